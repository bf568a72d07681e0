// Example C++ caller of the drop-in API (include/lsnif_gpu.hpp): loads a
// model, answers a row of camera-like rays with the closest-hit rule and
// prints the accepted hits. Build: make examples/query_cpp
#include <cstdio>
#include <vector>

#include "lsnif_gpu.hpp"

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "tests/golden/teapot_seed0.lsnif";
  try {
    const lsnif::gpu::Model model = lsnif::gpu::Model::load(path, 0);
    std::vector<lsnif_ray> rays;
    for (int i = 0; i < 64; ++i) {
      lsnif_ray r{{0.25f, 0.9f, 4.5f}, {(i - 32) * 0.005f, -0.05f, -1.0f}, 0.0f, 1e30f};
      rays.push_back(r);
    }
    const auto hits = lsnif::gpu::intersect(model, rays);
    int n = 0;
    for (const auto& h : hits) n += h.has_value();
    std::printf("%d of %zu rays accepted a neural hit\n", n, rays.size());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
