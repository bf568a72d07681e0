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

    // run_narrow_phase over given pairs: every ray with its [t_enter, t_exit]
    std::vector<lsnif_interval> pairs(rays.size(), lsnif_interval{3.0f, 6.0f});
    const auto nh = lsnif::gpu::infer_pairs(model, rays, pairs);
    int occ = 0;
    for (const auto& h : nh) occ += h.occluded;
    std::printf("infer_pairs: %d of %zu pairs occluded\n", occ, nh.size());

    // render() of a one-instance scene (PrimaryMode::lsnif), 64x36 x 2 spp
    const lsnif::gpu::Scene scene({model}, {{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0}});
    const lsnif_camera cam{{0.25f, 1.6f, 4.5f}, {0.25f, 0.87f, 0.0f}, {0.0f, 1.0f, 0.0f}, 40.0f};
    const std::vector<lsnif_light> lights{{LSNIF_LIGHT_POINT, {3.0f, 4.0f, 3.0f}, 0.0f, {20.0f, 20.0f, 20.0f}}};
    const float env[3] = {0.05f, 0.05f, 0.08f};
    lsnif_render_config cfg{64, 36, 2, 4, 0, 1e-3f, 0};
    lsnif_render_stats st{};
    const std::vector<float> img = lsnif::gpu::render(scene, {3.7f}, cam, lights, env, cfg, &st);
    double mean = 0;
    for (float v : img) mean += v;
    std::printf("render 64x36x2: %lld closest + %lld shadow rays, mean radiance %.5f\n",
                static_cast<long long>(st.closest_rays), static_cast<long long>(st.shadow_rays),
                mean / static_cast<double>(img.size()));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
