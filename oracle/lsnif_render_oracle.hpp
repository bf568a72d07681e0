// TEST INFRASTRUCTURE — NOT PRODUCT CODE. CPU restatement of render()
// (proj/src/renderer.cpp:330-542) for LSNIF-only scenes; see
// lsnif_render_oracle.cpp.
#pragma once

#include <cstdint>
#include <vector>

#include "lsnif_oracle.hpp"

namespace oracle {

struct RCamera {  // scene.hpp:12-17
  float position[3];
  float look_at[3];
  float up[3];
  float vfov_deg;
};

struct RLight {  // scene.hpp:19-26 (point = 0, sphere = 1)
  uint32_t type;
  float position[3];
  float radius;
  float radiance[3];
};

struct RenderSetup {  // RenderConfig (renderer.hpp:14-28) + PreparedScene state
  int width = 256, height = 256, spp = 16, max_bounces = 4;
  uint64_t seed = 0;
  float neural_eps_scale = 1e-3f;
  RCamera camera{};
  std::vector<RLight> lights;
  float environment[3] = {0, 0, 0};
  std::vector<float> world_diag;  // PreparedObject::world_diag per instance
};

// stats (nullable): [0] intersect_scene rays, [1] occluded_batch rays
void render(const RenderSetup& setup, const Instance* inst, int n_inst, float* image, int workers,
            int64_t* stats = nullptr);
void render_debug_paths(const RenderSetup& setup, int64_t first_path, int64_t n, Ray* rays, float* u, int k);

}  // namespace oracle
