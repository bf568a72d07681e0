// TEST INFRASTRUCTURE — NOT PRODUCT CODE. CPU restatement of the training
// math of one batch (training.cpp, loss.hpp, mlp.hpp, encoding.hpp); see
// lsnif_train_oracle.cpp.
#pragma once

#include <cstdint>

#include "lsnif_oracle.hpp"

namespace oracle {

struct TrainTarget {  // TrainSample targets (training.hpp:15-22) == lsnif_train_target
  int32_t occluded = 0;
  float local_t = 0;
  float normal[3] = {0, 0, 1};
  float albedo[3] = {0, 0, 0};
  int32_t material = 0;
};
static_assert(sizeof(TrainTarget) == 36, "TrainTarget must match lsnif_train_target");

struct TrainMesh {  // Mesh (geometry.hpp:62-85) as flat arrays
  const float* verts;
  const float* normals;      // nullable
  const int* faces;
  const int* face_normals;   // nullable
  const int* face_material;
  int n_faces;
  const float* albedo;       // 3 per material
};

bool label_ray(const TrainMesh& mesh, const Aabb& frame, const Ray& ray, TrainTarget& out);
// loss[6] = total, bce, mae, cosine, rel_l2, ce (batch means); g_mlp = w1|b1|w2|b2|w3|b3
void train_batch_grad(const Model& m, const Ray* rays, const TrainTarget* targets, int64_t n, float loss[6],
                      float* g_mlp, float* g_tab);

}  // namespace oracle
