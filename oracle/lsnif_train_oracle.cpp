// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU restatement of the reference's training math for one batch, used by
// tests/ as the checker of the GPU trainer (lsnif_trainer_*):
//   label_rays        label_ray (training.cpp:47-72) with the closest
//                     Moller-Trumbore hit over all faces (bvh.cpp:155-172,
//                     174-232: smallest t, ties to the lower face) and
//                     Mesh::shading_normal (geometry.cpp:58-67);
//   train_batch_grad  collect_boundary_hits + encode_ray_into (dda.cpp:119-124,
//                     encoding.hpp:166-176), forward_cached (mlp.hpp:117-130),
//                     composite_loss (loss.hpp:45-103) scaled by 1/batch
//                     (training.cpp:176-181), backward (mlp.hpp:188-225) and
//                     accumulate_grad_into (encoding.hpp:193-209).
// fp32 throughout, sequential sums (Eigen's GEMM order is library-internal:
// the GPU comparison is tolerance-based). Build with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "lsnif_oracle.hpp"
#include "lsnif_train_oracle.hpp"

namespace oracle {
namespace {

float dot3(const float* a, const float* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
void cross3(const float* a, const float* b, float* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

// bvh.cpp:155-172
bool intersect_triangle(const float* o, const float* d, float t_min, float t_max, const float* a, const float* b,
                        const float* c, float& t, float& u, float& v) {
  float e1[3], e2[3], p[3], s[3], q[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = b[k] - a[k];
    e2[k] = c[k] - a[k];
  }
  cross3(d, e2, p);
  const float det = dot3(e1, p);
  if (std::abs(det) < 1e-9f) return false;
  const float inv_det = 1.0f / det;
  for (int k = 0; k < 3; ++k) s[k] = o[k] - a[k];
  u = dot3(s, p) * inv_det;
  if (u < 0.0f || u > 1.0f) return false;
  cross3(s, e1, q);
  v = dot3(d, q) * inv_det;
  if (v < 0.0f || u + v > 1.0f) return false;
  t = dot3(e2, q) * inv_det;
  return !(t < t_min || t > t_max);
}

// intersect_closest over every face (the BVH only prunes; the winner is the
// smallest t with ties to the lower face index)
bool closest(const TrainMesh& M, const float* o, const float* d, float& t, float& u, float& v, int& face) {
  bool found = false;
  float best = std::numeric_limits<float>::infinity();
  for (int f = 0; f < M.n_faces; ++f) {
    const float* a = M.verts + 3 * M.faces[3 * f];
    const float* b = M.verts + 3 * M.faces[3 * f + 1];
    const float* c = M.verts + 3 * M.faces[3 * f + 2];
    float th, uh, vh;
    if (!intersect_triangle(o, d, 0.0f, std::numeric_limits<float>::infinity(), a, b, c, th, uh, vh)) continue;
    if (th < best || (th == best && !found)) {
      best = th;
      t = th;
      u = uh;
      v = vh;
      face = f;
      found = true;
    }
  }
  return found;
}

// geometry.cpp:35-43, 58-67
void shading_normal(const TrainMesh& M, int face, float u, float v, float* n) {
  if (M.normals && M.face_normals) {
    const float* n0 = M.normals + 3 * M.face_normals[3 * face];
    const float* n1 = M.normals + 3 * M.face_normals[3 * face + 1];
    const float* n2 = M.normals + 3 * M.face_normals[3 * face + 2];
    const float w0 = 1.0f - u - v;
    for (int a = 0; a < 3; ++a) n[a] = w0 * n0[a] + u * n1[a] + v * n2[a];
    const float len = std::sqrt(dot3(n, n));
    if (len > 1e-12f) {
      for (int a = 0; a < 3; ++a) n[a] = n[a] / len;
      return;
    }
  }
  const float* p0 = M.verts + 3 * M.faces[3 * face];
  const float* p1 = M.verts + 3 * M.faces[3 * face + 1];
  const float* p2 = M.verts + 3 * M.faces[3 * face + 2];
  float e0[3], e1[3];
  for (int a = 0; a < 3; ++a) {
    e0[a] = p1[a] - p0[a];
    e1[a] = p2[a] - p0[a];
  }
  cross3(e0, e1, n);
  const float len = std::sqrt(dot3(n, n));
  for (int a = 0; a < 3; ++a) n[a] = len > 0.0f ? n[a] / len : 0.0f;
}

float sigmoid(float v) { return 1.0f / (1.0f + std::exp(-v)); }

}  // namespace

// label_ray (training.cpp:47-72); returns false when the ray misses the box
bool label_ray(const TrainMesh& M, const Aabb& frame, const Ray& ray, TrainTarget& tg) {
  Ray r = ray;
  r.t_max = std::numeric_limits<float>::infinity();
  Interval iv;
  if (!ray_aabb_intersect(r, frame, &iv)) return false;
  float t = 0, u = 0, v = 0;
  int face = -1;
  const bool hit = closest(M, ray.o, ray.d, t, u, v, face);
  tg = TrainTarget{};
  tg.occluded = hit && t <= iv.exit;
  if (tg.occluded) {
    const float span = std::max(iv.exit - iv.enter, 1e-12f);
    tg.local_t = std::clamp((t - iv.enter) / span, 0.0f, 1.0f);
    float n[3];
    shading_normal(M, face, u, v, n);
    if (dot3(n, ray.d) > 0.0f)
      for (int a = 0; a < 3; ++a) n[a] = -n[a];
    const int mat = M.face_material[face];
    for (int a = 0; a < 3; ++a) {
      tg.normal[a] = n[a];
      tg.albedo[a] = M.albedo[3 * mat + a];
    }
    tg.material = mat;
  } else {
    tg.normal[2] = 1.0f;
  }
  return true;
}

void train_batch_grad(const Model& m, const Ray* rays, const TrainTarget* tg, int64_t n, float loss[6],
                      float* g_mlp, float* g_tab) {
  const int K1 = m.input_width(), hid = m.hidden, n_out = m.output_width(), n_mat = m.n_mat;
  const int L = m.n_levels, F = m.f_dim, H = m.hit_cap;
  const float inv_batch = 1.0f / static_cast<float>(n);
  // gradient layout: w1 | b1 | w2 | b2 | w3 | b3 (row-major), tables level-major
  const size_t o_w1 = 0, o_b1 = o_w1 + static_cast<size_t>(hid) * K1, o_w2 = o_b1 + hid,
               o_b2 = o_w2 + static_cast<size_t>(hid) * hid, o_w3 = o_b2 + hid,
               o_b3 = o_w3 + static_cast<size_t>(n_out) * hid, n_mlp = o_b3 + n_out;
  std::fill(g_mlp, g_mlp + n_mlp, 0.0f);
  std::fill(g_tab, g_tab + static_cast<size_t>(L) * m.table_size * F, 0.0f);
  for (int q = 0; q < 6; ++q) loss[q] = 0.0f;
  float inv_ext[3], o_local[3], d_local[3];
  for (int a = 0; a < 3; ++a) inv_ext[a] = 1.0f / (m.aabb.mx[a] - m.aabb.mn[a]);
  BoundaryHits hits;
  std::vector<float> x(K1), z1(hid), h1(hid), z2(hid), h2(hid), z3(n_out), p(n_out), dp(n_out), dz3(n_out),
      dh2(hid), dz2(hid), dh1(hid), dz1(hid), dx(K1);
  std::vector<PointCode> codes(static_cast<size_t>(H) * L);
  for (int64_t j = 0; j < n; ++j) {
    const Ray& r = rays[j];
    // collect_boundary_hits (dda.cpp:119-124) in the model frame
    for (int a = 0; a < 3; ++a) {
      o_local[a] = (r.o[a] - m.aabb.mn[a]) * inv_ext[a];
      d_local[a] = r.d[a] * inv_ext[a];
    }
    collect_boundary_hits_local(o_local, d_local, r.t_min, r.t_max, m.occupancy, m.voxel_res, H, hits);
    int npts = 0;
    encode_ray_into(m, hits, x.data(), codes.data(), npts);
    // forward_cached (mlp.hpp:117-130)
    for (int i = 0; i < hid; ++i) {
      float s = 0.0f;
      for (int k = 0; k < K1; ++k) s += m.w1[static_cast<size_t>(i) * K1 + k] * x[k];
      z1[i] = s + m.b1[i];
      h1[i] = z1[i] > 0.0f ? z1[i] : 0.01f * z1[i];
    }
    for (int i = 0; i < hid; ++i) {
      float s = 0.0f;
      for (int k = 0; k < hid; ++k) s += m.w2[static_cast<size_t>(i) * hid + k] * h1[k];
      z2[i] = s + m.b2[i];
      h2[i] = z2[i] > 0.0f ? z2[i] : 0.01f * z2[i];
    }
    for (int i = 0; i < n_out; ++i) {
      float s = 0.0f;
      for (int k = 0; k < hid; ++k) s += m.w3[static_cast<size_t>(i) * hid + k] * h2[k];
      z3[i] = s + m.b3[i];
    }
    // apply_heads (mlp.hpp:80-94)
    p[0] = sigmoid(z3[0]);
    p[1] = sigmoid(z3[1]);
    for (int k = 2; k < 5; ++k) p[k] = z3[k];
    for (int k = 5; k < 8; ++k) p[k] = sigmoid(z3[k]);
    float zmax = z3[8];
    for (int k = 1; k < n_mat; ++k) zmax = std::max(zmax, z3[8 + k]);
    float esum = 0.0f;
    std::vector<float> e(n_mat);
    for (int k = 0; k < n_mat; ++k) {
      e[k] = std::exp(z3[8 + k] - zmax);
      esum += e[k];
    }
    for (int k = 0; k < n_mat; ++k) p[8 + k] = e[k] / esum;
    // composite_loss (loss.hpp:45-103)
    float terms[6] = {0, 0, 0, 0, 0, 0};
    std::fill(dp.begin(), dp.end(), 0.0f);
    const TrainTarget& t = tg[j];
    {
      const float y = t.occluded ? 1.0f : 0.0f;
      const float prob = std::clamp(p[0], 1e-7f, 1.0f - 1e-7f);
      terms[1] = -(y * std::log(prob) + (1.0f - y) * std::log(1.0f - prob));
      dp[0] = (prob - y) / (prob * (1.0f - prob));
    }
    if (t.occluded) {
      const float diff = p[1] - t.local_t;
      terms[2] = std::abs(diff);
      dp[1] = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
      float tn[3] = {t.normal[0], t.normal[1], t.normal[2]};
      const float tl2 = dot3(tn, tn);
      if (tl2 > 0.0f)
        for (int a = 0; a < 3; ++a) tn[a] = tn[a] / std::sqrt(tl2);
      const float nv[3] = {p[2], p[3], p[4]};
      const float len = std::max(std::sqrt(dot3(nv, nv)), 1e-12f);
      const float ndt = dot3(nv, tn);
      terms[3] = 1.0f - ndt / len;
      for (int a = 0; a < 3; ++a) dp[2 + a] = -(tn[a] / len - (ndt / (len * len * len)) * nv[a]);
      for (int c = 0; c < 3; ++c) {
        const float a = p[5 + c], tt = t.albedo[c];
        const float denom = a * a + 1e-2f;
        const float diff2 = a - tt;
        terms[4] += diff2 * diff2 / denom;
        dp[5 + c] = (2.0f * diff2 * denom - diff2 * diff2 * 2.0f * a) / (denom * denom);
      }
      const float prob = std::clamp(p[8 + t.material], 1e-7f, 1.0f);
      terms[5] = -std::log(prob);
      dp[8 + t.material] = -1.0f / prob;
    }
    terms[0] = terms[1] + terms[2] + terms[3] + terms[4] + terms[5];
    for (int q = 0; q < 6; ++q) loss[q] += terms[q] * inv_batch;
    for (int r2 = 0; r2 < n_out; ++r2) dp[r2] = dp[r2] * inv_batch;
    // backward (mlp.hpp:188-225)
    for (int r2 : {0, 1, 5, 6, 7}) {
      const float pc = std::clamp(p[r2], 1e-7f, 1.0f - 1e-7f);
      dz3[r2] = dp[r2] * pc * (1.0f - pc);
    }
    for (int k = 0; k < 3; ++k) dz3[2 + k] = dp[2 + k];
    float dot = 0.0f;
    for (int k = 0; k < n_mat; ++k) dot += p[8 + k] * dp[8 + k];
    for (int k = 0; k < n_mat; ++k) dz3[8 + k] = p[8 + k] * (dp[8 + k] - dot);
    for (int i = 0; i < n_out; ++i) {
      for (int k = 0; k < hid; ++k) g_mlp[o_w3 + static_cast<size_t>(i) * hid + k] += dz3[i] * h2[k];
      g_mlp[o_b3 + i] += dz3[i];
    }
    for (int k = 0; k < hid; ++k) {
      float s = 0.0f;
      for (int i = 0; i < n_out; ++i) s += m.w3[static_cast<size_t>(i) * hid + k] * dz3[i];
      dh2[k] = s;
      dz2[k] = s * (z2[k] > 0.0f ? 1.0f : 0.01f);
    }
    for (int i = 0; i < hid; ++i) {
      for (int k = 0; k < hid; ++k) g_mlp[o_w2 + static_cast<size_t>(i) * hid + k] += dz2[i] * h1[k];
      g_mlp[o_b2 + i] += dz2[i];
    }
    for (int k = 0; k < hid; ++k) {
      float s = 0.0f;
      for (int i = 0; i < hid; ++i) s += m.w2[static_cast<size_t>(i) * hid + k] * dz2[i];
      dh1[k] = s;
      dz1[k] = s * (z1[k] > 0.0f ? 1.0f : 0.01f);
    }
    for (int i = 0; i < hid; ++i) {
      for (int k = 0; k < K1; ++k) g_mlp[o_w1 + static_cast<size_t>(i) * K1 + k] += dz1[i] * x[k];
      g_mlp[o_b1 + i] += dz1[i];
    }
    for (int k = 0; k < K1; ++k) {
      float s = 0.0f;
      for (int i = 0; i < hid; ++i) s += m.w1[static_cast<size_t>(i) * K1 + k] * dz1[i];
      dx[k] = s;
    }
    // accumulate_grad_into (encoding.hpp:193-209)
    for (int i = 0; i < npts; ++i)
      for (int l = 0; l < L; ++l) {
        const PointCode& c = codes[static_cast<size_t>(i) * L + l];
        float* g = g_tab + static_cast<size_t>(l) * m.table_size * F;
        const float* up = dx.data() + (i * L + l) * F;
        for (int k = 0; k < c.count; ++k)
          for (int f = 0; f < F; ++f) g[static_cast<size_t>(c.index[k]) * F + f] += c.weight[k] * up[f];
      }
  }
}

}  // namespace oracle
