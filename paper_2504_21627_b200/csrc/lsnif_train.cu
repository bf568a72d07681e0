// GPU training of an LSNIF model: lsnif::train
// (proj/src/training.cpp:95-230) as one device-resident step per call.
//
// Per step, for a batch of B samples (fp32 throughout, like the reference):
//   sample_kernel    draw_sample (training.cpp:74-93): external / surface rays
//                    (sample_external_ray 21-30, sample_surface_ray 32-45)
//                    labelled by label_ray (47-72) against the mesh: closest
//                    Moller-Trumbore hit over all triangles (bvh.cpp:155-172;
//                    equal t resolved to the lower face like intersect_closest),
//                    shading normal (geometry.cpp:58-67);
//   encode_kernel    collect_boundary_hits + encode_ray_into with the current
//                    fp32 tables (dda.cpp:119-124, encoding.hpp:166-176), the
//                    same walk / corner functions as the query kernels, and the
//                    point codes (hash index + weight per corner) for backward;
//   cuBLAS SGEMMs    z1 = W1 x, z2 = W2 h1, z3 = W3 h2 and the backward GEMMs
//                    (plain library GEMMs; forward_cached, backward: mlp.hpp);
//   heads_loss_kernel apply_heads + composite_loss (loss.hpp:45-103) + dz3;
//   scatter_kernel   accumulate_grad_into (encoding.hpp:193-209), atomics;
//   adam_kernel      adam_update_tensor (mlp.hpp:243-256) over MLP and tables.
// Random numbers come from per-sample counter streams (splitmix64), not the
// reference's per-worker mt19937 stream, whose retry loops make it serial.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "lsnif_gpu.h"
#include "lsnif_internal.hpp"

namespace lsnif_tr {

using lsnif_api::ck;
using lsnif_api::fail;
using lsnif_dev::DevModel;

constexpr float kPi = 3.14159265358979323846f;
constexpr float kLeakySlope = 0.01f;   // mlp.hpp:15
constexpr float kProbClamp = 1e-7f;    // loss.hpp:39
constexpr float kRelL2Stabilizer = 1e-2f;
constexpr int kSurfaceRetries = 64;    // training.cpp:12
constexpr int kExternalRetries = 4096; // the reference loops until the ray meets the box

// ------------------------------------------------------------- mesh + rng

struct MeshDev {
  const float4* tri;     // 3 per face: the corner positions (w unused), gathered once
  const float* v;        // 3 per vertex
  const float* n;        // 3 per normal (nullable)
  const int* f;          // 3 per face
  const int* fn;         // 3 per face (nullable)
  const int* fmat;       // per face
  int nf;
  const float* albedo;   // 3 per material
  int n_mats;
};

struct Rng {  // splitmix64 counter stream
  uint64_t s;
  __device__ float uniform() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return static_cast<float>(z >> 40) * 5.9604644775390625e-8f;  // [0, 1), 24 bits
  }
};

__device__ __forceinline__ float dot3(const float a[3], const float b[3]) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a[0], b[0]), __fmul_rn(a[1], b[1])), __fmul_rn(a[2], b[2]));
}
__device__ __forceinline__ void cross3(const float a[3], const float b[3], float o[3]) {
  o[0] = __fsub_rn(__fmul_rn(a[1], b[2]), __fmul_rn(a[2], b[1]));
  o[1] = __fsub_rn(__fmul_rn(a[2], b[0]), __fmul_rn(a[0], b[2]));
  o[2] = __fsub_rn(__fmul_rn(a[0], b[1]), __fmul_rn(a[1], b[0]));
}
__device__ __forceinline__ void normalize3(float v[3]) {
  const float n2 = dot3(v, v);
  if (n2 > 0.0f) {
    const float n = __fsqrt_rn(n2);
    for (int a = 0; a < 3; ++a) v[a] = __fdiv_rn(v[a], n);
  }
}

// sampling.hpp:18-46
__device__ void orthonormal_basis(const float n[3], float t[3], float b[3]) {
  const float sign = copysignf(1.0f, n[2]);
  const float a = __fdiv_rn(-1.0f, __fadd_rn(sign, n[2]));
  const float bb = __fmul_rn(__fmul_rn(n[0], n[1]), a);
  t[0] = __fadd_rn(1.0f, __fmul_rn(__fmul_rn(__fmul_rn(sign, n[0]), n[0]), a));
  t[1] = __fmul_rn(sign, bb);
  t[2] = -__fmul_rn(sign, n[0]);
  b[0] = bb;
  b[1] = __fadd_rn(sign, __fmul_rn(__fmul_rn(n[1], n[1]), a));
  b[2] = -n[1];
}
__device__ void uniform_sphere_dir(Rng& rng, float out[3]) {
  const float z = __fsub_rn(1.0f, __fmul_rn(2.0f, rng.uniform()));
  const float r = __fsqrt_rn(fmaxf(0.0f, __fsub_rn(1.0f, __fmul_rn(z, z))));
  const float phi = __fmul_rn(__fmul_rn(2.0f, kPi), rng.uniform());
  out[0] = __fmul_rn(r, cosf(phi));
  out[1] = __fmul_rn(r, sinf(phi));
  out[2] = z;
}
__device__ void cosine_hemisphere_dir(const float axis[3], Rng& rng, float out[3]) {
  const float u1 = rng.uniform();
  const float u2 = rng.uniform();
  const float r = __fsqrt_rn(u1);
  const float phi = __fmul_rn(__fmul_rn(2.0f, kPi), u2);
  const float x = __fmul_rn(r, cosf(phi)), y = __fmul_rn(r, sinf(phi));
  const float z = __fsqrt_rn(fmaxf(0.0f, __fsub_rn(1.0f, u1)));
  float t[3], b[3];
  orthonormal_basis(axis, t, b);
  for (int a = 0; a < 3; ++a) out[a] = __fadd_rn(__fadd_rn(__fmul_rn(x, t[a]), __fmul_rn(y, b[a])), __fmul_rn(z, axis[a]));
  normalize3(out);
}

// intersect_triangle (bvh.cpp:155-172)
__device__ __forceinline__ bool intersect_triangle(const float o[3], const float d[3], float t_min, float t_max,
                                                   const float a[3], const float b[3], const float c[3], float& t,
                                                   float& u, float& v) {
  float e1[3], e2[3], p[3], s[3], q[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = __fsub_rn(b[k], a[k]);
    e2[k] = __fsub_rn(c[k], a[k]);
  }
  cross3(d, e2, p);
  const float det = dot3(e1, p);
  if (fabsf(det) < 1e-9f) return false;
  const float inv_det = __fdiv_rn(1.0f, det);
  for (int k = 0; k < 3; ++k) s[k] = __fsub_rn(o[k], a[k]);
  u = __fmul_rn(dot3(s, p), inv_det);
  if (u < 0.0f || u > 1.0f) return false;
  cross3(s, e1, q);
  v = __fmul_rn(dot3(d, q), inv_det);
  if (v < 0.0f || __fadd_rn(u, v) > 1.0f) return false;
  t = __fmul_rn(dot3(e2, q), inv_det);
  return !(t < t_min || t > t_max);
}

// intersect_closest (bvh.cpp:174-232) over every face: smallest t, ties to
// the lower face index (a hit at exactly t_max is kept, like the reference).
// Warp-cooperative: the 32 lanes (which all hold the same ray) test faces
// lane, lane + 32, ... in increasing order, then reduce (t, face)
// lexicographically — the same winner as the sequential scan.
__device__ bool closest_hit(const MeshDev& M, const float o[3], const float d[3], float t_min, float t_max,
                            float& t, float& u, float& v, int& face) {
  const int lane = threadIdx.x & 31;
  float bt = __int_as_float(0x7f800000), bu = 0.0f, bv = 0.0f;
  int bf = 0x7fffffff;
  for (int f = lane; f < M.nf; f += 32) {
    const float4 A = __ldg(M.tri + 3 * f), B = __ldg(M.tri + 3 * f + 1), Cc = __ldg(M.tri + 3 * f + 2);
    const float a[3] = {A.x, A.y, A.z}, b[3] = {B.x, B.y, B.z}, c[3] = {Cc.x, Cc.y, Cc.z};
    float th, uh, vh;
    if (!intersect_triangle(o, d, t_min, t_max, a, b, c, th, uh, vh)) continue;
    if (th < bt || bf == 0x7fffffff) {  // first hit of this lane, or strictly closer
      bt = th;
      bu = uh;
      bv = vh;
      bf = f;
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const float ot = __shfl_xor_sync(0xffffffffu, bt, off);
    const int of = __shfl_xor_sync(0xffffffffu, bf, off);
    const float ou = __shfl_xor_sync(0xffffffffu, bu, off);
    const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
    if (ot < bt || (ot == bt && of < bf)) {
      bt = ot;
      bf = of;
      bu = ou;
      bv = ov;
    }
  }
  if (bf == 0x7fffffff) return false;
  t = bt;
  u = bu;
  v = bv;
  face = bf;
  return true;
}

// Mesh::shading_normal (geometry.cpp:58-67) / geometric_normal (35-43)
__device__ void shading_normal(const MeshDev& M, int face, float u, float v, float n[3]) {
  if (M.n && M.fn) {
    const int j0 = M.fn[3 * face], j1 = M.fn[3 * face + 1], j2 = M.fn[3 * face + 2];
    const float w0 = __fsub_rn(__fsub_rn(1.0f, u), v);
    for (int a = 0; a < 3; ++a)
      n[a] = __fadd_rn(__fadd_rn(__fmul_rn(w0, M.n[3 * j0 + a]), __fmul_rn(u, M.n[3 * j1 + a])),
                       __fmul_rn(v, M.n[3 * j2 + a]));
    const float len = __fsqrt_rn(dot3(n, n));
    if (len > 1e-12f) {
      for (int a = 0; a < 3; ++a) n[a] = __fdiv_rn(n[a], len);
      return;
    }
  }
  const int i0 = M.f[3 * face], i1 = M.f[3 * face + 1], i2 = M.f[3 * face + 2];
  float e0[3], e1[3];
  for (int a = 0; a < 3; ++a) {
    e0[a] = __fsub_rn(M.v[3 * i1 + a], M.v[3 * i0 + a]);
    e1[a] = __fsub_rn(M.v[3 * i2 + a], M.v[3 * i0 + a]);
  }
  cross3(e0, e1, n);
  const float len = __fsqrt_rn(dot3(n, n));
  if (len > 0.0f)
    for (int a = 0; a < 3; ++a) n[a] = __fdiv_rn(n[a], len);
  else
    n[0] = n[1] = n[2] = 0.0f;
}

struct Frame {  // the model's (inflated) frame box
  float mn[3], mx[3];
  float center[3], radius, eps;
};

// sample_external_ray (training.cpp:21-30)
__device__ void external_ray(const Frame& fr, Rng& rng, float o[3], float d[3]) {
  float s[3];
  uniform_sphere_dir(rng, s);
  for (int a = 0; a < 3; ++a) o[a] = __fadd_rn(fr.center[a], __fmul_rn(fr.radius, s[a]));
  float toward[3];
  for (int a = 0; a < 3; ++a) toward[a] = __fsub_rn(fr.center[a], o[a]);
  normalize3(toward);
  cosine_hemisphere_dir(toward, rng, d);
}

// ray_aabb_intersect (geometry.cpp:9-28) with t_max = inf
__device__ bool box_interval(const Frame& fr, const float o[3], const float d[3], float& enter, float& exit) {
  float t0 = 0.0f, t1 = __int_as_float(0x7f800000);
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0f) {
      if (o[a] < fr.mn[a] || o[a] > fr.mx[a]) return false;
      continue;
    }
    const float inv = __frcp_rn(d[a]);
    float ta = __fmul_rn(__fsub_rn(fr.mn[a], o[a]), inv), tb = __fmul_rn(__fsub_rn(fr.mx[a], o[a]), inv);
    if (ta > tb) {
      const float x = ta;
      ta = tb;
      tb = x;
    }
    t0 = t0 < ta ? ta : t0;
    t1 = tb < t1 ? tb : t1;
    if (t0 > t1) return false;
  }
  enter = t0;
  exit = t1;
  return true;
}

// label_ray (training.cpp:47-72)
__device__ bool label_ray(const MeshDev& M, const Frame& fr, const float o[3], const float d[3],
                          lsnif_train_target& tg) {
  float enter, exit;
  if (!box_interval(fr, o, d, enter, exit)) return false;
  float t, u, v;
  int face;
  const bool hit = closest_hit(M, o, d, 0.0f, __int_as_float(0x7f800000), t, u, v, face);
  tg.occluded = hit && t <= exit;
  if (tg.occluded) {
    const float span = fmaxf(__fsub_rn(exit, enter), 1e-12f);
    tg.local_t = fminf(fmaxf(__fdiv_rn(__fsub_rn(t, enter), span), 0.0f), 1.0f);
    float n[3];
    shading_normal(M, face, u, v, n);
    if (dot3(n, d) > 0.0f)
      for (int a = 0; a < 3; ++a) n[a] = -n[a];
    const int mat = M.fmat[face];
    for (int a = 0; a < 3; ++a) {
      tg.normal[a] = n[a];
      tg.albedo[a] = M.albedo[3 * mat + a];
    }
    tg.material = mat;
  } else {
    tg.local_t = 0.0f;
    tg.normal[0] = tg.normal[1] = 0.0f;
    tg.normal[2] = 1.0f;
    tg.albedo[0] = tg.albedo[1] = tg.albedo[2] = 0.0f;
    tg.material = 0;
  }
  return true;
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finalizer (types.hpp:25-31)
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t sample_seed(uint64_t seed, uint64_t step, uint64_t j) {
  return mix64(mix64(mix64(seed + 0x7e1ull) ^ step) ^ j);
}

// draw_sample (training.cpp:74-93)
// One warp per sample: every lane draws the same stream and takes the same
// path; the triangle scans are split over the lanes (closest_hit).
__global__ void __launch_bounds__(128) sample_kernel(MeshDev M, Frame fr, uint64_t seed, int64_t step,
                                                     float external_mix, int64_t n, lsnif_ray* rays,
                                                     lsnif_train_target* targets) {
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (j >= n) return;  // warp-uniform
  Rng rng{sample_seed(seed, static_cast<uint64_t>(step), static_cast<uint64_t>(j))};
  lsnif_train_target tg{};
  float o[3], d[3];
  bool ok = false;
  if (!(rng.uniform() < external_mix)) {
    for (int attempt = 0; attempt < kSurfaceRetries && !ok; ++attempt) {
      float po[3], pd[3];
      external_ray(fr, rng, po, pd);
      float t, u, v;
      int face;
      if (!closest_hit(M, po, pd, 0.0f, __int_as_float(0x7f800000), t, u, v, face)) continue;
      float nrm[3];
      shading_normal(M, face, u, v, nrm);
      if (dot3(nrm, pd) > 0.0f)
        for (int a = 0; a < 3; ++a) nrm[a] = -nrm[a];
      for (int a = 0; a < 3; ++a)  // probe.at(t) + eps * normal
        o[a] = __fadd_rn(__fadd_rn(po[a], __fmul_rn(t, pd[a])), __fmul_rn(fr.eps, nrm[a]));
      cosine_hemisphere_dir(nrm, rng, d);
      ok = label_ray(M, fr, o, d, tg);
    }
  }
  for (int attempt = 0; attempt < kExternalRetries && !ok; ++attempt) {
    external_ray(fr, rng, o, d);
    ok = label_ray(M, fr, o, d, tg);
  }
  lsnif_ray r;
  for (int a = 0; a < 3; ++a) {
    r.origin[a] = o[a];
    r.direction[a] = d[a];
  }
  r.t_min = 0.0f;
  r.t_max = __int_as_float(0x7f800000);
  if ((threadIdx.x & 31) == 0) {
    rays[j] = r;
    targets[j] = tg;
  }
}

// ------------------------------------------------------------- encode

// collect_boundary_hits + encode_ray_into (dda.cpp:40-124, encoding.hpp:84-176)
// with fp32 tables, one thread per sample; X column j = the sample's input
// (K1 values, zero padded), codes = (index, weight) of every corner used.
__global__ void __launch_bounds__(128) encode_kernel(const DevModel m, const float* __restrict__ tables,
                                                     const lsnif_ray* __restrict__ rays, int64_t n, float* X,
                                                     uint32_t* cidx, float* cw, int8_t* ccount) {
  extern __shared__ uint32_t stop[];
  for (int i = threadIdx.x; i < m.stop_words; i += blockDim.x) stop[i] = __ldg(m.stop + i);
  __syncthreads();
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int H = m.H, L = m.L, F = m.F, LF = L * F, K1 = m.K1;
  const lsnif_ray r = rays[j];
  float* x = X + j * K1;
  for (int k = 0; k < K1; ++k) x[k] = 0.0f;
  uint2 pool[lsnif_dev::kMaxHitCap];
  int count = 0;
  lsnif_dev::Walk w;
  if (lsnif_dev::walk_setup<0>(m, r.origin, r.direction, r.t_min, w)) {
    if (lsnif_dev::stop_bit(stop, w.idx)) pool[count++] = lsnif_dev::pack_point(w.t0, w.axis0, w.plane0);
    float tn;
    bool p1, p2;
    while (count < H && lsnif_dev::walk_step(w, tn, p1, p2)) {
      if (!lsnif_dev::stop_bit(stop, w.idx)) continue;
      int c[3];
      lsnif_dev::walk_cell<0>(m, w.idx, c);
      const int axis = p2 ? 2 : (p1 ? 1 : 0);
      const int ca = axis == 0 ? c[0] : axis == 1 ? c[1] : c[2];
      if (ca < 0 || ca >= m.V) break;  // left the grid (dda.cpp:112)
      const float da = axis == 0 ? w.d[0] : axis == 1 ? w.d[1] : w.d[2];
      pool[count++] = lsnif_dev::pack_point(tn, axis, static_cast<float>(da > 0.0f ? ca : ca + 1));
    }
  }
  for (int k = 0; k < H; ++k)
    for (int l = 0; l < L; ++l) ccount[(j * H + k) * L + l] = 0;
  for (int k = 0; k < count; ++k) {
    float p[3];
    bool volume;
    lsnif_dev::unpack_point(pool[k], w.o, w.d, m.inv_fres, p, volume);
    const int pa = volume ? -1 : lsnif_dev::plane_axis_of(p, m.fres);
    for (int l = 0; l < L; ++l) {
      const float* T = tables + static_cast<size_t>(l) * m.M * F;
      const int64_t cb = ((j * H + k) * L + l) * 8;
      uint32_t idx[8];
      float wt[8];
      int nc = 4;
      if (!volume) {
        lsnif_dev::boundary_corners<false>(m, l, p, pa, idx, wt);
      } else {  // encode_point_level with plane_axis = -1: 8 trilinear corners
        nc = 8;
        const int res = m.level_res[l];
        const float fres = static_cast<float>(res);
        int base[3];
        float frac[3];
        for (int a = 0; a < 3; ++a) {
          const float u = __fmul_rn(p[a], fres);
          base[a] = lsnif_dev::iclamp(static_cast<int>(floorf(u)), 0, res - 1);
          frac[a] = lsnif_dev::fclamp(__fsub_rn(u, static_cast<float>(base[a])), 0.0f, 1.0f);
        }
        for (int corner = 0; corner < 8; ++corner) {
          const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
          const float wx = dx ? frac[0] : __fsub_rn(1.0f, frac[0]);
          const float wy = dy ? frac[1] : __fsub_rn(1.0f, frac[1]);
          const float wz = dz ? frac[2] : __fsub_rn(1.0f, frac[2]);
          wt[corner] = __fmul_rn(__fmul_rn(wx, wy), wz);
          const uint32_t h = static_cast<uint32_t>(base[0] + dx) ^ static_cast<uint32_t>(base[1] + dy) * lsnif_dev::kP1 ^
                             static_cast<uint32_t>(base[2] + dz) * lsnif_dev::kP2;
          idx[corner] = lsnif_dev::hash_reduce<false>(m, h);
        }
      }
      float feat[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int c = 0; c < nc; ++c) {
        for (int f = 0; f < F; ++f) feat[f] = __fadd_rn(feat[f], __fmul_rn(wt[c], __ldg(T + static_cast<size_t>(idx[c]) * F + f)));
        cidx[cb + c] = idx[c];
        cw[cb + c] = wt[c];
      }
      ccount[(j * H + k) * L + l] = static_cast<int8_t>(nc);
      for (int f = 0; f < F; ++f) x[k * LF + l * F + f] = feat[f];
    }
  }
}

// ------------------------------------------------------------- MLP pieces

// z += b (per row), h = leaky(z): columns are samples (rows x n, col-major)
__global__ void bias_leaky_kernel(float* z, float* h, const float* b, int rows, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * n) return;
  const float v = __fadd_rn(z[i], b[i % rows]);
  z[i] = v;
  h[i] = v > 0.0f ? v : __fmul_rn(kLeakySlope, v);
}

// dz = dh * leaky'(z)
__global__ void leaky_back_kernel(const float* dh, const float* z, float* dz, int64_t total) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  dz[i] = __fmul_rn(dh[i], z[i] > 0.0f ? 1.0f : kLeakySlope);
}

// grad_b[r] = sum over samples of dz[r, j]
__global__ void rowsum_kernel(const float* dz, int rows, int64_t n, float* out) {
  const int r = blockIdx.x;
  float acc = 0.0f;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) acc += dz[j * rows + r];
  __shared__ float red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = red[0];
}

__device__ __forceinline__ float sig(float v) { return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-v))); }

// apply_heads (mlp.hpp:80-94) + composite_loss (loss.hpp:45-103, terms and dp
// scaled by 1/batch) + the head part of backward (mlp.hpp:188-204): dz3.
__global__ void heads_loss_kernel(const float* z3raw, const float* b3, int n_out, int n_mat, int64_t n,
                                  const lsnif_train_target* targets, float inv_batch, float* dz3, float* loss6) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  float terms[6] = {0, 0, 0, 0, 0, 0};  // total, bce, mae, cos, rel, ce
  if (j < n) {
    float z[16], p[16], dp[16];
    for (int r = 0; r < n_out; ++r) {
      z[r] = __fadd_rn(z3raw[j * n_out + r], b3[r]);
      dp[r] = 0.0f;
    }
    p[0] = sig(z[0]);
    p[1] = sig(z[1]);
    p[2] = z[2];
    p[3] = z[3];
    p[4] = z[4];
    for (int k = 0; k < 3; ++k) p[5 + k] = sig(z[5 + k]);
    float zmax = z[8];
    for (int k = 1; k < n_mat; ++k) zmax = z[8 + k] > zmax ? z[8 + k] : zmax;
    float e[8], esum = 0.0f;
    for (int k = 0; k < n_mat; ++k) {
      e[k] = expf(__fsub_rn(z[8 + k], zmax));
      esum = __fadd_rn(esum, e[k]);
    }
    for (int k = 0; k < n_mat; ++k) p[8 + k] = __fdiv_rn(e[k], esum);
    const lsnif_train_target tg = targets[j];
    {  // occlusion BCE
      const float y = tg.occluded ? 1.0f : 0.0f;
      const float prob = fminf(fmaxf(p[0], kProbClamp), __fsub_rn(1.0f, kProbClamp));
      terms[1] = -__fadd_rn(__fmul_rn(y, logf(prob)), __fmul_rn(__fsub_rn(1.0f, y), logf(__fsub_rn(1.0f, prob))));
      dp[0] = __fdiv_rn(__fsub_rn(prob, y), __fmul_rn(prob, __fsub_rn(1.0f, prob)));
    }
    if (tg.occluded) {
      const float diff = __fsub_rn(p[1], tg.local_t);
      terms[2] = fabsf(diff);
      dp[1] = diff > 0.0f ? 1.0f : (diff < 0.0f ? -1.0f : 0.0f);
      float t[3] = {tg.normal[0], tg.normal[1], tg.normal[2]};
      normalize3(t);
      const float nv[3] = {p[2], p[3], p[4]};
      const float len = fmaxf(__fsqrt_rn(dot3(nv, nv)), 1e-12f);
      const float ndt = dot3(nv, t);
      terms[3] = __fsub_rn(1.0f, __fdiv_rn(ndt, len));
      const float k3 = __fdiv_rn(ndt, __fmul_rn(__fmul_rn(len, len), len));
      for (int a = 0; a < 3; ++a) dp[2 + a] = -__fsub_rn(__fdiv_rn(t[a], len), __fmul_rn(k3, nv[a]));
      for (int c = 0; c < 3; ++c) {
        const float a = p[5 + c], tt = tg.albedo[c];
        const float denom = __fadd_rn(__fmul_rn(a, a), kRelL2Stabilizer);
        const float diff2 = __fsub_rn(a, tt);
        terms[4] = __fadd_rn(terms[4], __fdiv_rn(__fmul_rn(diff2, diff2), denom));
        dp[5 + c] = __fdiv_rn(__fsub_rn(__fmul_rn(__fmul_rn(2.0f, diff2), denom),
                                        __fmul_rn(__fmul_rn(__fmul_rn(diff2, diff2), 2.0f), a)),
                              __fmul_rn(denom, denom));
      }
      const int mat = tg.material < n_mat ? tg.material : n_mat - 1;
      const float prob = fminf(fmaxf(p[8 + mat], kProbClamp), 1.0f);
      terms[5] = -logf(prob);
      dp[8 + mat] = __fdiv_rn(-1.0f, prob);
    }
    terms[0] = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(terms[1], terms[2]), terms[3]), terms[4]), terms[5]);
    for (int q = 0; q < 6; ++q) terms[q] = __fmul_rn(terms[q], inv_batch);
    for (int r = 0; r < n_out; ++r) dp[r] = __fmul_rn(dp[r], inv_batch);
    // backward through the heads (mlp.hpp:192-204)
    float* d = dz3 + j * n_out;
    for (int r : {0, 1, 5, 6, 7}) {
      const float pc = fminf(fmaxf(p[r], 1e-7f), __fsub_rn(1.0f, 1e-7f));
      d[r] = __fmul_rn(__fmul_rn(dp[r], pc), __fsub_rn(1.0f, pc));
    }
    for (int k = 0; k < 3; ++k) d[2 + k] = dp[2 + k];
    float dot = 0.0f;
    for (int k = 0; k < n_mat; ++k) dot = __fadd_rn(dot, __fmul_rn(p[8 + k], dp[8 + k]));
    for (int k = 0; k < n_mat; ++k) d[8 + k] = __fmul_rn(p[8 + k], __fsub_rn(dp[8 + k], dot));
  }
  // block sums of the loss terms -> 6 atomics per block
  __shared__ float red[6][128];
  for (int q = 0; q < 6; ++q) red[q][threadIdx.x] = terms[q];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < 6; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) atomicAdd(loss6 + q, red[q][0]);
}

// accumulate_grad_into (encoding.hpp:193-209): gT[l][idx][f] += w * dx
__global__ void scatter_kernel(const float* dx, const uint32_t* cidx, const float* cw, const int8_t* ccount,
                               int64_t n, int H, int L, int F, uint32_t M, float* gT) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // (sample, point, level)
  if (i >= n * H * L) return;
  const int nc = ccount[i];
  if (nc == 0) return;
  const int64_t j = i / (H * L);
  const int kl = static_cast<int>(i - j * H * L);  // point * L + level
  const int l = kl % L;
  const float* up = dx + j * (static_cast<int64_t>(H) * L * F) + kl * F;
  float* g = gT + static_cast<size_t>(l) * M * F;
  for (int c = 0; c < nc; ++c) {
    const float wc = cw[i * 8 + c];
    const uint32_t idx = cidx[i * 8 + c];
    for (int f = 0; f < F; ++f) atomicAdd(g + static_cast<size_t>(idx) * F + f, __fmul_rn(wc, up[f]));
  }
}

// adam_update_tensor (mlp.hpp:243-256), every parameter
__global__ void adam_kernel(float* param, const float* grad, float* m, float* v, int64_t n, float lr, float b1,
                            float b2, float eps, float corr1, float corr2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float g = grad[i];
  const float mi = __fadd_rn(__fmul_rn(b1, m[i]), __fmul_rn(__fsub_rn(1.0f, b1), g));
  const float vi = __fadd_rn(__fmul_rn(b2, v[i]), __fmul_rn(__fsub_rn(1.0f, b2), __fmul_rn(g, g)));
  m[i] = mi;
  v[i] = vi;
  param[i] = __fsub_rn(param[i], __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mi, corr1)),
                                           __fadd_rn(__fsqrt_rn(__fdiv_rn(vi, corr2)), eps)));
}

}  // namespace lsnif_tr

// ================================================================== host

namespace lsnif_tr {

// tcgen05 split-TF32 GEMM (lsnif_tcgemm.cu), cublasSgemm semantics
cudaError_t tcgemm_colmajor(bool ta, bool tb, int mm, int nn, int kk, const float* A, int lda, const float* B, int ldb,
                            float* C, int ldc, float* work, size_t work_floats, int num_sms, cudaStream_t st);

struct Trainer {
  int device = 0;
  lsnif_model geo = nullptr;  // the init model: occupancy stop mask, frame, resolutions
  DevModel dm{};
  int V = 0, H = 0, L = 0, F = 0, K1 = 0, hid = 0, n_out = 0, n_mat = 0;
  uint32_t M = 0;
  std::vector<uint8_t> occupancy;
  std::vector<int32_t> level_res;
  std::vector<lsnif_material> materials;
  float aabb[6] = {};
  size_t n_tab = 0, off_w1 = 0, off_b1 = 0, off_w2 = 0, off_b2 = 0, off_w3 = 0, off_b3 = 0, n_params = 0;
  float *params = nullptr, *grads = nullptr, *m = nullptr, *v = nullptr;
  MeshDev mesh{};
  Frame frame{};
  lsnif_train_config cfg{};
  int64_t step = 0;
  int num_sms = 148;
  float* gemm_work = nullptr;  // split-K partials of the batch reductions
  size_t gemm_work_floats = 0;
  std::vector<void*> allocs;
  // batch buffers
  int64_t cap = 0;
  std::vector<void*> batch_allocs;
  lsnif_ray* rays = nullptr;
  lsnif_train_target* tg = nullptr;
  float *X = nullptr, *z1 = nullptr, *h1 = nullptr, *z2 = nullptr, *h2 = nullptr, *z3 = nullptr, *dz3 = nullptr;
  float *dh2 = nullptr, *dz2 = nullptr, *dh1 = nullptr, *dz1 = nullptr, *dx = nullptr, *cw = nullptr;
  float* loss6 = nullptr;
  uint32_t* cidx = nullptr;
  int8_t* ccount = nullptr;

  template <typename T>
  T* dalloc(size_t count, std::vector<void*>& list) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc(trainer)");
    list.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* upload(const T* src, size_t count) {
    T* p = dalloc<T>(count, allocs);
    if (count) ck(cudaMemcpy(p, src, count * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy(trainer)");
    return p;
  }
  void ensure_batch(int64_t n) {
    if (n <= cap) return;
    for (void* p : batch_allocs) cudaFree(p);
    batch_allocs.clear();
    rays = dalloc<lsnif_ray>(n, batch_allocs);
    tg = dalloc<lsnif_train_target>(n, batch_allocs);
    X = dalloc<float>(static_cast<size_t>(K1) * n, batch_allocs);
    dx = dalloc<float>(static_cast<size_t>(K1) * n, batch_allocs);
    for (float** p : {&z1, &h1, &z2, &h2, &dh2, &dz2, &dh1, &dz1})
      *p = dalloc<float>(static_cast<size_t>(hid) * n, batch_allocs);
    z3 = dalloc<float>(static_cast<size_t>(n_out) * n, batch_allocs);
    dz3 = dalloc<float>(static_cast<size_t>(n_out) * n, batch_allocs);
    cidx = dalloc<uint32_t>(static_cast<size_t>(n) * H * L * 8, batch_allocs);
    cw = dalloc<float>(static_cast<size_t>(n) * H * L * 8, batch_allocs);
    ccount = dalloc<int8_t>(static_cast<size_t>(n) * H * L, batch_allocs);
    loss6 = dalloc<float>(8, batch_allocs);
    cap = n;
  }
  ~Trainer() {
    if (device >= 0) cudaSetDevice(device);
    for (void* p : batch_allocs) cudaFree(p);
    for (void* p : allocs) cudaFree(p);
    cudaFree(params);
    cudaFree(grads);
    cudaFree(m);
    cudaFree(v);
    if (geo) lsnif_model_destroy(geo);
  }
};

template <typename K, typename... A>
void launch(K kern, int64_t n, int threads, size_t smem, cudaStream_t st, const char* what, A... args) {
  if (n <= 0) return;
  kern<<<static_cast<unsigned>((n + threads - 1) / threads), threads, smem, st>>>(args...);
  ck(cudaGetLastError(), what);
}

constexpr bool OP_N = false, OP_T = true;

void gemm(Trainer& T, cudaStream_t st, bool ta, bool tb, int mm, int nn, int kk, const float* A, int lda,
          const float* B, int ldb, float* Cm, int ldc) {
  ck(tcgemm_colmajor(ta, tb, mm, nn, kk, A, lda, B, ldb, Cm, ldc, T.gemm_work, T.gemm_work_floats, T.num_sms, st),
     "tcgemm_kernel");
}

// Forward + loss + backward of one batch into T.grads (zeroed first) and T.loss6.
void batch_grads(Trainer& T, const lsnif_ray* rays, const lsnif_train_target* tg, int64_t n, cudaStream_t st) {
  T.ensure_batch(n);
  ck(cudaMemsetAsync(T.grads, 0, T.n_params * sizeof(float), st), "cudaMemsetAsync");
  ck(cudaMemsetAsync(T.loss6, 0, 8 * sizeof(float), st), "cudaMemsetAsync");
  const int nn = static_cast<int>(n);
  const float* P = T.params;
  float* G = T.grads;
  launch(encode_kernel, n, 128, static_cast<size_t>(T.dm.stop_words) * 4, st, "encode_kernel", T.dm, P, rays, n, T.X,
         T.cidx, T.cw, T.ccount);
  // forward_cached (mlp.hpp:117-130); weights row-major [out][in] = col-major [in][out]
  gemm(T, st, OP_T, OP_N, T.hid, nn, T.K1, P + T.off_w1, T.K1, T.X, T.K1, T.z1, T.hid);
  launch(bias_leaky_kernel, static_cast<int64_t>(T.hid) * n, 256, 0, st, "bias_leaky", T.z1, T.h1, P + T.off_b1, T.hid, n);
  gemm(T, st, OP_T, OP_N, T.hid, nn, T.hid, P + T.off_w2, T.hid, T.h1, T.hid, T.z2, T.hid);
  launch(bias_leaky_kernel, static_cast<int64_t>(T.hid) * n, 256, 0, st, "bias_leaky", T.z2, T.h2, P + T.off_b2, T.hid, n);
  gemm(T, st, OP_T, OP_N, T.n_out, nn, T.hid, P + T.off_w3, T.hid, T.h2, T.hid, T.z3, T.n_out);
  launch(heads_loss_kernel, n, 128, 0, st, "heads_loss_kernel", static_cast<const float*>(T.z3), P + T.off_b3, T.n_out,
         T.n_mat, n, tg, 1.0f / static_cast<float>(n), T.dz3, T.loss6);
  // backward (mlp.hpp:206-225)
  gemm(T, st, OP_N, OP_T, T.hid, T.n_out, nn, T.h2, T.hid, T.dz3, T.n_out, G + T.off_w3, T.hid);
  rowsum_kernel<<<T.n_out, 256, 0, st>>>(T.dz3, T.n_out, n, G + T.off_b3);
  gemm(T, st, OP_N, OP_N, T.hid, nn, T.n_out, P + T.off_w3, T.hid, T.dz3, T.n_out, T.dh2, T.hid);
  launch(leaky_back_kernel, static_cast<int64_t>(T.hid) * n, 256, 0, st, "leaky_back", T.dh2, T.z2, T.dz2,
         static_cast<int64_t>(T.hid) * n);
  gemm(T, st, OP_N, OP_T, T.hid, T.hid, nn, T.h1, T.hid, T.dz2, T.hid, G + T.off_w2, T.hid);
  rowsum_kernel<<<T.hid, 256, 0, st>>>(T.dz2, T.hid, n, G + T.off_b2);
  gemm(T, st, OP_N, OP_N, T.hid, nn, T.hid, P + T.off_w2, T.hid, T.dz2, T.hid, T.dh1, T.hid);
  launch(leaky_back_kernel, static_cast<int64_t>(T.hid) * n, 256, 0, st, "leaky_back", T.dh1, T.z1, T.dz1,
         static_cast<int64_t>(T.hid) * n);
  gemm(T, st, OP_N, OP_T, T.K1, T.hid, nn, T.X, T.K1, T.dz1, T.hid, G + T.off_w1, T.K1);
  rowsum_kernel<<<T.hid, 256, 0, st>>>(T.dz1, T.hid, n, G + T.off_b1);
  gemm(T, st, OP_N, OP_N, T.K1, nn, T.hid, P + T.off_w1, T.K1, T.dz1, T.hid, T.dx, T.K1);
  ck(cudaGetLastError(), "rowsum_kernel");
  // hash-grid gradient (encoding.hpp:193-209)
  launch(scatter_kernel, n * T.H * T.L, 256, 0, st, "scatter_kernel", static_cast<const float*>(T.dx),
         static_cast<const uint32_t*>(T.cidx), static_cast<const float*>(T.cw),
         static_cast<const int8_t*>(T.ccount), n, T.H, T.L, T.F, T.M, G);
}

void read_loss(Trainer& T, cudaStream_t st, lsnif_train_loss* out) {
  if (!out) return;
  float h[8];
  ck(cudaMemcpyAsync(h, T.loss6, sizeof(h), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync(loss)");
  ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  out->total = h[0];
  out->occlusion_bce = h[1];
  out->local_t_mae = h[2];
  out->normal_cosine = h[3];
  out->albedo_rel_l2 = h[4];
  out->material_ce = h[5];
  out->step = T.step;
}

void sample(Trainer& T, int64_t step, int64_t n, lsnif_ray* rays, lsnif_train_target* tg, cudaStream_t st) {
  launch(sample_kernel, 32 * n, 128, 0, st, "sample_kernel", T.mesh, T.frame, T.cfg.seed, step,
         T.cfg.external_mix, n, rays, tg);
}

}  // namespace lsnif_tr

// ------------------------------------------------------------------ API glue

namespace lsnif_api {

using lsnif_tr::Trainer;

void* trainer_create(const lsnif_model_desc& d, const lsnif_mesh_desc& mesh, const lsnif_train_config& cfg,
                     int device, lsnif_model geo, const lsnif_dev::DevModel& dm) {
  if (cfg.batch < 1) fail(LSNIF_INVALID_ARGUMENT, "train: steps and batch must be >= 1");
  if (mesh.n_faces < 1 || mesh.n_vertices < 3 || !mesh.vertices || !mesh.faces || !mesh.face_material)
    fail(LSNIF_INVALID_ARGUMENT, "train: mesh needs vertices, faces and face materials");
  for (int i = 0; i < 3 * mesh.n_faces; ++i)
    if (mesh.faces[i] < 0 || mesh.faces[i] >= mesh.n_vertices) fail(LSNIF_RUNTIME_ERROR, "mesh face index out of range");
  auto T = std::make_unique<Trainer>();
  T->device = device;
  T->geo = geo;
  T->dm = dm;
  T->cfg = cfg;
  T->V = d.voxel_res;
  T->H = d.hit_cap;
  T->L = d.n_levels;
  T->F = d.f_dim;
  T->M = d.table_size;
  T->hid = d.hidden;
  T->n_mat = d.n_mat;
  T->n_out = 8 + d.n_mat;
  T->K1 = T->H * T->L * T->F;
  for (int i = 0; i < mesh.n_faces; ++i)
    if (mesh.face_material[i] < 0 || mesh.face_material[i] >= std::max(d.n_materials, 1))
      fail(LSNIF_RUNTIME_ERROR, "mesh face material out of range");
  T->occupancy.assign(d.occupancy, d.occupancy + static_cast<size_t>(T->V) * T->V * T->V / 8);
  T->level_res.assign(d.level_res, d.level_res + T->L);
  T->materials.assign(d.materials, d.materials + std::max(d.n_materials, 0));
  std::memcpy(T->aabb, d.aabb, sizeof(T->aabb));
  // parameters, fp32: tables | w1 | b1 | w2 | b2 | w3 | b3
  T->n_tab = static_cast<size_t>(T->L) * T->M * T->F;
  T->off_w1 = T->n_tab;
  T->off_b1 = T->off_w1 + static_cast<size_t>(T->hid) * T->K1;
  T->off_w2 = T->off_b1 + T->hid;
  T->off_b2 = T->off_w2 + static_cast<size_t>(T->hid) * T->hid;
  T->off_w3 = T->off_b2 + T->hid;
  T->off_b3 = T->off_w3 + static_cast<size_t>(T->n_out) * T->hid;
  T->n_params = T->off_b3 + T->n_out;
  std::vector<float> hp(T->n_params);
  auto dec = [](uint16_t h) { return __half2float(__ushort_as_half(h)); };
  for (int l = 0; l < T->L; ++l)
    for (size_t i = 0; i < static_cast<size_t>(T->M) * T->F; ++i)
      hp[static_cast<size_t>(l) * T->M * T->F + i] = dec(d.tables[l][i]);
  auto put = [&](size_t off, const uint16_t* src, size_t count) {
    for (size_t i = 0; i < count; ++i) hp[off + i] = dec(src[i]);
  };
  put(T->off_w1, d.w1, static_cast<size_t>(T->hid) * T->K1);
  put(T->off_b1, d.b1, T->hid);
  put(T->off_w2, d.w2, static_cast<size_t>(T->hid) * T->hid);
  put(T->off_b2, d.b2, T->hid);
  put(T->off_w3, d.w3, static_cast<size_t>(T->n_out) * T->hid);
  put(T->off_b3, d.b3, T->n_out);
  for (float** p : {&T->params, &T->grads, &T->m, &T->v})
    ck(cudaMalloc(p, T->n_params * sizeof(float)), "cudaMalloc(trainer params)");
  ck(cudaMemcpy(T->params, hp.data(), T->n_params * sizeof(float), cudaMemcpyHostToDevice), "cudaMemcpy");
  ck(cudaMemset(T->m, 0, T->n_params * sizeof(float)), "cudaMemset");
  ck(cudaMemset(T->v, 0, T->n_params * sizeof(float)), "cudaMemset");
  // mesh
  lsnif_tr::MeshDev& M = T->mesh;
  M.v = T->upload(mesh.vertices, 3 * static_cast<size_t>(mesh.n_vertices));
  M.f = T->upload(mesh.faces, 3 * static_cast<size_t>(mesh.n_faces));
  {  // corner positions per face, one 16-byte load each in the triangle loop
    std::vector<float4> tri(3 * static_cast<size_t>(mesh.n_faces));
    for (int f = 0; f < mesh.n_faces; ++f)
      for (int k = 0; k < 3; ++k) {
        const float* p = mesh.vertices + 3 * static_cast<size_t>(mesh.faces[3 * f + k]);
        tri[3 * static_cast<size_t>(f) + k] = make_float4(p[0], p[1], p[2], 0.0f);
      }
    M.tri = T->upload(tri.data(), tri.size());
  }
  M.fmat = T->upload(mesh.face_material, static_cast<size_t>(mesh.n_faces));
  M.n = nullptr;
  M.fn = nullptr;
  if (mesh.normals && mesh.n_normals > 0 && mesh.face_normals) {
    for (int i = 0; i < 3 * mesh.n_faces; ++i)
      if (mesh.face_normals[i] < 0 || mesh.face_normals[i] >= mesh.n_normals)
        fail(LSNIF_RUNTIME_ERROR, "mesh normal index out of range");
    M.n = T->upload(mesh.normals, 3 * static_cast<size_t>(mesh.n_normals));
    M.fn = T->upload(mesh.face_normals, 3 * static_cast<size_t>(mesh.n_faces));
  }
  M.nf = mesh.n_faces;
  std::vector<float> alb;
  for (const lsnif_material& mt : T->materials)
    for (int a = 0; a < 3; ++a) alb.push_back(mt.albedo[a]);
  if (alb.empty()) alb = {0.7f, 0.7f, 0.7f};
  M.albedo = T->upload(alb.data(), alb.size());
  M.n_mats = static_cast<int>(alb.size() / 3);
  // frame: the model's box (LocalFrame::for_mesh, already inflated)
  lsnif_tr::Frame& fr = T->frame;
  float ext[3];
  for (int a = 0; a < 3; ++a) {
    fr.mn[a] = d.aabb[a];
    fr.mx[a] = d.aabb[3 + a];
    fr.center[a] = 0.5f * (fr.mn[a] + fr.mx[a]);  // Aabb::center
    ext[a] = fr.mx[a] - fr.mn[a];
  }
  const float diag = std::sqrt((ext[0] * ext[0] + ext[1] * ext[1]) + ext[2] * ext[2]);  // Aabb::diagonal
  fr.radius = 0.5f * diag;
  fr.eps = 1e-4f * diag;  // self_intersection_eps (training.cpp:15-17)
  ck(cudaDeviceGetAttribute(&T->num_sms, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
  T->gemm_work_floats = static_cast<size_t>(T->num_sms) * 128 * 128;
  T->gemm_work = T->dalloc<float>(T->gemm_work_floats, T->allocs);
  return T.release();
}

void trainer_destroy(void* t) { delete static_cast<Trainer*>(t); }

void trainer_step(void* t, int steps, lsnif_train_loss* last, cudaStream_t st) {
  Trainer& T = *static_cast<Trainer*>(t);
  if (steps < 0) fail(LSNIF_INVALID_ARGUMENT, "train: negative step count");
  ck(cudaSetDevice(T.device), "cudaSetDevice");
  const int64_t B = T.cfg.batch;
  T.ensure_batch(B);
  for (int s = 0; s < steps; ++s) {
    lsnif_tr::sample(T, T.step, B, T.rays, T.tg, st);
    lsnif_tr::batch_grads(T, T.rays, T.tg, B, st);
    ++T.step;  // AdamState::step (mlp.hpp:266) == grid_states[l].step (training.cpp:209)
    const float corr1 = 1.0f - std::pow(0.9f, static_cast<float>(T.step));
    const float corr2 = 1.0f - std::pow(0.999f, static_cast<float>(T.step));
    lsnif_tr::launch(lsnif_tr::adam_kernel, static_cast<int64_t>(T.n_params), 256, 0, st, "adam_kernel", T.params,
                     static_cast<const float*>(T.grads), T.m, T.v, static_cast<int64_t>(T.n_params), T.cfg.lr, 0.9f,
                     0.999f, 1e-8f, corr1, corr2);
  }
  if (last) lsnif_tr::read_loss(T, st, last);
}

void trainer_batch_grad(void* t, const lsnif_ray* rays, const lsnif_train_target* tg, int64_t n,
                        lsnif_train_loss* loss, float* g_mlp, float* g_tab, cudaStream_t st) {
  Trainer& T = *static_cast<Trainer*>(t);
  if (n < 1 || !rays || !tg) fail(LSNIF_INVALID_ARGUMENT, "batch_grad: need n >= 1 rays and targets");
  ck(cudaSetDevice(T.device), "cudaSetDevice");
  lsnif_tr::batch_grads(T, rays, tg, n, st);
  if (g_tab) ck(cudaMemcpyAsync(g_tab, T.grads, T.n_tab * 4, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
  if (g_mlp)
    ck(cudaMemcpyAsync(g_mlp, T.grads + T.n_tab, (T.n_params - T.n_tab) * 4, cudaMemcpyDeviceToDevice, st),
       "cudaMemcpyAsync");
  lsnif_train_loss tmp;
  lsnif_tr::read_loss(T, st, loss ? loss : &tmp);
}

void trainer_sample(void* t, int64_t step, int64_t n, lsnif_ray* rays, lsnif_train_target* tg, cudaStream_t st) {
  Trainer& T = *static_cast<Trainer*>(t);
  if (n < 0 || (n > 0 && (!rays || !tg))) fail(LSNIF_INVALID_ARGUMENT, "sample: bad output");
  ck(cudaSetDevice(T.device), "cudaSetDevice");
  lsnif_tr::sample(T, step, n, rays, tg, st);
}

// save_model + load_model round trip (model_io.cpp:71-175): binary16 params.
void trainer_export(void* t, int device, lsnif_model* out) {
  Trainer& T = *static_cast<Trainer*>(t);
  ck(cudaSetDevice(T.device), "cudaSetDevice");
  ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  std::vector<float> hp(T.n_params);
  ck(cudaMemcpy(hp.data(), T.params, T.n_params * 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
  std::vector<uint16_t> hh(T.n_params);
  for (size_t i = 0; i < T.n_params; ++i) hh[i] = __half_as_ushort(__float2half_rn(hp[i]));
  std::vector<const uint16_t*> tabs(T.L);
  for (int l = 0; l < T.L; ++l) tabs[l] = hh.data() + static_cast<size_t>(l) * T.M * T.F;
  lsnif_model_desc d{};
  d.voxel_res = T.V;
  d.hit_cap = T.H;
  d.n_levels = T.L;
  d.f_dim = T.F;
  d.table_size = T.M;
  d.hidden = T.hid;
  d.n_mat = T.n_mat;
  d.occupancy = T.occupancy.data();
  d.level_res = T.level_res.data();
  d.tables = tabs.data();
  d.w1 = hh.data() + T.off_w1;
  d.b1 = hh.data() + T.off_b1;
  d.w2 = hh.data() + T.off_w2;
  d.b2 = hh.data() + T.off_b2;
  d.w3 = hh.data() + T.off_w3;
  d.b3 = hh.data() + T.off_b3;
  d.materials = T.materials.data();
  d.n_materials = static_cast<int32_t>(T.materials.size());
  std::memcpy(d.aabb, T.aabb, sizeof(d.aabb));
  const lsnif_status s = lsnif_model_create(&d, device, out);
  if (s != LSNIF_OK) fail(s, lsnif_last_error());
}

}  // namespace lsnif_api
