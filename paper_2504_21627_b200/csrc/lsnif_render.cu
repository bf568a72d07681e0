// Wavefront LSNIF path tracer for sm_100a.
//
// The reference's render() (proj/src/renderer.cpp:453-542) keeps paths in a
// host vector and calls intersect_scene / occluded_batch once per bounce on
// the active rays. Here the paths stay in HBM for the whole render: per wave
// of paths and per bounce
//   1. the active rays (compacted) go through lsnif_scene_query (CLOSEST),
//   2. shade_kernel applies shade_hit (renderer.cpp:378-442) per path: the
//      environment on a miss, next-event shadow rays into fixed per-path
//      slots, the BSDF sample and the compacted next-bounce ray list,
//   3. the shadow slots go through lsnif_scene_query (ANY) and
//      shadow_accum_kernel adds the unblocked contributions in light order,
// and resolve_kernel averages the samples of each pixel in sample order.
//
// Random numbers are the reference's exactly: each path owns the std::mt19937
// stream seeded with seed_stream(seed, pixel, sample) (renderer.cpp:470-471),
// read through uniform_real_distribution<float> (sampling.hpp:12-14). The
// first 227 outputs of a freshly seeded mt19937 depend only on the seeding
// words j, j+1 and j+397 (the first twist reads untwisted state), so a path
// carries four words instead of 624 — valid for up to 227 draws per path,
// which lsnif_render checks up front.
//
// Float expressions follow the reference's Eigen evaluation order (dot and
// squaredNorm as ((x + y) + z), scalar chains left to right, vector
// normalisation as division by the square root), unfused.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "lsnif_gpu.h"
#include "lsnif_internal.hpp"

namespace lsnif_pt {

using lsnif_api::ck;
using lsnif_api::fail;

constexpr int kMaxLights = 32;        // lights passed by value to the kernels
constexpr int kMaxShadows = 8;        // ShadeOutcome::shadows (renderer.cpp:368)
constexpr int kMaxDraws = 227;        // mt19937 outputs servable from the seeding words
constexpr float kPi = 3.14159265358979323846f;         // Real(M_PI)
constexpr float kInvPi = 0.318309886183790671538f;     // Real(M_1_PI)

// ------------------------------------------------------------- mt19937

struct Mt {
  uint32_t j;   // outputs drawn so far
  uint32_t a0;  // seeding word j
  uint32_t a1;  // seeding word j + 1
  uint32_t b;   // seeding word j + 397
};

__host__ __device__ __forceinline__ uint32_t mt_seed_step(uint32_t x, uint32_t i) {
  return 1812433253u * (x ^ (x >> 30)) + i;  // std::mt19937::seed
}

__device__ __forceinline__ Mt mt_seed(uint32_t s) {
  Mt m;
  m.j = 0;
  m.a0 = s;
  uint32_t x = mt_seed_step(s, 1);
  m.a1 = x;
  for (uint32_t i = 2; i <= 397; ++i) x = mt_seed_step(x, i);
  m.b = x;
  return m;
}

// Output j: the first twist's word j (needs untwisted words j, j+1, j+397),
// tempered.
__device__ __forceinline__ uint32_t mt_next(Mt& m) {
  const uint32_t y = (m.a0 & 0x80000000u) | (m.a1 & 0x7fffffffu);
  uint32_t v = m.b ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
  v ^= v >> 11;
  v ^= (v << 7) & 0x9d2c5680u;
  v ^= (v << 15) & 0xefc60000u;
  v ^= v >> 18;
  m.a0 = m.a1;
  m.a1 = mt_seed_step(m.a1, m.j + 2);
  m.b = mt_seed_step(m.b, m.j + 398);
  ++m.j;
  return v;
}

// uniform_real(rng) (sampling.hpp:12-14): libstdc++ generate_canonical<float,
// 24> with one 32-bit draw = float(x) / 2^32, clamped below 1.
__device__ __forceinline__ float mt_uniform(Mt& m) {
  const float f = __fmul_rn(__uint2float_rn(mt_next(m)), 2.3283064365386962890625e-10f);
  return f >= 1.0f ? 0.99999994f : f;
}

// seed_stream (types.hpp:25-39)
__host__ __device__ __forceinline__ uint64_t mix_bits(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint32_t seed_stream(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t h = mix_bits(seed + 0x632be59bd9b4e019ull);
  h = mix_bits(h ^ a);
  h = mix_bits(h ^ b);
  h = mix_bits(h ^ 0ull);
  return static_cast<uint32_t>(h >> 32);
}

// ------------------------------------------------------------- vectors

__device__ __forceinline__ float dot3(const float a[3], const float b[3]) {
  return __fadd_rn(__fadd_rn(__fmul_rn(a[0], b[0]), __fmul_rn(a[1], b[1])), __fmul_rn(a[2], b[2]));
}

// Eigen normalized(): v / sqrt(squaredNorm) when the norm is positive.
__device__ __forceinline__ void normalize3(float v[3]) {
  const float n2 = dot3(v, v);
  if (n2 > 0.0f) {
    const float n = __fsqrt_rn(n2);
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = __fdiv_rn(v[a], n);
  }
}

// orthonormal_basis (sampling.hpp:18-24)
__device__ __forceinline__ void orthonormal_basis(const float n[3], float t[3], float b[3]) {
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

// uniform_sphere_dir (sampling.hpp:26-31)
__device__ __forceinline__ void uniform_sphere_dir(Mt& rng, float out[3]) {
  const float z = __fsub_rn(1.0f, __fmul_rn(2.0f, mt_uniform(rng)));
  const float r = __fsqrt_rn(fmaxf(0.0f, __fsub_rn(1.0f, __fmul_rn(z, z))));
  const float phi = __fmul_rn(__fmul_rn(2.0f, kPi), mt_uniform(rng));
  out[0] = __fmul_rn(r, cosf(phi));
  out[1] = __fmul_rn(r, sinf(phi));
  out[2] = z;
}

// cosine_hemisphere_dir (sampling.hpp:35-46)
__device__ __forceinline__ void cosine_hemisphere_dir(const float axis[3], Mt& rng, float out[3]) {
  const float u1 = mt_uniform(rng);
  const float u2 = mt_uniform(rng);
  const float r = __fsqrt_rn(u1);
  const float phi = __fmul_rn(__fmul_rn(2.0f, kPi), u2);
  const float x = __fmul_rn(r, cosf(phi));
  const float y = __fmul_rn(r, sinf(phi));
  const float z = __fsqrt_rn(fmaxf(0.0f, __fsub_rn(1.0f, u1)));
  float t[3], b[3];
  orthonormal_basis(axis, t, b);
#pragma unroll
  for (int a = 0; a < 3; ++a) out[a] = __fadd_rn(__fadd_rn(__fmul_rn(x, t[a]), __fmul_rn(y, b[a])), __fmul_rn(z, axis[a]));
  normalize3(out);
}

// ------------------------------------------------------------- parameters

struct CameraBasis {  // make_camera_basis (renderer.cpp:334-344)
  float origin[3], forward[3], right[3], up[3];
  float half_w, half_h;
};

struct Params {
  CameraBasis cam;
  int width, height, spp, max_bounces;
  uint64_t seed;
  float eps_scale;
  float env[3];
  int n_lights, n_shadow_slots;
  lsnif_light lights[kMaxLights];
  const float* world_diag;  // per instance (DEVICE)
};

// Path state of one wave (structure of arrays, DEVICE). Counts live on the
// device (no host round trip between bounces): counts[d] = active rays at
// bounce d, counts[kMaxDepth + d] = shadow rays emitted at bounce d.
constexpr int kMaxDepth = 128;
struct Paths {
  lsnif_ray* rays[2];      // active rays of the current / next bounce (compacted)
  int32_t* slots[2];       // path of each active ray
  int32_t* counts;         // 2 * kMaxDepth device counters
  lsnif_scene_hit* hits;   // closest-hit results of the active rays
  float* thr;              // throughput, 3 per path
  float* rad;              // radiance, 3 per path
  uint4* rng;              // Mt per path
  int32_t* shadow_first;   // per active ray: first shadow ray, count in shadow_n
  int32_t* shadow_n;
  lsnif_ray* shadow_rays;  // compacted; each ray's shadows contiguous, in light order
  float* shadow_contrib;   // 3 per shadow ray
  lsnif_scene_hit* shadow_hits;
};

__device__ __forceinline__ Mt load_mt(const uint4& v) { return Mt{v.x, v.y, v.z, v.w}; }
__device__ __forceinline__ uint4 store_mt(const Mt& m) { return make_uint4(m.j, m.a0, m.a1, m.b); }

// camera_ray (renderer.cpp:347-361)
__device__ __forceinline__ void camera_ray(const Params& P, int px, int py, Mt& rng, lsnif_ray& ray) {
  const float u = mt_uniform(rng);
  const float v = mt_uniform(rng);
  const float sx = __fsub_rn(__fdiv_rn(__fmul_rn(2.0f, __fadd_rn(static_cast<float>(px), u)),
                                       static_cast<float>(P.width)), 1.0f);
  const float sy = __fsub_rn(1.0f, __fdiv_rn(__fmul_rn(2.0f, __fadd_rn(static_cast<float>(py), v)),
                                             static_cast<float>(P.height)));
  const float ax = __fmul_rn(sx, P.cam.half_w), ay = __fmul_rn(sy, P.cam.half_h);
  float d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    d[a] = __fadd_rn(__fadd_rn(P.cam.forward[a], __fmul_rn(ax, P.cam.right[a])), __fmul_rn(ay, P.cam.up[a]));
  normalize3(d);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ray.origin[a] = P.cam.origin[a];
    ray.direction[a] = d[a];
  }
  ray.t_min = 0.0f;
  ray.t_max = __int_as_float(0x7f800000);
}

// ------------------------------------------------------------- kernels

// Paths [0, n) of a wave starting at path `first` (path = pixel * spp + sample):
// seed the stream, draw the primary ray, reset throughput / radiance.
__global__ void __launch_bounds__(256) camera_kernel(const Params P, Paths S, int64_t first, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) S.counts[0] = static_cast<int32_t>(n);
  if (i >= n) return;
  const int64_t path = first + i;
  const int64_t pixel = path / P.spp;
  const int sample = static_cast<int>(path - pixel * P.spp);
  Mt rng = mt_seed(seed_stream(P.seed, static_cast<uint64_t>(pixel), static_cast<uint64_t>(sample)));
  lsnif_ray r;
  camera_ray(P, static_cast<int>(pixel % P.width), static_cast<int>(pixel / P.width), rng, r);
  S.rays[0][i] = r;
  S.slots[0][i] = static_cast<int32_t>(i);
  S.rng[i] = store_mt(rng);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    S.thr[3 * i + a] = 1.0f;
    S.rad[3 * i + a] = 0.0f;
  }
}

// One shading event per active ray (render loop body, renderer.cpp:506-534,
// with shade_hit, 378-442): miss -> environment; hit -> NEE shadow rays
// (appended, contiguous per path), then the BSDF sample; continuing paths are
// appended to the next bounce's list. The active count is read on the device.
__device__ __forceinline__ void shade_one(const Params& P, Paths& S, int cur, int depth, int spawn, int64_t n,
                                          int64_t k) {
  const int lane = threadIdx.x & 31;
  bool cont = false;
  lsnif_ray next{};
  int32_t path = 0;
  lsnif_ray srays[kMaxShadows];
  float scon[3 * kMaxShadows];
  int ns = 0;
  if (k < n) {
    path = (cur ? S.slots[1] : S.slots[0])[k];  // selects, not a dynamic index (keeps Paths out of local memory)
    const lsnif_ray ray = (cur ? S.rays[1] : S.rays[0])[k];
    const lsnif_scene_hit h = S.hits[k];
    float thr[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) thr[a] = S.thr[3 * path + a];
    if (!(h.flags & 1u)) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        S.rad[3 * path + a] = __fadd_rn(S.rad[3 * path + a], __fmul_rn(thr[a], P.env[a]));
    } else {
      Mt rng = load_mt(S.rng[path]);
      const float eps = __fmul_rn(P.eps_scale, P.world_diag[h.object_index]);  // neural hit
      float spawn_o[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) spawn_o[a] = __fadd_rn(h.position[a], __fmul_rn(eps, h.normal[a]));
      float ta[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) ta[a] = __fmul_rn(thr[a], h.albedo[a]);  // throughput ⊙ albedo
      if (h.kind == 0u) {  // diffuse: next-event estimation per light
        for (int li = 0; li < P.n_lights; ++li) {
          const lsnif_light& L = P.lights[li];
          float target[3] = {L.position[0], L.position[1], L.position[2]};
          float ln[3] = {0.0f, 0.0f, 0.0f};
          float pdf_area = 1.0f;
          if (L.type == LSNIF_LIGHT_SPHERE) {
            uniform_sphere_dir(rng, ln);
#pragma unroll
            for (int a = 0; a < 3; ++a) target[a] = __fadd_rn(L.position[a], __fmul_rn(L.radius, ln[a]));
            pdf_area = __fdiv_rn(1.0f, __fmul_rn(__fmul_rn(__fmul_rn(4.0f, kPi), L.radius), L.radius));
          }
          float tl[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) tl[a] = __fsub_rn(target[a], spawn_o[a]);
          const float dist2 = dot3(tl, tl);
          if (dist2 <= 0.0f) continue;
          const float dist = __fsqrt_rn(dist2);
          float wi[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) wi[a] = __fdiv_rn(tl[a], dist);
          const float cos_surf = dot3(h.normal, wi);
          if (cos_surf <= 0.0f) continue;
          float c[3];
          if (L.type == LSNIF_LIGHT_SPHERE) {
            const float nwi[3] = {-wi[0], -wi[1], -wi[2]};
            const float cos_light = dot3(ln, nwi);
            if (cos_light <= 0.0f) continue;
            const float den = __fmul_rn(dist2, pdf_area);
#pragma unroll
            for (int a = 0; a < 3; ++a)
              c[a] = __fdiv_rn(__fmul_rn(__fmul_rn(__fmul_rn(ta[a], kInvPi), cos_surf), cos_light), den);
          } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) c[a] = __fdiv_rn(__fmul_rn(__fmul_rn(ta[a], kInvPi), cos_surf), dist2);
          }
#pragma unroll
          for (int a = 0; a < 3; ++a) c[a] = __fmul_rn(c[a], L.radiance[a]);
          if (c[0] <= 0.0f && c[1] <= 0.0f && c[2] <= 0.0f) continue;
          if (ns >= kMaxShadows) continue;
          lsnif_ray& sr = srays[ns];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            sr.origin[a] = spawn_o[a];
            sr.direction[a] = wi[a];
            scon[3 * ns + a] = c[a];
          }
          sr.t_min = 0.0f;
          sr.t_max = __fmul_rn(dist, 0.9999f);  // dist * Real(1 - 1e-4)
          ++ns;
        }
      }
      if (spawn) {
        float dir[3];
        bool ok = true;
        if (h.kind == 0u) {
          cosine_hemisphere_dir(h.normal, rng, dir);
        } else {  // Phong lobe around the mirror direction
          const float dn = dot3(ray.direction, h.normal);
          float refl[3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
            refl[a] = __fsub_rn(ray.direction[a], __fmul_rn(__fmul_rn(2.0f, dn), h.normal[a]));
          normalize3(refl);
          const float exponent =
              fmaxf(0.0f, __fsub_rn(__fdiv_rn(2.0f, __fmul_rn(h.roughness, h.roughness)), 2.0f));
          const float u1 = mt_uniform(rng);
          const float u2 = mt_uniform(rng);
          const float cos_a = powf(u1, __fdiv_rn(1.0f, __fadd_rn(exponent, 1.0f)));
          const float sin_a = __fsqrt_rn(fmaxf(0.0f, __fsub_rn(1.0f, __fmul_rn(cos_a, cos_a))));
          const float phi = __fmul_rn(__fmul_rn(2.0f, kPi), u2);
          float t[3], b[3];
          orthonormal_basis(refl, t, b);
          const float sc = __fmul_rn(sin_a, cosf(phi)), ss = __fmul_rn(sin_a, sinf(phi));
#pragma unroll
          for (int a = 0; a < 3; ++a)
            dir[a] = __fadd_rn(__fadd_rn(__fmul_rn(sc, t[a]), __fmul_rn(ss, b[a])), __fmul_rn(cos_a, refl[a]));
          normalize3(dir);
          ok = dot3(dir, h.normal) > 0.0f;
        }
        if (ok) {
          cont = true;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            next.origin[a] = spawn_o[a];
            next.direction[a] = dir[a];
            S.thr[3 * path + a] = ta[a];
          }
          next.t_min = 0.0f;
          next.t_max = __int_as_float(0x7f800000);
        }
      }
      S.rng[path] = store_mt(rng);
    }
  }
  // ---- warp-aggregated appends: shadow rays (contiguous per path) and the
  //      continuing paths
  int incl = ns;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int sbase = 0;
  if (lane == 31 && total) sbase = atomicAdd(S.counts + kMaxDepth + depth, total);
  sbase = __shfl_sync(0xffffffffu, sbase, 31) + incl - ns;
  if (k < n) {
    S.shadow_first[k] = sbase;
    S.shadow_n[k] = ns;
    for (int q = 0; q < ns; ++q) {
      S.shadow_rays[sbase + q] = srays[q];
#pragma unroll
      for (int a = 0; a < 3; ++a) S.shadow_contrib[3 * (sbase + q) + a] = scon[3 * q + a];
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, cont);
  int base = 0;
  if (lane == 0 && m) base = atomicAdd(S.counts + depth + 1, __popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (cont) {
    const int j = base + __popc(m & ((1u << lane) - 1u));
    (cur ? S.rays[0] : S.rays[1])[j] = next;
    (cur ? S.slots[0] : S.slots[1])[j] = path;
  }
}

__global__ void __launch_bounds__(256) shade_kernel(const Params P, Paths S, int cur, int depth, int spawn) {
  const int64_t n = S.counts[depth];
  // block-stride over the device-side count (the grid is sized for the machine)
  for (int64_t kb = static_cast<int64_t>(blockIdx.x) * blockDim.x; kb < n;
       kb += static_cast<int64_t>(gridDim.x) * blockDim.x)
    shade_one(P, S, cur, depth, spawn, n, kb + threadIdx.x);
}

// occluded_batch result -> radiance (renderer.cpp:536-541), light order.
__global__ void __launch_bounds__(256) shadow_accum_kernel(Paths S, int cur, int depth) {
  const int64_t n = S.counts[depth];
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int ns = S.shadow_n[k];
    if (ns == 0) continue;
    const int first = S.shadow_first[k];
    const int32_t path = (cur ? S.slots[1] : S.slots[0])[k];
    float rad[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) rad[a] = S.rad[3 * path + a];
    for (int q = first; q < first + ns; ++q) {
      if (S.shadow_hits[q].flags & 1u) continue;  // blocked
#pragma unroll
      for (int a = 0; a < 3; ++a) rad[a] = __fadd_rn(rad[a], S.shadow_contrib[3 * q + a]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) S.rad[3 * path + a] = rad[a];
  }
}

// Image accumulation (renderer.cpp:538-545): pixel += radiance of its
// samples in sample order, then *= 1/spp.
__global__ void __launch_bounds__(256) resolve_kernel(const Params P, const float* rad, int64_t first_pixel,
                                                      int64_t n_pixels, float* image) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pixels) return;
  float acc[3] = {0.0f, 0.0f, 0.0f};
  for (int s = 0; s < P.spp; ++s) {
    const int64_t q = i * P.spp + s;
#pragma unroll
    for (int a = 0; a < 3; ++a) acc[a] = __fadd_rn(acc[a], rad[3 * q + a]);
  }
  const float inv_spp = __fdiv_rn(1.0f, static_cast<float>(P.spp));
#pragma unroll
  for (int a = 0; a < 3; ++a) image[3 * (first_pixel + i) + a] = __fmul_rn(acc[a], inv_spp);
}

__global__ void __launch_bounds__(256) debug_paths_kernel(const Params P, int64_t first, int64_t n,
                                                          lsnif_ray* rays, float* u, int k) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t path = first + i;
  const int64_t pixel = path / P.spp;
  const int sample = static_cast<int>(path - pixel * P.spp);
  Mt rng = mt_seed(seed_stream(P.seed, static_cast<uint64_t>(pixel), static_cast<uint64_t>(sample)));
  camera_ray(P, static_cast<int>(pixel % P.width), static_cast<int>(pixel / P.width), rng, rays[i]);
  for (int q = 0; q < k; ++q) u[i * k + q] = mt_uniform(rng);
}

// ------------------------------------------------------------- host side

// make_camera_basis (renderer.cpp:334-344) in float, reference order; the
// host compiler runs with -ffp-contract=off.
CameraBasis make_camera_basis(const lsnif_camera& cam, int width, int height) {
  auto normalized = [](float v[3]) {
    const float n2 = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
    if (n2 > 0.0f) {
      const float n = std::sqrt(n2);
      for (int a = 0; a < 3; ++a) v[a] = v[a] / n;
    }
  };
  auto cross = [](const float a[3], const float b[3], float o[3]) {  // Eigen cross
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
  };
  CameraBasis b{};
  for (int a = 0; a < 3; ++a) {
    b.origin[a] = cam.position[a];
    b.forward[a] = cam.look_at[a] - cam.position[a];
  }
  normalized(b.forward);
  cross(b.forward, cam.up, b.right);
  normalized(b.right);
  cross(b.right, b.forward, b.up);
  b.half_h = std::tan(0.5f * cam.vfov_deg * static_cast<float>(M_PI / 180.0));
  b.half_w = b.half_h * static_cast<float>(width) / static_cast<float>(height);
  return b;
}

Params make_params(const lsnif_camera& camera, const lsnif_render_config& cfg) {
  if (cfg.width <= 0 || cfg.height <= 0 || cfg.spp <= 0 || cfg.max_bounces < 0)
    fail(LSNIF_INVALID_ARGUMENT, "render: width, height, spp must be positive and max_bounces >= 0");
  Params P{};
  P.cam = make_camera_basis(camera, cfg.width, cfg.height);
  P.width = cfg.width;
  P.height = cfg.height;
  P.spp = cfg.spp;
  P.max_bounces = cfg.max_bounces;
  P.seed = cfg.seed;
  P.eps_scale = cfg.neural_eps_scale;
  return P;
}

template <typename K, typename... A>
void launch(K kern, int64_t n, cudaStream_t st, const char* what, A... args) {
  if (n <= 0) return;
  kern<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(args...);
  ck(cudaGetLastError(), what);
}

// For kernels bounded by a device-side count (upper bound n): a grid sized
// for the machine, the kernel strides over the real count.
template <typename K, typename... A>
void launch_strided(K kern, int64_t n, cudaStream_t st, const char* what, A... args) {
  if (n <= 0) return;
  kern<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(args...);
  ck(cudaGetLastError(), what);
}

// Path-state buffers of one (scene, stream), grown on demand and reused by
// later renders (a render allocates nothing in the steady state).
struct Workspace {
  std::vector<void*> bufs;
  int64_t cap = 0, shadow_cap = 0;
  int n_inst_cap = 0;
  Paths S{};
  float* diag = nullptr;
  int32_t* h_counts = nullptr;  // pinned copy of the device counters
  void release() {
    for (void* p : bufs) cudaFree(p);
    bufs.clear();
    cap = shadow_cap = 0;
  }
  ~Workspace() {
    release();
    cudaFree(diag);
    cudaFreeHost(h_counts);
  }
  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc(render)");
    bufs.push_back(p);
    return static_cast<T*>(p);
  }
  void ensure(int64_t paths, int slots) {
    const int64_t sh = paths * std::max(slots, 1);
    if (paths <= cap && sh <= shadow_cap) return;
    release();
    S.rays[0] = alloc<lsnif_ray>(paths);
    S.rays[1] = alloc<lsnif_ray>(paths);
    S.slots[0] = alloc<int32_t>(paths);
    S.slots[1] = alloc<int32_t>(paths);
    S.counts = alloc<int32_t>(2 * kMaxDepth);
    S.hits = alloc<lsnif_scene_hit>(paths);
    S.thr = alloc<float>(3 * paths);
    S.rad = alloc<float>(3 * paths);
    S.rng = alloc<uint4>(paths);
    S.shadow_first = alloc<int32_t>(paths);
    S.shadow_n = alloc<int32_t>(paths);
    S.shadow_rays = alloc<lsnif_ray>(sh);
    S.shadow_contrib = alloc<float>(3 * sh);
    S.shadow_hits = alloc<lsnif_scene_hit>(sh);
    cap = paths;
    shadow_cap = sh;
  }
};

void WorkspaceDeleter::operator()(Workspace* w) const { delete w; }

void render(WorkspacePtr& wsp, lsnif_scene scene, const float* world_diag, int n_instances,
            const lsnif_camera& camera, const lsnif_light* lights, int n_lights, const float environment[3],
            const lsnif_render_config& cfg, float* d_image, lsnif_render_stats* stats, cudaStream_t st) {
  Params P = make_params(camera, cfg);
  if (n_lights < 0 || n_lights > kMaxLights || (n_lights > 0 && !lights))
    fail(LSNIF_INVALID_ARGUMENT, "render: 0..32 lights");
  if (!d_image) fail(LSNIF_INVALID_ARGUMENT, "render: null image");
  if (cfg.max_bounces >= kMaxDepth) fail(LSNIF_UNSUPPORTED, "render: max_bounces must be < 128");
  int n_sphere = 0;
  for (int i = 0; i < n_lights; ++i) {
    if (lights[i].type != LSNIF_LIGHT_POINT && lights[i].type != LSNIF_LIGHT_SPHERE)
      fail(LSNIF_INVALID_ARGUMENT, "render: light type must be point or sphere (environment lights go in `environment`)");
    n_sphere += lights[i].type == LSNIF_LIGHT_SPHERE;
    P.lights[i] = lights[i];
  }
  const int64_t draws = 2 + static_cast<int64_t>(cfg.max_bounces + 1) * (2 * n_sphere + 2);
  if (draws > kMaxDraws)
    fail(LSNIF_UNSUPPORTED, "render: more than 227 random draws per path (max_bounces / sphere lights)");
  P.n_lights = n_lights;
  P.n_shadow_slots = std::min(n_lights, kMaxShadows);
  for (int a = 0; a < 3; ++a) P.env[a] = environment ? environment[a] : 0.0f;

  // waves of whole rows (renderer.cpp:458-466 bounds in-flight paths the same way)
  const int64_t row_paths = static_cast<int64_t>(cfg.width) * cfg.spp;
  const int64_t budget = cfg.max_paths_in_flight > 0 ? cfg.max_paths_in_flight : (int64_t(1) << 22);
  const int64_t rows_per_wave = std::max<int64_t>(1, std::min<int64_t>(cfg.height, budget / row_paths));
  const int64_t cap = rows_per_wave * row_paths;
  if (cap * std::max(1, P.n_shadow_slots) > INT32_MAX) fail(LSNIF_INVALID_ARGUMENT, "render: wave too large");

  if (!wsp) wsp.reset(new Workspace());
  Workspace& W = *wsp;
  W.ensure(cap, P.n_shadow_slots);
  if (n_instances > W.n_inst_cap) {
    cudaFree(W.diag);
    W.diag = nullptr;
    ck(cudaMalloc(&W.diag, n_instances * sizeof(float)), "cudaMalloc(render)");
    W.n_inst_cap = n_instances;
  }
  if (!W.h_counts) ck(cudaMallocHost(&W.h_counts, 2 * kMaxDepth * sizeof(int32_t)), "cudaMallocHost");
  if (n_instances > 0)
    ck(cudaMemcpyAsync(W.diag, world_diag, n_instances * sizeof(float), cudaMemcpyHostToDevice, st),
       "cudaMemcpyAsync");
  P.world_diag = W.diag;
  Paths& S = W.S;

  lsnif_render_stats rs{};
  const int waves = static_cast<int>((cfg.height + rows_per_wave - 1) / rows_per_wave);
  for (int wave = 0; wave < waves; ++wave) {
    const int64_t y0 = wave * rows_per_wave;
    const int64_t rows = std::min<int64_t>(rows_per_wave, cfg.height - y0);
    const int64_t n_paths = rows * row_paths;
    rs.paths += n_paths;
    ++rs.waves;
    // The whole wave is enqueued without a host round trip: each bounce's
    // active count lives in S.counts and bounds every kernel on the device.
    ck(cudaMemsetAsync(S.counts, 0, 2 * kMaxDepth * sizeof(int32_t), st), "cudaMemsetAsync");
    launch(camera_kernel, n_paths, st, "camera_kernel", P, S, y0 * row_paths, n_paths);
    int cur = 0;
    for (int depth = 0; depth <= cfg.max_bounces; ++depth) {
      lsnif_api::scene_query_async(scene, S.rays[cur], n_paths, S.counts + depth, LSNIF_QUERY_CLOSEST, S.hits,
                                   st);
      launch_strided(shade_kernel, n_paths, st, "shade_kernel", P, S, cur, depth, depth < cfg.max_bounces ? 1 : 0);
      if (P.n_shadow_slots > 0) {
        lsnif_api::scene_query_async(scene, S.shadow_rays, n_paths * P.n_shadow_slots,
                                     S.counts + kMaxDepth + depth, LSNIF_QUERY_ANY, S.shadow_hits, st);
        launch_strided(shadow_accum_kernel, n_paths, st, "shadow_accum_kernel", S, cur, depth);
      }
      cur ^= 1;
    }
    launch(resolve_kernel, rows * cfg.width, st, "resolve_kernel", P, static_cast<const float*>(S.rad),
           y0 * cfg.width, rows * cfg.width, d_image);
    ck(cudaMemcpyAsync(W.h_counts, S.counts, 2 * kMaxDepth * sizeof(int32_t), cudaMemcpyDeviceToHost, st),
       "cudaMemcpyAsync(counts)");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    for (int d = 0; d <= cfg.max_bounces; ++d) {
      rs.closest_rays += W.h_counts[d];
      rs.shadow_rays += W.h_counts[kMaxDepth + d];
      rs.shadow_slots += static_cast<int64_t>(W.h_counts[d]) * P.n_shadow_slots;
      if (W.h_counts[d] > 0) rs.max_depth_reached = std::max(rs.max_depth_reached, d);
    }
  }
  if (stats) *stats = rs;
}

void debug_paths(const lsnif_camera& camera, const lsnif_render_config& cfg, int64_t first_path,
                 int64_t n, lsnif_ray* d_rays, float* d_uniforms, int k, cudaStream_t st) {
  const Params P = make_params(camera, cfg);
  if (n < 0 || k < 0 || k + 2 > kMaxDraws || first_path < 0)
    fail(LSNIF_INVALID_ARGUMENT, "render_debug_paths: bad range or draw count");
  if (n > 0 && (!d_rays || (k > 0 && !d_uniforms))) fail(LSNIF_INVALID_ARGUMENT, "null output");
  launch(debug_paths_kernel, n, st, "debug_paths_kernel", P, first_path, n, d_rays, d_uniforms, k);
}

}  // namespace lsnif_pt
