// Device-side building blocks of the LSNIF query path (sm_100a).
//
// Every function here is used by BOTH the product kernels and the
// bit-exactness probe (lsnif_debug_traverse), so the probe's bit-exact
// comparison against the CPU oracle certifies the product code.
//
// Float semantics: the reference evaluates `a + b * c` with two roundings in
// the parity contract; nvcc would contract those into
// FMAs, so every such expression is spelled with __fmul_rn / __fadd_rn /
// __fsub_rn. Divisions are IEEE (-prec-div=true); floorf/roundf match
// std::floor/std::round. Never compile this with --use_fast_math.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "lsnif_gpu.h"

namespace lsnif_dev {

constexpr int kMaxLevels = 4;
constexpr int kMaxHitCap = 32;
constexpr int kTileM = 128;  // rays per MMA tile (TMEM lanes)

// Per-model constants, passed by value to every kernel (in the constant
// parameter bank). Pointers are device memory owned by the model.
struct DevModel {
  float mn[3], mx[3], inv_ext[3];
  int V;            // occupancy resolution (power of two)
  float fres, inv_fres;
  int H, L, F, LF;  // hit cap, levels, feature dim, L*F
  int K1;           // H*L*F (input width); column K1 holds the bias constant
  int K1P;          // K1 + 1 rounded up to 16
  uint32_t M, M_mask;
  int M_pow2;
  int level_res[kMaxLevels];
  const uint32_t* occ;                 // V^3/32 words
  const uint2* tables[kMaxLevels];     // M entries x 4 binary16 (F <= 4, zero padded)
  int hidden, n_out, n_mat, N3;        // N3: layer-3 MMA width (>= n_out, multiple of 16)
  const uint8_t* w_canon;              // W1 | W2 | W3, UMMA K-major canonical fp16
  uint32_t w1_bytes, w2_bytes, w3_bytes;
  const float* w_f32;                  // w1 | b1 | w2 | b2 | w3 | b3 (decoded fp32, row-major)
  float act_scale, inv_act_scale;      // power of two
  float occ_threshold;                 // smallest z with 1/(1+expf(-z)) > 0.5 under the host libm
  float z_zero[32];                    // logits of the all-zero input (rays without points)
};

// Row bookkeeping for rays that go through the MLP.
struct RowMeta {
  int32_t ray;
  float enter, exit, t_min, t_max;
  int32_t pad[3];
};
static_assert(sizeof(RowMeta) == 32, "RowMeta is 32 B");

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ float smax(float a, float b) { return (a < b) ? b : a; }
__device__ __forceinline__ float smin(float a, float b) { return (b < a) ? b : a; }
__device__ __forceinline__ int iclamp(int v, int lo, int hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}
__device__ __forceinline__ float fclamp(float v, float lo, float hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

// ------------------------------------------------------- pair / AABB clip

// ray_aabb_intersect (geometry.cpp:9-28) on the model frame box, with the
// pair-emission rule of collect_pairs (renderer.cpp:165-172): t_max = inf for
// the interval, pair kept iff enter < ray.t_max.
__device__ __forceinline__ bool frame_interval(const DevModel& m, const float o[3],
                                               const float d[3], float t_min, float t_max,
                                               float& enter, float& exit) {
  float t0 = t_min;
  float t1 = __int_as_float(0x7f800000);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0f) {
      if (o[a] < m.mn[a] || o[a] > m.mx[a]) return false;
      continue;
    }
    const float inv = __fdiv_rn(1.0f, d[a]);
    float ta = __fmul_rn(__fsub_rn(m.mn[a], o[a]), inv);
    float tb = __fmul_rn(__fsub_rn(m.mx[a], o[a]), inv);
    if (ta > tb) {
      const float s = ta;
      ta = tb;
      tb = s;
    }
    t0 = smax(t0, ta);
    t1 = smin(t1, tb);
    if (t0 > t1) return false;
  }
  enter = t0;
  exit = t1;
  return t0 < t_max;
}

// ------------------------------------------------------------------- DDA

// State of one Amanatides-Woo walk (dda.cpp:40-117) in local unit-cube space.
struct DdaState {
  float o[3], d[3];
  float t1;
  float t_next[3], t_delta[3];
  int cell[3];
  int entry_axis;
  float entry_t, entry_plane;
};

// dda.cpp:14-36 slab_interval
__device__ __forceinline__ bool slab_interval(const float o[3], const float d[3], float t_min,
                                              float& t0, float& t1, int& enter_axis) {
  t0 = t_min;
  t1 = __int_as_float(0x7f800000);
  enter_axis = -1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0f) {
      if (o[a] < 0.0f || o[a] > 1.0f) return false;
      continue;
    }
    const float inv = __fdiv_rn(1.0f, d[a]);
    float ta = __fmul_rn(__fsub_rn(0.0f, o[a]), inv);
    float tb = __fmul_rn(__fsub_rn(1.0f, o[a]), inv);
    if (ta > tb) {
      const float s = ta;
      ta = tb;
      tb = s;
    }
    if (ta > t0) {
      t0 = ta;
      enter_axis = a;
    }
    if (tb < t1) t1 = tb;
    if (t0 > t1) return false;
  }
  return true;
}

// dda.cpp:45-86: world->local (renderer.cpp:252-253), plane nudge, clip,
// start cell and stepping constants. Returns false when the local ray misses.
__device__ __forceinline__ bool dda_setup(const DevModel& m, const float wo[3], const float wd[3],
                                          float t_min, DdaState& s) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    s.o[a] = __fmul_rn(__fsub_rn(wo[a], m.mn[a]), m.inv_ext[a]);
    s.d[a] = __fmul_rn(wd[a], m.inv_ext[a]);
  }
  const float fres = m.fres;
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // dda.cpp:49-53
    const float scaled = __fmul_rn(s.o[a], fres);
    if (scaled == floorf(scaled)) s.o[a] = __fadd_rn(s.o[a], 1e-7f);
  }
  float t0;
  int entry_axis;
  if (!slab_interval(s.o, s.d, t_min, t0, s.t1, entry_axis)) return false;
  float start[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) start[a] = __fadd_rn(s.o[a], __fmul_rn(t0, s.d[a]));
  const float inf = __int_as_float(0x7f800000);
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // dda.cpp:64-79
    const int c = iclamp(static_cast<int>(floorf(__fmul_rn(start[a], fres))), 0, m.V - 1);
    s.cell[a] = c;
    const float da = s.d[a];
    if (da > 0.0f) {
      s.t_delta[a] = __fdiv_rn(1.0f, __fmul_rn(fres, da));
      // (c + 1) / fres is exact as a product by 1/fres (fres a power of two)
      s.t_next[a] = __fadd_rn(t0, __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(c + 1), m.inv_fres),
                                                      start[a]), da));
    } else if (da < 0.0f) {
      s.t_delta[a] = __fdiv_rn(-1.0f, __fmul_rn(fres, da));
      s.t_next[a] = __fadd_rn(t0, __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(c), m.inv_fres),
                                                      start[a]), da));
    } else {
      s.t_delta[a] = inf;
      s.t_next[a] = inf;
    }
  }
  s.entry_t = t0;
  s.entry_axis = entry_axis;
  s.entry_plane = -1.0f;
  if (entry_axis >= 0) {
    const float sa = entry_axis == 0 ? start[0] : entry_axis == 1 ? start[1] : start[2];
    s.entry_plane = roundf(__fmul_rn(sa, fres));
  }
  return true;
}

__device__ __forceinline__ bool occ_test(const uint32_t* occ, int V, int x, int y, int z) {
  const uint32_t i = static_cast<uint32_t>(x) + static_cast<uint32_t>(V) *
                     (static_cast<uint32_t>(y) + static_cast<uint32_t>(V) * static_cast<uint32_t>(z));
  return (occ[i >> 5] >> (i & 31)) & 1u;
}

// The entry point of the current cell (dda.cpp:90-95 + 113): o + entry_t*d
// with the entry-axis coordinate snapped to entry_plane / V. The reference
// computes entry_point at every step; it is a pure function of entry_t, so
// it is evaluated only when emitted.
__device__ __forceinline__ void dda_entry_point(const DdaState& s, float inv_fres, float p[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) p[a] = __fadd_rn(s.o[a], __fmul_rn(s.entry_t, s.d[a]));
  if (s.entry_axis >= 0) {
    const float snapped = __fmul_rn(s.entry_plane, inv_fres);  // == entry_plane / fres
    if (s.entry_axis == 0) p[0] = snapped;
    else if (s.entry_axis == 1) p[1] = snapped;
    else p[2] = snapped;
  }
}

// One advance (dda.cpp:103-115). Returns false when the walk ends.
__device__ __forceinline__ bool dda_advance(DdaState& s, int V) {
  int axis = 0;
  float tn = s.t_next[0];
  if (s.t_next[1] < tn) { axis = 1; tn = s.t_next[1]; }
  if (s.t_next[2] < tn) { axis = 2; tn = s.t_next[2]; }
  if (tn > s.t1) return false;
  s.entry_t = tn;
  const float da = axis == 0 ? s.d[0] : axis == 1 ? s.d[1] : s.d[2];
  const int ca = axis == 0 ? s.cell[0] : axis == 1 ? s.cell[1] : s.cell[2];
  const int step = da > 0.0f ? 1 : -1;  // t_next finite implies d != 0
  s.entry_plane = static_cast<float>(step > 0 ? ca + 1 : ca);
  const int nc = ca + step;
  if (nc < 0 || nc >= V) return false;
  s.entry_axis = axis;
  if (axis == 0) { s.cell[0] = nc; s.t_next[0] = __fadd_rn(s.t_next[0], s.t_delta[0]); }
  else if (axis == 1) { s.cell[1] = nc; s.t_next[1] = __fadd_rn(s.t_next[1], s.t_delta[1]); }
  else { s.cell[2] = nc; s.t_next[2] = __fadd_rn(s.t_next[2], s.t_delta[2]); }
  return true;
}

// ---------------------------------------------------------------- encode

// hash_vertex (encoding.hpp:18-23)
__device__ __forceinline__ uint32_t hash_vertex(const DevModel& m, int x, int y, int z) {
  const uint32_t h = static_cast<uint32_t>(x) ^ static_cast<uint32_t>(y) * 2654435761u ^
                     static_cast<uint32_t>(z) * 805459861u;
  return m.M_pow2 ? (h & m.M_mask) : (h % m.M);
}

__device__ __forceinline__ void unpack4(uint2 e, float f[4]) {
  const __half2 a = *reinterpret_cast<const __half2*>(&e.x);
  const __half2 b = *reinterpret_cast<const __half2*>(&e.y);
  f[0] = __low2float(a);
  f[1] = __high2float(a);
  f[2] = __low2float(b);
  f[3] = __high2float(b);
}

// encode_point_level (encoding.hpp:84-140): features[f] for one point on one
// level, fp32 accumulation in corner order 0..7. `hidx` (nullable) receives
// the hashed indices in visit order (debug probe).
__device__ __forceinline__ void encode_point_level(const DevModel& m, int level, const float p[3],
                                                   bool volume, float feat[4], uint32_t* hidx) {
  const int res = m.level_res[level];
  const float fres = static_cast<float>(res);
  float u[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) u[a] = __fmul_rn(p[a], fres);
  int plane_axis = -1;
  if (!volume) {
    float best = 3.402823466e38f;
    const float fv = static_cast<float>(m.V);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float scaled = __fmul_rn(p[a], fv);
      const float dist = fabsf(__fsub_rn(scaled, roundf(scaled)));
      if (dist < best) {
        best = dist;
        plane_axis = a;
      }
    }
  }
  int base[3];
  float frac[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a == plane_axis) {
      base[a] = iclamp(static_cast<int>(roundf(u[a])), 0, res);
      frac[a] = 0.0f;
    } else {
      base[a] = iclamp(static_cast<int>(floorf(u[a])), 0, res - 1);
      frac[a] = fclamp(__fsub_rn(u[a], static_cast<float>(base[a])), 0.0f, 1.0f);
    }
  }
  const uint2* table = m.tables[level];
  // Issue all gathers first (up to 8 independent 8-byte loads in flight).
  uint2 ent[8];
  float w[8];
  int cnt = 0;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const bool skip = (plane_axis == 0 && dx) || (plane_axis == 1 && dy) || (plane_axis == 2 && dz);
    const float wx = dx ? frac[0] : __fsub_rn(1.0f, frac[0]);
    const float wy = dy ? frac[1] : __fsub_rn(1.0f, frac[1]);
    const float wz = dz ? frac[2] : __fsub_rn(1.0f, frac[2]);
    w[corner] = __fmul_rn(__fmul_rn(wx, wy), wz);
    const uint32_t idx = hash_vertex(m, base[0] + dx, base[1] + dy, base[2] + dz);
    if (!skip) {
      ent[corner] = __ldg(table + idx);
      if (hidx) hidx[cnt] = idx;
      ++cnt;
    } else {
      ent[corner] = make_uint2(0u, 0u);
    }
  }
  feat[0] = feat[1] = feat[2] = feat[3] = 0.0f;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const bool skip = (plane_axis == 0 && dx) || (plane_axis == 1 && dy) || (plane_axis == 2 && dz);
    if (skip) continue;
    float t[4];
    unpack4(ent[corner], t);
#pragma unroll
    for (int f = 0; f < 4; ++f) feat[f] = __fadd_rn(feat[f], __fmul_rn(w[corner], t[f]));
  }
}

// ---------------------------------------------------------------- decode

// apply_heads (mlp.hpp:80-94) + NeuralHit decode (renderer.cpp:211-223) +
// accept rule (renderer.cpp:281-284 closest / 317-320 any).
__device__ __forceinline__ float sigmoid_ref(float v) {
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-v)));
}

// The occlusion decision sigmoid(z0) > 0.5 (renderer.cpp:212) is monotone in
// z0; it is taken as z0 >= occ_threshold, the boundary computed on the host
// with the reference's (correctly rounded) expf, so it does not depend on the
// last-ulp behaviour of the device expf.
__device__ __forceinline__ void decode_hit(const float* z, int n_mat, float occ_threshold,
                                           float enter, float exit, float t_min, float t_max,
                                           int mode, bool pair_flag, lsnif_hit& h) {
  const float lt = sigmoid_ref(z[1]);
  const bool occluded = z[0] >= occ_threshold;
  const float tw = __fadd_rn(enter, __fmul_rn(lt, __fsub_rn(exit, enter)));
  const float n0 = z[2], n1 = z[3], n2 = z[4];
  const float len = sqrtf(__fadd_rn(__fadd_rn(__fmul_rn(n0, n0), __fmul_rn(n1, n1)), __fmul_rn(n2, n2)));
  if (len > 1e-12f) {
    h.normal[0] = __fdiv_rn(n0, len);
    h.normal[1] = __fdiv_rn(n1, len);
    h.normal[2] = __fdiv_rn(n2, len);
  } else {
    h.normal[0] = h.normal[1] = h.normal[2] = 0.0f;
  }
  h.albedo[0] = sigmoid_ref(z[5]);
  h.albedo[1] = sigmoid_ref(z[6]);
  h.albedo[2] = sigmoid_ref(z[7]);
  float zmax = z[8];
  for (int k = 1; k < n_mat; ++k) zmax = (z[8 + k] > zmax) ? z[8 + k] : zmax;
  float sum = 0.0f;
  for (int k = 0; k < n_mat; ++k) sum = __fadd_rn(sum, expf(__fsub_rn(z[8 + k], zmax)));
  int arg = 0;
  float best = __fdiv_rn(expf(__fsub_rn(z[8], zmax)), sum);
  for (int k = 1; k < n_mat; ++k) {
    const float pk = __fdiv_rn(expf(__fsub_rn(z[8 + k], zmax)), sum);
    if (pk > best) {
      best = pk;
      arg = k;
    }
  }
  uint32_t flags = pair_flag ? LSNIF_HIT_PAIR : 0u;
  if (occluded) {
    flags |= LSNIF_HIT_OCCLUDED;
    const bool accept = (mode == LSNIF_QUERY_CLOSEST) ? !(tw >= t_max || tw < t_min)
                                                      : (tw >= t_min && tw <= t_max);
    if (accept && pair_flag) flags |= LSNIF_HIT_ACCEPTED;
  }
  h.flags_material = flags | (static_cast<uint32_t>(arg) << LSNIF_HIT_MATERIAL_SHIFT);
  h.t_world = tw;
}

__device__ __forceinline__ void store_hit(lsnif_hit* dst, const lsnif_hit& h) {
  float4* d4 = reinterpret_cast<float4*>(dst);
  d4[0] = make_float4(__uint_as_float(h.flags_material), h.t_world, h.normal[0], h.normal[1]);
  d4[1] = make_float4(h.normal[2], h.albedo[0], h.albedo[1], h.albedo[2]);
}

// Byte offset of element (row, col) of an fp16 operand tile in the UMMA
// K-major no-swizzle canonical layout: 8x8 core matrices (128 B), rows
// grouped by 8 at stride 128 B (SBO), K chunks of 8 at stride rows*16 B (LBO).
__device__ __host__ __forceinline__ uint32_t canon_offset(int row, int col, int rows) {
  return static_cast<uint32_t>((col >> 3) * rows * 16 + (row >> 3) * 128 + (row & 7) * 16 + (col & 7) * 2);
}

}  // namespace lsnif_dev
