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
constexpr int kInferMode = 2;  // MLP decode mode of lsnif_infer_batch (internal)
constexpr int kMaxHitCap = 32;
constexpr int kTileM = 128;  // rays per MMA tile (TMEM lanes)
// MLP rows are binned by their used input width: bin b holds the rows whose
// count * L * F features fit in K_b = 16 (b + 1) columns, so a tile of bin b
// is stored, loaded and multiplied with K_b columns instead of the padded
// input width.
constexpr int kMaxBins = 16;
constexpr uint32_t kBinTileBytes = kTileM * 16 * 2;  // one 16-column slab of a tile

// Byte offset of bin b's tile region when every bin holds cap_tiles tiles.
__device__ __host__ __forceinline__ uint64_t bin_x_offset(int b, int64_t cap_tiles) {
  return static_cast<uint64_t>(b) * (b + 1) / 2 * static_cast<uint64_t>(cap_tiles) * kBinTileBytes;
}

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
  const uint32_t* stop;                // (V+2)^3 bits: occupied cells + the outside border
  int stop_words;
  const uint32_t* stop2;               // (V+2)^3 2-bit codes: 0 free, 1 occupied, 2 border
  int stop2_words;
  int x_stages;                        // MLP X-tile ring depth (set at load from the SMEM budget)
  const uint2* tables[kMaxLevels];     // M entries x 4 binary16 (F <= 4, zero padded)
  int hidden, n_out, n_mat, N3;        // N3: layer-3 MMA width (>= n_out, multiple of 16)
  const uint8_t* w_canon;              // W1 | W2 | W3, UMMA K-major canonical fp16
  uint32_t w1_bytes, w2_bytes, w3_bytes;
  const float* w_f32;                  // w1 | b1 | w2 | b2 | w3 | b3 (decoded fp32, row-major)
  float act_scale, inv_act_scale;      // power of two
  float feat_bound;                    // max |feature| the scale was derived for (max |table entry|)
  float occ_threshold;                 // smallest z with 1/(1+expf(-z)) > 0.5 under the host libm
  const lsnif_material* materials;     // material table (model_io.cpp:159-164)
  int n_materials;
  float z_zero[32];                    // logits of the all-zero input (rays without points)
  float b3[16];                        // output bias, added in fp32 by the decode epilogue
  int n_bins;                          // K1P / 16
  // decode_hit of z_zero with enter = 0, exit = 1 (computed on the device at
  // load): rays with a pair but no point differ only in t_world and accept
  float zero_lt;                       // sigmoid(z_zero[1])
  float zero_normal[3], zero_albedo[3];
  uint32_t zero_flags;                 // OCCLUDED bit | material << shift
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
    const float inv = __frcp_rn(d[a]);  // == 1.0f / d (correctly rounded)
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
    const float inv = __frcp_rn(d[a]);  // == 1.0f / d (correctly rounded)
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

// State of one Amanatides-Woo walk (dda.cpp:40-117) in local unit-cube space.
// The current cell is a linear index into the padded (V+2)^3 stop mask (x
// fastest, voxel.hpp:30-34 order shifted by one), whose non-zero codes are
// the occupied cells (1) and the one-cell border outside the grid (2): one
// SMEM load per step finds both an occupied cell to emit and the walk leaving
// the grid (dda.cpp:112). The query kernel keeps 2-bit / byte codes
// (stop2); the trainer's encode the plain bitmask (stop) with walk_step.
struct Walk {
  float o[3], d[3];    // nudged local origin and local direction
  float t1;
  float tn[3], td[3];  // t_next, t_delta
  int lin[3];          // padded linear-index increment of one step per axis
  uint32_t idx;        // padded linear index of the current cell
  float t0;
  int axis0;           // entry axis of the start cell (-1: origin inside)
  float plane0;        // entry plane of the start cell (dda.cpp:86)
};

// dda.cpp:45-86 (+ renderer.cpp:252-253 world->local): nudge, clip, start
// cell and stepping constants. Returns false when the local ray misses.
template <int VS>
__device__ __forceinline__ bool walk_setup(const DevModel& m, const float wo[3], const float wd[3],
                                           float t_min, Walk& w) {
  const int V = VS ? VS : m.V;
  const int Vp = V + 2;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    w.o[a] = __fmul_rn(__fsub_rn(wo[a], m.mn[a]), m.inv_ext[a]);
    w.d[a] = __fmul_rn(wd[a], m.inv_ext[a]);
  }
  const float fres = static_cast<float>(V);
  const float inv_fres = m.inv_fres;
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // dda.cpp:49-53
    const float scaled = __fmul_rn(w.o[a], fres);
    if (scaled == floorf(scaled)) w.o[a] = __fadd_rn(w.o[a], 1e-7f);
  }
  float t0;
  int entry_axis;
  if (!slab_interval(w.o, w.d, t_min, t0, w.t1, entry_axis)) return false;
  float start[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) start[a] = __fadd_rn(w.o[a], __fmul_rn(t0, w.d[a]));
  const float inf = __int_as_float(0x7f800000);
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // dda.cpp:64-79
    c[a] = iclamp(static_cast<int>(floorf(__fmul_rn(start[a], fres))), 0, V - 1);
    const float da = w.d[a];
    const int stride = a == 0 ? 1 : a == 1 ? Vp : Vp * Vp;
    if (da > 0.0f) {
      w.td[a] = __frcp_rn(__fmul_rn(fres, da));
      // (c + 1) / fres is exact as a product by 1/fres (fres a power of two)
      w.tn[a] = __fadd_rn(t0, __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(c[a] + 1), inv_fres),
                                                  start[a]), da));
      w.lin[a] = stride;
    } else if (da < 0.0f) {
      w.td[a] = -__frcp_rn(__fmul_rn(fres, da));  // == -1 / (fres*da) exactly
      w.tn[a] = __fadd_rn(t0, __fdiv_rn(__fsub_rn(__fmul_rn(static_cast<float>(c[a]), inv_fres),
                                                  start[a]), da));
      w.lin[a] = -stride;
    } else {
      w.td[a] = inf;
      w.tn[a] = inf;
      w.lin[a] = 0;
    }
  }
  // A zero direction would never leave its cell (the reference loops forever);
  // such a walk stops after its start cell.
  if (w.lin[0] == 0 && w.lin[1] == 0 && w.lin[2] == 0) w.t1 = -inf;
  w.idx = static_cast<uint32_t>((c[0] + 1) + Vp * ((c[1] + 1) + Vp * (c[2] + 1)));
  w.t0 = t0;
  w.axis0 = entry_axis;
  w.plane0 = -1.0f;
  if (entry_axis >= 0) {
    const float sa = entry_axis == 0 ? start[0] : entry_axis == 1 ? start[1] : start[2];
    w.plane0 = roundf(__fmul_rn(sa, fres));
  }
  return true;
}

__device__ __forceinline__ bool stop_bit(const uint32_t* stop, uint32_t idx) {
  return (stop[idx >> 5] >> (idx & 31)) & 1u;
}

// One advance (dda.cpp:103-115): argmin of t_next with ties to the lower axis
// (p1: y beats x, p2: z beats the winner), stop when it exceeds t1; step the
// winning axis. Returns false at the t1 exit; `tn` is the new entry t.
__device__ __forceinline__ bool walk_step(Walk& w, float& tn, bool& p1, bool& p2) {
  p1 = w.tn[1] < w.tn[0];
  tn = p1 ? w.tn[1] : w.tn[0];
  p2 = w.tn[2] < tn;
  tn = p2 ? w.tn[2] : tn;
  if (tn > w.t1) return false;
  const bool a0 = !p1 && !p2;
  const bool a1 = p1 && !p2;
  if (a0) w.tn[0] = __fadd_rn(w.tn[0], w.td[0]);
  if (a1) w.tn[1] = __fadd_rn(w.tn[1], w.td[1]);
  if (p2) w.tn[2] = __fadd_rn(w.tn[2], w.td[2]);
  int dl = p1 ? w.lin[1] : w.lin[0];
  dl = p2 ? w.lin[2] : dl;
  w.idx += static_cast<uint32_t>(dl);
  return true;
}

// One advance of walk_step without its t1 test, for walks checked against a
// stop mask whose padded border is all set: the t_next sequence of a walk is
// non-decreasing, so the walk_step loop stops before a stop cell exactly when
// that cell's entry t exceeds t1, and no cell in between emits; the caller
// tests tn > t1 once per stop cell. Any moving walk reaches the border within
// 3 (V + 2) advances; not for a walk with no moving axis (t1 = -inf).
// Returns the step's padded-index increment, which also names the stepped
// axis (the pool code below), so no predicate state is carried around the
// caller's loop.
__device__ __forceinline__ int walk_advance_dl(Walk& w, float& tn) {
  const bool p1 = w.tn[1] < w.tn[0];
  tn = p1 ? w.tn[1] : w.tn[0];
  const bool p2 = w.tn[2] < tn;
  tn = p2 ? w.tn[2] : tn;
  const bool a0 = !p1 && !p2;
  const bool a1 = p1 && !p2;
  if (a0) w.tn[0] = __fadd_rn(w.tn[0], w.td[0]);
  if (a1) w.tn[1] = __fadd_rn(w.tn[1], w.td[1]);
  if (p2) w.tn[2] = __fadd_rn(w.tn[2], w.td[2]);
  int dl = p1 ? w.lin[1] : w.lin[0];
  dl = p2 ? w.lin[2] : dl;
  w.idx += static_cast<uint32_t>(dl);
  return dl;
}

// Trace-kernel stop-code mask size in 32-bit words: one byte per padded cell
// in the 1024-thread configuration, else 2 bits (16-byte multiple).
__host__ __device__ __forceinline__ int trace_mask_words(const DevModel& m, int warps_per_block) {
  return warps_per_block == 32 ? m.stop2_words * 4 : (m.stop2_words + 3) & ~3;
}

// Stop code of a padded cell in a 2-bit code mask (16 cells per word):
// 0 free, 1 occupied (emit), 2 border (the walk left the grid, dda.cpp:112).
__device__ __forceinline__ uint32_t stop_code2(const uint32_t* stop2, uint32_t idx) {
  return (stop2[idx >> 4] >> ((idx & 15u) << 1)) & 3u;
}

// One-byte pool code of a boundary point in the query kernel. The walk
// stores the low byte of the step's padded-index increment (+-1, +-(V+2),
// +-(V+2)^2: distinct low bytes for every power-of-two V <= 64, none in
// 0x80..0x83); the start point stores 0x80 | entry axis, or 0x83 when the
// origin is inside the cell (the "volume" first point, first_is_origin).
// point_axis_code maps either to: bits 0-1 the entry axis (3: volume), bit 2
// set for the start point, whose entry plane is round(start V) (dda.cpp:86);
// a later point crossed the plane nearest to V (o + t d) along the stepped
// axis (dda.cpp:89-95: t is within a few ulps of the exact crossing, far
// below half a cell). The plane is rebuilt from t in the encode, so the
// divergent emit path of the walk is a handful of instructions.
__device__ __forceinline__ uint32_t start_code(int axis0) {
  return axis0 < 0 ? 0x83u : (0x80u | static_cast<uint32_t>(axis0));
}
__device__ __forceinline__ uint32_t point_axis_code(uint32_t code, int V) {
  if ((code & 0xfcu) == 0x80u) return (code & 3u) == 3u ? 3u : ((code & 3u) | 4u);
  const uint32_t vp = static_cast<uint32_t>(V + 2) & 0xffu;
  return (code == 1u || code == 0xffu) ? 0u : ((code == vp || code == ((0u - vp) & 0xffu)) ? 1u : 2u);
}

// Entry point of a pooled boundary point (dda.cpp:90-95, 113): o + t d with
// the entry-axis coordinate snapped to plane / V (axis code as above).
__device__ __forceinline__ void point_from_code(float t, uint32_t code, const float o[3], const float d[3],
                                                float fres, float inv_fres, float p[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) p[a] = __fadd_rn(o[a], __fmul_rn(t, d[a]));
  const uint32_t axis = code & 3u;
  if (axis == 3u) return;
  const float s = __fmul_rn(axis == 0u ? p[0] : axis == 1u ? p[1] : p[2], fres);
  const float plane = (code & 4u) ? roundf(s) : rintf(s);
  const float snapped = __fmul_rn(plane, inv_fres);  // == plane / fres (fres a power of two)
  if (axis == 0u) p[0] = snapped;
  else if (axis == 1u) p[1] = snapped;
  else p[2] = snapped;
}

// Cell coordinates (unpadded, may be -1 or V when outside) of a padded index.
template <int VS>
__device__ __forceinline__ void walk_cell(const DevModel& m, uint32_t idx, int c[3]) {
  const uint32_t Vp = static_cast<uint32_t>((VS ? VS : m.V) + 2);
  const uint32_t q = idx / Vp;
  c[0] = static_cast<int>(idx - q * Vp) - 1;
  c[1] = static_cast<int>(q % Vp) - 1;
  c[2] = static_cast<int>(q / Vp) - 1;
}

// Pool entry of one boundary point: entry t and (axis | plane << 2), axis 3
// marking the origin-inside start point (first_is_origin).
__device__ __forceinline__ uint2 pack_point(float t, int axis, float plane) {
  const uint32_t code = axis < 0 ? 3u : (static_cast<uint32_t>(axis) | (static_cast<uint32_t>(plane) << 2));
  return make_uint2(__float_as_uint(t), code);
}

// Entry point of a pooled boundary point (dda.cpp:90-95, 113): o + t*d with
// the entry-axis coordinate snapped to plane / V.
__device__ __forceinline__ void unpack_point(uint2 e, const float o[3], const float d[3],
                                             float inv_fres, float p[3], bool& volume) {
  const float t = __uint_as_float(e.x);
  const uint32_t axis = e.y & 3u;
#pragma unroll
  for (int a = 0; a < 3; ++a) p[a] = __fadd_rn(o[a], __fmul_rn(t, d[a]));
  volume = axis == 3u;
  const float snapped = __fmul_rn(static_cast<float>(e.y >> 2), inv_fres);  // == plane / fres
  if (axis == 0u) p[0] = snapped;
  else if (axis == 1u) p[1] = snapped;
  else if (axis == 2u) p[2] = snapped;
}

// ---------------------------------------------------------------- encode

constexpr uint32_t kP1 = 2654435761u, kP2 = 805459861u;  // encoding.hpp:19-21

// hash_vertex (encoding.hpp:18-23) reduction
template <bool POW2>
__device__ __forceinline__ uint32_t hash_reduce(const DevModel& m, uint32_t h) {
  if (POW2) return h & m.M_mask;
  return m.M_pow2 ? (h & m.M_mask) : (h % m.M);
}

__device__ __forceinline__ void unpack4(uint2 e, float f[4]) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&e.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&e.y));
  f[0] = a.x;
  f[1] = a.y;
  f[2] = b.x;
  f[3] = b.y;
}

// The interpolation plane axis of a boundary point (encoding.hpp:95-108):
// argmin_a |p_a V - round(p_a V)| with the first minimum winning. The
// entry-axis coordinate is an exact multiple of 1/V (distance 0, the global
// minimum), so the argmin is the first axis whose p_a * V is an integer.
__device__ __forceinline__ int plane_axis_of(const float p[3], float fv) {
  const float s0 = __fmul_rn(p[0], fv), s1 = __fmul_rn(p[1], fv);
  return (s0 == rintf(s0)) ? 0 : (s1 == rintf(s1)) ? 1 : 2;
}

// encode_point_level (encoding.hpp:84-140) for a boundary point: the 4
// in-plane corners. With the plane axis a and free axes b < c, the
// reference's corner order (dx,dy,dz bits, skipping the +1 side of a) is
// (db,dc) = (0,0),(1,0),(0,1),(1,1) and its weight wx*wy*wz = wb*wc exactly
// (the plane factor is 1 - 0). Split into index/weight computation and the
// fp32 accumulation so callers can issue every gather of a point first.
template <bool POW2>
__device__ __forceinline__ void boundary_corners(const DevModel& m, int level, const float p[3], int pa,
                                                 uint32_t idx[4], float w[4]) {
  const int res = m.level_res[level];
  const float fres = static_cast<float>(res);
  const int b = pa == 0 ? 1 : 0;
  const int c = pa == 2 ? 1 : 2;
  const float pa_v = pa == 0 ? p[0] : pa == 1 ? p[1] : p[2];
  const float pb_v = b == 0 ? p[0] : p[1];
  const float pc_v = c == 1 ? p[1] : p[2];
  const int base_a = iclamp(static_cast<int>(roundf(__fmul_rn(pa_v, fres))), 0, res);
  const float ub = __fmul_rn(pb_v, fres), uc = __fmul_rn(pc_v, fres);
  const int base_b = iclamp(static_cast<int>(floorf(ub)), 0, res - 1);
  const int base_c = iclamp(static_cast<int>(floorf(uc)), 0, res - 1);
  const float fb = fclamp(__fsub_rn(ub, static_cast<float>(base_b)), 0.0f, 1.0f);
  const float fc = fclamp(__fsub_rn(uc, static_cast<float>(base_c)), 0.0f, 1.0f);
  const uint32_t Pa = pa == 0 ? 1u : pa == 1 ? kP1 : kP2;
  const uint32_t Pb = b == 0 ? 1u : kP1;
  const uint32_t Pc = c == 1 ? kP1 : kP2;
  const uint32_t ha = static_cast<uint32_t>(base_a) * Pa;
  const uint32_t hb0 = static_cast<uint32_t>(base_b) * Pb, hb1 = hb0 + Pb;
  const uint32_t hc0 = static_cast<uint32_t>(base_c) * Pc, hc1 = hc0 + Pc;
  idx[0] = hash_reduce<POW2>(m, ha ^ hb0 ^ hc0);
  idx[1] = hash_reduce<POW2>(m, ha ^ hb1 ^ hc0);
  idx[2] = hash_reduce<POW2>(m, ha ^ hb0 ^ hc1);
  idx[3] = hash_reduce<POW2>(m, ha ^ hb1 ^ hc1);
  const float wb0 = __fsub_rn(1.0f, fb), wc0 = __fsub_rn(1.0f, fc);
  w[0] = __fmul_rn(wb0, wc0);
  w[1] = __fmul_rn(fb, wc0);
  w[2] = __fmul_rn(wb0, fc);
  w[3] = __fmul_rn(fb, fc);
}

// features[f] = sum_k w[k] * entry_k[f] in corner order, fp32, unfused.
__device__ __forceinline__ void accumulate4(const uint2 ent[4], const float w[4], float feat[4]) {
  feat[0] = feat[1] = feat[2] = feat[3] = 0.0f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float t[4];
    unpack4(ent[k], t);
#pragma unroll
    for (int f = 0; f < 4; ++f) feat[f] = __fadd_rn(feat[f], __fmul_rn(w[k], t[f]));
  }
}

template <bool POW2>
__device__ __forceinline__ void encode_boundary_level(const DevModel& m, int level, const float p[3],
                                                      int pa, float feat[4], uint32_t* hidx) {
  uint32_t idx[4];
  float w[4];
  boundary_corners<POW2>(m, level, p, pa, idx, w);
  const uint2* table = m.tables[level];
  uint2 ent[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) ent[k] = __ldg(table + idx[k]);
  if (hidx) {
#pragma unroll
    for (int k = 0; k < 4; ++k) hidx[k] = idx[k];
  }
  accumulate4(ent, w, feat);
}

// Volume fallback (first point of a ray starting inside an occupied cell):
// all 8 corners, trilinear (encoding.hpp:109-139 with plane_axis = -1).
template <bool POW2>
__device__ __forceinline__ void encode_volume_level(const DevModel& m, int level, const float p[3],
                                                    float feat[4], uint32_t* hidx) {
  const int res = m.level_res[level];
  const float fres = static_cast<float>(res);
  int base[3];
  float frac[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float u = __fmul_rn(p[a], fres);
    base[a] = iclamp(static_cast<int>(floorf(u)), 0, res - 1);
    frac[a] = fclamp(__fsub_rn(u, static_cast<float>(base[a])), 0.0f, 1.0f);
  }
  const uint2* table = m.tables[level];
  uint2 ent[8];
  float w[8];
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    const float wx = dx ? frac[0] : __fsub_rn(1.0f, frac[0]);
    const float wy = dy ? frac[1] : __fsub_rn(1.0f, frac[1]);
    const float wz = dz ? frac[2] : __fsub_rn(1.0f, frac[2]);
    w[corner] = __fmul_rn(__fmul_rn(wx, wy), wz);
    const uint32_t h = static_cast<uint32_t>(base[0] + dx) ^ static_cast<uint32_t>(base[1] + dy) * kP1 ^
                       static_cast<uint32_t>(base[2] + dz) * kP2;
    const uint32_t idx = hash_reduce<POW2>(m, h);
    ent[corner] = __ldg(table + idx);
    if (hidx) hidx[corner] = idx;
  }
  feat[0] = feat[1] = feat[2] = feat[3] = 0.0f;
#pragma unroll
  for (int corner = 0; corner < 8; ++corner) {
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
  return __frcp_rn(__fadd_rn(1.0f, expf(-v)));  // == 1 / (1 + e^-v), correctly rounded
}

// The occlusion decision sigmoid(z0) > 0.5 (renderer.cpp:212) is monotone in
// z0; it is taken as z0 >= occ_threshold, the boundary computed on the host
// with the reference's (correctly rounded) expf, so it does not depend on the
// last-ulp behaviour of the device expf.
// The MLP epilogue splits the decode over the two warps that own a row:
// decode_flags (visibility, t_world, material, accept flags: z0, z1, z8..)
// and decode_normal + decode_albedo (z2..z7); decode_hit is all of them.
// zm points at the n_mat material logits.
__device__ __forceinline__ void decode_flags(float z0, float z1, const float* zm, int n_mat, float occ_threshold,
                                             float enter, float exit, float t_min, float t_max, int mode,
                                             bool pair_flag, uint32_t& flags_material, float& t_world) {
  const float lt = sigmoid_ref(z1);
  const bool occluded = z0 >= occ_threshold;
  const float tw = __fadd_rn(enter, __fmul_rn(lt, __fsub_rn(exit, enter)));
  // (loops unrolled to the compile-time maximum so the logits stay in registers)
  constexpr int kMaxMat = 8;
  float zmax = zm[0];
#pragma unroll
  for (int k = 1; k < kMaxMat; ++k)
    if (k < n_mat) zmax = (zm[k] > zmax) ? zm[k] : zmax;
  float e[kMaxMat];
  float sum = 0.0f;
#pragma unroll
  for (int k = 0; k < kMaxMat; ++k)
    if (k < n_mat) {
      e[k] = expf(__fsub_rn(zm[k], zmax));
      sum = __fadd_rn(sum, e[k]);
    }
  int arg = 0;
  float best = __fdiv_rn(e[0], sum);
#pragma unroll
  for (int k = 1; k < kMaxMat; ++k)
    if (k < n_mat) {
      const float pk = __fdiv_rn(e[k], sum);
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
  flags_material = flags | (static_cast<uint32_t>(arg) << LSNIF_HIT_MATERIAL_SHIFT);
  t_world = tw;
}

__device__ __forceinline__ void decode_normal(float n0, float n1, float n2, float normal[3]) {
  const float len = sqrtf(__fadd_rn(__fadd_rn(__fmul_rn(n0, n0), __fmul_rn(n1, n1)), __fmul_rn(n2, n2)));
  if (len > 1e-12f) {
    normal[0] = __fdiv_rn(n0, len);
    normal[1] = __fdiv_rn(n1, len);
    normal[2] = __fdiv_rn(n2, len);
  } else {
    normal[0] = normal[1] = normal[2] = 0.0f;
  }
}

__device__ __forceinline__ void decode_albedo(float z5, float z6, float z7, float albedo[3]) {
  albedo[0] = sigmoid_ref(z5);
  albedo[1] = sigmoid_ref(z6);
  albedo[2] = sigmoid_ref(z7);
}

// Reduced-instruction decode for the MLP epilogue (the outputs the parity
// contract takes within a tolerance: t_world, normal, albedo; SURVEY.md
// App. B): sigmoid from the hardware exp2 / reciprocal (a few ulp), the
// normal scaled by a hardware reciprocal square root, and the material as
// the first maximum of the logits (softmax is monotone: the same index as
// the reference's first maximum of the probabilities unless two logits
// round to the same probability). The visibility decision is unchanged
// (z0 >= occ_threshold).
__device__ __forceinline__ float sigmoid_fast(float v) {
  return __frcp_rn(__fadd_rn(1.0f, exp2f(__fmul_rn(v, -1.4426950408889634f))));
}

__device__ __forceinline__ void decode_flags_fast(float z0, float z1, const float* zm, int n_mat,
                                                  float occ_threshold, float enter, float exit, float t_min,
                                                  float t_max, int mode, uint32_t& flags_material,
                                                  float& t_world) {
  const float lt = sigmoid_fast(z1);
  const bool occluded = z0 >= occ_threshold;
  const float tw = __fadd_rn(enter, __fmul_rn(lt, __fsub_rn(exit, enter)));
  constexpr int kMaxMat = 8;
  int arg = 0;
  float best = zm[0];
#pragma unroll
  for (int k = 1; k < kMaxMat; ++k)
    if (k < n_mat && zm[k] > best) {
      best = zm[k];
      arg = k;
    }
  // kInferMode (lsnif_infer_batch): a bare NeuralHit, no pair / accept flags
  uint32_t flags = mode == kInferMode ? 0u : LSNIF_HIT_PAIR;
  if (occluded) {
    flags |= LSNIF_HIT_OCCLUDED;
    const bool accept = (mode == LSNIF_QUERY_CLOSEST) ? !(tw >= t_max || tw < t_min)
                                                      : (tw >= t_min && tw <= t_max);
    if (accept && mode != kInferMode) flags |= LSNIF_HIT_ACCEPTED;
  }
  flags_material = flags | (static_cast<uint32_t>(arg) << LSNIF_HIT_MATERIAL_SHIFT);
  t_world = tw;
}

__device__ __forceinline__ void decode_normal_fast(float n0, float n1, float n2, float normal[3]) {
  const float len2 = __fadd_rn(__fadd_rn(__fmul_rn(n0, n0), __fmul_rn(n1, n1)), __fmul_rn(n2, n2));
  const float inv = len2 > 1e-24f ? rsqrtf(len2) : 0.0f;
  normal[0] = __fmul_rn(n0, inv);
  normal[1] = __fmul_rn(n1, inv);
  normal[2] = __fmul_rn(n2, inv);
}

__device__ __forceinline__ void decode_albedo_fast(float z5, float z6, float z7, float albedo[3]) {
  albedo[0] = sigmoid_fast(z5);
  albedo[1] = sigmoid_fast(z6);
  albedo[2] = sigmoid_fast(z7);
}

__device__ __forceinline__ void decode_hit(const float* z, int n_mat, float occ_threshold,
                                           float enter, float exit, float t_min, float t_max,
                                           int mode, bool pair_flag, lsnif_hit& h) {
  decode_flags(z[0], z[1], z + 8, n_mat, occ_threshold, enter, exit, t_min, t_max, mode, pair_flag,
               h.flags_material, h.t_world);
  decode_normal(z[2], z[3], z[4], h.normal);
  decode_albedo(z[5], z[6], z[7], h.albedo);
}

// decode_hit(m.z_zero, ...) for a pair without boundary points (the all-zero
// MLP input): the constant heads come from the load-time decode, only
// t_world = enter + lt (exit - enter) and the accept rule depend on the ray.
__device__ __forceinline__ void decode_zero(const DevModel& m, float enter, float exit, float t_min,
                                            float t_max, int mode, lsnif_hit& h) {
  const float tw = __fadd_rn(enter, __fmul_rn(m.zero_lt, __fsub_rn(exit, enter)));
  uint32_t flags = m.zero_flags | LSNIF_HIT_PAIR;
  if (flags & LSNIF_HIT_OCCLUDED) {
    const bool accept = (mode == LSNIF_QUERY_CLOSEST) ? !(tw >= t_max || tw < t_min)
                                                      : (tw >= t_min && tw <= t_max);
    if (accept) flags |= LSNIF_HIT_ACCEPTED;
  }
  h.flags_material = flags;
  h.t_world = tw;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    h.normal[a] = m.zero_normal[a];
    h.albedo[a] = m.zero_albedo[a];
  }
}

__device__ __forceinline__ void store_hit(lsnif_hit* dst, const lsnif_hit& h) {
  float4* d4 = reinterpret_cast<float4*>(dst);
  d4[0] = make_float4(__uint_as_float(h.flags_material), h.t_world, h.normal[0], h.normal[1]);
  d4[1] = make_float4(h.normal[2], h.albedo[0], h.albedo[1], h.albedo[2]);
}

// ------------------------------------------------------------ wire form

// Packed 16 B result (lsnif_hit_wire, include/lsnif_gpu.h). The normal is
// the octahedral map of the unit vector (|x| + |y| + |z| = 1 projection,
// lower hemisphere folded) quantised to 2 x snorm16; the albedo 3 x unorm10.
// Host and device share the code (the host decode expands query results).
__host__ __device__ __forceinline__ float wire_sign(float v) { return v >= 0.0f ? 1.0f : -1.0f; }

__host__ __device__ __forceinline__ uint32_t wire_snorm16(float v) {
  v = v < -1.0f ? -1.0f : (v > 1.0f ? 1.0f : v);
  const int q = static_cast<int>(rintf(v * 32767.0f));
  return static_cast<uint32_t>(q) & 0xffffu;
}

__host__ __device__ __forceinline__ uint32_t wire_unorm10(float v) {
  v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
  return static_cast<uint32_t>(rintf(v * 1023.0f));
}

__host__ __device__ __forceinline__ void wire_pack_normal_albedo(const float n[3], const float a[3],
                                                                 uint32_t& normal_oct, uint32_t& albedo) {
  const float l1 = fabsf(n[0]) + fabsf(n[1]) + fabsf(n[2]);
  uint32_t zero = 0u;
  float u = 0.0f, v = 0.0f;
  if (l1 > 0.0f) {
    u = n[0] / l1;
    v = n[1] / l1;
    if (n[2] < 0.0f) {
      const float uu = (1.0f - fabsf(v)) * wire_sign(u);
      const float vv = (1.0f - fabsf(u)) * wire_sign(v);
      u = uu;
      v = vv;
    }
  } else {
    zero = LSNIF_WIRE_ZERO_NORMAL;
  }
  normal_oct = wire_snorm16(u) | (wire_snorm16(v) << 16);
  albedo = wire_unorm10(a[0]) | (wire_unorm10(a[1]) << 10) | (wire_unorm10(a[2]) << 20) | zero;
}

__host__ __device__ __forceinline__ void wire_unpack(const lsnif_hit_wire& w, lsnif_hit& h) {
  h.flags_material = w.flags_material;
  h.t_world = w.t_world;
  const float u = fmaxf(static_cast<float>(static_cast<int16_t>(w.normal_oct & 0xffffu)) / 32767.0f, -1.0f);
  const float v = fmaxf(static_cast<float>(static_cast<int16_t>(w.normal_oct >> 16)) / 32767.0f, -1.0f);
  if (w.albedo_unorm & LSNIF_WIRE_ZERO_NORMAL) {
    h.normal[0] = h.normal[1] = h.normal[2] = 0.0f;
  } else {
    float x = u, y = v;
    const float z = 1.0f - fabsf(u) - fabsf(v);
    if (z < 0.0f) {
      x = (1.0f - fabsf(v)) * wire_sign(u);
      y = (1.0f - fabsf(u)) * wire_sign(v);
    }
    const float len = sqrtf(x * x + y * y + z * z);
    h.normal[0] = x / len;
    h.normal[1] = y / len;
    h.normal[2] = z / len;
  }
  for (int c = 0; c < 3; ++c) h.albedo[c] = static_cast<float>((w.albedo_unorm >> (10 * c)) & 1023u) / 1023.0f;
}

__device__ __forceinline__ void store_hit_wire(lsnif_hit_wire* dst, const lsnif_hit& h) {
  uint32_t no, al;
  wire_pack_normal_albedo(h.normal, h.albedo, no, al);
  *reinterpret_cast<uint4*>(dst) = make_uint4(h.flags_material, __float_as_uint(h.t_world), no, al);
}

// One result into the caller's array: the 32 B parity record or the 16 B
// wire record.
__device__ __forceinline__ void store_result(void* out, int64_t i, bool wire, const lsnif_hit& h) {
  if (wire)
    store_hit_wire(static_cast<lsnif_hit_wire*>(out) + i, h);
  else
    store_hit(static_cast<lsnif_hit*>(out) + i, h);
}

// Byte offset of element (row, col) of an fp16 operand tile in the UMMA
// K-major no-swizzle canonical layout: 8x8 core matrices (128 B), rows
// grouped by 8 at stride 128 B (SBO), K chunks of 8 at stride rows*16 B (LBO).
// Within a K chunk the row term (row >> 3) * 128 + (row & 7) * 16 is row * 16.
__device__ __host__ __forceinline__ uint32_t canon_offset(int row, int col, int rows) {
  return static_cast<uint32_t>(((col >> 3) * rows + row) * 16 + (col & 7) * 2);
}

}  // namespace lsnif_dev
