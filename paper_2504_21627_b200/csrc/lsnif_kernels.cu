// LSNIF query kernels for sm_100a.
//
//  trace_encode_kernel<DEBUG>  one thread per ray: frame-box pair test,
//      3D-DDA over the SMEM-resident stop codes (points pooled per warp in
//      SMEM), then a warp-cooperative encode of the pooled points
//      (full SIMT efficiency regardless of per-ray point counts). Rays with
//      >= 1 point get a compacted row of the fp16 MLP operand X, written in
//      the UMMA canonical tile layout; other rays are answered directly.
//      DEBUG=true writes the bit-exactness probe instead of X.
//  mlp_tc_kernel   per 128-row tile: bulk-copy X into SMEM, three
//      tcgen05.mma layers (fp16 x fp16 -> fp32 in TMEM, biases folded in as
//      a constant operand column), leaky-ReLU epilogues TMEM -> regs -> TMEM
//      (half2), head decode + accept rule in the last epilogue, results
//      scattered to the caller's hit array.
//  infer_pack_kernel  lsnif_infer_batch's columns -> X tiles for mlp_tc_kernel.
//  infer_f32_kernel  fp32 CUDA-core infer_batch (renderer.cpp:183-226), the
//      reference summation order (validation and out-of-range fallback).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "lsnif_device.cuh"
#include "lsnif_internal.hpp"
#include "tc_ptx.cuh"

namespace lsnif_dev {

// ======================================================= trace + encode

// Persistent: each block loads the stop codes once; its warps claim 32-ray
// batches. Per warp: DDA per lane (points -> 5-byte pool entries), then a
// warp-cooperative encode of all pooled points. LS/FS: compile-time
// level/feature counts (0 = read from the model); POW2: M is a power of two.
// TW: warps per block. Every block holds one SMEM copy of the stop mask, so
// large blocks leave more of the unified L1 to the hash-table gathers and fill
// fewer masks (TW = 32: one 1024-thread block per SM, for launches of many
// waves); launches of about one wave use TW = 8, where 1024-thread blocks
// would leave SMs idle (profiles/experiments: C2 primary TW 4/8/16/32 =
// 0.144/0.140/0.138/0.135 ms, C2 shadow 0.041/0.039/0.043/0.048 ms).
template <bool DEBUG, int LS, int FS, bool POW2, int VS, int TW>
__global__ void __launch_bounds__(32 * TW, 32 / TW) trace_encode_kernel(const TraceParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  const DevModel& m = P.m;
  const int L = LS ? LS : m.L;
  const int F = FS ? FS : m.F;
  const int LF = L * F;
  const int H = m.H;
  const int V = VS ? VS : m.V;
  const int code_words = m.stop2_words;
  // the MLP kernel (launched as a programmatic dependent) may start its
  // prologue while this grid runs; it waits for our completion before reading
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // a chunk past the device-side ray count: nothing to trace
  if (P.n_dev && P.offset >= static_cast<int64_t>(*P.n_dev)) return;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // point pool per warp: entry t (fp32) and a one-byte code (start_code /
  // the step's index increment, point_axis_code) in separate arrays, H x 32
  // each (5 bytes per point)
  using code_t = uint8_t;
  // stop codes in SMEM (0 free, 1 occupied, 2 border): 2 bits per padded
  // cell, or (1024-thread blocks, one per SM) one byte per cell, which turns
  // the per-step test into a byte load
  constexpr bool kByteMask = TW == 32;
  const int mask_words = trace_mask_words(m, TW);
  float4* lane_ray = reinterpret_cast<float4*>(smem + mask_words) + warp * 64;
  float* pool_t = reinterpret_cast<float*>(smem + mask_words + TW * 64 * 4) + warp * (H * 32);
  code_t* pool_c = reinterpret_cast<code_t*>(pool_t - warp * (H * 32) + TW * H * 32) + warp * (H * 32);
  auto pool_put = [&](int i, uint2 e) {
    pool_t[i] = __uint_as_float(e.x);
    pool_c[i] = static_cast<code_t>(e.y);
  };
  auto pool_get = [&](int i) -> uint2 { return make_uint2(__float_as_uint(pool_t[i]), pool_c[i]); };
  const float scale = m.act_scale;
  uint32_t st_pair = 0, st_rows = 0, st_pts = 0, st_vol = 0;  // query statistics
  const int64_t n_rays = P.n_dev ? max(static_cast<int64_t>(0), min(P.n, static_cast<int64_t>(*P.n_dev) - P.offset))
                                 : P.n;
  const int64_t nwb = (n_rays + 31) / 32;  // 32-ray warp batches, fetched dynamically

  // Each warp claims 32-ray batches from a global counter; the next claim
  // and the next batch's ray loads are issued before the current batch is
  // traversed (software pipelining), so warps never wait on each other. The
  // first claim and ray loads overlap the stop-mask fill (small launches are
  // latency-bound: C2 shadow rays 51 -> 41 us). A static first batch
  // (block x 4 + warp) is no better there and costs C3 4%.
  // The claim is split: the atomic is issued at the top of a batch (the
  // reservation point is unchanged, so batches stay balanced across warps)
  // and its result is broadcast after the DDA, when the round trip of the
  // contended same-address atomic is long complete (ncu: the broadcast right
  // behind the atomic was the top stall, 13% of samples on C2); the next
  // batch's rays then load during the encode.
  unsigned int* const ctr = reinterpret_cast<unsigned int*>(P.batch_counter);
  unsigned int pending = 0;
  auto issue_claim = [&]() {
    if (lane == 0) pending = atomicAdd(ctr, 1u);
  };
  auto claimed = [&]() -> int64_t { return static_cast<int64_t>(__shfl_sync(0xffffffffu, pending, 0)); };
  float4 nra = make_float4(0, 0, 0, 0), nrb = nra;
  auto load_ray = [&](int64_t wb) {
    const int64_t r = wb * 32 + lane;
    if (wb < nwb && r < n_rays) {
      const float4* r4 = reinterpret_cast<const float4*>(P.rays + r);
      nra = __ldg(r4);
      nrb = __ldg(r4 + 1);
    }
  };
  issue_claim();
  int64_t next_wb = claimed();
  load_ray(next_wb);
  if (kByteMask) {
    for (int i = threadIdx.x; i < code_words * 4; i += blockDim.x) {  // 4 cells per 32-bit store
      const uint32_t w = __ldg(m.stop2 + (i >> 2)) >> ((i & 3) * 8);
      smem[i] = (w & 3u) | ((w & 0xcu) << 6) | ((w & 0x30u) << 12) | ((w & 0xc0u) << 18);
    }
  } else {
    for (int i = threadIdx.x; i < code_words; i += blockDim.x) smem[i] = __ldg(m.stop2 + i);
  }
  auto stop_at = [&](uint32_t idx) -> uint32_t {
    if (kByteMask) return reinterpret_cast<const uint8_t*>(smem)[idx];
    return stop_code2(smem, idx);
  };
  __syncthreads();
  while (next_wb < nwb) {
    const int64_t wbatch = next_wb;
    const int64_t ray_idx = wbatch * 32 + lane;
    const bool live = ray_idx < n_rays;
    const float4 ra = nra, rb = nrb;
    issue_claim();
    float o[3] = {ra.x, ra.y, ra.z}, d[3] = {ra.w, rb.x, rb.y};
    const float t_min = rb.z, t_max = rb.w;
    float enter = 0.0f, exit = 0.0f;
    bool pair;
    if (P.intervals) {  // given pairs (run_narrow_phase, renderer.cpp:232-265): every ray is one
      if (live) {
        const float2 iv = __ldg(reinterpret_cast<const float2*>(P.intervals) + ray_idx);
        enter = iv.x;
        exit = iv.y;
      }
      pair = live;
    } else {
      pair = live && frame_interval(m, o, d, t_min, t_max, enter, exit);
    }

    // ---- DDA (dda.cpp:88-116): occupied-cell entry points into the pool
    Walk w;
    int count = 0;
    bool fio = false;
    if (pair && walk_setup<VS>(m, o, d, t_min, w)) {
      // the encode reads the local ray back from SMEM: o, d are dead in the walk
      lane_ray[2 * lane] = make_float4(w.o[0], w.o[1], w.o[2], 0.0f);
      lane_ray[2 * lane + 1] = make_float4(w.d[0], w.d[1], w.d[2], 0.0f);
      if (stop_at(w.idx)) {  // start cell (always inside the grid)
        fio = w.axis0 < 0;
        pool_put(lane, make_uint2(__float_as_uint(w.t0), start_code(w.axis0)));
        if (DEBUG) {
          int c[3];
          walk_cell<VS>(m, w.idx, c);
          P.cells[ray_idx * H] = c[0] | c[1] << 8 | c[2] << 16;
        }
        count = 1;
      }
      float tn;
      if (count < H && w.t1 != -__int_as_float(0x7f800000)) {
        // one latch (the advance at the bottom) keeps this a single loop:
        // lanes at a stop cell emit while the others keep walking; the emit
        // stores t and the low byte of the step's index increment (the
        // stepped axis), the entry plane is rebuilt from t in the encode
        int dl = walk_advance_dl(w, tn);
        for (;;) {
          const uint32_t sc = stop_at(w.idx);
          if (sc != 0u) {
            // the border (the walk left the grid, dda.cpp:112), or the walk
            // ended before this cell (dda.cpp:106)
            if (sc > 1u || tn > w.t1) break;
            pool_put(count * 32 + lane, make_uint2(__float_as_uint(tn), static_cast<uint32_t>(dl) & 0xffu));
            if (DEBUG) {
              int c[3];
              walk_cell<VS>(m, w.idx, c);
              P.cells[ray_idx * H + count] = c[0] | c[1] << 8 | c[2] << 16;
            }
            if (++count >= H) break;  // first-H truncation (dda.cpp:99)
          }
          dl = walk_advance_dl(w, tn);
        }
      }
    }

    next_wb = claimed();
    load_ray(next_wb);

    // ---- rays answered without the MLP
    if (!DEBUG) {
      if (live && !pair) {
        lsnif_hit h{};
        store_result(P.out, ray_idx, P.wire, h);
      } else if (pair && count == 0) {
        lsnif_hit h;
        decode_zero(m, enter, exit, t_min, t_max, P.mode, h);
        store_result(P.out, ray_idx, P.wire, h);
      }
    } else if (live) {
      P.info[ray_idx] = pair ? (count | (fio ? 1 << 8 : 0) | (1 << 9)) : 0;
      P.interval[2 * ray_idx] = pair ? enter : 0.0f;
      P.interval[2 * ray_idx + 1] = pair ? exit : 0.0f;
    }

    // ---- row allocation (warp-aggregated per K bin) for rays that need the MLP
    const bool valid = pair && count > 0;
    const int bin = valid ? (count * LF + 15) / 16 - 1 : -1;
    int row = 0;
    if (!DEBUG) {
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (valid && lane == leader) base = atomicAdd(P.row_counter + bin, __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      row = base + __popc(peers & ((1u << lane) - 1u));
      if (valid) {
        float4* dst = reinterpret_cast<float4*>(P.meta + static_cast<int64_t>(bin) * P.cap_tiles * kTileM + row);
        dst[0] = make_float4(__int_as_float(static_cast<int32_t>(ray_idx)), enter, exit, t_min);
        dst[1] = make_float4(t_max, 0.0f, 0.0f, 0.0f);
      }
      st_pair += pair ? 1u : 0u;
      st_rows += valid ? 1u : 0u;
      st_pts += valid ? static_cast<uint32_t>(count) : 0u;
      st_vol += (valid && fio) ? 1u : 0u;
    }

    if (valid) {  // the row / bin of the stashed local ray
      reinterpret_cast<int*>(lane_ray)[8 * lane + 3] = row;
      reinterpret_cast<int*>(lane_ray)[8 * lane + 7] = bin;
    }
    __syncwarp();
    // ---- warp-cooperative encode of the pooled points (encoding.hpp:166-176):
    // boundary points in passes of 32 (any lane may take any lane's point),
    // then the rare inside-origin "volume" first points (8 corners per level)
    // in one pass of their own, so the boundary passes never diverge into the
    // volume path.
    // VOLT: std::integral_constant<bool, volume point> (compile time, so each
    // pass carries only its own path)
    auto encode_point = [&](auto VOLT, const float ro[3], const float rd[3], int64_t o_ray, int o_row, int o_bin,
                            int k, const uint2 e) {
      constexpr bool volume = decltype(VOLT)::value;
      float p[3];
      point_from_code(__uint_as_float(e.x), point_axis_code(e.y, V), ro, rd, m.fres, m.inv_fres, p);
      float fv[16];
      const int pa = volume ? -1 : plane_axis_of(p, m.fres);
      if (LS == 2 && !volume) {
        // both levels' 8 gathers in flight before any accumulation
        uint32_t i0[4], i1[4];
        float w0[4], w1[4];
        boundary_corners<POW2>(m, 0, p, pa, i0, w0);
        boundary_corners<POW2>(m, 1, p, pa, i1, w1);
        uint2 e0[4], e1[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          e0[q] = __ldg(m.tables[0] + i0[q]);
          e1[q] = __ldg(m.tables[1] + i1[q]);
        }
        float f0[4], f1[4];
        accumulate4(e0, w0, f0);
        accumulate4(e1, w1, f1);
#pragma unroll
        for (int f = 0; f < 4; ++f)
          if (f < F) {
            fv[f] = f0[f];
            fv[F + f] = f1[f];
          }
        if (DEBUG) {
          const int64_t hb = (o_ray * H + k) * L * 8;
          for (int q = 0; q < 4; ++q) {
            P.hidx[hb + q] = i0[q];
            P.hidx[hb + 8 + q] = i1[q];
          }
          for (int f = 0; f < F; ++f) {
            P.feat[o_ray * m.K1 + k * LF + f] = f0[f];
            P.feat[o_ray * m.K1 + k * LF + F + f] = f1[f];
          }
        }
      } else {
#pragma unroll
        for (int l = 0; l < (LS ? LS : kMaxLevels); ++l) {
          if (!LS && l >= L) break;
          float feat[4];
          uint32_t hidx[8];
          if (volume)
            encode_volume_level<POW2>(m, l, p, feat, DEBUG ? hidx : nullptr);
          else
            encode_boundary_level<POW2>(m, l, p, pa, feat, DEBUG ? hidx : nullptr);
          if (DEBUG) {
            const int64_t hb = ((o_ray * H + k) * L + l) * 8;
            const int nc = volume ? 8 : 4;
            for (int q = 0; q < nc; ++q) P.hidx[hb + q] = hidx[q];
            for (int f = 0; f < F; ++f) P.feat[o_ray * m.K1 + k * LF + l * F + f] = feat[f];
          }
#pragma unroll
          for (int f = 0; f < 4; ++f)
            if (f < F) fv[l * F + f] = feat[f];
        }
      }
      if (DEBUG) {
        P.t[o_ray * H + k] = __uint_as_float(e.x);
        P.pts[(o_ray * H + k) * 3 + 0] = p[0];
        P.pts[(o_ray * H + k) * 3 + 1] = p[1];
        P.pts[(o_ray * H + k) * 3 + 2] = p[2];
      } else {
        uint8_t* tile = P.X + bin_x_offset(o_bin, P.cap_tiles) +
                        static_cast<int64_t>(o_row >> 7) * (o_bin + 1) * kBinTileBytes;
        const int r = o_row & 127;
        const int col0 = k * LF;
        if ((LF & 1) == 0) {
#pragma unroll
          for (int q = 0; q < (LS && FS ? LS * FS : 16); q += 2) {
            if (!(LS && FS) && q >= LF) break;
            const __half2 hv = __floats2half2_rn(__fmul_rn(fv[q], scale), __fmul_rn(fv[q + 1], scale));
            *reinterpret_cast<__half2*>(tile + canon_offset(r, col0 + q, kTileM)) = hv;
          }
        } else {
          for (int q = 0; q < LF; ++q)
            *reinterpret_cast<__half*>(tile + canon_offset(r, col0 + q, kTileM)) =
                __float2half_rn(__fmul_rn(fv[q], scale));
        }
      }
    };
    const int vc = (valid && fio) ? 1 : 0;  // this lane's volume point (k = 0)
    const int c = valid ? count - vc : 0;   // its boundary points (k = vc .. count-1)
    int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    const int excl = incl - c;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int jb = 0; jb < total; jb += 32) {
      const int j = jb + lane;
      int owner = 0;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const int ex = __shfl_sync(0xffffffffu, excl, owner + st);
        if (ex <= j) owner += st;
      }
      const int o_excl = __shfl_sync(0xffffffffu, excl, owner);
      const int o_vc = __shfl_sync(0xffffffffu, vc, owner);
      if (j >= total) continue;
      const float4 rq = lane_ray[2 * owner], rr = lane_ray[2 * owner + 1];
      const float ro[3] = {rq.x, rq.y, rq.z}, rd[3] = {rr.x, rr.y, rr.z};
      const int k = o_vc + j - o_excl;
      encode_point(std::false_type{}, ro, rd, wbatch * 32 + owner, __float_as_int(rq.w), __float_as_int(rr.w), k,
                   pool_get(k * 32 + owner));
    }
    if (vc) {
      const float4 sq = lane_ray[2 * lane], sr = lane_ray[2 * lane + 1];
      const float so[3] = {sq.x, sq.y, sq.z}, sd[3] = {sr.x, sr.y, sr.z};
      encode_point(std::true_type{}, so, sd, ray_idx, row, bin, 0, pool_get(lane));
    }

    // ---- zero padding of the row tail up to the bin width (encoding.hpp:170)
    if (!DEBUG && valid) {
      uint8_t* tile = P.X + bin_x_offset(bin, P.cap_tiles) + static_cast<int64_t>(row >> 7) * (bin + 1) * kBinTileBytes;
      const int r = row & 127;
      const int kb = 16 * (bin + 1);
      int col = count * LF;
      if ((col & 1) == 0)
        for (; col < kb && (col & 7); col += 2) *reinterpret_cast<uint32_t*>(tile + canon_offset(r, col, kTileM)) = 0u;
      for (; col < kb && (col & 7); ++col) *reinterpret_cast<uint16_t*>(tile + canon_offset(r, col, kTileM)) = 0;
      for (; col < kb; col += 8) *reinterpret_cast<uint4*>(tile + canon_offset(r, col, kTileM)) = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();  // pool reuse by the next batch
  }
  if (!DEBUG) {  // one set of statistics atomics per warp
    const uint32_t a = __reduce_add_sync(0xffffffffu, st_pair);
    const uint32_t b = __reduce_add_sync(0xffffffffu, st_rows);
    const uint32_t c = __reduce_add_sync(0xffffffffu, st_pts);
    const uint32_t e = __reduce_add_sync(0xffffffffu, st_vol);
    if (lane == 0 && a) {
      atomicAdd(P.stats + 0, static_cast<unsigned long long>(a));
      atomicAdd(P.stats + 1, static_cast<unsigned long long>(b));
      atomicAdd(P.stats + 2, static_cast<unsigned long long>(c));
      atomicAdd(P.stats + 3, static_cast<unsigned long long>(e));
    }
  }
}

// ============================================================ tcgen05 MLP

// Warp-specialised persistent MLP over the compacted 128-row X tiles:
//   warp 0  loader: bulk-copies X tiles into a kXStages SMEM ring and keeps
//           kPrefetch tiles ahead in flight as L2 prefetches;
//   warp 1  TMEM allocator + the MMA-issuing thread of epilogue group 0;
//           the last warp issues group 1's MMAs (each blocks on its own
//           group's barriers; the tensor pipe interleaves the streams);
//   warps 2-9 / 10-17  two epilogue groups of 8 warps (2 per TMEM lane
//           quadrant, each taking half of the columns); group g owns TMEM
//           columns [256g, 256g+256): the fp32 accumulator D (128 cols) and
//           the fp16 hidden operand A_h (72 cols: 128 K-values + bias block).
// Per tile: L1 = X W1^T (A = X from SMEM, b1 via the constant column),
// h1 = leaky(D) -> fp16 A_h (tcgen05.st), L2 = A_h W2^T (A from TMEM, b2 via
// the constant column), h2 -> A_h, L3 = A_h W3^T (N = 16, K = 128), logits +
// b3 in fp32, heads/decode/accept -> global hits.
template <int HID>
struct MlpLayout {
  static constexpr int kK2 = HID + 16;        // hidden + bias block
  static constexpr int kEpiWarps = 8;         // per group
  static constexpr int kThreads = 32 * (3 + 2 * kEpiWarps);  // loader, 2 issuers, epilogues
  static constexpr int kXStages = 4;
  static constexpr uint32_t kGroupCols = HID == 128 ? 256 : 128;  // TMEM columns per group (D + A_h)
  static constexpr uint32_t kACol = HID;      // A_h column offset within a group
};

// leaky_relu(v, 0.01) (mlp.hpp:80-94) on a packed pair: the fp32 accumulator
// pair is rounded to fp16 once (F2FP), then max(h, 0.01 h) in half2 (HFMA2 +
// HMNMX2): 1.5 instructions per activation instead of 2.5 for the fp32 form
// (the epilogue is issue-bound). Non-negative activations are exactly their
// fp16 rounding, as before; negative ones are 0.01 (as fp16) times the
// rounded value, rounded (a second rounding on the 1%-slope side only).
__device__ __forceinline__ uint32_t leaky_pack(uint32_t a, uint32_t b) {
  const __half2 v = __floats2half2_rn(__uint_as_float(a), __uint_as_float(b));
  const __half2 h = __hmax2(v, __hmul2(v, __float2half2_rn(0.01f)));
  return *reinterpret_cast<const uint32_t*>(&h);
}

// h = leaky(D) for hidden columns [c0, c0 + NC) of this lane's row -> packed
// fp16 pairs in A_h columns [c0/2, c0/2 + NC/2) (NC = HID / 2: each of the
// two warps of a lane quadrant takes half of the columns). The bias is
// already in D (constant-operand K-step / A_h bias column) and the
// activation scale carries through the positively homogeneous leaky-ReLU.
template <int NC>
__device__ __forceinline__ void epi_hidden(uint32_t tD, uint32_t tA, int c0) {
  static_assert(NC == 64 || NC == 32, "32 or 64 columns per warp");
  uint32_t a0[32], a1[32], o[32];
  tc::tmem_ld32(tD + c0, a0);
  if (NC == 64) tc::tmem_ld32(tD + c0 + 32, a1);
  tc::tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = leaky_pack(a0[2 * j], a0[2 * j + 1]);
  if (NC == 64) {
#pragma unroll
    for (int j = 0; j < 16; ++j) o[16 + j] = leaky_pack(a1[2 * j], a1[2 * j + 1]);
    tc::tmem_st32(tA + c0 / 2, o);
  } else {
    tc::tmem_st16(tA + c0 / 2, o);
  }
}

// LSNIF_MLP_TIMELINE builds record, for CTA 0, clock64 stamps of the MMA
// issuer and of one warp per epilogue half and group (probe builds only).
#ifdef LSNIF_MLP_TIMELINE
__device__ unsigned long long g_mlp_timeline[1 << 16];
#define TL_STAMP(slot) g_mlp_timeline[(slot)] = clock64()
extern "C" int lsnif_probe_mlp_timeline(unsigned long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_mlp_timeline, sizeof(unsigned long long) * n));
}
#else
#define TL_STAMP(slot) (void)0
#endif

template <int HID, int NS>
__global__ void __launch_bounds__(MlpLayout<HID>::kThreads, 1) mlp_tc_kernel(const MlpParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using Lay = MlpLayout<HID>;
  constexpr int K2 = Lay::kK2;
  constexpr int EW = Lay::kEpiWarps;
  // NS: X ring depth, 4 or (inputs too wide for four stages next to the
  // weights, mlp_x_stages) 2; a compile-time constant keeps the ring
  // arithmetic off the issuing thread's critical path
  static_assert(NS == 4 || NS == 2, "X ring depth");
  static_assert(HID == 128 || HID == 64, "hidden width 64 (low-quality LSNIF) or 128 (high-quality)");
  const DevModel& m = P.m;
  if (blockIdx.x == 0 && threadIdx.x == 0) TL_STAMP(1023 * 64 + 0);  // kernel entry
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t xbytes = static_cast<uint32_t>(kTileM) * m.K1P * 2;
  const uint32_t xstage = (xbytes + 1023) & ~1023u;
  uint8_t* sW1 = base;
  uint8_t* sW2 = sW1 + m.w1_bytes;
  uint8_t* sW3 = sW2 + m.w2_bytes;
  uint8_t* sC = sW3 + ((m.w3_bytes + 1023) & ~1023u);  // constant bias slab (4 KB)
  uint8_t* sX = sC + kBinTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sX + NS * xstage);
  uint64_t* w_full = bars;                // 1
  uint64_t* x_full = bars + 1;            // NS
  uint64_t* x_empty = x_full + NS;        // NS
  uint64_t* l_done = x_empty + NS;        // 2
  uint64_t* h_ready = l_done + 2;         // 2
  uint64_t* acc_free = h_ready + 2;       // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);
  int* tstart = reinterpret_cast<int*>(tmem_slot + 4);  // first global tile of each K bin (+ total)
  int* x_bin = tstart + kMaxBins + 1;  // K bin of the tile in each X stage (loader -> MMA)
  int* bin_rows_n = x_bin + 8;         // rows of each K bin
  constexpr int kZSlots = 10;          // logits a thread keeps for its deferred decode
  float* zslots = reinterpret_cast<float*>(sX + NS * xstage + 1024);  // 16 warps x 10 x 32

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  // A chunk past the device-side ray count (renderer / scene queries sized by
  // an upper bound) has no rows: leave before the prologue. The count was
  // written before the trace kernel started, so it is visible here.
  if (P.n_dev && P.offset >= static_cast<int64_t>(*P.n_dev)) return;
  // ---- prologue, independent of the trace kernel's results: with
  // programmatic dependent launch it overlaps the trace kernel's tail
  if (tid == 0) {
    tc::mbar_init(w_full, 1);
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(x_full + s, 1);
      tc::mbar_init(x_empty + s, 1);
    }
    for (int g = 0; g < 2; ++g) {
      tc::mbar_init(l_done + g, 1);
      tc::mbar_init(h_ready + g, EW);   // one arrival per epilogue warp
      tc::mbar_init(acc_free + g, EW);
    }
    tc::fence_mbar_init();
  }
  // constant A slab of layer 1's bias K-step: column 0 = act_scale, 128 rows
  // (W1's last 16-column slab holds b1 in column 0)
  for (int r = threadIdx.x; r < kTileM; r += blockDim.x) {
    const uint32_t hs = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(m.act_scale)));
    *reinterpret_cast<uint4*>(sC + canon_offset(r, 0, kTileM)) = make_uint4(hs, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(sC + canon_offset(r, 8, kTileM)) = make_uint4(0u, 0u, 0u, 0u);
  }
  tc::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * Lay::kGroupCols);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) {  // the weights stay in SMEM for the kernel's lifetime
    tc::mbar_arrive_expect_tx(w_full, m.w1_bytes + m.w2_bytes + m.w3_bytes);
    tc::bulk_g2s(sW1, m.w_canon, m.w1_bytes, w_full);
    tc::bulk_g2s(sW2, m.w_canon + m.w1_bytes, m.w2_bytes, w_full);
    tc::bulk_g2s(sW3, m.w_canon + m.w1_bytes + m.w2_bytes, m.w3_bytes, w_full);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the trace kernel's rows are complete
  if (blockIdx.x == 0 && threadIdx.x == 0) TL_STAMP(1023 * 64 + 1);  // dependency resolved

  // tiles of all K bins, bin-major: global tile -> (bin b, tile t within b);
  // one global round trip for the row counters (written by the trace grid)
  const int nb = m.n_bins;
  if (tid < nb) bin_rows_n[tid] = P.row_counter[tid];
  __syncthreads();
  int ntiles = 0;
  for (int b = 0; b < nb; ++b) ntiles += (bin_rows_n[b] + kTileM - 1) / kTileM;
  if (static_cast<int>(blockIdx.x) >= ntiles) {  // nothing to do: release what the prologue took
    if (tid == 0) tc::mbar_wait(w_full, 0);
    __syncthreads();
    if (warp == 1) {
      tc::tc_fence_after();
      tc::tmem_dealloc(tmem, 2 * Lay::kGroupCols);
    }
    return;
  }
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = 0; b < nb; ++b) {
      tstart[b] = acc;
      acc += (bin_rows_n[b] + kTileM - 1) / kTileM;
    }
    tstart[nb] = acc;
  }
  __syncthreads();
  auto locate = [&](int tile, int& b, int& t) {
    b = 0;
    while (tile >= tstart[b + 1]) ++b;
    t = tile - tstart[b];
  };
  const int64_t bin_rows = P.cap_tiles * kTileM;
  const int my_tiles = (ntiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                       static_cast<int>(gridDim.x);

  if (warp == 0) {
    // ------------------------------------------------------------ loader
    if (lane == 0) {
      constexpr int kPrefetch = 8;
      auto tile_src = [&](int i, uint32_t& bytes) -> const uint8_t* {
        int b, t;
        locate(blockIdx.x + i * gridDim.x, b, t);
        bytes = (b + 1) * kBinTileBytes;
        return P.X + bin_x_offset(b, P.cap_tiles) + static_cast<int64_t>(t) * bytes;
      };
      uint32_t nbytes;
      // the first stages' copies go out before any L2 prefetch (they would
      // queue behind the prefetches in the copy engine)
      for (int i = 0; i < NS && i < my_tiles; ++i) {
        const uint8_t* src = tile_src(i, nbytes);
        x_bin[i] = static_cast<int>(nbytes / kBinTileBytes) - 1;
        tc::mbar_arrive_expect_tx(x_full + i, nbytes);
        tc::bulk_g2s(sX + i * xstage, src, nbytes, x_full + i);
      }
      for (int i = NS; i < NS + kPrefetch && i < my_tiles; ++i) {
        const uint8_t* src = tile_src(i, nbytes);
        tc::bulk_prefetch_l2(src, nbytes);
      }
      for (int i = NS; i < my_tiles; ++i) {
        const int st = i % NS, k = i / NS;
        if (i + kPrefetch < my_tiles) {
          const uint8_t* src = tile_src(i + kPrefetch, nbytes);
          tc::bulk_prefetch_l2(src, nbytes);
        }
        const uint8_t* src = tile_src(i, nbytes);
        if (k > 0) tc::mbar_wait(x_empty + st, (k - 1) & 1);
        x_bin[st] = static_cast<int>(nbytes / kBinTileBytes) - 1;  // released by the arrive below
        tc::mbar_arrive_expect_tx(x_full + st, nbytes);
        tc::bulk_g2s(sX + st * xstage, src, nbytes, x_full + st);
      }
    }
  } else if (warp == 1 || warp == 2 + 2 * EW) {
    // ------------------------------------------------------------ MMA issuers
    // one issuing thread per epilogue group (warp 1: group 0, the last warp:
    // group 1), each blocking on its own group's barriers; the tensor pipe
    // interleaves the two streams, so neither group's next layer waits for
    // the other group's MMA burst to be issued
    if (lane == 0) {
      const int g = warp == 1 ? 0 : 1;
      tc::mbar_wait(w_full, 0);
      if (blockIdx.x == 0 && g == 0) TL_STAMP(1023 * 64 + 2);  // weights in SMEM
      const uint32_t sW1_a = tc::smem_addr(sW1), sW2_a = tc::smem_addr(sW2), sW3_a = tc::smem_addr(sW3);
      const uint32_t sX_a = tc::smem_addr(sX), sC_a = tc::smem_addr(sC);
      constexpr uint32_t kIdescH = tc::idesc_f16_f32(kTileM, HID);
      const uint32_t idesc3 = tc::idesc_f16_f32(kTileM, m.N3);
      constexpr uint32_t a_lbo = kTileM * 16;
      const uint32_t tD = tmem + g * Lay::kGroupCols;
      const uint32_t tA = tD + Lay::kACol;
      uint32_t hc = 0;
      for (int i = g; i < my_tiles; i += 2) {
        const int st = i % NS, kx = i / NS, ka = i >> 1;
        tc::mbar_wait(x_full + st, kx & 1);
        if (ka > 0) tc::mbar_wait(acc_free + g, (ka - 1) & 1);
        if (blockIdx.x == 0 && i < 1024) TL_STAMP(i * 64 + 5);  // X + accumulator ready seen
        tc::tc_fence_after();
        const uint32_t a_base = sX_a + st * xstage;
        const int xb = x_bin[st];
        for (int ks = 0; ks <= xb; ++ks) {  // L1: A = X (SMEM), the tile's bin width
          // (the tile's SMEM stage holds K_b columns: LBO stays 128 x 16 B)
          const uint64_t ad = tc::smem_desc(a_base + ks * 2 * a_lbo, a_lbo, 128);
          const uint64_t bd = tc::smem_desc(sW1_a + ks * 2 * HID * 16, HID * 16, 128);
          tc::mma_f16_ss(tD, ad, bd, kIdescH, ks > 0 ? 1u : 0u);
        }
        {  // + b1: constant slab (act_scale in column 0) x W1's bias slab
          const uint64_t ad = tc::smem_desc(sC_a, a_lbo, 128);
          const uint64_t bd = tc::smem_desc(sW1_a + (m.K1P / 16) * 2 * HID * 16, HID * 16, 128);
          tc::mma_f16_ss(tD, ad, bd, kIdescH, 1u);
        }
        tc::mma_commit(x_empty + st);
        tc::mma_commit(l_done + g);
        if (blockIdx.x == 0 && i < 1024) TL_STAMP(i * 64 + 0);
        // L2: A = h1 (TMEM), K = HID + bias block
        tc::mbar_wait(h_ready + g, hc++ & 1);
        if (blockIdx.x == 0 && i < 1024) TL_STAMP(i * 64 + 3);  // h1 ready seen
        tc::tc_fence_after();
        for (int ks = 0; ks < K2 / 16; ++ks) {
          const uint64_t bd = tc::smem_desc(sW2_a + ks * 2 * HID * 16, HID * 16, 128);
          tc::mma_f16_ts(tD, tA + ks * 8, bd, kIdescH, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(l_done + g);
        if (blockIdx.x == 0 && i < 1024) TL_STAMP(i * 64 + 1);
        // L3: A = h2 (TMEM), K = HID, N = 16
        tc::mbar_wait(h_ready + g, hc++ & 1);
        if (blockIdx.x == 0 && i < 1024) TL_STAMP(i * 64 + 4);  // h2 ready seen
        tc::tc_fence_after();
        for (int ks = 0; ks < HID / 16; ++ks) {
          const uint64_t bd = tc::smem_desc(sW3_a + ks * 2 * m.N3 * 16, m.N3 * 16, 128);
          tc::mma_f16_ts(tD, tA + ks * 8, bd, idesc3, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(l_done + g);
        if (blockIdx.x == 0 && i < 1024) TL_STAMP(i * 64 + 2);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogues
    const int g = (warp - 2) / EW;
    const int e = (warp - 2) % EW;
    const int half = e / 4;  // column half; warps e and e+4 share a lane quadrant
    const int row = 32 * (warp & 3) + lane;
    const uint32_t lanes = static_cast<uint32_t>(32 * (warp & 3)) << 16;
    const uint32_t tD = tmem + lanes + g * Lay::kGroupCols;
    const uint32_t tA = tD + Lay::kACol;
    if (half == 0) {  // bias block of A_h: K = HID holds act_scale, HID+1..K2-1 zero
      const uint32_t hs = static_cast<uint32_t>(__half_as_ushort(__float2half_rn(m.act_scale)));
      const uint32_t blk[8] = {hs, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      tc::tmem_st8(tA + HID / 2, blk);
      tc::tmem_wait_st();
    }
    uint32_t lcount = 0;
    // Row metadata, prefetched one tile ahead: ray index (both halves),
    // interval and t range (the lower half, which decodes them).
    auto load_meta = [&](int i, float4& a, float4& b, bool& live) {
      a = b = make_float4(0.f, 0.f, 0.f, 0.f);
      live = false;
      if (i >= my_tiles) return;
      int tb, tt;
      locate(blockIdx.x + i * gridDim.x, tb, tt);
      const int grow = tt * kTileM + row;
      live = grow < bin_rows_n[tb];
      if (live) {
        const float4* mp = reinterpret_cast<const float4*>(P.meta + tb * bin_rows + grow);
        a = __ldg(mp);
        if (half == 0) b = __ldg(mp + 1);
      }
    };
    // The decode of a tile (heads, NeuralHit, accept; renderer.cpp:208-223,
    // 280-301) is deferred until after the group's next layer-1 epilogue, so
    // it overlaps the next tile's layer-2 MMAs instead of delaying its
    // layer 1. The logits wait in this thread's private SMEM slots; the two
    // warps of a row split the work: lower half z0, z1, z8.. (visibility,
    // t_world, material, accept), upper half z2..z7 (normal, albedo).
    float* zs = zslots + (warp - 2) * kZSlots * 32 + lane;
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = pa;  // pending tile's metadata
    bool plive = false;
    auto decode_pending = [&]() {
      if (!plive) return;
      const int64_t ray = __float_as_int(pa.x);
      float* dst = reinterpret_cast<float*>(static_cast<uint8_t*>(P.out) + ray * (P.wire ? 16 : 32));
      if (half == 0) {
        float zm[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) zm[k] = k < m.n_mat ? zs[(2 + k) * 32] : 0.0f;
        uint32_t fm;
        float tw;
        decode_flags_fast(zs[0], zs[32], zm, m.n_mat, m.occ_threshold, pa.y, pa.z, pa.w, pb.x, P.mode, fm, tw);
        *reinterpret_cast<float2*>(dst) = make_float2(__uint_as_float(fm), tw);
      } else {
        float nrm[3], alb[3];
        decode_normal_fast(zs[0], zs[32], zs[64], nrm);
        decode_albedo_fast(zs[96], zs[128], zs[160], alb);
        if (P.wire) {
          uint32_t no, al;
          wire_pack_normal_albedo(nrm, alb, no, al);
          *reinterpret_cast<uint2*>(dst + 2) = make_uint2(no, al);
        } else {
          *reinterpret_cast<float2*>(dst + 2) = make_float2(nrm[0], nrm[1]);
          *reinterpret_cast<float4*>(dst + 4) = make_float4(nrm[2], alb[0], alb[1], alb[2]);
        }
      }
      plive = false;
    };
    float4 na, nb_;
    bool nlive;
    load_meta(g, na, nb_, nlive);
    for (int i = g; i < my_tiles; i += 2) {
      const float4 ma = na, mb = nb_;
      const bool live = nlive;
      load_meta(i + 2, na, nb_, nlive);
      const bool tl = blockIdx.x == 0 && i < 1024 && lane == 0;
      (void)tl;
#pragma unroll 1
      for (int layer = 0; layer < 2; ++layer) {  // h1, h2 -> A_h
        tc::mbar_wait(l_done + g, lcount++ & 1);
        if (tl) TL_STAMP(i * 64 + 8 + 8 * layer + e);  // L1 / L2 done seen by warp e
        tc::tc_fence_after();
        epi_hidden<HID / 2>(tD, tA, half * (HID / 2));
        tc::tmem_wait_st();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(h_ready + g);
        if (tl) TL_STAMP(i * 64 + 24 + 8 * layer + e);  // h1 / h2 published by warp e
        if (layer == 0) decode_pending();             // previous tile of this group
      }
      // layer 3: logits (+ b3 in fp32, activation scale removed) -> SMEM
      tc::mbar_wait(l_done + g, lcount++ & 1);
      if (tl) TL_STAMP(i * 64 + 40 + e);  // L3 done seen
      tc::tc_fence_after();
      {
        uint32_t acc[16];
        tc::tmem_ld16(tD, acc);
        tc::tmem_wait_ld();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(acc_free + g);
        if (half == 0) {
          zs[0] = __fadd_rn(__fmul_rn(__uint_as_float(acc[0]), m.inv_act_scale), m.b3[0]);
          zs[32] = __fadd_rn(__fmul_rn(__uint_as_float(acc[1]), m.inv_act_scale), m.b3[1]);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k < m.n_mat) zs[(2 + k) * 32] = __fadd_rn(__fmul_rn(__uint_as_float(acc[8 + k]), m.inv_act_scale), m.b3[8 + k]);
        } else {
#pragma unroll
          for (int k = 0; k < 6; ++k)
            zs[k * 32] = __fadd_rn(__fmul_rn(__uint_as_float(acc[2 + k]), m.inv_act_scale), m.b3[2 + k]);
        }
      }
      pa = ma;
      pb = mb;
      plive = live;
      if (tl) TL_STAMP(i * 64 + 48 + e);  // tile's epilogue work done (decode deferred)
    }
    decode_pending();
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) TL_STAMP(1023 * 64 + 3);  // all tiles done
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 2 * Lay::kGroupCols);
  }
}

// ===================================================== multi-object scenes

// best_t = ray.t_max (no triangle objects, renderer.cpp:275), no hit.
__global__ void scene_init_kernel(const lsnif_ray* __restrict__ rays, int64_t n, const int32_t* n_dev,
                                  lsnif_scene_hit* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (n_dev) n = min(n, static_cast<int64_t>(*n_dev));
  if (i >= n) return;
  float4* o = reinterpret_cast<float4*>(out + i);
  const float t_max = rays[i].t_max;
  o[0] = make_float4(t_max, 0.f, 0.f, 0.f);
  o[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  o[2] = make_float4(0.f, 0.f, 0.f, 0.f);
  o[3] = make_float4(__int_as_float(-1), 0.f, 0.f, 0.f);  // object_index = -1, flags = 0
}

// object_space_ray (renderer.cpp:30-37): linear*p + translation, inner sum in
// index order, unfused.
__device__ __forceinline__ void to_object(const float* L, const float p[3], const float d[3], float op[3],
                                          float od[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float* r = L + 4 * i;
    op[i] = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(r[0], p[0]), __fmul_rn(r[1], p[1])), __fmul_rn(r[2], p[2])), r[3]);
    od[i] = __fadd_rn(__fadd_rn(__fmul_rn(r[0], d[0]), __fmul_rn(r[1], d[1])), __fmul_rn(r[2], d[2]));
  }
}

// collect_pairs (renderer.cpp:159-173) for one instance: object-space ray,
// interval on the frame box with t_max = inf, kept iff enter < max_t.
// Emits the compacted object-space rays (t_max = the pair gate) + slots.
__global__ void __launch_bounds__(256) broad_phase_kernel(const DevModel m, const InstanceParams ip,
                                                          const lsnif_ray* __restrict__ rays, int64_t n,
                                                          const int32_t* n_dev,
                                                          lsnif_ray* __restrict__ orays, int32_t* __restrict__ slots,
                                                          int32_t* count) {
  if (n_dev) n = min(n, static_cast<int64_t>(*n_dev));
  if (static_cast<int64_t>(blockIdx.x) * blockDim.x >= n) return;  // whole block past the count
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool keep = false;
  float op[3], od[3], t_min = 0.f, t_max = 0.f;
  if (i < n) {
    const float4* r4 = reinterpret_cast<const float4*>(rays + i);
    const float4 a = __ldg(r4), b = __ldg(r4 + 1);
    const float p[3] = {a.x, a.y, a.z}, d[3] = {a.w, b.x, b.y};
    t_min = b.z;
    t_max = b.w;
    to_object(ip.w2o, p, d, op, od);
    float enter, exit;
    keep = frame_interval(m, op, od, t_min, t_max, enter, exit);
  }
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  int base = 0;
  if (lane == 0 && mask) base = atomicAdd(count, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) {
    const int j = base + __popc(mask & ((1u << lane) - 1u));
    float4* dst = reinterpret_cast<float4*>(orays + j);
    dst[0] = make_float4(op[0], op[1], op[2], od[0]);
    dst[1] = make_float4(od[1], od[2], t_min, t_max);
    slots[j] = static_cast<int32_t>(i);
  }
}

// collect_pairs (renderer.cpp:154-181) for all instances in one pass: each
// ray is read once, its scene hit initialised (scene_init_kernel), and every
// instance whose frame box it meets before t_max gets the object-space ray
// appended to its own pair list (warp-aggregated per instance).
__device__ __forceinline__ void broad_phase_one(const InstanceBox* __restrict__ boxes, int n_inst,
                                                const lsnif_ray* __restrict__ rays, int64_t n, int64_t i,
                                                lsnif_ray* __restrict__ orays, int32_t* __restrict__ slots,
                                                int64_t stride, int32_t* counts, lsnif_scene_hit* out,
                                                unsigned long long* best) {
  const int lane = threadIdx.x & 31;
  const bool live = i < n;
  float p[3] = {0, 0, 0}, d[3] = {0, 0, 0}, t_min = 0.f, t_max = 0.f;
  if (live) {
    const float4* r4 = reinterpret_cast<const float4*>(rays + i);
    const float4 a = __ldg(r4), b = __ldg(r4 + 1);
    p[0] = a.x;
    p[1] = a.y;
    p[2] = a.z;
    d[0] = a.w;
    d[1] = b.x;
    d[2] = b.y;
    t_min = b.z;
    t_max = b.w;
    float4* o = reinterpret_cast<float4*>(out + i);  // best_t = t_max, no hit (renderer.cpp:275)
    o[0] = make_float4(t_max, 0.f, 0.f, 0.f);
    o[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    o[2] = make_float4(0.f, 0.f, 0.f, 0.f);
    o[3] = make_float4(__int_as_float(-1), 0.f, 0.f, 0.f);
    if (best) best[i] = ~0ull;
  }
  for (int k = 0; k < n_inst; ++k) {
    const InstanceBox& B = boxes[k];
    float op[3], od[3];
    bool keep = false;
    if (live) {
      to_object(B.w2o, p, d, op, od);
      // ray_aabb_intersect on the frame box, t_max = inf; kept iff enter < t_max
      float t0 = t_min, t1 = __int_as_float(0x7f800000);
      keep = true;
#pragma unroll
      for (int a = 0; a < 3 && keep; ++a) {
        if (od[a] == 0.0f) {
          if (op[a] < B.mn[a] || op[a] > B.mx[a]) keep = false;
          continue;
        }
        const float inv = __frcp_rn(od[a]);
        float ta = __fmul_rn(__fsub_rn(B.mn[a], op[a]), inv);
        float tb = __fmul_rn(__fsub_rn(B.mx[a], op[a]), inv);
        if (ta > tb) {
          const float x = ta;
          ta = tb;
          tb = x;
        }
        t0 = smax(t0, ta);
        t1 = smin(t1, tb);
        if (t0 > t1) keep = false;
      }
      keep = keep && t0 < t_max;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    if (!mask) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(counts + k, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
      const int64_t j = static_cast<int64_t>(k) * stride + base + __popc(mask & ((1u << lane) - 1u));
      float4* dst = reinterpret_cast<float4*>(orays + j);
      dst[0] = make_float4(op[0], op[1], op[2], od[0]);
      dst[1] = make_float4(od[1], od[2], t_min, t_max);
      slots[j] = static_cast<int32_t>(i);
    }
  }
}

__global__ void __launch_bounds__(256) broad_phase_all_kernel(const InstanceBox* __restrict__ boxes, int n_inst,
                                                              const lsnif_ray* __restrict__ rays, int64_t n,
                                                              const int32_t* n_dev, lsnif_ray* __restrict__ orays,
                                                              int32_t* __restrict__ slots, int64_t stride,
                                                              int32_t* counts, lsnif_scene_hit* out,
                                                              unsigned long long* best) {
  if (n_dev) n = min(n, static_cast<int64_t>(*n_dev));
  // block-stride over the (device-side) ray count: the grid is sized for the
  // machine, every warp iterates uniformly (warp-aggregated appends)
  for (int64_t kb = static_cast<int64_t>(blockIdx.x) * blockDim.x; kb < n;
       kb += static_cast<int64_t>(gridDim.x) * blockDim.x)
    broad_phase_one(boxes, n_inst, rays, n, kb + threadIdx.x, orays, slots, stride, counts, out, best);
}

cudaError_t launch_broad_phase_all(const InstanceBox* boxes, int n_inst, const lsnif_ray* rays, int64_t n,
                                   const int32_t* n_dev, lsnif_ray* orays, int32_t* slots, int64_t stride,
                                   int32_t* counts, lsnif_scene_hit* out, unsigned long long* best,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>(n_dev ? std::min<int64_t>((n + 255) / 256, 148 * 8) : (n + 255) / 256);
  broad_phase_all_kernel<<<grid, 256, 0, st>>>(boxes, n_inst, rays, n, n_dev, orays, slots, stride, counts, out, best);
  return cudaGetLastError();
}

// Order-preserving map of a float onto uint32 (total order of non-NaN values).
__device__ __forceinline__ uint32_t float_key(float t) {
  const uint32_t b = __float_as_uint(t);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Pass 1 of the fused merge: every accepted neural hit of every instance
// (grid.y = instance) offers its key. Closest (renderer.cpp:280-301): accept
// iff occluded, t_min <= t < best_t with best_t starting at t_max; the object
// loop keeps the smallest t and, among equal t, the first object, which is
// the minimum of (t, k * stride + pair) since pairs of instance k sort before
// those of k + 1. Any (316-321): occluded and t in [t_min, t_max]; the first
// occluding object is the minimum k.
__global__ void __launch_bounds__(256) merge_min_kernel(const lsnif_ray* __restrict__ rays,
                                                        const lsnif_hit* __restrict__ hits,
                                                        const int32_t* __restrict__ slots, int64_t stride,
                                                        const int32_t* __restrict__ counts, int mode,
                                                        unsigned long long* best) {
  const int k = blockIdx.y;
  const int64_t cnt = counts[k];  // device-side pair count: grid-stride over it (the grid is sized by SMs)
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cnt;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t g = k * stride + j;
    const uint32_t fm = hits[g].flags_material;
    if (!(fm & LSNIF_HIT_OCCLUDED)) continue;
    const float t = hits[g].t_world;
    const int32_t slot = slots[g];
    const float t_min = rays[slot].t_min, t_max = rays[slot].t_max;
    if (mode == LSNIF_QUERY_CLOSEST) {
      if (!(t < t_max) || t < t_min) continue;
      atomicMin(best + slot, (static_cast<unsigned long long>(float_key(t)) << 32) | static_cast<uint32_t>(g));
    } else if (t >= t_min && t <= t_max) {
      atomicMin(best + slot, static_cast<unsigned long long>(k));
    }
  }
}

// The winner's SurfaceHit (as merge_kernel writes it) for ray i.
__device__ __forceinline__ void merge_final_ray(const InstanceBox* __restrict__ boxes,
                                                const lsnif_ray* __restrict__ rays, int64_t i,
                                                const lsnif_hit* __restrict__ hits, int64_t stride, int mode,
                                                unsigned long long key, lsnif_scene_hit* out) {
  if (key == ~0ull) return;
  if (mode != LSNIF_QUERY_CLOSEST) {
    out[i].flags = 1u;
    out[i].object_index = static_cast<int32_t>(key);
    return;
  }
  const int64_t g = static_cast<int64_t>(key & 0xffffffffull);
  const int k = static_cast<int>(g / stride);
  const InstanceBox& B = boxes[k];
  const lsnif_hit h = hits[g];
  const lsnif_ray r = rays[i];
  const float t = h.t_world;
  lsnif_scene_hit o{};
  o.t = t;
  for (int a = 0; a < 3; ++a) o.position[a] = __fadd_rn(r.origin[a], __fmul_rn(t, r.direction[a]));
  const float* n0 = h.normal;
  float nw[3];
  const float nn = __fadd_rn(__fadd_rn(__fmul_rn(n0[0], n0[0]), __fmul_rn(n0[1], n0[1])), __fmul_rn(n0[2], n0[2]));
  if (nn == 0.0f) {
    for (int a = 0; a < 3; ++a) nw[a] = -r.direction[a];
  } else {  // normal_to_world (renderer.cpp:39-41): (W2O.linear^T n).normalized()
    const float* L = B.w2o;
    for (int a = 0; a < 3; ++a)
      nw[a] = __fadd_rn(__fadd_rn(__fmul_rn(L[a], n0[0]), __fmul_rn(L[4 + a], n0[1])), __fmul_rn(L[8 + a], n0[2]));
    const float len = sqrtf(__fadd_rn(__fadd_rn(__fmul_rn(nw[0], nw[0]), __fmul_rn(nw[1], nw[1])), __fmul_rn(nw[2], nw[2])));
    if (len > 0.0f)
      for (int a = 0; a < 3; ++a) nw[a] = __fdiv_rn(nw[a], len);
  }
  const float dd = __fadd_rn(__fadd_rn(__fmul_rn(nw[0], r.direction[0]), __fmul_rn(nw[1], r.direction[1])),
                             __fmul_rn(nw[2], r.direction[2]));
  for (int a = 0; a < 3; ++a) {
    o.normal[a] = dd > 0.0f ? -nw[a] : nw[a];
    o.albedo[a] = h.albedo[a];
  }
  const int mat = iclamp(static_cast<int>(h.flags_material >> LSNIF_HIT_MATERIAL_SHIFT), 0, B.n_materials - 1);
  o.kind = B.materials[mat].kind;
  o.roughness = B.materials[mat].roughness;
  o.object_index = k;
  o.flags = 1u;
  out[i] = o;
}

// Pass 2: the winners' SurfaceHits, grid-stride over the (device-side) ray count.
__global__ void __launch_bounds__(256) merge_final_kernel(const InstanceBox* __restrict__ boxes,
                                                          const lsnif_ray* __restrict__ rays, int64_t n,
                                                          const int32_t* n_dev, const lsnif_hit* __restrict__ hits,
                                                          int64_t stride, int mode,
                                                          const unsigned long long* __restrict__ best,
                                                          lsnif_scene_hit* out) {
  if (n_dev) n = min(n, static_cast<int64_t>(*n_dev));
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    merge_final_ray(boxes, rays, i, hits, stride, mode, best[i], out);
}

cudaError_t launch_merge_all(const InstanceBox* boxes, int n_inst, const lsnif_ray* rays, int64_t n,
                             const int32_t* n_dev, const lsnif_hit* hits, const int32_t* slots, int64_t stride,
                             const int32_t* counts, int mode, unsigned long long* best, lsnif_scene_hit* out,
                             cudaStream_t st) {
  if (n <= 0 || n_inst <= 0) return cudaSuccess;
  // grids sized for the machine, not for the upper-bound counts (the real
  // counts live on the device; most of an n_max grid would exit at once)
  constexpr int64_t kMaxBlocks = 148 * 8;
  const dim3 g1(static_cast<unsigned>(std::min<int64_t>((stride + 255) / 256, std::max<int64_t>(kMaxBlocks / n_inst, 16))),
                static_cast<unsigned>(n_inst));
  merge_min_kernel<<<g1, 256, 0, st>>>(rays, hits, slots, stride, counts, mode, best);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  merge_final_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, kMaxBlocks)), 256, 0, st>>>(
      boxes, rays, n, n_dev, hits, stride, mode, best, out);
  return cudaGetLastError();
}

// Accept + merge of one instance's neural hits into the scene result, in
// object order (renderer.cpp:280-301 closest, 316-321 any): each ray occurs
// at most once per instance list, so no atomics are needed.
__global__ void __launch_bounds__(256) merge_kernel(const DevModel m, const InstanceParams ip,
                                                    const lsnif_ray* __restrict__ rays,
                                                    const lsnif_hit* __restrict__ hits,
                                                    const int32_t* __restrict__ slots, const int32_t* count,
                                                    int mode, lsnif_scene_hit* out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= *count) return;
  const lsnif_hit h = hits[j];
  if (!(h.flags_material & LSNIF_HIT_OCCLUDED)) return;
  const int32_t slot = slots[j];
  const lsnif_ray r = rays[slot];
  lsnif_scene_hit& sh = out[slot];
  const float t = h.t_world;
  if (mode == LSNIF_QUERY_CLOSEST) {
    if (t >= sh.t || t < r.t_min) return;
    lsnif_scene_hit o{};
    o.t = t;
    for (int a = 0; a < 3; ++a) o.position[a] = __fadd_rn(r.origin[a], __fmul_rn(t, r.direction[a]));
    const float* n0 = h.normal;
    float nw[3];
    const float nn = __fadd_rn(__fadd_rn(__fmul_rn(n0[0], n0[0]), __fmul_rn(n0[1], n0[1])), __fmul_rn(n0[2], n0[2]));
    if (nn == 0.0f) {
      for (int a = 0; a < 3; ++a) nw[a] = -r.direction[a];
    } else {  // normal_to_world (renderer.cpp:39-41): (W2O.linear^T n).normalized()
      const float* L = ip.w2o;
      for (int a = 0; a < 3; ++a)
        nw[a] = __fadd_rn(__fadd_rn(__fmul_rn(L[a], n0[0]), __fmul_rn(L[4 + a], n0[1])), __fmul_rn(L[8 + a], n0[2]));
      const float len = sqrtf(__fadd_rn(__fadd_rn(__fmul_rn(nw[0], nw[0]), __fmul_rn(nw[1], nw[1])), __fmul_rn(nw[2], nw[2])));
      if (len > 0.0f)
        for (int a = 0; a < 3; ++a) nw[a] = __fdiv_rn(nw[a], len);
    }
    const float dd = __fadd_rn(__fadd_rn(__fmul_rn(nw[0], r.direction[0]), __fmul_rn(nw[1], r.direction[1])),
                               __fmul_rn(nw[2], r.direction[2]));
    for (int a = 0; a < 3; ++a) {
      o.normal[a] = dd > 0.0f ? -nw[a] : nw[a];
      o.albedo[a] = h.albedo[a];
    }
    const int mat = iclamp(static_cast<int>(h.flags_material >> LSNIF_HIT_MATERIAL_SHIFT), 0, m.n_materials - 1);
    o.kind = m.materials[mat].kind;
    o.roughness = m.materials[mat].roughness;
    o.object_index = ip.index;
    o.flags = 1u;
    sh = o;
  } else if (t >= r.t_min && t <= r.t_max) {
    sh.flags = 1u;
    if (sh.object_index < 0) sh.object_index = ip.index;
  }
}

cudaError_t launch_scene_init(const lsnif_ray* rays, int64_t n, const int32_t* n_dev, lsnif_scene_hit* out,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  scene_init_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(rays, n, n_dev, out);
  return cudaGetLastError();
}

cudaError_t launch_broad_phase(const DevModel& m, const InstanceParams& ip, const lsnif_ray* rays, int64_t n,
                               const int32_t* n_dev, lsnif_ray* orays, int32_t* slots, int32_t* count,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  broad_phase_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(m, ip, rays, n, n_dev, orays, slots,
                                                                            count);
  return cudaGetLastError();
}

cudaError_t launch_merge(const DevModel& m, const InstanceParams& ip, const lsnif_ray* rays,
                         const lsnif_hit* hits, const int32_t* slots, const int32_t* count, int64_t n_max,
                         int mode, lsnif_scene_hit* out, cudaStream_t st) {
  if (n_max <= 0) return cudaSuccess;
  merge_kernel<<<static_cast<unsigned>((n_max + 255) / 256), 256, 0, st>>>(m, ip, rays, hits, slots, count, mode, out);
  return cudaGetLastError();
}

// ==================================================== fp32 infer_batch

// One thread per column; exact fp32, sequential sum over the input index
// (the oracle's order), unfused multiply-add.
// lsnif_infer_batch on the tcgen05 MLP: the caller's encoded columns (column
// j = inputs[j * K1 .. + K1), the reference's MatX inputs(K1, n)) become rows
// of the top K bin's X tiles (fp16, times the activation scale, zero past
// K1) with row metadata {j, enter, exit}; the bin's row count is set so
// mlp_tc_kernel answers exactly these rows. An input beyond the bound the
// scale was derived for (|x| > feat_bound: not an encoder output) raises
// *overflow, which hands the whole call to the fp32 kernel below.
__global__ void __launch_bounds__(256) infer_pack_kernel(const DevModel m, const float* __restrict__ x, int64_t n,
                                                         const lsnif_interval* __restrict__ iv, uint8_t* X,
                                                         RowMeta* meta, int32_t* row_counter, int64_t cap_tiles,
                                                         int* overflow) {
  const int top = m.n_bins - 1;
  const int groups = m.K1P / 8;  // 16-byte column groups of a row
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t == 0) row_counter[top] = static_cast<int32_t>(n);
  if (t >= n * groups) return;
  const int64_t j = t / groups;
  const int c0 = static_cast<int>(t - j * groups) * 8;
  const float* xc = x + j * m.K1;
  uint32_t packed[4];
  bool big = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + 2 * q;
    const float a = c < m.K1 ? __ldg(xc + c) : 0.0f;
    const float b = c + 1 < m.K1 ? __ldg(xc + c + 1) : 0.0f;
    big |= !(fabsf(a) <= m.feat_bound) || !(fabsf(b) <= m.feat_bound);
    const __half2 h = __floats2half2_rn(__fmul_rn(a, m.act_scale), __fmul_rn(b, m.act_scale));
    packed[q] = *reinterpret_cast<const uint32_t*>(&h);
  }
  if (big) atomicOr(overflow, 1);
  uint8_t* tile = X + bin_x_offset(top, cap_tiles) + (j >> 7) * static_cast<int64_t>(top + 1) * kBinTileBytes;
  *reinterpret_cast<uint4*>(tile + canon_offset(static_cast<int>(j & 127), c0, kTileM)) =
      make_uint4(packed[0], packed[1], packed[2], packed[3]);
  if (c0 == 0) {
    float4* dst = reinterpret_cast<float4*>(meta + static_cast<int64_t>(top) * cap_tiles * kTileM + j);
    const lsnif_interval v = iv[j];
    dst[0] = make_float4(__int_as_float(static_cast<int32_t>(j)), v.enter, v.exit, 0.0f);
    dst[1] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
}

__global__ void __launch_bounds__(128) infer_f32_kernel(const DevModel m, const float* __restrict__ x,
                                                        int64_t n, const lsnif_interval* __restrict__ iv,
                                                        lsnif_hit* __restrict__ out, const int* only_if) {
  if (only_if && *only_if == 0) return;  // the tcgen05 path answered this call
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int in = m.K1, hid = m.hidden, no = m.n_out;
  const float* w1 = m.w_f32;
  const float* b1 = w1 + hid * in;
  const float* w2 = b1 + hid;
  const float* b2 = w2 + hid * hid;
  const float* w3 = b2 + hid;
  const float* b3 = w3 + no * hid;
  const float* xc = x + j * in;
  float h1[256], h2[256], z[32];
  for (int i = 0; i < hid; ++i) {
    float s = 0.0f;
    for (int k = 0; k < in; ++k) s = __fadd_rn(s, __fmul_rn(w1[i * in + k], xc[k]));
    s = __fadd_rn(s, b1[i]);
    h1[i] = s < 0.0f ? __fmul_rn(s, 0.01f) : s;
  }
  for (int i = 0; i < hid; ++i) {
    float s = 0.0f;
    for (int k = 0; k < hid; ++k) s = __fadd_rn(s, __fmul_rn(w2[i * hid + k], h1[k]));
    s = __fadd_rn(s, b2[i]);
    h2[i] = s < 0.0f ? __fmul_rn(s, 0.01f) : s;
  }
  for (int i = 0; i < no; ++i) {
    float s = 0.0f;
    for (int k = 0; k < hid; ++k) s = __fadd_rn(s, __fmul_rn(w3[i * hid + k], h2[k]));
    z[i] = __fadd_rn(s, b3[i]);
  }
  lsnif_hit h;
  decode_hit(z, m.n_mat, m.occ_threshold, iv[j].enter, iv[j].exit, 0.0f, 0.0f, LSNIF_QUERY_CLOSEST, false, h);
  store_hit(out + j, h);
}

// ================================================================ launch

__global__ void zero_hit_kernel(const DevModel m, lsnif_hit* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    lsnif_hit h;
    decode_hit(m.z_zero, m.n_mat, m.occ_threshold, 0.0f, 1.0f, 0.0f, 0.0f, LSNIF_QUERY_CLOSEST, false, h);
    *out = h;
  }
}

cudaError_t compute_zero_hit(const DevModel& m, lsnif_hit* host_out) {
  lsnif_hit* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(lsnif_hit));
  if (e != cudaSuccess) return e;
  zero_hit_kernel<<<1, 32>>>(m, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(host_out, d, sizeof(lsnif_hit), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e;
}

size_t trace_smem_bytes(const DevModel& m, int warps) {
  return static_cast<size_t>(trace_mask_words(m, warps)) * 4 + static_cast<size_t>(warps) * 64 * 16 +
         static_cast<size_t>(warps) * static_cast<size_t>(m.H) * 32 * 5;
}

size_t mlp_smem_bytes(const DevModel& m, int stages) {
  const size_t x = (static_cast<size_t>(kTileM) * m.K1P * 2 + 1023) & ~size_t(1023);
  // + barriers, TMEM slot, bin tile starts and the scaled b1 (1 KB tail)
  return 1024 + m.w1_bytes + m.w2_bytes + ((m.w3_bytes + 1023) & ~1023u) + kBinTileBytes +
         static_cast<size_t>(stages) * x + 1024 + 2 * MlpLayout<128>::kEpiWarps * 10 * 32 * 4;
}

int mlp_x_stages(const DevModel& m, size_t smem_limit) {
  if (mlp_smem_bytes(m, 4) <= smem_limit) return 4;
  if (mlp_smem_bytes(m, 2) <= smem_limit) return 2;
  return 0;
}

// Raise (never lower) a kernel's dynamic-SMEM limit on the current device:
// host threads launching the same kernel for models of different sizes must
// not shrink it under each other between the attribute call and the launch.
template <typename K>
static cudaError_t ensure_smem(K kern, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = granted[{reinterpret_cast<const void*>(kern), dev}];
  if (smem <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e == cudaSuccess) cur = smem;
  return e;
}

// Per-(kernel, device, smem size) launch configuration, computed once: the
// attribute and occupancy queries cost microseconds of host time per call.
struct LaunchCfg {
  int dev = -1;
  size_t smem = 0;
  int sms = 148, per_sm = 1;
};

template <bool DEBUG, int LS, int FS, bool POW2, int VS, int TW>
static cudaError_t launch_trace_t(const TraceParams& p, cudaStream_t st) {
  auto kern = trace_encode_kernel<DEBUG, LS, FS, POW2, VS, TW>;
  const size_t smem = trace_smem_bytes(p.m, TW);
  thread_local LaunchCfg cfg;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (cfg.dev != dev || cfg.smem != smem) {
    e = ensure_smem(kern, smem);
    if (e != cudaSuccess) return e;
    if (const char* c = std::getenv("LSNIF_TRACE_CARVEOUT")) {  // A/B probe: shared-memory share (%)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(c));
      if (e != cudaSuccess) return e;
    }
    e = cudaDeviceGetAttribute(&cfg.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cfg.per_sm, kern, 32 * TW, smem);
    if (e != cudaSuccess) return e;
    if (const char* c = std::getenv("LSNIF_TRACE_BLOCKS")) cfg.per_sm = std::min(cfg.per_sm, std::atoi(c));
    cfg.dev = dev;
    cfg.smem = smem;
  }
  const int sms = std::max(1, cfg.sms - reserved_sms()), per_sm = cfg.per_sm;
  const int64_t blocks = (p.n + 32 * TW - 1) / (32 * TW);  // one 32-ray batch per warp
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(blocks, static_cast<int64_t>(sms) * std::max(per_sm, 1)));
  kern<<<grid, 32 * TW, smem, st>>>(p);
  return cudaGetLastError();
}

int reserved_sms() {
  static const int r = [] {
    const char* e = std::getenv("LSNIF_RESERVE_SMS");
    const int v = e ? std::atoi(e) : 0;
    return v < 0 ? 0 : (v > 64 ? 64 : v);
  }();
  return r;
}

cudaError_t launch_trace(const TraceParams& p, bool debug, cudaStream_t st) {
  if (p.n <= 0) return cudaSuccess;
  const bool fast = p.m.L == 2 && p.m.F == 3 && p.m.M_pow2 && p.m.V == 32;
  if (debug)
    return fast ? launch_trace_t<true, 2, 3, true, 32, 8>(p, st) : launch_trace_t<true, 0, 0, false, 0, 8>(p, st);
  if (!fast) return launch_trace_t<false, 0, 0, false, 0, 8>(p, st);
  // many waves of 32-ray batches (>= 4 x the ~4.7k resident warps): 1024-thread
  // blocks; a device-side count (scene / renderer queries) may be far below its
  // upper bound p.n, so those keep the one-wave configuration
  // (and only while its SMEM - byte mask + 32 warps' pools - fits the 227 KB
  // per-block opt-in limit: a hit cap H above ~26 does not)
  const bool big = !p.n_dev && p.n >= int64_t(4) * 4736 * 32 && trace_smem_bytes(p.m, 32) <= 232448;
  return big ? launch_trace_t<false, 2, 3, true, 32, 32>(p, st) : launch_trace_t<false, 2, 3, true, 32, 8>(p, st);
}

template <int HID, int NS>
static cudaError_t launch_mlp_t(const MlpParams& p, int max_tiles, int num_sms, cudaStream_t st) {
  const size_t smem = mlp_smem_bytes(p.m, p.m.x_stages);
  const unsigned grid = static_cast<unsigned>(std::min(max_tiles, std::max(1, num_sms - reserved_sms())));
  thread_local LaunchCfg c;
  int dev = 0;
  cudaError_t de = cudaGetDevice(&dev);
  if (de != cudaSuccess) return de;
  if (c.dev != dev || c.smem != smem) {
    cudaError_t e = ensure_smem(mlp_tc_kernel<HID, NS>, smem);
    if (e != cudaSuccess) return e;
    c.dev = dev;
    c.smem = smem;
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(MlpLayout<HID>::kThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // programmatic dependent launch
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, mlp_tc_kernel<HID, NS>, p);
}

cudaError_t launch_mlp(const MlpParams& p, int max_tiles, int num_sms, cudaStream_t st) {
  if (max_tiles <= 0) return cudaSuccess;
  const bool deep = p.m.x_stages >= 4;  // else the 2-stage ring (wide inputs)
  if (p.m.hidden == 128)
    return deep ? launch_mlp_t<128, 4>(p, max_tiles, num_sms, st) : launch_mlp_t<128, 2>(p, max_tiles, num_sms, st);
  if (p.m.hidden == 64)
    return deep ? launch_mlp_t<64, 4>(p, max_tiles, num_sms, st) : launch_mlp_t<64, 2>(p, max_tiles, num_sms, st);
  return cudaErrorNotSupported;
}

cudaError_t launch_infer_f32(const DevModel& m, const float* x, int64_t n, const lsnif_interval* iv,
                             lsnif_hit* out, cudaStream_t st, const int* only_if) {
  if (n <= 0) return cudaSuccess;
  infer_f32_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(m, x, n, iv, out, only_if);
  return cudaGetLastError();
}

cudaError_t launch_infer_pack(const DevModel& m, const float* x, int64_t n, const lsnif_interval* iv, uint8_t* X,
                              RowMeta* meta, int32_t* row_counter, int64_t cap_tiles, int* overflow,
                              cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t total = n * (m.K1P / 8);
  infer_pack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(m, x, n, iv, X, meta, row_counter,
                                                                               cap_tiles, overflow);
  return cudaGetLastError();
}

}  // namespace lsnif_dev

#ifdef LSNIF_PROBE  // A/B probes only, never in the product build
const lsnif_dev::DevModel& lsnif_probe_devmodel(lsnif_model m);
#include "../../scripts/micro/dda_occupancy_probe.cuh"
#endif
