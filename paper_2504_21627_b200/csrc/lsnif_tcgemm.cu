// fp32 GEMM on the 5th-generation tensor cores for GPU training (F4): the
// forward and backward contractions of train()'s MLP (mlp.hpp:117-130,
// 206-225; training.cpp:153-216), replacing SIMT SGEMM.
//
//   C(m, n) = sum_k A(m, k) B(n, k)        (+ C when accumulate)
//
// Every operand is an arbitrary-strided fp32 view (A(m, k) = A[m sam + k sak]
// and so on), so the nine contractions of a training step (W x, W^T dz,
// h dz^T, ...) need no transposed copies. Accuracy is fp32-class through the
// split-TF32 scheme: each operand is split into a TF32 head and a TF32 tail
// (x = hi + lo, hi = x with the low 13 mantissa bits cleared, lo = x - hi
// exact in fp32), and the tile product is hi.hi + hi.lo + lo.hi, three
// tcgen05.mma.kind::tf32 per K-step into one fp32 TMEM accumulator (the
// dropped lo.lo term is ~2^-22 relative). Reductions over the batch (the
// weight gradients, K = batch) are split across CTAs into a partial buffer
// and summed in split order by a second kernel (deterministic).
//
// Tile: 128 (M, TMEM lanes) x 128 (N, TMEM columns) x 32 (K per stage), two
// SMEM stages of {A_hi, A_lo, B_hi, B_lo} in the canonical K-major layout
// (8-row x 16-byte core matrices). 128 threads: all load + split the next
// stage while thread 0's MMAs of the current one run; then warp w reads TMEM
// lanes [32w, 32w + 32) in the epilogue.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>
#include <vector>

#include "lsnif_internal.hpp"
#include "tc_ptx.cuh"

namespace lsnif_tr {

namespace {

constexpr int kBM = 128, kBK = 32;
constexpr int kThreads = 128;
constexpr uint32_t kOpBytes = kBM * kBK * 4;  // one A operand tile (16 KB)
// per stage: A_hi, A_lo (kBM rows), B_hi, B_lo (BN rows)
template <int BN>
__host__ __device__ constexpr uint32_t stage_bytes() { return 2 * kOpBytes + 2 * BN * kBK * 4; }
template <int BN>
__host__ __device__ constexpr uint32_t smem_bytes() { return 2 * stage_bytes<BN>() + 1024 + 64; }

// Instruction descriptor, kind::tf32: A = B = TF32, D = F32, K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Byte offset of element (row r, k) in a ROWS-row K-major canonical tile of
// 4-byte elements: core matrices of 8 rows x 16 B, rows-groups 128 B apart
// (SBO), K-groups of 4 elements ROWS x 16 B apart (LBO).
template <int ROWS>
__device__ __forceinline__ uint32_t canon32(int r, int k) {
  return static_cast<uint32_t>((k >> 2) * (ROWS * 16) + (r >> 3) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

struct GemmArgs {
  const float* A;
  int64_t sam, sak;
  const float* B;
  int64_t sbn, sbk;
  float* C;  // C or the split partials (split s at C + s * M * N, row-major M x N)
  int64_t scm, scn;
  int M, N, K;
  int k_per_split;  // K range of one split (multiple of kBK)
  int accumulate;   // C += (single split only)
  int partial;      // write split partials instead of C
};

// VA / VB: the operand is k-contiguous with 16-byte aligned rows (stride 1
// along k, row stride a multiple of 4 floats): 16-byte loads.
template <int BN, bool VA, bool VB>
__global__ void __launch_bounds__(kThreads, BN == 64 ? 2 : 1) tcgemm_kernel(const GemmArgs g) {
  constexpr uint32_t kStageBytes = stage_bytes<BN>();
  constexpr uint32_t kBOpBytes = BN * kBK * 4;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* done = reinterpret_cast<uint64_t*>(base + 2 * kStageBytes);  // per stage
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
  const int k_begin = blockIdx.z * g.k_per_split;
  const int k_end = min(g.K, k_begin + g.k_per_split);
  if (tid == 0) {
    tc::mbar_init(done, 1);
    tc::mbar_init(done + 1, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(tmem_slot, BN);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = idesc_tf32(kBM, BN);

  // one stage: every thread loads and splits 32 elements of each operand
  // (thread t: row r = t, all 32 k of the stage; for operands stored
  // k-fastest a thread walks one 128-byte line, otherwise the 128 rows of a k
  // are 128 consecutive threads) and stores them as 16-byte core-matrix rows
  auto split_store = [&](uint8_t* hi, uint8_t* lo, uint32_t off, const float* v) {
    float4 h, l;
    float* ph = &h.x;
    float* pl = &l.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ph[q] = __uint_as_float(__float_as_uint(v[q]) & 0xffffe000u);
      pl[q] = v[q] - ph[q];
    }
    *reinterpret_cast<float4*>(hi + off) = h;  // 4 consecutive k = one 16-byte core-matrix row
    *reinterpret_cast<float4*>(lo + off) = l;
  };
  auto load_stage = [&](int s, int k0) {
    uint8_t* st = base + s * kStageBytes;
    // A: thread t loads row t, all kBK k; B: row t % BN, kBK * BN / 128 k
    constexpr int kBk = kBK * BN / kThreads;
    const int m = m0 + tid;
    const int rb = tid % BN, kb0 = (tid / BN) * kBk;
    const int n = n0 + rb;
    float a[kBK], b[kBk];  // all of the stage's loads in flight before any split / store
    // 4 consecutive k of one row: a 16-byte load when the operand allows it
    // and the group lies inside the K range, else element by element
    auto load4 = [&](auto VEC, const float* base_row, int64_t sk, bool row_ok, int k, float* dst) {
      if (decltype(VEC)::value && row_ok && k + 3 < k_end) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(base_row + k));
        dst[0] = v.x;
        dst[1] = v.y;
        dst[2] = v.z;
        dst[3] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = (row_ok && k + q < k_end) ? __ldg(base_row + (k + q) * sk) : 0.0f;
      }
    };
    const float* arow = g.A + static_cast<int64_t>(m < g.M ? m : 0) * g.sam;
    const float* brow = g.B + static_cast<int64_t>(n < g.N ? n : 0) * g.sbn;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4)
      load4(std::integral_constant<bool, VA>{}, arow, g.sak, m < g.M, k0 + kk, a + kk);
#pragma unroll
    for (int kk = 0; kk < kBk; kk += 4)
      load4(std::integral_constant<bool, VB>{}, brow, g.sbk, n < g.N, k0 + kb0 + kk, b + kk);
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) split_store(st, st + kOpBytes, canon32<kBM>(tid, kk), a + kk);
#pragma unroll
    for (int kk = 0; kk < kBk; kk += 4)
      split_store(st + 2 * kOpBytes, st + 2 * kOpBytes + kBOpBytes, canon32<BN>(rb, kb0 + kk), b + kk);
    tc::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
  };

  const int nst = (k_end - k_begin + kBK - 1) / kBK;
  uint32_t ph[2] = {0u, 0u};
  if (nst > 0) load_stage(0, k_begin);
  for (int i = 0; i < nst; ++i) {
    const int s = i & 1;
    __syncthreads();  // stage s written by every thread
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t st = tc::smem_addr(base + s * kStageBytes);
#pragma unroll
      for (int ks = 0; ks < kBK / 8; ++ks) {  // 8 TF32 K per MMA = 2 core matrices
        const uint32_t koff = ks * 2 * (kBM * 16);
        const uint64_t ah = tc::smem_desc(st + koff, kBM * 16, 128);
        const uint64_t al = tc::smem_desc(st + kOpBytes + koff, kBM * 16, 128);
        const uint32_t kboff = ks * 2 * (BN * 16);
        const uint64_t bh = tc::smem_desc(st + 2 * kOpBytes + kboff, BN * 16, 128);
        const uint64_t bl = tc::smem_desc(st + 2 * kOpBytes + kBOpBytes + kboff, BN * 16, 128);
        const uint32_t acc0 = (i > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, al, bh, idesc, acc0);  // small terms first
        mma_tf32(tmem, ah, bl, idesc, 1u);
        mma_tf32(tmem, ah, bh, idesc, 1u);
      }
      tc::mma_commit(done + s);
    }
    if (i + 1 < nst) {
      const int s1 = (i + 1) & 1;
      if (i >= 1) {  // stage s1 was read by the MMAs of step i - 1
        tc::mbar_wait(done + s1, ph[s1]);
        ph[s1] ^= 1u;
      }
      load_stage(s1, k_begin + (i + 1) * kBK);
    }
  }
  if (nst > 0) {  // the last commit covers every MMA
    const int s = (nst - 1) & 1;
    tc::mbar_wait(done + s, ph[s]);
  }
  tc::tc_fence_after();

  // epilogue: warp w owns TMEM lanes (rows) [32 w, 32 w + 32)
  const int m = m0 + 32 * warp + lane;
  const uint32_t lanes = static_cast<uint32_t>(32 * warp) << 16;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    uint32_t v[32];
    if (nst > 0) {
      tc::tmem_ld32(tmem + lanes + c, v);
      tc::tmem_wait_ld();
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0u;
    }
    if (m < g.M) {
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const int n = n0 + c + j;
        if (n >= g.N) break;
        const float x = __uint_as_float(v[j]);
        if (g.partial) {
          g.C[static_cast<int64_t>(blockIdx.z) * g.M * g.N + static_cast<int64_t>(m) * g.N + n] = x;
        } else {
          float* dst = g.C + m * g.scm + n * g.scn;
          *dst = g.accumulate ? *dst + x : x;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, BN);
}

// C(m, n) (+)= sum over splits of the partials, in split order.
__global__ void split_sum_kernel(const float* __restrict__ part, int splits, int M, int N, float* C, int64_t scm,
                                 int64_t scn, int accumulate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(M) * N) return;
  float s = 0.0f;
  for (int z = 0; z < splits; ++z) s += part[static_cast<int64_t>(z) * M * N + i];
  const int m = static_cast<int>(i / N), n = static_cast<int>(i % N);
  float* dst = C + m * scm + n * scn;
  *dst = accumulate ? *dst + s : s;
}

}  // namespace

// Column-major BLAS-style entry used by the trainer: C (mm x nn, leading
// dimension ldc) = op(A) op(B), op = transpose when the flag is set, A / B
// column-major with leading dimensions lda / ldb (cublasSgemm semantics,
// alpha = 1, beta = 0). `work` holds split partials (work_floats floats).
cudaError_t tcgemm_colmajor(bool ta, bool tb, int mm, int nn, int kk, const float* A, int lda, const float* B, int ldb,
                            float* C, int ldc, float* work, size_t work_floats, int num_sms, cudaStream_t st) {
  if (mm <= 0 || nn <= 0) return cudaSuccess;
  // 128 x 128 output tiles (128 x 64 tiles, two CTAs per SM, measured slower
  // on the training step: 2.80 vs 2.69 ms at batch 65,536)
  constexpr int bn = 128;
  GemmArgs g{};
  // op(A)(m, k): column-major A is A[i + j lda]; op(A) = A -> (m, k) = A[m + k lda]
  g.A = A;
  g.sam = ta ? lda : 1;
  g.sak = ta ? 1 : lda;
  // C(m, n) = sum_k op(A)(m, k) op(B)(k, n); the kernel's B(n, k) = op(B)(k, n)
  g.B = B;
  g.sbn = tb ? 1 : ldb;
  g.sbk = tb ? ldb : 1;
  g.C = C;
  g.scm = 1;
  g.scn = ldc;
  g.M = mm;
  g.N = nn;
  g.K = kk;
  const int tiles = ((mm + kBM - 1) / kBM) * ((nn + bn - 1) / bn);
  // split the reduction when the output tiles alone leave SMs idle
  int splits = 1;
  const int kst = (kk + kBK - 1) / kBK;
  if (tiles < num_sms && kst > 4) {
    splits = std::min(std::max(num_sms / tiles, 1), kst / 4);
    while (splits > 1 && static_cast<size_t>(splits) * mm * nn > work_floats) --splits;
  }
  const int steps_per = (kst + splits - 1) / splits;
  splits = (kst + steps_per - 1) / steps_per;
  g.k_per_split = steps_per * kBK;
  g.accumulate = 0;
  g.partial = splits > 1;
  if (splits > 1) g.C = work;
  dim3 grid((mm + kBM - 1) / kBM, (nn + bn - 1) / bn, splits);
  auto aligned = [](const float* p, int64_t row_stride, int64_t k_stride) {
    return k_stride == 1 && row_stride % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  };
  const bool va = aligned(A, g.sam, g.sak), vb = aligned(B, g.sbn, g.sbk);
  auto launch = [&](auto kern) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem_bytes<bn>()));  // per device; cheap
    if (err != cudaSuccess) return err;
    kern<<<grid, kThreads, smem_bytes<bn>(), st>>>(g);
    return cudaGetLastError();
  };
  cudaError_t e = va ? (vb ? launch(tcgemm_kernel<bn, true, true>) : launch(tcgemm_kernel<bn, true, false>))
                     : (vb ? launch(tcgemm_kernel<bn, false, true>) : launch(tcgemm_kernel<bn, false, false>));
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = static_cast<int64_t>(mm) * nn;
  split_sum_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(work, splits, mm, nn, C, 1, ldc, 0);
  return cudaGetLastError();
}

}  // namespace lsnif_tr
