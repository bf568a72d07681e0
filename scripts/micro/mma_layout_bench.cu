// Microbenchmark: tcgen05.mma kind::f16 M=128 N=128 K=16 issue rate with
// SMEM operands in the SWIZZLE_NONE canonical layout vs SWIZZLE_128B K-major.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2504_21627_b200/csrc mma_layout_bench.cu
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for SW128 K-major)
  d |= static_cast<uint64_t>((1024 >> 4) & 0x3FFF) << 32;  // SBO: 8 rows x 128 B
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

__global__ void bench(int layout, int n_tiles, int N, int sts_warps, int rnd, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;            // 128 x 64 fp16 = 16 KB
  uint8_t* sB = base + 16384;    // N x 64 fp16
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (16384 + 16384) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = rnd ? make_uint4(0x3c003800u ^ (i * 2654435761u & 0x83ff83ffu), 0xbc003a00u ^ (i * 40503u & 0x03ff03ffu),
                                                         0x34003000u ^ (i * 97u & 0x03ff03ffu), 0xb800b400u ^ (i * 31u & 0x03ff03ffu))
                                                : make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 256);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp >= 1 && warp <= sts_warps) {  // concurrent SMEM store traffic (like epilogue H writes)
    uint4* dst = reinterpret_cast<uint4*>(base + 32768);
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    int it = 0;
    while (!stop) {
#pragma unroll 8
      for (int q = 0; q < 64; ++q) dst[((it + q) * 32 + (threadIdx.x & 31)) & 2047] = v;
      it += 64;
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t a0 = tc::smem_addr(sA), b0 = tc::smem_addr(sB);
    const uint32_t idesc = tc::idesc_f16_f32(128, N);
    unsigned long long t0 = clock64();
    uint32_t phase = 0;
    for (int t = 0; t < n_tiles; ++t) {
      for (int ks = 0; ks < 4; ++ks) {  // K = 64 per tile
        uint64_t ad, bd;
        if (layout == 0) {  // no swizzle: core matrices, LBO = rows*16 (K chunk), SBO = 128
          ad = tc::smem_desc(a0 + ks * 2 * 2048, 2048, 128);
          bd = tc::smem_desc(b0 + ks * 2 * N * 16, N * 16, 128);
        } else {            // SW128 K-major: rows of 128 B, K step = +32 B
          ad = desc_sw128(a0 + ks * 32);
          bd = desc_sw128(b0 + ks * 32);
        }
        tc::mma_f16_ss(tmem, ad, bd, idesc, (t | ks) ? 1u : 0u);
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, phase);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 256); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  for (int rnd : {0, 1}) for (int sts : {0}) for (int N : {128, 16}) for (int layout = 0; layout < 1; ++layout) {
    for (int rep = 0; rep < 2; ++rep) {
      const int tiles = 512;
      bench<<<148, 128, 80000>>>(layout, tiles, N, sts, rnd, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      if (rep) printf("random=%d sts_warps=%d N=%d layout=%s: %.1f cycles per MMA (K=16) [%s]\n", rnd, sts, N, layout ? "SW128" : "NONE",
                      avg / (tiles * 4), cudaGetErrorString(e));
    }
  }
  return 0;
}
