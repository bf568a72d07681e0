// Replicates mlp_tc_kernel's MMA stream (per tile: L1 7 K-steps N=128 from an
// X stage, L2 9 K-steps N=128 and L3 8 K-steps N=16 from an H buffer, two
// alternating TMEM accumulators) with the kernel's SMEM offsets, and variants.
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

__global__ void bench(int variant, int n_tiles, const uint8_t* gsrc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // kernel layout: W1 28672 | W2 36864 | W3 (4096 -> 5120) | X 2 x 28672 | H 2 x 36864
  uint8_t* sW1 = base;
  uint8_t* sW2 = sW1 + 28672;
  uint8_t* sW3 = sW2 + 36864;
  uint8_t* sX = sW3 + 5120;
  uint8_t* sH = sX + 2 * 28672;
  __shared__ uint64_t bar;
  __shared__ uint64_t lbar[2];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (28672 + 36864 + 5120 + 2 * 28672 + 2 * 36864) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::mbar_init(&lbar[0], 1); tc::mbar_init(&lbar[1], 1); tc::fence_mbar_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc(&slot, 256);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  __shared__ volatile int stop;
  __shared__ uint64_t tbar;
  if (threadIdx.x == 0) { stop = 0; tc::mbar_init(&tbar, 1); tc::fence_mbar_init(); }
  __syncthreads();
  if ((variant & 32) && threadIdx.x == 32) {  // concurrent TMA bulk copies into the X stages
    uint32_t ph = 0;
    int i = 0;
    while (!stop) {
      tc::mbar_arrive_expect_tx(&tbar, 28672);
      tc::bulk_g2s(sX + (i & 1) * 28672, gsrc + (static_cast<size_t>(blockIdx.x) * 64 + (i & 63)) * 28672, 28672, &tbar);
      tc::mbar_wait(&tbar, ph);
      ph ^= 1;
      ++i;
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t w1 = tc::smem_addr(sW1), w2 = tc::smem_addr(sW2), w3 = tc::smem_addr(sW3);
    const uint32_t x0 = tc::smem_addr(sX), h0 = tc::smem_addr(sH);
    const uint32_t i128 = tc::idesc_f16_f32(128, 128), i16 = tc::idesc_f16_f32(128, 16);
    auto layer = [&](uint32_t a, int ks_n, uint32_t b, uint32_t brows, uint32_t idesc, uint32_t d) {
      if (variant & 16) tc::tc_fence_after();
      for (int ks = 0; ks < ks_n; ++ks) {
        const uint64_t ad = tc::smem_desc(a + ks * 2 * 2048, 2048, 128);
        const uint64_t bd = tc::smem_desc(b + ks * 2 * brows * 16, brows * 16, 128);
        tc::mma_f16_ss(d, ad, bd, idesc, ks > 0 ? 1u : 0u);
      }
      if (variant & 8) tc::mma_commit(&lbar[(d >> 7) & 1]);
    };
    unsigned long long t0 = clock64();
    for (int t = 0; t < n_tiles; ++t) {
      const int g = (variant & 1) ? (t & 1) : 0;        // bit0: alternate accumulators
      const uint32_t d = tmem + g * 128;
      const uint32_t xa = x0 + ((variant & 2) ? g : 0) * 28672;
      const uint32_t ha = h0 + ((variant & 2) ? g : 0) * 36864;
      layer(xa, 7, w1, 128, i128, d);
      layer(ha, 9, w2, 128, i128, d);
      if (variant & 4) layer(ha, 8, w3, 16, i16, d);     // bit2: include the N=16 layer
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc::tc_fence_after(); tc::tmem_dealloc(tmem, 256); }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 202 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint8_t* g;
  cudaMalloc(&g, size_t(148) * 64 * 28672);
  cudaMemset(g, 0, size_t(148) * 64 * 28672);
  for (int tiles : {256, 10240}) for (int v : {7}) {
    for (int rep = 0; rep < 2; ++rep) {
      bench<<<148, 128, smem>>>(v, tiles, g, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      const int mmas = 16 + ((v & 4) ? 8 : 0);
      if (rep) printf("tiles/CTA %d: %.0f cycles/tile, %.1f per MMA [%s]\n", tiles, avg / tiles,
                      avg / tiles / mmas, cudaGetErrorString(e));
    }
  }
  return 0;
}
