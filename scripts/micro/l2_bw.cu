// L2 bandwidth microbenchmark (B200, sm_100a): the L2 peak is not in
// MEASURED_PEAKS.json. (1) streaming 16-byte loads over an L2-resident 48 MB
// buffer; (2) random 8-byte gathers from a 2 MiB table (the hash-grid level
// size), the trace kernel's access pattern. Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stream_kernel(const float4* __restrict__ a, size_t n, int reps, float* out) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(a + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void gather_kernel(const uint2* __restrict__ t, unsigned mask, int iters, unsigned* out) {
  unsigned h = blockIdx.x * 2654435761u + threadIdx.x * 805459861u, acc = 0;
  for (int i = 0; i < iters; ++i) {
    h = h * 1664525u + 1013904223u;
    const uint2 v = __ldcg(t + ((h >> 7) & mask));
    acc ^= v.x + v.y;
  }
  if (acc == 0x12345u) out[0] = acc;
}

int main() {
  const size_t bytes = 48ull << 20, n = bytes / 16;
  float4* a;
  float* o;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 0, bytes);
  cudaMalloc(&o, 64);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  stream_kernel<<<sms * 8, 512>>>(a, n, 2, o);
  cudaEventRecord(e0);
  stream_kernel<<<sms * 8, 512>>>(a, n, reps, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"l2_stream_read_GBps\": %.1f, ", (double)bytes * reps / (ms * 1e-3) / 1e9);
  const unsigned entries = (2u << 20) / 8;  // 2 MiB table of 8-byte entries
  uint2* t;
  cudaMalloc(&t, entries * 8);
  cudaMemset(t, 1, entries * 8);
  const int iters = 4096;
  gather_kernel<<<sms * 16, 256>>>(t, entries - 1, 64, (unsigned*)o);
  cudaEventRecord(e0);
  gather_kernel<<<sms * 16, 256>>>(t, entries - 1, iters, (unsigned*)o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double loads = (double)sms * 16 * 256 * iters;
  printf("\"gather8_Gloads_per_s\": %.1f, \"gather8_useful_GBps\": %.1f, \"gather8_sector_GBps\": %.1f}\n",
         loads / (ms * 1e-3) / 1e9, loads * 8 / (ms * 1e-3) / 1e9, loads * 32 / (ms * 1e-3) / 1e9);
  return 0;
}
