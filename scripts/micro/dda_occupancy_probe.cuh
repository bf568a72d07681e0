// DDA-only occupancy / ordering probe (built into an A/B library with
// -DLSNIF_PROBE, never into the product): the trace kernel's walk (frame clip,
// walk_setup, the byte-stop-code DDA loop with its emits reduced to a
// checksum) at 32 / 48 / 64 warps per SM, to measure how far a walk-only
// kernel with more resident warps gets on incoherent rays in input order and
// in walk-length order. Included at the end of lsnif_kernels.cu.
namespace lsnif_dev {
template <int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) dda_probe_kernel(const DevModel m, const lsnif_ray* rays, int64_t n,
                                                                uint32_t* out) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int code_words = m.stop2_words;
  for (int i = threadIdx.x; i < code_words * 4; i += blockDim.x) {
    const uint32_t w = __ldg(m.stop2 + (i >> 2)) >> ((i & 3) * 8);
    smem[i] = (w & 3u) | ((w & 0xcu) << 6) | ((w & 0x30u) << 12) | ((w & 0xc0u) << 18);
  }
  __syncthreads();
  const uint8_t* codes = reinterpret_cast<const uint8_t*>(smem);
  const int H = m.H;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * BLOCK + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * BLOCK) {
    const float4* r4 = reinterpret_cast<const float4*>(rays + i);
    const float4 ra = __ldg(r4), rb = __ldg(r4 + 1);
    float o[3] = {ra.x, ra.y, ra.z}, d[3] = {ra.w, rb.x, rb.y};
    float enter, exit;
    uint32_t sum = 0;
    int count = 0;
    Walk w;
    if (frame_interval(m, o, d, rb.z, rb.w, enter, exit) && walk_setup<32>(m, o, d, rb.z, w)) {
      if (codes[w.idx]) {
        sum = __float_as_uint(w.t0);
        count = 1;
      }
      float tn;
      if (count < H && w.t1 != -__int_as_float(0x7f800000)) {
        int dl = walk_advance_dl(w, tn);
        for (;;) {
          const uint32_t sc = codes[w.idx];
          if (sc != 0u) {
            if (sc > 1u || tn > w.t1) break;
            sum = sum * 31u + (__float_as_uint(tn) ^ static_cast<uint32_t>(dl));
            if (++count >= H) break;
          }
          dl = walk_advance_dl(w, tn);
        }
      }
    }
    out[i] = sum ^ static_cast<uint32_t>(count) << 24;
  }
}
}  // namespace lsnif_dev

extern "C" int lsnif_probe_dda(lsnif_model model, const lsnif_ray* d_rays, int64_t n, uint32_t* d_out, int warps_per_sm,
                               float* ms) {
  using namespace lsnif_dev;
  const DevModel& m = lsnif_probe_devmodel(model);
  const size_t smem = static_cast<size_t>(m.stop2_words) * 16;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, int per_sm) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const unsigned grid = 148u * per_sm;
    kern<<<grid, 512, smem>>>(m, d_rays, n, d_out);  // warm-up
    cudaEventRecord(a);
    kern<<<grid, 512, smem>>>(m, d_rays, n, d_out);
    cudaEventRecord(b);
  };
  if (warps_per_sm == 32) run(dda_probe_kernel<512, 2>, 2);
  else if (warps_per_sm == 48) run(dda_probe_kernel<512, 3>, 3);
  else run(dda_probe_kernel<512, 4>, 4);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return static_cast<int>(cudaGetLastError());
}
