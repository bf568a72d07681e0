// Host <-> kernel interface of liblsnif_gpu (not part of the public ABI).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lsnif_device.cuh"

namespace lsnif_dev {

struct TraceParams {
  DevModel m;
  const lsnif_ray* rays;
  int64_t n;
  int mode;
  lsnif_hit* out;
  uint8_t* X;                 // compacted MLP operand tiles
  RowMeta* meta;
  int32_t* row_counter;
  unsigned long long* batch_counter;  // dynamic 32-ray batch claims (zeroed per launch)
  unsigned long long* stats;  // pairs, rows, points, volume points
  uint32_t tile_bytes;
  // debug probe (DEBUG=true only)
  int32_t* info;
  float* interval;
  float* t;
  float* pts;
  uint32_t* cells;
  uint32_t* hidx;
  float* feat;
};

struct MlpParams {
  DevModel m;
  const uint8_t* X;
  const RowMeta* meta;
  const int32_t* row_counter;
  lsnif_hit* out;
  uint32_t tile_bytes;
  int mode;
};

size_t trace_smem_bytes(const DevModel& m);
size_t mlp_smem_bytes(const DevModel& m);
cudaError_t launch_trace(const TraceParams& p, bool debug, cudaStream_t st);
cudaError_t launch_mlp(const MlpParams& p, int max_tiles, int num_sms, cudaStream_t st);
cudaError_t launch_infer_f32(const DevModel& m, const float* x, int64_t n, const lsnif_interval* iv,
                             lsnif_hit* out, cudaStream_t st);

}  // namespace lsnif_dev
