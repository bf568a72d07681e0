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
  int64_t n;                  // rays in this launch (upper bound when n_dev is set)
  const int32_t* n_dev;       // optional device-side ray count of the whole query
  int64_t offset;             // first ray of this launch within the query
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

// Multi-object scenes: one instance's placement.
struct InstanceParams {
  float w2o[12];
  int32_t index;
};

size_t trace_smem_bytes(const DevModel& m);
cudaError_t compute_zero_hit(const DevModel& m, lsnif_hit* host_out);  // decode of z_zero, enter 0, exit 1
cudaError_t launch_scene_init(const lsnif_ray* rays, int64_t n, lsnif_scene_hit* out, cudaStream_t st);
cudaError_t launch_broad_phase(const DevModel& m, const InstanceParams& ip, const lsnif_ray* rays, int64_t n,
                               lsnif_ray* orays, int32_t* slots, int32_t* count, cudaStream_t st);
cudaError_t launch_merge(const DevModel& m, const InstanceParams& ip, const lsnif_ray* rays,
                         const lsnif_hit* hits, const int32_t* slots, const int32_t* count, int64_t n_max,
                         int mode, lsnif_scene_hit* out, cudaStream_t st);
size_t mlp_smem_bytes(const DevModel& m);
cudaError_t launch_trace(const TraceParams& p, bool debug, cudaStream_t st);
cudaError_t launch_mlp(const MlpParams& p, int max_tiles, int num_sms, cudaStream_t st);
cudaError_t launch_infer_f32(const DevModel& m, const float* x, int64_t n, const lsnif_interval* iv,
                             lsnif_hit* out, cudaStream_t st);

}  // namespace lsnif_dev
