// Host <-> kernel interface of liblsnif_gpu (not part of the public ABI).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>

#include "lsnif_device.cuh"

// Error plumbing shared by the C-ABI translation units: entry points throw
// ApiError and the guarded() wrapper in lsnif_capi.cu turns it into a status
// plus the thread-local message.
namespace lsnif_api {
struct ApiError {
  lsnif_status st;
  std::string msg;
};
[[noreturn]] inline void fail(lsnif_status st, const std::string& msg) { throw ApiError{st, msg}; }
inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(LSNIF_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace lsnif_api

namespace lsnif_dev {

struct TraceParams {
  DevModel m;
  const lsnif_ray* rays;
  const lsnif_interval* intervals;  // optional pair intervals (run_narrow_phase's t_enter/t_exit)
  int64_t n;                  // rays in this launch (upper bound when n_dev is set)
  const int32_t* n_dev;       // optional device-side ray count of the whole query
  int64_t offset;             // first ray of this launch within the query
  int mode;
  void* out;                  // lsnif_hit[] or (wire) lsnif_hit_wire[]
  int wire;
  uint8_t* X;                 // compacted MLP operand tiles, per K bin (bin_x_offset)
  RowMeta* meta;              // bin b's rows at meta + b * cap_tiles * 128
  int32_t* row_counter;       // one per K bin
  int64_t cap_tiles;          // tiles per bin region
  unsigned long long* batch_counter;  // dynamic 32-ray batch claims (zeroed per launch)
  unsigned long long* stats;  // pairs, rows, points, volume points
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
  const int32_t* row_counter;  // one per K bin
  int64_t cap_tiles;
  void* out;             // lsnif_hit[] or (wire) lsnif_hit_wire[]
  int wire;
  int mode;
  const int32_t* n_dev;  // optional device-side ray count of the query (as TraceParams)
  int64_t offset;        // first ray of this chunk within the query
};

// Multi-object scenes: one instance's placement.
struct InstanceParams {
  float w2o[12];
  int32_t index;
};

// One instance's broad-phase data (device array, one entry per instance).
struct InstanceBox {
  float w2o[12];
  float mn[3], mx[3];  // the model's frame box
  const lsnif_material* materials;  // the model's material table (DEVICE), for the merge
  int32_t n_materials;
};

// collect_pairs for every instance in one pass over the rays (scene_init
// fused): instance k's object-space rays / slots at orays / slots + k * stride,
// its pair count at counts[k].
// best (nullable): per-ray merge keys, reset to ~0 here for merge_all.
cudaError_t launch_broad_phase_all(const InstanceBox* boxes, int n_inst, const lsnif_ray* rays, int64_t n,
                                   const int32_t* n_dev, lsnif_ray* orays, int32_t* slots, int64_t stride,
                                   int32_t* counts, lsnif_scene_hit* out, unsigned long long* best,
                                   cudaStream_t st);
// Accept + merge of every instance's neural hits in two launches (closest:
// 64-bit atomicMin of (t, pair index) per ray, then the winner's SurfaceHit;
// any: lowest occluding instance). Needs n_inst * stride < 2^32.
cudaError_t launch_merge_all(const InstanceBox* boxes, int n_inst, const lsnif_ray* rays, int64_t n,
                             const int32_t* n_dev, const lsnif_hit* hits, const int32_t* slots, int64_t stride,
                             const int32_t* counts, int mode, unsigned long long* best, lsnif_scene_hit* out,
                             cudaStream_t st);

size_t trace_smem_bytes(const DevModel& m, int warps_per_block);
cudaError_t compute_zero_hit(const DevModel& m, lsnif_hit* host_out);  // decode of z_zero, enter 0, exit 1
// n_dev (nullable): device-side ray count, n its upper bound
cudaError_t launch_scene_init(const lsnif_ray* rays, int64_t n, const int32_t* n_dev, lsnif_scene_hit* out,
                              cudaStream_t st);
cudaError_t launch_broad_phase(const DevModel& m, const InstanceParams& ip, const lsnif_ray* rays, int64_t n,
                               const int32_t* n_dev, lsnif_ray* orays, int32_t* slots, int32_t* count,
                               cudaStream_t st);
cudaError_t launch_merge(const DevModel& m, const InstanceParams& ip, const lsnif_ray* rays,
                         const lsnif_hit* hits, const int32_t* slots, const int32_t* count, int64_t n_max,
                         int mode, lsnif_scene_hit* out, cudaStream_t st);
size_t mlp_smem_bytes(const DevModel& m, int x_stages);
// Deepest X ring (4..2 stages) whose SMEM fits smem_limit; 0 if none does.
int mlp_x_stages(const DevModel& m, size_t smem_limit);
// SMs the persistent query kernels leave free (LSNIF_RESERVE_SMS, read once;
// default 0). Both query kernels fill every SM they are given (the trace
// kernel's 1024-thread block takes the whole register file, the MLP CTA most
// of the shared memory), so a collective's kernels launched concurrently on
// another stream (the multi-GPU result gather) would otherwise wait for the
// query to finish instead of overlapping it.
int reserved_sms();
cudaError_t launch_trace(const TraceParams& p, bool debug, cudaStream_t st);
cudaError_t launch_mlp(const MlpParams& p, int max_tiles, int num_sms, cudaStream_t st);
cudaError_t launch_infer_pack(const DevModel& m, const float* x, int64_t n, const lsnif_interval* iv, uint8_t* X,
                              RowMeta* meta, int32_t* row_counter, int64_t cap_tiles, int* overflow,
                              cudaStream_t st);
cudaError_t launch_infer_f32(const DevModel& m, const float* x, int64_t n, const lsnif_interval* iv,
                             lsnif_hit* out, cudaStream_t st, const int* only_if = nullptr);

}  // namespace lsnif_dev

// Scene query with a device-side ray count (n_max bounds it): no host sync,
// so a caller can enqueue dependent work (lsnif_capi.cu).
namespace lsnif_api {
void scene_query_async(lsnif_scene scene, const lsnif_ray* d_rays, int64_t n_max, const int32_t* d_n, int mode,
                       lsnif_scene_hit* d_hits, cudaStream_t st);
}  // namespace lsnif_api

// Wavefront path tracer (lsnif_render.cu), driven by lsnif_render in lsnif_capi.cu.
namespace lsnif_pt {
struct Workspace;  // per (scene, stream) path-state buffers, reused across renders
struct WorkspaceDeleter {
  void operator()(Workspace* w) const;
};
using WorkspacePtr = std::unique_ptr<Workspace, WorkspaceDeleter>;
void render(WorkspacePtr& ws, lsnif_scene scene, const float* world_diag, int n_instances, const lsnif_camera& camera,
            const lsnif_light* lights, int n_lights, const float environment[3],
            const lsnif_render_config& cfg, float* d_image, lsnif_render_stats* stats, cudaStream_t st);
void debug_paths(const lsnif_camera& camera, const lsnif_render_config& cfg, int64_t first_path,
                 int64_t n, lsnif_ray* d_rays, float* d_uniforms, int k, cudaStream_t st);
}  // namespace lsnif_pt

// GPU trainer (lsnif_train.cu), driven by the lsnif_trainer_* entry points.
namespace lsnif_api {
void* trainer_create(const lsnif_model_desc& d, const lsnif_mesh_desc& mesh, const lsnif_train_config& cfg,
                     int device, lsnif_model geo, const lsnif_dev::DevModel& dm);
void trainer_destroy(void* t);
void trainer_step(void* t, int steps, lsnif_train_loss* last, cudaStream_t st);
void trainer_batch_grad(void* t, const lsnif_ray* rays, const lsnif_train_target* tg, int64_t n,
                        lsnif_train_loss* loss, float* g_mlp, float* g_tab, cudaStream_t st);
void trainer_sample(void* t, int64_t step, int64_t n, lsnif_ray* rays, lsnif_train_target* tg, cudaStream_t st);
void trainer_export(void* t, int device, lsnif_model* out);
}  // namespace lsnif_api
