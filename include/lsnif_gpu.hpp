// lsnif_gpu.hpp — header-only C++ host adapter over the C ABI (lsnif_gpu.h).
//
// Re-declares (does not copy) the reference's query surface
// (proj/include/lsnif/renderer.hpp:42-53, 110-116) so a caller of the CPU
// narrow phase can switch to the B200 path:
//   lsnif::gpu::Model            ~ std::shared_ptr<const LsnifModel> + upload
//   lsnif::gpu::infer_batch      ~ infer_batch (renderer.hpp:52-53)
//   lsnif::gpu::intersect        ~ the narrow phase + accept of intersect_scene
//                                  for one object (renderer.cpp:269-303)
//   lsnif::gpu::occluded_batch   ~ occluded_batch (renderer.cpp:305-323)
//   lsnif::gpu::Scene            ~ the LSNIF objects of PreparedScene
//                                  (renderer.hpp:80-131): intersect_scene /
//                                  occluded_batch over world rays
//   lsnif::gpu::render           ~ render() (renderer.cpp:453-542),
//                                  PrimaryMode::lsnif
//   lsnif::gpu::Trainer          ~ train() (training.cpp:95-230) on the GPU
// Errors are rethrown as the reference's exception types:
// std::invalid_argument for LSNIF_INVALID_ARGUMENT, std::runtime_error
// otherwise.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "lsnif_gpu.h"

namespace lsnif {
namespace gpu {

inline void check(lsnif_status st) {
  if (st == LSNIF_OK) return;
  const std::string msg = lsnif_last_error();
  if (st == LSNIF_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// renderer.hpp:42-48
struct NeuralHit {
  bool occluded = false;
  float t_world = 0;
  float normal[3] = {0, 0, 0};
  float albedo[3] = {0, 0, 0};
  int material_index = 0;
};

inline NeuralHit to_neural_hit(const lsnif_hit& h) {
  NeuralHit n;
  n.occluded = (h.flags_material & LSNIF_HIT_OCCLUDED) != 0;
  n.t_world = h.t_world;
  for (int k = 0; k < 3; ++k) {
    n.normal[k] = h.normal[k];
    n.albedo[k] = h.albedo[k];
  }
  n.material_index = static_cast<int>(h.flags_material >> LSNIF_HIT_MATERIAL_SHIFT);
  return n;
}

// A device-resident model; copies share the device upload (the reference
// shares one immutable LsnifModel across instances, renderer.cpp:55-76).
class Model {
 public:
  static Model load(const std::string& path, int device = 0) {
    lsnif_model m = nullptr;
    check(lsnif_model_load(path.c_str(), device, &m));
    return Model(m);
  }
  static Model create(const lsnif_model_desc& desc, int device = 0) {
    lsnif_model m = nullptr;
    check(lsnif_model_create(&desc, device, &m));
    return Model(m);
  }
  static Model adopt(lsnif_model m) { return Model(m); }  // takes ownership of a C-ABI handle
  lsnif_model handle() const { return h_.get(); }
  lsnif_model_info info() const {
    lsnif_model_info i{};
    check(lsnif_model_get_info(h_.get(), &i));
    return i;
  }
  int input_width() const {
    const lsnif_model_info i = info();
    return i.hit_cap * i.n_levels * i.f_dim;
  }

 private:
  explicit Model(lsnif_model m) : h_(m, [](lsnif_model p) { lsnif_model_destroy(p); }) {}
  std::shared_ptr<lsnif_model_s> h_;
};

// The model's device made current for the adapter's own allocations and
// copies, the caller's current device restored on exit (RAII).
class DeviceScope {
 public:
  explicit DeviceScope(const Model& model) : DeviceScope(model.info().device) {}
  explicit DeviceScope(int device) {  // device < 0: stay on the current device
    if (device < 0) return;
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
  }
  ~DeviceScope() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
  static void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }

 private:
  int prev_ = -1;
};

// Device buffer helper (RAII).
template <typename T>
struct DeviceBuffer {
  T* ptr = nullptr;
  explicit DeviceBuffer(size_t n) {
    if (n && cudaMalloc(&ptr, n * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
  }
  ~DeviceBuffer() { cudaFree(ptr); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

// infer_batch (renderer.cpp:183-226): `inputs` is MatX inputs(input_width, n)
// in column-major order, one interval per column.
inline std::vector<NeuralHit> infer_batch(const Model& model, const std::vector<float>& inputs,
                                          const std::vector<lsnif_interval>& intervals) {
  const int64_t rows = model.input_width();
  const int64_t n = rows ? static_cast<int64_t>(inputs.size()) / rows : 0;
  if (n * rows != static_cast<int64_t>(inputs.size()))
    throw std::invalid_argument("infer_batch: input width mismatch");
  DeviceScope on(model);
  DeviceBuffer<float> dx(inputs.size());
  DeviceBuffer<lsnif_interval> di(intervals.size());
  DeviceBuffer<lsnif_hit> dh(static_cast<size_t>(n));
  if (!inputs.empty())
    DeviceScope::cuda_check(cudaMemcpy(dx.ptr, inputs.data(), inputs.size() * 4, cudaMemcpyHostToDevice),
                            "cudaMemcpy(inputs)");
  if (!intervals.empty())
    DeviceScope::cuda_check(cudaMemcpy(di.ptr, intervals.data(), intervals.size() * sizeof(lsnif_interval),
                                       cudaMemcpyHostToDevice),
                            "cudaMemcpy(intervals)");
  check(lsnif_infer_batch(model.handle(), dx.ptr, rows, n, di.ptr, static_cast<int64_t>(intervals.size()),
                          dh.ptr, nullptr));
  std::vector<lsnif_hit> raw(static_cast<size_t>(n));
  if (n)
    DeviceScope::cuda_check(cudaMemcpy(raw.data(), dh.ptr, raw.size() * sizeof(lsnif_hit), cudaMemcpyDeviceToHost),
                            "cudaMemcpy(hits)");
  std::vector<NeuralHit> out;
  out.reserve(raw.size());
  for (const lsnif_hit& h : raw) out.push_back(to_neural_hit(h));
  return out;
}

// One query per ray (object-space rays), results in ray order.
inline std::vector<lsnif_hit> query(const Model& model, const std::vector<lsnif_ray>& rays, int mode) {
  std::vector<lsnif_hit> hits(rays.size());
  check(lsnif_query_host(model.handle(), rays.data(), static_cast<int64_t>(rays.size()), mode, hits.data(),
                         nullptr));
  return hits;
}

// run_narrow_phase (renderer.cpp:232-265) for one object group: the pairs'
// object-space rays and their [t_enter, t_exit] (RayLsnifPair); one NeuralHit
// per pair, in pair order, for the caller's accept lambdas. `mode` picks the
// kernel's own accept flag (LSNIF_HIT_ACCEPTED in the raw hits, see query()).
inline std::vector<NeuralHit> infer_pairs(const Model& model, const std::vector<lsnif_ray>& rays,
                                          const std::vector<lsnif_interval>& pairs,
                                          int mode = LSNIF_QUERY_CLOSEST) {
  if (rays.size() != pairs.size()) throw std::invalid_argument("infer_pairs: one interval per ray");
  const size_t n = rays.size();
  DeviceScope on(model);
  DeviceBuffer<lsnif_ray> dr(n);
  DeviceBuffer<lsnif_interval> di(n);
  DeviceBuffer<lsnif_hit> dh(n);
  if (n) {
    DeviceScope::cuda_check(cudaMemcpy(dr.ptr, rays.data(), n * sizeof(lsnif_ray), cudaMemcpyHostToDevice),
                            "cudaMemcpy(rays)");
    DeviceScope::cuda_check(cudaMemcpy(di.ptr, pairs.data(), n * sizeof(lsnif_interval), cudaMemcpyHostToDevice),
                            "cudaMemcpy(pairs)");
  }
  check(lsnif_query_pairs(model.handle(), dr.ptr, di.ptr, static_cast<int64_t>(n), mode, dh.ptr, nullptr));
  std::vector<lsnif_hit> raw(n);
  if (n)
    DeviceScope::cuda_check(cudaMemcpy(raw.data(), dh.ptr, n * sizeof(lsnif_hit), cudaMemcpyDeviceToHost),
                            "cudaMemcpy(hits)");
  std::vector<NeuralHit> out;
  out.reserve(n);
  for (const lsnif_hit& h : raw) out.push_back(to_neural_hit(h));
  return out;
}

// Closest-hit narrow phase of intersect_scene for one LSNIF object at identity
// transform: the accepted neural hit per ray, if any.
inline std::vector<std::optional<NeuralHit>> intersect(const Model& model, const std::vector<lsnif_ray>& rays) {
  const std::vector<lsnif_hit> hits = query(model, rays, LSNIF_QUERY_CLOSEST);
  std::vector<std::optional<NeuralHit>> out(hits.size());
  for (size_t i = 0; i < hits.size(); ++i)
    if (hits[i].flags_material & LSNIF_HIT_ACCEPTED) out[i] = to_neural_hit(hits[i]);
  return out;
}

// occluded_batch (renderer.cpp:305-323) for one LSNIF object.
inline std::vector<char> occluded_batch(const Model& model, const std::vector<lsnif_ray>& rays) {
  const std::vector<lsnif_hit> hits = query(model, rays, LSNIF_QUERY_ANY);
  std::vector<char> out(hits.size(), 0);
  for (size_t i = 0; i < hits.size(); ++i) out[i] = (hits[i].flags_material & LSNIF_HIT_ACCEPTED) ? 1 : 0;
  return out;
}

// The LSNIF objects of a PreparedScene: instances (model, world_to_object)
// in object order. Models are shared, as PreparedScene::prepare caches them.
class Scene {
 public:
  Scene(const std::vector<Model>& models, const std::vector<std::array<float, 12>>& world_to_object)
      : models_(models) {
    if (models.size() != world_to_object.size()) throw std::invalid_argument("one transform per instance");
    std::vector<lsnif_instance> inst(models.size());
    for (size_t i = 0; i < models.size(); ++i) {
      inst[i].model = models[i].handle();
      for (int k = 0; k < 12; ++k) inst[i].world_to_object[k] = world_to_object[i][static_cast<size_t>(k)];
    }
    lsnif_scene s = nullptr;
    check(lsnif_scene_create(inst.data(), static_cast<int32_t>(inst.size()), &s));
    h_.reset(s, [](lsnif_scene p) { lsnif_scene_destroy(p); });
  }
  lsnif_scene handle() const { return h_.get(); }
  size_t size() const { return models_.size(); }
  int device() const { return models_.empty() ? -1 : models_.front().info().device; }

  // intersect_scene (renderer.cpp:269-303) / occluded_batch (305-323) for a
  // scene without triangle objects; WORLD-space host rays.
  std::vector<lsnif_scene_hit> query(const std::vector<lsnif_ray>& rays, int mode) const {
    std::vector<lsnif_scene_hit> out(rays.size());
    check(lsnif_scene_query_host(h_.get(), rays.data(), static_cast<int64_t>(rays.size()), mode, out.data(),
                                 nullptr));
    return out;
  }
  std::vector<std::optional<lsnif_scene_hit>> intersect_scene(const std::vector<lsnif_ray>& rays) const {
    const auto hits = query(rays, LSNIF_QUERY_CLOSEST);
    std::vector<std::optional<lsnif_scene_hit>> out(hits.size());
    for (size_t i = 0; i < hits.size(); ++i)
      if (hits[i].flags & 1u) out[i] = hits[i];
    return out;
  }
  std::vector<char> occluded_batch(const std::vector<lsnif_ray>& rays) const {
    const auto hits = query(rays, LSNIF_QUERY_ANY);
    std::vector<char> out(hits.size());
    for (size_t i = 0; i < hits.size(); ++i) out[i] = (hits[i].flags & 1u) ? 1 : 0;
    return out;
  }

 private:
  std::vector<Model> models_;
  std::shared_ptr<lsnif_scene_s> h_;
};

// render() (renderer.cpp:453-542) with PrimaryMode::lsnif: returns the
// image as width * height RGB triples (the reference's Image::pixels).
inline std::vector<float> render(const Scene& scene, const std::vector<float>& world_diag,
                                 const lsnif_camera& camera, const std::vector<lsnif_light>& lights,
                                 const float environment[3], const lsnif_render_config& config,
                                 lsnif_render_stats* stats = nullptr) {
  const size_t px = static_cast<size_t>(config.width > 0 ? config.width : 0) *
                    static_cast<size_t>(config.height > 0 ? config.height : 0);
  DeviceScope on(scene.device());
  DeviceBuffer<float> img(3 * px);
  check(lsnif_render(scene.handle(), world_diag.data(), static_cast<int32_t>(world_diag.size()), &camera,
                     lights.data(), static_cast<int32_t>(lights.size()), environment, &config, img.ptr, stats,
                     nullptr));
  std::vector<float> out(3 * px);
  if (px)
    DeviceScope::cuda_check(cudaMemcpy(out.data(), img.ptr, out.size() * sizeof(float), cudaMemcpyDeviceToHost),
                            "cudaMemcpy(image)");
  return out;
}

// train() (training.cpp:95-230): the starting model + the mesh; step() runs
// optimizer steps on the device, model() exports the binary16 bundle as a
// query model (save_model + load_model).
class Trainer {
 public:
  Trainer(const lsnif_model_desc& init, const lsnif_mesh_desc& mesh, const lsnif_train_config& cfg,
          int device = 0) {
    lsnif_trainer t = nullptr;
    check(lsnif_trainer_create(&init, &mesh, &cfg, device, &t));
    h_.reset(t, [](lsnif_trainer p) { lsnif_trainer_destroy(p); });
  }
  lsnif_train_loss step(int steps) {
    lsnif_train_loss loss{};
    check(lsnif_trainer_step(h_.get(), steps, &loss, nullptr));
    return loss;
  }
  Model model() const {
    lsnif_model m = nullptr;
    check(lsnif_trainer_export(h_.get(), &m));
    return Model::adopt(m);
  }

 private:
  std::shared_ptr<lsnif_trainer_s> h_;
};

}  // namespace gpu
}  // namespace lsnif
