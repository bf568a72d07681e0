// TEST INFRASTRUCTURE — C ABI over the LSNIF REFERENCE ITSELF.
//
// oracle/Makefile.ref compiles the reference's own sources where they lie
// (/root/reference/proj/src/*.cpp, headers from /root/reference/proj/include)
// against the Eigen-subset shim in oracle/eigen_shim, and links them with
// this file into oracle/_ref/libref_{parity,fast}.so. Nothing here restates
// the reference's algorithms: every computational step below is a call into
// the reference (load_model, ray_aabb_intersect, collect_boundary_hits_local,
// encode_ray_into, infer_batch, PreparedScene::prepare / intersect_scene /
// occluded_batch, parallel_slices). The glue only converts records.
//
// Used by tests/ (to pin the oracle restatement and the GPU path to the
// reference's own code) and by bench.py's CPU arms (cpu_baseline /
// --impl reference, kind "reference"). Never linked by the product.
#include "lsnif/dda.hpp"
#include "lsnif/encoding.hpp"
#include "lsnif/geometry.hpp"
#include "lsnif/model_io.hpp"
#include "lsnif/parallel.hpp"
#include "lsnif/renderer.hpp"
#include "lsnif/obj.hpp"
#include "lsnif/scene.hpp"
#include "lsnif/shapes.hpp"
#include "lsnif/training.hpp"
#include "lsnif/voxel.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// Record layouts shared with oracle/oracle.py (lsnif::Ray and the query
// result record of include/lsnif_gpu.h).
struct RayRec {
  float o[3], d[3], t_min, t_max;
};
struct HitRec {
  uint32_t flags_material;
  float t_world, normal[3], albedo[3];
};
struct SceneHitRec {
  float t, position[3], normal[3], albedo[3];
  uint32_t kind;
  float roughness;
  int32_t object_index;
  uint32_t flags;
  uint32_t pad[2];
};
static_assert(sizeof(RayRec) == 32 && sizeof(HitRec) == 32 && sizeof(SceneHitRec) == 64, "records");

lsnif::Ray to_ray(const RayRec& r) {
  lsnif::Ray ray;
  ray.origin = lsnif::Vec3(r.o[0], r.o[1], r.o[2]);
  ray.direction = lsnif::Vec3(r.d[0], r.d[1], r.d[2]);
  ray.t_min = r.t_min;
  ray.t_max = r.t_max;
  return ray;
}

constexpr float kInf = std::numeric_limits<float>::infinity();

// One model as a single-object scene: the object-space path of
// collect_pairs / run_narrow_phase needs only the model; intersect_scene
// and occluded_batch need a PreparedScene (identity placement).
struct RefModel {
  std::string path;
  lsnif::LsnifModel model;
  lsnif::PreparedScene scene;
};

// The model's own frame box as a one-triangle stand-in mesh (prepare() uses
// the mesh only for the triangle BVH, which LSNIF queries never consult, and
// for world bounds; the frame box comes from the loaded model).
lsnif::Mesh frame_mesh(const lsnif::LsnifModel& m) {
  lsnif::Mesh mesh;
  mesh.vertices = {m.aabb.min, lsnif::Vec3(m.aabb.max.x(), m.aabb.min.y(), m.aabb.min.z()), m.aabb.max};
  mesh.faces = {lsnif::Vec3i(0, 1, 2)};
  mesh.face_material = {0};
  mesh.materials = m.materials.empty() ? std::vector<lsnif::Material>(1) : m.materials;
  return mesh;
}

// run_narrow_phase (renderer.cpp:232-265) for one object at identity
// placement, over a slice of rays, each ray its own pair when collect_pairs
// (renderer.cpp:165-172) emits one: the reference's functions for every step;
// results in the query-record layout (pair / occluded / accepted flags,
// NeuralHit fields) so they compare field by field with the GPU.
void narrow_slice(const lsnif::LsnifModel& m, const RayRec* rays, int64_t b, int64_t e, int mode, HitRec* out) {
  const lsnif::LocalFrame frame = m.frame();
  std::vector<int64_t> slot;
  std::vector<lsnif::RayInterval> intervals;
  for (int64_t i = b; i < e; ++i) {
    out[i] = HitRec{};
    lsnif::Ray oray = to_ray(rays[i]);
    oray.t_max = kInf;  // collect_pairs: interval over the whole frame box
    const auto iv = lsnif::ray_aabb_intersect(oray, m.aabb);
    if (!iv || iv->enter >= rays[i].t_max) continue;
    slot.push_back(i);
    intervals.push_back(*iv);
  }
  const int n = static_cast<int>(slot.size());
  if (!n) return;
  lsnif::MatX<lsnif::Real> inputs(m.input_width(), n);
  lsnif::BoundaryHits hits;
  for (int k = 0; k < n; ++k) {
    const lsnif::Ray ray = to_ray(rays[slot[k]]);
    lsnif::collect_boundary_hits_local(frame.to_local(ray.origin), ray.direction.cwiseProduct(frame.inv_extent),
                                       ray.t_min, kInf, m.occupancy, m.hit_cap, hits);
    int pc = 0;
    lsnif::encode_ray_into<lsnif::Real>(m.grid, hits, m.hit_cap, inputs.col(k).data(), nullptr, pc);
  }
  const std::vector<lsnif::NeuralHit> nh = lsnif::infer_batch(m, inputs, intervals);
  for (int k = 0; k < n; ++k) {
    HitRec& h = out[slot[k]];
    const lsnif::NeuralHit& x = nh[static_cast<size_t>(k)];
    const RayRec& r = rays[slot[k]];
    uint32_t f = 1u;
    if (x.occluded) {
      f |= 2u;
      const bool accept = mode == 0 ? !(x.t_world >= r.t_max || x.t_world < r.t_min)  // renderer.cpp:284
                                    : (x.t_world >= r.t_min && x.t_world <= r.t_max);  // renderer.cpp:319
      if (accept) f |= 4u;
    }
    h.flags_material = f | (static_cast<uint32_t>(x.material_index) << 8);
    h.t_world = x.t_world;
    for (int a = 0; a < 3; ++a) {
      h.normal[a] = x.normal[a];
      h.albedo[a] = x.albedo[a];
    }
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hardware_concurrency() { return lsnif::resolve_workers(0); }

void* ref_model_load(const char* path) {
  RefModel* out = nullptr;
  const int st = guarded([&] {
    auto r = std::make_unique<RefModel>();
    r->path = path;
    r->model = lsnif::load_model(path);
    lsnif::Scene sc;
    sc.meshes.push_back(frame_mesh(r->model));
    lsnif::SceneObject so;
    so.mesh_index = 0;
    so.representation = lsnif::Representation::lsnif;
    so.model_path = path;
    sc.objects.push_back(so);
    r->scene = lsnif::PreparedScene::prepare(sc);
    out = r.release();
  });
  return st == 0 ? out : nullptr;
}

void ref_model_free(void* m) { delete static_cast<RefModel*>(m); }

// V, H, L, F, M, hidden, n_mat, level_res[0..1]
void ref_model_info(void* mp, int64_t* info) {
  const lsnif::LsnifModel& m = static_cast<RefModel*>(mp)->model;
  info[0] = m.voxel_res;
  info[1] = m.hit_cap;
  info[2] = m.grid.n_levels();
  info[3] = m.grid.f_dim;
  info[4] = m.grid.table_size;
  info[5] = m.mlp.hidden_width();
  info[6] = m.mlp.n_mat();
  for (int l = 0; l < 2; ++l) info[7 + l] = l < m.grid.n_levels() ? m.grid.levels[l].resolution : 0;
}

void ref_model_aabb(void* mp, float* box) {
  const lsnif::LsnifModel& m = static_cast<RefModel*>(mp)->model;
  for (int a = 0; a < 3; ++a) {
    box[a] = m.aabb.min[a];
    box[3 + a] = m.aabb.max[a];
  }
}

// Per-ray pair interval, DDA boundary points, cells, hash indices and fp32
// features (the lsnif_debug_traverse layout), from the reference's
// ray_aabb_intersect / collect_boundary_hits_local / encode_ray_into.
int ref_trace(void* mp, const RayRec* rays, int64_t n, int32_t* info, float* interval, float* t, float* pts,
              uint32_t* cells, uint32_t* hidx, float* feat) {
  return guarded([&] {
    const lsnif::LsnifModel& m = static_cast<RefModel*>(mp)->model;
    const lsnif::LocalFrame frame = m.frame();
    const int H = m.hit_cap, L = m.grid.n_levels(), lf = L * m.grid.f_dim;
    lsnif::BoundaryHits hits;
    std::vector<float> column(static_cast<size_t>(H * lf));
    std::vector<lsnif::PointCodeT<float>> codes(static_cast<size_t>(H * L));
    for (int64_t i = 0; i < n; ++i) {
      info[i] = 0;
      interval[2 * i] = interval[2 * i + 1] = 0.0f;
      for (int k = 0; k < H; ++k) {
        t[i * H + k] = 0.0f;
        cells[i * H + k] = 0xffffffffu;
        for (int a = 0; a < 3; ++a) pts[(i * H + k) * 3 + a] = 0.0f;
        for (int c = 0; c < L * 8; ++c) hidx[(i * H + k) * L * 8 + c] = 0xffffffffu;
      }
      std::fill(feat + i * H * lf, feat + (i + 1) * H * lf, 0.0f);
      lsnif::Ray ray = to_ray(rays[i]);
      lsnif::Ray oray = ray;
      oray.t_max = kInf;
      const auto iv = lsnif::ray_aabb_intersect(oray, m.aabb);
      if (!iv || iv->enter >= ray.t_max) continue;
      interval[2 * i] = iv->enter;
      interval[2 * i + 1] = iv->exit;
      lsnif::collect_boundary_hits_local(frame.to_local(ray.origin), ray.direction.cwiseProduct(frame.inv_extent),
                                         ray.t_min, kInf, m.occupancy, m.hit_cap, hits);
      int pc = 0;
      lsnif::encode_ray_into<float>(m.grid, hits, H, column.data(), codes.data(), pc);
      info[i] = pc | (hits.first_is_origin ? 1 << 8 : 0) | (1 << 9);
      for (int k = 0; k < pc; ++k) {
        t[i * H + k] = hits.t_values[static_cast<size_t>(k)];
        for (int a = 0; a < 3; ++a) pts[(i * H + k) * 3 + a] = hits.points[static_cast<size_t>(k)][a];
        const lsnif::Vec3i& c = hits.cells[static_cast<size_t>(k)];
        cells[i * H + k] = static_cast<uint32_t>(c[0]) | static_cast<uint32_t>(c[1]) << 8 |
                           static_cast<uint32_t>(c[2]) << 16;
        for (int l = 0; l < L; ++l) {
          const auto& pcode = codes[static_cast<size_t>(k * L + l)];
          for (int q = 0; q < pcode.count; ++q) hidx[((i * H + k) * L + l) * 8 + q] = pcode.index[q];
        }
      }
      std::memcpy(feat + i * H * lf, column.data(), sizeof(float) * static_cast<size_t>(H * lf));
    }
  });
}

// infer_batch (renderer.cpp:183-226): inputs column-major (rows x n).
int ref_infer_batch(void* mp, const float* inputs, int64_t rows, int64_t n, const float* iv, int64_t n_iv,
                    HitRec* out) {
  return guarded([&] {
    const lsnif::LsnifModel& m = static_cast<RefModel*>(mp)->model;
    lsnif::MatX<lsnif::Real> x(rows, n);
    std::memcpy(x.data(), inputs, sizeof(float) * static_cast<size_t>(rows * n));
    std::vector<lsnif::RayInterval> ivs(static_cast<size_t>(n_iv));
    for (int64_t j = 0; j < n_iv; ++j) ivs[static_cast<size_t>(j)] = lsnif::RayInterval{iv[2 * j], iv[2 * j + 1]};
    const std::vector<lsnif::NeuralHit> nh = lsnif::infer_batch(m, x, ivs);
    for (int64_t j = 0; j < n; ++j) {
      const lsnif::NeuralHit& h = nh[static_cast<size_t>(j)];
      out[j].flags_material = (h.occluded ? 2u : 0u) | (static_cast<uint32_t>(h.material_index) << 8);
      out[j].t_world = h.t_world;
      for (int a = 0; a < 3; ++a) {
        out[j].normal[a] = h.normal[a];
        out[j].albedo[a] = h.albedo[a];
      }
    }
  });
}

// The narrow phase per ray (query-record layout), over `workers` threads in
// parallel_slices (parallel.hpp:18-37) with 65,536-ray blocks as render()
// batches them (renderer.cpp:478-480).
int ref_narrow_phase(void* mp, const RayRec* rays, int64_t n, int mode, HitRec* out, int workers) {
  return guarded([&] {
    const lsnif::LsnifModel& m = static_cast<RefModel*>(mp)->model;
    constexpr int64_t kBlock = 65536;
    const long nblocks = static_cast<long>((n + kBlock - 1) / kBlock);
    std::vector<std::string> errs(static_cast<size_t>(std::max(1, lsnif::resolve_workers(workers))));
    lsnif::parallel_slices(n, workers, [&](int w, long b, long e) {
      try {
        for (long s = b; s < e; s += kBlock) narrow_slice(m, rays, s, std::min<long>(e, s + kBlock), mode, out);
      } catch (const std::exception& ex) {
        errs[static_cast<size_t>(w)] = ex.what();
      }
    });
    (void)nblocks;
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// PreparedScene::intersect_scene (renderer.cpp:269-303, mode 0) or
// occluded_batch (305-323, mode 1) on a single-object scene, use_lsnif = true,
// called concurrently from `workers` threads on 65,536-ray blocks as render()
// does. Output: SurfaceHit fields (closest) / the occluded flag (any).
int ref_scene_query(void* mp, const RayRec* rays, int64_t n, int mode, SceneHitRec* out, int workers) {
  return guarded([&] {
    const lsnif::PreparedScene& scene = static_cast<RefModel*>(mp)->scene;
    constexpr long kBlock = 65536;
    const long nb = static_cast<long>((n + kBlock - 1) / kBlock);
    lsnif::parallel_slices(nb, workers, [&](int, long b, long e) {
      std::vector<lsnif::Ray> batch;
      for (long blk = b; blk < e; ++blk) {
        const int64_t s = blk * kBlock, t = std::min<int64_t>(n, s + kBlock);
        batch.resize(static_cast<size_t>(t - s));
        for (int64_t i = s; i < t; ++i) batch[static_cast<size_t>(i - s)] = to_ray(rays[i]);
        if (mode == 0) {
          const auto res = scene.intersect_scene(batch, true, true);
          for (int64_t i = s; i < t; ++i) {
            SceneHitRec& o = out[i];
            o = SceneHitRec{};
            o.t = rays[i].t_max;
            o.object_index = -1;
            const auto& r = res[static_cast<size_t>(i - s)];
            if (!r) continue;
            o.t = r->t;
            for (int a = 0; a < 3; ++a) {
              o.position[a] = r->position[a];
              o.normal[a] = r->normal[a];
              o.albedo[a] = r->albedo[a];
            }
            o.kind = static_cast<uint32_t>(r->kind);
            o.roughness = r->roughness;
            o.object_index = r->object_index;
            o.flags = 1u;
          }
        } else {
          const auto occ = scene.occluded_batch(batch, true);
          for (int64_t i = s; i < t; ++i) {
            out[i] = SceneHitRec{};
            out[i].object_index = -1;
            out[i].flags = occ[static_cast<size_t>(i - s)] ? 1u : 0u;
          }
        }
      }
    });
  });
}

// Best wall time (s) of `reps` ref_scene_query passes after one warm-up.
double ref_time_scene_query(void* mp, const RayRec* rays, int64_t n, int mode, SceneHitRec* out, int workers,
                            int reps) {
  double best = std::numeric_limits<double>::infinity();
  const int st = guarded([&] {
    if (ref_scene_query(mp, rays, n, mode, out, workers) != 0) throw std::runtime_error(g_err);
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      if (ref_scene_query(mp, rays, n, mode, out, workers) != 0) throw std::runtime_error(g_err);
      best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
  });
  return st < 0 ? st : best;
}

// The T = 0 state of train() (training.cpp:100-128: LocalFrame::for_mesh,
// voxelize_surface, make_sparse_hash_grid, make_mlp with TrainConfig's
// defaults and the given V, H, seed) saved with save_model — the reference
// generating the test fixtures the oracle generated.
static void save_setup_model(const lsnif::Mesh& mesh, int V, int H, uint64_t seed, const char* out) {
  lsnif::TrainConfig cfg;
  cfg.voxel_res = V;
  cfg.hit_cap = H;
  cfg.seed = seed;
  const lsnif::LocalFrame frame = lsnif::LocalFrame::for_mesh(mesh);
  lsnif::LsnifModel model;
  model.voxel_res = cfg.voxel_res;
  model.hit_cap = cfg.hit_cap;
  model.occupancy = lsnif::voxelize_surface(mesh, frame, cfg.voxel_res);
  model.grid = lsnif::make_sparse_hash_grid<lsnif::Real>(cfg.voxel_res, cfg.level_res, cfg.f_dim, cfg.table_size,
                                                         cfg.seed);
  const int input_width = cfg.hit_cap * model.grid.n_levels() * cfg.f_dim;
  model.mlp = lsnif::make_mlp<lsnif::Real>(input_width, cfg.hidden_width, mesh.n_materials(), cfg.seed);
  model.materials = mesh.materials;
  model.aabb = frame.aabb;
  lsnif::save_model(model, out);
}

int ref_build_obj_model(const char* obj_path, const char* out_path, int V, int H, uint64_t seed) {
  return guarded([&] { save_setup_model(lsnif::load_obj(obj_path), V, H, seed, out_path); });
}

// shape: 0 make_uv_sphere(), 1 make_box((1, .6, .8)), 2 make_torus() (shapes.cpp)
int ref_build_shape_model(int shape, uint64_t seed, const char* out_path) {
  return guarded([&] {
    lsnif::Mesh mesh = shape == 0   ? lsnif::make_uv_sphere()
                       : shape == 1 ? lsnif::make_box(lsnif::Vec3(1.0f, 0.6f, 0.8f))
                                    : lsnif::make_torus();
    save_setup_model(mesh, 32, 18, seed, out_path);
  });
}

}  // extern "C"
