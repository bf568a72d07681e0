// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
// Flat C entry points over the oracle for the Python test/bench harness
// (ctypes). Errors: functions return a negative status and set a
// thread-local message readable with oracle_last_error().
#include "lsnif_oracle.hpp"
#include "lsnif_render_oracle.hpp"
#include "lsnif_train_oracle.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>

using namespace oracle;

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

// Per-ray debug trace in the same flat layout lsnif_debug_traverse (GPU)
// produces; H/L/F are the model's.
struct TraceOut {
  int32_t* info;      // [n]  count | first_is_origin << 8 | pair << 9
  float* interval;    // [n][2]
  float* t;           // [n][H]
  float* pts;         // [n][H][3]
  uint32_t* cells;    // [n][H]  x | y << 8 | z << 16
  uint32_t* hidx;     // [n][H][L][8]  (unused corners 0xffffffff)
  float* feat;        // [n][H*L*F]
};
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

uint64_t oracle_mix_bits(uint64_t x) { return mix_bits(x); }
uint32_t oracle_seed_stream(uint64_t s, uint64_t a, uint64_t b, uint64_t c) {
  return seed_stream(s, a, b, c);
}
uint16_t oracle_float_to_half(float v) { return float_to_half(v); }
float oracle_half_to_float(uint16_t h) { return half_to_float(h); }
uint32_t oracle_hash_vertex(int x, int y, int z, uint32_t m) { return hash_vertex(x, y, z, m); }

int oracle_ray_aabb(const Ray* ray, const float box[6], float out[2]) {
  Aabb b;
  for (int a = 0; a < 3; ++a) {
    b.mn[a] = box[a];
    b.mx[a] = box[3 + a];
  }
  Interval iv;
  if (!ray_aabb_intersect(*ray, b, &iv)) return 0;
  out[0] = iv.enter;
  out[1] = iv.exit;
  return 1;
}

void oracle_inflate_frame(const float box[6], float out[6]) {
  Aabb b;
  for (int a = 0; a < 3; ++a) {
    b.mn[a] = box[a];
    b.mx[a] = box[3 + a];
  }
  b = inflate_frame(b);
  for (int a = 0; a < 3; ++a) {
    out[a] = b.mn[a];
    out[3 + a] = b.mx[a];
  }
}

int oracle_voxelize(const float* verts, int nv, const int* faces, int nf, const float frame[6],
                    int res, uint8_t* out) {
  return guarded([&] {
    Aabb f;
    for (int a = 0; a < 3; ++a) {
      f.mn[a] = frame[a];
      f.mx[a] = frame[3 + a];
    }
    std::vector<float> v(verts, verts + 3 * nv);
    std::vector<int> fc(faces, faces + 3 * nf);
    auto bits = voxelize_surface(v, fc, f, res);
    std::memcpy(out, bits.data(), bits.size());
  });
}

// DDA on a local-space ray (dda.cpp:40-117). Returns the point count.
int oracle_dda_local(const float o[3], const float d[3], float t_min, float t_max,
                     const uint8_t* occ, int res, int cap, float* pts, float* t, int* cells,
                     int* first_is_origin) {
  int n = -1;
  int st = guarded([&] {
    std::vector<uint8_t> bits(occ, occ + static_cast<size_t>(res) * res * res / 8);
    BoundaryHits h;
    collect_boundary_hits_local(o, d, t_min, t_max, bits, res, cap, h);
    n = h.count();
    std::memcpy(pts, h.points.data(), sizeof(float) * h.points.size());
    std::memcpy(t, h.t_values.data(), sizeof(float) * h.t_values.size());
    std::memcpy(cells, h.cells.data(), sizeof(int) * h.cells.size());
    *first_is_origin = h.first_is_origin ? 1 : 0;
  });
  return st < 0 ? st : n;
}

// ---- models ----

void* oracle_model_load(const char* path) {
  Model* m = nullptr;
  guarded([&] { m = new Model(load_model(path)); });
  return m;
}

void oracle_model_free(void* m) { delete static_cast<Model*>(m); }

int oracle_model_save(void* m, const char* path) {
  return guarded([&] { save_model(*static_cast<Model*>(m), path); });
}

// V, H, L, F, M, hidden, n_mat, level_res[0], level_res[1]
void oracle_model_info(void* mp, int64_t* out) {
  const Model& m = *static_cast<Model*>(mp);
  out[0] = m.voxel_res;
  out[1] = m.hit_cap;
  out[2] = m.n_levels;
  out[3] = m.f_dim;
  out[4] = m.table_size;
  out[5] = m.hidden;
  out[6] = m.n_mat;
  out[7] = m.level_res.size() > 0 ? m.level_res[0] : 0;
  out[8] = m.level_res.size() > 1 ? m.level_res[1] : 0;
}

void oracle_model_aabb(void* mp, float* out6) {
  const Model& m = *static_cast<Model*>(mp);
  for (int a = 0; a < 3; ++a) {
    out6[a] = m.aabb.mn[a];
    out6[3 + a] = m.aabb.mx[a];
  }
}

const uint8_t* oracle_model_occupancy(void* mp) {
  return static_cast<Model*>(mp)->occupancy.data();
}

// Random-init model (train() setup state, training.cpp:100-124) over a
// given occupancy grid and frame box. levels: n_levels resolutions.
void* oracle_model_random(const uint8_t* occ, int V, int H, int n_levels, const int* levels,
                          int F, uint32_t M, int hidden, int n_mat, const float frame[6],
                          uint64_t seed) {
  Model* out = nullptr;
  guarded([&] {
    Model m;
    m.voxel_res = V;
    m.hit_cap = H;
    m.n_levels = n_levels;
    m.f_dim = F;
    m.table_size = M;
    m.hidden = hidden;
    m.n_mat = n_mat;
    m.occupancy.assign(occ, occ + static_cast<size_t>(V) * V * V / 8);
    m.level_res.assign(levels, levels + n_levels);
    for (int a = 0; a < 3; ++a) {
      m.aabb.mn[a] = frame[a];
      m.aabb.mx[a] = frame[3 + a];
    }
    m.materials.assign(static_cast<size_t>(n_mat), Material{{0.7f, 0.7f, 0.7f}, 0u, 0.5f});
    init_random_model(m, seed);
    out = new Model(std::move(m));
  });
  return out;
}

// OBJ → LocalFrame::for_mesh → voxelize → random init (seed) → save_model:
// the reference train() setup with T = 0 steps (training.cpp:100-124).
int oracle_build_obj_model(const char* obj_path, int V, int H, uint64_t seed,
                           const char* out_path) {
  return guarded([&] {
    ObjMesh mesh = load_obj(obj_path);
    Aabb b;
    for (int a = 0; a < 3; ++a) {
      b.mn[a] = std::numeric_limits<float>::max();
      b.mx[a] = std::numeric_limits<float>::lowest();
    }
    for (size_t i = 0; i < mesh.verts.size() / 3; ++i)
      for (int a = 0; a < 3; ++a) {
        b.mn[a] = std::min(b.mn[a], mesh.verts[3 * i + a]);
        b.mx[a] = std::max(b.mx[a], mesh.verts[3 * i + a]);
      }
    const Aabb frame = inflate_frame(b);
    Model m;
    m.voxel_res = V;
    m.hit_cap = H;
    m.n_levels = 2;
    m.f_dim = 3;
    m.table_size = 1u << 17;
    m.hidden = 128;
    m.n_mat = mesh.n_mat;
    m.level_res = {64, 128};
    m.occupancy = voxelize_surface(mesh.verts, mesh.faces, frame, V);
    m.aabb = frame;
    m.materials.assign(static_cast<size_t>(mesh.n_mat), Material{{0.7f, 0.7f, 0.7f}, 0u, 0.5f});
    init_random_model(m, seed);
    save_model(m, out_path);
  });
}

// Encode one point on one level (encoding.hpp:84-140).
int oracle_encode_point(void* mp, int level, const float p[3], int volume, float* features,
                        uint32_t* idx, float* w, int* plane_axis) {
  PointCode code;
  encode_point_level(*static_cast<Model*>(mp), level, p, volume != 0, features, &code);
  for (int k = 0; k < code.count; ++k) {
    idx[k] = code.index[k];
    w[k] = code.weight[k];
  }
  *plane_axis = code.plane_axis;
  return code.count;
}

void oracle_mlp_logits(void* mp, const float* x, float* z) {
  mlp_logits(*static_cast<Model*>(mp), x, z);
}

static void to_record(const NeuralHit& nh, HitRecord* rec) {
  rec->flags_material = (nh.occluded ? 2u : 0u) | (static_cast<uint32_t>(nh.material_index) << 8);
  rec->t_world = nh.t_world;
  for (int k = 0; k < 3; ++k) {
    rec->normal[k] = nh.normal[k];
    rec->albedo[k] = nh.albedo[k];
  }
}

// infer_batch (renderer.cpp:183-226): x is n columns of input_width floats
// (column-major, as MatX inputs), intervals n pairs. Throws on shape
// mismatch like the reference.
int oracle_infer_batch(void* mp, const float* x, int64_t rows, int64_t n, const float* iv,
                       int64_t n_iv, HitRecord* out) {
  return guarded([&] {
    const Model& m = *static_cast<Model*>(mp);
    if (n != n_iv) throw std::invalid_argument("infer_batch: inputs/intervals size mismatch");
    if (rows != m.input_width()) throw std::invalid_argument("infer_batch: input width mismatch");
    for (int64_t j = 0; j < n; ++j)
      to_record(infer_one(m, x + j * rows, Interval{iv[2 * j], iv[2 * j + 1]}), out + j);
  });
}

int oracle_narrow_phase(void* mp, const Ray* rays, int64_t n, int mode, HitRecord* out,
                        int workers) {
  return guarded([&] { narrow_phase(*static_cast<Model*>(mp), rays, n, mode, out, workers); });
}

// Times narrow_phase over `reps` passes after one warm-up; returns the best
// wall time in seconds (steady clock), or a negative status.
double oracle_time_narrow_phase(void* mp, const Ray* rays, int64_t n, int mode, HitRecord* out,
                                int workers, int reps) {
  double best = std::numeric_limits<double>::infinity();
  int st = guarded([&] {
    const Model& m = *static_cast<Model*>(mp);
    narrow_phase(m, rays, n, mode, out, workers);
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      narrow_phase(m, rays, n, mode, out, workers);
      auto t1 = std::chrono::steady_clock::now();
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
  });
  return st < 0 ? st : best;
}

int oracle_hardware_concurrency() {
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

// Full per-ray trace (pair/interval, DDA points, hash indices, features) in
// the lsnif_debug_traverse layout.
int oracle_trace(void* mp, const Ray* rays, int64_t n, int32_t* info, float* interval, float* t,
                 float* pts, uint32_t* cells, uint32_t* hidx, float* feat) {
  return guarded([&] {
    const Model& m = *static_cast<Model*>(mp);
    const int H = m.hit_cap, L = m.n_levels, F = m.f_dim;
    const int lf = L * F;
    BoundaryHits hits;
    std::vector<float> column(static_cast<size_t>(m.input_width()));
    std::vector<PointCode> codes(static_cast<size_t>(H * L));
    for (int64_t i = 0; i < n; ++i) {
      const Ray& ray = rays[i];
      info[i] = 0;
      interval[2 * i] = interval[2 * i + 1] = 0.0f;
      for (int k = 0; k < H; ++k) {
        t[i * H + k] = 0.0f;
        cells[i * H + k] = 0xffffffffu;
        for (int a = 0; a < 3; ++a) pts[(i * H + k) * 3 + a] = 0.0f;
        for (int c = 0; c < L * 8; ++c) hidx[(i * H + k) * L * 8 + c] = 0xffffffffu;
      }
      for (int k = 0; k < H * lf; ++k) feat[i * H * lf + k] = 0.0f;
      Ray oray = ray;
      oray.t_max = std::numeric_limits<float>::infinity();
      Interval iv;
      if (!ray_aabb_intersect(oray, m.aabb, &iv) || !(iv.enter < ray.t_max)) continue;
      interval[2 * i] = iv.enter;
      interval[2 * i + 1] = iv.exit;
      float inv_ext[3], lo[3], ld[3];
      for (int a = 0; a < 3; ++a) inv_ext[a] = 1.0f / (m.aabb.mx[a] - m.aabb.mn[a]);
      for (int a = 0; a < 3; ++a) {
        lo[a] = (ray.o[a] - m.aabb.mn[a]) * inv_ext[a];
        ld[a] = ray.d[a] * inv_ext[a];
      }
      collect_boundary_hits_local(lo, ld, ray.t_min, std::numeric_limits<float>::infinity(),
                                  m.occupancy, m.voxel_res, H, hits);
      int pc = 0;
      encode_ray_into(m, hits, column.data(), codes.data(), pc);
      info[i] = pc | (hits.first_is_origin ? 1 << 8 : 0) | (1 << 9);
      for (int k = 0; k < pc; ++k) {
        t[i * H + k] = hits.t_values[static_cast<size_t>(k)];
        for (int a = 0; a < 3; ++a)
          pts[(i * H + k) * 3 + a] = hits.points[static_cast<size_t>(3 * k + a)];
        cells[i * H + k] = static_cast<uint32_t>(hits.cells[static_cast<size_t>(3 * k)]) |
                           static_cast<uint32_t>(hits.cells[static_cast<size_t>(3 * k + 1)]) << 8 |
                           static_cast<uint32_t>(hits.cells[static_cast<size_t>(3 * k + 2)]) << 16;
        for (int l = 0; l < L; ++l) {
          const PointCode& c = codes[static_cast<size_t>(k * L + l)];
          for (int q = 0; q < c.count; ++q) hidx[((i * H + k) * L + l) * 8 + q] = c.index[q];
        }
      }
      std::memcpy(feat + i * H * lf, column.data(), sizeof(float) * static_cast<size_t>(H * lf));
    }
  });
}

// Procedural fixture model (shapes.cpp) -> train() setup state -> file.
// shape: 0 sphere, 1 box, 2 torus.
int oracle_build_shape_model(int shape, uint64_t seed, const char* out_path) {
  return guarded([&] {
    ObjMesh mesh;
    if (shape == 0) mesh = make_uv_sphere(1.0f, 32, 16);
    else if (shape == 1) {
      const float h[3] = {1.0f, 0.6f, 0.8f};
      mesh = make_box(h);
    } else mesh = make_torus(1.0f, 0.35f, 48, 24);
    save_model(model_from_mesh(mesh, 32, 18, seed), out_path);
  });
}

int oracle_scene_query(void** models, const float* w2o, int n_inst, const Ray* rays, int64_t n,
                       int mode, SceneHit* out, int workers) {
  return guarded([&] {
    std::vector<Instance> inst(static_cast<size_t>(n_inst));
    for (int k = 0; k < n_inst; ++k) {
      inst[static_cast<size_t>(k)].model = static_cast<Model*>(models[k]);
      std::memcpy(inst[static_cast<size_t>(k)].w2o, w2o + 12 * k, 48);
    }
    scene_query(inst.data(), n_inst, rays, n, mode, out, workers);
  });
}

// setup layout (floats): width, height, spp, max_bounces, seed_lo, seed_hi (as
// u32 bit patterns), eps, camera[10], environment[3]; lights: 8 floats each
// (type as u32 bits, position, radius, radiance).
static RenderSetup unpack_setup(const float* sp, const float* lights, int n_lights, const float* diag, int n_inst) {
  RenderSetup S;
  const uint32_t* u = reinterpret_cast<const uint32_t*>(sp);
  S.width = static_cast<int>(u[0]);
  S.height = static_cast<int>(u[1]);
  S.spp = static_cast<int>(u[2]);
  S.max_bounces = static_cast<int>(u[3]);
  S.seed = static_cast<uint64_t>(u[4]) | (static_cast<uint64_t>(u[5]) << 32);
  S.neural_eps_scale = sp[6];
  std::memcpy(&S.camera, sp + 7, sizeof(RCamera));
  for (int a = 0; a < 3; ++a) S.environment[a] = sp[17 + a];
  for (int i = 0; i < n_lights; ++i) {
    RLight L;
    std::memcpy(&L, lights + 8 * i, sizeof(RLight));
    S.lights.push_back(L);
  }
  S.world_diag.assign(diag, diag + n_inst);
  return S;
}

int oracle_render(void** models, const float* w2o, int n_inst, const float* setup, const float* lights,
                  int n_lights, const float* world_diag, float* image, int workers, int64_t* stats) {
  return guarded([&] {
    std::vector<Instance> inst(static_cast<size_t>(n_inst));
    for (int k = 0; k < n_inst; ++k) {
      inst[static_cast<size_t>(k)].model = static_cast<Model*>(models[k]);
      std::memcpy(inst[static_cast<size_t>(k)].w2o, w2o + 12 * k, 48);
    }
    render(unpack_setup(setup, lights, n_lights, world_diag, n_inst), inst.data(), n_inst, image, workers,
           stats);
  });
}

int oracle_render_debug_paths(const float* setup, int64_t first, int64_t n, Ray* rays, float* u, int k) {
  return guarded([&] { render_debug_paths(unpack_setup(setup, nullptr, 0, nullptr, 0), first, n, rays, u, k); });
}

// mesh of a procedural fixture (shape 0 sphere, 1 box, 2 torus): counts first
// (verts/faces may be NULL), then the arrays.
int oracle_shape_mesh(int shape, float* verts, int* nv, int* faces, int* nf) {
  return guarded([&] {
    ObjMesh mesh;
    if (shape == 0) mesh = make_uv_sphere(1.0f, 32, 16);
    else if (shape == 1) {
      const float h[3] = {1.0f, 0.6f, 0.8f};
      mesh = make_box(h);
    } else mesh = make_torus(1.0f, 0.35f, 48, 24);
    *nv = static_cast<int>(mesh.verts.size() / 3);
    *nf = static_cast<int>(mesh.faces.size() / 3);
    if (verts) std::memcpy(verts, mesh.verts.data(), mesh.verts.size() * 4);
    if (faces) std::memcpy(faces, mesh.faces.data(), mesh.faces.size() * 4);
  });
}

int oracle_label_rays(const float* verts, const float* normals, const int* faces, const int* face_normals,
                      const int* face_material, int n_faces, const float* albedo, const float frame[6],
                      const Ray* rays, int64_t n, TrainTarget* out, int8_t* ok) {
  return guarded([&] {
    TrainMesh M{verts, normals, faces, face_normals, face_material, n_faces, albedo};
    Aabb box;
    for (int a = 0; a < 3; ++a) {
      box.mn[a] = frame[a];
      box.mx[a] = frame[3 + a];
    }
    for (int64_t i = 0; i < n; ++i) ok[i] = label_ray(M, box, rays[i], out[i]) ? 1 : 0;
  });
}

int oracle_train_batch_grad(void* mp, const Ray* rays, const TrainTarget* targets, int64_t n, float* loss,
                            float* g_mlp, float* g_tab) {
  return guarded([&] { train_batch_grad(*static_cast<Model*>(mp), rays, targets, n, loss, g_mlp, g_tab); });
}

}  // extern "C"
