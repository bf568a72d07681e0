// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU oracle for the LSNIF batched ray-query path: a line-by-line restatement
// (no Eigen) of the reference's hot-path functions, used only by tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// as the checker. The CUDA product path never links or calls it.
//
// Every function cites the reference file:line it restates (paths relative to
// the reference's proj/ directory). Float expressions keep the reference's
// operation order; the parity build compiles with -ffp-contract=off so that
// `a + b * c` is two roundings, as the GPU path reproduces with __fmul_rn /
// __fadd_rn. The timing build (-O3 -march=native, the reference's flags) may
// contract.
//
// Pinning: the reference cannot be compiled here (Eigen3 and CLI11 absent),
// and it ships no tests or golden vectors. The oracle is pinned against every
// known-answer example in SPEC.md (see tests/test_oracle_kats.py). MLP
// arithmetic is "parity unpinned" beyond those KATs: the reference's GEMV
// summation order is Eigen-internal; the oracle sums sequentially over the
// input index.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace oracle {

// types.hpp:10 (Real = float); geometry.hpp:11-18.
struct Ray {
  float o[3];
  float d[3];
  float t_min;
  float t_max;
};
static_assert(sizeof(Ray) == 32, "Ray must match lsnif_ray (32 B)");

struct Interval {  // geometry.hpp:47-50
  float enter;
  float exit;
};

struct Aabb {  // geometry.hpp:20-43
  float mn[3];
  float mx[3];
};

struct Material {  // geometry.hpp:56-60; model_io.cpp:159-164
  float albedo[3];
  uint32_t kind;  // 0 diffuse, 1 glossy
  float roughness;
};

// dda.hpp:13-28
struct BoundaryHits {
  std::vector<float> points;  // 3 per point
  std::vector<float> t_values;
  std::vector<int> cells;     // 3 per point
  bool first_is_origin = false;
  int count() const { return static_cast<int>(t_values.size()); }
  void clear() {
    points.clear();
    t_values.clear();
    cells.clear();
    first_is_origin = false;
  }
};

// model_io.hpp:18-36 with the tables/weights kept as decoded fp32 (exactly the
// values load_model produces from the fp16 file) plus the raw fp16 bits.
struct Model {
  int voxel_res = 32;  // V
  int hit_cap = 18;    // H
  int n_levels = 2;    // L
  int f_dim = 3;       // F
  uint32_t table_size = 1u << 17;  // M
  int hidden = 128;
  int n_mat = 1;
  std::vector<uint8_t> occupancy;            // V^3/8 bytes, voxel.hpp:10-11
  std::vector<int> level_res;                // per level R
  std::vector<std::vector<float>> tables;    // per level M*F, entry-major
  std::vector<float> w1, b1, w2, b2, w3, b3; // row-major [out][in]
  std::vector<float> w1t, w2t, w3t;          // transposed copies (finalize_model)
  std::vector<Material> materials;
  Aabb aabb{};

  int input_width() const { return hit_cap * n_levels * f_dim; }
  int output_width() const { return 8 + n_mat; }
};

// ---- L0 numerics (types.hpp:25-39, half.hpp:10-64) ----
uint64_t mix_bits(uint64_t x);
uint32_t seed_stream(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0);
uint16_t float_to_half(float v);
float half_to_float(uint16_t h);

// ---- geometry (geometry.cpp:9-28, 93-107) ----
bool ray_aabb_intersect(const Ray& ray, const Aabb& box, Interval* out);
Aabb inflate_frame(Aabb box);  // LocalFrame::for_aabb

// ---- voxel (voxel.hpp:10-36, voxel.cpp:47-127) ----
bool occupied(const std::vector<uint8_t>& bits, int res, int ix, int iy, int iz);
bool triangle_box_overlap(const float c[3], const float h[3], const float a[3],
                          const float b[3], const float cc[3]);
std::vector<uint8_t> voxelize_surface(const std::vector<float>& verts,  // 3 per vertex
                                      const std::vector<int>& faces,    // 3 per face
                                      const Aabb& frame, int res);

// ---- OBJ (obj.cpp:53-113), positions + faces + usemtl slots only ----
struct ObjMesh {
  std::vector<float> verts;
  std::vector<int> faces;
  std::vector<int> face_material;
  int n_mat = 1;
};
ObjMesh load_obj(const std::string& path);

// ---- DDA (dda.cpp:14-117) ----
void collect_boundary_hits_local(const float origin[3], const float dir[3], float t_min,
                                 float t_max, const std::vector<uint8_t>& occ, int res,
                                 int cap, BoundaryHits& out);

// ---- encoding (encoding.hpp:18-23, 84-176) ----
uint32_t hash_vertex(int ix, int iy, int iz, uint32_t table_size);
struct PointCode {  // encoding.hpp:75-79
  uint32_t index[8];
  float weight[8];
  int count = 0;
  int plane_axis = -1;
};
void encode_point_level(const Model& m, int level, const float p[3], bool volume,
                        float* features, PointCode* code);
void encode_ray_into(const Model& m, const BoundaryHits& hits, float* column,
                     PointCode* codes, int& point_count);

// ---- init (encoding.hpp:46-69, mlp.hpp:44-65) ----
void init_random_model(Model& m, uint64_t seed);  // tables + MLP, reference RNG order
void finalize_model(Model& m);                     // derived transposes

// ---- MLP + heads + decode (mlp.hpp:80-94; renderer.cpp:183-226) ----
struct NeuralHit {  // renderer.hpp:42-48
  bool occluded = false;
  float t_world = 0;
  float normal[3] = {0, 0, 0};
  float albedo[3] = {0, 0, 0};
  int material_index = 0;
};
void mlp_logits(const Model& m, const float* x, float* z3);  // z3: 8+n_mat
NeuralHit decode_logits(const Model& m, const float* z3, Interval iv);
NeuralHit infer_one(const Model& m, const float* x, Interval iv);

// ---- model file (model_io.cpp:71-175) ----
void save_model(const Model& m, const std::string& path);
Model load_model(const std::string& path);

// ---- narrow phase for one object at identity transform
//      (renderer.cpp:154-181 pair emission, 232-265 narrow phase,
//       280-301 / 316-321 accept rules) ----
enum QueryMode { kClosest = 0, kAny = 1 };
// Output record == lsnif_hit (include/lsnif_gpu.h).
struct HitRecord {
  uint32_t flags_material;  // bit0 pair, bit1 occluded head, bit2 accepted; material << 8
  float t_world;
  float normal[3];
  float albedo[3];
};
static_assert(sizeof(HitRecord) == 32, "HitRecord must match lsnif_hit (32 B)");
void narrow_phase(const Model& m, const Ray* rays, int64_t n, int mode, HitRecord* out,
                  int workers);

// ---- procedural fixture meshes (shapes.cpp:18-112) ----
ObjMesh make_uv_sphere(float radius, int segments, int rings);
ObjMesh make_box(const float half[3]);
ObjMesh make_torus(float major_radius, float minor_radius, int segments, int rings);
// train() setup state (T = 0) for a mesh: frame, V-voxelization, random init.
Model model_from_mesh(const ObjMesh& mesh, int V, int H, uint64_t seed);

// ---- multi-object query (renderer.cpp:154-181 collect_pairs with a
//      brute-force broad phase, stable sort by object, run_narrow_phase per
//      object group, accept rules 280-301 / 316-321) ----
struct Instance {
  const Model* model;
  float w2o[12];  // world_to_object, row-major 3x4 [linear | translation]
};
struct SceneHit {   // SurfaceHit (renderer.hpp:56-65) + bookkeeping, 64 B
  float t;
  float position[3];
  float normal[3];
  float albedo[3];
  uint32_t kind;
  float roughness;
  int32_t object_index;
  uint32_t flags;   // 1 = hit (closest) / occluded (any)
  uint32_t pad[2];
};
static_assert(sizeof(SceneHit) == 64, "SceneHit must match lsnif_scene_hit (64 B)");
void scene_query(const Instance* inst, int n_inst, const Ray* rays, int64_t n, int mode,
                 SceneHit* out, int workers);

}  // namespace oracle
