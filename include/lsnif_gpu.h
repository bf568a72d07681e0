/*
 * lsnif_gpu.h — C ABI of the B200-native LSNIF batched ray-query path.
 *
 * This is the drop-in boundary for the reference's narrow phase. The
 * reference has no plugin/FFI layer; its query surface is the C++ API in
 * proj/include/lsnif/renderer.hpp and the file-local driver
 * run_narrow_phase (proj/src/renderer.cpp:232-265). Each entry point below
 * names the reference interface it replaces. Plain pointers and sizes only;
 * CUDA streams are passed as `void*` (a cudaStream_t, NULL = legacy stream).
 *
 * Threading: every call is reentrant. Calls on distinct streams may run
 * concurrently (per-stream scratch); a model is read-only after creation
 * (reference: shared_ptr<const LsnifModel>, renderer.hpp:76).
 * Errors: a non-zero lsnif_status plus a thread-local message
 * (lsnif_last_error). LSNIF_INVALID_ARGUMENT corresponds to the reference's
 * std::invalid_argument (renderer.cpp:185-189), LSNIF_RUNTIME_ERROR to
 * std::runtime_error (model_io.cpp:118-141).
 */
#ifndef LSNIF_GPU_H_
#define LSNIF_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum lsnif_status {
  LSNIF_OK = 0,
  LSNIF_INVALID_ARGUMENT = 1,
  LSNIF_RUNTIME_ERROR = 2,
  LSNIF_CUDA_ERROR = 3,
  LSNIF_UNSUPPORTED = 4
} lsnif_status;

/* lsnif::Ray (geometry.hpp:11-18), object space of the model, 32 B. */
typedef struct lsnif_ray {
  float origin[3];
  float direction[3];
  float t_min;
  float t_max;
} lsnif_ray;

/* lsnif::RayInterval (geometry.hpp:47-50). */
typedef struct lsnif_interval {
  float enter;
  float exit;
} lsnif_interval;

/* One query result, 32 B. Carries lsnif::NeuralHit (renderer.hpp:42-48)
 * plus the pipeline flags around it:
 *   bit 0 PAIR      the ray overlaps the model's frame box before t_max
 *                   (pair emission, renderer.cpp:165-172);
 *   bit 1 OCCLUDED  NeuralHit::occluded (sigmoid(z0) > 0.5, renderer.cpp:212);
 *   bit 2 ACCEPTED  the closest-hit (renderer.cpp:281-284) or any-hit
 *                   (renderer.cpp:317-320) accept rule holds;
 *   bits 8..31      NeuralHit::material_index.
 * t_world / normal / albedo are NeuralHit's fields (valid when PAIR). */
typedef struct lsnif_hit {
  uint32_t flags_material;
  float t_world;
  float normal[3];
  float albedo[3];
} lsnif_hit;

#define LSNIF_HIT_PAIR 1u
#define LSNIF_HIT_OCCLUDED 2u
#define LSNIF_HIT_ACCEPTED 4u
#define LSNIF_HIT_MATERIAL_SHIFT 8

/* Packed 16 B "wire" form of lsnif_hit, SURVEY.md §2.1 (parity layout fp32
 * fields, wire layout packed): for results that cross PCIe or NVLink.
 *   flags_material, t_world   bit-identical to the lsnif_hit fields;
 *   normal_oct    the unit normal, octahedral map, 2 x snorm16 (u low,
 *                 v high); angular error < 0.01 degree;
 *   albedo_unorm  3 x unorm10 (r bits 0-9, g 10-19, b 20-29), error
 *                 <= 0.5/1023; bit 30 set when the normal is zero (NeuralHit's
 *                 zero-length normal, renderer.cpp:216-219).
 * lsnif_hits_from_wire expands it back to lsnif_hit on the host. */
typedef struct lsnif_hit_wire {
  uint32_t flags_material;
  float t_world;
  uint32_t normal_oct;
  uint32_t albedo_unorm;
} lsnif_hit_wire;

#define LSNIF_WIRE_ZERO_NORMAL 0x40000000u

/* lsnif::Material (geometry.hpp:56-60), as stored in the model file. */
typedef struct lsnif_material {
  float albedo[3];
  uint32_t kind; /* 0 diffuse, 1 glossy */
  float roughness;
} lsnif_material;

/* Host-side mirror of lsnif::LsnifModel (model_io.hpp:18-36) with the
 * binary16 payloads exactly as in the LSNF v1 file (model_io.hpp:38-43). */
typedef struct lsnif_model_desc {
  int32_t voxel_res;  /* V */
  int32_t hit_cap;    /* H */
  int32_t n_levels;   /* L */
  int32_t f_dim;      /* F */
  uint32_t table_size; /* M */
  int32_t hidden;
  int32_t n_mat;
  const uint8_t* occupancy;        /* V^3/8 bytes, x fastest (voxel.hpp:10-11) */
  const int32_t* level_res;        /* n_levels */
  const uint16_t* const* tables;   /* n_levels x (M*F binary16, entry-major) */
  const uint16_t* w1;              /* hidden x (H*L*F), row-major binary16 */
  const uint16_t* b1;
  const uint16_t* w2;              /* hidden x hidden */
  const uint16_t* b2;
  const uint16_t* w3;              /* (8+n_mat) x hidden */
  const uint16_t* b3;
  const lsnif_material* materials;
  int32_t n_materials;
  float aabb[6];                   /* inflated frame box: min xyz, max xyz */
} lsnif_model_desc;

typedef struct lsnif_model_info {
  int32_t voxel_res, hit_cap, n_levels, f_dim;
  uint32_t table_size;
  int32_t hidden, n_mat, n_materials;
  int32_t level_res[4];
  float aabb[6];
  float activation_scale; /* power-of-two fp16 operand scale */
  uint64_t device_bytes;
  int32_t device; /* CUDA device ordinal the model lives on */
} lsnif_model_info;

/* Counters of the last lsnif_query on a stream (filled when requested). */
typedef struct lsnif_query_stats {
  int64_t rays;        /* queries answered */
  int64_t pairs;       /* rays overlapping the frame box */
  int64_t mlp_rows;    /* pairs with >= 1 boundary point (run through the MLP) */
  int64_t points;      /* boundary points encoded */
  int64_t volume_points;
} lsnif_query_stats;

typedef struct lsnif_model_s* lsnif_model;

enum { LSNIF_QUERY_CLOSEST = 0, LSNIF_QUERY_ANY = 1 };

/* Replaces load_model (model_io.cpp:116-175) + the model upload done once per
 * object in PreparedScene::prepare (renderer.cpp:55-76). */
lsnif_status lsnif_model_load(const char* path, int device, lsnif_model* out);
/* Same, from host arrays mirroring LsnifModel. */
lsnif_status lsnif_model_create(const lsnif_model_desc* desc, int device, lsnif_model* out);
lsnif_status lsnif_model_destroy(lsnif_model model);
lsnif_status lsnif_model_get_info(lsnif_model model, lsnif_model_info* out);

/* Replaces run_narrow_phase (renderer.cpp:232-265) for one object group,
 * fused with pair emission (renderer.cpp:165-172) and the accept rule of
 * intersect_scene (mode CLOSEST, renderer.cpp:280-301) or occluded_batch
 * (mode ANY, renderer.cpp:316-321). Rays/hits are DEVICE pointers; one
 * result per ray, in ray order. Asynchronous on `stream`. Scratch is kept
 * per (model, stream) and sized by the largest query: queries run in launch
 * pairs of 2^24 rays (~18.8 GB of scratch for the teapot-size model) when a
 * quarter of the free device memory holds that at the stream's first query,
 * else 2^23 (~9.4 GB); LSNIF_CHUNK_LOG2 fixes the size. */
lsnif_status lsnif_query(lsnif_model model, const lsnif_ray* d_rays, int64_t n, int mode,
                         lsnif_hit* d_hits, void* stream);

/* run_narrow_phase proper (renderer.cpp:232-265): every ray is a pair of
 * this object whose interval [t_enter, t_exit] (RayLsnifPair, renderer.hpp:33-38,
 * from collect_pairs' ray_aabb_intersect, renderer.cpp:165-172) is given in
 * d_intervals[i] instead of being recomputed; it feeds the t_world decode
 * and the accept rule exactly as the recomputed one does. DEVICE pointers. */
lsnif_status lsnif_query_pairs(lsnif_model model, const lsnif_ray* d_rays, const lsnif_interval* d_intervals,
                               int64_t n, int mode, lsnif_hit* d_hits, void* stream);
/* The two accept rules as separate entry points; d_intervals may be NULL
 * (intervals clipped in the kernel, as lsnif_query) or the pairs' intervals
 * (as lsnif_query_pairs). */
lsnif_status lsnif_query_closest(lsnif_model model, const lsnif_ray* d_rays, const lsnif_interval* d_intervals,
                                 int64_t n, lsnif_hit* d_hits, void* stream);
lsnif_status lsnif_query_any(lsnif_model model, const lsnif_ray* d_rays, const lsnif_interval* d_intervals,
                             int64_t n, lsnif_hit* d_hits, void* stream);

/* Same with HOST rays/hits (pinned or pageable): chunked H2D / query / D2H,
 * overlapped on internal streams. Synchronous. */
lsnif_status lsnif_query_host(lsnif_model model, const lsnif_ray* h_rays, int64_t n, int mode,
                              lsnif_hit* h_hits, void* stream);

/* lsnif_query / lsnif_query_host writing the packed 16 B wire records
 * (half the result bytes of lsnif_hit; same flags, material and t_world). */
lsnif_status lsnif_query_wire(lsnif_model model, const lsnif_ray* d_rays, int64_t n, int mode,
                              lsnif_hit_wire* d_hits, void* stream);
lsnif_status lsnif_query_host_wire(lsnif_model model, const lsnif_ray* h_rays, int64_t n, int mode,
                                   lsnif_hit_wire* h_hits, void* stream);
/* Host-side expansion of wire records into lsnif_hit records, no device needed. */
lsnif_status lsnif_hits_from_wire(const lsnif_hit_wire* h_wire, int64_t n, lsnif_hit* h_out);

/* Replaces infer_batch (renderer.cpp:183-226): `inputs` is the reference's
 * MatX inputs(input_width, n) column-major fp32 (DEVICE), intervals n
 * entries (DEVICE). Throws-equivalent LSNIF_INVALID_ARGUMENT when
 * n != n_intervals or rows != input_width. Results carry OCCLUDED and the
 * NeuralHit fields; PAIR/ACCEPTED are not set. Runs the columns through the
 * tcgen05 MLP (fp16 operands, the query path's numerics); columns with an
 * input beyond the model's encoder range (|x| > max |table entry|) are
 * answered by the fp32 kernel instead (decided on the device). Asynchronous
 * on `stream`. */
lsnif_status lsnif_infer_batch(lsnif_model model, const float* d_inputs, int64_t rows, int64_t n,
                               const lsnif_interval* d_intervals, int64_t n_intervals,
                               lsnif_hit* d_hits, void* stream);
/* The same with fp32 CUDA-core arithmetic in the reference's summation order
 * (mlp.hpp:121-130): a validation mode, ~100x slower. */
lsnif_status lsnif_infer_batch_f32(lsnif_model model, const float* d_inputs, int64_t rows, int64_t n,
                                   const lsnif_interval* d_intervals, int64_t n_intervals,
                                   lsnif_hit* d_hits, void* stream);

/* Bit-exactness probe: per-ray pair/interval, DDA boundary points, t
 * values, cells, hash indices and fp32 features, produced by the same device
 * functions the query kernels use. DEVICE output arrays (H/L/F of the model):
 *   info[n] (count | first_is_origin<<8 | pair<<9), interval[n][2], t[n][H],
 *   pts[n][H][3], cells[n][H] (x | y<<8 | z<<16), hidx[n][H][L][8],
 *   feat[n][H*L*F]. */
lsnif_status lsnif_debug_traverse(lsnif_model model, const lsnif_ray* d_rays, int64_t n,
                                  int32_t* info, float* interval, float* t, float* pts,
                                  uint32_t* cells, uint32_t* hidx, float* feat, void* stream);

/* Counters of the most recent lsnif_query on `stream` (synchronises it). */
lsnif_status lsnif_last_query_stats(lsnif_model model, void* stream, lsnif_query_stats* out);

/* ---- multi-object scenes ----
 * An instance places a model in the world: world_to_object is the 3x4
 * row-major affine [linear | translation] the reference stores as
 * PreparedObject::world_to_object (renderer.hpp:67-71). Models may be shared
 * by several instances (renderer.cpp:55-76). */
typedef struct lsnif_instance {
  lsnif_model model;
  float world_to_object[12];
} lsnif_instance;

/* lsnif::SurfaceHit (renderer.hpp:56-65) for the merged multi-object query,
 * 64 B. object_index = -1 when no instance was accepted. In ANY mode only
 * flags / object_index (the first instance that occludes) are set. */
typedef struct lsnif_scene_hit {
  float t;
  float position[3];
  float normal[3];  /* unit, world space, facing the incoming ray */
  float albedo[3];
  uint32_t kind;    /* MaterialKind of the model's material table */
  float roughness;
  int32_t object_index;
  uint32_t flags;   /* 1: hit (CLOSEST) / occluded (ANY) */
  uint32_t pad[2];
} lsnif_scene_hit;

typedef struct lsnif_scene_s* lsnif_scene;

/* Replaces the LSNIF part of PreparedScene::prepare (renderer.cpp:83-97):
 * the instance list; the models must live on one device and outlive the scene. */
lsnif_status lsnif_scene_create(const lsnif_instance* instances, int32_t n, lsnif_scene* out);
lsnif_status lsnif_scene_destroy(lsnif_scene scene);
/* Replaces the LSNIF phases of intersect_scene (mode CLOSEST,
 * renderer.cpp:277-303) and occluded_batch (mode ANY, 310-323) for a scene
 * without triangle objects: broad phase (collect_pairs, 154-181, exact
 * per-instance frame-box test instead of the top-level BVH prefilter),
 * per-object narrow phase in object order, and the accept/merge rules.
 * WORLD-space DEVICE rays in, one lsnif_scene_hit per ray out. */
lsnif_status lsnif_scene_query(lsnif_scene scene, const lsnif_ray* d_rays, int64_t n, int mode,
                               lsnif_scene_hit* d_hits, void* stream);
/* The same from HOST rays / results (intersect_scene's std::vector<Ray> in,
 * one result per ray out): chunked H2D -> scene query -> D2H through
 * per-scene staging buffers, ordered after `stream`; returns when h_hits is
 * filled. Pinned host memory gets the full PCIe rate. */
lsnif_status lsnif_scene_query_host(lsnif_scene scene, const lsnif_ray* h_rays, int64_t n, int mode,
                                    lsnif_scene_hit* h_hits, void* stream);

/* ---- wavefront path tracer ----
 * lsnif::Camera (scene.hpp:12-17), lsnif::Light (scene.hpp:19-26; point and
 * sphere lights — environment lights are summed into `environment` as
 * PreparedScene::prepare does, renderer.cpp:46-51) and the RenderConfig
 * fields the renderer reads (renderer.hpp:14-28). */
typedef struct lsnif_camera {
  float position[3];
  float look_at[3];
  float up[3];
  float vfov_deg;
} lsnif_camera;

enum { LSNIF_LIGHT_POINT = 0, LSNIF_LIGHT_SPHERE = 1 };
typedef struct lsnif_light {
  uint32_t type;
  float position[3];
  float radius;
  float radiance[3];
} lsnif_light;

typedef struct lsnif_render_config {
  int32_t width, height, spp, max_bounces;
  uint64_t seed;
  float neural_eps_scale; /* respawn offset for neural hits, x object world diagonal */
  int32_t max_paths_in_flight; /* 0 = library default; bounds device memory per wave */
} lsnif_render_config;

/* Ray counts of one lsnif_render call (optional output). */
typedef struct lsnif_render_stats {
  int64_t paths;          /* width * height * spp */
  int64_t closest_rays;   /* intersect_scene queries: camera + bounce rays */
  int64_t shadow_slots;   /* occluded_batch queries (fixed per-path slots, incl. empty) */
  int64_t shadow_rays;    /* filled shadow slots */
  int32_t waves;
  int32_t max_depth_reached;
} lsnif_render_stats;

/* Replaces render() (renderer.cpp:453-542) with PrimaryMode::lsnif for a
 * scene whose objects are all LSNIF instances: per path the reference's
 * mt19937 stream (seed_stream(seed, pixel, sample)), camera_ray, and per
 * bounce intersect_scene (lsnif_scene_query, CLOSEST), shade_hit (NEE to
 * every light + BSDF sample, renderer.cpp:378-442) and occluded_batch on the
 * shadow rays (lsnif_scene_query, ANY); the environment on a miss. Paths are
 * device resident between bounces (wavefront). `world_diag[i]` is
 * PreparedObject::world_diag of instance i (renderer.cpp:73-74; the mesh is
 * not part of the model). d_image: DEVICE float[height][width][3], written
 * as the spp-average like the reference's Image. At most 227 random draws
 * per path (2 + (max_bounces+1) * (2 * n_sphere_lights + 2)); larger
 * configurations return LSNIF_UNSUPPORTED. `stats` may be NULL. Synchronous. */
lsnif_status lsnif_render(lsnif_scene scene, const float* world_diag, int32_t n_instances,
                          const lsnif_camera* camera, const lsnif_light* lights, int32_t n_lights,
                          const float environment[3], const lsnif_render_config* config,
                          float* d_image, lsnif_render_stats* stats, void* stream);

/* Test probe of the renderer's sampling: for paths [first_path, first_path+n)
 * (path = pixel * spp + sample) the primary ray (renderer.cpp:347-361) and the
 * next k uniform draws of the path's stream. DEVICE outputs. */
lsnif_status lsnif_render_debug_paths(const lsnif_camera* camera, const lsnif_render_config* config,
                                      int64_t first_path, int64_t n, lsnif_ray* d_rays,
                                      float* d_uniforms, int32_t k, void* stream);

/* ---- GPU training ----
 * lsnif::train (training.cpp:95-230): fresh balanced batches of external and
 * surface rays labelled against the mesh (the reference's BVH oracle:
 * closest Moller-Trumbore hit, ties to the lower face), DDA + hash-grid
 * encode with the current fp32 tables, fp32 forward, composite_loss
 * (loss.hpp), backward (mlp.hpp:188-225), hash-gradient scatter
 * (encoding.hpp:193-209) and dense bias-corrected Adam on the MLP and the
 * tables (mlp.hpp:243-272). Random numbers: per-sample counter streams
 * (the reference's per-worker sequential mt19937 stream with rejection
 * retries is inherently serial); same distributions. */
typedef struct lsnif_mesh_desc {
  const float* vertices;      /* 3 per vertex (object space) */
  int32_t n_vertices;
  const float* normals;       /* 3 per vertex normal; NULL / 0 = geometric normals */
  int32_t n_normals;
  const int32_t* faces;       /* 3 vertex indices per triangle */
  const int32_t* face_normals; /* 3 normal indices per triangle, or NULL */
  const int32_t* face_material; /* per triangle, index into the model's material table */
  int32_t n_faces;
} lsnif_mesh_desc;

typedef struct lsnif_train_config {
  int32_t batch;        /* TrainConfig::batch */
  float lr;             /* Adam step size (AdamConfig::lr) */
  float external_mix;   /* fraction of rays originating outside */
  uint64_t seed;
} lsnif_train_config;

typedef struct lsnif_train_loss { /* LossTerms (loss.hpp:25-31), batch means */
  float total, occlusion_bce, local_t_mae, normal_cosine, albedo_rel_l2, material_ce;
  int64_t step;
} lsnif_train_loss;

/* TrainSample targets (training.hpp:15-22) for the batch-gradient probe. */
typedef struct lsnif_train_target {
  int32_t occluded;
  float local_t;
  float normal[3];
  float albedo[3];
  int32_t material;
} lsnif_train_target;

typedef struct lsnif_trainer_s* lsnif_trainer;

/* `init`: the starting model (e.g. make_sparse_hash_grid + make_mlp, or a
 * file's contents); its occupancy grid, frame box and materials are kept. */
lsnif_status lsnif_trainer_create(const lsnif_model_desc* init, const lsnif_mesh_desc* mesh,
                                  const lsnif_train_config* config, int device, lsnif_trainer* out);
/* Same, starting from an LSNF v1 file (e.g. the reference's init state saved
 * with save_model, or a model to fine-tune). */
lsnif_status lsnif_trainer_create_from_file(const char* path, const lsnif_mesh_desc* mesh,
                                            const lsnif_train_config* config, int device, lsnif_trainer* out);
lsnif_status lsnif_trainer_destroy(lsnif_trainer trainer);
/* Runs `steps` optimizer steps; `last` (nullable) gets the last step's loss. */
lsnif_status lsnif_trainer_step(lsnif_trainer trainer, int32_t steps, lsnif_train_loss* last, void* stream);
/* The current parameters as a query model, quantised to binary16 exactly as
 * save_model + load_model would (model_io.cpp:71-175). */
lsnif_status lsnif_trainer_export(lsnif_trainer trainer, lsnif_model* out);
/* Parity probe: loss terms and gradients of a GIVEN batch (object-space rays
 * + targets, DEVICE), no update. d_grad_mlp: w1|b1|w2|b2|w3|b3 row-major
 * fp32; d_grad_tables: n_levels x M x F fp32. Either may be NULL. */
lsnif_status lsnif_trainer_batch_grad(lsnif_trainer trainer, const lsnif_ray* d_rays,
                                      const lsnif_train_target* d_targets, int64_t n,
                                      lsnif_train_loss* loss, float* d_grad_mlp, float* d_grad_tables,
                                      void* stream);
/* The trainer's own sampler: n labelled samples of training step `step`. */
lsnif_status lsnif_trainer_sample(lsnif_trainer trainer, int64_t step, int64_t n, lsnif_ray* d_rays,
                                  lsnif_train_target* d_targets, void* stream);

/* Kernel-level timing of queries (bench / roofline support). When enabled,
 * CUDA events are recorded on the query stream around every kernel launch;
 * lsnif_profile_read synchronises `stream` and returns the summed device
 * durations since the last reset. `launches` counts every kernel the query
 * entry points launched (always tracked). */
typedef struct lsnif_profile {
  uint64_t launches;
  uint64_t trace_launches, mlp_launches;
  double trace_ms, mlp_ms;
} lsnif_profile;
lsnif_status lsnif_profile_enable(lsnif_model model, int enable);
lsnif_status lsnif_profile_read(lsnif_model model, void* stream, int reset, lsnif_profile* out);

const char* lsnif_last_error(void);
const char* lsnif_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* LSNIF_GPU_H_ */
