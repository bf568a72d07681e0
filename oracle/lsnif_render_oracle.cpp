// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// CPU restatement of the reference's path tracer for LSNIF-only scenes with
// PrimaryMode::lsnif (proj/src/renderer.cpp:330-542 + sampling.hpp), used by
// tests/ as the checker of the GPU wavefront renderer (lsnif_render). The
// intersections go through the oracle's scene_query (intersect_scene /
// occluded_batch restatement). std::mt19937 + uniform_real_distribution<float>
// are the reference's own generator and distribution (same libstdc++), so the
// random streams are the reference's. Vector expressions keep Eigen's
// evaluation order for Vector3f ((x + y) + z reductions, scalar chains left to
// right, normalized() = v / sqrt(squaredNorm)); build with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "lsnif_oracle.hpp"
#include "lsnif_render_oracle.hpp"

namespace oracle {
namespace {

using Rng = std::mt19937;  // sampling.hpp:10

float uniform_real(Rng& rng) {  // sampling.hpp:12-14
  return std::uniform_real_distribution<float>(0.0f, 1.0f)(rng);
}

struct V3 {
  float x = 0, y = 0, z = 0;
  float operator[](int i) const { return i == 0 ? x : i == 1 ? y : z; }
};
V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 mul(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
V3 mul(float s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
V3 cwise(V3 a, V3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
V3 divs(V3 a, float s) { return {a.x / s, a.y / s, a.z / s}; }
float dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
V3 normalized(V3 v) {
  const float n2 = dot(v, v);
  return n2 > 0.0f ? divs(v, std::sqrt(n2)) : v;
}
V3 v3(const float* p) { return {p[0], p[1], p[2]}; }

constexpr float kInf = std::numeric_limits<float>::infinity();
constexpr float kPi = static_cast<float>(M_PI);
constexpr float kInvPi = static_cast<float>(M_1_PI);

// sampling.hpp:18-24
void orthonormal_basis(V3 n, V3& t, V3& b) {
  const float sign = std::copysign(1.0f, n.z);
  const float a = -1.0f / (sign + n.z);
  const float bb = n.x * n.y * a;
  t = {1.0f + sign * n.x * n.x * a, sign * bb, -sign * n.x};
  b = {bb, sign + n.y * n.y * a, -n.y};
}

V3 uniform_sphere_dir(Rng& rng) {  // sampling.hpp:26-31
  const float z = 1.0f - 2.0f * uniform_real(rng);
  const float r = std::sqrt(std::max(0.0f, 1.0f - z * z));
  const float phi = 2.0f * kPi * uniform_real(rng);
  return {r * std::cos(phi), r * std::sin(phi), z};
}

V3 cosine_hemisphere_dir(V3 axis, Rng& rng) {  // sampling.hpp:35-46
  const float u1 = uniform_real(rng);
  const float u2 = uniform_real(rng);
  const float r = std::sqrt(u1);
  const float phi = 2.0f * kPi * u2;
  const float x = r * std::cos(phi);
  const float y = r * std::sin(phi);
  const float z = std::sqrt(std::max(0.0f, 1.0f - u1));
  V3 t, b;
  orthonormal_basis(axis, t, b);
  return normalized(add(add(mul(x, t), mul(y, b)), mul(z, axis)));
}

struct CameraBasis {  // renderer.cpp:329-344
  V3 origin, forward, right, up;
  float half_w, half_h;
};

CameraBasis make_camera_basis(const RCamera& cam, int width, int height) {
  CameraBasis b;
  b.origin = v3(cam.position);
  b.forward = normalized(sub(v3(cam.look_at), v3(cam.position)));
  b.right = normalized(cross(b.forward, v3(cam.up)));
  b.up = cross(b.right, b.forward);
  b.half_h = std::tan(0.5f * cam.vfov_deg * static_cast<float>(M_PI / 180.0));
  b.half_w = b.half_h * static_cast<float>(width) / static_cast<float>(height);
  return b;
}

Ray camera_ray(const CameraBasis& basis, int px, int py, int width, int height, Rng& rng) {
  const float u = uniform_real(rng);  // renderer.cpp:347-361
  const float v = uniform_real(rng);
  const float sx = 2.0f * (static_cast<float>(px) + u) / static_cast<float>(width) - 1.0f;
  const float sy = 1.0f - 2.0f * (static_cast<float>(py) + v) / static_cast<float>(height);
  const V3 d = normalized(add(add(basis.forward, mul(sx * basis.half_w, basis.right)),
                              mul(sy * basis.half_h, basis.up)));
  Ray r;
  r.o[0] = basis.origin.x;
  r.o[1] = basis.origin.y;
  r.o[2] = basis.origin.z;
  r.d[0] = d.x;
  r.d[1] = d.y;
  r.d[2] = d.z;
  r.t_min = 0.0f;
  r.t_max = kInf;
  return r;
}

struct ShadowItem {
  Ray ray;
  V3 contribution;
};
struct ShadeOutcome {  // renderer.cpp:368-374
  ShadowItem shadows[8];
  int n_shadows = 0;
  bool continue_path = false;
  Ray next_ray;
  V3 next_throughput;
};

// shade_hit (renderer.cpp:378-442) for a neural hit.
void shade_hit(const RenderSetup& S, const Ray& ray, const SceneHit& hit, V3 throughput, bool spawn,
               Rng& rng, ShadeOutcome& out) {
  out.n_shadows = 0;
  out.continue_path = false;
  const float eps = S.neural_eps_scale * S.world_diag[static_cast<size_t>(hit.object_index)];
  const V3 n = v3(hit.normal), albedo = v3(hit.albedo);
  const V3 spawn_origin = add(v3(hit.position), mul(eps, n));

  if (hit.kind == 0u) {
    for (const RLight& light : S.lights) {
      V3 target = v3(light.position);
      V3 light_normal;
      float pdf_area = 1.0f;
      if (light.type == 1u) {
        light_normal = uniform_sphere_dir(rng);
        target = add(v3(light.position), mul(light.radius, light_normal));
        pdf_area = 1.0f / (4.0f * kPi * light.radius * light.radius);
      }
      const V3 to_light = sub(target, spawn_origin);
      const float dist2 = dot(to_light, to_light);
      if (dist2 <= 0.0f) continue;
      const float dist = std::sqrt(dist2);
      const V3 wi = divs(to_light, dist);
      const float cos_surf = dot(n, wi);
      if (cos_surf <= 0.0f) continue;
      V3 contribution;
      if (light.type == 1u) {
        const float cos_light = dot(light_normal, mul(wi, -1.0f));
        if (cos_light <= 0.0f) continue;
        contribution = divs(mul(mul(mul(cwise(throughput, albedo), kInvPi), cos_surf), cos_light),
                            dist2 * pdf_area);
      } else {
        contribution = divs(mul(mul(cwise(throughput, albedo), kInvPi), cos_surf), dist2);
      }
      contribution = cwise(contribution, v3(light.radiance));
      if (contribution.x <= 0.0f && contribution.y <= 0.0f && contribution.z <= 0.0f) continue;
      if (out.n_shadows >= 8) continue;
      ShadowItem& item = out.shadows[out.n_shadows++];
      item.ray.o[0] = spawn_origin.x;
      item.ray.o[1] = spawn_origin.y;
      item.ray.o[2] = spawn_origin.z;
      item.ray.d[0] = wi.x;
      item.ray.d[1] = wi.y;
      item.ray.d[2] = wi.z;
      item.ray.t_min = 0.0f;
      item.ray.t_max = dist * static_cast<float>(1 - 1e-4);
      item.contribution = contribution;
    }
  }
  if (!spawn) return;
  V3 dir;
  if (hit.kind == 0u) {
    dir = cosine_hemisphere_dir(n, rng);
  } else {
    const V3 d = v3(ray.d);
    const V3 refl = normalized(sub(d, mul(2.0f * dot(d, n), n)));
    const float exponent = std::max(0.0f, 2.0f / (hit.roughness * hit.roughness) - 2.0f);
    const float u1 = uniform_real(rng);
    const float u2 = uniform_real(rng);
    const float cos_alpha = std::pow(u1, 1.0f / (exponent + 1.0f));
    const float sin_alpha = std::sqrt(std::max(0.0f, 1.0f - cos_alpha * cos_alpha));
    const float phi = 2.0f * kPi * u2;
    V3 t, b;
    orthonormal_basis(refl, t, b);
    dir = normalized(add(add(mul(sin_alpha * std::cos(phi), t), mul(sin_alpha * std::sin(phi), b)),
                         mul(cos_alpha, refl)));
    if (dot(dir, n) <= 0.0f) return;
  }
  out.continue_path = true;
  for (int a = 0; a < 3; ++a) out.next_ray.o[a] = spawn_origin[a];
  out.next_ray.d[0] = dir.x;
  out.next_ray.d[1] = dir.y;
  out.next_ray.d[2] = dir.z;
  out.next_ray.t_min = 0.0f;
  out.next_ray.t_max = kInf;
  out.next_throughput = cwise(throughput, albedo);
}

struct PathState {  // renderer.cpp:444-451
  Rng rng;
  Ray ray;
  V3 throughput{1.0f, 1.0f, 1.0f};
  V3 radiance;
  int pixel = 0;
  bool active = true;
};

}  // namespace

// render() (renderer.cpp:453-542), PrimaryMode::lsnif, all objects LSNIF:
// intersect_scene / occluded_batch are the oracle's scene_query.
void render(const RenderSetup& S, const Instance* inst, int n_inst, float* image, int workers, int64_t* stats) {
  int64_t n_closest = 0, n_shadow = 0;
  const int W = S.width, H = S.height;
  std::vector<V3> pixels(static_cast<size_t>(W) * H);
  const CameraBasis basis = make_camera_basis(S.camera, W, H);
  const int rows_per_block = std::max(1, 65536 / std::max(1, W * S.spp));
  std::vector<PathState> paths;
  std::vector<Ray> rays, shadow_rays;
  std::vector<int> ray_owner, shadow_owner;
  std::vector<V3> shadow_contrib;
  std::vector<SceneHit> hits, blocked;
  ShadeOutcome outcome;
  for (int y0 = 0; y0 < H; y0 += rows_per_block) {
    const int y1 = std::min(H, y0 + rows_per_block);
    paths.clear();
    for (int y = y0; y < y1; ++y)
      for (int x = 0; x < W; ++x) {
        const int pixel = y * W + x;
        for (int s = 0; s < S.spp; ++s) {
          PathState p;
          p.rng = Rng(seed_stream(S.seed, static_cast<uint64_t>(pixel), static_cast<uint64_t>(s)));
          p.ray = camera_ray(basis, x, y, W, H, p.rng);
          p.pixel = pixel;
          paths.push_back(std::move(p));
        }
      }
    for (int depth = 0; depth <= S.max_bounces; ++depth) {
      rays.clear();
      ray_owner.clear();
      for (size_t i = 0; i < paths.size(); ++i) {
        if (!paths[i].active) continue;
        rays.push_back(paths[i].ray);
        ray_owner.push_back(static_cast<int>(i));
      }
      if (rays.empty()) break;
      n_closest += static_cast<int64_t>(rays.size());
      hits.assign(rays.size(), SceneHit{});
      scene_query(inst, n_inst, rays.data(), static_cast<int64_t>(rays.size()), kClosest, hits.data(), workers);
      shadow_rays.clear();
      shadow_contrib.clear();
      shadow_owner.clear();
      for (size_t k = 0; k < rays.size(); ++k) {
        PathState& path = paths[static_cast<size_t>(ray_owner[k])];
        if (!(hits[k].flags & 1u)) {
          path.radiance = add(path.radiance, cwise(path.throughput, v3(S.environment)));
          path.active = false;
          continue;
        }
        shade_hit(S, path.ray, hits[k], path.throughput, depth < S.max_bounces, path.rng, outcome);
        for (int s = 0; s < outcome.n_shadows; ++s) {
          shadow_rays.push_back(outcome.shadows[s].ray);
          shadow_contrib.push_back(outcome.shadows[s].contribution);
          shadow_owner.push_back(ray_owner[k]);
        }
        if (outcome.continue_path) {
          path.ray = outcome.next_ray;
          path.throughput = outcome.next_throughput;
        } else {
          path.active = false;
        }
      }
      if (!shadow_rays.empty()) {
        n_shadow += static_cast<int64_t>(shadow_rays.size());
        blocked.assign(shadow_rays.size(), SceneHit{});
        scene_query(inst, n_inst, shadow_rays.data(), static_cast<int64_t>(shadow_rays.size()), kAny,
                    blocked.data(), workers);
        for (size_t s = 0; s < shadow_rays.size(); ++s)
          if (!(blocked[s].flags & 1u)) {
            PathState& p = paths[static_cast<size_t>(shadow_owner[s])];
            p.radiance = add(p.radiance, shadow_contrib[s]);
          }
      }
    }
    for (const PathState& p : paths) {
      V3& px = pixels[static_cast<size_t>(p.pixel)];
      px = add(px, p.radiance);
    }
  }
  if (stats) {
    stats[0] = n_closest;
    stats[1] = n_shadow;
  }
  const float inv_spp = 1.0f / static_cast<float>(S.spp);
  for (size_t i = 0; i < pixels.size(); ++i) {
    image[3 * i + 0] = pixels[i].x * inv_spp;
    image[3 * i + 1] = pixels[i].y * inv_spp;
    image[3 * i + 2] = pixels[i].z * inv_spp;
  }
}

// Primary ray + the next k uniform draws of path (pixel * spp + sample).
void render_debug_paths(const RenderSetup& S, int64_t first_path, int64_t n, Ray* rays, float* u, int k) {
  const CameraBasis basis = make_camera_basis(S.camera, S.width, S.height);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t path = first_path + i;
    const int64_t pixel = path / S.spp;
    const int64_t s = path % S.spp;
    Rng rng(seed_stream(S.seed, static_cast<uint64_t>(pixel), static_cast<uint64_t>(s)));
    rays[i] = camera_ray(basis, static_cast<int>(pixel % S.width), static_cast<int>(pixel / S.width), S.width,
                         S.height, rng);
    for (int q = 0; q < k; ++q) u[i * k + q] = uniform_real(rng);
  }
}

}  // namespace oracle
