// TEST INFRASTRUCTURE — NOT PRODUCT CODE. See lsnif_oracle.hpp for the contract.
// All citations are reference paths relative to proj/.
#include "lsnif_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <random>
#include <sstream>
#include <stdexcept>
#include <thread>

namespace oracle {

// ---------------------------------------------------------------- L0 numerics

// types.hpp:25-31
uint64_t mix_bits(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// types.hpp:33-39
uint32_t seed_stream(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = mix_bits(seed + 0x632be59bd9b4e019ull);
  h = mix_bits(h ^ a);
  h = mix_bits(h ^ b);
  h = mix_bits(h ^ c);
  return static_cast<uint32_t>(h >> 32);
}

// half.hpp:10-37 (IEEE binary16, round to nearest even)
uint16_t float_to_half(float value) {
  uint32_t x;
  std::memcpy(&x, &value, 4);
  const uint16_t sign = static_cast<uint16_t>((x >> 16) & 0x8000u);
  const uint32_t exp_bits = (x >> 23) & 0xffu;
  uint32_t man = x & 0x7fffffu;
  if (exp_bits == 0xffu) return static_cast<uint16_t>(sign | 0x7c00u | (man ? 0x200u : 0u));
  const int exp = static_cast<int>(exp_bits) - 127 + 15;
  if (exp >= 31) return static_cast<uint16_t>(sign | 0x7c00u);
  if (exp <= 0) {
    if (exp < -10) return sign;
    man |= 0x800000u;
    const uint32_t shift = static_cast<uint32_t>(14 - exp);
    uint32_t half_man = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (half_man & 1u))) ++half_man;
    return static_cast<uint16_t>(sign | half_man);
  }
  uint16_t h = static_cast<uint16_t>(sign | (exp << 10) | (man >> 13));
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return h;
}

// half.hpp:39-64
float half_to_float(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1fu;
  uint32_t man = h & 0x3ffu;
  uint32_t x;
  if (exp == 0) {
    if (man == 0) {
      x = sign;
    } else {
      int shift = 0;
      while (!(man & 0x400u)) {
        man <<= 1;
        ++shift;
      }
      man &= 0x3ffu;
      x = sign | static_cast<uint32_t>(113 - shift) << 23 | (man << 13);
    }
  } else if (exp == 31) {
    x = sign | 0x7f800000u | (man << 13);
  } else {
    x = sign | ((exp - 15 + 127) << 23) | (man << 13);
  }
  float out;
  std::memcpy(&out, &x, 4);
  return out;
}

// ------------------------------------------------------------------ geometry

// std::max / std::min / std::clamp semantics spelled out (first argument wins
// ties), so the GPU path can mirror them with explicit selects.
static inline float smax(float a, float b) { return (a < b) ? b : a; }
static inline float smin(float a, float b) { return (b < a) ? b : a; }
template <typename T>
static inline T sclamp(T v, T lo, T hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// geometry.cpp:9-28
bool ray_aabb_intersect(const Ray& ray, const Aabb& box, Interval* out) {
  float t0 = ray.t_min;
  float t1 = ray.t_max;
  for (int a = 0; a < 3; ++a) {
    const float o = ray.o[a];
    const float d = ray.d[a];
    if (d == 0.0f) {
      if (o < box.mn[a] || o > box.mx[a]) return false;
      continue;
    }
    const float inv = 1.0f / d;
    float ta = (box.mn[a] - o) * inv;
    float tb = (box.mx[a] - o) * inv;
    if (ta > tb) std::swap(ta, tb);
    t0 = smax(t0, ta);
    t1 = smin(t1, tb);
    if (t0 > t1) return false;
  }
  out->enter = t0;
  out->exit = t1;
  return true;
}

// geometry.cpp:93-103 (LocalFrame::for_aabb)
Aabb inflate_frame(Aabb box) {
  float ext[3];
  for (int a = 0; a < 3; ++a) ext[a] = box.mx[a] - box.mn[a];
  float mx = ext[0];  // Eigen maxCoeff: first max wins
  if (ext[1] > mx) mx = ext[1];
  if (ext[2] > mx) mx = ext[2];
  float pad = 1e-4f * mx;
  if (!(pad > 0.0f)) pad = 1e-4f;
  for (int a = 0; a < 3; ++a) {
    box.mn[a] -= pad;
    box.mx[a] += pad;
  }
  return box;
}

// --------------------------------------------------------------------- voxel

// voxel.hpp:20-23, 30-34 (x fastest, bit i&7 of byte i>>3)
bool occupied(const std::vector<uint8_t>& bits, int res, int ix, int iy, int iz) {
  const size_t i = static_cast<size_t>(ix) +
                   static_cast<size_t>(res) *
                       (static_cast<size_t>(iy) + static_cast<size_t>(res) * iz);
  return (bits[i >> 3] >> (i & 7)) & 1u;
}

static inline void cross3(const float a[3], const float b[3], float out[3]) {
  out[0] = a[1] * b[2] - a[2] * b[1];
  out[1] = a[2] * b[0] - a[0] * b[2];
  out[2] = a[0] * b[1] - a[1] * b[0];
}
static inline float dot3(const float a[3], const float b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// voxel.cpp:37-42
static inline bool axis_separates(float pa, float pb, float pc, float rad) {
  const float lo = std::min(pa, std::min(pb, pc));
  const float hi = std::max(pa, std::max(pb, pc));
  return lo > rad || hi < -rad;
}

// voxel.cpp:47-80
bool triangle_box_overlap(const float center[3], const float half[3], const float a[3],
                          const float b[3], const float c[3]) {
  float v0[3], v1[3], v2[3];
  for (int i = 0; i < 3; ++i) {
    v0[i] = a[i] - center[i];
    v1[i] = b[i] - center[i];
    v2[i] = c[i] - center[i];
  }
  for (int i = 0; i < 3; ++i)
    if (axis_separates(v0[i], v1[i], v2[i], half[i])) return false;
  float e[3][3];
  for (int i = 0; i < 3; ++i) {
    e[0][i] = v1[i] - v0[i];
    e[1][i] = v2[i] - v1[i];
    e[2][i] = v0[i] - v2[i];
  }
  for (int k = 0; k < 3; ++k) {
    for (int i = 0; i < 3; ++i) {
      float axis[3] = {0, 0, 0};
      axis[i] = 1.0f;
      float n[3];
      cross3(axis, e[k], n);
      const float rad =
          half[0] * std::abs(n[0]) + half[1] * std::abs(n[1]) + half[2] * std::abs(n[2]);
      if (axis_separates(dot3(n, v0), dot3(n, v1), dot3(n, v2), rad)) return false;
    }
  }
  float normal[3];
  cross3(e[0], e[1], normal);
  const float d = dot3(normal, v0);
  const float rad = half[0] * std::abs(normal[0]) + half[1] * std::abs(normal[1]) +
                    half[2] * std::abs(normal[2]);
  return std::abs(d) <= rad;
}

// voxel.cpp:82-127
std::vector<uint8_t> voxelize_surface(const std::vector<float>& verts,
                                      const std::vector<int>& faces, const Aabb& frame,
                                      int resolution) {
  if (resolution < 2 || resolution > 256 || (resolution & (resolution - 1)) != 0)
    throw std::invalid_argument("occupancy resolution must be a power of two in [2, 256]");
  std::vector<uint8_t> bits(static_cast<size_t>(resolution) * resolution * resolution / 8, 0);
  float inv_ext[3];
  for (int a = 0; a < 3; ++a) inv_ext[a] = 1.0f / (frame.mx[a] - frame.mn[a]);
  auto to_local = [&](int v, float out[3]) {
    for (int a = 0; a < 3; ++a) out[a] = (verts[3 * v + a] - frame.mn[a]) * inv_ext[a];
  };
  const float res = static_cast<float>(resolution);
  const float cell = 1.0f / res;
  const float half[3] = {0.5f * cell, 0.5f * cell, 0.5f * cell};
  auto range_lo = [&](float lo) {
    return std::max(0, static_cast<int>(std::ceil(lo * res - 1.0f)));
  };
  auto range_hi = [&](float hi) {
    return std::min(resolution - 1, static_cast<int>(std::floor(hi * res)));
  };
  auto set = [&](int ix, int iy, int iz) {
    const size_t i = static_cast<size_t>(ix) +
                     static_cast<size_t>(resolution) *
                         (static_cast<size_t>(iy) + static_cast<size_t>(resolution) * iz);
    bits[i >> 3] |= static_cast<uint8_t>(1u << (i & 7));
  };
  const int n_faces = static_cast<int>(faces.size() / 3);
  for (int f = 0; f < n_faces; ++f) {
    float a[3], b[3], c[3];
    to_local(faces[3 * f + 0], a);
    to_local(faces[3 * f + 1], b);
    to_local(faces[3 * f + 2], c);
    float lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      // Eigen cwiseMin/cwiseMax: min(a, b) then min(., c)
      lo[k] = std::min(std::min(a[k], b[k]), c[k]);
      hi[k] = std::max(std::max(a[k], b[k]), c[k]);
    }
    const int x0 = range_lo(lo[0]), x1 = range_hi(hi[0]);
    const int y0 = range_lo(lo[1]), y1 = range_hi(hi[1]);
    const int z0 = range_lo(lo[2]), z1 = range_hi(hi[2]);
    float ba[3], ca[3], cr[3];
    for (int k = 0; k < 3; ++k) {
      ba[k] = b[k] - a[k];
      ca[k] = c[k] - a[k];
    }
    cross3(ba, ca, cr);
    const bool degenerate = std::sqrt(dot3(cr, cr)) < 1e-16f;
    for (int iz = z0; iz <= z1; ++iz)
      for (int iy = y0; iy <= y1; ++iy)
        for (int ix = x0; ix <= x1; ++ix) {
          if (degenerate) {
            set(ix, iy, iz);
            continue;
          }
          const float center[3] = {(ix + 0.5f) * cell, (iy + 0.5f) * cell,
                                   (iz + 0.5f) * cell};
          if (triangle_box_overlap(center, half, a, b, c)) set(ix, iy, iz);
        }
  }
  return bits;
}

// ----------------------------------------------------------------------- OBJ

// obj.cpp:17-21
static int resolve_index(int raw, int count, const std::string& name, int line) {
  const int idx = raw > 0 ? raw - 1 : count + raw;
  if (idx < 0 || idx >= count)
    throw std::runtime_error(name + ":" + std::to_string(line) + ": index out of range");
  return idx;
}

// obj.cpp:53-113 (positions, faces with fan triangulation, usemtl slots)
ObjMesh load_obj(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open OBJ file: " + path);
  ObjMesh mesh;
  std::map<std::string, int> material_slots;
  int current_material = 0;
  bool default_slot_used = false;
  std::string line;
  int line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      float p[3];
      if (!(ls >> p[0] >> p[1] >> p[2]))
        throw std::runtime_error(path + ":" + std::to_string(line_no) + ": bad vertex record");
      mesh.verts.insert(mesh.verts.end(), p, p + 3);
    } else if (tag == "usemtl") {
      std::string mat_name;
      ls >> mat_name;
      auto it = material_slots.find(mat_name);
      if (it == material_slots.end()) {
        const int slot = static_cast<int>(material_slots.size()) + (default_slot_used ? 1 : 0);
        it = material_slots.emplace(mat_name, slot).first;
      }
      current_material = it->second;
    } else if (tag == "f") {
      if (material_slots.empty() && !default_slot_used) default_slot_used = true;
      std::vector<int> corners;
      std::string token;
      const int nv = static_cast<int>(mesh.verts.size() / 3);
      while (ls >> token) {
        const size_t slash = token.find('/');
        const std::string head = token.substr(0, slash);
        corners.push_back(resolve_index(std::stoi(head), nv, path, line_no));
      }
      if (corners.size() < 3)
        throw std::runtime_error(path + ":" + std::to_string(line_no) +
                                 ": face with fewer than 3 vertices");
      for (size_t i = 2; i < corners.size(); ++i) {
        mesh.faces.push_back(corners[0]);
        mesh.faces.push_back(corners[i - 1]);
        mesh.faces.push_back(corners[i]);
        mesh.face_material.push_back(current_material);
      }
    }
  }
  int n_mat = 1;
  for (const auto& kv : material_slots) n_mat = std::max(n_mat, kv.second + 1);
  mesh.n_mat = n_mat;
  return mesh;
}

// ----------------------------------------------------------------------- DDA

// dda.cpp:14-36
static bool slab_interval(const float o[3], const float d[3], float t_min, float t_max,
                          float& t0, float& t1, int& enter_axis) {
  t0 = t_min;
  t1 = t_max;
  enter_axis = -1;
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0f) {
      if (o[a] < 0.0f || o[a] > 1.0f) return false;
      continue;
    }
    const float inv = 1.0f / d[a];
    float ta = (0.0f - o[a]) * inv;
    float tb = (1.0f - o[a]) * inv;
    if (ta > tb) std::swap(ta, tb);
    if (ta > t0) {
      t0 = ta;
      enter_axis = a;
    }
    if (tb < t1) t1 = tb;
    if (t0 > t1) return false;
  }
  return true;
}

// dda.cpp:40-117
void collect_boundary_hits_local(const float origin[3], const float direction[3],
                                 float t_min, float t_max, const std::vector<uint8_t>& occ,
                                 int res, int cap, BoundaryHits& out) {
  out.clear();
  if (cap < 1) throw std::invalid_argument("hit cap must be >= 1");
  const float fres = static_cast<float>(res);

  float o[3] = {origin[0], origin[1], origin[2]};
  for (int a = 0; a < 3; ++a) {  // dda.cpp:49-53
    const float scaled = o[a] * fres;
    if (scaled == std::floor(scaled)) o[a] += 1e-7f;
  }

  float t0, t1;
  int entry_axis;
  if (!slab_interval(o, direction, t_min, t_max, t0, t1, entry_axis)) return;

  float start[3];
  for (int a = 0; a < 3; ++a) start[a] = o[a] + t0 * direction[a];
  int cell[3], step[3];
  float t_next[3], t_delta[3];
  const float kInf = std::numeric_limits<float>::infinity();
  for (int a = 0; a < 3; ++a) {  // dda.cpp:64-79
    cell[a] = sclamp(static_cast<int>(std::floor(start[a] * fres)), 0, res - 1);
    if (direction[a] > 0.0f) {
      step[a] = 1;
      t_delta[a] = 1.0f / (fres * direction[a]);
      t_next[a] = t0 + ((cell[a] + 1) / fres - start[a]) / direction[a];
    } else if (direction[a] < 0.0f) {
      step[a] = -1;
      t_delta[a] = -1.0f / (fres * direction[a]);
      t_next[a] = t0 + (cell[a] / fres - start[a]) / direction[a];
    } else {
      step[a] = 0;
      t_delta[a] = kInf;
      t_next[a] = kInf;
    }
  }

  float entry_t = t0;
  float entry_point[3] = {start[0], start[1], start[2]};
  float entry_plane = -1.0f;
  if (entry_axis >= 0) entry_plane = std::round(start[entry_axis] * fres);

  while (true) {  // dda.cpp:88-116
    if (occupied(occ, res, cell[0], cell[1], cell[2])) {
      float p[3] = {entry_point[0], entry_point[1], entry_point[2]};
      if (entry_axis >= 0) {
        p[entry_axis] = entry_plane / fres;
      } else if (out.count() == 0) {
        out.first_is_origin = true;
      }
      out.points.insert(out.points.end(), p, p + 3);
      out.t_values.push_back(entry_t);
      out.cells.insert(out.cells.end(), cell, cell + 3);
      if (out.count() >= cap) return;
    }
    int axis = 0;
    if (t_next[1] < t_next[axis]) axis = 1;
    if (t_next[2] < t_next[axis]) axis = 2;
    if (t_next[axis] > t1) return;
    entry_t = t_next[axis];
    entry_plane = static_cast<float>(step[axis] > 0 ? cell[axis] + 1 : cell[axis]);
    cell[axis] += step[axis];
    if (cell[axis] < 0 || cell[axis] >= res) return;
    for (int a = 0; a < 3; ++a) entry_point[a] = o[a] + entry_t * direction[a];
    entry_axis = axis;
    t_next[axis] += t_delta[axis];
  }
}

// ------------------------------------------------------------------ encoding

// encoding.hpp:18-23
uint32_t hash_vertex(int ix, int iy, int iz, uint32_t table_size) {
  const uint32_t h = static_cast<uint32_t>(ix) * 1u ^ static_cast<uint32_t>(iy) * 2654435761u ^
                     static_cast<uint32_t>(iz) * 805459861u;
  return h % table_size;
}

// encoding.hpp:84-140
void encode_point_level(const Model& m, int level, const float p[3], bool volume,
                        float* features, PointCode* code) {
  const int res = m.level_res[static_cast<size_t>(level)];
  const float fres = static_cast<float>(res);
  float u[3];
  for (int a = 0; a < 3; ++a) u[a] = p[a] * fres;
  int base[3];
  float frac[3];
  int plane_axis = -1;
  if (!volume) {
    float best = std::numeric_limits<float>::max();
    for (int a = 0; a < 3; ++a) {
      const float scaled = p[a] * static_cast<float>(m.voxel_res);
      const float dist = std::abs(scaled - std::round(scaled));
      if (dist < best) {
        best = dist;
        plane_axis = a;
      }
    }
  }
  for (int a = 0; a < 3; ++a) {
    if (a == plane_axis) {
      base[a] = sclamp(static_cast<int>(std::round(u[a])), 0, res);
      frac[a] = 0.0f;
    } else {
      base[a] = sclamp(static_cast<int>(std::floor(u[a])), 0, res - 1);
      frac[a] = sclamp(u[a] - static_cast<float>(base[a]), 0.0f, 1.0f);
    }
  }
  if (code) {
    code->count = 0;
    code->plane_axis = plane_axis;
  }
  const std::vector<float>& table = m.tables[static_cast<size_t>(level)];
  for (int f = 0; f < m.f_dim; ++f) features[f] = 0.0f;
  for (int corner = 0; corner < 8; ++corner) {
    const int dx = corner & 1, dy = (corner >> 1) & 1, dz = (corner >> 2) & 1;
    if (plane_axis == 0 && dx) continue;
    if (plane_axis == 1 && dy) continue;
    if (plane_axis == 2 && dz) continue;
    const float wx = dx ? frac[0] : 1.0f - frac[0];
    const float wy = dy ? frac[1] : 1.0f - frac[1];
    const float wz = dz ? frac[2] : 1.0f - frac[2];
    const float w = wx * wy * wz;
    const uint32_t idx = hash_vertex(base[0] + dx, base[1] + dy, base[2] + dz, m.table_size);
    if (code) {
      code->index[code->count] = idx;
      code->weight[code->count] = w;
      ++code->count;
    }
    for (int f = 0; f < m.f_dim; ++f)
      features[f] += w * table[static_cast<size_t>(idx) * m.f_dim + f];
  }
}

// encoding.hpp:148-154, 166-176
void encode_ray_into(const Model& m, const BoundaryHits& hits, float* column,
                     PointCode* codes, int& point_count) {
  const int lf = m.n_levels * m.f_dim;
  point_count = std::min(hits.count(), m.hit_cap);
  for (int i = 0; i < m.hit_cap * lf; ++i) column[i] = 0.0f;
  for (int i = 0; i < point_count; ++i) {
    const bool volume = (i == 0) && hits.first_is_origin;
    for (int l = 0; l < m.n_levels; ++l)
      encode_point_level(m, l, &hits.points[static_cast<size_t>(3 * i)], volume,
                         column + i * lf + l * m.f_dim,
                         codes ? codes + i * m.n_levels + l : nullptr);
  }
}

// ---------------------------------------------------------------------- init

// encoding.hpp:46-69 + mlp.hpp:44-65 (kaiming_init draws a fresh
// normal_distribution per matrix, row-major order; biases zero).
void init_random_model(Model& m, uint64_t seed) {
  {
    std::mt19937 rng(seed_stream(seed, 0x9dd1));
    std::uniform_real_distribution<double> dist(-1e-4, 1e-4);
    m.tables.assign(m.level_res.size(), {});
    for (size_t l = 0; l < m.level_res.size(); ++l) {
      if (m.level_res[l] % m.voxel_res != 0)
        throw std::invalid_argument("level resolution must be a multiple of the voxel resolution");
      std::vector<float>& t = m.tables[l];
      t.assign(static_cast<size_t>(m.table_size) * m.f_dim, 0.0f);
      for (uint32_t e = 0; e < m.table_size; ++e)
        for (int f = 0; f < m.f_dim; ++f)
          t[static_cast<size_t>(e) * m.f_dim + f] = static_cast<float>(dist(rng));
    }
  }
  std::mt19937 rng(seed_stream(seed, 0x3b8d));
  auto kaiming = [&](int rows, int cols, std::vector<float>& w) {
    std::normal_distribution<double> dist(0.0, std::sqrt(2.0 / cols));
    w.assign(static_cast<size_t>(rows) * cols, 0.0f);
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) w[static_cast<size_t>(r) * cols + c] = static_cast<float>(dist(rng));
  };
  const int in = m.input_width();
  kaiming(m.hidden, in, m.w1);
  m.b1.assign(static_cast<size_t>(m.hidden), 0.0f);
  kaiming(m.hidden, m.hidden, m.w2);
  m.b2.assign(static_cast<size_t>(m.hidden), 0.0f);
  kaiming(8 + m.n_mat, m.hidden, m.w3);
  m.b3.assign(static_cast<size_t>(8 + m.n_mat), 0.0f);
  finalize_model(m);
}

// ----------------------------------------------------------------------- MLP

// renderer.cpp:197-207: z = W x + b per layer, leaky slope 0.01 on z < 0.
// Each output sums its products sequentially over the input index (Eigen's
// GEMV order is library-internal). The loop is written in column (axpy) form
// over transposed weights so the timing build vectorises like a column-major
// Eigen GEMV; the per-output summation order is unchanged.
static void dense_axpy(const float* wt, const float* x, int in, int out, float* z) {
  for (int i = 0; i < out; ++i) z[i] = 0.0f;
  for (int j = 0; j < in; ++j) {
    const float xj = x[j];
    const float* col = wt + static_cast<size_t>(j) * out;
    for (int i = 0; i < out; ++i) z[i] += col[i] * xj;
  }
}

void mlp_logits(const Model& m, const float* x, float* z3) {
  const int in = m.input_width();
  const int h = m.hidden;
  float z1[512], z2[512];
  if (h > 512) throw std::invalid_argument("hidden width > 512 unsupported by the oracle");
  dense_axpy(m.w1t.data(), x, in, h, z1);
  for (int i = 0; i < h; ++i) {
    z1[i] = z1[i] + m.b1[static_cast<size_t>(i)];
    if (z1[i] < 0.0f) z1[i] *= 0.01f;
  }
  dense_axpy(m.w2t.data(), z1, h, h, z2);
  for (int i = 0; i < h; ++i) {
    z2[i] = z2[i] + m.b2[static_cast<size_t>(i)];
    if (z2[i] < 0.0f) z2[i] *= 0.01f;
  }
  const int out = m.output_width();
  dense_axpy(m.w3t.data(), z2, h, out, z3);
  for (int i = 0; i < out; ++i) z3[i] = z3[i] + m.b3[static_cast<size_t>(i)];
}

static std::vector<float> transpose(const std::vector<float>& w, int rows, int cols) {
  std::vector<float> t(w.size());
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c)
      t[static_cast<size_t>(c) * rows + r] = w[static_cast<size_t>(r) * cols + c];
  return t;
}

void finalize_model(Model& m) {
  m.w1t = transpose(m.w1, m.hidden, m.input_width());
  m.w2t = transpose(m.w2, m.hidden, m.hidden);
  m.w3t = transpose(m.w3, m.output_width(), m.hidden);
}

// mlp.hpp:80-94 (apply_heads) + renderer.cpp:211-223 (decode)
NeuralHit decode_logits(const Model& m, const float* z, Interval iv) {
  auto sig = [](float v) { return 1.0f / (1.0f + std::exp(-v)); };
  NeuralHit nh;
  const float occ = sig(z[0]);
  const float local_t = sig(z[1]);
  nh.occluded = occ > 0.5f;
  nh.t_world = iv.enter + local_t * (iv.exit - iv.enter);
  const float n0 = z[2], n1 = z[3], n2 = z[4];
  const float len = std::sqrt(n0 * n0 + n1 * n1 + n2 * n2);
  if (len > 1e-12f) {
    nh.normal[0] = n0 / len;
    nh.normal[1] = n1 / len;
    nh.normal[2] = n2 / len;
  }
  for (int k = 0; k < 3; ++k) nh.albedo[k] = sig(z[5 + k]);
  // softmax with max subtraction, then first argmax of the probabilities
  const int n_mat = m.n_mat;
  float zmax = z[8];
  for (int k = 1; k < n_mat; ++k)
    if (z[8 + k] > zmax) zmax = z[8 + k];
  std::vector<float> e(static_cast<size_t>(n_mat));
  float sum = 0.0f;
  for (int k = 0; k < n_mat; ++k) {
    e[static_cast<size_t>(k)] = std::exp(z[8 + k] - zmax);
    sum += e[static_cast<size_t>(k)];
  }
  int arg = 0;
  float best = e[0] / sum;
  for (int k = 1; k < n_mat; ++k) {
    const float pk = e[static_cast<size_t>(k)] / sum;
    if (pk > best) {
      best = pk;
      arg = k;
    }
  }
  nh.material_index = arg;
  return nh;
}

NeuralHit infer_one(const Model& m, const float* x, Interval iv) {
  std::vector<float> z(static_cast<size_t>(m.output_width()));
  mlp_logits(m, x, z.data());
  return decode_logits(m, z.data(), iv);
}

// ---------------------------------------------------------------- model file

namespace {
void write_u32(std::ostream& out, uint32_t v) { out.write(reinterpret_cast<const char*>(&v), 4); }
void write_f32(std::ostream& out, float v) { out.write(reinterpret_cast<const char*>(&v), 4); }
void write_half(std::ostream& out, float v) {
  const uint16_t h = float_to_half(v);
  out.write(reinterpret_cast<const char*>(&h), 2);
}
uint32_t read_u32(std::istream& in) {
  uint32_t v;
  if (!in.read(reinterpret_cast<char*>(&v), 4)) throw std::runtime_error("model file truncated");
  return v;
}
float read_f32(std::istream& in) {
  float v;
  if (!in.read(reinterpret_cast<char*>(&v), 4)) throw std::runtime_error("model file truncated");
  return v;
}
float read_half(std::istream& in) {
  uint16_t h;
  if (!in.read(reinterpret_cast<char*>(&h), 2)) throw std::runtime_error("model file truncated");
  return half_to_float(h);
}
}  // namespace

// model_io.cpp:71-114
void save_model(const Model& m, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open model file for writing: " + path);
  out.write("LSNF", 4);
  write_u32(out, 1u);
  write_u32(out, static_cast<uint32_t>(m.voxel_res));
  write_u32(out, static_cast<uint32_t>(m.hit_cap));
  write_u32(out, static_cast<uint32_t>(m.n_levels));
  write_u32(out, static_cast<uint32_t>(m.f_dim));
  write_u32(out, m.table_size);
  write_u32(out, static_cast<uint32_t>(m.hidden));
  write_u32(out, static_cast<uint32_t>(m.n_mat));
  out.write(reinterpret_cast<const char*>(m.occupancy.data()),
            static_cast<std::streamsize>(m.occupancy.size()));
  for (size_t l = 0; l < m.tables.size(); ++l) {
    write_u32(out, static_cast<uint32_t>(m.level_res[l]));
    for (float v : m.tables[l]) write_half(out, v);
  }
  for (const auto* t : {&m.w1, &m.b1, &m.w2, &m.b2, &m.w3, &m.b3})
    for (float v : *t) write_half(out, v);
  write_u32(out, static_cast<uint32_t>(m.materials.size()));
  for (const Material& mat : m.materials) {
    for (int c = 0; c < 3; ++c) write_f32(out, mat.albedo[c]);
    write_u32(out, mat.kind);
    write_f32(out, mat.roughness);
  }
  for (int c = 0; c < 3; ++c) write_f32(out, m.aabb.mn[c]);
  for (int c = 0; c < 3; ++c) write_f32(out, m.aabb.mx[c]);
  if (!out) throw std::runtime_error("failed writing model file: " + path);
}

// model_io.cpp:116-175
Model load_model(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open model file: " + path);
  char magic[4];
  if (!in.read(magic, 4)) throw std::runtime_error("model file truncated");
  if (std::memcmp(magic, "LSNF", 4) != 0)
    throw std::runtime_error("not an LSNIF model file (bad magic): " + path);
  const uint32_t version = read_u32(in);
  if (version != 1u) throw std::runtime_error("unsupported model version " + std::to_string(version));
  Model m;
  m.voxel_res = static_cast<int>(read_u32(in));
  m.hit_cap = static_cast<int>(read_u32(in));
  m.n_levels = static_cast<int>(read_u32(in));
  m.f_dim = static_cast<int>(read_u32(in));
  m.table_size = read_u32(in);
  m.hidden = static_cast<int>(read_u32(in));
  m.n_mat = static_cast<int>(read_u32(in));
  if (m.voxel_res < 2 || m.voxel_res > 256 || (m.voxel_res & (m.voxel_res - 1)) != 0)
    throw std::invalid_argument("occupancy resolution must be a power of two in [2, 256]");
  m.occupancy.assign(static_cast<size_t>(m.voxel_res) * m.voxel_res * m.voxel_res / 8, 0);
  if (!in.read(reinterpret_cast<char*>(m.occupancy.data()),
               static_cast<std::streamsize>(m.occupancy.size())))
    throw std::runtime_error("model file truncated");
  for (int l = 0; l < m.n_levels; ++l) {
    m.level_res.push_back(static_cast<int>(read_u32(in)));
    std::vector<float> t(static_cast<size_t>(m.table_size) * m.f_dim);
    for (float& v : t) v = read_half(in);
    m.tables.push_back(std::move(t));
  }
  const int in_w = m.input_width();
  auto read_vec = [&](std::vector<float>& v, size_t n) {
    v.resize(n);
    for (float& x : v) x = read_half(in);
  };
  read_vec(m.w1, static_cast<size_t>(m.hidden) * in_w);
  read_vec(m.b1, static_cast<size_t>(m.hidden));
  read_vec(m.w2, static_cast<size_t>(m.hidden) * m.hidden);
  read_vec(m.b2, static_cast<size_t>(m.hidden));
  read_vec(m.w3, static_cast<size_t>(8 + m.n_mat) * m.hidden);
  read_vec(m.b3, static_cast<size_t>(8 + m.n_mat));
  const uint32_t mat_count = read_u32(in);
  m.materials.resize(mat_count);
  for (Material& mat : m.materials) {
    for (int c = 0; c < 3; ++c) mat.albedo[c] = read_f32(in);
    mat.kind = read_u32(in) == 1u ? 1u : 0u;
    mat.roughness = read_f32(in);
  }
  for (int c = 0; c < 3; ++c) m.aabb.mn[c] = read_f32(in);
  for (int c = 0; c < 3; ++c) m.aabb.mx[c] = read_f32(in);
  finalize_model(m);
  return m;
}

// -------------------------------------------------------------- narrow phase

// One (ray, object) query at identity object transform, as the reference
// pipeline performs it:
//  * pair emission: ray_aabb_intersect on the object-space ray with t_max = inf
//    against the frame box, kept iff enter < max_t (renderer.cpp:165-172;
//    max_t = ray.t_max for a scene with no triangle objects, 275, 314);
//  * narrow phase: to_local + d*inv_extent, DDA with (t_min, inf), encode,
//    infer (renderer.cpp:251-261);
//  * accept: closest-hit (renderer.cpp:281-284) or any-hit (317-320).
static HitRecord query_one(const Model& m, const Ray& ray, int mode, BoundaryHits& hits,
                           std::vector<float>& column) {
  HitRecord rec{};
  Ray oray = ray;
  oray.t_max = std::numeric_limits<float>::infinity();
  Interval iv;
  if (!ray_aabb_intersect(oray, m.aabb, &iv) || !(iv.enter < ray.t_max)) return rec;
  float inv_ext[3], lo[3], ld[3];
  for (int a = 0; a < 3; ++a) inv_ext[a] = 1.0f / (m.aabb.mx[a] - m.aabb.mn[a]);
  for (int a = 0; a < 3; ++a) {
    lo[a] = (ray.o[a] - m.aabb.mn[a]) * inv_ext[a];
    ld[a] = ray.d[a] * inv_ext[a];
  }
  collect_boundary_hits_local(lo, ld, ray.t_min, std::numeric_limits<float>::infinity(),
                              m.occupancy, m.voxel_res, m.hit_cap, hits);
  int pc = 0;
  encode_ray_into(m, hits, column.data(), nullptr, pc);
  const NeuralHit nh = infer_one(m, column.data(), iv);
  uint32_t flags = 1u;
  if (nh.occluded) {
    flags |= 2u;
    bool accept;
    if (mode == kClosest)
      accept = !(nh.t_world >= ray.t_max || nh.t_world < ray.t_min);
    else
      accept = nh.t_world >= ray.t_min && nh.t_world <= ray.t_max;
    if (accept) flags |= 4u;
  }
  rec.flags_material = flags | (static_cast<uint32_t>(nh.material_index) << 8);
  rec.t_world = nh.t_world;
  for (int k = 0; k < 3; ++k) {
    rec.normal[k] = nh.normal[k];
    rec.albedo[k] = nh.albedo[k];
  }
  return rec;
}

// parallel.hpp:18-37 slicing over contiguous ranges
void narrow_phase(const Model& m, const Ray* rays, int64_t n, int mode, HitRecord* out,
                  int workers) {
  if (workers < 1) {
    const unsigned hw = std::thread::hardware_concurrency();
    workers = hw > 0 ? static_cast<int>(hw) : 1;
  }
  auto run = [&](int64_t b, int64_t e) {
    BoundaryHits hits;
    std::vector<float> column(static_cast<size_t>(m.input_width()));
    for (int64_t i = b; i < e; ++i) out[i] = query_one(m, rays[i], mode, hits, column);
  };
  if (n <= 0) return;
  if (workers > n) workers = static_cast<int>(n);
  if (workers == 1) {
    run(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t chunk = (n + workers - 1) / workers;
  for (int w = 0; w < workers; ++w) {
    const int64_t b = w * chunk;
    const int64_t e = std::min<int64_t>(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&run, b, e] { run(b, e); });
  }
  for (auto& t : pool) t.join();
}

// ------------------------------------------------------ procedural meshes

static void mesh_finalize(ObjMesh& m) {  // shapes.cpp:10-14
  m.face_material.assign(m.faces.size() / 3, 0);
  m.n_mat = 1;
}

// shapes.cpp:18-58
ObjMesh make_uv_sphere(float radius, int segments, int rings) {
  const float kPi = 3.14159265358979323846f;
  ObjMesh m;
  auto push = [&](float x, float y, float z) { m.verts.insert(m.verts.end(), {x, y, z}); };
  push(0, radius, 0);
  for (int r = 1; r < rings; ++r) {
    const float phi = kPi * static_cast<float>(r) / static_cast<float>(rings);
    for (int s = 0; s < segments; ++s) {
      const float theta = 2.0f * kPi * static_cast<float>(s) / static_cast<float>(segments);
      push(radius * (std::sin(phi) * std::cos(theta)), radius * std::cos(phi),
           radius * (std::sin(phi) * std::sin(theta)));
    }
  }
  push(0, -radius, 0);
  const int south = static_cast<int>(m.verts.size() / 3) - 1;
  auto rv = [&](int r, int s) { return 1 + (r - 1) * segments + (s % segments); };
  auto face = [&](int a, int b, int c) { m.faces.insert(m.faces.end(), {a, b, c}); };
  for (int s = 0; s < segments; ++s) face(0, rv(1, s + 1), rv(1, s));
  for (int r = 1; r < rings - 1; ++r)
    for (int s = 0; s < segments; ++s) {
      const int a = rv(r, s), b = rv(r, s + 1), c = rv(r + 1, s), d = rv(r + 1, s + 1);
      face(a, b, d);
      face(a, d, c);
    }
  for (int s = 0; s < segments; ++s) face(south, rv(rings - 1, s), rv(rings - 1, s + 1));
  mesh_finalize(m);
  return m;
}

// shapes.cpp:60-87
ObjMesh make_box(const float h[3]) {
  ObjMesh m;
  const int axes[6][2] = {{1, 2}, {2, 0}, {0, 1}, {2, 1}, {0, 2}, {1, 0}};
  for (int face = 0; face < 6; ++face) {
    const int axis = face % 3;
    const float sign = face < 3 ? 1.0f : -1.0f;
    float n[3] = {0, 0, 0}, u[3] = {0, 0, 0}, v[3] = {0, 0, 0}, c[3];
    n[axis] = sign;
    u[axes[face][0]] = h[axes[face][0]];
    v[axes[face][1]] = h[axes[face][1]];
    for (int k = 0; k < 3; ++k) c[k] = n[k] * h[k];
    const int base = static_cast<int>(m.verts.size() / 3);
    for (int k = 0; k < 3; ++k) m.verts.push_back(c[k] - u[k] - v[k]);
    for (int k = 0; k < 3; ++k) m.verts.push_back(c[k] + u[k] - v[k]);
    for (int k = 0; k < 3; ++k) m.verts.push_back(c[k] + u[k] + v[k]);
    for (int k = 0; k < 3; ++k) m.verts.push_back(c[k] - u[k] + v[k]);
    m.faces.insert(m.faces.end(), {base, base + 1, base + 2, base, base + 2, base + 3});
  }
  mesh_finalize(m);
  return m;
}

// shapes.cpp:89-112
ObjMesh make_torus(float R, float r0, int segments, int rings) {
  const float kPi = 3.14159265358979323846f;
  ObjMesh m;
  for (int s = 0; s < segments; ++s) {
    const float theta = 2.0f * kPi * static_cast<float>(s) / static_cast<float>(segments);
    const float cx = R * std::cos(theta), cz = R * std::sin(theta);
    const float rx = std::cos(theta), rz = std::sin(theta);
    for (int r = 0; r < rings; ++r) {
      const float phi = 2.0f * kPi * static_cast<float>(r) / static_cast<float>(rings);
      const float nx = std::cos(phi) * rx, ny = std::sin(phi), nz = std::cos(phi) * rz;
      m.verts.insert(m.verts.end(), {cx + r0 * nx, r0 * ny, cz + r0 * nz});
    }
  }
  auto vid = [&](int s, int r) { return (s % segments) * rings + (r % rings); };
  for (int s = 0; s < segments; ++s)
    for (int r = 0; r < rings; ++r) {
      const int a = vid(s, r), b = vid(s + 1, r), c = vid(s + 1, r + 1), d = vid(s, r + 1);
      m.faces.insert(m.faces.end(), {a, b, c, a, c, d});
    }
  mesh_finalize(m);
  return m;
}

Model model_from_mesh(const ObjMesh& mesh, int V, int H, uint64_t seed) {
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
  return m;
}

// ----------------------------------------------------------- scene query

// object_space_ray (renderer.cpp:30-37): Eigen Affine3f * point = linear*p +
// translation with the product summed over the inner index in order.
static Ray object_space_ray(const float w2o[12], const Ray& r, float t_max) {
  Ray o;
  for (int i = 0; i < 3; ++i) {
    const float* L = w2o + 4 * i;
    o.o[i] = ((L[0] * r.o[0] + L[1] * r.o[1]) + L[2] * r.o[2]) + L[3];
    o.d[i] = (L[0] * r.d[0] + L[1] * r.d[1]) + L[2] * r.d[2];
  }
  o.t_min = r.t_min;
  o.t_max = t_max;
  return o;
}

void scene_query(const Instance* inst, int n_inst, const Ray* rays, int64_t n, int mode,
                 SceneHit* out, int workers) {
  const float inf = std::numeric_limits<float>::infinity();
  for (int64_t i = 0; i < n; ++i) {
    out[i] = SceneHit{};
    out[i].t = rays[i].t_max;  // best_t with no triangle objects (renderer.cpp:275, 314)
    out[i].object_index = -1;
  }
  // Pairs in stable object order (renderer.cpp:175-179): object-major loop.
  std::vector<Ray> oray;
  std::vector<int64_t> slot;
  std::vector<HitRecord> hits;
  for (int k = 0; k < n_inst; ++k) {
    const Model& m = *inst[k].model;
    oray.clear();
    slot.clear();
    for (int64_t i = 0; i < n; ++i) {
      // collect_pairs: interval on the unclipped object-space ray, kept iff
      // enter < max_t (renderer.cpp:165-172); max_t = t_max (no triangles)
      Ray o = object_space_ray(inst[k].w2o, rays[i], inf);
      Interval iv;
      if (!ray_aabb_intersect(o, m.aabb, &iv) || !(iv.enter < rays[i].t_max)) continue;
      o.t_max = rays[i].t_max;  // carries the pair gate into narrow_phase
      oray.push_back(o);
      slot.push_back(i);
    }
    hits.assign(oray.size(), HitRecord{});
    narrow_phase(m, oray.data(), static_cast<int64_t>(oray.size()), mode, hits.data(), workers);
    for (size_t p = 0; p < oray.size(); ++p) {
      const HitRecord& h = hits[p];
      if (!(h.flags_material & 2u)) continue;  // !nh.occluded
      const Ray& ray = rays[slot[p]];
      SceneHit& sh = out[slot[p]];
      const float t = h.t_world;
      if (mode == kClosest) {
        if (t >= sh.t || t < ray.t_min) continue;  // renderer.cpp:284
        sh.t = t;
        for (int a = 0; a < 3; ++a) sh.position[a] = ray.o[a] + t * ray.d[a];  // Ray::at
        const float* n0 = h.normal;
        float nw[3];
        if (n0[0] * n0[0] + n0[1] * n0[1] + n0[2] * n0[2] == 0.0f) {
          for (int a = 0; a < 3; ++a) nw[a] = -ray.d[a];
        } else {  // normal_to_world: (W2O.linear^T n).normalized()
          const float* L = inst[k].w2o;
          for (int a = 0; a < 3; ++a) nw[a] = (L[a] * n0[0] + L[4 + a] * n0[1]) + L[8 + a] * n0[2];
          const float len = std::sqrt((nw[0] * nw[0] + nw[1] * nw[1]) + nw[2] * nw[2]);
          if (len > 0.0f)
            for (int a = 0; a < 3; ++a) nw[a] = nw[a] / len;
        }
        if ((nw[0] * ray.d[0] + nw[1] * ray.d[1]) + nw[2] * ray.d[2] > 0.0f)
          for (int a = 0; a < 3; ++a) nw[a] = -nw[a];
        for (int a = 0; a < 3; ++a) {
          sh.normal[a] = nw[a];
          sh.albedo[a] = h.albedo[a];
        }
        const int mat = std::clamp(static_cast<int>(h.flags_material >> 8), 0,
                                   static_cast<int>(m.materials.size()) - 1);
        sh.kind = m.materials[static_cast<size_t>(mat)].kind;
        sh.roughness = m.materials[static_cast<size_t>(mat)].roughness;
        sh.object_index = k;
        sh.flags = 1u;
      } else if (t >= ray.t_min && t <= ray.t_max) {  // renderer.cpp:319
        sh.flags = 1u;
        if (sh.object_index < 0) sh.object_index = k;
      }
    }
  }
}

}  // namespace oracle
