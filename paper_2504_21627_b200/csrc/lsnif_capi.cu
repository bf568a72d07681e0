// C ABI of liblsnif_gpu (include/lsnif_gpu.h): model ingest and device
// residency, per-stream scratch, query orchestration, host staging.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "lsnif_gpu.h"
#include "lsnif_internal.hpp"

using lsnif_dev::DevModel;
using lsnif_dev::RowMeta;
using lsnif_dev::kTileM;

namespace {

thread_local std::string g_err;

using lsnif_api::ApiError;
using lsnif_api::ck;
using lsnif_api::fail;

// Every entry point restores the caller's current device on return (the
// body switches to the model's / scene's device).
struct DeviceRestore {
  int dev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  }
  ~DeviceRestore() {
    if (dev >= 0) cudaSetDevice(dev);
  }
};

template <typename F>
lsnif_status guarded(F&& f) {
  DeviceRestore restore;
  try {
    f();
    return LSNIF_OK;
  } catch (const ApiError& e) {
    g_err = e.msg;
    return e.st;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return LSNIF_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LSNIF_RUNTIME_ERROR;
  }
}

// ------------------------------------------------------------ fp16 decode
float half_bits_to_float(uint16_t h) {  // IEEE binary16 -> fp32 (exact)
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
  float f;
  std::memcpy(&f, &x, 4);
  return f;
}


// ------------------------------------------------------------- workspace
struct Workspace {
  uint8_t* X = nullptr;
  size_t x_tiles = 0;
  int64_t chunk = 0;  // rays per trace/MLP launch pair (pick_chunk)
  RowMeta* meta = nullptr;
  size_t meta_cap = 0;
  uint8_t* counters = nullptr;  // per chunk: u64 batch counter + one i32 row counter per K bin
  unsigned long long* stats = nullptr;
  int64_t last_rays = 0;
  // profiling: event pairs around each launch (kind 0 trace, 1 mlp). The
  // query thread appends and lsnif_profile_read (any thread) drains them:
  // both hold prof_mu.
  std::mutex prof_mu;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  uint64_t launches[2] = {0, 0};
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
  }
  ~Workspace() {
    for (auto& u : ev_used) {
      cudaEventDestroy(u.second.first);
      cudaEventDestroy(u.second.second);
    }
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    cudaFree(X);
    cudaFree(meta);
    cudaFree(stats);
  }
};

// Host staging for lsnif_query_host: kSlots device buffers, each with its own
// stream, so the H2D copy engine, the kernels and the D2H copy engine work on
// different chunks at once (PCIe-bound; copies of a slot are stream-ordered).
constexpr int kSlots = 4;
template <typename Hit>
struct HostStagingT {
  cudaStream_t streams[kSlots] = {};
  lsnif_ray* d_rays[kSlots] = {};
  Hit* d_hits[kSlots] = {};
  int64_t cap = 0;
  ~HostStagingT() {
    for (int i = 0; i < kSlots; ++i) {
      cudaFree(d_rays[i]);
      cudaFree(d_hits[i]);
      if (streams[i]) cudaStreamDestroy(streams[i]);
    }
  }
};
using HostStaging = HostStagingT<lsnif_hit>;

// Rays per trace/MLP launch pair, chosen per stream workspace (pick_chunk):
// fewer, longer launches amortise each launch's fixed costs (stop-mask fill,
// weight copy and TMEM allocation, both kernels' tails): C5 device rays/s at
// 2^21 / 2^22 / 2^23 / 2^24 / 2^25 = 5.65 / 5.97 / 6.15 / 6.25 / 6.29 e9. The
// workspace grows with the launch (per-bin X regions sized for every row:
// ~9.4 GB at 2^23 rows, ~18.8 GB at 2^24, only for queries that large).
// LSNIF_CHUNK_LOG2 (read once) fixes the size.
inline int64_t chunk_override() {
  static const int64_t c = [] {
    const char* e = std::getenv("LSNIF_CHUNK_LOG2");
    if (!e) return int64_t(0);
    const int l = std::atoi(e);
    return int64_t(1) << (l < 16 ? 16 : (l > 25 ? 25 : l));
  }();
  return c;
}
// Largest host staging step in rays (LSNIF_HOST_CHUNK overrides); a call is
// cut into ~8 steps of at least 64K rays up to this cap. Larger steps cut the
// per-copy overhead of big calls: C5 e2e 1.44e9 -> 1.63e9 rays/s, C3 1.44 ->
// 1.51e9, C2 1.18 -> 1.29e9 with a 2^21 cap instead of 2^17 (2^22: no better).
constexpr int64_t kHostChunk = int64_t(1) << 21;

int64_t host_chunk(int64_t dflt = kHostChunk) {
  const char* e = std::getenv("LSNIF_HOST_CHUNK");
  const long long v = e ? std::atoll(e) : 0;
  return v >= 1024 ? static_cast<int64_t>(v) : dflt;
}
// Chunked host round trip through kSlots staging slots: per chunk H2D of
// the rays, query(d_rays, n, d_hits, stream), D2H of the results, each slot
// on its own stream so the copy engines and the kernels overlap. The slots
// are ordered after prior work on the caller's stream; returns when the
// results are in host memory.
// `chunk` = rays per staging step (LSNIF_HOST_CHUNK overrides).
template <typename Hit, typename Query>
void host_round_trip(std::unique_ptr<HostStagingT<Hit>>& staging, int64_t chunk, const lsnif_ray* h_rays,
                     int64_t n, Hit* h_hits, cudaStream_t stream, Query&& query) {
  if (!staging) {
    auto s = std::make_unique<HostStagingT<Hit>>();
    const int64_t cap = host_chunk(chunk);
    for (int i = 0; i < kSlots; ++i) {
      ck(cudaStreamCreateWithFlags(&s->streams[i], cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaMalloc(&s->d_rays[i], cap * sizeof(lsnif_ray)), "cudaMalloc(staging)");
      ck(cudaMalloc(&s->d_hits[i], cap * sizeof(Hit)), "cudaMalloc(staging)");
    }
    s->cap = cap;
    staging = std::move(s);
  }
  HostStagingT<Hit>& S = *staging;
  cudaEvent_t ev;
  ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  struct EventGuard {
    cudaEvent_t e;
    ~EventGuard() { cudaEventDestroy(e); }
  } guard{ev};
  ck(cudaEventRecord(ev, stream), "cudaEventRecord");
  for (int i = 0; i < kSlots; ++i) ck(cudaStreamWaitEvent(S.streams[i], ev, 0), "cudaStreamWaitEvent");
  // ~8 chunks per call so the H2D of one chunk, the kernels of the previous
  // and the D2H of the one before overlap, but no chunk below 64K rays: a
  // query launch pair has ~40 us of fixed latency (C2 shadow call, 116k rays:
  // 16K-ray chunks 0.27 ms, 64K 0.19 ms; scripts/e2e_min.sh).
  static const int64_t min_step = [] {
    const char* e = std::getenv("LSNIF_HOST_MIN_CHUNK");  // A/B probe
    return e ? std::max<int64_t>(1024, std::atoll(e)) : int64_t(65536);
  }();
  const int64_t step = std::min(S.cap, std::max<int64_t>(min_step, ((n + 7) / 8 + 1023) / 1024 * 1024));
  int64_t k = 0;
  for (int64_t s = 0; s < n; s += step, ++k) {
    const int slot = static_cast<int>(k % kSlots);
    const int64_t cn = std::min(step, n - s);
    cudaStream_t st = S.streams[slot];
    ck(cudaMemcpyAsync(S.d_rays[slot], h_rays + s, cn * sizeof(lsnif_ray), cudaMemcpyHostToDevice, st),
       "cudaMemcpyAsync(H2D)");
    query(S.d_rays[slot], cn, S.d_hits[slot], st);
    ck(cudaMemcpyAsync(h_hits + s, S.d_hits[slot], cn * sizeof(Hit), cudaMemcpyDeviceToHost, st),
       "cudaMemcpyAsync(D2H)");
  }
  for (int i = 0; i < kSlots; ++i) ck(cudaStreamSynchronize(S.streams[i]), "cudaStreamSynchronize");
}

constexpr size_t kMaxChunks = 1024;                // chunks per query (>= 2^31 rays / 2^21)
// Counter block, zeroed by one memset per query (only the chunks it uses):
// 4 x u64 stats, then per chunk {u64 batch counter, i32 row counter per K bin}.
constexpr size_t kStatsBytes = 32;
constexpr size_t kChunkCounterBytes = 8 + 4 * lsnif_dev::kMaxBins + 8;  // 80 B
constexpr size_t kCounterBytes = kStatsBytes + kChunkCounterBytes * kMaxChunks;

}  // namespace

struct lsnif_model_s {
  int device = 0;
  int num_sms = 148;
  DevModel dm{};
  lsnif_model_info info{};
  std::vector<void*> allocations;
  std::mutex mu;
  std::map<cudaStream_t, std::unique_ptr<Workspace>> ws;
  std::unique_ptr<HostStaging> staging;
  std::unique_ptr<HostStagingT<lsnif_hit_wire>> staging_wire;
  std::mutex staging_mu;
  std::atomic<bool> profiling{false};

  ~lsnif_model_s() {
    cudaSetDevice(device);
    ws.clear();
    staging.reset();
    staging_wire.reset();
    for (void* p : allocations) cudaFree(p);
  }

  template <typename T>
  T* upload(const void* src, size_t bytes) {
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes), "cudaMalloc(model)");
    allocations.push_back(p);
    ck(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy(model)");
    info.device_bytes += bytes;
    return static_cast<T*>(p);
  }

  // Workspace bytes for launches of `rows` rays (X regions + row meta).
  size_t workspace_bytes(int64_t rows) const {
    const int64_t tiles = (rows + kTileM - 1) / kTileM;
    return lsnif_dev::bin_x_offset(dm.n_bins, tiles) + static_cast<size_t>(dm.n_bins) * tiles * kTileM * sizeof(RowMeta);
  }
  // 2^24-ray launches while their workspace is at most a quarter of the free
  // HBM (decided once per stream), else 2^23.
  int64_t pick_chunk() const {
    if (const int64_t c = chunk_override()) return c;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return int64_t(1) << 23;
    return workspace_bytes(int64_t(1) << 24) * 4 <= free_b ? int64_t(1) << 24 : int64_t(1) << 23;
  }

  Workspace& workspace(cudaStream_t st, int64_t n) {
    std::lock_guard<std::mutex> lock(mu);
    auto& slot = ws[st];
    if (!slot) {
      slot = std::make_unique<Workspace>();
      // one allocation, reset by a single memset per query
      ck(cudaMalloc(&slot->stats, kCounterBytes), "cudaMalloc(counters)");
      slot->counters = reinterpret_cast<uint8_t*>(slot->stats) + kStatsBytes;
      slot->chunk = pick_chunk();
    }
    Workspace& w = *slot;
    // X / meta: one region per K bin, each able to hold every row of a chunk
    for (;;) {
      const int64_t rows = std::min<int64_t>(n, w.chunk);
      const size_t tiles = static_cast<size_t>((rows + kTileM - 1) / kTileM);
      if (tiles <= w.x_tiles) break;
      cudaFree(w.X);
      cudaFree(w.meta);
      w.X = nullptr;
      w.meta = nullptr;
      w.x_tiles = 0;
      cudaError_t e = cudaMalloc(&w.X, lsnif_dev::bin_x_offset(dm.n_bins, static_cast<int64_t>(tiles)));
      if (e == cudaSuccess)
        e = cudaMalloc(&w.meta, static_cast<size_t>(dm.n_bins) * tiles * kTileM * sizeof(RowMeta));
      if (e == cudaSuccess) {
        w.x_tiles = tiles;
        break;
      }
      cudaFree(w.X);
      w.X = nullptr;
      w.meta = nullptr;
      (void)cudaGetLastError();  // allocation failures are not sticky
      if (e == cudaErrorMemoryAllocation && w.chunk > (int64_t(1) << 23) && !chunk_override()) {
        w.chunk = int64_t(1) << 23;  // memory got tighter since pick_chunk: smaller launches
        continue;
      }
      ck(e, "cudaMalloc(query workspace)");
    }
    return w;
  }
};

namespace {

// Builds the device model from a host description (model_io.hpp:18-36).
void build_model(lsnif_model_s& M, const lsnif_model_desc& d) {
  const int V = d.voxel_res, H = d.hit_cap, L = d.n_levels, F = d.f_dim, hid = d.hidden;
  if (V < 2 || V > 256 || (V & (V - 1)) != 0)
    fail(LSNIF_INVALID_ARGUMENT, "occupancy resolution must be a power of two in [2, 256]");
  if (H < 1) fail(LSNIF_INVALID_ARGUMENT, "hit cap must be >= 1");
  if (L < 1) fail(LSNIF_INVALID_ARGUMENT, "need at least one grid level");
  if (d.n_mat < 1) fail(LSNIF_INVALID_ARGUMENT, "n_mat must be >= 1");
  if (d.table_size < 1) fail(LSNIF_INVALID_ARGUMENT, "table size must be >= 1");
  for (int l = 0; l < L; ++l)
    if (d.level_res[l] % V != 0)
      fail(LSNIF_INVALID_ARGUMENT, "level resolution must be a multiple of the voxel resolution");
  // Fast-path envelope of this build.
  if (V > 64) fail(LSNIF_UNSUPPORTED, "voxel resolution > 64 is not supported by the GPU path");
  if (H > lsnif_dev::kMaxHitCap) fail(LSNIF_UNSUPPORTED, "hit cap > 32 is not supported");
  if (L > lsnif_dev::kMaxLevels || F > 4 || L * F > 16)
    fail(LSNIF_UNSUPPORTED, "need n_levels <= 4, f_dim <= 4, n_levels * f_dim <= 16");
  if (hid != 128 && hid != 64)
    fail(LSNIF_UNSUPPORTED, "hidden width must be 128 or 64 (the paper's high- / low-quality LSNIF)");
  const int n_out = 8 + d.n_mat;
  if (n_out > 16) fail(LSNIF_UNSUPPORTED, "n_mat > 8 is not supported");
  const int K1 = H * L * F;
  const int K1P = (K1 + 15) / 16 * 16;

  if (K1P / 16 > lsnif_dev::kMaxBins) fail(LSNIF_UNSUPPORTED, "input width H*L*F must be <= 256");

  DevModel& m = M.dm;
  m = DevModel{};
  for (int a = 0; a < 3; ++a) {
    m.mn[a] = d.aabb[a];
    m.mx[a] = d.aabb[3 + a];
    m.inv_ext[a] = 1.0f / (m.mx[a] - m.mn[a]);  // model_io.hpp:33 cwiseInverse
  }
  m.V = V;
  m.fres = static_cast<float>(V);
  m.inv_fres = 1.0f / static_cast<float>(V);
  m.H = H;
  m.L = L;
  m.F = F;
  m.LF = L * F;
  m.K1 = K1;
  m.K1P = K1P;
  m.n_bins = K1P / 16;
  m.M = d.table_size;
  m.M_pow2 = (d.table_size & (d.table_size - 1)) == 0;
  m.M_mask = d.table_size - 1;
  for (int l = 0; l < L; ++l) m.level_res[l] = d.level_res[l];
  m.hidden = hid;
  m.n_out = n_out;
  m.n_mat = d.n_mat;
  m.N3 = 16;

  // occupancy bitset as 32-bit words (same bit order as the byte stream)
  const size_t occ_bytes = static_cast<size_t>(V) * V * V / 8;
  std::vector<uint32_t> occ((occ_bytes + 3) / 4, 0u);
  std::memcpy(occ.data(), d.occupancy, occ_bytes);
  m.occ = M.upload<uint32_t>(occ.data(), occ.size() * 4);
  // padded stop mask: occupied cells + the border one cell outside the grid
  {
    const int Vp = V + 2;
    const size_t nbits = static_cast<size_t>(Vp) * Vp * Vp;
    std::vector<uint32_t> stop((nbits + 31) / 32, 0u);
    // the same cells as 2-bit codes (0 free, 1 occupied, 2 border) for the
    // query kernel, whose walk tells an occupied cell from the border
    std::vector<uint32_t> stop2((nbits + 15) / 16, 0u);
    for (int z = 0; z < Vp; ++z)
      for (int y = 0; y < Vp; ++y)
        for (int x = 0; x < Vp; ++x) {
          const bool inside = x >= 1 && x <= V && y >= 1 && y <= V && z >= 1 && z <= V;
          uint32_t code = 2u;
          if (inside) {
            const size_t i = static_cast<size_t>(x - 1) + static_cast<size_t>(V) *
                             (static_cast<size_t>(y - 1) + static_cast<size_t>(V) * (z - 1));
            code = (d.occupancy[i >> 3] >> (i & 7)) & 1u;
          }
          const size_t j = static_cast<size_t>(x) + static_cast<size_t>(Vp) * (y + static_cast<size_t>(Vp) * z);
          if (code) stop[j >> 5] |= 1u << (j & 31);
          stop2[j >> 4] |= code << ((j & 15) * 2);
        }
    m.stop = M.upload<uint32_t>(stop.data(), stop.size() * 4);
    m.stop_words = static_cast<int>(stop.size());
    m.stop2 = M.upload<uint32_t>(stop2.data(), stop2.size() * 4);
    m.stop2_words = static_cast<int>(stop2.size());
  }

  // hash tables: 4 binary16 per entry (8 B, one load per corner)
  float xmax = 0.0f;
  for (int l = 0; l < L; ++l) {
    std::vector<uint16_t> t(static_cast<size_t>(d.table_size) * 4, 0);
    for (uint32_t e = 0; e < d.table_size; ++e)
      for (int f = 0; f < F; ++f) {
        const uint16_t h = d.tables[l][static_cast<size_t>(e) * F + f];
        t[static_cast<size_t>(e) * 4 + f] = h;
        xmax = std::max(xmax, std::fabs(half_bits_to_float(h)));
      }
    m.tables[l] = M.upload<uint2>(t.data(), t.size() * 2);
  }

  // decoded fp32 weights (row-major) for the fp32 infer_batch kernel + bounds
  auto dec = [](const uint16_t* src, size_t n) {
    std::vector<float> v(n);
    for (size_t i = 0; i < n; ++i) v[i] = half_bits_to_float(src[i]);
    return v;
  };
  const std::vector<float> w1 = dec(d.w1, static_cast<size_t>(hid) * K1), b1 = dec(d.b1, hid);
  const std::vector<float> w2 = dec(d.w2, static_cast<size_t>(hid) * hid), b2 = dec(d.b2, hid);
  const std::vector<float> w3 = dec(d.w3, static_cast<size_t>(n_out) * hid), b3 = dec(d.b3, n_out);
  {
    std::vector<float> all;
    for (const auto* v : {&w1, &b1, &w2, &b2, &w3, &b3}) all.insert(all.end(), v->begin(), v->end());
    m.w_f32 = M.upload<float>(all.data(), all.size() * 4);
  }

  // Activation scale: a power of two s with s * |activation| <= 2^14 for
  // every fp16 operand, from rigorous bounds (|feature| <= max|entry|,
  // |z_i| <= sum_j |W_ij| * bound + |b_i|).
  auto layer_bound = [](const std::vector<float>& w, const std::vector<float>& b, int rows, int cols,
                        double in_bound) {
    double mx = 0.0;
    for (int i = 0; i < rows; ++i) {
      double s = std::fabs(b[static_cast<size_t>(i)]);
      for (int j = 0; j < cols; ++j) s += std::fabs(w[static_cast<size_t>(i) * cols + j]) * in_bound;
      mx = std::max(mx, s);
    }
    return mx;
  };
  const double B1 = layer_bound(w1, b1, hid, K1, xmax);
  const double B2 = layer_bound(w2, b2, hid, hid, B1);
  const double B3 = layer_bound(w3, b3, n_out, hid, B2);
  const double bmax = std::max({static_cast<double>(xmax), B1, B2, B3, 1e-30});
  int e = static_cast<int>(std::floor(std::log2(16384.0 / bmax)));
  e = std::max(-14, std::min(15, e));
  m.act_scale = std::ldexp(1.0f, e);
  m.inv_act_scale = std::ldexp(1.0f, -e);
  m.feat_bound = xmax;
  M.info.activation_scale = m.act_scale;

  // UMMA canonical fp16 operands with the bias folded in as column K:
  //   W1: hid x (K1P+16) (col K1P = b1), W2: hid x (hid+16) (col hid = b2),
  //   W3: 16 x hid (rows >= n_out zero).
  const int K2 = hid + 16;
  auto canon = [&](int rows, int cols, auto&& get) {
    std::vector<uint8_t> buf(static_cast<size_t>(rows) * cols * 2, 0);
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c) {
        const uint16_t h = get(r, c);
        std::memcpy(buf.data() + lsnif_dev::canon_offset(r, c, rows), &h, 2);
      }
    return buf;
  };
  // W1's bias lives in its own trailing 16-column slab (column K1P = b1),
  // multiplied by a constant A slab, so an X tile can stop at its K bin
  const auto c1 = canon(hid, K1P + 16, [&](int r, int c) -> uint16_t {
    if (c < K1) return d.w1[static_cast<size_t>(r) * K1 + c];
    return c == K1P ? d.b1[r] : uint16_t(0);
  });
  const auto c2 = canon(hid, K2, [&](int r, int c) -> uint16_t {
    if (c < hid) return d.w2[static_cast<size_t>(r) * hid + c];
    return c == hid ? d.b2[r] : uint16_t(0);
  });
  // W3 has no bias column: b3 is added in fp32 by the decode epilogue (an
  // N = 16 MMA K-step costs ~50 cycles, as much as most of a layer's work)
  const auto c3 = canon(16, hid, [&](int r, int c) -> uint16_t {
    if (r >= n_out) return 0;
    return d.w3[static_cast<size_t>(r) * hid + c];
  });
  for (int i = 0; i < 16; ++i) m.b3[i] = i < n_out ? b3[i] : 0.0f;
  std::vector<uint8_t> wc;
  wc.insert(wc.end(), c1.begin(), c1.end());
  wc.insert(wc.end(), c2.begin(), c2.end());
  wc.insert(wc.end(), c3.begin(), c3.end());
  m.w_canon = M.upload<uint8_t>(wc.data(), wc.size());
  m.w1_bytes = static_cast<uint32_t>(c1.size());
  m.w2_bytes = static_cast<uint32_t>(c2.size());
  m.w3_bytes = static_cast<uint32_t>(c3.size());
  {  // X-tile ring depth: the deepest that fits the per-block SMEM opt-in limit
    int dev = 0, optin = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "cudaDeviceGetAttribute");
    m.x_stages = lsnif_dev::mlp_x_stages(m, static_cast<size_t>(optin));
    if (m.x_stages == 0)
      fail(LSNIF_UNSUPPORTED, "input width H*L*F too large for the MLP kernel's shared memory at this hidden "
                              "width (weights + two X tiles must fit one SM)");
  }

  // Logits of the all-zero input (rays without boundary points), fp32 with
  // the reference's sequential order (renderer.cpp:197-207).
  {
    std::vector<float> h1(hid), h2(hid);
    for (int i = 0; i < hid; ++i) {
      float s = 0.0f;
      for (int j = 0; j < K1; ++j) s += w1[static_cast<size_t>(i) * K1 + j] * 0.0f;
      s = s + b1[i];
      h1[i] = s < 0.0f ? s * 0.01f : s;
    }
    for (int i = 0; i < hid; ++i) {
      float s = 0.0f;
      for (int j = 0; j < hid; ++j) {
        const float p = w2[static_cast<size_t>(i) * hid + j] * h1[j];
        s = s + p;
      }
      s = s + b2[i];
      h2[i] = s < 0.0f ? s * 0.01f : s;
    }
    for (int i = 0; i < n_out; ++i) {
      float s = 0.0f;
      for (int j = 0; j < hid; ++j) {
        const float p = w3[static_cast<size_t>(i) * hid + j] * h2[j];
        s = s + p;
      }
      m.z_zero[i] = s + b3[i];
    }
  }

  // Occlusion boundary: smallest float z with 1/(1+expf(-z)) > 0.5, found by
  // bisection over the ordered bit patterns of [0, 1].
  {
    auto occ = [](float z) { return 1.0f / (1.0f + std::exp(-z)) > 0.5f; };
    uint32_t lo = 0u, hi = 0x3f800000u;  // occ(0) false, occ(1) true
    while (hi - lo > 1u) {
      const uint32_t mid = lo + (hi - lo) / 2;
      float z;
      std::memcpy(&z, &mid, 4);
      if (occ(z)) hi = mid; else lo = mid;
    }
    std::memcpy(&m.occ_threshold, &hi, 4);
  }

  {  // material table (model_io.cpp:159-164); one default entry if empty
    std::vector<lsnif_material> mats(d.materials, d.materials + std::max(d.n_materials, 0));
    if (mats.empty()) mats.push_back(lsnif_material{{0.7f, 0.7f, 0.7f}, 0u, 0.5f});
    m.materials = M.upload<lsnif_material>(mats.data(), mats.size() * sizeof(lsnif_material));
    m.n_materials = static_cast<int>(mats.size());
  }

  {  // constant heads of the all-zero input (rays with a pair but no point)
    lsnif_hit zh{};
    ck(lsnif_dev::compute_zero_hit(m, &zh), "zero_hit_kernel");
    m.zero_lt = zh.t_world;
    for (int a = 0; a < 3; ++a) {
      m.zero_normal[a] = zh.normal[a];
      m.zero_albedo[a] = zh.albedo[a];
    }
    m.zero_flags = zh.flags_material & ~static_cast<uint32_t>(LSNIF_HIT_PAIR | LSNIF_HIT_ACCEPTED);
  }

  M.info.device = M.device;
  M.info.voxel_res = V;
  M.info.hit_cap = H;
  M.info.n_levels = L;
  M.info.f_dim = F;
  M.info.table_size = d.table_size;
  M.info.hidden = hid;
  M.info.n_mat = d.n_mat;
  M.info.n_materials = d.n_materials;
  for (int l = 0; l < L && l < 4; ++l) M.info.level_res[l] = d.level_res[l];
  for (int a = 0; a < 6; ++a) M.info.aabb[a] = d.aabb[a];
}

// LSNF v1 reader (model_io.cpp:116-175): same checks and messages.
struct FileModel {
  lsnif_model_desc desc{};
  std::vector<uint8_t> occ;
  std::vector<int32_t> levels;
  std::vector<std::vector<uint16_t>> tables;
  std::vector<const uint16_t*> table_ptrs;
  std::vector<uint16_t> w1, b1, w2, b2, w3, b3;
  std::vector<lsnif_material> materials;
};

void read_model_file(const std::string& path, FileModel& fm) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(LSNIF_RUNTIME_ERROR, "cannot open model file: " + path);
  auto rd = [&](void* dst, size_t n) {
    if (!in.read(static_cast<char*>(dst), static_cast<std::streamsize>(n)))
      fail(LSNIF_RUNTIME_ERROR, "model file truncated");
  };
  auto u32 = [&]() {
    uint32_t v;
    rd(&v, 4);
    return v;
  };
  char magic[4];
  rd(magic, 4);
  if (std::memcmp(magic, "LSNF", 4) != 0)
    fail(LSNIF_RUNTIME_ERROR, "not an LSNIF model file (bad magic): " + path);
  const uint32_t version = u32();
  if (version != 1u) fail(LSNIF_RUNTIME_ERROR, "unsupported model version " + std::to_string(version));
  lsnif_model_desc& d = fm.desc;
  d.voxel_res = static_cast<int32_t>(u32());
  d.hit_cap = static_cast<int32_t>(u32());
  d.n_levels = static_cast<int32_t>(u32());
  d.f_dim = static_cast<int32_t>(u32());
  d.table_size = u32();
  d.hidden = static_cast<int32_t>(u32());
  d.n_mat = static_cast<int32_t>(u32());
  const int V = d.voxel_res;
  if (V < 2 || V > 256 || (V & (V - 1)) != 0)
    fail(LSNIF_INVALID_ARGUMENT, "occupancy resolution must be a power of two in [2, 256]");
  if (d.n_levels < 1 || d.n_levels > 64 || d.f_dim < 1 || d.f_dim > 64 || d.hidden < 1 ||
      d.hidden > 4096 || d.n_mat < 1 || d.n_mat > 4096 || d.hit_cap < 1 || d.hit_cap > 4096)
    fail(LSNIF_RUNTIME_ERROR, "model header out of range: " + path);
  fm.occ.resize(static_cast<size_t>(V) * V * V / 8);
  rd(fm.occ.data(), fm.occ.size());
  for (int l = 0; l < d.n_levels; ++l) {
    fm.levels.push_back(static_cast<int32_t>(u32()));
    std::vector<uint16_t> t(static_cast<size_t>(d.table_size) * d.f_dim);
    rd(t.data(), t.size() * 2);
    fm.tables.push_back(std::move(t));
  }
  const size_t K1 = static_cast<size_t>(d.hit_cap) * d.n_levels * d.f_dim;
  const size_t hid = static_cast<size_t>(d.hidden), no = 8 + static_cast<size_t>(d.n_mat);
  auto vec = [&](std::vector<uint16_t>& v, size_t n) {
    v.resize(n);
    rd(v.data(), n * 2);
  };
  vec(fm.w1, hid * K1);
  vec(fm.b1, hid);
  vec(fm.w2, hid * hid);
  vec(fm.b2, hid);
  vec(fm.w3, no * hid);
  vec(fm.b3, no);
  const uint32_t nm = u32();
  if (nm > 1u << 20) fail(LSNIF_RUNTIME_ERROR, "model file truncated");
  fm.materials.resize(nm);
  for (auto& mt : fm.materials) {
    rd(mt.albedo, 12);
    mt.kind = u32() == 1u ? 1u : 0u;
    rd(&mt.roughness, 4);
  }
  rd(d.aabb, 24);
  for (auto& t : fm.tables) fm.table_ptrs.push_back(t.data());
  d.occupancy = fm.occ.data();
  d.level_res = fm.levels.data();
  d.tables = fm.table_ptrs.data();
  d.w1 = fm.w1.data();
  d.b1 = fm.b1.data();
  d.w2 = fm.w2.data();
  d.b2 = fm.b2.data();
  d.w3 = fm.w3.data();
  d.b3 = fm.b3.data();
  d.materials = fm.materials.data();
  d.n_materials = static_cast<int32_t>(nm);
}

void check_model(lsnif_model m) {
  if (!m) fail(LSNIF_INVALID_ARGUMENT, "null model");
}

void create_into(const lsnif_model_desc& d, int device, lsnif_model* out) {
  if (!out) fail(LSNIF_INVALID_ARGUMENT, "null output handle");
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) fail(LSNIF_INVALID_ARGUMENT, "invalid device ordinal");
  ck(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop{};
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10)
    fail(LSNIF_UNSUPPORTED, std::string("liblsnif_gpu is built for sm_100a; device is ") + prop.name);
  auto M = std::make_unique<lsnif_model_s>();
  M->device = device;
  M->num_sms = prop.multiProcessorCount;
  build_model(*M, d);
  *out = M.release();
}

// n is the ray count, or its upper bound when n_dev (device-side count) is set.
// wire: d_hits holds lsnif_hit_wire records (16 B) instead of lsnif_hit.
void run_query(lsnif_model_s& M, const lsnif_ray* d_rays, int64_t n, int mode, void* d_hits,
               cudaStream_t st, const int32_t* n_dev = nullptr, const lsnif_interval* d_intervals = nullptr,
               bool wire = false) {
  if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative ray count");
  if (mode != LSNIF_QUERY_CLOSEST && mode != LSNIF_QUERY_ANY) fail(LSNIF_INVALID_ARGUMENT, "bad query mode");
  if (n > 0 && (!d_rays || !d_hits)) fail(LSNIF_INVALID_ARGUMENT, "null ray or hit pointer");
  if (n > INT32_MAX) fail(LSNIF_INVALID_ARGUMENT, "more than 2^31-1 rays in one call");
  ck(cudaSetDevice(M.device), "cudaSetDevice");
  Workspace& w = M.workspace(st, std::max<int64_t>(n, 1));
  const int64_t kChunk = w.chunk;
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  if (static_cast<size_t>(nchunks) > kMaxChunks) fail(LSNIF_INVALID_ARGUMENT, "too many rays in one call");
  ck(cudaMemsetAsync(w.stats, 0, kStatsBytes + kChunkCounterBytes * std::max<int64_t>(nchunks, 1), st),
     "cudaMemsetAsync");
  w.last_rays = n;
  for (int64_t s = 0, ci = 0; s < n; s += kChunk, ++ci) {
    const int64_t cn = std::min(kChunk, n - s);
    lsnif_dev::TraceParams tp{};
    tp.m = M.dm;
    tp.rays = d_rays + s;
    tp.intervals = d_intervals ? d_intervals + s : nullptr;
    tp.n = cn;
    tp.n_dev = n_dev;
    tp.offset = s;
    tp.mode = mode;
    const size_t rec = wire ? sizeof(lsnif_hit_wire) : sizeof(lsnif_hit);
    tp.out = static_cast<uint8_t*>(d_hits) + s * rec;
    tp.wire = wire ? 1 : 0;
    tp.X = w.X;
    tp.meta = w.meta;
    uint8_t* cc = w.counters + kChunkCounterBytes * ci;
    tp.batch_counter = reinterpret_cast<unsigned long long*>(cc);
    tp.row_counter = reinterpret_cast<int32_t*>(cc + 8);
    tp.cap_tiles = static_cast<int64_t>(w.x_tiles);
    tp.stats = w.stats;
    // one read of the flag per chunk; the event bookkeeping under prof_mu
    const bool prof = M.profiling.load(std::memory_order_relaxed);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto record = [&](cudaEvent_t& e) {
      std::lock_guard<std::mutex> lk(w.prof_mu);
      e = w.take_event();
      ck(cudaEventRecord(e, st), "cudaEventRecord");
    };
    auto finish = [&](int kind) {
      std::lock_guard<std::mutex> lk(w.prof_mu);
      ++w.launches[kind];
      if (prof) w.ev_used.push_back({kind, {e0, e1}});
    };
    if (prof) record(e0);
    ck(lsnif_dev::launch_trace(tp, false, st), "trace_encode_kernel");
    if (prof) record(e1);
    finish(0);
    lsnif_dev::MlpParams mp{};
    mp.m = M.dm;
    mp.X = w.X;
    mp.meta = w.meta;
    mp.row_counter = reinterpret_cast<int32_t*>(cc + 8);
    mp.cap_tiles = static_cast<int64_t>(w.x_tiles);
    mp.out = static_cast<uint8_t*>(d_hits) + s * rec;
    mp.wire = wire ? 1 : 0;
    mp.mode = mode;
    mp.n_dev = n_dev;
    mp.offset = s;

    if (prof) record(e0);
    ck(lsnif_dev::launch_mlp(mp, static_cast<int>((cn + kTileM - 1) / kTileM) + M.dm.n_bins, M.num_sms, st),
       "mlp_tc_kernel");
    if (prof) record(e1);
    finish(1);
  }
}

}  // namespace

struct lsnif_scene_s {
  int device = 0;
  std::vector<lsnif_model> models;
  std::vector<lsnif_dev::InstanceParams> inst;
  lsnif_dev::InstanceBox* boxes = nullptr;  // device: per-instance transform + frame box
  // Per-instance narrow phases run concurrently on side streams (fork/join
  // with events around them; the merges stay in object order on the caller's
  // stream). The enqueue section is serialised by side_mu.
  std::mutex side_mu;
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> side_done;
  cudaEvent_t fork = nullptr;
  struct Scratch {
    lsnif_ray* orays = nullptr;   // instance k's pairs at k * cap
    int32_t* slots = nullptr;
    lsnif_hit* hits = nullptr;    // instance k's results at k * cap
    int32_t* count = nullptr;     // per instance
    unsigned long long* best = nullptr;  // per ray: merge key (launch_merge_all)
    int64_t cap = 0;
    ~Scratch() {
      cudaFree(orays);
      cudaFree(slots);
      cudaFree(hits);
      cudaFree(count);
      cudaFree(best);
    }
  };
  std::mutex mu;
  std::map<cudaStream_t, std::unique_ptr<Scratch>> scratch;
  std::mutex render_mu;
  std::map<cudaStream_t, lsnif_pt::WorkspacePtr> render_ws;  // renderer path state per stream
  std::mutex staging_mu;
  std::unique_ptr<HostStagingT<lsnif_scene_hit>> staging;     // lsnif_scene_query_host

  ~lsnif_scene_s() {
    cudaSetDevice(device);
    staging.reset();
    scratch.clear();
    cudaFree(boxes);
    for (cudaStream_t x : side) cudaStreamDestroy(x);
    for (cudaEvent_t e : side_done) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
  }

  Scratch& get(cudaStream_t st, int64_t n) {
    std::lock_guard<std::mutex> lock(mu);
    auto& s = scratch[st];
    const size_t ni = std::max<size_t>(inst.size(), 1);
    if (!s) {
      s = std::make_unique<Scratch>();
      ck(cudaMalloc(&s->count, ni * sizeof(int32_t)), "cudaMalloc(scene count)");
    }
    if (n > s->cap) {
      cudaFree(s->orays);
      cudaFree(s->slots);
      cudaFree(s->hits);
      cudaFree(s->best);
      s->orays = nullptr;
      s->slots = nullptr;
      s->hits = nullptr;
      s->best = nullptr;
      ck(cudaMalloc(&s->orays, ni * n * sizeof(lsnif_ray)), "cudaMalloc(scene rays)");
      ck(cudaMalloc(&s->slots, ni * n * sizeof(int32_t)), "cudaMalloc(scene slots)");
      ck(cudaMalloc(&s->hits, ni * n * sizeof(lsnif_hit)), "cudaMalloc(scene hits)");
      ck(cudaMalloc(&s->best, n * sizeof(unsigned long long)), "cudaMalloc(scene merge keys)");
      s->cap = n;
    }
    return *s;
  }
};

namespace lsnif_api {

void scene_query_async(lsnif_scene scene, const lsnif_ray* d_rays, int64_t n, const int32_t* d_n, int mode,
                       lsnif_scene_hit* d_hits, cudaStream_t st) {
  if (!scene) fail(LSNIF_INVALID_ARGUMENT, "null scene");
  if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative ray count");
  if (mode != LSNIF_QUERY_CLOSEST && mode != LSNIF_QUERY_ANY) fail(LSNIF_INVALID_ARGUMENT, "bad query mode");
  if (n > 0 && (!d_rays || !d_hits)) fail(LSNIF_INVALID_ARGUMENT, "null ray or hit pointer");
  if (n > INT32_MAX) fail(LSNIF_INVALID_ARGUMENT, "more than 2^31-1 rays in one call");
  if (n == 0) return;
  ck(cudaSetDevice(scene->device), "cudaSetDevice");
  auto& S = scene->get(st, n);
  const int ni = static_cast<int>(scene->inst.size());
  if (ni == 0) {
    ck(lsnif_dev::launch_scene_init(d_rays, n, d_n, d_hits, st), "scene_init_kernel");
    return;
  }
  // one pass over the rays: scene hits initialised + every instance's pairs
  ck(cudaMemsetAsync(S.count, 0, ni * sizeof(int32_t), st), "cudaMemsetAsync");
  // fused merge (two launches) unless pair indices overflow its 32-bit key
  const bool fused = static_cast<uint64_t>(ni) * static_cast<uint64_t>(S.cap) < (uint64_t(1) << 32);
  ck(lsnif_dev::launch_broad_phase_all(scene->boxes, ni, d_rays, n, d_n, S.orays, S.slots, S.cap, S.count, d_hits,
                                       fused ? S.best : nullptr, st),
     "broad_phase_all_kernel");
  // narrow phases: independent per instance, concurrently on side streams
  constexpr int kMaxSide = 8;
  std::lock_guard<std::mutex> lock(scene->side_mu);
  const int nside = std::min(ni, kMaxSide);
  while (static_cast<int>(scene->side.size()) < nside) {
    cudaStream_t x;
    cudaEvent_t e;
    ck(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    scene->side.push_back(x);
    scene->side_done.push_back(e);
  }
  if (!scene->fork) ck(cudaEventCreateWithFlags(&scene->fork, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaEventRecord(scene->fork, st), "cudaEventRecord");
  for (int q = 0; q < nside; ++q) ck(cudaStreamWaitEvent(scene->side[q], scene->fork, 0), "cudaStreamWaitEvent");
  for (int k = 0; k < ni; ++k)
    run_query(*scene->models[k], S.orays + k * S.cap, n, mode, S.hits + k * S.cap, scene->side[k % nside],
              S.count + k);
  for (int q = 0; q < nside; ++q) {
    ck(cudaEventRecord(scene->side_done[q], scene->side[q]), "cudaEventRecord");
    ck(cudaStreamWaitEvent(st, scene->side_done[q], 0), "cudaStreamWaitEvent");
  }
  if (fused) {
    ck(lsnif_dev::launch_merge_all(scene->boxes, ni, d_rays, n, d_n, S.hits, S.slots, S.cap, S.count, mode, S.best,
                                   d_hits, st),
       "merge_all");
  } else {
    for (int k = 0; k < ni; ++k)  // merges in object order (renderer.cpp:175-179)
      ck(lsnif_dev::launch_merge(scene->models[k]->dm, scene->inst[k], d_rays, S.hits + k * S.cap,
                                 S.slots + k * S.cap, S.count + k, n, mode, d_hits, st),
         "merge_kernel");
  }
}

}  // namespace lsnif_api

extern "C" {

const char* lsnif_last_error(void) { return g_err.c_str(); }

lsnif_status lsnif_scene_create(const lsnif_instance* instances, int32_t n, lsnif_scene* out) {
  return guarded([&] {
    if (!out) fail(LSNIF_INVALID_ARGUMENT, "null output handle");
    if (n < 0 || (n > 0 && !instances)) fail(LSNIF_INVALID_ARGUMENT, "bad instance list");
    auto S = std::make_unique<lsnif_scene_s>();
    for (int32_t k = 0; k < n; ++k) {
      check_model(instances[k].model);
      if (k > 0 && instances[k].model->device != instances[0].model->device)
        fail(LSNIF_INVALID_ARGUMENT, "scene instances must share one device");
      lsnif_dev::InstanceParams ip{};
      std::memcpy(ip.w2o, instances[k].world_to_object, sizeof(ip.w2o));
      ip.index = k;
      S->models.push_back(instances[k].model);
      S->inst.push_back(ip);
    }
    S->device = n > 0 ? instances[0].model->device : 0;
    if (n > 0) {
      std::vector<lsnif_dev::InstanceBox> boxes(static_cast<size_t>(n));
      for (int32_t k = 0; k < n; ++k) {
        std::memcpy(boxes[k].w2o, instances[k].world_to_object, sizeof(boxes[k].w2o));
        for (int a = 0; a < 3; ++a) {
          boxes[k].mn[a] = instances[k].model->dm.mn[a];
          boxes[k].mx[a] = instances[k].model->dm.mx[a];
        }
        boxes[k].materials = instances[k].model->dm.materials;
        boxes[k].n_materials = instances[k].model->dm.n_materials;
      }
      ck(cudaSetDevice(S->device), "cudaSetDevice");
      ck(cudaMalloc(&S->boxes, boxes.size() * sizeof(lsnif_dev::InstanceBox)), "cudaMalloc(scene boxes)");
      ck(cudaMemcpy(S->boxes, boxes.data(), boxes.size() * sizeof(lsnif_dev::InstanceBox), cudaMemcpyHostToDevice),
         "cudaMemcpy(scene boxes)");
    }
    *out = S.release();
  });
}

lsnif_status lsnif_scene_destroy(lsnif_scene scene) {
  return guarded([&] { delete scene; });
}

lsnif_status lsnif_scene_query(lsnif_scene scene, const lsnif_ray* d_rays, int64_t n, int mode,
                               lsnif_scene_hit* d_hits, void* stream) {
  return guarded([&] {
    lsnif_api::scene_query_async(scene, d_rays, n, nullptr, mode, d_hits, static_cast<cudaStream_t>(stream));
  });
}

lsnif_status lsnif_scene_query_host(lsnif_scene scene, const lsnif_ray* h_rays, int64_t n, int mode,
                                    lsnif_scene_hit* h_hits, void* stream) {
  return guarded([&] {
    if (!scene) fail(LSNIF_INVALID_ARGUMENT, "null scene");
    if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative ray count");
    if (mode != LSNIF_QUERY_CLOSEST && mode != LSNIF_QUERY_ANY) fail(LSNIF_INVALID_ARGUMENT, "bad query mode");
    if (n > 0 && (!h_rays || !h_hits)) fail(LSNIF_INVALID_ARGUMENT, "null ray or hit pointer");
    if (n == 0) return;
    ck(cudaSetDevice(scene->device), "cudaSetDevice");
    std::lock_guard<std::mutex> lock(scene->staging_mu);
    // larger steps than the single-model path: a scene chunk is ~4 launches
    // per instance (scripts/scene_e2e_probe.py: C4 2^17 3.77 ms, 2^18 3.13 ms)
    host_round_trip(scene->staging, int64_t(1) << 18, h_rays, n, h_hits, static_cast<cudaStream_t>(stream),
                    [&](const lsnif_ray* r, int64_t cn, lsnif_scene_hit* h, cudaStream_t st) {
                      lsnif_api::scene_query_async(scene, r, cn, nullptr, mode, h, st);
                    });
  });
}

lsnif_status lsnif_render(lsnif_scene scene, const float* world_diag, int32_t n_instances,
                          const lsnif_camera* camera, const lsnif_light* lights, int32_t n_lights,
                          const float environment[3], const lsnif_render_config* config,
                          float* d_image, lsnif_render_stats* stats, void* stream) {
  return guarded([&] {
    if (!scene || !camera || !config) fail(LSNIF_INVALID_ARGUMENT, "null scene, camera or config");
    if (n_instances != static_cast<int32_t>(scene->inst.size()))
      fail(LSNIF_INVALID_ARGUMENT, "render: world_diag needs one entry per scene instance");
    if (n_instances > 0 && !world_diag) fail(LSNIF_INVALID_ARGUMENT, "render: null world_diag");
    ck(cudaSetDevice(scene->device), "cudaSetDevice");
    lsnif_pt::WorkspacePtr* ws = nullptr;
    {
      std::lock_guard<std::mutex> lock(scene->render_mu);
      ws = &scene->render_ws[static_cast<cudaStream_t>(stream)];
    }
    lsnif_pt::render(*ws, scene, world_diag, n_instances, *camera, lights, n_lights, environment, *config,
                     d_image, stats, static_cast<cudaStream_t>(stream));
  });
}

lsnif_status lsnif_render_debug_paths(const lsnif_camera* camera, const lsnif_render_config* config,
                                      int64_t first_path, int64_t n, lsnif_ray* d_rays,
                                      float* d_uniforms, int32_t k, void* stream) {
  return guarded([&] {
    if (!camera || !config) fail(LSNIF_INVALID_ARGUMENT, "null camera or config");
    lsnif_pt::debug_paths(*camera, *config, first_path, n, d_rays, d_uniforms, k,
                              static_cast<cudaStream_t>(stream));
  });
}

struct lsnif_trainer_s {
  int device = 0;
  void* impl = nullptr;
  ~lsnif_trainer_s() {
    if (impl) lsnif_api::trainer_destroy(impl);
  }
};

lsnif_status lsnif_trainer_create(const lsnif_model_desc* init, const lsnif_mesh_desc* mesh,
                                  const lsnif_train_config* config, int device, lsnif_trainer* out) {
  return guarded([&] {
    if (!init || !mesh || !config || !out) fail(LSNIF_INVALID_ARGUMENT, "null trainer argument");
    lsnif_model geo = nullptr;
    create_into(*init, device, &geo);  // validates the model, builds the stop mask / frame constants
    auto T = std::make_unique<lsnif_trainer_s>();
    T->device = device;
    try {
      T->impl = lsnif_api::trainer_create(*init, *mesh, *config, device, geo, geo->dm);
    } catch (...) {
      lsnif_model_destroy(geo);
      throw;
    }
    *out = T.release();
  });
}

lsnif_status lsnif_trainer_create_from_file(const char* path, const lsnif_mesh_desc* mesh,
                                            const lsnif_train_config* config, int device, lsnif_trainer* out) {
  FileModel fm;
  const lsnif_status st = guarded([&] {
    if (!path) fail(LSNIF_INVALID_ARGUMENT, "null path");
    read_model_file(path, fm);
  });
  if (st != LSNIF_OK) return st;
  return lsnif_trainer_create(&fm.desc, mesh, config, device, out);
}

lsnif_status lsnif_trainer_destroy(lsnif_trainer trainer) {
  return guarded([&] { delete trainer; });
}

lsnif_status lsnif_trainer_step(lsnif_trainer trainer, int32_t steps, lsnif_train_loss* last, void* stream) {
  return guarded([&] {
    if (!trainer) fail(LSNIF_INVALID_ARGUMENT, "null trainer");
    lsnif_api::trainer_step(trainer->impl, steps, last, static_cast<cudaStream_t>(stream));
  });
}

lsnif_status lsnif_trainer_export(lsnif_trainer trainer, lsnif_model* out) {
  return guarded([&] {
    if (!trainer || !out) fail(LSNIF_INVALID_ARGUMENT, "null trainer or output");
    lsnif_api::trainer_export(trainer->impl, trainer->device, out);
  });
}

lsnif_status lsnif_trainer_batch_grad(lsnif_trainer trainer, const lsnif_ray* d_rays,
                                      const lsnif_train_target* d_targets, int64_t n, lsnif_train_loss* loss,
                                      float* d_grad_mlp, float* d_grad_tables, void* stream) {
  return guarded([&] {
    if (!trainer) fail(LSNIF_INVALID_ARGUMENT, "null trainer");
    lsnif_api::trainer_batch_grad(trainer->impl, d_rays, d_targets, n, loss, d_grad_mlp, d_grad_tables,
                                  static_cast<cudaStream_t>(stream));
  });
}

lsnif_status lsnif_trainer_sample(lsnif_trainer trainer, int64_t step, int64_t n, lsnif_ray* d_rays,
                                  lsnif_train_target* d_targets, void* stream) {
  return guarded([&] {
    if (!trainer) fail(LSNIF_INVALID_ARGUMENT, "null trainer");
    lsnif_api::trainer_sample(trainer->impl, step, n, d_rays, d_targets, static_cast<cudaStream_t>(stream));
  });
}

const char* lsnif_build_info(void) {
  return "liblsnif_gpu sm_100a: trace_encode_kernel + mlp_tc_kernel (tcgen05 kind::f16, TMEM), "
         "infer_f32_kernel; wavefront renderer (camera/shade/shadow_accum/resolve kernels)";
}

lsnif_status lsnif_model_create(const lsnif_model_desc* desc, int device, lsnif_model* out) {
  return guarded([&] {
    if (!desc) fail(LSNIF_INVALID_ARGUMENT, "null model description");
    create_into(*desc, device, out);
  });
}

lsnif_status lsnif_model_load(const char* path, int device, lsnif_model* out) {
  return guarded([&] {
    if (!path) fail(LSNIF_INVALID_ARGUMENT, "null path");
    FileModel fm;
    read_model_file(path, fm);
    create_into(fm.desc, device, out);
  });
}

lsnif_status lsnif_model_destroy(lsnif_model model) {
  return guarded([&] { delete model; });
}

lsnif_status lsnif_model_get_info(lsnif_model model, lsnif_model_info* out) {
  return guarded([&] {
    check_model(model);
    if (!out) fail(LSNIF_INVALID_ARGUMENT, "null output");
    *out = model->info;
  });
}

lsnif_status lsnif_query(lsnif_model model, const lsnif_ray* d_rays, int64_t n, int mode,
                         lsnif_hit* d_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    run_query(*model, d_rays, n, mode, d_hits, static_cast<cudaStream_t>(stream));
  });
}

lsnif_status lsnif_query_pairs(lsnif_model model, const lsnif_ray* d_rays, const lsnif_interval* d_intervals,
                               int64_t n, int mode, lsnif_hit* d_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    if (n > 0 && !d_intervals) fail(LSNIF_INVALID_ARGUMENT, "null interval pointer");
    run_query(*model, d_rays, n, mode, d_hits, static_cast<cudaStream_t>(stream), nullptr, d_intervals);
  });
}

lsnif_status lsnif_query_closest(lsnif_model model, const lsnif_ray* d_rays, const lsnif_interval* d_intervals,
                                 int64_t n, lsnif_hit* d_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    run_query(*model, d_rays, n, LSNIF_QUERY_CLOSEST, d_hits, static_cast<cudaStream_t>(stream), nullptr,
              d_intervals);
  });
}

lsnif_status lsnif_query_any(lsnif_model model, const lsnif_ray* d_rays, const lsnif_interval* d_intervals,
                             int64_t n, lsnif_hit* d_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    run_query(*model, d_rays, n, LSNIF_QUERY_ANY, d_hits, static_cast<cudaStream_t>(stream), nullptr,
              d_intervals);
  });
}

lsnif_status lsnif_query_host(lsnif_model model, const lsnif_ray* h_rays, int64_t n, int mode,
                              lsnif_hit* h_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative ray count");
    if (n > 0 && (!h_rays || !h_hits)) fail(LSNIF_INVALID_ARGUMENT, "null ray or hit pointer");
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    std::lock_guard<std::mutex> lock(model->staging_mu);
    host_round_trip(model->staging, kHostChunk, h_rays, n, h_hits, static_cast<cudaStream_t>(stream),
                    [&](const lsnif_ray* r, int64_t cn, lsnif_hit* h, cudaStream_t st) {
                      run_query(*model, r, cn, mode, h, st);
                    });
  });
}

lsnif_status lsnif_query_wire(lsnif_model model, const lsnif_ray* d_rays, int64_t n, int mode,
                              lsnif_hit_wire* d_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    run_query(*model, d_rays, n, mode, d_hits, static_cast<cudaStream_t>(stream), nullptr, nullptr, true);
  });
}

lsnif_status lsnif_query_host_wire(lsnif_model model, const lsnif_ray* h_rays, int64_t n, int mode,
                                   lsnif_hit_wire* h_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative ray count");
    if (n > 0 && (!h_rays || !h_hits)) fail(LSNIF_INVALID_ARGUMENT, "null ray or hit pointer");
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    std::lock_guard<std::mutex> lock(model->staging_mu);
    host_round_trip(model->staging_wire, kHostChunk, h_rays, n, h_hits, static_cast<cudaStream_t>(stream),
                    [&](const lsnif_ray* r, int64_t cn, lsnif_hit_wire* h, cudaStream_t st) {
                      run_query(*model, r, cn, mode, h, st, nullptr, nullptr, true);
                    });
  });
}

lsnif_status lsnif_hits_from_wire(const lsnif_hit_wire* h_wire, int64_t n, lsnif_hit* h_out) {
  return guarded([&] {
    if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative count");
    if (n > 0 && (!h_wire || !h_out)) fail(LSNIF_INVALID_ARGUMENT, "null pointer");
    for (int64_t i = 0; i < n; ++i) lsnif_dev::wire_unpack(h_wire[i], h_out[i]);
  });
}

lsnif_status lsnif_infer_batch(lsnif_model model, const float* d_inputs, int64_t rows, int64_t n,
                               const lsnif_interval* d_intervals, int64_t n_intervals,
                               lsnif_hit* d_hits, void* stream) {
  return guarded([&] {
    check_model(model);
    if (n != n_intervals) fail(LSNIF_INVALID_ARGUMENT, "infer_batch: inputs/intervals size mismatch");
    if (rows != model->dm.K1) fail(LSNIF_INVALID_ARGUMENT, "infer_batch: input width mismatch");
    if (n > 0 && (!d_inputs || !d_intervals || !d_hits)) fail(LSNIF_INVALID_ARGUMENT, "null pointer");
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    if (n == 0) return;
    // the caller's columns through the tcgen05 MLP (chunks of kChunk rows);
    // a chunk with an input beyond the scale's operand bound is answered
    // again by the fp32 kernel (device-side flag, no host round trip)
    lsnif_model_s& M = *model;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Workspace& w = M.workspace(st, n);
    const int64_t kChunk = w.chunk;
    const int64_t nchunks = (n + kChunk - 1) / kChunk;
    if (static_cast<size_t>(nchunks) > kMaxChunks) fail(LSNIF_INVALID_ARGUMENT, "too many columns in one call");
    ck(cudaMemsetAsync(w.counters, 0, kChunkCounterBytes * nchunks, st), "cudaMemsetAsync");
    for (int64_t s = 0, ci = 0; s < n; s += kChunk, ++ci) {
      const int64_t cn = std::min(kChunk, n - s);
      uint8_t* cc = w.counters + kChunkCounterBytes * ci;
      int32_t* rows = reinterpret_cast<int32_t*>(cc + 8);
      int* overflow = reinterpret_cast<int*>(cc + 8 + 4 * lsnif_dev::kMaxBins);
      ck(lsnif_dev::launch_infer_pack(M.dm, d_inputs + s * M.dm.K1, cn, d_intervals + s, w.X, w.meta, rows,
                                      static_cast<int64_t>(w.x_tiles), overflow, st),
         "infer_pack_kernel");
      lsnif_dev::MlpParams mp{};
      mp.m = M.dm;
      mp.X = w.X;
      mp.meta = w.meta;
      mp.row_counter = rows;
      mp.cap_tiles = static_cast<int64_t>(w.x_tiles);
      mp.out = d_hits + s;
      mp.wire = 0;
      mp.mode = lsnif_dev::kInferMode;
      ck(lsnif_dev::launch_mlp(mp, static_cast<int>((cn + kTileM - 1) / kTileM) + M.dm.n_bins, M.num_sms, st),
         "mlp_tc_kernel");
      ck(lsnif_dev::launch_infer_f32(M.dm, d_inputs + s * M.dm.K1, cn, d_intervals + s, d_hits + s, st,
                                     overflow),
         "infer_f32_kernel");
    }
  });
}

lsnif_status lsnif_infer_batch_f32(lsnif_model model, const float* d_inputs, int64_t rows, int64_t n,
                                   const lsnif_interval* d_intervals, int64_t n_intervals, lsnif_hit* d_hits,
                                   void* stream) {
  return guarded([&] {
    check_model(model);
    if (n != n_intervals) fail(LSNIF_INVALID_ARGUMENT, "infer_batch: inputs/intervals size mismatch");
    if (rows != model->dm.K1) fail(LSNIF_INVALID_ARGUMENT, "infer_batch: input width mismatch");
    if (n > 0 && (!d_inputs || !d_intervals || !d_hits)) fail(LSNIF_INVALID_ARGUMENT, "null pointer");
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    ck(lsnif_dev::launch_infer_f32(model->dm, d_inputs, n, d_intervals, d_hits,
                                   static_cast<cudaStream_t>(stream)),
       "infer_f32_kernel");
  });
}

lsnif_status lsnif_debug_traverse(lsnif_model model, const lsnif_ray* d_rays, int64_t n, int32_t* info,
                                  float* interval, float* t, float* pts, uint32_t* cells, uint32_t* hidx,
                                  float* feat, void* stream) {
  return guarded([&] {
    check_model(model);
    if (n < 0) fail(LSNIF_INVALID_ARGUMENT, "negative ray count");
    if (n == 0) return;
    if (!d_rays || !info || !interval || !t || !pts || !cells || !hidx || !feat)
      fail(LSNIF_INVALID_ARGUMENT, "null pointer");
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    const DevModel& m = model->dm;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t H = m.H, L = m.L;
    ck(cudaMemsetAsync(t, 0, n * H * 4, st), "memset");
    ck(cudaMemsetAsync(pts, 0, n * H * 12, st), "memset");
    ck(cudaMemsetAsync(cells, 0xff, n * H * 4, st), "memset");
    ck(cudaMemsetAsync(hidx, 0xff, n * H * L * 8 * 4, st), "memset");
    ck(cudaMemsetAsync(feat, 0, n * static_cast<size_t>(m.K1) * 4, st), "memset");
    Workspace& w = model->workspace(st, 1);
    ck(cudaMemsetAsync(w.stats, 0, kStatsBytes + kChunkCounterBytes, st), "cudaMemsetAsync");
    lsnif_dev::TraceParams tp{};
    tp.m = m;
    tp.rays = d_rays;
    tp.n = n;
    tp.batch_counter = reinterpret_cast<unsigned long long*>(w.counters);
    tp.row_counter = reinterpret_cast<int32_t*>(w.counters + 8);
    tp.stats = w.stats;
    tp.info = info;
    tp.interval = interval;
    tp.t = t;
    tp.pts = pts;
    tp.cells = cells;
    tp.hidx = hidx;
    tp.feat = feat;
    ck(lsnif_dev::launch_trace(tp, true, st), "trace_encode_kernel<debug>");
  });
}

lsnif_status lsnif_profile_enable(lsnif_model model, int enable) {
  return guarded([&] {
    check_model(model);
    model->profiling.store(enable != 0);
  });
}

lsnif_status lsnif_profile_read(lsnif_model model, void* stream, int reset, lsnif_profile* out) {
  return guarded([&] {
    check_model(model);
    if (!out) fail(LSNIF_INVALID_ARGUMENT, "null output");
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    *out = lsnif_profile{};
    std::lock_guard<std::mutex> lock(model->mu);
    for (auto& kv : model->ws) {
      if (stream && kv.first != static_cast<cudaStream_t>(stream)) continue;
      Workspace& w = *kv.second;
      ck(cudaStreamSynchronize(kv.first), "cudaStreamSynchronize");
      std::lock_guard<std::mutex> plk(w.prof_mu);
      out->trace_launches += w.launches[0];
      out->mlp_launches += w.launches[1];
      for (auto& u : w.ev_used) {
        float ms = 0.0f;
        ck(cudaEventElapsedTime(&ms, u.second.first, u.second.second), "cudaEventElapsedTime");
        (u.first == 0 ? out->trace_ms : out->mlp_ms) += ms;
      }
      if (reset) {
        for (auto& u : w.ev_used) {
          w.ev_pool.push_back(u.second.first);
          w.ev_pool.push_back(u.second.second);
        }
        w.ev_used.clear();
        w.launches[0] = w.launches[1] = 0;
      }
    }
    out->launches = out->trace_launches + out->mlp_launches;
  });
}

lsnif_status lsnif_last_query_stats(lsnif_model model, void* stream, lsnif_query_stats* out) {
  return guarded([&] {
    check_model(model);
    if (!out) fail(LSNIF_INVALID_ARGUMENT, "null output");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Workspace* w = nullptr;
    {
      std::lock_guard<std::mutex> lock(model->mu);
      auto it = model->ws.find(st);
      if (it == model->ws.end()) fail(LSNIF_INVALID_ARGUMENT, "no query has run on this stream");
      w = it->second.get();
    }
    ck(cudaSetDevice(model->device), "cudaSetDevice");
    unsigned long long s[4];
    ck(cudaMemcpyAsync(s, w->stats, sizeof(s), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    out->rays = w->last_rays;
    out->pairs = static_cast<int64_t>(s[0]);
    out->mlp_rows = static_cast<int64_t>(s[1]);
    out->points = static_cast<int64_t>(s[2]);
    out->volume_points = static_cast<int64_t>(s[3]);
  });
}

}  // extern "C"

#ifdef LSNIF_PROBE  // A/B probes only (scripts/micro/dda_occupancy_probe.cuh)
const lsnif_dev::DevModel& lsnif_probe_devmodel(lsnif_model m) { return m->dm; }
#endif
