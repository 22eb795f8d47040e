// The extern "C" boundary (include/tcsl_cuda.h): argument checks with the
// reference's error classes, workspace carving, and kernel dispatch.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "tcsl_internal.cuh"

namespace tcslk {
int auto_split(uint32_t m, uint32_t k, int n, double avg_entries_per_tile);
}

namespace {

thread_local char g_cuda_err[256] = "";

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return TCSL_STATUS_OK;
  std::snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  return TCSL_STATUS_CUDA_ERROR;
}

// TileConfig::validate (proj/src/matrix.cpp:11-18).
bool tile_ok(int m_tb, int k_tb) {
  return m_tb > 0 && k_tb > 0 && m_tb % 8 == 0 && k_tb % 8 == 0 && static_cast<long long>(m_tb) * k_tb <= 65536;
}

uint32_t num_tiles(uint32_t m, uint32_t k, int m_tb, int k_tb) {
  return static_cast<uint32_t>(tcslk::div_up_i(m, m_tb)) * static_cast<uint32_t>(tcslk::div_up_i(k, k_tb));
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool is_default_tile(int m_tb, int k_tb) { return m_tb == 128 && k_tb == 64; }

// Row pitch (elements) the tensor-core path uses for X: TMA wants 16-B rows.
int x_pitch(int n) { return (n + 7) / 8 * 8; }

// The split the kernel will run: the request (or the heuristic's choice),
// clamped by the plan (at most tiles_k splits, bounded units per CTA pair).
int planned_split(uint32_t m, uint32_t k, int n, int split) {
  tcslk::SpmmPlan plan;
  tcslk::spmm_sm100_plan(m, k, n, split, &plan);
  return plan.split;
}

int effective_split(uint32_t m, uint32_t k, int n, int split_k) {
  if (split_k > 0) return planned_split(m, k, n, split_k);
  // the heuristic simulates the persistent schedule (SM count of the current
  // device); memoise it per device and shape
  static std::mutex mu;
  static std::map<std::tuple<int, uint32_t, uint32_t, int>, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) cudaGetLastError();
  const auto key = std::make_tuple(dev, m, k, n);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int s = planned_split(m, k, n, tcslk::auto_split(m, k, n, 0.2 * 8192));
  cache.emplace(key, s);
  return s;
}

struct SpmmWs {
  size_t x_pad, partials, total;
};

SpmmWs spmm_ws_layout(uint32_t m, uint32_t k, int n, int split, bool pad_x) {
  SpmmWs w{};
  w.x_pad = pad_x ? align256(static_cast<size_t>(k) * x_pitch(n) * 2) : 0;
  w.partials = split > 1 ? align256(static_cast<size_t>(split) * m * n * 4) : 0;
  w.total = w.x_pad + w.partials;
  return w;
}

}  // namespace

extern "C" {

int tcsl_cuda_abi_version(void) { return TCSL_CUDA_ABI_VERSION; }

const char* tcsl_cuda_status_string(int st) {
  switch (st) {
    case 0: return "ok";
    case 1: return "bad magic";
    case 2: return "unsupported version";
    case 3: return "bad header";
    case 4: return "wrong dtype";
    case 5: return "truncated file";
    case 6: return "trailing data";
    case 7: return "inconsistent offsets";
    case 8: return "location out of range";
    case 9: return "dimension mismatch";
    case 10: return "invalid argument";
    case 11: return "i/o failure";
    case TCSL_STATUS_CUDA_ERROR: return "cuda error";
    case TCSL_STATUS_UNSUPPORTED: return "unsupported";
    case TCSL_STATUS_WORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

const char* tcsl_cuda_last_cuda_error(void) { return g_cuda_err; }

int tcsl_cuda_read_error(const int* dErr, void* stream) {
  int h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, dErr, sizeof(int), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_status(e);
  return h;
}

// ------------------------------------------------------------------ encode
int tcsl_cuda_encode_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, size_t* ws_bytes) {
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  const uint32_t t = num_tiles(m, k, m_tb, k_tb);
  *ws_bytes = align256((static_cast<size_t>(t) + 1) * 4) + align256(tcslk::encode_scan_temp_bytes(t));
  return TCSL_STATUS_OK;
}

int tcsl_cuda_encode_count(const uint16_t* dW, uint32_t m, uint32_t k, int m_tb, int k_tb, uint32_t* dOffsets,
                           void* ws, size_t ws_bytes, void* stream) {
  // tcsl_format.cpp:37-38: validate cfg, reject empty matrices
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !dW || !dOffsets) return TCSL_STATUS_INVALID_ARGUMENT;
  size_t need = 0;
  tcsl_cuda_encode_workspace(m, k, m_tb, k_tb, &need);
  if (!ws || ws_bytes < need) return TCSL_STATUS_WORKSPACE;
  auto s = static_cast<cudaStream_t>(stream);
  const uint32_t t = num_tiles(m, k, m_tb, k_tb);
  uint32_t* counts = static_cast<uint32_t*>(ws);
  void* temp = static_cast<char*>(ws) + align256((static_cast<size_t>(t) + 1) * 4);
  cudaError_t e = cudaMemsetAsync(counts + t, 0, 4, s);
  if (e == cudaSuccess) e = tcslk::launch_encode_count(dW, m, k, m_tb, k_tb, counts, s);
  if (e == cudaSuccess)
    e = tcslk::launch_encode_scan(counts, dOffsets, t, temp, ws_bytes - align256((static_cast<size_t>(t) + 1) * 4), s);
  return cuda_status(e);
}

int tcsl_cuda_encode_emit(const uint16_t* dW, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                          const uint32_t* dOffsets, uint32_t* dEntries, int* dErr, void* stream) {
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !dW || !dOffsets) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_encode_emit(dW, m, k, m_tb, k_tb, reorder, dOffsets, dEntries, dErr,
                                               static_cast<cudaStream_t>(stream)));
}

int tcsl_cuda_encode_fused_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, size_t* ws_bytes) {
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  *ws_bytes = tcslk::encode_fused_ws_bytes(num_tiles(m, k, m_tb, k_tb));
  return TCSL_STATUS_OK;
}

int tcsl_cuda_encode_fused(const uint16_t* dW, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                           uint32_t* dOffsets, uint32_t* dEntries, uint64_t capacity, void* ws, size_t ws_bytes,
                           int* dErr, void* stream) {
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !dW || !dOffsets || (capacity && !dEntries))
    return TCSL_STATUS_INVALID_ARGUMENT;
  if (!tcslk::encode_fused_supported(dW, dEntries, k, m_tb, k_tb, reorder)) return TCSL_STATUS_UNSUPPORTED;
  size_t need = 0;
  tcsl_cuda_encode_fused_workspace(m, k, m_tb, k_tb, &need);
  if (!ws || ws_bytes < need) return TCSL_STATUS_WORKSPACE;
  return cuda_status(tcslk::launch_encode_fused(dW, m, k, m_tb, k_tb, reorder, dOffsets, dEntries, capacity, ws,
                                                dErr, static_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------ decode
int tcsl_cuda_decode(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m, uint32_t k,
                     int m_tb, int k_tb, uint16_t* dOut, int* dErr, void* stream) {
  if (!tile_ok(m_tb, k_tb)) return TCSL_STATUS_INVALID_ARGUMENT;
  if (m == 0 || k == 0) return 3;  // bad_header (tcsl_format.cpp:128)
  if (!dOffsets || !dOut) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_decode(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dOut, dErr, 1,
                                          static_cast<cudaStream_t>(stream)));
}

int tcsl_cuda_validate(const uint32_t* dOffsets, uint64_t n_entries, uint32_t m, uint32_t k, int m_tb, int k_tb,
                       int* dErr, void* stream) {
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !dOffsets) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_validate(dOffsets, n_entries, num_tiles(m, k, m_tb, k_tb), dErr,
                                            static_cast<cudaStream_t>(stream)));
}

int tcsl_cuda_validate_entries(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                               uint32_t k, int m_tb, int k_tb, int mode, uint32_t* dFlags, int* dErr, void* stream) {
  if (!tile_ok(m_tb, k_tb) || m == 0 || k == 0 || !dOffsets || (n_entries && !dEntries)) return TCSL_STATUS_INVALID_ARGUMENT;
  if (mode < TCSL_CHECK_SPMM || mode > TCSL_CHECK_INGEST) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_validate_entries(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, mode, dFlags,
                                                    dErr, static_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------ ingest
// deserialize_tcsl (proj/src/tcsl_format.cpp:180-222): header fields and their
// checks in the reference's order.
int tcsl_cuda_parse_header(const void* bytes, size_t size, tcsl_cuda_header* out) {
  if (!out || (!bytes && size)) return TCSL_STATUS_INVALID_ARGUMENT;
  const uint8_t* p = static_cast<const uint8_t*>(bytes);
  size_t at = 0;
  auto le = [&](int nb, uint32_t* v) {
    if (size - at < static_cast<size_t>(nb)) return false;
    *v = 0;
    for (int i = 0; i < nb; ++i) *v |= static_cast<uint32_t>(p[at + i]) << (8 * i);
    at += nb;
    return true;
  };
  constexpr int kTruncated = 5, kBadMagic = 1, kBadVersion = 2, kBadHeader = 3, kTrailing = 6;
  if (size < 4) return kTruncated;
  if (std::memcmp(p, "TCSL", 4) != 0) return kBadMagic;
  at = 4;
  uint32_t version = 0, flags = 0, m = 0, k = 0, m_tb = 0, k_tb = 0, nt = 0;
  if (!le(2, &version)) return kTruncated;
  if (version != 1) return kBadVersion;
  if (!le(2, &flags)) return kTruncated;
  if (flags & ~1u) return kBadVersion;
  if (!le(4, &m) || !le(4, &k) || !le(4, &m_tb) || !le(4, &k_tb)) return kTruncated;
  if (m == 0 || k == 0) return kBadHeader;
  if (m_tb == 0 || k_tb == 0 || m_tb > 65536 || k_tb > 65536) return kBadHeader;
  if (!tile_ok(static_cast<int>(m_tb), static_cast<int>(k_tb))) return kBadHeader;
  if (!le(4, &nt)) return kTruncated;
  const uint64_t want_tiles = static_cast<uint64_t>(tcslk::div_up_i(m, m_tb)) * tcslk::div_up_i(k, k_tb);
  if (nt != want_tiles) return kBadHeader;
  const size_t off_bytes = 4 * (static_cast<size_t>(nt) + 1);
  if (size - at < off_bytes) return kTruncated;
  uint32_t last = 0;
  std::memcpy(&last, p + at + off_bytes - 4, 4);
  const size_t payload = size - at - off_bytes;
  if (payload != 4 * static_cast<size_t>(last)) {
    // The reference checks the offset table before the payload size: report
    // inconsistent_offsets when the table itself is malformed (host scan, error path only).
    uint32_t prev = 0;
    for (uint32_t i = 0; i <= nt; ++i) {
      uint32_t o = 0;
      std::memcpy(&o, p + at + 4 * static_cast<size_t>(i), 4);
      if ((i == 0 && o != 0) || (i > 0 && (o < prev || ((o - prev) & 31u)))) return TCSL_STATUS_INCONSISTENT_OFFSETS;
      prev = o;
    }
    return payload < 4 * static_cast<size_t>(last) ? kTruncated : kTrailing;
  }
  out->m = m;
  out->k = k;
  out->m_tb = m_tb;
  out->k_tb = k_tb;
  out->num_tiles = nt;
  out->reordered = flags & 1u;
  out->n_entries = last;
  return TCSL_STATUS_OK;
}

int tcsl_cuda_ingest(const void* bytes, size_t size, const tcsl_cuda_header* h, uint32_t* dOffsets,
                     uint32_t* dEntries, void* staging, size_t staging_bytes, uint32_t* dFlags, int* dErr,
                     void* stream) {
  if (!bytes || !h || !dOffsets || (h->n_entries && !dEntries)) return TCSL_STATUS_INVALID_ARGUMENT;
  if (staging && staging_bytes < (1u << 20)) return TCSL_STATUS_INVALID_ARGUMENT;
  const size_t off_bytes = 4 * (static_cast<size_t>(h->num_tiles) + 1), ent_bytes = 4 * h->n_entries;
  if (size != 28 + off_bytes + ent_bytes) return TCSL_STATUS_INVALID_ARGUMENT;  // parse_header first
  auto s = static_cast<cudaStream_t>(stream);
  const uint8_t* src = static_cast<const uint8_t*>(bytes) + 28;
  cudaError_t e = cudaSuccess;
  if (!staging) {  // caller's buffer is pinned (or accepts a synchronous pageable copy)
    e = cudaMemcpyAsync(dOffsets, src, off_bytes, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && ent_bytes)
      e = cudaMemcpyAsync(dEntries, src + off_bytes, ent_bytes, cudaMemcpyHostToDevice, s);
  } else {
    // pageable source: two pinned halves, host memcpy of chunk i+1 overlaps the DMA of chunk i
    const size_t half = (staging_bytes / 2) & ~size_t(255);
    cudaEvent_t ev[2];
    bool ev_ok[2] = {false, false};
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
      ev_ok[i] = e == cudaSuccess;
    }
    struct Part {
      uint8_t* dst;
      const uint8_t* src;
      size_t n;
    } parts[2] = {{reinterpret_cast<uint8_t*>(dOffsets), src, off_bytes},
                  {reinterpret_cast<uint8_t*>(dEntries), src + off_bytes, ent_bytes}};
    int slot = 0;
    bool used[2] = {false, false};
    for (const Part& part : parts) {
      for (size_t pos = 0; pos < part.n && e == cudaSuccess; pos += half, slot ^= 1) {
        const size_t c = std::min(half, part.n - pos);
        uint8_t* buf = static_cast<uint8_t*>(staging) + slot * half;
        if (used[slot]) e = cudaEventSynchronize(ev[slot]);
        if (e != cudaSuccess) break;
        std::memcpy(buf, part.src + pos, c);
        e = cudaMemcpyAsync(part.dst + pos, buf, c, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[slot], s);
        used[slot] = true;
      }
    }
    for (int i = 0; i < 2; ++i) {
      if (ev_ok[i] && used[i]) {
        const cudaError_t e2 = cudaEventSynchronize(ev[i]);
        if (e == cudaSuccess) e = e2;
      }
      if (ev_ok[i]) cudaEventDestroy(ev[i]);
    }
  }
  if (e != cudaSuccess) return cuda_status(e);
  return cuda_status(tcslk::launch_validate_entries(dOffsets, dEntries, h->n_entries, h->m, h->k,
                                                    static_cast<int>(h->m_tb), static_cast<int>(h->k_tb),
                                                    TCSL_CHECK_INGEST, dFlags, dErr, s));
}

// -------------------------------------------------------------------- prune
int tcsl_cuda_prune_workspace(uint64_t count, size_t* ws_bytes) {
  if (!ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  *ws_bytes = tcslk::prune_workspace_bytes(count);
  return TCSL_STATUS_OK;
}

int tcsl_cuda_prune_magnitude(const uint16_t* dA, uint64_t count, double beta, uint16_t* dOut, void* ws,
                              size_t ws_bytes, void* stream) {
  // matrix.cpp:69-75: beta in [0, 1], cut = floor(beta * n) clamped to [0, n]
  if (!(beta >= 0.0 && beta <= 1.0)) return TCSL_STATUS_INVALID_ARGUMENT;
  if (count && (!dA || !dOut)) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!ws || ws_bytes < tcslk::prune_workspace_bytes(count)) return TCSL_STATUS_WORKSPACE;
  long long cut = static_cast<long long>(std::floor(beta * static_cast<double>(count)));
  cut = std::max(0ll, std::min(cut, static_cast<long long>(count)));
  return cuda_status(tcslk::launch_prune(dA, count, static_cast<uint64_t>(cut), dOut, ws, ws_bytes,
                                         static_cast<cudaStream_t>(stream)));
}

// -------------------------------------------------------------------- spmm
int tcsl_cuda_spmm_auto_split(uint32_t m, uint32_t k, int n) { return effective_split(m, k, n, 0); }

int tcsl_cuda_spmm_estimate(uint32_t m, uint32_t k, int n, uint64_t n_entries, int split_k, double hbm_gbs,
                            tcsl_cuda_estimate* out) {
  if (!out || m == 0 || k == 0 || n <= 0 || split_k < 0) return TCSL_STATUS_INVALID_ARGUMENT;
  constexpr double kClockMHz = 1965.0;     // B200 SM clock under load (bench clocks)
  constexpr double kMmaCycles = 32.0;      // per tcgen05.mma M=256 instruction, in situ (ncu)
  constexpr double kChain0 = 284.3, kChainG = 3.95, kChainN = 0.763;  // cycles per tile (fit)
  constexpr double kFixedUs = 10.89, kSplitUs = 2.42;                  // per launch, split-K pass (fit)
  if (hbm_gbs <= 0) hbm_gbs = 6558.7;      // MEASURED_PEAKS.json copy bandwidth
  const uint32_t tiles_m = (m + 127) / 128, tiles_k = (k + 63) / 64;
  const double tiles = static_cast<double>(tiles_m) * tiles_k;
  const int split = effective_split(m, k, n, split_k);
  const int clusters = std::max(1, tcslk::num_sms() / 2);
  const uint64_t units = static_cast<uint64_t>((tiles_m + 1) / 2) * split;
  const double per_cta = static_cast<double>((units + clusters - 1) / clusters) *
                         static_cast<double>((tiles_k + split - 1) / split);
  const double g = static_cast<double>(n_entries) / 32.0 / tiles;
  const double clear = g <= 32.0 ? 1.5 * g : (g <= 81.0 ? 128.0 : 1.5 * g);  // rescatter or zero fill
  const double wavefronts = g * (1.0 + 1.5) + clear + 136.0 + 4.0 * n_entries / tiles / 128.0;
  const double bytes = 4.0 * n_entries + 4.0 * (tiles + 1) + 2.0 * k * n + 4.0 * static_cast<double>(m) * n;
  out->split = split;
  out->hbm_us = bytes / (hbm_gbs * 1e3);
  out->tensor_us = per_cta * 4.0 * kMmaCycles / kClockMHz;
  out->smem_us = per_cta * wavefronts / kClockMHz;
  out->chain_us = per_cta * (kChain0 + kChainG * g + kChainN * n) / kClockMHz;
  out->fixed_us = kFixedUs + (split > 1 ? kSplitUs : 0.0);
  double worst = out->hbm_us;
  out->bound = TCSL_BOUND_HBM;
  if (out->tensor_us > worst) { worst = out->tensor_us; out->bound = TCSL_BOUND_TENSOR; }
  if (out->smem_us > worst) { worst = out->smem_us; out->bound = TCSL_BOUND_SMEM; }
  if (out->chain_us > worst) { worst = out->chain_us; out->bound = TCSL_BOUND_CHAIN; }
  out->us = out->fixed_us + worst;
  return TCSL_STATUS_OK;
}

int tcsl_cuda_spmm_exact_workspace(uint32_t m, uint32_t k, size_t* ws_bytes) {
  if (!ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  *ws_bytes = align256(static_cast<size_t>(m) * k * 2);
  return TCSL_STATUS_OK;
}

int tcsl_cuda_spmm_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, int n, int split_k, size_t* ws_bytes) {
  return tcsl_cuda_spmm_ex_workspace(m, k, m_tb, k_tb, n, split_k, 0, ws_bytes);
}

int tcsl_cuda_spmm_ex_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, int n, int split_k, int exact,
                                size_t* ws_bytes) {
  if (!tile_ok(m_tb, k_tb) || n <= 0 || split_k < 0 || !ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  if (exact || !is_default_tile(m_tb, k_tb)) {
    // dense reconstruction + an fp32 staging buffer for the fused epilogue
    *ws_bytes = align256(static_cast<size_t>(m) * k * 2) + align256(static_cast<size_t>(m) * n * 4);
    return TCSL_STATUS_OK;
  }
  *ws_bytes = spmm_ws_layout(m, k, n, effective_split(m, k, n, split_k), true).total;
  return TCSL_STATUS_OK;
}

int tcsl_cuda_spmm_exact(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                         uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, float* dY, void* ws,
                         size_t ws_bytes, int* dErr, void* stream) {
  return tcsl_cuda_spmm_ex(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dX, n, dY, TCSL_OUT_F32, nullptr,
                           TCSL_ACT_NONE, 0, 1, ws, ws_bytes, dErr, stream);
}

int tcsl_cuda_spmm(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m, uint32_t k,
                   int m_tb, int k_tb, const uint16_t* dX, int n, float* dY, int split_k, void* ws,
                   size_t ws_bytes, int* dErr, void* stream) {
  return tcsl_cuda_spmm_ex(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dX, n, dY, TCSL_OUT_F32, nullptr,
                           TCSL_ACT_NONE, split_k, 0, ws, ws_bytes, dErr, stream);
}

namespace {

// tcsl_cuda_spmm_ex and tcsl_cuda_spmm_push: Y to dY, or (n_peers > 0) to every
// dPeers[g] (device array of base pointers) through the epilogue pass.
int spmm_core(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m, uint32_t k,
              int m_tb, int k_tb, const uint16_t* dX, int n, void* dY, int out_dtype, void* const* dPeers,
              int n_peers, const float* dBias, int activation, int split_k, int exact, void* ws, size_t ws_bytes,
              int* dErr, void* stream) {
  // engine.cpp:28-32 (the dimension check is the caller's: no B shape crosses the ABI)
  if (!tile_ok(m_tb, k_tb) || n <= 0 || m == 0 || k == 0 || split_k < 0) return TCSL_STATUS_INVALID_ARGUMENT;
  if (out_dtype != TCSL_OUT_F32 && out_dtype != TCSL_OUT_F16) return TCSL_STATUS_INVALID_ARGUMENT;
  if (activation < TCSL_ACT_NONE || activation > TCSL_ACT_GELU_TANH) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!dOffsets || !dX || (n_peers > 0 ? !dPeers : !dY) || n_peers < 0 || (n_entries && !dEntries))
    return TCSL_STATUS_INVALID_ARGUMENT;
  auto s = static_cast<cudaStream_t>(stream);
  const bool push = n_peers > 0;
  const bool fused = dBias != nullptr || activation != TCSL_ACT_NONE || out_dtype == TCSL_OUT_F16 || push;
  float* y32 = out_dtype == TCSL_OUT_F32 ? static_cast<float*>(dY) : nullptr;
  uint16_t* y16 = out_dtype == TCSL_OUT_F16 ? static_cast<uint16_t*>(dY) : nullptr;
  cudaError_t e = cudaSuccess;
  if (exact || !is_default_tile(m_tb, k_tb)) {
    const size_t need = align256(static_cast<size_t>(m) * k * 2) + (fused ? align256(static_cast<size_t>(m) * n * 4) : 0);
    if (!ws || ws_bytes < need) return TCSL_STATUS_WORKSPACE;
    uint16_t* dense = static_cast<uint16_t*>(ws);
    float* tmp = reinterpret_cast<float*>(static_cast<char*>(ws) + align256(static_cast<size_t>(m) * k * 2));
    e = tcslk::launch_decode(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dense, dErr, 0, s);
    if (e == cudaSuccess) e = tcslk::launch_dense_gemm_exact(dense, m, k, dX, n, fused ? tmp : y32, s);
    if (e == cudaSuccess && fused)
      e = tcslk::launch_reduce_epilogue(tmp, 1, m, n, dBias, activation, y32, y16, s, dPeers, n_peers,
                                        out_dtype == TCSL_OUT_F16);
    return cuda_status(e);
  }
  // cp.async.bulk streams 128-B spans of the entries: they must be 16-B aligned
  if (reinterpret_cast<uintptr_t>(dEntries) & 15u) return TCSL_STATUS_INVALID_ARGUMENT;
  const int split = effective_split(m, k, n, split_k);
  const bool pad_x = (n % 8) != 0 || (reinterpret_cast<uintptr_t>(dX) & 15u) != 0;
  const SpmmWs lay = spmm_ws_layout(m, k, n, split, pad_x);
  if (lay.total && (!ws || ws_bytes < lay.total)) return TCSL_STATUS_WORKSPACE;
  const uint16_t* x = dX;
  int ldx = n;
  if (pad_x) {
    uint16_t* xp = static_cast<uint16_t*>(ws);
    ldx = x_pitch(n);
    e = cudaMemsetAsync(xp, 0, static_cast<size_t>(k) * ldx * 2, s);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(xp, static_cast<size_t>(ldx) * 2, dX, static_cast<size_t>(n) * 2,
                            static_cast<size_t>(n) * 2, k, cudaMemcpyDeviceToDevice, s);
    x = xp;
    if (e != cudaSuccess) return cuda_status(e);
  }
  tcslk::SpmmPlan plan;
  tcslk::spmm_sm100_plan(m, k, n, split, &plan);
  if (split > 1) {
    float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + lay.x_pad);
    e = tcslk::launch_spmm_sm100(plan, dOffsets, dEntries, n_entries, m, k, x, ldx, part, dErr, s);
    if (e == cudaSuccess)
      e = fused ? tcslk::launch_reduce_epilogue(part, split, m, n, dBias, activation, y32, y16, s, dPeers, n_peers,
                                                out_dtype == TCSL_OUT_F16)
                : tcslk::launch_splitk_reduce(part, split, static_cast<size_t>(m) * n, y32, s);
  } else {
    tcslk::Epilogue epi;
    epi.bias = dBias;
    epi.act = activation;
    epi.out16 = y16;
    epi.peers = dPeers;
    epi.n_peers = n_peers;
    epi.peers_f16 = out_dtype == TCSL_OUT_F16;
    e = tcslk::launch_spmm_sm100(plan, dOffsets, dEntries, n_entries, m, k, x, ldx, y32, dErr, s, epi);
  }
  return cuda_status(e);
}

}  // namespace

int tcsl_cuda_spmm_ex(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                      uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, void* dY, int out_dtype,
                      const float* dBias, int activation, int split_k, int exact, void* ws, size_t ws_bytes,
                      int* dErr, void* stream) {
  if (!dY) return TCSL_STATUS_INVALID_ARGUMENT;
  return spmm_core(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dX, n, dY, out_dtype, nullptr, 0, dBias,
                   activation, split_k, exact, ws, ws_bytes, dErr, stream);
}

int tcsl_cuda_spmm_push(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                        uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, void* const* dPeerY, int n_peers,
                        int out_dtype, const float* dBias, int activation, int split_k, int exact, void* ws,
                        size_t ws_bytes, int* dErr, void* stream) {
  if (n_peers <= 0 || n_peers > TCSL_MAX_PEERS || !dPeerY) return TCSL_STATUS_INVALID_ARGUMENT;
  return spmm_core(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dX, n, nullptr, out_dtype, dPeerY, n_peers,
                   dBias, activation, split_k, exact, ws, ws_bytes, dErr, stream);
}

int tcsl_cuda_splitk_reduce(const float* dPartials, int split_k, size_t count, float* dY, void* stream) {
  if (split_k < 1 || !dPartials || !dY) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_splitk_reduce(dPartials, split_k, count, dY, static_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- sharding
int tcsl_cuda_rebase_offsets(const uint32_t* dOffsets, uint32_t tile0, uint32_t tile1, uint32_t* dOut,
                             void* stream) {
  if (!dOffsets || !dOut || tile1 < tile0) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_rebase(dOffsets, tile0, tile1, dOut, static_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------- memory plumbing
int tcsl_cuda_malloc(void** dptr, size_t bytes) {
  if (!dptr) return TCSL_STATUS_INVALID_ARGUMENT;
  *dptr = nullptr;
  return bytes ? cuda_status(cudaMalloc(dptr, bytes)) : TCSL_STATUS_OK;
}
int tcsl_cuda_free(void* dptr) { return dptr ? cuda_status(cudaFree(dptr)) : TCSL_STATUS_OK; }
int tcsl_cuda_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (!bytes) return TCSL_STATUS_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
}
int tcsl_cuda_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  if (!bytes) return TCSL_STATUS_OK;
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
}
int tcsl_cuda_memset(void* dptr, int value, size_t bytes, void* stream) {
  if (!bytes) return TCSL_STATUS_OK;
  return cuda_status(cudaMemsetAsync(dptr, value, bytes, static_cast<cudaStream_t>(stream)));
}
int tcsl_cuda_stream_sync(void* stream) {
  return cuda_status(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
}
int tcsl_cuda_device_count(int* count) {
  if (!count) return TCSL_STATUS_INVALID_ARGUMENT;
  *count = 0;
  const cudaError_t e = cudaGetDeviceCount(count);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    *count = 0;
    return TCSL_STATUS_OK;
  }
  return cuda_status(e);
}

int tcsl_cuda_gen_synthetic(uint16_t* dW, uint64_t count, double beta, uint64_t seed, void* stream) {
  if (!dW || !(beta >= 0.0 && beta <= 1.0)) return TCSL_STATUS_INVALID_ARGUMENT;
  return cuda_status(tcslk::launch_gen_synthetic(dW, count, beta, seed, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
