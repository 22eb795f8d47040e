// The extern "C" boundary (include/tcsl_cuda.h): argument checks with the
// reference's error classes, workspace carving, and kernel dispatch.
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
  // the heuristic simulates the persistent schedule; memoise it per shape
  static std::mutex mu;
  static std::map<std::tuple<uint32_t, uint32_t, int>, int> cache;
  const auto key = std::make_tuple(m, k, n);
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

// -------------------------------------------------------------------- spmm
int tcsl_cuda_spmm_auto_split(uint32_t m, uint32_t k, int n) { return effective_split(m, k, n, 0); }

int tcsl_cuda_spmm_exact_workspace(uint32_t m, uint32_t k, size_t* ws_bytes) {
  if (!ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  *ws_bytes = align256(static_cast<size_t>(m) * k * 2);
  return TCSL_STATUS_OK;
}

int tcsl_cuda_spmm_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, int n, int split_k, size_t* ws_bytes) {
  if (!tile_ok(m_tb, k_tb) || n <= 0 || !ws_bytes) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!is_default_tile(m_tb, k_tb)) return tcsl_cuda_spmm_exact_workspace(m, k, ws_bytes);
  *ws_bytes = spmm_ws_layout(m, k, n, effective_split(m, k, n, split_k), true).total;
  return TCSL_STATUS_OK;
}

int tcsl_cuda_spmm_exact(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                         uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, float* dY, void* ws,
                         size_t ws_bytes, int* dErr, void* stream) {
  // engine.cpp:28-32
  if (!tile_ok(m_tb, k_tb) || n <= 0 || m == 0 || k == 0) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!dOffsets || !dX || !dY) return TCSL_STATUS_INVALID_ARGUMENT;
  size_t need = 0;
  tcsl_cuda_spmm_exact_workspace(m, k, &need);
  if (!ws || ws_bytes < need) return TCSL_STATUS_WORKSPACE;
  auto s = static_cast<cudaStream_t>(stream);
  uint16_t* dense = static_cast<uint16_t*>(ws);
  cudaError_t e = tcslk::launch_decode(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dense, dErr, 0, s);
  if (e == cudaSuccess) e = tcslk::launch_dense_gemm_exact(dense, m, k, dX, n, dY, s);
  return cuda_status(e);
}

int tcsl_cuda_spmm(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m, uint32_t k,
                   int m_tb, int k_tb, const uint16_t* dX, int n, float* dY, int split_k, void* ws,
                   size_t ws_bytes, int* dErr, void* stream) {
  if (!tile_ok(m_tb, k_tb) || n <= 0 || m == 0 || k == 0 || split_k < 0) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!dOffsets || !dX || !dY || (n_entries && !dEntries)) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!is_default_tile(m_tb, k_tb))
    return tcsl_cuda_spmm_exact(dOffsets, dEntries, n_entries, m, k, m_tb, k_tb, dX, n, dY, ws, ws_bytes, dErr,
                                stream);
  auto s = static_cast<cudaStream_t>(stream);
  const int split = effective_split(m, k, n, split_k);
  const bool pad_x = (n % 8) != 0 || (reinterpret_cast<uintptr_t>(dX) & 15u) != 0;
  const SpmmWs lay = spmm_ws_layout(m, k, n, split, pad_x);
  if (lay.total && (!ws || ws_bytes < lay.total)) return TCSL_STATUS_WORKSPACE;
  const uint16_t* x = dX;
  int ldx = n;
  cudaError_t e = cudaSuccess;
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
  float* out = split > 1 ? reinterpret_cast<float*>(static_cast<char*>(ws) + lay.x_pad) : dY;
  e = tcslk::launch_spmm_sm100(plan, dOffsets, dEntries, n_entries, m, k, x, ldx, out, dErr, s);
  if (e == cudaSuccess && split > 1) e = tcslk::launch_splitk_reduce(out, split, static_cast<size_t>(m) * n, dY, s);
  return cuda_status(e);
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
