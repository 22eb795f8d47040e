/* tcsl_cuda.h — the C-ABI drop-in boundary of the B200 Tiled-CSL hot path.
 *
 * Plain C, plain pointers and sizes: no torch or C++ types cross this line.
 * Every function is stream-ordered on the caller's `cudaStream_t` (passed as
 * `void*`), works on caller-allocated DEVICE buffers, and returns 0 on success
 * or a status code:
 *     1..11  tcsl::Errc ordinal + 1 (reference: proj/include/tcsl/errors.hpp:10-22)
 *     TCSL_STATUS_CUDA_ERROR, TCSL_STATUS_UNSUPPORTED, TCSL_STATUS_WORKSPACE
 * Errors discovered on the device (bad locations, inconsistent offsets) are
 * recorded in the caller's `int* dErr` (device memory, zero it before use);
 * collect them with tcsl_cuda_read_error() after the stream work completes.
 *
 * Each entry point replaces one reference function on the Flash-LLM LSCD path:
 *   tcsl_cuda_encode_count/emit  <- tcsl::encode      proj/src/tcsl_format.cpp:36-124
 *                                   (decl proj/include/tcsl/tcsl_format.hpp:62)
 *   tcsl_cuda_decode             <- tcsl::decode      proj/src/tcsl_format.cpp:126-155
 *   tcsl_cuda_spmm               <- tcsl::spmm        proj/src/engine.cpp:27-78
 *                                   (decl proj/include/tcsl/engine.hpp:18); split_k
 *                                   mirrors upstream SpMM_SplitK_API
 *   tcsl_cuda_splitk_reduce      <- the upstream Reduction_Workspace sum
 *   tcsl_cuda_spmm_exact         <- tcsl::spmm bit-exact mode (dense_gemm_ref order,
 *                                   proj/src/gemm.cpp:36-40), any TileConfig
 *   tcsl_cuda_validate           <- check_offsets     proj/src/tcsl_format.cpp:19-32
 *   tcsl_cuda_rebase_offsets     <- row-shard slicing
 */
#ifndef TCSL_CUDA_H
#define TCSL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCSL_CUDA_ABI_VERSION 1

enum {
  TCSL_STATUS_OK = 0,
  /* 1..11: tcsl::Errc + 1 */
  TCSL_STATUS_INCONSISTENT_OFFSETS = 7,
  TCSL_STATUS_LOCATION_OUT_OF_RANGE = 8,
  TCSL_STATUS_DIMENSION_MISMATCH = 9,
  TCSL_STATUS_INVALID_ARGUMENT = 10,
  TCSL_STATUS_CUDA_ERROR = 64,
  TCSL_STATUS_UNSUPPORTED = 65,
  TCSL_STATUS_WORKSPACE = 66
};

int tcsl_cuda_abi_version(void);
const char* tcsl_cuda_status_string(int status);
/* Last CUDA error string seen by the library on this thread ("" if none). */
const char* tcsl_cuda_last_cuda_error(void);

/* Synchronises `stream`, reads *dErr (device) and returns it as a status. */
int tcsl_cuda_read_error(const int* dErr, void* stream);

/* ---------------------------------------------------------------- encode */
/* Workspace for tcsl_cuda_encode_count (scan temporaries). */
int tcsl_cuda_encode_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, size_t* ws_bytes);
/* Pass 1: dOffsets[0..T] = exclusive prefix of the 32-padded per-tile entry
 * counts, T = ceil(m/m_tb)*ceil(k/k_tb). dW is m x k row-major binary16 bits.
 * The host reads dOffsets[T] (4 bytes) to size dEntries. */
int tcsl_cuda_encode_count(const uint16_t* dW, uint32_t m, uint32_t k, int m_tb, int k_tb,
                           uint32_t* dOffsets, void* ws, size_t ws_bytes, void* stream);
/* Pass 2: writes the packed entries in exactly the reference's order
 * (bank-greedy reorder or natural scan order, +0.0 pads at the first zero
 * positions). Bit-exact with tcsl::encode. */
int tcsl_cuda_encode_emit(const uint16_t* dW, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                          const uint32_t* dOffsets, uint32_t* dEntries, int* dErr, void* stream);

/* ---------------------------------------------------------------- decode */
/* Dense m x k binary16 reconstruction (zeros as +0.0). Errors -> *dErr. */
int tcsl_cuda_decode(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                     uint32_t k, int m_tb, int k_tb, uint16_t* dOut, int* dErr, void* stream);

/* Structural check of a device-resident matrix (monotone offsets, whole
 * 32-entry groups, last offset == n_entries). Errors -> *dErr. */
int tcsl_cuda_validate(const uint32_t* dOffsets, uint64_t n_entries, uint32_t m, uint32_t k, int m_tb,
                       int k_tb, int* dErr, void* stream);

/* ------------------------------------------------------------------ spmm */
/* Y[m x n] (fp32, row-major, ld = n) = W_tcsl x X[k x n] (binary16, row-major,
 * ld = n). Tensor-core path (tcgen05, fp32 accumulate) for TileConfig
 * {128, 64}; any other TileConfig runs the bit-exact CUDA-core path.
 * split_k: 0 = automatic, 1 = none, S > 1 = S partial sums reduced in fixed
 * order by tcsl_cuda_splitk_reduce (deterministic). */
int tcsl_cuda_spmm_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, int n, int split_k,
                             size_t* ws_bytes);
int tcsl_cuda_spmm(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                   uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, float* dY, int split_k,
                   void* ws, size_t ws_bytes, int* dErr, void* stream);
/* The split the automatic heuristic picks for this shape on this device. */
int tcsl_cuda_spmm_auto_split(uint32_t m, uint32_t k, int n);
/* Y = sum_{s=0}^{S-1} P[s] in ascending s (P is S x count floats). */
int tcsl_cuda_splitk_reduce(const float* dPartials, int split_k, size_t count, float* dY, void* stream);
/* Bit-exact mode: same multiply/add sequence as tcsl::spmm / dense_gemm_ref
 * (proj/src/gemm.cpp:36-40), any TileConfig. ws >= tcsl_cuda_spmm_exact_workspace. */
int tcsl_cuda_spmm_exact_workspace(uint32_t m, uint32_t k, size_t* ws_bytes);
int tcsl_cuda_spmm_exact(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries,
                         uint32_t m, uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, float* dY,
                         void* ws, size_t ws_bytes, int* dErr, void* stream);

/* --------------------------------------------------------------- sharding */
/* Row shard [tile row tr0, tr1): dOut[i] = dOffsets[tr0*tk + i] - dOffsets[tr0*tk],
 * i in [0, (tr1-tr0)*tk]. The shard's entries are dEntries + dOffsets[tr0*tk]. */
int tcsl_cuda_rebase_offsets(const uint32_t* dOffsets, uint32_t tile0, uint32_t tile1, uint32_t* dOut,
                             void* stream);

/* ------------------------------------------------------- memory plumbing */
/* Thin wrappers so host bindings (C++, ctypes, cgo, JNI) never link a CUDA
 * runtime of their own. Same semantics as the CUDA runtime calls. */
int tcsl_cuda_malloc(void** dptr, size_t bytes);
int tcsl_cuda_free(void* dptr);
int tcsl_cuda_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int tcsl_cuda_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int tcsl_cuda_memset(void* dptr, int value, size_t bytes, void* stream);
int tcsl_cuda_stream_sync(void* stream);
int tcsl_cuda_device_count(int* count);

/* -------------------------------------------------------- bench utilities */
/* Synthetic random-sparse binary16 weights: each element is +0.0 with
 * probability beta, else a value with the reference's value law (uniform
 * sign, exponent field 13..17, uniform mantissa; proj/src/matrix.cpp:56-63).
 * Positions come from a counter hash, NOT from gen_random_sparse's
 * mt19937_64 stream (that one is inherently sequential). */
int tcsl_cuda_gen_synthetic(uint16_t* dW, uint64_t count, double beta, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TCSL_CUDA_H */
