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
 *   tcsl_cuda_validate_entries   <- check_offsets + decode's per-entry checks
 *                                   (location range, fringe payload, tcsl_format.cpp:137-152)
 *   tcsl_cuda_parse_header /     <- deserialize_tcsl  proj/src/tcsl_format.cpp:180-222
 *   tcsl_cuda_ingest                (host header checks, pinned upload, device validation)
 *   tcsl_cuda_spmm_ex            <- tcsl::spmm + the CLI's --out-f16 narrowing
 *                                   (tcsl_main.cpp:182-186, f16_from_f32 half.cpp:10-40),
 *                                   with an optional per-row bias and activation
 *   tcsl_cuda_prune_magnitude    <- prune_magnitude   proj/src/matrix.cpp:69-100
 *   tcsl_cuda_rebase_offsets     <- row-shard slicing
 *   tcsl_cuda_allgather_rows     <- the multi-GPU exchange of SURVEY.md §8(b)/(e)
 *                                   (the reference is single-process)
 */
#ifndef TCSL_CUDA_H
#define TCSL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCSL_CUDA_ABI_VERSION 2

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

/* One pass (W read once): per-tile counts, a decoupled look-back scan for the
 * offsets, and the entries, in a single kernel. TileConfig {128, 64} with the
 * bank reorder only (else TCSL_STATUS_UNSUPPORTED); dEntries 16-byte aligned.
 * dOffsets[0..T] are always written. A tile's entries are written only if
 * they end within `capacity` entries: when dOffsets[T] exceeds `capacity`,
 * the caller sizes dEntries from it and runs tcsl_cuda_encode_emit with the
 * same dOffsets. Same bits as count + emit.
 * ws: tcsl_cuda_encode_fused_workspace bytes (look-back status words). */
int tcsl_cuda_encode_fused_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, size_t* ws_bytes);
int tcsl_cuda_encode_fused(const uint16_t* dW, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                           uint32_t* dOffsets, uint32_t* dEntries, uint64_t capacity, void* ws, size_t ws_bytes,
                           int* dErr, void* stream);

/* ---------------------------------------------------------------- decode */
/* Dense m x k binary16 reconstruction (zeros as +0.0). Errors -> *dErr. */
int tcsl_cuda_decode(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                     uint32_t k, int m_tb, int k_tb, uint16_t* dOut, int* dErr, void* stream);

/* Structural check of a device-resident matrix (monotone offsets, whole
 * 32-entry groups, last offset == n_entries). Errors -> *dErr. */
int tcsl_cuda_validate(const uint32_t* dOffsets, uint64_t n_entries, uint32_t m, uint32_t k, int m_tb,
                       int k_tb, int* dErr, void* stream);

/* Whole-matrix validation on the device (offsets AND entries), one pass over E.
 *   mode TCSL_CHECK_DECODE:  the checks tcsl::decode makes (check_offsets, location
 *                            < m_tb*k_tb, no nonzero value in the padded fringe) raise
 *                            inconsistent_offsets / location_out_of_range in *dErr.
 *   mode TCSL_CHECK_SPMM:    the checks tcsl::spmm makes (engine.cpp:8-25: each tile's
 *                            span inside [0, n_entries], locations in range).
 *   mode TCSL_CHECK_INGEST:  the checks deserialize_tcsl makes (check_offsets only);
 *                            per-entry problems are reported as flags, not errors.
 * *dFlags (device, zero it first) |= TCSL_FLAG_* in every mode. */
enum { TCSL_CHECK_SPMM = 0, TCSL_CHECK_DECODE = 1, TCSL_CHECK_INGEST = 2 };
#define TCSL_FLAG_DUPLICATE_LOCATIONS 1u /* a tile repeats a location (the last entry wins) */
#define TCSL_FLAG_PARTIAL_GROUPS 2u      /* a tile span is not whole 32-entry groups */
#define TCSL_FLAG_FRINGE_PAYLOAD 4u      /* a nonzero value sits in the padded fringe */
#define TCSL_FLAG_LOCATION_RANGE 8u      /* a location >= m_tb * k_tb */
int tcsl_cuda_validate_entries(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries,
                               uint32_t m, uint32_t k, int m_tb, int k_tb, int mode, uint32_t* dFlags,
                               int* dErr, void* stream);

/* ---------------------------------------------------------------- ingest */
/* TCSL container -> device (reference byte layout, tcsl_format.hpp:68-71).
 * tcsl_cuda_parse_header runs deserialize_tcsl's host-side checks in its order
 * (bad_magic, bad_version, bad_header, truncated / trailing_data from the sizes)
 * and fills *out. tcsl_cuda_ingest then copies the offset table and the entries
 * from `bytes` (host memory; pageable data is staged through `staging`, a pinned
 * buffer of staging_bytes >= 1 MiB, or pass bytes already pinned and staging =
 * NULL) into dOffsets[num_tiles + 1] / dEntries[n_entries] (16-byte aligned) and
 * validates them on the device with TCSL_CHECK_INGEST. */
typedef struct tcsl_cuda_header {
  uint32_t m, k, m_tb, k_tb, num_tiles, reordered;
  uint64_t n_entries;
} tcsl_cuda_header;
int tcsl_cuda_parse_header(const void* bytes, size_t size, tcsl_cuda_header* out);
int tcsl_cuda_ingest(const void* bytes, size_t size, const tcsl_cuda_header* h, uint32_t* dOffsets,
                     uint32_t* dEntries, void* staging, size_t staging_bytes, uint32_t* dFlags, int* dErr,
                     void* stream);

/* ------------------------------------------------------------------ spmm */
/* Y[m x n] (fp32, row-major, ld = n) = W_tcsl x X[k x n] (binary16, row-major,
 * ld = n). Tensor-core path (tcgen05, fp32 accumulate) for TileConfig
 * {128, 64}; any other TileConfig runs the bit-exact CUDA-core path.
 * split_k: 0 = automatic, 1 = none, S > 1 = S partial sums reduced in fixed
 * order by tcsl_cuda_splitk_reduce (deterministic).
 * Preconditions of the tensor-core path (tcsl::encode output always meets
 * them; tcsl_cuda_validate_entries reports violations as flags):
 *   - every tile span is whole 32-entry groups (else inconsistent_offsets);
 *     tcsl_cuda_spmm_exact accepts partial groups like the reference;
 *   - no location repeats inside a tile (TCSL_FLAG_DUPLICATE_LOCATIONS): for
 *     such inputs use tcsl_cuda_spmm_exact, which resolves them last-writer-wins
 *     like tcsl::extract_tile (the tensor-core scatter would race);
 *   - dEntries is 16-byte aligned (bulk copies), else invalid_argument. */
int tcsl_cuda_spmm_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, int n, int split_k,
                             size_t* ws_bytes);
int tcsl_cuda_spmm(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                   uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, float* dY, int split_k,
                   void* ws, size_t ws_bytes, int* dErr, void* stream);
/* Fused epilogue: Y = act(W x X + bias) stored as fp32 or as binary16 bits
 * narrowed round-to-nearest-even with the canonical NaN 0x7E00 (f16_from_f32,
 * half.cpp:10-40; the CLI's --out-f16, tcsl_main.cpp:182-186). dBias: m floats
 * (one per output row) or NULL. activation: TCSL_ACT_*. out_dtype: TCSL_OUT_*.
 * exact != 0 runs the bit-exact CUDA-core product first (any TileConfig). */
enum { TCSL_ACT_NONE = 0, TCSL_ACT_RELU = 1, TCSL_ACT_GELU_TANH = 2 };
enum { TCSL_OUT_F32 = 0, TCSL_OUT_F16 = 1 };
int tcsl_cuda_spmm_ex_workspace(uint32_t m, uint32_t k, int m_tb, int k_tb, int n, int split_k, int exact,
                                size_t* ws_bytes);
int tcsl_cuda_spmm_ex(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                      uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, void* dY, int out_dtype,
                      const float* dBias, int activation, int split_k, int exact, void* ws, size_t ws_bytes,
                      int* dErr, void* stream);
/* The split the automatic heuristic picks for this shape on this device. */
/* Row-sharded SpMM with the all-gather fused into the epilogue (SURVEY.md §8e,
 * configs[4]): as tcsl_cuda_spmm_ex, but every finished Y row block is stored
 * into each of the n_peers (<= TCSL_MAX_PEERS) destinations dPeerY[g] (a DEVICE
 * array of device pointers: rank g's full-Y buffer, already offset to this
 * shard's first row; peer pointers are NVLink-mapped, e.g. symmetric memory), so
 * no collective runs after the kernel; the caller's cross-rank barrier makes the
 * rows visible. With split-K the epilogue pass (K3) does the pushing. */
#define TCSL_MAX_PEERS 64
int tcsl_cuda_spmm_push(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries, uint32_t m,
                        uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, void* const* dPeerY, int n_peers,
                        int out_dtype, const float* dBias, int activation, int split_k, int exact, void* ws,
                        size_t ws_bytes, int* dErr, void* stream);
/* A-priori time model of tcsl_cuda_spmm on a B200 (the B200 counterpart of the
 * reference's estimate_time, proj/src/pipeline.cpp:214-273, which models the
 * A100 kernel as max(gmem, smem, tensor) time): per persistent CTA,
 *   t = fixed + max(HBM, tensor, smem, chain),
 * HBM = (4E + 4(T+1) + 2KN + 4MN) / hbm_gbs (0: the measured 6558.7 GB/s);
 * tensor = 4 tcgen05.mma per tile at the in-situ 32 cycles (ncu); smem = the
 * shared-memory wavefronts of one tile (ring LDS, scatter, clear or zero fill,
 * bulk-copy landing, tensor-core operand reads) at 1 per cycle; chain = the
 * per-tile decode/issue handshake latency, 284 + 3.95 g + 0.76 N cycles for g
 * groups per tile (fitted to the 84 cold cells of profiles/r02_bench_v3.json);
 * fixed = 10.9 us per launch + 2.4 us for the split-K pass; clock 1965 MHz.
 * split_k 0 = the auto choice. Host only (no GPU needed). */
enum { TCSL_BOUND_HBM = 0, TCSL_BOUND_TENSOR = 1, TCSL_BOUND_SMEM = 2, TCSL_BOUND_CHAIN = 3 };
typedef struct {
  double us, hbm_us, tensor_us, smem_us, chain_us, fixed_us;
  int split, bound;
} tcsl_cuda_estimate;
int tcsl_cuda_spmm_estimate(uint32_t m, uint32_t k, int n, uint64_t n_entries, int split_k, double hbm_gbs,
                            tcsl_cuda_estimate* out);
int tcsl_cuda_spmm_auto_split(uint32_t m, uint32_t k, int n);
/* Y = sum_{s=0}^{S-1} P[s] in ascending s (P is S x count floats). */
int tcsl_cuda_splitk_reduce(const float* dPartials, int split_k, size_t count, float* dY, void* stream);
/* Bit-exact mode: same multiply/add sequence as tcsl::spmm / dense_gemm_ref
 * (proj/src/gemm.cpp:36-40), any TileConfig. ws >= tcsl_cuda_spmm_exact_workspace. */
int tcsl_cuda_spmm_exact_workspace(uint32_t m, uint32_t k, size_t* ws_bytes);
int tcsl_cuda_spmm_exact(const uint32_t* dOffsets, const uint32_t* dEntries, uint64_t n_entries,
                         uint32_t m, uint32_t k, int m_tb, int k_tb, const uint16_t* dX, int n, float* dY,
                         void* ws, size_t ws_bytes, int* dErr, void* stream);

/* ------------------------------------------------------------------ prune */
/* Magnitude pruning on the device, bit-exact with prune_magnitude: the
 * floor(beta * count) elements smallest by |value| (NaN ranks as +inf) become
 * +0.0; among equal magnitudes the larger row-major index goes first. dOut may
 * equal dA. beta outside [0, 1] -> invalid_argument. */
int tcsl_cuda_prune_workspace(uint64_t count, size_t* ws_bytes);
int tcsl_cuda_prune_magnitude(const uint16_t* dA, uint64_t count, double beta, uint16_t* dOut, void* ws,
                              size_t ws_bytes, void* stream);

/* --------------------------------------------------------------- sharding */
/* Row shard [tile row tr0, tr1): dOut[i] = dOffsets[tr0*tk + i] - dOffsets[tr0*tk],
 * i in [0, (tr1-tr0)*tk]. The shard's entries are dEntries + dOffsets[tr0*tk]. */
int tcsl_cuda_rebase_offsets(const uint32_t* dOffsets, uint32_t tile0, uint32_t tile1, uint32_t* dOut,
                             void* stream);

/* Row-sharded Y: rank r holds rows [r*rows_per_rank, ...) of
 * the m x n fp32 result in dYg (rows_per_rank x n); after the call every rank
 * holds the whole dY (nranks*rows_per_rank x n, rank-major). One
 * ncclAllGather on `comm` (an ncclComm_t) over NVLink, stream-ordered.
 * NCCL is resolved at run time (dlopen "libnccl.so.2", the copy torch already
 * loaded when there is one), so the library itself has no NCCL dependency.
 * out_dtype TCSL_OUT_F16 gathers binary16 rows (half the bytes). */
int tcsl_cuda_nccl_available(void);
int tcsl_cuda_nccl_unique_id(void* id128);
int tcsl_cuda_nccl_comm_init(void** comm, int nranks, const void* id128, int rank);
int tcsl_cuda_nccl_comm_destroy(void* comm);
int tcsl_cuda_allgather_rows(const void* dYg, void* dY, size_t rows_per_rank, int n, int out_dtype, void* comm,
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
