// Shared declarations between the kernel translation units and the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/tcsl_cuda.h"

namespace tcslk {

constexpr int kGroup = 32;  // entries per group (proj/include/tcsl/tcsl_format.hpp:12)

// Device error codes (stored in *dErr). The smallest status wins, so the class
// matches the reference's check order (check_offsets -> inconsistent_offsets (7)
// before any per-entry location_out_of_range (8), tcsl_format.cpp:126-155)
// whatever order the threads report in.
__device__ __forceinline__ void raise_dev(int* err, int status) {
  if (!err) return;
  int cur = atomicCAS(err, 0, status);
  while (cur != 0 && status < cur) {
    const int prev = atomicCAS(err, cur, status);
    if (prev == cur) return;
    cur = prev;
  }
}

// tcsl_cuda_validate_entries flag bits (see include/tcsl_cuda.h).
constexpr uint32_t kFlagDuplicates = TCSL_FLAG_DUPLICATE_LOCATIONS;
constexpr uint32_t kFlagPartialGroups = TCSL_FLAG_PARTIAL_GROUPS;
constexpr uint32_t kFlagFringePayload = TCSL_FLAG_FRINGE_PAYLOAD;

inline int div_up_i(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Programmatic dependent launch for the SpMM-path kernels (env TCSL_PDL=0 turns it off).
bool pdl_enabled();

// binary16 bits of v, round to nearest even, overflow to +-inf, every NaN the
// canonical quiet NaN 0x7E00: f16_from_f32 (proj/src/half.cpp:10-40).
__device__ __forceinline__ uint32_t f16_bits_rne(float v) {
  if (v != v) return 0x7E00u;
  uint16_t h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(v));
  return h;
}

// Epilogue of tcsl_cuda_spmm_ex: act(acc + bias), one fp32 add (no FMA).
__device__ __forceinline__ float epilogue_value(float acc, float bias, int act) {
  float v = __fadd_rn(acc, bias);
  if (act == TCSL_ACT_RELU) {
    v = v > 0.0f ? v : (v != v ? v : 0.0f);
  } else if (act == TCSL_ACT_GELU_TANH) {
    // 0.5 v (1 + tanh(sqrt(2/pi) (v + 0.044715 v^3)))
    const float u = 0.7978845608028654f * (v + 0.044715f * v * v * v);
    v = 0.5f * v * (1.0f + tanhf(u));
  }
  return v;
}

// Host launchers (return cudaError_t as int, 0 on success).
cudaError_t launch_encode_count(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb,
                                uint32_t* counts, cudaStream_t s);
cudaError_t launch_encode_emit(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                               const uint32_t* offsets, uint32_t* entries, int* err, cudaStream_t s);
// strict = 1: tcsl::decode (check_offsets, fringe payloads rejected); strict = 0:
// tcsl::extract_tile semantics as used by spmm (per-tile spans only, fringe
// entries dropped). Repeated locations inside a tile resolve to the last entry
// (last writer wins, engine.cpp:17-22, tcsl_format.cpp:137-152).
cudaError_t launch_decode(const uint32_t* off, const uint32_t* ent, uint64_t n_entries, uint32_t m,
                          uint32_t k, int m_tb, int k_tb, uint16_t* out, int* err, int strict, cudaStream_t s);
// Structural validation without output (modes as launch_decode); flags |= kFlag*.
cudaError_t launch_validate_entries(const uint32_t* off, const uint32_t* ent, uint64_t n_entries, uint32_t m,
                                    uint32_t k, int m_tb, int k_tb, int strict, uint32_t* flags, int* err,
                                    cudaStream_t s);
size_t encode_scan_temp_bytes(uint32_t tiles);
// One-pass encoder (count + emit with a decoupled look-back; TileConfig {128, 64}, reorder).
size_t encode_fused_ws_bytes(uint32_t tiles);
bool encode_fused_supported(const void* w, const void* entries, uint32_t k, int m_tb, int k_tb, int reorder);
cudaError_t launch_encode_fused(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                                uint32_t* offsets, uint32_t* entries, uint64_t capacity, void* ws, int* err,
                                cudaStream_t s);
cudaError_t launch_encode_scan(uint32_t* counts_in, uint32_t* offsets, uint32_t tiles, void* temp,
                               size_t temp_bytes, cudaStream_t s);
cudaError_t launch_validate(const uint32_t* off, uint64_t n_entries, uint32_t tiles, int* err,
                            cudaStream_t s);
cudaError_t launch_dense_gemm_exact(const uint16_t* a, uint32_t m, uint32_t k, const uint16_t* x, int n,
                                    float* y, cudaStream_t s);
cudaError_t launch_splitk_reduce(const float* p, int split, size_t count, float* y, cudaStream_t s);
// Split-K reduce (or, split == 1, a pure epilogue pass) with the fused epilogue:
// y[i] = act(sum_s p[s][i] + bias[i / n]) as fp32 (y32) or binary16 (y16).
// peers / n_peers > 0: the result goes to n_peers destinations (device array of
// base pointers, each laid out like y32 / y16) instead of y32 / y16.
cudaError_t launch_reduce_epilogue(const float* p, int split, uint32_t m, int n, const float* bias, int act,
                                   float* y32, uint16_t* y16, cudaStream_t s, void* const* peers = nullptr,
                                   int n_peers = 0, bool peers_f16 = false);
// tcsl_cuda_prune_magnitude (prune.cu)
size_t prune_workspace_bytes(uint64_t count);
cudaError_t launch_prune(const uint16_t* a, uint64_t count, uint64_t cut, uint16_t* out, void* ws, size_t ws_bytes,
                         cudaStream_t s);
cudaError_t launch_rebase(const uint32_t* off, uint32_t t0, uint32_t t1, uint32_t* out, cudaStream_t s);
cudaError_t launch_gen_synthetic(uint16_t* w, uint64_t count, double beta, uint64_t seed, cudaStream_t s);

// Tensor-core SpMM (TileConfig {128, 64}).
struct SpmmPlan {
  int n;          // true N
  int n_pad;      // MMA N (8, 16, 32, 64, 128, 192, 256)
  int split;      // k splits
  int units;      // tiles_m * split
  int grid;       // persistent CTAs
  size_t smem;    // dynamic smem bytes
};
int spmm_sm100_plan(uint32_t m, uint32_t k, int n, int split_k, SpmmPlan* plan);
struct Epilogue {
  const float* bias = nullptr;  // per row
  int act = 0;                  // TCSL_ACT_*
  uint16_t* out16 = nullptr;    // binary16 output instead of fp32
  void* const* peers = nullptr;  // > 0 peers: Y rows go to every peers[g] (device array) instead of out
  int n_peers = 0;
  bool peers_f16 = false;        // the peers' dtype (binary16 or fp32)
};
cudaError_t launch_spmm_sm100(const SpmmPlan& plan, const uint32_t* off, const uint32_t* ent,
                              uint64_t n_entries, uint32_t m, uint32_t k, const uint16_t* x, int ldx,
                              float* out, int* err, cudaStream_t s, const Epilogue& epi = Epilogue{});
int num_sms();

}  // namespace tcslk
