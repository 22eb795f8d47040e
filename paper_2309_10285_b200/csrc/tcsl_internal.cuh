// Shared declarations between the kernel translation units and the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/tcsl_cuda.h"

namespace tcslk {

constexpr int kGroup = 32;  // entries per group (proj/include/tcsl/tcsl_format.hpp:12)

// Device error codes (stored in *dErr; first error wins).
__device__ __forceinline__ void raise_dev(int* err, int status) {
  if (err) atomicCAS(err, 0, status);
}

inline int div_up_i(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Host launchers (return cudaError_t as int, 0 on success).
cudaError_t launch_encode_count(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb,
                                uint32_t* counts, cudaStream_t s);
cudaError_t launch_encode_emit(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                               const uint32_t* offsets, uint32_t* entries, int* err, cudaStream_t s);
cudaError_t launch_decode(const uint32_t* off, const uint32_t* ent, uint64_t n_entries, uint32_t m,
                          uint32_t k, int m_tb, int k_tb, uint16_t* out, int* err, int strict, cudaStream_t s);
size_t encode_scan_temp_bytes(uint32_t tiles);
cudaError_t launch_encode_scan(uint32_t* counts_in, uint32_t* offsets, uint32_t tiles, void* temp,
                               size_t temp_bytes, cudaStream_t s);
cudaError_t launch_validate(const uint32_t* off, uint64_t n_entries, uint32_t tiles, int* err,
                            cudaStream_t s);
cudaError_t launch_dense_gemm_exact(const uint16_t* a, uint32_t m, uint32_t k, const uint16_t* x, int n,
                                    float* y, cudaStream_t s);
cudaError_t launch_splitk_reduce(const float* p, int split, size_t count, float* y, cudaStream_t s);
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
cudaError_t launch_spmm_sm100(const SpmmPlan& plan, const uint32_t* off, const uint32_t* ent,
                              uint64_t n_entries, uint32_t m, uint32_t k, const uint16_t* x, int ldx,
                              float* out, int* err, cudaStream_t s);
int num_sms();

}  // namespace tcslk
