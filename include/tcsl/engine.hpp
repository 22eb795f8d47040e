// LSCD SpMM engine — drop-in for proj/include/tcsl/engine.hpp:9-25.
#pragma once

#include <vector>

#include "tcsl/tcsl_format.hpp"

namespace tcsl {

// Dense m_tb x k_tb reconstruction of one tile (host).
std::vector<HalfBits> extract_tile(const TcslMatrix& t, std::uint32_t tile);

// Y = A x B on the GPU. Default TileConfig {128,64}: tcgen05 tensor cores, fp32
// accumulate, within the north-star tolerance of the reference's serial fp32
// sum (SpmmOptions::exact switches to the bit-exact CUDA-core path, which every
// other TileConfig uses anyway). dimension_mismatch when a.k != b.rows().
struct SpmmOptions {
  int split_k = 0;     // 0 auto, 1 none, S > 1: S partial sums reduced in fixed order
  bool exact = false;  // bit-identical to the reference (dense_gemm_ref order)
};
FloatMatrix spmm(const TcslMatrix& a, const HalfMatrix& b);
FloatMatrix spmm(const TcslMatrix& a, const HalfMatrix& b, const SpmmOptions& opt);

// Registers per thread a kernel holding each tile's entries would need.
int reg_pressure(const TcslMatrix& t);
inline constexpr int kRegPressureWarnLimit = 64;

}  // namespace tcsl
