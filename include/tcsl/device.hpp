// Weights-resident form of the drop-in (an addition to the reference API, which is
// value-in / value-out: proj/include/tcsl/engine.hpp:14-18). tcsl::spmm uploads the
// Tiled-CSL matrix on every call; a DeviceMatrix uploads it once (and runs the
// one-pass device check of the tensor-core preconditions once), so serving-style
// callers pay only X up and Y down per call.
#pragma once

#include <cstdint>

#include "tcsl/engine.hpp"
#include "tcsl/tcsl_format.hpp"

namespace tcsl {

class DeviceMatrix {
 public:
  explicit DeviceMatrix(const TcslMatrix& t);  // errors as tcsl::spmm's argument checks
  ~DeviceMatrix();
  DeviceMatrix(const DeviceMatrix&) = delete;
  DeviceMatrix& operator=(const DeviceMatrix&) = delete;

  // Y = A x B, the semantics of tcsl::spmm(A, B, opt) (engine.cpp:27-78).
  FloatMatrix spmm(const HalfMatrix& b, const SpmmOptions& opt = {}) const;

  std::uint32_t rows() const { return m_; }
  std::uint32_t cols() const { return k_; }
  std::uint64_t entries() const { return n_entries_; }
  // false when the matrix needs the bit-exact path (repeated locations inside a
  // tile, or tile spans that are not whole 32-entry groups)
  bool tensor_core_ready() const { return tc_ready_; }

 private:
  std::uint32_t m_ = 0, k_ = 0;
  TileConfig cfg_;
  std::uint64_t n_entries_ = 0;
  void* off_ = nullptr;
  void* ent_ = nullptr;
  bool tc_ready_ = false;
};

}  // namespace tcsl
