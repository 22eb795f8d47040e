// Host-side pieces of the tcsl API that carry no device work: error names,
// binary16 conversions, tile-config checks and synthetic inputs.
// Behaviour follows proj/src/{errors,half,matrix}.cpp (cited per function).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#include "tcsl/errors.hpp"
#include "tcsl/half.hpp"
#include "tcsl/matrix.hpp"
#include "tcsl_host.h"

namespace tcsl {

const char* errc_name(Errc c) {  // proj/src/errors.cpp:5-20
  static const char* const names[] = {"bad magic",        "unsupported version",  "bad header",
                                      "wrong dtype",      "truncated file",       "trailing data",
                                      "inconsistent offsets", "location out of range", "dimension mismatch",
                                      "invalid argument", "i/o failure"};
  const int i = static_cast<int>(c);
  return (i >= 0 && i < 11) ? names[i] : "error";
}

// proj/src/half.cpp:10-40. Finite values go through the compiler's IEEE
// binary16 conversion (round-to-nearest-even, overflow to inf); every NaN
// becomes the canonical quiet NaN.
HalfBits f16_from_f32(float v) {
  if (std::isnan(v)) return kHalfQuietNan;
  const _Float16 h = static_cast<_Float16>(v);
  HalfBits b;
  std::memcpy(&b, &h, sizeof b);
  return b;
}

// proj/src/half.cpp:42-66. Exact; inf/NaN keep their payload bits verbatim.
float f32_from_f16(HalfBits b) {
  if ((b & 0x7C00u) == 0x7C00u) {
    const std::uint32_t w = (static_cast<std::uint32_t>(b & 0x8000u) << 16) | 0x7F800000u |
                            (static_cast<std::uint32_t>(b & 0x03FFu) << 13);
    float f;
    std::memcpy(&f, &w, sizeof f);
    return f;
  }
  _Float16 h;
  std::memcpy(&h, &b, sizeof h);
  return static_cast<float>(h);
}

void TileConfig::validate() const {  // proj/src/matrix.cpp:11-18
  if (m_tb <= 0 || k_tb <= 0) raise(Errc::invalid_argument, "tile dims must be positive");
  if (m_tb % 8 || k_tb % 8) raise(Errc::invalid_argument, "tile dims must be multiples of 8");
  if (static_cast<long long>(m_tb) * k_tb > 65536) raise(Errc::invalid_argument, "tile locations must fit 16 bits");
  if (threads_per_block <= 0) raise(Errc::invalid_argument, "threads_per_block must be positive");
}

int tile_n_for(int n) { return n <= 8 ? 8 : n <= 16 ? 16 : n <= 64 ? 32 : 64; }  // proj/src/matrix.cpp:20-25

// proj/src/matrix.cpp:35-67: one mt19937_64 draw decides zero/non-zero for
// each position (selection sampling keeps the zero count exact); a second
// draw builds a non-zero value.
namespace {

void gen_into(std::int64_t total, double beta, std::uint64_t seed, std::uint16_t* dst) {
  std::int64_t zeros_left = std::clamp<std::int64_t>(std::llround(beta * static_cast<double>(total)), 0, total);
  std::mt19937_64 rng(seed);
  for (std::int64_t pos = 0; pos < total; ++pos) {
    const std::uint64_t unfilled = static_cast<std::uint64_t>(total - pos);
    if (rng() % unfilled < static_cast<std::uint64_t>(zeros_left)) {
      dst[pos] = kHalfPosZero;
      --zeros_left;
      continue;
    }
    const std::uint64_t bits = rng();
    const HalfBits mantissa = static_cast<HalfBits>(bits & 0x3FFu);
    const HalfBits exponent = static_cast<HalfBits>(13u + (bits >> 10) % 5u);
    const HalfBits sign = static_cast<HalfBits>((bits >> 63) << 15);
    dst[pos] = static_cast<HalfBits>(sign | (exponent << 10) | mantissa);
  }
}

}  // namespace

HalfMatrix gen_random_sparse(int rows, int cols, double beta, std::uint64_t seed) {
  if (rows <= 0 || cols <= 0) raise(Errc::invalid_argument, "matrix dims must be positive");
  if (!(beta >= 0.0 && beta <= 1.0)) raise(Errc::invalid_argument, "sparsity must be in [0, 1]");
  HalfMatrix out(rows, cols);
  gen_into(static_cast<std::int64_t>(rows) * cols, beta, seed, reinterpret_cast<std::uint16_t*>(out.data()));
  return out;
}

double sparsity(const HalfMatrix& a) {  // proj/src/matrix.cpp:102-109
  if (a.size() == 0) return 0.0;
  std::int64_t z = 0;
  for (std::int64_t i = 0; i < a.size(); ++i) z += f16_is_zero(bits_of(a.data()[i]));
  return static_cast<double>(z) / static_cast<double>(a.size());
}

HalfMatrix normalize_zeros(HalfMatrix a) {  // proj/src/matrix.cpp:111-116
  for (std::int64_t i = 0; i < a.size(); ++i) a.data()[i] = half_from_bits(f16_normalize_zero(bits_of(a.data()[i])));
  return a;
}

}  // namespace tcsl

// C entry point of the host library for bindings (include/tcsl_host.h).
extern "C" int tcsl_host_gen_random_sparse(int rows, int cols, double beta, std::uint64_t seed, std::uint16_t* out) {
  if (rows <= 0 || cols <= 0 || !out || !(beta >= 0.0 && beta <= 1.0)) return 10;  // Errc::invalid_argument + 1
  tcsl::gen_into(static_cast<std::int64_t>(rows) * cols, beta, seed, out);
  return 0;
}
