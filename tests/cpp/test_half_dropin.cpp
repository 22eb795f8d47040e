// Host-only checks of the drop-in's binary16 conversions (include/tcsl/half.hpp,
// host/support.cpp), the same cases as the reference's proj/tests/test_half.cpp:
// spot values (:19-37), canonical NaN (:39-47), overflow / tie boundaries
// (:49-66), every binary16 value decoded exactly and round-tripped (:68-87), a
// strided sweep of binary32 narrowing (:89-101) and every representable
// midpoint (:103-123). The independent oracle below works on doubles with
// std::nearbyint (round-half-even in the default rounding mode), not on bits.
// Needs no GPU. Exit code 0 = all checks passed.
#include <bit>
#include <cfenv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <limits>

#include "tcsl/half.hpp"

using tcsl::f16_from_f32;
using tcsl::f32_from_f16;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

namespace indep {

// binary16 value of bit pattern h as a double (exact), NaN for NaNs.
double value(std::uint16_t h) {
  const int e = (h >> 10) & 31, f = h & 1023;
  const double s = (h & 0x8000) ? -1.0 : 1.0;
  if (e == 31) return f ? std::numeric_limits<double>::quiet_NaN() : s * std::numeric_limits<double>::infinity();
  if (e == 0) return s * std::ldexp(static_cast<double>(f), -24);
  return s * std::ldexp(static_cast<double>(1024 + f), e - 25);
}

// Round-to-nearest-even narrowing: scale by the quantum of the target binade and
// let nearbyint (ties to even) pick the integer multiple.
std::uint16_t narrow(float v) {
  if (std::isnan(v)) return 0x7E00;
  const std::uint16_t sign = std::signbit(v) ? 0x8000 : 0;
  const double a = std::fabs(static_cast<double>(v));
  if (std::isinf(a)) return sign | 0x7C00;
  // quantum: 2^-24 below 2^-14 (subnormals), else 2^(floor(log2 a) - 10)
  int q = -24;
  if (a >= std::ldexp(1.0, -14)) q = static_cast<int>(std::floor(std::log2(a))) - 10;
  if (a >= std::ldexp(1.0, -14) && std::ldexp(1.0, q + 10) > a) --q;  // log2 rounding guard
  if (a >= std::ldexp(1.0, -14) && std::ldexp(1.0, q + 11) <= a) ++q;
  const double units = std::nearbyint(std::ldexp(a, -q));
  const double r = std::ldexp(units, q);
  if (r >= 65520.0) return sign | 0x7C00;  // rounds past the largest finite value
  if (r == 0.0) return sign;
  // encode r (exactly representable now)
  if (r < std::ldexp(1.0, -14)) return sign | static_cast<std::uint16_t>(std::ldexp(r, 24));
  int e = static_cast<int>(std::floor(std::log2(r)));
  if (std::ldexp(1.0, e) > r) --e;
  if (std::ldexp(1.0, e + 1) <= r) ++e;
  const int man = static_cast<int>(std::ldexp(r, 10 - e)) - 1024;
  return sign | static_cast<std::uint16_t>(((e + 15) << 10) | man);
}

}  // namespace indep

static float bits32(std::uint32_t u) { return std::bit_cast<float>(u); }

int main() {
  std::fesetround(FE_TONEAREST);
  // spot values
  CHECK(f16_from_f32(0.0f) == 0x0000);
  CHECK(f16_from_f32(-0.0f) == 0x8000);
  CHECK(f16_from_f32(1.0f) == 0x3C00);
  CHECK(f16_from_f32(-1.0f) == 0xBC00);
  CHECK(f16_from_f32(0.5f) == 0x3800);
  CHECK(f16_from_f32(65504.0f) == 0x7BFF);
  CHECK(f16_from_f32(std::ldexp(1.0f, -24)) == 0x0001);
  CHECK(f16_from_f32(std::ldexp(1.0f, -14)) == 0x0400);
  CHECK(f16_from_f32(std::numeric_limits<float>::infinity()) == 0x7C00);
  CHECK(f16_from_f32(-std::numeric_limits<float>::infinity()) == 0xFC00);
  CHECK(f32_from_f16(0x3C00) == 1.0f);
  CHECK(f32_from_f16(0x7BFF) == 65504.0f);
  CHECK(f32_from_f16(0x0001) == std::ldexp(1.0f, -24));
  CHECK(std::bit_cast<std::uint32_t>(f32_from_f16(0x8000)) == 0x80000000u);
  // canonical NaN
  CHECK(f16_from_f32(std::numeric_limits<float>::quiet_NaN()) == 0x7E00);
  CHECK(f16_from_f32(-std::numeric_limits<float>::quiet_NaN()) == 0x7E00);
  CHECK(f16_from_f32(bits32(0x7F800001u)) == 0x7E00);
  CHECK(f16_from_f32(bits32(0xFFC12345u)) == 0x7E00);
  CHECK(std::isnan(f32_from_f16(0x7C01)) && std::isnan(f32_from_f16(0xFE00)) && std::isnan(f32_from_f16(0x7FFF)));
  // overflow and ties
  CHECK(f16_from_f32(65520.0f) == 0x7C00);
  CHECK(f16_from_f32(std::nextafterf(65520.0f, 0.0f)) == 0x7BFF);
  CHECK(f16_from_f32(-65520.0f) == 0xFC00);
  CHECK(f16_from_f32(1e30f) == 0x7C00);
  CHECK(f16_from_f32(std::ldexp(1.0f, -25)) == 0x0000);
  CHECK(f16_from_f32(-std::ldexp(1.0f, -25)) == 0x8000);
  CHECK(f16_from_f32(std::nextafterf(std::ldexp(1.0f, -25), 1.0f)) == 0x0001);
  CHECK(f16_from_f32(std::ldexp(3.0f, -25)) == 0x0002);
  CHECK(f16_from_f32(std::ldexp(1.0f, -26)) == 0x0000);

  // every binary16 value widens exactly and narrows back to itself
  int bad = 0;
  for (std::uint32_t h = 0; h <= 0xFFFF; ++h) {
    const auto hb = static_cast<tcsl::HalfBits>(h);
    const float got = f32_from_f16(hb);
    const double want = indep::value(hb);
    bool ok;
    if (tcsl::f16_is_nan(hb))
      ok = std::isnan(got);
    else
      ok = static_cast<double>(got) == want && std::signbit(got) == std::signbit(want) && f16_from_f32(got) == hb;
    bad += !ok;
  }
  CHECK(bad == 0);

  // strided binary32 sweep against the independent oracle
  bad = 0;
  for (std::uint64_t u = 0; u <= 0xFFFFFFFFull; u += 997) {
    const float f = bits32(static_cast<std::uint32_t>(u));
    bad += f16_from_f32(f) != indep::narrow(f);
  }
  CHECK(bad == 0);

  // every representable midpoint ties to even, its neighbours round away from it
  bad = 0;
  for (std::uint32_t h = 0; h + 1 <= 0x7BFF; ++h) {
    const double lo = f32_from_f16(static_cast<tcsl::HalfBits>(h)), hi = f32_from_f16(static_cast<tcsl::HalfBits>(h + 1));
    const float mid = static_cast<float>((lo + hi) / 2.0);
    const std::uint16_t even = (h & 1) ? static_cast<std::uint16_t>(h + 1) : static_cast<std::uint16_t>(h);
    bool ok = f16_from_f32(mid) == even && f16_from_f32(std::nextafterf(mid, -1e30f)) == h &&
              f16_from_f32(std::nextafterf(mid, 1e30f)) == h + 1 && f16_from_f32(-mid) == (even | 0x8000);
    bad += !ok;
  }
  CHECK(bad == 0);

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
