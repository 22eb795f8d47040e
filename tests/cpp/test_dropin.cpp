// Drop-in check of the C++ API (include/tcsl/*.hpp over the C-ABI), written
// against the same signatures and expectations as the reference's own tests
// (proj/tests/test_codec.cpp, test_engine.cpp, test_gemm.cpp, acceptance.cpp:60-64).
// Exit code 0 = all checks passed. Needs a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <optional>
#include <random>
#include <string>

#include "tcsl/device.hpp"
#include "tcsl/engine.hpp"
#include "tcsl/gemm.hpp"
#include "tcsl/tcsl_format.hpp"

using namespace tcsl;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (cond) {                                                              \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                        \
  } while (0)

template <class F>
static std::optional<Errc> thrown(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.code();
  }
  return std::nullopt;
}

static std::uint64_t fnv1a(const std::vector<std::uint8_t>& b) {
  std::uint64_t h = 1469598103934665603ull;
  for (std::uint8_t c : b) h = (h ^ c) * 1099511628211ull;
  return h;
}

static bool same(const HalfMatrix& a, const HalfMatrix& b) {
  return a.rows() == b.rows() && a.cols() == b.cols() && std::memcmp(a.data(), b.data(), 2 * a.size()) == 0;
}
static bool same(const FloatMatrix& a, const FloatMatrix& b) {
  return a.rows() == b.rows() && a.cols() == b.cols() && std::memcmp(a.data(), b.data(), 4 * a.size()) == 0;
}

int main() {
  // golden artifacts (acceptance.cpp:60-64)
  struct G {
    int r, c;
    double beta;
    std::uint64_t seed;
    bool reorder;
    std::uint64_t hash;
  } golden[] = {{128, 64, 0.3, 11, true, 0xa57f18792a5f0447ull},
                {256, 128, 0.8, 22, true, 0x2a290613b42e2457ull},
                {130, 70, 0.5, 33, false, 0xf68ef9afd7dea93aull}};
  for (const G& g : golden) {
    const HalfMatrix a = gen_random_sparse(g.r, g.c, g.beta, g.seed);
    const TcslMatrix t = encode(a, {}, g.reorder);
    CHECK(fnv1a(serialize_tcsl(t)) == g.hash);
    CHECK(same(decode(t), normalize_zeros(a)));
    CHECK(serialize_tcsl(deserialize_tcsl(serialize_tcsl(t))) == serialize_tcsl(t));
  }

  {  // worked example and greedy order (test_codec.cpp:48-84)
    HalfMatrix a(128, 64);
    a.setZero();
    a(0, 0) = Eigen::half(1.0f);
    a(1, 2) = Eigen::half(2.0f);
    const TcslMatrix t = encode(a);
    CHECK(t.tile_offsets == (std::vector<std::uint32_t>{0, 32}));
    CHECK(t.entries[0].raw == 0x3C000000u && t.entries[1].raw == 0x40000042u);
    for (int i = 2; i < 32; ++i) CHECK(t.entries[i].value_bits() == 0 && t.entries[i].location() == i - 1);
    HalfMatrix b(128, 64);
    b.setZero();
    b(0, 0) = Eigen::half(1.0f);
    b(1, 0) = Eigen::half(2.0f);
    b(1, 1) = Eigen::half(3.0f);
    const TcslMatrix r = encode(b, {}, true);
    CHECK(r.entries[0].location() == 64 && r.entries[1].location() == 0 && r.entries[2].location() == 65);
  }

  {  // round trips incl. -0 and fringes (test_codec.cpp:98-138)
    std::mt19937_64 rng(88);
    for (int it = 0; it < 12; ++it) {
      const int m = 1 + static_cast<int>(rng() % 300), k = 1 + static_cast<int>(rng() % 150);
      HalfMatrix a = gen_random_sparse(m, k, static_cast<double>(rng() % 1001) / 1000.0, rng());
      if (a.size() > 3) a.data()[2] = half_from_bits(kHalfNegZero);
      const TcslMatrix t = encode(a, {}, it % 2 == 0);
      CHECK(same(decode(t), normalize_zeros(a)));
    }
  }

  {  // error classes (test_codec.cpp:242-273, test_engine.cpp:95-99)
    CHECK(thrown([] { encode(HalfMatrix{}); }) == Errc::invalid_argument);
    CHECK(thrown([] { encode(gen_random_sparse(16, 16, 0.5, 2), TileConfig{12, 8, 32}); }) == Errc::invalid_argument);
    HalfMatrix a(128, 64);
    a.setZero();
    a(0, 0) = Eigen::half(1.0f);
    TcslMatrix bad = encode(a);
    bad.entries[1] = TcslEntry::make(0, 8192);
    CHECK(thrown([&] { decode(bad); }) == Errc::location_out_of_range);
    const TcslMatrix t = encode(gen_random_sparse(32, 16, 0.5, 1), TileConfig{16, 8, 32});
    CHECK(thrown([&] { spmm(t, gen_random_sparse(17, 4, 0.0, 2)); }) == Errc::dimension_mismatch);
    std::vector<std::uint8_t> buf = serialize_tcsl(encode(gen_random_sparse(130, 70, 0.5, 9)));
    buf[0] = 'Y';
    CHECK(thrown([&] { deserialize_tcsl(buf); }) == Errc::bad_magic);
  }

  {  // spmm: bit-exact mode and non-default tiles (test_engine.cpp:64-93)
    std::mt19937_64 rng(77);
    const TileConfig small{16, 8, 32};
    for (int it = 0; it < 10; ++it) {
      const int m = 1 + static_cast<int>(rng() % 50), k = 1 + static_cast<int>(rng() % 40), n = 1 + static_cast<int>(rng() % 12);
      const HalfMatrix a = gen_random_sparse(m, k, static_cast<double>(rng() % 1001) / 1000.0, rng());
      const HalfMatrix b = gen_random_sparse(k, n, 0.1, rng());
      const TcslMatrix t = encode(a, small, it % 2 == 0);
      CHECK(same(spmm(t, b), dense_gemm_ref(decode(t), b, small)));
    }
    const HalfMatrix a = gen_random_sparse(256, 128, 0.8, rng());
    const HalfMatrix b = gen_random_sparse(128, 16, 0.0, rng());
    const TcslMatrix t = encode(a);
    const FloatMatrix want = dense_gemm_ref(decode(t), b);
    CHECK(same(spmm(t, b, SpmmOptions{0, true}), want));
    // tensor-core path: north-star tolerance against the exact result
    const FloatMatrix got = spmm(t, b);
    double num = 0, den = 0;
    bool elem_ok = true;
    const HalfMatrix aa = [&] {
      HalfMatrix c = a;
      for (std::int64_t i = 0; i < c.size(); ++i) c.data()[i] = half_from_bits(bits_of(c.data()[i]) & 0x7FFF);
      return c;
    }();
    const HalfMatrix bb = [&] {
      HalfMatrix c = b;
      for (std::int64_t i = 0; i < c.size(); ++i) c.data()[i] = half_from_bits(bits_of(c.data()[i]) & 0x7FFF);
      return c;
    }();
    const FloatMatrix bound = dense_gemm_ref(aa, bb);
    for (std::int64_t i = 0; i < got.size(); ++i) {
      const double d = double(got.data()[i]) - double(want.data()[i]);
      num += d * d;
      den += double(want.data()[i]) * want.data()[i];
      elem_ok = elem_ok && std::fabs(d) <= std::ldexp(double(bound.data()[i]), -10);
    }
    CHECK(elem_ok);
    CHECK(std::sqrt(num / den) <= 1e-3);
    CHECK(reg_pressure(encode(gen_random_sparse(128, 64, 0.0, 3))) == 64);  // test_engine.cpp:101-113
  }

  {  // lenient spans (engine.cpp:8-14 only checks per-tile spans): accepted, bit-exact
    const TileConfig cfg{16, 8, 32};
    const HalfMatrix a = gen_random_sparse(32, 16, 0.5, 4);
    TcslMatrix t = encode(a, cfg, false);
    TcslMatrix loose = t;  // drop the +0.0 padding of tile 0 -> count not a multiple of 32
    const std::uint32_t pad = [&] {
      std::uint32_t p = 0;
      for (std::uint32_t e = t.tile_offsets[0]; e < t.tile_offsets[1]; ++e) p += t.entries[e].value_bits() == 0;
      return p;
    }();
    if (pad > 0 && pad < 32) {
      loose.entries.erase(loose.entries.begin() + (t.tile_offsets[1] - pad), loose.entries.begin() + t.tile_offsets[1]);
      for (std::size_t i = 1; i < loose.tile_offsets.size(); ++i) loose.tile_offsets[i] -= pad;
      const HalfMatrix b = gen_random_sparse(16, 5, 0.0, 5);
      CHECK(same(spmm(loose, b), spmm(t, b)));
    }
  }

  {  // prune_magnitude on the GPU (proj/tests/test_matrix.cpp:54-104)
    HalfMatrix a(2, 2);
    a(0, 0) = Eigen::half(1.0f);
    a(0, 1) = Eigen::half(-4.0f);
    a(1, 0) = Eigen::half(2.0f);
    a(1, 1) = Eigen::half(3.0f);
    const HalfMatrix p = prune_magnitude(a, 0.5);
    CHECK(bits_of(p(0, 0)) == 0x0000 && bits_of(p(0, 1)) == 0xC400 && bits_of(p(1, 0)) == 0x0000 &&
          bits_of(p(1, 1)) == 0x4200);
    HalfMatrix t(1, 4);
    for (int j = 0; j < 4; ++j) t(0, j) = Eigen::half(2.0f);
    const HalfMatrix q = prune_magnitude(t, 0.5);
    CHECK(bits_of(q(0, 0)) == 0x4000 && bits_of(q(0, 1)) == 0x4000 && bits_of(q(0, 2)) == 0 && bits_of(q(0, 3)) == 0);
    CHECK(thrown([&] { prune_magnitude(t, 1.5); }) == Errc::invalid_argument);
    HalfMatrix n(1, 4);
    n(0, 0) = half_from_bits(kHalfQuietNan);
    n(0, 1) = Eigen::half(1.0f);
    n(0, 2) = Eigen::half(2.0f);
    n(0, 3) = Eigen::half(3.0f);
    const HalfMatrix pn = prune_magnitude(n, 0.5);
    CHECK(f16_is_nan(bits_of(pn(0, 0))) && bits_of(pn(0, 1)) == 0 && bits_of(pn(0, 2)) == 0 && bits_of(pn(0, 3)) == 0x4200);
  }

  {  // a location repeated inside a tile: last writer wins, like extract_tile (engine.cpp:17-22)
    const HalfMatrix a = gen_random_sparse(256, 128, 0.7, 31);
    TcslMatrix t = encode(a);
    for (std::uint32_t e = t.tile_offsets[0] + 1; e < t.tile_offsets[1]; e += 3)
      t.entries[e] = TcslEntry::make(t.entries[e].value_bits(), t.entries[e - 1].location());
    const HalfMatrix b = gen_random_sparse(128, 16, 0.0, 32);
    const FloatMatrix want = dense_gemm_ref(decode(t), b);
    CHECK(same(spmm(t, b), want));  // routed to the bit-exact path
    HalfMatrix dense(256, 128);
    dense.setZero();
    for (std::uint32_t tile = 0; tile < t.num_tiles(); ++tile) {
      const std::vector<HalfBits> d = extract_tile(t, tile);
      const int r0 = static_cast<int>(tile) / t.tiles_k() * 128, c0 = static_cast<int>(tile) % t.tiles_k() * 64;
      for (int x = 0; x < 128; ++x)
        for (int y = 0; y < 64; ++y) dense(r0 + x, c0 + y) = half_from_bits(d[static_cast<std::size_t>(x) * 64 + y]);
    }
    CHECK(same(decode(t), dense));
  }

  {  // weights-resident handle: the same bits as tcsl::spmm, call after call
    const HalfMatrix a = gen_random_sparse(640, 1024, 0.8, 41);
    const TcslMatrix t = encode(a);
    const DeviceMatrix dm(t);
    CHECK(dm.rows() == 640 && dm.cols() == 1024 && dm.entries() == t.entries.size() && dm.tensor_core_ready());
    for (int n : {8, 24, 64}) {
      const HalfMatrix b = gen_random_sparse(1024, n, 0.0, 42 + n);
      CHECK(same(dm.spmm(b), spmm(t, b)));
      CHECK(same(dm.spmm(b, SpmmOptions{3, false}), spmm(t, b, SpmmOptions{3, false})));
      CHECK(same(dm.spmm(b, SpmmOptions{0, true}), dense_gemm_ref(decode(t), b)));
    }
    CHECK(thrown([&] { (void)dm.spmm(gen_random_sparse(1000, 8, 0.0, 2)); }) == Errc::dimension_mismatch);
    TcslMatrix dup = t;  // a repeated location: the handle routes every call to the bit-exact path
    dup.entries[1] = TcslEntry::make(dup.entries[1].value_bits(), dup.entries[0].location());
    const DeviceMatrix dd(dup);
    CHECK(!dd.tensor_core_ready());
    const HalfMatrix b = gen_random_sparse(1024, 16, 0.0, 43);
    CHECK(same(dd.spmm(b), dense_gemm_ref(decode(dup), b)));
  }

  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
