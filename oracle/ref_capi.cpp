// extern "C" veneer over the UNMODIFIED reference library — TEST/BASELINE ONLY.
//
// oracle/Makefile compiles /root/reference/proj/src/*.cpp in place (read-only,
// never copied) together with this file into oracle/_ref/libtcsl_ref.so, using
// the reference's own Release flags (proj/CMakeLists.txt:3-13). tests/ use it
// to pin the C restatement (tcsl_oracle.c) and the GPU path; bench.py's
// `--impl reference` arm and `cpu_baseline` time tcsl::spmm through it.
//
// Threading: the reference is single-threaded. ref_spmm_run
// splits the row blocks into independent row shards (each shard's Tiled-CSL
// is exactly `encode` of that row block) and
// calls the reference tcsl::spmm on each shard in its own std::thread. The
// per-row arithmetic is untouched, so the bits equal the 1-thread call.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>
#include <vector>

#include "tcsl/engine.hpp"
#include "tcsl/gemm.hpp"
#include "tcsl/matrix.hpp"
#include "tcsl/tcsl_format.hpp"

namespace {

int status_of(const tcsl::Error& e) { return static_cast<int>(e.code()) + 1; }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const tcsl::Error& e) {
    return status_of(e);
  } catch (const std::bad_alloc&) {
    return 100;
  } catch (...) {
    return 101;
  }
}

tcsl::HalfMatrix half_matrix(const std::uint16_t* p, int rows, int cols) {
  tcsl::HalfMatrix m(rows, cols);
  if (rows > 0 && cols > 0) std::memcpy(m.data(), p, sizeof(std::uint16_t) * m.size());
  return m;
}

tcsl::TcslMatrix tcsl_from(const std::uint32_t* offsets, const std::uint32_t* entries, std::uint64_t n_entries,
                           std::uint32_t m, std::uint32_t k, int m_tb, int k_tb, int reordered) {
  tcsl::TcslMatrix t;
  t.m = m;
  t.k = k;
  t.cfg.m_tb = m_tb;
  t.cfg.k_tb = k_tb;
  t.reordered = reordered != 0;
  t.tile_offsets.assign(offsets, offsets + t.num_tiles() + 1);
  t.entries.resize(n_entries);
  if (n_entries) std::memcpy(t.entries.data(), entries, 4 * n_entries);
  return t;
}

struct SpmmPlan {
  std::vector<tcsl::TcslMatrix> shards;
  std::vector<std::uint32_t> row0;
};

}  // namespace

extern "C" {

int ref_gen_random_sparse(int rows, int cols, double beta, std::uint64_t seed, std::uint16_t* out) {
  return guarded([&] {
    const tcsl::HalfMatrix a = tcsl::gen_random_sparse(rows, cols, beta, seed);
    std::memcpy(out, a.data(), sizeof(std::uint16_t) * a.size());
  });
}

// Encodes and returns an opaque handle; read it back with ref_tcsl_* below.
int ref_encode(const std::uint16_t* a, int rows, int cols, int m_tb, int k_tb, int reorder, void** handle) {
  return guarded([&] {
    tcsl::TileConfig cfg;
    cfg.m_tb = m_tb;
    cfg.k_tb = k_tb;
    auto t = std::make_unique<tcsl::TcslMatrix>(tcsl::encode(half_matrix(a, rows, cols), cfg, reorder != 0));
    *handle = t.release();
  });
}

std::uint32_t ref_tcsl_num_tiles(void* h) { return static_cast<tcsl::TcslMatrix*>(h)->num_tiles(); }
std::uint64_t ref_tcsl_num_entries(void* h) { return static_cast<tcsl::TcslMatrix*>(h)->entries.size(); }
void ref_tcsl_copy(void* h, std::uint32_t* offsets, std::uint32_t* entries) {
  auto* t = static_cast<tcsl::TcslMatrix*>(h);
  std::memcpy(offsets, t->tile_offsets.data(), 4 * t->tile_offsets.size());
  if (!t->entries.empty()) std::memcpy(entries, t->entries.data(), 4 * t->entries.size());
}
void ref_tcsl_free(void* h) { delete static_cast<tcsl::TcslMatrix*>(h); }

int ref_serialize_fnv(void* h, std::uint64_t* hash, std::uint64_t* size) {
  return guarded([&] {
    const auto bytes = tcsl::serialize_tcsl(*static_cast<tcsl::TcslMatrix*>(h));
    std::uint64_t x = 1469598103934665603ull;
    for (std::uint8_t c : bytes) {
      x ^= c;
      x *= 1099511628211ull;
    }
    *hash = x;
    *size = bytes.size();
  });
}

int ref_decode(const std::uint32_t* offsets, const std::uint32_t* entries, std::uint64_t n_entries, std::uint32_t m,
               std::uint32_t k, int m_tb, int k_tb, std::uint16_t* out) {
  return guarded([&] {
    const tcsl::HalfMatrix d = tcsl::decode(tcsl_from(offsets, entries, n_entries, m, k, m_tb, k_tb, 0));
    std::memcpy(out, d.data(), sizeof(std::uint16_t) * d.size());
  });
}

int ref_dense_gemm(const std::uint16_t* a, int m, int k, const std::uint16_t* b, int n, int m_tb, int k_tb,
                   float* y) {
  return guarded([&] {
    tcsl::TileConfig cfg;
    cfg.m_tb = m_tb;
    cfg.k_tb = k_tb;
    const tcsl::FloatMatrix c = tcsl::dense_gemm_ref(half_matrix(a, m, k), half_matrix(b, k, n), cfg);
    std::memcpy(y, c.data(), sizeof(float) * c.size());
  });
}

// Builds row shards (no arithmetic) for ref_spmm_run.
int ref_spmm_prepare(const std::uint32_t* offsets, const std::uint32_t* entries, std::uint64_t n_entries,
                     std::uint32_t m, std::uint32_t k, int m_tb, int k_tb, int nshards, void** plan) {
  return guarded([&] {
    auto p = std::make_unique<SpmmPlan>();
    const int tm = tcsl::div_up(m, m_tb), tk = tcsl::div_up(k, k_tb);
    if (nshards < 1) nshards = 1;
    if (nshards > tm) nshards = tm;
    for (int s = 0; s < nshards; ++s) {
      const int rb0 = static_cast<int>(static_cast<std::int64_t>(tm) * s / nshards);
      const int rb1 = static_cast<int>(static_cast<std::int64_t>(tm) * (s + 1) / nshards);
      const std::uint32_t t0 = static_cast<std::uint32_t>(rb0) * tk, t1 = static_cast<std::uint32_t>(rb1) * tk;
      const std::uint32_t r0 = static_cast<std::uint32_t>(rb0) * m_tb;
      const std::uint32_t r1 = std::min<std::uint32_t>(m, static_cast<std::uint32_t>(rb1) * m_tb);
      tcsl::TcslMatrix sh;
      sh.m = r1 - r0;
      sh.k = k;
      sh.cfg.m_tb = m_tb;
      sh.cfg.k_tb = k_tb;
      sh.tile_offsets.resize(t1 - t0 + 1);
      for (std::uint32_t t = t0; t <= t1; ++t) sh.tile_offsets[t - t0] = offsets[t] - offsets[t0];
      sh.entries.resize(offsets[t1] - offsets[t0]);
      if (!sh.entries.empty())
        std::memcpy(sh.entries.data(), entries + offsets[t0], 4 * sh.entries.size());
      p->shards.push_back(std::move(sh));
      p->row0.push_back(r0);
    }
    (void)n_entries;
    *plan = p.release();
  });
}

void ref_spmm_free(void* plan) { delete static_cast<SpmmPlan*>(plan); }

// Runs the reference tcsl::spmm on every shard, one std::thread per shard.
int ref_spmm_run(void* plan, const std::uint16_t* b, int k, int n, float* y) {
  auto* p = static_cast<SpmmPlan*>(plan);
  const tcsl::HalfMatrix bm = half_matrix(b, k, n);
  std::vector<int> status(p->shards.size(), 0);
  auto work = [&](std::size_t s) {
    status[s] = guarded([&] {
      const tcsl::FloatMatrix c = tcsl::spmm(p->shards[s], bm);
      std::memcpy(y + static_cast<std::size_t>(p->row0[s]) * n, c.data(), sizeof(float) * c.size());
    });
  };
  if (p->shards.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (std::size_t s = 0; s < p->shards.size(); ++s) th.emplace_back(work, s);
    for (auto& t : th) t.join();
  }
  for (int s : status)
    if (s) return s;
  return 0;
}

}  // extern "C"
