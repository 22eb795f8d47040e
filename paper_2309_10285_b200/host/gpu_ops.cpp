// Hot-path entry points of the tcsl API, executed on the GPU through the
// C-ABI (include/tcsl_cuda.h). Host arrays are staged through a per-thread
// cache of device buffers, so repeated calls do not re-allocate.
//   encode        proj/src/tcsl_format.cpp:36-124   -> tcsl_cuda_encode_count/emit
//   decode        proj/src/tcsl_format.cpp:126-155  -> tcsl_cuda_decode
//   spmm          proj/src/engine.cpp:27-78         -> tcsl_cuda_spmm / _exact
//   dense_gemm_ref proj/src/gemm.cpp:7-44           -> tcsl_cuda_spmm_exact on encode(A)
//   prune_magnitude proj/src/matrix.cpp:69-100      -> tcsl_cuda_prune_magnitude (radix select)
//   extract_tile, reg_pressure (engine.cpp:8-25, 80-91) stay on the host (O(entries of a tile)).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "tcsl/device.hpp"
#include "tcsl/engine.hpp"
#include "tcsl/gemm.hpp"
#include "tcsl/tcsl_format.hpp"
#include "tcsl_cuda.h"

namespace tcsl {

namespace {

void check(int status, const char* what) {
  if (status == TCSL_STATUS_OK) return;
  if (status >= 1 && status <= 11) raise(static_cast<Errc>(status - 1), what);
  throw CudaError(std::string(what) + ": " + tcsl_cuda_status_string(status) + " " + tcsl_cuda_last_cuda_error());
}

// Grow-only device scratch buffers, one set per host thread.
class DeviceSlot {
 public:
  ~DeviceSlot() { tcsl_cuda_free(ptr_); }
  void* get(std::size_t bytes) {
    if (bytes > cap_) {
      tcsl_cuda_free(ptr_);
      ptr_ = nullptr;
      cap_ = 0;
      check(tcsl_cuda_malloc(&ptr_, bytes), "device allocation");
      cap_ = bytes;
    }
    return ptr_;
  }

 private:
  void* ptr_ = nullptr;
  std::size_t cap_ = 0;
};

struct Scratch {
  DeviceSlot dense, offsets, entries, x, y, ws, err, flags;
};

Scratch& scratch() {
  thread_local Scratch s;
  return s;
}

int* fresh_error_word() {
  int* err = static_cast<int*>(scratch().err.get(sizeof(int)));
  check(tcsl_cuda_memset(err, 0, sizeof(int), nullptr), "memset");
  return err;
}

void collect_errors(int* err, const char* what) { check(tcsl_cuda_read_error(err, nullptr), what); }

struct DeviceTcsl {
  const std::uint32_t* off;
  const std::uint32_t* ent;
};

DeviceTcsl upload(const TcslMatrix& t) {
  Scratch& s = scratch();
  auto* off = static_cast<std::uint32_t*>(s.offsets.get(4 * std::max<std::size_t>(t.tile_offsets.size(), 1)));
  auto* ent = static_cast<std::uint32_t*>(s.entries.get(4 * std::max<std::size_t>(t.entries.size(), 1)));
  check(tcsl_cuda_memcpy_h2d(off, t.tile_offsets.data(), 4 * t.tile_offsets.size(), nullptr), "upload offsets");
  check(tcsl_cuda_memcpy_h2d(ent, t.entries.data(), 4 * t.entries.size(), nullptr), "upload entries");
  return {off, ent};
}

const std::uint16_t* upload_half(DeviceSlot& slot, const HalfMatrix& a) {
  auto* d = static_cast<std::uint16_t*>(slot.get(2 * std::max<std::size_t>(static_cast<std::size_t>(a.size()), 1)));
  check(tcsl_cuda_memcpy_h2d(d, a.data(), 2 * static_cast<std::size_t>(a.size()), nullptr), "upload");
  return d;
}

}  // namespace

TcslMatrix encode(const HalfMatrix& a, const TileConfig& cfg, bool reorder) {
  cfg.validate();
  if (a.rows() <= 0 || a.cols() <= 0) raise(Errc::invalid_argument, "cannot encode an empty matrix");
  Scratch& s = scratch();
  const auto m = static_cast<std::uint32_t>(a.rows()), k = static_cast<std::uint32_t>(a.cols());
  const std::uint16_t* w = upload_half(s.dense, a);
  TcslMatrix t;
  t.m = m;
  t.k = k;
  t.cfg = cfg;
  t.reordered = reorder;
  const std::size_t n_off = static_cast<std::size_t>(t.num_tiles()) + 1;
  std::size_t ws_bytes = 0;
  check(tcsl_cuda_encode_workspace(m, k, cfg.m_tb, cfg.k_tb, &ws_bytes), "encode");
  auto* off = static_cast<std::uint32_t*>(s.offsets.get(4 * n_off));
  void* ws = s.ws.get(ws_bytes);
  check(tcsl_cuda_encode_count(w, m, k, cfg.m_tb, cfg.k_tb, off, ws, ws_bytes, nullptr), "encode");
  t.tile_offsets.resize(n_off);
  check(tcsl_cuda_memcpy_d2h(t.tile_offsets.data(), off, 4 * n_off, nullptr), "encode");
  check(tcsl_cuda_stream_sync(nullptr), "encode");
  const std::size_t n_ent = t.tile_offsets.back();
  auto* ent = static_cast<std::uint32_t*>(s.entries.get(4 * std::max<std::size_t>(n_ent, 1)));
  int* err = fresh_error_word();
  check(tcsl_cuda_encode_emit(w, m, k, cfg.m_tb, cfg.k_tb, reorder ? 1 : 0, off, ent, err, nullptr), "encode");
  t.entries.resize(n_ent);
  check(tcsl_cuda_memcpy_d2h(t.entries.data(), ent, 4 * n_ent, nullptr), "encode");
  collect_errors(err, "encode");
  return t;
}

HalfMatrix decode(const TcslMatrix& t) {
  t.cfg.validate();
  if (t.m == 0 || t.k == 0) raise(Errc::bad_header, "matrix dims must be positive");
  if (t.tile_offsets.size() != static_cast<std::size_t>(t.num_tiles()) + 1)
    raise(Errc::inconsistent_offsets, "offset table must have num_tiles+1 entries");
  const DeviceTcsl d = upload(t);
  Scratch& s = scratch();
  auto* out = static_cast<std::uint16_t*>(s.dense.get(2ull * t.m * t.k));
  int* err = fresh_error_word();
  check(tcsl_cuda_decode(d.off, d.ent, t.entries.size(), t.m, t.k, t.cfg.m_tb, t.cfg.k_tb, out, err, nullptr),
        "decode");
  HalfMatrix h(t.m, t.k);
  check(tcsl_cuda_memcpy_d2h(h.data(), out, 2ull * t.m * t.k, nullptr), "decode");
  collect_errors(err, "decode");
  return h;
}

std::vector<HalfBits> extract_tile(const TcslMatrix& t, std::uint32_t tile) {
  t.cfg.validate();
  if (tile >= t.num_tiles()) raise(Errc::invalid_argument, "tile index out of range");
  if (t.tile_offsets.size() != static_cast<std::size_t>(t.num_tiles()) + 1 ||
      t.tile_offsets[tile + 1] < t.tile_offsets[tile] || t.tile_offsets[tile + 1] > t.entries.size())
    raise(Errc::inconsistent_offsets, "offset table does not match entries");
  std::vector<HalfBits> dense(static_cast<std::size_t>(t.cfg.tile_elems()), kHalfPosZero);
  for (std::uint32_t e = t.tile_offsets[tile]; e < t.tile_offsets[tile + 1]; ++e) {
    const TcslEntry entry = t.entries[e];
    if (entry.location() >= t.cfg.tile_elems()) raise(Errc::location_out_of_range, "entry location exceeds tile size");
    dense[entry.location()] = f16_normalize_zero(entry.value_bits());
  }
  return dense;
}

FloatMatrix spmm(const TcslMatrix& a, const HalfMatrix& b) { return spmm(a, b, SpmmOptions{}); }

namespace {

// Argument checks of tcsl::spmm (engine.cpp:28-32) and extract_tile's per-tile
// spans (engine.cpp:11-14) on the host copy of the offsets.
void check_spmm_args(const TcslMatrix& a) {
  a.cfg.validate();
  if (a.tile_offsets.size() != static_cast<std::size_t>(a.num_tiles()) + 1)
    raise(Errc::inconsistent_offsets, "offset table does not match tile count");
  for (std::uint32_t t = 0; t < a.num_tiles(); ++t)  // the per-tile checks of extract_tile (engine.cpp:11-14)
    if (a.tile_offsets[t + 1] < a.tile_offsets[t] || a.tile_offsets[t + 1] > a.entries.size())
      raise(Errc::inconsistent_offsets, "offset table does not match entries");
}

// The reference accepts tiles whose spans are not whole 32-entry groups and
// locations repeated inside a tile (last writer wins, engine.cpp:8-25); the
// tensor-core decoders need neither. One device pass over the uploaded entries
// finds out; such matrices take the bit-exact path, which handles both.
bool tc_preconditions(const std::uint32_t* off, const std::uint32_t* ent, std::uint64_t n_entries, std::uint32_t m,
                      std::uint32_t k, const TileConfig& cfg) {
  if (cfg.m_tb != 128 || cfg.k_tb != 64) return false;
  auto* flags = static_cast<std::uint32_t*>(scratch().flags.get(sizeof(std::uint32_t)));
  check(tcsl_cuda_memset(flags, 0, sizeof(std::uint32_t), nullptr), "memset");
  int* verr = fresh_error_word();
  check(tcsl_cuda_validate_entries(off, ent, n_entries, m, k, cfg.m_tb, cfg.k_tb, TCSL_CHECK_SPMM, flags, verr,
                                   nullptr),
        "spmm");
  std::uint32_t h = 0;
  check(tcsl_cuda_memcpy_d2h(&h, flags, sizeof h, nullptr), "spmm");
  collect_errors(verr, "spmm");
  return (h & (TCSL_FLAG_DUPLICATE_LOCATIONS | TCSL_FLAG_PARTIAL_GROUPS)) == 0;
}

FloatMatrix spmm_device(const std::uint32_t* off, const std::uint32_t* ent, std::uint64_t n_entries, std::uint32_t m,
                        std::uint32_t k, const TileConfig& cfg, bool tc_ready, const HalfMatrix& b,
                        const SpmmOptions& opt) {
  if (b.rows() <= 0 || b.cols() <= 0) raise(Errc::invalid_argument, "B must be non-empty");
  if (static_cast<std::int64_t>(k) != b.rows())
    raise(Errc::dimension_mismatch, "A has " + std::to_string(k) + " columns, B has " + std::to_string(b.rows()) +
                                        " rows");
  const int n = static_cast<int>(b.cols());
  FloatMatrix c(m, n);
  Scratch& s = scratch();
  const bool exact = opt.exact || !tc_ready;
  const std::uint16_t* x = upload_half(s.x, b);
  auto* y = static_cast<float*>(s.y.get(4ull * m * n));
  std::size_t ws_bytes = 0;
  if (exact)
    check(tcsl_cuda_spmm_exact_workspace(m, k, &ws_bytes), "spmm");
  else
    check(tcsl_cuda_spmm_workspace(m, k, cfg.m_tb, cfg.k_tb, n, opt.split_k, &ws_bytes), "spmm");
  void* ws = s.ws.get(std::max<std::size_t>(ws_bytes, 256));
  int* err = fresh_error_word();
  if (exact)
    check(tcsl_cuda_spmm_exact(off, ent, n_entries, m, k, cfg.m_tb, cfg.k_tb, x, n, y, ws, ws_bytes, err, nullptr),
          "spmm");
  else
    check(tcsl_cuda_spmm(off, ent, n_entries, m, k, cfg.m_tb, cfg.k_tb, x, n, y, opt.split_k, ws, ws_bytes, err,
                         nullptr),
          "spmm");
  check(tcsl_cuda_memcpy_d2h(c.data(), y, 4ull * m * n, nullptr), "spmm");
  collect_errors(err, "spmm");
  return c;
}

}  // namespace

FloatMatrix spmm(const TcslMatrix& a, const HalfMatrix& b, const SpmmOptions& opt) {
  check_spmm_args(a);
  if (b.rows() <= 0 || b.cols() <= 0) raise(Errc::invalid_argument, "B must be non-empty");
  if (static_cast<std::int64_t>(a.k) != b.rows())
    raise(Errc::dimension_mismatch,
          "A has " + std::to_string(a.k) + " columns, B has " + std::to_string(b.rows()) + " rows");
  const DeviceTcsl d = upload(a);
  const bool tc_ready = !opt.exact && tc_preconditions(d.off, d.ent, a.entries.size(), a.m, a.k, a.cfg);
  return spmm_device(d.off, d.ent, a.entries.size(), a.m, a.k, a.cfg, tc_ready, b, opt);
}

DeviceMatrix::DeviceMatrix(const TcslMatrix& t) : m_(t.m), k_(t.k), cfg_(t.cfg), n_entries_(t.entries.size()) {
  check_spmm_args(t);
  check(tcsl_cuda_malloc(&off_, 4 * t.tile_offsets.size()), "device allocation");
  check(tcsl_cuda_malloc(&ent_, 4 * std::max<std::size_t>(t.entries.size(), 1)), "device allocation");
  check(tcsl_cuda_memcpy_h2d(off_, t.tile_offsets.data(), 4 * t.tile_offsets.size(), nullptr), "upload offsets");
  check(tcsl_cuda_memcpy_h2d(ent_, t.entries.data(), 4 * t.entries.size(), nullptr), "upload entries");
  tc_ready_ = tc_preconditions(static_cast<const std::uint32_t*>(off_), static_cast<const std::uint32_t*>(ent_),
                                n_entries_, m_, k_, cfg_);
}

DeviceMatrix::~DeviceMatrix() {
  tcsl_cuda_free(off_);
  tcsl_cuda_free(ent_);
}

FloatMatrix DeviceMatrix::spmm(const HalfMatrix& b, const SpmmOptions& opt) const {
  return spmm_device(static_cast<const std::uint32_t*>(off_), static_cast<const std::uint32_t*>(ent_), n_entries_,
                     m_, k_, cfg_, tc_ready_, b, opt);
}

int reg_pressure(const TcslMatrix& t) {
  t.cfg.validate();
  if (t.tile_offsets.size() != static_cast<std::size_t>(t.num_tiles()) + 1)
    raise(Errc::inconsistent_offsets, "offset table does not match tile count");
  int worst = 0;
  for (std::uint32_t tile = 0; tile < t.num_tiles(); ++tile)
    worst = std::max(worst, div_up(t.tile_entry_count(tile), t.cfg.threads_per_block));
  return worst;
}

HalfMatrix prune_magnitude(const HalfMatrix& a, double beta) {
  if (!(beta >= 0.0 && beta <= 1.0)) raise(Errc::invalid_argument, "sparsity must be in [0, 1]");
  HalfMatrix out = a;
  const auto n = static_cast<std::uint64_t>(a.size());
  if (n == 0) return out;
  Scratch& s = scratch();
  auto* d = static_cast<std::uint16_t*>(s.dense.get(2 * n));
  check(tcsl_cuda_memcpy_h2d(d, a.data(), 2 * n, nullptr), "prune");
  std::size_t ws_bytes = 0;
  check(tcsl_cuda_prune_workspace(n, &ws_bytes), "prune");
  void* ws = s.ws.get(ws_bytes);
  check(tcsl_cuda_prune_magnitude(d, n, beta, d, ws, ws_bytes, nullptr), "prune");
  check(tcsl_cuda_memcpy_d2h(out.data(), d, 2 * n, nullptr), "prune");
  check(tcsl_cuda_stream_sync(nullptr), "prune");
  return out;
}

FloatMatrix dense_gemm_ref(const HalfMatrix& a, const HalfMatrix& b, const TileConfig& cfg) {
  cfg.validate();
  if (a.rows() <= 0 || a.cols() <= 0 || b.cols() <= 0) raise(Errc::invalid_argument, "operands must be non-empty");
  if (a.cols() != b.rows())
    raise(Errc::dimension_mismatch, "A is " + std::to_string(a.rows()) + "x" + std::to_string(a.cols()) +
                                        ", B has " + std::to_string(b.rows()) + " rows");
  // The bit-exact GPU path consumes Tiled-CSL; encode A with the same tiling.
  return spmm(encode(a, cfg, false), b, SpmmOptions{0, true});
}

}  // namespace tcsl
