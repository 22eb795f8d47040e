// TCSL container I/O (host). Byte layout per proj/include/tcsl/tcsl_format.hpp:68-71,
// validation order and error classes per proj/src/tcsl_format.cpp:19-32, 157-245,
// so reference artifacts (and their FNV-1a hashes) round-trip unchanged.
#include <cstring>
#include <fstream>
#include <iterator>

#include "tcsl/tcsl_format.hpp"

namespace tcsl {

namespace {

constexpr std::uint16_t kFormatVersion = 1;
constexpr std::uint16_t kReorderedFlag = 1;
constexpr std::size_t kHeaderBytes = 28;

void require_whole_groups(const TcslMatrix& t) {
  const std::uint32_t nt = t.num_tiles();
  if (t.tile_offsets.size() != static_cast<std::size_t>(nt) + 1)
    raise(Errc::inconsistent_offsets, "offset table must have num_tiles+1 entries");
  if (t.tile_offsets[0] != 0) raise(Errc::inconsistent_offsets, "first offset must be 0");
  for (std::uint32_t i = 0; i < nt; ++i) {
    const std::uint32_t lo = t.tile_offsets[i], hi = t.tile_offsets[i + 1];
    if (hi < lo) raise(Errc::inconsistent_offsets, "offsets must be non-decreasing");
    if ((hi - lo) % kGroupSize) raise(Errc::inconsistent_offsets, "tile entry counts must be multiples of 32");
  }
  if (t.tile_offsets[nt] != t.entries.size()) raise(Errc::inconsistent_offsets, "last offset must equal the entry count");
}

void put_le(std::vector<std::uint8_t>& out, std::uint32_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

// Little-endian cursor; reading past the end is Errc::truncated.
class Cursor {
 public:
  Cursor(const std::uint8_t* p, std::size_t n) : p_(p), n_(n) {}
  void need(std::size_t k) const {
    if (k > n_ - at_) raise(Errc::truncated, "unexpected end of file");
  }
  std::uint32_t le(int bytes) {
    need(static_cast<std::size_t>(bytes));
    std::uint32_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint32_t>(p_[at_ + i]) << (8 * i);
    at_ += static_cast<std::size_t>(bytes);
    return v;
  }
  void copy(void* dst, std::size_t k) {
    need(k);
    if (k) std::memcpy(dst, p_ + at_, k);
    at_ += k;
  }
  void magic() {
    need(4);
    if (std::memcmp(p_ + at_, "TCSL", 4) != 0) raise(Errc::bad_magic, "not a TCSL file");
    at_ += 4;
  }
  void finish() const {
    if (at_ != n_) raise(Errc::trailing_data, "trailing bytes after payload");
  }

 private:
  const std::uint8_t* p_;
  std::size_t n_;
  std::size_t at_ = 0;
};

}  // namespace

std::vector<std::uint8_t> serialize_tcsl(const TcslMatrix& t) {
  t.cfg.validate();
  if (t.m == 0 || t.k == 0) raise(Errc::bad_header, "matrix dims must be positive");
  require_whole_groups(t);
  std::vector<std::uint8_t> out;
  out.reserve(footprint_bytes(t));
  out.insert(out.end(), {'T', 'C', 'S', 'L'});
  put_le(out, kFormatVersion, 2);
  put_le(out, t.reordered ? kReorderedFlag : 0, 2);
  put_le(out, t.m, 4);
  put_le(out, t.k, 4);
  put_le(out, static_cast<std::uint32_t>(t.cfg.m_tb), 4);
  put_le(out, static_cast<std::uint32_t>(t.cfg.k_tb), 4);
  put_le(out, t.num_tiles(), 4);
  const std::size_t off_bytes = 4 * t.tile_offsets.size(), ent_bytes = 4 * t.entries.size();
  out.resize(kHeaderBytes + off_bytes + ent_bytes);
  std::memcpy(out.data() + kHeaderBytes, t.tile_offsets.data(), off_bytes);
  if (ent_bytes) std::memcpy(out.data() + kHeaderBytes + off_bytes, t.entries.data(), ent_bytes);
  return out;
}

TcslMatrix deserialize_tcsl(const std::uint8_t* data, std::size_t size) {
  Cursor in(data, size);
  in.magic();
  if (in.le(2) != kFormatVersion) raise(Errc::bad_version, "unknown TCSL version");
  const std::uint32_t flags = in.le(2);
  if (flags & ~static_cast<std::uint32_t>(kReorderedFlag)) raise(Errc::bad_version, "unknown TCSL flag bits");
  TcslMatrix t;
  t.reordered = flags & kReorderedFlag;
  t.m = in.le(4);
  t.k = in.le(4);
  const std::uint32_t m_tb = in.le(4), k_tb = in.le(4);
  if (t.m == 0 || t.k == 0) raise(Errc::bad_header, "matrix dims must be positive");
  if (m_tb == 0 || k_tb == 0 || m_tb > 65536 || k_tb > 65536) raise(Errc::bad_header, "implausible tile dims");
  t.cfg.m_tb = static_cast<int>(m_tb);
  t.cfg.k_tb = static_cast<int>(k_tb);
  try {
    t.cfg.validate();
  } catch (const Error& e) {
    raise(Errc::bad_header, e.what());
  }
  const std::uint32_t nt = in.le(4);
  if (nt != t.num_tiles()) raise(Errc::bad_header, "tile count does not match dims");
  t.tile_offsets.resize(static_cast<std::size_t>(nt) + 1);
  in.copy(t.tile_offsets.data(), 4 * t.tile_offsets.size());
  if (t.tile_offsets[0] != 0) raise(Errc::inconsistent_offsets, "first offset must be 0");
  for (std::uint32_t i = 0; i < nt; ++i) {
    if (t.tile_offsets[i + 1] < t.tile_offsets[i]) raise(Errc::inconsistent_offsets, "offsets must be non-decreasing");
    if ((t.tile_offsets[i + 1] - t.tile_offsets[i]) % kGroupSize)
      raise(Errc::inconsistent_offsets, "tile entry counts must be multiples of 32");
  }
  const std::size_t n = t.tile_offsets[nt];
  in.need(4 * n);
  t.entries.resize(n);
  in.copy(t.entries.data(), 4 * n);
  in.finish();
  return t;
}

TcslMatrix deserialize_tcsl(const std::vector<std::uint8_t>& bytes) { return deserialize_tcsl(bytes.data(), bytes.size()); }

void save_tcsl(const std::string& path, const TcslMatrix& t) {
  const std::vector<std::uint8_t> bytes = serialize_tcsl(t);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) raise(Errc::io_failure, "cannot open " + path + " for writing");
  f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
  if (!f) raise(Errc::io_failure, "cannot write " + path);
}

TcslMatrix load_tcsl(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) raise(Errc::io_failure, "cannot open " + path);
  const std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (f.bad()) raise(Errc::io_failure, "cannot read " + path);
  return deserialize_tcsl(bytes);
}

std::size_t footprint_bytes(const TcslMatrix& t) {
  return kHeaderBytes + 4 * t.tile_offsets.size() + 4 * t.entries.size();
}

double footprint_ratio(const TcslMatrix& t) {
  return static_cast<double>(footprint_bytes(t)) / (2.0 * static_cast<double>(t.m) * static_cast<double>(t.k));
}

}  // namespace tcsl
