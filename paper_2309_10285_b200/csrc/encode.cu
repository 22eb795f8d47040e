// K1: GPU Tiled-CSL encoder, bit-exact with tcsl::encode
// (reference: proj/src/tcsl_format.cpp:36-124, layout proj/include/tcsl/tcsl_format.hpp:12-54).
//
// The reference emits each tile's nonzeros with a sequential greedy loop:
// "pull from the bank bucket with the most entries left, smallest bank id on
// ties, FIFO inside a bucket" (tcsl_format.cpp:81-97). That loop is a pure
// function of the 32 bucket sizes c_b and each entry's FIFO index k inside its
// bucket: the entry is emitted when its bucket has L = c_b - k entries left,
// and every entry with a larger "level" L' > L (from any bucket) or the same
// level in a smaller bank precedes it. Hence
//     pos = F(L) + popc(Mask(L) & ((1 << b) - 1)),
//     F(L) = sum_b' max(0, c_b' - L),  Mask(L) = {b' : c_b' >= L},
// a closed form every thread evaluates independently.
// Padding: +0.0 entries at the tile's first (32 - nnz % 32) % 32 zero
// positions in row-major order, fringe included (tcsl_format.cpp:103-119).
//
// Two passes: encode_count_kernel -> exclusive scan (CUB) -> encode_emit_kernel.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "tcsl_internal.cuh"

namespace tcslk {

namespace {

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// One block per tile: number of nonzero (bit pattern & 0x7FFF != 0) elements
// inside the matrix, rounded up to whole 32-entry groups.
__global__ void __launch_bounds__(256) encode_count_kernel(const uint16_t* __restrict__ w, uint32_t m,
                                                           uint32_t k, int m_tb, int k_tb, int tiles_k,
                                                           uint32_t* __restrict__ counts) {
  const uint32_t tile = blockIdx.x;
  const long long r0 = static_cast<long long>(tile / tiles_k) * m_tb;
  const int c0 = static_cast<int>(tile % tiles_k) * k_tb;
  const int x_end = static_cast<int>(min(static_cast<long long>(m_tb), static_cast<long long>(m) - r0));
  const int y_end = min(k_tb, static_cast<int>(k) - c0);
  uint32_t cnt = 0;
  if ((k & 7u) == 0 && (reinterpret_cast<uintptr_t>(w) & 15u) == 0) {
    // 16-byte vector loads: rows start 16-B aligned because k % 8 == 0 and c0 % 8 == 0.
    const int vpr = (y_end + 7) >> 3;
    const int total = x_end * vpr;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int x = i / vpr, v = i - x * vpr;
      const uint16_t* p = w + (r0 + x) * k + c0 + v * 8;
      if (v * 8 + 8 <= y_end) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
        const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) cnt += ((wd[e] & 0x7FFFu) != 0) + ((wd[e] & 0x7FFF0000u) != 0);
      } else {
        for (int y = v * 8; y < y_end; ++y) cnt += (p[y - v * 8] & 0x7FFFu) != 0;
      }
    }
  } else {
    const int total = x_end * y_end;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int x = i / y_end, y = i - x * y_end;
      cnt += (w[(r0 + x) * k + c0 + y] & 0x7FFFu) != 0;
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  __shared__ uint32_t part[32];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) part[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int i = 0; i < (blockDim.x >> 5); ++i) s += part[i];
    counts[tile] = (s + 31u) & ~31u;
  }
}

struct EmitLayout {
  int items;     // m_tb * ceil(k_tb / 64): one (row, 64-column chunk) per warp step
  int max_level; // m_tb * k_tb / 32: the largest possible bank count
  bool stage;    // stage the tile's entries in smem (tile_elems <= 8192)
  size_t cnt4, nzz, bpre, npre, zpre, cb, fl, ml, stg, bytes;
};

__host__ __device__ inline EmitLayout emit_layout(int m_tb, int k_tb) {
  EmitLayout L{};
  const int nch = (k_tb + 63) / 64;
  L.items = m_tb * nch;
  L.max_level = m_tb * k_tb / 32;
  L.stage = m_tb * k_tb <= 8192;
  size_t o = 0;
  L.cnt4 = o; o += 4ull * L.items;
  L.nzz = o;  o += 4ull * L.items;
  L.npre = o; o += 4ull * L.items;
  L.zpre = o; o += 4ull * L.items;
  L.bpre = o; o += 8ull * L.items;
  L.cb = o;   o += 4ull * 32 + 16;
  L.fl = o;   o += 4ull * (L.max_level + 2);
  L.ml = o;   o += 4ull * (L.max_level + 2);
  o = (o + 15) & ~size_t(15);
  L.stg = o;  o += L.stage ? 4ull * m_tb * k_tb : 0;
  L.bytes = o;
  return L;
}

struct Pair {
  uint32_t v0, v1;  // element bits (0 when outside)
  bool nz0, nz1;    // numerically nonzero inside the matrix
  bool in0, in1;    // position exists inside the m_tb x k_tb tile
};

__device__ __forceinline__ Pair load_pair(const uint16_t* __restrict__ w, uint32_t k, long long r0, int c0,
                                          int x, int y0, int x_end, int y_end, int k_tb) {
  Pair p;
  p.in0 = y0 < k_tb;
  p.in1 = y0 + 1 < k_tb;
  const bool val0 = x < x_end && y0 < y_end;
  const bool val1 = x < x_end && y0 + 1 < y_end;
  p.v0 = p.v1 = 0;
  if (val0) {
    const uint16_t* src = w + (r0 + x) * k + c0 + y0;
    if (val1 && ((reinterpret_cast<uintptr_t>(src) & 3u) == 0)) {
      const uint32_t both = __ldg(reinterpret_cast<const uint32_t*>(src));
      p.v0 = both & 0xFFFFu;
      p.v1 = both >> 16;
    } else {
      p.v0 = __ldg(src);
      if (val1) p.v1 = __ldg(src + 1);
    }
  }
  p.nz0 = (p.v0 & 0x7FFFu) != 0;
  p.nz1 = (p.v1 & 0x7FFFu) != 0;
  return p;
}

// The two elements at (x, y0), (x, y0 + 1) as one word (v0 | v1 << 16), 0 outside.
__device__ __forceinline__ uint32_t load_raw(const uint16_t* __restrict__ w, uint32_t k, long long r0, int c0, int x,
                                             int y0, int x_end, int y_end) {
  const bool val0 = x < x_end && y0 < y_end;
  const bool val1 = x < x_end && y0 + 1 < y_end;
  if (!val0) return 0u;
  const uint16_t* src = w + (r0 + x) * k + c0 + y0;
  if (val1 && ((reinterpret_cast<uintptr_t>(src) & 3u) == 0)) return __ldg(reinterpret_cast<const uint32_t*>(src));
  return static_cast<uint32_t>(__ldg(src)) | (val1 ? static_cast<uint32_t>(__ldg(src + 1)) << 16 : 0u);
}
__device__ __forceinline__ Pair pair_from_raw(uint32_t raw, int y0, int k_tb) {
  Pair p;
  p.in0 = y0 < k_tb;
  p.in1 = y0 + 1 < k_tb;
  p.v0 = raw & 0xFFFFu;
  p.v1 = raw >> 16;
  p.nz0 = (p.v0 & 0x7FFFu) != 0;
  p.nz1 = (p.v1 & 0x7FFFu) != 0;
  return p;
}

// Items (rows x 64-column chunks) per warp kept in registers between the two
// passes when the tile shape allows (128 x 64 with 8 warps): the tile is read
// from HBM once, with all 16 loads of a warp in flight at once.
constexpr int kEmitIpw = 16;

// One block (8 warps) per tile. See the file comment for the closed form.
__global__ void __launch_bounds__(256) encode_emit_kernel(const uint16_t* __restrict__ w, uint32_t m,
                                                          uint32_t k, int m_tb, int k_tb, int tiles_k,
                                                          int reorder, const uint32_t* __restrict__ offsets,
                                                          uint32_t* __restrict__ entries, int* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const EmitLayout lay = emit_layout(m_tb, k_tb);
  uint32_t* cnt4 = reinterpret_cast<uint32_t*>(smem + lay.cnt4);
  uint32_t* nzz = reinterpret_cast<uint32_t*>(smem + lay.nzz);
  uint32_t* npre = reinterpret_cast<uint32_t*>(smem + lay.npre);
  uint32_t* zpre = reinterpret_cast<uint32_t*>(smem + lay.zpre);
  uint16_t* bpre = reinterpret_cast<uint16_t*>(smem + lay.bpre);
  uint32_t* cb = reinterpret_cast<uint32_t*>(smem + lay.cb);
  uint32_t* fl = reinterpret_cast<uint32_t*>(smem + lay.fl);
  uint32_t* ml = reinterpret_cast<uint32_t*>(smem + lay.ml);
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem + lay.stg);

  const uint32_t tile = blockIdx.x;
  const long long r0 = static_cast<long long>(tile / tiles_k) * m_tb;
  const int c0 = static_cast<int>(tile % tiles_k) * k_tb;
  const int x_end = static_cast<int>(min(static_cast<long long>(m_tb), static_cast<long long>(m) - r0));
  const int y_end = min(k_tb, static_cast<int>(k) - c0);
  const int nch = (k_tb + 63) / 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const uint32_t lt = lanemask_lt();

  const bool regs = lay.items == kEmitIpw * nwarps && nch == 1;  // the warp's items fit in registers (item = row)
  uint32_t raw[kEmitIpw];
  if (regs) {
    if (x_end == m_tb && y_end == 64 && (k & 1u) == 0) {
      // full tile, 4-byte aligned rows: one strided pointer, no per-item bounds
      const uint32_t* rp = reinterpret_cast<const uint32_t*>(w + (r0 + warp) * k + c0) + lane;
      const size_t stride = static_cast<size_t>(nwarps) * (k >> 1);
#pragma unroll
      for (int q = 0; q < kEmitIpw; ++q) raw[q] = __ldg(rp + q * stride);
    } else {
#pragma unroll
      for (int q = 0; q < kEmitIpw; ++q) raw[q] = load_raw(w, k, r0, c0, warp + q * nwarps, 2 * lane, x_end, y_end);
    }
  }

  // ---- pass A: per (row, chunk) item, per-bank-column counts and nz / zero counts
#pragma unroll
  for (int q = 0; q < kEmitIpw; ++q) {
    if (!regs) break;
    const int it = warp + q * nwarps;
    const Pair p = pair_from_raw(raw[q], 2 * lane, k_tb);
    // per bank column j = lane % 4: nonzeros of the lanes l = j (mod 4), summed
    // by three xor-shuffles; lane j < 4 stores byte j of cnt4[it]
    uint32_t v = (p.nz0 ? 1u : 0u) + (p.nz1 ? 1u : 0u);
    uint32_t zc = (p.in0 && !p.nz0 ? 1u : 0u) + (p.in1 && !p.nz1 ? 1u : 0u);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    const uint32_t nt = __reduce_add_sync(0xffffffffu, (p.nz0 ? 1u : 0u) + (p.nz1 ? 1u : 0u));
    zc = __reduce_add_sync(0xffffffffu, zc);
    if (lane < 4) reinterpret_cast<uint8_t*>(cnt4)[4 * it + lane] = static_cast<uint8_t>(v);
    if (lane == 0) nzz[it] = nt | (zc << 16);
  }
  for (int it = warp; it < lay.items && !regs; it += nwarps) {
    const int x = it / nch, ch = it - x * nch;
    const Pair p = load_pair(w, k, r0, c0, x, ch * 64 + 2 * lane, x_end, y_end, k_tb);
    const uint32_t b0 = __ballot_sync(0xffffffffu, p.nz0), b1 = __ballot_sync(0xffffffffu, p.nz1);
    const uint32_t z0 = __ballot_sync(0xffffffffu, p.in0 && !p.nz0);
    const uint32_t z1 = __ballot_sync(0xffffffffu, p.in1 && !p.nz1);
    if (lane == 0) {
      uint32_t c4 = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t mj = 0x11111111u << j;
        c4 |= static_cast<uint32_t>(__popc(b0 & mj) + __popc(b1 & mj)) << (8 * j);
      }
      cnt4[it] = c4;
      nzz[it] = static_cast<uint32_t>(__popc(b0) + __popc(b1)) |
                (static_cast<uint32_t>(__popc(z0) + __popc(z1)) << 16);
    }
  }
  __syncthreads();

  // ---- prefixes: per bank over its items (warp 0), scan order over all items (warp 1)
  if (warp == 0) {
    const int x0 = lane >> 2, j = lane & 3;
    uint32_t run = 0;
    if (regs && m_tb == 8 * kEmitIpw) {
      // all 16 counts loaded first (independent LDS), then the running sum
      uint32_t cv[kEmitIpw];
#pragma unroll
      for (int q = 0; q < kEmitIpw; ++q) cv[q] = reinterpret_cast<const uint8_t*>(cnt4)[4 * (x0 + 8 * q) + j];
#pragma unroll
      for (int q = 0; q < kEmitIpw; ++q) {
        bpre[(x0 + 8 * q) * 4 + j] = static_cast<uint16_t>(run);
        run += cv[q];
      }
    } else {
      for (int x = x0; x < m_tb; x += 8) {
        for (int ch = 0; ch < nch; ++ch) {
          const int it = x * nch + ch;
          bpre[it * 4 + j] = static_cast<uint16_t>(run);
          run += (cnt4[it] >> (8 * j)) & 0xFFu;
        }
      }
    }
    cb[lane] = run;
    const uint32_t tot = __reduce_add_sync(0xffffffffu, run);
    const uint32_t mx = __reduce_max_sync(0xffffffffu, run);
    if (lane == 0) {
      cb[32] = tot;
      cb[33] = mx;
    }
  } else if (warp == 1) {
    uint32_t carry_n = 0, carry_z = 0;
    for (int base = 0; base < lay.items; base += 32) {
      const int it = base + lane;
      const uint32_t v = it < lay.items ? nzz[it] : 0u;
      uint32_t n = v & 0xFFFFu, z = v >> 16;
      uint32_t in = n, iz = z;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t tn = __shfl_up_sync(0xffffffffu, in, d), tz = __shfl_up_sync(0xffffffffu, iz, d);
        if (lane >= d) {
          in += tn;
          iz += tz;
        }
      }
      if (it < lay.items) {
        npre[it] = carry_n + in - n;
        zpre[it] = carry_z + iz - z;
      }
      carry_n += __shfl_sync(0xffffffffu, in, 31);
      carry_z += __shfl_sync(0xffffffffu, iz, 31);
    }
  }
  __syncthreads();

  const uint32_t nnz = cb[32];
  const uint32_t maxc = cb[33];
  const uint32_t pad = (32u - (nnz & 31u)) & 31u;
  const uint32_t base = offsets[tile];
  if (offsets[tile + 1] - base != nnz + pad) {  // count pass / offsets disagree
    if (threadIdx.x == 0) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
    return;
  }
  if (reorder) {
    for (uint32_t L = threadIdx.x + 1; L <= maxc; L += blockDim.x) {
      uint32_t f = 0, mask = 0;
#pragma unroll 8
      for (int b = 0; b < 32; ++b) {
        const uint32_t c = cb[b];
        f += c > L ? c - L : 0u;
        mask |= static_cast<uint32_t>(c >= L) << b;
      }
      fl[L] = f;
      ml[L] = mask;
    }
    __syncthreads();
  }

  // ---- pass B: place every nonzero and the first `pad` zero positions
  uint32_t* out = lay.stage ? stg : entries + base;
  auto place = [&](int it, int x, int y0, const Pair& p) {
    const uint32_t b0 = __ballot_sync(0xffffffffu, p.nz0), b1 = __ballot_sync(0xffffffffu, p.nz1);
    const bool zp0 = p.in0 && !p.nz0, zp1 = p.in1 && !p.nz1;
    const uint32_t z0 = __ballot_sync(0xffffffffu, zp0), z1 = __ballot_sync(0xffffffffu, zp1);
    const uint32_t loc0 = static_cast<uint32_t>(x * k_tb + y0);
    if (p.nz0 || p.nz1) {
      uint32_t pos0, pos1;
      if (reorder) {
        const int j = lane & 3;
        const uint32_t mj = 0x11111111u << j;
        const int b = (x & 7) * 4 + j;
        const uint32_t kb = bpre[it * 4 + j] + __popc(b0 & mj & lt) + __popc(b1 & mj & lt);
        const uint32_t c = cb[b];
        const uint32_t below = (1u << b) - 1u;
        const uint32_t L0 = c - kb;
        pos0 = fl[L0] + __popc(ml[L0] & below);
        const uint32_t L1 = c - kb - (p.nz0 ? 1u : 0u);
        pos1 = fl[L1] + __popc(ml[L1] & below);
      } else {
        pos0 = npre[it] + __popc(b0 & lt) + __popc(b1 & lt);
        pos1 = pos0 + (p.nz0 ? 1u : 0u);
      }
      if (p.nz0) out[pos0] = (p.v0 << 16) | loc0;
      if (p.nz1) out[pos1] = (p.v1 << 16) | (loc0 + 1);
    }
    if (pad && (zp0 || zp1)) {
      const uint32_t zr0 = zpre[it] + __popc(z0 & lt) + __popc(z1 & lt);
      const uint32_t zr1 = zr0 + (zp0 ? 1u : 0u);
      if (zp0 && zr0 < pad) out[nnz + zr0] = loc0;
      if (zp1 && zr1 < pad) out[nnz + zr1] = loc0 + 1;
    }
  };
  if (regs) {
#pragma unroll
    for (int q = 0; q < kEmitIpw; ++q) {
      const int it = warp + q * nwarps;
      place(it, it, 2 * lane, pair_from_raw(raw[q], 2 * lane, k_tb));
    }
  } else {
    for (int it = warp; it < lay.items; it += nwarps) {
      const int x = it / nch, ch = it - x * nch;
      const int y0 = ch * 64 + 2 * lane;
      place(it, x, y0, load_pair(w, k, r0, c0, x, y0, x_end, y_end, k_tb));
    }
  }
  if (lay.stage) {
    __syncthreads();
    const uint32_t total = nnz + pad;  // multiple of 32, base multiple of 32: 128-B aligned spans
    uint4* dst = reinterpret_cast<uint4*>(entries + base);
    const uint4* src = reinterpret_cast<const uint4*>(stg);
    for (uint32_t i = threadIdx.x; i < total / 4; i += blockDim.x) dst[i] = src[i];
  }
}

// ============================================================================
// Fast path for the default TileConfig {128, 64} (every BASELINE shape).
//
// Count: one warp per tile (persistent grid), 16-byte loads, a branch-free
// nonzero test on two binary16 at once: t = v & 0x7FFF7FFF; t + 0x7FFF7FFF has
// bit 15 (31) set iff the low (high) half is nonzero (no carry crosses halves).
//
// Emit (bank reorder): warp w owns the tile rows x = w + 8q (q = 0..15), i.e.
// exactly the four buckets (w, j) of bank_id(x, y) = (x%8)*4 + (y%8)/2 with
// j = lane % 4 (lane holds elements y = 2*lane, 2*lane + 1, both in bank column
// j). The FIFO index of an entry inside its bucket is therefore a running
// count inside the warp (ballots, no shared memory); only the 32 bucket sizes
// cross warps (one barrier). Then pos = F(L) + popc(Mask(L) & below(b)) (see
// the file comment) from a per-tile table of (F, Mask) over L = 1..max c_b, the
// entries are staged in shared memory and written out with 16-byte stores.
// ============================================================================

__device__ __forceinline__ uint32_t nz_bits2(uint32_t v) {  // bit 15 / 31 = low / high half nonzero
  return ((v & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x80008000u;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ldg_nc_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_u32_if(uint32_t addr, uint32_t v, uint32_t pred) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}" ::"r"(addr), "r"(v),
               "r"(pred)
               : "memory");
}
// The look-back status word is self-contained (flag and value in one 64-bit word,
// nothing else published through it), so relaxed loads suffice; an acquire load
// would hold back the warp's later shared-memory work until it completes.
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Requires k % 8 == 0 and a 16-byte aligned W (rows and 8-column chunks are
// 16-byte aligned; a tile's column fringe is then a whole number of chunks).
#ifndef TCSL_COUNT_MINB
#define TCSL_COUNT_MINB 4  // 64 registers, 32 warps per SM: 130 us vs 137 us (128 registers) on ffn1
#endif
__global__ void __launch_bounds__(256, TCSL_COUNT_MINB) encode_count128_kernel(const uint16_t* __restrict__ w, uint32_t m, uint32_t k,
                                                              int tiles_k, uint32_t tiles,
                                                              uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const int ch = lane & 7, rr = lane >> 3;  // 8-column chunk, row within a 4-row slab
  const size_t ld4 = k >> 3;                // row stride in uint4
  for (uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < tiles; tile += nw) {
    const uint32_t tr = tile / tiles_k, tc = tile - tr * tiles_k;
    const long long r0 = static_cast<long long>(tr) * 128;
    const int x_end = static_cast<int>(min(128ll, static_cast<long long>(m) - r0));
    const bool col_ok = static_cast<uint32_t>(tc * 64 + ch * 8) < k;
    const uint4* p = reinterpret_cast<const uint4*>(w + r0 * k + tc * 64) + ch + rr * ld4;
    uint32_t cnt = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = 4 * (8 * b + i) + rr;
        v[i] = (col_ok && row < x_end) ? ldg_nc_v4(p + static_cast<size_t>(4 * (8 * b + i)) * ld4) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t a = nz_bits2(v[i].x) | (nz_bits2(v[i].y) >> 15);
        const uint32_t c = nz_bits2(v[i].z) | (nz_bits2(v[i].w) >> 15);
        cnt += __popc(a) + __popc(c);
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) counts[tile] = (cnt + 31u) & ~31u;
  }
}

// Decoupled look-back status word of the fused (one-pass) encoder: bits 32-33
// = 1 (tile aggregate) or 2 (inclusive prefix), bits 0-31 = the value.
constexpr unsigned long long kAggregate = 1ull << 32, kPrefix = 2ull << 32;

// FUSED = false: offsets come from the count pass (checked against the tile's
// own count). FUSED = true: one pass; each tile takes a ticket (tiles in
// ticket order, so every earlier tile is resident or done), publishes its
// entry count, finds its base with a warp-wide look-back over earlier tiles'
// status words, writes offsets[tile + 1], and writes its entries only when
// they fit in `capacity`.
//
// Layout: lane = (rr, ch) holds the 8 elements y = 8ch .. 8ch+7 of row
// x = w + 8(4q + rr) for slices q = 0..3 (one 16-byte load each). Word j of
// the load holds both elements of bank column j (y % 8 = 2j, 2j+1), so the
// four per-column counts of a lane pack into the bytes of one register and a
// single byte-packed warp scan per slice gives every element's FIFO index
// (lane order inside a slice is row-major, slices are in row order).
// One 128 x 64 tile's loads: lane (rr, ch), slice q -> v[q][j] = elements
// (x, 8ch + 2j), (x, 8ch + 2j + 1) of row x = warp + 8(4q + rr), 0 outside.
__device__ __forceinline__ void load_tile128(const uint16_t* __restrict__ w, uint32_t m, uint32_t k, int tiles_k,
                                             uint32_t tile, int warp, int rr, int ch, uint32_t (&v)[4][4]) {
  const uint32_t tr = tile / tiles_k, tc = tile - tr * tiles_k;
  const long long r0 = static_cast<long long>(tr) * 128;
  const int c0 = static_cast<int>(tc) * 64;
  const int x_end = static_cast<int>(min(128ll, static_cast<long long>(m) - r0));
  const int y_end = min(64, static_cast<int>(k) - c0);
  if (x_end == 128 && y_end == 64 && (k & 7u) == 0 && (reinterpret_cast<uintptr_t>(w) & 15u) == 0) {
    const uint4* p = reinterpret_cast<const uint4*>(w + (r0 + warp + 8 * rr) * k + c0) + ch;
    const size_t st = static_cast<size_t>(k) * 4;  // 32 rows, in 16-byte units
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 t = ldg_nc_v4(p + q * st);
      v[q][0] = t.x;
      v[q][1] = t.y;
      v[q][2] = t.z;
      v[q][3] = t.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) v[q][j] = load_raw(w, k, r0, c0, warp + 8 * (4 * q + rr), 8 * ch + 2 * j, x_end, y_end);
  }
}

// FUSED = false: offsets come from the count pass (checked against the tile's
// own count). FUSED = true: one pass; tiles are taken by ticket (so every
// earlier tile is held by a running block), each publishes its entry count,
// finds its base with a warp-wide look-back over earlier tiles' status words,
// writes offsets[tile + 1], and writes its entries only when they fit in
// `capacity`.
//
// One tile per block (persistent blocks that prefetch the next tile measured
// 17 % slower: fewer resident blocks at the higher register count).
//
// Layout: lane = (rr, ch) holds the 8 elements y = 8ch .. 8ch+7 of row
// x = w + 8(4q + rr) for slices q = 0..3 (one 16-byte load each). Word j of
// the load holds both elements of bank column j (y % 8 = 2j, 2j+1), so the
// four per-column counts of a lane pack into the bytes of one register and a
// single byte-packed warp scan per slice gives every element's FIFO index
// (lane order inside a slice is row-major, slices are in row order).
#ifndef TCSL_EMIT_MINB
#define TCSL_EMIT_MINB 6  // 40 registers, 6 blocks per SM (the 36 KB smem limit): 386 us vs 392 (5) and 409 (4)
#endif
template <bool FUSED>
__global__ void __launch_bounds__(256, TCSL_EMIT_MINB) encode_emit128_kernel(const uint16_t* __restrict__ w, uint32_t m,
                                                                 uint32_t k, int tiles_k, uint32_t tiles,
                                                                 const uint32_t* __restrict__ offsets_in,
                                                                 uint32_t* __restrict__ offsets_out,
                                                                 uint32_t* __restrict__ entries, uint64_t capacity,
                                                                 unsigned long long* status, uint32_t* ticket,
                                                                 int* err) {
  __shared__ uint32_t s_cb[32];
  __shared__ uint2 s_tab[258];   // (F(L), Mask(L)), L = 1 .. max c_b <= 256
  __shared__ uint8_t s_zb[1024]; // per (row, 8-column chunk): zero positions (bit = y % 8)
  __shared__ uint32_t s_misc[4];
  extern __shared__ __align__(16) uint32_t s_stg[];  // [8192] staged entries
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rr = lane >> 3, ch = lane & 7;
  const uint32_t stg = static_cast<uint32_t>(__cvta_generic_to_shared(s_stg));
  uint32_t tile = blockIdx.x;
  if (FUSED) {
    if (threadIdx.x == 0) s_misc[0] = atomicAdd(ticket, 1u);
    __syncthreads();
    tile = s_misc[0];
  }
  uint32_t v[4][4];
  load_tile128(w, m, k, tiles_k, tile, warp, rr, ch, v);
  {
    // ---- FIFO index of each lane's first element per column, packed in bytes
    uint32_t kidp[4];
    uint32_t runp = 0;  // per-column counts of the earlier slices (<= 192 each)
    uint32_t cfin[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t c4 = 0, zm = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t nb = nz_bits2(v[q][j]);
        c4 |= static_cast<uint32_t>(__popc(nb)) << (8 * j);
        zm |= (((~nb) >> 15) & 1u) << (2 * j) | (((~nb) >> 31) & 1u) << (2 * j + 1);
      }
      uint32_t inc = c4;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
      kidp[q] = runp + inc - c4;
      if (q < 3) {
        runp += tot;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) cfin[j] = ((runp >> (8 * j)) & 0xFFu) + ((tot >> (8 * j)) & 0xFFu);
      }
      s_zb[(warp + 8 * (4 * q + rr)) * 8 + ch] = static_cast<uint8_t>(zm);
    }
    if (lane < 4) s_cb[warp * 4 + lane] = lane == 0 ? cfin[0] : (lane == 1 ? cfin[1] : (lane == 2 ? cfin[2] : cfin[3]));
    __syncthreads();  // (1)

    // ---- (F, Mask) table, tile totals
    const uint32_t cl = s_cb[lane];
    const uint32_t nnz = __reduce_add_sync(0xffffffffu, cl);
    const uint32_t maxc = __reduce_max_sync(0xffffffffu, cl);
    const uint32_t pad = (32u - (nnz & 31u)) & 31u;
    const uint32_t total = nnz + pad;
    for (uint32_t L = warp + 1; L <= maxc; L += 8) {
      const uint32_t f = __reduce_add_sync(0xffffffffu, cl > L ? cl - L : 0u);
      const uint32_t mk = __ballot_sync(0xffffffffu, cl >= L);
      if (lane == 0) s_tab[L] = make_uint2(f, mk);
    }
    // one pass: publish this tile's count now; the look-back for its base runs after
    // the place phase, when the earlier tiles have had that time to publish prefixes
    if (FUSED && warp == 0 && lane == 0) st_release_gpu_u64(status + tile, (tile == 0 ? kPrefix : kAggregate) | total);
    uint32_t base = 0;
    if (!FUSED) {
      base = offsets_in[tile];
      if (offsets_in[tile + 1] - base != total) {  // count pass / offsets disagree
        if (threadIdx.x == 0) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
        return;
      }
    }
    __syncthreads();  // (2)

    // ---- +0.0 pads at the first `pad` zero positions, row-major (fringe included)
    if (pad && warp == 7) {
      uint32_t zb = 0;
      for (int x0 = 0; x0 < 128 && zb < pad; x0 += 4) {
        const uint32_t zm = s_zb[x0 * 8 + lane];  // row x0 + lane / 8, chunk lane % 8: lanes in row-major order
        const uint32_t n = __popc(zm);
        uint32_t inc = n;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
          if (lane >= d) inc += t;
        }
        uint32_t r = zb + inc - n, mm = zm;
        const uint32_t loc = static_cast<uint32_t>(x0 + (lane >> 3)) * 64u + 8u * (lane & 7);
        while (mm && r < pad) {
          const int bit = __ffs(mm) - 1;
          mm &= mm - 1;
          s_stg[nnz + r] = loc + bit;
          ++r;
        }
        zb += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    // ---- place: pos = F(L) + popc(Mask(L) & below(b)), b = 4 * warp + j;
    //      branch-free (a zero element's table reads stay in range, 0 <= L <= 256;
    //      only the stores are predicated)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t xloc = static_cast<uint32_t>(warp + 8 * (4 * q + rr)) * 64u + 8u * ch;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t below = (1u << (warp * 4 + j)) - 1u;
        const uint32_t r = v[q][j], nb = nz_bits2(r);
        const uint32_t n0 = (nb >> 15) & 1u;
        const uint32_t L0 = cfin[j] - ((kidp[q] >> (8 * j)) & 0xFFu);
        const uint32_t loc0 = xloc + 2u * j;
        const uint2 t0 = s_tab[L0];
        const uint2 t1 = s_tab[L0 - n0];
        sts_u32_if(stg + 4u * (t0.x + __popc(t0.y & below)), __byte_perm(r, loc0, 0x1054), n0);
        sts_u32_if(stg + 4u * (t1.x + __popc(t1.y & below)), __byte_perm(r, loc0 + 1u, 0x3254), nb >> 31);
      }
    }
    if (FUSED && warp == 0) {
      // decoupled look-back
      uint32_t acc = 0;
      for (long long jt = static_cast<long long>(tile) - 1; jt >= 0; jt -= 32) {
        const long long idx = jt - lane;
        unsigned long long sv = 0;
        if (idx >= 0) {
          while ((sv >> 32) == 0) sv = ld_relaxed_gpu_u64(status + idx);
        }
        const uint32_t pm = __ballot_sync(0xffffffffu, idx >= 0 && (sv >> 32) == 2);
        const uint32_t val = idx >= 0 ? static_cast<uint32_t>(sv) : 0u;
        if (pm) {
          const int f = __ffs(pm) - 1;
          acc += __reduce_add_sync(0xffffffffu, lane <= f ? val : 0u);
          break;
        }
        acc += __reduce_add_sync(0xffffffffu, val);
      }
      if (lane == 0) {
        if (tile) st_release_gpu_u64(status + tile, kPrefix | (acc + total));
        offsets_out[tile + 1] = acc + total;
        if (tile == 0) offsets_out[0] = 0;
        s_misc[1] = acc;
      }
    }
    __syncthreads();  // (3)
    if (FUSED) base = s_misc[1];
    if (!FUSED || static_cast<uint64_t>(base) + total <= capacity) {  // else the host sees offsets[T] > capacity
      uint4* dst = reinterpret_cast<uint4*>(entries + base);
      const uint4* src = reinterpret_cast<const uint4*>(s_stg);
      for (uint32_t i = threadIdx.x; i < total / 4; i += blockDim.x) dst[i] = src[i];
    }
  }
}

constexpr size_t kEmit128Dyn = 8192 * 4;

bool fast128(const void* w, uint32_t k, int m_tb, int k_tb) {
  return m_tb == 128 && k_tb == 64 && (k & 7u) == 0 && (reinterpret_cast<uintptr_t>(w) & 15u) == 0;
}

}  // namespace

cudaError_t launch_encode_count(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb,
                                uint32_t* counts, cudaStream_t s) {
  const int tk = div_up_i(k, k_tb);
  const long long tiles = static_cast<long long>(div_up_i(m, m_tb)) * tk;
  if (tiles <= 0) return cudaSuccess;
  if (fast128(w, k, m_tb, k_tb) && !getenv("TCSL_ENCODE_SLOW")) {
    const long long blocks = std::min<long long>((tiles + 7) / 8, 148ll * 16);
    encode_count128_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(w, m, k, tk, static_cast<uint32_t>(tiles),
                                                                        counts);
    return cudaGetLastError();
  }
  encode_count_kernel<<<static_cast<unsigned>(tiles), 256, 0, s>>>(w, m, k, m_tb, k_tb, tk, counts);
  return cudaGetLastError();
}

size_t encode_fused_ws_bytes(uint32_t tiles) { return 256 + 8ull * tiles; }

cudaError_t launch_encode_fused(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                                uint32_t* offsets, uint32_t* entries, uint64_t capacity, void* ws, int* err,
                                cudaStream_t s) {
  (void)m_tb;
  (void)k_tb;
  (void)reorder;
  const int tk = div_up_i(k, 64);
  const long long tiles = static_cast<long long>(div_up_i(m, 128)) * tk;
  cudaError_t e = cudaMemsetAsync(ws, 0, encode_fused_ws_bytes(static_cast<uint32_t>(tiles)), s);
  if (e != cudaSuccess || tiles <= 0) return e;
  auto* ticket = static_cast<uint32_t*>(ws);
  auto* status = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256);
  e = cudaFuncSetAttribute(encode_emit128_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kEmit128Dyn));
  if (e != cudaSuccess) return e;
  encode_emit128_kernel<true><<<static_cast<unsigned>(tiles), 256, kEmit128Dyn, s>>>(w, m, k, tk, static_cast<uint32_t>(tiles), nullptr, offsets, entries,
                                                                            capacity, status, ticket, err);
  return cudaGetLastError();
}

bool encode_fused_supported(const void* w, const void* entries, uint32_t k, int m_tb, int k_tb, int reorder) {
  (void)w;
  (void)k;
  return reorder && m_tb == 128 && k_tb == 64 && (reinterpret_cast<uintptr_t>(entries) & 15u) == 0;
}

size_t encode_scan_temp_bytes(uint32_t tiles) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                static_cast<int>(tiles) + 1);
  return bytes;
}

cudaError_t launch_encode_scan(uint32_t* counts_in, uint32_t* offsets, uint32_t tiles, void* temp,
                               size_t temp_bytes, cudaStream_t s) {
  return cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts_in, offsets, static_cast<int>(tiles) + 1, s);
}

cudaError_t launch_encode_emit(const uint16_t* w, uint32_t m, uint32_t k, int m_tb, int k_tb, int reorder,
                               const uint32_t* offsets, uint32_t* entries, int* err, cudaStream_t s) {
  const int tk = div_up_i(k, k_tb);
  const long long tiles = static_cast<long long>(div_up_i(m, m_tb)) * tk;
  if (tiles > 0 && reorder && m_tb == 128 && k_tb == 64 && (reinterpret_cast<uintptr_t>(entries) & 15u) == 0 &&
      !getenv("TCSL_ENCODE_SLOW")) {
    cudaError_t e = cudaFuncSetAttribute(encode_emit128_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kEmit128Dyn));
    if (e != cudaSuccess) return e;
    encode_emit128_kernel<false><<<static_cast<unsigned>(tiles), 256, kEmit128Dyn, s>>>(w, m, k, tk, static_cast<uint32_t>(tiles), offsets, nullptr, entries,
                                                                               0, nullptr, nullptr, err);
    return cudaGetLastError();
  }
  const EmitLayout lay = emit_layout(m_tb, k_tb);
  cudaError_t e = cudaFuncSetAttribute(encode_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(lay.bytes));
  if (e != cudaSuccess) return e;
  if (tiles > 0)
    encode_emit_kernel<<<static_cast<unsigned>(tiles), 256, lay.bytes, s>>>(w, m, k, m_tb, k_tb, tk, reorder,
                                                                           offsets, entries, err);
  return cudaGetLastError();
}

}  // namespace tcslk
