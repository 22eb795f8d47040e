// K2: Load-as-Sparse / Compute-as-Dense SpMM on sm_100a (TileConfig {128, 64}).
//
// Reference semantics: tcsl::spmm, proj/src/engine.cpp:27-78 — per 128-row
// block, per 64-column k-tile: rebuild the dense tile from its Tiled-CSL
// entries (extract_tile, engine.cpp:8-25) and run a dense product over every
// element, zeros included. Here the dense product is a tcgen05 MMA with an
// fp32 accumulator in TMEM; the reference's serial fp32 add order is not
// reproduced (tolerance per BASELINE.json north_star), see spmm_exact for the
// bit-exact CUDA-core mode.
//
// One persistent CTA per SM, warp-specialised (512 threads):
//   warp 0      entry producer: streams each unit's contiguous entry span
//               [off[t0], off[t1]) with cp.async.bulk into a ring of 2 KB chunks
//   warp 1      X producer: TMA-loads the 64 x NPAD activation tile per k-tile
//               (MN-major, hardware swizzle = 2*NPAD bytes)
//   warp 2      TMEM owner + single-thread tcgen05.mma issuer (M=128, N=NPAD, K=16 x 4)
//   warps 4-7   epilogue: tcgen05.ld accumulator -> fp32 Y rows (or split-K partials)
//   warps 8-15  decode, two teams of 4 warps working on alternate k-tiles: zero
//               the dense tile, then scatter each 32-entry group (one entry per
//               lane) into the SWIZZLE_NONE K-major core-matrix layout
// The core-matrix layout puts element (x, y) in bank (x%8)*4 + (y%8)/2, which is
// exactly the reference's bank_id (proj/include/tcsl/tcsl_format.hpp:18), so the
// encoder's ahead-of-time bank reordering keeps the scatter near one wavefront
// per group.
//
// Work unit = (row block rb, k-split s): k-tiles [s*tk/S, (s+1)*tk/S).
// S == 1 writes Y directly; S > 1 writes partial sums P[s] that
// tcsl_cuda_splitk_reduce adds in ascending s (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>

#include "sm100_ptx.cuh"
#include "tcsl_internal.cuh"

namespace tcslk {

namespace {

constexpr int kMTB = 128, kKTB = 64;
constexpr uint32_t kABytes = kMTB * kKTB * 2;  // dense fp16 tile, 16 KB
constexpr int kNA = 4;                         // dense-tile buffers (2 per decode team)
constexpr int kTeamWarps = 4;                  // warps per decode team
constexpr uint32_t kChunk = 512;               // entries per ring chunk (2 KB); chunks are tile-aligned
constexpr uint32_t kRingT = 20;                // chunks per team ring (40 KB; >= one dense tile + slack)
constexpr int kThreads = 512;
constexpr int kWarpEpi = 4, kWarpDec = 8;

template <int NPAD>
struct Cfg {
  static constexpr int kBoxW = NPAD < 64 ? NPAD : 64;       // TMA box / swizzle atom width
  static constexpr int kBoxes = NPAD / kBoxW;
  static constexpr uint32_t kBoxBytes = 64u * kBoxW * 2;    // 64 k-rows
  static constexpr uint32_t kXStage = kBoxBytes * kBoxes;
  static constexpr int kNX = (32768 / kXStage) < 2 ? 2 : ((32768 / kXStage) > 8 ? 8 : (32768 / kXStage));
  static constexpr uint32_t kRowBytes = kBoxW * 2;
  static constexpr uint32_t kLayout = kRowBytes == 16 ? 0u : (kRowBytes == 32 ? 6u : (kRowBytes == 64 ? 4u : 2u));
  // SWIZZLE_NONE (NPAD=8): LBO = k-group stride (8 rows x 16 B); swizzled: SBO = 8-row
  // k-group stride, LBO = stride between 64-column atoms.
  static constexpr uint32_t kLBO = kRowBytes == 16 ? 128u : kBoxBytes;
  static constexpr uint32_t kSBO = kRowBytes == 16 ? 128u : 8u * kRowBytes;
  static constexpr uint32_t kKStep = 16u * kRowBytes;       // 16 k-rows per MMA
  static constexpr uint32_t kTmemCols = (2 * NPAD) <= 32 ? 32 : ((2 * NPAD) <= 64 ? 64 : ((2 * NPAD) <= 128 ? 128 : ((2 * NPAD) <= 256 ? 256 : 512)));
  static constexpr uint32_t kIdesc = idesc_f16_f32(128, NPAD, 1);
  // smem carve-up (from a 1024-aligned base)
  static constexpr uint32_t kOffX = kNA * kABytes;
  static constexpr uint32_t kOffE = kOffX + kNX * kXStage;
  static constexpr uint32_t kOffBar = kOffE + 2 * kRingT * kChunk * 4;
  static constexpr uint32_t kNumBars = 2 * kNA + 2 * kNX + 4 * kRingT + 4;
  static constexpr uint32_t kSmem = 1024 + kOffBar + 8 * kNumBars + 16;
};

struct Params {
  const uint32_t* off;
  const uint32_t* ent;
  uint64_t n_entries;
  uint32_t m, k;
  int tiles_m, tiles_k;
  int n, col0, split, units;
  float* out;
  int ldo;
  int* err;
  unsigned long long* trace;  // TCSL_TRACE builds only: per-event clock64 stamps of CTA 0
};

#ifdef TCSL_TRACE
#define TRACE(slot, idx) \
  do { if (blockIdx.x == 0 && p.trace && (idx) < 4096) p.trace[(slot) * 4096 + (idx)] = clock64(); } while (0)
#else
#define TRACE(slot, idx) do { } while (0)
#endif

struct Unit {
  int rb, s, kt0, kt1;
};
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
  Unit x;
  x.rb = u / p.split;
  x.s = u - x.rb * p.split;
  x.kt0 = static_cast<int>(static_cast<long long>(x.s) * p.tiles_k / p.split);
  x.kt1 = static_cast<int>(static_cast<long long>(x.s + 1) * p.tiles_k / p.split);
  return x;
}
// The unit's entry span; every role derives the same (sanitised) span.
__device__ __forceinline__ bool unit_span(const Params& p, const Unit& u, uint32_t& e0, uint32_t& e1) {
  const uint32_t t0 = static_cast<uint32_t>(u.rb) * p.tiles_k + u.kt0;
  const uint32_t t1 = static_cast<uint32_t>(u.rb) * p.tiles_k + u.kt1;
  e0 = __ldg(p.off + t0);
  e1 = __ldg(p.off + t1);
  if (e1 < e0 || e1 > p.n_entries || (e0 & 31u) || ((e1 - e0) & 31u)) {
    e1 = e0;
    return false;
  }
  return true;
}
// A tile's span is streamed / decoded only when it sits inside the unit span
// as whole 32-entry groups; producer and decoders apply the same rule.
__device__ __forceinline__ uint32_t tile_groups(uint32_t e0, uint32_t e1, uint32_t a0, uint32_t a1) {
  return (e0 <= a0 && a0 <= a1 && a1 <= e1 && ((a1 - a0) & 31u) == 0) ? (a1 - a0) >> 5 : 0u;
}

// Byte offset of tile element `loc` (= x*64 + y) in the K-major SWIZZLE_NONE
// canonical layout: (x/8)*1024 + (y/8)*128 + (x%8)*16 + (y%8)*2. Bits >= 13 of
// loc are ignored, so the address is always inside the 16 KB tile.
__device__ __forceinline__ uint32_t a_offset(uint32_t loc) {
  return ((loc << 1) & 0x3C0Eu)  // (y%8)*2 from loc[2:0], (x/8)*1024 from loc[12:9]
         | ((loc >> 2) & 0x70u)  // (x%8)*16 from loc[8:6]
         | ((loc << 4) & 0x380u);  // (y/8)*128 from loc[5:3]
}

template <int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
    spmm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  using C = Cfg<NPAD>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t s_a = (raw + 1023u) & ~1023u;
  const uint32_t s_x = s_a + C::kOffX;
  const uint32_t s_e = s_a + C::kOffE;  // team t ring at s_e + t * kRingT * kChunk * 4
  const uint32_t s_bar = s_a + C::kOffBar;
  const uint32_t b_afull = s_bar, b_aempty = s_bar + 8 * kNA;
  const uint32_t b_xfull = s_bar + 8 * (2 * kNA), b_xempty = b_xfull + 8 * C::kNX;
  const uint32_t b_efull = b_xempty + 8 * C::kNX;  // [team][kRingT]
  const uint32_t b_eempty = b_efull + 8 * 2 * kRingT;
  const uint32_t b_dfull = b_eempty + 8 * 2 * kRingT, b_dempty = b_dfull + 16;
  const uint32_t s_tmem_slot = b_dempty + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (s_tmem_slot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNA; ++i) {
      mbar_init(b_afull + 8 * i, kTeamWarps);
      mbar_init(b_aempty + 8 * i, 1);
    }
    for (int i = 0; i < C::kNX; ++i) {
      mbar_init(b_xfull + 8 * i, 1);
      mbar_init(b_xempty + 8 * i, 1);
    }
    for (uint32_t i = 0; i < 2 * kRingT; ++i) {
      mbar_init(b_efull + 8 * i, 1);
      mbar_init(b_eempty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(b_dfull + 8 * i, 1);
      mbar_init(b_dempty + 8 * i, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1 && lane == 0) prefetch_tmap(&tmap_x);
  if (warp == 2) tmem_alloc_dyn(s_tmem_slot, C::kTmemCols);
  for (uint32_t i = threadIdx.x; i < kNA * kABytes / 16; i += kThreads) sts128_zero(s_a + 16 * i);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == 3) {
    // ------------------------------------------------------ entry producers (one per team)
    // Streams the entry span of every k-tile of its team (gt % 2 == team) into
    // the team ring, in tile-aligned 2 KB chunks.
    if (lane == 0) {
      const uint32_t team = warp == 0 ? 0u : 1u;
      const uint32_t ring = s_e + team * kRingT * kChunk * 4;
      const uint32_t efull = b_efull + 8 * team * kRingT, eempty = b_eempty + 8 * team * kRingT;
      const uint64_t pol = policy_evict_first();
      uint32_t g = 0, gt = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit un = unit_of(p, u);
        uint32_t e0, e1;
        if (!unit_span(p, un, e0, e1) && team == 0) raise_dev(p.err, TCSL_STATUS_INCONSISTENT_OFFSETS);
        const uint32_t tile0 = static_cast<uint32_t>(un.rb) * p.tiles_k + un.kt0;
        for (int kt = un.kt0; kt < un.kt1; ++kt, ++gt) {
          if ((gt & 1u) != team) continue;
          const uint32_t t = tile0 + (kt - un.kt0);
          const uint32_t a0 = __ldg(p.off + t), a1 = __ldg(p.off + t + 1);
          const uint32_t ng = tile_groups(e0, e1, a0, a1);
          for (uint32_t c0 = 0; c0 < 32 * ng; c0 += kChunk, ++g) {
            const uint32_t slot = g % kRingT;
            const uint32_t use = g / kRingT;
            if (team == 0) TRACE(9, g);
            if (use > 0) mbar_wait_sleep(eempty + 8 * slot, (use - 1) & 1);
            if (team == 0) TRACE(10, g);
            const uint32_t bytes = min(kChunk, 32 * ng - c0) * 4;
            mbar_arrive_expect_tx(efull + 8 * slot, bytes);
            bulk_g2s(ring + slot * kChunk * 4, p.ent + a0 + c0, bytes, efull + 8 * slot, pol);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- X producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      uint32_t gt = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit un = unit_of(p, u);
        for (int kt = un.kt0; kt < un.kt1; ++kt, ++gt) {
          const uint32_t slot = gt % C::kNX;
          const uint32_t use = gt / C::kNX;
          if (use > 0) mbar_wait_sleep(b_xempty + 8 * slot, (use - 1) & 1);
          mbar_arrive_expect_tx(b_xfull + 8 * slot, C::kXStage);
#pragma unroll
          for (int bx = 0; bx < C::kBoxes; ++bx)
            tma_load_2d(s_x + slot * C::kXStage + bx * C::kBoxBytes, &tmap_x, p.col0 + bx * C::kBoxW, kt * kKTB,
                        b_xfull + 8 * slot, pol);
        }
      }
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      uint32_t gt = 0, ui = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
        const Unit un = unit_of(p, u);
        const uint32_t acc = ui & 1;
        if (ui >= 2) mbar_wait_sleep(b_dempty + 8 * acc, ((ui >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * NPAD;
        for (int kt = un.kt0; kt < un.kt1; ++kt, ++gt) {
          const uint32_t b = gt % kNA;
          const uint32_t xs = gt % C::kNX;
          TRACE(5, gt);
          mbar_wait(b_afull + 8 * b, (gt / kNA) & 1);
          TRACE(6, gt);
          mbar_wait(b_xfull + 8 * xs, (gt / C::kNX) & 1);
          TRACE(7, gt);
          tc_fence_after();
          const uint32_t a0 = s_a + b * kABytes;
          const uint32_t x0 = s_x + xs * C::kXStage;
#pragma unroll
          for (int s = 0; s < kKTB / 16; ++s) {
            const uint64_t ad = smem_desc(a0 + s * 256, 128, 1024, 0);
            const uint64_t bd = smem_desc(x0 + s * C::kKStep, C::kLBO, C::kSBO, C::kLayout);
            mma_f16_ss(d_tmem, ad, bd, C::kIdesc, (kt > un.kt0 || s > 0) ? 1u : 0u);
          }
          mma_commit(b_aempty + 8 * b);
          mma_commit(b_xempty + 8 * xs);
#ifdef TCSL_TRACE
          if (blockIdx.x == 0 && p.trace) {  // debug only: measure MMA completion latency
            mbar_wait(b_aempty + 8 * b, (gt / kNA) & 1);
            TRACE(8, gt);
          }
#endif
        }
        mma_commit(b_dfull + 8 * acc);
      }
    }
    __syncwarp();
  } else if (warp >= kWarpEpi && warp < kWarpEpi + 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lanes 32q..32q+31
    uint32_t ui = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
      const Unit un = unit_of(p, u);
      const uint32_t acc = ui & 1;
      mbar_wait_sleep(b_dfull + 8 * acc, (ui >> 1) & 1);
      tc_fence_after();
      const long long row = static_cast<long long>(un.rb) * kMTB + q * 32 + lane;
      float* dst = p.out + (p.split > 1 ? static_cast<long long>(un.s) * p.m * p.ldo : 0ll) + row * p.ldo + p.col0;
      const bool row_ok = row < p.m;
      const uint32_t t_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * NPAD;
      const int ncol = min(NPAD, p.n - p.col0);
      if constexpr (NPAD == 8) {
        uint32_t r[8];
        tmem_ld8(t_base, r);
        tmem_ld_wait();
        if (row_ok) {
          if (ncol == 8 && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
            reinterpret_cast<float4*>(dst)[0] =
                make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]), __uint_as_float(r[3]));
            reinterpret_cast<float4*>(dst)[1] =
                make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]), __uint_as_float(r[7]));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < ncol) dst[j] = __uint_as_float(r[j]);
          }
        }
      } else {
#pragma unroll
        for (int c0 = 0; c0 < NPAD; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(t_base + c0, r);
          tmem_ld_wait();
          if (row_ok) {
            if (c0 + 16 <= ncol && ((reinterpret_cast<uintptr_t>(dst + c0) & 15u) == 0)) {
              float4* d4 = reinterpret_cast<float4*>(dst + c0);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                d4[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                    __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (c0 + j < ncol) dst[c0 + j] = __uint_as_float(r[j]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(b_dempty + 8 * acc);
    }
  } else if (warp >= kWarpDec) {
    // ---------------------------------------------------------------- decode
    // Team t (4 warps) decodes the k-tiles with gt % 2 == t into buffers t, t+2.
    const int dw = warp - kWarpDec;
    const uint32_t team = dw / kTeamWarps;
    const int tw = dw % kTeamWarps;
    const uint32_t ring = s_e + team * kRingT * kChunk * 4;
    const uint32_t efull = b_efull + 8 * team * kRingT, eempty = b_eempty + 8 * team * kRingT;
    uint32_t gt = 0;
    uint32_t cbase = 0;                   // first team-ring chunk of the current tile
    uint32_t prev_base = 0, prev_n = 0;   // chunks of this team's previous tile (released after the barrier)
    uint32_t nxt = 0;                     // team-ring chunks < nxt have been waited full by this warp
    uint32_t err_or = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const Unit un = unit_of(p, u);
      uint32_t e0, e1;
      unit_span(p, un, e0, e1);
      const uint32_t tile0 = static_cast<uint32_t>(un.rb) * p.tiles_k + un.kt0;
      const int ntiles = un.kt1 - un.kt0;
      // offsets window: lane l holds off[tile0 + 32*w + l]
      const uint32_t last_off = tile0 + ntiles;
      uint32_t win_cur = __ldg(p.off + min(tile0 + lane, last_off));
      uint32_t win_nxt = __ldg(p.off + min(tile0 + 32 + lane, last_off));
      int win = 0;
      for (int i = 0; i < ntiles; ++i, ++gt) {
        if ((i >> 5) != win) {  // slide the window by 32 tiles
          win_cur = win_nxt;
          ++win;
          win_nxt = __ldg(p.off + min(tile0 + 32 * (win + 1) + lane, last_off));
        }
        if ((gt & 1u) != team) continue;
        const uint32_t a0 = __shfl_sync(0xffffffffu, win_cur, i & 31);
        const uint32_t a1n = __shfl_sync(0xffffffffu, win_nxt, 0);
        const uint32_t a1c = __shfl_sync(0xffffffffu, win_cur, (i + 1) & 31);
        const uint32_t a1 = ((i & 31) == 31) ? a1n : a1c;
        const uint32_t ng = tile_groups(e0, e1, a0, a1);
        const uint32_t b = gt % kNA;
        const uint32_t use = gt / kNA;
        const uint32_t a_tile = s_a + b * kABytes;
        if (tw == 0 && lane == 0) TRACE(0, gt);
        if (use > 0) {
          mbar_wait(b_aempty + 8 * b, (use - 1) & 1);
          const uint32_t q0 = a_tile + tw * (kABytes / kTeamWarps);
#pragma unroll
          for (int r = 0; r < static_cast<int>(kABytes / kTeamWarps / 512); ++r) sts128_zero(q0 + 512 * r + 16 * lane);
        }
        if (tw == 0 && lane == 0) TRACE(1, gt);
        named_bar_sync(1 + team, kTeamWarps * 32);
        if (tw == 0 && lane == 0) {
          TRACE(2, gt);
          // every warp of the team is past its previous tile: hand its chunks back
          for (uint32_t c = prev_base; c < prev_base + prev_n; ++c) mbar_arrive(eempty + 8 * (c % kRingT));
        }
        if (a1 != a0 + 32 * ng && tw == 0 && lane == 0) raise_dev(p.err, TCSL_STATUS_INCONSISTENT_OFFSETS);
        // contiguous quarter of the tile's groups
        const uint32_t g0 = ng * tw / kTeamWarps, g1 = ng * (tw + 1) / kTeamWarps;
        uint32_t g = g0;
#ifdef TCSL_TRACE
        long long wait_cyc = 0, n_waits = 0;
#endif
        for (; g + 4 <= g1; g += 4) {
          const uint32_t c_hi = cbase + (32 * (g + 3)) / kChunk;
#ifdef TCSL_TRACE
          const long long tw0 = clock64();
          if (nxt <= c_hi) ++n_waits;
#endif
          while (nxt <= c_hi) {
            mbar_wait(efull + 8 * (nxt % kRingT), (nxt / kRingT) & 1);
            ++nxt;
          }
#ifdef TCSL_TRACE
          wait_cyc += clock64() - tw0;
#endif
          uint32_t e[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t pj = 32 * (g + j);
            e[j] = lds32(ring + 4 * (((cbase + pj / kChunk) % kRingT) * kChunk + (pj % kChunk) + lane));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            err_or |= e[j];
            sts16(a_tile + a_offset(e[j]), e[j] >> 16);
          }
        }
        for (; g < g1; ++g) {
          const uint32_t pj = 32 * g;
          const uint32_t c = cbase + pj / kChunk;
          while (nxt <= c) {
            mbar_wait(efull + 8 * (nxt % kRingT), (nxt / kRingT) & 1);
            ++nxt;
          }
          const uint32_t e = lds32(ring + 4 * ((c % kRingT) * kChunk + (pj % kChunk) + lane));
          err_or |= e;
          sts16(a_tile + a_offset(e), e >> 16);
        }
        if (tw == 0 && lane == 0) TRACE(3, gt);
#ifdef TCSL_TRACE
        if (tw == 0 && lane == 0 && blockIdx.x == 0 && p.trace && gt < 4096) {
          p.trace[11 * 4096 + gt] = wait_cyc;
          p.trace[12 * 4096 + gt] = n_waits;
        }
#endif
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_afull + 8 * b);
        if (tw == 0 && lane == 0) TRACE(4, gt);
        const uint32_t nch = (32 * ng + kChunk - 1) / kChunk;
        prev_base = cbase;
        prev_n = nch;
        cbase += nch;
        if (nxt < cbase) nxt = cbase;  // chunks of this tile that this warp never read
      }
    }
    // locations >= 8192 leave the 128x64 tile (the scatter masked them into range)
    if (__any_sync(0xffffffffu, (err_or & 0xE000u) != 0) && lane == 0)
      raise_dev(p.err, TCSL_STATUS_LOCATION_OUT_OF_RANGE);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

int pad_n(int n) {
  if (n <= 8) return 8;
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

// Estimated runtime (us) of a split choice: max over persistent CTAs of their
// units' tile work + per-unit overhead, plus the reduction pass.
double split_cost(int tiles_m, int tiles_k, int split, int sms, double t_tile, double mn_bytes) {
  const int units = tiles_m * split;
  const int grid = std::min(units, sms);
  std::vector<double> load(grid, 0.0);
  for (int u = 0; u < units; ++u) {
    const int s = u % split;
    const int kt0 = static_cast<int>(static_cast<long long>(s) * tiles_k / split);
    const int kt1 = static_cast<int>(static_cast<long long>(s + 1) * tiles_k / split);
    load[u % grid] += (kt1 - kt0) * t_tile + 0.8;
  }
  double worst = 0.0;
  for (double l : load) worst = std::max(worst, l);
  if (split > 1) worst += 2.5 + (split + 2) * mn_bytes / 5.0e6;
  return worst;
}

template <int NPAD>
cudaError_t launch_npad(const Params& p, const CUtensorMap& tm, int grid, cudaStream_t s) {
  using C = Cfg<NPAD>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(spmm_sm100_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(C::kSmem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  spmm_sm100_kernel<NPAD><<<grid, kThreads, C::kSmem, s>>>(tm, p);
  return cudaGetLastError();
}

}  // namespace

unsigned long long* g_trace = nullptr;

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

int auto_split(uint32_t m, uint32_t k, int n, double avg_entries_per_tile) {
  const int tiles_m = div_up_i(m, kMTB), tiles_k = div_up_i(k, kKTB);
  const int sms = num_sms();
  // per-SM streaming rate ~ 6.5 TB/s / 148; dense-tile smem floor ~0.12 us per tile
  const double t_tile = std::max(avg_entries_per_tile * 4.0 / 44.0e3, 0.12);
  const double mn_bytes = static_cast<double>(m) * std::min(n, 256) * 4.0;
  int best = 1;
  double best_cost = split_cost(tiles_m, tiles_k, 1, sms, t_tile, mn_bytes);
  for (int s = 2; s <= std::min(32, tiles_k); ++s) {
    const double c = split_cost(tiles_m, tiles_k, s, sms, t_tile, mn_bytes);
    if (c < best_cost * 0.97) {
      best = s;
      best_cost = c;
    }
  }
  return best;
}

int spmm_sm100_plan(uint32_t m, uint32_t k, int n, int split_k, SpmmPlan* plan) {
  const int tiles_m = div_up_i(m, kMTB), tiles_k = div_up_i(k, kKTB);
  plan->n = n;
  plan->n_pad = pad_n(std::min(n, 256));
  plan->split = split_k > 0 ? std::min(split_k, tiles_k) : 1;
  plan->units = tiles_m * plan->split;
  plan->grid = std::min(plan->units, num_sms());
  plan->smem = 0;
  return 0;
}

cudaError_t launch_spmm_sm100(const SpmmPlan& plan, const uint32_t* off, const uint32_t* ent,
                              uint64_t n_entries, uint32_t m, uint32_t k, const uint16_t* x, int ldx,
                              float* out, int* err, cudaStream_t s) {
  auto encode = tensor_map_encoder();
  if (!encode) return cudaErrorNotSupported;
  Params p{};
  p.off = off;
  p.ent = ent;
  p.n_entries = n_entries;
  p.m = m;
  p.k = k;
  p.tiles_m = div_up_i(m, kMTB);
  p.tiles_k = div_up_i(k, kKTB);
  p.n = plan.n;
  p.split = plan.split;
  p.units = plan.units;
  p.out = out;
  p.ldo = plan.n;
  p.err = err;
  p.trace = g_trace;
  // Column slabs of <= 256 (one TMEM accumulator pair each).
  for (int col0 = 0; col0 < plan.n; col0 += 256) {
    const int n_pad = pad_n(std::min(256, plan.n - col0));
    const int box_w = std::min(n_pad, 64);
    p.col0 = col0;
    const uint32_t row_bytes = box_w * 2;
    const CUtensorMapSwizzle swz =
        row_bytes == 16 ? CU_TENSOR_MAP_SWIZZLE_NONE
                        : (row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B));
    CUtensorMap tm;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(plan.n), static_cast<cuuint64_t>(k)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_w), 64u};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(x), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    cudaError_t e;
    switch (n_pad) {
      case 8: e = launch_npad<8>(p, tm, plan.grid, s); break;
      case 16: e = launch_npad<16>(p, tm, plan.grid, s); break;
      case 32: e = launch_npad<32>(p, tm, plan.grid, s); break;
      case 64: e = launch_npad<64>(p, tm, plan.grid, s); break;
      case 128: e = launch_npad<128>(p, tm, plan.grid, s); break;
      default: e = launch_npad<256>(p, tm, plan.grid, s); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tcslk

#ifdef TCSL_TRACE
extern "C" void tcsl_cuda_debug_set_trace(unsigned long long* d_trace) { tcslk::g_trace = d_trace; }
#endif
