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
// One persistent CTA per SM, warp-specialised (640 threads). The scheduler
// favours higher warp ids, so the pacing role gets the highest id:
//   warps 0-11  decode, three teams of 4 warps on k-tiles gt % 3 == team: zero the
//               dense tile, then each warp scatters its contiguous share of the
//               tile's 32-entry groups (one entry per lane, loaded from L2 straight
//               into registers one team-tile ahead) into the SWIZZLE_NONE K-major
//               core-matrix layout
//   warps 12-15 epilogue: tcgen05.ld accumulator -> fp32 Y rows (or split-K partials)
//   warp 16     X producer: TMA-loads kTX k-tiles x NPAD activations per stage
//               (MN-major, hardware swizzle = 2*NPAD bytes)
//   warp 17     L2 prefetcher: cp.async.bulk.prefetch.L2 of the entry spans of the
//               next kPrefetchAhead k-tiles, paced by the MMA's progress
//   warp 19     TMEM owner + tcgen05.mma issuer (M=128, N=NPAD, K=16 x 4 per k-tile).
//               A tcgen05.mma of this shape holds the issuing thread ~45 cycles and
//               the tensor pipe does not queue behind it, so every cycle this loop
//               spends outside MMA issue is tensor-pipe idle time: it polls plain
//               smem counters (not mbarriers) and syncs/commits once per PAIR of
//               k-tiles.
// The core-matrix layout puts element (x, y) in bank (x%8)*4 + (y%8)/2, which is
// exactly the reference's bank_id (proj/include/tcsl/tcsl_format.hpp:18), so the
// encoder's ahead-of-time bank reordering keeps the scatter close to one wavefront
// per group.
//
// Work unit = (row block rb, k-split s): k-tiles [s*tk/S, (s+1)*tk/S).
// S == 1 writes Y directly; S > 1 writes partial sums P[s] that
// tcsl_cuda_splitk_reduce adds in ascending s (deterministic).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "sm100_ptx.cuh"
#include "tcsl_internal.cuh"

namespace tcslk {

namespace {

constexpr int kMTB = 128, kKTB = 64;
constexpr uint32_t kABytes = kMTB * kKTB * 2;  // dense fp16 tile, 16 KB
constexpr int kTeams = 3;                      // decode teams
constexpr int kTeamWarps = 4;                  // warps per team
constexpr int kWarpDec = 0;                    // decode warps 0 .. 11
constexpr int kWarpEpi = kTeams * kTeamWarps;  // epilogue warps 12 .. 15 (id % 4 = TMEM lane quarter)
constexpr int kWarpX = kWarpEpi + 4;           // 16
constexpr int kWarpPf = kWarpX + 1;            // 17
constexpr int kWarpMma = kWarpX + 3;           // 19
constexpr int kThreads = 32 * (kWarpMma + 1);
constexpr int kChunkG = 24;                    // groups per warp held in registers per team-tile
constexpr int kPrefetchAhead = 32;             // k-tiles of entries kept in flight toward L2
constexpr int kPfChunk = 4;                    // k-tiles per L2 prefetch

template <int NPAD>
struct Cfg {
  static constexpr int kBoxW = NPAD < 64 ? NPAD : 64;        // TMA box / swizzle atom width
  static constexpr int kBoxes = NPAD / kBoxW;
  static constexpr int kTX = NPAD <= 32 ? 4 : (NPAD == 64 ? 2 : 1);  // k-tiles per X stage
  static constexpr uint32_t kBoxBytes = 64u * kTX * kBoxW * 2;
  static constexpr uint32_t kXStage = kBoxBytes * kBoxes;
  static constexpr int kNX = (49152 / kXStage) < 2 ? 2 : ((49152 / kXStage) > 4 ? 4 : (49152 / kXStage));
  static constexpr int kNA = NPAD <= 128 ? 10 : 8;           // dense-tile buffers (even: MMA pairs)
  static constexpr uint32_t kRowBytes = kBoxW * 2;
  static constexpr uint32_t kLayout = kRowBytes == 16 ? 0u : (kRowBytes == 32 ? 6u : (kRowBytes == 64 ? 4u : 2u));
  // SWIZZLE_NONE (NPAD=8): LBO = k-group stride (8 rows x 16 B); swizzled: SBO = 8-row
  // k-group stride, LBO = stride between 64-column atoms.
  static constexpr uint32_t kLBO = kRowBytes == 16 ? 128u : kBoxBytes;
  static constexpr uint32_t kSBO = kRowBytes == 16 ? 128u : 8u * kRowBytes;
  static constexpr uint32_t kKStep = 16u * kRowBytes;        // 16 k-rows per MMA
  static constexpr uint32_t kTileStep = 64u * kRowBytes;     // next k-tile inside a stage
  static constexpr uint32_t kTmemCols = (2 * NPAD) <= 32 ? 32 : ((2 * NPAD) <= 64 ? 64 : ((2 * NPAD) <= 128 ? 128 : ((2 * NPAD) <= 256 ? 256 : 512)));
  static constexpr uint32_t kIdesc = idesc_f16_f32(128, NPAD, 1);
  // smem carve-up (from a 1024-aligned base)
  static constexpr uint32_t kOffX = kNA * kABytes;
  static constexpr uint32_t kOffBar = kOffX + kNX * kXStage;
  static constexpr uint32_t kNumBars = kNA / 2 + 2 * kNX + 4;
  static constexpr uint32_t kOffFlags = kOffBar + 8 * kNumBars;
  static constexpr uint32_t kSmem = 1024 + kOffFlags + 4 * kNA + 16;
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
// debug-only experiment switches (env TCSL_DEBUG): 2 skip scatter, 4 skip zeroing,
// 32 skip entry loads
__constant__ int c_debug;
#define DBG(bit) (c_debug & (bit))
#else
#define DBG(bit) 0
#endif

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

// Walks this CTA's k-tiles in schedule order: (unit, kt, global tile index t).
struct TileWalk {
  int u, kt, kt1;
  uint32_t t;
  __device__ __forceinline__ bool start(const Params& p) {
    u = blockIdx.x;
    return load(p);
  }
  __device__ __forceinline__ bool load(const Params& p) {
    if (u >= p.units) return false;
    const Unit un = unit_of(p, u);
    kt = un.kt0;
    kt1 = un.kt1;
    t = static_cast<uint32_t>(un.rb) * p.tiles_k + un.kt0;
    return true;
  }
  // advance by `steps` tiles (crossing units as needed)
  __device__ __forceinline__ bool advance(const Params& p, int steps) {
    while (steps > 0) {
      const int left = kt1 - kt;
      if (steps < left) {
        kt += steps;
        t += steps;
        return true;
      }
      steps -= left;
      u += gridDim.x;
      if (!load(p)) return false;
    }
    return true;
  }
};

// Number of 32-entry groups of tile [a0, a1); 0 when malformed.
__device__ __forceinline__ uint32_t tile_groups(const Params& p, uint32_t a0, uint32_t a1) {
  return (a0 <= a1 && a1 <= p.n_entries && ((a1 - a0) & 31u) == 0) ? (a1 - a0) >> 5 : 0u;
}

// Byte offset of tile element `loc` (= x*64 + y) in the K-major SWIZZLE_NONE
// canonical layout: (x/8)*1024 + (y/8)*128 + (x%8)*16 + (y%8)*2. Bits >= 13 of
// loc are ignored, so the address is always inside the 16 KB tile.
__device__ __forceinline__ uint32_t a_offset(uint32_t loc) {
  return ((loc << 1) & 0x3C0Eu)  // (y%8)*2 from loc[2:0], (x/8)*1024 from loc[12:9]
         | ((loc >> 2) & 0x70u)  // (x%8)*16 from loc[8:6]
         | ((loc << 4) & 0x380u);  // (y/8)*128 from loc[5:3]
}

__device__ __forceinline__ uint32_t ld_acquire_smem(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_smem_add(uint32_t addr, uint32_t v) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_shared_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Spin on an smem counter until it reaches `target` (watchdog as in mbar_wait).
__device__ __forceinline__ void wait_counter(uint32_t addr, uint32_t target) {
  if (static_cast<int32_t>(ld_acquire_smem(addr) - target) >= 0) return;
  const long long t0 = clock64();
  while (static_cast<int32_t>(ld_acquire_smem(addr) - target) < 0) {
    if (clock64() - t0 > 40000000000LL) __trap();
  }
}

// One decode warp's share of a team-tile: E holds its first kChunkG groups
// (loaded earlier); meanwhile F is filled with its share of the team's next tile.
template <int NA>
__device__ __forceinline__ void decode_tile(const Params& p, uint32_t (&E)[kChunkG], uint32_t (&F)[kChunkG],
                                            uint32_t a_tile, uint32_t a0, uint32_t g0, uint32_t g1,
                                            uint32_t n0, uint32_t ng0, uint32_t ng1, int lane,
                                            uint32_t& err_or) {
  // Straight-line code in blocks of 8 groups: loads are unconditional (clamped to
  // the last valid group), stores predicated in PTX — no per-group branches.
  // Next team-tile's share first, so its L2 latency overlaps this tile's scatter.
  const uint32_t ncnt = ng1 - ng0;
  if (ncnt) {
    const uint32_t* nsrc = p.ent + n0 + 32 * ng0 + lane;
    const uint32_t last = ncnt - 1;
#pragma unroll
    for (int jb = 0; jb < kChunkG; jb += 8) {
      if (static_cast<uint32_t>(jb) >= ncnt) break;
#pragma unroll
      for (int j = jb; j < jb + 8; ++j)
        if (!DBG(32)) F[j] = ldg_stream(nsrc + 32 * min(static_cast<uint32_t>(j), last));
    }
  }
  const uint32_t cnt = g1 - g0;
#pragma unroll
  for (int jb = 0; jb < kChunkG; jb += 8) {
    if (static_cast<uint32_t>(jb) >= cnt) break;
#pragma unroll
    for (int j = jb; j < jb + 8; ++j) {
      // slots past cnt hold duplicates of valid entries (or zeros): harmless for err_or
      err_or |= E[j];
      sts16_if(a_tile + a_offset(E[j]), E[j] >> 16, static_cast<uint32_t>(j) < cnt && !DBG(2));
    }
  }
  // rare: more than kChunkG groups for this warp (density above ~25 %)
  for (uint32_t g = g0 + kChunkG; g < g1; ++g) {
    const uint32_t e = ldg_stream(p.ent + a0 + 32 * g + lane);
    err_or |= e;
    sts16(a_tile + a_offset(e), e >> 16);
  }
}

template <int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
    spmm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  using C = Cfg<NPAD>;
  constexpr int NA = C::kNA;
  constexpr int NX = C::kNX;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t s_a = (raw + 1023u) & ~1023u;
  const uint32_t s_x = s_a + C::kOffX;
  const uint32_t s_bar = s_a + C::kOffBar;
  const uint32_t b_aempty = s_bar;  // [NA/2] MMAs of both tiles of a buffer pair complete
  const uint32_t b_xfull = s_bar + 8 * (NA / 2), b_xempty = b_xfull + 8 * NX;
  const uint32_t b_dfull = b_xempty + 8 * NX, b_dempty = b_dfull + 16;
  const uint32_t s_flags = s_a + C::kOffFlags;  // [NA] decode-warp completions per buffer
  const uint32_t s_tmem_slot = s_flags + 4 * NA;
  const uint32_t s_progress = s_tmem_slot + 4;  // k-tiles the MMA has consumed (prefetch pacing)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + (s_tmem_slot - raw));
  volatile uint32_t* progress = reinterpret_cast<volatile uint32_t*>(smem_raw + (s_progress - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NA / 2; ++i) mbar_init(b_aempty + 8 * i, 1);
    for (int i = 0; i < NA; ++i) st_shared_u32(s_flags + 4 * i, 0);
    for (int i = 0; i < NX; ++i) {
      mbar_init(b_xfull + 8 * i, 1);
      mbar_init(b_xempty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(b_dfull + 8 * i, 1);
      mbar_init(b_dempty + 8 * i, 4);
    }
    *progress = 0;
    fence_barrier_init();
  }
  if (warp == kWarpX && lane == 0) prefetch_tmap(&tmap_x);
  if (warp == kWarpMma) tmem_alloc_dyn(s_tmem_slot, C::kTmemCols);
  for (uint32_t i = threadIdx.x; i < NA * kABytes / 16; i += kThreads) sts128_zero(s_a + 16 * i);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kWarpX) {
    // ---------------------------------------------------------------- X producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      uint32_t gs = 0;  // global X stage counter
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit un = unit_of(p, u);
        for (int kt = un.kt0; kt < un.kt1; kt += C::kTX, ++gs) {
          const uint32_t slot = gs % NX;
          const uint32_t use = gs / NX;
          if (use > 0) mbar_wait_sleep(b_xempty + 8 * slot, (use - 1) & 1);
          mbar_arrive_expect_tx(b_xfull + 8 * slot, C::kXStage);
#pragma unroll
          for (int bx = 0; bx < C::kBoxes; ++bx)
            tma_load_2d(s_x + slot * C::kXStage + bx * C::kBoxBytes, &tmap_x, p.col0 + bx * C::kBoxW, kt * kKTB,
                        b_xfull + 8 * slot, pol);
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ---------------------------------------------------------------- MMA issuer
    // The whole warp walks the schedule (warp-uniform values stay in uniform
    // registers); one elected lane issues. Descriptors are base + byte offset/16.
    const uint64_t a_desc0 = smem_desc(s_a, 128, 1024, 0);
    const uint64_t b_desc0 = smem_desc(s_x, C::kLBO, C::kSBO, C::kLayout);
    uint32_t total = 0;  // k-tiles of this CTA
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const Unit un = unit_of(p, u);
      total += un.kt1 - un.kt0;
    }
    uint32_t gt = 0, ui = 0, gs = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
      const Unit un = unit_of(p, u);
      const uint32_t acc = ui & 1;
      if (ui >= 2) mbar_wait_sleep(b_dempty + 8 * acc, ((ui >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * NPAD;
      for (int kt = un.kt0; kt < un.kt1; ++kt, ++gt) {
        const int in_stage = (kt - un.kt0) % C::kTX;
        const uint32_t xs = gs % NX;
        if (in_stage == 0) mbar_wait(b_xfull + 8 * xs, (gs / NX) & 1);
        const uint32_t b = gt % NA;
        if ((gt & 1u) == 0) {
          // both tiles of the pair decoded? (one sync point per two k-tiles)
          if (lane == 0) TRACE(5, gt);
          wait_counter(s_flags + 4 * b, kTeamWarps * (gt / NA + 1));
          if (gt + 1 < total) wait_counter(s_flags + 4 * (b + 1), kTeamWarps * ((gt + 1) / NA + 1));
          if (lane == 0) TRACE(6, gt);
          tc_fence_after();
        }
        const uint64_t ad = a_desc0 + ((b * kABytes) >> 4);
        const uint64_t bd = b_desc0 + ((xs * C::kXStage + in_stage * C::kTileStep) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int s = 0; s < kKTB / 16; ++s)
            mma_f16_ss(d_tmem, ad + (s * 256 >> 4), bd + (s * C::kKStep >> 4), C::kIdesc,
                       (kt > un.kt0 || s > 0) ? 1u : 0u);
          if ((gt & 1u) || gt + 1 == total) mma_commit(b_aempty + 8 * (b >> 1));
          if (in_stage == C::kTX - 1 || kt + 1 == un.kt1) mma_commit(b_xempty + 8 * xs);
          if ((gt & 3u) == 3u) *progress = gt + 1;
        }
        __syncwarp();
        if (in_stage == C::kTX - 1 || kt + 1 == un.kt1) ++gs;
        if (lane == 0 && (gt & 1u)) TRACE(7, gt - 1);
      }
      if (elect_one()) mma_commit(b_dfull + 8 * acc);
      __syncwarp();
    }
  } else if (warp == kWarpPf) {
    // ---------------------------------------------------------------- L2 prefetcher
    // Keeps the entry spans of the next kPrefetchAhead k-tiles on their way to
    // L2 so the decode warps' loads hit L2 instead of waiting on HBM.
    // A unit's tiles are contiguous in the entry array, so the warp prefetches
    // chunks of kPfChunk tiles; each lane loads the bounds of one chunk (32
    // chunks per offset round trip) and the chunks are issued in order, paced.
    uint32_t base = 0;  // schedule index of the unit's first k-tile
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const Unit un = unit_of(p, u);
      const uint32_t t0 = static_cast<uint32_t>(un.rb) * p.tiles_k + un.kt0;
      const uint32_t nt = un.kt1 - un.kt0;
      for (uint32_t c = 0; c < nt; c += 32 * kPfChunk) {
        const uint32_t my0 = min(c + lane * kPfChunk, nt), my1 = min(my0 + kPfChunk, nt);
        uint32_t lo = 0, hi = 0;
        if (my1 > my0) {
          lo = __ldg(p.off + t0 + my0);
          hi = __ldg(p.off + t0 + my1);
        }
        const bool ok = hi > lo && hi <= p.n_entries && (lo & 3u) == 0;
        for (int i = 0; i < 32; ++i) {
          const uint32_t first = c + i * kPfChunk;
          if (first >= nt) break;
          if (lane == 0)
            while (base + first >= *progress + kPrefetchAhead) __nanosleep(64);
          __syncwarp();
          if (lane == i && ok) bulk_prefetch_l2(p.ent + lo, ((hi - lo) * 4u) & ~15u);
        }
      }
      base += nt;
    }
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
  } else if (warp >= kWarpDec && warp < kWarpDec + kTeams * kTeamWarps) {
    // ---------------------------------------------------------------- decode teams
    // Team t owns the k-tiles gt = t, t + kTeams, ...; each of its 4 warps owns a
    // contiguous quarter of the tile's groups. Two register sets alternate
    // between team-tiles (no copies): while one tile is scattered, the next
    // team-tile's entries are in flight; offsets run two team-tiles ahead.
    const int dw = warp - kWarpDec;
    const int team = dw / kTeamWarps;
    const int tw = dw % kTeamWarps;
    TileWalk w;
    bool more = w.start(p) && w.advance(p, team);
    uint32_t gt = team;
    uint32_t err_or = 0;
    bool bad_off = false;
    uint32_t a0 = 0, a1 = 0, n0 = 0, n1 = 0;
    uint32_t E0[kChunkG], E1[kChunkG];
#pragma unroll
    for (int j = 0; j < kChunkG; ++j) E0[j] = E1[j] = 0u;  // unused slots must not look like bad locations
    bool has_n = false;
    if (more) {
      a0 = __ldg(p.off + w.t);
      a1 = __ldg(p.off + w.t + 1);
      const uint32_t ng = tile_groups(p, a0, a1);
      const uint32_t g0 = ng * tw / kTeamWarps, g1 = ng * (tw + 1) / kTeamWarps;
#pragma unroll
      for (int j = 0; j < kChunkG; ++j)
        if (g0 + j < g1) E0[j] = ldg_stream(p.ent + a0 + 32 * (g0 + j) + lane);
      has_n = w.advance(p, kTeams);
      if (has_n) {
        n0 = __ldg(p.off + w.t);
        n1 = __ldg(p.off + w.t + 1);
      }
    }
    int parity = 0;  // which register set holds the current tile
    while (more) {
      const uint32_t ng = tile_groups(p, a0, a1);
      if (a1 != a0 + 32 * ng) bad_off = true;
      const uint32_t g0 = ng * tw / kTeamWarps, g1 = ng * (tw + 1) / kTeamWarps;
      // offsets of the team's tile after next
      const bool has_nn = has_n && w.advance(p, kTeams);
      uint32_t nn0 = 0, nn1 = 0;
      if (has_nn) {
        nn0 = __ldg(p.off + w.t);
        nn1 = __ldg(p.off + w.t + 1);
      }
      const uint32_t nng = has_n ? tile_groups(p, n0, n1) : 0u;
      const uint32_t ng0 = nng * tw / kTeamWarps, ng1 = nng * (tw + 1) / kTeamWarps;

      const uint32_t b = gt % NA;
      const uint32_t use = gt / NA;
      const uint32_t a_tile = s_a + b * kABytes;
      if (tw == 0 && lane == 0) TRACE(0, gt);
      if (use > 0) {
        // sleep in hardware: spinning try_waits from 12 warps starve the tcgen05 issue path
        mbar_wait_sleep(b_aempty + 8 * (b >> 1), (use - 1) & 1);
        const uint32_t q0 = a_tile + tw * (kABytes / kTeamWarps);
#pragma unroll
        for (int r = 0; r < static_cast<int>(kABytes / kTeamWarps / 512); ++r)
          if (!DBG(4)) sts128_zero(q0 + 512 * r + 16 * lane);
      }
      if (tw == 0 && lane == 0) TRACE(1, gt);
      named_bar_sync(1 + team, kTeamWarps * 32);
      if (tw == 0 && lane == 0) TRACE(2, gt);
      if (DBG(1024)) {
      } else if (parity == 0)
        decode_tile<NA>(p, E0, E1, a_tile, a0, g0, g1, n0, ng0, ng1, lane, err_or);
      else
        decode_tile<NA>(p, E1, E0, a_tile, a0, g0, g1, n0, ng0, ng1, lane, err_or);
      if (tw == 0 && lane == 0) TRACE(3, gt);
      if (!DBG(64)) fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (DBG(128))
          asm volatile("red.relaxed.cta.shared::cta.add.u32 [%0], %1;" ::"r"(s_flags + 4 * b), "r"(1u) : "memory");
        else
          red_release_smem_add(s_flags + 4 * b, 1u);
      }
      if (tw == 0 && lane == 0) TRACE(4, gt);
      parity ^= 1;
      more = has_n;
      a0 = n0;
      a1 = n1;
      has_n = has_nn;
      n0 = nn0;
      n1 = nn1;
      gt += kTeams;
    }
    // locations >= 8192 leave the 128x64 tile (the scatter masked them into range)
    if (__any_sync(0xffffffffu, (err_or & 0xE000u) != 0) && lane == 0)
      raise_dev(p.err, TCSL_STATUS_LOCATION_OUT_OF_RANGE);
    if (__any_sync(0xffffffffu, bad_off) && lane == 0) raise_dev(p.err, TCSL_STATUS_INCONSISTENT_OFFSETS);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
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
  static_assert(C::kSmem <= 227 * 1024, "shared memory budget");
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
  // per-SM streaming rate ~ 6.5 TB/s / 148; MMA floor ~0.1 us per tile
  const double t_tile = std::max(avg_entries_per_tile * 4.0 / 44.0e3, 0.1);
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
#ifdef TCSL_TRACE
  {
    const int dbg = getenv("TCSL_DEBUG") ? atoi(getenv("TCSL_DEBUG")) : 0;
    cudaMemcpyToSymbolAsync(c_debug, &dbg, sizeof dbg, 0, cudaMemcpyHostToDevice, s);
  }
#endif
  // Column slabs of <= 256 (one TMEM accumulator pair each).
  for (int col0 = 0; col0 < plan.n; col0 += 256) {
    const int n_pad = pad_n(std::min(256, plan.n - col0));
    const int box_w = std::min(n_pad, 64);
    const int box_rows = 64 * (n_pad <= 32 ? 4 : (n_pad == 64 ? 2 : 1));  // Cfg<NPAD>::kTX k-tiles per stage
    p.col0 = col0;
    const uint32_t row_bytes = box_w * 2;
    const CUtensorMapSwizzle swz =
        row_bytes == 16 ? CU_TENSOR_MAP_SWIZZLE_NONE
                        : (row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B));
    CUtensorMap tm;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(plan.n), static_cast<cuuint64_t>(k)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_rows)};
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
