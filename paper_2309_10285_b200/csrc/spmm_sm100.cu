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
//   warp 0      entry producer: streams the unit's contiguous entry span
//               [off[t0], off[t1]) with cp.async.bulk into a ring of 4 KB chunks
//   warp 1      X producer: TMA-loads the 64 x n_pad activation tile per k-tile
//               (MN-major, hardware swizzle = 2*n_pad bytes)
//   warp 2      TMEM owner + single-thread tcgen05.mma issuer (M=128, N=n_pad, K=16 x 4)
//   warps 4-7   epilogue: tcgen05.ld accumulator -> fp32 Y rows (or split-K partials)
//   warps 8-15  decode: scatter each 32-entry group (one entry per lane) into the
//               dense tile in the SWIZZLE_NONE K-major core-matrix layout
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
constexpr int kABytes = kMTB * kKTB * 2;  // dense fp16 tile, 16 KB
constexpr int kNA = 3;                    // dense-tile buffers
constexpr int kNDec = 8;                  // decode warps
constexpr int kChunk = 1024;              // entries per ring chunk (4 KB)
constexpr int kThreads = 512;
constexpr int kWarpEpi = 4, kWarpDec = 8;

struct Params {
  const uint32_t* off;
  const uint32_t* ent;
  uint64_t n_entries;
  uint32_t m, k;
  int tiles_m, tiles_k;
  int n, n_pad, col0, split, units;
  float* out;
  int ldo;
  int* err;
  int nx, ring;
  uint32_t x_stage, x_box_bytes;
  int x_boxes, box_w;
  uint32_t tmem_cols, idesc, b_layout, b_lbo, b_sbo, b_kstep;
};

struct Bars {
  uint32_t base;
  int nx, ring;
  __device__ uint32_t afull(int i) const { return base + 8 * i; }
  __device__ uint32_t aempty(int i) const { return base + 8 * (kNA + i); }
  __device__ uint32_t xfull(int i) const { return base + 8 * (2 * kNA + i); }
  __device__ uint32_t xempty(int i) const { return base + 8 * (2 * kNA + nx + i); }
  __device__ uint32_t efull(int i) const { return base + 8 * (2 * kNA + 2 * nx + i); }
  __device__ uint32_t eempty(int i) const { return base + 8 * (2 * kNA + 2 * nx + ring + i); }
  __device__ uint32_t dfull(int i) const { return base + 8 * (2 * kNA + 2 * nx + 2 * ring + i); }
  __device__ uint32_t dempty(int i) const { return base + 8 * (2 * kNA + 2 * nx + 2 * ring + 2 + i); }
  __device__ uint32_t count() const { return 2 * kNA + 2 * nx + 2 * ring + 4; }
};

__host__ __device__ inline size_t bar_bytes(int nx, int ring) { return 8ull * (2 * kNA + 2 * nx + 2 * ring + 4) + 16; }

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

// Byte offset of tile element `loc` (= x*64 + y) in the K-major SWIZZLE_NONE
// canonical layout: (x/8)*1024 + (y/8)*128 + (x%8)*16 + (y%8)*2.
__device__ __forceinline__ uint32_t a_offset(uint32_t loc) {
  return ((loc << 1) & 0x3C0Eu)      // (y%8)*2 from loc[2:0], (x/8)*1024 from loc[12:9]
         | ((loc >> 2) & 0x70u)      // (x%8)*16 from loc[8:6]
         | ((loc << 4) & 0x380u);    // (y/8)*128 from loc[5:3]
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    spmm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t s_a = smem_u32(smem);
  const uint32_t s_x = s_a + kNA * kABytes;
  const uint32_t s_e = s_x + p.nx * p.x_stage;
  const uint32_t* ring_e = reinterpret_cast<const uint32_t*>(smem + (s_e - s_a));
  Bars bars{s_e + static_cast<uint32_t>(p.ring) * kChunk * 4, p.nx, p.ring};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + (bars.base - s_a) + 8 * bars.count());

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNA; ++i) {
      mbar_init(bars.afull(i), kNDec);
      mbar_init(bars.aempty(i), 1);
    }
    for (int i = 0; i < p.nx; ++i) {
      mbar_init(bars.xfull(i), 1);
      mbar_init(bars.xempty(i), 1);
    }
    for (int i = 0; i < p.ring; ++i) {
      mbar_init(bars.efull(i), 1);
      mbar_init(bars.eempty(i), kNDec);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bars.dfull(i), 1);
      mbar_init(bars.dempty(i), 4);
    }
    fence_barrier_init();
  }
  if (warp == 1 && lane == 0) prefetch_tmap(&tmap_x);
  if (warp == 2) tmem_alloc_dyn(smem_u32(tmem_slot), p.tmem_cols);
  {  // dense tiles start as +0.0 everywhere
    uint4* a4 = reinterpret_cast<uint4*>(smem);
    for (int i = threadIdx.x; i < kNA * kABytes / 16; i += kThreads) a4[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- entry producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t g = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit un = unit_of(p, u);
        uint32_t e0, e1;
        if (!unit_span(p, un, e0, e1)) raise_dev(p.err, TCSL_STATUS_INCONSISTENT_OFFSETS);
        for (uint32_t c0 = e0; c0 < e1; c0 += kChunk, ++g) {
          const int slot = static_cast<int>(g % p.ring);
          const uint32_t use = g / p.ring;
          if (use > 0) mbar_wait(bars.eempty(slot), (use - 1) & 1);
          const uint32_t bytes = min(static_cast<uint32_t>(kChunk), e1 - c0) * 4;
          mbar_arrive_expect_tx(bars.efull(slot), bytes);
          bulk_g2s(s_e + slot * kChunk * 4, p.ent + c0, bytes, bars.efull(slot), pol);
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
          const int slot = static_cast<int>(gt % p.nx);
          const uint32_t use = gt / p.nx;
          if (use > 0) mbar_wait(bars.xempty(slot), (use - 1) & 1);
          mbar_arrive_expect_tx(bars.xfull(slot), p.x_stage);
          for (int bx = 0; bx < p.x_boxes; ++bx)
            tma_load_2d(s_x + slot * p.x_stage + bx * p.x_box_bytes, &tmap_x, p.col0 + bx * p.box_w, kt * kKTB,
                        bars.xfull(slot), pol);
        }
      }
    }
  } else if (warp == 2) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      uint32_t gt = 0, ui = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
        const Unit un = unit_of(p, u);
        const int acc = static_cast<int>(ui & 1);
        if (ui >= 2) mbar_wait(bars.dempty(acc), ((ui >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + static_cast<uint32_t>(acc * p.n_pad);
        for (int kt = un.kt0; kt < un.kt1; ++kt, ++gt) {
          const int b = static_cast<int>(gt % kNA);
          const int xs = static_cast<int>(gt % p.nx);
          mbar_wait(bars.afull(b), (gt / kNA) & 1);
          mbar_wait(bars.xfull(xs), (gt / p.nx) & 1);
          tc_fence_after();
          const uint32_t a0 = s_a + b * kABytes;
          const uint32_t b0 = s_x + xs * p.x_stage;
#pragma unroll
          for (int s = 0; s < kKTB / 16; ++s) {
            const uint64_t ad = smem_desc(a0 + s * 256, 128, 1024, 0);
            const uint64_t bd = smem_desc(b0 + s * p.b_kstep, p.b_lbo, p.b_sbo, p.b_layout);
            mma_f16_ss(d_tmem, ad, bd, p.idesc, (kt > un.kt0 || s > 0) ? 1u : 0u);
          }
          mma_commit(bars.aempty(b));
          mma_commit(bars.xempty(xs));
        }
        mma_commit(bars.dfull(acc));
      }
    }
    __syncwarp();
  } else if (warp >= kWarpEpi && warp < kWarpEpi + 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lanes 32q..32q+31
    uint32_t ui = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++ui) {
      const Unit un = unit_of(p, u);
      const int acc = static_cast<int>(ui & 1);
      mbar_wait(bars.dfull(acc), (ui >> 1) & 1);
      tc_fence_after();
      const long long row = static_cast<long long>(un.rb) * kMTB + q * 32 + lane;
      float* dst = p.out + (p.split > 1 ? static_cast<long long>(un.s) * p.m * p.ldo : 0ll) + row * p.ldo + p.col0;
      const bool row_ok = row < p.m;
      const uint32_t t_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * p.n_pad);
      const int ncol = min(p.n_pad, p.n - p.col0);
      if (p.n_pad == 8) {
        uint32_t r[8];
        tmem_ld8(t_base, r);
        tmem_ld_wait();
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < ncol) dst[j] = __uint_as_float(r[j]);
        }
      } else {
        for (int c0 = 0; c0 < p.n_pad; c0 += 16) {
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
      if (lane == 0) mbar_arrive(bars.dempty(acc));
    }
  } else if (warp >= kWarpDec) {
    // ---------------------------------------------------------------- decode
    const int dw = warp - kWarpDec;
    uint32_t gt = 0;
    uint32_t g_base = 0;  // first ring chunk of the current unit
    uint32_t nxt = 0;     // chunks < nxt have been waited full
    uint32_t rel = 0;     // chunks < rel have been released
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const Unit un = unit_of(p, u);
      uint32_t e0, e1;
      unit_span(p, un, e0, e1);
      const uint32_t nchunks = (e1 - e0 + kChunk - 1) / kChunk;
      for (int kt = un.kt0; kt < un.kt1; ++kt, ++gt) {
        const int b = static_cast<int>(gt % kNA);
        const uint32_t use = gt / kNA;
        uint8_t* a_tile = smem + b * kABytes;
        if (use > 0) {
          mbar_wait(bars.aempty(b), (use - 1) & 1);
          uint4* a4 = reinterpret_cast<uint4*>(a_tile);
          for (int i = dw * 32 + lane; i < kABytes / 16; i += kNDec * 32) a4[i] = make_uint4(0, 0, 0, 0);
        }
        named_bar_sync(1, kNDec * 32);
        const uint32_t t = static_cast<uint32_t>(un.rb) * p.tiles_k + kt;
        const uint32_t a0 = __ldg(p.off + t), a1 = __ldg(p.off + t + 1);
        uint32_t ng = 0;
        if (e0 <= a0 && a0 <= a1 && a1 <= e1 && ((a1 - a0) & 31u) == 0) {
          ng = (a1 - a0) >> 5;
        } else if (dw == 0 && lane == 0) {
          raise_dev(p.err, TCSL_STATUS_INCONSISTENT_OFFSETS);
        }
        for (uint32_t gi = dw; gi < ng; gi += kNDec) {
          const uint32_t pos = a0 - e0 + gi * 32;
          const uint32_t c = g_base + pos / kChunk;
          while (nxt <= c) {
            mbar_wait(bars.efull(nxt % p.ring), (nxt / p.ring) & 1);
            ++nxt;
          }
          while (rel < c) {
            __syncwarp();
            if (lane == 0) mbar_arrive(bars.eempty(rel % p.ring));
            ++rel;
          }
          const uint32_t e = ring_e[(c % p.ring) * kChunk + (pos % kChunk) + lane];
          const uint32_t loc = e & 0xFFFFu;
          if (loc < kMTB * kKTB) {
            *reinterpret_cast<uint16_t*>(a_tile + a_offset(loc)) = static_cast<uint16_t>(e >> 16);
          } else {
            raise_dev(p.err, TCSL_STATUS_LOCATION_OUT_OF_RANGE);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bars.afull(b));
      }
      // release every chunk of this unit (waiting for each first: see SURVEY-style
      // phase rule — an arrival may only count toward the chunk it belongs to)
      const uint32_t g_end = g_base + nchunks;
      while (nxt < g_end) {
        mbar_wait(bars.efull(nxt % p.ring), (nxt / p.ring) & 1);
        ++nxt;
      }
      __syncwarp();
      while (rel < g_end) {
        if (lane == 0) mbar_arrive(bars.eempty(rel % p.ring));
        ++rel;
      }
      g_base = g_end;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, p.tmem_cols);
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
  return std::min(256, (n + 63) / 64 * 64);
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

}  // namespace

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
  plan->n_pad = pad_n(n);
  plan->split = split_k > 0 ? std::min(split_k, tiles_k) : 1;
  plan->units = tiles_m * plan->split;
  plan->grid = std::min(plan->units, num_sms());
  const uint32_t x_stage = 64u * plan->n_pad * 2;
  const int nx = std::max(2, std::min(8, static_cast<int>((48u * 1024) / x_stage)));
  const size_t fixed = 1024 + static_cast<size_t>(kNA) * kABytes + static_cast<size_t>(nx) * x_stage;
  int ring = static_cast<int>((200u * 1024 - fixed) / (kChunk * 4));
  ring = std::max(4, std::min(32, ring));
  plan->smem = fixed + static_cast<size_t>(ring) * kChunk * 4 + bar_bytes(nx, ring);
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
  const uint32_t x_stage_full = 64u * plan.n_pad * 2;
  p.nx = std::max(2, std::min(8, static_cast<int>((48u * 1024) / x_stage_full)));
  const size_t fixed = 1024 + static_cast<size_t>(kNA) * kABytes + static_cast<size_t>(p.nx) * x_stage_full;
  p.ring = std::max(4, std::min(32, static_cast<int>((200u * 1024 - fixed) / (kChunk * 4))));

  // Column slabs of <= 256 (one TMEM accumulator pair each).
  for (int col0 = 0; col0 < plan.n; col0 += 256) {
    const int n_here = std::min(256, plan.n - col0);
    const int n_pad = pad_n(n_here);
    p.col0 = col0;
    p.n_pad = n_pad;
    p.box_w = std::min(n_pad, 64);
    p.x_boxes = n_pad / p.box_w;
    p.x_box_bytes = 64u * p.box_w * 2;
    p.x_stage = p.x_box_bytes * p.x_boxes;
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(2 * n_pad)) cols <<= 1;
    p.tmem_cols = cols;
    p.idesc = idesc_f16_f32(128, n_pad, 1);
    CUtensorMapSwizzle swz;
    if (p.box_w == 8) {
      swz = CU_TENSOR_MAP_SWIZZLE_NONE;
      p.b_layout = 0;
      p.b_lbo = 128;  // k-group (8 rows x 16 B) stride
      p.b_sbo = 128;
    } else {
      const uint32_t row_bytes = p.box_w * 2;  // 32 / 64 / 128
      swz = row_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                            : (row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
      p.b_layout = row_bytes == 32 ? 6u : (row_bytes == 64 ? 4u : 2u);
      p.b_sbo = 8 * row_bytes;    // stride between 8-row k-groups
      p.b_lbo = p.x_box_bytes;    // stride between 64-column atoms (n_pad > 64)
    }
    p.b_kstep = 16 * p.box_w * 2;  // 16 k-rows per MMA
    CUtensorMap tm;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(plan.n), static_cast<cuuint64_t>(k)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(p.box_w), 64u};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<uint16_t*>(x), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    const size_t smem = 1024 + static_cast<size_t>(kNA) * kABytes + static_cast<size_t>(p.nx) * p.x_stage +
                        static_cast<size_t>(p.ring) * kChunk * 4 + bar_bytes(p.nx, p.ring);
    cudaError_t e = cudaFuncSetAttribute(spmm_sm100_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    spmm_sm100_kernel<<<plan.grid, kThreads, smem, s>>>(tm, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tcslk
