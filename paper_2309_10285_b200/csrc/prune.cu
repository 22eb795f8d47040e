// GPU magnitude pruning, bit-exact with tcsl::prune_magnitude
// (reference: proj/src/matrix.cpp:69-100; KATs proj/tests/test_matrix.cpp:54-104).
//
// The reference ranks every element by |value| (NaN as +inf), breaks ties by
// row-major index DESCENDING (the larger index is pruned first), and zeroes the
// first cut = floor(beta * n) elements of that strict total order (nth_element).
// For binary16, |value| ordering is the ordering of the 15-bit pattern
// (b & 0x7FFF) for non-NaN values, and NaN shares +inf's rank, so the rank key
// is key(b) = min(b & 0x7FFF, 0x7C00): 31745 distinct keys. Radix select:
//   1. histogram of the keys (one HBM read of A);
//   2. one block scans the histogram: threshold key T with
//      #(key < T) < cut <= #(key <= T), and r = cut - #(key < T) elements of key
//      T to prune — the r with the LARGEST indices among the E_T elements of key T;
//   3. per 8192-element chunk, the number of key-T elements; exclusive scan;
//   4. write: prune key < T, and key == T with global rank (in index order) >= E_T - r.
// Every pass is a coalesced stream over A (HBM-bound); the result does not
// depend on thread scheduling.
#include <cub/cub.cuh>

#include "tcsl_internal.cuh"

namespace tcslk {

namespace {

constexpr uint32_t kKeys = 0x7C01;    // keys 0 .. 0x7C00
constexpr int kChunk = 8192;          // elements per chunk in passes 3-4
constexpr int kThreads = 256;
constexpr int kPerThread = kChunk / kThreads;  // 32

__device__ __forceinline__ uint32_t rank_key(uint32_t b) {
  const uint32_t k = b & 0x7FFFu;
  return k > 0x7C00u ? 0x7C00u : k;  // NaN ranks with +inf (matrix.cpp:80-81)
}

struct PruneWs {
  size_t hist, sel, cnt, pre, temp, total, temp_bytes;
};

__host__ PruneWs prune_layout(uint64_t count) {
  PruneWs w{};
  auto a256 = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t chunks = (count + kChunk - 1) / kChunk;
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                static_cast<int>(chunks > 0 ? chunks : 1));
  size_t o = 0;
  w.hist = o; o += a256(8ull * kKeys);
  w.sel = o;  o += a256(64);
  w.cnt = o;  o += a256(4ull * (chunks + 1));
  w.pre = o;  o += a256(4ull * (chunks + 1));
  w.temp = o; o += a256(temp);
  w.temp_bytes = temp;
  w.total = o;
  return w;
}

// Pass 1: key histogram. Block-private smem histogram (124 KB), flushed with
// 64-bit global atomics for the non-empty bins.
__global__ void __launch_bounds__(1024) prune_hist_kernel(const uint16_t* __restrict__ a, uint64_t count,
                                                          unsigned long long* __restrict__ hist) {
  extern __shared__ uint32_t h[];
  for (uint32_t i = threadIdx.x; i < kKeys; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n2 = count / 2;  // pairs: 32-bit loads (the base is 2-byte aligned at worst, checked on host)
  const uint32_t* a2 = reinterpret_cast<const uint32_t*>(a);
  if ((reinterpret_cast<uintptr_t>(a) & 3u) == 0) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) {
      const uint32_t v = __ldg(a2 + i);
      atomicAdd(&h[rank_key(v & 0xFFFFu)], 1u);
      atomicAdd(&h[rank_key(v >> 16)], 1u);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (count & 1)) atomicAdd(&h[rank_key(a[count - 1])], 1u);
  } else {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
      atomicAdd(&h[rank_key(a[i])], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kKeys; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, static_cast<unsigned long long>(h[i]));
}

// Pass 2 (one block): sel[0] = T, sel[1] = E_T - r (first pruned rank among key T),
// sel[2] = 1 when anything is pruned.
__global__ void __launch_bounds__(1024) prune_select_kernel(const unsigned long long* __restrict__ hist,
                                                            uint64_t cut, unsigned long long* __restrict__ sel) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr uint32_t kPer = (kKeys + 1023) / 1024;  // 31 bins per thread
  const uint32_t b0 = threadIdx.x * kPer;
  unsigned long long mine = 0;
  for (uint32_t i = 0; i < kPer; ++i)
    if (b0 + i < kKeys) mine += hist[b0 + i];
  unsigned long long before = 0;
  Scan(tmp).ExclusiveSum(mine, before);
  if (threadIdx.x == 0) sel[2] = cut > 0 ? 1ull : 0ull;
  if (cut == 0) return;
  // the thread whose bins hold the cut-th element (1-based) finds T
  if (before < cut && cut <= before + mine) {
    unsigned long long cum = before;
    for (uint32_t i = 0; i < kPer; ++i) {
      const unsigned long long c = hist[b0 + i];
      if (cum + c >= cut) {
        const unsigned long long r = cut - cum;  // prune r of the c elements with key T
        sel[0] = b0 + i;
        sel[1] = c - r;
        break;
      }
      cum += c;
    }
  }
}

// Pass 3: number of key-T elements per chunk.
__global__ void __launch_bounds__(kThreads) prune_count_kernel(const uint16_t* __restrict__ a, uint64_t count,
                                                               const unsigned long long* __restrict__ sel,
                                                               uint32_t* __restrict__ cnt) {
  if (sel[2] == 0) return;
  const uint32_t T = static_cast<uint32_t>(sel[0]);
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kChunk;
  uint32_t c = 0;
#pragma unroll 8
  for (int j = 0; j < kPerThread; ++j) {
    const uint64_t i = base + static_cast<uint64_t>(j) * kThreads + threadIdx.x;
    if (i < count) c += rank_key(__ldg(a + i)) == T;
  }
  using Red = cub::BlockReduce<uint32_t, kThreads>;
  __shared__ typename Red::TempStorage tmp;
  const uint32_t tot = Red(tmp).Sum(c);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

// Pass 4: write the pruned copy. Element i of key T has global rank
// pre[chunk] + (its rank inside the chunk, in index order).
__global__ void __launch_bounds__(kThreads) prune_write_kernel(const uint16_t* __restrict__ a, uint64_t count,
                                                               const unsigned long long* __restrict__ sel,
                                                               const uint32_t* __restrict__ pre,
                                                               uint16_t* __restrict__ out) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kChunk;
  const bool any = sel[2] != 0;
  const uint32_t T = any ? static_cast<uint32_t>(sel[0]) : 0xFFFFFFFFu;
  const unsigned long long first = any ? sel[1] : 0ull;
  using Scan = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename Scan::TempStorage tmp;
  unsigned long long rank = any ? pre[blockIdx.x] : 0ull;  // key-T elements before this chunk
  for (int j = 0; j < kPerThread; ++j) {
    const uint64_t i = base + static_cast<uint64_t>(j) * kThreads + threadIdx.x;
    const uint16_t v = i < count ? a[i] : 0;
    const uint32_t key = rank_key(v);
    const uint32_t eq = (i < count && key == T) ? 1u : 0u;
    uint32_t ex = 0, agg = 0;
    Scan(tmp).ExclusiveSum(eq, ex, agg);
    __syncthreads();  // tmp reuse
    if (i < count) {
      const bool prune = any && (key < T || (eq && rank + ex >= first));
      out[i] = prune ? 0 : v;
    }
    rank += agg;
  }
}

}  // namespace

size_t prune_workspace_bytes(uint64_t count) { return prune_layout(count).total; }

cudaError_t launch_prune(const uint16_t* a, uint64_t count, uint64_t cut, uint16_t* out, void* ws, size_t ws_bytes,
                         cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const PruneWs L = prune_layout(count);
  if (ws_bytes < L.total) return cudaErrorInvalidValue;
  char* w = static_cast<char*>(ws);
  auto* hist = reinterpret_cast<unsigned long long*>(w + L.hist);
  auto* sel = reinterpret_cast<unsigned long long*>(w + L.sel);
  auto* cnt = reinterpret_cast<uint32_t*>(w + L.cnt);
  auto* pre = reinterpret_cast<uint32_t*>(w + L.pre);
  const uint64_t chunks = (count + kChunk - 1) / kChunk;
  if (chunks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(hist, 0, 8ull * kKeys, s);
  if (e != cudaSuccess) return e;
  const int hsm = static_cast<int>(4 * kKeys);
  e = cudaFuncSetAttribute(prune_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, hsm);
  if (e != cudaSuccess) return e;
  const int blocks = static_cast<int>(std::min<uint64_t>((count + 2047) / 2048, static_cast<uint64_t>(num_sms())));
  prune_hist_kernel<<<blocks, 1024, hsm, s>>>(a, count, hist);
  prune_select_kernel<<<1, 1024, 0, s>>>(hist, cut, sel);
  prune_count_kernel<<<static_cast<unsigned>(chunks), kThreads, 0, s>>>(a, count, sel, cnt);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  size_t tb = L.temp_bytes;
  e = cub::DeviceScan::ExclusiveSum(w + L.temp, tb, cnt, pre, static_cast<int>(chunks), s);
  if (e != cudaSuccess) return e;
  prune_write_kernel<<<static_cast<unsigned>(chunks), kThreads, 0, s>>>(a, count, sel, pre, out);
  return cudaGetLastError();
}

}  // namespace tcslk
