// Microbenchmark (debug tool, not product): latencies of the synchronisation
// primitives the SpMM's producer warps use, measured with clock64 on one SM.
//  1. try_wait loop: iterations and wake-up latency when the phase completes
//     T cycles after the waiter started (another warp arrives)
//  2. same with test_wait (non-blocking) polling
//  3. cost per op, single thread, back to back: arrive.expect_tx, test_wait on a
//     completed phase, cp.async.bulk issue (8 KB, 16 KB), remote arrive (cluster)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sync_bench tools/sync_bench.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

__global__ void __cluster_dims__(2, 1, 1) bench(const uint8_t* src, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = smem_u32(smem);
  const uint32_t bars = base;           // 64 barriers
  const uint32_t buf = base + 1024;     // 64 KB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) mbar_init(bars + 8 * i, (i >= 8 && i < 40) ? 2 : (i == 63 ? 1000 : 1));
    fence_barrier_init();
  }
  cluster_sync_all();
  if (rank != 0) {
    cluster_sync_all();
    return;
  }
  long long* o = out;
  // ---- 1/2: waiter warp 0, arriver warp 1 (after `delay` cycles)
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      const uint32_t bar = bars + 8 * (mode * 3 + rep);
      const long long delay = 20000;
      __syncthreads();
      __shared__ long long t_start, t_arrive;
      if (warp == 1 && lane == 0) {
        const long long t0 = clock64();
        t_start = t0;
        while (clock64() - t0 < delay) {
        }
        t_arrive = clock64();
        mbar_arrive(bar);
      }
      if (warp == 0 && lane == 0) {
        long long iters = 0;
        if (mode == 0) {
          while (!mbar_try_wait(bar, 0)) ++iters;
        } else {
          while (!mbar_test_wait(bar, 0)) ++iters;
        }
        const long long t_done = clock64();
        __syncwarp(1);
        o[mode * 8 + rep * 2] = iters;
        o[mode * 8 + rep * 2 + 1] = t_done;  // fixed up below
      }
      __syncthreads();
      if (threadIdx.x == 0) o[mode * 8 + rep * 2 + 1] -= t_arrive;
    }
  }
  __syncthreads();
  // ---- 3: single-thread op costs
  if (threadIdx.x == 0) {
    const int n = 64;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) mbar_arrive_expect_tx(bars + 8 * (8 + (i & 31)), 128);
    long long t1 = clock64();
    o[16] = (t1 - t0) / n;
    // test_wait on incomplete phase
    t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < n; ++i) acc += mbar_test_wait(bars + 8 * (8 + (i & 31)), 0);
    t1 = clock64();
    o[17] = (t1 - t0) / n + (acc == 12345);
    // try_wait on incomplete phase (times out)
    t0 = clock64();
    for (int i = 0; i < 4; ++i) acc += mbar_try_wait(bars + 8 * (8 + i), 0);
    t1 = clock64();
    o[18] = (t1 - t0) / 4 + (acc == 12345);
    // bulk copy issue, 8 KB, into 8 slots (fresh barriers 40..47)
    const uint64_t pol = policy_evict_first();
    t0 = clock64();
    for (int i = 0; i < 8; ++i) {
      mbar_arrive_expect_tx(bars + 8 * (40 + i), 8192);
      bulk_g2s(buf + 8192 * i, src + 8192 * i, 8192, bars + 8 * (40 + i), pol);
    }
    t1 = clock64();
    o[19] = (t1 - t0) / 8;
    for (int i = 0; i < 8; ++i) mbar_wait(bars + 8 * (40 + i), 0);
    long long t2 = clock64();
    o[20] = t2 - t0;  // 64 KB landed
    // remote arrive to the peer (cluster) barrier 63
    const uint32_t remote = mapa_shared(bars + 8 * 63, 1);
    t0 = clock64();
    for (int i = 0; i < 16; ++i) mbar_arrive_cluster(remote);
    t1 = clock64();
    o[21] = (t1 - t0) / 16;
    // lds latency chain
    t0 = clock64();
    uint32_t v = 0;
    for (int i = 0; i < 16; ++i) v = lds32(buf + (v & 4));
    t1 = clock64();
    o[22] = (t1 - t0) / 16 + (v == 12345);
  }
  __syncthreads();
  cluster_sync_all();
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 1 << 20);
  cudaMemset(src, 1, 1 << 20);
  long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaMemset(d, 0, 64 * 8);
  const int smem = 1024 + 65536;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<<<2, 64, smem>>>(src, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[64];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("status %s\n", cudaGetErrorString(e));
  for (int rep = 0; rep < 3; ++rep)
    printf("try_wait  loop (arrive after 20000 cyc): %lld iterations, wake-up %lld cycles after the arrive\n",
           h[rep * 2], h[rep * 2 + 1]);
  for (int rep = 0; rep < 3; ++rep)
    printf("test_wait loop (arrive after 20000 cyc): %lld iterations, wake-up %lld cycles after the arrive\n",
           h[8 + rep * 2], h[8 + rep * 2 + 1]);
  printf("arrive.expect_tx: %lld cyc/op\n", h[16]);
  printf("test_wait (incomplete): %lld cyc/op\n", h[17]);
  printf("try_wait (incomplete, returns false): %lld cyc/op\n", h[18]);
  printf("expect_tx + cp.async.bulk 8 KB issue: %lld cyc/op; 64 KB landed after %lld cyc\n", h[19], h[20]);
  printf("remote mbarrier arrive: %lld cyc/op\n", h[21]);
  printf("dependent LDS: %lld cyc/op\n", h[22]);
  return 0;
}
