// Microbenchmark (debug tool, not product): cycles per iteration of the SpMM's
// MMA-issuer loop shape on a CTA pair: wait on an already-completed mbarrier,
// elect, 4 x tcgen05.mma.cta_group::2 (M=256, N=16, K=16), multicast commit to
// both CTAs; optionally with 16 busy warps per CTA doing STS (decode-like load).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_loop_bench tools/mma_loop_bench.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

// WAIT: 0 none, 1 try_wait, 2 test_wait; TPI tiles per iteration (one wait per iteration)
template <int BUSY, int DO_MMA, int COMMIT_EVERY, int WAIT = 1, int TPI = 1, int ONE_THREAD = 0, int CLK = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(576, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + 8 * 16384, bars = sb + 16384;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < (8 * 16384 + 16384) / 16; i += blockDim.x) sts128_zero(base + 16 * i);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(bars + 8 * i, 1);
    mbar_arrive(bars + 8 * 15);  // bar 15: completed phase 0 (the "A full" the issuer polls)
    stop = 0;
    fence_barrier_init();
  }
  if (warp == 17) tmem_alloc_pair(smem_u32(&tslot), 512);
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 17) {
    if (rank == 0 && (!ONE_THREAD || lane == 0)) {
      const uint32_t idesc = idesc_f16_f32(256, 16, 1);
      const uint64_t a0 = smem_desc(sa, 128, 1024, 0), b0 = smem_desc(sb, 128, 128, 0);
      const long long t0 = clock64();
      long long acc_clk = 0;
      for (int it = 0; it < iters; it += TPI) {
#pragma unroll
        for (int c = 0; c < CLK; ++c) acc_clk += clock64() * (c + 1);
        if (WAIT == 1) mbar_wait(bars + 8 * 15, 0);
        if (WAIT == 2) while (!mbar_test_wait(bars + 8 * 15, 0)) {}
        tc_fence_after();
        if (ONE_THREAD || elect_one()) {
#pragma unroll
          for (int t = 0; t < TPI; ++t) {
            const uint64_t ad = a0 + ((((it + t) & 7) * 16384) >> 4);
            if (DO_MMA) {
#pragma unroll
              for (int k4 = 0; k4 < 4; ++k4) mma_f16_ss_pair(tmem, ad + (k4 * 256 >> 4), b0 + (k4 * 256 >> 4), idesc, 1u);
            }
            if (((it + t) % COMMIT_EVERY) == COMMIT_EVERY - 1) mma_commit_pair(bars + 8 * ((it + t) & 7), 3);
          }
        }
        if (!ONE_THREAD) __syncwarp();
      }
      if (ONE_THREAD || elect_one()) mma_commit_pair(bars + 8 * 8, 3);
      if (!ONE_THREAD) __syncwarp();
      mbar_wait(bars + 8 * 8, 0);
      if (lane == 0) out[blockIdx.x] = (clock64() - t0) / iters + (acc_clk == 42 ? 1 : 0);
      stop = 1;
    }
  } else if (BUSY && warp < 16) {
    // decode-like load: 16 warps scattering 16-bit stores into buffers the MMA does not read
    uint32_t v = threadIdx.x * 2654435761u;
    const uint32_t zone = sb;  // B region (the MMA reads only the first 512 B)
    const long long tb = clock64();
    while (!stop && clock64() - tb < 3000000) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        v = v * 1664525u + 1013904223u;
        sts16(zone + 4096 + ((v >> 8) & 0x2FFEu), v);
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 17) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

template <int BUSY, int DO_MMA, int COMMIT_EVERY, int WAIT = 1, int TPI = 1, int ONE_THREAD = 0, int CLK = 0>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaMemset(d, 0, 148 * 8);
  const int smem = 9 * 16384 + 2048;
  cudaFuncSetAttribute(bench<BUSY, DO_MMA, COMMIT_EVERY, WAIT, TPI, ONE_THREAD, CLK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<BUSY, DO_MMA, COMMIT_EVERY, WAIT, TPI, ONE_THREAD, CLK><<<148, 576, smem>>>(2000, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; i += 2) mx = h[i] > mx ? h[i] : mx;
  printf("%-44s %6lld cycles per pair-tile iteration [%s]\n", name, mx, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 0, 1000000, 0, 1, 1, 0>("idle, 1 thread, empty loop");
  run<0, 0, 1000000, 0, 1, 1, 6>("idle, 1 thread, 6 clock64 reads");
  run<1, 0, 1000000, 0, 1, 1, 6>("busy, 1 thread, 6 clock64 reads");
  run<1, 1, 1, 0, 1, 1, 0>("busy, 1 thread, MMA, commit/tile");
  run<1, 1, 1, 0, 1, 1, 6>("busy, 1 thread, MMA, commit/tile, 6 clocks");
  run<1, 1, 1, 1, 1, 1, 0>("busy, 1 thread, MMA, commit/tile, try_wait");
  run<0, 0, 1000000, 0>("idle, no MMA, no commit, no wait");
  run<0, 0, 1, 0>("idle, no MMA, commit/tile, no wait");
  run<0, 0, 1, 1>("idle, no MMA, commit/tile, try_wait");
  run<0, 1, 1000000, 0>("idle, MMA, no commit, no wait");
  run<1, 0, 1000000, 0>("busy, no MMA, no commit, no wait");
  run<1, 0, 1, 0>("busy, no MMA, commit/tile, no wait");
  run<1, 0, 1, 1>("busy, no MMA, commit/tile, try_wait");
  run<0, 1, 1>("idle, MMA, commit/tile, try_wait");
  run<0, 1, 1, 0>("idle, MMA, commit/tile, no wait");
  run<0, 1, 1, 2>("idle, MMA, commit/tile, test_wait");
  run<0, 1, 1, 1, 1, 1>("idle, MMA, commit/tile, try_wait, 1 thread");
  run<0, 1, 1, 1, 2>("idle, MMA, commit/tile, try_wait, 2 tiles/iter");
  run<0, 1, 1, 1, 4>("idle, MMA, commit/tile, try_wait, 4 tiles/iter");
  run<1, 1, 1>("busy, MMA, commit/tile, try_wait");
  run<1, 1, 1, 0>("busy, MMA, commit/tile, no wait");
  run<1, 1, 1, 1, 2>("busy, MMA, commit/tile, try_wait, 2 tiles/iter");
  run<1, 1, 1, 1, 4>("busy, MMA, commit/tile, try_wait, 4 tiles/iter");
  run<1, 1, 2, 1, 4>("busy, MMA, commit/2 tiles, try_wait, 4 tiles/iter");
  return 0;
}
