// Microbenchmark (debug tool, not product): does a CTA pair (cta_group::2,
// M=256) double the per-SM rate of small-N tcgen05.mma compared with one CTA
// (cta_group::1, M=128)? Each "tile" = 4 MMAs of K=16 (one 64-wide k-tile).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench4 tools/mma_bench4.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

__device__ __forceinline__ uint32_t cluster_rank() { return cluster_ctarank(); }
__device__ __forceinline__ void mma2_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2_mc(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"(mask)
               : "memory");
}

template <int N, int PAIR, int COMMIT_EVERY = 0>
__global__ void __cluster_dims__(2, 1, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + 4 * 16384, bar = sb + 16384 + 64;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < (4 * 16384 + 16384) / 16; i += blockDim.x) sts128_zero(base + 16 * i);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc_dyn(smem_u32(&tslot), 512);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (threadIdx.x == 0 && (!PAIR || rank == 0)) {
    const uint32_t idesc = idesc_f16_f32(PAIR ? 256 : 128, N, 0);
    for (int it = 0; it < iters; ++it) {
      const uint32_t a0 = sa + (it & 3) * 16384;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t bd = smem_desc(sb + s * 256, 128, 1024, 0);
        const uint64_t ad = smem_desc(a0 + s * 256, 128, 1024, 0);
        if (PAIR)
          mma2_f16_ss(tmem, ad, bd, idesc, it > 0 ? 1u : 0u);
        else
          mma_f16_ss(tmem, ad, bd, idesc, it > 0 ? 1u : 0u);
      }
      if (COMMIT_EVERY && (it % COMMIT_EVERY) == COMMIT_EVERY - 1) {
        if (PAIR)
          commit2_mc(bar + 8, 3);
        else
          mma_commit(bar + 8);
      }
    }
    if (PAIR)
      commit2_mc(bar, 3);
    else
      mma_commit(bar);
  }
  if (threadIdx.x == 0) mbar_wait(bar, 0);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    else
      tmem_dealloc(tmem, 512);
  }
}

template <int N, int PAIR, int COMMIT_EVERY = 0>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 5 * 16384 + 2048;
  cudaFuncSetAttribute(bench<N, PAIR, COMMIT_EVERY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  bench<N, PAIR, COMMIT_EVERY><<<148, 128, smem>>>(iters, d);
  bench<N, PAIR, COMMIT_EVERY><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s N=%3d commit every %d tiles: %6.1f cycles per instruction; %6.1f cycles per 128x64 tile per SM [%s]\n",
         PAIR ? "cta_group::2 M=256" : "cta_group::1 M=128", N, COMMIT_EVERY, mx / iters / 4, mx / iters / (PAIR ? 2 : 1),
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, 1>();
  run<16, 1, 1>();
  run<16, 1, 2>();
  run<16, 1, 4>();
  run<16, 0>();
  run<16, 0, 1>();
  run<64, 1, 1>();
  return 0;
}
