// Microbenchmark (debug tool, not product): tcgen05.mma kind::f16 throughput
// with A read from shared memory in SWIZZLE_NONE vs SWIZZLE_128B K-major
// layouts, for the SpMM tile shape (M=128, K=64 per tile, small N).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

template <int N, int LAYOUT_A, int MODE = 0>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sa = base;                 // 4 x 16 KB A tiles
  const uint32_t sb = base + 4 * 16384;     // B tile
  const uint32_t bar = sb + 8192 + 64;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (4 * 16384 + 8192) / 16; i += blockDim.x) sts128_zero(base + 16 * i);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 8, 1);
    mbar_init(bar + 16, 1);
    mbar_arrive(bar + 16);  // phase 0 of bar+16 completes: a barrier that is always ready
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_dyn(smem_u32(&tslot), 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(128, N, 1);
    const uint32_t b_row = N * 2 < 16 ? 16 : N * 2;
    const uint32_t b_layout = b_row == 16 ? 0u : (b_row == 32 ? 6u : (b_row == 64 ? 4u : 2u));
    const uint32_t b_lbo = b_row == 16 ? 128u : 8192u, b_sbo = b_row == 16 ? 128u : 8u * b_row;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t a0 = sa + (it & 3) * 16384;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        uint64_t ad;
        if (LAYOUT_A == 0)
          ad = smem_desc(a0 + s * 256, 128, 1024, 0);  // SWIZZLE_NONE, core matrices K-fastest
        else
          ad = smem_desc(a0 + s * 32, 16, 1024, 2);    // SWIZZLE_128B K-major, rows of 128 B
        const uint64_t bd = smem_desc(sb + s * 16 * b_row, b_lbo, b_sbo, b_layout);
        mma_f16_ss(tmem, ad, bd, idesc, (it | s) ? 1u : 0u);
      }
      if (MODE >= 1) mma_commit(bar + 8);
      if (MODE >= 2) mma_commit(bar + 8);
      if (MODE >= 3) tc_fence_after();
      if (MODE >= 4) {
        mbar_wait(bar + 16, 0);
        mbar_wait(bar + 16, 0);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

template <int N, int L, int MODE = 0>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 4 * 16384 + 8192 + 2048;
  cudaFuncSetAttribute(bench<N, L, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  bench<N, L, MODE><<<148, 128, smem>>>(iters, d);
  bench<N, L, MODE><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%-28s mode %d N=%3d: %7.1f cycles per 128x64 tile (4 MMAs)  [%s]\n", name, MODE, N, double(h[0]) / iters,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<8, 0>("A SWIZZLE_NONE");
  run<16, 0>("A SWIZZLE_NONE");
  run<32, 0>("A SWIZZLE_NONE");
  run<64, 0>("A SWIZZLE_NONE");
  run<16, 2>("A SWIZZLE_128B");
  run<64, 2>("A SWIZZLE_128B");
  run<8, 2>("A SWIZZLE_128B");
  run<16, 0, 1>("+commit");
  run<16, 0, 2>("+2 commits");
  run<16, 0, 3>("+fence after");
  run<16, 0, 4>("+2 ready try_waits");
  return 0;
}
