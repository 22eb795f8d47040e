// Microbenchmark (debug tool, not product): is the ~45-cycle cost of one
// tcgen05.mma (M=128, K=16, small N) a per-instruction throughput limit or the
// read-modify-write dependency on one TMEM accumulator? One thread issues
// kind::f16 SS MMAs round-robin over NACC independent accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench3 tools/mma_bench3.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

// BK: 0 = B MN-major (as the SpMM), 1 = B K-major SWIZZLE_NONE, 2 = A and B K-major SWIZZLE_128B
template <int N, int NACC, int M, int BK>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + 4 * 16384, bar = sb + 16384 + 64;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (4 * 16384 + 16384) / 16; i += blockDim.x) sts128_zero(base + 16 * i);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_dyn(smem_u32(&tslot), 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b_row = N * 2;
  const uint32_t b_layout = b_row == 16 ? 0u : (b_row == 32 ? 6u : (b_row == 64 ? 4u : 2u));
  const uint32_t b_sbo = b_row == 16 ? 128u : 8u * b_row;
  const uint32_t b_lbo = b_row == 16 ? 128u : 8192u;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16_f32(M, N, BK == 0 ? 1 : 0);
    for (int it = 0; it < iters; ++it) {
      const uint32_t a0 = sa + (it & 3) * 16384;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        uint64_t bd, ad;
        if (BK == 0) {
          bd = smem_desc(sb + s * 16 * b_row, b_lbo, b_sbo, b_layout);
          ad = smem_desc(a0 + s * 256, 128, 1024, 0);
        } else if (BK == 1) {  // core matrices 8 (n) x 16 B (k): LBO = k step, SBO = n step
          bd = smem_desc(sb + s * 256, 128, 1024, 0);
          ad = smem_desc(a0 + s * 256, 128, 1024, 0);
        } else {  // rows of 128 B (64 k), 8-row atoms of 1 KB, k-step = +32 B
          bd = smem_desc(sb + s * 32, 16, 1024, 2);
          ad = smem_desc(a0 + s * 32, 16, 1024, 2);
        }
        const int acc = (it * 4 + s) % NACC;
        mma_f16_ss(tmem + acc * N, ad, bd, idesc, it > 0 ? 1u : 0u);
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, int NACC, int M = 128, int BK = 0>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 5 * 16384 + 2048;
  cudaFuncSetAttribute(bench<N, NACC, M, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  bench<N, NACC, M, BK><<<148, 128, smem>>>(iters, d);
  bench<N, NACC, M, BK><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("BK=%d M=%3d N=%3d accumulators=%d: %6.1f cycles/MMA (%6.1f per 128x64 tile, max CTA) [%s]\n", BK, M, N, NACC,
         mx / iters / 4, mx / iters, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, 1>();
  run<64, 1>();
  run<16, 1, 128, 1>();
  run<64, 1, 128, 1>();
  run<16, 1, 128, 2>();
  run<64, 1, 128, 2>();
  run<16, 2, 128, 2>();
  run<8, 1, 128, 1>();
  return 0;
}
