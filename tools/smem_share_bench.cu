// Microbenchmark (debug tool, not product): do tcgen05.mma shared-memory
// operand reads compete with LSU shared-memory traffic? Per SM:
//   mode 0: MMA only        (one thread issues cta_group::1 M=128 N=16 K=16 SS MMAs)
//   mode 1: STS.U16 only    (8 warps scatter 16-bit stores, 1 wavefront per instruction)
//   mode 2: both concurrently, each timed on its own
// Reports MMA bytes of A read per cycle and LSU wavefronts per cycle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/smem_share_bench tools/smem_share_bench.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

template <int MODE>
__global__ void bench(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + 4 * 16384, sc = sb + 16384, bar = sc + 32768;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (4 * 16384 + 16384 + 32768) / 16; i += blockDim.x) sts128_zero(base + 16 * i);
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
  __syncthreads();
  if (warp == 0) {
    if (MODE != 1 && lane == 0) {
      const uint32_t idesc = idesc_f16_f32(128, 16, 1);
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        const uint32_t a0 = sa + (it & 3) * 16384;
#pragma unroll
        for (int s = 0; s < 4; ++s)
          mma_f16_ss(tmem, smem_desc(a0 + s * 256, 128, 1024, 0), smem_desc(sb + s * 16 * 32, 8192, 256, 6), idesc,
                     it > 0 ? 1u : 0u);
      }
      mma_commit(bar);
      mbar_wait(bar, 0);
      out[blockIdx.x * 2] = clock64() - t0;
    }
  } else if (warp <= 8) {
    if (MODE != 0) {
      // scatter: lane l stores to bank l (one wavefront per instruction), 16 KB region
      const long long t0 = clock64();
      uint32_t off = (warp * 997u) & 0x3F80u;
      for (int it = 0; it < iters * 8; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) sts16(sc + ((off + 4 * lane + 128 * j) & 0x7FFEu), it);
        off += 1024;
      }
      __syncwarp();
      if (lane == 0 && warp == 1) out[blockIdx.x * 2 + 1] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * 2 * 8);
  cudaMemset(d, 0, 148 * 2 * 8);
  const int smem = 4 * 16384 + 16384 + 32768 + 2048;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2048;
  bench<MODE><<<148, 288, smem>>>(iters, d);
  bench<MODE><<<148, 288, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double mma_cyc = h[0] ? double(h[0]) : 0, st_cyc = h[1] ? double(h[1]) : 0;
  printf("%-22s MMA: %7.1f cyc/tile (%5.1f B/cyc of A)   STS (8 warps): %6.3f wavefronts/cyc  [%s]\n", name,
         mma_cyc / iters, mma_cyc ? 16384.0 * iters / mma_cyc : 0.0,
         st_cyc ? 8.0 * iters * 8 * 8 / st_cyc : 0.0, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("MMA only");
  run<1>("STS only");
  run<2>("MMA + STS");
  return 0;
}
