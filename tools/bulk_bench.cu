// Microbenchmark (debug tool, not product): HBM streaming rate of one
// producer thread per SM issuing cp.async.bulk global->smem copies of CH bytes
// into a ring of DEPTH slots (the SpMM's entry-ring pattern), vs. a plain
// vectorised LDG stream by 512 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bulk_bench tools/bulk_bench.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

template <int CH, int DEPTH>
__global__ void __launch_bounds__(64, 1) bulk_stream(const uint8_t* src, size_t bytes_per_cta, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t ring = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t bars = ring + CH * DEPTH;
  const uint8_t* base = src + blockIdx.x * bytes_per_cta;
  const uint32_t nchunks = static_cast<uint32_t>(bytes_per_cta / CH);
  if (threadIdx.x == 0) {
    for (int i = 0; i < DEPTH; ++i) mbar_init(bars + 8 * i, 1);
    fence_barrier_init();
  }
  __syncthreads();
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    // prologue
    for (uint32_t c = 0; c < DEPTH && c < nchunks; ++c) {
      mbar_arrive_expect_tx(bars + 8 * c, CH);
      bulk_g2s(ring + c * CH, base + static_cast<size_t>(c) * CH, CH, bars + 8 * c, pol);
    }
    for (uint32_t c = 0; c < nchunks; ++c) {
      const uint32_t s = c % DEPTH;
      mbar_wait(bars + 8 * s, (c / DEPTH) & 1);
      acc += lds32(ring + s * CH);
      const uint32_t nc = c + DEPTH;
      if (nc < nchunks) {
        mbar_arrive_expect_tx(bars + 8 * s, CH);
        bulk_g2s(ring + s * CH, base + static_cast<size_t>(nc) * CH, CH, bars + 8 * s, pol);
      }
    }
    sink[blockIdx.x] = acc;
  }
}

__global__ void __launch_bounds__(512, 1) ldg_stream_k(const uint4* src, size_t vec_per_cta, unsigned long long* sink) {
  const uint4* base = src + blockIdx.x * vec_per_cta;
  unsigned int acc = 0;
#pragma unroll 8
  for (size_t i = threadIdx.x; i < vec_per_cta; i += blockDim.x) {
    const uint4 v = __ldg(base + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

template <int CH, int DEPTH>
void run_bulk(const uint8_t* d, size_t total, unsigned long long* sink) {
  const int grid = 148;
  const size_t per = (total / grid) / CH * CH;
  const int smem = CH * DEPTH + 1024 + 8 * DEPTH;
  cudaFuncSetAttribute(bulk_stream<CH, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  bulk_stream<CH, DEPTH><<<grid, 64, smem>>>(d, per, sink);
  cudaEventRecord(a);
  bulk_stream<CH, DEPTH><<<grid, 64, smem>>>(d, per, sink);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("bulk CH=%6d DEPTH=%2d (in flight %6d B/SM): %7.1f GB/s [%s]\n", CH, DEPTH, CH * DEPTH,
         per * grid / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
}

int main() {
  const size_t total = size_t(2) << 30;
  uint8_t* d;
  cudaMalloc(&d, total);
  cudaMemset(d, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 148 * 8);
  run_bulk<4096, 4>(d, total, sink);
  run_bulk<4096, 8>(d, total, sink);
  run_bulk<4096, 16>(d, total, sink);
  run_bulk<4096, 32>(d, total, sink);
  run_bulk<8192, 8>(d, total, sink);
  run_bulk<8192, 16>(d, total, sink);
  run_bulk<16384, 4>(d, total, sink);
  run_bulk<16384, 8>(d, total, sink);
  run_bulk<2048, 32>(d, total, sink);
  run_bulk<2048, 64>(d, total, sink);
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t per = total / 148 / 16;
    ldg_stream_k<<<148, 512>>>(reinterpret_cast<const uint4*>(d), per, sink);
    cudaEventRecord(a);
    ldg_stream_k<<<148, 512>>>(reinterpret_cast<const uint4*>(d), per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128 stream, 512 thr/SM: %7.1f GB/s\n", per * 16 * 148 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
