// Microbenchmark (debug tool, not product): per-tile cost of the MMA shapes the
// SpMM can use for one 128x64 fp16 A tile:
//   SS  M=128 / M=64, N in {16,32,64}   (A and B from shared memory)
//   TS  M=128, A from TMEM              (A written to TMEM beforehand)
//   tcgen05.cp 128x256b smem->TMEM      (4 per tile)
//   tcgen05.st 32x32b.x32 regs->TMEM    (one 128x64 tile = 4 warps x 32 columns)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_bench2 tools/mma_bench2.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE: 0 SS M=128, 1 SS M=64, 2 TS M=128 (A in TMEM), 3 tcgen05.cp only, 4 tcgen05.st only (4 warps)
template <int MODE, int N>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t sa = base, sb = base + 4 * 16384, bar = sb + 16384 + 64;
  __shared__ uint32_t tslot;
  __shared__ uint32_t st_flag_done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) st_flag_done = 0;
  for (int i = threadIdx.x; i < (4 * 16384 + 16384) / 16; i += blockDim.x) sts128_zero(base + 16 * i);
  if (MODE == 9) {  // random fp16 data (|v| in [0.25, 8)), 80 % zeros in A like a sparse tile
    __syncthreads();
    for (int i = threadIdx.x; i < (4 * 16384 + 16384) / 2; i += blockDim.x) {
      uint32_t h = (i + 1) * 2654435761u;
      h ^= h >> 13;
      h *= 0x5bd1e995u;
      h ^= h >> 15;
      const bool zero = i < 4 * 16384 / 2 && (h % 10) < 8;
      const uint16_t v = zero ? 0 : static_cast<uint16_t>(((h >> 8) & 0x83FF) | ((13 + (h >> 20) % 5) << 10));
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(base + 2 * i), "h"(v));
    }
    fence_proxy_async_smem();
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, MODE == 5 ? 2 : (MODE == 6 ? 4 : 1));
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_dyn(smem_u32(&tslot), 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;  // D at cols [0, N); A tiles at cols 256.. (32 cols each)
  const uint32_t b_row = N * 2;
  const uint32_t b_layout = b_row == 32 ? 6u : (b_row == 64 ? 4u : 2u);
  const uint32_t b_sbo = 8u * b_row;
  long long t0 = clock64();
  if (MODE == 4) {
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = j;
    for (int it = 0; it < iters; ++it) {
      tmem_st32(tmem + ((warp * 32u) << 16) + 256 + (it & 7) * 32, r);
    }
    tmem_st_wait();
  } else if (MODE == 5 || MODE == 6) {
    // several issuing threads (one per warp), separate accumulators
    const int issuers = MODE == 5 ? 2 : 4;
    if (warp < issuers && (threadIdx.x & 31) == 0) {
      const uint32_t idesc = idesc_f16_f32(128, N, 1);
      const uint32_t d = tmem + warp * 64;
      for (int it = 0; it < iters / issuers; ++it) {
        const uint32_t a0 = sa + (it & 3) * 16384;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t bd = smem_desc(sb + s * 16 * b_row, 8192, b_sbo, b_layout);
          const uint64_t ad = smem_desc(a0 + s * 256, 128, 1024, 0);
          mma_f16_ss(d, ad, bd, idesc, (it | s) ? 1u : 0u);
        }
      }
      mma_commit(bar);
    }
    if (threadIdx.x == 0) {
      for (int i = 0; i < 1; ++i) mbar_wait(bar, 0);
    }
    __syncthreads();
  } else if (MODE == 7 || MODE == 8) {
    // MMA issue (7: SS, 8: TS) while warps 1-3 stream STS.128 into a separate
    // region (the decode warps' memset/scatter traffic)
    if (threadIdx.x == 0) {
      const uint32_t idesc = idesc_f16_f32(128, N, 1);
      for (int it = 0; it < iters; ++it) {
        const uint32_t a0 = sa + (it & 1) * 16384;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t bd = smem_desc(sb + s * 16 * b_row, 8192, b_sbo, b_layout);
          if (MODE == 7)
            mma_f16_ss(tmem, smem_desc(a0 + s * 256, 128, 1024, 0), bd, idesc, (it | s) ? 1u : 0u);
          else
            mma_f16_ts(tmem, tmem + 256 + (it & 3) * 32 + s * 8, bd, idesc, (it | s) ? 1u : 0u);
        }
      }
      mma_commit(bar);
      mbar_wait(bar, 0);
      st_flag_done = 1;
    } else if (warp >= 1) {
      const uint32_t zone = sa + 2 * 16384;  // tiles 2,3: not read by the MMA
      volatile uint32_t* done = &st_flag_done;
      uint32_t i = threadIdx.x - 32;
      while (!*done) {
#pragma unroll 8
        for (int r = 0; r < 8; ++r) {
          sts128_zero(zone + ((i * 16) & 32767));
          i += 96;
        }
      }
    }
    __syncthreads();
  } else if (MODE == 10 || MODE == 11) {
    // production-like issue loop: last warp of a 640-thread CTA, whole warp walks,
    // elect_one issues; MODE 11 also commits + polls an smem flag per tile pair
    if (warp == (int)(blockDim.x / 32) - 1) {
      const uint32_t idesc = idesc_f16_f32(128, N, 1);
      const uint64_t a_desc0 = smem_desc(sa, 128, 1024, 0);
      const uint64_t b_desc0 = smem_desc(sb, 8192, b_sbo, b_layout);
      for (int it = 0; it < iters; ++it) {
        const uint64_t ad = a_desc0 + (((it & 3) * 16384) >> 4);
        if (MODE == 11 && (it & 1) == 0) {
          uint32_t v;
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&st_flag_done)) : "memory");
          if (v == 12345) __trap();
          tc_fence_after();
        }
        if (elect_one()) {
#pragma unroll
          for (int s = 0; s < 4; ++s)
            mma_f16_ss(tmem + 16, ad + (s * 256 >> 4), b_desc0 + (s * 16 * b_row >> 4), idesc, (it | s) ? 1u : 0u);
          if (MODE == 11 && (it & 1)) mma_commit(bar + 8);
        }
        __syncwarp();
      }
      if (elect_one()) {
        mma_commit(bar);
      }
      __syncwarp();
      mbar_wait(bar, 0);
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    constexpr uint32_t M = MODE == 1 ? 64 : 128;  // MODE 9 behaves like MODE 0 on random data
    const uint32_t idesc = idesc_f16_f32(M, N, 1);
    for (int it = 0; it < iters; ++it) {
      const uint32_t a0 = sa + (it & 3) * 16384;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t bd = smem_desc(sb + s * 16 * b_row, 8192, b_sbo, b_layout);
        if (MODE == 0 || MODE == 1 || MODE == 9) {
          const uint64_t ad = smem_desc(a0 + s * 256, 128, 1024, 0);
          mma_f16_ss(tmem, ad, bd, idesc, (it | s) ? 1u : 0u);
        } else if (MODE == 2) {
          mma_f16_ts(tmem, tmem + 256 + (it & 3) * 32 + s * 8, bd, idesc, (it | s) ? 1u : 0u);
        } else {
          const uint64_t ad = smem_desc(a0 + s * 256, 128, 1024, 0);
          tmem_cp_128x256b(tmem + 256 + (it & 3) * 32 + s * 8, ad);
        }
      }
    }
    mma_commit(bar);
    mbar_wait(bar, 0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int MODE, int N>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 5 * 16384 + 2048;
  cudaFuncSetAttribute(bench<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  const int threads = MODE >= 10 && MODE <= 11 ? 640 : 128;
  bench<MODE, N><<<148, threads, smem>>>(iters, d);
  bench<MODE, N><<<148, threads, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%-34s N=%3d: %7.1f cycles per 128x64 tile  [%s]\n", name, N, double(h[0]) / iters, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 16>("SS M=128");
  run<0, 32>("SS M=128");
  run<0, 64>("SS M=128");
  run<1, 32>("SS M=64 (half tile)");
  run<2, 16>("TS M=128 (A in TMEM)");
  run<2, 32>("TS M=128 (A in TMEM)");
  run<2, 64>("TS M=128 (A in TMEM)");
  run<3, 32>("tcgen05.cp 4x128x256b");
  run<4, 32>("tcgen05.st x32 per warp (4 warps)");
  run<5, 32>("SS M=128, 2 issuing warps");
  run<6, 32>("SS M=128, 4 issuing warps");
  run<5, 16>("SS M=128, 2 issuing warps");
  run<10, 16>("640 thr, warp 19, elect");
  run<11, 16>("640 thr, warp 19, +flag+commit");
  run<9, 16>("SS random data");
  run<9, 64>("SS random data");
  run<7, 16>("SS + 3 warps STS.128 stream");
  run<8, 16>("TS + 3 warps STS.128 stream");
  return 0;
}
