// Microbenchmark (debug tool, not product): shared-memory cost of scattering
// real bank-reordered Tiled-CSL groups into the dense tile (SWIZZLE_NONE
// core-matrix layout), STS.U16 vs STS.32 (word-granular, wrong values on
// purpose), to compare measured wavefronts with the reference's bank model.
// Input: entries of one encoded matrix (uint32) + offsets, passed from Python.
#include <cstdint>
#include <cstdio>

#include "../paper_2309_10285_b200/csrc/sm100_ptx.cuh"

using namespace tcslk;

__device__ __forceinline__ uint32_t a_offset(uint32_t loc) {
  return ((loc << 1) & 0x3C0Eu) | ((loc >> 2) & 0x70u) | ((loc << 4) & 0x380u);
}

template <int MODE>
__global__ void scatter(const uint32_t* ent, const uint32_t* off, int tiles, int reps, unsigned long long* cyc) {
  __shared__ __align__(16) uint8_t tile[16384];
  const uint32_t base = smem_u32(tile);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const uint32_t a0 = off[t], a1 = off[t + 1];
      for (uint32_t g = a0 + 32 * warp; g < a1; g += 32 * (blockDim.x / 32)) {
        const uint32_t e = __ldg(ent + g + lane);
        if (MODE == 0) sts16(base + a_offset(e), e >> 16);
        if (MODE == 1) asm volatile("st.shared.u32 [%0], %1;" ::"r"(base + (a_offset(e) & ~3u)), "r"(e) : "memory");
        if (MODE == 2) sts16(base + ((e & 0x1FFF) << 1), e >> 16);  // plain row-major (bank-unaware)
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  uint32_t tiles, ne;
  fread(&tiles, 4, 1, f);
  fread(&ne, 4, 1, f);
  uint32_t* hoff = new uint32_t[tiles + 1];
  uint32_t* hent = new uint32_t[ne];
  fread(hoff, 4, tiles + 1, f);
  fread(hent, 4, ne, f);
  fclose(f);
  uint32_t *doff, *dent;
  unsigned long long* dc;
  cudaMalloc(&doff, 4 * (tiles + 1));
  cudaMalloc(&dent, 4ull * ne);
  cudaMalloc(&dc, 8 * 148);
  cudaMemcpy(doff, hoff, 4 * (tiles + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(dent, hent, 4ull * ne, cudaMemcpyHostToDevice);
  const char* names[3] = {"STS.U16 core-matrix", "STS.32 word", "STS.U16 row-major"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int it = 0; it < 2; ++it) {
      if (mode == 0) scatter<0><<<148, 128>>>(dent, doff, tiles, 4, dc);
      if (mode == 1) scatter<1><<<148, 128>>>(dent, doff, tiles, 4, dc);
      if (mode == 2) scatter<2><<<148, 128>>>(dent, doff, tiles, 4, dc);
    }
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, dc, sizeof h, cudaMemcpyDeviceToHost);
    const double groups = double(ne) / 32 * 4 / 148;
    printf("%-22s %.1f cycles per group per SM (%s)\n", names[mode], double(h[0]) / groups,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
