// Auxiliary kernels of the hot path:
//   decode            <- tcsl::decode       proj/src/tcsl_format.cpp:126-155
//   validate          <- check_offsets      proj/src/tcsl_format.cpp:19-32
//   dense_gemm_exact  <- dense_gemm_ref     proj/src/gemm.cpp:7-44 (bit-exact order)
//   splitk_reduce     <- upstream split-K Reduction_Workspace
//   rebase            <- row-shard slicing
//   gen_synthetic     <- bench inputs with gen_random_sparse's value law (matrix.cpp:56-63)
#include <cuda_fp16.h>

#include <cstdlib>

#include "sm100_ptx.cuh"
#include "tcsl_internal.cuh"

namespace tcslk {

namespace {

// One block per tile; `strict` is a TCSL_CHECK_* mode. DECODE: decode's rules (tcsl_format.cpp:126-155 after
// check_offsets :19-32): whole 32-entry groups, first offset 0, last == E, and a
// nonzero value in the padded fringe is location_out_of_range. INGEST:
// deserialize_tcsl's rules (check_offsets only; entry problems become flags). SPMM:
// extract_tile's rules as spmm uses them (engine.cpp:8-25): only the tile's own
// span is checked and fringe entries are dropped. A location repeated inside a
// tile is detected with a bitmap (tile_elems <= 65536 bits = 8 KB of smem); such
// a tile is rewritten serially in entry order so the last entry wins, as in the
// reference's sequential loops. out == nullptr: validation only.
__global__ void decode_kernel(const uint32_t* __restrict__ off, const uint32_t* __restrict__ ent,
                              uint64_t n_entries, uint32_t m, uint32_t k, int m_tb, int k_tb, int tiles_k,
                              uint32_t tiles, uint16_t* __restrict__ out, int* err, int strict,
                              uint32_t* flags) {
  extern __shared__ uint32_t seen[];
  const uint32_t tile = blockIdx.x;
  const uint32_t a = off[tile], b = off[tile + 1];
  if (threadIdx.x == 0 && strict) {
    if (tile == 0 && a != 0) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
    if (tile + 1 == tiles && b != n_entries) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
  }
  if (b < a || b > n_entries || (strict && ((b - a) & 31u))) {
    if (threadIdx.x == 0) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
    return;
  }
  if (threadIdx.x == 0 && flags && (((b - a) & 31u) || (a & 31u))) atomicOr(flags, kFlagPartialGroups);
  const long long r0 = static_cast<long long>(tile / tiles_k) * m_tb;
  const long long c0 = static_cast<long long>(tile % tiles_k) * k_tb;
  const uint32_t elems = static_cast<uint32_t>(m_tb) * k_tb;
  for (uint32_t w = threadIdx.x; w < (elems + 31) / 32; w += blockDim.x) seen[w] = 0;
  __syncthreads();
  bool dup = false, fringe = false, range = false;
  for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
    const uint32_t v = ent[e];
    const uint32_t loc = v & 0xFFFFu;
    if (loc >= elems) {
      range = true;
      if (strict != TCSL_CHECK_INGEST) raise_dev(err, TCSL_STATUS_LOCATION_OUT_OF_RANGE);
      continue;
    }
    const uint32_t bit = 1u << (loc & 31u);
    dup |= (atomicOr(&seen[loc >> 5], bit) & bit) != 0;
    const long long r = r0 + loc / k_tb, c = c0 + loc % k_tb;
    uint16_t val = static_cast<uint16_t>(v >> 16);
    if ((val & 0x7FFFu) == 0) val = 0;  // -0 -> +0 (half.hpp:27)
    if (r >= m || c >= k) {
      // decode rejects fringe payloads (tcsl_format.cpp:146-149); spmm's extract_tile
      // (engine.cpp:8-25) lets them through and the crop / zero-padded B removes them.
      if (val) {
        fringe = true;
        if (strict == TCSL_CHECK_DECODE) raise_dev(err, TCSL_STATUS_LOCATION_OUT_OF_RANGE);
      }
      continue;
    }
    if (out) out[r * k + c] = val;
  }
  if (__syncthreads_or(fringe) && flags && threadIdx.x == 0) atomicOr(flags, kFlagFringePayload);
  if (__syncthreads_or(range) && flags && threadIdx.x == 0) atomicOr(flags, TCSL_FLAG_LOCATION_RANGE);
  if (__syncthreads_or(dup) && threadIdx.x == 0) {
    if (flags) atomicOr(flags, kFlagDuplicates);
    for (uint32_t e = a; e < b && out; ++e) {  // sequential replay: the last entry wins
      const uint32_t v = ent[e];
      const uint32_t loc = v & 0xFFFFu;
      if (loc >= elems) continue;
      const long long r = r0 + loc / k_tb, c = c0 + loc % k_tb;
      if (r >= m || c >= k) continue;
      uint16_t val = static_cast<uint16_t>(v >> 16);
      if ((val & 0x7FFFu) == 0) val = 0;
      out[r * k + c] = val;
    }
  }
}

__global__ void validate_kernel(const uint32_t* __restrict__ off, uint64_t n_entries, uint32_t tiles,
                                int* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && off[0] != 0) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
  if (i == 0 && off[tiles] != n_entries) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
  if (i < tiles) {
    const uint32_t a = off[i], b = off[i + 1];
    if (b < a || ((b - a) & 31u)) raise_dev(err, TCSL_STATUS_INCONSISTENT_OFFSETS);
  }
}

// Y = A x X with one binary32 multiply and one binary32 add per k, k ascending
// (gemm.cpp:36-40). __fmul_rn/__fadd_rn are never contracted into FMA.
constexpr int kGT = 16;  // output tile 16 x 16, one output per thread
constexpr int kGK = 32;  // k chunk
__global__ void __launch_bounds__(256) dense_gemm_exact_kernel(const uint16_t* __restrict__ a, uint32_t m,
                                                               uint32_t k, const uint16_t* __restrict__ x,
                                                               int n, float* __restrict__ y) {
  __shared__ float as[kGT][kGK + 1];
  __shared__ float xs[kGK][kGT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long i = static_cast<long long>(blockIdx.y) * kGT + ty;
  const int j = blockIdx.x * kGT + tx;
  float acc = 0.0f;
  for (uint32_t k0 = 0; k0 < k; k0 += kGK) {
    for (int t = threadIdx.x; t < kGT * kGK; t += 256) {
      const int r = t / kGK, c = t % kGK;
      const long long gi = static_cast<long long>(blockIdx.y) * kGT + r;
      const uint32_t gk = k0 + c;
      as[r][c] = (gi < m && gk < k) ? __half2float(__ushort_as_half(a[gi * k + gk])) : 0.0f;
      const int rr = t / kGT, cc = t % kGT;
      const uint32_t gk2 = k0 + rr;
      const int gj = blockIdx.x * kGT + cc;
      xs[rr][cc] = (gk2 < k && gj < n) ? __half2float(__ushort_as_half(x[static_cast<long long>(gk2) * n + gj]))
                                       : 0.0f;
    }
    __syncthreads();
    const int kc = min(kGK, static_cast<int>(k - k0));
    for (int kk = 0; kk < kc; ++kk) acc = __fadd_rn(acc, __fmul_rn(as[ty][kk], xs[kk][tx]));
    __syncthreads();
  }
  if (i < m && j < n) y[i * n + j] = acc;
}

__global__ void splitk_reduce_kernel(const float* __restrict__ p, int split, size_t count,
                                     float* __restrict__ y) {
  griddep_wait();  // launched with programmatic serialization: the partials come from the previous grid
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  if ((count & 3u) == 0) {
    const size_t c4 = count / 4;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < c4; i += stride) {
      float4 acc = reinterpret_cast<const float4*>(p)[i];
      for (int s = 1; s < split; ++s) {
        const float4 v = reinterpret_cast<const float4*>(p + static_cast<size_t>(s) * count)[i];
        acc.x = __fadd_rn(acc.x, v.x);
        acc.y = __fadd_rn(acc.y, v.y);
        acc.z = __fadd_rn(acc.z, v.z);
        acc.w = __fadd_rn(acc.w, v.w);
      }
      reinterpret_cast<float4*>(y)[i] = acc;
    }
  } else {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
      float acc = p[i];
      for (int s = 1; s < split; ++s) acc = __fadd_rn(acc, p[static_cast<size_t>(s) * count + i]);
      y[i] = acc;
    }
  }
}

// Split-K sum in ascending s (as splitk_reduce_kernel) followed by the fused
// epilogue of tcsl_cuda_spmm_ex; split == 1 is a pure epilogue pass.
__global__ void reduce_epilogue_kernel(const float* __restrict__ p, int split, size_t count, int n,
                                       const float* __restrict__ bias, int act, float* __restrict__ y32,
                                       uint16_t* __restrict__ y16, void* const* __restrict__ peers, int n_peers,
                                       int peers_f16) {
  griddep_wait();
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    float acc = p[i];
    for (int s = 1; s < split; ++s) acc = __fadd_rn(acc, p[static_cast<size_t>(s) * count + i]);
    const float v = epilogue_value(acc, bias ? __ldg(bias + i / static_cast<size_t>(n)) : 0.0f, act);
    if (n_peers > 0) {  // rows pushed to every peer's Y (NVLink stores for remote peers)
      const uint32_t h = f16_bits_rne(v);
      for (int g = 0; g < n_peers; ++g) {
        void* base = peers[g];
        if (peers_f16)
          static_cast<uint16_t*>(base)[i] = static_cast<uint16_t>(h);
        else
          static_cast<float*>(base)[i] = v;
      }
    } else if (y16) {
      y16[i] = static_cast<uint16_t>(f16_bits_rne(v));
    } else {
      y32[i] = v;
    }
  }
}

__global__ void rebase_kernel(const uint32_t* __restrict__ off, uint32_t t0, uint32_t n,
                              uint32_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) out[i] = off[t0 + i] - off[t0];
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen_synthetic_kernel(uint16_t* __restrict__ w, uint64_t count, uint64_t thresh,
                                     uint64_t seed) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const uint64_t h = splitmix64(seed ^ (i * 0xD1B54A32D192ED03ull));
    uint16_t v = 0;
    if ((h >> 11) >= thresh) {  // P(zero) = thresh / 2^53 = beta
      const uint64_t r = splitmix64(h);
      const uint16_t man = static_cast<uint16_t>(r & 0x3FFu);
      const uint16_t expf = static_cast<uint16_t>(13 + (r >> 10) % 5);
      const uint16_t sign = static_cast<uint16_t>(((r >> 63) & 1u) << 15);
      v = static_cast<uint16_t>(sign | (expf << 10) | man);
    }
    w[i] = v;
  }
}

// Launch with programmatic stream serialization (the kernel calls griddep_wait first).
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int blocks, int threads, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace

bool pdl_enabled() {
  static const bool on = !(getenv("TCSL_PDL") && atoi(getenv("TCSL_PDL")) == 0);
  return on;
}

cudaError_t launch_decode(const uint32_t* off, const uint32_t* ent, uint64_t n_entries, uint32_t m,
                          uint32_t k, int m_tb, int k_tb, uint16_t* out, int* err, int strict, cudaStream_t s) {
  const int tk = div_up_i(k, k_tb);
  const uint32_t tiles = static_cast<uint32_t>(div_up_i(m, m_tb)) * tk;
  cudaError_t e = cudaMemsetAsync(out, 0, static_cast<size_t>(m) * k * 2, s);
  if (e != cudaSuccess) return e;
  const size_t smem = 4 * ((static_cast<size_t>(m_tb) * k_tb + 31) / 32);
  if (tiles)
    decode_kernel<<<tiles, 256, smem, s>>>(off, ent, n_entries, m, k, m_tb, k_tb, tk, tiles, out, err, strict,
                                           nullptr);
  return cudaGetLastError();
}

cudaError_t launch_validate_entries(const uint32_t* off, const uint32_t* ent, uint64_t n_entries, uint32_t m,
                                    uint32_t k, int m_tb, int k_tb, int strict, uint32_t* flags, int* err,
                                    cudaStream_t s) {
  const int tk = div_up_i(k, k_tb);
  const uint32_t tiles = static_cast<uint32_t>(div_up_i(m, m_tb)) * tk;
  const size_t smem = 4 * ((static_cast<size_t>(m_tb) * k_tb + 31) / 32);
  if (tiles)
    decode_kernel<<<tiles, 256, smem, s>>>(off, ent, n_entries, m, k, m_tb, k_tb, tk, tiles, nullptr, err, strict,
                                           flags);
  return cudaGetLastError();
}

cudaError_t launch_validate(const uint32_t* off, uint64_t n_entries, uint32_t tiles, int* err,
                            cudaStream_t s) {
  validate_kernel<<<(tiles + 256) / 256, 256, 0, s>>>(off, n_entries, tiles, err);
  return cudaGetLastError();
}

cudaError_t launch_dense_gemm_exact(const uint16_t* a, uint32_t m, uint32_t k, const uint16_t* x, int n,
                                    float* y, cudaStream_t s) {
  dim3 grid((n + kGT - 1) / kGT, (m + kGT - 1) / kGT);
  dense_gemm_exact_kernel<<<grid, 256, 0, s>>>(a, m, k, x, n, y);
  return cudaGetLastError();
}

cudaError_t launch_splitk_reduce(const float* p, int split, size_t count, float* y, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  const size_t work = (count & 3u) == 0 ? count / 4 : count;
  const int blocks = static_cast<int>(std::min<size_t>((work + 255) / 256, 148 * 8));
  return launch_pdl(splitk_reduce_kernel, blocks, 256, s, p, split, count, y);
}

cudaError_t launch_reduce_epilogue(const float* p, int split, uint32_t m, int n, const float* bias, int act,
                                   float* y32, uint16_t* y16, cudaStream_t s, void* const* peers, int n_peers,
                                   bool peers_f16) {
  const size_t count = static_cast<size_t>(m) * n;
  if (count == 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 8));
  return launch_pdl(reduce_epilogue_kernel, blocks, 256, s, p, split, count, n, bias, act, y32, y16, peers,
                    n_peers, peers_f16 ? 1 : 0);
}

cudaError_t launch_rebase(const uint32_t* off, uint32_t t0, uint32_t t1, uint32_t* out, cudaStream_t s) {
  const uint32_t n = t1 - t0;
  rebase_kernel<<<(n + 256) / 256, 256, 0, s>>>(off, t0, n, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_synthetic(uint16_t* w, uint64_t count, double beta, uint64_t seed, cudaStream_t s) {
  double t = beta * 9007199254740992.0;  // 2^53
  if (t < 0) t = 0;
  if (t > 9007199254740992.0) t = 9007199254740992.0;
  const uint64_t thresh = static_cast<uint64_t>(t);
  const int blocks = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 148ull * 16));
  if (count) gen_synthetic_kernel<<<blocks, 256, 0, s>>>(w, count, thresh, seed);
  return cudaGetLastError();
}

}  // namespace tcslk
