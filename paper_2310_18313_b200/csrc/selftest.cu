// selftest.cu — on-device verification that the branch-free sqrt / division fast
// paths of device.cuh return exactly what __fsqrt_rn / __fdiv_rn return wherever
// their range predicate accepts the input (diagnostic entry fp8lm_selftest_fastmath).
#include <cuda_runtime.h>
#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace fp8lm {

// every positive binary32 bit pattern [lo, hi): sqrt fast vs intrinsic
__global__ void k_check_sqrt(uint32_t lo, uint32_t hi, unsigned long long* bad,
                             unsigned long long* accepted) {
  unsigned long long nb = 0, na = 0;
  for (uint64_t b = (uint64_t)lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < hi;
       b += (uint64_t)gridDim.x * blockDim.x) {
    const float x = __uint_as_float((uint32_t)b);
    const bool ok = sqrt_chk(x) >= kSqrtChkMin && x < 1.2676506e30f;
    const float f = sqrt_rn_core(x);
    if (ok) {
      ++na;
      const float r = __fsqrt_rn(x);
      nb += (__float_as_uint(f) != __float_as_uint(r));
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(accepted, na);
}

__device__ __forceinline__ uint32_t mix(uint64_t x) {   // splitmix64 -> 32 bits
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)((x ^ (x >> 31)) >> 16);
}

// `pairs` pseudo-random (a, b): a any sign, exponents spanning the predicate's
// range and beyond, b > 0; every 64th pair uses a mantissa-boundary pattern
__global__ void k_check_div(uint64_t pairs, uint64_t seed, unsigned long long* bad,
                            unsigned long long* accepted) {
  unsigned long long nb = 0, na = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < pairs;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t ra = mix(seed ^ (2 * i)), rb = mix(seed ^ (2 * i + 1));
    uint32_t ea = 40u + (ra >> 24) % 176u, eb = 50u + (rb >> 24) % 156u;   // wide exponent spread
    uint32_t ma = ra & 0x7FFFFFu, mb = rb & 0x7FFFFFu;
    if ((i & 63u) == 0) { ma = (i & 64u) ? 0x7FFFFFu : 0u; mb = (i & 128u) ? 0x7FFFFFu : 1u; }
    const float a = __uint_as_float(((ra & 1u) << 31) | (ea << 23) | ma);
    const float b = __uint_as_float((eb << 23) | mb);
    const bool ok = div_chk(a) >= kDivChkMin && fabsf(a) < 2.3058430e18f &&
                    b >= 8.6736174e-19f && b < 2.3058430e18f;          // 2^-60 .. 2^61
    const float f = div_rn_core(a, b);
    if (ok) {
      ++na;
      const float r = __fdiv_rn(a, b);
      nb += (__float_as_uint(f) != __float_as_uint(r));
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(accepted, na);
}

}  // namespace fp8lm

using namespace fp8lm;

extern "C" int fp8lm_selftest_fastmath(uint64_t div_pairs, uint64_t seed, uint64_t* out4) {
  if (!out4) return FP8LM_EINVAL;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 4 * sizeof(unsigned long long)) != cudaSuccess) return FP8LM_ECUDA;
  cudaMemset(d, 0, 4 * sizeof(unsigned long long));
  const int grid = num_sms() * 8;
  k_check_sqrt<<<grid, 256>>>(0u, 0x80000000u, d, d + 1);   // every x >= +0, incl. inf/NaN
  k_check_div<<<grid, 256>>>(div_pairs, seed, d + 2, d + 3);
  unsigned long long h[4] = {0, 0, 0, 0};
  cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return FP8LM_ECUDA;
  for (int i = 0; i < 4; ++i) out4[i] = h[i];
  return FP8LM_OK;
}
