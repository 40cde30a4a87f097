// strategies.cu — the FP8 all-reduce strategies of PAPER.md §2.1 (pre-scaling Eq. 1,
// post-scaling Eq. 2, automatic scaling Eq. 3-6) over N ranks' gradients held on one
// device, with the Fig. 6 statistics (SNR, underflow rate, overflow rate).
// SURVEY §8(f) row f3; readings R28-R30; ABI: fp8lm_allreduce_strategy.
//
// Two streaming kernels over the N x n gradient block (HBM-bound: every value is read
// twice, 8 B per rank-element):
//   k_strat_amax    A = max |g| over ranks and elements (Eq. 4's MIN of the ranks' JIT
//                   scales is the scale of the largest amax, RN being monotone); its last
//                   CTA sets the shared scale s, the result scale and zeroes the sums
//   k_strat_reduce  per element: the N rank encodes in rank order (pre: fl(fl(g s)/N)),
//                   the binary32 rank-order sum, the encode of the sum, the dequantized
//                   result against the binary64 mean; event counts and the two error
//                   sums flush once per warp; the last CTA runs the mu update (AUTO)
#include <cuda_runtime.h>
#include <cstdint>

#include "device.cuh"
#include "internal.h"

namespace fp8lm {

namespace {

constexpr int kST = 256;        // threads per CTA
constexpr float kMuGrowth = 1.00069344043731689453125f;   // 0x3F8016B9 = fl(2^(1/1000)) (R2)

enum { SCR_AMAX = 0, SCR_NONFINITE = 1, SCR_TICKET_A = 2, SCR_TICKET_R = 3 };

__device__ __forceinline__ bool last_cta(uint32_t* ticket) {
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(ticket, 1u);
    last = t == gridDim.x - 1;
    if (last) *ticket = 0;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t range_first(int64_t n) { return n * blockIdx.x / gridDim.x; }
__device__ __forceinline__ int64_t range_end(int64_t n) { return n * (blockIdx.x + 1) / gridDim.x; }

// ------------------------------------------------------------------ A and the scales
template <bool VEC>
__global__ void __launch_bounds__(kST) k_strat_amax(const float* __restrict__ g, int64_t total,
                                                    fp8lm_commstats* st, const float* mu, int strategy,
                                                    int N) {
  uint32_t m = 0, bad = 0;
  if (VEC) {
    const int64_t nv = total / 4;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const int64_t b = range_first(nv), e = range_end(nv);
    for (int64_t i = b + threadIdx.x; i < e; i += kST) {
      const float4 x = __ldg(g4 + i);
      const uint32_t a0 = abs_bits(x.x), a1 = abs_bits(x.y), a2 = abs_bits(x.z), a3 = abs_bits(x.w);
      m = max(m, max(max(a0, a1), max(a2, a3)));
      bad |= (a0 >= 0x7F800000u) | (a1 >= 0x7F800000u) | (a2 >= 0x7F800000u) | (a3 >= 0x7F800000u);
    }
    if (blockIdx.x == gridDim.x - 1)
      for (int64_t i = nv * 4 + threadIdx.x; i < total; i += kST) {
        const uint32_t a = abs_bits(__ldg(g + i));
        m = max(m, a);
        bad |= a >= 0x7F800000u;
      }
  } else {
    const int64_t b = range_first(total), e = range_end(total);
    for (int64_t i = b + threadIdx.x; i < e; i += kST) {
      const uint32_t a = abs_bits(__ldg(g + i));
      m = max(m, a);
      bad |= a >= 0x7F800000u;
    }
  }
  m = warp_max(m);
  bad = __any_sync(0xffffffffu, bad) ? 1u : 0u;
  if ((threadIdx.x & 31) == 0) {
    if (m) atomicMax(&st->scratch[SCR_AMAX], m);
    if (bad) atomicOr(&st->scratch[SCR_NONFINITE], 1u);
  }
  if (!last_cta(&st->scratch[SCR_TICKET_A])) return;
  if (threadIdx.x != 0) return;
  // Eq. 4 through the pipeline's scale rules (R7, R14): s = fl(fl(448 / A) mu)
  const uint32_t ab = st->scratch[SCR_AMAX];
  const uint32_t nf = st->scratch[SCR_NONFINITE];
  const float A = __uint_as_float(ab);
  const float mu_used = strategy == FP8LM_STRATEGY_AUTO ? *mu : 1.0f;
  float s;
  if (nf) {
    s = 0.0f;
  } else if (ab == 0) {
    s = 1.0f;
  } else {
    const float r = __fdiv_rn(448.0f, A);
    s = isinf(r) ? 1.0f : __fmul_rn(r, mu_used);
    if (isinf(s)) s = 1.0f;
  }
  const float scale = strategy == FP8LM_STRATEGY_PRE ? s : __fmul_rn((float)N, s);
  st->amax = nf ? __int_as_float(0x7FC00000) : A;
  st->nonfinite = nf;
  st->s = s;
  st->scale = scale;
  st->scale_inv = __fdiv_rn(1.0f, scale);
  st->mu_used = mu_used;
  st->sig2 = 0.0;
  st->err2 = 0.0;
  st->underflow = 0;
  st->overflow = 0;
  st->sat = 0;
  st->scratch[SCR_AMAX] = 0;
  st->scratch[SCR_NONFINITE] = 0;
}

// ------------------------------------------------------------------ the strategies
struct Acc {
  double sig2 = 0.0, err2 = 0.0;
  uint32_t under = 0, over = 0, sat = 0;
};

// encode events (R29): underflow = nonzero input -> zero code, overflow = |in| > 448
// (integer tests on the bit patterns: 448 = 0x43E00000; inputs are finite)
__device__ __forceinline__ void count_events(float y, uint32_t code, Acc& a) {
  const uint32_t ab = abs_bits(y);
  a.under += (ab != 0u) & ((code & 0x7Fu) == 0u);
  a.over += ab > 0x43E00000u;
}

// two encodes with one cvt each way: codes (lo byte = y0) and the exact decoded values
__device__ __forceinline__ void enc_dec2(float y0, float y1, Acc& a, uint32_t& c0, uint32_t& c1,
                                         float& d0, float& d1) {
  const uint32_t c = e4m3x2(y0, y1);
  dec_e4m3x2(c, d0, d1);
  c0 = c & 0xFFu;
  c1 = c >> 8;
  count_events(y0, c0, a);
  count_events(y1, c1, a);
}

template <int STRAT, int V>
__device__ __forceinline__ void strat_elems(const float* __restrict__ g, int N, int64_t n, int64_t i,
                                            float s, float inv_n, bool pow2, float sinv,
                                            uint8_t* codes, Acc& a) {
  constexpr int V2 = V < 2 ? 2 : V;       // V = 1 runs the pair code with a dummy lane
  float S[V2];
  double msum[V2];
#pragma unroll 4
  for (int r = 0; r < N; ++r) {
    float x[V2];
    if (V == 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(g + (int64_t)r * n + i));
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
      x[0] = __ldg(g + (int64_t)r * n + i);
      x[1] = 0.0f;
    }
    float y[V2];
#pragma unroll
    for (int j = 0; j < V2; ++j) {
      y[j] = __fmul_rn(x[j], s);                                  // fl(g s)
      if (STRAT == FP8LM_STRATEGY_PRE)                            // Eq. 1: fl(fl(g s) / N)
        y[j] = pow2 ? __fmul_rn(y[j], inv_n) : __fdiv_rn(y[j], (float)N);
    }
#pragma unroll
    for (int j = 0; j < V2; j += 2) {
      uint32_t c0, c1;
      float d0, d1;
      enc_dec2(y[j], y[j + 1], a, c0, c1, d0, d1);
      if (r == 0) {                                               // rank order (R12)
        S[j] = d0; S[j + 1] = d1;
        msum[j] = (double)x[j]; msum[j + 1] = (double)x[j + 1];
      } else {
        S[j] = __fadd_rn(S[j], d0); S[j + 1] = __fadd_rn(S[j + 1], d1);
        msum[j] = __dadd_rn(msum[j], (double)x[j]);
        msum[j + 1] = __dadd_rn(msum[j + 1], (double)x[j + 1]);
      }
    }
  }
  uint32_t cw = 0;
#pragma unroll
  for (int j = 0; j < V2; j += 2) {
    uint32_t c0, c1;
    float d0, d1;
    enc_dec2(S[j], S[j + 1], a, c0, c1, d0, d1);   // E4M3 of the sum (R13); a dummy lane is 0
    const uint32_t cc[2] = {c0, c1};
    const float dd[2] = {d0, d1};
#pragma unroll
    for (int h = 0; h < (V == 1 ? 1 : 2); ++h) {
      a.sat += (cc[h] & 0x7Fu) == 0x7Eu;
      const float gh = __fmul_rn(dd[h], sinv);                    // A6 dequantize
      const double m = __ddiv_rn(msum[j + h], (double)N);
      const double e = __dsub_rn((double)gh, m);
      a.sig2 = __fma_rn(m, m, a.sig2);
      a.err2 = __fma_rn(e, e, a.err2);
      cw |= cc[h] << (8 * (j + h));
    }
  }
  if (codes) {
    if (V == 4) *reinterpret_cast<uint32_t*>(codes + i) = cw;
    else codes[i] = (uint8_t)cw;
  }
}

template <int STRAT, bool VEC>
__global__ void __launch_bounds__(kST) k_strat_reduce(const float* __restrict__ g, int N, int64_t n,
                                                      uint8_t* codes, fp8lm_commstats* st, float* mu) {
  const float s = st->s, sinv = st->scale_inv;
  const bool pow2 = (N & (N - 1)) == 0;
  const float inv_n = __fdiv_rn(1.0f, (float)N);
  Acc a;
  if (VEC) {
    const int64_t nv = n / 4;
    const int64_t b = range_first(nv), e = range_end(nv);
    for (int64_t q = b + threadIdx.x; q < e; q += kST)
      strat_elems<STRAT, 4>(g, N, n, q * 4, s, inv_n, pow2, sinv, codes, a);
    if (blockIdx.x == gridDim.x - 1)
      for (int64_t i = nv * 4 + threadIdx.x; i < n; i += kST)
        strat_elems<STRAT, 1>(g, N, n, i, s, inv_n, pow2, sinv, codes, a);
  } else {
    const int64_t b = range_first(n), e = range_end(n);
    for (int64_t i = b + threadIdx.x; i < e; i += kST)
      strat_elems<STRAT, 1>(g, N, n, i, s, inv_n, pow2, sinv, codes, a);
  }
  // one flush per warp (the error sums are binary64 atomics: their order varies, the
  // tests compare them with a relative tolerance; every count is exact)
  const double s2 = warp_sum_f64(a.sig2), e2 = warp_sum_f64(a.err2);
  const unsigned long long un = warp_sum_u64(a.under), ov = warp_sum_u64(a.over);
  const uint32_t sa = warp_sum(a.sat);
  if ((threadIdx.x & 31) == 0) {
    if (s2 != 0.0) atomicAdd(&st->sig2, s2);
    if (e2 != 0.0) atomicAdd(&st->err2, e2);
    if (un) atomicAdd(reinterpret_cast<unsigned long long*>(&st->underflow), un);
    if (ov) atomicAdd(reinterpret_cast<unsigned long long*>(&st->overflow), ov);
    if (sa) atomicAdd(&st->sat, sa);
  }
  if (!last_cta(&st->scratch[SCR_TICKET_R])) return;
  if (threadIdx.x != 0) return;
  st->events = (uint64_t)(N + 1) * (uint64_t)n;
  if (STRAT == FP8LM_STRATEGY_AUTO) {
    // mu update (R1-R3): halve if sat / n > 1e-5, else grow by 2^(1/1000), cap 2
    const float mu_u = st->mu_used;
    const uint64_t sat = st->sat;
    const float next = sat * 100000ull > (uint64_t)n ? __fmul_rn(mu_u, 0.5f)
                                                     : fminf(2.0f, __fmul_rn(mu_u, kMuGrowth));
    st->mu_next = next;
    *mu = next;
  } else {
    st->mu_next = 1.0f;
  }
}

template <typename K>
int occupancy_grid(K kernel, int64_t work) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kST, 0);
  const int64_t want = (work + kST - 1) / kST;
  int64_t grid = (int64_t)sms * (per > 0 ? per : 1);
  if (want < grid) grid = want;
  return (int)(grid < 1 ? 1 : grid);
}

template <int STRAT>
cudaError_t launch_reduce_t(const float* g, int N, int64_t n, uint8_t* codes, fp8lm_commstats* st,
                            float* mu, bool vec, cudaStream_t s) {
  if (vec) {
    auto k = k_strat_reduce<STRAT, true>;
    k<<<occupancy_grid(k, n / 4 + 1), kST, 0, s>>>(g, N, n, codes, st, mu);
  } else {
    auto k = k_strat_reduce<STRAT, false>;
    k<<<occupancy_grid(k, n), kST, 0, s>>>(g, N, n, codes, st, mu);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_allreduce_strategy(int strategy, const float* g, int N, int64_t n, float* mu,
                                      uint8_t* codes, fp8lm_commstats* st, cudaStream_t s) {
  const int64_t total = (int64_t)N * n;
  const bool vec_a = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  {
    ProfScope ps_(P_STRAT_AMAX, s);
    if (vec_a) {
      auto k = k_strat_amax<true>;
      k<<<occupancy_grid(k, total / 4 + 1), kST, 0, s>>>(g, total, st, mu, strategy, N);
    } else {
      auto k = k_strat_amax<false>;
      k<<<occupancy_grid(k, total), kST, 0, s>>>(g, total, st, mu, strategy, N);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // float4 rows need 16-byte aligned rows (and codes 4-byte aligned)
  const bool vec = vec_a && n % 4 == 0 && (reinterpret_cast<uintptr_t>(codes) & 3) == 0;
  ProfScope ps_(P_STRAT_REDUCE, s);
  switch (strategy) {
    case FP8LM_STRATEGY_PRE: return launch_reduce_t<FP8LM_STRATEGY_PRE>(g, N, n, codes, st, mu, vec, s);
    case FP8LM_STRATEGY_POST: return launch_reduce_t<FP8LM_STRATEGY_POST>(g, N, n, codes, st, mu, vec, s);
    default: return launch_reduce_t<FP8LM_STRATEGY_AUTO>(g, N, n, codes, st, mu, vec, s);
  }
}

}  // namespace fp8lm
