// sp.cu — the FP8 activation converter g between the sequence- and tensor-parallel
// regions (§2.3, Fig. 5; readings R31-R32):
// "We add an FP8 datatype conversion prior to g, such that the all-gather (or
// reduce-scatter) operation uses FP8 low-bit activation to save communication cost".
//
// Transport: NVLink peer memory (CUDA IPC windows of fp8lm_sp), no NCCL on the data
// path.  Every op is ONE cooperative kernel in three phases separated by grid barriers:
//   1  local amax -> s_r; the last CTA publishes s_r into every rank's pad, waits for all
//      ranks and takes the MIN (Eq. 4)
//   2  all-gather: quantize the local partition into the own receive window at
//      rank * m; reduce-scatter: quantize the full local gradient into the own send
//      window; the last CTA releases "data" to every rank, all CTAs wait for every
//      rank's "data"
//   3  all-gather: LOAD rank r's codes from rank r's receive window (pull over NVLink)
//      and copy them out and / or dequantize them into the caller's buffers;
//      reduce-scatter: LOAD chunk `rank` from every rank's send window, sum in rank
//      order in binary32, fl(S * fl(1/s)) -> out
// Flags carry the op's epoch (host counter, identical on every rank): "scale" (s_r
// published), "data" (codes stored / quantized) and "done" (this rank no longer reads
// its receive window / peers' send windows for that epoch), each one u32 per source
// rank in every rank's pad.  A push / quantize waits for the previous epoch's "done"
// of every rank before overwriting a window somebody may still read.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device.cuh"
#include "internal.h"

namespace fp8lm {

namespace {

constexpr int kSpT = 256;

__device__ __forceinline__ uint32_t* sp_flags(uint32_t* pad, size_t off) {
  return reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pad) + off);
}

// this CTA's copy of the peer table (device copy lives in the own pad)
template <int NR>
struct Peers {
  uint8_t* recv[NR];
  uint8_t* send[NR];
  uint32_t* pad[NR];
};
template <int NR>
__device__ __forceinline__ Peers<NR> load_peers(const SpArgs& a) {
  __shared__ uint8_t* r_[kMaxPeers];
  __shared__ uint8_t* s_[kMaxPeers];
  __shared__ uint32_t* p_[kMaxPeers];
  const SpTable* tab = reinterpret_cast<const SpTable*>(reinterpret_cast<const uint8_t*>(a.pad) + kSpPadTable);
  if (threadIdx.x < NR) {
    r_[threadIdx.x] = tab->recv[threadIdx.x];
    s_[threadIdx.x] = tab->send[threadIdx.x];
    p_[threadIdx.x] = tab->pad[threadIdx.x];
  }
  __syncthreads();
  Peers<NR> P;
#pragma unroll
  for (int q = 0; q < NR; ++q) { P.recv[q] = r_[q]; P.send[q] = s_[q]; P.pad[q] = p_[q]; }
  return P;
}

// sys: this CTA wrote memory that peers read (peer stores, the own send window)
__device__ __forceinline__ bool sp_last_cta(uint32_t* ticket, bool sys) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    // one fence per CTA after the barrier: cumulative over every thread's writes
    if (sys) __threadfence_system();
    else __threadfence();
    const uint32_t t = atomicAdd(ticket, 1u);
    last = t == gridDim.x - 1;
    if (last) *ticket = 0;
  }
  __syncthreads();
  if (last) {
    if (sys) __threadfence_system();
    else __threadfence();
  }
  return last;
}

template <int NR>
__device__ __forceinline__ void release_all(const Peers<NR>& P, size_t off, int rank, uint32_t e) {
  // one system fence, then relaxed flag stores (a release pattern per flag): N sequential
  // st.release.sys would cost N x ~1.5 us in this one thread
  __threadfence_system();
#pragma unroll
  for (int q = 0; q < NR; ++q) st_relaxed_sys(sp_flags(P.pad[q], off) + rank, e);
}

__device__ __forceinline__ int64_t cta_lo(int64_t n) { return n * blockIdx.x / gridDim.x; }
__device__ __forceinline__ int64_t cta_hi(int64_t n) { return n * (blockIdx.x + 1) / gridDim.x; }

template <typename T> struct In;
template <> struct In<float> {
  static __device__ __forceinline__ float get(const float* p, int64_t i) { return __ldg(p + i); }
  static __device__ __forceinline__ void get16(const float* p, int64_t i, float* x) {
    const F8 a = ld256_f32(p + i), b = ld256_f32(p + i + 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) { x[k] = a.v[k]; x[8 + k] = b.v[k]; }
  }
};
template <> struct In<__nv_bfloat16> {
  static __device__ __forceinline__ float get(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
  static __device__ __forceinline__ void get16(const __nv_bfloat16* p, int64_t i, float* x) {
    const U8 a = ld256_b32(p + i);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x[2 * k] = __uint_as_float(a.v[k] << 16);
      x[2 * k + 1] = __uint_as_float(a.v[k] & 0xFFFF0000u);
    }
  }
};

template <typename O> struct Out;
template <> struct Out<float> {
  static __device__ __forceinline__ void put(float* p, int64_t i, float v) { p[i] = v; }
  static __device__ __forceinline__ void put16(float* p, int64_t i, const float* v) {
#pragma unroll
    for (int k = 0; k < 16; k += 4)
      st128(p + i + k, make_uint4(__float_as_uint(v[k]), __float_as_uint(v[k + 1]),
                                  __float_as_uint(v[k + 2]), __float_as_uint(v[k + 3])));
  }
};
template <> struct Out<__nv_bfloat16> {
  static __device__ __forceinline__ void put(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }
  static __device__ __forceinline__ uint32_t pack(float lo, float hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);     // RNE, lo in the low half
    return *reinterpret_cast<const uint32_t*>(&h);
  }
  static __device__ __forceinline__ void put16(__nv_bfloat16* p, int64_t i, const float* v) {
    st128(p + i, make_uint4(pack(v[0], v[1]), pack(v[2], v[3]), pack(v[4], v[5]), pack(v[6], v[7])));
    st128(p + i + 8, make_uint4(pack(v[8], v[9]), pack(v[10], v[11]), pack(v[12], v[13]), pack(v[14], v[15])));
  }
};

// grid-wide barrier of a cooperative launch: the last CTA to arrive runs `last` (thread
// 0), then releases the others through a local flag holding the op's epoch
template <typename F>
__device__ __forceinline__ void grid_phase(const SpArgs& a, int ticket, int flag, bool sys, F&& last) {
  if (sp_last_cta(a.scratch + ticket, sys)) {
    if (threadIdx.x == 0) {
      last();
      __threadfence();
      atomicExch(a.scratch + flag, a.epoch);
    }
  }
  if (threadIdx.x == 0) {
    volatile uint32_t* f = a.scratch + flag;
    while (*f != a.epoch) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------------------ phase 1: A, s_r, MIN
template <typename T, int NR>
__device__ __forceinline__ void phase_scale(const T* __restrict__ x, int64_t n, const SpArgs& a,
                                            const Peers<NR>& P, float* scale_out) {
  uint32_t m = 0, bad = 0;
  const int64_t ng = a.vec ? n / 16 : 0;
  for (int64_t gi = cta_lo(ng) + threadIdx.x, e = cta_hi(ng); gi < e; gi += kSpT) {
    float v[16];
    In<T>::get16(x, gi * 16, v);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t b = abs_bits(v[k]);
      m = max(m, b);
      bad |= b >= 0x7F800000u;
    }
  }
  const int64_t t0 = ng * 16;
  for (int64_t i = t0 + cta_lo(n - t0) + threadIdx.x, e = t0 + cta_hi(n - t0); i < e; i += kSpT) {
    const uint32_t b = abs_bits(In<T>::get(x, i));
    m = max(m, b);
    bad |= b >= 0x7F800000u;
  }
  m = warp_max(m);
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (m) atomicMax(a.scratch + kSpScrAmax, m);
    if (bad) atomicOr(a.scratch + kSpScrBad, 1u);
  }
  grid_phase(a, kSpScrTicketA, kSpScrFlag1, false, [&] {
    // s_r = fl(448 / A_r): 0 if non-finite, +inf if A_r = 0 or the ratio overflows (R14)
    const uint32_t ab = a.scratch[kSpScrAmax];
    float sr;
    if (a.scratch[kSpScrBad]) sr = 0.0f;
    else if (ab == 0) sr = __int_as_float(0x7F800000);
    else sr = __fdiv_rn(448.0f, __uint_as_float(ab));
    a.scratch[kSpScrAmax] = 0;
    a.scratch[kSpScrBad] = 0;
#pragma unroll
    for (int q = 0; q < NR; ++q)
      reinterpret_cast<volatile float*>(sp_flags(P.pad[q], kSpPadScales))[a.rank] = sr;
    release_all<NR>(P, kSpPadFlagScale, a.rank, a.epoch);
    wait_epoch(sp_flags(a.pad, kSpPadFlagScale), NR, a.epoch);
    // Eq. 4: the MIN of the ranks' scales; every rank zero / tiny -> 1
    const volatile float* sc = reinterpret_cast<const volatile float*>(sp_flags(a.pad, kSpPadScales));
    float s = sc[0];
#pragma unroll
    for (int q = 1; q < NR; ++q) s = fminf(s, sc[q]);
    if (isinf(s)) s = 1.0f;
    const float sinv = __fdiv_rn(1.0f, s);
    a.scratch[kSpScrS] = __float_as_uint(s);
    a.scratch[kSpScrSinv] = __float_as_uint(sinv);
    if (scale_out) { scale_out[0] = s; scale_out[1] = sinv; }
  });
}

// 16 values -> 16 E4M3 codes of fl(x * s)
__device__ __forceinline__ uint4 quant16(const float* x, float s) {
  uint4 c;
  c.x = e4m3x4(__fmul_rn(x[0], s), __fmul_rn(x[1], s), __fmul_rn(x[2], s), __fmul_rn(x[3], s));
  c.y = e4m3x4(__fmul_rn(x[4], s), __fmul_rn(x[5], s), __fmul_rn(x[6], s), __fmul_rn(x[7], s));
  c.z = e4m3x4(__fmul_rn(x[8], s), __fmul_rn(x[9], s), __fmul_rn(x[10], s), __fmul_rn(x[11], s));
  c.w = e4m3x4(__fmul_rn(x[12], s), __fmul_rn(x[13], s), __fmul_rn(x[14], s), __fmul_rn(x[15], s));
  return c;
}

// ------------------------------------------------------------------ phase 2: quantize
// PUSH: codes of x[0, n) to every rank's receive window at rank * n (all-gather);
// else: to the own send window (reduce-scatter).  Waits first until every rank is done
// with the previous epoch's windows; the last CTA then releases "data" to every rank.
template <typename T, int NR, bool PUSH>
__device__ __forceinline__ void phase_quant(const T* __restrict__ x, int64_t n, const SpArgs& a,
                                            const Peers<NR>& P) {
  if (threadIdx.x == 0) wait_epoch(sp_flags(a.pad, kSpPadFlagDone), NR, a.epoch - 1);
  __syncthreads();
  const float s = __uint_as_float(*(volatile uint32_t*)(a.scratch + kSpScrS));
  const int64_t dst_off = PUSH ? (int64_t)a.rank * n : 0;
  uint8_t* own_send = P.send[0];
  uint8_t* own_recv = P.recv[0];
#pragma unroll
  for (int q = 1; q < NR; ++q)
    if (q == a.rank) { own_send = P.send[q]; own_recv = P.recv[q]; }
  const int64_t ng = a.vec ? n / 16 : 0;
  for (int64_t gi = cta_lo(ng) + threadIdx.x, e = cta_hi(ng); gi < e; gi += kSpT) {
    float v[16];
    In<T>::get16(x, gi * 16, v);
    const uint4 c = quant16(v, s);
    if (PUSH) st128(own_recv + dst_off + gi * 16, c);   // all-gather: pulled by the peers
    else st128(own_send + gi * 16, c);
  }
  const int64_t t0 = ng * 16;
  for (int64_t i = t0 + cta_lo(n - t0) + threadIdx.x, e = t0 + cta_hi(n - t0); i < e; i += kSpT) {
    const uint8_t c = (uint8_t)(e4m3x2(__fmul_rn(In<T>::get(x, i), s), 0.0f) & 0xFFu);
    if (PUSH) own_recv[dst_off + i] = c;
    else own_send[i] = c;
  }
  // the codes are local (own window): a gpu-scope ticket, release_all's fence.sys covers them
  grid_phase(a, kSpScrTicketB, kSpScrFlag2, false, [&] { release_all<NR>(P, kSpPadFlagData, a.rank, a.epoch); });
  if (threadIdx.x == 0) wait_epoch(sp_flags(a.pad, kSpPadFlagData), NR, a.epoch);
  __syncthreads();
}

// ------------------------------------------------------------------ all-gather kernel
template <typename T, typename O, int NR>
__global__ void __launch_bounds__(kSpT) k_sp_allgather(const T* __restrict__ x, int64_t m, uint8_t* codes_out,
                                                       O* out, float* scale_out, SpArgs a) {
  const Peers<NR> P = load_peers<NR>(a);
  phase_scale<T, NR>(x, m, a, P, scale_out);
  phase_quant<T, NR, true>(x, m, a, P);
  // phase 3: every rank's codes have landed: copy them out and / or dequantize
  // PULL: rank r's codes are read straight from rank r's receive window (NVLink), so
  // the transfer and the dequantize are one pass instead of a push followed by a read
  const float sinv = __uint_as_float(*(volatile uint32_t*)(a.scratch + kSpScrSinv));
  const int64_t total = m * NR;
  if (codes_out || out) {
    const int64_t ng = a.vec ? total / 16 : 0;
    const int64_t gm = m / 16;                       // groups per rank (vector path)
    constexpr int U = 4;                             // 16-byte peer loads in flight
    for (int64_t g0 = cta_lo(ng) + threadIdx.x, e = cta_hi(ng); g0 < e; g0 += (int64_t)kSpT * U) {
      uint4 c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t gi = g0 + (int64_t)u * kSpT;
        if (gi < e) c[u] = ld128_peer(P.recv[(int)(gi / gm)] + gi * 16);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t gi = g0 + (int64_t)u * kSpT;
        if (gi >= e) continue;
        if (codes_out) st128(codes_out + gi * 16, c[u]);
        if (out) {
          float d[16];
          dec_e4m3x4(c[u].x, d); dec_e4m3x4(c[u].y, d + 4); dec_e4m3x4(c[u].z, d + 8); dec_e4m3x4(c[u].w, d + 12);
#pragma unroll
          for (int k = 0; k < 16; ++k) d[k] = __fmul_rn(d[k], sinv);
          Out<O>::put16(out, gi * 16, d);
        }
      }
    }
    const int64_t t0 = ng * 16;
    for (int64_t i = t0 + cta_lo(total - t0) + threadIdx.x, e = t0 + cta_hi(total - t0); i < e; i += kSpT) {
      const uint8_t c = P.recv[(int)(i / m)][i];
      if (codes_out) codes_out[i] = c;
      if (out) {
        float d, u;
        dec_e4m3x2(c, d, u);
        Out<O>::put(out, i, __fmul_rn(d, sinv));
      }
    }
  }
  if (sp_last_cta(a.scratch + kSpScrTicketC, false) && threadIdx.x == 0) {
    release_all<NR>(P, kSpPadFlagDone, a.rank, a.epoch);
  }
}

// ------------------------------------------------------------------ reduce-scatter kernel
// phase 3: pull chunk `rank` (m codes) from every rank's send window over NVLink, sum in
// rank order (binary32, R12), out = fl(S * fl(1/s)) (R32)
template <typename T, typename O, int NR>
__global__ void __launch_bounds__(kSpT) k_sp_reduce_scatter(const T* __restrict__ dy, int64_t m, O* out,
                                                            float* scale_out, SpArgs a) {
  const Peers<NR> P = load_peers<NR>(a);
  phase_scale<T, NR>(dy, m * NR, a, P, scale_out);
  phase_quant<T, NR, false>(dy, m * NR, a, P);
  const float sinv = __uint_as_float(*(volatile uint32_t*)(a.scratch + kSpScrSinv));
  const int64_t base = (int64_t)a.rank * m;
  const int64_t ng = a.vec ? m / 16 : 0;
  for (int64_t gi = cta_lo(ng) + threadIdx.x, e = cta_hi(ng); gi < e; gi += kSpT) {
    uint4 c[NR];
#pragma unroll
    for (int q = 0; q < NR; ++q) c[q] = ld128_peer(P.send[q] + base + gi * 16);
    float S[16];
    dec_e4m3x4(c[0].x, S); dec_e4m3x4(c[0].y, S + 4); dec_e4m3x4(c[0].z, S + 8); dec_e4m3x4(c[0].w, S + 12);
#pragma unroll
    for (int q = 1; q < NR; ++q) {
      float d[16];
      dec_e4m3x4(c[q].x, d); dec_e4m3x4(c[q].y, d + 4); dec_e4m3x4(c[q].z, d + 8); dec_e4m3x4(c[q].w, d + 12);
#pragma unroll
      for (int k = 0; k < 16; ++k) S[k] = __fadd_rn(S[k], d[k]);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) S[k] = __fmul_rn(S[k], sinv);
    Out<O>::put16(out, gi * 16, S);
  }
  const int64_t t0 = ng * 16;
  for (int64_t i = t0 + cta_lo(m - t0) + threadIdx.x, e = t0 + cta_hi(m - t0); i < e; i += kSpT) {
    float S = 0.0f;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
      float d, u;
      dec_e4m3x2(P.send[q][base + i], d, u);
      S = q == 0 ? d : __fadd_rn(S, d);
    }
    Out<O>::put(out, i, __fmul_rn(S, sinv));
  }
  if (sp_last_cta(a.scratch + kSpScrTicketC, false) && threadIdx.x == 0) {
    release_all<NR>(P, kSpPadFlagDone, a.rank, a.epoch);
  }
}

// cooperative launch: the phases' grid barriers need every CTA resident
template <typename K, typename... Args>
cudaError_t coop_launch(K kernel, int64_t work, cudaStream_t s, Args... args) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kSpT, 0);
  // 2 CTAs per SM: the three grid barriers and their flag polling cost more than the
  // extra occupancy buys (measured 1, 2, 4, 8 per SM)
  if (per > 2) per = 2;
  const int64_t want = (work + kSpT - 1) / kSpT;
  int64_t grid = (int64_t)sms * (per > 0 ? per : 1);
  if (want < grid) grid = want;
  if (grid < 1) grid = 1;
  void* params[] = {&args...};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3((unsigned)grid), dim3(kSpT),
                                     params, 0, s);
}

template <int NR, typename T>
cudaError_t sp_allgather_t(const void* x, int64_t m, uint8_t* codes_out, void* out, int out_dtype,
                           float* scale_out, const SpArgs& a, cudaStream_t s) {
  ProfScope ps_(P_SP_ALLGATHER, s);
  const int64_t work = std::max<int64_t>(m, m * NR / 16);
  if (out_dtype == FP8LM_BF16)
    return coop_launch(k_sp_allgather<T, __nv_bfloat16, NR>, work, s, static_cast<const T*>(x), m, codes_out,
                       static_cast<__nv_bfloat16*>(out), scale_out, a);
  return coop_launch(k_sp_allgather<T, float, NR>, work, s, static_cast<const T*>(x), m, codes_out,
                     static_cast<float*>(out), scale_out, a);
}

template <int NR>
cudaError_t sp_allgather_n(const void* x, int x_dtype, int64_t m, uint8_t* codes_out, void* out,
                           int out_dtype, float* scale_out, const SpArgs& a, cudaStream_t s) {
  return x_dtype == FP8LM_F32 ? sp_allgather_t<NR, float>(x, m, codes_out, out, out_dtype, scale_out, a, s)
                              : sp_allgather_t<NR, __nv_bfloat16>(x, m, codes_out, out, out_dtype, scale_out, a, s);
}

template <int NR, typename T>
cudaError_t sp_reduce_scatter_t(const void* dy, int64_t m, void* out, int out_dtype, float* scale_out,
                                const SpArgs& a, cudaStream_t s) {
  ProfScope ps_(P_SP_REDUCE_SCATTER, s);
  const int64_t work = m * NR;
  if (out_dtype == FP8LM_BF16)
    return coop_launch(k_sp_reduce_scatter<T, __nv_bfloat16, NR>, work, s, static_cast<const T*>(dy), m,
                       static_cast<__nv_bfloat16*>(out), scale_out, a);
  return coop_launch(k_sp_reduce_scatter<T, float, NR>, work, s, static_cast<const T*>(dy), m,
                     static_cast<float*>(out), scale_out, a);
}

template <int NR>
cudaError_t sp_reduce_scatter_n(const void* dy, int dtype, int64_t m, void* out, int out_dtype,
                                float* scale_out, const SpArgs& a, cudaStream_t s) {
  return dtype == FP8LM_F32 ? sp_reduce_scatter_t<NR, float>(dy, m, out, out_dtype, scale_out, a, s)
                            : sp_reduce_scatter_t<NR, __nv_bfloat16>(dy, m, out, out_dtype, scale_out, a, s);
}

}  // namespace

cudaError_t launch_sp_allgather(const void* x, int x_dtype, int64_t m, uint8_t* codes_out, void* out,
                                int out_dtype, float* scale_out, const SpArgs& a, cudaStream_t s) {
  switch (a.nranks) {
    case 1: return sp_allgather_n<1>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 2: return sp_allgather_n<2>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 3: return sp_allgather_n<3>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 4: return sp_allgather_n<4>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 5: return sp_allgather_n<5>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 6: return sp_allgather_n<6>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 7: return sp_allgather_n<7>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    case 8: return sp_allgather_n<8>(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_sp_reduce_scatter(const void* dy, int dtype, int64_t m, void* out, int out_dtype,
                                     float* scale_out, const SpArgs& a, cudaStream_t s) {
  switch (a.nranks) {
    case 1: return sp_reduce_scatter_n<1>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 2: return sp_reduce_scatter_n<2>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 3: return sp_reduce_scatter_n<3>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 4: return sp_reduce_scatter_n<4>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 5: return sp_reduce_scatter_n<5>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 6: return sp_reduce_scatter_n<6>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 7: return sp_reduce_scatter_n<7>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    case 8: return sp_reduce_scatter_n<8>(dy, dtype, m, out, out_dtype, scale_out, a, s);
    default: return cudaErrorInvalidValue;
  }
}

FP8LM_WAIT_WATCHDOG_HOOK(wait_watchdog_set_sp)

}  // namespace fp8lm
