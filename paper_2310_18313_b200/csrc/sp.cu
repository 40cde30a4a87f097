// sp.cu — the FP8 activation converter g between the sequence- and tensor-parallel
// regions (§2.3, Fig. 5; readings R31-R32):
// "We add an FP8 datatype conversion prior to g, such that the all-gather (or
// reduce-scatter) operation uses FP8 low-bit activation to save communication cost".
//
// Transport: NVLink peer memory (CUDA IPC windows of fp8lm_sp), no NCCL on the data
// path.  Every op is three kernels on the caller's stream:
//   k_sp_amax        local amax -> s_r; the last CTA publishes s_r into every rank's pad,
//                    waits for all ranks and takes the MIN (Eq. 4)
//   all-gather:      k_sp_push      quantize the local partition and STORE the codes into
//                                   every rank's receive window (push all-gather)
//                    k_sp_gather    wait for every rank's data, copy the gathered codes
//                                   and / or dequantize them into the caller's buffers
//   reduce-scatter:  k_sp_quant     quantize the full local gradient into the own send
//                                   window
//                    k_sp_pull      wait, LOAD chunk `rank` from every rank's send window,
//                                   rank-order binary32 sum, fl(S * fl(1/s)) -> out
// Flags carry the op's epoch (host counter, identical on every rank): "scale" (s_r
// published), "data" (codes stored / quantized) and "done" (this rank no longer reads
// its receive window / peers' send windows for that epoch), each one u32 per source
// rank in every rank's pad.  A push / quantize waits for the previous epoch's "done"
// of every rank before overwriting a window somebody may still read.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

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

__device__ __forceinline__ bool sp_last_cta(uint32_t* ticket) {
  __shared__ int last;
  __threadfence_system();       // this CTA's peer stores / local writes
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(ticket, 1u);
    last = t == gridDim.x - 1;
    if (last) *ticket = 0;
  }
  __syncthreads();
  if (last) __threadfence_system();
  return last;
}

template <int NR>
__device__ __forceinline__ void release_all(const Peers<NR>& P, size_t off, int rank, uint32_t e) {
#pragma unroll
  for (int q = 0; q < NR; ++q) st_release_sys(sp_flags(P.pad[q], off) + rank, e);
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

// ------------------------------------------------------------------ A, s_r, MIN
template <typename T, int NR>
__global__ void __launch_bounds__(kSpT) k_sp_amax(const T* __restrict__ x, int64_t n, SpArgs a,
                                                  float* scale_out) {
  const Peers<NR> P = load_peers<NR>(a);
  uint32_t m = 0, bad = 0;
  for (int64_t i = cta_lo(n) + threadIdx.x, e = cta_hi(n); i < e; i += kSpT) {
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
  if (!sp_last_cta(a.scratch + kSpScrTicketA)) return;
  if (threadIdx.x != 0) return;
  // s_r = fl(448 / A_r): 0 if non-finite, +inf if A_r = 0 or the ratio overflows (R14)
  const uint32_t ab = a.scratch[kSpScrAmax];
  float sr;
  if (a.scratch[kSpScrBad]) {
    sr = 0.0f;
  } else if (ab == 0) {
    sr = __int_as_float(0x7F800000);
  } else {
    sr = __fdiv_rn(448.0f, __uint_as_float(ab));
  }
  a.scratch[kSpScrAmax] = 0;
  a.scratch[kSpScrBad] = 0;
#pragma unroll
  for (int q = 0; q < NR; ++q)
    reinterpret_cast<volatile float*>(sp_flags(P.pad[q], kSpPadScales))[a.rank] = sr;
  __threadfence_system();
  release_all<NR>(P, kSpPadFlagScale, a.rank, a.epoch);
  wait_epoch(sp_flags(a.pad, kSpPadFlagScale), NR, a.epoch);
  const volatile float* sc = reinterpret_cast<const volatile float*>(sp_flags(a.pad, kSpPadScales));
  float s = sc[0];
#pragma unroll
  for (int q = 1; q < NR; ++q) s = fminf(s, sc[q]);
  if (isinf(s)) s = 1.0f;                       // every rank zero / tiny
  const float sinv = __fdiv_rn(1.0f, s);
  a.scratch[kSpScrS] = __float_as_uint(s);
  a.scratch[kSpScrSinv] = __float_as_uint(sinv);
  if (scale_out) { scale_out[0] = s; scale_out[1] = sinv; }
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

template <int NR>
__device__ __forceinline__ void wait_done_prev(const SpArgs& a) {
  if (threadIdx.x == 0) wait_epoch(sp_flags(a.pad, kSpPadFlagDone), NR, a.epoch - 1);
  __syncthreads();
}

// ------------------------------------------------------------------ all-gather
// PUSH = true: codes of x[0, m) go to every rank's receive window at rank * m (k_sp_push)
// PUSH = false: codes of x[0, n) go to the own send window at 0 (k_sp_quant, RS)
template <typename T, int NR, bool PUSH>
__global__ void __launch_bounds__(kSpT) k_sp_quant(const T* __restrict__ x, int64_t n, SpArgs a) {
  const Peers<NR> P = load_peers<NR>(a);
  wait_done_prev<NR>(a);
  const float s = __uint_as_float(a.scratch[kSpScrS]);
  const int64_t dst_off = PUSH ? (int64_t)a.rank * n : 0;
  const bool vec = a.vec;
  if (vec) {
    const int64_t ng = n / 16;
    for (int64_t gi = cta_lo(ng) + threadIdx.x, e = cta_hi(ng); gi < e; gi += kSpT) {
      float v[16];
      In<T>::get16(x, gi * 16, v);
      const uint4 c = quant16(v, s);
      if (PUSH) {
#pragma unroll
        for (int q = 0; q < NR; ++q) st128(P.recv[q] + dst_off + gi * 16, c);
      } else {
        st128(P.send[a.rank] + gi * 16, c);
      }
    }
  }
  const int64_t tail0 = vec ? n / 16 * 16 : 0;
  for (int64_t i = tail0 + cta_lo(n - tail0) + threadIdx.x, e = tail0 + cta_hi(n - tail0); i < e; i += kSpT) {
    const uint8_t c = (uint8_t)(e4m3x2(__fmul_rn(In<T>::get(x, i), s), 0.0f) & 0xFFu);
    if (PUSH) {
#pragma unroll
      for (int q = 0; q < NR; ++q) P.recv[q][dst_off + i] = c;
    } else {
      P.send[a.rank][i] = c;
    }
  }
  if (sp_last_cta(a.scratch + kSpScrTicketB) && threadIdx.x == 0)
    release_all<NR>(P, kSpPadFlagData, a.rank, a.epoch);
}

template <typename O> struct Out;
template <> struct Out<float> {
  static __device__ __forceinline__ void put(float* p, int64_t i, float v) { p[i] = v; }
};
template <> struct Out<__nv_bfloat16> {
  static __device__ __forceinline__ void put(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }
};

// wait for every rank's codes, copy them out and / or dequantize fl(dec(c) * sinv)
template <typename O, int NR>
__global__ void __launch_bounds__(kSpT) k_sp_gather(int64_t total, uint8_t* codes_out, O* out, SpArgs a) {
  const Peers<NR> P = load_peers<NR>(a);
  if (threadIdx.x == 0) wait_epoch(sp_flags(a.pad, kSpPadFlagData), NR, a.epoch);
  __syncthreads();
  const float sinv = __uint_as_float(a.scratch[kSpScrSinv]);
  const uint8_t* src = P.recv[a.rank];
  if (codes_out || out) {
    const int64_t ng = a.vec ? total / 16 : 0;
    for (int64_t gi = cta_lo(ng) + threadIdx.x, e = cta_hi(ng); gi < e; gi += kSpT) {
      const uint4 c = ld128_nc(src + gi * 16);
      if (codes_out) st128(codes_out + gi * 16, c);
      if (out) {
        float d[16];
        dec_e4m3x4(c.x, d); dec_e4m3x4(c.y, d + 4); dec_e4m3x4(c.z, d + 8); dec_e4m3x4(c.w, d + 12);
#pragma unroll
        for (int k = 0; k < 16; ++k) Out<O>::put(out, gi * 16 + k, __fmul_rn(d[k], sinv));
      }
    }
    const int64_t t0 = ng * 16;
    for (int64_t i = t0 + cta_lo(total - t0) + threadIdx.x, e = t0 + cta_hi(total - t0); i < e; i += kSpT) {
      const uint8_t c = src[i];
      if (codes_out) codes_out[i] = c;
      if (out) {
        float d, u;
        dec_e4m3x2(c, d, u);
        Out<O>::put(out, i, __fmul_rn(d, sinv));
      }
    }
  }
  if (sp_last_cta(a.scratch + kSpScrTicketC) && threadIdx.x == 0)
    release_all<NR>(P, kSpPadFlagDone, a.rank, a.epoch);
}

// ------------------------------------------------------------------ reduce-scatter
// wait for every rank's quantized gradient, pull chunk `rank` (m codes) from each send
// window over NVLink, sum in rank order (binary32, R12), out = fl(S * fl(1/s)) (R32)
template <typename O, int NR>
__global__ void __launch_bounds__(kSpT) k_sp_pull(int64_t m, O* out, SpArgs a) {
  const Peers<NR> P = load_peers<NR>(a);
  if (threadIdx.x == 0) wait_epoch(sp_flags(a.pad, kSpPadFlagData), NR, a.epoch);
  __syncthreads();
  const float sinv = __uint_as_float(a.scratch[kSpScrSinv]);
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
    for (int k = 0; k < 16; ++k) Out<O>::put(out, gi * 16 + k, __fmul_rn(S[k], sinv));
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
  if (sp_last_cta(a.scratch + kSpScrTicketC) && threadIdx.x == 0)
    release_all<NR>(P, kSpPadFlagDone, a.rank, a.epoch);
}

template <typename K>
int sp_grid(K kernel, int64_t work) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kSpT, 0);
  const int64_t want = (work + kSpT - 1) / kSpT;
  int64_t grid = (int64_t)sms * (per > 0 ? per : 1);
  if (want < grid) grid = want;
  return (int)(grid < 1 ? 1 : grid);
}

template <typename T, int NR>
cudaError_t sp_amax(const void* x, int64_t n, const SpArgs& a, float* scale_out, cudaStream_t s) {
  auto k = k_sp_amax<T, NR>;
  k<<<sp_grid(k, n), kSpT, 0, s>>>(static_cast<const T*>(x), n, a, scale_out);
  return cudaGetLastError();
}

template <int NR>
cudaError_t sp_allgather_n(const void* x, int x_dtype, int64_t m, uint8_t* codes_out, void* out,
                           int out_dtype, float* scale_out, const SpArgs& a, cudaStream_t s) {
  cudaError_t e;
  {
    ProfScope ps_(P_SP_AMAX, s);
    e = x_dtype == FP8LM_F32 ? sp_amax<float, NR>(x, m, a, scale_out, s)
                             : sp_amax<__nv_bfloat16, NR>(x, m, a, scale_out, s);
    if (e != cudaSuccess) return e;
  }
  {
    ProfScope ps_(P_SP_PUSH, s);
    if (x_dtype == FP8LM_F32) {
      auto k = k_sp_quant<float, NR, true>;
      k<<<sp_grid(k, m / 16 + 1), kSpT, 0, s>>>(static_cast<const float*>(x), m, a);
    } else {
      auto k = k_sp_quant<__nv_bfloat16, NR, true>;
      k<<<sp_grid(k, m / 16 + 1), kSpT, 0, s>>>(static_cast<const __nv_bfloat16*>(x), m, a);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  ProfScope ps_(P_SP_GATHER, s);
  const int64_t total = m * NR;
  if (out_dtype == FP8LM_BF16) {
    auto k = k_sp_gather<__nv_bfloat16, NR>;
    k<<<sp_grid(k, total / 16 + 1), kSpT, 0, s>>>(total, codes_out, static_cast<__nv_bfloat16*>(out), a);
  } else {
    auto k = k_sp_gather<float, NR>;
    k<<<sp_grid(k, total / 16 + 1), kSpT, 0, s>>>(total, codes_out, static_cast<float*>(out), a);
  }
  return cudaGetLastError();
}

template <int NR>
cudaError_t sp_reduce_scatter_n(const void* dy, int dtype, int64_t m, void* out, int out_dtype,
                                float* scale_out, const SpArgs& a, cudaStream_t s) {
  const int64_t n = m * NR;
  cudaError_t e;
  {
    ProfScope ps_(P_SP_AMAX, s);
    e = dtype == FP8LM_F32 ? sp_amax<float, NR>(dy, n, a, scale_out, s)
                           : sp_amax<__nv_bfloat16, NR>(dy, n, a, scale_out, s);
    if (e != cudaSuccess) return e;
  }
  {
    ProfScope ps_(P_SP_QUANT, s);
    if (dtype == FP8LM_F32) {
      auto k = k_sp_quant<float, NR, false>;
      k<<<sp_grid(k, n / 16 + 1), kSpT, 0, s>>>(static_cast<const float*>(dy), n, a);
    } else {
      auto k = k_sp_quant<__nv_bfloat16, NR, false>;
      k<<<sp_grid(k, n / 16 + 1), kSpT, 0, s>>>(static_cast<const __nv_bfloat16*>(dy), n, a);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  ProfScope ps_(P_SP_PULL, s);
  if (out_dtype == FP8LM_BF16) {
    auto k = k_sp_pull<__nv_bfloat16, NR>;
    k<<<sp_grid(k, m / 16 + 1), kSpT, 0, s>>>(m, static_cast<__nv_bfloat16*>(out), a);
  } else {
    auto k = k_sp_pull<float, NR>;
    k<<<sp_grid(k, m / 16 + 1), kSpT, 0, s>>>(m, static_cast<float*>(out), a);
  }
  return cudaGetLastError();
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

}  // namespace fp8lm
