// store_probe.cu — how fast can a 6 B in / 6 B out per element streaming pass run on
// B200, by store path?  (pass 2 of the FP8 AdamW: g8 u8, m1 u8, v u16, w u16 in; w8 u8,
// m1 u8, v u16, w u16 out).  Trivial compute; the question is the memory pipeline.
//   A: 1-D TMA load ring (4 x 24 KB stages, producer warp) + st.global from registers
//   B: the same ring, results written back into the stage, TMA bulk stores by a storer warp
//   C: plain 128-bit ld.global.nc / st.global, no shared memory
//   D: cudaMemcpy D2D of the same byte count (12 B per element, half read / half write)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe store_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kT = 256, kG = 16, kTile = kT * kG, kSt = 4;
struct Stage { uint8_t g[kTile]; uint8_t m[kTile]; uint16_t v[kTile]; uint16_t w[kTile]; };

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" :: "r"(su(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory"); }
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(d), "r"(su(s)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory"); }

struct Args { const uint8_t* g; uint8_t* m; uint16_t* v; uint16_t* w; uint8_t* w8; int64_t ntiles; };

__device__ __forceinline__ void issue(const Args& a, int64_t t, Stage* st, uint64_t* full) {
  const int64_t e = t * kTile;
  mb_expect(full, 6 * kTile);
  g2s(st->g, a.g + e, kTile, full);
  g2s(st->m, a.m + e, kTile, full);
  g2s(st->v, a.v + e, 2 * kTile, full);
  g2s(st->w, a.w + e, 2 * kTile, full);
}

// ---------------- A: TMA load ring + st.global
__global__ void __launch_bounds__(kT + 32, 2) kA(Args a) {
  extern __shared__ __align__(128) uint8_t sm[];
  Stage* st = reinterpret_cast<Stage*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + sizeof(Stage) * kSt);
  uint64_t* empty = full + kSt;
  if (threadIdx.x == 0) { for (int s = 0; s < kSt; ++s) { mb_init(full + s, 1); mb_init(empty + s, kT / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x >= kT) {
    if ((threadIdx.x & 31) == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++k) {
        const int s = k % kSt;
        if (k >= kSt) mb_wait(empty + s, ((k / kSt) + 1) & 1);
        issue(a, t, st + s, full + s);
      }
    }
    return;
  }
  int k = 0;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++k) {
    const int s = k % kSt;
    mb_wait(full + s, (k / kSt) & 1);
    const Stage& S = st[s];
    const int b = threadIdx.x * kG;
    uint4 g = *reinterpret_cast<const uint4*>(S.g + b), m = *reinterpret_cast<const uint4*>(S.m + b);
    uint4 v0 = *reinterpret_cast<const uint4*>(S.v + b), v1 = *reinterpret_cast<const uint4*>(S.v + b + 8);
    uint4 w0 = *reinterpret_cast<const uint4*>(S.w + b), w1 = *reinterpret_cast<const uint4*>(S.w + b + 8);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mb_arrive(empty + s);
    const int64_t e = t * kTile + b;
    m.x += g.x; v0.x ^= 1; w1.y ^= 3; g.z += 1;
    *reinterpret_cast<uint4*>(a.m + e) = m;
    *reinterpret_cast<uint4*>(a.v + e) = v0; *reinterpret_cast<uint4*>(a.v + e + 8) = v1;
    *reinterpret_cast<uint4*>(a.w + e) = w0; *reinterpret_cast<uint4*>(a.w + e + 8) = w1;
    *reinterpret_cast<uint4*>(a.w8 + e) = g;
  }
}

// ---------------- B: TMA load ring + in-place results + TMA bulk stores by a storer warp
template <int NST, int WD>
__global__ void __launch_bounds__(kT + 64, 1) kB(Args a) {
  constexpr int kSt = NST;
  extern __shared__ __align__(128) uint8_t sm[];
  Stage* st = reinterpret_cast<Stage*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + sizeof(Stage) * kSt);
  uint64_t* empty = full + kSt;
  uint64_t* done = empty + kSt;
  if (threadIdx.x == 0) { for (int s = 0; s < kSt; ++s) { mb_init(full + s, 1); mb_init(empty + s, 1); mb_init(done + s, kT / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kT / 32) {                       // producer
    if (lane == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++k) {
        const int s = k % kSt;
        if (k >= kSt) mb_wait(empty + s, ((k / kSt) + 1) & 1);
        issue(a, t, st + s, full + s);
      }
    }
    return;
  }
  if (warp == kT / 32 + 1) {                   // storer
    if (lane == 0) {
      int k = 0, prev = -1;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++k) {
        const int s = k % kSt;
        mb_wait(done + s, (k / kSt) & 1);
        const int64_t e = t * kTile;
        Stage& S = st[s];
        s2g(a.w8 + e, S.g, kTile);
        s2g(a.m + e, S.m, kTile);
        s2g(a.v + e, S.v, 2 * kTile);
        s2g(a.w + e, S.w, 2 * kTile);
        bulk_commit();
        // release the stage whose store is WD tiles old once its smem has been read
        if (k >= WD) { bulk_wait_read<WD>(); mb_arrive(empty + (k - WD) % kSt); }
        prev = s;
      }
      bulk_wait<0>();
      for (int j = (k > WD ? k - WD : 0); j < k; ++j) mb_arrive(empty + j % kSt);
    }
    return;
  }
  int k = 0;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++k) {
    const int s = k % kSt;
    mb_wait(full + s, (k / kSt) & 1);
    Stage& S = st[s];
    const int b = threadIdx.x * kG;
    uint4 g = *reinterpret_cast<const uint4*>(S.g + b), m = *reinterpret_cast<const uint4*>(S.m + b);
    uint4 v0 = *reinterpret_cast<const uint4*>(S.v + b), v1 = *reinterpret_cast<const uint4*>(S.v + b + 8);
    uint4 w0 = *reinterpret_cast<const uint4*>(S.w + b), w1 = *reinterpret_cast<const uint4*>(S.w + b + 8);
    m.x += g.x; v0.x ^= 1; w1.y ^= 3; g.z += 1;
    *reinterpret_cast<uint4*>(S.m + b) = m;
    *reinterpret_cast<uint4*>(S.v + b) = v0; *reinterpret_cast<uint4*>(S.v + b + 8) = v1;
    *reinterpret_cast<uint4*>(S.w + b) = w0; *reinterpret_cast<uint4*>(S.w + b + 8) = w1;
    *reinterpret_cast<uint4*>(S.g + b) = g;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mb_arrive(done + s);
  }
}

// ---------------- C: plain vector loads / stores
__global__ void __launch_bounds__(kT) kC(Args a) {
  const int64_t n = a.ntiles * kTile / kG;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const int64_t e = i * kG;
    uint4 g = __ldg(reinterpret_cast<const uint4*>(a.g + e)), m = __ldg(reinterpret_cast<const uint4*>(a.m + e));
    uint4 v0 = __ldg(reinterpret_cast<const uint4*>(a.v + e)), v1 = __ldg(reinterpret_cast<const uint4*>(a.v + e + 8));
    uint4 w0 = __ldg(reinterpret_cast<const uint4*>(a.w + e)), w1 = __ldg(reinterpret_cast<const uint4*>(a.w + e + 8));
    m.x += g.x; v0.x ^= 1; w1.y ^= 3; g.z += 1;
    *reinterpret_cast<uint4*>(a.m + e) = m;
    *reinterpret_cast<uint4*>(a.v + e) = v0; *reinterpret_cast<uint4*>(a.v + e + 8) = v1;
    *reinterpret_cast<uint4*>(a.w + e) = w0; *reinterpret_cast<uint4*>(a.w + e + 8) = w1;
    *reinterpret_cast<uint4*>(a.w8 + e) = g;
  }
}

int main() {
  const int64_t n = (int64_t)1 << 30;        // elements: 6 GB in, 6 GB out
  Args a;
  a.ntiles = n / kTile;
  uint8_t *g, *m, *w8; uint16_t *v, *w;
  cudaMalloc(&g, n); cudaMalloc(&m, n); cudaMalloc(&w8, n); cudaMalloc(&v, 2 * n); cudaMalloc(&w, 2 * n);
  cudaMemset(g, 1, n); cudaMemset(m, 2, n); cudaMemset(v, 3, 2 * n); cudaMemset(w, 4, 2 * n);
  a.g = g; a.m = m; a.v = v; a.w = w; a.w8 = w8;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smA = sizeof(Stage) * kSt + 128;
  cudaFuncSetAttribute(kA, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA);
  uint8_t *cs, *cd; cudaMalloc(&cs, 6 * n); cudaMalloc(&cd, 6 * n); cudaMemset(cs, 5, 6 * n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = 12.0 * n;
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-28s %.3f ms  %.0f GB/s  %s\n", name, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("A tma-load + st.global", [&] { kA<<<2 * sms, kT + 32, smA>>>(a); });
#define VB(NST, WD, CPS)                                                                     \
  {                                                                                          \
    const size_t smb = sizeof(Stage) * NST + 256;                                            \
    cudaFuncSetAttribute(kB<NST, WD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb); \
    timeit("B tma st=" #NST " wd=" #WD " cta/sm=" #CPS, [&] { kB<NST, WD><<<CPS * sms, kT + 64, smb>>>(a); }); \
  }
  VB(4, 1, 2) VB(4, 2, 2) VB(3, 1, 2) VB(8, 1, 1) VB(8, 2, 1) VB(8, 4, 1) VB(3, 1, 3) VB(2, 1, 3) VB(2, 1, 4)
  timeit("C plain ld/st", [&] { kC<<<4 * sms, kT>>>(a); });
  timeit("D cudaMemcpy 6n", [&] { cudaMemcpyAsync(cd, cs, (size_t)(6 * n), cudaMemcpyDeviceToDevice); });
  return 0;
}
