// fence_probe.cu — latency of the memory-ordering operations the flag handshakes use, one
// thread, 10000 iterations each (globaltimer ns per op): fence.sc.sys (__threadfence_system),
// fence.acq_rel.sys, fence.acq_rel.gpu (__threadfence), st.release.sys + ld.acquire.sys on
// local memory, and a kernel launch round trip (empty kernels back to back).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void probe(uint32_t* buf, uint64_t* out) {
  const int R = 10000;
  uint64_t t0 = gt();
  for (int i = 0; i < R; ++i) { buf[i & 255] = i; __threadfence_system(); }
  uint64_t t1 = gt();
  for (int i = 0; i < R; ++i) { buf[i & 255] = i; asm volatile("fence.acq_rel.sys;" ::: "memory"); }
  uint64_t t2 = gt();
  for (int i = 0; i < R; ++i) { buf[i & 255] = i; __threadfence(); }
  uint64_t t3 = gt();
  for (int i = 0; i < R; ++i) asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(buf + (i & 255)), "r"(i) : "memory");
  uint64_t t4 = gt();
  uint32_t acc = 0;
  for (int i = 0; i < R; ++i) { uint32_t v; asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(buf + (i & 255)) : "memory"); acc += v; }
  uint64_t t5 = gt();
  for (int i = 0; i < R; ++i) { uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(buf + (i & 255)) : "memory"); acc += v; }
  uint64_t t6 = gt();
  out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5; out[6] = acc;
}
__global__ void empty() {}
int main() {
  uint32_t* buf; uint64_t* out; cudaMalloc(&buf, 4096); cudaMallocManaged(&out, 64);
  probe<<<1, 1>>>(buf, out); cudaDeviceSynchronize();
  probe<<<1, 1>>>(buf, out); cudaDeviceSynchronize();
  const char* names[6] = {"st + fence.sc.sys (__threadfence_system)", "st + fence.acq_rel.sys", "st + fence.acq_rel.gpu (__threadfence)",
                          "st.release.sys", "ld.acquire.sys", "ld.relaxed.gpu"};
  for (int k = 0; k < 6; ++k) printf("%-45s %8.1f ns/op\n", names[k], out[k] / 10000.0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 100; ++i) empty<<<1, 32>>>();
  cudaEventRecord(a); for (int i = 0; i < 1000; ++i) empty<<<1, 32>>>(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); printf("%-45s %8.2f us/launch\n", "empty kernel back to back", ms);
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(32);
  cudaLaunchAttribute at; at.id = cudaLaunchAttributeCooperative; at.val.cooperative = 1; cfg.attrs = &at; cfg.numAttrs = 1;
  cudaEventRecord(a); for (int i = 0; i < 1000; ++i) cudaLaunchKernelEx(&cfg, empty); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("%-45s %8.2f us/launch\n", "empty cooperative kernel back to back", ms);
  return 0;
}
