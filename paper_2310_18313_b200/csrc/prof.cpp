// prof.cpp — launch tracing (the "tracing / profiling" auxiliary subsystem of SURVEY §5):
// CUDA-event brackets around every kernel and NCCL call the library enqueues, enabled
// on demand, aggregated per name.  Disabled (the default) it costs one branch.
#include <atomic>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "internal.h"

namespace fp8lm {

static const char* kNames[P_COUNT] = {
    "amax", "scale", "scale_fix", "quantize", "reduce", "allreduce_finalize", "adam_pass1",
    "adam_pass2", "adam_finalize", "adam_wfix", "state_init", "quantize_single", "dequantize_single",
    "memset", "nccl_allreduce_min", "nccl_alltoall", "nccl_allgather+sum", "reduce_p2p", "quantize+adam_pass1", "w8_broadcast", "adam_delayed",
    "quantize+adam_delayed", "strategy_amax", "strategy_reduce",
    "sp_allgather", "sp_reduce_scatter"};
static const bool kIsOurs[P_COUNT] = {true, true, true, true, true, true, true, true, true,
                                      true, true, true, true, false, false, false, false, true,
                                      true, true, true, true, true, true, true, true};

struct Rec {
  int id;
  cudaEvent_t a, b;
};

static std::mutex g_mu;
static std::atomic<bool> g_on{false};
static std::vector<Rec> g_recs;
static std::vector<cudaEvent_t> g_free;

static cudaEvent_t get_event() {
  if (!g_free.empty()) {
    cudaEvent_t e = g_free.back();
    g_free.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

bool prof_on() { return g_on.load(std::memory_order_relaxed); }

ProfScope::ProfScope(int id_, cudaStream_t s_) : id(id_), s(s_) {
  if (!prof_on()) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t e = get_event();
  cudaEventRecord(e, s);
  a = e;
}

ProfScope::~ProfScope() {
  if (!a) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t e = get_event();
  cudaEventRecord(e, s);
  g_recs.push_back(Rec{id, static_cast<cudaEvent_t>(a), e});
}

}  // namespace fp8lm

using namespace fp8lm;

extern "C" {

int fp8lm_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (on) {   // a new window: recycle the previous window's events
    for (auto& r : g_recs) { g_free.push_back(r.a); g_free.push_back(r.b); }
    g_recs.clear();
  }
  g_on.store(on != 0);
  return FP8LM_OK;
}

int fp8lm_prof_read(int32_t id, const char** name, int64_t* launches, double* total_ms,
                    int32_t* is_ours) {
  if (id < 0 || id >= P_COUNT) return FP8LM_EINVAL;
  std::lock_guard<std::mutex> lk(g_mu);
  int64_t n = 0;
  double ms = 0.0;
  for (auto& r : g_recs) {
    if (r.id != id) continue;
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return FP8LM_ECUDA;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return FP8LM_ECUDA;
    ++n;
    ms += t;
  }
  if (name) *name = kNames[id];
  if (launches) *launches = n;
  if (total_ms) *total_ms = ms;
  if (is_ours) *is_ours = kIsOurs[id] ? 1 : 0;
  return FP8LM_OK;
}

int fp8lm_prof_ids(void) { return P_COUNT; }

}  // extern "C"
