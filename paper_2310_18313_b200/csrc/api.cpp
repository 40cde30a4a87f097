// api.cpp — the C ABI declared in include/fp8lm.h: argument checking, the flat-layout
// plan, the NCCL communicator, and the sequencing of kernels + collectives for the
// four hot-path calls.  Every step of the hot path runs in kernels.cu or in NCCL; this
// file only validates arguments and enqueues work on the caller's stream.
#include <algorithm>
#include <cstdarg>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#ifdef FP8LM_WITH_NCCL
#include <nccl.h>
#endif

#include "config.h"
#include "internal.h"

using namespace fp8lm;

// ---------------------------------------------------------------- error plumbing
static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(FP8LM_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_));            \
  } while (0)

#ifdef FP8LM_WITH_NCCL
#define NCCL_TRY(expr)                                                              \
  do {                                                                              \
    ncclResult_t r_ = (expr);                                                       \
    if (r_ != ncclSuccess)                                                          \
      return fail(FP8LM_ENCCL, "%s: %s", #expr, ncclGetErrorString(r_));            \
  } while (0)
#endif

struct fp8lm_comm {
#ifdef FP8LM_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  int32_t nranks = 0;
  int32_t rank = 0;
  bool owned = true;         // false: attached (fp8lm_comm_attach), not destroyed here
};

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static inline bool aligned(const void* p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

extern "C" {

int fp8lm_version(void) { return FP8LM_ABI_VERSION; }
const char* fp8lm_last_error(void) { return g_err.c_str(); }
int fp8lm_has_nccl(void) {
#ifdef FP8LM_WITH_NCCL
  return 1;
#else
  return 0;
#endif
}

// ---------------------------------------------------------------- host scalars (R24)
int fp8lm_adam_hp_make(double lr, double beta1, double beta2, double eps, double weight_decay,
                       int64_t step, fp8lm_adam_hp* out) {
  if (!out) return fail(FP8LM_EINVAL, "adam_hp_make: out is NULL");
  if (step < 1) return fail(FP8LM_EINVAL, "adam_hp_make: step must be >= 1 (got %lld)", (long long)step);
  if (!std::isfinite(lr) || !std::isfinite(beta1) || !std::isfinite(beta2) || !std::isfinite(eps) ||
      !std::isfinite(weight_decay) || beta1 < 0 || beta1 >= 1 || beta2 < 0 || beta2 >= 1)
    return fail(FP8LM_EINVAL, "adam_hp_make: invalid hyper-parameters");
  out->beta1 = (float)beta1;
  out->beta2 = (float)beta2;
  out->one_minus_beta1 = (float)(1.0 - beta1);
  out->one_minus_beta2 = (float)(1.0 - beta2);
  out->eps = (float)eps;
  out->decay = (float)(1.0 - lr * weight_decay);
  out->step_size = (float)(lr / (1.0 - std::pow(beta1, (double)step)));
  out->inv_bc2_sqrt = (float)(1.0 / std::sqrt(1.0 - std::pow(beta2, (double)step)));
  return FP8LM_OK;
}

// ---------------------------------------------------------------- Alg. 1
int fp8lm_zero_plan(int32_t T, const int64_t* numels, int32_t nranks, int32_t* owner_out,
                    int64_t* load_out) {
  if (T < 0 || nranks < 1) return fail(FP8LM_EINVAL, "zero_plan: T=%d nranks=%d", T, nranks);
  if (T > 0 && (!numels || !owner_out)) return fail(FP8LM_EINVAL, "zero_plan: NULL array");
  if (!load_out) return fail(FP8LM_EINVAL, "zero_plan: load_out is NULL");
  // line 1: sort by size, descending; equal sizes keep ascending original index (R21)
  std::vector<int32_t> order(T);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return numels[a] > numels[b]; });
  // line 2: u_j = 0
  for (int j = 0; j < nranks; ++j) load_out[j] = 0;
  for (int32_t i : order) {                       // line 3
    int j = 0;                                    // line 4: argmin u_j, lowest index on ties
    for (int k = 1; k < nranks; ++k)
      if (load_out[k] < load_out[j]) j = k;
    owner_out[i] = j;                             // line 5
    load_out[j] += numels[i];                     // line 6
  }
  return FP8LM_OK;
}

// ---------------------------------------------------------------- communicator
int fp8lm_comm_unique_id(uint8_t* id_out) {
#ifdef FP8LM_WITH_NCCL
  if (!id_out) return fail(FP8LM_EINVAL, "comm_unique_id: NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
  return FP8LM_OK;
#else
  (void)id_out;
  return fail(FP8LM_EUNSUPPORTED, "built without NCCL");
#endif
}

int fp8lm_comm_init(int32_t nranks, int32_t rank, const uint8_t* id, fp8lm_comm** out) {
#ifdef FP8LM_WITH_NCCL
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FP8LM_EINVAL, "comm_init: bad arguments (nranks=%d rank=%d)", nranks, rank);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  auto* c = new fp8lm_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(FP8LM_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return FP8LM_OK;
#else
  (void)nranks; (void)rank; (void)id; (void)out;
  return fail(FP8LM_EUNSUPPORTED, "built without NCCL");
#endif
}

int fp8lm_comm_attach(void* nccl_comm, int32_t nranks, int32_t rank, fp8lm_comm** out) {
#ifdef FP8LM_WITH_NCCL
  if (!nccl_comm || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(FP8LM_EINVAL, "comm_attach: bad arguments (nranks=%d rank=%d)", nranks, rank);
  ncclComm_t c = static_cast<ncclComm_t>(nccl_comm);
  int cnt = -1, rk = -1;
  NCCL_TRY(ncclCommCount(c, &cnt));
  NCCL_TRY(ncclCommUserRank(c, &rk));
  if (cnt != nranks || rk != rank)
    return fail(FP8LM_EINVAL, "comm_attach: communicator is rank %d of %d, expected %d of %d", rk, cnt,
                rank, nranks);
  auto* w = new fp8lm_comm();
  w->comm = c;
  w->nranks = nranks;
  w->rank = rank;
  w->owned = false;
  *out = w;
  return FP8LM_OK;
#else
  (void)nccl_comm; (void)nranks; (void)rank; (void)out;
  return fail(FP8LM_EUNSUPPORTED, "built without NCCL");
#endif
}

int fp8lm_commstats_metrics(const fp8lm_commstats* st, double* out3) {
  if (!st || !out3) return fail(FP8LM_EINVAL, "commstats_metrics: NULL");
  const double g = st->sig2, e = st->err2;
  if (e == 0.0) out3[0] = g > 0.0 ? HUGE_VAL : NAN;
  else out3[0] = g > 0.0 ? 10.0 * std::log10(g / e) : -HUGE_VAL;
  out3[1] = st->events ? (double)st->underflow / (double)st->events : 0.0;
  out3[2] = st->events ? (double)st->overflow / (double)st->events : 0.0;
  return FP8LM_OK;
}

int fp8lm_comm_destroy(fp8lm_comm* comm) {
  if (!comm) return FP8LM_OK;
#ifdef FP8LM_WITH_NCCL
  if (comm->comm && comm->owned) {
    ncclCommFinalize(comm->comm);
    ncclCommDestroy(comm->comm);
  }
#endif
  delete comm;
  return FP8LM_OK;
}

// ---------------------------------------------------------------- plan
int fp8lm_plan_create(int32_t T, const int64_t* numels, int32_t mode, int32_t nranks,
                      int32_t rank, fp8lm_plan** out) {
  if (!out) return fail(FP8LM_EINVAL, "plan_create: out is NULL");
  if (T < 0 || (T > 0 && !numels)) return fail(FP8LM_EINVAL, "plan_create: bad T / numels");
  if (mode < FP8LM_MODE_LOCAL || mode > FP8LM_MODE_ZERO)
    return fail(FP8LM_EINVAL, "plan_create: bad mode %d", mode);
  if (nranks < 1) return fail(FP8LM_EINVAL, "plan_create: nranks must be >= 1");
  if (mode == FP8LM_MODE_LOCAL && nranks != 1)
    return fail(FP8LM_EINVAL, "plan_create: mode LOCAL needs nranks == 1");
  if (mode == FP8LM_MODE_SIMULATED && nranks > FP8LM_MAX_SIM_RANKS)
    return fail(FP8LM_EINVAL, "plan_create: at most %d simulated ranks", FP8LM_MAX_SIM_RANKS);
  const bool peer = mode == FP8LM_MODE_P2P || mode == FP8LM_MODE_ZERO;
  const bool dist = mode == FP8LM_MODE_NCCL || peer;
  if (dist && (rank < 0 || rank >= nranks))
    return fail(FP8LM_EINVAL, "plan_create: rank %d out of range", rank);
  if (peer && (nranks < 2 || nranks > FP8LM_MAX_P2P_RANKS))
    return fail(FP8LM_EINVAL, "plan_create: modes P2P / ZERO need 2..%d ranks", FP8LM_MAX_P2P_RANKS);
  for (int t = 0; t < T; ++t)
    if (numels[t] < 0) return fail(FP8LM_EINVAL, "plan_create: numel[%d] < 0", t);

  auto* p = new fp8lm_plan();
  p->T = T;
  p->mode = mode;
  p->nranks = nranks;
  p->rank = dist ? rank : 0;
  if (nranks > 1) p->oneshot_raw_max_bytes = FP8LM_ONESHOT_RAW_PULL / ((int64_t)(nranks - 1) * 4);
  p->numel.assign(numels, numels + T);
  p->offset.resize(T);
  p->item_start.resize(T + 1);
  int64_t run = 0, items = 0;
  for (int t = 0; t < T; ++t) {
    p->offset[t] = run;
    run += round_up(p->numel[t], FP8LM_ALIGN_ELEMS);
    p->item_start[t] = items;
    items += (p->numel[t] + kChunk - 1) / kChunk;
  }
  p->item_start[T] = items;
  p->items.reserve(items);
  for (int t = 0; t < T; ++t)
    for (int64_t x = 0; x < p->numel[t]; x += kChunk)
      p->items.push_back(ShardItem{p->offset[t] + x, t, (int32_t)std::min<int64_t>(kChunk, p->numel[t] - x)});
  p->total = run;
  p->g8_bytes = run;
  if (dist) {
    // reduce-scatter shards: N contiguous byte ranges of the flat code buffer, each a
    // multiple of 64 bytes so that every shard item starts 16-byte aligned
    const int64_t N = nranks;
    p->shard = std::max<int64_t>(round_up((run + N - 1) / N, FP8LM_ALIGN_ELEMS), FP8LM_ALIGN_ELEMS);
    p->g8_bytes = p->shard * N;
    const int64_t lo = p->shard * p->rank, hi = lo + p->shard;
    for (int t = 0; t < T; ++t) {
      const int64_t a = std::max(lo, p->offset[t]);
      const int64_t b = std::min(hi, p->offset[t] + p->numel[t]);
      for (int64_t x = a; x < b; x += kChunk)
        p->shard_items.push_back(ShardItem{x, t, (int32_t)std::min<int64_t>(kChunk, b - x)});
    }
  }
  // workspace layout
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (size_t)round_up((int64_t)bytes, 256); return o; };
  const int nsim = mode == FP8LM_MODE_SIMULATED ? nranks : 1;
  p->off_numel = take(sizeof(int64_t) * std::max(T, 1));
  p->off_offset = take(sizeof(int64_t) * std::max(T, 1));
  p->off_item_start = take(sizeof(int64_t) * (T + 1));
  p->off_items = take(sizeof(ShardItem) * std::max<size_t>(p->items.size(), 1));
  p->off_shard_items = take(sizeof(ShardItem) * std::max<size_t>(p->shard_items.size(), 1));
  p->off_acc_amax = take(sizeof(uint32_t) * std::max(nsim * T, 1));
  p->off_acc_state = take(sizeof(uint32_t) * std::max(3 * T, 1));
  p->off_sat_part = take(sizeof(uint32_t) * std::max(T, 1));
  p->off_sat_acc = take(sizeof(uint32_t) * std::max(T, 1));
  p->off_ctr = take(sizeof(uint32_t) * kCtrWords);
  p->off_acc_end = off;
  if (mode == FP8LM_MODE_NCCL) {
    p->off_send = take((size_t)(p->shard * nranks));
    p->off_recv = take((size_t)(p->shard * nranks));
  }
  if (mode == FP8LM_MODE_SIMULATED) p->off_sim = take((size_t)(p->total * nranks));
  if (mode == FP8LM_MODE_ZERO) {
    // Alg. 1: whole tensors to owners; this rank keeps optimizer state only
    // for its own tensors, packed in a compact LOCAL sub-plan
    p->owner.resize(std::max(T, 1));
    std::vector<int64_t> load(nranks);
    fp8lm_zero_plan(T, numels, nranks, p->owner.data(), load.data());
    std::vector<int64_t> own_numel;
    for (int t = 0; t < T; ++t)
      if (p->owner[t] == p->rank) {
        p->own2full.push_back(t);
        p->own_gpos.push_back(p->offset[t]);
        own_numel.push_back(p->numel[t]);
      }
    int rc = fp8lm_plan_create((int32_t)own_numel.size(), own_numel.data(), FP8LM_MODE_LOCAL, 1, 0,
                               &p->own);
    if (rc) { delete p; return rc; }
    p->full2own_off.assign(std::max(T, 1), -1);
    for (size_t j = 0; j < p->own2full.size(); ++j) p->full2own_off[p->own2full[j]] = p->own->offset[j];
    // A3's push layout: every rank quantizes tensor t straight into slot `rank` of its
    // owner's window, in the owner's compact layout (the same Alg. 1 packing every rank
    // computes), so the owner reduce reads N local slots instead of pulling over NVLink
    std::vector<int64_t> qtot(nranks, 0), coff(std::max(T, 1), 0);
    for (int t = 0; t < T; ++t) {
      coff[t] = qtot[p->owner[t]];
      qtot[p->owner[t]] += round_up(p->numel[t], FP8LM_ALIGN_ELEMS);
    }
    if (qtot[p->rank] != p->own->total) { delete p; return fail(FP8LM_EINVAL, "plan_create: owned layout mismatch"); }
    p->push_base.assign(std::max(T, 1), 0);
    for (int t = 0; t < T; ++t) p->push_base[t] = (int64_t)p->rank * qtot[p->owner[t]] + coff[t] - p->offset[t];
    p->off_push_base = take(sizeof(int64_t) * std::max(T, 1));
    p->off_owner_of = take(sizeof(int32_t) * std::max(T, 1));
    const size_t To = std::max<size_t>(p->own2full.size(), 1);
    p->off_own_ws = take(p->own->ws_bytes);
    p->off_own_gpos = take(sizeof(int64_t) * To);
    p->off_own2full = take(sizeof(int32_t) * To);
    p->off_gsinv_own = take(sizeof(float) * To);
  }
  p->ws_bytes = off;
  *out = p;
  return FP8LM_OK;
}

int fp8lm_plan_destroy(fp8lm_plan* plan) {
  if (!plan) return FP8LM_OK;
  for (void* m : plan->mapped) cudaIpcCloseMemHandle(m);
  if (plan->win_send) cudaFree(plan->win_send);
  if (plan->win_g8) cudaFree(plan->win_g8);
  if (plan->win_pad) cudaFree(plan->win_pad);
  if (plan->win_w8) cudaFree(plan->win_w8);
  for (auto& g : plan->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
    if (g.log) adam_log_free(g.log);
  }
  if (plan->xs) cudaStreamDestroy(plan->xs);
  if (plan->gs) cudaStreamDestroy(plan->gs);
  if (plan->ev_q) cudaEventDestroy(plan->ev_q);
  if (plan->ev_x) cudaEventDestroy(plan->ev_x);
  if (plan->own) fp8lm_plan_destroy(plan->own);
  delete plan;
  return FP8LM_OK;
}

int32_t fp8lm_plan_owner(const fp8lm_plan* p, int32_t t) {
  if (!p || p->mode != FP8LM_MODE_ZERO || t < 0 || t >= p->T) return -1;
  return p->owner[t];
}
int64_t fp8lm_plan_owned_offset(const fp8lm_plan* p, int32_t t) {
  if (!p || p->mode != FP8LM_MODE_ZERO || t < 0 || t >= p->T) return -1;
  return p->full2own_off[t];
}
int64_t fp8lm_plan_owned_total(const fp8lm_plan* p) {
  return (p && p->mode == FP8LM_MODE_ZERO) ? p->own->total : -1;
}
int32_t fp8lm_plan_owned_count(const fp8lm_plan* p) {
  return (p && p->mode == FP8LM_MODE_ZERO) ? (int32_t)p->own2full.size() : -1;
}

// ---------------------------------------------------------------- mode P2P windows
// this rank's symmetric windows (send, g8, w8, pad), zeroed where a peer may read first
static int peer_alloc(fp8lm_plan* p) {
  const bool zero = p->mode == FP8LM_MODE_ZERO;
  // ZERO: N slots of this rank's compact (owned) layout, written by every rank's quantize
  size_t win = zero ? std::max<size_t>((size_t)p->nranks * p->own->total, 256) : (size_t)p->g8_bytes;
  if (!zero && p->T > 0 && p->g8_bytes <= kRawAllocMax) {   // the raw one-shot's two copies
    p->raw_off = (int64_t)round_up((int64_t)win, 256);
    p->raw_half = (int64_t)round_up(p->total * (int64_t)sizeof(float), 256);
    win = (size_t)(p->raw_off + 2 * p->raw_half);
  }
  p->pad_bytes = pad_bytes_for(p->nranks, p->T);
  CUDA_TRY(cudaMalloc(&p->win_send, win));
  CUDA_TRY(cudaMalloc(&p->win_g8, zero ? 256 : win));     // ZERO: the owner's g8 is compact
  CUDA_TRY(cudaMalloc(&p->win_w8, zero ? std::max<size_t>(p->total, 256) : 256));
  CUDA_TRY(cudaMalloc(&p->win_pad, p->pad_bytes));
  CUDA_TRY(cudaMemset(p->win_pad, 0, p->pad_bytes));
  CUDA_TRY(cudaMemset(p->win_send, 0, win));
  return FP8LM_OK;
}

static int peer_table_upload(fp8lm_plan* p, const PeerTable& tab) {
  CUDA_TRY(cudaMemcpy(reinterpret_cast<uint8_t*>(p->win_pad) + kPadTable, &tab, sizeof tab,
                      cudaMemcpyHostToDevice));
  p->dev.send = p->win_send;
  p->p2p_ready = true;
  return FP8LM_OK;
}

// ---------------------------------------------------------------- peer-wait watchdog
static uint32_t* g_report = nullptr;                 // host-mapped {hit, flag, epoch, seen}
static unsigned long long g_timeout_ns = 600ull * 1000000000ull;

static int watchdog_install() {
  if (!g_report) {
    void* h = nullptr;
    CUDA_TRY(cudaHostAlloc(&h, 16, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(h, 0, 16);
    g_report = static_cast<uint32_t*>(h);
  }
  uint32_t* dev = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), g_report, 0));
  CUDA_TRY(wait_watchdog_set_kernels(g_timeout_ns, dev));
  CUDA_TRY(wait_watchdog_set_sp(g_timeout_ns, dev));
  return FP8LM_OK;
}

int fp8lm_set_peer_timeout(double seconds) {
  if (!(seconds >= 0) || seconds > 1e9) return fail(FP8LM_EINVAL, "set_peer_timeout: bad seconds");
  g_timeout_ns = (unsigned long long)(seconds * 1e9);
  return watchdog_install();
}

int fp8lm_peer_timeout_report(uint32_t* out4) {
  if (!out4) return fail(FP8LM_EINVAL, "peer_timeout_report: NULL");
  for (int k = 0; k < 4; ++k) out4[k] = g_report ? reinterpret_cast<volatile uint32_t*>(g_report)[k] : 0u;
  return FP8LM_OK;
}

int fp8lm_peer_setup(fp8lm_plan* p, fp8lm_comm* comm, void* stream) {
  if (!p || (p->mode != FP8LM_MODE_P2P && p->mode != FP8LM_MODE_ZERO))
    return fail(FP8LM_EINVAL, "peer_setup: plan mode is not P2P / ZERO");
  if (!p->bound) return fail(FP8LM_EWORKSPACE, "peer_setup: plan not bound");
  if (p->p2p_ready) return FP8LM_OK;
#ifdef FP8LM_WITH_NCCL
  if (!comm || comm->nranks != p->nranks || comm->rank != p->rank)
    return fail(FP8LM_EINVAL, "peer_setup: communicator does not match the plan");
  const int N = p->nranks;
  int rc = watchdog_install();
  if (rc || (rc = peer_alloc(p))) return rc;
  struct Handles { cudaIpcMemHandle_t send, g8, pad, w8; };
  Handles mine;
  CUDA_TRY(cudaIpcGetMemHandle(&mine.send, p->win_send));
  CUDA_TRY(cudaIpcGetMemHandle(&mine.g8, p->win_g8));
  CUDA_TRY(cudaIpcGetMemHandle(&mine.pad, p->win_pad));
  CUDA_TRY(cudaIpcGetMemHandle(&mine.w8, p->win_w8));
  Handles* dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, sizeof(Handles) * N));
  CUDA_TRY(cudaMemcpy(dev + p->rank, &mine, sizeof(Handles), cudaMemcpyHostToDevice));
  cudaStream_t s = S(stream);
  NCCL_TRY(ncclAllGather(dev + p->rank, dev, sizeof(Handles), ncclUint8, comm->comm, s));
  std::vector<Handles> all(N);
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaMemcpy(all.data(), dev, sizeof(Handles) * N, cudaMemcpyDeviceToHost));
  cudaFree(dev);
  PeerTable tab{};
  for (int q = 0; q < N; ++q) {
    if (q == p->rank) {
      tab.send[q] = p->win_send;
      tab.g8[q] = p->win_g8;
      tab.pad[q] = p->win_pad;
      tab.w8[q] = p->win_w8;
      continue;
    }
    void *ps = nullptr, *pg = nullptr, *pp = nullptr, *pw = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ps, all[q].send, cudaIpcMemLazyEnablePeerAccess));
    p->mapped.push_back(ps);
    CUDA_TRY(cudaIpcOpenMemHandle(&pg, all[q].g8, cudaIpcMemLazyEnablePeerAccess));
    p->mapped.push_back(pg);
    CUDA_TRY(cudaIpcOpenMemHandle(&pp, all[q].pad, cudaIpcMemLazyEnablePeerAccess));
    p->mapped.push_back(pp);
    CUDA_TRY(cudaIpcOpenMemHandle(&pw, all[q].w8, cudaIpcMemLazyEnablePeerAccess));
    p->mapped.push_back(pw);
    tab.send[q] = static_cast<uint8_t*>(ps);
    tab.g8[q] = static_cast<uint8_t*>(pg);
    tab.pad[q] = static_cast<uint32_t*>(pp);
    tab.w8[q] = static_cast<uint8_t*>(pw);
  }
  // (every peer zeroed its pad before contributing its handles to the all-gather above,
  // so no signal can land in an uninitialised pad)
  return peer_table_upload(p, tab);
#else
  (void)comm; (void)stream;
  return fail(FP8LM_EUNSUPPORTED, "built without NCCL");
#endif
}

int fp8lm_peer_setup_loopback(fp8lm_plan* const* plans, int32_t n, void* stream) {
  (void)stream;
  if (!plans || n < 2 || n > FP8LM_MAX_P2P_RANKS)
    return fail(FP8LM_EINVAL, "peer_setup_loopback: need 2..%d plans", FP8LM_MAX_P2P_RANKS);
  for (int r = 0; r < n; ++r) {
    const fp8lm_plan* p = plans[r];
    if (!p || (p->mode != FP8LM_MODE_P2P && p->mode != FP8LM_MODE_ZERO) || p->mode != plans[0]->mode)
      return fail(FP8LM_EINVAL, "peer_setup_loopback: plan %d is not P2P / ZERO like plan 0", r);
    if (!p->bound) return fail(FP8LM_EWORKSPACE, "peer_setup_loopback: plan %d not bound", r);
    if (p->p2p_ready) return fail(FP8LM_EINVAL, "peer_setup_loopback: plan %d already set up", r);
    if (p->nranks != n || p->rank != r)
      return fail(FP8LM_EINVAL, "peer_setup_loopback: plan %d has rank %d of %d", r, p->rank, p->nranks);
    if (p->numel != plans[0]->numel) return fail(FP8LM_EINVAL, "peer_setup_loopback: plan %d differs", r);
  }
  int rc = watchdog_install();
  if (rc) return rc;
  CUDA_TRY(preload_kernels());
  PeerTable tab{};
  for (int r = 0; r < n; ++r) {
    if ((rc = peer_alloc(plans[r]))) return rc;
    tab.send[r] = plans[r]->win_send;
    tab.g8[r] = plans[r]->win_g8;
    tab.pad[r] = plans[r]->win_pad;
    tab.w8[r] = plans[r]->win_w8;
  }
  // half the SMs per rank's kernel: with the split step two kernels of a rank (its stream
  // and its exchange stream) can be in flight
  const int ctas = std::max(1, num_sms() / (2 * n));
  for (int r = 0; r < n; ++r) {
    plans[r]->loopback_ctas = ctas;
    if (plans[r]->own) plans[r]->own->loopback_ctas = ctas;
    if ((rc = peer_table_upload(plans[r], tab))) return rc;
  }
  return FP8LM_OK;
}

uint8_t* fp8lm_peer_g8(const fp8lm_plan* p) {
  return (p && p->p2p_ready && p->mode == FP8LM_MODE_P2P) ? p->win_g8 : nullptr;
}
uint8_t* fp8lm_peer_w8(const fp8lm_plan* p) {
  return (p && p->p2p_ready && p->mode == FP8LM_MODE_ZERO) ? p->win_w8 : nullptr;
}
float* fp8lm_peer_w8_scalars(const fp8lm_plan* p) {
  if (!(p && p->p2p_ready && p->mode == FP8LM_MODE_ZERO)) return nullptr;
  return reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(p->win_pad) + kPadData +
                                  (size_t)p->nranks * p->T * 8);
}

int fp8lm_plan_set_oneshot(fp8lm_plan* p, int64_t max_bytes) {
  if (!p || max_bytes < 0) return fail(FP8LM_EINVAL, "plan_set_oneshot: bad arguments");
  p->oneshot_max_bytes = max_bytes;
  return FP8LM_OK;
}
int fp8lm_plan_set_oneshot_raw(fp8lm_plan* p, int64_t max_bytes) {
  if (!p || max_bytes < 0) return fail(FP8LM_EINVAL, "plan_set_oneshot_raw: bad arguments");
  p->oneshot_raw_max_bytes = max_bytes;
  return FP8LM_OK;
}

int64_t fp8lm_plan_offset(const fp8lm_plan* p, int32_t t) {
  if (!p || t < 0 || t >= p->T) return -1;
  return p->offset[t];
}
int64_t fp8lm_plan_total(const fp8lm_plan* p) { return p ? p->total : -1; }
int64_t fp8lm_plan_g8_bytes(const fp8lm_plan* p) { return p ? p->g8_bytes : -1; }
int64_t fp8lm_plan_shard_bytes(const fp8lm_plan* p) { return p ? p->shard : -1; }
int64_t fp8lm_plan_shard_begin(const fp8lm_plan* p, int32_t rank) {
  if (!p || rank < 0 || rank >= p->nranks) return -1;
  return p->shard * rank;
}
size_t fp8lm_plan_workspace_bytes(const fp8lm_plan* p) { return p ? p->ws_bytes : 0; }

int fp8lm_plan_bind(fp8lm_plan* p, void* ws, size_t ws_bytes, void* stream) {
  if (!p) return fail(FP8LM_EINVAL, "plan_bind: plan is NULL");
  if (!ws || ws_bytes < p->ws_bytes || !aligned(ws, 256))
    return fail(FP8LM_EWORKSPACE, "plan_bind: need %zu bytes, 256-aligned (got %zu at %p)",
                p->ws_bytes, ws_bytes, ws);
  uint8_t* b = static_cast<uint8_t*>(ws);
  cudaStream_t s = S(stream);
  if (p->T > 0) {
    CUDA_TRY(cudaMemcpyAsync(b + p->off_numel, p->numel.data(), sizeof(int64_t) * p->T, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(b + p->off_offset, p->offset.data(), sizeof(int64_t) * p->T, cudaMemcpyHostToDevice, s));
  }
  CUDA_TRY(cudaMemcpyAsync(b + p->off_item_start, p->item_start.data(), sizeof(int64_t) * (p->T + 1), cudaMemcpyHostToDevice, s));
  if (!p->items.empty())
    CUDA_TRY(cudaMemcpyAsync(b + p->off_items, p->items.data(), sizeof(ShardItem) * p->items.size(), cudaMemcpyHostToDevice, s));
  if (!p->shard_items.empty())
    CUDA_TRY(cudaMemcpyAsync(b + p->off_shard_items, p->shard_items.data(), sizeof(ShardItem) * p->shard_items.size(), cudaMemcpyHostToDevice, s));
  // accumulators (acc_amax, acc_state, sat_part, sat_acc, counters: consecutive) zero at rest
  CUDA_TRY(cudaMemsetAsync(b + p->off_acc_amax, 0, p->off_acc_end - p->off_acc_amax, s));
  CUDA_TRY(cudaStreamSynchronize(s));   // host tables are pageable: finish before returning
  DevPlan& d = p->dev;
  d.T = p->T;
  d.nranks = p->nranks;
  d.total = p->total;
  d.n_items = p->item_start[p->T];
  d.numel = reinterpret_cast<const int64_t*>(b + p->off_numel);
  d.offset = reinterpret_cast<const int64_t*>(b + p->off_offset);
  d.item_start = reinterpret_cast<const int64_t*>(b + p->off_item_start);
  d.items = reinterpret_cast<const ShardItem*>(b + p->off_items);
  d.shard_items = reinterpret_cast<const ShardItem*>(b + p->off_shard_items);
  d.n_shard_items = (int64_t)p->shard_items.size();
  d.shard = p->shard;
  d.acc_amax = reinterpret_cast<uint32_t*>(b + p->off_acc_amax);
  d.acc_state = reinterpret_cast<uint32_t*>(b + p->off_acc_state);
  d.sat_part = reinterpret_cast<uint32_t*>(b + p->off_sat_part);
  d.send = p->mode == FP8LM_MODE_NCCL ? b + p->off_send : nullptr;
  d.recv = p->mode == FP8LM_MODE_NCCL ? b + p->off_recv : nullptr;
  d.sim_codes = p->mode == FP8LM_MODE_SIMULATED ? b + p->off_sim : nullptr;
  d.sat_acc = reinterpret_cast<uint32_t*>(b + p->off_sat_acc);
  d.counters = reinterpret_cast<uint32_t*>(b + p->off_ctr);
  d.T_own = 0;
  if (p->mode == FP8LM_MODE_ZERO) {
    int rc = fp8lm_plan_bind(p->own, b + p->off_own_ws, p->own->ws_bytes, stream);
    if (rc) return rc;
    const size_t To = p->own2full.size();
    if (To) {
      CUDA_TRY(cudaMemcpyAsync(b + p->off_own_gpos, p->own_gpos.data(), sizeof(int64_t) * To, cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(b + p->off_own2full, p->own2full.data(), sizeof(int32_t) * To, cudaMemcpyHostToDevice, s));
    }
    if (p->T > 0) {
      CUDA_TRY(cudaMemcpyAsync(b + p->off_push_base, p->push_base.data(), sizeof(int64_t) * p->T,
                               cudaMemcpyHostToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(b + p->off_owner_of, p->owner.data(), sizeof(int32_t) * p->T,
                               cudaMemcpyHostToDevice, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    d.push_base = reinterpret_cast<const int64_t*>(b + p->off_push_base);
    d.owner_of = reinterpret_cast<const int32_t*>(b + p->off_owner_of);
    d.own_slot = p->own->total;
    d.T_own = (int32_t)To;
    d.own_gpos = reinterpret_cast<const int64_t*>(b + p->off_own_gpos);
    d.own2full = reinterpret_cast<const int32_t*>(b + p->off_own2full);
    d.gsinv_own = reinterpret_cast<float*>(b + p->off_gsinv_own);
  }
  p->ws = ws;
  p->bound = true;
  return FP8LM_OK;
}

// ---------------------------------------------------------------- shared checks
static int check_plan(const fp8lm_plan* p, const fp8lm_comm* comm, const char* who) {
  if (!p) return fail(FP8LM_EINVAL, "%s: plan is NULL", who);
  if (!p->bound) return fail(FP8LM_EWORKSPACE, "%s: plan not bound to a workspace", who);
  if (p->mode == FP8LM_MODE_NCCL) {
    if (!comm) return fail(FP8LM_EINVAL, "%s: mode NCCL needs a communicator", who);
    if (comm->nranks != p->nranks || comm->rank != p->rank)
      return fail(FP8LM_EINVAL, "%s: communicator (%d/%d) does not match plan (%d/%d)", who,
                  comm->rank, comm->nranks, p->rank, p->nranks);
  } else if (p->mode == FP8LM_MODE_P2P || p->mode == FP8LM_MODE_ZERO) {
    if (!p->p2p_ready) return fail(FP8LM_EINVAL, "%s: modes P2P / ZERO need fp8lm_peer_setup first", who);
  } else if (comm) {
    return fail(FP8LM_EINVAL, "%s: communicator given but plan mode is not NCCL", who);
  }
  return FP8LM_OK;
}

static P2PArgs p2p_args(const fp8lm_plan* p) {
  P2PArgs x;
  x.tab = reinterpret_cast<const PeerTable*>(reinterpret_cast<uint8_t*>(p->win_pad) + kPadTable);
  x.pad = p->win_pad;
  x.rank = p->rank;
  x.nranks = p->nranks;
  return x;
}

// resolve the gradient source(s): SIMULATED -> host array of nranks device pointers
static int grad_sources(const fp8lm_plan* p, const void* grads, int32_t dtype,
                        const void** srcs, int* nsrc, const char* who) {
  if (dtype != FP8LM_F32 && dtype != FP8LM_BF16)
    return fail(FP8LM_EUNSUPPORTED, "%s: gradients must be F32 or BF16", who);
  if (!grads) return fail(FP8LM_EINVAL, "%s: grads is NULL", who);
  if (p->mode == FP8LM_MODE_SIMULATED) {
    const void* const* arr = static_cast<const void* const*>(grads);
    *nsrc = p->nranks;
    for (int r = 0; r < p->nranks; ++r) srcs[r] = arr[r];
  } else {
    *nsrc = 1;
    srcs[0] = grads;
  }
  for (int r = 0; r < *nsrc; ++r)
    if (!srcs[r] || !aligned(srcs[r], 256))
      return fail(FP8LM_EINVAL, "%s: gradient buffer %d is NULL or not 256-byte aligned", who, r);
  return FP8LM_OK;
}

// ---------------------------------------------------------------- (1) fp8_quantize
int fp8lm_quantize(const void* src, int32_t src_dtype, int64_t n, int32_t fmt, void* dst,
                   float* scale, float* scale_inv, float* amax, int32_t jit, uint32_t* sat_count,
                   void* stream) {
  if (n < 0) return fail(FP8LM_EINVAL, "quantize: n < 0");
  if (src_dtype != FP8LM_F32 && src_dtype != FP8LM_BF16)
    return fail(FP8LM_EUNSUPPORTED, "quantize: src dtype must be F32 or BF16");
  if (fmt != FP8LM_E4M3 && fmt != FP8LM_E5M2 && fmt != FP8LM_F16)
    return fail(FP8LM_EINVAL, "quantize: fmt must be E4M3, E5M2 or F16");
  if (n > 0 && (!src || !dst)) return fail(FP8LM_EINVAL, "quantize: NULL src/dst");
  if (!scale || (jit && (!scale_inv || !amax)))
    return fail(FP8LM_EINVAL, "quantize: NULL scale pointers");
  CUDA_TRY(launch_q_single(src, src_dtype, n, fmt, dst, scale, scale_inv, amax, jit, sat_count, S(stream)));
  return FP8LM_OK;
}

int fp8lm_dequantize(const void* codes, int32_t fmt, int64_t n, const float* scale_inv,
                     float* dst, void* stream) {
  if (n < 0) return fail(FP8LM_EINVAL, "dequantize: n < 0");
  if (fmt != FP8LM_E4M3 && fmt != FP8LM_E5M2 && fmt != FP8LM_F16)
    return fail(FP8LM_EINVAL, "dequantize: fmt must be E4M3, E5M2 or F16");
  if (n > 0 && (!codes || !dst || !scale_inv)) return fail(FP8LM_EINVAL, "dequantize: NULL pointer");
  CUDA_TRY(launch_dq_single(codes, fmt, n, scale_inv, dst, S(stream)));
  return FP8LM_OK;
}

// ---------------------------------------------------------------- (8) FP8 SP converter (f4)
struct fp8lm_sp {
  int32_t nranks = 1, rank = 0;
  int64_t max_elems = 0;
  uint8_t* recv = nullptr;
  uint8_t* send = nullptr;
  uint32_t* pad = nullptr;
  uint32_t* scratch = nullptr;
  std::vector<void*> mapped;
  uint32_t epoch = 0;
};

int fp8lm_sp_create(fp8lm_comm* comm, int64_t max_elems, void* stream, fp8lm_sp** out) {
  if (!out) return fail(FP8LM_EINVAL, "sp_create: NULL out");
  *out = nullptr;
  if (max_elems < 0) return fail(FP8LM_EINVAL, "sp_create: max_elems < 0");
  const int N = comm ? comm->nranks : 1;
  const int rank = comm ? comm->rank : 0;
  if (N > FP8LM_MAX_P2P_RANKS) return fail(FP8LM_EINVAL, "sp_create: at most %d ranks", FP8LM_MAX_P2P_RANKS);
  auto* sp = new fp8lm_sp();
  sp->nranks = N;
  sp->rank = rank;
  sp->max_elems = max_elems;
  const size_t win = (size_t)std::max<int64_t>(round_up(max_elems, 256), 256);
  auto bail = [&](int rc) { fp8lm_sp_destroy(sp); return rc; };
  if (cudaMalloc(&sp->recv, win) != cudaSuccess || cudaMalloc(&sp->send, win) != cudaSuccess ||
      cudaMalloc(&sp->pad, kSpPadBytes) != cudaSuccess ||
      cudaMalloc(&sp->scratch, sizeof(uint32_t) * kSpScrWords) != cudaSuccess)
    return bail(fail(FP8LM_ECUDA, "sp_create: cudaMalloc failed"));
  if (cudaMemset(sp->pad, 0, kSpPadBytes) != cudaSuccess ||
      cudaMemset(sp->scratch, 0, sizeof(uint32_t) * kSpScrWords) != cudaSuccess)
    return bail(fail(FP8LM_ECUDA, "sp_create: cudaMemset failed"));
  SpTable tab{};
  tab.recv[rank] = sp->recv;
  tab.send[rank] = sp->send;
  tab.pad[rank] = sp->pad;
  if (N > 1) {
#ifdef FP8LM_WITH_NCCL
    if (int rc = watchdog_install()) return bail(rc);
    struct Handles { cudaIpcMemHandle_t recv, send, pad; };
    Handles mine;
    if (cudaIpcGetMemHandle(&mine.recv, sp->recv) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine.send, sp->send) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine.pad, sp->pad) != cudaSuccess)
      return bail(fail(FP8LM_ECUDA, "sp_create: cudaIpcGetMemHandle failed"));
    Handles* dev = nullptr;
    if (cudaMalloc(&dev, sizeof(Handles) * N) != cudaSuccess)
      return bail(fail(FP8LM_ECUDA, "sp_create: cudaMalloc failed"));
    cudaMemcpy(dev + rank, &mine, sizeof(Handles), cudaMemcpyHostToDevice);
    cudaStream_t s = S(stream);
    const ncclResult_t nr = ncclAllGather(dev + rank, dev, sizeof(Handles), ncclUint8, comm->comm, s);
    std::vector<Handles> all(N);
    const cudaError_t ce = cudaStreamSynchronize(s);
    cudaMemcpy(all.data(), dev, sizeof(Handles) * N, cudaMemcpyDeviceToHost);
    cudaFree(dev);
    if (nr != ncclSuccess || ce != cudaSuccess) return bail(fail(FP8LM_ENCCL, "sp_create: handle exchange failed"));
    for (int q = 0; q < N; ++q) {
      if (q == rank) continue;
      void *pr = nullptr, *ps = nullptr, *pp = nullptr;
      if (cudaIpcOpenMemHandle(&pr, all[q].recv, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
          cudaIpcOpenMemHandle(&ps, all[q].send, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
          cudaIpcOpenMemHandle(&pp, all[q].pad, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return bail(fail(FP8LM_ECUDA, "sp_create: cudaIpcOpenMemHandle failed"));
      sp->mapped.push_back(pr);
      sp->mapped.push_back(ps);
      sp->mapped.push_back(pp);
      tab.recv[q] = static_cast<uint8_t*>(pr);
      tab.send[q] = static_cast<uint8_t*>(ps);
      tab.pad[q] = static_cast<uint32_t*>(pp);
    }
#else
    (void)stream;
    return bail(fail(FP8LM_EUNSUPPORTED, "sp_create: built without NCCL"));
#endif
  }
  if (cudaMemcpy(reinterpret_cast<uint8_t*>(sp->pad) + kSpPadTable, &tab, sizeof tab,
                 cudaMemcpyHostToDevice) != cudaSuccess)
    return bail(fail(FP8LM_ECUDA, "sp_create: table upload failed"));
  *out = sp;
  return FP8LM_OK;
}

int fp8lm_sp_destroy(fp8lm_sp* sp) {
  if (!sp) return FP8LM_OK;
  for (void* m : sp->mapped) cudaIpcCloseMemHandle(m);
  if (sp->recv) cudaFree(sp->recv);
  if (sp->send) cudaFree(sp->send);
  if (sp->pad) cudaFree(sp->pad);
  if (sp->scratch) cudaFree(sp->scratch);
  delete sp;
  return FP8LM_OK;
}

static int sp_check(const fp8lm_sp* sp, const void* src, int32_t dtype, int64_t m, const void* out,
                    int32_t out_dtype, const char* who) {
  if (!sp) return fail(FP8LM_EINVAL, "%s: sp is NULL", who);
  if (m < 0) return fail(FP8LM_EINVAL, "%s: m < 0", who);
  if (m * sp->nranks > sp->max_elems)
    return fail(FP8LM_EINVAL, "%s: N*m = %lld exceeds max_elems %lld", who, (long long)(m * sp->nranks),
                (long long)sp->max_elems);
  if (dtype != FP8LM_F32 && dtype != FP8LM_BF16) return fail(FP8LM_EUNSUPPORTED, "%s: input must be F32 or BF16", who);
  if (out && out_dtype != FP8LM_F32 && out_dtype != FP8LM_BF16)
    return fail(FP8LM_EUNSUPPORTED, "%s: output must be F32 or BF16", who);
  if (m > 0 && !src) return fail(FP8LM_EINVAL, "%s: NULL input", who);
  return FP8LM_OK;
}

int fp8lm_sp_allgather(fp8lm_sp* sp, const void* x, int32_t x_dtype, int64_t m, uint8_t* codes_out,
                       void* out, int32_t out_dtype, float* scale_out, void* stream) {
  int rc = sp_check(sp, x, x_dtype, m, out, out_dtype, "sp_allgather");
  if (rc) return rc;
  SpArgs a{sp->pad, sp->scratch, sp->rank, sp->nranks, ++sp->epoch, false};
  a.vec = m % 16 == 0 && aligned(x, 32) && (!codes_out || aligned(codes_out, 16)) &&
          (!out || aligned(out, 16));
  CUDA_TRY(launch_sp_allgather(x, x_dtype, m, codes_out, out, out_dtype, scale_out, a, S(stream)));
  return FP8LM_OK;
}

int fp8lm_sp_reduce_scatter(fp8lm_sp* sp, const void* dy, int32_t dtype, int64_t m, void* out,
                            int32_t out_dtype, float* scale_out, void* stream) {
  int rc = sp_check(sp, dy, dtype, m, out, out_dtype, "sp_reduce_scatter");
  if (rc) return rc;
  if (m > 0 && !out) return fail(FP8LM_EINVAL, "sp_reduce_scatter: NULL out");
  SpArgs a{sp->pad, sp->scratch, sp->rank, sp->nranks, ++sp->epoch, false};
  a.vec = m % 16 == 0 && aligned(dy, 32) && aligned(out, 16);
  CUDA_TRY(launch_sp_reduce_scatter(dy, dtype, m, out, out_dtype, scale_out, a, S(stream)));
  return FP8LM_OK;
}

// ---------------------------------------------------------------- (7) strategies (f3)
static_assert(sizeof(fp8lm_commstats) == 88, "fp8lm_commstats layout (the binding unpacks 88 bytes)");
static_assert(offsetof(fp8lm_commstats, sat) == 40 && offsetof(fp8lm_commstats, amax) == 48 &&
              offsetof(fp8lm_commstats, scratch) == 72, "fp8lm_commstats layout");
int fp8lm_allreduce_strategy(int32_t strategy, const float* grads, int32_t nranks, int64_t n,
                             float* mu, uint8_t* codes, fp8lm_commstats* stats, void* stream) {
  if (strategy < FP8LM_STRATEGY_PRE || strategy > FP8LM_STRATEGY_AUTO)
    return fail(FP8LM_EINVAL, "allreduce_strategy: bad strategy %d", strategy);
  if (nranks < 1) return fail(FP8LM_EINVAL, "allreduce_strategy: nranks must be >= 1");
  if (n < 0) return fail(FP8LM_EINVAL, "allreduce_strategy: n < 0");
  if (!stats) return fail(FP8LM_EINVAL, "allreduce_strategy: NULL stats");
  if (n > 0 && !grads) return fail(FP8LM_EINVAL, "allreduce_strategy: NULL grads");
  if (strategy == FP8LM_STRATEGY_AUTO && !mu) return fail(FP8LM_EINVAL, "allreduce_strategy: AUTO needs mu");
  if (!aligned(stats, 8)) return fail(FP8LM_EINVAL, "allreduce_strategy: stats must be 8-byte aligned");
  CUDA_TRY(launch_allreduce_strategy(strategy, grads, nranks, n, mu, codes, stats, S(stream)));
  return FP8LM_OK;
}

// ---------------------------------------------------------------- (2) amax_scale_sync
int fp8lm_amax_scale_sync(fp8lm_plan* p, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                          const float* mu, float* amax_out, float* s_g, int32_t* skip,
                          void* stream) {
  const LaunchScope ls_(p);   // loopback plans: capped grids
  int rc = check_plan(p, comm, "amax_scale_sync");
  if (rc) return rc;
  const void* srcs[FP8LM_MAX_SIM_RANKS];
  int nsrc = 0;
  if (p->T > 0 && (rc = grad_sources(p, grads, src_dtype, srcs, &nsrc, "amax_scale_sync"))) return rc;
  if (!mu || !amax_out || !s_g || !skip) return fail(FP8LM_EINVAL, "amax_scale_sync: NULL output");
  cudaStream_t s = S(stream);
  if (p->T == 0) {
    CUDA_TRY(cudaMemsetAsync(skip, 0, sizeof(int32_t), s));
    return FP8LM_OK;
  }
  const bool nccl = p->mode == FP8LM_MODE_NCCL;
  if (p->mode == FP8LM_MODE_P2P || p->mode == FP8LM_MODE_ZERO) {
    // A1 amax; its last CTA exchanges the local scales through the peers' pads (Eq. 4)
    const P2PArgs x = p2p_args(p);
    CUDA_TRY(launch_amax(p->dev, srcs, nsrc, src_dtype, mu, amax_out, s_g, skip, true, &x, s));
    return FP8LM_OK;
  }
  // A1 amax; its last CTA computes the scales (A2) and, without an exchange, s_g + skip
  CUDA_TRY(launch_amax(p->dev, srcs, nsrc, src_dtype, mu, amax_out, s_g, skip, !nccl, nullptr, s));
  if (nccl) {
#ifdef FP8LM_WITH_NCCL
    // Eq. 4: s'_g = min(s'_1, ..., s'_N) — T floats over NVLink
    {
      ProfScope ps_(P_NCCL_MIN, s);
      NCCL_TRY(ncclAllReduce(s_g, s_g, (size_t)p->T, ncclFloat32, ncclMin, comm->comm, s));
    }
    CUDA_TRY(launch_scale_fix(p->dev, s_g, skip, s));
#else
    return fail(FP8LM_EUNSUPPORTED, "built without NCCL");
#endif
  }
  return FP8LM_OK;
}

// ---------------------------------------------------------------- (3) fp8_grad_allreduce
int fp8lm_grad_allreduce(fp8lm_plan* p, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                         const float* s_g, const int32_t* skip, uint8_t* g8, float* g_scale,
                         float* g_scale_inv, uint32_t* sat, float* mu, void* stream) {
  const LaunchScope ls_(p);   // loopback plans: capped grids
  int rc = check_plan(p, comm, "grad_allreduce");
  if (rc) return rc;
  const void* srcs[FP8LM_MAX_SIM_RANKS];
  int nsrc = 0;
  if (p->T > 0 && (rc = grad_sources(p, grads, src_dtype, srcs, &nsrc, "grad_allreduce"))) return rc;
  if (!s_g || !skip || !g_scale || !g_scale_inv || !sat || !mu)
    return fail(FP8LM_EINVAL, "grad_allreduce: NULL scalar array");
  if (p->T > 0 && (!g8 || !aligned(g8, 256)))
    return fail(FP8LM_EINVAL, "grad_allreduce: g8 NULL or not 256-byte aligned");
  cudaStream_t s = S(stream);
  if (p->T == 0) return FP8LM_OK;
  const DevPlan& d = p->dev;
  const TailArgs tail{p->nranks, skip, sat, g_scale, g_scale_inv, mu};
  if (p->mode == FP8LM_MODE_LOCAL) {
    // N = 1: the reduce-scatter / all-gather are the identity (A4, A5); quantize counts
    // saturation and its last CTA runs the Eq. 6 / mu tail
    uint8_t* dst[1] = {g8};
    CUDA_TRY(launch_quantize(d, srcs, dst, 1, src_dtype, s_g, &tail, s));
  } else if (p->mode == FP8LM_MODE_ZERO) {
    if (!p->p2p_ready) return fail(FP8LM_EINVAL, "grad_allreduce: mode ZERO needs fp8lm_peer_setup first");
    CUDA_TRY(launch_quantize_push(d, p2p_args(p), srcs[0], src_dtype, s_g, s));
    // each owner reduces its whole tensors from the N slots of its window
    CUDA_TRY(launch_reduce_owner(d, p->own->dev, p2p_args(p), g8, s_g, tail, s));
  } else if (p->mode == FP8LM_MODE_P2P) {
    if (g8 != p->win_g8) return fail(FP8LM_EINVAL, "grad_allreduce: mode P2P needs g8 == fp8lm_peer_g8(plan)");
    if (p->g8_bytes <= p->oneshot_max_bytes) {   // small message: one kernel, one handshake
      CUDA_TRY(launch_oneshot(d, p2p_args(p), srcs[0], src_dtype, g8, s_g, tail, s));
      return FP8LM_OK;
    }
    // A3 pushes every code group into its shard owner's window slot (the reduce-scatter's
    // NVLink transfer rides on the quantize pass), then A4 + A5 in one kernel
    P2PArgs x = p2p_args(p);
    x.slots = 1;
    CUDA_TRY(launch_quantize_push(d, x, srcs[0], src_dtype, s_g, s, /*shard_slots=*/true));
    CUDA_TRY(launch_reduce_p2p(d, x, g8, s_g, tail, s));
  } else if (p->mode == FP8LM_MODE_SIMULATED) {
    uint8_t* dst[FP8LM_MAX_SIM_RANKS];
    for (int r = 0; r < nsrc; ++r) dst[r] = d.sim_codes + (int64_t)r * p->total;
    CUDA_TRY(launch_quantize(d, srcs, dst, nsrc, src_dtype, s_g, nullptr, s));
    CUDA_TRY(launch_reduce(d, d.sim_codes, p->total, nsrc, 0, false, g8, s_g, &tail, s));
  } else {
#ifdef FP8LM_WITH_NCCL
    const int64_t S_ = p->shard;
    uint8_t* dst[1] = {d.send};
    CUDA_TRY(launch_quantize(d, srcs, dst, 1, src_dtype, s_g, nullptr, s));
    // reduce-scatter transport: chunk j of the flat code buffer goes to rank j
    {
      ProfScope ps_(P_NCCL_A2A, s);
      NCCL_TRY(ncclAlltoAll(d.send, d.recv, (size_t)S_, ncclUint8, comm->comm, s));
    }
    // own shard: rank-order FP32 sum, requantize, per-shard saturation counts (sat_part
    // was zeroed by this step's amax epilogue)
    CUDA_TRY(launch_reduce(d, d.recv, S_, p->nranks, S_ * p->rank, true, g8, s_g, nullptr, s));
    // all-gather of the reduced shards (in place) + global saturation counts
    {
      ProfScope ps_(P_NCCL_AG_SUM, s);
      NCCL_TRY(ncclGroupStart());
      NCCL_TRY(ncclAllGather(g8 + S_ * p->rank, g8, (size_t)S_, ncclUint8, comm->comm, s));
      NCCL_TRY(ncclAllReduce(d.sat_part, sat, (size_t)p->T, ncclUint32, ncclSum, comm->comm, s));
      NCCL_TRY(ncclGroupEnd());
    }
    CUDA_TRY(launch_allreduce_finalize(d, s_g, tail, s));
#else
    return fail(FP8LM_EUNSUPPORTED, "built without NCCL");
#endif
  }
  return FP8LM_OK;
}

// ---------------------------------------------------------------- (2) + (3) in one call
int fp8lm_allreduce_jit(fp8lm_plan* p, fp8lm_comm* comm, const void* grads, int32_t src_dtype, float* mu,
                        float* amax_out, float* s_g, int32_t* skip, uint8_t* g8, float* g_scale,
                        float* g_scale_inv, uint32_t* sat, void* stream) {
  const LaunchScope ls_(p);
  int rc = check_plan(p, comm, "allreduce_jit");
  if (rc) return rc;
  if (p->mode == FP8LM_MODE_P2P && p->T > 0 && p->g8_bytes <= p->oneshot_max_bytes) {
    const void* srcs[1];
    int nsrc = 0;
    if ((rc = grad_sources(p, grads, src_dtype, srcs, &nsrc, "allreduce_jit"))) return rc;
    if (!mu || !amax_out || !s_g || !skip || !g_scale || !g_scale_inv || !sat)
      return fail(FP8LM_EINVAL, "allreduce_jit: NULL output");
    if (g8 != p->win_g8) return fail(FP8LM_EINVAL, "allreduce_jit: mode P2P needs g8 == fp8lm_peer_g8(plan)");
    const TailArgs tail{p->nranks, skip, sat, g_scale, g_scale_inv, mu};
    if (p->raw_half > 0 && p->g8_bytes <= p->oneshot_raw_max_bytes)   // one handshake
      CUDA_TRY(launch_oneshot_raw(p->dev, p2p_args(p), srcs[0], src_dtype, mu, amax_out, s_g, skip, g8, tail,
                                  p->raw_off, p->raw_half, S(stream)));
    else
      CUDA_TRY(launch_oneshot_full(p->dev, p2p_args(p), srcs[0], src_dtype, mu, amax_out, s_g, skip, g8, tail,
                                   S(stream)));
    return FP8LM_OK;
  }
  if ((rc = fp8lm_amax_scale_sync(p, comm, grads, src_dtype, mu, amax_out, s_g, skip, stream))) return rc;
  return fp8lm_grad_allreduce(p, comm, grads, src_dtype, s_g, skip, g8, g_scale, g_scale_inv, sat, mu, stream);
}

// ---------------------------------------------------------------- (4) fp8_adam_step
static int check_stensors(const fp8lm_plan* p, const fp8lm_stensors* x, const char* name,
                          const char* who) {
  if (!x) return fail(FP8LM_EINVAL, "%s: %s is NULL", who, name);
  if (!x->scale || !x->scale_inv || !x->amax)
    return fail(FP8LM_EINVAL, "%s: %s scalar arrays must be non-NULL", who, name);
  if (p->T > 0 && (!x->data || !aligned(x->data, 256)))
    return fail(FP8LM_EINVAL, "%s: %s.data NULL or not 256-byte aligned", who, name);
  return FP8LM_OK;
}

int fp8lm_adam_step(fp8lm_plan* p, const uint8_t* g8, const float* g_scale_inv,
                    const fp8lm_stensors* m1, const fp8lm_stensors* v,
                    const fp8lm_stensors* master, const fp8lm_stensors* w8,
                    const fp8lm_adam_hp* hp, const int32_t* skip, void* stream) {
  const LaunchScope ls_(p);   // loopback plans: capped grids
  if (!p) return fail(FP8LM_EINVAL, "adam_step: plan is NULL");
  if (!p->bound) return fail(FP8LM_EWORKSPACE, "adam_step: plan not bound");
  int rc;
  if ((rc = check_stensors(p, m1, "m1", "adam_step")) || (rc = check_stensors(p, v, "v", "adam_step")) ||
      (rc = check_stensors(p, master, "master", "adam_step")) || (rc = check_stensors(p, w8, "w8", "adam_step")))
    return rc;
  if (!hp || !skip || !g_scale_inv) return fail(FP8LM_EINVAL, "adam_step: NULL hp / skip / g_scale_inv");
  if (p->mode == FP8LM_MODE_ZERO) {
    // ZeRO: AdamW on the owned tensors (compact sub-plan), then the owners write w8 into
    // every rank's replicated copy
    if (!p->p2p_ready) return fail(FP8LM_EINVAL, "adam_step: mode ZERO needs fp8lm_peer_setup first");
    if (p->own->T > 0 && (!g8 || !aligned(g8, 256))) return fail(FP8LM_EINVAL, "adam_step: g8 NULL or misaligned");
    CUDA_TRY(launch_adam(p->own->dev, g8, p->dev.gsinv_own, *m1, *v, *master, *w8, *hp, skip, S(stream)));
    CUDA_TRY(launch_w8_bcast(p->dev, p->own->dev, p2p_args(p),
                             static_cast<const uint8_t*>(w8->data), *w8, S(stream)));
    return FP8LM_OK;
  }
  if (p->T > 0 && (!g8 || !aligned(g8, 256))) return fail(FP8LM_EINVAL, "adam_step: g8 NULL or misaligned");
  CUDA_TRY(launch_adam(p->dev, g8, g_scale_inv, *m1, *v, *master, *w8, *hp, skip, S(stream)));
  return FP8LM_OK;
}

int fp8lm_adam_step_delayed(fp8lm_plan* p, const uint8_t* g8, const float* g_scale_inv,
                            const fp8lm_stensors* m1, const fp8lm_stensors* v,
                            const fp8lm_stensors* master, const fp8lm_stensors* w8,
                            const fp8lm_adam_hp* hp, const int32_t* skip, float* w_hist,
                            int32_t hist_slot, void* stream) {
  const LaunchScope ls_(p);   // loopback plans: capped grids
  if (!p) return fail(FP8LM_EINVAL, "adam_step_delayed: plan is NULL");
  if (!p->bound) return fail(FP8LM_EWORKSPACE, "adam_step_delayed: plan not bound");
  int rc;
  if ((rc = check_stensors(p, m1, "m1", "adam_step_delayed")) ||
      (rc = check_stensors(p, v, "v", "adam_step_delayed")) ||
      (rc = check_stensors(p, master, "master", "adam_step_delayed")) ||
      (rc = check_stensors(p, w8, "w8", "adam_step_delayed")))
    return rc;
  if (!hp || !skip || !g_scale_inv || !w_hist)
    return fail(FP8LM_EINVAL, "adam_step_delayed: NULL hp / skip / g_scale_inv / w_hist");
  if (hist_slot < 0 || hist_slot >= 16) return fail(FP8LM_EINVAL, "adam_step_delayed: hist_slot not in [0, 16)");
  if (p->mode == FP8LM_MODE_ZERO) {
    if (!p->p2p_ready) return fail(FP8LM_EINVAL, "adam_step_delayed: mode ZERO needs fp8lm_peer_setup first");
    CUDA_TRY(launch_adam_delayed(p->own->dev, g8, p->dev.gsinv_own, *m1, *v, *master, *w8, *hp, skip,
                                 w_hist, hist_slot, S(stream)));
    CUDA_TRY(launch_w8_bcast(p->dev, p->own->dev, p2p_args(p),
                             static_cast<const uint8_t*>(w8->data), *w8, S(stream)));
    return FP8LM_OK;
  }
  if (p->T > 0 && (!g8 || !aligned(g8, 256))) return fail(FP8LM_EINVAL, "adam_step_delayed: g8 NULL or misaligned");
  CUDA_TRY(launch_adam_delayed(p->dev, g8, g_scale_inv, *m1, *v, *master, *w8, *hp, skip, w_hist,
                               hist_slot, S(stream)));
  return FP8LM_OK;
}

// ---------------------------------------------------------------- the whole step
// the exchange stream of a split step (phase 1 launches the exchange kernel there, phase 2
// makes the caller's stream wait for it): created on first use, highest priority so its
// CTAs are scheduled ahead of the HBM passes they run beside
static int split_resources(fp8lm_plan* p) {
  if (p->xs) return FP8LM_OK;
  int lo = 0, hi = 0;
  CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CUDA_TRY(cudaStreamCreateWithPriority(&p->xs, cudaStreamNonBlocking, hi));
  CUDA_TRY(cudaEventCreateWithFlags(&p->ev_q, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&p->ev_x, cudaEventDisableTiming));
  return FP8LM_OK;
}

// Split-step grid caps: the exchange kernel of phase 1 runs at 1.5 CTAs per SM (its
// launch bounds keep it <= 85 registers, 3 CTAs/SM possible), so that it is resident
// beside the HBM passes of the other buckets instead of taking every slot (highest
// stream priority) and serialising them; FP8LM_SPLIT_HCAP (CTAs per SM, 0 = off) caps the
// HBM passes as well.  Measured at GPT-7B N = 4 with 4 buckets (profiles/r2/split):
// 1 CTA/SM 29.5 ms, 1.25 30.0, 1.5 28.8, 2 28.5-30.0, uncapped 33.8, unsplit 31.5.  At
// N = 2 the exchange kernel also runs pass 1 on half the tensors (a quarter at N = 4) and
// needs more room: 6 buckets, 1.25 CTAs/SM 30.9 ms, 1.5 30.3-30.6, 2 29.1-29.2
// (profiles/r2/n2ab).
#ifndef FP8LM_SPLIT_XCAP
#define FP8LM_SPLIT_XCAP 0           /* 0: 2 * #SMs at N = 2, 3 * #SMs / 2 above */
#endif
#ifndef FP8LM_SPLIT_HCAP
#define FP8LM_SPLIT_HCAP 0
#endif
static int split_xcap(const fp8lm_plan* p) {
  if (p->loopback_ctas) return p->loopback_ctas;
  if (FP8LM_SPLIT_XCAP) return FP8LM_SPLIT_XCAP;
  return p->nranks <= 2 ? 2 * num_sms() : 3 * num_sms() / 2;
}
struct CapScope {
  LaunchPolicy saved;
  explicit CapScope(int ctas) : saved(launch_policy()) {
    if (ctas > 0 && (saved.max_ctas == 0 || ctas < saved.max_ctas)) launch_policy().max_ctas = ctas;
  }
  ~CapScope() { launch_policy() = saved; }
};

// phase 0: the whole step on `stream`; 1: amax + quantize on `stream`, the exchange kernel
// on the plan's exchange stream; 2: `stream` waits for that exchange, then the AdamW pass
static int dp_step_impl(fp8lm_plan* p, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                        float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                        float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                        const fp8lm_stensors* v, const fp8lm_stensors* master,
                        const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                        int32_t hist_slot, void* stream, int phase) {
  const LaunchScope ls_(p);   // loopback plans: capped grids
  const CapScope hcap_(phase ? FP8LM_SPLIT_HCAP * num_sms() : 0);
  int rc;
  const bool delayed = w_hist != nullptr;
  if (phase == 0 && p && p->mode == FP8LM_MODE_P2P && p->T > 0 && p->g8_bytes <= p->oneshot_max_bytes) {
    // small message: A1-A5 in one kernel (the one-shot exchange leaves the whole reduced
    // set in g8), then both AdamW passes locally
    if ((rc = check_stensors(p, m1, "m1", "dp_step")) || (rc = check_stensors(p, v, "v", "dp_step")) ||
        (rc = check_stensors(p, master, "master", "dp_step")) || (rc = check_stensors(p, w8, "w8", "dp_step")))
      return rc;
    if (!hp) return fail(FP8LM_EINVAL, "dp_step: NULL hp");
    if (delayed && (hist_slot < 0 || hist_slot >= 16)) return fail(FP8LM_EINVAL, "dp_step: hist_slot not in [0, 16)");
    if ((rc = fp8lm_allreduce_jit(p, comm, grads, src_dtype, mu, amax_out, s_g, skip, g8, g_scale, g_scale_inv,
                                  sat, stream)))
      return rc;
    if (delayed)
      CUDA_TRY(launch_adam_delayed(p->dev, g8, g_scale_inv, *m1, *v, *master, *w8, *hp, skip, w_hist,
                                   hist_slot, S(stream)));
    else
      CUDA_TRY(launch_adam(p->dev, g8, g_scale_inv, *m1, *v, *master, *w8, *hp, skip, S(stream)));
    return FP8LM_OK;
  }
  if (phase != 2 && (rc = fp8lm_amax_scale_sync(p, comm, grads, src_dtype, mu, amax_out, s_g, skip, stream)))
    return rc;
  if (delayed && (hist_slot < 0 || hist_slot >= 16)) return fail(FP8LM_EINVAL, "dp_step: hist_slot not in [0, 16)");
  // SIMULATED with 2..4 ranks (config C1): quantize + rank-order reduce + Adam pass 1 in one
  // kernel, like LOCAL; more ranks (tests up to 16) and delayed scaling take the three calls
  const bool sim_fused = p->mode == FP8LM_MODE_SIMULATED && p->nranks <= 4 && !delayed;
  if ((p->mode != FP8LM_MODE_LOCAL && p->mode != FP8LM_MODE_P2P && p->mode != FP8LM_MODE_ZERO &&
       !sim_fused) ||
      p->T == 0 || (delayed && p->mode == FP8LM_MODE_ZERO)) {
    rc = fp8lm_grad_allreduce(p, comm, grads, src_dtype, s_g, skip, g8, g_scale, g_scale_inv, sat,
                              mu, stream);
    if (rc) return rc;
    if (delayed)
      return fp8lm_adam_step_delayed(p, g8, g_scale_inv, m1, v, master, w8, hp, skip, w_hist,
                                     hist_slot, stream);
    return fp8lm_adam_step(p, g8, g_scale_inv, m1, v, master, w8, hp, skip, stream);
  }
  if (p->mode == FP8LM_MODE_ZERO) {
    // the owner reduce runs Adam pass 1 on the reduced codes of its whole tensors
    if (!p->p2p_ready) return fail(FP8LM_EINVAL, "dp_step: mode ZERO needs fp8lm_peer_setup first");
    if (!hp || !g_scale || !g_scale_inv || !sat || !m1 || !v || !master || !w8)
      return fail(FP8LM_EINVAL, "dp_step: NULL argument");
    if (p->own->T > 0 && (!g8 || !aligned(g8, 256))) return fail(FP8LM_EINVAL, "dp_step: g8 NULL or misaligned");
    const TailArgs tail{p->nranks, skip, sat, g_scale, g_scale_inv, mu};
    cudaStream_t ps = S(stream);   // the stream pass 2 (+ w8 broadcast) runs on
    if (phase != 2) {
      const void* srcs[1];
      int nsrc = 0;
      if ((rc = grad_sources(p, grads, src_dtype, srcs, &nsrc, "dp_step"))) return rc;
      CUDA_TRY(launch_quantize_push(p->dev, p2p_args(p), srcs[0], src_dtype, s_g, S(stream)));
      cudaStream_t xs = S(stream);
      if (phase == 1) {
        CUDA_TRY(cudaEventRecord(p->ev_q, S(stream)));
        CUDA_TRY(cudaStreamWaitEvent(p->xs, p->ev_q, 0));
        xs = p->xs;
      }
      {
        LaunchPolicy keep = launch_policy();
        if (phase == 1) launch_policy().max_ctas = split_xcap(p);
        rc = launch_reduce_owner_a1(p->dev, p->own->dev, p2p_args(p), s_g, tail, g8, *m1, *v,
                                    *master, *w8, *hp, skip, xs);
        launch_policy() = keep;
        CUDA_TRY((cudaError_t)rc);
      }
      // split step: pass 2 follows on the exchange stream (GPT-13B N = 4, 4 buckets:
      // 44.8 ms with it on the rank stream, 41.1-41.7 here; profiles/r2/zero_push)
      if (phase == 1) ps = p->xs;
    } else {
      CUDA_TRY(cudaStreamWaitEvent(S(stream), p->ev_x, 0));
      return FP8LM_OK;
    }
    // pass 2 on the owned tensors also stores every w8 group into every rank's window
    // (the broadcast overlaps the HBM-bound pass); its last CTA publishes the scalars.
    // In a split step it follows the owner reduce on the exchange stream: both are
    // NVLink-bound, and there they overlap the other buckets' amax / quantize passes
    Pass2Ext ext;
    ext.bcast = p2p_args(p);
    ext.own_gpos = p->dev.own_gpos;
    ext.own2full = p->dev.own2full;
    ext.T_full = p->T;
    {
      LaunchPolicy keep = launch_policy();
      if (ps != S(stream)) launch_policy().max_ctas = split_xcap(p);
      if (p->own->dev.n_items > 0) {
        rc = launch_adam(p->own->dev, g8, p->dev.gsinv_own, *m1, *v, *master, *w8, *hp, skip, ps,
                         /*pass1=*/false, &ext);
      } else {   // a rank that owns nothing still meets the others at flag W8
        rc = launch_w8_bcast(p->dev, p->own->dev, ext.bcast, static_cast<const uint8_t*>(w8->data),
                             *w8, ps);
      }
      launch_policy() = keep;
      CUDA_TRY((cudaError_t)rc);
    }
    if (ps != S(stream)) CUDA_TRY(cudaEventRecord(p->ev_x, p->xs));
    return FP8LM_OK;
  }
  if (p->mode == FP8LM_MODE_P2P) {
    // the exchange kernel runs Adam pass 1 on its own shard; maxima combined in its tail
    if ((rc = check_stensors(p, m1, "m1", "dp_step")) || (rc = check_stensors(p, v, "v", "dp_step")) ||
        (rc = check_stensors(p, master, "master", "dp_step")) ||
        (rc = check_stensors(p, w8, "w8", "dp_step")))
      return rc;
    if (!hp || !g_scale || !g_scale_inv || !sat) return fail(FP8LM_EINVAL, "dp_step: NULL argument");
    if (g8 != p->win_g8) return fail(FP8LM_EINVAL, "dp_step: mode P2P needs g8 == fp8lm_peer_g8(plan)");
    const TailArgs tail{p->nranks, skip, sat, g_scale, g_scale_inv, mu};
    P2PArgs x = p2p_args(p);
    if (phase != 2) {
      const void* srcs[1];
      int nsrc = 0;
      if ((rc = grad_sources(p, grads, src_dtype, srcs, &nsrc, "dp_step"))) return rc;
      // the whole step (phase 0): the quantize pushes each code group into its shard
      // owner's slot, so the exchange kernel reads locally (unsplit GPT-7B N = 4: 31.7 ->
      // 30.4 ms).  A split step keeps the codes in the own window and the exchange pulls
      // them on the exchange stream, where the transfer hides under the other buckets'
      // passes (a pushing quantize is NVLink-bound on the rank's stream: 28.4 -> 31.8 ms)
      x.slots = phase == 0 ? 1 : 0;
      if (x.slots) {
        CUDA_TRY(launch_quantize_push(p->dev, x, srcs[0], src_dtype, s_g, S(stream), /*shard_slots=*/true));
      } else {
        uint8_t* dst[1] = {p->win_send};
        CUDA_TRY(launch_quantize(p->dev, srcs, dst, 1, src_dtype, s_g, nullptr, S(stream)));
      }
      cudaStream_t xs = S(stream);
      if (phase == 1) {
        CUDA_TRY(cudaEventRecord(p->ev_q, S(stream)));
        CUDA_TRY(cudaStreamWaitEvent(p->xs, p->ev_q, 0));
        xs = p->xs;
      }
      {
        LaunchPolicy keep = launch_policy();
        if (phase == 1) launch_policy().max_ctas = split_xcap(p);
        if (delayed)            // reduce-scatter only (the single delayed pass pulls the rest)
          rc = launch_reduce_p2p(p->dev, x, g8, s_g, tail, xs, /*ag=*/false);
        else
          rc = launch_reduce_p2p_a1(p->dev, x, s_g, tail, g8, *m1, *v, *master, *w8, *hp, skip, xs);
        launch_policy() = keep;
        CUDA_TRY((cudaError_t)rc);
      }
      if (phase == 1) {
        CUDA_TRY(cudaEventRecord(p->ev_x, p->xs));
        return FP8LM_OK;
      }
    } else {
      CUDA_TRY(cudaStreamWaitEvent(S(stream), p->ev_x, 0));
    }
    // the exchange leaves each rank's reduced shard in its own window; the AdamW pass
    // that encodes the states pulls the other shards' codes from the peers' windows (the
    // all-gather, overlapped with its HBM traffic), walking its work items from this
    // rank's shard on so that the ranks pull from different owners at any moment
    const int64_t lo = p->shard * p->rank;
    const auto first = std::lower_bound(p->items.begin(), p->items.end(), lo,
                                        [](const ShardItem& a, int64_t v) { return a.pos < v; });
    Pass2Ext ext;
    ext.pull_tab = x.tab;
    ext.pull_shard = p->shard;
    ext.rot = (int64_t)(first - p->items.begin());
    if (delayed) {            // the single delayed pass
      CUDA_TRY(launch_adam_delayed(p->dev, g8, g_scale_inv, *m1, *v, *master, *w8, *hp, skip,
                                   w_hist, hist_slot, S(stream), &ext));
      return FP8LM_OK;
    }
    CUDA_TRY(launch_adam(p->dev, g8, g_scale_inv, *m1, *v, *master, *w8, *hp, skip, S(stream),
                         /*pass1=*/false, &ext));
    return FP8LM_OK;
  }
  if (phase != 0) return fail(FP8LM_EINVAL, "dp_step_split: modes P2P / ZERO only");
  // LOCAL: the codes quantize produces are final, so Adam pass 1 runs in the same kernel;
  // SIMULATED (2..4 ranks): the same kernel quantizes every rank's value and reduces them
  if ((rc = check_stensors(p, m1, "m1", "dp_step")) || (rc = check_stensors(p, v, "v", "dp_step")) ||
      (rc = check_stensors(p, master, "master", "dp_step")) ||
      (rc = check_stensors(p, w8, "w8", "dp_step")))
    return rc;
  if (!hp || !g_scale || !g_scale_inv || !sat) return fail(FP8LM_EINVAL, "dp_step: NULL argument");
  if (!g8 || !aligned(g8, 256)) return fail(FP8LM_EINVAL, "dp_step: g8 NULL or misaligned");
  const void* srcs[FP8LM_MAX_SIM_RANKS];
  int nsrc = 0;
  if ((rc = grad_sources(p, grads, src_dtype, srcs, &nsrc, "dp_step"))) return rc;
  const TailArgs tail{nsrc, skip, sat, g_scale, g_scale_inv, mu};
  CUDA_TRY(launch_adam_fused_local(p->dev, srcs, nsrc, src_dtype, s_g, g8, tail, *m1, *v, *master, *w8,
                                   *hp, skip, S(stream), w_hist, hist_slot));
  return FP8LM_OK;
}

int fp8lm_dp_step(fp8lm_plan* p, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                  float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                  float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                  const fp8lm_stensors* v, const fp8lm_stensors* master,
                  const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                  int32_t hist_slot, void* stream) {
  return dp_step_impl(p, comm, grads, src_dtype, mu, amax_out, s_g, skip, g8, g_scale, g_scale_inv, sat,
                      m1, v, master, w8, hp, w_hist, hist_slot, stream, 0);
}

int fp8lm_dp_step_split(fp8lm_plan* p, int32_t phase, const void* grads, int32_t src_dtype,
                        float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                        float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                        const fp8lm_stensors* v, const fp8lm_stensors* master,
                        const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                        int32_t hist_slot, void* stream) {
  if (!p || (p->mode != FP8LM_MODE_P2P && p->mode != FP8LM_MODE_ZERO))
    return fail(FP8LM_EINVAL, "dp_step_split: modes P2P / ZERO only");
  if (phase != 1 && phase != 2) return fail(FP8LM_EINVAL, "dp_step_split: phase must be 1 or 2");
  if (w_hist && p->mode == FP8LM_MODE_ZERO)
    return fail(FP8LM_EINVAL, "dp_step_split: mode ZERO with delayed state scaling has no split form");
  if ((phase == 2) != p->split_open)
    return fail(FP8LM_EINVAL, "dp_step_split: phase %d out of order (phases 1 and 2 alternate)", phase);
  int rc = split_resources(p);
  if (rc) return rc;
  rc = dp_step_impl(p, nullptr, grads, src_dtype, mu, amax_out, s_g, skip, g8, g_scale, g_scale_inv, sat,
                    m1, v, master, w8, hp, w_hist, hist_slot, stream, phase);
  if (!rc) p->split_open = phase == 1;
  return rc;
}

int fp8lm_dp_step_graphed(fp8lm_plan* p, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                          float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                          float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                          const fp8lm_stensors* v, const fp8lm_stensors* master,
                          const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                          int32_t hist_slot, void* stream) {
  if (!p) return fail(FP8LM_EINVAL, "dp_step_graphed: plan is NULL");
  auto eager = [&] {
    return dp_step_impl(p, comm, grads, src_dtype, mu, amax_out, s_g, skip, g8, g_scale, g_scale_inv, sat, m1, v,
                        master, w8, hp, w_hist, hist_slot, stream, 0);
  };
  if (p->mode == FP8LM_MODE_NCCL || !hp || !m1 || !v || !master || !w8) return eager();
  // the graph is valid for one set of buffers: every pointer argument, the dtype, the
  // state scaling and the stream
  std::vector<uintptr_t> key = {(uintptr_t)comm, (uintptr_t)src_dtype, (uintptr_t)mu, (uintptr_t)amax_out,
                                (uintptr_t)s_g, (uintptr_t)skip, (uintptr_t)g8, (uintptr_t)g_scale,
                                (uintptr_t)g_scale_inv, (uintptr_t)sat, (uintptr_t)w_hist, (uintptr_t)stream};
  if (p->mode == FP8LM_MODE_SIMULATED) {
    const void* const* arr = static_cast<const void* const*>(grads);
    for (int r = 0; arr && r < p->nranks; ++r) key.push_back((uintptr_t)arr[r]);
  } else {
    key.push_back((uintptr_t)grads);
  }
  for (const fp8lm_stensors* st : {m1, v, master, w8}) {
    key.push_back((uintptr_t)st->data); key.push_back((uintptr_t)st->scale);
    key.push_back((uintptr_t)st->scale_inv); key.push_back((uintptr_t)st->amax);
  }
  cudaStream_t s = S(stream);
  constexpr size_t kMaxGraphs = 4;
  fp8lm_plan::GraphEntry* ge = nullptr;
  for (auto& g : p->graphs)
    if (g.key == key) ge = &g;
  if (!ge) {                          // new buffers: a new entry (the least recently used goes)
    if (p->graphs.size() >= kMaxGraphs) {
      auto lru = std::min_element(p->graphs.begin(), p->graphs.end(),
                                  [](const auto& x, const auto& y) { return x.used < y.used; });
      if (lru->exec) cudaGraphExecDestroy(lru->exec);
      if (lru->graph) cudaGraphDestroy(lru->graph);
      if (lru->log) adam_log_free(lru->log);
      p->graphs.erase(lru);
    }
    p->graphs.emplace_back();
    ge = &p->graphs.back();
    ge->key = key;
  }
  ge->used = ++p->graph_clock;
  if (!ge->exec && ge->seen++ == 0) return eager();   // first call: modules load, caches fill
  if (!ge->exec) {                    // second call: capture this step, then launch it
    if (ge->log) adam_log_free(ge->log);
    ge->log = adam_log_new();
    // capture on a plan-owned stream (the caller's may be the legacy default stream,
    // which cannot be captured); the graph is then launched on the caller's stream
    if (!p->gs) CUDA_TRY(cudaStreamCreateWithFlags(&p->gs, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamBeginCapture(p->gs, cudaStreamCaptureModeThreadLocal));
    adam_log_activate(ge->log);
    const int rc = dp_step_impl(p, comm, grads, src_dtype, mu, amax_out, s_g, skip, g8, g_scale, g_scale_inv, sat,
                                m1, v, master, w8, hp, w_hist, hist_slot, p->gs, 0);
    adam_log_activate(nullptr);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(p->gs, &g);
    if (rc) { if (g) cudaGraphDestroy(g); return rc; }
    CUDA_TRY(ce);
    ge->graph = g;
    CUDA_TRY(cudaGraphInstantiate(&ge->exec, g, 0));
    CUDA_TRY(cudaGraphLaunch(ge->exec, s));
    return FP8LM_OK;
  }
  // replay: patch this step's scalars into the AdamW nodes, launch
  CUDA_TRY(adam_log_update(ge->log, ge->exec, *hp, hist_slot));
  CUDA_TRY(cudaGraphLaunch(ge->exec, s));
  return FP8LM_OK;
}

int fp8lm_state_init(fp8lm_plan* p, const float* w0, const fp8lm_stensors* m1,
                     const fp8lm_stensors* v, const fp8lm_stensors* master,
                     const fp8lm_stensors* w8, void* stream) {
  const LaunchScope ls_(p);   // loopback plans: capped grids
  if (!p) return fail(FP8LM_EINVAL, "state_init: plan is NULL");
  if (!p->bound) return fail(FP8LM_EWORKSPACE, "state_init: plan not bound");
  int rc;
  if ((rc = check_stensors(p, m1, "m1", "state_init")) || (rc = check_stensors(p, v, "v", "state_init")) ||
      (rc = check_stensors(p, master, "master", "state_init")) || (rc = check_stensors(p, w8, "w8", "state_init")))
    return rc;
  if (p->mode == FP8LM_MODE_ZERO) {
    if (!p->p2p_ready) return fail(FP8LM_EINVAL, "state_init: mode ZERO needs fp8lm_peer_setup first");
    if (p->own->T > 0 && (!w0 || !aligned(w0, 256))) return fail(FP8LM_EINVAL, "state_init: w0 NULL or misaligned");
    CUDA_TRY(launch_state_init(p->own->dev, w0, *m1, *v, *master, *w8, S(stream)));
    CUDA_TRY(launch_w8_bcast(p->dev, p->own->dev, p2p_args(p),
                             static_cast<const uint8_t*>(w8->data), *w8, S(stream)));
    return FP8LM_OK;
  }
  if (p->T > 0 && (!w0 || !aligned(w0, 256))) return fail(FP8LM_EINVAL, "state_init: w0 NULL or misaligned");
  CUDA_TRY(launch_state_init(p->dev, w0, *m1, *v, *master, *w8, S(stream)));
  return FP8LM_OK;
}

}  // extern "C"
