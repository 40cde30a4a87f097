// internal.h — host-side structures shared by the C-ABI layer (api.cpp) and the
// kernel launchers (kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fp8lm.h"

namespace fp8lm {

// one reduce-scatter work item: bytes [pos, pos+len) of tensor t (global flat coords)
struct ShardItem {
  int64_t pos;
  int32_t t;
  int32_t len;
};

// device views of the plan tables inside the caller's workspace
struct DevPlan {
  int32_t T;
  int32_t nranks;
  int64_t total;            // elements of each flat buffer
  int64_t n_items;          // full-tensor work items
  const int64_t* numel;     // [T]
  const int64_t* offset;    // [T]
  const int64_t* item_start;// [T+1]
  const ShardItem* items;   // [n_items] full-tensor work items (pos, t, len): one 16-B load
  const ShardItem* shard_items;
  int64_t n_shard_items;
  uint32_t* acc_amax;       // [nsim*T]  float bits, atomicMax accumulators (zero at rest)
  uint32_t* acc_state;      // [3*T]     amax of m', v', w' (zero at rest)
  uint32_t* sat_part;       // [T]       per-shard saturation counts (NCCL)
  uint8_t* send;            // [N*S]     NCCL send buffer (quantized codes, flat)
  uint8_t* recv;            // [N*S]     NCCL all-to-all receive buffer
  uint8_t* sim_codes;       // [nsim*total] simulated ranks' quantized codes
  uint32_t* sat_acc;        // [T]       saturation counts of the step (zero at rest)
  uint32_t* counters;       // [8]       grid_last_block tickets, grid barrier (zero at rest)
  // mode ZERO: owned tensors j = 0..T_own-1 (ascending t)
  int32_t T_own;
  const int64_t* own_gpos;  // [T_own] full-layout offset of owned tensor j
  const int32_t* own2full;  // [T_own] its global index t
  float* gsinv_own;         // [T_own] compact copy of g_scale_inv (written by the reduce tail)
  // mode ZERO push layout: rank r's codes of tensor t go to window(owner_of[t]) +
  // push_base[t] + pos (slot r of the owner's compact layout); own_slot = this rank's
  // slot size (its compact total), so slot r of its own window starts at r * own_slot
  const int64_t* push_base; // [T]
  const int32_t* owner_of;  // [T]
  int64_t own_slot;
  // mode P2P push layout: rank r's codes of shard q go to window(q) + r * shard + (pos - q * shard)
  int64_t shard;
};

constexpr int kCtrAmax = 0, kCtrTail = 1, kCtrAdam = 2, kCtrFix = 3, kCtrFixGen = 4, kCtrOneshot = 5,
              kCtrPhase = 6 /* k_oneshot_full's phase word: the last released epoch */, kCtrWords = 8;

// ---------------------------------------------------------------- mode P2P windows
// Signal / exchange pad of one rank (bytes): three flag arrays (one u32 epoch slot per
// source rank), the peer pointer table, then the exchanged per-tensor data:
// scales[N][T] (float, local scales for the MIN of Eq. 4) and sat[N][T] (u32,
// per-shard saturation counts).
constexpr int kMaxPeers = FP8LM_MAX_P2P_RANKS;
constexpr size_t kPadFlagScale = 0, kPadFlagReady = 64, kPadFlagDone = 128, kPadFlagW8 = 192,
                 kPadTable = 256, kPadCtl = 512, kPadData = 1024;
// kPadCtl: this rank's epoch counters, device-resident so that a captured (CUDA-graph)
// step advances them on every replay: [0] the step epoch (bumped by k_amax's exchange
// epilogue, read by the step's later kernels), [1] the w8-broadcast epoch (mode ZERO)
struct PeerTable {
  uint8_t* send[kMaxPeers];
  uint8_t* g8[kMaxPeers];
  uint32_t* pad[kMaxPeers];
  uint8_t* w8[kMaxPeers];   // mode ZERO: replicated FP8 weight copy (full layout)
};
static_assert(kPadTable + sizeof(PeerTable) <= kPadCtl && kPadCtl + 8 <= kPadData, "pad layout");
// pad data region: scales [N][T] f32 | sat [N][T] u32 | (ZERO) w8 scalars [3][T] f32 |
// pass-1 state maxima [N][3T] u32 (fused P2P step)
inline size_t pad_bytes_for(int N, int T) {
  const size_t t = T > 0 ? T : 1;
  return kPadData + (size_t)N * t * 8 + 3 * t * 4 + (size_t)N * 3 * t * 4;
}
struct P2PArgs {
  const PeerTable* tab;   // device copy inside this rank's pad
  uint32_t* pad;          // this rank's pad
  int rank;
  int nranks;
  // mode P2P: 1 — this step's quantize pushed the codes into the shard owners' window
  // slots (the reduce-scatter reads N local slots); 0 — each rank's codes are in its own
  // send window, full layout (the reduce-scatter pulls them)
  int slots = 0;
};
// the step's epoch (flags hold the epoch of their last signal) / the w8 epoch, from the
// own pad's counters
__host__ __device__ inline uint32_t* pad_ctl(uint32_t* pad) {
  return reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(pad) + kPadCtl);
}

// ---------------------------------------------------------------- FP8 SP converter (f4)
// pad of one rank (bytes): three flag rows (one u32 epoch per source rank), the ranks'
// local scales, then the peer table
constexpr size_t kSpPadFlagScale = 0, kSpPadFlagData = 64, kSpPadFlagDone = 128, kSpPadScales = 192,
                 kSpPadTable = 256, kSpPadBytes = 512;
struct SpTable {
  uint8_t* recv[kMaxPeers];   // all-gather receive windows (N m bytes)
  uint8_t* send[kMaxPeers];   // reduce-scatter send windows (N m bytes)
  uint32_t* pad[kMaxPeers];
};
static_assert(kSpPadTable + sizeof(SpTable) <= kSpPadBytes, "sp pad layout");
// local scratch (u32 words, zero at rest except s / sinv)
constexpr int kSpScrAmax = 0, kSpScrBad = 1, kSpScrTicketA = 2, kSpScrTicketB = 3, kSpScrTicketC = 4,
              kSpScrS = 5, kSpScrSinv = 6, kSpScrFlag1 = 7, kSpScrFlag2 = 8, kSpScrWords = 16;
struct SpArgs {
  uint32_t* pad;       // this rank's pad (its table copy at kSpPadTable)
  uint32_t* scratch;
  int rank;
  int nranks;
  uint32_t epoch;
  bool vec;            // 16-element vector paths (sizes multiples of 16, aligned buffers)
};

// pass 2 of the fused multi-GPU steps (fp8lm_dp_step)
struct Pass2Ext {
  // mode P2P: the all-gather pulled from the owners' g8 windows, work order rotated
  const PeerTable* pull_tab = nullptr;
  int64_t pull_shard = 0;
  int64_t rot = 0;
  // mode ZERO: w8 stored into every rank's window (tab == nullptr: off)
  P2PArgs bcast{};
  const int64_t* own_gpos = nullptr;
  const int32_t* own2full = nullptr;
  int T_full = 0;
};

struct GraphAdamLog;   // kernels.cu: the captured AdamArgs launches of a graphed step

// outputs of the Eq. 6 / mu tail of fp8lm_grad_allreduce
struct TailArgs {
  int nranks;
  const int32_t* skip;
  uint32_t* sat;
  float* g_scale;
  float* g_scale_inv;
  float* mu;
};

}  // namespace fp8lm

// raw one-shot sizes: the window copy is allocated for plans up to kRawAllocMax code bytes
// and used, by default, while a rank's raw pull ((N-1) * 4 * n bytes) is at most
// FP8LM_ONESHOT_RAW_PULL — measured (profiles/r2/c5_raw): the raw kernel wins up to 256K
// elements at N = 2 and 64K at N = 4 (fp8lm_plan_set_oneshot_raw changes it per plan)
#ifndef FP8LM_ONESHOT_RAW_PULL
#define FP8LM_ONESHOT_RAW_PULL (1 << 20)
#endif
constexpr int64_t kRawAllocMax = 1 << 20;

struct fp8lm_plan {
  int32_t T = 0;
  int32_t mode = 0;
  int32_t nranks = 1;
  int32_t rank = 0;
  std::vector<int64_t> numel, offset, item_start;
  std::vector<fp8lm::ShardItem> items, shard_items;
  int64_t total = 0;        // elements per flat buffer
  int64_t shard = 0;        // S bytes (NCCL)
  int64_t g8_bytes = 0;
  // workspace layout (byte offsets)
  size_t off_numel = 0, off_offset = 0, off_item_start = 0, off_items = 0, off_shard_items = 0;
  size_t off_acc_amax = 0, off_acc_state = 0, off_sat_part = 0, off_sat_acc = 0, off_ctr = 0,
         off_acc_end = 0;
  size_t off_send = 0, off_recv = 0, off_sim = 0, ws_bytes = 0;
  void* ws = nullptr;
  fp8lm::DevPlan dev{};
  bool bound = false;
  // mode P2P: symmetric windows owned by the plan, peer mappings, step epoch
  uint8_t* win_send = nullptr;
  uint8_t* win_g8 = nullptr;
  uint32_t* win_pad = nullptr;
  size_t pad_bytes = 0;
  std::vector<void*> mapped;
  bool p2p_ready = false;
  uint8_t* win_w8 = nullptr;
  // single-process loopback of modes P2P / ZERO (fp8lm_peer_setup_loopback): the N ranks
  // are N plans of one process on one GPU; every kernel of this plan launches at most
  // loopback_ctas CTAs (num_sms / N, so the N ranks' kernels are all resident at once:
  // the spin-waits need that) without the cooperative / PDL attributes.  0: off.
  int loopback_ctas = 0;
  // mode P2P: a plan whose reduced codes fit in this many bytes takes the one-shot
  // exchange (fp8lm_plan_set_oneshot; default 1 MiB)
  int64_t oneshot_max_bytes = 1 << 20;
  // raw one-shot (launch_oneshot_raw): the send window carries two fp32 copies of the set
  // behind the codes when g8_bytes <= kRawAllocMax; used up to oneshot_raw_max_bytes
  int64_t raw_off = 0, raw_half = 0;
  int64_t oneshot_raw_max_bytes = 0;   // set by fp8lm_plan_create from N
  // split step (fp8lm_dp_step_split): the exchange stream and its two events
  cudaStream_t xs = nullptr;
  cudaEvent_t ev_q = nullptr, ev_x = nullptr;
  bool split_open = false;
  // fp8lm_dp_step_graphed: captured steps, one per set of pointer arguments (and dtype,
  // state scaling, stream) — a few, for callers that rotate gradient buffers
  struct GraphEntry {
    std::vector<uintptr_t> key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    fp8lm::GraphAdamLog* log = nullptr;
    int seen = 0;                    // calls with this key (the 2nd one captures)
    uint64_t used = 0;               // LRU stamp
  };
  std::vector<GraphEntry> graphs;
  uint64_t graph_clock = 0;
  cudaStream_t gs = nullptr;         // the capture stream
  // mode ZERO: Alg. 1 owners, the owned tensors and the compact sub-plan over them
  std::vector<int32_t> owner, own2full;
  std::vector<int64_t> own_gpos, full2own_off;
  fp8lm_plan* own = nullptr;
  size_t off_own_ws = 0, off_own_gpos = 0, off_own2full = 0, off_gsinv_own = 0;
  std::vector<int64_t> push_base;
  size_t off_push_base = 0, off_owner_of = 0;
};

namespace fp8lm {
// ------------------------------------------------------------------ launch tracing
// When enabled (fp8lm_prof_enable), every kernel / collective the library enqueues is
// bracketed by two CUDA events on its own stream; fp8lm_prof_read aggregates the
// durations per name.  Used by bench.py for the per-kernel roofline and launch count.
enum ProfId : int {
  P_AMAX = 0, P_SCALE, P_SCALE_FIX, P_QUANTIZE, P_REDUCE, P_AR_FINALIZE, P_ADAM1, P_ADAM2,
  P_ADAM_FINALIZE, P_ADAM_WFIX, P_STATE_INIT, P_Q_SINGLE, P_DQ_SINGLE, P_MEMSET,
  P_NCCL_MIN, P_NCCL_A2A, P_NCCL_AG_SUM, P_REDUCE_P2P, P_QADAM1, P_W8_BCAST, P_ADAM_DELAYED,
  P_QADAM_DELAYED, P_STRAT_AMAX, P_STRAT_REDUCE, P_SP_ALLGATHER, P_SP_REDUCE_SCATTER,
  P_COUNT
};
bool prof_on();
struct ProfScope {
  int id;
  cudaStream_t s;
  void* a = nullptr;
  ProfScope(int id_, cudaStream_t s_);
  ~ProfScope();
};

// kernel launchers (kernels.cu); return cudaError_t of the launch
cudaError_t launch_amax(const DevPlan& p, const void* const* srcs, int nsrc, int src_dtype,
                        const float* mu, float* amax_out, float* s_out, int32_t* skip,
                        bool finalize, const P2PArgs* x, cudaStream_t s);
cudaError_t launch_reduce_p2p(const DevPlan& p, const P2PArgs& x, uint8_t* g8, const float* s_g,
                              const TailArgs& tail, cudaStream_t s, bool ag = true);
// mode P2P, small messages: quantize into the own send window, then every rank pulls and
// reduces the WHOLE tensor set from every rank (one kernel, one cross-rank handshake)
cudaError_t launch_oneshot(const DevPlan& p, const P2PArgs& x, const void* src, int src_dtype,
                           uint8_t* g8, const float* s_g, const TailArgs& tail, cudaStream_t s);
// A1-A5 of a small plan in one kernel: amax, MIN through the pads, then the one-shot body
cudaError_t launch_oneshot_full(const DevPlan& p, const P2PArgs& x, const void* src, int src_dtype,
                                const float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                                const TailArgs& tail, cudaStream_t s);
// the same with ONE cross-rank handshake: the gradient copied into the send window's raw
// half (epoch & 1) at raw_off + half * raw_half; every rank pulls and encodes every rank's
cudaError_t launch_oneshot_raw(const DevPlan& p, const P2PArgs& x, const void* src, int src_dtype,
                               const float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                               const TailArgs& tail, int64_t raw_off, int64_t raw_half, cudaStream_t s);
// mode ZERO: A3 pushing every code into its owner's window (slot = this rank), then one
// system-scope fence per CTA so the owners' reduce (after its "ready" flag) sees them
// mode P2P (shard_slots): the same into slot `rank` of each shard owner's window
cudaError_t launch_quantize_push(const DevPlan& p, const P2PArgs& x, const void* src, int src_dtype,
                                 const float* s_g, cudaStream_t s, bool shard_slots = false);
// mode ZERO: owner reduce over the compact sub-plan `o` (items), tails on the full plan `p`
cudaError_t launch_reduce_owner(const DevPlan& p, const DevPlan& o, const P2PArgs& x, uint8_t* g8,
                                const float* s_g, const TailArgs& tail, cudaStream_t s);
// mode ZERO: owned w8 codes (compact) + scalars -> every rank's w8 window / pad rows
cudaError_t launch_w8_bcast(const DevPlan& p, const DevPlan& o, const P2PArgs& x,
                            const uint8_t* w8_own, const fp8lm_stensors& w8s, cudaStream_t s);
cudaError_t launch_scale_fix(const DevPlan& p, float* s_g, int32_t* skip, cudaStream_t s);
cudaError_t launch_quantize(const DevPlan& p, const void* const* srcs, uint8_t* const* dsts,
                            int nsrc, int src_dtype, const float* s_g, const TailArgs* tail,
                            cudaStream_t s);
cudaError_t launch_reduce(const DevPlan& p, const uint8_t* base, int64_t stride, int nsrc,
                          int64_t shift, bool shard_items, uint8_t* dst, const float* s_g,
                          const TailArgs* tail, cudaStream_t s);
cudaError_t launch_allreduce_finalize(const DevPlan& p, const float* s_g, const TailArgs& tail,
                                      cudaStream_t s);
cudaError_t launch_adam(const DevPlan& p, const uint8_t* g8, const float* g_sinv,
                        const fp8lm_stensors& m1, const fp8lm_stensors& v,
                        const fp8lm_stensors& w, const fp8lm_stensors& w8,
                        const fp8lm_adam_hp& hp, const int32_t* skip, cudaStream_t s,
                        bool pass1 = true, const Pass2Ext* ext = nullptr);
// fused quantize (+ the rank-order reduce of nsrc = 2..4 simulated ranks) + Adam pass 1,
// then pass 2; nsrc = 1: LOCAL (also the delayed single pass when w_hist != nullptr)
cudaError_t launch_adam_fused_local(const DevPlan& p, const void* const* srcs, int nsrc, int src_dtype,
                                   const float* s_g, uint8_t* g8, const TailArgs& tail,
                                   const fp8lm_stensors& m1, const fp8lm_stensors& v,
                                   const fp8lm_stensors& w, const fp8lm_stensors& w8,
                                   const fp8lm_adam_hp& hp, const int32_t* skip, cudaStream_t s,
                                   float* w_hist = nullptr, int hist_slot = 0);
// delayed state scaling: one AdamW pass (App. B)
cudaError_t launch_adam_delayed(const DevPlan& p, const uint8_t* g8, const float* g_sinv,
                                const fp8lm_stensors& m1, const fp8lm_stensors& v,
                                const fp8lm_stensors& w, const fp8lm_stensors& w8,
                                const fp8lm_adam_hp& hp, const int32_t* skip, float* w_hist,
                                int hist_slot, cudaStream_t s, const Pass2Ext* ext = nullptr);
// mode P2P fused step: exchange + reduce + Adam pass 1 on the own shard (+ maxima exchange)
cudaError_t launch_reduce_p2p_a1(const DevPlan& p, const P2PArgs& x, const float* s_g,
                                 const TailArgs& tail, uint8_t* g8, const fp8lm_stensors& m1,
                                 const fp8lm_stensors& v, const fp8lm_stensors& w,
                                 const fp8lm_stensors& w8, const fp8lm_adam_hp& hp,
                                 const int32_t* skip, cudaStream_t s);
cudaError_t launch_state_init(const DevPlan& p, const float* w0, const fp8lm_stensors& m1,
                              const fp8lm_stensors& v, const fp8lm_stensors& w,
                              const fp8lm_stensors& w8, cudaStream_t s);
// single-tensor codec (fp8lm_quantize / fp8lm_dequantize)
cudaError_t launch_q_single(const void* src, int src_dtype, int64_t n, int fmt, void* dst,
                            float* scale, float* scale_inv, float* amax, int jit,
                            uint32_t* sat, cudaStream_t s);
cudaError_t launch_allreduce_strategy(int strategy, const float* g, int N, int64_t n, float* mu,
                                      uint8_t* codes, fp8lm_commstats* st, cudaStream_t s);
cudaError_t launch_sp_allgather(const void* x, int x_dtype, int64_t m, uint8_t* codes_out, void* out,
                                int out_dtype, float* scale_out, const SpArgs& a, cudaStream_t s);
cudaError_t launch_sp_reduce_scatter(const void* dy, int dtype, int64_t m, void* out, int out_dtype,
                                     float* scale_out, const SpArgs& a, cudaStream_t s);
cudaError_t launch_reduce_owner_a1(const DevPlan& p, const DevPlan& o, const P2PArgs& x, const float* s_g,
                                   const TailArgs& tail, uint8_t* g8, const fp8lm_stensors& m1,
                                   const fp8lm_stensors& v, const fp8lm_stensors& w,
                                   const fp8lm_stensors& w8, const fp8lm_adam_hp& hp,
                                   const int32_t* skip, cudaStream_t s);
cudaError_t launch_dq_single(const void* codes, int fmt, int64_t n, const float* scale_inv,
                             float* dst, cudaStream_t s);
int num_sms();

// Launch policy of the current API call (thread-local, set by LaunchScope in api.cpp):
// max_ctas > 0 caps every grid (loopback); plain = no cooperative / PDL attributes.
struct LaunchPolicy {
  int max_ctas = 0;
  bool plain = false;
};
LaunchPolicy& launch_policy();
struct LaunchScope {
  LaunchPolicy saved;
  explicit LaunchScope(const fp8lm_plan* p);
  ~LaunchScope() { launch_policy() = saved; }
};

// CUDA-graph capture of a step (kernels.cu): the log of the captured AdamArgs launches
struct GraphAdamLog;
GraphAdamLog* adam_log_new();
void adam_log_free(GraphAdamLog* l);
void adam_log_activate(GraphAdamLog* l);      // thread-local; nullptr = off
size_t adam_log_size(const GraphAdamLog* l);
cudaError_t adam_log_update(const GraphAdamLog* l, cudaGraphExec_t exec, const fp8lm_adam_hp& hp,
                            int hist_slot);

// the peer-wait watchdog of every compilation unit that spins on peer flags (device.cuh)
cudaError_t wait_watchdog_set_kernels(unsigned long long ns, uint32_t* report);
cudaError_t wait_watchdog_set_sp(unsigned long long ns, uint32_t* report);
// load the code of every kernel a peer-mode step can launch (see kernels.cu)
cudaError_t preload_kernels();
}  // namespace fp8lm
