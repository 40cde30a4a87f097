/*
 * fp8lm.h — C ABI of the FP8-LM data-parallel hot path on B200 (sm_100a).
 *
 * FP8-LM (arXiv 2310.18313), PAPER.md:
 *   §2.1 "FP8 Gradient and All-Reduce Communication"  P:95-142  (Eq. 3-6)
 *   §2.2 "FP8 Optimizer"                              P:146-179 (Eq. 7-8)
 *   §2.3 FP8 ZeRO, Alg. 1
 *   App. A FP8 formats, Table 5
 *   App. B JIT / delayed tensor scaling
 * Readings of ambiguous passages are numbered R1..R24 in DESIGN.md §3.
 *
 * CONVENTIONS (apply to every call)
 *   - Pointers are DEVICE pointers unless the parameter says "host".
 *   - The caller owns all memory (PyTorch allocates it).  The library allocates
 *     nothing on the hot path; it owns only plan / communicator objects.
 *   - Every device-side call is asynchronous on `stream` (a cudaStream_t; NULL =
 *     legacy default stream) and performs no host synchronisation.
 *   - Return value: FP8LM_OK (0) or a negative fp8lm_status.  Argument errors are
 *     detected on the host and returned before anything is enqueued.  CUDA / NCCL
 *     launch errors return FP8LM_ECUDA / FP8LM_ENCCL.  fp8lm_last_error() gives a
 *     thread-local message.  Nothing throws across the ABI.
 *   - A non-finite gradient is NOT an error: it sets the device flag *skip = 1,
 *     the optimizer step becomes a no-op and mu halves (R14).
 *
 * FLAT LAYOUT ("plan")
 *   A plan describes T tensors (numel[t]) packed into flat buffers, tensor t at
 *   element offset fp8lm_plan_offset(t) (a multiple of FP8LM_ALIGN_ELEMS).  The
 *   gradient buffer (fp32 or bf16), the E4M3 gradient codes and every optimizer
 *   state buffer use the same element offsets (DDP-bucket style: autograd writes
 *   into views of the flat gradient buffer).  Per-tensor scalars are arrays [T].
 *
 * SCALING TENSORS ("(g'_i, s'_i) ... The actual weight gradient is g'_i/s'_i")
 *   logical value = decode(code) * scale_inv, with scale_inv = fl(1/scale)  (R8).
 */
#ifndef FP8LM_H
#define FP8LM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP8LM_ABI_VERSION 1
#define FP8LM_ALIGN_ELEMS 64      /* tensor offsets in flat buffers are multiples of this */
#define FP8LM_MAX_SIM_RANKS 16    /* simulated ranks on one device (config C1) */

typedef enum {
  FP8LM_OK = 0,
  FP8LM_EINVAL = -1,        /* bad argument (host-side check)               */
  FP8LM_ECUDA = -2,         /* CUDA runtime / launch error                   */
  FP8LM_ENCCL = -3,         /* NCCL error                                    */
  FP8LM_EWORKSPACE = -4,    /* workspace missing / too small / plan unbound  */
  FP8LM_EUNSUPPORTED = -5   /* built without NCCL, or unsupported dtype     */
} fp8lm_status;

typedef enum {
  FP8LM_E4M3 = 0,   /* App. A: S1E4M3, bias 7, max 448, NaN = S.1111.111, no inf  */
  FP8LM_E5M2 = 1,   /* App. A: S1E5M2, bias 15, max 57344, inf, NaN              */
  FP8LM_F16 = 2,
  FP8LM_BF16 = 3,
  FP8LM_F32 = 4
} fp8lm_dtype;

typedef enum {
  FP8LM_MODE_LOCAL = 0,      /* nranks must be 1: one process, one GPU, no exchange     */
  FP8LM_MODE_SIMULATED = 1,  /* nranks simulated ranks whose gradients all live on this
                                device (config C1); the exchange is a local read       */
  FP8LM_MODE_NCCL = 2,       /* one process per GPU; exchange over NCCL (NVLink)       */
  FP8LM_MODE_P2P = 3,        /* one process per GPU; the exchange runs inside this
                                library's kernels over NVLink peer memory (CUDA IPC
                                windows of fp8lm_peer_setup); NCCL only bootstraps      */
  FP8LM_MODE_ZERO = 4        /* P2P transport with FP8 ZeRO whole-tensor ownership (Alg. 1,
                                P:206-237): tensor t is reduced and optimised only by its
                                owner, which then writes w8 + scale into every rank    */
} fp8lm_mode;

#define FP8LM_MAX_P2P_RANKS 8     /* ranks of one NVLink / NVSwitch domain in mode P2P */

typedef struct fp8lm_plan fp8lm_plan;   /* opaque */
typedef struct fp8lm_comm fp8lm_comm;   /* opaque: owns an ncclComm_t */

/* A set of T scaling tensors in one flat buffer (D1/D4 of SURVEY §2.2).
 * data: flat codes (uint8 for E4M3, uint16 for FP16) at the plan's offsets.
 * scale / scale_inv / amax: device float[T]. */
typedef struct {
  void* data;
  float* scale;
  float* scale_inv;
  float* amax;
} fp8lm_stensors;

/* AdamW scalars for one step (P:301 beta1 = 0.9, beta2 = 0.95, weight decay 0.1;
 * eps, bias correction R15).  Each field is computed on the host in double and
 * rounded once to float (R24) — see fp8lm_adam_hp_make. */
typedef struct {
  float beta1, beta2;
  float one_minus_beta1, one_minus_beta2;
  float eps;
  float decay;          /* fl(1 - lr * weight_decay)            */
  float step_size;      /* fl(lr / (1 - beta1^step))             */
  float inv_bc2_sqrt;   /* fl(1 / sqrt(1 - beta2^step))          */
} fp8lm_adam_hp;

/* ------------------------------------------------------------------ misc (host) */
int fp8lm_version(void);                       /* FP8LM_ABI_VERSION */
const char* fp8lm_last_error(void);            /* thread-local message of the last failure */
int fp8lm_has_nccl(void);                      /* 1 if built with NCCL */

/* Host: fill *out (host) from the hyper-parameters; step >= 1.  EINVAL on step < 1 or
 * non-finite inputs. */
int fp8lm_adam_hp_make(double lr, double beta1, double beta2, double eps,
                       double weight_decay, int64_t step, fp8lm_adam_hp* out);

/* Host: Alg. 1 "Greedy Distribution Algorithm for ZeRO".  numels [T]
 * (host) are the tensor sizes c_i; owner_out [T] (host) receives the GPU of each
 * tensor; load_out [nranks] (host) the loads u_j.  Ties: stable sort by ascending
 * index, argmin by lowest device (R21).  EINVAL if nranks < 1 or T < 0. */
int fp8lm_zero_plan(int32_t T, const int64_t* numels, int32_t nranks,
                    int32_t* owner_out, int64_t* load_out);

/* ------------------------------------------------------------- communicator (NCCL) */
/* Host: ncclGetUniqueId into id_out[128] (host).  Rank 0 calls it and broadcasts the
 * bytes with torch.distributed (plumbing). */
int fp8lm_comm_unique_id(uint8_t* id_out);
/* Host: ncclCommInitRank on the CURRENT CUDA device.  *out receives the handle. */
int fp8lm_comm_init(int32_t nranks, int32_t rank, const uint8_t* id, fp8lm_comm** out);
/* Host: wrap an EXISTING NCCL communicator — e.g. torch.distributed's own, from
 * ProcessGroupNCCL._comm_ptr() (one communicator per process, shared with
 * the framework) — without taking ownership: fp8lm_comm_destroy then only frees the
 * wrapper.  nccl_comm is an ncclComm_t of the NCCL library this one links (the torch-
 * bundled libnccl.so.2, the same one torch loads); nranks / rank must match its count
 * and rank (checked with ncclCommCount / ncclCommUserRank: EINVAL otherwise). */
int fp8lm_comm_attach(void* nccl_comm, int32_t nranks, int32_t rank, fp8lm_comm** out);
int fp8lm_comm_destroy(fp8lm_comm* comm);

/* --------------------------------------------------------------------- the plan */
/* Host: build the flat layout, chunk tables and (mode NCCL) the reduce-scatter shard
 * map for T tensors.  numels (host) [T], each >= 0.  nranks >= 1; rank in [0,nranks)
 * (ignored unless mode == NCCL).  EINVAL on bad arguments. */
int fp8lm_plan_create(int32_t T, const int64_t* numels, int32_t mode, int32_t nranks,
                      int32_t rank, fp8lm_plan** out);
int fp8lm_plan_destroy(fp8lm_plan* plan);
int64_t fp8lm_plan_offset(const fp8lm_plan* plan, int32_t t);  /* element offset of tensor t, -1 if bad */
int64_t fp8lm_plan_total(const fp8lm_plan* plan);              /* elements of every flat buffer */
int64_t fp8lm_plan_g8_bytes(const fp8lm_plan* plan);           /* bytes of the reduced-code buffer g8
                                                                  (>= total; N*S in mode NCCL) */
int64_t fp8lm_plan_shard_bytes(const fp8lm_plan* plan);        /* S: bytes each rank reduces (NCCL) */
int64_t fp8lm_plan_shard_begin(const fp8lm_plan* plan, int32_t rank); /* = rank * S */
size_t fp8lm_plan_workspace_bytes(const fp8lm_plan* plan);
/* Upload the plan's tables into the caller-owned device workspace `ws` (>=
 * fp8lm_plan_workspace_bytes, 256-byte aligned) and zero its accumulators on
 * `stream`; synchronises `stream` before returning (one-time setup, host tables are
 * pageable).  Must precede every call below that takes the plan.
 * EWORKSPACE if ws is NULL / too small / misaligned. */
int fp8lm_plan_bind(fp8lm_plan* plan, void* ws, size_t ws_bytes, void* stream);

/* Mode ZERO: owner of tensor t (Alg. 1 with the R21 ties), its element offset in this
 * rank's COMPACT layout of owned tensors (-1 if another rank owns it), and the elements
 * of that compact layout (the size of the owned g8 / m1 / v / master / w8 buffers).
 * In mode ZERO the per-tensor state arrays (scale, scale_inv, amax) are indexed by the
 * owned-tensor ordinal j = 0..fp8lm_plan_owned_count-1 (owned tensors in ascending t). */
int32_t fp8lm_plan_owner(const fp8lm_plan* plan, int32_t t);
int64_t fp8lm_plan_owned_offset(const fp8lm_plan* plan, int32_t t);
int64_t fp8lm_plan_owned_total(const fp8lm_plan* plan);
int32_t fp8lm_plan_owned_count(const fp8lm_plan* plan);

/* Mode P2P, collective (every rank, after fp8lm_plan_bind): allocate this rank's
 * symmetric windows — the quantized send buffer (N*S bytes), the reduced-code buffer
 * g8 (N*S bytes) and a small signal / exchange pad — exchange their CUDA IPC handles over
 * `comm` (ncclAllGather) and map every peer's windows.  The windows are owned by the
 * plan (freed by fp8lm_plan_destroy): the one exception to "the caller owns all memory".
 * Synchronous.  EINVAL unless mode == P2P and comm matches the plan; ECUDA / ENCCL on
 * failure. */
int fp8lm_peer_setup(fp8lm_plan* plan, fp8lm_comm* comm, void* stream);
/* Single-process loopback of modes P2P / ZERO (tests, and any host that drives several
 * logical ranks on one GPU): plans[r] (r = 0..n-1) are n bound plans of one process,
 * created with the same numels and mode (P2P or ZERO), nranks = n and rank = r.  Each
 * gets its windows as in fp8lm_peer_setup, but the peer table points at the other
 * plans' local windows (no IPC, no communicator).  The ranks then run the same call
 * sequence, each on its OWN stream (the kernels meet at the same flags as over NVLink,
 * so the n ranks' launches must be able to run concurrently); every kernel of a
 * loopback plan launches at most floor(#SMs / n) CTAs and without the cooperative / PDL
 * attributes, so that all ranks' kernels are resident together.  Same arithmetic and
 * bit-identical results as n processes; not a performance configuration.  Synchronous.
 * EINVAL on mismatched plans or a plan already set up. */
int fp8lm_peer_setup_loopback(fp8lm_plan* const* plans, int32_t n, void* stream);

/* Peer-wait watchdog (modes P2P / ZERO and the SP converter).  The kernels that meet
 * other ranks spin on epoch flags in the peers' pads.  A flag still behind its epoch
 * after `seconds` (default 600: a peer may save a checkpoint or evaluate between steps)
 * makes the waiting kernel record {1, flag index, epoch wanted, value seen} in a
 * host-mapped report and trap (a sticky CUDA error: the job must restart, as after an
 * NCCL timeout).  seconds = 0: wait forever.  Applies to kernels launched after the
 * call; EINVAL on a negative / non-finite value.  fp8lm_peer_timeout_report copies the
 * report (all zero if no wait timed out); readable after the trap. */
int fp8lm_set_peer_timeout(double seconds);
int fp8lm_peer_timeout_report(uint32_t* out4);

/* Mode P2P, small messages: a plan whose reduced-code buffer (fp8lm_plan_g8_bytes) is at
 * most max_bytes (default 1 MiB; 0 = never) exchanges with the ONE-SHOT kernel instead of
 * quantize + reduce-scatter + all-gather: it quantizes into the own send window, meets the
 * ranks at one flag, and every rank pulls and reduces the whole set from every rank
 * (rank order, R12) — the same results with one kernel and one cross-rank handshake,
 * (N-1) n bytes of NVLink per rank instead of 2 (N-1)/N n (config C5's small sizes).
 * fp8lm_grad_allreduce and fp8lm_dp_step (not the split step); every rank must set the
 * same value.  Host call; EINVAL on a NULL plan or a negative size. */
int fp8lm_plan_set_oneshot(fp8lm_plan* plan, int64_t max_bytes);

/* Mode P2P, the smallest messages: a one-shot plan whose code buffer is at most max_bytes
 * (default 1 MiB / (4 (N-1)): 256 KiB at N = 2, 85 KiB at N = 4 — where it measured faster;
 * 0 = never; effective only for plans of at most 1 MiB, whose send
 * window fp8lm_peer_setup sizes for it) runs fp8lm_allreduce_jit / fp8lm_dp_step with the
 * RAW one-shot kernel: each rank copies its gradient (fp32 / bf16 as given) into its send
 * window during the amax pass, the Eq. 4 MIN handshake publishes the copy with the scale,
 * and every rank pulls every rank's gradient and encodes it itself with s_g (Eq. 5 — the
 * same codes) before the rank-order sum: one cross-rank handshake and no quantize pass,
 * for (N-1) n sizeof(src) bytes of NVLink per rank.  Same results bit for bit.  Every rank
 * must set the same value.  Host call; EINVAL on a NULL plan or a negative size. */
int fp8lm_plan_set_oneshot_raw(fp8lm_plan* plan, int64_t max_bytes);

/* Mode P2P: this rank's g8 window (device); pass it as g8 to the calls below.  NULL if
 * fp8lm_peer_setup has not run. */
uint8_t* fp8lm_peer_g8(const fp8lm_plan* plan);
/* Mode ZERO (also set up by fp8lm_peer_setup): the replicated FP8 weight copy of ALL
 * tensors in the full layout (every owner writes its tensors' w8 codes here on every
 * rank) and its per-tensor scalars, three device float[T] rows: scale, scale_inv, amax. */
uint8_t* fp8lm_peer_w8(const fp8lm_plan* plan);
float* fp8lm_peer_w8_scalars(const fp8lm_plan* plan);

/* ------------------------------------------- (1) fp8_quantize: one scaling tensor */
/* App. B JIT scaling + App. A encode.  src: n elements of src_dtype (F32 or BF16),
 * any alignment.  fmt: E4M3 or E5M2 (codes to dst, uint8[n]) or F16 (uint16[n]).
 * jit = 1: amax = max|src| -> *amax, scale = fl(fmt_max / amax) (1 if amax is 0 or
 *          the ratio overflows) -> *scale, *scale_inv = fl(1/scale), then encode.
 * jit = 0: use the scale already in *scale (amax not written).
 * Encode: code = satRNE(fl(src * scale)) (R11: saturating round-to-nearest-even).
 * sat_count (nullable): += number of codes whose magnitude is the format max. */
int fp8lm_quantize(const void* src, int32_t src_dtype, int64_t n, int32_t fmt, void* dst,
                   float* scale, float* scale_inv, float* amax, int32_t jit,
                   uint32_t* sat_count, void* stream);
/* dst[i] = fl(decode(codes[i]) * (*scale_inv)), fp32 output. */
int fp8lm_dequantize(const void* codes, int32_t fmt, int64_t n, const float* scale_inv,
                     float* dst, void* stream);

/* ---------------------------- (2) amax_scale_sync: Eq. 3-4, A1 + A2 */
/* grads: flat gradient buffer (src_dtype F32 or BF16) in plan layout.  In mode
 * SIMULATED, grads is a HOST array of nranks device pointers (one flat buffer per
 * simulated rank) cast to const void*; otherwise it is the device pointer itself.
 *   amax_r[t] = max_i |g_r[t][i]|                 -> amax_out [T] (SIMULATED: [nranks*T],
 *                                                   rank-major); NaN/inf propagate (R14)
 *   s_r[t]    = fl(fl(448 / amax_r[t]) * mu[t])   (0 if non-finite, +inf if amax == 0)
 *   s_g[t]    = min_r s_r[t]  (Eq. 4; NCCL: ncclAllReduce MIN over `comm`)
 *   s_g == 0 -> *skip = 1;  s_g == +inf -> s_g = 1.         -> s_g [T], skip [1]
 * mu [T] is read only.  comm must be non-NULL iff mode == NCCL.  Mode P2P: the MIN over
 * ranks is exchanged through the peers' pads by the amax kernel's last CTA (comm unused,
 * may be NULL). */
int fp8lm_amax_scale_sync(fp8lm_plan* plan, fp8lm_comm* comm, const void* grads,
                          int32_t src_dtype, const float* mu, float* amax_out,
                          float* s_g, int32_t* skip, void* stream);

/* ----------------------------- (3) fp8_grad_allreduce: Eq. 5-6, A3-A5 */
/* c_r = E4M3(fl(g_r * s_g))  (quantized once from FP32, R9)
 * S   = sum over r = 0..N-1 of decode(c_r), binary32, rank order (exact, R12)
 * g8  = E4M3(S): the reduced codes, on every rank (reduce-scatter + all-gather, NCCL)
 * g_scale[t] = fl(N * s_g[t]) (Eq. 6), g_scale_inv[t] = fl(1 / g_scale[t])
 * sat[t]     = #{i : |decode(g8[t][i])| == 448}  ("attains the maximum", R4)
 * mu[t]     <- mu_next: halve if *skip or sat*1e5 > numel[t], else min(2, fl(mu*2^(1/1000)))
 *              (R1-R3) — updated in place for the next step.
 * grads as in (2).  g8: fp8lm_plan_g8_bytes bytes.  All outputs are device arrays [T].
 * Mode P2P: g8 must be fp8lm_peer_g8(plan); one kernel reads every rank's quantized
 * shard over NVLink, reduces in rank order and stores the result into every rank's g8
 * (reduce-scatter + all-gather fused), with sys-scope flag barriers in the peers' pads.
 * Mode ZERO: g8 is this rank's COMPACT buffer (fp8lm_plan_owned_total bytes); every
 * rank's quantize pushes each code into its owner's window (slot = the rank, in the
 * owner's compact layout) and the owner reduces its whole tensors from those N local
 * slots (no all-gather: only the owner needs them).  sat / mu / g_scale / g_scale_inv stay
 * full [T] arrays, replicated on every rank. */
int fp8lm_grad_allreduce(fp8lm_plan* plan, fp8lm_comm* comm, const void* grads,
                         int32_t src_dtype, const float* s_g, const int32_t* skip,
                         uint8_t* g8, float* g_scale, float* g_scale_inv, uint32_t* sat,
                         float* mu, void* stream);

/* (2) + (3) in one call: fp8lm_amax_scale_sync then fp8lm_grad_allreduce, same
 * arguments and results.  Mode P2P with a small plan (fp8lm_plan_set_oneshot): ONE kernel
 * — amax, the Eq. 4 MIN through the pads, the one-shot exchange — one launch and two
 * cross-rank handshakes per step (config C5's small messages); one handshake for the
 * smallest plans (fp8lm_plan_set_oneshot_raw).  Other modes / sizes: the
 * two calls. */
int fp8lm_allreduce_jit(fp8lm_plan* plan, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                        float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                        float* g_scale, float* g_scale_inv, uint32_t* sat, void* stream);

/* --------------------------------- (4) fp8_adam_step: §2.2, A6 + A7 */
/* Precision-decoupled AdamW on every tensor of the plan, JIT state scaling (R18):
 *   g  = fl(decode(g8) * g_scale_inv[t])        (dequantize, A6)
 *   m  = fl(decode_e4m3(m1) * m1.scale_inv[t]);  v = fl(f16(v) * v.scale_inv[t]);
 *   w  = fl(f16(master) * master.scale_inv[t])
 *   m' = fl(fl(b1 m) + fl(omb1 g));  v' = fl(fl(b2 v) + fl(fl(omb2 g) g))
 *   u  = fl(m' / fl(fl(sqrt(v') * inv_bc2_sqrt) + eps));  w' = fl(fl(w decay) - fl(step_size u))
 *   new scales from the exact amax of m', v', w' (pass 1), then encode (pass 2):
 *   m1 <- E4M3(fl(m' * 448/A_m)),  v <- F16(fl(v' * 65504/A_v)),
 *   master <- F16(fl(w' * 65504/A_w)),  w8 <- E4M3(fl(w' * 448/A_w))
 *   (scale = 1 where the amax is 0); each stensor's scale/scale_inv/amax updated.
 * If *skip != 0 nothing changes.  hp is a HOST pointer.  m1/w8 data: uint8 flat,
 * v/master data: uint16 (FP16 bits) flat, all at the plan's offsets.
 * Mode ZERO: g8 and the four states are COMPACT (owned tensors only, scalars indexed
 * by the owned ordinal; g_scale_inv is the full [T] array); after the update every
 * owner stores its tensors' w8 codes and scalars into every rank's fp8lm_peer_w8 /
 * fp8lm_peer_w8_scalars (collective: returns once all ranks' copies have landed). */
int fp8lm_adam_step(fp8lm_plan* plan, const uint8_t* g8, const float* g_scale_inv,
                    const fp8lm_stensors* m1, const fp8lm_stensors* v,
                    const fp8lm_stensors* master, const fp8lm_stensors* w8,
                    const fp8lm_adam_hp* hp, const int32_t* skip, void* stream);

/* Delayed state scaling (App. B: "maximum absolute values observed in a certain
 * number of preceding iterations"; readings R25-R27): ONE AdamW pass, 12 B/param
 * instead of 18.  The new scales are fixed before the update: m1 and v from a-priori
 * bounds on |m'| and v' (they never saturate), master (16x headroom) and w8 from the
 * maximum of w_hist; the exact new amaxes are still recorded and amax(w') is written
 * into slot hist_slot of w_hist.  w_hist: device float[16 * T] (ring of exact amax(w')
 * values, slot-major; start it with amax(w0) in slot 0 and zeros elsewhere);
 * hist_slot = (step - 1) % 16.  Mode ZERO: w_hist and states are compact (owned). */
int fp8lm_adam_step_delayed(fp8lm_plan* plan, const uint8_t* g8, const float* g_scale_inv,
                            const fp8lm_stensors* m1, const fp8lm_stensors* v,
                            const fp8lm_stensors* master, const fp8lm_stensors* w8,
                            const fp8lm_adam_hp* hp, const int32_t* skip, float* w_hist,
                            int32_t hist_slot, void* stream);

/* ------------------------------------------------ the whole data-parallel step */
/* (2) + (3) + (4) in one call, with the fusions the separate calls cannot express;
 * results are bit-identical to calling fp8lm_amax_scale_sync, fp8lm_grad_allreduce and
 * fp8lm_adam_step in sequence (same arguments).  Mode LOCAL: the codes of A3 are final
 * (N = 1), so the quantize kernel also runs Adam pass 1 on them (4 launches per step,
 * 26 B/param instead of 27).  Mode P2P: the quantize pushes every 16-code group into
 * slot `rank` of its shard owner's send window (the reduce-scatter's NVLink transfer
 * rides on the quantize pass); the exchange kernel runs Adam pass 1 on the
 * elements of its own shard (1/N of pass 1 per rank) and combines the ranks' partial
 * state maxima through the pads; the all-gather (A5) is a PULL inside pass 2 (delayed
 * state scaling: inside the single pass), which reads each code from its owner's g8
 * window over NVLink while it streams the local states.
 * So after a P2P dp_step, g8 (this rank's window) holds the reduced codes of this
 * rank's shard [fp8lm_plan_shard_begin(rank), +shard bytes) only — every other result
 * (scales, sat, mu, the four states) is bit-identical to the three calls; use
 * fp8lm_grad_allreduce for a fully gathered g8.  Other modes: the three calls in sequence.
 * w_hist != NULL selects delayed state scaling (fp8lm_adam_step_delayed semantics); in
 * mode LOCAL the quantize kernel then also runs the single AdamW pass (20 B/param).
 * Mode ZERO: the owner's pass 2 also broadcasts w8 (+ scalars) into every rank's window
 * (JIT; delayed state scaling runs the three calls). */
int fp8lm_dp_step(fp8lm_plan* plan, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                  float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                  float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                  const fp8lm_stensors* v, const fp8lm_stensors* master,
                  const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                  int32_t hist_slot, void* stream);

/* The P2P / ZERO step in two phases, so that the exchange of one bucket of tensors runs
 * beside the HBM passes of another (the exchange overlaps compute; f2).  A bucket
 * is a plan over a subset of the tensors (its own windows, flags and epochs).  phase 1:
 * amax + scale MIN + quantize on `stream`, then the exchange kernel (reduce-scatter +
 * rank-order reduce + Adam pass 1 on the own shard; ZERO: the owner reduce + pass 1) on
 * the plan's own high-priority exchange stream (ZERO: followed there by the owner's pass 2
 * + w8 broadcast, NVLink-bound); phase 2: `stream` waits for that
 * exchange, then (P2P) the AdamW pass with the pulled all-gather.  A
 * caller with buckets b = 0..B-1 issues phase 1 for every bucket, then phase 2 for every
 * bucket: the exchange of bucket b overlaps the amax / quantize of b+1 and pass 2 of b-1.
 * Same arguments and results as fp8lm_dp_step (comm unused: modes P2P / ZERO only; ZERO
 * JIT only).  EINVAL on another mode or when phases do not alternate 1, 2, 1, 2, ...
 * Every rank must issue the same sequence (the phases are collective). */
int fp8lm_dp_step_split(fp8lm_plan* plan, int32_t phase, const void* grads, int32_t src_dtype,
                        float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                        float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                        const fp8lm_stensors* v, const fp8lm_stensors* master,
                        const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                        int32_t hist_slot, void* stream);

/* fp8lm_dp_step as a CUDA graph: same arguments and results.  The first call with a set
 * of buffers runs eagerly; the second captures the step on `stream`
 * (cudaStreamCaptureModeThreadLocal), instantiates and launches the graph; later calls
 * patch the step's scalars (hp, hist_slot) into the graph's AdamW kernel nodes and
 * relaunch it — one host call and no per-kernel launch work per step.  Every other
 * per-step value is device-resident (μ, scales, the P2P / ZERO flag epochs in the pads).
 * A graph belongs to one set of pointers (grads, outputs, states, w_hist, comm, stream)
 * and dtype; the plan keeps the 4 most recently used (callers that rotate gradient
 * buffers).  Mode NCCL: plain fp8lm_dp_step.  The caller must not capture `stream`
 * itself around this call. */
int fp8lm_dp_step_graphed(fp8lm_plan* plan, fp8lm_comm* comm, const void* grads, int32_t src_dtype,
                          float* mu, float* amax_out, float* s_g, int32_t* skip, uint8_t* g8,
                          float* g_scale, float* g_scale_inv, uint32_t* sat, const fp8lm_stensors* m1,
                          const fp8lm_stensors* v, const fp8lm_stensors* master,
                          const fp8lm_stensors* w8, const fp8lm_adam_hp* hp, float* w_hist,
                          int32_t hist_slot, void* stream);

/* Initial optimizer state: m1, v = zero codes with scale 1,
 * amax 0; master / w8 JIT-encoded from the FP32 flat weights w0 (plan layout).
 * Mode ZERO: w0 and the states are COMPACT (owned tensors); the replicated w8 copy is
 * then broadcast as after a step (collective). */
int fp8lm_state_init(fp8lm_plan* plan, const float* w0, const fp8lm_stensors* m1,
                     const fp8lm_stensors* v, const fp8lm_stensors* master,
                     const fp8lm_stensors* w8, void* stream);

/* ------------------------------------------------------- launch tracing (auxiliary) */
/* Host: when enabled, every kernel, memset and NCCL call the library enqueues is
 * bracketed by CUDA events on its stream.  fp8lm_prof_enable(1) starts a new window
 * (clears records), (0) stops recording.  fp8lm_prof_ids() = number of trace ids;
 * fp8lm_prof_read(id, ...) synchronises the recorded events and returns the name,
 * number of launches and summed device milliseconds of that id, and whether it is a
 * kernel of this library (is_ours = 1) rather than a memset / NCCL collective. */
int fp8lm_prof_enable(int on);
int fp8lm_prof_ids(void);
int fp8lm_prof_read(int32_t id, const char** name, int64_t* launches, double* total_ms,
                    int32_t* is_ours);

/* ------------------- (7) FP8 all-reduce strategies and Fig. 6 statistics (f3) */
/* PAPER.md §2.1 P:102-121 compares three ways to aggregate FP8 gradients over N ranks:
 * pre-scaling (Eq. 1, g = g_1/N + ... + g_N/N), post-scaling (Eq. 2, (g_1 + ... + g_N)/N)
 * and automatic scaling (Eq. 3-6, the method); Fig. 6 reports their SNR,
 * underflow rate and overflow rate.  Readings R28-R30:
 *   s = Eq. 4's shared scale = fl(fl(448 / A) * mu), A = max over ranks and elements of
 *       |g|, mu = *mu for AUTO and 1 for PRE / POST (1 if A = 0 or 448/A overflows)
 *   PRE   c_r = E4M3(fl(fl(g_r * s) / N)), result scale s
 *   POST  c_r = E4M3(fl(g_r * s)),          result scale fl(N * s)
 *   AUTO  as POST with mu; *mu <- the mu update (R1-R3) from the result's saturation
 *   then S = rank-order binary32 sum of decode(c_r), code = E4M3(S) (all three)
 *   events = (N + 1) n encodes; underflow: nonzero input -> zero code; overflow: |input|
 *   > 448; sig2 = sum m^2, err2 = sum (g_hat - m)^2 in binary64, m = binary64 rank-order
 *   mean of g_r, g_hat = fl(decode(code) * fl(1 / result scale)); SNR = 10 log10(sig2/err2).
 * grads: device, N rows of n binary32 values (row r = rank r), contiguous, any alignment.
 * mu: device float[1], read by AUTO and replaced by the next step's mu (untouched by PRE
 * and POST).  codes: device uint8[n] (the aggregated E4M3 codes) or NULL.  stats: device
 * fp8lm_commstats, zero-initialised once by the caller; every call overwrites its
 * outputs and returns its scratch fields to zero.  Non-finite gradients are not supported
 * (s = 0: the statistics are then meaningless).  Asynchronous on `stream`; EINVAL on bad
 * arguments (strategy, N < 1, n < 0, NULL pointers). */
#define FP8LM_STRATEGY_PRE 0
#define FP8LM_STRATEGY_POST 1
#define FP8LM_STRATEGY_AUTO 2
typedef struct {
  double sig2;             /* sum over elements of m^2 */
  double err2;             /* sum over elements of (g_hat - m)^2 */
  uint64_t underflow;      /* encodes of a nonzero input that gave a zero code */
  uint64_t overflow;       /* encodes whose input magnitude exceeded 448 */
  uint64_t events;         /* (N + 1) * n */
  uint32_t sat;            /* result codes attaining 448 (the mu statistic, R4) */
  uint32_t nonfinite;      /* 1 if any input was inf / NaN */
  float amax;              /* A */
  float s;                 /* the shared scale used for the rank encodes */
  float scale;             /* result scale (s for PRE, fl(N s) otherwise) */
  float scale_inv;         /* fl(1 / scale) */
  float mu_used;
  float mu_next;
  uint32_t scratch[4];     /* internal accumulators / tickets: zero at rest */
} fp8lm_commstats;
int fp8lm_allreduce_strategy(int32_t strategy, const float* grads, int32_t nranks, int64_t n,
                             float* mu, uint8_t* codes, fp8lm_commstats* stats, void* stream);
/* Host: the Fig. 6 metrics of one fp8lm_commstats already copied to the host (R29-R30):
 * out3[0] = SNR in dB = 10 log10(sig2 / err2) (+inf if err2 = 0 < sig2, NaN if both are
 * 0, -inf if sig2 = 0 < err2); out3[1] = underflow rate = underflow / events; out3[2] =
 * overflow rate = overflow / events (0 when events = 0).  EINVAL on NULL pointers. */
int fp8lm_commstats_metrics(const fp8lm_commstats* host_stats, double* out3);

/* ------------------ (8) FP8 sequence/tensor-parallel activation converter g (f4) */
/* PAPER.md §2.3, Fig. 5: "We add an FP8 datatype conversion prior to g, such
 * that the all-gather (or reduce-scatter) operation uses FP8 low-bit activation to save
 * communication cost across GPUs."  Readings R31-R32:
 *   s = Eq. 4's shared scale over the ranks' inputs, mu = 1: min_r fl(448 / amax_r)
 *       (+inf for all-zero ranks; 1 if every rank is zero; 0 if any input is inf/NaN)
 *   all-gather (forward):  rank r holds x_r (m elements); every rank receives the
 *       gathered codes E4M3(fl(x_r * s)), rank-major (N m bytes), scale s;
 *       out = fl(decode(code) * fl(1/s)) in out_dtype (bf16: round-to-nearest-even)
 *   reduce-scatter (backward): rank r holds dy_r (N m elements); every rank quantizes
 *       E4M3(fl(dy_r * s)); rank k receives S = rank-order binary32 sum of chunk k of
 *       every rank's codes, out = fl(S * fl(1/s)) (no requantization, no mu)
 * Transport: NVLink peer memory between the ranks of `comm` (CUDA IPC windows owned by
 * the fp8lm_sp object), no NCCL call on the data path; 1 B per element crosses NVLink
 * instead of 2 for bf16.  Every call is COLLECTIVE: all ranks call the same sequence of
 * ops with the same m (ops are matched by a per-object counter), asynchronous on
 * `stream`; a rank that never arrives makes the others trap after the peer-wait
 * watchdog timeout (fp8lm_set_peer_timeout, default 600 s).
 *
 * fp8lm_sp_create: collective over comm (NULL = a single rank, no peers); max_elems
 * bounds N*m of every later op.  Allocates two windows of max_elems bytes and a 512-byte
 * pad per rank, exchanges IPC handles (ncclAllGather on `stream`, synchronised).  EINVAL
 * on bad arguments, ECUDA / ENCCL on failure.  fp8lm_sp_destroy: unmaps and frees.
 * fp8lm_sp_allgather: x (device, x_dtype F32 or BF16, m elements); codes_out (device
 * uint8[N m] or NULL); out (device [N m] of out_dtype F32 or BF16, or NULL); scale_out
 * (device float[2]: s, fl(1/s), or NULL).  The op is complete for this rank's readers
 * when the stream reaches its end (the kernels wait for every peer's data).
 * fp8lm_sp_reduce_scatter: dy (device, dtype F32 or BF16, N m elements: the full
 * tensor, chunk k = elements [k m, (k+1) m)); out (device [m] of out_dtype) receives
 * this rank's chunk of the sum; scale_out as above.
 * Sizes with m % 16 == 0 and 32-byte aligned inputs take the vector kernels; others
 * are correct but slower. */
typedef struct fp8lm_sp fp8lm_sp;   /* opaque */
int fp8lm_sp_create(fp8lm_comm* comm, int64_t max_elems, void* stream, fp8lm_sp** out);
int fp8lm_sp_destroy(fp8lm_sp* sp);
int fp8lm_sp_allgather(fp8lm_sp* sp, const void* x, int32_t x_dtype, int64_t m, uint8_t* codes_out,
                       void* out, int32_t out_dtype, float* scale_out, void* stream);
int fp8lm_sp_reduce_scatter(fp8lm_sp* sp, const void* dy, int32_t dtype, int64_t m, void* out,
                            int32_t out_dtype, float* scale_out, void* stream);

/* ----------------------------------------------------------- diagnostics (auxiliary) */
/* Device self-test of the branch-free IEEE sqrt / division fast paths used by the
 * AdamW kernels: every non-negative binary32 input for sqrt, `div_pairs` seeded
 * pseudo-random (a, b) pairs for division, each compared bit-for-bit with
 * __fsqrt_rn / __fdiv_rn wherever the fast path's range predicate accepts it.
 * out4 (host): {sqrt mismatches, sqrt inputs accepted, div mismatches, div pairs
 * accepted}.  Synchronous (allocates 32 bytes of device scratch; not a hot-path call). */
int fp8lm_selftest_fastmath(uint64_t div_pairs, uint64_t seed, uint64_t* out4);

#ifdef __cplusplus
}
#endif
#endif /* FP8LM_H */
