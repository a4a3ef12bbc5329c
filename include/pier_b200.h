/*
 * pier_b200.h -- C-ABI of the B200-native Pier optimizer hot path.
 *
 * Plain pointers, sizes and scalars; no torch types.  Device pointers point to
 * CUDA global memory; `stream` is a cudaStream_t passed as void* so the header
 * needs no CUDA include.  Every call is asynchronous on `stream` unless stated,
 * never allocates device memory (only the *_create / *_init / *_alloc_* setup
 * calls do -- a communicator maps its round signal block and norm slots into
 * every rank when it is created), never
 * throws, and returns 0 on success or a negative PIER_E* code; the message of
 * the last failure on the calling thread is in pier_last_error().
 *
 * The reference (Pier desk simulator, /root/reference/pkg/src/pier) is pure
 * NumPy; each entry point below cites the reference function it replaces.
 * Scalars arrive as double and are rounded to the array dtype on the host
 * exactly where the reference applies `dtype.type(...)` (optim.py:96-102,
 * 245, 271), so the f32 kernels are bitwise comparable with NumPy float32.
 */
#ifndef PIER_B200_H
#define PIER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define PIER_OK 0
#define PIER_EINVAL -1    /* bad size / pointer / alignment  -> ConfigError / ValueError */
#define PIER_ECUDA -2     /* CUDA runtime error                                           */
#define PIER_ENCCL -3     /* NCCL error                                                   */
#define PIER_EPROTOCOL -4 /* offload misuse (driver.py:136-146)  -> ProtocolError         */
#define PIER_ENOMEM -5    /* host / setup allocation failed                               */
#define PIER_EABORTED -6  /* a virtual group was aborted by a failing rank (driver.py:494-501) */

const char* pier_last_error(void);
int pier_version(void); /* 10000*major + 100*minor + patch */
int pier_device_sm_count(int device);
/* number of kernels this library has launched in the process (bench evidence) */
unsigned long long pier_launch_count(void);
/* cudaDeviceSynchronize with the library's error plumbing (a trapped round's
 * timeout record is appended to pier_last_error) */
int pier_device_sync(void);

/* ---- K1: pseudo-gradient  delta = theta - anchor -------------------------
 * replaces driver.py:415 (`theta_now - snapshot`) and driver.py:434
 * (`theta_avg - snapshot`).  256-bit (32-byte aligned) or 128-bit vector access. */
int pier_pseudograd_f32(const float* theta, const float* anchor, float* delta, int64_t n,
                        void* stream);
int pier_pseudograd_f64(const double* theta, const double* anchor, double* delta, int64_t n,
                        void* stream);

/* ---- a1: fold_momentum (optim.py:243-245)  out = (mu*mom) + delta -------- */
int pier_fold_momentum_f32(const float* mom, const float* delta, float* out, int64_t n,
                           double mu, void* stream);
int pier_fold_momentum_f64(const double* mom, const double* delta, double* out, int64_t n,
                           double mu, void* stream);

/* ---- a2: outer_step (optim.py:248-276), pure form --------------------------
 * mom_out = fold(mom, delta, mu); upd = lr*fold(mom_out, delta, mu);
 * theta_out = anchor ? anchor + (upd - delta) : snapshot + upd.
 * `anchor` may be NULL (snapshot form); outputs may alias nothing. */
int pier_outer_step_f32(const float* mom, const float* snapshot, const float* delta,
                        const float* anchor, float* theta_out, float* mom_out, int64_t n,
                        double lr, double mu, void* stream);
int pier_outer_step_f64(const double* mom, const double* snapshot, const double* delta,
                        const double* anchor, double* theta_out, double* mom_out, int64_t n,
                        double lr, double mu, void* stream);

/* ---- K3: fused outer update, one HBM pass (driver.py:428-440 after the mean)
 * avg = avg_or_sum / divisor (divisor 1: already averaged; the division is
 * the `acc /= n` of topology.py:121);  d = avg - anchor;
 * mom = mu*mom + d;  theta = avg + (lr*(mu*mom + d) - d);  anchor = theta.
 * `theta_out` may alias `avg_or_sum` (in-place on the reduced buffer). */
int pier_outer_update_f32(const float* avg_or_sum, float* anchor, float* mom, float* theta_out,
                          int64_t n, double lr, double mu, int32_t divisor, void* stream);
int pier_outer_update_f64(const double* avg_or_sum, double* anchor, double* mom,
                          double* theta_out, int64_t n, double lr, double mu, int32_t divisor,
                          void* stream);

/* ---- K3b: warmup fold (driver.py:412-420)  mom = mu*mom + (theta-anchor); anchor = theta */
int pier_warmup_fold_f32(const float* theta, float* anchor, float* mom, int64_t n, double mu,
                         void* stream);
int pier_warmup_fold_f64(const double* theta, double* anchor, double* mom, int64_t n, double mu,
                         void* stream);

/* ---- K6: ascending left-fold mean of up to 64 replicas (topology.py:104-122)
 * `parts` is a HOST array of `nparts` device pointers. out may alias parts[0]. */
#define PIER_MAX_PARTS 64
int pier_mean_left_fold_f32(const float* const* parts, int32_t nparts, float* out, int64_t n,
                            void* stream);
int pier_mean_left_fold_f64(const double* const* parts, int32_t nparts, double* out, int64_t n,
                            void* stream);

/* ---- K4a: global gradient norm + clip scale (optim.py:70-79) --------------
 * Writes a PierClip record at the start of the caller-owned device workspace
 * `ws` (pier_norm_ws_bytes() bytes, zero-initialised once).  Deterministic:
 * fixed partition, fp64 accumulation, fixed-order final sum. */
typedef struct PierClip {
    double sqnorm;   /* sum g^2, fp64 accumulation                          */
    double norm;     /* sqrt as the reference computes it (fp32 for f32)    */
    double scale;    /* dtype(max_norm/norm) if norm > max_norm else 1      */
    int32_t clipped; /* 1 iff norm > max_norm                               */
    int32_t nonfinite;
} PierClip;
size_t pier_norm_ws_bytes(void);
int pier_grad_sqnorm_f32(const float* g, int64_t n, double max_norm, void* ws, void* stream);
int pier_grad_sqnorm_f64(const double* g, int64_t n, double max_norm, void* ws, void* stream);
/* Recompute norm/scale/clipped from the record's sqnorm -- after the callers
 * summed the partial square sums of a replica's tensor-parallel shards into
 * it, so the clip stays GLOBAL over the replica (optim.py:76).  dtype_code
 * 0 = f32 rounding rules, 1 = f64. */
int pier_clip_finalize(void* ws, double max_norm, int32_t dtype_code, void* stream);
/* K4c: out = g * scale (the clipped copy of optim.py:78), scale from `ws` */
int pier_apply_clip_f32(const float* g, float* out, int64_t n, const void* ws, void* stream);
int pier_apply_clip_f64(const double* g, double* out, int64_t n, const void* ws, void* stream);

/* ---- K4b: fused AdamW (optim.py:82-103) with the clip applied in-flight ---
 * `step` is the NEW step count (state.step + 1).  `clip_ws` = workspace
 * written by pier_grad_sqnorm_* on the same stream, or NULL for no clip. */
typedef struct PierAdamW {
    double lr, beta1, beta2, eps, weight_decay;
    int64_t step;
} PierAdamW;
int pier_adamw_f32(float* theta, const float* g, float* m, float* v, int64_t n,
                   const PierAdamW* hp, const void* clip_ws, void* stream);
int pier_adamw_f64(double* theta, const double* g, double* m, double* v, int64_t n,
                   const PierAdamW* hp, const void* clip_ws, void* stream);
/* K5: one group (no exchange) at a boundary iteration: clip+AdamW then the
 * anchor-form outer step in ONE pass (driver.py:395-399 + :428-440 with
 * n = 1); bitwise equal to pier_adamw_* followed by pier_outer_update_*. */
int pier_adamw_outer_f32(float* theta, const float* g, float* m, float* v, float* anchor,
                         float* mom, int64_t n, const PierAdamW* hp, const void* clip_ws,
                         double outer_lr, double mu, void* stream);
int pier_adamw_outer_f64(double* theta, const double* g, double* m, double* v, double* anchor,
                         double* mom, int64_t n, const PierAdamW* hp, const void* clip_ws,
                         double outer_lr, double mu, void* stream);
/* bf16 live params with an fp32 master (7B config): master/m/v fp32, grad bf16;
 * writes master and its RNE bf16 copy in the same pass. */
int pier_adamw_bf16_f32(float* master, uint16_t* theta_bf16, const uint16_t* g_bf16, float* m,
                        float* v, int64_t n, const PierAdamW* hp, const void* clip_ws,
                        void* stream);
int pier_grad_sqnorm_bf16(const uint16_t* g, int64_t n, double max_norm, void* ws, void* stream);
/* refresh bf16 live params from the fp32 master after an outer step (RNE) */
int pier_cast_bf16(const float* src, uint16_t* dst, int64_t n, void* stream);

/* launch tuning of the streaming kernels on the calling thread.  ctas_per_sm
 * > 0 caps the grids at that many CTAs per SM (grid-stride loop); < 0 restores
 * the default, one tile per CTA (uncapped); 0 keeps the current value.
 * k5_unroll: K5's 256-bit vectors per thread per array (1 or 2; default 2;
 * <= 0 keeps). */
int pier_kernel_tune(int ctas_per_sm, int k5_unroll);

/* ---- multi-tensor (torch param lists; one launch over all tensors) ------- */
typedef struct PierTensorDesc {
    void* param;
    const void* grad;
    void* exp_avg;
    void* exp_avg_sq;
    int64_t numel;
} PierTensorDesc;
typedef struct PierTensorList PierTensorList;
/* setup call: uploads the chunk table once; dtype_code 0 = f32, 1 = f64 */
int pier_tensor_list_create(const PierTensorDesc* descs, int32_t ntensors, int32_t dtype_code,
                            PierTensorList** out);
int pier_tensor_list_destroy(PierTensorList* list);
int pier_grad_sqnorm_mt(const PierTensorList* list, double max_norm, void* ws, void* stream);
int pier_adamw_mt(const PierTensorList* list, const PierAdamW* hp, const void* clip_ws,
                  void* stream);

/* ---- outer-step schedule (optim.py:162-219), host-side, exact ------------ */
double pier_momentum_mu(int64_t t, int64_t total_iters);          /* < 0 on domain error */
int pier_outer_lr(int64_t t, int64_t total_iters, double* out);   /* EINVAL off-domain   */

/* ---- NCCL group communicator (one process per GPU, one group per GPU) ---- */
typedef struct PierComm PierComm;
int pier_nccl_unique_id_bytes(void);
int pier_nccl_get_unique_id(void* out);
/* Collective over all ranks: NCCL communicator + the persistent round's
 * signal block, the norm slots and a host-mapped timeout record, mapped into
 * every rank (CUDA IPC).  No later call allocates device memory implicitly. */
int pier_comm_init(const void* unique_id, int32_t rank, int32_t nranks, PierComm** out);
int pier_comm_destroy(PierComm* comm);
/* Virtual group: `nranks` (1..8) communicator handles out[0..n) for ranks
 * living on the CURRENT device, each driven by its own host thread -- the
 * reference's in-process groups (driver.py:476-529) on one B200.  Collectives
 * rendezvous on the host and order the ranks' streams with events instead of
 * NCCL; the P2P exchanges read/write the other ranks' buffers on the same
 * device; the persistent round runs ONE cooperative launch for all ranks.
 * NCCL-only entry points (bucketed RS/AG, NCCL means, NVLS) return EINVAL. */
int pier_vgroup_create(int32_t nranks, PierComm** out);
/* a failing rank's thread aborts the group: every rank blocked in (or later
 * entering) a collective returns PIER_EABORTED (driver.py:494-501) */
int pier_vgroup_abort(PierComm* any_rank);
int pier_comm_is_virtual(const PierComm* comm);
/* spin limit of the persistent round's waits (default 20 s or
 * PIER_ROUND_TIMEOUT_S); on expiry the kernel records what it waited on and
 * traps; pier_last_error of the failing call then names the rank and counter */
int pier_comm_set_timeout(PierComm* comm, double seconds);
/* the timeout record: {flag, team rank, span, observed, target, kind (0 ready,
 * 1 done), peer} (flag 1 = a wait timed out) */
int pier_comm_diag(const PierComm* comm, uint32_t* out7);
/* Mode B outer step: per bucket b, in-place ReduceScatter(sum) of
 * theta[b*n*B .. (b+1)*n*B) -> K3 on this rank's B-slice with divisor n ->
 * in-place AllGather; comm on an internal stream, K3 on `stream`, ordered by
 * events so RS(b+1) and AG(b-1) overlap K3(b).  theta length = n_padded,
 * a multiple of nranks*bucket_elems... see pier_shard_layout. */
int pier_outer_step_sharded_f32(PierComm* comm, float* theta, float* anchor_shard,
                                float* mom_shard, int64_t n_padded, int64_t bucket_elems,
                                double lr, double mu, void* stream);
/* lazy-phase fold on this rank's shard (replicas identical, no exchange) */
int pier_warmup_fold_sharded_f32(PierComm* comm, const float* theta, float* anchor_shard,
                                 float* mom_shard, int64_t n_padded, int64_t bucket_elems,
                                 double mu, void* stream);
/* bucketed in-place all-reduce mean (lazy-phase gradient sync, driver.py:380-393) */
int pier_allreduce_mean_f32(PierComm* comm, float* buf, int64_t n, int64_t bucket_elems,
                            void* stream);
/* bf16 gradients: bucketed NCCL average (bf16 partial sums in ring order).
 * Comparison point only -- the engine's 7B recipe uses
 * pier_allreduce_mean_p2p_bf16 (fp32 left fold, one rounding). */
int pier_allreduce_mean_bf16(PierComm* comm, uint16_t* buf, int64_t n, int64_t bucket_elems,
                             void* stream);
/* gather this rank's shard of a sharded array into a contiguous replica
 * (used to report M / anchor with the reference layout) */
int pier_shard_allgather_f32(PierComm* comm, const float* shard, float* full, int64_t n_padded,
                             int64_t bucket_elems, void* stream);

/* ---- fused peer-memory path (NVLink P2P through CUDA IPC) ----------------
 * Collective: every rank calls with the same `bytes`; allocates a zeroed
 * device buffer mapped into all ranks (ids agree across ranks). */
int pier_comm_alloc_shared(PierComm* comm, size_t bytes, void** out_local, int32_t* out_id);
int pier_comm_free_shared(PierComm* comm, int32_t id);
/* ONE kernel over all spans: each rank pulls its slice from every rank's theta,
 * folds them in ascending rank order (bitwise = topology.py:113-121), applies
 * the fused outer update (K3) with its anchor/momentum shard and pushes the
 * new params into every rank's theta.  Same shard layout as
 * pier_outer_step_sharded_f32.  Stream-ordered NCCL barriers bracket it. */
int pier_outer_step_p2p_f32(PierComm* comm, int32_t theta_id, float* anchor_shard,
                            float* mom_shard, int64_t n_padded, int64_t bucket_elems, double lr,
                            double mu, void* stream);
/* The same exchange (over `team`, NULL: every rank) when members hold identical
 * params (the dp replicas of one group after their group step, driver.py:375-378):
 * reps[q] (one per member) is the rank whose copy stands in for member q in the
 * ascending fold -- bitwise the fold over every member, but consecutive members with
 * the same stand-in are pulled once (with reps[q] = (group of q, this rank's dp and
 * tp index) the wire drops from 2(n-1)/n * 4N to (groups-1 + n-1)/n * 4N per
 * direction). */
int pier_outer_step_p2p_reps_f32(PierComm* comm, int32_t theta_id, const int32_t* team, int32_t nteam,
                                 const int32_t* reps, float* anchor_shard, float* mom_shard,
                                 int64_t n_padded, int64_t bucket_elems, double lr, double mu,
                                 void* stream);
/* The same exchange on the region [offset, offset + len) of the buffer only
 * (offset a multiple of n*bucket_elems; len a multiple of 4n, the whole span
 * tail allowed at the end): the shards point at the region's first slice
 * (shard offset offset/n).  Lets a host-resident caller pipeline uploads,
 * exchange and downloads chunk by chunk (PierEngine.step_host). */
int pier_outer_step_p2p_region_f32(PierComm* comm, int32_t theta_id, int64_t offset, int64_t len,
                                   float* anchor_shard, float* mom_shard, int64_t bucket_elems,
                                   double lr, double mu, void* stream);
/* in-place mean over ranks of a shared buffer, left-fold order (bitwise =
 * inner_gradient_sync, topology.py:125-127) */
int pier_allreduce_mean_p2p_f32(PierComm* comm, int32_t buf_id, int64_t n_padded, void* stream);
/* The same mean fused with K4a on its result (lazy phase: driver.py:380-399):
 * each rank sums the squares of the means it produces, the ranks' shares are
 * added in rank order, and `clip_ws` receives the clip record of the averaged
 * gradient -- identical on every rank -- without a second pass over it. */
int pier_allreduce_mean_norm_p2p_f32(PierComm* comm, int32_t buf_id, int64_t n_padded,
                                     double max_norm, void* clip_ws, void* stream);
/* A whole lazy-phase inner step, sharded over the ranks (driver.py:380-399 for
 * t <= lazy_end, where every replica holds the same theta, m, v).  Rank r's shard
 * is its B-slice of every span of n*B elements (B = bucket_elems; 0 = one span:
 * the contiguous r-th 1/n), the layout of the outer exchange.  The mean of the
 * shard (ascending left fold) lands in rank r's gradient buffer with the clip
 * record of the whole mean in `clip_ws` (as pier_allreduce_mean_norm_p2p_f32);
 * rank r then runs AdamW (clip, optim.py:76-102) on its shard only and stores the
 * new params into EVERY rank's theta.  Bitwise equal to the mean + replicated clip
 * + AdamW; the AdamW pass is 1/n of the buffer and overlaps the all-gather.  m and
 * v are current on the shard only afterwards: pier_gather_p2p_f32 (same B) on their
 * shared buffers restores the replicas.  `m`, `v`: this rank's full-length buffers
 * (16-byte aligned).  Collective; stream-ordered barriers bracket the exchanges. */
int pier_lazy_step_p2p_f32(PierComm* comm, int32_t theta_id, int32_t grad_id, float* m, float* v,
                           int64_t n_padded, int64_t bucket_elems, const PierAdamW* hp,
                           double max_norm, void* clip_ws, void* stream);
/* The same step over a team (strictly ascending ranks containing the caller,
 * resolved like pier_outer_step_p2p_team_f32; shard = the caller's position in
 * the team): the replicas of one tensor shard (outer_participant_ranks,
 * topology.py:81-92) in the lazy phase, the dp replicas of one group after it
 * (driver.py:375-378).  `norm_team` (NULL: none): the ranks holding the other
 * tensor shards of this replica -- their square sums are added
 * (pier_norm_allreduce_team) so the clip norm stays global (optim.py:76).
 * Collective over the whole communicator (its barriers). */
int pier_lazy_step_p2p_team_f32(PierComm* comm, int32_t theta_id, int32_t grad_id, const int32_t* team,
                                int32_t nteam, const int32_t* norm_team, int32_t n_norm_team, float* m,
                                float* v, int64_t n_padded, int64_t bucket_elems, const PierAdamW* hp,
                                double max_norm, void* clip_ws, void* stream);
/* The step overlapped with the backward pass: as soon as every rank's gradient of
 * span `span` (elements [span*n*B, (span+1)*n*B), n = team size) is final, each
 * rank calls pier_lazy_pull_span_p2p_f32 (same spans, same order on every rank of
 * the communicator; typically on a side stream behind an event of the backward):
 * the ranks meet and the COPY ENGINES bring the caller's slice of every team
 * member's copy into `staging` (local, n_padded floats; member q's shard at
 * q*n_padded/n) -- no SMs are taken from the backward.  After every span,
 * pier_lazy_finish_staged_p2p_f32 folds the staged copies in ascending rank order
 * (+ the norm of the mean, shared as in the one-call step; `norm_team` as in the
 * team step), then AdamW on the shard + the all-gather.  Team = NULL: every rank.
 * Same params as pier_lazy_step_p2p_team_f32 given the clip scale (the norm's fp64
 * partial sums are added in another order). */
int pier_lazy_pull_span_p2p_f32(PierComm* comm, int32_t grad_id, const int32_t* team, int32_t nteam,
                                float* staging, int64_t n_padded, int64_t bucket_elems, int32_t span,
                                void* stream);
int pier_lazy_finish_staged_p2p_f32(PierComm* comm, int32_t theta_id, int32_t grad_id,
                                    const int32_t* team, int32_t nteam, const int32_t* norm_team,
                                    int32_t n_norm_team, const float* staging, float* m, float* v,
                                    int64_t n_padded, int64_t bucket_elems, const PierAdamW* hp,
                                    double max_norm, void* clip_ws, int32_t push, void* stream);
/* push = 0 above defers the all-gather: the new params stay on each rank's shard
 * (a closing barrier: every shard final), and pier_allgather_span_p2p_f32 then
 * pulls every team member's slice of one span into this rank's buffer with the
 * COPY ENGINES -- called span by span in forward order on a side stream, so the
 * next forward (waiting per span) overlaps the all-gather. */
int pier_allgather_span_p2p_f32(PierComm* comm, int32_t buf_id, const int32_t* team, int32_t nteam,
                                int64_t n_padded, int64_t bucket_elems, int32_t span, void* stream);
/* The sharded lazy step of the 7B recipe (bf16 live params and gradients, fp32
 * master / m / v): the bf16 mean of the shard (fp32 left fold, one RNE rounding,
 * as pier_allreduce_mean_norm_p2p_bf16) with the clip record of the whole mean,
 * AdamW on the shard of the master (master, m, v updated there only), and the RNE
 * bf16 of the new master stored into EVERY rank's live params (`live_id`,
 * n_padded bf16).  The master's other slices go stale: pier_gather_p2p_f32 on
 * `master_id` restores them (before a warmup fold, and when the groups diverge).
 * n_padded a multiple of 8*n, bucket_elems of 8.  Collective. */
int pier_lazy_step_p2p_bf16(PierComm* comm, int32_t master_id, int32_t live_id, int32_t grad_id,
                            float* m, float* v, int64_t n_padded, int64_t bucket_elems,
                            const PierAdamW* hp, double max_norm, void* clip_ws, void* stream);
/* The 7B recipe's step overlapped with the backward (as pier_lazy_pull_span_p2p_f32 /
 * pier_lazy_finish_staged_p2p_f32 on bf16 gradients): copy-engine pulls of the bf16
 * spans into `staging` (n_padded bf16), then the fp32 left fold with one RNE rounding
 * + the norm of the mean, AdamW on the master shard and the live params pushed. */
int pier_lazy_pull_span_p2p_bf16(PierComm* comm, int32_t grad_id, uint16_t* staging, int64_t n_padded,
                                 int64_t bucket_elems, int32_t span, void* stream);
int pier_lazy_finish_staged_p2p_bf16(PierComm* comm, int32_t master_id, int32_t live_id, int32_t grad_id,
                                     const uint16_t* staging, float* m, float* v, int64_t n_padded,
                                     int64_t bucket_elems, const PierAdamW* hp, double max_norm,
                                     void* clip_ws, void* stream);
/* all-gather of a buffer whose rank-r shard (its B-slice of every span of n*B
 * elements; B = 0: the r-th 1/n) is current on rank r: every rank stores its
 * shard into every peer's copy.  Collective. */
int pier_gather_p2p_f32(PierComm* comm, int32_t buf_id, int64_t n_padded, int64_t bucket_elems,
                        void* stream);
/* the same within a team (shard = the caller's position in the team) */
int pier_gather_p2p_team_f32(PierComm* comm, int32_t buf_id, const int32_t* team, int32_t nteam,
                             int64_t n_padded, int64_t bucket_elems, void* stream);
/* A whole Pier round at a boundary iteration, pipelined per span: this group's
 * AdamW (with the clip scale already in `clip_ws`, pier_grad_sqnorm_*) runs
 * span by span on `stream`; as soon as every rank finished span b, the fused
 * pull-fold-update-push kernel for span b runs on a high-priority exchange
 * stream, overlapping the AdamW of span b+1.  Bitwise equal to
 * pier_adamw_f32 followed by pier_outer_step_p2p_f32. */
int pier_round_p2p_f32(PierComm* comm, int32_t theta_id, const float* g, float* m, float* v,
                       float* anchor_shard, float* mom_shard, int64_t n_padded,
                       int64_t bucket_elems, const PierAdamW* hp, const void* clip_ws,
                       double outer_lr, double mu, void* stream);
/* ---- in-switch reduction path (NVLink SHARP / NVLS multicast) ------------
 * Collective: an NCCL symmetric window (ncclMemAlloc + ncclCommWindowRegister)
 * with a multicast mapping; creates the device communicator on first use. */
int pier_comm_alloc_window(PierComm* comm, size_t bytes, void** out_local, int32_t* out_id);
/* one kernel per span: multimem.ld_reduce (switch sums every rank's copy) ->
 * fused outer update on this rank's anchor/momentum shard -> multimem.st to
 * every rank; device-side LSA barriers.  Within fp32 tolerance (switch order). */
int pier_outer_step_nvls_f32(PierComm* comm, int32_t theta_win, float* anchor_shard,
                             float* mom_shard, int64_t n_padded, int64_t bucket_elems, double lr,
                             double mu, void* stream);
int pier_round_nvls_f32(PierComm* comm, int32_t theta_win, const float* g, float* m, float* v,
                        float* anchor_shard, float* mom_shard, int64_t n_padded,
                        int64_t bucket_elems, const PierAdamW* hp, const void* clip_ws,
                        double outer_lr, double mu, void* stream);
int pier_allreduce_mean_nvls_f32(PierComm* comm, int32_t win_id, int64_t n_padded, void* stream);
/* The same round as ONE persistent cooperative kernel per rank: 3 of the 4
 * co-resident CTAs per SM run this group's AdamW (tiles claimed in address
 * order) and publish a per-span ready counter (system-scope release); the
 * fourth pulls-folds-updates-pushes each span as soon as every rank's counter
 * shows it done (acquire loads over NVLink).  Collective: the ranks meet at a
 * stream-ordered barrier (1-element all-reduce) right before the launch, so the
 * spins cover only the round; a wait longer than the communicator's timeout
 * records {rank, span, counter, target} (pier_comm_diag) and traps.  No host
 * synchronisation; bitwise equal to pier_adamw_f32 + pier_outer_step_p2p_f32.
 * On a virtual group every rank's grid is one cooperative launch.
 * 256-bit accesses: g, m, v and the shards 32-byte aligned, n_padded a
 * multiple of 8*n and bucket_elems of 8 (the engine pads to 64*n / 64). */
int pier_round_fused_f32(PierComm* comm, int32_t theta_id, const float* g, float* m, float* v,
                         float* anchor_shard, float* mom_shard, int64_t n_padded,
                         int64_t bucket_elems, const PierAdamW* hp, const void* clip_ws,
                         double outer_lr, double mu, void* stream);
/* 7B recipe (bf16 live params and grads, fp32 master/m/v/anchor/momentum):
 * the same persistent round with bf16 gradients -- the AdamW role is
 * pier_adamw_bf16_f32's master update (driver.py:395-399), the exchange runs
 * on the fp32 master `theta_id` (driver.py:428-440).  The bf16 live copy is
 * NOT written (the outer step replaces it): refresh it with pier_cast_bf16
 * afterwards.  Bitwise equal to pier_adamw_bf16_f32 + pier_outer_step_p2p_f32
 * on the master.  g_bf16 16-byte aligned, m, v and the shards 32-byte aligned. */
int pier_round_fused_bf16_f32(PierComm* comm, int32_t theta_id, const uint16_t* g_bf16, float* m,
                              float* v, float* anchor_shard, float* mom_shard, int64_t n_padded,
                              int64_t bucket_elems, const PierAdamW* hp, const void* clip_ws,
                              double outer_lr, double mu, void* stream);
/* Test harness for the round kernel without a communicator: n (2..8)
 * VIRTUAL ranks on the calling device, every rank's grid (adamw_ctas +
 * exchange_ctas CTAs each) in ONE cooperative launch of k_round_multi<n>
 * (co-resident by construction), peer "NVLink" loads/stores going to the other
 * virtual ranks' buffers.  Exercises every rank-count instantiation (incl. the
 * 8-group one a 4-GPU box cannot launch) on one GPU.  Every per-rank argument
 * is a HOST array of n device pointers; sig[r] = pier_round_sig_bytes() zeroed
 * bytes per virtual rank, kept across rounds like the communicator's block. */
size_t pier_round_sig_bytes(void);
/* (pier_round_virtual_f32 below launches every virtual rank's grid as ONE
 * cooperative kernel on streams[0], so the grids are co-resident.) */
/* The same for the P2P exchange kernel (pier_outer_step_p2p_f32 when outer
 * != 0, pier_allreduce_mean_p2p_f32 when 0): one launch per virtual rank. */
int pier_p2p_virtual_f32(int32_t n, int32_t outer, float* const* buf, float* const* anchor_shards,
                         float* const* mom_shards, int64_t n_padded, int64_t bucket_elems,
                         double outer_lr, double mu, void* const* streams);
int pier_round_virtual_f32(int32_t n, float* const* theta, const float* const* g, float* const* m,
                           float* const* v, float* const* anchor_shards, float* const* mom_shards,
                           uint32_t* const* sig, int64_t n_padded, int64_t bucket_elems,
                           const PierAdamW* hp, const void* const* clip_ws, double outer_lr,
                           double mu, int32_t adamw_ctas, int32_t exchange_ctas,
                           void* const* streams);
/* CTAs per SM of the AdamW role (<= 0 keeps) and the total number of
 * exchange-role CTAs (0 = one per SM, < 0 keeps) of pier_round_fused_f32;
 * clamped so the whole grid stays co-resident. */
int pier_round_split(int adamw_ctas_per_sm, int exchange_ctas);
/* Team variants (groups x dp x tp layouts, topology.py:31-92): the exchange
 * runs among `team` (strictly ascending ranks incl. the caller) -- e.g. the
 * outer participants of one tensor shard (outer_participant_ranks) or the dp
 * replicas of one group (_sync_groups, driver.py:372-378); folding stays in
 * ascending rank order.  Every team of the job must run its exchange at the
 * same point (the ordering barriers span the whole communicator). */
int pier_outer_step_p2p_team_f32(PierComm* comm, int32_t theta_id, const int32_t* team,
                                 int32_t nteam, float* anchor_shard, float* mom_shard,
                                 int64_t n_padded, int64_t bucket_elems, double lr, double mu,
                                 void* stream);
int pier_allreduce_mean_p2p_team_f32(PierComm* comm, int32_t buf_id, const int32_t* team,
                                     int32_t nteam, int64_t n_padded, void* stream);
int pier_round_fused_team_f32(PierComm* comm, int32_t theta_id, const int32_t* team, int32_t nteam,
                              const float* g, float* m, float* v, float* anchor_shard,
                              float* mom_shard, int64_t n_padded, int64_t bucket_elems,
                              const PierAdamW* hp, const void* clip_ws, double outer_lr, double mu,
                              void* stream);
/* Lazy-phase mean of bf16 gradients (7B recipe, driver.py:380-393): each
 * owner folds its 1/n of every rank's shared bf16 buffer in ascending rank
 * order in fp32 (topology.py:113-121), divides by n, rounds once to bf16
 * (RNE) and pushes the result to every rank; barriers bracket it.
 * n_padded (bf16 elements) a multiple of 8*nranks. */
int pier_allreduce_mean_p2p_bf16(PierComm* comm, int32_t buf_id, int64_t n_padded, void* stream);
/* the same mean fused with K4a: each owner also sums the squares of the bf16
 * means it produces (fp64), the ranks' shares are added in rank order -> the
 * clip record of the averaged gradient in `clip_ws`, identical on every rank,
 * without a second pass over the gradient (optim.py:76 on driver.py:380-393) */
int pier_allreduce_mean_norm_p2p_bf16(PierComm* comm, int32_t buf_id, int64_t n_padded, double max_norm,
                                      void* clip_ws, void* stream);
/* Global clip norm over the tensor shards of one replica (optim.py:76 on the
 * concatenated gradient; tp_size > 1): every member's K4a square sum in `ws`
 * goes to every member, each adds the team's sums in ascending rank order and
 * re-finalises its clip record (same formula as pier_clip_finalize, f32). */
int pier_norm_allreduce_team(PierComm* comm, const int32_t* team, int32_t nteam, void* clip_ws,
                             double max_norm, void* stream);
/* launch tuning of the fused kernels (process-wide): CTAs per SM (>0; default 4,
 * 6 for the two kernels of pier_lazy_step_p2p_f32 / pier_gather_p2p_f32 -- a value
 * set here applies to all),
 * 16-B vectors per thread per rank (0 = auto), and diagnostic flags
 * (bit0: loads from peers, bit1: stores to peers; 3 = normal). <0 keeps. */
int pier_p2p_tune(int ctas_per_sm, int unroll, int flags);
/* pier_round_p2p_f32 grid sizes: CTAs per SM for its AdamW spans and for its
 * exchange kernels (both run concurrently). <= 0 keeps the current value. */
int pier_round_tune(int adamw_ctas_per_sm, int p2p_ctas_per_sm);

/* ---- host offload of outer state (driver.py:115-164, 318-329) ------------ */
typedef struct PierOffload PierOffload;
/* setup: `nslots` pinned host slots of `slot_bytes` each and two side streams
 * (D2H parks, H2D fetches); both move 64 MB pieces and the fetch of a piece
 * waits only for that piece's park, so a fetch can run behind a park */
int pier_offload_create(int32_t nslots, size_t slot_bytes, PierOffload** out);
int pier_offload_destroy(PierOffload* off);
/* D2H of `bytes` from `dev` into slot, on the side stream, after all work
 * queued so far on `producer`.  PIER_EPROTOCOL if the slot is already live. */
int pier_offload_park(PierOffload* off, int32_t slot, const void* dev, size_t bytes,
                      void* producer);
/* H2D back into `dev`; `consumer` waits for it.  PIER_EPROTOCOL if not live. */
int pier_offload_fetch(PierOffload* off, int32_t slot, void* dev, size_t bytes, void* consumer);
/* split form of fetch: issue the H2D now (after work queued on `consumer`),
 * and make `consumer` wait for it later, so the copy overlaps inner steps */
int pier_offload_prefetch(PierOffload* off, int32_t slot, void* dev, size_t bytes, void* consumer);
int pier_offload_wait(PierOffload* off, int32_t slot, void* consumer);
/* block until the slot's transfer finished (tests / teardown) */
int pier_offload_sync(PierOffload* off);
/* counters: to_host_bytes, from_host_bytes, store_events, load_events, resident_bytes */
int pier_offload_counters(const PierOffload* off, double* out5);
void* pier_offload_host_ptr(PierOffload* off, int32_t slot);
/* the side streams (cudaStream_t) of parks (D2H) and fetches (H2D), so callers
 * can order allocator reuse of the device buffers on them */
void* pier_offload_stream(PierOffload* off);
void* pier_offload_stream_h2d(PierOffload* off);

#ifdef __cplusplus
}
#endif
#endif /* PIER_B200_H */
