/*
 * spz.h -- C ABI of the B200-native Spreeze update hot path.
 *
 * Spreeze (arXiv 2312.06126) "Network Update" (§3.2):
 * experience is "transmitted to a single network update process for
 * parallelization by GPU" with "a large batch size", and the SAC
 * update uses "two value networks Q1 and Q2 ... updated ... together with the
 * target network".  This library implements exactly that step, from a
 * device-resident replay ring (the paper's shared-memory experience pool,
 * P:278-288) to the Adam/Polyak parameter update, as hand-written sm_100a
 * CUDA.  The semantics of every call are those of the float64 oracle in
 * oracle/ (DESIGN.md "Readings").
 *
 * Conventions (all calls):
 *  - Every call returns spz_status; on a non-OK return spz_last_error() gives a
 *    thread-local human-readable message naming the failing argument/kernel.
 *  - Handles are opaque and caller-owned; *_destroy frees them (NULL is a no-op).
 *  - Input arrays are borrowed for the duration of the call only.
 *  - Pointers documented "device" must be device pointers on the handle's device
 *    (any allocator: cudaMalloc, torch); "host" pointers are ordinary host memory.
 *  - A handle is single-owner: calls on one handle must not run concurrently;
 *    calls on different handles may ("single-owner").
 *  - There is no CPU fallback: without a usable sm_100 device every creating
 *    call fails with SPZ_ECUDA.
 */
#ifndef SPZ_H_
#define SPZ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPZ_OK = 0,
  SPZ_EINVAL = -1,        /* bad argument (dims, sizes, NULL, batch > max_batch)    */
  SPZ_ENODATA = -2,       /* ring fill < batch ("caller retries")             */
  SPZ_ENONFINITE = -3,    /* non-finite loss/gradient; learner halted */
  SPZ_ECUDA = -4,         /* CUDA runtime/driver error or no sm_100 device          */
  SPZ_ENCCL = -5,         /* NCCL error                                             */
  SPZ_ENOMEM = -6,        /* device allocation failed                               */
  SPZ_ESTATE = -7,        /* call not valid in the handle's current state           */
  SPZ_ETIMEOUT = -8,      /* split-mode peer missed the step barrier        */
  SPZ_EUNSUPPORTED = -9   /* configuration not built in this library                */
} spz_status;

/* Thread-local message for the last non-OK return on this thread ("" if none). */
const char* spz_last_error(void);
/* Library version string and the build's target ("sm_100a"). */
const char* spz_version(void);

/* ------------------------------------------------------------------ replay ring
 * Device-resident ring of transitions ("state s, action a, next state s2,
 * reward r, and done flag d"; SPEC ReplayRing S:172-179).  Record layout: one
 * fp32 record per transition, [s(o) | a(m) | r | d | s2(o) | pad], padded to
 * R = round_up(2o+m+2, 4) floats (16-byte aligned rows, read with 128-bit loads).
 * Global index i lives in slot i mod C; fill = min(cursor, C).
 */
typedef struct spz_replay spz_replay;

typedef struct {
  int32_t obs_dim;      /* o >= 1                                   */
  int32_t act_dim;      /* m >= 1                                   */
  int64_t capacity;     /* C >= 1 (capacity 0 is SPZ_EINVAL) */
  int32_t device;       /* CUDA device ordinal that holds the ring  */
} spz_replay_desc;

spz_status spz_replay_create(const spz_replay_desc* desc, spz_replay** out);

/* Append n transitions (S:195 ring_push).  obs/next_obs are [n x o] row-major,
 * act [n x m], rew [n], done [n] (d in {0,1}; time-limit truncation stored as 0,
 * S:230).  If src_on_device == 0 the arrays are host memory (staged through a
 * pinned buffer, copied in at most two pieces split at the wrap point); if 1 they
 * are device pointers on the ring's device.  Synchronous with respect to the
 * source buffers.  *first_global_index (nullable) receives the global index of
 * the first record; the oldest records are overwritten when full. */
spz_status spz_replay_push(spz_replay* r, int64_t n, const float* obs, const float* act,
                           const float* rew, const float* next_obs, const float* done,
                           int32_t src_on_device, int64_t* first_global_index);
/* As spz_replay_push, but for page-locked host fields it returns once the copies are enqueued: the
 * caller keeps the five buffers unchanged until the NEXT spz_replay_push / spz_replay_push_async on this
 * ring returns, or spz_replay_sync(r) does (so two alternating host buffer sets suffice).  Pageable or
 * device sources behave exactly like spz_replay_push.  Lets a producer stream transitions without
 * waiting for each H2D copy (P:278-288 ingest; the e2e loop of bench.py). */
spz_status spz_replay_push_async(spz_replay* r, int64_t n, const float* obs, const float* act,
                                 const float* rew, const float* next_obs, const float* done,
                                 int32_t src_on_device, int64_t* first_global_index);
/* Wait until the host buffers of the last spz_replay_push_async have been read. */
spz_status spz_replay_sync(spz_replay* r);

/* Uniform sample with replacement over slots [0, F), F = current fill (S:203,
 * S:228): for j in [0, batch), (x0,x1,x2,x3) = Philox4x32-10(key = seed,
 * ctr = (j, 0, step, 1)) and idx_j = floor((x1*2^32 + x0) * F / 2^64).  Writes
 * (each output nullable, all device pointers, row-major): idx int32[batch],
 * obs [batch x o], act [batch x m], rew [batch], next_obs [batch x o],
 * done [batch].  Returns SPZ_ENODATA if F < batch.  Synchronous. This is the same
 * draw the learner makes internally at its global step `step`. */
spz_status spz_replay_sample(spz_replay* r, int64_t batch, uint64_t seed, uint64_t step,
                             int32_t* idx, float* obs, float* act, float* rew,
                             float* next_obs, float* done);

spz_status spz_replay_info(const spz_replay* r, int64_t* cursor, int64_t* fill, int64_t* capacity);
/* Device pointer to the record array [C x R] fp32 and R (for zero-copy inspection). */
spz_status spz_replay_records(const spz_replay* r, const float** records, int32_t* record_floats);
/* Experience transmission loss (Table 3 column): the fraction of
 * pushed records overwritten before ever being sampled.  spz_replay_track(r, 1) starts accounting
 * (a one-bit "sampled" tag per slot, set by every sample -- the learners' gathers and
 * spz_replay_sample; a push counts each unsampled tracked record it overwrites, and every record
 * of a push longer than the capacity that never lands); 0 stops it.  Learners pick the change up
 * at their next update (their plan is rebuilt).  spz_replay_loss reports, since tracking started:
 * pushed = lost + resident_unsampled + sampled_at_least_once.  SPZ_ESTATE if tracking is
 * off.  Synchronous.  (Row-sharded learners each mark their own ring replica.) */
spz_status spz_replay_track(spz_replay* r, int32_t on);
spz_status spz_replay_loss(spz_replay* r, int64_t* pushed, int64_t* lost, int64_t* resident_unsampled);
void spz_replay_destroy(spz_replay* r);

/* ------------------------------------------------------------------ learner
 * One SAC (or TD3, DDPG) update step per the oracle, Jacobi order:
 * all losses at (theta_k, phi_k, alpha_k), then Adam on each trained network
 * (own step counter), then Polyak theta' <- tau theta + (1-tau) theta'.
 * DDPG (§8(f) f4, oracle/ddpg.py: one critic, no target smoothing, no policy delay) runs on the TD3
 * kernels with the twin critic tied to the first: Q2 = Q1 and Q2' = Q1' at creation and on every
 * spz_set_params of Q1 / Q1_TARG (setting Q2 / Q2_TARG directly is SPZ_EINVAL), so both receive
 * identical updates and min(Q1', Q2') = Q1'; the reported critic_loss is DDPG's (half the twins' sum).
 * spz_config_default(SPZ_DDPG) sets td3_policy_delay = 1 and td3_noise = td3_noise_clip = 0.
 * SPZ_SACV1 (§8(f) f4, oracle/sacv1.py, reading #24): the original soft actor-critic the
 * paper cites -- a state-value network V(s) (in = o, out 1, same hidden stack) with a Polyak
 * target V'; the twin critics regress to y_Q = r + gamma (1-d) V'(s2) (no target critics, no a'), V to
 * y_V = min_i Q_i(s, a~) - alpha log pi(a~|s), L_V = (1/B) sum (V(s) - y_V)^2 (stats value_loss); the
 * policy and temperature losses are SAC's.  V is trained with lr_critic.  spz_config_default(SPZ_SACV1)
 * sets alpha_auto = 0 (v1's fixed temperature).  Role ALL only.
 */
typedef enum { SPZ_SAC = 0, SPZ_TD3 = 1, SPZ_DDPG = 2, SPZ_SACV1 = 3 } spz_algo;
/* FP32: every dense layer as 3xTF32 on tcgen05 (hi = rna_tf32(x), lo = rna_tf32(x - hi),
 * D = hi*hi + hi*lo + lo*hi, 64-deep TMEM chunk sums added in fp32 registers; readings #15, #22);
 * BF16: GEMM operands rounded to bf16 (RNE) on tcgen05 tensor cores with fp32 accumulation.  Every
 * epilogue, master weight and optimizer state stays fp32 in both (reading #15). */
typedef enum { SPZ_FP32 = 0, SPZ_BF16 = 1 } spz_precision;
/* Role of this rank (P:239-247 actor/critic model parallelism). */
typedef enum { SPZ_ROLE_ALL = 0, SPZ_ROLE_CRITIC = 1, SPZ_ROLE_ACTOR = 2 } spz_role;

typedef struct {
  spz_algo algo;
  spz_precision precision;
  int32_t obs_dim, act_dim;        /* o, m                                       */
  int32_t hidden, n_hidden;        /* h, L: L hidden ReLU layers of width h      */
  int64_t max_batch;               /* upper bound on the (global) batch          */
  double gamma, tau;               /* 0.99, 0.005                                */
  double lr_actor, lr_critic, lr_alpha, beta1, beta2, adam_eps; /* 3e-4 x3, 0.9, 0.999, 1e-8 */
  int32_t alpha_auto;              /* 1: learn log alpha (target entropy below)  */
  double alpha_init, target_entropy, log_std_min, log_std_max; /* 0.2, -m, -20, 2 */
  double td3_noise, td3_noise_clip; int32_t td3_policy_delay;  /* 0.2, 0.5, 2 */
  uint64_t seed;                   /* sampling/noise key (Philox)                */
  uint64_t init_seed;              /* parameter init key (Philox stream 5)       */
  int32_t device;                  /* CUDA device ordinal                        */
  int32_t world_size, rank;        /* row sharding: rank handles a contiguous slice of global rows */
  int32_t n_critic_ranks, n_actor_ranks; /* split roles over world_size ranks: ranks [0, n_critic_ranks)
                                            are the critic group, the rest the actor group */
  spz_role role;                   /* ALL (default), or one half of the Jacobi step  */
  const uint8_t* nccl_unique_id;   /* 128 bytes, identical on all ranks; NULL if world_size == 1 */
  int32_t use_graph;               /* 1 (default): replay the step as a CUDA graph */
  int32_t comm_mode;               /* world_size > 1: 0 = NCCL allreduce (default); 1 = no exchange
                                      (diagnostics: each rank applies its own shard's gradient);
                                      2 = (world_size 1 only) run the sharded path through a
                                      single-rank NCCL communicator (diagnostics) */
} spz_config;

/* Fill *out with the defaults above for (algo, o, m); h = 256, L = 2, max_batch 8192. */
spz_status spz_config_default(spz_algo algo, int32_t obs_dim, int32_t act_dim, spz_config* out);
/* Generate a fresh NCCL unique id (rank 0 calls this and broadcasts the bytes).  NCCL is
 * loaded at run time (libnccl.so.2); SPZ_ENCCL if unavailable. */
spz_status spz_nccl_unique_id(uint8_t out[128]);

/* Host-side multi-GPU plan of one rank (reading #17; P:239-247 for the
 * actor/critic split, P:170-173 for the row-sharded group).  Pure host arithmetic, no device: the
 * learner builds its own partition, communicator split and exchange from this function, and the
 * world-size-2 gloo tests check the same function across processes.
 *   role ALL:    one group of world_size ranks;  role CRITIC / ACTOR (world_size > 1): the critic group
 *                is ranks [0, n_critic_ranks), the actor group the rest.
 *   rows:        the group's global batch B split contiguously by global row id, the first B % G
 *                ranks one row longer; every group reads all B rows.
 *   exchange:    split roles broadcast phi_{k+1} (+ log alpha, TD3 phi') from actor_root and
 *                theta_{k+1} from critic_root over the world communicator at the step boundary.
 * Errors: SPZ_EINVAL (NULL, bad world/rank/role layout, batch < group_size). */
typedef struct {
  int32_t role;         /* SPZ_ROLE_* this rank computes                                   */
  int32_t group_size;   /* ranks in its row-sharded group                                  */
  int32_t group_rank;   /* index inside the group (the communicator-split key)             */
  int32_t group_color;  /* 0 = critic group or all ranks, 1 = actor group (the split color) */
  int64_t row0, rows;   /* its share [row0, row0 + rows) of the global batch               */
  int32_t actor_root;   /* world rank broadcasting the actor side (split), else -1         */
  int32_t critic_root;  /* world rank broadcasting the critics (split), else -1            */
  int32_t allreduce;    /* 1: the group all-reduces [gradients | loss totals] every step   */
  int32_t pad_;
} spz_plan;
spz_status spz_plan_rank(const spz_config* cfg, int64_t batch, spz_plan* out);

typedef struct spz_learner spz_learner;

typedef struct {
  int64_t step;                    /* global step k of the last completed update          */
  double critic_loss, actor_loss;  /* L_Q, L_pi at step k (TD3: L_pi on delayed steps)    */
  double alpha, alpha_loss;        /* alpha_k and L_alpha                                 */
  double q1_mean, q2_mean;         /* mean Q_i(s, a) over the batch                       */
  double logp_mean;                /* mean log pi(a~|s)                                   */
  double value_loss;               /* SAC v1: L_V at step k (else 0)                      */
} spz_stats;

/* Create a learner on cfg->device that samples from `ring` (borrowed: the ring
 * must outlive the learner and live on the same device).  Parameters are
 * initialised W, b ~ U(+-1/sqrt(fan_in)) from Philox(init_seed, stream 5); the
 * targets copy the online networks; log alpha = ln(alpha_init). */
spz_status spz_learner_create(const spz_config* cfg, spz_replay* ring, spz_learner** out);

/* Run n_steps update steps with (global) batch B, each exactly the oracle's step
 * k = current step.  Step k samples exactly spz_replay_sample(ring, B, seed, k).
 * Requires fill >= B (else SPZ_ENODATA, nothing run) and B <= max_batch.  B may
 * change between calls; Adam moments are preserved.  Synchronous at
 * return (one device->host read of the stats and the non-finite flag).  On a
 * non-finite loss the learner stops at the state before the failing step and
 * returns SPZ_ENONFINITE (message names the step).  *last (nullable) receives
 * the statistics of the last completed step. */
spz_status spz_update(spz_learner* L, int64_t batch, int64_t n_steps, spz_stats* last);

/* The two halves of spz_update, so a caller can overlap its next spz_replay_push with the update
 * running on the GPU -- the paper's updater "reads the experience pool without waiting for the
 * samplers" (§3.3.2).  spz_update_async enqueues the n_steps steps (same semantics and
 * errors as spz_update except SPZ_ENONFINITE of *these* steps, which spz_update_wait reports) and
 * returns without waiting; up to two calls are in flight per learner (a third first completes the
 * oldest), so the host's next push and launch hide under the running update.  Ring pushes issued
 * meanwhile are ordered on the device: their records are written only after the reads of every update
 * enqueued before them, and the next update waits for them, so results are identical to the
 * synchronous sequence push, update, push, update.  spz_update_wait blocks until the oldest call in
 * flight finishes and fills *last (nullable) with its statistics like spz_update; with nothing in
 * flight it returns the statistics of the last completed update. */
spz_status spz_update_async(spz_learner* L, int64_t batch, int64_t n_steps);
spz_status spz_update_wait(spz_learner* L, spz_stats* last);

/* Use `stream` (a cudaStream_t on the learner's device, e.g. a torch stream) for
 * all subsequent work; NULL restores the learner's private stream. */
spz_status spz_learner_set_stream(spz_learner* L, void* stream);

typedef enum {
  SPZ_T_ACTOR = 0, SPZ_T_Q1 = 1, SPZ_T_Q2 = 2, SPZ_T_Q1_TARG = 3, SPZ_T_Q2_TARG = 4,
  SPZ_T_ACTOR_TARG = 5, /* TD3 only */
  SPZ_T_LOG_ALPHA = 6,
  SPZ_T_V = 7, SPZ_T_V_TARG = 8 /* SAC v1 only: the state-value network and its target */
} spz_tensor;
typedef enum { SPZ_S_PARAM = 0, SPZ_S_ADAM_M = 1, SPZ_S_ADAM_V = 2 } spz_slot; /* Adam slots: trained nets only */

/* Flat fp32 layout (the oracle's): for each layer l = 1..L+1, W_l row-major
 * [out x in] then b_l[out].  Actor: in = o, hidden h, out = 2m (SAC: rows 0..m-1
 * mu, m..2m-1 log sigma) or m (TD3).  Critics: in = o + m (input [s | a]), out 1.  V: in = o, out 1.
 * LOG_ALPHA is 1 float.  get: n < n_required -> SPZ_EINVAL and *n_required set. */
spz_status spz_get_params(spz_learner* L, spz_tensor t, spz_slot s, float* host_out, int64_t n,
                          int64_t* n_required);
spz_status spz_set_params(spz_learner* L, spz_tensor t, spz_slot s, const float* host_in, int64_t n);
/* Adam step counters t of (critic, actor, alpha) optimizers and the global step. */
spz_status spz_get_counters(spz_learner* L, int64_t* step, int64_t* t_critic, int64_t* t_actor, int64_t* t_alpha);

/* Actor publication buffer ("never a blend", S:248/S:271 monotone version):
 *   bytes [0, 64)  header: u64 version (last published; 0 = none) | u64 n_floats | u64 seq[2] | 32 B reserved
 *   slot s at SPZ_SYNC_HEADER_BYTES + s * SPZ_SYNC_SLOT_BYTES(n): n_floats fp32 (the flat actor)
 * Version v lives in slot v & 1.  seq[s] is the per-slot seqlock word: 2v - 1 (odd) while version v's
 * payload is being written into slot s, 2v once it is complete. */
#define SPZ_SYNC_HEADER_BYTES 64
#define SPZ_SYNC_SLOT_BYTES(n) ((((int64_t)(n) * 4 + 63) / 64) * 64)
#define SPZ_SYNC_BYTES(n) (SPZ_SYNC_HEADER_BYTES + 2 * SPZ_SYNC_SLOT_BYTES(n))

/* Push the actor parameters peer-to-peer (north_star "actor parameters pushed
 * peer-to-peer") into a publication buffer (layout above) on dst_device.  Publishing version v, in
 * stream order: seq[v & 1] = 2v - 1, the payload into slot v & 1, seq[v & 1] = 2v, then the header
 * version = v.  Version v - 1 (the other slot) stays intact while v is written, so a reader always has
 * one complete version to copy, and a reader that overlaps a rewrite of its slot sees seq change and
 * retries (spz_policy_load) -- it never accepts a blend.  The version is monotone per learner
 * and returned in *version (nullable).  dst must be device memory on dst_device (peer access is
 * enabled when available, else the copy is staged by the driver), zero-initialised before the first
 * publication, 16-byte aligned; dst_bytes >= SPZ_SYNC_BYTES(n_floats).  Synchronous.
 * Errors: SPZ_EINVAL (NULL / too small), SPZ_ECUDA. */
spz_status spz_sync_actor(spz_learner* L, int32_t dst_device, void* dst, int64_t dst_bytes,
                          uint64_t* version);

/* Actor/critic model parallelism on one host process: after each spz_update of a
 * critic-role learner and an actor-role learner (each world_size 1, any devices), copy the
 * updated actor parameters and log alpha (TD3: also the target actor) into the critic side and
 * the online critics into the actor side (peer copies), refreshing the receivers' operand
 * shadows.  With world_size > 1 and NCCL the same exchange runs inside every step instead.
 * Together the two halves compute exactly the single-learner step (Jacobi order, reading #3). */
spz_status spz_split_exchange(spz_learner* critic_side, spz_learner* actor_side);

/* Per kernel-class device time (ms per step, averaged over n_steps steps run
 * un-graphed with CUDA events around each class) -- measurement only; the steps
 * run are real updates.  names/ms arrays of capacity `cap`; *count set. */
spz_status spz_learner_profile(spz_learner* L, int64_t batch, int64_t n_steps, int32_t cap,
                               const char** names, double* ms, int32_t* count);
/* Number of kernel launches one update step performs (for the bench's gpu_launches). */
spz_status spz_learner_launches_per_step(spz_learner* L, int64_t batch, int32_t* launches);

/* Copy an internal step buffer (as left by the last completed step) to host memory, for
 * tests and diagnosis only.  Names: "Xa", "Xc", "H", "dH", "Aact<l>", "dZa<l>",
 * "Aon<i>_<l>", "Atg<i>_<l>", "dZc<i>_<l>", "q_on<i>", "q_tg<i>", "gq<i>", "dXc<i>",
 * "logp", "logp2", "r", "d", "y", "idx".  Raw bytes in the buffer's element type
 * (*elem_size = 2 for bf16 operand buffers, 4 for fp32 / int32), sized for max_batch
 * rows.  host_out == NULL only reports *bytes_required. */
spz_status spz_learner_debug_buffer(spz_learner* L, const char* name, void* host_out, int64_t bytes,
                                    int64_t* bytes_required, int32_t* elem_size);

/* ---------------------------------------------------------------- batch-size adaptation (§8(f) f3)
 * The paper adapts its batch size to the largest one the GPU sustains ("BS mainly loads
 * the GPU"; enumeration assuming a unimodal response).  spz_tune_batch probes the
 * ascending ladder[0..n): at each B it runs max(warmup, 1) untimed then `steps` timed update steps
 * (CUDA events on the learner's stream) and records the update frequency and frames/s = B x
 * updates/s.  It stops climbing once frames/s falls more than `tol` (relative) below the best so far
 * (past the peak) or the update frequency falls below min_update_hz; *best = the probed B with the
 * most frames/s among those meeting min_update_hz (ladder[0] if none does).  With restore != 0 the
 * parameters, Adam moments, step counters and the non-finite flag are restored afterwards, so training
 * continues exactly as if the tuner had not run; else the probe steps count as training.  Needs
 * fill >= B and B <= max_batch for every probed B (else SPZ_EINVAL / SPZ_ENODATA); the ladder must
 * be strictly ascending.  out[0..*n_out) receives the probed points (caller-allocated, n entries). */
typedef struct {
  int64_t batch;
  double updates_per_s;
  double frames_per_s;
  double ms_per_update;
} spz_tune_point;
spz_status spz_tune_batch(spz_learner* L, const int64_t* ladder, int32_t n, int64_t warmup, int64_t steps,
                          double min_update_hz, double tol, int32_t restore, spz_tune_point* out, int32_t* n_out,
                          int64_t* best);

void spz_learner_destroy(spz_learner* L);

/* ------------------------------------------------------------------ diagnostics
 * spz_diag_tc_trace: enable (on = 1) / disable per-tile %globaltimer stamps in the tcgen05 GEMM
 * (160 CTAs x 8 tiles x 4 events: producer start, MMA issued, accumulator ready, epilogue done) and,
 * if host_out != NULL, copy up to n stamps of the last traced launch.  on = k >= 2 traces only the
 * (k-2)-th launch from now.  on >= 100 addresses the fused MLP forward instead (mode on - 100;
 * 160 CTAs x 4 units x 3 layers x 4 events: MMA start, MMA issued, accumulator ready, epilogue
 * done).  Synchronous. */
spz_status spz_diag_tc_trace(int32_t device, int32_t on, uint64_t* host_out, int32_t n);

/* The dense-layer GEMM of the update on its own, for kernel tests: on `device`,
 * C[m, n] (fp32, row pitch ldc) = sum_k A(m, k) B(n, k) over bf16 device operands with
 * A(m,k) = a_mn ? A[k*lda + m] : A[m*lda + k] and B(n,k) = b_mn ? B[k*ldb + n] : B[n*ldb + k].
 * With splits > 1 the contraction is cut into chunks of k_per_split (multiple of 64) and
 * chunk s is written to C + s*M*ldc.  tensor_cores = 1 runs the tcgen05 kernel (SPZ_EUNSUPPORTED
 * if the problem does not qualify), 0 the SIMT kernel.  Synchronous. */
spz_status spz_diag_gemm_bf16(int32_t device, int32_t tensor_cores, int64_t M, int64_t N, int64_t K,
                              const void* A, int64_t lda, int32_t a_mn, const void* B, int64_t ldb,
                              int32_t b_mn, float* C, int64_t ldc, int32_t splits, int64_t k_per_split);

/* ---------------------------------------------------------------- sampler-side policy (§8(f) f1)
 * Batched actor inference for the samplers, fed by spz_sync_actor (sampler actions are
 * "generate[d] ... by forward propagation"; the test process acts deterministically).
 *   SAC  deterministic a = tanh(mu);  stochastic a = tanh(mu + exp(clamp(l, lo, hi)) * n)
 *   TD3  deterministic a = tanh(z);   stochastic a = clip(tanh(z) + expl_noise * n, -1, 1)
 * n[j, i]: normal i of call row j, Philox(seed, (j, i / 4, step, S_ACT = 7)) Box-Muller as in the
 * update (readings #13, #21).  Same dense layers as the update: bf16 tcgen05 GEMMs, or
 * 3xTF32 in FP32 precision. */
typedef struct spz_policy spz_policy;     /* opaque, caller-owned */
typedef struct {
  spz_algo algo;
  spz_precision precision;
  int32_t obs_dim, act_dim, hidden, n_hidden;  /* must match the learner whose actor is loaded */
  int64_t max_batch;                           /* rows per spz_policy_act call                  */
  int32_t device;
  double log_std_min, log_std_max;             /* SAC clamp (learner defaults: -20, 2)           */
  double expl_noise;                           /* TD3 exploration std (0.1)                      */
} spz_policy_desc;
/* Errors: SPZ_EINVAL (bad dims), SPZ_ENOMEM, SPZ_ECUDA. */
spz_status spz_policy_create(const spz_policy_desc* desc, spz_policy** out);
/* Load the actor from a spz_sync_actor publication buffer (layout above; device or host memory, borrowed
 * for the call).  Seqlock read of the newest version v: header, seq[v & 1] == 2v, payload of slot v & 1,
 * seq[v & 1] again; any change (a writer reached that slot again) restarts the read, so the loaded
 * parameters are exactly one version's; *version (nullable) receives it.  SPZ_ESTATE if nothing
 * was published yet; SPZ_EINVAL if n_floats does not match the policy's shape or bytes is too small;
 * SPZ_ETIMEOUT if 64 attempts all overlapped a writer.  Synchronous. */
spz_status spz_policy_load(spz_policy* P, const void* payload, int64_t bytes, uint64_t* version);
/* Actions act [n x m] (fp32, row-major) for observations obs [n x o]; each pointer may be host or
 * device memory (detected).  0 <= n <= max_batch.  deterministic != 0 selects the test-process
 * action.  SPZ_ESTATE before the first spz_policy_load.  Synchronous. */
spz_status spz_policy_act(spz_policy* P, int64_t n, const float* obs, int32_t deterministic, uint64_t seed,
                          uint64_t step, float* act);
/* Copy the currently loaded flat actor (fp32, the spz_get_params layout) to host memory; n >= n_floats. */
spz_status spz_policy_get_params(spz_policy* P, float* host_out, int64_t n);
void spz_policy_destroy(spz_policy* P);

/* Diagnostics (GEMM unit tests): the FP32-precision GEMM, C = A * B in fp32 with the same operand
 * conventions as spz_diag_gemm_bf16 but fp32 operands (row pitches multiple of 4 elements, 16-byte
 * aligned device pointers).  tensor_cores = 1 runs the 3xTF32 tcgen05 kernel (SURVEY.md §8(a) a3,
 * §8(c) reading 15: hi = x with the low 13 mantissa bits cleared, lo = x - hi, D = hi*hi + hi*lo +
 * lo*hi accumulated in fp32; k_per_split a multiple of 32), 0 the fp32 SIMT kernel.  Synchronous.
 * Errors: SPZ_EINVAL (bad sizes / NULL), SPZ_EUNSUPPORTED (layout the kernel does not take),
 * SPZ_ECUDA. */
spz_status spz_diag_gemm_f32(int32_t device, int32_t tensor_cores, int64_t M, int64_t N, int64_t K,
                             const float* A, int64_t lda, int32_t a_mn, const float* B, int64_t ldb,
                             int32_t b_mn, float* C, int64_t ldc, int32_t splits, int64_t k_per_split);

#ifdef __cplusplus
}
#endif
#endif /* SPZ_H_ */
