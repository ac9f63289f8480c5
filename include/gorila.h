/* gorila.h — C-ABI of the B200-native Gorila DQN learner update.
 *
 * Paper: Nair et al. 2015, "Massively Parallel Methods for Deep Reinforcement
 * Learning" (arXiv:1507.04296), /root/reference/PAPER.md. Citations are
 * PAPER.md line numbers (P:L) with the section / equation / algorithm.
 *
 * The library implements Algorithm 1's learner half and the
 * sharded parameter server for the Nature-DQN Q-network
 * (§5.1), one process per GPU. All compute runs in the library's own
 * sm_100a kernels. When world > 1 the gradient sum and the parameter broadcast
 * run inside one library kernel over NVLink peer memory (every rank maps every
 * peer's workspace through CUDA IPC); NCCL (the copy torch loads) is used only
 * to bootstrap those mappings and, if peer mappings are unavailable, as the
 * fallback reduce-scatter / all-gather.
 *
 * Conventions (all entry points):
 *  - Ownership: the caller owns the workspace (device memory, e.g. a torch
 *    tensor of gorila_workspace_bytes()), the stream and every host buffer.
 *    The context owns sub-allocations of the workspace and its NCCL
 *    communicator (destroyed by gorila_destroy). No pointer argument is retained
 *    after a call returns, except config.workspace and config.stream.
 *  - Asynchrony: every call enqueues work on config.stream and returns without
 *    synchronising, unless stated. *_info / *_out host buffers are written by
 *    cudaMemcpyAsync on that stream: valid after the stream synchronises
 *    (pass pinned memory for a fully asynchronous copy).
 *  - Collectives: gorila_init (world > 1) and ps_apply_shard are collective —
 *    every rank calls them in the same order with the same arguments.
 *  - Errors: every call returns a gorila_status; no C++ exception crosses the
 *    ABI; gorila_last_error() returns a thread-local message. After
 *    GORILA_E_CUDA / GORILA_E_NCCL the context is poisoned: only
 *    gorila_destroy is legal. Outcomes (outlier-rejected, stale, not ready)
 *    are NOT errors; they are reported in gorila_learner_info.
 *  - Parameter layout at the boundary ("canonical"): flat float32 vector
 *    [W1,b1,W2,b2,W3,b3,W4,b4,W5,b5]; conv weights OIHW, FC weights
 *    [out][in]; fc4's input index = c*49 + y*7 + x (CHW flatten, reading R18).
 *    P = 1,684,128 + 513*nA (1,693,362 for nA = 18). Internal layouts are private.
 */
#ifndef GORILA_H
#define GORILA_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GORILA_API __attribute__((visibility("default")))
#else
#define GORILA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gorila_ctx gorila_ctx; /* opaque; one per rank */

typedef enum {
    GORILA_OK = 0,
    GORILA_E_INVALID = 1,   /* invalid config or argument */
    GORILA_E_SHAPE = 2,     /* wrong buffer size / count */
    GORILA_E_RANGE = 3,     /* learner id or action out of range */
    GORILA_E_NOT_READY = 4, /* replay below the warm-up size (replay_sample only) */
    GORILA_E_CUDA = 5,
    GORILA_E_NCCL = 6,
    GORILA_E_OOM = 7        /* workspace too small */
} gorila_status;

typedef enum {
    GORILA_MATH_FP32 = 0, /* fp32 SIMT check mode: parity 1e-5 vs the exact oracle */
    GORILA_MATH_BF16 = 2  /* bf16 operands on tcgen05 tensor cores, fp32 accumulate (reading R16) */
} gorila_math;

typedef enum {
    GORILA_OPT_RMSPROP = 0, /* centered RMSProp (BASELINE north_star; reading R2) */
    GORILA_OPT_ADAGRAD = 1  /* the paper's rule, "we used the AdaGrad update rule" */
} gorila_optimizer;

typedef struct {
    int32_t n_actions;         /* nA in [1, 32]: "a single output unit for each valid action" */
    int32_t batch;             /* B in [1, 4096], minibatch per learner (Alg.1) */
    float gamma;               /* discount, Alg.1 target P:125 */
    int64_t replay_capacity;   /* C frames per learner ("1 million frames"); >= 2 */
    int32_t n_learners_local;  /* learners (bundles) hosted by this rank, >= 1 */
    int32_t learner_id_base;   /* global id of local learner 0 (ids feed the sampler's Philox counter) */
    int32_t rank, world;       /* this rank; number of ranks = parameter-server shards */
    const void* nccl_unique_id;/* 128-byte ncclUniqueId broadcast by the caller; NULL if world == 1 or
                                  the caller bootstraps the peer mappings (gorila_peer_connect) */
    void* stream;              /* cudaStream_t every call enqueues on (0 = legacy default stream) */
    void* workspace;           /* device memory, >= gorila_workspace_bytes(cfg), 256-B aligned */
    uint64_t workspace_bytes;
    int32_t optimizer;         /* gorila_optimizer */
    float lr;                  /* learning rate eta (2.5e-4, reading R2) */
    float rms_rho;             /* RMSProp decay of both averages (0.95) */
    float rms_eps;             /* RMSProp epsilon inside the sqrt (0.01) */
    float ada_eps;             /* AdaGrad epsilon outside the sqrt (1e-8) */
    int64_t target_period;     /* N: theta^- <- theta^+ once V >= last + N (Alg.1) */
    int64_t max_staleness;     /* discard iff V0 - base > max_staleness; < 0 disables */
    int32_t outlier_enabled;   /* discard batches with |loss| > mu + k*sigma */
    int32_t outlier_warmup;    /* batches observed before the filter may reject */
    float outlier_k;           /* "several standard deviations": k */
    double outlier_beta;       /* EMA decay of the running mean / variance */
    int64_t min_replay;        /* learner waits until size-1 >= max(1, min_replay) */
    uint64_t seed;             /* Philox key of the minibatch sampler */
    int32_t math;              /* gorila_math */
    int32_t history;           /* parameter-replica history depth H >= 1: learner_step accepts
                                  scheduled staleness s < H (deterministic fixed-staleness mode) */
    const float* theta0;       /* host, canonical layout, P floats: theta^+ = theta = theta^- at init (Alg.1) */
    int32_t ps_mode;           /* 0: aggregate, one optimizer step per round on the mean of the accepted
                                  gradients (reading R12); 1: per message (NEXT row f1, readings R32, R37):
                                  the learners' gradients arrive at the PS in ascending global learner id;
                                  each is discarded if stale against the version at its arrival (V0 + the
                                  messages applied before it), else applied as its own
                                  optimizer step (V += 1), after which every learner's target net
                                  syncs if V >= last + N, possibly inside the round: theta^- is
                                  theta^+ at that version. In this mode the stale / accepted fields of
                                  learner_step's info are provisional (accepted = message sent); the final
                                  decisions are in gorila_round's info and after ps_apply_shard, which also
                                  takes every learner's sync decisions (sync_target only reports them,
                                  unless force). 1 needs world == 1 or the peer-memory exchange (E_INVALID
                                  on the NCCL fallback) and world * n_learners_local <= 64. */
    int32_t replay_mode;       /* 0: local, each learner samples its own ring (P:140 first form);
                                  1: global (NEXT row f4, reading R36): every minibatch is drawn uniformly
                                  from the union D of all learners' rings on all ranks ("a global replay
                                  memory aggregates the experience into a distributed database", P:140;
                                  "sampled from either a local or global experience replay memory D",
                                  P:142), gathered from peer HBM over NVLink. Needs learner_id_base ==
                                  rank * n_learners_local, world * n_learners_local <= 256 and, when
                                  world > 1, the peer-memory mapping (E_INVALID otherwise). learner_step,
                                  gorila_round and replay_sample then start with a device barrier over
                                  the ranks (COLLECTIVE): inserts issued before them on any rank are
                                  part of D. */
} gorila_config;

/* Per-learner outcome of one learner_step (Alg.1). */
typedef struct {
    float loss;               /* mean delta^2 over the batch (Eq.1; reading R6) */
    float abs_loss;           /* mean |delta| — the outlier statistic (reading R7) */
    double mu, var;           /* running stats AFTER this batch (reading R8) */
    double threshold;         /* mu + k*sigma BEFORE this batch (the decision threshold) */
    uint64_t base_version;    /* V of the replica the gradient was computed on */
    uint32_t stats_count;     /* batches observed before this one */
    uint8_t not_ready;        /* replay below warm-up: no batch, no gradient */
    uint8_t rejected_outlier; /* discarded by the loss filter (learner side) */
    uint8_t stale;            /* discarded by the staleness rule (PS side) */
    uint8_t accepted;         /* contributed to this round's update */
} gorila_learner_info;

/* Outcome of one ps_apply_shard. */
typedef struct {
    uint32_t n_accepted;      /* |Acc|: learner gradients applied this round (all ranks) */
    uint32_t pad_;
    uint64_t version_before;  /* V0 */
    uint64_t version_after;   /* V0 + |Acc| (reading R12) */
} gorila_round_info;

/* P for nA actions (closed form from P:182). */
GORILA_API int64_t gorila_param_count(int32_t n_actions);
/* Device workspace bytes cfg needs (all learners' replay included). */
GORILA_API uint64_t gorila_workspace_bytes(const gorila_config* cfg);
/* Validate cfg, carve the workspace, set theta^+ = theta = theta^- = theta0,
 * m = v = 0, V = 0, last_sync = 0, empty loss stats, empty replays. When world > 1
 * with an NCCL id: create the communicator and map the peers' workspaces (collective);
 * without one, the caller connects the peers afterwards (gorila_peer_connect).
 * Synchronises the stream. */
GORILA_API gorila_status gorila_init(const gorila_config* cfg, gorila_ctx** out);
GORILA_API void gorila_destroy(gorila_ctx* ctx);
GORILA_API const char* gorila_last_error(void);

/* Store steps (o_t, a_t, r_t, d_t) for t = n .. n+count-1 into local learner
 * `learner`'s frame ring (slot t mod C; Alg.1 P:119 "Store ... in D"; P:140
 * local replay; reading R14). frames: count*84*84 u8 (row-major 84x84 each,
 * "84x84" preprocessed luminance); actions u8 (< nA, else E_RANGE is
 * NOT checked on device data), rewards f32, terminals u8 (d_t = 1 iff s_{t+1}
 * is terminal, Alg.1). src_on_device != 0: all four are device pointers,
 * read asynchronously on the library stream: the caller must not overwrite them
 * until that stream has passed this call (order its own stream after ours, as
 * the Python binding does). Host pointers are copied before the call returns:
 * up to 4 MB into a pinned staging ring allocated by gorila_init (no stream
 * synchronisation; a scatter kernel reads slots up to 64 KB over the bus and
 * larger ones after one upload), beyond that with a stream synchronisation. */
GORILA_API gorila_status replay_insert(gorila_ctx* ctx, int32_t learner, int64_t count, const uint8_t* frames,
                            const uint8_t* actions, const float* rewards, const uint8_t* terminals,
                            int32_t src_on_device);

/* Draw and gather learner `learner`'s minibatch for `round` exactly as
 * learner_step does ("sampled uniformly from the replay memory D", §3.3;
 * Alg.1): tau_i uniform over [n-size, n-2] from Philox4x32-10, then
 * s_i = stack(tau_i), s'_i = stack(tau_i + 1) (4 frames, oldest first, P:181,
 * zero-padded across episode ends and evicted slots, reading R15). Outputs
 * (host pointers, each may be NULL): idx_out int64[B] (absolute step tau_i),
 * s_out / s2_out u8 [B][4][84][84], a_out u8[B], r_out f32[B], d_out u8[B].
 * Returns E_NOT_READY (no side effects) if size-1 < max(1, min_replay).
 * Synchronises the stream (parity / debugging entry point). */
/* The shard of each sample of the most recent draw (replay_sample, or the last learner of
 * learner_step): the global learner id whose ring it was gathered from (global replay), 0 in
 * local mode. shard_out: host int32[B]. Synchronises the stream. */
GORILA_API gorila_status replay_sample_shards(gorila_ctx* ctx, int32_t* shard_out);
GORILA_API gorila_status replay_sample(gorila_ctx* ctx, int32_t learner, uint64_t round, int64_t* idx_out,
                            uint8_t* s_out, uint8_t* s2_out, uint8_t* a_out, float* r_out,
                            uint8_t* d_out);

/* One learner update for each listed local learner (Alg.1):
 * theta <- replica of round max(round - s_j, 0) (fixed-staleness schedule
 * s_j = staleness[j] or 0 if staleness == NULL, s_j < history), sample, online
 * forward Q(s;theta), target forward Q(s';theta^-_j), y = r or r + gamma max Q(s')
 * (P:122-126), delta = y - Q(s,a), loss, outlier decision + EMA update,
 * stale decision V0 - base > max_staleness, backward of Eq.2
 * with delta clipped to [-1,1] (BASELINE north_star; reading R3) unless discarded,
 * and accumulation into this rank's gradient buffer. learners: local ids
 * (ascending, each at most once); n >= 1. info_out: n entries or NULL.
 * Rounds must be issued in increasing order; one learner_step per round. */
GORILA_API gorila_status learner_step(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                           const int32_t* staleness, gorila_learner_info* info_out);

/* Parameter-server step for `round` ("split disjointly across N_param
 * machines", "applies the updates that are accumulated from many
 * learners"; reading R12): the gradient slices of this rank's shard summed in
 * rank order, one optimizer step on the shard with the mean of the accepted
 * gradients (skipped if none), V += |Acc|, and the updated slice broadcast into
 * every rank's next replica (Alg.1 P:116/"Update theta from theta^+").
 * When world > 1 this is one kernel reading and writing the peers' workspaces
 * over NVLink (k_apply_p2p); without peer mappings, NCCL reduce-scatter +
 * all-gather. COLLECTIVE. info_out may be NULL. */
GORILA_API gorila_status ps_apply_shard(gorila_ctx* ctx, uint64_t round, gorila_round_info* info_out);

/* Target sync (Alg.1 P:130 "Every global N steps sync theta^- with theta^+";
 * P:158-160 N counts PS updates; reading R13): for each listed local learner,
 * if force or V >= last_j + N then theta^-_j <- theta^+ and last_j <- V. The
 * predicate is evaluated on the device (no host sync). synced_out: n bytes or NULL. */
GORILA_API gorila_status sync_target(gorila_ctx* ctx, const int32_t* learners, int32_t n, int32_t force,
                          uint8_t* synced_out);

/* One whole round = learner_step + ps_apply_shard + sync_target(force = 0) for
 * the listed learners, replayed from a CUDA graph captured on first reuse (key:
 * learner list, staleness schedule, replica slot round mod history). Semantics
 * are exactly those of the three calls in sequence; rounds with a not-ready
 * learner (or round < max staleness) run them eagerly instead. Outputs (each may
 * be NULL) are copied after the round: info n entries, round_info, synced n
 * bytes; any non-NULL output synchronises the stream. COLLECTIVE. */
GORILA_API gorila_status gorila_round(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                                      const int32_t* staleness, gorila_learner_info* info_out,
                                      gorila_round_info* round_info_out, uint8_t* synced_out);
/* As gorila_round, but the result copies (info_out, round_info_out, synced_out) are only
 * enqueued on the library stream: they must point to pinned host (or device) memory that
 * stays valid until the stream passes them (synchronise the stream or an event recorded on
 * it after this call). Lets a caller read round k's result while round k+1 runs. When every
 * output is device-accessible (pinned, mapped or device memory) and n <= 11, one small kernel
 * stores them; otherwise they are copy-engine copies (pageable memory then serialises). */
GORILA_API gorila_status gorila_round_async(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                                           const int32_t* staleness, gorila_learner_info* info_out,
                                           gorila_round_info* round_info_out, uint8_t* synced_out);
/* Posted round: gorila_round's semantics, and the round's results (learner infos, round info,
 * sync flags) are stored by the round's own last kernel into slot round % 16 of a library-owned
 * pinned result ring (no copy operation outside the round's CUDA graph). gorila_round_fetch
 * waits for that slot by polling host memory (no CUDA call; a failed stream is reported as its
 * CUDA error) and copies it out: info_out n entries, round_info_out, synced_out n bytes (each may
 * be NULL; n = the posted round's learner count). Fetch a round before 16 further rounds are
 * posted (E_INVALID: overwritten). At most 32 learners per posted round (E_SHAPE). COLLECTIVE
 * as gorila_round. */
GORILA_API gorila_status gorila_round_post(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                                           const int32_t* staleness);
GORILA_API gorila_status gorila_round_fetch(gorila_ctx* ctx, uint64_t round, gorila_learner_info* info_out,
                                            gorila_round_info* round_info_out, uint8_t* synced_out);

/* State access for checkpointing and teacher-forced parity (canonical layout,
 * host buffers, any may be NULL; synchronises the stream). m / v are the full
 * optimizer state vectors (world == 1), or zeros outside this rank's shard.
 * stats: per local learner {mu, var, count(as double), last_sync(as double)}. */
GORILA_API gorila_status gorila_get_state(gorila_ctx* ctx, float* theta, float* m, float* v, uint64_t* version);
GORILA_API gorila_status gorila_set_state(gorila_ctx* ctx, const float* theta, const float* m, const float* v,
                               uint64_t version);
GORILA_API gorila_status gorila_get_learner_state(gorila_ctx* ctx, int32_t learner, float* theta_minus,
                                       double* stats4);
GORILA_API gorila_status gorila_set_learner_state(gorila_ctx* ctx, int32_t learner, const float* theta_minus,
                                       const double* stats4);
/* The gradient buffer G (canonical layout, sum over this rank's accepted
 * learners of the last learner_step, before the reduce-scatter). */
GORILA_API gorila_status gorila_get_grad(gorila_ctx* ctx, float* g);
/* Q and Q-hat [B][nA] of the last learner_step of local learner `learner`. */
GORILA_API gorila_status gorila_get_q(gorila_ctx* ctx, int32_t learner, float* q, float* qhat);
/* NEXT row f3 (acting). epsilon-greedy actions for n <= batch stacked states on the
 * latest theta^+ replica (Alg.1 P:118 "select a_t with the epsilon-greedy policy on
 * Q(s; theta)"; P:187 epsilon annealed linearly from 1 to eps_final over anneal_steps
 * global steps). states: u8 [n][4][84][84] (replay_sample's s layout), device pointer if
 * states_on_device else host. Per state i, x = Philox4x32-10(ctr = {i, actor_id,
 * step lo, (step hi & 0xffffff) | 5 << 24}, key = seed): explore iff x0 < eps * 2^32
 * (fp64), action = floor(x1 * nA / 2^32); else the argmax of Q with the lowest index on
 * ties. actions_out: host int32 [n]; q_out (nullable): host f32 [n][nA]. Synchronises the
 * library stream; uses the learner scratch (not concurrently with learner_step).
 * E_SHAPE if n < 1 or n > batch. */
GORILA_API gorila_status gorila_act(gorila_ctx* ctx, const uint8_t* states, int32_t n, uint64_t global_step,
                                    uint64_t actor_id, double eps_final, int64_t anneal_steps,
                                    int32_t states_on_device, int32_t* actions_out, float* q_out);
/* Intermediate tensors of the last learner step (diagnostics; the scratch is
 * shared by the local learners, so this is the last learner that ran). which:
 * 0 s, 1 a1, 2 a2, 3 a3 (NHWC [B][H][W][C], element type of the math mode:
 * bf16 as uint16 or fp32), 4 a4 ([B][512] fp32), 5 g1, 6 g2, 7 g3, 8 g4 (the
 * masked output gradients, same layouts / types as a1..a4 except g4 in the math
 * type). bytes must equal the tensor size (GORILA_E_SHAPE otherwise); host is a
 * host pointer; the call synchronises the library stream. */
GORILA_API gorila_status gorila_get_activation(gorila_ctx* ctx, int32_t which, void* host, uint64_t bytes);
/* Parity diagnostics (teacher-forced ReLU decisions, R30): enable != 0 makes every
 * later learner_step copy each learner's a1..a3 (NHWC, math type) and a4 ([B][512] fp32) after its
 * forward into a per-learner buffer (cudaMalloc'ed by the library on first enable, L x the
 * activation bytes; freed by gorila_destroy); 0 stops the copies. Drops the cached round graphs.
 * gorila_get_learner_activation reads learner `learner`'s copy of its last step: which 1..4 =
 * a1..a4 with gorila_get_activation's layouts and sizes (E_SHAPE on a size mismatch, E_RANGE on a
 * bad learner / which, E_INVALID while capture is off); synchronises the library stream. */
GORILA_API gorila_status gorila_capture_activations(gorila_ctx* ctx, int32_t enable);
GORILA_API gorila_status gorila_get_learner_activation(gorila_ctx* ctx, int32_t learner, int32_t which, void* host,
                                                       uint64_t bytes);
/* Per-phase device timing (diagnostics for the roofline report). When enabled,
 * learner_step / ps_apply_shard / sync_target record a CUDA event after each
 * phase on the stream; gorila_profile_read synchronises, returns the summed
 * milliseconds per phase (n entries, phase names from gorila_profile_phase_name)
 * and the number of learner steps covered, and resets the accumulators. */
GORILA_API gorila_status gorila_profile_enable(gorila_ctx* ctx, int32_t enable);
GORILA_API gorila_status gorila_profile_read(gorila_ctx* ctx, double* ms, int32_t n, uint64_t* n_steps);
GORILA_API int32_t gorila_profile_phase_count(void);
GORILA_API const char* gorila_profile_phase_name(int32_t i);
/* Diagnostics: re-launch the kernels of one phase (index < gorila_profile_phase_count();
 * learner phases act on local learner `learner`'s buffers from its last learner_step)
 * `iters` times back-to-back on the stream and return the mean device time per
 * repetition in microseconds (CUDA events; warm L2; launches overlap through PDL as in a
 * round). Results written by the repeated kernels are scratch: call it outside the
 * parity-checked sequence. Synchronises the stream. */
GORILA_API gorila_status gorila_bench_phase(gorila_ctx* ctx, int32_t learner, int32_t phase, int32_t iters,
                                            double* us_per_iter);
/* Diagnostics build only (-DGORILA_TRACE): clock64 timeline of CTA (0,0,0) of the last GEMM. */
GORILA_API gorila_status gorila_debug_trace(uint64_t* out64);
/* Diagnostics build only: per-tile events of CTA 0 of the last shifted-window GEMM, out512[ev * 64 +
 * tile] (clock64; ev 0/1 converter start / buffer handed over, 2/3/4 MMA operands ready / accumulator
 * free / issued, 5/6/7 epilogue wait / accumulator ready / done). E_INVALID in the normal build. */
GORILA_API gorila_status gorila_debug_trace_tiles(uint64_t* out512);
/* NEXT row f2: the asynchronous parameter server (config.ps_mode == 2; §3.1, P:144,
 * P:165-169). Runs `steps` learner steps for each listed local learner (ascending ids; round robin on
 * the library stream, rounds round0 .. round0 + steps - 1 for the sampler) while this rank's shard is
 * served by a persistent kernel of server_blocks blocks (<= 0: 32) on a second stream. A learner step
 * fetches the live replica (waiting only until its own previous message was consumed), records every
 * shard's live version as its base, syncs its target net if min V >= last + N, runs the learner update
 * and sends one message per shard unless outlier-rejected. Each shard's server applies messages in
 * arrival order, discarding those with V_arrival - base > max_staleness, one optimizer
 * step each (V += 1). Nothing orders learners and servers beyond those device counters: the result is
 * not deterministic and has no parity oracle (throughput and discard statistics); the deterministic
 * modes stay the parity path. COLLECTIVE when world > 1 (peer-memory mapping required). Returns after
 * every rank's messages are drained; the deterministic entry points (learner_step, ps_apply_shard,
 * gorila_round) return E_INVALID in this mode. out (may be NULL): counts and observed delays. */
typedef struct {
    uint64_t steps;          /* learner steps run on this rank */
    uint64_t sent;           /* messages sent by this rank's learners (to every shard) */
    uint64_t fresh, stale;   /* messages applied / discarded by this rank's shard */
    uint64_t rejected;       /* this rank's outlier-rejected steps (no message) */
    uint64_t version_after;  /* this shard's version at the end */
    uint64_t max_delay;      /* largest V_arrival - base this shard saw */
    double mean_delay;       /* mean V_arrival - base over this shard's messages */
} gorila_async_stats;
GORILA_API gorila_status gorila_async_run(gorila_ctx* ctx, const int32_t* learners, int32_t n, int64_t steps,
                                          uint64_t round0, int32_t server_blocks, gorila_async_stats* out);

/* Writes a fresh 128-byte ncclUniqueId (rank 0 calls it and broadcasts the bytes). */
GORILA_API gorila_status gorila_nccl_unique_id(void* out128);
/* Caller-bootstrapped exchange (world > 1 and config.nccl_unique_id == NULL; e.g. a gloo process
 * group, or several ranks sharing one GPU, where NCCL cannot form a communicator): after
 * gorila_init, every rank writes its 128-byte peer record (the CUDA IPC handle of its workspace
 * allocation + the workspace's offset in it) with gorila_peer_record, the caller all-gathers the
 * records in rank order, and every rank passes all `world` of them to gorila_peer_connect, which
 * maps every peer's workspace ("split disjointly": each shard owner then reads the peers'
 * gradient slices and writes the new replica chunks over NVLink peer memory, k_apply_p2p). Until
 * then learner_step / ps_apply_shard / replay_sample return E_INVALID. E_CUDA if the workspace
 * cannot be exported or a peer's cannot be opened (nothing stays mapped; the caller should agree
 * on the outcome across ranks); E_SHAPE if world differs from config.world; world <= 8. */
GORILA_API gorila_status gorila_peer_record(gorila_ctx* ctx, void* out128);
GORILA_API gorila_status gorila_peer_connect(gorila_ctx* ctx, const void* records, int32_t world);
/* Number of kernels this library launched so far (evidence counter). */
GORILA_API uint64_t gorila_kernel_launches(gorila_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
