// async.cuh — NEXT row f2: the asynchronous parameter server (ps_mode 2).
//
// The paper's Gorila is asynchronous SGD (§3.1; §4): learners compute
// gradients on whatever parameters they last fetched and send them to the parameter-server shards,
// which apply each one when it arrives; a shard "discards gradients that are older than a
// threshold" — the safeguard against "disappearing nodes, slowdowns".
//
// Here each rank's shard is served by a persistent kernel (k_ps_server, a few dozen blocks beside
// the learners) that drains a device message queue in arrival order: block 0 takes the stale /
// fresh decision of message m against the shard's live version V (applied messages so far), every
// block applies a fresh message to its own element range of the shard (so blocks never wait for
// each other; per element the messages stay in arrival order) and emits the new values into every
// rank's live replica; the last block to finish a message bumps V and marks the learner's gradient
// buffer consumed. Learners run on their own stream: fetch (wait until their previous message is
// consumed everywhere, read every shard's V, copy the live replica, target sync if V >= last + N),
// the learner step on the fetched copy, and send (one queue ticket per shard, an atomic on the
// shard owner's memory over NVLink when it is a peer). Nothing is ordered between learners and
// servers except through these device counters, so staleness is whatever the hardware produces.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace gorila {

constexpr int QCAP = 256;  // > every learner's one outstanding message (<= 64): a ticket's slot is free
struct AsyncMsg {
    uint64_t seq;       // ticket + 1 once the message is written (0: free)
    uint64_t decision;  // (ticket + 1) << 1 | fresh, published by server block 0
    uint64_t base;      // the shard's version the learner fetched (its replica's version)
    int32_t gid, pad_;
};
struct AsyncState {            // one per rank: its shard's queue and counters, its learners' flags
    uint64_t tail;             // tickets taken (learners of every rank, atomics over NVLink)
    uint64_t V;                // live shard version = fresh messages applied
    uint64_t n_fresh, n_stale; // server counters
    uint64_t ranks_done;       // ranks whose learners sent their last message
    uint64_t max_delay_seen;   // largest V - base at arrival (fresh or stale)
    uint64_t delay_sum;        // sum of V - base over all messages (mean staleness)
    uint64_t n_rejected;       // this rank's outlier-rejected learner steps (learner side)
    uint64_t progress;         // learner-side kernels completed on this rank (fetch, send): diagnostics
    uint64_t err;              // nonzero: a bounded wait timed out (1 server: message, 2 server: decision,
                               // 3 learner: its previous message not consumed) -- reported, never a hang
    uint64_t sent[32];         // per local learner: messages sent
    uint64_t consumed[MAX_W][32];  // [shard][local learner]: messages applied / discarded by that shard
    uint64_t base[32][MAX_W];  // per local learner: the shards' versions at its last fetch
    AsyncMsg ring[QCAP];
    uint32_t done_cnt[QCAP];
};

struct ServerParams {
    ApplyParams p;               // this shard's slice (theta, m, v), optimizer constants, nA, base, n_real
    AsyncState* st;              // this rank's state
    const float* G[MAX_MSG];     // global learner's gradient buffer at this shard's slice (this process)
    uint64_t* consumed[MAX_MSG]; // &consumed[this shard][local id] on the learner's rank (this process)
    void* live_t[MAX_W];         // every rank's live replica (T area, fp32 area)
    float* live_f[MAX_W];
    int W;
    int64_t max_delay;
};

template <typename T>
__global__ void __launch_bounds__(256) k_ps_server(ServerParams sp) {
    AsyncState* st = sp.st;
    const ApplyParams& p = sp.p;
    __shared__ int s_exit;
    __shared__ uint64_t s_dec;
    __shared__ int s_gid;
    const int64_t n4 = (p.n_real + 3) / 4;
    const int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(n4, lo + per);
    uint64_t applied = ld_acquire_sys(&st->V);  // block 0: the version a message arrives at
    for (uint64_t m = 0;; ++m) {
        AsyncMsg* msg = &st->ring[m % QCAP];
        if (threadIdx.x == 0) {
            for (uint32_t n = 0;; ++n) {
                if (ld_acquire_sys(&msg->seq) == m + 1) {
                    s_exit = 0;
                    break;
                }
                // every rank finished sending and no ticket beyond m was taken: drained
                if (ld_acquire_sys(&st->ranks_done) == (uint64_t)sp.W && ld_acquire_sys(&st->tail) == m) {
                    s_exit = 1;
                    break;
                }
                if (n > (1u << 26) || ld_acquire_sys(&st->err)) {  // tens of seconds without a message
                    atomicCAS(reinterpret_cast<unsigned long long*>(&st->err), 0ull, 1ull);
                    s_exit = 1;
                    break;
                }
                __nanosleep(n < 64 ? 32 : 256);
            }
            if (!s_exit) {
                if (blockIdx.x == 0) {  // discard if older than the threshold at arrival
                    const uint64_t delay = applied - msg->base;
                    const bool fresh = !(sp.max_delay >= 0 && (int64_t)delay > sp.max_delay);
                    applied += fresh ? 1 : 0;
                    st->delay_sum += delay;
                    if (delay > st->max_delay_seen) st->max_delay_seen = delay;
                    st_release_sys(&msg->decision, ((m + 1) << 1) | (fresh ? 1ull : 0ull));
                }
                uint64_t d;
                for (uint32_t n = 0; ((d = ld_acquire_sys(&msg->decision)) >> 1) != m + 1; ++n) {
                    if (n > (1u << 26)) {
                        atomicCAS(reinterpret_cast<unsigned long long*>(&st->err), 0ull, 2ull);
                        s_exit = 1;
                        break;
                    }
                    __nanosleep(32);
                }
                s_dec = d & 1ull;
                s_gid = msg->gid;
            }
        }
        __syncthreads();
        if (s_exit) break;
        if (s_dec) {
            const float4* g4 = reinterpret_cast<const float4*>(sp.G[s_gid]);
            for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
                float4 th = reinterpret_cast<float4*>(p.theta)[e];
                float4 mm = reinterpret_cast<float4*>(p.m)[e];
                float4 vv4 = reinterpret_cast<float4*>(p.v)[e];
                float tv[4] = {th.x, th.y, th.z, th.w}, mv[4] = {mm.x, mm.y, mm.z, mm.w},
                      vv[4] = {vv4.x, vv4.y, vv4.z, vv4.w};
                opt_step4(p, tv, mv, vv, __ldcg(g4 + e));
                reinterpret_cast<float4*>(p.theta)[e] = make_float4(tv[0], tv[1], tv[2], tv[3]);
                reinterpret_cast<float4*>(p.m)[e] = make_float4(mv[0], mv[1], mv[2], mv[3]);
                reinterpret_cast<float4*>(p.v)[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
                for (int q = 0; q < sp.W; ++q) emit4_to<T>(sp.live_t[q], sp.live_f[q], p.nA, p.base + 4 * e, tv);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // the last block to finish message m publishes it
            __threadfence_system();
            const uint32_t prev = atomicAdd(&st->done_cnt[m % QCAP], 1u);
            if (prev == gridDim.x - 1) {
                st->done_cnt[m % QCAP] = 0;
                if (s_dec) {
                    st->n_fresh += 1;
                    st_release_sys(&st->V, ld_acquire_sys(&st->V) + 1);
                } else {
                    st->n_stale += 1;
                }
                msg->seq = 0;  // the slot is free again
                __threadfence_system();
                uint64_t* c = sp.consumed[s_gid];
                st_release_sys(c, ld_acquire_sys(c) + 1);
            }
        }
    }
}

struct FetchParams {
    AsyncState* st;               // this rank's state
    const uint64_t* V[MAX_W];     // every shard's live version (this process's address)
    int W, j;                     // local learner
    LearnerStats* stats;          // its target-sync state
    uint8_t* sync_flag;
    DevLearnerInfo* info;
    int64_t period;
    uint64_t* vhist;              // the fetched replica's version record (learner step's base_V)
};
// learner j, before its step: its previous message consumed by every shard (its gradient buffer is
// free), then the shards' versions (the fetched replica's base) and the target-sync decision on the
// smallest of them (N updates applied by the PS); the replica copy follows.
__global__ void k_async_fetch(FetchParams f) {
    pdl_wait();
    pdl_trigger();
    AsyncState* st = f.st;
    const uint64_t want = st->sent[f.j];
    for (int s = 0; s < f.W; ++s)
        for (uint32_t n = 0; ld_acquire_sys(&st->consumed[s][f.j]) < want; ++n) {
            if (n > (1u << 26) || ld_acquire_sys(&st->err)) {
                atomicCAS(reinterpret_cast<unsigned long long*>(&st->err), 0ull, 3ull);
                break;
            }
            __nanosleep(64);
        }
    uint64_t vmin = ~0ull;
    for (int s = 0; s < f.W; ++s) {
        const uint64_t v = ld_acquire_sys(f.V[s]);
        st->base[f.j][s] = v;
        vmin = v < vmin ? v : vmin;
    }
    *f.vhist = vmin;
    st->progress += 1;
    const bool doit = vmin >= f.stats->last_sync + (uint64_t)f.period;
    if (doit) f.stats->last_sync = vmin;
    *f.sync_flag = doit;
}

struct SendParams {
    AsyncState* st;               // this rank's state
    AsyncState* shard[MAX_W];     // every shard's state (this process's address)
    int W, j, gid;
    const DevLearnerInfo* info;
};
// learner j, after its step: one message per shard unless its minibatch was outlier-rejected
__global__ void k_async_send(SendParams s) {
    pdl_wait();
    pdl_trigger();
    AsyncState* st = s.st;
    st->progress += 100;
    if (!s.info->accepted) {  // rejected (or not ready): no message
        st->n_rejected += s.info->rejected_outlier ? 1 : 0;
        return;
    }
    st->sent[s.j] += 1;
    for (int q = 0; q < s.W; ++q) {
        AsyncState* sh = s.shard[q];
        const uint64_t t = atomicAdd(reinterpret_cast<unsigned long long*>(&sh->tail), 1ull);
        AsyncMsg* msg = &sh->ring[t % QCAP];
        msg->base = st->base[s.j][q];
        msg->gid = s.gid;
        __threadfence_system();
        st_release_sys(&msg->seq, t + 1);
    }
}

// every shard: this rank's learners are done (the servers drain and exit)
__global__ void k_async_done(SendParams s) {
    pdl_wait();
    pdl_trigger();
    __threadfence_system();
    for (int q = 0; q < s.W; ++q) atomicAdd(reinterpret_cast<unsigned long long*>(&s.shard[q]->ranks_done), 1ull);
}

__global__ void k_copy_u64(uint64_t* dst, const uint64_t* src) { *dst = *src; }

// every rank reached this point of gorila_async_run (epoch ep): flags[q][FLAG_ASYNC + rank] = ep
__global__ void k_async_barrier(P2PParams x, uint64_t ep) {
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x != 0) return;
    __threadfence_system();
    for (int q = 0; q < x.W; ++q)
        if (q != x.rank) st_release_sys(x.flags[q] + FLAG_ASYNC + x.rank, ep);
    for (int q = 0; q < x.W; ++q)
        if (q != x.rank) wait_flag(x.flags[x.rank] + FLAG_ASYNC + q, ep);
}

}  // namespace gorila
