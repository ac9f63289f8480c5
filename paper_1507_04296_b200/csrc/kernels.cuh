// kernels.cuh — the non-GEMM kernels of the learner update (SIMT, HBM / latency bound).
#pragma once
#include "common.cuh"
#include "layout.cuh"

namespace gorila {

constexpr uint32_t TAG_SAMPLE = 3u;
constexpr int RING_MAXL = 32, RING_HDR = 8 + 8 + 24 + 64;  // result ring slot: see k_emit_ring

// one learner's replay ring as seen from this rank (local or a peer's, mapped over NVLink)
struct ShardPtrs {
    const uint8_t* frames;
    const uint8_t* a;
    const float* r;
    const uint8_t* d;
    const uint64_t* n;  // steps inserted so far (device counter)
};
constexpr int MAX_SHARDS = 256;

// u8 path (large batches): per sample, the addresses of the five ring frames tau-3 .. tau+1 and the
// episode / eviction masks. conv1's forward and weight-gradient operands gather their input straight
// from the replay ring through these (shift_gemm.cuh U8Planes): no stacked copy of s / s' is written.
// s channel c = frame[c], s' channel c = frame[c + 1]; keep bit c (s) / 4 + c (s'): 0 = zero channel.
struct SampleDesc {
    const uint8_t* frame[5];
    uint32_t keep;
    uint32_t pad_;
};


// ------------------------------------------------------------------------- K1 sampler
// Alg.1 P:121 "Sample random mini-batch from D"; "(s,a,r,s') ~ U(D)"; P:181 4-frame stack.
// Block (cx, b): tau_b from Philox4x32-10 (counter {b/2, learner, round lo, round hi | TAG}),
// tau = (n - size) + floor(u * (size-1) / 2^64); thread = one 16-pixel chunk of the 84x84
// frame: reads the 5 frames o_{tau-3} .. o_{tau+1} (16 B each, coalesced), applies the
// episode / eviction zero mask and writes s, s' as NHWC [B][84][84][4] in T.
// Global replay (NEXT row f4, reading R36; tab != nullptr): the draw is over the union of the G
// shards' valid transitions, T = sum_j (size_j - 1), g = floor(u * T / 2^64), and (shard, tau) is
// the g-th transition in (shard, tau) order; the gather then reads that shard's ring, local or in
// a peer's HBM over NVLink. G = 1 is exactly the local draw.
template <typename T>
__global__ void __launch_bounds__(256) k_sample(const uint8_t* __restrict__ frames, const uint8_t* __restrict__ ring_a,
                                                const float* __restrict__ ring_r, const uint8_t* __restrict__ ring_d,
                                                int64_t C, const uint64_t* __restrict__ ring_n,
                                                const ShardPtrs* __restrict__ tab, int G,
                                                const uint64_t* __restrict__ n_snap, int32_t* __restrict__ shard_out,
                                                uint2 key,
                                                uint32_t learner_gid, const uint64_t* __restrict__ round_ptr, int B,
                                                T* __restrict__ s_out,
                                                T* __restrict__ s2_out, uint8_t* __restrict__ a_out,
                                                float* __restrict__ r_out, uint8_t* __restrict__ d_out,
                                                int64_t* __restrict__ idx_out, uint32_t* __restrict__ n_acc_reset) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    if (n_acc_reset && b == 0 && blockIdx.x == 0 && threadIdx.x == 0) *n_acc_reset = 0;  // first learner of a round
    const uint64_t round = *round_ptr;  // device-resident round counter (graph replay friendly)
    const uint4 x = philox4x32_10(make_uint4((uint32_t)(b >> 1), learner_gid, (uint32_t)round,
                                             (uint32_t)((round >> 32) & 0xffffffu) | (TAG_SAMPLE << 24)),
                                  key);
    const uint64_t u = (b & 1) ? ((uint64_t)x.z | ((uint64_t)x.w << 32)) : ((uint64_t)x.x | ((uint64_t)x.y << 32));
    int64_t n, tau;
    int shard = 0;
#ifdef GORILA_TRACE
    long long tr[5] = {clock64(), 0, 0, 0, 0};
    bool tr_own = true;
#endif
    if (tab) {  // f4: every shard's counter (read after the round's replay barrier), then the union index
        __shared__ uint64_t s_n[MAX_SHARDS];
        __shared__ int64_t s_tau;
        __shared__ int s_shard;
        // world > 1: the counters every rank pushed into n_snap with its barrier flag (local reads)
        for (int j = threadIdx.x; j < G; j += blockDim.x)
            s_n[j] = n_snap ? n_snap[j] : *(volatile const uint64_t*)tab[j].n;
        __syncthreads();
#ifdef GORILA_TRACE
        tr[1] = clock64();
#endif
        if (threadIdx.x == 0) {
            uint64_t Tot = 0;
            for (int j = 0; j < G; ++j) {
                const int64_t sz = (int64_t)s_n[j] < C ? (int64_t)s_n[j] : C;
                Tot += sz >= 2 ? (uint64_t)(sz - 1) : 0;
            }
            const uint64_t g = __umul64hi(u, Tot);
            uint64_t pos = 0;
            for (int j = 0; j < G; ++j) {
                const int64_t nj = (int64_t)s_n[j], sz = nj < C ? nj : C;
                const uint64_t M = sz >= 2 ? (uint64_t)(sz - 1) : 0;
                if (g < pos + M) {
                    s_shard = j;
                    s_tau = (nj - sz) + (int64_t)(g - pos);
                    break;
                }
                pos += M;
            }
        }
        __syncthreads();
        shard = s_shard;
        tau = s_tau;
        n = (int64_t)s_n[shard];
#ifdef GORILA_TRACE
        tr[2] = clock64();
        tr_own = tab[shard].frames == frames;
#endif
        frames = tab[shard].frames;
        ring_a = tab[shard].a;
        ring_r = tab[shard].r;
        ring_d = tab[shard].d;
    } else {
        n = (int64_t)*ring_n;
        const int64_t size = n < C ? n : C;
        tau = (n - size) + (int64_t)__umul64hi(u, (uint64_t)(size - 1));
    }
    const int64_t size = n < C ? n : C;
    const int64_t oldest = n - size;

    // the four episode flags and a_tau / r_tau: loaded once per block (a peer's ring is read over
    // NVLink, where 441 threads re-reading the same bytes would be 441 remote requests each), and
    // issued before the frame loads so that they do not queue behind the frame traffic
    __shared__ uint8_t s_d[4], s_a;
    __shared__ float s_r;
    uint8_t dv = 1, av = 0;
    float rv = 0.f;
    if (threadIdx.x < 4) {
        const int64_t st = tau - 3 + threadIdx.x;
        if (st >= oldest) dv = __ldcg(ring_d + st % C);  // d_tau itself: tau >= oldest always
    } else if (threadIdx.x == 32) {
        av = __ldcg(ring_a + tau % C);
    } else if (threadIdx.x == 64) {
        rv = __ldcg(ring_r + tau % C);
    }
    const int chunk = blockIdx.x * blockDim.x + threadIdx.x;
    uint4 f[5];  // issued before the flags are used: the keep masks zero channels later
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        int64_t st = tau - 3 + t;
        f[t] = (sizeof(T) != 1 && st >= 0 && chunk < FRAME_BYTES / 16)  // (u8 path: no frame reads here)
                   ? __ldcg(reinterpret_cast<const uint4*>(frames + (st % C) * FRAME_BYTES + chunk * 16))
                   : make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x < 4) s_d[threadIdx.x] = dv != 0;
    else if (threadIdx.x == 32) s_a = av;
    else if (threadIdx.x == 64) s_r = rv;
    __syncthreads();
#ifdef GORILA_TRACE
    tr[3] = clock64();
#endif
    // keep[f] for frames tau-3+f, f = 0..4 (s uses f = 0..3, s' uses f = 1..4)
    bool keep_s[4], keep_s2[4];
    {
        bool dflag[4];  // d_{tau-3+t}, t = 0..3 (only used when the frame is retained)
#pragma unroll
        for (int t = 0; t < 4; ++t) dflag[t] = s_d[t] != 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            // s channel c = frame tau-3+c: zero if evicted or an episode ended at t' in [tau-3+c, tau-1]
            bool k = (tau - 3 + c) >= oldest;
            for (int t = c; t < 3; ++t) k = k && !dflag[t];
            keep_s[c] = k;
            // s' channel c = frame tau-2+c: zero if evicted or an episode ended at t' in [tau-2+c, tau]
            bool k2 = (tau - 2 + c) >= oldest;
            for (int t = c + 1; t < 4; ++t) k2 = k2 && !dflag[t];
            keep_s2[c] = k2;
        }
    }
    if constexpr (sizeof(T) == 1) {
        // u8 path: the sample's frame addresses and masks only (conv1's operands gather the frames)
        if (threadIdx.x == 0) {
            SampleDesc ds;
#pragma unroll
            for (int t = 0; t < 5; ++t) {
                const int64_t st = tau - 3 + t;  // frames before the ring start are never kept
                ds.frame[t] = frames + (st >= 0 ? st % C : 0) * FRAME_BYTES;
            }
            uint32_t keep = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) keep |= (keep_s[c] ? 1u : 0u) << c | (keep_s2[c] ? 1u : 0u) << (4 + c);
            ds.keep = keep;
            ds.pad_ = 0;
            reinterpret_cast<SampleDesc*>(s_out)[b] = ds;
        }
    } else if constexpr (sizeof(T) == 2) {
        // bf16: each thread's 16 pixels x 4 channels = 8 uint4 per stack, staged in shared memory
        // (rows XOR-rotated: conflict-free) and written out block-contiguously (every warp store one
        // 512-B run instead of 32 runs of 16 B at a 128-B stride)
        __shared__ uint4 stage[256 * 8];
        const uint8_t* fb[5];
#pragma unroll
        for (int t = 0; t < 5; ++t) fb[t] = reinterpret_cast<const uint8_t*>(&f[t]);
        const int nvalid = min(FRAME_BYTES / 16 - (int)(blockIdx.x * blockDim.x), (int)blockDim.x);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            if (chunk < FRAME_BYTES / 16) {
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float x2[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int el = v * 8 + 2 * e + h, px = el >> 2, c = el & 3;
                            const bool keep = half ? keep_s2[c] : keep_s[c];
                            x2[h] = keep ? (float)fb[c + half][px] : 0.f;
                        }
                        __nv_bfloat162 hh = __floats2bfloat162_rn(x2[0], x2[1]);
                        w[e] = *reinterpret_cast<uint32_t*>(&hh);
                    }
                    stage[threadIdx.x * 8 + ((v + threadIdx.x) & 7)] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
            __syncthreads();
            T* dst = (half ? s2_out : s_out) + ((int64_t)b * FRAME_BYTES + (int64_t)blockIdx.x * blockDim.x * 16) * NSTACK;
            for (int o = threadIdx.x; o < nvalid * 8; o += blockDim.x) {
                const int i = o >> 3, v = o & 7;
                reinterpret_cast<uint4*>(dst)[o] = stage[i * 8 + ((v + i) & 7)];
            }
            __syncthreads();
        }
    } else if (chunk < FRAME_BYTES / 16) {
        const uint8_t* fb[5];
#pragma unroll
        for (int t = 0; t < 5; ++t) fb[t] = reinterpret_cast<const uint8_t*>(&f[t]);
        T* so = s_out + ((int64_t)b * FRAME_BYTES + chunk * 16) * NSTACK;
        T* so2 = s2_out + ((int64_t)b * FRAME_BYTES + chunk * 16) * NSTACK;
        // NHWC: 16 pixels x 4 channels, written as 16-byte vectors
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            T* dst = half ? so2 : so;
#pragma unroll
            for (int v = 0; v < 64 * (int)sizeof(T) / 16; ++v) {  // 16-B vectors per 16 pixels
                float x[16 / sizeof(T)];
#pragma unroll
                for (int e = 0; e < (int)(16 / sizeof(T)); ++e) {
                    const int el = v * (16 / sizeof(T)) + e, px = el >> 2, c = el & 3;
                    const bool keep = half ? keep_s2[c] : keep_s[c];
                    x[e] = keep ? (float)fb[c + half][px] : 0.f;
                }
                if constexpr (sizeof(T) == 2) {
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
                        w[e] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    reinterpret_cast<uint4*>(dst)[v] = make_uint4(w[0], w[1], w[2], w[3]);
                } else {
                    reinterpret_cast<float4*>(dst)[v] = make_float4(x[0], x[1], x[2], x[3]);
                }
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a_out[b] = s_a;
        r_out[b] = s_r;
        d_out[b] = s_d[3];
        idx_out[b] = tau;
        if (shard_out) shard_out[b] = shard;
#ifdef GORILA_TRACE
        tr[4] = clock64();
        const int o = tr_own ? 0 : 8;
        for (int i = 1; i < 5; ++i) atomicAdd(&gorila_trace_buf[o + i - 1], (unsigned long long)(tr[i] - tr[i - 1]));
        atomicAdd(&gorila_trace_buf[o + 4], 1ull);
#endif
    }
}

// ------------------------------------------------------------------------- K7 TD + decisions
struct LearnerStats {  // device-resident per learner (reading R8)
    double mu, var;
    uint32_t count, pad_;
    uint64_t last_sync;
};

struct DevLearnerInfo {  // mirrors gorila_learner_info
    float loss, abs_loss;
    double mu, var, threshold;
    uint64_t base_version;
    uint32_t stats_count;
    uint8_t not_ready, rejected_outlier, stale, accepted;
};

struct TdParams {
    const float* Q;
    const float* Qhat;
    const uint8_t* a;
    const float* r;
    const uint8_t* d;
    float* dQ;
    int B, nA;
    float gamma;
    LearnerStats* stats;
    DevLearnerInfo* info;
    const uint64_t* V;        // V0 (PS version before this round's apply)
    const uint64_t* base_V;   // version of the replica used (history)
    uint32_t* n_acc_local;
    int64_t max_staleness;
    int outlier_enabled, outlier_warmup;
    float outlier_k;
    double outlier_beta;
};

// batch loss, outlier decision (on the pre-update stats) + EMA update (reading R8), stale decision
// (reading R10), info record and accepted count. One thread. Returns "accepted".
GORILA_DEV int td_decide(const TdParams& p, const float* s_sq, const float* s_ab, int nwarps) {
    float tsq = 0.f, tab = 0.f;
    for (int w = 0; w < nwarps; ++w) {
        tsq += s_sq[w];
        tab += s_ab[w];
    }
    const float loss = tsq / (float)p.B, ell = tab / (float)p.B;
    LearnerStats st = *p.stats;
    const double thr = st.mu + (double)p.outlier_k * sqrt(st.var);
    const bool rejected = p.outlier_enabled && st.count >= (uint32_t)p.outlier_warmup && (double)ell > thr;
    DevLearnerInfo inf{};
    inf.stats_count = st.count;
    if (st.count == 0) {
        st.mu = ell;
        st.var = 0.0;
    } else {
        const double e = (double)ell - st.mu;
        st.mu = st.mu + (1.0 - p.outlier_beta) * e;
        st.var = p.outlier_beta * (st.var + (1.0 - p.outlier_beta) * e * e);
    }
    st.count += 1;
    *p.stats = st;
    const uint64_t V0 = *p.V, base = *p.base_V;
    const bool stale = p.max_staleness >= 0 && (int64_t)(V0 - base) > p.max_staleness;
    const bool accepted = !rejected && !stale;
    inf.loss = loss;
    inf.abs_loss = ell;
    inf.mu = st.mu;
    inf.var = st.var;
    inf.threshold = thr;
    inf.base_version = base;
    inf.rejected_outlier = rejected;
    inf.stale = stale;
    inf.accepted = accepted;
    *p.info = inf;
    if (accepted) *p.n_acc_local += 1;
    return accepted;
}

// ------------------------------------------------------------------------- fc5 forward + K7
// Grid (B): block b computes Q(s_b, .) and Q-hat(s'_b, .) (fc5, fp32), the TD target, delta and
// dQ of sample b (Alg.1; reading R3), and its delta^2 / |delta| into per_sample[b];
// the last block to finish (device counter) sums the batch in sample order and takes the outlier
// and stale decisions (td_decide); a rejected batch has its dQ zeroed there.
struct Fc5TdParams {
    const float *a4, *t4, *w5, *b5, *w5t, *b5t;
    unsigned int* counter;  // zero between launches (the last block resets it)
    float* per_sample;      // [B][2]
    TdParams td;
    // fused fc5 backward (gridDim == B <= 32, every block resident): after the decision every block
    // writes its sample's g4 row and a column slice of the single-chunk fc5 gradient partial
    int fuse_bwd;
    unsigned int* gen;      // [2]: launch generation, decision-published generation
    float* part5;           // [nA * 513]
    void* g4;               // T [B][512]
    int bf16;               // g4 element type
};
// fused fc5 backward of one block (fuse_bwd): wait until the last block published the decision
// (dQ final), then this block's sample's g4 row and its column slice of dW5 / db5 (one chunk)
GORILA_DEV void fc5_bwd_fused(const Fc5TdParams& p, unsigned int gen) {
    if (threadIdx.x == 0)
        while (*(volatile unsigned int*)&p.gen[1] != gen + 1) __nanosleep(32);
    __syncthreads();
    __threadfence();
    const TdParams& t = p.td;
    const int B = t.B, nA = t.nA, b = blockIdx.x;
    __shared__ float dq[32 * 32];
    for (int i = threadIdx.x; i < B * nA; i += blockDim.x) dq[i] = __ldcg(&t.dQ[i]);
    __syncthreads();
    for (int n = threadIdx.x; n < FC4_OUT; n += blockDim.x) {  // g4[b][n] = mask(sum_a dQ[b][a] W5[a][n])
        float g = 0.f;
        for (int a = 0; a < nA; ++a) g = fmaf(dq[b * nA + a], p.w5[a * FC4_OUT + n], g);
        const float x = p.a4[(int64_t)b * FC4_OUT + n];
        const float v = x > 0.f ? g : 0.f;
        if (p.bf16) reinterpret_cast<__nv_bfloat16*>(p.g4)[(int64_t)b * FC4_OUT + n] = __float2bfloat16_rn(v);
        else reinterpret_cast<float*>(p.g4)[(int64_t)b * FC4_OUT + n] = v;
    }
    // dW5[a][n] = sum_b dQ[b][a] a4[b][n] for this block's columns; db5 by block 0
    const int per = (FC4_OUT + gridDim.x - 1) / gridDim.x, n0 = b * per, n1 = min(FC4_OUT, n0 + per);
    for (int e = threadIdx.x; e < nA * (n1 - n0); e += blockDim.x) {
        const int a = e / (n1 - n0), n = n0 + (e - a * (n1 - n0));
        float acc = 0.f;
        for (int bb = 0; bb < B; ++bb) acc = fmaf(dq[bb * nA + a], p.a4[(int64_t)bb * FC4_OUT + n], acc);
        p.part5[a * FC4_OUT + n] = acc;
    }
    if (b == 0 && (int)threadIdx.x < nA) {
        float sb = 0.f;
        for (int bb = 0; bb < B; ++bb) sb += dq[bb * nA + threadIdx.x];
        p.part5[nA * FC4_OUT + threadIdx.x] = sb;
    }
}

// 16 warps: warps 0..7 the online net, 8..15 the target net; every operand of a warp's (up to
// four) actions is requested before the first FMA (one memory round trip for the whole layer)
__global__ void __launch_bounds__(512) k_fc5_td(Fc5TdParams p) {
    const TdParams& t = p.td;
    const int nA = t.nA;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int z = warp >> 3, wz = warp & 7;
    __shared__ float q[2][2][32];  // [sample parity][net][action]
    // this warp's W5 rows stay in registers for all the block's samples
    const float* w5 = z ? p.w5t : p.w5;
    const float* b5 = z ? p.b5t : p.b5;
    float wv[4][FC4_OUT / 32];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int a = wz + 8 * u;
#pragma unroll
        for (int k = 0; k < FC4_OUT / 32; ++k) wv[u][k] = a < nA ? __ldcg(w5 + a * FC4_OUT + lane + 32 * k) : 0.f;
    }
    // W5 / b5 (the replica and theta^-) were written two or more kernels back: loaded before the
    // wait for fc4's output (PDL: the preceding kernel has passed its own wait when this one starts).
    // Loads issued before the wait go through L2 (ld.global.cg): an SM's L1 may still hold lines of
    // an older value of these addresses, and only the wait orders this grid after the flush
    float bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) bv[u] = wz + 8 * u < nA ? __ldcg(b5 + wz + 8 * u) : 0.f;
    pdl_wait();
    pdl_trigger();
    int it = 0;
    for (int b = blockIdx.x; b < t.B; b += gridDim.x, ++it) {
        const int par = it & 1;
        const float* x = (z ? p.t4 : p.a4) + (int64_t)b * FC4_OUT;
        float xv[FC4_OUT / 32];
#pragma unroll
        for (int k = 0; k < FC4_OUT / 32; ++k) xv[k] = x[lane + 32 * k];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int a = wz + 8 * u;
            if (a >= nA) break;
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < FC4_OUT / 32; ++k) acc = fmaf(xv[k], wv[u][k], acc);
            acc = warp_sum(acc);
            if (lane == 0) q[par][z][a] = acc + bv[u];
        }
        __syncthreads();
        if (warp == 0) {
            const float qv = lane < nA ? q[par][0][lane] : 0.f, qh = lane < nA ? q[par][1][lane] : -INFINITY;
            if (lane < nA) {
                const_cast<float*>(t.Q)[b * nA + lane] = qv;
                const_cast<float*>(t.Qhat)[b * nA + lane] = qh;
            }
            const float mx = warp_max(qh);
            const int ab = t.a[b];
            const float y = t.d[b] ? t.r[b] : t.r[b] + t.gamma * mx;  // Alg.1
            const float delta = y - q[par][0][ab];
            if (lane < nA) {
                const float cl = fminf(fmaxf(delta, -1.f), 1.f);  // reading R3
                t.dQ[b * nA + lane] = (lane == ab) ? -cl / (float)t.B : 0.f;
            }
            if (lane == 0) {
                p.per_sample[2 * b] = delta * delta;
                p.per_sample[2 * b + 1] = fabsf(delta);
            }
        }
        // the next sample writes the other parity of q: one barrier per sample suffices
    }
    __shared__ unsigned int s_last, s_gen;
    if (threadIdx.x == 0 && p.fuse_bwd) s_gen = *(volatile unsigned int*)&p.gen[0];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) {
        if (p.fuse_bwd) fc5_bwd_fused(p, s_gen);
        return;
    }
    __threadfence();
    // last block: fixed-order batch sums (8 interleaved partials, then in order), decisions
    __shared__ float s_sq[16], s_ab[16];
    __shared__ int s_keep;
    float sq = 0.f, sa = 0.f;
    for (int i = threadIdx.x; i < t.B; i += blockDim.x) {
        sq += __ldcg(&p.per_sample[2 * i]);
        sa += __ldcg(&p.per_sample[2 * i + 1]);
    }
    sq = warp_sum(sq);
    sa = warp_sum(sa);
    if (lane == 0) {
        s_sq[warp] = sq;
        s_ab[warp] = sa;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s_keep = td_decide(t, s_sq, s_ab, 16);
        *p.counter = 0;
    }
    __syncthreads();
    if (!s_keep)
        for (int e = threadIdx.x; e < t.B * nA; e += blockDim.x) t.dQ[e] = 0.f;
    if (p.fuse_bwd) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            p.gen[0] = s_gen + 1;                               // the next launch's generation
            atomicExch(&p.gen[1], s_gen + 1);                   // publish: dQ is final
        }
        fc5_bwd_fused(p, s_gen);
    }
}

// Large batches (B >= 256): the same fc5 forward + TD + decisions with one warp per S samples (both
// nets) instead of all warps on one sample at a time. W5 / W5t sit in shared memory (loaded before
// the PDL wait: written two or more kernels back); each W5 element read from shared memory feeds S
// FMAs, and three actions' warp sums are in flight together (the shuffles' latency, not the FMAs,
// bounds this kernel: 16 warps per block, S chosen so the grid fills the SMs). The last block sums
// the per-sample terms in sample order and decides (td_decide), as k_fc5_td.
constexpr int FC5W_WARPS = 16;
template <int S>
__global__ void __launch_bounds__(FC5W_WARPS * 32) k_fc5_td_wide(Fc5TdParams p) {
    const TdParams& t = p.td;
    const int nA = t.nA;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    extern __shared__ __align__(16) float sw[];  // [2][nA][512] weights, then [2][32] biases
    __shared__ __align__(8) uint64_t wbar;
    if (threadIdx.x == 0) {  // the two W5 matrices: one bulk copy each (contiguous [nA][512] fp32)
        mbar_init(&wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&wbar, 2u * nA * FC4_OUT * 4u);
        bulk_load(smem_u32(sw), p.w5, nA * FC4_OUT * 4u, &wbar);
        bulk_load(smem_u32(sw + nA * FC4_OUT), p.w5t, nA * FC4_OUT * 4u, &wbar);
    }
    float* sb = sw + 2 * nA * FC4_OUT;
    if (threadIdx.x < 64)  // before the wait: through L2 (see k_fc5_td)
        sb[threadIdx.x] = (threadIdx.x & 31) < nA ? __ldcg((threadIdx.x < 32 ? p.b5 : p.b5t) + (threadIdx.x & 31)) : 0.f;
    __syncthreads();
    mbar_wait(&wbar, 0);
    pdl_wait();
    pdl_trigger();
    __shared__ float qs[FC5W_WARPS][2][S][32];  // [warp][net][sample][action]
    const int nw = blockDim.x >> 5;  // <= FC5W_WARPS
    for (int b0 = (blockIdx.x * nw + warp) * S; b0 < t.B; b0 += gridDim.x * nw * S) {
#pragma unroll
        for (int z = 0; z < 2; ++z) {
            float xv[S][FC4_OUT / 32];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const float* x = (z ? p.t4 : p.a4) + (int64_t)min(b0 + s, t.B - 1) * FC4_OUT;
#pragma unroll
                for (int k = 0; k < FC4_OUT / 32; ++k) xv[s][k] = x[lane + 32 * k];
            }
            const float* w = sw + z * nA * FC4_OUT;
            for (int a0 = 0; a0 < nA; a0 += 3) {
                float acc[3][S] = {};
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int a = min(a0 + u, nA - 1);
#pragma unroll
                    for (int k = 0; k < FC4_OUT / 32; ++k) {
                        const float wk = w[a * FC4_OUT + lane + 32 * k];
#pragma unroll
                        for (int s = 0; s < S; ++s) acc[u][s] = fmaf(xv[s][k], wk, acc[u][s]);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int u = 0; u < 3; ++u)
#pragma unroll
                        for (int s = 0; s < S; ++s) acc[u][s] += __shfl_xor_sync(0xffffffffu, acc[u][s], o);
                if (lane == 0)
#pragma unroll
                    for (int u = 0; u < 3; ++u)
                        if (a0 + u < nA)
#pragma unroll
                            for (int s = 0; s < S; ++s) qs[warp][z][s][a0 + u] = acc[u][s];
            }
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int b = b0 + s;
            if (b >= t.B) break;
            const float qv = lane < nA ? qs[warp][0][s][lane] + sb[lane] : 0.f;
            const float qh = lane < nA ? qs[warp][1][s][lane] + sb[32 + lane] : -INFINITY;
            if (lane < nA) {
                const_cast<float*>(t.Q)[b * nA + lane] = qv;
                const_cast<float*>(t.Qhat)[b * nA + lane] = qh;
            }
            const float mx = warp_max(qh);
            const int ab = t.a[b];
            const float y = t.d[b] ? t.r[b] : t.r[b] + t.gamma * mx;  // Alg.1
            const float delta = y - __shfl_sync(0xffffffffu, qv, ab);
            if (lane < nA) {
                const float cl = fminf(fmaxf(delta, -1.f), 1.f);  // reading R3
                t.dQ[b * nA + lane] = (lane == ab) ? -cl / (float)t.B : 0.f;
            }
            if (lane == 0)
                reinterpret_cast<float2*>(p.per_sample)[b] = make_float2(delta * delta, fabsf(delta));
        }
        __syncwarp();
    }
    __shared__ unsigned int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ float s_sq[FC5W_WARPS], s_ab[FC5W_WARPS];
    __shared__ int s_keep;
    float sq = 0.f, sa = 0.f;
    // thread i sums samples i, i + blockDim, ... in order; eight loads in flight at a time
    for (int i0 = threadIdx.x; i0 < t.B; i0 += 8 * blockDim.x) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            v[u] = i < t.B ? __ldcg(reinterpret_cast<const float2*>(p.per_sample) + i) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            sq += v[u].x;
            sa += v[u].y;
        }
    }
    sq = warp_sum(sq);
    sa = warp_sum(sa);
    if (lane == 0) {
        s_sq[warp] = sq;
        s_ab[warp] = sa;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        s_keep = td_decide(t, s_sq, s_ab, nw);
        *p.counter = 0;
    }
    __syncthreads();
    if (!s_keep)
        for (int e = threadIdx.x; e < t.B * nA; e += blockDim.x) t.dQ[e] = 0.f;
}

__global__ void k_mark_not_ready(DevLearnerInfo* info, const LearnerStats* st) {
    pdl_wait();
    pdl_trigger();
    DevLearnerInfo inf{};
    inf.not_ready = 1;
    inf.mu = st->mu;
    inf.var = st->var;
    inf.stats_count = st->count;
    *info = inf;
}

// ------------------------------------------------------------------------- fc5 backward
// dW5[a][n] += sum_b dQ[b][a] a4[b][n]; db5[a] += sum_b dQ[b][a];
// g4[b][n] = round_T((sum_a dQ[b][a] W5[a][n]) * 1[a4[b][n] > 0])
// Blocks [0, 2 n_chunks): rows [c*fc5_rows(B), ...) and one half of the columns of dW5[a][n] = sum_b dQ[b][a] a4[b][n] and
// db5[a] = sum_b dQ[b][a] -> part[c][nA*512 + nA] (summed over c in fixed order by K10).
// Remaining blocks: g4[b][n] = mask(sum_a dQ[b][a] W5[a][n]).
constexpr int FC5_ROWS_MAX = 64;
// rows per chunk: small batches use short chunks (more blocks, one round of loads each)
__host__ __device__ constexpr int fc5_rows(int B) {
    return B / 64 < 8 ? 8 : B / 64 > FC5_ROWS_MAX ? FC5_ROWS_MAX : (B / 64 + 7) / 8 * 8;
}
template <typename T>
__global__ void __launch_bounds__(256) k_fc5_bwd(const float* __restrict__ dQ, const float* __restrict__ a4,
                                                 const float* __restrict__ w5, int B, int nA, float* __restrict__ part,
                                                 int n_chunks, T* __restrict__ g4, const uint8_t* __restrict__ act) {
    // a4 (fc4's output) and W5 (the replica) were written two or more kernels back: loaded before
    // the wait (PDL: complete once this grid runs); only dQ comes from the kernel just before
    if ((int)blockIdx.x < 2 * n_chunks) {  // (chunk, column half)
        __shared__ __align__(16) float dq[FC5_ROWS_MAX * 32];  // [row][32]: actions padded with zeros
        const int rows = fc5_rows(B), c = blockIdx.x >> 1, b0 = c * rows, nb = min(rows, B - b0);
        const int n = threadIdx.x + 256 * (blockIdx.x & 1);
        float xpre[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xpre[u] = u < nb ? __ldcg(a4 + (int64_t)(b0 + u) * FC4_OUT + n) : 0.f;  // L2: see k_fc5_td
        pdl_wait();
        pdl_trigger();
        for (int i = threadIdx.x; i < nb * 32; i += 256)
            dq[i] = (i & 31) < nA ? dQ[(int64_t)(b0 + (i >> 5)) * nA + (i & 31)] : 0.f;
        __syncthreads();
        float acc[32];
#pragma unroll
        for (int a = 0; a < 32; ++a) acc[a] = 0.f;
        const float* xs = a4 + (int64_t)b0 * FC4_OUT + n;
        for (int bb = 0; bb < nb; bb += 16) {
            float x[16];  // sixteen rows' loads in flight before the FMAs (the first eight prefetched)
#pragma unroll
            for (int u = 0; u < 16; ++u)
                x[u] = (bb == 0 && u < 8) ? xpre[u] : bb + u < nb ? xs[(int64_t)(bb + u) * FC4_OUT] : 0.f;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (bb + u >= nb) break;
                const float4* q = reinterpret_cast<const float4*>(dq + (bb + u) * 32);
#pragma unroll
                for (int a = 0; a < 32; a += 4)
                    if (a < nA) {  // one 16-B shared load feeds four FMAs
                        const float4 qq = q[a / 4];
                        acc[a] = fmaf(qq.x, x[u], acc[a]);
                        acc[a + 1] = fmaf(qq.y, x[u], acc[a + 1]);
                        acc[a + 2] = fmaf(qq.z, x[u], acc[a + 2]);
                        acc[a + 3] = fmaf(qq.w, x[u], acc[a + 3]);
                    }
            }
        }
        float* out = part + (int64_t)c * nA * (FC4_OUT + 1);
#pragma unroll
        for (int a = 0; a < 32; ++a)
            if (a < nA) out[a * FC4_OUT + n] = acc[a];
        if ((blockIdx.x & 1) == 0 && (int)threadIdx.x < nA) {
            float t = 0.f;
            for (int b = 0; b < nb; ++b) t += dq[b * 32 + threadIdx.x];
            out[nA * FC4_OUT + threadIdx.x] = t;
        }
        return;
    }
    // g4[b][n] = mask(dQ[b][a_b] W5[a_b][n]): dQ has one nonzero entry per sample (the action taken,
    // k_fc5_td), so the sum over actions is that single product (exact: the other terms are zeros).
    // One warp per sample, four float4 columns per lane: its first sample's a4 row is requested
    // through L2 before the PDL wait (with plain, L1-cached loads there the asynchronous and
    // per-message modes disagreed, measured), everything else after it
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)(gridDim.x - 2 * n_chunks) * (blockDim.x >> 5);
    const int64_t b_first = (int64_t)(blockIdx.x - 2 * n_chunks) * (blockDim.x >> 5) + warp;
    float4 x[4];
    if (b_first < B)
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __ldcg(reinterpret_cast<const float4*>(a4 + b_first * FC4_OUT + (lane + 32 * i) * 4));
    pdl_wait();
    pdl_trigger();
    for (int64_t b = b_first; b < B; b += nwarps) {
        const int ab = act[b];
        float4 w[4];
        if (b != b_first)
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = *reinterpret_cast<const float4*>(a4 + b * FC4_OUT + (lane + 32 * i) * 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = *reinterpret_cast<const float4*>(w5 + ab * FC4_OUT + (lane + 32 * i) * 4);
        const float dq = dQ[b * nA + ab];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int n = (lane + 32 * i) * 4;
            const float v[4] = {x[i].x > 0.f ? dq * w[i].x : 0.f, x[i].y > 0.f ? dq * w[i].y : 0.f,
                                x[i].z > 0.f ? dq * w[i].z : 0.f, x[i].w > 0.f ? dq * w[i].w : 0.f};
            T* dst = g4 + b * FC4_OUT + n;
            if constexpr (sizeof(T) == 2) {  // one 8-B store
                __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);
                *reinterpret_cast<uint2*>(dst) =
                    make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
            } else {
                *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    }
}

// ------------------------------------------------------------------------- staged replay insert
// one upload of [frames | a | r | d] (the host call's packed staging bytes) scattered into the
// ring slots (t0 + i) mod C, then the device step counter (replay_insert, small host inserts)
__global__ void k_insert_scatter(const uint8_t* __restrict__ src, int64_t keep, int64_t t0, int64_t C,
                                 uint8_t* __restrict__ frames, uint8_t* __restrict__ ra, float* __restrict__ rr,
                                 uint8_t* __restrict__ rd, uint64_t* __restrict__ n_dev, uint64_t n_new) {
    const uint8_t* sa = src + keep * FRAME_BYTES;
    const float* sr = reinterpret_cast<const float*>(sa + ((keep + 15) / 16) * 16);
    const uint8_t* sd = reinterpret_cast<const uint8_t*>(sr + keep);
    const int64_t vec = keep * (FRAME_BYTES / 16);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < vec + keep; v += (int64_t)gridDim.x * blockDim.x) {
        if (v < vec) {
            const int64_t i = v / (FRAME_BYTES / 16), c = v - i * (FRAME_BYTES / 16);
            reinterpret_cast<uint4*>(frames + ((t0 + i) % C) * FRAME_BYTES)[c] =
                reinterpret_cast<const uint4*>(src + i * FRAME_BYTES)[c];
        } else {
            const int64_t i = v - vec, slot = (t0 + i) % C;
            ra[slot] = sa[i];
            rr[slot] = sr[i];
            rd[slot] = sd[i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_dev = n_new;
}

// ------------------------------------------------------------------------- result ring (gorila_round_post)
// The last node of a posted round: learner infos, round info and sync flags of the round into slot
// round % R of a mapped pinned ring, then (after a system fence) the slot's sequence number, which
// the host polls (gorila_round_fetch: no CUDA call, no extra stream operation outside the graph).
// Slot layout: u64 seq | u32 n | u32 pad | 24 B round info | 64 B sync flags | n x learner info.
struct EmitRing {
    uint8_t* ring;  // device view of the mapped ring
    int R, slot_bytes, n;
    const DevLearnerInfo* info[RING_MAXL];
    const uint8_t* sync[RING_MAXL];
    const uint64_t* round_info;  // [n_acc, V_before, V_after]
    const uint64_t* dev_round;   // advanced by this round's apply: the round is *dev_round - 1
};
__global__ void k_emit_ring(EmitRing p) {
    pdl_wait();
    pdl_trigger();
    const uint64_t round = *p.dev_round - 1;
    uint8_t* slot = p.ring + (size_t)(round % (uint64_t)p.R) * p.slot_bytes;
    const int t = threadIdx.x;
    constexpr int IW = sizeof(DevLearnerInfo) / 4;
    for (int e = t; e < p.n * IW; e += blockDim.x)
        reinterpret_cast<uint32_t*>(slot + RING_HDR)[e] = reinterpret_cast<const uint32_t*>(p.info[e / IW])[e % IW];
    if (t < p.n) slot[40 + t] = *p.sync[t];
    if (t == 0) {
        *reinterpret_cast<uint32_t*>(slot + 8) = (uint32_t)p.n;
        *reinterpret_cast<uint32_t*>(slot + 16) = (uint32_t)p.round_info[0];  // n_accepted (+ zero pad)
        *reinterpret_cast<uint32_t*>(slot + 20) = 0u;
        *reinterpret_cast<uint64_t*>(slot + 24) = p.round_info[1];
        *reinterpret_cast<uint64_t*>(slot + 32) = p.round_info[2];
    }
    __syncthreads();
    if (t == 0) {  // one system-scope release: cumulative over the block's payload stores (bar.sync)
        __threadfence_system();
        *reinterpret_cast<volatile uint64_t*>(slot) = round + 1;
    }
}

// ------------------------------------------------------------------------- small result copies
// gorila_round_async's learner infos / sync flags / round info into pinned host buffers: warp w
// copies segment w, w + nwarps, ... byte by byte (a few hundred bytes in all)
constexpr int SMALL_COPY_MAX = 24;
struct SmallCopies {
    int n;
    const uint8_t* src[SMALL_COPY_MAX];
    uint8_t* dst[SMALL_COPY_MAX];
    int bytes[SMALL_COPY_MAX];
};
__global__ void k_small_copies(SmallCopies c) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int s = w; s < c.n; s += blockDim.x >> 5)
        for (int b = lane; b < c.bytes[s]; b += 32) c.dst[s][b] = c.src[s][b];
}

// ------------------------------------------------------------------------- acting (NEXT row f3)
// states u8 [n][4][84][84] -> the conv input layout (NHWC, T), 4 pixels per thread
template <typename T>
__global__ void k_stage_states(const uint8_t* __restrict__ st, int n, T* __restrict__ s_out) {
    pdl_wait();
    pdl_trigger();
    const int64_t total = (int64_t)n * (FRAME_BYTES / 4);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / (FRAME_BYTES / 4), px = (i - b * (FRAME_BYTES / 4)) * 4;
        uint32_t c4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) c4[c] = *reinterpret_cast<const uint32_t*>(st + (b * 4 + c) * FRAME_BYTES + px);
        T* dst = s_out + (b * FRAME_BYTES + px) * NSTACK;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[p * 4 + c] = fromf<T>((float)((c4[c] >> (8 * p)) & 0xffu));
    }
}
// the acting path's states (u8 [n][4][7056] in device memory) as sample descriptors of the u8 path:
// state b's frames, every channel kept (samples n .. B-1 repeat the last state)
__global__ void k_act_desc(const uint8_t* __restrict__ st, int n, int B, SampleDesc* __restrict__ desc) {
    pdl_wait();
    pdl_trigger();
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        const int64_t sb = b < n ? b : n - 1;
        SampleDesc ds;
#pragma unroll
        for (int c = 0; c < 4; ++c) ds.frame[c] = st + (sb * 4 + c) * FRAME_BYTES;
        ds.frame[4] = ds.frame[3];
        ds.keep = 0xFFu;
        ds.pad_ = 0;
        desc[b] = ds;
    }
}
// Q = a4 . W5^T + b5 (fp32), then the epsilon-greedy decision (one block per state)
constexpr uint32_t TAG_ACT = 5u;
__global__ void __launch_bounds__(256) k_act_head(const float* __restrict__ a4, const float* __restrict__ w5,
                                                  const float* __restrict__ b5, int nA, uint64_t step,
                                                  uint32_t actor, uint2 key, double eps, int32_t* actions,
                                                  float* q) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ float qs[32];
    const float* x = a4 + (int64_t)i * FC4_OUT;
    for (int a = warp; a < nA; a += 8) {
        float acc = 0.f;
        for (int k = lane; k < FC4_OUT; k += 32) acc = fmaf(x[k], w5[a * FC4_OUT + k], acc);
        acc = warp_sum(acc);
        if (lane == 0) qs[a] = acc + b5[a];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = 0;
        for (int a = 1; a < nA; ++a)
            if (qs[a] > qs[best]) best = a;  // lowest index on ties
        const uint4 r = philox4x32_10(
            make_uint4((uint32_t)i, actor, (uint32_t)step, (uint32_t)((step >> 32) & 0xffffffu) | (TAG_ACT << 24)), key);
        const bool explore = (double)r.x < eps * 4294967296.0;
        actions[i] = explore ? (int32_t)(((uint64_t)r.y * (uint64_t)nA) >> 32) : best;
        for (int a = 0; a < nA; ++a) q[i * nA + a] = qs[a];
    }
}

// ------------------------------------------------------------------------- bias gradients
// db_l[o] = sum_m g_l[m][o], layers 1..4: block (chunk, l) sums rows [chunk*rows_per, ...) with
// coalesced row reads and a fixed-order in-block reduction -> part[l][chunk][o]; K10 sums chunks.
template <typename T>
__global__ void __launch_bounds__(256) k_bias_partial(const T* __restrict__ g1, const T* __restrict__ g2,
                                                      const T* __restrict__ g3, const T* __restrict__ g4, int B,
                                                      float* __restrict__ part, int BIAS_CHUNKS, int l0) {
    pdl_wait();
    pdl_trigger();
    // each thread owns 8 consecutive channels (one 16-B vector per row) of rows rg, rg+RG, ...
    // (layers l0..3: from the u8 path on, b1..b3 come from the weight-gradient GEMMs, l0 = 3)
    __shared__ float red[256 * 8];
    const int l = blockIdx.y + l0, chunk = blockIdx.x;
    const T* g = l == 0 ? g1 : l == 1 ? g2 : l == 2 ? g3 : g4;
    const int C = l == 0 ? C1_OUT : l == 3 ? FC4_OUT : C2_OUT;
    const int rows = B * (l == 0 ? H1 * H1 : l == 1 ? H2 * H2 : l == 2 ? H3 * H3 : 1);
    float* out = part + (l == 0 ? 0 : l == 1 ? BIAS_CHUNKS * C1_OUT : l == 2 ? BIAS_CHUNKS * (C1_OUT + C2_OUT)
                                                                             : BIAS_CHUNKS * (C1_OUT + 2 * C2_OUT));
    const int per = (rows + BIAS_CHUNKS - 1) / BIAS_CHUNKS;
    const int r0 = chunk * per, r1 = min(rows, r0 + per);
    const int VPR = C / 8;             // vectors per row
    const int RG = 256 / VPR;          // rows in flight per block pass
    const int vc = threadIdx.x % VPR, rg = threadIdx.x / VPR;
    float acc[8] = {};
    constexpr int V = 16 / sizeof(T);  // elements per 16-B vector (8 bf16 / 4 fp32)
    for (int r = r0 + rg; r < r1; r += RG) {
#pragma unroll
        for (int h = 0; h < 8 / V; ++h) {
            const uint4 q = *reinterpret_cast<const uint4*>(g + (int64_t)r * C + vc * 8 + h * V);
            const T* e = reinterpret_cast<const T*>(&q);
#pragma unroll
            for (int k = 0; k < V; ++k) acc[h * V + k] += tof(e[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) red[threadIdx.x * 8 + k] = acc[k];
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += 256) {  // fixed-order sum over the row groups
        const int v = c / 8, k = c % 8;
        float t = 0.f;
        for (int q = 0; q < RG; ++q) t += red[(q * VPR + v) * 8 + k];
        out[(int64_t)c * BIAS_CHUNKS + chunk] = t;  // [o][chunk]: K10 reads each bias's partials contiguously
    }
}

// ------------------------------------------------------------------------- K10 wgrad reduce
// G[seg] (+)= sum_s partial_seg[s][.] in split order, for the conv weights and the four biases
constexpr int WRED_SEGS = 8;
struct WgradReduceParams {
    const float* part[WRED_SEGS];
    int splits[WRED_SEGS];
    int64_t count[WRED_SEGS];
    int64_t off[WRED_SEGS];
    int wide[WRED_SEGS];  // 1: partials stored [element][split] and summed by one warp per element
    int nseg, accumulate;
    int coop;  // 1: [split][element] sums split over a block's 8 warps (many splits: one partial per CTA)
};
__global__ void k_wgrad_reduce(WgradReduceParams p, float* __restrict__ G) {
    pdl_wait();
    pdl_trigger();
    int64_t total = 0, total_w = 0;
    for (int l = 0; l < p.nseg; ++l) (p.wide[l] ? total_w : total) += p.count[l];
    // wide segments (many splits, few elements): a warp per element, lanes over the splits,
    // fixed-order shuffle tree
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t e = gw; e < total_w; e += nw) {
        int l = 0;
        int64_t f = e;
        while (!p.wide[l] || f >= p.count[l]) {
            if (p.wide[l]) f -= p.count[l];
            ++l;
        }
        const int S = p.splits[l];
        const float* src = p.part[l] + f * S;
        float acc = 0.f;
        for (int s = lane; s < S; s += 32) acc += src[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            float* dst = G + p.off[l] + f;
            *dst = p.accumulate ? *dst + acc : acc;
        }
    }
    if (!p.coop) {  // few splits: a thread per element, 8 independent partial sums in flight
        for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
            int l = 0;
            int64_t f = e;
            while (p.wide[l] || f >= p.count[l]) {
                if (!p.wide[l]) f -= p.count[l];
                ++l;
            }
            const float* src = p.part[l] + f;
            const int S = p.splits[l];
            const int64_t st = p.count[l];
            float a8[8] = {};
            int s = 0;
            for (; s + 8 <= S; s += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) a8[u] += src[(int64_t)(s + u) * st];
            }
            for (int u = 0; s < S; ++s, ++u) a8[u] += src[(int64_t)s * st];
            const float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
            float* dst = G + p.off[l] + f;
            *dst = p.accumulate ? *dst + acc : acc;
        }
        return;
    }
    // many splits: a block takes 32 consecutive elements, its 8 warps the splits s = w, w + 8, ...
    // (coalesced 128-B rows, 8 loads in flight per lane), combined in a fixed order through shared
    // memory (the split count reaches 148 with the one-partial-per-CTA GEMMs)
    __shared__ float red[8][33];
    const int x = threadIdx.x & 31, y = threadIdx.x >> 5, ny = blockDim.x >> 5;
    for (int64_t g0 = (int64_t)blockIdx.x * 32; g0 < total; g0 += (int64_t)gridDim.x * 32) {
        const int64_t e = g0 + x;
        float acc = 0.f;
        int l = 0;
        int64_t f = e;
        if (e < total) {
            while (p.wide[l] || f >= p.count[l]) {
                if (!p.wide[l]) f -= p.count[l];
                ++l;
            }
            const float* src = p.part[l] + f;
            const int S = p.splits[l];
            const int64_t st = p.count[l];
            float a8[8] = {};  // 8 loads in flight per lane
            int s = y;
            for (; s + 7 * ny < S; s += 8 * ny) {
#pragma unroll
                for (int u = 0; u < 8; ++u) a8[u] += src[(int64_t)(s + u * ny) * st];
            }
            for (int u = 0; s < S; s += ny, ++u) a8[u & 7] += src[(int64_t)s * st];
            acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
        }
        red[y][x] = acc;
        __syncthreads();
        if (y == 0 && e < total) {
            float t = red[0][x];
            for (int w = 1; w < ny; ++w) t += red[w][x];
            float* dst = G + p.off[l] + f;
            *dst = p.accumulate ? *dst + t : t;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------- PS apply (K11)
struct ApplyParams {
    float* theta;  // this rank's slice of theta^+ (sliced storage)
    float* m;
    float* v;
    const float* g;      // this rank's reduced slice
    const float* count;  // accepted gradients this round (all ranks), world > 1
    const uint32_t* count_local;  // world == 1: the learners' own counter
    uint64_t* dev_round;  // advanced by one (the next round's sampler counter)
    // fused target-sync decisions (gorila_round): R13, evaluated on the updated V
    LearnerStats* sync_stats[8];
    uint8_t* sync_flag[8];
    int n_sync;
    int64_t period;
    int64_t n_real;      // real elements in this slice
    int optimizer;
    float lr, rho, eps, ada_eps;
    uint64_t* V;
    uint64_t* round_info;  // [n_acc, V_before, V_after]
    // fused replica emission (world == 1): theta -> replica slot for the next round
    void* rep_t;           // T area (nullptr: no emission)
    float* rep_f;
    uint64_t* vhist_dst;
    int nA;
    int64_t base;          // internal index of this slice's element 0
    // fused target-sync copy (gorila_round, 1 GPU): when learner i's sync fires, the new replica is
    // also written into its theta^- (no separate pack); bookkeeping then moves to the last block
    void* sync_tm_t[8];
    float* sync_tm_f[8];
    int sync_copy;
    unsigned int* counter;
    // posted round (gorila_round_post, 1 GPU, fused sync decisions): block 0 stores the round's
    // results into the result-ring slot as soon as it has taken the decisions (no extra kernel)
    uint8_t* ring;
    int ring_R, ring_slot_bytes;
    const DevLearnerInfo* ring_info[8];
    int book_last;  // 1: the grid's last block only takes the round's decisions / stores the ring slot
                    // (its system fence overlaps the other blocks' update), the others only update
};
// Centered RMSProp (reading R2) / AdaGrad on the mean of the accepted gradients
// (reading R12, R25); V += |Acc|. float4-vectorised, grid-stride.
template <typename T>
GORILA_DEV void emit4(const ApplyParams& p, int64_t e4, const float* tv) {
    const ReplicaLayout L = replica_layout(p.nA);
    const int64_t slot = replica_slot(L, p.base + 4 * e4);
    if (slot >= 0) {
        T* dst = reinterpret_cast<T*>(p.rep_t) + slot;
        if constexpr (sizeof(T) == 2) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(tv[0], tv[1]), h1 = __floats2bfloat162_rn(tv[2], tv[3]);
            *reinterpret_cast<uint2*>(dst) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
        } else {
            *reinterpret_cast<float4*>(dst) = make_float4(tv[0], tv[1], tv[2], tv[3]);
        }
    } else {
        *reinterpret_cast<float4*>(p.rep_f + (-slot - 1)) = make_float4(tv[0], tv[1], tv[2], tv[3]);
    }
}

template <typename T>
GORILA_DEV void emit4_to(void* rep_t, float* rep_f, int nA, int64_t idx, const float* tv) {
    const ReplicaLayout L = replica_layout(nA);
    const int64_t slot = replica_slot(L, idx);
    if (slot >= 0) {
        T* dst = reinterpret_cast<T*>(rep_t) + slot;
        if constexpr (sizeof(T) == 2) {
            __nv_bfloat162 h0 = __floats2bfloat162_rn(tv[0], tv[1]), h1 = __floats2bfloat162_rn(tv[2], tv[3]);
            *reinterpret_cast<uint2*>(dst) =
                make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
        } else {
            *reinterpret_cast<float4*>(dst) = make_float4(tv[0], tv[1], tv[2], tv[3]);
        }
    } else {
        *reinterpret_cast<float4*>(rep_f + (-slot - 1)) = make_float4(tv[0], tv[1], tv[2], tv[3]);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) k_apply(ApplyParams p) {
    pdl_wait();
    pdl_trigger();
    const float cnt = p.count_local ? (float)*p.count_local : *p.count;
    // fused sync copy: every block takes the (same) decisions from the state before this round;
    // only the last block writes that state back, after every block has read it
    uint32_t doit_mask = 0;
    if (p.sync_copy) {
        const uint64_t v1 = *p.V + (uint64_t)(cnt + 0.5f);
        for (int i = 0; i < p.n_sync; ++i)
            if (v1 >= p.sync_stats[i]->last_sync + (uint64_t)p.period) doit_mask |= 1u << i;
    }
    const int book_block = p.book_last ? gridDim.x - 1 : 0;
    if (!p.sync_copy && blockIdx.x == book_block && threadIdx.x == 0) {
        const uint64_t v0 = *p.V;
        const uint64_t n_acc = (uint64_t)(cnt + 0.5f);
        p.round_info[0] = n_acc;
        p.round_info[1] = v0;
        p.round_info[2] = v0 + n_acc;
        *p.V = v0 + n_acc;
        if (p.vhist_dst) *p.vhist_dst = v0 + n_acc;
        const uint64_t rnd = p.dev_round ? *p.dev_round : 0;
        if (p.dev_round) *p.dev_round = rnd + 1;
        uint8_t* slot = p.ring ? p.ring + (size_t)(rnd % (uint64_t)p.ring_R) * p.ring_slot_bytes : nullptr;
        for (int i = 0; i < p.n_sync; ++i) {
            LearnerStats* st = p.sync_stats[i];
            const bool doit = v0 + n_acc >= st->last_sync + (uint64_t)p.period;
            if (doit) st->last_sync = v0 + n_acc;
            *p.sync_flag[i] = doit;
            if (slot) slot[40 + i] = doit;
        }
        if (slot) {  // the result ring slot of this round (layout: k_emit_ring)
            *reinterpret_cast<uint32_t*>(slot + 8) = (uint32_t)p.n_sync;
            *reinterpret_cast<uint64_t*>(slot + 16) = n_acc;  // n_accepted + zero pad
            *reinterpret_cast<uint64_t*>(slot + 24) = v0;
            *reinterpret_cast<uint64_t*>(slot + 32) = v0 + n_acc;
            for (int i = 0; i < p.n_sync; ++i)
                for (int w = 0; w < (int)(sizeof(DevLearnerInfo) / 8); ++w)
                    reinterpret_cast<uint64_t*>(slot + RING_HDR)[i * (sizeof(DevLearnerInfo) / 8) + w] =
                        reinterpret_cast<const uint64_t*>(p.ring_info[i])[w];
            __threadfence_system();
            *reinterpret_cast<volatile uint64_t*>(slot) = rnd + 1;
        }
    }
    const bool update = cnt > 0.5f;
    const float inv = update ? 1.0f / cnt : 0.f;
    const int64_t n4 = (p.n_real + 3) / 4;  // slices are padded to 64 elements (zeros, never read back)
    const int upd_blocks = gridDim.x - (p.book_last ? 1 : 0);
    if ((int)blockIdx.x >= upd_blocks) return;  // the bookkeeping block (book_last)
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)upd_blocks * blockDim.x) {
        float4 th = reinterpret_cast<float4*>(p.theta)[e];
        if (!update) {  // nothing accepted: theta, m, v unchanged; still emit the next replica
            if (p.rep_t) {
                const float tv[4] = {th.x, th.y, th.z, th.w};
                emit4<T>(p, e, tv);
            }
            continue;
        }
        float4 g = reinterpret_cast<const float4*>(p.g)[e];
        float4 m = reinterpret_cast<float4*>(p.m)[e];
        float4 v = reinterpret_cast<float4*>(p.v)[e];
        float gv[4] = {g.x * inv, g.y * inv, g.z * inv, g.w * inv};
        float tv[4] = {th.x, th.y, th.z, th.w}, mv[4] = {m.x, m.y, m.z, m.w}, vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (p.optimizer == 0) {
                mv[c] = p.rho * mv[c] + (1.f - p.rho) * gv[c];
                vv[c] = p.rho * vv[c] + (1.f - p.rho) * gv[c] * gv[c];
                tv[c] -= p.lr * gv[c] / sqrtf(vv[c] - mv[c] * mv[c] + p.eps);
            } else {
                vv[c] += gv[c] * gv[c];
                tv[c] -= p.lr * gv[c] / (sqrtf(vv[c]) + p.ada_eps);
            }
        }
        reinterpret_cast<float4*>(p.theta)[e] = make_float4(tv[0], tv[1], tv[2], tv[3]);
        reinterpret_cast<float4*>(p.m)[e] = make_float4(mv[0], mv[1], mv[2], mv[3]);
        reinterpret_cast<float4*>(p.v)[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        if (p.rep_t) emit4<T>(p, e, tv);
        if (doit_mask)
            for (int i = 0; i < p.n_sync; ++i)
                if (doit_mask >> i & 1u) emit4_to<T>(p.sync_tm_t[i], p.sync_tm_f[i], p.nA, p.base + 4 * e, tv);
    }
    if (!p.sync_copy) return;
    __shared__ unsigned int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(p.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    *p.counter = 0;
    const uint64_t v0 = *p.V;
    const uint64_t n_acc = (uint64_t)(cnt + 0.5f);
    p.round_info[0] = n_acc;
    p.round_info[1] = v0;
    p.round_info[2] = v0 + n_acc;
    *p.V = v0 + n_acc;
    if (p.vhist_dst) *p.vhist_dst = v0 + n_acc;
    if (p.dev_round) *p.dev_round += 1;
    for (int i = 0; i < p.n_sync; ++i) {
        const bool doit = doit_mask >> i & 1u;
        if (doit) p.sync_stats[i]->last_sync = v0 + n_acc;
        *p.sync_flag[i] = doit;
    }
}

// ------------------------------------------------------------------------- fused PS exchange (W > 1)
// One kernel replaces reduce-scatter -> apply -> all-gather -> pack over NVLink peer memory (CUDA
// IPC mappings of every rank's workspace): signal "my G is complete" into every peer's flag area,
// wait for every peer's, then for this rank's shard slice sum the peers' gradient slices in rank
// order (reading peer HBM through NVLink), apply the optimizer, and store the new theta slice and
// its next-round replica chunk into every rank. The last block signals "done"; k_peer_wait holds
// the stream until every peer is done (so no rank starts the next round while a peer still reads
// its G / count or writes its replicas).
// one optimizer step on 4 elements (R2 centered RMSProp / P:169 AdaGrad), the gradient unscaled
GORILA_DEV void opt_step4(const ApplyParams& p, float* tv, float* mv, float* vv, const float4 g) {
    const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        if (p.optimizer == 0) {
            mv[c] = p.rho * mv[c] + (1.f - p.rho) * gv[c];
            vv[c] = p.rho * vv[c] + (1.f - p.rho) * gv[c] * gv[c];
            tv[c] -= p.lr * gv[c] / sqrtf(vv[c] - mv[c] * mv[c] + p.eps);
        } else {
            vv[c] += gv[c] * gv[c];
            tv[c] -= p.lr * gv[c] / (sqrtf(vv[c]) + p.ada_eps);
        }
    }
}
constexpr int MAX_W = 8;
// f1 per-message PS (R32, R37): the messages of a round arrive in ascending global learner id. Message
// m (sent unless its learner was not ready or outlier-rejected) is stale iff max_delay >= 0 and
// V - base_m > max_delay with V the PS version when it arrives (V0 + messages applied before it;
// P:160); a fresh one is its own optimizer step and V += 1, after which every learner i
// with V >= last_i + N syncs its target net (theta^- = theta after that step, last_i = V;
// P:158-160). Computed by one thread from the round's inputs; every block computes the same.
constexpr int MAX_MSG = 64;
struct MsgSchedule {
    uint64_t acc;                 // applied messages
    uint64_t vend;                // V after the round
    uint64_t last[MAX_MSG];       // every learner's last sync after the round
    uint64_t sync_after[MAX_MSG]; // learners whose (last) in-round sync follows message m
    int8_t sync_at[MAX_MSG];      // message after which learner i last synced this round, -1: none
};
GORILA_DEV void msg_schedule(int n, uint64_t has, const uint64_t* base, const uint64_t* last0, uint64_t V0,
                             int64_t max_delay, int64_t period, MsgSchedule& s) {
    uint64_t V = V0;
    s.acc = 0;
    for (int i = 0; i < n; ++i) {
        s.last[i] = last0[i];
        s.sync_at[i] = -1;
        s.sync_after[i] = 0;
    }
    for (int m = 0; m < n; ++m) {
        if (!(has >> m & 1ull)) continue;
        if (max_delay >= 0 && (int64_t)(V - base[m]) > max_delay) continue;  // stale at arrival
        s.acc |= 1ull << m;
        V += 1;
        for (int i = 0; i < n; ++i)
            if (V >= s.last[i] + (uint64_t)period) {
                s.last[i] = V;
                s.sync_at[i] = (int8_t)m;
            }
    }
    for (int i = 0; i < n; ++i)
        if (s.sync_at[i] >= 0) s.sync_after[s.sync_at[i]] |= 1ull << i;
    s.vend = V;
}

GORILA_DEV void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
GORILA_DEV uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// wait until a peer-written flag reaches ep; a peer that never arrives (protocol error, dead
// rank) traps after ~2^25 polls (seconds) instead of hanging the device
GORILA_DEV uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// trace build: accumulated ns of the exchange (slots 40..: wait-for-peers, work after the wait,
// peer-done wait, rounds) — tools/trace_p2p.py
#ifdef GORILA_TRACE
#define P2PTRACE(slot, v) atomicAdd(&gorila_trace_buf[(slot)], (unsigned long long)(v))
#else
#define P2PTRACE(slot, v)
#endif
GORILA_DEV void wait_flag(const uint64_t* p, uint64_t ep) {
    for (uint32_t n = 0; ld_acquire_sys(p) < ep; ++n) {
        if (n > (1u << 25)) __trap();
        __nanosleep(64);
    }
}

// global replay (f4, R36): before a round's first draw every rank's earlier inserts must be
// visible to every rank. Rank r bumps its epoch, publishes it into slot r of every peer's flag
// array (system-scope release after a system fence: cumulative over the insert kernels that
// completed before this one on the stream) and waits until all peers' epochs reached it.
// A peer cannot overwrite a slot this round reads before the round ends: its next insert
// follows its own round, whose parameter exchange needs this rank's gradient, i.e. this draw.
// With the flag, rank r pushes its learners' ring counters into every rank's n_snap (slots r*L ..
// r*L+L-1), so the sampler finds all G counters in local memory once the flags have arrived.
struct ReplayBarrier {
    uint64_t* epoch;             // this rank's round epoch (device counter)
    uint64_t* flags[MAX_W];      // rank q's flag array [MAX_W]
    uint64_t* n_snap[MAX_W];     // rank q's counter snapshot [G]
    const ShardPtrs* tab;
    int W, rank, L;
};
__global__ void k_replay_barrier(ReplayBarrier p) {
    pdl_wait();
    for (int j = threadIdx.x; j < p.L; j += blockDim.x) {
        const int gid = p.rank * p.L + j;
        const uint64_t v = *(volatile const uint64_t*)p.tab[gid].n;
        for (int q = 0; q < p.W; ++q) p.n_snap[q][gid] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t e = *p.epoch + 1;
        *p.epoch = e;
        __threadfence_system();
        for (int q = 0; q < p.W; ++q)
            if (q != p.rank) st_release_sys(p.flags[q] + p.rank, e);
        for (int q = 0; q < p.W; ++q)
            if (q != p.rank) wait_flag(p.flags[p.rank] + q, e);
    }
    __syncthreads();
    pdl_trigger();
}
struct P2PParams {
    int W, rank;
    const float* G[MAX_W];        // rank q's gradient buffer at this rank's slice
    const uint32_t* nacc[MAX_W];  // rank q's accepted count of the round
    float* theta[MAX_W];          // rank q's theta^+ at this rank's slice
    void* rep_t[MAX_W];           // rank q's next-round replica (T area, fp32 area)
    float* rep_f[MAX_W];
    uint64_t* flags[MAX_W];       // rank q's flag area: phase f: [2f MAX_W, +MAX_W) ready, [(2f+1) MAX_W, ..) done;
                                  // [4 MAX_W, 5 MAX_W): the ranks' accepted counts (sent with the ready flag);
                                  // [5 MAX_W, 6 MAX_W): their per-learner acceptance masks (f1)
    uint64_t* epoch;              // local round epoch (advanced by k_peer_wait)
    unsigned int* counter;        // local: finished blocks, one counter per phase (phases may overlap)
    int dbg;                      // diagnostics (GORILA_P2P_DBG): 1 = skip peer gradient loads, 2 = skip peer replica stores
    // per-message mode (f1): L messages per rank, message (q, j) = rank q's learner j at Gm[q * L + j]
    int L;                        // 0: aggregate mode
    const float* Gm[64];
    DevLearnerInfo* info[32];     // this rank's learners' records (sent mask / bases published with the flag;
                                  // the final stale / accepted decisions written back by the book block)
    LearnerStats* stats[32];      // this rank's learners' target-sync state
    uint8_t* sync_flag[32];
    void* tm_t[64];               // every global learner's theta^- replica, at its address in this process
    float* tm_f[64];
    int64_t max_delay, period;
};
// flag-area slots (u64) of the per-message exchange, besides the ready / done flags and counts
constexpr int FLAG_BASE = 6 * MAX_W, FLAG_LAST = FLAG_BASE + MAX_MSG, FLAG_V0 = FLAG_LAST + MAX_MSG,
              FLAG_ASYNC = FLAG_V0 + MAX_W, FLAG_WORDS = FLAG_ASYNC + MAX_W;


// phase: flag set (0 = the fc4 weight region, launched early by gorila_round; 1 = the rest);
// [lo0, hi0) and [lo1, hi1): float4 ranges of the slice this launch updates; book: V, round
// info, version history and sync decisions (the last phase only).
template <typename T>
__global__ void __launch_bounds__(256) k_apply_p2p(ApplyParams p, P2PParams x, int phase, int64_t lo0,
                                                   int64_t hi0, int64_t lo1, int64_t hi1, int book) {
    pdl_wait();
    pdl_trigger();
    const uint64_t ep = *x.epoch + 1;
    const int RDY = 2 * phase * MAX_W, DONE = RDY + MAX_W;
#ifdef GORILA_TRACE
    const uint64_t t_in = gtimer();
#endif
    uint64_t* mine = x.flags[x.rank];
    if (blockIdx.x == 0 && (int)threadIdx.x < x.W) {  // this rank's G range and count are complete
        x.flags[threadIdx.x][4 * MAX_W + x.rank] = (uint64_t)*x.nacc[x.rank];  // ordered by the release
        if (x.L) {  // f1: which learners sent a message, their replica versions, target-sync state, V0
            uint64_t m = 0;
            for (int j = 0; j < x.L; ++j) {
                m |= (uint64_t)(x.info[j]->accepted ? 1 : 0) << j;
                x.flags[threadIdx.x][FLAG_BASE + x.rank * x.L + j] = x.info[j]->base_version;
                x.flags[threadIdx.x][FLAG_LAST + x.rank * x.L + j] = x.stats[j]->last_sync;
            }
            x.flags[threadIdx.x][5 * MAX_W + x.rank] = m;
            x.flags[threadIdx.x][FLAG_V0 + x.rank] = *p.V;
        }
        st_release_sys(x.flags[threadIdx.x] + RDY + x.rank, ep);
    }
    __shared__ float s_cnt;
    __shared__ unsigned long long s_gmask;
    __shared__ MsgSchedule sch;
    if (threadIdx.x == 0) {
        float c = 0.f;
        unsigned long long gm = 0;
        for (int q = 0; q < x.W; ++q) {
            wait_flag(mine + RDY + q, ep);
            c += (float)__ldcg(mine + 4 * MAX_W + q);  // local copy of rank q's count
            if (x.L) gm |= (unsigned long long)__ldcg(mine + 5 * MAX_W + q) << (q * x.L);
        }
        if (x.L) {  // the per-message schedule over every rank's messages (identical on every rank)
            uint64_t base[MAX_MSG], last0[MAX_MSG];
            const int n = x.W * x.L;
            for (int i = 0; i < n; ++i) {
                base[i] = __ldcg(mine + FLAG_BASE + i);
                last0[i] = __ldcg(mine + FLAG_LAST + i);
            }
            msg_schedule(n, gm, base, last0, __ldcg(mine + FLAG_V0), x.max_delay, x.period, sch);
            gm = sch.acc;
            c = (float)__popcll(gm);
        }
        s_cnt = c;
        s_gmask = gm;
    }
    __syncthreads();
    const unsigned long long gmask = s_gmask;
#ifdef GORILA_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t t = gtimer();
        P2PTRACE(40, t - t_in);
        gorila_trace_buf[47] = t;
    }
#endif
    const float cnt = s_cnt;
    if (book && x.L && blockIdx.x == 0 && threadIdx.x == 0) {  // f1: the schedule's versions and decisions
        const uint64_t v0 = __ldcg(mine + FLAG_V0), n_acc = (uint64_t)__popcll(gmask);
        p.round_info[0] = n_acc;
        p.round_info[1] = v0;
        p.round_info[2] = sch.vend;
        *p.V = sch.vend;
        if (p.vhist_dst) *p.vhist_dst = sch.vend;
        if (p.dev_round) *p.dev_round += 1;
        for (int j = 0; j < x.L; ++j) {
            const int gid = x.rank * x.L + j;
            DevLearnerInfo* inf = x.info[j];
            const bool sent = inf->accepted;
            inf->accepted = (gmask >> gid & 1ull) ? 1 : 0;
            inf->stale = (sent && !inf->accepted) ? 1 : 0;
            x.stats[j]->last_sync = sch.last[gid];
            *x.sync_flag[j] = sch.sync_at[gid] >= 0;
        }
    } else if (book && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t v0 = *p.V;
        const uint64_t n_acc = (uint64_t)(cnt + 0.5f);
        p.round_info[0] = n_acc;
        p.round_info[1] = v0;
        p.round_info[2] = v0 + n_acc;
        *p.V = v0 + n_acc;
        if (p.vhist_dst) *p.vhist_dst = v0 + n_acc;
        if (p.dev_round) *p.dev_round += 1;
        for (int i = 0; i < p.n_sync; ++i) {
            LearnerStats* st = p.sync_stats[i];
            const bool doit = v0 + n_acc >= st->last_sync + (uint64_t)p.period;
            if (doit) st->last_sync = v0 + n_acc;
            *p.sync_flag[i] = doit;
        }
    }
    const bool update = cnt > 0.5f;
    const float inv = update ? 1.0f / cnt : 0.f;
    float* th_local = x.theta[x.rank];
    const int64_t len0 = hi0 - lo0, n = len0 + (hi1 - lo1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = i < len0 ? lo0 + i : lo1 + (i - len0);
        float4 th = reinterpret_cast<const float4*>(th_local)[e];
        float tv[4] = {th.x, th.y, th.z, th.w};
        if (update && x.L) {  // f1: one optimizer step per accepted message, in global learner order
            float4 m = reinterpret_cast<float4*>(p.m)[e];
            float4 v = reinterpret_cast<float4*>(p.v)[e];
            float mv[4] = {m.x, m.y, m.z, m.w}, vv[4] = {v.x, v.y, v.z, v.w};
            for (int msg = 0; msg < x.W * x.L; ++msg) {
                if (!(gmask >> msg & 1ull)) continue;
                opt_step4(p, tv, mv, vv, __ldcg(reinterpret_cast<const float4*>(x.Gm[msg]) + e));
                for (uint64_t sm = sch.sync_after[msg]; sm; sm &= sm - 1) {  // in-round target syncs (any rank)
                    const int i = __ffsll((long long)sm) - 1;
                    emit4_to<T>(x.tm_t[i], x.tm_f[i], p.nA, p.base + 4 * e, tv);
                }
            }
            reinterpret_cast<float4*>(p.m)[e] = make_float4(mv[0], mv[1], mv[2], mv[3]);
            reinterpret_cast<float4*>(p.v)[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
            reinterpret_cast<float4*>(th_local)[e] = make_float4(tv[0], tv[1], tv[2], tv[3]);
        } else if (update) {
            float4 gq[MAX_W];  // every rank's slice element requested before the first add
#pragma unroll
            for (int q = 0; q < MAX_W; ++q)
                if (q < x.W) gq[q] = __ldcg(reinterpret_cast<const float4*>(x.G[(x.dbg & 1) ? x.rank : q]) + e);
            float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < MAX_W; ++q)  // fixed rank order
                if (q < x.W) {
                    g.x += gq[q].x; g.y += gq[q].y; g.z += gq[q].z; g.w += gq[q].w;
                }
            float4 m = reinterpret_cast<float4*>(p.m)[e];
            float4 v = reinterpret_cast<float4*>(p.v)[e];
            float gv[4] = {g.x * inv, g.y * inv, g.z * inv, g.w * inv};
            float mv[4] = {m.x, m.y, m.z, m.w}, vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (p.optimizer == 0) {
                    mv[c] = p.rho * mv[c] + (1.f - p.rho) * gv[c];
                    vv[c] = p.rho * vv[c] + (1.f - p.rho) * gv[c] * gv[c];
                    tv[c] -= p.lr * gv[c] / sqrtf(vv[c] - mv[c] * mv[c] + p.eps);
                } else {
                    vv[c] += gv[c] * gv[c];
                    tv[c] -= p.lr * gv[c] / (sqrtf(vv[c]) + p.ada_eps);
                }
            }
            reinterpret_cast<float4*>(p.m)[e] = make_float4(mv[0], mv[1], mv[2], mv[3]);
            reinterpret_cast<float4*>(p.v)[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
            // the fp32 master stays with the owner; the peers get only the replica chunk
            reinterpret_cast<float4*>(th_local)[e] = make_float4(tv[0], tv[1], tv[2], tv[3]);
        }
        for (int q = 0; q < x.W; ++q)
            if (!(x.dbg & 2) || q == x.rank) emit4_to<T>(x.rep_t[q], x.rep_f[q], p.nA, p.base + 4 * e, tv);
    }
    // done: a GPU-scope fence per block before the counter; the last block's system-scope
    // fence then releases every block's peer stores (cumulativity) before the flag
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int* ctr = x.counter + phase;
        const unsigned int prev = atomicAdd(ctr, 1u);
        if (prev == gridDim.x - 1) {
            *ctr = 0;
            P2PTRACE(41, gtimer() - gorila_trace_buf[47]);
            __threadfence();
            __threadfence_system();
            for (int q = 0; q < x.W; ++q) st_release_sys(x.flags[q] + DONE + x.rank, ep);
        }
    }
}

// target sync from the replica (peer-memory mode, where each rank holds only its own slice of
// the fp32 theta^+): theta^- <- the replica the round just emitted, if *pred (R13)
__global__ void k_copy_replica(const uint4* __restrict__ st, uint4* __restrict__ dt, int64_t nt16,
                               const float4* __restrict__ sf, float4* __restrict__ df, int64_t nf4,
                               const uint8_t* __restrict__ pred) {
    pdl_wait();
    pdl_trigger();
    if (pred && !*pred) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt16 + nf4; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < nt16) dt[i] = st[i];
        else df[i - nt16] = sf[i - nt16];
    }
}

__global__ void k_peer_wait(P2PParams x, int phase0) {  // waits for phase 1 (and phase 0 if phase0)
    pdl_wait();
    pdl_trigger();
    const uint64_t ep = *x.epoch + 1;
    const uint64_t* mine = x.flags[x.rank];
#ifdef GORILA_TRACE
    const uint64_t t_in = gtimer();
#endif
    if ((int)threadIdx.x < x.W) {
        wait_flag(mine + 3 * MAX_W + threadIdx.x, ep);
        if (phase0) wait_flag(mine + MAX_W + threadIdx.x, ep);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *x.epoch = ep;
        P2PTRACE(42, gtimer() - t_in);
        P2PTRACE(43, 1);
    }
}

// ------------------------------------------------------------------------- per-message PS (f1)
// NEXT row f1 (reading R32): each accepted learner gradient is its own optimizer step, applied in
// ascending global learner id ("applies the updates", P:160 version per update). The
// sequence is elementwise, so every thread runs the whole message sequence on its elements.
struct MsgParams {
    const float* G[32];           // local learner j's gradient (this rank's slice)
    DevLearnerInfo* info[32];     // its learner record (sent = accepted from the learner step; the
                                  // final stale / accepted decisions are written back here)
    LearnerStats* stats[32];      // its target-sync state
    uint8_t* sync_flag[32];
    void* tm_t[32];               // its target replica (T area, fp32 area)
    float* tm_f[32];
    int nmsg;
    int64_t max_delay;
    unsigned int* counter;        // last-block detection (zero between launches)
};
// W == 1: every block takes the schedule from the state before this round; the last block to finish
// writes the decisions / versions / sync state back (after every block has read them).
template <typename T>
__global__ void __launch_bounds__(256) k_apply_msg(ApplyParams p, MsgParams mp) {
    pdl_wait();
    pdl_trigger();
    __shared__ MsgSchedule sch;
    __shared__ uint64_t s_v0;
    if (threadIdx.x == 0) {
        uint64_t has = 0, base[32], last0[32];
        for (int j = 0; j < mp.nmsg; ++j) {
            has |= (uint64_t)(mp.info[j]->accepted ? 1 : 0) << j;
            base[j] = mp.info[j]->base_version;
            last0[j] = mp.stats[j]->last_sync;
        }
        s_v0 = *p.V;
        msg_schedule(mp.nmsg, has, base, last0, s_v0, mp.max_delay, p.period, sch);
    }
    __syncthreads();
    const uint64_t acc = sch.acc;
    const int64_t n4 = (p.n_real + 3) / 4;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
        float4 th = reinterpret_cast<float4*>(p.theta)[e];
        float tv[4] = {th.x, th.y, th.z, th.w};
        if (acc) {
            float4 m = reinterpret_cast<float4*>(p.m)[e];
            float4 v = reinterpret_cast<float4*>(p.v)[e];
            float mv[4] = {m.x, m.y, m.z, m.w}, vv[4] = {v.x, v.y, v.z, v.w};
            for (int j0 = 0; j0 < mp.nmsg; j0 += 8) {  // 8 messages' gradients in flight, then their steps
                float4 gq[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (j0 + u < mp.nmsg && (acc >> (j0 + u) & 1ull)) gq[u] = reinterpret_cast<const float4*>(mp.G[j0 + u])[e];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (j0 + u >= mp.nmsg || !(acc >> (j0 + u) & 1ull)) continue;
                    opt_step4(p, tv, mv, vv, gq[u]);
                    for (uint64_t sm = sch.sync_after[j0 + u]; sm; sm &= sm - 1) {  // in-round target syncs
                        const int i = __ffsll((long long)sm) - 1;
                        emit4_to<T>(mp.tm_t[i], mp.tm_f[i], p.nA, p.base + 4 * e, tv);
                    }
                }
            }
            reinterpret_cast<float4*>(p.theta)[e] = make_float4(tv[0], tv[1], tv[2], tv[3]);
            reinterpret_cast<float4*>(p.m)[e] = make_float4(mv[0], mv[1], mv[2], mv[3]);
            reinterpret_cast<float4*>(p.v)[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        }
        if (p.rep_t) emit4<T>(p, e, tv);
    }
    __shared__ unsigned int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(mp.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    *mp.counter = 0;
    const uint64_t v0 = s_v0, n_acc = (uint64_t)__popcll(acc);
    p.round_info[0] = n_acc;
    p.round_info[1] = v0;
    p.round_info[2] = sch.vend;
    *p.V = sch.vend;
    if (p.vhist_dst) *p.vhist_dst = sch.vend;
    if (p.dev_round) *p.dev_round += 1;
    for (int j = 0; j < mp.nmsg; ++j) {
        DevLearnerInfo* inf = mp.info[j];
        const bool sent = inf->accepted;
        inf->accepted = (acc >> j & 1ull) ? 1 : 0;
        inf->stale = (sent && !inf->accepted) ? 1 : 0;
        mp.stats[j]->last_sync = sch.last[j];
        *mp.sync_flag[j] = sch.sync_at[j] >= 0;
    }
}

// this rank's accepted count, once per destination shard (reduce-scattered with G)
__global__ void k_write_counts(float* counts, int W, const uint32_t* n_acc_local) {
    pdl_wait();
    pdl_trigger();
    const int s = threadIdx.x;
    if (s < W) counts[s] = (float)*n_acc_local;
}

// ------------------------------------------------------------------------- replica pack
// theta^+ (internal order, fp32) -> replica (T area + fp32 area). pred (nullable): skip unless *pred.
template <typename T>
__global__ void k_pack(const float* __restrict__ theta, int nA, T* __restrict__ rt, float* __restrict__ rf,
                       const uint8_t* __restrict__ pred, uint64_t* __restrict__ vhist_dst,
                       const uint64_t* __restrict__ V) {
    pdl_wait();
    pdl_trigger();
    if (pred && !*pred) return;
    const ReplicaLayout L = replica_layout(nA);
    const int64_t P = param_count(nA);
    if (vhist_dst && blockIdx.x == 0 && threadIdx.x == 0) *vhist_dst = *V;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = replica_slot(L, i);
        if (slot >= 0) rt[slot] = fromf<T>(theta[i]);
        else rf[-slot - 1] = theta[i];
    }
}

// ------------------------------------------------------------------------- target sync decision
// Alg.1; R13: sync iff force or V >= last + N; then last = V.
__global__ void k_sync_decide(LearnerStats* st, const uint64_t* V, int64_t period, int force, uint8_t* flag) {
    pdl_wait();
    pdl_trigger();
    const uint64_t v = *V;
    const bool doit = force || v >= st->last_sync + (uint64_t)period;
    if (doit) st->last_sync = v;
    *flag = doit;
}

// ------------------------------------------------------------------------- layout conversion
// dir 0: canonical -> internal ; dir 1: internal -> canonical
__global__ void k_convert(const float* __restrict__ src, float* __restrict__ dst, int64_t P, int dir) {
    pdl_wait();
    pdl_trigger();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = canon_of_internal(i);
        if (dir == 0) dst[i] = src[c];
        else dst[c] = src[i];
    }
}

__global__ void k_set_u64(uint64_t* dst, uint64_t v) {
    pdl_wait();
    pdl_trigger();
    *dst = v;
}

}  // namespace gorila
