// gorila.cu — context, workspace, orchestration and the C-ABI (include/gorila.h).
//
// One learner update (Alg.1) for local learner j at round k, all on `stream`:
//   K1 sample -> conv1..fc4 fwd (online + target batched per launch) -> fc5 fwd -> K7 TD +
//   decisions -> fc5 bwd -> fc4 dgrad/wgrad -> conv3/conv2 dgrad + wgrad -> conv1 wgrad ->
//   bias grads -> K10 wgrad reduce into G.
// ps_apply_shard: [NCCL reduce-scatter] -> K11 apply -> [NCCL all-gather] -> replica pack.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <atomic>
#include <memory>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/gorila.h"
#include "common.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "layout.cuh"
#include "tma_gemm.cuh"
#include "shift_gemm.cuh"
#include "tower.cuh"
#include "async.cuh"

using namespace gorila;

namespace {

thread_local std::string g_last_error;

gorila_status fail(gorila_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

#define CU(expr)                                                                                     \
    do {                                                                                             \
        cudaError_t _e = (expr);                                                                     \
        if (_e != cudaSuccess) {                                                                     \
            ctx->poisoned = true;                                                                    \
            return fail(GORILA_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
        }                                                                                            \
    } while (0)

#define NC(expr)                                                                                     \
    do {                                                                                             \
        ncclResult_t _r = (expr);                                                                    \
        if (_r != ncclSuccess) {                                                                     \
            ctx->poisoned = true;                                                                    \
            return fail(GORILA_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));          \
        }                                                                                            \
    } while (0)

#define LAUNCHED() (ctx->launches++)

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct Learner {
    uint8_t* frames;
    uint8_t* a;
    float* r;
    uint8_t* d;
    uint64_t* n_dev;
    int64_t n_host = 0;
    void* tminus_t;   // target replica (fwd only), element type T
    float* tminus_f;  // fp32 area
    LearnerStats* stats;
    DevLearnerInfo* info;
    float* Q;
    float* Qhat;
    uint8_t* sync_flag;
};

// carve helper over the caller's workspace (256-B aligned bump allocator; nullptr base = dry run)
struct Carver {
    uint8_t* base;
    uint64_t off = 0;
    template <typename X>
    X* take(int64_t count) {
        off = (uint64_t)round_up((int64_t)off, 256);
        X* p = base ? reinterpret_cast<X*>(base + off) : nullptr;
        off += (uint64_t)count * sizeof(X);
        return p;
    }
};

}  // namespace

struct gorila_ctx {
    gorila_config cfg;
    cudaStream_t stream;
    bool poisoned = false;
    uint64_t launches = 0;
    int nA, B, L, W, rank;
    int64_t P, q;       // params, elements per shard slice (P padded to W*q)
    size_t esz;         // sizeof(T)
    ReplicaLayout rl;
    // PS state
    float* theta;   // [W*q] full theta^+ (internal layout, contiguous shard slices)
    float* m;       // [q] own slice
    float* v;
    float* G;       // [W*q] gradient
    float* counts;  // [W] accepted-gradient counts (reduce-scattered with G)
    uint64_t* V;
    uint64_t* round_info;  // [3]
    uint32_t* n_acc_local;
    // history of replicas (H slots)
    int H;
    std::vector<void*> rep_t;
    std::vector<float*> rep_f;
    uint64_t* Vhist;
    // learners
    std::vector<Learner> learners;
    // per-step scratch (shared by the local learners)
    void *s, *s2, *a1, *a2, *a3, *t1, *t2, *t3, *g1, *g2, *g3, *g4;
    float *a4, *t4;  // fp32 (fc5 runs in fp32)
    uint8_t *sa, *sd;
    float* sr;
    int64_t* sidx;
    int32_t* sshard;         // shard (global learner id) of each sample of the last draw (f4)
    // global replay (NEXT row f4, cfg.replay_mode == 1): every learner's ring on every rank
    bool replay_global = false;
    ShardPtrs* shard_tab = nullptr;  // [W * L], rank-major (q, j): index = global learner id
    int n_shards = 0;
    uint64_t* rflags = nullptr;      // [MAX_W] replay-barrier epochs published by each rank
    uint64_t* replay_epoch = nullptr;
    uint64_t* n_snap = nullptr;      // [W * L] ring counters pushed by every rank at the replay barrier
    float* dQ;
    float* td_partial;  // [B][2] per-sample delta^2, |delta|
    int bias_chunks;
    float* part_w[3];  // conv wgrad partials
    float* part_b;     // bias-gradient partials [4 layers][C][BIAS_CHUNKS]
    float* part5;      // fc5 weight + bias gradient partials [B/FC5_ROWS][nA*513]
    int split_w[3];
    float* tmp_canon;  // [P]
    float* tmp_int;    // [W*q]
    ncclComm_t comm = nullptr;
    // per-phase profiling (gorila_profile_*)
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> marks;
    double prof_ms[32] = {};
    uint64_t prof_steps = 0;
    // CUDA-graph cache of whole rounds (gorila_round)
    uint64_t* dev_round = nullptr;  // round counter the sampler reads
    uint64_t dev_round_expect = ~0ull;  // value dev_round will hold when the queued work completes
    unsigned int* head_counter = nullptr;
    bool pdl = true;               // programmatic dependent launch between the round's kernels
    bool fused_sync = false;       // gorila_round: k_apply takes the target-sync decisions
    int sync_ids[8] = {};
    int sync_n = 0;
    bool capturing = false;
    std::map<std::vector<int64_t>, cudaGraphExec_t> graphs;
    std::map<std::vector<int64_t>, uint64_t> graph_kernels;
    std::map<std::vector<int64_t>, int> graph_seen;
    std::map<std::vector<int64_t>, std::vector<std::pair<int, cudaEvent_t>>> graph_marks;  // profiling graphs
    std::map<std::vector<uint64_t>, CUtensorMap> tmaps;  // TMA descriptors, encoded once per (buffer, view)
    bool tma_failed = false;
    int num_sms = 148;
    unsigned int* fc5_gen = nullptr;  // [2] generation counters of the fused fc5 backward
    // pinned staging ring for host-source replay_insert: the call copies the caller's bytes here
    // (CPU memcpy) and enqueues the upload without synchronising; a slot is reused only after the
    // event of its previous upload has completed
    static constexpr int kStage = 4;
    uint8_t* stage[kStage] = {};
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[kStage] = {};
    int stage_next = 0;
    uint8_t* stage_dev = nullptr;  // device landing buffer of a staged insert (4 MB)
    // result ring of gorila_round_post / gorila_round_fetch (mapped pinned host memory)
    static constexpr int kRing = 16;
    uint8_t* ring_host = nullptr;
    uint8_t* ring_dev = nullptr;
    int ring_slot = 0;
    bool ring_pending = false;  // a posted round whose results are not stored yet (k_apply or k_emit_ring)
    uint8_t* stage_dptr[kStage] = {};  // device view of the mapped pinned slots (small inserts read them directly)
    unsigned int* apply_counter = nullptr;  // last-block detection of k_apply's fused sync copy
    bool sync_fused_now = false;            // this round's k_apply did the target-sync copy
    // L2 persistence window over the parameter-server state (theta, m, v, G, replicas): the
    // optimizer's working set stays resident across rounds (GORILA_L2_PERSIST=1: on)
    cudaAccessPolicyWindow l2win{};
    bool l2_on = false;
    // fused PS exchange over NVLink peer memory (W > 1; CUDA IPC mappings of the peers' workspaces)
    bool p2p = false;
    uint8_t* ws_local = nullptr;
    uint8_t* peer_ws[MAX_W] = {};   // peer q's workspace base in this process (nullptr for self)
    void* peer_raw[MAX_W] = {};     // the opened IPC allocations (closed in gorila_destroy)
    uint64_t* pflags = nullptr;     // [4 * MAX_W] ready / done flags (two phases) written by the peers
    // gorila_round overlaps the exchange of the fc4 weight region (95% of theta) with the conv
    // backward: phase 0 of the apply runs on side2 right after the last learner's fc4 wgrad
    bool in_round = false, early_pending = false;
    // per-message PS (f1, cfg.ps_mode == 1): every local learner keeps its own gradient buffer
    bool per_msg = false;    // ps_mode 1 or 2: one gradient buffer per learner
    bool async_mode = false; // ps_mode 2 (NEXT row f2): gorila_async_run only
    AsyncState* ast = nullptr;
    uint64_t async_epoch = 0;  // gorila_async_run calls (the cross-rank start barrier's epoch)
    float* G_all = nullptr;  // [L][W*q]; G points at learner 0's
    int early_learner = -1;
    cudaStream_t side2 = nullptr;
    cudaEvent_t ev_s2_fork = nullptr, ev_s2_join = nullptr;
    uint64_t* p2p_epoch = nullptr;
    unsigned int* p2p_counter = nullptr;
    int fc4_normal_min = 256;  // batch from which fc4 runs with M = samples (GORILA_FC4_NORMAL_MIN)
    // shifted-window implicit GEMM per layer (bit 1 conv1 fwd, 2 conv2 fwd, 4 conv3 fwd, 8 conv3 dgrad,
    // 16 conv2 dgrad; the forward layers only when there are more tiles than SMs);
    // GORILA_SHIFT=<mask> selects, 0 = im2col boxes everywhere
    int shift = 31;
    bool tower = true;  // small-batch bf16 forward: conv1..conv3 fused per (net, sample) (GORILA_TOWER=0: off)
    // large-batch bf16 (B > 74): s / s' staged as u8 in row-phase-major order, expanded to bf16 inside
    // conv1's forward and weight-gradient kernels (shift_gemm.cuh U8Planes; GORILA_U8=0: bf16 NHWC)
    bool u8 = false;
    // u8 path: conv1 / conv2 forward also store their ReLU decisions as bits (EpAct::mask), which the
    // conv2 / conv3 data gradients read (EpMaskBits) instead of the activations
    uint32_t* mbits1 = nullptr;  // [B * 400] one word (32 channels) per a1 row
    uint32_t* mbits2 = nullptr;  // [B * 81][2]
    uint32_t* mbits3 = nullptr;  // [B * 49][2] = [B][98]: conv3 forward's decisions, read by fc4's data gradient
    float* part_bias[3] = {};    // u8 path: b1..b3 partials [split_w[l]][C] from the weight-gradient GEMMs
    SampleDesc* sdesc = nullptr; // u8 path: [B] the samples' ring frames (the sampler's output)
    // side stream for the weight-gradient GEMMs, which are off the dgrad critical path
    // (a fork / join of the round; a graph captures it as parallel branches)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork[4] = {}, ev_join = nullptr;
    cudaEvent_t ev_join2 = nullptr;  // side2 -> main (small batches: conv3 / conv2 weight gradients on side2)
    bool fork = true;
    // parity diagnostics (gorila_capture_activations): every learner's a1..a4 copied after its
    // forward, so that tests can read the ReLU decisions of each learner of a multi-learner step
    bool cap_acts = false;
    uint8_t* cap_buf = nullptr;  // [L][a1 | a2 | a3 (B x A* x esz) | a4 (B x 512 fp32)], cudaMalloc'ed
};

extern "C" void early_apply_p2p(gorila_ctx* ctx, uint64_t round);  // defined with the PS calls below

namespace {

enum Phase {
    PH_SAMPLE, PH_CONV1F, PH_CONV2F, PH_CONV3F, PH_FC4F, PH_FC5F, PH_TD, PH_FC5B, PH_FC4DG, PH_FC4WG,
    PH_CONV3DG, PH_CONV3WG, PH_CONV2DG, PH_CONV2WG, PH_CONV1WG, PH_BIASG, PH_WGRED, PH_STEP_MISC,
    PH_RS, PH_APPLY, PH_AG, PH_PACK, PH_SYNC, PH_COUNT
};
const char* kPhaseNames[PH_COUNT] = {
    "sample", "conv1_fwd", "conv2_fwd", "conv3_fwd", "fc4_fwd", "fc5_fwd", "td", "fc5_bwd", "fc4_dgrad",
    "fc4_wgrad", "conv3_dgrad", "conv3_wgrad", "conv2_dgrad", "conv2_wgrad", "conv1_wgrad", "bias_grad",
    "wgrad_reduce", "step_misc", "reduce_scatter", "apply", "all_gather", "pack", "target_sync"};

// record "phase ph ends here" (ph < 0: a boundary that starts the next phase)
void mark(gorila_ctx* ctx, int ph) {
    if (!ctx->prof) return;
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
    }
    if (ctx->capturing)  // becomes an event-record node of the graph, readable after each replay
        cudaEventRecordWithFlags(ctx->ev_pool[ctx->ev_used], ctx->stream, cudaEventRecordExternal);
    else
        cudaEventRecord(ctx->ev_pool[ctx->ev_used], ctx->stream);
    ctx->marks.push_back({ph, ctx->ev_used});
    ctx->ev_used++;
}

// fork: the side stream waits for everything issued so far on the main stream
void fork_side(gorila_ctx* ctx, int i) {
    cudaEventRecord(ctx->ev_fork[i], ctx->stream);
    cudaStreamWaitEvent(ctx->side, ctx->ev_fork[i], 0);
}
// join: the main stream waits for the side stream
void join_side(gorila_ctx* ctx) {
    cudaEventRecord(ctx->ev_join, ctx->side);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
}
// launches issued inside this scope go to the side stream (if `on`)
struct OnSide {
    gorila_ctx* c;
    cudaStream_t saved;
    OnSide(gorila_ctx* c_, bool on) : c(c_), saved(c_->stream) {
        if (on) c->stream = c->side;
    }
    ~OnSide() { c->stream = saved; }
};
struct OnSide2 {
    gorila_ctx* c;
    cudaStream_t saved;
    explicit OnSide2(gorila_ctx* c_) : c(c_), saved(c_->stream) { c->stream = c->side2; }
    ~OnSide2() { c->stream = saved; }
};

// fold recorded marks into the per-phase accumulators (events must be complete)
cudaError_t fold_marks(gorila_ctx* ctx, const std::vector<std::pair<int, cudaEvent_t>>& m) {
    for (size_t i = 1; i < m.size(); ++i) {
        if (m[i].first < 0) continue;
        float t = 0.f;
        cudaError_t e = cudaEventElapsedTime(&t, m[i - 1].second, m[i].second);
        if (e != cudaSuccess) return e;
        ctx->prof_ms[m[i].first] += t;
    }
    return cudaSuccess;
}

// launch attributes shared by every kernel of the library: programmatic dependent launch and the
// L2 persistence window; returns the number written (at has room for 2 more after `na`)
int base_attrs(const gorila_ctx* ctx, cudaLaunchAttribute* at, int na, bool pdl) {
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (ctx->l2_on) {
        at[na].id = cudaLaunchAttributeAccessPolicyWindow;
        at[na].val.accessPolicyWindow = ctx->l2win;
        ++na;
    }
    return na;
}

// every kernel of the round goes through here: programmatic dependent launch (the next kernel's
// launch / prologue overlaps this one; kernels griddepcontrol.wait before reading inputs)
template <typename... KP, typename... A>
void launch(gorila_ctx* ctx, void (*kern)(KP...), dim3 grid, dim3 block, size_t smem, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[3];
    cfg.attrs = at;
    cfg.numAttrs = base_attrs(ctx, at, 0, ctx->pdl);
    cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
    ctx->launches++;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// bf16 tensor map over `base` with `rank` dims (dims[0] innermost, = 8 elements = 16 B),
// byte strides of dims 1.., box and element strides. Cached per argument set.
CUtensorMap tmap(gorila_ctx* ctx, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                 const uint32_t* box, const uint32_t* es = nullptr, int swizzle = 0) {
    std::vector<uint64_t> key{(uint64_t)(uintptr_t)base, (uint64_t)rank, (uint64_t)swizzle};
    for (int i = 0; i < rank; ++i) key.push_back(dims[i]);
    for (int i = 0; i < rank - 1; ++i) key.push_back(strides[i]);
    for (int i = 0; i < rank; ++i) key.push_back(box[i]);
    for (int i = 0; i < rank; ++i) key.push_back(es ? es[i] : 1);
    auto it = ctx->tmaps.find(key);
    if (it != ctx->tmaps.end()) return it->second;
    CUtensorMap m;
    memset(&m, 0, sizeof(m));
    cuuint64_t d[5], st[4];
    cuuint32_t b[5], e[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        e[i] = es ? es[i] : 1;
    }
    for (int i = 0; i < rank - 1; ++i) st[i] = strides[i];
    auto enc = tma_encoder();
    CUresult r = enc ? enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), d, st, b, e,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                           : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                           : swizzle == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
                     : CUDA_ERROR_NOT_INITIALIZED;
    if (r != CUDA_SUCCESS) {
        ctx->tma_failed = true;
        g_last_error = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    }
    ctx->tmaps[key] = m;
    return m;
}

// K-major [rows][K] matrix (ld elements per row), tile TR rows
template <int TR>
OpMatK<TR> op_matk(gorila_ctx* ctx, const void* x, int rows, int K, int64_t ld) {
    OpMatK<TR> o;
    const uint64_t dims[3] = {8, (uint64_t)rows, (uint64_t)K / 8}, str[2] = {(uint64_t)ld * 2, 16};
    const uint32_t box[3] = {8, TR, 8};
    o.map = tmap(ctx, x, 3, dims, str, box);
    o.rows = rows;
    return o;
}
// the same, SWIZZLE_128B: map (K, rows), box (64, TR)
template <int TR>
OpMatKS<TR> op_matks(gorila_ctx* ctx, const void* x, int rows, int K, int64_t ld) {
    OpMatKS<TR> o;
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)rows}, str[1] = {(uint64_t)ld * 2};
    const uint32_t box[2] = {64, TR};
    o.map = tmap(ctx, x, 2, dims, str, box, nullptr, 128);
    o.rows = rows;
    return o;
}
// MN-major [Krows][MN] matrix (ld elements per row), tile TR columns
template <int TR>
OpMatMN<TR> op_matmn(gorila_ctx* ctx, const void* x, int krows, int mn, int64_t ld) {
    OpMatMN<TR> o;
    const uint64_t dims[3] = {8, (uint64_t)krows, (uint64_t)mn / 8}, str[2] = {(uint64_t)ld * 2, 16};
    const uint32_t box[3] = {8, 64, TR / 8};
    o.map = tmap(ctx, x, 3, dims, str, box);
    o.mn = mn;
    return o;
}
// NHWC view (8, W, H, B, G) of an activation, box (8, bw, bh, bb, bc), element strides (1, s, s, 1, 1).
// The group dimension has stride 16 B; G may exceed C/8 (groups then run into the next pixels of
// the row: used to cover several adjacent taps with one copy).
template <class SH>
CUtensorMap nhwc_map(gorila_ctx* ctx, const void* x, int B, int bw, int bh, int bb, int bc, int s) {
    const uint64_t C = SH::C;
    const uint64_t dims[5] = {8, (uint64_t)SH::W, (uint64_t)SH::H, (uint64_t)B, (uint64_t)bc};
    const uint64_t str[4] = {C * 2, SH::W * C * 2, (uint64_t)SH::H * SH::W * C * 2, 16};
    const uint32_t box[5] = {8, (uint32_t)bw, (uint32_t)bh, (uint32_t)bb, (uint32_t)bc};
    const uint32_t es[5] = {1, (uint32_t)s, (uint32_t)s, 1, 1};
    return tmap(ctx, x, 5, dims, str, box, es);
}
// swizzled forward im2col views (OpConvFwdS): 128-B rows of 64 K-elements per output pixel.
// conv3: (64 c, W, H, B); conv2: (64 = 2 pixels x 32 c, W-1 [x stride C*2], H, B), element strides 2
template <class SH>
CUtensorMap fwd_map_sw(gorila_ctx* ctx, const void* x, int B, int nb) {
    constexpr int TPC = 64 / SH::C;
    const uint64_t dims[4] = {64, (uint64_t)(SH::W - (TPC - 1)), (uint64_t)SH::H, (uint64_t)B};
    const uint64_t str[3] = {SH::C * 2, SH::W * SH::C * 2, (uint64_t)SH::H * SH::W * SH::C * 2};
    const uint32_t box[4] = {64, (uint32_t)(SH::OW * SH::S), (uint32_t)(SH::OH * SH::S), (uint32_t)nb};
    const uint32_t es[4] = {1, (uint32_t)SH::S, (uint32_t)SH::S, 1};
    return tmap(ctx, x, 4, dims, str, box, es, 128);
}
// conv1 (OpConv1FwdS): 64-B rows = 8 pixels x 4 channels at x = 4*ox: (32, 20 ox, 84 y, B)
CUtensorMap conv1_map_sw(gorila_ctx* ctx, const void* s, int B, int nb, int out_rows = H1) {
    const uint64_t dims[4] = {32, H1, 84, (uint64_t)B};
    const uint64_t str[3] = {32, 84 * 8, 84 * 84 * 8};
    const uint32_t box[4] = {32, H1, (uint32_t)(4 * out_rows), (uint32_t)nb};
    const uint32_t es[4] = {1, 1, 4, 1};
    return tmap(ctx, s, 4, dims, str, box, es, 64);
}
// swizzled output-gradient view (OpDgradS): (64 co, OW, OH, B), box (64, bw, bh, nb)
template <class SH>
CUtensorMap grad_map_sw(gorila_ctx* ctx, const void* g, int B, int bw, int bh, int bb) {
    static_assert(SH::CO == 64, "one 128-B row per tap");
    const uint64_t dims[4] = {64, (uint64_t)SH::OW, (uint64_t)SH::OH, (uint64_t)B};
    const uint64_t str[3] = {128, (uint64_t)SH::OW * 128, (uint64_t)SH::OH * SH::OW * 128};
    const uint32_t box[4] = {64, (uint32_t)bw, (uint32_t)bh, (uint32_t)bb};
    return tmap(ctx, g, 4, dims, str, box, nullptr, 128);
}
// MN-major [Krows][MN] matrix, SWIZZLE_128B: map (MN, Krows), box (64, 64)
template <int TR>
OpMatMNS<TR> op_matmns(gorila_ctx* ctx, const void* x, int krows, int mn, int64_t ld) {
    OpMatMNS<TR> o;
    const uint64_t dims[2] = {(uint64_t)mn, (uint64_t)krows}, str[1] = {(uint64_t)ld * 2};
    const uint32_t box[2] = {64, 64};
    o.map = tmap(ctx, x, 2, dims, str, box, nullptr, 128);
    o.mn = mn;
    return o;
}
// conv weight [CO][K][K][C] as (C, CO, K*K), box (C, 64, 1), swizzle = C*2 bytes
template <class SH>
CUtensorMap wdgrad_map_sw(gorila_ctx* ctx, const void* w) {
    const uint64_t dims[3] = {SH::C, SH::CO, (uint64_t)SH::K * SH::K};
    const uint64_t str[2] = {(uint64_t)SH::R * 2, SH::C * 2};
    const uint32_t box[3] = {SH::C, 64, 1};
    return tmap(ctx, w, 3, dims, str, box, nullptr, SH::C * 2);
}
// weight-gradient output-gradient operand, swizzled rows of CO*2 bytes
template <int CO, int KC, bool FLAT>
OpWgradOutS<CO, KC, FLAT> op_wgout_s(gorila_ctx* ctx, const void* g, int npix, int B) {
    OpWgradOutS<CO, KC, FLAT> o;
    if (FLAT) {
        const uint64_t dims[2] = {CO, (uint64_t)B * npix}, str[1] = {CO * 2};
        const uint32_t box[2] = {CO, KC};
        o.map = tmap(ctx, g, 2, dims, str, box, nullptr, CO * 2);
    } else {
        const uint64_t dims[3] = {CO, (uint64_t)npix, (uint64_t)B}, str[2] = {CO * 2, (uint64_t)npix * CO * 2};
        const uint32_t box[3] = {CO, KC, 1};
        o.map = tmap(ctx, g, 3, dims, str, box, nullptr, CO * 2);
    }
    return o;
}
// output-gradient view g [B][OH][OW][CO=64]: (8, OW, OH, B, 8), box (8, bw, bh, NB, 8)
template <class SH>
CUtensorMap grad_map(gorila_ctx* ctx, const void* g, int B, int bw, int bh, int bb) {
    const uint64_t dims[5] = {8, (uint64_t)SH::OW, (uint64_t)SH::OH, (uint64_t)B, SH::CO / 8};
    const uint64_t str[4] = {SH::CO * 2, (uint64_t)SH::OW * SH::CO * 2, (uint64_t)SH::OH * SH::OW * SH::CO * 2, 16};
    const uint32_t box[5] = {8, (uint32_t)bw, (uint32_t)bh, (uint32_t)bb, SH::CO / 8};
    return tmap(ctx, g, 5, dims, str, box);
}
// conv weight [CO][K][K][C] seen MN-major over c: (8, CO, C/8, K*K)
template <class SH>
CUtensorMap wdgrad_map(gorila_ctx* ctx, const void* w) {
    const uint64_t dims[4] = {8, SH::CO, SH::C / 8, (uint64_t)SH::K * SH::K};
    const uint64_t str[3] = {(uint64_t)SH::R * 2, 16, SH::C * 2};
    const uint32_t box[4] = {8, 64, SH::C / 8, 1};
    return tmap(ctx, w, 4, dims, str, box);
}

// weight-gradient output-gradient operand: g [B][npix][CO] per-sample chunks of KC rows (zero tail),
// or flat chunks of KC rows over B*npix (conv1)
template <int CO, int KC, bool FLAT>
OpWgradOut<CO, KC, FLAT> op_wgout(gorila_ctx* ctx, const void* g, int npix, int B) {
    OpWgradOut<CO, KC, FLAT> o;
    if (FLAT) {
        const uint64_t dims[3] = {8, (uint64_t)B * npix, CO / 8}, str[2] = {CO * 2, 16};
        const uint32_t box[3] = {8, KC, CO / 8};
        o.map = tmap(ctx, g, 3, dims, str, box);
    } else {
        const uint64_t dims[4] = {8, (uint64_t)npix, (uint64_t)B, CO / 8};
        const uint64_t str[3] = {CO * 2, (uint64_t)npix * CO * 2, 16};
        const uint32_t box[4] = {8, KC, 1, CO / 8};
        o.map = tmap(ctx, g, 4, dims, str, box);
    }
    return o;
}

bool cluster_env_on() {
    static const int v = [] {
        const char* e = getenv("GORILA_CLUSTER");  // GORILA_CLUSTER=0: no in-cluster split-K
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

// persistent launch: grid = min(tiles, SMs x resident CTAs per SM)
template <int BN, int MB, class OA, class OB, class EP>
void gemm_tma_p_launch(gorila_ctx* ctx, const TmaProb<OA, OB, EP>* probs, int nprob, int tilesA, int tilesB,
                       int nchunks, int splits, int N, int max_grid = 0) {
    using CFG = TmaPCfg<BN, MB, OA, OB>;
    static int occ = 0;
    if (!occ) {
        cudaFuncSetAttribute(gemm_tma_p<BN, MB, OA, OB, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, CFG::SMEM);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_tma_p<BN, MB, OA, OB, EP>, CFG::THREADS,
                                                          CFG::SMEM) != cudaSuccess ||
            occ < 1)
            occ = 1;
        occ = std::min(occ, (int)(512 / CFG::TCOLS));  // TMEM columns per SM
    }
    TmaBatch<OA, OB, EP> gb;
    memset((void*)&gb, 0, sizeof(gb));
    for (int i = 0; i < nprob; ++i) gb.prob[i] = probs[i];
    gb.nchunks = nchunks;
    gb.N = N;
    splits = std::max(1, std::min(splits, nchunks));
    gb.chunks_per_split = (nchunks + splits - 1) / splits;
    gb.splits = (nchunks + gb.chunks_per_split - 1) / gb.chunks_per_split;
    gb.cluster = 1;
    const int tiles = tilesA * tilesB * nprob * gb.splits;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min(std::min(tiles, ctx->num_sms * occ), max_grid > 0 ? max_grid : 1 << 30));
    cfg.blockDim = dim3(CFG::THREADS);
    cfg.dynamicSmemBytes = CFG::SMEM;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[3];
    cfg.attrs = at;
    cfg.numAttrs = base_attrs(ctx, at, 0, ctx->pdl);
    cudaLaunchKernelEx(&cfg, gemm_tma_p<BN, MB, OA, OB, EP>, gb, tilesA, tilesB, nprob);
    ctx->launches++;
}

// shifted-window engine: one CTA per SM, A-buffer ring as deep as shared memory allows (2..4)
template <int BN, int MB, class OA, class OB, class EP>
void gemm_shift_launch(gorila_ctx* ctx, const ShiftProb<OA, OB, EP>* probs, int nprob, int N) {
    using CFG = ShiftCfg<BN, MB, OA, OB>;
    constexpr int SMEM_MAX = 227 * 1024;
    int nbuf = SHIFT_MAX_BUF;
    while (nbuf > 2 && CFG::smem(nprob, nbuf) > SMEM_MAX) --nbuf;
    const int smem = CFG::smem(nprob, nbuf);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gemm_shift<BN, MB, OA, OB, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
        attr_set = true;
    }
    ShiftBatch<OA, OB, EP> gb;
    memset((void*)&gb, 0, sizeof(gb));
    for (int i = 0; i < nprob; ++i) gb.prob[i] = probs[i];
    gb.nprob = nprob;
    gb.nbuf = nbuf;
    gb.N = N;
    const int tiles = probs[0].a.ntiles() * nprob;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min(tiles, ctx->num_sms));
    cfg.blockDim = dim3(CFG::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[3];
    cfg.attrs = at;
    cfg.numAttrs = base_attrs(ctx, at, 0, ctx->pdl);
    cudaLaunchKernelEx(&cfg, gemm_shift<BN, MB, OA, OB, EP>, gb);
    ctx->launches++;
}
template <class W>
void wgrad_shift_launch(gorila_ctx* ctx, const WgradShiftParams& wp, int grid) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_wgrad_shift<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, wgs::Cfg<W>::SMEM);
        attr = true;
    }
    launch(ctx, k_wgrad_shift<W>, dim3(grid), dim3(192), wgs::Cfg<W>::SMEM, wp);
}
// tensor maps of the shifted-window operands
CUtensorMap sh_conv3_map(gorila_ctx* ctx, const void* a2, int B) {  // flat (64, B*81), box (64, 148)
    const uint64_t dims[2] = {64, (uint64_t)B * 81}, str[1] = {128};
    const uint32_t box[2] = {64, ShConv3Fwd::ROWS};
    return tmap(ctx, a2, 2, dims, str, box, nullptr, 128);
}
template <class SH>  // output gradient (64, OW, OH, B), box (64, 11, 11, 1)
CUtensorMap sh_grad_map(gorila_ctx* ctx, const void* g, int B) {
    const uint64_t dims[4] = {64, (uint64_t)SH::OW, (uint64_t)SH::OH, (uint64_t)B};
    const uint64_t str[3] = {128, (uint64_t)SH::OW * 128, (uint64_t)SH::OH * SH::OW * 128};
    const uint32_t box[4] = {64, 11, 11, 1};
    return tmap(ctx, g, 4, dims, str, box, nullptr, 128);
}
CUtensorMap sh_conv2_map(gorila_ctx* ctx, const void* a1, int B) {  // phase planes of a1 (64-B rows)
    const uint64_t dims[4] = {32, 20, 20, (uint64_t)B};
    const uint64_t str[3] = {64, 20 * 64, 400 * 64};
    const uint32_t box[4] = {32, 20, 20, 1}, es[4] = {1, 2, 2, 1};
    return tmap(ctx, a1, 4, dims, str, box, es, 64);
}
CUtensorMap sh_conv1_map(gorila_ctx* ctx, const void* s, int B) {  // row phases of s (32-B rows)
    const uint64_t dims[4] = {16, 21, 84, (uint64_t)B};
    const uint64_t str[3] = {32, 84 * 8, 84 * 84 * 8};
    const uint32_t box[4] = {16, 21, 84, 1}, es[4] = {1, 1, 4, 1};
    return tmap(ctx, s, 4, dims, str, box, es, 32);
}
template <int CO, int RB, int NCH, int KOFF>  // K-major weight [CO][Ktot], box (RB/2, CO)
ShWeightK<CO, RB, NCH, KOFF> sh_wk(gorila_ctx* ctx, const void* w, int ktot) {
    ShWeightK<CO, RB, NCH, KOFF> o;
    const uint64_t dims[2] = {(uint64_t)ktot, CO}, str[1] = {(uint64_t)ktot * 2};
    const uint32_t box[2] = {RB / 2, CO};
    o.map = tmap(ctx, w, 2, dims, str, box, nullptr, RB);
    return o;
}

// grid + launch of the TMA engine (cluster split-K when cluster_target > 0)
template <int BN, int MB, class OA, class OB, class EP>
void gemm_tma_launch(gorila_ctx* ctx, const TmaProb<OA, OB, EP>* probs, int nprob, int tilesA, int tilesB,
                     int nchunks, int splits, int cluster_target, int N, int cl_cap = 0) {
    using CFG = TmaCfg<BN, MB, OA, OB>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gemm_tma<BN, MB, OA, OB, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, CFG::SMEM);
        cudaFuncSetAttribute(gemm_tma<BN, MB, OA, OB, EP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr_set = true;
    }
    static const bool persist_env = [] {
        const char* e = getenv("GORILA_PERSIST");  // GORILA_PERSIST=0: one CTA per tile (gemm_tma)
        return !(e && atoi(e) == 0);
    }();
    int cl = 1;  // in-cluster split-K size
    if (MB == 1 && cluster_target > 0 && cluster_env_on()) {
        const int tiles = tilesA * tilesB * nprob;
        const int want = std::max(1, (cluster_target + tiles - 1) / tiles);
        static const int cl_max = [] {
            const char* e = getenv("GORILA_CLUSTER_MAX");  // in-cluster split-K size cap (default 8)
            return e ? std::max(1, std::min(16, atoi(e))) : 8;
        }();
        while (cl * 2 <= std::min(cl_cap > 0 ? cl_cap : cl_max, std::min(want, nchunks))) cl *= 2;
    }
    if (persist_env && cl == 1 &&
        (int64_t)tilesA * tilesB * nprob * std::max(1, std::min(splits, nchunks)) > ctx->num_sms) {
        gemm_tma_p_launch<BN, MB>(ctx, probs, nprob, tilesA, tilesB, nchunks, splits, N);
        return;
    }
    TmaBatch<OA, OB, EP> gb;
    memset((void*)&gb, 0, sizeof(gb));
    for (int i = 0; i < nprob; ++i) gb.prob[i] = probs[i];
    gb.nchunks = nchunks;
    gb.N = N;
    splits = std::max(1, std::min(splits, nchunks));
    gb.chunks_per_split = (nchunks + splits - 1) / splits;
    gb.splits = (nchunks + gb.chunks_per_split - 1) / gb.chunks_per_split;
    gb.cluster = 1;
    if (cl > 1) {
        gb.cluster = cl;
        gb.splits = cl;
        gb.chunks_per_split = (nchunks + cl - 1) / cl;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(tilesA, tilesB, nprob * gb.splits);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = CFG::SMEM;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[4];
    int na = 0;
    if (gb.cluster > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = 1;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = gb.cluster;
        ++na;
    }
    na = base_attrs(ctx, at, na, ctx->pdl);
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, gemm_tma<BN, MB, OA, OB, EP>, gb);
    ctx->launches++;
}

int pick_splits(int64_t chunks_total, int64_t base_ctas, int target_ctas, int max_splits) {
    int64_t s = std::max<int64_t>(1, std::min<int64_t>(max_splits, (target_ctas + base_ctas - 1) / base_ctas));
    s = std::min<int64_t>(s, chunks_total);
    return (int)s;
}

// ------------------------------------------------------------------ GEMM dispatch
template <typename LA, typename LB, typename EP>
void launch_simt(GemmBatch<LA, LB, EP> gb, int nprob, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((gb.M + SM_BI - 1) / SM_BI, (gb.N + SM_BJ - 1) / SM_BJ, nprob * gb.splits);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, gemm_simt<LA, LB, EP>, gb);
}

// fp32 check mode: C[M][N] = sum_r A(i,r) B(j,r) on the SIMT engine. `splits` requested split of
// the reduction (rounded to whole chunks) into partial outputs (the epilogue gets the split index).
// The last argument is ignored (call sites keep the CTA target their bf16 twin uses).
template <typename T, int BN, typename LA, typename LB, typename EP>
void gemm(gorila_ctx* ctx, const GemmProb<LA, LB, EP>* probs, int nprob, int M, int N, int R, int splits,
          int = 0) {
    static_assert(std::is_same<T, float>::value, "the bf16 path runs the TMA / shifted-window engines");
    GemmBatch<LA, LB, EP> gb{};
    for (int i = 0; i < nprob; ++i) gb.prob[i] = probs[i];
    if (nprob == 1) gb.prob[1] = probs[0];
    gb.M = M;
    gb.N = N;
    gb.R = R;
    const int chunks = std::max(1, (R + SM_BR - 1) / SM_BR);
    splits = std::max(1, std::min(splits, chunks));
    gb.chunks_per_split = (chunks + splits - 1) / splits;
    gb.splits = (chunks + gb.chunks_per_split - 1) / gb.chunks_per_split;
    gb.cluster = 1;
    launch_simt(gb, nprob, ctx->stream, ctx->pdl);
    LAUNCHED();
}

template <typename T>
T* P_(void* p) {
    return reinterpret_cast<T*>(p);
}

// number of effective splits the gemm() call will use (so partial buffers are consistent)
int eff_splits(bool fp32, int R, int splits) {
    const int chunk = fp32 ? SM_BR : TC_BK;
    const int chunks = std::max(1, (R + chunk - 1) / chunk);
    splits = std::max(1, std::min(splits, chunks));
    const int cps = (chunks + splits - 1) / splits;
    return (chunks + cps - 1) / cps;
}

// the fc4 forward / dgrad N tile (= batch columns)
#define DISPATCH_BN_BATCH(B, CALL) \
    do {                           \
        if ((B) <= 32) { CALL(32); } else if ((B) <= 64) { CALL(64); } else if ((B) <= 128) { CALL(128); } else { CALL(256); } \
    } while (0)

// ------------------------------------------------------------------ one learner update
// GORILA_REPLAY_BARRIER=0: diagnostics only (timing; no parity guarantee across ranks)
static bool replay_barrier_off() {
    static const bool off = [] {
        const char* e = getenv("GORILA_REPLAY_BARRIER");
        return e && atoi(e) == 0;
    }();
    return off;
}

template <typename T>
gorila_status run_learner(gorila_ctx* ctx, int j, uint64_t round, int s_j, int accumulate,
                          uint32_t phases = 0xffffffffu) {
#define PHASE(ph) if (phases & (1u << (ph)))
    // fork the weight-gradient GEMMs and the bias partials onto the side stream (full rounds only;
    // phase profiling keeps one stream so that its marks bracket single kernels)
    const bool fk = ctx->fork && ctx->side && !ctx->prof && phases == ~0u;
    const gorila_config& cfg = ctx->cfg;
    Learner& Lr = ctx->learners[j];
    const int B = ctx->B, nA = ctx->nA;
    constexpr bool fp32v = std::is_same<T, float>::value;
    const uint64_t k_src = round >= (uint64_t)s_j ? round - (uint64_t)s_j : 0;
    // asynchronous mode (f2): the replica the learner fetched (slot 1; slot 0 is the servers' live one)
    const int slot = ctx->async_mode ? 1 : (int)(k_src % (uint64_t)ctx->H);
    // gradient destination: the shared sum, or (per-message mode) this learner's own buffer
    float* const Gd = ctx->per_msg ? ctx->G_all + (int64_t)j * ctx->W * ctx->q : ctx->G;
    // the round's first learner resets the accepted count; the others add to it (also in
    // per-message mode, where every learner writes its own gradient buffer: accumulate = 0)
    const bool first_learner = accumulate == 0;
    if (ctx->per_msg) accumulate = 0;
    const T* rt = P_<T>(ctx->rep_t[slot]);
    const float* rf = ctx->rep_f[slot];
    const T* tt = P_<T>(Lr.tminus_t);
    const float* tf = Lr.tminus_f;
    const ReplicaLayout& RL = ctx->rl;
    const ReplicaLayout& RT = ctx->rl;

    T *s = P_<T>(ctx->s), *s2 = P_<T>(ctx->s2);
    T *a1 = P_<T>(ctx->a1), *a2 = P_<T>(ctx->a2), *a3 = P_<T>(ctx->a3);
    T *t1 = P_<T>(ctx->t1), *t2 = P_<T>(ctx->t2), *t3 = P_<T>(ctx->t3);
    float *a4 = ctx->a4, *t4 = ctx->t4;
    T *g1 = P_<T>(ctx->g1), *g2 = P_<T>(ctx->g2), *g3 = P_<T>(ctx->g3), *g4 = P_<T>(ctx->g4);

    const float in_scale = 1.0f / 255.0f;  // reading R17 (fp32 constant, folded into conv1's epilogue)
    PHASE(PH_SAMPLE) {
    // K1: sample + gather + stack (Alg.1)
    {
        dim3 grid((FRAME_BYTES / 16 + 255) / 256, B);
        uint2 key = make_uint2((uint32_t)cfg.seed, (uint32_t)(cfg.seed >> 32));
        using ST = std::conditional_t<fp32v, T, uint8_t>;  // (bf16: u8 staging when ctx->u8)
        if (!fp32v && ctx->u8)  // the samples' frame addresses only (one block of three warps per sample:
                                // threads 0-3 / 32 / 64 load the flags / action / reward)
            launch(ctx, k_sample<ST>, dim3(1, B), dim3(96), 0, (const uint8_t*)Lr.frames, (const uint8_t*)Lr.a,
                   (const float*)Lr.r, (const uint8_t*)Lr.d, (int64_t)cfg.replay_capacity, (const uint64_t*)Lr.n_dev,
                   (const ShardPtrs*)(ctx->replay_global ? ctx->shard_tab : nullptr), ctx->n_shards,
                   (const uint64_t*)(ctx->replay_global && ctx->W > 1 && !replay_barrier_off() ? ctx->n_snap : nullptr),
                   ctx->sshard, key,
                   (uint32_t)(cfg.learner_id_base + j), (const uint64_t*)ctx->dev_round, B, (ST*)ctx->sdesc, (ST*)nullptr,
                   ctx->sa, ctx->sr, ctx->sd, ctx->sidx, first_learner ? ctx->n_acc_local : (uint32_t*)nullptr);
        else
        launch(ctx, k_sample<T>, grid, dim3(256), 0, (const uint8_t*)Lr.frames, (const uint8_t*)Lr.a,
               (const float*)Lr.r, (const uint8_t*)Lr.d, (int64_t)cfg.replay_capacity, (const uint64_t*)Lr.n_dev,
               (const ShardPtrs*)(ctx->replay_global ? ctx->shard_tab : nullptr), ctx->n_shards,
               (const uint64_t*)(ctx->replay_global && ctx->W > 1 && !replay_barrier_off() ? ctx->n_snap : nullptr),
               ctx->sshard, key,
               (uint32_t)(cfg.learner_id_base + j), (const uint64_t*)ctx->dev_round, B, s, s2, ctx->sa, ctx->sr,
               ctx->sd, ctx->sidx, first_learner ? ctx->n_acc_local : (uint32_t*)nullptr);
    }
    }
    mark(ctx, PH_SAMPLE);
    // GORILA_FC5_FUSE=1 (B <= 32): the fc5 backward runs inside k_fc5_td after a grid-wide wait on
    // the TD decision (one launch fewer). Opt-in: measured 12.39k vs 12.57k updates/s unfused, the
    // spin on the decision costs more than the launch it saves.
    static const bool fc5_fuse_env = [] {
        const char* e = getenv("GORILA_FC5_FUSE");
        return e && atoi(e) != 0;
    }();
    const bool fc5_fused = fc5_fuse_env && B <= 32 && (phases & (1u << PH_FC5F)) && (phases & (1u << PH_FC5B));
    // small batches (bf16): conv1 -> conv2 -> conv3 of a (net, sample) in one CTA (tower.cuh)
    const bool use_tower = !fp32v && ctx->tower && 2 * B <= ctx->num_sms;
    PHASE(PH_CONV1F) if (use_tower) {
        TowerParams tp{};
        tp.in_scale = in_scale;
        tp.batch = B;
        for (int z = 0; z < 2; ++z) {
            TowerNet& N = tp.net[z];
            N.s_map = sh_conv1_map(ctx, z ? (const void*)s2 : (const void*)s, B);
            N.w1_map = sh_wk<32, 32, 16, 2>(ctx, z ? (const void*)(tt + RT.w1) : (const void*)(rt + RL.w1), K1).map;
            N.w2_map = sh_wk<64, 64, 16, 1>(ctx, z ? (const void*)(tt + RT.w2) : (const void*)(rt + RL.w2), K2).map;
            N.w3_map = sh_wk<64, 128, 9, 0>(ctx, z ? (const void*)(tt + RT.w3) : (const void*)(rt + RL.w3), K3).map;
            N.a1 = (__nv_bfloat16*)(z ? t1 : a1);
            N.a2 = (__nv_bfloat16*)(z ? t2 : a2);
            N.a3 = (__nv_bfloat16*)(z ? t3 : a3);
            N.b1 = z ? tf + RT.b1 : rf + RL.b1;
            N.b2 = z ? tf + RT.b2 : rf + RL.b2;
            N.b3 = z ? tf + RT.b3 : rf + RL.b3;
        }
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_conv_tower, cudaFuncAttributeMaxDynamicSharedMemorySize, tower::SMEM);
            attr = true;
        }
        launch(ctx, k_conv_tower, dim3(B, 2), dim3(tower::THREADS), tower::SMEM, tp);
    } else {
    // conv1 fwd (online on s with theta, target on s' with theta^-)
    {
        const int M = B * H1 * H1;
        if constexpr (fp32v) {
            using LA = LdConvIn<T, Conv1>; using LB = LdRows<T>; using EP = EpAct<T>;
            GemmProb<LA, LB, EP> pr[2] = {
                {{s, M}, {rt + RL.w1, K1, C1_OUT, K1}, {a1, C1_OUT, rf + RL.b1, in_scale, M, C1_OUT, 1}},
                {{s2, M}, {tt + RT.w1, K1, C1_OUT, K1}, {t1, C1_OUT, tf + RT.b1, in_scale, M, C1_OUT, 1}}};
            gemm<T, 32>(ctx, pr, 2, M, C1_OUT, K1, 1);
        } else if (ctx->u8) {  // shifted windows over the row phases, expanded from the u8 staging
            using OA = ShConv1FwdU8; using OB = ShWeightK<32, 32, 16, 2>; using EP = EpAct<T>;
            ShiftProb<OA, OB, EP> pr[2];
            for (int z = 0; z < 2; ++z) {
                pr[z].a.desc = ctx->sdesc;
                pr[z].a.z = z;
                pr[z].a.batch = B;
                pr[z].b = sh_wk<32, 32, 16, 2>(ctx, z ? (const void*)(tt + RT.w1) : (const void*)(rt + RL.w1), K1);
                pr[z].ep = {z ? t1 : a1, C1_OUT, z ? tf + RT.b1 : rf + RL.b1, in_scale, M, C1_OUT, 1};
            }
            pr[0].ep.mask = ctx->mbits1;  // the online net's ReLU decisions for conv2's data gradient
            gemm_shift_launch<32, 4>(ctx, pr, 2, C1_OUT);
        } else if ((ctx->shift & 1) && 2 * B > ctx->num_sms) {  // shifted windows over the row phases of s
#define SH_C1(MS_, MB_)                                                                                        \
    {                                                                                                          \
        using OA = ShConv1Fwd<MS_>; using OB = ShWeightK<32, 32, 16, 2>; using EP = EpAct<T>;                  \
        ShiftProb<OA, OB, EP> pr[2];                                                                           \
        for (int z = 0; z < 2; ++z) {                                                                          \
            pr[z].a.map = sh_conv1_map(ctx, z ? (const void*)s2 : (const void*)s, B);                          \
            pr[z].a.batch = B;                                                                                 \
            pr[z].b = sh_wk<32, 32, 16, 2>(ctx, z ? (const void*)(tt + RT.w1) : (const void*)(rt + RL.w1), K1); \
            pr[z].ep = {z ? t1 : a1, C1_OUT, z ? tf + RT.b1 : rf + RL.b1, in_scale, M, C1_OUT, 1};             \
        }                                                                                                      \
        gemm_shift_launch<32, MB_>(ctx, pr, 2, C1_OUT);                                                        \
    }
            SH_C1(1, 4)
#undef SH_C1
        } else {  // TMA: one sample (400 rows = 4 M-blocks) per tile, pixel-pair im2col boxes
            using OA = OpConv1FwdS<4>; using OB = OpMatKS<32>; using EP = EpAct<T>;
            TmaProb<OA, OB, EP> pr[2];
            for (int z = 0; z < 2; ++z) {
                pr[z].a.map = conv1_map_sw(ctx, z ? (const void*)s2 : (const void*)s, B, 1);
                pr[z].a.nb = 1;
                pr[z].a.batch = B;
                pr[z].b = op_matks<32>(ctx, z ? (const void*)(tt + RT.w1) : (const void*)(rt + RL.w1), C1_OUT, K1, K1);
                pr[z].ep = {z ? t1 : a1, C1_OUT, z ? tf + RT.b1 : rf + RL.b1, in_scale, M, C1_OUT, 1};
            }
            gemm_tma_launch<32, 4>(ctx, pr, 2, B, 1, K1 / 64, 1, 0, C1_OUT);
        }
    }
    }
    mark(ctx, PH_CONV1F);
    PHASE(PH_CONV2F) if (!use_tower) {
    // conv2 fwd
    {
        const int M = B * H2 * H2;
        if constexpr (fp32v) {
            using LA = LdConvIn<T, Conv2>; using LB = LdRows<T>; using EP = EpAct<T>;
            GemmProb<LA, LB, EP> pr[2] = {
                {{a1, M}, {rt + RL.w2, K2, C2_OUT, K2}, {a2, C2_OUT, rf + RL.b2, 1.f, M, C2_OUT, 1}},
                {{t1, M}, {tt + RT.w2, K2, C2_OUT, K2}, {t2, C2_OUT, tf + RT.b2, 1.f, M, C2_OUT, 1}}};
            gemm<T, 64>(ctx, pr, 2, M, C2_OUT, K2, 1, 148);
        } else if ((ctx->shift & 2) && 2 * B > ctx->num_sms) {  // shifted windows over the stride phases of a1
            using OA = ShConv2Fwd; using OB = ShWeightK<64, 64, 16, 1>; using EP = EpAct<T>;
            ShiftProb<OA, OB, EP> pr[2];
            for (int z = 0; z < 2; ++z) {
                pr[z].a.map = sh_conv2_map(ctx, z ? (const void*)t1 : (const void*)a1, B);
                pr[z].a.batch = B;
                pr[z].b = sh_wk<64, 64, 16, 1>(ctx, z ? (const void*)(tt + RT.w2) : (const void*)(rt + RL.w2), K2);
                pr[z].ep = {z ? t2 : a2, C2_OUT, z ? tf + RT.b2 : rf + RL.b2, 1.f, M, C2_OUT, 1};
            }
            if (ctx->u8) pr[0].ep.mask = ctx->mbits2;
            gemm_shift_launch<64, 1>(ctx, pr, 2, C2_OUT);
        } else {  // TMA: one sample (81 rows) per tile, stride-2 boxes; in-cluster split of K = 512
            using OA = OpConvFwdS<Conv2, 1>; using OB = OpMatKS<64>; using EP = EpAct<T>;
            TmaProb<OA, OB, EP> pr[2];
            for (int z = 0; z < 2; ++z) {
                pr[z].a.map = fwd_map_sw<Conv2>(ctx, z ? (const void*)t1 : (const void*)a1, B, 1);
                pr[z].a.nb = 1;
                pr[z].a.batch = B;
                pr[z].b = op_matks<64>(ctx, z ? (const void*)(tt + RT.w2) : (const void*)(rt + RL.w2), C2_OUT, K2, K2);
                pr[z].ep = {z ? t2 : a2, C2_OUT, z ? tf + RT.b2 : rf + RL.b2, 1.f, M, C2_OUT, 1};
            }
            gemm_tma_launch<64, 1>(ctx, pr, 2, B, 1, K2 / 64, 1, 0, C2_OUT);
        }
    }
    }
    mark(ctx, PH_CONV2F);
    PHASE(PH_CONV3F) if (!use_tower) {
    // conv3 fwd
    {
        const int M = B * H3 * H3;
        if constexpr (fp32v) {
            using LA = LdConvIn<T, Conv3>; using LB = LdRows<T>; using EP = EpAct<T>;
            GemmProb<LA, LB, EP> pr[2] = {
                {{a2, M}, {rt + RL.w3, K3, C3_OUT, K3}, {a3, C3_OUT, rf + RL.b3, 1.f, M, C3_OUT, 1}},
                {{t2, M}, {tt + RT.w3, K3, C3_OUT, K3}, {t3, C3_OUT, tf + RT.b3, 1.f, M, C3_OUT, 1}}};
            gemm<T, 64>(ctx, pr, 2, M, C3_OUT, K3, 1, 148);
        } else if ((ctx->shift & 4) && 2 * B > ctx->num_sms) {  // shifted windows over the pixel rows of a2
            using OA = ShConv3Fwd; using OB = ShWeightK<64, 128, 9, 0>; using EP = EpAct<T>;
            ShiftProb<OA, OB, EP> pr[2];
            for (int z = 0; z < 2; ++z) {
                pr[z].a.map = sh_conv3_map(ctx, z ? (const void*)t2 : (const void*)a2, B);
                pr[z].a.batch = B;
                pr[z].b = sh_wk<64, 128, 9, 0>(ctx, z ? (const void*)(tt + RT.w3) : (const void*)(rt + RL.w3), K3);
                pr[z].ep = {z ? t3 : a3, C3_OUT, z ? tf + RT.b3 : rf + RL.b3, 1.f, M, C3_OUT, 1};
            }
            if (ctx->u8) pr[0].ep.mask = ctx->mbits3;
            gemm_shift_launch<64, 1>(ctx, pr, 2, C3_OUT);
        } else {  // TMA: two samples (98 rows) per tile, one tap per K-chunk
            using OA = OpConvFwdS<Conv3, 1>; using OB = OpMatKS<64>; using EP = EpAct<T>;
            TmaProb<OA, OB, EP> pr[2];
            for (int z = 0; z < 2; ++z) {
                pr[z].a.map = fwd_map_sw<Conv3>(ctx, z ? (const void*)t2 : (const void*)a2, B, 2);
                pr[z].a.nb = 2;
                pr[z].a.batch = B;
                pr[z].b = op_matks<64>(ctx, z ? (const void*)(tt + RT.w3) : (const void*)(rt + RL.w3), C3_OUT, K3, K3);
                pr[z].ep = {z ? t3 : a3, C3_OUT, z ? tf + RT.b3 : rf + RL.b3, 1.f, M, C3_OUT, 1};
            }
            gemm_tma_launch<64, 1>(ctx, pr, 2, (B + 1) / 2, 1, K3 / 64, 1, 0, C3_OUT);
        }
    }
    }
    mark(ctx, PH_CONV3F);
    PHASE(PH_FC4F) {
    // fc4 fwd, swap-AB (i = n, j = b): a4[b][n] = ReLU(W4[n] . a3[b] + b4[n]) in fp32, the split of
    // K = 3136 reduced inside the cluster (no partial buffers, no finalize kernel)
    {
        if constexpr (fp32v) {
            using LA = LdRows<T>; using LB = LdRows<T>; using EP = EpActT;
            GemmProb<LA, LB, EP> pr[2] = {
                {{rt + RL.w4, FC4_IN, FC4_OUT, FC4_IN}, {a3, FC4_IN, B, FC4_IN}, {a4, FC4_OUT, rf + RL.b4, FC4_OUT, B}},
                {{tt + RT.w4, FC4_IN, FC4_OUT, FC4_IN}, {t3, FC4_IN, B, FC4_IN}, {t4, FC4_OUT, tf + RT.b4, FC4_OUT, B}}};
            gemm<T, 32>(ctx, pr, 2, FC4_OUT, B, FC4_IN, 1, 148);
        } else {
#define FC4F(BN_)                                                                                              \
    {                                                                                                          \
        using OA = OpMatKS<128>; using OB = OpMatKS<BN_>; using EP = EpActT;                                   \
        TmaProb<OA, OB, EP> pr[2];                                                                             \
        for (int z = 0; z < 2; ++z) {                                                                          \
            pr[z].a = op_matks<128>(ctx, z ? (const void*)(tt + RT.w4) : (const void*)(rt + RL.w4), FC4_OUT,    \
                                   FC4_IN, FC4_IN);                                                            \
            pr[z].b = op_matks<BN_>(ctx, z ? (const void*)t3 : (const void*)a3, B, FC4_IN, FC4_IN);            \
            pr[z].ep = {z ? t4 : a4, FC4_OUT, z ? tf + RT.b4 : rf + RL.b4, FC4_OUT, B};                        \
        }                                                                                                      \
        gemm_tma_launch<BN_, 1>(ctx, pr, 2, FC4_OUT / 128, (B + BN_ - 1) / BN_, FC4_IN / 64, 1, 148, B);      \
    }
            if (B >= ctx->fc4_normal_min) {  // large batch: M = samples, N = 512 outputs (row-major stores)
                using OA = OpMatKS<128>; using OB = OpMatKS<128>; using EP = EpAct<float>;
                TmaProb<OA, OB, EP> pr[2];
                for (int z = 0; z < 2; ++z) {
                    pr[z].a = op_matks<128>(ctx, z ? (const void*)t3 : (const void*)a3, B, FC4_IN, FC4_IN);
                    pr[z].b = op_matks<128>(ctx, z ? (const void*)(tt + RT.w4) : (const void*)(rt + RL.w4), FC4_OUT,
                                            FC4_IN, FC4_IN);
                    pr[z].ep = {z ? t4 : a4, FC4_OUT, z ? tf + RT.b4 : rf + RL.b4, 1.f, B, FC4_OUT, 1};
                }
                gemm_tma_launch<128, 1>(ctx, pr, 2, (B + 127) / 128, FC4_OUT / 128, FC4_IN / 64, 1, 0, FC4_OUT);
            } else {
                DISPATCH_BN_BATCH(B, FC4F);
            }
#undef FC4F
        }
    }
    }
    mark(ctx, PH_FC4F);
    PHASE(PH_FC5F) {
    // fc5 forward (both nets) + K7: TD target, clipped error, loss, outlier + stale decisions
    {
        Fc5TdParams p{};
        p.a4 = a4; p.t4 = t4; p.w5 = rf + RL.w5; p.b5 = rf + RL.b5; p.w5t = tf + RT.w5; p.b5t = tf + RT.b5;
        p.counter = ctx->head_counter;
        TdParams& t = p.td;
        t.Q = Lr.Q; t.Qhat = Lr.Qhat; t.a = ctx->sa; t.r = ctx->sr; t.d = ctx->sd; t.dQ = ctx->dQ;
        t.B = B; t.nA = nA; t.gamma = cfg.gamma; t.stats = Lr.stats; t.info = Lr.info; t.V = ctx->V;
        t.base_V = ctx->Vhist + slot; t.n_acc_local = ctx->n_acc_local; t.max_staleness = ctx->per_msg ? -1 : cfg.max_staleness;  // per-message: judged at the PS (R37)
        t.outlier_enabled = cfg.outlier_enabled; t.outlier_warmup = cfg.outlier_warmup;
        t.outlier_k = cfg.outlier_k; t.outlier_beta = cfg.outlier_beta;
        p.per_sample = ctx->td_partial;
        if (fc5_fused) {
            p.fuse_bwd = 1;
            p.gen = ctx->fc5_gen;
            p.part5 = ctx->part5;
            p.g4 = g4;
            p.bf16 = !fp32v;
        }
        if (B >= 256 && !fc5_fused) {  // large batch: one warp per sample, W5 in shared memory
            const size_t smem = (size_t)(2 * nA * FC4_OUT + 64) * sizeof(float);
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_fc5_td_wide<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * 32 * FC4_OUT + 64) * 4);
                cudaFuncSetAttribute(k_fc5_td_wide<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * 32 * FC4_OUT + 64) * 4);
                cudaFuncSetAttribute(k_fc5_td_wide<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * 32 * FC4_OUT + 64) * 4);
                attr = true;
            }
            // S samples per warp, nw warps per block: every W5 element read from shared memory feeds S
            // FMAs (shared-memory bandwidth) while nw warps hide the warp sums' latency
            static const int env_s = [] { const char* e = getenv("GORILA_FC5W_S"); return e ? atoi(e) : 0; }();
            static const int env_w = [] { const char* e = getenv("GORILA_FC5W_WARPS"); return e ? atoi(e) : 0; }();
            const int per_sm = (B + ctx->num_sms - 1) / ctx->num_sms;
            // measured (tools/fc5w_sweep.sh, phase us at B = 256 / 1024 / 4096): S = 2 with 4 warps
            // 9.7 / 9.9 / 21.7, with 8 warps 10.8 / 11.1 / 19.4; S = 1 x 16 warps 14.2 / 14.5 / 23.7;
            // S = 4 x 4 / 8 warps 14.2-16.8 / 20.6-21.9
            const int S = env_s == 1 || env_s == 2 || env_s == 4 ? env_s : 2;
            const int nw = env_w > 0 ? std::min(env_w, FC5W_WARPS) : per_sm >= 16 ? 8 : 4;
            const dim3 grid(std::min((B + nw * S - 1) / (nw * S), 2 * ctx->num_sms));
            if (S == 1) launch(ctx, k_fc5_td_wide<1>, grid, dim3(nw * 32), smem, p);
            else if (S == 2) launch(ctx, k_fc5_td_wide<2>, grid, dim3(nw * 32), smem, p);
            else launch(ctx, k_fc5_td_wide<4>, grid, dim3(nw * 32), smem, p);
        } else {
            launch(ctx, k_fc5_td, dim3(fc5_fused ? B : std::min(B, 2 * 148)), dim3(512), 0, p);
        }
    }
    }
    mark(ctx, PH_FC5F);
    mark(ctx, PH_TD);
    PHASE(PH_FC5B) if (!fc5_fused) {
    // fc5 bwd: dW5, db5 into G; g4 = mask(dQ W5)
    {
        const int nch = (B + fc5_rows(B) - 1) / fc5_rows(B);
        const int g4_blocks = (B + 7) / 8;  // one warp per sample
        launch(ctx, k_fc5_bwd<T>, dim3(2 * nch + g4_blocks), dim3(256), 0,
               (const float*)ctx->dQ, (const float*)a4, (const float*)(rf + RL.w5), B, nA, ctx->part5, nch, g4,
               (const uint8_t*)ctx->sa);
    }
    }
    mark(ctx, PH_FC5B);
    if (fk) fork_side(ctx, 0);  // g4 ready: fc4 wgrad may start
    PHASE(PH_FC4DG) {
    // fc4 dgrad (i = k, j = b, red = n): g3[b][k] = mask(sum_n W4[n][k] g4[b][n])
    {
        if constexpr (fp32v) {
            using LA = LdRowsMN<T>; using LB = LdRows<T>; using EP = EpMaskT<T>;
            GemmProb<LA, LB, EP> pr[1] = {{{rt + RL.w4, FC4_IN, FC4_IN, FC4_OUT}, {g4, FC4_OUT, B, FC4_OUT},
                                           {g3, a3, FC4_IN, FC4_IN, B}}};
            gemm<T, 32>(ctx, pr, 1, FC4_IN, B, FC4_OUT, 1, 148);
        } else {
#define FC4D(BN_)                                                                                              \
    {                                                                                                          \
        using OA = OpMatMNS<128>; using OB = OpMatKS<BN_>; using EP = EpMaskT<T>;                              \
        TmaProb<OA, OB, EP> pr[1];                                                                             \
        pr[0].a = op_matmns<128>(ctx, rt + RL.w4, FC4_OUT, FC4_IN, FC4_IN);                                    \
        pr[0].b = op_matks<BN_>(ctx, g4, B, FC4_OUT, FC4_OUT);                                                 \
        pr[0].ep = {g3, a3, FC4_IN, FC4_IN, B};                                                                \
        gemm_tma_launch<BN_, 1>(ctx, pr, 1, (FC4_IN + 127) / 128, (B + BN_ - 1) / BN_, FC4_OUT / 64, 1, 148, B); \
    }
            if (B >= ctx->fc4_normal_min && ctx->u8 && (ctx->shift & 4)) {  // as below, decisions as bits
                using OA = OpMatKS<128>; using OB = OpMatMNS<256>; using EP = EpMaskBits<T>;
                TmaProb<OA, OB, EP> pr[1];
                pr[0].a = op_matks<128>(ctx, g4, B, FC4_OUT, FC4_OUT);
                pr[0].b = op_matmns<256>(ctx, rt + RL.w4, FC4_OUT, FC4_IN, FC4_IN);
                pr[0].ep = {g3, ctx->mbits3, FC4_IN, B, FC4_IN, FC4_IN / 32};
                gemm_tma_launch<256, 1>(ctx, pr, 1, (B + 127) / 128, (FC4_IN + 255) / 256, FC4_OUT / 64, 1, 0, FC4_IN);
            } else if (B >= ctx->fc4_normal_min) {  // large batch: M = samples, N = 3136 (row-major masked stores)
                using OA = OpMatKS<128>; using OB = OpMatMNS<256>; using EP = EpMask<T>;
                TmaProb<OA, OB, EP> pr[1];
                pr[0].a = op_matks<128>(ctx, g4, B, FC4_OUT, FC4_OUT);
                pr[0].b = op_matmns<256>(ctx, rt + RL.w4, FC4_OUT, FC4_IN, FC4_IN);
                pr[0].ep = {g3, a3, FC4_IN, B, FC4_IN};
                gemm_tma_launch<256, 1>(ctx, pr, 1, (B + 127) / 128, (FC4_IN + 255) / 256, FC4_OUT / 64, 1, 0, FC4_IN);
            } else {
                DISPATCH_BN_BATCH(B, FC4D);
            }
#undef FC4D
        }
    }
    }
    mark(ctx, PH_FC4DG);
    // K10's segments: 0 W1, 1 W2, 2 W3, 3..6 b1..b4 (wide: many partials per element), 7 W5 + b5
    WgradReduceParams all{};
    {
        all.part[0] = ctx->part_w[0]; all.part[1] = ctx->part_w[1]; all.part[2] = ctx->part_w[2];
        all.splits[0] = ctx->split_w[0];
        all.splits[1] = ctx->split_w[1];
        all.splits[2] = ctx->split_w[2];
        all.count[0] = (int64_t)C1_OUT * K1; all.count[1] = (int64_t)C2_OUT * K2; all.count[2] = (int64_t)C3_OUT * K3;
        all.off[0] = OFF_W1; all.off[1] = OFF_W2; all.off[2] = OFF_W3;
        const int bc[4] = {C1_OUT, C2_OUT, C3_OUT, FC4_OUT};
        const int64_t boff[4] = {OFF_B1, OFF_B2, OFF_B3, OFF_B4};
        const float* bp = ctx->part_b;
        for (int l = 0; l < 4; ++l) {
            all.part[3 + l] = bp; all.splits[3 + l] = ctx->bias_chunks; all.count[3 + l] = bc[l];
            all.off[3 + l] = boff[l];
            bp += (int64_t)ctx->bias_chunks * bc[l];
        }
        all.part[7] = ctx->part5;  // W5 and b5 (contiguous); the fused head writes one chunk
        all.splits[7] = fc5_fused ? 1 : (B + fc5_rows(B) - 1) / fc5_rows(B);
        all.count[7] = (int64_t)nA * (FC4_OUT + 1); all.off[7] = OFF_W5;
        for (int l = 3; l < 7; ++l) all.wide[l] = 1;
        if (ctx->u8)  // b1..b3 from the weight-gradient GEMMs' ones accumulators, one partial per CTA
            for (int l = 0; l < 3; ++l) {
                all.part[3 + l] = ctx->part_bias[l]; all.splits[3 + l] = ctx->split_w[l]; all.wide[3 + l] = 0;
            }
        all.nseg = 8;
        all.accumulate = accumulate;
        for (int l = 0; l < all.nseg; ++l) all.coop |= !all.wide[l] && all.splits[l] >= 64 ? 1 : 0;
    }
    auto pick = [&](std::initializer_list<int> segs) {
        WgradReduceParams p{};
        for (int l : segs) {
            p.part[p.nseg] = all.part[l]; p.splits[p.nseg] = all.splits[l]; p.count[p.nseg] = all.count[l];
            p.off[p.nseg] = all.off[l]; p.wide[p.nseg] = all.wide[l];
            ++p.nseg;
        }
        p.accumulate = all.accumulate;
        for (int l = 0; l < p.nseg; ++l) p.coop |= !p.wide[l] && p.splits[l] >= 64 ? 1 : 0;
        return p;
    };
    static const bool split_red = [] {  // GORILA_SPLIT_REDUCE=0: one K10 after the join
        const char* e = getenv("GORILA_SPLIT_REDUCE");
        return !(e && atoi(e) == 0);
    }();
    // grid of a K10 launch: one block per 32 [split][element] elements, one warp per wide element
    auto red_grid = [](const WgradReduceParams& q) {
        int64_t tot = 0, totw = 0;
        for (int l = 0; l < q.nseg; ++l) (q.wide[l] ? totw : tot) += q.count[l];
        if (!q.coop) return 148 * 2;  // a thread per element
        return (int)std::min<int64_t>(4096, std::max<int64_t>({148, (tot + 31) / 32, (totw + 7) / 8}));
    };
    // u8 path, forked round: b4's partials right after fc4's weight gradient and the side stream's
    // reduction right after conv2's weight gradient (neither waits for g1), so both run under the
    // main stream's conv2 data gradient / conv1 weight gradient
    const bool early_side = fk && ctx->u8 && split_red;
    // small batches, one GPU: the conv3 / conv2 weight gradients run on side2 as soon as g3 / g2
    // exist (instead of queueing behind fc4's weight gradient on side), the bias partials on side
    // after fc4's; no side reduction: one K10 on the main stream after both joins
    // (GORILA_SIDE2=0: everything on side)
    static const bool side2_env = [] {
        const char* e = getenv("GORILA_SIDE2");
        return !(e && atoi(e) == 0);
    }();
    // (not in asynchronous mode: side2 then hosts the persistent shard server)
    // (several ranks: only without the opt-in early exchange, which also uses side2)
    const bool on2 = fk && !ctx->u8 && (ctx->W == 1 || ctx->early_learner < 0) && !ctx->async_mode && side2_env &&
                     ctx->side2 != nullptr;
    // on2, first learner: conv1's weight gradient reduced in-cluster straight into G and fc5's
    // partials reduced by the side stream, so no reduction kernel is left on the main path
    static const bool c1d_env = [] {  // B = 32: 65.0 vs 65.3 us per step (GORILA_C1_DIRECT=0: off)
        const char* e = getenv("GORILA_C1_DIRECT");
        return !(e && atoi(e) == 0);
    }();
    // (aggregate mode only: the in-cluster order of the sum differs from K10's, and the per-message
    // mode must stay bitwise equal to the asynchronous one, which does not fork)
    const bool c1_direct = on2 && split_red && accumulate == 0 && !fp32v && !ctx->per_msg && c1d_env &&
                           cluster_env_on();
    PHASE(PH_FC4WG) {
    // fc4 wgrad (i = k, j = n, red = b): G[W4][n][k] += sum_b a3[b][k] g4[b][n]
    {
        OnSide on_side(ctx, fk);
        if constexpr (fp32v) {
            using LA = LdRowsMN<T>; using LB = LdRowsMN<T>; using EP = EpAddT;
            GemmProb<LA, LB, EP> pr[1] = {{{a3, FC4_IN, FC4_IN, B}, {g4, FC4_OUT, FC4_OUT, B},
                                           {Gd + OFF_W4, FC4_IN, FC4_IN, FC4_OUT, accumulate}}};
            gemm<T, 64>(ctx, pr, 1, FC4_IN, FC4_OUT, B, 1);
        } else {
            using OA = OpMatMNS<128>; using OB = OpMatMNS<64>; using EP = EpAddT;
            TmaProb<OA, OB, EP> pr[1];
            pr[0].a = op_matmns<128>(ctx, a3, B, FC4_IN, FC4_IN);
            pr[0].b = op_matmns<64>(ctx, g4, B, FC4_OUT, FC4_OUT);
            pr[0].ep = {Gd + OFF_W4, FC4_IN, FC4_IN, FC4_OUT, accumulate};
            // small batches: this GEMM runs on the side stream beside the dgrad chain, so fewer,
            // longer CTAs leave that chain its SMs (B = 32, 200 tiles: 60 CTAs 69.6-69.7 us per step,
            // 80: 70.2-70.5, 148 x 2: 71.5; 20 / 50: 71.9 / 72.1; GORILA_FC4WG_GRID overrides, 0 = uncapped)
            static const int fc4wg_env = [] {
                const char* e = getenv("GORILA_FC4WG_GRID");
                return e ? atoi(e) : -1;
            }();
            const int fc4wg_grid = fc4wg_env >= 0 ? fc4wg_env : (2 * B <= ctx->num_sms ? 60 : 0);
            if (fc4wg_grid > 0)
                gemm_tma_p_launch<64, 1>(ctx, pr, 1, (FC4_IN + 127) / 128, FC4_OUT / 64, (B + 63) / 64, 1, FC4_OUT, fc4wg_grid);
            else
                gemm_tma_launch<64, 1>(ctx, pr, 1, (FC4_IN + 127) / 128, FC4_OUT / 64, (B + 63) / 64, 1, 0, FC4_OUT);
        }
    }
    }
    mark(ctx, PH_FC4WG);
    if (fk && j == ctx->early_learner) {  // this rank's fc4 weight gradient is complete on the side stream
        cudaStream_t m = ctx->stream;
        ctx->stream = ctx->side;
        early_apply_p2p(ctx, round);
        ctx->stream = m;
    }
    if (early_side) {
        OnSide on_side(ctx, true);
        launch(ctx, k_bias_partial<T>, dim3(ctx->bias_chunks, 1), dim3(256), 0, (const T*)g1, (const T*)g2,
               (const T*)g3, (const T*)g4, B, ctx->part_b, ctx->bias_chunks, 3);
    }
    if (fk) fork_side(ctx, 1);  // g3 ready (fc4 dgrad is on the main stream before this point)
    if (on2) cudaStreamWaitEvent(ctx->side2, ctx->ev_fork[1], 0);
    PHASE(PH_CONV3DG) {
    // conv3 dgrad: g2 = mask(conv3^T(g3))
    {
        const int M = B * H2 * H2;
        if constexpr (fp32v) {
            using LA = LdDgrad<T, Conv3>; using LB = LdWdgradMN<T, Conv3>; using EP = EpMask<T>;
            GemmProb<LA, LB, EP> pr[1] = {{{g3, M}, {rt + RL.w3}, {g2, a2, C2_OUT, M, C2_OUT}}};
            gemm<T, 64>(ctx, pr, 1, M, C2_OUT, K3, 1, 148);
        } else if ((ctx->shift & 8) && (ctx->shift & 2) && ctx->u8) {  // as below, decisions as bits (conv2 fwd)
            using OA = ShDgrad3; using OB = ShWeightDgrad<Conv3, false>; using EP = EpMaskBits<T>;
            ShiftProb<OA, OB, EP> pr[1];
            pr[0].a.map = sh_grad_map<Conv3>(ctx, g3, B);
            pr[0].a.batch = B;
            pr[0].b.map = wdgrad_map_sw<Conv3>(ctx, rt + RL.w3);
            pr[0].ep = {g2, ctx->mbits2, C2_OUT, M, C2_OUT, 2};
            gemm_shift_launch<64, 1>(ctx, pr, 1, C2_OUT);
        } else if (ctx->shift & 8) {  // shifted windows over the zero-padded g3 of each sample
            using OA = ShDgrad3; using OB = ShWeightDgrad<Conv3, false>; using EP = EpMask<T>;
            ShiftProb<OA, OB, EP> pr[1];
            pr[0].a.map = sh_grad_map<Conv3>(ctx, g3, B);
            pr[0].a.batch = B;
            pr[0].b.map = wdgrad_map_sw<Conv3>(ctx, rt + RL.w3);
            pr[0].ep = {g2, a2, C2_OUT, M, C2_OUT};
            gemm_shift_launch<64, 1>(ctx, pr, 1, C2_OUT);
        } else {  // TMA: one sample (81 input pixels) per tile, shifted boxes with zero fill
            using OA = OpDgradS<Conv3, 1>; using OB = OpWdgradMNS<Conv3>; using EP = EpMask<T>;
            TmaProb<OA, OB, EP> pr[1];
            pr[0].a.map = grad_map_sw<Conv3>(ctx, g3, B, H2, H2, 1);
            pr[0].a.nb = 1;
            pr[0].a.batch = B;
            pr[0].a.phase = -1;
            pr[0].b.map = wdgrad_map_sw<Conv3>(ctx, rt + RL.w3);
            pr[0].b.phase = -1;
            pr[0].ep = {g2, a2, C2_OUT, M, C2_OUT};
            gemm_tma_launch<64, 1>(ctx, pr, 1, B, 1, C3_K * C3_K, 1, 0, C2_OUT);
        }
    }
    }
    mark(ctx, PH_CONV3DG);
    PHASE(PH_CONV3WG) {
    // conv3 wgrad (i = r, j = o, red = m): partial[s][o][r]
    {
        OnSide on_side(ctx, fk && !on2);
        std::unique_ptr<OnSide2> on_side2(on2 ? new OnSide2(ctx) : nullptr);
        const int Mred = B * H3 * H3;
        if constexpr (fp32v) {
            using LA = LdConvInMN<T, Conv3>; using LB = LdRowsMN<T>; using EP = EpStoreT;
            GemmProb<LA, LB, EP> pr[1] = {{{a2, Mred}, {g3, C3_OUT, C3_OUT, Mred},
                                           {ctx->part_w[2], K3, (int64_t)C3_OUT * K3, 1.f, K3, C3_OUT}}};
            gemm<T, 64>(ctx, pr, 1, K3, C3_OUT, Mred, ctx->split_w[2]);
        } else if (ctx->u8) {  // shifted windows: every tap a start row of a2 (k_wgrad_shift)
            WgradShiftParams wp;
            {
                const uint64_t dims[3] = {64, 81, (uint64_t)B}, str[2] = {128, 81 * 128};
                const uint32_t box[3] = {64, 81, 1};
                wp.a_map = tmap(ctx, a2, 3, dims, str, box, nullptr, 128);
            }
            {
                const uint64_t dims[4] = {64, 7, 7, (uint64_t)B}, str[3] = {128, 7 * 128, 49 * 128};
                const uint32_t box[4] = {64, 9, 9, 1};
                wp.g_map = tmap(ctx, g3, 4, dims, str, box, nullptr, 128);
            }
            wp.part = ctx->part_w[2];
            wp.part_b = ctx->part_bias[2];
            wp.batch = B;
            wgrad_shift_launch<WgConv3>(ctx, wp, ctx->split_w[2]);
        } else {  // TMA: K-chunk = one sample's 49 pixels (64 rows, zero tail in the gradient operand)
            using OA = OpWgradInS<Conv3, 64>; using OB = OpWgradOutS<64, 64, false>; using EP = EpStoreT;
            TmaProb<OA, OB, EP> pr[1];
            pr[0].a.map = fwd_map_sw<Conv3>(ctx, a2, B, 1);
            pr[0].b = op_wgout_s<64, 64, false>(ctx, g3, H3 * H3, B);
            pr[0].ep = {ctx->part_w[2], K3, (int64_t)C3_OUT * K3, 1.f, K3, C3_OUT};
            gemm_tma_launch<64, 1>(ctx, pr, 1, (K3 + 127) / 128, 1, B, ctx->split_w[2], 0, C3_OUT);
        }
    }
    }
    mark(ctx, PH_CONV3WG);
    if (fk) fork_side(ctx, 2);  // g2 ready
    if (on2) cudaStreamWaitEvent(ctx->side2, ctx->ev_fork[2], 0);
    PHASE(PH_CONV2DG) {
    // conv2 dgrad: g1 = mask(conv2^T(g2))
    {
        const int M = B * H1 * H1;
        if constexpr (fp32v) {
            using LA = LdDgrad<T, Conv2>; using LB = LdWdgradMN<T, Conv2>; using EP = EpMask<T>;
            GemmProb<LA, LB, EP> pr[1] = {{{g2, M}, {rt + RL.w2}, {g1, a1, C1_OUT, M, C1_OUT}}};
            gemm<T, 32>(ctx, pr, 1, M, C1_OUT, Conv2::RD, 1, 296);
        } else if (ctx->shift & 16) {  // the four output phases as M-blocks over one padded g2 per sample
#define SH_D2(MS_, MB_)                                                                                        \
    {                                                                                                          \
        using OA = ShDgrad2<MS_>; using OB = ShWeightDgrad<Conv2, true>; using EP = EpMask<T>;                 \
        ShiftProb<OA, OB, EP> pr[1];                                                                           \
        pr[0].a.map = sh_grad_map<Conv2>(ctx, g2, B);                                                          \
        pr[0].a.batch = B;                                                                                     \
        pr[0].b.map = wdgrad_map_sw<Conv2>(ctx, rt + RL.w2);                                                   \
        pr[0].ep = {g1, a1, C1_OUT, M, C1_OUT};                                                                \
        gemm_shift_launch<32, MB_>(ctx, pr, 1, C1_OUT);                                                        \
    }
#define SH_D2B(MS_, MB_)                                                                                       \
    {                                                                                                          \
        using OA = ShDgrad2<MS_>; using OB = ShWeightDgrad<Conv2, true>; using EP = EpMaskBits<T>;             \
        ShiftProb<OA, OB, EP> pr[1];                                                                           \
        pr[0].a.map = sh_grad_map<Conv2>(ctx, g2, B);                                                          \
        pr[0].a.batch = B;                                                                                     \
        pr[0].b.map = wdgrad_map_sw<Conv2>(ctx, rt + RL.w2);                                                   \
        pr[0].ep = {g1, ctx->mbits1, C1_OUT, M, C1_OUT, 1};                                                    \
        gemm_shift_launch<32, MB_>(ctx, pr, 1, C1_OUT);                                                        \
    }
            if (ctx->u8) {  // the ReLU decisions as bits (conv1's forward stored them)
                if (B < ctx->num_sms) SH_D2B(4, 1) else SH_D2B(1, 4)
            } else if (B < ctx->num_sms) SH_D2(4, 1) else SH_D2(1, 4)  // few samples: one phase per tile
#undef SH_D2B
#undef SH_D2
        } else {  // TMA: the stride-2 transpose as 4 phase problems of 2x2 taps (no zero taps)
            using OA = OpDgradS<Conv2, 1>; using OB = OpWdgradMNS<Conv2>; using EP = EpMask<T>;
            TmaProb<OA, OB, EP> pr[4];
            for (int ph = 0; ph < 4; ++ph) {
                pr[ph].a.map = grad_map_sw<Conv2>(ctx, g2, B, 10, 10, 1);
                pr[ph].a.nb = 1;
                pr[ph].a.batch = B;
                pr[ph].a.phase = ph;
                pr[ph].b.map = wdgrad_map_sw<Conv2>(ctx, rt + RL.w2);
                pr[ph].b.phase = ph;
                pr[ph].ep = {g1, a1, C1_OUT, M, C1_OUT};
            }
            gemm_tma_launch<32, 1>(ctx, pr, 4, B, 1, 4, 1, 0, C1_OUT);
        }
    }
    }
    mark(ctx, PH_CONV2DG);
    PHASE(PH_CONV2WG) {
    // conv2 wgrad
    {
        OnSide on_side(ctx, fk && !on2);
        std::unique_ptr<OnSide2> on_side2(on2 ? new OnSide2(ctx) : nullptr);
        const int Mred = B * H2 * H2;
        if constexpr (fp32v) {
            using LA = LdConvInMN<T, Conv2>; using LB = LdRowsMN<T>; using EP = EpStoreT;
            GemmProb<LA, LB, EP> pr[1] = {{{a1, Mred}, {g2, C2_OUT, C2_OUT, Mred},
                                           {ctx->part_w[1], K2, (int64_t)C2_OUT * K2, 1.f, K2, C2_OUT}}};
            gemm<T, 64>(ctx, pr, 1, K2, C2_OUT, Mred, ctx->split_w[1]);
        } else if (ctx->u8) {  // shifted windows over the stride phases of a1 (k_wgrad_shift)
            WgradShiftParams wp;
            wp.a_map = sh_conv2_map(ctx, a1, B);
            {
                const uint64_t dims[4] = {64, 9, 9, (uint64_t)B}, str[3] = {128, 9 * 128, 81 * 128};
                const uint32_t box[4] = {64, 10, 9, 1};
                wp.g_map = tmap(ctx, g2, 4, dims, str, box, nullptr, 128);
            }
            wp.part = ctx->part_w[1];
            wp.part_b = ctx->part_bias[1];
            wp.batch = B;
            wgrad_shift_launch<WgConv2>(ctx, wp, ctx->split_w[1]);
        } else {  // TMA: K-chunk = one sample's 81 pixels (96 rows, zero tail)
            using OA = OpWgradInS<Conv2, 96>; using OB = OpWgradOutS<64, 96, false>; using EP = EpStoreT;
            TmaProb<OA, OB, EP> pr[1];
            pr[0].a.map = fwd_map_sw<Conv2>(ctx, a1, B, 1);
            pr[0].b = op_wgout_s<64, 96, false>(ctx, g2, H2 * H2, B);
            pr[0].ep = {ctx->part_w[1], K2, (int64_t)C2_OUT * K2, 1.f, K2, C2_OUT};
            gemm_tma_launch<64, 1>(ctx, pr, 1, K2 / 128, 1, B, ctx->split_w[1], 0, C2_OUT);
        }
    }
    }
    mark(ctx, PH_CONV2WG);
    if (on2 && split_red && (phases & (1u << PH_WGRED))) {  // conv2 / conv3 weights, on side2 behind them
        OnSide2 on_side2(ctx);
        const WgradReduceParams q = pick({1, 2});
        launch(ctx, k_wgrad_reduce, dim3(red_grid(q)), dim3(256), 0, q, Gd);
    }
    if (early_side) {
        OnSide on_side(ctx, true);
        const WgradReduceParams q = pick({1, 2, 4, 5, 6});
        launch(ctx, k_wgrad_reduce, dim3(red_grid(q)), dim3(256), 0, q, Gd);
    }
    if (fk) fork_side(ctx, 3);  // g1 ready
    PHASE(PH_CONV1WG) {
    // conv1 wgrad (input scale 1/255 folded into the store)
    {
        const int Mred = B * H1 * H1;
        if constexpr (fp32v) {
            using LA = LdConvInMN<T, Conv1>; using LB = LdRowsMN<T>; using EP = EpStoreT;
            GemmProb<LA, LB, EP> pr[1] = {{{s, Mred}, {g1, C1_OUT, C1_OUT, Mred},
                                           {ctx->part_w[0], K1, (int64_t)C1_OUT * K1, in_scale, K1, C1_OUT}}};
            gemm<T, 32>(ctx, pr, 1, K1, C1_OUT, Mred, ctx->split_w[0]);
        } else if (ctx->u8) {  // shifted windows over the u8-staged s, one partial per CTA
            Conv1WgradU8 wp;
            {
                const uint64_t dims[4] = {32, 20, 20, (uint64_t)B}, str[3] = {64, 20 * 64, 400 * 64};
                const uint32_t box[4] = {32, 21, 20, 1};
                wp.g1_map = tmap(ctx, g1, 4, dims, str, box, nullptr, 64);
            }
            wp.desc = ctx->sdesc;
            wp.part = ctx->part_w[0];
            wp.part_b = ctx->part_bias[0];
            wp.scale = in_scale;
            wp.batch = B;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(k_conv1_wgrad_u8, cudaFuncAttributeMaxDynamicSharedMemorySize, c1wg::SMEM);
                attr = true;
            }
            launch(ctx, k_conv1_wgrad_u8, dim3(ctx->split_w[0]), dim3(c1wg::THREADS), c1wg::SMEM, wp);
        } else if (c1_direct) {  // the splits of a tile reduced in the cluster (DSMEM), stored into G
            using OA = OpWgradIn1S; using OB = OpWgradOutS<32, 80, true>; using EP = EpStoreT;
            TmaProb<OA, OB, EP> pr[1];
            pr[0].a.map = conv1_map_sw(ctx, s, B, 1, 4);
            pr[0].b = op_wgout_s<32, 80, true>(ctx, g1, H1 * H1, B);
            pr[0].ep = {Gd + OFF_W1, K1, 0, in_scale, K1, C1_OUT};
            gemm_tma_launch<32, 1>(ctx, pr, 1, K1 / 128, 1, B * 5, 1, 148, C1_OUT, 16);
        } else {  // TMA: K-chunk = 4 output rows (80 pixels) of one sample
            using OA = OpWgradIn1S; using OB = OpWgradOutS<32, 80, true>; using EP = EpStoreT;
            TmaProb<OA, OB, EP> pr[1];
            pr[0].a.map = conv1_map_sw(ctx, s, B, 1, 4);
            pr[0].b = op_wgout_s<32, 80, true>(ctx, g1, H1 * H1, B);
            pr[0].ep = {ctx->part_w[0], K1, (int64_t)C1_OUT * K1, in_scale, K1, C1_OUT};
            gemm_tma_launch<32, 1>(ctx, pr, 1, K1 / 128, 1, B * 5, ctx->split_w[0], 0, C1_OUT);
        }
    }
    }
    mark(ctx, PH_CONV1WG);
    PHASE(PH_BIASG) if (!early_side) {
    // bias gradients b1..b4 (coalesced partials; reduced by K10)
    OnSide on_side(ctx, fk);
    const int l0 = ctx->u8 ? 3 : 0;  // u8 path: only b4 here (b1..b3 came with the weight gradients)
    launch(ctx, k_bias_partial<T>, dim3(ctx->bias_chunks, 4 - l0), dim3(256), 0, (const T*)g1, (const T*)g2,
           (const T*)g3, (const T*)g4, B, ctx->part_b, ctx->bias_chunks, l0);
    // forked round: the side stream reduces what it produced (conv2 / conv3 weights, the biases)
    // while the main stream finishes conv1's weight gradient
    if (split_red && fk && (phases & (1u << PH_WGRED))) {
        // on2: the side stream reduces only the biases (side2 reduced conv2 / conv3's weights)
        const WgradReduceParams q = c1_direct ? pick({3, 4, 5, 6, 7}) : on2 ? pick({3, 4, 5, 6}) : pick({1, 2, 3, 4, 5, 6});
        launch(ctx, k_wgrad_reduce, dim3(red_grid(q)), dim3(256), 0, q, Gd);
    }
    }
    mark(ctx, PH_BIASG);
    // on2: the main reduction (conv1's weight, fc5) runs before the joins, beside the other two
    auto main_reduce = [&]() {
        PHASE(PH_WGRED) {
        // K10: fixed-order reduction of the conv wgrad partials into G (the rest of it when forked)
        // (u8 path: b1 comes from conv1's weight gradient on the main stream, so the main reduce takes it)
        const WgradReduceParams q = (fk && split_red) ? (ctx->u8 ? pick({0, 3, 7}) : pick({0, 7})) : all;
        launch(ctx, k_wgrad_reduce, dim3(red_grid(q)), dim3(256), 0, q, Gd);
        }
    };
    if (on2 && split_red && !c1_direct) main_reduce();
    if (on2) {
        cudaEventRecord(ctx->ev_join2, ctx->side2);
        cudaStreamWaitEvent(ctx->stream, ctx->ev_join2, 0);
    }
    if (fk) join_side(ctx);
    if (!(on2 && split_red)) main_reduce();
    mark(ctx, PH_WGRED);
    CU(cudaGetLastError());
    return GORILA_OK;
#undef PHASE
}

template <typename T>
gorila_status pack_replica(gorila_ctx* ctx, const float* theta, void* rt, float* rf, const uint8_t* pred,
                           uint64_t* vhist_dst) {
    launch(ctx, k_pack<T>, dim3(148 * 4), dim3(256), 0, theta, ctx->nA, P_<T>(rt), rf, pred, vhist_dst,
           (const uint64_t*)ctx->V);
    CU(cudaGetLastError());
    return GORILA_OK;
}

gorila_status pack_any(gorila_ctx* ctx, const float* theta, void* rt, float* rf, const uint8_t* pred,
                       uint64_t* vhist_dst) {
    if (ctx->cfg.math == GORILA_MATH_FP32) return pack_replica<float>(ctx, theta, rt, rf, pred, vhist_dst);
    return pack_replica<__nv_bfloat16>(ctx, theta, rt, rf, pred, vhist_dst);
}

// ---------------------------------------------------------------- NVLink peer mappings
// Every rank maps every peer's workspace (same carve on every rank, so a peer's buffer is at the
// same offset): IPC handle of the workspace's allocation + the workspace offset inside it. The
// 128-byte records are exchanged either with one NCCL all-gather (gorila_init with an NCCL id) or by
// the caller (gorila_peer_record / gorila_peer_connect: any process group, e.g. gloo, which also
// covers several ranks sharing one GPU, where NCCL cannot form a communicator).
struct PeerRec {
    cudaIpcMemHandle_t h;
    uint64_t off;
    int32_t ok, dev;
    uint8_t pad[128 - sizeof(cudaIpcMemHandle_t) - 16];
};
static_assert(sizeof(PeerRec) == 128, "record size");

void peer_record(gorila_ctx* ctx, PeerRec* mine) {
    typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<GetRange>(f);
    }();
    memset(mine, 0, sizeof(*mine));
    ctx->ws_local = (uint8_t*)ctx->cfg.workspace;
    CUdeviceptr base = 0;
    size_t size = 0;
    mine->ok = get_range && get_range(&base, &size, (CUdeviceptr)ctx->ws_local) == CUDA_SUCCESS &&
               cudaIpcGetMemHandle(&mine->h, (void*)base) == cudaSuccess;
    cudaGetLastError();
    mine->off = (uint64_t)((CUdeviceptr)ctx->ws_local - base);
    cudaGetDevice(&mine->dev);
}

void peer_close(gorila_ctx* ctx) {
    for (int q = 0; q < MAX_W; ++q)
        if (ctx->peer_raw[q]) {
            cudaIpcCloseMemHandle(ctx->peer_raw[q]);
            ctx->peer_raw[q] = nullptr;
            ctx->peer_ws[q] = nullptr;
        }
    cudaGetLastError();
}

// open every peer's record (all: W records in rank order); false (nothing left open) on any failure
bool peer_open(gorila_ctx* ctx, const PeerRec* all) {
    const int W = ctx->W, r = ctx->rank;
    bool ok = true;
    for (int q = 0; q < W; ++q) ok = ok && all[q].ok;
    for (int q = 0; q < W && ok; ++q) {
        if (q == r) continue;
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, all[q].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
            break;
        }
        ctx->peer_raw[q] = p;
        ctx->peer_ws[q] = (uint8_t*)p + all[q].off;
    }
    if (!ok) peer_close(ctx);
    return ok;
}

// NCCL bootstrap: records all-gathered on the library's communicator, the verdict all-reduced (min)
bool p2p_setup(gorila_ctx* ctx) {
    const int W = ctx->W, r = ctx->rank;
    PeerRec mine;
    peer_record(ctx, &mine);
    uint8_t* dbuf = reinterpret_cast<uint8_t*>(ctx->tmp_int);  // scratch: [W][128 B] records
    if (cudaMemcpyAsync(dbuf + (size_t)r * 128, &mine, 128, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        ncclAllGather(dbuf + (size_t)r * 128, dbuf, 128, ncclChar, ctx->comm, ctx->stream) != ncclSuccess)
        return false;
    std::vector<PeerRec> all(W);
    if (cudaMemcpyAsync(all.data(), dbuf, (size_t)W * 128, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
        return false;
    const bool ok = peer_open(ctx, all.data());
    int32_t* vb = reinterpret_cast<int32_t*>(dbuf);
    const int32_t v = ok ? 1 : 0;
    if (cudaMemcpyAsync(vb, &v, 4, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
        ncclAllReduce(vb, vb, 1, ncclInt32, ncclMin, ctx->comm, ctx->stream) != ncclSuccess)
        return false;
    int32_t all_ok = 0;
    cudaMemcpyAsync(&all_ok, vb, 4, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (!all_ok) peer_close(ctx);
    return all_ok != 0;
}
// rank q's copy of a workspace pointer
template <typename P>
P* peer_ptr(gorila_ctx* ctx, int q, P* local) {
    if (q == ctx->rank) return local;
    return reinterpret_cast<P*>(ctx->peer_ws[q] + ((uint8_t*)local - ctx->ws_local));
}

// the u8 staging of s / s' (large-batch bf16, conv1 on the shifted-window path)
bool u8_staging(const gorila_config* cfg) {
    static const bool off = [] {
        const char* e = getenv("GORILA_U8");
        return e && atoi(e) == 0;
    }();
    static const int shift = [] {
        const char* e = getenv("GORILA_SHIFT");
        return e ? atoi(e) : 31;
    }();
    return !off && (shift & 1) && cfg->math != GORILA_MATH_FP32 && 2 * cfg->batch > 148;
}

uint64_t layout_bytes(const gorila_config* cfg, gorila_ctx* ctx, uint8_t* base) {
    // computes the carve; if ctx != nullptr and base != nullptr fills the pointers
    const int nA = cfg->n_actions, B = cfg->batch, L = cfg->n_learners_local, W = cfg->world;
    const int64_t P = param_count(nA);
    const int64_t q = round_up((P + W - 1) / W, 64);
    const size_t esz = cfg->math == GORILA_MATH_FP32 ? 4 : 2;
    const ReplicaLayout rl = replica_layout(nA);
    const int H = std::max(1, cfg->history);
    const bool fp32 = cfg->math == GORILA_MATH_FP32;
    Carver c{base};
    float* theta = c.take<float>(W * q);
    float* m = c.take<float>(q);
    float* v = c.take<float>(q);
    float* G = c.take<float>((cfg->ps_mode >= 1 ? L : 1) * W * q);  // per-message / async: one per learner
    float* counts = c.take<float>(W + 64);
    uint64_t* V = c.take<uint64_t>(4);
    uint64_t* rinfo = c.take<uint64_t>(4);
    uint32_t* nacc = c.take<uint32_t>(4);
    uint64_t* Vhist = c.take<uint64_t>(H);
    uint64_t* dev_round = c.take<uint64_t>(1);
    unsigned int* head_counter = c.take<unsigned int>(1);
    uint64_t* pflags = c.take<uint64_t>(FLAG_WORDS);
    uint64_t* p2p_epoch = c.take<uint64_t>(1);
    unsigned int* p2p_counter = c.take<unsigned int>(2);
    unsigned int* apply_counter = c.take<unsigned int>(1);
    unsigned int* fc5_gen = c.take<unsigned int>(2);
    std::vector<void*> rep_t(H);
    std::vector<float*> rep_f(H);
    for (int h = 0; h < H; ++h) {
        rep_t[h] = c.take<uint8_t>(rl.n_t * esz);
        rep_f[h] = c.take<float>(rl.n_f);
    }
    std::vector<Learner> lrs(L);
    for (int j = 0; j < L; ++j) {
        Learner& l = lrs[j];
        l.frames = c.take<uint8_t>(cfg->replay_capacity * FRAME_BYTES);
        l.a = c.take<uint8_t>(cfg->replay_capacity);
        l.r = c.take<float>(cfg->replay_capacity);
        l.d = c.take<uint8_t>(cfg->replay_capacity);
        l.n_dev = c.take<uint64_t>(1);
        l.tminus_t = c.take<uint8_t>(rl.n_t * esz);
        l.tminus_f = c.take<float>(rl.n_f);
        l.stats = c.take<LearnerStats>(1);
        l.info = c.take<DevLearnerInfo>(1);
        l.Q = c.take<float>((int64_t)B * nA);
        l.Qhat = c.take<float>((int64_t)B * nA);
        l.sync_flag = c.take<uint8_t>(1);
    }
    const int64_t Bs = B;
    void* s = c.take<uint8_t>(Bs * FRAME_BYTES * NSTACK * esz);
    void* s2 = c.take<uint8_t>(Bs * FRAME_BYTES * NSTACK * esz);
    void* a1 = c.take<uint8_t>(Bs * A1 * esz);
    void* a2 = c.take<uint8_t>(Bs * A2 * esz);
    void* a3 = c.take<uint8_t>(Bs * A3 * esz);
    float* a4 = c.take<float>(Bs * A4);
    void* t1 = c.take<uint8_t>(Bs * A1 * esz);
    void* t2 = c.take<uint8_t>(Bs * A2 * esz);
    void* t3 = c.take<uint8_t>(Bs * A3 * esz);
    float* t4 = c.take<float>(Bs * A4);
    void* g1 = c.take<uint8_t>(Bs * A1 * esz);
    void* g2 = c.take<uint8_t>(Bs * A2 * esz);
    void* g3 = c.take<uint8_t>(Bs * A3 * esz);
    void* g4 = c.take<uint8_t>(Bs * A4 * esz);
    uint32_t* mbits1 = c.take<uint32_t>(u8_staging(cfg) ? Bs * H1 * H1 : 0);
    uint32_t* mbits2 = c.take<uint32_t>(u8_staging(cfg) ? Bs * H2 * H2 * 2 : 0);
    uint32_t* mbits3 = c.take<uint32_t>(u8_staging(cfg) ? Bs * H3 * H3 * 2 : 0);
    SampleDesc* sdesc = c.take<SampleDesc>(Bs);
    uint8_t* sa = c.take<uint8_t>(Bs);
    uint8_t* sd = c.take<uint8_t>(Bs);
    float* sr = c.take<float>(Bs);
    int64_t* sidx = c.take<int64_t>(Bs);
    int32_t* sshard = c.take<int32_t>(Bs);
    ShardPtrs* shard_tab = c.take<ShardPtrs>((int64_t)W * L);
    uint64_t* rflags = c.take<uint64_t>(MAX_W);
    uint64_t* replay_epoch = c.take<uint64_t>(1);
    uint64_t* n_snap = c.take<uint64_t>((int64_t)W * L);
    float* dQ = c.take<float>(Bs * nA);
    float* td_partial = c.take<float>(Bs * 2);
    static const int bias_min = [] {
        const char* e = getenv("GORILA_BIAS_CHUNKS");
        return e ? std::max(1, atoi(e)) : 64;
    }();
    const int bias_chunks = std::max(bias_min, std::min(2048, 2 * B));
    // split choices (reduction chunks of 64 for tc, 16 for simt)
    const int chunk = fp32 ? SM_BR : TC_BK;
    int split_w[3];
    const int Mred[3] = {B * H1 * H1, B * H2 * H2, B * H3 * H3};
    const int64_t wcount[3] = {(int64_t)C1_OUT * K1, (int64_t)C2_OUT * K2, (int64_t)C3_OUT * K3};
    const int tiles[3] = {fp32 ? 4 * 1 : 2, fp32 ? 8 : 4, fp32 ? 9 : 5};
    float* part_w[3];
    for (int l = 0; l < 3; ++l) {
        if (fp32) {
            int want = pick_splits((Mred[l] + chunk - 1) / chunk, tiles[l], 148, 128);
            split_w[l] = eff_splits(fp32, Mred[l], want);
        } else {  // TMA engine: chunks are 80-pixel rows (conv1) or whole samples (conv2, conv3)
            const int nch = l == 0 ? 5 * B : B, ta = l == 0 ? 2 : l == 1 ? 4 : 5;
            // partials per weight (the critical-path reduce reads them all); conv1's weight gradient
            // is itself on the critical path (the last GEMM of the dgrad chain): it keeps more splits
            static const int cap23_env = [] {  // B = 32 sweep (tools/knob_sweep2.sh): 4: 76.9, 6: 76.9,
                const char* e = getenv("GORILA_WSPLIT_MAX");  // 8: 75.7, 11: 78.5, 16: 78.5 us/step
                return e ? std::max(1, atoi(e)) : 0;
            }();
            static const int cap1_env = [] {
                const char* e = getenv("GORILA_WSPLIT1_MAX");
                return e ? std::max(1, atoi(e)) : 0;
            }();
            // B = 256 sweep (r02): conv1 37 / conv2-3 16 splits: 162.9 us/step vs 173.7 with 16 / 8;
            // no change at B = 128
            const int cap1 = cap1_env ? cap1_env : (B <= 128 ? 16 : 37);
            const int cap23 = cap23_env ? cap23_env : (B <= 128 ? 8 : 16);
            const int cap = l == 0 ? cap1 : cap23;
            // small batches: the weight-gradient GEMMs run beside the dgrad chain and can afford
            // fewer, longer splits; large batches need every SM on them
            const int lim = B <= 256 ? std::min(nch, cap) : nch;
            const int want = std::max(1, std::min(lim, (148 + ta - 1) / ta));
            const int cps = (nch + want - 1) / want;
            split_w[l] = (nch + cps - 1) / cps;
            // k_conv1_wgrad_u8 / k_wgrad_shift: one partial per CTA. conv2 / conv3 (144 / 128 KB of
            // partials per CTA) balance the kernel (samples per CTA x ~0.6-0.9 us) against the
            // reduction's partial traffic: about sqrt(25 B) CTAs below B = 876
            if (u8_staging(cfg))
                split_w[l] = l == 0 ? std::min(148, B)
                                    : std::min(148, std::max(1, (int)std::lround(std::sqrt(25.0 * B))));
        }
        part_w[l] = c.take<float>((int64_t)split_w[l] * wcount[l]);
    }
    float* part_b = c.take<float>((int64_t)bias_chunks * (C1_OUT + C2_OUT + C3_OUT + FC4_OUT));
    float* part_bias[3];
    {
        const int bc[3] = {C1_OUT, C2_OUT, C3_OUT};
        for (int l = 0; l < 3; ++l) part_bias[l] = c.take<float>(u8_staging(cfg) ? (int64_t)split_w[l] * bc[l] : 0);
    }
    float* part5 = c.take<float>((int64_t)((B + fc5_rows(B) - 1) / fc5_rows(B)) * nA * (FC4_OUT + 1));
    float* tmp_canon = c.take<float>(P);
    float* tmp_int = c.take<float>(W * q);
    AsyncState* ast = c.take<AsyncState>(1);  // f2 queue / counters (small; carved in every mode)
    if (ctx) {
        ctx->nA = nA; ctx->B = B; ctx->L = L; ctx->W = W; ctx->P = P; ctx->q = q; ctx->esz = esz;
        ctx->u8 = u8_staging(cfg);
        ctx->rl = rl; ctx->H = H;
        ctx->theta = theta; ctx->m = m; ctx->v = v; ctx->G = G; ctx->counts = counts; ctx->V = V;
        ctx->G_all = G; ctx->per_msg = cfg->ps_mode >= 1; ctx->async_mode = cfg->ps_mode == 2;
        ctx->ast = ast;
        ctx->round_info = rinfo;
        ctx->n_acc_local = nacc; ctx->Vhist = Vhist; ctx->dev_round = dev_round; ctx->head_counter = head_counter;
        ctx->pflags = pflags; ctx->p2p_epoch = p2p_epoch; ctx->p2p_counter = p2p_counter;
        ctx->apply_counter = apply_counter;
        ctx->fc5_gen = fc5_gen; ctx->rep_t = rep_t; ctx->rep_f = rep_f; ctx->learners = lrs;
        ctx->s = s; ctx->s2 = s2; ctx->a1 = a1; ctx->a2 = a2; ctx->a3 = a3; ctx->a4 = a4;
        ctx->t1 = t1; ctx->t2 = t2; ctx->t3 = t3; ctx->t4 = t4;
        ctx->g1 = g1; ctx->g2 = g2; ctx->g3 = g3; ctx->g4 = g4;
        ctx->mbits1 = mbits1; ctx->mbits2 = mbits2; ctx->mbits3 = mbits3; ctx->sdesc = sdesc;
        ctx->sa = sa; ctx->sd = sd; ctx->sr = sr; ctx->sidx = sidx; ctx->dQ = dQ;
        ctx->sshard = sshard; ctx->shard_tab = shard_tab; ctx->rflags = rflags; ctx->replay_epoch = replay_epoch;
        ctx->n_snap = n_snap;
        ctx->n_shards = W * L; ctx->replay_global = cfg->replay_mode == 1;
        ctx->td_partial = td_partial; ctx->bias_chunks = bias_chunks;
        for (int l = 0; l < 3; ++l) { ctx->part_w[l] = part_w[l]; ctx->split_w[l] = split_w[l]; }
        ctx->part_b = part_b;
        for (int l = 0; l < 3; ++l) ctx->part_bias[l] = part_bias[l];
        ctx->part5 = part5;
        ctx->tmp_canon = tmp_canon; ctx->tmp_int = tmp_int;
    }
    return c.off + 256;
}

gorila_status check_learner(gorila_ctx* ctx, int32_t j) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned by an earlier CUDA/NCCL error");
    if (j < 0 || j >= ctx->L) return fail(GORILA_E_RANGE, "learner id out of range");
    return GORILA_OK;
}

}  // namespace

// ==================================================================== C-ABI
extern "C" {

int64_t gorila_param_count(int32_t n_actions) { return param_count(n_actions); }

const char* gorila_last_error(void) { return g_last_error.c_str(); }

uint64_t gorila_workspace_bytes(const gorila_config* cfg) {
    if (!cfg) return 0;
    return layout_bytes(cfg, nullptr, nullptr);
}

uint64_t gorila_kernel_launches(gorila_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t gorila_profile_phase_count(void) { return PH_COUNT; }

const char* gorila_profile_phase_name(int32_t i) { return (i >= 0 && i < PH_COUNT) ? kPhaseNames[i] : ""; }

gorila_status gorila_profile_enable(gorila_ctx* ctx, int32_t enable) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    ctx->prof = enable != 0;
    return GORILA_OK;
}

gorila_status gorila_profile_read(gorila_ctx* ctx, double* ms, int32_t n, uint64_t* n_steps) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    CU(cudaStreamSynchronize(ctx->stream));
    std::vector<std::pair<int, cudaEvent_t>> m;
    for (auto& mk : ctx->marks) m.push_back({mk.first, ctx->ev_pool[mk.second]});
    CU(fold_marks(ctx, m));
    ctx->marks.clear();
    ctx->ev_used = 0;
    for (int i = 0; i < n && i < PH_COUNT; ++i) ms[i] = ctx->prof_ms[i];
    if (n_steps) *n_steps = ctx->prof_steps;
    for (double& x : ctx->prof_ms) x = 0.0;
    ctx->prof_steps = 0;
    return GORILA_OK;
}

gorila_status gorila_bench_phase(gorila_ctx* ctx, int32_t learner, int32_t phase, int32_t iters,
                                double* us_per_iter) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    if (phase < 0 || phase >= PH_COUNT || iters < 1 || !us_per_iter) return fail(GORILA_E_INVALID, "bad argument");
    cudaStream_t st = ctx->stream;
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    const bool prof = ctx->prof;
    ctx->prof = false;
    CU(cudaEventRecord(e0, st));
    for (int it = 0; it < iters && s == GORILA_OK; ++it) {
        if (phase == PH_APPLY || phase == PH_RS || phase == PH_AG || phase == PH_PACK) {
            s = ps_apply_shard(ctx, ctx->dev_round_expect - 1, nullptr);
        } else if (phase == PH_SYNC) {
            s = sync_target(ctx, &learner, 1, 0, nullptr);
        } else {
            s = ctx->cfg.math == GORILA_MATH_FP32
                    ? run_learner<float>(ctx, learner, 0, 0, 0, 1u << phase)
                    : run_learner<__nv_bfloat16>(ctx, learner, 0, 0, 0, 1u << phase);
        }
    }
    CU(cudaEventRecord(e1, st));
    CU(cudaEventSynchronize(e1));
    ctx->prof = prof;
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *us_per_iter = 1000.0 * ms / iters;
    return s;
}

gorila_status gorila_debug_trace(uint64_t* out64) {
#ifdef GORILA_TRACE
    cudaMemcpyFromSymbol(out64, gorila_trace_buf, sizeof(unsigned long long) * 64);
    cudaMemset(nullptr, 0, 0);
    return GORILA_OK;
#else
    (void)out64;
    return fail(GORILA_E_INVALID, "built without GORILA_TRACE");
#endif
}

gorila_status gorila_debug_trace_tiles(uint64_t* out512) {
#ifdef GORILA_TRACE
    cudaMemcpyFromSymbol(out512, gorila_trace_tiles, sizeof(unsigned long long) * 512);
    return GORILA_OK;
#else
    (void)out512;
    return fail(GORILA_E_INVALID, "built without GORILA_TRACE");
#endif
}

gorila_status gorila_nccl_unique_id(void* out128) {
    if (!out128) return fail(GORILA_E_INVALID, "null argument");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(GORILA_E_NCCL, ncclGetErrorString(r));
    memcpy(out128, &id, sizeof(id));
    return GORILA_OK;
}

static cudaError_t stage_alloc(gorila_ctx* ctx);

// f4: the shard table, every rank's rings at their address in this process (after the peer mappings)
static cudaError_t shard_table(gorila_ctx* ctx) {
    if (!ctx->replay_global) return cudaSuccess;
    std::vector<ShardPtrs> tab;
    for (int q = 0; q < ctx->W; ++q)
        for (const Learner& l : ctx->learners)
            tab.push_back({peer_ptr(ctx, q, l.frames), peer_ptr(ctx, q, l.a), peer_ptr(ctx, q, l.r),
                           peer_ptr(ctx, q, l.d), peer_ptr(ctx, q, l.n_dev)});
    cudaError_t e = cudaMemcpyAsync(ctx->shard_tab, tab.data(), sizeof(ShardPtrs) * tab.size(),
                                    cudaMemcpyHostToDevice, ctx->stream);
    return e ? e : cudaStreamSynchronize(ctx->stream);
}

// world > 1: the exchange is set up (peer mappings, or the NCCL fallback)
static bool exchange_ready(const gorila_ctx* ctx) { return ctx->W == 1 || ctx->p2p || ctx->comm; }

gorila_status gorila_peer_record(gorila_ctx* ctx, void* out128) {
    if (!ctx || !out128) return fail(GORILA_E_INVALID, "null argument");
    PeerRec r;
    peer_record(ctx, &r);
    memcpy(out128, &r, sizeof(r));
    if (!r.ok) return fail(GORILA_E_CUDA, "cannot export the workspace allocation (cudaIpcGetMemHandle)");
    return GORILA_OK;
}

gorila_status gorila_peer_connect(gorila_ctx* ctx, const void* records, int32_t world) {
    if (!ctx || !records) return fail(GORILA_E_INVALID, "null argument");
    if (ctx->W == 1) return GORILA_OK;
    if (world != ctx->W) return fail(GORILA_E_SHAPE, "records must hold world entries");
    if (ctx->comm || ctx->p2p) return fail(GORILA_E_INVALID, "peers already connected");
    if (ctx->W > MAX_W) return fail(GORILA_E_INVALID, "peer-memory exchange: world <= 8");
    if (!peer_open(ctx, reinterpret_cast<const PeerRec*>(records)))
        return fail(GORILA_E_CUDA, "cudaIpcOpenMemHandle of a peer's workspace failed");
    ctx->p2p = true;
    CU(shard_table(ctx));
    return GORILA_OK;
}

gorila_status gorila_init(const gorila_config* cfg, gorila_ctx** out) {
    if (!cfg || !out) return fail(GORILA_E_INVALID, "null argument");
    *out = nullptr;
    if (cfg->n_actions < 1 || cfg->n_actions > 32) return fail(GORILA_E_INVALID, "n_actions must be in [1, 32]");
    if (cfg->batch < 1 || cfg->batch > 4096) return fail(GORILA_E_INVALID, "batch must be in [1, 4096]");
    if (cfg->replay_capacity < 2) return fail(GORILA_E_INVALID, "replay_capacity must be >= 2");
    if (cfg->n_learners_local < 1) return fail(GORILA_E_INVALID, "n_learners_local must be >= 1");
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return fail(GORILA_E_INVALID, "bad rank/world");
    if (cfg->math != GORILA_MATH_FP32 && cfg->math != GORILA_MATH_BF16) return fail(GORILA_E_INVALID, "bad math");
    if (cfg->optimizer != GORILA_OPT_RMSPROP && cfg->optimizer != GORILA_OPT_ADAGRAD)
        return fail(GORILA_E_INVALID, "bad optimizer");
    if (cfg->history < 1 || cfg->history > 64) return fail(GORILA_E_INVALID, "history must be in [1, 64]");
    if (cfg->target_period < 1) return fail(GORILA_E_INVALID, "target_period must be >= 1");
    if (cfg->ps_mode < 0 || cfg->ps_mode > 2) return fail(GORILA_E_INVALID, "ps_mode must be 0, 1 or 2");
    if (cfg->ps_mode == 2 && cfg->replay_mode != 0)
        return fail(GORILA_E_INVALID, "asynchronous mode (ps_mode 2) runs local replay only");
    if (cfg->ps_mode == 2 && cfg->history < 2)
        return fail(GORILA_E_INVALID, "asynchronous mode (ps_mode 2) needs history >= 2 (live + fetched replica)");
    if (cfg->replay_mode != 0 && cfg->replay_mode != 1) return fail(GORILA_E_INVALID, "replay_mode must be 0 or 1");
    if (cfg->replay_mode == 1 && (cfg->learner_id_base != cfg->rank * cfg->n_learners_local ||
                                  cfg->world * cfg->n_learners_local > MAX_SHARDS))
        return fail(GORILA_E_INVALID, "global replay: learner_id_base must be rank * n_learners_local, "
                                      "at most 256 learners in total");
    if (cfg->ps_mode >= 1 && (cfg->n_learners_local > 32 || cfg->world * cfg->n_learners_local > 64))
        return fail(GORILA_E_INVALID, "per-message / asynchronous mode: at most 32 learners per rank, 64 in total");
    if (!cfg->theta0) return fail(GORILA_E_INVALID, "theta0 is required");
    if (!cfg->workspace) return fail(GORILA_E_INVALID, "workspace is required");
    if (((uintptr_t)cfg->workspace) % 256) return fail(GORILA_E_INVALID, "workspace must be 256-byte aligned");
    const uint64_t need = layout_bytes(cfg, nullptr, nullptr);
    if (cfg->workspace_bytes < need) return fail(GORILA_E_OOM, "workspace too small: need " + std::to_string(need));

    gorila_ctx* ctx = new gorila_ctx();
    struct InitGuard {  // any early return below destroys the partial context (streams, pinned buffers, comm)
        gorila_ctx* c;
        ~InitGuard() { if (c) gorila_destroy(c); }
    } guard{ctx};
    ctx->cfg = *cfg;
    ctx->cfg.theta0 = nullptr;
    ctx->cfg.nccl_unique_id = nullptr;
    ctx->stream = (cudaStream_t)cfg->stream;
    ctx->rank = cfg->rank;
    layout_bytes(cfg, ctx, (uint8_t*)cfg->workspace);
    cudaStream_t st = ctx->stream;
    // zero the PS state, gradient buffer, counters, learner state
    CU(cudaMemsetAsync(ctx->theta, 0, sizeof(float) * ctx->W * ctx->q, st));
    CU(cudaMemsetAsync(ctx->m, 0, sizeof(float) * ctx->q, st));
    CU(cudaMemsetAsync(ctx->v, 0, sizeof(float) * ctx->q, st));
    CU(cudaMemsetAsync(ctx->G, 0, sizeof(float) * ctx->W * ctx->q * (ctx->per_msg ? ctx->L : 1), st));
    CU(cudaMemsetAsync(ctx->V, 0, sizeof(uint64_t) * 4, st));
    CU(cudaMemsetAsync(ctx->n_acc_local, 0, sizeof(uint32_t) * 4, st));
    CU(cudaMemsetAsync(ctx->Vhist, 0, sizeof(uint64_t) * ctx->H, st));
    CU(cudaMemsetAsync(ctx->head_counter, 0, sizeof(unsigned int), st));
    CU(cudaMemsetAsync(ctx->dev_round, 0, sizeof(uint64_t), st));
    CU(cudaMemsetAsync(ctx->pflags, 0, sizeof(uint64_t) * FLAG_WORDS, st));
    CU(cudaMemsetAsync(ctx->p2p_epoch, 0, sizeof(uint64_t), st));
    CU(cudaMemsetAsync(ctx->p2p_counter, 0, sizeof(unsigned int) * 2, st));
    CU(cudaMemsetAsync(ctx->apply_counter, 0, sizeof(unsigned int), st));
    CU(cudaMemsetAsync(ctx->fc5_gen, 0, sizeof(unsigned int) * 2, st));
    CU(cudaMemsetAsync(ctx->rflags, 0, sizeof(uint64_t) * MAX_W, st));
    CU(cudaMemsetAsync(ctx->replay_epoch, 0, sizeof(uint64_t), st));
    ctx->dev_round_expect = 0;
    {
        // programmatic dependent launch: on for small batches (a kernel's launch and prologue overlap its
        // predecessor: the B = 32 step is a latency chain); off from B = 2048, where the early-resident
        // CTAs of the next persistent GEMM measured 1.5% slower at B = 4096 (965 vs 980 us/step; at
        // B <= 1024 it is 3-8% faster).
        // GORILA_PDL=0 / 1 forces it.
        const char* e = getenv("GORILA_PDL");
        ctx->pdl = e ? atoi(e) != 0 : cfg->batch < 2048;
        const char* tw = getenv("GORILA_TOWER");
        if (tw && atoi(tw) == 0) ctx->tower = false;
        const char* sh = getenv("GORILA_SHIFT");
        if (sh) ctx->shift = atoi(sh);
        const char* fn = getenv("GORILA_FC4_NORMAL_MIN");
        if (fn) ctx->fc4_normal_min = atoi(fn);
        const char* f = getenv("GORILA_FORK");  // GORILA_FORK=0 keeps the round on one stream
        ctx->fork = !(f && atoi(f) == 0);
    }
    {
        int dev = 0;
        CU(cudaGetDevice(&dev));
        CU(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    {  // L2 persistence window: theta, m, v, G, counters and the replica history (carved contiguously)
        const char* e = getenv("GORILA_L2_PERSIST");
        int dev = 0, maxwin = 0, maxpersist = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, dev);
        const uint8_t* lo = (const uint8_t*)ctx->theta;
        const uint8_t* hi = (const uint8_t*)(ctx->rep_f[ctx->H - 1] + ctx->rl.n_f);
        size_t bytes = std::min<size_t>((size_t)(hi - lo), (size_t)std::min(maxwin, maxpersist));
        if (e && atoi(e) != 0 && bytes > 0 &&  // opt-in: measured no gain at B = 32 (12.07k vs 12.08k)
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) == cudaSuccess) {
            ctx->l2win.base_ptr = (void*)lo;
            ctx->l2win.num_bytes = bytes;
            ctx->l2win.hitRatio = 1.0f;
            ctx->l2win.hitProp = cudaAccessPropertyPersisting;
            ctx->l2win.missProp = cudaAccessPropertyStreaming;
            ctx->l2_on = true;
        }
        cudaGetLastError();
    }
    CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&ctx->ev_s2_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->ev_s2_join, cudaEventDisableTiming));
    for (auto& e : ctx->ev_fork) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->ev_join2, cudaEventDisableTiming));
    for (auto& l : ctx->learners) {
        CU(cudaMemsetAsync(l.n_dev, 0, sizeof(uint64_t), st));
        CU(cudaMemsetAsync(l.stats, 0, sizeof(LearnerStats), st));
        CU(cudaMemsetAsync(l.info, 0, sizeof(DevLearnerInfo), st));
        CU(cudaMemsetAsync(l.d, 0, cfg->replay_capacity, st));
    }
    // theta^+ = theta0 (canonical -> internal sliced)
    CU(cudaMemcpyAsync(ctx->tmp_canon, cfg->theta0, sizeof(float) * ctx->P, cudaMemcpyHostToDevice, st));
    k_convert<<<148 * 4, 256, 0, st>>>(ctx->tmp_canon, ctx->theta, ctx->P, 0);
    ctx->launches++;
    // replica slot 0 and every learner's theta^- (Alg.1 P:113 theta^- = theta)
    gorila_status s;
    if ((s = pack_any(ctx, ctx->theta, ctx->rep_t[0], ctx->rep_f[0], nullptr, ctx->Vhist)) != GORILA_OK) return s;
    for (auto& l : ctx->learners)
        if ((s = pack_any(ctx, ctx->theta, l.tminus_t, l.tminus_f, nullptr, nullptr)) != GORILA_OK) return s;
    if (cfg->world > 1 && cfg->world > MAX_W && (!cfg->nccl_unique_id || ctx->per_msg || ctx->replay_global))
        return fail(GORILA_E_INVALID, "world > 8 runs only the NCCL aggregate exchange (needs nccl_unique_id)");
    if (cfg->world > 1 && cfg->nccl_unique_id) {
        ncclUniqueId id;
        memcpy(&id, cfg->nccl_unique_id, sizeof(id));
        NC(ncclCommInitRank(&ctx->comm, cfg->world, id, cfg->rank));
        const char* pe = getenv("GORILA_P2P");  // GORILA_P2P=0: NCCL reduce-scatter / all-gather
        if (!(pe && atoi(pe) == 0) && cfg->world <= MAX_W) ctx->p2p = p2p_setup(ctx);
        if (ctx->per_msg && !ctx->p2p) {
            return fail(GORILA_E_INVALID, "per-message mode needs the peer-memory exchange (world > 1)");
        }
        if (ctx->replay_global && !ctx->p2p) {
            return fail(GORILA_E_INVALID, "global replay needs the peer-memory mapping (world > 1)");
        }
    }
    // world > 1 without an NCCL id: the caller exchanges the peer records (gorila_peer_connect)
    if (cfg->world == 1 || ctx->p2p) CU(shard_table(ctx));
    CU(stage_alloc(ctx));
    ctx->ring_slot = (RING_HDR + std::min(ctx->L, RING_MAXL) * (int)sizeof(DevLearnerInfo) + 63) / 64 * 64;
    CU(cudaHostAlloc((void**)&ctx->ring_host, (size_t)gorila_ctx::kRing * ctx->ring_slot, cudaHostAllocMapped));
    memset(ctx->ring_host, 0, (size_t)gorila_ctx::kRing * ctx->ring_slot);
    CU(cudaHostGetDevicePointer((void**)&ctx->ring_dev, ctx->ring_host, 0));
    CU(cudaStreamSynchronize(st));
    guard.c = nullptr;
    *out = ctx;
    return GORILA_OK;
}

void gorila_destroy(gorila_ctx* ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    for (auto e : ctx->ev_fork)
        if (e) cudaEventDestroy(e);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->ev_join2) cudaEventDestroy(ctx->ev_join2);
    if (ctx->side2) {
        cudaStreamSynchronize(ctx->side2);
        cudaStreamDestroy(ctx->side2);
    }
    if (ctx->ev_s2_fork) cudaEventDestroy(ctx->ev_s2_fork);
    if (ctx->ev_s2_join) cudaEventDestroy(ctx->ev_s2_join);
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : ctx->graph_marks)
        for (auto& m : kv.second) cudaEventDestroy(m.second);
    peer_close(ctx);
    for (int i = 0; i < gorila_ctx::kStage; ++i) {
        if (ctx->stage_ev[i]) {
            cudaEventSynchronize(ctx->stage_ev[i]);
            cudaEventDestroy(ctx->stage_ev[i]);
        }
        if (ctx->stage[i]) cudaFreeHost(ctx->stage[i]);
    }
    if (ctx->stage_dev) cudaFree(ctx->stage_dev);
    if (ctx->cap_buf) cudaFree(ctx->cap_buf);
    if (ctx->ring_host) cudaFreeHost(ctx->ring_host);
    if (ctx->comm) {
        if (ctx->poisoned) ncclCommAbort(ctx->comm);
        else ncclCommDestroy(ctx->comm);
    }
    delete ctx;
}

// the staging ring of small host inserts (allocated by gorila_init: pinned allocation takes
// milliseconds and must not land inside a caller's first training step)
static cudaError_t stage_alloc(gorila_ctx* ctx) {
    ctx->stage_bytes = (size_t)1 << 22;
    for (int i = 0; i < gorila_ctx::kStage; ++i) {
        cudaError_t e;
        if (!ctx->stage_ev[i] && (e = cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming))) return e;
        if ((e = cudaHostAlloc((void**)&ctx->stage[i], ctx->stage_bytes, cudaHostAllocMapped))) return e;
        if ((e = cudaHostGetDevicePointer((void**)&ctx->stage_dptr[i], ctx->stage[i], 0))) return e;
        if ((e = cudaEventRecord(ctx->stage_ev[i], ctx->stream))) return e;
    }
    return ctx->stage_dev ? cudaSuccess : cudaMalloc((void**)&ctx->stage_dev, ctx->stage_bytes);
}

gorila_status replay_insert(gorila_ctx* ctx, int32_t learner, int64_t count, const uint8_t* frames,
                            const uint8_t* actions, const float* rewards, const uint8_t* terminals,
                            int32_t src_on_device) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    if (count < 0) return fail(GORILA_E_SHAPE, "negative count");
    if (count == 0) return GORILA_OK;
    if (!frames || !actions || !rewards || !terminals) return fail(GORILA_E_INVALID, "null buffer");
    if (!src_on_device) {  // a host action outside [0, nA) would index past the TD kernel's Q rows
        const int64_t from = count > ctx->cfg.replay_capacity ? count - ctx->cfg.replay_capacity : 0;
        for (int64_t i = from; i < count; ++i)
            if (actions[i] >= ctx->nA)
                return fail(GORILA_E_RANGE, "action " + std::to_string((int)actions[i]) + " at " + std::to_string(i) +
                                                " is not below n_actions");
    }
    Learner& l = ctx->learners[learner];
    const int64_t C = ctx->cfg.replay_capacity;
    cudaMemcpyKind kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    cudaStream_t st = ctx->stream;
    // host sources of a small insert go through the pinned staging ring (no stream synchronisation)
    const int64_t keep = std::min<int64_t>(count, C);
    const size_t need = (size_t)keep * (FRAME_BYTES + 1 + sizeof(float) + 1) + 64;
    bool staged = false;
    if (!src_on_device && need <= ((size_t)1 << 22)) {
        const int k = ctx->stage_next;
        if (!ctx->stage[k]) CU(stage_alloc(ctx));
        CU(cudaEventSynchronize(ctx->stage_ev[k]));  // its previous upload is done (normally long ago)
        const int64_t skip0 = count - keep;
        uint8_t* sb = ctx->stage[k];
        memcpy(sb, frames + skip0 * FRAME_BYTES, (size_t)keep * FRAME_BYTES);
        uint8_t* sa = sb + (size_t)keep * FRAME_BYTES;
        memcpy(sa, actions + skip0, keep);
        float* sr = reinterpret_cast<float*>(sa + ((keep + 15) / 16) * 16);
        memcpy(sr, rewards + skip0, keep * sizeof(float));
        uint8_t* sd = reinterpret_cast<uint8_t*>(sr + keep);
        memcpy(sd, terminals + skip0, keep);
        frames = sb - skip0 * FRAME_BYTES;  // the loop below indexes from the original start
        actions = sa - skip0;
        rewards = sr - skip0;
        terminals = sd - skip0;
        staged = true;
    }
    if (staged) {  // one scatter kernel (+ one upload for larger inserts); the slot is reused after its event
        const int k = ctx->stage_next;
        const size_t bytes = (size_t)keep * FRAME_BYTES + ((keep + 15) / 16) * 16 + keep * sizeof(float) + keep;
        // up to 64 KB the kernel reads the mapped pinned slot itself: one stream operation instead
        // of a copy-engine hop plus a kernel (the e2e loop inserts one 7 KB transition per step)
        const uint8_t* src = ctx->stage_dptr[k];
        if (bytes > ((size_t)1 << 16)) {
            CU(cudaMemcpyAsync(ctx->stage_dev, ctx->stage[k], bytes, cudaMemcpyHostToDevice, st));
            src = ctx->stage_dev;
        }
        const int64_t t0 = l.n_host + (count - keep);
        l.n_host += count;
        const int64_t work = keep * (FRAME_BYTES / 16) + keep;
        k_insert_scatter<<<(unsigned)std::min<int64_t>(148 * 4, (work + 255) / 256), 256, 0, st>>>(
            src, keep, t0, C, l.frames, l.a, l.r, l.d, l.n_dev, (uint64_t)l.n_host);
        ctx->launches++;
        CU(cudaGetLastError());
        CU(cudaEventRecord(ctx->stage_ev[k], st));
        ctx->stage_next = (k + 1) % gorila_ctx::kStage;
        return GORILA_OK;
    }
    // only the last min(count, C) steps survive; copy them in at most two contiguous segments
    int64_t skip = count > C ? count - C : 0;
    int64_t t = l.n_host + skip, left = count - skip, src = skip;
    while (left > 0) {
        const int64_t slot = t % C, seg = std::min(left, C - slot);
        CU(cudaMemcpyAsync(l.frames + slot * FRAME_BYTES, frames + src * FRAME_BYTES, seg * FRAME_BYTES, kind, st));
        CU(cudaMemcpyAsync(l.a + slot, actions + src, seg, kind, st));
        CU(cudaMemcpyAsync(l.r + slot, rewards + src, seg * sizeof(float), kind, st));
        CU(cudaMemcpyAsync(l.d + slot, terminals + src, seg, kind, st));
        t += seg; src += seg; left -= seg;
    }
    if (!src_on_device) {
        CU(cudaStreamSynchronize(st));  // large host inserts: the caller's buffers may be reused on return
    }
    l.n_host += count;
    k_set_u64<<<1, 1, 0, st>>>(l.n_dev, (uint64_t)l.n_host);
    ctx->launches++;
    CU(cudaGetLastError());
    return GORILA_OK;
}

static void replay_barrier(gorila_ctx* ctx);

gorila_status replay_sample_shards(gorila_ctx* ctx, int32_t* shard_out) {
    if (!ctx || !shard_out) return fail(GORILA_E_INVALID, "null argument");
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(shard_out, ctx->sshard, sizeof(int32_t) * ctx->B, cudaMemcpyDeviceToHost));
    return GORILA_OK;
}

gorila_status replay_sample(gorila_ctx* ctx, int32_t learner, uint64_t round, int64_t* idx_out, uint8_t* s_out,
                            uint8_t* s2_out, uint8_t* a_out, float* r_out, uint8_t* d_out) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    if (!exchange_ready(ctx)) return fail(GORILA_E_INVALID, "world > 1: connect the peers first (gorila_peer_connect)");
    Learner& l = ctx->learners[learner];
    const int64_t size = std::min<int64_t>(l.n_host, ctx->cfg.replay_capacity);
    if (size - 1 < std::max<int64_t>(1, ctx->cfg.min_replay)) return fail(GORILA_E_NOT_READY, "replay not ready");
    const int B = ctx->B;
    cudaStream_t st = ctx->stream;
    const gorila_config& cfg = ctx->cfg;
    // sample into u8-valued T buffers of the scratch (same kernel as learner_step)
    launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->dev_round, (uint64_t)round);
    ctx->dev_round_expect = round;
    dim3 grid((FRAME_BYTES / 16 + 255) / 256, B);
    uint2 key = make_uint2((uint32_t)cfg.seed, (uint32_t)(cfg.seed >> 32));
    replay_barrier(ctx);
    const ShardPtrs* tab = ctx->replay_global ? ctx->shard_tab : nullptr;
    const uint64_t* snap = ctx->replay_global && ctx->W > 1 && !replay_barrier_off() ? ctx->n_snap : nullptr;
    if (cfg.math == GORILA_MATH_FP32)
        k_sample<float><<<grid, 256, 0, st>>>(l.frames, l.a, l.r, l.d, cfg.replay_capacity, l.n_dev, tab,
                                              ctx->n_shards, snap, ctx->sshard, key,
                                              (uint32_t)(cfg.learner_id_base + learner), ctx->dev_round, B, (float*)ctx->s,
                                              (float*)ctx->s2, ctx->sa, ctx->sr, ctx->sd, ctx->sidx, nullptr);
    else
        k_sample<__nv_bfloat16><<<grid, 256, 0, st>>>(l.frames, l.a, l.r, l.d, cfg.replay_capacity, l.n_dev, tab,
                                                      ctx->n_shards, snap, ctx->sshard, key,
                                                      (uint32_t)(cfg.learner_id_base + learner), ctx->dev_round,
                                                      B, (__nv_bfloat16*)ctx->s, (__nv_bfloat16*)ctx->s2, ctx->sa,
                                                      ctx->sr, ctx->sd, ctx->sidx, nullptr);
    ctx->launches++;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st));
    if (idx_out) CU(cudaMemcpy(idx_out, ctx->sidx, sizeof(int64_t) * B, cudaMemcpyDeviceToHost));
    if (a_out) CU(cudaMemcpy(a_out, ctx->sa, B, cudaMemcpyDeviceToHost));
    if (r_out) CU(cudaMemcpy(r_out, ctx->sr, sizeof(float) * B, cudaMemcpyDeviceToHost));
    if (d_out) CU(cudaMemcpy(d_out, ctx->sd, B, cudaMemcpyDeviceToHost));
    // NHWC T -> NCHW u8 on the host side of the boundary (debug / parity entry point)
    const int64_t n_el = (int64_t)B * FRAME_BYTES * NSTACK;
    std::vector<uint8_t> raw(n_el * ctx->esz);
    for (int which = 0; which < 2; ++which) {
        uint8_t* dst = which ? s2_out : s_out;
        if (!dst) continue;
        CU(cudaMemcpy(raw.data(), which ? ctx->s2 : ctx->s, raw.size(), cudaMemcpyDeviceToHost));
        for (int64_t b = 0; b < B; ++b)
            for (int64_t p = 0; p < FRAME_BYTES; ++p)
                for (int c = 0; c < NSTACK; ++c) {
                    const int64_t src = (b * FRAME_BYTES + p) * NSTACK + c;
                    float val;
                    if (ctx->esz == 4) {
                        memcpy(&val, raw.data() + src * 4, 4);
                    } else {
                        uint16_t h;
                        memcpy(&h, raw.data() + src * 2, 2);
                        uint32_t bits = (uint32_t)h << 16;
                        memcpy(&val, &bits, 4);
                    }
                    dst[(b * NSTACK + c) * FRAME_BYTES + p] = (uint8_t)val;
                }
    }
    return GORILA_OK;
}

// global replay across ranks (f4): the device barrier of k_replay_barrier (no-op otherwise)
static void replay_barrier(gorila_ctx* ctx) {
    if (!ctx->replay_global || ctx->W == 1 || replay_barrier_off()) return;
    ReplayBarrier p{};
    p.epoch = ctx->replay_epoch;
    for (int q = 0; q < ctx->W; ++q) {
        p.flags[q] = peer_ptr(ctx, q, ctx->rflags);
        p.n_snap[q] = peer_ptr(ctx, q, ctx->n_snap);
    }
    p.tab = ctx->shard_tab;
    p.W = ctx->W;
    p.rank = ctx->rank;
    p.L = ctx->L;
    launch(ctx, k_replay_barrier, dim3(1), dim3(32), 0, p);
}

gorila_status learner_step(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                           const int32_t* staleness, gorila_learner_info* info_out) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (ctx->async_mode) return fail(GORILA_E_INVALID, "asynchronous mode (ps_mode 2): use gorila_async_run");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned");
    if (!exchange_ready(ctx)) return fail(GORILA_E_INVALID, "world > 1: connect the peers first (gorila_peer_connect)");
    if (!learners || n < 1 || n > ctx->L) return fail(GORILA_E_SHAPE, "bad learner list");
    for (int i = 0; i < n; ++i) {
        if (learners[i] < 0 || learners[i] >= ctx->L) return fail(GORILA_E_RANGE, "learner id out of range");
        if (i && learners[i] <= learners[i - 1]) return fail(GORILA_E_INVALID, "learners must be ascending");
        if (staleness && (staleness[i] < 0 || staleness[i] >= ctx->H))
            return fail(GORILA_E_RANGE, "staleness must be in [0, history)");
    }
    cudaStream_t st = ctx->stream;
    mark(ctx, -1);
    ctx->prof_steps += ctx->prof ? 1 : 0;
    if (ctx->dev_round_expect != round) {  // the device counter is advanced by k_apply each round
        launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->dev_round, (uint64_t)round);
        ctx->dev_round_expect = round;
    }
    mark(ctx, PH_STEP_MISC);
    if (ctx->per_msg && n != ctx->L)
        return fail(GORILA_E_INVALID, "per-message mode: every local learner runs each round");
    ctx->early_learner = -1;
    static const bool early_env = [] {
        // GORILA_EARLY=1: overlap the fc4-region exchange with the conv backward (measured slower at
        // N=2: 122 vs 118.5 us/step, so off by default)
        const char* e = getenv("GORILA_EARLY");
        return e && atoi(e) != 0;
    }();
    if (early_env && ctx->in_round && ctx->p2p && ctx->W > 1 && ctx->H >= 2 && ctx->fork && !ctx->prof &&
        !ctx->early_pending)
        for (int i = 0; i < n; ++i) {  // the last learner that runs
            const Learner& l = ctx->learners[learners[i]];
            const int64_t size = std::min<int64_t>(l.n_host, ctx->cfg.replay_capacity);
            if (size - 1 >= std::max<int64_t>(1, ctx->cfg.min_replay)) ctx->early_learner = learners[i];
        }
    replay_barrier(ctx);  // f4: every rank's earlier inserts visible before the first draw
    int ran = 0;  // the first learner that runs stores G, later ones accumulate (no memset)
    for (int i = 0; i < n; ++i) {
        const int j = learners[i];
        Learner& l = ctx->learners[j];
        const int64_t size = std::min<int64_t>(l.n_host, ctx->cfg.replay_capacity);
        if (size - 1 < std::max<int64_t>(1, ctx->cfg.min_replay)) {
            launch(ctx, k_mark_not_ready, dim3(1), dim3(1), 0, l.info, (const LearnerStats*)l.stats);
            continue;
        }
        const int s_j = staleness ? staleness[i] : 0;
        gorila_status s = ctx->cfg.math == GORILA_MATH_FP32 ? run_learner<float>(ctx, j, round, s_j, ran > 0)
                                                             : run_learner<__nv_bfloat16>(ctx, j, round, s_j, ran > 0);
        if (s != GORILA_OK) return s;
        if (ctx->cap_acts) {  // a1..a4 are final once the forward ran (the backward only reads them)
            const size_t e = ctx->esz, Bs = (size_t)ctx->B;
            const size_t n1 = Bs * A1 * e, n2 = Bs * A2 * e, n3 = Bs * A3 * e, n4 = Bs * A4 * 4;
            uint8_t* dst = ctx->cap_buf + (size_t)j * (n1 + n2 + n3 + n4);
            CU(cudaMemcpyAsync(dst, ctx->a1, n1, cudaMemcpyDeviceToDevice, st));
            CU(cudaMemcpyAsync(dst + n1, ctx->a2, n2, cudaMemcpyDeviceToDevice, st));
            CU(cudaMemcpyAsync(dst + n1 + n2, ctx->a3, n3, cudaMemcpyDeviceToDevice, st));
            CU(cudaMemcpyAsync(dst + n1 + n2 + n3, ctx->a4, n4, cudaMemcpyDeviceToDevice, st));
        }
        ++ran;
    }
    if (ran == 0) {
        CU(cudaMemsetAsync(ctx->G, 0, sizeof(float) * ctx->W * ctx->q, st));
        CU(cudaMemsetAsync(ctx->n_acc_local, 0, sizeof(uint32_t), st));
    }
    if (ctx->W > 1)
        launch(ctx, k_write_counts, dim3(1), dim3(64), 0, ctx->counts, ctx->W, (const uint32_t*)ctx->n_acc_local);
    mark(ctx, PH_STEP_MISC);
    if (info_out)
        for (int i = 0; i < n; ++i)
            CU(cudaMemcpyAsync(&info_out[i], ctx->learners[learners[i]].info, sizeof(gorila_learner_info),
                               cudaMemcpyDeviceToHost, st));
    CU(cudaGetLastError());
    return GORILA_OK;
}

// W > 1 over peer memory: k_apply_p2p (gradient sum + optimizer + replica broadcast) and
// k_peer_wait (everyone done) instead of reduce-scatter / apply / all-gather / pack
void p2p_params(gorila_ctx* ctx, uint64_t round, ApplyParams& p, P2PParams& x) {
    const int W = ctx->W, r = ctx->rank;
    const int64_t lo = (int64_t)r * ctx->q;
    const int slot = (int)((round + 1) % (uint64_t)ctx->H);
    p = ApplyParams{};
    p.m = ctx->m;
    p.v = ctx->v;
    p.dev_round = ctx->dev_round;
    p.period = ctx->cfg.target_period;
    if (ctx->fused_sync)
        for (int i = 0; i < ctx->sync_n; ++i) {
            p.sync_stats[p.n_sync] = ctx->learners[ctx->sync_ids[i]].stats;
            p.sync_flag[p.n_sync] = ctx->learners[ctx->sync_ids[i]].sync_flag;
            ++p.n_sync;
        }
    p.n_real = std::max<int64_t>(0, std::min<int64_t>(ctx->q, ctx->P - lo));
    p.optimizer = ctx->cfg.optimizer;
    p.lr = ctx->cfg.lr; p.rho = ctx->cfg.rms_rho; p.eps = ctx->cfg.rms_eps; p.ada_eps = ctx->cfg.ada_eps;
    p.V = ctx->V;
    p.round_info = ctx->round_info;
    p.vhist_dst = ctx->Vhist + slot;
    p.nA = ctx->nA;
    p.base = lo;
    x = P2PParams{};
    x.W = W;
    x.rank = r;
    for (int q = 0; q < W; ++q) {
        x.G[q] = peer_ptr(ctx, q, ctx->G) + lo;
        x.nacc[q] = peer_ptr(ctx, q, ctx->n_acc_local);
        x.theta[q] = peer_ptr(ctx, q, ctx->theta) + lo;
        x.rep_t[q] = peer_ptr(ctx, q, (uint8_t*)ctx->rep_t[slot]);
        x.rep_f[q] = peer_ptr(ctx, q, ctx->rep_f[slot]);
        x.flags[q] = peer_ptr(ctx, q, ctx->pflags);
        if (ctx->per_msg)
            for (int j = 0; j < ctx->L; ++j)
                x.Gm[q * ctx->L + j] = peer_ptr(ctx, q, ctx->G_all + (int64_t)j * W * ctx->q) + lo;
    }
    x.L = ctx->per_msg ? ctx->L : 0;
    for (int j = 0; j < (ctx->per_msg ? ctx->L : 0); ++j) {
        const Learner& l = ctx->learners[j];
        x.info[j] = l.info;
        x.stats[j] = l.stats;
        x.sync_flag[j] = l.sync_flag;
    }
    if (ctx->per_msg)  // f1: every global learner's theta^- (in-round target syncs write this rank's slice)
        for (int q = 0; q < W; ++q)
            for (int j = 0; j < ctx->L; ++j) {
                const Learner& l = ctx->learners[j];
                x.tm_t[q * ctx->L + j] = peer_ptr(ctx, q, (uint8_t*)l.tminus_t);
                x.tm_f[q * ctx->L + j] = peer_ptr(ctx, q, l.tminus_f);
            }
    x.max_delay = ctx->cfg.max_staleness;
    x.period = ctx->cfg.target_period;
    x.epoch = ctx->p2p_epoch;
    x.counter = ctx->p2p_counter;
    static const int dbg = [] {
        const char* e = getenv("GORILA_P2P_DBG");
        return e ? atoi(e) : 0;
    }();
    x.dbg = dbg;
}
// the fc4 weight region of this rank's slice, float4 units relative to the slice start
void w4_range(gorila_ctx* ctx, int64_t& a, int64_t& b) {
    const int64_t lo = (int64_t)ctx->rank * ctx->q, n = std::max<int64_t>(0, std::min<int64_t>(ctx->q, ctx->P - lo));
    a = std::min(n, std::max<int64_t>(0, OFF_W4 - lo));
    b = std::min(n, std::max<int64_t>(0, OFF_W4 + (int64_t)FC4_OUT * FC4_IN - lo));
    a = (a + 3) / 4;
    b = (b + 3) / 4;
    if (b < a) b = a;
}
void launch_apply_p2p(gorila_ctx* ctx, const ApplyParams& p, const P2PParams& x, int phase, int64_t lo0, int64_t hi0,
                      int64_t lo1, int64_t hi1, int book, int blocks) {
    if (ctx->cfg.math == GORILA_MATH_FP32)
        launch(ctx, k_apply_p2p<float>, dim3(blocks), dim3(256), 0, p, x, phase, lo0, hi0, lo1, hi1, book);
    else
        launch(ctx, k_apply_p2p<__nv_bfloat16>, dim3(blocks), dim3(256), 0, p, x, phase, lo0, hi0, lo1, hi1, book);
}
// phase 0 (gorila_round): the fc4 weight part of the slice, on side2 once this rank's fc4
// weight gradient (the last learner's) is in G
void early_apply_p2p(gorila_ctx* ctx, uint64_t round) {
    ApplyParams p;
    P2PParams x;
    p2p_params(ctx, round, p, x);
    int64_t a, b;
    w4_range(ctx, a, b);
    cudaEventRecord(ctx->ev_s2_fork, ctx->stream);
    cudaStreamWaitEvent(ctx->side2, ctx->ev_s2_fork, 0);
    OnSide2 on(ctx);
    launch_apply_p2p(ctx, p, x, 0, a, b, 0, 0, 0, 148);
    ctx->early_pending = true;
}

gorila_status ps_apply_p2p(gorila_ctx* ctx, uint64_t round, gorila_round_info* info_out) {
    ApplyParams p;
    P2PParams x;
    p2p_params(ctx, round, p, x);
    const int64_t n4 = (p.n_real + 3) / 4;
    const bool early = ctx->early_pending;
    if (early) {  // the rest of the slice (at most two pieces around the fc4 weight region)
        int64_t a, b;
        w4_range(ctx, a, b);
        launch_apply_p2p(ctx, p, x, 1, 0, a, b, n4, 1, 148 * 2);
    } else {
        launch_apply_p2p(ctx, p, x, 1, 0, n4, 0, 0, 1, 148 * 2);
    }
    ctx->dev_round_expect = round + 1;
    mark(ctx, PH_APPLY);
    if (early) {
        cudaEventRecord(ctx->ev_s2_join, ctx->side2);
        cudaStreamWaitEvent(ctx->stream, ctx->ev_s2_join, 0);
        ctx->early_pending = false;
    }
    launch(ctx, k_peer_wait, dim3(1), dim3(32), 0, x, early ? 1 : 0);
    mark(ctx, PH_AG);
    if (info_out) {
        uint64_t tmp[3];
        CU(cudaMemcpyAsync(tmp, ctx->round_info, sizeof(tmp), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        info_out->n_accepted = (uint32_t)tmp[0];
        info_out->pad_ = 0;
        info_out->version_before = tmp[1];
        info_out->version_after = tmp[2];
    }
    CU(cudaGetLastError());
    return GORILA_OK;
}

gorila_status ps_apply_shard(gorila_ctx* ctx, uint64_t round, gorila_round_info* info_out) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (ctx->async_mode) return fail(GORILA_E_INVALID, "asynchronous mode (ps_mode 2): use gorila_async_run");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned");
    if (!exchange_ready(ctx)) return fail(GORILA_E_INVALID, "world > 1: connect the peers first (gorila_peer_connect)");
    cudaStream_t st = ctx->stream;
    const int W = ctx->W, r = ctx->rank;
    float* gsl = ctx->G + (int64_t)r * ctx->q;
    mark(ctx, -1);
    if (W > 1 && ctx->p2p) return ps_apply_p2p(ctx, round, info_out);
    if (W > 1) {  // gradient + accepted counts onto the owning shard, one grouped launch
        NC(ncclGroupStart());
        NC(ncclReduceScatter(ctx->G, gsl, ctx->q, ncclFloat, ncclSum, ctx->comm, st));
        NC(ncclReduceScatter(ctx->counts, ctx->counts + r, 1, ncclFloat, ncclSum, ctx->comm, st));
        NC(ncclGroupEnd());
    }
    mark(ctx, PH_RS);
    ApplyParams p{};
    p.theta = ctx->theta + (int64_t)r * ctx->q;
    p.m = ctx->m;
    p.v = ctx->v;
    p.g = gsl;
    p.count = ctx->counts + (W > 1 ? r : 0);
    p.count_local = W > 1 ? nullptr : ctx->n_acc_local;
    p.dev_round = ctx->dev_round;
    p.period = ctx->cfg.target_period;
    p.n_sync = 0;
    if (ctx->fused_sync)
        for (int i = 0; i < ctx->sync_n; ++i) {
            p.sync_stats[p.n_sync] = ctx->learners[ctx->sync_ids[i]].stats;
            p.sync_flag[p.n_sync] = ctx->learners[ctx->sync_ids[i]].sync_flag;
            ++p.n_sync;
        }
    p.n_real = std::max<int64_t>(0, std::min<int64_t>(ctx->q, ctx->P - (int64_t)r * ctx->q));
    p.optimizer = ctx->cfg.optimizer;
    p.lr = ctx->cfg.lr; p.rho = ctx->cfg.rms_rho; p.eps = ctx->cfg.rms_eps; p.ada_eps = ctx->cfg.ada_eps;
    p.V = ctx->V;
    p.round_info = ctx->round_info;
    const int slot = (int)((round + 1) % (uint64_t)ctx->H);
    p.nA = ctx->nA;
    p.base = (int64_t)r * ctx->q;
    if (W == 1) {  // the optimizer emits the next round's replica directly (no separate pack)
        p.rep_t = ctx->rep_t[slot];
        p.rep_f = ctx->rep_f[slot];
        p.vhist_dst = ctx->Vhist + slot;
        // gorila_round: the optimizer also writes theta^- of the learners whose sync fires
        static const bool sync_fuse = [] {  // opt-in: measured 0.9 us/step slower than the predicated pack
            const char* e = getenv("GORILA_SYNC_FUSE");
            return e && atoi(e) != 0;
        }();
        ctx->sync_fused_now = sync_fuse && ctx->fused_sync && !ctx->per_msg;
        if (ctx->ring_pending && !ctx->sync_fused_now && !ctx->per_msg && ctx->fused_sync && p.n_sync <= 8) {
            p.ring = ctx->ring_dev;  // k_apply block 0 stores the results (no k_emit_ring)
            p.ring_R = gorila_ctx::kRing;
            p.ring_slot_bytes = ctx->ring_slot;
            for (int i = 0; i < p.n_sync; ++i) p.ring_info[i] = ctx->learners[ctx->sync_ids[i]].info;
            ctx->ring_pending = false;
        }
        if (ctx->sync_fused_now) {
            p.sync_copy = 1;
            p.counter = ctx->apply_counter;
            for (int i = 0; i < p.n_sync; ++i) {
                const Learner& l = ctx->learners[ctx->sync_ids[i]];
                p.sync_tm_t[i] = l.tminus_t;
                p.sync_tm_f[i] = l.tminus_f;
            }
        }
    }
    if (ctx->per_msg) {  // W == 1 here (W > 1 runs the peer-memory exchange)
        MsgParams mp{};
        mp.nmsg = ctx->L;
        for (int j = 0; j < ctx->L; ++j) {
            const Learner& l = ctx->learners[j];
            mp.G[j] = ctx->G_all + (int64_t)j * ctx->W * ctx->q;
            mp.info[j] = l.info;
            mp.stats[j] = l.stats;
            mp.sync_flag[j] = l.sync_flag;
            mp.tm_t[j] = l.tminus_t;
            mp.tm_f[j] = l.tminus_f;
        }
        mp.max_delay = ctx->cfg.max_staleness;
        mp.counter = ctx->apply_counter;
        if (ctx->cfg.math == GORILA_MATH_FP32) launch(ctx, k_apply_msg<float>, dim3(148 * 4), dim3(256), 0, p, mp);
        else launch(ctx, k_apply_msg<__nv_bfloat16>, dim3(148 * 4), dim3(256), 0, p, mp);
    } else {
        p.book_last = p.sync_copy ? 0 : 1;  // one extra block takes the decisions / stores the ring slot
        const dim3 grid(148 * 4 + p.book_last);
        if (ctx->cfg.math == GORILA_MATH_FP32) launch(ctx, k_apply<float>, grid, dim3(256), 0, p);
        else launch(ctx, k_apply<__nv_bfloat16>, grid, dim3(256), 0, p);
    }
    ctx->dev_round_expect = round + 1;
    mark(ctx, PH_APPLY);
    if (W > 1) {
        NC(ncclAllGather(p.theta, ctx->theta, ctx->q, ncclFloat, ctx->comm, st));
        mark(ctx, PH_AG);
        gorila_status s = pack_any(ctx, ctx->theta, ctx->rep_t[slot], ctx->rep_f[slot], nullptr, ctx->Vhist + slot);
        if (s != GORILA_OK) return s;
        mark(ctx, PH_PACK);
    }
    if (info_out) {
        uint64_t tmp[3];
        CU(cudaMemcpyAsync(tmp, ctx->round_info, sizeof(tmp), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        info_out->n_accepted = (uint32_t)tmp[0];
        info_out->pad_ = 0;
        info_out->version_before = tmp[1];
        info_out->version_after = tmp[2];
    }
    CU(cudaGetLastError());
    return GORILA_OK;
}

gorila_status sync_target(gorila_ctx* ctx, const int32_t* learners, int32_t n, int32_t force, uint8_t* synced_out) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned");
    if (!learners || n < 1) return fail(GORILA_E_SHAPE, "bad learner list");
    cudaStream_t st = ctx->stream;
    mark(ctx, -1);
    for (int i = 0; i < n; ++i) {
        gorila_status s = check_learner(ctx, learners[i]);
        if (s != GORILA_OK) return s;
        Learner& l = ctx->learners[learners[i]];
        // per-message mode (f1, R37): ps_apply_shard took every learner's in-round sync decisions and
        // wrote theta^- at the version each fired; only a forced sync acts here
        const bool msg_done = ctx->per_msg && !force;
        if (!ctx->fused_sync && !msg_done)  // gorila_round: k_apply already took the decision
            launch(ctx, k_sync_decide, dim3(1), dim3(1), 0, l.stats, (const uint64_t*)ctx->V,
                   (int64_t)ctx->cfg.target_period, (int)force, l.sync_flag);
        if (msg_done || (ctx->sync_fused_now && !force)) {  // k_apply wrote theta^- when it fired
        } else if (ctx->p2p && ctx->W > 1) {  // ranks hold only their own fp32 slice: copy the latest replica
            const int slot = (int)(ctx->dev_round_expect % (uint64_t)ctx->H);
            const int64_t nt = (int64_t)ctx->rl.n_t * ctx->esz;
            launch(ctx, k_copy_replica, dim3(148 * 2), dim3(256), 0, (const uint4*)ctx->rep_t[slot],
                   (uint4*)l.tminus_t, nt / 16, (const float4*)ctx->rep_f[slot], (float4*)l.tminus_f,
                   (int64_t)ctx->rl.n_f / 4, (const uint8_t*)l.sync_flag);
        } else if ((s = pack_any(ctx, ctx->theta, l.tminus_t, l.tminus_f, l.sync_flag, nullptr)) != GORILA_OK) {
            return s;
        }
        if (synced_out) CU(cudaMemcpyAsync(&synced_out[i], l.sync_flag, 1, cudaMemcpyDeviceToHost, st));
    }
    mark(ctx, PH_SYNC);
    CU(cudaGetLastError());
    return GORILA_OK;
}

// pinned / registered host memory or device memory: a kernel may store to it (UVA: same address)
static bool device_accessible(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return true;
    return at.type == cudaMemoryTypeHost && at.devicePointer == p;
}

// the last node of a posted round (k_emit_ring): results into the ring slot of this round
static void emit_ring(gorila_ctx* ctx, const int32_t* learners, int32_t n) {
    EmitRing p{};
    p.ring = ctx->ring_dev;
    p.R = gorila_ctx::kRing;
    p.slot_bytes = ctx->ring_slot;
    p.n = n;
    for (int i = 0; i < n; ++i) {
        p.info[i] = ctx->learners[learners[i]].info;
        p.sync[i] = ctx->learners[learners[i]].sync_flag;
    }
    p.round_info = ctx->round_info;
    p.dev_round = ctx->dev_round;
    launch(ctx, k_emit_ring, dim3(1), dim3(128), 0, p);
}

static gorila_status round_impl(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                                const int32_t* staleness, gorila_learner_info* info_out,
                                gorila_round_info* round_info_out, uint8_t* synced_out, bool sync,
                                bool ring = false) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned");
    if (!learners || n < 1 || n > ctx->L) return fail(GORILA_E_SHAPE, "bad learner list");
    cudaStream_t st = ctx->stream;
    bool graphable = st != nullptr;  // the legacy default stream cannot be captured
    std::vector<int64_t> key;
    for (int i = 0; i < n; ++i) {
        if (learners[i] < 0 || learners[i] >= ctx->L) return fail(GORILA_E_RANGE, "learner id out of range");
        const Learner& l = ctx->learners[learners[i]];
        const int64_t size = std::min<int64_t>(l.n_host, ctx->cfg.replay_capacity);
        if (size - 1 < std::max<int64_t>(1, ctx->cfg.min_replay)) graphable = false;
        const int s_i = staleness ? staleness[i] : 0;
        if ((uint64_t)s_i > round) graphable = false;
        key.push_back(learners[i]);
        key.push_back(s_i);
    }
    key.push_back((int64_t)(round % (uint64_t)ctx->H));
    key.push_back(ctx->prof ? 1 : 0);  // profiling graphs carry event-record nodes
    key.push_back(ring ? 1 : 0);       // posted rounds end with the result-ring node
    gorila_status s;
    auto eager = [&]() -> gorila_status {
        ctx->in_round = true;
        gorila_status r = learner_step(ctx, learners, n, round, staleness, nullptr);
        ctx->in_round = false;
        if (r != GORILA_OK) return r;
        ctx->fused_sync = n <= 8;  // k_apply takes the target-sync decisions (same predicate, R13)
        ctx->sync_n = n;
        for (int i = 0; i < n && i < 8; ++i) ctx->sync_ids[i] = learners[i];
        ctx->ring_pending = ring;
        r = ps_apply_shard(ctx, round, nullptr);
        if (r == GORILA_OK) r = sync_target(ctx, learners, n, 0, nullptr);
        if (r == GORILA_OK && ctx->ring_pending) emit_ring(ctx, learners, n);  // not stored by k_apply
        ctx->ring_pending = false;
        ctx->fused_sync = false;
        ctx->sync_fused_now = false;
        return r;
    };
    auto it = graphable ? ctx->graphs.find(key) : ctx->graphs.end();
    if (it != ctx->graphs.end()) {
        if (ctx->dev_round_expect != round)
            launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->dev_round, (uint64_t)round);
        CU(cudaGraphLaunch(it->second, st));
        ctx->dev_round_expect = round + 1;
        ctx->launches += ctx->graph_kernels[key];
        if (ctx->prof) {  // the graph's events are re-recorded by every replay: fold them now
            CU(cudaStreamSynchronize(st));
            CU(fold_marks(ctx, ctx->graph_marks[key]));
            ctx->prof_steps += 1;
        }
    } else if (!graphable || ctx->graph_seen[key]++ == 0) {
        if ((s = eager()) != GORILA_OK) return s;  // first use: eager (also sets lazy kernel attributes)
    } else {
        // capture the round once; the captured sampler reads ctx->dev_round (advanced by k_apply)
        if (ctx->dev_round_expect != round)
            launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->dev_round, (uint64_t)round);
        ctx->dev_round_expect = round;
        CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        ctx->capturing = true;
        const uint64_t launches0 = ctx->launches;
        const size_t marks0 = ctx->marks.size();
        const size_t used0 = ctx->ev_used;
        s = eager();
        ctx->capturing = false;
        if (ctx->prof) {  // these marks belong to the graph, not to the eager accumulator
            std::vector<std::pair<int, cudaEvent_t>> gm;
            for (size_t i = marks0; i < ctx->marks.size(); ++i)
                gm.push_back({ctx->marks[i].first, ctx->ev_pool[ctx->marks[i].second]});
            ctx->graph_marks[key] = gm;
            ctx->marks.resize(marks0);
            // hand the graph's events over (they must not be re-recorded by eager marks)
            ctx->ev_pool.erase(ctx->ev_pool.begin() + used0, ctx->ev_pool.begin() + ctx->ev_used);
            ctx->ev_used = used0;
            ctx->prof_steps -= 1;  // the capture itself executed nothing
        }
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (s != GORILA_OK) {
            if (graph) cudaGraphDestroy(graph);
            return s;
        }
        CU(ce);
        cudaGraphExec_t exec = nullptr;
        CU(cudaGraphInstantiate(&exec, graph, 0));
        cudaGraphDestroy(graph);
        ctx->graphs[key] = exec;
        ctx->graph_kernels[key] = ctx->launches - launches0;
        CU(cudaGraphLaunch(exec, st));
        ctx->dev_round_expect = round + 1;
        if (ctx->prof) {
            CU(cudaStreamSynchronize(st));
            CU(fold_marks(ctx, ctx->graph_marks[key]));
            ctx->prof_steps += 1;
        }
    }
    // asynchronous results into device-accessible (pinned) host buffers: one small copy kernel
    // instead of up to 2n+1 copy-engine operations on the stream
    if (!sync && n <= SMALL_COPY_MAX / 2 - 1 && (info_out || synced_out || round_info_out) &&
        device_accessible(info_out) && device_accessible(synced_out) && device_accessible(round_info_out)) {
        SmallCopies sc{};
        auto add = [&](void* dst, const void* src, int bytes) {
            sc.dst[sc.n] = (uint8_t*)dst; sc.src[sc.n] = (const uint8_t*)src; sc.bytes[sc.n] = bytes; sc.n++;
        };
        for (int i = 0; i < n && info_out; ++i)
            add(&info_out[i], ctx->learners[learners[i]].info, (int)sizeof(gorila_learner_info));
        for (int i = 0; i < n && synced_out; ++i) add(&synced_out[i], ctx->learners[learners[i]].sync_flag, 1);
        if (round_info_out) add(round_info_out, ctx->round_info, (int)sizeof(gorila_round_info));
        k_small_copies<<<1, 32 * std::min(sc.n, 8), 0, st>>>(sc);
        ctx->launches++;
        CU(cudaGetLastError());
        return GORILA_OK;
    }
    if (info_out)
        for (int i = 0; i < n; ++i)
            CU(cudaMemcpyAsync(&info_out[i], ctx->learners[learners[i]].info, sizeof(gorila_learner_info),
                               cudaMemcpyDeviceToHost, st));
    if (synced_out)
        for (int i = 0; i < n; ++i)
            CU(cudaMemcpyAsync(&synced_out[i], ctx->learners[learners[i]].sync_flag, 1, cudaMemcpyDeviceToHost, st));
    static_assert(sizeof(gorila_round_info) == 3 * sizeof(uint64_t), "round info = [n_acc, V_before, V_after]");
    if (round_info_out && !sync)  // same bytes: n_accepted (+ zero pad) and the two versions
        CU(cudaMemcpyAsync(round_info_out, ctx->round_info, sizeof(gorila_round_info), cudaMemcpyDeviceToHost, st));
    if (round_info_out && sync) {
        uint64_t tmp[3];
        CU(cudaMemcpyAsync(tmp, ctx->round_info, sizeof(tmp), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        round_info_out->n_accepted = (uint32_t)tmp[0];
        round_info_out->pad_ = 0;
        round_info_out->version_before = tmp[1];
        round_info_out->version_after = tmp[2];
    }
    if (sync && (info_out || synced_out)) CU(cudaStreamSynchronize(st));
    CU(cudaGetLastError());
    return GORILA_OK;
}

// ---------------------------------------------------------------- NEXT row f2: asynchronous PS
gorila_status gorila_async_run(gorila_ctx* ctx, const int32_t* learners, int32_t n, int64_t steps, uint64_t round0,
                               int32_t server_blocks, gorila_async_stats* out) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned");
    if (!ctx->async_mode) return fail(GORILA_E_INVALID, "gorila_async_run needs ps_mode 2 (asynchronous)");
    if (!exchange_ready(ctx)) return fail(GORILA_E_INVALID, "world > 1: connect the peers first (gorila_peer_connect)");
    if (ctx->W > 1 && !ctx->p2p) return fail(GORILA_E_INVALID, "asynchronous mode needs the peer-memory mapping");
    if (!learners || n < 1 || n > ctx->L || steps < 0) return fail(GORILA_E_SHAPE, "bad learner list / steps");
    for (int i = 0; i < n; ++i) {
        if (learners[i] < 0 || learners[i] >= ctx->L) return fail(GORILA_E_RANGE, "learner id out of range");
        if (i && learners[i] <= learners[i - 1]) return fail(GORILA_E_INVALID, "learners must be ascending");
        const Learner& l = ctx->learners[learners[i]];
        if (std::min<int64_t>(l.n_host, ctx->cfg.replay_capacity) - 1 < std::max<int64_t>(1, ctx->cfg.min_replay))
            return fail(GORILA_E_NOT_READY, "replay not ready");
    }
    cudaStream_t st = ctx->stream;
    const int W = ctx->W, r = ctx->rank, L = ctx->L;
    const bool fp32 = ctx->cfg.math == GORILA_MATH_FP32;
    // the live replica (slot 0) = the latest one; the state and counters start from zero
    const int latest = (int)(ctx->dev_round_expect % (uint64_t)ctx->H);
    if (latest != 0)
        launch(ctx, k_copy_replica, dim3(148 * 2), dim3(256), 0, (const uint4*)ctx->rep_t[latest], (uint4*)ctx->rep_t[0],
               (int64_t)ctx->rl.n_t * (int64_t)ctx->esz / 16, (const float4*)ctx->rep_f[latest], (float4*)ctx->rep_f[0],
               (int64_t)ctx->rl.n_f / 4, (const uint8_t*)nullptr);
    // CUDA's lazy module loading blocks a kernel's first launch until the running kernels finish, which
    // would stall every learner kernel behind the persistent server: load them all now, with one learner
    // step whose only lasting effect (the outlier statistics, info) is undone
    {
        Learner& l0 = ctx->learners[learners[0]];
        CU(cudaMemcpyAsync(ctx->tmp_canon, l0.stats, sizeof(LearnerStats), cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync((uint8_t*)ctx->tmp_canon + 256, l0.info, sizeof(DevLearnerInfo), cudaMemcpyDeviceToDevice, st));
        launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->dev_round, round0);
        gorila_status s0 = fp32 ? run_learner<float>(ctx, learners[0], round0, 0, 0)
                                : run_learner<__nv_bfloat16>(ctx, learners[0], round0, 0, 0);
        if (s0 != GORILA_OK) return s0;
        CU(cudaMemcpyAsync(l0.stats, ctx->tmp_canon, sizeof(LearnerStats), cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(l0.info, (uint8_t*)ctx->tmp_canon + 256, sizeof(DevLearnerInfo), cudaMemcpyDeviceToDevice, st));
        cudaFuncAttributes fa;
        CU(cudaFuncGetAttributes(&fa, k_async_fetch));
        CU(cudaFuncGetAttributes(&fa, k_async_send));
        CU(cudaFuncGetAttributes(&fa, k_async_done));
        CU(cudaFuncGetAttributes(&fa, k_async_barrier));
        CU(cudaFuncGetAttributes(&fa, k_copy_replica));
        CU(cudaFuncGetAttributes(&fa, k_set_u64));
        CU(cudaFuncGetAttributes(&fa, k_copy_u64));
        CU(cudaFuncGetAttributes(&fa, k_ps_server<float>));
        CU(cudaFuncGetAttributes(&fa, k_ps_server<__nv_bfloat16>));
    }
    CU(cudaMemsetAsync(ctx->ast, 0, sizeof(AsyncState), st));
    k_copy_u64<<<1, 1, 0, st>>>(&ctx->ast->V, ctx->V);  // the shard's versions continue from V
    ctx->launches++;
    ApplyParams ap{};
    P2PParams x{};
    p2p_params(ctx, round0, ap, x);  // this rank's slice bounds / optimizer constants; peer flag areas
    const uint64_t ep = ++ctx->async_epoch;
    if (W > 1) launch(ctx, k_async_barrier, dim3(1), dim3(32), 0, x, ep);  // every rank reset before any send
    CU(cudaStreamSynchronize(st));
    // the server: a persistent kernel on side2, beside the learner stream
    ServerParams sp{};
    sp.p = ap;
    sp.p.theta = ctx->theta + (int64_t)r * ctx->q;
    sp.st = ctx->ast;
    for (int q = 0; q < W; ++q)
        for (int j = 0; j < L; ++j) {
            sp.G[q * L + j] = peer_ptr(ctx, q, ctx->G_all + (int64_t)j * W * ctx->q) + (int64_t)r * ctx->q;
            sp.consumed[q * L + j] = peer_ptr(ctx, q, &ctx->ast->consumed[r][j]);
        }
    for (int q = 0; q < W; ++q) {
        sp.live_t[q] = peer_ptr(ctx, q, (uint8_t*)ctx->rep_t[0]);
        sp.live_f[q] = peer_ptr(ctx, q, ctx->rep_f[0]);
    }
    sp.W = W;
    sp.max_delay = ctx->cfg.max_staleness;
    const int nsrv = server_blocks > 0 ? server_blocks : 32;
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(nsrv);
        cfg.blockDim = dim3(256);
        cfg.stream = ctx->side2;
        if (fp32) CU(cudaLaunchKernelEx(&cfg, k_ps_server<float>, sp));
        else CU(cudaLaunchKernelEx(&cfg, k_ps_server<__nv_bfloat16>, sp));
        ctx->launches++;
    }
    // the learners, round robin on the library stream
    FetchParams fp{};
    fp.st = ctx->ast;
    fp.W = W;
    fp.period = ctx->cfg.target_period;
    fp.vhist = ctx->Vhist + 1;
    for (int q = 0; q < W; ++q) fp.V[q] = &peer_ptr(ctx, q, ctx->ast)->V;
    SendParams sd{};
    sd.st = ctx->ast;
    sd.W = W;
    for (int q = 0; q < W; ++q) sd.shard[q] = peer_ptr(ctx, q, ctx->ast);
    const int64_t nt16 = (int64_t)ctx->rl.n_t * (int64_t)ctx->esz / 16, nf4 = (int64_t)ctx->rl.n_f / 4;
    for (int64_t k = 0; k < steps; ++k) {
        launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->dev_round, round0 + (uint64_t)k);
        ctx->dev_round_expect = round0 + (uint64_t)k;
        for (int i = 0; i < n; ++i) {
            const int j = learners[i];
            Learner& l = ctx->learners[j];
            fp.j = j;
            fp.stats = l.stats;
            fp.sync_flag = l.sync_flag;
            fp.info = l.info;
            launch(ctx, k_async_fetch, dim3(1), dim3(1), 0, fp);
            launch(ctx, k_copy_replica, dim3(148), dim3(256), 0, (const uint4*)ctx->rep_t[0], (uint4*)ctx->rep_t[1],
                   nt16, (const float4*)ctx->rep_f[0], (float4*)ctx->rep_f[1], nf4, (const uint8_t*)nullptr);
            launch(ctx, k_copy_replica, dim3(148), dim3(256), 0, (const uint4*)ctx->rep_t[1], (uint4*)l.tminus_t, nt16,
                   (const float4*)ctx->rep_f[1], (float4*)l.tminus_f, nf4, (const uint8_t*)l.sync_flag);
            gorila_status s = fp32 ? run_learner<float>(ctx, j, round0 + (uint64_t)k, 0, 0)
                                   : run_learner<__nv_bfloat16>(ctx, j, round0 + (uint64_t)k, 0, 0);
            if (s != GORILA_OK) return s;
            sd.j = j;
            sd.gid = ctx->cfg.learner_id_base + j;
            sd.info = l.info;
            launch(ctx, k_async_send, dim3(1), dim3(1), 0, sd);
        }
    }
    launch(ctx, k_async_done, dim3(1), dim3(1), 0, sd);
    CU(cudaStreamSynchronize(st));
    CU(cudaStreamSynchronize(ctx->side2));
    AsyncState h;
    CU(cudaMemcpy(&h, ctx->ast, sizeof(AsyncState), cudaMemcpyDeviceToHost));
    if (h.err)
        return fail(GORILA_E_CUDA, "asynchronous run: a bounded wait timed out (code " + std::to_string(h.err) +
                                       "; 1 server/message, 2 server/decision, 3 learner/consumed; learner progress " +
                                       std::to_string(h.progress) + ", tail " + std::to_string(h.tail) + ")");
    // the deterministic API's version record and next replica slot follow the live state
    launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->V, h.V);
    ctx->dev_round_expect = 0;  // the live replica is slot 0
    CU(cudaStreamSynchronize(st));
    if (out) {
        out->steps = (uint64_t)steps * (uint64_t)n;
        uint64_t sent = 0;
        for (int j = 0; j < L; ++j) sent += h.sent[j];
        out->sent = sent;
        out->fresh = h.n_fresh;
        out->stale = h.n_stale;
        out->rejected = h.n_rejected;
        out->version_after = h.V;
        out->max_delay = h.max_delay_seen;
        out->mean_delay = (h.n_fresh + h.n_stale) ? (double)h.delay_sum / (double)(h.n_fresh + h.n_stale) : 0.0;
    }
    CU(cudaGetLastError());
    return GORILA_OK;
}

gorila_status gorila_round(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                           const int32_t* staleness, gorila_learner_info* info_out, gorila_round_info* round_info_out,
                           uint8_t* synced_out) {
    return round_impl(ctx, learners, n, round, staleness, info_out, round_info_out, synced_out, true);
}

gorila_status gorila_round_async(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                                 const int32_t* staleness, gorila_learner_info* info_out,
                                 gorila_round_info* round_info_out, uint8_t* synced_out) {
    return round_impl(ctx, learners, n, round, staleness, info_out, round_info_out, synced_out, false);
}

gorila_status gorila_round_post(gorila_ctx* ctx, const int32_t* learners, int32_t n, uint64_t round,
                                const int32_t* staleness) {
    if (ctx && n > RING_MAXL) return fail(GORILA_E_SHAPE, "gorila_round_post: at most 32 learners per round");
    return round_impl(ctx, learners, n, round, staleness, nullptr, nullptr, nullptr, false, true);
}

gorila_status gorila_round_fetch(gorila_ctx* ctx, uint64_t round, gorila_learner_info* info_out,
                                 gorila_round_info* round_info_out, uint8_t* synced_out) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    const uint8_t* slot = ctx->ring_host + (size_t)(round % gorila_ctx::kRing) * ctx->ring_slot;
    const volatile uint64_t* seq = reinterpret_cast<const volatile uint64_t*>(slot);
    for (uint64_t spin = 0;; ++spin) {  // the posting stream writes the slot; poll it (no CUDA call)
        const uint64_t v = *seq;
        if (v == round + 1) break;
        if (v > round + 1) return fail(GORILA_E_INVALID, "gorila_round_fetch: result overwritten (fetch within 16 rounds)");
        __builtin_ia32_pause();  // keep the polled line cool for the device's write
        if ((spin & 0xfffff) == 0xfffff) {  // a failed stream would never write it: surface its error
            const cudaError_t e = cudaStreamQuery(ctx->stream);
            if (e != cudaSuccess && e != cudaErrorNotReady) CU(e);
            if (e == cudaSuccess && *seq != round + 1)
                return fail(GORILA_E_INVALID, "gorila_round_fetch: round was not posted");
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const uint32_t n = *reinterpret_cast<const uint32_t*>(slot + 8);
    if (round_info_out) memcpy(round_info_out, slot + 16, sizeof(gorila_round_info));
    if (synced_out) memcpy(synced_out, slot + 40, n);
    if (info_out) memcpy(info_out, slot + RING_HDR, sizeof(gorila_learner_info) * n);
    return GORILA_OK;
}

gorila_status gorila_get_state(gorila_ctx* ctx, float* theta, float* m, float* v, uint64_t* version) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    cudaStream_t st = ctx->stream;
    const int64_t P = ctx->P;
    struct Item { const float* src_slice; float* dst; bool full; } items[3] = {
        {ctx->theta, theta, true}, {ctx->m, m, false}, {ctx->v, v, false}};
    for (auto& it : items) {
        if (!it.dst) continue;
        if (it.full && ctx->p2p && ctx->W > 1) {  // each rank holds only its own fp32 slice: gather them
            CU(cudaStreamSynchronize(st));
            for (int q = 0; q < ctx->W; ++q)
                CU(cudaMemcpyAsync(ctx->tmp_int + (int64_t)q * ctx->q, peer_ptr(ctx, q, ctx->theta) + (int64_t)q * ctx->q,
                                   sizeof(float) * ctx->q, cudaMemcpyDefault, st));
        } else if (it.full) {
            CU(cudaMemcpyAsync(ctx->tmp_int, it.src_slice, sizeof(float) * ctx->W * ctx->q, cudaMemcpyDeviceToDevice, st));
        } else {  // own slice only; other slices zero
            CU(cudaMemsetAsync(ctx->tmp_int, 0, sizeof(float) * ctx->W * ctx->q, st));
            CU(cudaMemcpyAsync(ctx->tmp_int + (int64_t)ctx->rank * ctx->q, it.src_slice, sizeof(float) * ctx->q,
                               cudaMemcpyDeviceToDevice, st));
        }
        k_convert<<<148 * 4, 256, 0, st>>>(ctx->tmp_int, ctx->tmp_canon, P, 1);
        ctx->launches++;
        CU(cudaMemcpyAsync(it.dst, ctx->tmp_canon, sizeof(float) * P, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    if (version) CU(cudaMemcpy(version, ctx->V, sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return GORILA_OK;
}

gorila_status gorila_set_state(gorila_ctx* ctx, const float* theta, const float* m, const float* v, uint64_t version) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    cudaStream_t st = ctx->stream;
    const int64_t P = ctx->P;
    struct Item { const float* src; float* dst_slice; bool full; } items[3] = {
        {theta, ctx->theta, true}, {m, ctx->m, false}, {v, ctx->v, false}};
    for (auto& it : items) {
        if (!it.src) continue;
        CU(cudaMemcpyAsync(ctx->tmp_canon, it.src, sizeof(float) * P, cudaMemcpyHostToDevice, st));
        CU(cudaMemsetAsync(ctx->tmp_int, 0, sizeof(float) * ctx->W * ctx->q, st));
        k_convert<<<148 * 4, 256, 0, st>>>(ctx->tmp_canon, ctx->tmp_int, P, 0);
        ctx->launches++;
        if (it.full)
            CU(cudaMemcpyAsync(it.dst_slice, ctx->tmp_int, sizeof(float) * ctx->W * ctx->q, cudaMemcpyDeviceToDevice, st));
        else
            CU(cudaMemcpyAsync(it.dst_slice, ctx->tmp_int + (int64_t)ctx->rank * ctx->q, sizeof(float) * ctx->q,
                               cudaMemcpyDeviceToDevice, st));
        CU(cudaStreamSynchronize(st));
    }
    launch(ctx, k_set_u64, dim3(1), dim3(1), 0, ctx->V, version);
    // every replica slot = the new theta (teacher forcing restarts the history)
    for (int h = 0; h < ctx->H; ++h) {
        gorila_status s = pack_any(ctx, ctx->theta, ctx->rep_t[h], ctx->rep_f[h], nullptr, ctx->Vhist + h);
        if (s != GORILA_OK) return s;
    }
    CU(cudaStreamSynchronize(st));
    return GORILA_OK;
}

gorila_status gorila_get_learner_state(gorila_ctx* ctx, int32_t learner, float* theta_minus, double* stats4) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    cudaStream_t st = ctx->stream;
    Learner& l = ctx->learners[learner];
    CU(cudaStreamSynchronize(st));
    if (stats4) {
        LearnerStats h;
        CU(cudaMemcpy(&h, l.stats, sizeof(h), cudaMemcpyDeviceToHost));
        stats4[0] = h.mu; stats4[1] = h.var; stats4[2] = (double)h.count; stats4[3] = (double)h.last_sync;
    }
    if (theta_minus) {
        // unpack the fwd replica (T) + fp32 area back to canonical fp32 on the host
        const ReplicaLayout& R = ctx->rl;
        std::vector<uint8_t> t(R.n_t * ctx->esz);
        std::vector<float> f(R.n_f);
        CU(cudaMemcpy(t.data(), l.tminus_t, t.size(), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(f.data(), l.tminus_f, f.size() * sizeof(float), cudaMemcpyDeviceToHost));
        auto tval = [&](int64_t e) -> float {
            if (ctx->esz == 4) { float x; memcpy(&x, t.data() + e * 4, 4); return x; }
            uint16_t h; memcpy(&h, t.data() + e * 2, 2); uint32_t bits = (uint32_t)h << 16; float x; memcpy(&x, &bits, 4); return x;
        };
        for (int64_t i = 0; i < ctx->P; ++i) {
            float w;
            if (i < OFF_B1) w = tval(R.w1 + i);
            else if (i < OFF_W2) w = f[R.b1 + i - OFF_B1];
            else if (i < OFF_B2) w = tval(R.w2 + i - OFF_W2);
            else if (i < OFF_W3) w = f[R.b2 + i - OFF_B2];
            else if (i < OFF_B3) w = tval(R.w3 + i - OFF_W3);
            else if (i < OFF_W4) w = f[R.b3 + i - OFF_B3];
            else if (i < OFF_B4) w = tval(R.w4 + i - OFF_W4);
            else if (i < OFF_W5) w = f[R.b4 + i - OFF_B4];
            else w = f[R.w5 + i - OFF_W5];
            theta_minus[canon_of_internal(i)] = w;
        }
    }
    return GORILA_OK;
}

gorila_status gorila_set_learner_state(gorila_ctx* ctx, int32_t learner, const float* theta_minus,
                                       const double* stats4) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    cudaStream_t st = ctx->stream;
    Learner& l = ctx->learners[learner];
    if (stats4) {
        LearnerStats h{};
        h.mu = stats4[0]; h.var = stats4[1]; h.count = (uint32_t)stats4[2]; h.last_sync = (uint64_t)stats4[3];
        CU(cudaMemcpyAsync(l.stats, &h, sizeof(h), cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    }
    if (theta_minus) {
        CU(cudaMemcpyAsync(ctx->tmp_canon, theta_minus, sizeof(float) * ctx->P, cudaMemcpyHostToDevice, st));
        CU(cudaMemsetAsync(ctx->tmp_int, 0, sizeof(float) * ctx->W * ctx->q, st));
        k_convert<<<148 * 4, 256, 0, st>>>(ctx->tmp_canon, ctx->tmp_int, ctx->P, 0);
        ctx->launches++;
        if ((s = pack_any(ctx, ctx->tmp_int, l.tminus_t, l.tminus_f, nullptr, nullptr)) != GORILA_OK) return s;
        CU(cudaStreamSynchronize(st));
    }
    return GORILA_OK;
}

gorila_status gorila_get_grad(gorila_ctx* ctx, float* g) {
    if (!ctx || !g) return fail(GORILA_E_INVALID, "null argument");
    cudaStream_t st = ctx->stream;
    const float* src = ctx->G;
    if (ctx->per_msg && ctx->L > 1) {  // the sum over this rank's learners (as the aggregate mode's G)
        const int64_t n = (int64_t)ctx->W * ctx->q;
        std::vector<float> acc(n, 0.f), one(n);
        CU(cudaStreamSynchronize(st));
        for (int j = 0; j < ctx->L; ++j) {
            CU(cudaMemcpy(one.data(), ctx->G_all + (int64_t)j * n, sizeof(float) * n, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < n; ++i) acc[i] += one[i];
        }
        // on the library stream: a pageable cudaMemcpy may return before its DMA lands, and the
        // (non-blocking) library stream would not wait for it
        CU(cudaMemcpyAsync(ctx->tmp_int, acc.data(), sizeof(float) * n, cudaMemcpyHostToDevice, st));
        src = ctx->tmp_int;
    }
    k_convert<<<148 * 4, 256, 0, st>>>(src, ctx->tmp_canon, ctx->P, 1);
    ctx->launches++;
    CU(cudaMemcpyAsync(g, ctx->tmp_canon, sizeof(float) * ctx->P, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return GORILA_OK;
}

gorila_status gorila_act(gorila_ctx* ctx, const uint8_t* states, int32_t n, uint64_t global_step,
                        uint64_t actor_id, double eps_final, int64_t anneal_steps, int32_t states_on_device,
                        int32_t* actions_out, float* q_out) {
    if (!ctx || !states || !actions_out) return fail(GORILA_E_INVALID, "null argument");
    if (ctx->poisoned) return fail(GORILA_E_INVALID, "context poisoned");
    if (n < 1 || n > ctx->B) return fail(GORILA_E_SHAPE, "n must be in [1, batch]");
    cudaStream_t st = ctx->stream;
    const size_t sbytes = (size_t)n * NSTACK * FRAME_BYTES;
    const uint8_t* src = states;
    if (!states_on_device) {  // land the u8 states in the s' staging buffer: B * 4 * 7056 * sizeof(T) >= sbytes
        static_assert(NSTACK * FRAME_BYTES > 0, "");
        CU(cudaMemcpyAsync(ctx->s2, states, sbytes, cudaMemcpyHostToDevice, st));
        src = reinterpret_cast<const uint8_t*>(ctx->s2);
    } else if (ctx->u8 && ((uintptr_t)states & 15u)) {  // the u8 path bulk-copies frames: 16-B aligned
        CU(cudaMemcpyAsync(ctx->s2, states, sbytes, cudaMemcpyDeviceToDevice, st));
        src = reinterpret_cast<const uint8_t*>(ctx->s2);
    }
    const bool fp32 = ctx->cfg.math == GORILA_MATH_FP32;
    const int64_t total = (int64_t)n * (FRAME_BYTES / 4);
    const int grid = (int)std::min<int64_t>(148 * 8, (total + 255) / 256);
    if (fp32) launch(ctx, k_stage_states<float>, dim3(grid), dim3(256), 0, src, n, (float*)ctx->s);
    else if (ctx->u8) launch(ctx, k_act_desc, dim3((ctx->B + 255) / 256), dim3(256), 0, src, n, ctx->B, ctx->sdesc);
    else launch(ctx, k_stage_states<__nv_bfloat16>, dim3(grid), dim3(256), 0, src, n, (__nv_bfloat16*)ctx->s);
    // the forward phases of a learner step on the latest replica (slot of round dev_round_expect)
    const uint32_t fwd = (1u << PH_CONV1F) | (1u << PH_CONV2F) | (1u << PH_CONV3F) | (1u << PH_FC4F);
    const uint64_t rnd = ctx->dev_round_expect == ~0ull ? 0 : ctx->dev_round_expect;
    gorila_status s = fp32 ? run_learner<float>(ctx, 0, rnd, 0, 0, fwd) : run_learner<__nv_bfloat16>(ctx, 0, rnd, 0, 0, fwd);
    if (s != GORILA_OK) return s;
    const int slot = (int)(rnd % (uint64_t)ctx->H);
    const float* rf = ctx->rep_f[slot];
    const double eps = anneal_steps <= 0 || (int64_t)global_step >= anneal_steps
                           ? eps_final
                           : 1.0 - (1.0 - eps_final) * ((double)global_step / (double)anneal_steps);
    const uint2 key = make_uint2((uint32_t)ctx->cfg.seed, (uint32_t)(ctx->cfg.seed >> 32));
    int32_t* dact = reinterpret_cast<int32_t*>(ctx->sidx);  // learner scratch (rewritten by the sampler)
    float* dq = ctx->dQ;                                     // learner scratch [B][nA]
    launch(ctx, k_act_head, dim3(n), dim3(256), 0, (const float*)ctx->a4, rf + ctx->rl.w5, rf + ctx->rl.b5, ctx->nA,
           global_step, (uint32_t)actor_id, key, eps, dact, dq);
    CU(cudaMemcpyAsync(actions_out, dact, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    if (q_out) CU(cudaMemcpyAsync(q_out, dq, sizeof(float) * n * ctx->nA, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return GORILA_OK;
}

gorila_status gorila_get_activation(gorila_ctx* ctx, int32_t which, void* host, uint64_t bytes) {
    if (!ctx || !host) return fail(GORILA_E_INVALID, "null argument");
    const uint64_t B = ctx->B, e = ctx->esz;
    const void* src = nullptr;
    uint64_t n = 0;
    switch (which) {
        case 0: src = ctx->s; n = B * IMG * IMG * NSTACK * e; break;
        case 1: src = ctx->a1; n = B * H1 * H1 * C1_OUT * e; break;
        case 2: src = ctx->a2; n = B * H2 * H2 * C2_OUT * e; break;
        case 3: src = ctx->a3; n = B * H3 * H3 * C3_OUT * e; break;
        case 4: src = ctx->a4; n = B * FC4_OUT * 4; break;
        case 5: src = ctx->g1; n = B * H1 * H1 * C1_OUT * e; break;
        case 6: src = ctx->g2; n = B * H2 * H2 * C2_OUT * e; break;
        case 7: src = ctx->g3; n = B * H3 * H3 * C3_OUT * e; break;
        case 8: src = ctx->g4; n = B * FC4_OUT * e; break;
        default: return fail(GORILA_E_RANGE, "which must be in [0, 8]");
    }
    if (bytes != n) return fail(GORILA_E_SHAPE, "bytes must be " + std::to_string(n));
    CU(cudaStreamSynchronize(ctx->stream));
    if (which == 0 && ctx->u8) {  // u8 path: gathered from the ring (row-phase-major u8), as bf16 NHWC
        k_stage_from_desc<<<148 * 4, 256, 0, ctx->stream>>>(ctx->sdesc, (int)B, (uint8_t*)ctx->s);
        CU(cudaStreamSynchronize(ctx->stream));
        std::vector<uint8_t> st((size_t)B * FRAME_BYTES * NSTACK);
        CU(cudaMemcpy(st.data(), ctx->s, st.size(), cudaMemcpyDeviceToHost));
        uint16_t* out = static_cast<uint16_t*>(host);
        for (uint64_t b = 0; b < B; ++b)
            for (int y = 0; y < IMG; ++y)
                for (int x = 0; x < IMG; ++x)
                    for (int c = 0; c < NSTACK; ++c) {
                        const uint8_t u = st[b * FRAME_BYTES * NSTACK +
                                             ((((y & 3) * 21 + (y >> 2)) * 21 + (x >> 2)) * 16) + (x & 3) * 4 + c];
                        const float f = (float)u;
                        uint32_t bits;
                        memcpy(&bits, &f, 4);
                        out[((b * IMG + y) * IMG + x) * NSTACK + c] = (uint16_t)(bits >> 16);
                    }
        return GORILA_OK;
    }
    CU(cudaMemcpy(host, src, n, cudaMemcpyDeviceToHost));
    return GORILA_OK;
}

gorila_status gorila_capture_activations(gorila_ctx* ctx, int32_t enable) {
    if (!ctx) return fail(GORILA_E_INVALID, "null context");
    if (enable && !ctx->cap_buf) {
        const size_t e = ctx->esz, Bs = (size_t)ctx->B;
        const size_t per = Bs * (A1 + A2 + A3) * e + Bs * A4 * 4;
        CU(cudaMalloc((void**)&ctx->cap_buf, per * (size_t)ctx->L));
    }
    ctx->cap_acts = enable != 0;
    // the cached round graphs were captured without (or with) the copies: re-capture
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    ctx->graphs.clear();
    ctx->graph_kernels.clear();
    ctx->graph_seen.clear();
    return GORILA_OK;
}

gorila_status gorila_get_learner_activation(gorila_ctx* ctx, int32_t learner, int32_t which, void* host,
                                            uint64_t bytes) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    if (!host) return fail(GORILA_E_INVALID, "null argument");
    if (!ctx->cap_acts) return fail(GORILA_E_INVALID, "activation capture is off (gorila_capture_activations)");
    if (which < 1 || which > 4) return fail(GORILA_E_RANGE, "which must be in [1, 4]");
    const uint64_t e = ctx->esz, Bs = (uint64_t)ctx->B;
    const uint64_t n[4] = {Bs * A1 * e, Bs * A2 * e, Bs * A3 * e, Bs * A4 * 4};
    uint64_t off = (uint64_t)learner * (n[0] + n[1] + n[2] + n[3]);
    for (int i = 1; i < which; ++i) off += n[i - 1];
    if (bytes != n[which - 1]) return fail(GORILA_E_SHAPE, "bytes must be " + std::to_string(n[which - 1]));
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(host, ctx->cap_buf + off, bytes, cudaMemcpyDeviceToHost));
    return GORILA_OK;
}

gorila_status gorila_get_q(gorila_ctx* ctx, int32_t learner, float* q, float* qhat) {
    gorila_status s = check_learner(ctx, learner);
    if (s != GORILA_OK) return s;
    Learner& l = ctx->learners[learner];
    CU(cudaStreamSynchronize(ctx->stream));
    if (q) CU(cudaMemcpy(q, l.Q, sizeof(float) * ctx->B * ctx->nA, cudaMemcpyDeviceToHost));
    if (qhat) CU(cudaMemcpy(qhat, l.Qhat, sizeof(float) * ctx->B * ctx->nA, cudaMemcpyDeviceToHost));
    return GORILA_OK;
}

}  // extern "C"
