// gemm.cuh — the contraction engine of the learner update.
//
// Every conv / FC layer of the Nature-DQN forward and backward (Eq.2)
// is one "implicit GEMM"  C[i][j] = sum_r A(i, r) * B(j, r)  whose operands are
// produced on the fly by a loader (im2col of an NHWC activation, a shifted output
// gradient for dgrad, a transposed read for wgrad, or a plain row-major matrix)
// and whose result goes through a fused epilogue (scale, bias, ReLU, ReLU-mask,
// bf16 rounding, transposed gradient store, split-K partials).
//
// Two engines share the loaders / epilogues:
//   gemm_tc   — sm_100a tensor cores: bf16 operands staged in shared memory in the
//               UMMA canonical K-major layout, tcgen05.mma (M=128, N=BN, K=16) issued
//               by one thread, fp32 accumulator in TMEM, tcgen05.commit -> mbarrier
//               pipeline (2 smem stages + register prefetch), tcgen05.ld epilogue.
//   gemm_simt — fp32 FFMA tiles for the fp32 check mode (parity 1e-5).
#pragma once
#include "common.cuh"

namespace gorila {

// ====================================================================== loaders
// value(i, r); out of range -> 0. load8: 8 consecutive r (r0 % 8 == 0) as bf16x8.

template <typename T>
struct LdRows {  // X[i][r], row-major with leading dimension ld
    const T* x;
    int64_t ld;
    int rows, cols;
    GORILA_DEV float load(int i, int r) const { return (i < rows && r < cols) ? tof(x[(int64_t)i * ld + r]) : 0.f; }
    GORILA_DEV uint4 load8(int i, int r0) const {
        if (i >= rows || r0 >= cols) return make_uint4(0, 0, 0, 0);
        return *reinterpret_cast<const uint4*>(x + (int64_t)i * ld + r0);
    }
};

template <typename T>
struct LdRowsT {  // X[r][i] read transposed: value(i, r) = X[r * ld + i]
    const T* x;
    int64_t ld;
    int rows, cols;  // i extent, r extent
    GORILA_DEV float load(int i, int r) const { return (i < rows && r < cols) ? tof(x[(int64_t)r * ld + i]) : 0.f; }
    GORILA_DEV uint4 load8(int i, int r0) const {
        uint32_t w[4] = {0, 0, 0, 0};
        if (i < rows) {
            const unsigned short* p = reinterpret_cast<const unsigned short*>(x);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                int r = r0 + e;
                uint32_t h = (r < cols) ? (uint32_t)p[(int64_t)r * ld + i] : 0u;
                w[e >> 1] |= h << (16 * (e & 1));
            }
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};

// im2col of an NHWC input for a valid conv (k x k, stride s):
// value(i = (b, oy, ox), r = (ky*k + kx)*C + c) = in[b][oy*s+ky][ox*s+kx][c]
template <typename T>
struct LdConvIn {
    const T* in;
    int H, W, C, k, s, OH, OW, M, R;
    GORILA_DEV int64_t addr(int i, int r) const {
        int b = i / (OH * OW), p = i - b * (OH * OW), oy = p / OW, ox = p - oy * OW;
        int ky = r / (k * C), rem = r - ky * (k * C), kx = rem / C, c = rem - kx * C;
        return (((int64_t)b * H + oy * s + ky) * W + ox * s + kx) * C + c;
    }
    GORILA_DEV float load(int i, int r) const { return (i < M && r < R) ? tof(in[addr(i, r)]) : 0.f; }
    GORILA_DEV uint4 load8(int i, int r0) const {  // C % 8 == 0, or C == 4 (two adjacent pixels)
        if (i >= M || r0 >= R) return make_uint4(0, 0, 0, 0);
        return *reinterpret_cast<const uint4*>(in + addr(i, r0));
    }
};

// the same im2col read transposed (wgrad operand): value(i = r, red = m)
template <typename T>
struct LdConvInT {
    LdConvIn<T> f;
    GORILA_DEV float load(int i, int m) const { return f.load(m, i); }
    GORILA_DEV uint4 load8(int i, int m0) const {
        uint32_t w[4] = {0, 0, 0, 0};
        if (i < f.R) {
            const unsigned short* p = reinterpret_cast<const unsigned short*>(f.in);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                int m = m0 + e;
                uint32_t h = (m < f.M) ? (uint32_t)p[f.addr(m, i)] : 0u;
                w[e >> 1] |= h << (16 * (e & 1));
            }
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};

// conv dgrad operand: the output gradient g (NHWC [B][OH][OW][Co]) seen from input position
// i = (b, y, x), r = (ky*k + kx)*Co + o:  g[b][(y-ky)/s][(x-kx)/s][o] if that position exists, else 0
template <typename T>
struct LdDgrad {
    const T* g;
    int H, W, Co, k, s, OH, OW, M, R;
    GORILA_DEV int64_t addr(int i, int r) const {  // -1 if the tap does not exist
        int b = i / (H * W), p = i - b * (H * W), y = p / W, x = p - y * W;
        int ky = r / (k * Co), rem = r - ky * (k * Co), kx = rem / Co, o = rem - kx * Co;
        int ty = y - ky, tx = x - kx;
        if (ty < 0 || tx < 0 || ty % s || tx % s) return -1;
        int oy = ty / s, ox = tx / s;
        if (oy >= OH || ox >= OW) return -1;
        return (((int64_t)b * OH + oy) * OW + ox) * Co + o;
    }
    GORILA_DEV float load(int i, int r) const {
        if (i >= M || r >= R) return 0.f;
        int64_t a = addr(i, r);
        return a < 0 ? 0.f : tof(g[a]);
    }
    GORILA_DEV uint4 load8(int i, int r0) const {
        if (i >= M || r0 >= R) return make_uint4(0, 0, 0, 0);
        int64_t a = addr(i, r0);
        return a < 0 ? make_uint4(0, 0, 0, 0) : *reinterpret_cast<const uint4*>(g + a);
    }
};

// ====================================================================== epilogues
// apply(i, j, v, split): v = fp32 accumulator of C[i][j] (of split `split`).

template <typename T>
struct EpAct {  // out[i][j] = round_T(act(v * scale + bias[j]))
    T* out;
    int64_t ld;
    const float* bias;
    float scale;
    int M, N, relu;
    GORILA_DEV void apply(int i, int j, float v, int) const {
        if (i >= M || j >= N) return;
        float z = v * scale + bias[j];
        if (relu) z = fmaxf(z, 0.f);
        out[(int64_t)i * ld + j] = fromf<T>(z);
    }
};

template <typename T>
struct EpMask {  // out[i][j] = round_T(v * 1[act[i][j] > 0])  (ReLU' with ReLU'(0) = 0, reading R19)
    T* out;
    const T* act;
    int64_t ld;
    int M, N;
    GORILA_DEV void apply(int i, int j, float v, int) const {
        if (i >= M || j >= N) return;
        int64_t a = (int64_t)i * ld + j;
        out[a] = fromf<T>(tof(act[a]) > 0.f ? v : 0.f);
    }
};

template <typename T>
struct EpMaskT {  // transposed: out[j][i] = round_T(v * 1[act[j][i] > 0])
    T* out;
    const T* act;
    int64_t ld;
    int M, N;
    GORILA_DEV void apply(int i, int j, float v, int) const {
        if (i >= M || j >= N) return;
        int64_t a = (int64_t)j * ld + i;
        out[a] = fromf<T>(tof(act[a]) > 0.f ? v : 0.f);
    }
};

struct EpStoreT {  // dst[split][j][i] = v * scale (transposed fp32 store: weight-gradient partials)
    float* dst;
    int64_t ld, split_stride;
    float scale;
    int M, N;
    GORILA_DEV void apply(int i, int j, float v, int split) const {
        if (i >= M || j >= N) return;
        dst[split * split_stride + (int64_t)j * ld + i] = v * scale;
    }
};

struct EpStore {  // dst[split][i][j] = v (fp32 split-K partials)
    float* dst;
    int64_t ld, split_stride;
    int M, N;
    GORILA_DEV void apply(int i, int j, float v, int split) const {
        if (i >= M || j >= N) return;
        dst[split * split_stride + (int64_t)i * ld + j] = v;
    }
};

// ====================================================================== problem batch
template <typename LA, typename LB, typename EP>
struct GemmProb {
    LA a;
    LB b;
    EP ep;
};

template <typename LA, typename LB, typename EP>
struct GemmBatch {
    GemmProb<LA, LB, EP> prob[2];
    int M, N, R;   // shared by all problems of the batch
    int splits;    // split of the reduction range
    int chunks_per_split;  // in units of 64 (tc) / 16 (simt) reduction elements
};

// ====================================================================== tcgen05 engine
constexpr int TC_BM = 128, TC_BK = 64, TC_THREADS = 128;

__host__ __device__ constexpr uint32_t tmem_cols_for(int bn) {
    return bn <= 32 ? 32u : bn <= 64 ? 64u : bn <= 128 ? 128u : 256u;
}
__host__ __device__ constexpr int tc_smem_bytes(int bn) { return 2 * (TC_BM * TC_BK * 2 + bn * TC_BK * 2) + 64; }

// canonical K-major no-swizzle offset of (row, 16-byte k-chunk) inside a [rows][64] bf16 tile
GORILA_DEV uint32_t tc_off(int row, int kch) { return (uint32_t)((row >> 3) * 1024 + kch * 128 + (row & 7) * 16); }

template <int BN, typename LA, typename LB, typename EP>
__global__ void __launch_bounds__(TC_THREADS) gemm_tc(const __grid_constant__ GemmBatch<LA, LB, EP> p) {
    constexpr int A_BYTES = TC_BM * TC_BK * 2, B_BYTES = BN * TC_BK * 2;
    constexpr int A_ITERS = TC_BM * 8 / TC_THREADS, B_ITERS = BN * 8 / TC_THREADS;
    static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
    static_assert((BN * 8) % TC_THREADS == 0, "B tile split");
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;                        // [2][A_BYTES]
    uint8_t* sB = smem + 2 * A_BYTES;          // [2][B_BYTES]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 2 * (A_BYTES + B_BYTES));
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int prob = blockIdx.z / p.splits, split = blockIdx.z - prob * p.splits;
    const GemmProb<LA, LB, EP>& P = p.prob[prob];
    const int i0 = blockIdx.x * TC_BM, j0 = blockIdx.y * BN;
    const int n_chunks_total = (p.R + TC_BK - 1) / TC_BK;
    const int kc_begin = split * p.chunks_per_split;
    const int kc_end = min(n_chunks_total, kc_begin + p.chunks_per_split);
    const int nK = max(0, kc_end - kc_begin);

    if (warp == 0) tmem_alloc(tmem_slot, tmem_cols_for(BN));
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t IDESC = umma_idesc_bf16(TC_BM, BN);

    uint4 ra[A_ITERS], rb[B_ITERS];
    auto load_regs = [&](int kc) {
        const int r0 = (kc_begin + kc) * TC_BK;
#pragma unroll
        for (int q = 0; q < A_ITERS; ++q) {
            int idx = tid + TC_THREADS * q;
            int row = (idx >> 6) * 8 + (idx & 7), kch = (idx >> 3) & 7;
            ra[q] = P.a.load8(i0 + row, r0 + kch * 8);
        }
#pragma unroll
        for (int q = 0; q < B_ITERS; ++q) {
            int idx = tid + TC_THREADS * q;
            int row = (idx >> 6) * 8 + (idx & 7), kch = (idx >> 3) & 7;
            rb[q] = P.b.load8(j0 + row, r0 + kch * 8);
        }
    };

    if (nK > 0) load_regs(0);
    for (int kc = 0; kc < nK; ++kc) {
        const int s = kc & 1;
        if (kc >= 2) mbar_wait(&mbar[s], ((kc - 2) >> 1) & 1);  // MMAs of chunk kc-2 released stage s
        uint8_t* a_st = sA + s * A_BYTES;
        uint8_t* b_st = sB + s * B_BYTES;
#pragma unroll
        for (int q = 0; q < A_ITERS; ++q) {
            int idx = tid + TC_THREADS * q;
            int row = (idx >> 6) * 8 + (idx & 7), kch = (idx >> 3) & 7;
            *reinterpret_cast<uint4*>(a_st + tc_off(row, kch)) = ra[q];
        }
#pragma unroll
        for (int q = 0; q < B_ITERS; ++q) {
            int idx = tid + TC_THREADS * q;
            int row = (idx >> 6) * 8 + (idx & 7), kch = (idx >> 3) & 7;
            *reinterpret_cast<uint4*>(b_st + tc_off(row, kch)) = rb[q];
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t a_base = smem_u32(a_st), b_base = smem_u32(b_st);
#pragma unroll
            for (int kk = 0; kk < TC_BK / 16; ++kk) {
                uint64_t ad = umma_desc(a_base + kk * 256, 128, 1024);
                uint64_t bd = umma_desc(b_base + kk * 256, 128, 1024);
                umma_bf16(tmem, ad, bd, IDESC, (kc > 0 || kk > 0) ? 1u : 0u);
            }
            umma_commit(&mbar[s]);
        }
        if (kc + 1 < nK) load_regs(kc + 1);
    }
    if (nK > 0) {
        const int last = nK - 1;
        mbar_wait(&mbar[last & 1], (last >> 1) & 1);
        if (last >= 1) mbar_wait(&mbar[(last - 1) & 1], ((last - 1) >> 1) & 1);
    }
    tc_fence_after();

    // epilogue: warp w owns TMEM lanes (= rows) 32w .. 32w+31
    const int row = i0 + warp * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16];
        if (nK > 0) {
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) P.ep.apply(row, j0 + c0 + e, v[e], split);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols_for(BN));
}

// ====================================================================== fp32 SIMT engine
constexpr int SM_BI = 64, SM_BJ = 64, SM_BR = 16;

template <typename LA, typename LB, typename EP>
__global__ void __launch_bounds__(256) gemm_simt(const __grid_constant__ GemmBatch<LA, LB, EP> p) {
    __shared__ float As[SM_BR][SM_BI + 4];
    __shared__ float Bs[SM_BR][SM_BJ + 4];
    const int tid = threadIdx.x;
    const int prob = blockIdx.z / p.splits, split = blockIdx.z - prob * p.splits;
    const GemmProb<LA, LB, EP>& P = p.prob[prob];
    const int i0 = blockIdx.x * SM_BI, j0 = blockIdx.y * SM_BJ;
    const int r_begin = split * p.chunks_per_split * SM_BR;
    const int r_end = min(p.R, r_begin + p.chunks_per_split * SM_BR);
    const int ti = tid & 15, tj = tid >> 4;
    float acc[4][4] = {};
    for (int r0 = r_begin; r0 < r_end; r0 += SM_BR) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int idx = tid + 256 * q;
            int ii = idx & 63, rr = idx >> 6;
            int r = r0 + rr;
            As[rr][ii] = (r < r_end) ? P.a.load(i0 + ii, r) : 0.f;
            Bs[rr][ii] = (r < r_end) ? P.b.load(j0 + ii, r) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int rr = 0; rr < SM_BR; ++rr) {
            float av[4], bv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                av[q] = As[rr][ti + 16 * q];
                bv[q] = Bs[rr][tj + 16 * q];
            }
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) P.ep.apply(i0 + ti + 16 * x, j0 + tj + 16 * y, acc[x][y], split);
}

}  // namespace gorila
