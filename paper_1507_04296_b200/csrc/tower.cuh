// tower.cuh — the three conv layers of one (net, sample) in one CTA (small batches).
//
// At B = 32 each conv layer is a separate latency-bound launch (one sample per CTA, a handful of
// K-chunks). Here one CTA runs conv1 -> conv2 -> conv3 for one sample of one net, with the
// activations handed from layer to layer in shared memory, already in the next layer's
// shifted-window operand layout (shift_gemm.cuh): conv1's epilogue writes a1 into conv2's four
// stride-phase planes (64-B rows, SWIZZLE_64B applied by hand), conv2's epilogue writes a2 into
// conv3's flat 128-B rows (SWIZZLE_128B by hand); a fence.proxy.async makes those generic-proxy
// stores visible to the tensor core. a1, a2, a3 also go to global memory (the backward reads them).
// The weights of all three layers (152 KB, bf16, per-chunk TMA boxes with their own mbarriers)
// and the sample's conv1 input planes arrive by TMA at the start.
// Warp 0: TMA; warp 1: tcgen05.mma issuer; warps 2..9: epilogues (TMEM lanes 32*(w%4).., warps
// 2..5 the first half of each layer's columns, 6..9 the second). conv1 is committed per M-block:
// the epilogue of block mb (TMEM -> bias, ReLU, bf16 -> global) runs under the MMAs of mb+1 and
// keeps its packed a1 in registers; the scatter into conv2's planes (which overlap the conv1 input
// planes) waits for the last block.
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "layout.cuh"
#include "shift_gemm.cuh"

namespace gorila {

struct TowerNet {
    alignas(64) CUtensorMap s_map;   // conv1 input row phases (as ShConv1Fwd)
    alignas(64) CUtensorMap w1_map;  // (256, 32), box (16, 32), SWIZZLE_32B   (ShWeightK<32, 32, 16, 2>)
    alignas(64) CUtensorMap w2_map;  // (512, 64), box (32, 64), SWIZZLE_64B   (ShWeightK<64, 64, 16, 1>)
    alignas(64) CUtensorMap w3_map;  // (576, 64), box (64, 64), SWIZZLE_128B  (ShWeightK<64, 128, 9, 0>)
    __nv_bfloat16 *a1, *a2, *a3;     // global outputs (NHWC)
    const float *b1, *b2, *b3;
};
struct TowerParams {
    TowerNet net[2];
    float in_scale;
    int batch;
};

namespace tower {
// shared memory carve (1024-aligned offsets)
constexpr int W1_OFF = 0, W1_CH = 1024;             // 16 chunks [32 co][32 B]
constexpr int W2_OFF = 16 * 1024, W2_CH = 4096;     // 16 chunks [64 co][64 B]
constexpr int W3_OFF = 80 * 1024, W3_CH = 8192;     // 9 chunks  [64 co][128 B]
constexpr int A_OFF = 152 * 1024;                   // s planes (4 x 17408) / later a1 planes + a2
constexpr int S_PLANE = ShConv1Fwd<1>::PLANE;       // 17408
constexpr int A1_PLANE = ShConv2Fwd::PLANE;         // 9216: 144 rows x 64 B
constexpr int A2_OFF = A_OFF + 4 * A1_PLANE;        // 148 rows x 128 B
constexpr int A2_BYTES = 19456;
constexpr int BAR_OFF = A_OFF + 4 * S_PLANE;        // 221184
constexpr int NB_W = 16 + 16 + 9;
constexpr int NB_ACC = 6;                           // conv1 per M-block [0, 4), conv2 [4], conv3 [5]
constexpr int BIAS_OFF = BAR_OFF + 8 * (NB_W + 12);  // 160 floats: b1, b2, b3
constexpr int THREADS = 320;
constexpr int SMEM = BIAS_OFF + 160 * 4 + 1024;
static_assert(A2_OFF + A2_BYTES <= BAR_OFF, "a1 / a2 fit in the s-plane region");
}  // namespace tower

// trace build: clock64 of CTA (0, 0) at the tower's hand-off points (slots 48.., tools/trace_tower.py)
#ifdef GORILA_TRACE
#define TTRACE(slot)                                                        \
    do {                                                                    \
        if (blockIdx.x == 0 && blockIdx.y == 0) {                           \
            unsigned long long t_;                                          \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));              \
            gorila_trace_buf[(slot)] = t_;                                  \
        }                                                                   \
    } while (0)
#else
#define TTRACE(slot) \
    do {             \
    } while (0)
#endif

// swizzled 16-B store: logical byte offset o inside a region aligned to the swizzle atom;
// SWIZZLE_{32,64,128}B XOR address bits [4, 4+b) with bits [7, 7+b), b = 1, 2, 3
GORILA_DEV void st_swz16(uint8_t* region, uint32_t o, int b, uint4 v) {
    const uint32_t mask = (1u << b) - 1u;
    const uint32_t po = o ^ (((o >> 7) & mask) << 4);
    *reinterpret_cast<uint4*>(region + po) = v;
}

__global__ void __launch_bounds__(tower::THREADS) k_conv_tower(const __grid_constant__ TowerParams p) {
    using namespace tower;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* w_full = reinterpret_cast<uint64_t*>(sm + BAR_OFF);  // [41] weight chunks
    uint64_t* s_full = w_full + NB_W;                               // conv1 input planes
    uint64_t* acc_full = s_full + 1;                                // [NB_ACC] MMA -> epilogue
    uint64_t* act_ready = acc_full + NB_ACC;                        // [2] a1 / a2 in smem (epilogue -> MMA)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_ready + 2);
    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    const int z = blockIdx.y, b = blockIdx.x;
    const TowerNet& N = p.net[z];

    if (warp == 0) tmem_alloc(tmem_slot, 256);
    // rows of the s planes past the 441 loaded ones are read by dropped output rows only
    for (int q = 0; q < 4; ++q)
        for (int o = 441 * 32 + tid * 16; o < S_PLANE; o += THREADS * 16)
            *reinterpret_cast<uint4*>(sm + A_OFF + q * S_PLANE + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid == 32) {
        // act_ready[0]: 256 epilogue threads + warp 0 (which zeroes the operand tails); [1]: 256
        const int n_bar = NB_W + 1 + NB_ACC + 2;
        for (int i = 0; i < n_bar; ++i) mbar_init(&w_full[i], i == n_bar - 2 ? 288 : i == n_bar - 1 ? 256 : 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_nu = *tmem_slot, base_nu = smem_u32(sm);
    const uint32_t tmem = tmem_nu, base = base_nu;
    float* s_bias = reinterpret_cast<float*>(sm + BIAS_OFF);
    // The weights (this round's replica / theta^-) were written by the previous round's apply and
    // target sync, two or more kernels back: with PDL those are complete when this grid starts
    // (the kernel just before has passed its own griddepcontrol.wait), so they stream in while the
    // sampler finishes. Only the sample's planes wait for the sampler.
    if (warp == 0 && lane == 0) {
        for (int c = 0; c < 16; ++c) {
            tma_load(&N.w1_map, base + W1_OFF + c * W1_CH, &w_full[c], ShWeightK<32, 32, 16, 2>::koff(c), 0);
            mbar_expect_tx(&w_full[c], 32 * 32);
        }
        for (int c = 0; c < 16; ++c) {
            tma_load(&N.w2_map, base + W2_OFF + c * W2_CH, &w_full[16 + c], ShWeightK<64, 64, 16, 1>::koff(c), 0);
            mbar_expect_tx(&w_full[16 + c], 64 * 64);
        }
        for (int c = 0; c < 9; ++c) {
            tma_load(&N.w3_map, base + W3_OFF + c * W3_CH, &w_full[32 + c], c * 64, 0);
            mbar_expect_tx(&w_full[32 + c], 64 * 128);
        }
    }
    pdl_wait();
    pdl_trigger();
    if (tid == 0) TTRACE(48);
    if (warp == 0) {
        if (lane == 0) {  // the sample's conv1 input planes
#pragma unroll
            for (int q = 0; q < 4; ++q) tma_load(&N.s_map, base + A_OFF + q * S_PLANE, s_full, 0, 0, q, b);
            mbar_expect_tx(s_full, 4 * 441 * 32);
        }
        // once conv1's MMAs are done the s planes are dead: zero the rows of the a1 planes and of
        // the a2 buffer that no output row writes (read only by dropped output rows)
        __syncwarp();
        mbar_wait(&acc_full[3], 0);  // the last conv1 block: every MMA reading the s planes is done
        for (int q = 0; q < 4; ++q)
            for (int o = 100 * 64 + lane * 16; o < A1_PLANE; o += 32 * 16)
                *reinterpret_cast<uint4*>(sm + A_OFF + q * A1_PLANE + o) = make_uint4(0, 0, 0, 0);
        for (int o = 81 * 128 + lane * 16; o < A2_BYTES; o += 32 * 16)
            *reinterpret_cast<uint4*>(sm + A2_OFF + o) = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
        mbar_arrive(&act_ready[0]);
    } else if (warp == 1) {
        {  // MMA issuer (warp-uniform): conv1 -> TMEM [0,128), conv2 -> [128,192), conv3 -> [192,256)
            const uint32_t tmem = uniform_u32(tmem_nu), base = uniform_u32(base_nu);
            constexpr uint32_t ID32 = umma_idesc_bf16(128, 32), ID64 = umma_idesc_bf16(128, 64);
            mbar_wait(s_full, 0);
            TTRACE(49);
            tc_fence_after();
            {
                const uint64_t ad0 = umma_desc_sw(base + A_OFF, 32), bd0 = umma_desc_sw(base + W1_OFF, 32);
#pragma unroll
                for (int mb = 0; mb < 4; ++mb) {
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        if (mb == 0) {
                            mbar_wait(&w_full[c], 0);
                            tc_fence_after();
                        }
                        const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
                        umma_bf16_w(tmem + mb * 32, ad0 + ((q * S_PLANE + (mb * 128 + dy * 21 + dx) * 32) >> 4),
                                  bd0 + ((c * W1_CH) >> 4), ID32, c > 0 ? 1u : 0u);
                    }
                    umma_commit_w(&acc_full[mb]);  // block mb's epilogue runs under the next block's MMAs
                }
                TTRACE(50);
            }
            mbar_wait(&act_ready[0], 0);  // a1 planes written by the epilogue warps
            TTRACE(51);
            tc_fence_after();
            {
                const uint64_t ad0 = umma_desc_sw(base + A_OFF, 64), bd0 = umma_desc_sw(base + W2_OFF, 64);
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    mbar_wait(&w_full[16 + c], 0);
                    tc_fence_after();
                    const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk)
                        umma_bf16_w(tmem + 128, ad0 + ((q * A1_PLANE + (dy * 10 + dx) * 64 + kk * 32) >> 4),
                                  bd0 + ((c * W2_CH + kk * 32) >> 4), ID64, (c > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit_w(&acc_full[4]);
                TTRACE(52);
            }
            mbar_wait(&act_ready[1], 0);  // a2 rows written
            TTRACE(53);
            tc_fence_after();
            {
                const uint64_t ad0 = umma_desc_sw(base + A2_OFF, 128), bd0 = umma_desc_sw(base + W3_OFF, 128);
#pragma unroll
                for (int c = 0; c < 9; ++c) {
                    mbar_wait(&w_full[32 + c], 0);
                    tc_fence_after();
                    const int ky = c / 3, kx = c - 3 * ky;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_bf16_w(tmem + 192, ad0 + (((ky * 9 + kx) * 128 + kk * 32) >> 4),
                                  bd0 + ((c * W3_CH + kk * 32) >> 4), ID64, (c > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit_w(&acc_full[5]);
                TTRACE(54);
            }
        }
    } else {  // epilogue warps 2..9
        const int quad = warp & 3, half = (warp - 2) >> 2, etid = tid - 64;  // etid 0..255
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
        for (int i = etid; i < 160; i += 256)  // the layers' biases, once (not per output element)
            s_bias[i] = i < 32 ? N.b1[i] : i < 96 ? N.b2[i - 32] : N.b3[i - 96];
        asm volatile("bar.sync 1, 256;" ::: "memory");  // the epilogue warps only
        const float* sb1 = s_bias + half * 16;
        const float* sb2 = s_bias + 32 + half * 32;
        const float* sb3 = s_bias + 96 + half * 32;
        // ---- conv1: a1 = bf16(ReLU(v / 255 + b1)), columns [16 half, 16 half + 16) -> global now,
        // -> conv2's phase planes once the last block's MMAs no longer read the s planes
        uint4 a1r[4][2];
#pragma unroll
        for (int mb = 0; mb < 4; ++mb) {
            mbar_wait(&acc_full[mb], 0);
            if (etid == 0 && mb == 0) TTRACE(55);
            tc_fence_after();
            const int m = mb * 128 + quad * 32 + lane, Y = m / 21, X = m - 21 * Y;
            const bool ok = m < 441 && Y < 20 && X < 20;
            float v[16];
            tmem_ld16(lane_base + (uint32_t)(mb * 32 + half * 16), v);
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float x0 = fmaxf(v[2 * e] * p.in_scale + sb1[2 * e], 0.f);
                const float x1 = fmaxf(v[2 * e + 1] * p.in_scale + sb1[2 * e + 1], 0.f);
                __nv_bfloat162 t = __floats2bfloat162_rn(x0, x1);
                w[e] = *reinterpret_cast<uint32_t*>(&t);
            }
            a1r[mb][0] = make_uint4(w[0], w[1], w[2], w[3]);
            a1r[mb][1] = make_uint4(w[4], w[5], w[6], w[7]);
            if (ok) {
                uint4* g = reinterpret_cast<uint4*>(N.a1 + ((int64_t)b * 400 + Y * 20 + X) * 32);
                g[2 * half] = a1r[mb][0];
                g[2 * half + 1] = a1r[mb][1];
            }
        }
#pragma unroll
        for (int mb = 0; mb < 4; ++mb) {
            const int m = mb * 128 + quad * 32 + lane, Y = m / 21, X = m - 21 * Y;
            if (m < 441 && Y < 20 && X < 20) {
                uint8_t* plane = sm + A_OFF + ((Y & 1) * 2 + (X & 1)) * A1_PLANE;
                const int prow = (Y >> 1) * 10 + (X >> 1);
                st_swz16(plane, prow * 64 + (2 * half) * 16, 2, a1r[mb][0]);
                st_swz16(plane, prow * 64 + (2 * half + 1) * 16, 2, a1r[mb][1]);
            }
        }
        fence_proxy_async_smem();  // generic-proxy smem stores -> visible to tcgen05.mma
        tc_fence_before();
        if (etid == 0) TTRACE(56);
        mbar_arrive(&act_ready[0]);
        // ---- conv2: a2 -> global and conv3's flat rows (columns [32 half, 32 half + 32))
        mbar_wait(&acc_full[4], 0);
        if (etid == 0) TTRACE(57);
        tc_fence_after();
        {
            const int r = quad * 32 + lane, Y = r / 10, X = r - 10 * Y;
            const bool ok = r < 100 && Y < 9 && X < 9;
            __nv_bfloat16* g = N.a2 + ((int64_t)b * 81 + Y * 9 + X) * 64;
            const int frow = Y * 9 + X;
            float v[32];
            tmem_ld16x2(lane_base + (uint32_t)(128 + half * 32), v);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int h = 2 * half + hh;
                if (!ok) continue;
                uint32_t w[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float x0 = fmaxf(v[hh * 16 + 2 * e] + sb2[hh * 16 + 2 * e], 0.f);
                    const float x1 = fmaxf(v[hh * 16 + 2 * e + 1] + sb2[hh * 16 + 2 * e + 1], 0.f);
                    __nv_bfloat162 t = __floats2bfloat162_rn(x0, x1);
                    w[e] = *reinterpret_cast<uint32_t*>(&t);
                }
                const uint4 u0 = make_uint4(w[0], w[1], w[2], w[3]), u1 = make_uint4(w[4], w[5], w[6], w[7]);
                reinterpret_cast<uint4*>(g)[2 * h] = u0;
                reinterpret_cast<uint4*>(g)[2 * h + 1] = u1;
                st_swz16(sm + A2_OFF, frow * 128 + (2 * h) * 16, 3, u0);
                st_swz16(sm + A2_OFF, frow * 128 + (2 * h + 1) * 16, 3, u1);
            }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        if (etid == 0) TTRACE(58);
        mbar_arrive(&act_ready[1]);
        // ---- conv3: a3 -> global
        mbar_wait(&acc_full[5], 0);
        if (etid == 0) TTRACE(59);
        tc_fence_after();
        {
            const int r = quad * 32 + lane, y = r / 9, x = r - 9 * y;
            const bool ok = r < 81 && y < 7 && x < 7;
            __nv_bfloat16* g = N.a3 + ((int64_t)b * 49 + y * 7 + x) * 64;
            float v[32];
            tmem_ld16x2(lane_base + (uint32_t)(192 + half * 32), v);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int h = 2 * half + hh;
                if (!ok) continue;
                uint32_t w[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float x0 = fmaxf(v[hh * 16 + 2 * e] + sb3[hh * 16 + 2 * e], 0.f);
                    const float x1 = fmaxf(v[hh * 16 + 2 * e + 1] + sb3[hh * 16 + 2 * e + 1], 0.f);
                    __nv_bfloat162 t = __floats2bfloat162_rn(x0, x1);
                    w[e] = *reinterpret_cast<uint32_t*>(&t);
                }
                reinterpret_cast<uint4*>(g)[2 * h] = make_uint4(w[0], w[1], w[2], w[3]);
                reinterpret_cast<uint4*>(g)[2 * h + 1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
        }
    }
    if (tid == 64) TTRACE(60);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

}  // namespace gorila
