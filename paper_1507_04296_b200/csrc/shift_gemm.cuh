// shift_gemm.cuh — shifted-window implicit GEMM for the conv layers (forward and data gradient).
//
// A convolution output row m (one output pixel, laid out on a "virtual" grid as wide as the
// input rows) reads, for kernel tap (dy, dx), input row m + dy*W + dx of the same grid. So the
// layer input of a tile is loaded into shared memory ONCE (one TMA box, K-major swizzled rows of
// 128 / 64 / 32 bytes) and every reduction chunk (tap, or tap of a stride phase plane) is the same
// buffer read from a shifted start address: the swizzle is a function of the absolute address, so
// any whole-row shift is a valid UMMA operand (tools/umma_shift_probe.cu). Compared with one
// im2col box per chunk this removes the K*K-fold re-read of the input from L2 and most TMA
// requests. Rows of the virtual grid that are not output pixels are computed and dropped.
//
// Strided layers use phase planes: conv2 (stride 2) reads the four planes a1[2Y+py][2X+px]
// (64-B rows of 32 channels) with 2x2 taps each; conv1 (stride 4) reads the four row phases
// s[4Y+py][4X..4X+3] (32-B rows of 4 pixels x 4 channels) with 2x2 taps each; the stride-2 data
// gradient runs its four output phases as four M-blocks over one zero-padded gradient buffer.
//
// The weights of every chunk stay resident in shared memory for the whole (persistent) CTA.
// Warp roles as in gemm_tma_p: warp 0 lane 0 loads (weights once per problem, then the A
// buffers through a ring), warp 1 lane 0 issues tcgen05.mma into one of two TMEM accumulators,
// warps 2..5 run the epilogue.
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "layout.cuh"

namespace gorila {

// ---------------------------------------------------------------- A operands (input windows)
// Interface: RB (row bytes), NCHUNK, KSTEPS (16-element K steps per chunk), BUF (bytes of one A
// buffer, 1024-aligned), NPLANE / PLANE / WRITTEN (the buffer's planes and the bytes TMA writes
// into each: the rest is zeroed once), MS (a sample's M-blocks split over MS tiles),
// load(tile, dst, bar) -> bytes, mb0(tile) -> the tile's first global M-block, addr(base, c, mbg)
// -> start address of chunk c's rows for global M-block mbg, row(tile, mbg, r) -> output row or -1.

// conv3 forward (stride 1, 3x3 over 9x9x64): the flat pixel array [B*81][64]; tile = 128
// consecutive rows of it, buffer = 148 rows (the largest tap shift is 2*9+2 = 20).
struct ShConv3Fwd {
    static constexpr int RB = 128, NCHUNK = 9, KSTEPS = 4, ROWS = 148, BUF = (ROWS * RB + 1023) / 1024 * 1024;
    static constexpr int NPLANE = 1, PLANE = BUF, WRITTEN = ROWS * RB, MS = 1;
    alignas(64) CUtensorMap map;  // (64, B*81), box (64, 148), SWIZZLE_128B
    int batch;
    __host__ __device__ int ntiles() const { return (batch * 81 + 127) / 128; }
    GORILA_DEV int mb0(int) const { return 0; }
    GORILA_DEV uint32_t load(int t, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, 0, t * 128);
        return ROWS * RB;
    }
    GORILA_DEV uint32_t addr(uint32_t base, int c, int) const {
        const int ky = c / 3, kx = c - 3 * ky;
        return base + (ky * 9 + kx) * RB;
    }
    GORILA_DEV int row(int t, int, int r) const {
        const int m = t * 128 + r, b = m / 81, p = m - 81 * b, y = p / 9, x = p - 9 * y;
        return (b < batch && y < 7 && x < 7) ? b * 49 + y * 7 + x : -1;
    }
};

// conv3 data gradient (full 3x3 convolution of g3 7x7x64): per sample, g3 zero-padded by 2
// (an 11x11 box at (-2, -2)); output (y, x) in 9x9 at grid row y*11 + x reads tap (ky, kx) at
// row + (2-ky)*11 + (2-kx). Tail rows 121.. of the buffer stay zero (read by dropped rows only).
struct ShDgrad3 {
    static constexpr int RB = 128, NCHUNK = 9, KSTEPS = 4, ROWS = 152, BUF = (ROWS * RB + 1023) / 1024 * 1024;
    static constexpr int NPLANE = 1, PLANE = BUF, WRITTEN = 121 * RB, MS = 1;
    alignas(64) CUtensorMap map;  // (64, 7, 7, B), box (64, 11, 11, 1), SWIZZLE_128B
    int batch;
    __host__ __device__ int ntiles() const { return batch; }
    GORILA_DEV int mb0(int) const { return 0; }
    GORILA_DEV uint32_t load(int t, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, 0, -2, -2, t);
        return 121 * RB;
    }
    GORILA_DEV uint32_t addr(uint32_t base, int c, int) const {
        const int ky = c / 3, kx = c - 3 * ky;
        return base + ((2 - ky) * 11 + (2 - kx)) * RB;
    }
    GORILA_DEV int row(int t, int, int r) const {
        const int y = r / 11, x = r - 11 * y;
        return (r < 121 && y < 9 && x < 9) ? (t * 9 + y) * 9 + x : -1;
    }
};

// conv2 data gradient (stride-2 transposed 4x4 convolution of g2 9x9x64): per sample, g2 padded
// by one row / column on each side (an 11x11 box at (-1, -1)); the four output phases
// (py, px) = M-blocks: g1[2Y+py][2X+px] at grid row Y*11 + X reads tap (dy, dx) (kernel
// (2dy+py, 2dx+px)) at row + (1-dy)*11 + (1-dx).
// MS_ = 4: one phase per tile (small batches: four times the CTAs, the buffer loaded per phase).
template <int MS_>
struct ShDgrad2 {
    static constexpr int RB = 128, NCHUNK = 4, KSTEPS = 4, ROWS = 140, BUF = (ROWS * RB + 1023) / 1024 * 1024;
    static constexpr int NPLANE = 1, PLANE = BUF, WRITTEN = 121 * RB, MS = MS_;
    alignas(64) CUtensorMap map;  // (64, 9, 9, B), box (64, 11, 11, 1), SWIZZLE_128B
    int batch;
    __host__ __device__ int ntiles() const { return batch * MS; }
    GORILA_DEV int mb0(int t) const { return (t % MS) * (4 / MS); }
    GORILA_DEV uint32_t load(int t, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, 0, -1, -1, t / MS);
        return 121 * RB;
    }
    GORILA_DEV uint32_t addr(uint32_t base, int c, int) const {
        const int dy = c >> 1, dx = c & 1;
        return base + ((1 - dy) * 11 + (1 - dx)) * RB;
    }
    GORILA_DEV int row(int t, int mb, int r) const {
        const int Y = r / 11, X = r - 11 * Y;
        return (r < 121 && Y < 10 && X < 10) ? ((t / MS) * 20 + 2 * Y + (mb >> 1)) * 20 + 2 * X + (mb & 1) : -1;
    }
};

// conv2 forward (stride 2, 4x4 over 20x20x32): per sample the four phase planes
// P(py,px)[Y][X] = a1[2Y+py][2X+px] (10x10 rows of 64 B); chunk c = plane*4 + tap (dy, dx)
// (kernel (2dy+py, 2dx+px)) reads plane rows Y*10 + X + dy*10 + dx.
struct ShConv2Fwd {
    static constexpr int RB = 64, NCHUNK = 16, KSTEPS = 2, PROWS = 144, PLANE = PROWS * RB;  // 9216 B
    static constexpr int BUF = 4 * PLANE, NPLANE = 4, WRITTEN = 100 * RB, MS = 1;
    alignas(64) CUtensorMap map;  // (32, 20, 20, B), box (32, 10, 10, 1), es (1, 2, 2, 1), SWIZZLE_64B
    int batch;
    __host__ __device__ int ntiles() const { return batch; }
    GORILA_DEV int mb0(int) const { return 0; }
    GORILA_DEV uint32_t load(int t, uint32_t dst, uint64_t* bar) const {
#pragma unroll
        for (int q = 0; q < 4; ++q) tma_load(&map, dst + q * PLANE, bar, 0, q & 1, q >> 1, t);
        return 4 * 100 * RB;
    }
    GORILA_DEV uint32_t addr(uint32_t base, int c, int) const {
        const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
        return base + q * PLANE + (dy * 10 + dx) * RB;
    }
    GORILA_DEV int row(int t, int, int r) const {
        const int Y = r / 10, X = r - 10 * Y;
        return (r < 100 && Y < 9 && X < 9) ? t * 81 + Y * 9 + X : -1;
    }
};

// conv1 forward (stride 4, 8x8 over 84x84x4): per sample the four row phases
// Q(py)[Y][X] = s[4Y+py][4X .. 4X+3][0..3] (21x21 rows of 32 B); chunk c = py*4 + tap (dy, dx)
// (kernel rows 4dy+py, columns 4dx .. 4dx+3) reads rows Y*21 + X + dy*21 + dx. M = 4 blocks.
// MS_ > 1: a sample's four M-blocks split over MS_ tiles (small batches).
template <int MS_>
struct ShConv1Fwd {
    static constexpr int RB = 32, NCHUNK = 16, KSTEPS = 1, PROWS = 544, PLANE = PROWS * RB;  // 17408 B
    static constexpr int BUF = 4 * PLANE, NPLANE = 4, WRITTEN = 441 * RB, MS = MS_;
    alignas(64) CUtensorMap map;  // (16, 21, 84, B), box (16, 21, 84, 1), es (1, 1, 4, 1), SWIZZLE_32B
    int batch;
    __host__ __device__ int ntiles() const { return batch * MS; }
    GORILA_DEV int mb0(int t) const { return (t % MS) * (4 / MS); }
    GORILA_DEV uint32_t load(int t, uint32_t dst, uint64_t* bar) const {
#pragma unroll
        for (int q = 0; q < 4; ++q) tma_load(&map, dst + q * PLANE, bar, 0, 0, q, t / MS);
        return 4 * 441 * RB;
    }
    GORILA_DEV uint32_t addr(uint32_t base, int c, int mb) const {
        const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
        return base + q * PLANE + (mb * 128 + dy * 21 + dx) * RB;
    }
    GORILA_DEV int row(int t, int mb, int r) const {
        const int m = mb * 128 + r, Y = m / 21, X = m - 21 * Y;
        return (m < 441 && Y < 20 && X < 20) ? (t / MS) * 400 + Y * 20 + X : -1;
    }
};

// ---------------------------------------------------------------- B operands (resident weights)
// Interface: kMN, CHUNK (bytes per chunk, multiple of 1024), NCH (chunks incl. M-block variants),
// load_chunk(ch, dst, bar) -> bytes, chunk_of(c, mb), desc0(base) (descriptor of the block start)
// and off(c, kk, mb) (byte offset of a K step: a descriptor's address field is linear).

// K-major weight [CO][Ktot] (conv forward): chunk c = the CO x (RB/2) block at K offset koff(c).
// map (Ktot, CO), box (RB/2, CO), swizzle RB. KOFF: 0 = c*RB/2; 1 = conv2 phase chunks; 2 = conv1.
template <int CO, int RB_, int NCH_, int KOFF>
struct ShWeightK {
    static constexpr bool kMN = false;
    static constexpr int RB = RB_, NCH = NCH_, CHUNK = (CO * RB + 1023) / 1024 * 1024;
    alignas(64) CUtensorMap map;
    GORILA_DEV static int koff(int c) {
        if (KOFF == 0) return c * (RB / 2);
        if (KOFF == 1) {  // conv2: plane (py, px), tap (dy, dx) -> kernel (2dy+py, 2dx+px), 32 channels
            const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
            return ((2 * dy + (q >> 1)) * 4 + 2 * dx + (q & 1)) * 32;
        }
        const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;  // conv1: row 4dy+py, columns 4dx..4dx+3
        return ((4 * dy + q) * 8 + 4 * dx) * 4;
    }
    GORILA_DEV uint32_t load_chunk(int c, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, koff(c), 0);
        return CO * RB;
    }
    GORILA_DEV static uint64_t desc0(uint32_t base) { return umma_desc_sw(base, RB); }
    GORILA_DEV static uint32_t off(int c, int kk, int) { return c * CHUNK + kk * 32; }
    GORILA_DEV static int chunk_of(int c, int) { return c; }
};

// MN-major conv weight for the data gradient: W [CO=64][K][K][C] over c (N = C), chunk = one tap
// x 64 o (K rows). map (C, 64, K*K), box (C, 64, 1), swizzle C*2. Stride-2 layer: chunk of
// M-block (phase) mb and tap c = kernel (2dy+py, 2dx+px).
template <class SH, bool PHASED>
struct ShWeightDgrad {
    static constexpr bool kMN = true;
    static constexpr int RB = SH::C * 2, NCH = PHASED ? 16 : SH::K * SH::K, CHUNK = (64 * RB + 1023) / 1024 * 1024;
    alignas(64) CUtensorMap map;
    GORILA_DEV static int tap(int ch) {
        if (!PHASED) return ch;
        const int mb = ch >> 2, c = ch & 3, dy = c >> 1, dx = c & 1;
        return (2 * dy + (mb >> 1)) * SH::K + 2 * dx + (mb & 1);
    }
    GORILA_DEV uint32_t load_chunk(int ch, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, 0, 0, tap(ch));
        return 64 * RB;
    }
    GORILA_DEV static int chunk_of(int c, int mb) { return PHASED ? mb * 4 + c : c; }
    GORILA_DEV static uint64_t desc0(uint32_t base) { return umma_desc_mn_sw(base, 0, RB); }
    GORILA_DEV static uint32_t off(int c, int kk, int mb) { return chunk_of(c, mb) * CHUNK + kk * 16 * RB; }
};

// ---------------------------------------------------------------- the engine
template <class OA, class OB, class EP>
struct ShiftProb {
    OA a;
    OB b;
    EP ep;
};
template <class OA, class OB, class EP>
struct ShiftBatch {
    ShiftProb<OA, OB, EP> prob[2];
    int nprob, nbuf, N;
};

constexpr int SHIFT_MAX_BUF = 4, SHIFT_MAX_BCH = 16;

template <int BN, int MB, class OA, class OB>
struct ShiftCfg {
    static constexpr uint32_t ACC = MB * BN;
    static constexpr uint32_t TCOLS = tmem_cols_for(2 * MB * BN);
    static_assert(2 * MB * BN <= 512, "TMEM columns");
    static_assert(OB::NCH <= SHIFT_MAX_BCH, "weight chunks");
    static constexpr int BAR_BYTES = 8 * (2 * SHIFT_MAX_BCH + 2 * SHIFT_MAX_BUF + 4) + 16;
    static constexpr int THREADS = 192;
    // dynamic smem for nprob problems and nbuf A buffers
    static constexpr int smem(int nprob, int nbuf) {
        return 1024 + nprob * OB::NCH * OB::CHUNK + nbuf * OA::BUF + BAR_BYTES;
    }
};

template <int BN, int MB, class OA, class OB, class EP>
__global__ void __launch_bounds__(192) gemm_shift(const __grid_constant__ ShiftBatch<OA, OB, EP> p) {
    using CFG = ShiftCfg<BN, MB, OA, OB>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int nprob = p.nprob, nbuf = p.nbuf;
    uint8_t* bsm = smem;                                   // [nprob][NCH][CHUNK]
    uint8_t* asm_ = smem + nprob * OB::NCH * OB::CHUNK;    // [nbuf][BUF]
    uint64_t* bars = reinterpret_cast<uint64_t*>(asm_ + nbuf * OA::BUF);
    uint64_t* b_full = bars;                               // [2][SHIFT_MAX_BCH]
    uint64_t* a_full = b_full + 2 * SHIFT_MAX_BCH;         // [SHIFT_MAX_BUF]
    uint64_t* a_empty = a_full + SHIFT_MAX_BUF;
    uint64_t* acc_full = a_empty + SHIFT_MAX_BUF;          // [2]
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_per = p.prob[0].a.ntiles(), ntiles = tiles_per * nprob;
    if (warp == 0) tmem_alloc(tmem_slot, CFG::TCOLS);
    if (OA::WRITTEN < OA::PLANE)  // rows past the loaded boxes are read by dropped output rows only:
        for (int b = 0; b < nbuf * OA::NPLANE; ++b)  // zero them once (TMA never writes them)
            for (int o = OA::WRITTEN + tid * 16; o < OA::PLANE; o += CFG::THREADS * 16)
                *reinterpret_cast<uint4*>(asm_ + b * OA::PLANE + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid == 32) {
        for (int i = 0; i < 2 * SHIFT_MAX_BCH; ++i) mbar_init(&b_full[i], 1);
        for (int i = 0; i < SHIFT_MAX_BUF; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_trigger();
    const uint32_t tmem = *tmem_slot;
    const uint32_t bbase = smem_u32(bsm), abase = smem_u32(asm_);
    constexpr uint32_t IDESC = umma_idesc_bf16(TC_BM, BN) | (OB::kMN ? (1u << 16) : 0u);

    if (warp == 0) {
        if (lane == 0) {  // loads: a problem's weights when its first tile comes up, then A buffers
            uint32_t loaded = 0;
            int tl = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const int prob = t / tiles_per, tile = t - prob * tiles_per;
                if (!(loaded & (1u << prob))) {
                    loaded |= 1u << prob;
                    for (int c = 0; c < OB::NCH; ++c) {
                        uint64_t* bar = &b_full[prob * SHIFT_MAX_BCH + c];
                        const uint32_t bytes =
                            p.prob[prob].b.load_chunk(c, bbase + (prob * OB::NCH + c) * OB::CHUNK, bar);
                        mbar_expect_tx(bar, bytes);
                    }
                }
                const int buf = tl % nbuf;
                if (tl >= nbuf) mbar_wait(&a_empty[buf], ((tl / nbuf) - 1) & 1);
                const uint32_t bytes = p.prob[prob].a.load(tile, abase + buf * OA::BUF, &a_full[buf]);
                mbar_expect_tx(&a_full[buf], bytes);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            uint32_t waited = 0;
            int tl = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const int prob = t / tiles_per;
                const ShiftProb<OA, OB, EP>& P = p.prob[prob];
                const int buf = tl % nbuf;
                const uint32_t abuf = tl & 1;
                mbar_wait(&a_full[buf], (tl / nbuf) & 1);
                if (tl >= 2) mbar_wait(&acc_empty[abuf], ((tl >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t acc = tmem + abuf * CFG::ACC;
                const uint32_t a0 = abase + buf * OA::BUF, b0 = bbase + prob * OB::NCH * OB::CHUNK;
                const int m0 = P.a.mb0(t - prob * tiles_per);
                const bool first = !(waited & (1u << prob));  // the problem's weights may still be landing
                waited |= 1u << prob;
                const uint64_t ad0 = umma_desc_sw(a0, OA::RB), bd0 = OB::desc0(b0);
#pragma unroll
                for (int c = 0; c < OA::NCHUNK; ++c) {
                    if (first) {
#pragma unroll
                        for (int mb = 0; mb < MB; ++mb) mbar_wait(&b_full[prob * SHIFT_MAX_BCH + OB::chunk_of(c, m0 + mb)], 0);
                        tc_fence_after();
                    }
#pragma unroll
                    for (int kk = 0; kk < OA::KSTEPS; ++kk)
#pragma unroll
                        for (int mb = 0; mb < MB; ++mb)
                            umma_bf16(acc + mb * BN, ad0 + ((P.a.addr(0, c, m0 + mb) + kk * 32) >> 4),
                                      bd0 + (OB::off(c, kk, m0 + mb) >> 4), IDESC, (c > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&a_empty[buf]);
                umma_commit(&acc_full[abuf]);
            }
        }
    } else {  // epilogue warps 2..5 (warp w reads TMEM lanes 32*(w%4) ..)
        const int quad = warp & 3;
        int tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int prob = t / tiles_per, tile = t - prob * tiles_per;
            const ShiftProb<OA, OB, EP>& P = p.prob[prob];
            const EP ep = P.ep;
            using PT = EpPre<EP>;
            constexpr int NC = BN / 16, PD = NC < 4 ? NC : 4;
            typename PT::type pre[PD];
            const uint32_t abuf = tl & 1;
            const int m0 = P.a.mb0(tile);
            {
                const int i = P.a.row(tile, m0, quad * 32 + lane);
#pragma unroll
                for (int d = 0; d < PD; ++d)
                    if (i >= 0) pre[d] = PT::load(ep, i, d * 16);
            }
            mbar_wait(&acc_full[abuf], (tl >> 1) & 1);
            tc_fence_after();
            const uint32_t acc = tmem + abuf * CFG::ACC + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
            for (int mb = 0; mb < MB; ++mb) {
                const int i = P.a.row(tile, m0 + mb, quad * 32 + lane);
                if (mb > 0)
#pragma unroll
                    for (int d = 0; d < PD; ++d)
                        if (i >= 0) pre[d] = PT::load(ep, i, d * 16);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    float v[16];
                    tmem_ld16(acc + (uint32_t)(mb * BN + c * 16), v);
                    const typename PT::type cur = pre[c % PD];
                    if (c + PD < NC && i >= 0) pre[c % PD] = PT::load(ep, i, (c + PD) * 16);
                    if (i >= 0 && c * 16 < p.N) PT::apply(ep, i, c * 16, v, cur, 0);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[abuf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, CFG::TCOLS);
}

}  // namespace gorila
