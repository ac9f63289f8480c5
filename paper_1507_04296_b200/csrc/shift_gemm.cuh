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

// ---------------------------------------------------------------- ring-gathered input (large batches)
// From B = 75 (the GEMM path) conv1's operands read their input straight from the replay ring: the
// sampler only records each sample's five frame addresses and masks (SampleDesc). A converter expands
// a sample into the bf16 row-phase planes of ShConv1Fwd: row (q, r = Y*21 + X) of plane q holds
// pixels s[4Y+q][4X .. 4X+3] x channels 0..3 (32 B), the same image the TMA boxes of ShConv1Fwd write
// from a bf16 NHWC stack; the four channels are four frames (net z: frames z .. z+3), one 4-byte
// load each, byte-transposed to pixel-major order. 16-B half h of a row sits at byte r*32 + 16h of
// the plane with address bit 7 XORed into bit 4 (SWIZZLE_32B).
constexpr int U8_ROWS = 4 * 441;  // plane rows per sample

// bytes (2hi, 2hi + 1) of w as bf16x2: u8 -> fp32 exactly (magic 2^23), the upper halves exact
GORILA_DEV uint32_t u8x2_bf16x2(uint32_t w, int hi) {
    const float f0 = __uint_as_float(__byte_perm(w, 0x4B000000u, hi ? 0x7442u : 0x7440u)) - 8388608.f;
    const float f1 = __uint_as_float(__byte_perm(w, 0x4B000000u, hi ? 0x7443u : 0x7441u)) - 8388608.f;
    return __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632u);
}

// NT threads expand one sample: load() issues its global reads (into registers, so that the next
// sample's loads are in flight while this one is stored), store() transposes, converts and writes
template <int NT>
struct U8Planes {
    static constexpr int PER = (U8_ROWS + NT - 1) / NT;
    uint32_t w[PER][4];  // per row: channel c's four pixels
    GORILA_DEV void load(const SampleDesc* __restrict__ d, int z, int t) {
        const uint8_t* fr[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) fr[c] = d->frame[c + z];
        const uint32_t keep = d->keep >> (4 * z);
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = t + k * NT;
            if (i >= U8_ROWS) continue;
            const int q = i / 441, r = i - 441 * q, Y = r / 21, X = r - 21 * Y;
            const int off = (4 * Y + q) * 84 + 4 * X;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                w[k][c] = (keep >> c) & 1u ? __ldcg(reinterpret_cast<const uint32_t*>(fr[c] + off)) : 0u;
        }
    }
    // the same rows from the sample's four frames staged in shared memory (channel c at c * 7056)
    GORILA_DEV void load_smem(uint32_t raw, uint32_t keep, int t) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = t + k * NT;
            if (i >= U8_ROWS) continue;
            const int q = i / 441, r = i - 441 * q, Y = r / 21, X = r - 21 * Y;
            const uint32_t off = (4 * Y + q) * 84 + 4 * X;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t v = 0;
                if ((keep >> c) & 1u) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(raw + c * FRAME_BYTES + off));
                w[k][c] = v;
            }
        }
    }
    GORILA_DEV void store(uint32_t planes, uint32_t plane_bytes, int t) const {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int i = t + k * NT;
            if (i >= U8_ROWS) continue;
            const int q = i / 441, r = i - 441 * q;
            const uint32_t row = planes + q * plane_bytes + r * 32;
            // 4 x 4 byte transpose: word px = channels 0..3 of pixel px
            const uint32_t lo01 = __byte_perm(w[k][0], w[k][1], 0x5140u), lo23 = __byte_perm(w[k][2], w[k][3], 0x5140u);
            const uint32_t hi01 = __byte_perm(w[k][0], w[k][1], 0x7362u), hi23 = __byte_perm(w[k][2], w[k][3], 0x7362u);
            const uint32_t px[4] = {__byte_perm(lo01, lo23, 0x5410u), __byte_perm(lo01, lo23, 0x7632u),
                                    __byte_perm(hi01, hi23, 0x5410u), __byte_perm(hi01, hi23, 0x7632u)};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t a = row + 16 * h, pa = a ^ ((a >> 3) & 16u);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(pa), "r"(u8x2_bf16x2(px[2 * h], 0)),
                             "r"(u8x2_bf16x2(px[2 * h], 1)), "r"(u8x2_bf16x2(px[2 * h + 1], 0)),
                             "r"(u8x2_bf16x2(px[2 * h + 1], 1))
                             : "memory");
            }
        }
    }
};

// diagnostics (gorila_get_activation "s" on the u8 path): sample b's s as row-phase-major u8
// [q][Y][X][px][c] (4 x 441 rows of 16 B), through the same gather as the converters
__global__ void k_stage_from_desc(const SampleDesc* __restrict__ desc, int B, uint8_t* __restrict__ out) {
    const int64_t total = (int64_t)B * U8_ROWS;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / U8_ROWS;
        const int i = (int)(e - b * U8_ROWS), q = i / 441, r = i - 441 * q, Y = r / 21, X = r - 21 * Y;
        const SampleDesc& d = desc[b];
        uint32_t w[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
            w[c] = (d.keep >> c) & 1u ? *reinterpret_cast<const uint32_t*>(d.frame[c] + (4 * Y + q) * 84 + 4 * X) : 0u;
        const uint32_t lo01 = __byte_perm(w[0], w[1], 0x5140u), lo23 = __byte_perm(w[2], w[3], 0x5140u);
        const uint32_t hi01 = __byte_perm(w[0], w[1], 0x7362u), hi23 = __byte_perm(w[2], w[3], 0x7362u);
        reinterpret_cast<uint4*>(out)[e] = make_uint4(__byte_perm(lo01, lo23, 0x5410u), __byte_perm(lo01, lo23, 0x7632u),
                                                      __byte_perm(hi01, hi23, 0x5410u), __byte_perm(hi01, hi23, 0x7632u));
    }
}

// conv1 forward from the ring gather: ShConv1Fwd<1>'s planes, written by the engine's converter warps
struct ShConv1FwdU8 {
    static constexpr bool CONVERT = true;
    static constexpr int RB = 32, NCHUNK = 16, KSTEPS = 1, PROWS = 544, PLANE = PROWS * RB;
    static constexpr int BUF = 4 * PLANE, NPLANE = 4, WRITTEN = 441 * RB, MS = 1;
    const SampleDesc* desc;  // [B]
    int z;                   // 0: s (frames 0..3), 1: s' (frames 1..4)
    int batch;
    __host__ __device__ int ntiles() const { return batch; }
    GORILA_DEV int mb0(int) const { return 0; }
    GORILA_DEV uint32_t addr(uint32_t base, int c, int mb) const {
        const int q = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
        return base + q * PLANE + (mb * 128 + dy * 21 + dx) * RB;
    }
    GORILA_DEV int row(int t, int mb, int r) const {
        const int m = mb * 128 + r, Y = m / 21, X = m - 21 * Y;
        return (m < 441 && Y < 20 && X < 20) ? t * 400 + Y * 20 + X : -1;
    }
};
template <class E, class = void>
struct ep_has_mask : std::false_type {};
template <class E>
struct ep_has_mask<E, std::void_t<decltype(std::declval<E>().mask)>> : std::true_type {};
template <class O, class = void>
struct shift_convert : std::false_type {};
template <class O>
struct shift_convert<O, std::void_t<decltype(O::CONVERT)>> : std::integral_constant<bool, O::CONVERT> {};
#ifndef GORILA_CONV_WARPS
#define GORILA_CONV_WARPS 8
#endif
constexpr int SHIFT_CONV_WARPS = GORILA_CONV_WARPS;  // converter warps of a CONVERT operand

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
    static constexpr int BAR_BYTES = 8 * (2 * SHIFT_MAX_BCH + 2 * SHIFT_MAX_BUF + 8) + 16;
    static constexpr bool CONV = shift_convert<OA>::value;
    // epilogue warp groups: two for the converting multi-block operand (conv1, MB = 4: each group
    // drains half of a tile's M-blocks, so the accumulator is released twice as fast)
    static constexpr int ES = (CONV && MB >= 2) ? 2 : 1;
    static constexpr int EPI_END = 2 + 4 * ES;  // epilogue warps 2 .. EPI_END - 1, converters after
    // converter warps avoid the MMA warp's scheduler (warp w runs on sub-partition w % 4; warp 1
    // issues the MMAs): with ES = 2 they are warps 10, 11, 12, 14, 15, 16, 18, 19 (13, 17 idle)
    // (ES == 2: the converter warps skip sub-partition 1 -> SHIFT_CONV_WARPS / 3 * 4 warp slots)
    static constexpr int conv_span() {
        int w = EPI_END, k = 0;
        while (k < SHIFT_CONV_WARPS) k += ((w++ & 3) != 1) ? 1 : 0;
        return w - EPI_END;
    }
    static constexpr int CONV_SPAN = CONV ? (ES == 2 ? conv_span() : SHIFT_CONV_WARPS) : 0;
    static constexpr int THREADS = 32 * (EPI_END + CONV_SPAN);
    static GORILA_DEV int conv_index(int w) {  // converter number 0..SHIFT_CONV_WARPS-1 of warp w, or -1
        const int o = w - EPI_END;
        if (o < 0 || o >= CONV_SPAN) return -1;
        if (ES != 2) return o;
        if ((w & 3) == 1) return -1;
        int k = 0;  // converters before warp w (warps on sub-partition 1 skipped)
        for (int u = EPI_END; u < w; ++u) k += (u & 3) != 1;
        return k < SHIFT_CONV_WARPS ? k : -1;
    }
    // CONVERT: the tile's four ring frames, bulk-copied (cp.async.bulk) by the load warp
    static constexpr int RAW = CONV ? 2 * 4 * FRAME_BYTES : 0;  // two tiles' frames
    // dynamic smem for nprob problems and nbuf A buffers
    static constexpr int smem(int nprob, int nbuf) {
        return 1024 + nprob * OB::NCH * OB::CHUNK + nbuf * OA::BUF + RAW + BAR_BYTES;
    }
};

template <int BN, int MB, class OA, class OB, class EP>
__global__ void __launch_bounds__(ShiftCfg<BN, MB, OA, OB>::THREADS)
    gemm_shift(const __grid_constant__ ShiftBatch<OA, OB, EP> p) {
    using CFG = ShiftCfg<BN, MB, OA, OB>;
    constexpr bool CONV = CFG::CONV;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int nprob = p.nprob, nbuf = p.nbuf;
    uint8_t* bsm = smem;                                   // [nprob][NCH][CHUNK]
    uint8_t* asm_ = smem + nprob * OB::NCH * OB::CHUNK;    // [nbuf][BUF]
    uint8_t* raw = asm_ + nbuf * OA::BUF;                  // [RAW] (CONVERT)
    uint64_t* bars = reinterpret_cast<uint64_t*>(raw + CFG::RAW);
    uint64_t* b_full = bars;                               // [2][SHIFT_MAX_BCH]
    uint64_t* a_full = b_full + 2 * SHIFT_MAX_BCH;         // [SHIFT_MAX_BUF]
    uint64_t* a_empty = a_full + SHIFT_MAX_BUF;
    uint64_t* acc_full = a_empty + SHIFT_MAX_BUF;          // [2]
    uint64_t* acc_empty = acc_full + 2;
    uint64_t* raw_full = acc_empty + 2;                    // [2] CONVERT: frames landed / read
    uint64_t* raw_empty = raw_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + 2);

    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
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
            mbar_init(&a_full[i], CONV ? SHIFT_CONV_WARPS : 1);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4 * CFG::ES);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&raw_full[i], 1);
            mbar_init(&raw_empty[i], SHIFT_CONV_WARPS);
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
                if constexpr (!CONV) {  // (CONVERT operands: the converter warps fill the buffers)
                    const int buf = tl % nbuf;
                    if (tl >= nbuf) mbar_wait(&a_empty[buf], ((tl / nbuf) - 1) & 1);
                    const uint32_t bytes = p.prob[prob].a.load(tile, abase + buf * OA::BUF, &a_full[buf]);
                    mbar_expect_tx(&a_full[buf], bytes);
                } else {  // the tile's four frames into the raw buffer once the converters have read it
                    const int rs = tl & 1;
                    if (tl >= 2) mbar_wait(&raw_empty[rs], ((tl >> 1) - 1) & 1);
                    const SampleDesc* d = p.prob[prob].a.desc + tile;
                    const int z = p.prob[prob].a.z;
                    const uint32_t rb = smem_u32(raw) + rs * 4 * FRAME_BYTES;
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        bulk_load(rb + c * FRAME_BYTES, d->frame[c + z], FRAME_BYTES, &raw_full[rs]);
                    mbar_expect_tx(&raw_full[rs], 4 * FRAME_BYTES);
                }
            }
        }
    } else if (warp == 1) {
        {  // MMA issuer (warp-uniform; one elected lane issues)
            const uint32_t tmem_u = uniform_u32(tmem), abase_u = uniform_u32(abase), bbase_u = uniform_u32(bbase);
            uint32_t waited = 0;
            int tl = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const int prob = t / tiles_per;
                const ShiftProb<OA, OB, EP>& P = p.prob[prob];
                const int buf = tl % nbuf;
                const uint32_t abuf = tl & 1;
                mbar_wait(&a_full[buf], (tl / nbuf) & 1);
                if (lane == 0) GTRACE_T(2, tl);
                if (tl >= 2) mbar_wait(&acc_empty[abuf], ((tl >> 1) - 1) & 1);
                if (lane == 0) GTRACE_T(3, tl);
                tc_fence_after();
                const uint32_t acc = tmem_u + abuf * CFG::ACC;
                const uint32_t a0 = abase_u + buf * OA::BUF, b0 = bbase_u + prob * OB::NCH * OB::CHUNK;
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
                            umma_bf16_w(acc + mb * BN, ad0 + ((P.a.addr(0, c, m0 + mb) + kk * 32) >> 4),
                                        bd0 + (OB::off(c, kk, m0 + mb) >> 4), IDESC, (c > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit_w(&a_empty[buf]);
                umma_commit_w(&acc_full[abuf]);
                if (lane == 0) GTRACE_T(4, tl);
            }
        }
    } else if (CONV && warp >= CFG::EPI_END) {  // converter warps: ring frames -> the tile's bf16 planes
        if constexpr (CONV) {
            const int cw = CFG::conv_index(warp);
            // per tile: read the landed frames (releasing the raw buffer for the next tile's copy),
            // then transpose / convert into the tile's A buffer
            constexpr int NT = 32 * SHIFT_CONV_WARPS;
            const int ct = cw * 32 + lane;
            const uint32_t rb = smem_u32(raw);
            U8Planes<NT> r;
            int tl = 0;
            for (int t = cw < 0 ? ntiles : (int)blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const int pr = t / tiles_per;
                const uint32_t keep = p.prob[pr].a.desc[t - pr * tiles_per].keep >> (4 * p.prob[pr].a.z);
                if (ct == 0) GTRACE_T(0, tl);
                const int rs = tl & 1;
                mbar_wait(&raw_full[rs], (tl >> 1) & 1);
                r.load_smem(rb + rs * 4 * FRAME_BYTES, keep, ct);
                __syncwarp();
                if (lane == 0) mbar_arrive(&raw_empty[rs]);
                const int buf = tl % nbuf;
                if (tl >= nbuf) mbar_wait(&a_empty[buf], ((tl / nbuf) - 1) & 1);
                r.store(abase + buf * OA::BUF, OA::PLANE, ct);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[buf]);
                if (lane == 0) GTRACE_C(cw, tl);  // (every converter warp's hand-over)
                if (ct == 0) GTRACE_T(1, tl);
            }
        }
    } else if constexpr (ep_col_pre<EP>::value && BN <= 64) {
        // epilogue warps 2..5, column-only inputs (the biases): loaded once per CTA (per problem);
        // the accumulator is read 32 columns per TMEM wait
        const int quad = warp & 3, eh = (warp - 2) >> 2;  // lane quarter, epilogue group
        using PT = EpPre<EP>;
        constexpr int NC = BN / 16;
        typename PT::type pre[NC];
        int pre_prob = -1;  // a CTA's tiles run in increasing order: its problem changes at most nprob - 1 times
        int tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int prob = t / tiles_per, tile = t - prob * tiles_per;
            const ShiftProb<OA, OB, EP>& P = p.prob[prob];
            const EP ep = P.ep;
            if (prob != pre_prob) {
#pragma unroll
                for (int c = 0; c < NC; ++c) pre[c] = PT::load(ep, 0, c * 16);
                pre_prob = prob;
            }
            const uint32_t abuf = tl & 1;
            const int m0 = P.a.mb0(tile);
            if (quad == 2 && eh == 0 && lane == 0) GTRACE_T(5, tl);
            mbar_wait(&acc_full[abuf], (tl >> 1) & 1);
            if (quad == 2 && eh == 0 && lane == 0) GTRACE_T(6, tl);
            tc_fence_after();
            const uint32_t acc = tmem + abuf * CFG::ACC + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
            for (int mb = eh; mb < MB; mb += CFG::ES) {
                const int i = P.a.row(tile, m0 + mb, quad * 32 + lane);
#pragma unroll
                for (int c2 = 0; c2 < NC; c2 += 2) {
                    float v[32];
                    if (c2 + 1 < NC) tmem_ld16x2(acc + (uint32_t)(mb * BN + c2 * 16), v);
                    else tmem_ld16(acc + (uint32_t)(mb * BN + c2 * 16), v);
                    if constexpr (ep_has_mask<EP>::value) {
                        if (ep.mask != nullptr) {  // the ReLU decisions as bits, one word per 32 columns
                            if (i >= 0 && c2 + 1 < NC && (c2 + 2) * 16 <= p.N) {
                                const uint32_t lo = ep.apply16m(i, c2 * 16, v, pre[c2]);
                                const uint32_t hi = ep.apply16m(i, c2 * 16 + 16, v + 16, pre[c2 + 1]);
                                ep.mask[(int64_t)i * (p.N >> 5) + (c2 >> 1)] = lo | (hi << 16);
                            }
                            continue;
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if (c2 + h < NC && i >= 0 && (c2 + h) * 16 < p.N)
                            PT::apply(ep, i, (c2 + h) * 16, v + 16 * h, pre[c2 + h], 0);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[abuf]);
            if (quad == 2 && eh == 0 && lane == 0) GTRACE_T(7, tl);
        }
    } else {  // epilogue warps 2..5 (warp w reads TMEM lanes 32*(w%4) ..)
        static_assert(CFG::ES == 1, "generic epilogue runs one warp group");
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
            if (quad == 2 && lane == 0) GTRACE_T(5, tl);
            mbar_wait(&acc_full[abuf], (tl >> 1) & 1);
            if (quad == 2 && lane == 0) GTRACE_T(6, tl);
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
            if (quad == 2 && lane == 0) GTRACE_T(7, tl);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, CFG::TCOLS);
}


// ---------------------------------------------------------------- conv1 weight gradient (u8 staging)
// dW1[o][ky][kx][c] = sum over samples and output pixels (oy, ox) of g1[oy][ox][o] * s[4oy+ky][4ox+kx][c].
// With ky = 4dy + py and kx = 4dx + px the input element is row (oy+dy)*21 + (ox+dx) of phase plane
// py (element (px, c)): the virtual-grid pixel p = oy*21 + ox shifted by dy*21 + dx rows. So per
// (dy, dx) one M = 64 accumulator (the 4 planes x 16 (px, c): MN-major A, 16-element blocks PLANE
// bytes apart) runs over K = the sample's 21 x 20 virtual pixels from a shifted start row, against
// B = g1 on the same virtual grid (MN-major over o, 64-B rows; the 21st column is TMA zero fill, so
// the rows a shift wraps into contribute nothing). No im2col: the planes are expanded once per
// sample from the u8 staging (U8Planes) and every tap is a start address.
// One CTA per sample stride; the four accumulators (M = 64 each: two per TMEM column block, at lane
// offsets 0 and 16) stay in TMEM across all of the CTA's samples; the epilogue stores the CTA's
// partial dW1 [o][k] (times the input scale) for the fixed-order reduction (k_wgrad_reduce).
struct Conv1WgradU8 {
    CUtensorMap g1_map;  // (32, 20, 20, B) bf16, box (32, 21, 20, 1), SWIZZLE_64B
    const SampleDesc* desc;  // [B]: the samples' ring frames (s = frames 0..3)
    float* part;         // [gridDim.x][32][256]
    float* part_b;       // [gridDim.x][32]: the CTA's sum of g1 (bias b1's gradient)
    float scale;
    int batch;
};
// The bias gradient rides along as one more accumulator: D[m][o] += sum_p ONE[m][p] g[p][o] with an
// A operand of ones (every row of D is the column sum of g). One 16-row block of bf16 ones (M = 64
// rows of 128 B, MN-major) serves every K step.
constexpr int ONES_BYTES = 16 * 128;
GORILA_DEV void fill_ones(uint8_t* dst, int tid, int nthr) {
    for (int o = tid * 16; o < ONES_BYTES; o += nthr * 16)
        *reinterpret_cast<uint4*>(dst + o) = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
}
namespace c1wg {
constexpr int KSTEPS = 27;                           // 432 virtual rows, 420 of them g1 rows (21 x 20)
constexpr int PLANE = ShConv1FwdU8::PLANE;           // 544 rows of 32 B (rows <= 431 + 22 are read)
constexpr int ABUF = 4 * PLANE, BBUF = KSTEPS * 16 * 64, STAGE = ABUF + BBUF;  // 69632 + 27648
// converters: warps 2, 3, 4, 6, 7, 8, 10, 11 (off the MMA warp's sub-partition 1); epilogue 2..5
constexpr int NBUF = 2, CONV_WARPS = 8, THREADS = 32 * 12;
constexpr int RAW = 4 * FRAME_BYTES;  // the sample's four ring frames (cp.async.bulk)
constexpr int SMEM = 1024 + NBUF * STAGE + ONES_BYTES + RAW + 128;
GORILA_DEV int conv_index(int w) { return (w < 2 || w > 11 || (w & 3) == 1) ? -1 : w - 2 - (w > 5) - (w > 9); }
constexpr uint32_t TCOLS = 128;  // 4 (dy, dx) accumulators in columns 0..63, the ones accumulator 64..95
}  // namespace c1wg

__global__ void __launch_bounds__(c1wg::THREADS) k_conv1_wgrad_u8(const __grid_constant__ Conv1WgradU8 p) {
    using namespace c1wg;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ones = smem + NBUF * STAGE;
    uint8_t* raw = ones + ONES_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(raw + RAW);
    uint64_t* a_full = bars;               // [NBUF] converter warps
    uint64_t* b_full = a_full + NBUF;      // [NBUF] TMA of g1
    uint64_t* empty = b_full + NBUF;       // [NBUF] MMA commit
    uint64_t* done = empty + NBUF;
    uint64_t* raw_full = done + 1;         // the frames landed / read by the converters
    uint64_t* raw_empty = raw_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(raw_empty + 1);
    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    const int nt = p.batch > (int)blockIdx.x ? (p.batch - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (warp == 0) tmem_alloc(tmem_slot, TCOLS);
    // plane rows past the 441 written ones and g1 rows past the 420 loaded ones: zero once
    for (int b = 0; b < NBUF; ++b) {
        uint8_t* st = smem + b * STAGE;
        for (int q = 0; q < 4; ++q)
            for (int o = 441 * 32 + tid * 16; o < PLANE; o += THREADS * 16)
                *reinterpret_cast<uint4*>(st + q * PLANE + o) = make_uint4(0, 0, 0, 0);
        for (int o = 420 * 64 + tid * 16; o < BBUF; o += THREADS * 16)
            *reinterpret_cast<uint4*>(st + ABUF + o) = make_uint4(0, 0, 0, 0);
    }
    fill_ones(ones, tid, THREADS);
    fence_proxy_async_smem();
    if (tid == 32) {
        for (int i = 0; i < NBUF; ++i) {
            mbar_init(&a_full[i], CONV_WARPS);
            mbar_init(&b_full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        mbar_init(raw_full, 1);
        mbar_init(raw_empty, CONV_WARPS);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_trigger();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = smem_u32(smem);
    if (warp == 0) {
        if (lane == 0) {  // per sample: its four frames (once the converters read the last ones), g1
            const uint32_t rb = smem_u32(raw);
            for (int tl = 0; tl < nt; ++tl) {
                const int b = blockIdx.x + tl * gridDim.x, s = tl % NBUF;
                if (tl >= 1) mbar_wait(raw_empty, (tl - 1) & 1);
                const SampleDesc* d = p.desc + b;
#pragma unroll
                for (int c = 0; c < 4; ++c) bulk_load(rb + c * FRAME_BYTES, d->frame[c], FRAME_BYTES, raw_full);
                mbar_expect_tx(raw_full, 4 * FRAME_BYTES);
                if (tl >= NBUF) mbar_wait(&empty[s], ((tl / NBUF) - 1) & 1);
                tma_load(&p.g1_map, sbase + s * STAGE + ABUF, &b_full[s], 0, 0, 0, b);
                mbar_expect_tx(&b_full[s], 420 * 64);
            }
        }
    } else if (warp == 1) {
        {  // MMA issuer (warp-uniform): per sample 27 K-steps x 4 (dy, dx) accumulators
            constexpr uint32_t IDESC = umma_idesc_bf16(64, 32) | (1u << 15) | (1u << 16);
            const uint32_t tmem_u = uniform_u32(tmem), sbase_u = uniform_u32(sbase);
            const uint64_t od = umma_desc_mn_sw(sbase_u + NBUF * STAGE, 0, 128);  // the ones block
            for (int tl = 0; tl < nt; ++tl) {
                const int s = tl % NBUF;
                mbar_wait(&a_full[s], (tl / NBUF) & 1);
                mbar_wait(&b_full[s], (tl / NBUF) & 1);
                tc_fence_after();
                const uint32_t a0 = sbase_u + s * STAGE, b0 = a0 + ABUF;
#pragma unroll 1
                for (int kk = 0; kk < KSTEPS; ++kk) {
                    const uint64_t bd = umma_desc_mn_sw(b0 + kk * 1024, 0, 64);
                    umma_bf16_w(tmem_u + 64, od, bd, IDESC, (tl > 0 || kk > 0) ? 1u : 0u);  // sum of g1
#pragma unroll
                    for (int acc = 0; acc < 4; ++acc) {
                        const int dy = acc >> 1, dx = acc & 1;
                        const uint64_t ad = umma_desc_mn_sw(a0 + (kk * 16 + dy * 21 + dx) * 32, PLANE, 32);
                        umma_bf16_w(tmem_u + ((uint32_t)(16 * dx) << 16) + 32 * dy, ad, bd, IDESC,
                                    (tl > 0 || kk > 0) ? 1u : 0u);
                    }
                }
                umma_commit_w(&empty[s]);
            }
            umma_commit_w(done);
        }
    } else {  // converter warps (conv_index >= 0): the samples' frames -> bf16 planes
        constexpr int NT = 32 * CONV_WARPS;
        const int cw = conv_index(warp), ct = cw * 32 + lane;
        const uint32_t rb = smem_u32(raw);
        U8Planes<NT> r;
        for (int tl = 0; cw >= 0 && tl < nt; ++tl) {
            const uint32_t keep = p.desc[blockIdx.x + tl * gridDim.x].keep;
            mbar_wait(raw_full, tl & 1);
            r.load_smem(rb, keep, ct);
            __syncwarp();
            if (lane == 0) mbar_arrive(raw_empty);
            const int s = tl % NBUF;
            if (tl >= NBUF) mbar_wait(&empty[s], ((tl / NBUF) - 1) & 1);
            r.store(sbase + s * STAGE, PLANE, ct);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_full[s]);
        }
        if (warp < 6) {  // epilogue (warps 2..5 = TMEM lane quarters 2, 3, 0, 1)
            const int quad = warp & 3;
            if (nt > 0) {
                mbar_wait(done, 0);
                tc_fence_after();
            }
            float* dst = p.part + (int64_t)blockIdx.x * (32 * K1);
            // lane l of quarter quad: row 16*quad + (l & 15) of accumulator (dy, dx = l >> 4) in column
            // block dy -> k = (4dy + quad) * 32 + 16dx + (l & 15) = (4dy + quad) * 32 + l
#pragma unroll 1
            for (int dy = 0; dy < 2; ++dy)
#pragma unroll 1
                for (int c0 = 0; c0 < 32; c0 += 16) {
                    float v[16];
                    if (nt > 0) tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(32 * dy + c0), v);
                    else
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    const int k = (4 * dy + quad) * 32 + lane;
#pragma unroll
                    for (int e = 0; e < 16; ++e) dst[(c0 + e) * K1 + k] = v[e] * p.scale;
                }
            if (quad == 0) {  // row 0 of the ones accumulator (lane 0): the CTA's sum of g1 per channel
                float v[32];
                if (nt > 0) tmem_ld16x2(tmem + 64, v);
                else
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                if (lane == 0)
#pragma unroll
                    for (int e = 0; e < 32; ++e) p.part_b[blockIdx.x * 32 + e] = v[e];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, TCOLS);
}


// ---------------------------------------------------------------- conv2 / conv3 weight gradients
// Same construction as k_conv1_wgrad_u8 over bf16 activations loaded by TMA: per sample the layer
// input (MN-major over input channels) and the output gradient g on the layer's virtual grid (the
// input grid's width; columns / rows past the output are TMA zero fill); tap (ky, kx) of the kernel
// reads the input rows shifted by its offset on that grid. One CTA per sample stride, all taps'
// accumulators in TMEM across the CTA's samples, partial dW [o][k] per CTA (k_wgrad_reduce).
//   conv3 (3x3, stride 1, a2 9x9x64 -> g3 7x7x64): grid 9 wide, 9 taps = 9 accumulators M = 64
//     (the 64 input channels; two per TMEM column block at lane offsets 0 / 16), k = tap*64 + c.
//   conv2 (4x4, stride 2, a1 20x20x32 -> g2 9x9x64): the four stride phases of a1 as planes (10 x 10
//     rows of 32 channels, as conv2's forward loads them); per (dy, dx) one accumulator M = 128 =
//     4 planes x 32 channels (kernel (2dy + py, 2dx + px)), grid 10 wide.
struct WgConv3 {
    static constexpr int NPLANE = 1, A_RB = 128, PROWS = 120, PLANE = PROWS * A_RB, A_LOADED = 81 * A_RB;
    static constexpr int B_ROWS_LOADED = 81, NACC = 9, M = 64, TCOLS = 512;
    static GORILA_DEV int shift(int a) { return (a / 3) * 9 + (a % 3); }
    static GORILA_DEV uint32_t dtmem(int a) { return ((uint32_t)(16 * (a & 1)) << 16) + 64 * (a >> 1); }
    static constexpr uint32_t ONES_TMEM = (16u << 16) + 256, ONES_LANE = 16;  // the free 10th M = 64 slot
    static GORILA_DEV void load_a(const CUtensorMap* m, uint32_t dst, uint64_t* bar, int b) { tma_load(m, dst, bar, 0, 0, b); }
    static GORILA_DEV void load_b(const CUtensorMap* m, uint32_t dst, uint64_t* bar, int b) { tma_load(m, dst, bar, 0, 0, 0, b); }
};
struct WgConv2 {
    static constexpr int NPLANE = 4, A_RB = 64, PROWS = 112, PLANE = PROWS * A_RB, A_LOADED = 4 * 100 * A_RB;
    static constexpr int B_ROWS_LOADED = 90, NACC = 4, M = 128, TCOLS = 512;
    static GORILA_DEV int shift(int a) { return (a >> 1) * 10 + (a & 1); }
    static GORILA_DEV uint32_t dtmem(int a) { return 64 * a; }
    static constexpr uint32_t ONES_TMEM = 256, ONES_LANE = 0;  // an M = 64 accumulator after the four M = 128
    static GORILA_DEV void load_a(const CUtensorMap* m, uint32_t dst, uint64_t* bar, int b) {
#pragma unroll
        for (int q = 0; q < 4; ++q) tma_load(m, dst + q * PLANE, bar, 0, q & 1, q >> 1, b);
    }
    static GORILA_DEV void load_b(const CUtensorMap* m, uint32_t dst, uint64_t* bar, int b) { tma_load(m, dst, bar, 0, 0, 0, b); }
};
struct WgradShiftParams {
    CUtensorMap a_map;  // conv3: (64, 81, B) box (64, 81, 1) SW128; conv2: sh_conv2_map (phase planes)
    CUtensorMap g_map;  // conv3: (64, 7, 7, B) box (64, 9, 9, 1); conv2: (64, 9, 9, B) box (64, 10, 9, 1); SW128
    float* part;        // [gridDim.x][64][K]
    float* part_b;      // [gridDim.x][64]: the CTA's sum of g (the layer's bias gradient)
    int batch;
};
namespace wgs {
constexpr int KSTEPS = 6, B_BUF = KSTEPS * 16 * 128, NBUF = 4;  // 96 virtual rows of g
template <class W>
struct Cfg {
    static constexpr int A_BUF = W::NPLANE * W::PLANE, STAGE = A_BUF + B_BUF;
    static constexpr int SMEM = 1024 + NBUF * STAGE + ONES_BYTES + 128;
};
}  // namespace wgs

template <class W>
__global__ void __launch_bounds__(192) k_wgrad_shift(const __grid_constant__ WgradShiftParams p) {
    using CF = wgs::Cfg<W>;
    constexpr int NBUF = wgs::NBUF, STAGE = CF::STAGE, A_BUF = CF::A_BUF;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ones = smem + NBUF * STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(ones + ONES_BYTES);
    uint64_t* empty = full + NBUF;
    uint64_t* done = empty + NBUF;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    const int nt = p.batch > (int)blockIdx.x ? (p.batch - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (warp == 0) tmem_alloc(tmem_slot, W::TCOLS);
    fill_ones(ones, tid, 192);
    for (int s = 0; s < NBUF; ++s) {  // rows the loads never write (read only against zero rows of g)
        uint8_t* st = smem + s * STAGE;
        for (int q = 0; q < W::NPLANE; ++q)
            for (int o = W::A_LOADED / W::NPLANE + tid * 16; o < W::PLANE; o += 192 * 16)
                *reinterpret_cast<uint4*>(st + q * W::PLANE + o) = make_uint4(0, 0, 0, 0);
        for (int o = W::B_ROWS_LOADED * 128 + tid * 16; o < wgs::B_BUF; o += 192 * 16)
            *reinterpret_cast<uint4*>(st + A_BUF + o) = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
    if (tid == 32) {
        for (int i = 0; i < NBUF; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_trigger();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = smem_u32(smem);
    if (warp == 0) {
        if (lane == 0) {  // per sample: the layer input and the output gradient
            for (int tl = 0; tl < nt; ++tl) {
                const int b = blockIdx.x + tl * gridDim.x, s = tl % NBUF;
                if (tl >= NBUF) mbar_wait(&empty[s], ((tl / NBUF) - 1) & 1);
                const uint32_t a0 = sbase + s * STAGE;
                W::load_a(&p.a_map, a0, &full[s], b);
                W::load_b(&p.g_map, a0 + A_BUF, &full[s], b);
                mbar_expect_tx(&full[s], W::A_LOADED + W::B_ROWS_LOADED * 128);
            }
        }
    } else if (warp == 1) {  // MMA issuer (warp-uniform)
        constexpr uint32_t IDESC = umma_idesc_bf16(W::M, 64) | (1u << 15) | (1u << 16);
        constexpr uint32_t IDESC1 = umma_idesc_bf16(64, 64) | (1u << 15) | (1u << 16);
        const uint32_t tmem_u = uniform_u32(tmem), sbase_u = uniform_u32(sbase);
        const uint64_t od = umma_desc_mn_sw(sbase_u + NBUF * STAGE, 0, 128);  // the ones block
        for (int tl = 0; tl < nt; ++tl) {
            const int s = tl % NBUF;
            mbar_wait(&full[s], (tl / NBUF) & 1);
            tc_fence_after();
            const uint32_t a0 = sbase_u + s * STAGE, b0 = a0 + A_BUF;
#pragma unroll 1
            for (int kk = 0; kk < wgs::KSTEPS; ++kk) {
                const uint64_t bd = umma_desc_mn_sw(b0 + kk * 16 * 128, 0, 128);
                umma_bf16_w(tmem_u + W::ONES_TMEM, od, bd, IDESC1, (tl > 0 || kk > 0) ? 1u : 0u);  // sum of g
#pragma unroll
                for (int a = 0; a < W::NACC; ++a) {
                    const uint64_t ad = umma_desc_mn_sw(a0 + (kk * 16 + W::shift(a)) * W::A_RB, W::PLANE, W::A_RB);
                    umma_bf16_w(tmem_u + W::dtmem(a), ad, bd, IDESC, (tl > 0 || kk > 0) ? 1u : 0u);
                }
            }
            umma_commit_w(&empty[s]);
        }
        umma_commit_w(done);
    } else {  // epilogue warps 2..5: the CTA's partial dW [o][k]
        const int quad = warp & 3;
        if (nt > 0) {
            mbar_wait(done, 0);
            tc_fence_after();
        }
        constexpr int K = W::M == 64 ? 9 * 64 : 16 * 32;
        float* dst = p.part + (int64_t)blockIdx.x * (64 * K);
        constexpr int NBLK = W::M == 64 ? (W::NACC + 1) / 2 : W::NACC;
#pragma unroll 1
        for (int j = 0; j < NBLK; ++j) {
            int k;
            bool ok = true;
            if (W::M == 64) {  // lanes 0-15: accumulator 2j, 16-31: 2j + 1; row 16 * quad + (lane & 15)
                const int a = 2 * j + (lane >> 4);
                ok = a < W::NACC;
                k = a * 64 + 16 * quad + (lane & 15);
            } else {  // accumulator j = (dy, dx); lane quarter = phase plane (py, px), lane = channel
                const int dy = j >> 1, dx = j & 1, py = quad >> 1, px = quad & 1;
                k = ((2 * dy + py) * 4 + 2 * dx + px) * 32 + lane;
            }
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 32) {
                float v[32];
                if (nt > 0) tmem_ld16x2(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(64 * j + c0), v);
                else
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                if (ok)
#pragma unroll
                    for (int e = 0; e < 32; ++e) dst[(c0 + e) * K + k] = v[e];
            }
        }
        if (quad == 0)  // row 0 of the ones accumulator: the CTA's sum of g per output channel
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 32) {
                float v[32];
                if (nt > 0) tmem_ld16x2(tmem + W::ONES_TMEM - ((W::ONES_TMEM >> 16) << 16) + (uint32_t)c0, v);
                else
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                if (lane == (int)W::ONES_LANE)
#pragma unroll
                    for (int e = 0; e < 32; ++e) p.part_b[blockIdx.x * 64 + c0 + e] = v[e];
            }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, W::TCOLS);
}

}  // namespace gorila
