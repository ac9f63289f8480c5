// tma_gemm.cuh — TMA-fed tcgen05 implicit GEMM (the bf16 engine of every conv / FC layer).
//
// C[i][j] = sum_r A(i, r) B(j, r). Each operand tile of one K-chunk arrives in shared memory
// through one to four cp.async.bulk.tensor (TMA) copies issued by a single producer thread:
// multi-dimensional boxes with element strides express the conv im2col windows (conv1's
// 8x8 / stride-4 taps over pixel pairs, conv2's stride 2), negative start coordinates with
// hardware zero fill express the dgrad "full" convolution (the stride-2 one decomposed into
// four phases), and a 16-byte innermost box dimension lands every tile directly in the UMMA
// canonical no-swizzle layout (8-row x 16-byte core matrices; K-major or MN-major).
// One thread issues tcgen05.mma (M = 128 per block, N = BN, K = 16) into TMEM and commits to
// per-stage "empty" mbarriers; the epilogue (all 4 warps) reads TMEM with tcgen05.ld and runs
// the fused epilogue of gemm.cuh. Split-K runs across a thread-block cluster with a DSMEM
// reduction (cluster > 1) or into fp32 partials (splits > 1, cluster == 1).
#pragma once
#include "common.cuh"
#include "gemm.cuh"
#include "layout.cuh"

namespace gorila {

// ============================================================ operand kinds
// Interface: kMN; chunk rows KC (reduction elements per chunk, multiple of 16);
// stage bytes; issue(tile, kc, dst, bar) -> bytes; desc(base, kk, mb); row(tile, r) -> global
// row index or -1 (A side only).

// K-major plain matrix X[rows][K] (row-major, ld = K): tile = TR rows, chunk = 64 columns.
// map: dims (8, rows, K/8), strides (ld*2, 16), box (8, TR, 8)  ->  smem [kgroup][row][8]
template <int TR>
struct OpMatK {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = TR * 128;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    int rows;
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, 0, tile * TR, kc * 8);
        return TR * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const {
        return umma_desc(base + mb * 2048 + kk * 2 * TR * 16, TR * 16, 128);
    }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * TR + r;
        return (r < TR && i < rows) ? i : -1;
    }
};

// MN-major plain matrix X[Krows][MN] (row-major, ld = MN): tile = TR columns, chunk = 64 rows.
// map: dims (8, Krows, MN/8), strides (ld*2, 16), box (8, 64, TR/8)  ->  smem [mngroup][k][8]
template <int TR>
struct OpMatMN {
    static constexpr bool kMN = true;
    static constexpr int KC = 64, STAGE = TR * 128;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    int mn;  // valid MN extent
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, 0, kc * 64, tile * (TR / 8));
        return TR * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc(base + kk * 256, 128, 1024); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * TR + r;
        return (r < TR && i < mn) ? i : -1;
    }
};

// conv forward im2col (K-major), C >= 8: tile = NB samples (rows = NB*OH*OW <= 128*MB),
// chunk = 64 reduction elements = 64/C taps x C channels of one kernel row.
// map over the NHWC input: dims (8, W, H, B, 64/8), strides (C*2, W*C*2, H*W*C*2, 16),
// box (8, OW*S, OH*S, NB, 8), element strides (1, S, S, 1, 1); coords (0, kx0, ky, b0, 0)
// -> smem [group][b][oy][ox][8]. With C = 32 the 8 groups span the two adjacent taps kx0, kx0+1
// (the next pixel starts 64 B later), so one 128-B aligned copy covers the chunk.
template <class SH, int MB>
struct OpConvFwd {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = MB * 128 * 128, TPC = 64 / SH::C;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    int nb, batch;
    GORILA_DEV int rows_tile() const { return nb * SH::OH * SH::OW; }
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        static_assert(SH::K % TPC == 0, "a chunk's taps lie in one kernel row");
        const int t = kc * TPC, ky = t / SH::K, kx = t - ky * SH::K;
        tma_load(&map, dst, bar, 0, kx, ky, tile * nb, 0);
        return 64 * rows_tile() * 2;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const {
        const uint32_t lbo = rows_tile() * 16;
        return umma_desc(base + mb * 2048 + kk * 2 * lbo, lbo, 128);
    }
    GORILA_DEV int row(int tile, int r) const {
        const int b = tile * nb + r / (SH::OH * SH::OW);
        return (r < rows_tile() && b < batch) ? tile * rows_tile() + r : -1;
    }
};

// conv1 forward (C = 4): K groups are pixel pairs (2 x 4 ch = 16 B). View the input as
// (8, 42 pairs, 84 rows, B, 4 pair offsets): strides (16, 672, 56448, 16), box (8, 40, 80, NB, 4),
// element strides (1, 2, 4, 1, 1). Chunk kc = kernel rows ky = 2kc, 2kc+1 (2 copies of 4 groups).
template <int MB>
struct OpConv1Fwd {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = MB * 128 * 128;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    int nb, batch;
    GORILA_DEV int rows_tile() const { return nb * H1 * H1; }
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        const int rt = rows_tile();
#pragma unroll
        for (int u = 0; u < 2; ++u) tma_load(&map, dst + u * 4 * rt * 16, bar, 0, 0, 2 * kc + u, tile * nb, 0);
        return 64 * rt * 2;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const {
        const uint32_t lbo = rows_tile() * 16;
        return umma_desc(base + mb * 2048 + kk * 2 * lbo, lbo, 128);
    }
    GORILA_DEV int row(int tile, int r) const {
        const int b = tile * nb + r / (H1 * H1);
        return (r < rows_tile() && b < batch) ? tile * rows_tile() + r : -1;
    }
};

// conv dgrad: the output gradient g (NHWC [B][OH][OW][CO], CO = 64) seen from the input
// positions (K-major), chunk = one tap x 64 output channels.
// PH < 0 (stride 1): rows = NB*H*W input pixels, map box (8, W, H, NB, 8), coords (0, -kx, -ky, b0, 0).
// PH = 0..3 (stride 2, phase py = PH/2, px = PH%2): rows = NB*10*10 pixels (2yy+py, 2xx+px),
// taps (kyi, kxi) with ky = py + 2kyi, coords (0, -kxi, -kyi, b0, 0), box (8, 10, 10, NB, 8).
// map: dims (8, OW, OH, B, 8), strides (128, OW*128, OH*OW*128, 16); zero fill out of bounds.
template <class SH, int MB>
struct OpDgrad {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = MB * 128 * 128;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    int nb, batch, phase;  // phase < 0: stride-1 layer
    GORILA_DEV int side_y() const { return phase < 0 ? SH::H : (SH::H + 1) / 2; }
    GORILA_DEV int side_x() const { return phase < 0 ? SH::W : (SH::W + 1) / 2; }
    GORILA_DEV int rows_tile() const { return nb * side_y() * side_x(); }
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        int dy, dx;
        if (phase < 0) {
            dy = kc / SH::K;
            dx = kc - dy * SH::K;
        } else {
            dy = kc >> 1;
            dx = kc & 1;
        }
        tma_load(&map, dst, bar, 0, -dx, -dy, tile * nb, 0);
        return 64 * rows_tile() * 2;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const {
        const uint32_t lbo = rows_tile() * 16;
        return umma_desc(base + mb * 2048 + kk * 2 * lbo, lbo, 128);
    }
    GORILA_DEV int row(int tile, int r) const {
        const int sy = side_y(), sx = side_x(), per = sy * sx;
        const int bb = r / per, b = tile * nb + bb;
        if (r >= rows_tile() || b >= batch) return -1;
        if (phase < 0) return tile * rows_tile() + r;
        const int rem = r - bb * per, yy = rem / sx, xx = rem - yy * sx;
        return (b * SH::H + 2 * yy + (phase >> 1)) * SH::W + 2 * xx + (phase & 1);
    }
};

// conv dgrad weight operand, MN-major over input channels c (N tile = C), chunk = one tap x 64 o.
// map over W [CO][K][K][C]: dims (8, CO, C/8, K*K), strides (R*2, 16, C*2), box (8, 64, C/8, 1)
// -> smem [cg][o][8]
template <class SH>
struct OpWdgradMN {
    static constexpr bool kMN = true;
    static constexpr int KC = 64, STAGE = SH::C * 128;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    int phase;
    GORILA_DEV uint32_t issue(int, int kc, uint32_t dst, uint64_t* bar) const {
        int t;
        if (phase < 0) t = kc;
        else t = ((phase >> 1) + 2 * (kc >> 1)) * SH::K + (phase & 1) + 2 * (kc & 1);
        tma_load(&map, dst, bar, 0, 0, 0, t);
        return SH::C * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc(base + kk * 256, 128, 1024); }
};

// weight-gradient input operand (MN-major over r = (ky, kx, c), tile = 128 r), chunk = the
// output pixels of one sample (conv2 / conv3; KC = 96 / 64 rows, the tail multiplies zeros of
// the gradient operand) -> smem [group][pixel][8], group stride SBO = OH*OW*16.
// map over the NHWC input: dims (8, W, H, B, G), box (8, OW*S, OH*S, 1, G), es (1, S, S, 1, 1);
// conv3: G = 8, one copy per tap (2 per tile); conv2: G = 16 groups = the 4 adjacent taps of
// one kernel row (one copy per tile).
template <class SH, int KC_>
struct OpWgradIn {
    static constexpr bool kMN = true;
    static constexpr int KC = KC_, TPT = 128 / SH::C, NPIX = SH::OH * SH::OW;
    static constexpr int STAGE = (16 * NPIX * 16 + KC * 16 + 127) / 128 * 128;
    // the K-tail of the last group reads past the copies: that slack is zeroed once (the tail
    // rows multiply zero rows of the gradient operand, and must not hold NaN patterns)
    static constexpr int WRITTEN = 16 * NPIX * 16;
    alignas(64) CUtensorMap map;
    static constexpr bool ROW = SH::K == TPT;  // the tile is one kernel row: a single copy
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        if (ROW) {
            tma_load(&map, dst, bar, 0, 0, tile, kc, 0);
        } else {
#pragma unroll
            for (int u = 0; u < TPT; ++u) {
                const int t = tile * TPT + u, ky = t / SH::K, kx = t - ky * SH::K;
                tma_load(&map, dst + u * (SH::C / 8) * NPIX * 16, bar, 0, kx, ky, kc, 0);
            }
        }
        return 128 * NPIX * 2;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc(base + kk * 256, 128, NPIX * 16); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * 128 + r;
        return i < SH::R ? i : -1;
    }
};

// conv1 weight-gradient input operand: groups (ky, pair) over 4 kernel rows per tile; chunk =
// 4 output rows (80 pixels) of one sample. Same pair view as OpConv1Fwd, box (8, 40, 16, 1, 4).
struct OpWgradIn1 {
    static constexpr bool kMN = true;
    static constexpr int KC = 80, NPIX = 80;
    static constexpr int STAGE = 16 * NPIX * 16 + 128;
    static constexpr int WRITTEN = 16 * NPIX * 16;
    alignas(64) CUtensorMap map;
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        const int b = kc / 5, oy0 = (kc - b * 5) * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) tma_load(&map, dst + u * 4 * NPIX * 16, bar, 0, 0, 4 * oy0 + tile * 4 + u, b, 0);
        return 128 * NPIX * 2;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc(base + kk * 256, 128, NPIX * 16); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * 128 + r;
        return i < K1 ? i : -1;
    }
};

// weight-gradient output-gradient operand g [B][NPIX][CO] (MN-major over o, N tile = CO),
// chunk = the same pixels as the input operand; rows past the sample are zero filled.
// per-sample chunks: dims (8, NPIX, B, CO/8), box (8, KC, 1, CO/8); flat chunks (conv1):
// dims (8, B*NPIX, CO/8), box (8, KC, CO/8).
template <int CO, int KC_, bool FLAT>
struct OpWgradOut {
    static constexpr bool kMN = true;
    static constexpr int KC = KC_, STAGE = CO * KC * 2;
    static constexpr int WRITTEN = STAGE;  // bytes a stage's copies define
    alignas(64) CUtensorMap map;
    GORILA_DEV uint32_t issue(int, int kc, uint32_t dst, uint64_t* bar) const {
        if (FLAT) tma_load(&map, dst, bar, 0, kc * KC, 0);
        else tma_load(&map, dst, bar, 0, 0, kc, 0);
        return CO * KC * 2;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc(base + kk * 256, 128, KC * 16); }
};

// ---------------------------------------------------------------- swizzled K-major operands
// (fewer, larger TMA requests: one 128-B (64-B) row per output row and K-chunk)

// K-major plain matrix X[rows][K]: map dims (K, rows), box (64, TR), SWIZZLE_128B -> [row][128 B]
template <int TR>
struct OpMatKS {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = TR * 128, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    int rows;
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        tma_load(&map, dst, bar, kc * 64, tile * TR);
        return TR * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const { return umma_desc_sw(base + mb * 16384 + kk * 32, 128); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * TR + r;
        return (r < TR && i < rows) ? i : -1;
    }
};

// conv2 / conv3 forward im2col, SWIZZLE_128B: one 128-B row (64 K) per output pixel and chunk.
// conv3 (C = 64): dims (64, W, H, B), box (64, OW, OH, NB), coords (0, kx, ky, b0).
// conv2 (C = 32): the chunk = taps (ky, kx0), (ky, kx0+1) = two adjacent pixels = 128 contiguous
// bytes: dims (64, W-1, H, B) with x stride C*2, box (64, OW*2, OH*2, NB), element strides (1,2,2,1).
template <class SH, int MB>
struct OpConvFwdS {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = MB * 128 * 128, WRITTEN = STAGE, TPC = 64 / SH::C;
    alignas(64) CUtensorMap map;
    int nb, batch;
    GORILA_DEV int rows_tile() const { return nb * SH::OH * SH::OW; }
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        const int t = kc * TPC, ky = t / SH::K, kx = t - ky * SH::K;
        tma_load(&map, dst, bar, 0, kx, ky, tile * nb);
        return rows_tile() * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const { return umma_desc_sw(base + mb * 16384 + kk * 32, 128); }
    GORILA_DEV int row(int tile, int r) const {
        const int b = tile * nb + r / (SH::OH * SH::OW);
        return (r < rows_tile() && b < batch) ? tile * rows_tile() + r : -1;
    }
};

// conv1 forward, SWIZZLE_64B: one 64-B row (the 8 pixels x 4 channels of one kernel row) per
// output pixel, two kernel rows per chunk. View s as (32, 20 ox [stride 32 B], 84 y, B), box
// (32, 20, 80, NB), element strides (1, 1, 4, 1): x = 4*ox .. 4*ox+7 at row 4*oy + ky.
template <int MB>
struct OpConv1FwdS {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = 2 * MB * 128 * 64, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    int nb, batch;
    GORILA_DEV int rows_tile() const { return nb * H1 * H1; }
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
#pragma unroll
        for (int u = 0; u < 2; ++u) tma_load(&map, dst + u * MB * 128 * 64, bar, 0, 0, 2 * kc + u, tile * nb);
        return 2 * rows_tile() * 64;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const {
        return umma_desc_sw(base + (kk >> 1) * MB * 128 * 64 + mb * 8192 + (kk & 1) * 32, 64);
    }
    GORILA_DEV int row(int tile, int r) const {
        const int b = tile * nb + r / (H1 * H1);
        return (r < rows_tile() && b < batch) ? tile * rows_tile() + r : -1;
    }
};

// conv dgrad (shifted output gradient, CO = 64 = one 128-B row per tap), SWIZZLE_128B:
// dims (64, OW, OH, B), box (8.. -> 64, side_x, side_y, NB), coords (0, -dx, -dy, b0)
template <class SH, int MB>
struct OpDgradS {
    static constexpr bool kMN = false;
    static constexpr int KC = 64, STAGE = MB * 128 * 128, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    int nb, batch, phase;
    GORILA_DEV int side_y() const { return phase < 0 ? SH::H : (SH::H + 1) / 2; }
    GORILA_DEV int side_x() const { return phase < 0 ? SH::W : (SH::W + 1) / 2; }
    GORILA_DEV int rows_tile() const { return nb * side_y() * side_x(); }
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        int dy, dx;
        if (phase < 0) {
            dy = kc / SH::K;
            dx = kc - dy * SH::K;
        } else {
            dy = kc >> 1;
            dx = kc & 1;
        }
        tma_load(&map, dst, bar, 0, -dx, -dy, tile * nb);
        return rows_tile() * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int mb) const { return umma_desc_sw(base + mb * 16384 + kk * 32, 128); }
    GORILA_DEV int row(int tile, int r) const {
        const int sy = side_y(), sx = side_x(), per = sy * sx;
        const int bb = r / per, b = tile * nb + bb;
        if (r >= rows_tile() || b >= batch) return -1;
        if (phase < 0) return tile * rows_tile() + r;
        const int rem = r - bb * per, yy = rem / sx, xx = rem - yy * sx;
        return (b * SH::H + 2 * yy + (phase >> 1)) * SH::W + 2 * xx + (phase & 1);
    }
};

// ---------------------------------------------------------------- swizzled MN-major operands
// smem [MN block][K row][64 (32) elements]: 128-B (64-B) rows, one TMA box per MN block.

// MN-major plain matrix X[Krows][MN]: map dims (MN, Krows), box (64, 64), SWIZZLE_128B;
// tile = TR columns (TR/64 boxes), chunk = 64 K rows
template <int TR>
struct OpMatMNS {
    static constexpr bool kMN = true, ZERO_ALL = false;
    static constexpr int KC = 64, STAGE = TR * 128, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    int mn;
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
#pragma unroll
        for (int h = 0; h < TR / 64; ++h) tma_load(&map, dst + h * 8192, bar, tile * TR + h * 64, kc * 64);
        return TR * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc_mn_sw(base + kk * 2048, 8192, 128); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * TR + r;
        return (r < TR && i < mn) ? i : -1;
    }
};

// conv dgrad weight operand, MN-major over c (N = C): chunk = one tap x 64 o.
// map over W [CO][K][K][C]: dims (C, CO, K*K), strides (R*2, C*2), box (C, 64, 1) -> [o][C]
template <class SH>
struct OpWdgradMNS {
    static constexpr bool kMN = true, ZERO_ALL = false;
    static constexpr int RB = SH::C * 2;  // row bytes (128 or 64)
    static constexpr int KC = 64, STAGE = 64 * RB, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    int phase;
    GORILA_DEV uint32_t issue(int, int kc, uint32_t dst, uint64_t* bar) const {
        int t;
        if (phase < 0) t = kc;
        else t = ((phase >> 1) + 2 * (kc >> 1)) * SH::K + (phase & 1) + 2 * (kc & 1);
        tma_load(&map, dst, bar, 0, 0, t);
        return 64 * RB;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc_mn_sw(base + kk * 16 * RB, 0, RB); }
};

// conv2 / conv3 weight-gradient input operand, MN-major over r = (ky, kx, c), tile = 128 r =
// two MN blocks of 64 (conv3: one tap each; conv2: two adjacent taps = pixels x, x+1 each);
// chunk = the output pixels of one sample (KC = 64 / 96 rows; the tail rows stay zero and meet
// zero rows of the gradient operand). Map as fwd_map_sw with NB = 1.
template <class SH, int KC_>
struct OpWgradInS {
    static constexpr bool kMN = true, ZERO_ALL = true;
    static constexpr int KC = KC_, NPIX = SH::OH * SH::OW, TPB = 64 / SH::C;  // taps per MN block
    static constexpr int REG = KC * 128;                                      // bytes of one MN block
    static constexpr int STAGE = 2 * REG, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = (tile * 2 + h) * TPB, ky = t / SH::K, kx = t - ky * SH::K;
            tma_load(&map, dst + h * REG, bar, 0, kx, ky, kc);
        }
        return 2 * NPIX * 128;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc_mn_sw(base + kk * 2048, REG, 128); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * 128 + r;
        return i < SH::R ? i : -1;
    }
};

// conv1 weight-gradient input operand, MN-major over r = (ky, kx, c): tile = 4 kernel rows = 4
// MN blocks of 32 (8 pixels x 4 channels, 64-B rows, SWIZZLE_64B); chunk = 4 output rows (80
// pixels) of one sample. Map as conv1_map_sw with NB = 1 and a box of 4 output rows.
struct OpWgradIn1S {
    static constexpr bool kMN = true, ZERO_ALL = false;
    static constexpr int KC = 80, REG = 80 * 64, STAGE = 4 * REG, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    GORILA_DEV uint32_t issue(int tile, int kc, uint32_t dst, uint64_t* bar) const {
        const int b = kc / 5, oy0 = (kc - b * 5) * 4;
#pragma unroll
        for (int u = 0; u < 4; ++u) tma_load(&map, dst + u * REG, bar, 0, 0, 4 * oy0 + tile * 4 + u, b);
        return 4 * REG;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc_mn_sw(base + kk * 1024, REG, 64); }
    GORILA_DEV int row(int tile, int r) const {
        const int i = tile * 128 + r;
        return i < K1 ? i : -1;
    }
};

// weight-gradient output-gradient operand g [B][NPIX][CO], MN-major over o (N = CO), rows of
// CO*2 bytes (SWIZZLE_128B / 64B); per-sample chunks: dims (CO, NPIX, B), box (CO, KC, 1) (rows
// past the sample zero filled); flat chunks (conv1): dims (CO, B*NPIX), box (CO, KC).
template <int CO, int KC_, bool FLAT>
struct OpWgradOutS {
    static constexpr bool kMN = true, ZERO_ALL = false;
    static constexpr int RB = CO * 2, KC = KC_, STAGE = KC * RB, WRITTEN = STAGE;
    alignas(64) CUtensorMap map;
    GORILA_DEV uint32_t issue(int, int kc, uint32_t dst, uint64_t* bar) const {
        if (FLAT) tma_load(&map, dst, bar, 0, kc * KC);
        else tma_load(&map, dst, bar, 0, 0, kc);
        return KC * RB;
    }
    GORILA_DEV uint64_t desc(uint32_t base, int kk, int) const { return umma_desc_mn_sw(base + kk * 16 * RB, 0, RB); }
};

// ============================================================ the engine
template <class O, class = void>
struct zero_all : std::false_type {};
template <class O>
struct zero_all<O, std::void_t<decltype(O::ZERO_ALL)>> : std::integral_constant<bool, O::ZERO_ALL> {};

template <class OA, class OB, class EP>
struct TmaProb {
    OA a;
    OB b;
    EP ep;
};

template <class OA, class OB, class EP>
struct TmaBatch {
    TmaProb<OA, OB, EP> prob[4];
    int nchunks;           // K-chunks of the whole reduction
    int splits;            // reduction split (grid.z = nprob * splits)
    int chunks_per_split;
    int cluster;           // > 1: the splits of a tile form a cluster and reduce through DSMEM
    int N;                 // output columns (epilogue bound)
};

template <int BN, int MB, class OA, class OB>
struct TmaCfg {
    static constexpr int A_ST = (OA::STAGE + 1023) / 1024 * 1024;
    static constexpr int B_ST = (OB::STAGE + 1023) / 1024 * 1024;
    static constexpr int BUDGET = 200 * 1024;
    static constexpr int STAGES = (A_ST + B_ST) * 4 <= BUDGET ? 4 : (A_ST + B_ST) * 3 <= BUDGET ? 3 : 2;
    static constexpr int PIPE = STAGES * (A_ST + B_ST);
    static constexpr int RED = MB == 1 ? tc_red_bytes(BN) + tc_slice_bytes(BN) : 0;
    static constexpr int SMEM = (PIPE > RED ? PIPE : RED) + 128 + 1024;  // + alignment slack
    static constexpr uint32_t TCOLS = tmem_cols_for(MB * BN);
    static_assert(MB * BN <= 256, "TMEM columns");
};

template <int BN, int MB, class OA, class OB, class EP>
__global__ void __launch_bounds__(128) gemm_tma(const __grid_constant__ TmaBatch<OA, OB, EP> p) {
    using CFG = TmaCfg<BN, MB, OA, OB>;
    constexpr int STAGES = CFG::STAGES;
    static_assert(OA::KC == OB::KC && OA::KC % 16 == 0, "chunk rows");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // swizzle atoms (and so every stage) must sit on 1024-B boundaries of the shared window
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + CFG::SMEM - 128);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    GTRACE(0);
    const int prob = blockIdx.z / p.splits, split = blockIdx.z - prob * p.splits;
    const TmaProb<OA, OB, EP>& P = p.prob[prob];
    const int ta = blockIdx.x, tb = blockIdx.y;
    const int kc0 = split * p.chunks_per_split;
    const int nK = max(0, min(p.nchunks, kc0 + p.chunks_per_split) - kc0);

    if (warp == 0) tmem_alloc(tmem_slot, CFG::TCOLS);
    if (OA::WRITTEN < CFG::A_ST || zero_all<OA>::value)  // zero the never-copied rows of the A stages
        for (int s = 0; s < STAGES; ++s)
            for (int o = (zero_all<OA>::value ? 0 : OA::WRITTEN) + tid * 16; o < CFG::A_ST; o += 128 * 16)
                *reinterpret_cast<uint4*>(smem + s * (CFG::A_ST + CFG::B_ST) + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid == 32) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
        tma_prefetch_desc(&P.a.map);
        tma_prefetch_desc(&P.b.map);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    GTRACE(1);
    pdl_wait();     // operands are produced by the preceding kernel(s)
    pdl_trigger();  // the next kernel may start its prologue
    GTRACE(2);
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t IDESC =
        umma_idesc_bf16(TC_BM, BN) | (OA::kMN ? (1u << 15) : 0u) | (OB::kMN ? (1u << 16) : 0u);
    const uint32_t sbase = smem_u32(smem);

    if (warp == 0) {  // (warp-uniform branch: keeps the MMA warp's branch below uniform)
        if (lane == 0) {  // TMA producer
            for (int kc = 0; kc < nK; ++kc) {
                const int s = kc % STAGES;
                if (kc >= STAGES) mbar_wait(&empty[s], ((kc / STAGES) - 1) & 1);
                const uint32_t a_dst = sbase + s * (CFG::A_ST + CFG::B_ST), b_dst = a_dst + CFG::A_ST;
                // issue first, then arrive with the transaction count (full boxes, zero fill included);
                // the phase cannot complete before this arrival
                uint32_t bytes = P.a.issue(ta, kc0 + kc, a_dst, &full[s]);
                bytes += P.b.issue(tb, kc0 + kc, b_dst, &full[s]);
                mbar_expect_tx(&full[s], bytes);
                GTRACE(8 + (kc & 7));
            }
        }
    } else if (warp == 1) {  // MMA issuer (warp-uniform; one elected lane issues)
        // a K step / M-block only moves a descriptor's start address: per stage one base
        // descriptor plus these address-field deltas
        const uint32_t tmem_u = uniform_u32(tmem), sbase_u = uniform_u32(sbase);
        constexpr int KS = OA::KC / 16;
        uint32_t adl[KS][MB], bdl[KS];
        const uint64_t a00 = P.a.desc(0, 0, 0), b00 = P.b.desc(0, 0, 0);
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            bdl[kk] = uniform_u32((uint32_t)(P.b.desc(0, kk, 0) - b00));
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) adl[kk][mb] = uniform_u32((uint32_t)(P.a.desc(0, kk, mb) - a00));
        }
        for (int kc = 0; kc < nK; ++kc) {
            const int s = kc % STAGES;
            mbar_wait(&full[s], (kc / STAGES) & 1);
            tc_fence_after();
            const uint32_t a_base = sbase_u + s * (CFG::A_ST + CFG::B_ST), b_base = a_base + CFG::A_ST;
            const uint64_t ad0 = uniform_u64(P.a.desc(a_base, 0, 0)), bd0 = uniform_u64(P.b.desc(b_base, 0, 0));
#pragma unroll
            for (int kk = 0; kk < KS; ++kk) {
#pragma unroll
                for (int mb = 0; mb < MB; ++mb)
                    umma_bf16_w(tmem_u + mb * BN, ad0 + adl[kk][mb], bd0 + bdl[kk], IDESC, (kc > 0 || kk > 0) ? 1u : 0u);
            }
            umma_commit_w(&empty[s]);
        }
        if (nK > 0) umma_commit_w(done);
    }
    __syncwarp();
    GTRACE(3);
    // the functor is copied to registers once: indexed by the problem, its fields would otherwise
    // be re-read from the parameter bank before every store (the compiler cannot rule out aliasing)
    const EP ep = P.ep;
    using PT = EpPre<EP>;
    constexpr int NC = BN / 16, PD = NC < 4 ? NC : 4;  // epilogue prefetch distance (chunks)
    typename PT::type pre[PD];
    const int i0 = P.a.row(ta, warp * 32 + lane);
    if (!(MB == 1 && p.cluster > 1))  // first chunks' epilogue inputs in flight during the main loop
#pragma unroll
        for (int d = 0; d < PD; ++d)
            if (i0 >= 0) pre[d] = PT::load(ep, i0, tb * BN + d * 16);
    if (nK > 0) mbar_wait(done, 0);
    tc_fence_after();
    GTRACE(4);

    // ---------------------------------------------------------------- epilogue
    if (MB == 1 && p.cluster > 1) {
        float* red = reinterpret_cast<float*>(smem);  // the stage ring is dead now
        const int lrow = warp * 32 + lane;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16];
            if (nK > 0) tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            else
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = 0.f;
            float4* dst = reinterpret_cast<float4*>(red + ((c0 / 16) * TC_BM + lrow) * 20);
#pragma unroll
            for (int e = 0; e < 4; ++e) dst[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
        }
        cluster_sync();
        const int CL = p.cluster, rows_per = TC_BM / CL;
        const int q = (int)cluster_ctarank();
        float* slice = reinterpret_cast<float*>(smem + tc_red_bytes(BN));
        const int n4 = rows_per * BN / 4;
        // every float4 of this CTA's row slice: all CL peer reads in flight before any add
        for (int it0 = 0; it0 < n4; it0 += 128 * 2) {
            float4 x[2][16];
            uint32_t ad[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int it = it0 + h * 128 + tid;
                const int r_loc = it / (BN / 4), c4 = (it % (BN / 4)) * 4;
                ad[h] = smem_u32(red + ((c4 / 16) * TC_BM + q * rows_per + r_loc) * 20 + (c4 % 16));
                if (it < n4)
#pragma unroll
                    for (int pr = 0; pr < 16; ++pr)
                        if (pr < CL) x[h][pr] = dsmem_ld4(dsmem_map(ad[h], (uint32_t)pr));
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int it = it0 + h * 128 + tid;
                if (it >= n4) continue;
                const int r_loc = it / (BN / 4), c4 = (it % (BN / 4)) * 4;
                float4 acc = x[h][0];
#pragma unroll
                for (int pr = 1; pr < 16; ++pr)
                    if (pr < CL) {
                        acc.x += x[h][pr].x; acc.y += x[h][pr].y; acc.z += x[h][pr].z; acc.w += x[h][pr].w;
                    }
                *reinterpret_cast<float4*>(slice + r_loc * (BN + 4) + c4) = acc;
            }
        }
        __syncthreads();
        for (int item = tid; item < rows_per * (BN / 16); item += 128) {
            const int r_loc = item % rows_per, c0 = (item / rows_per) * 16;
            const int i = P.a.row(ta, q * rows_per + r_loc);
            float v[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = slice[r_loc * (BN + 4) + c0 + e];
            if (i >= 0 && tb * BN + c0 < p.N) ep.apply16(i, tb * BN + c0, v, 0);
        }
        cluster_sync();
    } else {
#pragma unroll 1
        for (int mb = 0; mb < MB; ++mb) {
            const int i = P.a.row(ta, mb * 128 + warp * 32 + lane);
            if (mb > 0)
#pragma unroll
                for (int d = 0; d < PD; ++d)
                    if (i >= 0) pre[d] = PT::load(ep, i, tb * BN + d * 16);
            GTRACE(16);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const int c0 = c * 16;
                float v[16];
                if (nK > 0) {
                    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(mb * BN + c0), v);
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0.f;
                }
                const typename PT::type cur = pre[c % PD];
                if (c + PD < NC && i >= 0) pre[c % PD] = PT::load(ep, i, tb * BN + c0 + PD * 16);
                if (c0 < 64) GTRACE(17 + 2 * (c0 / 16));
                if (i >= 0 && tb * BN + c0 < p.N) PT::apply(ep, i, tb * BN + c0, v, cur, split);
                if (c0 < 64) GTRACE(18 + 2 * (c0 / 16));
            }
        }
    }
    GTRACE(5);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, CFG::TCOLS);
    GTRACE(6);
}

// ============================================================ persistent engine
// One CTA per SM slot loops over the tiles (prob, split, tb, ta) of the launch, ta fastest.
// Warp 0: TMA producer (stage ring continues across tiles). Warp 1: MMA issuer into one of two
// TMEM accumulators. Warps 2..5: epilogue (warp w reads TMEM lanes 32*(w%4)..): tile t's epilogue
// overlaps tile t+1's loads and MMAs. No cluster reduction here (launches with cluster > 1 use
// gemm_tma above).
template <int BN, int MB, class OA, class OB>
struct TmaPCfg {
    static constexpr int A_ST = TmaCfg<BN, MB, OA, OB>::A_ST;
    static constexpr int B_ST = TmaCfg<BN, MB, OA, OB>::B_ST;
    static constexpr int BUDGET = 200 * 1024;
    static constexpr int STAGES = (A_ST + B_ST) * 6 <= BUDGET   ? 6
                                  : (A_ST + B_ST) * 4 <= BUDGET ? 4
                                  : (A_ST + B_ST) * 3 <= BUDGET ? 3
                                                                : 2;
    static constexpr int SMEM = STAGES * (A_ST + B_ST) + 256 + 1024;
    static constexpr uint32_t ACC = MB * BN;  // columns of one accumulator
    static constexpr uint32_t TCOLS = tmem_cols_for(2 * MB * BN);
    static_assert(2 * MB * BN <= 512, "TMEM columns");
    static constexpr int THREADS = 192;
};

template <int BN, int MB, class OA, class OB, class EP>
__global__ void __launch_bounds__(192) gemm_tma_p(const __grid_constant__ TmaBatch<OA, OB, EP> p, int tilesA,
                                                  int tilesB, int nprob) {
    using CFG = TmaPCfg<BN, MB, OA, OB>;
    constexpr int STAGES = CFG::STAGES;
    static_assert(OA::KC == OB::KC && OA::KC % 16 == 0, "chunk rows");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + CFG::SMEM - 256);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;  // [2] MMA -> epilogue
    uint64_t* acc_empty = acc_full + 2;   // [2] epilogue -> MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int tid = threadIdx.x, warp = warp_uniform(), lane = tid & 31;
    const int ntiles = tilesA * tilesB * nprob * p.splits;
    if (warp == 0) tmem_alloc(tmem_slot, CFG::TCOLS);
    if (OA::WRITTEN < CFG::A_ST || zero_all<OA>::value)  // zero the never-copied rows of the A stages
        for (int s = 0; s < STAGES; ++s)
            for (int o = (zero_all<OA>::value ? 0 : OA::WRITTEN) + tid * 16; o < CFG::A_ST; o += CFG::THREADS * 16)
                *reinterpret_cast<uint4*>(smem + s * (CFG::A_ST + CFG::B_ST) + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid == 32) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_trigger();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sbase = smem_u32(smem);
    constexpr uint32_t IDESC =
        umma_idesc_bf16(TC_BM, BN) | (OA::kMN ? (1u << 15) : 0u) | (OB::kMN ? (1u << 16) : 0u);

    // tile t -> (prob, split, tb, ta)
    auto decode = [&](int t, int& prob, int& split, int& ta, int& tb) {
        ta = t % tilesA;
        t /= tilesA;
        tb = t % tilesB;
        t /= tilesB;
        split = t % p.splits;
        prob = t / p.splits;
    };
    auto chunks = [&](int split, int& kc0) {
        kc0 = split * p.chunks_per_split;
        return max(0, min(p.nchunks, kc0 + p.chunks_per_split) - kc0);
    };

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            uint32_t it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int prob, split, ta, tb, kc0;
                decode(t, prob, split, ta, tb);
                const int nK = chunks(split, kc0);
                const TmaProb<OA, OB, EP>& P = p.prob[prob];
                for (int kc = 0; kc < nK; ++kc, ++it) {
                    const int s = it % STAGES;
                    if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
                    const uint32_t a_dst = sbase + s * (CFG::A_ST + CFG::B_ST), b_dst = a_dst + CFG::A_ST;
                    uint32_t bytes = P.a.issue(ta, kc0 + kc, a_dst, &full[s]);
                    bytes += P.b.issue(tb, kc0 + kc, b_dst, &full[s]);
                    mbar_expect_tx(&full[s], bytes);
                }
            }
        }
    } else if (warp == 1) {
        {  // MMA issuer (warp-uniform; one elected lane issues)
            const uint32_t tmem_u = uniform_u32(tmem), sbase_u = uniform_u32(sbase);
            uint32_t it = 0, tl = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                int prob, split, ta, tb, kc0;
                decode(t, prob, split, ta, tb);
                const int nK = chunks(split, kc0);
                const TmaProb<OA, OB, EP>& P = p.prob[prob];
                const uint32_t buf = tl & 1;
                if (tl >= 2) mbar_wait(&acc_empty[buf], ((tl >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t acc = tmem_u + buf * CFG::ACC;
                constexpr int KS = OA::KC / 16;  // descriptor deltas of the K steps / M-blocks
                uint32_t adl[KS][MB], bdl[KS];
                const uint64_t a00 = P.a.desc(0, 0, 0), b00 = P.b.desc(0, 0, 0);
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) {
                    bdl[kk] = (uint32_t)(P.b.desc(0, kk, 0) - b00);
#pragma unroll
                    for (int mb = 0; mb < MB; ++mb) adl[kk][mb] = (uint32_t)(P.a.desc(0, kk, mb) - a00);
                }
                for (int kc = 0; kc < nK; ++kc, ++it) {
                    const int s = it % STAGES;
                    mbar_wait(&full[s], (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a_base = sbase_u + s * (CFG::A_ST + CFG::B_ST), b_base = a_base + CFG::A_ST;
                    const uint64_t ad0 = P.a.desc(a_base, 0, 0), bd0 = P.b.desc(b_base, 0, 0);
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
                        for (int mb = 0; mb < MB; ++mb)
                            umma_bf16_w(acc + mb * BN, ad0 + adl[kk][mb], bd0 + bdl[kk], IDESC,
                                        (kc > 0 || kk > 0) ? 1u : 0u);
                    umma_commit_w(&empty[s]);
                }
                umma_commit_w(&acc_full[buf]);  // also arrives when the tile had no chunks
            }
        }
    } else {  // epilogue warps 2..5
        const int quad = warp & 3;
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            int prob, split, ta, tb, kc0;
            decode(t, prob, split, ta, tb);
            const int nK = chunks(split, kc0);
            const TmaProb<OA, OB, EP>& P = p.prob[prob];
            const EP ep = P.ep;
            using PT = EpPre<EP>;
            constexpr int NC = BN / 16, PD = NC < 4 ? NC : 4;  // epilogue prefetch distance (chunks)
            typename PT::type pre[PD];
            const uint32_t buf = tl & 1;
            {  // the first chunks' epilogue inputs are requested before the accumulator is ready
                const int i = P.a.row(ta, quad * 32 + lane);
#pragma unroll
                for (int d = 0; d < PD; ++d)
                    if (i >= 0) pre[d] = PT::load(ep, i, tb * BN + d * 16);
            }
            mbar_wait(&acc_full[buf], (tl >> 1) & 1);
            tc_fence_after();
            const uint32_t acc = tmem + buf * CFG::ACC + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
            for (int mb = 0; mb < MB; ++mb) {
                const int i = P.a.row(ta, mb * 128 + quad * 32 + lane);
                if (mb > 0)
#pragma unroll
                    for (int d = 0; d < PD; ++d)
                        if (i >= 0) pre[d] = PT::load(ep, i, tb * BN + d * 16);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const int c0 = c * 16;
                    float v[16];
                    if (nK > 0) {
                        tmem_ld16(acc + (uint32_t)(mb * BN + c0), v);
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = 0.f;
                    }
                    const typename PT::type cur = pre[c % PD];
                    if (c + PD < NC && i >= 0) pre[c % PD] = PT::load(ep, i, tb * BN + c0 + PD * 16);
                    if (i >= 0 && tb * BN + c0 < p.N) PT::apply(ep, i, tb * BN + c0, v, cur, split);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, CFG::TCOLS);
}

}  // namespace gorila
