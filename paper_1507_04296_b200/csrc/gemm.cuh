// gemm.cuh — the contraction engine of the learner update.
//
// Every conv / FC layer of the Nature-DQN forward and backward (Eq.2)
// is one "implicit GEMM"  C[i][j] = sum_r A(i, r) * B(j, r)  whose operands are
// produced on the fly by a loader (im2col of an NHWC activation, a shifted output
// gradient for dgrad, a plain row-major matrix) and whose result goes through a
// fused epilogue (scale, bias, ReLU, ReLU-mask, bf16 rounding, transposed gradient
// store, split-K partials).
//
// Loaders are either K-major (8 consecutive reduction elements of one row are
// contiguous: forward im2col, dgrad, weights) or MN-major (8 consecutive rows at one
// reduction index are contiguous: the weight-gradient operands, whose reduction runs
// over batch x pixels). Both are staged with 16-byte vector loads into the matching
// UMMA canonical (SWIZZLE_NONE) shared-memory layout.
//
// gemm_simt (fp32 FFMA tiles) runs the fp32 check mode (parity 1e-5) on these loaders and
// epilogues; the bf16 path runs the tcgen05 engines of tma_gemm.cuh / shift_gemm.cuh / tower.cuh,
// which share the epilogues and the split / cluster helpers below.
#pragma once
#include "common.cuh"
#include "layout.cuh"

namespace gorila {

// compile-time conv geometry (valid padding): input H x W x C, kernel K, stride S
template <int H_, int W_, int C_, int K_, int S_, int CO_>
struct ConvShape {
    static constexpr int H = H_, W = W_, C = C_, K = K_, S = S_, CO = CO_;
    static constexpr int OH = (H - K) / S + 1, OW = (W - K) / S + 1;
    static constexpr int R = K * K * C;    // forward / wgrad reduction (ky, kx, c)
    static constexpr int RD = K * K * CO;  // dgrad reduction (ky, kx, o)
};
using Conv1 = ConvShape<IMG, IMG, NSTACK, C1_K, C1_S, C1_OUT>;
using Conv2 = ConvShape<H1, H1, C1_OUT, C2_K, C2_S, C2_OUT>;
using Conv3 = ConvShape<H2, H2, C2_OUT, C3_K, C3_S, C3_OUT>;

// ====================================================================== loaders

template <typename T>
struct LdRows {  // K-major: value(i, r) = X[i][r] (row-major, leading dimension ld)
    static constexpr bool kMN = false;
    const T* x;
    int64_t ld;
    int rows, cols;
    GORILA_DEV float load(int i, int r) const { return (i < rows && r < cols) ? tof(x[(int64_t)i * ld + r]) : 0.f; }
    GORILA_DEV const T* src8(int i, int r0) const {
        return (i >= rows || r0 >= cols) ? nullptr : x + (int64_t)i * ld + r0;
    }
    GORILA_DEV const void* gptr() const { return x; }  // any valid global address (zero-fill source)
};

template <typename T>
struct LdRowsMN {  // MN-major: value(i, r) = X[r][i]; src8(i0, r) = &X[r][i0] (8 consecutive i)
    static constexpr bool kMN = true;
    const T* x;
    int64_t ld;
    int rows, cols;  // i extent (multiple of 8), r extent
    GORILA_DEV float load(int i, int r) const { return (i < rows && r < cols) ? tof(x[(int64_t)r * ld + i]) : 0.f; }
    GORILA_DEV const T* src8(int i0, int r) const {
        return (i0 >= rows || r >= cols) ? nullptr : x + (int64_t)r * ld + i0;
    }
    GORILA_DEV const void* gptr() const { return x; }  // any valid global address (zero-fill source)
};

// im2col of an NHWC input: value(m = (b, oy, ox), r = (ky*K + kx)*C + c) = in[b][oy*S+ky][ox*S+kx][c]
template <typename SH>
GORILA_DEV int64_t conv_in_addr(int m, int r) {
    const int b = m / (SH::OH * SH::OW), p = m - b * (SH::OH * SH::OW);
    const int oy = p / SH::OW, ox = p - oy * SH::OW;
    const int ky = r / (SH::K * SH::C), rem = r - ky * (SH::K * SH::C);
    const int kx = rem / SH::C, c = rem - kx * SH::C;
    return (((int64_t)b * SH::H + oy * SH::S + ky) * SH::W + ox * SH::S + kx) * SH::C + c;
}

template <typename T, typename SH>
struct LdConvIn {  // K-major forward operand (8 consecutive r = same pixel channels, or 2 pixels x 4 ch)
    static constexpr bool kMN = false;
    const T* in;
    int M;
    GORILA_DEV float load(int m, int r) const { return (m < M && r < SH::R) ? tof(in[conv_in_addr<SH>(m, r)]) : 0.f; }
    GORILA_DEV const T* src8(int m, int r0) const {
        return (m >= M || r0 >= SH::R) ? nullptr : in + conv_in_addr<SH>(m, r0);
    }
    GORILA_DEV const void* gptr() const { return in; }  // any valid global address (zero-fill source)
};

template <typename T, typename SH>
struct LdConvInMN {  // MN-major weight-gradient operand: value(i = r, red = m); src8(r0, m)
    static constexpr bool kMN = true;
    const T* in;
    int M;
    GORILA_DEV float load(int r, int m) const { return (m < M && r < SH::R) ? tof(in[conv_in_addr<SH>(m, r)]) : 0.f; }
    GORILA_DEV const T* src8(int r0, int m) const {
        return (m >= M || r0 >= SH::R) ? nullptr : in + conv_in_addr<SH>(m, r0);
    }
    GORILA_DEV const void* gptr() const { return in; }  // any valid global address (zero-fill source)
};

// conv dgrad operand: output gradient g (NHWC [B][OH][OW][CO]) seen from input position
// i = (b, y, x), r = (ky*K + kx)*CO + o: g[b][(y-ky)/S][(x-kx)/S][o] if that tap exists, else 0
template <typename SH>
GORILA_DEV int64_t dgrad_addr(int i, int r) {
    const int b = i / (SH::H * SH::W), p = i - b * (SH::H * SH::W);
    const int y = p / SH::W, x = p - y * SH::W;
    const int ky = r / (SH::K * SH::CO), rem = r - ky * (SH::K * SH::CO);
    const int kx = rem / SH::CO, o = rem - kx * SH::CO;
    const int ty = y - ky, tx = x - kx;
    if (ty < 0 || tx < 0 || ty % SH::S || tx % SH::S) return -1;
    const int oy = ty / SH::S, ox = tx / SH::S;
    if (oy >= SH::OH || ox >= SH::OW) return -1;
    return (((int64_t)b * SH::OH + oy) * SH::OW + ox) * SH::CO + o;
}

template <typename T, typename SH>
struct LdDgrad {
    static constexpr bool kMN = false;
    const T* g;
    int M;  // B * H * W
    GORILA_DEV float load(int i, int r) const {
        if (i >= M || r >= SH::RD) return 0.f;
        const int64_t a = dgrad_addr<SH>(i, r);
        return a < 0 ? 0.f : tof(g[a]);
    }
    GORILA_DEV const T* src8(int i, int r0) const {
        if (i >= M || r0 >= SH::RD) return nullptr;
        const int64_t a = dgrad_addr<SH>(i, r0);
        return a < 0 ? nullptr : g + a;
    }
    GORILA_DEV const void* gptr() const { return g; }  // any valid global address (zero-fill source)
};

// conv dgrad weight operand read straight from the forward (KRSC) weight, MN-major over c:
// value(i = c, r = (ky*K + kx)*CO + o) = W[o][ky][kx][c]
template <typename T, typename SH>
struct LdWdgradMN {
    static constexpr bool kMN = true;
    const T* w;
    GORILA_DEV int64_t addr(int c, int r) const {
        const int t = r / SH::CO, o = r - t * SH::CO;
        return (int64_t)o * SH::R + t * SH::C + c;
    }
    GORILA_DEV float load(int c, int r) const { return (c < SH::C && r < SH::RD) ? tof(w[addr(c, r)]) : 0.f; }
    GORILA_DEV const T* src8(int c0, int r) const {
        return (c0 >= SH::C || r >= SH::RD) ? nullptr : w + addr(c0, r);
    }
    GORILA_DEV const void* gptr() const { return w; }  // any valid global address (zero-fill source)
};

// ====================================================================== epilogues
// apply1(i, j, v, split): scalar; apply16(i, j0, v[16], split): 16 consecutive columns.

template <typename T>
GORILA_DEV void store16(T* dst, const float* v) {  // 16 values, 16-B aligned destination
    if constexpr (sizeof(T) == 2) {
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            w[e] = *reinterpret_cast<uint32_t*>(&h);
        }
#ifdef GORILA_EXP_NOSTORE  // timing experiment only: the stores are skipped (results wrong)
        if ((w[0] ^ w[1] ^ w[2] ^ w[3] ^ w[4] ^ w[5] ^ w[6] ^ w[7]) != 0x12345678u) return;
#endif
        if (((uintptr_t)dst & 31u) == 0) {  // one 256-bit store (half the L1 wavefronts of two 128-bit)
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(w[0]), "r"(w[1]),
                         "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
        } else {
            reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
            reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            reinterpret_cast<float4*>(dst)[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
    }
}
template <typename T>
GORILA_DEV void load16(const T* src, float* v) {
    if constexpr (sizeof(T) == 2) {
        const uint4 a = reinterpret_cast<const uint4*>(src)[0], b = reinterpret_cast<const uint4*>(src)[1];
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[e]);
            float2 f = __bfloat1622float2(h);
            v[2 * e] = f.x;
            v[2 * e + 1] = f.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float4 f = reinterpret_cast<const float4*>(src)[e];
            v[4 * e] = f.x; v[4 * e + 1] = f.y; v[4 * e + 2] = f.z; v[4 * e + 3] = f.w;
        }
    }
}

template <typename T>
struct EpAct {  // out[i][j] = round_T(act(v * scale + bias[j]))   (ld % 8 == 0)
    T* out;
    int64_t ld;
    const float* bias;
    float scale;
    int M, N, relu;
    // optional (shifted-window engine, N <= 64): the ReLU decisions of the stored values as bits,
    // mask[i * (N / 32) + j / 32] bit j % 32 = (out[i][j] > 0), read back by the data gradient
    // (EpMaskBits) instead of the activation itself
    uint32_t* mask = nullptr;
    GORILA_DEV float f(float v, int j) const {
        float z = v * scale + bias[j];
        return relu ? fmaxf(z, 0.f) : z;
    }
    GORILA_DEV void apply1(int i, int j, float v, int) const {
        if (i < M && j < N) out[(int64_t)i * ld + j] = fromf<T>(f(v, j));
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int s) const {
        if (i >= M) return;
        if (j0 + 16 <= N) {
            float o[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = f(v[e], j0 + e);
            store16<T>(out + (int64_t)i * ld + j0, o);
        } else {
            for (int e = 0; e < 16; ++e) apply1(i, j0 + e, v[e], s);
        }
    }
    // prefetch: the 16 biases of a column chunk, requested ahead of the accumulator (they depend on
    // the column only: COL_PRE engines load them once per CTA)
    static constexpr bool COL_PRE = true;
    struct Pre {
        float b[16];
    };
    GORILA_DEV Pre prefetch(int, int j0) const {
        Pre p;
#pragma unroll
        for (int e = 0; e < 16; ++e) p.b[e] = j0 + e < N ? bias[j0 + e] : 0.f;
        return p;
    }
    // apply16p that also returns the 16 decisions (out > 0) of the ROUNDED stored values
    GORILA_DEV uint32_t apply16m(int i, int j0, const float* v, const Pre& p) const {
        float o[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const float z = v[e] * scale + p.b[e];
            o[e] = relu ? fmaxf(z, 0.f) : z;
        }
        uint32_t bits = 0;
        if constexpr (sizeof(T) == 2) {  // decided on the packed bf16 words (= the stored values)
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                __nv_bfloat162 h = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
                w[e] = *reinterpret_cast<uint32_t*>(&h);
                const bool neg_lo = (w[e] & 0x8000u) != 0, neg_hi = (w[e] & 0x80000000u) != 0;
                bits |= ((w[e] & 0x7fffu) != 0 && !neg_lo ? 1u : 0u) << (2 * e);
                bits |= ((w[e] & 0x7fff0000u) != 0 && !neg_hi ? 1u : 0u) << (2 * e + 1);
            }
            T* dst = out + (int64_t)i * ld + j0;
            if (((uintptr_t)dst & 31u) == 0) {
                asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(w[0]), "r"(w[1]),
                             "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                             : "memory");
            } else {
                reinterpret_cast<uint4*>(dst)[0] = make_uint4(w[0], w[1], w[2], w[3]);
                reinterpret_cast<uint4*>(dst)[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) bits |= (o[e] > 0.f ? 1u : 0u) << e;
            store16<T>(out + (int64_t)i * ld + j0, o);
        }
        return bits;
    }
    GORILA_DEV void apply16p(int i, int j0, const float* v, const Pre& p, int s) const {
        if (i >= M) return;
        if (j0 + 16 <= N) {
            float o[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const float z = v[e] * scale + p.b[e];
                o[e] = relu ? fmaxf(z, 0.f) : z;
            }
            store16<T>(out + (int64_t)i * ld + j0, o);
        } else {
            for (int e = 0; e < 16; ++e) apply1(i, j0 + e, v[e], s);
        }
    }
};

// out[i][j] = round_T(v * 1[act[i][j] > 0]) with the decisions read as bits (EpAct::mask):
// 4 bytes per row of 32 channels instead of the activation row (64 B), same values as EpMask
template <typename T>
struct EpMaskBits {
    T* out;
    const uint32_t* bits;
    int64_t ld;
    int M, N, words;  // words = N / 32
    static constexpr bool ROW_PRE = true;
    struct Pre {
        uint32_t w;
    };
    GORILA_DEV Pre prefetch(int i, int j0) const {
        Pre p;
        p.w = i < M ? __ldg(bits + (int64_t)i * words + (j0 >> 5)) : 0u;
        return p;
    }
    GORILA_DEV void apply16p(int i, int j0, const float* v, const Pre& p, int) const {
        if (i >= M || j0 + 16 > N) return;
        const uint32_t b = p.w >> (j0 & 16);
        float o[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) o[e] = (b >> e) & 1u ? v[e] : 0.f;
        store16<T>(out + (int64_t)i * ld + j0, o);
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int s) const { apply16p(i, j0, v, prefetch(i, j0), s); }
};

template <typename T>
struct EpMask {  // out[i][j] = round_T(v * 1[act[i][j] > 0])  (ReLU'(0) = 0, reading R19; ld % 8 == 0)
    T* out;
    const T* act;
    int64_t ld;
    int M, N;
    GORILA_DEV void apply1(int i, int j, float v, int) const {
        if (i >= M || j >= N) return;
        const int64_t a = (int64_t)i * ld + j;
        out[a] = fromf<T>(tof(act[a]) > 0.f ? v : 0.f);
    }
    // epilogue prefetch (issued ahead of the accumulator): the 16 activations of a row chunk
    static constexpr bool ROW_PRE = true;
    struct Pre {
        uint4 q[sizeof(T)];
    };
    GORILA_DEV Pre prefetch(int i, int j0) const {
        Pre p;
#ifdef GORILA_EXP_NOSTORE  // timing experiment only: no mask loads either
        if (i >= 0) {
#pragma unroll
            for (int u = 0; u < (int)sizeof(T); ++u) p.q[u] = make_uint4(i, j0, i, j0);
            return p;
        }
#endif
        if (i < M && j0 + 16 <= N) {
            const T* src = act + (int64_t)i * ld + j0;
            if (sizeof(T) == 2 && ((uintptr_t)src & 31u) == 0) {  // one 256-bit load
                uint32_t* q = reinterpret_cast<uint32_t*>(p.q);
                asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                             : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]),
                               "=r"(q[7])
                             : "l"(src));
            } else {
#pragma unroll
                for (int u = 0; u < (int)sizeof(T); ++u) p.q[u] = reinterpret_cast<const uint4*>(src)[u];
            }
        } else {
#pragma unroll
            for (int u = 0; u < (int)sizeof(T); ++u) p.q[u] = make_uint4(0, 0, 0, 0);
        }
        return p;
    }
    GORILA_DEV void apply16p(int i, int j0, const float* v, const Pre& p, int s) const {
        if (i >= M) return;
        if (j0 + 16 <= N) {
            float h[16], o[16];
            load16<T>(reinterpret_cast<const T*>(p.q), h);
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = h[e] > 0.f ? v[e] : 0.f;
            store16<T>(out + (int64_t)i * ld + j0, o);
        } else {
            for (int e = 0; e < 16; ++e) apply1(i, j0 + e, v[e], s);
        }
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int s) const {
        if (i >= M) return;
        if (j0 + 16 <= N) {
            float h[16], o[16];
            load16<T>(act + (int64_t)i * ld + j0, h);
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = h[e] > 0.f ? v[e] : 0.f;
            store16<T>(out + (int64_t)i * ld + j0, o);
        } else {
            for (int e = 0; e < 16; ++e) apply1(i, j0 + e, v[e], s);
        }
    }
};

template <typename T>
struct EpMaskT {  // transposed: out[j][i] = round_T(v * 1[act[j][i] > 0])  (coalesced across the warp's rows)
    T* out;
    const T* act;
    int64_t ld;
    int M, N;
    GORILA_DEV void apply1(int i, int j, float v, int) const {
        if (i >= M || j >= N) return;
        const int64_t a = (int64_t)j * ld + i;
        out[a] = fromf<T>(tof(act[a]) > 0.f ? v : 0.f);
    }
    struct Pre {
        float h[16];
    };
    GORILA_DEV Pre prefetch(int i, int j0) const {
        Pre p;
#pragma unroll
        for (int e = 0; e < 16; ++e) p.h[e] = (i < M && j0 + e < N) ? tof(act[(int64_t)(j0 + e) * ld + i]) : 0.f;
        return p;
    }
    GORILA_DEV void apply16p(int i, int j0, const float* v, const Pre& p, int) const {
        if (i >= M) return;
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if (j0 + e < N) out[(int64_t)(j0 + e) * ld + i] = fromf<T>(p.h[e] > 0.f ? v[e] : 0.f);
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int) const {
        if (i >= M) return;
        float h[16];  // all loads before any store (no load/store aliasing chain)
#pragma unroll
        for (int e = 0; e < 16; ++e) h[e] = (j0 + e < N) ? tof(act[(int64_t)(j0 + e) * ld + i]) : 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if (j0 + e < N) out[(int64_t)(j0 + e) * ld + i] = fromf<T>(h[e] > 0.f ? v[e] : 0.f);
    }
};

struct EpStoreT {  // dst[split][j][i] = v * scale (transposed fp32 store: weight-gradient partials)
    float* dst;
    int64_t ld, split_stride;
    float scale;
    int M, N;
    GORILA_DEV void apply1(int i, int j, float v, int split) const {
        if (i < M && j < N) dst[split * split_stride + (int64_t)j * ld + i] = v * scale;
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int s) const {
        if (i < M && j0 + 16 <= N) {  // common case: no per-element bounds branches
            float* d = dst + s * split_stride + (int64_t)j0 * ld + i;
#pragma unroll
            for (int e = 0; e < 16; ++e) d[(int64_t)e * ld] = v[e] * scale;
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) apply1(i, j0 + e, v[e], s);
        }
    }
};

struct EpActT {  // out[j][i] = ReLU(v + bias[i]) in fp32 (fc4 forward computed as W4 . a3^T)
    float* out;
    int64_t ld;
    const float* bias;
    int M, N;
    GORILA_DEV void apply1(int i, int j, float v, int) const {
        if (i < M && j < N) out[(int64_t)j * ld + i] = fmaxf(v + bias[i], 0.f);
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int s) const {
        if (i >= M) return;
        const float b = bias[i];
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if (j0 + e < N) out[(int64_t)(j0 + e) * ld + i] = fmaxf(v[e] + b, 0.f);
    }
};

struct EpStore {  // dst[split][i][j] = v (fp32 split-K partials)
    float* dst;
    int64_t ld, split_stride;
    int M, N;
    GORILA_DEV void apply1(int i, int j, float v, int split) const {
        if (i < M && j < N) dst[split * split_stride + (int64_t)i * ld + j] = v;
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int s) const {
        if (i < M && j0 + 16 <= N && (ld & 3) == 0) {
            store16<float>(dst + s * split_stride + (int64_t)i * ld + j0, v);
        } else {
            for (int e = 0; e < 16; ++e) apply1(i, j0 + e, v[e], s);
        }
    }
};

struct EpAddT {  // G[j*ld + i] (+)= v (fp32, transposed, coalesced across the warp's rows)
    float* G;
    int64_t ld;
    int M, N, accumulate;
    GORILA_DEV void apply1(int i, int j, float v, int) const {
        if (i < M && j < N) G[(int64_t)j * ld + i] = accumulate ? G[(int64_t)j * ld + i] + v : v;
    }
    GORILA_DEV void apply16(int i, int j0, const float* v, int) const {
        if (i >= M) return;
        float* d = G + (int64_t)j0 * ld + i;
        if (j0 + 16 <= N && !accumulate) {  // first learner of the round: plain stores
#pragma unroll
            for (int e = 0; e < 16; ++e) d[(int64_t)e * ld] = v[e];
            return;
        }
        float o[16];  // all loads before any store
#pragma unroll
        for (int e = 0; e < 16; ++e) o[e] = (accumulate && j0 + e < N) ? d[(int64_t)e * ld] : 0.f;
#pragma unroll
        for (int e = 0; e < 16; ++e)
            if (j0 + e < N) d[(int64_t)e * ld] = o[e] + v[e];
    }
};

// epilogues whose prefetched inputs depend on the output row (ROW_PRE): the shifted-window engine
// requests a whole tile of them one tile ahead
template <class EP, class = void>
struct ep_row_pre : std::false_type {};
template <class EP>
struct ep_row_pre<EP, std::void_t<decltype(EP::ROW_PRE)>> : std::integral_constant<bool, EP::ROW_PRE> {};
template <class EP, class = void>
struct ep_col_pre : std::false_type {};
template <class EP>
struct ep_col_pre<EP, std::void_t<decltype(EP::COL_PRE)>> : std::integral_constant<bool, EP::COL_PRE> {};
// prefetch interface: epilogues with a `Pre` type load their inputs ahead of the accumulator
template <class EP, class = void>
struct EpPre {
    struct type {};
    static GORILA_DEV type load(const EP&, int, int) { return {}; }
    static GORILA_DEV void apply(const EP& ep, int i, int j0, const float* v, const type&, int s) {
        ep.apply16(i, j0, v, s);
    }
};
template <class EP>
struct EpPre<EP, std::void_t<typename EP::Pre>> {
    using type = typename EP::Pre;
    static GORILA_DEV type load(const EP& ep, int i, int j0) { return ep.prefetch(i, j0); }
    static GORILA_DEV void apply(const EP& ep, int i, int j0, const float* v, const type& p, int s) {
        ep.apply16p(i, j0, v, p, s);
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
    int M, N, R;           // shared by all problems of the batch
    int splits;            // split of the reduction range
    int chunks_per_split;  // in units of 64 (tc) / 16 (simt) reduction elements
    int cluster;           // > 1: the `splits` CTAs of one tile form a cluster and reduce through DSMEM
};

// ====================================================================== tcgen05 engine
constexpr int TC_BM = 128, TC_BK = 64, TC_THREADS = 128;

__host__ __device__ constexpr uint32_t tmem_cols_for(int bn) {
    return bn <= 32 ? 32u : bn <= 64 ? 64u : bn <= 128 ? 128u : bn <= 256 ? 256u : 512u;
}
// fp32 partial tile for the cluster reduction: [BN/16][128 rows][20 floats] (80-B row pitch: conflict-free)
__host__ __device__ constexpr int tc_red_bytes(int bn) { return (bn / 16) * TC_BM * 80; }
__host__ __device__ constexpr int tc_slice_bytes(int bn) { return 64 * (bn + 4) * 4; }
// ====================================================================== fp32 SIMT engine
constexpr int SM_BI = 64, SM_BJ = 64, SM_BR = 16;

template <typename LA, typename LB, typename EP>
__global__ void __launch_bounds__(256) gemm_simt(const __grid_constant__ GemmBatch<LA, LB, EP> p) {
    __shared__ float As[SM_BR][SM_BI + 4];
    __shared__ float Bs[SM_BR][SM_BJ + 4];
    pdl_wait();
    pdl_trigger();
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
            const int idx = tid + 256 * q;
            const int ii = idx & 63, rr = idx >> 6;
            const int r = r0 + rr;
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
        for (int y = 0; y < 4; ++y) P.ep.apply1(i0 + ti + 16 * x, j0 + tj + 16 * y, acc[x][y], split);
}

}  // namespace gorila
