/* oracle.c — plain, slow, obviously-correct CPU oracle for the Gorila DQN learner update.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code
 * with the CUDA path (paper_1507_04296_b200/csrc) and neither includes the other.
 *
 * What is here (the heavy loops; the round logic is in gorila_oracle.py):
 *   - Philox4x32-10 and the uniform index map           (§3.3, Alg.1)
 *   - 4-frame stacking with episode/eviction zero-pad   (§5.1; readings R14/R15)
 *   - Nature-DQN Q-network forward / backward in fp64   (§5.1; Eq.2)
 *     with an optional bf16 rounding emulation that mirrors the GPU precision
 *     contract (reading R16): rounding happens ONLY at the listed points.
 *
 * Layouts are the paper-natural ones: images NCHW, conv weights OIHW, FC
 * weights [out][in], canonical flat θ = [W1,b1,W2,b2,W3,b3,W4,b4,W5,b5].
 * Loops are direct definitions (no blocking, no reordering); OpenMP only
 * splits independent outputs across threads, so results do not depend on the
 * thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ---------------- Philox4x32-10 (Salmon et al. 2011) ---------------- */
EXPORT void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    memcpy(out, c, sizeof(c));
}

#define ORC_TAG_SAMPLE 3u

/* O2: minibatch indices, uniform with replacement over the
 * valid slots tau in [n-size, n-2] ("sampled uniformly from the replay memory",
 * P:87 §3.3; Alg.1). M = size-1 valid slots; u is a 64-bit uniform word and
 * tau = (n-size) + floor(u*M / 2^64). Returns 0, or -1 if fewer than one valid slot. */
EXPORT int orc_sample_indices(int64_t n, int64_t size, int32_t B, uint64_t seed, int32_t learner,
                              uint64_t round, int64_t* tau) {
    int64_t M = size - 1;
    if (M < 1) return -1;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int32_t i = 0; i < B; ++i) {
        uint32_t ctr[4] = {(uint32_t)(i / 2), (uint32_t)learner, (uint32_t)round,
                           (uint32_t)((round >> 32) & 0xffffffu) | (ORC_TAG_SAMPLE << 24)};
        uint32_t x[4];
        orc_philox(ctr, key, x);
        uint64_t u = (i % 2 == 0) ? ((uint64_t)x[0] | ((uint64_t)x[1] << 32))
                                  : ((uint64_t)x[2] | ((uint64_t)x[3] << 32));
        unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)(uint64_t)M;
        tau[i] = (n - size) + (int64_t)(uint64_t)(prod >> 64);
    }
    return 0;
}

/* f4 (reading R36): a minibatch drawn uniformly from the GLOBAL
 * replay memory D ("a global replay memory aggregates the experience into a distributed
 * database", §4; "sampled from either a local or global experience replay memory D",
 * P:142; uniform sampling from D, §3.3). D is the union of the G shards' valid transitions,
 * enumerated shard by shard (ascending global learner id j) and within shard j by tau ascending
 * over [n_j - size_j, n_j - 2], size_j = min(n_j, C). With T = |D| and u the same 64-bit word as
 * O2 (counter of the drawing learner), g = floor(u*T / 2^64) and (shard, tau) is the g-th element
 * of that enumeration, found here by walking the enumeration. Returns 0, or -1 if T = 0. */
EXPORT int orc_sample_indices_global(int32_t G, const int64_t* n, int64_t C, int32_t B, uint64_t seed,
                                     int32_t learner, uint64_t round, int32_t* shard, int64_t* tau) {
    uint64_t T = 0;
    for (int32_t j = 0; j < G; ++j) {
        int64_t size = n[j] < C ? n[j] : C;
        if (size >= 2) T += (uint64_t)(size - 1);
    }
    if (T == 0) return -1;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int32_t i = 0; i < B; ++i) {
        uint32_t ctr[4] = {(uint32_t)(i / 2), (uint32_t)learner, (uint32_t)round,
                           (uint32_t)((round >> 32) & 0xffffffu) | (ORC_TAG_SAMPLE << 24)};
        uint32_t x[4];
        orc_philox(ctr, key, x);
        uint64_t u = (i % 2 == 0) ? ((uint64_t)x[0] | ((uint64_t)x[1] << 32))
                                  : ((uint64_t)x[2] | ((uint64_t)x[3] << 32));
        uint64_t g = (uint64_t)(((unsigned __int128)u * (unsigned __int128)T) >> 64);
        uint64_t pos = 0;  /* index of the first element of shard j in the enumeration */
        for (int32_t j = 0; j < G; ++j) {
            int64_t size = n[j] < C ? n[j] : C;
            uint64_t M = size >= 2 ? (uint64_t)(size - 1) : 0;
            if (g < pos + M) {
                shard[i] = j;
                tau[i] = (n[j] - size) + (int64_t)(g - pos);
                break;
            }
            pos += M;
        }
    }
    return 0;
}

/* O3: stack(t)[c] = o_{t-3+c}, c = 0..3 (oldest -> newest; "concatenating the
 * images from four previous preprocessed frames"). Frame t-3+c is
 * replaced by zeros if it is no longer (or never was) in the ring
 * (t-3+c < n-size) or if an episode ended at any step t' in [t-3+c, t-1]
 * (d_{t'} = 1 means s_{t'+1} is terminal, so frames up to t' belong to an
 * earlier episode). Ring slot of step t is t mod C. */
EXPORT void orc_stack(int64_t C, int64_t n, const uint8_t* frames, const uint8_t* d, int64_t t,
                      uint8_t* out /* [4][84*84] */) {
    const int64_t FB = 84 * 84;
    int64_t size = n < C ? n : C;
    for (int c = 0; c < 4; ++c) {
        int64_t f = t - 3 + c;
        int zero = (f < n - size);
        if (!zero)
            for (int64_t tp = f; tp <= t - 1; ++tp)
                if (d[tp % C]) zero = 1;
        if (zero) memset(out + c * FB, 0, FB);
        else memcpy(out + c * FB, frames + (f % C) * FB, FB);
    }
}

/* gather the minibatch: s_i = stack(tau_i), s'_i = stack(tau_i + 1), a, r, d at tau_i */
EXPORT void orc_gather(int64_t C, int64_t n, const uint8_t* frames, const uint8_t* a, const float* r,
                       const uint8_t* d, int32_t B, const int64_t* tau, uint8_t* s, uint8_t* s2,
                       uint8_t* a_out, float* r_out, uint8_t* d_out) {
    const int64_t SB = 4 * 84 * 84;
    for (int32_t i = 0; i < B; ++i) {
        orc_stack(C, n, frames, d, tau[i], s + i * SB);
        orc_stack(C, n, frames, d, tau[i] + 1, s2 + i * SB);
        a_out[i] = a[tau[i] % C];
        r_out[i] = r[tau[i] % C];
        d_out[i] = d[tau[i] % C];
    }
}

/* ---------------- layer primitives (fp64, NCHW / OIHW, valid padding) ---------------- */

/* y[b][o][oy][ox] = bias[o] + sum_{c,ky,kx} x[b][c][oy*s+ky][ox*s+kx] * w[o][c][ky][kx] */
EXPORT void orc_conv2d_fwd(int B, int Cin, int H, int W, int Cout, int k, int s, const double* x,
                           const double* w, const double* bias, double* y) {
    int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
#pragma omp parallel for schedule(static)
    for (int b = 0; b < B; ++b)
        for (int o = 0; o < Cout; ++o)
            for (int oy = 0; oy < OH; ++oy)
                for (int ox = 0; ox < OW; ++ox) {
                    double acc = 0.0;
                    for (int c = 0; c < Cin; ++c)
                        for (int ky = 0; ky < k; ++ky)
                            for (int kx = 0; kx < k; ++kx)
                                acc += x[(((int64_t)b * Cin + c) * H + oy * s + ky) * W + ox * s + kx] *
                                       w[(((int64_t)o * Cin + c) * k + ky) * k + kx];
                    y[(((int64_t)b * Cout + o) * OH + oy) * OW + ox] = acc + (bias ? bias[o] : 0.0);
                }
}

/* dx = transpose of the forward map applied to dy: every forward product
 * x[..]*w[..] contributes dy*w to dx at the same input position. */
EXPORT void orc_conv2d_bwd_data(int B, int Cin, int H, int W, int Cout, int k, int s, const double* dy,
                                const double* w, double* dx) {
    int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
    memset(dx, 0, sizeof(double) * (size_t)B * Cin * H * W);
#pragma omp parallel for schedule(static)
    for (int b = 0; b < B; ++b)
        for (int o = 0; o < Cout; ++o)
            for (int oy = 0; oy < OH; ++oy)
                for (int ox = 0; ox < OW; ++ox) {
                    double g = dy[(((int64_t)b * Cout + o) * OH + oy) * OW + ox];
                    for (int c = 0; c < Cin; ++c)
                        for (int ky = 0; ky < k; ++ky)
                            for (int kx = 0; kx < k; ++kx)
                                dx[(((int64_t)b * Cin + c) * H + oy * s + ky) * W + ox * s + kx] +=
                                    g * w[(((int64_t)o * Cin + c) * k + ky) * k + kx];
                }
}

/* dw[o][c][ky][kx] = sum_{b,oy,ox} dy[b][o][oy][ox] * x[b][c][oy*s+ky][ox*s+kx]; db[o] = sum dy[b][o][..] */
EXPORT void orc_conv2d_bwd_weight(int B, int Cin, int H, int W, int Cout, int k, int s, const double* dy,
                                  const double* x, double* dw, double* db) {
    int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
#pragma omp parallel for schedule(static)
    for (int o = 0; o < Cout; ++o) {
        for (int c = 0; c < Cin; ++c)
            for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                    double acc = 0.0;
                    for (int b = 0; b < B; ++b)
                        for (int oy = 0; oy < OH; ++oy)
                            for (int ox = 0; ox < OW; ++ox)
                                acc += dy[(((int64_t)b * Cout + o) * OH + oy) * OW + ox] *
                                       x[(((int64_t)b * Cin + c) * H + oy * s + ky) * W + ox * s + kx];
                    dw[(((int64_t)o * Cin + c) * k + ky) * k + kx] = acc;
                }
        if (db) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b)
                for (int p = 0; p < OH * OW; ++p) acc += dy[((int64_t)b * Cout + o) * OH * OW + p];
            db[o] = acc;
        }
    }
}

/* y[b][n] = bias[n] + sum_k x[b][k] * w[n][k] */
EXPORT void orc_linear_fwd(int B, int K, int N, const double* x, const double* w, const double* bias,
                           double* y) {
#pragma omp parallel for schedule(static)
    for (int b = 0; b < B; ++b)
        for (int n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int k = 0; k < K; ++k) acc += x[(int64_t)b * K + k] * w[(int64_t)n * K + k];
            y[(int64_t)b * N + n] = acc + (bias ? bias[n] : 0.0);
        }
}

/* dx[b][k] = sum_n dy[b][n] * w[n][k] */
EXPORT void orc_linear_bwd_data(int B, int K, int N, const double* dy, const double* w, double* dx) {
#pragma omp parallel for schedule(static)
    for (int b = 0; b < B; ++b)
        for (int k = 0; k < K; ++k) {
            double acc = 0.0;
            for (int n = 0; n < N; ++n) acc += dy[(int64_t)b * N + n] * w[(int64_t)n * K + k];
            dx[(int64_t)b * K + k] = acc;
        }
}

/* dw[n][k] = sum_b dy[b][n] * x[b][k]; db[n] = sum_b dy[b][n] */
EXPORT void orc_linear_bwd_weight(int B, int K, int N, const double* dy, const double* x, double* dw,
                                  double* db) {
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N; ++n) {
        for (int k = 0; k < K; ++k) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b) acc += dy[(int64_t)b * N + n] * x[(int64_t)b * K + k];
            dw[(int64_t)n * K + k] = acc;
        }
        if (db) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b) acc += dy[(int64_t)b * N + n];
            db[n] = acc;
        }
    }
}

/* ---------------- precision emulation (reading R16) ---------------- */

/* round to bfloat16 precision: 8 significant bits, round-to-nearest-even
 * (values here are far from bf16 overflow / subnormal range). */
EXPORT double orc_round_bf16(double x) {
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    double m = frexp(x, &e);            /* x = m * 2^e, 0.5 <= |m| < 1 */
    double r = nearbyint(ldexp(m, 8));  /* default FE_TONEAREST: ties to even */
    return ldexp(r, e - 8);
}

/* ---------------- Nature-DQN Q-network (§5.1) ---------------- */

enum { ORC_EXACT = 0, ORC_BF16 = 2 };

/* conv1 32x(4x8x8)/4: 84->20; conv2 64x(32x4x4)/2: 20->9; conv3 64x(64x3x3)/1: 9->7;
 * fc4 3136->512; fc5 512->nA. */
#define L1_OUT (32 * 20 * 20)
#define L2_OUT (64 * 9 * 9)
#define L3_OUT (64 * 7 * 7)
#define L4_OUT 512
#define ACTS_PER_SAMPLE (L1_OUT + L2_OUT + L3_OUT + L4_OUT)

#define OFF_W1 0
#define OFF_B1 (OFF_W1 + 32 * 4 * 8 * 8)
#define OFF_W2 (OFF_B1 + 32)
#define OFF_B2 (OFF_W2 + 64 * 32 * 4 * 4)
#define OFF_W3 (OFF_B2 + 64)
#define OFF_B3 (OFF_W3 + 64 * 64 * 3 * 3)
#define OFF_W4 (OFF_B3 + 64)
#define OFF_B4 (OFF_W4 + 512 * 3136)
#define OFF_W5 (OFF_B4 + 512)

/* 1/255 rounded to fp32: the input scale of the precision contract (R16, R17) */
static const float kInScaleF32 = 1.0f / 255.0f;

EXPORT int64_t orc_param_count(int nA) { return (int64_t)OFF_W5 + 512 * (int64_t)nA + nA; }
EXPORT int64_t orc_acts_per_sample(void) { return ACTS_PER_SAMPLE; }

static double* quantised_copy(const double* src, int64_t n, int mode) {
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) q[i] = (mode == ORC_BF16) ? orc_round_bf16(src[i]) : src[i];
    return q;
}

/* post-activation h = ReLU(z); in BF16 mode h is rounded to bf16 (stored and used as the next operand) */
static void relu_store(double* z, int64_t n, int mode) {
    for (int64_t i = 0; i < n; ++i) {
        double h = z[i] > 0.0 ? z[i] : 0.0;
        z[i] = (mode == ORC_BF16) ? orc_round_bf16(h) : h;
    }
}

/* Forward Q(s,.;theta) for a batch of stacked frames s [B][4][84][84] (u8).
 * EXACT: x = u8/255, everything fp64. BF16: x = u8 (exact integers), conv1..fc4
 * weights rounded to bf16, conv1 pre-activation = acc * fp32(1/255) + b1, the
 * conv activations a1..a3 rounded to bf16 after the ReLU (they are tensor-core
 * operands); a4, fc5 weights / biases and Q unrounded (fc5 runs in fp32). acts (nullable) receives [B][a1|a2|a3|a4] (CHW per sample).
 * zs (nullable) receives the pre-activations z1..z4 in the same layout (the values the ReLU decides
 * on, before rounding) — read-only diagnostics for the parity tests; nothing below depends on it. */
static void save_pre(double* zs, const double* z, int B, int64_t per, int64_t off) {
    if (!zs) return;
    for (int b = 0; b < B; ++b) memcpy(zs + (int64_t)b * ACTS_PER_SAMPLE + off, z + (int64_t)b * per, sizeof(double) * per);
}
EXPORT void orc_qnet_forward(int nA, int B, const double* theta, const uint8_t* s, int mode, double* Q,
                             double* acts, double* zs) {
    double* x0 = (double*)malloc(sizeof(double) * (size_t)B * 4 * 84 * 84);
    for (int64_t i = 0; i < (int64_t)B * 4 * 84 * 84; ++i)
        x0[i] = (mode == ORC_BF16) ? (double)s[i] : (double)s[i] / 255.0;
    double* w1 = quantised_copy(theta + OFF_W1, 32 * 4 * 8 * 8, mode);
    double* w2 = quantised_copy(theta + OFF_W2, 64 * 32 * 4 * 4, mode);
    double* w3 = quantised_copy(theta + OFF_W3, 64 * 64 * 3 * 3, mode);
    double* w4 = quantised_copy(theta + OFF_W4, 512 * 3136, mode);
    double* a1 = (double*)malloc(sizeof(double) * (size_t)B * L1_OUT);
    double* a2 = (double*)malloc(sizeof(double) * (size_t)B * L2_OUT);
    double* a3 = (double*)malloc(sizeof(double) * (size_t)B * L3_OUT);
    double* a4 = (double*)malloc(sizeof(double) * (size_t)B * L4_OUT);

    if (mode == ORC_BF16) {
        orc_conv2d_fwd(B, 4, 84, 84, 32, 8, 4, x0, w1, NULL, a1);
        for (int b = 0; b < B; ++b)
            for (int o = 0; o < 32; ++o)
                for (int p = 0; p < 400; ++p) {
                    double* z = &a1[((int64_t)b * 32 + o) * 400 + p];
                    *z = *z * (double)kInScaleF32 + theta[OFF_B1 + o];
                }
    } else {
        orc_conv2d_fwd(B, 4, 84, 84, 32, 8, 4, x0, w1, theta + OFF_B1, a1);
    }
    save_pre(zs, a1, B, L1_OUT, 0);
    relu_store(a1, (int64_t)B * L1_OUT, mode);
    orc_conv2d_fwd(B, 32, 20, 20, 64, 4, 2, a1, w2, theta + OFF_B2, a2);
    save_pre(zs, a2, B, L2_OUT, L1_OUT);
    relu_store(a2, (int64_t)B * L2_OUT, mode);
    orc_conv2d_fwd(B, 64, 9, 9, 64, 3, 1, a2, w3, theta + OFF_B3, a3);
    save_pre(zs, a3, B, L3_OUT, L1_OUT + L2_OUT);
    relu_store(a3, (int64_t)B * L3_OUT, mode);
    /* fc4 input = a3 flattened in (C,H,W) order (reading R18) — the NCHW memory order */
    orc_linear_fwd(B, 3136, 512, a3, w4, theta + OFF_B4, a4);
    save_pre(zs, a4, B, L4_OUT, L1_OUT + L2_OUT + L3_OUT);
    /* a4 feeds only the fp32 fc5 layer (not a tensor-core operand): never rounded (R16) */
    relu_store(a4, (int64_t)B * L4_OUT, ORC_EXACT);
    orc_linear_fwd(B, 512, nA, a4, theta + OFF_W5, theta + OFF_W5 + 512 * nA, Q);

    if (acts)
        for (int b = 0; b < B; ++b) {
            double* dst = acts + (int64_t)b * ACTS_PER_SAMPLE;
            memcpy(dst, a1 + (int64_t)b * L1_OUT, sizeof(double) * L1_OUT);
            memcpy(dst + L1_OUT, a2 + (int64_t)b * L2_OUT, sizeof(double) * L2_OUT);
            memcpy(dst + L1_OUT + L2_OUT, a3 + (int64_t)b * L3_OUT, sizeof(double) * L3_OUT);
            memcpy(dst + L1_OUT + L2_OUT + L3_OUT, a4 + (int64_t)b * L4_OUT, sizeof(double) * L4_OUT);
        }
    free(x0); free(w1); free(w2); free(w3); free(w4);
    free(a1); free(a2); free(a3); free(a4);
}

/* g = upstream * 1[h > 0] (ReLU'(0) := 0, reading R19); BF16 mode rounds g to bf16 */
static void relu_grad(double* g, const double* h, int64_t n, int mode) {
    for (int64_t i = 0; i < n; ++i) {
        double v = h[i] > 0.0 ? g[i] : 0.0;
        g[i] = (mode == ORC_BF16) ? orc_round_bf16(v) : v;
    }
}

/* Backward: G = sum_b sum_a dQ[b][a] * dQ(s_b,a;theta)/dtheta (canonical layout), given the
 * saved activations of orc_qnet_forward (same mode). Eq.2: the caller passes
 * dQ[b][a_b] = -clip(delta_b)/B and 0 elsewhere (R3/R4). */
EXPORT void orc_qnet_backward(int nA, int B, const double* theta, const uint8_t* s, const double* acts,
                              const double* dQ, int mode, double* G) {
    double* x0 = (double*)malloc(sizeof(double) * (size_t)B * 4 * 84 * 84);
    for (int64_t i = 0; i < (int64_t)B * 4 * 84 * 84; ++i)
        x0[i] = (mode == ORC_BF16) ? (double)s[i] : (double)s[i] / 255.0;
    double* w2 = quantised_copy(theta + OFF_W2, 64 * 32 * 4 * 4, mode);
    double* w3 = quantised_copy(theta + OFF_W3, 64 * 64 * 3 * 3, mode);
    double* w4 = quantised_copy(theta + OFF_W4, 512 * 3136, mode);
    double* a1 = (double*)malloc(sizeof(double) * (size_t)B * L1_OUT);
    double* a2 = (double*)malloc(sizeof(double) * (size_t)B * L2_OUT);
    double* a3 = (double*)malloc(sizeof(double) * (size_t)B * L3_OUT);
    double* a4 = (double*)malloc(sizeof(double) * (size_t)B * L4_OUT);
    for (int b = 0; b < B; ++b) {
        const double* src = acts + (int64_t)b * ACTS_PER_SAMPLE;
        memcpy(a1 + (int64_t)b * L1_OUT, src, sizeof(double) * L1_OUT);
        memcpy(a2 + (int64_t)b * L2_OUT, src + L1_OUT, sizeof(double) * L2_OUT);
        memcpy(a3 + (int64_t)b * L3_OUT, src + L1_OUT + L2_OUT, sizeof(double) * L3_OUT);
        memcpy(a4 + (int64_t)b * L4_OUT, src + L1_OUT + L2_OUT + L3_OUT, sizeof(double) * L4_OUT);
    }
    double* g4 = (double*)malloc(sizeof(double) * (size_t)B * L4_OUT);
    double* g3 = (double*)malloc(sizeof(double) * (size_t)B * L3_OUT);
    double* g2 = (double*)malloc(sizeof(double) * (size_t)B * L2_OUT);
    double* g1 = (double*)malloc(sizeof(double) * (size_t)B * L1_OUT);

    /* fc5 (unrounded weights in both modes) */
    orc_linear_bwd_weight(B, 512, nA, dQ, a4, G + OFF_W5, G + OFF_W5 + 512 * nA);
    orc_linear_bwd_data(B, 512, nA, dQ, theta + OFF_W5, g4);
    relu_grad(g4, a4, (int64_t)B * L4_OUT, mode);
    /* fc4 */
    orc_linear_bwd_weight(B, 3136, 512, g4, a3, G + OFF_W4, G + OFF_B4);
    orc_linear_bwd_data(B, 3136, 512, g4, w4, g3);
    relu_grad(g3, a3, (int64_t)B * L3_OUT, mode);
    /* conv3 */
    orc_conv2d_bwd_weight(B, 64, 9, 9, 64, 3, 1, g3, a2, G + OFF_W3, G + OFF_B3);
    orc_conv2d_bwd_data(B, 64, 9, 9, 64, 3, 1, g3, w3, g2);
    relu_grad(g2, a2, (int64_t)B * L2_OUT, mode);
    /* conv2 */
    orc_conv2d_bwd_weight(B, 32, 20, 20, 64, 4, 2, g2, a1, G + OFF_W2, G + OFF_B2);
    orc_conv2d_bwd_data(B, 32, 20, 20, 64, 4, 2, g2, w2, g1);
    relu_grad(g1, a1, (int64_t)B * L1_OUT, mode);
    /* conv1: weight gradient only (the input is data). BF16 mode folds the 1/255 into the end. */
    orc_conv2d_bwd_weight(B, 4, 84, 84, 32, 8, 4, g1, x0, G + OFF_W1, G + OFF_B1);
    if (mode == ORC_BF16)
        for (int i = 0; i < 32 * 4 * 8 * 8; ++i) G[OFF_W1 + i] *= (double)kInScaleF32;

    free(x0); free(w2); free(w3); free(w4);
    free(a1); free(a2); free(a3); free(a4);
    free(g1); free(g2); free(g3); free(g4);
}
