/* synth.c — host implementation of the synthetic input definition in synth.h. */
#include "synth.h"
#include <math.h>
#include <string.h>

static void mulhilo32(uint32_t a, uint32_t b, uint32_t* hi, uint32_t* lo) {
    uint64_t p = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(p >> 32);
    *lo = (uint32_t)p;
}

void synth_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint32_t hi0, lo0, hi1, lo1;
        mulhilo32(0xD2511F53u, c0, &hi0, &lo0);
        mulhilo32(0xCD9E8D57u, c2, &hi1, &lo1);
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void synth_frames(uint64_t seed, int32_t learner, int64_t t0, int64_t count, uint8_t* out) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t f = 0; f < count; ++f) {
        uint64_t t = (uint64_t)(t0 + f);
        for (uint32_t c = 0; c < SYNTH_FRAME_BYTES / 16; ++c) {
            uint32_t ctr[4] = {c, (uint32_t)learner, (uint32_t)t,
                               (uint32_t)((t >> 32) & 0xffffffu) | (SYNTH_TAG_FRAME << 24)};
            uint32_t x[4];
            synth_philox(ctr, key, x);
            uint8_t* dst = out + f * SYNTH_FRAME_BYTES + 16 * c;
            for (int w = 0; w < 4; ++w)
                for (int b = 0; b < 4; ++b) dst[4 * w + b] = (uint8_t)(x[w] >> (8 * b));
        }
    }
}

void synth_meta(uint64_t seed, int32_t learner, int64_t t0, int64_t count, int32_t n_actions,
                uint32_t poison_thr, uint8_t* a, float* r, uint8_t* d) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t f = 0; f < count; ++f) {
        uint64_t t = (uint64_t)(t0 + f);
        uint32_t ctr[4] = {(uint32_t)t, (uint32_t)learner, (uint32_t)(t >> 32), SYNTH_TAG_META << 24};
        uint32_t x[4];
        synth_philox(ctr, key, x);
        a[f] = (uint8_t)(((uint64_t)x[0] * (uint64_t)n_actions) >> 32);
        float rew = 0.0f;
        if (x[1] < SYNTH_R_POS_THR) rew = 1.0f;
        else if (x[1] < SYNTH_R_NEG_THR) rew = -1.0f;
        if (x[3] < poison_thr) rew = SYNTH_POISON_REWARD;
        r[f] = rew;
        d[f] = (uint8_t)(x[2] < SYNTH_D_THR);
    }
}

int64_t synth_theta0(uint64_t seed, int32_t n_actions, float* out) {
    /* (count, fan_in) per tensor in canonical order; architecture of P:180-183 */
    const int64_t cnt[10] = {32 * 4 * 8 * 8, 32, 64 * 32 * 4 * 4, 64, 64 * 64 * 3 * 3, 64,
                             512 * 3136, 512, (int64_t)n_actions * 512, n_actions};
    const int fan[10] = {256, 256, 512, 512, 576, 576, 3136, 3136, 512, 512};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int64_t i = 0;
    for (int t = 0; t < 10; ++t) {
        double bound = 1.0 / sqrt((double)fan[t]);
        for (int64_t e = 0; e < cnt[t]; ++e, ++i) {
            uint32_t ctr[4] = {(uint32_t)i, 0u, 0u, SYNTH_TAG_INIT << 24};
            uint32_t x[4];
            synth_philox(ctr, key, x);
            double u = (double)x[0] * (1.0 / 4294967296.0);
            if (out) out[i] = (float)((2.0 * u - 1.0) * bound);
        }
    }
    return i;
}
