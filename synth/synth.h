/* synth.h — seeded synthetic Atari-shaped replay input (shared input generator).
 *
 * This module is the ONE piece both sides of the parity check may use: it
 * defines the synthetic inputs (frames and per-step meta) and holds none of
 * the method's arithmetic (no sampling, no stacking, no network, no update).
 * The oracle (oracle/) reads frames from the host implementation; the
 * benchmark fills the device replay from the device implementation
 * (synth_fill.cu). Both implement the same counter-based definition below,
 * and tests check them bit-exact against each other.
 *
 * Definition:
 *   Philox4x32-10 (Salmon et al., SC'11), key = {seed & 0xffffffff, seed >> 32}.
 *   Frame t of learner j is 84x84 u8 (paper P:176-181, §5.1 "84x84" luminance
 *   frames) = 441 chunks of 16 B; chunk c = little-endian bytes of
 *   Philox(ctr = {c, j, t & 0xffffffff, ((t >> 32) & 0xffffff) | TAG_FRAME << 24}).
 *   Meta of step t: x = Philox(ctr = {t & 0xffffffff, j, (t >> 32) & 0xffffffff, TAG_META << 24})
 *     a_t = (x0 * nA) >> 32                        (uniform action in [0, nA))
 *     r_t = +1 if x1 <  R_POS_THR, -1 if x1 < R_NEG_THR, else 0   (2% / 1%)
 *     d_t = x2 < D_THR                             (episodes average 1000 steps)
 *     poison: r_t = 1e6 if x3 < poison_thr          (SPEC S:600 poison injection)
 */
#ifndef GORILA_SYNTH_H
#define GORILA_SYNTH_H
#include <stdint.h>

#define SYNTH_FRAME_BYTES 7056
#define SYNTH_TAG_FRAME 1u
#define SYNTH_TAG_META 2u
#define SYNTH_R_POS_THR 85899345u   /* floor(0.02 * 2^32) */
#define SYNTH_R_NEG_THR 128849018u  /* floor(0.03 * 2^32) */
#define SYNTH_D_THR 4294967u        /* floor(2^32 / 1000) */
#define SYNTH_POISON_REWARD 1.0e6f

#ifdef __cplusplus
extern "C" {
#endif

/* frames t0 .. t0+count-1 of learner j -> out[count][7056] */
void synth_frames(uint64_t seed, int32_t learner, int64_t t0, int64_t count, uint8_t* out);
/* meta of steps t0 .. t0+count-1. poison_thr = floor(p_poison * 2^32) (0 = off) */
void synth_meta(uint64_t seed, int32_t learner, int64_t t0, int64_t count, int32_t n_actions,
                uint32_t poison_thr, uint8_t* a, float* r, uint8_t* d);
/* theta0 (reading R24: "random network initializations"): canonical flat layout
 * [W1,b1,W2,b2,W3,b3,W4,b4,W5,b5]; element i = (2u-1)/sqrt(fan_in of its layer) rounded to
 * fp32, u = x0 * 2^-32 with x = Philox(ctr = {i, 0, 0, TAG_INIT << 24}, key = seed). */
#define SYNTH_TAG_INIT 4u
int64_t synth_theta0(uint64_t seed, int32_t n_actions, float* out);
/* raw Philox4x32-10 block (exported for the generator's own known-answer test) */
void synth_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* device implementation (synth_fill.cu, libsynth_dev.so). Pointers are device
 * pointers; stream is a cudaStream_t. Returns 0 on success, else a cudaError_t. */
int synth_fill_frames_dev(uint64_t seed, int32_t learner, int64_t t0, int64_t count,
                          uint8_t* out, void* stream);
int synth_fill_meta_dev(uint64_t seed, int32_t learner, int64_t t0, int64_t count,
                        int32_t n_actions, uint32_t poison_thr, uint8_t* a, float* r,
                        uint8_t* d, void* stream);
#ifdef __cplusplus
}
#endif
#endif
