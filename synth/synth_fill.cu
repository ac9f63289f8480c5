// synth_fill.cu — device implementation of the synthetic input definition in synth.h.
// Used by bench.py / GPU tests to fill a 1M-frame device replay without a host round trip.
#include <cuda_runtime.h>
#include <stdint.h>
#include "synth.h"

namespace {

__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__global__ void fill_frames(uint2 key, uint32_t learner, int64_t t0, int64_t count, uint4* out) {
    const int64_t total = count * (SYNTH_FRAME_BYTES / 16);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t f = (uint64_t)(i / (SYNTH_FRAME_BYTES / 16));
        uint32_t c = (uint32_t)(i - (int64_t)f * (SYNTH_FRAME_BYTES / 16));
        uint64_t t = (uint64_t)t0 + f;
        uint4 x = philox(make_uint4(c, learner, (uint32_t)t,
                                    (uint32_t)((t >> 32) & 0xffffffu) | (SYNTH_TAG_FRAME << 24)),
                         key);
        out[i] = x;  // little-endian bytes of x0..x3
    }
}

__global__ void fill_meta(uint2 key, uint32_t learner, int64_t t0, int64_t count, int32_t n_actions,
                          uint32_t poison_thr, uint8_t* a, float* r, uint8_t* d) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < count;
         f += (int64_t)gridDim.x * blockDim.x) {
        uint64_t t = (uint64_t)t0 + f;
        uint4 x = philox(make_uint4((uint32_t)t, learner, (uint32_t)(t >> 32), SYNTH_TAG_META << 24), key);
        a[f] = (uint8_t)(((uint64_t)x.x * (uint64_t)n_actions) >> 32);
        float rew = 0.0f;
        if (x.y < SYNTH_R_POS_THR) rew = 1.0f;
        else if (x.y < SYNTH_R_NEG_THR) rew = -1.0f;
        if (x.w < poison_thr) rew = SYNTH_POISON_REWARD;
        r[f] = rew;
        d[f] = (uint8_t)(x.z < SYNTH_D_THR);
    }
}

}  // namespace

extern "C" int synth_fill_frames_dev(uint64_t seed, int32_t learner, int64_t t0, int64_t count,
                                     uint8_t* out, void* stream) {
    if (count <= 0) return 0;
    uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    fill_frames<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(key, (uint32_t)learner, t0, count, (uint4*)out);
    return (int)cudaGetLastError();
}

extern "C" int synth_fill_meta_dev(uint64_t seed, int32_t learner, int64_t t0, int64_t count,
                                   int32_t n_actions, uint32_t poison_thr, uint8_t* a, float* r,
                                   uint8_t* d, void* stream) {
    if (count <= 0) return 0;
    uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    fill_meta<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(key, (uint32_t)learner, t0, count, n_actions,
                                                         poison_thr, a, r, d);
    return (int)cudaGetLastError();
}
