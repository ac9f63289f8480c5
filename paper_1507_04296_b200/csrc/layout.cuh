// layout.cuh — Nature-DQN shapes (§5.1) and the library's private layouts.
//
// Canonical (boundary) flat vector: [W1,b1,W2,b2,W3,b3,W4,b4,W5,b5], conv weights OIHW,
// FC [out][in], fc4 input index c*49 + y*7 + x.
// Internal flat vector (theta^+, m, v, G): same tensor offsets, each conv weight
// permuted to O,KH,KW,C ("KRSC", matches NHWC activations) and W4 to [512][y][x][c]
// (matches the NHWC flatten of conv3's output). The optimizer is elementwise, so the
// permutation and the shard split do not change results.
#pragma once
#include <stdint.h>

namespace gorila {

constexpr int IMG = 84, FRAME_BYTES = IMG * IMG, NSTACK = 4;
// conv1 32x(4x8x8)/4 -> 20x20x32 ; conv2 64x(32x4x4)/2 -> 9x9x64 ; conv3 64x(64x3x3)/1 -> 7x7x64
constexpr int C1_OUT = 32, C1_K = 8, C1_S = 4, H1 = 20;
constexpr int C2_OUT = 64, C2_K = 4, C2_S = 2, H2 = 9;
constexpr int C3_OUT = 64, C3_K = 3, C3_S = 1, H3 = 7;
constexpr int FC4_IN = H3 * H3 * C3_OUT;  // 3136
constexpr int FC4_OUT = 512;
constexpr int K1 = C1_K * C1_K * NSTACK;  // 256
constexpr int K2 = C2_K * C2_K * C1_OUT;  // 512
constexpr int K3 = C3_K * C3_K * C2_OUT;  // 576
constexpr int A1 = H1 * H1 * C1_OUT;      // 12800 per sample
constexpr int A2 = H2 * H2 * C2_OUT;      // 5184
constexpr int A3 = FC4_IN;                // 3136
constexpr int A4 = FC4_OUT;               // 512

constexpr int64_t OFF_W1 = 0;
constexpr int64_t OFF_B1 = OFF_W1 + (int64_t)C1_OUT * K1;
constexpr int64_t OFF_W2 = OFF_B1 + C1_OUT;
constexpr int64_t OFF_B2 = OFF_W2 + (int64_t)C2_OUT * K2;
constexpr int64_t OFF_W3 = OFF_B2 + C2_OUT;
constexpr int64_t OFF_B3 = OFF_W3 + (int64_t)C3_OUT * K3;
constexpr int64_t OFF_W4 = OFF_B3 + C3_OUT;
constexpr int64_t OFF_B4 = OFF_W4 + (int64_t)FC4_OUT * FC4_IN;
constexpr int64_t OFF_W5 = OFF_B4 + FC4_OUT;
__host__ __device__ constexpr int64_t off_b5(int nA) { return OFF_W5 + (int64_t)nA * FC4_OUT; }
__host__ __device__ constexpr int64_t param_count(int nA) { return off_b5(nA) + nA; }

// canonical index of internal index i (a permutation within each tensor)
__host__ __device__ inline int64_t canon_of_internal(int64_t i) {
    if (i < OFF_B1) {  // W1: internal [o][ky][kx][c] <- canonical [o][c][ky][kx]
        int64_t o = i / K1, r = i % K1;
        int ky = (int)(r / (C1_K * NSTACK)), kx = (int)(r / NSTACK) % C1_K, c = (int)(r % NSTACK);
        return OFF_W1 + o * K1 + ((int64_t)c * C1_K + ky) * C1_K + kx;
    }
    if (i >= OFF_W2 && i < OFF_B2) {
        int64_t j = i - OFF_W2, o = j / K2, r = j % K2;
        int ky = (int)(r / (C2_K * C1_OUT)), kx = (int)(r / C1_OUT) % C2_K, c = (int)(r % C1_OUT);
        return OFF_W2 + o * K2 + ((int64_t)c * C2_K + ky) * C2_K + kx;
    }
    if (i >= OFF_W3 && i < OFF_B3) {
        int64_t j = i - OFF_W3, o = j / K3, r = j % K3;
        int ky = (int)(r / (C3_K * C2_OUT)), kx = (int)(r / C2_OUT) % C3_K, c = (int)(r % C2_OUT);
        return OFF_W3 + o * K3 + ((int64_t)c * C3_K + ky) * C3_K + kx;
    }
    if (i >= OFF_W4 && i < OFF_B4) {  // W4: internal [n][y][x][c] <- canonical [n][c*49+y*7+x]
        int64_t j = i - OFF_W4, n = j / FC4_IN, r = j % FC4_IN;
        int y = (int)(r / (H3 * C3_OUT)), x = (int)(r / C3_OUT) % H3, c = (int)(r % C3_OUT);
        return OFF_W4 + n * FC4_IN + (int64_t)c * (H3 * H3) + y * H3 + x;
    }
    return i;  // biases, W5, b5 are identical
}

// ------------------------------------------------------------ packed replica
// A replica ("what the kernels read") of theta: the conv / fc4 weights in element type T
// (internal KRSC order; the backward reads the same copy through MN-major descriptors),
// and an fp32 area with the biases and fc5.
//   T:    w1 [32][256], w2 [64][512], w3 [64][576], w4 [512][3136]
//   fp32: b1 b2 b3 b4 w5 [nA][512] b5
struct ReplicaLayout {
    int64_t w1, w2, w3, w4, n_t;     // element offsets / count in T
    int64_t b1, b2, b3, b4, w5, b5, n_f;  // element offsets / count in the fp32 area
};
__host__ __device__ inline ReplicaLayout replica_layout(int nA) {
    ReplicaLayout L{};
    L.w1 = 0;
    L.w2 = L.w1 + (int64_t)C1_OUT * K1;
    L.w3 = L.w2 + (int64_t)C2_OUT * K2;
    L.w4 = L.w3 + (int64_t)C3_OUT * K3;
    L.n_t = (L.w4 + (int64_t)FC4_OUT * FC4_IN + 127) / 128 * 128;
    L.b1 = 0; L.b2 = 32; L.b3 = 96; L.b4 = 160; L.w5 = 672;
    L.b5 = L.w5 + (int64_t)nA * FC4_OUT;
    L.n_f = (L.b5 + nA + 4 + 63) / 64 * 64;  // room for the 4-wide tail of the optimizer's emission
    return L;
}

// where internal element i lives in the replica: returns the T-area offset (>= 0) or
// -(fp32-area offset) - 1
__host__ __device__ inline int64_t replica_slot(const ReplicaLayout& L, int64_t i) {
    if (i < OFF_B1) return L.w1 + i;
    if (i < OFF_W2) return -(L.b1 + (i - OFF_B1)) - 1;
    if (i < OFF_B2) return L.w2 + (i - OFF_W2);
    if (i < OFF_W3) return -(L.b2 + (i - OFF_B2)) - 1;
    if (i < OFF_B3) return L.w3 + (i - OFF_W3);
    if (i < OFF_W4) return -(L.b3 + (i - OFF_B3)) - 1;
    if (i < OFF_B4) return L.w4 + (i - OFF_W4);
    if (i < OFF_W5) return -(L.b4 + (i - OFF_B4)) - 1;
    return -(L.w5 + (i - OFF_W5)) - 1;  // W5 then b5 are contiguous in both layouts
}

}  // namespace gorila
