// umma_shift_probe.cu — does a K-major SWIZZLE_128B UMMA operand tolerate a start address
// (and 64-B / 32-B) shifted by r rows (not a multiple of the 8-row swizzle atom)? And what must the
// descriptor's base-offset field (bits 49..51) hold then? (Run on a B200.)
//
// A [256][64] and B [32][64] bf16 land in shared memory through TMA (SWIZZLE_128B). For each
// shift r, D[128][32] = A[r .. r+128) . B^T is computed with 4 tcgen05.mma K-steps, once with
// base_offset = 0 and once with base_offset = r & 7, and compared with the host product.
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_1507_04296_b200/csrc tools/umma_shift_probe.cu -o tools/umma_shift_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "common.cuh"

using namespace gorila;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

GORILA_DEV uint64_t desc_rb(uint32_t saddr, uint32_t rb) {
    const uint64_t layout = rb == 128 ? 2ull : rb == 64 ? 4ull : 6ull;
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(((8 * rb) >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= layout << 61;
    return d;
}
__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap ma,
                                             const __grid_constant__ CUtensorMap mb, int shift, int base_off_mode,
                                             int rb, float* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar, done;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tmem_alloc(&slot, 32);
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_init(&done, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t a = smem_u32(sm), b = a + 256 * 128;
    if (tid == 0) {
        tma_load(&ma, a, &bar, 0, 0);
        tma_load(&mb, b, &bar, 0, 0);
        mbar_expect_tx(&bar, 256 * rb + 32 * rb);
    }
    mbar_wait(&bar, 0);
    const uint32_t tmem = slot;
    if (tid == 0) {
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, 32);
        for (int kk = 0; kk < rb / 32; ++kk) {
            const uint32_t start = a + shift * rb + kk * 32;
            uint64_t ad = desc_rb(start, rb);
            if (base_off_mode == 1) ad |= (uint64_t)((start >> 7) & 7) << 49;
            umma_bf16(tmem, ad, desc_rb(b + kk * 32, rb), idesc, kk > 0 ? 1u : 0u);
        }
        umma_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
    tc_fence_after();
    float v[16];
    for (int c0 = 0; c0 < 32; c0 += 16) {
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        for (int e = 0; e < 16; ++e) out[(warp * 32 + lane) * 32 + c0 + e] = v[e];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 32);
}

static float bf(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    int all_ok = 1;
    for (int rb : {128, 64, 32}) {
    const int K = rb / 2;
    std::vector<uint16_t> A(256 * K), B(32 * K);
    srand(7 + rb);
    for (auto& x : A) x = (uint16_t)(0x3f80 + (rand() % 64) - 32);  // ~[0.5, 2) bf16
    for (auto& x : B) x = (uint16_t)(0x3f80 + (rand() % 64) - 32);
    uint16_t *dA, *dB;
    float* dO;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dO, 128 * 32 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CUtensorMap ma, mb;
    cuuint64_t da[2] = {(cuuint64_t)K, 256}, db[2] = {(cuuint64_t)K, 32}, st[1] = {(cuuint64_t)rb};
    cuuint32_t ba[2] = {(cuuint32_t)K, 256}, bb[2] = {(cuuint32_t)K, 32}, es[2] = {1, 1};
    const CUtensorMapSwizzle sw = rb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                                      : CU_TENSOR_MAP_SWIZZLE_32B;
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, da, st, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
        enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, db, st, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
        printf("encode failed\n");
        return 1;
    }
    const int smem = 1024 + 256 * 128 + 32 * 128;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    std::vector<float> o(128 * 32);
    int ok_mode[2] = {1, 1};
    const int shifts[] = {0, 1, 3, 7, 8, 9, 13, 21};
    for (int mode = 0; mode < 2; ++mode)
        for (int r : shifts) {
            probe<<<1, 128, smem>>>(ma, mb, r, mode, rb, dO);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (int i = 0; i < 128; ++i)
                for (int j = 0; j < 32; ++j) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k) ref += (double)bf(A[(i + r) * K + k]) * bf(B[j * K + k]);
                    if (fabs(o[i * 32 + j] - ref) > 1e-3 * fabs(ref) + 1e-3) ++bad;
                }
            if (bad) ok_mode[mode] = 0;
            if (bad || r == 21) printf("rb %3d base_offset mode %d shift %2d: %d mismatches\n", rb, mode, r, bad);
        }
    printf("RESULT rb %d: mode0(base_offset=0)=%s mode1(base_offset=(start>>7)&7)=%s\n", rb,
           ok_mode[0] ? "OK" : "FAIL", ok_mode[1] ? "OK" : "FAIL");
    all_ok &= ok_mode[0];
    }
    printf(all_ok ? "SHIFT PROBE OK\n" : "SHIFT PROBE FAILED\n");
    return 0;
}
