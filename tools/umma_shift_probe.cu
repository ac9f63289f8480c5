// umma_shift_probe.cu — does a K-major SWIZZLE_128B UMMA operand tolerate a start address
// shifted by r 128-B rows (not a multiple of the 8-row / 1024-B swizzle atom)? And what must the
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

__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap ma,
                                             const __grid_constant__ CUtensorMap mb, int shift, int base_off_mode,
                                             float* out) {
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
        mbar_expect_tx(&bar, 256 * 128 + 32 * 128);
    }
    mbar_wait(&bar, 0);
    const uint32_t tmem = slot;
    if (tid == 0) {
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, 32);
        for (int kk = 0; kk < 4; ++kk) {
            const uint32_t start = a + shift * 128 + kk * 32;
            uint64_t ad = umma_desc_sw(start, 128);
            if (base_off_mode == 1) ad |= (uint64_t)((start >> 7) & 7) << 49;
            umma_bf16(tmem, ad, umma_desc_sw(b + kk * 32, 128), idesc, kk > 0 ? 1u : 0u);
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
    std::vector<uint16_t> A(256 * 64), B(32 * 64);
    srand(7);
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
    cuuint64_t da[2] = {64, 256}, db[2] = {64, 32}, st[1] = {128};
    cuuint32_t ba[2] = {64, 256}, bb[2] = {64, 32}, es[2] = {1, 1};
    if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, da, st, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
        enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dB, db, st, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
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
            probe<<<1, 128, smem>>>(ma, mb, r, mode, dO);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (int i = 0; i < 128; ++i)
                for (int j = 0; j < 32; ++j) {
                    double ref = 0;
                    for (int k = 0; k < 64; ++k) ref += (double)bf(A[(i + r) * 64 + k]) * bf(B[j * 64 + k]);
                    if (fabs(o[i * 32 + j] - ref) > 1e-3 * fabs(ref) + 1e-3) ++bad;
                }
            printf("base_offset mode %d shift %2d: %d mismatches\n", mode, r, bad);
            if (bad) ok_mode[mode] = 0;
        }
    printf("RESULT mode0(base_offset=0)=%s mode1(base_offset=(start>>7)&7)=%s\n", ok_mode[0] ? "OK" : "FAIL",
           ok_mode[1] ? "OK" : "FAIL");
    return 0;
}
