// tma_probe.cu — checks the TMA features the GEMM engine relies on (run on a B200):
//  (1) a 3-D view of a row-major [rows][K] bf16 matrix as (8, rows, K/8) with strides
//      (2*K bytes, 16 bytes): non-monotonic strides, box (8, 128, 8) -> [kgroup][row][8];
//  (2) a 5-D NHWC view with element strides (1,2,2,1,1) and negative start coordinates
//      (zero fill out of bounds).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void probe(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3, int c4, int bytes,
                      uint16_t* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes));
        if (RANK == 3)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                "[%5];" ::"r"(smem_u32(smem)),
                "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar))
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
                "%6}], [%7];" ::"r"(smem_u32(smem)),
                "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(&bar))
                : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra WAIT;\n\t}" ::"r"(
            smem_u32(&bar)));
    for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(smem)[i];
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    int fails = 0;
    // ---- (1) K-major 3-D trick
    {
        const int rows = 300, K = 192;
        uint16_t* h = (uint16_t*)malloc(rows * K * 2);
        for (int r = 0; r < rows; ++r)
            for (int k = 0; k < K; ++k) h[r * K + k] = (uint16_t)(r * 1000 + k);
        uint16_t *d, *o;
        CK(cudaMalloc(&d, rows * K * 2));
        CK(cudaMalloc(&o, 128 * 64 * 2));
        CK(cudaMemcpy(d, h, rows * K * 2, cudaMemcpyHostToDevice));
        CUtensorMap map;
        cuuint64_t dims[3] = {8, (cuuint64_t)rows, (cuuint64_t)K / 8};
        cuuint64_t strides[2] = {(cuuint64_t)K * 2, 16};
        cuuint32_t box[3] = {8, 128, 8}, es[3] = {1, 1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode 3d: %d\n", (int)r);
        if (r == CUDA_SUCCESS) {
            const int row0 = 250, kg0 = 8;  // rows 250..377 (OOB beyond 299), k 64..127
            probe<3><<<1, 128, 128 * 64 * 2>>>(map, 0, row0, kg0, 0, 0, 128 * 64 * 2, o);
            CK(cudaDeviceSynchronize());
            uint16_t* ho = (uint16_t*)malloc(128 * 64 * 2);
            CK(cudaMemcpy(ho, o, 128 * 64 * 2, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (int kg = 0; kg < 8; ++kg)
                for (int rr = 0; rr < 128; ++rr)
                    for (int e = 0; e < 8; ++e) {
                        int row = row0 + rr, k = (kg0 + kg) * 8 + e;
                        uint16_t expect = row < rows ? (uint16_t)(row * 1000 + k) : 0;
                        if (ho[(kg * 128 + rr) * 8 + e] != expect) ++bad;
                    }
            printf("3d trick: %d mismatches\n", bad);
            fails += bad != 0;
        } else {
            fails++;
        }
    }
    // ---- (2) 5-D NHWC strided box with negative coordinates
    {
        const int B = 3, H = 20, W = 20, C = 32;
        size_t n = (size_t)B * H * W * C;
        uint16_t* h = (uint16_t*)malloc(n * 2);
        for (size_t i = 0; i < n; ++i) h[i] = (uint16_t)(i % 60000 + 1);
        uint16_t *d, *o;
        CK(cudaMalloc(&d, n * 2));
        CK(cudaMalloc(&o, 65536));
        CK(cudaMemcpy(d, h, n * 2, cudaMemcpyHostToDevice));
        // dims (8 c_in, W, H, B, C/8) ; strides (C*2, W*C*2, H*W*C*2, 16)
        CUtensorMap map;
        cuuint64_t dims[5] = {8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)C / 8};
        cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, 16};
        cuuint32_t box[5] = {8, 18, 18, 2, 4}, es[5] = {1, 2, 2, 1, 1};  // 9 x 9 pixels with stride 2
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode 5d: %d\n", (int)r);
        if (r == CUDA_SUCCESS) {
            const int x0 = -1, y0 = 1, b0 = 1;
            const int bytes = 4 * 2 * 9 * 9 * 8 * 2;
            probe<5><<<1, 128, bytes>>>(map, 0, x0, y0, b0, 0, bytes, o);
            CK(cudaDeviceSynchronize());
            uint16_t* ho = (uint16_t*)malloc(bytes);
            CK(cudaMemcpy(ho, o, bytes, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (int cg = 0; cg < 4; ++cg)
                for (int bb = 0; bb < 2; ++bb)
                    for (int yy = 0; yy < 9; ++yy)
                        for (int xx = 0; xx < 9; ++xx)
                            for (int e = 0; e < 8; ++e) {
                                int b = b0 + bb, y = y0 + 2 * yy, x = x0 + 2 * xx, c = cg * 8 + e;
                                bool in = b < B && y >= 0 && y < H && x >= 0 && x < W;
                                uint16_t expect = in ? h[(((size_t)b * H + y) * W + x) * C + c] : 0;
                                size_t idx = ((((size_t)cg * 2 + bb) * 9 + yy) * 9 + xx) * 8 + e;
                                if (ho[idx] != expect) ++bad;
                            }
            printf("5d strided/negative: %d mismatches\n", bad);
            fails += bad != 0;
        } else {
            fails++;
        }
    }
    printf(fails ? "TMA PROBE FAILED\n" : "TMA PROBE OK\n");
    return fails;
}
