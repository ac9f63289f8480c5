// mma_rate_probe.cu — issue rate of tcgen05.mma (kind::f16, cta_group::1) by shape and operand
// layout, every SM running the same loop: cycles per MMA for M x N x 16 with A / B in shared memory
// (K-major SWIZZLE_32B / 128B, MN-major SWIZZLE_32B) or A in TMEM, one accumulator or four
// interleaved. Which operand fetch bounds the N = 32 GEMMs of conv1 / conv2? (Run on a B200.)
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_1507_04296_b200/csrc tools/mma_rate_probe.cu -o /tmp/mma_rate_probe
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

using namespace gorila;

GORILA_DEV uint64_t desc_k(uint32_t saddr, uint32_t rb) {  // K-major swizzled
    const uint64_t layout = rb == 128 ? 2ull : rb == 64 ? 4ull : 6ull;
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(((8 * rb) >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= layout << 61;
    return d;
}
GORILA_DEV void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

// mode: 0 SS A K-major (rb_a), 1 SS A MN-major SW32 (M blocks 16 el, LBO 4096), 2 A in TMEM
__global__ void __launch_bounds__(128) probe(int mode, int M, int N, int rb_a, int nacc, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    for (int o = tid * 16; o < 160 * 1024; o += 128 * 16) *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid < 32) tmem_alloc(&slot, 512);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        const uint32_t a0 = smem_u32(smem), b0 = a0 + 64 * 1024;
        uint32_t idesc = umma_idesc_bf16(M, N);
        if (mode == 1) idesc |= 1u << 15;
        const uint64_t bd = desc_k(b0, 128);
        const uint64_t ad = mode == 1 ? umma_desc_mn_sw(a0, 4096, 32) : desc_k(a0, rb_a);
        const uint32_t ncol = N;  // accumulator columns
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int a = i % nacc;
            const uint32_t d = tmem + a * ncol;
            // K steps walk through the operand buffers (32 B per step, rows stay in place)
            const uint32_t koff = (uint32_t)((i / nacc) & 3) * 32;
            if (mode == 2) umma_ts(d, tmem + 384 + ((i / nacc) & 3) * 8, bd + (koff >> 4), idesc, 1u);
            else umma_bf16(d, ad + (koff >> 4), bd + (koff >> 4), idesc, 1u);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(tmem, 512);
}


GORILA_DEV void umma_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
GORILA_DEV void umma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
GORILA_DEV void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
// unrolled: NACC accumulators x 4 K steps per iteration, constant descriptor deltas (as the GEMM
// engines). MODE 0: A K-major (RA-byte swizzle rows), 1: A MN-major SWIZZLE_32B (16-element blocks
// 4 KB apart), 2: A in TMEM; B K-major (RB-byte swizzle rows). WARP: the whole warp runs the loop
// and elect.sync picks the issuing lane inside the asm (else one thread).
template <int MODE, int M, int N, int RA, int RB, int NACC, bool WARP, int SHIFT = 0, int LBO = 4096>
__global__ void __launch_bounds__(128) probe2(int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    for (int o = tid * 16; o < 160 * 1024; o += 128 * 16) *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (tid < 32) tmem_alloc(&slot, 512);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // warp-uniform values (a __shfl_sync result is known uniform): the descriptors and the TMEM
    // address can then live in uniform registers, with no R2UR per MMA
    const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);
    const int warp_u = __shfl_sync(0xffffffffu, tid >> 5, 0);
    constexpr uint32_t IDESC = umma_idesc_bf16(M, N) | (MODE == 1 ? (1u << 15) : 0u);
    const uint32_t a0 = __shfl_sync(0xffffffffu, smem_u32(smem), 0), b0 = a0 + 64 * 1024;
    const uint64_t ad = MODE == 1 ? umma_desc_mn_sw(a0 + SHIFT * 32, LBO, 32) : desc_k(a0 + SHIFT * RA, RA),
                   bd = desc_k(b0, RB);
    // K step deltas (descriptor address units of 16 B): K-major 32 B; MN-major 16 rows of 32 B
    constexpr int DA = MODE == 1 ? 32 : 2, DB = 2;
    if (WARP ? warp_u == 0 : tid == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters / (4 * NACC); ++i) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                for (int a = 0; a < NACC; ++a) {
                    const uint32_t d = tmem + a * N;
                    if (MODE == 2 && WARP) umma_ts_elect(d, tmem + 384 + kk * 8, bd + kk * DB, IDESC, 1u);
                    else if (MODE == 2) umma_ts(d, tmem + 384 + kk * 8, bd + kk * DB, IDESC, 1u);
                    else if (WARP) umma_elect(d, ad + kk * DA, bd + kk * DB, IDESC, 1u);
                    else umma_bf16(d, ad + kk * DA, bd + kk * DB, IDESC, 1u);
                }
        }
        if (WARP) commit_elect(&bar);
        else umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (tid == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(tmem, 512);
}
template <int MODE, int M, int N, int RA, int RB, int NACC, bool WARP, int SHIFT = 0, int LBO = 4096>
void run2(long long* d, const char* what) {
    const int iters = 4096;
    auto k = probe2<MODE, M, N, RA, RB, NACC, WARP, SHIFT, LBO>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024 + 1024);
    k<<<148, 128, 161 * 1024 + 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s M%d N%d: %s\n", what, M, N, cudaGetErrorString(e)); exit(1); }
    long long h[148];
    cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cyc = (double)mx / iters;
    printf("%-34s sh%d lbo%5d M%3d N%3d acc%d %s: %6.1f cyc/MMA  %5.0f MAC/cyc/SM (%3.0f%%)\n", what, SHIFT, LBO, M, N, NACC,
           WARP ? "warp" : "1thr", cyc, (double)M * N * 16 / cyc, 100.0 * M * N * 16 / cyc / 4096);
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024 + 1024);
    struct V { int mode, M, N, rb, nacc; const char* what; } vs[] = {
        {0, 128, 32, 32, 1, "SS K-major SW32 A"}, {0, 128, 32, 32, 4, "SS K-major SW32 A"},
        {0, 128, 32, 128, 4, "SS K-major SW128 A"}, {0, 128, 64, 32, 4, "SS K-major SW32 A"},
        {0, 128, 64, 128, 4, "SS K-major SW128 A"}, {0, 128, 128, 128, 2, "SS K-major SW128 A"},
        {0, 128, 256, 128, 1, "SS K-major SW128 A"}, {1, 64, 32, 32, 4, "SS MN-major SW32 A"},
        {1, 128, 32, 32, 4, "SS MN-major SW32 A"}, {0, 64, 32, 128, 4, "SS K-major SW128 A"},
        {2, 128, 32, 0, 4, "TS (A in TMEM)"}, {2, 128, 64, 0, 4, "TS (A in TMEM)"},
        {2, 128, 128, 0, 2, "TS (A in TMEM)"},
    };
    run2<0, 128, 32, 32, 32, 4, true>(d, "SS A K SW32, B K SW32 (conv1 fwd)");
    run2<0, 128, 32, 32, 32, 4, true, 1>(d, "SS A K SW32, B K SW32 (conv1 fwd)");
    run2<0, 128, 32, 32, 32, 4, true, 5>(d, "SS A K SW32, B K SW32 (conv1 fwd)");
    run2<0, 128, 32, 32, 32, 4, false, 5>(d, "SS A K SW32, B K SW32 (conv1 fwd)");
    run2<1, 64, 32, 32, 64, 4, true>(d, "SS A MN SW32, B MN SW64 (c1 wgrad)");
    run2<1, 64, 32, 32, 64, 4, true, 1>(d, "SS A MN SW32 (c1 wgrad u8)");
    run2<1, 64, 32, 32, 64, 4, true, 5, 17408>(d, "SS A MN SW32 (c1 wgrad u8)");
    run2<1, 64, 32, 32, 64, 4, false, 5, 17408>(d, "SS A MN SW32 (c1 wgrad u8)");
    run2<0, 128, 64, 128, 128, 4, true, 3>(d, "SS A K SW128, B K SW128");
    return 0;
    const int iters = 4096;
    for (auto& v : vs)
        for (int grid : {1, 148}) {
            probe<<<grid, 128, 161 * 1024 + 1024>>>(v.mode, v.M, v.N, v.rb, v.nacc, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("%s M%d N%d: %s\n", v.what, v.M, v.N, cudaGetErrorString(e));
                return 1;
            }
            long long h[148];
            cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            const double cyc = (double)mx / iters;
            printf("%-22s M%3d N%3d acc%d grid%3d: %6.1f cyc/MMA  %7.0f MAC/cyc/SM (%.0f%% of 4096)\n", v.what, v.M, v.N,
                   v.nacc, grid, cyc, (double)v.M * v.N * 16 / cyc, 100.0 * v.M * v.N * 16 / cyc / 4096);
        }
    return 0;
}
