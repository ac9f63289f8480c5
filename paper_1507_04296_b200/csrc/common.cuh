// common.cuh — shared device helpers of the Gorila B200 library (no method arithmetic here).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

#define GORILA_DEV __device__ __forceinline__

namespace gorila {

// ----------------------------------------------------------------- element types
template <typename T> struct Elem;
template <> struct Elem<float> {
    static GORILA_DEV float to_f(float v) { return v; }
    static GORILA_DEV float from_f(float v) { return v; }
};
template <> struct Elem<__nv_bfloat16> {
    static GORILA_DEV float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
    // round-to-nearest-even (reading R16)
    static GORILA_DEV __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }
};

template <typename T> GORILA_DEV float tof(T v) { return Elem<T>::to_f(v); }
template <typename T> GORILA_DEV T fromf(float v) { return Elem<T>::from_f(v); }

// ----------------------------------------------------------------- Philox4x32-10
GORILA_DEV uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// ----------------------------------------------------------------- warp helpers
GORILA_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
GORILA_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ----------------------------------------------------------------- sm_100a PTX wrappers
GORILA_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

GORILA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
GORILA_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
GORILA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
GORILA_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// make generic-proxy st.shared visible to the tensor core (async proxy)
GORILA_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

GORILA_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
GORILA_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
GORILA_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
GORILA_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate (kind::f16), issued by one thread.
GORILA_DEV void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-uniform issue: the whole warp executes the call and elect.sync picks the issuing lane. With
// the issuing loop and its operands warp-uniform (warp_uniform() / uniform_u32() make that visible
// to the compiler), descriptors and TMEM addresses stay in uniform registers and an MMA issues with
// no R2UR moves or ELECT waterfall per instruction (tools/mma_rate_probe.cu, every SM issuing:
// M64 N32 24 vs 45 cycles per MMA, M128 N32 40 vs 45).
GORILA_DEV void umma_bf16_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
GORILA_DEV void umma_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
GORILA_DEV int warp_uniform() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
GORILA_DEV uint32_t uniform_u32(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }
GORILA_DEV uint64_t uniform_u64(uint64_t v) { return __shfl_sync(0xffffffffu, (unsigned long long)v, 0); }
// arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete
GORILA_DEV void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread
GORILA_DEV void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// two 16-column loads in flight, one wait: columns [c, c + 32) of the warp's 32 lanes
GORILA_DEV void tmem_ld16x2(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr + 16u));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- optional per-CTA timeline instrumentation (diagnostics build only: -DGORILA_TRACE)
#ifdef GORILA_TRACE
__device__ unsigned long long gorila_trace_buf[64];
#define GTRACE(slot)                                                                              \
    do {                                                                                          \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) {         \
            unsigned long long t_;                                                               \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                  \
            gorila_trace_buf[(slot)] = t_;                                                       \
        }                                                                                         \
    } while (0)
// per-tile events of CTA 0 of a persistent engine: gorila_trace_tiles[ev][tile] (tile < 64);
// -DGORILA_TRACE_CONV: instead every converter warp's hand-over time (GTRACE_C)
__device__ unsigned long long gorila_trace_tiles[8 * 64];
#ifdef GORILA_TRACE_CONV
#define GTRACE_C(ev, tl) GTRACE_T_(ev, tl)
#define GTRACE_T(ev, tl) \
    do {                 \
    } while (0)
#else
#define GTRACE_C(ev, tl) \
    do {                 \
    } while (0)
#define GTRACE_T(ev, tl) GTRACE_T_(ev, tl)
#endif
#define GTRACE_T_(ev, tl)                                                                         \
    do {                                                                                          \
        if (blockIdx.x == 0 && (tl) < 64) {                                                       \
            unsigned long long t_;                                                               \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                  \
            gorila_trace_tiles[(ev) * 64 + (tl)] = t_;                                           \
        }                                                                                         \
    } while (0)
#else
#define GTRACE(slot) \
    do {             \
    } while (0)
#define GTRACE_T(ev, tl) \
    do {                 \
    } while (0)
#define GTRACE_C(ev, tl) \
    do {                 \
    } while (0)
#endif

// ---- cp.async (LDGSTS): 16-byte global -> shared copies; src_bytes = 0 zero-fills the destination
GORILA_DEV void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
GORILA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
GORILA_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- TMA (cp.async.bulk.tensor) into shared memory, completion counted on an mbarrier
GORILA_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// contiguous bytes (multiple of 16, 16-B aligned) global -> shared in one bulk copy
GORILA_DEV void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
GORILA_DEV void tma_load(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
GORILA_DEV void tma_load(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
GORILA_DEV void tma_load(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
GORILA_DEV void tma_load(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int c0, int c1, int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
        "[%7];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}
GORILA_DEV void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---- programmatic dependent launch: wait for the preceding grid's results / let the next grid launch
GORILA_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
GORILA_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- thread-block clusters / distributed shared memory
GORILA_DEV uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
GORILA_DEV void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same smem location in CTA `rank` of the cluster
GORILA_DEV uint32_t dsmem_map(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
GORILA_DEV float4 dsmem_ld4(uint32_t caddr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(caddr) : "memory");
    return v;
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major canonical layout:
// core matrix = 8 rows x 16 B contiguous; LBO = byte step between K-adjacent core
// matrices; SBO = byte step between M/N-adjacent 8-row groups; version 1 (sm_100).
GORILA_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;                // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
}
// K-major swizzled layouts written by TMA with SWIZZLE_128B / 64B / 32B: rows of 128 / 64 / 32 B,
// 8-row atoms (SBO = 8 rows), K steps of 16 elements advance the start address by 32 B inside the
// row; layout_type 2 / 4 / 6. The swizzle follows the absolute shared-memory address, so a start
// address shifted by whole rows (not atoms) is valid with base offset 0 (tools/umma_shift_probe.cu).
GORILA_DEV uint64_t umma_desc_sw(uint32_t saddr, uint32_t row_bytes) {
    const uint64_t layout = row_bytes == 128 ? 2ull : row_bytes == 64 ? 4ull : 6ull;  // 6: SWIZZLE_32B
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                            // LBO (unused for swizzled K-major)
    d |= (uint64_t)(((8 * row_bytes) >> 4) & 0x3FFF) << 32;  // SBO = one 8-row atom
    d |= (uint64_t)1 << 46;                            // version
    d |= layout << 61;
    return d;
}
// MN-major swizzled layouts (SWIZZLE_128B / 64B / 32B, blocks of 64 / 32 / 16 MN elements): K rows
// of 128 / 64 / 32 B, 8-row atoms; LBO = byte stride between MN blocks, SBO = byte stride between
// 8-row K groups (the roles are swapped relative to the no-swizzle layout).
GORILA_DEV uint64_t umma_desc_mn_sw(uint32_t saddr, uint32_t lbo, uint32_t row_bytes) {
    const uint64_t layout = row_bytes == 128 ? 2ull : row_bytes == 64 ? 4ull : 6ull;
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)(((8 * row_bytes) >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= layout << 61;
    return d;
}
// instruction descriptor: D f32, A/B bf16, both K-major, M x N
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace gorila
