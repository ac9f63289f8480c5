// Remote (NVLink peer) random-frame gather cost vs local: the f4 sampler's access pattern.
// grid (2, B) x 256 threads, each thread 5 x 16-B loads at a random frame of a ring of `span` bytes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int FB = 7056;
__global__ void gather(const uint8_t* ring, int64_t nframes, uint64_t seed, uint8_t* out, int mode) {
    const int b = blockIdx.y;
    uint64_t h = (seed + b) * 0x9E3779B97F4A7C15ull; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    const int64_t tau = 3 + (int64_t)(h % (uint64_t)(nframes - 5));
    const int chunk = blockIdx.x * blockDim.x + threadIdx.x;
    if (chunk >= FB / 16) return;
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        uint4 v;
        const uint4* p = reinterpret_cast<const uint4*>(ring + (tau - 3 + t) * FB + chunk * 16);
        if (mode == 0) v = __ldcg(p); else v = *p;
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    reinterpret_cast<uint4*>(out)[(int64_t)b * (FB / 16) + chunk] = acc;
}
__global__ void chain(const uint64_t* p, int n, uint64_t* out) {  // dependent remote loads: latency
    uint64_t i = 0;
    for (int k = 0; k < n; ++k) i = __ldcg(p + (i & 1023));
    *out = i;
}
int main() {
    int nd = 0; cudaGetDeviceCount(&nd);
    if (nd < 2) { printf("need 2 GPUs\n"); return 1; }
    const size_t big = (size_t)1000000 * FB;
    uint8_t *r0, *r1, *out; uint64_t* o8;
    CK(cudaSetDevice(1)); CK(cudaMalloc(&r1, big)); CK(cudaMemset(r1, 1, big));
    CK(cudaSetDevice(0)); CK(cudaMalloc(&r0, big)); CK(cudaMemset(r0, 1, big));
    CK(cudaMalloc(&out, 1 << 24)); CK(cudaMalloc(&o8, 8));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int B : {32, 256}) for (int mode = 0; mode < 2; ++mode)
    for (int remote = 0; remote < 2; ++remote) for (int64_t nf : {(int64_t)1000000, (int64_t)10000}) {
        const uint8_t* ring = remote ? r1 : r0;
        for (int w = 0; w < 20; ++w) gather<<<dim3(2, B), 256>>>(ring, nf, w * 77, out, mode);
        cudaEventRecord(e0);
        const int it = 200;
        for (int w = 0; w < it; ++w) gather<<<dim3(2, B), 256>>>(ring, nf, 1000 + w * 131, out, mode);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("B %3d %s %s span %5.0f MB: %6.2f us per launch\n", B, mode ? "ld   " : "ldcg ", remote ? "remote" : "local ",
               nf * FB / 1e6, ms * 1000 / it);
    }
    for (int remote = 0; remote < 2; ++remote) {
        const uint64_t* p = (const uint64_t*)(remote ? r1 : r0);
        CK(cudaMemset(remote ? (void*)nullptr : (void*)r0, 0, 0));
        cudaEventRecord(e0);
        chain<<<1, 1>>>(p, 1000, o8);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("dependent %s load latency: %.2f us\n", remote ? "remote" : "local ", ms * 1000 / 1000);
    }
    return 0;
}
