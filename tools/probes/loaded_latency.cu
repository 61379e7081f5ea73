// Probe: dependent-load latency (pointer chase) with the GPU idle and while a
// persistent streaming copy saturates HBM, for an HBM-resident and an
// L2-resident chase array.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void stream_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            uint4 v;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
            asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
}
__global__ void chase(const unsigned* __restrict__ next, int hops, long long* out, int delay_ns) {
    if (delay_ns) {
        unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        unsigned long long t; do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)delay_ns);
    }
    unsigned p = threadIdx.x * 977;
    long long c0 = clock64();
    for (int h = 0; h < hops; ++h) p = __ldcg(next + p);
    long long c1 = clock64();
    if (threadIdx.x == 0) { out[0] = (c1 - c0) / hops; out[1] = p; }
}
int main() {
    const size_t big = 512ull << 20;  // bytes per copy buffer
    uint4 *a, *b;
    cudaMalloc(&a, big); cudaMalloc(&b, big);
    cudaMemset(a, 1, big);
    long long* out; cudaMalloc(&out, 16);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t words : {size_t(1) << 18 /*1 MB*/, size_t(1) << 24 /*64 MB*/, size_t(1) << 27 /*512 MB*/}) {
        std::vector<unsigned> perm(words), nxt(words);
        for (size_t i = 0; i < words; ++i) perm[i] = (unsigned)i;
        srand(1);
        for (size_t i = words - 1; i > 0; --i) { size_t j = ((size_t)rand() * 65536 + rand()) % (i + 1); std::swap(perm[i], perm[j]); }
        for (size_t i = 0; i < words; ++i) nxt[perm[i]] = perm[(i + 1) % words];
        unsigned* d; cudaMalloc(&d, words * 4);
        cudaMemcpy(d, nxt.data(), words * 4, cudaMemcpyHostToDevice);
        for (int ctas_per_sm : {0, 1, 2, 3, 4, 6}) {
            long long h[2];
            chase<<<1, 32, 0, s2>>>(d, 64, out, 0);  // warm L2 for the small case
            cudaDeviceSynchronize();
            if (ctas_per_sm) stream_copy<<<sms * ctas_per_sm, 128, 0, s1>>>(a, b, big / 16, 4);
            chase<<<1, 32, 0, s2>>>(d, 2000, out, ctas_per_sm ? 20000 : 0);
            cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s2);
            cudaDeviceSynchronize();
            printf("chase array %4zu MB  copy CTAs/SM %d : %6lld cycles/hop (%.2f us)\n", words * 4 >> 20, ctas_per_sm, h[0], h[0] / 1965.0);
        }
        cudaFree(d);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
