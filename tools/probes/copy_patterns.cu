// Probe: achievable bandwidth of the replay step's copy patterns on this GPU
// (read+write bytes / time, L2 cleared by a 256 MB read before each run).
//  A: contiguous -> contiguous          (reference copy)
//  B: contiguous -> scattered 16 KB rows (payload insert pattern)
//  C: scattered 16 KB rows -> contiguous (gather pattern)
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void flush(const float4* p, size_t n, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += p[i].x;
    if (s == 1234.5f) *out = s;
}
template <int U>
__global__ void copy_rows(const uint4* __restrict__ src, uint4* __restrict__ dst, const int* srow,
                          const int* drow, int nrows, int qpr /* quads per row */) {
    const long long total = (long long)nrows * qpr;
    for (long long b = (long long)blockIdx.x * blockDim.x * U; b < total; b += (long long)gridDim.x * blockDim.x * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = b + threadIdx.x + (long long)u * blockDim.x;
            if (i < total) {
                const int r = (int)(i / qpr), q = (int)(i % qpr);
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + (size_t)srow[r] * qpr + q));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = b + threadIdx.x + (long long)u * blockDim.x;
            if (i < total) {
                const int r = (int)(i / qpr), q = (int)(i % qpr);
                asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst + (size_t)drow[r] * qpr + q), "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w) : "memory");
            }
        }
    }
}
int main() {
    const int qpr = 1024;                 // 16 KB rows
    const int nrows_buf = 32768;          // 512 MB slot store
    const size_t big = (size_t)nrows_buf * qpr;
    uint4 *store, *packed;
    cudaMalloc(&store, big * 16);
    cudaMalloc(&packed, (size_t)8192 * qpr * 16);
    float4* fl; cudaMalloc(&fl, 256u << 20); float* fo; cudaMalloc(&fo, 4);
    cudaMemset(store, 1, big * 16); cudaMemset(packed, 2, (size_t)8192 * qpr * 16); cudaMemset(fl, 0, 256u << 20);
    int *ident, *scat;
    cudaMalloc(&ident, 32768 * 4); cudaMalloc(&scat, 32768 * 4);
    std::vector<int> h(32768), hs(32768);
    for (int i = 0; i < 32768; ++i) h[i] = i, hs[i] = i;
    std::mt19937 g(1); std::shuffle(hs.begin(), hs.end(), g);
    cudaMemcpy(ident, h.data(), 32768 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(scat, hs.data(), 32768 * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    struct Case { const char* name; int rows; bool scat_src, scat_dst; };
    Case cases[] = {{"A contiguous->contiguous 2x1293 rows", 2586, false, false},
                    {"B contiguous->scattered  2x1293 rows", 2586, false, true},
                    {"C scattered->contiguous  4096 rows   ", 4096, true, false},
                    {"C scattered->contiguous  8192 rows   ", 8192, true, false}};
    for (auto& c : cases) {
        for (int ctas : {2, 4, 8}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                flush<<<sms * 4, 256>>>(fl, (256u << 20) / 16, fo);
                cudaEventRecord(e0);
                if (c.scat_src)
                    copy_rows<4><<<sms * ctas, 128>>>(store, packed, scat, ident, c.rows, qpr);
                else
                    copy_rows<4><<<sms * ctas, 128>>>(packed, store, ident, c.scat_dst ? scat : ident, c.rows, qpr);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
            }
            const double bytes = 2.0 * c.rows * qpr * 16;
            printf("%s ctas/SM %d: %.1f us  %.0f GB/s\n", c.name, ctas, best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
