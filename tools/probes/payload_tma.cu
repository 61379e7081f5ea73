// Probe: payload-insert copy designs for the C4 pattern (1293 records x 2
// arrays x 16 KB, packed source -> slot rows), L2 flushed before each run.
//   lsu<U>      128-bit LDG/STG grid-stride copy, U quads in flight per thread
//   tma<W,S,CH> W warps per CTA, each warp's lane 0 an independent
//               cp.async.bulk pipeline of S shared-memory stages of CH bytes
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/payload_tma tools/probes/payload_tma.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__global__ void flush(const float4* p, size_t n, float* out) {
    float s = 0.f;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        s += p[i].x;
    if (s == 1234.5f) *out = s;
}

template <int U>
__global__ void lsu(const uint4* __restrict__ s0, const uint4* __restrict__ s1, uint4* d0, uint4* d1,
                    const int* drow, int nrec, int qpr) {
    const long long total = 2LL * nrec * qpr;
    for (long long b = (long long)blockIdx.x * blockDim.x * U; b < total;
         b += (long long)gridDim.x * blockDim.x * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = b + threadIdx.x + (long long)u * blockDim.x;
            if (i < total) {
                const long long ii = i % ((long long)nrec * qpr);
                const uint4* s = i < (long long)nrec * qpr ? s0 : s1;
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(s + ii));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = b + threadIdx.x + (long long)u * blockDim.x;
            if (i < total) {
                const long long ii = i % ((long long)nrec * qpr);
                const int r = (int)(ii / qpr), q = (int)(ii % qpr);
                uint4* d = i < (long long)nrec * qpr ? d0 : d1;
                asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(d + (size_t)drow[r] * qpr + q),
                             "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                             : "memory");
            }
        }
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int W, int S, int CH, int L>
__global__ void __launch_bounds__(32 * W) tma(const char* s0, const char* s1, char* d0, char* d1,
                                              const int* drow, int nrec, int row_bytes) {
    extern __shared__ __align__(128) char sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane) return;
    char* stg = sm + (size_t)w * S * CH;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)W * S * CH) + w * S;
    for (int s = 0; s < S; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int cpr = row_bytes / CH;             // chunks per row
    const long long items = 2LL * nrec * cpr;   // (array, record, chunk)
    const long long P = (long long)gridDim.x * W, p = (long long)blockIdx.x * W + w;
    const long long mine = p < items ? (items - 1 - p) / P + 1 : 0;
    auto addr = [&](long long k, const char** src, char** dst) {
        const long long it = p + k * P;
        const int a = (int)(it / ((long long)nrec * cpr));
        const long long rc = it % ((long long)nrec * cpr);
        const int r = (int)(rc / cpr), c = (int)(rc % cpr);
        *src = (a ? s1 : s0) + (size_t)r * row_bytes + (size_t)c * CH;
        *dst = (a ? d1 : d0) + (size_t)drow[r] * row_bytes + (size_t)c * CH;
    };
    for (long long k = 0; k < mine + L; ++k) {
        if (k < mine) {  // load item k into stage k % S (its previous store has read it)
            const int st = (int)(k % S);
            if (k >= S) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - L - 1) : "memory");
            const char* src;
            char* dst;
            addr(k, &src, &dst);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])),
                         "r"(CH)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(stg + (size_t)st * CH)),
                "l"(src), "r"(CH), "r"(smem_u32(&bar[st]))
                : "memory");
        }
        const long long j = k - L;
        if (j >= 0) {  // store item j
            const int st = (int)(j % S);
            const uint32_t par = (uint32_t)((j / S) & 1);
            asm volatile(
                "{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                    smem_u32(&bar[st])),
                "r"(par)
                : "memory");
            const char* src;
            char* dst;
            addr(j, &src, &dst);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                         "r"(smem_u32(stg + (size_t)st * CH)), "r"(CH)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const int nrec = argc > 1 ? atoi(argv[1]) : 1293, row_bytes = 16384, qpr = row_bytes / 16;
    const int store_rows = 16384 > nrec ? 16384 : nrec;
    char *s0, *s1, *d0, *d1;
    cudaMalloc(&s0, (size_t)nrec * row_bytes);
    cudaMalloc(&s1, (size_t)nrec * row_bytes);
    cudaMalloc(&d0, (size_t)store_rows * row_bytes);
    cudaMalloc(&d1, (size_t)store_rows * row_bytes);
    cudaMemset(s0, 1, (size_t)nrec * row_bytes);
    cudaMemset(s1, 2, (size_t)nrec * row_bytes);
    float4* fl;
    cudaMalloc(&fl, 512u << 20);
    cudaMemset(fl, 0, 512u << 20);
    float* fo;
    cudaMalloc(&fo, 4);
    std::vector<int> h(nrec);
    for (int i = 0; i < nrec; ++i) h[i] = (9000 + i) % store_rows;  // ring slots
    int* drow;
    cudaMalloc(&drow, nrec * 4);
    cudaMemcpy(drow, h.data(), nrec * 4, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 2.0 * 2 * nrec * (double)row_bytes;
    auto run = [&](const char* name, auto launch) {
        float best = 1e9, sum = 0;
        for (int rep = 0; rep < 7; ++rep) {
            flush<<<sms * 4, 256>>>(fl, (512u << 20) / 16, fo);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) sum += ms;
            best = std::min(best, ms);
        }
        printf("%-34s best %6.2f us (%5.0f GB/s)  mean %6.2f us  %s\n", name, best * 1e3,
               bytes / (best * 1e-3) / 1e9, sum / 6 * 1e3, cudaGetErrorString(cudaGetLastError()));
    };
#define TMA(W, S, CH, L, CPS)                                                                     \
    {                                                                                             \
        const size_t smem = (size_t)(W) * (S) * (CH) + (W) * (S) * 8;                             \
        cudaFuncSetAttribute(tma<W, S, CH, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        char nm[64];                                                                              \
        snprintf(nm, sizeof nm, "tma W%d S%d CH%d L%d x %d/SM", W, S, CH, L, CPS);                 \
        run(nm, [&] { tma<W, S, CH, L><<<sms * (CPS), 32 * (W), smem>>>(s0, s1, d0, d1, drow, nrec, row_bytes); }); \
    }
    for (int c : {8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "lsu<4> 128thr x %d/SM", c);
        run(nm, [&] { lsu<4><<<sms * c, 128>>>((uint4*)s0, (uint4*)s1, (uint4*)d0, (uint4*)d1, drow, nrec, qpr); });
    }
    TMA(2, 3, 16384, 1, 2)
    TMA(1, 4, 16384, 2, 3)
    TMA(4, 3, 8192, 1, 2)
    TMA(2, 4, 16384, 2, 1)
    TMA(1, 4, 16384, 2, 2)
    TMA(2, 2, 16384, 1, 2)
    TMA(1, 3, 16384, 1, 2)
    TMA(2, 3, 8192, 1, 2)
    TMA(4, 2, 8192, 1, 2)
    TMA(1, 2, 16384, 1, 3)
    TMA(1, 2, 16384, 1, 4)
    TMA(4, 2, 4096, 1, 4)
    TMA(2, 3, 4096, 1, 4)
    return 0;
}
