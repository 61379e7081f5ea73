// Probe: time twisting 105 MT19937-64 blocks (one C4-at-8-GPUs call) into a
// ring in global memory, one warp with the block in registers vs a 128-thread
// CTA with the block in shared memory.  nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -std=c++17 -I include -I paper_2604_08706_b200/csrc tools/probes/mt_twist.cu -o tools/probes/mt_twist
#include <cstdio>
#include "common.cuh"
using namespace rb;

__global__ void k_warp(uint64_t* ring, int nblk) {
    if (threadIdx.x >= 32) return;
    const int l = threadIdx.x;
    uint64_t w[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) w[k] = (l + 32 * k < MT_N) ? ring[l + 32 * k] : 0;
    for (int q = 1; q <= nblk; ++q) {
        mt_twist_warp(w);
        uint64_t* dst = ring + (size_t)q * MT_N;
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if (l + 32 * k < MT_N) dst[l + 32 * k] = w[k];
    }
}
__global__ void k_warp_nostore(uint64_t* ring, int nblk) {
    if (threadIdx.x >= 32) return;
    const int l = threadIdx.x;
    uint64_t w[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) w[k] = (l + 32 * k < MT_N) ? ring[l + 32 * k] : 0;
    for (int q = 1; q <= nblk; ++q) mt_twist_warp(w);
    uint64_t* dst = ring + (size_t)(nblk + 1) * MT_N;
#pragma unroll
    for (int k = 0; k < 10; ++k)
        if (l + 32 * k < MT_N) dst[l + 32 * k] = w[k];
}
__global__ void k_block(uint64_t* ring, int nblk) {
    __shared__ uint64_t mt[MT_N];
    for (int i = threadIdx.x; i < MT_N; i += blockDim.x) mt[i] = ring[i];
    __syncthreads();
    for (int q = 1; q <= nblk; ++q) {
        mt_twist_block(mt);
        uint64_t* dst = ring + (size_t)q * MT_N;
        for (int i = threadIdx.x; i < MT_N; i += blockDim.x) dst[i] = mt[i];
    }
}
int main() {
    const int nblk = 105;
    uint64_t* ring;
    cudaMalloc(&ring, (size_t)(nblk + 2) * MT_N * 8);
    cudaMemset(ring, 1, (size_t)(nblk + 2) * MT_N * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        float t[3];
        for (int v = 0; v < 3; ++v) {
            cudaEventRecord(a);
            if (v == 0) k_warp<<<1, 32>>>(ring, nblk);
            if (v == 1) k_warp_nostore<<<1, 32>>>(ring, nblk);
            if (v == 2) k_block<<<1, 128>>>(ring, nblk);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&t[v], a, b);
        }
        printf("105 blocks: warp+store %.2f us, warp no store %.2f us, block(128)+store %.2f us\n",
               t[0] * 1e3, t[1] * 1e3, t[2] * 1e3);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
