// Probe: does a programmatic-dependent launch chain A -> B -> C let C start
// while A still runs (B triggers at its start)?  Prints kernel start/end
// times (globaltimer, ns) for eager and graph launches.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_t[8];
__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ void spin_ns(unsigned long long ns) {
    const unsigned long long t0 = now();
    while (now() - t0 < ns) {}
}
template <int K>
__global__ void k(int trig, unsigned long long ns) {
    if (threadIdx.x == 0) atomicMin(&g_t[2 * K], now());
    if (trig) asm volatile("griddepcontrol.launch_dependents;");
    spin_ns(ns);
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&g_t[2 * K + 1], now());
}
template <class Kern>
void launch(Kern kern, int grid, int pdl, cudaStream_t s, int trig, unsigned long long ns) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl;
    cudaLaunchKernelEx(&cfg, kern, trig, ns);
}
void reset() {
    unsigned long long init[8];
    for (int i = 0; i < 8; ++i) init[i] = (i & 1) ? 0 : ~0ULL;
    cudaMemcpyToSymbol(g_t, init, sizeof init);
}
void show(const char* tag) {
    unsigned long long t[8];
    cudaMemcpyFromSymbol(t, g_t, sizeof t);
    printf("%-28s A [%6.2f %6.2f]  B [%6.2f %6.2f]  C [%6.2f %6.2f] us\n", tag, 0.0,
           (t[1] - t[0]) / 1e3, (t[2] - t[0]) / 1e3, (t[3] - t[0]) / 1e3, (t[4] - t[0]) / 1e3,
           (t[5] - t[0]) / 1e3);
}
int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (int mode = 0; mode < 4; ++mode) {
        // mode 0: eager chain; 1: graph chain; 2: graph chain with an event record between B and C;
        // 3: graph, B grid fills the GPU (888 CTAs)
        const int gridB = mode == 3 ? 888 : 16;
        for (int rep = 0; rep < 3; ++rep) {
            reset();
            cudaDeviceSynchronize();
            if (mode == 0) {
                launch(k<0>, 8, 0, s, 1, 20000);
                launch(k<1>, gridB, 1, s, 1, 20000);
                launch(k<2>, 4, 1, s, 0, 2000);
            } else {
                cudaGraph_t g;
                cudaGraphExec_t ge;
                cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
                launch(k<0>, 8, 0, s, 1, 20000);
                launch(k<1>, gridB, 1, s, 1, 20000);
                if (mode == 2) cudaEventRecord(ev, s);
                launch(k<2>, 4, 1, s, 0, 2000);
                cudaStreamEndCapture(s, &g);
                if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
                    printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
                    return 1;
                }
                cudaGraphLaunch(ge, s);
                cudaStreamSynchronize(s);
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(g);
            }
            cudaDeviceSynchronize();
            char tag[64];
            snprintf(tag, sizeof tag, "mode %d rep %d", mode, rep);
            show(tag);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
