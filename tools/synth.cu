// synth.cu — synthetic inference-worker / trainer stand-ins for tests and
// bench.py (NOT part of the replay-step product).  Generates on the GPU the
// exact workload of include/replay_synth.h so CPU checkers and GPU runs see
// bit-identical inputs.
#include <cuda_runtime.h>
#include <stdint.h>

#include "replay_synth.h"

namespace {

__global__ void k_payload(uint64_t seed, const uint64_t* ids, const int64_t* toff, long long n,
                          int32_t* tokens, float* logp_old) {
    const long long i = blockIdx.x;
    if (i >= n) return;
    const uint64_t id = ids[i];
    const long long o0 = toff[i], o1 = toff[i + 1];
    for (long long t = o0 + threadIdx.x; t < o1; t += blockDim.x) {
        const uint64_t tt = (uint64_t)(t - o0);
        if (tokens) tokens[t] = rs_token(seed, id, tt);
        if (logp_old) logp_old[t] = rs_logp_old(seed, id, tt);
    }
}

__global__ void k_meta(uint64_t seed, const uint64_t* ids, long long n, int32_t lmax, int ragged,
                       double* reward, int32_t* len, double* blp) {
    const long long i = blockIdx.x;
    if (i >= n) return;
    const uint64_t id = ids[i];
    const int32_t L = rs_length(seed, id, lmax, ragged);
    // every logp_old is a multiple of 2^-21 with |.| <= 8: the fp64 sum is
    // exact in any order, so this block reduction equals the sequential sum.
    double s = 0.0;
    for (int32_t t = threadIdx.x; t < L; t += blockDim.x) s += (double)rs_logp_old(seed, id, (uint64_t)t);
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        reward[i] = rs_reward(seed, id);
        len[i] = L;
        if (blp) blp[i] = red[0];
    }
}

__global__ void k_logp_now(uint64_t seed, uint64_t version, const uint64_t* ids,
                           const int64_t* off, long long n, float* out) {
    const long long i = blockIdx.x;
    if (i >= n) return;
    const uint64_t id = ids[i];
    const long long o0 = off[i], o1 = off[i + 1];
    for (long long t = o0 + threadIdx.x; t < o1; t += blockDim.x)
        out[t] = rs_logp_now(seed, id, (uint64_t)(t - o0), version);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int rs_fill_payload(uint64_t seed, const uint64_t* ids,
                                                           const int64_t* toff, long long n,
                                                           int32_t* tokens, float* logp_old,
                                                           void* stream) {
    if (n > 0) k_payload<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(seed, ids, toff, n, tokens, logp_old);
    return (int)cudaGetLastError();
}

__attribute__((visibility("default"))) int rs_fill_meta(uint64_t seed, const uint64_t* ids,
                                                        long long n, int32_t lmax, int ragged,
                                                        double* reward, int32_t* len, double* blp,
                                                        void* stream) {
    if (n > 0) k_meta<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(seed, ids, n, lmax, ragged, reward, len, blp);
    return (int)cudaGetLastError();
}

__attribute__((visibility("default"))) int rs_logp_now(uint64_t seed, uint64_t version,
                                                       const uint64_t* ids, const int64_t* off,
                                                       long long n, float* out, void* stream) {
    if (n > 0) k_logp_now<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(seed, version, ids, off, n, out);
    return (int)cudaGetLastError();
}

}  // extern "C"
