/* replay_synth.h — the synthetic trajectory workload shared by the GPU
 * producer (bench.py / tests), the CPU oracle and the reference-arm driver.
 *
 * This is NOT part of the replay-step product: it stands in for the
 * inference workers (inbound trajectories) and for the trainer forward pass
 * (logp_now), so that CPU and GPU see bit-identical inputs.
 * fixes the shape of the workload; the concrete formulas are chosen here so
 * that every value is exactly reproducible on host and device (integer
 * hashing + exactly-representable fp32 arithmetic, no transcendental calls):
 *
 *   token id   = h mod 151936                         (Qwen vocab size)
 *   logp_old   = -8 * (k/4096)^2, k = 12 hash bits    (exact in fp32, in [-8,0])
 *   logp_now   = fl32(logp_old + 0.1732 * (u1+u2+u3+u4 - 2)), u_i 16-bit grid
 *                (Irwin–Hall(4), std ≈ 0.1; ratio in [0.707, 1.414] so both
 *                 GRPO clip branches are exercised)
 *   reward     = one hash bit (Bernoulli(0.5)); is_correct = (reward == 1)
 *   length     = fixed L, or U{1..Lmax} for the ragged configs
 *   behavior_logprob = sum_t logp_old — every term is a multiple of 2^-21
 *                with |.| <= 8, so the fp64 sum is exact in any order.
 */
#ifndef REPLAY_SYNTH_H
#define REPLAY_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define RS_HD __host__ __device__ __forceinline__
#else
#define RS_HD static inline
#endif

#define RS_VOCAB 151936u

/* splitmix64 finaliser (the same mixing constants as rng.cpp:17-23, used
 * here as a stateless counter hash). */
RS_HD uint64_t rs_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* Counter hash of (seed, rollout id, token position, purpose). */
RS_HD uint64_t rs_hash(uint64_t seed, uint64_t rollout_id, uint64_t t, uint64_t purpose) {
    return rs_mix64(seed ^ rs_mix64(rollout_id * 0x9E3779B97F4A7C15ULL ^
                                    (t * 0xC2B2AE3D27D4EB4FULL) ^ (purpose << 56)));
}

enum { RS_TOKEN = 1, RS_LOGP = 2, RS_NOW = 3, RS_REWARD = 4, RS_LEN = 5 };

RS_HD int32_t rs_token(uint64_t seed, uint64_t id, uint64_t t) {
    return (int32_t)(rs_hash(seed, id, t, RS_TOKEN) % RS_VOCAB);
}

RS_HD float rs_logp_old(uint64_t seed, uint64_t id, uint64_t t) {
    const uint32_t k = (uint32_t)(rs_hash(seed, id, t, RS_LOGP) >> 52); /* 12 bits */
    /* k*k < 2^24 is exact as a float; the scale by -8/2^24 is a power of two. */
    return (float)(k * k) * -4.76837158203125e-07f; /* -8 / 2^24 = -2^-21 */
}

/* logp_now for the synthetic trainer.  `version` lets a test move the policy. */
RS_HD float rs_logp_now(uint64_t seed, uint64_t id, uint64_t t, uint64_t version) {
    const uint64_t h = rs_hash(seed ^ (version * 0xD6E8FEB86659FD93ULL), id, t, RS_NOW);
    const uint32_t s = (uint32_t)(h & 0xffff) + (uint32_t)((h >> 16) & 0xffff) +
                       (uint32_t)((h >> 32) & 0xffff) + (uint32_t)(h >> 48);
    /* (s - 2*65536) is an exact integer below 2^18: exact in fp32. */
    const float centered = (float)((int32_t)s - 131072) * 1.52587890625e-05f; /* /65536 */
#if defined(__CUDA_ARCH__)
    return __fadd_rn(rs_logp_old(seed, id, t), __fmul_rn(centered, 0.1732f));
#else
    volatile float d = centered * 0.1732f; /* keep the host from contracting */
    return rs_logp_old(seed, id, t) + d;
#endif
}

RS_HD double rs_reward(uint64_t seed, uint64_t id) {
    return (rs_hash(seed, id, 0, RS_REWARD) >> 63) ? 1.0 : 0.0;
}

/* Length of trajectory `id`: fixed when ragged == 0, else U{1..lmax}. */
RS_HD int32_t rs_length(uint64_t seed, uint64_t id, int32_t lmax, int ragged) {
    if (!ragged) return lmax;
    return (int32_t)(rs_hash(seed, id, 0, RS_LEN) % (uint64_t)lmax) + 1;
}

#endif /* REPLAY_SYNTH_H */
