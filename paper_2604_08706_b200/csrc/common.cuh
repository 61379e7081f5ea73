// common.cuh — internals shared by the libreplay_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "replay_b200.h"

namespace rb {

// ---- error plumbing: C++ exceptions inside, status codes at the ABI -----
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string& msg);

#define RB_CUDA(expr)                                                                  \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess)                                                         \
            throw ::rb::Error(RB_ECUDA, std::string("CUDA error: ") +                  \
                                            cudaGetErrorString(_e) + " at " #expr);    \
    } while (0)

[[noreturn]] inline void invalid(const std::string& m) { throw Error(RB_EINVAL, m); }

template <class F>
int guard(F&& f) {
    try {
        f();
        return RB_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of memory");
        return RB_ENOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return RB_ELOGIC;
    }
}

// Fails loudly when no sm_100 device is usable (there is no CPU fallback).
void require_device();

// Pointer classification: true if `p` is device memory / page-locked host memory.
bool is_device_ptr(const void* p);
bool is_pinned_ptr(const void* p);
// Packed device arrays are accessed with 16-byte vector loads / stores and
// bulk copies: a misaligned device pointer (e.g. a torch slice x[1:]) is an
// RB_EINVAL, not a misaligned-address fault that poisons the context.
inline void require_aligned16(const void* p, const char* what) {
    if (p && ((uintptr_t)p & 15) != 0 && is_device_ptr(p))
        throw Error(RB_EINVAL, std::string(what) + ": device array must be 16-byte aligned");
}

// ---- MT19937-64 (rng.hpp:68, std::mt19937_64 per [rand.predef]) --------
constexpr int MT_N = 312;
constexpr int MT_M = 156;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ULL;
constexpr uint64_t MT_LM = 0x000000007FFFFFFFULL;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;

struct MtState {  // identical layout on host and device
    uint64_t mt[MT_N];
    uint32_t idx;
    uint32_t pad;
    uint64_t draws;
};

__host__ __device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
__host__ __device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b) {
    const uint64_t x = (a & MT_UM) | (b & MT_LM);
    return (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
}
// Sequential twist (one thread; used by the scalar device paths and the host).
__host__ __device__ inline void mt_twist_scalar(uint64_t* mt) {
    for (int i = 0; i < MT_N; ++i) {
        const int i1 = (i + 1 == MT_N) ? 0 : i + 1;
        const int im = (i + MT_M >= MT_N) ? i + MT_M - MT_N : i + MT_M;
        mt[i] = mt[im] ^ mt_mix(mt[i], mt[i1]);
    }
}
__host__ __device__ inline uint64_t mt_next_scalar(uint64_t* mt, uint32_t* idx,
                                                   uint64_t* draws) {
    if (*idx >= MT_N) {
        mt_twist_scalar(mt);
        *idx = 0;
    }
    ++*draws;
    return mt_temper(mt[(*idx)++]);
}
// Device home of a stream: a ring of twisted MT blocks.  Block q is the
// state after q twists of the ring's base state (block 0); the current state
// is (block q_state, idx) and blocks (q_state, q_hi] are twisted AHEAD by a
// generator kernel off the sampler's critical path, so a sampler only tempers
// words it reads.  Word o (o >= 0) after the current position is word
// (idx + o) % MT_N of block q_state + (idx + o) / MT_N.  Any consumer that
// twists itself produces the same blocks (the stream is deterministic).
constexpr int MT_KR = 256;  // ring capacity in blocks (79872 outputs: a call of up to ~38k draws is twisted ahead by the previous one)
struct MtRing {
    long long q_state;  // block of the current state
    long long q_hi;     // last block held; [q_state, q_hi] are resident
    uint32_t idx;       // next word of block q_state (MT_N: block exhausted)
    uint32_t pad;
    uint64_t draws;     // outputs consumed since seeding (parity aid)
    long long gen_q;    // generator progress within a fused sampler (<= q_hi otherwise)
    uint64_t blk[MT_KR][MT_N];
};
struct MtRingHead {  // the first bytes of MtRing (host-side header copies)
    long long q_state, q_hi;
    uint32_t idx, pad;
    uint64_t draws;
    long long gen_q;
};
static_assert(sizeof(MtRingHead) == 40, "MtRing header layout");
// Advance (q, idx) past d outputs, keeping idx in [1, MT_N] once moved.
__host__ __device__ __forceinline__ void ring_advance(long long& q, uint32_t& idx,
                                                     unsigned long long d) {
    if (d == 0) return;
    const unsigned long long o = (unsigned long long)idx + d;
    q += (long long)((o - 1) / MT_N);
    idx = (uint32_t)((o - 1) % MT_N + 1);
}

// rng.cpp:44: values >= limit are rejected.
__host__ __device__ __forceinline__ uint64_t below_limit(uint64_t bound) {
    return UINT64_MAX - UINT64_MAX % bound;
}

// Block-cooperative twist of a shared-memory MT state in three dependency
// phases (i < 156 reads only old words; 156 <= i < 311 reads new words
// i-156; i = 311 reads new word 0).  Any blockDim.x >= 52 (each thread
// computes up to three words per phase into registers); every thread of the
// block must call it.
__device__ __forceinline__ void mt_twist_block(uint64_t* mt) {
    // new[i] = old[i+156] ^ mix(old[i], old[i+1])            i in [0, 156)
    // new[j] = new[j-156] ^ mix(old[j], old[j+1])            j in [156, 311)
    // new[311] = new[155] ^ mix(old[311], new[0])
    // Thread t owns i = t + r*nt and j = i + 156, so new[j-156] is its own
    // register: every old word is read before any write (one barrier), the
    // words are written, and thread 0 finishes word 311 (one more barrier).
    const int t = threadIdx.x, nt = blockDim.x;
    uint64_t a[3], b[3], old311 = 0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int i = t + r * nt;
        if (i < 156) {
            a[r] = mt[i + 156] ^ mt_mix(mt[i], mt[i + 1]);
            if (i + 156 < 311) b[r] = a[r] ^ mt_mix(mt[i + 156], mt[i + 157]);
        }
    }
    if (t == 0) old311 = mt[311];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const int i = t + r * nt;
        if (i < 156) {
            mt[i] = a[r];
            if (i + 156 < 311) mt[i + 156] = b[r];
        }
    }
    __syncthreads();
    if (t == 0) mt[311] = mt[155] ^ mt_mix(old311, mt[0]);
    __syncthreads();
}

// One warp, block held in registers: lane l holds word l + 32k in w[k]
// (k < 10; slot 9 exists for lanes < 24).  Twists w in place with shuffles
// only (no shared memory, no barriers): the ring generator's serial chain.
//   new[i] = old[i+156] ^ mix(old[i], old[i+1])     i < 156
//   new[j] = new[j-156] ^ mix(old[j], old[j+1])     156 <= j < 311
//   new[311] = new[155] ^ mix(old[311], new[0])
__device__ __forceinline__ void mt_twist_warp(uint64_t (&w)[10]) {
    const int l = threadIdx.x & 31;
    const unsigned F = 0xffffffffu;
    uint64_t nw[10];
    // old[i+1] for every slot (lane 31 takes lane 0 of the next slot)
    uint64_t o1[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) {
        const uint64_t dn = __shfl_down_sync(F, w[k], 1);
        const uint64_t nx = __shfl_sync(F, w[k < 9 ? k + 1 : 9], 0);
        o1[k] = l == 31 ? nx : dn;
    }
    // phase 1: slots 0..4 (index < 156: every lane of slots 0..3, lanes < 28 of slot 4);
    // old[i+156] = lane (l+28)&31, slot k+4 (source lane >= 28) or k+5
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const uint64_t src = l >= 28 ? w[k + 4] : w[k + 5 < 10 ? k + 5 : 9];
        const uint64_t o156 = __shfl_sync(F, src, (l + 28) & 31);
        nw[k] = o156 ^ mt_mix(w[k], o1[k]);
    }
    // phase 2: slots 4..9 (156 <= j < 311); new[j-156] = lane (l+4)&31,
    // slot k-5 (source lane >= 4) or k-4 (source lane < 4)
#pragma unroll
    for (int k = 4; k < 10; ++k) {
        const uint64_t src = l < 4 ? nw[k - 4] : nw[k - 5 >= 0 ? k - 5 : 0];
        const uint64_t n156 = __shfl_sync(F, src, (l + 4) & 31);
        const int j = l + 32 * k;
        if (j >= 156 && j < 311) nw[k] = n156 ^ mt_mix(w[k], o1[k]);
    }
    // word 311 (lane 23, slot 9): new[155] (lane 27, slot 4), new[0] (lane 0, slot 0)
    const uint64_t n155 = __shfl_sync(F, nw[4], 27);
    const uint64_t n0 = __shfl_sync(F, nw[0], 0);
    if (l == 23) nw[9] = n155 ^ mt_mix(w[9], n0);
#pragma unroll
    for (int k = 0; k < 10; ++k) w[k] = nw[k];
}

// Block-wide: twist ring blocks (qhi, target] from block qhi (shared scratch
// `mt`, blockDim.x >= 52; every thread calls with the same arguments).
// The caller guarantees target - q_state < MT_KR.
__device__ __forceinline__ void ring_extend(MtRing* r, uint64_t* mt, long long qhi,
                                            long long target) {
    if (qhi >= target) return;
    const uint64_t* src = r->blk[qhi % MT_KR];
    for (int i = threadIdx.x; i < MT_N; i += blockDim.x) mt[i] = src[i];
    __syncthreads();
    for (long long q = qhi + 1; q <= target; ++q) {
        mt_twist_block(mt);
        uint64_t* dst = r->blk[q % MT_KR];
        for (int i = threadIdx.x; i < MT_N; i += blockDim.x) dst[i] = mt[i];
    }
    __syncthreads();
}
// Block-wide: copy the current state's block into shared `mt`.
__device__ __forceinline__ void ring_load_block(const MtRing* r, long long q, uint64_t* mt) {
    const uint64_t* src = r->blk[q % MT_KR];
    for (int i = threadIdx.x; i < MT_N; i += blockDim.x) mt[i] = src[i];
    __syncthreads();
}
// Block-wide: a consumer that advanced a shared copy `mt` of block q0 by
// `tw` twists to index idx publishes the new state (block q0 + tw).
__device__ __forceinline__ void ring_store_state(MtRing* r, const uint64_t* mt, long long q0,
                                                 long long tw, uint32_t idx, uint64_t draws) {
    const long long q = q0 + tw, qhi = r->q_hi;
    __syncthreads();
    if (q > qhi) {
        uint64_t* dst = r->blk[q % MT_KR];
        for (int i = threadIdx.x; i < MT_N; i += blockDim.x) dst[i] = mt[i];
    }
    if (threadIdx.x == 0) {
        r->q_state = q;
        r->q_hi = q > qhi ? q : qhi;
        r->idx = idx;
        r->draws = draws;
    }
    __syncthreads();
}

// ---- small device helpers ----------------------------------------------
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long x) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long x;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ void st_release_i32(int* p, int x) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ int ld_acquire_i32(const int* p) {
    int x;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    return x;
}
// Done counters of the multi-CTA kernels: one acq_rel atomic by thread 0
// after a CTA barrier publishes the CTA's writes (release, cumulative over
// the barrier) and, for the last CTA, acquires everyone else's — instead of
// a sequentially consistent __threadfence() plus a relaxed atomic.
__device__ __forceinline__ unsigned done_add_u32(unsigned* p) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long done_add_u64(unsigned long long* p) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(p) : "memory");
    return old;
}

// Bounded spins on a flag published by a kernel that runs concurrently
// (programmatic dependent launch): a producer that never publishes is a bug,
// so after ~4 s the waiting kernel traps (a sticky launch error) instead of
// hanging the device.
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
static __device__ __noinline__ int spin_while_eq(const int* f, int v) {
    int x = ld_acquire_i32(f);
    if (x != v) return x;
    const unsigned long long t0 = gtimer_ns();
    while ((x = ld_acquire_i32(f)) == v) {
        __nanosleep(64);
        if (gtimer_ns() - t0 > 4000000000ULL) __trap();
    }
    return x;
}

// Epoch-tagged flags of an insert (verdict, route done, copy done):
// value = epoch << 2 | state.  A waiter knows the epoch it waits for, so a
// flag left by an earlier insert is simply "not yet": nothing is reset (no
// reset store has to become visible before a dependent launches).
// Returns the state once the flag carries `epoch`; bounded like spin_while_eq.
constexpr int RB_EPOCH_MASK = (1 << 29) - 1;
static __device__ __noinline__ int spin_epoch(const int* f, int epoch) {
    int x = ld_acquire_i32(f);
    if ((x >> 2) == epoch) return x & 3;
    const unsigned long long t0 = gtimer_ns();
    while (((x = ld_acquire_i32(f)) >> 2) != epoch) {
        __nanosleep(64);
        if (gtimer_ns() - t0 > 4000000000ULL) __trap();
    }
    return x & 3;
}

// Writes made before a programmatic trigger, performed before it executes.
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

static __device__ __noinline__ void spin_until_ge_u64(const unsigned long long* f,
                                                      unsigned long long v) {
    if (ld_acquire_u64(f) >= v) return;
    const unsigned long long t0 = gtimer_ns();
    while (ld_acquire_u64(f) < v) {
        __nanosleep(32);
        if (gtimer_ns() - t0 > 4000000000ULL) __trap();
    }
}

// Programmatic dependent launch: let the next kernel of the stream (launched
// with programmatic serialization) start while this one runs.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Waits until the grid this one programmatically depends on has completed and
// its writes are visible (returns at once without such a dependency).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Phase clocks for tuning the single-CTA kernels (debug builds only:
// -DRB_PHASE_CLOCKS; read back with rb_debug_phase_clocks).
#ifdef RB_PHASE_CLOCKS
static __device__ long long g_phase_clock[64];
// kernel timeline in global-timer ns: [64 + 2k] = first CTA start, [65 + 2k] = last CTA end
static __device__ unsigned long long g_timeline[64];
__device__ __forceinline__ unsigned long long rb_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RB_CLOCK(i)                                                  \
    do {                                                             \
        if (threadIdx.x == 0 && blockIdx.x == 0) g_phase_clock[i] = clock64(); \
    } while (0)
// globaltimer stamp of phase i by thread 0 when `cond` holds (one CTA)
#define RB_GCLOCK(i, cond)                                           \
    do {                                                             \
        if (threadIdx.x == 0 && (cond)) g_phase_clock[i] = (long long)rb_globaltimer(); \
    } while (0)
#define RB_TSTART(k)                                             \
    do {                                                         \
        if (threadIdx.x == 0) {                                  \
            const unsigned long long _t = rb_globaltimer();      \
            atomicMin(&g_timeline[2 * (k)], _t);                 \
            atomicMax(&g_timeline[32 + (k)], _t); /* latest CTA start */ \
        }                                                        \
    } while (0)
#define RB_TEND(k)                                                                 \
    do {                                                                           \
        __syncthreads();                                                           \
        if (threadIdx.x == 0) atomicMax(&g_timeline[2 * (k) + 1], rb_globaltimer()); \
    } while (0)
#else
#define RB_CLOCK(i) \
    do {            \
    } while (0)
#define RB_TSTART(k) \
    do {             \
    } while (0)
#define RB_GCLOCK(i, cond) \
    do {                   \
    } while (0)
#define RB_TEND(k) \
    do {           \
    } while (0)
#endif

// Device-side loss accumulator (one per buffer; reset by the sampler).
struct DevLossAcc {
    double obj_sum;
    unsigned long long included;
    unsigned long long excluded;
    unsigned long long done_blocks;
    long long total_tokens;  // normaliser used for the optimistic scale
    double objective;
    int need_fixup;
    int kind;      // loss that filled the accumulator: 0 GRPO, 1 AsymRE
    double* red3;  // registered reduce vector {objective_sum, included, excluded} (or NULL)
    unsigned claim;   // claimed work units of a dynamic loss launch (reset by its last CTA)
    unsigned fin_cnt; // CTAs of a finalize kernel past their reads of the accumulator
    double inv_b;    // AsymRE: 1 / B (objective = obj_sum * inv_b)
    double cur_div;  // GRPO: the divisor D baked into dlogp (dlogp = -g / D); 0 = total_tokens
};

}  // namespace rb
