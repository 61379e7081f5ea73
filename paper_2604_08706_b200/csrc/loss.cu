// loss.cu — group advantages and the two policy-gradient losses.
//
//   rb_loss_grpo      grpo_loss_grad (bandit.cpp:363-408) per token of the
//                     current batch: logp_old read straight from the slot row
//                     (never packed), logp_now / dlogp packed; 20 B/token with
//                     the gather.
//   rb_loss_asymre    asymre_loss_grad (bandit.cpp:410-438) per token.
//   rb_group_advantages, rb_grpo_tokens, rb_grpo_records, rb_asymre_*:
//                     the same arithmetic over explicit arrays.
//
// Precision: the ratio is evaluated in fp32 (one ex2.approx) and the branch
// decided in fp32 unless the token sits within 4e-6 (relative) of a clip
// edge, has |logp_now - logp_old| >= RB_FAST_D (16) or is non-finite; those
// tokens are recomputed exactly as the reference does, in fp64 (exp, clamp,
// r*A <= c*A with ties to the unclipped branch, non-finite => excluded).  On
// the fast path the fp32 difference d (<= 0.5 ulp(16)), the product
// d*log2(e) (<= 0.5 ulp(23)) and ex2.approx (~2 ulp) bound the ratio's
// relative error by ~2e-6, inside the north star's 1e-5
// (tests/test_gpu_bench_shapes.py sweeps |d| up to 79 at 1e-5).  Objective
// terms accumulate in fp64 (per-thread unit sums included).  dlogp is
// written with the optimistic scale -1/total_tokens; if any token was
// excluded, the last CTA flags a rescale to -1/included.
#include <dlfcn.h>
#include <nccl.h>  // types and enums; the symbols are resolved at run time

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "buffer_internal.cuh"

using namespace rb;

namespace rb {

// |logp_now - logp_old| below which the fp32 fast path evaluates a token
#define RB_FAST_D 16.f

struct GrpoParams {
    float lo_f, hi_f;    // 1-eps_low, 1+eps_high (fp32)
    double lo, hi;       // same in fp64
};

struct GrpoPartial {
    double obj = 0.0;
    long long inc = 0, exc = 0;
};

// One token (bandit.cpp:380-400).  Returns the un-normalised coefficient.
__device__ __forceinline__ float grpo_token(float lpn, float lpo, double A, float Af,
                                            const GrpoParams& p, GrpoPartial& acc) {
    const float d = lpn - lpo;
    const float r = __expf(d);
    const bool edge = !(fabsf(d) < RB_FAST_D) || fabsf(r - p.hi_f) <= 4e-6f * p.hi_f ||
                      fabsf(r - p.lo_f) <= 4e-6f * p.lo_f;
    if (!edge) {
        ++acc.inc;
        bool unclipped;
        if (A > 0.0)
            unclipped = r <= p.hi_f;
        else if (A < 0.0)
            unclipped = r >= p.lo_f;
        else
            unclipped = true;
        if (unclipped) {
            acc.obj += (double)r * A;
            return Af * r;
        }
        acc.obj += (A > 0.0 ? p.hi : p.lo) * A;
        return 0.f;
    }
    const double rd = exp((double)lpn - (double)lpo);
    if (!isfinite(rd)) {  // bandit.cpp:381-386
        ++acc.exc;
        return 0.f;
    }
    ++acc.inc;
    const double c = rd < p.lo ? p.lo : (p.hi < rd ? p.hi : rd);  // std::clamp
    const double uv = __dmul_rn(rd, A), cv = __dmul_rn(c, A);
    if (uv <= cv) {  // ties -> unclipped (bandit.cpp:392)
        acc.obj += uv;
        return (float)(A * rd);
    }
    acc.obj += cv;
    return 0.f;
}

// e^d as one ex2.approx.ftz (results below 2^-126 flush to 0; __expf adds a
// denormal-range fix-up of four instructions per token).  Used only on the
// fast path, whose branch decisions are at least 4e-6 away from a clip edge.
__device__ __forceinline__ float exp_ftz(float d) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d * 1.4426950408889634f));
    return r;
}

__device__ __forceinline__ uint4 funnel4(const uint4& lo, const uint4& hi, int a) {
    switch (a & 3) {
        case 0: return lo;
        case 1: return make_uint4(lo.y, lo.z, lo.w, hi.x);
        case 2: return make_uint4(lo.z, lo.w, hi.x, hi.y);
        default: return make_uint4(lo.w, hi.x, hi.y, hi.z);
    }
}
__device__ __forceinline__ uint4 shfl_up_q(const uint4& q) {
    return make_uint4(__shfl_up_sync(0xffffffffu, q.x, 1), __shfl_up_sync(0xffffffffu, q.y, 1),
                      __shfl_up_sync(0xffffffffu, q.z, 1), __shfl_up_sync(0xffffffffu, q.w, 1));
}
__device__ __forceinline__ float qf(const uint4& q, int i) {
    return __uint_as_float(i == 0 ? q.x : i == 1 ? q.y : i == 2 ? q.z : q.w);
}

// Block reduction of the partials + one atomic per CTA + last-CTA finalize.
__device__ void grpo_block_commit(GrpoPartial p, DevLossAcc* acc) {
    __shared__ double s_obj[32];
    __shared__ long long s_inc[32], s_exc[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    p.obj = warp_sum_f64(p.obj);
    p.inc = warp_sum_i64(p.inc);
    p.exc = warp_sum_i64(p.exc);
    if (lane == 0) {
        s_obj[wid] = p.obj;
        s_inc[wid] = p.inc;
        s_exc[wid] = p.exc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double o = 0;
        long long i = 0, e = 0;
        for (int w = 0; w < nw; ++w) {
            o += s_obj[w];
            i += s_inc[w];
            e += s_exc[w];
        }
        atomicAdd(&acc->obj_sum, o);
        atomicAdd(&acc->included, (unsigned long long)i);
        atomicAdd(&acc->excluded, (unsigned long long)e);
        __threadfence();
        const unsigned long long t = atomicAdd(&acc->done_blocks, 1ULL);
        if (t == gridDim.x - 1) {  // last CTA: objective and rescale flag
            __threadfence();
            const unsigned long long inc = atomicAdd(&acc->included, 0ULL);
            const unsigned long long exc = atomicAdd(&acc->excluded, 0ULL);
            const double obj = atomicAdd(&acc->obj_sum, 0.0);
            acc->objective = inc ? obj / (double)inc : 0.0;
            acc->need_fixup = exc > 0 && inc > 0;
        }
    }
}

// Per-CTA loss partial of the persistent kernels (32 B).
struct Partial {
    double obj;
    long long inc, exc, pad;
};

// d[0, n) *= f by threads [tid, tid + nthr) of a grid or a CTA: 16-byte
// accesses, 4 in flight per thread (a one-float-per-iteration loop is
// latency-bound: 200 µs for 16.7 M floats over 148 CTAs).  d is 16-B aligned
// (require_aligned16 on every dlogp the library writes).
__device__ __forceinline__ void scale_f32(float* d, long long n, float f, long long tid,
                                          long long nthr) {
    float4* d4 = reinterpret_cast<float4*>(d);
    const long long n4 = n >> 2;
    long long i = tid;
    for (; i + 3 * nthr < n4; i += 4 * nthr) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = d4[i + k * nthr];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k].x *= f;
            v[k].y *= f;
            v[k].z *= f;
            v[k].w *= f;
            d4[i + k * nthr] = v[k];
        }
    }
    for (; i < n4; i += nthr) {
        float4 v = d4[i];
        v.x *= f;
        v.y *= f;
        v.z *= f;
        v.w *= f;
        d4[i] = v;
    }
    for (long long t = 4 * n4 + tid; t < n; t += nthr) d[t] *= f;
}

// Block-reduce the thread partials into parts[blockIdx.x]; the last CTA to
// finish (one ticket atomic per CTA) folds all partials in a fixed order
// (bitwise-reproducible objective), writes the accumulator and the optional
// device stats, and — single-process buffers only — applies the rare
// -1/total -> -1/included correction itself when a token was excluded.
__device__ void loss_commit(GrpoPartial p, Partial* parts, DevLossAcc* acc,
                            rb_loss_stats* stats, int asym, double inv_b, float* dlogp,
                            const long long* n_local, int local_fix, int part_base, int nparts,
                            double opt_div = 0.0) {
    __shared__ double s_obj[32];
    __shared__ long long s_inc[32], s_exc[32];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    p.obj = warp_sum_f64(p.obj);
    p.inc = warp_sum_i64(p.inc);
    p.exc = warp_sum_i64(p.exc);
    if (lane == 0) {
        s_obj[wid] = p.obj;
        s_inc[wid] = p.inc;
        s_exc[wid] = p.exc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial q{0.0, 0, 0, 0};
        for (int w = 0; w < nw; ++w) {
            q.obj += s_obj[w];
            q.inc += s_inc[w];
            q.exc += s_exc[w];
        }
        parts[part_base + blockIdx.x] = q;
        s_last = done_add_u64(&acc->done_blocks) == (unsigned long long)nparts - 1;
    }
    __syncthreads();
    if (!s_last) return;
    RB_GCLOCK(3, true);
    double o = 0.0;
    long long inc = 0, exc = 0;
    // FB partials per thread per round, all loads in flight together; the
    // order of the additions is fixed (bitwise-reproducible objective)
    // (16 in flight raised the whole kernel to 128 registers: 41 µs vs 37)
    constexpr int FB = 8;
    for (int base = threadIdx.x; base < nparts; base += FB * blockDim.x) {
        double ob[FB];
        long long ib[FB], eb[FB];
#pragma unroll
        for (int k = 0; k < FB; ++k) {
            const int i = base + k * blockDim.x;
            const bool ok = i < nparts;
            ob[k] = ok ? __ldcg(&parts[i].obj) : 0.0;
            ib[k] = ok ? __ldcg(&parts[i].inc) : 0;
            eb[k] = ok ? __ldcg(&parts[i].exc) : 0;
        }
#pragma unroll
        for (int k = 0; k < FB; ++k) {
            o += ob[k];
            inc += ib[k];
            exc += eb[k];
        }
    }
    o = warp_sum_f64(o);
    inc = warp_sum_i64(inc);
    exc = warp_sum_i64(exc);
    __syncthreads();
    if (lane == 0) {
        s_obj[wid] = o;
        s_inc[wid] = inc;
        s_exc[wid] = exc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        o = 0.0;
        inc = exc = 0;
        for (int w = 0; w < nw; ++w) {
            o += s_obj[w];
            inc += s_inc[w];
            exc += s_exc[w];
        }
        acc->obj_sum = o;
        acc->included = (unsigned long long)inc;
        acc->excluded = (unsigned long long)exc;
        if (double* r3 = acc->red3) {  // one-collective multi-GPU reduction
            r3[0] = o;
            r3[1] = (double)inc;
            r3[2] = (double)exc;
        }
        acc->objective = asym ? o * inv_b : (inc ? o / (double)inc : 0.0);
        acc->need_fixup = !asym && exc > 0 && inc > 0;
        acc->kind = asym;
        acc->inv_b = inv_b;
        // dlogp was written as -g / opt_div (the token mode: total_tokens; the
        // sequence modes: the selection count); the local fix below makes it -g / included
        const double od = opt_div > 0.0 ? opt_div : (double)acc->total_tokens;
        acc->cur_div = (acc->need_fixup && local_fix) ? (double)inc : od;
        acc->done_blocks = 0;
        acc->claim = 0;  // every CTA has made its last claim
        if (stats) {
            stats->objective_sum = o;
            stats->objective = acc->objective;
            stats->included = inc;
            stats->excluded = exc;
            stats->total_tokens = acc->total_tokens;
        }
        s_last = acc->need_fixup && local_fix;
        RB_GCLOCK(4, true);
    }
    __syncthreads();
    if (s_last) {  // rare: some ratio was non-finite
        const double od = opt_div > 0.0 ? opt_div : (double)acc->total_tokens;
        const float f = (float)(od / (double)acc->included);
        const long long n = *n_local;
        scale_f32(dlogp, n, f, threadIdx.x, blockDim.x);
    }
}

// Exact fp64 evaluation of one token, as the reference does (bandit.cpp:380-400).
__device__ __noinline__ float grpo_token_exact(float lpn, float lpo, double A,
                                               const GrpoParams& p, GrpoPartial& acc) {
    const double rd = exp((double)lpn - (double)lpo);
    if (!isfinite(rd)) {  // bandit.cpp:381-386
        ++acc.exc;
        return 0.f;
    }
    ++acc.inc;
    const double c = rd < p.lo ? p.lo : (p.hi < rd ? p.hi : rd);  // std::clamp
    const double uv = __dmul_rn(rd, A), cv = __dmul_rn(c, A);
    if (uv <= cv) {  // ties -> unclipped (bandit.cpp:392)
        acc.obj += uv;
        return (float)(A * rd);
    }
    acc.obj += cv;
    return 0.f;
}

// GRPO over the current batch: persistent over nloc * ceil(max_nq/(128*U))
// virtual units.  Per token 12 B of compulsory traffic: logp_old (slot row,
// funnel-shifted to the packed alignment) and logp_now (packed) in, dlogp out.
// Fast path per token: one ex2, the branch as two threshold compares chosen
// per unit from sign(A), and an fp32 per-unit objective sum; tokens near a
// clip edge or with |d| >= 80 / non-finite take grpo_token_exact.
//
// Unit order.  Selection-major (chunk c of selection b is unit b*ups + c)
// keeps a selection's chunks together (DRAM page locality: C4).  CM
// (chunk-major, unit c*nloc + b; long trajectories) deals every CTA of the
// static stride one chunk of each rank, so ragged batches — whose later
// chunks are mostly empty — leave no CTA with all the full units (it
// is the gather's order for long rows; for the loss it measured level with
// DYN, C3 24.6 vs 24.0 µs).  DYN (long rows, default): units claimed from a
// counter, the next claim in flight while the current unit runs.
// One work unit of the GRPO loss: QU destination quads of selection `un`
// (chunk c).  BOUNDED: the batch's last selection, whose last quad may end
// the caller's logp_now array — loaded word by word there (every other
// selection's last quad reads into the next selection's tokens, in bounds).
// The whole unit is instantiated twice so the hot path has no branch between
// its loads and their first use.
template <int U, bool BOUNDED>
__device__ __forceinline__ void grpo_unit(const BufView& v, const Unit& un, int c, int nq, int a,
                                          const float* lpn_packed, float* dlogp,
                                          const GrpoParams& prm, float scale, float tol_hi,
                                          float tol_lo, GrpoPartial& part, long long& inc_fast) {
    constexpr int QU = UNIT_THREADS * U;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nsq = (un.len + 3) >> 2;
    const long long P0 = un.off >> 2;
    const int kw = c * QU + wid * 32 * U;
    uint4 now[U], old[U];
#pragma unroll
    for (int s = 0; s < U; ++s) {
        const int k = kw + 32 * s + lane;
        now[s] = k < nq ? (BOUNDED ? ld_stream_lim(lpn_packed, P0 + k, un.off + un.len)
                                   : ld_stream(lpn_packed + 4 * (P0 + k)))
                        : make_uint4(0, 0, 0, 0);
    }
    row_to_packed_quads<U>(
        reinterpret_cast<const uint4*>(v.lpo + (size_t)un.row * v.stride), nsq, a, kw, old);
    const double A = un.adv;
    const float Af = (float)A;
    const float Afs = Af * scale;
    // Per unit the branch depends on one threshold only: A > 0 clips above
    // 1+eps_high (r near 1-eps_low is unclipped either way), A < 0 below
    // 1-eps_low, A = 0 never contributes.  Only tokens within tol of that
    // threshold, or with d >= 80 / NaN (fp32 overflow vs fp64), go exact.
    const int sgn = A > 0.0 ? 1 : (A < 0.0 ? -1 : 0);
    const float thr = sgn > 0 ? prm.hi_f : prm.lo_f;
    const float tol = sgn > 0 ? tol_hi : tol_lo;
    double fsum = 0.0;  // fp64: the objective matches the reference's fp64 sum
#pragma unroll
    for (int s = 0; s < U; ++s) {
        const int k = kw + 32 * s + lane;
        if (k < nq) {
            const int e0 = 4 * k - a;
            const bool full = e0 >= 0 && e0 + 3 < un.len;
            float o[4] = {0.f, 0.f, 0.f, 0.f};
            bool slow = !full;
            if (full) {
                float r[4];
                bool edge = false;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float d = qf(now[s], i) - qf(old[s], i);
                    r[i] = exp_ftz(d);
                    edge |= !(fabsf(d) < RB_FAST_D) || (sgn != 0 && fabsf(r[i] - thr) <= tol);
                }
                if (!edge) {
                    if (sgn > 0) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const bool unc = r[i] <= thr;
                            o[i] = unc ? Afs * r[i] : 0.f;
                            fsum += (double)(unc ? r[i] : thr);
                        }
                    } else if (sgn < 0) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const bool unc = r[i] >= thr;
                            o[i] = unc ? Afs * r[i] : 0.f;
                            fsum += (double)(unc ? r[i] : thr);
                        }
                    }
                    inc_fast += 4;
                } else {
                    slow = true;
                }
            }
            if (slow) {  // boundary quads and edge tokens: exact fp64, per token
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (e0 + i >= 0 && e0 + i < un.len)
                        o[i] = grpo_token_exact(qf(now[s], i), qf(old[s], i), A, prm, part) *
                               scale;
            }
            store_quad_masked(reinterpret_cast<uint32_t*>(dlogp), P0 + k,
                              make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]),
                                         __float_as_uint(o[2]), __float_as_uint(o[3])),
                              e0, un.len);
        }
    }
    part.obj += fsum * A;
}

template <int U, bool DYN, bool CM = false>
// (More CTAs per SM via a register cap spill and run slower: 44 µs at 10
// CTAs per SM vs 37 µs at 8.  The claimed-unit variant for ragged long rows
// is capped to 8 CTAs per SM (64 registers): C3 loss 24.4 vs 25.6 µs; the
// static-stride one to 7 (72 registers; uncapped it takes 96): C4 step 82.9
// vs 84.6 µs.)
#ifndef RB_LOSS_MINB
#define RB_LOSS_MINB 7
#endif
__global__ void __launch_bounds__(UNIT_THREADS, DYN ? 8 : RB_LOSS_MINB) k_loss_grpo_buf(
    BufView v, const Unit* units, const int* maxq_p, int nloc, const float* lpn_packed,
    float* dlogp, GrpoParams prm, DevLossAcc* acc, Partial* parts, rb_loss_stats* stats,
    const long long* n_local, int local_fix, int part_base, int nparts) {
    constexpr int QU = UNIT_THREADS * U;
    const float scale = -1.f / (float)acc->total_tokens;
    const float tol_hi = 4e-6f * prm.hi_f, tol_lo = 4e-6f * prm.lo_f;
    RB_TSTART(5);
    RB_GCLOCK(0, blockIdx.x == 0);
    pdl_trigger();  // the next step's route may start on its batch (it waits before the buffer)
    const int ups = (*maxq_p + QU - 1) / QU;
    const int nu = nloc * ups;
    GrpoPartial part;
    long long inc_fast = 0;
    __shared__ int s_claim[2];
    int u = blockIdx.x, p = 0;
    if (DYN) {
        if (threadIdx.x == 0) s_claim[0] = (int)atomicAdd(&acc->claim, 1u);
        __syncthreads();
        u = s_claim[0];
    }
    Unit nxt;  // static stride: descriptor of the next unit, loaded one unit ahead
    if (!DYN && u < nu) nxt = ld_unit(units + (CM ? u % nloc : u / ups));
    for (; u < nu;) {
        if (DYN && threadIdx.x == 0) s_claim[p ^ 1] = (int)atomicAdd(&acc->claim, 1u);
        const int b = CM ? u % nloc : u / ups;
        const int c = CM ? u / nloc : u - b * ups;
        const Unit un = DYN ? ld_unit(units + b) : nxt;
        const int un_next = DYN ? 0 : u + (int)gridDim.x;
        if (!DYN && un_next < nu) nxt = ld_unit(units + (CM ? un_next % nloc : un_next / ups));
        const int a = (int)(un.off & 3);
        const int nq = (a + un.len + 3) >> 2;
        if (c * QU < nq) {
            if (b == nloc - 1)
                grpo_unit<U, true>(v, un, c, nq, a, lpn_packed, dlogp, prm, scale, tol_hi, tol_lo,
                                   part, inc_fast);
            else
                grpo_unit<U, false>(v, un, c, nq, a, lpn_packed, dlogp, prm, scale, tol_hi, tol_lo,
                                    part, inc_fast);
        }
        if (DYN) {
            __syncthreads();
            u = s_claim[p ^ 1];
            p ^= 1;
        } else {
            u = un_next;
        }
    }
    part.inc += inc_fast;
    RB_GCLOCK(1, blockIdx.x == 0);
    RB_TEND(5);
    loss_commit(part, parts, acc, stats, 0, 0.0, dlogp, n_local, local_fix, part_base, nparts);
    RB_GCLOCK(2, blockIdx.x == 0);
}
#ifndef RB_LOSS_U
#define RB_LOSS_U 4
#endif
constexpr int LOSS_U = RB_LOSS_U;

template <int U>
__global__ void __launch_bounds__(UNIT_THREADS) k_loss_asymre_buf(
    BufView v, const Unit* units, const int* maxq_p, int nloc, const float* lpn_packed,
    float* dlogp, double delta_v, double inv_b, DevLossAcc* acc, Partial* parts,
    rb_loss_stats* stats, int part_base, int nparts);

// ---- GRPO normalisation modes 1 and 2 (oracle: or_loss_grpo_tokens_mode) ---
// One CTA per sequence (persistent over the batch's selections).
//   mode 1  per-sequence mean: n_i included tokens counted first (a token is
//           excluded iff exp(logp_now - logp_old) is not finite in fp64), then
//           every token's coefficient (same arithmetic as the token mode) is
//           written as -g_t / (n_i * S0) and the sequence contributes
//           mean_t(term_t) to the objective; included = sequences with n_i > 0.
//   mode 2  sequence ratio exp(sum_t logp_now_t - behavior_logprob) (PAPER.md
//           :1022-1025; bandit.cpp:375-406 with the record's logp = the sum):
//           one fp64 ratio / clip / tie decision per sequence; every token gets
//           -c_i / S0; included / excluded count sequences.
// S0 = the number of sequences of the (global) batch, the optimistic divisor;
// an exclusion that empties a sequence (mode 1) or excludes one (mode 2)
// rescales to -1/included afterwards like the token mode.
constexpr int SEQ_THREADS = 256;
__device__ __forceinline__ double block_sum_f64(double x) {
    __shared__ double s_r[32];
    __shared__ double s_tot;
    x = warp_sum_f64(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_r[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_r[w];
        s_tot = t;
    }
    __syncthreads();
    return s_tot;
}
__device__ __forceinline__ long long block_sum_i64(long long x) {
    __shared__ long long s_r[32];
    __shared__ long long s_tot;
    x = warp_sum_i64(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s_r[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_r[w];
        s_tot = t;
    }
    __syncthreads();
    return s_tot;
}
// bandit.cpp:381: a ratio is excluded iff exp(logp_now - logp_old) is not
// finite in fp64 (NaN, or d above ln(DBL_MAX) ~ 709.78).
__device__ __forceinline__ bool ratio_finite(float lpn, float lpo) {
    const double d = (double)lpn - (double)lpo;
    return d <= 709.0 || (d < 710.0 && isfinite(exp(d)));
}
// One sequence (block-wide).  lpn / lpo / dl are the sequence's first token;
// blp: the record's behavior_logprob, or NaN to use sum_t logp_old (mode 2).
template <int MODE>
__device__ __forceinline__ void seq_loss_cta(const float* lpn, const float* lpo, float* dl,
                                             int len, double A, double blp, double s0,
                                             const GrpoParams& prm, GrpoPartial& part) {
    const int tid = threadIdx.x;
    if (MODE == 2) {
        const bool own_blp = isnan(blp);
        double sn = 0.0, so = 0.0;
        for (int t = tid; t < len; t += blockDim.x) {
            sn += (double)lpn[t];
            if (own_blp) so += (double)lpo[t];
        }
        sn = block_sum_f64(sn);
        if (own_blp) so = block_sum_f64(so);
        __shared__ double s_c;
        if (tid == 0) {
            const double rd = exp(sn - (own_blp ? so : blp));  // bandit.cpp:380
            double c = 0.0;
            if (!isfinite(rd)) {  // 381-386
                ++part.exc;
            } else {
                ++part.inc;
                const double cl = rd < prm.lo ? prm.lo : (prm.hi < rd ? prm.hi : rd);
                const double uv = __dmul_rn(rd, A), cv = __dmul_rn(cl, A);
                if (uv <= cv) {  // ties -> unclipped (392)
                    part.obj += uv;
                    c = __dmul_rn(A, rd);
                } else {
                    part.obj += cv;
                }
            }
            s_c = c;
        }
        __syncthreads();
        const float g = (float)(-s_c / s0);
        for (int t = tid; t < len; t += blockDim.x) dl[t] = g;
        __syncthreads();  // s_c is reused by the next sequence
    } else {
        long long bad = 0;
        for (int t = tid; t < len; t += blockDim.x) bad += ratio_finite(lpn[t], lpo[t]) ? 0 : 1;
        bad = block_sum_i64(bad);
        const long long ni = (long long)len - bad;
        const float scale = ni > 0 ? (float)(-1.0 / ((double)ni * s0)) : 0.f;
        const float Af = (float)A;
        GrpoPartial tmp;  // this thread's terms of the sequence
        for (int t = tid; t < len; t += blockDim.x)
            dl[t] = ni > 0 ? grpo_token(lpn[t], lpo[t], A, Af, prm, tmp) * scale : 0.f;
        const double ssum = block_sum_f64(tmp.obj);
        if (tid == 0) {
            part.exc += bad;
            if (ni > 0) {
                ++part.inc;
                part.obj += ssum / (double)ni;
            }
        }
    }
}
// The buffer path: selection u's logp_old from its slot row, logp_now /
// dlogp packed at its offset, behavior_logprob from the record column.
template <int MODE>
__global__ void __launch_bounds__(SEQ_THREADS) k_loss_grpo_seq_buf(
    BufView v, const Unit* units, int nloc, const float* lpn, float* dlogp, GrpoParams prm,
    double s0, DevLossAcc* acc, Partial* parts, rb_loss_stats* stats, const long long* n_local,
    int local_fix, int part_base, int nparts) {
    GrpoPartial part;
    for (int u = blockIdx.x; u < nloc; u += gridDim.x) {
        const Unit un = ld_unit(units + u);
        if (un.len <= 0) continue;
        seq_loss_cta<MODE>(lpn + un.off, v.lpo + (size_t)un.row * v.stride, dlogp + un.off,
                           un.len, un.adv, MODE == 2 ? v.blp[un.g] : 0.0, s0, prm, part);
    }
    loss_commit(part, parts, acc, stats, 0, 0.0, dlogp, n_local, local_fix, part_base, nparts, s0);
}
// The stateless path over explicit packed arrays (one CTA per trajectory).
template <int MODE>
__global__ void __launch_bounds__(SEQ_THREADS) k_loss_grpo_seq_packed(
    const float* lpn, const float* lpo, const double* adv, const double* blp,
    const int64_t* offsets, float* dlogp, GrpoParams prm, double s0, DevLossAcc* acc) {
    const long long i = blockIdx.x;
    const long long o0 = offsets[i], o1 = offsets[i + 1];
    GrpoPartial part;
    seq_loss_cta<MODE>(lpn + o0, lpo + o0, dlogp + o0, (int)(o1 - o0), adv[i],
                       blp ? blp[i] : __longlong_as_double(0x7ff8000000000000LL), s0, prm, part);
    grpo_block_commit(part, acc);
}

int loss_grid(int sms) {
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_loss_grpo_buf<LOSS_U, false>, UNIT_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_loss_asymre_buf<LOSS_U>, UNIT_THREADS, 0);
    return sms * std::max(1, std::min(a, b));
}

// GRPO over explicit packed arrays (stateless API): CTA per trajectory.
__global__ void __launch_bounds__(256) k_loss_grpo_packed(const float* lpn, const float* lpo,
                                                          const double* adv,
                                                          const int64_t* offsets, float* dlogp,
                                                          GrpoParams prm, DevLossAcc* acc,
                                                          long long n_traj) {
    const long long i = blockIdx.x;
    const long long o0 = offsets[i], o1 = offsets[i + 1];
    const int len = (int)(o1 - o0);
    const double A = adv[i];
    const float Af = (float)A;
    const long long total = offsets[n_traj] - offsets[0];
    const float scale = total > 0 ? -1.f / (float)total : 0.f;
    const long long q0 = o0 >> 2, q1 = (o1 + 3) >> 2;
    GrpoPartial part;
    for (long long q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        const uint4 now = ld_stream_lim(lpn, q, o1);
        const uint4 old = ld_stream_lim(lpo, q, o1);
        float* dq = dlogp + 4 * q;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const long long t = 4 * q + e;
            if (t >= o0 && t < o1) dq[e] = grpo_token(qf(now, e), qf(old, e), A, Af, prm, part) * scale;
        }
    }
    (void)len;
    grpo_block_commit(part, acc);
}

__global__ void k_set_cur_div_included(DevLossAcc* acc) {
    if (acc->need_fixup) acc->cur_div = (double)acc->included;
}
__global__ void k_dlogp_rescale(float* d, long long n, const long long* n_dev,
                                const DevLossAcc* acc) {
    if (!acc->need_fixup) return;
    if (n_dev) n = *n_dev;
    const double cur = acc->cur_div > 0.0 ? acc->cur_div : (double)acc->total_tokens;
    const float f = (float)(cur / (double)acc->included);
    scale_f32(d, n, f, blockIdx.x * (long long)blockDim.x + threadIdx.x,
              (long long)gridDim.x * blockDim.x);
}

// AsymRE over the current batch: dlogp = -coef/B on every token.
// AsymRE over the current batch (persistent over the virtual units): 8 B/token,
// logp_now in, dlogp = -coef/B out; objective sum coef * sum_t logp_now.
template <int U>
__global__ void __launch_bounds__(UNIT_THREADS) k_loss_asymre_buf(
    BufView v, const Unit* units, const int* maxq_p, int nloc, const float* lpn_packed,
    float* dlogp, double delta_v, double inv_b, DevLossAcc* acc, Partial* parts,
    rb_loss_stats* stats, int part_base, int nparts) {
    constexpr int QU = UNIT_THREADS * U;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    pdl_trigger();  // the next step's route may start on its batch (it waits before the buffer)
    const int ups = (*maxq_p + QU - 1) / QU;
    const int nu = nloc * ups;
    GrpoPartial part;
    Unit nxt;  // descriptor of the next unit, loaded one unit ahead
    if ((int)blockIdx.x < nu) nxt = ld_unit(units + blockIdx.x / ups);
    for (int u = blockIdx.x; u < nu; u += gridDim.x) {
        const int b = u / ups, c = u - b * ups;
        const Unit un = nxt;
        if (u + (int)gridDim.x < nu) nxt = ld_unit(units + (u + (int)gridDim.x) / ups);
        const int a = (int)(un.off & 3);
        const int nq = (a + un.len + 3) >> 2;
        if (c * QU >= nq) continue;
        const long long P0 = un.off >> 2;
        const int kw = c * QU + wid * 32 * U;
        const double coef = v.reward[un.g] - (v.gmean[un.g] + delta_v);  // bandit.cpp:429
        const float gc = (float)(coef * -inv_b);
        const uint4 gq = make_uint4(__float_as_uint(gc), __float_as_uint(gc), __float_as_uint(gc),
                                    __float_as_uint(gc));
        uint4 now[U];
#pragma unroll
        for (int s = 0; s < U; ++s) {
            const int k = kw + 32 * s + lane;
            now[s] = k < nq ? ld_stream_lim(lpn_packed, P0 + k, un.off + un.len)
                            : make_uint4(0, 0, 0, 0);
        }
        double fs = 0.0;  // fp64 sum of logp_now (the reference's objective is fp64)
#pragma unroll
        for (int s = 0; s < U; ++s) {
            const int k = kw + 32 * s + lane;
            if (k < nq) {
                const int e0 = 4 * k - a;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (e0 + i >= 0 && e0 + i < un.len) fs += (double)qf(now[s], i);
                store_quad_masked(reinterpret_cast<uint32_t*>(dlogp), P0 + k, gq, e0, un.len);
            }
        }
        part.obj += coef * fs;
    }
    loss_commit(part, parts, acc, stats, 1, inv_b, dlogp, nullptr, 0, part_base, nparts);
}

__global__ void __launch_bounds__(256) k_loss_asymre_packed(const float* lpn, const double* reward,
                                                            const double* gmean,
                                                            const int64_t* offsets, float* dlogp,
                                                            double delta_v, double inv_b,
                                                            DevLossAcc* acc) {
    const long long i = blockIdx.x;
    const long long o0 = offsets[i], o1 = offsets[i + 1];
    const double coef = reward[i] - (gmean[i] + delta_v);
    const float gcoef = (float)(coef * -inv_b);
    double seq = 0.0;
    for (long long t = o0 + threadIdx.x; t < o1; t += blockDim.x) {
        seq += (double)lpn[t];
        dlogp[t] = gcoef;
    }
    GrpoPartial p;
    p.obj = coef * seq;
    grpo_block_commit(p, acc);
}

// Record-level fp64 forms (L = 1): the reference's arithmetic per record.
__global__ void k_grpo_records(const double* lpn, const double* blp, const double* adv,
                               long long n, double lo, double hi, double* coef_out,
                               DevLossAcc* acc) {
    GrpoPartial p;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double ratio = exp(lpn[i] - blp[i]);
        if (!isfinite(ratio)) {
            ++p.exc;
            coef_out[i] = 0.0;
            continue;
        }
        ++p.inc;
        const double A = adv[i];
        const double c = ratio < lo ? lo : (hi < ratio ? hi : ratio);
        const double uv = __dmul_rn(ratio, A), cv = __dmul_rn(c, A);
        if (uv <= cv) {
            p.obj += uv;
            coef_out[i] = __dmul_rn(A, ratio);
        } else {
            p.obj += cv;
            coef_out[i] = 0.0;
        }
    }
    grpo_block_commit(p, acc);
}
__global__ void k_scale_records(double* d, long long n, const DevLossAcc* acc) {
    const unsigned long long inc = acc->included;
    const double s = inc ? 1.0 / (double)inc : 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        d[i] = inc ? __dmul_rn(d[i], -s) : 0.0;
}
__global__ void k_asymre_records(const double* lpn, const double* reward, const double* gmean,
                                 long long n, double delta_v, double* d, DevLossAcc* acc) {
    GrpoPartial p;
    const double s = 1.0 / (double)n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double coef = reward[i] - (gmean[i] + delta_v);
        p.obj += __dmul_rn(coef, lpn[i]);
        d[i] = __dmul_rn(coef, -s);
    }
    grpo_block_commit(p, acc);
}

// group_advantages (bandit.cpp:276-294), segmented; bit-exact fp64.
__global__ void k_group_adv(const double* r, const int64_t* off, long long ng, double* adv,
                            double* mean_out, int* bad) {
    for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < ng;
         gi += (long long)gridDim.x * blockDim.x) {
        const long long b = off[gi], e = off[gi + 1], m = e - b;
        if (m < 2) {
            *bad = 1;
            continue;
        }
        const double dn = (double)m;
        double mean = 0.0;
        for (long long k = b; k < e; ++k) mean = __dadd_rn(mean, r[k]);
        mean = __ddiv_rn(mean, dn);
        double var = 0.0;
        for (long long k = b; k < e; ++k) {
            const double d = __dsub_rn(r[k], mean);
            var = __dadd_rn(var, __dmul_rn(d, d));
        }
        var = __ddiv_rn(var, dn);
        const double sd = __dsqrt_rn(var);
        for (long long k = b; k < e; ++k)
            adv[k] = sd < 1e-8 ? 0.0 : __ddiv_rn(__dsub_rn(r[k], mean), sd);
        if (mean_out) mean_out[gi] = mean;
    }
}

__global__ void k_acc_reset(DevLossAcc* acc, long long total) {
    acc->cur_div = 0.0;
    acc->obj_sum = 0.0;
    acc->included = 0;
    acc->excluded = 0;
    acc->done_blocks = 0;
    acc->total_tokens = total;
    acc->objective = 0.0;
    acc->need_fixup = 0;
}
__global__ void k_acc_set_total(DevLossAcc* acc, const long long* total_or_null, long long v) {
    acc->total_tokens = total_or_null ? *total_or_null : v;
    acc->obj_sum = 0.0;
    acc->included = 0;
    acc->excluded = 0;
    acc->done_blocks = 0;
    acc->objective = 0.0;
    acc->need_fixup = 0;
}
__global__ void k_stats_out(const DevLossAcc* acc, rb_loss_stats* out, int asym, double inv_b) {
    out->objective_sum = acc->obj_sum;
    out->objective = asym ? acc->obj_sum * inv_b : acc->objective;
    out->included = (long long)acc->included;
    out->excluded = (long long)acc->excluded;
    out->total_tokens = acc->total_tokens;
}

// ---- stateless context: stream + staging per process ---------------------
struct Ctx {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    DevLossAcc* acc = nullptr;
    rb_loss_stats* dstats = nullptr;
    int* dflag = nullptr;
    std::vector<void*> temps;
    Ctx() {}
    void init() {
        if (stream) return;
        require_device();
        RB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        RB_CUDA(cudaMalloc(&acc, sizeof(DevLossAcc)));
        RB_CUDA(cudaMemset(acc, 0, sizeof(DevLossAcc)));  // no reduce vector (red3 = NULL)
        RB_CUDA(cudaMalloc(&dstats, sizeof(rb_loss_stats)));
        RB_CUDA(cudaMalloc(&dflag, sizeof(int)));
    }
    // device view of a (possibly host) input array
    template <class T>
    const T* in(const T* p, size_t n) {
        if (!p || is_device_ptr(p)) return p;
        void* d;
        RB_CUDA(cudaMallocAsync(&d, std::max<size_t>(n, 1) * sizeof(T) + 16, stream));
        RB_CUDA(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, stream));
        temps.push_back(d);
        return (const T*)d;
    }
    template <class T>
    T* out(T* p, size_t n, std::vector<std::pair<void*, std::pair<void*, size_t>>>& back) {
        if (!p || is_device_ptr(p)) return p;
        void* d;
        RB_CUDA(cudaMallocAsync(&d, std::max<size_t>(n, 1) * sizeof(T) + 16, stream));
        temps.push_back(d);
        back.push_back({(void*)p, {d, n * sizeof(T)}});
        return (T*)d;
    }
    void finish(std::vector<std::pair<void*, std::pair<void*, size_t>>>& back) {
        for (auto& b : back)
            RB_CUDA(cudaMemcpyAsync(b.first, b.second.first, b.second.second,
                                    cudaMemcpyDeviceToHost, stream));
        for (void* t : temps) RB_CUDA(cudaFreeAsync(t, stream));
        temps.clear();
        RB_CUDA(cudaStreamSynchronize(stream));
    }
    void stats(rb_loss_stats* s, int asym, double inv_b,
               std::vector<std::pair<void*, std::pair<void*, size_t>>>& back) {
        if (!s) return;
        rb_loss_stats* d = is_device_ptr(s) ? s : dstats;
        k_stats_out<<<1, 1, 0, stream>>>(acc, d, asym, inv_b);
        RB_CUDA(cudaGetLastError());
        if (d != s) back.push_back({(void*)s, {(void*)d, sizeof(rb_loss_stats)}});
    }
};
Ctx& ctx() {
    static Ctx c;
    return c;
}

void copy_stats(rb_buffer* b, rb_loss_stats* stats, int asym, double inv_b) {
    if (!stats) return;
    const bool host = !is_device_ptr(stats);
    rb_loss_stats* d = host ? (rb_loss_stats*)b->scratch(sizeof(rb_loss_stats)) : stats;
    k_stats_out<<<1, 1, 0, b->stream>>>(b->acc, d, asym, inv_b);
    RB_CUDA(cudaGetLastError());
    if (host) {
        RB_CUDA(cudaMemcpyAsync(stats, d, sizeof *stats, cudaMemcpyDeviceToHost, b->stream));
        b->sync();
    }
}

// Host logp_now / dlogp for the buffer losses: staged through the buffer's
// ST_LOSS_IN / ST_LOSS_OUT device areas (H2D before, D2H after).
unsigned grid_for(long long n) {
    return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
}

// One loss evaluation over the current batch.
struct LossCall {
    int kind = 0;  // 0 GRPO, 1 AsymRE
    int mode = 0;  // GRPO normalisation: RB_GRPO_TOKEN_MEAN / SEQ_MEAN / SEQ_RATIO
    GrpoParams p{};
    double delta_v = 0.0, inv_b = 0.0;
    double s0 = 0.0;  // sequence modes: the optimistic divisor (sequences in the batch)
};

// Launch the loss kernel over owned selections [s0, s1) (part slots
// [part_base, part_base + grid) of `nparts` folded by the last CTA overall).
// CTAs for a launch over `nsel` selections: the resident grid, or fewer
// when the batch has fewer work units (small batches: fewer idle CTAs and
// fewer partials for the last CTA to fold).
int loss_grid_for(const rb_buffer* b, long long nsel);
// CTAs of the call's kernel over nsel selections (the sequence modes: one
// 256-thread CTA per selection, at most 8 resident per SM).
int call_grid(const rb_buffer* b, const LossCall& c, long long nsel) {
    if (c.kind == 0 && c.mode != RB_GRPO_TOKEN_MEAN)
        return (int)std::max<long long>(1, std::min<long long>(nsel, (long long)b->sms * 8));
    return loss_grid_for(b, nsel);
}
int loss_grid_for(const rb_buffer* b, long long nsel) {
    const long long qmax = ((long long)b->max_tokens + 3) / 4 + 1;  // quads per selection (bound)
    const long long ups = (qmax + UNIT_THREADS * LOSS_U - 1) / (UNIT_THREADS * LOSS_U);
    const long long units = std::max(1LL, nsel * ups);
    return (int)std::min<long long>(b->grid_loss, std::max<long long>(units, b->sms));
}

void launch_loss(rb_buffer* b, const LossCall& c, const float* lpn, float* dl, long long s0,
                 long long s1, int part_base, int nparts, rb_loss_stats* kst, int local_fix) {
    const Unit* u = b->units_sel + s0;
    const int grid = call_grid(b, c, s1 - s0);
    if (c.kind == 0 && c.mode != RB_GRPO_TOKEN_MEAN) {
        if (c.mode == RB_GRPO_SEQ_MEAN)
            k_loss_grpo_seq_buf<1><<<grid, SEQ_THREADS, 0, b->stream>>>(
                b->v, u, (int)(s1 - s0), lpn, dl, c.p, c.s0, b->acc, (Partial*)b->loss_partials,
                kst, b->sel_total, local_fix, part_base, nparts);
        else
            k_loss_grpo_seq_buf<2><<<grid, SEQ_THREADS, 0, b->stream>>>(
                b->v, u, (int)(s1 - s0), lpn, dl, c.p, c.s0, b->acc, (Partial*)b->loss_partials,
                kst, b->sel_total, local_fix, part_base, nparts);
        RB_CUDA(cudaGetLastError());
        return;
    }
    // claimed units for long (ragged-prone) trajectories in a one-launch loss
    const bool dyn = b->max_tokens > 2 * UNIT_THREADS * LOSS_U * 4 && part_base == 0 &&
                     nparts == grid;
    if (c.kind == 0 && dyn && b->loss_dyn)
        k_loss_grpo_buf<LOSS_U, true><<<grid, UNIT_THREADS, 0, b->stream>>>(
            b->v, u, b->n_units_sel, (int)(s1 - s0), lpn, dl, c.p, b->acc,
            (Partial*)b->loss_partials, kst, b->sel_total, local_fix, part_base, nparts);
    else if (c.kind == 0 && b->chunk_major && b->max_tokens > 2 * UNIT_THREADS * LOSS_U * 4)
        k_loss_grpo_buf<LOSS_U, false, true><<<grid, UNIT_THREADS, 0, b->stream>>>(
            b->v, u, b->n_units_sel, (int)(s1 - s0), lpn, dl, c.p, b->acc,
            (Partial*)b->loss_partials, kst, b->sel_total, local_fix, part_base, nparts);
    else if (c.kind == 0)
        k_loss_grpo_buf<LOSS_U, false><<<grid, UNIT_THREADS, 0, b->stream>>>(
            b->v, u, b->n_units_sel, (int)(s1 - s0), lpn, dl, c.p, b->acc,
            (Partial*)b->loss_partials, kst, b->sel_total, local_fix, part_base, nparts);
    else
        k_loss_asymre_buf<LOSS_U><<<grid, UNIT_THREADS, 0, b->stream>>>(
            b->v, u, b->n_units_sel, (int)(s1 - s0), lpn, dl, c.delta_v, c.inv_b, b->acc,
            (Partial*)b->loss_partials, kst, part_base, nparts);
    RB_CUDA(cudaGetLastError());
}

constexpr int LOSS_CHUNKS = 8;  // host-buffer pipeline depth (16 measured slower: per-copy setup)

// Device buffers: one launch.  Host buffers: the batch is cut into up to
// LOSS_CHUNKS selection ranges; per chunk the logp_now upload (copy stream
// 1), the loss kernel (buffer stream) and the dlogp download (copy stream 2)
// are chained by events, so upload and download overlap (PCIe is full
// duplex).  A token excluded anywhere (non-finite ratio, rare) rescales and
// re-downloads dlogp after the pipeline.
void run_loss(rb_buffer* b, const LossCall& c, const float* lpn, float* dl,
              rb_loss_stats* stats) {
    require_aligned16(lpn, "loss: logp_now");
    require_aligned16(dl, "loss: out_dlogp");
    b->other_work();
    b->join_lookahead();  // the step's ring lookahead rejoins the stream here (graph capture)
    const size_t per = b->T ? b->B / b->T : 0;
    const long long lo = (long long)std::min(b->sb * per, b->B);
    const long long hi = (long long)std::min(b->se * per, b->B);
    const long long nloc = hi - lo;
    const bool dev_stats = stats && is_device_ptr(stats);
    rb_loss_stats* kst = dev_stats ? stats : (stats ? (rb_loss_stats*)b->scratch(64) : nullptr);
    const bool host_in = lpn && !is_device_ptr(lpn);
    const bool host_out = dl && !is_device_ptr(dl);
    const bool single = b->sb == 0 && b->se == b->T;
    if (nloc <= 0) {
        if (kst) k_stats_out<<<1, 1, 0, b->stream>>>(b->acc, kst, c.kind, c.inv_b);
    } else if (!host_in && !host_out) {
        launch_loss(b, c, lpn, dl, 0, nloc, 0, call_grid(b, c, nloc), kst, single && c.kind == 0);
    } else {
        // packed offsets of the owned selections (and the total) on the host
        std::vector<long long> off(nloc + 1);
        b->fetch(off.data(), b->sel_off, (nloc + 1) * 8);
        const long long total = off[nloc];
        const size_t bytes = (((size_t)total + 3) & ~size_t(3)) * 4 + 16;
        b->wait_outputs_on(b->stream);  // the last async download still reads the staging output
        float* din = host_in ? (float*)b->dev_stage(bytes, rb_buffer::ST_LOSS_IN) : (float*)lpn;
        float* dout = host_out ? (float*)b->dev_stage(bytes, rb_buffer::ST_LOSS_OUT) : dl;
        const bool pin_in = !host_in || is_pinned_ptr(lpn);
        const bool pin_out = !host_out || is_pinned_ptr(dl);
        b->ensure_copy_streams();
        // chunk boundaries: ~equal token counts, at selection boundaries
        std::vector<long long> cut{0};
        for (int k = 1; k < LOSS_CHUNKS; ++k) {
            const long long want = total * k / LOSS_CHUNKS;
            const long long s = std::lower_bound(off.begin(), off.end(), want) - off.begin();
            if (s > cut.back() && s < nloc) cut.push_back(s);
        }
        cut.push_back(nloc);
        const int nch = (int)cut.size() - 1;
        std::vector<int> pbase(nch + 1, 0);  // partial slots of each chunk's launch
        for (int k = 0; k < nch; ++k) pbase[k + 1] = pbase[k] + call_grid(b, c, cut[k + 1] - cut[k]);
        const int nparts = pbase[nch];
        if ((size_t)nparts * 32 > b->loss_partials_bytes) b->grow_loss_partials((size_t)nparts * 32);
        const float* hin = lpn;
        if (host_in && !pin_in) {  // pageable: one staged copy (no overlap)
            void* hs = b->host_stage(total * 4 + 16);
            std::memcpy(hs, lpn, total * 4);
            hin = (const float*)hs;
        }
        RB_CUDA(cudaEventRecord(b->ev_io[0], b->stream));
        RB_CUDA(cudaStreamWaitEvent(b->cs_in, b->ev_io[0], 0));
        RB_CUDA(cudaStreamWaitEvent(b->cs_out, b->ev_io[0], 0));
        for (int k = 0; k < nch; ++k) {
            const long long t0 = off[cut[k]], t1 = off[cut[k + 1]];
            if (host_in) {
                RB_CUDA(cudaMemcpyAsync(din + t0, hin + t0, (t1 - t0) * 4, cudaMemcpyHostToDevice,
                                        b->cs_in));
                RB_CUDA(cudaEventRecord(b->ev_io[1 + 2 * k], b->cs_in));
                RB_CUDA(cudaStreamWaitEvent(b->stream, b->ev_io[1 + 2 * k], 0));
            }
            launch_loss(b, c, din, dout, cut[k], cut[k + 1], pbase[k], nparts, kst, 0);
            if (host_out && pin_out) {
                RB_CUDA(cudaEventRecord(b->ev_io[2 + 2 * k], b->stream));
                RB_CUDA(cudaStreamWaitEvent(b->cs_out, b->ev_io[2 + 2 * k], 0));
                RB_CUDA(cudaMemcpyAsync(dl + t0, dout + t0, (t1 - t0) * 4, cudaMemcpyDeviceToHost,
                                        b->cs_out));
            }
        }
        if (host_in && !pin_in) b->host_stage_issued_on(b->cs_in);
        const bool async_dl = b->async_out && host_out && pin_out;
        if (async_dl) {  // the download drains beside the caller's next call
            if (!b->out_done) RB_CUDA(cudaEventCreateWithFlags(&b->out_done, cudaEventDisableTiming));
            RB_CUDA(cudaEventRecord(b->out_done, b->cs_out));
            b->out_pending = true;
        } else {
            RB_CUDA(cudaStreamSynchronize(b->cs_out));
        }
        RB_CUDA(cudaStreamSynchronize(b->stream));
        DevLossAcc acc;
        b->fetch(&acc, b->acc, sizeof acc);
        const bool fix = c.kind == 0 && acc.need_fixup && single;
        if (fix) b->drain_outputs();  // the rescaled array is downloaded again below
        if (fix) {  // -1/total -> -1/included (rare: a non-finite ratio)
            k_dlogp_rescale<<<grid_for(total), 256, 0, b->stream>>>(dout, total, nullptr, b->acc);
            k_set_cur_div_included<<<1, 1, 0, b->stream>>>(b->acc);  // after every rescale CTA read it
            RB_CUDA(cudaGetLastError());
        }
        if (host_out && (!pin_out || fix)) {
            RB_CUDA(cudaMemcpyAsync(dl, dout, total * 4, cudaMemcpyDeviceToHost, b->stream));
            b->sync();
        }
    }
    if (stats && !dev_stats) {
        b->fetch(stats, kst, sizeof *stats);
        if (b->async_unchecked) b->sync_checked();
    }
}

}  // namespace rb

// ====================================================================== C ABI
extern "C" {

int rb_loss_grpo(rb_buffer* b, const float* logp_now, float* out_dlogp, double eps_low,
                 double eps_high, int64_t norm_tokens, rb_loss_stats* stats) {
    return rb_loss_grpo_ex(b, logp_now, out_dlogp, eps_low, eps_high, RB_GRPO_TOKEN_MEAN,
                           norm_tokens, stats);
}

int rb_loss_grpo_ex(rb_buffer* b, const float* logp_now, float* out_dlogp, double eps_low,
                    double eps_high, int mode, int64_t norm, rb_loss_stats* stats) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (mode < RB_GRPO_TOKEN_MEAN || mode > RB_GRPO_SEQ_RATIO)
            invalid("rb_loss_grpo_ex: unknown normalisation mode");
        if (mode != RB_GRPO_TOKEN_MEAN) {
            if (b->stride == 0) invalid("rb_loss_grpo: buffer holds no token payload");
            if (eps_low < 0.0 || eps_high < 0.0) invalid("loss spec: clip bounds must be >= 0");
            if (!std::isfinite(eps_low) || !std::isfinite(eps_high))
                invalid("loss spec: parameters must be finite");
            if (b->B == 0) invalid("loss gradient needs a non-empty batch");
            LossCall c;
            c.kind = 0;
            c.mode = mode;
            c.p.lo = 1.0 - eps_low;
            c.p.hi = 1.0 + eps_high;
            c.p.lo_f = (float)c.p.lo;
            c.p.hi_f = (float)c.p.hi;
            c.s0 = (double)(norm > 0 ? norm : (int64_t)b->B);
            if (b->acc_norm_explicit) {  // back to the batch's token count (stats)
                k_acc_set_total<<<1, 1, 0, b->stream>>>(b->acc, b->sel_total + 1, 0);
                RB_CUDA(cudaGetLastError());
            }
            b->last_loss = 0;
            b->acc_norm_explicit = false;
            run_loss(b, c, logp_now, out_dlogp, stats);
            return;
        }
        const int64_t norm_tokens = norm;
        if (b->stride == 0) invalid("rb_loss_grpo: buffer holds no token payload");
        if (eps_low < 0.0 || eps_high < 0.0) invalid("loss spec: clip bounds must be >= 0");
        if (!std::isfinite(eps_low) || !std::isfinite(eps_high))
            invalid("loss spec: parameters must be finite");
        if (b->B == 0) invalid("loss gradient needs a non-empty batch");
        LossCall c;
        c.kind = 0;
        c.p.lo = 1.0 - eps_low;
        c.p.hi = 1.0 + eps_high;
        c.p.lo_f = (float)c.p.lo;
        c.p.hi_f = (float)c.p.hi;
        if (norm_tokens > 0 || b->acc_norm_explicit) {
            // explicit normaliser (or back to the batch's token count after
            // one); the accumulator fields are rewritten by the last CTA, so a
            // repeated loss on the same batch needs no reset
            k_acc_set_total<<<1, 1, 0, b->stream>>>(b->acc, norm_tokens > 0 ? nullptr : b->sel_total + 1,
                                                    norm_tokens);
            RB_CUDA(cudaGetLastError());
        }
        b->last_loss = 0;
        b->acc_norm_explicit = norm_tokens > 0;
        run_loss(b, c, logp_now, out_dlogp, stats);
    });
}

int rb_loss_asymre(rb_buffer* b, const float* logp_now, float* out_dlogp, double delta_v,
                   int64_t norm_batch, rb_loss_stats* stats) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (!std::isfinite(delta_v)) invalid("loss spec: parameters must be finite");
        if (b->B == 0) invalid("loss gradient needs a non-empty batch");
        LossCall c;
        c.kind = 1;
        c.delta_v = delta_v;
        c.inv_b = 1.0 / (double)(norm_batch > 0 ? norm_batch : (int64_t)b->B);
        if (b->acc_norm_explicit) {
            k_acc_set_total<<<1, 1, 0, b->stream>>>(b->acc, b->sel_total + 1, 0);
            RB_CUDA(cudaGetLastError());
        }
        b->last_loss = 1;
        b->acc_norm_explicit = false;
        run_loss(b, c, logp_now, out_dlogp, stats);
    });
}

// After the all-reduce of the reduce vector: every CTA derives the global
// normalisation from it and rescales its slice of dlogp if a token was
// excluded anywhere (GRPO); CTA 0 updates the accumulator and the stats.
// The global GRPO normalisation: dlogp holds -g / acc->cur_div (the loss
// kernel's total_tokens, or the single-process fix's included count); the
// target is -g / inc (bandit.cpp:402-406).  Idempotent: a second finalize
// (or one after the local fix) finds cur_div == inc and leaves dlogp alone.
__device__ __forceinline__ bool finalize_scale(const DevLossAcc* acc, unsigned long long inc,
                                               float* f) {
    if (inc == 0) return false;  // every token excluded: dlogp is already all zeros
    const double cur = acc->cur_div > 0.0 ? acc->cur_div : (double)acc->total_tokens;
    if (cur == (double)inc) return false;
    *f = (float)(cur / (double)inc);
    return true;
}
// Barrier over the finalize grid's reads of acc (before CTA 0 rewrites it):
// every CTA reads cur_div first, then CTA 0 waits for the others.
__device__ __forceinline__ void finalize_publish_wait(unsigned* cnt) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = done_add_u32(cnt);
        if (blockIdx.x == 0) {
            const unsigned long long t0 = gtimer_ns();
            while (ld_acquire_i32((const int*)cnt) < (int)gridDim.x) {
                __nanosleep(32);
                if (gtimer_ns() - t0 > 4000000000ULL) __trap();
            }
        }
        (void)t;
    }
    __syncthreads();
}
__global__ void k_finalize_vec(DevLossAcc* acc, const double* v3, float* dlogp,
                               const long long* n_dev, rb_loss_stats* st, int grpo) {
    pdl_trigger();  // the next step's route may start on its batch (it waits before the buffer)
    const double obj = v3[0];
    const unsigned long long inc = (unsigned long long)v3[1], exc = (unsigned long long)v3[2];
    float f = 1.f;
    const bool fix = grpo && finalize_scale(acc, inc, &f);
    if (fix && dlogp) {
        scale_f32(dlogp, *n_dev, f, blockIdx.x * (long long)blockDim.x + threadIdx.x,
                  (long long)gridDim.x * blockDim.x);
    }
    finalize_publish_wait(&acc->fin_cnt);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        acc->fin_cnt = 0;
        acc->obj_sum = obj;
        acc->included = inc;
        acc->excluded = exc;
        acc->objective = grpo ? (inc ? obj / (double)inc : 0.0) : obj * acc->inv_b;
        if (grpo && inc) acc->cur_div = (double)inc;
        acc->need_fixup = 0;  // applied
        if (st) {
            st->objective_sum = obj;
            st->objective = acc->objective;
            st->included = (int64_t)inc;
            st->excluded = (int64_t)exc;
            st->total_tokens = acc->total_tokens;
        }
    }
}
__global__ void k_set_red3(DevLossAcc* acc, double* v) { acc->red3 = v; }

// rb_loss_finalize in one kernel (reduced rb_loss_stats in, stats out).
__global__ void k_finalize_stats(DevLossAcc* acc, rb_loss_stats* st, float* dlogp,
                                 const long long* n_dev, int grpo) {
    pdl_trigger();  // the next step's route may start on its batch (it waits before the buffer)
    const double obj = st->objective_sum;
    const long long inc = st->included, exc = st->excluded;
    float f = 1.f;
    if (grpo && dlogp && finalize_scale(acc, (unsigned long long)(inc > 0 ? inc : 0), &f)) {
        scale_f32(dlogp, *n_dev, f, blockIdx.x * (long long)blockDim.x + threadIdx.x,
                  (long long)gridDim.x * blockDim.x);
    }
    finalize_publish_wait(&acc->fin_cnt);  // every CTA has read st and acc before they are rewritten
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        acc->fin_cnt = 0;
        acc->obj_sum = obj;
        acc->included = (unsigned long long)inc;
        acc->excluded = (unsigned long long)exc;
        acc->objective = grpo ? (inc ? obj / (double)inc : 0.0) : obj * acc->inv_b;
        if (grpo && inc > 0) acc->cur_div = (double)inc;
        acc->need_fixup = 0;  // applied
        st->objective_sum = obj;
        st->objective = acc->objective;
        st->included = inc;
        st->excluded = exc;
        st->total_tokens = acc->total_tokens;
    }
}

int rb_loss_set_reduce_vector(rb_buffer* b, double* vec3) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (vec3 && !is_device_ptr(vec3)) invalid("rb_loss_set_reduce_vector: device memory required");
        b->other_work();
        k_set_red3<<<1, 1, 0, b->stream>>>(b->acc, vec3);
        RB_CUDA(cudaGetLastError());
        b->red3 = vec3;
    });
}

namespace {
// ncclAllReduce of the NCCL library already in the process (e.g. torch's
// bundled one, found by soname without loading a second copy), else of the
// system's libnccl.so.2.  Resolved at run time: a communicator is only valid
// with the library instance that created it, so the product never links one.
using NcclAllReduceFn = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                         ncclComm_t, cudaStream_t);
using NcclErrFn = const char* (*)(ncclResult_t);
struct NcclSyms {
    NcclAllReduceFn allreduce = nullptr;
    NcclErrFn errstr = nullptr;
};
const NcclSyms& nccl_syms() {
    static NcclSyms s;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        s.allreduce = (NcclAllReduceFn)dlsym(h, "ncclAllReduce");
        s.errstr = (NcclErrFn)dlsym(h, "ncclGetErrorString");
    });
    return s;
}
}  // namespace

int rb_allreduce_loss_stats(rb_buffer* b, void* nccl_comm, float* dlogp, rb_loss_stats* stats) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (!nccl_comm) invalid("rb_allreduce_loss_stats: NULL communicator");
        if (!b->red3)
            throw Error(RB_ELOGIC, "rb_allreduce_loss_stats: register a reduce vector first "
                                   "(rb_loss_set_reduce_vector)");
        const NcclSyms& nc = nccl_syms();
        if (!nc.allreduce) throw Error(RB_ECUDA, "rb_allreduce_loss_stats: libnccl.so.2 not found");
        b->other_work();
        // the 24-B {objective_sum, included, excluded} the loss fold wrote, in place
        const ncclResult_t r = nc.allreduce(b->red3, b->red3, 3, ncclFloat64, ncclSum,
                                            (ncclComm_t)nccl_comm, b->stream);
        if (r != ncclSuccess)
            throw Error(RB_ECUDA, std::string("ncclAllReduce: ") +
                                      (nc.errstr ? nc.errstr(r) : std::to_string((int)r)));
        const int st = rb_loss_finalize_vec(b, dlogp, b->red3, stats);
        if (st != RB_OK) throw Error(st, rb_last_error());
    });
}

// The north star's priority-mass all-reduce: this rank's per-shard masses
// (owned shards, zeros elsewhere) summed in place over the communicator, so
// every rank holds every shard's W_s (e.g. for importance weights w_i / W).
int rb_allreduce_priority_mass(rb_buffer* b, void* nccl_comm, uint64_t* masses) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);
        if (!nccl_comm) invalid("rb_allreduce_priority_mass: NULL communicator");
        if (!masses || !is_device_ptr(masses))
            invalid("rb_allreduce_priority_mass: device vector of num_shards uint64 required");
        const NcclSyms& nc = nccl_syms();
        if (!nc.allreduce) throw Error(RB_ECUDA, "rb_allreduce_priority_mass: libnccl.so.2 not found");
        b->other_work();
        rb::prio_mass_launch(b, (unsigned long long*)masses);
        const ncclResult_t r = nc.allreduce(masses, masses, b->T, ncclUint64, ncclSum,
                                            (ncclComm_t)nccl_comm, b->stream);
        if (r != ncclSuccess)
            throw Error(RB_ECUDA, std::string("ncclAllReduce: ") +
                                      (nc.errstr ? nc.errstr(r) : std::to_string((int)r)));
    });
}

int rb_loss_finalize_vec(rb_buffer* b, float* dlogp, const double* vec3, rb_loss_stats* stats) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (!vec3 || !is_device_ptr(vec3)) invalid("rb_loss_finalize_vec: device vector required");
        b->other_work();
        const bool host = stats && !is_device_ptr(stats);
        rb_loss_stats* dst = host ? (rb_loss_stats*)b->scratch(sizeof(rb_loss_stats)) : stats;
        // the normalisation needs the tokens of this rank's batch: sel_total[0]
        k_finalize_vec<<<148, 256, 0, b->stream>>>(b->acc, vec3, dlogp, b->sel_total, dst,
                                                   b->last_loss == 0 ? 1 : 0);
        RB_CUDA(cudaGetLastError());
        if (host) {
            RB_CUDA(cudaMemcpyAsync(stats, dst, sizeof(rb_loss_stats), cudaMemcpyDeviceToHost,
                                    b->stream));
            b->sync();
        }
    });
}

int rb_loss_finalize(rb_buffer* b, float* dlogp, rb_loss_stats* stats) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        b->other_work();
        // Asynchronous when stats is a device pointer (the multi-GPU hot path:
        // allreduce the device stats, then finalize without a host round trip).
        if (!stats) invalid("rb_loss_finalize: stats required");
        const bool host = !is_device_ptr(stats);
        rb_loss_stats* dst = stats;
        if (host) {
            dst = (rb_loss_stats*)b->scratch(sizeof(rb_loss_stats));
            RB_CUDA(cudaMemcpyAsync(dst, stats, sizeof(rb_loss_stats), cudaMemcpyHostToDevice,
                                    b->stream));
        }
        // one kernel: every CTA reads the reduced stats and rescales its slice
        // of dlogp if a token was excluded anywhere; CTA 0 updates the
        // accumulator and writes the stats back
        k_finalize_stats<<<148, 256, 0, b->stream>>>(b->acc, dst, b->last_loss == 0 ? dlogp : nullptr,
                                                     b->sel_total, b->last_loss == 0 ? 1 : 0);
        RB_CUDA(cudaGetLastError());
        if (host) {
            RB_CUDA(cudaMemcpyAsync(stats, dst, sizeof(rb_loss_stats), cudaMemcpyDeviceToHost,
                                    b->stream));
            b->sync();
        }
    });
}

int rb_group_advantages(const double* rewards, const int64_t* offsets, size_t n_groups,
                        double* out_adv, double* out_mean) {
    return guard([&] {
        Ctx& c = ctx();
        std::lock_guard<std::mutex> lk(c.mu);
        c.init();
        int64_t last = 0;
        if (is_device_ptr(offsets))
            RB_CUDA(cudaMemcpy(&last, offsets + n_groups, 8, cudaMemcpyDeviceToHost));
        else
            last = offsets[n_groups];
        if (!is_device_ptr(offsets)) {
            for (size_t g = 0; g < n_groups; ++g)
                if (offsets[g + 1] - offsets[g] < 2) invalid("group advantages need >= 2 rewards");
        }
        std::vector<std::pair<void*, std::pair<void*, size_t>>> back;
        const double* r = c.in(rewards, (size_t)last);
        const int64_t* o = c.in(offsets, n_groups + 1);
        double* a = c.out(out_adv, (size_t)last, back);
        double* m = c.out(out_mean, n_groups, back);
        RB_CUDA(cudaMemsetAsync(c.dflag, 0, sizeof(int), c.stream));
        k_group_adv<<<grid_for((long long)n_groups), 256, 0, c.stream>>>(r, o, (long long)n_groups, a, m,
                                                                         c.dflag);
        RB_CUDA(cudaGetLastError());
        int bad = 0;
        RB_CUDA(cudaMemcpyAsync(&bad, c.dflag, sizeof bad, cudaMemcpyDeviceToHost, c.stream));
        c.finish(back);
        if (bad) invalid("group advantages need >= 2 rewards");
    });
}

int rb_grpo_tokens(const float* logp_now, const float* logp_old, const double* adv,
                   const int64_t* offsets, size_t n_traj, double eps_low, double eps_high,
                   float* out_dlogp, rb_loss_stats* stats) {
    return guard([&] {
        if (eps_low < 0.0 || eps_high < 0.0) invalid("loss spec: clip bounds must be >= 0");
        if (!std::isfinite(eps_low) || !std::isfinite(eps_high))
            invalid("loss spec: parameters must be finite");
        if (n_traj == 0) invalid("loss gradient needs a non-empty batch");
        Ctx& c = ctx();
        std::lock_guard<std::mutex> lk(c.mu);
        c.init();
        int64_t first = 0, last = 0;
        if (is_device_ptr(offsets)) {
            RB_CUDA(cudaMemcpy(&first, offsets, 8, cudaMemcpyDeviceToHost));
            RB_CUDA(cudaMemcpy(&last, offsets + n_traj, 8, cudaMemcpyDeviceToHost));
        } else {
            first = offsets[0];
            last = offsets[n_traj];
        }
        if (first != 0) invalid("rb_grpo_tokens: offsets must start at 0");
        require_aligned16(logp_now, "rb_grpo_tokens: logp_now");
        require_aligned16(logp_old, "rb_grpo_tokens: logp_old");
        require_aligned16(out_dlogp, "rb_grpo_tokens: out_dlogp");
        const size_t nt = ((size_t)last + 3) & ~size_t(3);
        std::vector<std::pair<void*, std::pair<void*, size_t>>> back;
        const float* lpn = c.in(logp_now, (size_t)last);
        const float* lpo = c.in(logp_old, (size_t)last);
        const double* a = c.in(adv, n_traj);
        const int64_t* o = c.in(offsets, n_traj + 1);
        float* d = c.out(out_dlogp, nt, back);
        if (back.size()) back.back().second.second = (size_t)last * sizeof(float);
        GrpoParams p;
        p.lo = 1.0 - eps_low;
        p.hi = 1.0 + eps_high;
        p.lo_f = (float)p.lo;
        p.hi_f = (float)p.hi;
        k_acc_reset<<<1, 1, 0, c.stream>>>(c.acc, last);
        k_loss_grpo_packed<<<(unsigned)n_traj, 256, 0, c.stream>>>(lpn, lpo, a, o, d, p, c.acc,
                                                                  (long long)n_traj);
        k_dlogp_rescale<<<148, 256, 0, c.stream>>>(d, last, nullptr, c.acc);
        RB_CUDA(cudaGetLastError());
        c.stats(stats, 0, 0.0, back);
        c.finish(back);
    });
}

int rb_grpo_tokens_ex(const float* logp_now, const float* logp_old, const double* adv,
                      const double* behavior_logprob, const int64_t* offsets, size_t n_traj,
                      double eps_low, double eps_high, int mode, float* out_dlogp,
                      rb_loss_stats* stats) {
    if (mode == RB_GRPO_TOKEN_MEAN)
        return rb_grpo_tokens(logp_now, logp_old, adv, offsets, n_traj, eps_low, eps_high,
                              out_dlogp, stats);
    return guard([&] {
        if (mode < RB_GRPO_TOKEN_MEAN || mode > RB_GRPO_SEQ_RATIO)
            invalid("rb_grpo_tokens_ex: unknown normalisation mode");
        if (eps_low < 0.0 || eps_high < 0.0) invalid("loss spec: clip bounds must be >= 0");
        if (!std::isfinite(eps_low) || !std::isfinite(eps_high))
            invalid("loss spec: parameters must be finite");
        if (n_traj == 0) invalid("loss gradient needs a non-empty batch");
        Ctx& c = ctx();
        std::lock_guard<std::mutex> lk(c.mu);
        c.init();
        int64_t first = 0, last = 0;
        if (is_device_ptr(offsets)) {
            RB_CUDA(cudaMemcpy(&first, offsets, 8, cudaMemcpyDeviceToHost));
            RB_CUDA(cudaMemcpy(&last, offsets + n_traj, 8, cudaMemcpyDeviceToHost));
        } else {
            first = offsets[0];
            last = offsets[n_traj];
        }
        if (first != 0) invalid("rb_grpo_tokens: offsets must start at 0");
        require_aligned16(out_dlogp, "rb_grpo_tokens_ex: out_dlogp");
        std::vector<std::pair<void*, std::pair<void*, size_t>>> back;
        const float* lpn = c.in(logp_now, (size_t)last);
        const float* lpo = c.in(logp_old, (size_t)last);
        const double* a = c.in(adv, n_traj);
        const double* bl = c.in(behavior_logprob, n_traj);
        const int64_t* o = c.in(offsets, n_traj + 1);
        float* d = c.out(out_dlogp, (size_t)last, back);
        GrpoParams p;
        p.lo = 1.0 - eps_low;
        p.hi = 1.0 + eps_high;
        p.lo_f = (float)p.lo;
        p.hi_f = (float)p.hi;
        const double s0 = (double)n_traj;
        k_acc_reset<<<1, 1, 0, c.stream>>>(c.acc, (long long)n_traj);  // divisor: sequences
        if (mode == RB_GRPO_SEQ_MEAN)
            k_loss_grpo_seq_packed<1><<<(unsigned)n_traj, SEQ_THREADS, 0, c.stream>>>(
                lpn, lpo, a, bl, o, d, p, s0, c.acc);
        else
            k_loss_grpo_seq_packed<2><<<(unsigned)n_traj, SEQ_THREADS, 0, c.stream>>>(
                lpn, lpo, a, bl, o, d, p, s0, c.acc);
        k_dlogp_rescale<<<148, 256, 0, c.stream>>>(d, last, nullptr, c.acc);
        RB_CUDA(cudaGetLastError());
        c.stats(stats, 0, 0.0, back);
        c.finish(back);
    });
}

int rb_grpo_records(const double* logp_now, const double* behavior_logprob, const double* adv,
                    size_t n, double eps_low, double eps_high, double* out_dlogp,
                    rb_loss_stats* stats) {
    return guard([&] {
        if (eps_low < 0.0 || eps_high < 0.0) invalid("loss spec: clip bounds must be >= 0");
        if (!std::isfinite(eps_low) || !std::isfinite(eps_high))
            invalid("loss spec: parameters must be finite");
        if (n == 0) invalid("loss gradient needs a non-empty batch");
        Ctx& c = ctx();
        std::lock_guard<std::mutex> lk(c.mu);
        c.init();
        std::vector<std::pair<void*, std::pair<void*, size_t>>> back;
        const double* lpn = c.in(logp_now, n);
        const double* blp = c.in(behavior_logprob, n);
        const double* a = c.in(adv, n);
        double* d = c.out(out_dlogp, n, back);
        k_acc_reset<<<1, 1, 0, c.stream>>>(c.acc, (long long)n);
        const unsigned g = grid_for((long long)n);
        k_grpo_records<<<g, 256, 0, c.stream>>>(lpn, blp, a, (long long)n, 1.0 - eps_low,
                                                1.0 + eps_high, d, c.acc);
        k_scale_records<<<g, 256, 0, c.stream>>>(d, (long long)n, c.acc);
        RB_CUDA(cudaGetLastError());
        c.stats(stats, 0, 0.0, back);
        c.finish(back);
    });
}

int rb_asymre_tokens(const float* logp_now, const double* reward, const double* group_mean,
                     const int64_t* offsets, size_t n_traj, double delta_v, float* out_dlogp,
                     rb_loss_stats* stats) {
    return guard([&] {
        if (!std::isfinite(delta_v)) invalid("loss spec: parameters must be finite");
        if (n_traj == 0) invalid("loss gradient needs a non-empty batch");
        Ctx& c = ctx();
        std::lock_guard<std::mutex> lk(c.mu);
        c.init();
        int64_t last = 0;
        if (is_device_ptr(offsets))
            RB_CUDA(cudaMemcpy(&last, offsets + n_traj, 8, cudaMemcpyDeviceToHost));
        else
            last = offsets[n_traj];
        std::vector<std::pair<void*, std::pair<void*, size_t>>> back;
        const float* lpn = c.in(logp_now, (size_t)last);
        const double* r = c.in(reward, n_traj);
        const double* gm = c.in(group_mean, n_traj);
        const int64_t* o = c.in(offsets, n_traj + 1);
        float* d = c.out(out_dlogp, (size_t)last, back);
        const double inv_b = 1.0 / (double)n_traj;
        k_acc_reset<<<1, 1, 0, c.stream>>>(c.acc, last);
        k_loss_asymre_packed<<<(unsigned)n_traj, 256, 0, c.stream>>>(lpn, r, gm, o, d, delta_v,
                                                                    inv_b, c.acc);
        RB_CUDA(cudaGetLastError());
        c.stats(stats, 1, inv_b, back);
        c.finish(back);
    });
}

int rb_asymre_records(const double* logp_now, const double* reward, const double* group_mean,
                      size_t n, double delta_v, double* out_dlogp, rb_loss_stats* stats) {
    return guard([&] {
        if (!std::isfinite(delta_v)) invalid("loss spec: parameters must be finite");
        if (n == 0) invalid("loss gradient needs a non-empty batch");
        Ctx& c = ctx();
        std::lock_guard<std::mutex> lk(c.mu);
        c.init();
        std::vector<std::pair<void*, std::pair<void*, size_t>>> back;
        const double* lpn = c.in(logp_now, n);
        const double* r = c.in(reward, n);
        const double* gm = c.in(group_mean, n);
        double* d = c.out(out_dlogp, n, back);
        k_acc_reset<<<1, 1, 0, c.stream>>>(c.acc, (long long)n);
        k_asymre_records<<<grid_for((long long)n), 256, 0, c.stream>>>(lpn, r, gm, (long long)n,
                                                                       delta_v, d, c.acc);
        RB_CUDA(cudaGetLastError());
        c.stats(stats, 1, 1.0 / (double)n, back);
        c.finish(back);
    });
}

}  // extern "C"

// Tuning aid (debug builds): the loss kernels' part of the kernel timeline
// (each translation unit has its own copy of the timeline array).
extern "C" __attribute__((visibility("default"))) int rb_debug_phase_clocks_loss(long long* out) {
    return guard([&] {
#ifdef RB_PHASE_CLOCKS
        RB_CUDA(cudaDeviceSynchronize());
        RB_CUDA(cudaMemcpyFromSymbol(out, g_phase_clock, 64 * sizeof(long long)));
#else
        for (int i = 0; i < 64; ++i) out[i] = 0;
#endif
    });
}
extern "C" __attribute__((visibility("default"))) int rb_debug_timeline_loss(unsigned long long* out,
                                                                             int reset) {
    return guard([&] {
#ifdef RB_PHASE_CLOCKS
        RB_CUDA(cudaDeviceSynchronize());
        RB_CUDA(cudaMemcpyFromSymbol(out, g_timeline, 64 * sizeof(unsigned long long)));
        if (reset) {
            unsigned long long init[64];
            for (int i = 0; i < 64; ++i) init[i] = (i < 32 && !(i & 1)) ? ~0ULL : 0ULL;
            RB_CUDA(cudaMemcpyToSymbol(g_timeline, init, sizeof init));
        }
#else
        for (int i = 0; i < 64; ++i) out[i] = 0;
#endif
    });
}
