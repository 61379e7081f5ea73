// buffer.cu — ShardedReplayBuffer on the GPU (replay_buffer.hpp:57-108).
//
// Kernels of one replay step, all on the buffer's stream:
//   k_route_fifo          FIFO insert, ids promised unique: one record per
//                         thread, whole-batch validation per CTA (split over
//                         the CTAs above 4096 records), group advantages
//                         (bandit.cpp:276-294), routing and victims in closed
//                         form (replay_buffer.cpp:83-133); extra CTAs keep a
//                         copy of the token offsets for the sampler.
//   k_insert_payload_tma  closed-form payload copy over cp.async.bulk, a
//                         programmatic dependent of the route (gated on its
//                         verdict); k_insert_payload: the table-driven copy.
//   k_sample_fused        uniform_with_replacement: MT19937-64 ring twisted
//                         ahead, draws, arrival index -> slot, look-back scan
//                         of the packed offsets (replay_buffer.cpp:135-217).
//                         Above 8192 draws the next call's blocks come from
//                         the Rng's side-stream lookahead (rng.cu).
//   k_gather              ragged 128-bit gather of the sampled rows;
//                         k_gather_early (opt-in) overlaps it with the copy.
// General paths: k_insert_route (exact sequential semantics: duplicate ids,
// positive bias validation) + k_posbias_batch (positive bias as O(1) queues),
// k_sample_without + k_sample_map (without-replacement strategies),
// k_sample_records (record copies with post-increment use counts, ledger).
#include <algorithm>
#include <charconv>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_set>
#include <vector>

#include "buffer_internal.cuh"
#include "rng_internal.cuh"
#include "stream_copy.cuh"


using namespace rb;

namespace rb {

constexpr uint64_t NONE_ID = UINT64_MAX;

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ int fifo_head(long long P, int C) {
    return P >= C ? (int)(P % C) : 0;
}
// Arrival head of shard s (FIFO: implicit ring; positive bias: v.order is
// materialised densely after every insert, head 0).
__device__ __forceinline__ int shard_head(const BufView& v, int s) {
    return v.retention == RB_POSITIVE_BIAS ? 0 : fifo_head(v.pushes[s], v.C);
}
// Local slot of arrival rank i (0 = oldest) given the shard's head.
__device__ __forceinline__ int arrival_slot_h(const BufView& v, int s, long long i, int head) {
    long long x = head + i;
    if (x >= v.C) x -= v.C;
    return v.retention == RB_POSITIVE_BIAS ? v.order[(size_t)s * v.C + x] : (int)x;
}
__device__ __forceinline__ int arrival_slot(const BufView& v, int s, long long i) {
    return arrival_slot_h(v, s, i, shard_head(v, s));
}
__device__ __forceinline__ long long occupancy(const BufView& v, int s) {
    const long long P = v.pushes[s];
    return P < v.C ? P : v.C;
}

// Block-wide: for items [0, n) with count(i) units each, emit(i, first, count)
// in item order; returns the total.  Items are split into contiguous
// per-thread runs so one block scan suffices.
template <class CountF, class EmitF>
__device__ long long block_build_units(long long n, CountF count, EmitF emit) {
    const long long per = (n + blockDim.x - 1) / blockDim.x;
    const long long i0 = threadIdx.x * per, i1 = i0 + per < n ? i0 + per : n;
    long long local = 0;
    for (long long i = i0; i < i1; ++i) local += count(i);
    long long total;
    long long pos = block_exclusive_scan(local, &total);
    for (long long i = i0; i < i1; ++i) {
        const long long c = count(i);
        emit(i, pos, c);
        pos += c;
    }
    return total;
}

struct InsertIn {
    long long n;
    const uint64_t *id, *prompt, *group;
    const int64_t *cstep, *pver;
    const double *reward, *blp, *adv, *gmean;
    const uint8_t* correct;
    const int64_t* goff;
    long long ngroups;
    const int64_t* toff;  // n+1 payload offsets (may be NULL: length 0)
    int64_t* toff_keep;   // closed-form route: copy of toff for a sampler that overlaps it
    int pay_follows;      // closed-form route: the payload copy is launched next
    int split_validate;   // closed-form route: validation split over the CTAs (large batches)
    int keep_ctas;        // closed-form route: extra CTAs copying toff into toff_keep
    unsigned long long* keep_cnt;  // route CTAs that finished their toff_keep slice (monotonic)
    int32_t maxlen;
    int32_t* len;         // scratch: per-record length
    double *adv_out, *gmean_out;
    int32_t* tslot;
    uint8_t* surv;
    uint64_t* evid;
    rb_record* evrec;     // may be NULL
    Unit* units;          // payload copy work units (owned survivors)
    int* n_units;
    // owned-metadata buffers (rb_insert_owned): the batch holds only the
    // records of the global batch of n_global routed to the one owned shard
    // v.sb, in arrival order (global arrival j0 + k*T for record k)
    int own_only;
    long long n_global;
    int epoch;            // closed-form route: the flag epoch of this insert (pay_sync tags)
};

__device__ __forceinline__ bool in_correct(const InsertIn& in, long long j) {
    return in.correct ? in.correct[j] != 0 : in.reward[j] == 1.0;
}
__device__ __forceinline__ rb_record in_record(const InsertIn& in, long long j) {
    rb_record r;
    r.rollout_id = in.id[j];
    r.prompt_id = in.prompt ? in.prompt[j] : 0;
    r.group_id = in.group ? in.group[j] : 0;
    r.creation_step = in.cstep ? in.cstep[j] : 0;
    r.policy_version = in.pver ? in.pver[j] : 0;
    r.reward = in.reward[j];
    r.is_correct = in_correct(in, j);
    r.behavior_logprob = in.blp ? in.blp[j] : 0.0;
    r.advantage = in.adv_out[j];
    r.use_count = 0;
    return r;
}
__device__ __forceinline__ rb_record slot_record(const BufView& v, size_t g) {
    rb_record r;
    r.rollout_id = v.id[g];
    r.prompt_id = v.prompt[g];
    r.group_id = v.group[g];
    r.creation_step = v.cstep[g];
    r.policy_version = v.pver[g];
    r.reward = v.reward[g];
    r.is_correct = v.correct[g];
    r.behavior_logprob = v.blp[g];
    r.advantage = v.adv[g];
    r.use_count = v.use[g];
    return r;
}
__device__ __forceinline__ void write_meta(const BufView& v, size_t g, const InsertIn& in,
                                           long long j) {
    v.id[g] = in.id[j];
    v.prompt[g] = in.prompt ? in.prompt[j] : 0;
    v.group[g] = in.group ? in.group[j] : 0;
    v.cstep[g] = in.cstep ? in.cstep[j] : 0;
    v.pver[g] = in.pver ? in.pver[j] : 0;
    v.reward[g] = in.reward[j];
    v.correct[g] = in_correct(in, j);
    v.blp[g] = in.blp ? in.blp[j] : 0.0;
    v.adv[g] = in.adv_out[j];
    v.gmean[g] = in.gmean_out[j];
    v.use[g] = 0;
    v.len[g] = in.len ? in.len[j] : 0;
}

// ---- present-id hash set (exact path only) ------------------------------
__device__ __forceinline__ unsigned long long hmix(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    return k;
}
__device__ bool h_find(const BufView& v, uint64_t k, unsigned long long* at) {
    unsigned long long i = hmix(k) & (v.hcap - 1);
    for (;;) {
        const uint32_t st = v.hstate[i];
        if (st == 0) return false;
        if (st == 1 && v.hkeys[i] == k) {
            *at = i;
            return true;
        }
        i = (i + 1) & (v.hcap - 1);
    }
}
__device__ void h_insert_seq(const BufView& v, uint64_t k) {  // caller checked absence
    unsigned long long i = hmix(k) & (v.hcap - 1);
    while (v.hstate[i] == 1) i = (i + 1) & (v.hcap - 1);
    v.hkeys[i] = k;
    v.hstate[i] = 1;
}
__device__ void h_erase(const BufView& v, uint64_t k) {
    unsigned long long at;
    if (h_find(v, k, &at)) v.hstate[at] = 2;
}
__device__ void h_insert_par(const BufView& v, uint64_t k) {  // distinct keys, no tombstones
    unsigned long long i = hmix(k) & (v.hcap - 1);
    while (atomicCAS(&v.hstate[i], 0u, 3u) != 0u) i = (i + 1) & (v.hcap - 1);
    v.hkeys[i] = k;
    __threadfence_block();
    v.hstate[i] = 1;
}
// Rebuild the set from the occupied slots (block-wide).
__device__ void h_rebuild(const BufView& v) {
    for (unsigned long long i = threadIdx.x; i < v.hcap; i += blockDim.x) v.hstate[i] = 0;
    __syncthreads();
    const long long N = (long long)v.T * v.C;
    for (long long g = threadIdx.x; g < N; g += blockDim.x) {
        const int s = (int)(g / v.C), x = (int)(g % v.C);
        if (x < occupancy(v, s)) h_insert_par(v, v.id[g]);
    }
    __syncthreads();
}

// ---- positive-bias retention (replay_buffer.cpp:98-133) as two queues ------
// The reference keeps a shard in arrival order and, once full, evicts the
// first !is_correct record among the oldest cs+1 arrivals (cs =
// correct_slots; that window is the reserve plus the record that just aged
// out of the newest fs = fresh_slots), else the oldest record, erasing it
// from the middle of the vector.  Equivalently: a FIFO F of the newest fs
// records and the reserve split into two arrival-ordered queues, W (wrong)
// and Q (correct).  A push appends x to F and moves F's oldest to W or Q;
// the victim is W's head if W is non-empty, else Q's head.  (fs == 0: x
// itself enters the reserve and may be the victim.)  Every push is O(1).
// Arrival order for sampling is materialised per shard after each insert:
// merge(W, Q) by arrival sequence number, then F (v.order, dense).
// Queue entries: local slot | is_correct << 31.
constexpr uint32_t PB_XMARK = 0x7fffffffu;  // "the record being pushed" (fs == 0)

__device__ __forceinline__ int32_t* pb_ring(const BufView& v, int r, int s) {
    return v.pbq + ((size_t)r * v.T + s) * (size_t)(v.C + 1);
}
struct GQ {  // a ring in global memory (sequential use by one thread)
    uint32_t* ring;
    int rc, h, n;
    __device__ int len() const { return n; }
    __device__ uint32_t pop() {
        const uint32_t e = ring[h];
        h = h + 1 == rc ? 0 : h + 1;
        --n;
        return e;
    }
    __device__ void push(uint32_t e) {
        int p = h + n;
        if (p >= rc) p -= rc;
        ring[p] = e;
        ++n;
    }
    __device__ void patch_tail(uint32_t e) {
        int p = h + n - 1;
        if (p >= rc) p -= rc;
        ring[p] = e;
    }
};
struct VQ {  // a ring's loaded prefix + the entries appended in this chunk (shared memory)
    const uint32_t* pre;
    uint32_t* app;
    int exist, pre_h, app_n, app_h;
    __device__ int len() const { return (exist - pre_h) + (app_n - app_h); }
    __device__ uint32_t pop() { return pre_h < exist ? pre[pre_h++] : app[app_h++]; }
    __device__ void push(uint32_t e) { app[app_n++] = e; }
    __device__ void patch_tail(uint32_t e) { app[app_n - 1] = e; }
};
// One push; returns x's local slot, or -1 when x itself is evicted.  *vict =
// local slot of the evicted record (-1: no eviction; -2: x itself).
template <class Qu>
__device__ __forceinline__ int pb_push_logic(int C, int fs, Qu& F, Qu& W, Qu& Q, int& size,
                                             bool xc, int* vict) {
    const uint32_t cb = xc ? 0x80000000u : 0u;
    if (size < C) {  // filling: no eviction
        const int gx = size++;
        if (fs > 0) {
            F.push((uint32_t)gx | cb);
            if (F.len() > fs) {
                const uint32_t y = F.pop();
                (y >> 31 ? Q : W).push(y);
            }
        } else {
            (xc ? Q : W).push((uint32_t)gx | cb);
        }
        *vict = -1;
        return gx;
    }
    if (fs > 0) {
        const uint32_t y = F.pop();
        (y >> 31 ? Q : W).push(y);
    } else {
        (xc ? Q : W).push(PB_XMARK | cb);
    }
    const uint32_t ve = W.len() ? W.pop() : Q.pop();
    const uint32_t vs = ve & 0x7fffffffu;
    if (vs == PB_XMARK) {
        *vict = -2;
        return -1;
    }
    const int gx = (int)vs;
    if (fs > 0) F.push((uint32_t)gx | cb);
    else (xc ? Q : W).patch_tail((uint32_t)gx | cb);
    *vict = gx;
    return gx;
}

// Block-wide: v.order of shard s = merge(W, Q) by arrival sequence, then F.
__device__ void pb_materialize(const BufView& v, int s) {
    const PbState st = v.pbs[s];
    const int C = v.C, RC = C + 1;
    const uint32_t* F = (const uint32_t*)pb_ring(v, 0, s);
    const uint32_t* W = (const uint32_t*)pb_ring(v, 1, s);
    const uint32_t* Q = (const uint32_t*)pb_ring(v, 2, s);
    const long long* seq = v.seq + (size_t)s * C;
    int32_t* ord = v.order + (size_t)s * C;
    auto at = [&](const uint32_t* ring, int h, int k) {
        int p = h + k;
        if (p >= RC) p -= RC;
        return (int)(ring[p] & 0x7fffffffu);
    };
    // rank of an element of one queue in the merge = its index + the number
    // of the other queue's elements that arrived earlier (binary search)
    const int nw = st.n[1], nq = st.n[2], nf = st.n[0];
    for (int k = threadIdx.x; k < nw + nq; k += blockDim.x) {
        const bool inw = k < nw;
        const int a = inw ? k : k - nw;
        const int slot = inw ? at(W, st.h[1], a) : at(Q, st.h[2], a);
        const long long sq = seq[slot];
        const uint32_t* O = inw ? Q : W;
        const int oh = inw ? st.h[2] : st.h[1], on = inw ? nq : nw;
        int lo = 0, hi = on;  // first index with seq > sq
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (seq[at(O, oh, mid)] < sq) lo = mid + 1;
            else hi = mid;
        }
        ord[a + lo] = slot;
    }
    for (int k = threadIdx.x; k < nf; k += blockDim.x) ord[nw + nq + k] = at(F, st.h[0], k);
}

// Positive-bias insert for ids promised new and increasing: one CTA per
// shard runs the O(1)-per-push queue simulation on shared memory (thread
// 0), in chunks of PB_CH pushes whose queue prefixes the whole CTA loads
// first; then, in parallel, evicted ids, the survivors' metadata, payload
// descriptors, the ring write-back and the materialised arrival order.
// k_insert_route ran before it (lengths, group advantages, validation) and
// set ctl->pb_go when this kernel is to apply the batch.
constexpr int PB_THREADS = 256;
constexpr int PB_CH = 512;
__global__ void __launch_bounds__(PB_THREADS) k_posbias_batch(BufView v, InsertIn in,
                                                              unsigned long long cur0) {
    extern __shared__ uint32_t pb_sm[];
    __shared__ int s_size;
    __shared__ PbState s_st;
    __shared__ int s_maxq, s_a0[3], s_a1[3];
    const int s = blockIdx.x, tid = threadIdx.x;
    const int T = v.T, C = v.C, RC = C + 1, fs = v.fs;
    if (!v.ctl->pb_go) return;
    const int n = (int)in.n;
    const int j0 = (int)(((long long)s - (long long)(cur0 % (unsigned long long)T)) % T + T) % T;
    const int ns = n > j0 ? (n - 1 - j0) / T + 1 : 0;
    uint32_t* Fpre = pb_sm;
    uint32_t* Wpre = Fpre + PB_CH;
    uint32_t* Qpre = Wpre + PB_CH;
    uint32_t* Fapp = Qpre + PB_CH;
    uint32_t* Wapp = Fapp + PB_CH;
    uint32_t* Qapp = Wapp + PB_CH;
    int* gxs = (int*)(Qapp + PB_CH);  // per push of this chunk: x's slot
    int* vic = gxs + PB_CH;           // evicted local slot / -1 / -2
    int* vocc = vic + PB_CH;          // occupant of the victim slot: batch index or -1
    int* occ = vocc + PB_CH;          // [C] batch index now holding each slot (-1: pre-batch)
    const long long P0 = v.pushes[s];
    for (int x = tid; x < C; x += PB_THREADS) occ[x] = -1;
    if (tid == 0) {
        s_st = v.pbs[s];
        s_size = (int)(P0 < C ? P0 : C);
        s_maxq = 0;
    }
    __syncthreads();
    uint32_t* Fr = (uint32_t*)pb_ring(v, 0, s);
    uint32_t* Wr = (uint32_t*)pb_ring(v, 1, s);
    uint32_t* Qr = (uint32_t*)pb_ring(v, 2, s);
    for (int c0 = 0; c0 < ns; c0 += PB_CH) {
        const int ch = ns - c0 < PB_CH ? ns - c0 : PB_CH;
        const PbState st = s_st;
        // queue prefixes (a chunk pops at most `ch` entries from each)
        for (int k = tid; k < ch; k += PB_THREADS) {
            int p;
            if (k < st.n[0]) { p = st.h[0] + k; if (p >= RC) p -= RC; Fpre[k] = (uint32_t)Fr[p]; }
            if (k < st.n[1]) { p = st.h[1] + k; if (p >= RC) p -= RC; Wpre[k] = (uint32_t)Wr[p]; }
            if (k < st.n[2]) { p = st.h[2] + k; if (p >= RC) p -= RC; Qpre[k] = (uint32_t)Qr[p]; }
            const int j = j0 + (c0 + k) * T;
            gxs[k] = in_correct(in, j) ? 1 : 0;  // x's correctness (overwritten below)
        }
        __syncthreads();
        if (tid == 0) {
            VQ F{Fpre, Fapp, st.n[0], 0, 0, 0}, W{Wpre, Wapp, st.n[1], 0, 0, 0},
                Q{Qpre, Qapp, st.n[2], 0, 0, 0};
            int size = s_size;
            for (int k = 0; k < ch; ++k) {
                const int j = j0 + (c0 + k) * T;
                int vs;
                const int gx = pb_push_logic(C, fs, F, W, Q, size, gxs[k] != 0, &vs);
                vocc[k] = vs >= 0 ? occ[vs] : -1;
                if (gx >= 0) occ[gx] = j;
                gxs[k] = gx;
                vic[k] = vs;
            }
            s_size = size;
            // ring write-back bookkeeping: new heads / counts (entries below)
            VQ* qs[3] = {&F, &W, &Q};
            for (int r = 0; r < 3; ++r) {
                const int pops = qs[r]->pre_h + qs[r]->app_h;
                s_st.h[r] = (st.h[r] + pops) % RC;
                s_st.n[r] = st.n[r] + qs[r]->app_n - pops;
                // appended entries still queued: app[app_h..app_n) at old tail + index
                s_a0[r] = qs[r]->app_h;
                s_a1[r] = qs[r]->app_n;
            }
        }
        __syncthreads();
        // write back the live appended entries at the rings' tails
        {
            const uint32_t* apps[3] = {Fapp, Wapp, Qapp};
            uint32_t* rings[3] = {Fr, Wr, Qr};
            for (int r = 0; r < 3; ++r) {
                const int a0 = s_a0[r], a1 = s_a1[r];
                for (int k = a0 + tid; k < a1; k += PB_THREADS) {
                    int p = st.h[r] + st.n[r] + k;
                    p %= RC;
                    rings[r][p] = apps[r][k];
                }
            }
        }
        // per push: evicted id (the victim's occupant before this push), seq
        for (int k = tid; k < ch; k += PB_THREADS) {
            const int j = j0 + (c0 + k) * T;
            const int vs = vic[k], gx = gxs[k];
            uint64_t ev = NONE_ID;
            if (vs == -2) {
                ev = in.id[j];
                if (in.evrec) in.evrec[j] = in_record(in, j);
            } else if (vs >= 0) {
                const int o = vocc[k];
                ev = o >= 0 ? in.id[o] : v.id[(size_t)s * C + vs];
                if (in.evrec) in.evrec[j] = o >= 0 ? in_record(in, o) : slot_record(v, (size_t)s * C + vs);
            }
            in.evid[j] = ev;
            in.tslot[j] = gx >= 0 ? (int32_t)((size_t)s * C + gx) : -1;
            if (gx >= 0) v.seq[(size_t)s * C + gx] = P0 + c0 + k;
        }
        __syncthreads();
    }
    // survivors (final occupant of their slot): metadata + payload descriptors
    int maxq = 0;
    for (int r = tid; r < ns; r += PB_THREADS) {
        const int j = j0 + r * T;
        const int32_t g = in.tslot[j];
        const bool surv = g >= 0 && occ[g - s * C] == j;
        in.surv[j] = surv;
        Unit d;
        d.row = -1;
        d.len = in.len[j];
        d.k0 = 0;
        d.g = j;
        d.off = in.toff ? in.toff[j] : 0;
        d.adv = 0.0;
        if (surv) {
            write_meta(v, (size_t)g, in, j);
            if (s >= v.sb && s < v.se && d.len > 0 && v.stride > 0) {
                d.row = (s - v.sb) * C + (g - s * C);
                const int q = (d.len + 3) >> 2;
                maxq = q > maxq ? q : maxq;
            }
        }
        in.units[j] = d;
    }
    maxq = __reduce_max_sync(0xffffffffu, maxq);
    if ((tid & 31) == 0 && maxq) atomicMax(&s_maxq, maxq);
    if (tid == 0) {
        PbState st = s_st;
        v.pbs[s] = st;
        v.pushes[s] = P0 + ns;
    }
    __syncthreads();
    if (tid == 0 && s_maxq) atomicMax(in.n_units, s_maxq);
    pb_materialize(v, s);
}

// ---------------------------------------------------------------- insert
__global__ void __launch_bounds__(1024) k_insert_route(BufView v, InsertIn in) {
    __shared__ int s_bad;
    __shared__ long long s_applied;
    const int tid = threadIdx.x, nt = blockDim.x;
    const long long n = in.n;
    DevCtl* ctl = v.ctl;
    if (tid == 0) ctl->pb_go = 0;  // set again below when k_posbias_batch is to apply
    if (ctl->err_code != 0) {  // sticky error: buffer frozen until rb_check
        if (tid == 0) *in.n_units = 0;
        for (long long j = tid; j < n; j += nt) {
            in.surv[j] = 0;
            in.tslot[j] = -1;
            in.evid[j] = NONE_ID;
        }
        return;
    }
    if (tid == 0) {
        s_bad = 0;
        s_applied = n;
    }
    __syncthreads();
    RB_CLOCK(10);
    // 0. lengths from the payload offsets
    for (long long j = tid; j < n; j += nt) {
        long long l = in.toff ? in.toff[j + 1] - in.toff[j] : 0;
        if (l < 0 || l > in.maxlen) {
            s_bad = 3;
            l = 0;
        }
        in.len[j] = (int32_t)l;
    }

    RB_CLOCK(11);
    // 1. group-relative advantages, frozen at insertion (bandit.cpp:276-294),
    //    fp64 with the reference's operation order (no FMA contraction).
    if (in.adv == nullptr) {
        if (tid == 0 && (in.goff[0] != 0 || in.goff[in.ngroups] != n)) s_bad = 1;
        // One thread per group, the reference's sequential fp64 order; the
        // group's reward loads are independent and pipeline (unrolled).
        for (long long g = tid; g < in.ngroups; g += nt) {
            const long long b = in.goff[g], e = in.goff[g + 1], m = e - b;
            if (m < 2 || b < 0 || e > n) {
                s_bad = 1;
                continue;
            }
            const double dn = (double)m;
            double mean = 0.0;
#pragma unroll 8
            for (long long k = b; k < e; ++k) mean = __dadd_rn(mean, in.reward[k]);
            mean = __ddiv_rn(mean, dn);
            double var = 0.0;
#pragma unroll 8
            for (long long k = b; k < e; ++k) {
                const double d = __dsub_rn(in.reward[k], mean);
                var = __dadd_rn(var, __dmul_rn(d, d));
            }
            var = __ddiv_rn(var, dn);
            const double sd = __dsqrt_rn(var);
            const double inv_ok = sd < 1e-8 ? 0.0 : 1.0;
#pragma unroll 8
            for (long long k = b; k < e; ++k) {
                in.adv_out[k] = inv_ok == 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(in.reward[k], mean), sd);
                in.gmean_out[k] = mean;  // bandit.cpp:316-318 (same sequential sum)
            }
        }
    } else {
        for (long long j = tid; j < n; j += nt) {
            in.adv_out[j] = in.adv[j];
            in.gmean_out[j] = in.gmean ? in.gmean[j] : 0.0;
        }
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) {
            ctl->err_code = RB_EINVAL;
            ctl->err_index = s_bad == 3 ? -3 : -2;
        }
        if (tid == 0) *in.n_units = 0;
        for (long long j = tid; j < n; j += nt) {
            in.surv[j] = 0;
            in.tslot[j] = -1;
            in.evid[j] = NONE_ID;
        }
        return;
    }

    RB_CLOCK(12);
    // 2. duplicate screening: strictly increasing ids above every id ever
    //    pushed cannot collide (all reference callers allocate ids that way).
    int risk = 0;
    for (long long j = tid; j < n; j += nt) {
        const uint64_t x = in.id[j];
        if (j > 0 ? x <= in.id[j - 1] : (ctl->has_any && x <= ctl->max_id)) risk = 1;
    }
    risk = __syncthreads_or(risk);
    RB_CLOCK(13);
    const unsigned long long cur0 = ctl->cursor;
    const int T = v.T, C = v.C;

    if (!risk && v.retention == RB_PLAIN_FIFO) {
        // 3a. FIFO closed form: push j -> shard (cur0+j)%T, per-shard arrival
        //     p = pushes_s + j/T, slot p % C; the victim is whatever held the
        //     slot C arrivals earlier (pre-batch record or an earlier push).
        // 32-bit index arithmetic (n, T, C < 2^31); the 64-bit push counts
        // enter only through a per-shard P mod C computed once.
        const int c0 = (int)(cur0 % (unsigned long long)T), n32 = (int)n;
        for (int j = tid; j < n32; j += nt) {
            int s = c0 + j % T;
            if (s >= T) s -= T;
            const int rank = j / T, j0 = j % T;
            const int ns = (n32 - 1 - j0) / T + 1;
            const long long P = v.pushes[s];
            const long long p = P + rank;
            const int pm = (int)(P % C);
            int x = pm + rank % C;
            if (x >= C) x -= C;
            const size_t g = (size_t)s * C + (size_t)x;
            in.tslot[j] = (int32_t)g;
            in.surv[j] = (rank + C >= ns);
            uint64_t ev = NONE_ID;
            if (p >= C) {
                if (rank >= C) {
                    const long long jv = j - (long long)C * T;
                    ev = in.id[jv];
                    if (in.evrec) in.evrec[j] = in_record(in, jv);
                } else {
                    ev = v.id[g];
                    if (in.evrec) in.evrec[j] = slot_record(v, g);
                }
            }
            in.evid[j] = ev;
        }
        __syncthreads();
        for (long long j = tid; j < n; j += nt)
            if (in.surv[j]) write_meta(v, (size_t)in.tslot[j], in, j);
        __syncthreads();
        for (int s = tid; s < T; s += nt) {
            const long long j0 = (((long long)s - (long long)(cur0 % T)) % T + T) % T;
            const long long ns = n > j0 ? (n - 1 - j0) / T + 1 : 0;
            v.pushes[s] += ns;
        }
        if (tid == 0) ctl->cursor = (cur0 + n) % T;
    } else if (!risk) {
        // 3b. positive bias, ids promised new: k_posbias_batch (launched next)
        //     applies the batch, writes the descriptors and the unit bound.
        if (tid == 0) {
            ctl->pb_go = 1;
            ctl->cursor = (cur0 + n) % T;
            *in.n_units = 0;
        }
    } else {
        // 3c. exact sequential path (possible duplicates): replay_buffer.cpp:83-96
        //     push by push against the present-id set.
        h_rebuild(v);
        if (tid == 0) {
            unsigned long long cur = cur0;
            long long j = 0;
            for (; j < n; ++j) {
                const uint64_t x = in.id[j];
                unsigned long long at;
                if (h_find(v, x, &at)) {
                    ctl->err_code = RB_EINVAL;
                    ctl->err_index = j;
                    ctl->err_id = x;
                    break;
                }
                h_insert_seq(v, x);
                const int s = (int)cur;
                cur = (cur + 1) % T;
                if (v.retention == RB_PLAIN_FIFO) {
                    const long long P = v.pushes[s];
                    const size_t g = (size_t)s * C + (size_t)(P % C);
                    uint64_t ev = NONE_ID;
                    if (P >= C) {
                        ev = v.id[g];
                        if (in.evrec) in.evrec[j] = slot_record(v, g);
                    }
                    write_meta(v, g, in, j);
                    in.tslot[j] = (int32_t)g;
                    v.owner[g] = (int32_t)j;
                    in.evid[j] = ev;
                    v.pushes[s] = P + 1;
                } else {
                    const long long P = v.pushes[s];
                    PbState st = v.pbs[s];
                    const int RC = C + 1;
                    GQ F{(uint32_t*)pb_ring(v, 0, s), RC, st.h[0], st.n[0]};
                    GQ W{(uint32_t*)pb_ring(v, 1, s), RC, st.h[1], st.n[1]};
                    GQ Q{(uint32_t*)pb_ring(v, 2, s), RC, st.h[2], st.n[2]};
                    int size = (int)(P < C ? P : C), vs;
                    const int gx = pb_push_logic(C, v.fs, F, W, Q, size, in_correct(in, j), &vs);
                    uint64_t ev = NONE_ID;
                    if (vs == -2) {
                        ev = in.id[j];
                        if (in.evrec) in.evrec[j] = in_record(in, j);
                    } else if (vs >= 0) {
                        const size_t gv = (size_t)s * C + vs;
                        ev = v.id[gv];
                        if (in.evrec) in.evrec[j] = slot_record(v, gv);
                    }
                    in.tslot[j] = -1;
                    if (gx >= 0) {
                        const size_t g = (size_t)s * C + gx;
                        write_meta(v, g, in, j);
                        in.tslot[j] = (int32_t)g;
                        v.owner[g] = (int32_t)j;
                        v.seq[g] = P;
                    }
                    in.evid[j] = ev;
                    st.h[0] = F.h;
                    st.n[0] = F.n;
                    st.h[1] = W.h;
                    st.n[1] = W.n;
                    st.h[2] = Q.h;
                    st.n[2] = Q.n;
                    v.pbs[s] = st;
                    v.pushes[s] = P + 1;
                }
                if (in.evid[j] != NONE_ID) h_erase(v, in.evid[j]);
            }
            s_applied = j;
            ctl->cursor = cur;
            for (long long k = j; k < n; ++k) {
                in.tslot[k] = -1;
                in.evid[k] = NONE_ID;
            }
        }
        __syncthreads();
        if (v.retention == RB_POSITIVE_BIAS)
            for (int s = 0; s < T; ++s) pb_materialize(v, s);
    }
    const bool pb_fast = !risk && v.retention == RB_POSITIVE_BIAS;  // k_posbias_batch applies
    if (risk || (v.retention != RB_PLAIN_FIFO && !pb_fast)) {
        for (long long j = tid; j < n; j += nt) {
            const int32_t g = in.tslot[j];
            in.surv[j] = g >= 0 && v.owner[g] == (int32_t)j;
        }
    }
    __syncthreads();
    RB_CLOCK(14);
    // 4. payload descriptors: one per record (row = -1 unless it survived the
    //    batch in a shard held here) and the max units per record; the
    //    payload kernel strides over n * ups virtual units.
    if (!pb_fast) {
        int ups = 0;
        if (in.toff && v.stride > 0) {
            for (long long j = tid; j < n; j += nt) {
                Unit d;
                d.row = -1;
                d.len = in.len[j];
                d.k0 = 0;
                d.g = (int32_t)j;
                d.off = in.toff[j];
                d.adv = 0.0;
                if (in.surv[j]) {
                    const int g = in.tslot[j], s = g / v.C;
                    if (s >= v.sb && s < v.se && d.len > 0) {
                        d.row = (s - v.sb) * v.C + (g - s * v.C);
                        const int u = (d.len + 3) >> 2;  // row quads
                        ups = u > ups ? u : ups;
                    }
                }
                in.units[j] = d;
            }
        }
        ups = __reduce_max_sync(0xffffffffu, ups);
        __shared__ int s_ups[32];
        if ((tid & 31) == 0) s_ups[tid >> 5] = ups;
        __syncthreads();
        if (tid == 0) {
            int m = 0;
            for (int w = 0; w < (nt >> 5); ++w) m = s_ups[w] > m ? s_ups[w] : m;
            *in.n_units = m;  // max quads per record
        }
    }
    RB_CLOCK(15);
    // 5. bookkeeping: largest id ever pushed (block max over the applied prefix)
    __shared__ unsigned long long s_mx[32];
    const long long applied = s_applied;
    unsigned long long mx = 0;
    for (long long j = tid; j < applied; j += nt) mx = in.id[j] > mx ? in.id[j] : mx;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((tid & 31) == 0) s_mx[tid >> 5] = mx;
    __syncthreads();
    if (tid == 0) {
        mx = ctl->has_any ? ctl->max_id : 0ULL;
        for (int w = 0; w < (nt >> 5); ++w) mx = s_mx[w] > mx ? s_mx[w] : mx;
        if (applied > 0) {
            ctl->max_id = mx;
            ctl->has_any = 1;
        }
        ctl->hash_stale = risk ? 0 : 1;
        RB_CLOCK(16);
    }
}

// ---- payload insert: persistent over n * ceil(max_nq / QPU) virtual units --
// Each unit copies 128*U quads of one surviving trajectory from the packed
// inbound batch (any alignment) into its 16-byte aligned slot row, tokens and
// logp_old interleaved so every thread keeps 2*U 16-byte loads in flight.
//
// Two descriptor sources: the route kernel's table (general path), or the
// FIFO closed form evaluated here from the pre-batch cursor and per-shard
// push counts (host mirrors, exact on this path), so the copy does not wait
// for the route: it is launched as a programmatic dependent of the route
// (PDL) and only its first store waits for the route's whole-batch
// validation flag (1 = valid, 2 = rejected; reset by the last CTA).
struct FifoPlan {
    int c0, T, C, ups;  // cursor % T, shards, capacity per shard, units per record
    int own;            // owned-metadata batch: the owned shard (its records only), else -1
    int epoch;          // the insert's flag epoch (verdict wait, copy-done publish)
    int pm[64];         // pushes_s % C before the batch
};
__device__ __forceinline__ Unit fifo_unit(const BufView& v, const FifoPlan& p,
                                          const int64_t* toff, int n, int j) {
    int s = p.c0 + j % p.T;
    if (s >= p.T) s -= p.T;
    int rank = j / p.T;
    const int j0 = j % p.T;
    int ns = (n - 1 - j0) / p.T + 1;
    if (p.own >= 0) {  // record j is the owned shard's j-th push of the batch
        s = p.own;
        rank = j;
        ns = n;
    }
    Unit d;
    d.off = toff[j];
    const long long l = toff[j + 1] - d.off;
    d.len = (int32_t)(l < 0 ? 0 : l);
    d.k0 = 0;
    d.g = j;
    d.adv = 0.0;
    d.row = -1;
    if (rank + p.C >= ns && s >= v.sb && s < v.se && l > 0) {
        int x = p.pm[s] + rank % p.C;
        if (x >= p.C) x -= p.C;
        d.row = (s - v.sb) * p.C + x;
    }
    return d;
}

// Completion flag of the closed-form payload copy for the early gather:
// sync[2] = 1 while the copy runs (set by the route kernel before any
// dependent can launch), cleared by the last CTA to finish (sync[3] counts
// them).
__device__ __forceinline__ void payload_pending_end(int* sync, int epoch) {  // thread 0, CTA's stores done
    if (done_add_u32(reinterpret_cast<unsigned*>(&sync[3])) == gridDim.x - 1) {
        sync[3] = 0;
        st_release_i32(&sync[2], epoch << 2 | 2);  // the copy of this insert is complete
    }
}

template <int U, bool CLOSED>
__device__ __forceinline__ void payload_body(const BufView& v, const Unit* desc, const FifoPlan& p,
                                             const int64_t* toff, int ups, int n,
                                             const int32_t* tokens, const float* logp_old,
                                             int* sync) {
    constexpr int QU = UNIT_THREADS * U;
    __shared__ int s_flag;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nu = n * ups;
    auto load_desc = [&](int u) { return CLOSED ? fifo_unit(v, p, toff, n, u / ups) : ld_unit(desc + u / ups); };
    bool ready = !CLOSED;
    // the sampler may launch: it waits for the route itself (closed form), or
    // the insert kernels before this copy are complete (table form); it never
    // reads the rows this copy writes, and waits for the copy before it exits
    pdl_trigger();
    Unit nxt;  // descriptor of the next unit, loaded one unit ahead
    if ((int)blockIdx.x < nu) nxt = load_desc(blockIdx.x);
    const long long tend = CLOSED ? toff[n] : 0;
    for (int u = blockIdx.x; u < nu; u += gridDim.x) {
        const int c = u % ups;
        const Unit un = nxt;
        if (u + (int)gridDim.x < nu) nxt = load_desc(u + (int)gridDim.x);
        const int nq = (un.len + 3) >> 2;  // destination (row) quads
        if (un.row < 0 || c * QU >= nq) continue;
        const int a = (int)(un.off & 3);
        const int nsq = (a + un.len + 3) >> 2;  // source quads touched
        const int kw = c * QU + wid * 32 * U;
        const size_t row = (size_t)un.row * v.stride;
        uint4 ot[U], ol[U];
        const uint4* tq = reinterpret_cast<const uint4*>(tokens) + (un.off >> 2);
        const uint4* lq = reinterpret_cast<const uint4*>(logp_old) + (un.off >> 2);
        // closed form: only a record whose last quad crosses the batch's end
        // (toff[n]) reads word by word; any other record's last quad reads
        // into the next record's tokens, inside the caller's arrays
        if (!CLOSED || ((un.off + un.len + 3) & ~3LL) > tend) {
            if (tokens) packed_to_row_quads<U, true>(tq, nsq, a, kw, ot, a + un.len);
            if (logp_old) packed_to_row_quads<U, true>(lq, nsq, a, kw, ol, a + un.len);
        } else {
            if (tokens) packed_to_row_quads<U, false>(tq, nsq, a, kw, ot, a + un.len);
            if (logp_old) packed_to_row_quads<U, false>(lq, nsq, a, kw, ol, a + un.len);
        }
        if (CLOSED && !ready) {  // CTA-uniform: first store of this CTA
            if (threadIdx.x == 0) {
                s_flag = spin_epoch(&sync[0], p.epoch);
            }
            __syncthreads();
            if (s_flag != 1) break;  // batch rejected: nothing is applied
            ready = true;
        }
#pragma unroll
        for (int s = 0; s < U; ++s) {
            const int k = kw + 32 * s + lane;
            if (k < nq) {
                if (tokens)
                    store_quad_masked(reinterpret_cast<uint32_t*>(v.tok + row), k, ot[s], 4 * k,
                                      un.len);
                if (logp_old)
                    store_quad_masked(reinterpret_cast<uint32_t*>(v.lpo + row), k, ol[s], 4 * k,
                                      un.len);
            }
        }
    }
    if (CLOSED) {
        __syncthreads();
        if (threadIdx.x == 0) payload_pending_end(sync, p.epoch);
        // completion of this copy implies completion of the route before it
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
}
template <int U>
__global__ void __launch_bounds__(UNIT_THREADS) k_insert_payload(BufView v, const Unit* desc,
                                                                 const int* maxq_p, int n,
                                                                 const int32_t* tokens,
                                                                 const float* logp_old) {
    RB_TSTART(1);
    const int ups = (*maxq_p + UNIT_THREADS * U - 1) / (UNIT_THREADS * U);
    payload_body<U, false>(v, desc, FifoPlan{}, nullptr, ups, n, tokens, logp_old, nullptr);
    RB_TEND(1);
}
template <int U>
__global__ void __launch_bounds__(UNIT_THREADS) k_insert_payload_fifo(BufView v, FifoPlan p,
                                                                      const int64_t* toff, int n,
                                                                      const int32_t* tokens,
                                                                      const float* logp_old,
                                                                      int* sync) {
    RB_TSTART(1);
    payload_body<U, true>(v, nullptr, p, toff, p.ups, n, tokens, logp_old, sync);
    RB_TEND(1);
}
#ifndef RB_PAYLOAD_U
#define RB_PAYLOAD_U 4
#endif
constexpr int PAYLOAD_U = RB_PAYLOAD_U;


// ---- payload insert over the bulk-copy engine (TMA) ------------------------
// The closed-form FIFO copy as independent cp.async.bulk pipelines, one per
// single-warp CTA (PB_CTAS per SM), each a ring of PB_S shared-memory stages
// of up to PB_CH tokens.  An item is one array (tokens or logp_old) of one
// chunk of one surviving trajectory: a 16-byte aligned source goes global ->
// smem -> slot row untouched; otherwise the aligned-down source quads are
// loaded and the warp shifts them in place before the bulk store (rows are
// 16-byte aligned and padded to a multiple of 4 tokens, so a store may round
// its length up to whole quads).  Lane 0 issues; the warp builds the list of
// its next 32 candidate items' descriptors in parallel (fifo_unit, one per
// lane) so descriptor loads never serialise the pipeline.  Descriptors come
// from the closed form; stores start once the route kernel has published a
// valid verdict.  tools/probes/payload_tma.cu: many small independent
// pipelines of 16 KB items reach the HBM copy rate (6.6-6.9 TB/s on 339 MB),
// a single thread issuing 4 KB items per SM does not (1.6 TB/s).
#ifndef RB_PB_S
#define RB_PB_S 2
#define RB_PB_L 1
#define RB_PB_CTAS 3
#endif
constexpr int PB_S = RB_PB_S;                  // stages per pipeline
constexpr int PB_L = RB_PB_L;                  // loads issued ahead of the stores
constexpr int PB_CTAS = RB_PB_CTAS;            // pipelines (single-warp CTAs) per SM
constexpr int PB_CHT = 4096;                   // tokens per item (16 KB)
constexpr int PB_RAW = PB_CHT + 4;             // words per stage (aligned-down source + spill)
constexpr size_t PB_SMEM = (size_t)PB_S * PB_RAW * 4 + PB_S * 8 + 32 * 16 + PB_S * 16;
static_assert(PB_S - PB_L - 1 >= 0, "bulk pipeline lag");
static_assert((PB_RAW * 4) % 16 == 0, "bulk-copy alignment");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct PbItem {
    int64_t src;  // packed element index of the item's first token
    int32_t row;  // slot row (local), -1 = none
    int32_t n;    // tokens | array << 30 | chunk << 20
};

__global__ void __launch_bounds__(32) k_insert_payload_tma(BufView v, FifoPlan p, const int64_t* toff,
                                                           int n, const int32_t* tokens,
                                                           const float* logp_old, int* sync) {
    extern __shared__ __align__(128) uint32_t pb_smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(pb_smem + PB_S * PB_RAW);
    PbItem* list = reinterpret_cast<PbItem*>(bar + PB_S);
    PbItem* meta = list + 32;  // the item held by each stage
    RB_TSTART(1);
    pdl_trigger();  // the sampler may launch (it waits for the route itself)
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < PB_S; ++s) mbar_init(&bar[s]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int cpr = (v.stride + PB_CHT - 1) / PB_CHT;  // chunks per record (bound)
    const int arrays = 2;                              // tokens, logp_old
    const long long nitems = (long long)n * arrays * cpr;
    const long long P = gridDim.x;
    long long issued = 0, stored = 0;
    int flag = 0;  // route verdict (1 valid, 2 rejected), read before the first store
    // store step of item g (whole warp): wait for its load, shift, bulk store
    auto store_one = [&](long long g) {
        const int st = (int)(g % PB_S);
        if (lane == 0) mbar_wait(&bar[st], (uint32_t)((g / PB_S) & 1));
        __syncwarp();
        const PbItem x = meta[st];
        const int cnt = x.n & 0xfffff, c = (x.n >> 20) & 0x3ff, arr = x.n >> 30;
        const int a = (int)(x.src & 3);
        const int words = (cnt + 3) & ~3;
        uint32_t* stg = pb_smem + (size_t)st * PB_RAW;
        {  // the source's last partial quad: word loads (the bulk copy stops at a quad boundary)
            const int full = (a + cnt) & ~3, tw = (a + cnt) & 3;
            const uint32_t* srcb = arr ? reinterpret_cast<const uint32_t*>(logp_old)
                                       : reinterpret_cast<const uint32_t*>(tokens);
            if (lane < tw) stg[full + lane] = __ldg(srcb + (x.src - a) + full + lane);
            if (tw && a == 0)  // generic-proxy writes read by the bulk store below
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
        }
        if (a != 0) {  // shift the aligned-down source quads down by `a`, in place
            for (int e0 = 0; e0 < words; e0 += 128) {
                uint32_t r[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = e0 + lane + 32 * q;
                    r[q] = e < words ? stg[a + e] : 0u;
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = e0 + lane + 32 * q;
                    if (e < words) stg[e] = r[q];
                }
                __syncwarp();
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
        }
        if (lane == 0) {
            if (flag == 0) flag = spin_epoch(&sync[0], p.epoch);
            if (flag == 1) {
                const size_t row = (size_t)x.row * v.stride + (size_t)c * PB_CHT;
                uint32_t* dst = arr ? reinterpret_cast<uint32_t*>(v.lpo) + row
                                    : reinterpret_cast<uint32_t*>(v.tok) + row;
                bulk_s2g(dst, stg, (uint32_t)words * 4);
            }
            bulk_commit();  // (an empty group when rejected keeps the count in step)
        }
    };
    for (long long base = blockIdx.x; base < nitems; base += 32 * P) {
        // this warp's next 32 candidate items: descriptors in parallel, compacted
        const long long u = base + (long long)lane * P;
        PbItem it{0, -1, 0};
        if (u < nitems) {
            const int j = (int)(u / (arrays * cpr));
            const int r = (int)(u - (long long)j * arrays * cpr);
            const int arr = r / cpr, c = r - arr * cpr;
            const Unit d = fifo_unit(v, p, toff, n, j);
            const int rest = d.len - c * PB_CHT;
            const bool have = arr ? logp_old != nullptr : tokens != nullptr;
            if (d.row >= 0 && rest > 0 && have) {
                it.row = d.row;
                it.src = d.off + (long long)c * PB_CHT;
                it.n = (rest < PB_CHT ? rest : PB_CHT) | (c << 20) | (arr << 30);
            }
        }
        const unsigned ok = __ballot_sync(0xffffffffu, it.row >= 0);
        if (it.row >= 0) list[__popc(ok & ((1u << lane) - 1))] = it;
        __syncwarp();
        const int m = __popc(ok);
        for (int i = 0; i < m; ++i) {
            if (lane == 0) {  // load item `issued` into its stage
                const long long g = issued;
                const int st = (int)(g % PB_S);
                if (g >= PB_S) bulk_wait_read<PB_S - PB_L - 1>();  // its stage's last store has read it
                const PbItem x = list[i];
                meta[st] = x;
                const int cnt = x.n & 0xfffff, arr = x.n >> 30;
                const int a = (int)(x.src & 3);
                const uint32_t bytes = (uint32_t)((a + cnt) & ~3) * 4;  // whole quads only
                const uint32_t* srcb = arr ? reinterpret_cast<const uint32_t*>(logp_old)
                                           : reinterpret_cast<const uint32_t*>(tokens);
                mbar_expect_tx(&bar[st], bytes);
                if (bytes) bulk_g2s(pb_smem + (size_t)st * PB_RAW, srcb + (x.src - a), bytes, &bar[st]);
            }
            ++issued;
            __syncwarp();
            if (issued - stored > PB_L) store_one(stored++);
        }
    }
    while (stored < issued) store_one(stored++);
    if (lane == 0) {
        bulk_wait_all();  // this CTA's row writes are complete
        asm volatile("fence.proxy.async.global;" ::: "memory");
        payload_pending_end(sync, p.epoch);
    }
    RB_TEND(1);
    // completion of this copy implies completion of the route before it
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- sample
struct SampleArgs {
    int nsh;            // shards to draw from (error semantics: [0, nsh))
    long long per;      // draws per shard
    int32_t* sel_shard;
    int64_t* sel_index;
    // map phase
    long long nsel, lo, hi;  // selections; owned range [lo, hi)
    int32_t* sel_slot;
    int32_t* sel_len;
    int64_t* off;
    long long* totals;
    DevLossAcc* acc;
    Unit* units;
    int* n_units;
    PendingIns pend;          // a closed-form FIFO insert that may still be running
    int early;                // publish the early-gather flags (seg, fin)
    int gen_ahead;            // the generator CTA also twists the next call's blocks
    long long occ[64];        // per-shard occupancy after the preceding inserts (draws)
    const long long* occ_dev;  // the same for more than 64 shards (device), else NULL
    const int* verdict;       // the pending insert's whole-batch verdict (1 valid, 2 rejected)
    int own_only;             // owned-metadata buffer: map (use counts, lengths, totals) only [lo, hi)
    int chk_frozen;           // k_sample_map after k_sample_prio: a sticky error freezes it too
};

// A rejected insert leaves a sticky error and freezes the buffer until
// rb_check: a fused sampler enqueued behind it applies nothing (no use
// counts, no RNG consumption, an empty batch).  Thread 0; block-uniform via
// the caller's shared copy.  While the insert may still run, its verdict
// flag decides (published before any of its records is applied).
__device__ __forceinline__ int sampler_frozen(const BufView& v, const SampleArgs& a) {
    if (a.pend.pending) return spin_epoch(a.verdict, a.pend.epoch) == 2;
    return *(volatile const int*)&v.ctl->err_code != 0;
}

// x % n without a 64-bit division: q from a precomputed reciprocal
// m = floor((2^64-1)/n) underestimates floor(x/n) by at most 2.
__device__ __forceinline__ uint64_t fast_mod(uint64_t x, uint64_t n, uint64_t m) {
    const uint64_t q = __umul64hi(x, m);
    uint64_t r = x - q * n;
    while (r >= n) r -= n;
    return r;
}

#ifdef RB_PHASE_CLOCKS
static __device__ long long g_dbg_locb[2];
#else
static __device__ long long g_dbg_locb[2];
#endif
// Per-shard heads of one sampling call, cached in shared memory for the
// first MAP_NSH shards (more shards read them from global memory).
constexpr int MAP_NSH = 128;
__device__ __forceinline__ int cached_head(const BufView& v, const int* heads, int s) {
    return s < MAP_NSH ? heads[s] : shard_head(v, s);
}

// Arrival head of shard s once the preceding insert is applied: from the
// insert's plan while it may still be running (closed-form FIFO, <= 64
// shards), else from the device counters.
__device__ __forceinline__ int head_after(const BufView& v, const PendingIns& pi, int s) {
    if (!pi.pending) return shard_head(v, s);
    const int T = v.T, C = v.C;
    const int j0 = ((s - pi.c0) % T + T) % T;
    const int ns = pi.n > j0 ? (pi.n - 1 - j0) / T + 1 : 0;
    const long long P = pi.P[s] + ns;
    return P >= C ? (int)(P % C) : 0;
}

// Grid-wide bookkeeping of the multi-CTA kernels (no grid barrier): CTAs
// take tickets in launch order, publish look-back words, and the last CTA
// to finish (done counter) finalises and resets the control block.
constexpr int GRID_MAX_CTAS = 4096;
struct GridCtl {
    unsigned int ticket, done;
    unsigned long long gsum;
    int first_rej;                      // fused sampler: first map CTA that saw a rejection
    int pad;
    long long gen_hi;                   // fused sampler: last ring block after the generator
    unsigned long long word[GRID_MAX_CTAS];  // look-back: status (2 bits) | value (62 bits)
    int cta_max[GRID_MAX_CTAS];
    // fused sampler -> early gather (k_gather_early): per map CTA, 0 = not
    // mapped yet, 1 = its units are final, 2 = a rejected draw at or before
    // it (final only once `fin` is set); fin = the last CTA has finalised
    int seg[GRID_MAX_CTAS];
    int fin;
    unsigned gwork, gdone;  // early gather: unit claim counter, done counter
    unsigned long long keep_cnt;  // route: CTAs that copied their offsets slice (monotonic)
    unsigned vdone, vbad;         // route (split validation): CTAs past it, OR of their bits
};
constexpr unsigned long long LB_AGG = 1ULL << 62, LB_INC = 2ULL << 62,
                             LB_VAL = (1ULL << 62) - 1;
// Warp 0: exclusive prefix of map CTA `t` over the aggregates / inclusive
// values of its predecessors (decoupled look-back).  Predecessors hold
// lower tickets, so they are running and publish without waiting.
__device__ __forceinline__ unsigned long long lookback(GridCtl* gc, int t) {
    const int lane = threadIdx.x & 31;
    unsigned long long excl = 0;
    for (int p = t - 1; p >= 0; p -= 32) {
        const int q = p - lane;
        unsigned long long w = 0;
        if (q >= 0) {
            do {
                w = ld_acquire_u64(&gc->word[q]);
            } while ((w >> 62) == 0);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, q >= 0 && (w >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 32;
        unsigned long long x = (q >= 0 && lane <= stop) ? (w & LB_VAL) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        excl += x;
        if (inc) break;
    }
    return excl;
}

// ---- map phase (every sampler): arrival index -> slot, use counts
// (replay_buffer.cpp:201), lengths, advantages; packed offsets of the owned
// selections by a decoupled look-back scan over the map CTAs; the gather /
// loss work descriptors.  Each thread maps MAP_R consecutive selections
// with every dependent load in flight together.
//
// DRAW = true (uniform_with_replacement, replay_buffer.cpp:141-145 and
// rng.cpp:40-51): the CTA also makes its selections' draws.  Shard 0 takes
// its `per` below(n_0) draws first, then shard 1, ...; draw k is word k of
// the MT19937-64 stream from the current position, tempered from the ring
// (blocks twisted ahead; blocks not resident yet are waited for from the
// generator CTA).  A rejected value (v >= limit; probability ~n/2^64 per
// draw) shifts every later draw: its CTA and every later one publish the
// fact through the look-back word, apply nothing, and the last CTA replays
// the rest exactly.
#ifndef RB_MAP_THREADS
#define RB_MAP_THREADS 128
#endif
constexpr int MAP_THREADS = RB_MAP_THREADS;  // small: co-resides with the persistent payload grid
#ifndef RB_MAP_R
#define RB_MAP_R 2
#endif
constexpr int MAP_R = RB_MAP_R;
constexpr int MAP_SPC = MAP_THREADS * MAP_R;  // selections per map CTA
constexpr int DRAW_NSH = 64;                  // shards whose occupancy rides in the arguments
constexpr unsigned long long LB_REJ = 1ULL << 61;
constexpr unsigned long long LB_SUM = LB_REJ - 1;

struct DrawCtx {  // ring position at the start of the call (header is constant meanwhile)
    const MtRing* r;
    long long q0, qhi0;
    uint32_t idx0;
};

template <bool DRAW>
__device__ void map_cta(const BufView& v, const SampleArgs& a, GridCtl* gc, int t,
                        const DrawCtx& dc, const int* route_done) {
    __shared__ int s_head[MAP_NSH], s_newfrom[MAP_NSH], s_ns[MAP_NSH], s_j0[MAP_NSH];
    __shared__ int s_occ_after[MAP_NSH];
    __shared__ unsigned long long s_lim[DRAW_NSH], s_mag[DRAW_NSH];
    __shared__ long long s_occ[DRAW_NSH];
    __shared__ unsigned long long s_excl, s_w[MAP_THREADS / 32];
    __shared__ int s_m[MAP_THREADS / 32];
    const int tid = threadIdx.x;
    const PendingIns& pi = a.pend;
    // Shard heads after the preceding insert.  While a closed-form FIFO
    // insert may still be running (pi.pending), they and the position of its
    // records follow from its plan: the newest min(ns, C) records of shard s
    // are its pushes to s; their lengths come from its offsets, so the map
    // needs the route kernel only for the use counts and advantages (last).
    for (int s = tid; s < a.nsh && s < MAP_NSH; s += MAP_THREADS) {
        if (pi.pending) {
            const int T = v.T, C = v.C;
            const int j0 = ((s - pi.c0) % T + T) % T;
            const int ns = pi.n > j0 ? (pi.n - 1 - j0) / T + 1 : 0;
            const long long P = pi.P[s] + ns;
            const int occ = (int)(P < C ? P : C);
            s_head[s] = P >= C ? (int)(P % C) : 0;
            s_newfrom[s] = occ - (ns < C ? ns : C);
            s_ns[s] = ns;
            s_j0[s] = j0;
            s_occ_after[s] = occ;
        } else {
            s_head[s] = shard_head(v, s);
            s_newfrom[s] = INT_MAX;
        }
    }
    if (DRAW)
        for (int s = tid; s < a.nsh && s < DRAW_NSH; s += MAP_THREADS) {
            const unsigned long long n = (unsigned long long)a.occ[s];
            s_occ[s] = (long long)n;
            s_lim[s] = below_limit(n);
            s_mag[s] = UINT64_MAX / n;
        }
    const long long kc = (long long)t * MAP_SPC;  // first selection of this CTA
    RB_GCLOCK(41 + 8 * (t & 1), t < 2);
    // Blocks past the ring's resident range (first call, or a larger batch
    // than the generator planned for) are twisted here into shared memory
    // (the ring itself is written only by the generator CTA).  A CTA's
    // MAP_SPC draws span at most LOC_BLKS blocks.
    constexpr int LOC_BLKS = MAP_SPC / MT_N + 2;
    __shared__ uint64_t s_loc[LOC_BLKS][MT_N];
    __shared__ uint64_t s_tw[MT_N];
    long long locb = LLONG_MAX;  // first block held in s_loc
    if (DRAW && kc < a.nsel) {
        const long long kl = (kc + MAP_SPC < a.nsel ? kc + MAP_SPC : a.nsel) - 1;
        const long long firstb = dc.q0 + (long long)((dc.idx0 + (unsigned long long)kc) / MT_N);
        const long long lastb = dc.q0 + (long long)((dc.idx0 + (unsigned long long)kl) / MT_N);
        if (lastb > dc.qhi0) {  // block-uniform
            locb = firstb > dc.qhi0 + 1 ? firstb : dc.qhi0 + 1;
            for (int i = tid; i < MT_N; i += MAP_THREADS) s_tw[i] = __ldcg(&dc.r->blk[dc.qhi0 % MT_KR][i]);
            __syncthreads();
            for (long long q = dc.qhi0 + 1; q <= lastb; ++q) {
                mt_twist_block(s_tw);
                if (q >= locb)
                    for (int i = tid; i < MT_N; i += MAP_THREADS) s_loc[q - locb][i] = s_tw[i];
            }
        }
    }
    __syncthreads();
    RB_GCLOCK(42 + 8 * (t & 1), t < 2);
    if (threadIdx.x == 0 && t < 2) g_dbg_locb[t] = locb == LLONG_MAX ? -1 : locb - dc.qhi0;
    const long long k0 = kc + (long long)tid * MAP_R;
    const int per = (int)a.per;
    int sh[MAP_R], ix[MAP_R], g[MAP_R], L[MAP_R];
    bool ok[MAP_R];
    bool rej = false;
    // Branch-free: every load of a stage is issued before any is consumed
    // (out-of-range lanes read a valid dummy address), so each stage costs one
    // memory round trip instead of MAP_R.
    uint64_t w[MAP_R];
#pragma unroll
    for (int r = 0; r < MAP_R; ++r) {
        const long long k = k0 + r;
        ok[r] = k < a.nsel;
        const long long kk = ok[r] ? k : 0;
        if (DRAW) {
            const unsigned long long o = dc.idx0 + (unsigned long long)kk;
            const long long qb = dc.q0 + (long long)(o / MT_N);
            const long long qr = qb < locb ? qb : dc.q0;  // resident block (or a dummy)
            const uint64_t wr = __ldcg(&dc.r->blk[qr % MT_KR][o % MT_N]);
            const uint64_t wl = s_loc[qb < locb ? 0 : qb - locb][o % MT_N];
            w[r] = qb < locb ? wr : wl;
        } else {
            sh[r] = a.sel_shard[kk];
            ix[r] = (int)a.sel_index[kk];
        }
    }
    if (DRAW) {
#pragma unroll
        for (int r = 0; r < MAP_R; ++r) {
            const long long kk = ok[r] ? k0 + r : 0;
            const uint64_t y = mt_temper(w[r]);
            const int s = (int)kk / per;
            unsigned long long n, lim, mag;
            if (s < DRAW_NSH) {
                n = (unsigned long long)s_occ[s];
                lim = s_lim[s];
                mag = s_mag[s];
            } else {
                n = (unsigned long long)a.occ_dev[s];
                lim = below_limit(n);
                mag = UINT64_MAX / n;
            }
            rej |= ok[r] && y >= lim;
            sh[r] = s;
            ix[r] = (int)fast_mod(y, n, mag);
        }
    }
    RB_GCLOCK(46 + 8 * (t & 1), t < 2);
    if (pi.pending && pi.toff) {  // the route kernel's copy of the insert's offsets
        if (tid == 0) spin_until_ge_u64(pi.keep_cnt, pi.keep_target);  // bounded: traps, never hangs
        __syncthreads();
    }
    int lv[MAP_R];
    double av[MAP_R];
    long long t0[MAP_R], t1[MAP_R];
    bool nw[MAP_R];
#pragma unroll
    for (int r = 0; r < MAP_R; ++r) {
        const int s = sh[r];
        g[r] = s * v.C + arrival_slot_h(v, s, ix[r], cached_head(v, s_head, s));
        const int nf = s < MAP_NSH ? s_newfrom[s] : INT_MAX;
        nw[r] = ix[r] >= nf;  // a record of the pending insert: length from its offsets
        const bool has_off = nw[r] && pi.toff != nullptr;  // no offsets: length 0
        const int jr = s_ns[s] - (s_occ_after[s] - ix[r]);  // its push index within shard s
        const int j = has_off ? (pi.own ? jr : s_j0[s] + jr * v.T) : 0;
        const int64_t* to = has_off ? pi.toff : reinterpret_cast<const int64_t*>(v.pushes);
        lv[r] = v.len[g[r]];
        av[r] = v.adv[g[r]];  // old records' advantages (new ones: after the route)
        t0[r] = to[j];
        t1[r] = to[j + (has_off ? 1 : 0)];
    }
    // live: mapped selections (an owned-metadata buffer maps its own slice only;
    // the other draws still count for the rejection check above)
    bool live[MAP_R];
#pragma unroll
    for (int r = 0; r < MAP_R; ++r)
        live[r] = ok[r] && (!a.own_only || (k0 + r >= a.lo && k0 + r < a.hi));
#pragma unroll
    for (int r = 0; r < MAP_R; ++r) {
        const long long l = t1[r] - t0[r];
        L[r] = !live[r] ? 0 : nw[r] ? (int)(l < 0 ? 0 : l) : lv[r];
    }
    unsigned long long own = 0, all = 0;
#pragma unroll
    for (int r = 0; r < MAP_R; ++r) {
        all += (unsigned long long)L[r];
        if (ok[r] && k0 + r >= a.lo && k0 + r < a.hi) own += (unsigned long long)L[r];
    }
    RB_GCLOCK(47 + 8 * (t & 1), t < 2);
    // v.dbg_replay (tests): every CTA takes the exact-replay path
    const bool cta_rej = DRAW && __syncthreads_or(rej || v.dbg_replay);
    RB_GCLOCK(43 + 8 * (t & 1), t < 2);
    long long cta_own;
    const long long pre = block_exclusive_scan((long long)own, &cta_own);
#pragma unroll
    for (int o = 16; o; o >>= 1) all += __shfl_xor_sync(0xffffffffu, all, o);
    if ((tid & 31) == 0) s_w[tid >> 5] = all;
    __syncthreads();
    const unsigned long long rbit = cta_rej ? LB_REJ : 0;
    if (tid < 32) {
        if (tid == 0)
            st_release_u64(&gc->word[t], (t ? LB_AGG : LB_INC) | rbit | (unsigned long long)cta_own);
        const unsigned long long excl = t ? lookback(gc, t) : 0;  // sums and OR of reject bits
        if (tid == 0) {
            const unsigned long long inc = ((excl & LB_SUM) + (unsigned long long)cta_own) |
                                           (excl & LB_REJ) | rbit;
            if (t) st_release_u64(&gc->word[t], LB_INC | inc);
            s_excl = excl | rbit;
        }
    }
    __syncthreads();
    RB_GCLOCK(44 + 8 * (t & 1), t < 2);
    if (DRAW || a.chk_frozen) {
        __shared__ int s_frozen;
        if (tid == 0) s_frozen = sampler_frozen(v, a);
        __syncthreads();
        if (s_frozen) {  // empty batch: zero-length work units, nothing mutated
#pragma unroll
            for (int r = 0; r < MAP_R; ++r) {
                const long long k = k0 + r;
                if (!ok[r] || k < a.lo || k >= a.hi) continue;
                Unit d{};
                a.units[k - a.lo] = d;
                a.off[k - a.lo] = 0;
            }
            if (tid == 0) gc->cta_max[t] = 0;
            if (a.early && tid == 0) st_release_i32(&gc->seg[t], 1);
            return;
        }
    }
    if (s_excl & LB_REJ) {  // a rejection at or before this CTA: the last CTA replays
        if (tid == 0) atomicMin(&gc->first_rej, t);
        if (tid == 0) gc->cta_max[t] = 0;
        if (a.early && tid == 0) st_release_i32(&gc->seg[t], 2);
        return;
    }
    if (tid == 0) {
        unsigned long long ca = 0;
        for (int w = 0; w < MAP_THREADS / 32; ++w) ca += s_w[w];
        atomicAdd(&gc->gsum, ca);
    }
    long long pos = (long long)(s_excl & LB_SUM) + pre;
    int maxq = 0;
#pragma unroll
    for (int r = 0; r < MAP_R; ++r) {
        const long long k = k0 + r;
        if (!ok[r]) continue;
        if (DRAW) {
            a.sel_shard[k] = sh[r];
            a.sel_index[k] = ix[r];
        }
        if (!live[r]) continue;
        a.sel_slot[k] = g[r];
        a.sel_len[k] = L[r];
        if (k < a.lo || k >= a.hi) continue;
        a.off[k - a.lo] = pos;
        Unit d;
        d.row = (sh[r] - v.sb) * v.C + (g[r] - sh[r] * v.C);
        d.len = L[r];
        d.k0 = nw[r] ? 1 : 0;  // a record of the pending insert (its row may still be copied)
        d.g = g[r];
        d.off = pos;
        d.adv = av[r];  // new records: patched below once the route kernel wrote it
        a.units[k - a.lo] = d;
        const int nq = ((int)(pos & 3) + L[r] + 3) >> 2;
        if (L[r]) maxq = nq > maxq ? nq : maxq;
        pos += L[r];
    }
    maxq = __reduce_max_sync(0xffffffffu, maxq);
    if ((tid & 31) == 0) s_m[tid >> 5] = maxq;
    // use counts (replay_buffer.cpp:201): records older than the pending
    // insert now (its route kernel leaves their slots alone) ...
    bool any_new = false;
#pragma unroll
    for (int r = 0; r < MAP_R; ++r) {
        if (!live[r]) continue;
        if (nw[r]) any_new = true;
        else atomicAdd(&v.use[g[r]], 1u);
    }
    // ... and its own records once the route kernel has written them
    const bool cta_new = __syncthreads_or(any_new);
    if (DRAW && a.early && tid == 0) st_release_i32(&gc->seg[t], 1);  // this CTA's units are final
    if (cta_new) {
        if (tid == 0) spin_epoch(route_done, pi.epoch);
        __syncthreads();
        double adv[MAP_R];
#pragma unroll
        for (int r = 0; r < MAP_R; ++r) adv[r] = v.adv[g[r]];
#pragma unroll
        for (int r = 0; r < MAP_R; ++r) {
            if (!live[r] || !nw[r]) continue;
            atomicAdd(&v.use[g[r]], 1u);
            const long long k = k0 + r;
            if (k >= a.lo && k < a.hi) reinterpret_cast<double*>(&a.units[k - a.lo])[3] = adv[r];
        }
    }
    if (tid == 0) {
        int m = 0;
        for (int w = 0; w < MAP_THREADS / 32; ++w) m = s_m[w] > m ? s_m[w] : m;
        gc->cta_max[t] = m;
    }
    RB_GCLOCK(45 + 8 * (t & 1), t < 2);
}
// Done counter; returns (block-uniform) whether this CTA finished last.
__device__ __forceinline__ bool last_to_finish(GridCtl* gc) {
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) s_last = done_add_u32(&gc->done) == gridDim.x - 1;
    __syncthreads();
    return s_last;
}

// Exact sequential replay of draws [k0, k1) from a shared copy of the
// block holding the current position (thread 0; rejections shift the stream).
__device__ __noinline__ void draw_exact(int32_t* sel_shard, int64_t* sel_index, long long per,
                                        const long long* occ, uint64_t* mt, long long k0,
                                        long long k1, uint32_t* idx, long long* tw,
                                        unsigned long long* dr) {
    for (long long kk = k0; kk < k1; ++kk) {
        const int ss = (int)(kk / per);
        const unsigned long long n = (unsigned long long)occ[ss];
        const uint64_t lim = below_limit(n);
        uint64_t y;
        do {
            if (*idx >= MT_N) {
                mt_twist_scalar(mt);
                *idx = 0;
                ++*tw;
            }
            y = mt_temper(mt[(*idx)++]);
            ++*dr;
        } while (y >= lim);
        sel_shard[kk] = ss;
        sel_index[kk] = (int64_t)(y % n);
    }
}

// Last CTA: (replay of a rejected tail,) totals, work-unit bound,
// loss-accumulator reset, control reset; the new ring position when drawing.
template <bool DRAW>
__device__ void map_finalize(const BufView& v, const SampleArgs& a, GridCtl* gc, int nmap,
                             const DrawCtx& dc, MtRing* r, const int* route_done) {
    __shared__ int s_m[32];
    __shared__ uint64_t mt[MT_N];
    __shared__ long long s_q;
    __shared__ uint32_t s_idx;
    __shared__ long long s_total, s_genhi;
    __shared__ unsigned long long s_g;
    // every map CTA's writes were acquired by the done counter: the loads
    // of the common path are independent and issued together with `first`
    unsigned long long wl = 0, dr = 0, gs = 0;
    long long gh = 0;
    if (threadIdx.x == 0) {
        wl = __ldcg(&gc->word[nmap - 1]);
        gs = __ldcg(&gc->gsum);
        if (DRAW) {
            dr = r->draws;
            gh = __ldcg(&gc->gen_hi);
        }
    }
    const int first = DRAW ? __ldcg(&gc->first_rej) : INT_MAX;
    const long long D = a.nsel;
    const long long nloc = a.hi - a.lo;
    __shared__ int s_frozen;
    if (threadIdx.x == 0) s_frozen = (DRAW || a.chk_frozen) ? sampler_frozen(v, a) : 0;  // final: a map CTA waited for it
    __syncthreads();
    const bool frozen = s_frozen != 0;
    if (frozen) {  // a rejected insert before this sampler: empty batch, ring position unchanged
        if (threadIdx.x == 0) {
            s_total = 0;
            s_g = 0;
            s_m[0] = 0;
            s_q = dc.q0;
            s_idx = dc.idx0;
            s_genhi = gh;
        }
        __syncthreads();
    } else if (DRAW && first != INT_MAX) {
        // the stream had no rejection before selection k0
        const long long k0 = (long long)first * MAP_SPC;
        long long q = dc.q0;
        uint32_t idx = dc.idx0;
        ring_advance(q, idx, (unsigned long long)k0);
        for (int i = threadIdx.x; i < MT_N; i += blockDim.x) mt[i] = __ldcg(&dc.r->blk[q % MT_KR][i]);
        __syncthreads();
        __shared__ long long s_occ[DRAW_NSH];
        for (int s = threadIdx.x; s < a.nsh && s < DRAW_NSH; s += blockDim.x) s_occ[s] = a.occ[s];
        __syncthreads();
        if (threadIdx.x == 0) {
            long long tw = 0;
            unsigned long long dr = 0;
            draw_exact(a.sel_shard, a.sel_index, a.per, a.occ_dev ? a.occ_dev : s_occ, mt, k0, D,
                       &idx, &tw, &dr);
            s_q = q + tw;
            s_idx = idx;
            r->draws = r->draws + (unsigned long long)k0 + dr;
        }
        __syncthreads();
        // map the replayed tail, then rescan every owned offset (shard heads
        // from the insert's plan: the route kernel may still be advancing
        // the device counters; the metadata it writes is read below)
        if (threadIdx.x == 0 && a.pend.pending) spin_epoch(route_done, a.pend.epoch);
        __shared__ int s_head[MAP_NSH];
        for (int s = threadIdx.x; s < a.nsh && s < MAP_NSH; s += blockDim.x)
            s_head[s] = head_after(v, a.pend, s);
        __syncthreads();
        unsigned long long tail = 0;
        const long long kb = a.own_only ? (k0 > a.lo ? k0 : a.lo) : k0;
        const long long ke = a.own_only ? (D < a.hi ? D : a.hi) : D;
        for (long long k = kb + threadIdx.x; k < ke; k += blockDim.x) {
            const int s = a.sel_shard[k];
            const int g = s * v.C + arrival_slot_h(v, s, a.sel_index[k], cached_head(v, s_head, s));
            atomicAdd(&v.use[g], 1u);
            a.sel_slot[k] = g;
            const int L = v.len[g];
            a.sel_len[k] = L;
            tail += (unsigned long long)L;
            if (k >= a.lo && k < a.hi) {
                Unit d;
                d.row = (s - v.sb) * v.C + (g - s * v.C);
                d.len = L;
                d.k0 = 0;
                d.g = g;
                d.off = 0;
                d.adv = v.adv[g];
                a.units[k - a.lo] = d;
            }
        }
        tail = warp_sum_i64((long long)tail);
        if ((threadIdx.x & 31) == 0) atomicAdd(&gc->gsum, tail);
        __syncthreads();
        long long carry = 0;
        int maxq = 0;
        for (long long cb = 0; cb < nloc; cb += blockDim.x) {
            const long long i = cb + threadIdx.x;
            const long long L = i < nloc ? a.sel_len[a.lo + i] : 0;
            long long ct;
            const long long ex = block_exclusive_scan(L, &ct);
            if (i < nloc) {
                const long long pos = carry + ex;
                a.off[i] = pos;
                reinterpret_cast<long long*>(&a.units[i])[2] = pos;  // Unit::off
                const int nq = ((int)(pos & 3) + (int)L + 3) >> 2;
                if (L) maxq = nq > maxq ? nq : maxq;
            }
            carry += ct;
        }
        maxq = __reduce_max_sync(0xffffffffu, maxq);
        if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = maxq;
        __syncthreads();
        if (threadIdx.x == 0) {
            int mm = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = s_m[w] > mm ? s_m[w] : mm;
            s_total = carry;
            s_m[0] = mm;
        }
        __syncthreads();
    } else {
        int m = 0;
        for (int c = threadIdx.x; c < nmap; c += blockDim.x) m = max(m, __ldcg(&gc->cta_max[c]));
        m = __reduce_max_sync(0xffffffffu, m);
        if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            int mm = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mm = s_m[w] > mm ? s_m[w] : mm;
            s_m[0] = mm;
            s_total = (long long)(wl & LB_SUM);
            s_g = gs;
            s_genhi = gh;
            if (DRAW) {
                long long q = dc.q0;
                uint32_t idx = dc.idx0;
                ring_advance(q, idx, (unsigned long long)D);
                s_q = q;
                s_idx = idx;
                r->draws = dr + (unsigned long long)D;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const unsigned long long global =
            (DRAW && first != INT_MAX && !frozen) ? atomicAdd(&gc->gsum, 0ULL) : s_g;
        s_g = global;
        a.off[nloc] = s_total;
        a.totals[0] = s_total;
        a.totals[1] = (long long)global;
        *a.n_units = s_m[0];  // max destination quads per selection
        DevLossAcc* acc = a.acc;
        acc->obj_sum = 0.0;
        acc->included = 0;
        acc->excluded = 0;
        acc->done_blocks = 0;
        acc->total_tokens = (long long)global;
        acc->objective = 0.0;
        acc->need_fixup = 0;
        if (DRAW) {
            const long long qhi = (first != INT_MAX && !frozen) ? __ldcg(&gc->gen_hi) : s_genhi;
            const long long qn = s_q;
            r->q_state = qn;
            r->idx = s_idx;
            r->q_hi = qhi > qn ? qhi : qn;
        }
        gc->ticket = 0;
        gc->done = 0;
        gc->gsum = 0;
        gc->first_rej = INT_MAX;
    }
    __syncthreads();
    if (DRAW && first != INT_MAX && !frozen && s_q > __ldcg(&gc->gen_hi)) {  // replay went past the ring
        uint64_t* dst = r->blk[s_q % MT_KR];
        for (int i = threadIdx.x; i < MT_N; i += blockDim.x) dst[i] = mt[i];
    }
    for (int c = threadIdx.x; c < nmap; c += blockDim.x) gc->word[c] = 0;
    if (DRAW && a.early) {
        __syncthreads();
        if (threadIdx.x == 0) st_release_i32(&gc->fin, 1);  // every unit is final
    }
}

// Map phase after k_sample_without (selections already drawn).
__global__ void __launch_bounds__(MAP_THREADS) k_sample_map(BufView v, SampleArgs a, GridCtl* gc,
                                                          const int* route_done) {
    __shared__ int s_t;
    RB_TSTART(3);
    if (threadIdx.x == 0) s_t = (int)atomicAdd(&gc->ticket, 1u);
    __syncthreads();
    const DrawCtx dc{};
    map_cta<false>(v, a, gc, s_t, dc, route_done);
    if (last_to_finish(gc)) map_finalize<false>(v, a, gc, (int)gridDim.x, dc, nullptr, route_done);
    RB_TEND(3);
}

// ---- fused uniform_with_replacement sampler: ticket 0 is the ring
// generator (twists the blocks this call needs that are not resident yet,
// publishing progress block by block, then as many again ahead for the next
// call); tickets 1.. are map CTAs with their own draws, which wait for the
// route kernel's completion flag (the metadata they map).  Launched as a
// programmatic dependent of the payload copy, so it overlaps the insert;
// griddepcontrol.wait at the end keeps "this kernel complete => the copy
// complete" for the gather that follows.
__device__ void gen_role(MtRing* r, const SampleArgs& a, GridCtl* gc) {
    const long long q0 = r->q_state, qhi0 = r->q_hi;
    const uint32_t idx0 = r->idx;
    const unsigned long long D = (unsigned long long)a.nsel;
    const long long need = q0 + (long long)((idx0 + D + MT_N - 1) / MT_N);
    // this call's blocks only (a first call, or a larger batch than the
    // lookahead planned for); the next call's come from the Rng's lookahead
    // (or, with RB_NO_LOOKAHEAD, from here: as many again ahead)
    long long target = a.gen_ahead ? need + (need - q0) + 1 : need;
    if (target > q0 + MT_KR - 1) target = q0 + MT_KR - 1;
    if (target > qhi0 && threadIdx.x < 32) {  // one warp, the block in registers
        const int l = threadIdx.x;
        uint64_t w[10];
        const uint64_t* src = r->blk[qhi0 % MT_KR];
#pragma unroll
        for (int k = 0; k < 10; ++k) w[k] = (l + 32 * k < MT_N) ? src[l + 32 * k] : 0;
        for (long long q = qhi0 + 1; q <= target; ++q) {
            mt_twist_warp(w);
            uint64_t* dst = r->blk[q % MT_KR];
#pragma unroll
            for (int k = 0; k < 10; ++k)
                if (l + 32 * k < MT_N) dst[l + 32 * k] = w[k];
        }
    }
    if (threadIdx.x == 0) gc->gen_hi = target > qhi0 ? target : qhi0;
}

__global__ void __launch_bounds__(MAP_THREADS, 4) k_sample_fused(BufView v, MtRing* r, SampleArgs a,
                                                                 GridCtl* gc, const int* route_done) {
    __shared__ int s_t;
    // the early-gather flags (seg, fin) start clear: reset by the early
    // gather that consumed them, or by the host before this launch
    pdl_trigger();  // the early gather may launch (it waits for the flags)
    if (threadIdx.x == 0) s_t = (int)atomicAdd(&gc->ticket, 1u);
    const DrawCtx dc{r, r->q_state, r->q_hi, r->idx};
    __syncthreads();
    const int t = s_t;
    if (t == 0) {
        RB_TSTART(6);
        gen_role(r, a, gc);
        RB_TEND(6);
    } else {
        RB_TSTART(3);
        RB_GCLOCK(40, t == 1);
        map_cta<true>(v, a, gc, t - 1, dc, route_done);
        RB_TEND(3);
    }
    if (last_to_finish(gc)) {
        RB_GCLOCK(58, true);
        map_finalize<true>(v, a, gc, (int)gridDim.x - 1, dc, r, route_done);
        RB_GCLOCK(59, true);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ uint64_t mt_below_scalar(uint64_t* mt, uint32_t* idx,
                                                    uint64_t* draws, long long* tw,
                                                    uint64_t bound) {
    const uint64_t lim = below_limit(bound);
    uint64_t x;
    do {
        if (*idx >= MT_N) {
            mt_twist_scalar(mt);
            *idx = 0;
            ++*tw;
        }
        ++*draws;
        x = mt_temper(mt[(*idx)++]);
    } while (x >= lim);
    return x % bound;
}

// uniform_without_replacement / unused_first_without_replacement
// (replay_buffer.cpp:146-179): sequential partial Fisher-Yates over the
// arrival indices with the reference's exact draw consumption.
__global__ void k_sample_without(BufView v, MtRing* r, SampleArgs a, int strategy,
                                 int64_t* scratch /* >= 2*C */) {
    __shared__ uint64_t mt[MT_N];
    __shared__ uint32_t s_idx;
    __shared__ uint64_t s_draws;
    __shared__ long long s_tw;
    const long long q0 = r->q_state;
    ring_load_block(r, q0, mt);
    if (threadIdx.x == 0) {
        uint32_t idx = r->idx;
        uint64_t draws = r->draws;
        long long tw = 0;
        long long pos = 0;
        int64_t* perm = scratch;
        int64_t* used = scratch + v.C;
        for (int s = 0; s < a.nsh; ++s) {
            const long long n = occupancy(v, s), k = a.per;
            long long picked = 0;
            if (strategy == RB_UNUSED_FIRST_WITHOUT_REPLACEMENT) {
                for (long long i = n - 1; i >= 0 && picked < k; --i) {
                    const size_t g = (size_t)s * v.C + arrival_slot(v, s, i);
                    if (v.use[g] == 0) {
                        a.sel_shard[pos + picked] = s;
                        a.sel_index[pos + picked] = i;
                        ++picked;
                    }
                }
                if (picked == k) {
                    pos += k;
                    continue;
                }
            }
            // population: all arrival indices, or the used ones (ascending)
            long long m = 0;
            if (strategy == RB_UNUSED_FIRST_WITHOUT_REPLACEMENT) {
                for (long long i = 0; i < n; ++i) {
                    const size_t g = (size_t)s * v.C + arrival_slot(v, s, i);
                    if (v.use[g] != 0) used[m++] = i;
                }
            } else {
                for (long long i = 0; i < n; ++i) used[m++] = i;
            }
            for (long long i = 0; i < m; ++i) perm[i] = i;
            const long long need = k - picked;
            for (long long i = 0; i < need; ++i) {
                const long long jj =
                    i + (long long)mt_below_scalar(mt, &idx, &draws, &tw, (uint64_t)(m - i));
                const int64_t t = perm[i];
                perm[i] = perm[jj];
                perm[jj] = t;
                a.sel_shard[pos + picked + i] = s;
                a.sel_index[pos + picked + i] = used[perm[i]];
            }
            pos += k;
        }
        s_idx = idx;
        s_draws = draws;
        s_tw = tw;
    }
    __syncthreads();
    ring_store_state(r, mt, q0, s_tw, s_idx, s_draws);
}

// priority_with_replacement (builder extension, no reference counterpart;
// SURVEY.md §8e): per shard, in shard order, `per` draws with probability
// w_i / W over the arrival indices, w_i = prio_weight (integer, so the CDF is
// exact and order-independent), each draw x = below(W) with the reference's
// rejection rule (rng.cpp:40-51) and index = upper_bound(cdf, x).  With every
// weight 1 it is pick_indices' uniform_with_replacement (replay_buffer.cpp:
// 141-145) draw for draw.  One CTA: the CDF is a block scan in chunks, the
// draws take one MT word per thread (a block scan of the accept flags ranks
// them, so a rejected word shifts the later draws exactly as the serial
// loop does), then one binary search per draw over the CDF (L2-resident).
constexpr int PR_THREADS = 1024;
__device__ __forceinline__ unsigned long long prio_weight(const BufView& v, size_t g,
                                                          const PrioParams& p) {
    double a = fabs(v.adv[g]);
    if (!(a <= 32768.0)) a = a > 32768.0 ? 32768.0 : 0.0;  // clamp; NaN -> 0
    unsigned long long w = (unsigned long long)p.base +
                           (unsigned long long)__dmul_rn(a, (double)p.adv_scale);
    if (p.pos_bonus != 0 && v.reward[g] > 0.0) w += p.pos_bonus;
    return w;
}
// CDF of up to PR_SMEM_CDF records in dynamic shared memory (the searches
// are then shared-memory round trips), else in global scratch.  The draws
// read MT words from the stream's ring (the Rng's twisted-ahead blocks);
// missing blocks are twisted into the ring by the whole CTA a chunk ahead
// (ring_extend: a one-warp twist chain was 3/4 of the kernel at 14 blocks).  A chunk is PR_R consecutive words per
// thread: the accept flags (x < below_limit(W)) are ranked by one block
// scan, so a rejected word shifts the later draws exactly as rng.cpp:40-51's
// loop does.
constexpr int PR_SMEM_CDF = 22528;  // 187 KB padded
constexpr int PR_G = 4096;          // guide-table buckets (16 KB)
// CDF word i lives at i + i / 16 (one pad word per 16: per-thread runs of 16
// read distinct banks)
__host__ __device__ __forceinline__ long long pr_pad(long long i) { return i + (i >> 4); }
constexpr int PR_R = 4;
constexpr long long PR_CH = (long long)PR_THREADS * PR_R;  // words per chunk
constexpr int PR_MS = 64;  // all-shards-at-once path: at most this many shards
template <bool SM>
__global__ void __launch_bounds__(PR_THREADS) k_sample_prio(BufView v, MtRing* r, SampleArgs a,
                                                            PrioParams p,
                                                            unsigned long long* g_cdf,
                                                            long long cdf_cap /* >= C */) {
    extern __shared__ unsigned long long s_cdf[];  // [pr_pad(cap)] cdf, then [PR_G] int32 guide
    __shared__ uint64_t s_mt[MT_N];
    __shared__ long long s_consumed;
    unsigned long long* cdf = SM ? s_cdf : g_cdf;
    int* guide = reinterpret_cast<int*>(cdf + pr_pad(cdf_cap));
    RB_GCLOCK(8, true);
    // a rejected asynchronous insert before this call (sticky error): no
    // draws, the stream position unchanged; k_sample_map (chk_frozen) maps
    // an empty batch, as the fused uniform sampler does
    if (*(volatile const int*)&v.ctl->err_code != 0) {
        for (long long i = threadIdx.x; i < a.nsel; i += PR_THREADS) {  // in-range, never mapped
            a.sel_shard[i] = 0;
            a.sel_index[i] = 0;
        }
        return;
    }
    const long long q0 = r->q_state;
    const uint32_t idx0 = r->idx;
    const uint64_t draws0 = r->draws;
    long long qhi = r->q_hi;  // block-uniform: twisted blocks are [q0, qhi]
    long long o = 0, pos = 0;  // words consumed past (q0, idx0); selections written
    // ring block holding word o + d (d < PR_CH), capped to what the ring holds
    auto chunk_target = [&](long long oo) {
        const long long first = q0 + ((long long)idx0 + oo) / MT_N;
        const long long last = q0 + ((long long)idx0 + oo + PR_CH - 1) / MT_N;
        return last < first + MT_KR - 1 ? last : first + MT_KR - 1;
    };
    // ---- several shards at once: one CDF over all their records (each
    // shard's values are differences from the prefix before it), per-shard
    // guide segments, and the draws taken as if no below() rejection occurs
    // (probability < W / 2^64 per draw), which the same pass verifies; any
    // rejection falls back to the shard-by-shard loop below (same ring).
    __shared__ long long s_base[PR_MS + 1];
    __shared__ unsigned long long s_pre[PR_MS], s_W[PR_MS], s_lim[PR_MS], s_mag[PR_MS];
    __shared__ int s_head[PR_MS], s_sh[PR_MS], s_G[PR_MS], s_flag;
    const long long D = (long long)a.nsh * a.per;
    if (SM && a.nsh > 1 && a.nsh <= PR_MS && D <= 60000) {
        const int T = a.nsh;
        if (threadIdx.x < T) {
            s_base[threadIdx.x + 1] = occupancy(v, threadIdx.x);
            s_head[threadIdx.x] = shard_head(v, threadIdx.x);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_base[0] = 0;
            for (int t = 0; t < T; ++t) s_base[t + 1] += s_base[t];
            s_flag = 0;
        }
        __syncthreads();
        const long long M = s_base[T], k = a.per;
        auto shard_of = [&](long long g) {  // last t with s_base[t] <= g
            int lo = 0, hi = T;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_base[mid] <= g) lo = mid;
                else hi = mid;
            }
            return lo;
        };
        if (M <= cdf_cap) {
#pragma unroll 4
            for (long long g = threadIdx.x; g < M; g += PR_THREADS) {
                const int t = shard_of(g);
                const long long i = g - s_base[t];
                cdf[pr_pad(g)] = prio_weight(
                    v, (size_t)t * v.C + arrival_slot_h(v, t, i, s_head[t]), p);
            }
            __syncthreads();
            const long long per = (M + PR_THREADS - 1) / PR_THREADS;
            const long long i0 = threadIdx.x * per, i1 = i0 + per < M ? i0 + per : M;
            long long run = 0;
            for (long long i = i0; i < i1; ++i) run += (long long)cdf[pr_pad(i)];
            long long tot;
            long long acc = block_exclusive_scan(run, &tot);
            for (long long i = i0; i < i1; ++i) {
                acc += (long long)cdf[pr_pad(i)];
                cdf[pr_pad(i)] = (unsigned long long)acc;
            }
            __syncthreads();
            const int gbits = 31 - __clz(PR_G / T);  // guide buckets per shard: 2^gbits
            if (threadIdx.x < T) {
                const int t = threadIdx.x;
                const unsigned long long pre = s_base[t] ? cdf[pr_pad(s_base[t] - 1)] : 0;
                const unsigned long long W = cdf[pr_pad(s_base[t + 1] - 1)] - pre;
                s_pre[t] = pre;
                s_W[t] = W;
                s_lim[t] = below_limit(W);
                s_mag[t] = UINT64_MAX / W;  // fast_mod's reciprocal (one division per shard)
                s_sh[t] = max(0, 64 - __clzll((long long)W) - gbits);
                s_G[t] = (int)((W - 1) >> s_sh[t]) + 1;
            }
            __syncthreads();
            for (long long g = threadIdx.x; g < M; g += PR_THREADS) {
                const int t = shard_of(g);
                const long long i = g - s_base[t];
                const unsigned long long prev = (i ? cdf[pr_pad(g - 1)] : s_pre[t]) - s_pre[t];
                const unsigned long long cur = cdf[pr_pad(g)] - s_pre[t];
                const int sh = s_sh[t];
                const unsigned long long msk = (1ULL << sh) - 1;
                const int b0 = (int)((prev + msk) >> sh), b1 = (int)((cur + msk) >> sh);
                for (int b = b0; b < b1 && b < s_G[t]; ++b) guide[(t << gbits) + b] = (int)i;
            }
            __syncthreads();
            for (long long c = 0; c < D; c += PR_CH) {
                const long long tgt = chunk_target(c);
                if (tgt > qhi) {
                    ring_extend(r, s_mt, qhi, tgt);  // ends with a CTA barrier
                    qhi = tgt;
                }
#pragma unroll
                for (int j = 0; j < PR_R; ++j) {
                    const long long d = c + (long long)threadIdx.x * PR_R + j;
                    if (d >= D) continue;
                    const long long gw = (long long)idx0 + d;
                    const uint64_t x = mt_temper(__ldcg(&r->blk[(q0 + gw / MT_N) % MT_KR][gw % MT_N]));
                    const int t = (int)(d / k);
                    if (x >= s_lim[t]) {
                        s_flag = 1;
                        continue;
                    }
                    const unsigned long long xr = fast_mod(x, s_W[t], s_mag[t]), pre = s_pre[t];
                    const int b = (int)(xr >> s_sh[t]);
                    int lo = guide[(t << gbits) + b];
                    int hi = b + 1 < s_G[t] ? guide[(t << gbits) + b + 1]
                                            : (int)(s_base[t + 1] - s_base[t]);
                    const long long bt = s_base[t];
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (cdf[pr_pad(bt + mid)] - pre > xr) hi = mid;
                        else lo = mid + 1;
                    }
                    a.sel_shard[d] = t;
                    a.sel_index[d] = lo;
                }
            }
            __syncthreads();
            if (!s_flag && !v.dbg_replay) {  // (tests: RB_DEBUG_FORCE_DRAW_REPLAY takes the fallback)
                if (threadIdx.x == 0) {
                    long long q = q0;
                    uint32_t idx = idx0;
                    ring_advance(q, idx, (unsigned long long)D);
                    r->q_state = q;
                    r->q_hi = qhi > q ? qhi : q;
                    r->idx = idx;
                    r->draws = draws0 + (uint64_t)D;
                }
                return;
            }
            // a rejection: the exact shard-by-shard loop (the ring blocks stay)
        }
    }
    for (int s = 0; s < a.nsh; ++s) {
        const long long n = occupancy(v, s), k = a.per;
        const int head = shard_head(v, s);
        // weights in arrival order (oldest first), coalesced, 8 loads in flight
        // (fused into the scan loop below they were not hoisted past the
        // shuffles: 12.6 vs 5.4 us at 16384 records)
#pragma unroll 8
        for (long long i = threadIdx.x; i < n; i += PR_THREADS)
            cdf[pr_pad(i)] = prio_weight(v, (size_t)s * v.C + arrival_slot_h(v, s, i, head), p);
        __syncthreads();
        RB_GCLOCK(9, s == 0);
        // inclusive scan: a contiguous run per thread in registers (the CDF is
        // padded one word per 16, so the runs' strided reads are free of bank
        // conflicts — unpadded they were 32-way, 26 us at 16384 records; a
        // warp-segment shuffle scan took 10 us), one block scan of the run sums
        const long long per = (n + PR_THREADS - 1) / PR_THREADS;
        const long long i0 = threadIdx.x * per, i1 = i0 + per < n ? i0 + per : n;
        long long run = 0;
        for (long long i = i0; i < i1; ++i) run += (long long)cdf[pr_pad(i)];
        long long W;
        long long acc = block_exclusive_scan(run, &W);
        for (long long i = i0; i < i1; ++i) {
            acc += (long long)cdf[pr_pad(i)];
            cdf[pr_pad(i)] = (unsigned long long)acc;
        }
        __syncthreads();
        // guide table: bucket b of values [b << sh, (b + 1) << sh) starts at the
        // record holding value b << sh (each record writes the buckets whose
        // first value it holds: they partition [0, W)), so a search is over
        // [guide[b], guide[b + 1]] — usually one or two records
        const int sh = max(0, 64 - __clzll((long long)W) - 12);  // W >> sh < PR_G
        const int G = (int)(((uint64_t)W - 1) >> sh) + 1;
        const unsigned long long msk = (1ULL << sh) - 1;
        for (long long i = threadIdx.x; i < n; i += PR_THREADS) {
            const unsigned long long prev = i ? cdf[pr_pad(i - 1)] : 0;
            const int b0 = (int)((prev + msk) >> sh), b1 = (int)((cdf[pr_pad(i)] + msk) >> sh);
            for (int b = b0; b < b1 && b < G; ++b) guide[b] = (int)i;
        }
        __syncthreads();
        RB_GCLOCK(10, s == 0);
        const uint64_t lim = below_limit((uint64_t)W);
        const uint64_t mag = UINT64_MAX / (uint64_t)W;  // x % W by multiply-high (fast_mod)
        long long got = 0;
        while (got < k) {
            const long long tgt = chunk_target(o);
            if (tgt > qhi) {
                ring_extend(r, s_mt, qhi, tgt);  // ends with a CTA barrier
                qhi = tgt;
            }
            RB_GCLOCK(11, s == 0 && got == 0);
            const long long ow = o + (long long)threadIdx.x * PR_R;
            uint64_t x[PR_R];
            unsigned okm = 0;
#pragma unroll
            for (int j = 0; j < PR_R; ++j) {
                const long long gw = (long long)idx0 + ow + j;
                const long long q = q0 + gw / MT_N;
                x[j] = mt_temper(__ldcg(&r->blk[q % MT_KR][gw % MT_N]));
                if (x[j] < lim) okm |= 1u << j;
            }
            const int cnt = __popc(okm);
            long long nacc;
            long long rank = block_exclusive_scan(cnt, &nacc);
            const long long need = k - got;
            if (threadIdx.x == 0) s_consumed = PR_CH;
            __syncthreads();
            RB_GCLOCK(12, s == 0 && got == 0);
            // the PR_R searches advance together (ILP): upper_bound over the
            // guide bucket's records [guide[b], guide[b + 1]]
            int lo[PR_R], hi[PR_R];
            uint64_t xr[PR_R];
#pragma unroll
            for (int j = 0; j < PR_R; ++j) {
                const bool ok = (okm >> j) & 1u;
                if (ok && rank == need - 1) s_consumed = (long long)threadIdx.x * PR_R + j + 1;
                const bool take = ok && rank < need;
                xr[j] = take ? fast_mod(x[j], (uint64_t)W, mag) : 0;
                const int b = (int)(xr[j] >> sh);
                lo[j] = take ? guide[b] : 0;
                hi[j] = !take ? 0 : (b + 1 < G ? guide[b + 1] : (int)n);
                rank += ok ? 1 : 0;
            }
            RB_GCLOCK(13, s == 0 && got == 0);
            for (bool more = true; more;) {
                more = false;
#pragma unroll
                for (int j = 0; j < PR_R; ++j) {
                    if (lo[j] < hi[j]) {
                        const int mid = (lo[j] + hi[j]) >> 1;
                        if (cdf[pr_pad(mid)] > xr[j]) hi[j] = mid;
                        else lo[j] = mid + 1;
                        more |= lo[j] < hi[j];
                    }
                }
            }
            RB_GCLOCK(15, s == 0 && got == 0);
            rank -= cnt;
#pragma unroll
            for (int j = 0; j < PR_R; ++j) {
                const bool ok = (okm >> j) & 1u;
                if (ok && rank < need) {
                    a.sel_shard[pos + got + rank] = s;
                    a.sel_index[pos + got + rank] = lo[j];
                }
                rank += ok ? 1 : 0;
            }
            __syncthreads();
            o += s_consumed;
            got += nacc < need ? nacc : need;
            __syncthreads();
        }
        pos += k;
        RB_GCLOCK(14, s == 0);
    }
    if (threadIdx.x == 0) {
        long long q = q0;
        uint32_t idx = idx0;
        ring_advance(q, idx, (unsigned long long)o);
        r->q_state = q;
        r->q_hi = qhi > q ? qhi : q;
        r->idx = idx;
        r->draws = draws0 + (uint64_t)o;
    }
}

// Per-shard priority mass W_s (uint64, exact, order-free): one CTA per owned
// shard.  The all-reduce of these T-vectors over the ranks is the global
// priority mass (rb_allreduce_priority_mass).
__global__ void __launch_bounds__(256) k_prio_mass(BufView v, PrioParams p,
                                                   unsigned long long* out) {
    const int s = v.sb + (int)blockIdx.x;
    const long long n = occupancy(v, s);
    const int head = shard_head(v, s);
    unsigned long long w = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x)
        w += prio_weight(v, (size_t)s * v.C + arrival_slot_h(v, s, i, head), p);
#pragma unroll
    for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    __shared__ unsigned long long s_w[8];
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += s_w[k];
        out[s] = t;
    }
}

// ---------------------------------------------------------------- FIFO route
// FIFO routing + eviction + group advantages + metadata scatter for ids
// promised new and increasing (replay_buffer.cpp:83-133 in closed form;
// bandit.cpp:276-294 per group), one record per thread, no grid barrier:
// every CTA validates the whole batch itself (lengths, id order, group
// offsets; ~16 B per record from L2) so it may apply its own records at
// once, each record recomputes its group's statistics (the reference's
// sequential fp64 order; the group's rewards are register-resident), and
// the last CTA to finish advances the per-shard counters.  Nothing is
// applied if the batch is invalid (the error is sticky until rb_check).
#ifndef RB_RT_THREADS
#define RB_RT_THREADS 256
#endif
constexpr int RT_THREADS = RB_RT_THREADS;  // one record per thread; 256 measured ~0.5-1 µs better than 128
constexpr int RT_NSH = 256;
constexpr int RT_GOFF = 2048;
constexpr int GR = 16;  // rewards per register batch
__device__ __forceinline__ void group_adv_one(const double* rw, long long b, long long e,
                                              double rj, double* adv, double* mean_out) {
    const long long m = e - b;
    const double dn = (double)m;
    double mean = 0.0, var = 0.0;
    if (m <= GR) {
        double r[GR];
#pragma unroll
        for (int k = 0; k < GR; ++k) r[k] = k < m ? rw[b + k] : 0.0;
#pragma unroll
        for (int k = 0; k < GR; ++k)
            if (k < m) mean = __dadd_rn(mean, r[k]);
        mean = __ddiv_rn(mean, dn);
#pragma unroll
        for (int k = 0; k < GR; ++k)
            if (k < m) {
                const double d = __dsub_rn(r[k], mean);
                var = __dadd_rn(var, __dmul_rn(d, d));
            }
    } else {
        for (long long k = b; k < e; ++k) mean = __dadd_rn(mean, rw[k]);
        mean = __ddiv_rn(mean, dn);
        for (long long k = b; k < e; ++k) {
            const double d = __dsub_rn(rw[k], mean);
            var = __dadd_rn(var, __dmul_rn(d, d));
        }
    }
    var = __ddiv_rn(var, dn);
    const double sd = __dsqrt_rn(var);
    // bandit.cpp:289-292: zeros when the population std < 1e-8
    *adv = sd < 1e-8 ? 0.0 : __ddiv_rn(__dsub_rn(rj, mean), sd);
    *mean_out = mean;  // bandit.cpp:316-318 (same sequential sum)
}

// Batches above this size split the route's validation over its CTAs (at
// 1293 records the whole-batch sweep per CTA publishes the verdict ~2 µs
// sooner than the counter; at 8 GPUs' 10344 records it is ~7 µs later).
constexpr int RT_SPLIT_MIN = 4096;
#ifndef RB_RT_UNROLL
#define RB_RT_UNROLL 8
#endif
constexpr int RT_UNROLL = RB_RT_UNROLL;  // whole-batch validation sweep: records in flight per thread
constexpr int RT_KEEP = 1024;  // token offsets copied per extra route CTA

__global__ void __launch_bounds__(RT_THREADS) k_route_fifo(BufView v, InsertIn in, GridCtl* gc,
                                                          int* pay_sync) {
    __shared__ long long s_P[RT_NSH];
    __shared__ long long s_goff[RT_GOFF + 1];
    __shared__ int s_bad, s_last, s_m[RT_THREADS / 32];
    const int tid = threadIdx.x;
    const int n = (int)in.n;
    const long long ng = in.ngroups;
    DevCtl* ctl = v.ctl;
    RB_TSTART(0);
    RB_GCLOCK(30, blockIdx.x == 0);
    // This insert's flags (verdict, done; the copy's completion) carry its
    // epoch: the dependents wait for the epoch, so nothing is reset here.
    const int E = in.epoch;
    RB_GCLOCK(31, blockIdx.x == 0);
    pdl_trigger();  // the closed-form payload copy may start now (it waits for the verdict)
    // the route proper runs on the first nrt CTAs
    const unsigned nrt = gridDim.x - (in.toff_keep ? (unsigned)in.keep_ctas : 0u);
    if (blockIdx.x >= nrt) {
        // Extra CTAs (RT_KEEP offsets each, all loads in flight): the caller
        // may reuse its offsets as soon as later stream work runs, but an
        // overlapping sampler reads the new records' lengths after this
        // call: keep a copy, published by a monotonic counter (the sampler
        // waits for its target).  The previous insert's sampler may still
        // read the copy area: written after the wait.
        pdl_wait();
        const int base = (int)(blockIdx.x - nrt) * RT_KEEP + tid;
        int64_t t[RT_KEEP / RT_THREADS];
#pragma unroll
        for (int k = 0; k < RT_KEEP / RT_THREADS; ++k) {
            const int i = base + k * RT_THREADS;
            t[k] = i <= n ? in.toff[i] : 0;
        }
#pragma unroll
        for (int k = 0; k < RT_KEEP / RT_THREADS; ++k) {
            const int i = base + k * RT_THREADS;
            if (i <= n) in.toff_keep[i] = t[k];
        }
        __syncthreads();
        if (tid == 0)
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(in.keep_cnt) : "memory");
        return;
    }
    // ---- before the wait: the caller's batch only (when launched as a
    // programmatic dependent of the previous step's sampler or loss, this
    // overlaps its tail; nothing of the buffer is read or written yet)
    if (tid == 0) s_bad = 0;
    const bool goff_smem = !in.adv && ng <= RT_GOFF;
    if (goff_smem)
        for (long long gi = tid; gi <= ng; gi += RT_THREADS) s_goff[gi] = in.goff[gi];
    // own record (all loads issued before the validation sweep)
    const int j = blockIdx.x * RT_THREADS + tid;
    const bool mine = j < n;
    uint64_t id = 0, prompt = 0, group = 0;
    int64_t cstep = 0, pver = 0;
    double reward = 0.0, blp = 0.0, adv = 0.0, gmean = 0.0;
    bool correct = false;
    long long off0 = 0, len = 0;
    if (mine) {
        id = in.id[j];
        prompt = in.prompt ? in.prompt[j] : 0;
        group = in.group ? in.group[j] : 0;
        cstep = in.cstep ? in.cstep[j] : 0;
        pver = in.pver ? in.pver[j] : 0;
        reward = in.reward[j];
        correct = in.correct ? in.correct[j] != 0 : reward == 1.0;
        blp = in.blp ? in.blp[j] : 0.0;
        if (in.adv) {
            adv = in.adv[j];
            gmean = in.gmean ? in.gmean[j] : 0.0;
        }
        if (in.toff) {
            off0 = in.toff[j];
            len = in.toff[j + 1] - off0;
        }
    }
    // whole-batch validation (replay_buffer.cpp:85-88 order: nothing applied).
    // Up to RT_SPLIT_MIN records every CTA sweeps the whole batch and reaches
    // the verdict alone; larger batches (many GPUs: the metadata of every
    // shard's records) split it: each CTA checks its own records and a stride
    // of the groups, the last CTA to finish ORs the bits and publishes the
    // verdict, the others wait for it.  The first id's check against the
    // buffer's largest id comes after the wait.
    const bool split = in.split_validate != 0;
    int bad = 0;
    if (split) {
        if (mine) {
            if (in.toff && (len < 0 || len > in.maxlen)) bad |= 2;
            if (j > 0 && id <= in.id[j - 1]) bad |= 1;
        }
        if (!in.adv) {
            if (blockIdx.x == 0 && tid == 0 && (in.goff[0] != 0 || in.goff[ng] != n)) bad |= 4;
            for (long long gi = (long long)blockIdx.x * RT_THREADS + tid; gi < ng;
                 gi += (long long)nrt * RT_THREADS) {
                const long long b = in.goff[gi], e = in.goff[gi + 1];
                if (e - b < 2 || b < 0 || e > n) bad |= 4;
            }
        }
    } else {
#pragma unroll (RT_UNROLL)
        for (int jj = tid; jj < n; jj += RT_THREADS) {
            if (in.toff) {
                const long long l = in.toff[jj + 1] - in.toff[jj];
                if (l < 0 || l > in.maxlen) bad |= 2;
            }
            if (jj > 0 && in.id[jj] <= in.id[jj - 1]) bad |= 1;
        }
        if (!in.adv) {
            if (tid == 0 && (in.goff[0] != 0 || in.goff[ng] != n)) bad |= 4;
            for (long long gi = tid; gi < ng; gi += RT_THREADS) {
                const long long b = in.goff[gi], e = in.goff[gi + 1];
                if (e - b < 2 || b < 0 || e > n) bad |= 4;
            }
        }
    }
    const uint64_t id0 = n > 0 ? in.id[0] : 0;
    __syncthreads();  // s_bad and s_goff written
    // group advantages of the own record (bandit.cpp:276-294), from the batch
    if (mine && !in.adv && !bad) {
        long long lo = 0, hi = ng;  // group gi: goff[gi] <= j < goff[gi+1]
        while (hi - lo > 1) {
            const long long mid = (lo + hi) >> 1;
            const long long gm = goff_smem ? s_goff[mid] : in.goff[mid];
            if (gm <= j) lo = mid;
            else hi = mid;
        }
        const long long b = goff_smem ? s_goff[lo] : in.goff[lo];
        const long long e = goff_smem ? s_goff[lo + 1] : in.goff[lo + 1];
        if (e - b >= 2 && b >= 0 && e <= n) group_adv_one(in.reward, b, e, reward, &adv, &gmean);
    }
    // ---- the buffer's state: after the previous kernel (if a programmatic
    // dependency) has completed
    pdl_wait();
    const int sticky = ctl->err_code;
    const unsigned long long cur0 = ctl->cursor;
    RB_GCLOCK(32, blockIdx.x == 0);  // (debug builds: after the control-block loads are issued)
    const int has_any = ctl->has_any;
    const unsigned long long max_id = ctl->max_id;
    const int T = v.T, C = v.C;
    const int c0 = (int)(cur0 % (unsigned long long)T);
    for (int s = tid; s < T && s < RT_NSH; s += RT_THREADS) s_P[s] = v.pushes[s];
    if (sticky) bad |= 8;
    if (tid == 0 && (split ? blockIdx.x == 0 : true) && n > 0 && has_any && id0 <= max_id) bad |= 1;
    RB_GCLOCK(60, blockIdx.x == 0);
    if (bad) atomicOr(&s_bad, bad);
    __syncthreads();
    if (split) {
        if (tid == 0) {
            if (s_bad) atomicOr(&gc->vbad, (unsigned)s_bad);
            if (done_add_u32(&gc->vdone) == nrt - 1) {  // acquires every CTA's bits
                const int vb = (int)atomicOr(&gc->vbad, 0u);
                s_bad = vb;
                st_release_i32(&pay_sync[0], E << 2 | (vb ? 2 : 1));
            } else {
                const int f = spin_epoch(&pay_sync[0], E);
                s_bad = f == 2 ? (int)__ldcg(&gc->vbad) : 0;
            }
        }
        __syncthreads();
    }
    RB_GCLOCK(61, blockIdx.x == 0);
    const int bb = s_bad;
    // unsplit: every CTA reached the same verdict; CTA 0 alone publishes it
    if (!split && blockIdx.x == 0 && tid == 0) st_release_i32(&pay_sync[0], E << 2 | (bb ? 2 : 1));
    // no payload copy follows: its completion flag is trivially this insert's
    if (!in.pay_follows && blockIdx.x == 0 && tid == 0) st_release_i32(&pay_sync[2], E << 2 | 2);
    int maxq = 0;
    if (mine) {
        int32_t slot = -1;
        uint8_t surv = 0;
        uint64_t ev = NONE_ID;
        bool ev_by_survivor = false;
        Unit d;
        d.row = -1;
        d.len = (int32_t)(len < 0 ? 0 : len);
        d.k0 = 0;
        d.g = j;
        d.off = off0;
        d.adv = 0.0;
        if (!bb) {
            int s = c0 + j % T;
            if (s >= T) s -= T;
            int rank = j / T, j0 = j % T;
            int ns = (n - 1 - j0) / T + 1;
            // owned-metadata batch: record j is the owned shard's j-th push
            // (its records only; an evictee of this batch is record j - C)
            const int jst = in.own_only ? 1 : T;
            if (in.own_only) {
                s = v.sb;
                rank = j;
                j0 = 0;
                ns = n;
            }
            const long long P = s < RT_NSH ? s_P[s] : v.pushes[s];
            int x2 = (int)(P % C) + rank % C;
            if (x2 >= C) x2 -= C;
            const size_t g = (size_t)s * C + (size_t)x2;
            slot = (int32_t)g;
            surv = rank + C >= ns;
            // The id a push evicts: an earlier record of this batch, or the
            // slot's resident one.  A slot pushed again later in this batch
            // is overwritten by its survivor (another CTA): that survivor
            // reports the resident id for the slot's first push instead
            // (read before its own write, same thread).
            if (P + rank >= C) ev = rank >= C ? in.id[j - C * jst] : v.id[g];
            if (rank < C && !surv) ev_by_survivor = true;
            if (surv && rank >= C) {
                const int r0 = rank % C;
                in.evid[r0 * jst + j0] = P + r0 >= C ? v.id[g] : NONE_ID;
            }
            // (advantages: computed from the batch before the wait)
            if (surv) {
                v.id[g] = id;
                v.prompt[g] = prompt;
                v.group[g] = group;
                v.cstep[g] = cstep;
                v.pver[g] = pver;
                v.reward[g] = reward;
                v.correct[g] = correct;
                v.blp[g] = blp;
                v.adv[g] = adv;
                v.gmean[g] = gmean;
                v.use[g] = 0;
                v.len[g] = (int32_t)len;
                if (s >= v.sb && s < v.se && len > 0 && v.stride > 0) {
                    d.row = (s - v.sb) * C + x2;
                    maxq = (int)((len + 3) >> 2);
                }
            }
        }
        in.len[j] = (int32_t)(len < 0 ? 0 : len);
        in.tslot[j] = slot;
        in.surv[j] = surv;
        if (!ev_by_survivor) in.evid[j] = ev;
        in.adv_out[j] = adv;
        in.gmean_out[j] = gmean;
        in.units[j] = d;
    }
    RB_GCLOCK(62, blockIdx.x == 0);
    maxq = __reduce_max_sync(0xffffffffu, maxq);
    if ((tid & 31) == 0) s_m[tid >> 5] = maxq;
    __syncthreads();
    if (tid == 0) {
        int m = 0;
        for (int w = 0; w < RT_THREADS / 32; ++w) m = s_m[w] > m ? s_m[w] : m;
        gc->cta_max[blockIdx.x] = m;
        s_last = done_add_u32(&gc->done) == nrt - 1;
    }
    __syncthreads();
    RB_GCLOCK(63, blockIdx.x == 0);
    if (!s_last) return;
    RB_GCLOCK(56, true);
    // last CTA: every CTA's records are written (each released by its done
    // increment, acquired by ours): the sampler's map may read the metadata
    // now; the counters below are not read by it (it uses the insert's plan)
    if (tid == 0) st_release_i32(&pay_sync[1], E << 2 | 1);
    int m = 0;
    for (int c = tid; c < (int)nrt; c += RT_THREADS) m = max(m, __ldcg(&gc->cta_max[c]));
    m = __reduce_max_sync(0xffffffffu, m);
    if ((tid & 31) == 0) s_m[tid >> 5] = m;
    const int nG = in.own_only ? (int)in.n_global : n;  // the global batch
    if (!bb)
        for (int s = tid; s < T; s += RT_THREADS) {
            const int j0 = ((s - c0) % T + T) % T;
            const int ns = nG > j0 ? (nG - 1 - j0) / T + 1 : 0;
            v.pushes[s] += ns;
        }
    __syncthreads();
    if (tid == 0) {
        int mm = 0;
        for (int w = 0; w < RT_THREADS / 32; ++w) mm = s_m[w] > mm ? s_m[w] : mm;
        *in.n_units = bb ? 0 : mm;
        if (!bb) {
            ctl->cursor = (cur0 + (unsigned long long)nG) % T;
            ctl->max_id = in.id[n - 1];  // strictly increasing and above the old max
            ctl->has_any = 1;
            ctl->hash_stale = 1;
        } else if (!sticky) {
            ctl->err_code = RB_EINVAL;
            ctl->err_index = (bb & 2) ? -3 : (bb & 4) ? -2 : -4;
        }
        gc->done = 0;
        gc->vdone = 0;
        gc->vbad = 0;
        RB_GCLOCK(57, true);
    }
    RB_TEND(0);
}

// ---- positive bias, ids promised new: one launch, one CTA per shard -------
// Replaces k_insert_route + k_posbias_batch for RB_INSERT_ASSUME_UNIQUE
// batches whose shard state fits shared memory (C <= PBP_CMAX, <= PBP_NSMAX
// pushes per shard).  Every CTA validates the whole batch itself (the
// reference's all-or-nothing order, replay_buffer.cpp:85-88) and computes
// its own records' group advantages (bandit.cpp:276-294, fp64, sequential
// order).  The queue update (replay_buffer.cpp:98-133 as F/W/Q queues, see
// pb_push_logic) runs in parallel once the shard is full:
//   * push k moves e_k — the k-th element of (F ++ batch) — from F into the
//     reserve (W if wrong, Q if correct) and then evicts W's head if W is
//     non-empty, else Q's head;
//   * |W| follows the Lindley recursion w_k = max(w_{k-1} + wrong_k - 1, 0),
//     whose prefix is a block scan of the max-plus maps w -> max(w + A, B)
//     ((A1,B1) then (A2,B2) = (A1+A2, max(B1+A2, B2)));
//   * the m-th W pop takes the m-th element of (W ++ wrong entries), the
//     m-th Q pop likewise (prefix counts), so every victim is known at once;
//   * a pushed record takes its victim's slot: chains through earlier pushes
//     of the batch are resolved by pointer jumping.
// While a shard is still filling (or fresh_slots == 0) thread 0 runs the
// O(1)-per-push simulation on the shared-memory rings instead.  Then, per
// shard in parallel: evicted ids, survivors' metadata, payload descriptors,
// rings rewritten from head 0, and the materialised arrival order
// (merge(W, Q) by arrival sequence, then F).
constexpr int PBP_THREADS = 1024;
constexpr int PBP_CMAX = 4096;
constexpr int PBP_NSMAX = 4096;
constexpr int PBP_NMAX = 65536;

struct MaxPlus {
    int a, b;  // w -> max(w + a, b)
};
__device__ __forceinline__ MaxPlus mp_then(MaxPlus x, MaxPlus y) {  // x first, then y
    return MaxPlus{x.a + y.a, max(x.b + y.a, y.b)};
}
// Block-wide exclusive scan of max-plus maps (identity {0, INT_MIN/2}),
// together with an exclusive sum of one int per thread (*cex; *ctot the total).
__device__ MaxPlus block_scan_mp(MaxPlus x, int c, int* cex, int* ctot) {
    __shared__ int s_a[32], s_b[32], s_c[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    MaxPlus inc = x;
    int ci = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const MaxPlus y{__shfl_up_sync(0xffffffffu, inc.a, o), __shfl_up_sync(0xffffffffu, inc.b, o)};
        const int yc = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) {
            inc = mp_then(y, inc);
            ci += yc;
        }
    }
    if (lane == 31) {
        s_a[wid] = inc.a;
        s_b[wid] = inc.b;
        s_c[wid] = ci;
    }
    __syncthreads();
    if (wid == 0) {
        MaxPlus w = lane < nw ? MaxPlus{s_a[lane], s_b[lane]} : MaxPlus{0, INT_MIN / 2};
        int wc = lane < nw ? s_c[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const MaxPlus y{__shfl_up_sync(0xffffffffu, w.a, o), __shfl_up_sync(0xffffffffu, w.b, o)};
            const int yc = __shfl_up_sync(0xffffffffu, wc, o);
            if (lane >= o) {
                w = mp_then(y, w);
                wc += yc;
            }
        }
        s_a[lane] = w.a;
        s_b[lane] = w.b;
        s_c[lane] = wc;
    }
    __syncthreads();
    const MaxPlus base = wid ? MaxPlus{s_a[wid - 1], s_b[wid - 1]} : MaxPlus{0, INT_MIN / 2};
    *cex = (wid ? s_c[wid - 1] : 0) + ci - c;
    *ctot = s_c[nw - 1];
    // exclusive within the warp: the inclusive value of the lane before
    MaxPlus ex{__shfl_up_sync(0xffffffffu, inc.a, 1), __shfl_up_sync(0xffffffffu, inc.b, 1)};
    if (lane == 0) ex = MaxPlus{0, INT_MIN / 2};
    __syncthreads();
    return mp_then(base, ex);
}

__global__ void __launch_bounds__(PBP_THREADS) k_posbias_par(BufView v, InsertIn in,
                                                             unsigned long long cur0,
                                                             GridCtl* gc, int nsp) {
    extern __shared__ __align__(16) unsigned char pbp_sm[];
    __shared__ long long s_goff[RT_GOFF + 1];
    __shared__ int s_maxq;
    __shared__ PbState s_st;
    const int s = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int T = v.T, C = v.C, RC = C + 1, fs = v.fs;
    DevCtl* ctl = v.ctl;
    const int n = (int)in.n;
    const long long ng = in.ngroups;
    const int j0 = (int)(((long long)s - (long long)(cur0 % (unsigned long long)T)) % T + T) % T;
    const int ns = n > j0 ? (n - 1 - j0) / T + 1 : 0;
    RB_TSTART(0);
    RB_GCLOCK(20, s == 0);
    // shared memory: preseq / preid [C] (i64), rings [3][RC], occb [C], per
    // push: vk, slotk, WE, QE (i32), cx, evw (u8)
    long long* preseq = reinterpret_cast<long long*>(pbp_sm);
    uint64_t* preid = reinterpret_cast<uint64_t*>(preseq + C);
    uint32_t* ring = reinterpret_cast<uint32_t*>(preid + C);
    int* occb = reinterpret_cast<int*>(ring + 3 * RC);
    int* vk = occb + C;       // victim of push k: -1 none, -2 itself, < C pre slot, C + k'' push k''
    int* slotk = vk + nsp;  // local slot of push k's record (-1: evicted on arrival)
    int* WE = slotk + nsp;  // wrong entries in order (element ids)
    int* QE = WE + nsp;     // correct entries in order
    uint8_t* cx = reinterpret_cast<uint8_t*>(QE + nsp);  // correctness of push k
    uint8_t* evw = cx + nsp;                             // push k pops W
    // ---- before the wait: the caller's batch only (a programmatic dependent
    // of the previous kernel: this overlaps its tail; the buffer is read and
    // written only after griddepcontrol.wait)
    const bool goff_smem = !in.adv && ng <= RT_GOFF;
    if (goff_smem)
        for (long long gi = tid; gi <= ng; gi += nt) s_goff[gi] = in.goff[gi];
    // whole-batch validation (nothing applied if any check fails); the first
    // id against the buffer's largest id after the wait
    int bad = 0;
    for (int jj = tid; jj < n; jj += nt) {
        if (in.toff) {
            const long long l = in.toff[jj + 1] - in.toff[jj];
            if (l < 0 || l > in.maxlen) bad |= 2;
        }
        if (jj > 0 && in.id[jj] <= in.id[jj - 1]) bad |= 1;
    }
    if (!in.adv) {
        if (tid == 0 && (in.goff[0] != 0 || in.goff[ng] != n)) bad |= 4;
        for (long long gi = tid; gi < ng; gi += nt) {
            const long long b = in.goff[gi], e = in.goff[gi + 1];
            if (e - b < 2 || b < 0 || e > n) bad |= 4;
        }
    }
    const uint64_t id0 = n > 0 ? in.id[0] : 0;
    const uint64_t idl = n > 0 ? in.id[n - 1] : 0;  // the buffer's new largest id
    __syncthreads();  // s_goff written
    // own records: lengths, advantages (frozen at insertion, bandit.cpp:276-294,
    // the reference's fp64 order), correctness — into the insert's own scratch
    // columns (no kernel before this one reads them)
    for (int k = tid; k < ns; k += nt) {
        const int j = j0 + k * T;
        const long long l = in.toff ? in.toff[j + 1] - in.toff[j] : 0;
        in.len[j] = (int32_t)l;
        double adv = 0.0, gmean = 0.0;
        if (in.adv) {
            adv = in.adv[j];
            gmean = in.gmean ? in.gmean[j] : 0.0;
        } else if (!bad) {
            long long lo = 0, hi = ng;
            while (hi - lo > 1) {
                const long long mid = (lo + hi) >> 1;
                const long long gm = goff_smem ? s_goff[mid] : in.goff[mid];
                if (gm <= j) lo = mid;
                else hi = mid;
            }
            const long long b = goff_smem ? s_goff[lo] : in.goff[lo];
            const long long e = goff_smem ? s_goff[lo + 1] : in.goff[lo + 1];
            if (e - b >= 2 && b >= 0 && e <= n) group_adv_one(in.reward, b, e, in.reward[j], &adv, &gmean);
        }
        in.adv_out[j] = adv;
        in.gmean_out[j] = gmean;
        cx[k] = in_correct(in, j) ? 1 : 0;
    }
    // ---- the buffer's state
    pdl_wait();
    RB_GCLOCK(29, s == 0);
    const int sticky = ctl->err_code;
    const int has_any = ctl->has_any;
    const unsigned long long max_id = ctl->max_id;
    const long long P0 = v.pushes[s];
    if (tid == 0) {
        s_st = v.pbs[s];
        s_maxq = 0;
        if (n > 0 && has_any && id0 <= max_id) bad |= 1;
    }
    for (int x = tid; x < C; x += nt) {
        preseq[x] = v.seq[(size_t)s * C + x];
        preid[x] = v.id[(size_t)s * C + x];
        occb[x] = -1;
    }
    const int bb = (sticky ? 8 : 0) | (__syncthreads_or(bad & 1) ? 1 : 0) |
                   (__syncthreads_or(bad & 2) ? 2 : 0) | (__syncthreads_or(bad & 4) ? 4 : 0);
    RB_GCLOCK(21, s == 0);
    if (bb) {  // frozen or rejected: nothing applied
        for (int k = tid; k < ns; k += nt) {
            const int j = j0 + k * T;
            in.surv[j] = 0;
            in.tslot[j] = -1;
            in.evid[j] = NONE_ID;
            Unit d{};
            d.row = -1;
            d.g = j;
            in.units[j] = d;
        }
        if (tid == 0 && done_add_u32(&gc->done) == (unsigned)T - 1) {
            *in.n_units = 0;
            if (!sticky) {
                ctl->err_code = RB_EINVAL;
                ctl->err_index = (bb & 2) ? -3 : (bb & 4) ? -2 : -4;
            }
            gc->done = 0;
        }
        return;
    }
    // the shard's rings (pre-batch heads, rebased to 0)
    const PbState st = s_st;
    uint32_t* gring[3] = {(uint32_t*)pb_ring(v, 0, s), (uint32_t*)pb_ring(v, 1, s),
                          (uint32_t*)pb_ring(v, 2, s)};
    for (int r = 0; r < 3; ++r)
        for (int i = tid; i < st.n[r]; i += nt) {
            int p = st.h[r] + i;
            if (p >= RC) p -= RC;
            ring[r * RC + i] = gring[r][p];
        }
    __syncthreads();
    RB_GCLOCK(22, s == 0);
    const int size0 = (int)(P0 < C ? P0 : C);
    const bool par = size0 == C && fs > 0 && st.n[0] == fs && ns > 0;
    const uint32_t* Fp = ring;
    const uint32_t* Wp = ring + RC;
    const uint32_t* Qp = ring + 2 * RC;
    const int w0 = st.n[1], q0 = st.n[2];
    // element e: < C a pre-batch record (its local slot), else push e - C
    PbState nst;
    if (par) {
        // 1. e_k = (F ++ batch)[k]; |W| by the max-plus scan; pops from W
        const int per = (ns + nt - 1) / nt;
        const int k0 = tid * per, k1 = min(ns, k0 + per);
        auto ent = [&](int k, bool* wrong) {
            if (k < fs) {
                const uint32_t x = Fp[k];
                *wrong = (x >> 31) == 0;
                return (int)(x & 0x7fffffffu);
            }
            *wrong = cx[k - fs] == 0;
            return C + (k - fs);
        };
        MaxPlus loc{0, INT_MIN / 2};
        int nwr = 0, npw = 0;
        for (int k = k0; k < k1; ++k) {
            bool wr;
            ent(k, &wr);
            loc = mp_then(loc, MaxPlus{wr ? 0 : -1, 0});
            nwr += wr;
        }
        int ew, tot_wr;  // wrong entries before k0, in all
        const MaxPlus pre = block_scan_mp(loc, nwr, &ew, &tot_wr);
        int w = max(w0 + pre.a, pre.b);
        for (int k = k0; k < k1; ++k) {
            bool wr;
            ent(k, &wr);
            const bool pw = w + (wr ? 1 : 0) >= 1;
            evw[k] = pw;
            npw += pw;
            w = max(w + (wr ? 0 : -1), 0);
        }
        long long tot_pw;
        int cw = (int)block_exclusive_scan(npw, &tot_pw);  // W pops before k0
        // 2. entries in order
        {
            int e_w = ew;
            for (int k = k0; k < k1; ++k) {
                bool wr;
                const int e = ent(k, &wr);
                if (wr) WE[e_w++] = e;
                else QE[k - e_w] = e;  // correct entries before k = k - wrong entries before k
            }
        }
        __syncthreads();
        // 3. victims
        {
            int c_w = cw;
            for (int k = k0; k < k1; ++k) {
                int e;
                if (evw[k]) {
                    const int m = c_w++;
                    e = m < w0 ? (int)(Wp[m] & 0x7fffffffu) : WE[m - w0];
                } else {
                    const int m = k - c_w;  // Q pops before k
                    e = m < q0 ? (int)(Qp[m] & 0x7fffffffu) : QE[m - q0];
                }
                vk[k] = e;
                slotk[k] = e;
            }
        }
        __syncthreads();
        // 4. slots: push k takes its victim's slot (pointer jumping)
        RB_GCLOCK(23, s == 0);
        // (reads and writes of a round separated by a barrier: at most 4 pushes
        // per thread, the CTA has >= min(1024, pushes) threads)
        for (;;) {
            int nv[4];
            int ch = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = tid + i * nt;
                nv[i] = 0;
                if (k < ns) {
                    const int e = slotk[k];
                    nv[i] = e >= C ? slotk[e - C] : e;
                    ch |= e >= C;
                }
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = tid + i * nt;
                if (k < ns) slotk[k] = nv[i];
            }
            if (!__syncthreads_or(ch)) break;
        }
        // 5. survivors: the pushes no later push evicted
        RB_GCLOCK(24, s == 0);
        // mark batch victims
        for (int k = tid; k < ns; k += nt)
            if (vk[k] >= C) cx[vk[k] - C] |= 2;  // bit 1: evicted within the batch
        __syncthreads();
        for (int k = tid; k < ns; k += nt)
            if (!(cx[k] & 2)) occb[slotk[k]] = k;
        // 6. new queues (head 0): F = (F ++ batch)[ns, ns + fs), W / Q = unpopped entries
        const int nw_new = w0 + (int)tot_wr - (int)tot_pw;
        const int nq_new = q0 + (ns - (int)tot_wr) - (ns - (int)tot_pw);
        nst.h[0] = nst.h[1] = nst.h[2] = 0;
        nst.n[0] = fs;
        nst.n[1] = nw_new;
        nst.n[2] = nq_new;
        // Every new entry is computed (reads of the old rings), then stored:
        // F_new[i] = (F ++ batch)[ns + i], W_new[i] = (W ++ WE)[pops_W + i],
        // Q_new[i] = (Q ++ QE)[pops_Q + i]; entry = slot | correct << 31
        auto entry_of = [&](int e, bool pre_bit) -> uint32_t {
            const int sl = e < C ? e : slotk[e - C];
            const bool c = e < C ? pre_bit : (cx[e - C] & 1) != 0;
            return (uint32_t)sl | (c ? 0x80000000u : 0u);
        };
        const int tot = fs + nw_new + nq_new;  // == C
        uint32_t val[4];  // C <= PBP_CMAX = 4 * blockDim.x at most (see the launch)
        int cnt = 0;
        for (int i = tid; i < tot; i += nt, ++cnt) {
            uint32_t x;
            if (i < fs) {
                const int t = ns + i;
                x = t < fs ? Fp[t] : entry_of(C + (t - fs), false);
            } else if (i < fs + nw_new) {
                const int m = (int)tot_pw + (i - fs);
                x = m < w0 ? Wp[m] : entry_of(WE[m - w0], false);
            } else {
                const int m = (ns - (int)tot_pw) + (i - fs - nw_new);
                x = m < q0 ? Qp[m] : entry_of(QE[m - q0], true);
            }
            val[cnt] = x;
        }
        __syncthreads();
        cnt = 0;
        for (int i = tid; i < tot; i += nt, ++cnt) {
            const uint32_t x = val[cnt];
            if (i < fs) ring[i] = x;
            else if (i < fs + nw_new) ring[RC + (i - fs)] = x;
            else ring[2 * RC + (i - fs - nw_new)] = x;
        }
    } else if (tid == 0) {
        // filling (or fresh_slots == 0): the sequential queue simulation
        GQ F{ring, RC, 0, st.n[0]}, W{ring + RC, RC, 0, st.n[1]}, Q{ring + 2 * RC, RC, 0, st.n[2]};
        int size = size0;
        for (int k = 0; k < ns; ++k) {
            int vs;
            const int gx = pb_push_logic(C, fs, F, W, Q, size, (cx[k] & 1) != 0, &vs);
            int e = -1;  // victim element
            if (vs == -2) e = -2;
            else if (vs >= 0) e = occb[vs] >= 0 ? C + occb[vs] : vs;
            if (e >= C) cx[e - C] |= 2;
            vk[k] = e;
            slotk[k] = gx;
            if (gx >= 0) occb[gx] = k;
        }
        nst.h[0] = F.h;
        nst.n[0] = F.n;
        nst.h[1] = W.h;
        nst.n[1] = W.n;
        nst.h[2] = Q.h;
        nst.n[2] = Q.n;
        s_st = nst;
    }
    __syncthreads();
    if (!par) nst = s_st;
    RB_GCLOCK(25, s == 0);
    // per push: evicted id (pre-batch occupants from the shared copy, so no
    // write below races with it), slot, survivor, metadata, payload descriptor
    int maxq = 0;
    for (int k = tid; k < ns; k += nt) {
        const int j = j0 + k * T;
        const int e = vk[k];
        uint64_t ev = NONE_ID;
        if (e == -2) ev = in.id[j];
        else if (e >= C) ev = in.id[j0 + (e - C) * T];
        else if (e >= 0) ev = preid[e];
        const int sl = slotk[k];
        const bool surv = sl >= 0 && !(cx[k] & 2);
        in.evid[j] = ev;
        in.tslot[j] = sl >= 0 ? (int32_t)((size_t)s * C + sl) : -1;
        in.surv[j] = surv;
        Unit d;
        d.row = -1;
        d.len = in.len[j];
        d.k0 = 0;
        d.g = j;
        d.off = in.toff ? in.toff[j] : 0;
        d.adv = 0.0;
        if (surv) {
            const size_t g = (size_t)s * C + sl;
            write_meta(v, g, in, j);
            v.seq[g] = P0 + k;
            if (s >= v.sb && s < v.se && d.len > 0 && v.stride > 0) {
                d.row = (s - v.sb) * C + sl;
                const int q = (d.len + 3) >> 2;
                maxq = q > maxq ? q : maxq;
            }
        }
        in.units[j] = d;
    }
    maxq = __reduce_max_sync(0xffffffffu, maxq);
    if ((tid & 31) == 0 && maxq) atomicMax(&s_maxq, maxq);
    RB_GCLOCK(26, s == 0);
    // rings back to global memory (rebased), state, push count
    for (int r = 0; r < 3; ++r)
        for (int i = tid; i < nst.n[r]; i += nt) {
            int p = nst.h[r] + i;
            if (p >= RC) p -= RC;
            gring[r][i] = ring[r * RC + p];
        }
    // arrival order: merge(W, Q) by sequence number, then F
    auto seqof = [&](uint32_t x) -> long long {
        const int sl = (int)(x & 0x7fffffffu);
        const int k = occb[sl];
        return k >= 0 ? P0 + k : preseq[sl];
    };
    auto at = [&](int r, int i) -> uint32_t {
        int p = nst.h[r] + i;
        if (p >= RC) p -= RC;
        return ring[r * RC + p];
    };
    int32_t* ord = v.order + (size_t)s * C;
    const int nw = nst.n[1], nq = nst.n[2], nf = nst.n[0];
    for (int k = tid; k < nw + nq; k += nt) {
        const bool inw = k < nw;
        const int a = inw ? k : k - nw;
        const uint32_t x = at(inw ? 1 : 2, a);
        const long long sq = seqof(x);
        const int orr = inw ? 2 : 1, on = inw ? nq : nw;
        int lo = 0, hi = on;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (seqof(at(orr, mid)) < sq) lo = mid + 1;
            else hi = mid;
        }
        ord[a + lo] = (int32_t)(x & 0x7fffffffu);
    }
    for (int k = tid; k < nf; k += nt) ord[nw + nq + k] = (int32_t)(at(0, k) & 0x7fffffffu);
    __syncthreads();
    RB_GCLOCK(27, s == 0);
    if (tid == 0) {
        PbState o;
        for (int r = 0; r < 3; ++r) {
            o.h[r] = 0;
            o.n[r] = nst.n[r];
        }
        v.pbs[s] = o;
        v.pushes[s] = P0 + ns;
        if (T == 1) {  // one CTA: no grid-wide counters
            *in.n_units = s_maxq;
            ctl->cursor = 0;
            if (n > 0) {
                ctl->max_id = idl;
                ctl->has_any = 1;
            }
            ctl->hash_stale = 1;
            RB_GCLOCK(28, true);
        } else if (s_maxq) {
            atomicMax(&gc->cta_max[0], s_maxq);
        }
        if (T > 1 && done_add_u32(&gc->done) == (unsigned)T - 1) {
            *in.n_units = atomicExch(&gc->cta_max[0], 0);
            ctl->cursor = (cur0 + (unsigned long long)n) % T;
            if (n > 0) {
                ctl->max_id = in.id[n - 1];
                ctl->has_any = 1;
            }
            ctl->hash_stale = 1;
            gc->done = 0;
            RB_GCLOCK(28, true);
        }
    }
    RB_TEND(0);
}

// Record copies with the post-increment use count in draw order
// (replay_buffer.cpp:201-202) and optional UseEvents (205-215).
__global__ void k_sample_records(BufView v, long long nsel, long long per,
                                 const int32_t* sel_slot, rb_record* out, rb_use_event* ev,
                                 long long batch_id, long long use_step) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nsel;
         i += (long long)gridDim.x * blockDim.x) {
        const int32_t g = sel_slot[i];
        const long long seg = (i / per) * per, end = seg + per;
        long long rank = 0, count = 0;
        for (long long k = seg; k < end; ++k) {
            if (sel_slot[k] == g) {
                ++count;
                if (k < i) ++rank;
            }
        }
        rb_record r = slot_record(v, g);
        r.use_count = (uint32_t)(v.use[g] - count + rank + 1);
        if (out) out[i] = r;
        if (ev) {
            rb_use_event e;
            e.rollout_id = r.rollout_id;
            e.creation_step = r.creation_step;
            e.use_step = use_step;
            e.batch_id = batch_id;
            e.within_batch_rank = i;
            ev[i] = e;
        }
    }
}

// ---------------------------------------------------------------- gather
// Persistent over nloc * ceil(max_nq / (128*U)) virtual units: 128*U quads of
// one selection's slot row -> the packed batch at its offset (funnel-shifted
// 128-bit stores; boundary quads shared with the neighbouring trajectory use
// masked stores).
// CM: chunk-major unit order for long rows (see k_loss_grpo_buf).
template <int U, bool CM = false>
// Registers capped so 8 CTAs per SM leave room for one more warp: the Rng's
// ring lookahead (one warp, launched when the sampler completes) runs beside
// the gather without displacing a CTA of this static-stride grid.
__global__ void __launch_bounds__(UNIT_THREADS, 9) k_gather(BufView v, const Unit* desc,
                                                        const int* maxq_p, int nloc,
                                                        int32_t* out_tok, float* out_lpo) {
    constexpr int QU = UNIT_THREADS * U;
    RB_TSTART(4);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int ups = (*maxq_p + QU - 1) / QU;  // units per selection
    const int nu = nloc * ups;
    Unit nxt;  // descriptor of the next unit, loaded one unit ahead
    auto sel = [&](int x) { return CM ? x % nloc : x / ups; };
    if ((int)blockIdx.x < nu) nxt = ld_unit(desc + sel(blockIdx.x));
    for (int u = blockIdx.x; u < nu; u += gridDim.x) {
        const int b = sel(u), c = CM ? u / nloc : u - b * ups;
        const Unit un = nxt;
        if (u + (int)gridDim.x < nu) nxt = ld_unit(desc + sel(u + (int)gridDim.x));
        const int a = (int)(un.off & 3);
        const int nq = (a + un.len + 3) >> 2;
        if (c * QU >= nq) continue;
        const int nsq = (un.len + 3) >> 2;
        const long long P0 = un.off >> 2;
        const int kw = c * QU + wid * 32 * U;
        const size_t row = (size_t)un.row * v.stride;
        uint4 ot[U], ol[U];
        if (out_tok)
            row_to_packed_quads<U>(reinterpret_cast<const uint4*>(v.tok + row), nsq, a, kw, ot);
        if (out_lpo)
            row_to_packed_quads<U>(reinterpret_cast<const uint4*>(v.lpo + row), nsq, a, kw, ol);
#pragma unroll
        for (int s = 0; s < U; ++s) {
            const int k = kw + 32 * s + lane;
            if (k < nq) {
                if (out_tok)
                    store_quad_masked(reinterpret_cast<uint32_t*>(out_tok), P0 + k, ot[s], 4 * k - a,
                                      un.len);
                if (out_lpo)
                    store_quad_masked(reinterpret_cast<uint32_t*>(out_lpo), P0 + k, ol[s], 4 * k - a,
                                      un.len);
            }
        }
    }
    RB_TEND(4);
}
#ifndef RB_GATHER_U
#define RB_GATHER_U 4
#endif
constexpr int GATHER_U = RB_GATHER_U;

// ---- early gather: a programmatic dependent of the fused sampler, which is
// itself a dependent of the insert's payload copy.  It starts while the copy
// and the sampler run: a unit (QU quads of one selection) is claimed from a
// counter and copied as soon as its map CTA has published its descriptors
// (gc->seg), so the gather of the records that were already resident overlaps
// the insert.  Units of the pending insert's records wait for the copy's
// completion flag (pay_sync[2]); units behind a rejected draw wait for the
// sampler's exact replay (gc->fin).  Deferred units are kept in shared memory
// and copied as soon as their condition holds.  Rows written by the
// concurrent copy are read through L2 (ld.cg), never the non-coherent path.
__device__ __forceinline__ Unit ld_unit_cg(const Unit* u) {
    const uint4 a = __ldcg(reinterpret_cast<const uint4*>(u));
    const uint4 b = __ldcg(reinterpret_cast<const uint4*>(u) + 1);
    Unit r;
    r.row = (int32_t)a.x;
    r.len = (int32_t)a.y;
    r.k0 = (int32_t)a.z;
    r.g = (int32_t)a.w;
    r.off = (int64_t)(((uint64_t)b.y << 32) | b.x);
    r.adv = __hiloint2double((int)b.w, (int)b.z);
    return r;
}
template <int U, bool CG>
__device__ __forceinline__ void row_to_packed_quads_l2(const uint4* rowq, int nsq, int a, int kw,
                                                       uint4 (&o)[U]) {
    if (!CG) {
        row_to_packed_quads<U>(rowq, nsq, a, kw, o);
        return;
    }
    const int lane = threadIdx.x & 31;
    uint4 cur[U];
#pragma unroll
    for (int s = 0; s < U; ++s) {
        const int k = kw + 32 * s + lane;
        cur[s] = (k >= 0 && k < nsq) ? __ldcg(rowq + k) : make_uint4(0, 0, 0, 0);
    }
    if (a == 0) {
#pragma unroll
        for (int s = 0; s < U; ++s) o[s] = cur[s];
        return;
    }
    uint4 first_prev = make_uint4(0, 0, 0, 0);
    if (lane == 0 && kw >= 1 && kw - 1 < nsq) first_prev = __ldcg(rowq + kw - 1);
#pragma unroll
    for (int s = 0; s < U; ++s) {
        uint4 prev = shfl_up4(cur[s]);
        const uint4 carry = s ? shfl4(cur[s > 0 ? s - 1 : 0], 31) : first_prev;
        if (lane == 0) prev = carry;
        o[s] = funnel(prev, cur[s], 4 - a);
    }
}
// Chunk c of a selection's destination quads: [c*QU, (c+1)*QU), the last
// chunk (c == ups-1) running to the end.
template <int U, bool CG>
__device__ __forceinline__ void gather_chunk(const uint4* tok_row, const uint4* lpo_row, int len,
                                          long long off, int c, int ups, int32_t* out_tok,
                                          float* out_lpo) {
    constexpr int QU = UNIT_THREADS * U;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int a = (int)(off & 3);
    const int nq = (a + len + 3) >> 2;
    const int nsq = (len + 3) >> 2;
    const long long P0 = off >> 2;
    const int end = c == ups - 1 ? nq : min(nq, (c + 1) * QU);
    for (int cq = c * QU; cq < end; cq += QU) {
        const int kw = cq + wid * 32 * U;
        uint4 q[U];
        if (out_tok) {
            row_to_packed_quads_l2<U, CG>(tok_row, nsq, a, kw, q);
#pragma unroll
            for (int s = 0; s < U; ++s) {
                const int k = kw + 32 * s + lane;
                if (k < end)
                    store_quad_masked(reinterpret_cast<uint32_t*>(out_tok), P0 + k, q[s], 4 * k - a, len);
            }
        }
        if (out_lpo) {
            row_to_packed_quads_l2<U, CG>(lpo_row, nsq, a, kw, q);
#pragma unroll
            for (int s = 0; s < U; ++s) {
                const int k = kw + 32 * s + lane;
                if (k < end)
                    store_quad_masked(reinterpret_cast<uint32_t*>(out_lpo), P0 + k, q[s], 4 * k - a, len);
            }
        }
    }
}
template <int U, bool CG>
__device__ __forceinline__ void gather_unit(const BufView& v, const Unit& un, int c, int ups,
                                            int32_t* out_tok, float* out_lpo) {
    const size_t row = (size_t)un.row * v.stride;
    gather_chunk<U, CG>(reinterpret_cast<const uint4*>(v.tok + row),
                        reinterpret_cast<const uint4*>(v.lpo + row), un.len, un.off, c, ups,
                        out_tok, out_lpo);
}
constexpr int GE_DEFER = 64;  // deferred units held per CTA
template <int U>
__global__ void __launch_bounds__(UNIT_THREADS, 8) k_gather_early(BufView v, const Unit* desc, int nloc,
                                                              long long lo, int ups, GridCtl* gc,
                                                              int nseg, const int* pay_pending,
                                                              int pay_epoch,
                                                              int32_t* out_tok, float* out_lpo) {
    __shared__ int s_claim[2], s_state, s_pay, s_fin, s_ndef;
    __shared__ int s_def[GE_DEFER];
    RB_TSTART(4);
    const int tid = threadIdx.x;
    const int nu = nloc * ups;
    if (tid == 0) {
        s_claim[0] = (int)atomicAdd(&gc->gwork, 1u);
        s_pay = 0;
        s_fin = 0;
        s_ndef = 0;
    }
    __syncthreads();
    // Copies the deferred units whose condition now holds (block-uniform).
    auto drain = [&](bool wait) {
        if (tid == 0) {
            if (!s_pay)  // the copy of the pending insert has completed
                s_pay = wait ? (spin_epoch(pay_pending, pay_epoch), 1)
                             : ld_acquire_i32(pay_pending) == (pay_epoch << 2 | 2);
            if (!s_fin) s_fin = wait ? (spin_while_eq(&gc->fin, 0), 1) : ld_acquire_i32(&gc->fin) != 0;
        }
        __syncthreads();
        if (!s_pay) return;  // every deferred unit needs the copy (replayed ones too)
        int keep = 0;
        const int n = s_ndef;
        for (int i = 0; i < n; ++i) {
            const int u = s_def[i];
            const bool replayed = u < 0;  // encoded as -(u+1)
            const int uu = replayed ? -(u + 1) : u;
            const int bb = uu / ups, c = uu - bb * ups;
            if (replayed && !s_fin) {
                __syncthreads();
                if (tid == 0) s_def[keep] = u;
                ++keep;
                continue;
            }
            const Unit un = ld_unit_cg(desc + bb);
            if (un.len > 0) gather_unit<U, true>(v, un, c, ups, out_tok, out_lpo);
        }
        __syncthreads();
        if (tid == 0) s_ndef = keep;
        __syncthreads();
    };
    int p = 0;
    for (;;) {
        const int u = s_claim[p];
        if (u >= nu) break;
        if (tid == 0) {
            s_claim[p ^ 1] = (int)atomicAdd(&gc->gwork, 1u);  // next claim, in flight meanwhile
            s_state = spin_while_eq(&gc->seg[(int)((lo + u / ups) / MAP_SPC)], 0);
            if (!s_pay) s_pay = ld_acquire_i32(pay_pending) == (pay_epoch << 2 | 2);
        }
        __syncthreads();
        const int b = u / ups, c = u - b * ups;
        const Unit un = ld_unit_cg(desc + b);
        if (s_state == 2) {  // behind a rejected draw: after the replay
            if (tid == 0) s_def[s_ndef++] = -(u + 1);
        } else if (un.k0 && !s_pay) {  // a record of the pending insert
            if (tid == 0) s_def[s_ndef++] = u;
        } else if (un.len > 0) {
            if (un.k0) gather_unit<U, true>(v, un, c, ups, out_tok, out_lpo);
            else gather_unit<U, false>(v, un, c, ups, out_tok, out_lpo);
        }
        __syncthreads();
        if (s_ndef == GE_DEFER) drain(true);
        else if (s_ndef && s_pay) drain(false);
        p ^= 1;
    }
    while (s_ndef) drain(true);
    __syncthreads();
    __shared__ int s_lastg;
    if (tid == 0) s_lastg = done_add_u32(&gc->gdone) == gridDim.x - 1;
    __syncthreads();
    if (s_lastg) {  // every CTA is past its waits: reset the flags for the next call
        for (int t = tid; t < nseg; t += UNIT_THREADS) gc->seg[t] = 0;
        if (tid == 0) {
            gc->fin = 0;
            gc->gwork = 0;
            gc->gdone = 0;
        }
    }
    RB_TEND(4);
    // completion of this gather implies completion of the sampler and the copy
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------- inspect
__global__ void k_shard_contents(BufView v, int s, long long n, rb_record* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = slot_record(v, (size_t)s * v.C + arrival_slot(v, s, i));
}
__global__ void k_slot_of(BufView v, int s, long long i, int32_t* out) {
    *out = (int32_t)((size_t)s * v.C + arrival_slot(v, s, i));
}

// Load: records written densely to slots 0..n-1 of shard s, arrival order.
__global__ void k_load_shard(BufView v, int s, long long n, const rb_record* recs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const size_t g = (size_t)s * v.C + i;
        const rb_record r = recs[i];
        v.id[g] = r.rollout_id;
        v.prompt[g] = r.prompt_id;
        v.group[g] = r.group_id;
        v.cstep[g] = r.creation_step;
        v.pver[g] = r.policy_version;
        v.reward[g] = r.reward;
        v.correct[g] = r.is_correct;
        v.blp[g] = r.behavior_logprob;
        v.adv[g] = r.advantage;
        v.gmean[g] = 0.0;
        v.use[g] = r.use_count;
        v.len[g] = 0;
        if (v.retention == RB_POSITIVE_BIAS) {
            v.order[g] = (int32_t)i;
            v.seq[g] = i;
        }
    }
}
// Positive-bias queues of a loaded shard (records at slots 0..n-1 in arrival
// order): F = the newest min(n, fs), the rest split into W / Q.
__global__ void k_load_posbias(BufView v, int s, int n, const rb_record* recs) {
    if (threadIdx.x != 0) return;
    const int C = v.C, RC = C + 1;
    const int nf = n < v.fs ? n : v.fs;
    uint32_t* F = (uint32_t*)pb_ring(v, 0, s);
    uint32_t* W = (uint32_t*)pb_ring(v, 1, s);
    uint32_t* Q = (uint32_t*)pb_ring(v, 2, s);
    PbState st{};
    for (int i = 0; i < n; ++i) {
        const uint32_t e = (uint32_t)i | (recs[i].is_correct ? 0x80000000u : 0u);
        if (i >= n - nf) F[st.n[0]++] = e;
        else if (recs[i].is_correct) Q[st.n[2]++] = e;
        else W[st.n[1]++] = e;
    }
    (void)RC;
    v.pbs[s] = st;
}

}  // namespace rb

// ====================================================================== host
rb_buffer::~rb_buffer() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (out_pending) cudaEventSynchronize(out_done);
    if (out_done) cudaEventDestroy(out_done);
    if (hmap_h) cudaFreeHost(hmap_h);
    if (gout_pending) cudaEventSynchronize(gather_done);
    if (gather_done) cudaEventDestroy(gather_done);
    if (gather_ready) cudaEventDestroy(gather_ready);
    if (look_ev) {
        if (cudaEventSynchronize(look_ev) != cudaSuccess) cudaDeviceSynchronize();  // captured
        cudaEventDestroy(look_ev);
    }
    void* ptrs[] = {v.id, v.prompt, v.group, v.cstep, v.pver, v.reward, v.blp, v.adv, v.gmean,
                    v.correct, v.use, v.len, v.order, v.head, v.pushes, v.owner, v.tok, v.lpo, v.pbq, v.pbs, v.seq,
                    v.hkeys, v.hstate, v.ctl, s_tslot, s_surv, s_evid, s_evrec, s_adv, s_gmean,
                    s_len, s_toff, sel_slot, sel_shard, sel_index, sel_off, sel_total,
                    acc, misc, n_units_ins, n_units_sel, loss_partials, route_ctl, map_ctl, pay_sync};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (void* p : stage_dev)
        if (p) cudaFree(p);
    if (stage_host) cudaFreeHost(stage_host);
    if (stage_event) cudaEventDestroy(stage_event);
    if (cs_in) cudaStreamSynchronize(cs_in);
    if (cs_out) cudaStreamSynchronize(cs_out);
    for (auto e : ev_io)
        if (e) cudaEventDestroy(e);
    if (cs_in) cudaStreamDestroy(cs_in);
    if (cs_out) cudaStreamDestroy(cs_out);
    cudaGetLastError();  // destructors report nothing: leave no error behind
    if (own_stream && stream) cudaStreamDestroy(stream);
}

template <class T>
static T* dalloc(size_t n) {
    T* p = nullptr;
    RB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    RB_CUDA(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}

void* rb_buffer::scratch(size_t bytes) {
    if (bytes > misc_cap) {
        if (misc) {
            sync();
            cudaFree(misc);
        }
        misc_cap = std::max(bytes, misc_cap * 2);
        RB_CUDA(cudaMalloc(&misc, misc_cap));
    }
    return misc;
}
void* rb_buffer::host_stage(size_t bytes) {
    if (stage_event) RB_CUDA(cudaEventSynchronize(stage_event));
    if (bytes > stage_host_cap) {
        sync();
        if (stage_host) cudaFreeHost(stage_host);
        stage_host_cap = std::max(bytes, stage_host_cap * 2);
        RB_CUDA(cudaMallocHost(&stage_host, stage_host_cap));
    }
    return stage_host;
}
void* rb_buffer::dev_stage(size_t bytes, int slot) {
    if (bytes > stage_dev_cap[slot]) {
        sync();
        drain_outputs();  // an asynchronous download may still read the old area
        if (stage_dev[slot]) cudaFree(stage_dev[slot]);
        stage_dev_cap[slot] = std::max(bytes, stage_dev_cap[slot] * 2);
        RB_CUDA(cudaMalloc(&stage_dev[slot], stage_dev_cap[slot]));
    }
    return stage_dev[slot];
}
void rb_buffer::host_stage_issued_on(cudaStream_t s) {
    if (!stage_event) RB_CUDA(cudaEventCreateWithFlags(&stage_event, cudaEventDisableTiming));
    RB_CUDA(cudaEventRecord(stage_event, s));
}
void rb_buffer::ensure_copy_streams() {
    if (cs_in) return;
    RB_CUDA(cudaStreamCreateWithFlags(&cs_in, cudaStreamNonBlocking));
    RB_CUDA(cudaStreamCreateWithFlags(&cs_out, cudaStreamNonBlocking));
    for (auto& e : ev_io) RB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}
void rb_buffer::grow_loss_partials(size_t bytes) {
    sync();
    if (loss_partials) cudaFree(loss_partials);
    RB_CUDA(cudaMalloc(&loss_partials, bytes));
    loss_partials_bytes = bytes;
}
void rb_buffer::host_stage_issued() {
    if (!stage_event) RB_CUDA(cudaEventCreateWithFlags(&stage_event, cudaEventDisableTiming));
    RB_CUDA(cudaEventRecord(stage_event, stream));
}
void rb_buffer::join_lookahead() {
    if (!look_pending) return;
    if (!look_captured && cudaEventQuery(look_ev) == cudaSuccess) {  // complete, uncaptured
        look_pending = false;
        joined_uid = look_uid;
        joined_seq = look_seq;
        return;
    }
    RB_CUDA(cudaStreamWaitEvent(stream, look_ev, 0));
    look_pending = false;
    joined_uid = look_uid;
    joined_seq = look_seq;
}
void rb_buffer::ensure_insert(size_t n) {
    if (n <= ins_cap) return;
    sync();
    void* ps[] = {s_tslot, s_surv, s_evid, s_evrec, s_adv, s_gmean, s_len, s_toff, units_ins};
    for (void* p : ps)
        if (p) cudaFree(p);
    ins_cap = std::max(n, ins_cap * 2);
    units_ins_cap = ins_cap;  // one descriptor per record
    units_ins = dalloc<Unit>(units_ins_cap);
    s_tslot = dalloc<int32_t>(ins_cap);
    s_surv = dalloc<uint8_t>(ins_cap);
    s_evid = dalloc<uint64_t>(ins_cap);
    s_evrec = dalloc<rb_record>(ins_cap);
    s_adv = dalloc<double>(ins_cap);
    s_gmean = dalloc<double>(ins_cap);
    s_len = dalloc<int32_t>(ins_cap);
    s_toff = dalloc<int64_t>(ins_cap + 1);
}
void rb_buffer::ensure_select(size_t n) {
    if (n <= sel_cap) return;
    sync();
    void* ps[] = {sel_slot, sel_shard, sel_index, sel_off, sel_len, units_sel};
    for (void* p : ps)
        if (p) cudaFree(p);
    sel_cap = std::max(n, sel_cap * 2);
    sel_len = dalloc<int32_t>(sel_cap);
    units_sel_cap = sel_cap;  // one descriptor per selection
    units_sel = dalloc<Unit>(units_sel_cap);
    sel_slot = dalloc<int32_t>(sel_cap);
    sel_shard = dalloc<int32_t>(sel_cap);
    sel_index = dalloc<int64_t>(sel_cap);
    sel_off = dalloc<int64_t>(sel_cap + 1);
}
void rb_buffer::sync() { RB_CUDA(cudaStreamSynchronize(stream)); }
namespace rb {
// dst (mapped host or device) <- src (device), 8-byte words (bytes % 8 == 0)
// or bytes; one CTA.
__global__ void k_copy_small(void* dst, const void* src, size_t bytes) {
    if (((uintptr_t)dst | (uintptr_t)src | bytes) % 8 == 0) {
        uint64_t* d = (uint64_t*)dst;
        const uint64_t* s = (const uint64_t*)src;
        for (size_t i = threadIdx.x; i < bytes / 8; i += blockDim.x) d[i] = s[i];
    } else {
        for (size_t i = threadIdx.x; i < bytes; i += blockDim.x)
            ((char*)dst)[i] = ((const char*)src)[i];
    }
}
}  // namespace rb
void rb_buffer::fetch(void* host_dst, const void* dev_src, size_t bytes) {
    if (bytes > hmap_cap) {
        sync();
        if (hmap_h) cudaFreeHost(hmap_h);
        hmap_cap = std::max<size_t>(bytes, std::max<size_t>(4096, hmap_cap * 2));
        RB_CUDA(cudaHostAlloc(&hmap_h, hmap_cap, cudaHostAllocMapped));
        RB_CUDA(cudaHostGetDevicePointer(&hmap_d, hmap_h, 0));
    }
    k_copy_small<<<1, 256, 0, stream>>>(hmap_d, dev_src, bytes);
    RB_CUDA(cudaGetLastError());
    sync();
    std::memcpy(host_dst, hmap_h, bytes);
}
void rb_buffer::to_host_async(void* host_dst, const void* dev_src, size_t bytes) {
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, host_dst, 0) != cudaSuccess) {  // pinned but not mapped
        cudaGetLastError();
        RB_CUDA(cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, stream));
        return;
    }
    k_copy_small<<<1, 256, 0, stream>>>(d, dev_src, bytes);
    RB_CUDA(cudaGetLastError());
}
void rb_buffer::wait_outputs_on(cudaStream_t s) {
    if (out_pending) RB_CUDA(cudaStreamWaitEvent(s, out_done, 0));
}
void rb_buffer::drain_outputs() {
    if (gout_pending) {
        RB_CUDA(cudaEventSynchronize(gather_done));
        gout_pending = false;
    }
    if (!out_pending) return;
    RB_CUDA(cudaEventSynchronize(out_done));
    out_pending = false;
}

namespace {

struct DeviceScope {  // make the buffer's device current for the call
    int prev = -1;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Device view of a caller array: returns a device pointer, staging host
// memory through the buffer's device staging area at `*cursor`.
struct Stager {
    rb_buffer* b;
    std::vector<std::pair<const void*, size_t>> host_items;
    size_t total = 0;
    explicit Stager(rb_buffer* b_) : b(b_) {}
};

void check_sticky(rb_buffer* b) {
    DevCtl c;
    b->fetch(&c, b->v.ctl, sizeof c);
    b->async_unchecked = false;
    if (c.err_code) {
        DevCtl z = c;
        z.err_code = 0;
        z.err_index = 0;
        RB_CUDA(cudaMemcpyAsync(b->v.ctl, &z, sizeof z, cudaMemcpyHostToDevice, b->stream));
        // The host mirrors assumed every asynchronous insert applied: resync
        // them from the device, which is authoritative.
        RB_CUDA(cudaMemcpyAsync(b->h_pushes.data(), b->v.pushes, b->T * sizeof(long long),
                                cudaMemcpyDeviceToHost, b->stream));
        RB_CUDA(cudaStreamSynchronize(b->stream));
        b->h_cursor = (size_t)c.cursor;
        if (c.err_index == -2) invalid("group advantages need >= 2 rewards");
        if (c.err_index == -3) invalid("rb_insert: trajectory length exceeds max_tokens");
        if (c.err_index == -4)
            invalid("rb_insert: RB_INSERT_ASSUME_UNIQUE violated (ids not new and strictly increasing)");
        invalid("ShardedReplayBuffer: rollout id " + std::to_string(c.err_id) +
                " is already stored");
    }
}

}  // namespace
void rb_buffer::sync_checked() {
    sync();
    if (async_unchecked) check_sticky(this);
}
namespace {

std::string fmt_double(double x) {  // text_io.cpp:10-14 (shortest round trip)
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, x);
    return std::string(buf, r.ptr);
}

std::string strategy_name(int s) {
    switch (s) {
        case RB_UNIFORM_WITH_REPLACEMENT: return "uniform_with_replacement";
        case RB_UNIFORM_WITHOUT_REPLACEMENT: return "uniform_without_replacement";
        case RB_UNUSED_FIRST_WITHOUT_REPLACEMENT: return "unused_first_without_replacement";
        case RB_PRIORITY_WITH_REPLACEMENT: return "priority_with_replacement";
    }
    throw Error(RB_ELOGIC, "bad SamplingStrategy");
}

rb_buffer* create(size_t T, size_t N, int strategy, int retention, double delta,
                  int32_t max_tokens, int device, size_t sb, size_t se) {
    require_device();
    if (T == 0) invalid("ShardedReplayBuffer: need at least one shard");
    if (N == 0 || N % T != 0)
        invalid("ShardedReplayBuffer: capacity must be a positive multiple of the shard count");
    if (retention == RB_POSITIVE_BIAS && !(delta >= 0.0 && delta <= 1.0))
        invalid("RetentionPolicy: delta must be in [0, 1]");
    if (strategy < 0 || strategy > 3) throw Error(RB_ELOGIC, "bad SamplingStrategy");
    if (max_tokens < 0) invalid("rb_create: max_tokens must be >= 0");
    if (sb == 0 && se == 0) se = T;
    if (sb >= se || se > T) invalid("rb_create: bad owned shard range");
    if (N / T > (size_t)INT32_MAX / 2 || N > (size_t)INT32_MAX / 2)
        invalid("rb_create: capacity too large");
    if (device < 0) RB_CUDA(cudaGetDevice(&device));
    DeviceScope ds(device);
    auto* b = new rb_buffer();
    try {
        b->T = T;
        b->N = N;
        b->C = N / T;
        b->strategy = strategy;
        b->retention = retention;
        b->delta = retention == RB_POSITIVE_BIAS ? delta : 0.0;
        b->max_tokens = max_tokens;
        b->stride = (max_tokens + 3) & ~3;
        b->device = device;
        b->sb = sb;
        b->se = se;
        RB_CUDA(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
        b->own_stream = true;
        BufView& v = b->v;
        v.T = (int)T;
        v.C = (int)b->C;
        v.stride = b->stride;
        v.retention = retention;
        v.sb = (int)sb;
        v.se = (int)se;
        // replay_buffer.cpp:110-112
        const size_t cs = retention == RB_POSITIVE_BIAS
                              ? (size_t)std::floor(b->delta * (double)b->C + 1e-9)
                              : 0;
        v.cs = (int)cs;
        v.fs = (int)(b->C - cs);
        v.id = dalloc<uint64_t>(N);
        v.prompt = dalloc<uint64_t>(N);
        v.group = dalloc<uint64_t>(N);
        v.cstep = dalloc<int64_t>(N);
        v.pver = dalloc<int64_t>(N);
        v.reward = dalloc<double>(N);
        v.blp = dalloc<double>(N);
        v.adv = dalloc<double>(N);
        v.gmean = dalloc<double>(N);
        v.correct = dalloc<uint8_t>(N);
        v.use = dalloc<uint32_t>(N);
        v.len = dalloc<int32_t>(N);
        v.order = dalloc<int32_t>(N);
        v.head = dalloc<int32_t>(T);
        if (retention == RB_POSITIVE_BIAS) {
            v.pbq = dalloc<int32_t>(3 * T * (b->C + 1));
            v.pbs = dalloc<PbState>(T);
            v.seq = dalloc<long long>(N);
            const size_t smem = (9 * (size_t)PB_CH + b->C) * sizeof(uint32_t);
            if (smem > 48 * 1024) {
                if (smem > 200 * 1024) invalid("rb_create: positive-bias shard capacity too large");
                RB_CUDA(cudaFuncSetAttribute(k_posbias_batch,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            }
        }
        v.pushes = dalloc<long long>(T);
        v.owner = dalloc<int32_t>(N);
        const size_t rows = (se - sb) * b->C * (size_t)b->stride;
        v.tok = rows ? dalloc<int32_t>(rows) : nullptr;
        v.lpo = rows ? dalloc<float>(rows) : nullptr;
        unsigned long long hc = 64;
        while (hc < 4ULL * N + 131072) hc <<= 1;  // batches up to hc/4 per kernel
        v.hcap = hc;
        v.hkeys = dalloc<uint64_t>(hc);
        v.hstate = dalloc<uint32_t>(hc);
        v.ctl = dalloc<DevCtl>(1);
        b->sel_total = dalloc<long long>(2);
        b->acc = dalloc<DevLossAcc>(1);
        int sms = 148;
        RB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        // One shared-memory carveout for the kernels that run side by side: an
        // SM configured for a smem-less streaming kernel (max L1) cannot take
        // a CTA that needs shared memory until it drains, which would
        // serialise the route / sampler CTAs behind the persistent copy grid.
        // The copy bypasses L1 (ld.global.nc.L1::no_allocate).
        {
            const void* ks[] = {(const void*)k_route_fifo, (const void*)k_sample_fused,
                                (const void*)k_sample_map, (const void*)k_insert_payload<PAYLOAD_U>,
                                (const void*)k_insert_payload_fifo<PAYLOAD_U>,
                                (const void*)k_insert_payload_tma,
                                (const void*)k_insert_route};
            for (const void* k : ks)
                RB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             cudaSharedmemCarveoutMaxShared));
        }
        b->unit_grid = sms * UNIT_CTAS_PER_SM;
        // Persistent grids: exactly the resident CTAs of each kernel.  The
        // payload copy overlaps the sampler's draw CTA, so it leaves room.
        int occ = 0;
        RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<GATHER_U>,
                                                              UNIT_THREADS, 0));
        b->grid_gather = sms * std::max(std::min(occ, 8), 1);
        RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_insert_payload<PAYLOAD_U>,
                                                              UNIT_THREADS, 0));
        {
            int occ2 = 0;
            RB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &occ2, k_insert_payload_fifo<PAYLOAD_U>, UNIT_THREADS, 0));
            occ = std::min(occ, occ2);
        }
        // The copy overlaps the latency-bound route / sampler kernels: keep
        // only the bytes in flight that saturate HBM (more only deepens the
        // memory queues those kernels' dependent loads wait in), and leave
        // room on every SM for their CTAs.
        {
            int per_sm = 3;
            if (const char* e = std::getenv("RB_PAYLOAD_CTAS")) per_sm = std::atoi(e);
            b->payload_grid = sms * std::max(1, std::min(per_sm, occ - 2));
        }
        b->grid_loss = loss_grid(sms);
        b->route_ctl = dalloc<GridCtl>(1);
        b->pay_sync = dalloc<int>(4);
        {  // no insert yet: the route-completion flag starts set
            const int one = 1;
            RB_CUDA(cudaMemcpy(b->pay_sync + 1, &one, sizeof one, cudaMemcpyHostToDevice));
        }
        b->pdl = std::getenv("RB_NO_PDL") == nullptr;
        b->lookahead = std::getenv("RB_NO_LOOKAHEAD") == nullptr;
        if (const char* e = std::getenv("RB_LOOKAHEAD_MIN_DRAWS")) b->lookahead_min_draws = std::atoll(e);
        // early gather (k_gather_early): opt-in, see DESIGN.md §4 — overlapping
        // the gather with the payload copy did not raise their combined HBM
        // throughput on C4 (both are bandwidth-bound)
        b->early_gather_ok = b->pdl && std::getenv("RB_EARLY_GATHER") != nullptr;
        b->tma_payload = std::getenv("RB_PAYLOAD_LSU") == nullptr;
        b->pb_par = std::getenv("RB_NO_PB_PAR") == nullptr;
        b->route_pdl = b->pdl && std::getenv("RB_NO_ROUTE_PDL") == nullptr;
        b->loss_dyn = std::getenv("RB_LOSS_CHUNK_MAJOR") == nullptr;
        b->tma_long = std::getenv("RB_PAYLOAD_TMA_LONG") != nullptr;
        b->chunk_major = std::getenv("RB_NO_CHUNK_MAJOR") == nullptr;
        b->tma_ctas = PB_CTAS;  // the build default (RB_PB_CTAS), overridable per process
        if (const char* e = std::getenv("RB_TMA_CTAS")) b->tma_ctas = std::max(1, std::atoi(e));
        b->sms = sms;
        RB_CUDA(cudaFuncSetAttribute(k_insert_payload_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)PB_SMEM));
        // test hook: force the sampler's exact draw replay (must not change results)
        v.dbg_replay = std::getenv("RB_DEBUG_FORCE_DRAW_REPLAY") != nullptr;
        b->map_ctl = dalloc<GridCtl>(1);
        {
            const int none = INT_MAX;
            RB_CUDA(cudaMemcpy(&b->map_ctl->first_rej, &none, sizeof none, cudaMemcpyHostToDevice));
        }
        b->n_units_ins = dalloc<int>(1);
        b->n_units_sel = dalloc<int>(1);
        b->loss_partials = dalloc<char>((size_t)b->unit_grid * 32);
        b->loss_partials_bytes = (size_t)b->unit_grid * 32;
        b->h_pushes.assign(T, 0);
    } catch (...) {
        delete b;
        throw;
    }
    return b;
}


// Insert `bt` (pointers already resolved to device memory; lens/toff device)
void launch_insert(rb_buffer* b, const rb_insert_batch& bt, bool want_evrec, bool unique) {
    InsertIn in{};
    in.n = (long long)bt.n;
    in.id = bt.rollout_id;
    in.prompt = bt.prompt_id;
    in.group = bt.group_id;
    in.cstep = bt.creation_step;
    in.pver = bt.policy_version;
    in.reward = bt.reward;
    in.correct = bt.is_correct;
    in.blp = bt.behavior_logprob;
    in.adv = bt.advantage;
    in.gmean = bt.group_mean;
    in.goff = bt.group_offsets;
    in.ngroups = (long long)bt.n_groups;
    in.toff = bt.tok_offsets;
    in.maxlen = b->max_tokens;
    in.len = b->s_len;
    in.adv_out = b->s_adv;
    in.gmean_out = b->s_gmean;
    in.tslot = b->s_tslot;
    in.surv = b->s_surv;
    in.evid = b->s_evid;
    in.evrec = want_evrec ? b->s_evrec : nullptr;
    const bool payload = bt.tok_offsets && b->stride > 0 && (bt.tokens || bt.logp_old);
    in.units = b->units_ins;
    in.n_units = b->n_units_ins;
    if (!payload) in.toff = bt.tok_offsets;  // lengths only
    bool closed = false;
    const bool fifo_route = unique && b->retention == RB_PLAIN_FIFO && !want_evrec &&
                            bt.n <= (size_t)RT_THREADS * GRID_MAX_CTAS;
    in.own_only = b->own_n_global ? 1 : 0;
    in.n_global = b->own_n_global ? (long long)b->own_n_global : in.n;
    if (in.own_only && !fifo_route)
        throw Error(RB_ELOGIC, "rb_insert_owned: FIFO retention and ids promised unique required");
    if (fifo_route) {
        // ids promised new and increasing: the closed-form FIFO route
        b->ins_epoch = (b->ins_epoch + 1) & RB_EPOCH_MASK;
        in.epoch = b->ins_epoch;
        const unsigned grid = (unsigned)((bt.n + RT_THREADS - 1) / RT_THREADS);
        closed = payload && b->T <= 64 && b->pdl;
        // a sampler enqueued next reads the new records' lengths from the
        // offsets after this call returns: the route kernel keeps a copy
        in.toff_keep = bt.tok_offsets && b->T <= 64 && b->pdl ? b->s_toff : nullptr;
        in.pay_follows = closed ? 1 : 0;
        in.split_validate = bt.n > (size_t)RT_SPLIT_MIN ? 1 : 0;
        in.keep_cnt = &b->route_ctl->keep_cnt;
        in.keep_ctas = in.toff_keep ? (int)((bt.n + 1 + RT_KEEP - 1) / RT_KEEP) : 0;
        b->keep_total += (unsigned long long)in.keep_ctas;  // extra CTAs copy them
        // a programmatic dependent of the previous kernel (the last step's
        // sampler or loss trigger at their start): the batch's loads,
        // validation and group advantages overlap that kernel's tail; the
        // buffer is touched only after griddepcontrol.wait
        cudaLaunchConfig_t rcfg = {};
        rcfg.gridDim = dim3(grid + (unsigned)in.keep_ctas);
        rcfg.blockDim = dim3(RT_THREADS);
        rcfg.stream = b->stream;
        cudaLaunchAttribute rat[1];
        rat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        rat[0].val.programmaticStreamSerializationAllowed = 1;
        rcfg.attrs = rat;
        rcfg.numAttrs = b->route_pdl ? 1 : 0;
        RB_CUDA(cudaLaunchKernelEx(&rcfg, k_route_fifo, b->v, in, b->route_ctl, b->pay_sync));
    } else if (unique && b->retention == RB_POSITIVE_BIAS && !want_evrec && b->pb_par &&
               b->C <= (size_t)PBP_CMAX && bt.n <= (size_t)PBP_NMAX &&
               (bt.n + b->T - 1) / b->T <= (size_t)PBP_NSMAX) {
        // ids promised new: validation, advantages and the queue update in one
        // launch, one CTA per shard (k_posbias_par)
        const int nsp = (int)((bt.n + b->T - 1) / b->T + 3) & ~3;
        const size_t smem = b->C * 16 + 3 * (b->C + 1) * 4 + b->C * 4 + (size_t)nsp * 18;
        static bool attr_set = false;  // per process: the kernel's opt-in limit
        if (!attr_set) {
            RB_CUDA(cudaFuncSetAttribute(k_posbias_par, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         208 * 1024));
            attr_set = true;
        }
        // CTA size from the work: every phase ends in a CTA barrier, whose cost
        // grows with the warp count (C2: 162 pushes -> 192 threads); at least
        // C/4 threads (the ring rewrite keeps 4 entries per thread in registers)
        const int need = std::max({nsp, (int)(b->C + 3) / 4, 128});
        const int nthr = std::min(PBP_THREADS, (need + 31) & ~31);
        // a programmatic dependent of the previous kernel, like the FIFO route
        cudaLaunchConfig_t pcfg = {};
        pcfg.gridDim = dim3((unsigned)b->T);
        pcfg.blockDim = dim3((unsigned)nthr);
        pcfg.dynamicSmemBytes = smem;
        pcfg.stream = b->stream;
        cudaLaunchAttribute pat[1];
        pat[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pat[0].val.programmaticStreamSerializationAllowed = 1;
        pcfg.attrs = pat;
        pcfg.numAttrs = b->route_pdl ? 1 : 0;
        RB_CUDA(cudaLaunchKernelEx(&pcfg, k_posbias_par, b->v, in, (unsigned long long)b->h_cursor,
                                   b->route_ctl, nsp));
    } else {
        k_insert_route<<<1, 1024, 0, b->stream>>>(b->v, in);
        if (b->retention == RB_POSITIVE_BIAS) {
            RB_CUDA(cudaGetLastError());
            const size_t smem = (9 * (size_t)PB_CH + b->C) * sizeof(uint32_t);
            k_posbias_batch<<<(unsigned)b->T, PB_THREADS, smem, b->stream>>>(
                b->v, in, (unsigned long long)b->h_cursor);
        }
    }
    RB_CUDA(cudaGetLastError());
    if (payload && closed) {
        // closed-form copy as a programmatic dependent of the route
        FifoPlan p{};
        p.c0 = (int)(b->h_cursor % b->T);
        p.T = (int)b->T;
        p.C = (int)b->C;
        p.own = b->own_n_global ? (int)b->sb : -1;
        p.epoch = in.epoch;
        const int maxq = (b->max_tokens + 3) / 4;
        p.ups = std::max(1, (maxq + UNIT_THREADS * PAYLOAD_U - 1) / (UNIT_THREADS * PAYLOAD_U));
        for (size_t s = 0; s < b->T; ++s) p.pm[s] = (int)(b->h_pushes[s] % (long long)b->C);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(b->payload_grid);
        cfg.blockDim = dim3(UNIT_THREADS);
        cfg.stream = b->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        // Bulk copy for rows of up to one item (PB_CHT tokens) per array; longer
        // (ragged-prone) rows split into several items per pipeline and the
        // LSU copy measured faster (C3: 59.4 vs 68.5 µs per step).
        if (b->tma_payload && (b->stride <= PB_CHT || b->tma_long) && b->stride <= 1023 * PB_CHT) {
            cfg.gridDim = dim3(b->sms * b->tma_ctas);
            cfg.blockDim = dim3(32);
            cfg.dynamicSmemBytes = PB_SMEM;
            RB_CUDA(cudaLaunchKernelEx(&cfg, k_insert_payload_tma, b->v, p, bt.tok_offsets,
                                       (int)bt.n, bt.tokens, bt.logp_old, b->pay_sync));
        } else {
            RB_CUDA(cudaLaunchKernelEx(&cfg, k_insert_payload_fifo<PAYLOAD_U>, b->v, p,
                                       bt.tok_offsets, (int)bt.n, bt.tokens, bt.logp_old,
                                       b->pay_sync));
        }
        b->pdl_tail = true;  // a sampler launched next may overlap this copy
        b->pend.pending = 1;
        b->pend.c0 = p.c0;
        b->pend.n = b->own_n_global ? (int)b->own_n_global : (int)bt.n;
        b->pend.own = b->own_n_global ? 1 : 0;
        b->pend.epoch = in.epoch;
        b->pend.toff = b->s_toff;  // the route kernel's copy
        b->pend.keep_cnt = &b->route_ctl->keep_cnt;
        b->pend.keep_target = b->keep_total;
        for (size_t s = 0; s < b->T; ++s) b->pend.P[s] = b->h_pushes[s];
    } else if (payload) {
        k_insert_payload<PAYLOAD_U><<<b->payload_grid, UNIT_THREADS, 0, b->stream>>>(
            b->v, b->units_ins, b->n_units_ins, (int)bt.n, bt.tokens, bt.logp_old);
        RB_CUDA(cudaGetLastError());
        // the insert's metadata is final once this copy starts: a fused sampler
        // launched next may run beside the copy (no pending plan)
        b->pdl_tail = b->pdl;
        b->pend.pending = 0;
    } else if (fifo_route && b->T <= 64 && b->pdl) {
        // no payload: the route kernel (which triggers its dependents at its
        // start) is the tail; a sampler may overlap it with the insert's plan
        b->pdl_tail = true;
        b->pend.pending = 1;
        b->pend.c0 = (int)(b->h_cursor % b->T);
        b->pend.n = b->own_n_global ? (int)b->own_n_global : (int)bt.n;
        b->pend.own = b->own_n_global ? 1 : 0;
        b->pend.epoch = in.epoch;
        b->pend.toff = bt.tok_offsets ? b->s_toff : nullptr;  // lengths only (or NULL: length 0)
        b->pend.keep_cnt = &b->route_ctl->keep_cnt;
        b->pend.keep_target = b->keep_total;
        for (size_t s = 0; s < b->T; ++s) b->pend.P[s] = b->h_pushes[s];
    } else {
        b->pdl_tail = false;
    }
}

}  // namespace

// helper launchers defined at the end of this file (C++ linkage)
void rb_lengths_from_offsets(const int64_t* toff, size_t n, int32_t* len, int32_t maxlen,
                             DevCtl* ctl, cudaStream_t s);
void rb_widen_i32(const int32_t* a, int64_t* b, size_t n, cudaStream_t s);
void rb_batch_ids_dev(const BufView& v, const int32_t* sel_slot, long long lo, long long hi,
                      uint64_t* ids, int32_t* lens, cudaStream_t s);

// ---------------------------------------------------------------- C ABI
extern "C" {

int rb_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor) {
    return guard([&] {
        require_device();
        int d = 0;
        RB_CUDA(cudaGetDevice(&d));
        if (device) *device = d;
        if (sm_count) RB_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, d));
        if (cc_major) RB_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, d));
        if (cc_minor) RB_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, d));
    });
}

int rb_create(size_t num_shards, size_t total_capacity, int strategy, int retention,
              double delta, int32_t max_tokens, int device, size_t shard_begin,
              size_t shard_end, rb_buffer** out) {
    return guard([&] {
        *out = create(num_shards, total_capacity, strategy, retention, delta, max_tokens,
                      device, shard_begin, shard_end);
    });
}

void rb_destroy(rb_buffer* b) { delete b; }

int rb_set_stream(rb_buffer* b, void* stream) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->gather_early = false;
        b->sync();
        if (b->own_stream && b->stream) cudaStreamDestroy(b->stream);
        // Any handle is taken as given; NULL is the legacy default stream.
        b->stream = (cudaStream_t)stream;
        b->own_stream = false;
    });
}
void* rb_get_stream(rb_buffer* b) { return (void*)b->stream; }

int rb_insert(rb_buffer* b, const rb_insert_batch* bt_in, uint64_t* out_evicted_ids,
              size_t* out_applied, int flags) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->gather_early = false;
        b->join_lookahead();  // before the route: the sampler that follows stays a PDL dependent
        {  // an error left by an unrelated earlier call must not be blamed on this one
            const cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess)
                throw Error(RB_ECUDA, std::string("CUDA error pending before rb_insert: ") +
                                          cudaGetErrorString(e));
        }
        rb_insert_batch bt = *bt_in;
        if (out_applied) *out_applied = 0;
        if (bt.n == 0) return;
        if (!bt.rollout_id || !bt.reward) invalid("rb_insert: rollout_id and reward are required");
        if (!bt.advantage && !bt.group_offsets)
            invalid("rb_insert: need advantage or group_offsets");
        // Split very large batches so the exact path's hash set stays sparse.
        const size_t chunk_max = (size_t)(b->v.hcap / 4);
        if (bt.n > chunk_max && !b->own_n_global) {  // (an owned batch takes the closed form)
            if (!bt.advantage) invalid("rb_insert: batch too large for device advantages");
            size_t done = 0;
            while (done < bt.n) {
                const size_t m = std::min(chunk_max, bt.n - done);
                rb_insert_batch c = bt;
                auto adv = [&](auto* p) { return p ? p + done : p; };
                c.n = m;
                c.rollout_id = adv(bt.rollout_id);
                c.prompt_id = adv(bt.prompt_id);
                c.group_id = adv(bt.group_id);
                c.creation_step = adv(bt.creation_step);
                c.policy_version = adv(bt.policy_version);
                c.reward = adv(bt.reward);
                c.is_correct = adv(bt.is_correct);
                c.behavior_logprob = adv(bt.behavior_logprob);
                c.advantage = adv(bt.advantage);
                c.group_mean = adv(bt.group_mean);
                c.tok_offsets = adv(bt.tok_offsets);
                size_t applied = 0;
                int st = rb_insert(b, &c, out_evicted_ids ? out_evicted_ids + done : nullptr,
                                   &applied, flags);
                if (out_applied) *out_applied = done + applied;
                if (st != RB_OK) throw Error(st, rb_last_error());
                done += m;
            }
            return;
        }
        b->ensure_insert(bt.n);
        const size_t n = bt.n;

        // Resolve every input array to device memory (host arrays staged).
        struct Item {
            const void** ptr;
            size_t bytes;  // device staging size
            size_t copy;   // bytes read from the caller's array (<= bytes; the rest is zeroed)
        };
        std::vector<Item> items;
        const int64_t* toff_user = bt.tok_offsets;
        auto add = [&](const void** p, size_t bytes, size_t copy = SIZE_MAX) {
            if (*p && !is_device_ptr(*p)) items.push_back({p, bytes, std::min(bytes, copy)});
        };
        // packed device arrays are read with 16-byte vector loads / bulk copies
        require_aligned16(bt.tokens, "rb_insert: tokens");
        require_aligned16(bt.logp_old, "rb_insert: logp_old");
        add((const void**)&bt.rollout_id, n * 8);
        add((const void**)&bt.prompt_id, n * 8);
        add((const void**)&bt.group_id, n * 8);
        add((const void**)&bt.creation_step, n * 8);
        add((const void**)&bt.policy_version, n * 8);
        add((const void**)&bt.reward, n * 8);
        add((const void**)&bt.is_correct, n);
        add((const void**)&bt.behavior_logprob, n * 8);
        add((const void**)&bt.advantage, n * 8);
        add((const void**)&bt.group_mean, n * 8);
        add((const void**)&bt.group_offsets, (bt.n_groups + 1) * 8);
        const bool toff_host = toff_user && !is_device_ptr(toff_user);
        add((const void**)&bt.tok_offsets, (n + 1) * 8);
        size_t payload_elems = 0;
        const bool host_payload = (bt.tokens && !is_device_ptr(bt.tokens)) ||
                                  (bt.logp_old && !is_device_ptr(bt.logp_old));
        if (toff_user && host_payload) {  // size needed only to stage host payload
            if (toff_host) {
                payload_elems = (size_t)toff_user[n];
            } else {
                int64_t last = 0;
                RB_CUDA(cudaMemcpy(&last, toff_user + n, 8, cudaMemcpyDeviceToHost));
                payload_elems = (size_t)last;
            }
            const size_t pbytes = ((payload_elems + 3) & ~size_t(3)) * 4;
            add((const void**)&bt.tokens, pbytes, payload_elems * 4);
            add((const void**)&bt.logp_old, pbytes, payload_elems * 4);
        }
        if (toff_host) {
            for (size_t j = 0; j < n; ++j) {
                const int64_t l = toff_user[j + 1] - toff_user[j];
                if (l < 0 || l > b->max_tokens)
                    invalid("rb_insert: trajectory length " + std::to_string(l) +
                            " exceeds max_tokens " + std::to_string(b->max_tokens));
            }
        }
        if (!items.empty()) {
            // Large pinned host arrays (the token payload) are copied straight
            // to the device, issued first; pageable ones and the small
            // per-record columns are packed into the pinned staging area
            // while those copies run, then sent in one H2D (a copy per
            // column would cost a PCIe round trip each).
            constexpr size_t DIRECT_MIN = 1 << 20;
            auto direct = [&](const Item& it) { return it.bytes >= DIRECT_MIN && is_pinned_ptr(*it.ptr); };
            size_t total = 0, paged = 0;
            for (auto& it : items) {
                total += (it.bytes + 255) & ~size_t(255);
                if (!direct(it)) paged += (it.bytes + 255) & ~size_t(255);
            }
            char* dsg = (char*)b->dev_stage(total, rb_buffer::ST_INSERT);
            char* hs = paged ? (char*)b->host_stage(paged) : nullptr;
            size_t o = 0, ho = 0;
            // A rank holding one of the shards reads only its own records'
            // payload (every T-th record from the cursor).  With the offsets
            // on the host and equal lengths, only those rows cross PCIe, as
            // one strided 2-D copy per array (a batch of per-record copies
            // measured slower than the whole array: ~2.4 µs per range).
            bool partial = b->se == b->sb + 1 && b->T > 1 && toff_host && n > 0 && !b->own_n_global;
            const int64_t L0 = partial ? toff_user[1] - toff_user[0] : 0;
            for (size_t j = 1; partial && j < n; ++j)
                if (toff_user[j + 1] - toff_user[j] != L0) partial = false;
            partial = partial && L0 > 0;
            const size_t j0 = partial ? (b->sb + b->T - b->h_cursor % b->T) % b->T : 0;
            const size_t rows = partial && j0 < n ? (n - 1 - j0) / b->T + 1 : 0;
            for (auto& it : items) {
                const size_t sz = (it.bytes + 255) & ~size_t(255);
                if (direct(it)) {
                    const bool payload_arr = it.ptr == (const void**)&bt.tokens ||
                                             it.ptr == (const void**)&bt.logp_old;
                    if (partial && payload_arr) {
                        if (rows) {
                            const size_t t0 = (size_t)toff_user[j0] * 4, w = (size_t)L0 * 4;
                            const size_t pitch = w * b->T;
                            RB_CUDA(cudaMemcpy2DAsync(dsg + o + t0, pitch, (const char*)*it.ptr + t0,
                                                      pitch, w, rows, cudaMemcpyHostToDevice,
                                                      b->stream));
                        }
                    } else {
                        RB_CUDA(cudaMemcpyAsync(dsg + o, *it.ptr, it.copy,
                                                cudaMemcpyHostToDevice, b->stream));
                        if (it.copy < it.bytes)
                            RB_CUDA(cudaMemsetAsync(dsg + o + it.copy, 0, it.bytes - it.copy, b->stream));
                    }
                    *it.ptr = dsg + o;
                    o += sz;
                }
            }

            const size_t paged_base = o;
            for (auto& it : items) {
                const size_t sz = (it.bytes + 255) & ~size_t(255);
                if (*it.ptr >= (const void*)dsg && *it.ptr < (const void*)(dsg + total)) continue;
                std::memcpy(hs + ho, *it.ptr, it.copy);
                if (it.copy < it.bytes) std::memset(hs + ho + it.copy, 0, it.bytes - it.copy);
                *it.ptr = dsg + paged_base + ho;
                ho += sz;
            }
            if (paged) {
                RB_CUDA(cudaMemcpyAsync(dsg + paged_base, hs, paged, cudaMemcpyHostToDevice,
                                        b->stream));
                b->host_stage_issued();
            }
        }
        if (flags & RB_INSERT_ASSUME_UNIQUE) b->async_unchecked = true;
        const bool want_evrec = (flags & 0x100) != 0;  // internal: rb_push
        launch_insert(b, bt, want_evrec, (flags & RB_INSERT_ASSUME_UNIQUE) != 0);
        if (out_evicted_ids) {
            RB_CUDA(cudaMemcpyAsync(out_evicted_ids, b->s_evid, n * 8, cudaMemcpyDefault,
                                    b->stream));
            b->pdl_tail = false;  // the copy, not the payload kernel, is the stream's tail
        }
        // host mirrors: assume fully applied, corrected below when synchronous
        const size_t nG = b->own_n_global ? b->own_n_global : n;  // the global batch
        for (size_t j = 0; j < nG; ++j) b->h_pushes[(b->h_cursor + j) % b->T]++;
        const size_t cursor_before = b->h_cursor;
        std::vector<long long> pushes_before;
        b->h_cursor = (b->h_cursor + nG) % b->T;
        if (!(flags & RB_INSERT_ASSUME_UNIQUE)) {
            DevCtl c;
            RB_CUDA(cudaMemcpyAsync(&c, b->v.ctl, sizeof c, cudaMemcpyDeviceToHost, b->stream));
            RB_CUDA(cudaStreamSynchronize(b->stream));
            if (c.err_code) {
                // roll the mirrors back to the applied prefix
                for (size_t j = 0; j < n; ++j) b->h_pushes[(cursor_before + j) % b->T]--;
                const size_t applied = c.err_index >= 0 ? (size_t)c.err_index : 0;
                for (size_t j = 0; j < applied; ++j) b->h_pushes[(cursor_before + j) % b->T]++;
                b->h_cursor = (cursor_before + applied) % b->T;
                if (out_applied) *out_applied = applied;
                check_sticky(b);  // clears and throws
            }
            if (out_applied) *out_applied = n;
        } else if (out_applied) {
            *out_applied = n;
        }
    });
}

int rb_set_owned_metadata(rb_buffer* b, int on) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (on && !(b->T > 1 && b->se == b->sb + 1 && b->T <= 64))
            throw Error(RB_ELOGIC, "rb_set_owned_metadata: one owned shard of 2..64 required");
        if (on && (b->retention != RB_PLAIN_FIFO || b->strategy != RB_UNIFORM_WITH_REPLACEMENT))
            throw Error(RB_ELOGIC,
                        "rb_set_owned_metadata: FIFO retention and uniform draws with replacement required");
        b->owned_meta = on != 0;
    });
}

int rb_insert_owned(rb_buffer* b, const rb_insert_batch* batch, size_t n_global, int flags) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (!b->owned_meta) throw Error(RB_ELOGIC, "rb_insert_owned: rb_set_owned_metadata first");
        if (!(flags & RB_INSERT_ASSUME_UNIQUE))
            throw Error(RB_ELOGIC, "rb_insert_owned: ids must be promised unique (RB_INSERT_ASSUME_UNIQUE)");
        if (!batch->advantage && batch->n > 0)
            invalid("rb_insert_owned: advantages required (groups span the shards of other ranks)");
        // the owned shard's arrival positions among the global batch (round robin
        // from the cursor, replay_buffer.cpp:89-90)
        const size_t T = b->T, j0 = (b->sb + T - b->h_cursor % T) % T;
        const size_t mine = n_global > j0 ? (n_global - 1 - j0) / T + 1 : 0;
        if (batch->n != mine)
            invalid("rb_insert_owned: the batch must hold exactly the owned shard's " +
                    std::to_string(mine) + " records of the global batch of " +
                    std::to_string(n_global));
        if (n_global == 0) return;
        if (batch->n == 0) {  // only the other shards' counters and the cursor advance
            b->other_work();  // no insert plan is pending for a sampler
            b->sync_checked();
            for (size_t j = 0; j < n_global; ++j) b->h_pushes[(b->h_cursor + j) % T]++;
            b->h_cursor = (b->h_cursor + n_global) % T;
            DevCtl c;
            b->fetch(&c, b->v.ctl, sizeof c);
            c.cursor = b->h_cursor;
            RB_CUDA(cudaMemcpy(b->v.pushes, b->h_pushes.data(), T * sizeof(long long),
                               cudaMemcpyHostToDevice));
            RB_CUDA(cudaMemcpy(b->v.ctl, &c, sizeof c, cudaMemcpyHostToDevice));
            return;
        }
        b->own_n_global = n_global;
        struct Reset {
            rb_buffer* b;
            ~Reset() { b->own_n_global = 0; }
        } reset{b};
        const int st = rb_insert(b, batch, nullptr, nullptr, flags);
        if (st != RB_OK) throw Error(st, rb_last_error());
    });
}

int rb_push(rb_buffer* b, const rb_record* rec, const int32_t* tokens, const float* logp_old,
            int32_t n_tokens, rb_record* evicted, int* has_evicted) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->gather_early = false;
        if (has_evicted) *has_evicted = 0;
        if (n_tokens < 0 || n_tokens > b->max_tokens)
            invalid("rb_push: n_tokens exceeds max_tokens");
        rb_insert_batch bt{};
        bt.n = 1;
        const rb_record r = *rec;
        bt.rollout_id = &r.rollout_id;
        bt.prompt_id = &r.prompt_id;
        bt.group_id = &r.group_id;
        bt.creation_step = &r.creation_step;
        bt.policy_version = &r.policy_version;
        bt.reward = &r.reward;
        bt.is_correct = &r.is_correct;
        bt.behavior_logprob = &r.behavior_logprob;
        bt.advantage = &r.advantage;
        int64_t toff[2] = {0, n_tokens};
        if (tokens || logp_old) {
            bt.tok_offsets = toff;
            bt.tokens = tokens;
            bt.logp_old = logp_old;
        } else {
            bt.tok_offsets = toff;  // records the length (0) without payload
            toff[1] = 0;
        }
        uint64_t evid = NONE_ID;
        int st = rb_insert(b, &bt, &evid, nullptr, 0x100);
        if (st != RB_OK) throw Error(st, rb_last_error());
        if (evid != NONE_ID) {
            rb_record ev;
            RB_CUDA(cudaMemcpyAsync(&ev, b->s_evrec, sizeof ev, cudaMemcpyDeviceToHost, b->stream));
            RB_CUDA(cudaStreamSynchronize(b->stream));
            if (evicted) *evicted = ev;
            if (has_evicted) *has_evicted = 1;
        }
    });
}

int rb_sample(rb_buffer* b, size_t batch_size, rb_rng* rng, rb_record* out_records,
              int64_t* out_shard, int64_t* out_index, rb_use_event* out_events,
              int64_t batch_id, int64_t use_step) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        const size_t T = b->T;
        if (batch_size == 0 || batch_size % T != 0)  // replay_buffer.cpp:189-192
            invalid("ShardedReplayBuffer: batch size must be a positive multiple of the shard count");
        const size_t per = batch_size / T;
        // An asynchronous insert may have been rejected on the device (sticky
        // error): the fused sampler checks that itself (it freezes, applying
        // nothing); the serial without-replacement path, which sizes its
        // draws from the host mirrors, checks first.
        if (b->strategy != RB_UNIFORM_WITH_REPLACEMENT &&
            b->strategy != RB_PRIORITY_WITH_REPLACEMENT && b->async_unchecked)
            check_sticky(b);
        // The reference fails at the first empty (197-199) or too-small
        // (148-150, without replacement) shard after mutating earlier shards.
        size_t nsh = T;
        std::string err;
        for (size_t s = 0; s < T; ++s) {
            const long long occ = std::min<long long>(b->h_pushes[s], (long long)b->C);
            if (occ == 0) {
                nsh = s;
                err = "ShardedReplayBuffer: cannot sample from an empty shard";
                break;
            }
            const bool without = b->strategy == RB_UNIFORM_WITHOUT_REPLACEMENT ||
                                 b->strategy == RB_UNUSED_FIRST_WITHOUT_REPLACEMENT;
            if (without && (long long)per > occ) {
                nsh = s;
                err = "ShardedReplayBuffer: batch exceeds shard occupancy for sampling without "
                      "replacement";
                break;
            }
        }
        const size_t nsel = nsh * per;
        b->ensure_select(std::max<size_t>(batch_size, 1));
        const long long lo = (long long)std::min(b->sb * per, nsel);
        const long long hi = (long long)std::min(b->se * per, nsel);
        SampleArgs a{};
        a.nsh = (int)nsh;
        a.per = (long long)per;
        a.sel_shard = b->sel_shard;
        a.sel_index = b->sel_index;
        a.nsel = (long long)nsel;
        a.lo = lo;
        a.hi = hi;
        a.sel_slot = b->sel_slot;
        a.sel_len = b->sel_len;
        a.off = b->sel_off;
        a.totals = b->sel_total;
        a.acc = b->acc;
        a.units = b->units_sel;
        a.n_units = b->n_units_sel;
        a.verdict = b->pay_sync;
        a.own_only = b->owned_meta ? 1 : 0;
        a.chk_frozen = b->strategy == RB_PRIORITY_WITH_REPLACEMENT ? 1 : 0;
        if (b->owned_meta && b->strategy != RB_UNIFORM_WITH_REPLACEMENT)
            throw Error(RB_ELOGIC, "owned-metadata buffers sample uniformly with replacement");
        const unsigned nmap = (unsigned)std::max<size_t>(1, (nsel + MAP_SPC - 1) / MAP_SPC);
        if (nmap > (unsigned)GRID_MAX_CTAS) invalid("rb_sample: batch too large");
        bool fused = false;
        if (b->strategy == RB_UNIFORM_WITH_REPLACEMENT) {
            // One fused launch (ring generator + draws + map), a programmatic
            // dependent of the insert's payload copy when that is the last
            // kernel on the stream: it overlaps the copy and waits for the
            // route kernel's completion flag itself.
            for (size_t s = 0; s < nsh && s < (size_t)DRAW_NSH; ++s)
                a.occ[s] = std::min<long long>(b->h_pushes[s], (long long)b->C);
            a.occ_dev = nullptr;
            if (nsh > (size_t)DRAW_NSH) {  // occupancies for every shard, staged on the stream
                std::vector<long long> occ(nsh);
                for (size_t s = 0; s < nsh; ++s) occ[s] = std::min<long long>(b->h_pushes[s], (long long)b->C);
                long long* d = (long long*)b->dev_stage(nsh * sizeof(long long), rb_buffer::ST_OCC);
                RB_CUDA(cudaMemcpyAsync(d, occ.data(), nsh * sizeof(long long), cudaMemcpyHostToDevice,
                                        b->stream));
                RB_CUDA(cudaStreamSynchronize(b->stream));  // `occ` is a host temporary
                a.occ_dev = d;
            }
            // early-gather flags only when an early gather can follow
            a.early = b->early_gather_ok && !(nsel > 0 && (out_records || out_events));
            // The next call's blocks: twisted by the sampler's generator CTA
            // while the batch is small (it finishes inside the payload copy),
            // by the Rng's side-stream lookahead once that serial chain would
            // outlast it (measured: 8192 draws faster inside, 16384 beside).
            const bool side = b->lookahead && nsel > (size_t)b->lookahead_min_draws;
            a.gen_ahead = side ? 0 : 1;
            if (b->seg_used) {  // flags of a sampling call no early gather consumed
                RB_CUDA(cudaMemsetAsync(b->map_ctl->seg, 0, (size_t)b->seg_used * sizeof(int),
                                        b->stream));
                RB_CUDA(cudaMemsetAsync(&b->map_ctl->fin, 0, sizeof(int), b->stream));
                b->pdl_tail = false;  // the memsets are now the stream's tail
                b->seg_used = 0;
            }
            // a lookahead this buffer already joined on its stream needs no
            // second wait (which would sit between the payload and the sampler)
            if (rng->gen_pending && rng->uid == b->joined_uid && rng->gen_seq == b->joined_seq)
                rng->gen_pending = false;
            MtRing* ring = rng->to_device(b->stream);
            if (b->pdl_tail) a.pend = b->pend;  // the insert just enqueued may still run
            b->gather_epoch = a.pend.pending ? a.pend.epoch : b->gather_epoch;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nmap + 1);
            cfg.blockDim = dim3(MAP_THREADS);
            cfg.stream = b->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = b->pdl_tail ? 1 : 0;
            const int* route_done = b->pay_sync + 1;
            RB_CUDA(cudaLaunchKernelEx(&cfg, k_sample_fused, b->v, ring, a, b->map_ctl, route_done));
            rng->used_on(b->stream);
            fused = true;
            // the next call's MT blocks, twisted beside the rest of the step
            if (side) rng->launch_lookahead(b->stream, (unsigned long long)nsel);
            if (rng->gen_pending) {
                if (!b->look_ev) RB_CUDA(cudaEventCreateWithFlags(&b->look_ev, cudaEventDisableTiming));
                RB_CUDA(cudaEventRecord(b->look_ev, rng->gen_stream));
                b->look_captured = rng->gen_captured;
                b->look_pending = true;
                b->look_uid = rng->uid;
                b->look_seq = rng->gen_seq;
            }
            b->seg_used = a.early ? (int)nmap : 0;
        } else {
            MtRing* ring = rng->to_device(b->stream);
            if (nsh > 0 && b->strategy == RB_PRIORITY_WITH_REPLACEMENT) {
                // several shards' records at once when they all fit in shared memory
                const size_t cap = (b->T > 1 && b->N <= (size_t)PR_SMEM_CDF) ? b->N : b->C;
                const bool sm = cap <= (size_t)PR_SMEM_CDF;
                const size_t need_b = (size_t)pr_pad((long long)cap) * sizeof(unsigned long long) +
                                      PR_G * sizeof(int);
                const size_t smem = sm ? need_b : 0;
                auto* cdf = sm ? nullptr : (unsigned long long*)b->scratch(need_b + 16);
                static bool attr_set = false;  // per process; the attribute is per function
                if (!attr_set) {
                    RB_CUDA(cudaFuncSetAttribute(k_sample_prio<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)(pr_pad(PR_SMEM_CDF) * sizeof(unsigned long long) +
                                                       PR_G * sizeof(int))));
                    attr_set = true;
                }
                if (sm)
                    k_sample_prio<true><<<1, PR_THREADS, smem, b->stream>>>(b->v, ring, a, b->prio, cdf,
                                                                            (long long)cap);
                else
                    k_sample_prio<false><<<1, PR_THREADS, 0, b->stream>>>(b->v, ring, a, b->prio, cdf,
                                                                         (long long)cap);
                RB_CUDA(cudaGetLastError());
            } else if (nsh > 0) {
                int64_t* scr = (int64_t*)b->scratch(2 * b->C * sizeof(int64_t) + 16);
                k_sample_without<<<1, 32, 0, b->stream>>>(b->v, ring, a, b->strategy, scr);
                RB_CUDA(cudaGetLastError());
            }
            // (a programmatic launch of the map after the prioritised sampler
            // measured no faster: C4 sampling call 46.7 vs 42 us)
            k_sample_map<<<nmap, MAP_THREADS, 0, b->stream>>>(b->v, a, b->map_ctl, b->pay_sync + 1);
            RB_CUDA(cudaGetLastError());
            rng->used_on(b->stream);
            // prioritised: the next call's MT blocks, twisted on the Rng's side
            // stream beside the rest of the step (joined by the next to_device)
            if (nsh > 0 && b->strategy == RB_PRIORITY_WITH_REPLACEMENT && b->lookahead) {
                rng->launch_lookahead(b->stream, (unsigned long long)nsel);
                if (!b->look_ev) RB_CUDA(cudaEventCreateWithFlags(&b->look_ev, cudaEventDisableTiming));
                RB_CUDA(cudaEventRecord(b->look_ev, rng->gen_stream));
                b->look_captured = rng->gen_captured;
                b->look_pending = true;
                b->look_uid = rng->uid;
                b->look_seq = rng->gen_seq;
            }
        }
        b->pdl_tail = false;
        // the next rb_gather may overlap the sampler (and the insert before it)
        // when nothing else is enqueued after the sampler
        b->gather_early = fused && b->seg_used > 0;
        b->B = nsel;
        b->last_loss = -1;
        b->acc_norm_explicit = false;
        if (nsel > 0 && (out_records || out_events)) {
            rb_record* dr = out_records;
            rb_use_event* de = out_events;
            const bool hr = out_records && !is_device_ptr(out_records);
            const bool he = out_events && !is_device_ptr(out_events);
            char* scr = nullptr;
            if (hr || he) scr = (char*)b->dev_stage(nsel * (sizeof(rb_record) + sizeof(rb_use_event)), rb_buffer::ST_SAMPLE);
            if (hr) dr = (rb_record*)scr;
            if (he) de = (rb_use_event*)(scr + nsel * sizeof(rb_record));
            const unsigned grid = (unsigned)std::min<size_t>((nsel + 255) / 256, 1184);
            k_sample_records<<<grid, 256, 0, b->stream>>>(b->v, (long long)nsel, (long long)per,
                                                          b->sel_slot, dr, de, batch_id, use_step);
            RB_CUDA(cudaGetLastError());
            if (hr)
                RB_CUDA(cudaMemcpyAsync(out_records, dr, nsel * sizeof(rb_record),
                                        cudaMemcpyDeviceToHost, b->stream));
            if (he)
                RB_CUDA(cudaMemcpyAsync(out_events, de, nsel * sizeof(rb_use_event),
                                        cudaMemcpyDeviceToHost, b->stream));
        }
        if (nsel > 0 && (out_shard || out_index)) {
            // (shard, arrival index) as int64 pairs
            std::vector<int32_t> sh;
            if (out_shard) {
                if (is_device_ptr(out_shard)) {
                    rb_widen_i32(b->sel_shard, out_shard, nsel, b->stream);
                } else {
                    sh.resize(nsel);
                    RB_CUDA(cudaMemcpyAsync(sh.data(), b->sel_shard, nsel * 4,
                                            cudaMemcpyDeviceToHost, b->stream));
                }
            }
            if (out_index)
                RB_CUDA(cudaMemcpyAsync(out_index, b->sel_index, nsel * 8, cudaMemcpyDefault,
                                        b->stream));
            if (!sh.empty()) {
                b->sync();
                for (size_t i = 0; i < nsel; ++i) out_shard[i] = sh[i];
            }
        }
        const bool host_out = (out_records && !is_device_ptr(out_records)) ||
                              (out_events && !is_device_ptr(out_events)) ||
                              (out_index && !is_device_ptr(out_index));
        if (host_out) {
            b->sync();
            // results handed back while an asynchronous insert was rejected
            // would be those of an empty (frozen) batch: report the error
            if (b->async_unchecked) check_sticky(b);
        }
        if (!err.empty()) {
            b->sync();
            invalid(err);
        }
    });
}

int rb_batch_size(const rb_buffer* b, size_t* n) {
    std::lock_guard<std::recursive_mutex> lk(const_cast<rb_buffer*>(b)->mu);
    *n = b->B;
    return RB_OK;
}

int rb_batch_total_tokens(rb_buffer* b, int64_t* total) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        long long t[2];
        RB_CUDA(cudaMemcpyAsync(t, b->sel_total, sizeof t, cudaMemcpyDeviceToHost, b->stream));
        b->sync_checked();
        *total = t[0];
    });
}

int rb_gather(rb_buffer* b, int32_t* out_tokens, float* out_logp_old, int64_t* out_offsets) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        if (b->stride == 0 && (out_tokens || out_logp_old))
            invalid("rb_gather: buffer holds no token payload (max_tokens = 0)");
        require_aligned16(out_tokens, "rb_gather: out_tokens");
        require_aligned16(out_logp_old, "rb_gather: out_logp_old");
        const size_t per = b->T ? (b->B / b->T) : 0;
        const long long lo = (long long)std::min(b->sb * per, b->B);
        const long long hi = (long long)std::min(b->se * per, b->B);
        const long long nloc = hi - lo;
        const bool ht = out_tokens && !is_device_ptr(out_tokens);
        const bool hl = out_logp_old && !is_device_ptr(out_logp_old);
        long long total = 0;
        if (ht || hl) {
            long long t[2];
            b->fetch(t, b->sel_total, sizeof t);
            total = t[0];
        }
        int32_t* dt = out_tokens;
        float* dl = out_logp_old;
        char* stage = nullptr;
        const size_t pb = (((size_t)total + 3) & ~size_t(3)) * 4;
        if (ht || hl) stage = (char*)b->dev_stage(2 * pb + 16, rb_buffer::ST_GATHER);
        if (ht) dt = (int32_t*)stage;
        if (hl) dl = (float*)(stage + pb);
        // the previous gather's asynchronous download still reads the staging area
        if (b->gout_pending && stage) RB_CUDA(cudaStreamWaitEvent(b->stream, b->gather_done, 0));
        const bool early = b->gather_early;
        b->gather_early = false;  // one early gather per sampling call (it consumes the claims)
        if (nloc > 0 && (dt || dl) && early) {
            // programmatic dependent of the fused sampler: overlaps the insert
            constexpr int QU = UNIT_THREADS * GATHER_U;
            const int ups = std::max(1, (int)(((b->stride + 3) / 4 + QU - 1) / QU));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(b->grid_gather);
            cfg.blockDim = dim3(UNIT_THREADS);
            cfg.stream = b->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            RB_CUDA(cudaLaunchKernelEx(&cfg, k_gather_early<GATHER_U>, b->v,
                                       (const Unit*)b->units_sel, (int)nloc, lo, ups, b->map_ctl,
                                       b->seg_used, (const int*)(b->pay_sync + 2),
                                       b->gather_epoch, dt, dl));
            b->seg_used = 0;  // the early gather resets the flags it consumed
        } else if (nloc > 0 && (dt || dl)) {
            // the resident grid, or one CTA per work unit for small batches
            constexpr int QU = UNIT_THREADS * GATHER_U;
            const long long ups = (((long long)b->stride + 3) / 4 + 1 + QU - 1) / QU;
            const long long units = std::max<long long>(1, nloc * ups);
            const unsigned grid = (unsigned)std::min<long long>(b->grid_gather,
                                                                std::max<long long>(units, b->sms));
            if (b->chunk_major && b->stride > 2 * UNIT_THREADS * GATHER_U * 4)
                k_gather<GATHER_U, true><<<grid, UNIT_THREADS, 0, b->stream>>>(
                    b->v, b->units_sel, b->n_units_sel, (int)nloc, dt, dl);
            else
                k_gather<GATHER_U><<<grid, UNIT_THREADS, 0, b->stream>>>(
                    b->v, b->units_sel, b->n_units_sel, (int)nloc, dt, dl);
            RB_CUDA(cudaGetLastError());
        }
        // Pinned host outputs with rb_set_async_outputs: the download drains on
        // the copy stream (complete after rb_synchronize) while the caller's
        // next call runs, e.g. the loss's logp_now upload (full-duplex PCIe).
        const bool async_g = b->async_out && (ht || hl) && (!ht || is_pinned_ptr(out_tokens)) &&
                             (!hl || is_pinned_ptr(out_logp_old));
        cudaStream_t cs = b->stream;
        if (async_g) {
            b->ensure_copy_streams();
            if (!b->gather_ready) {
                RB_CUDA(cudaEventCreateWithFlags(&b->gather_ready, cudaEventDisableTiming));
                RB_CUDA(cudaEventCreateWithFlags(&b->gather_done, cudaEventDisableTiming));
            }
            RB_CUDA(cudaEventRecord(b->gather_ready, b->stream));
            RB_CUDA(cudaStreamWaitEvent(b->cs_out, b->gather_ready, 0));
            cs = b->cs_out;
        }
        if (ht) RB_CUDA(cudaMemcpyAsync(out_tokens, dt, total * 4, cudaMemcpyDeviceToHost, cs));
        if (hl) RB_CUDA(cudaMemcpyAsync(out_logp_old, dl, total * 4, cudaMemcpyDeviceToHost, cs));
        if (async_g) {
            RB_CUDA(cudaEventRecord(b->gather_done, b->cs_out));
            b->gout_pending = true;
        }
        const bool host_off = out_offsets && !is_device_ptr(out_offsets);
        if (host_off && is_pinned_ptr(out_offsets))  // kernel store into the mapped array
            b->to_host_async(out_offsets, b->sel_off, (nloc + 1) * 8);
        else if (out_offsets)
            RB_CUDA(cudaMemcpyAsync(out_offsets, b->sel_off, (nloc + 1) * 8, cudaMemcpyDefault,
                                    b->stream));
        if (((ht || hl) && !async_g) || host_off) b->sync_checked();
    });
}

// ---- DLPack export (ABI v0.8 structs, declared here: no header dependency)
namespace {
struct DLDevice_ { int32_t device_type, device_id; };  // kDLCUDA = 2
struct DLDataType_ { uint8_t code, bits; uint16_t lanes; };  // kDLInt 0, kDLFloat 2
struct DLTensor_ {
    void* data;
    DLDevice_ device;
    int32_t ndim;
    DLDataType_ dtype;
    int64_t* shape;
    int64_t* strides;
    uint64_t byte_offset;
};
struct DLManagedTensor_ {
    DLTensor_ dl_tensor;
    void* manager_ctx;
    void (*deleter)(DLManagedTensor_*);
};
struct DlHolder {
    DLManagedTensor_ mt;
    int64_t shape[1];
    void* mem;
    int device;
};
void dl_delete(DLManagedTensor_* m) {
    DlHolder* h = static_cast<DlHolder*>(m->manager_ctx);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    cudaFree(h->mem);
    cudaSetDevice(prev);
    delete h;
}
DlHolder* dl_alloc(int device, int64_t n, uint8_t code, uint8_t bits) {
    DlHolder* h = new DlHolder();
    h->device = device;
    h->shape[0] = n;
    if (cudaMalloc(&h->mem, (size_t)std::max<int64_t>(n, 1) * (bits / 8) + 16) != cudaSuccess) {
        delete h;
        throw Error(RB_ECUDA, "rb_gather_dlpack: device allocation failed");
    }
    DLTensor_& t = h->mt.dl_tensor;
    t.data = h->mem;
    t.device = DLDevice_{2, device};
    t.ndim = 1;
    t.dtype = DLDataType_{code, bits, 1};
    t.shape = h->shape;
    t.strides = nullptr;  // compact
    t.byte_offset = 0;
    h->mt.manager_ctx = h;
    h->mt.deleter = dl_delete;
    return h;
}
}  // namespace

void rb_dlpack_free(void* managed_tensor) {
    if (auto* m = static_cast<DLManagedTensor_*>(managed_tensor))
        if (m->deleter) m->deleter(m);
}

int rb_gather_dlpack(rb_buffer* b, void** out_tokens, void** out_logp_old, void** out_offsets) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        if (b->stride == 0 && (out_tokens || out_logp_old))
            invalid("rb_gather_dlpack: buffer holds no token payload (max_tokens = 0)");
        const size_t per = b->T ? (b->B / b->T) : 0;
        const long long lo = (long long)std::min(b->sb * per, b->B);
        const long long hi = (long long)std::min(b->se * per, b->B);
        const long long nloc = hi - lo;
        long long t[2] = {0, 0};
        RB_CUDA(cudaMemcpyAsync(t, b->sel_total, sizeof t, cudaMemcpyDeviceToHost, b->stream));
        b->sync_checked();
        std::unique_ptr<DlHolder, void (*)(DlHolder*)> ht(nullptr, [](DlHolder* h) { if (h) dl_delete(&h->mt); }),
            hl(nullptr, [](DlHolder* h) { if (h) dl_delete(&h->mt); }),
            ho(nullptr, [](DlHolder* h) { if (h) dl_delete(&h->mt); });
        if (out_tokens) ht.reset(dl_alloc(b->device, t[0], 0, 32));
        if (out_logp_old) hl.reset(dl_alloc(b->device, t[0], 2, 32));
        if (out_offsets) ho.reset(dl_alloc(b->device, nloc + 1, 0, 64));
        const int rc = rb_gather(b, ht ? (int32_t*)ht->mem : nullptr, hl ? (float*)hl->mem : nullptr,
                                 ho ? (int64_t*)ho->mem : nullptr);
        if (rc != RB_OK) throw Error(rc, rb_last_error());
        b->sync_checked();  // the arrays are complete for a consumer on any stream
        if (out_tokens) *out_tokens = &ht.release()->mt;
        if (out_logp_old) *out_logp_old = &hl.release()->mt;
        if (out_offsets) *out_offsets = &ho.release()->mt;
    });
}

int rb_batch_ids(rb_buffer* b, uint64_t* out_ids, int32_t* out_lengths, int64_t* out_offsets) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        const size_t per = b->T ? (b->B / b->T) : 0;
        const long long lo = (long long)std::min(b->sb * per, b->B);
        const long long hi = (long long)std::min(b->se * per, b->B);
        const long long n = hi - lo;
        const bool hid = out_ids && !is_device_ptr(out_ids);
        const bool hlen = out_lengths && !is_device_ptr(out_lengths);
        char* st = (char*)b->dev_stage(n * 12 + 64, rb_buffer::ST_IDS);
        uint64_t* di = hid ? (uint64_t*)st : out_ids;
        int32_t* dlen = hlen ? (int32_t*)(st + n * 8 + 16) : out_lengths;
        if (n > 0) rb_batch_ids_dev(b->v, b->sel_slot, lo, hi, di, dlen, b->stream);
        if (hid) RB_CUDA(cudaMemcpyAsync(out_ids, di, n * 8, cudaMemcpyDeviceToHost, b->stream));
        if (hlen) RB_CUDA(cudaMemcpyAsync(out_lengths, dlen, n * 4, cudaMemcpyDeviceToHost, b->stream));
        if (out_offsets)
            RB_CUDA(cudaMemcpyAsync(out_offsets, b->sel_off, (n + 1) * 8, cudaMemcpyDefault, b->stream));
        if (hid || hlen || (out_offsets && !is_device_ptr(out_offsets))) b->sync_checked();
    });
}

int rb_num_shards(const rb_buffer* b, size_t* out) {
    *out = b->T;
    return RB_OK;
}
int rb_total_capacity(const rb_buffer* b, size_t* out) {
    *out = b->N;
    return RB_OK;
}
int rb_shard_capacity(const rb_buffer* b, size_t* out) {
    *out = b->C;
    return RB_OK;
}
int rb_size(rb_buffer* b, size_t* out) {
    std::lock_guard<std::recursive_mutex> lk(b->mu);
    size_t t = 0;
    for (size_t s = 0; s < b->T; ++s) t += (size_t)std::min<long long>(b->h_pushes[s], (long long)b->C);
    *out = t;
    return RB_OK;
}
int rb_shard_size(rb_buffer* b, size_t shard, size_t* out) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        if (shard >= b->T) throw Error(RB_ELOGIC, "vector::_M_range_check: shard out of range");
        *out = (size_t)std::min<long long>(b->h_pushes[shard], (long long)b->C);
    });
}
int rb_shard_contents(rb_buffer* b, size_t shard, rb_record* out, size_t capacity,
                      size_t* count) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        if (shard >= b->T) throw Error(RB_ELOGIC, "vector::_M_range_check: shard out of range");
        const size_t n = (size_t)std::min<long long>(b->h_pushes[shard], (long long)b->C);
        *count = n;
        if (!out || n == 0) return;
        if (capacity < n) invalid("rb_shard_contents: output too small");
        rb_record* d = (rb_record*)b->dev_stage(n * sizeof(rb_record), rb_buffer::ST_INSPECT);
        k_shard_contents<<<(unsigned)std::min<size_t>((n + 255) / 256, 1024), 256, 0, b->stream>>>(
            b->v, (int)shard, (long long)n, d);
        RB_CUDA(cudaGetLastError());
        RB_CUDA(cudaMemcpyAsync(out, d, n * sizeof(rb_record), cudaMemcpyDefault, b->stream));
        b->sync();
    });
}

int rb_record_tokens(rb_buffer* b, size_t shard, size_t index, int32_t* tokens,
                     float* logp_old, int32_t capacity, int32_t* n_tokens) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        if (shard >= b->T) invalid("rb_record_tokens: shard out of range");
        const size_t n = (size_t)std::min<long long>(b->h_pushes[shard], (long long)b->C);
        if (index >= n) invalid("rb_record_tokens: index out of range");
        if (shard < b->sb || shard >= b->se) invalid("rb_record_tokens: shard not held here");
        int32_t* d = (int32_t*)b->scratch(64);
        k_slot_of<<<1, 1, 0, b->stream>>>(b->v, (int)shard, (long long)index, d);
        int32_t g = 0, len = 0;
        RB_CUDA(cudaMemcpyAsync(&g, d, 4, cudaMemcpyDeviceToHost, b->stream));
        b->sync();
        RB_CUDA(cudaMemcpy(&len, b->v.len + g, 4, cudaMemcpyDeviceToHost));
        *n_tokens = len;
        if (len > capacity) invalid("rb_record_tokens: output too small");
        const size_t row = ((size_t)(shard - b->sb) * b->C + (g % b->C)) * (size_t)b->stride;
        if (tokens) RB_CUDA(cudaMemcpy(tokens, b->v.tok + row, len * 4, cudaMemcpyDefault));
        if (logp_old) RB_CUDA(cudaMemcpy(logp_old, b->v.lpo + row, len * 4, cudaMemcpyDefault));
    });
}

int rb_strategy(const rb_buffer* b, int* out) {
    *out = b->strategy;
    return RB_OK;
}
extern "C++" {
namespace rb {
void prio_mass_launch(rb_buffer* b, unsigned long long* out) {
    RB_CUDA(cudaMemsetAsync(out, 0, b->T * sizeof(unsigned long long), b->stream));
    k_prio_mass<<<(unsigned)(b->se - b->sb), 256, 0, b->stream>>>(b->v, b->prio, out);
    RB_CUDA(cudaGetLastError());
}
}  // namespace rb
}  // extern "C++"

int rb_priority_mass(rb_buffer* b, uint64_t* out) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);
        DeviceScope ds(b->device);
        if (!out) invalid("rb_priority_mass: NULL output");
        if (b->async_unchecked) check_sticky(b);
        b->other_work();
        const bool host = !is_device_ptr(out);
        auto* d = host ? (unsigned long long*)b->scratch(b->T * sizeof(uint64_t))
                       : (unsigned long long*)out;
        rb::prio_mass_launch(b, d);
        if (host) {
            RB_CUDA(cudaMemcpyAsync(out, d, b->T * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    b->stream));
            b->sync();
        }
    });
}

// priority_with_replacement weights (builder extension; k_sample_prio).
int rb_set_priority(rb_buffer* b, uint32_t base, uint32_t adv_scale, uint32_t pos_bonus) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);
        if (base == 0) invalid("rb_set_priority: base weight must be >= 1");
        if (adv_scale > 65536u) invalid("rb_set_priority: adv_scale must be <= 65536");
        b->prio = rb::PrioParams{base, adv_scale, pos_bonus};
    });
}
int rb_get_priority(const rb_buffer* b, uint32_t* base, uint32_t* adv_scale, uint32_t* pos_bonus) {
    *base = b->prio.base;
    *adv_scale = b->prio.adv_scale;
    *pos_bonus = b->prio.pos_bonus;
    return RB_OK;
}
int rb_retention(const rb_buffer* b, int* kind, double* delta) {
    *kind = b->retention;
    *delta = b->delta;
    return RB_OK;
}
int rb_route_cursor(rb_buffer* b, size_t* out) {
    std::lock_guard<std::recursive_mutex> lk(b->mu);
    *out = b->h_cursor;
    return RB_OK;
}

namespace {
// ---- replay diagnostics ------------------------------------------------------
// Histogram of integer values (shared-memory bins, one global atomic per bin
// per CTA) and their sum.
__global__ void k_hist_staleness(const BufView v, const int32_t* sel_slot, long long n,
                                 long long use_step, int max_bin, unsigned long long* hist,
                                 long long* sum) {
    extern __shared__ unsigned long long sh[];
    for (int i = threadIdx.x; i <= max_bin; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    long long s = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long st = use_step - v.cstep[sel_slot[i]];  // metrics.cpp:37-39
        s += st;
        const long long b = st < 0 ? 0 : (st > max_bin ? max_bin : st);
        atomicAdd(&sh[b], 1ULL);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= max_bin; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
    s = warp_sum_i64(s);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd((unsigned long long*)sum, (unsigned long long)s);
}
__global__ void k_hist_use(const BufView v, int max_bin, unsigned long long* hist,
                           unsigned long long* sum) {
    extern __shared__ unsigned long long sh[];
    for (int i = threadIdx.x; i <= max_bin; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    unsigned long long s = 0;
    const long long N = (long long)v.T * v.C;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < N;
         g += (long long)gridDim.x * blockDim.x) {
        const int sh_ = (int)(g / v.C), x = (int)(g % v.C);
        if (x >= occupancy(v, sh_)) continue;  // resident slots only
        const unsigned u = v.use[g];
        s += u;
        atomicAdd(&sh[u > (unsigned)max_bin ? max_bin : u], 1ULL);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= max_bin; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
    s = (unsigned long long)warp_sum_i64((long long)s);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(sum, s);
}
}  // namespace
}  // extern "C"
namespace {
template <class T, class F>
void run_hist(rb_buffer* b, int32_t max_bin, uint64_t* hist, T* sum, F launch) {
    if (max_bin < 0 || max_bin > 4095) invalid("histogram: max_bin must be in [0, 4095]");
    const size_t hb = ((size_t)max_bin + 1) * 8;
    char* d = (char*)b->scratch(hb + 16);
    RB_CUDA(cudaMemsetAsync(d, 0, hb + 16, b->stream));
    launch((unsigned long long*)d, (T*)(d + hb), (size_t)hb);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaMemcpyAsync(hist, d, hb, cudaMemcpyDefault, b->stream));
    if (sum) RB_CUDA(cudaMemcpyAsync(sum, d + hb, sizeof(T), cudaMemcpyDefault, b->stream));
    b->sync();
}
}  // namespace
extern "C" {
namespace {

// ---- binary snapshot (rb_snapshot / rb_restore) ---------------------------
struct SnapHeader {
    char magic[8];  // "RBSNAP01"
    uint64_t T, N, C;
    int32_t max_tokens, strategy, retention, pad;
    double delta;
    uint64_t sb, se, sections;
};
struct Section {
    void* ptr;
    size_t bytes;
};
std::vector<Section> snap_sections(rb_buffer* b) {
    const BufView& v = b->v;
    const size_t N = b->N, T = b->T, C = b->C;
    std::vector<Section> s = {
        {v.ctl, sizeof(DevCtl)}, {v.pushes, T * 8}, {v.id, N * 8}, {v.prompt, N * 8},
        {v.group, N * 8}, {v.cstep, N * 8}, {v.pver, N * 8}, {v.reward, N * 8}, {v.blp, N * 8},
        {v.adv, N * 8}, {v.gmean, N * 8}, {v.correct, N}, {v.use, N * 4}, {v.len, N * 4},
        {v.order, N * 4}};
    if (b->retention == RB_POSITIVE_BIAS) {
        s.push_back({v.pbq, 3 * T * (C + 1) * 4});
        s.push_back({v.pbs, T * sizeof(PbState)});
        s.push_back({v.seq, N * 8});
    }
    const size_t rows = (b->se - b->sb) * C * (size_t)b->stride;
    if (rows) {
        s.push_back({v.tok, rows * 4});
        s.push_back({v.lpo, rows * 4});
    }
    return s;
}
SnapHeader snap_header(rb_buffer* b, size_t nsec) {
    SnapHeader h{};
    std::memcpy(h.magic, "RBSNAP01", 8);
    h.T = b->T;
    h.N = b->N;
    h.C = b->C;
    h.max_tokens = b->max_tokens;
    h.strategy = b->strategy;
    h.retention = b->retention;
    h.delta = b->delta;
    h.sb = b->sb;
    h.se = b->se;
    h.sections = nsec;
    return h;
}
}  // namespace

int rb_batch_staleness_hist(rb_buffer* b, int64_t use_step, int32_t max_bin, uint64_t* hist,
                            int64_t* sum) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        run_hist(b, max_bin, hist, sum, [&](unsigned long long* h, int64_t* sm, size_t hb) {
            if (b->B)
                k_hist_staleness<<<std::max<unsigned>(1, std::min<unsigned>((unsigned)((b->B + 255) / 256), 148)),
                                   256, hb, b->stream>>>(b->v, b->sel_slot, (long long)b->B,
                                                         (long long)use_step, max_bin, h,
                                                         (long long*)sm);
        });
    });
}

int rb_use_count_hist(rb_buffer* b, int32_t max_bin, uint64_t* hist, uint64_t* sum) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        run_hist(b, max_bin, hist, sum, [&](unsigned long long* h, uint64_t* sm, size_t hb) {
            k_hist_use<<<std::max<unsigned>(1, std::min<unsigned>((unsigned)((b->N + 255) / 256), 148)),
                         256, hb, b->stream>>>(b->v, max_bin, h, (unsigned long long*)sm);
        });
    });
}

int rb_snapshot(rb_buffer* b, void* dst, size_t cap, size_t* len) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        const auto secs = snap_sections(b);
        size_t total = sizeof(SnapHeader);
        for (auto& x : secs) total += 8 + x.bytes;
        if (len) *len = total;
        if (!dst) return;
        if (cap < total) invalid("rb_snapshot: destination too small");
        check_sticky(b);  // synchronises; the state is consistent
        const SnapHeader h = snap_header(b, secs.size());
        char* o = (char*)dst;
        RB_CUDA(cudaMemcpy(o, &h, sizeof h, cudaMemcpyDefault));
        o += sizeof h;
        for (auto& x : secs) {
            const uint64_t n = x.bytes;
            RB_CUDA(cudaMemcpy(o, &n, 8, cudaMemcpyDefault));
            RB_CUDA(cudaMemcpy(o + 8, x.ptr, x.bytes, cudaMemcpyDefault));
            o += 8 + x.bytes;
        }
    });
}

int rb_restore(rb_buffer* b, const void* src, size_t len) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->other_work();
        const auto secs = snap_sections(b);
        SnapHeader h;
        if (!src || len < sizeof h) invalid("rb_restore: snapshot truncated");
        RB_CUDA(cudaMemcpy(&h, src, sizeof h, cudaMemcpyDefault));
        const SnapHeader want = snap_header(b, secs.size());
        if (std::memcmp(h.magic, want.magic, 8) != 0) invalid("rb_restore: not a buffer snapshot");
        if (h.T != want.T || h.N != want.N || h.C != want.C || h.max_tokens != want.max_tokens ||
            h.strategy != want.strategy || h.retention != want.retention ||
            h.delta != want.delta || h.sb != want.sb || h.se != want.se ||
            h.sections != want.sections)
            invalid("rb_restore: snapshot of a buffer with a different shape");
        size_t total = sizeof h;
        for (auto& x : secs) total += 8 + x.bytes;
        if (len < total) invalid("rb_restore: snapshot truncated");
        b->sync();
        const char* o = (const char*)src + sizeof h;
        for (auto& x : secs) {
            uint64_t n = 0;
            RB_CUDA(cudaMemcpy(&n, o, 8, cudaMemcpyDefault));
            if (n != x.bytes) invalid("rb_restore: section size mismatch");
            RB_CUDA(cudaMemcpy(x.ptr, o + 8, x.bytes, cudaMemcpyDefault));
            o += 8 + x.bytes;
        }
        // host mirrors from the restored device state
        DevCtl c;
        RB_CUDA(cudaMemcpy(&c, b->v.ctl, sizeof c, cudaMemcpyDeviceToHost));
        RB_CUDA(cudaMemcpy(b->h_pushes.data(), b->v.pushes, b->T * 8, cudaMemcpyDeviceToHost));
        b->h_cursor = (size_t)c.cursor;
        b->B = 0;  // no current batch after a restore
    });
}

int rb_check(rb_buffer* b) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        check_sticky(b);
    });
}
int rb_synchronize(rb_buffer* b) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        b->join_lookahead();
        b->sync();
        b->drain_outputs();
    });
}

int rb_set_async_outputs(rb_buffer* b, int on) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        DeviceScope ds(b->device);
        if (!on) b->drain_outputs();
        b->async_out = on != 0;
    });
}

// replay_buffer.cpp:238-255
int rb_dump(rb_buffer* b, char* out, size_t cap, size_t* len) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lk(b->mu);  // one total order (replay_buffer.cpp:84, 188)
        std::string s;
        s += "# sharded_replay_buffer v1\n";
        s += "# shards = " + std::to_string(b->T) + "\n";
        s += "# capacity = " + std::to_string(b->N) + "\n";
        s += "# strategy = " + strategy_name(b->strategy) + "\n";
        s += "# retention = " +
             std::string(b->retention == RB_PLAIN_FIFO ? "plain_fifo"
                                                       : "positive_bias delta=" + fmt_double(b->delta)) +
             "\n";
        s += "# route_cursor = " + std::to_string(b->h_cursor) + "\n";
        std::vector<rb_record> recs(b->C + 1);
        for (size_t sh = 0; sh < b->T; ++sh) {
            s += "# shard " + std::to_string(sh) + "\n";
            size_t n = 0;
            int st = rb_shard_contents(b, sh, recs.data(), recs.size(), &n);
            if (st != RB_OK) throw Error(st, rb_last_error());
            for (size_t i = 0; i < n; ++i) {  // rollout.cpp:9-15
                const rb_record& r = recs[i];
                s += std::to_string(r.rollout_id) + "," + std::to_string(r.prompt_id) + "," +
                     std::to_string(r.group_id) + "," + std::to_string(r.creation_step) + "," +
                     std::to_string(r.policy_version) + "," + fmt_double(r.reward) + "," +
                     (r.is_correct ? "1" : "0") + "," + fmt_double(r.behavior_logprob) + "," +
                     fmt_double(r.advantage) + "," + std::to_string(r.use_count) + "\n";
            }
        }
        *len = s.size();
        if (out && cap) {
            const size_t m = std::min(s.size(), cap - 1);
            std::memcpy(out, s.data(), m);
            out[m] = 0;
        }
    });
}

}  // extern "C"

// ---- load (replay_buffer.cpp:276-324) -----------------------------------
namespace {
std::string_view trim(std::string_view s) {  // text_io trim
    size_t a = 0, e = s.size();
    while (a < e && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r' || s[a] == '\n')) ++a;
    while (e > a && (s[e - 1] == ' ' || s[e - 1] == '\t' || s[e - 1] == '\r' || s[e - 1] == '\n')) --e;
    return s.substr(a, e - a);
}
[[noreturn]] void bad_field(std::string_view what, std::string_view text) {
    invalid(std::string(what) + ": '" + std::string(text) + "'");
}
uint64_t parse_u64(std::string_view t0) {
    auto t = trim(t0);
    uint64_t v = 0;
    auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec != std::errc() || r.ptr != t.data() + t.size() || t.empty())
        bad_field("not an unsigned integer", t0);
    return v;
}
int64_t parse_i64(std::string_view t0) {
    auto t = trim(t0);
    int64_t v = 0;
    auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec != std::errc() || r.ptr != t.data() + t.size() || t.empty())
        bad_field("not an integer", t0);
    return v;
}
double parse_f64(std::string_view t0) {
    auto t = trim(t0);
    double v = 0;
    auto r = std::from_chars(t.data(), t.data() + t.size(), v);
    if (r.ec != std::errc() || r.ptr != t.data() + t.size() || t.empty())
        bad_field("not a number", t0);
    return v;
}
bool parse_bool(std::string_view t0) {
    auto t = trim(t0);
    if (t == "true" || t == "1") return true;
    if (t == "false" || t == "0") return false;
    bad_field("not a boolean", t0);
}
std::vector<std::string_view> split(std::string_view s, char d) {
    std::vector<std::string_view> out;
    size_t a = 0;
    for (;;) {
        size_t e = s.find(d, a);
        if (e == std::string_view::npos) {
            out.push_back(s.substr(a));
            return out;
        }
        out.push_back(s.substr(a, e - a));
        a = e + 1;
    }
}
std::string_view header_value(std::string_view line, std::string_view key) {
    const size_t eq = line.find('=');
    if (eq == std::string_view::npos)
        invalid("buffer dump: malformed header line '" + std::string(line) + "'");
    const std::string_view name = trim(line.substr(1, eq - 1));
    if (name != key)
        invalid("buffer dump: expected header '" + std::string(key) + "', got '" + std::string(name) + "'");
    return trim(line.substr(eq + 1));
}
rb_record record_from_line(std::string_view line) {  // rollout.cpp:17-35
    const auto f = split(line, ',');
    if (f.size() != 10)
        invalid("RolloutRecord: expected 10 fields, got " + std::to_string(f.size()));
    rb_record r{};
    r.rollout_id = parse_u64(f[0]);
    r.prompt_id = parse_u64(f[1]);
    r.group_id = parse_u64(f[2]);
    r.creation_step = parse_i64(f[3]);
    r.policy_version = parse_i64(f[4]);
    r.reward = parse_f64(f[5]);
    r.is_correct = parse_bool(f[6]);
    r.behavior_logprob = parse_f64(f[7]);
    r.advantage = parse_f64(f[8]);
    r.use_count = (uint32_t)parse_u64(f[9]);
    return r;
}
}  // namespace

extern "C" int rb_load(const char* text, int32_t max_tokens, int device, rb_buffer** out) {
    return guard([&] {
        std::vector<std::string> lines;
        for (auto l : split(text, '\n')) {
            auto t = trim(l);
            if (!t.empty()) lines.emplace_back(t);
        }
        if (lines.size() < 6 || lines[0] != "# sharded_replay_buffer v1")
            invalid("buffer dump: missing or unsupported header");
        const uint64_t T = parse_u64(header_value(lines[1], "shards"));
        const uint64_t N = parse_u64(header_value(lines[2], "capacity"));
        const std::string_view sname = header_value(lines[3], "strategy");
        int strategy;
        if (sname == "uniform_with_replacement") strategy = 0;
        else if (sname == "uniform_without_replacement") strategy = 1;
        else if (sname == "unused_first_without_replacement") strategy = 2;
        else if (sname == "priority_with_replacement") strategy = 3;
        else invalid("unknown sampling strategy: '" + std::string(sname) + "'");
        const std::string_view rname = header_value(lines[4], "retention");
        int retention = RB_PLAIN_FIFO;
        double delta = 0.0;
        constexpr std::string_view kPrefix = "positive_bias delta=";
        if (rname == "plain_fifo") {
        } else if (rname.substr(0, kPrefix.size()) == kPrefix) {
            retention = RB_POSITIVE_BIAS;
            delta = parse_f64(rname.substr(kPrefix.size()));
            if (!(delta >= 0.0) || !(delta <= 1.0)) invalid("RetentionPolicy: delta must be in [0, 1]");
        } else {
            invalid("unknown retention policy: '" + std::string(rname) + "'");
        }
        const uint64_t cursor = parse_u64(header_value(lines[5], "route_cursor"));
        rb_buffer* b = create(T, N, strategy, retention, delta, max_tokens, device, 0, 0);
        try {
            if (cursor >= T) invalid("buffer dump: route cursor out of range");
            std::vector<std::vector<rb_record>> shards(T);
            std::unordered_set<uint64_t> ids;
            size_t shard = 0;
            bool in_shard = false;
            for (size_t i = 6; i < lines.size(); ++i) {
                const std::string& line = lines[i];
                if (line.rfind("# shard ", 0) == 0) {
                    shard = parse_u64(std::string_view(line).substr(8));
                    if (shard >= T) invalid("buffer dump: shard index out of range");
                    in_shard = true;
                    continue;
                }
                if (!in_shard) invalid("buffer dump: record before any shard marker");
                shards[shard].push_back(record_from_line(line));
                if (shards[shard].size() > b->C) invalid("buffer dump: shard exceeds capacity");
                if (!ids.insert(shards[shard].back().rollout_id).second)
                    invalid("buffer dump: duplicate rollout id " +
                            std::to_string(shards[shard].back().rollout_id));
            }
            DeviceScope ds(b->device);
        b->other_work();
            unsigned long long mx = 0;
            for (size_t s = 0; s < T; ++s) {
                const size_t n = shards[s].size();
                b->h_pushes[s] = (long long)n;
                for (auto& r : shards[s]) mx = std::max<unsigned long long>(mx, r.rollout_id);
                if (!n) continue;
                rb_record* d = (rb_record*)b->dev_stage(n * sizeof(rb_record), rb_buffer::ST_INSPECT);
                RB_CUDA(cudaMemcpyAsync(d, shards[s].data(), n * sizeof(rb_record),
                                        cudaMemcpyHostToDevice, b->stream));
                k_load_shard<<<(unsigned)((n + 255) / 256), 256, 0, b->stream>>>(b->v, (int)s,
                                                                                (long long)n, d);
                RB_CUDA(cudaGetLastError());
                if (b->retention == RB_POSITIVE_BIAS) {
                    k_load_posbias<<<1, 32, 0, b->stream>>>(b->v, (int)s, (int)n, d);
                    RB_CUDA(cudaGetLastError());
                }
                b->sync();
            }
            RB_CUDA(cudaMemcpy(b->v.pushes, b->h_pushes.data(), T * sizeof(long long),
                               cudaMemcpyHostToDevice));
            DevCtl c{};
            c.cursor = cursor;
            c.max_id = mx;
            c.has_any = ids.empty() ? 0 : 1;
            c.hash_stale = 1;
            RB_CUDA(cudaMemcpy(b->v.ctl, &c, sizeof c, cudaMemcpyHostToDevice));
            b->h_cursor = cursor;
        } catch (...) {
            delete b;
            throw;
        }
        *out = b;
    });
}

// ---- small helper kernels referenced above --------------------------------
namespace {
__global__ void k_lengths(const int64_t* toff, long long n, int32_t* len, int32_t maxlen,
                          DevCtl* ctl) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n;
         j += (long long)gridDim.x * blockDim.x) {
        long long l = toff[j + 1] - toff[j];
        if (l < 0 || l > maxlen) {
            ctl->err_code = RB_EINVAL;
            ctl->err_index = -3;
            l = 0;
        }
        len[j] = (int32_t)l;
    }
}
__global__ void k_widen(const int32_t* a, int64_t* b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = a[i];
}
__global__ void k_batch_ids(BufView v, const int32_t* sel_slot, long long lo, long long hi,
                            uint64_t* ids, int32_t* lens) {
    for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi;
         i += (long long)gridDim.x * blockDim.x) {
        const int g = sel_slot[i];
        if (ids) ids[i - lo] = v.id[g];
        if (lens) lens[i - lo] = v.len[g];
    }
}
}  // namespace

void rb_lengths_from_offsets(const int64_t* toff, size_t n, int32_t* len, int32_t maxlen,
                             DevCtl* ctl, cudaStream_t s) {
    k_lengths<<<(unsigned)std::min<size_t>((n + 255) / 256, 1024), 256, 0, s>>>(toff, (long long)n, len,
                                                                                maxlen, ctl);
    RB_CUDA(cudaGetLastError());
}
void rb_widen_i32(const int32_t* a, int64_t* b, size_t n, cudaStream_t s) {
    k_widen<<<(unsigned)std::min<size_t>((n + 255) / 256, 1024), 256, 0, s>>>(a, b, (long long)n);
    RB_CUDA(cudaGetLastError());
}
void rb_batch_ids_dev(const BufView& v, const int32_t* sel_slot, long long lo, long long hi,
                      uint64_t* ids, int32_t* lens, cudaStream_t s) {
    const long long n = hi - lo;
    k_batch_ids<<<(unsigned)std::min<long long>((n + 255) / 256, 1024), 256, 0, s>>>(v, sel_slot, lo, hi,
                                                                                    ids, lens);
    RB_CUDA(cudaGetLastError());
}

// Tuning aid: phase clocks of the single-CTA kernels (zeros unless the
// library was built with -DRB_PHASE_CLOCKS).
extern "C" __attribute__((visibility("default"))) int rb_debug_timeline(unsigned long long* out,
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

extern "C" __attribute__((visibility("default"))) int rb_debug_locb(long long* out) {
    return guard([&] { RB_CUDA(cudaMemcpyFromSymbol(out, g_dbg_locb, 2 * sizeof(long long))); });
}
extern "C" __attribute__((visibility("default"))) int rb_debug_phase_clocks(long long* out) {
    return guard([&] {
#ifdef RB_PHASE_CLOCKS
        RB_CUDA(cudaMemcpyFromSymbol(out, g_phase_clock, 64 * sizeof(long long)));
#else
        for (int i = 0; i < 64; ++i) out[i] = 0;
#endif
    });
}
