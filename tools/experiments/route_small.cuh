// ---- FIFO route for small batches: one CTA, one memory round trip ---------
// k_route_fifo's semantics (replay_buffer.cpp:83-96 closed form, group
// advantages bandit.cpp:276-294) for batches of at most RS_NMAX records over
// <= 64 shards, without its grid-wide done counter and last-CTA pass: the
// per-shard push counts come from the host mirrors (exact on this path, as
// for the closed-form payload copy), so every slot, survivor and evictee is
// known before any load; the batch (ids, rewards, offsets, group offsets)
// and the evictees' ids are all loaded at once into registers / shared
// memory, validated, and the records applied by the same 1024 threads.  The
// verdict and done flags, the offsets copy for an overlapping sampler and
// the counters follow k_route_fifo's protocol.
constexpr int RS_THREADS = 1024;
constexpr int RS_PER = 2;
constexpr int RS_NMAX = RS_THREADS * RS_PER;
constexpr int RS_GMAX = RS_NMAX / 2;  // groups have >= 2 records
struct SmallPlan {
    int c0;          // cursor % T before the batch
    long long P[64]; // per-shard push counts before the batch
};
// group_adv_one over shared-memory rewards (the same fp64 operation order)
__device__ __forceinline__ void group_adv_smem(const double* rw, int b, int e, double rj,
                                               double* adv, double* mean_out) {
    const double dn = (double)(e - b);
    double mean = 0.0, var = 0.0;
    for (int k = b; k < e; ++k) mean = __dadd_rn(mean, rw[k]);
    mean = __ddiv_rn(mean, dn);
    for (int k = b; k < e; ++k) {
        const double d = __dsub_rn(rw[k], mean);
        var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, dn);
    const double sd = __dsqrt_rn(var);
    *adv = sd < 1e-8 ? 0.0 : __ddiv_rn(__dsub_rn(rj, mean), sd);
    *mean_out = mean;
}

__global__ void __launch_bounds__(RS_THREADS) k_route_small(BufView v, InsertIn in, SmallPlan sp,
                                                             int* pay_sync) {
    __shared__ double s_rw[RS_NMAX];
    __shared__ uint64_t s_id[RS_NMAX];
    __shared__ long long s_goff[RS_GMAX + 1];
    __shared__ int s_m[RS_THREADS / 32];
    const int tid = threadIdx.x;
    const int n = (int)in.n, ng = (int)in.ngroups;
    const int T = v.T, C = v.C;
    DevCtl* ctl = v.ctl;
    RB_TSTART(0);
    if (tid == 0) {  // this insert's verdict / completion flags
        st_release_i32(&pay_sync[0], 0);
        st_release_i32(&pay_sync[1], 0);
        if (in.pay_follows) st_release_i32(&pay_sync[2], 1);  // the copy's completion flag
        fence_gpu();
    }
    __syncthreads();
    pdl_trigger();
    // ---- the one round trip: control block, batch, evictees
    const int sticky = ctl->err_code;
    const int has_any = ctl->has_any;
    const unsigned long long max_id = ctl->max_id;
    uint64_t id[RS_PER], prompt[RS_PER], group[RS_PER], evres[RS_PER];
    int64_t cstep[RS_PER], pver[RS_PER], off0[RS_PER], off1[RS_PER];
    double reward[RS_PER], blp[RS_PER], adv[RS_PER], gmean[RS_PER];
    bool correct[RS_PER];
    int slot[RS_PER], rank_[RS_PER], j0_[RS_PER], ns_[RS_PER];
    long long Pj[RS_PER];
#pragma unroll
    for (int r = 0; r < RS_PER; ++r) {
        const int j = tid + r * RS_THREADS;
        evres[r] = NONE_ID;
        if (j >= n) continue;
        id[r] = in.id[j];
        prompt[r] = in.prompt ? in.prompt[j] : 0;
        group[r] = in.group ? in.group[j] : 0;
        cstep[r] = in.cstep ? in.cstep[j] : 0;
        pver[r] = in.pver ? in.pver[j] : 0;
        reward[r] = in.reward[j];
        correct[r] = in.correct ? in.correct[j] != 0 : false;
        blp[r] = in.blp ? in.blp[j] : 0.0;
        adv[r] = in.adv ? in.adv[j] : 0.0;
        gmean[r] = in.adv && in.gmean ? in.gmean[j] : 0.0;
        off0[r] = in.toff ? in.toff[j] : 0;
        off1[r] = in.toff ? in.toff[j + 1] : 0;
        int s = sp.c0 + j % T;
        if (s >= T) s -= T;
        const int rank = j / T, j0 = j % T;
        const long long P = sp.P[s];
        int x2 = (int)(P % C) + rank % C;
        if (x2 >= C) x2 -= C;
        slot[r] = s * C + x2;
        rank_[r] = rank;
        j0_[r] = j0;
        ns_[r] = (n - 1 - j0) / T + 1;
        Pj[r] = P;
        // the slot's resident record before the batch (its first push evicts it)
        if (P + (rank % C) >= C) evres[r] = v.id[slot[r]];
    }
    if (!in.adv)
        for (int gi = tid; gi <= ng; gi += RS_THREADS) s_goff[gi] = in.goff[gi];
#pragma unroll
    for (int r = 0; r < RS_PER; ++r) {
        const int j = tid + r * RS_THREADS;
        if (j < n) {
            s_id[j] = id[r];
            s_rw[j] = reward[r];
            if (in.toff_keep) {
                in.toff_keep[j] = off0[r];
                if (j == n - 1) in.toff_keep[n] = off1[r];
            }
        }
    }
    __syncthreads();
    // ---- whole-batch validation (replay_buffer.cpp:85-88 order: nothing applied)
    int bad = 0;
#pragma unroll
    for (int r = 0; r < RS_PER; ++r) {
        const int j = tid + r * RS_THREADS;
        if (j >= n) continue;
        const long long l = off1[r] - off0[r];
        if (in.toff && (l < 0 || l > in.maxlen)) bad |= 2;
        if (j > 0 ? id[r] <= s_id[j - 1] : (has_any && id[r] <= max_id)) bad |= 1;
    }
    if (!in.adv) {
        if (tid == 0 && (s_goff[0] != 0 || s_goff[ng] != n)) bad |= 4;
        for (int gi = tid; gi < ng; gi += RS_THREADS) {
            const long long b = s_goff[gi], e = s_goff[gi + 1];
            if (e - b < 2 || b < 0 || e > n) bad |= 4;
        }
    }
    const int bb = (sticky ? 8 : 0) | (__syncthreads_or(bad & 1) ? 1 : 0) |
                   (__syncthreads_or(bad & 2) ? 2 : 0) | (__syncthreads_or(bad & 4) ? 4 : 0);
    if (tid == 0) st_release_i32(&pay_sync[0], bb ? 2 : 1);
    RB_GCLOCK(60, true);
    // ---- apply: slots, evictions, advantages, metadata, payload descriptors
    int maxq = 0;
#pragma unroll
    for (int r = 0; r < RS_PER; ++r) {
        const int j = tid + r * RS_THREADS;
        if (j >= n) continue;
        const long long len = off1[r] - off0[r];
        int32_t sl = -1;
        uint8_t surv = 0;
        uint64_t ev = NONE_ID;
        bool ev_by_survivor = false;
        Unit d;
        d.row = -1;
        d.len = (int32_t)(len < 0 ? 0 : len);
        d.k0 = 0;
        d.g = j;
        d.off = off0[r];
        d.adv = 0.0;
        double a = adv[r], gm = gmean[r];
        if (!bb) {
            const int rank = rank_[r], j0 = j0_[r], ns = ns_[r];
            const int g = slot[r], s = g / C;
            sl = g;
            surv = rank + C >= ns;
            if (Pj[r] + rank >= C) ev = rank >= C ? s_id[j - C * T] : evres[r];
            if (rank < C && !surv) ev_by_survivor = true;
            if (surv && rank >= C) {
                const int r0 = rank % C;
                in.evid[r0 * T + j0] = Pj[r] + r0 >= C ? evres[r] : NONE_ID;
            }
            if (!in.adv) {
                int lo = 0, hi = ng;  // group gi: goff[gi] <= j < goff[gi+1]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_goff[mid] <= j) lo = mid;
                    else hi = mid;
                }
                group_adv_smem(s_rw, (int)s_goff[lo], (int)s_goff[lo + 1], reward[r], &a, &gm);
            }
            if (surv) {
                v.id[g] = id[r];
                v.prompt[g] = prompt[r];
                v.group[g] = group[r];
                v.cstep[g] = cstep[r];
                v.pver[g] = pver[r];
                v.reward[g] = reward[r];
                v.correct[g] = in.correct ? correct[r] : reward[r] == 1.0;
                v.blp[g] = blp[r];
                v.adv[g] = a;
                v.gmean[g] = gm;
                v.use[g] = 0;
                v.len[g] = (int32_t)len;
                if (s >= v.sb && s < v.se && len > 0 && v.stride > 0) {
                    d.row = (s - v.sb) * C + (g - s * C);
                    maxq = max(maxq, (int)((len + 3) >> 2));
                }
            }
        }
        in.len[j] = (int32_t)(len < 0 ? 0 : len);
        in.tslot[j] = sl;
        in.surv[j] = surv;
        if (!ev_by_survivor) in.evid[j] = ev;
        in.adv_out[j] = a;
        in.gmean_out[j] = gm;
        in.units[j] = d;
    }
    maxq = __reduce_max_sync(0xffffffffu, maxq);
    if ((tid & 31) == 0) s_m[tid >> 5] = maxq;
    __syncthreads();
    RB_GCLOCK(62, true);
    if (tid == 0) {
        // every record of the batch is written: the sampler may read them
        st_release_i32(&pay_sync[1], 1);
        if (in.toff_keep)  // the offsets copy for an overlapping sampler
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(in.keep_cnt) : "memory");
        int m = 0;
        for (int w = 0; w < RS_THREADS / 32; ++w) m = max(m, s_m[w]);
        *in.n_units = bb ? 0 : m;
        if (!bb) {
            ctl->cursor = ((unsigned long long)sp.c0 + (unsigned long long)n) % T;
            ctl->max_id = id[0];  // overwritten below by the batch's last id
            ctl->has_any = 1;
            ctl->hash_stale = 1;
        } else if (!sticky) {
            ctl->err_code = RB_EINVAL;
            ctl->err_index = (bb & 2) ? -3 : (bb & 4) ? -2 : -4;
        }
    }
    if (!bb) {
        if (tid == ((n - 1) & (RS_THREADS - 1))) ctl->max_id = s_id[n - 1];
        for (int s = tid; s < T; s += RS_THREADS) {
            const int j0 = ((s - sp.c0) % T + T) % T;
            const int ns = n > j0 ? (n - 1 - j0) / T + 1 : 0;
            v.pushes[s] += ns;
        }
    }
    RB_GCLOCK(57, true);
    RB_TEND(0);
}

