// ---- one launch per small replay step: insert + sample (rb_insert_sample) --
// The record-level step of the reference's loops — push a batch of whole
// groups, then sample B (bandit.cpp:596-615, async_sim.cpp:138-139) — for
// FIFO retention, ids promised new, uniform draws with replacement, at most
// SS_NMAX records and SS_BMAX draws over <= 64 shards, in ONE CTA and one
// launch.  The multi-kernel path (route -> sampler, flags and done counters
// across CTAs and kernels) costs ~13 µs per record-level step in a CUDA graph
// whatever the size (tools/c5_probe.py: 9 µs for either kernel alone); here
// the whole step is three dependent memory round trips:
//   1. the batch, the control block, the evictees' ids, the ring header;
//   2. the MT19937-64 words of this call's draws (blocks twisted ahead by the
//      previous call; missing ones twisted into the ring first);
//   3. the sampled slots' lengths and advantages (+ use-count atomics).
// Routing, eviction and advantages follow k_route_fifo (replay_buffer.cpp:
// 83-96 in closed form from the host's exact per-shard push counts,
// bandit.cpp:276-294 fp64 in the reference's order); the draws follow
// k_sample_fused (shard s takes draws [s*per, (s+1)*per), below() rejection
// -> exact sequential replay of the whole call by one thread,
// replay_buffer.cpp:141-145 / rng.cpp:40-51).  A rejected batch (or a
// sticky error) freezes the sampler as on the multi-kernel path: empty
// batch, ring unchanged.  The payload copy (if any) is launched next as a
// programmatic dependent and waits for this kernel's verdict flag.
constexpr int SS_THREADS = 1024;
constexpr int SS_RPT = 2;                       // records per thread
constexpr int SS_DPT = 4;                       // draws per thread
constexpr int SS_NMAX = SS_THREADS * SS_RPT;    // 2048 records
constexpr int SS_BMAX = SS_THREADS * SS_DPT;    // 4096 draws
constexpr int SS_GMAX = SS_NMAX / 2;            // groups of >= 2 records

struct StepPlan {
    int c0;          // cursor % T before the batch
    int gen_ahead;   // twist the next call's blocks too
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

__global__ void __launch_bounds__(SS_THREADS) k_step_small(BufView v, InsertIn in, StepPlan sp,
                                                            MtRing* r, SampleArgs a, int* pay_sync) {
    __shared__ double s_rw[SS_NMAX];
    __shared__ uint64_t s_id[SS_NMAX];
    __shared__ long long s_goff[SS_GMAX + 1];
    __shared__ uint64_t s_mt[MT_N];
    __shared__ long long s_occ[64], s_q;
    __shared__ uint64_t s_lim[64], s_mag[64];
    __shared__ int s_head[64], s_m[SS_THREADS / 32], s_rej;
    __shared__ uint32_t s_idx;
    const int tid = threadIdx.x;
    const int n = (int)in.n, ng = (int)in.ngroups;
    const int T = v.T, C = v.C;
    DevCtl* ctl = v.ctl;
    RB_TSTART(0);
    if (tid == 0) {  // this insert's verdict / completion flags (payload copy protocol)
        st_release_i32(&pay_sync[0], 0);
        st_release_i32(&pay_sync[1], 0);
        if (in.pay_follows) st_release_i32(&pay_sync[2], 1);
        fence_gpu();
    }
    __syncthreads();
    pdl_trigger();  // the closed-form payload copy may start (it waits for the verdict)
    // ---- round trip 1: control block, ring header, batch, evictees
    const int sticky = ctl->err_code;
    const int has_any = ctl->has_any;
    const unsigned long long max_id = ctl->max_id;
    const long long q0 = r->q_state, qhi0 = r->q_hi;
    const uint32_t idx0 = r->idx;
    const unsigned long long draws0 = r->draws;
    uint64_t id[SS_RPT], evres[SS_RPT];
    int64_t off0[SS_RPT], off1[SS_RPT];
    double reward[SS_RPT];
#pragma unroll
    for (int k = 0; k < SS_RPT; ++k) {
        const int j = tid + k * SS_THREADS;
        evres[k] = NONE_ID;
        if (j >= n) continue;
        id[k] = in.id[j];
        reward[k] = in.reward[j];
        off0[k] = in.toff ? in.toff[j] : 0;
        off1[k] = in.toff ? in.toff[j + 1] : 0;
        int s = sp.c0 + j % T;
        if (s >= T) s -= T;
        const int rank = j / T;
        const long long P = sp.P[s];
        // the slot's pre-batch resident, evicted by the slot's first push
        if (rank < C && P + rank >= C) {
            int x = (int)(P % C) + rank;
            if (x >= C) x -= C;
            evres[k] = v.id[(size_t)s * C + x];
        }
    }
    if (!in.adv)
        for (int gi = tid; gi <= ng; gi += SS_THREADS) s_goff[gi] = in.goff[gi];
#pragma unroll
    for (int k = 0; k < SS_RPT; ++k) {
        const int j = tid + k * SS_THREADS;
        if (j < n) {
            s_id[j] = id[k];
            s_rw[j] = reward[k];
        }
    }
    __syncthreads();
    // ---- whole-batch validation (replay_buffer.cpp:85-88: nothing applied on failure)
    int bad = 0;
#pragma unroll
    for (int k = 0; k < SS_RPT; ++k) {
        const int j = tid + k * SS_THREADS;
        if (j >= n) continue;
        const long long l = off1[k] - off0[k];
        if (in.toff && (l < 0 || l > in.maxlen)) bad |= 2;
        if (j > 0 ? id[k] <= s_id[j - 1] : (has_any && id[k] <= max_id)) bad |= 1;
    }
    if (!in.adv) {
        if (tid == 0 && (s_goff[0] != 0 || s_goff[ng] != n)) bad |= 4;
        for (int gi = tid; gi < ng; gi += SS_THREADS) {
            const long long b = s_goff[gi], e = s_goff[gi + 1];
            if (e - b < 2 || b < 0 || e > n) bad |= 4;
        }
    }
    const int bb = (sticky ? 8 : 0) | (__syncthreads_or(bad & 1) ? 1 : 0) |
                   (__syncthreads_or(bad & 2) ? 2 : 0) | (__syncthreads_or(bad & 4) ? 4 : 0);
    if (tid == 0) st_release_i32(&pay_sync[0], bb ? 2 : 1);
    // ---- apply the batch (k_route_fifo's outputs)
    if (!bb) {
#pragma unroll
        for (int k = 0; k < SS_RPT; ++k) {
            const int j = tid + k * SS_THREADS;
            if (j >= n) continue;
            int s = sp.c0 + j % T;
            if (s >= T) s -= T;
            const int rank = j / T, j0 = j % T;
            const int ns = (n - 1 - j0) / T + 1;
            const long long P = sp.P[s];
            int x = (int)(P % C) + rank % C;
            if (x >= C) x -= C;
            const size_t g = (size_t)s * C + x;
            const bool surv = rank + C >= ns;
            uint64_t ev = NONE_ID;
            if (P + rank >= C) ev = rank >= C ? s_id[j - C * T] : evres[k];
            const long long len = off1[k] - off0[k];
            double adv, gm;
            if (in.adv) {
                adv = in.adv[j];
                gm = in.gmean ? in.gmean[j] : 0.0;
            } else {
                int lo = 0, hi = ng;  // group gi: goff[gi] <= j < goff[gi+1]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_goff[mid] <= j) lo = mid;
                    else hi = mid;
                }
                group_adv_smem(s_rw, (int)s_goff[lo], (int)s_goff[lo + 1], reward[k], &adv, &gm);
            }
            if (surv) {
                v.id[g] = id[k];
                v.prompt[g] = in.prompt ? in.prompt[j] : 0;
                v.group[g] = in.group ? in.group[j] : 0;
                v.cstep[g] = in.cstep ? in.cstep[j] : 0;
                v.pver[g] = in.pver ? in.pver[j] : 0;
                v.reward[g] = reward[k];
                v.correct[g] = in.correct ? in.correct[j] != 0 : reward[k] == 1.0;
                v.blp[g] = in.blp ? in.blp[j] : 0.0;
                v.adv[g] = adv;
                v.gmean[g] = gm;
                v.use[g] = 0;
                v.len[g] = (int32_t)len;
            }
            in.len[j] = (int32_t)len;
            in.tslot[j] = (int32_t)g;
            in.surv[j] = surv;
            in.evid[j] = ev;
            in.adv_out[j] = adv;
            in.gmean_out[j] = gm;
        }
    }
    // ---- the sampler: shard occupancies / heads after the batch (closed form)
    const bool frozen = bb != 0;
    if (tid < T) {
        const int s = tid;
        const int j0 = ((s - sp.c0) % T + T) % T;
        const int ns = (!bb && n > j0) ? (n - 1 - j0) / T + 1 : 0;
        const long long P = sp.P[s] + ns;
        const long long occ = P < C ? P : C;
        s_occ[s] = occ;
        s_head[s] = P >= C ? (int)(P % C) : 0;
        s_lim[s] = occ ? below_limit((uint64_t)occ) : 0;
        s_mag[s] = occ ? UINT64_MAX / (uint64_t)occ : 0;
        if (!bb) v.pushes[s] = P;
    }
    const long long D = frozen ? 0 : a.nsel;
    const long long need = q0 + (long long)((idx0 + (unsigned long long)D + MT_N - 1) / MT_N);
    __syncthreads();  // the batch's metadata is written (visible to this CTA below)
    if (!frozen && need > qhi0) ring_extend(r, s_mt, qhi0, need);  // first call / large batch
    // ---- round trip 2: the draws
    const int per = (int)a.per;
    long long kd[SS_DPT];
    int sh[SS_DPT], ix[SS_DPT];
    bool rej = false;
#pragma unroll
    for (int d = 0; d < SS_DPT; ++d) {
        const long long k = (long long)tid * SS_DPT + d;
        kd[d] = k;
        sh[d] = 0;
        ix[d] = 0;
        if (k >= D) continue;
        const unsigned long long o = idx0 + (unsigned long long)k;
        const uint64_t y = mt_temper(__ldcg(&r->blk[(q0 + (long long)(o / MT_N)) % MT_KR][o % MT_N]));
        const int s = (int)(k / per);
        rej |= y >= s_lim[s];
        sh[d] = s;
        ix[d] = (int)fast_mod(y, (uint64_t)s_occ[s], s_mag[s]);
    }
    const bool any_rej = __syncthreads_or(rej || v.dbg_replay);
    long long qn = q0;
    uint32_t idxn = idx0;
    unsigned long long drn = draws0;
    if (any_rej) {  // an exact sequential replay of the whole call (probability ~D*n/2^64)
        if (tid == 0) s_rej = 0;
        for (int i = tid; i < MT_N; i += SS_THREADS) s_mt[i] = __ldcg(&r->blk[q0 % MT_KR][i]);
        __syncthreads();
        if (tid == 0) {
            uint32_t idx = idx0;
            long long tw = 0;
            unsigned long long dr = 0;
            draw_exact(a.sel_shard, a.sel_index, a.per, s_occ, s_mt, 0, D, &idx, &tw, &dr);
            s_q = q0 + tw;
            s_idx = idx;
            s_rej = (int)(dr - (unsigned long long)D);
            r->draws = draws0 + dr;
        }
        __syncthreads();
        qn = s_q;
        idxn = s_idx;
#pragma unroll
        for (int d = 0; d < SS_DPT; ++d)
            if (kd[d] < D) {
                sh[d] = a.sel_shard[kd[d]];
                ix[d] = (int)a.sel_index[kd[d]];
            }
    } else if (!frozen) {
        ring_advance(qn, idxn, (unsigned long long)D);
        drn = draws0 + (unsigned long long)D;
    }
    // ---- round trip 3: sampled slots (use counts, lengths, advantages)
    int g[SS_DPT], L[SS_DPT];
    double av[SS_DPT];
#pragma unroll
    for (int d = 0; d < SS_DPT; ++d) {
        g[d] = 0;
        L[d] = 0;
        av[d] = 0.0;
        if (kd[d] >= D) continue;
        const int s = sh[d];
        int x = s_head[s] + ix[d];
        if (x >= C) x -= C;
        g[d] = s * C + x;
        L[d] = v.len[g[d]];
        av[d] = v.adv[g[d]];
        atomicAdd(&v.use[g[d]], 1u);  // replay_buffer.cpp:201
    }
    // packed offsets of the owned selections, totals
    long long own = 0, all = 0;
#pragma unroll
    for (int d = 0; d < SS_DPT; ++d) {
        if (kd[d] >= D) continue;
        all += L[d];
        if (kd[d] >= a.lo && kd[d] < a.hi) own += L[d];
    }
    long long own_tot, all_tot;
    long long pos = block_exclusive_scan(own, &own_tot);
    block_exclusive_scan(all, &all_tot);
    int maxq = 0;
#pragma unroll
    for (int d = 0; d < SS_DPT; ++d) {
        const long long k = kd[d];
        if (k >= a.nsel) continue;
        const bool live = k < D;
        if (!any_rej && live) {
            a.sel_shard[k] = sh[d];
            a.sel_index[k] = ix[d];
        }
        if (live) {
            a.sel_slot[k] = g[d];
            a.sel_len[k] = L[d];
        }
        if (k < a.lo || k >= a.hi) continue;
        Unit u{};
        if (live) {
            u.row = (sh[d] - v.sb) * C + (g[d] - sh[d] * C);
            u.len = L[d];
            u.g = g[d];
            u.off = pos;
            u.adv = av[d];
            const int nq = ((int)(pos & 3) + L[d] + 3) >> 2;
            if (L[d]) maxq = nq > maxq ? nq : maxq;
        }
        a.units[k - a.lo] = u;
        a.off[k - a.lo] = live ? pos : 0;
        if (live) pos += L[d];
    }
    maxq = __reduce_max_sync(0xffffffffu, maxq);
    if ((tid & 31) == 0) s_m[tid >> 5] = maxq;
    __syncthreads();
    if (tid == 0) {
        int m = 0;
        for (int w = 0; w < SS_THREADS / 32; ++w) m = max(m, s_m[w]);
        const long long nloc = a.hi - a.lo;
        a.off[nloc] = own_tot;
        a.totals[0] = own_tot;
        a.totals[1] = all_tot;
        *a.n_units = m;
        DevLossAcc* acc = a.acc;
        acc->obj_sum = 0.0;
        acc->included = 0;
        acc->excluded = 0;
        acc->done_blocks = 0;
        acc->total_tokens = all_tot;
        acc->objective = 0.0;
        acc->need_fixup = 0;
        // the insert's bookkeeping (k_route_fifo's last CTA)
        *in.n_units = 0;  // no separate descriptor table: the copy uses the closed form
        if (!bb) {
            ctl->cursor = ((unsigned long long)sp.c0 + (unsigned long long)n) % T;
            ctl->max_id = s_id[n - 1];  // strictly increasing and above the old max
            ctl->has_any = 1;
            ctl->hash_stale = 1;
        } else if (!sticky) {
            ctl->err_code = RB_EINVAL;
            ctl->err_index = (bb & 2) ? -3 : (bb & 4) ? -2 : -4;
        }
        st_release_i32(&pay_sync[1], 1);
        // the ring position after this call (unchanged when frozen)
        if (!frozen) {
            r->q_state = qn;
            r->idx = idxn;
            if (!any_rej) r->draws = drn;
        }
    }
    // the next call's blocks (what k_sample_fused's generator CTA does)
    if (!frozen) {
        long long hi = need > qhi0 ? need : qhi0;
        if (any_rej && qn > hi) {  // the replay went past the ring: store its block
            __syncthreads();
            for (int i = tid; i < MT_N; i += SS_THREADS) r->blk[qn % MT_KR][i] = s_mt[i];
            hi = qn;
        }
        long long target = sp.gen_ahead ? need + (need - q0) + 1 : need;
        if (target > qn + MT_KR - 1) target = qn + MT_KR - 1;
        if (target > hi) ring_extend(r, s_mt, hi, target);
        if (tid == 0) r->q_hi = target > hi ? target : hi;
    }
    RB_TEND(0);
}

