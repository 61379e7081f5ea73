// ---- GRPO over the current batch with TMA-staged operands -----------------
// The same per-token arithmetic as k_loss_grpo_buf (fast fp32 path with one
// threshold per item, exact fp64 replay near a clip edge / |d| >= 16 /
// non-finite / boundary quads), but the 8 B of operands per token reach the
// SM by bulk copies (cp.async.bulk global -> shared, mbarrier-tracked) issued
// LT_S items ahead by one thread, so every CTA keeps LT_S x 16 KB in flight
// independently of its registers and computes one item while the next ones
// load (the register-staged kernel waits one full memory latency per unit).
// Item = up to LT_CH tokens of one selection: logp_now from the packed batch
// (16-B aligned-down source, the shift absorbed by indexing the staged
// quads), logp_old from the selection's slot row (16-B aligned).  dlogp is
// stored from registers with 128-bit streaming stores (masked at the
// selection's boundary quads, which neighbouring selections share).  Items
// of a CTA: a static stride over (selection, chunk), the descriptors of up
// to LT_THREADS candidates loaded in parallel and compacted (empty chunks
// of short rows skipped).  Objective: fp64 per item, folded as the other
// loss kernels (fixed order, bitwise-reproducible).
constexpr int LT_CH = 2048;                 // tokens per item
constexpr int LT_S = 4;                     // stages per CTA
#ifndef RB_LT_THREADS
#define RB_LT_THREADS 256
#endif
constexpr int LT_THREADS = RB_LT_THREADS;
constexpr int LT_NOW = LT_CH + 8;           // staged logp_now floats (aligned-down start + spill)
constexpr int LT_OLD = LT_CH + 4;
struct LtItem {
    long long P;  // packed offset of the item's first token
    int row;      // slot row (local)
    int cnt;      // tokens
    int c;        // chunk within the selection
    int pad;
    double A;     // the selection's advantage
};
constexpr size_t LT_SMEM = (size_t)LT_S * (LT_NOW + LT_OLD) * 4 + 2 * LT_S * 8 +
                           (LT_S + LT_THREADS) * sizeof(LtItem) + 64;

__global__ void __launch_bounds__(LT_THREADS + 32) k_loss_grpo_tma(
    BufView v, const Unit* units, const int* maxq_p, int nloc, const float* lpn_packed,
    float* dlogp, GrpoParams prm, DevLossAcc* acc, Partial* parts, rb_loss_stats* stats,
    const long long* n_local, int local_fix) {
    extern __shared__ __align__(128) unsigned char lt_sm[];
    float* nowb = reinterpret_cast<float*>(lt_sm);
    float* oldb = nowb + LT_S * LT_NOW;
    uint64_t* bar = reinterpret_cast<uint64_t*>(oldb + LT_S * LT_OLD);  // [S] full, [S] empty
    uint64_t* ebar = bar + LT_S;
    LtItem* held = reinterpret_cast<LtItem*>(ebar + LT_S);  // the item in each stage
    LtItem* list = held + LT_S;                            // compacted candidates
    __shared__ int s_wcnt[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const float scale = -1.f / (float)acc->total_tokens;
    const float tol_hi = 4e-6f * prm.hi_f, tol_lo = 4e-6f * prm.lo_f;
    RB_TSTART(5);
    // warps 0..LT_THREADS/32-1 compute; the last warp issues the bulk copies
    const bool producer = tid >= LT_THREADS;
    if (tid == 0) {
        for (int s = 0; s < LT_S; ++s) {
            mbar_init(&bar[s]);
            mbar_init_n(&ebar[s], LT_THREADS / 32);  // one arrival per compute warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int maxt = 4 * *maxq_p;  // tokens of the longest selection (bound)
    const int ups = (maxt + LT_CH - 1) / LT_CH;
    const long long nitems = (long long)nloc * ups;
    const long long G = gridDim.x;
    GrpoPartial part;
    long long inc_fast = 0;
    long long g = 0;  // items of this CTA so far (stage g % LT_S, phase (g / LT_S) & 1)
    __syncthreads();
    auto issue = [&](const LtItem& it, long long gi) {  // the producer's lane 0
        const int st = (int)(gi % LT_S);
        held[st] = it;
        const long long Pa = it.P & ~3LL;
        const int a = (int)(it.P - Pa);
        const uint32_t bn = (uint32_t)(((a + it.cnt + 3) & ~3) * 4);
        const uint32_t bo = (uint32_t)(((it.cnt + 3) & ~3) * 4);
        mbar_expect_tx(&bar[st], bn + bo);
        bulk_g2s(nowb + (size_t)st * LT_NOW, lpn_packed + Pa, bn, &bar[st]);
        bulk_g2s(oldb + (size_t)st * LT_OLD,
                 v.lpo + (size_t)it.row * v.stride + (size_t)it.c * LT_CH, bo, &bar[st]);
    };
    for (long long base = blockIdx.x; base < nitems; base += (long long)LT_THREADS * G) {
        // this window's candidates: descriptors in parallel, non-empty ones compacted
        const long long u = base + (long long)tid * G;
        LtItem it{};
        bool ok = false;
        if (!producer && u < nitems) {
            const int b = (int)(u / ups), c = (int)(u - (long long)b * ups);
            const Unit un = ld_unit(units + b);
            const int cnt = min(un.len - c * LT_CH, LT_CH);
            if (un.row >= 0 && cnt > 0) {
                it.P = un.off + (long long)c * LT_CH;
                it.row = un.row;
                it.cnt = cnt;
                it.c = c;
                it.A = un.adv;
                ok = true;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (lane == 0 && !producer) s_wcnt[wid] = __popc(m);
        __syncthreads();
        int wbase = 0, total = 0;
        for (int w = 0; w < LT_THREADS / 32; ++w) {
            if (w < wid) wbase += s_wcnt[w];
            total += s_wcnt[w];
        }
        if (ok) list[wbase + __popc(m & ((1u << lane) - 1))] = it;
        __syncthreads();
        // pipeline over the window: LT_S items in flight; a stage is refilled
        // once every compute warp has released it (no CTA barrier per item)
        if (producer) {
            if (lane == 0)
                for (int i = 0; i < total; ++i) {
                    const long long gi = g + i;
                    if (gi >= LT_S) mbar_wait(&ebar[gi % LT_S], (uint32_t)(((gi / LT_S) - 1) & 1));
                    issue(list[i], gi);
                }
            g += total;
            __syncthreads();  // the list is rewritten by the next window
            continue;
        }
        for (int i = 0; i < total; ++i, ++g) {
            const int st = (int)(g % LT_S);
            mbar_wait(&bar[st], (uint32_t)((g / LT_S) & 1));
            const LtItem x = held[st];
            const int a = (int)(x.P & 3);
            const long long K0 = x.P >> 2;  // first destination quad
            const int nq = (int)(((x.P + x.cnt - 1) >> 2) - K0 + 1);
            const double A = x.A;
            const float Afs = (float)A * scale;
            const int sgn = A > 0.0 ? 1 : (A < 0.0 ? -1 : 0);
            const float thr = sgn > 0 ? prm.hi_f : prm.lo_f;
            const float tol = sgn > 0 ? tol_hi : tol_lo;
            const float* nw = nowb + (size_t)st * LT_NOW;
            const float* od = oldb + (size_t)st * LT_OLD;
            double fsum = 0.0;
            for (int q = tid; q < nq; q += LT_THREADS) {
                const float4 n4 = *reinterpret_cast<const float4*>(nw + 4 * q);
                const float nv[4] = {n4.x, n4.y, n4.z, n4.w};
                const int e0 = 4 * q - a;  // local index of the quad's first element
                float ov[4];
                if (a == 0) {  // the staged row quads line up with the destination's
                    const float4 o4 = *reinterpret_cast<const float4*>(od + 4 * q);
                    ov[0] = o4.x;
                    ov[1] = o4.y;
                    ov[2] = o4.z;
                    ov[3] = o4.w;
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int e = e0 + i;
                        ov[i] = (e >= 0 && e < x.cnt) ? od[e] : 0.f;
                    }
                }
                const bool full = e0 >= 0 && e0 + 3 < x.cnt;
                float o[4] = {0.f, 0.f, 0.f, 0.f};
                bool slow = !full;
                if (full) {
                    float r[4];
                    bool edge = false;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float d = nv[i] - ov[i];
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
                if (slow) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (e0 + i >= 0 && e0 + i < x.cnt)
                            o[i] = grpo_token_exact(nv[i], ov[i], A, prm, part) * scale;
                }
                store_quad_masked(reinterpret_cast<uint32_t*>(dlogp), K0 + q,
                                  make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]),
                                             __float_as_uint(o[2]), __float_as_uint(o[3])),
                                  e0, x.cnt);
            }
            part.obj += fsum * A;
            __syncwarp();
            if (lane == 0) mbar_arrive(&ebar[st]);  // this warp is done with stage st
        }
        __syncthreads();  // the list is rewritten by the next window
    }
    part.inc += inc_fast;
    RB_TEND(5);
    loss_commit(part, parts, acc, stats, 0, 0.0, dlogp, n_local, local_fix, 0, (int)gridDim.x);
}


