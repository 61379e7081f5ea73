// packed_range.cuh — balanced persistent iteration over a packed batch.
//
// The gather and the token losses walk the PACKED token space of the
// batch, not its selections: [T0, T1) with T0 = off[0], T1 = off[nsel],
// off = the exclusive scan of the selected trajectories' lengths.  Its
// 16-byte quads are tiled into warp units of PK_WQ quads; CTA c owns a
// contiguous run of equal numbers of warp units, so ragged lengths cost
// nothing in balance and no unit is empty (the per-selection unit tables
// they replace spent ~half their units on nothing at U{1..8192}).
//
// Per CTA, the selections holding the run stage their offsets, slot rows,
// metadata slots and advantages in shared memory (pk_setup).  A warp unit
// that lies inside one selection (the common case) is then a funnel-shifted
// 128-bit row copy with neighbour quads by shuffle; in a unit that straddles
// selections each lane handles its quads alone: a quad inside one selection
// is still two 128-bit row loads and a funnel shift, only the quad holding a
// boundary goes token by token (each lane writes whole quads, so no quad is
// written by two threads).  Runs covering more than PK_SL selections (tiny
// trajectories) search off[] in global memory per token: correct, slower.
#pragma once

#include "stream_copy.cuh"

namespace rb {

constexpr int PK_U = 4;             // quads per lane per warp unit
constexpr int PK_WQ = 32 * PK_U;    // quads per warp unit (512 tokens)
constexpr int PK_SL = 256;          // selections staged per CTA
constexpr int PK_THREADS = 128;     // 4 warps

struct PkSlice {
    long long off[PK_SL + 1];
    int32_t row[PK_SL];
    int32_t g[PK_SL];
    double adv[PK_SL];
    long long q_lo, q_hi;  // this CTA's quads [q_lo, q_hi)
    long long T0, T1;      // the batch's token range
    int b0, n;             // staged selections [b0, b0 + n); n < 0: not staged
    int cur0;              // staged index of the run's first selection
};

// Largest b in [0, nsel) with off[b] <= t (off non-decreasing, off[0] <= t):
// the selection holding token t (zero-length selections are skipped).
__device__ __forceinline__ int pk_warp_search(const int64_t* off, int nsel, long long t) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = nsel;
    while (hi - lo > 1) {
        const int step = (hi - lo + 31) >> 5;
        const int idx = lo + lane * step;
        const bool p = idx < hi && off[idx] <= t;
        const unsigned m = __ballot_sync(0xffffffffu, p);
        lo += (31 - __clz(m)) * step;  // lane 0 holds by the invariant off[lo] <= t
        hi = min(hi, lo + step);
    }
    return lo;
}
// Per-thread binary search (the unstaged fallback).
__device__ __forceinline__ int pk_thread_search(const int64_t* off, int nsel, long long t) {
    int lo = 0, hi = nsel;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Block-wide: this CTA's quad run and its staged selections.  Returns false
// (block-uniform) when the CTA has no work.  Two dependent loads in the
// common case: the range ends off[0], off[nsel]; then a window of
// blockDim.x offsets and descriptors around the interpolated position of the
// run's first token (exact for equal lengths; ragged prefixes stay close),
// which holds the run's first and last selections unless lengths are very
// uneven — then 32-ary searches and a slice load (3 + 1 more).
__device__ __forceinline__ bool pk_setup(PkSlice& s, const int64_t* off, const Unit* desc,
                                         int nsel) {
    const int tid = threadIdx.x, wid = tid >> 5, nt = blockDim.x;
    __shared__ long long s_T[2];
    __shared__ int s_bb[2];
    if (tid < 2) s_T[tid] = nsel > 0 ? off[tid ? nsel : 0] : 0;
    __syncthreads();
    const long long T0 = s_T[0], T1 = s_T[1];
    const long long Q0 = T0 >> 2, Q1 = (T1 + 3) >> 2;
    const long long nwu = T1 > T0 ? (Q1 - Q0 + PK_WQ - 1) / PK_WQ : 0;
    const long long per = (nwu + gridDim.x - 1) / gridDim.x;
    const long long w0 = (long long)blockIdx.x * per, w1 = min(nwu, w0 + per);
    if (w1 <= w0) return false;
    const long long q_lo = Q0 + w0 * PK_WQ, q_hi = min(Q1, Q0 + w1 * PK_WQ);
    const long long ta = max(T0, 4 * q_lo), tb = min(T1, 4 * q_hi) - 1;
    // window [b_w, b_w + nt - 1) of selections, offsets [b_w, b_w + nt - 1]
    const long long guess = (long long)((double)(ta - T0) / (double)(T1 - T0) * (double)nsel);
    const int W = min(nt - 1, nsel);
    const int b_w = (int)max(0LL, min((long long)(nsel - W), guess - 8));
    if (tid == 0) s_bb[0] = s_bb[1] = -1;
    if (tid <= W) s.off[tid] = off[b_w + tid];
    if (tid < W) {
        const Unit d = ld_unit(desc + b_w + tid);
        s.row[tid] = d.row;
        s.g[tid] = d.g;
        s.adv[tid] = d.adv;
    }
    __syncthreads();
    if (tid < W) {  // the unique window entry holding ta / tb, if any
        const long long o0 = s.off[tid], o1 = s.off[tid + 1];
        if (o0 <= ta && ta < o1) s_bb[0] = tid;
        if (o0 <= tb && tb < o1) s_bb[1] = tid;
    }
    __syncthreads();
    if (s_bb[0] >= 0 && s_bb[1] >= 0) {
        if (tid == 0) {
            s.b0 = b_w;
            s.n = W;
            s.cur0 = s_bb[0];
            s.q_lo = q_lo;
            s.q_hi = q_hi;
            s.T0 = T0;
            s.T1 = T1;
        }
        __syncthreads();
        return true;
    }
    __syncthreads();  // every thread has read s_bb before the fallback rewrites it
    // fallback: exact searches, then the slice (or no staging at all)
    if (wid < 2) {
        const int b = pk_warp_search(off, nsel, wid == 0 ? ta : tb);
        if ((tid & 31) == 0) s_bb[wid] = b;
    }
    __syncthreads();
    const int b0 = s_bb[0], n = s_bb[1] - s_bb[0] + 1;
    if (n <= PK_SL) {
        for (int i = tid; i <= n; i += nt) s.off[i] = off[b0 + i];
        for (int i = tid; i < n; i += nt) {
            const Unit d = ld_unit(desc + b0 + i);
            s.row[i] = d.row;
            s.g[i] = d.g;
            s.adv[i] = d.adv;
        }
    }
    if (tid == 0) {
        s.b0 = b0;
        s.n = n <= PK_SL ? n : -1;
        s.cur0 = 0;
        s.q_lo = q_lo;
        s.q_hi = q_hi;
        s.T0 = T0;
        s.T1 = T1;
    }
    __syncthreads();
    return true;
}

// Selection of token t (t in [T0, T1)), as an index into the staged slice
// (staged) or a global selection index (unstaged); `cur` is a hint that only
// moves forward.
__device__ __forceinline__ int pk_find(const PkSlice& s, const int64_t* off, int nsel, long long t,
                                       int cur) {
    if (s.n >= 0) {
        while (cur + 1 < s.n && s.off[cur + 1] <= t) ++cur;
        return cur;
    }
    return pk_thread_search(off, nsel, t);
}

// Fields of the selection found by pk_find.
struct PkSel {
    long long off, end;
    int32_t row, g;
    double adv;
};
__device__ __forceinline__ PkSel pk_sel(const PkSlice& s, const int64_t* off, const Unit* desc,
                                        int j) {
    PkSel r;
    if (s.n >= 0) {
        r.off = s.off[j];
        r.end = s.off[j + 1];
        r.row = s.row[j];
        r.g = s.g[j];
        r.adv = s.adv[j];
    } else {
        const Unit d = ld_unit(desc + j);
        r.off = off[j];
        r.end = off[j + 1];
        r.row = d.row;
        r.g = d.g;
        r.adv = d.adv;
    }
    return r;
}

// Row elements [e, e+4) of a 16-byte aligned row as one quad (e >= 0, e + 3
// inside the row): two 128-bit loads and a funnel shift.
__device__ __forceinline__ uint4 pk_row_quad(const uint32_t* row, long long e) {
    const uint4* rq = reinterpret_cast<const uint4*>(row) + (e >> 2);
    const int a = (int)(e & 3);
    const uint4 lo = ld_stream(rq);
    return a ? funnel(lo, ld_stream(rq + 1), a) : lo;
}

// Store the valid elements [lo, hi) of destination quad q (tokens 4q..4q+3).
__device__ __forceinline__ void pk_store_quad(uint32_t* base, long long q, const uint4& v,
                                              long long lo, long long hi) {
    const long long t = 4 * q;
    if (t >= lo && t + 4 <= hi) {
        st_stream(reinterpret_cast<uint4*>(base) + q, v);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (t + i >= lo && t + i < hi) base[t + i] = q_at(v, i);
    }
}

}  // namespace rb
