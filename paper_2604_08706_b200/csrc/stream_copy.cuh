// stream_copy.cuh — persistent work units and 128-bit funnel-shifted row I/O
// shared by the payload insert, the ragged gather and the token losses.
//
// Every heavy kernel of the step is a persistent grid (UNIT_GRID CTAs of
// UNIT_THREADS) striding over a device-built table of work units.  A unit is
// QPU = UNIT_THREADS * UNIT_U 16-byte quads of one trajectory, so ragged
// lengths balance across CTAs; its 32-byte descriptor carries everything the
// kernel needs (row, length, packed offset, advantage) so a unit costs one
// descriptor load, prefetched one unit ahead.
//
// Rows of the slot store are 16-byte aligned (stride % 4 == 0); packed
// (gathered) arrays start at arbitrary token offsets.  A warp owns 32*U
// consecutive quads; the neighbour quad a funnel shift needs comes from the
// adjacent lane by shuffle, so each quad is loaded from memory once.
#pragma once

#include <stdint.h>

namespace rb {

constexpr int UNIT_THREADS = 128;
constexpr int UNIT_U = 2;                          // quads per thread per unit
constexpr int QPU = UNIT_THREADS * UNIT_U;         // 256 quads = 1024 tokens
constexpr int UNIT_CTAS_PER_SM = 2048 / UNIT_THREADS;

struct __align__(16) Unit {
    int32_t row;    // payload row (local), or -1
    int32_t len;    // trajectory length in tokens
    int32_t k0;     // first quad of this unit (in the loop's quad space)
    int32_t g;      // global metadata slot (selection units) / record index (insert units)
    int64_t off;    // packed token offset (gather/loss: destination; insert: source)
    double adv;     // frozen advantage (selection units)
};
static_assert(sizeof(Unit) == 32, "unit descriptor is 32 bytes");

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& q) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(q.x), "r"(q.y),
                 "r"(q.z), "r"(q.w)
                 : "memory");
}
// Quad q of a packed 4-byte array whose valid elements end at element `lim`
// (exclusive): one 128-bit load when the quad lies before `lim`, else the
// valid words one by one (zeros past `lim`) — a batch's last quad never
// reads past the caller's array.
__device__ __forceinline__ uint4 ld_stream_lim(const void* base, long long q, long long lim) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(base) + 4 * q;
    if (4 * q + 4 <= lim) return ld_stream(w);
    const long long e = lim - 4 * q;
    return make_uint4(e > 0 ? __ldg(w) : 0u, e > 1 ? __ldg(w + 1) : 0u, e > 2 ? __ldg(w + 2) : 0u, 0u);
}
__device__ __forceinline__ Unit ld_unit(const Unit* u) {
    const uint4 a = *reinterpret_cast<const uint4*>(u);
    const uint4 b = *(reinterpret_cast<const uint4*>(u) + 1);
    Unit r;
    r.row = (int32_t)a.x;
    r.len = (int32_t)a.y;
    r.k0 = (int32_t)a.z;
    r.g = (int32_t)a.w;
    r.off = (int64_t)(((uint64_t)b.y << 32) | b.x);
    r.adv = __hiloint2double((int)b.w, (int)b.z);
    return r;
}
// out[i] = concat(lo, hi)[a + i]
__device__ __forceinline__ uint4 funnel(const uint4& lo, const uint4& hi, int a) {
    switch (a & 3) {
        case 0: return lo;
        case 1: return make_uint4(lo.y, lo.z, lo.w, hi.x);
        case 2: return make_uint4(lo.z, lo.w, hi.x, hi.y);
        default: return make_uint4(lo.w, hi.x, hi.y, hi.z);
    }
}
__device__ __forceinline__ uint4 shfl4(const uint4& q, int src) {
    return make_uint4(__shfl_sync(0xffffffffu, q.x, src), __shfl_sync(0xffffffffu, q.y, src),
                      __shfl_sync(0xffffffffu, q.z, src), __shfl_sync(0xffffffffu, q.w, src));
}
__device__ __forceinline__ uint4 shfl_up4(const uint4& q) {
    return make_uint4(__shfl_up_sync(0xffffffffu, q.x, 1), __shfl_up_sync(0xffffffffu, q.y, 1),
                      __shfl_up_sync(0xffffffffu, q.z, 1), __shfl_up_sync(0xffffffffu, q.w, 1));
}
__device__ __forceinline__ uint4 shfl_down4(const uint4& q) {
    return make_uint4(__shfl_down_sync(0xffffffffu, q.x, 1),
                      __shfl_down_sync(0xffffffffu, q.y, 1),
                      __shfl_down_sync(0xffffffffu, q.z, 1),
                      __shfl_down_sync(0xffffffffu, q.w, 1));
}
__device__ __forceinline__ uint32_t q_at(const uint4& q, int i) {
    return i == 0 ? q.x : i == 1 ? q.y : i == 2 ? q.z : q.w;
}

// Row (aligned) -> packed quads.  The warp's quads are kq[s] = kw + 32*s + lane
// of the DESTINATION quad space of a row packed at element offset `doff`
// (a = doff & 3): destination quad k holds row elements 4k-a .. 4k-a+3, i.e.
// funnel(src quad k-1, src quad k, 4-a).  Returns the U destination quads.
template <int U>
__device__ __forceinline__ void row_to_packed_quads(const uint4* rowq, int nsq, int a, int kw,
                                                    uint4 (&o)[U]) {
    const int lane = threadIdx.x & 31;
    uint4 cur[U];
#pragma unroll
    for (int s = 0; s < U; ++s) {
        const int k = kw + 32 * s + lane;
        cur[s] = (k >= 0 && k < nsq) ? ld_stream(rowq + k) : make_uint4(0, 0, 0, 0);
    }
    if (a == 0) {
#pragma unroll
        for (int s = 0; s < U; ++s) o[s] = cur[s];
        return;
    }
    uint4 first_prev = make_uint4(0, 0, 0, 0);
    if (lane == 0 && kw >= 1 && kw - 1 < nsq) first_prev = ld_stream(rowq + kw - 1);
#pragma unroll
    for (int s = 0; s < U; ++s) {
        uint4 prev = shfl_up4(cur[s]);
        const uint4 carry = s ? shfl4(cur[s > 0 ? s - 1 : 0], 31) : first_prev;
        if (lane == 0) prev = carry;
        o[s] = funnel(prev, cur[s], 4 - a);
    }
}

// Packed (element offset `soff`, any alignment) -> aligned row quads: row
// quad k = funnel(src quad Q0+k, src quad Q0+k+1, a), a = soff & 3.
// (lim = a + len: the valid elements counted from quad Q0's first element;
// the last quad is read word by word, never past the caller's array)
// (BOUNDED = false: the caller knows quad nsq-1 ends inside its array)
template <int U, bool BOUNDED = true>
__device__ __forceinline__ void packed_to_row_quads(const uint4* srcq0 /* quad Q0 */, int nsq,
                                                    int a, int kw, uint4 (&o)[U], int lim) {
    const int lane = threadIdx.x & 31;
    uint4 cur[U];
#pragma unroll
    for (int s = 0; s < U; ++s) {
        const int k = kw + 32 * s + lane;
        cur[s] = (k < nsq) ? (BOUNDED ? ld_stream_lim(srcq0, k, lim) : ld_stream(srcq0 + k))
                           : make_uint4(0, 0, 0, 0);
    }
    if (a == 0) {
#pragma unroll
        for (int s = 0; s < U; ++s) o[s] = cur[s];
        return;
    }
    const int klast = kw + 32 * U;  // first quad after the warp's span
    uint4 last_next = make_uint4(0, 0, 0, 0);
    if (lane == 31 && klast < nsq)
        last_next = BOUNDED ? ld_stream_lim(srcq0, klast, lim) : ld_stream(srcq0 + klast);
#pragma unroll
    for (int s = 0; s < U; ++s) {
        uint4 next = shfl_down4(cur[s]);
        const uint4 carry = (s + 1 < U) ? shfl4(cur[s + 1 < U ? s + 1 : s], 0) : last_next;
        if (lane == 31) next = carry;
        o[s] = funnel(cur[s], next, a);
    }
}

// Store destination quad `k` (global quad index `gq`) of which only the
// elements with 0 <= e0+i < len are valid.
__device__ __forceinline__ void store_quad_masked(uint32_t* base, long long gq, const uint4& q,
                                                  int e0, int len) {
    if (e0 >= 0 && e0 + 3 < len) {
        st_stream(reinterpret_cast<uint4*>(base) + gq, q);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (e0 + i >= 0 && e0 + i < len) base[4 * gq + i] = q_at(q, i);
    }
}

// Block-wide exclusive scan helper (blockDim.x <= 1024, multiple of 32).
// Each thread contributes `x`; returns the exclusive prefix and the total.
__device__ __forceinline__ long long block_exclusive_scan(long long x, long long* total) {
    __shared__ long long s_w[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        long long w = lane < nw ? s_w[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    const long long base = wid ? s_w[wid - 1] : 0;
    *total = s_w[nw - 1];
    __syncthreads();
    return base + incl - x;
}

}  // namespace rb
