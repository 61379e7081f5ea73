// ledger.cu — the UseEvent ledger and its replay diagnostics on the device
// (replab MetricsLedger, metrics.hpp:36-93, metrics.cpp).
//
//   rb_ledger_record_batch   sample(..., &ledger, batch_id, use_step)
//                            (replay_buffer.cpp:205-215, metrics.cpp:56-69):
//                            one event per selection of the buffer's current
//                            batch, appended by a kernel on the buffer's
//                            stream (no host round trip on the step).
//   rb_ledger_replay_counts  replay_counts (metrics.cpp:123-131): radix sort
//                            of the event ids (+ generated ids at count 0),
//                            reduce by key -> ascending ids, as std::map.
//   rb_ledger_global_use_order  global_use_order (metrics.cpp:133-151): events
//                            sorted by (use_step, batch_id, within_batch_rank)
//                            (three stable radix passes), then every batch
//                            Fisher-Yates shuffled with Rng::shuffle's draws
//                            (rng.hpp:59-64) taken from the caller's
//                            MT19937-64 stream bit-exactly.
//   rb_ledger_steps_since_last_use (metrics.cpp:153-170): the gap to the
//                            previous use of the same rollout in that order,
//                            by a stable sort of (id, position).
// The shuffle's draws: one CTA generates the stream block by block (twist in
// shared memory, one tempered word per thread); draw d takes the next word
// unless a below() rejection (probability bound/2^64) skips it, so a block is
// consumed in parallel up to its first rejection.  The swaps of a batch are
// sequential by definition: one thread per batch in shared memory.
//
// Validation follows the reference: generated twice / duplicate batch slot
// throw at the call (host-side sets); a use before creation is detected on
// the device and reported by the next diagnostics call or rb_ledger_check,
// which drops that event and every later one (the reference's state after
// its throw).
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <set>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "buffer_internal.cuh"
#include "rng_internal.cuh"

using namespace rb;

struct rb_ledger {
    int device = 0;
    cudaStream_t stream = nullptr;  // the ledger's own stream (appends and diagnostics)
    cudaEvent_t ev = nullptr;       // cross-stream ordering with the buffer's stream
    size_t n_ev = 0, cap_ev = 0;
    uint64_t* id = nullptr;
    int64_t *cstep = nullptr, *ustep = nullptr, *batch = nullptr, *rank = nullptr;
    size_t n_gen = 0, cap_gen = 0;
    uint64_t* gen = nullptr;
    unsigned long long* bad = nullptr;  // first event index with use_step < creation_step (~0: none)
    std::unordered_set<uint64_t> gen_set;
    std::unordered_set<int64_t> batch_whole;               // batch ids recorded by record_batch
    std::unordered_map<int64_t, std::set<int64_t>> pairs;  // (batch, rank) from record_uses
    std::unordered_map<int64_t, size_t> batch_size;        // B of each record_batch
    std::mutex mu;
};

namespace {

struct DevScope {
    int prev = 0;
    explicit DevScope(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DevScope() { cudaSetDevice(prev); }
};

template <class T>
void grow(T*& p, size_t n_keep, size_t cap, cudaStream_t s) {
    T* q = nullptr;
    RB_CUDA(cudaMallocAsync(&q, std::max<size_t>(cap, 1) * sizeof(T), s));
    if (p && n_keep) RB_CUDA(cudaMemcpyAsync(q, p, n_keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) RB_CUDA(cudaFreeAsync(p, s));
    p = q;
}

void reserve_events(rb_ledger* l, size_t need, cudaStream_t s) {
    if (need <= l->cap_ev) return;
    const size_t cap = std::max(need, 2 * l->cap_ev + 1024);
    grow(l->id, l->n_ev, cap, s);
    grow(l->cstep, l->n_ev, cap, s);
    grow(l->ustep, l->n_ev, cap, s);
    grow(l->batch, l->n_ev, cap, s);
    grow(l->rank, l->n_ev, cap, s);
    l->cap_ev = cap;
}

// scratch device memory of one diagnostics call (freed in order on the stream)
struct Scratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    template <class T>
    T* get(size_t n) {
        void* p = nullptr;
        RB_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), s));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
};

__global__ void k_ledger_append(const uint64_t* vid, const int64_t* vcstep, const int32_t* sel_slot,
                                long long n, int64_t batch_id, int64_t use_step, uint64_t* id,
                                int64_t* cstep, int64_t* ustep, int64_t* batch, int64_t* rank,
                                unsigned long long base, unsigned long long* bad) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const int32_t g = sel_slot[k];
        const int64_t c = vcstep[g];
        id[k] = vid[g];
        cstep[k] = c;
        ustep[k] = use_step;
        batch[k] = batch_id;
        rank[k] = k;
        if (use_step < c) atomicMin(bad, base + (unsigned long long)k);  // metrics.cpp:58-62
    }
}

__global__ void k_ledger_unpack(const rb_use_event* ev, long long n, uint64_t* id, int64_t* cstep,
                                int64_t* ustep, int64_t* batch, int64_t* rank) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const rb_use_event e = ev[k];
        id[k] = e.rollout_id;
        cstep[k] = e.creation_step;
        ustep[k] = e.use_step;
        batch[k] = e.batch_id;
        rank[k] = e.within_batch_rank;
    }
}

__global__ void k_ledger_pack(const uint64_t* id, const int64_t* cstep, const int64_t* ustep,
                              const int64_t* batch, const int64_t* rank, long long n,
                              rb_use_event* out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        out[k] = rb_use_event{id[k], cstep[k], ustep[k], batch[k], rank[k]};
}

__global__ void k_iota(uint64_t* p, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        p[k] = (uint64_t)k;
}
template <class T>
__global__ void k_gather_key(const T* key, const uint64_t* perm, long long n, T* out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        out[k] = key[perm[k]];
}
template <class T>
__global__ void k_fill(T* p, long long n, T v) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        p[k] = v;
}
// head flags of the (use_step, batch_id) groups of the sorted events
__global__ void k_group_heads(const int64_t* ustep, const int64_t* batch, const uint64_t* perm,
                              long long n, uint8_t* head) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const uint64_t e = perm[k];
        bool h = k == 0;
        if (!h) {
            const uint64_t p = perm[k - 1];
            h = ustep[e] != ustep[p] || batch[e] != batch[p];
        }
        head[k] = h;
    }
}
// per group: size m and draws m - 1 (Rng::shuffle: i = m .. 2)
__global__ void k_group_sizes(const uint64_t* starts, long long ng, long long n, int64_t* draws) {
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < ng;
         g += (long long)gridDim.x * blockDim.x) {
        const long long m = (long long)((g + 1 < ng ? starts[g + 1] : (uint64_t)n) - starts[g]);
        draws[g] = m > 1 ? m - 1 : 0;
    }
}
// bound of every draw: group g's draws are below(m), below(m-1), ..., below(2)
__global__ void k_draw_bounds(const uint64_t* starts, const int64_t* doff, long long ng, long long n,
                              uint64_t* bound) {
    for (long long g = blockIdx.x; g < ng; g += gridDim.x) {
        const long long m = (long long)((g + 1 < ng ? starts[g + 1] : (uint64_t)n) - starts[g]);
        for (long long t = threadIdx.x; t < m - 1; t += blockDim.x) bound[doff[g] + t] = (uint64_t)(m - t);
    }
}

// The draws of Rng::below (rng.cpp:40-51) for every bound, from the MT state
// `st` (advanced in place).  One CTA of >= 312 threads.
__global__ void __launch_bounds__(320) k_ledger_draws(MtState* st, const uint64_t* bound,
                                                      long long D, uint64_t* out) {
    __shared__ uint64_t mt[MT_N];
    __shared__ int s_first;
    const int t = threadIdx.x;
    for (int i = t; i < MT_N; i += blockDim.x) mt[i] = st->mt[i];
    long long d = 0;
    int w = (int)st->idx;
    unsigned long long words = 0;
    __syncthreads();
    while (d < D) {
        if (w >= MT_N) {
            mt_twist_block(mt);
            w = 0;
        }
        const long long k = min((long long)(MT_N - w), D - d);
        if (t == 0) s_first = INT32_MAX;
        __syncthreads();
        uint64_t y = 0, b = 1;
        bool ok = true;
        if (t < k) {
            y = mt_temper(mt[w + t]);
            b = bound[d + t];
            ok = y < below_limit(b);
            if (!ok) atomicMin(&s_first, t);
        }
        __syncthreads();
        const int r = s_first;  // words before the first rejection map 1:1 to draws
        if (t < k && t < r) out[d + t] = y % b;
        if (r == INT32_MAX) {
            d += k;
            w += (int)k;
            words += (unsigned long long)k;
        } else {  // draw d + r rejected word w + r: it retries from the next word
            d += r;
            w += r + 1;
            words += (unsigned long long)r + 1;
        }
        __syncthreads();
    }
    for (int i = t; i < MT_N; i += blockDim.x) st->mt[i] = mt[i];
    if (t == 0) {
        st->idx = (uint32_t)w;
        st->draws += words;
    }
}

// Rng::shuffle (rng.hpp:59-64) of every group in place: for i = m .. 2,
// swap(v[i-1], v[below(i)]).  One CTA per group, thread 0 swaps in shared
// memory (groups larger than the buffer swap in global memory).
constexpr int SHUF_SMEM = 12288;  // entries (96 KB)
__global__ void k_ledger_shuffle(uint64_t* perm, const uint64_t* starts, const int64_t* doff,
                                 long long ng, long long n, const uint64_t* draw) {
    extern __shared__ uint64_t sv[];
    for (long long g = blockIdx.x; g < ng; g += gridDim.x) {
        const long long s0 = (long long)starts[g];
        const long long m = (long long)((g + 1 < ng ? starts[g + 1] : (uint64_t)n) - s0);
        if (m < 2) continue;
        const uint64_t* dr = draw + doff[g];
        uint64_t* v = perm + s0;
        if (m <= SHUF_SMEM) {
            for (long long i = threadIdx.x; i < m; i += blockDim.x) sv[i] = v[i];
            __syncthreads();
            if (threadIdx.x == 0)
                for (long long i = m; i > 1; --i) {
                    const long long j = (long long)dr[m - i];
                    const uint64_t x = sv[i - 1];
                    sv[i - 1] = sv[j];
                    sv[j] = x;
                }
            __syncthreads();
            for (long long i = threadIdx.x; i < m; i += blockDim.x) v[i] = sv[i];
            __syncthreads();
        } else if (threadIdx.x == 0) {
            for (long long i = m; i > 1; --i) {
                const long long j = (long long)dr[m - i];
                const uint64_t x = v[i - 1];
                v[i - 1] = v[j];
                v[j] = x;
            }
        }
    }
}

// gaps: sorted (id, position) pairs; the previous entry with the same id is
// the previous use in the global order (metrics.cpp:160-168)
__global__ void k_ledger_gaps(const uint64_t* sid, const uint64_t* spos, const uint64_t* order,
                              const int64_t* ustep, long long n, int64_t* gap, uint8_t* has) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const uint64_t p = spos[k];
        if (k > 0 && sid[k - 1] == sid[k]) {
            gap[p] = ustep[order[p]] - ustep[order[spos[k - 1]]];
            has[p] = 1;
        } else {
            gap[p] = 0;
            has[p] = 0;
        }
    }
}

struct SumOp {
    __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const { return a + b; }
};

unsigned grid_of(long long n) { return (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8)); }

// Sticky use-before-creation check (metrics.cpp:58-62): drop the offending
// event and everything after it, then throw the reference's message.
void check_bad(rb_ledger* l) {
    unsigned long long b = ~0ULL;
    RB_CUDA(cudaMemcpyAsync(&b, l->bad, sizeof b, cudaMemcpyDeviceToHost, l->stream));
    RB_CUDA(cudaStreamSynchronize(l->stream));
    if (b == ~0ULL) return;
    uint64_t rid = 0;
    RB_CUDA(cudaMemcpy(&rid, l->id + b, sizeof rid, cudaMemcpyDeviceToHost));
    const unsigned long long none = ~0ULL;
    RB_CUDA(cudaMemcpy(l->bad, &none, sizeof none, cudaMemcpyHostToDevice));
    l->n_ev = (size_t)b;
    invalid("use event for rollout " + std::to_string(rid) + " precedes its creation step");
}

// global_use_order into `order` (device, n_ev entries), consuming rng.
void use_order(rb_ledger* l, rb_rng* rng, uint64_t* order, Scratch& sc) {
    const long long n = (long long)l->n_ev;
    cudaStream_t s = l->stream;
    if (n == 0) return;
    uint64_t* perm = order;
    uint64_t* perm2 = sc.get<uint64_t>(n);
    int64_t* key = sc.get<int64_t>(n);
    int64_t* key2 = sc.get<int64_t>(n);
    k_iota<<<grid_of(n), 256, 0, s>>>(perm, n);
    size_t tb = 0;
    RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, perm, perm2, (int)n, 0, 64, s));
    void* tmp = sc.get<char>(tb);
    // LSD: within_batch_rank, batch_id, use_step (each pass stable)
    const int64_t* keys[3] = {l->rank, l->batch, l->ustep};
    for (int pass = 0; pass < 3; ++pass) {
        k_gather_key<<<grid_of(n), 256, 0, s>>>(keys[pass], perm, n, key);
        RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, perm, perm2, (int)n, 0, 64, s));
        RB_CUDA(cudaMemcpyAsync(perm, perm2, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    }
    // groups and their draws
    uint8_t* head = sc.get<uint8_t>(n);
    k_group_heads<<<grid_of(n), 256, 0, s>>>(l->ustep, l->batch, perm, n, head);
    uint64_t* iota = sc.get<uint64_t>(n);
    k_iota<<<grid_of(n), 256, 0, s>>>(iota, n);
    uint64_t* starts = sc.get<uint64_t>(n);
    long long* ng_d = sc.get<long long>(1);
    size_t tb2 = 0;
    RB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, iota, head, starts, ng_d, (int)n, s));
    void* tmp2 = sc.get<char>(tb2);
    RB_CUDA(cub::DeviceSelect::Flagged(tmp2, tb2, iota, head, starts, ng_d, (int)n, s));
    long long ng = 0;
    RB_CUDA(cudaMemcpyAsync(&ng, ng_d, sizeof ng, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    int64_t* dcount = sc.get<int64_t>(ng + 1);
    int64_t* doff = sc.get<int64_t>(ng + 1);
    k_group_sizes<<<grid_of(ng), 256, 0, s>>>(starts, ng, n, dcount);
    k_fill<int64_t><<<1, 1, 0, s>>>(dcount + ng, 1, 0);
    size_t tb3 = 0;
    RB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, dcount, doff, (int)(ng + 1), s));
    void* tmp3 = sc.get<char>(tb3);
    RB_CUDA(cub::DeviceScan::ExclusiveSum(tmp3, tb3, dcount, doff, (int)(ng + 1), s));
    long long D = 0;
    RB_CUDA(cudaMemcpyAsync(&D, doff + ng, sizeof D, cudaMemcpyDeviceToHost, s));
    RB_CUDA(cudaStreamSynchronize(s));
    if (D == 0) return;
    uint64_t* bound = sc.get<uint64_t>(D);
    uint64_t* draw = sc.get<uint64_t>(D);
    k_draw_bounds<<<(unsigned)std::min<long long>(ng, 148 * 8), 256, 0, s>>>(starts, doff, ng, n, bound);
    // the caller's stream: host-authoritative state -> device -> back
    rng->to_host();
    MtState* st = sc.get<MtState>(1);
    RB_CUDA(cudaMemcpyAsync(st, &rng->host, sizeof(MtState), cudaMemcpyHostToDevice, s));
    k_ledger_draws<<<1, 320, 0, s>>>(st, bound, D, draw);
    RB_CUDA(cudaMemcpyAsync(&rng->host, st, sizeof(MtState), cudaMemcpyDeviceToHost, s));
    static bool attr = false;
    if (!attr) {
        RB_CUDA(cudaFuncSetAttribute(k_ledger_shuffle, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     SHUF_SMEM * 8));
        attr = true;
    }
    k_ledger_shuffle<<<(unsigned)std::min<long long>(ng, 148 * 4), 128, SHUF_SMEM * 8, s>>>(
        perm, starts, doff, ng, n, draw);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaStreamSynchronize(s));  // rng->host is written back
}

template <class T>
void copy_out(T* dst, const T* src, size_t n, cudaStream_t s) {
    if (dst && n) RB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDefault, s));
}

}  // namespace

extern "C" {

int rb_ledger_create(int device, rb_ledger** out) {
    return guard([&] {
        require_device();
        rb_ledger* l = new rb_ledger();
        if (device < 0) RB_CUDA(cudaGetDevice(&device));
        l->device = device;
        DevScope ds(device);
        RB_CUDA(cudaMalloc(&l->bad, sizeof(unsigned long long)));
        const unsigned long long none = ~0ULL;
        RB_CUDA(cudaMemcpy(l->bad, &none, sizeof none, cudaMemcpyHostToDevice));
        *out = l;
    });
}

void rb_ledger_destroy(rb_ledger* l) {
    if (!l) return;
    DevScope ds(l->device);
    if (l->stream) cudaStreamSynchronize(l->stream);
    if (l->ev) cudaEventDestroy(l->ev);
    for (void* p : {(void*)l->id, (void*)l->cstep, (void*)l->ustep, (void*)l->batch, (void*)l->rank,
                    (void*)l->gen, (void*)l->bad})
        if (p) cudaFree(p);
    if (l->stream) cudaStreamDestroy(l->stream);
    delete l;
}

// metrics.cpp:44-53
int rb_ledger_note_generated(rb_ledger* l, const uint64_t* ids, size_t n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
        std::vector<uint64_t> h(n);
        if (n) RB_CUDA(cudaMemcpy(h.data(), ids, n * 8, cudaMemcpyDefault));
        for (size_t i = 0; i < n; ++i) {
            if (!l->gen_set.insert(h[i]).second) {
                for (size_t k = 0; k < i; ++k) l->gen_set.erase(h[k]);  // nothing applied
                invalid("rollout " + std::to_string(h[i]) + " noted as generated twice");
            }
        }
        if (l->n_gen + n > l->cap_gen) {
            const size_t cap = std::max(l->n_gen + n, 2 * l->cap_gen + 1024);
            grow(l->gen, l->n_gen, cap, l->stream);
            l->cap_gen = cap;
        }
        if (n) RB_CUDA(cudaMemcpyAsync(l->gen + l->n_gen, h.data(), n * 8, cudaMemcpyHostToDevice, l->stream));
        RB_CUDA(cudaStreamSynchronize(l->stream));
        l->n_gen += n;
    });
}

// sample(batch, rng, &ledger, batch_id, use_step): the current batch's events
int rb_ledger_record_batch(rb_ledger* l, rb_buffer* b, int64_t batch_id, int64_t use_step) {
    return guard([&] {
        std::lock_guard<std::recursive_mutex> lb(b->mu);
        std::lock_guard<std::mutex> lk(l->mu);
        if (b->device != l->device) invalid("rb_ledger_record_batch: buffer on another device");
        DevScope ds(l->device);
        const size_t n = b->B;
        if (l->batch_whole.count(batch_id) || (l->pairs.count(batch_id) && n > 0 &&
                                                *l->pairs[batch_id].begin() < (int64_t)n))
            invalid("duplicate batch slot (batch " + std::to_string(batch_id) + ", rank " +
                    std::to_string(l->batch_whole.count(batch_id) ? 0 : *l->pairs[batch_id].begin()) + ")");
        if (n == 0) return;
        // the ledger's own stream, ordered after the sampler on the buffer's
        // stream, and the buffer's later work (an insert may overwrite the
        // sampled slots) ordered after the append: no host wait
        if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
        if (!l->ev) RB_CUDA(cudaEventCreateWithFlags(&l->ev, cudaEventDisableTiming));
        RB_CUDA(cudaEventRecord(l->ev, b->stream));
        RB_CUDA(cudaStreamWaitEvent(l->stream, l->ev, 0));
        reserve_events(l, l->n_ev + n, l->stream);
        const size_t o = l->n_ev;
        k_ledger_append<<<grid_of((long long)n), 256, 0, l->stream>>>(
            b->v.id, b->v.cstep, b->sel_slot, (long long)n, batch_id, use_step, l->id + o,
            l->cstep + o, l->ustep + o, l->batch + o, l->rank + o, (unsigned long long)o, l->bad);
        RB_CUDA(cudaGetLastError());
        RB_CUDA(cudaEventRecord(l->ev, l->stream));
        RB_CUDA(cudaStreamWaitEvent(b->stream, l->ev, 0));
        l->n_ev += n;
        l->batch_whole.insert(batch_id);
        l->batch_size[batch_id] = n;
    });
}

// record_use for explicit events (host or device), metrics.cpp:56-69
int rb_ledger_record_uses(rb_ledger* l, const rb_use_event* ev, size_t n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        std::vector<rb_use_event> h(n);
        if (n) RB_CUDA(cudaMemcpy(h.data(), ev, n * sizeof(rb_use_event), cudaMemcpyDefault));
        std::vector<std::pair<int64_t, int64_t>> added;
        for (size_t i = 0; i < n; ++i) {
            const rb_use_event& e = h[i];
            std::string err;
            if (e.use_step < e.creation_step)
                err = "use event for rollout " + std::to_string(e.rollout_id) + " precedes its creation step";
            else if ((l->batch_whole.count(e.batch_id) && e.within_batch_rank >= 0 &&
                      (size_t)e.within_batch_rank < l->batch_size[e.batch_id]) ||
                     !l->pairs[e.batch_id].insert(e.within_batch_rank).second)
                err = "duplicate batch slot (batch " + std::to_string(e.batch_id) + ", rank " +
                      std::to_string(e.within_batch_rank) + ")";
            if (!err.empty()) {
                // the events before it are recorded, as in the reference's loop
                n = i;
                h.resize(i);
                if (n) {
                    if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
                    reserve_events(l, l->n_ev + n, l->stream);
                    rb_use_event* d = nullptr;
                    RB_CUDA(cudaMallocAsync(&d, n * sizeof(rb_use_event), l->stream));
                    RB_CUDA(cudaMemcpyAsync(d, h.data(), n * sizeof(rb_use_event), cudaMemcpyHostToDevice, l->stream));
                    const size_t o = l->n_ev;
                    k_ledger_unpack<<<grid_of((long long)n), 256, 0, l->stream>>>(
                        d, (long long)n, l->id + o, l->cstep + o, l->ustep + o, l->batch + o, l->rank + o);
                    RB_CUDA(cudaFreeAsync(d, l->stream));
                    RB_CUDA(cudaStreamSynchronize(l->stream));
                    l->n_ev += n;
                }
                invalid(err);
            }
        }
        if (!n) return;
        if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
        reserve_events(l, l->n_ev + n, l->stream);
        rb_use_event* d = nullptr;
        RB_CUDA(cudaMallocAsync(&d, n * sizeof(rb_use_event), l->stream));
        RB_CUDA(cudaMemcpyAsync(d, h.data(), n * sizeof(rb_use_event), cudaMemcpyHostToDevice, l->stream));
        const size_t o = l->n_ev;
        k_ledger_unpack<<<grid_of((long long)n), 256, 0, l->stream>>>(
            d, (long long)n, l->id + o, l->cstep + o, l->ustep + o, l->batch + o, l->rank + o);
        RB_CUDA(cudaFreeAsync(d, l->stream));
        RB_CUDA(cudaStreamSynchronize(l->stream));
        l->n_ev += n;
    });
}

int rb_ledger_check(rb_ledger* l) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (l->stream) check_bad(l);
    });
}

int rb_ledger_sizes(rb_ledger* l, size_t* n_events, size_t* n_generated) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (l->stream) check_bad(l);
        if (n_events) *n_events = l->n_ev;
        if (n_generated) *n_generated = l->n_gen;
    });
}

int rb_ledger_events(rb_ledger* l, rb_use_event* out, size_t cap, size_t* n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (l->stream) check_bad(l);
        *n = l->n_ev;
        if (!out || !l->n_ev) return;
        if (cap < l->n_ev) invalid("rb_ledger_events: capacity below the event count");
        Scratch sc(l->stream);
        rb_use_event* d = sc.get<rb_use_event>(l->n_ev);
        k_ledger_pack<<<grid_of((long long)l->n_ev), 256, 0, l->stream>>>(
            l->id, l->cstep, l->ustep, l->batch, l->rank, (long long)l->n_ev, d);
        copy_out(out, d, l->n_ev, l->stream);
        RB_CUDA(cudaStreamSynchronize(l->stream));
    });
}

// replay_counts(ledger, include_zero_use), metrics.cpp:123-131
int rb_ledger_replay_counts(rb_ledger* l, int include_zero_use, uint64_t* out_ids,
                            uint64_t* out_counts, size_t cap, size_t* n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
        check_bad(l);
        cudaStream_t s = l->stream;
        const long long ne = (long long)l->n_ev, ng = include_zero_use ? (long long)l->n_gen : 0;
        const long long m = ne + ng;
        *n = 0;
        if (m == 0) return;
        Scratch sc(s);
        uint64_t* k = sc.get<uint64_t>(m);
        uint64_t* v = sc.get<uint64_t>(m);
        uint64_t* k2 = sc.get<uint64_t>(m);
        uint64_t* v2 = sc.get<uint64_t>(m);
        if (ne) RB_CUDA(cudaMemcpyAsync(k, l->id, ne * 8, cudaMemcpyDeviceToDevice, s));
        if (ng) RB_CUDA(cudaMemcpyAsync(k + ne, l->gen, ng * 8, cudaMemcpyDeviceToDevice, s));
        if (ne) k_fill<uint64_t><<<grid_of(ne), 256, 0, s>>>(v, ne, 1);
        if (ng) k_fill<uint64_t><<<grid_of(ng), 256, 0, s>>>(v + ne, ng, 0);
        size_t tb = 0;
        RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k, k2, v, v2, (int)m, 0, 64, s));
        void* tmp = sc.get<char>(tb);
        RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k, k2, v, v2, (int)m, 0, 64, s));
        long long* runs = sc.get<long long>(1);
        size_t tb2 = 0;
        RB_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, tb2, k2, k, v2, v, runs, SumOp(), (int)m, s));
        void* tmp2 = sc.get<char>(tb2);
        RB_CUDA(cub::DeviceReduce::ReduceByKey(tmp2, tb2, k2, k, v2, v, runs, SumOp(), (int)m, s));
        long long r = 0;
        RB_CUDA(cudaMemcpyAsync(&r, runs, sizeof r, cudaMemcpyDeviceToHost, s));
        RB_CUDA(cudaStreamSynchronize(s));
        *n = (size_t)r;
        if (!out_ids && !out_counts) return;
        if (cap < (size_t)r) invalid("rb_ledger_replay_counts: capacity below the id count");
        copy_out(out_ids, k, r, s);
        copy_out(out_counts, v, r, s);
        RB_CUDA(cudaStreamSynchronize(s));
    });
}

// global_use_order(ledger.events(), rng), metrics.cpp:133-151
int rb_ledger_global_use_order(rb_ledger* l, rb_rng* rng, uint64_t* out_order, size_t cap,
                               size_t* n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
        check_bad(l);
        *n = l->n_ev;
        if (!l->n_ev) return;
        if (cap < l->n_ev) invalid("rb_ledger_global_use_order: capacity below the event count");
        Scratch sc(l->stream);
        uint64_t* order = sc.get<uint64_t>(l->n_ev);
        use_order(l, rng, order, sc);
        copy_out(out_order, order, l->n_ev, l->stream);
        RB_CUDA(cudaStreamSynchronize(l->stream));
    });
}

// steps_since_last_use(ledger, rng), metrics.cpp:153-170: labels in the
// global use order; has_gap 0 = first use (nullopt).
int rb_ledger_steps_since_last_use(rb_ledger* l, rb_rng* rng, uint64_t* out_event_index,
                                   int64_t* out_gap, uint8_t* out_has_gap, size_t cap, size_t* n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(l->mu);
        DevScope ds(l->device);
        if (!l->stream) RB_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
        check_bad(l);
        const long long ne = (long long)l->n_ev;
        *n = (size_t)ne;
        if (!ne) return;
        if (cap < (size_t)ne) invalid("rb_ledger_steps_since_last_use: capacity below the event count");
        cudaStream_t s = l->stream;
        Scratch sc(s);
        uint64_t* order = sc.get<uint64_t>(ne);
        use_order(l, rng, order, sc);
        uint64_t* kid = sc.get<uint64_t>(ne);
        uint64_t* pos = sc.get<uint64_t>(ne);
        uint64_t* kid2 = sc.get<uint64_t>(ne);
        uint64_t* pos2 = sc.get<uint64_t>(ne);
        k_gather_key<uint64_t><<<grid_of(ne), 256, 0, s>>>(l->id, order, ne, kid);
        k_iota<<<grid_of(ne), 256, 0, s>>>(pos, ne);
        size_t tb = 0;
        RB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kid, kid2, pos, pos2, (int)ne, 0, 64, s));
        void* tmp = sc.get<char>(tb);
        RB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kid, kid2, pos, pos2, (int)ne, 0, 64, s));
        int64_t* gap = sc.get<int64_t>(ne);
        uint8_t* has = sc.get<uint8_t>(ne);
        k_ledger_gaps<<<grid_of(ne), 256, 0, s>>>(kid2, pos2, order, l->ustep, ne, gap, has);
        RB_CUDA(cudaGetLastError());
        copy_out(out_event_index, order, ne, s);
        copy_out(out_gap, gap, ne, s);
        copy_out(out_has_gap, has, ne, s);
        RB_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
