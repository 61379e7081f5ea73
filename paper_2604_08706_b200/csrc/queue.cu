// queue.cu — replab::TransferQueue on the GPU (transfer_queue.hpp:12-35,
// transfer_queue.cpp:1-50): the consume-once LIFO hand-off of the paper's
// no-buffer baseline, with the token payload kept in HBM next to the records.
//
// Layout: records (80-B rb_record, stack order), lengths, and fixed-stride
// payload rows (row i = stack position i).  The stack height lives on the
// host (every push / pop is host-driven, so it is exact); an unbounded queue
// grows its device storage by doubling.  push_group is all-or-nothing
// (transfer_queue.cpp:22-29): a group that does not fit is refused before
// anything is copied; one with a length over max_tokens is refused too.
// pop(k) is k reference pops: the most recent record first.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "stream_copy.cuh"

using namespace rb;

struct rb_queue {
    size_t cap = 0;     // 0 = unbounded (capacity nullopt)
    size_t alloc = 0;   // device slots allocated
    size_t size = 0;    // stack height (exact: host-driven)
    int32_t max_tokens = 0, stride = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    rb_record* rec = nullptr;
    int32_t* len = nullptr;
    int32_t* tok = nullptr;
    float* lpo = nullptr;
    int* err = nullptr;          // device flag of the last push (1 = a length out of range)
    int64_t* off = nullptr;      // pop scratch: packed offsets
    size_t off_cap = 0;
    void* stage = nullptr;       // device staging of host inputs / outputs
    size_t stage_cap = 0;
    ~rb_queue();
    void reserve(size_t n);
    void* staging(size_t bytes);
};

namespace {

struct QIn {
    long long n, base;
    const uint64_t *id, *prompt, *group;
    const int64_t *cstep, *pver;
    const double *reward, *blp, *adv;
    const uint8_t* correct;
    const int64_t* goff;
    long long ngroups;
    const int64_t* toff;
    int32_t maxlen;
};

// Records (+ advantages per group when not given, bandit.cpp:276-294) and
// lengths of one pushed group, after checking every length: one CTA.
__global__ void __launch_bounds__(1024) k_queue_push(QIn in, rb_record* rec, int32_t* len, int* err) {
    int bad = 0;
    for (long long j = threadIdx.x; j < in.n; j += blockDim.x) {
        const long long l = in.toff ? in.toff[j + 1] - in.toff[j] : 0;
        if (l < 0 || l > in.maxlen) bad = 1;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) *err = bad;
    if (bad) return;
    for (long long j = threadIdx.x; j < in.n; j += blockDim.x) {
        double adv = in.adv ? in.adv[j] : 0.0;
        if (!in.adv && in.goff) {  // the record's group: binary search, then its statistics
            long long lo = 0, hi = in.ngroups;
            while (hi - lo > 1) {
                const long long mid = (lo + hi) >> 1;
                if (in.goff[mid] <= j) lo = mid;
                else hi = mid;
            }
            const long long b = in.goff[lo], e = in.goff[lo + 1], m = e - b;
            double mean = 0.0, var = 0.0;
            for (long long k = b; k < e; ++k) mean = __dadd_rn(mean, in.reward[k]);
            mean = __ddiv_rn(mean, (double)m);
            for (long long k = b; k < e; ++k) {
                const double d = __dsub_rn(in.reward[k], mean);
                var = __dadd_rn(var, __dmul_rn(d, d));
            }
            const double sd = __dsqrt_rn(__ddiv_rn(var, (double)m));
            adv = sd < 1e-8 ? 0.0 : __ddiv_rn(__dsub_rn(in.reward[j], mean), sd);
        }
        rb_record r;
        r.rollout_id = in.id[j];
        r.prompt_id = in.prompt ? in.prompt[j] : 0;
        r.group_id = in.group ? in.group[j] : 0;
        r.creation_step = in.cstep ? in.cstep[j] : 0;
        r.policy_version = in.pver ? in.pver[j] : 0;
        r.reward = in.reward[j];
        r.is_correct = in.correct ? in.correct[j] != 0 : in.reward[j] == 1.0;
        r.behavior_logprob = in.blp ? in.blp[j] : 0.0;
        r.advantage = adv;
        r.use_count = 0;
        rec[in.base + j] = r;
        len[in.base + j] = in.toff ? (int32_t)(in.toff[j + 1] - in.toff[j]) : 0;
    }
}

// Payload of record j -> row base + j: one CTA per record, coalesced words.
__global__ void k_queue_rows_in(const int64_t* toff, const int32_t* tokens, const float* lpo_in,
                                long long base, int stride, const int* err, int32_t* tok,
                                float* lpo) {
    if (*err) return;
    const long long j = blockIdx.x;
    const long long o = toff[j], l = toff[j + 1] - o;
    const size_t row = (size_t)(base + j) * stride;
    for (long long t = threadIdx.x; t < l; t += blockDim.x) {
        if (tokens) tok[row + t] = tokens[o + t];
        if (lpo_in) lpo[row + t] = lpo_in[o + t];
    }
}

// pop(n): records of stack positions size-1 .. size-n (most recent first),
// their lengths scanned into packed offsets: one CTA.
__global__ void __launch_bounds__(1024) k_queue_pop(const rb_record* rec, const int32_t* len,
                                                    long long size, long long n, rb_record* out,
                                                    int64_t* off) {
    long long carry = 0;
    for (long long c = 0; c < n; c += blockDim.x) {
        const long long i = c + threadIdx.x;
        const long long L = i < n ? len[size - 1 - i] : 0;
        if (i < n && out) out[i] = rec[size - 1 - i];
        long long tot;
        const long long ex = block_exclusive_scan(L, &tot);
        if (i < n) off[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) off[n] = carry;
}

// Payload of popped record i (row size-1-i) -> packed at off[i].
__global__ void k_queue_rows_out(const int32_t* tok, const float* lpo, long long size, int stride,
                                 const int32_t* len, const int64_t* off, int32_t* out_tok,
                                 float* out_lpo) {
    const long long i = blockIdx.x;
    const long long p = size - 1 - i;
    const long long l = len[p], o = off[i];
    const size_t row = (size_t)p * stride;
    for (long long t = threadIdx.x; t < l; t += blockDim.x) {
        if (out_tok) out_tok[o + t] = tok[row + t];
        if (out_lpo) out_lpo[o + t] = lpo[row + t];
    }
}

template <class T>
T* qalloc(size_t n) {
    T* p = nullptr;
    RB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}

struct QDeviceScope {
    int prev = -1;
    explicit QDeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~QDeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

rb_queue::~rb_queue() {
    if (device >= 0) cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    void* ps[] = {rec, len, tok, lpo, err, off, stage};
    for (void* p : ps)
        if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
    cudaGetLastError();
}

void rb_queue::reserve(size_t n) {
    if (n <= alloc) return;
    size_t a = std::max<size_t>(alloc ? alloc * 2 : 64, n);
    if (cap) a = std::min(a, cap);
    rb_record* r2 = qalloc<rb_record>(a);
    int32_t* l2 = qalloc<int32_t>(a);
    int32_t* t2 = stride ? qalloc<int32_t>(a * (size_t)stride) : nullptr;
    float* p2 = stride ? qalloc<float>(a * (size_t)stride) : nullptr;
    RB_CUDA(cudaStreamSynchronize(stream));
    if (size) {
        RB_CUDA(cudaMemcpy(r2, rec, size * sizeof(rb_record), cudaMemcpyDeviceToDevice));
        RB_CUDA(cudaMemcpy(l2, len, size * 4, cudaMemcpyDeviceToDevice));
        if (stride) {
            RB_CUDA(cudaMemcpy(t2, tok, size * (size_t)stride * 4, cudaMemcpyDeviceToDevice));
            RB_CUDA(cudaMemcpy(p2, lpo, size * (size_t)stride * 4, cudaMemcpyDeviceToDevice));
        }
    }
    void* old[] = {rec, len, tok, lpo};
    for (void* p : old)
        if (p) cudaFree(p);
    rec = r2;
    len = l2;
    tok = t2;
    lpo = p2;
    alloc = a;
}

void* rb_queue::staging(size_t bytes) {
    if (bytes > stage_cap) {
        RB_CUDA(cudaStreamSynchronize(stream));
        if (stage) cudaFree(stage);
        stage_cap = std::max(bytes, stage_cap * 2);
        RB_CUDA(cudaMalloc(&stage, stage_cap));
    }
    return stage;
}

extern "C" {

int rb_queue_create(size_t capacity, int32_t max_tokens, int device, rb_queue** out) {
    return guard([&] {
        require_device();
        if (max_tokens < 0) invalid("rb_queue_create: max_tokens must be >= 0");
        if (device < 0) RB_CUDA(cudaGetDevice(&device));
        QDeviceScope ds(device);
        auto* q = new rb_queue();
        try {
            q->cap = capacity;
            q->max_tokens = max_tokens;
            q->stride = (max_tokens + 3) & ~3;
            q->device = device;
            RB_CUDA(cudaStreamCreateWithFlags(&q->stream, cudaStreamNonBlocking));
            q->err = qalloc<int>(1);
            q->reserve(capacity ? std::min<size_t>(capacity, 1 << 16) : 64);
        } catch (...) {
            delete q;
            throw;
        }
        *out = q;
    });
}

void rb_queue_destroy(rb_queue* q) { delete q; }

int rb_queue_size(const rb_queue* q, size_t* out) {
    *out = q->size;
    return RB_OK;
}

int rb_queue_capacity(const rb_queue* q, size_t* capacity, int* bounded) {
    if (capacity) *capacity = q->cap;
    if (bounded) *bounded = q->cap != 0;
    return RB_OK;
}

int rb_queue_push_group(rb_queue* q, const rb_insert_batch* bt_in, int* accepted) {
    return guard([&] {
        QDeviceScope ds(q->device);
        *accepted = 0;
        rb_insert_batch bt = *bt_in;
        const size_t n = bt.n;
        if (n == 0) {
            *accepted = 1;
            return;
        }
        if (!bt.rollout_id || !bt.reward) invalid("rb_queue_push_group: rollout_id and reward are required");
        if (q->cap && q->size + n > q->cap) return;  // transfer_queue.cpp:24-26: back-pressure
        if (bt.tok_offsets && (bt.tokens || bt.logp_old) && q->stride == 0)
            invalid("rb_queue_push_group: queue holds no token payload (max_tokens = 0)");
        q->reserve(q->size + n);
        // host inputs -> one device staging area (synchronous copies: a baseline path)
        struct Item {
            const void** ptr;
            size_t bytes;
        };
        std::vector<Item> items;
        auto add = [&](const void** p, size_t bytes) {
            if (*p && !is_device_ptr(*p)) items.push_back({p, bytes});
        };
        add((const void**)&bt.rollout_id, n * 8);
        add((const void**)&bt.prompt_id, n * 8);
        add((const void**)&bt.group_id, n * 8);
        add((const void**)&bt.creation_step, n * 8);
        add((const void**)&bt.policy_version, n * 8);
        add((const void**)&bt.reward, n * 8);
        add((const void**)&bt.is_correct, n);
        add((const void**)&bt.behavior_logprob, n * 8);
        add((const void**)&bt.advantage, n * 8);
        add((const void**)&bt.group_offsets, (bt.n_groups + 1) * 8);
        size_t elems = 0;
        if (bt.tok_offsets) {
            int64_t last = 0;
            RB_CUDA(cudaMemcpy(&last, bt.tok_offsets + n, 8, cudaMemcpyDefault));
            elems = (size_t)std::max<int64_t>(last, 0);
        }
        add((const void**)&bt.tok_offsets, (n + 1) * 8);
        add((const void**)&bt.tokens, elems * 4);
        add((const void**)&bt.logp_old, elems * 4);
        size_t total = 0;
        for (auto& it : items) total += (it.bytes + 255) & ~size_t(255);
        char* st = total ? (char*)q->staging(total) : nullptr;
        size_t o = 0;
        for (auto& it : items) {
            RB_CUDA(cudaMemcpyAsync(st + o, *it.ptr, it.bytes, cudaMemcpyHostToDevice, q->stream));
            *it.ptr = st + o;
            o += (it.bytes + 255) & ~size_t(255);
        }
        QIn in{};
        in.n = (long long)n;
        in.base = (long long)q->size;
        in.id = bt.rollout_id;
        in.prompt = bt.prompt_id;
        in.group = bt.group_id;
        in.cstep = bt.creation_step;
        in.pver = bt.policy_version;
        in.reward = bt.reward;
        in.blp = bt.behavior_logprob;
        in.adv = bt.advantage;
        in.correct = bt.is_correct;
        in.goff = bt.group_offsets;
        in.ngroups = (long long)bt.n_groups;
        in.toff = bt.tok_offsets;
        in.maxlen = q->max_tokens;
        k_queue_push<<<1, 1024, 0, q->stream>>>(in, q->rec, q->len, q->err);
        RB_CUDA(cudaGetLastError());
        if (bt.tok_offsets && (bt.tokens || bt.logp_old) && q->stride) {
            k_queue_rows_in<<<(unsigned)n, 256, 0, q->stream>>>(bt.tok_offsets, bt.tokens,
                                                                bt.logp_old, in.base, q->stride,
                                                                q->err, q->tok, q->lpo);
            RB_CUDA(cudaGetLastError());
        }
        int e = 0;
        RB_CUDA(cudaMemcpyAsync(&e, q->err, sizeof e, cudaMemcpyDeviceToHost, q->stream));
        RB_CUDA(cudaStreamSynchronize(q->stream));
        if (e) invalid("rb_queue_push_group: trajectory length exceeds max_tokens");
        q->size += n;
        *accepted = 1;
    });
}

int rb_queue_pop(rb_queue* q, size_t k, rb_record* out_records, size_t* n_popped,
                 int32_t* out_tokens, float* out_logp_old, int64_t* out_offsets) {
    return guard([&] {
        QDeviceScope ds(q->device);
        const size_t n = std::min(k, q->size);
        if (n_popped) *n_popped = n;
        if (n == 0) {
            if (out_offsets) {
                const int64_t zero = 0;
                RB_CUDA(cudaMemcpy(out_offsets, &zero, 8, cudaMemcpyDefault));
            }
            return;
        }
        if ((out_tokens || out_logp_old) && q->stride == 0)
            invalid("rb_queue_pop: queue holds no token payload (max_tokens = 0)");
        if (n + 1 > q->off_cap) {
            RB_CUDA(cudaStreamSynchronize(q->stream));
            if (q->off) cudaFree(q->off);
            q->off_cap = std::max(n + 1, q->off_cap * 2);
            q->off = qalloc<int64_t>(q->off_cap);
        }
        const bool hr = out_records && !is_device_ptr(out_records);
        rb_record* dr = out_records;
        if (hr) dr = (rb_record*)q->staging(n * sizeof(rb_record));
        k_queue_pop<<<1, 1024, 0, q->stream>>>(q->rec, q->len, (long long)q->size, (long long)n, dr,
                                               q->off);
        RB_CUDA(cudaGetLastError());
        if (hr)
            RB_CUDA(cudaMemcpyAsync(out_records, dr, n * sizeof(rb_record), cudaMemcpyDeviceToHost,
                                    q->stream));
        if (out_tokens || out_logp_old) {
            int64_t total = 0;
            RB_CUDA(cudaMemcpyAsync(&total, q->off + n, 8, cudaMemcpyDeviceToHost, q->stream));
            RB_CUDA(cudaStreamSynchronize(q->stream));
            const bool ht = out_tokens && !is_device_ptr(out_tokens);
            const bool hl = out_logp_old && !is_device_ptr(out_logp_old);
            char* st = (ht || hl) ? (char*)q->staging((size_t)total * 8 + 64) : nullptr;
            int32_t* dt = ht ? (int32_t*)st : out_tokens;
            float* dl = hl ? (float*)(st + total * 4 + 32) : out_logp_old;
            k_queue_rows_out<<<(unsigned)n, 256, 0, q->stream>>>(q->tok, q->lpo, (long long)q->size,
                                                                 q->stride, q->len, q->off, dt, dl);
            RB_CUDA(cudaGetLastError());
            if (ht) RB_CUDA(cudaMemcpyAsync(out_tokens, dt, total * 4, cudaMemcpyDeviceToHost, q->stream));
            if (hl) RB_CUDA(cudaMemcpyAsync(out_logp_old, dl, total * 4, cudaMemcpyDeviceToHost, q->stream));
        }
        if (out_offsets)
            RB_CUDA(cudaMemcpyAsync(out_offsets, q->off, (n + 1) * 8, cudaMemcpyDefault, q->stream));
        RB_CUDA(cudaStreamSynchronize(q->stream));
        q->size -= n;
    });
}

}  // extern "C"
