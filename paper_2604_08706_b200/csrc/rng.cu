// rng.cu — replab::Rng (rng.hpp:22-69, rng.cpp) reproduced bit-exactly.
//
// The MT19937-64 state has one authoritative home at a time: the GPU while
// the sampler consumes it (the hot path never copies it back), the host when
// a caller asks for a host-side draw (test code that interleaves
// rng.uniform01() with buffer.sample(), as the reference's own tests do).
// Migration is a 2.5 KB copy on the owning stream.  On the device the state
// lives in a ring of twisted blocks (MtRing); a sampler that consumed a
// large batch forks the next call's block twisting onto a side stream
// (k_ring_lookahead, one warp with the block in registers), and every later
// user of the ring joins it first (join / to_device / to_host).
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <string>

#include "common.cuh"
#include "rng_internal.cuh"

namespace rb {

static thread_local std::string g_err;
void set_last_error(const std::string& msg) { g_err = msg; }

void require_device() {
    static int ok = -1;
    if (ok < 0) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        ok = (e == cudaSuccess && n > 0) ? 1 : 0;
        if (ok) {
            int dev = 0, major = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
            if (major < 10) ok = 2;
        }
    }
    if (ok == 0) throw Error(RB_ECUDA, "libreplay_b200: no CUDA device available (no CPU fallback)");
    if (ok == 2) throw Error(RB_ECUDA, "libreplay_b200: built for sm_100a; device is older");
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// rng.cpp:8-15
uint64_t hash_name(const char* name) {
    uint64_t h = 1469598103934665603ULL;
    for (const unsigned char* c = (const unsigned char*)name; *c; ++c) {
        h ^= *c;
        h *= 1099511628211ULL;
    }
    return h;
}
// rng.cpp:17-23
static uint64_t splitmix64(uint64_t& state) {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

}  // namespace rb

using namespace rb;

static void mt_seed(MtState& s, uint64_t seed) {  // [rand.predef] seeding
    s.mt[0] = seed;
    for (int i = 1; i < MT_N; ++i) s.mt[i] = 6364136223846793005ULL * (s.mt[i - 1] ^ (s.mt[i - 1] >> 62)) + i;
    s.idx = MT_N;  // libstdc++ twists lazily on the first draw
    s.pad = 0;
    s.draws = 0;
}

static std::atomic<unsigned long long> g_rng_uid{1};
rb_rng::rb_rng(uint64_t seed_) : seed(seed_) {
    mt_seed(host, seed_);
    where = 0;
    uid = g_rng_uid.fetch_add(1);
}
rb_rng::~rb_rng() {
    wait_lookahead();
    if (gen_fork) cudaEventDestroy(gen_fork);
    if (gen_done) cudaEventDestroy(gen_done);
    if (gen_stream) cudaStreamDestroy(gen_stream);
    if (done) {
        // an event last recorded inside a stream capture cannot be waited on
        if (cudaEventSynchronize(done) != cudaSuccess) cudaDeviceSynchronize();
        cudaEventDestroy(done);
    }
    if (dev) cudaFree(dev);
    cudaGetLastError();  // destructors report nothing: leave no error behind
}

void rb_rng::wait_lookahead() {
    if (!gen_pending) return;
    if (cudaEventSynchronize(gen_done) != cudaSuccess) {  // recorded inside a capture
        cudaGetLastError();
        cudaDeviceSynchronize();
    }
    gen_pending = false;
}
void rb_rng::join(cudaStream_t s) {
    if (!gen_pending) return;
    // a lookahead launched outside any capture and already complete needs no
    // wait (and a capture must not wait on uncaptured work)
    if (!gen_captured && cudaEventQuery(gen_done) == cudaSuccess) {
        gen_pending = false;
        return;
    }
    RB_CUDA(cudaStreamWaitEvent(s, gen_done, 0));
    gen_pending = false;
}

void rb_rng::to_host() {
    wait_lookahead();
    if (where == 0) return;
    if (done && cudaEventSynchronize(done) != cudaSuccess) {
        // last recorded inside a stream capture: wait for the device instead
        cudaGetLastError();
        RB_CUDA(cudaDeviceSynchronize());
    }
    MtRingHead h;
    static_assert(offsetof(MtRing, blk) == sizeof(MtRingHead), "MtRing header layout");
    RB_CUDA(cudaMemcpy(&h, dev, sizeof h, cudaMemcpyDeviceToHost));
    RB_CUDA(cudaMemcpy(host.mt, dev->blk[h.q_state % MT_KR], sizeof host.mt,
                       cudaMemcpyDeviceToHost));
    host.idx = h.idx;
    host.draws = h.draws;
    where = 0;
}

MtRing* rb_rng::to_device(cudaStream_t s) {
    require_device();
    if (!dev) {
        RB_CUDA(cudaMalloc(&dev, sizeof(MtRing)));
        RB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        RB_CUDA(cudaGetDevice(&device));
    }
    if (where == 0) {
        // the previous device user (and any lookahead) must be finished
        // before we overwrite; the host state becomes ring block 0
        wait_lookahead();
        if (cudaEventSynchronize(done) != cudaSuccess) {
            cudaGetLastError();
            RB_CUDA(cudaDeviceSynchronize());
        }
        MtRingHead h;
        h.q_state = 0;
        h.q_hi = 0;
        h.idx = host.idx;
        h.pad = 0;
        h.draws = host.draws;
        h.gen_q = 0;
        RB_CUDA(cudaMemcpyAsync(dev, &h, sizeof h, cudaMemcpyHostToDevice, s));
        RB_CUDA(cudaMemcpyAsync(dev->blk[0], host.mt, sizeof host.mt, cudaMemcpyHostToDevice, s));
        // host copies must stay alive until the copies complete
        RB_CUDA(cudaStreamSynchronize(s));
    } else if (gen_pending) {
        // a lookahead still extends the ring: order after it (and so after
        // the previous user, which it follows)
        join(s);
    } else if (s != last_stream) {
        // order after the previous user of the device state on another stream
        // (same-stream users are ordered already; skipping the wait keeps the
        // sampler capturable in CUDA graphs)
        RB_CUDA(cudaStreamWaitEvent(s, done, 0));
    }
    where = 1;
    return dev;
}

void rb_rng::used_on(cudaStream_t s) {
    RB_CUDA(cudaEventRecord(done, s));
    last_stream = s;
}

uint64_t rb_rng::next() {
    to_host();
    return mt_next_scalar(host.mt, &host.idx, &host.draws);
}

// ---- device bulk generator (parity aid for the sampler's stream) -------
// Ring lookahead (one warp, blocks in registers): extend the ring so the next
// call of `draws` draws finds its blocks twisted: (q_hi, need + 1], capped by
// the ring's capacity from the current block.
__global__ void __launch_bounds__(32) k_ring_lookahead(MtRing* r, unsigned long long draws) {
    const int l = threadIdx.x;
    const long long q0 = r->q_state, qhi = r->q_hi;
    const long long need = q0 + (long long)((r->idx + draws + MT_N - 1) / MT_N);
    long long target = need + 1;
    if (target > q0 + MT_KR - 1) target = q0 + MT_KR - 1;
    if (target <= qhi) return;
    uint64_t w[10];
    const uint64_t* src = r->blk[qhi % MT_KR];
#pragma unroll
    for (int k = 0; k < 10; ++k) w[k] = (l + 32 * k < MT_N) ? src[l + 32 * k] : 0;
    for (long long q = qhi + 1; q <= target; ++q) {
        mt_twist_warp(w);
        uint64_t* dst = r->blk[q % MT_KR];
#pragma unroll
        for (int k = 0; k < 10; ++k)
            if (l + 32 * k < MT_N) dst[l + 32 * k] = w[k];
    }
    __syncwarp();
    if (l == 0) r->q_hi = target;  // the joiners see it after this kernel completes
}

void rb_rng::launch_lookahead(cudaStream_t s, unsigned long long draws) {
    if (!dev) return;
    if (!gen_stream) {
        RB_CUDA(cudaStreamCreateWithFlags(&gen_stream, cudaStreamNonBlocking));
        RB_CUDA(cudaEventCreateWithFlags(&gen_fork, cudaEventDisableTiming));
        RB_CUDA(cudaEventCreateWithFlags(&gen_done, cudaEventDisableTiming));
    }
    join(s);  // at most one lookahead in flight
    RB_CUDA(cudaEventRecord(gen_fork, s));
    RB_CUDA(cudaStreamWaitEvent(gen_stream, gen_fork, 0));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    RB_CUDA(cudaStreamIsCapturing(s, &cs));
    gen_captured = cs != cudaStreamCaptureStatusNone;
    k_ring_lookahead<<<1, 32, 0, gen_stream>>>(dev, draws);
    RB_CUDA(cudaGetLastError());
    RB_CUDA(cudaEventRecord(gen_done, gen_stream));
    gen_pending = true;
    ++gen_seq;
}

__global__ void __launch_bounds__(320) k_mt_fill(MtRing* r, uint64_t n, uint64_t* out) {
    __shared__ uint64_t mt[MT_N];
    const long long q0 = r->q_state;
    uint32_t idx = r->idx;
    const uint64_t draws = r->draws;
    ring_load_block(r, q0, mt);
    uint64_t pos = 0;
    long long tw = 0;
    while (pos < n) {
        if (idx >= MT_N) {
            mt_twist_block(mt);
            idx = 0;
            ++tw;
        }
        const uint64_t avail = (uint64_t)(MT_N - idx);
        const uint64_t take = avail < n - pos ? avail : n - pos;
        if (threadIdx.x < take) out[pos + threadIdx.x] = mt_temper(mt[idx + threadIdx.x]);
        idx += (uint32_t)take;
        pos += take;
    }
    ring_store_state(r, mt, q0, tw, idx, draws + n);
}

extern "C" {

const char* rb_last_error(void) { return rb::g_err.c_str(); }

uint64_t rb_hash_name(const char* name) { return hash_name(name); }

int rb_rng_create(uint64_t seed, rb_rng** out) {
    return guard([&] { *out = new rb_rng(seed); });
}

int rb_rng_stream(const rb_rng* p, const char* name, rb_rng** out) {
    return guard([&] {  // rng.cpp:27-30
        uint64_t state = p->seed ^ hash_name(name);
        *out = new rb_rng(splitmix64(state));
    });
}

int rb_rng_stream_index(const rb_rng* p, const char* name, uint64_t index, rb_rng** out) {
    return guard([&] {  // rng.cpp:32-36
        uint64_t state = p->seed ^ hash_name(name);
        state = splitmix64(state) ^ (index * 0x9e3779b97f4a7c15ULL);
        *out = new rb_rng(splitmix64(state));
    });
}

int rb_rng_clone(const rb_rng* r, rb_rng** out) {
    return guard([&] {
        rb_rng* c = new rb_rng(r->seed);
        const_cast<rb_rng*>(r)->to_host();
        c->host = r->host;
        *out = c;
    });
}

void rb_rng_destroy(rb_rng* r) { delete r; }

uint64_t rb_rng_seed(const rb_rng* r) { return r->seed; }

uint64_t rb_rng_draws(const rb_rng* r) {
    const_cast<rb_rng*>(r)->to_host();
    return r->host.draws;
}

int rb_rng_next_u64(rb_rng* r, uint64_t* out) {
    return guard([&] { *out = r->next(); });
}

int rb_rng_below(rb_rng* r, uint64_t bound, uint64_t* out) {
    return guard([&] {  // rng.cpp:40-51
        if (bound == 0) invalid("Rng::below: bound must be positive");
        const uint64_t limit = below_limit(bound);
        uint64_t v;
        do {
            v = r->next();
        } while (v >= limit);
        *out = v % bound;
    });
}

int rb_rng_uniform01(rb_rng* r, double* out) {
    return guard([&] { *out = static_cast<double>(r->next() >> 11) * 0x1.0p-53; });
}

int rb_rng_normal(rb_rng* r, double* out) {
    return guard([&] {  // rng.cpp:59-70
        for (;;) {
            const double u = 2.0 * (static_cast<double>(r->next() >> 11) * 0x1.0p-53) - 1.0;
            const double v = 2.0 * (static_cast<double>(r->next() >> 11) * 0x1.0p-53) - 1.0;
            const double s = u * u + v * v;
            if (s > 0.0 && s < 1.0) {
                *out = u * std::sqrt(-2.0 * std::log(s) / s);
                return;
            }
        }
    });
}

int rb_rng_sample_without_replacement(rb_rng* r, uint64_t n, uint64_t k, uint64_t* out) {
    return guard([&] {  // rng.cpp:108-121
        if (k > n) invalid("Rng::sample_without_replacement: k exceeds population");
        std::vector<uint64_t> idx(n);
        for (uint64_t i = 0; i < n; ++i) idx[i] = i;
        for (uint64_t i = 0; i < k; ++i) {
            const uint64_t bound = n - i, limit = below_limit(bound);
            uint64_t v;
            do {
                v = r->next();
            } while (v >= limit);
            std::swap(idx[i], idx[i + v % bound]);
        }
        std::memcpy(out, idx.data(), k * sizeof(uint64_t));
    });
}

int rb_rng_get_state(rb_rng* r, uint64_t* mt312, uint32_t* idx, uint64_t* draws) {
    return guard([&] {
        r->to_host();
        if (mt312) std::memcpy(mt312, r->host.mt, sizeof r->host.mt);
        if (idx) *idx = r->host.idx;
        if (draws) *draws = r->host.draws;
    });
}

int rb_rng_set_state(rb_rng* r, const uint64_t* mt312, uint32_t idx, uint64_t draws) {
    return guard([&] {
        if (!mt312 || idx > (uint32_t)MT_N) invalid("rb_rng_set_state: bad state");
        r->to_host();  // the device ring (if any) is superseded
        std::memcpy(r->host.mt, mt312, sizeof r->host.mt);
        r->host.idx = idx;
        r->host.draws = draws;
    });
}

int rb_rng_fill_u64(rb_rng* r, uint64_t n, uint64_t* out) {
    return guard([&] {
        require_device();
        cudaStream_t s = 0;  // legacy default stream
        MtRing* st = r->to_device(s);
        uint64_t* d = out;
        const bool dev_out = is_device_ptr(out);
        if (!dev_out) RB_CUDA(cudaMallocAsync((void**)&d, n * sizeof(uint64_t) + 8, s));
        k_mt_fill<<<1, 320, 0, s>>>(st, n, d);
        RB_CUDA(cudaGetLastError());
        r->used_on(s);
        if (!dev_out) {
            RB_CUDA(cudaMemcpyAsync(out, d, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
            RB_CUDA(cudaFreeAsync(d, s));
            RB_CUDA(cudaStreamSynchronize(s));
        }
    });
}

}  // extern "C"
