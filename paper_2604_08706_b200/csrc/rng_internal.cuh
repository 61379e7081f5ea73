// rng_internal.cuh — the rb_rng object behind the C handle.
#pragma once

#include <vector>

#include "common.cuh"

struct rb_rng {
    explicit rb_rng(uint64_t seed);
    ~rb_rng();
    rb_rng(const rb_rng&) = delete;
    rb_rng& operator=(const rb_rng&) = delete;

    // Make the host copy authoritative (synchronises the owning stream).
    void to_host();
    // Make the device ring authoritative for kernels on stream `s`; the
    // caller enqueues its kernels and then calls used_on(s).
    rb::MtRing* to_device(cudaStream_t s);
    void used_on(cudaStream_t s);  // record completion of the last device use
    uint64_t next();               // host draw (rng.cpp:38)
    // Ring lookahead: after a sampler on stream `s` consumed the ring, twist
    // the next call's blocks (assuming `draws` draws) on a side stream, so
    // the serial MT chain runs beside the rest of the step instead of inside
    // the sampler.  The next device user joins it (join / to_device).
    void launch_lookahead(cudaStream_t s, unsigned long long draws);
    void join(cudaStream_t s);     // order stream s after a pending lookahead
    void wait_lookahead();         // host-side wait (to_host, destruction)

    uint64_t seed;
    rb::MtState host{};
    rb::MtRing* dev = nullptr;
    int where = 0;                   // 0 = host authoritative, 1 = device authoritative
    cudaEvent_t done = nullptr;      // completes after the last kernel that used `dev`
    cudaStream_t last_stream = nullptr;  // stream of that kernel (compared, never used)
    int device = -1;
    cudaStream_t gen_stream = nullptr;   // lookahead stream (non-blocking)
    cudaEvent_t gen_fork = nullptr, gen_done = nullptr;
    bool gen_pending = false;            // a lookahead not yet joined by a device user
    bool gen_captured = false;           // that lookahead was launched inside a stream capture
    unsigned long long gen_seq = 0;      // lookaheads launched (pairs with the joiner's record)
    unsigned long long uid = 0;          // process-unique id (buffers remember who they joined)
};

namespace rb {
uint64_t hash_name(const char* name);
}
