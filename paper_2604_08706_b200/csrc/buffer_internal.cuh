// buffer_internal.cuh — the HBM-resident ShardedReplayBuffer behind rb_buffer.
//
// Data layout:
//   metadata  SoA columns of N = T*C slots (slot g = shard*C + local slot),
//             replicated on every rank: id, prompt, group, creation_step,
//             policy_version, reward, is_correct, behavior_logprob,
//             advantage (frozen), group_mean (AsymRE baseline), use_count,
//             length;
//   arrival   FIFO: implicit ring, arrival rank i of shard s lives in local
//             slot (head_s + i) % C with head_s = pushes_s % C once full;
//             positive bias: explicit ring order[s*C + (head_s + i) % C];
//   payload   owned shards only: tokens int32[C][stride], logp_old
//             fp32[C][stride], stride = max_tokens rounded up to 4 (16 B rows).
#pragma once

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "stream_copy.cuh"

namespace rb {

struct DevCtl {
    unsigned long long max_id;  // largest rollout id ever pushed
    unsigned long long cursor;  // route cursor (replay_buffer.hpp:105)
    long long err_index;        // first duplicate push of the last insert
    unsigned long long err_id;
    int err_code;  // sticky asynchronous error (RB_EINVAL)
    int has_any;   // max_id valid
    int hash_stale;
    int pb_go;  // k_posbias_batch applies the current insert
    int pad[2];
};

// Positive-bias queue state of one shard: head and count of F, W, Q.
struct PbState {
    int h[3], n[3];
};

// Everything a kernel needs, passed by value.
struct BufView {
    int T, C, stride, retention;
    int sb, se;  // owned shards [sb, se)
    int cs, fs;  // positive bias: correct_slots, fresh_slots (replay_buffer.cpp:110-112)
    int dbg_replay;  // test hook: the sampler replays its draws exactly
    uint64_t *id, *prompt, *group;
    int64_t *cstep, *pver;
    double *reward, *blp, *adv, *gmean;
    uint8_t* correct;
    uint32_t* use;
    int32_t* len;
    int32_t* order;      // [N] positive-bias arrival rings
    int32_t* head;       // [T]
    long long* pushes;   // [T]
    int32_t* owner;      // [N] last writer in the current insert
    int32_t* pbq;        // positive bias: rings F, W, Q per shard [3][T][C+1] (slot | correct<<31)
    struct PbState* pbs; // positive bias: ring heads / counts per shard [T]
    long long* seq;      // positive bias: arrival sequence number per slot [N]
    int32_t* tok;        // owned payload
    float* lpo;
    uint64_t* hkeys;     // present-id set (exact path)
    uint32_t* hstate;
    unsigned long long hcap;
    DevCtl* ctl;
};

// priority_with_replacement weights (rb_set_priority): w = base +
// floor(min(|advantage|, 2^15) * adv_scale) + pos_bonus * [reward > 0].
struct PrioParams {
    uint32_t base, adv_scale, pos_bonus;
};

int loss_grid(int sms);
// priority_with_replacement: enqueue this buffer's per-shard priority mass
// (sum of the record weights of owned shards [sb, se), 0 elsewhere) into
// out[T] (device) on the buffer's stream (buffer.cu).
void prio_mass_launch(struct ::rb_buffer* b, unsigned long long* out);
struct GridCtl;  // buffer.cu: multi-CTA bookkeeping
struct PendingIns {
    int pending;          // 1: the last insert (closed-form FIFO, <= 64 shards) may be running
    int c0, n;            // its cursor % T and (global) record count
    int own;              // owned-metadata insert: its offsets index the owned shard's records only
    int epoch;            // its flag epoch (verdict / done / copy-done carry it)
    const int64_t* toff;  // its payload offsets (the route kernel's copy)
    const unsigned long long* keep_cnt;  // the copy is complete once *keep_cnt >= keep_target
    unsigned long long keep_target;
    long long P[64];      // per-shard push counts before it
};  // loss.cu: resident CTAs of the loss kernels

}  // namespace rb

struct rb_buffer {
    // Every C-ABI call on a buffer holds this lock, as every method of the
    // reference's ShardedReplayBuffer holds its mutex (replay_buffer.cpp:84,
    // 188, 220, 229, 234, 239; replay_buffer.hpp:106-107): concurrent callers
    // see one total order of pushes and samples.  Recursive: entry points
    // call one another (rb_push -> rb_insert).
    std::recursive_mutex mu;
    size_t T = 0, N = 0, C = 0;
    int strategy = 0, retention = 0;
    rb::PrioParams prio{1, 0, 0};  // priority_with_replacement weights
    double delta = 0.0;
    int32_t max_tokens = 0, stride = 0;
    int device = 0;
    size_t sb = 0, se = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    rb::BufView v{};

    // host mirrors (exact; updated when an insert is applied)
    std::vector<long long> h_pushes;
    size_t h_cursor = 0;
    bool async_unchecked = false;  // an RB_INSERT_ASSUME_UNIQUE insert ran since the last sticky check
    // owned metadata (rb_set_owned_metadata): one owned shard keeps the
    // metadata of its own records only; inserts carry only those records
    // (rb_insert_owned, own_n_global = the global batch size during the call)
    bool owned_meta = false;
    size_t own_n_global = 0;

    // scratch (device), grown on demand
    size_t ins_cap = 0;
    int32_t* s_tslot = nullptr;
    uint8_t* s_surv = nullptr;
    uint64_t* s_evid = nullptr;
    rb_record* s_evrec = nullptr;
    double* s_adv = nullptr;
    double* s_gmean = nullptr;
    int32_t* s_len = nullptr;
    int64_t* s_toff = nullptr;
    // staging of host-side insert inputs (device side) and pinned mirrors
    enum { ST_INSERT = 0, ST_SAMPLE, ST_GATHER, ST_IDS, ST_INSPECT, ST_LOSS_IN, ST_LOSS_OUT, ST_OCC, ST_N };
    void* stage_dev[ST_N] = {};
    size_t stage_dev_cap[ST_N] = {};
    void* stage_host = nullptr;
    size_t stage_host_cap = 0;
    cudaEvent_t stage_event = nullptr;  // last async read of stage_host

    // persistent-kernel work units (stream_copy.cuh)
    int unit_grid = 0;                  // SMs * UNIT_CTAS_PER_SM
    int payload_grid = 0, grid_gather = 0, grid_loss = 0;
    rb::GridCtl* route_ctl = nullptr;   // multi-CTA route bookkeeping
    rb::GridCtl* map_ctl = nullptr;     // multi-CTA sampler-map bookkeeping
    int* pay_sync = nullptr;            // [verdict, done] of the last FIFO route (0 = pending;
                                        // verdict 1 valid / 2 rejected), read by the payload copy
                                        // and the fused sampler
    bool pdl = true;                    // programmatic dependent launch of the payload copy
    bool tma_payload = true;            // bulk-copy (TMA) payload kernel (else 128-bit LSU)
    bool pb_par = true;                 // positive bias, unique ids: k_posbias_par (one launch)
    bool route_pdl = true;              // FIFO route as a programmatic dependent of the previous kernel
    int sms = 148;
    int tma_ctas = 3;                   // bulk-copy payload pipelines (single-warp CTAs) per SM
    bool pdl_tail = false;              // the stream's last kernel is the closed-form payload copy
    int ins_epoch = 0;                  // epoch of the last closed-form FIFO insert (pay_sync tags)
    int gather_epoch = 0;               // epoch of the insert pending at the last fused sampler
    rb::PendingIns pend{};              // its insert's plan (for a sampler that overlaps it)
    unsigned long long keep_total = 0;  // route CTAs launched with an offsets copy (host count)
    int seg_used = 0;                   // map CTAs whose early-gather flags are set (to reset)
    // the ring lookahead launched after the last fused sampler (on the Rng's
    // side stream): joined by the next insert / loss / synchronize, or by the
    // next sampler itself
    cudaEvent_t look_ev = nullptr;
    bool look_pending = false;
    bool lookahead = true;              // RB_NO_LOOKAHEAD unset
    long long lookahead_min_draws = 8192;  // side-stream lookahead above this batch
    unsigned long long look_uid = 0, look_seq = 0;  // the lookahead recorded in look_ev
    bool look_captured = false;  // look_ev recorded inside a stream capture
    unsigned long long joined_uid = 0, joined_seq = 0;  // the last one joined on `stream`
    void join_lookahead();
    bool gather_early = false;          // the last kernel on the stream is the fused sampler
    bool early_gather_ok = true;        // RB_NO_EARLY_GATHER unset
    bool loss_dyn = true;               // long rows: claimed loss units (RB_LOSS_CHUNK_MAJOR: static)
    bool tma_long = false;              // RB_PAYLOAD_TMA_LONG: bulk copy for rows > PB_CHT too
    bool chunk_major = true;            // RB_NO_CHUNK_MAJOR unset: long rows, chunk-major units
    void other_work() { pdl_tail = false; gather_early = false; }  // anything else enqueued
    rb::Unit* units_ins = nullptr;      // payload copy units of the last insert
    int* n_units_ins = nullptr;
    size_t units_ins_cap = 0;
    rb::Unit* units_sel = nullptr;      // gather/loss units of the current batch
    int* n_units_sel = nullptr;
    size_t units_sel_cap = 0;
    int32_t* sel_len = nullptr;
    void* loss_partials = nullptr;      // per-CTA loss partials (32 B each)
    size_t loss_partials_bytes = 0;
    // host-buffer loss pipeline: upload / download streams and chunk events
    cudaStream_t cs_in = nullptr, cs_out = nullptr;
    cudaEvent_t ev_io[1 + 2 * 8] = {};  // LOSS_CHUNKS = 8
    // rb_set_async_outputs: a loss with pinned host dlogp returns once its
    // stats are final; the download drains on cs_out beside the next call
    // (an insert's upload runs the other way over PCIe).  out_done marks it.
    bool async_out = false;
    bool out_pending = false;
    cudaEvent_t out_done = nullptr;
    // the same for a gather into pinned host arrays: its download (from the
    // ST_GATHER staging area) drains on cs_out beside the loss's logp_now
    // upload on cs_in; gather_done marks it
    bool gout_pending = false;
    cudaEvent_t gather_ready = nullptr, gather_done = nullptr;
    void wait_outputs_on(cudaStream_t s);  // order s after a pending loss download
    void drain_outputs();                  // host wait for every pending download

    // current batch (selection)
    size_t sel_cap = 0, B = 0;
    int32_t* sel_slot = nullptr;
    int32_t* sel_shard = nullptr;
    int64_t* sel_index = nullptr;
    int64_t* sel_off = nullptr;      // packed offsets over owned selections (B+1)
    long long* sel_total = nullptr;  // [0] local tokens, [1] global tokens
    rb::DevLossAcc* acc = nullptr;
    int last_loss = -1;              // 0 grpo, 1 asymre
    double* red3 = nullptr;          // registered reduce vector (rb_loss_set_reduce_vector)
    bool acc_norm_explicit = false;  // the accumulator holds an explicit GRPO normaliser

    // misc scratch
    void* misc = nullptr;
    size_t misc_cap = 0;

    ~rb_buffer();
    void* scratch(size_t bytes);          // device misc scratch
    void* host_stage(size_t bytes);       // pinned host scratch (waits for its last reader)
    // Small device->host results (totals, offsets, stats, the loss
    // accumulator, the control block) are written by a one-CTA kernel
    // straight into mapped pinned memory: a cudaMemcpy of a few bytes would
    // queue behind a pending multi-MB download on the D2H copy engine
    // (rb_set_async_outputs) and stall the call for a millisecond.
    void* hmap_h = nullptr;
    void* hmap_d = nullptr;
    size_t hmap_cap = 0;
    void fetch(void* host_dst, const void* dev_src, size_t bytes);  // stream-ordered, synchronous
    void to_host_async(void* host_dst, const void* dev_src, size_t bytes);  // pinned dst, no sync
    void host_stage_issued();             // record that the stream reads stage_host
    void host_stage_issued_on(cudaStream_t s);  // ... that stream `s` reads it
    void ensure_copy_streams();
    void grow_loss_partials(size_t bytes);
    void* dev_stage(size_t bytes, int slot);  // device staging areas (one per use)
    void ensure_insert(size_t n);
    void ensure_select(size_t n);
    void sync();
    void sync_checked();  // sync(), then report a sticky error left by an asynchronous insert
};
