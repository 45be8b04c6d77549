// internal.h -- shared internals of the CUDA path (NOT part of the C-ABI).
//
// The oracle never includes this file and this file never includes the oracle's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <string>
#include <deque>
#include <vector>

#include "../../include/ingpu_replay.h"

namespace rpl {

// ---- error reporting -------------------------------------------------------------------
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what);   // records the message, returns RPL_ECUDA
extern std::atomic<uint64_t> g_launches;            // kernels launched by this library

#define RPL_CUDA(call)                                            \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return ::rpl::cuda_fail(_e, #call); \
    } while (0)

#define RPL_LAUNCHED()                                                   \
    do {                                                                 \
        cudaError_t _e = cudaGetLastError();                             \
        if (_e != cudaSuccess) return ::rpl::cuda_fail(_e, "kernel launch"); \
        ::rpl::g_launches.fetch_add(1, std::memory_order_relaxed);        \
    } while (0)

// sticky device-side error bits (written by kernels with atomicOr)
enum : uint32_t { ERRBIT_CORRUPT = 1u, ERRBIT_NUMERIC = 2u, ERRBIT_RANGE = 4u, ERRBIT_PEER = 8u };

// Philox counter word 3 = (TAG << 24) | rank  (reading Q3)
constexpr uint32_t TAG_SAMPLE = 1u;

// ---- the replay ring ---------------------------------------------------------------------
// Device row layout: row stride RS floats (multiple of 32,
// i.e. 128-byte aligned rows):  [ s (D f32) | s' (D f32) | a (i32) | r (f32) | done (u32) | 0 ]
// RPL_U8 rings (byte states, SURVEY config 5): row = [s u8 (D) | s' u8 (D) | pad to 16 B |
// a | r | done | pad], row stride a multiple of 128 B; `so` is the byte offset of a.
struct Ring {
    float *rows = nullptr;     // capacity * rs words
    int host = 0;              // RPL_RING_HOST: rows in pinned, mapped host memory;
                               // RPL_RING_HOST_BATCH (2): pageable host rows, CPU sampler
    int owned = 1;             // 0: rows are the caller's opts.storage (not freed)
    int64_t capacity = 0;
    int32_t D = 0;
    int32_t rs = 0;            // row stride in 4-byte words
    int32_t u8 = 0;            // states stored as bytes
    int32_t so = 0;            // u8 rings: byte offset of the scalars (a, r, done)
    int32_t shared = 0;        // shared states: s' of slot i = s of slot i + 1
    int32_t sw = 0;            // fp32 rings: word offset of the scalars (2D, or D if shared)
};

inline int32_t ring_row_stride(int32_t D, bool shared = false)
{
    return (((shared ? 1 : 2) * D + 3) + 31) / 32 * 32;
}
inline int32_t ring_u8_scalar_offset(int32_t D, bool shared = false)
{
    return ((shared ? 1 : 2) * D + 15) / 16 * 16;
}
inline int32_t ring_u8_row_bytes(int32_t D, bool shared = false)
{
    return (ring_u8_scalar_offset(D, shared) + 12 + 127) / 128 * 128;
}

}  // namespace rpl

struct rpl_replay {
    int device = 0;
    cudaStream_t stream = nullptr;
    rpl::Ring ring;
    int64_t burn_in = 1;
    uint64_t seed = 2;
    uint32_t rank = 0;
    // P:73 update-size queue (update_size > 0): host experiences waiting for their block,
    // SoA like replay_add's inputs
    int64_t qU = 0, qk = 0;
    std::vector<uint8_t> qs, qs2, qdone;
    std::vector<int32_t> qa;
    std::vector<float> qr;
    // host mirror of the ring state (exact: every add is host-initiated with a known k)
    int64_t cursor = 0, size = 0;
    uint64_t total = 0, events = 0, h2d_bytes = 0;
    // pinned host staging + device staging for RPL_HOST adds: one arena (room for two adds of
    // max_host_add experiences) used as a ring of spans, one per add, so the host can run many
    // small adds ahead of the device; a span is reused once its event -- recorded when the
    // device has read it (H2D copy, or the step / insert kernel consuming a zero-copy insert)
    // -- has fired (stage_alloc)
    int64_t max_host_add = 65536;
    char *pinned = nullptr, *dstage = nullptr;
    size_t arena = 0, head = 0;
    struct Span {
        size_t off, len;
        int ev;
    };
    std::deque<Span> live;                 // spans the device may still read
    std::vector<cudaEvent_t> evs;          // event pool (index = Pending::slot)
    std::vector<int> free_evs;
    cudaStream_t copy_stream = nullptr;    // H2D copies of host adds (overlap the work stream)
    cudaEvent_t copy_done = nullptr;
    uint32_t *err_dev = nullptr;   // sticky device error word
    // device control block read by graph-replayed train steps: [0] sampler events consumed,
    // [1] filled size, [2] cursor (kept equal to the host mirror by the kernels that change them)
    uint64_t *ctrl_dev = nullptr;
    // At most one small insert whose ring write is deferred into the next fast train step's
    // K1 (which reads sampled pending slots straight from these sources: "read-through").
    // Any other operation on the replay first flushes it with the insert kernel.  The host
    // mirror (cursor / size / total) already includes it.
    struct Pending {
        int64_t k = 0, cursor = 0, new_size = 0;
        const void *s = nullptr, *s2 = nullptr;   // fp32 (or u8) states
        const float *r = nullptr;
        const int32_t *a = nullptr;
        const uint8_t *done = nullptr;
        int slot = -1;   // zero-copy host add: the pinned staging slot its sources live in
    } pend;
    bool zero_copy = true;   // host adds read by the device from pinned memory (RPL_NO_ZC=1: H2D copy)
    bool no_defer = false;   // RPL_NO_DEFER=1: every insert is an immediate kernel
    bool distinct = false;   // RPL_SAMPLE_DISTINCT (distinct.cuh)
    int32_t *ds_idx = nullptr;   // scratch indices of distinct replay_sample calls
    int64_t ds_cap = 0;
    // RPL_RING_HOST_BATCH (the paper's in-RAM replay): per-step batch staging -- two pinned
    // buffers [rows B x rs words | idx B] used alternately (an event per buffer marks its H2D
    // copy done), and the device batch the step's kernels read
    char *bpin[2] = {nullptr, nullptr};
    cudaEvent_t bev[2] = {nullptr, nullptr};
    int bcur = 0;
    int64_t bcap = 0;          // rows the staging holds
    float *bdev = nullptr;     // device rows [bcap x rs] then idx [bcap]
};

namespace rpl {
// launch helpers implemented in replay.cu, used by dqn.cu
int launch_gather(rpl_replay *rp, int64_t n, const int32_t *idx_dev, uint64_t event,
                  int use_sampler, const rpl_batch *out);
const void *insert_kernel_ptr();
// distinct batch indices of the replay's current event into out[0..B) (distinct.cuh);
// ctrl != null also advances the device event counter
int launch_distinct(const rpl_replay *rp, int B, int32_t *out, uint32_t *err, uint64_t *ctrl,
                    cudaStream_t st);
// experiences the sampler draws from (shared states: all but the newest, reading Q30) and the
// slot of logical position 0 (shared states: the oldest experience; else 0, slot == u)
int64_t sampleable(const rpl_replay *rp);
uint64_t oldest_slot(const rpl_replay *rp);
// the sampling gather of a graph-captured byte-state train step (control block read on device)
int launch_gather_u8_dev(rpl_replay *rp, int64_t n, const rpl_batch *out, cudaStream_t st);
// enqueue the pending deferred insert (if any) as an insert-kernel launch
int replay_flush(rpl_replay *rp);
// the pending insert was enqueued for consumption on `st`: a zero-copy staging slot may be
// reused once the stream passes this point
int replay_consumed(rpl_replay *rp, int slot, cudaStream_t st);
// RPL_RING_HOST_BATCH: sample B indices of event rp->events on the CPU, gather their rows on
// the CPU into pinned staging and enqueue one H2D copy on `st` into the device batch (rows
// at *rows, indices at *idx); the caller advances the event
int host_batch_stage(rpl_replay *rp, int B, cudaStream_t st, const float **rows, const int32_t **idx);
// largest insert that may be deferred into K1 (K1's CTAs write its rows)
constexpr int64_t kMaxDeferredRows = 4096;
}  // namespace rpl
