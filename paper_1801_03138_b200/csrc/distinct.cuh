// distinct.cuh -- distinct-index sampling ("I plan on switching back to sampling distinct
// integers once TensorFlow has an efficient way to do so").  CUDA path only.
//
// Definition (reading Q29): the batch is the first B DISTINCT values of the same
// Philox index stream the uniform sampler uses (stream position t = sample_pair call t/2, word
// t % 2), in stream order -- identical to the uniform batch whenever that has no repeat.
//
// One CTA walks the stream in chunks of its thread count: every candidate is inserted into an
// open-addressing table in shared memory that keeps, per distinct value, the smallest stream
// position (atomicMin: independent of the order the threads get there), a candidate is a
// first occurrence iff its position is the one kept, and a block-wide prefix count of the
// first occurrences in stream order gives each its batch slot.  Stops once B are found.
#pragma once
#include <stdint.h>

#include "philox.cuh"
#include "ring_row.cuh"

namespace rpl {

constexpr int DS_T = 1024;   // threads of the sampling CTA (stream positions per chunk)
constexpr int DS_MAXB = 7168;  // largest distinct batch (its table fits in shared memory)

// table slots for batch B: a power of two >= 2 (B + DS_T)
__host__ __device__ inline int ds_table_slots(int B)
{
    int ts = 1024;
    while (ts < 2 * (B + DS_T)) ts <<= 1;
    return ts;
}
__host__ inline size_t ds_smem_bytes(int B) { return (size_t)ds_table_slots(B) * 8; }

// out[i] = slot_of(i-th distinct logical position, oldest, capacity) (identity for a plain
// ring: oldest = 0)
__device__ inline void distinct_sample(uint64_t seed, uint32_t rank, uint64_t event, uint64_t n,
                                       int B, int32_t *out, uint32_t *err, int *keys, int *pos,
                                       uint64_t oldest, int64_t capacity)
{
    __shared__ int wsum[DS_T / 32];
    __shared__ int s_total;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int TS = ds_table_slots(B);
    int lg = 0;
    while ((1 << lg) < TS) ++lg;
    for (int i = tid; i < TS; i += DS_T) {
        keys[i] = -1;
        pos[i] = 0x7FFFFFFF;
    }
    __syncthreads();
    int count = 0;
    // a stream longer than this means n < B (excluded by the callers) -- flag, don't spin
    const int64_t limit = (int64_t)64 * (B + DS_T);
    for (int64_t t0 = 0; count < B; t0 += DS_T) {
        if (t0 > limit) {
            if (tid == 0 && err) atomicOr(err, 4u);   // ERRBIT_RANGE
            break;
        }
        const int64_t t = t0 + tid;
        int32_t i0, i1;
        sample_pair(seed, rank, event, (uint32_t)(t >> 1), n, i0, i1);
        const int32_t v = (t & 1) ? i1 : i0;
        uint32_t h = ((uint32_t)v * 0x9E3779B1u) >> (32 - lg);
        while (true) {
            const int k = atomicCAS(&keys[h], -1, v);
            if (k == -1 || k == v) break;
            h = (h + 1) & (uint32_t)(TS - 1);
        }
        atomicMin(&pos[h], (int)t);
        __syncthreads();
        const bool first = pos[h] == (int)t;
        // exclusive prefix count of first occurrences in stream (= thread) order
        const unsigned bal = __ballot_sync(0xFFFFFFFFu, first);
        const int excl_w = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            int x = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            wsum[lane] = x;   // inclusive
            if (lane == 31) s_total = x;
        }
        __syncthreads();
        const int excl = (warp ? wsum[warp - 1] : 0) + excl_w;
        if (first && count + excl < B) out[count + excl] = slot_of(v, oldest, capacity);
        count += s_total;
        __syncthreads();   // wsum / s_total reuse
    }
}

}  // namespace rpl
