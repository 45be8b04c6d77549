// ring_row.cuh -- the one definition of a packed ring row write (CUDA path only), shared by
// the insert kernel (replay.cu) and the deferred insert that K3 of the fast train step
// performs (train_fast.cuh: rows loaded into registers at K3's start, stored at its end).  Row layout: [s (D) | s' (D) | a (i32 bits) |
// r | done (u32 bits) | zero pad], rs words, or [s | a | r | done | pad] with shared states.
// experience j goes to slot (cursor + j) mod capacity.

// sampler slot of logical position u: the uniform stream draws u over the n sampleable
// experiences; with shared states the newest is excluded and u counts from the oldest
__device__ __forceinline__ int32_t slot_of(int32_t u, uint64_t oldest, int64_t capacity)
{
    const uint64_t s = oldest + (uint64_t)u;   // u < capacity and oldest < capacity
    return (int32_t)(s >= (uint64_t)capacity ? s - (uint64_t)capacity : s);
}
#pragma once
#include <stdint.h>

#include "internal.h"

namespace rpl {

// warp-cooperative: lane c writes words c, c + 32, ... of experience j's row.  sw = first
// scalar word: 2D, or D for shared-state rows [s | a | r | done] (no s' stored)
__device__ __forceinline__ void ring_write_row(float *row, int rs, int D, int sw, int lane, int64_t j,
                                               const float *__restrict__ s,
                                               const int32_t *__restrict__ a,
                                               const float *__restrict__ r,
                                               const float *__restrict__ s2,
                                               const uint8_t *__restrict__ done, uint32_t *err)
{
    for (int c = lane; c < rs; c += 32) {
        float v = 0.0f;
        if (c < D) {
            v = s[j * D + c];
        } else if (c < sw) {
            v = s2[j * D + (c - D)];
        } else if (c == sw) {
            v = __int_as_float(a[j]);
        } else if (c == sw + 1) {
            v = r[j];
        } else if (c == sw + 2) {
            uint32_t d = done[j];
            if (d > 1u) {   // a device-sourced done > 1 is stored as 1 and flagged
                atomicOr(err, ERRBIT_CORRUPT);
                d = 1u;
            }
            v = __uint_as_float(d);
        }
        row[c] = v;
    }
}

// the same row in two halves: every word of a row of <= 32 RW_PRE words into registers first
// (all loads in flight at once: one round trip, e.g. over PCIe for a zero-copy source) ...
constexpr int RW_PRE = 4;
__device__ __forceinline__ void ring_load_row(float v[RW_PRE], int rs, int D, int sw, int lane, int64_t j,
                                              const float *__restrict__ s, const int32_t *__restrict__ a,
                                              const float *__restrict__ r, const float *__restrict__ s2,
                                              const uint8_t *__restrict__ done, uint32_t *err)
{
#pragma unroll
    for (int q = 0; q < RW_PRE; ++q) {
        const int c = lane + 32 * q;
        float x = 0.0f;
        if (c < rs) {
            if (c < D) {
                x = s[j * D + c];
            } else if (c < sw) {
                x = s2[j * D + (c - D)];
            } else if (c == sw) {
                x = __int_as_float(a[j]);
            } else if (c == sw + 1) {
                x = r[j];
            } else if (c == sw + 2) {
                uint32_t d = done[j];
                if (d > 1u) {
                    atomicOr(err, ERRBIT_CORRUPT);
                    d = 1u;
                }
                x = __uint_as_float(d);
            }
        }
        v[q] = x;
    }
}
// ... and stored later
__device__ __forceinline__ void ring_store_row(float *row, const float v[RW_PRE], int rs, int lane)
{
#pragma unroll
    for (int q = 0; q < RW_PRE; ++q)
        if (lane + 32 * q < rs) row[lane + 32 * q] = v[q];
}

}  // namespace rpl
