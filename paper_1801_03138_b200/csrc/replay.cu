// replay.cu -- the device FIFO ring of experiences: insert (replay_add), Philox sample +
// gather + unpack (replay_sample / replay_gather), and the library's error plumbing.
//
// Paper: P:71-75 [Methods] (packed 1,000,000 x 57 Variable, block inserts, uniform integer
// sampling + gather + unpack), P:44 (FIFO, burn-in).  B200 design: DESIGN.md "Kernels".
#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "philox.cuh"
#include "ring_row.cuh"
#include "distinct.cuh"
#include <vector>

namespace rpl {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_err;

void set_error(const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
}

int cuda_fail(cudaError_t e, const char *what)
{
    set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
    return RPL_ECUDA;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------------------------------------
// K1: insert.  One warp per experience; the warp writes the whole 128B-aligned row (one or
// more fully coalesced 128-byte stores per 32 floats).  Slot = (cursor + j) mod capacity.
// ------------------------------------------------------------------------------------------
// One CTA inserts tiles of INS_R (64) consecutive experiences: the tile's SoA sources (contiguous
// runs of s / s' / a / r / done) are read with coalesced loads into shared memory, then the
// packed rows (consecutive slots) leave as 16-byte stores, every warp writing whole 128-byte
// lines -- all loads of a tile in flight at once (P:73 block insert).  Rows wider than
// INS_RS words take one warp per row.
constexpr int INS_R = 64, INS_RS = 64;
__global__ void __launch_bounds__(256) insert_kernel(float *__restrict__ rows, int rs, int D, int sw,
                                                     int64_t capacity, int64_t cursor, int64_t k,
                                                     const float *__restrict__ s,
                                                     const int32_t *__restrict__ a,
                                                     const float *__restrict__ r,
                                                     const float *__restrict__ s2,
                                                     const uint8_t *__restrict__ done,
                                                     uint32_t *err, uint64_t *ctrl, int64_t new_size)
{
    __shared__ __align__(16) float tile[INS_R * INS_RS];
    const int tid = threadIdx.x, lane = tid & 31;
    if (blockIdx.x == 0 && tid == 0) {
        ctrl[1] = (uint64_t)new_size;
        ctrl[2] = (uint64_t)((cursor + k) % capacity);
    }
    if (rs > INS_RS) {
        const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
        for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (tid >> 5); j < k; j += nwarps) {
            int64_t slot = cursor + j;
            if (slot >= capacity) slot -= capacity;   // k <= capacity, cursor < capacity
            ring_write_row(rows + slot * rs, rs, D, sw, lane, j, s, a, r, s2, done, err);
        }
        return;
    }
    const int nq = rs / 4;   // 16-byte pieces per row (rs is a multiple of 32 words)
    for (int64_t j0 = (int64_t)blockIdx.x * INS_R; j0 < k; j0 += (int64_t)gridDim.x * INS_R) {
        const int nr = (int)(k - j0 < INS_R ? k - j0 : INS_R);
        const int ns = nr * D;
        for (int e = tid; e < ns; e += blockDim.x) {
            const int rr = e / D, c = e - rr * D;
            tile[rr * INS_RS + c] = s[j0 * D + e];
            if (sw > D) tile[rr * INS_RS + D + c] = s2[j0 * D + e];
        }
        for (int e = tid; e < nr * (rs - sw); e += blockDim.x) {
            const int rr = e / (rs - sw), c = sw + (e - rr * (rs - sw));
            float v = 0.0f;
            if (c == sw) {
                v = __int_as_float(a[j0 + rr]);
            } else if (c == sw + 1) {
                v = r[j0 + rr];
            } else if (c == sw + 2) {
                uint32_t d = done[j0 + rr];
                if (d > 1u) {   // a device-sourced done > 1 is stored as 1 and flagged
                    atomicOr(err, ERRBIT_CORRUPT);
                    d = 1u;
                }
                v = __uint_as_float(d);
            }
            tile[rr * INS_RS + c] = v;
        }
        __syncthreads();
        for (int e = tid; e < nr * nq; e += blockDim.x) {
            const int rr = e / nq, q = e - rr * nq;
            int64_t slot = cursor + j0 + rr;
            if (slot >= capacity) slot -= capacity;
            *reinterpret_cast<float4 *>(rows + slot * rs + 4 * q) =
                *reinterpret_cast<const float4 *>(tile + rr * INS_RS + 4 * q);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------------
// Shared-state rows (reading Q30): sample over the experiences with a stored successor
// (logical position u -> slot (oldest + u) mod C), the new state from the next slot's row.
// One warp per entry.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gather_shared_kernel(const float *__restrict__ rows, int rs, int D,
                                                            int sw, int64_t capacity, int64_t nvalid,
                                                            uint64_t oldest, int64_t size, int64_t n,
                                                            const int32_t *__restrict__ idx_in,
                                                            uint64_t seed, uint32_t rank, uint64_t event,
                                                            float *s, float *s2, int32_t *a, float *r,
                                                            uint8_t *done, int32_t *idx_out, uint32_t *err,
                                                            uint64_t *ctrl)
{
    if (idx_in == nullptr && ctrl && blockIdx.x == 0 && threadIdx.x == 0) ctrl[0] = event + 1;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < n; e += nwarps) {
        int32_t ix;
        if (idx_in == nullptr) {
            int32_t i0, i1;
            sample_pair(seed, rank, event, (uint32_t)(e >> 1), (uint64_t)nvalid, i0, i1);
            ix = slot_of((e & 1) ? i1 : i0, oldest, capacity);
        } else {
            ix = idx_in[e];
            if (ix < 0 || ix >= size) {
                if (lane == 0) atomicOr(err, ERRBIT_RANGE);
                ix = min(max(ix, 0), (int32_t)size - 1);
            }
        }
        const int64_t nx = (ix + 1) % capacity;
        const float *row = rows + (int64_t)ix * rs, *nrow = rows + nx * rs;
        for (int c = lane; c < D; c += 32) {
            if (s) s[e * D + c] = __ldg(row + c);
            if (s2) s2[e * D + c] = __ldg(nrow + c);
        }
        if (lane == 0) {
            if (idx_out) idx_out[e] = ix;
            if (a) a[e] = __float_as_int(__ldg(row + sw));
            if (r) r[e] = __ldg(row + sw + 1);
            if (done) done[e] = (uint8_t)(__float_as_uint(__ldg(row + sw + 2)) != 0u);
        }
    }
}

// ------------------------------------------------------------------------------------------
// K2+K3: Philox sample (or caller indices) + gather + unpack.  A warp owns groups of 64
// consecutive batch entries: lane l draws entries (2l, 2l+1) with ONE Philox call (call j =
// group/2 + l), then each half-warp gathers one row per iteration with 16-byte loads, 8 rows
// per half-warp in flight, and scatters the fields into the five SoA outputs.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void store_field(int c, float v, int64_t i, int D, float *s,
                                            float *s2, int32_t *a, float *r, uint8_t *done)
{
    if (c < D) {
        if (s) s[i * D + c] = v;
    } else if (c < 2 * D) {
        if (s2) s2[i * D + (c - D)] = v;
    } else if (c == 2 * D) {
        if (a) a[i] = __float_as_int(v);
    } else if (c == 2 * D + 1) {
        if (r) r[i] = v;
    } else if (c == 2 * D + 2) {
        if (done) done[i] = (uint8_t)(__float_as_uint(v) != 0u);
    }
}

template <bool kRow64>
__global__ void __launch_bounds__(256) gather_kernel(const float *__restrict__ rows, int rs, int D,
                                                     int64_t size, int64_t n,
                                                     const int32_t *__restrict__ idx_in,
                                                     uint64_t seed, uint32_t rank, uint64_t event,
                                                     float *s, float *s2, int32_t *a, float *r,
                                                     uint8_t *done, int32_t *idx_out, uint32_t *err,
                                                     uint64_t *ctrl)
{
    if (idx_in == nullptr && ctrl && blockIdx.x == 0 && threadIdx.x == 0) ctrl[0] = event + 1;
    const int lane = threadIdx.x & 31;
    const int half = lane >> 4, p = lane & 15;
    const int64_t ngroups = (n + 63) / 64;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < ngroups;
         g += nwarps) {
        const int64_t base = g * 64;
        int32_t i0, i1;
        const int64_t e0 = base + 2 * lane;
        if (idx_in == nullptr) {
            sample_pair(seed, rank, event, (uint32_t)(g * 32 + lane), (uint64_t)size, i0, i1);
        } else {
            i0 = e0 < n ? idx_in[e0] : 0;
            i1 = e0 + 1 < n ? idx_in[e0 + 1] : 0;
            if (i0 < 0 || i0 >= size || i1 < 0 || i1 >= size) {
                if (e0 < n) atomicOr(err, ERRBIT_RANGE);
                i0 = min(max(i0, 0), (int32_t)size - 1);
                i1 = min(max(i1, 0), (int32_t)size - 1);
            }
        }
        if (idx_out) {
            if (e0 < n) idx_out[e0] = i0;
            if (e0 + 1 < n) idx_out[e0 + 1] = i1;
        }
        if (kRow64) {
#pragma unroll
            for (int u0 = 0; u0 < 32; u0 += 8) {
                float4 v[8];
                int64_t ent[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int32_t iA = __shfl_sync(0xffffffffu, i0, u0 + q);
                    const int32_t iB = __shfl_sync(0xffffffffu, i1, u0 + q);
                    const int32_t row = half ? iB : iA;
                    ent[q] = base + 2 * (u0 + q) + half;
                    if (ent[q] < n)
                        v[q] = __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)row * 64) + p);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (ent[q] < n) {
                        store_field(4 * p + 0, v[q].x, ent[q], D, s, s2, a, r, done);
                        store_field(4 * p + 1, v[q].y, ent[q], D, s, s2, a, r, done);
                        store_field(4 * p + 2, v[q].z, ent[q], D, s, s2, a, r, done);
                        store_field(4 * p + 3, v[q].w, ent[q], D, s, s2, a, r, done);
                    }
                }
            }
        } else {
            for (int u = 0; u < 32; ++u) {
                const int32_t iA = __shfl_sync(0xffffffffu, i0, u);
                const int32_t iB = __shfl_sync(0xffffffffu, i1, u);
                const int32_t row = half ? iB : iA;
                const int64_t ent = base + 2 * u + half;
                if (ent >= n) continue;
                const float4 *src = reinterpret_cast<const float4 *>(rows + (int64_t)row * rs);
                for (int c4 = p; c4 < rs / 4; c4 += 16) {
                    const float4 v = __ldg(src + c4);
                    store_field(4 * c4 + 0, v.x, ent, D, s, s2, a, r, done);
                    store_field(4 * c4 + 1, v.y, ent, D, s, s2, a, r, done);
                    store_field(4 * c4 + 2, v.z, ent, D, s, s2, a, r, done);
                    store_field(4 * c4 + 3, v.w, ent, D, s, s2, a, r, done);
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// Bandwidth-oriented gather for 256-byte rows (D <= 30): a warp owns 32 consecutive entries,
// issues all 32 row loads (16 B per lane, 16 float4 in flight per lane) before using any, stages
// the rows in shared memory, then writes every output tensor as full, coalesced lines (s and s'
// as float4 runs of 32*D floats; a, r, done, idx as 32-wide vectors).
// ------------------------------------------------------------------------------------------
constexpr int GS_W = 8;   // warps per CTA
template <int KD>
__global__ void __launch_bounds__(GS_W * 32) gather_staged_kernel(
    const float *__restrict__ rows, int64_t size, int64_t n, const int32_t *__restrict__ idx_in,
    uint64_t seed, uint32_t rank, uint64_t event, float *s, float *s2, int32_t *a, float *r,
    uint8_t *done, int32_t *idx_out, uint32_t *err, uint64_t *ctrl, int vec_ok)
{
    constexpr int RW = 2 * KD + 3;   // used words of a row: s | s' | a | r | done
    constexpr int SP = RW + 1;       // staging row stride
    extern __shared__ float4 gs_smem[];
    float *st = reinterpret_cast<float *>(gs_smem) + (threadIdx.x >> 5) * 32 * SP;
    if (idx_in == nullptr && ctrl && blockIdx.x == 0 && threadIdx.x == 0) ctrl[0] = event + 1;
    const int lane = threadIdx.x & 31, half = lane >> 4, p = lane & 15;
    const int64_t ngroups = (n + 31) / 32;
    const int64_t nwarps = (int64_t)gridDim.x * GS_W;
    for (int64_t grp = (int64_t)blockIdx.x * GS_W + (threadIdx.x >> 5); grp < ngroups; grp += nwarps) {
        const int64_t base = grp * 32, e = base + lane;
        int32_t ix;
        if (idx_in == nullptr) {
            int32_t i0, i1;
            sample_pair(seed, rank, event, (uint32_t)(e >> 1), (uint64_t)size, i0, i1);
            ix = (lane & 1) ? i1 : i0;
        } else {
            ix = e < n ? idx_in[e] : 0;
            if (ix < 0 || ix >= size) {
                if (e < n) atomicOr(err, ERRBIT_RANGE);
                ix = min(max(ix, 0), (int32_t)size - 1);
            }
        }
        if (idx_out && e < n) idx_out[e] = ix;
        float4 v[16];
#pragma unroll
        for (int it = 0; it < 16; ++it) {
            const int ent = 2 * it + half;
            const int32_t rix = __shfl_sync(0xffffffffu, ix, ent);
            v[it] = (base + ent < n) ? __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)rix * 64) + p)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int it = 0; it < 16; ++it) {
            const int ent = 2 * it + half;
            float *dst = st + ent * SP;
            const float c[4] = {v[it].x, v[it].y, v[it].z, v[it].w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (4 * p + q < RW) dst[4 * p + q] = c[q];
        }
        __syncwarp();
        const int cnt = (int)(n - base < 32 ? n - base : 32);
        if (cnt == 32 && vec_ok) {
            // 32 * KD floats per state tensor, 16-byte aligned (base % 32 == 0)
            float4 *so = reinterpret_cast<float4 *>(s + base * KD);
            float4 *s2o = reinterpret_cast<float4 *>(s2 + base * KD);
            for (int q = lane; q < 8 * KD; q += 32) {
                float w0[4], w1[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int el = 4 * q + k, rr = el / KD, cc = el - rr * KD;
                    w0[k] = st[rr * SP + cc];
                    w1[k] = st[rr * SP + KD + cc];
                }
                if (s) so[q] = make_float4(w0[0], w0[1], w0[2], w0[3]);
                if (s2) s2o[q] = make_float4(w1[0], w1[1], w1[2], w1[3]);
            }
        } else {
            for (int el = lane; el < cnt * KD; el += 32) {
                const int rr = el / KD, cc = el - rr * KD;
                if (s) s[base * KD + el] = st[rr * SP + cc];
                if (s2) s2[base * KD + el] = st[rr * SP + KD + cc];
            }
        }
        if (lane < cnt) {
            const float *row = st + lane * SP + 2 * KD;
            if (a) a[e] = __float_as_int(row[0]);
            if (r) r[e] = row[1];
            if (done) done[e] = (uint8_t)(__float_as_uint(row[2]) != 0u);
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------------------------------
// RPL_U8 rings (Atari-shaped byte states, SURVEY config 5): rows of round_up(2D, 16) + 12
// bytes padded to 128 B.  One CTA per experience: the states move as 16-byte vectors (four
// loads in flight per thread before their stores) when both sides are 16-byte aligned.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void copy_bytes_cta(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src,
                                               int64_t nbytes)
{
    const int tid = threadIdx.x, nt = blockDim.x;
    if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
        const int64_t n16 = nbytes >> 4;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        int64_t i = tid;
        for (; i + 3 * nt < n16; i += 4 * nt) {
            const uint4 v0 = __ldg(s4 + i), v1 = __ldg(s4 + i + nt), v2 = __ldg(s4 + i + 2 * nt),
                        v3 = __ldg(s4 + i + 3 * nt);
            d4[i] = v0;
            d4[i + nt] = v1;
            d4[i + 2 * nt] = v2;
            d4[i + 3 * nt] = v3;
        }
        for (; i < n16; i += nt) d4[i] = __ldg(s4 + i);
        for (int64_t b = (n16 << 4) + tid; b < nbytes; b += nt) dst[b] = src[b];
    } else {
        for (int64_t b = tid; b < nbytes; b += nt) dst[b] = src[b];
    }
}

constexpr int64_t kInsPiece = 4096;   // bytes of a byte-state row per insert CTA

__global__ void __launch_bounds__(256) insert_u8_kernel(uint8_t *__restrict__ rows, int64_t rsb, int so,
                                                        int D, int shared, int64_t capacity, int64_t cursor,
                                                        int64_t k, const uint8_t *__restrict__ s,
                                                        const int32_t *__restrict__ a,
                                                        const float *__restrict__ r,
                                                        const uint8_t *__restrict__ s2,
                                                        const uint8_t *__restrict__ done, uint32_t *err,
                                                        uint64_t *ctrl, int64_t new_size)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctrl[1] = (uint64_t)new_size;
        ctrl[2] = (uint64_t)((cursor + k) % capacity);
    }
    // a row's state bytes (s, then s' unless shared) are cut into kInsPiece-byte pieces, one
    // CTA each: a few ~56 KB Atari rows are spread over many SMs instead of one CTA per row
    const int64_t L = (int64_t)(shared ? 1 : 2) * D;
    const int64_t np = (L + kInsPiece - 1) / kInsPiece;
    for (int64_t w = blockIdx.x; w < k * np; w += gridDim.x) {
        const int64_t j = w / np, q = w % np;
        int64_t slot = cursor + j;
        if (slot >= capacity) slot -= capacity;   // k <= capacity, cursor < capacity
        uint8_t *row = rows + slot * rsb;
        const int64_t b0 = q * kInsPiece, b1 = b0 + kInsPiece < L ? b0 + kInsPiece : L;
        if (b0 < D) copy_bytes_cta(row + b0, s + j * D + b0, (b1 < D ? b1 : D) - b0);
        if (b1 > D) {   // shared: s' is the next row's s (L == D, never taken)
            const int64_t c0 = b0 > D ? b0 : D;
            copy_bytes_cta(row + c0, s2 + j * D + (c0 - D), b1 - c0);
        }
        if (q != np - 1) continue;
        for (int b = (shared ? 1 : 2) * D + threadIdx.x; b < so; b += blockDim.x) row[b] = 0;
        if (threadIdx.x == 0) {
            uint32_t d = done[j];
            if (d > 1u) {   // a device-sourced done > 1 is stored as 1 and flagged
                atomicOr(err, ERRBIT_CORRUPT);
                d = 1u;
            }
            uint32_t *sc = reinterpret_cast<uint32_t *>(row + so);
            sc[0] = (uint32_t)a[j];
            sc[1] = __float_as_uint(r[j]);
            sc[2] = d;
        }
    }
}

// Philox sample (or caller indices) + gather + unpack of byte-state rows: one CTA per entry
__global__ void __launch_bounds__(256) gather_u8_kernel(const uint8_t *__restrict__ rows, int64_t rsb,
                                                        int so, int D, int shared, int64_t capacity,
                                                        uint64_t oldest, int64_t nvalid, int64_t size, int64_t n,
                                                        const int32_t *__restrict__ idx_in,
                                                        uint64_t seed, uint32_t rank, uint64_t event,
                                                        uint8_t *s, uint8_t *s2, int32_t *a, float *r,
                                                        uint8_t *done, int32_t *idx_out, uint32_t *err,
                                                        uint64_t *ctrl, const uint64_t *ctrl_in)
{
    __shared__ int32_t ix_s;
    if (ctrl_in) {   // graph-replayed train steps: event / size / cursor from the control block
        event = ctrl_in[0];
        size = (int64_t)ctrl_in[1];
        nvalid = shared ? size - 1 : size;
        oldest = (shared && size == capacity) ? ctrl_in[2] : 0;
    }
    if (idx_in == nullptr && ctrl && blockIdx.x == 0 && threadIdx.x == 0) ctrl[0] = event + 1;
    for (int64_t e = blockIdx.x; e < n; e += gridDim.x) {
        if (threadIdx.x == 0) {
            int32_t ix;
            if (idx_in == nullptr) {
                int32_t i0, i1;
                sample_pair(seed, rank, event, (uint32_t)(e >> 1), (uint64_t)nvalid, i0, i1);
                ix = slot_of((e & 1) ? i1 : i0, oldest, capacity);
            } else {
                ix = idx_in[e];
                if (ix < 0 || ix >= size) {
                    atomicOr(err, ERRBIT_RANGE);
                    ix = min(max(ix, 0), (int32_t)size - 1);
                }
            }
            ix_s = ix;
            if (idx_out) idx_out[e] = ix;
            const uint32_t *sc = reinterpret_cast<const uint32_t *>(rows + (int64_t)ix * rsb + so);
            if (a) a[e] = (int32_t)__ldg(sc);
            if (r) r[e] = __uint_as_float(__ldg(sc + 1));
            if (done) done[e] = (uint8_t)(__ldg(sc + 2) != 0u);
        }
        __syncthreads();
        const uint8_t *row = rows + (int64_t)ix_s * rsb;
        if (s) copy_bytes_cta(s + e * D, row, D);
        if (s2) copy_bytes_cta(s2 + e * D, shared ? rows + (int64_t)((ix_s + 1) % capacity) * rsb : row + D, D);
        __syncthreads();   // ix_s reuse
    }
}

// host-driven calls (replay_sample / replay_gather path, the generic train step)
// (ctrl != null: the replay_sample path consumes the event: ctrl[0] = event + 1)
__global__ void __launch_bounds__(DS_T, 1) distinct_kernel(uint64_t seed, uint32_t rank, uint64_t event,
                                                           uint64_t n, int B, int32_t *out, uint32_t *err,
                                                           uint64_t *ctrl, uint64_t oldest, int64_t capacity)
{
    extern __shared__ int ds_smem[];
    const int TS = ds_table_slots(B);
    distinct_sample(seed, rank, event, n, B, out, err, ds_smem, ds_smem + TS, oldest, capacity);
    if (ctrl && threadIdx.x == 0) ctrl[0] = event + 1;
}

// launcher for the other translation units (the generic train step)
int launch_distinct(const rpl_replay *rp, int B, int32_t *out, uint32_t *err, uint64_t *ctrl,
                    cudaStream_t st)
{
    static bool attr = false;
    if (!attr) {
        RPL_CUDA(cudaFuncSetAttribute(distinct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)ds_smem_bytes(DS_MAXB)));
        attr = true;
    }
    distinct_kernel<<<1, DS_T, ds_smem_bytes(B), st>>>(rp->seed, rp->rank, rp->events,
                                                       (uint64_t)sampleable(rp), B, out, err, ctrl,
                                                       oldest_slot(rp), rp->ring.capacity);
    RPL_LAUNCHED();
    return RPL_OK;
}

const void *insert_kernel_ptr() { return (const void *)insert_kernel; }

// the sampling gather of a graph-captured byte-state step: event, size and cursor are read
// from the control block on the device, the event is advanced by the step's last kernel
// Byte-state gather with no CTA-wide barrier (states a multiple of 16 bytes): the 2D state
// bytes of a sample ([s | s'], s' from the next slot's row with shared states) are cut into
// GU_PIECE-byte pieces, one CTA task each; every thread draws the sample's index itself
// (one Philox call) and moves GU_V 16-byte vectors with all loads in flight before its
// stores.  Piece 0's thread 0 also writes the index and the scalars.
constexpr int GU_V = 4, GU_T = 256;
constexpr int64_t GU_PIECE = (int64_t)GU_T * GU_V * 16;   // 16 KB
__global__ void __launch_bounds__(GU_T) gather_u8_pieces_kernel(
    const uint8_t *__restrict__ rows, int64_t rsb, int so, int D, int shared, int64_t capacity,
    uint64_t oldest, int64_t nvalid, int64_t size, int64_t n, const int32_t *__restrict__ idx_in,
    uint64_t seed, uint32_t rank, uint64_t event, uint8_t *s, uint8_t *s2, int32_t *a, float *r,
    uint8_t *done, int32_t *idx_out, uint32_t *err, uint64_t *ctrl, const uint64_t *ctrl_in)
{
    if (ctrl_in) {   // graph-replayed train steps: event / size / cursor from the control block
        event = ctrl_in[0];
        size = (int64_t)ctrl_in[1];
        nvalid = shared ? size - 1 : size;
        oldest = (shared && size == capacity) ? ctrl_in[2] : 0;
    }
    if (idx_in == nullptr && ctrl && blockIdx.x == 0 && threadIdx.x == 0) ctrl[0] = event + 1;
    const int64_t L = 2 * (int64_t)D, np = (L + GU_PIECE - 1) / GU_PIECE;
    for (int64_t task = blockIdx.x; task < n * np; task += gridDim.x) {
        const int64_t e = task / np, q = task - e * np;
        // the sample's slot: lane 0 of every warp draws it (one Philox call), a shuffle shares it
        int32_t ix = 0;
        bool bad = false;
        if ((threadIdx.x & 31) == 0) {
            if (idx_in == nullptr) {
                int32_t i0, i1;
                sample_pair(seed, rank, event, (uint32_t)(e >> 1), (uint64_t)nvalid, i0, i1);
                ix = slot_of((e & 1) ? i1 : i0, oldest, capacity);
            } else {
                ix = idx_in[e];
                if (ix < 0 || ix >= size) {
                    bad = true;
                    ix = min(max(ix, 0), (int32_t)size - 1);
                }
            }
        }
        ix = __shfl_sync(0xffffffffu, ix, 0);
        const uint8_t *row = rows + (int64_t)ix * rsb;
        const uint8_t *row2 = shared ? rows + (int64_t)((ix + 1) % capacity) * rsb : row + D;
        uint4 v[GU_V];
        int64_t off[GU_V];
#pragma unroll
        for (int i = 0; i < GU_V; ++i) {
            off[i] = q * GU_PIECE + (int64_t)(i * GU_T + threadIdx.x) * 16;
            if (off[i] < L)
                v[i] = __ldg(reinterpret_cast<const uint4 *>(off[i] < D ? row + off[i] : row2 + (off[i] - D)));
        }
#pragma unroll
        for (int i = 0; i < GU_V; ++i) {
            if (off[i] >= L) continue;
            if (off[i] < D) {
                if (s) *reinterpret_cast<uint4 *>(s + e * D + off[i]) = v[i];
            } else if (s2) {
                *reinterpret_cast<uint4 *>(s2 + e * D + (off[i] - D)) = v[i];
            }
        }
        if (q == 0 && threadIdx.x == 0) {
            if (bad) atomicOr(err, ERRBIT_RANGE);
            if (idx_out) idx_out[e] = ix;
            const uint32_t *sc = reinterpret_cast<const uint32_t *>(row + so);
            if (a) a[e] = (int32_t)__ldg(sc);
            if (r) r[e] = __uint_as_float(__ldg(sc + 1));
            if (done) done[e] = (uint8_t)(__ldg(sc + 2) != 0u);
        }
    }
}

// the byte-state gather for n samples: the piece kernel when states are 16-byte multiples
static void launch_gather_u8_any(const rpl::Ring &R, int dev_sms, uint64_t oldest, int64_t nvalid,
                                 int64_t size, int64_t n, const int32_t *idx_in, uint64_t seed,
                                 uint32_t rank, uint64_t event, const rpl_batch *out, uint32_t *err,
                                 uint64_t *ctrl, const uint64_t *ctrl_in, cudaStream_t st)
{
    const uint8_t *rows = reinterpret_cast<const uint8_t *>(R.rows);
    if (R.D % 16 == 0) {
        const int64_t tasks = n * ((2 * (int64_t)R.D + GU_PIECE - 1) / GU_PIECE);
        int64_t nb = tasks < (int64_t)dev_sms * 8 ? tasks : (int64_t)dev_sms * 8;
        if (nb < 1) nb = 1;
        gather_u8_pieces_kernel<<<(unsigned)nb, GU_T, 0, st>>>(
            rows, (int64_t)R.rs * 4, R.so, R.D, R.shared, R.capacity, oldest, nvalid, size, n, idx_in,
            seed, rank, event, static_cast<uint8_t *>(out->s), static_cast<uint8_t *>(out->s_next),
            out->a, out->r, out->done, out->idx, err, ctrl, ctrl_in);
        return;
    }
    int64_t nb = n < (int64_t)dev_sms * 8 ? n : (int64_t)dev_sms * 8;
    if (nb < 1) nb = 1;
    gather_u8_kernel<<<(unsigned)nb, 256, 0, st>>>(
        rows, (int64_t)R.rs * 4, R.so, R.D, R.shared, R.capacity, oldest, nvalid, size, n, idx_in, seed,
        rank, event, static_cast<uint8_t *>(out->s), static_cast<uint8_t *>(out->s_next), out->a,
        out->r, out->done, out->idx, err, ctrl, ctrl_in);
}

int launch_gather_u8_dev(rpl_replay *rp, int64_t n, const rpl_batch *out, cudaStream_t st)
{
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, rp->device);
    launch_gather_u8_any(rp->ring, dev_sms, 0, 0, 0, n, nullptr, rp->seed, rp->rank, 0, out,
                         rp->err_dev, nullptr, rp->ctrl_dev, st);
    RPL_LAUNCHED();
    return RPL_OK;
}

int64_t sampleable(const rpl_replay *rp)
{
    return rp->ring.shared ? (rp->size > 0 ? rp->size - 1 : 0) : rp->size;
}
uint64_t oldest_slot(const rpl_replay *rp)
{
    return (rp->ring.shared && rp->size == rp->ring.capacity) ? (uint64_t)rp->cursor : 0;
}

int replay_consumed(rpl_replay *rp, int slot, cudaStream_t st)
{
    if (slot >= 0) RPL_CUDA(cudaEventRecord(rp->evs[slot], st));
    return RPL_OK;
}

// the next staging span of `len` bytes (a multiple of 64): wraps to the arena start when the
// tail is too short, and waits for every live span it would overwrite (their events were all
// recorded: an add first flushes the previous deferred insert, which records its span's).
// Every live span is checked, not only the oldest: a span left near the arena's end by an
// earlier wrap can be older than the ones the new span overlaps.
static int stage_alloc(rpl_replay *rp, size_t len, size_t *off, int *ev)
{
    if (rp->head + len > rp->arena) rp->head = 0;
    for (auto it = rp->live.begin(); it != rp->live.end();) {
        if (it->off < rp->head + len && rp->head < it->off + it->len) {
            RPL_CUDA(cudaEventSynchronize(rp->evs[it->ev]));
            rp->free_evs.push_back(it->ev);
            it = rp->live.erase(it);
        } else {
            ++it;
        }
    }
    if (rp->free_evs.empty()) {
        cudaEvent_t e = nullptr;
        RPL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        rp->evs.push_back(e);
        rp->free_evs.push_back((int)rp->evs.size() - 1);
    }
    *ev = rp->free_evs.back();
    rp->free_evs.pop_back();
    *off = rp->head;
    rp->live.push_back({rp->head, len, *ev});
    rp->head += len;
    return RPL_OK;
}

int replay_flush(rpl_replay *rp)
{
    rpl_replay::Pending &q = rp->pend;
    if (q.k == 0) return RPL_OK;
    const int64_t k = q.k;
    q.k = 0;
    const int zslot = q.slot;
    q.slot = -1;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, rp->device);
    int64_t blocks = rp->ring.rs > INS_RS ? (k + 7) / 8 : (k + INS_R - 1) / INS_R;
    if (blocks > (int64_t)dev_sms * 8) blocks = (int64_t)dev_sms * 8;
    if (rp->ring.u8) {
        // one CTA per 4 KB piece of a row (rows are ~56 KB for Atari-shaped states)
        const int64_t pieces = k * (((rp->ring.shared ? 1 : 2) * (int64_t)rp->ring.D + kInsPiece - 1) / kInsPiece);
        const int64_t ublocks = pieces < (int64_t)dev_sms * 16 ? pieces : (int64_t)dev_sms * 16;
        insert_u8_kernel<<<(unsigned)ublocks, 256, 0, rp->stream>>>(
            reinterpret_cast<uint8_t *>(rp->ring.rows), (int64_t)rp->ring.rs * 4, rp->ring.so,
            rp->ring.D, rp->ring.shared, rp->ring.capacity, q.cursor, k, static_cast<const uint8_t *>(q.s), q.a, q.r,
            static_cast<const uint8_t *>(q.s2), q.done, rp->err_dev, rp->ctrl_dev, q.new_size);
    } else {
        insert_kernel<<<(unsigned)blocks, 256, 0, rp->stream>>>(
            rp->ring.rows, rp->ring.rs, rp->ring.D, rp->ring.sw, rp->ring.capacity, q.cursor, k,
            static_cast<const float *>(q.s), q.a, q.r, static_cast<const float *>(q.s2), q.done,
            rp->err_dev, rp->ctrl_dev, q.new_size);
    }
    RPL_LAUNCHED();
    return replay_consumed(rp, zslot, rp->stream);
}

int launch_gather(rpl_replay *rp, int64_t n, const int32_t *idx_dev, uint64_t event,
                  int use_sampler, const rpl_batch *out)
{
    if (int rc = replay_flush(rp)) return rc;
    if (use_sampler && rp->distinct) {
        // distinct sampler (distinct.cuh) into the caller's idx (or scratch), then an
        // explicit-index gather; the sampling kernel consumes the event
        int32_t *buf = out->idx;
        if (!buf) {
            if (rp->ds_cap < n) {
                if (rp->ds_idx) cudaFree(rp->ds_idx);
                rp->ds_idx = nullptr;
                rp->ds_cap = 0;
                RPL_CUDA(cudaMalloc(&rp->ds_idx, (size_t)n * sizeof(int32_t)));
                rp->ds_cap = n;
            }
            buf = rp->ds_idx;
        }
        (void)event;   // == rp->events on this path
        if (int rc = launch_distinct(rp, (int)n, buf, rp->err_dev, rp->ctrl_dev, rp->stream)) return rc;
        idx_dev = buf;
        use_sampler = 0;
    }
    const int64_t groups = (n + 63) / 64;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, rp->device);
    const int64_t warps_per_block = 8;
    int64_t blocks = (groups + warps_per_block - 1) / warps_per_block;
    const int64_t max_blocks = (int64_t)dev_sms * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    const rpl::Ring &R = rp->ring;
    float *os = static_cast<float *>(out->s), *os2 = static_cast<float *>(out->s_next);
    const int64_t nvalid = sampleable(rp);
    const uint64_t oldest = oldest_slot(rp);
    if (R.u8) {
        launch_gather_u8_any(R, dev_sms, oldest, nvalid, rp->size, n, use_sampler ? nullptr : idx_dev,
                             rp->seed, rp->rank, event, out, rp->err_dev, rp->ctrl_dev, nullptr, rp->stream);
    } else if (R.shared) {
        gather_shared_kernel<<<(unsigned)blocks, 256, 0, rp->stream>>>(
            R.rows, R.rs, R.D, R.sw, R.capacity, nvalid, oldest, rp->size, n,
            use_sampler ? nullptr : idx_dev, rp->seed, rp->rank, event, os, os2, out->a, out->r,
            out->done, out->idx, rp->err_dev, rp->ctrl_dev);
    } else if (R.rs == 64 && R.D == 27) {
        // staged, line-coalesced writes (the Melee row: 27-float states)
        constexpr int KD = 27;
        const size_t smem = (size_t)GS_W * 32 * (2 * KD + 4) * sizeof(float);
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(gather_staged_kernel<KD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr_set = true;
        }
        const int64_t g32 = (n + 31) / 32;
        int64_t nb = (g32 + GS_W - 1) / GS_W;
        if (nb > (int64_t)dev_sms * 4) nb = (int64_t)dev_sms * 4;
        if (nb < 1) nb = 1;
        const int vec_ok = ((uintptr_t)out->s % 16 == 0) && ((uintptr_t)out->s_next % 16 == 0);
        gather_staged_kernel<KD><<<(unsigned)nb, GS_W * 32, smem, rp->stream>>>(
            R.rows, rp->size, n, use_sampler ? nullptr : idx_dev, rp->seed, rp->rank, event,
            os, os2, out->a, out->r, out->done, out->idx, rp->err_dev, rp->ctrl_dev, vec_ok);
    } else if (R.rs == 64) {
        gather_kernel<true><<<(unsigned)blocks, 256, 0, rp->stream>>>(
            R.rows, R.rs, R.D, rp->size, n, use_sampler ? nullptr : idx_dev, rp->seed, rp->rank,
            event, os, os2, out->a, out->r, out->done, out->idx, rp->err_dev, rp->ctrl_dev);
    } else {
        gather_kernel<false><<<(unsigned)blocks, 256, 0, rp->stream>>>(
            R.rows, R.rs, R.D, rp->size, n, use_sampler ? nullptr : idx_dev, rp->seed, rp->rank,
            event, os, os2, out->a, out->r, out->done, out->idx, rp->err_dev, rp->ctrl_dev);
    }
    RPL_LAUNCHED();
    return RPL_OK;
}

}  // namespace rpl

using namespace rpl;

// ==========================================================================================
// C-ABI
// ==========================================================================================
extern "C" const char *rpl_last_error(void) { return rpl::t_err.c_str(); }
extern "C" uint64_t rpl_kernel_launches(void) { return rpl::g_launches.load(); }

// bytes of one host-sourced add of k experiences (the SoA inputs, copied once: P:32)
static size_t host_add_bytes(int64_t k, int32_t D, bool u8)
{
    return (size_t)k * (2 * (size_t)D * (u8 ? 1 : 4) + 4 + 4 + 1);
}

extern "C" int replay_ring_bytes(int64_t capacity, int32_t state_dim, const rpl_replay_opts *opts,
                                 size_t *bytes)
{
    if (!bytes || capacity < 1 || capacity >= (int64_t(1) << 31) || state_dim < 1 || state_dim > 1 << 20) {
        set_error("replay_ring_bytes: invalid argument");
        return RPL_EINVAL;
    }
    const bool u8 = opts && opts->state_dtype == RPL_U8;
    const bool sh = opts && opts->state_sharing != 0;
    const int64_t rs = u8 ? ring_u8_row_bytes(state_dim, sh) / 4 : ring_row_stride(state_dim, sh);
    *bytes = (size_t)capacity * rs * sizeof(float);
    return RPL_OK;
}

extern "C" int replay_create(int64_t capacity, int32_t state_dim, const rpl_replay_opts *opts,
                             rpl_replay **out)
{
    if (!out) { set_error("replay_create: out is NULL"); return RPL_EINVAL; }
    *out = nullptr;
    rpl_replay_opts o{};
    o.device = 0; o.cuda_stream = nullptr; o.burn_in = 1; o.seed = 2; o.rank = 0;
    o.max_host_add = 0;
    if (opts) o = *opts;
    if (capacity < 1 || capacity >= (int64_t(1) << 31) || state_dim < 1 || state_dim > 1 << 20 ||
        o.rank >= (1u << 24) || o.burn_in < 1 || o.max_host_add < 0 ||
        (o.state_dtype != RPL_F32 && o.state_dtype != RPL_U8) ||
        (o.sampling != RPL_SAMPLE_UNIFORM && o.sampling != RPL_SAMPLE_DISTINCT) ||
        (o.state_sharing != 0 && o.state_sharing != 1) ||
        (o.ring_memory != RPL_RING_DEVICE && o.ring_memory != RPL_RING_HOST &&
         o.ring_memory != RPL_RING_HOST_BATCH) ||
        (o.ring_memory == RPL_RING_HOST_BATCH && (o.state_dtype != RPL_F32 || o.state_sharing)) ||
        o.update_size < 0 || o.update_size > capacity) {
        set_error("replay_create: invalid argument (capacity=%lld state_dim=%d rank=%u burn_in=%lld)",
                  (long long)capacity, state_dim, o.rank, (long long)o.burn_in);
        return RPL_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || o.device < 0 || o.device >= ndev) {
        set_error("replay_create: no CUDA device %d (count %d)", o.device, ndev);
        return RPL_ECUDA;
    }
    DeviceGuard g(o.device);
    rpl_replay *rp = new rpl_replay();
    rp->device = o.device;
    rp->stream = (cudaStream_t)o.cuda_stream;
    rp->burn_in = o.burn_in;
    rp->seed = o.seed;
    rp->rank = o.rank;
    if (const char *nd = getenv("RPL_NO_DEFER")) rp->no_defer = atoi(nd) != 0;
    if (const char *nz = getenv("RPL_NO_ZC")) rp->zero_copy = atoi(nz) == 0;
    const bool u8 = o.state_dtype == RPL_U8;
    rp->max_host_add = o.max_host_add ? o.max_host_add : 65536;
    // pinned + device staging is two slots of max_host_add experiences: at most 256 MB each
    const int64_t cap_rows = (int64_t)((256ull << 20) / host_add_bytes(1, state_dim, u8));
    if (rp->max_host_add > cap_rows) rp->max_host_add = cap_rows > 0 ? cap_rows : 1;
    if (rp->max_host_add > capacity) rp->max_host_add = capacity;
    if (o.update_size > 0) {
        // P:73 block updates: a block of U is one host add, so staging must hold U
        if (o.update_size > cap_rows) {
            set_error("replay_create: update_size %lld exceeds the %lld-experience staging",
                      (long long)o.update_size, (long long)cap_rows);
            delete rp;
            return RPL_EINVAL;
        }
        if (rp->max_host_add < o.update_size) rp->max_host_add = o.update_size;
        const size_t sb = (size_t)o.update_size * state_dim * (u8 ? 1 : 4);
        rp->qU = o.update_size;
        rp->qs.resize(sb);
        rp->qs2.resize(o.state_sharing ? 0 : sb);
        rp->qa.resize(o.update_size);
        rp->qr.resize(o.update_size);
        rp->qdone.resize(o.update_size);
    }
    rp->ring.capacity = capacity;
    rp->ring.D = state_dim;
    rp->ring.u8 = u8 ? 1 : 0;
    const bool sh = o.state_sharing != 0;
    rp->ring.shared = sh ? 1 : 0;
    rp->ring.rs = u8 ? ring_u8_row_bytes(state_dim, sh) / 4 : ring_row_stride(state_dim, sh);
    rp->ring.so = u8 ? ring_u8_scalar_offset(state_dim, sh) : 0;
    rp->ring.sw = sh ? state_dim : 2 * state_dim;
    if (u8) rp->no_defer = true;   // deferral is a fast-path (fp32 states) feature
    rp->distinct = o.sampling == RPL_SAMPLE_DISTINCT;
    const size_t ring_bytes = (size_t)capacity * rp->ring.rs * sizeof(float);
    rp->ring.host = o.ring_memory == RPL_RING_HOST ? 1 : o.ring_memory == RPL_RING_HOST_BATCH ? 2 : 0;
    if (o.storage) {
        // caller-owned device rows (e.g. a torch tensor): checked, zeroed, never freed here
        cudaPointerAttributes pa{};
        const bool dev_ok = cudaPointerGetAttributes(&pa, o.storage) == cudaSuccess &&
                            pa.type == cudaMemoryTypeDevice && pa.device == o.device;
        cudaGetLastError();
        if (rp->ring.host || o.storage_bytes < ring_bytes || ((uintptr_t)o.storage & 255) != 0 || !dev_ok) {
            set_error("replay_create: opts.storage must be a 256-byte aligned device buffer of >= %zu bytes "
                      "on device %d (got %zu bytes), and RPL_RING_DEVICE", ring_bytes, o.device, o.storage_bytes);
            delete rp;
            return RPL_EINVAL;
        }
        rp->ring.rows = (float *)o.storage;
        rp->ring.owned = 0;
    } else if (rp->ring.host == 2) {
        // the paper's in-RAM replay: ordinary pageable host memory, written and read by the CPU
        void *mem = nullptr;
        if (posix_memalign(&mem, 4096, ring_bytes) != 0) {
            set_error("replay_create: %zu bytes of host ring memory unavailable", ring_bytes);
            delete rp;
            return RPL_ENOMEM;
        }
        rp->ring.rows = (float *)mem;
        std::memset(rp->ring.rows, 0, ring_bytes);
    } else if (rp->ring.host) {
        // in-RAM comparison mode: pinned host rows the kernels address directly (UVA)
        if (cudaHostAlloc(&rp->ring.rows, ring_bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            rp->ring.rows = nullptr;
            set_error("replay_create: cudaHostAlloc of %zu pinned ring bytes failed", ring_bytes);
            delete rp;
            return RPL_ENOMEM;
        }
        std::memset(rp->ring.rows, 0, ring_bytes);
    } else {
        cudaError_t e = cudaMalloc(&rp->ring.rows, ring_bytes);
        if (e != cudaSuccess) {
            size_t fr = 0, tot = 0;
            cudaMemGetInfo(&fr, &tot);
            set_error("replay_create: cudaMalloc of %zu ring bytes failed (%zu free)", ring_bytes, fr);
            rp->ring.rows = nullptr;
            delete rp;
            return RPL_ENOMEM;
        }
    }
    const size_t st = host_add_bytes(rp->max_host_add, state_dim, u8) + 64 * 5;
    rp->arena = 2 * st;
    bool ok = cudaMalloc(&rp->err_dev, sizeof(uint32_t)) == cudaSuccess &&
              cudaMalloc(&rp->ctrl_dev, 3 * sizeof(uint64_t)) == cudaSuccess &&
              cudaMemsetAsync(rp->ctrl_dev, 0, 3 * sizeof(uint64_t), rp->stream) == cudaSuccess &&
              cudaHostAlloc((void **)&rp->pinned, rp->arena, cudaHostAllocDefault) == cudaSuccess &&
              cudaMalloc((void **)&rp->dstage, rp->arena) == cudaSuccess &&
              cudaStreamCreateWithFlags(&rp->copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&rp->copy_done, cudaEventDisableTiming) == cudaSuccess;
    if (!ok || cudaMemsetAsync(rp->err_dev, 0, sizeof(uint32_t), rp->stream) != cudaSuccess ||
        (!rp->ring.host && cudaMemsetAsync(rp->ring.rows, 0, ring_bytes, rp->stream) != cudaSuccess)) {
        set_error("replay_create: staging allocation of %zu bytes failed", st);
        replay_destroy(rp);
        return RPL_ENOMEM;
    }
    *out = rp;
    return RPL_OK;
}

extern "C" int replay_destroy(rpl_replay *rp)
{
    if (!rp) return RPL_OK;
    DeviceGuard g(rp->device);
    rp->pend.k = 0;   // a never-consumed deferred insert is dropped with the ring
    rp->pend.slot = -1;
    cudaStreamSynchronize(rp->stream);
    for (cudaEvent_t ev : rp->evs) cudaEventDestroy(ev);
    if (rp->copy_stream) {
        cudaStreamSynchronize(rp->copy_stream);
        cudaStreamDestroy(rp->copy_stream);
    }
    if (rp->copy_done) cudaEventDestroy(rp->copy_done);
    if (rp->pinned) cudaFreeHost(rp->pinned);
    if (rp->dstage) cudaFree(rp->dstage);
    if (rp->err_dev) cudaFree(rp->err_dev);
    if (rp->ctrl_dev) cudaFree(rp->ctrl_dev);
    if (rp->ds_idx) cudaFree(rp->ds_idx);
    for (int i = 0; i < 2; ++i) {
        if (rp->bev[i]) cudaEventDestroy(rp->bev[i]);
        if (rp->bpin[i]) cudaFreeHost(rp->bpin[i]);
    }
    if (rp->bdev) cudaFree(rp->bdev);
    if (rp->ring.rows && rp->ring.owned) {
        if (rp->ring.host == 2) free(rp->ring.rows);
        else if (rp->ring.host) cudaFreeHost(rp->ring.rows);
        else cudaFree(rp->ring.rows);
    }
    delete rp;
    return RPL_OK;
}

static int add_rows(rpl_replay *rp, int64_t k, const void *s, const int32_t *a, const float *r,
                    const void *s_next, const uint8_t *done, int mem);

extern "C" int replay_add(rpl_replay *rp, int64_t k, const void *s, const int32_t *a,
                          const float *r, const void *s_next, const uint8_t *done, int mem)
{
    if (!rp) { set_error("replay_add: null handle"); return RPL_EINVAL; }
    if (rp->qU == 0) return add_rows(rp, k, s, a, r, s_next, done, mem);
    // P:73 block updates: append to the host queue; every U queued experiences are one insert
    if (mem != RPL_HOST) {
        set_error("replay_add: update_size > 0 queues host experiences only (mem=%d)", mem);
        return RPL_EINVAL;
    }
    if (k < 0 || k > rp->ring.capacity) {
        set_error("replay_add: invalid k=%lld (capacity %lld)", (long long)k, (long long)rp->ring.capacity);
        return RPL_EINVAL;
    }
    if (k == 0) return RPL_OK;
    if (!s || !a || !r || (!s_next && !rp->ring.shared) || !done) {
        set_error("replay_add: null input pointer");
        return RPL_EINVAL;
    }
    for (int64_t j = 0; j < k; ++j)
        if (done[j] > 1) {
            set_error("replay_add: done[%lld]=%u not in {0,1}", (long long)j, done[j]);
            return RPL_ECORRUPT;
        }
    const size_t es = (size_t)rp->ring.D * (rp->ring.u8 ? 1 : 4);   // bytes of one state
    int64_t j = 0;
    while (j < k) {
        const int64_t m = std::min(k - j, rp->qU - rp->qk);
        std::memcpy(rp->qs.data() + rp->qk * es, (const char *)s + j * es, m * es);
        if (!rp->ring.shared) std::memcpy(rp->qs2.data() + rp->qk * es, (const char *)s_next + j * es, m * es);
        std::memcpy(rp->qa.data() + rp->qk, a + j, m * 4);
        std::memcpy(rp->qr.data() + rp->qk, r + j, m * 4);
        std::memcpy(rp->qdone.data() + rp->qk, done + j, m);
        rp->qk += m;
        j += m;
        if (rp->qk == rp->qU) {
            if (int rc = add_rows(rp, rp->qU, rp->qs.data(), rp->qa.data(), rp->qr.data(),
                                  rp->ring.shared ? nullptr : rp->qs2.data(), rp->qdone.data(), RPL_HOST))
                return rc;
            rp->qk = 0;
        }
    }
    return RPL_OK;
}

extern "C" int replay_flush_queue(rpl_replay *rp, int64_t *flushed)
{
    if (!rp) return RPL_EINVAL;
    const int64_t k = rp->qk;
    if (flushed) *flushed = k;
    if (k == 0) return RPL_OK;
    if (int rc = add_rows(rp, k, rp->qs.data(), rp->qa.data(), rp->qr.data(),
                          rp->ring.shared ? nullptr : rp->qs2.data(), rp->qdone.data(), RPL_HOST))
        return rc;
    rp->qk = 0;
    return RPL_OK;
}

extern "C" int replay_queued(const rpl_replay *rp, int64_t *queued)
{
    if (!rp || !queued) return RPL_EINVAL;
    *queued = rp->qk;
    return RPL_OK;
}

// RPL_RING_HOST_BATCH insert: the CPU writes the rows of the host ring (the paper's in-RAM
// replay keeps its experiences in RAM; no transfer until a batch is sampled)
static int host_ring_add(rpl_replay *rp, int64_t k, const float *s, const int32_t *a, const float *r,
                         const float *s_next, const uint8_t *done, int mem)
{
    if (mem != RPL_HOST) {
        set_error("replay_add: an RPL_RING_HOST_BATCH replay takes host inputs only (mem=%d)", mem);
        return RPL_EINVAL;
    }
    for (int64_t j = 0; j < k; ++j)
        if (done[j] > 1) {
            set_error("replay_add: done[%lld]=%u not in {0,1}", (long long)j, done[j]);
            return RPL_ECORRUPT;
        }
    const int32_t D = rp->ring.D, rs = rp->ring.rs;
    for (int64_t j = 0; j < k; ++j) {
        float *row = rp->ring.rows + ((rp->cursor + j) % rp->ring.capacity) * rs;
        std::memcpy(row, s + j * D, (size_t)D * 4);
        std::memcpy(row + D, s_next + j * D, (size_t)D * 4);
        const uint32_t dn = done[j];
        std::memcpy(row + 2 * D, a + j, 4);
        std::memcpy(row + 2 * D + 1, r + j, 4);
        std::memcpy(row + 2 * D + 2, &dn, 4);
    }
    rp->cursor = (rp->cursor + k) % rp->ring.capacity;
    rp->size = std::min<int64_t>(rp->size + k, rp->ring.capacity);
    rp->total += (uint64_t)k;
    return RPL_OK;
}

// the CPU sampler of RPL_RING_HOST_BATCH: the device sampler's Philox stream (Q3)
// (distinct sampling, reading Q29 -- the paper's in-RAM `random.sample`: the first B distinct
// values of the same uniform stream, in stream order; needs size >= B, checked by the callers)
static void host_sample(const rpl_replay *rp, int B, uint64_t event, int32_t *idx)
{
    const uint64_t n = (uint64_t)rp->size;
    if (!rp->distinct) {
        for (int i = 0; i < B; i += 2) {
            int32_t i0, i1;
            sample_pair(rp->seed, rp->rank, event, (uint32_t)(i / 2), n, i0, i1);
            idx[i] = i0;
            if (i + 1 < B) idx[i + 1] = i1;
        }
        return;
    }
    // an open-addressing set (power-of-two table of 4B slots, linear probing; -1 = empty)
    static thread_local std::vector<int32_t> table;
    size_t cap = 16;
    while (cap < (size_t)4 * B) cap <<= 1;
    table.assign(cap, -1);
    const size_t mask = cap - 1;
    int got = 0;
    for (uint32_t j = 0; got < B; ++j) {   // stream positions 2j, 2j + 1
        int32_t v[2];
        sample_pair(rp->seed, rp->rank, event, j, n, v[0], v[1]);
        for (int h = 0; h < 2 && got < B; ++h) {
            size_t t = ((uint32_t)v[h] * 2654435761u) & mask;
            while (table[t] != -1 && table[t] != v[h]) t = (t + 1) & mask;
            if (table[t] == -1) {
                table[t] = v[h];
                idx[got++] = v[h];
            }
        }
    }
}

// grow the batch staging to B rows (waits for the copies in flight)
static int host_batch_reserve(rpl_replay *rp, int64_t B)
{
    if (B <= rp->bcap) return RPL_OK;
    const size_t rowb = (size_t)rp->ring.rs * 4, bytes = (size_t)B * (rowb + 4);
    for (int i = 0; i < 2; ++i) {
        if (rp->bev[i]) RPL_CUDA(cudaEventSynchronize(rp->bev[i]));
        if (rp->bpin[i]) cudaFreeHost(rp->bpin[i]);
        rp->bpin[i] = nullptr;
        if (!rp->bev[i]) RPL_CUDA(cudaEventCreateWithFlags(&rp->bev[i], cudaEventDisableTiming));
    }
    if (rp->bdev) {
        RPL_CUDA(cudaDeviceSynchronize());
        cudaFree(rp->bdev);
        rp->bdev = nullptr;
    }
    rp->bcap = 0;
    for (int i = 0; i < 2; ++i)
        if (cudaHostAlloc((void **)&rp->bpin[i], bytes, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            set_error("in-RAM batch staging: %zu pinned bytes unavailable", bytes);
            return RPL_ENOMEM;
        }
    if (cudaMalloc((void **)&rp->bdev, bytes) != cudaSuccess) {
        cudaGetLastError();
        set_error("in-RAM batch staging: %zu device bytes unavailable", bytes);
        return RPL_ENOMEM;
    }
    rp->bcap = B;
    return RPL_OK;
}

namespace rpl {
int host_batch_stage(rpl_replay *rp, int B, cudaStream_t st, const float **rows, const int32_t **idx)
{
    DeviceGuard g(rp->device);
    if (int rc = host_batch_reserve(rp, B)) return rc;
    const int c = rp->bcur;
    rp->bcur ^= 1;
    RPL_CUDA(cudaEventSynchronize(rp->bev[c]));   // the copy that last read this buffer is done
    const size_t rowb = (size_t)rp->ring.rs * 4;
    char *pin = rp->bpin[c];
    int32_t *pidx = reinterpret_cast<int32_t *>(pin + (size_t)B * rowb);
    host_sample(rp, B, rp->events, pidx);
    for (int i = 0; i < B; ++i)
        std::memcpy(pin + (size_t)i * rowb, rp->ring.rows + (int64_t)pidx[i] * rp->ring.rs, rowb);
    // one transfer: the rows then the indices, packed at the front of the device batch
    char *dst = reinterpret_cast<char *>(rp->bdev);
    RPL_CUDA(cudaMemcpyAsync(dst, pin, (size_t)B * (rowb + 4), cudaMemcpyHostToDevice, st));
    RPL_CUDA(cudaEventRecord(rp->bev[c], st));
    rp->h2d_bytes += (uint64_t)B * (rowb + 4);
    *rows = rp->bdev;
    *idx = reinterpret_cast<const int32_t *>(dst + (size_t)B * rowb);
    return RPL_OK;
}
}  // namespace rpl

static int add_rows(rpl_replay *rp, int64_t k, const void *s, const int32_t *a, const float *r,
                    const void *s_next, const uint8_t *done, int mem)
{
    const int32_t D = rp->ring.D;
    if (k < 0 || k > rp->ring.capacity ||
        (mem != RPL_HOST && mem != RPL_DEVICE && mem != RPL_DEVICE_DEFER)) {
        set_error("replay_add: invalid k=%lld (capacity %lld) or mem=%d", (long long)k,
                  (long long)rp->ring.capacity, mem);
        return RPL_EINVAL;
    }
    if (k == 0) return RPL_OK;
    if (!s || !a || !r || (!s_next && !rp->ring.shared) || !done) {
        set_error("replay_add: null input pointer");
        return RPL_EINVAL;
    }
    if (rp->ring.host == 2) return host_ring_add(rp, k, (const float *)s, a, r, (const float *)s_next, done, mem);
    DeviceGuard g(rp->device);
    if (int rc = replay_flush(rp)) return rc;   // inserts stay in call order
    const void *ds = s, *ds2 = nullptr;
    if (mem != RPL_HOST) ds2 = s_next;
    const float *dr = r;
    int zslot = -1;
    const int32_t *da = a;
    const uint8_t *dd = done;
    bool direct = false;   // host inputs already in pinned memory: the insert kernel reads them
    if (mem == RPL_HOST && k > kMaxDeferredRows) {
        // large host blocks from pinned (page-locked, device-mapped) memory: no staging copy --
        // the insert kernel reads the caller's arrays across PCIe once, and the call returns
        // after it (the caller may reuse its buffers, as for any RPL_HOST add)
        const void *ps[5] = {s, a, r, rp->ring.shared ? s : s_next, done};
        const void *pd[5] = {};
        direct = true;
        for (int i = 0; i < 5 && direct; ++i) {
            cudaPointerAttributes at{};
            direct = cudaPointerGetAttributes(&at, ps[i]) == cudaSuccess &&
                     at.type == cudaMemoryTypeHost && at.devicePointer != nullptr;
            if (direct) pd[i] = at.devicePointer;
        }
        cudaGetLastError();
        if (direct) {
            for (int64_t j = 0; j < k; ++j)
                if (done[j] > 1) {
                    set_error("replay_add: done[%lld]=%u not in {0,1}", (long long)j, done[j]);
                    return RPL_ECORRUPT;
                }
            ds = pd[0];
            da = (const int32_t *)pd[1];
            dr = (const float *)pd[2];
            ds2 = rp->ring.shared ? nullptr : pd[3];
            dd = (const uint8_t *)pd[4];
            const size_t bs = (size_t)k * D * (rp->ring.u8 ? 1 : sizeof(float));
            rp->h2d_bytes += bs * (rp->ring.shared ? 1 : 2) + (size_t)k * 9;
        }
    }
    if (mem == RPL_HOST && !direct) {
        if (k > rp->max_host_add) {
            set_error("replay_add: k=%lld exceeds max_host_add=%lld", (long long)k,
                      (long long)rp->max_host_add);
            return RPL_EINVAL;
        }
        for (int64_t j = 0; j < k; ++j)
            if (done[j] > 1) {
                set_error("replay_add: done[%lld]=%u not in {0,1}", (long long)j, done[j]);
                return RPL_ECORRUPT;
            }
        // [r | a | s | s' | done], each section 64-byte aligned, in the next span of the arena
        const size_t bs = (size_t)k * D * (rp->ring.u8 ? 1 : sizeof(float));
        auto up = [](size_t x) { return (x + 63) & ~(size_t)63; };
        const size_t len = up((size_t)k * 4) * 2 + up(bs) * (rp->ring.shared ? 1 : 2) + up((size_t)k);
        size_t base = 0;
        int slot = -1;
        if (int rc = stage_alloc(rp, len, &base, &slot)) return rc;
        char *hp = rp->pinned + base;
        char *dp = rp->dstage + base;
        size_t off = 0, bytes = 0;
        memcpy(hp + off, r, (size_t)k * 4); dr = (const float *)(dp + off); off += up((size_t)k * 4);
        memcpy(hp + off, a, (size_t)k * 4); da = (const int32_t *)(dp + off); off += up((size_t)k * 4);
        memcpy(hp + off, s, bs); ds = dp + off; off += up(bs);
        bytes = (size_t)k * 8 + bs;
        if (!rp->ring.shared) {   // shared states: one state per experience crosses PCIe
            memcpy(hp + off, s_next, bs); ds2 = dp + off; off += up(bs);
            bytes += bs;
        }
        memcpy(hp + off, done, (size_t)k); dd = (const uint8_t *)(dp + off); off += up((size_t)k);
        bytes += (size_t)k;
        rp->h2d_bytes += bytes;
        if (rp->zero_copy && !rp->ring.u8 && !rp->no_defer && k <= kMaxDeferredRows) {
            // zero-copy: the deferred insert's sources are the pinned slot itself -- the
            // device reads them over PCIe (once, for the ring write) when it consumes the
            // insert, so no copy op enters the stream; the slot's event is recorded then
            const char *dev0 = dp;
            auto host_of = [&](const void *d) { return (const void *)(hp + ((const char *)d - dev0)); };
            ds = host_of(ds);
            if (ds2) ds2 = host_of(ds2);
            dr = (const float *)host_of(dr);
            da = (const int32_t *)host_of(da);
            dd = (const uint8_t *)host_of(dd);
            zslot = slot;
        } else if (rp->copy_stream) {
            // the H2D copy runs on the replay's copy stream, overlapping whatever the work
            // stream is doing (typically the previous train step); the work stream waits for
            // it before the insert reads the span, and the span's event is recorded once that
            // consumer has run (its region is then free for a later add's copy)
            RPL_CUDA(cudaMemcpyAsync(dp, hp, off, cudaMemcpyHostToDevice, rp->copy_stream));
            RPL_CUDA(cudaEventRecord(rp->copy_done, rp->copy_stream));
            RPL_CUDA(cudaStreamWaitEvent(rp->stream, rp->copy_done, 0));
            zslot = slot;
        } else {
            RPL_CUDA(cudaMemcpyAsync(dp, hp, off, cudaMemcpyHostToDevice, rp->stream));
            RPL_CUDA(cudaEventRecord(rp->evs[slot], rp->stream));
        }
    }
    const int64_t new_size = rp->size + k < rp->ring.capacity ? rp->size + k : rp->ring.capacity;
    // Defer the ring write of a small insert into the next fast train step (its K1 reads
    // sampled pending slots from the sources and writes the rows).  RPL_DEVICE inputs are
    // only deferred on request (RPL_DEVICE_DEFER): the caller must keep them unchanged.
    rpl_replay::Pending &q = rp->pend;
    q.cursor = rp->cursor;
    q.new_size = new_size;
    q.s = ds;
    q.s2 = ds2;
    q.r = dr;
    q.a = da;
    q.done = dd;
    q.slot = zslot;
    q.k = k;
    if (mem == RPL_DEVICE || k > kMaxDeferredRows || rp->no_defer) {
        if (int rc = replay_flush(rp)) return rc;
    }
    if (direct) RPL_CUDA(cudaStreamSynchronize(rp->stream));   // the caller's pinned arrays are read
    rp->cursor = (rp->cursor + k) % rp->ring.capacity;
    rp->size = new_size;
    rp->total += (uint64_t)k;
    return RPL_OK;
}

extern "C" int replay_sample(rpl_replay *rp, int32_t batch, const rpl_batch *out)
{
    if (!rp || !out || batch < 1) {
        set_error("replay_sample: invalid argument (batch=%d)", batch);
        return RPL_EINVAL;
    }
    if (rp->distinct && batch > DS_MAXB) {
        set_error("replay_sample: distinct batch %d > %d", batch, DS_MAXB);
        return RPL_EINVAL;
    }
    const int64_t nvalid = sampleable(rp);
    if (rp->size < rp->burn_in || nvalid < 1 || (rp->distinct && nvalid < batch)) return RPL_NOT_READY;
    DeviceGuard g(rp->device);
    if (rp->ring.host == 2) {
        // in-RAM replay: CPU sample + CPU unpack into pinned staging, then the batch tensors
        // cross PCIe (the paper's feed of sampled batches)
        const int32_t D = rp->ring.D, rs = rp->ring.rs;
        if (int rc = host_batch_reserve(rp, (int64_t)batch * 2)) return rc;
        const int c = rp->bcur;
        rp->bcur ^= 1;
        RPL_CUDA(cudaEventSynchronize(rp->bev[c]));
        char *pin = rp->bpin[c];
        float *ps = reinterpret_cast<float *>(pin), *ps2 = ps + (size_t)batch * D;
        int32_t *pa = reinterpret_cast<int32_t *>(ps2 + (size_t)batch * D);
        float *pr = reinterpret_cast<float *>(pa + batch);
        int32_t *pidx = reinterpret_cast<int32_t *>(pr + batch);
        uint8_t *pd = reinterpret_cast<uint8_t *>(pidx + batch);
        host_sample(rp, batch, rp->events, pidx);
        for (int i = 0; i < batch; ++i) {
            const float *row = rp->ring.rows + (int64_t)pidx[i] * rs;
            std::memcpy(ps + (size_t)i * D, row, (size_t)D * 4);
            std::memcpy(ps2 + (size_t)i * D, row + D, (size_t)D * 4);
            std::memcpy(pa + i, row + 2 * D, 4);
            std::memcpy(pr + i, row + 2 * D + 1, 4);
            uint32_t dn;
            std::memcpy(&dn, row + 2 * D + 2, 4);
            pd[i] = (uint8_t)(dn != 0u);
        }
        const size_t sb = (size_t)batch * D * 4;
        RPL_CUDA(cudaMemcpyAsync(out->s, ps, sb, cudaMemcpyHostToDevice, rp->stream));
        RPL_CUDA(cudaMemcpyAsync(out->s_next, ps2, sb, cudaMemcpyHostToDevice, rp->stream));
        RPL_CUDA(cudaMemcpyAsync(out->a, pa, (size_t)batch * 4, cudaMemcpyHostToDevice, rp->stream));
        RPL_CUDA(cudaMemcpyAsync(out->r, pr, (size_t)batch * 4, cudaMemcpyHostToDevice, rp->stream));
        RPL_CUDA(cudaMemcpyAsync(out->done, pd, (size_t)batch, cudaMemcpyHostToDevice, rp->stream));
        if (out->idx) RPL_CUDA(cudaMemcpyAsync(out->idx, pidx, (size_t)batch * 4, cudaMemcpyHostToDevice, rp->stream));
        RPL_CUDA(cudaEventRecord(rp->bev[c], rp->stream));
        rp->h2d_bytes += 2 * sb + (size_t)batch * 9;
        rp->events += 1;
        return RPL_OK;
    }
    int rc = launch_gather(rp, batch, nullptr, rp->events, 1, out);
    if (rc != RPL_OK) return rc;
    rp->events += 1;
    return RPL_OK;
}

extern "C" int replay_gather(rpl_replay *rp, int64_t n, const int32_t *idx_dev,
                             const rpl_batch *out)
{
    if (!rp || !out || n < 0 || (n > 0 && !idx_dev)) {
        set_error("replay_gather: invalid argument");
        return RPL_EINVAL;
    }
    if (n == 0) return RPL_OK;
    if (rp->size < 1) {
        set_error("replay_gather: empty replay");
        return RPL_ESTATE;
    }
    if (rp->ring.host == 2) {
        set_error("replay_gather: device-index gathers need device-addressable rows (not RPL_RING_HOST_BATCH)");
        return RPL_ESTATE;
    }
    DeviceGuard g(rp->device);
    return launch_gather(rp, n, idx_dev, 0, 0, out);
}

extern "C" int rpl_time_adds(rpl_replay *rp, int64_t n_calls, int64_t k, const void *s, const int32_t *a,
                             const float *r, const void *s_next, const uint8_t *done, int mem, double *seconds)
{
    if (!rp || n_calls < 0 || !seconds) return RPL_EINVAL;
    const auto t0 = std::chrono::steady_clock::now();
    for (int64_t i = 0; i < n_calls; ++i)
        if (int rc = replay_add(rp, k, s, a, r, s_next, done, mem)) return rc;
    if (int rc = replay_flush(rp)) return rc;
    DeviceGuard g(rp->device);
    RPL_CUDA(cudaStreamSynchronize(rp->stream));
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return RPL_OK;
}

extern "C" int replay_size(const rpl_replay *rp, int64_t *size)
{
    if (!rp || !size) return RPL_EINVAL;
    *size = rp->size;
    return RPL_OK;
}

extern "C" int replay_state(const rpl_replay *rp, int64_t *cursor, int64_t *size,
                            uint64_t *total, uint64_t *events, uint64_t *h2d_bytes)
{
    if (!rp) return RPL_EINVAL;
    if (cursor) *cursor = rp->cursor;
    if (size) *size = rp->size;
    if (total) *total = rp->total;
    if (events) *events = rp->events;
    if (h2d_bytes) *h2d_bytes = rp->h2d_bytes;
    return RPL_OK;
}
