// dp_peer.cuh -- data-parallel gradient mean + SGD over peer memory (P:144
// "synchronized every train step").  CUDA path only.
//
// Every rank exports one exchange buffer (cudaIpc): two gradient slots [2][P + 1] (slot t % 2
// holds step t's gradient, loss in word P) and a flag word.  After its step's gradient is
// complete, rank r's dp_peer_sgd_kernel publishes flag_r = t (release, system scope), waits until
// every rank's flag reaches t (acquire), then every CTA reads its slice of all ranks' gradients
// straight from their memory over NVLink, forms the mean in rank order (identical arithmetic on
// every rank: replicas stay bit-identical), applies SGD / the target copy and writes the mean
// (the API's RPL_GRAD).  Reuse of a slot two steps later is safe: a rank only passes step
// t + 1's flag wait once every rank has started step t + 1, i.e. finished reading step t - 1.
//
// The same kernel emulates `nloc` ranks in one cooperative launch on one device (rank groups
// of blocks, all buffers local): the multi-rank protocol is testable without more GPUs.
#pragma once
#include <stdint.h>

#include "internal.h"

namespace rpl {

constexpr int DP_MAXR = 8;                  // ranks of one node
constexpr int64_t kDpRsMin = 1 << 20;      // gradients longer than this use the reduce-scatter kernel
constexpr int kDpRsWorld = 4;              // ... and so does every gradient from this many ranks up
constexpr int DP_U = 8;                    // elements per thread and round (loads in flight)
// all-read moves (world - 1) x P words into each rank per step, reduce-scatter about 2 x P plus
// a second handshake: from 4 ranks up (C2 at 8 GPUs: 3.9 MB vs 1.1 MB per rank) the bytes win
inline bool dp_use_rs(int64_t P, int world) { return P + 1 > kDpRsMin || world >= kDpRsWorld; }

struct DPArgs {
    int nloc, world, rank0;              // ranks run by this launch: rank0 .. rank0 + nloc - 1
    int64_t P;                           // parameters (the gradient slot holds P + 1 words)
    unsigned long long t;                // step number (> 0), parity selects the slot
    float lr;
    const float *xbuf[DP_MAXR];          // rank q's exchange buffer (peer-mapped or local)
    unsigned long long *flag[DP_MAXR];   // rank q's flag word
    float *online[DP_MAXR], *target[DP_MAXR], *gmean[DP_MAXR];   // per local rank
    const int32_t *sync_flag[DP_MAXR];
    uint32_t *err[DP_MAXR];
    float *loss_out[DP_MAXR];            // the mean loss for the caller (or null), per local rank
    // byte-state learners (wide.cuh): W0's bf16 planes, rewritten by the SGD for the W0 entries,
    // so the next step needs no re-split (.bf null: no planes); local rank 0 only
    struct { uint16_t *bf; int64_t n, pe; int D, planes; } w0;
};

// W0's bf16 planes of a byte-state learner ([online, target][planes][pe], null: none): the first
// n = N0 * D blob words are W0 [N0][D]
struct W0Planes {
    uint16_t *bf;
    int64_t n, pe;
    int D, planes;
};
// the SGD of blob word i (the new weight w) into W0's bf16 planes, when i is a W0 entry
__device__ __forceinline__ void dp_w0_planes(const W0Planes &q, int64_t i, float w, int do_sync)
{
    if (!q.bf || i >= q.n) return;
    const int ii = (int)i, u = ii / q.D, k = ii - u * q.D;
    const int64_t t = wd_tix_k(u, k);
    uint16_t h, m, l;
    umma::split3_bf16(w, h, m, l);
    uint16_t *pl = q.bf;
    for (int net = 0; net < (do_sync ? 2 : 1); ++net, pl += 3 * q.pe) {
        pl[t] = h;
        if (q.planes > 1) pl[q.pe + t] = m;
        if (q.planes > 2) pl[2 * q.pe + t] = l;
    }
}
// the same for the float4 group j (blob words 4j .. 4j + 3): with D % 4 == 0 the four words are
// consecutive inputs of one unit row, i.e. 8 bytes of one core-matrix row per plane
__device__ __forceinline__ void dp_w0_planes4(const W0Planes &q, int64_t j, float4 w, int do_sync)
{
    if (!q.bf || 4 * j >= q.n) return;
    if ((q.D & 3) != 0) {
        dp_w0_planes(q, 4 * j, w.x, do_sync);
        dp_w0_planes(q, 4 * j + 1, w.y, do_sync);
        dp_w0_planes(q, 4 * j + 2, w.z, do_sync);
        dp_w0_planes(q, 4 * j + 3, w.w, do_sync);
        return;
    }
    const int ii = (int)(4 * j), u = ii / q.D, k = ii - u * q.D;
    const int64_t t = wd_tix_k(u, k);
    uint2 h, m, l;
    umma::split3_pack2(w.x, w.y, h.x, m.x, l.x);
    umma::split3_pack2(w.z, w.w, h.y, m.y, l.y);
    uint16_t *pl = q.bf;
    for (int net = 0; net < (do_sync ? 2 : 1); ++net, pl += 3 * q.pe) {
        *reinterpret_cast<uint2 *>(pl + t) = h;
        if (q.planes > 1) *reinterpret_cast<uint2 *>(pl + q.pe + t) = m;
        if (q.planes > 2) *reinterpret_cast<uint2 *>(pl + 2 * q.pe + t) = l;
    }
}


// exchange buffer: [2][S] gradient slots, [S] mean (reduce-scatter variant; S = P + 1 rounded to
// 16 bytes: dp_slot_stride), then a
// 256-byte flag area: flag (u64) at +0, broken (u32) at +64, flag2 (u64) at +128, a block
// counter (u32) at +192
// slot stride: P + 1 words rounded up to 16 bytes, so a step can write its gradient straight
// into its slot with the same vector stores it uses for the learner's own gradient buffer
__host__ __device__ inline int64_t dp_slot_stride(int64_t P) { return (P + 1 + 3) & ~(int64_t)3; }
__host__ __device__ inline size_t dp_flag_offset(int64_t P) { return ((size_t)3 * dp_slot_stride(P) * sizeof(float) + 255) / 256 * 256; }
__host__ __device__ inline size_t dp_xbuf_bytes(int64_t P) { return dp_flag_offset(P) + 256; }
__host__ __device__ inline unsigned long long *dp_flag_of(const float *xbuf, int64_t P)
{
    return (unsigned long long *)((char *)xbuf + dp_flag_offset(P));
}

// host: make `dev` current for a scope
struct DeviceGuardDqn {
    int prev = -1;
    explicit DeviceGuardDqn(int dev)
    {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuardDqn()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

__device__ __forceinline__ unsigned long long dp_ld_acquire(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void dp_st_release(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned *dp_broken_of(unsigned long long *flag) { return reinterpret_cast<unsigned *>(flag + 8); }
__device__ __forceinline__ bool dp_is_broken(unsigned long long *flag)
{
    return *reinterpret_cast<volatile unsigned *>(dp_broken_of(flag)) != 0;
}

// thread 0: wait until every rank's flag word (at word offset `which` of its flag area) reaches
// t (the own rank's only for `own`: its step-t gradient precedes the kernel in stream order).
// Fails -- returns true, marks this rank's exchange broken and raises ERRBIT_PEER -- when this
// rank's exchange is already broken, when a peer's is (a broken rank stops publishing, so every
// rank of the group fails at the same step instead of averaging a frozen replica's gradient),
// or after ~10 s without the flag.
__device__ inline bool dp_wait_all(const DPArgs &a, int rank, int rl, int which, bool own)
{
    bool failed = dp_is_broken(a.flag[rank]);
    const long long t0 = clock64();
    for (int q = 0; q < a.world && !failed; ++q) {
        if (q == rank && !own) continue;
        while (dp_ld_acquire(a.flag[q] + which) < a.t) {
            if (dp_is_broken(a.flag[q]) || clock64() - t0 > 20000000000ll) {
                failed = true;
                break;
            }
        }
    }
    if (failed) {
        atomicExch(dp_broken_of(a.flag[rank]), 1u);
        atomicOr(a.err[rl], ERRBIT_PEER);
    }
    return failed;
}

// Reduce-scatter variant for large P (config 5's 15 MB gradient): rank r averages only its
// 1/world of the P + 1 words, reading them from every rank, and stores the mean into every
// rank's mean buffer; its last block to finish publishes flag2; after every rank's flag2 each
// rank applies SGD from its own mean buffer.  Each rank moves ~2 P words over NVLink instead of
// world x P.  Cooperative launch: a rank's blocks wait for its own last block.  The mean buffer
// needs no second slot: rank r writes rank q's again only after q's next flag, i.e. after q
// finished reading it.
__global__ void __launch_bounds__(256) dp_peer_rs_sgd_kernel(const __grid_constant__ DPArgs a)
{
    const int bpr = gridDim.x / a.nloc;
    const int rl = blockIdx.x / bpr, bi = blockIdx.x % bpr;
    if (rl >= a.nloc) return;
    const int rank = a.rank0 + rl;
    const int64_t n = a.P + 1, ss = dp_slot_stride(a.P), slot = (int64_t)(a.t & 1ull) * ss;
    __shared__ int timed_out;
    if (bi == 0 && threadIdx.x == 0 && !dp_is_broken(a.flag[rank])) {   // a broken rank stops publishing
        __threadfence_system();
        dp_st_release(a.flag[rank], a.t);
    }
    if (threadIdx.x == 0) timed_out = dp_wait_all(a, rank, rl, 0, false);
    __syncthreads();
    if (timed_out) return;
    __threadfence();
    // this rank's slice of the mean, into every rank's mean buffer
    // this rank's slice (whole float4 groups: slots and the mean buffer are 16-byte aligned and
    // padded) of the mean, into every rank's mean buffer; DP_U groups per thread and round with
    // all their loads in flight (the same rank-order sums)
    const int64_t n4 = (n + 3) / 4, lo4 = n4 * rank / a.world, hi4 = n4 * (rank + 1) / a.world;
    const int64_t S = (int64_t)bpr * blockDim.x;
    for (int64_t j0 = lo4 + (int64_t)bi * blockDim.x + threadIdx.x; j0 < hi4; j0 += DP_U * S) {
        float4 g[DP_U];
#pragma unroll
        for (int u = 0; u < DP_U; ++u) g[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < a.world; ++q) {
            float4 v[DP_U];
            const float4 *src = reinterpret_cast<const float4 *>(a.xbuf[q] + slot);
#pragma unroll
            for (int u = 0; u < DP_U; ++u) v[u] = j0 + u * S < hi4 ? __ldcv(src + j0 + u * S) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < DP_U; ++u) {
                g[u].x += v[u].x; g[u].y += v[u].y; g[u].z += v[u].z; g[u].w += v[u].w;
            }
        }
        const float fw = (float)a.world;
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            if (j0 + u * S >= hi4) continue;
            const float4 m = make_float4(g[u].x / fw, g[u].y / fw, g[u].z / fw, g[u].w / fw);
            for (int q = 0; q < a.world; ++q)
                reinterpret_cast<float4 *>(const_cast<float *>(a.xbuf[q]) + 2 * ss)[j0 + u * S] = m;
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned *cnt = reinterpret_cast<unsigned *>(a.flag[rank] + 24);
        if (atomicAdd(cnt, 1u) == (unsigned)bpr - 1) {   // this rank's last block: publish
            atomicExch(cnt, 0u);
            __threadfence_system();
            dp_st_release(a.flag[rank] + 16, a.t);
        }
        timed_out = dp_wait_all(a, rank, rl, 16, true);   // co-resident (cooperative launch)
    }
    __syncthreads();
    if (timed_out) return;
    __threadfence();
    const float *mean = a.xbuf[rank] + 2 * ss;
    const float loss = __ldcv(mean + a.P);
    const bool ok = isfinite(loss);
    const int do_sync = *a.sync_flag[rl];
    float *on = a.online[rl], *tg = a.target[rl], *gm = a.gmean[rl];
    // the learner's own arrays 16-byte aligned (the real learner; emulated ranks may not be):
    // float4 groups, then the scalar tail
    const bool vec = ((reinterpret_cast<uintptr_t>(on) | reinterpret_cast<uintptr_t>(tg) |
                       reinterpret_cast<uintptr_t>(gm)) & 15) == 0;
    const int64_t P4 = vec ? a.P / 4 : 0;
    for (int64_t j0 = (int64_t)bi * blockDim.x + threadIdx.x; j0 < P4; j0 += DP_U * S) {
        float4 g[DP_U], w[DP_U];
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            const bool in = j0 + u * S < P4;
            g[u] = in ? __ldcv(reinterpret_cast<const float4 *>(mean) + j0 + u * S) : make_float4(0.f, 0.f, 0.f, 0.f);
            w[u] = in ? reinterpret_cast<const float4 *>(on)[j0 + u * S] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            const int64_t j = j0 + u * S;
            if (j >= P4) continue;
            reinterpret_cast<float4 *>(gm)[j] = g[u];
            if (ok) {
                const float4 nw = make_float4(w[u].x - a.lr * g[u].x, w[u].y - a.lr * g[u].y, w[u].z - a.lr * g[u].z,
                                              w[u].w - a.lr * g[u].w);
                reinterpret_cast<float4 *>(on)[j] = nw;
                if (do_sync) reinterpret_cast<float4 *>(tg)[j] = nw;
                if (rl == 0) dp_w0_planes4(W0Planes{a.w0.bf, a.w0.n, a.w0.pe, a.w0.D, a.w0.planes}, j, nw, do_sync);
            }
        }
    }
    for (int64_t i0 = 4 * P4 + (int64_t)bi * blockDim.x + threadIdx.x; i0 < a.P; i0 += DP_U * S) {
        float g[DP_U], w[DP_U];
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            const bool in = i0 + u * S < a.P;
            g[u] = in ? __ldcv(mean + i0 + u * S) : 0.0f;
            w[u] = in ? on[i0 + u * S] : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            const int64_t i = i0 + u * S;
            if (i >= a.P) continue;
            gm[i] = g[u];
            if (ok) {
                const float nw = w[u] - a.lr * g[u];
                on[i] = nw;
                if (do_sync) tg[i] = nw;
                if (rl == 0) dp_w0_planes(W0Planes{a.w0.bf, a.w0.n, a.w0.pe, a.w0.D, a.w0.planes}, i, nw, do_sync);
            }
        }
    }
    if (bi == 0 && threadIdx.x == 0) {
        gm[a.P] = loss;
        if (a.loss_out[rl]) *a.loss_out[rl] = loss;
        if (!ok) atomicOr(a.err[rl], ERRBIT_NUMERIC);
    }
}

__global__ void __launch_bounds__(256) dp_peer_sgd_kernel(const __grid_constant__ DPArgs a)
{
    const int bpr = gridDim.x / a.nloc;
    const int rl = blockIdx.x / bpr, bi = blockIdx.x % bpr;
    if (rl >= a.nloc) return;
    const int rank = a.rank0 + rl;
    const int64_t slot = (int64_t)(a.t & 1ull) * dp_slot_stride(a.P);
    // (1) this rank's step-t gradient is complete (written before this kernel): publish it
    if (bi == 0 && threadIdx.x == 0 && !dp_is_broken(a.flag[rank])) {   // a broken rank stops publishing
        __threadfence_system();
        dp_st_release(a.flag[rank], a.t);
    }
    // (2) wait for every other rank's (no block waits on this rank's own flag, so a plain launch
    // needs no co-residency); a rank that never arrives, or whose exchange is broken, ends the
    // wait with the sticky ERRBIT_PEER and the update skipped, and marks this rank's exchange
    // broken so every later step skips at once on every rank (fail fast instead of a hang)
    __shared__ int timed_out;
    if (threadIdx.x == 0) timed_out = dp_wait_all(a, rank, rl, 0, false);
    __syncthreads();
    if (timed_out) return;
    __threadfence();
    // (3) the mean loss decides the update for every CTA alike
    float ls = 0.0f;
    for (int q = 0; q < a.world; ++q) ls += __ldcv(a.xbuf[q] + slot + a.P);
    const float loss = ls / (float)a.world;
    const bool ok = isfinite(loss);
    const int do_sync = *a.sync_flag[rl];
    float *on = a.online[rl], *tg = a.target[rl], *gm = a.gmean[rl];
    // (4) mean of the ranks' gradients in rank order, SGD, target copy on sync steps
    const int64_t S = (int64_t)bpr * blockDim.x;
    for (int64_t i0 = (int64_t)bi * blockDim.x + threadIdx.x; i0 < a.P; i0 += DP_U * S) {
        float g[DP_U], w[DP_U];
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            g[u] = 0.0f;
            w[u] = i0 + u * S < a.P ? on[i0 + u * S] : 0.0f;
        }
        for (int q = 0; q < a.world; ++q) {
            float v[DP_U];
#pragma unroll
            for (int u = 0; u < DP_U; ++u) v[u] = i0 + u * S < a.P ? __ldcv(a.xbuf[q] + slot + i0 + u * S) : 0.0f;
#pragma unroll
            for (int u = 0; u < DP_U; ++u) g[u] += v[u];
        }
#pragma unroll
        for (int u = 0; u < DP_U; ++u) {
            const int64_t i = i0 + u * S;
            if (i >= a.P) continue;
            const float m = g[u] / (float)a.world;
            gm[i] = m;
            if (ok) {
                const float nw = w[u] - a.lr * m;
                on[i] = nw;
                if (do_sync) tg[i] = nw;
                if (rl == 0) dp_w0_planes(W0Planes{a.w0.bf, a.w0.n, a.w0.pe, a.w0.D, a.w0.planes}, i, nw, do_sync);
            }
        }
    }
    if (bi == 0 && threadIdx.x == 0) {
        gm[a.P] = loss;
        if (a.loss_out[rl]) *a.loss_out[rl] = loss;
        if (!ok) atomicOr(a.err[rl], ERRBIT_NUMERIC);
    }
}

}  // namespace rpl
