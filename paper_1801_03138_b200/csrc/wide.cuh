// wide.cuh -- the wide-input layer 0 of byte-state learners (SURVEY config 5: 84x84x4 uint8
// states, 28,224 inputs) on the 5th-generation tensor cores (tcgen05, umma.cuh).  CUDA path only.
//
// The input x = u8 / 255 (reading Q27) is carried exactly as the integer u (0..255 is exact in
// bf16) with the 1/255 applied to the fp32 result; every fp32 weight / gradient operand w is
// split into three bf16 terms hi + mid + lo that hold all 24 of its significand bits
// (umma::split3_bf16), so the three bf16 MMAs u*hi + u*mid + u*lo accumulate the exact
// products in fp32 -- an FP32-accurate layer 0 (tests/test_gpu_u8.py checks it against the
// fp64 oracle) at tensor-core rate.
//
//   wide_l0_kernel : Z0 partials.  CTA (net, k-chunk) computes D[128 units][B] =
//                    W0_net[:, chunk] . U_net[:, chunk]^T (A = W0 K-major, B = U K-major) and
//                    writes it (still x 255) to PF0[chunk][net][b][unit]; the reduction adds the
//                    chunks in order, divides by 255 once, adds the bias and applies the ReLU.
//   wide_dw0_kernel: dW0 tile [128 units][256 inputs] = dZ0^T U over the batch (A = dZ0^T
//                    MN-major, B = U^T MN-major), then g = D / 255 -> grad, SGD (and the target
//                    sync) of those W0 entries: layer 0's gradient never makes a round trip.
// The fp32 operands are split once, not per CTA: W0's planes live next to the fp32 master
// weights (rewritten by the dW0 epilogue's SGD, re-split by wide_split_kernel after any host
// write or target sync) and dZ0's planes are written by the train kernel.  Both sets of planes
// are stored PRE-TILED: each 64-deep K slice of a plane is the 16 KB canonical shared-memory
// image of that slice (wd_tix_k / wd_tix_mn), so one bulk copy on the TMA engine
// (cp.async.bulk, completing on an mbarrier) moves a slice plane.  Both kernels stage 64-deep
// K slices through two shared-memory buffers: the loads of slice i + 1 overlap the MMAs of
// slice i (tcgen05.commit -> mbarrier per buffer).
#pragma once
#include <cooperative_groups.h>
#include <stdint.h>

#include "umma.cuh"

namespace rpl {

constexpr int WD_M = 128;                 // units of layer 0 (the UMMA M)
constexpr int WD_KS = 64;                 // K slice per stage
constexpr int WD_T = 256;                 // threads
constexpr int WD_MAXN = 256;              // UMMA N at most (batch for the forward, inputs for dW0)
constexpr int WD_A_PLANE = WD_M * WD_KS * 2;            // bytes of one bf16 A plane
constexpr int WD_B_BYTES = WD_MAXN * WD_KS * 2;         // bytes of the bf16 B slice
constexpr int WD_STAGE = 3 * WD_A_PLANE + WD_B_BYTES;   // 80 KB
constexpr int WD_SMEM = 2 * WD_STAGE + 1024;            // + alignment slack
constexpr int WD_SMEM_MAX = 226 * 1024;                 // the per-CTA opt-in limit (227 KB) less static smem
// wide_dw0_kernel's epilogue: the accumulator tile [128][N + 4] plus, when it fits, the tile's
// fp32 weights [128][N + 4] prefetched with cp.async (one memory latency for the whole tile)
__host__ __device__ inline int wd_dw0_need(int ntile) { return 1024 + 2 * WD_M * (ntile + 4) * 4; }
__host__ __device__ inline bool wd_dw0_wpre(int ntile) { return wd_dw0_need(ntile) <= WD_SMEM_MAX; }
__host__ __device__ inline int wd_dw0_smem(int ntile)
{
    return wd_dw0_wpre(ntile) && wd_dw0_need(ntile) > WD_SMEM ? wd_dw0_need(ntile) : WD_SMEM;
}

struct WideArgs {
    int D, B, N0, nets, ks;          // inputs, batch, layer-0 units (== 128), nets, k-chunks
    int cs;                          // wide_l0_kernel cluster size: ks % cs == 0, the cs chunks of a
                                     // cluster sum their partials over DSMEM (PF0 holds ks / cs)
    const uint8_t *U0, *U1;          // gathered byte states s, s' [B][D]
    const float *online, *target;
    int64_t w0;                      // offset of W0 [N0][D] in the parameter blob
    float *PF0;                      // [ks][nets][B][N0]
    const float *dZ0;                // [B][N0] (materialised by the train kernel)
    const uint16_t *dZ0bf;           // its bf16 hi / mid / lo planes [3][wd_plane_elems(B)], MN-major tiles
    uint16_t *W0bf;                  // bf16 planes of W0: [net 0 online, 1 target][3][wd_plane_elems(D)], K-major tiles
    float *grad;                     // [P + 1] (grad[P] = batch-mean loss, set by the train kernel)
    int64_t P;
    float *online_w, *target_w;      // SGD targets (== online / target)
    float lr;
    int apply_update;
    const int32_t *sync_flag;
    int64_t b0;                      // offset of b0 (the fast-path variant: db0 is this kernel's)
    int do_db0;
    int ntile;                       // dW0 inputs per CTA (multiple of 16, <= 256)
    int wpre;                        // wd_dw0_wpre(ntile): the launch has wd_dw0_smem(ntile) bytes
    unsigned long long *trace;       // RPL_TRACE=1: per-CTA %globaltimer marks (kernel slots 4, 5)
    int nplanes;                     // bf16 terms per fp32 operand: 3 (FP32), 2 (TF32), 1 (BF16)
};

// RPL_TRACE=1: thread 0 of each CTA stores %globaltimer at marks 0 .. 7 of its slot
struct WdTrace {
    unsigned long long *slot;
    __device__ WdTrace(unsigned long long *tr, int kernel)
        : slot(tr && threadIdx.x == 0 ? tr + 8 * ((size_t)kernel * 2048 + blockIdx.x) : nullptr)
    {
        mark(0);
    }
    __device__ void mark(int i)
    {
        if (!slot) return;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        slot[i] = t;
    }
};

// chunk q of ks: 64-deep slices [q S / ks, (q + 1) S / ks) of the S = ceil(D / 64) slices
__host__ __device__ inline void wd_chunk(int64_t D, int ks, int q, int64_t &kb, int64_t &ke)
{
    const int64_t S = (D + WD_KS - 1) / WD_KS;
    kb = q * S / ks * WD_KS;
    ke = (q + 1) * S / ks * WD_KS;
    if (ke > D) ke = D;
}

// layer-0 partials wide_l0_kernel leaves in PF0 for batch B: ks / cs when the cluster sums
// apply (the rounded batch splits into 8-column pieces per owner), else ks
__host__ __device__ inline int wd_l0_partials(int ks, int cs, int B)
{
    const int N = (B + 15) & ~15;
    return cs > 1 && N % (8 * cs) == 0 ? ks / cs : ks;
}

// canonical no-swizzle offsets (umma.cuh): K-major rows x 64-deep slice, and MN-major
__device__ __forceinline__ uint32_t wd_off_k(int r, int k) { return (r >> 3) * 1024 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2; }
__device__ __forceinline__ uint32_t wd_off_mn(int r, int k, int R) { return (k >> 3) * (R / 8) * 128 + (r >> 3) * 128 + (k & 7) * 16 + (r & 7) * 2; }

// pre-tiled global planes (128 rows, K padded to the 64-deep slice, padding zero): element
// (row u, k) of a K-major plane (W0: u = unit, k = input) and of an MN-major one (dZ0^T:
// u = unit, k = sample)
__host__ __device__ inline int64_t wd_plane_elems(int64_t K) { return (int64_t)WD_M * ((K + WD_KS - 1) / WD_KS * WD_KS); }
__device__ __forceinline__ int64_t wd_tix_k(int u, int64_t k) { return (k >> 6) * (WD_M * WD_KS) + wd_off_k(u, (int)(k & 63)) / 2; }
__device__ __forceinline__ int64_t wd_tix_mn(int u, int64_t k) { return (k >> 6) * (WD_M * WD_KS) + wd_off_mn(u, (int)(k & 63), WD_M) / 2; }

__device__ __forceinline__ void wd_cp16(void *smem, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(umma::smem_u32(smem)), "l"(gmem) : "memory");
}

__device__ __forceinline__ uint32_t pack2(uint16_t a, uint16_t b) { return (uint32_t)a | ((uint32_t)b << 16); }

// planes[p] = split3(W0)_p (p = hi, mid, lo) for W0 [N0][D] row-major, K-major tiles
__global__ void __launch_bounds__(256) wide_split_kernel(const float *__restrict__ src, uint16_t *planes, int N0, int64_t D)
{
    const int64_t n = (int64_t)N0 * D, pe = wd_plane_elems(D);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint16_t h, m, l;
        umma::split3_bf16(src[i], h, m, l);
        const int64_t t = wd_tix_k((int)(i / D), i % D);
        planes[t] = h;
        planes[pe + t] = m;
        planes[2 * pe + t] = l;
    }
}
// the same for D % 8 == 0 and a 16-byte aligned source: a thread splits 8 consecutive inputs
// of one unit row (two 16-byte loads) into one 16-byte core-matrix row per plane; the grid's
// y dimension is the unit, so no 64-bit division per element
__global__ void __launch_bounds__(256) wide_split8_kernel(const float *__restrict__ src, uint16_t *planes, int64_t D)
{
    const int u = blockIdx.y;
    const int64_t pe = wd_plane_elems(D), G = D >> 3;
    const float *row = src + (int64_t)u * D;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (int64_t)gridDim.x * blockDim.x) {
        const float4 x0 = __ldg(reinterpret_cast<const float4 *>(row) + 2 * g);
        const float4 x1 = __ldg(reinterpret_cast<const float4 *>(row) + 2 * g + 1);
        const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        uint32_t hw[4], mw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) umma::split3_pack2(x[2 * i], x[2 * i + 1], hw[i], mw[i], lw[i]);
        const int64_t t = wd_tix_k(u, g << 3);   // 8 consecutive k of one row: 16 contiguous bytes
        *reinterpret_cast<uint4 *>(planes + t) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4 *>(planes + pe + t) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        *reinterpret_cast<uint4 *>(planes + 2 * pe + t) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}
inline void launch_wide_split(const float *src, uint16_t *planes, int N0, int64_t D, int sms, cudaStream_t st)
{
    if (D % 8 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && N0 <= 65535) {
        const int64_t G = D / 8;
        const unsigned gx = (unsigned)std::min<int64_t>((G + 255) / 256, std::max(1, 4 * sms / std::max(1, N0)) * 8);
        wide_split8_kernel<<<dim3(gx, (unsigned)N0), 256, 0, st>>>(src, planes, D);
    } else {
        wide_split_kernel<<<sms * 4, 256, 0, st>>>(src, planes, N0, D);
    }
}
// a byte 0..255 as bf16: exact in fp32 and in bf16 (<= 8 significant bits), so the bf16 is the
// fp32's upper half -- one I2F and a shift instead of the general rounding conversion
__device__ __forceinline__ uint16_t u8_bf16(uint32_t v) { return (uint16_t)(__float_as_uint((float)v) >> 16); }

// ------------------------------------------------------------------------------------------
// layer-0 forward partials
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(WD_T, 1) wide_l0_kernel(const __grid_constant__ WideArgs p)
{
    extern __shared__ uint8_t wd_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(((uintptr_t)wd_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t mbar[2], full[2];   // MMAs done with / weight planes landed in a stage
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int net = blockIdx.x / p.ks, kq = blockIdx.x % p.ks;
    WdTrace tr(p.trace, 4);
    int64_t kb, ke;
    wd_chunk(p.D, p.ks, kq, kb, ke);
    const int nsl = (int)((ke - kb + WD_KS - 1) / WD_KS);
    const int N = (p.B + 15) & ~15;                  // UMMA N: the batch rounded up to 16
    const uint8_t *U = net == 0 ? p.U0 : p.U1;
    if (warp == 0) umma::tmem_alloc(&tbase, 256);
    if (tid == 0) {
        umma::mbar_init(&mbar[0], 1);
        umma::mbar_init(&mbar[1], 1);
        umma::mbar_init(&full[0], 1);
        umma::mbar_init(&full[1], 1);
        umma::fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tbase;
    const uint32_t idesc = umma::idesc_bf16(WD_M, N, false, false);
    // software pipeline over the K slices: slice sl + 1's weight planes (cp.async group) and
    // byte states (registers) are in flight while slice sl is converted and multiplied; a
    // stage is refilled once the MMAs that read it two slices earlier have committed
    const int64_t pe = wd_plane_elems(p.D);
    const uint16_t *Wp = p.W0bf + (net == 1 ? 3 * pe : 0);
    auto issue_A = [&](int sl) {
        // thread 0: the hi / mid / lo tiles of W0[:, k0 .. k0+63], one 16 KB bulk copy each
        if (tid != 0) return;
        uint8_t *A = sm + (sl & 1) * WD_STAGE;
        const int64_t t0 = (kb + (int64_t)sl * WD_KS) / WD_KS * (WD_M * WD_KS);
        umma::mbar_expect_tx(&full[sl & 1], p.nplanes * WD_A_PLANE);
        for (int pl = 0; pl < p.nplanes; ++pl) umma::bulk_g2s(A + pl * WD_A_PLANE, Wp + pl * pe + t0, WD_A_PLANE, &full[sl & 1]);
    };
    const int totalB = N * (WD_KS / 16);   // 16-byte pieces of a slice's states (<= 4 per thread)
    auto load_B = [&](int sl, uint4 v[4]) {
        const int64_t k0 = kb + (int64_t)sl * WD_KS;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + q * WD_T;
            v[q] = make_uint4(0u, 0u, 0u, 0u);
            if (e >= totalB) continue;
            const int b = e / (WD_KS / 16), k = 16 * (e % (WD_KS / 16));
            if (b < p.B) {
                const uint8_t *src = U + (int64_t)b * p.D + k0 + k;
                if (k0 + k + 15 < ke && ((uintptr_t)src & 15) == 0) {
                    v[q] = __ldg(reinterpret_cast<const uint4 *>(src));
                } else {
                    uint8_t t[16];
                    for (int i = 0; i < 16; ++i) t[i] = (k0 + k + i < ke) ? src[i] : 0;
                    v[q] = make_uint4(t[0] | t[1] << 8 | t[2] << 16 | (uint32_t)t[3] << 24,
                                      t[4] | t[5] << 8 | t[6] << 16 | (uint32_t)t[7] << 24,
                                      t[8] | t[9] << 8 | t[10] << 16 | (uint32_t)t[11] << 24,
                                      t[12] | t[13] << 8 | t[14] << 16 | (uint32_t)t[15] << 24);
                }
            }
        }
    };
    auto store_B = [&](int sl, const uint4 v[4]) {   // u8 -> bf16, K-major
        uint8_t *Bs = sm + (sl & 1) * WD_STAGE + 3 * WD_A_PLANE;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + q * WD_T;
            if (e >= totalB) continue;
            const int b = e / (WD_KS / 16), k = 16 * (e % (WD_KS / 16));
            const uint32_t w4[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
            uint32_t o8[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                o8[2 * i] = pack2(u8_bf16(w4[i] & 0xFF), u8_bf16((w4[i] >> 8) & 0xFF));
                o8[2 * i + 1] = pack2(u8_bf16((w4[i] >> 16) & 0xFF), u8_bf16(w4[i] >> 24));
            }
            *reinterpret_cast<uint4 *>(Bs + wd_off_k(b, k)) = make_uint4(o8[0], o8[1], o8[2], o8[3]);
            *reinterpret_cast<uint4 *>(Bs + wd_off_k(b, k + 8)) = make_uint4(o8[4], o8[5], o8[6], o8[7]);
        }
    };
    uint4 vb[4], vn[4];
    tr.mark(1);
    issue_A(0);
    load_B(0, vb);
    for (int sl = 0; sl < nsl; ++sl) {
        const int st = sl & 1;
        uint8_t *A = sm + st * WD_STAGE, *Bs = A + 3 * WD_A_PLANE;
        store_B(sl, vb);   // stage st was freed before A(sl) was issued
        if (sl + 1 < nsl) {
            // the other stage last fed the MMAs of slice sl - 1: wait for them, then refill it
            if (sl >= 1) umma::mbar_wait(&mbar[st ^ 1], ((sl - 1) >> 1) & 1);
            issue_A(sl + 1);
            load_B(sl + 1, vn);
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            umma::fence_after_sync();
            umma::mbar_wait(&full[st], (sl >> 1) & 1);   // A(sl) has landed
            for (int s = 0; s < WD_KS / 16; ++s) {
                const uint64_t bd = umma::desc(Bs + 2 * s * 128, 128, 1024);
                for (int pl = 0; pl < p.nplanes; ++pl)
                    umma::mma_bf16(tmem, umma::desc(A + pl * WD_A_PLANE + 2 * s * 128, 128, 1024), bd,
                                   idesc, sl > 0 || s > 0 || pl > 0);
            }
            umma::commit(&mbar[st]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) vb[q] = vn[q];
    }
    // the last slice's commit covers every earlier MMA
    {
        const int last = nsl - 1;
        umma::mbar_wait(&mbar[last & 1], (last >> 1) & 1);
    }
    tr.mark(2);
    umma::fence_after_sync();
    // epilogue: warp w reads TMEM lanes (units) 32 (w % 4) .. + 31, columns (samples) of its half
    if (p.cs == 1 || N % (8 * p.cs) != 0) {   // (a batch that does not split: ks partials)
        const int q = warp & 3, half = warp >> 2, u = 32 * q + lane;
        const int c0 = half * (N / 2), c1 = c0 + N / 2;
        float *out = p.PF0 + ((int64_t)kq * p.nets + net) * p.B * p.N0;
        // 32 columns per round: four TMEM loads in flight, one wait, then the stores
        for (int c = c0; c < c1; c += 32) {
            uint32_t r[4][8];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c + 8 * j < c1) umma::tmem_ld8_nowait(tmem + ((uint32_t)(32 * q) << 16) + c + 8 * j, r[j]);
            umma::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int cc = c + 8 * j + i;
                    if (cc < c1 && cc < p.B && u < p.N0)
                        out[(int64_t)cc * p.N0 + u] = __uint_as_float(r[j][i]);   // x 255
                }
        }
    } else {
        // cluster of cs consecutive chunks: CTA r owns sample columns [r Nc, (r + 1) Nc) of the
        // cluster's sum.  Every CTA pushes each 8-column piece of its accumulator straight from
        // TMEM into the owner's shared memory (distributed shared memory stores: no round
        // trip), one slot per source rank; after one cluster barrier each owner adds its cs
        // slots in rank order and writes the cluster's single partial -- PF0 traffic and
        // wide_reduce_kernel's work drop cs-fold
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        const int rk = (int)cl.block_rank();
        const int Nc = N / p.cs, RS = Nc + 4;               // columns per owner, slot row stride
        float *R = reinterpret_cast<float *>(sm);            // [cs source ranks][128 units][RS]
        {
            const int q = warp & 3, half = warp >> 2, u = 32 * q + lane;
            const int c0 = half * (N / 2), c1 = c0 + N / 2;
            for (int c = c0; c < c1; c += 8) {
                float v[8];
                umma::tmem_ld8(tmem + ((uint32_t)(32 * q) << 16) + c, v);
                const int ow = c / Nc;
                float *dst = cl.map_shared_rank(R, ow) + ((int64_t)rk * WD_M + u) * RS + (c - ow * Nc);
                *reinterpret_cast<float4 *>(dst) = make_float4(v[0], v[1], v[2], v[3]);
                *reinterpret_cast<float4 *>(dst + 4) = make_float4(v[4], v[5], v[6], v[7]);
            }
        }
        cl.sync();   // every slot of every owner is written
        float *out = p.PF0 + ((int64_t)(kq / p.cs) * p.nets + net) * p.B * p.N0;
        for (int f = tid; f < WD_M * (Nc / 4); f += WD_T) {
            const int u = f % WD_M, c = 4 * (f / WD_M);     // consecutive threads: consecutive units
            float4 acc = *reinterpret_cast<const float4 *>(R + (int64_t)u * RS + c);
            for (int r = 1; r < p.cs; ++r) {
                const float4 v = *reinterpret_cast<const float4 *>(R + ((int64_t)r * WD_M + u) * RS + c);
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            const int b = rk * Nc + c;
            if (u < p.N0) {
                const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
                for (int i2 = 0; i2 < 4; ++i2)
                    if (b + i2 < p.B) out[(int64_t)(b + i2) * p.N0 + u] = a4[i2];   // x 255
            }
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    tr.mark(3);
    if (warp == 0) umma::tmem_free(tmem, 256);
}

// ------------------------------------------------------------------------------------------
// dW0 + SGD of W0
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(WD_T, 1) wide_dw0_kernel(const __grid_constant__ WideArgs p)
{
    extern __shared__ uint8_t wd_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(((uintptr_t)wd_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t n0 = (int64_t)blockIdx.x * p.ntile;                  // first input of the tile
    WdTrace tr(p.trace, 5);
    const int nn = (int)(p.D - n0 < p.ntile ? p.D - n0 : p.ntile);    // inputs in the tile
    const int N = (nn + 15) & ~15;
    const int nsl = (p.B + WD_KS - 1) / WD_KS;
    __shared__ uint64_t full[2];
    if (warp == 0) umma::tmem_alloc(&tbase, 256);
    if (tid == 0) {
        umma::mbar_init(&mbar[0], 1);
        umma::mbar_init(&mbar[1], 1);
        umma::mbar_init(&full[0], 1);
        umma::mbar_init(&full[1], 1);
        umma::fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tbase;
    const uint32_t idesc = umma::idesc_bf16(WD_M, N, true, true);
    const float loss = __ldcg(p.grad + p.P);
    const bool upd = p.apply_update && isfinite(loss);
    const bool sync = *p.sync_flag != 0;
    if (p.do_db0 && warp == WD_T / 32 - 1) {
        // db0 = sum_b dZ0[b][u] (the last warp of CTA u, lanes stride the samples, fixed
        // shuffle tree) and its SGD, first thing: its loads overlap the first slice's
        for (int u = blockIdx.x; u < p.N0; u += gridDim.x) {
            float acc = 0.0f;
#pragma unroll 8
            for (int bb = lane; bb < p.B; bb += 32) acc += __ldcg(p.dZ0 + (int64_t)bb * p.N0 + u);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
            if (lane == 0) {
                p.grad[p.b0 + u] = acc;
                if (upd) {
                    const float w = p.online_w[p.b0 + u] - p.lr * acc;
                    p.online_w[p.b0 + u] = w;
                    if (sync) p.target_w[p.b0 + u] = w;
                }
            }
        }
    }
    // software pipeline as in wide_l0_kernel: slice sl + 1's dZ0 planes (bulk copies) and byte
    // states (registers) are in flight while slice sl is converted and multiplied
    auto issue_A = [&](int sl) {
        // A = dZ0^T slice: element (unit u, sample b) = dZ0[b][u], MN-major: the train
        // kernel's pre-tiled bf16 planes, one 16 KB bulk copy each (thread 0)
        if (tid != 0) return;
        uint8_t *A = sm + (sl & 1) * WD_STAGE;
        const int64_t pz = wd_plane_elems(p.B), t0 = (int64_t)sl * (WD_M * WD_KS);
        umma::mbar_expect_tx(&full[sl & 1], p.nplanes * WD_A_PLANE);
        for (int pl = 0; pl < p.nplanes; ++pl)
            umma::bulk_g2s(A + pl * WD_A_PLANE, p.dZ0bf + pl * pz + t0, WD_A_PLANE, &full[sl & 1]);
    };
    // B = U^T slice: element (input n, sample b) = U[b][n0 + n], MN-major (contiguous in n);
    // 16-byte pieces, at most 4 per thread
    const int totalB = WD_KS * (N / 16);
    auto load_B = [&](int sl, uint4 v[4]) {
        const int b0 = sl * WD_KS;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + q * WD_T;
            v[q] = make_uint4(0u, 0u, 0u, 0u);
            if (e >= totalB) continue;
            const int bb = e / (N / 16), n = 16 * (e % (N / 16));
            if (b0 + bb < p.B) {
                const uint8_t *src = p.U0 + (int64_t)(b0 + bb) * p.D + n0 + n;
                if (n + 15 < nn && ((uintptr_t)src & 15) == 0) {
                    v[q] = __ldg(reinterpret_cast<const uint4 *>(src));
                } else {
                    uint8_t t[16];
                    for (int i = 0; i < 16; ++i) t[i] = (n + i < nn) ? src[i] : 0;
                    v[q] = make_uint4(t[0] | t[1] << 8 | t[2] << 16 | (uint32_t)t[3] << 24,
                                      t[4] | t[5] << 8 | t[6] << 16 | (uint32_t)t[7] << 24,
                                      t[8] | t[9] << 8 | t[10] << 16 | (uint32_t)t[11] << 24,
                                      t[12] | t[13] << 8 | t[14] << 16 | (uint32_t)t[15] << 24);
                }
            }
        }
    };
    auto store_B = [&](int sl, const uint4 v[4]) {
        uint8_t *Bs = sm + (sl & 1) * WD_STAGE + 3 * WD_A_PLANE;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + q * WD_T;
            if (e >= totalB) continue;
            const int bb = e / (N / 16), n = 16 * (e % (N / 16));
            const uint32_t w4[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
            uint32_t o8[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                o8[2 * i] = pack2(u8_bf16(w4[i] & 0xFF), u8_bf16((w4[i] >> 8) & 0xFF));
                o8[2 * i + 1] = pack2(u8_bf16((w4[i] >> 16) & 0xFF), u8_bf16(w4[i] >> 24));
            }
            *reinterpret_cast<uint4 *>(Bs + wd_off_mn(n, bb, N)) = make_uint4(o8[0], o8[1], o8[2], o8[3]);
            *reinterpret_cast<uint4 *>(Bs + wd_off_mn(n + 8, bb, N)) = make_uint4(o8[4], o8[5], o8[6], o8[7]);
        }
    };
    tr.mark(1);
    uint4 vb[4], vn[4];
    issue_A(0);
    load_B(0, vb);
    for (int sl = 0; sl < nsl; ++sl) {
        const int st = sl & 1;
        const uint8_t *A = sm + st * WD_STAGE, *Bs = A + 3 * WD_A_PLANE;
        store_B(sl, vb);   // stage st was freed before A(sl) was issued
        if (sl + 1 < nsl) {
            // the other stage last fed the MMAs of slice sl - 1: wait for them, then refill it
            if (sl >= 1) umma::mbar_wait(&mbar[st ^ 1], ((sl - 1) >> 1) & 1);
            issue_A(sl + 1);
            load_B(sl + 1, vn);
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
            umma::fence_after_sync();
            umma::mbar_wait(&full[st], (sl >> 1) & 1);
            const int ksteps = (min(WD_KS, p.B - sl * WD_KS) + 15) / 16;
            for (int s = 0; s < ksteps; ++s) {
                const uint64_t bd = umma::desc(Bs + 2 * s * (N / 8) * 128, (N / 8) * 128, 128);
                for (int pl = 0; pl < p.nplanes; ++pl)
                    umma::mma_bf16(tmem, umma::desc(A + pl * WD_A_PLANE + 2 * s * (WD_M / 8) * 128,
                                                    (WD_M / 8) * 128, 128),
                                   bd, idesc, sl > 0 || s > 0 || pl > 0);
            }
            umma::commit(&mbar[st]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) vb[q] = vn[q];
    }
    tr.mark(2);
    {
        const int last = nsl - 1;
        umma::mbar_wait(&mbar[last & 1], (last >> 1) & 1);
    }
    tr.mark(4);
    umma::fence_after_sync();
    // epilogue: the accumulator tile goes TMEM -> registers -> shared memory (the staging
    // buffers are free: every MMA has completed) while the tile's weights stream into shared
    // memory behind it (wpre), then each warp walks whole W0 rows so the weight, gradient and
    // plane accesses are coalesced: g = D / 255 -> grad; w -= lr g (skipped on a non-finite
    // loss); the target copy on sync steps
    const int TS = N + 4;                           // tile row stride (floats)
    float *T = reinterpret_cast<float *>(sm);       // [128][TS]
    float *Wt = T + WD_M * TS;                      // [128][TS] (wpre)
    const bool wpre = p.wpre && upd;
    if (wpre) {
        const int nq = nn / 4;
        // e = pu * nq + pc, advanced by WD_T = du * nq + dc without divisions
        const int du = WD_T / nq, dc = WD_T % nq;
        int pu = tid / nq, pc = tid % nq;
        for (int e = tid; e < p.N0 * nq; e += WD_T) {
            wd_cp16(Wt + pu * TS + 4 * pc, p.online_w + p.w0 + (int64_t)pu * p.D + n0 + 4 * pc);
            pu += du;
            pc += dc;
            if (pc >= nq) {
                pc -= nq;
                ++pu;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    {
        const int q = warp & 3, half = warp >> 2, u = 32 * q + lane;
        const int c0 = half * (N / 2), c1 = c0 + N / 2;
        for (int c = c0; c < c1; c += 32) {   // four TMEM loads in flight per wait
            uint32_t r[4][8];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c + 8 * j < c1) umma::tmem_ld8_nowait(tmem + ((uint32_t)(32 * q) << 16) + c + 8 * j, r[j]);
            umma::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c + 8 * j < c1) {
                    float *dst = T + u * TS + c + 8 * j;
                    *reinterpret_cast<float4 *>(dst) = make_float4(__uint_as_float(r[j][0]), __uint_as_float(r[j][1]),
                                                                   __uint_as_float(r[j][2]), __uint_as_float(r[j][3]));
                    *reinterpret_cast<float4 *>(dst + 4) = make_float4(__uint_as_float(r[j][4]), __uint_as_float(r[j][5]),
                                                                       __uint_as_float(r[j][6]), __uint_as_float(r[j][7]));
                }
        }
    }
    if (wpre) asm volatile("cp.async.wait_group 0;" ::: "memory");
    tr.mark(5);
    umma::fence_before_sync();
    __syncthreads();
    {
        const int64_t pe = wd_plane_elems(p.D);
        const float k255 = 1.0f / 255.0f;
        // task (8-row group G, 16-input chunk): lane 4 r + q takes row 8 G + r, inputs
        // 16 chunk + 4 q .. + 3, so the fp32 rows go out in 64-byte runs and the bf16 plane
        // tiles in 256-byte runs (two whole core matrices): every store fills its sectors
        constexpr int NWE = WD_T / 32;
        const int r8 = lane >> 2, q4 = lane & 3;
        const int nch = nn / 16, ntask = (p.N0 / 8) * nch;
#pragma unroll 2
        int tg = warp / nch, tc = warp % nch;   // task = tg * nch + tc, advanced without divisions
        for (int task = warp; task < ntask; task += NWE, tc += NWE) {
                while (tc >= nch) {
                    tc -= nch;
                    ++tg;
                }
                {
                    const int u = 8 * tg + r8, c = 16 * tc + 4 * q4;
                    const int64_t j = (int64_t)u * p.D + n0 + c;   // index within W0
                    const int64_t wi = p.w0 + j;
                    const float4 t = *reinterpret_cast<const float4 *>(T + u * TS + c);
                    const float4 g = make_float4(t.x * k255, t.y * k255, t.z * k255, t.w * k255);
                    *reinterpret_cast<float4 *>(p.grad + wi) = g;
                    if (!upd) continue;
                    float4 w = wpre ? *reinterpret_cast<const float4 *>(Wt + u * TS + c)
                                    : *reinterpret_cast<const float4 *>(p.online_w + wi);
                    w.x -= p.lr * g.x;
                    w.y -= p.lr * g.y;
                    w.z -= p.lr * g.z;
                    w.w -= p.lr * g.w;
                    *reinterpret_cast<float4 *>(p.online_w + wi) = w;
                    // the next step's forward operand: W0's bf16 planes, split once here
                    uint2 ph, pm, pl;
                    umma::split3_pack2(w.x, w.y, ph.x, pm.x, pl.x);
                    umma::split3_pack2(w.z, w.w, ph.y, pm.y, pl.y);
                    const int64_t tx = wd_tix_k(u, n0 + c);   // 4 inputs of one core-matrix row
                    *reinterpret_cast<uint2 *>(p.W0bf + tx) = ph;
                    if (p.nplanes > 1) *reinterpret_cast<uint2 *>(p.W0bf + pe + tx) = pm;
                    if (p.nplanes > 2) *reinterpret_cast<uint2 *>(p.W0bf + 2 * pe + tx) = pl;
                    if (sync) {
                        *reinterpret_cast<float4 *>(p.target_w + wi) = w;
                        *reinterpret_cast<uint2 *>(p.W0bf + 3 * pe + tx) = ph;
                        if (p.nplanes > 1) *reinterpret_cast<uint2 *>(p.W0bf + 4 * pe + tx) = pm;
                        if (p.nplanes > 2) *reinterpret_cast<uint2 *>(p.W0bf + 5 * pe + tx) = pl;
                    }
                }
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    tr.mark(6);
    if (warp == 0) umma::tmem_free(tmem, 256);
}

// wide inputs on the fast path: H0[net][b][u] = ReLU(b0_net[u] + (sum of the wide_l0_kernel
// partials) / 255) for the fast kernels above layer 0.  A CTA takes 32 float4 groups of 4
// consecutive elements; its 8 warps take the chunks q = w, w + 8, ... (all <= ks / 8 + 1 loads
// of a thread in flight at once), and warp 0 adds the 8 residue sums in warp order: a fixed
// summation order, one memory round trip per thread
constexpr int WR_G = 32, WR_S = 8, WR_MAXQ = 10;   // groups per CTA, residues, ks <= 80
__global__ void __launch_bounds__(256) wide_reduce_kernel(const float *__restrict__ PF0, int ks, int nets,
                                                          int B, int N0, const float *online,
                                                          const float *target, int64_t b0, float *H0)
{
    __shared__ float4 part[WR_S][WR_G];
    const int64_t per = (int64_t)B * N0, total = (int64_t)nets * per, G = total / 4;   // N0 % 4 == 0
    const int gl = threadIdx.x % WR_G, res = threadIdx.x / WR_G;
    for (int64_t gb = (int64_t)blockIdx.x * WR_G; gb < G; gb += (int64_t)gridDim.x * WR_G) {
        const int64_t g = gb + gl;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g < G) {
            const float4 *src = reinterpret_cast<const float4 *>(PF0) + g;
            float4 pv[WR_MAXQ];
#pragma unroll
            for (int r = 0; r < WR_MAXQ; ++r) {
                const int q = res + WR_S * r;
                pv[r] = q < ks ? __ldcg(src + (int64_t)q * G) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int r = 0; r < WR_MAXQ; ++r) {
                acc.x += pv[r].x;
                acc.y += pv[r].y;
                acc.z += pv[r].z;
                acc.w += pv[r].w;
            }
        }
        part[res][gl] = acc;
        __syncthreads();
        if (res == 0 && g < G) {
            float4 t = part[0][gl];
#pragma unroll
            for (int w = 1; w < WR_S; ++w) {
                const float4 o = part[w][gl];
                t.x += o.x;
                t.y += o.y;
                t.z += o.z;
                t.w += o.w;
            }
            const float a4[4] = {t.x, t.y, t.z, t.w};
            float4 h;
            float *hv = reinterpret_cast<float *>(&h);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t i = 4 * g + r;
                const int net = (int)(i / per), u = (int)(i % N0);
                const float v = a4[r] / 255.0f + __ldg((net == 1 ? target : online) + b0 + u);
                hv[r] = v > 0.0f ? v : 0.0f;
            }
            reinterpret_cast<float4 *>(H0)[g] = h;
        }
        __syncthreads();
    }
}

}  // namespace rpl
