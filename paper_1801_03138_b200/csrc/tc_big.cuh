// tc_big.cuh -- the train step at large batch (B >= kTcbMinBatch) with its three dense
// contractions on the 5th-generation tensor cores (tcgen05 kind::f16, fp32 accumulators in
// tensor memory, operands staged by the TMA engine with cp.async.bulk).  Nets: two trunk
// layers with 128 layer-0 units, the paper's dueling net 27 -> 128 -> [V 512 | A 512] -> 1 + |A|
// and plain MLPs with N1 % 128 == 0.  CUDA path only; FastArgs / td_warp / the SGD
// kernel K4 are train_fast.cuh's.
//
// One step, six kernels in one CUDA graph (B = batch, Bp = B rounded up to 128):
//   T0 tcb_l0_kernel   Philox sample + gather of s / s', the deferred insert's ring rows
//                      (P:73), layer 0 of every net in FP32 FMA (K = state_dim is tiny) ->
//                      H0 images (bf16 planes) per net, H0 (fp32, online net on s), the
//                      [x | 1] image of s
//   T1 tcb_fwd_kernel  layer 1 of every net: D1[b][u] = H0 W1^T (M = 128 samples, N = 128
//                      units, K = 128), + b1, ReLU, the head's partial dot products per
//                      64-unit column group (FMA), H1 (fp32) of the online net on s.
//                      Persistent per (net, unit tile): the W1 tile stays in shared memory,
//                      the H0 tiles stream through a 4-slot ring; one producer warp (TMA),
//                      one MMA warp, 8 epilogue warps on a double-buffered accumulator
//   TD tcb_td_kernel   head sums, dueling combine, DQN / Double-DQN target, Huber,
//                      dHead -- a warp per sample (train_fast.cuh td_warp)
//   T3a tcb_dw1_kernel per (unit tile, batch chunk group): dZ1 = (dHead . W_head) * [H1 > 0]
//                      into shared memory (and its image to global for T3b), dW1 += dZ1^T H0
//                      on the tensor cores (K = samples), db1 / dW_head / db_head by FMA
//   T3b tcb_dh0_kernel per (128-row batch tile, split of the layer-1 units):
//                      dH0 = dZ1 W1 (K = units), dZ0 = dH0 * [H0 > 0] (the mask distributes
//                      over the split sum), dW0 | db0 share = dZ0^T [x | 1] (K = samples)
//   K4                 sums of the partials in a fixed order, SGD, target sync, and the
//                      bf16 image of the new W1 (train_fast.cuh fast_bwd0_sgd_kernel)
//
// FP32 accuracy (BASELINE north star: 1e-5): every operand x is carried as three bf16 terms
// hi + mid + lo holding all 24 significand bits (umma::split3_bf16), and a product is formed
// from the six term products whose order is above 2^-24 (lo.hi, hi.lo, mid.mid, mid.hi,
// hi.mid, hi.hi, smallest first), accumulated in fp32.  Six kind::f16 MMAs of K = 16 cost the
// same tensor time as three kind::tf32 MMAs of K = 8 per 16 products of fp32 operands ("3xTF32"),
// and bf16 operands may be MN-major in the no-swizzle layout, so each matrix here needs ONE
// image for both the K-major and the MN-major uses.  rpl_dqn_config.precision BF16 (reading Q33):
// the hi.hi product only.
//
// Image layout (all operands, global and shared): "row-group major" core matrices.  Element
// (r, c) of an R x C matrix (C % 8 == 0) lives at bf16 offset
//     ((r / 8) * (C / 8) + c / 8) * 64 + (r % 8) * 8 + c % 8
// i.e. 8 rows x 8 consecutive columns (16 bytes per row) form one 128-byte core matrix; core
// matrices run along the columns, then down the row groups.  As a K-major operand with K =
// the columns: LBO = 128 B, SBO = (C / 8) * 128 B; as an MN-major operand with MN = the
// columns and K = the rows: SBO = 128 B, LBO = (C / 8) * 128 B (umma.cuh).  A block of whole
// row groups is contiguous; a column range of one row group is contiguous.  Each plane (hi,
// mid, lo) of a matrix is a separate image.
#pragma once
#include "umma.cuh"

namespace rpl {
namespace tcb {

constexpr int N0 = 128;       // layer-0 units (the M of the dW0 MMA, the K of layer 1)
constexpr int JW = 8;         // head outputs one unit tile contributes to (dueling A stream: |A|)
constexpr int JPMAX = 16;     // padded head width of dHead rows (J <= 16)
constexpr int T0_ROWS = 16, T0_T = 256;   // T0: 16 half-warps, one sampled row each
#ifndef RPL_T1_EPW
#define RPL_T1_EPW 8
#endif
#ifndef RPL_T1_SLOTS
#define RPL_T1_SLOTS 4
#endif
constexpr int T1_EPW = RPL_T1_EPW;   // T1 epilogue warps (a multiple of 4: per TMEM lane quarter)
constexpr int T1_PSL = 1;                   // head partial slots per 128-unit tile (TD sums N1 / 128)
constexpr int T1_CPW = 128 / (T1_EPW / 4);  // accumulator columns per epilogue thread
constexpr int T1_HN = 16;                   // head MMA N: the tile's head outputs, padded (J <= 16)
// T1 tensor memory (512 columns): two layer-1 accumulators [0, 256), the head accumulator
// [256, 272), the head MMA's A operand = H1 of the tile as 3 bf16 planes of 64 columns
// (two bf16 per 32-bit column, even k in the low half) [320, 512)
constexpr int T1_TM_DH = 256, T1_TM_AH = 320;
constexpr int T1_T = (T1_EPW + 2) * 32;     // + producer warp, MMA warp
constexpr int T1_SLOTS = RPL_T1_SLOTS;   // H0 ring slots (one 32-deep K quarter of a 128-row tile each)
constexpr int T1_SLOT = 3 * 128 * 32 * 2;   // bytes of one slot (three planes)
constexpr int T3A_T = 256;
constexpr int T3A_STAGE_A = 3 * 64 * 128 * 2;   // dZ1 chunk: 64 samples x 128 units, 3 planes
constexpr int T3A_STAGE_B = 3 * 64 * N0 * 2;    // H0 chunk: 64 samples x 128 layer-0 units
constexpr int T3B_T = 128;
constexpr int T3B_STAGE_A = 3 * 128 * 64 * 2;   // dZ1: 128 samples x 64 units
constexpr int T3B_STAGE_B = 3 * 64 * N0 * 2;    // W1: 64 units x 128
constexpr int XW = 32;                          // [x | 1] image width (state_dim <= 31)

__host__ __device__ __forceinline__ int64_t img(int64_t r, int c, int C)
{
    return ((r >> 3) * (C >> 3) + (c >> 3)) * 64 + (r & 7) * 8 + (c & 7);
}

// H0 image as T1 reads it: 128-row x 32-column (tile, K quarter) blocks of 8 KB, each block
// row-group major with C = 32 (so one bulk copy per plane fills a T1 ring slot)
__host__ __device__ __forceinline__ int64_t qimg(int64_t r, int c)
{
    return ((r >> 7) * (N0 / 32) + (c >> 5)) * (128 * 32) + (((r & 127) >> 3) * 4 + ((c & 31) >> 3)) * 64 + (r & 7) * 8 + (c & 7);
}

// dZ1 image as T3b reads it: 128-row x 64-unit (tile, unit chunk) blocks of 16 KB, each block
// row-group major with C = 64 (one bulk copy per plane fills a T3b stage)
__host__ __device__ __forceinline__ int64_t dzimg(int64_t r, int u, int N1)
{
    return ((r >> 7) * (N1 >> 6) + (u >> 6)) * (128 * 64) + (((r & 127) >> 3) * 8 + ((u & 63) >> 3)) * 64 + (r & 7) * 8 + (u & 7);
}

// eight consecutive fp32 values -> their hi / mid / lo bf16 terms, 16 bytes per plane
__device__ __forceinline__ void split8(const float (&x)[8], uint4 &h, uint4 &m, uint4 &l)
{
    uint32_t hw[4], mw[4], lw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) umma::split3_pack2(x[2 * i], x[2 * i + 1], hw[i], mw[i], lw[i]);
    h = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    m = make_uint4(mw[0], mw[1], mw[2], mw[3]);
    l = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}
// store the three planes of 8 values at image offset `off` (bf16 elements, 16-byte aligned)
__device__ __forceinline__ void store8(uint16_t *base, int64_t plane, int64_t off, const float (&x)[8])
{
    uint4 h, m, l;
    split8(x, h, m, l);
    *reinterpret_cast<uint4 *>(base + off) = h;
    *reinterpret_cast<uint4 *>(base + plane + off) = m;
    *reinterpret_cast<uint4 *>(base + 2 * plane + off) = l;
}
__device__ __forceinline__ void store8_smem(char *base, int plane_bytes, int off_bytes, const float (&x)[8])
{
    uint4 h, m, l;
    split8(x, h, m, l);
    *reinterpret_cast<uint4 *>(base + off_bytes) = h;
    *reinterpret_cast<uint4 *>(base + plane_bytes + off_bytes) = m;
    *reinterpret_cast<uint4 *>(base + 2 * plane_bytes + off_bytes) = l;
}

// the six term products of one K = 16 step (small terms first); hi.hi only at BF16 precision
__device__ __forceinline__ void mma6(uint32_t d, const uint64_t (&a)[3], const uint64_t (&b)[3], uint32_t id,
                                     bool acc, bool fp32)
{
    if (fp32) {
        umma::mma_bf16(d, a[2], b[0], id, acc);
        umma::mma_bf16(d, a[0], b[2], id, true);
        umma::mma_bf16(d, a[1], b[1], id, true);
        umma::mma_bf16(d, a[1], b[0], id, true);
        umma::mma_bf16(d, a[0], b[1], id, true);
        umma::mma_bf16(d, a[0], b[0], id, true);
    } else {
        umma::mma_bf16(d, a[0], b[0], id, acc);
    }
}

// 16 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void ld16(uint32_t a, uint32_t (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st16(uint32_t a, const uint32_t *r)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                    "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]^T (kind::f16, A: M lanes x K packed two bf16 per column)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, bool acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(id), "r"((uint32_t)acc) : "memory");
}
// mma6 with the A terms in tensor memory (same product order)
__device__ __forceinline__ void mma6_ts(uint32_t d, const uint32_t (&a)[3], const uint64_t (&b)[3], uint32_t id,
                                        bool acc, bool fp32)
{
    if (fp32) {
        mma_bf16_ts(d, a[2], b[0], id, acc);
        mma_bf16_ts(d, a[0], b[2], id, true);
        mma_bf16_ts(d, a[1], b[1], id, true);
        mma_bf16_ts(d, a[1], b[0], id, true);
        mma_bf16_ts(d, a[0], b[1], id, true);
        mma_bf16_ts(d, a[0], b[0], id, true);
    } else {
        mma_bf16_ts(d, a[0], b[0], id, acc);
    }
}
__device__ __forceinline__ uint32_t lane_addr(uint32_t base, int quarter, int col)
{
    return base + ((uint32_t)(32 * quarter) << 16) + (uint32_t)col;
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(umma::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t phase)
{
    umma::mbar_wait(bar, phase);
    umma::fence_after_sync();
}
// bulk (TMA engine) copy shared -> global, tracked by the issuing thread's bulk groups
__device__ __forceinline__ void bulk_s2g(void *gmem, const void *smem, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(gmem), "r"(umma::smem_u32(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void epi_sync(int n) { asm volatile("bar.sync 1, %0;" :: "r"(n) : "memory"); }

// the head outputs a 128-unit tile of layer 1 feeds: dueling V stream j = 0, A stream
// j = 1 .. |A|, plain MLP j = 0 .. J-1 (DESIGN.md §6 parameter blob)
__device__ __forceinline__ void head_range(const FastArgs &p, int u0, int &jlo, int &jhi)
{
    if (!p.dueling) {
        jlo = 0;
        jhi = p.J;
    } else if (u0 < p.S) {
        jlo = 0;
        jhi = 1;
    } else {
        jlo = 1;
        jhi = p.J;
    }
}
// head weight of output j for layer-1 unit u (0 where u does not feed j)
__device__ __forceinline__ float head_w(const FastArgs &p, const float *theta, int j, int u)
{
    if (!p.dueling) return __ldg(theta + p.wh + (int64_t)j * p.N1 + u);
    if (u < p.S) return j == 0 ? __ldg(theta + p.wh + u) : 0.0f;
    return j > 0 ? __ldg(theta + p.wh + (int64_t)j * p.S + (u - p.S)) : 0.0f;
}

// the head weights [J][128] of the unit tile at u0 into shared memory: every load of a thread
// issued before the first store (J <= JPMAX, nt >= 256: at most 8 per thread)
__device__ __forceinline__ void stage_head(const FastArgs &p, const float *theta, int u0, float *Whs, int tid, int nt)
{
    const int n = p.J * 128;
    float v[JPMAX * 128 / 256];
#pragma unroll
    for (int i = 0; i < JPMAX * 128 / 256; ++i) {
        const int e = tid + i * nt;
        v[i] = e < n ? head_w(p, theta, e >> 7, u0 + (e & 127)) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < JPMAX * 128 / 256; ++i) {
        const int e = tid + i * nt;
        if (e < n) Whs[e] = v[i];
    }
}

struct T1Smem {
    int oW1, oA, oWh, ob1, oH, obar, total;
    __host__ __device__ T1Smem(int)
    {
        oW1 = 0;                               // W1 tile: 3 planes x [128 units x 128]
        oA = oW1 + 3 * 128 * N0 * 2;           // H0 ring: T1_SLOTS x 3 planes x [128 x 32]
        oWh = oA + T1_SLOTS * T1_SLOT;         // the tile's head weights: 3 planes x [16 x 128] bf16
        ob1 = oWh + 3 * T1_HN * 128 * 2;       // b1 of the tile [128]
        oH = ob1 + 128 * 4;                    // H1 store staging: per epilogue warp [32 rows][20]
        obar = (oH + T1_EPW * 32 * 20 * 4 + 15) & ~15;   // 15 mbarriers + the TMEM base
        total = obar + 16 * 8;
    }
};
struct T3aSmem {
    int oA, oB, oWh, ored, obar, total;
    __host__ __device__ T3aSmem(int J)
    {
        oA = 0;                                  // dZ1 chunks: 2 stages
        oB = oA + 2 * T3A_STAGE_A;               // H0 chunks: 2 stages
        oWh = oB + 2 * T3A_STAGE_B;              // online head weights of the tile [J][128]
        ored = oWh + J * 128 * 4;                // cross-warp sums [2 row halves][16 groups][8 + 8 JW] + [JPMAX]
        obar = (ored + (2 * 16 * (8 + 8 * JW) + JPMAX) * 4 + 15) & ~15;
        total = obar + 6 * 8;
    }
};
struct T3bSmem {
    int oA, oB, oX, obar, total;
    __host__ __device__ T3bSmem()
    {
        oA = 0;                                  // dZ1 chunks: 2 stages (stage 0 then dZ0)
        oB = oA + 2 * T3B_STAGE_A;               // W1 chunks: 2 stages
        oX = oB + 2 * T3B_STAGE_B;               // [x | 1] image of the tile: 3 x [128 x 32]
        obar = oX + 3 * 128 * XW * 2;
        total = obar + 8 * 8;
    }
};

}  // namespace tcb

// ------------------------------------------------------------------------------------------
// T0: sample, gather, deferred insert, layer 0 (FP32 FMA) -- 16 batch rows per CTA.  Every
// global load a phase needs is in flight at once: W0 / b0 by 16-byte cp.async (waited for only
// before layer 0), a sampled row by one half-warp with 16-byte loads (the whole row, scalars
// included, in one or two loads per lane)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(tcb::T0_T) tcb_l0_kernel(const __grid_constant__ FastArgs p)
{
    using namespace tcb;
    extern __shared__ __align__(16) float sm0[];
    const int D = p.D, B = p.B, tid = threadIdx.x, lane = tid & 31;
    constexpr int XS = 33;   // staged state pitch (>= D + 1, odd: conflict-free)
    float *W0s = sm0;                      // [online | target] W0^T [D][N0]
    float *b0s = W0s + 2 * N0 * D;         // [online | target] [N0]
    float *xs = b0s + 2 * N0;              // [T0_ROWS rows][s, s'][XS]
    __shared__ int32_t idxs[T0_ROWS], pjs[T0_ROWS], pjs2[T0_ROWS];
    // (0) W0^T [D][N0] (kept by K4 / tcb_w1_split_kernel) and b0 of both nets into shared
    // memory, asynchronously (N0 * D and N0 are multiples of 4 floats; b0's blob offset is
    // 16-byte aligned when b0 % 4 == 0)
    for (int c = tid; c < 2 * N0 * D / 4; c += T0_T) cp_async16(W0s + 4 * c, p.w0t + 4 * c);
    if ((p.b0 & 3) == 0) {
        for (int c = tid; c < N0 / 4; c += T0_T) {
            cp_async16(b0s + 4 * c, p.online + p.b0 + 4 * c);
            cp_async16(b0s + N0 + 4 * c, p.target + p.b0 + 4 * c);
        }
    } else {
        for (int e = tid; e < N0; e += T0_T) {
            b0s[e] = __ldg(p.online + p.b0 + e);
            b0s[N0 + e] = __ldg(p.target + p.b0 + e);
        }
    }
    const uint64_t event = p.rctrl[0];
    const uint64_t size = p.pend_k ? p.pend_size : p.rctrl[1];
    const uint64_t cursor = p.pend_k ? (uint64_t)((p.pend_cur + p.pend_k) % p.capacity) : p.rctrl[2];
    const uint64_t nvalid = p.shared ? size - 1 : size;   // reading Q30
    const uint64_t oldest = (p.shared && size == (uint64_t)p.capacity) ? cursor : 0;
    if (p.pend_k && blockIdx.x == 0 && tid == 0) {
        p.rctrl[1] = p.pend_size;
        p.rctrl[2] = cursor;
    }
    const int rb = blockIdx.x * T0_ROWS;
    // (1) batch indices (Q3): Philox call j gives rows 2j and 2j + 1
    auto pend_j = [&](int64_t slot) {
        int64_t j = slot - p.pend_cur;
        if (j < 0) j += p.capacity;
        return j < p.pend_k ? (int)j : -1;
    };
    if (tid < T0_ROWS / 2) {
        int32_t i0 = 0, i1 = 0;
        const int r0 = rb + 2 * tid;
        if (p.bidx) {
            i0 = r0 < B ? p.bidx[r0] : 0;
            i1 = r0 + 1 < B ? p.bidx[r0 + 1] : 0;
        } else if (p.distinct) {
            i0 = r0 < B ? p.idx[r0] : 0;
            i1 = r0 + 1 < B ? p.idx[r0 + 1] : 0;
        } else if (r0 < B) {
            sample_pair(p.seed, p.rank, event, (uint32_t)(r0 / 2), nvalid, i0, i1);
            i0 = slot_of(i0, oldest, p.capacity);
            i1 = slot_of(i1, oldest, p.capacity);
        }
        idxs[2 * tid] = i0;
        idxs[2 * tid + 1] = i1;
        pjs[2 * tid] = pend_j(i0);
        pjs[2 * tid + 1] = pend_j(i1);
        pjs2[2 * tid] = p.shared ? pend_j((i0 + 1) % p.capacity) : -1;
        pjs2[2 * tid + 1] = p.shared ? pend_j((i1 + 1) % p.capacity) : -1;
    }
    __syncthreads();
    // (2) s and s' of the rows (shared states: s' is the next slot's s); a sampled slot
    // of the pending insert is read from the insert's sources
    const bool rvec = !p.shared && (p.rs & 3) == 0 && (reinterpret_cast<uintptr_t>(p.ring) & 15) == 0;
    {
        // half-warp h owns row h: lane l16 loads floats 4 (l16 + 16 i) .. + 3 of the row
        const int r = tid >> 4, l16 = tid & 15, b = rb + r;
        const bool mine = rvec && b < B && pjs[r] < 0;
        const int nv = (p.sw + 3 + 3) >> 2;   // float4s up to the terminal flag
        float4 v[2];
        if (mine) {
            const float4 *row = reinterpret_cast<const float4 *>(p.ring + (int64_t)(p.bidx ? b : idxs[r]) * p.rs);
#pragma unroll
            for (int i = 0; i < 2; ++i)
                if (l16 + 16 * i < nv) v[i] = __ldg(row + l16 + 16 * i);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                if (l16 + 16 * i >= nv) continue;
                const float f[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c = 4 * (l16 + 16 * i) + q;
                    if (c < D) {
                        xs[(r * 2) * XS + c] = f[q];
                    } else if (c < 2 * D) {
                        xs[(r * 2 + 1) * XS + c - D] = f[q];
                    } else if (c == p.sw) {
                        p.a[b] = __float_as_int(f[q]);
                    } else if (c == p.sw + 1) {
                        p.r[b] = f[q];
                    } else if (c == p.sw + 2) {
                        p.done[b] = (uint8_t)(__float_as_uint(f[q]) != 0u);
                    }
                }
            }
        }
    }
    // rows the vector path does not take: shared-state rings, pending slots, rows past B
    for (int e = tid; e < T0_ROWS * 2 * D; e += T0_T) {
        const int r = e / (2 * D), rem = e - r * 2 * D, which = rem / D, dd = rem - which * D;
        const int b = rb + r;
        if (rvec && b < B && pjs[r] < 0) continue;
        float v = 0.0f;
        if (b < B) {
            const bool nxt = which == 1 && p.shared;
            const int j = nxt ? pjs2[r] : pjs[r];
            const int64_t slot = p.bidx ? b : nxt ? (idxs[r] + 1) % p.capacity : idxs[r];
            const int col0 = which == 0 || p.shared ? 0 : D;
            v = j < 0 ? __ldg(p.ring + slot * p.rs + col0 + dd)
                      : (which == 0 || p.shared ? p.pend_s : p.pend_s2)[(int64_t)j * D + dd];
        }
        xs[(r * 2 + which) * XS + dd] = v;
    }
    if (tid < T0_ROWS && rb + tid < B) {
        const int b = rb + tid, j = pjs[tid];
        if (!(rvec && j < 0)) {
            int32_t ra;
            float rr;
            uint32_t rd;
            if (j < 0) {
                const float *row = p.ring + (int64_t)(p.bidx ? b : idxs[tid]) * p.rs + p.sw;
                ra = __float_as_int(__ldg(row));
                rr = __ldg(row + 1);
                rd = __float_as_uint(__ldg(row + 2));
            } else {
                ra = p.pend_a[j];
                rr = p.pend_r[j];
                rd = p.pend_done[j];
            }
            p.a[b] = ra;
            p.r[b] = rr;
            p.done[b] = (uint8_t)(rd != 0u);
        }
        p.idx[b] = idxs[tid];
    }
    cp_async_wait_all();
    __syncthreads();
    // the gathered states of the batch (the learner's batch tensors)
    for (int e = tid; e < T0_ROWS * 2 * D; e += T0_T) {
        const int which = e / (T0_ROWS * D), rem = e - which * T0_ROWS * D, r = rem / D, dd = rem - r * D;
        if (rb + r < B) (which == 0 ? p.Xs : p.Xs2)[(int64_t)(rb + r) * D + dd] = xs[(r * 2 + which) * XS + dd];
    }
    // (3) the [x | 1] image of s (the B operand of T3b's dW0 | db0 MMA), zero past D + 1 and
    // for rows past B
    if (tid < T0_ROWS * (XW / 8)) {
        const int r = tid >> 2, cg = tid & 3, b = rb + r;
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int c = 8 * cg + i;
            x[i] = b < B ? (c < D ? xs[(r * 2) * XS + c] : c == D ? 1.0f : 0.0f) : 0.0f;
        }
        store8(p.ximg, p.xpl, img(b, 8 * cg, XW), x);
    }
    // (4) layer 0 of every net: H0 = ReLU(x W0^T + b0); thread = (row, 8 units)
    {
        const int r = tid % T0_ROWS, g = tid / T0_ROWS, b = rb + r, k0 = 8 * g;
        const bool ok = b < B;
        for (int net = 0; net < p.nets; ++net) {
            const float *x = xs + (r * 2 + (net == 0 ? 0 : 1)) * XS;
            const float *W = W0s + (net == 1 ? N0 * D : 0) + k0;
            const float *bb = b0s + (net == 1 ? N0 : 0);
            float h[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) h[i] = bb[k0 + i];
            for (int dd = 0; dd < D; ++dd) {
                const float xv = x[dd];
                const float4 wa = *reinterpret_cast<const float4 *>(W + dd * N0);
                const float4 wb = *reinterpret_cast<const float4 *>(W + dd * N0 + 4);
                const float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) h[i] = fmaf(w[i], xv, h[i]);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) h[i] = ok ? fmaxf(h[i], 0.0f) : 0.0f;
            // T1's A operand (tile-quarter blocks), and T3a's B operand for the online net on s
            store8(p.h0img + (int64_t)net * 3 * p.h0pl, p.h0pl, qimg(b, k0), h);
            if (net == 0) store8(p.h0img + (int64_t)p.nets * 3 * p.h0pl, p.h0pl, img(b, k0, N0), h);
            if (net == 0 && ok) {
                float *ho = p.H0 + (int64_t)b * N0 + k0;
                *reinterpret_cast<float4 *>(ho) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4 *>(ho + 4) = make_float4(h[4], h[5], h[6], h[7]);
            }
        }
    }
    // (5) the deferred insert's rows into the ring: no sampled read of this step goes
    // to a pending slot's ring row (those read the insert's sources), so the order is free
    if (p.pend_k)
        for (int64_t j = (int64_t)blockIdx.x * (T0_T / 32) + (tid >> 5); j < p.pend_k; j += (int64_t)gridDim.x * (T0_T / 32))
            ring_write_row(p.ring + ((p.pend_cur + j) % p.capacity) * p.rs, p.rs, D, p.sw, lane, j, p.pend_s,
                           p.pend_a, p.pend_r, p.pend_s2, p.pend_done, p.pend_err);
}

// ------------------------------------------------------------------------------------------
// T1: layer 1 + head partials, persistent per (net, 128-unit tile); CTAs c, c + ncombo, ...
// share a combo and take its batch tiles bt0, bt0 + cpc, ...
// TMEM: two 128-column accumulators.  Barriers: wbar (W1 tile), full / empty [T1_SLOTS]
// (H0 ring), accf / acce [2] (accumulator written / drained).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(tcb::T1_T, 1) tcb_fwd_kernel(const __grid_constant__ FastArgs p)
{
    using namespace tcb;
    extern __shared__ __align__(1024) char smc[];
    const int N1 = p.N1, B = p.B, J = p.J;
    const T1Smem L(J);
    char *W1s = smc + L.oW1, *As = smc + L.oA;
    char *Whs = smc + L.oWh;
    float *b1s = reinterpret_cast<float *>(smc + L.ob1);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smc + L.obar);
    uint64_t *wbar = bar, *full = bar + 1, *empty = bar + 1 + T1_SLOTS, *accf = bar + 1 + 2 * T1_SLOTS,
             *acce = accf + 2, *hready = acce + 2, *hdone = hready + 1;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 15);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nut = N1 / 128, ncombo = p.nets * nut;
    const int combo = blockIdx.x % ncombo, cpc = gridDim.x / ncombo, bt0 = blockIdx.x / ncombo;
    const int net = combo / nut, ut = combo % nut, u0 = ut * 128;
    const int nbt = p.Bp / 128, nq = N0 / 32;
    const int ntile = bt0 < nbt ? (nbt - bt0 + cpc - 1) / cpc : 0;
    // RPL_TRACE: per-CTA cycle totals (kernel slot 4): 2 MMA thread waiting for H0 slots, 3 MMA
    // thread waiting for a drained accumulator, 4 epilogue waiting for an accumulator, 5
    // epilogue work per tile, 6 producer waiting for a free slot
    CtaTrace tr_(p.trace, 4);
    const int mma_tid = 32 * (T1_EPW + 1), prod_tid = 32 * T1_EPW;
    if (warp == 0) umma::tmem_alloc(tslot, 512);
    if (tid == 0) {
        umma::mbar_init(hready, T1_EPW);
        umma::mbar_init(hdone, 1);
        umma::mbar_init(wbar, 1);
        for (int i = 0; i < T1_SLOTS; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&accf[i], 1);
            umma::mbar_init(&acce[i], T1_EPW);
        }
        umma::fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = *tslot;
    const uint16_t *h0 = p.h0img + (int64_t)net * 3 * p.h0pl;
    const uint16_t *w1 = p.w1img + (net == 1 ? 3 * p.w1pl : 0);   // the target's image for net 1
    const float *theta = net == 1 ? p.target : p.online;
    if (warp == T1_EPW) {
        // ---- producer: the W1 tile once, then the H0 quarters through the ring -------------
        if (lane == 0) {
            umma::mbar_expect_tx(wbar, 3 * 128 * N0 * 2);
            for (int pl = 0; pl < 3; ++pl)
                umma::bulk_g2s(W1s + pl * 128 * N0 * 2, w1 + pl * p.w1pl + (int64_t)u0 * N0, 128 * N0 * 2, wbar);
        }
        for (int n = 0; n < ntile * nq; ++n) {
            const int it = n / nq, q = n - it * nq, bt = bt0 + it * cpc, slot = n % T1_SLOTS;
            long long t0 = tr_.now_by(prod_tid);
            if (n >= T1_SLOTS) umma::mbar_wait(&empty[slot], (uint32_t)(((n / T1_SLOTS) - 1) & 1));
            tr_.acc_by(prod_tid, 6, t0);
            if (lane == 0) umma::mbar_expect_tx(&full[slot], T1_SLOT);
            __syncwarp();
            char *dst = As + slot * T1_SLOT;
            // a (tile, K quarter) block of the H0 image is one contiguous 8 KB piece per plane
            if (lane < 3)
                umma::bulk_g2s(dst + lane * (128 * 32 * 2), h0 + lane * p.h0pl + qimg((int64_t)bt * 128, 32 * q),
                               128 * 32 * 2, &full[slot]);
        }
    } else if (warp == T1_EPW + 1) {
        // ---- MMA issue ------------------------------------------------------------------------
        if (lane == 0) {
            const uint32_t id = umma::idesc_bf16(128, 128, false, false);
            const uint32_t idh = umma::idesc_bf16(128, T1_HN, false, false);
            const bool fp32 = p.prec != RPL_PREC_BF16;
            // the head contraction of tile t: D_head[b][j] = sum_u H1[b][u] W_head[j][u]
            // (M = 128 samples, N = 16 outputs, K = 128 units; A = the H1 planes the epilogue
            // wrote into tensor memory, B = the tile's head-weight image)
            auto head = [&](int t) {
                tcb::wait(hready, (uint32_t)(t & 1));
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    uint32_t ad[3];
                    uint64_t bd[3];
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl) {
                        ad[pl] = tb + (uint32_t)(T1_TM_AH + 64 * pl + 8 * ks);
                        bd[pl] = umma::desc(Whs + pl * (T1_HN * 128 * 2) + ks * 2 * 128, 128, (128 / 8) * 128);
                    }
                    mma6_ts(tb + T1_TM_DH, ad, bd, idh, ks > 0, fp32);
                }
                umma::commit(hdone);
            };
            tcb::wait(wbar, 0);
            for (int it = 0; it < ntile; ++it) {
                const int acc = it & 1;
                long long t0 = tr_.now_by(mma_tid);
                if (it >= 2) tcb::wait(&acce[acc], (uint32_t)(((it >> 1) - 1) & 1));
                tr_.acc_by(mma_tid, 3, t0);
                const uint32_t dcol = tb + (uint32_t)(acc * 128);
                for (int q = 0; q < nq; ++q) {
                    const int n = it * nq + q, slot = n % T1_SLOTS;
                    long long t1 = tr_.now_by(mma_tid);
                    tcb::wait(&full[slot], (uint32_t)((n / T1_SLOTS) & 1));
                    tr_.acc_by(mma_tid, 2, t1);
                    const char *a = As + slot * T1_SLOT;
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        uint64_t ad[3], bd[3];
#pragma unroll
                        for (int pl = 0; pl < 3; ++pl) {
                            ad[pl] = umma::desc(a + pl * (128 * 32 * 2) + s * 256, 128, 512);
                            bd[pl] = umma::desc(W1s + pl * 128 * N0 * 2 + ((32 * q + 16 * s) >> 3) * 128, 128,
                                                (N0 / 8) * 128);
                        }
                        mma6(dcol, ad, bd, id, q > 0 || s > 0, fp32);
                    }
                    umma::commit(&empty[slot]);
                }
                umma::commit(&accf[acc]);
                if (it >= 1) head(it - 1);
            }
            if (ntile > 0) head(ntile - 1);
        }
    } else {
        // ---- epilogue (warps 0 .. T1_EPW-1): warp w reads TMEM lane quarter w % 4, columns
        // T1_CPW (w / 4) ...: bias, ReLU, H1 of the online net; H1's bf16 planes into tensor
        // memory for the head MMA; the previous tile's head sums out as partials
        if (tid < T1_HN * 16) {   // the tile's head-weight image (rows j < J of head_w, zero
            // where unit u does not feed j and for the padding rows): thread = (output j, 8
            // consecutive units)
            const int j = tid >> 4, ug = tid & 15;
            float w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = j < J ? head_w(p, theta, j, u0 + 8 * ug + i) : 0.0f;
            store8_smem(Whs, T1_HN * 128 * 2, (int)img(j, 8 * ug, 128) * 2, w);
        }
        for (int c = tid; c < 128; c += 32 * T1_EPW) b1s[c] = __ldg(theta + p.b1 + u0 + c);
        umma::fence_async_smem();   // the head image is read by the tensor cores
        epi_sync(32 * T1_EPW);
        const int quarter = warp & 3, half = warp >> 2, nps = (N1 / 128) * T1_PSL;
        // the head sums of tile t (its D_head, complete) -> this row's partials
        auto head_out = [&](int t) {
            tcb::wait(hdone, (uint32_t)(t & 1));
            uint32_t dh[16];
            ld16(lane_addr(tb + T1_TM_DH, quarter, 0), dh);
            wait_ld();
            const int b = (bt0 + t * cpc) * 128 + 32 * quarter + lane;
            if (half == 0 && b < B) {
                float *po = p.part + (((int64_t)net * nps + ut) * B + b) * J;
#pragma unroll
                for (int j = 0; j < T1_HN; ++j)
                    if (j < J) po[j] = __uint_as_float(dh[j]);
            }
        };
        for (int it = 0; it < ntile; ++it) {
            const int acc = it & 1, bt = bt0 + it * cpc, b = bt * 128 + 32 * quarter + lane;
            long long t0 = tr_.now();
            tcb::wait(&accf[acc], (uint32_t)((it >> 1) & 1));
            tr_.acc(4, t0);
            t0 = tr_.now();
            uint32_t v[T1_CPW / 16][16];
#pragma unroll
            for (int c = 0; c < T1_CPW / 16; ++c) ld16(lane_addr(tb + (uint32_t)(acc * 128), quarter, T1_CPW * half + 16 * c), v[c]);
            wait_ld();
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[acc]);   // accumulator drained into registers
            uint32_t pk[3][T1_CPW / 2];               // H1 planes, two bf16 per word
#pragma unroll
            for (int c = 0; c < T1_CPW / 16; ++c) {
                const int c0 = T1_CPW * half + 16 * c;
                float h[16], bb[16];
                // 16-byte shared loads (broadcast: every lane of the warp reads the same words)
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 t = *reinterpret_cast<const float4 *>(b1s + c0 + i);
                    bb[i] = t.x; bb[i + 1] = t.y; bb[i + 2] = t.z; bb[i + 3] = t.w;
                }
#pragma unroll
                for (int i = 0; i < 16; ++i) h[i] = fmaxf(__uint_as_float(v[c][i]) + bb[i], 0.0f);
#ifndef RPL_T1_NOH1   // (timing experiment only: results invalid without H1)
                if (net == 0) {
#else
                if (net < 0) {
#endif
                    // H1 of the online net (T3a's input): the warp's 32 rows x 16 columns go
                    // through shared memory so every global store is a whole 64-byte row
                    // segment (8 rows per instruction) instead of a 16-byte piece of 32 rows
                    float *st = reinterpret_cast<float *>(smc + L.oH) + warp * (32 * 20);
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        *reinterpret_cast<float4 *>(st + lane * 20 + i) = make_float4(h[i], h[i + 1], h[i + 2], h[i + 3]);
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int rr = 8 * i + (lane >> 2), c4 = lane & 3;
                        const int bb2 = bt * 128 + 32 * quarter + rr;
                        const float4 t = *reinterpret_cast<const float4 *>(st + rr * 20 + 4 * c4);
                        if (bb2 < B) *reinterpret_cast<float4 *>(p.H1 + (int64_t)bb2 * N1 + u0 + c0 + 4 * c4) = t;
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int i = 0; i < 16; i += 2)
                    umma::split3_pack2(h[i], h[i + 1], pk[0][8 * c + i / 2], pk[1][8 * c + i / 2], pk[2][8 * c + i / 2]);
            }
            // the previous tile's head MMAs have read the A planes and written D_head
            if (it >= 1) head_out(it - 1);
#pragma unroll
            for (int pl = 0; pl < 3; ++pl)
#pragma unroll
                for (int c = 0; c < T1_CPW / 32; ++c)
                    st16(lane_addr(tb + (uint32_t)(T1_TM_AH + 64 * pl), quarter, (T1_CPW / 2) * half + 16 * c),
                         &pk[pl][16 * c]);
            wait_st();
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(hready);
            tr_.acc(5, t0);
        }
        if (ntile > 0) head_out(ntile - 1);
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tb, 512);
}

// ------------------------------------------------------------------------------------------
// TD: a warp per sample: head sums (bias + the N1 / 64 partials in order), td_warp (dueling
// combine, target, Huber, dHead), dHead padded to jp words per row
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) tcb_td_kernel(const __grid_constant__ FastArgs p)
{
    // the partials of the CTA's 8 consecutive samples: for each (net, unit half-tile q) the
    // 8 x J words are contiguous in p.part (T1 writes [net][q][b][j]), so the CTA loads them
    // with coalesced loads, 8 in flight per thread, into raw[net][q][8][J]
    extern __shared__ float raw[];
    __shared__ float hs[8][3 * (F_MAXJ + 1)];
    __shared__ float dhs[8][F_MAXJ + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t t = *p.step_dev + 1;
        *p.sync_flag = (p.sync_period > 0 && t % p.sync_period == 0) ? 1 : 0;
    }
    const int J = p.J, B = p.B, nut2 = (p.N1 / 128) * tcb::T1_PSL, b0 = blockIdx.x * 8;
    const int nb = min(8, B - b0), span = nb * J, nseg = p.nets * nut2, n = nseg * span;
    // the sample's action / reward / terminal and the head biases, requested with the partials
    const int b = b0 + warp;
    const bool live = b < B;
    const int ab = live ? p.a[b] : 0;
    const float rb = live ? p.r[b] : 0.0f;
    const uint8_t db = live ? p.done[b] : 0;
    float bias[3];
#pragma unroll
    for (int net = 0; net < 3; ++net)
        bias[net] = (net < p.nets && lane < J) ? __ldg((net == 1 ? p.target : p.online) + p.bh + lane) : 0.0f;
#pragma unroll 8
    for (int e = threadIdx.x; e < n; e += 256) {
        const int seg = e / span, w = e - seg * span;
        raw[seg * 8 * J + w] = __ldcg(p.part + ((int64_t)seg * B + b0) * J + w);
    }
    __syncthreads();
    if (!live) return;
#pragma unroll
    for (int net = 0; net < 3; ++net) {
        if (net < p.nets && lane < J) {
            // bias, then the partials in unit-tile order
            const float *src = raw + (int64_t)net * nut2 * 8 * J + warp * J + lane;
            float v = bias[net];
            for (int q = 0; q < nut2; ++q) v += src[q * 8 * J];
            hs[warp][net * (F_MAXJ + 1) + lane] = v;
        }
    }
    __syncwarp();
    td_warp(p, hs[warp], F_MAXJ + 1, ab, rb, db, b, lane, dhs[warp]);
    __syncwarp();
    if (lane < p.jp) p.dheadp[(int64_t)b * p.jp + lane] = lane < J ? dhs[warp][lane] : 0.0f;
}
inline size_t tcb_td_smem(int nets, int N1, int J) { return (size_t)nets * (N1 / 128) * tcb::T1_PSL * 8 * J * sizeof(float); }

// ------------------------------------------------------------------------------------------
// T3a: per (128-unit tile ut, chunk group g): 64-row chunks c = g, g + G, ... of the batch.
// Per chunk: all threads form dZ1[b][u] (thread = 8 rows of one 8-unit column group per
// pass) into the stage's A image and straight into the global dZ1 image (T3b, dzimg blocks);
// thread 0 issues dW1 += dZ1^T H0 (M = units, N = 128, K = 64 samples; both MN-major).
// Partials -> gpart[g] (dW1, db1, dW_head of the tile; db_head from ut == 0).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(tcb::T3A_T, 1) tcb_dw1_kernel(const __grid_constant__ FastArgs p)
{
    using namespace tcb;
    extern __shared__ __align__(1024) char smc[];
    const int N1 = p.N1, B = p.B, J = p.J, jp = p.jp;
    const T3aSmem L(J);
    float *Whs = reinterpret_cast<float *>(smc + L.oWh), *red = reinterpret_cast<float *>(smc + L.ored);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smc + L.obar);
    uint64_t *full = bar, *mfree = bar + 2, *mdone = bar + 4;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 5);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nut = N1 / 128, ut = blockIdx.x % nut, g = blockIdx.x / nut, G = gridDim.x / nut;
    // RPL_TRACE: thread 0's cycle totals (kernel slot 5): 2 chunk start (stage free + barrier),
    // 3 the four dZ1 passes, 4 the barrier after them, 5 waiting for the H0 chunk (MMA issue)
    CtaTrace tr_(p.trace, 5);
    const int u0 = ut * 128, nch = p.Bp / 64;
    if (warp == 0) umma::tmem_alloc(tslot, 128);
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&mfree[i], 1);
        }
        umma::mbar_init(mdone, 1);
        umma::fence_mbar_init();
    }
    stage_head(p, p.online, u0, Whs, tid, T3A_T);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = *tslot;
    int jlo, jhi;
    head_range(p, u0, jlo, jhi);
    const int r8 = lane & 7, cg = 4 * (warp & 3) + (lane >> 3), rh = warp >> 2;
    const bool fp32 = p.prec != RPL_PREC_BF16;
    const uint32_t id = umma::idesc_bf16(128, N0, true, true);
    float db1[8], wacc[JW][8], bha[JPMAX];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        db1[i] = 0.0f;
#pragma unroll
        for (int j = 0; j < JW; ++j) wacc[j][i] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < JPMAX; ++j) bha[j] = 0.0f;
    // the H1 / dHead rows of pass (chunk c, pass ps) -- loaded one pass ahead, so the next
    // pass's (and across chunks, the next chunk's first pass's) L2 loads are in flight while
    // this pass computes
    auto load_pass = [&](int c, int ps, float (&h1)[8], float (&dh)[JPMAX]) {
        const int b = 64 * c + 16 * ps + 8 * rh + r8;
        if (c < nch && b < B) {
            const float4 *hp = reinterpret_cast<const float4 *>(p.H1 + (int64_t)b * N1 + u0 + 8 * cg);
            const float4 x0 = __ldcg(hp), x1 = __ldcg(hp + 1);
            h1[0] = x0.x; h1[1] = x0.y; h1[2] = x0.z; h1[3] = x0.w;
            h1[4] = x1.x; h1[5] = x1.y; h1[6] = x1.z; h1[7] = x1.w;
#pragma unroll
            for (int q = 0; q < JPMAX / 4; ++q) {
                float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
                if (4 * q < jp) t = __ldcg(reinterpret_cast<const float4 *>(p.dheadp + (int64_t)b * jp) + q);
                dh[4 * q] = t.x; dh[4 * q + 1] = t.y; dh[4 * q + 2] = t.z; dh[4 * q + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) h1[k] = 0.0f;
#pragma unroll
            for (int j = 0; j < JPMAX; ++j) dh[j] = 0.0f;
        }
    };
    // two passes of loads in flight: (h1n, dhn) for the next pass, (h1m, dhm) for the one after
    float h1n[8], dhn[JPMAX], h1m[8], dhm[JPMAX];
    load_pass(g, 0, h1n, dhn);
    load_pass(g, 1, h1m, dhm);
    int i = 0;
#ifndef RPL_T3A_EPI_TRACE
    tr_.mark(6);   // setup done (cycles since the CTA started; overwritten per step)
#endif
    for (int c = g; c < nch; c += G, ++i) {
        const int s = i & 1;
        char *Ast = smc + L.oA + s * T3A_STAGE_A, *Bst = smc + L.oB + s * T3A_STAGE_B;
        long long t0 = tr_.now();
        if (i >= 2) umma::mbar_wait(&mfree[s], (uint32_t)(((i >> 1) - 1) & 1));   // chunk i - 2's MMAs
        __syncthreads();
        tr_.acc(2, t0);
        t0 = tr_.now();
        umma::fence_after_sync();
        if (tid == 0) {
            umma::mbar_expect_tx(&full[s], T3A_STAGE_B);
            for (int pl = 0; pl < 3; ++pl)
                umma::bulk_g2s(Bst + pl * (64 * N0 * 2), p.h0img + ((int64_t)p.nets * 3 + pl) * p.h0pl + (int64_t)c * 64 * N0, 64 * N0 * 2,
                               &full[s]);
        }
#pragma unroll 1
        for (int ps = 0; ps < 4; ++ps) {
            const int rr = 16 * ps + 8 * rh + r8;
            float h1[8], dh[JPMAX];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                h1[k] = h1n[k];
                h1n[k] = h1m[k];
            }
#pragma unroll
            for (int j = 0; j < JPMAX; ++j) {
                dh[j] = dhn[j];
                dhn[j] = dhm[j];
            }
            if (ps < 2) load_pass(c, ps + 2, h1m, dhm);
            else load_pass(c + G, ps - 2, h1m, dhm);
            // the tile's head outputs start at jlo (0 or 1, head_range)
            float dsel[JW];
#pragma unroll
            for (int j = 0; j < JW; ++j) dsel[j] = jlo ? dh[j + 1] : dh[j];
            float dz[8], gs[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) gs[k] = 0.0f;
            // head weights of the 8 units, two 16-byte shared loads per output
#pragma unroll
            for (int j = 0; j < JW; ++j)
                if (jlo + j < jhi) {
                    const float4 *w4 = reinterpret_cast<const float4 *>(Whs + (jlo + j) * 128 + 8 * cg);
                    const float4 wa = w4[0], wb = w4[1];
                    const float w[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        gs[k] = fmaf(dsel[j], w[k], gs[k]);
                        wacc[j][k] = fmaf(dsel[j], h1[k], wacc[j][k]);
                    }
                }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                dz[k] = h1[k] > 0.0f ? gs[k] : 0.0f;
                db1[k] += dz[k];
            }
            if (cg == 0) {
#pragma unroll
                for (int j = 0; j < JPMAX; ++j) bha[j] += dh[j];
            }
            // the stage's A image, and straight into the global dZ1 image T3b reads (8 lanes
            // write one 128-byte core matrix per plane); one split for both
            {
                uint4 zh, zm, zl;
                split8(dz, zh, zm, zl);
                char *sa = Ast + (rr >> 3) * 2048 + cg * 128 + (rr & 7) * 16;
                *reinterpret_cast<uint4 *>(sa) = zh;
                *reinterpret_cast<uint4 *>(sa + 64 * 128 * 2) = zm;
                *reinterpret_cast<uint4 *>(sa + 2 * 64 * 128 * 2) = zl;
                uint16_t *g = p.dz1img + dzimg(64 * (int64_t)c + rr, u0 + 8 * cg, N1);
                *reinterpret_cast<uint4 *>(g) = zh;
                *reinterpret_cast<uint4 *>(g + p.dzpl) = zm;
                *reinterpret_cast<uint4 *>(g + 2 * p.dzpl) = zl;
            }
        }
        tr_.acc(3, t0);
        t0 = tr_.now();
        umma::fence_async_smem();
        __syncthreads();
        tr_.acc(4, t0);
        if (tid == 0) {
            long long t1 = tr_.now();
            tcb::wait(&full[s], (uint32_t)((i >> 1) & 1));
            tr_.acc(5, t1);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint64_t ad[3], bd[3];
#pragma unroll
                for (int pl = 0; pl < 3; ++pl) {
                    ad[pl] = umma::desc(Ast + pl * (64 * 128 * 2) + ks * 2 * 2048, 2048, 128);
                    bd[pl] = umma::desc(Bst + pl * (64 * N0 * 2) + ks * 2 * (N0 / 8) * 128, (N0 / 8) * 128, 128);
                }
                mma6(tb, ad, bd, id, i > 0 || ks > 0, fp32);
            }
            umma::commit(&mfree[s]);
        }
    }
    if (tid == 0) umma::commit(mdone);
#ifndef RPL_T3A_EPI_TRACE
    tr_.mark(7);   // chunk loop done
#else
    tr_.mark(5);   // (epilogue trace build: 5 loop done, 6 shuffles done, 7 partial writes done)
#endif
    // the tile's db1 / dW_head / db_head: sums over the 8 rows of a lane group (shuffles), then
    // over the two row halves (shared memory), in a fixed order
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            db1[k] += __shfl_xor_sync(0xffffffffu, db1[k], o);
#pragma unroll
            for (int j = 0; j < JW; ++j) wacc[j][k] += __shfl_xor_sync(0xffffffffu, wacc[j][k], o);
        }
#pragma unroll
        for (int j = 0; j < JPMAX; ++j) bha[j] += __shfl_xor_sync(0xffffffffu, bha[j], o);
    }
#ifdef RPL_T3A_EPI_TRACE
    tr_.mark(6);
#endif
    // both row halves' lane-group sums into shared memory, then every thread writes whole
    // coalesced runs of the tile's db1 / dW_head (row half 0 + row half 1, the former order)
    constexpr int RW = 8 + 8 * JW;
    float *red1 = red + 16 * RW + JPMAX;   // row half 0 (red: row half 1, then db_head)
    if (r8 == 0) {
        float *rp = (rh == 1 ? red : red1) + cg * RW;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            rp[k] = db1[k];
#pragma unroll
            for (int j = 0; j < JW; ++j) rp[8 + 8 * j + k] = wacc[j][k];
        }
        if (rh == 1 && cg == 0)
#pragma unroll
            for (int j = 0; j < JPMAX; ++j) red[16 * RW + j] = bha[j];
    }
    __syncthreads();
    float *gp = p.gpart + (int64_t)g * p.gps;
    for (int o = tid; o < 128 * (1 + JW); o += T3A_T) {
        const int ul = o & 127, sl = o >> 7, cgo = ul >> 3, k = ul & 7, u = u0 + ul;
        const int idx = sl == 0 ? k : 8 + 8 * (sl - 1) + k;
        const float v = red1[cgo * RW + idx] + red[cgo * RW + idx];
        if (sl == 0) {
            gp[p.b1 + u] = v;
        } else {
            const int jj = jlo + sl - 1;
            if (jj >= jhi) continue;
            int64_t off;
            if (!p.dueling) off = (int64_t)jj * N1 + u;
            else if (jj == 0) off = u;
            else off = (int64_t)jj * p.S + (u - p.S);
            gp[p.wh + off] = v;
        }
    }
    if (tid == 0 && ut == 0)   // db_head: row half 0's group 0 sums (registers of thread 0) + row half 1's
        for (int j = 0; j < J; ++j) gp[p.bh + j] = bha[j] + red[16 * RW + j];
#ifdef RPL_T3A_EPI_TRACE
    tr_.mark(7);
#endif
    // dW1 of the tile: TMEM lane = unit, column = layer-0 unit; warps w, w + 4 split the columns
    tcb::wait(mdone, 0);
    {
        const int quarter = warp & 3, half = warp >> 2, u = u0 + 32 * quarter + lane;
        float *dst = gp + p.w1 + (int64_t)u * N0 + 64 * half;
        uint32_t v[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c) ld16(lane_addr(tb, quarter, 64 * half + 16 * c), v[c]);
        wait_ld();
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int k = 0; k < 16; k += 4)
                *reinterpret_cast<float4 *>(dst + 16 * c + k) =
                    make_float4(__uint_as_float(v[c][k]), __uint_as_float(v[c][k + 1]), __uint_as_float(v[c][k + 2]),
                                __uint_as_float(v[c][k + 3]));
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tb, 128);
}

// ------------------------------------------------------------------------------------------
// T3b: per (128-row batch tile bt, unit split q): dH0 = sum_u dZ1[b][u] W1[u][k] over the
// split's 64-unit chunks (A = dZ1 K-major, B = W1 MN-major; warp 1 produces, thread 0 of
// warp 0 issues), then dZ0 = dH0 * [H0 > 0] into shared memory and its [dW0 | db0] share
// dZ0^T [x | 1] (M = 128 layer-0 units, N = 32, K = 128 samples) -> w0part[q * nbt + bt].
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(tcb::T3B_T, 1) tcb_dh0_kernel(const __grid_constant__ FastArgs p)
{
    using namespace tcb;
    extern __shared__ __align__(1024) char smc[];
    const int N1 = p.N1, B = p.B, D = p.D;
    const T3bSmem L;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smc + L.obar);
    uint64_t *full = bar, *mfree = bar + 2, *xbar = bar + 4, *mdone = bar + 5, *mdone2 = bar + 6;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 7);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nbt = p.Bp / 128, bt = blockIdx.x % nbt, q = blockIdx.x / nbt, NQ = gridDim.x / nbt;
    const int UQ = N1 / NQ, nck = UQ / 64;
    if (warp == 0) umma::tmem_alloc(tslot, 256);
    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&mfree[i], 1);
        }
        umma::mbar_init(xbar, 1);
        umma::mbar_init(mdone, 1);
        umma::mbar_init(mdone2, 1);
        umma::fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = *tslot;
    const bool fp32 = p.prec != RPL_PREC_BF16;
    char *Xs = smc + L.oX;
    // this thread's H0 row (sample bt * 128 + tid: the ReLU mask of dZ0), loaded now so the
    // L2 round trips overlap the dH0 main loop
    float4 h0r[N0 / 4];
    {
        const int b = bt * 128 + tid;
        const float4 *h0 = reinterpret_cast<const float4 *>(p.H0 + (int64_t)b * N0);
#pragma unroll
        for (int i = 0; i < N0 / 4; ++i) h0r[i] = b < B ? __ldcg(h0 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (warp == 1) {
        // ---- producer ------------------------------------------------------------------------
        if (lane == 0) {
            umma::mbar_expect_tx(xbar, 3 * 128 * XW * 2);
            for (int pl = 0; pl < 3; ++pl)
                umma::bulk_g2s(Xs + pl * (128 * XW * 2), p.ximg + pl * p.xpl + (int64_t)bt * 128 * XW, 128 * XW * 2, xbar);
        }
        for (int i = 0; i < nck; ++i) {
            const int s = i & 1, uc = q * UQ + 64 * i;
            if (i >= 2) umma::mbar_wait(&mfree[s], (uint32_t)(((i >> 1) - 1) & 1));
            if (lane == 0) umma::mbar_expect_tx(&full[s], T3B_STAGE_A + T3B_STAGE_B);
            __syncwarp();
            char *A = smc + L.oA + s * T3B_STAGE_A, *Bq = smc + L.oB + s * T3B_STAGE_B;
            if (lane < 3) {   // the (tile, 64-unit chunk) block of dZ1: one 16 KB piece per plane
                umma::bulk_g2s(A + lane * (128 * 64 * 2), p.dz1img + lane * p.dzpl + dzimg((int64_t)bt * 128, uc, N1),
                               128 * 64 * 2, &full[s]);
            } else if (lane < 6) {   // W1 rows [uc, uc + 64) of the online net
                const int pl = lane - 3;
                umma::bulk_g2s(Bq + pl * (64 * N0 * 2), p.w1img + pl * p.w1pl + (int64_t)uc * N0, 64 * N0 * 2, &full[s]);
            }
        }
    } else if (warp == 0 && lane == 0) {
        // ---- MMA issue: dH0 (M = 128 samples, N = 128, K = 64 units per chunk) ---------------
        const uint32_t id = umma::idesc_bf16(128, N0, false, true);
        for (int i = 0; i < nck; ++i) {
            const int s = i & 1;
            tcb::wait(&full[s], (uint32_t)((i >> 1) & 1));
            const char *A = smc + L.oA + s * T3B_STAGE_A, *Bq = smc + L.oB + s * T3B_STAGE_B;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint64_t ad[3], bd[3];
#pragma unroll
                for (int pl = 0; pl < 3; ++pl) {
                    ad[pl] = umma::desc(A + pl * (128 * 64 * 2) + ks * 256, 128, 1024);
                    bd[pl] = umma::desc(Bq + pl * (64 * N0 * 2) + ks * 2 * (N0 / 8) * 128, (N0 / 8) * 128, 128);
                }
                mma6(tb, ad, bd, id, i > 0 || ks > 0, fp32);
            }
            umma::commit(&mfree[s]);
        }
        umma::commit(mdone);
    }
    __syncwarp();
    tcb::wait(mdone, 0);
    // ---- dZ0 of the tile (thread = sample row = TMEM lane) into an MN-major image ----------
    char *Z = smc + L.oA;   // stage 0 and 1 of A: 3 planes x [128 x 128]
    {
        const int r = tid;
#pragma unroll
        for (int c0 = 0; c0 < N0; c0 += 16) {
            uint32_t v[16];
            ld16(lane_addr(tb, warp, c0), v);
            float hm[16];
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
                const float4 t = h0r[(c0 + i) >> 2];
                hm[i] = t.x; hm[i + 1] = t.y; hm[i + 2] = t.z; hm[i + 3] = t.w;
            }
            wait_ld();
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                float z[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) z[i] = hm[8 * hf + i] > 0.0f ? __uint_as_float(v[8 * hf + i]) : 0.0f;
                store8_smem(Z, 128 * N0 * 2, (r >> 3) * (N0 / 8) * 128 + ((c0 >> 3) + hf) * 128 + (r & 7) * 16, z);
            }
        }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
        umma::fence_after_sync();
        tcb::wait(xbar, 0);
        const uint32_t id = umma::idesc_bf16(128, XW, true, true);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            uint64_t ad[3], bd[3];
#pragma unroll
            for (int pl = 0; pl < 3; ++pl) {
                ad[pl] = umma::desc(Z + pl * (128 * N0 * 2) + ks * 2 * (N0 / 8) * 128, (N0 / 8) * 128, 128);
                bd[pl] = umma::desc(Xs + pl * (128 * XW * 2) + ks * 2 * (XW / 8) * 128, (XW / 8) * 128, 128);
            }
            mma6(tb + 128, ad, bd, id, ks > 0, fp32);
        }
        umma::commit(mdone2);
    }
    __syncwarp();
    tcb::wait(mdone2, 0);
    {
        const int k = tid;   // TMEM lane = layer-0 unit
        uint32_t v[2][16];
        ld16(lane_addr(tb + 128, warp, 0), v[0]);
        ld16(lane_addr(tb + 128, warp, 16), v[1]);
        wait_ld();
        float *w0p = p.w0part + (int64_t)(q * nbt + bt) * p.w1;
        for (int dd = 0; dd < D; ++dd) w0p[(int64_t)k * D + dd] = __uint_as_float(v[dd >> 4][dd & 15]);
        w0p[(int64_t)N0 * D + k] = __uint_as_float(v[D >> 4][D & 15]);
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tb, 256);
}

// the bf16 image of W1 (online and target) from the fp32 weights: after create, set_params,
// sync_target and any update that is not K4's
__global__ void __launch_bounds__(256) tcb_w1_split_kernel(const float *__restrict__ w1, uint16_t *__restrict__ im,
                                                           int64_t plane, int N1, const float *__restrict__ w0,
                                                           float *__restrict__ w0t, int D)
{
    using namespace tcb;
    // W0 transposed ([D][N0], T0's layer-0 operand)
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)N0 * D; e += (int64_t)gridDim.x * blockDim.x) {
        const int u = (int)(e / D), dd = (int)(e - (int64_t)u * D);
        w0t[(int64_t)dd * N0 + u] = w0[e];
    }
    const int64_t n8 = (int64_t)N1 * N0 / 8;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = e / (N0 / 8);
        const int k = 8 * (int)(e % (N0 / 8));
        float x[8];
        const float4 a = *reinterpret_cast<const float4 *>(w1 + u * N0 + k);
        const float4 c = *reinterpret_cast<const float4 *>(w1 + u * N0 + k + 4);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = c.x; x[5] = c.y; x[6] = c.z; x[7] = c.w;
        store8(im, plane, img(u, k, N0), x);
    }
}

}  // namespace rpl
