// tc_fast.cuh -- the fast path's contractions on the 5th-generation tensor cores (tcgen05
// kind::tf32, fp32 accumulators in tensor memory), for the two-trunk-layer nets of the fast path
// (the paper's dueling net 27 -> 128 -> [V 512 | A 512] -> 1 + |A|; the plain
// 27 -> 64 -> 64 -> |A| MLP of configs[0]).  CUDA path only; FastArgs / K2 / K4 in
// train_fast.cuh.
//
//   K1 tc_fwd_kernel : per (net, 128-row batch tile, unit tile of UN layer-1 units), 128 threads
//       (thread t <-> batch row t <-> TMEM lane t):
//         Philox sample + gather of the tile's rows -> X (tf32 hi / lo planes, shared memory)
//         layer 0: D0[b][n] = X W0^T                           (tcgen05, A and B in smem)
//         H0 = ReLU(D0 + b0) -> its hi / lo planes back into TMEM     (tcgen05.ld / .st)
//         layer 1: D1[b][u] = H0 W1_tile^T                      (tcgen05, A in TMEM)
//         H1 = ReLU(D1 + b1); the tile's head partial sums H1 . W_head (FP32 FMA)
//   K3 tc_bwd_kernel : 128 threads, two task kinds
//       (A) 128 layer-1 units x a batch split:  dW1[u][k] = sum_b dZ1[b][u] H0[b][k]  and the
//           head-weight gradient dWh[j][u] = sum_b dHead[b][j] H1[b][u], M = units (TMEM lanes),
//           K = samples; A operands (dZ1^T, H1^T) built in TMEM by their lane's thread, dZ1
//           computed on the fly from K2's dHead: dZ1 = (dHead . W_head) * [H1 > 0]
//       (B) 128-row batch tile x a split of the layer-1 units:  dH0^T[k][b] = sum_u W1[u][k] dZ1[b][u]
//           (M = layer-0 units, N = samples), then its share of dW0 / db0:
//           dZ0 = dH0 * [H0 > 0] (the mask distributes over the split sum) and
//           dW0_share[k][d] = sum_b dZ0[k][b] [x | 1][b][d]    (second MMA, A = dZ0 in TMEM)
//
// FP32 accuracy (BASELINE north star 1e-5): every fp32 operand x is carried as two tf32 terms,
// hi = tf32(x) and lo = x - hi (exact in fp32, read as tf32 by the MMA), and a product is
// lo.hi + hi.lo + hi.hi accumulated in fp32 -- the dropped lo.lo term is ~2^-22 of the product
// ("3xTF32", the same arithmetic as mma_tf32.cuh's legacy-MMA path).  Reduced precision
// (rpl_dqn_config.precision TF32 / BF16, reading Q33): one product of tf32- / bf16-rounded
// operands.
//
// Operand layouts (sm_100 no-swizzle canonical, 32-bit elements): a K-major tile of R rows x
// kc columns is 8-row x 16-byte core matrices, LBO = 128 B between core matrices along K,
// SBO = kc * 32 B between 8-row groups (off_k); one MMA consumes K = 8 (two core matrices).
// An A operand in TMEM holds row r in lane r, one element per 32-bit column.
// (kind::tf32 MN-major operands need the 32-byte-atom swizzle: every transposed operand here
// is transposed by the thread that stages it instead -- scripts/mb_tc32.cu.)
#pragma once
#include "umma.cuh"
#include "mma_tf32.cuh"

namespace rpl {
namespace tc {

constexpr int T = 128;      // threads per CTA (4 warps: warp w <-> TMEM lanes 32w .. 32w + 31)
constexpr int KC = 32;      // contraction chunk of a staged operand (32 tf32 = 8 core matrices)
constexpr int MAXJ = 33;    // head outputs (1 + 32 actions)

__device__ __forceinline__ uint32_t off_k(int r, int k, int kc)
{
    return (uint32_t)((r >> 3) * (kc * 32) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
// descriptor of k-step s (K = 8) of a K-major tile with kc-element rows
__device__ __forceinline__ uint64_t kdesc(const void *tile, int s, int kc)
{
    return umma::desc(static_cast<const char *>(tile) + s * 256, 128, (uint32_t)kc * 32);
}
// instruction descriptor: kind::tf32, D fp32, A and B K-major, M x N
__host__ __device__ constexpr uint32_t idesc(int M, int N)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
// the 3xTF32 product sequence (small terms first); prec != 0: hi.hi only
__device__ __forceinline__ void mma3_ss(uint32_t d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                        uint32_t id, uint32_t acc, int prec)
{
    if (prec == 0) {
        mma_ss(d, al, bh, id, acc);
        mma_ss(d, ah, bl, id, 1u);
        mma_ss(d, ah, bh, id, 1u);
    } else {
        mma_ss(d, ah, bh, id, acc);
    }
}
__device__ __forceinline__ void mma3_ts(uint32_t d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                        uint32_t id, uint32_t acc, int prec)
{
    if (prec == 0) {
        mma_ts(d, al, bh, id, acc);
        mma_ts(d, ah, bl, id, 1u);
        mma_ts(d, ah, bh, id, 1u);
    } else {
        mma_ts(d, ah, bh, id, acc);
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
__device__ __forceinline__ void st16(uint32_t a, const uint32_t (&r)[16])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                    "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM address of column `col` in this warp's lane quarter
__device__ __forceinline__ uint32_t lane_addr(uint32_t base, int warp, int col)
{
    return base + ((uint32_t)(32 * warp) << 16) + (uint32_t)col;
}

// a 4-element group split into its hi / lo tf32 planes and stored as one 16-byte chunk each
__device__ __forceinline__ void split_store4(char *hi, char *lo, uint32_t off, float x0, float x1, float x2,
                                            float x3, int prec)
{
    uint4 h, l;
    split_p(x0, h.x, l.x, prec);
    split_p(x1, h.y, l.y, prec);
    split_p(x2, h.z, l.z, prec);
    split_p(x3, h.w, l.w, prec);
    *reinterpret_cast<uint4 *>(hi + off) = h;
    if (prec == 0) *reinterpret_cast<uint4 *>(lo + off) = l;
}

// every thread of the CTA waits for phase `ph` of an mbarrier (then flips its parity)
__device__ __forceinline__ void wait_bar(uint64_t *bar, uint32_t &ph)
{
    umma::mbar_wait(bar, ph);
    ph ^= 1u;
    umma::fence_after_sync();
}
// make this thread's TMEM stores and shared-memory operand writes visible to the MMA issuer
__device__ __forceinline__ void operands_ready()
{
    wait_st();
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
}

// ---- K1 shared-memory layout (bytes); the host sizes the launch with the same formula ----
constexpr int T1 = 256;     // K1 threads: group 0 (warps 0-3) gather / layer 0, group 1 (warps 4-7) layer-1 epilogue
struct FwdSmem {
    int oX, oW0, oW1, oWh, ob0, ob1, oidx, opj, opj2, obar, total;
    __host__ __device__ FwdSmem(int N0, int UN, int J)
    {
        oX = 0;                                   // X hi | lo: 2 x [128 rows x 32] tf32
        oW0 = oX + 2 * 128 * KC * 4;              // W0 hi | lo: 2 x [128 units x 32]
        oW1 = oW0 + 2 * 128 * KC * 4;             // W1 tile hi | lo: 2 x [UN units x N0]
        oWh = oW1 + 2 * UN * N0 * 4;              // head weights of the tile [J][UN] fp32
        ob0 = oWh + J * UN * 4;                   // b0 [N0]
        ob1 = ob0 + N0 * 4;                       // b1 tile [UN]
        oidx = ob1 + UN * 4;                      // sampled slots [128]
        opj = oidx + 128 * 4;                     // deferred-insert index of a row, or -1 [128]
        opj2 = opj + 128 * 4;                     // the same for its s' row (shared states)
        obar = (opj2 + 128 * 4 + 15) & ~15;       // mbarriers f0, f1[2], free[2] + TMEM base
        total = obar + 64;
    }
};

__device__ __forceinline__ void group0_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(umma::smem_u32(bar)) : "memory");
}

}  // namespace tc

// ------------------------------------------------------------------------------------------
// K1 (tensor cores), persistent per (net, unit tile of UN layer-1 units): a CTA stages its
// weight tile once, then runs batch tiles bt = b0, b0 + cpc, ... (cpc CTAs per combo) as a
// pipeline of two thread groups (TMEM lane = batch row; warp w owns lanes 32 (w % 4) ..):
//   group 0 (warps 0-3): gather X(i) -> wait F1(i-1) (its A operand, H0, occupies TMEM
//     [0, 256)) -> F0(i) = X W0^T (thread 0 issues) -> H0 = ReLU(+b0) split into TMEM hi / lo
//     -> thread 0 issues F1(i) = H0 W1_tile^T into accumulator i % 2
//   group 1 (warps 4-7): F1(i) done -> H1 = ReLU(+b1) (kept for the online net on s), head
//     partial sums H1 . W_head -> releases accumulator i % 2
// so the gather of tile i + 1 and the layer-1 epilogue of tile i overlap the MMAs of F1(i).
// TMEM columns: [0, 128) layer-0 accumulator, then the hi plane of H0; [128, 256) its lo
// plane; [256, 256 + UN) and [256 + UN, 256 + 2 UN) the two layer-1 accumulators.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(tc::T1, 1) tc_fwd_kernel(const __grid_constant__ FastArgs p)
{
    using namespace tc;
    CtaTrace trace_(p.trace, 0);
    extern __shared__ __align__(1024) char smc[];
    const int N0 = p.N0, N1 = p.N1, B = p.B, J = p.J, D = p.D, UN = p.UT, prec = p.prec;
    const int N0p = (N0 + 15) & ~15;
    const FwdSmem L(N0, UN, J);
    char *Xh = smc + L.oX, *Xl = Xh + 128 * KC * 4;
    char *W0h = smc + L.oW0, *W0l = W0h + 128 * KC * 4;
    char *W1h = smc + L.oW1, *W1l = W1h + UN * N0 * 4;
    float *Whs = reinterpret_cast<float *>(smc + L.oWh);
    float *b0s = reinterpret_cast<float *>(smc + L.ob0), *b1s = reinterpret_cast<float *>(smc + L.ob1);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smc + L.obar);   // [0] f0, [1,2] f1, [3,4] free
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smc + L.obar + 40);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, grp = tid >> 7, r = tid & 127;
    const int wq = warp & 3;   // TMEM lane quarter of this warp
    if (warp == 0) umma::tmem_alloc(tslot, 512);
    if (tid == 0) {
        umma::mbar_init(&bar[0], 1);
        umma::mbar_init(&bar[1], 1);
        umma::mbar_init(&bar[2], 1);
        umma::mbar_init(&bar[3], 128);
        umma::mbar_init(&bar[4], 128);
        umma::fence_mbar_init();
    }
    const int nbt = (B + 127) / 128, nut = p.nut;
    const uint64_t event = p.rctrl[0];
    const uint64_t size = p.pend_k ? p.pend_size : p.rctrl[1];
    const uint64_t cursor = p.pend_k ? (uint64_t)((p.pend_cur + p.pend_k) % p.capacity) : p.rctrl[2];
    const uint64_t nvalid = p.shared ? size - 1 : size;   // reading Q30
    const uint64_t oldest = (p.shared && size == (uint64_t)p.capacity) ? cursor : 0;
    if (p.pend_k && blockIdx.x == 0 && tid == 0) {
        p.rctrl[1] = p.pend_size;
        p.rctrl[2] = cursor;
    }
    // this CTA's combo and first batch tile: CTAs c, c + ncombo, ... share combo c
    const int ncombo = p.nets * nut;
    const int combo = blockIdx.x % ncombo, cpc = gridDim.x / ncombo, bt0 = blockIdx.x / ncombo;
    const int net = combo / nut, ut = combo % nut, u0 = ut * UN;
    const float *theta = net == 1 ? p.target : p.online;
    const bool vtile = p.dueling && u0 < p.S;
    // (1) the weight tile -> tf32 planes, once.  W1 rows u < UN (K = N0): a warp stores 8 rows
    // x 16 columns per instruction (conflict-free 16-byte stores, 64-byte global row pieces)
    {
        const int kq = N0 / 16, r8 = lane & 7, qq = lane >> 3;
        for (int g = warp; g < (UN / 8) * kq; g += T1 / 32) {
            const int u = (g / kq) * 8 + r8, k = (g % kq) * 16 + qq * 4;
            const float4 w = __ldg(reinterpret_cast<const float4 *>(theta + p.w1 + (int64_t)(u0 + u) * N0 + k));
            split_store4(W1h, W1l, off_k(u, k, N0), w.x, w.y, w.z, w.w, prec);
        }
        if (!p.h0_in) {   // W0 [N0p rows x 32] (K = D, zero past D): 4 consecutive inputs per item
            for (int e = tid; e < N0p * (KC / 4); e += T1) {
                const int n = e / (KC / 4), d4 = 4 * (e % (KC / 4));
                float w[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    w[i] = (n < N0 && d4 + i < D) ? __ldg(theta + p.w0 + (int64_t)n * D + d4 + i) : 0.0f;
                split_store4(W0h, W0l, off_k(n, d4, KC), w[0], w[1], w[2], w[3], prec);
            }
        }
        for (int n = tid; n < N0; n += T1) b0s[n] = __ldg(theta + p.b0 + n);
        for (int u = tid; u < UN; u += T1) b1s[u] = __ldg(theta + p.b1 + u0 + u);
        // head weights of the tile's units: dueling V row (j = 0) over V units, A rows
        // (j >= 1) over A units (a tile never straddles the streams: S % UN == 0)
        for (int e = tid; e < J * UN; e += T1) {
            const int j = e / UN, c = e - j * UN;
            float w = 0.0f;
            if (!p.dueling) w = __ldg(theta + p.wh + (int64_t)j * N1 + u0 + c);
            else if (vtile && j == 0) w = __ldg(theta + p.wh + u0 + c);
            else if (!vtile && j > 0) w = __ldg(theta + p.wh + (int64_t)j * p.S + (u0 - p.S) + c);
            Whs[e] = w;
        }
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = *tslot;
    trace_.mark(2);
    int it = 0;
    for (int bt = bt0; bt < nbt; bt += cpc, ++it) {
        const int rb = bt * 128, nb = min(128, B - rb);
        const uint32_t accA = tb + 256 + (uint32_t)(UN * (it & 1));
        if (grp == 0) {
            // ---------------- group 0: gather, layer 0, issue layer 1 ----------------------
            long long tg = trace_.now();
            if (!p.h0_in) {
                // (2) Philox sample of row rb + r (Q3): index 2j / 2j + 1 of call j
                const int row = rb + r;
                int32_t slot = 0;
                if (p.bidx) {
                    slot = row < B ? p.bidx[row] : 0;
                } else if (p.distinct) {
                    slot = row < B ? p.idx[row] : 0;
                } else {
                    int32_t i0, i1;
                    sample_pair(p.seed, p.rank, event, (uint32_t)(row >> 1), nvalid, i0, i1);
                    slot = slot_of((row & 1) ? i1 : i0, oldest, p.capacity);
                }
                auto pend_j = [&](int64_t sl) {
                    int64_t j = sl - p.pend_cur;
                    if (j < 0) j += p.capacity;
                    return j < p.pend_k ? (int)j : -1;
                };
                const int pj = pend_j(slot);
                const bool nxt = net != 0 && p.shared;    // shared states: s' = next slot's s
                const int64_t sslot = nxt ? (slot + 1) % p.capacity : slot;
                const int pjx = nxt ? pend_j(sslot) : pj;
                const int col0 = net == 0 || p.shared ? 0 : D;
                // (3) the row's state into registers (pending slots read through from the
                // insert's sources, possibly pinned host memory)
                float x[KC];
                const int64_t rslot = p.bidx ? min(row, B - 1) : sslot;   // in-RAM: the copied batch
                const float *src = pjx < 0 ? p.ring + rslot * p.rs + col0
                                           : (net == 0 || p.shared ? p.pend_s : p.pend_s2) + (int64_t)pjx * D;
#pragma unroll
                for (int d = 0; d < KC; ++d) x[d] = (d < D && r < nb) ? src[d] : 0.0f;
                if (net == 0 && ut == 0 && r < nb) {
                    int32_t ra;
                    float rr;
                    uint32_t rd;
                    if (pj < 0) {
                        const float *sc = p.ring + (int64_t)(p.bidx ? row : slot) * p.rs + p.sw;
                        ra = __float_as_int(__ldg(sc));
                        rr = __ldg(sc + 1);
                        rd = __float_as_uint(__ldg(sc + 2));
                    } else {
                        ra = p.pend_a[pj];
                        rr = p.pend_r[pj];
                        rd = p.pend_done[pj];
                    }
                    p.idx[row] = slot;
                    p.a[row] = ra;
                    p.r[row] = rr;
                    p.done[row] = (uint8_t)(rd != 0u);
                }
                if (ut == 0 && net <= 1 && r < nb) {
                    float *xo = (net == 0 ? p.Xs : p.Xs2) + (int64_t)row * D;
                    for (int d = 0; d < D; ++d) xo[d] = x[d];
                }
#pragma unroll
                for (int q = 0; q < KC / 4; ++q)
                    split_store4(Xh, Xl, off_k(r, 4 * q, KC), x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3], prec);
                umma::fence_async_smem();
            }
            trace_.acc(3, tg);   // phase 3: gather
            tg = trace_.now();
            // F1(it - 1) has finished reading H0 (TMEM [0, 256))
            if (it > 0) umma::mbar_wait(&bar[1 + ((it - 1) & 1)], (uint32_t)(((it - 1) >> 1) & 1));
            umma::fence_after_sync();
            trace_.acc(4, tg);   // phase 4: wait for F1(it - 1)
            tg = trace_.now();
            if (p.h0_in) {
                // wide inputs (config 5): layer 0 came from wide.cuh -> its activations into TMEM
                const float *h0 = p.h0_in + ((int64_t)net * B + rb + r) * N0;
                for (int c0 = 0; c0 < N0p; c0 += 16) {
                    uint32_t hh[16], hl[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float h = (r < nb && c0 + i < N0) ? __ldcg(h0 + c0 + i) : 0.0f;
                        split_p(h, hh[i], hl[i], prec);
                    }
                    st16(lane_addr(tb, wq, c0), hh);
                    if (prec == 0) st16(lane_addr(tb, wq, 128 + c0), hl);
                }
            } else {
                group0_sync();   // every row of X is in shared memory
                // (4) layer 0 on the tensor cores: D0[128][N0p] = X W0^T
                if (tid == 0) {
                    umma::fence_after_sync();
                    const uint32_t id = idesc(128, N0p);
#pragma unroll
                    for (int s = 0; s < KC / 8; ++s)
                        mma3_ss(tb, kdesc(Xh, s, KC), kdesc(Xl, s, KC), kdesc(W0h, s, KC), kdesc(W0l, s, KC), id,
                                s > 0 ? 1u : 0u, prec);
                    umma::commit(&bar[0]);
                }
                umma::mbar_wait(&bar[0], (uint32_t)(it & 1));
                umma::fence_after_sync();
                trace_.acc(5, tg);   // phase 5: layer-0 MMAs (issue + wait)
                tg = trace_.now();
                // H0 = ReLU(D0 + b0) -> hi plane over D0, lo plane at column 128
                const bool keep = net == 0 && ut == 0 && r < nb;
                for (int c0 = 0; c0 < N0p; c0 += 16) {
                    uint32_t v[16], hl[16];
                    ld16(lane_addr(tb, wq, c0), v);
                    wait_ld();
                    float h[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int c = c0 + i;
                        h[i] = c < N0 ? fmaxf(__uint_as_float(v[i]) + b0s[c], 0.0f) : 0.0f;
                        split_p(h[i], v[i], hl[i], prec);
                    }
                    if (keep) {
                        float *ho = p.H0 + (int64_t)(rb + r) * N0 + c0;
#pragma unroll
                        for (int i = 0; i < 16; i += 4)
                            if (c0 + i < N0) *reinterpret_cast<float4 *>(ho + i) = make_float4(h[i], h[i + 1], h[i + 2], h[i + 3]);
                    }
                    st16(lane_addr(tb, wq, c0), v);
                    if (prec == 0) st16(lane_addr(tb, wq, 128 + c0), hl);
                }
            }
            wait_st();
            umma::fence_before_sync();
            group0_sync();   // H0 complete in TMEM
            trace_.acc(6, tg);   // phase 6: layer-0 epilogue
            // (5) layer 1: D1[128][UN] = H0 W1_tile^T into accumulator it % 2 (free once group 1
            // has drained it for tile it - 2)
            if (tid == 0) {
                umma::fence_after_sync();
                if (it >= 2) umma::mbar_wait(&bar[3 + (it & 1)], (uint32_t)(((it - 2) >> 1) & 1));
                umma::fence_after_sync();
                const uint32_t id = idesc(128, UN);
                for (int s = 0; s < N0 / 8; ++s)
                    mma3_ts(accA, tb + 8 * s, tb + 128 + 8 * s, kdesc(W1h, s, N0), kdesc(W1l, s, N0), id,
                            s > 0 ? 1u : 0u, prec);
                umma::commit(&bar[1 + (it & 1)]);
            }
        } else {
            // ---------------- group 1: layer-1 epilogue of tile it ----------------------------
            const long long tw = trace_.now_by(128);
            umma::mbar_wait(&bar[1 + (it & 1)], (uint32_t)((it >> 1) & 1));
            umma::fence_after_sync();
            trace_.acc_by(128, 7, tw);   // phase 7: group 1 waiting for F1(it)
            // (6) H1 = ReLU(D1 + b1) (kept for the online net on s) and the tile's head partials
            float acc[MAXJ];
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) acc[j] = 0.0f;
            const bool keep1 = net == 0 && r < nb;
            for (int c0 = 0; c0 < UN; c0 += 16) {
                uint32_t v[16];
                ld16(lane_addr(accA, wq, c0), v);
                wait_ld();
                float h[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) h[i] = fmaxf(__uint_as_float(v[i]) + b1s[c0 + i], 0.0f);
                if (keep1) {
                    float *ho = p.H1 + (int64_t)(rb + r) * N1 + u0 + c0;
#pragma unroll
                    for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4 *>(ho + i) = make_float4(h[i], h[i + 1], h[i + 2], h[i + 3]);
                }
                if (vtile) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) acc[0] = fmaf(h[i], Whs[c0 + i], acc[0]);
                } else {
#pragma unroll
                    for (int j = 0; j < MAXJ; ++j) {
                        if (j < J && (p.dueling ? j > 0 : true)) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) acc[j] = fmaf(h[i], Whs[j * UN + c0 + i], acc[j]);
                        }
                    }
                }
            }
            umma::fence_before_sync();
            mbar_arrive(&bar[3 + (it & 1)]);   // accumulator it % 2 drained
            if (r < nb) {
                float *po = p.part + (((int64_t)net * nut + ut) * B + rb + r) * J;
#pragma unroll
                for (int j = 0; j < MAXJ; ++j)
                    if (j < J) po[j] = acc[j];
            }
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tb, 512);
}

// ------------------------------------------------------------------------------------------
// K3 (tensor cores).  Task kinds (A) dW1 + dWh for 128 units x one batch split, (B) dH0 for
// one 128-row batch tile x one split of the layer-1 units, with its dW0 / db0 share.
// ------------------------------------------------------------------------------------------
namespace tc {
struct BwdSmem {
    int oS0, oS1, oX, owh, obar, total;   // two operand stages, x^T planes, W_head chunks
    __host__ __device__ BwdSmem()
    {
        // a stage: (A tasks) H0^T hi | lo 2 x [128 x 32] + dHead^T hi | lo 2 x [32 x 32]
        //          (B tasks) dZ1 hi | lo 2 x [128 x 32]
        oS0 = 0;
        oS1 = oS0 + (2 * 128 * KC + 2 * 32 * KC) * 4;
        oX = oS1 + (2 * 128 * KC + 2 * 32 * KC) * 4;    // [x | 1]^T hi | lo: 2 x [32 x 128]
        owh = oX + 2 * 32 * 128 * 4;                    // [2][MAXJ][32] fp32 (W_head or dHead chunk)
        obar = (owh + 2 * MAXJ * 32 * 4 + 15) & ~15;    // 3 mbarriers + TMEM base
        // >= half the shared memory of an SM: one CTA per SM (each allocates all 512 TMEM columns)
        total = obar + 32 < 120 * 1024 ? 120 * 1024 : obar + 32;
    }
};
}  // namespace tc

__global__ void __launch_bounds__(tc::T, 1) tc_bwd_kernel(const __grid_constant__ FastArgs p)
{
    using namespace tc;
    CtaTrace trace_(p.trace, 2);
    extern __shared__ __align__(1024) char smc[];
    const BwdSmem L;
    const int N0 = p.N0, N1 = p.N1, B = p.B, J = p.J, D = p.D, prec = p.prec;
    const int N0p = (N0 + 15) & ~15, JP = (J + 15) & ~15;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smc + L.obar);
    uint32_t *tslot = reinterpret_cast<uint32_t *>(smc + L.obar + 24);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // the deferred insert's ring rows: a warp's first row loaded before the tasks (a zero-copy
    // source's PCIe round trip overlaps them), every row written after them
    const int64_t pj0 = (int64_t)blockIdx.x * (T / 32) + warp;
    const bool pre = p.pend_k && pj0 < p.pend_k && p.rs <= 32 * RW_PRE;
    float prow[RW_PRE];
    if (pre) ring_load_row(prow, p.rs, p.D, p.sw, lane, pj0, p.pend_s, p.pend_a, p.pend_r, p.pend_s2,
                           p.pend_done, p.pend_err);
    if (warp == 0) umma::tmem_alloc(tslot, 512);
    if (tid == 0) {
        for (int i = 0; i < 3; ++i) umma::mbar_init(&bar[i], 1);
        umma::fence_mbar_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = *tslot;
    uint32_t ph[3] = {0u, 0u, 0u};
    pdl_wait();   // K2's dHead (no-op without a programmatic launch)
    const int nut3 = (N1 + 127) / 128, nA = nut3 * p.nsb;
    const int nbt = (B + 127) / 128, nB = nbt * p.NS;
    const int ucs = N1 / p.NS;   // units per B-task split (a multiple of 32)
    for (int task = blockIdx.x; task < nA + nB; task += gridDim.x) {
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
        if (task < nB) {
            // ---------------- (B) dH0^T[k][b] over a split of the units, dW0 share ---------
            const int s = task / nbt, bt = task % nbt;
            const int rb = bt * 128, nb = min(128, B - rb), Nb = max(16, (nb + 15) & ~15);
            const int ua = s * ucs, ue = min(N1, ua + ucs), nch = (ue - ua + KC - 1) / KC;
            const int b = rb + tid;   // B-operand row (sample) of this thread
            float dh[MAXJ];
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) dh[j] = (j < J && tid < nb) ? __ldcg(p.dHead + (int64_t)b * J + j) : 0.0f;
            bool pend[2] = {false, false};
            for (int c = 0; c < nch; ++c) {
                const int st = c & 1;
                long long tw = trace_.now();
                if (pend[st]) {   // the MMAs of chunk c - 2 are done with this stage
                    wait_bar(&bar[st], ph[st]);
                    pend[st] = false;
                }
                trace_.acc(3, tw);
                const long long ts = trace_.now();
                char *Sh = smc + (st ? L.oS1 : L.oS0), *Sl = Sh + 128 * KC * 4;
                float *whs = reinterpret_cast<float *>(smc + L.owh) + st * MAXJ * KC;
                const int uc = ua + KC * c;
                // W_head chunk [j][i] for units uc + i (dueling: V row over V units, A rows
                // over A units)
                for (int e = tid; e < J * KC; e += T) {
                    const int j = e / KC, i = e - j * KC, u = uc + i;
                    float w = 0.0f;
                    if (u < ue) {
                        if (!p.dueling) w = __ldg(p.online + p.wh + (int64_t)j * N1 + u);
                        else if (u < p.S) w = j == 0 ? __ldg(p.online + p.wh + u) : 0.0f;
                        else w = j > 0 ? __ldg(p.online + p.wh + (int64_t)j * p.S + (u - p.S)) : 0.0f;
                    }
                    whs[e] = w;
                }
                // A = W1^T[k][u] into TMEM (lane k = tid), columns 128 + 64 st: hi 32 | lo 32
                {
                    uint32_t ah[16], al[16];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int u = uc + 16 * h + i;
                            const float w = (tid < N0 && u < ue) ? __ldg(p.online + p.w1 + (int64_t)u * N0 + tid) : 0.0f;
                            split_p(w, ah[i], al[i], prec);
                        }
                        st16(lane_addr(tb, warp, 128 + 64 * st + 16 * h), ah);
                        if (prec == 0) st16(lane_addr(tb, warp, 128 + 64 * st + 32 + 16 * h), al);
                    }
                }
                __syncthreads();   // whs
                // B = dZ1[b][u] (rows b, K = u): dZ1 = (dHead . W_head) * [H1 > 0] (P:94's
                // combine backward folded into dHead by K2)
#pragma unroll
                for (int q = 0; q < KC / 4; ++q) {
                    const int u = uc + 4 * q;
                    float z[4] = {0.f, 0.f, 0.f, 0.f};
                    if (tid < nb && u < ue) {
                        const float4 h1 = __ldcg(reinterpret_cast<const float4 *>(p.H1 + (int64_t)b * N1 + u));
                        const float hv[4] = {h1.x, h1.y, h1.z, h1.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float a = 0.0f;
#pragma unroll
                            for (int j = 0; j < MAXJ; ++j)
                                if (j < J) a = fmaf(dh[j], whs[j * KC + 4 * q + e], a);
                            z[e] = hv[e] > 0.0f ? a : 0.0f;
                        }
                    }
                    split_store4(Sh, Sl, off_k(tid, 4 * q, KC), z[0], z[1], z[2], z[3], prec);
                }
                operands_ready();
                trace_.acc(2, ts);
                if (tid == 0) {
                    const uint32_t id = idesc(128, Nb);
#pragma unroll
                    for (int k = 0; k < KC / 8; ++k)
                        mma3_ts(tb, tb + 128 + 64 * st + 8 * k, tb + 128 + 64 * st + 32 + 8 * k, kdesc(Sh, k, KC),
                                kdesc(Sl, k, KC), id, (c > 0 || k > 0) ? 1u : 0u, prec);
                    umma::commit(&bar[st]);
                }
                pend[st] = true;
            }
            // drain in chunk order
            long long tw = trace_.now();
            for (int c = max(0, nch - 2); c < nch; ++c)
                if (pend[c & 1]) {
                    wait_bar(&bar[c & 1], ph[c & 1]);
                    pend[c & 1] = false;
                }
            trace_.acc(3, tw);
            const long long te = trace_.now();
            const int k = tid;   // TMEM lane = layer-0 unit
            if (p.PdH0) {
                // wide inputs: the partial dH0 goes to memory; K4 forms dZ0 (wide.cuh dW0)
                float *out = p.PdH0 + (int64_t)s * B * N0;
                for (int c0 = 0; c0 < Nb; c0 += 16) {
                    uint32_t v[16];
                    ld16(lane_addr(tb, warp, c0), v);
                    wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (k < N0 && c0 + i < nb) out[(int64_t)(rb + c0 + i) * N0 + k] = __uint_as_float(v[i]);
                }
                continue;
            }
            // [x | 1]^T planes (rows d, K = the tile's samples): row D = 1 gives db0
            {
                char *Xh = smc + L.oX, *Xl = Xh + 32 * 128 * 4;
                const int d = tid & 31;
                for (int b4 = tid >> 5; b4 < 32; b4 += 4) {
                    float xv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int bb = 4 * b4 + e;
                        xv[e] = bb >= nb ? 0.0f : d < D ? __ldcg(p.Xs + (int64_t)(rb + bb) * D + d) : d == D ? 1.0f : 0.0f;
                    }
                    split_store4(Xh, Xl, off_k(d, 4 * b4, 128), xv[0], xv[1], xv[2], xv[3], prec);
                }
            }
            // dZ0 = dH0 * ReLU'(z0): hi plane over the accumulator, lo plane at column 384
            for (int c0 = 0; c0 < Nb; c0 += 16) {
                uint32_t v[16], zl[16];
                ld16(lane_addr(tb, warp, c0), v);
                wait_ld();
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int bb = c0 + i;
                    const float h0 = (k < N0 && bb < nb) ? __ldcg(p.H0 + (int64_t)(rb + bb) * N0 + k) : 0.0f;
                    const float z = h0 > 0.0f ? __uint_as_float(v[i]) : 0.0f;
                    split_p(z, v[i], zl[i], prec);
                }
                st16(lane_addr(tb, warp, c0), v);
                if (prec == 0) st16(lane_addr(tb, warp, 384 + c0), zl);
            }
            operands_ready();
            if (tid == 0) {
                const uint32_t id = idesc(128, 32);
                const char *Xh = smc + L.oX, *Xl = Xh + 32 * 128 * 4;
                for (int k8 = 0; k8 < Nb / 8; ++k8)
                    mma3_ts(tb + 256, tb + 8 * k8, tb + 384 + 8 * k8, kdesc(Xh, k8, 128), kdesc(Xl, k8, 128), id,
                            k8 > 0 ? 1u : 0u, prec);
                umma::commit(&bar[2]);
            }
            wait_bar(&bar[2], ph[2]);
            if (k < N0) {
                float *w0p = p.w0part + (int64_t)(s * nbt + bt) * (p.b0 + N0);
                for (int c0 = 0; c0 < 32; c0 += 16) {
                    uint32_t v[16];
                    ld16(lane_addr(tb, warp, 256 + c0), v);
                    wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int d = c0 + i;
                        if (d < D) w0p[p.w0 + (int64_t)k * D + d] = __uint_as_float(v[i]);
                        else if (d == D) w0p[p.b0 + k] = __uint_as_float(v[i]);
                    }
                }
            } else {
                // keep every lane's TMEM loads collective (.sync.aligned): lanes past N0 load too
                for (int c0 = 0; c0 < 32; c0 += 16) {
                    uint32_t v[16];
                    ld16(lane_addr(tb, warp, 256 + c0), v);
                    wait_ld();
                }
            }
            trace_.acc(5, te);
        } else {
            // ---------------- (A) dW1 and dWh for 128 units over one batch split ------------
            const int a = task - nB;
            const int s = a / nut3, ut3 = a % nut3;
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit), nch = (ke - kb + KC - 1) / KC;
            const int u = ut3 * 128 + tid;   // this thread's unit / TMEM lane
            const bool uv = u < N1;
            // W_head column of the unit: dueling V unit -> j = 0, A unit -> j >= 1; plain all j
            float wcol[MAXJ];
#pragma unroll
            for (int j = 0; j < MAXJ; ++j) {
                float w = 0.0f;
                if (uv && j < J) {
                    if (!p.dueling) w = __ldg(p.online + p.wh + (int64_t)j * N1 + u);
                    else if (u < p.S) w = j == 0 ? __ldg(p.online + p.wh + u) : 0.0f;
                    else w = j > 0 ? __ldg(p.online + p.wh + (int64_t)j * p.S + (u - p.S)) : 0.0f;
                }
                wcol[j] = w;
            }
            float db1 = 0.0f, dbh = 0.0f;
            bool pend[2] = {false, false};
            for (int c = 0; c < nch; ++c) {
                const int st = c & 1;
                long long tw = trace_.now();
                if (pend[st]) {
                    wait_bar(&bar[st], ph[st]);
                    pend[st] = false;
                }
                trace_.acc(3, tw);
                const long long ts = trace_.now();
                char *Hh = smc + (st ? L.oS1 : L.oS0), *Hl = Hh + 128 * KC * 4;
                char *Gh = Hl + 128 * KC * 4, *Gl = Gh + 32 * KC * 4;
                float *dhs = reinterpret_cast<float *>(smc + L.owh) + st * MAXJ * KC;   // [i][J]
                const int b0 = kb + KC * c;
                for (int e = tid; e < KC * J; e += T) {
                    const int i = e / J, j = e - i * J;
                    dhs[e] = b0 + i < ke ? __ldcg(p.dHead + (int64_t)(b0 + i) * J + j) : 0.0f;
                }
                // B operands: H0^T [k][b] (rows k = tid) and dHead^T [j][b] (rows j)
                if (tid < N0p) {
#pragma unroll
                    for (int q = 0; q < KC / 4; ++q) {
                        float hv[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int bb = b0 + 4 * q + e;
                            hv[e] = (bb < ke && tid < N0) ? __ldcg(p.H0 + (int64_t)bb * N0 + tid) : 0.0f;
                        }
                        split_store4(Hh, Hl, off_k(tid, 4 * q, KC), hv[0], hv[1], hv[2], hv[3], prec);
                    }
                }
                for (int e = tid; e < JP * (KC / 4); e += T) {
                    const int j = e / (KC / 4), q = e % (KC / 4);
                    float gv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int bb = b0 + 4 * q + i;
                        gv[i] = (bb < ke && j < J) ? __ldcg(p.dHead + (int64_t)bb * J + j) : 0.0f;
                    }
                    split_store4(Gh, Gl, off_k(j, 4 * q, KC), gv[0], gv[1], gv[2], gv[3], prec);
                }
                __syncthreads();   // dhs
                // A operands into TMEM (lane = unit): dZ1^T and H1^T, columns 256 + 128 st:
                // [dZ1 hi 32 | dZ1 lo 32 | H1 hi 32 | H1 lo 32]
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t zh[16], zl[16], hh[16], hl[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int ii = 16 * h + i, bb = b0 + ii;
                        const float h1 = (uv && bb < ke) ? __ldcg(p.H1 + (int64_t)bb * N1 + u) : 0.0f;
                        float acc = 0.0f;
#pragma unroll
                        for (int j = 0; j < MAXJ; ++j)
                            if (j < J) acc = fmaf(dhs[ii * J + j], wcol[j], acc);
                        const float z = h1 > 0.0f ? acc : 0.0f;
                        db1 += z;
                        split_p(z, zh[i], zl[i], prec);
                        split_p(h1, hh[i], hl[i], prec);
                    }
                    const int cb = 256 + 128 * st + 16 * h;
                    st16(lane_addr(tb, warp, cb), zh);
                    st16(lane_addr(tb, warp, cb + 64), hh);
                    if (prec == 0) {
                        st16(lane_addr(tb, warp, cb + 32), zl);
                        st16(lane_addr(tb, warp, cb + 96), hl);
                    }
                }
                if (ut3 == 0 && tid < J)   // head-bias gradient sum_b dHead[b][j], by task ut3 = 0
                    for (int i = 0; i < KC; ++i) dbh += dhs[i * J + tid];
                operands_ready();
                trace_.acc(4, ts);
                if (tid == 0) {
                    const uint32_t idw = idesc(128, N0p), idh = idesc(128, JP);
                    const uint32_t cb = tb + 256 + 128 * st;
#pragma unroll
                    for (int k = 0; k < KC / 8; ++k) {
                        const uint32_t acc = (c > 0 || k > 0) ? 1u : 0u;
                        mma3_ts(tb, cb + 8 * k, cb + 32 + 8 * k, kdesc(Hh, k, KC), kdesc(Hl, k, KC), idw, acc, prec);
                        mma3_ts(tb + 128, cb + 64 + 8 * k, cb + 96 + 8 * k, kdesc(Gh, k, KC), kdesc(Gl, k, KC), idh, acc, prec);
                    }
                    umma::commit(&bar[st]);
                }
                pend[st] = true;
            }
            for (int c = max(0, nch - 2); c < nch; ++c)
                if (pend[c & 1]) {
                    wait_bar(&bar[c & 1], ph[c & 1]);
                    pend[c & 1] = false;
                }
            float *gp = p.gpart + (int64_t)s * p.gps;
            for (int c0 = 0; c0 < N0p; c0 += 16) {
                uint32_t v[16];
                ld16(lane_addr(tb, warp, c0), v);
                wait_ld();
                if (uv) {
                    float *o = gp + p.w1 + (int64_t)u * N0 + c0;
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        if (c0 + i < N0)
                            *reinterpret_cast<float4 *>(o + i) = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                                             __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                }
            }
            if (uv) gp[p.b1 + u] = db1;
            for (int c0 = 0; c0 < JP; c0 += 16) {
                uint32_t v[16];
                ld16(lane_addr(tb, warp, 128 + c0), v);
                wait_ld();
                if (uv) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int j = c0 + i;
                        if (j >= J) continue;
                        if (!p.dueling) gp[p.wh + (int64_t)j * N1 + u] = __uint_as_float(v[i]);
                        else if (u < p.S && j == 0) gp[p.wh + u] = __uint_as_float(v[i]);
                        else if (u >= p.S && j > 0) gp[p.wh + (int64_t)j * p.S + (u - p.S)] = __uint_as_float(v[i]);
                    }
                }
            }
            if (ut3 == 0 && tid < J) gp[p.bh + tid] = dbh;
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tb, 512);
    // the deferred insert's rows
    if (p.pend_k) {
        for (int64_t j = (int64_t)blockIdx.x * (T / 32) + warp; j < p.pend_k; j += (int64_t)gridDim.x * (T / 32)) {
            int64_t slot = p.pend_cur + j;
            if (slot >= p.capacity) slot -= p.capacity;
            if (pre && j == pj0)
                ring_store_row(p.ring + slot * p.rs, prow, p.rs, lane);
            else
                ring_write_row(p.ring + slot * p.rs, p.rs, p.D, p.sw, lane, j, p.pend_s, p.pend_a, p.pend_r,
                               p.pend_s2, p.pend_done, p.pend_err);
        }
    }
}

}  // namespace rpl
