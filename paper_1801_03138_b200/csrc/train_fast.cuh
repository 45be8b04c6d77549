// train_fast.cuh -- the fast path of the device-resident train step for two trunk layers
// (the paper's dueling net 27 -> 128 -> [V 512 | A 512] -> 1 + |A|, and the plain
// 27 -> 64 -> 64 -> |A| MLP of configs[0]).  Four kernels, captured once per batch size into a
// CUDA graph:
//
//   K1 fwd  : per (net, 16-row batch tile, unit tile of layer 1): Philox sample + gather the 16
//             rows (pending-insert slots read through from the insert's source), layer 0 for
//             those rows (recomputed per unit tile: 55 kMAC, cheaper than a grid-wide
//             exchange), the tile's layer-1 units and its partial sums of the V/A heads, all as
//             3xTF32 mma.sync tiles (mma_tf32.cuh).  All weights stream into shared memory
//             with cp.async while the sampled rows are being gathered from HBM.
//   K2 td   : per sample: reduce head partials, dueling combine, max / argmax (warp shuffles),
//             TD target, Huber, dQ, dV/dA, and dZ1 = dHead . W_head (*) ReLU'(z1).
//   K3 bwd1 : (programmatic launch: stages K1's operands while K2 runs) dW1 = dZ1^T H0 (+ db1)
//             32x32 tiles, split-K partials of dH0 = dZ1 W1 with their dW0 / db0 shares, head
//             gradients -- 3xTF32 mma.sync; its first CTAs also write the deferred insert's
//             ring rows.
//   K4 bwd0 : W0 / b0 = fixed-order sum of K3's partials, then SGD of every parameter
//             (non-finite guard), target sync, counters; the loss is stored first.
//
// Step-varying state (sampler event, ring size, step counter) lives in device memory so the
// same graph replays every step with no host input.
#pragma once
#include "philox.cuh"
#include "simt_gemm.cuh"
#include "mma_tf32.cuh"
#include "ring_row.cuh"
#include "distinct.cuh"
#include "umma.cuh"
#include "wide.cuh"

namespace rpl {

constexpr int F_BT = 16;          // batch rows per K1 task
constexpr int F_MAXJ = 33;        // head outputs (1 + 32 actions)
constexpr int F_JT = (F_MAXJ + 7) / 8;   // 8-wide MMA n-tiles of the head outputs
constexpr int F_JP = 8 * F_JT;           // head outputs padded to the n-tiles
constexpr int F_NT1 = 512;        // threads per K1 CTA
constexpr int F_NT3 = 256;        // threads per K3 CTA

struct FastArgs {
    // replay (rctrl[0] = sampler events consumed, rctrl[1] = filled size, rctrl[2] = cursor)
    float *ring;
    int rs, D;
    int shared, sw;      // shared states (s' = next slot's s); scalar word offset
    uint64_t *rctrl;
    uint64_t seed;
    uint32_t rank;
    // deferred insert (pend_k > 0, K1 only): experience j < pend_k belongs in slot
    // (pend_cur + j) mod capacity; K1 reads sampled pending slots from these SoA sources,
    // writes the rows and sets rctrl[1] = pend_size (replay.cu replay_add)
    const float *pend_s, *pend_s2, *pend_r;
    const int32_t *pend_a;
    const uint8_t *pend_done;
    uint32_t *pend_err;   // the replay's sticky error word (corrupt done)
    int64_t pend_cur, capacity;
    uint64_t pend_size;
    int pend_k;
    // network
    int A, dueling, J, S, N0, N1, nets, ddqn;
    int64_t w0, b0, w1, b1, wh, bh, P;
    int B;
    float gamma, lr, kappa;
    int kinf;
    int64_t sync_period;
    float *online, *target;
    // workspaces
    float *Xs, *Xs2, *r;
    int32_t *a, *idx;
    uint8_t *done;
    float *H0, *H1;      // online net on s: [B][N0], [B][N1]
    float *part;         // [nets][nut][B][J]
    int nut, UT;
    float *dHead;        // [B][J]
    float *dZ1;          // [B][N1]
    float *w0part;       // [NS][ceil(B/32)][N0*D + N0] dW0 / db0 partials (K3 -> K4)
    int NS;
    float *gpart;        // [nsb][gps] (== grad when nsb == 1)
    int64_t gps;         // gpart split stride: P rounded up to 4 (16-byte aligned splits)
    int nsb, bsplit;
    float *grad;         // [P + 1]
    float *loss_part, *Qs, *Qt2, *Qo2, *y;
    int32_t *astar;
    float *loss_out;
    int64_t *step_dev;
    int32_t *sync_flag;  // written by K2 (step t+1 is a sync step), read by K4 / sgd_kernel
    int apply_update;
    int distinct;        // 1: the batch indices come from distinct_fast_kernel (in idx)
    const int32_t *bidx; // in-RAM replay (RPL_RING_HOST_BATCH): the CPU-sampled indices of the
                         // batch copied to the device; then `ring` is that batch, row b = sample b
    // wide inputs (config 5): layer 0 runs in wide.cuh; the fast kernels run the layers above it
    const float *h0_in;  // [nets][B][N0] layer-0 activations (K1 skips sample, gather, layer 0)
    float *PdH0;         // [NS][B][N0] K3's dH0 split-K partials (no dW0 shares)
    float *dZ0;          // [B][N0] dZ0 materialised by K4 for wide_dw0_kernel
    uint16_t *dZ0bf;     // its bf16 hi / mid / lo planes [3][B][N0]
    int event_advanced;  // 1: the step's sampling kernel advanced rctrl[0] already
    int loss_early;      // 1: loss_out_kernel (a side branch after K3) writes *loss_out, K4 does not
    uint32_t *err;
    unsigned long long *trace;   // optional per-CTA [kernel][cta][start, end] %globaltimer (ns)
    int prec;            // rpl_dqn_config.precision (split_p / mma_3xtf32, mma_tf32.cuh)
    int tc;              // 1: K1 / K3 are the tensor-core kernels of tc_fast.cuh (K2 skips dZ1,
                         //    which K3 forms on the fly; K4 sums nw0 dW0 / db0 partials)
    int nw0;             // tc / tcb: dW0 / db0 partials in w0part
    // large-batch tensor-core path (tc_big.cuh): bf16 hi / mid / lo images of the operands
    int tcb;             // 1: the step runs tc_big.cuh's kernels (K4 writes the W1 image)
    int Bp;              // B rounded up to 128 (rows past B are zero in every image)
    int jp;              // dheadp row pitch (J rounded up to 4)
    uint16_t *h0img;     // [nets + 1][3][Bp * 128] H0 of every net (tile-quarter blocks, T1), then the online net on s (row-group major, T3a)
    uint16_t *ximg;      // [3][Bp * 32] [x | 1] of s
    uint16_t *dz1img;    // [3][Bp * N1] dZ1
    uint16_t *w1img;     // [online, target][3][N1 * 128] W1
    float *w0t;          // [online, target][D][N0] W0 transposed (T0's operand; K4 keeps it)
    int64_t h0pl, xpl, dzpl, w1pl;   // plane strides (elements)
    float *dheadp;       // [B][jp] dHead
};

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// records the CTA's start / end %globaltimer (ns) and phase marks as SM-clock cycles since
// the CTA started when tracing is on (RPL_TRACE=1)
struct CtaTrace {
    unsigned long long *slot;
    unsigned long long *any;   // this CTA's trace words, for any thread (acc_by)
    long long c0;
    __device__ CtaTrace(unsigned long long *tr, int kernel)
        : slot(tr && threadIdx.x == 0 ? tr + 8 * ((size_t)kernel * 2048 + blockIdx.x) : nullptr),
          any(tr ? tr + 8 * ((size_t)kernel * 2048 + blockIdx.x) : nullptr), c0(0)
    {
        if (slot) {
            slot[0] = gtimer();
            c0 = clock64();
        }
    }
    __device__ ~CtaTrace()
    {
        if (slot) slot[1] = gtimer();
    }
    __device__ void mark(int i)
    {
        if (slot) slot[i] = (unsigned long long)(clock64() - c0);
    }
    // accumulate the cycles since `t` into slot i (phase totals of a CTA)
    __device__ void acc(int i, long long t)
    {
        if (slot) slot[i] += (unsigned long long)(clock64() - t);
    }
    __device__ long long now() const { return slot ? clock64() : 0; }
    // the same from thread `who` of the CTA (e.g. the first thread of another warp group)
    __device__ long long now_by(int who) const { return any && (int)threadIdx.x == who ? clock64() : 0; }
    __device__ void acc_by(int who, int i, long long t)
    {
        if (any && (int)threadIdx.x == who) any[i] += (unsigned long long)(clock64() - t);
    }
};

// programmatic dependent launch: let the next kernel of the graph start early / wait for the
// previous one's results (no-ops when the launch is not programmatic)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// n floats (n % 4 == 0, both pointers 16-byte aligned) global -> shared, 16-byte cp.async
__device__ __forceinline__ void cp_async_row(float *dst, const float *src, int n, int tid, int nt)
{
    for (int c = tid; c < n / 4; c += nt) cp_async16(dst + 4 * c, src + 4 * c);
}

__device__ __forceinline__ float f_huber(float d, float kappa, int kinf)
{
    const float ad = fabsf(d);
    if (kinf || ad <= kappa) return 0.5f * d * d;
    return kappa * (ad - 0.5f * kappa);
}

// TD target, Huber loss and the head-output gradient of one sample, by one warp (lane j owns
// head output j / action j).  hs[net * hsld + j]: head outputs (bias included) of the online
// net on s (net 0), the target net on s' (1), the online net on s' (2, Double DQN).  Writes the
// step's exported Q / y / loss / a* for sample b and dhs[0, J).
__device__ __forceinline__ void td_warp(const FastArgs &p, const float *hs, int hsld, int ab, float rb,
                                        uint8_t db, int b, int lane, float *dhs)
{
    const int A = p.A, B = p.B;
    float q[3];
#pragma unroll
    for (int net = 0; net < 3; ++net) {
        float qa = 0.0f;
        if (net < p.nets) {
            if (p.dueling) {
                // Q(s,a) = V(s) + A(s,a) - (1/|A|) sum_a' A(s,a'); the mean by a
                // fixed shuffle tree over the lanes (A <= 32)
                const float av = lane < A ? hs[net * hsld + 1 + lane] : 0.0f;
                const float mean = warp_sum(av) / (float)A;
                if (lane < A) qa = hs[net * hsld + 0] + av - mean;
            } else if (lane < A) {
                qa = hs[net * hsld + lane];
            }
        }
        q[net] = qa;
    }
    // TD target (Q9): DQN max_a Q_t(s',a); Double DQN Q_t(s', argmax_a Q_o(s',a))
    float boot;
    int astar = -1;
    if (!p.ddqn) {
        float m = lane < A ? q[1] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        boot = m;
    } else {
        float v = lane < A ? q[2] : -INFINITY;
        int ix = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
            if (ov > v || (ov == v && oi < ix)) { v = ov; ix = oi; }   // ties: lowest
        }
        astar = ix;
        boot = __shfl_sync(0xffffffffu, q[1], astar);
    }
    const float notdone = db ? 0.0f : 1.0f;
    const float yb = rb + p.gamma * notdone * boot;
    const float qsel = __shfl_sync(0xffffffffu, q[0], ab & 31);   // Q[i*A + a_i]
    // an action outside [0, A) (a corrupt experience; the replay does not know A) poisons the
    // loss, so the non-finite guard skips the whole update, and raises the sticky ECORRUPT
    const bool bad = (unsigned)ab >= (unsigned)A;
    if (bad && lane == 0) atomicOr(p.err, ERRBIT_CORRUPT);
    const float delta = bad ? __int_as_float(0x7fc00000) : qsel - yb;
    const float g = (p.kinf ? delta : fminf(fmaxf(delta, -p.kappa), p.kappa)) / (float)B;
    if (p.dueling) {
        // dV = sum_a dQ_a = g ; dA_a = dQ_a - (1/|A|) sum_a' dQ_a'
        if (lane < A) dhs[1 + lane] = (lane == ab ? g : 0.0f) - g / (float)A;
        if (lane == 0) dhs[0] = g;
    } else if (lane < A) {
        dhs[lane] = lane == ab ? g : 0.0f;
    }
    if (lane < A) {
        p.Qs[(int64_t)b * A + lane] = q[0];
        p.Qt2[(int64_t)b * A + lane] = q[1];
        if (p.ddqn) p.Qo2[(int64_t)b * A + lane] = q[2];
    }
    if (lane == 0) {
        p.y[b] = yb;
        p.loss_part[b] = f_huber(delta, p.kappa, p.kinf);
        if (p.ddqn) p.astar[b] = astar;
    }
}

// the distinct sampler of the fast path (graph-replayed: event and filled size read on the
// device, the deferred insert's size included) -> idx[B], read by K1
__global__ void __launch_bounds__(DS_T, 1) distinct_fast_kernel(const __grid_constant__ FastArgs p)
{
    extern __shared__ int ds_smem[];
    const uint64_t event = p.rctrl[0];
    const uint64_t size = p.pend_k ? p.pend_size : p.rctrl[1];
    const uint64_t cursor = p.pend_k ? (uint64_t)((p.pend_cur + p.pend_k) % p.capacity) : p.rctrl[2];
    const uint64_t nvalid = p.shared ? size - 1 : size;
    const uint64_t oldest = (p.shared && size == (uint64_t)p.capacity) ? cursor : 0;
    distinct_sample(p.seed, p.rank, event, nvalid, p.B, p.idx, p.err, ds_smem,
                    ds_smem + ds_table_slots(p.B), oldest, p.capacity);
}

// shared-memory layout of K1 (32-bit words); the same formula sizes the launch on the host
struct FwdLayout {
    int XP, N0P, UT, UTP;
    int oW0, oX, oXh, oXl, oH0h, oH0l, oW1, oH1, oWh, ob0, ob1, oidx, opj, opj2, ored, total;
    __host__ __device__ FwdLayout(int D, int N0, int UT_, int J)
    {
        (void)J;
        XP = ((D + 7) & ~7) + 4;         // X row stride: K padded to the MMA k-step, +4 words
        N0P = ((N0 + 31) & ~31) + 4;     // row stride == 4 (mod 32): conflict-free fragments
        UT = UT_;
        UTP = UT + 4;
        oW0 = 0;                         // W0 flat [N0 * D], 16-byte aligned
        oX = (N0 * D + 3) & ~3;          // [BT][XP] fp32 gathered states
        oXh = oX + F_BT * XP;            // [BT][XP] tf32 hi
        oXl = oXh + F_BT * XP;           // [BT][XP] tf32 lo
        oH0h = oXl + F_BT * XP;          // [BT][N0P] tf32 hi of H0
        oH0l = oH0h + F_BT * N0P;        // [BT][N0P] tf32 lo of H0
        oW1 = oH0l + F_BT * N0P;         // [UT][N0P] fp32 layer-1 weight tile
        oH1 = oW1 + UT * N0P;            // [BT][UTP] fp32 H1 tile
        oWh = oH1 + F_BT * UTP;          // [F_JP][UTP] fp32 head-weight tile (rows >= J zero)
        ob0 = oWh + F_JP * UTP;          // [N0]
        ob1 = ob0 + ((N0 + 3) & ~3);     // [UT]
        oidx = ob1 + UT;                 // [BT]
        opj = oidx + F_BT;               // [BT] deferred-insert index j of the row, or -1
        opj2 = opj + F_BT;               // [BT] the same for its s' row (shared states)
        ored = opj2 + F_BT;              // [16 warps][16][F_JP] head partials
        total = ored + 16 * 16 * F_JP;
    }
};

// ------------------------------------------------------------------------------------------
// K1.  512 threads = 16 warps; layer 0, layer 1 and the head partials are 16-row
// tensor-core products (3xTF32 mma.sync.m16n8k8, FP32-accurate): warp w owns n-tiles
// w, w+16, ... of 8 output units.  Compile-time dims (KD, KN0, KJ) for the paper's /
// configs[0] nets; 0 = read at run time.
// ------------------------------------------------------------------------------------------
// MC > 1: the kernel runs in clusters of MC CTAs that share one weight tile (consecutive
// batch tiles of one (net, unit tile)); each CTA loads 1/MC of the tile's rows with TMA
// multicast into every CTA of the cluster, so L2 serves the weights once per cluster
template <int UT, int KD, int KN0, int KJ, int MC>
__device__ __forceinline__ void fast_fwd_body(const FastArgs &p)
{
    CtaTrace trace_(p.trace, 0);
    __shared__ uint64_t wbar;   // MC > 1: the multicast weight bytes have landed
    pdl_trigger();
    extern __shared__ float4 smem4[];
    float *sm = reinterpret_cast<float *>(smem4);
    constexpr int NW = F_NT1 / 32;
    const int D = KD ? KD : p.D, N0 = KN0 ? KN0 : p.N0, J = KJ ? KJ : p.J;
    const int N1 = p.N1, B = p.B;
    const FwdLayout L(D, N0, UT, J);
    float *W0f = sm + L.oW0, *Xs = sm + L.oX, *W1s = sm + L.oW1;
    uint32_t *Xh = reinterpret_cast<uint32_t *>(sm + L.oXh), *Xl = reinterpret_cast<uint32_t *>(sm + L.oXl);
    uint32_t *H0h = reinterpret_cast<uint32_t *>(sm + L.oH0h), *H0l = reinterpret_cast<uint32_t *>(sm + L.oH0l);
    float *H1s = sm + L.oH1, *Whs = sm + L.oWh, *b0s = sm + L.ob0, *b1s = sm + L.ob1, *red = sm + L.ored;
    int *idxs = reinterpret_cast<int *>(sm + L.oidx), *pjs = reinterpret_cast<int *>(sm + L.opj);
    int *pjs2 = reinterpret_cast<int *>(sm + L.opj2);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int nbt = (B + F_BT - 1) / F_BT, nut = p.nut;
    const uint64_t event = p.rctrl[0];
    const uint64_t size = p.pend_k ? p.pend_size : p.rctrl[1];
    const uint64_t cursor = p.pend_k ? (uint64_t)((p.pend_cur + p.pend_k) % p.capacity) : p.rctrl[2];
    // shared states: the newest experience has no stored successor (reading Q30)
    const uint64_t nvalid = p.shared ? size - 1 : size;
    const uint64_t oldest = (p.shared && size == (uint64_t)p.capacity) ? cursor : 0;
    if (p.pend_k && blockIdx.x == 0 && threadIdx.x == 0) {
        p.rctrl[1] = p.pend_size;
        p.rctrl[2] = cursor;
    }
    const int ntasks = p.nets * nbt * nut;
    // tasks are (net, unit tile)-major: with the grid a multiple of nets x nut (large batches),
    // a CTA keeps one weight tile resident and walks batch tiles, loading the weights once.
    // MC > 1 (one task per CTA): batch tiles fastest, so a cluster shares its weight tile
    const int ncombo = p.nets * nut;
    int loaded = -1;
    if (MC > 1) {
        if (tid == 0) {
            umma::mbar_init(&wbar, 1);
            umma::fence_mbar_init();
        }
        cooperative_groups::this_cluster().sync();   // every peer's barrier exists before data lands
    }
    for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
        const int combo = MC > 1 ? task / nbt : task % ncombo, bt = MC > 1 ? task % nbt : task / ncombo;
        const int net = combo / nut, ut = combo % nut;
        const int rb = bt * F_BT, u0 = ut * UT;
        const int nu = min(UT, N1 - u0);   // valid units in this tile (multiple of 4)
        const float *theta = net == 1 ? p.target : p.online;
        const bool reload = combo != loaded;
        loaded = combo;
        __syncthreads();   // the previous task is done with shared memory
        // (1) weights -> shared memory, all 16-byte cp.async (no load waits on another)
        if (reload && MC > 1) {
            // rows u = rank, rank + MC, ... of the W1 tile and 1/MC of W0 from this CTA, each
            // bulk copy multicast to the whole cluster; the barrier expects the full tile
            const int rk = (int)(blockIdx.x % MC);
            const uint16_t all = (uint16_t)((1u << MC) - 1u);
            const uint32_t w0b = (uint32_t)(N0 * D * 4), w0c = w0b / MC;
            const bool w0split = !p.h0_in && w0c % 16 == 0;
            if (tid == 0)
                umma::mbar_expect_tx(&wbar, (uint32_t)(nu * N0 * 4) + (p.h0_in ? 0u : w0b));
            if (warp == 0) {
                for (int u = rk + MC * lane; u < nu; u += MC * 32)
                    umma::bulk_g2s_mc(W1s + u * L.N0P, theta + p.w1 + (int64_t)(u0 + u) * N0, N0 * 4, &wbar, all);
                if (lane == 0 && !p.h0_in) {
                    if (w0split)
                        umma::bulk_g2s_mc(reinterpret_cast<char *>(W0f) + rk * w0c,
                                          reinterpret_cast<const char *>(theta + p.w0) + rk * w0c, w0c, &wbar, all);
                    else if (rk == 0)
                        umma::bulk_g2s_mc(W0f, theta + p.w0, w0b, &wbar, all);
                }
            }
            const int c4 = N0 / 4;
            for (int e = nu * c4 + tid; e < UT * c4; e += F_NT1) {
                const int u = e / c4, c = e - u * c4;
                *reinterpret_cast<float4 *>(W1s + u * L.N0P + 4 * c) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (!p.h0_in) cp_async_row(b0s, theta + p.b0, N0, tid, F_NT1);
        } else if (reload) {
            const int c4 = N0 / 4;
            for (int e = tid; e < UT * c4; e += F_NT1) {
                const int u = e / c4, c = e - u * c4;
                float *dst = W1s + u * L.N0P + 4 * c;
                if (u < nu) cp_async16(dst, theta + p.w1 + (int64_t)(u0 + u) * N0 + 4 * c);
                else *reinterpret_cast<float4 *>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (!p.h0_in) {
                cp_async_row(W0f, theta + p.w0, N0 * D, tid, F_NT1);
                cp_async_row(b0s, theta + p.b0, N0, tid, F_NT1);
            }
        }
        if (reload) {
            cp_async_row(b1s, theta + p.b1 + u0, nu, tid, F_NT1);
            for (int u = nu + tid; u < UT; u += F_NT1) b1s[u] = 0.0f;
        }
        if (reload) {
            // head weights of the tile's units: dueling V row (j = 0) over V units, A rows
            // (j >= 1) over A units (a tile never straddles the streams: S % UT == 0)
            const bool vtile = p.dueling && u0 < p.S;
            for (int e = tid; e < F_JP * (UT / 4); e += F_NT1) {
                const int j = e / (UT / 4), c = e - j * (UT / 4);
                float *dst = Whs + j * L.UTP + 4 * c;
                const float *src = nullptr;
                if (j < J && 4 * c < nu) {
                    if (!p.dueling) src = theta + p.wh + (int64_t)j * N1 + u0 + 4 * c;
                    else if (vtile && j == 0) src = theta + p.wh + u0 + 4 * c;
                    else if (!vtile && j > 0) src = theta + p.wh + (int64_t)j * p.S + (u0 - p.S) + 4 * c;
                }
                if (src) cp_async16(dst, src);
                else *reinterpret_cast<float4 *>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        if (p.h0_in) {
            // wide inputs: layer 0 came from the tensor-core kernels -- load the tile's H0 rows
            // of this net and split them into tf32 hi / lo
            const float *h0 = p.h0_in + ((int64_t)net * B + rb) * N0;
            cp_async_wait_all();   // the weight tiles
            if (MC > 1 && reload) umma::mbar_wait(&wbar, 0);
            for (int e = tid; e < F_BT * N0; e += F_NT1) {
                const int rr = e / N0, cc = e - rr * N0;
                const float h = rb + rr < B ? __ldcg(h0 + (int64_t)rr * N0 + cc) : 0.0f;
                uint32_t hi, lo;
                split_p(h, hi, lo, p.prec);
                H0h[rr * L.N0P + cc] = hi;
                H0l[rr * L.N0P + cc] = lo;
            }
            __syncthreads();
        } else {
            // (2) Philox sample of the tile's rows (Q3)
            if (tid < F_BT / 2) {
                int32_t i0, i1;
                if (p.bidx) {       // in-RAM replay: sampled on the CPU, rows already gathered
                    i0 = rb + 2 * tid < B ? p.bidx[rb + 2 * tid] : 0;
                    i1 = rb + 2 * tid + 1 < B ? p.bidx[rb + 2 * tid + 1] : 0;
                } else if (p.distinct) {   // written by distinct_fast_kernel (rows past B: any valid slot)
                    i0 = rb + 2 * tid < B ? p.idx[rb + 2 * tid] : 0;
                    i1 = rb + 2 * tid + 1 < B ? p.idx[rb + 2 * tid + 1] : 0;
                } else {
                    sample_pair(p.seed, p.rank, event, (uint32_t)(rb / 2 + tid), nvalid, i0, i1);
                    i0 = slot_of(i0, oldest, p.capacity);
                    i1 = slot_of(i1, oldest, p.capacity);
                }
                idxs[2 * tid] = i0;
                idxs[2 * tid + 1] = i1;
                // deferred-insert index of a slot (read-through), or -1
                auto pend_j = [&](int64_t slot) {
                    int64_t j = slot - p.pend_cur;
                    if (j < 0) j += p.capacity;
                    return j < p.pend_k ? (int)j : -1;
                };
                pjs[2 * tid] = pend_j(i0);
                pjs[2 * tid + 1] = pend_j(i1);
                pjs2[2 * tid] = p.shared ? pend_j((i0 + 1) % p.capacity) : -1;
                pjs2[2 * tid + 1] = p.shared ? pend_j((i1 + 1) % p.capacity) : -1;
            }
            __syncthreads();
            // (3) gather the 16 sampled rows: s for online(s), s' for target(s') / online(s')
            // shared states: s' is the old state of the next slot
            const bool nxt = net != 0 && p.shared;
            const int col0 = net == 0 || p.shared ? 0 : D;
            for (int e = tid; e < F_BT * D; e += F_NT1) {
                const int rr = e / D, d = e - rr * D, j = nxt ? pjs2[rr] : pjs[rr];
                const int64_t slot = p.bidx ? min(rb + rr, B - 1) : nxt ? (idxs[rr] + 1) % p.capacity : idxs[rr];
                if (j < 0) {
                    cp_async4(Xs + rr * L.XP + d, p.ring + slot * p.rs + col0 + d);
                } else {   // pending insert: its sources (possibly pinned host memory: plain loads)
                    Xs[rr * L.XP + d] = (net == 0 || p.shared ? p.pend_s : p.pend_s2)[(int64_t)j * D + d];
                }
            }
            int32_t ra_ = 0;
            float rr_ = 0.0f;
            uint32_t rd_ = 0;
            const bool unpack_scalars = net == 0 && ut == 0 && tid < F_BT && rb + tid < B;
            if (unpack_scalars) {
                const int j = pjs[tid];
                if (j < 0) {
                    const float *row = p.ring + (int64_t)(p.bidx ? rb + tid : idxs[tid]) * p.rs + p.sw;
                    ra_ = __float_as_int(__ldg(row));
                    rr_ = __ldg(row + 1);
                    rd_ = __float_as_uint(__ldg(row + 2));
                } else {
                    ra_ = p.pend_a[j];
                    rr_ = p.pend_r[j];
                    rd_ = p.pend_done[j];
                }
            }
            trace_.mark(2);
            cp_async_wait_all();
            if (MC > 1 && reload) umma::mbar_wait(&wbar, 0);   // the multicast W1 / W0 tiles
            __syncthreads();
            trace_.mark(3);
            // split X into tf32 hi / lo (zero beyond D); unpack the batch once for the backward
            // pass and the debug export
            for (int e = tid; e < F_BT * L.XP; e += F_NT1) {
                const int rr = e / L.XP, d = e - rr * L.XP;
                const float x = d < D ? Xs[e] : 0.0f;
                uint32_t hi, lo;
                split_p(x, hi, lo, p.prec);
                Xh[e] = hi;
                Xl[e] = lo;
                if (ut == 0 && net <= 1 && d < D && rb + rr < B)
                    (net == 0 ? p.Xs : p.Xs2)[(int64_t)(rb + rr) * D + d] = x;
            }
            if (unpack_scalars) {
                p.idx[rb + tid] = idxs[tid];
                p.a[rb + tid] = ra_;
                p.r[rb + tid] = rr_;
                p.done[rb + tid] = (uint8_t)(rd_ != 0u);
            }
            __syncthreads();
            // (4) layer 0: H0[16][N0] = ReLU(X W0^T + b0)
            for (int nt = warp; nt < N0 / 8; nt += NW) {
                const int n = nt * 8 + g;
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                for (int k0 = 0; k0 < D; k0 += 8) {
                    uint32_t ah[4], al[4], bh[2], bl[2];
                    ah[0] = Xh[g * L.XP + k0 + t];       al[0] = Xl[g * L.XP + k0 + t];
                    ah[1] = Xh[(g + 8) * L.XP + k0 + t]; al[1] = Xl[(g + 8) * L.XP + k0 + t];
                    ah[2] = Xh[g * L.XP + k0 + t + 4];   al[2] = Xl[g * L.XP + k0 + t + 4];
                    ah[3] = Xh[(g + 8) * L.XP + k0 + t + 4]; al[3] = Xl[(g + 8) * L.XP + k0 + t + 4];
                    const float w0 = k0 + t < D ? W0f[n * D + k0 + t] : 0.0f;
                    const float w1 = k0 + t + 4 < D ? W0f[n * D + k0 + t + 4] : 0.0f;
                    split_p(w0, bh[0], bl[0], p.prec);
                    split_p(w1, bh[1], bl[1], p.prec);
                    mma_3xtf32(c, ah, al, bh, bl, p.prec);
                }
                const int col = nt * 8 + 2 * t;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rr = g + (q >> 1) * 8, cc = col + (q & 1);
                    float h = c[q] + b0s[cc];
                    h = h > 0.0f ? h : 0.0f;
                    uint32_t hi, lo;
                    split_p(h, hi, lo, p.prec);
                    H0h[rr * L.N0P + cc] = hi;
                    H0l[rr * L.N0P + cc] = lo;
                    if (net == 0 && ut == 0 && rb + rr < B) p.H0[(int64_t)(rb + rr) * N0 + cc] = h;
                }
            }
            __syncthreads();
            trace_.mark(4);
        }
        // (5) layer 1: H1[16][UT] = ReLU(H0 W1_tile^T + b1)
        for (int nt = warp; nt < UT / 8; nt += NW) {
            const float *wrow = W1s + (nt * 8 + g) * L.N0P;
            float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
            for (int k0 = 0; k0 < N0; k0 += 8) {
                uint32_t ah[4], al[4], bh[2], bl[2];
                ah[0] = H0h[g * L.N0P + k0 + t];       al[0] = H0l[g * L.N0P + k0 + t];
                ah[1] = H0h[(g + 8) * L.N0P + k0 + t]; al[1] = H0l[(g + 8) * L.N0P + k0 + t];
                ah[2] = H0h[g * L.N0P + k0 + t + 4];   al[2] = H0l[g * L.N0P + k0 + t + 4];
                ah[3] = H0h[(g + 8) * L.N0P + k0 + t + 4]; al[3] = H0l[(g + 8) * L.N0P + k0 + t + 4];
                split_p(wrow[k0 + t], bh[0], bl[0], p.prec);
                split_p(wrow[k0 + t + 4], bh[1], bl[1], p.prec);
                mma_3xtf32(c, ah, al, bh, bl, p.prec);
            }
            const int col = nt * 8 + 2 * t;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rr = g + (q >> 1) * 8, cc = col + (q & 1);
                float h = c[q] + b1s[cc];
                h = h > 0.0f ? h : 0.0f;
                H1s[rr * L.UTP + cc] = h;
                if (net == 0 && rb + rr < B && cc < nu) p.H1[(int64_t)(rb + rr) * N1 + u0 + cc] = h;
            }
        }
        __syncthreads();
        trace_.mark(5);
        // (6) head partials [16 rows][JP = 8 * ceil(J / 8)]: warp w takes k-steps w, w+16, ...
        //     of the tile's units; the per-warp products are reduced in a fixed order
        {
            const int JT = (J + 7) / 8;
            float c[F_JT][4];
#pragma unroll
            for (int jt = 0; jt < F_JT; ++jt)
#pragma unroll
                for (int q = 0; q < 4; ++q) c[jt][q] = 0.0f;
            for (int k0 = warp * 8; k0 < UT; k0 += NW * 8) {
                uint32_t ah[4], al[4], bh[2], bl[2];
                split_p(H1s[g * L.UTP + k0 + t], ah[0], al[0], p.prec);
                split_p(H1s[(g + 8) * L.UTP + k0 + t], ah[1], al[1], p.prec);
                split_p(H1s[g * L.UTP + k0 + t + 4], ah[2], al[2], p.prec);
                split_p(H1s[(g + 8) * L.UTP + k0 + t + 4], ah[3], al[3], p.prec);
#pragma unroll
                for (int jt = 0; jt < F_JT; ++jt) {
                    if (jt < JT) {
                        split_p(Whs[(8 * jt + g) * L.UTP + k0 + t], bh[0], bl[0], p.prec);
                        split_p(Whs[(8 * jt + g) * L.UTP + k0 + t + 4], bh[1], bl[1], p.prec);
                        mma_3xtf32(c[jt], ah, al, bh, bl, p.prec);
                    }
                }
            }
            float *rw = red + warp * (16 * F_JP);
#pragma unroll
            for (int jt = 0; jt < F_JT; ++jt) {
                if (jt < JT) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int rr = g + (q >> 1) * 8, cc = 8 * jt + 2 * t + (q & 1);
                        rw[rr * F_JP + cc] = c[jt][q];
                    }
                }
            }
        }
        __syncthreads();
        for (int o = tid; o < F_BT * J; o += F_NT1) {
            const int rr = o / J, j = o - rr * J;
            float v = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += red[w * (16 * F_JP) + rr * F_JP + j];
            if (rb + rr < B) p.part[(((int64_t)net * nut + ut) * B + rb + rr) * J + j] = v;
        }
    }
    if (MC > 1) cooperative_groups::this_cluster().sync();   // no CTA leaves while peers' copies fly
}

template <int UT, int KD, int KN0, int KJ>
__global__ void __launch_bounds__(F_NT1, 1) fast_fwd_kernel(const __grid_constant__ FastArgs p)
{
    fast_fwd_body<UT, KD, KN0, KJ, 1>(p);
}

constexpr int K1_MC = 4;   // cluster size of the multicast K1 (co-residency: scripts/mb_cluster.cu)
template <int UT, int KD, int KN0, int KJ>
__global__ void __cluster_dims__(K1_MC, 1, 1) __launch_bounds__(F_NT1, 1)
    fast_fwd_mc_kernel(const __grid_constant__ FastArgs p)
{
    fast_fwd_body<UT, KD, KN0, KJ, K1_MC>(p);
}

// ------------------------------------------------------------------------------------------
// K2: one CTA per sample
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) fast_td_kernel(const __grid_constant__ FastArgs p)
{
    CtaTrace trace_(p.trace, 1);
    extern __shared__ float4 smem4[];
    const int A = p.A, J = p.J, B = p.B, N1 = p.N1, S = p.S;
    const int HS = p.dueling ? S : N1;
    float *Whs = reinterpret_cast<float *>(smem4);      // the online head weights (J x HS)
    float *h1s = Whs + J * HS;                          // this sample's H1 row
    __shared__ float hs[3][F_MAXJ + 1];
    __shared__ float dhs[F_MAXJ + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (blockIdx.x == 0 && tid == 0) {
        const int64_t t = *p.step_dev + 1;
        *p.sync_flag = (p.sync_period > 0 && t % p.sync_period == 0) ? 1 : 0;
    }
    // the head weights are reused for every sample of this CTA: stream them in once (they are
    // step-invariant, so before waiting for the forward kernel)
    pdl_trigger();
    if (!p.tc) cp_async_row(Whs, p.online + p.wh, J * HS, tid, NT);
    pdl_wait();
    for (int b = blockIdx.x; b < B; b += gridDim.x) {
        __syncthreads();
        if (!p.tc) cp_async_row(h1s, p.H1 + (int64_t)b * N1, N1, tid, NT);
        // the sample's action / reward / terminal, needed after the reduction (prefetched)
        int ab = 0;
        float rb = 0.0f;
        uint8_t db = 0;
        if (warp == 0) {
            ab = p.a[b];
            rb = p.r[b];
            db = p.done[b];
        }
        if (warp < p.nets) {
            const float *theta = warp == 1 ? p.target : p.online;
            for (int j = lane; j < J; j += 32) {
                const float *src = p.part + ((int64_t)warp * p.nut * B + b) * J + j;
                const int64_t stride = (int64_t)B * J;
                float pv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pv[q] = q < p.nut ? __ldcg(src + q * stride) : 0.0f;
                float v = __ldg(theta + p.bh + j);
#pragma unroll
                for (int q = 0; q < 8; ++q) v += pv[q];
                for (int q = 8; q < p.nut; ++q) v += __ldcg(src + q * stride);
                hs[warp][j] = v;
            }
        }
        __syncthreads();
        trace_.mark(2);
        if (warp == 0) td_warp(p, &hs[0][0], F_MAXJ + 1, ab, rb, db, b, lane, dhs);
        trace_.mark(3);
        cp_async_wait_all();
        __syncthreads();
        trace_.mark(4);
        for (int j = tid; j < J; j += NT) p.dHead[(int64_t)b * J + j] = dhs[j];
        if (p.tc) continue;   // tc_bwd_kernel forms dZ1 from dHead itself
        // dZ1[b][u] = (dHead . W_head)[u] * ReLU'(z1[b][u]), 4 consecutive units per thread
        // (N1 % 4 == 0; a dueling stream boundary S % 4 == 0 never splits a group)
        for (int u4 = tid; u4 < N1 / 4; u4 += NT) {
            const int u = 4 * u4;
            float4 dh = make_float4(0.f, 0.f, 0.f, 0.f);
            auto acc = [&](float d, const float *w) {
                const float4 wv = *reinterpret_cast<const float4 *>(w);
                dh.x = fmaf(d, wv.x, dh.x); dh.y = fmaf(d, wv.y, dh.y);
                dh.z = fmaf(d, wv.z, dh.z); dh.w = fmaf(d, wv.w, dh.w);
            };
            if (p.dueling) {
                if (u < S) {
                    const float4 wv = *reinterpret_cast<const float4 *>(Whs + u);
                    dh = make_float4(dhs[0] * wv.x, dhs[0] * wv.y, dhs[0] * wv.z, dhs[0] * wv.w);
                } else {
                    for (int k = 0; k < A; ++k) acc(dhs[1 + k], Whs + (1 + k) * S + (u - S));
                }
            } else {
                for (int k = 0; k < A; ++k) acc(dhs[k], Whs + k * N1 + u);
            }
            const float4 h = *reinterpret_cast<const float4 *>(h1s + u);
            const float4 z = make_float4(h.x > 0.0f ? dh.x : 0.0f, h.y > 0.0f ? dh.y : 0.0f,
                                         h.z > 0.0f ? dh.z : 0.0f, h.w > 0.0f ? dh.w : 0.0f);
            *reinterpret_cast<float4 *>(p.dZ1 + (int64_t)b * N1 + u) = z;
        }
    }
}

// K3 operand: element (r, kk) is p[kk * ld + r] (source rows are kk) or p[r * ld + kk]
struct Opnd {
    const float *p;
    int ld, R;
};

// ------------------------------------------------------------------------------------------
// K3 tensor-core tile: C[32 x K3N] = sum_{kk in [kb, ke)} A(m, kk) B(n, kk) with 3xTF32
// mma.sync.m16n8k8 (FP32-accurate), 256 threads = 8 warps as 2 (m16) x 4 (n8 per K3N/4).  The
// whole contraction range (up to MM_SK per pass) is copied global -> shared with 16-byte
// cp.async in one go (one L2 round trip), in the source's own orientation: an operand whose
// source rows are kk (kRc) is stored [kk][r] with row stride MM_KS == 8 (mod 32) words, one whose
// source rows are r is stored [r][kk] with stride MM_RS == 4 (mod 32): both make every
// fragment load conflict-free.  Values are split into tf32 hi / lo while loading fragments.
// Operand element (r, kk) is p[kk * ld + r] (kRc) or p[r * ld + kk]; r, kk multiples of 4 are
// whole 16-byte chunks (all dims here are multiples of 4), missing chunks are zero-filled.
// ------------------------------------------------------------------------------------------
constexpr int MM_T = 256;
constexpr int K3N = 32;                      // K3 tile columns (32 x 32 tiles: 2 CTAs / SM)
constexpr int MM_SK = 128;                   // contraction per pass
constexpr int MM_KS = 40;                    // [kk][r] stride (>= BM, K3N; == 8 mod 32)
constexpr int MM_RS = MM_SK + 4;             // [r][kk] stride (== 4 mod 32)
constexpr int MM_OPF = MM_SK * MM_KS > BM * MM_RS ? MM_SK * MM_KS : BM * MM_RS;   // one operand
constexpr int MM_FLOATS = 2 * MM_OPF;

__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, bool valid)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}

// stage [k0, k0 + MM_SK) of an operand with TR rows: kRc -> S[kk][r], else S[r][kk]
template <bool kRc, int TR>
__device__ __forceinline__ void mm_stage(float *S, const Opnd &o, int r0, int k0, int kend, int tid)
{
    if (kRc) {
        // source rows are kk: TR/4 chunks of 16 B per kk
        for (int e = tid; e < MM_SK * (TR / 4); e += MM_T) {
            const int kk = e / (TR / 4), r4 = e % (TR / 4);
            const int r = r0 + 4 * r4, k = k0 + kk;
            const bool v = r < o.R && k < kend;
            cp_async16_zfill(S + kk * MM_KS + 4 * r4, v ? o.p + (int64_t)k * o.ld + r : o.p, v);
        }
    } else {
        // source rows are r: MM_SK/4 chunks of 16 B per r
        for (int e = tid; e < TR * (MM_SK / 4); e += MM_T) {
            const int r = e / (MM_SK / 4), k4 = e % (MM_SK / 4);
            const int rr = r0 + r, k = k0 + 4 * k4;
            const bool v = rr < o.R && k < kend;
            cp_async16_zfill(S + r * MM_RS + 4 * k4, v ? o.p + (int64_t)rr * o.ld + k : o.p, v);
        }
    }
}

// element (r, kk) of a staged operand
template <bool kRc>
__device__ __forceinline__ float mm_at(const float *S, int r, int kk)
{
    return kRc ? S[kk * MM_KS + r] : S[r * MM_RS + kk];
}

template <bool kARc, bool kBRc, class EPI, class RSUM>
__device__ __forceinline__ void gemm_mma_tile(const Opnd &a, const Opnd &b, int m0, int n0, int kb, int ke,
                                              const EPI &epi, bool want_rowsum, const RSUM &rs, float *smf,
                                              int prec, CtaTrace *tr = nullptr, int mk = 0)
{
    // 8 warps = 2 (m16 halves of the tile) x 4 (k-step residues): warp (wm, wk) computes rows
    // 16 wm .. 16 wm + 15 x all K3N columns over the k-steps ks == wk (mod 4) of every pass --
    // each A fragment feeds K3N / 8 MMAs and every staged word is read by one or two warps
    // (shared-memory bandwidth, not the HMMA pipe, bounds this loop).  The four k-residue
    // partials are added in a fixed order at the end.
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3, wm = warp & 1, wk = warp >> 1;
    float *As = smf, *Bs = smf + MM_OPF;
    constexpr int NT8 = K3N / 8;                  // n8 tiles per warp
    float c[NT8][4], cl[NT8][4], cm[NT8][4], cs[NT8][4];   // hi*hi, hi*lo, lo*hi partials; sums
#pragma unroll
    for (int i = 0; i < NT8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) cs[i][q] = 0.0f;
    float rsum = 0.0f;
    const int mr = 16 * wm + g;
    for (int k0 = kb; k0 < ke; k0 += MM_SK) {
        __syncthreads();   // the previous pass / task is done with the staging buffers
        mm_stage<kBRc, K3N>(Bs, b, n0, k0, ke, tid);
        if (k0 == kb) pdl_wait();   // A is K2's dZ1 (no-op without a programmatic launch)
        mm_stage<kARc, BM>(As, a, m0, k0, ke, tid);
        cp_async_wait_all();
        __syncthreads();
        if (tr && k0 == kb) tr->mark(mk);
        const int ksteps = (min(MM_SK, ke - k0) + 7) / 8;
#pragma unroll
        for (int i = 0; i < NT8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) c[i][q] = cl[i][q] = cm[i][q] = 0.0f;
        // this warp's k-steps of the pass: at most MM_SK / 32 = 4, one 32-deep chunk of the
        // round-to-nearest FP32 sums (long contractions keep FP32-level accuracy)
        for (int ks = wk; ks < ksteps; ks += 4) {
            const int k = 8 * ks;
            uint32_t ah[4], al[4];
            split_p(mm_at<kARc>(As, mr, k + t), ah[0], al[0], prec);
            split_p(mm_at<kARc>(As, mr + 8, k + t), ah[1], al[1], prec);
            split_p(mm_at<kARc>(As, mr, k + t + 4), ah[2], al[2], prec);
            split_p(mm_at<kARc>(As, mr + 8, k + t + 4), ah[3], al[3], prec);
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) {
                const int nc = 8 * nt + g;
                uint32_t bh[2], bl[2];
                split_p(mm_at<kBRc>(Bs, nc, k + t), bh[0], bl[0], prec);
                split_p(mm_at<kBRc>(Bs, nc, k + t + 4), bh[1], bl[1], prec);
                mma_3xtf32_sep(c[nt], cl[nt], cm[nt], ah, al, bh, bl, prec);
            }
        }
#pragma unroll
        for (int i = 0; i < NT8; ++i)
#pragma unroll
            for (int q = 0; q < 4; ++q) cs[i][q] += acc3_sum(c[i][q], cl[i][q], cm[i][q]);
        if (want_rowsum && tid < BM) {
            const int kn = min(MM_SK, ke - k0);
            for (int k = 0; k < kn; ++k) rsum += mm_at<kARc>(As, tid, k);
        }
    }
    if (tr) tr->mark(mk + 1);
    // k-residue partials -> shared memory (the staging buffers are free), fixed-order sum
    __syncthreads();
    float *red = smf;                                   // [4][BM][K3N + 1]
    constexpr int RP = K3N + 1;
#pragma unroll
    for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q)
            red[(wk * BM + 16 * wm + g + 8 * (q >> 1)) * RP + 8 * nt + 2 * t + (q & 1)] = cs[nt][q];
    __syncthreads();
    for (int e = tid; e < BM * K3N; e += MM_T) {
        const int m = e / K3N, n = e - m * K3N;
        const float v = ((red[(0 * BM + m) * RP + n] + red[(1 * BM + m) * RP + n]) +
                         red[(2 * BM + m) * RP + n]) + red[(3 * BM + m) * RP + n];
        epi(m0 + m, n0 + n, v);
    }
    if (want_rowsum && tid < BM) rs(m0 + tid, rsum);
}

constexpr int HD_U = 64;                                   // head-gradient unit tile
constexpr int K3_HD_FLOATS = 128 * HD_U + 128 * F_MAXJ + 4 * HD_U * 8;   // head-gradient staging
constexpr int K3_GEMM_FLOATS = MM_FLOATS;
// + the dH0 tile and the batch tile's states (D <= 64)
constexpr int K3_DH_FLOATS = K3_GEMM_FLOATS + BM * (K3N + 4) + BM * 36 + BM * K3N;
constexpr int K3_SMEM_FLOATS = K3_DH_FLOATS > K3_HD_FLOATS ? K3_DH_FLOATS : K3_HD_FLOATS;

// the batch-mean loss exactly as K4 forms it (NT = 256 threads: thread t sums samples t, t + 256,
// ... in order, warp sums, the 8 warp sums in warp order, / B): every thread of the CTA calls it
__device__ __forceinline__ float block_batch_loss(const FastArgs &p, float *red8)
{
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    float ls = 0.0f;
    for (int b = tid; b < p.B; b += 256) ls += __ldcg(p.loss_part + b);
    ls = warp_sum(ls);
    if (lane == 0) red8[wq] = ls;
    __syncthreads();
    float lsum = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) lsum += red8[w];
    return lsum / (float)p.B;
}

__global__ void __launch_bounds__(F_NT3) fast_bwd1_kernel(const __grid_constant__ FastArgs p)
{
    // K3 is launched programmatically after K2: every operand K1 (or an earlier step) wrote
    // -- H0, H1, W1, the states -- is requested before griddepcontrol.wait, K2's dZ1 / dHead
    // after it, so the weight / activation half of the staging overlaps K2
    CtaTrace trace_(p.trace, 2);
    extern __shared__ float4 smem4[];
    float *k3raw = reinterpret_cast<float *>(smem4);   // K3_SMEM_FLOATS
    const int N0 = p.N0, N1 = p.N1, B = p.B, J = p.J;
    const int wmt = (N1 + BM - 1) / BM, wnt = (N0 + K3N - 1) / K3N;
    const int n_w = wmt * wnt * p.nsb;
    const int hmt = (B + BM - 1) / BM, hnt = (N0 + K3N - 1) / K3N;
    const int n_h = hmt * hnt * p.NS;
    // head-weight gradient tasks: (128-unit tile) x (pass of <= 8 head rows), + 1 bias task
    const int hd_passes = p.dueling ? (p.A + 7) / 8 : (J + 7) / 8;
    const int hd_tasks = ((N1 + HD_U - 1) / HD_U) * hd_passes;
    const int n_hd = (hd_tasks + 1) * p.nsb;
    const int ntasks = n_w + n_h + n_hd;
    // the deferred insert's ring rows (no sampled row of this step reads them from the ring;
    // the next step's K1 follows K4): written by the first CTAs -- dW1 tasks, the shortest --
    // after their task, so the (possibly PCIe) source loads stay off the critical path
    // A warp's first row (rows <= 128 words) is loaded into registers before the CTA's task, so
    // a zero-copy source's PCIe round trip overlaps the task instead of following it
    const int pw = threadIdx.x >> 5, plane = threadIdx.x & 31;
    const int64_t pj0 = (int64_t)blockIdx.x * (F_NT3 / 32) + pw;
    const bool pre = p.pend_k && pj0 < p.pend_k && p.rs <= 32 * RW_PRE;
    float prow[RW_PRE];
    if (pre) ring_load_row(prow, p.rs, p.D, p.sw, plane, pj0, p.pend_s, p.pend_a, p.pend_r, p.pend_s2,
                           p.pend_done, p.pend_err);
    auto write_pending = [&]() {
        if (!p.pend_k) return;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = F_NT3 / 32;
        for (int64_t j = blockIdx.x * nw + warp; j < p.pend_k; j += (int64_t)gridDim.x * nw) {
            int64_t slot = p.pend_cur + j;
            if (slot >= p.capacity) slot -= p.capacity;
            if (pre && j == pj0)
                ring_store_row(p.ring + slot * p.rs, prow, p.rs, lane);
            else
                ring_write_row(p.ring + slot * p.rs, p.rs, p.D, p.sw, lane, j, p.pend_s, p.pend_a,
                               p.pend_r, p.pend_s2, p.pend_done, p.pend_err);
        }
    };
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        if (t < n_w) {
            // dW1[u][k] = sum_b dZ1[b][u] H0[b][k]  (+ db1[u] = sum_b dZ1[b][u])
            const int s = t / (wmt * wnt), rem = t % (wmt * wnt);
            const int m0 = (rem / wnt) * BM, n0 = (rem % wnt) * K3N;
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit);
            float *gp = p.gpart + (int64_t)s * p.gps;
            const Opnd a{p.dZ1, N1, N1}, bo{p.H0, N0, N0};
            auto epi = [&](int m, int n, float v) {
                if (m < N1 && n < N0) gp[p.w1 + (int64_t)m * N0 + n] = v;
            };
            auto rs = [&](int m, float v) {
                if (m < N1) gp[p.b1 + m] = v;
            };
            gemm_mma_tile<true, true>(a, bo, m0, n0, kb, ke, epi, n0 == 0, rs, k3raw, p.prec);
        } else if (t < n_w + n_h) {
            // dH0 partial [s][b][k] = sum_{u in split s} dZ1[b][u] W1[u][k]
            const int u = t - n_w;
            const int s = u / (hmt * hnt), rem = u % (hmt * hnt);
            const int m0 = (rem / hnt) * BM, n0 = (rem % hnt) * K3N;
            const int chunk = (N1 + p.NS - 1) / p.NS;
            const int kb = s * chunk, ke = min(N1, kb + chunk);
            if (p.PdH0) {
                // wide inputs: the partial goes to memory; K4 forms dZ0, wide_dw0_kernel dW0
                const Opnd a{p.dZ1, N1, B}, bo{p.online + p.w1, N0, N0};
                float *out = p.PdH0 + (int64_t)s * B * N0;
                auto epi = [&](int m, int n, float v) {
                    if (m < B && n < N0) out[(int64_t)m * N0 + n] = v;
                };
                gemm_mma_tile<false, true>(a, bo, m0, n0, kb, ke, epi, false, NoRowsum{}, k3raw, p.prec);
                continue;
            }
            // the partial dH0 tile stays in shared memory; masked by ReLU'(z0) it gives this
            // (split, batch tile)'s share of dW0 = dZ0^T X and db0 = sum_b dZ0 (the mask
            // distributes over the split-K sum), reduced in K4 in a fixed order
            float *tile = k3raw + K3_GEMM_FLOATS;          // [BM][K3N + 4] partial dH0
            float *xs = tile + BM * (K3N + 4);              // [BM][XS] states, column D = 1
            constexpr int XS = 36;
            const int D = p.D, nb = min(BM, B - m0), nk = min(K3N, N0 - n0);
            float *h0t = xs + BM * XS;                     // [BM][K3N] H0 of the tile (ReLU mask)
            // the tile's states and H0 (ReLU mask) are requested first: they arrive with the
            // GEMM operands (whose wait covers them)
            __syncthreads();   // a previous task of this CTA is done with xs / h0t
            for (int e = threadIdx.x; e < nb * D; e += F_NT3) {
                const int bb = e / D, d = e - bb * D;
                cp_async4(xs + bb * XS + d, p.Xs + (int64_t)m0 * D + e);
            }
            for (int e = threadIdx.x; e < nb * (nk / 4); e += F_NT3) {
                const int bb = e / (nk / 4), q = e % (nk / 4);
                cp_async16(h0t + bb * K3N + 4 * q, p.H0 + (int64_t)(m0 + bb) * N0 + n0 + 4 * q);
            }
            for (int e = threadIdx.x; e < BM * XS; e += F_NT3) {
                const int bb = e / XS, d = e - bb * XS;
                if (bb >= nb || d >= D) xs[e] = (d == D && bb < nb) ? 1.0f : 0.0f;   // ones column -> db0
            }
            for (int e = threadIdx.x; e < (BM - nb) * K3N; e += F_NT3) h0t[nb * K3N + e] = 0.0f;
            const Opnd a{p.dZ1, N1, B}, bo{p.online + p.w1, N0, N0};
            auto epi = [&](int m, int n, float v) { tile[(m - m0) * (K3N + 4) + (n - n0)] = v; };
            gemm_mma_tile<false, true>(a, bo, m0, n0, kb, ke, epi, false, NoRowsum{}, k3raw, p.prec, &trace_, 2);
            __syncthreads();
            trace_.mark(4);
            // dW0 / db0 share: C[unit k][d] = sum_b dZ0[b][k] xs[b][d] over the tile's rows with
            // dZ0 = dH0 * ReLU'(z0) (column D of xs is 1 -> db0); thread = (unit kk, 4
            // consecutive columns): 8 threads per unit
            float *w0p = p.w0part + ((int64_t)s * ((B + BM - 1) / BM) + m0 / BM) * (p.b0 + N0);
            {
                const int kk = threadIdx.x >> 3, d0 = 4 * (threadIdx.x & 7);
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
                for (int bb = 0; bb < BM; ++bb) {
                    const float z = h0t[bb * K3N + kk] > 0.0f ? tile[bb * (K3N + 4) + kk] : 0.0f;
                    const float4 x0 = *reinterpret_cast<const float4 *>(xs + bb * XS + d0);
                    acc[0] = fmaf(z, x0.x, acc[0]); acc[1] = fmaf(z, x0.y, acc[1]);
                    acc[2] = fmaf(z, x0.z, acc[2]); acc[3] = fmaf(z, x0.w, acc[3]);
                }
                const int k = n0 + kk;
                trace_.mark(6);
                if (kk < nk) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int d = d0 + q;
                        if (d < D) w0p[p.w0 + (int64_t)k * D + d] = acc[q];
                        else if (d == D) w0p[p.b0 + k] = acc[q];
                    }
                }
            }
            trace_.mark(7);
        } else {
            // head-weight gradients g_Wh[j][u] = sum_b dHead[b][j] H1[b][u]: a task owns 128
            // head-input units and a pass of up to 8 head rows j (dueling: the V row over V
            // units, the A rows over A units); H1 / dHead chunks of 32 samples are staged in
            // shared memory.  The last task of a b-split does the biases sum_b dHead[b][j].
            const int u = t - n_w - n_h;
            const int s = u / (hd_tasks + 1), c = u % (hd_tasks + 1);
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit);
            float *gp = p.gpart + (int64_t)s * p.gps;
            if (c == hd_tasks) {
                // warp w reduces head rows j = w, w + 4, ...: lanes stride the samples
                pdl_wait();
                const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
                for (int j = w; j < J; j += F_NT3 / 32) {
                    float acc = 0.0f;
                    for (int bb = kb + lane; bb < ke; bb += 32) acc += __ldcg(p.dHead + (int64_t)bb * J + j);
                    acc = warp_sum(acc);
                    if (lane == 0) gp[p.bh + j] = acc;
                }
            } else {
                // 64-unit tile; thread = (unit, quarter of the samples); fixed-order reduction
                const int ut = c / hd_passes, pass = c % hd_passes;
                const int u0 = ut * HD_U, ul = threadIdx.x % HD_U, qtr = threadIdx.x / HD_U;
                int jlo, jn;   // head rows of this tile and pass
                if (p.dueling) {
                    if (u0 < p.S) { jlo = 0; jn = pass == 0 ? 1 : 0; }
                    else { jlo = 1 + 8 * pass; jn = min(8, p.A - 8 * pass); }
                } else {
                    jlo = 8 * pass; jn = min(8, J - 8 * pass);
                }
                float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                float *hsm = k3raw;                    // [<=128][HD_U]
                float *dsm = k3raw + 128 * HD_U;       // [<=128][J]
                float *red = dsm + 128 * F_MAXJ;       // [4][HD_U][8]
                for (int c0 = kb; c0 < ke; c0 += 128) {
                    const int cn = min(128, ke - c0);
                    __syncthreads();
                    if (u0 + HD_U <= N1) {
                        for (int e = threadIdx.x; e < cn * (HD_U / 4); e += F_NT3) {
                            const int bb = e / (HD_U / 4), q = e % (HD_U / 4);
                            cp_async16(hsm + bb * HD_U + 4 * q, p.H1 + (int64_t)(c0 + bb) * N1 + u0 + 4 * q);
                        }
                    } else {
                        for (int e = threadIdx.x; e < cn * HD_U; e += F_NT3) {
                            const int bb = e / HD_U, q = e % HD_U;
                            hsm[e] = u0 + q < N1 ? __ldcg(p.H1 + (int64_t)(c0 + bb) * N1 + u0 + q) : 0.0f;
                        }
                    }
                    pdl_wait();   // dHead is K2's
                    for (int e = threadIdx.x; e < cn * J; e += F_NT3) cp_async4(dsm + e, p.dHead + (int64_t)c0 * J + e);
                    cp_async_wait_all();
                    __syncthreads();
                    const int q0 = (cn * qtr) / 4, q1 = (cn * (qtr + 1)) / 4;
                    for (int bb = q0; bb < q1; ++bb) {
                        const float h = hsm[bb * HD_U + ul];
                        const float *dr = dsm + bb * J + jlo;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj)
                            if (jj < jn) acc[jj] = fmaf(dr[jj], h, acc[jj]);
                    }
                }
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) red[(qtr * HD_U + ul) * 8 + jj] = acc[jj];
                __syncthreads();
                for (int o = threadIdx.x; o < HD_U * 8; o += F_NT3) {
                    const int uu = o / 8, jj = o % 8, unit = u0 + uu;
                    if (jj >= jn || unit >= N1) continue;
                    const float v = ((red[(0 * HD_U + uu) * 8 + jj] + red[(1 * HD_U + uu) * 8 + jj]) +
                                     red[(2 * HD_U + uu) * 8 + jj]) + red[(3 * HD_U + uu) * 8 + jj];
                    const int j = jlo + jj;
                    int64_t dst;
                    if (!p.dueling) dst = p.wh + (int64_t)j * N1 + unit;
                    else if (j == 0) dst = p.wh + unit;
                    else dst = p.wh + (int64_t)j * p.S + (unit - p.S);
                    gp[dst] = v;
                }
            }
        }
    }
    write_pending();
}

// the step's loss into the caller's slot (possibly pinned host memory) from a one-CTA kernel on
// a side branch of the step graph that forks after K3 and joins after K4: the PCIe write and
// its completion overlap K4 instead of delaying the end of the step's last kernel
// (its own small argument struct: the destination changes every step, and a graph node update
// of a small parameter block is cheaper than one of FastArgs)
struct LossArgs {
    const float *loss_part;
    int B;
    float *loss_out;
};
__global__ void __launch_bounds__(256) loss_out_kernel(const __grid_constant__ LossArgs a)
{
    // the batch-mean loss exactly as K4 forms it (block_batch_loss's order)
    __shared__ float red8[8];
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    float ls = 0.0f;
    for (int b = tid; b < a.B; b += 256) ls += __ldcg(a.loss_part + b);
    ls = warp_sum(ls);
    if (lane == 0) red8[wq] = ls;
    __syncthreads();
    float lsum = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) lsum += red8[w];
    if (tid == 0) *a.loss_out = lsum / (float)a.B;
}

// ------------------------------------------------------------------------------------------
// K4: layer-0 backward + SGD of every parameter + target sync + counters
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) fast_bwd0_sgd_kernel(const __grid_constant__ FastArgs p)
{
    pdl_wait();
    CtaTrace trace_(p.trace, 3);
    constexpr int NWK4 = NT / 32;
    __shared__ float red[NWK4];
    __shared__ float wsum[NWK4][32];
    const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    const int B = p.B;
    const int64_t stride = (int64_t)gridDim.x * NT;
    // Every load of the kernel's first round is issued before anything waits on one: the
    // loss partials, the sync flag, this thread's first W0 partials and its first float4 of
    // [w1, P) (grad + weights).
    // (1) batch-mean loss (fixed-order reduction, identical in every CTA)
    float ls = 0.0f;
    for (int b = tid; b < B; b += NT) ls += __ldcg(p.loss_part + b);
    const int do_sync = __ldcg(p.sync_flag);
    // (2) W0, b0: the fixed-order sum of the (split, batch tile) partials written by K3.  A
    // CTA owns 32 consecutive elements; warp w sums partials q = w, w + 8, ... (compensated,
    // in order; coalesced 128-B loads), then the 8 warp sums are added in warp order.
    // (wide inputs: W0 / b0 are wide_dw0_kernel's, which also gets dZ0 from here)
    const int64_t n0el = p.PdH0 ? 0 : p.w1;     // W0 and b0 lead the blob
    const int nparts = (p.tc || p.tcb) ? p.nw0 : p.NS * ((B + BM - 1) / BM);
    auto w0_partial = [&](int64_t i) {
        float g = 0.0f, comp = 0.0f;
        if (i >= n0el) return g;
        for (int q0 = wq; q0 < nparts; q0 += 8 * NWK4) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int qq = q0 + q * NWK4;
                v[q] = qq < nparts ? __ldcg(p.w0part + (int64_t)qq * n0el + i) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float yv = v[q] - comp;
                const float tv = g + yv;
                comp = (tv - g) - yv;
                g = tv;
            }
        }
        return g;
    };
    // (3) first float4 of the elementwise SGD over [w1, P)
    const int64_t lo = p.w1, n_el = p.P - p.w1;
    // float4 groups: the single-split gradient, or (large-batch path, w1 % 4 == 0) the sum of
    // the batch-split partials with W1's bf16 image written from the new weights
    const bool split4 = p.nsb > 1 && (p.w1 & 3) == 0 && (p.gps & 3) == 0 && (!p.w1img || (p.N0 & 3) == 0);
    const int64_t n4 = ((p.nsb == 1 && !p.w1img) || split4) ? n_el / 4 : 0;
    int64_t e4 = (int64_t)blockIdx.x * NT + tid;
    float4 g4 = make_float4(0.f, 0.f, 0.f, 0.f), w4 = g4;
    if (e4 < n4 && p.nsb == 1) {
        g4 = __ldcg(reinterpret_cast<const float4 *>(p.grad + lo + 4 * e4));
        w4 = *reinterpret_cast<const float4 *>(p.online + lo + 4 * e4);
    }
    int64_t i0 = (int64_t)blockIdx.x * 32;
    float g = w0_partial(i0 + lane);
    ls = warp_sum(ls);
    if (lane == 0) red[wq] = ls;
    wsum[wq][lane] = g;
    __syncthreads();
    float lsum = 0.0f;
    for (int w = 0; w < NWK4; ++w) lsum += red[w];
    const float loss = lsum / (float)B;
    const bool ok = isfinite(loss);
    const bool upd = p.apply_update && ok;
    // the loss leaves first: a caller's loss_out may be pinned host memory, and that PCIe write
    // then completes while the SGD below runs instead of at the kernel's end
    if (blockIdx.x == 0 && tid == 0) {
        p.grad[p.P] = loss;
        if (p.loss_out && !p.loss_early) *p.loss_out = loss;
    }
    const float lr = p.lr;
    trace_.mark(2);
    auto w0_finish = [&](int64_t i) {
        if (wq != 0 || i >= n0el) return;
        float t = 0.0f;
#pragma unroll
        for (int w = 0; w < NWK4; ++w) t += wsum[w][lane];
        p.grad[i] = t;
        if (upd) {
            const float w = p.online[i] - lr * t;
            p.online[i] = w;
            if (do_sync) p.target[i] = w;
            if (p.w0t && i < (int64_t)p.N0 * p.D) {   // the large-batch path's W0^T for T0
                const int ii = (int)i, u = ii / p.D, dd = ii - u * p.D;   // (W0 indices fit in 32 bits)
                p.w0t[(int64_t)dd * p.N0 + u] = w;
                if (do_sync) p.w0t[(int64_t)(p.D + dd) * p.N0 + u] = w;
            }
        }
    };
    w0_finish(i0 + lane);
    for (i0 += (int64_t)gridDim.x * 32; i0 < n0el; i0 += (int64_t)gridDim.x * 32) {
        g = w0_partial(i0 + lane);
        __syncthreads();   // wsum reuse
        wsum[wq][lane] = g;
        __syncthreads();
        w0_finish(i0 + lane);
    }
    if (p.PdH0) {
        // wide inputs: dZ0 = ReLU'(z0) * (sum of K3's dH0 split-K partials, in split order)
        // and its bf16 planes in wide_dw0_kernel's pre-tiled MN-major layout; the samples up
        // to the next multiple of 16 (read by its last MMA) get zero planes
        const int64_t nz = (int64_t)B * p.N0, pz = wd_plane_elems(B);
        const int64_t nz16 = (int64_t)((B + 15) & ~15) * p.N0;
        for (int64_t i = (int64_t)blockIdx.x * NT + tid; i < nz16; i += stride) {
            float z = 0.0f;
            if (i < nz) {
                for (int q = 0; q < p.NS; ++q) z += __ldcg(p.PdH0 + (int64_t)q * nz + i);
                z = __ldcg(p.h0_in + i) > 0.0f ? z : 0.0f;
                p.dZ0[i] = z;
            }
            uint16_t h, m, l;
            umma::split3_bf16(z, h, m, l);
            const int64_t t = wd_tix_mn((int)(i % p.N0), i / p.N0);
            p.dZ0bf[t] = h;
            p.dZ0bf[pz + t] = m;
            p.dZ0bf[2 * pz + t] = l;
        }
    }
    trace_.mark(3);
    // (4) every other parameter: [w1, P), float4 where whole
    for (; e4 < n4; e4 += stride) {
        const int64_t i = lo + 4 * e4;
        if (split4) {
            // the partials in split order, 8 float4 loads in flight (the same per-element sums)
            float4 t[8];
            g4 = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int sb0 = 0; sb0 < p.nsb; sb0 += 8) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (sb0 + k < p.nsb) t[k] = __ldcg(reinterpret_cast<const float4 *>(p.gpart + (int64_t)(sb0 + k) * p.gps + i));
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (sb0 + k < p.nsb) {
                        g4.x += t[k].x;
                        g4.y += t[k].y;
                        g4.z += t[k].z;
                        g4.w += t[k].w;
                    }
            }
            *reinterpret_cast<float4 *>(p.grad + i) = g4;
            w4 = *reinterpret_cast<const float4 *>(p.online + i);
        } else if (e4 != (int64_t)blockIdx.x * NT + tid) {
            g4 = __ldcg(reinterpret_cast<const float4 *>(p.grad + i));
            w4 = *reinterpret_cast<const float4 *>(p.online + i);
        }
        if (upd) {
            w4.x -= lr * g4.x;
            w4.y -= lr * g4.y;
            w4.z -= lr * g4.z;
            w4.w -= lr * g4.w;
            *reinterpret_cast<float4 *>(p.online + i) = w4;
            if (do_sync) *reinterpret_cast<float4 *>(p.target + i) = w4;
            if (p.w1img && i < p.w1 + (int64_t)p.N1 * p.N0) {
                // four consecutive inputs of one W1 row: 8 bytes of one core-matrix row per plane
                const int64_t e = i - p.w1, u = p.N0 == 128 ? e >> 7 : e / p.N0;
                const int k = (int)(e - u * p.N0);
                const int64_t o = ((u >> 3) * (p.N0 >> 3) + (k >> 3)) * 64 + (u & 7) * 8 + (k & 7);
                const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
                uint32_t pk[3][2];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) umma::split3_pack2(wv[2 * h2], wv[2 * h2 + 1], pk[0][h2], pk[1][h2], pk[2][h2]);
                for (int net = 0; net < (do_sync ? 2 : 1); ++net) {
                    uint16_t *im = p.w1img + net * 3 * p.w1pl;
#pragma unroll
                    for (int pl = 0; pl < 3; ++pl)
                        *reinterpret_cast<uint2 *>(im + pl * p.w1pl + o) = make_uint2(pk[pl][0], pk[pl][1]);
                }
            }
        }
    }
    for (int64_t e = 4 * n4 + (int64_t)blockIdx.x * NT + tid; e < n_el; e += stride) {
        const int64_t i = lo + e;
        float gs;
        if (p.nsb == 1) {
            gs = __ldcg(p.grad + i);
        } else {
            gs = 0.0f;
            for (int sb = 0; sb < p.nsb; ++sb) gs += __ldcg(p.gpart + (int64_t)sb * p.gps + i);
            p.grad[i] = gs;
        }
        if (upd) {
            const float w = p.online[i] - lr * gs;
            p.online[i] = w;
            if (do_sync) p.target[i] = w;
            if (p.w1img && i < p.w1 + (int64_t)p.N1 * p.N0) {
                // the large-batch path's bf16 image of W1 (tc_big.cuh) for the next step
                const int64_t e = i - p.w1, u = p.N0 == 128 ? e >> 7 : e / p.N0;
                const int k = (int)(e - u * p.N0);
                const int64_t o = ((u >> 3) * (p.N0 >> 3) + (k >> 3)) * 64 + (u & 7) * 8 + (k & 7);
                uint16_t h, m, l;
                umma::split3_bf16(w, h, m, l);
                for (int net = 0; net < (do_sync ? 2 : 1); ++net) {
                    uint16_t *im = p.w1img + net * 3 * p.w1pl;
                    im[o] = h;
                    im[p.w1pl + o] = m;
                    im[2 * p.w1pl + o] = l;
                }
            }
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        if (!ok) atomicOr(p.err, ERRBIT_NUMERIC);
        // fire-and-forget reductions (no load round trip on the kernel's tail); with wide
        // inputs the sampling gather has advanced the event already
        if (!p.event_advanced) atomicAdd(reinterpret_cast<unsigned long long *>(p.rctrl), 1ull);   // sampler event consumed
        atomicAdd(reinterpret_cast<unsigned long long *>(p.step_dev), 1ull); // executed train steps
    }
}

}  // namespace rpl
