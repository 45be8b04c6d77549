// dqn.cu -- the fused, device-resident DQN / Double-DQN train step (one cooperative launch).
//
// Paper: P:79-84 [Integration]: once the replay is on the GPU "all logic for a single train
// step can be moved to the GPU" with "no inputs copied from the CPU"; P:88-94 [Deep Q-Network
// Model]: dueling DQN (shared 128, V/A streams of 512, Q = V + A - mean A), target fixing,
// the update rule w <- w + alpha (r + gamma max Q(s',a') - Q(s,a)) grad Q(s,a).
//
// B200 design: one persistent cooperative kernel, one CTA of 256
// threads per SM, phases separated by a grid barrier:
//   F0    Philox sample + gather ring rows + layer 0 of every needed forward (online(s),
//         target(s'), [online(s')]) -- 32x64 FP32 register-tiled SIMT GEMM tiles
//   F1.. remaining trunk layers (dueling: the 128 -> [V 512 | A 512] stream layer)
//   Head  one warp per sample: V/A heads, dueling combine, max / argmax (warp shuffles), TD
//         target, Huber, dQ, dueling backward, dZ of the last trunk layer
//   Bl    backward of trunk layer l: dW_l (contraction over the batch, + bias row sums) and
//         split-K partials of dH_{l-1}; head-weight gradients in the last layer's phase
//   SGD   deterministic reduction of gradient partials, non-finite guard, w -= lr g,
//         target sync on sync steps
// All reductions run in a fixed order, so a step is bit-reproducible.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"
#include "philox.cuh"
#include "simt_gemm.cuh"
#include "train_fast.cuh"
#include "tc_fast.cuh"
#include "tc_big.cuh"
#include "wide.cuh"
#include "dp_peer.cuh"

// Variants measured slower than the default path are compiled in, and their
// environment switches read, only in an experiments build (RPL_NVCC_FLAGS=-DRPL_EXPERIMENTS);
// the default library has one kernel sequence per shape.
#ifdef RPL_EXPERIMENTS
static bool exp_flag(const char *name)
{
    const char *v = getenv(name);
    return v && v[0] == '1';
}
#else
static bool exp_flag(const char *) { return false; }
#endif

namespace rpl {

constexpr int MAXL = 5;   // trunk layers (4 shared + dueling stream layer)
constexpr int MAXA = 32;  // actions (one warp)
constexpr int MAXJ = MAXA + 1;

constexpr int kWideInput = 1024;   // state_dim above which layer 0 is split-K (wide inputs)
constexpr int kKs0Max = 80;        // layer-0 split-K chunks at most

struct TrainArgs {
    // replay
    const float *ring;
    int rs, D;
    int u8, so;            // byte states (x = u8 / 255, reading Q27); scalars at byte `so`
    int shared, sw;        // shared states (s' = next slot's s); fp32 scalar word offset
    int64_t cursor, capacity;
    int64_t size;
    uint64_t seed, event;
    uint32_t rank;
    // network layout
    int A, dueling, T, J, S, NH, nets, ddqn;
    int N[MAXL], K[MAXL];
    int64_t woff[MAXL], boff[MAXL], hw_off, hb_off, P;
    // batch
    int B;
    float gamma, lr, kappa;
    int kappa_inf;
    // parameters
    float *online, *target;
    // workspaces
    float *Xs, *Xs2, *r;
    int32_t *a, *idx;
    uint8_t *done;
    float *H[MAXL];        // [nets][B][N_l]
    float *dZlast;         // [B][NH]
    float *dO;             // [B][J]
    float *PdH[MAXL];      // layer l >= 1: [nsplit_n[l]][B][K_l]
    int nsplit_n[MAXL];
    float *gpart;          // [nsplit_b][P] (== grad when nsplit_b == 1)
    int nsplit_b, bsplit;
    float *grad;           // [P + 1] (grad[P] = batch-mean loss)
    float *loss_part;      // [B]
    float *Qs, *Qt2, *Qo2, *y;
    int32_t *astar;
    float *loss_out;
    int apply_update, do_sync;
    int wide_tc;           // layer 0 (forward partials, dW0 + its SGD) runs in wide.cuh kernels
                           // (its partials are x 255: phase_l0_reduce divides the sum)
    int distinct;          // batch indices precomputed by distinct_kernel into idx
    uint16_t *dZ0bf;       // wide_tc: bf16 hi / mid / lo planes of dZ0 [3][B][N0]
    unsigned long long *trace;   // RPL_TRACE=1: per-phase %globaltimer of CTA 0 (else null)
    int ks0;               // split-K of the layer-0 forward (wide inputs): partials in PF0
    float *PF0;            // [ks0][nets][B][N0]
    unsigned *bar;         // [0] arrivals, [1] generation
    uint32_t *err;
    uint64_t *rctrl;       // replay control block: [0] events, [1] size
    int64_t *step_dev;
    int32_t *sync_flag;
};

struct __align__(16) TileSmem : GemmSmem {
    int idx[BM];
    int idx2[BM];          // the s' row of each sampled slot (== idx unless shared states)
    float red[NT / 32];
    float head[NT / 32][MAXJ + 3];
};

// ------------------------------------------------------------------------------------------
// grid barrier (all CTAs co-resident: cooperative launch)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier(unsigned *bar)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(bar + 1);
        __threadfence();
        const unsigned arrived = atomicAdd(bar, 1u);
        if (arrived == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (ld_acquire(bar + 1) == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ float dz_val(const TrainArgs &p, int l, int b, int n)
{
    const int N = p.N[l];
    if (l == p.T - 1) return __ldcg(p.dZlast + (int64_t)b * N + n);
    if (l == 0 && p.ks0 > 1) return __ldcg(p.PF0 + (int64_t)b * N + n);   // materialised dZ0
    const float *q = p.PdH[l + 1] + (int64_t)b * N + n;
    const int64_t stride = (int64_t)p.B * N;
    float s = 0.0f;
    for (int i = 0; i < p.nsplit_n[l + 1]; ++i) s += __ldcg(q + i * stride);
    const float h = __ldcg(p.H[l] + (int64_t)b * N + n);
    return h > 0.0f ? s : 0.0f;
}
// (m = unit n, kk = sample b), contiguous along n (for dW)
struct LdDzT {
    static constexpr bool kKContig = false;
    const TrainArgs *p;
    int l, N, KB, KE;
    __device__ float operator()(int n, int b) const
    {
        return (n < N && b >= KB && b < KE) ? dz_val(*p, l, b, n) : 0.0f;
    }
};
// (m = sample b, kk = unit n), contiguous along n (for dH)
struct LdDz {
    static constexpr bool kKContig = true;
    const TrainArgs *p;
    int l, B, KB, KE;
    __device__ float operator()(int b, int n) const
    {
        return (b < B && n >= KB && n < KE) ? dz_val(*p, l, b, n) : 0.0f;
    }
};

// byte-state operands (RPL_U8 replays): x = u8 / 255 (reading Q27), an exactly rounded fp32
// quotient.  Gathered ring rows (m = sample, k = input), and the unpacked batch [B][D]
// read as (r = input, kk = sample) for dW0.
__device__ __forceinline__ float u8_input(uint8_t v) { return __fdiv_rn((float)v, 255.0f); }
struct LdRingU8 {
    static constexpr bool kKContig = true;
    const uint8_t *ring;
    const int *idx_s;
    int m0;
    int64_t rsb;
    int col0, R, KE;
    __device__ float operator()(int m, int k) const
    {
        return (m < R && k < KE) ? u8_input(__ldg(ring + (int64_t)idx_s[m - m0] * rsb + col0 + k)) : 0.0f;
    }
};
struct LdRMajorU8 {
    static constexpr bool kKContig = false;
    const uint8_t *p;
    int ld, R, KB, KE;
    __device__ float operator()(int r, int kk) const
    {
        return (r < R && kk >= KB && kk < KE) ? u8_input(__ldcg(p + (int64_t)kk * ld + r)) : 0.0f;
    }
};

// ------------------------------------------------------------------------------------------
// phases
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ const float *net_params(const TrainArgs &p, int net)
{
    return net == 1 ? p.target : p.online;
}

// F0 / Fl: forward of trunk layer l for every needed net.  Layer 0 samples + gathers its
// rows; with a wide input (ks0 > 1) its contraction is split into ks0 chunks whose partial
// sums go to PF0 and are reduced (+ bias, ReLU) by phase_l0_reduce after a grid barrier.
__device__ void phase_forward(const TrainArgs &p, int l, TileSmem &sm)
{
    const int N = p.N[l], K = p.K[l], B = p.B;
    const int mt = (B + BM - 1) / BM, nt = (N + BN - 1) / BN;
    const int ks = l == 0 ? p.ks0 : 1;
    const int kchunk = ((K + ks - 1) / ks + BK - 1) / BK * BK;
    const int ntasks = p.nets * mt * nt * ks;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        const int kq = t / (p.nets * mt * nt), tt = t % (p.nets * mt * nt);
        const int net = tt / (mt * nt), rem = tt % (mt * nt);
        const int m0 = (rem / nt) * BM, n0 = (rem % nt) * BN;
        const int kb = kq * kchunk, ke = min(K, kb + kchunk);
        const float *theta = net_params(p, net);
        const float *W = theta + p.woff[l];
        const float *bias = theta + p.boff[l];
        float *Hout = p.H[l] + (int64_t)net * B * N;
        float *Pout = ks > 1 ? p.PF0 + ((int64_t)kq * p.nets + net) * B * N : nullptr;
        auto epi = [&](int m, int n, float v) {
            if (m < B && n < N) {
                if (Pout) {
                    Pout[(int64_t)m * N + n] = v;
                } else {
                    v += __ldg(bias + n);
                    Hout[(int64_t)m * N + n] = v > 0.0f ? v : 0.0f;
                }
            }
        };
        LdKMajor lw{W, K, N, ke};
        if (l == 0) {
            // sample (Philox, event E) + gather: the batch rows m0..m0+BM
            __syncthreads();
            if (threadIdx.x < BM / 2) {
                const int pair = (m0 >> 1) + threadIdx.x;
                int32_t i0, i1;
                if (p.distinct) {
                    i0 = 2 * pair < B ? p.idx[2 * pair] : 0;
                    i1 = 2 * pair + 1 < B ? p.idx[2 * pair + 1] : 0;
                } else {
                    // shared states: logical positions over all but the newest experience
                    const int64_t nvalid = p.shared ? p.size - 1 : p.size;
                    const uint64_t oldest = (p.shared && p.size == p.capacity) ? (uint64_t)p.cursor : 0;
                    sample_pair(p.seed, p.rank, p.event, (uint32_t)pair, (uint64_t)nvalid, i0, i1);
                    i0 = slot_of(i0, oldest, p.capacity);
                    i1 = slot_of(i1, oldest, p.capacity);
                }
                sm.idx[2 * threadIdx.x] = i0;
                sm.idx[2 * threadIdx.x + 1] = i1;
                sm.idx2[2 * threadIdx.x] = p.shared ? (int)((i0 + 1) % p.capacity) : i0;
                sm.idx2[2 * threadIdx.x + 1] = p.shared ? (int)((i1 + 1) % p.capacity) : i1;
            }
            __syncthreads();
            const int D = p.D;
            // s for online(s), s' for the others: the same row's second state, or the next
            // slot's state with shared states
            const int col0 = (net == 0 || p.shared) ? 0 : D;
            const int *rows_s = (net == 0) ? sm.idx : sm.idx2;
            // unpack the batch once (online(s) / target(s') tasks of the first column tile)
            if (n0 == 0 && net <= 1 && kq == 0) {
                if (p.u8) {
                    const uint8_t *rb = reinterpret_cast<const uint8_t *>(p.ring);
                    uint8_t *xo = reinterpret_cast<uint8_t *>(net == 0 ? p.Xs : p.Xs2);
                    for (int e = threadIdx.x; e < BM * D; e += NT) {
                        const int r = e / D, c = e % D;
                        if (m0 + r < B)
                            xo[(int64_t)(m0 + r) * D + c] = __ldg(rb + (int64_t)rows_s[r] * p.rs * 4 + col0 + c);
                    }
                } else {
                    for (int e = threadIdx.x; e < BM * D; e += NT) {
                        const int r = e / D, c = e % D;
                        if (m0 + r < B)
                            (net == 0 ? p.Xs : p.Xs2)[(int64_t)(m0 + r) * D + c] =
                                __ldg(p.ring + (int64_t)rows_s[r] * p.rs + col0 + c);
                    }
                }
                if (net == 0 && threadIdx.x < BM && m0 + threadIdx.x < B) {
                    const int r = threadIdx.x, b = m0 + r;
                    const float *row = p.u8 ? reinterpret_cast<const float *>(
                                                  reinterpret_cast<const uint8_t *>(p.ring) +
                                                  (int64_t)sm.idx[r] * p.rs * 4 + p.so)
                                            : p.ring + (int64_t)sm.idx[r] * p.rs + p.sw;
                    p.idx[b] = sm.idx[r];
                    p.a[b] = __float_as_int(__ldg(row));
                    p.r[b] = __ldg(row + 1);
                    p.done[b] = (uint8_t)(__float_as_uint(__ldg(row + 2)) != 0u);
                }
            }
            if (p.u8) {
                LdRingU8 lx{reinterpret_cast<const uint8_t *>(p.ring), rows_s, m0, (int64_t)p.rs * 4,
                            col0, B, ke};
                gemm_tile(lx, lw, m0, n0, kb, ke, epi, false, NoRowsum{}, sm);
            } else {
                LdRing lx{p.ring, rows_s, m0, p.rs, col0, B, ke};
                gemm_tile(lx, lw, m0, n0, kb, ke, epi, false, NoRowsum{}, sm);
            }
        } else {
            LdKMajor lh{p.H[l - 1] + (int64_t)net * B * K, K, B, K};
            gemm_tile(lh, lw, m0, n0, 0, K, epi, false, NoRowsum{}, sm);
        }
    }
}

// wide inputs: dZ0 = (sum of the dH0 split-K partials) * ReLU'(z0) materialised once in PF0
// (free after the layer-0 reduction) for the many dW0 tiles, in dz_val's order
__device__ void phase_dz0(const TrainArgs &p)
{
    const int N = p.N[0];
    const int64_t total = (int64_t)p.B * N, stride = (int64_t)gridDim.x * NT;
    const int64_t pstride = (int64_t)p.B * N;
    // wide_tc: the samples up to the next multiple of 16 get zero planes (wide_dw0_kernel)
    const int64_t total16 = p.wide_tc ? (int64_t)((p.B + 15) & ~15) * N : total;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < total16; i += stride) {
        float z = 0.0f;
        if (i < total) {
            float s = 0.0f;
            for (int q = 0; q < p.nsplit_n[1]; ++q) s += __ldcg(p.PdH[1] + q * pstride + i);
            z = __ldcg(p.H[0] + i) > 0.0f ? s : 0.0f;
            p.PF0[i] = z;
        }
        if (p.wide_tc) {   // the dW0 kernel's tensor-core operand, split once, pre-tiled
            uint16_t h, m, l;
            umma::split3_bf16(z, h, m, l);
            const int64_t t = wd_tix_mn((int)(i % N), i / N), pz = wd_plane_elems(p.B);
            p.dZ0bf[t] = h;
            p.dZ0bf[pz + t] = m;
            p.dZ0bf[2 * pz + t] = l;
        }
    }
}

// layer-0 split-K reduction: H0 = ReLU(sum_q PF0[q] + b0), partials added in chunk order
__device__ void phase_l0_reduce(const TrainArgs &p)
{
    const int N = p.N[0], B = p.B;
    const int64_t per_net = (int64_t)B * N, total = (int64_t)p.nets * per_net;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < total; i += stride) {
        const int net = (int)(i / per_net), n = (int)(i % N);
        float v = 0.0f;
        for (int q = 0; q < p.ks0; ++q) v += __ldcg(p.PF0 + (int64_t)q * total + i);
        if (p.wide_tc) v = v / 255.0f;   // tensor-core partials carry u, not u / 255
        v += __ldg(net_params(p, net) + p.boff[0] + n);
        p.H[0][i] = v > 0.0f ? v : 0.0f;
    }
}

__device__ __forceinline__ float huber(float d, float kappa, int kinf)
{
    const float ad = fabsf(d);
    if (kinf || ad <= kappa) return 0.5f * d * d;
    return kappa * (ad - 0.5f * kappa);
}

// Head: one warp per sample
__device__ void phase_head(const TrainArgs &p, TileSmem &sm)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nw = NT / 32;
    const int A = p.A, J = p.J, S = p.S, NH = p.NH, B = p.B;
    const int L = p.T - 1;
    float *hs = sm.head[wib];
    for (int b = blockIdx.x + gridDim.x * wib; b < B; b += gridDim.x * nw) {
        float q0 = 0.0f, q1 = 0.0f, q2 = 0.0f;   // lane a < A holds Q_net(., a)
        for (int net = 0; net < p.nets; ++net) {
            const float *theta = net_params(p, net);
            const float *Wh = theta + p.hw_off;
            const float *bh = theta + p.hb_off;
            const float *h = p.H[L] + ((int64_t)net * B + b) * NH;
            for (int j = 0; j < J; ++j) {
                // head row j over its input units: dueling V row over the V units, A rows over
                // the A units; float4 loads, four in flight per lane where aligned
                const int len = p.dueling ? S : NH;
                const float *w = Wh + (int64_t)j * len;
                const float *hh = p.dueling ? h + (j == 0 ? 0 : S) : h;
                float acc = 0.0f;
                if ((len & 3) == 0 && (((uintptr_t)w | (uintptr_t)hh) & 15) == 0) {
                    const float4 *w4 = reinterpret_cast<const float4 *>(w);
                    const float4 *h4 = reinterpret_cast<const float4 *>(hh);
                    const int n4 = len >> 2;
                    int u = lane;
                    for (; u + 96 < n4; u += 128) {
                        float4 wv[4], hv[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            wv[q] = __ldg(w4 + u + 32 * q);
                            hv[q] = __ldcg(h4 + u + 32 * q);
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            acc = fmaf(wv[q].x, hv[q].x, acc);
                            acc = fmaf(wv[q].y, hv[q].y, acc);
                            acc = fmaf(wv[q].z, hv[q].z, acc);
                            acc = fmaf(wv[q].w, hv[q].w, acc);
                        }
                    }
                    for (; u < n4; u += 32) {
                        const float4 wv = __ldg(w4 + u), hv = __ldcg(h4 + u);
                        acc = fmaf(wv.x, hv.x, acc);
                        acc = fmaf(wv.y, hv.y, acc);
                        acc = fmaf(wv.z, hv.z, acc);
                        acc = fmaf(wv.w, hv.w, acc);
                    }
                } else {
                    for (int u = lane; u < len; u += 32) acc = fmaf(__ldg(w + u), __ldcg(hh + u), acc);
                }
                acc = warp_sum(acc);
                if (lane == 0) hs[j] = acc + __ldg(bh + j);
            }
            __syncwarp();
            float qa = 0.0f;
            if (p.dueling) {
                // Q(s,a) = V(s) + A(s,a) - (1/|A|) sum_a' A(s,a')
                float mean = 0.0f;
                for (int a = 0; a < A; ++a) mean += hs[1 + a];
                mean /= (float)A;
                if (lane < A) qa = hs[0] + hs[1 + lane] - mean;
            } else if (lane < A) {
                qa = hs[lane];
            }
            if (net == 0) q0 = qa; else if (net == 1) q1 = qa; else q2 = qa;
            __syncwarp();
        }
        // TD target (Q9): DQN max_a Q_t(s',a); DDQN Q_t(s', argmax_a Q_o(s',a))
        float boot;
        int astar = -1;
        if (!p.ddqn) {
            float m = lane < A ? q1 : -INFINITY;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            boot = m;
        } else {
            float v = lane < A ? q2 : -INFINITY;
            int ix = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
                if (ov > v || (ov == v && oi < ix)) { v = ov; ix = oi; }   // ties: lowest index
            }
            astar = ix;
            boot = __shfl_sync(0xffffffffu, q1, astar);
        }
        const int ab = p.a[b];
        const float rb = p.r[b];
        const float notdone = p.done[b] ? 0.0f : 1.0f;
        const float yb = rb + p.gamma * notdone * boot;
        // the enumerate-mask gather Q[i*A + a_i] is a register select here
        const float qsel = __shfl_sync(0xffffffffu, q0, ab & 31);
        // an action outside [0, A) poisons the loss (the update is skipped) and raises ECORRUPT
        const bool bad = (unsigned)ab >= (unsigned)A;
        if (bad && lane == 0) atomicOr(p.err, ERRBIT_CORRUPT);
        const float delta = bad ? __int_as_float(0x7fc00000) : qsel - yb;
        const float g = (p.kappa_inf ? delta : fminf(fmaxf(delta, -p.kappa), p.kappa)) / (float)B;
        // dL/dhead: plain dO_j = [j==a]g ; dueling dV = g, dA_j = [j==a]g - g/|A|
        if (p.dueling) {
            if (lane == 0) hs[0] = g;
            if (lane < A) hs[1 + lane] = (lane == ab ? g : 0.0f) - g / (float)A;
        } else if (lane < A) {
            hs[lane] = lane == ab ? g : 0.0f;
        }
        __syncwarp();
        for (int j = lane; j < J; j += 32) p.dO[(int64_t)b * J + j] = hs[j];
        if (lane < A) {
            p.Qs[(int64_t)b * A + lane] = q0;
            p.Qt2[(int64_t)b * A + lane] = q1;
            if (p.ddqn) p.Qo2[(int64_t)b * A + lane] = q2;
        }
        if (lane == 0) {
            p.y[b] = yb;
            p.loss_part[b] = huber(delta, p.kappa, p.kappa_inf);
            if (p.ddqn) p.astar[b] = astar;
        }
        // dZ of the last trunk layer: (dO . W_head) * ReLU'(z)
        const float *Wh = p.online + p.hw_off;
        const float *h0 = p.H[L] + (int64_t)b * NH;
        for (int u = lane; u < NH; u += 32) {
            float dh = 0.0f;
            if (p.dueling) {
                if (u < S) {
                    dh = hs[0] * __ldg(Wh + u);
                } else {
                    for (int a = 0; a < A; ++a) dh = fmaf(hs[1 + a], __ldg(Wh + (int64_t)(1 + a) * S + (u - S)), dh);
                }
            } else {
                for (int a = 0; a < A; ++a) dh = fmaf(hs[a], __ldg(Wh + (int64_t)a * NH + u), dh);
            }
            p.dZlast[(int64_t)b * NH + u] = __ldcg(h0 + u) > 0.0f ? dh : 0.0f;
        }
        __syncwarp();
    }
}

// backward of trunk layer l (+ the head weights when l == T-1)
__device__ void phase_backward(const TrainArgs &p, int l, TileSmem &sm)
{
    const int N = p.N[l], K = p.K[l], B = p.B;
    // (i) dW_l tiles: M = N units, N-dim = K inputs, contraction over the b-split
    const int wmt = (N + BM - 1) / BM, wnt = (K + BN - 1) / BN;
    const int n_w = wmt * wnt * p.nsplit_b;
    // (ii) dH_{l-1} split-K partials: M = B, N-dim = K, contraction over units
    const int hmt = (B + BM - 1) / BM, hnt = (K + BN - 1) / BN;
    const int n_h = l > 0 ? hmt * hnt * p.nsplit_n[l] : 0;
    // (iii) head weight gradients (l == T-1) as GEMM tiles over (head row j, head-input unit u):
    //       g_Wh[j][u] = sum_b dO[b][j] h[b][u], per b-split; the bias rows come with n0 == 0
    const int hjt = (p.J + BM - 1) / BM, hut = (p.NH + BN - 1) / BN;
    const int n_hd = (l == p.T - 1) ? hjt * hut * p.nsplit_b : 0;
    const float *Hprev = (l == 0) ? p.Xs : p.H[l - 1];
    const int ntasks = n_w + n_h + n_hd;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        if (t < n_w) {
            const int s = t / (wmt * wnt), rem = t % (wmt * wnt);
            const int m0 = (rem / wnt) * BM, n0 = (rem % wnt) * BN;
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit);
            float *gp = p.gpart + (int64_t)s * p.P;
            LdDzT la{&p, l, N, kb, ke};
            auto epi = [&](int m, int n, float v) {
                if (m < N && n < K) gp[p.woff[l] + (int64_t)m * K + n] = v;
            };
            auto rs = [&](int m, float v) {
                if (m < N) gp[p.boff[l] + m] = v;
            };
            if (l == 0 && p.u8) {
                LdRMajorU8 lb{reinterpret_cast<const uint8_t *>(Hprev), K, K, kb, ke};
                gemm_tile(la, lb, m0, n0, kb, ke, epi, n0 == 0, rs, sm);
            } else {
                LdRMajor lb{Hprev, K, K, kb, ke};
                gemm_tile(la, lb, m0, n0, kb, ke, epi, n0 == 0, rs, sm);
            }
        } else if (t < n_w + n_h) {
            const int u = t - n_w;
            const int s = u / (hmt * hnt), rem = u % (hmt * hnt);
            const int m0 = (rem / hnt) * BM, n0 = (rem % hnt) * BN;
            const int chunk = (N + p.nsplit_n[l] - 1) / p.nsplit_n[l];
            const int kb = s * chunk, ke = min(N, kb + chunk);
            float *out = p.PdH[l] + (int64_t)s * B * K;
            LdDz la{&p, l, B, kb, ke};
            LdRMajor lb{p.online + p.woff[l], K, K, kb, ke};
            auto epi = [&](int m, int n, float v) {
                if (m < B && n < K) out[(int64_t)m * K + n] = v;
            };
            gemm_tile(la, lb, m0, n0, kb, ke, epi, false, NoRowsum{}, sm);
        } else {
            // head gradients: g_Wh[j][u] = sum_b dO[b][j] h[b][u]; g_bh[j] = sum_b dO[b][j]
            const int u = t - n_w - n_h;
            const int s = u / (hjt * hut), rem = u % (hjt * hut);
            const int m0 = (rem / hut) * BM, n0 = (rem % hut) * BN;
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit);
            float *gp = p.gpart + (int64_t)s * p.P;
            const int J = p.J, NH = p.NH, S = p.S;
            LdRMajor la{p.dO, J, J, kb, ke};
            LdRMajor lb{p.H[p.T - 1], NH, NH, kb, ke};   // online net on s
            auto epi = [&](int j, int unit, float v) {
                if (j >= J || unit >= NH) return;
                if (!p.dueling) gp[p.hw_off + (int64_t)j * NH + unit] = v;
                else if (j == 0 && unit < S) gp[p.hw_off + unit] = v;                          // V head
                else if (j > 0 && unit >= S) gp[p.hw_off + (int64_t)j * S + (unit - S)] = v;   // A head
            };
            auto rs = [&](int j, float v) {
                if (j < J) gp[p.hb_off + j] = v;
            };
            gemm_tile(la, lb, m0, n0, kb, ke, epi, n0 == 0, rs, sm);
        }
    }
}

__device__ float block_sum_fixed(float v, TileSmem &sm)
{
    v = warp_sum(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
    __syncthreads();
    float s = 0.0f;
    for (int w = 0; w < NT / 32; ++w) s += sm.red[w];   // same order in every thread/CTA
    return s;
}

// SGD: deterministic reduction of the b-split partials, non-finite guard,
// w -= lr g, target sync on sync steps
__device__ void phase_sgd(const TrainArgs &p, TileSmem &sm)
{
    float ls = 0.0f;
    for (int b = threadIdx.x; b < p.B; b += NT) ls += __ldcg(p.loss_part + b);
    const float loss = block_sum_fixed(ls, sm) / (float)p.B;
    const bool ok = isfinite(loss);
    const int64_t stride = (int64_t)gridDim.x * NT;
    const int64_t w0b = p.woff[0], w0e = p.woff[0] + (int64_t)p.N[0] * p.K[0];
    for (int64_t i = (int64_t)blockIdx.x * NT + threadIdx.x; i < p.P; i += stride) {
        float g;
        if (p.wide_tc && i >= w0b && i < w0e) continue;   // W0: wide_dw0_kernel
        if (p.wide_tc && i >= p.boff[0] && i < p.boff[0] + p.N[0]) {
            // db0 = sum_b dZ0[b][u] (dZ0 materialised in PF0), in sample order
            const int u = (int)(i - p.boff[0]);
            g = 0.0f;
            for (int b = 0; b < p.B; ++b) g += __ldcg(p.PF0 + (int64_t)b * p.N[0] + u);
            p.grad[i] = g;
        } else if (p.nsplit_b == 1) {
            g = __ldcg(p.grad + i);
        } else {
            g = 0.0f;
            for (int s = 0; s < p.nsplit_b; ++s) g += __ldcg(p.gpart + (int64_t)s * p.P + i);
            p.grad[i] = g;
        }
        if (p.apply_update && ok) {
            const float w = p.online[i] - p.lr * g;
            p.online[i] = w;
            if (p.do_sync) p.target[i] = w;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.grad[p.P] = loss;
        if (p.loss_out) *p.loss_out = loss;
        if (!ok) atomicOr(p.err, ERRBIT_NUMERIC);
        p.rctrl[0] = p.event + 1;
        *p.step_dev += 1;
        *p.sync_flag = p.do_sync;
    }
}

__global__ void __launch_bounds__(NT, 1) train_step_kernel(const __grid_constant__ TrainArgs p)
{
    __shared__ TileSmem sm;
    // RPL_TRACE=1: %globaltimer after every phase (CTA 0), slots of kernel 0 in the trace
    int mk = 0;
    auto mark = [&]() {
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            p.trace[mk] = t;
        }
        ++mk;
    };
    mark();
    for (int l = 0; l < p.T; ++l) {
        if (!(l == 0 && p.wide_tc)) {   // wide_tc: sampled, gathered and multiplied already
            phase_forward(p, l, sm);
            grid_barrier(p.bar);
        }
        mark();
        if (l == 0 && p.ks0 > 1) {
            phase_l0_reduce(p);
            grid_barrier(p.bar);
        }
        mark();
    }
    phase_head(p, sm);
    grid_barrier(p.bar);
    mark();
    for (int l = p.T - 1; l >= 0; --l) {
        if (l == 0 && p.ks0 > 1 && p.T > 1) {
            phase_dz0(p);
            grid_barrier(p.bar);
        }
        mark();
        if (l == 0 && p.wide_tc) break;   // dW0 and its SGD follow in wide_dw0_kernel
        phase_backward(p, l, sm);
        grid_barrier(p.bar);
        mark();
    }
    phase_sgd(p, sm);
    mark();
}

// SGD after an NCCL all-reduce (world > 1): grad[P] holds the rank-averaged loss
// the SGD after an NCCL all-reduce (grad = the ranks' mean, word P = the mean loss): DP_U float4
// groups per thread and round with their loads in flight, the scalar tail after; W0's bf16
// planes rewritten for byte-state learners (as the peer-memory exchange does: DPArgs fields)
struct SgdArgs {
    float *online, *target;
    const float *grad;
    int64_t P;
    float lr;
    const int32_t *sync_flag;
    uint32_t *err;
    float *loss_out;      // the mean loss for the caller (or null)
    W0Planes planes;      // byte-state learners: W0's bf16 planes rewritten with W0 (.bf null: none)
};
__global__ void __launch_bounds__(256) sgd_kernel(const __grid_constant__ SgdArgs a)
{
    const int do_sync = *a.sync_flag;
    const float loss = a.grad[a.P];
    const bool ok = isfinite(loss);
    if (a.loss_out && blockIdx.x == 0 && threadIdx.x == 0) *a.loss_out = loss;   // the ranks' mean loss
    const int64_t S = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(a.online) | reinterpret_cast<uintptr_t>(a.target) |
                       reinterpret_cast<uintptr_t>(a.grad)) & 15) == 0;
    const int64_t P4 = vec ? a.P / 4 : 0;
    if (ok) {
        for (int64_t j0 = t0; j0 < P4; j0 += DP_U * S) {
            float4 g[DP_U], w[DP_U];
#pragma unroll
            for (int u = 0; u < DP_U; ++u) {
                const bool in = j0 + u * S < P4;
                g[u] = in ? __ldcg(reinterpret_cast<const float4 *>(a.grad) + j0 + u * S) : make_float4(0.f, 0.f, 0.f, 0.f);
                w[u] = in ? reinterpret_cast<const float4 *>(a.online)[j0 + u * S] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < DP_U; ++u) {
                const int64_t j = j0 + u * S;
                if (j >= P4) continue;
                const float4 nw = make_float4(w[u].x - a.lr * g[u].x, w[u].y - a.lr * g[u].y, w[u].z - a.lr * g[u].z,
                                              w[u].w - a.lr * g[u].w);
                reinterpret_cast<float4 *>(a.online)[j] = nw;
                if (do_sync) reinterpret_cast<float4 *>(a.target)[j] = nw;
                dp_w0_planes4(a.planes, j, nw, do_sync);
            }
        }
        for (int64_t i = 4 * P4 + t0; i < a.P; i += S) {
            const float w = a.online[i] - a.lr * a.grad[i];
            a.online[i] = w;
            if (do_sync) a.target[i] = w;
            dp_w0_planes(a.planes, i, w, do_sync);
        }
    }
    if (!ok && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.err, ERRBIT_NUMERIC);
}

// ------------------------------------------------------------------------------------------
// NCCL (dlopen of the process's libnccl.so.2 -- the one torch loaded)
// ------------------------------------------------------------------------------------------
typedef struct { char internal[128]; } nccl_uid;
typedef int (*fn_get_uid)(nccl_uid *);
typedef int (*fn_init_rank)(void **, int, nccl_uid, int);
typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*fn_destroy)(void *);
typedef const char *(*fn_errstr)(int);
struct NcclApi {
    bool loaded = false;
    fn_get_uid get_uid = nullptr;
    fn_init_rank init_rank = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_destroy destroy = nullptr;
    fn_errstr errstr = nullptr;
};
static NcclApi g_nccl;
static int nccl_load()
{
    if (g_nccl.loaded) return RPL_OK;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        set_error("NCCL: dlopen(libnccl.so.2) failed: %s", dlerror());
        return RPL_ENCCL;
    }
    g_nccl.get_uid = (fn_get_uid)dlsym(h, "ncclGetUniqueId");
    g_nccl.init_rank = (fn_init_rank)dlsym(h, "ncclCommInitRank");
    g_nccl.allreduce = (fn_allreduce)dlsym(h, "ncclAllReduce");
    g_nccl.destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
    g_nccl.errstr = (fn_errstr)dlsym(h, "ncclGetErrorString");
    if (!g_nccl.get_uid || !g_nccl.init_rank || !g_nccl.allreduce || !g_nccl.destroy) {
        set_error("NCCL: missing symbols in libnccl.so.2");
        return RPL_ENCCL;
    }
    g_nccl.loaded = true;
    return RPL_OK;
}
constexpr int kNcclFloat = 7;   // ncclFloat32
constexpr int kNcclAvg = 4;     // ncclAvg

}  // namespace rpl

using namespace rpl;

// ==========================================================================================
// learner handle + C-ABI
// ==========================================================================================
struct rpl_dqn {
    int device = 0;
    cudaStream_t stream = nullptr;
    rpl_dqn_config cfg{};
    // layout
    int T = 0, J = 0, NH = 0;
    int N[MAXL] = {}, K[MAXL] = {};
    int64_t woff[MAXL] = {}, boff[MAXL] = {}, hw_off = 0, hb_off = 0, P = 0, Htot = 0;
    int sms = 148;
    // device memory
    float *online = nullptr, *target = nullptr, *grad = nullptr, *gpart = nullptr;
    float *Xs = nullptr, *Xs2 = nullptr, *r = nullptr;
    int32_t *a = nullptr, *idx = nullptr, *astar = nullptr;
    uint8_t *done = nullptr;
    float *H[MAXL] = {}, *dZlast = nullptr, *dO = nullptr, *PdH[MAXL] = {};
    float *loss_part = nullptr, *Qs = nullptr, *Qt2 = nullptr, *Qo2 = nullptr, *y = nullptr;
    float *loss_dev = nullptr;
    unsigned *bar = nullptr;
    uint32_t *err = nullptr;
    int64_t gpart_elems = 0, pdh_elems[MAXL] = {};
    int64_t steps = 0;
    int last_B = 0;
    int last_u8 = 0;                 // the last step's replay stores byte states
    // wide inputs: layer-0 forward split-K partials [kKs0Max][nets][max_batch][N0]
    float *PF0 = nullptr;
    // fast path (two trunk layers): head partials, dH0 split-K partials, device counters
    bool fast = false;
    bool tc = false;                 // the fast path's K1 / K3 on tcgen05 (tc_fast.cuh)
    bool tcb = false;                // large batches: tc_big.cuh's step (B >= kTcbMinBatch)
    uint16_t *h0img = nullptr, *ximg = nullptr, *dz1img = nullptr, *w1img = nullptr;
    float *w0t = nullptr;                  // tcb: [online, target] W0^T [D][N0]
    float *dheadp = nullptr;
    int64_t tcb_h0pl = 0, tcb_xpl = 0, tcb_dzpl = 0, tcb_w1pl = 0;
    float *part = nullptr, *dH0p = nullptr;
    int64_t part_elems = 0, dh0p_elems = 0;
    int64_t *step_dev = nullptr;
    int32_t *sync_flag = nullptr;
    cudaStream_t cap_stream = nullptr;
    cudaStream_t loss_stream = nullptr;    // the step's side branch (loss_out_kernel)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    struct PtypeSlot { uint64_t page; bool host; };
    PtypeSlot ptype_cache[64] = {};        // loss destinations: memory type per 4 KB page (+1)
    struct GraphEntry {
        const rpl_replay *rp;
        int B;
        int apply;                  // 0: data-parallel step (SGD after the all-reduce)
        int le;                     // FastArgs.loss_early: the graph has the loss side branch
        cudaGraph_t graph;          // kept alive: its nodes are updated in place
        cudaGraphExec_t exec;
        // nodes whose args change between replays: K1 and the distinct sampler (deferred
        // insert read-through, control block), K3 (the deferred insert's ring write), K4
        // (the loss destination)
        cudaGraphNode_t k1, ds, k3, k4;
        cudaGraphNode_t kl;         // loss_out_kernel (the loss side branch), or null
        cudaGraphNode_t ksgd;       // NCCL data parallelism: the captured SGD after the all-reduce
        float *sgd_loss;            // ... and the loss destination its node holds
        int par;                    // peer-memory data parallelism: the exchange slot (step parity), else -1
        cudaGraphNode_t kdp;        // ... and the captured exchange kernel (its DPArgs change every step)
        FastArgs args;              // the args those nodes currently hold
    };
    std::vector<GraphEntry> graphs;
    struct WideGraph {
        const rpl_replay *rp;
        int B, apply;
        int par;                   // peer-memory data parallelism: the exchange slot written, else -1
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        cudaGraphNode_t k4;        // the loss destination
        FastArgs args;
    };
    std::vector<WideGraph> wide_graphs;
    bool use_graphs = true;
    bool use_pdl = false;                  // programmatic dependent launch inside the graph
    bool k3_pdl = true;                    // K3 programmatic after K2
    bool k2_pdl = false, k4_pdl = false;   // experiments: RPL_K2PDL=1, RPL_K4PDL=1
    bool wide_tc = false;                  // byte-state wide inputs: layer 0 on tcgen05 (wide.cuh)
    bool wide_fast = false;                // ... and the layers above it on the fast kernels
    float *PdH0 = nullptr;                 // wide_fast: K3's dH0 partials [32][max_batch][N0]
    uint16_t *w0bf = nullptr;              // bf16 planes of W0 [online, target][3][N0 * D]
    uint16_t *dz0bf = nullptr;             // bf16 planes of dZ0 [3][max_batch][N0]
    // bf16 operand images to be re-split from the fp32 weights: bit 0 the online net's, bit 1
    // the target net's (a data-parallel update rewrites the online weights, and the target
    // only on a sync step)
    int w0bf_stale = 3;                    // wide W0 planes
    int w1img_stale = 3;                   // tcb: W1 images (any update not K4's)
    int wide_ks = 0, wide_cs = 1;          // wide_l0_kernel chunks and cluster size (wide_l0_plan)
    int k1_mc_clusters = 0;                // co-resident clusters of the multicast K1 (0: not used)
    unsigned long long *trace = nullptr;   // RPL_TRACE=1: per-CTA timestamps of the fast kernels
    // data parallel
    void *comm = nullptr;
    int rank = 0, world = 1;
    // peer-memory data parallelism (dqn_attach_peers, dp_peer.cuh): this rank's exchange buffer
    // [2][P + 1] gradient slots + a flag word, and every rank's, mapped through cudaIpc
    float *xbuf = nullptr;
    bool p2p = false;
    float *peer_xbuf[DP_MAXR] = {};
    int64_t dp_base = 0;                   // d->steps at dqn_attach_peers: exchange step = steps - base
    bool peer_opened[DP_MAXR] = {};
    std::vector<void *> allocs;
};

static int config_layout(const rpl_dqn_config *c, rpl_dqn *d)
{
    if (!c || c->state_dim < 1 || c->n_actions < 1 || c->n_actions > MAXA || c->n_hidden < 1 ||
        c->n_hidden > 4 || !(c->gamma >= 0.0f && c->gamma <= 1.0f) || !(c->lr >= 0.0f) ||
        !(c->huber_kappa > 0.0f) || c->sync_period < 0 || c->max_batch < 1 ||
        c->max_batch > (1 << 20) || (c->dueling && (c->stream < 1 || c->stream > 4096)) ||
        c->precision < RPL_PREC_FP32 || c->precision > RPL_PREC_BF16)
        return RPL_EINVAL;
    for (int l = 0; l < c->n_hidden; ++l)
        if (c->hidden[l] < 1 || c->hidden[l] > 4096) return RPL_EINVAL;
    int64_t P = 0;
    int K = c->state_dim, T = 0;
    for (int l = 0; l < c->n_hidden; ++l, ++T) {
        d->N[T] = c->hidden[l];
        d->K[T] = K;
        d->woff[T] = P;
        d->boff[T] = P + (int64_t)d->N[T] * K;
        P += (int64_t)d->N[T] * K + d->N[T];
        K = d->N[T];
    }
    if (c->dueling) {
        d->N[T] = 2 * c->stream;
        d->K[T] = K;
        d->woff[T] = P;
        d->boff[T] = P + (int64_t)d->N[T] * K;
        P += (int64_t)d->N[T] * K + d->N[T];
        ++T;
        d->J = 1 + c->n_actions;
        d->NH = 2 * c->stream;
        d->hw_off = P;
        d->hb_off = P + (int64_t)d->J * c->stream;
        P += (int64_t)d->J * c->stream + d->J;
    } else {
        d->J = c->n_actions;
        d->NH = K;
        d->hw_off = P;
        d->hb_off = P + (int64_t)d->J * K;
        P += (int64_t)d->J * K + d->J;
    }
    d->T = T;
    d->P = P;
    d->Htot = 0;
    for (int l = 0; l < T; ++l) d->Htot += d->N[l];
    return RPL_OK;
}

extern "C" int dqn_param_count(const rpl_dqn_config *cfg, int64_t *n)
{
    rpl_dqn tmp;
    if (!n || config_layout(cfg, &tmp) != RPL_OK) {
        set_error("dqn_param_count: invalid config");
        return RPL_EINVAL;
    }
    *n = tmp.P;
    return RPL_OK;
}

// split choices (host): b-split of 256 samples for weight gradients; split-K of dH so a
// phase has about one task per SM
static int nsplit_b_for(int B) { return (B + 255) / 256; }
static int nsplit_n_for(const rpl_dqn *d, int l, int B)
{
    const int tiles = ((B + BM - 1) / BM) * ((d->K[l] + BN - 1) / BN);
    int ns = (d->sms + tiles - 1) / tiles;
    const int maxs = (d->N[l] + BK - 1) / BK;
    if (ns > maxs) ns = maxs;
    if (ns < 1) ns = 1;
    return ns;
}

template <class T>
static bool dalloc(rpl_dqn *d, T **p, size_t n)
{
    void *q = nullptr;
    if (cudaMalloc(&q, n * sizeof(T) + 16) != cudaSuccess) return false;
    d->allocs.push_back(q);
    *p = (T *)q;
    return true;
}

// ---- fast-path sizing (host) ---------------------------------------------------------------
// layer-1 unit tile of K1: the largest of 128 / 64 / 32 that keeps every tile inside one
// dueling stream (S % UT == 0); 0 = no valid tile (the generic kernel runs instead)
static int fast_ut_cfg(const rpl_dqn_config &c, int N1)
{
    for (int ut : {128, 64, 32}) {
        if (c.dueling ? (c.stream % ut == 0) : (ut == 32 || N1 > ut / 2)) return ut;
    }
    return 0;
}
static int fast_ut(const rpl_dqn *d) { return fast_ut_cfg(d->cfg, d->N[1]); }
typedef void (*fwd_fn)(FastArgs);
// K1 instantiation: compile-time dims for the paper's dueling net and configs[0]'s MLP
static fwd_fn fast_fwd_fn(const rpl_dqn *d)
{
    const int ut = fast_ut(d), D = d->cfg.state_dim, N0 = d->N[0], J = d->J;
    if (ut == 128 && D == 27 && N0 == 128 && J == 9) return fast_fwd_kernel<128, 27, 128, 9>;
    if (ut == 64 && D == 27 && N0 == 64 && J == 8) return fast_fwd_kernel<64, 27, 64, 8>;
    if (ut == 128) return fast_fwd_kernel<128, 0, 0, 0>;
    if (ut == 64) return fast_fwd_kernel<64, 0, 0, 0>;
    return fast_fwd_kernel<32, 0, 0, 0>;
}
// the clustered K1 with multicast weight staging (paper net only), or null
static fwd_fn fast_fwd_mc_fn(const rpl_dqn *d)
{
    const int ut = fast_ut(d), D = d->cfg.state_dim, N0 = d->N[0], J = d->J;
#ifdef RPL_EXPERIMENTS
    if (ut == 128 && D == 27 && N0 == 128 && J == 9) return fast_fwd_mc_kernel<128, 27, 128, 9>;
#else
    (void)ut, (void)D, (void)N0, (void)J;
#endif
    return nullptr;
}
static size_t fast_fwd_smem(const rpl_dqn *d, int ut, int D = -1)
{
    const FwdLayout L(D < 0 ? d->cfg.state_dim : D, d->N[0], ut, d->J);
    return (size_t)L.total * sizeof(float);
}
static size_t fast_td_smem(const rpl_dqn *d)
{
    const int hs = d->cfg.dueling ? d->cfg.stream : d->N[1];
    return ((size_t)d->J * hs + d->N[1]) * sizeof(float);
}
// split-K count of dH0 = dZ1 W1 so that K3 has about one task per SM
static int fast_ns(const rpl_dqn *d, int B)
{
    // K3 runs two CTAs per SM: aim at ~2 tasks per SM in total
    const int n_w = ((d->N[1] + BM - 1) / BM) * ((d->N[0] + K3N - 1) / K3N) * ((B + 511) / 512);
    const int tiles = ((B + BM - 1) / BM) * ((d->N[0] + K3N - 1) / K3N);
    int want = (2 * d->sms - n_w) / tiles;
    int ns = 1;
    while (ns * 2 <= want && ns * 2 * 32 <= d->N[1]) ns *= 2;
    return ns;
}

// ---- tensor-core fast path (tc_fast.cuh) sizing --------------------------------------------
// shapes: layer-0 units a multiple of 16 up to 128 (the layer-0 accumulator and both H0 planes
// share 256 TMEM columns), inputs up to 31 (32 with the ones column of db0), layer-1 units
// and the dueling streams multiples of 32
static bool tc_shape_ok(const rpl_dqn *d)
{
    const rpl_dqn_config &c = d->cfg;
    return d->T == 2 && d->N[0] % 16 == 0 && d->N[0] <= 128 && d->N[1] % 32 == 0 &&
           (!c.dueling || c.stream % 32 == 0) && d->J <= tc::MAXJ && d->woff[1] % 4 == 0;
}
// K1 unit tile: the largest of 128 / 64 / 32 dividing N1 and a dueling stream (K1 CTAs are
// persistent per (net, unit tile) and run that combo's batch tiles)
static int tc_un_for(const rpl_dqn *d, int B)
{
    (void)B;
    const int S = d->cfg.dueling ? d->cfg.stream : d->N[1];
    for (int un : {128, 64})
        if (d->N[1] % un == 0 && S % un == 0) return un;
    return 32;
}
// the tensor-core kernels take batches from kTcMinBatch up (below it the mma.sync kernels are
// faster: the step is latency-bound there)
static constexpr int kTcMinBatch = 1 << 30;
static int tc_min_batch()
{
#ifdef RPL_EXPERIMENTS
    if (const char *v = getenv("RPL_TC_MIN")) return atoi(v);
#endif
    return kTcMinBatch;
}
static constexpr int kTcBsplit = 256;   // K3 (A) tasks: samples per batch split
// K3 (B) tasks: splits of the layer-1 units (a power of two, >= 2 chunks of 32 units each)
static int tc_ns_for(const rpl_dqn *d, int B)
{
    const int nbt = (B + 127) / 128, nA = ((d->N[1] + 127) / 128) * ((B + kTcBsplit - 1) / kTcBsplit);
    const int mx = std::max(1, d->N[1] / 64);
    const int want = std::max(4, (d->sms - nA) / nbt);
    int ns = 1;
    while (ns * 2 <= mx && ns * 2 <= want && (d->N[1] / (ns * 2)) % 32 == 0) ns *= 2;
    return ns;
}
static size_t tc_fwd_smem(const rpl_dqn *d, int un) { return (size_t)tc::FwdSmem(d->N[0], un, d->J).total; }

// ---- large-batch tensor-core step (tc_big.cuh) ----------------------------------------------
// shapes: 128 layer-0 units, fp32 states of <= 31 floats, layer-1 units and dueling streams in
// 128-unit tiles, at most tcb::JW head outputs per tile (dueling |A| <= 8), FP32 or BF16
// precision (TF32 keeps the mma.sync kernels)
static bool tcb_shape_ok(const rpl_dqn *d)
{
    const rpl_dqn_config &c = d->cfg;
    const int hw = c.dueling ? c.n_actions : d->J;
    return d->T == 2 && d->N[0] == tcb::N0 && c.state_dim <= 31 && d->N[1] % 128 == 0 &&
           (!c.dueling || c.stream % 128 == 0) && hw <= tcb::JW && d->J <= tcb::JPMAX &&
           d->woff[1] % 4 == 0 && c.precision != RPL_PREC_TF32;
}
// batches from here up take the tensor-core step (below it the mma.sync kernels: the step is
// latency-bound there)
static constexpr int kTcbMinBatch = 640;
static int tcb_min_batch()
{
#ifdef RPL_EXPERIMENTS
    if (const char *v = getenv("RPL_TCB_MIN")) return atoi(v);
#endif
    return kTcbMinBatch;
}
// T3a chunk groups: one CTA per (unit tile, group), about one wave
static int tcb_G(const rpl_dqn *d, int Bp)
{
    const int nch = Bp / 64, nut = d->N[1] / 128;
    return std::max(1, std::min(nch, d->sms / nut));
}
// T3b splits of the layer-1 units (64-unit chunks): a power of two with splits x tiles <= sms
static int tcb_NQ(const rpl_dqn *d, int Bp)
{
    const int nbt = Bp / 128, mx = d->N[1] / 64;
    int q = 1;
    while (q * 2 <= mx && q * 2 * nbt <= d->sms && d->N[1] % (q * 2 * 64) == 0) q *= 2;
    return q;
}
static int tcb_t0_smem(const rpl_dqn *d) { return (2 * tcb::N0 * d->cfg.state_dim + 2 * tcb::N0 + tcb::T0_ROWS * 2 * 33) * 4; }

extern "C" int dqn_destroy(rpl_dqn *d)
{
    if (!d) return RPL_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(d->device);
    cudaStreamSynchronize(d->stream);
    if (d->comm && g_nccl.destroy) g_nccl.destroy(d->comm);
    for (int q = 0; q < DP_MAXR; ++q)
        if (d->peer_opened[q]) cudaIpcCloseMemHandle(d->peer_xbuf[q]);
    if (d->xbuf) cudaFree(d->xbuf);
    for (auto &g : d->graphs) {
        cudaGraphExecDestroy(g.exec);
        cudaGraphDestroy(g.graph);
    }
    for (auto &g : d->wide_graphs) {
        cudaGraphExecDestroy(g.exec);
        cudaGraphDestroy(g.graph);
    }
    if (d->cap_stream) cudaStreamDestroy(d->cap_stream);
    if (d->loss_stream) cudaStreamDestroy(d->loss_stream);
    if (d->ev_fork) cudaEventDestroy(d->ev_fork);
    if (d->ev_join) cudaEventDestroy(d->ev_join);
    for (void *p : d->allocs) cudaFree(p);
    delete d;
    if (prev >= 0) cudaSetDevice(prev);
    return RPL_OK;
}

static void wide_l0_plan(rpl_dqn *d, int nets, int64_t D);

extern "C" int dqn_create(const rpl_dqn_config *cfg, const float *init, rpl_dqn **out)
{
    if (!out || !init) {
        set_error("dqn_create: null argument");
        return RPL_EINVAL;
    }
    *out = nullptr;
    rpl_dqn *d = new rpl_dqn();
    if (config_layout(cfg, d) != RPL_OK) {
        delete d;
        set_error("dqn_create: invalid config");
        return RPL_EINVAL;
    }
    d->cfg = *cfg;
    d->device = cfg->device;
    d->stream = (cudaStream_t)cfg->cuda_stream;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || d->device < 0 || d->device >= ndev) {
        delete d;
        set_error("dqn_create: no CUDA device %d", cfg->device);
        return RPL_ECUDA;
    }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(d->device);
    cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, d->device);
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, d->device);
    const int Bm = cfg->max_batch, D = cfg->state_dim, A = cfg->n_actions;
    const int nets = cfg->double_dqn ? 3 : 2;
    bool ok = coop != 0;
    ok = ok && dalloc(d, &d->online, d->P) && dalloc(d, &d->target, d->P) &&
         dalloc(d, &d->grad, d->P + 1);
    d->gpart_elems = (int64_t)nsplit_b_for(Bm) * ((d->P + 3) & ~(int64_t)3);
    ok = ok && (nsplit_b_for(Bm) == 1 || dalloc(d, &d->gpart, d->gpart_elems));
    ok = ok && dalloc(d, &d->Xs, (size_t)Bm * D) && dalloc(d, &d->Xs2, (size_t)Bm * D) &&
         dalloc(d, &d->r, Bm) && dalloc(d, &d->a, Bm) && dalloc(d, &d->idx, Bm) &&
         dalloc(d, &d->astar, Bm) && dalloc(d, &d->done, Bm) && dalloc(d, &d->dZlast, (size_t)Bm * d->NH) &&
         dalloc(d, &d->dO, (size_t)Bm * d->J) && dalloc(d, &d->loss_part, Bm) &&
         dalloc(d, &d->Qs, (size_t)Bm * A) && dalloc(d, &d->Qt2, (size_t)Bm * A) &&
         dalloc(d, &d->Qo2, (size_t)Bm * A) && dalloc(d, &d->y, Bm) && dalloc(d, &d->loss_dev, 1) &&
         dalloc(d, &d->bar, 2) && dalloc(d, &d->err, 1);
    if (ok && D > kWideInput)
        ok = dalloc(d, &d->PF0, (size_t)kKs0Max * nets * Bm * d->N[0]);
    {
        // tcgen05 layer 0 for byte-state replays (used when the replay is RPL_U8): 128 units,
        // 16-byte input rows, batches up to 256 (RPL_NO_WIDE_TC=1 disables)
        const char *nw = getenv("RPL_NO_WIDE_TC");
        d->wide_tc = ok && D > kWideInput && D % 16 == 0 && d->N[0] == WD_M && d->T >= 2 &&
                     !(nw && nw[0] == '1');
        if (d->wide_tc) {
            ok = cudaFuncSetAttribute(wide_l0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WD_SMEM) == cudaSuccess &&
                 cudaFuncSetAttribute(wide_dw0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WD_SMEM_MAX) == cudaSuccess &&
                 dalloc(d, &d->w0bf, (size_t)6 * wd_plane_elems(D)) &&
                 dalloc(d, &d->dz0bf, (size_t)3 * wd_plane_elems(Bm)) &&
                 // the tiles' padding (inputs past D) is never written: zero once
                 cudaMemset(d->w0bf, 0, (size_t)6 * wd_plane_elems(D) * 2) == cudaSuccess &&
                 cudaMemset(d->dz0bf, 0, (size_t)3 * wd_plane_elems(Bm) * 2) == cudaSuccess;
            if (ok) wide_l0_plan(d, d->cfg.double_dqn ? 3 : 2, D);
        }
    }
    for (int l = 0; l < d->T && ok; ++l) {
        ok = dalloc(d, &d->H[l], (size_t)nets * Bm * d->N[l]);
        if (ok && l > 0) {
            // nsplit_n * B <= (sms / tiles + 1) * B with tiles >= B / BM, so
            // nsplit_n * B <= sms * BM + B for every batch size B <= max_batch
            d->pdh_elems[l] = ((int64_t)d->sms * BM + Bm) * d->K[l];
            ok = dalloc(d, &d->PdH[l], d->pdh_elems[l]);
        }
    }
    // fast path: two trunk layers (dueling with one shared layer, or a plain 2-hidden-layer MLP)
    const char *path = getenv("RPL_PATH");
    d->fast = d->T == 2 && d->N[0] % 4 == 0 && d->N[0] <= 256 && D <= 31 && d->J <= F_MAXJ &&
              d->N[1] % 4 == 0 && (!cfg->dueling || cfg->stream % 4 == 0) && fast_ut_cfg(*cfg, d->N[1]) > 0 &&
              d->woff[1] % 4 == 0 && !(path && strcmp(path, "generic") == 0);
    // the fast kernels' contractions on tcgen05 (fp32 rings: inputs <= 31; byte-state wide
    // inputs: layer 0 is wide.cuh's, the tc kernels run the layers above it)
    d->tc = tc_shape_ok(d) && (D <= 31 || D > kWideInput);
    const char *ng = getenv("RPL_NO_GRAPH");
    d->use_graphs = !(ng && ng[0] == '1');
    // programmatic dependent launch measured slower on this structure (dependent CTAs that
    // start early compete for SM slots); opt in with RPL_PDL=1
    d->use_pdl = exp_flag("RPL_PDL");
    ok = ok && cudaFuncSetAttribute(distinct_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ds_smem_bytes(DS_MAXB)) == cudaSuccess;
    d->k3_pdl = !exp_flag("RPL_NO_K3PDL");
    d->k2_pdl = exp_flag("RPL_K2PDL");
    d->k4_pdl = exp_flag("RPL_K4PDL");
    ok = ok && dalloc(d, &d->step_dev, 1) && dalloc(d, &d->sync_flag, 1);
    const char *tr = getenv("RPL_TRACE");
    if (ok && tr && tr[0] == '1') {
        ok = dalloc(d, &d->trace, 8 * 2048 * 8);
        if (ok) cudaMemset(d->trace, 0, 8 * 2048 * 8 * sizeof(unsigned long long));
    }
    // wide byte-state inputs: the fast kernels run the layers above the tensor-core layer 0
    {
        const char *nf = getenv("RPL_NO_WIDE_FAST");
        d->wide_fast = ok && d->wide_tc && d->T == 2 && d->N[0] % 4 == 0 && d->J <= F_MAXJ &&
                       d->N[1] % 4 == 0 && (!cfg->dueling || cfg->stream % 4 == 0) &&
                       fast_ut_cfg(*cfg, d->N[1]) > 0 && Bm <= WD_MAXN &&
                       !(path && strcmp(path, "generic") == 0) && !(nf && nf[0] == '1');
        if (d->wide_fast) {
            const int ut = fast_ut(d);
            const int nut = (d->N[1] + (d->tc ? 32 : ut) - 1) / (d->tc ? 32 : ut);
            d->part_elems = (int64_t)nets * nut * Bm * d->J;
            ok = dalloc(d, &d->part, d->part_elems) && dalloc(d, &d->PdH0, (size_t)32 * Bm * d->N[0]);
            ok = ok && cudaFuncSetAttribute(fast_fwd_fn(d), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            fast_fwd_smem(d, ut, 0)) == cudaSuccess &&
                 cudaFuncSetAttribute(fast_bwd1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      K3_SMEM_FLOATS * sizeof(float)) == cudaSuccess &&
                 fast_td_smem(d) <= 200 * 1024 &&
                 cudaFuncSetAttribute(fast_td_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      fast_td_smem(d)) == cudaSuccess;
        }
    }
    if (ok && d->tc) {
        ok = cudaFuncSetAttribute(tc_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)tc_fwd_smem(d, 128)) == cudaSuccess &&
             cudaFuncSetAttribute(tc_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  tc::BwdSmem().total) == cudaSuccess;
    }
    if (ok && d->fast) {
        const int ut = fast_ut(d);   // the mma.sync K1's unit tile (its shared memory below)
        const int nut = (d->N[1] + (d->tc ? 32 : ut) - 1) / (d->tc ? 32 : ut);   // tc: up to N1 / 32 partials
        d->part_elems = (int64_t)nets * nut * Bm * d->J;
        // dW0 / db0 partials: NS(B) x ceil(B / 32) x (N0 D + N0); NS(B) x tiles(B) <= sms
        // with tiles(B) = ceil(B / 32) * ceil(N0 / 64) >= ceil(B / 32), so the product is
        // bounded by sms + ceil(B / 32) for every B <= max_batch; tc: NS <= N1 / 64 splits of
        // every 128-row batch tile
        int64_t w0p = d->sms + (Bm + BM - 1) / BM;
        if (d->tc) w0p = std::max<int64_t>(w0p, (int64_t)std::max(1, d->N[1] / 64) * ((Bm + 127) / 128));
        d->dh0p_elems = w0p * (d->woff[1]);
        ok = dalloc(d, &d->part, d->part_elems) && dalloc(d, &d->dH0p, d->dh0p_elems);
        ok = ok && cudaStreamCreateWithFlags(&d->cap_stream, cudaStreamNonBlocking) == cudaSuccess &&
             cudaStreamCreateWithFlags(&d->loss_stream, cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaFuncSetAttribute(fast_fwd_fn(d), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        fast_fwd_smem(d, ut)) == cudaSuccess;
        // clustered K1 (multicast weights; opt-in RPL_K1MC=1: 9.6 vs 7.9 us per K1 measured,
        // DESIGN.md §12): how many K1_MC-CTA clusters can be co-resident
        if (ok && fast_fwd_mc_fn(d)) {
            if (exp_flag("RPL_K1MC") &&
                cudaFuncSetAttribute(fast_fwd_mc_fn(d), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     fast_fwd_smem(d, ut)) == cudaSuccess) {
                cudaLaunchConfig_t lc = {};
                lc.gridDim = dim3(K1_MC);
                lc.blockDim = dim3(F_NT1);
                lc.dynamicSmemBytes = fast_fwd_smem(d, ut);
                int n = 0;
                if (cudaOccupancyMaxActiveClusters(&n, fast_fwd_mc_fn(d), &lc) == cudaSuccess) d->k1_mc_clusters = n;
            }
            cudaGetLastError();
        }

        ok = ok && cudaFuncSetAttribute(fast_bwd1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        K3_SMEM_FLOATS * sizeof(float)) == cudaSuccess;
        // one shared-memory carveout for every kernel of the step: no L1/shared
        // reconfiguration between consecutive kernels
        if (ok) {
            const void *fns[] = {(const void *)fast_fwd_fn(d), (const void *)fast_td_kernel,
                                 (const void *)fast_bwd1_kernel, (const void *)fast_bwd0_sgd_kernel,
                                 (const void *)insert_kernel_ptr(), (const void *)tc_fwd_kernel,
                                 (const void *)tc_bwd_kernel};
            for (const void *f : fns)
                ok = ok && cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                cudaSharedmemCarveoutMaxShared) == cudaSuccess;
            if (ok && fast_fwd_mc_fn(d))
                ok = cudaFuncSetAttribute((const void *)fast_fwd_mc_fn(d), cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared) == cudaSuccess;
        }
        ok = ok && fast_td_smem(d) <= 200 * 1024 &&
             cudaFuncSetAttribute(fast_td_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  fast_td_smem(d)) == cudaSuccess;
    }
    if (ok && d->fast && tcb_shape_ok(d) && Bm >= tcb_min_batch()) {
        const int64_t Bpm = ((int64_t)Bm + 127) / 128 * 128;
        d->tcb = true;
        d->tcb_h0pl = Bpm * tcb::N0;
        d->tcb_xpl = Bpm * tcb::XW;
        d->tcb_dzpl = Bpm * d->N[1];
        d->tcb_w1pl = (int64_t)d->N[1] * tcb::N0;
        const int jp = (d->J + 3) & ~3;
        ok = dalloc(d, &d->h0img, (size_t)3 * (nets + 1) * d->tcb_h0pl) && dalloc(d, &d->ximg, (size_t)3 * d->tcb_xpl) &&
             dalloc(d, &d->dz1img, (size_t)3 * d->tcb_dzpl) && dalloc(d, &d->w1img, (size_t)6 * d->tcb_w1pl) &&
             dalloc(d, &d->w0t, (size_t)2 * tcb::N0 * d->cfg.state_dim) &&
             dalloc(d, &d->dheadp, (size_t)Bpm * jp);
        // T3a partial gradients [G][gps]; T3b dW0 | db0 partials [NQ * tiles][w1] with
        // NQ * tiles <= max(sms, tiles)
        const int64_t gps = (d->P + 3) & ~(int64_t)3;
        const int64_t gneed = (int64_t)tcb_G(d, (int)Bpm) * gps;
        if (ok && gneed > d->gpart_elems) {
            ok = dalloc(d, &d->gpart, (size_t)gneed);
            d->gpart_elems = gneed;
        }
        const int64_t wneed = (int64_t)std::max<int64_t>(d->sms, Bpm / 128) * d->woff[1];
        if (ok && wneed > d->dh0p_elems) {
            ok = dalloc(d, &d->dH0p, (size_t)wneed);
            d->dh0p_elems = wneed;
        }
        const int64_t pneed = (int64_t)nets * (d->N[1] / 128) * tcb::T1_PSL * Bm * d->J;
        if (ok && pneed > d->part_elems) {
            ok = dalloc(d, &d->part, (size_t)pneed);
            d->part_elems = pneed;
        }
        ok = ok && cudaFuncSetAttribute(tcb_l0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tcb_t0_smem(d)) == cudaSuccess &&
             cudaFuncSetAttribute(tcb_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tcb::T1Smem(d->J).total) == cudaSuccess &&
             cudaFuncSetAttribute(tcb_dw1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tcb::T3aSmem(d->J).total) == cudaSuccess &&
             cudaFuncSetAttribute(tcb_dh0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tcb::T3bSmem().total) == cudaSuccess &&
             cudaFuncSetAttribute(tcb_td_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)tcb_td_smem(3, d->N[1], d->J)) == cudaSuccess;
    }
    if (!ok) {
        if (!coop) set_error("dqn_create: device %d lacks cooperative launch", d->device);
        else set_error("dqn_create: device allocation failed");
        dqn_destroy(d);
        if (prev >= 0) cudaSetDevice(prev);
        return coop ? RPL_ENOMEM : RPL_ECUDA;
    }
    const size_t pb = (size_t)d->P * sizeof(float);
    cudaError_t e = cudaMemcpyAsync(d->online, init, pb, cudaMemcpyHostToDevice, d->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d->target, init, pb, cudaMemcpyHostToDevice, d->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->bar, 0, 2 * sizeof(unsigned) + 16, d->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->err, 0, sizeof(uint32_t), d->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->grad, 0, (d->P + 1) * sizeof(float), d->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->step_dev, 0, sizeof(int64_t), d->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d->sync_flag, 0, sizeof(int32_t), d->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
    if (prev >= 0) cudaSetDevice(prev);
    if (e != cudaSuccess) {
        int rc = cuda_fail(e, "dqn_create init copies");
        dqn_destroy(d);
        return rc;
    }
    *out = d;
    return RPL_OK;
}

// split-K of the layer-0 forward for wide inputs: as many chunks as fill the grid in one
// wave (the state_dim > kWideInput case, e.g. 84x84x4 byte states)
static int ks0_for(const rpl_dqn *d, int B)
{
    if (d->cfg.state_dim <= kWideInput) return 1;
    const int nets = d->cfg.double_dqn ? 3 : 2;
    const int base = nets * ((B + BM - 1) / BM) * ((d->N[0] + BN - 1) / BN);
    int ks = d->sms / base;
    const int maxk = (d->cfg.state_dim + BK - 1) / BK;
    if (ks > kKs0Max) ks = kKs0Max;
    if (ks > maxk) ks = maxk;
    return ks < 1 ? 1 : ks;
}

static void fill_args(rpl_dqn *d, rpl_replay *rp, int B, float *loss_dev, int apply, int do_sync,
                      TrainArgs &p)
{
    memset(&p, 0, sizeof p);
    p.ring = rp->ring.rows;
    p.rs = rp->ring.rs;
    p.D = rp->ring.D;
    p.u8 = rp->ring.u8;
    p.so = rp->ring.so;
    p.shared = rp->ring.shared;
    p.sw = rp->ring.sw;
    p.cursor = rp->cursor;
    p.capacity = rp->ring.capacity;
    p.size = rp->size;
    p.seed = rp->seed;
    p.event = rp->events;
    p.rank = rp->rank;
    const rpl_dqn_config &c = d->cfg;
    p.A = c.n_actions;
    p.dueling = c.dueling;
    p.T = d->T;
    p.J = d->J;
    p.S = c.dueling ? c.stream : 0;
    p.NH = d->NH;
    p.nets = c.double_dqn ? 3 : 2;
    p.ddqn = c.double_dqn;
    for (int l = 0; l < d->T; ++l) {
        p.N[l] = d->N[l];
        p.K[l] = d->K[l];
        p.woff[l] = d->woff[l];
        p.boff[l] = d->boff[l];
        p.H[l] = d->H[l];
        p.PdH[l] = d->PdH[l];
        p.nsplit_n[l] = l > 0 ? nsplit_n_for(d, l, B) : 1;
    }
    p.hw_off = d->hw_off;
    p.hb_off = d->hb_off;
    p.P = d->P;
    p.B = B;
    p.gamma = c.gamma;
    p.lr = c.lr;
    p.kappa_inf = std::isinf(c.huber_kappa) ? 1 : 0;
    p.kappa = p.kappa_inf ? 0.0f : c.huber_kappa;
    p.online = d->online;
    p.target = d->target;
    p.Xs = d->Xs;
    p.Xs2 = d->Xs2;
    p.r = d->r;
    p.a = d->a;
    p.idx = d->idx;
    p.done = d->done;
    p.dZlast = d->dZlast;
    p.dO = d->dO;
    p.nsplit_b = nsplit_b_for(B);
    p.bsplit = 256;
    p.gpart = p.nsplit_b == 1 ? d->grad : d->gpart;
    p.grad = d->grad;
    p.loss_part = d->loss_part;
    p.Qs = d->Qs;
    p.Qt2 = d->Qt2;
    p.Qo2 = d->Qo2;
    p.y = d->y;
    p.astar = d->astar;
    p.loss_out = loss_dev ? loss_dev : d->loss_dev;
    p.apply_update = apply;
    p.do_sync = do_sync;
    p.ks0 = ks0_for(d, B);
    p.distinct = rp->distinct ? 1 : 0;
    p.PF0 = d->PF0;
    p.dZ0bf = d->dz0bf;
    p.trace = d->trace;
    p.bar = d->bar;
    p.err = d->err;
    p.rctrl = rp->ctrl_dev;
    p.step_dev = d->step_dev;
    p.sync_flag = d->sync_flag;
}

// wide_l0_kernel launch: nets x ks CTAs in clusters of cs along the chunks (wide.cuh)
static cudaError_t launch_wide_l0(const WideArgs &w, cudaStream_t st)
{
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(w.nets * w.ks));
    lc.blockDim = dim3(WD_T);
    lc.dynamicSmemBytes = WD_SMEM;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)w.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, wide_l0_kernel, w);
}

// chunks (ks) and cluster size (cs) of wide_l0_kernel for `nets` nets: as many co-resident
// clusters as the GPU holds (one CTA per SM; cudaOccupancyMaxActiveClusters), ks a multiple of
// cs, ks <= kKs0Max.  Default cs = 1: the cluster sums measured slower than writing every
// partial (cs = 2: epilogue 8.6 vs 5.0 us); RPL_WIDE_CS = 2..16 selects them
static void wide_l0_plan(rpl_dqn *d, int nets, int64_t D)
{
    const int64_t S = (D + WD_KS - 1) / WD_KS;
    int cs = 1;
#ifdef RPL_EXPERIMENTS
    if (const char *c = getenv("RPL_WIDE_CS")) cs = std::max(1, std::min(16, atoi(c)));
#endif
    for (; cs >= 1; --cs) {
        if (cs > 8) cudaFuncSetAttribute(wide_l0_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)(cs * nets));
        lc.blockDim = dim3(WD_T);
        lc.dynamicSmemBytes = WD_SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, wide_l0_kernel, &lc) != cudaSuccess) {
            cudaGetLastError();
            n = cs == 1 ? d->sms : 0;
        }
        int ks = (n / nets) * cs;
        ks = (int)std::min<int64_t>(ks, std::min<int64_t>(S, kKs0Max) / cs * cs);
        if (ks >= 2 * cs || (cs == 1 && ks >= 1)) {
            d->wide_ks = ks;
            d->wide_cs = cs;
            return;
        }
    }
    d->wide_ks = 1;
    d->wide_cs = 1;
}

// a loss destination in (pinned / mapped) host memory: the step writes it from a side branch
// (loss_out_kernel) so the PCIe write overlaps K3 / K4; device memory keeps the write in K4 (the
// branch's fork / join costs ~1 us of graph time that only a host write wins back)
// (the memory type is looked up once per 4 KB page: cudaPointerGetAttributes costs several us
// of host time per call; host-pinned and device allocations never share a page of the unified
// address space)
static bool loss_in_host_memory(rpl_dqn *d, const void *ptr)
{
    const uint64_t page = reinterpret_cast<uintptr_t>(ptr) >> 12;
    auto &slot = d->ptype_cache[page % 64];
    if (slot.page == page + 1) return slot.host;
    cudaPointerAttributes a{};
    bool host = false;
    if (cudaPointerGetAttributes(&a, ptr) == cudaSuccess) host = a.type == cudaMemoryTypeHost;
    else cudaGetLastError();   // unregistered pageable memory: not a valid kernel destination anyway
    slot.page = page + 1;
    slot.host = host;
    return host;
}

static void fill_fast(rpl_dqn *d, rpl_replay *rp, int B, float *loss_dev, int apply, FastArgs &p)
{
    memset(&p, 0, sizeof p);
    const rpl_dqn_config &c = d->cfg;
    p.prec = c.precision;
    p.ring = rp->ring.rows;
    p.rs = rp->ring.rs;
    p.D = rp->ring.D;
    p.shared = rp->ring.shared;
    p.sw = rp->ring.sw;
    p.rctrl = rp->ctrl_dev;
    p.seed = rp->seed;
    p.rank = rp->rank;
    p.A = c.n_actions;
    p.dueling = c.dueling;
    p.J = d->J;
    p.S = c.dueling ? c.stream : 0;
    p.N0 = d->N[0];
    p.N1 = d->N[1];
    p.nets = c.double_dqn ? 3 : 2;
    p.ddqn = c.double_dqn;
    p.w0 = d->woff[0];
    p.b0 = d->boff[0];
    p.w1 = d->woff[1];
    p.b1 = d->boff[1];
    p.wh = d->hw_off;
    p.bh = d->hb_off;
    p.P = d->P;
    p.B = B;
    p.gamma = c.gamma;
    p.lr = c.lr;
    p.kinf = std::isinf(c.huber_kappa) ? 1 : 0;
    p.kappa = p.kinf ? 0.0f : c.huber_kappa;
    p.sync_period = c.sync_period;
    p.online = d->online;
    p.target = d->target;
    p.Xs = d->Xs;
    p.Xs2 = d->Xs2;
    p.r = d->r;
    p.a = d->a;
    p.idx = d->idx;
    p.done = d->done;
    p.H0 = d->H[0];
    p.H1 = d->H[1];
    p.part = d->part;
    p.UT = fast_ut(d);
    p.nut = (p.N1 + p.UT - 1) / p.UT;
    p.dHead = d->dO;
    p.dZ1 = d->dZlast;
    p.w0part = d->dH0p;
    p.NS = fast_ns(d, B);
    p.nsb = (B + 511) / 512;
    p.bsplit = 512;
    p.gps = (p.P + 3) & ~(int64_t)3;
    p.gpart = p.nsb == 1 ? d->grad : d->gpart;
    p.grad = d->grad;
    p.loss_part = d->loss_part;
    p.Qs = d->Qs;
    p.Qt2 = d->Qt2;
    p.Qo2 = d->Qo2;
    p.y = d->y;
    p.astar = d->astar;
    p.loss_out = loss_dev ? loss_dev : d->loss_dev;
    p.step_dev = d->step_dev;
    p.sync_flag = d->sync_flag;
    p.apply_update = apply;
    p.err = d->err;
    p.trace = d->trace;
    p.distinct = rp->distinct ? 1 : 0;
    p.capacity = rp->ring.capacity;
    if (d->tc && B >= tc_min_batch()) {
        p.tc = 1;
        p.UT = tc_un_for(d, B);
        p.nut = p.N1 / p.UT;
        p.NS = tc_ns_for(d, B);
        p.bsplit = kTcBsplit;
        p.nsb = (B + kTcBsplit - 1) / kTcBsplit;
        p.gpart = p.nsb == 1 ? d->grad : d->gpart;
        p.nw0 = p.NS * ((B + 127) / 128);
    }
    if (d->tcb && B >= tcb_min_batch()) {
        p.tc = 0;
        p.tcb = 1;
        p.Bp = (B + 127) / 128 * 128;
        p.jp = (d->J + 3) & ~3;
        p.h0img = d->h0img;
        p.ximg = d->ximg;
        p.dz1img = d->dz1img;
        p.w1img = d->w1img;
        p.w0t = d->w0t;
        p.h0pl = d->tcb_h0pl;
        p.xpl = d->tcb_xpl;
        p.dzpl = d->tcb_dzpl;
        p.w1pl = d->tcb_w1pl;
        p.dheadp = d->dheadp;
        p.nsb = tcb_G(d, p.Bp);           // T3a chunk groups = K4's gradient splits
        p.gpart = p.nsb == 1 ? d->grad : d->gpart;
        p.NS = tcb_NQ(d, p.Bp);
        p.nw0 = p.NS * (p.Bp / 128);
    }
    const rpl_replay::Pending &q = rp->pend;
    if (q.k > 0) {   // consumed by this step's K1 (dqn_train_step clears it)
        p.pend_k = (int)q.k;
        p.pend_cur = q.cursor;
        p.pend_size = (uint64_t)q.new_size;
        p.pend_s = static_cast<const float *>(q.s);
        p.pend_s2 = static_cast<const float *>(q.s2);
        p.pend_r = q.r;
        p.pend_a = q.a;
        p.pend_done = q.done;
        p.pend_err = rp->err_dev;
    }
    // the loss leaves from a side branch of the step (loss_out_kernel after K2), so its
    // possibly-PCIe write overlaps K3 / K4 (not in data-parallel steps: there the exchanged
    // mean is the loss)
    p.loss_early = (loss_dev && apply && !p.tc && loss_in_host_memory(d, loss_dev)) ? 1 : 0;
}

// the four fast-path kernels, enqueued on `st`
// launch with programmatic dependent launch: the kernel may start while its predecessor is
// finishing; it prefetches step-invariant data, then waits (griddepcontrol.wait) before
// touching the predecessor's outputs
template <class K>
static cudaError_t launch_pdl(K kernel, int grid, int block, size_t smem, cudaStream_t st, bool pdl,
                              const FastArgs &p)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, p);
}

// the loss side branch of a step (FastArgs.loss_early): fork after K3, join before the step ends
static cudaError_t fork_loss(rpl_dqn *d, const FastArgs &p, cudaStream_t st)
{
    if (!p.loss_early) return cudaSuccess;
    cudaError_t e = cudaEventRecord(d->ev_fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(d->loss_stream, d->ev_fork, 0);
    if (e == cudaSuccess) {
        // highest launch priority: the scheduler places its one CTA ahead of K3's pending ones
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(1);
        lc.blockDim = dim3(256);
        lc.stream = d->loss_stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributePriority;
        at[0].val.priority = hi;
        lc.attrs = at;
        lc.numAttrs = 1;
        const LossArgs la{p.loss_part, p.B, p.loss_out};
        e = cudaLaunchKernelEx(&lc, loss_out_kernel, la);
    }
    if (e == cudaSuccess) e = cudaEventRecord(d->ev_join, d->loss_stream);
    return e;
}
static cudaError_t join_loss(rpl_dqn *d, const FastArgs &p, cudaStream_t st)
{
    return p.loss_early ? cudaStreamWaitEvent(st, d->ev_join, 0) : cudaSuccess;
}

// the fast-path kernels, enqueued on `st`
static cudaError_t tc_enqueue(rpl_dqn *d, const FastArgs &p, cudaStream_t st)
{
    const bool pdl = d->use_pdl;
    cudaError_t e;
    if (p.distinct) {   // distinct batch indices first (distinct.cuh)
        e = launch_pdl(distinct_fast_kernel, 1, DS_T, ds_smem_bytes(p.B), st, false, p);
        if (e != cudaSuccess) return e;
    }
    // K1: (net, unit tile) combos x 128-row batch tiles; with more tasks than SMs the grid is a
    // multiple of the combos, so a CTA keeps one weight tile staged across its batch tiles
    // one CTA per SM, persistent: cpc CTAs per (net, unit tile) combo split its batch tiles
    const int nbt = (p.B + 127) / 128, ncombo = p.nets * p.nut;
    const int cpc = std::max(1, std::min(nbt, d->sms / ncombo));
    e = launch_pdl(tc_fwd_kernel, ncombo * cpc, tc::T1, tc_fwd_smem(d, p.UT), st, false, p);
    if (e != cudaSuccess) return e;
    e = launch_pdl(fast_td_kernel, std::min(p.B, 4 * d->sms), NT, fast_td_smem(d), st, pdl || d->k2_pdl, p);
    if (e != cudaSuccess) return e;
    const int k3_tasks = ((p.N1 + 127) / 128) * p.nsb + nbt * p.NS;
    e = launch_pdl(tc_bwd_kernel, std::min(k3_tasks, d->sms), tc::T, tc::BwdSmem().total, st,
                   pdl || d->k3_pdl, p);
    if (e != cudaSuccess) return e;
    e = launch_pdl(fast_bwd0_sgd_kernel, d->sms, NT, 0, st, pdl || d->k4_pdl, p);
    return e == cudaSuccess ? join_loss(d, p, st) : e;
}

// the large-batch step (tc_big.cuh), enqueued on `st`
static cudaError_t tcb_enqueue(rpl_dqn *d, const FastArgs &p, cudaStream_t st)
{
    cudaError_t e;
    if (p.distinct) {   // distinct batch indices first (distinct.cuh)
        e = launch_pdl(distinct_fast_kernel, 1, DS_T, ds_smem_bytes(p.B), st, false, p);
        if (e != cudaSuccess) return e;
    }
    const int nbt = p.Bp / 128, nut = p.N1 / 128, ncombo = p.nets * nut;
    e = launch_pdl(tcb_l0_kernel, p.Bp / tcb::T0_ROWS, tcb::T0_T, tcb_t0_smem(d), st, false, p);
    if (e != cudaSuccess) return e;
    const int cpc = std::max(1, std::min(nbt, d->sms / ncombo));
    e = launch_pdl(tcb_fwd_kernel, ncombo * cpc, tcb::T1_T, tcb::T1Smem(p.J).total, st, false, p);
    if (e != cudaSuccess) return e;
    e = launch_pdl(tcb_td_kernel, (p.B + 7) / 8, 256, tcb_td_smem(p.nets, p.N1, p.J), st, false, p);
    if (e != cudaSuccess) return e;
    e = launch_pdl(tcb_dw1_kernel, nut * p.nsb, tcb::T3A_T, tcb::T3aSmem(p.J).total, st, false, p);
    if (e != cudaSuccess) return e;
    e = launch_pdl(tcb_dh0_kernel, nbt * p.NS, tcb::T3B_T, tcb::T3bSmem().total, st, false, p);
    if (e == cudaSuccess) e = fork_loss(d, p, st);
    if (e != cudaSuccess) return e;
    e = launch_pdl(fast_bwd0_sgd_kernel, d->sms, NT, 0, st, false, p);
    return e == cudaSuccess ? join_loss(d, p, st) : e;
}

static cudaError_t fast_enqueue(rpl_dqn *d, const FastArgs &p, cudaStream_t st)
{
    if (p.tcb) return tcb_enqueue(d, p, st);
    if (p.tc) return tc_enqueue(d, p, st);
    const int nbt = (p.B + F_BT - 1) / F_BT;
    const int k1_tasks = p.nets * nbt * p.nut;
    // large batches: a multiple of the nets x unit-tile combinations, so every CTA keeps one
    // weight tile resident across its batch tiles
    const int ncombo = p.nets * p.nut;
    int g1 = std::min(k1_tasks, d->sms);
    if (k1_tasks > d->sms && ncombo <= d->sms) g1 = (d->sms / ncombo) * ncombo;
    const size_t sm1 = fast_fwd_smem(d, p.UT, p.D);
    const bool pdl = d->use_pdl;
    cudaError_t e;
    if (p.distinct) {   // distinct batch indices first (distinct.cuh)
        e = launch_pdl(distinct_fast_kernel, 1, DS_T, ds_smem_bytes(p.B), st, false, p);
        if (e != cudaSuccess) return e;
    }
    // one task per CTA in whole co-resident clusters sharing a weight tile: the multicast K1
    const bool mc = d->k1_mc_clusters > 0 && g1 == k1_tasks && nbt % K1_MC == 0 &&
                    k1_tasks <= d->k1_mc_clusters * K1_MC && fast_fwd_mc_fn(d) && p.h0_in == nullptr;
    e = launch_pdl(mc ? fast_fwd_mc_fn(d) : fast_fwd_fn(d), g1, F_NT1, sm1, st, false, p);
    if (e != cudaSuccess) return e;
    e = launch_pdl(fast_td_kernel, std::min(p.B, 4 * d->sms), NT, fast_td_smem(d), st,
                   pdl || d->k2_pdl, p);
    if (e != cudaSuccess) return e;
    const int n_w = ((p.N1 + BM - 1) / BM) * ((p.N0 + K3N - 1) / K3N) * p.nsb;
    const int n_h = ((p.B + BM - 1) / BM) * ((p.N0 + K3N - 1) / K3N) * p.NS;
    const int hd_passes = p.dueling ? (p.A + 7) / 8 : (p.J + 7) / 8;
    const int n_hd = (((p.N1 + HD_U - 1) / HD_U) * hd_passes + 1) * p.nsb;
    // K3 always programmatic: it stages K1's operands while K2 finishes (griddepcontrol.wait
    // before K2's outputs); RPL_NO_K3PDL=1 serialises it
    e = launch_pdl(fast_bwd1_kernel, std::min(n_w + n_h + n_hd, 2 * d->sms), F_NT3,
                   K3_SMEM_FLOATS * sizeof(float), st, pdl || d->k3_pdl, p);
    // the loss branch forks after K3: its PCIe write then runs beside K4, which reads no host
    // memory (beside K3 it would hold up K3's zero-copy reads of a host-sourced insert: PCIe
    // reads do not pass posted writes)
    if (e == cudaSuccess) e = fork_loss(d, p, st);
    if (e != cudaSuccess) return e;
    e = launch_pdl(fast_bwd0_sgd_kernel, d->sms, NT, 0, st, pdl || d->k4_pdl, p);
    return e == cudaSuccess ? join_loss(d, p, st) : e;
}

static int grid_for(const rpl_dqn *d, const TrainArgs &p)
{
    // the largest phase task count, capped at one CTA per SM
    int64_t mx = 1;
    for (int l = 0; l < p.T; ++l) {
        const int64_t f = (int64_t)p.nets * ((p.B + BM - 1) / BM) * ((p.N[l] + BN - 1) / BN) *
                          (l == 0 ? p.ks0 : 1);
        const int64_t w = (int64_t)((p.N[l] + BM - 1) / BM) * ((p.K[l] + BN - 1) / BN) * p.nsplit_b;
        const int64_t h = l > 0 ? (int64_t)((p.B + BM - 1) / BM) * ((p.K[l] + BN - 1) / BN) * p.nsplit_n[l] : 0;
        mx = std::max(mx, std::max(f, w + h));
    }
    mx = std::max<int64_t>(mx, (p.B + NT / 32 - 1) / (NT / 32));
    mx = std::max<int64_t>(mx, (p.P + NT - 1) / NT);
    return (int)std::min<int64_t>(mx, d->sms);
}

// FastArgs of the fast kernels above a tensor-core layer 0 (byte-state wide inputs)
static void wide_fast_args(rpl_dqn *d, rpl_replay *rp, int B, float *loss_dev, int apply, FastArgs &fp)
{
    fill_fast(d, rp, B, loss_dev, apply, fp);
    fp.loss_early = 0;        // the byte-state step ends with wide_dw0_kernel: K4's write overlaps it
    fp.D = 0;                 // K1 neither gathers nor computes layer 0
    fp.distinct = 0;          // the batch is sampled by the byte gather
    fp.h0_in = d->H[0];       // [nets][B][N0] (the debug export's layer-0 activations)
    fp.H0 = d->H[0];          // the online net's block [B][N0]
    fp.PdH0 = d->PdH0;
    fp.dZ0 = d->PF0;
    fp.dZ0bf = d->dz0bf;
    fp.NS = fast_ns(d, B);
}

// the byte-state wide step captured once per (replay, batch, mode) and replayed: gather
// (event / size / cursor from the control block), tcgen05 layer 0, split-K reduction, the
// fast kernels above it (K4 advances the event), dW0 + its SGD
static cudaError_t wide_graph_step(rpl_dqn *d, rpl_replay *rp, int B, float *loss_dev, int apply,
                                   const WideArgs &w0, int par)
{
    FastArgs fp;
    wide_fast_args(d, rp, B, loss_dev, apply, fp);
    fp.event_advanced = 0;
    WideArgs w = w0;
    if (par >= 0) {   // peer-memory data parallelism: the gradient goes straight into its exchange slot
        float *slot = d->xbuf + (int64_t)par * dp_slot_stride(d->P);
        if (fp.gpart == fp.grad) fp.gpart = slot;
        fp.grad = slot;
        w.grad = slot;
    }
    rpl_dqn::WideGraph *ge = nullptr;
    for (auto &g : d->wide_graphs)
        if (g.rp == rp && g.B == B && g.apply == apply && g.par == par) ge = &g;
    cudaError_t e = cudaSuccess;
    if (!ge) {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaStream_t cs = d->cap_stream;
        if (!cs && (e = cudaStreamCreateWithFlags(&d->cap_stream, cudaStreamNonBlocking)) != cudaSuccess)
            return e;
        cs = d->cap_stream;
        e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return e;
        rpl_batch bt{d->Xs, d->Xs2, d->a, d->r, d->done, d->idx};
        int rc = launch_gather_u8_dev(rp, B, &bt, cs);
        cudaError_t el = launch_wide_l0(w, cs);
        wide_reduce_kernel<<<d->sms * 4, 256, 0, cs>>>(d->PF0, wd_l0_partials(w.ks, w.cs, B), w.nets, B, d->N[0], d->online,
                                                       d->target, d->boff[0], d->H[0]);
        cudaError_t e2 = rc == RPL_OK ? fast_enqueue(d, fp, cs) : cudaErrorUnknown;
        wide_dw0_kernel<<<(unsigned)((w.D + w.ntile - 1) / w.ntile), WD_T, wd_dw0_smem(w.ntile), cs>>>(w);
        e = cudaStreamEndCapture(cs, &graph);
        if (e == cudaSuccess) e = el;
        if (e == cudaSuccess) e = e2;
        if (e == cudaSuccess) e = cudaGetLastError();
        cudaGraphNode_t k4 = nullptr;
        if (e == cudaSuccess) {
            size_t n = 0;
            e = cudaGraphGetNodes(graph, nullptr, &n);
            std::vector<cudaGraphNode_t> nodes(n);
            if (e == cudaSuccess && n) e = cudaGraphGetNodes(graph, nodes.data(), &n);
            for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
                cudaGraphNodeType ty;
                cudaKernelNodeParams kp = {};
                if (cudaGraphNodeGetType(nodes[i], &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel &&
                    cudaGraphKernelNodeGetParams(nodes[i], &kp) == cudaSuccess &&
                    kp.func == (void *)fast_bwd0_sgd_kernel)
                    k4 = nodes[i];
            }
            if (e == cudaSuccess && !k4) e = cudaErrorInvalidValue;
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
        if (e != cudaSuccess) {
            if (graph) cudaGraphDestroy(graph);
            return e;
        }
        if (d->wide_graphs.size() >= 8) {
            cudaGraphExecDestroy(d->wide_graphs.front().exec);
            cudaGraphDestroy(d->wide_graphs.front().graph);
            d->wide_graphs.erase(d->wide_graphs.begin());
        }
        d->wide_graphs.push_back({rp, B, apply, par, graph, exec, k4, fp});
        ge = &d->wide_graphs.back();
    } else if (memcmp(&ge->args, &fp, sizeof fp) != 0) {
        // between replays only the loss destination may change (K4 writes it)
        void *args[] = {&fp};
        cudaKernelNodeParams kp = {};
        e = cudaGraphKernelNodeGetParams(ge->k4, &kp);
        kp.kernelParams = args;
        kp.extra = nullptr;
        if (e == cudaSuccess) e = cudaGraphExecKernelNodeSetParams(ge->exec, ge->k4, &kp);
        if (e != cudaSuccess) return e;
        ge->args = fp;
    }
    e = cudaGraphLaunch(ge->exec, d->stream);
    if (e == cudaSuccess) g_launches.fetch_add(8);
    return e;
}

// the SGD after an NCCL all-reduce; W0's planes for byte-state learners whose planes are current
static SgdArgs sgd_args(const rpl_dqn *d, const rpl_replay *rp, float *loss_out)
{
    SgdArgs a{};
    a.online = d->online;
    a.target = d->target;
    a.grad = d->grad;
    a.P = d->P;
    a.lr = d->cfg.lr;
    a.sync_flag = d->sync_flag;
    a.err = d->err;
    a.loss_out = loss_out;
    if (d->w0bf && rp->ring.u8 && d->wide_tc && d->woff[0] == 0 && !d->w0bf_stale) {
        a.planes.bf = d->w0bf;
        a.planes.n = (int64_t)d->N[0] * d->cfg.state_dim;
        a.planes.pe = wd_plane_elems(d->cfg.state_dim);
        a.planes.D = d->cfg.state_dim;
        a.planes.planes = d->cfg.precision == RPL_PREC_BF16 ? 1 : d->cfg.precision == RPL_PREC_TF32 ? 2 : 3;
    }
    return a;
}

// the exchange kernel's arguments for exchange step tx (dp_peer.cuh)
static void fill_dp(const rpl_dqn *d, int64_t tx, float *loss_out, DPArgs &a)
{
    a = DPArgs{};
    a.nloc = 1;
    a.world = d->world;
    a.rank0 = d->rank;
    a.P = d->P;
    a.t = (unsigned long long)tx;
    a.lr = d->cfg.lr;
    for (int q = 0; q < d->world; ++q) {
        a.xbuf[q] = d->peer_xbuf[q];
        a.flag[q] = dp_flag_of(d->peer_xbuf[q], d->P);
    }
    a.online[0] = d->online;
    a.target[0] = d->target;
    a.gmean[0] = d->grad;
    a.sync_flag[0] = d->sync_flag;
    a.err[0] = d->err;
    a.loss_out[0] = loss_out;
}
static cudaError_t launch_dp(const rpl_dqn *d, const DPArgs &a, cudaStream_t st)
{
    if (dp_use_rs(d->P, d->world)) {   // large gradients or >= 4 ranks: the reduce-scatter variant
        void *args[] = {const_cast<DPArgs *>(&a)};
        return cudaLaunchCooperativeKernel((const void *)dp_peer_rs_sgd_kernel, dim3(d->sms), dim3(256), args, 0, st);
    }
    dp_peer_sgd_kernel<<<(unsigned)d->sms, 256, 0, st>>>(a);
    return cudaGetLastError();
}
// cached step graphs that end in a data-parallel exchange: rebuilt after an attach / detach
static void drop_dp_graphs(rpl_dqn *d)
{
    for (size_t i = 0; i < d->wide_graphs.size();) {
        if (d->wide_graphs[i].apply == 0) {
            cudaGraphExecDestroy(d->wide_graphs[i].exec);
            cudaGraphDestroy(d->wide_graphs[i].graph);
            d->wide_graphs.erase(d->wide_graphs.begin() + i);
        } else {
            ++i;
        }
    }
    for (size_t i = 0; i < d->graphs.size();) {
        if (d->graphs[i].apply == 0) {
            cudaGraphExecDestroy(d->graphs[i].exec);
            cudaGraphDestroy(d->graphs[i].graph);
            d->graphs.erase(d->graphs.begin() + i);
        } else {
            ++i;
        }
    }
}

extern "C" int dqn_train_step(rpl_dqn *d, rpl_replay *rp, int32_t batch, float *loss_dev)
{
    if (!d || !rp || batch < 1 || batch > d->cfg.max_batch || rp->ring.D != d->cfg.state_dim ||
        rp->device != d->device) {
        set_error("dqn_train_step: invalid argument (batch=%d max=%d)", batch,
                  d ? d->cfg.max_batch : 0);
        return RPL_EINVAL;
    }
    if (rp->size < rp->burn_in || rp->size < 1) return RPL_NOT_READY;   // P:44, nothing advances
    if (sampleable(rp) < 1) return RPL_NOT_READY;                        // reading Q30
    if (rp->distinct && sampleable(rp) < batch) return RPL_NOT_READY;    // reading Q29
    if (rp->distinct && batch > DS_MAXB) {
        set_error("dqn_train_step: distinct batch %d > %d", batch, DS_MAXB);
        return RPL_EINVAL;
    }
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(d->device);
    const int64_t t = d->steps + 1;
    const int do_sync = d->cfg.sync_period > 0 && t % d->cfg.sync_period == 0;
    // data parallel: per-step gradient mean (dp), or local SGD + periodic parameter mean (avg)
    const bool avg = d->comm != nullptr && d->cfg.avg_period > 0;
    const bool dp = (d->comm != nullptr || d->p2p) && !avg;
    bool dp_graphed = false;   // the NCCL all-reduce + SGD captured in the fast step's graph
    int wide_par = -1;         // the byte-state graph wrote the gradient into this exchange slot
    cudaError_t e = cudaSuccess;
    // a deferred insert is consumed by the fast path's K1 on the shared stream; otherwise it
    // is written now by the insert kernel
    const bool fast = d->fast && !rp->ring.u8;   // the fast kernels read fp32 rows
    if (rp->ring.host == 2 && !fast) {
        if (prev >= 0) cudaSetDevice(prev);
        set_error("dqn_train_step: an RPL_RING_HOST_BATCH replay needs the fast path's net shape");
        return RPL_ESTATE;
    }
    if (!fast || rp->stream != d->stream) {
        if (int rc = replay_flush(rp)) {
            if (prev >= 0) cudaSetDevice(prev);
            return rc;
        }
    }
    if (fast) {
        FastArgs fp;
        fill_fast(d, rp, batch, dp ? nullptr : loss_dev, dp ? 0 : 1, fp);
        if (rp->ring.host == 2) {
            // the paper's in-RAM replay: CPU sample + CPU gather into pinned
            // staging, one H2D copy of the batch, then the same kernels on the copied rows
            const float *rows = nullptr;
            const int32_t *bidx = nullptr;
            if (int rc = host_batch_stage(rp, batch, d->stream, &rows, &bidx)) {
                if (prev >= 0) cudaSetDevice(prev);
                return rc;
            }
            fp.ring = const_cast<float *>(rows);
            fp.bidx = bidx;
            fp.distinct = 0;   // (distinct batches are drawn by the CPU sampler too)
        }
        if (fp.tcb && d->w1img_stale) {   // after create / set_params / sync_target / a DP or small-batch update
            if (d->w1img_stale & 1) {
                tcb_w1_split_kernel<<<d->sms, 256, 0, d->stream>>>(d->online + d->woff[1], d->w1img, d->tcb_w1pl, d->N[1],
                                                                   d->online + d->woff[0], d->w0t, d->cfg.state_dim);
                g_launches.fetch_add(1);
            }
            if (d->w1img_stale & 2) {
                tcb_w1_split_kernel<<<d->sms, 256, 0, d->stream>>>(d->target + d->woff[1], d->w1img + 3 * d->tcb_w1pl,
                                                                   d->tcb_w1pl, d->N[1], d->target + d->woff[0],
                                                                   d->w0t + (int64_t)tcb::N0 * d->cfg.state_dim,
                                                                   d->cfg.state_dim);
                g_launches.fetch_add(1);
            }
            e = cudaGetLastError();
            if (e != cudaSuccess) {
                if (prev >= 0) cudaSetDevice(prev);
                return cuda_fail(e, "tcb_w1_split_kernel");
            }
            d->w1img_stale = 0;
        }
        if (!fp.tcb && !dp) d->w1img_stale = 3;   // the mma.sync step's K4 updates W1 without its image
        const int zslot = rp->pend.slot;   // zero-copy staging slot the insert reads (or -1)
        rp->pend.k = 0;
        rp->pend.slot = -1;
        if (d->use_graphs) {
            rpl_dqn::GraphEntry *ge = nullptr;
            const int apply = dp ? 0 : 1;
            // NCCL data parallelism: the all-reduce (mean of gradient + loss word) and the SGD
            // after it are captured into the same graph -- one launch per step, the loss written
            // by the SGD kernel
            const bool nccl_tail = dp && d->comm && !d->p2p;
            float *sgd_loss = loss_dev ? loss_dev : d->loss_dev;
            // peer-memory data parallelism: the step writes its gradient straight into the
            // exchange slot of its parity (one graph per parity) and the exchange kernel is
            // captured after K4 (its DPArgs -- step number, loss destination -- set per step)
            const bool peer_tail = dp && d->p2p;
            const int64_t tx = t - d->dp_base;
            const int par = peer_tail ? (int)(tx & 1) : -1;
            if (peer_tail) {
                if (fp.gpart == fp.grad) fp.gpart = d->xbuf + (int64_t)par * dp_slot_stride(d->P);   // one batch split: K3 writes the gradient itself
                fp.grad = d->xbuf + (int64_t)par * dp_slot_stride(d->P);
            }
            DPArgs dpa;
            if (peer_tail) fill_dp(d, tx, loss_dev, dpa);
            for (auto &g : d->graphs)
                if (g.rp == rp && g.B == batch && g.apply == apply && g.le == fp.loss_early && g.par == par) ge = &g;
            if (!ge) {
                cudaGraph_t graph = nullptr;
                cudaGraphExec_t exec = nullptr;
                cudaGraphNode_t k1 = nullptr, ds = nullptr, k3 = nullptr, k4 = nullptr, kl = nullptr, ksgd = nullptr,
                                kdp = nullptr;
                e = cudaStreamBeginCapture(d->cap_stream, cudaStreamCaptureModeThreadLocal);
                if (e == cudaSuccess) {
                    cudaError_t e2 = fast_enqueue(d, fp, d->cap_stream);
                    if (e2 == cudaSuccess && nccl_tail) {
                        const int nr = g_nccl.allreduce(d->grad, d->grad, (size_t)d->P + 1, kNcclFloat, kNcclAvg,
                                                        d->comm, d->cap_stream);
                        if (nr != 0) {
                            set_error("ncclAllReduce (graph capture) failed: %s", g_nccl.errstr ? g_nccl.errstr(nr) : "?");
                            e2 = cudaErrorUnknown;
                        } else {
                            sgd_kernel<<<(unsigned)d->sms, 256, 0, d->cap_stream>>>(sgd_args(d, rp, sgd_loss));
                            e2 = cudaGetLastError();
                        }
                    }
                    if (e2 == cudaSuccess && peer_tail) e2 = launch_dp(d, dpa, d->cap_stream);
                    e = cudaStreamEndCapture(d->cap_stream, &graph);
                    if (e2 != cudaSuccess) e = e2;
                }
                if (e == cudaSuccess) {
                    size_t n = 0;
                    e = cudaGraphGetNodes(graph, nullptr, &n);
                    std::vector<cudaGraphNode_t> nodes(n);
                    if (e == cudaSuccess && n) e = cudaGraphGetNodes(graph, nodes.data(), &n);
                    for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
                        cudaGraphNodeType ty;
                        cudaKernelNodeParams kp = {};
                        if (cudaGraphNodeGetType(nodes[i], &ty) == cudaSuccess &&
                            ty == cudaGraphNodeTypeKernel &&
                            cudaGraphKernelNodeGetParams(nodes[i], &kp) == cudaSuccess) {
                            if (kp.func == (void *)fast_fwd_fn(d) || kp.func == (void *)tc_fwd_kernel ||
                                (fast_fwd_mc_fn(d) && kp.func == (void *)fast_fwd_mc_fn(d)))
                                k1 = nodes[i];
                            if (kp.func == (void *)distinct_fast_kernel) ds = nodes[i];
                            if (kp.func == (void *)fast_bwd1_kernel || kp.func == (void *)tc_bwd_kernel) k3 = nodes[i];
                            if (kp.func == (void *)fast_bwd0_sgd_kernel) k4 = nodes[i];
                            if (kp.func == (void *)loss_out_kernel) kl = nodes[i];
                            if (kp.func == (void *)sgd_kernel) ksgd = nodes[i];
                            if (kp.func == (void *)dp_peer_sgd_kernel || kp.func == (void *)dp_peer_rs_sgd_kernel)
                                kdp = nodes[i];
                            if (kp.func == (void *)tcb_l0_kernel) k1 = k3 = nodes[i];   // T0 also writes the insert
                        }
                    }
                    // NCCL's captured kernel nodes (a foreign module) fail the params query with
                    // cudaErrorInvalidDeviceFunction: a non-sticky error, cleared here so the next
                    // launch check does not report it
                    cudaGetLastError();
                    if (e == cudaSuccess && (!k1 || !k3 || !k4 || (nccl_tail && !ksgd) || (peer_tail && !kdp)))
                        e = cudaErrorInvalidValue;
                }
                if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
                if (e == cudaSuccess) {
                    if (d->graphs.size() >= 16) {
                        cudaGraphExecDestroy(d->graphs.front().exec);
                        cudaGraphDestroy(d->graphs.front().graph);
                        d->graphs.erase(d->graphs.begin());
                    }
                    d->graphs.push_back({rp, batch, apply, fp.loss_early, graph, exec, k1, ds, k3, k4,
                                         fp.loss_early ? kl : nullptr, nccl_tail ? ksgd : nullptr, sgd_loss, par,
                                         peer_tail ? kdp : nullptr, fp});
                    ge = &d->graphs.back();
                } else if (graph) {
                    cudaGraphDestroy(graph);
                }
            } else if (memcmp(&ge->args, &fp, sizeof fp) != 0) {
                // between replays only the deferred insert and the loss destination change:
                // update the nodes that read them
                const bool pend_changed = ge->args.pend_k != fp.pend_k || ge->args.pend_cur != fp.pend_cur ||
                                          ge->args.pend_s != fp.pend_s || ge->args.pend_size != fp.pend_size ||
                                          ge->args.pend_s2 != fp.pend_s2 || ge->args.pend_r != fp.pend_r ||
                                          ge->args.pend_a != fp.pend_a || ge->args.pend_done != fp.pend_done;
                const bool loss_changed = ge->args.loss_out != fp.loss_out;
                FastArgs cmp = ge->args;
                cmp.pend_k = fp.pend_k; cmp.pend_cur = fp.pend_cur; cmp.pend_s = fp.pend_s;
                cmp.pend_s2 = fp.pend_s2; cmp.pend_r = fp.pend_r; cmp.pend_a = fp.pend_a;
                cmp.pend_done = fp.pend_done; cmp.pend_size = fp.pend_size; cmp.pend_err = fp.pend_err;
                cmp.loss_out = fp.loss_out;
                void *args[] = {&fp};
                auto update = [&](cudaGraphNode_t nd) {
                    if (!nd || e != cudaSuccess) return;
                    cudaKernelNodeParams kp = {};
                    e = cudaGraphKernelNodeGetParams(nd, &kp);
                    if (e == cudaSuccess && (kp.func == (void *)sgd_kernel || kp.func == (void *)dp_peer_sgd_kernel ||
                                             kp.func == (void *)dp_peer_rs_sgd_kernel || kp.func == (void *)loss_out_kernel))
                        return;   // not a FastArgs kernel
                    if (e == cudaErrorInvalidDeviceFunction) {   // a foreign (NCCL) kernel node: not ours
                        cudaGetLastError();
                        e = cudaSuccess;
                        return;
                    }
                    kp.kernelParams = args;
                    kp.extra = nullptr;
                    if (e == cudaSuccess) e = cudaGraphExecKernelNodeSetParams(ge->exec, nd, &kp);
                };
                if (memcmp(&cmp, &fp, sizeof fp) != 0) {
                    // anything else differs (not expected): every node of the step
                    size_t n = 0;
                    e = cudaGraphGetNodes(ge->graph, nullptr, &n);
                    std::vector<cudaGraphNode_t> nodes(n);
                    if (e == cudaSuccess && n) e = cudaGraphGetNodes(ge->graph, nodes.data(), &n);
                    for (size_t i = 0; e == cudaSuccess && i < n; ++i) update(nodes[i]);
                } else {
                    if (pend_changed) {
                        update(ge->k1);
                        update(ge->ds);
                        update(ge->k3);
                    }
                    if (loss_changed && !ge->kl) update(ge->k4);
                }
                if (loss_changed && ge->kl && e == cudaSuccess) {
                    // the loss side branch alone writes it (K4 skips it with loss_early)
                    LossArgs la{fp.loss_part, fp.B, fp.loss_out};
                    void *largs[] = {&la};
                    cudaKernelNodeParams kp = {};
                    e = cudaGraphKernelNodeGetParams(ge->kl, &kp);
                    kp.kernelParams = largs;
                    kp.extra = nullptr;
                    if (e == cudaSuccess) e = cudaGraphExecKernelNodeSetParams(ge->exec, ge->kl, &kp);
                }
                if (e == cudaSuccess) ge->args = fp;
            }
            if (e == cudaSuccess && ge && ge->ksgd && ge->sgd_loss != sgd_loss) {
                // the SGD node's loss destination (its other arguments are fixed)
                SgdArgs sa = sgd_args(d, rp, sgd_loss);
                void *sargs[] = {&sa};
                cudaKernelNodeParams kp = {};
                e = cudaGraphKernelNodeGetParams(ge->ksgd, &kp);
                kp.kernelParams = sargs;
                kp.extra = nullptr;
                if (e == cudaSuccess) e = cudaGraphExecKernelNodeSetParams(ge->exec, ge->ksgd, &kp);
                if (e == cudaSuccess) ge->sgd_loss = sgd_loss;
            }
            if (e == cudaSuccess && ge && ge->kdp) {
                // the exchange kernel's step number and loss destination
                void *dargs[] = {&dpa};
                cudaKernelNodeParams kp = {};
                e = cudaGraphKernelNodeGetParams(ge->kdp, &kp);
                kp.kernelParams = dargs;
                kp.extra = nullptr;
                if (e == cudaSuccess) e = cudaGraphExecKernelNodeSetParams(ge->exec, ge->kdp, &kp);
            }
            if (e == cudaSuccess) e = cudaGraphLaunch(ge->exec, d->stream);
            if (e == cudaSuccess && ge && ge->kdp) {
                dp_graphed = true;
                g_launches.fetch_add(1);   // the captured exchange kernel
            }
            if (e == cudaSuccess && ge && ge->ksgd) {
                dp_graphed = true;
                g_launches.fetch_add(1);   // the captured sgd_kernel (NCCL's own kernels not counted)
            }
        } else {
            e = fast_enqueue(d, fp, d->stream);
        }
        if (e == cudaSuccess) {
            // the zero-copy staging slot may be rewritten once the stream passes this step
            if (zslot >= 0 && cudaEventRecord(rp->evs[zslot], d->stream) != cudaSuccess)
                e = cudaGetLastError();
        }
        if (e != cudaSuccess) {
            if (prev >= 0) cudaSetDevice(prev);
            return cuda_fail(e, "fast train step");
        }
        g_launches.fetch_add((fp.distinct ? 1 : 0) + (fp.tcb ? 6 : 4) + (fp.loss_early ? 1 : 0));
    } else {
        d->w1img_stale = 3;   // the generic kernels update W1 without the tcb image
        TrainArgs p;
        fill_args(d, rp, batch, loss_dev, dp ? 0 : 1, do_sync, p);
        // byte states with a wide input: layer 0 on the tensor cores (wide.cuh) around the
        // cooperative kernel, which then runs the layers above it
        const bool wide = d->wide_tc && rp->ring.u8 && batch <= WD_MAXN;
        WideArgs w{};
        if (wide) {
            const int nets = p.nets;
            w.D = p.D;
            w.B = batch;
            w.N0 = d->N[0];
            w.nets = nets;
            w.ks = d->wide_ks;
            w.cs = d->wide_cs;
            w.U0 = reinterpret_cast<const uint8_t *>(d->Xs);
            w.U1 = reinterpret_cast<const uint8_t *>(d->Xs2);
            w.online = d->online;
            w.target = d->target;
            w.w0 = d->woff[0];
            w.PF0 = d->PF0;
            w.dZ0 = d->PF0;
            w.dZ0bf = d->dz0bf;
            w.W0bf = d->w0bf;
            w.grad = d->grad;
            w.P = d->P;
            w.online_w = d->online;
            w.target_w = d->target;
            w.lr = d->cfg.lr;
            w.apply_update = dp ? 0 : 1;
            w.sync_flag = d->sync_flag;
            p.wide_tc = 1;
            p.ks0 = wd_l0_partials(w.ks, w.cs, batch);   // partials left in PF0
            if (d->w0bf_stale) {   // after create / set_params / sync_target / a DP step
                const int64_t pe = wd_plane_elems(p.D);
                if (d->w0bf_stale & 1) launch_wide_split(d->online + d->woff[0], d->w0bf, d->N[0], p.D, d->sms, d->stream);
                if (d->w0bf_stale & 2)
                    launch_wide_split(d->target + d->woff[0], d->w0bf + 3 * pe, d->N[0], p.D, d->sms, d->stream);
                e = cudaGetLastError();
                if (e != cudaSuccess) {
                    if (prev >= 0) cudaSetDevice(prev);
                    return cuda_fail(e, "wide_split_kernel");
                }
                g_launches.fetch_add(d->w0bf_stale == 3 ? 2 : 1);
                d->w0bf_stale = 0;
            }
            w.ntile = (int)std::min<int64_t>(WD_MAXN, ((p.D + d->sms - 1) / d->sms + 15) / 16 * 16);
            w.wpre = wd_dw0_wpre(w.ntile) ? 1 : 0;
            // bf16 terms of the fp32 weights / dZ0 per product: 3 (FP32), 2 (TF32), 1 (BF16)
            w.nplanes = d->cfg.precision == RPL_PREC_BF16 ? 1 : d->cfg.precision == RPL_PREC_TF32 ? 2 : 3;
            w.trace = d->trace;
            w.do_db0 = d->wide_fast ? 1 : 0;
            w.b0 = d->boff[0];
            if (d->wide_fast && d->use_graphs && !rp->distinct) {
                // the whole byte-state step as one CUDA graph (control block read on device)
                wide_par = dp && d->p2p ? (int)((t - d->dp_base) & 1) : -1;
                e = wide_graph_step(d, rp, batch, dp ? nullptr : loss_dev, dp ? 0 : 1, w, wide_par);
                if (e != cudaSuccess) {
                    if (prev >= 0) cudaSetDevice(prev);
                    return cuda_fail(e, "wide graph step");
                }
                goto after_step;
            }
            // (1) Philox sample + gather + unpack into the learner's batch buffers
            rpl_batch bt{d->Xs, d->Xs2, d->a, d->r, d->done, d->idx};
            if (int rc = launch_gather(rp, batch, nullptr, rp->events, 1, &bt)) {
                if (prev >= 0) cudaSetDevice(prev);
                return rc;
            }
            // (2) layer-0 forward partials of every net
            e = launch_wide_l0(w, d->stream);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) {
                if (prev >= 0) cudaSetDevice(prev);
                return cuda_fail(e, "wide_l0_kernel");
            }
        }
        if (p.distinct && !wide) {   // distinct batch indices into d->idx (distinct.cuh)
            if (int rc = launch_distinct(rp, batch, d->idx, d->err, nullptr, d->stream)) {
                if (prev >= 0) cudaSetDevice(prev);
                return rc;
            }
        }
        if (wide && d->wide_fast) {
            // (3) layers above layer 0 on the fast kernels: H0 from the partials, then K1 (H0
            // in), K2, K3 (dH0 partials out), K4 (dZ0 for step 4, every SGD but layer 0's)
            wide_reduce_kernel<<<d->sms * 4, 256, 0, d->stream>>>(d->PF0, wd_l0_partials(w.ks, w.cs, batch), p.nets, batch, d->N[0],
                                                                   d->online, d->target, d->boff[0], d->H[0]);
            FastArgs fp;
            wide_fast_args(d, rp, batch, dp ? nullptr : loss_dev, dp ? 0 : 1, fp);
            fp.event_advanced = 1;    // the sampling gather advanced the event
            e = cudaGetLastError();
            if (e == cudaSuccess) e = fast_enqueue(d, fp, d->stream);
            if (e != cudaSuccess) {
                if (prev >= 0) cudaSetDevice(prev);
                return cuda_fail(e, "wide fast step");
            }
            g_launches.fetch_add(5);
        } else {
        const int grid = grid_for(d, p);
        void *args[] = {&p};
        e = cudaLaunchCooperativeKernel((const void *)train_step_kernel, dim3(grid), dim3(NT), args,
                                        0, d->stream);
        if (e != cudaSuccess) {
            if (prev >= 0) cudaSetDevice(prev);
            return cuda_fail(e, "cudaLaunchCooperativeKernel(train_step_kernel)");
        }
        g_launches.fetch_add(1);
        }
        if (wide) {
            // (4) dW0 = dZ0^T x per 256-input tile, then its SGD / target sync
            // dW0 tiles: one wave over the SMs (28,224 inputs -> 147 tiles of 192)
            wide_dw0_kernel<<<(unsigned)((p.D + w.ntile - 1) / w.ntile), WD_T, wd_dw0_smem(w.ntile), d->stream>>>(w);
            e = cudaGetLastError();
            if (e != cudaSuccess) {
                if (prev >= 0) cudaSetDevice(prev);
                return cuda_fail(e, "wide_dw0_kernel");
            }
            g_launches.fetch_add(2);
        }
    }
after_step:
    if (dp && d->p2p) {
        // gradient mean + SGD over peer memory (dp_peer.cuh): this step's gradient into its
        // exchange slot, then one kernel publishes it, waits for every rank's and updates
        // exchange step numbers count from the attach (every rank attached at the same point
        // of its stream, after the flag area was cleared), not from the learner's own steps
        // (the byte-state and generic steps; the fast step captures all of this in its graph)
        const int64_t tx = t - d->dp_base;
        float *mine = d->xbuf + (int64_t)(tx & 1) * dp_slot_stride(d->P);
        bool planes = false;   // the exchange's SGD rewrites W0's bf16 planes (byte-state learners)
        if (!dp_graphed) {
            if (wide_par < 0)   // (the byte-state graph wrote it into the slot already)
                e = cudaMemcpyAsync(mine, d->grad, (size_t)(d->P + 1) * sizeof(float), cudaMemcpyDeviceToDevice, d->stream);
            DPArgs a;
            fill_dp(d, tx, loss_dev, a);
#ifndef RPL_NO_DP_PLANES   // (A/B timing builds only)
            if (d->w0bf && rp->ring.u8 && d->wide_tc && d->woff[0] == 0 && !d->w0bf_stale) {
#else
            if (false) {
#endif
                a.w0.bf = d->w0bf;
                a.w0.n = (int64_t)d->N[0] * d->cfg.state_dim;
                a.w0.pe = wd_plane_elems(d->cfg.state_dim);
                a.w0.D = d->cfg.state_dim;
                a.w0.planes = d->cfg.precision == RPL_PREC_BF16 ? 1 : d->cfg.precision == RPL_PREC_TF32 ? 2 : 3;
                planes = true;
            }
            if (e == cudaSuccess) e = launch_dp(d, a, d->stream);
            if (e != cudaSuccess) {
                if (prev >= 0) cudaSetDevice(prev);
                return cuda_fail(e, "dp_peer_sgd_kernel");
            }
            g_launches.fetch_add(1);
        }
        // the update rewrote the online W0 / W1 without their images (the target too on a sync
        // step) -- except W0's planes when the exchange wrote them
        if (!planes) d->w0bf_stale |= do_sync ? 3 : 1;
        d->w1img_stale |= do_sync ? 3 : 1;
    } else if (dp && dp_graphed) {
        // the all-reduce and the SGD after it ran inside the step's graph (nccl_tail)
        d->w0bf_stale |= do_sync ? 3 : 1;
        d->w1img_stale |= do_sync ? 3 : 1;
    } else if (dp) {
        int nr = g_nccl.allreduce(d->grad, d->grad, (size_t)d->P + 1, kNcclFloat, kNcclAvg,
                                  d->comm, d->stream);
        if (nr != 0) {
            set_error("ncclAllReduce failed: %s", g_nccl.errstr ? g_nccl.errstr(nr) : "?");
            if (prev >= 0) cudaSetDevice(prev);
            return RPL_ENCCL;
        }
        const SgdArgs sa = sgd_args(d, rp, loss_dev);
        // the all-reduced update rewrote the online W0 / W1 without their images (the target
        // too on a sync step) -- except W0's planes when the SGD writes them
        if (!sa.planes.bf) d->w0bf_stale |= do_sync ? 3 : 1;
        d->w1img_stale |= do_sync ? 3 : 1;
        sgd_kernel<<<(unsigned)d->sms, 256, 0, d->stream>>>(sa);
        e = cudaGetLastError();
        if (e != cudaSuccess) {
            if (prev >= 0) cudaSetDevice(prev);
            return cuda_fail(e, "sgd_kernel");
        }
        g_launches.fetch_add(1);
    }
    if (avg && t % d->cfg.avg_period == 0) {
        // iterative parameter mixing (reading Q31): online and target <- their mean over ranks
        for (float *w : {d->online, d->target}) {
            int nr = g_nccl.allreduce(w, w, (size_t)d->P, kNcclFloat, kNcclAvg, d->comm, d->stream);
            if (nr != 0) {
                set_error("ncclAllReduce failed: %s", g_nccl.errstr ? g_nccl.errstr(nr) : "?");
                if (prev >= 0) cudaSetDevice(prev);
                return RPL_ENCCL;
            }
        }
        d->w0bf_stale = 3;
        d->w1img_stale = 3;
    }
    if (prev >= 0) cudaSetDevice(prev);
    rp->events += 1;
    d->steps = t;
    d->last_B = batch;
    d->last_u8 = rp->ring.u8;
    return RPL_OK;
}

extern "C" int sync_target(rpl_dqn *d)
{
    if (!d) return RPL_EINVAL;
    RPL_CUDA(cudaMemcpyAsync(d->target, d->online, (size_t)d->P * sizeof(float),
                             cudaMemcpyDeviceToDevice, d->stream));
    d->w0bf_stale = 3;
    d->w1img_stale = 3;
    return RPL_OK;
}

static float *which_ptr(rpl_dqn *d, int which)
{
    return which == RPL_ONLINE ? d->online : which == RPL_TARGET ? d->target
                                           : which == RPL_GRAD ? d->grad : nullptr;
}

extern "C" int dqn_get_params(rpl_dqn *d, int which, float *host_out, int64_t n)
{
    if (!d || !host_out || n != d->P || !which_ptr(d, which)) {
        set_error("dqn_get_params: invalid argument");
        return RPL_EINVAL;
    }
    RPL_CUDA(cudaMemcpyAsync(host_out, which_ptr(d, which), (size_t)n * sizeof(float),
                             cudaMemcpyDeviceToHost, d->stream));
    RPL_CUDA(cudaStreamSynchronize(d->stream));
    return RPL_OK;
}

extern "C" int dqn_set_params(rpl_dqn *d, int which, const float *host_in, int64_t n)
{
    if (!d || !host_in || n != d->P || (which != RPL_ONLINE && which != RPL_TARGET)) {
        set_error("dqn_set_params: invalid argument");
        return RPL_EINVAL;
    }
    RPL_CUDA(cudaMemcpyAsync(which_ptr(d, which), host_in, (size_t)n * sizeof(float),
                             cudaMemcpyHostToDevice, d->stream));
    RPL_CUDA(cudaStreamSynchronize(d->stream));
    d->w0bf_stale = 3;
    d->w1img_stale = 3;
    return RPL_OK;
}

extern "C" int dqn_step_count(const rpl_dqn *d, int64_t *steps)
{
    if (!d || !steps) return RPL_EINVAL;
    *steps = d->steps;
    return RPL_OK;
}

extern "C" int dqn_debug_export(rpl_dqn *d, int what, void *host_out, int64_t bytes)
{
    if (!d || !host_out || d->last_B < 1) {
        set_error("dqn_debug_export: no step executed yet");
        return RPL_ESTATE;
    }
    const int64_t B = d->last_B, D = d->cfg.state_dim, A = d->cfg.n_actions;
    const void *src = nullptr;
    int64_t need = 0;
    switch (what) {
    case RPL_DBG_IDX: src = d->idx; need = B * 4; break;
    case RPL_DBG_S: src = d->Xs; need = B * D * (d->last_u8 ? 1 : 4); break;
    case RPL_DBG_S_NEXT: src = d->Xs2; need = B * D * (d->last_u8 ? 1 : 4); break;
    case RPL_DBG_A: src = d->a; need = B * 4; break;
    case RPL_DBG_R: src = d->r; need = B * 4; break;
    case RPL_DBG_DONE: src = d->done; need = B; break;
    case RPL_DBG_Q: src = d->Qs; need = B * A * 4; break;
    case RPL_DBG_QT_NEXT: src = d->Qt2; need = B * A * 4; break;
    case RPL_DBG_QO_NEXT: src = d->Qo2; need = B * A * 4; break;
    case RPL_DBG_Y: src = d->y; need = B * 4; break;
    case RPL_DBG_ASTAR: src = d->astar; need = B * 4; break;
    case RPL_DBG_LOSS: src = d->grad + d->P; need = 4; break;
    case RPL_DBG_H: need = B * d->Htot * 4; break;
    case RPL_DBG_TRACE:
        if (!d->trace) { set_error("dqn_debug_export: tracing is off (set RPL_TRACE=1)"); return RPL_ESTATE; }
        src = d->trace; need = 8 * 2048 * 8 * 8; break;
    default: set_error("dqn_debug_export: unknown item %d", what); return RPL_EINVAL;
    }
    if (bytes != need) {
        set_error("dqn_debug_export: item %d needs %lld bytes, got %lld", what, (long long)need,
                  (long long)bytes);
        return RPL_EINVAL;
    }
    if (what == RPL_DBG_H) {
        // hidden-unit space per sample: layer 0 units, layer 1 units, ... (online net on s)
        std::vector<float> tmp;
        int64_t off = 0;
        float *o = (float *)host_out;
        for (int l = 0; l < d->T; ++l) {
            tmp.resize((size_t)B * d->N[l]);
            RPL_CUDA(cudaMemcpyAsync(tmp.data(), d->H[l], tmp.size() * 4, cudaMemcpyDeviceToHost, d->stream));
            RPL_CUDA(cudaStreamSynchronize(d->stream));
            for (int64_t b = 0; b < B; ++b)
                memcpy(o + b * d->Htot + off, tmp.data() + b * d->N[l], (size_t)d->N[l] * 4);
            off += d->N[l];
        }
        return RPL_OK;
    }
    RPL_CUDA(cudaMemcpyAsync(host_out, src, (size_t)need, cudaMemcpyDeviceToHost, d->stream));
    RPL_CUDA(cudaStreamSynchronize(d->stream));
    return RPL_OK;
}

extern "C" int rpl_nccl_unique_id(void *out128)
{
    if (!out128) return RPL_EINVAL;
    int rc = nccl_load();
    if (rc != RPL_OK) return rc;
    nccl_uid id;
    int nr = g_nccl.get_uid(&id);
    if (nr != 0) {
        set_error("ncclGetUniqueId failed (%d)", nr);
        return RPL_ENCCL;
    }
    memcpy(out128, &id, sizeof id);
    return RPL_OK;
}

extern "C" int dqn_attach_nccl(rpl_dqn *d, int32_t rank, int32_t world, const void *id128)
{
    if (!d || !id128 || world < 1 || rank < 0 || rank >= world) return RPL_EINVAL;
    if (d->comm) {
        set_error("dqn_attach_nccl: already attached");
        return RPL_ESTATE;
    }
    // a world of one needs no communicator -- unless RPL_DP_FORCE=1 (tests run the whole NCCL
    // path, all-reduces over a single rank included, on one GPU)
    const char *ff = getenv("RPL_DP_FORCE");
    const bool force = ff && ff[0] == '1';
    if (world == 1 && !force) return RPL_OK;
    int rc = nccl_load();
    if (rc != RPL_OK) return rc;
    nccl_uid id;
    memcpy(&id, id128, sizeof id);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(d->device);
    int nr = g_nccl.init_rank(&d->comm, world, id, rank);
    if (prev >= 0) cudaSetDevice(prev);
    if (nr != 0) {
        d->comm = nullptr;
        set_error("ncclCommInitRank failed: %s", g_nccl.errstr ? g_nccl.errstr(nr) : "?");
        return RPL_ENCCL;
    }
    d->rank = rank;
    d->world = world;
    return RPL_OK;
}

// ---- peer-memory data parallelism (dp_peer.cuh) ----------------------------------------------
extern "C" int dqn_peer_handle(rpl_dqn *d, void *handle_out)
{
    if (!d || !handle_out) return RPL_EINVAL;
    DeviceGuardDqn g(d->device);
    if (!d->xbuf) {
        const size_t bytes = dp_xbuf_bytes(d->P);
        RPL_CUDA(cudaMalloc((void **)&d->xbuf, bytes));
        RPL_CUDA(cudaMemset(d->xbuf, 0, bytes));
    }
    cudaIpcMemHandle_t h;
    RPL_CUDA(cudaIpcGetMemHandle(&h, d->xbuf));
    memcpy(handle_out, &h, sizeof h);
    return RPL_OK;
}

extern "C" int dqn_attach_peers(rpl_dqn *d, int32_t rank, int32_t world, const void *handles)
{
    if (!d || !handles || world < 1 || world > DP_MAXR || rank < 0 || rank >= world) return RPL_EINVAL;
    if (d->comm || d->p2p || !d->xbuf || d->cfg.avg_period > 0) {
        set_error("dqn_attach_peers: needs dqn_peer_handle first, no NCCL attach, avg_period 0");
        return RPL_ESTATE;
    }
    DeviceGuardDqn g(d->device);
    // a fresh protocol state: step flags, the broken word and the block counter are cleared and
    // exchange steps count from here (a learner re-attached after a detach, a
    // timeout or solo steps would otherwise read stale flags); the caller synchronises the
    // ranks after every rank's attach and before the first step (dp.attach_auto's final
    // all-reduce), so no peer can publish into a flag area before it is cleared
    RPL_CUDA(cudaStreamSynchronize(d->stream));
    RPL_CUDA(cudaMemset((char *)d->xbuf + dp_flag_offset(d->P), 0, 256));
    RPL_CUDA(cudaDeviceSynchronize());
    d->dp_base = d->steps;
    drop_dp_graphs(d);   // their exchange kernels were captured for the previous attach
    const cudaIpcMemHandle_t *hs = static_cast<const cudaIpcMemHandle_t *>(handles);
    for (int q = 0; q < world; ++q) {
        if (q == rank) {
            d->peer_xbuf[q] = d->xbuf;
            continue;
        }
        void *ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, hs[q], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int r = 0; r < q; ++r)
                if (d->peer_opened[r]) {
                    cudaIpcCloseMemHandle(d->peer_xbuf[r]);
                    d->peer_opened[r] = false;
                }
            return cuda_fail(e, "cudaIpcOpenMemHandle");
        }
        d->peer_xbuf[q] = (float *)ptr;
        d->peer_opened[q] = true;
    }
    d->rank = rank;
    d->world = world;
    d->p2p = true;
    return RPL_OK;
}

extern "C" int dqn_detach_peers(rpl_dqn *d)
{
    if (!d) return RPL_EINVAL;
    DeviceGuardDqn g(d->device);
    cudaStreamSynchronize(d->stream);
    for (int q = 0; q < DP_MAXR; ++q) {
        if (d->peer_opened[q]) cudaIpcCloseMemHandle(d->peer_xbuf[q]);
        d->peer_opened[q] = false;
        d->peer_xbuf[q] = nullptr;
    }
    if (d->p2p) {
        d->p2p = false;
        d->rank = 0;
        d->world = 1;
    }
    drop_dp_graphs(d);
    return RPL_OK;
}

// test entry: `world` ranks emulated by one cooperative launch on this device (dp_peer.cuh)
extern "C" int rpl_dp_emulate(int32_t world, int64_t P, float *xbufs, float *online, float *target,
                              float *gmean, const int32_t *sync_flag, uint32_t *err, float lr,
                              uint64_t t, int32_t reduce_scatter)
{
    if (world < 1 || world > DP_MAXR || P < 1 || !xbufs || !online || !target || !gmean ||
        !sync_flag || !err || t == 0)
        return RPL_EINVAL;
    const size_t stride = dp_xbuf_bytes(P) / sizeof(float);
    DPArgs a{};
    a.nloc = world;
    a.world = world;
    a.rank0 = 0;
    a.P = P;
    a.t = t;
    a.lr = lr;
    for (int q = 0; q < world; ++q) {
        a.xbuf[q] = xbufs + q * stride;
        a.flag[q] = dp_flag_of(xbufs + q * stride, P);
        a.online[q] = online + q * P;
        a.target[q] = target + q * P;
        a.gmean[q] = gmean + q * (P + 1);
        a.sync_flag[q] = sync_flag;
        a.err[q] = err;
    }
    const int bpr = 8;
    void *args[] = {&a};
    RPL_CUDA(cudaLaunchCooperativeKernel(reduce_scatter ? (const void *)dp_peer_rs_sgd_kernel
                                                        : (const void *)dp_peer_sgd_kernel,
                                         dim3(world * bpr), dim3(256), args, 0, nullptr));
    RPL_CUDA(cudaDeviceSynchronize());
    return RPL_OK;
}

extern "C" int rpl_check(void *handle, int kind)
{
    if (!handle || (kind != 0 && kind != 1)) return RPL_EINVAL;
    cudaStream_t st;
    uint32_t *err;
    if (kind == 0) {
        if (int rc = replay_flush((rpl_replay *)handle)) return rc;
        st = ((rpl_replay *)handle)->stream;
        err = ((rpl_replay *)handle)->err_dev;
    } else {
        st = ((rpl_dqn *)handle)->stream;
        err = ((rpl_dqn *)handle)->err;
    }
    RPL_CUDA(cudaStreamSynchronize(st));
    uint32_t h = 0;
    RPL_CUDA(cudaMemcpy(&h, err, sizeof h, cudaMemcpyDeviceToHost));
    if (h) RPL_CUDA(cudaMemset(err, 0, sizeof h));
    if (h & ERRBIT_CORRUPT) {
        set_error("corrupt experience: a device-sourced terminal flag > 1 or a sampled action outside [0, A) "
                  "(that step's update was skipped)");
        return RPL_ECORRUPT;
    }
    if (h & ERRBIT_NUMERIC) { set_error("non-finite loss: update skipped"); return RPL_ENUMERIC; }
    if (h & ERRBIT_RANGE) { set_error("gather index out of range (clamped)"); return RPL_EINVAL; }
    if (h & ERRBIT_PEER) {
        set_error("peer-memory data parallelism: a rank did not publish its gradient (update skipped)");
        return RPL_ENCCL;
    }
    return RPL_OK;
}
