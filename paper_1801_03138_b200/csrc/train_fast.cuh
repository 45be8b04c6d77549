// train_fast.cuh -- the fast path of the device-resident train step for two trunk layers
// (the paper's dueling net 27 -> 128 -> [V 512 | A 512] -> 1 + |A|, and the plain
// 27 -> 64 -> 64 -> |A| MLP of configs[0]).  Four kernels, captured once per batch size into a
// CUDA graph:
//
//   K1 fwd  : per (net, 16-row batch tile, 128-unit tile): Philox sample + gather the 16 rows,
//             layer 0 for the tile's rows (recomputed per unit tile: 55 kMAC, cheaper than a
//             grid-wide exchange), layer-1 units of the tile, and the tile's partial sums of the
//             V/A heads.  Weight tiles stream into shared memory with cp.async while the gather
//             is in flight.
//   K2 td   : per sample: reduce head partials, dueling combine, max / argmax (warp shuffles),
//             TD target, Huber, dQ, dV/dA, and dZ1 = dHead . W_head (*) ReLU'(z1).
//   K3 bwd1 : dW1 = dZ1^T H0 and split-K partials of dH0 = dZ1 W1 (32x64 SIMT GEMM tiles),
//             head-weight gradients.
//   K4 bwd0 : dZ0 = (sum of dH0 partials) (*) ReLU'(z0), dW0 = dZ0^T X, then SGD of every
//             parameter (non-finite guard), target sync, counters.
//
// Step-varying state (sampler event, ring size, step counter) lives in device memory so the
// same graph replays every step with no host input.
#pragma once
#include "philox.cuh"
#include "simt_gemm.cuh"

namespace rpl {

constexpr int F_BT = 16;          // batch rows per K1 task
constexpr int F_MAXJ = 33;        // head outputs (1 + 32 actions)

struct FastArgs {
    // replay (rctrl[0] = sampler events consumed, rctrl[1] = filled size)
    const float *ring;
    int rs, D;
    uint64_t *rctrl;
    uint64_t seed;
    uint32_t rank;
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
    float *dH0p;         // [NS][B][N0]
    int NS;
    float *gpart;        // [nsb][P] (== grad when nsb == 1)
    int nsb, bsplit;
    float *grad;         // [P + 1]
    float *loss_part, *Qs, *Qt2, *Qo2, *y;
    int32_t *astar;
    float *loss_out;
    int64_t *step_dev;
    int32_t *sync_flag;  // written by K2 (step t+1 is a sync step), read by K4 / sgd_kernel
    int apply_update;
    uint32_t *err;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// shared-memory layout of K1 (floats); identical formula on the host (fast_fwd_smem_bytes)
struct FwdLayout {
    int DP, SW0, N0P, UT;
    int oX, oW0, oH0, oW1, oH1, oWh, ob0, ob1, oidx, total;
    __host__ __device__ FwdLayout(int D, int N0, int UT_, int J)
    {
        DP = (D + 3) & ~3;
        SW0 = ((DP + 31) & ~31) + 4;     // row stride == 4 (mod 32): conflict-free LDS.128
        N0P = ((N0 + 31) & ~31) + 4;
        UT = UT_;
        oX = 0;
        oW0 = oX + F_BT * DP;
        oH0 = oW0 + N0 * SW0;
        oW1 = oH0 + F_BT * N0P;
        oH1 = oW1 + UT * N0P;
        oWh = oH1 + F_BT * (UT + 1);
        ob0 = oWh + J * (UT + 1);
        ob1 = ob0 + N0;
        oidx = ob1 + UT;
        total = oidx + F_BT;
    }
};

// ------------------------------------------------------------------------------------------
// K1
// ------------------------------------------------------------------------------------------
template <int UT>
__global__ void __launch_bounds__(NT, 2) fast_fwd_kernel(const __grid_constant__ FastArgs p)
{
    extern __shared__ float4 smem4[];
    float *sm = reinterpret_cast<float *>(smem4);
    constexpr int RPT = F_BT * UT / NT;   // rows per thread in layer 1
    static_assert(RPT >= 1 && F_BT * UT == RPT * NT, "tile shape");
    const int D = p.D, N0 = p.N0, N1 = p.N1, J = p.J, B = p.B;
    const FwdLayout L(D, N0, UT, J);
    float *Xs = sm + L.oX, *W0s = sm + L.oW0, *H0s = sm + L.oH0, *W1s = sm + L.oW1;
    float *H1s = sm + L.oH1, *Whs = sm + L.oWh, *b0s = sm + L.ob0, *b1s = sm + L.ob1;
    int *idxs = reinterpret_cast<int *>(sm + L.oidx);
    const int tid = threadIdx.x;
    const int nbt = (B + F_BT - 1) / F_BT, nut = p.nut;
    const uint64_t event = p.rctrl[0];
    const uint64_t size = p.rctrl[1];
    const int ntasks = p.nets * nbt * nut;
    for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
        const int net = task / (nbt * nut), rem = task % (nbt * nut);
        const int bt = rem / nut, ut = rem % nut;
        const int rb = bt * F_BT, u0 = ut * UT;
        const float *theta = net == 1 ? p.target : p.online;
        __syncthreads();   // the previous task is done with shared memory
        // (1) stream the layer-1 weight tile into shared memory (rows stride N0P)
        {
            const int c4 = N0 / 4;
            for (int e = tid; e < UT * c4; e += NT) {
                const int u = e / c4, c = e % c4;
                float *dst = W1s + u * L.N0P + 4 * c;
                if (u0 + u < N1)
                    cp_async16(dst, theta + p.w1 + (int64_t)(u0 + u) * N0 + 4 * c);
                else
                    *reinterpret_cast<float4 *>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        // (2) Philox sample of the tile's rows (Q3)
        if (tid < F_BT / 2) {
            int32_t i0, i1;
            sample_pair(p.seed, p.rank, event, (uint32_t)(rb / 2 + tid), size, i0, i1);
            idxs[2 * tid] = i0;
            idxs[2 * tid + 1] = i1;
        }
        // (3) layer-0 weights (transposed copy, zero-padded), biases, head-weight tile
        for (int e = tid; e < N0 * L.DP; e += NT) {
            const int n = e / L.DP, d = e % L.DP;
            W0s[n * L.SW0 + d] = d < D ? __ldg(theta + p.w0 + (int64_t)n * D + d) : 0.0f;
        }
        for (int n = tid; n < N0; n += NT) b0s[n] = __ldg(theta + p.b0 + n);
        for (int u = tid; u < UT; u += NT) b1s[u] = (u0 + u < N1) ? __ldg(theta + p.b1 + u0 + u) : 0.0f;
        for (int e = tid; e < J * UT; e += NT) {
            const int j = e / UT, u = e % UT, g = u0 + u;
            float w = 0.0f;
            if (g < N1) {
                if (!p.dueling) w = __ldg(theta + p.wh + (int64_t)j * N1 + g);
                else if (j == 0 && g < p.S) w = __ldg(theta + p.wh + g);
                else if (j > 0 && g >= p.S) w = __ldg(theta + p.wh + (int64_t)j * p.S + (g - p.S));
            }
            Whs[j * (UT + 1) + u] = w;
        }
        __syncthreads();
        // (4) gather the 16 sampled rows: s for online(s), s' for target(s') / online(s')
        const int col0 = net == 0 ? 0 : D;
        for (int e = tid; e < F_BT * L.DP; e += NT) {
            const int rr = e / L.DP, d = e % L.DP;
            Xs[rr * L.DP + d] = d < D ? __ldg(p.ring + (int64_t)idxs[rr] * p.rs + col0 + d) : 0.0f;
        }
        if (ut == 0 && net <= 1) {
            // unpack the batch once for the backward pass and the debug export
            for (int e = tid; e < F_BT * D; e += NT) {
                const int rr = e / D, d = e % D;
                if (rb + rr < B)
                    (net == 0 ? p.Xs : p.Xs2)[(int64_t)(rb + rr) * D + d] =
                        __ldg(p.ring + (int64_t)idxs[rr] * p.rs + col0 + d);
            }
            if (net == 0 && tid < F_BT && rb + tid < B) {
                const float *row = p.ring + (int64_t)idxs[tid] * p.rs + 2 * D;
                p.idx[rb + tid] = idxs[tid];
                p.a[rb + tid] = __float_as_int(__ldg(row));
                p.r[rb + tid] = __ldg(row + 1);
                p.done[rb + tid] = (uint8_t)(__float_as_uint(__ldg(row + 2)) != 0u);
            }
        }
        __syncthreads();
        // (5) layer 0 for the tile's rows: H0 = ReLU(X W0^T + b0)
        for (int o = tid; o < F_BT * N0; o += NT) {
            const int rr = o / N0, n = o % N0;
            const float4 *x4 = reinterpret_cast<const float4 *>(Xs + rr * L.DP);
            const float4 *w4 = reinterpret_cast<const float4 *>(W0s + n * L.SW0);
            float acc = b0s[n];
            for (int q = 0; q < L.DP / 4; ++q) {
                const float4 x = x4[q], w = w4[q];
                acc = fmaf(x.x, w.x, acc);
                acc = fmaf(x.y, w.y, acc);
                acc = fmaf(x.z, w.z, acc);
                acc = fmaf(x.w, w.w, acc);
            }
            const float h = acc > 0.0f ? acc : 0.0f;
            H0s[rr * L.N0P + n] = h;
            if (net == 0 && ut == 0 && rb + rr < B) p.H0[(int64_t)(rb + rr) * N0 + n] = h;
        }
        cp_async_wait_all();
        __syncthreads();
        // (6) layer 1: thread (u, row group): RPT rows x 1 unit, float4 over k
        {
            const int u = tid % UT, r0 = (tid / UT) * RPT;
            float acc[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) acc[i] = b1s[u];
            const float4 *w4 = reinterpret_cast<const float4 *>(W1s + u * L.N0P);
            for (int q = 0; q < N0 / 4; ++q) {
                const float4 w = w4[q];
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const float4 h = reinterpret_cast<const float4 *>(H0s + (r0 + i) * L.N0P)[q];
                    acc[i] = fmaf(h.x, w.x, acc[i]);
                    acc[i] = fmaf(h.y, w.y, acc[i]);
                    acc[i] = fmaf(h.z, w.z, acc[i]);
                    acc[i] = fmaf(h.w, w.w, acc[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const float h = acc[i] > 0.0f ? acc[i] : 0.0f;
                H1s[(r0 + i) * (UT + 1) + u] = h;
                if (net == 0 && rb + r0 + i < B && u0 + u < N1)
                    p.H1[(int64_t)(rb + r0 + i) * N1 + u0 + u] = h;
            }
        }
        __syncthreads();
        // (7) this tile's partial sums of the head outputs
        for (int o = tid; o < F_BT * J; o += NT) {
            const int rr = o / J, j = o % J;
            const float *h = H1s + rr * (UT + 1);
            const float *w = Whs + j * (UT + 1);
            float acc = 0.0f;
            for (int u = 0; u < UT; ++u) acc = fmaf(w[u], h[u], acc);
            if (rb + rr < B) p.part[(((int64_t)net * nut + ut) * B + rb + rr) * J + j] = acc;
        }
    }
}

// ------------------------------------------------------------------------------------------
// K2: one CTA per sample
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float f_huber(float d, float kappa, int kinf)
{
    const float ad = fabsf(d);
    if (kinf || ad <= kappa) return 0.5f * d * d;
    return kappa * (ad - 0.5f * kappa);
}

__global__ void __launch_bounds__(NT) fast_td_kernel(const __grid_constant__ FastArgs p)
{
    __shared__ float hs[3][F_MAXJ + 1];
    __shared__ float dhs[F_MAXJ + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int A = p.A, J = p.J, B = p.B, N1 = p.N1, S = p.S;
    if (blockIdx.x == 0 && tid == 0) {
        const int64_t t = *p.step_dev + 1;
        *p.sync_flag = (p.sync_period > 0 && t % p.sync_period == 0) ? 1 : 0;
    }
    for (int b = blockIdx.x; b < B; b += gridDim.x) {
        __syncthreads();
        if (warp < p.nets) {
            const float *theta = warp == 1 ? p.target : p.online;
            for (int j = lane; j < J; j += 32) {
                float v = __ldg(theta + p.bh + j);
                for (int ut = 0; ut < p.nut; ++ut)
                    v += __ldcg(p.part + (((int64_t)warp * p.nut + ut) * B + b) * J + j);
                hs[warp][j] = v;
            }
        }
        __syncthreads();
        if (warp == 0) {
            float q[3];
#pragma unroll
            for (int net = 0; net < 3; ++net) {
                float qa = 0.0f;
                if (net < p.nets) {
                    if (p.dueling) {
                        // Q(s,a) = V(s) + A(s,a) - (1/|A|) sum_a' A(s,a')
                        float mean = 0.0f;
                        for (int k = 0; k < A; ++k) mean += hs[net][1 + k];
                        mean /= (float)A;
                        if (lane < A) qa = hs[net][0] + hs[net][1 + lane] - mean;
                    } else if (lane < A) {
                        qa = hs[net][lane];
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
            const int ab = p.a[b];
            const float notdone = p.done[b] ? 0.0f : 1.0f;
            const float yb = p.r[b] + p.gamma * notdone * boot;
            const float qsel = __shfl_sync(0xffffffffu, q[0], ab);   // Q[i*A + a_i]
            const float delta = qsel - yb;
            const float g = (p.kinf ? delta : fminf(fmaxf(delta, -p.kappa), p.kappa)) / (float)B;
            if (p.dueling) {
                if (lane == 0) dhs[0] = g;
                if (lane < A) dhs[1 + lane] = (lane == ab ? g : 0.0f) - g / (float)A;
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
        __syncthreads();
        for (int j = tid; j < J; j += NT) p.dHead[(int64_t)b * J + j] = dhs[j];
        // dZ1[b][u] = (dHead . W_head)[u] * ReLU'(z1[b][u])
        const float *Wh = p.online + p.wh;
        for (int u = tid; u < N1; u += NT) {
            float dh = 0.0f;
            if (p.dueling) {
                if (u < S) {
                    dh = dhs[0] * __ldg(Wh + u);
                } else {
                    for (int k = 0; k < A; ++k) dh = fmaf(dhs[1 + k], __ldg(Wh + (int64_t)(1 + k) * S + (u - S)), dh);
                }
            } else {
                for (int k = 0; k < A; ++k) dh = fmaf(dhs[k], __ldg(Wh + (int64_t)k * N1 + u), dh);
            }
            p.dZ1[(int64_t)b * N1 + u] = __ldcg(p.H1 + (int64_t)b * N1 + u) > 0.0f ? dh : 0.0f;
        }
    }
}

// ------------------------------------------------------------------------------------------
// K3: dW1 / db1 tiles, dH0 split-K tiles, head-weight gradients
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) fast_bwd1_kernel(const __grid_constant__ FastArgs p)
{
    __shared__ GemmSmem sm;
    __shared__ float dhs[128 * F_MAXJ];
    const int N0 = p.N0, N1 = p.N1, B = p.B, J = p.J;
    const int wmt = (N1 + BM - 1) / BM, wnt = (N0 + BN - 1) / BN;
    const int n_w = wmt * wnt * p.nsb;
    const int hmt = (B + BM - 1) / BM, hnt = (N0 + BN - 1) / BN;
    const int n_h = hmt * hnt * p.NS;
    const int hu_tasks = (N1 + NT - 1) / NT;
    const int n_hd = (hu_tasks + 1) * p.nsb;
    const int ntasks = n_w + n_h + n_hd;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
        if (t < n_w) {
            const int s = t / (wmt * wnt), rem = t % (wmt * wnt);
            const int m0 = (rem / wnt) * BM, n0 = (rem % wnt) * BN;
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit);
            float *gp = p.gpart + (int64_t)s * p.P;
            LdRMajor la{p.dZ1, N1, N1, kb, ke};
            LdRMajor lb{p.H0, N0, N0, kb, ke};
            auto epi = [&](int m, int n, float v) {
                if (m < N1 && n < N0) gp[p.w1 + (int64_t)m * N0 + n] = v;
            };
            auto rs = [&](int m, float v) {
                if (m < N1) gp[p.b1 + m] = v;
            };
            gemm_tile(la, lb, m0, n0, kb, ke, epi, n0 == 0, rs, sm);
        } else if (t < n_w + n_h) {
            const int u = t - n_w;
            const int s = u / (hmt * hnt), rem = u % (hmt * hnt);
            const int m0 = (rem / hnt) * BM, n0 = (rem % hnt) * BN;
            const int chunk = (N1 + p.NS - 1) / p.NS;
            const int kb = s * chunk, ke = min(N1, kb + chunk);
            float *out = p.dH0p + (int64_t)s * B * N0;
            LdKMajor la{p.dZ1, N1, B, ke};
            LdRMajor lb{p.online + p.w1, N0, N0, kb, ke};
            auto epi = [&](int m, int n, float v) {
                if (m < B && n < N0) out[(int64_t)m * N0 + n] = v;
            };
            gemm_tile(la, lb, m0, n0, kb, ke, epi, false, NoRowsum{}, sm);
        } else {
            // g_Wh[j][u] = sum_b dHead[b][j] H1[b][u]; g_bh[j] = sum_b dHead[b][j]
            const int u = t - n_w - n_h;
            const int s = u / (hu_tasks + 1), c = u % (hu_tasks + 1);
            const int kb = s * p.bsplit, ke = min(B, kb + p.bsplit);
            float *gp = p.gpart + (int64_t)s * p.P;
            const int unit = c * NT + threadIdx.x;
            const bool is_bias = (c == hu_tasks);
            float acc[F_MAXJ];
#pragma unroll
            for (int j = 0; j < F_MAXJ; ++j) acc[j] = 0.0f;
            for (int c0 = kb; c0 < ke; c0 += 128) {
                const int c1 = min(ke, c0 + 128);
                __syncthreads();
                for (int e = threadIdx.x; e < (c1 - c0) * J; e += NT)
                    dhs[e] = __ldcg(p.dHead + (int64_t)c0 * J + e);
                __syncthreads();
                if (is_bias) {
                    if (threadIdx.x < J)
                        for (int bb = 0; bb < c1 - c0; ++bb) acc[0] += dhs[bb * J + threadIdx.x];
                } else if (unit < N1) {
                    int jlo = 0, jhi = J;
                    if (p.dueling) {
                        if (unit < p.S) jhi = 1;
                        else jlo = 1;
                    }
#pragma unroll 4
                    for (int bb = 0; bb < c1 - c0; ++bb) {
                        const float h = __ldcg(p.H1 + (int64_t)(c0 + bb) * N1 + unit);
#pragma unroll
                        for (int j = 0; j < F_MAXJ; ++j)
                            if (j >= jlo && j < jhi) acc[j] = fmaf(dhs[bb * J + j], h, acc[j]);
                    }
                }
            }
            if (is_bias) {
                if (threadIdx.x < J) gp[p.bh + threadIdx.x] = acc[0];
            } else if (unit < N1) {
#pragma unroll
                for (int j = 0; j < F_MAXJ; ++j) {
                    if (j >= J) break;
                    if (!p.dueling) gp[p.wh + (int64_t)j * N1 + unit] = acc[j];
                    else if (j == 0 && unit < p.S) gp[p.wh + unit] = acc[0];
                    else if (j > 0 && unit >= p.S) gp[p.wh + (int64_t)j * p.S + (unit - p.S)] = acc[j];
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// K4: layer-0 backward + SGD of every parameter + target sync + counters
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) fast_bwd0_sgd_kernel(const __grid_constant__ FastArgs p)
{
    __shared__ float dzs[NT];
    __shared__ float red[NT];
    const int tid = threadIdx.x;
    const int N0 = p.N0, D = p.D, B = p.B;
    // batch-mean loss (fixed-order reduction, identical in every CTA)
    float ls = 0.0f;
    for (int b = tid; b < B; b += NT) ls += __ldcg(p.loss_part + b);
    ls = warp_sum(ls);
    if ((tid & 31) == 0) red[tid >> 5] = ls;
    __syncthreads();
    float lsum = 0.0f;
    for (int w = 0; w < NT / 32; ++w) lsum += red[w];
    const float loss = lsum / (float)B;
    const bool ok = isfinite(loss);
    const bool upd = p.apply_update && ok;
    const bool do_sync = *p.sync_flag != 0;
    __syncthreads();
    // (a) one CTA per layer-0 unit n: dZ0[:, n], dW0[n][:], db0[n], then its SGD
    for (int n = blockIdx.x; n < N0; n += gridDim.x) {
        // thread (d = tid % 32, group g = tid / 32) accumulates sum_b dZ0[b][n] X[b][d]
        const int d = tid & 31, grp = tid >> 5;
        float accw = 0.0f, accb = 0.0f;
        for (int c0 = 0; c0 < B; c0 += NT) {
            const int b = c0 + tid;
            float dz = 0.0f;
            if (b < B) {
                for (int s = 0; s < p.NS; ++s) dz += __ldcg(p.dH0p + ((int64_t)s * B + b) * N0 + n);
                dz = __ldcg(p.H0 + (int64_t)b * N0 + n) > 0.0f ? dz : 0.0f;
            }
            __syncthreads();
            dzs[tid] = dz;
            __syncthreads();
            const int cn = min(NT, B - c0);
            for (int bb = grp; bb < cn; bb += NT / 32) {
                const float z = dzs[bb];
                if (d < D) accw = fmaf(z, __ldcg(p.Xs + (int64_t)(c0 + bb) * D + d), accw);
                if (d == 0) accb += z;
            }
        }
        __syncthreads();
        red[tid] = accw;
        __syncthreads();
        if (tid < 32) {
            float s = 0.0f;
            for (int g = 0; g < NT / 32; ++g) s += red[g * 32 + tid];
            if (tid < D) {
                const int64_t i = p.w0 + (int64_t)n * D + tid;
                p.grad[i] = s;
                if (upd) {
                    const float w = p.online[i] - p.lr * s;
                    p.online[i] = w;
                    if (do_sync) p.target[i] = w;
                }
            }
        }
        __syncthreads();
        red[tid] = accb;
        __syncthreads();
        if (tid == 0) {
            float s = 0.0f;
            for (int g = 0; g < NT / 32; ++g) s += red[g * 32];
            const int64_t i = p.b0 + n;
            p.grad[i] = s;
            if (upd) {
                const float w = p.online[i] - p.lr * s;
                p.online[i] = w;
                if (do_sync) p.target[i] = w;
            }
        }
        __syncthreads();
    }
    // (b) every other parameter: [w1, P) (the blob stores W0, b0 first)
    const int64_t lo = p.w1, n_el = p.P - p.w1;
    for (int64_t e = (int64_t)blockIdx.x * NT + tid; e < n_el; e += (int64_t)gridDim.x * NT) {
        const int64_t i = lo + e;
        float g;
        if (p.nsb == 1) {
            g = __ldcg(p.grad + i);
        } else {
            g = 0.0f;
            for (int s = 0; s < p.nsb; ++s) g += __ldcg(p.gpart + (int64_t)s * p.P + i);
            p.grad[i] = g;
        }
        if (upd) {
            const float w = p.online[i] - p.lr * g;
            p.online[i] = w;
            if (do_sync) p.target[i] = w;
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        p.grad[p.P] = loss;
        if (p.loss_out) *p.loss_out = loss;
        if (!ok) atomicOr(p.err, ERRBIT_NUMERIC);
        p.rctrl[0] += 1;          // sampler event consumed
        *p.step_dev += 1;         // executed train steps
    }
}

}  // namespace rpl
