// simt_gemm.cuh -- FP32 register-tiled SIMT GEMM tile + operand loaders shared by the train-step
// kernels (CUDA path only).
#pragma once
#include <stdint.h>

namespace rpl {

constexpr int NT = 256;   // threads per CTA
constexpr int BM = 32;    // tile rows
constexpr int BN = 64;    // tile cols
constexpr int BK = 32;    // contraction chunk

struct __align__(16) GemmSmem {
    float As[BK][BM + 4];
    float Bs[BK][BN + 4];
};

// ------------------------------------------------------------------------------------------
// 32x64 register-tiled FP32 GEMM tile: C[m][n] = sum_{kk in [kb,ke)} A(m,kk) * B(n,kk).
// Operand loaders return 0 outside their bounds.  Each thread owns a 2x4 block of C.
// The next chunk is fetched into registers while the current one is multiplied.
// If want_rowsum, rs(m, sum_kk A(m,kk)) is also produced (bias gradients).
// ------------------------------------------------------------------------------------------
template <class LA, class LB, class EPI, class RSUM>
__device__ __forceinline__ void gemm_tile(const LA &la, const LB &lb, int m0, int n0, int kb,
                                          int ke, const EPI &epi, bool want_rowsum,
                                          const RSUM &rs, GemmSmem &sm)
{
    const int tid = threadIdx.x, tn = tid & 15, tm = tid >> 4;
    float acc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    float rsum0 = 0.0f, rsum1 = 0.0f;
    constexpr int NA = BM * BK / NT, NB = BN * BK / NT;
    float ra[NA], rb[NB];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int e = i * NT + tid;
            const int r = LA::kKContig ? e / BK : e % BM;
            const int kk = LA::kKContig ? e % BK : e / BM;
            ra[i] = la(m0 + r, k0 + kk);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int e = i * NT + tid;
            const int r = LB::kKContig ? e / BK : e % BN;
            const int kk = LB::kKContig ? e % BK : e / BN;
            rb[i] = lb(n0 + r, k0 + kk);
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            const int e = i * NT + tid;
            const int r = LA::kKContig ? e / BK : e % BM;
            const int kk = LA::kKContig ? e % BK : e / BM;
            sm.As[kk][r] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int e = i * NT + tid;
            const int r = LB::kKContig ? e / BK : e % BN;
            const int kk = LB::kKContig ? e % BK : e / BN;
            sm.Bs[kk][r] = rb[i];
        }
    };
    const int nchunks = (ke - kb + BK - 1) / BK;
    if (nchunks > 0) {
        fetch(kb);
        stash();
        __syncthreads();
        for (int c = 0; c < nchunks; ++c) {
            if (c + 1 < nchunks) fetch(kb + (c + 1) * BK);
#pragma unroll 8
            for (int k = 0; k < BK; ++k) {
                const float2 av = *reinterpret_cast<const float2 *>(&sm.As[k][2 * tm]);
                const float4 bv = *reinterpret_cast<const float4 *>(&sm.Bs[k][4 * tn]);
                acc[0][0] = fmaf(av.x, bv.x, acc[0][0]);
                acc[0][1] = fmaf(av.x, bv.y, acc[0][1]);
                acc[0][2] = fmaf(av.x, bv.z, acc[0][2]);
                acc[0][3] = fmaf(av.x, bv.w, acc[0][3]);
                acc[1][0] = fmaf(av.y, bv.x, acc[1][0]);
                acc[1][1] = fmaf(av.y, bv.y, acc[1][1]);
                acc[1][2] = fmaf(av.y, bv.z, acc[1][2]);
                acc[1][3] = fmaf(av.y, bv.w, acc[1][3]);
            }
            if (want_rowsum && tn == 0) {
                for (int k = 0; k < BK; ++k) {
                    rsum0 += sm.As[k][2 * tm];
                    rsum1 += sm.As[k][2 * tm + 1];
                }
            }
            __syncthreads();
            if (c + 1 < nchunks) {
                stash();
                __syncthreads();
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) epi(m0 + 2 * tm + i, n0 + 4 * tn + j, acc[i][j]);
    if (want_rowsum && tn == 0) {
        rs(m0 + 2 * tm, rsum0);
        rs(m0 + 2 * tm + 1, rsum1);
    }
}

// ---- operand loaders --------------------------------------------------------------------
// row-major [rows x ld] matrix, element (r, kk) = p[r*ld + kk], valid for r < R, kk < KE
struct LdKMajor {
    static constexpr bool kKContig = true;
    const float *p;
    int ld, R, KE;
    __device__ float operator()(int r, int kk) const
    {
        return (r < R && kk < KE) ? __ldcg(p + (int64_t)r * ld + kk) : 0.0f;
    }
};
// element (r, kk) = p[kk*ld + r] (contiguous along r), valid for r < R, kk in [KB, KE)
struct LdRMajor {
    static constexpr bool kKContig = false;
    const float *p;
    int ld, R, KB, KE;
    __device__ float operator()(int r, int kk) const
    {
        return (r < R && kk >= KB && kk < KE) ? __ldcg(p + (int64_t)kk * ld + r) : 0.0f;
    }
};
// gathered replay rows: element (m, k) = ring[idx[m - m0] * rs + col0 + k]
struct LdRing {
    static constexpr bool kKContig = true;
    const float *ring;
    const int *idx_s;
    int m0, rs, col0, R, KE;
    __device__ float operator()(int m, int k) const
    {
        return (m < R && k < KE) ? __ldg(ring + (int64_t)idx_s[m - m0] * rs + col0 + k) : 0.0f;
    }
};

struct NoRowsum {
    __device__ void operator()(int, float) const {}
};

__device__ __forceinline__ float warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


}  // namespace rpl
