// mma_tf32.cuh -- FP32-accurate warp-level tensor-core products for the small 16-row tiles of
// the fast path: "3xTF32" on mma.sync.m16n8k8 (CUDA path only).
//
// x = hi + lo with hi = tf32(x), lo = x - hi (read as tf32 by the MMA); a.b ~= hi_a hi_b + hi_a lo_b + lo_a hi_b
// (the dropped lo_a lo_b term is ~2^-22 relative), accumulated in FP32.  Small terms are
// accumulated first.  The error is at FP32 round-off level, which keeps the 1e-5 normwise
// parity of the FP32 path (BASELINE north star); tests/test_gpu_train.py checks it.
//
// Fragment layouts of m16n8k8.row.col.f32.tf32.tf32.f32 (g = lane / 4, t = lane % 4):
//   A 16x8 : a0 (g, t)   a1 (g+8, t)   a2 (g, t+4)   a3 (g+8, t+4)
//   B 8x8  : b0 (k=t, n=g)             b1 (k=t+4, n=g)
//   C 16x8 : c0 (g, 2t)  c1 (g, 2t+1)  c2 (g+8, 2t)  c3 (g+8, 2t+1)
#pragma once
#include <stdint.h>

namespace rpl {

// hi = x rounded to tf32 (half away from zero: +half an ulp of the 10-bit mantissa, then
// truncate; 2 integer ops instead of the multi-instruction cvt.rna.tf32 sequence sm_100a emits);
// lo = x - hi is exact in fp32 and is passed raw: the MMA reads only its tf32 bits (the
// dropped bits are ~2^-21 of x)
__device__ __forceinline__ void tf32_split(float x, uint32_t &hi, uint32_t &lo)
{
    hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

// precision of a learner's tensor-core products (rpl_dqn_config.precision): 0 = FP32 (the
// 3xTF32 split above), 1 = TF32 (one product of tf32-rounded operands), 2 = BF16 (one product
// of bf16-rounded operands: exact in the fp32 accumulator, i.e. a BF16 MMA's numerics).  The
// reduced modes leave lo = 0 and skip the correction products.
__device__ __forceinline__ void split_p(float x, uint32_t &hi, uint32_t &lo, int prec)
{
    if (prec == 0) {
        tf32_split(x, hi, lo);
        return;
    }
    hi = prec == 2 ? (__float_as_uint(x) + 0x8000u) & 0xffff0000u : (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    lo = 0u;
}

__device__ __forceinline__ void mma_tf32(float c[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1)
{
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// c += A(16x8) B(8x8) with both operands given as hi/lo pairs
__device__ __forceinline__ void mma_3xtf32(float c[4], const uint32_t ah[4], const uint32_t al[4],
                                           const uint32_t bh[2], const uint32_t bl[2], int prec = 0)
{
    if (prec == 0) {
        mma_tf32(c, al[0], al[1], al[2], al[3], bh[0], bh[1]);
        mma_tf32(c, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
    }
    mma_tf32(c, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
}

// The three products into three independent accumulators (no dependent-HMMA chain inside a
// k-step); combine small terms first with acc3_sum.
__device__ __forceinline__ void mma_3xtf32_sep(float chh[4], float chl[4], float clh[4],
                                               const uint32_t ah[4], const uint32_t al[4],
                                               const uint32_t bh[2], const uint32_t bl[2], int prec = 0)
{
    if (prec == 0) {
        mma_tf32(clh, al[0], al[1], al[2], al[3], bh[0], bh[1]);
        mma_tf32(chl, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
    }
    mma_tf32(chh, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
}
__device__ __forceinline__ float acc3_sum(float hh, float hl, float lh) { return (lh + hl) + hh; }

}  // namespace rpl
