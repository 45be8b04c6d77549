// umma.cuh -- 5th-generation tensor-core (tcgen05 / UMMA) building blocks for sm_100a: shared-
// memory matrix descriptors for the no-swizzle canonical layouts, the kind::f16 instruction
// descriptor (bf16 x bf16 -> fp32), MMA issue / commit, mbarriers, TMEM allocation and loads.
// CUDA path only.
//
// Canonical no-swizzle layouts (both majors): the operand is tiled into 128-byte "core
// matrices" of 8 rows x 16 bytes, rows 16 bytes apart:
//   K-major  : a core matrix = 8 M/N rows x 8 bf16 along K;
//   MN-major : a core matrix = 8 K rows  x 8 bf16 along M/N.
// SBO = byte distance between core matrices adjacent along M/N, LBO = along K.  One
// kind::f16 MMA consumes K = 16 (two core matrices along K).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace rpl {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

// shared-memory matrix descriptor, SWIZZLE_NONE, base offset 0, version 1 (sm_100)
__device__ __forceinline__ uint64_t desc(const void *smem, uint32_t lbo_bytes, uint32_t sbo_bytes)
{
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
    return d;                 // layout type bits [61,64) = 0: no swizzle
}

// instruction descriptor of tcgen05.mma kind::f16: A, B bf16, D fp32, M x N, majors
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn_major, bool b_mn_major)
{
    return (1u << 4)                          // D format fp32
         | (1u << 7)                          // A format bf16
         | (1u << 10)                         // B format bf16
         | ((a_mn_major ? 1u : 0u) << 15)
         | ((b_mn_major ? 1u : 0u) << 16)
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread for the whole CTA
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate ? 1u : 0u)
        : "memory");
}

// arrive on an mbarrier when every previously issued MMA of this thread has completed
__device__ __forceinline__ void commit(uint64_t *mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n"
        :: "r"(smem_u32(mbar)), "r"(phase) : "memory");
}

// one thread arms the mbarrier with the bytes its bulk copies will deliver (its arrival)
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(mbar)), "r"(bytes) : "memory");
}

// bulk (TMA engine) copy of `bytes` (multiple of 16, both ends 16-byte aligned) global ->
// shared memory, completing as transaction bytes on `mbar`
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, uint32_t bytes, uint64_t *mbar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}

// the same copy delivered to the same shared-memory offset (data and mbarrier) of every CTA
// of the cluster in ctaMask (TMA multicast)
__device__ __forceinline__ void bulk_g2s_mc(void *smem, const void *gmem, uint32_t bytes, uint64_t *mbar,
                                            uint16_t mask)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
                 "[%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(mbar)), "h"(mask) : "memory");
}

// operands written with ordinary st.shared must be made visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// TMEM: one warp allocates `cols` (power of two >= 32) columns; the address lands in smem
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t cols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst_smem)), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t cols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(cols) : "memory");
}

// warp w (mod 4) of a warpgroup reads TMEM lanes 32 (w % 4) .. + 31: thread t gets lane
// 32 (w % 4) + t, 8 consecutive fp32 columns starting at column `col`
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float v[8])
{
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// the same load without its wait: several loads in flight, then one tmem_wait_ld()
__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t r[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// fp32 -> three bf16 terms hi + mid + lo that carry all 24 significand bits (round-to-nearest
// at each stage): x - (hi + mid + lo) is 0 for normal x outside the bf16 underflow range
__device__ __forceinline__ void split3_bf16(float x, uint16_t &hi, uint16_t &mid, uint16_t &lo)
{
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(m);
    const __nv_bfloat16 l = __float2bfloat16_rn(r2);
    hi = __bfloat16_as_ushort(h);
    mid = __bfloat16_as_ushort(m);
    lo = __bfloat16_as_ushort(l);
}
// the same for two consecutive values, packed two per word (x0 in the low half): one paired
// conversion (F2FP ... PACK_AB) per term instead of two
__device__ __forceinline__ void split3_pack2(float x0, float x1, uint32_t &h, uint32_t &m, uint32_t &l)
{
    auto bits = [](__nv_bfloat162 v) { return *reinterpret_cast<uint32_t *>(&v); };
    h = bits(__floats2bfloat162_rn(x0, x1));
    const float r0 = x0 - __uint_as_float(h << 16), r1 = x1 - __uint_as_float(h & 0xffff0000u);
    m = bits(__floats2bfloat162_rn(r0, r1));
    const float q0 = r0 - __uint_as_float(m << 16), q1 = r1 - __uint_as_float(m & 0xffff0000u);
    l = bits(__floats2bfloat162_rn(q0, q1));
}

}  // namespace umma
}  // namespace rpl
