// philox.cuh -- Philox4x32-10 and the index mapping of the sampler (library: the device
// sampler, and the host sampler of the in-RAM comparison mode RPL_RING_HOST_BATCH).
//
// Written independently of the oracle (oracle/oracle.c); both follow Salmon et al., SC'11
// and DESIGN.md reading Q3.  Parity of the two is checked bit-exactly by tests/test_gpu_*.
#pragma once
#include <stdint.h>

namespace rpl {

struct u32x4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b)
{
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}
__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b)
{
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = mulhi32(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = mulhi32(0xCD9E8D57u, c.z);
        c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;   // the bump after the last round is never used
        k1 += 0xBB67AE85u;
    }
    return c;
}

// The two sampled indices of Philox call j of event `event`: (index 2j, index 2j+1).
// u = hi:lo of one word pair, idx = floor(u * n / 2^64)  (n < 2^31).
__host__ __device__ __forceinline__ void sample_pair(uint64_t seed, uint32_t rank, uint64_t event,
                                            uint32_t j, uint64_t n, int32_t &i0, int32_t &i1)
{
    u32x4 c{j, (uint32_t)event, (uint32_t)(event >> 32), (1u << 24) | (rank & 0xFFFFFFu)};
    u32x4 x = philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t u0 = ((uint64_t)x.y << 32) | x.x;
    const uint64_t u1 = ((uint64_t)x.w << 32) | x.z;
    i0 = (int32_t)mulhi64(u0, n);
    i1 = (int32_t)mulhi64(u1, n);
}

}  // namespace rpl
