// mb_tc32.cu -- correctness + timing probe of the kind::tf32 tcgen05 building blocks the fast
// path's tensor-core kernels use: one CTA computes D[128 x N] = A[128 x K] B[N x K]^T with
//   (a) A and B in shared memory, each K-major or MN-major (no-swizzle canonical layouts of
//       32-bit elements: a core matrix is 8 rows x 16 bytes = 4 tf32),
//   (b) A in tensor memory (written with tcgen05.st, lane = row, one element per column).
// Exact small-integer inputs make every product exact, so D must equal a CPU product bit for bit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1801_03138_b200/csrc mb_tc32.cu -o mb_tc32
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace rpl;

constexpr int M = 128;

// byte offset of element (r, k) of an R x K tf32 operand in the canonical layouts
__host__ __device__ inline uint32_t off_k(int r, int k, int K) { return (r / 8) * (K / 4) * 128 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4; }
__host__ __device__ inline uint32_t off_mn(int r, int k, int R) { return (k / 8) * (R / 4) * 128 + (r / 4) * 128 + (k % 8) * 16 + (r % 4) * 4; }

__host__ __device__ constexpr uint32_t idesc_tf32(int Mm, int N, bool amn, bool bmn)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(Mm >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc ? 1u : 0u) : "memory");
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, bool acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                 :: "r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc ? 1u : 0u) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float v[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
                    "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
                    "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}

// MODE 0: A, B in smem; MODE 1: A in TMEM (columns [N_alloc_D, ...)), B in smem
template <int N, int K, bool AMN, bool BMN, int MODE>
__global__ void k_tc(const float *A, const float *B, float *D, long long *cyc)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *As = sm, *Bs = sm + M * K * 4;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr int DC = N < 32 ? 32 : N;
    constexpr int COLS = MODE == 1 ? 512 : (DC <= 32 ? 32 : DC <= 64 ? 64 : DC <= 128 ? 128 : 256);
    if (MODE == 0)
        for (int e = tid; e < M * K; e += blockDim.x) {
            const int r = e / K, k = e % K;
            *reinterpret_cast<float *>(As + (AMN ? off_mn(r, k, M) : off_k(r, k, K))) = A[e];
        }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        *reinterpret_cast<float *>(Bs + (BMN ? off_mn(r, k, N) : off_k(r, k, K))) = B[e];
    }
    if (warp == 0) umma::tmem_alloc(&tbase, COLS);
    if (tid == 0) {
        umma::mbar_init(&mbar, 1);
        umma::fence_mbar_init();
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tbase;
    const uint32_t ta = tmem + 256;   // A's columns (MODE 1)
    if (MODE == 1 && warp < 4) {
        const int row = 32 * warp + (tid & 31);
        for (int c = 0; c < K; c += 8) {
            float v[8];
            for (int i = 0; i < 8; ++i) v[i] = A[row * K + c + i];
            tmem_st8(ta + ((uint32_t)(32 * warp) << 16) + c, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const long long t0 = clock64();
    if (tid == 0) {
        constexpr uint32_t idesc = idesc_tf32(M, N, AMN, BMN);
        for (int s = 0; s < K / 8; ++s) {
            const uint64_t bd = BMN ? umma::desc(Bs + s * (N / 4) * 128, (N / 4) * 128, 128)
                                    : umma::desc(Bs + 2 * s * 128, 128, (K / 4) * 128);
            if (MODE == 0) {
                const uint64_t ad = AMN ? umma::desc(As + s * (M / 4) * 128, (M / 4) * 128, 128)
                                        : umma::desc(As + 2 * s * 128, 128, (K / 4) * 128);
                mma_tf32_ss(tmem, ad, bd, idesc, s > 0);
            } else {
                mma_tf32_ts(tmem, ta + 8 * s, bd, idesc, s > 0);
            }
        }
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after_sync();
    const long long t1 = clock64();
    if (warp < 4) {
        const int row = 32 * warp + (tid & 31);
        for (int c = 0; c < N; c += 8) {
            float v[8];
            umma::tmem_ld8(tmem + ((uint32_t)(32 * warp) << 16) + c, v);
            for (int i = 0; i < 8; ++i) D[row * N + c + i] = v[i];
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_free(tmem, COLS);
    if (tid == 0) cyc[0] = t1 - t0;
}

template <int N, int K, bool AMN, bool BMN, int MODE>
int run()
{
    std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N, 0.0);
    srand(1);
    // tf32 keeps 10 mantissa bits: small integers and their products / sums are exact
    for (auto &x : A) x = (float)(rand() % 17 - 8);
    for (auto &x : B) x = (float)(rand() % 13 - 6) * 0.25f;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
            R[m * N + n] = (float)s;
        }
    float *dA, *dB, *dD;
    long long *dc, cyc = 0;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    const int smem = (M + N) * K * 4;
    cudaFuncSetAttribute(k_tc<N, K, AMN, BMN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_tc<N, K, AMN, BMN, MODE><<<1, 128, smem>>>(dA, dB, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i)
        if (D[i] != R[i]) {
            if (bad < 5) printf("  mismatch at (%d,%d): got %f want %f\n", i / N, i % N, D[i], R[i]);
            ++bad;
        }
    printf("tf32 N=%3d K=%3d A %s B %s: %s (%d bad), %lld cycles for %d MMAs, err=%s\n", N, K,
           MODE == 1 ? "TM" : AMN ? "MN" : "K ", BMN ? "MN" : "K ", bad ? "FAIL" : "ok", bad, cyc,
           K / 8, cudaGetErrorString(e));
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
    return bad || e != cudaSuccess;
}

int main()
{
    int bad = 0;
    bad += run<64, 32, false, false, 0>();
    bad += run<64, 32, true, false, 0>();
    bad += run<64, 32, false, true, 0>();
    bad += run<64, 32, true, true, 0>();
    bad += run<128, 128, false, false, 0>();
    bad += run<128, 128, true, true, 0>();
    bad += run<256, 64, false, true, 0>();
    bad += run<32, 64, false, false, 0>();
    bad += run<64, 64, false, false, 1>();
    bad += run<128, 128, false, false, 1>();
    bad += run<128, 128, false, true, 1>();
    bad += run<256, 128, false, false, 1>();
    printf(bad ? "FAILURES\n" : "all ok\n");
    return 0;
}
