// mb_umma.cu -- correctness + timing probe of the tcgen05 building blocks in umma.cuh: one CTA
// computes D[128 x N] = A[128 x K] B[N x K]^T (bf16 in, fp32 accumulate in TMEM) with each
// operand K-major or MN-major in the no-swizzle canonical layout; exact integer inputs are
// checked against a CPU product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1801_03138_b200/csrc mb_umma.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace rpl;

constexpr int M = 128;

// byte offset of element (r, k) of an R x K operand in the canonical layout
__host__ __device__ inline uint32_t off_kmajor(int r, int k, int K) { return (r / 8) * (K / 8) * 128 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2; }
__host__ __device__ inline uint32_t off_mnmajor(int r, int k, int R) { return (k / 8) * (R / 8) * 128 + (r / 8) * 128 + (k % 8) * 16 + (r % 8) * 2; }

template <int N, int K, bool AMN, bool BMN>
__global__ void k_umma(const float *A, const float *B, float *D, long long *cyc)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *As = sm, *Bs = sm + M * K * 2;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < M * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        const uint32_t o = AMN ? off_mnmajor(r, k, M) : off_kmajor(r, k, K);
        *reinterpret_cast<__nv_bfloat16 *>(As + o) = __float2bfloat16_rn(A[e]);
    }
    for (int e = tid; e < N * K; e += blockDim.x) {
        const int r = e / K, k = e % K;
        const uint32_t o = BMN ? off_mnmajor(r, k, N) : off_kmajor(r, k, K);
        *reinterpret_cast<__nv_bfloat16 *>(Bs + o) = __float2bfloat16_rn(B[e]);
    }
    if (warp == 0) umma::tmem_alloc(&tbase, N < 32 ? 32 : N);
    if (tid == 0) {
        umma::mbar_init(&mbar, 1);
        umma::fence_mbar_init();
    }
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tbase;
    const long long t0 = clock64();
    if (tid == 0) {
        constexpr uint32_t idesc = umma::idesc_bf16(M, N, AMN, BMN);
        for (int s = 0; s < K / 16; ++s) {
            // K-major: the 2 core matrices along K are LBO = 128 B apart, 8-row groups SBO apart;
            // MN-major: 8-element MN groups are SBO = 128 B apart, K groups LBO apart
            const uint64_t ad = AMN ? umma::desc(As + 2 * s * (M / 8) * 128, (M / 8) * 128, 128)
                                    : umma::desc(As + 2 * s * 128, 128, (K / 8) * 128);
            const uint64_t bd = BMN ? umma::desc(Bs + 2 * s * (N / 8) * 128, (N / 8) * 128, 128)
                                    : umma::desc(Bs + 2 * s * 128, 128, (K / 8) * 128);
            umma::mma_bf16(tmem, ad, bd, idesc, s > 0);
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
    if (warp == 0) umma::tmem_free(tmem, N < 32 ? 32 : N);
    if (tid == 0) cyc[0] = t1 - t0;
}

template <int N, int K, bool AMN, bool BMN>
int run()
{
    std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N, 0.0);
    srand(1);
    for (auto &x : A) x = (float)(rand() % 17 - 8);
    for (auto &x : B) x = (float)(rand() % 13 - 6);
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
    const int smem = (M + N) * K * 2;
    cudaFuncSetAttribute(k_umma<N, K, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_umma<N, K, AMN, BMN><<<1, 128, smem>>>(dA, dB, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i)
        if (D[i] != R[i]) {
            if (bad < 5) printf("  mismatch at (%d,%d): got %f want %f\n", i / N, i % N, D[i], R[i]);
            ++bad;
        }
    printf("N=%3d K=%3d A %s B %s: %s (%d bad), %lld cycles for %d MMAs, err=%s\n", N, K,
           AMN ? "MN" : "K ", BMN ? "MN" : "K ", bad ? "FAIL" : "ok", bad, cyc, K / 16,
           cudaGetErrorString(e));
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
    return bad;
}

int main()
{
    int bad = 0;
    bad += run<64, 64, false, false>();
    bad += run<64, 64, true, false>();
    bad += run<64, 64, false, true>();
    bad += run<64, 64, true, true>();
    bad += run<256, 64, false, false>();
    bad += run<256, 128, true, true>();
    printf(bad ? "FAILURES\n" : "all ok\n");
    return 0;
}
