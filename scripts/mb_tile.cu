// mb_tile.cu -- per-CTA cost of the K3 building blocks on B200: cp.async staging of a
// 32x128 + 64x128 fp32 operand pair, the 3xTF32 mma.sync tile loop, and both together.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1801_03138_b200/csrc mb_tile.cu
#include <cstdio>
#include <vector>

#include "../paper_1801_03138_b200/csrc/internal.h"
#include "../paper_1801_03138_b200/csrc/train_fast.cuh"

using namespace rpl;

__global__ void __launch_bounds__(256) k_tile(const float *A, const float *B, float *out, int mode,
                                              long long *cyc, int reps)
{
    extern __shared__ float4 smem4[];
    float *smf = reinterpret_cast<float *>(smem4);
    const long long t0 = clock64();
    const Opnd a{A + (size_t)blockIdx.x * 128 * 1024, 1024, 1024}, b{B + (size_t)blockIdx.x * 128 * 128, 128, 128};
    float sink = 0.0f;
    for (int rep = 0; rep < reps; ++rep) {
        if (mode == 0) {
            __syncthreads();
            mm_stage<true, BM>(smf, a, 0, 0, 128, threadIdx.x);
            mm_stage<true, K3N>(smf + MM_OPF, b, 0, 0, 128, threadIdx.x);
            cp_async_wait_all();
            __syncthreads();
            sink += smf[threadIdx.x];
        } else {
            auto epi = [&](int m, int n, float v) { sink += v; };
            gemm_mma_tile<true, true>(a, b, 0, 0, 0, 128, epi, false, NoRowsum{}, smf);
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (sink == 12345.0f) out[0] = sink;
}

int main()
{
    const int G = 145;
    float *A, *B, *o;
    long long *cyc;
    cudaMalloc(&A, (size_t)G * 128 * 1024 * 4);
    cudaMalloc(&B, (size_t)G * 128 * 128 * 4);
    cudaMemset(A, 0, (size_t)G * 128 * 1024 * 4);
    cudaMemset(B, 0, (size_t)G * 128 * 128 * 4);
    cudaMalloc(&o, 64);
    cudaMalloc(&cyc, G * 8);
    const size_t sm = MM_FLOATS * 4;
    cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int mode = 0; mode < 2; ++mode) {
        for (int reps : {1, 10}) {
            for (int w = 0; w < 3; ++w) k_tile<<<G, 256, sm>>>(A, B, o, mode, cyc, reps);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_tile<<<G, 256, sm>>>(A, B, o, mode, cyc, reps);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> h(G);
            cudaMemcpy(h.data(), cyc, G * 8, cudaMemcpyDeviceToHost);
            double mean = 0, mx = 0;
            for (auto v : h) { mean += v; mx = v > mx ? v : mx; }
            mean /= G;
            printf("mode %s reps %2d: kernel %.2f us, per-CTA cycles mean %.0f (%.2f us) max %.0f\n",
                   mode == 0 ? "stage" : "stage+mma", reps, 1000 * ms, mean, mean / 1965.0, mx);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
