// mb_graph.cu -- device-side cost of back-to-back CUDA graph launches on B200: graphs of n
// short kernels launched 2000x on one stream (host far ahead), per launch vs per kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mb_graph.cu -o mb_graph
#include <cstdio>
#include <chrono>
__global__ void k_spin(int ns, int *p)
{
    extern __shared__ float smem[];
    if (ns < -1) smem[threadIdx.x] = 1.0f;
    const long long t0 = clock64();
    while (clock64() - t0 < ns) {}
    if (threadIdx.x == 0 && blockIdx.x == 0 && ns < 0) p[0] = 1;
}
int main()
{
    int *p;
    cudaMalloc(&p, 64);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    for (unsigned flags : {0u}) {
        for (int n : {1, 4}) {
            for (int spin : {0, 10000}) {
              for (int smem : {0, 140 * 1024}) {
                cudaGraph_t g;
                cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
                for (int i = 0; i < n; ++i) k_spin<<<148, 256, i == 0 ? smem : 0, st>>>(spin, p);
                cudaStreamEndCapture(st, &g);
                cudaGraphExec_t ge;
                if (cudaGraphInstantiateWithFlags(&ge, g, flags) != cudaSuccess) { printf("inst fail\n"); continue; }
                cudaGraphUpload(ge, st);
                for (int i = 0; i < 50; ++i) cudaGraphLaunch(ge, st);
                cudaStreamSynchronize(st);
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                const int L = 2000;
                auto h0 = std::chrono::steady_clock::now();
                cudaEventRecord(a, st);
                for (int i = 0; i < L; ++i) cudaGraphLaunch(ge, st);
                cudaEventRecord(b, st);
                auto h1 = std::chrono::steady_clock::now();
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                printf("smem %6d graph of %d kernel(s) spin %5d cyc: %.2f us per launch on device (%.2f us host enqueue)\n", smem, n, spin,
                       1000.0 * ms / L, std::chrono::duration<double, std::micro>(h1 - h0).count() / L);
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(g);
              }
            }
        }
    }
    // plain stream launches for comparison
    for (int spin : {0, 10000}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int L = 4000;
        cudaEventRecord(a, st);
        for (int i = 0; i < L; ++i) k_spin<<<148, 256, 0, st>>>(spin, p);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("stream launches spin %5d: %.2f us per kernel\n", spin, 1000.0 * ms / L);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
