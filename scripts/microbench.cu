// microbench.cu -- B200 latency floors that shape the fused train-step design:
// back-to-back launch cost (plain / cooperative / cluster), grid-barrier cost, cluster-barrier
// cost, DSMEM and L2 round trips.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// barrier A: the train-step kernel's current one
__device__ void bar_a(unsigned *bar)
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
            while (ld_acquire(bar + 1) == gen) {}
        }
        __threadfence();
    }
    __syncthreads();
}
// barrier B: monotonically increasing counter, release-add, relaxed polling, one acquire fence
__device__ void bar_b(unsigned *cnt, unsigned target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        while (ld_relaxed(cnt) < target) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

__global__ void k_empty(int) {}
__global__ void k_bar_a(unsigned *bar, int n) { for (int i = 0; i < n; ++i) bar_a(bar); }
__global__ void k_bar_b(unsigned *cnt, unsigned base, int n)
{
    for (int i = 0; i < n; ++i) bar_b(cnt, base + (unsigned)(i + 1) * gridDim.x);
}
__global__ void k_bar_cg(int n) { cg::grid_group g = cg::this_grid(); for (int i = 0; i < n; ++i) g.sync(); }
__global__ void k_cluster(int n, float *out)
{
    cg::cluster_group c = cg::this_cluster();
    __shared__ float s[256];
    s[threadIdx.x] = threadIdx.x;
    float acc = 0;
    for (int i = 0; i < n; ++i) {
        c.sync();
        float *peer = c.map_shared_rank(s, (c.block_rank() + 1) % c.num_blocks());
        acc += peer[threadIdx.x];
    }
    if (acc == 12345.f) out[0] = acc;
}
// L2 pointer chase (one thread): latency of dependent loads
__global__ void k_chase(const unsigned *p, int n, unsigned *out, long long *cyc)
{
    unsigned i = 0;
    long long t0 = clock64();
    for (int k = 0; k < n; ++k) i = __ldcg(p + i);
    long long t1 = clock64();
    out[0] = i;
    cyc[0] = t1 - t0;
}


// barrier C: arrivals counted by red.release; CTA 0 gathers, then releases per-CTA flags
__device__ void bar_c(unsigned *cnt, unsigned *flags, unsigned epoch)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    }
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) { while (ld_relaxed(cnt) < epoch * gridDim.x) {} asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
        __syncthreads();
        for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + 32 * i), "r"(epoch) : "memory");
    } else if (threadIdx.x == 0) {
        while (ld_relaxed(flags + 32 * blockIdx.x) < epoch) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}
__global__ void k_bar_c(unsigned *cnt, unsigned *flags, unsigned base, int n)
{
    for (int i = 0; i < n; ++i) bar_c(cnt, flags, base + i + 1);
}
// barrier D: barrier B with nanosleep backoff in the poll
__device__ void bar_d(unsigned *cnt, unsigned target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        while (ld_relaxed(cnt) < target) { __nanosleep(32); }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}
__global__ void k_bar_d(unsigned *cnt, unsigned base, int n)
{
    for (int i = 0; i < n; ++i) bar_d(cnt, base + (unsigned)(i + 1) * gridDim.x);
}

template <class F>
float time_ms(F f, int reps)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    unsigned *bar; CK(cudaMalloc(&bar, 64)); CK(cudaMemset(bar, 0, 64));
    float *out; CK(cudaMalloc(&out, 64));
    const int R = 2000;
    // 1. launch floors
    printf("empty <<<148,256>>>            : %.2f us\n", 1000 * time_ms([&] { k_empty<<<sms, 256>>>(0); }, R));
    printf("empty <<<1,32>>>               : %.2f us\n", 1000 * time_ms([&] { k_empty<<<1, 32>>>(0); }, R));
    {
        int n = 0; void *args[] = {&n};
        printf("empty cooperative 148x256      : %.2f us\n", 1000 * time_ms([&] {
            cudaLaunchCooperativeKernel((void *)k_empty, sms, 256, args, 0, 0); }, R));
    }
    // 2. grid barrier cost
    for (int nb : {0, 20}) {
        int n = nb; void *args[] = {&bar, &n};
        float ms = time_ms([&] { cudaLaunchCooperativeKernel((void *)k_bar_a, sms, 256, args, 0, 0); }, 500);
        printf("coop + %2d barrier-A           : %.2f us\n", nb, 1000 * ms);
    }
    {
        unsigned *cnt; CK(cudaMalloc(&cnt, 64)); CK(cudaMemset(cnt, 0, 64));
        unsigned base = 0;
        int n = 20;
        void *args[] = {&cnt, &base, &n};
        float ms = time_ms([&] {
            cudaLaunchCooperativeKernel((void *)k_bar_b, sms, 256, args, 0, 0);
            base += 20u * sms; }, 500);
        printf("coop + 20 barrier-B (red/relax): %.2f us\n", 1000 * ms);
    }
    for (int nb : {0, 20}) {
        int n = nb; void *args[] = {&n};
        float ms = time_ms([&] { cudaLaunchCooperativeKernel((void *)k_bar_cg, sms, 256, args, 0, 0); }, 500);
        printf("coop + %2d cg grid.sync         : %.2f us\n", nb, 1000 * ms);
    }

    {
        unsigned *cnt, *flags; CK(cudaMalloc(&cnt, 64)); CK(cudaMemset(cnt, 0, 64));
        CK(cudaMalloc(&flags, 4 * 32 * 256)); CK(cudaMemset(flags, 0, 4 * 32 * 256));
        unsigned base = 0; int n = 20;
        void *args[] = {&cnt, &flags, &base, &n};
        float ms = time_ms([&] { cudaLaunchCooperativeKernel((void *)k_bar_c, sms, 256, args, 0, 0); base += 20; }, 500);
        printf("coop + 20 barrier-C (flags)    : %.2f us\n", 1000 * ms);
        unsigned *cnt2; CK(cudaMalloc(&cnt2, 64)); CK(cudaMemset(cnt2, 0, 64));
        unsigned base2 = 0;
        void *args2[] = {&cnt2, &base2, &n};
        ms = time_ms([&] { cudaLaunchCooperativeKernel((void *)k_bar_d, sms, 256, args2, 0, 0); base2 += 20u * sms; }, 500);
        printf("coop + 20 barrier-D (nanosleep): %.2f us\n", 1000 * ms);
        ms = time_ms([&] { cudaLaunchCooperativeKernel((void *)k_bar_d, 64, 256, args2, 0, 0); base2 += 20u * 64; }, 500);
        printf("coop64 + 20 barrier-D          : %.2f us (wrong base ok)\n", 1000 * ms);
    }
    // graphs of sequential kernels
    {
        cudaStream_t st; CK(cudaStreamCreate(&st));
        for (int coop = 0; coop < 2; ++coop) {
            cudaGraph_t g; cudaGraphExec_t ge;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
            for (int i = 0; i < 100; ++i) {
                if (coop) { int n = 0; void *args[] = {&n}; cudaLaunchCooperativeKernel((void *)k_empty, sms, 256, args, 0, st); }
                else k_empty<<<sms, 256, 0, st>>>(0);
            }
            CK(cudaStreamEndCapture(st, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
            cudaEventRecord(a, st);
            for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, st);
            cudaEventRecord(b, st); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("graph of 100 sequential empty %s kernels: %.2f us per kernel\n", coop ? "coop" : "plain", 1000 * ms / 2000);
        }
        // PDL launches back to back
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(sms); cfg.blockDim = dim3(256); cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
        float ms = time_ms([&] { cudaLaunchKernelEx(&cfg, k_empty, 0); }, R);
        printf("PDL empty 148x256 back-to-back : %.2f us\n", 1000 * ms);
    }
    // 3. clusters
    for (int cs : {2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs == 16 ? 128 : (sms / cs) * cs);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        if (cs == 16) CK(cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        int ncl = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)k_cluster, &cfg);
        printf("cluster %2d: max active clusters %d (%s)\n", cs, ncl, cudaGetErrorString(e));
        for (int nb : {0, 50}) {
            float ms = time_ms([&] { cudaLaunchKernelEx(&cfg, k_cluster, nb, out); }, 500);
            printf("  cluster %2d grid %d + %2d cluster.sync+DSMEM: %.2f us\n", cs, cfg.gridDim.x, nb, 1000 * ms);
        }
        CK(cudaGetLastError());
    }
    // 4. L2 / DRAM dependent-load latency
    {
        const int N = 1 << 24;
        unsigned *h = new unsigned[N], *d;
        for (int i = 0; i < N; ++i) h[i] = (unsigned)(((long long)i * 7919 + 4099) % N);
        CK(cudaMalloc(&d, N * 4)); CK(cudaMemcpy(d, h, N * 4, cudaMemcpyHostToDevice));
        unsigned *o; long long *c, hc;
        CK(cudaMalloc(&o, 8)); CK(cudaMalloc(&c, 8));
        k_chase<<<1, 1>>>(d, 10000, o, c); CK(cudaDeviceSynchronize());
        k_chase<<<1, 1>>>(d, 10000, o, c); CK(cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost));
        printf("dependent __ldcg chase over 64 MB (L2-resident after warm): %.0f cycles/load\n", hc / 10000.0);
        // small footprint: 4 KB
        for (int i = 0; i < 1024; ++i) h[i] = (i * 17 + 5) % 1024;
        CK(cudaMemcpy(d, h, 4096, cudaMemcpyHostToDevice));
        k_chase<<<1, 1>>>(d, 10000, o, c); CK(cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost));
        printf("dependent __ldcg chase over 4 KB: %.0f cycles/load\n", hc / 10000.0);
    }
    CK(cudaDeviceSynchronize());
    printf("done\n");
    return 0;
}
