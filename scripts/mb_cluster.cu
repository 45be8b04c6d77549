// How many thread-block clusters of a 1-CTA-per-SM kernel (161 KB dynamic smem, 256 threads)
// can be co-resident on this GPU, per cluster size -- the cluster-reduction sizing of
// wide_l0_kernel.   nvcc -gencode arch=compute_100a,code=sm_100a -o mb_cluster mb_cluster.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float *x) { extern __shared__ float s[]; if (x) x[threadIdx.x] = s[threadIdx.x]; }
int main()
{
    const int smem = 161 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int smem_kb : {161, 100}) {
        for (int cs : {1, 2, 3, 4, 6, 7, 8, 9, 12, 16}) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(cs * 64);
            lc.blockDim = dim3(256);
            lc.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &lc);
            printf("smem %3d KB cluster %2d: max active clusters %3d -> %4d CTAs (of %d SMs) %s\n", smem_kb, cs, n,
                   n * cs, sms, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
