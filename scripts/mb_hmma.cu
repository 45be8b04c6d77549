// mb_hmma.cu -- issue rate of legacy mma.sync m16n8k8 TF32 vs FFMA on this B200 (8 warps/SM)
#include <cstdio>
#include <cstdint>
__global__ void k_hmma(float *out, int iters)
{
    float c[8][4] = {};
    uint32_t a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    const long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0) / (iters * 8);
    if (s == 1234.f) out[1] = s;
}
__global__ void k_ffma(float *out, int iters)
{
    float c[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    const float a = threadIdx.x * 1e-3f, b = 0.999f;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fmaf(c[j], b, a);
    }
    const long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j];
    if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = (float)(t1 - t0) / (iters * 8);
    if (s == 1234.f) out[3] = s;
}
int main()
{
    float *o, h[4];
    cudaMalloc(&o, 64);
    for (int w : {1, 4, 8, 16}) {
        k_hmma<<<148, 32 * w>>>(o, 4096);
        k_ffma<<<148, 32 * w>>>(o, 4096);
        cudaDeviceSynchronize();
        cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        // cycles per instruction per warp; per-SM MAC/cycle = warps * (MACs per instr) / cycles
        printf("warps/SM %2d: HMMA tf32 m16n8k8 %.1f cyc/instr/warp -> %.0f MAC/cyc/SM ; FFMA %.1f cyc/instr/warp -> %.0f MAC/cyc/SM\n",
               w, h[0], w * 1024.0 / h[0], h[2], w * 32.0 / h[2]);
    }
    return 0;
}
