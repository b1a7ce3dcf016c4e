// Dependent fp32 add chain latency on B200 (the router's floor): one warp,
// a chain of 4096 __fadd_rn on values from registers / shared memory.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_reg(const float *x, float *out, long long *cyc) {
    float a = x[threadIdx.x], b = x[threadIdx.x + 32], acc = 0.0f;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < 4096; ++i) acc = __fadd_rn(acc, (i & 1) ? a : b);
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void chain_fmul_fadd_smem(const float *x, float *out, long long *cyc) {
    __shared__ float xs[4096], ws[4096];
    for (int i = threadIdx.x; i < 4096; i += 32) xs[i] = x[i], ws[i] = x[4096 + i];
    __syncwarp();
    float acc = 0.0f;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) acc = __fadd_rn(acc, __fmul_rn(xs[i], ws[i]));
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    float *x, *out;
    long long *cyc, h;
    cudaMalloc(&x, 8192 * 4);
    cudaMalloc(&out, 128);
    cudaMalloc(&cyc, 8);
    cudaMemset(x, 0, 8192 * 4);
    for (int r = 0; r < 2; ++r) {
        chain_reg<<<1, 32>>>(x, out, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("register chain: %.2f cycles per dependent FADD\n", h / 4096.0);
        chain_fmul_fadd_smem<<<1, 32>>>(x, out, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("smem x*w + chain: %.2f cycles per element\n", h / 4096.0);
    }
    return 0;
}
