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

// The router_chain_kernel pattern: products in shared memory read 4 at a time
// (LDS.128), 16 columns loaded ahead.  chunk > 0: in chunks of `chunk` columns
// with a runtime trip count per chunk (the kernel's shape).
__global__ void chain_lds128(const float *x, float *out, long long *cyc, int chunk) {
    __shared__ __align__(16) float ps[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) ps[i] = x[i];
    __syncthreads();
    const float4 *pr = reinterpret_cast<const float4 *>(ps);
    const int kc = chunk > 0 ? chunk : 4096;
    float acc = 0.0f;
    long long t0 = clock64();
    for (int c = 0; c < 4096; c += kc) {
        const float4 *p = pr + c / 4;
        float4 cur[4], nxt[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = p[u];
        for (int j = 16; j < kc; j += 16) {
#pragma unroll
            for (int u = 0; u < 4; ++u) nxt[u] = p[(j >> 2) + u];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc = __fadd_rn(acc, cur[u].x);
                acc = __fadd_rn(acc, cur[u].y);
                acc = __fadd_rn(acc, cur[u].z);
                acc = __fadd_rn(acc, cur[u].w);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, cur[u].x), cur[u].y), cur[u].z), cur[u].w);
    }
    asm volatile("" : "+f"(acc));
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
        for (int chunk : {0, 256}) {
            chain_lds128<<<1, 32>>>(x, out, cyc, chunk);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("LDS.128 products + chain, chunk %d: %.2f cycles per element\n", chunk, h / 4096.0);
        }
    }
    return 0;
}
