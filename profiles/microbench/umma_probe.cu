// Microbenchmark: tcgen05.mma kind::i8 issue/complete throughput on one SM
// for the shapes the LUT GEMM uses (M=128, K=32, N=16..256), A from TMEM vs
// A from shared memory, one accumulator vs R rotating accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__global__ void probe(int n, int iters, int rot, int a_smem, int conv, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    // B: n rows x 32 k at smem+32K ; A (smem mode): 128 rows x 32 k at smem 0
    const uint64_t bdesc = sdesc(sa(smem + 32768), 128, 256);
    const uint64_t adesc = sdesc(sa(smem), 128, 256);
    if (conv && threadIdx.x < 32) {
        // whole warp converged; one lane elected inside the asm; 4 accumulators
        // addressed by constants, unrolled x4 (no per-MMA address arithmetic)
        long long t0 = clock64();
        const uint32_t a0 = tmem + 448;
        for (int i = 0; i < iters; i += 4) {
            const uint32_t acc = i >= 4 ? 1u : 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t d = tmem + (uint32_t)(u * (rot > 1 ? n : 0));
                asm volatile("{\n\t.reg .pred p, e;\n\t"
                             "elect.sync _|e, 0xffffffff;\n\t"
                             "setp.ne.b32 p, %4, 0;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5,%5,%5,%5}, p;\n\t}" ::"r"(d),
                             "r"(a0 + u * 8), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u));
            }
        }
        long long t1 = clock64();
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(sa(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n}" ::"r"(
            sa(&bar)));
        long long t2 = clock64();
        if (threadIdx.x == 0) {
            cycles[blockIdx.x * 2] = t1 - t0;
            cycles[blockIdx.x * 2 + 1] = t2 - t0;
        }
    }
    if (!conv && threadIdx.x == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tmem + (uint32_t)((i % rot) * n);
            const uint32_t acc = i >= rot ? 1u : 0u;
            if (a_smem) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
            } else {
                const uint32_t a = tmem + 448 + (uint32_t)((i & 1) * 8);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5,%5,%5,%5}, p;\n\t}" ::"r"(d),
                             "r"(a), "l"(bdesc), "r"(idesc), "r"(acc), "r"(0u));
            }
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            sa(&bar)));
        long long t2 = clock64();
        cycles[blockIdx.x * 2] = t1 - t0;
        cycles[blockIdx.x * 2 + 1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long *d, h[2 * 148];
    cudaMalloc(&d, sizeof(h));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 4096;
    printf("mode n rot : issue_cyc/mma total_cyc/mma  (1 CTA/SM, 148 CTAs; MACs/clk/SM)\n");
    for (int mode = 2; mode < 3; ++mode)
        for (int n : {16, 32, 64, 128, 256})
            for (int rot : {1, 4}) {
                if (rot * n > 448 || (rot == 4 && n > 64)) continue;
                const int a_smem = mode == 1, conv = mode == 2;
                probe<<<148, 128, 64 * 1024>>>(n, iters, rot, a_smem, conv, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                double tot = 0, iss = 0;
                for (int b = 0; b < 148; ++b) {
                    iss += h[2 * b];
                    tot += h[2 * b + 1];
                }
                iss /= 148.0 * iters;
                tot /= 148.0 * iters;
                printf("%s n=%3d rot=%d : issue %6.1f  total %6.1f  cyc/mma   -> %7.0f MAC/clk/SM\n",
                       conv ? "TSconv" : (a_smem ? "SS" : "TS"), n, rot, iss, tot, 128.0 * n * 32 / tot);
            }
    return 0;
}
