// Microbenchmark: the LUT GEMM's digit-plane expansion alone (no data path, no
// MMAs) on every SM: per 128x128 chunk, 4 k-steps of 32 packed ids per row,
// P 16-entry byte tables per thread, 2 PRMT + 1 IMAD merge per 4 weights per
// plane, tcgen05.st.32x32b.x8 into TMEM, tcgen05.wait::st per chunk.  Chunks
// are dealt to warpgroups round robin (as the GEMM's chunk streams).
// Modes: 0 full, 1 no TMEM stores (results XOR-sunk), 2 one PRMT per 4
// weights (K <= 8 tables), 3 TMEM stores only (no lookups), 5 full with the
// previous k-step's stored registers kept live until the next k-step's lookups
// are done (no write-after-read wait on tcgen05.st sources)
// Caveat (found later): the ids are the same for every chunk except w.x, so the compiler hoists
// three quarters of the lookups out of the chunk loop; the absolute cycles understate the
// expansion cost ~4x (the GEMM's own ncu profile, profiles/r02/README.md, is the measurement).
// The relative effects of store scheduling and unrolling are what this probe showed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o expand_probe expand_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}
__device__ __forceinline__ uint32_t merge(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t hi16(uint32_t x) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, 65536;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ void st8(uint32_t t, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

template <int P, int MODE, int WGS>
__global__ void __launch_bounds__(WGS * 128, 1) expand(int chunks, long long *cycles, uint32_t *sink) {
    extern __shared__ __align__(1024) uint8_t smem[];  // ids: 4 k-steps x 128 rows x 16 B, tables: 128 x P x 16 B
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (8192 + 128 * P * 16) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(smem)[i] = (uint32_t)(i * 2654435761u) & (MODE == 2 ? 0x77777777u : 0xffffffffu);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const int wg = warp >> 2, quarter = warp & 3, row = quarter * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    const uint4 *tab = reinterpret_cast<const uint4 *>(smem + 8192) + row * P;
    uint4 L[P];
#pragma unroll
    for (int p = 0; p < P; ++p) L[p] = tab[p];
    uint32_t acc = 0;
    uint32_t prev[P][8];
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) prev[p][cc] = 0;
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int c = wg; c < chunks; c += WGS) {
        const uint32_t abase0 = tmem + lane_addr + 128 + (uint32_t)(wg * 96);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            uint4 w = reinterpret_cast<const uint4 *>(smem)[ks * 128 + row];
            if (MODE == 3) w.x ^= (uint32_t)c;
            const uint32_t wv[4] = {w.x ^ (uint32_t)c, w.y, w.z, w.w};
            uint32_t sel[8], xsel[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t xx = wv[q] ^ 0x88888888u;
                sel[2 * q] = wv[q];
                sel[2 * q + 1] = hi16(wv[q]);
                xsel[2 * q] = xx;
                xsel[2 * q + 1] = hi16(xx);
            }
            if (MODE == 7) {  // one k-step: all planes' lookups, then its stores
                uint32_t v[P][8];
#pragma unroll
                for (int p = 0; p < P; ++p)
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc)
                        v[p][cc] = merge(prmt(L[p].x, L[p].y, sel[cc]), prmt(L[p].z, L[p].w, xsel[cc]));
#pragma unroll
                for (int p = 0; p < P; ++p) st8(abase0 + (uint32_t)(ks * 8 * P + p * 8), v[p]);
                continue;
            }
            if (MODE == 6) {  // pairs of k-steps: both k-steps' lookups, then their stores
                if (ks & 1) continue;
                const uint4 w2 = reinterpret_cast<const uint4 *>(smem)[(ks + 1) * 128 + row];
                const uint32_t wv2[4] = {w2.x ^ (uint32_t)c, w2.y, w2.z, w2.w};
                uint32_t sel2[8], xsel2[8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t xx = wv2[q] ^ 0x88888888u;
                    sel2[2 * q] = wv2[q];
                    sel2[2 * q + 1] = hi16(wv2[q]);
                    xsel2[2 * q] = xx;
                    xsel2[2 * q + 1] = hi16(xx);
                }
                uint32_t v[2][P][8];
#pragma unroll
                for (int p = 0; p < P; ++p)
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) {
                        v[0][p][cc] = merge(prmt(L[p].x, L[p].y, sel[cc]), prmt(L[p].z, L[p].w, xsel[cc]));
                        v[1][p][cc] = merge(prmt(L[p].x, L[p].y, sel2[cc]), prmt(L[p].z, L[p].w, xsel2[cc]));
                    }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int p = 0; p < P; ++p) st8(abase0 + (uint32_t)((ks + h) * 8 * P + p * 8), v[h][p]);
                continue;
            }
            if (MODE == 5) {
                uint32_t v[P][8];
#pragma unroll
                for (int p = 0; p < P; ++p)
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc)
                        v[p][cc] = merge(prmt(L[p].x, L[p].y, sel[cc]), prmt(L[p].z, L[p].w, xsel[cc]));
                // the previous k-step's stores have had this k-step's lookups to drain their sources
#pragma unroll
                for (int p = 0; p < P; ++p)
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) asm volatile("" ::"r"(prev[p][cc]));
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    st8(abase0 + (uint32_t)(ks * 8 * P + p * 8), v[p]);
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) prev[p][cc] = v[p][cc];
                }
                continue;
            }
#pragma unroll
            for (int p = 0; p < P; ++p) {
                uint32_t v[8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    if (MODE == 2)
                        v[cc] = prmt(L[p].x, L[p].y, sel[cc]);
                    else if (MODE == 3)
                        v[cc] = sel[cc] + p;
                    else
                        v[cc] = merge(prmt(L[p].x, L[p].y, sel[cc]), prmt(L[p].z, L[p].w, xsel[cc]));
                }
                if (MODE == 1) {
#pragma unroll
                    for (int cc = 0; cc < 8; ++cc) acc ^= v[cc];
                } else {
                    st8(abase0 + (uint32_t)(ks * 8 * P + p * 8), v);
                }
            }
        }
        if (MODE != 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    const long long t1 = clock64();
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;
    __syncthreads();
    if (lane == 0) atomicMax((unsigned long long *)&cycles[blockIdx.x], (unsigned long long)(t1 - t0));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int P, int MODE, int WGS>
void run(const char *name, int chunks) {
    long long *d;
    uint32_t *sink;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&sink, 4096);
    const int smem = 8192 + 128 * P * 16;
    cudaFuncSetAttribute(expand<P, MODE, WGS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 148 * 8);
        expand<P, MODE, WGS><<<148, WGS * 128, smem>>>(chunks, d, sink);
        cudaDeviceSynchronize();
    }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long x : h) mx = x > mx ? x : mx;
    printf("%-34s P=%d warpgroups=%d: %7.1f cycles per chunk per SM (%s)\n", name, P, WGS, (double)mx / chunks,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(sink);
}

int main() {
    const int C = 400;
    run<3, 0, 4>("full (2 PRMT + IMAD, st.x8)", C);
    run<3, 1, 4>("no TMEM stores", C);
    run<3, 2, 4>("1 PRMT per 4 weights (K<=8)", C);
    run<3, 3, 4>("TMEM stores only", C);
    run<3, 0, 2>("full, 2 warpgroups", C);
    run<3, 1, 2>("no TMEM stores, 2 warpgroups", C);
    run<2, 0, 4>("full (2 PRMT + IMAD, st.x8)", C);
    run<3, 5, 4>("full, stored regs kept live 1 k-step", C);
    run<2, 5, 4>("full, stored regs kept live 1 k-step", C);
    run<3, 6, 4>("k-step pairs: lookups then stores", C);
    run<3, 7, 4>("per k-step: lookups then stores", C);
    return 0;
}
