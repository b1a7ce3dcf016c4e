// The expert-segment permutation of a routed batch, computed by one CTA in
// shared memory (permute_kernel's result; the builder-defined permutation of
// SURVEY.md §8(a) a11): routes grouped by local expert, experts ascending,
// tokens ascending inside an expert.  Used by the tcgen05 GEMM's B build at
// decode sizes, where every CTA derives it from `selected` instead of waiting
// for separate top-k / permute launches.
#pragma once

#include "common.cuh"

namespace cq {

constexpr int MAX_TOPK = 16;
constexpr int RP_MAX_LOCAL = 32;     // local experts (one ballot per expert)
constexpr int RP_MAX_ROUTES = 4096;  // n * k held in shared memory

// s_off [n_local + 1] and s_perm [n * k] are shared memory.  perm_slot / inv
// (global, nullable) are written when given (one CTA does that).  Every
// thread of the CTA (NT threads) must call this.
template <int NT>
__device__ void route_permute(const int32_t *__restrict__ selected, int64_t n, int k, int64_t local_begin,
                              int n_local, int32_t *s_off, int32_t *s_perm, int32_t *__restrict__ perm_slot,
                              int32_t *__restrict__ inv) {
    __shared__ int32_t s_cnt[RP_MAX_LOCAL];
    __shared__ int32_t s_wtot[NT / 32][RP_MAX_LOCAL];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < n_local) s_cnt[tid] = 0;
    __syncthreads();
    for (int64_t x = tid; x < n * k; x += NT) {
        const int64_t e = selected[x] - local_begin;
        if (e >= 0 && e < n_local) atomicAdd(&s_cnt[e], 1);
    }
    __syncthreads();
    if (tid == 0) {
        int32_t run = 0;
        for (int e = 0; e < n_local; ++e) {
            s_off[e] = run;
            run += s_cnt[e];
        }
        s_off[n_local] = run;
    }
    __syncthreads();
    if (tid < n_local) s_cnt[tid] = s_off[tid];  // running base per expert
    __syncthreads();
    for (int64_t t0 = 0; t0 < n; t0 += NT) {
        const int64_t t = t0 + tid;
        int le[MAX_TOPK], pre[MAX_TOPK];
        uint32_t mine = 0;
#pragma unroll
        for (int s = 0; s < MAX_TOPK; ++s) {
            le[s] = -1;
            pre[s] = 0;
            if (s < k && t < n) {
                const int64_t e = selected[t * k + s] - local_begin;
                if (e >= 0 && e < n_local) {
                    le[s] = (int)e;
                    mine |= 1u << e;
                }
            }
        }
        for (int e = 0; e < n_local; ++e) {
            const uint32_t b = __ballot_sync(0xffffffffu, (mine >> e) & 1u);
            if (lane == 0) s_wtot[warp][e] = __popc(b);
#pragma unroll
            for (int s = 0; s < MAX_TOPK; ++s)
                if (le[s] == e) pre[s] = __popc(b & ((1u << lane) - 1u));
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < MAX_TOPK; ++s) {
            if (le[s] < 0) continue;
            int32_t pos = s_cnt[le[s]] + pre[s];
            for (int w = 0; w < warp; ++w) pos += s_wtot[w][le[s]];
            s_perm[pos] = (int32_t)t;
            if (perm_slot != nullptr) perm_slot[pos] = s;
            if (inv != nullptr) inv[t * k + s] = pos;
        }
        __syncthreads();
        if (tid < n_local) {
            int32_t tot = 0;
            for (int w = 0; w < NT / 32; ++w) tot += s_wtot[w][tid];
            s_cnt[tid] += tot;
        }
        __syncthreads();
    }
}

}  // namespace cq
