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
constexpr int RP_MAX_LOCAL = 32;     // local experts (one ballot per expert; a 256-expert variant
                                     // with 8 masks measured slower than separate kernels at E = 128)
constexpr int RP_MAX_ROUTES = 4096;  // n * k held in shared memory

// numpy's float32 sum of a short row: a plain loop below 8 elements, eight
// interleaved partial sums combined as a tree from 8 up (pairwise_sum).
__device__ __forceinline__ float np_sum(const float *v, int n) {
    if (n < 8) {
        float r = 0.0f;  // numpy starts from the first element; 0 + x == x exactly
        for (int i = 0; i < n; ++i) r = __fadd_rn(r, v[i]);
        return r;
    }
    float r[8];
    for (int j = 0; j < 8; ++j) r[j] = v[j];
    int i = 8;
    for (; i + 8 <= n; i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], v[i + j]);
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __fadd_rn(res, v[i]);
    return res;
}

// One warp per token: the lanes hold the token's logits (expert e in lane e % 32),
// and each of the k rounds is a warp argmax (larger logit first, ties -> lower
// expert id, +0 and -0 equal like numpy's sort): the stable descending
// selection of model.py:324-330.  Lane 0 then forms the softmax over the
// selected logits and counts the routes of the local expert range.
// `row`: the token's n_exp logits, global or shared memory; weights and counts
// are nullable.
// PER: logits per lane (n_exp <= 32 PER).
template <int PER = 8>
__device__ __forceinline__ void topk_token(const float *row, int64_t t, int64_t n_exp, int64_t k, int lane,
                                           int32_t *__restrict__ selected, float *__restrict__ weights,
                                           int32_t *__restrict__ counts, int64_t local_begin, int64_t n_local) {
    float lv[PER];
    uint32_t taken = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int64_t e = lane + 32 * i;
        lv[i] = e < n_exp ? row[e] : 0.0f;
        if (e >= n_exp) taken |= 1u << i;
    }
    // round s's winner is kept by lane s (registers, no local-memory arrays)
    int my_sel = -1;
    float my_val = 0.0f;
    for (int s = 0; s < k; ++s) {
        int best = -1;
        float bv = 0.0f;
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (!(taken >> i & 1) && (best < 0 || lv[i] > bv)) {  // lane-local: ids ascending with i
                best = lane + 32 * i;
                bv = lv[i];
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int ob = __shfl_xor_sync(0xffffffffu, best, o);
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            if (ob >= 0 && (best < 0 || ov > bv || (!(bv > ov) && ob < best))) {
                best = ob;
                bv = ov;
            }
        }
        if (lane == s) {
            my_sel = best;
            my_val = bv;
        }
        if ((best & 31) == lane) taken |= 1u << (best >> 5);
    }
    // softmax over the selected logits, one lane per route; the sum is np_sum's order exactly
    const float m = __shfl_sync(0xffffffffu, my_val, 0);  // max of the selected logits
    const float ex = lane < k ? expf(__fsub_rn(my_val, m)) : 0.0f;
    float tot;
    if (k < 8) {
        tot = 0.0f;  // numpy starts from the first element; 0 + x == x exactly
        for (int i = 0; i < k; ++i) tot = __fadd_rn(tot, __shfl_sync(0xffffffffu, ex, i));
    } else {
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __shfl_sync(0xffffffffu, ex, j);
        int i = 8;
        for (; i + 8 <= k; i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], __shfl_sync(0xffffffffu, ex, i + j));
        tot = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
        for (; i < k; ++i) tot = __fadd_rn(tot, __shfl_sync(0xffffffffu, ex, i));
    }
    if (lane < k) {
        selected[t * k + lane] = my_sel;
        if (weights != nullptr) weights[t * k + lane] = __fdiv_rn(ex, tot);
        const int64_t le = my_sel - local_begin;
        if (counts != nullptr && le >= 0 && le < n_local) atomicAdd(counts + le, 1);
    }
}

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
    for (int e = tid; e < n_local; e += NT) s_cnt[e] = 0;
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
    for (int e = tid; e < n_local; e += NT) s_cnt[e] = s_off[e];  // running base per expert
    __syncthreads();
    constexpr int NG = RP_MAX_LOCAL / 32;  // expert groups of 32, one bit mask each
    for (int64_t t0 = 0; t0 < n; t0 += NT) {
        const int64_t t = t0 + tid;
        int le[MAX_TOPK], pre[MAX_TOPK];
        uint32_t mine[NG];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) mine[gi] = 0;
#pragma unroll
        for (int s = 0; s < MAX_TOPK; ++s) {
            le[s] = -1;
            pre[s] = 0;
            if (s < k && t < n) {
                const int64_t e = selected[t * k + s] - local_begin;
                if (e >= 0 && e < n_local) {
                    le[s] = (int)e;
#pragma unroll
                    for (int gi = 0; gi < NG; ++gi)  // static indices keep the masks in registers
                        if ((e >> 5) == gi) mine[gi] |= 1u << (e & 31);
                }
            }
        }
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
            if (32 * gi >= n_local) break;
            const int eb = n_local - 32 * gi < 32 ? n_local - 32 * gi : 32;
            for (int b = 0; b < eb; ++b) {
                const int e = 32 * gi + b;
                const bool has = (mine[gi] >> b) & 1u;
                const uint32_t bal = __ballot_sync(0xffffffffu, has);
                if (lane == 0) s_wtot[warp][e] = __popc(bal);
                if (has) {
#pragma unroll
                    for (int s = 0; s < MAX_TOPK; ++s)
                        if (le[s] == e) pre[s] = __popc(bal & ((1u << lane) - 1u));
                }
            }
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
        for (int e = tid; e < n_local; e += NT) {
            int32_t tot = 0;
            for (int w = 0; w < NT / 32; ++w) tot += s_wtot[w][e];
            s_cnt[e] += tot;
        }
        __syncthreads();
    }
}

}  // namespace cq
