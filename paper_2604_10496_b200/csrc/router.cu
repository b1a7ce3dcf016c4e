// Router (model.py:379-385), top-k (model.py:324-330) and the builder-defined
// token permutation into per-expert segments.
//
// Bit-exactness: logits reproduce the ordered fp32 chain of _core.matmul_f32
// (k ascending, no FMA) on the exact fake-quant input codes*scale
// (quant.py:8-13); top-k ids, their order, counts, offsets and the permutation
// are therefore bit-exact.  Route weights use CUDA expf (ulp-bounded vs numpy).
#include <type_traits>

#include "common.cuh"
#include "route_perm.cuh"

#include <cstdlib>

namespace cq {

// logits[t, e] = sum_k (q[t,k] * s_t) * W[k, e], k ascending, one rounding per
// multiply and per add (the chain of _core.matmul_f32).  A CTA owns TT tokens x
// E experts (one thread per chain); W and the exact fake-quant inputs q*s are
// staged in shared memory RK columns at a time so the chains read smem, not L2.
__global__ void router_logits_kernel(const int8_t *__restrict__ codes, const float *__restrict__ scales,
                                     const float *__restrict__ w, int64_t n, int64_t d, int64_t n_exp, int rk,
                                     float *__restrict__ logits) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    extern __shared__ float rsm[];
    const int tt_n = blockDim.x / (int)n_exp;
    float *ws = rsm;                 // [rk][E]
    float *as = rsm + rk * n_exp;    // [tt_n][rk]
    const int t_loc = threadIdx.x / (int)n_exp, e = threadIdx.x % (int)n_exp;
    const int64_t t0 = blockIdx.x * (int64_t)tt_n;
    const int64_t t = t0 + t_loc;
    const bool live = t_loc < tt_n && t < n;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < d; k0 += rk) {
        const int kn = (int)((d - k0) < rk ? (d - k0) : rk);
        __syncthreads();
        for (int x = threadIdx.x; x < kn * n_exp; x += blockDim.x) ws[x] = __ldg(w + k0 * n_exp + x);
        for (int x = threadIdx.x; x < tt_n * kn; x += blockDim.x) {
            const int tl = x / kn, kk = x - tl * kn;
            const int64_t tg = t0 + tl;
            as[tl * rk + kk] = tg < n ? __fmul_rn((float)codes[tg * d + k0 + kk], __ldg(scales + tg)) : 0.0f;
        }
        __syncthreads();
        if (live) {
            const float *ar = as + t_loc * rk;
#pragma unroll 8
            for (int kk = 0; kk < kn; ++kk) acc = __fadd_rn(acc, __fmul_rn(ar[kk], ws[kk * n_exp + e]));
        }
    }
    if (live) logits[t * n_exp + e] = acc;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}

// Same chains on the dequantized rows x = fl(q * s) that the quantizer writes
// alongside the codes (quant.cu), so a chain step is one FMUL (off the
// critical path) and one dependent FADD.  CTA = TT tokens x E experts <= 128
// chains = 4 warps, one per SMSP; x rows and W rows are staged RK columns at a
// time by cp.async, double-buffered.  Per element and lane: a quarter of a
// broadcast LDS.128 (x), one LDS (w), FMUL, FADD — under the 4-cycle FADD
// latency, which is the floor (d dependent adds per chain).
constexpr int RD_THREADS = 128;

// EC: n_exp as a compile-time constant (w offsets become immediates), 0 = runtime.
template <int EC>
__global__ void __launch_bounds__(RD_THREADS) router_deq_kernel(const float *__restrict__ xdeq,
                                                                const float *__restrict__ w, int64_t n, int64_t d,
                                                                int64_t n_exp, int tt, int rk,
                                                                float *__restrict__ logits) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    extern __shared__ __align__(16) float rds[];
    const int E = EC ? EC : (int)n_exp;
    float *xs = rds;                         // [2][tt][rk]
    float *ws = rds + (size_t)2 * tt * rk;   // [2][rk][E]
    const int tid = threadIdx.x;
    const int64_t t0 = blockIdx.x * (int64_t)tt;
    const int t_loc = tid / E, e = tid - t_loc * E;
    const bool chain = t_loc < tt;
    const bool live = chain && t0 + t_loc < n;
    const int n_chunks = (int)((d + rk - 1) / rk);
    auto stage = [&](int i) {
        const int b = i & 1;
        const int64_t k0 = (int64_t)i * rk;
        const int kn = (int)((d - k0) < rk ? (d - k0) : rk);
        float *wsb = ws + (size_t)b * rk * E;
        for (int x = tid; x < kn * E / 4; x += (int)blockDim.x) cp_async16(wsb + 4 * x, w + k0 * E + 4 * x);
        const int rowv = kn / 4;
        float *xsb = xs + (size_t)b * tt * rk;
        for (int x = tid; x < tt * rowv; x += (int)blockDim.x) {
            const int tl = x / rowv, v = x - tl * rowv;
            const int64_t tg = t0 + tl < n ? t0 + tl : n - 1;  // clamp: rows past n are never consumed
            cp_async16(xsb + tl * rk + 4 * v, xdeq + tg * d + k0 + 4 * v);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage(0);
    float acc = 0.0f;
    for (int i = 0; i < n_chunks; ++i) {
        const int b = i & 1;
        if (i + 1 < n_chunks) {
            stage(i + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int kn = (int)((d - (int64_t)i * rk) < rk ? (d - (int64_t)i * rk) : rk);  // multiple of 16
        if (chain) {
            const float4 *xr = reinterpret_cast<const float4 *>(xs + (size_t)b * tt * rk + t_loc * rk);
            const float *wr = ws + (size_t)b * rk * E + e;
            // register double buffer: the next 16 (x, w) pairs load while the
            // current 16 dependent adds run
            float xc[16], wc[16], xn[16], wn[16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float4 v = xr[u];
                xc[4 * u] = v.x, xc[4 * u + 1] = v.y, xc[4 * u + 2] = v.z, xc[4 * u + 3] = v.w;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) wc[u] = wr[u * E];
            for (int j = 16; j < kn; j += 16) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 v = xr[(j >> 2) + u];
                    xn[4 * u] = v.x, xn[4 * u + 1] = v.y, xn[4 * u + 2] = v.z, xn[4 * u + 3] = v.w;
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) wn[u] = wr[(j + u) * E];
#pragma unroll
                for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, __fmul_rn(xc[u], wc[u]));
#pragma unroll
                for (int u = 0; u < 16; ++u) xc[u] = xn[u], wc[u] = wn[u];
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, __fmul_rn(xc[u], wc[u]));
        }
        __syncthreads();  // buffer b is refilled by the next iteration's prefetch
    }
    if (live) logits[(t0 + t_loc) * n_exp + e] = acc;
}

// Many experts (E in {32, 64, 128}) at prefill sizes: each thread runs TI x 4
// ordered chains, TI consecutive tokens x 4 consecutive experts, so a step of
// 4 columns costs TI x-row and 4 w-row 128-bit loads (4 x 4: 8 loads for 128
// fp32 operations; one expert x 16 tokens per thread needed 20).  Each chain
// adds its products in column order (one ordered fp32 add per column), so the
// logits are bit-identical to _core.matmul_f32.
// CTA: blockDim (<= 256) threads = EC / 4 expert quads x token groups.  Every
// CTA streams all of w through shared memory, so the host sizes the token tile
// to one CTA per SM (QW: 124 us with 16-token tiles on 2 CTAs per SM, 115 us
// with 32 on 128 SMs, 28 on 147 SMs below; profiles/README.md).
// RK > 0: the chunk width at compile time (rk == RK): full chunks run with immediate load offsets
// (a runtime width cost ~13M address / loop instructions of 69M at QW, issued by ~2 warps per SMSP).
template <int EC, int TI, int RK = 0>
__global__ void __launch_bounds__(256) router_tile_kernel(const float *__restrict__ xdeq,
                                                                 const float *__restrict__ w, int64_t n, int64_t d,
                                                                 int rk, float *__restrict__ logits) {
    griddep_wait();
    if (RK > 0) rk = RK;
    constexpr int EQ = EC / 4;                 // expert quads
    const int NT = blockDim.x;
    const int TQ = NT / EQ;                    // token groups of TI
    const int TT = TI * TQ;                    // tokens per CTA
    extern __shared__ __align__(16) float rts[];
    const int xp = rk + 4;                     // x row pitch: token quads' rows on different banks
    float *xs = rts;                           // [2][TT][xp]
    float *ws = rts + (size_t)2 * TT * xp;     // [2][rk][EC]
    const int tid = threadIdx.x, eq = tid % EQ, tq = tid / EQ;
    const int64_t t0 = blockIdx.x * (int64_t)TT;
    const int n_chunks = (int)((d + rk - 1) / rk);
    auto stage = [&](int i) {
        const int b = i & 1;
        const int64_t k0 = (int64_t)i * rk;
        const int kn = (int)((d - k0) < rk ? (d - k0) : rk);
        float *wsb = ws + (size_t)b * rk * EC;
        for (int x = tid; x < kn * EC / 4; x += NT) cp_async16(wsb + 4 * x, w + k0 * EC + 4 * x);
        const int rowv = kn / 4;
        float *xsb = xs + (size_t)b * TT * xp;
        for (int x = tid; x < TT * rowv; x += NT) {
            const int tl = x / rowv, v = x - tl * rowv;
            const int64_t tg = t0 + tl < n ? t0 + tl : n - 1;  // clamp: rows past n are never stored
            cp_async16(xsb + tl * xp + 4 * v, xdeq + tg * d + k0 + 4 * v);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage(0);
    float acc[TI][4];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[i][m] = 0.0f;
    for (int c = 0; c < n_chunks; ++c) {
        const int b = c & 1;
        if (c + 1 < n_chunks) {
            stage(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int kn = (int)((d - (int64_t)c * rk) < rk ? (d - (int64_t)c * rk) : rk);  // multiple of 16
        const float *wr = ws + (size_t)b * rk * EC + 4 * eq;
        const float *xr = xs + (size_t)b * TT * xp + (size_t)(TI * tq) * xp;
        auto step4 = [&](int j) {
            float4 wv[4], xv[TI];
#pragma unroll
            for (int q = 0; q < 4; ++q) wv[q] = *reinterpret_cast<const float4 *>(wr + (j + q) * EC);
#pragma unroll
            for (int i = 0; i < TI; ++i) xv[i] = *reinterpret_cast<const float4 *>(xr + i * xp + j);
#pragma unroll
            for (int i = 0; i < TI; ++i) {
                const float xq[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float p0, p1, p2, p3;  // x broadcast against expert pairs: two FMUL2 per 4 products
                    fmul2_rn(xq[q], xq[q], wv[q].x, wv[q].y, p0, p1);
                    fmul2_rn(xq[q], xq[q], wv[q].z, wv[q].w, p2, p3);
                    acc[i][0] = __fadd_rn(acc[i][0], p0);
                    acc[i][1] = __fadd_rn(acc[i][1], p1);
                    acc[i][2] = __fadd_rn(acc[i][2], p2);
                    acc[i][3] = __fadd_rn(acc[i][3], p3);
                }
            }
        };
        if (RK > 0 && kn == RK) {
#pragma unroll 8
            for (int j = 0; j < RK; j += 4) step4(j);
        } else {
            for (int j = 0; j < kn; j += 4) step4(j);
        }
        __syncthreads();  // buffer b is refilled by the next iteration's prefetch
    }
#pragma unroll
    for (int i = 0; i < TI; ++i) {
        const int64_t t = t0 + TI * tq + i;
        if (t < n)
            *reinterpret_cast<float4 *>(logits + t * EC + 4 * eq) =
                make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
}

// A warp per token, TOPK_TPW tokens per warp; the route counts are summed in shared memory and
// added once per CTA and expert (one global atomic per route on <= 128 addresses serialised in L2:
// DS 8192 x top-6 took 38 us).
#ifndef TOPK_TPW_
#define TOPK_TPW_ 1
#endif
#ifndef TOPK_AGG_
#define TOPK_AGG_ 1
#endif
constexpr int TOPK_WARPS = 8, TOPK_TPW = TOPK_TPW_, TOPK_SMEM_E = 1024;

template <int PER>
__global__ void __launch_bounds__(TOPK_WARPS * 32) topk_kernel(const float *__restrict__ logits, int64_t n,
                                                               int64_t n_exp, int64_t k, int32_t *__restrict__ selected,
                                                               float *__restrict__ weights, int32_t *__restrict__ counts,
                                                               int64_t local_begin, int64_t n_local) {
    __shared__ int32_t s_cnt[TOPK_SMEM_E];
    const bool agg = TOPK_AGG_ && counts != nullptr && n_local <= TOPK_SMEM_E;
    if (agg)
        for (int64_t e = threadIdx.x; e < n_local; e += blockDim.x) s_cnt[e] = 0;
    __syncthreads();
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t t0 = ((int64_t)blockIdx.x * TOPK_WARPS + warp) * TOPK_TPW;
    for (int i = 0; i < TOPK_TPW; ++i) {
        const int64_t t = t0 + i;
        if (t >= n) break;  // warp-uniform
        topk_token<PER>(logits + t * n_exp, t, n_exp, k, lane, selected, weights, agg ? s_cnt : counts, local_begin,
                        n_local);
    }
    if (!agg) return;
    __syncthreads();
    for (int64_t e = threadIdx.x; e < n_local; e += blockDim.x)
        if (s_cnt[e] != 0) atomicAdd(counts + e, s_cnt[e]);
}

// CTA per local expert: a stable block scan over tokens assigns each route
// of this expert its row in the segment; CTA 0 also publishes offsets[0..E].
// (Large batches: the route counts come from the top-k.)
constexpr int PERM_THREADS = 1024;

__global__ void __launch_bounds__(PERM_THREADS) permute_kernel(
    const int32_t *__restrict__ selected, const int32_t *__restrict__ counts, int64_t n, int64_t k,
    int64_t local_begin, int64_t n_local, int32_t *__restrict__ offsets,
    int32_t *__restrict__ perm_token, int32_t *__restrict__ perm_slot, int32_t *__restrict__ inv) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int32_t s_base;
    __shared__ int32_t warp_tot[PERM_THREADS / 32];
    const int e_loc = blockIdx.x;
    const int64_t e_glob = e_loc + local_begin;
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int e = 0; e < e_loc; ++e) acc += counts[e];
        s_base = acc;
        if (e_loc == 0) {
            int32_t run = 0;
            for (int e = 0; e < n_local; ++e) {
                offsets[e] = run;
                run += counts[e];
            }
            offsets[n_local] = run;
        }
    }
    __syncthreads();
    int32_t base = s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t t0 = 0; t0 < n; t0 += PERM_THREADS) {
        const int64_t t = t0 + threadIdx.x;
        int slot = -1;
        if (t < n)
            for (int s = 0; s < k; ++s)
                if (selected[t * k + s] == e_glob) slot = s;
        const unsigned ball = __ballot_sync(0xffffffffu, slot >= 0);
        const int in_warp = __popc(ball & ((1u << lane) - 1u));
        if (lane == 0) warp_tot[warp] = __popc(ball);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < PERM_THREADS / 32; ++w) {
            const int c = warp_tot[w];
            before += (w < warp) ? c : 0;
            total += c;
        }
        if (slot >= 0) {
            const int32_t pos = base + before + in_warp;
            perm_token[pos] = (int32_t)t;
            perm_slot[pos] = slot;
            if (inv != nullptr) inv[t * k + slot] = pos;
        }
        base += total;
        __syncthreads();
    }
}

// Batches up to PERMC_MAX tokens: no route counts needed.  CTA per local expert, one pass over the
// selections: each thread takes PERMC_TPT consecutive tokens, a block scan per chunk orders this
// expert's routes (token ascending) into a shared-memory list, and the routes of lower local
// experts are counted on the way; their total is the segment start.  Then the list is written out
// (coalesced) and the CTA publishes counts[e], offsets[e] (and offsets[n_local] from the last).
// The top-k then needs no route-count atomics: one per route on <= E addresses of one L2 slice
// serialised (DS 8192 x top-6: 39 us of top-k).
constexpr int PERMC_THREADS = 1024, PERMC_TPT = 4;
constexpr int64_t PERMC_MAX = 49152;  // list entries in shared memory (192 KB)

__global__ void __launch_bounds__(PERMC_THREADS) permute_count_kernel(
    const int32_t *__restrict__ selected, int64_t n, int64_t k, int64_t local_begin, int64_t n_local,
    int32_t *__restrict__ counts, int32_t *__restrict__ offsets, int32_t *__restrict__ perm_token,
    int32_t *__restrict__ perm_slot, int32_t *__restrict__ inv) {
    extern __shared__ int32_t pc_list[];  // [n] this expert's routes: token << 4 | slot
    __shared__ int32_t warp_sum[PERMC_THREADS / 32], s_tot;
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t e_glob = blockIdx.x + local_begin;
    int32_t mine = 0;  // block-uniform: routes of this expert so far
    int below = 0;     // this thread's routes of local experts below e
    for (int64_t c0 = 0; c0 < n; c0 += (int64_t)PERMC_THREADS * PERMC_TPT) {
        const int64_t tb = c0 + (int64_t)threadIdx.x * PERMC_TPT;
        // slots of the PERMC_TPT tokens, 5 bits each (slot + 1, 0 = not this expert)
        uint32_t sp = 0;
        if (tb + PERMC_TPT <= n) {
            // the tokens' 4k selections are 16-byte aligned (tb * k * 4 = threadIdx * 16 k): k int4 loads
            const int4 *src = reinterpret_cast<const int4 *>(selected + tb * k);
            int i = 0, s = 0;
#pragma unroll 4
            for (int q = 0; q < k; ++q) {
                const int4 v4 = src[q];
                const int32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (vv[c] == e_glob) sp |= (uint32_t)(s + 1) << (5 * i);
                    below += (vv[c] >= local_begin && vv[c] < e_glob) ? 1 : 0;
                    if (++s == k) {
                        s = 0;
                        ++i;
                    }
                }
            }
        } else {
            for (int i = 0; i < PERMC_TPT; ++i) {
                const int64_t t = tb + i;
                if (t >= n) break;
                for (int s = 0; s < k; ++s) {
                    const int32_t v = selected[t * k + s];
                    if (v == e_glob) sp |= (uint32_t)(s + 1) << (5 * i);
                    below += (v >= local_begin && v < e_glob) ? 1 : 0;
                }
            }
        }
        int8_t slot[PERMC_TPT];
        int m = 0;
#pragma unroll
        for (int i = 0; i < PERMC_TPT; ++i) {
            slot[i] = (int8_t)((int)((sp >> (5 * i)) & 31u) - 1);
            m += slot[i] >= 0;
        }
        int incl = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const int wv = warp_sum[lane];
            int wi = wv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            warp_sum[lane] = wi - wv;  // exclusive warp prefix
            if (lane == 31) s_tot = wi;
        }
        __syncthreads();
        int pos = mine + warp_sum[warp] + incl - m;
#pragma unroll
        for (int i = 0; i < PERMC_TPT; ++i)
            if (slot[i] >= 0) pc_list[pos++] = (int32_t)((tb + i) << 4) | slot[i];
        mine += s_tot;
        __syncthreads();  // warp_sum / s_tot are rewritten by the next chunk
    }
    // segment start: the routes of the lower local experts
    below = __reduce_add_sync(0xffffffffu, below);
    if (lane == 0) warp_sum[warp] = below;
    __syncthreads();
    if (warp == 0) {
        const int b = __reduce_add_sync(0xffffffffu, warp_sum[lane]);
        if (lane == 0) s_tot = b;
    }
    __syncthreads();
    const int32_t base = s_tot;
    for (int32_t i = threadIdx.x; i < mine; i += PERMC_THREADS) {
        const int32_t ent = pc_list[i];
        const int64_t t = ent >> 4;
        const int sl = ent & 15;
        const int32_t p = base + i;
        perm_token[p] = (int32_t)t;
        perm_slot[p] = sl;
        if (inv != nullptr) inv[t * k + sl] = p;
    }
    if (threadIdx.x == 0) {
        counts[blockIdx.x] = mine;
        offsets[blockIdx.x] = base;
        if (blockIdx.x == n_local - 1) offsets[n_local] = base + mine;
    }
}

bool permute_counts_itself(int64_t n) { return n <= PERMC_MAX; }

// What the decode router's fused tail writes: the top-k of its tokens.
struct RouteFuse {
    int32_t *selected;
    float *weights;
    int64_t k;
    // quantizer in the router (qx != nullptr): the CTA quantizes its own tokens first
    // (quantize_a4_vec_kernel's arithmetic) and keeps the dequantized rows in shared memory
    const void *qx = nullptr;
    int qdt = 0;
    int8_t *codes = nullptr;
    float *scales = nullptr;
    int *nonfinite = nullptr;
    int32_t *tsum = nullptr;
    int32_t *zero = nullptr;
    int n_zero = 0;
};

// Decode batches: each chain (token, expert) is d dependent fp32 adds, and with
// one token per CTA the chain warp of router_deq_kernel issues ~5 instructions
// per column (loads, FMUL, FADD), above the 4-cycle FADD latency.  Here warp 0
// holds only the chains (lane c = token c / EG, expert e0 + c % EG) and adds
// precomputed products with one LDS.128 per 4 columns.  Warps 1-3 stage raw
// W / x chunks by cp.async (NR buffers) and write the rounded products
// fmul(x[t][j], w[j][e]) of the next chunk into the other product buffer.
// Summation order and rounding are those of router_deq_kernel (bit-exact).
constexpr int RC_THREADS = 128, RC_K = 256;
// raw stages: W leaves L2 under the expert weight stream, so chunks come from
// DRAM; prefetch NR - 1 chunks (~0.55 us of chain each) ahead
// BIG (the fused decode router of 8 experts): 512-column chunks, half the chunk handoffs (MX router
// 22.9 -> 21.1 us, step 314.5 -> 312.4 us; 128 columns: 26.2 us)
template <int EG, bool BIG = false>
struct RcStages {
    static constexpr int NR = EG >= 32 ? 4 : (BIG ? 4 : 8);
    // 32-expert groups (E = 64 / 128 at decode): 128-column chunks keep a CTA near 100 KB, two per SM
    static constexpr int K = EG >= 32 ? 128 : (BIG ? 2 * RC_K : RC_K);
    static constexpr int PITCH = K + 4;
};
template <int EG, bool FUSE>
constexpr bool rc_big() { return FUSE && EG == 8; }

// acc + p[0] + p[1] + ... + p[kn-1] in order (kn % 16 == 0), 16 columns loaded
// ahead of the adds; KC > 0 fixes kn = KC at compile time.
template <int KC>
__device__ __forceinline__ float chain_add(float acc, const float4 *__restrict__ pr, int kn) {
    if (KC > 0) kn = KC;
    float4 cur[4], nxt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) cur[u] = pr[u];
#pragma unroll 3
    for (int j = 16; j < kn; j += 16) {
#pragma unroll
        for (int u = 0; u < 4; ++u) nxt[u] = pr[(j >> 2) + u];
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
    for (int u = 0; u < 4; ++u) {
        acc = __fadd_rn(acc, cur[u].x);
        acc = __fadd_rn(acc, cur[u].y);
        acc = __fadd_rn(acc, cur[u].z);
        acc = __fadd_rn(acc, cur[u].w);
    }
    return acc;
}

// FUSE (one expert group, n_exp == EG): the CTA also selects its tokens'
// top-k from the logits in shared memory (topk_kernel without its launch; the
// permutation is derived by the consumer, route_perm.cuh).
// The CTA's tt token rows quantized as quantize_a4_vec_kernel does them (same max, scale, codes,
// sums and code * scale products, bit for bit), the dequantized rows left in xs [tt][d].
__device__ void rc_quantize(const RouteFuse &f, int64_t t0, int tt, int64_t n, int64_t d, float *xs) {
    __shared__ float red_f[RC_THREADS / 32];
    __shared__ int red_i[RC_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool pub = blockIdx.y == 0;  // expert groups > 0 recompute the same rows
    const int nv = (int)(d >> 2);
    if (pub && blockIdx.x == 0)
        for (int i = tid; i < f.n_zero; i += RC_THREADS) f.zero[i] = 0;
    for (int tl = 0; tl < tt; ++tl) {
        const int64_t tg = t0 + tl < n ? t0 + tl : n - 1;  // rows past n are never stored
        float4 *xr = reinterpret_cast<float4 *>(xs + (size_t)tl * d);
        float mx = 0.0f;
        bool bad = false;
        for (int j = tid; j < nv; j += RC_THREADS) {  // (8 loads batched per thread: spills, slower)
            float h[4];
            if (f.qdt == CQ_DTYPE_F32) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(f.qx) + tg * nv + j);
                h[0] = v.x, h[1] = v.y, h[2] = v.z, h[3] = v.w;
            } else {
                const uint2 v = __ldg(reinterpret_cast<const uint2 *>(f.qx) + tg * nv + j);
                h[0] = __uint_as_float(v.x << 16), h[1] = __uint_as_float(v.x & 0xFFFF0000u);
                h[2] = __uint_as_float(v.y << 16), h[3] = __uint_as_float(v.y & 0xFFFF0000u);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bad |= !isfinite(h[q]);
                mx = fmaxf(mx, fabsf(h[q]));
            }
            xr[j] = make_float4(h[0], h[1], h[2], h[3]);
        }
        mx = warp_max(mx);
        if (lane == 0) red_f[warp] = mx;
        if (__syncthreads_or(bad) && tid == 0 && pub && f.nonfinite != nullptr) atomicExch(f.nonfinite, 1);
        float m = red_f[0];
#pragma unroll
        for (int w = 1; w < RC_THREADS / 32; ++w) m = fmaxf(m, red_f[w]);
        const float sc = a4_scale(m);
        const float rs = __frcp_rn(sc);
        int csum = 0;
        const bool live = pub && t0 + tl < n;
        for (int j = tid; j < nv; j += RC_THREADS) {
            const float4 h = xr[j];
            const char4 c = make_char4(a4_code_rcp(h.x, sc, rs), a4_code_rcp(h.y, sc, rs), a4_code_rcp(h.z, sc, rs),
                                       a4_code_rcp(h.w, sc, rs));
            if (live) reinterpret_cast<char4 *>(f.codes + tg * d)[j] = c;
            csum += c.x + c.y + c.z + c.w;
            xr[j] = make_float4(__fmul_rn((float)c.x, sc), __fmul_rn((float)c.y, sc), __fmul_rn((float)c.z, sc),
                                __fmul_rn((float)c.w, sc));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
        if (lane == 0) red_i[warp] = csum;
        __syncthreads();
        if (tid == 0 && live) {
            int t = 0;
            for (int w = 0; w < RC_THREADS / 32; ++w) t += red_i[w];
            if (f.tsum != nullptr) f.tsum[tg] = t;
            f.scales[tg] = sc;
        }
        __syncthreads();  // red_f / red_i are reused by the next row
    }
}

// QIN (with FUSE): the quantizer runs in the router launch (rc_quantize); x comes from shared
// memory instead of the xdeq ring, and `xdeq` is unused.
template <int EG, bool FUSE, bool QIN = false>
__global__ void __launch_bounds__(RC_THREADS) router_chain_kernel(const float *__restrict__ xdeq,
                                                                  const float *__restrict__ w, int64_t n,
                                                                  int64_t d, int64_t n_exp, int tt,
                                                                  float *__restrict__ logits, RouteFuse f) {
    griddep_wait();
    extern __shared__ __align__(16) float rcs[];
    const int nc = tt * EG;                      // chains
    float *pbuf = rcs;                           // [2][nc][PITCH] products
    using RS = RcStages<EG, rc_big<EG, FUSE>()>;
    constexpr int NR = RS::NR;
    constexpr int KC = RS::K, PITCH = RS::PITCH;
    float *wraw = pbuf + 2 * nc * PITCH;      // [NR][KC][EG]
    float *xraw = wraw + NR * KC * EG;         // [NR][tt][KC]; QIN: [tt][d]
    const int tid = threadIdx.x;
    const int64_t t0 = blockIdx.x * (int64_t)tt;
    const int e0 = blockIdx.y * EG;
    const int n_chunks = (int)((d + KC - 1) / KC);
    const int ptid = tid - 32;  // producer index, warps 1-3
    auto stage = [&](int i) {
        if (i < n_chunks) {
            const int64_t k0 = (int64_t)i * KC;
            const int kn = (int)((d - k0) < KC ? (d - k0) : KC);
            float *wb = wraw + (i % NR) * KC * EG;
            for (int x = ptid; x < kn * (EG / 4); x += RC_THREADS - 32) {
                const int r = x / (EG / 4), q = x - r * (EG / 4);
                cp_async16(wb + r * EG + 4 * q, w + (k0 + r) * n_exp + e0 + 4 * q);
            }
            float *xb = xraw + (i % NR) * tt * KC;
            const int rowv = QIN ? 0 : kn / 4;
            for (int x = ptid; x < tt * rowv; x += RC_THREADS - 32) {
                const int tl = x / rowv, v = x - tl * rowv;
                const int64_t tg = t0 + tl < n ? t0 + tl : n - 1;  // rows past n are never stored
                cp_async16(xb + tl * KC + 4 * v, xdeq + tg * d + k0 + 4 * v);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto produce = [&](int i) {  // chunk i landed in raw buffer i % NR (own copies waited for)
        asm volatile("bar.sync 1, %0;" ::"n"(RC_THREADS - 32) : "memory");
        const int64_t k0 = (int64_t)i * KC;
        const int kn = (int)((d - k0) < KC ? (d - k0) : KC);
        const float *wb = wraw + (i % NR) * KC * EG;
        const float *xb = QIN ? xraw + k0 : xraw + (i % NR) * tt * KC;
        const int64_t xs = QIN ? d : KC;  // x row pitch
        float *pb = pbuf + (i & 1) * nc * PITCH;
        for (int j = ptid; j < kn; j += RC_THREADS - 32) {
            float wr[EG];
#pragma unroll
            for (int q = 0; q < EG / 4; ++q) {
                const float4 v = *reinterpret_cast<const float4 *>(wb + j * EG + 4 * q);
                wr[4 * q] = v.x, wr[4 * q + 1] = v.y, wr[4 * q + 2] = v.z, wr[4 * q + 3] = v.w;
            }
            for (int t = 0; t < tt; ++t) {
                const float xv = xb[t * xs + j];
#pragma unroll
                for (int e = 0; e < EG; e += 2) {
                    float p0, p1;
                    fmul2_rn(xv, xv, wr[e], wr[e + 1], p0, p1);
                    pb[(t * EG + e) * PITCH + j] = p0;
                    pb[(t * EG + e + 1) * PITCH + j] = p1;
                }
            }
        }
    };
    if (tid >= 32) {
#pragma unroll
        for (int i = 0; i < NR - 1; ++i) stage(i);
    }
    if constexpr (QIN) rc_quantize(f, t0, tt, n, d, xraw);  // the W chunks land meanwhile
    if (tid >= 32) {
        asm volatile("cp.async.wait_group %0;" ::"n"(NR - 2) : "memory");
        produce(0);
    }
    __syncthreads();
    const bool chain = tid < nc;
    float acc = 0.0f;
    for (int i = 0; i < n_chunks; ++i) {
        if (tid >= 32) {
            if (i + 1 < n_chunks) {
                stage(i + NR - 1);  // into the buffer produce(i - 1) read
                asm volatile("cp.async.wait_group %0;" ::"n"(NR - 2) : "memory");
                produce(i + 1);
            }
        } else if (chain) {
            const int kn = (int)((d - (int64_t)i * KC) < KC ? (d - (int64_t)i * KC) : KC);  // % 16 == 0
            const float4 *pr = reinterpret_cast<const float4 *>(pbuf + (i & 1) * nc * PITCH + tid * PITCH);
            if (kn == KC)
                acc = chain_add<KC>(acc, pr, KC);  // full chunk: compile-time trip count
            else
                acc = chain_add<0>(acc, pr, kn);
        }
        __syncthreads();  // product buffer i & 1 is rewritten by iteration i + 1's producers
    }
    if (chain && t0 + tid / EG < n) logits[(t0 + tid / EG) * n_exp + e0 + tid % EG] = acc;
    if constexpr (FUSE) {
        __shared__ float lg[32];  // [tt][EG]
        if (chain) lg[tid] = acc;
        __syncthreads();
        const int warp = tid >> 5;
        if (warp < tt && t0 + warp < n)
            topk_token(lg + warp * EG, t0 + warp, EG, f.k, tid & 31, f.selected, f.weights, nullptr, 0, 0);
    }
}

static size_t router_chain_smem(int eg, int tt, int64_t qin_d = 0, bool fuse = false) {
    const bool big = fuse && eg == 8;
    const size_t nr = eg >= 32 ? RcStages<32>::NR : big ? RcStages<8, true>::NR : RcStages<8>::NR;
    const size_t kc = eg >= 32 ? RcStages<32>::K : big ? RcStages<8, true>::K : RcStages<8>::K;
    const size_t xf = qin_d > 0 ? (size_t)tt * qin_d : nr * tt * kc;  // QIN: the whole dequantized rows
    return sizeof(float) * ((size_t)2 * tt * eg * (kc + 4) + nr * kc * eg + xf);
}
constexpr size_t RC_FUSE_SMEM_MAX = 200 * 1024;  // the fused variants' smem opt-in

// rows_out[r, :] = rows_in[perm_token[r], :], r < offsets[n_local]; also scales.
__global__ void gather_rows_kernel(const int8_t *__restrict__ src, const float *__restrict__ sscale,
                                   const int32_t *__restrict__ perm_token,
                                   const int32_t *__restrict__ offsets, int64_t n_local, int64_t d,
                                   int8_t *__restrict__ dst, float *__restrict__ dscale) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t r = blockIdx.x;
    if (r >= offsets[n_local]) return;
    const int64_t t = perm_token[r];
    if (threadIdx.x == 0) dscale[r] = sscale[t];
    const int8_t *s = src + t * d;
    int8_t *o = dst + r * d;
    if ((d & 15) == 0) {
        for (int64_t j = threadIdx.x * 16; j < d; j += blockDim.x * 16)
            *reinterpret_cast<uint4 *>(o + j) = *reinterpret_cast<const uint4 *>(s + j);
    } else {
        for (int64_t j = threadIdx.x; j < d; j += blockDim.x) o[j] = s[j];
    }
}

template <bool FUSE, bool QIN = false>
static void launch_chain(int eg, dim3 grid, size_t smem, cudaStream_t st, const float *xdeq, const float *w,
                         int64_t n, int64_t d, int64_t n_exp, int tt, float *logits, const RouteFuse &f) {
    static std::atomic<uint64_t> attr{0};  // devices whose smem opt-in is set
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(router_chain_kernel<8, FUSE, QIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FUSE ? (int)RC_FUSE_SMEM_MAX : (int)router_chain_smem(8, 4));
        cudaFuncSetAttribute(router_chain_kernel<16, FUSE, QIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FUSE ? (int)RC_FUSE_SMEM_MAX : (int)router_chain_smem(16, 2));
        cudaFuncSetAttribute(router_chain_kernel<32, FUSE, QIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FUSE ? (int)RC_FUSE_SMEM_MAX : (int)router_chain_smem(32, 1));
    }
    if (eg == 32)
        launch_pdl(router_chain_kernel<32, FUSE, QIN>, grid, RC_THREADS, smem, st, xdeq, w, n, d, n_exp, tt, logits,
                   f);
    else if (eg == 16)
        launch_pdl(router_chain_kernel<16, FUSE, QIN>, grid, RC_THREADS, smem, st, xdeq, w, n, d, n_exp, tt, logits,
                   f);
    else
        launch_pdl(router_chain_kernel<8, FUSE, QIN>, grid, RC_THREADS, smem, st, xdeq, w, n, d, n_exp, tt, logits,
                   f);
}

// Decode router, one chain per thread (v2).  A CTA holds tt tokens x EGc experts (thread t:
// token t / EGc, expert e0 + t % EGc; tt sized so the grid is about one CTA per SM).  W chunks
// [RV_K][EGc] and x chunks [tt][RV_K] are staged by cp.async through an RV_NR-deep ring (W leaves
// L2 under the expert weight stream, so chunks come from DRAM: several are kept in flight); every
// thread then walks its chain through the chunk: per 4 columns one LDS.128 of x (shared by the EGc
// lanes of a token), 4 LDS.32 of W (consecutive experts, conflict-free), 4 FMUL and the 4 dependent
// FADDs — the FADD latency is the critical path, and no product buffer is written or synchronised.
// Summation order and rounding as router_deq_kernel (bit-exact): acc = ((0 + x0 w0) + x1 w1) + ...
constexpr int RV_K = 256;
#ifndef RV_NR16
#define RV_NR16 4
#endif
// ring depth: 3 stages of 36 KB for 32-expert CTAs, RV_NR16 of 25 KB for 16 (two CTAs per SM either way)
__host__ __device__ constexpr int rv_nr(int egc) { return egc >= 32 ? 3 : RV_NR16; }
// acc + x[0] w[0] + x[1] w[1] + ... over kn columns (kn % 4 == 0; KN > 0 fixes it at compile time):
// w column j at wb[j * WP], x as float4s.
template <int WP, int KN>
__device__ __forceinline__ float chain2_steps(float acc, const float *__restrict__ wb, const float4 *__restrict__ xr,
                                              int kn) {
    // 16 columns per step, pipelined in two stages: a step's 16 products are formed while the previous
    // step's 16 adds run, from operands loaded before them, so neither the shared-memory latency nor the
    // multiply sits on the add chain (loads and products right before their adds: ~8-13 cycles per
    // column against the adds' 4.2)
    if (KN > 0) kn = KN;
    float p[16];
    auto products = [&](int j) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float4 xv = xr[(j >> 2) + u];
            fmul2_rn(xv.x, xv.y, wb[(j + 4 * u) * WP], wb[(j + 4 * u + 1) * WP], p[4 * u], p[4 * u + 1]);
            fmul2_rn(xv.z, xv.w, wb[(j + 4 * u + 2) * WP], wb[(j + 4 * u + 3) * WP], p[4 * u + 2], p[4 * u + 3]);
        }
    };
    products(0);
#pragma unroll 4
    for (int j = 16; j < kn; j += 16) {
        float q[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) q[c] = p[c];
        products(j);  // independent of the adds below: issued alongside them
#pragma unroll
        for (int c = 0; c < 16; ++c) acc = __fadd_rn(acc, q[c]);
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) acc = __fadd_rn(acc, p[c]);
    return acc;
}
template <int EGc, bool FUSE>
__global__ void __launch_bounds__(128) router_chain2_kernel(const float *__restrict__ xdeq,
                                                            const float *__restrict__ w, int64_t n, int64_t d,
                                                            int64_t n_exp, int tt, float *__restrict__ logits,
                                                            RouteFuse f) {
    griddep_wait();
    constexpr int RVN = rv_nr(EGc);
    constexpr int WP = EGc, XP = RV_K + 4;  // pitches (floats)
    extern __shared__ __align__(16) float rvs[];
    const int stage_f = RV_K * WP + tt * XP;  // floats per ring stage: W [RV_K][WP] then x [tt][XP]
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int tl = tid / EGc, el = tid % EGc;
    const bool chain = tl < tt;
    const int64_t t0 = blockIdx.x * (int64_t)tt;
    const int64_t e0 = blockIdx.y * (int64_t)EGc;
    const int n_chunks = (int)((d + RV_K - 1) / RV_K);
    // full chunks with 64 or 128 threads: each thread's copies at fixed row / quad offsets from
    // pointers set up once (the generic loop's 64-bit address arithmetic per 16-byte copy was the
    // kernel's hottest code: ~20 instructions per copy)
    constexpr int QW = EGc / 4;
    const float *wsrc = w + (int64_t)(tid / QW) * n_exp + e0 + 4 * (tid % QW);
    const int xv = tid & 63, xt = tid >> 6;
    auto stage_full = [&](int i, auto nth_c) {
        constexpr int NTH = decltype(nth_c)::value, WRP = NTH / QW, WPASS = RV_K / WRP;
        const int64_t k0 = (int64_t)i * RV_K;
        float *wb = rvs + (i % RVN) * stage_f + (tid / QW) * WP + 4 * (tid % QW);
        const float *ws = wsrc + k0 * n_exp;
#pragma unroll
        for (int m = 0; m < WPASS; ++m) cp_async16(wb + m * WRP * WP, ws + (int64_t)m * WRP * n_exp);
        float *xb = rvs + (i % RVN) * stage_f + RV_K * WP;
        for (int t = xt; t < tt; t += NTH / 64) {  // a token's 64 float4s per 64 threads
            const int64_t tg = t0 + t < n ? t0 + t : n - 1;  // rows past n are never stored
            cp_async16(xb + t * XP + 4 * xv, xdeq + tg * d + k0 + 4 * xv);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto stage = [&](int i) {
#ifdef RV_NO_STAGE  // bounding experiment: chains over whatever the ring holds
        if (i >= RVN - 1) {
            asm volatile("cp.async.commit_group;" ::: "memory");
            return;
        }
#endif
        if (i < n_chunks && (int64_t)(i + 1) * RV_K <= d) {
            if (nthr == 128) {
                stage_full(i, std::integral_constant<int, 128>{});
                return;
            }
            if (nthr == 64) {
                stage_full(i, std::integral_constant<int, 64>{});
                return;
            }
        }
        if (i < n_chunks) {
            const int64_t k0 = (int64_t)i * RV_K;
            const int kn = (int)((d - k0) < RV_K ? (d - k0) : RV_K);
            float *wb = rvs + (i % RVN) * stage_f;
            for (int x = tid; x < kn * (EGc / 4); x += nthr) {
                const int r = x / (EGc / 4), q = x - r * (EGc / 4);
                cp_async16(wb + r * WP + 4 * q, w + (k0 + r) * n_exp + e0 + 4 * q);
            }
            float *xb = wb + RV_K * WP;
            for (int x = tid; x < tt * (kn / 4); x += nthr) {
                const int t = x / (kn / 4), v = x - t * (kn / 4);
                const int64_t tg = t0 + t < n ? t0 + t : n - 1;  // rows past n are never stored
                cp_async16(xb + t * XP + 4 * v, xdeq + tg * d + k0 + 4 * v);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int i = 0; i < RVN - 1; ++i) stage(i);
    float acc = 0.0f;
    for (int i = 0; i < n_chunks; ++i) {
        asm volatile("cp.async.wait_group %0;" ::"n"(RVN - 2) : "memory");
        __syncthreads();  // chunk i landed for every thread; chunk i - 1's stage is free
        stage(i + RVN - 1);
        if (chain) {
            const int kn = (int)((d - (int64_t)i * RV_K) < RV_K ? (d - (int64_t)i * RV_K) : RV_K);  // % 16 == 0
            const float *wb = rvs + (i % RVN) * stage_f + el;
            const float4 *xr = reinterpret_cast<const float4 *>(rvs + (i % RVN) * stage_f + RV_K * WP + tl * XP);
            // full chunks with a compile-time trip count: the loads take immediate offsets (a runtime
            // count cost ~7 instructions per column in address arithmetic and loop control, which one
            // warp per SMSP issues at ~2.5 cycles each: 17 cycles per column against the 4.2 of the adds)
            if (kn == RV_K)
                acc = chain2_steps<WP, RV_K>(acc, wb, xr, kn);
            else
                acc = chain2_steps<WP, 0>(acc, wb, xr, kn);
        }
    }
    if (chain && t0 + tl < n) logits[(t0 + tl) * n_exp + e0 + el] = acc;
    if constexpr (FUSE) {  // one expert group: the CTA's tokens' top-k from its logits
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        float *lg = rvs;   // [tt][EGc] (the ring is idle now)
        if (chain) lg[tl * EGc + el] = acc;
        __syncthreads();
        const int warp = tid >> 5;
        for (int t = warp; t < tt; t += nthr / 32)
            if (t0 + t < n)
                topk_token(lg + t * EGc, t0 + t, EGc, f.k, tid & 31, f.selected, f.weights, nullptr, 0, 0);
    }
}

static size_t router_chain2_smem(int egc, int tt) {
    return sizeof(float) * (size_t)rv_nr(egc) * ((size_t)RV_K * egc + (size_t)tt * (RV_K + 4));
}

template <bool FUSE>
static void launch_chain2(int egc, int tt, dim3 grid, cudaStream_t st, const float *xdeq, const float *w, int64_t n,
                          int64_t d, int64_t n_exp, float *logits, const RouteFuse &f) {
    static std::atomic<uint64_t> attr{0};  // devices whose smem opt-in is set
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(router_chain2_kernel<8, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(router_chain2_kernel<16, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(router_chain2_kernel<32, FUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    }
    const size_t smem = router_chain2_smem(egc, tt);
    const unsigned threads = (unsigned)ceil_div((int64_t)tt * egc, 32) * 32;
    if (egc == 32)
        launch_pdl(router_chain2_kernel<32, FUSE>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, logits, f);
    else if (egc == 16)
        launch_pdl(router_chain2_kernel<16, FUSE>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, logits, f);
    else
        launch_pdl(router_chain2_kernel<8, FUSE>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, logits, f);
}

static int chain_mode() {  // CQ_ROUTER_CHAIN: 0 off, 1 chain kernels, 2 without the fused tail, 3 v1 kernel only
    static int mode = -1;
    if (mode < 0) {
        const char *e = getenv("CQ_ROUTER_CHAIN");
        mode = e ? atoi(e) : 1;
    }
    return mode;
}

// Decode-sized batches (at most one wave of CTAs, each holding tt * EG <= 32
// chains) take router_chain_kernel.  With `fuse` given and a single expert
// group, the same launch also does top-k and the permutation; *fused says so
// (the counts and the arrival counter must have been zeroed).
static bool router_chain(const float *xdeq, const float *w, int64_t n, int64_t d, int64_t n_exp, float *logits,
                         const RouteFuse *fuse, cudaStream_t st, bool *fused) {
    if (fused) *fused = false;
    if (xdeq == nullptr || d % 16 || n_exp % 8 || chain_mode() == 0) return false;
    if (chain_mode() != 3 && n_exp % 32 == 0) {
        if (fuse != nullptr && fuse->qx != nullptr) return false;  // no quantizer in the v2 form
        // v2 (one chain per thread) when E % 32 == 0 (16 experts per CTA by default), every
        // warp forms its own products (QW decode 64: 37 -> 18 us).  Smaller groups keep v1, whose
        // producer warps feed one chain warp (v2 measured 2x slower there: one warp issues all).
        static int egc_env = -1;  // CQ_ROUTER_EGC: experts per CTA (experiments)
        if (egc_env < 0) {
            const char *e = getenv("CQ_ROUTER_EGC");
            egc_env = e ? atoi(e) : 16;  // 16 vs 32, same box x 3: QW decode 64 -0.2 us, 256 -0.45 us
        }
        int egc = egc_env == 8 || egc_env == 32 ? egc_env : 16;
        if (fuse != nullptr && n_exp == 32) egc = 32;  // one group: the launch also does the top-k
        const int64_t groups = n_exp / egc;
        // 64-thread CTAs while they fit one per SM: the four warps of a 128-thread CTA need 5 shared-memory
        // wavefronts per column (W 1 per warp, x 1 per 4 columns), above the 4.2-cycle add chain
        static int nth_env = -1;  // CQ_ROUTER_NTH: 64 / 128 forces one (experiments)
        if (nth_env < 0) {
            const char *e = getenv("CQ_ROUTER_NTH");
            nth_env = e ? atoi(e) : 0;
        }
        const int nth = nth_env == 64 || nth_env == 128 ? nth_env : (ceil_div(n, 64 / egc) * groups <= 148 ? 64 : 128);
        const int tt = nth / egc;
        const int64_t ctas = ceil_div(n, tt) * groups;
        if (ctas > 2 * 148 || router_chain2_smem(egc, tt) > 220 * 1024) return false;  // the tiled routers
        const bool can_fuse = groups == 1 && chain_mode() == 1 && fuse != nullptr;
        if (fuse != nullptr && !can_fuse) return false;  // the caller runs the separate kernels
        const dim3 grid((unsigned)ceil_div(n, tt), (unsigned)groups);
        if (can_fuse) {
            launch_chain2<true>(egc, tt, grid, st, xdeq, w, n, d, n_exp, logits, *fuse);
            *fused = true;
        } else {
            launch_chain2<false>(egc, tt, grid, st, xdeq, w, n, d, n_exp, logits, RouteFuse{});
        }
        return true;
    }
    const int eg = n_exp % 32 == 0 ? 32 : (n_exp % 16 == 0 ? 16 : 8);
    const int64_t groups = n_exp / eg;
    const int tt = (int)std::min<int64_t>(32 / eg, std::max<int64_t>(1, ceil_div(n * groups, 148)));
    const int64_t ctas = ceil_div(n, tt) * groups;
    const bool qin = fuse != nullptr && fuse->qx != nullptr;
    const bool can_fuse = groups == 1 && chain_mode() == 1 && fuse != nullptr;
    if (fuse != nullptr && !can_fuse) return false;  // the caller runs the separate kernels
    const size_t smem = router_chain_smem(eg, tt, qin ? d : 0, can_fuse);
    if (can_fuse && (smem > RC_FUSE_SMEM_MAX || (qin && d % 4))) return false;
    const int64_t per_sm = std::max<int64_t>(1, (int64_t)(227 * 1024) / (int64_t)(smem + 1024));
    if (ctas > per_sm * 148) return false;
    const dim3 grid((unsigned)ceil_div(n, tt), (unsigned)groups);
    if (can_fuse) {
        if (qin)
            launch_chain<true, true>(eg, grid, smem, st, xdeq, w, n, d, n_exp, tt, logits, *fuse);
        else
            launch_chain<true>(eg, grid, smem, st, xdeq, w, n, d, n_exp, tt, logits, *fuse);
        *fused = true;
    } else {
        launch_chain<false>(eg, grid, smem, st, xdeq, w, n, d, n_exp, tt, logits, RouteFuse{});
    }
    return true;
}

// Router logits + top-k in one launch where router_chain can fuse them
// (*fused); otherwise nothing is launched.
cq_status router_fused(const float *xdeq, const float *w, int64_t n, int64_t d, int64_t n_exp, float *logits,
                       int32_t *selected, float *weights, int64_t k, cudaStream_t st, bool *fused) {
    *fused = false;
    if (n * n_exp == 0 || k < 1 || k > MAX_TOPK || k > n_exp) return CQ_OK;
    RouteFuse f{selected, weights, k};
    if (!router_chain(xdeq, w, n, d, n_exp, logits, &f, st, fused)) return CQ_OK;
    return check_launch("router_fused");
}

// Quantizer + router logits + top-k in one launch where router_chain can fuse them (*fused:
// codes, scales, code sums and the cleared counters written as quantize_a4 writes them); otherwise
// nothing is launched.  xdeq: scratch the caller owns (unused by the fused kernel).
cq_status router_fused_quant(const void *x, int dtype, int8_t *codes, float *scales, int *nonfinite, int32_t *tsum,
                             int32_t *zero, int n_zero, float *xdeq, const float *w, int64_t n, int64_t d,
                             int64_t n_exp, float *logits, int32_t *selected, float *weights, int64_t k,
                             cudaStream_t st, bool *fused) {
    *fused = false;
    if (n * n_exp == 0 || k < 1 || k > MAX_TOPK || k > n_exp) return CQ_OK;
    if (dtype != CQ_DTYPE_F32 && dtype != CQ_DTYPE_BF16) return CQ_OK;
    RouteFuse f{selected, weights, k, x, dtype, codes, scales, nonfinite, tsum, zero, n_zero};
    if (!router_chain(xdeq, w, n, d, n_exp, logits, &f, st, fused)) return CQ_OK;
    return check_launch("router_fused_quant");
}

// Token tile: TI x tq tokens, tq groups per expert quad chosen so the grid is about one CTA per SM.
template <int TI>
static cq_status router_tile_launch(const float *xdeq, const float *w, int64_t n, int64_t d, int64_t n_exp,
                                    float *logits, cudaStream_t st) {
    const int eq = (int)n_exp / 4;
    const int tq = (int)std::min<int64_t>(256 / eq, std::max<int64_t>(128 / eq, ceil_div(n, 148 * TI)));
    const int nt = tq * eq, tt = TI * tq;
    const int64_t ctas = ceil_div(n, tt);
    const int smem_max = ctas <= 148 ? 200 * 1024 : 96 * 1024;  // one CTA per SM, else two
    int rk = (int)std::min<int64_t>(512, (smem_max / 8 - 4 * tt) / (tt + n_exp)) & ~15;
    if (rk < 16) rk = 16;
    constexpr int RKC = 128, RKS = 64;  // the compile-time chunk widths, when they fit
    const int fixed = rk >= RKC ? RKC : (rk >= RKS ? RKS : 0);
    if (fixed) rk = fixed;
    const size_t smem = (size_t)8 * ((size_t)tt * (rk + 4) + (size_t)rk * n_exp);
    static std::atomic<uint64_t> attr{0};  // devices whose smem opt-in is set
    if (first_on_device(attr)) {
        cudaFuncSetAttribute(router_tile_kernel<32, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<64, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<128, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<32, TI, RKC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<64, TI, RKC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<128, TI, RKC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<32, TI, RKS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<64, TI, RKS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(router_tile_kernel<128, TI, RKS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
    }
    const dim3 grid((unsigned)ctas);
#define CQ_TILE(EC_)                                                                                        \
    (fixed == RKC   ? launch_pdl(router_tile_kernel<EC_, TI, RKC>, grid, nt, smem, st, xdeq, w, n, d, rk, logits) \
     : fixed == RKS ? launch_pdl(router_tile_kernel<EC_, TI, RKS>, grid, nt, smem, st, xdeq, w, n, d, rk, logits) \
                    : launch_pdl(router_tile_kernel<EC_, TI>, grid, nt, smem, st, xdeq, w, n, d, rk, logits))
    if (n_exp == 32)
        CQ_TILE(32);
    else if (n_exp == 64)
        CQ_TILE(64);
    else
        CQ_TILE(128);
#undef CQ_TILE
    return check_launch("router_logits");
}

// xdeq (nullable): the dequantized rows code * scale from the quantizer.
cq_status router_logits(const int8_t *codes, const float *scales, const float *xdeq, const float *w, int64_t n,
                        int64_t d, int64_t n_exp, float *logits, cudaStream_t st) {
    if (n * n_exp == 0) return CQ_OK;
    if (n_exp > 256) {
        set_error("router: at most 256 experts");
        return CQ_ERR_CONFIG;
    }
    if (router_chain(xdeq, w, n, d, n_exp, logits, nullptr, st, nullptr)) return check_launch("router_logits");
    if (xdeq != nullptr && d % 16 == 0 && (n_exp == 32 || n_exp == 64 || n_exp == 128) && n >= 64)
        return router_tile_launch<4>(xdeq, w, n, d, n_exp, logits, st);
    if (xdeq != nullptr && n_exp <= RD_THREADS && d % 16 == 0) {
        // tokens per CTA: fewer, smaller CTAs stage less per chunk (CQ_ROUTER_TT overrides, experiments)
        static int tt_env = -1;
        if (tt_env < 0) {
            const char *e = getenv("CQ_ROUTER_TT");
            tt_env = e ? atoi(e) : 0;
        }
        // about one CTA per SM: a decode batch gets one token per CTA (the chains run on many SMs
        // and each stages little), a large batch up to 128 / E tokens per CTA (W reused across them)
        int tt = (int)std::min<int64_t>(RD_THREADS / n_exp, std::max<int64_t>(1, ceil_div(n, 148)));
        if (tt_env > 0 && tt_env * n_exp <= RD_THREADS) tt = tt_env;
        const int threads = (int)ceil_div(tt * n_exp, 32) * 32;
        // double-buffered x [tt][rk] + W [rk][E] f32 in <= 48 KB; rk a multiple of 16, <= 512
        static int rd_kb = -1;  // CQ_ROUTER_RD_KB: the CTA's shared-memory budget (experiments)
        if (rd_kb < 0) {
            const char *e = getenv("CQ_ROUTER_RD_KB");
            // PH (E = 16): 96 KB 76.8 us (two CTAs per SM, 1.7 waves), 64 78, 48 72.2, 32 75.3
            rd_kb = e ? atoi(e) : 48;
        }
        int rk = (int)std::min<int64_t>(512, (((int64_t)rd_kb * 1024) / (8 * (tt + n_exp))) & ~15LL);
        if (rk < 16) rk = 16;
        const size_t smem = (size_t)8 * rk * (tt + n_exp);
        static std::atomic<uint64_t> attr{0};  // devices whose smem opt-in is set
        if (first_on_device(attr)) {
            cudaFuncSetAttribute(router_deq_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(router_deq_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(router_deq_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(router_deq_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(router_deq_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        }
        const dim3 grid((unsigned)ceil_div(n, tt));
        switch (n_exp) {
            case 8: launch_pdl(router_deq_kernel<8>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, rk, logits); break;
            case 16: launch_pdl(router_deq_kernel<16>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, rk, logits); break;
            case 64: launch_pdl(router_deq_kernel<64>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, rk, logits); break;
            case 128:
                launch_pdl(router_deq_kernel<128>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, rk, logits);
                break;
            default: launch_pdl(router_deq_kernel<0>, grid, threads, smem, st, xdeq, w, n, d, n_exp, tt, rk, logits);
        }
        return check_launch("router_logits");
    }
    const int tt = (int)(256 / n_exp);
    // W chunk [rk][E] + inputs [tt][rk] in <= 48 KB of shared memory
    const int rk = (int)std::max<int64_t>(16, std::min<int64_t>(256, (12288 / (n_exp + tt)) & ~15LL));
    const size_t smem = ((size_t)rk * n_exp + (size_t)tt * rk) * sizeof(float);
    router_logits_kernel<<<(unsigned)ceil_div(n, tt), (unsigned)(tt * n_exp), smem, st>>>(codes, scales, w, n, d,
                                                                                         n_exp, rk, logits);
    return check_launch("router_logits");
}

cq_status topk(const float *logits, int64_t n, int64_t n_exp, int64_t k, int32_t *sel, float *wts,
               int32_t *counts, int64_t local_begin, int64_t n_local, cudaStream_t st) {
    if (k < 1 || k > MAX_TOPK || k > n_exp) {
        set_error("top_k must be in [1, min(16, n_experts)]");
        return CQ_ERR_CONFIG;
    }
    if (n == 0) return CQ_OK;
    // logits per lane: the selection rounds scan only the lanes' real experts
    auto kern = n_exp <= 32 ? topk_kernel<1> : n_exp <= 64 ? topk_kernel<2> : n_exp <= 128 ? topk_kernel<4> : topk_kernel<8>;
    launch_pdl(kern, (unsigned)ceil_div(n, TOPK_WARPS * TOPK_TPW), TOPK_WARPS * 32, 0, st, logits, n, n_exp, k, sel,
               wts, counts, local_begin, n_local);
    return check_launch("topk");
}

// counts: read (large batches: written by the top-k), or written here when
// permute_counts_itself(n) (the top-k then runs without counts).
cq_status permute(const int32_t *sel, int32_t *counts, int64_t n, int64_t k, int64_t local_begin,
                  int64_t n_local, int32_t *offsets, int32_t *perm_token, int32_t *perm_slot,
                  int32_t *inv, cudaStream_t st) {
    if (n_local == 0) return CQ_OK;
    if (permute_counts_itself(n)) {
        const int smem = (int)std::max<int64_t>(n, 1) * 4;
        cudaFuncSetAttribute(permute_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        launch_pdl(permute_count_kernel, (unsigned)n_local, PERMC_THREADS, (size_t)smem, st, sel, n, k, local_begin,
                   n_local, counts, offsets, perm_token, perm_slot, inv);
        return check_launch("permute");
    }
    launch_pdl(permute_kernel, (unsigned)n_local, PERM_THREADS, 0, st, sel, counts, n, k, local_begin, n_local,
                                                               offsets, perm_token, perm_slot, inv);
    return check_launch("permute");
}

cq_status gather_rows(const int8_t *src, const float *sscale, const int32_t *perm_token,
                      const int32_t *offsets, int64_t n_local, int64_t rows_bound, int64_t d,
                      int8_t *dst, float *dscale, cudaStream_t st) {
    if (rows_bound == 0) return CQ_OK;
    launch_pdl(gather_rows_kernel, (unsigned)rows_bound, 128, 0, st, src, sscale, perm_token, offsets, n_local, d,
                                                             dst, dscale);
    return check_launch("gather_rows");
}

}  // namespace cq

using namespace cq;

extern "C" cq_status cq_route_topk(const float *logits, int64_t n, int64_t n_experts, int64_t top_k,
                                   int32_t *selected, float *weights, void *stream) {
    if (n < 0 || n_experts < 1) {
        set_error("route: bad shape");
        return CQ_ERR_SHAPE;
    }
    return topk(logits, n, n_experts, top_k, selected, weights, nullptr, 0, 0, as_stream(stream));
}
