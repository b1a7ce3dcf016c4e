// Router (model.py:379-385), top-k (model.py:324-330) and the builder-defined
// token permutation into per-expert segments.
//
// Bit-exactness: logits reproduce the ordered fp32 chain of _core.matmul_f32
// (k ascending, no FMA) on the exact fake-quant input codes*scale
// (quant.py:8-13); top-k ids, their order, counts, offsets and the permutation
// are therefore bit-exact.  Route weights use CUDA expf (ulp-bounded vs numpy).
#include "common.cuh"

namespace cq {

// logits[t, e] = sum_k (q[t,k] * s_t) * W[k, e], k ascending, one rounding per
// multiply and per add (the chain of _core.matmul_f32).  A CTA owns TT tokens x
// E experts (one thread per chain); W and the exact fake-quant inputs q*s are
// staged in shared memory RK columns at a time so the chains read smem, not L2.
__global__ void router_logits_kernel(const int8_t *__restrict__ codes, const float *__restrict__ scales,
                                     const float *__restrict__ w, int64_t n, int64_t d, int64_t n_exp, int rk,
                                     float *__restrict__ logits) {
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

// Same chains, with the W / code chunks double-buffered by cp.async so the
// next chunk lands while the current one is consumed (d % 16 == 0 and
// rk * E % 4 == 0; the kernel above covers every other shape).
__global__ void router_logits_async_kernel(const int8_t *__restrict__ codes, const float *__restrict__ scales,
                                           const float *__restrict__ w, int64_t n, int64_t d, int64_t n_exp, int rk,
                                           float *__restrict__ logits) {
    extern __shared__ __align__(16) float rsm[];
    const int tt_n = blockDim.x / (int)n_exp;
    const int wsz = rk * (int)n_exp, csz = tt_n * rk;  // floats of W, bytes of codes per buffer
    float *wbuf[2] = {rsm, rsm + wsz};
    int8_t *cbuf[2] = {reinterpret_cast<int8_t *>(rsm + 2 * wsz), reinterpret_cast<int8_t *>(rsm + 2 * wsz) + csz};
    const int t_loc = threadIdx.x / (int)n_exp, e = threadIdx.x % (int)n_exp;
    const int64_t t0 = blockIdx.x * (int64_t)tt_n;
    const int64_t t = t0 + t_loc;
    const bool live = t_loc < tt_n && t < n;
    const float s = live ? __ldg(scales + t) : 0.0f;
    const int n_chunks = (int)((d + rk - 1) / rk);
    auto load = [&](int ci, int b) {
        const int64_t k0 = (int64_t)ci * rk;
        const int kn = (int)((d - k0) < rk ? (d - k0) : rk);
        for (int x = threadIdx.x * 4; x < kn * n_exp; x += blockDim.x * 4) cp_async16(wbuf[b] + x, w + k0 * n_exp + x);
        const int rowv = kn / 16;
        for (int x = threadIdx.x; x < tt_n * rowv; x += blockDim.x) {
            const int tl = x / rowv, v = x - tl * rowv;
            const int64_t tg = t0 + tl < n ? t0 + tl : n - 1;  // clamp: rows past n are never consumed
            cp_async16(cbuf[b] + tl * rk + v * 16, codes + tg * d + k0 + v * 16);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    load(0, 0);
    float acc = 0.0f;
    for (int ci = 0; ci < n_chunks; ++ci) {
        const int b = ci & 1;
        if (ci + 1 < n_chunks) {
            load(ci + 1, b ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int64_t k0 = (int64_t)ci * rk;
        const int kn = (int)((d - k0) < rk ? (d - k0) : rk);
        if (live) {
            const int8_t *cr = cbuf[b] + t_loc * rk;
            const float *wr = wbuf[b] + e;
#pragma unroll 8
            for (int kk = 0; kk < kn; ++kk)
                acc = __fadd_rn(acc, __fmul_rn(__fmul_rn((float)cr[kk], s), wr[kk * n_exp]));
        }
        __syncthreads();  // buffer b is refilled by the next iteration's prefetch
    }
    if (live) logits[t * n_exp + e] = acc;
}

// Same chains, split so the serial part is only the additions: 128 producer
// threads form the products p[k][j] = fl(fl(q[t,k] * s_t) * W[k,e]) for a
// chunk of RK columns into shared memory while the chain threads (one per
// (token, expert) pair, CH per CTA) add the previous chunk in k order.  Named
// barriers double-buffer the product chunks.  The dependent fp32 adds are
// the floor (~4 cycles each).
constexpr int RC_PROD = 128;

// Shared-memory plan of router_chain_kernel for chunk size rk: double-buffered
// codes [tt][rk] i8, W [rk][E] f32 and products [rk][ch] f32.
struct RcPlan {
    int rk;
    size_t codes, wts, prod, total;
};

__host__ __device__ inline RcPlan rc_plan(int rk, int tt, int ch, int64_t n_exp) {
    RcPlan p;
    p.rk = rk;
    p.codes = 0;
    p.wts = (((size_t)2 * tt * rk + 15) / 16) * 16;
    p.prod = p.wts + (size_t)2 * rk * n_exp * 4;
    p.total = p.prod + (size_t)2 * rk * ch * 4;
    return p;
}

__global__ void router_chain_kernel(const int8_t *__restrict__ codes, const float *__restrict__ scales,
                                    const float *__restrict__ w, int64_t n, int64_t d, int64_t n_exp, int tt, int ch,
                                    int rk, float *__restrict__ logits) {
    extern __shared__ __align__(16) uint8_t rsm_raw[];
    const RcPlan plan = rc_plan(rk, tt, ch, n_exp);
    int8_t *cst = reinterpret_cast<int8_t *>(rsm_raw + plan.codes);   // [2][tt][rk]
    float *wst = reinterpret_cast<float *>(rsm_raw + plan.wts);       // [2][rk][E]
    float *prod = reinterpret_cast<float *>(rsm_raw + plan.prod);     // [2][rk][ch]
    const int tid = threadIdx.x;
    const int64_t t0 = blockIdx.x * (int64_t)tt;
    const int n_chunks = (int)((d + rk - 1) / rk);
    const int nthreads = ch + RC_PROD;
    if (tid < ch) {
        // ---- chain threads: the ordered adds only
        const int t_loc = tid / (int)n_exp, e = tid % (int)n_exp;
        const bool live = t_loc < tt && t0 + t_loc < n;
        float acc = 0.0f;
        for (int i = 0; i < n_chunks; ++i) {
            const int b = i & 1;
            asm volatile("bar.sync %0, %1;" ::"r"(1 + b), "r"(nthreads) : "memory");
            const int kn = (int)((d - (int64_t)i * rk) < rk ? (d - (int64_t)i * rk) : rk);
            const float *pb = prod + (size_t)b * rk * ch + tid;
            int kk = 0;
            if (kn >= 16) {
                float cur[16], nxt[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) cur[u] = pb[u * ch];
                for (kk = 16; kk + 16 <= kn; kk += 16) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) nxt[u] = pb[(kk + u) * ch];
#pragma unroll
                    for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, cur[u]);
#pragma unroll
                    for (int u = 0; u < 16; ++u) cur[u] = nxt[u];
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, cur[u]);
            }
            for (; kk < kn; ++kk) acc = __fadd_rn(acc, pb[kk * ch]);
            if (i + 2 < n_chunks) asm volatile("bar.arrive %0, %1;" ::"r"(3 + b), "r"(nthreads) : "memory");
        }
        if (live) logits[(t0 + t_loc) * n_exp + e] = acc;
    } else {
        // ---- helpers: stage codes + W of chunk i+1 (cp.async) while forming
        // the products of chunk i from shared memory
        const int pt = tid - ch;
        auto stage = [&](int i) {
            const int b = i & 1;
            const int64_t k0 = (int64_t)i * rk;
            const int kn = (int)((d - k0) < rk ? (d - k0) : rk);
            for (int x = pt * 4; x < kn * (int)n_exp; x += RC_PROD * 4)
                cp_async16(wst + (size_t)b * rk * n_exp + x, w + k0 * n_exp + x);
            const int rowv = kn / 16;
            for (int x = pt; x < tt * rowv; x += RC_PROD) {
                const int tl = x / rowv, v = x - tl * rowv;
                const int64_t tg = t0 + tl < n ? t0 + tl : n - 1;
                cp_async16(cst + (size_t)b * tt * rk + tl * rk + v * 16, codes + tg * d + k0 + v * 16);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        const int j = pt % ch, kk0 = pt / ch, kstep = RC_PROD / ch;
        const int t_loc = j / (int)n_exp, e = j - t_loc * (int)n_exp;
        const bool live = t_loc < tt && t0 + t_loc < n;
        const float s = live ? __ldg(scales + t0 + t_loc) : 0.0f;
        stage(0);
        for (int i = 0; i < n_chunks; ++i) {
            const int b = i & 1;
            if (i + 1 < n_chunks) {
                stage(i + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            asm volatile("bar.sync 5, %0;" ::"r"(RC_PROD) : "memory");  // chunk i staged by every helper
            if (i >= 2) asm volatile("bar.sync %0, %1;" ::"r"(3 + b), "r"(nthreads) : "memory");
            const int kn = (int)((d - (int64_t)i * rk) < rk ? (d - (int64_t)i * rk) : rk);
            const int8_t *cr = cst + (size_t)b * tt * rk + (live ? t_loc : 0) * rk;
            const float *wr = wst + (size_t)b * rk * n_exp + e;
            float *pb = prod + (size_t)b * rk * ch + j;
            for (int kk = kk0; kk < kn; kk += kstep)
                pb[kk * ch] = live ? __fmul_rn(__fmul_rn((float)cr[kk], s), wr[kk * n_exp]) : 0.0f;
            asm volatile("bar.arrive %0, %1;" ::"r"(1 + b), "r"(nthreads) : "memory");
            asm volatile("bar.sync 5, %0;" ::"r"(RC_PROD) : "memory");  // stage buffer b reusable
        }
    }
}

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

constexpr int MAX_TOPK = 16;

// One thread per token: stable descending selection (ties -> lower id; +0 and
// -0 compare equal like numpy's sort), softmax over the selected logits, and
// per-expert route counts for the local expert range.
__global__ void topk_kernel(const float *__restrict__ logits, int64_t n, int64_t n_exp, int64_t k,
                            int32_t *__restrict__ selected, float *__restrict__ weights,
                            int32_t *__restrict__ counts, int64_t local_begin, int64_t n_local) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const float *row = logits + t * n_exp;
    int sel[MAX_TOPK];
    float val[MAX_TOPK];
    for (int s = 0; s < k; ++s) {
        int best = -1;
        float bv = 0.0f;
        for (int e = 0; e < n_exp; ++e) {
            bool taken = false;
            for (int p = 0; p < s; ++p) taken |= (sel[p] == e);
            if (taken) continue;
            const float v = row[e];
            if (best < 0 || v > bv) {
                best = e;
                bv = v;
            }
        }
        sel[s] = best;
        val[s] = bv;
    }
    const float m = val[0];  // max of the selected logits
    float ex[MAX_TOPK];
    for (int s = 0; s < k; ++s) ex[s] = expf(__fsub_rn(val[s], m));
    const float tot = np_sum(ex, (int)k);
    for (int s = 0; s < k; ++s) {
        selected[t * k + s] = sel[s];
        weights[t * k + s] = __fdiv_rn(ex[s], tot);
        const int64_t le = sel[s] - local_begin;
        if (counts != nullptr && le >= 0 && le < n_local) atomicAdd(counts + le, 1);
    }
}

// CTA per local expert: a stable block scan over tokens assigns each route of
// this expert its row in the segment; CTA 0 also publishes offsets[0..E].
constexpr int PERM_THREADS = 1024;

__global__ void __launch_bounds__(PERM_THREADS) permute_kernel(
    const int32_t *__restrict__ selected, const int32_t *__restrict__ counts, int64_t n, int64_t k,
    int64_t local_begin, int64_t n_local, int32_t *__restrict__ offsets,
    int32_t *__restrict__ perm_token, int32_t *__restrict__ perm_slot, int32_t *__restrict__ inv) {
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

// rows_out[r, :] = rows_in[perm_token[r], :], r < offsets[n_local]; also scales.
__global__ void gather_rows_kernel(const int8_t *__restrict__ src, const float *__restrict__ sscale,
                                   const int32_t *__restrict__ perm_token,
                                   const int32_t *__restrict__ offsets, int64_t n_local, int64_t d,
                                   int8_t *__restrict__ dst, float *__restrict__ dscale) {
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

cq_status router_logits(const int8_t *codes, const float *scales, const float *w, int64_t n,
                        int64_t d, int64_t n_exp, float *logits, cudaStream_t st) {
    if (n * n_exp == 0) return CQ_OK;
    if (n_exp > 256) {
        set_error("router: at most 256 experts");
        return CQ_ERR_CONFIG;
    }
    if (n_exp <= 128 && d % 16 == 0) {
        // chains per CTA: >= one warp; staging + products double-buffered in <= 48 KB
        const int tt2 = (int)std::max<int64_t>(1, 32 / n_exp);
        const int ch = (int)(ceil_div(tt2 * n_exp, 32) * 32);
        int rk = 256;
        while (rk > 16 && rc_plan(rk, tt2, ch, n_exp).total > 48 * 1024) rk -= 16;
        const size_t smem = rc_plan(rk, tt2, ch, n_exp).total;
        router_chain_kernel<<<(unsigned)ceil_div(n, tt2), (unsigned)(ch + RC_PROD), smem, st>>>(
            codes, scales, w, n, d, n_exp, tt2, ch, rk, logits);
        return check_launch("router_logits");
    }
    const int tt = (int)(256 / n_exp);
    if (d % 16 == 0) {
        // double-buffered W chunk [rk][E] f32 + codes [tt][rk] i8 in <= 48 KB of shared memory
        const int rk = (int)std::max<int64_t>(16, std::min<int64_t>(256, (24576 / (4 * n_exp + tt)) & ~15LL));
        const size_t smem = 2 * ((size_t)rk * n_exp * sizeof(float) + (size_t)tt * rk);
        router_logits_async_kernel<<<(unsigned)ceil_div(n, tt), (unsigned)(tt * n_exp), smem, st>>>(
            codes, scales, w, n, d, n_exp, rk, logits);
        return check_launch("router_logits");
    }
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
    topk_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(logits, n, n_exp, k, sel, wts, counts,
                                                            local_begin, n_local);
    return check_launch("topk");
}

cq_status permute(const int32_t *sel, const int32_t *counts, int64_t n, int64_t k, int64_t local_begin,
                  int64_t n_local, int32_t *offsets, int32_t *perm_token, int32_t *perm_slot,
                  int32_t *inv, cudaStream_t st) {
    if (n_local == 0) return CQ_OK;
    permute_kernel<<<(unsigned)n_local, PERM_THREADS, 0, st>>>(sel, counts, n, k, local_begin, n_local,
                                                               offsets, perm_token, perm_slot, inv);
    return check_launch("permute");
}

cq_status gather_rows(const int8_t *src, const float *sscale, const int32_t *perm_token,
                      const int32_t *offsets, int64_t n_local, int64_t rows_bound, int64_t d,
                      int8_t *dst, float *dscale, cudaStream_t st) {
    if (rows_bound == 0) return CQ_OK;
    gather_rows_kernel<<<(unsigned)rows_bound, 128, 0, st>>>(src, sscale, perm_token, offsets, n_local, d,
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
