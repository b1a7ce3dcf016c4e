// Certified A4 quantization of the tensor-core rotation (pipeline.py:516 then
// quant.py:89-100): the codes and scale the reference gets from its ordered
// fp32 chain v = x @ R (linalg.py:66-75 -> _core.pyx:27-38), bit for bit, at
// tensor-core speed.
//
// rot_gemm (rotate_tc.cu) gives v_tc with |v_tc - v_chain| <= eps_rel * max|v|
// per row (measured: tools/rot_err.py, max 2.6e-5 over 50M PH elements; the
// default band is 6x that).  The quantizer only needs, per row, the exact
// max|v| (-> the snapped scale) and, per element, which side of a rounding
// boundary v lies on.  So one warp per row:
//   1. mx = max|v_tc|; every element with |v_tc| >= mx - 2 eps is a candidate
//      for the true maximum: recompute those with the ordered chain (one lane
//      per element), take the exact maximum, s = snap(max / 7);
//   2. an element whose interval [v_tc - eps, v_tc + eps] maps to one code is
//      settled; the others (a few per 4096-wide row) are recomputed with the
//      ordered chain and coded from the exact value.
// The chains (k ascending, separate fp32 multiply and add, as the reference)
// read R^T rows, prepared once next to the bf16 planes.
#include "common.cuh"

namespace cq {

constexpr int RQ_WARPS = 8;       // rows per CTA
constexpr int RQ_LIST = 128;      // elements collected per warp and round
constexpr int RQ_RB = 8;          // row loads in flight per lane in the row scans
// Band tests use t = v * (1/s) with approximate reciprocals: a code boundary counts as inside the
// band when it is within RQ_SLACK (code units) of it, far above their ~1e-6 error.  A settled
// element's band then clears every boundary by more than that error, so its code from the
// approximate t equals quant.py's IEEE-division code.
constexpr float RQ_SLACK = 1e-4f;

// v[row, j] in the reference's ordered chain: ((0 + x0 R0j) + x1 R1j) + ...  (k ascending, separate
// fp32 multiply and add, _core.pyx:27-38).  All lanes of a warp walk the same token row in lockstep,
// so the x loads are warp-uniform (broadcast); each lane streams its own R^T row.  (Deeper register
// prefetch of the R^T stream and shared-memory copies of x measured slower: occupancy.)
template <int DT>
__device__ float rq_chain(const void *__restrict__ x, int64_t row, int64_t d, const float *__restrict__ Rt,
                          int64_t j) {
    const float4 *r4 = reinterpret_cast<const float4 *>(Rt + j * d);
    float acc = 0.0f;
#pragma unroll 4
    for (int64_t k8 = 0; k8 < d / 8; ++k8) {
        const float4 ra = __ldg(r4 + 2 * k8), rb = __ldg(r4 + 2 * k8 + 1);
        float xv[8];
        if (DT == CQ_DTYPE_F32) {
            const float4 *x4 = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(x) + row * d);
            const float4 xa = __ldg(x4 + 2 * k8), xb = __ldg(x4 + 2 * k8 + 1);
            xv[0] = xa.x, xv[1] = xa.y, xv[2] = xa.z, xv[3] = xa.w, xv[4] = xb.x, xv[5] = xb.y, xv[6] = xb.z, xv[7] = xb.w;
        } else {
            const uint4 u = __ldg(reinterpret_cast<const uint4 *>(reinterpret_cast<const uint16_t *>(x) + row * d) + k8);
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                xv[2 * q] = __uint_as_float(w[q] << 16);
                xv[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
            }
        }
        const float rv[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __fadd_rn(acc, __fmul_rn(xv[q], rv[q]));
    }
    return acc;
}

// The collected elements idx[0..cnt) -> exact values val[], one lane per element.
template <int DT>
__device__ __forceinline__ void rq_resolve(const void *x, int64_t row, int64_t d, const float *Rt,
                                           const int32_t *idx, float *val, int cnt, int lane) {
    for (int i = lane; i < cnt; i += 32) val[i] = rq_chain<DT>(x, row, d, Rt, idx[i]);
    __syncwarp();
}

// The A4 code of t = x / s given t (round half away from zero, clip to [-8, 7]; quant.py:69-100).
__device__ __forceinline__ int rq_code_t(float t) { return (int)fminf(fmaxf(roundf(t), -8.0f), 7.0f); }

// Collect the row's elements selected by pick(value) -> (index) into idx[] in ascending order:
// entries with rank in [lo, lo + RQ_LIST); returns the total count.  One scan of the row.
template <class Pick>
__device__ __forceinline__ int rq_collect(const float4 *v4, int64_t nv, int lane, int lo, int32_t *idx, Pick pick) {
    int total = 0;
    // RQ_RB iterations' loads are issued before their (warp-synchronous) scans: the row streams with
    // RQ_RB loads in flight per lane instead of one memory latency per 128 elements
    for (int64_t b0 = 0; b0 < nv; b0 += 32 * RQ_RB) {
        float4 a[RQ_RB];
#pragma unroll
        for (int r = 0; r < RQ_RB; ++r) {
            const int64_t j = b0 + r * 32 + lane;
            a[r] = j < nv ? v4[j] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
#pragma unroll
        for (int r = 0; r < RQ_RB; ++r) {
            const int64_t j = b0 + r * 32 + lane;
            unsigned m = 0;
            if (j < nv)
                m = (pick(a[r].x) ? 1u : 0u) | (pick(a[r].y) ? 2u : 0u) | (pick(a[r].z) ? 4u : 0u) |
                    (pick(a[r].w) ? 8u : 0u);
            const unsigned any = __ballot_sync(0xffffffffu, m != 0);
            if (any == 0) continue;  // the common case: nothing picked in these 128 elements
            const int mine = __popc(m);
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int pos = total + incl - mine;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (m >> e & 1u) {
                    if (pos >= lo && pos < lo + RQ_LIST) idx[pos - lo] = (int32_t)(4 * j + e);
                    ++pos;
                }
            total += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncwarp();
    return total;
}

// Per-row band state: the approximate max, the error band and the scale range it allows.
struct RqRow {
    float mx, eps, thr, s_lo, s_hi, r_lo, r_hi;
    __device__ RqRow(float mx_, float eps_rel) : mx(mx_) {
        eps = eps_rel * mx;
        thr = mx > 0.0f ? mx - 2.0f * eps : INFINITY;  // an all-zero row has no candidates
        s_lo = a4_scale(fmaxf(mx - eps, 0.0f));
        s_hi = a4_scale(mx + eps);
        r_lo = 1.0f / s_lo;  // s_lo <= s <= s_hi
        r_hi = 1.0f / s_hi;
    }
    // a candidate for the true maximum
    __device__ __forceinline__ bool cand(float a) const { return fabsf(a) >= thr; }
    // recomputed in the one-round path: a max candidate, or a code that differs between the ends of
    // the value band under the two ends of the scale range
    __device__ __forceinline__ bool picked(float a) const {
        if (cand(a)) return true;
        const float lo = a - eps, hi = a + eps;
        const float tmin = fminf(lo * r_lo, lo * r_hi), tmax = fmaxf(hi * r_lo, hi * r_hi);
        return rq_code_t(tmin - RQ_SLACK) != rq_code_t(tmax + RQ_SLACK);
    }
};

// Approximate row max (and the non-finite flag).
__device__ __forceinline__ float rq_row_max(const float4 *v4, int64_t nv, int lane, int *nonfinite) {
    float mx = 0.0f;
    bool bad = false;
#pragma unroll 8
    for (int64_t j = lane; j < nv; j += 32) {
        const float4 a = v4[j];
        bad |= !isfinite(a.x) || !isfinite(a.y) || !isfinite(a.z) || !isfinite(a.w);
        mx = fmaxf(fmaxf(mx, fabsf(a.x)), fmaxf(fabsf(a.y), fmaxf(fabsf(a.z), fabsf(a.w))));
    }
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad) && lane == 0 && nonfinite != nullptr) atomicExch(nonfinite, 1);
    return mx;
}

// One-round finish: the picked elements idx[0..total) (ascending) have their exact values in val[];
// the exact max over the candidates gives the scale, settled codes come from v_tc, the others from val.
__device__ void rq_finish_fast(const float *__restrict__ v, int64_t row, int64_t d, int lane, const RqRow &rr,
                               const int32_t *idx, const float *val, int total, int8_t *__restrict__ codes,
                               float *__restrict__ scales, float *__restrict__ deq, int32_t *__restrict__ tsum,
                               int *__restrict__ recomputed) {
    const float4 *v4 = reinterpret_cast<const float4 *>(v + row * d);
    const int64_t nv = d / 4;
    float mxe = 0.0f;
    for (int i = lane; i < total; i += 32)
        if (rr.cand(v[row * d + idx[i]])) mxe = fmaxf(mxe, fabsf(val[i]));
    mxe = warp_max(mxe);
    const float sc = a4_scale(mxe);  // quant.py:76-100 on the exact maximum
    const float rc = 1.0f / sc;
    if (lane == 0) scales[row] = sc;
    int8_t *crow = codes + row * d;
    float4 *drow = deq != nullptr ? reinterpret_cast<float4 *>(deq + row * d) : nullptr;
    int csum = 0;
    // 1. every element with the settled formula (no band test, no scan) ...
#pragma unroll 4
    for (int64_t j = lane; j < nv; j += 32) {
        const float4 a = v4[j];
        const int8_t c0 = (int8_t)rq_code_t(a.x * rc), c1 = (int8_t)rq_code_t(a.y * rc);
        const int8_t c2 = (int8_t)rq_code_t(a.z * rc), c3 = (int8_t)rq_code_t(a.w * rc);
        reinterpret_cast<char4 *>(crow)[j] = make_char4(c0, c1, c2, c3);
        csum += c0 + c1 + c2 + c3;
        // dequantized value, rounded exactly as codes.astype(f32) * scales (model.py:379-381)
        if (drow != nullptr)
            drow[j] = make_float4(__fmul_rn((float)c0, sc), __fmul_rn((float)c1, sc), __fmul_rn((float)c2, sc),
                                  __fmul_rn((float)c3, sc));
    }
    __syncwarp();  // the recomputed elements below overwrite what step 1 wrote for them
    // 2. ... then the recomputed ones (every picked element) from their exact values
    for (int i = lane; i < total; i += 32) {
        const int32_t j = idx[i];
        const int cw = rq_code_t(v[row * d + j] * rc), c = a4_code(val[i], sc);
        crow[j] = (int8_t)c;
        csum += c - cw;
        if (deq != nullptr) deq[row * d + j] = __fmul_rn((float)c, sc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if (lane == 0) {
        if (tsum != nullptr) tsum[row] = csum;
        if (recomputed != nullptr) atomicAdd(recomputed, total);
    }
}

// General path (more than RQ_LIST picked elements): the exact max over the candidates first, in
// rounds, then the unsettled elements under the exact scale, in rounds.  idx / val: RQ_LIST slots.
template <int DT>
__device__ void rq_general(const float *__restrict__ v, const void *__restrict__ x, const float *__restrict__ Rt,
                           int64_t row, int64_t d, int lane, const RqRow &rr, int32_t *idx, float *val,
                           int8_t *__restrict__ codes, float *__restrict__ scales, float *__restrict__ deq,
                           int32_t *__restrict__ tsum, int *__restrict__ recomputed) {
    const float4 *v4 = reinterpret_cast<const float4 *>(v + row * d);
    const int64_t nv = d / 4;
    const float eps = rr.eps;
    auto is_cand = [&](float a) { return rr.cand(a); };
    int n_chain = 0;
    float mxe = 0.0f;
    for (int lo = 0;; lo += RQ_LIST) {
        const int total = rq_collect(v4, nv, lane, lo, idx, is_cand);
        const int cnt = min(RQ_LIST, total - lo);
        if (cnt <= 0) break;
        rq_resolve<DT>(x, row, d, Rt, idx, val, cnt, lane);
        for (int i = lane; i < cnt; i += 32) mxe = fmaxf(mxe, fabsf(val[i]));
        n_chain += cnt;
        __syncwarp();
        if (lo + RQ_LIST >= total) break;
    }
    mxe = warp_max(mxe);
    const float s = a4_scale(mxe);  // quant.py:76-100 on the exact maximum
    if (lane == 0) scales[row] = s;

    // ---- codes: settled where v_tc +- eps give one code, else from the exact chain value
    const float rs = 1.0f / s;
    auto unsettled = [&](float a) {
        return rq_code_t((a - eps) * rs - RQ_SLACK) != rq_code_t((a + eps) * rs + RQ_SLACK);
    };
    int8_t *crow = codes + row * d;
    float4 *drow = deq != nullptr ? reinterpret_cast<float4 *>(deq + row * d) : nullptr;
    int csum = 0;
    for (int lo = 0;; lo += RQ_LIST) {
        const int total = rq_collect(v4, nv, lane, lo, idx, unsettled);
        const int cnt = max(0, min(RQ_LIST, total - lo));
        rq_resolve<DT>(x, row, d, Rt, idx, val, cnt, lane);
        n_chain += cnt;
        // write the row: round 0 the settled codes, every round the unsettled ones of its window
        int seen = 0;
        for (int64_t base = 0; base < nv; base += 32) {
            const int64_t j = base + lane;
            int8_t c[4] = {0, 0, 0, 0};
            unsigned m = 0;
            if (j < nv) {
                const float4 a = v4[j];
                const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    c[e] = (int8_t)rq_code_t(av[e] * rs);  // settled: equals a4_code(av[e], s)
                    if (unsettled(av[e])) m |= 1u << e;
                }
            }
            const int mine = __popc(m);
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int pos = seen + incl - mine;
            // this round writes the settled codes (round 0 only) and the unsettled ones of its window
            unsigned wr = lo == 0 ? (~m & 0xFu) : 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (m >> e & 1u) {
                    if (pos >= lo && pos < lo + RQ_LIST) {
                        c[e] = a4_code(val[pos - lo], s);
                        wr |= 1u << e;
                    }
                    ++pos;
                }
            seen += __shfl_sync(0xffffffffu, incl, 31);
            if (j < nv && wr) {
                // dequantized value, rounded exactly as codes.astype(f32) * scales (model.py:379-381)
                if (wr == 0xFu) {
                    reinterpret_cast<char4 *>(crow)[j] = make_char4(c[0], c[1], c[2], c[3]);
                    if (drow != nullptr)
                        drow[j] = make_float4(__fmul_rn((float)c[0], s), __fmul_rn((float)c[1], s),
                                              __fmul_rn((float)c[2], s), __fmul_rn((float)c[3], s));
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (wr >> e & 1u) {
                            crow[4 * j + e] = c[e];
                            if (drow != nullptr) deq[row * d + 4 * j + e] = __fmul_rn((float)c[e], s);
                        }
                }
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (wr >> e & 1u) csum += c[e];
            }
        }
        if (lo + RQ_LIST >= total) break;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if (lane == 0) {
        if (tsum != nullptr) tsum[row] = csum;
        if (recomputed != nullptr) atomicAdd(recomputed, n_chain);
    }
}

// Single-kernel form: one warp per row does pick, chains and codes (the fallback when the
// scheduled form's scratch does not fit).
template <int DT>
__global__ void __launch_bounds__(RQ_WARPS * 32) rot_certify_kernel(
    const float *__restrict__ v, const void *__restrict__ x, const float *__restrict__ Rt, int64_t n, int64_t d,
    float eps_rel, int8_t *__restrict__ codes, float *__restrict__ scales, int *__restrict__ nonfinite,
    float *__restrict__ deq, int32_t *__restrict__ tsum, int32_t *__restrict__ zero, int n_zero,
    int *__restrict__ recomputed) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int32_t idx_sh[RQ_WARPS][RQ_LIST];
    __shared__ float val_sh[RQ_WARPS][RQ_LIST];
    if (blockIdx.x == 0)  // counters the next kernels accumulate into (route counts)
        for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * RQ_WARPS + warp;
    if (row >= n) return;
    int32_t *idx = idx_sh[warp];
    float *val = val_sh[warp];
    const float4 *v4 = reinterpret_cast<const float4 *>(v + row * d);
    const RqRow rr(rq_row_max(v4, d / 4, lane, nonfinite), eps_rel);
    const int total = rq_collect(v4, d / 4, lane, 0, idx, [&](float a) { return rr.picked(a); });
    if (total <= RQ_LIST) {
        rq_resolve<DT>(x, row, d, Rt, idx, val, total, lane);
        rq_finish_fast(v, row, d, lane, rr, idx, val, total, codes, scales, deq, tsum, recomputed);
    } else {
        rq_general<DT>(v, x, Rt, row, d, lane, rr, idx, val, codes, scales, deq, tsum, recomputed);
    }
}

// ---- Scheduled form (three kernels).  The single-kernel form runs ~12 chains per row on 12 lanes
// of the row's warp, each lane streaming its own R^T row: 50k R^T rows (800 MB, mostly DRAM) per PH
// step.  Here the chains are grouped by column: (1) per row, pick the elements and push one task per
// element into its column's bucket; (2) one warp per column runs that column's chains, the R^T row
// shared by all lanes (warp-uniform loads: each R^T row read once) and each lane reading its token's
// x row (L2-resident); (3) per row, the exact max, the scale and the codes from the values.
struct RqScratch {
    int32_t *col_cnt;  // [d] tasks pushed per column, then [d] = overflow count
    int32_t *tok_cnt;  // [n] picked elements of the row, -1: general path
    float *tok_mx;     // [n] approximate row max
    int32_t *tok_idx;  // [n][RQ_LIST] picked element indices (ascending)
    float *tok_val;    // [n][RQ_LIST] their exact values
    int32_t *bucket;   // [d][cap] tasks (row << 8 | slot)
    int32_t *ovf;      // [ovf_cap] tasks past a full bucket
    int64_t ovf_cap;
    int cap;           // bucket capacity: n when it fits (a column may be picked by every row)
};

static int64_t rq_scratch_layout(int64_t n, int64_t d, int64_t cap, void *base, RqScratch *sc) {
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        const int64_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    const int64_t o_cc = take((d + 1) * 4), o_tc = take(n * 4), o_mx = take(n * 4);
    const int64_t o_ti = take(n * RQ_LIST * 4), o_tv = take(n * RQ_LIST * 4), o_b = take(d * cap * 4);
    const int64_t ovf_cap = 4 * n + 1024;
    const int64_t o_o = take(ovf_cap * 4);
    if (sc != nullptr) {
        char *b = reinterpret_cast<char *>(base);
        sc->col_cnt = reinterpret_cast<int32_t *>(b + o_cc);
        sc->tok_cnt = reinterpret_cast<int32_t *>(b + o_tc);
        sc->tok_mx = reinterpret_cast<float *>(b + o_mx);
        sc->tok_idx = reinterpret_cast<int32_t *>(b + o_ti);
        sc->tok_val = reinterpret_cast<float *>(b + o_tv);
        sc->bucket = reinterpret_cast<int32_t *>(b + o_b);
        sc->ovf = reinterpret_cast<int32_t *>(b + o_o);
        sc->ovf_cap = ovf_cap;
        sc->cap = (int)cap;
    }
    return off;
}

__global__ void __launch_bounds__(RQ_WARPS * 32) rq_pick_kernel(const float *__restrict__ v, int64_t n, int64_t d,
                                                                 float eps_rel, int *__restrict__ nonfinite,
                                                                 RqScratch sc) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int32_t idx_sh[RQ_WARPS][RQ_LIST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * RQ_WARPS + warp;
    if (row >= n) return;
    int32_t *idx = idx_sh[warp];
    const float4 *v4 = reinterpret_cast<const float4 *>(v + row * d);
    const float mx = rq_row_max(v4, d / 4, lane, nonfinite);
    const RqRow rr(mx, eps_rel);
    const int total = rq_collect(v4, d / 4, lane, 0, idx, [&](float a) { return rr.picked(a); });
    bool ok = total <= RQ_LIST;
    if (ok) {
        for (int i = lane; i < total; i += 32) {
            const int32_t j = idx[i];
            sc.tok_idx[row * RQ_LIST + i] = j;
            const int32_t task = (int32_t)(row << 8) | i;
            const int pos = atomicAdd(sc.col_cnt + j, 1);
            if (pos < sc.cap) {
                sc.bucket[(int64_t)j * sc.cap + pos] = task;
            } else {
                const int opos = atomicAdd(sc.col_cnt + d, 1);
                if (opos < sc.ovf_cap)
                    sc.ovf[opos] = task;
                else
                    ok = false;  // lost task: the row takes the general path
            }
        }
        ok = __all_sync(0xffffffffu, ok);
    }
    if (lane == 0) {
        sc.tok_cnt[row] = ok ? total : -1;
        sc.tok_mx[row] = mx;
    }
}

// One warp per column: the lanes share j, so each R^T row is read once per call, and each lane runs
// the chain of one task (its token's x row, L2-resident).  The operands stream through a per-warp
// shared-memory ring (cp.async, RC_S stages of RC_K columns): the chain's dependent adds then
// overlap the loads of the next stages.  (Direct loads: one memory latency per 32 columns, 167 us
// at PH; one task per thread in column order: 381 us, a quarter of the loads in flight.)
#ifndef RC_K_
#define RC_K_ 32
#endif
#ifndef RC_S_
#define RC_S_ 4
#endif
constexpr int RC_K = RC_K_;  // chain steps (columns of x / R^T) per stage
constexpr int RC_S = RC_S_;  // ring stages
constexpr int RC_DMAX = 8192;  // columns of the in-CTA work-unit scan (shared memory)
template <int DT>
struct RcCfg {
    static constexpr int XB = DT == CQ_DTYPE_F32 ? 4 : 2;
#ifndef RC_W_
#define RC_W_ 16
#endif
    static constexpr int WPC = DT == CQ_DTYPE_F32 ? RC_W_ / 2 : RC_W_;  // warps per CTA (one CTA per SM)
    static constexpr int XLS = RC_K * XB + 16;             // a lane's x chunk, padded: conflict-free LDS.128
    static constexpr int STAGE = 32 * XLS + 2 * RC_K * 4;   // x chunks of 32 lanes, then two R^T chunks
    static constexpr int SMEM = WPC * RC_S * STAGE;
};

__device__ __forceinline__ void rc_cp16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}

template <int DT>
__global__ void __launch_bounds__(RcCfg<DT>::WPC * 32) rq_chain_kernel(const void *__restrict__ x,
                                                                      const float *__restrict__ Rt, int64_t d,
                                                                      RqScratch sc) {
    using C = RcCfg<DT>;
    constexpr int XCH = RC_K * C::XB / 16;  // 16-byte pieces of a lane's x chunk
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    extern __shared__ __align__(16) uint8_t rc_sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t *ring = rc_sm + (size_t)warp * RC_S * C::STAGE;
    int32_t *off = reinterpret_cast<int32_t *>(rc_sm + C::SMEM);  // [d + 1] work units before column c
    // work units: (column, round of 32 tasks); exclusive scan of ceil(cnt / 32) over the columns,
    // thread i owning columns [i * per, (i + 1) * per)
    {
        __shared__ int32_t wsum[C::WPC];
        const int per = (int)((d + blockDim.x - 1) / blockDim.x);
        const int c0 = threadIdx.x * per, c1 = min((int)d, c0 + per);
        int run = 0;
        for (int c = c0; c < c1; ++c) {
            off[c] = run;
            run += (min(sc.col_cnt[c], sc.cap) + 15) >> 4;
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int base = incl - run;
        for (int w = 0; w < warp; ++w) base += wsum[w];
        for (int c = c0; c < c1; ++c) off[c] += base;
        if (threadIdx.x == blockDim.x - 1) off[d] = base + run;
        __syncthreads();
    }
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nst = d / RC_K;
    // a half-warp per unit (column, round of 16 tasks): ~12 tasks per column at PH, so a whole warp
    // per column left most lanes idle; each half has its own R^T chunk in the stage
    const int half = lane >> 4, hl = lane & 15;
    for (int64_t up = gw; 2 * up < off[d]; up += nw) {
        const int64_t u = 2 * up + half;
        const bool uvalid = u < off[d];
        int j;
        {
            // the last column with off[c] <= u (columns without units share the next one's offset)
            int lo = 0, hi = (int)d - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (off[mid] <= u) lo = mid; else hi = mid - 1;
            }
            j = lo;
        }
        const int cnt = min(sc.col_cnt[j], sc.cap);
        const float *rg = Rt + (int64_t)j * d;
        {
            const int r0 = (int)(u - off[j]) * 16;
            const bool act = uvalid && r0 + hl < cnt;
            const int32_t task = act ? sc.bucket[(int64_t)j * sc.cap + r0 + hl] : 0;
            const int64_t row = task >> 8;
            const uint8_t *xg = reinterpret_cast<const uint8_t *>(x) + row * d * C::XB;
            // the warp loads its rows' x chunks cooperatively: piece i of this lane is piece q of row r
            // (XCH consecutive lanes per row), so a copy instruction touches 32 / XCH rows instead of 32
            // scattered 16-byte pieces (the L1 tag lookups of scattered pieces bound the kernel)
            const uint8_t *xsrc[XCH];
            int xdst[XCH];
            bool xok[XCH];
#pragma unroll
            for (int i = 0; i < XCH; ++i) {
                const int pc = lane + 32 * i, r = pc / XCH, q = pc - r * XCH;
                const uint64_t rp = __shfl_sync(0xffffffffu, (uint64_t)xg, r);
                xok[i] = __shfl_sync(0xffffffffu, (int)act, r) != 0;
                xsrc[i] = reinterpret_cast<const uint8_t *>(rp) + q * 16;
                xdst[i] = r * C::XLS + q * 16;
            }
            auto issue = [&](int64_t g) {
                if (g < nst) {
                    uint8_t *st = ring + (g % RC_S) * C::STAGE;
#pragma unroll
                    for (int i = 0; i < XCH; ++i)
                        if (xok[i]) rc_cp16(st + xdst[i], xsrc[i] + g * RC_K * C::XB);
                    if (uvalid && hl < RC_K / 4)
                        rc_cp16(st + 32 * C::XLS + half * RC_K * 4 + hl * 16, rg + g * RC_K + hl * 4);
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
#pragma unroll
            for (int g = 0; g < RC_S - 1; ++g) issue(g);
            float acc = 0.0f;
            for (int64_t g = 0; g < nst; ++g) {
                issue(g + RC_S - 1);
                asm volatile("cp.async.wait_group %0;" ::"n"(RC_S - 1) : "memory");
                __syncwarp();
                const uint8_t *st = ring + (g % RC_S) * C::STAGE;
                const float4 *r4 = reinterpret_cast<const float4 *>(st + 32 * C::XLS + half * RC_K * 4);
                const uint4 *x4 = reinterpret_cast<const uint4 *>(st + lane * C::XLS);
                if (act) {
                    // the reference's order: k ascending, separate fp32 multiply and add (rq_chain)
#pragma unroll
                    for (int q = 0; q < XCH; ++q) {
                        const uint4 u = x4[q];
                        float xv[8];
                        int nx;
                        if (DT == CQ_DTYPE_F32) {
                            xv[0] = __uint_as_float(u.x), xv[1] = __uint_as_float(u.y);
                            xv[2] = __uint_as_float(u.z), xv[3] = __uint_as_float(u.w);
                            nx = 4;
                        } else {
                            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                xv[2 * e] = __uint_as_float(w[e] << 16);
                                xv[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
                            }
                            nx = 8;
                        }
                        const int k0 = q * nx;  // first column of this piece within the stage
#pragma unroll
                        for (int e = 0; e < 8; e += 4) {
                            if (e < nx) {
                                const float4 rv = r4[(k0 + e) / 4];
                                acc = __fadd_rn(acc, __fmul_rn(xv[e], rv.x));
                                acc = __fadd_rn(acc, __fmul_rn(xv[e + 1], rv.y));
                                acc = __fadd_rn(acc, __fmul_rn(xv[e + 2], rv.z));
                                acc = __fadd_rn(acc, __fmul_rn(xv[e + 3], rv.w));
                            }
                        }
                    }
                }
                __syncwarp();  // every lane is done with this stage before it is refilled
            }
            if (act) sc.tok_val[row * RQ_LIST + (task & 255)] = acc;
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    // the overflow tasks, one lane each
    const int64_t n_ovf = sc.col_cnt[d] < sc.ovf_cap ? (int64_t)sc.col_cnt[d] : sc.ovf_cap;
    for (int64_t t = gw * 32 + lane; t < n_ovf; t += nw * 32) {
        const int32_t task = sc.ovf[t];
        const int64_t row = task >> 8;
        const int slot = task & 255;
        sc.tok_val[row * RQ_LIST + slot] = rq_chain<DT>(x, row, d, Rt, sc.tok_idx[row * RQ_LIST + slot]);
    }
}

template <int DT>
__global__ void __launch_bounds__(RQ_WARPS * 32) rq_finish_kernel(
    const float *__restrict__ v, const void *__restrict__ x, const float *__restrict__ Rt, int64_t n, int64_t d,
    float eps_rel, RqScratch sc, int8_t *__restrict__ codes, float *__restrict__ scales,
    float *__restrict__ deq, int32_t *__restrict__ tsum, int32_t *__restrict__ zero, int n_zero,
    int *__restrict__ recomputed) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int32_t idx_sh[RQ_WARPS][RQ_LIST];
    __shared__ float val_sh[RQ_WARPS][RQ_LIST];
    if (blockIdx.x == 0)  // counters the next kernels accumulate into (route counts)
        for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * RQ_WARPS + warp;
    if (row >= n) return;
    int32_t *idx = idx_sh[warp];
    float *val = val_sh[warp];
    const RqRow rr(sc.tok_mx[row], eps_rel);
    const int total = sc.tok_cnt[row];
    if (total < 0) {
        rq_general<DT>(v, x, Rt, row, d, lane, rr, idx, val, codes, scales, deq, tsum, recomputed);
        return;
    }
    for (int i = lane; i < total; i += 32) {
        idx[i] = sc.tok_idx[row * RQ_LIST + i];
        val[i] = sc.tok_val[row * RQ_LIST + i];
    }
    __syncwarp();
    rq_finish_fast(v, row, d, lane, rr, idx, val, total, codes, scales, deq, tsum, recomputed);
}

// The chain kernel's grid: one CTA per SM (its rings fill the shared memory), work units grid-strided.
static int rc_grid() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}

// v (n, d) f32 from rot_gemm, x the layer input (dtype), Rt = R^T (d, d) f32.  scratch (nullable):
// device memory free for this call (the rotation's consumed operand planes); the scheduled form
// runs when it fits, else the single-kernel form (CQ_ROT_CERT_SCHED=0 forces that).
cq_status rot_certify(const float *v, const void *x, int dtype, const float *Rt, int64_t n, int64_t d, int8_t *codes,
                      float *scales, int *nonfinite, float *deq, int32_t *tsum, int32_t *zero, int n_zero,
                      int *recomputed, void *scratch, int64_t scratch_bytes, cudaStream_t st) {
    if (n == 0) return CQ_OK;
    if (d % 8) {
        set_error("rotation: certified quantizer needs d_model % 8 == 0");
        return CQ_ERR_UNSUPPORTED;
    }
    const char *env = getenv("CQ_ROT_CERT_EPS");  // tests / experiments: the recompute band
    const float eps_rel = env ? (float)atof(env) : 1.5e-4f;
    static int sched_env = -1;
    if (sched_env < 0) {
        const char *e = getenv("CQ_ROT_CERT_SCHED");
        sched_env = e ? atoi(e) : 1;
    }
    const unsigned grid = (unsigned)ceil_div(n, RQ_WARPS);
    const bool bf = dtype == CQ_DTYPE_BF16;
    // bucket capacity: n (no overflow) when the scratch holds it, else what fits (>= 64)
    int64_t cap = n;
    if (scratch != nullptr && rq_scratch_layout(n, d, cap, nullptr, nullptr) > scratch_bytes)
        cap = (scratch_bytes - rq_scratch_layout(n, d, 0, nullptr, nullptr)) / (4 * d) - 64;
    if (sched_env && scratch != nullptr && n < (1LL << 23) && d % RC_K == 0 && d <= RC_DMAX && cap >= std::min<int64_t>(n, 64) &&
        rq_scratch_layout(n, d, cap, nullptr, nullptr) <= scratch_bytes) {
        RqScratch sc;
        rq_scratch_layout(n, d, cap, scratch, &sc);
        if (cudaMemsetAsync(sc.col_cnt, 0, (d + 1) * 4, st) != cudaSuccess) return check_launch("rotation_certify");
        launch_pdl(rq_pick_kernel, grid, RQ_WARPS * 32, 0, st, v, n, d, eps_rel, nonfinite, sc);
        CQ_TRY(check_launch("rotation_certify_pick"));
        // one warp per column; the smem opt-in is per device: set on every launch
        if (bf) {
            using C = RcCfg<CQ_DTYPE_BF16>;
            const int sm = C::SMEM + (int)(d + 1) * 4;
            cudaFuncSetAttribute(rq_chain_kernel<CQ_DTYPE_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            launch_pdl(rq_chain_kernel<CQ_DTYPE_BF16>, (unsigned)rc_grid(), C::WPC * 32, (size_t)sm, st, x, Rt, d, sc);
        } else {
            using C = RcCfg<CQ_DTYPE_F32>;
            const int sm = C::SMEM + (int)(d + 1) * 4;
            cudaFuncSetAttribute(rq_chain_kernel<CQ_DTYPE_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
            launch_pdl(rq_chain_kernel<CQ_DTYPE_F32>, (unsigned)rc_grid(), C::WPC * 32, (size_t)sm, st, x, Rt, d, sc);
        }
        CQ_TRY(check_launch("rotation_certify_chains"));
        if (bf)
            launch_pdl(rq_finish_kernel<CQ_DTYPE_BF16>, grid, RQ_WARPS * 32, 0, st, v, x, Rt, n, d, eps_rel, sc, codes,
                       scales, deq, tsum, zero, n_zero, recomputed);
        else
            launch_pdl(rq_finish_kernel<CQ_DTYPE_F32>, grid, RQ_WARPS * 32, 0, st, v, x, Rt, n, d, eps_rel, sc, codes,
                       scales, deq, tsum, zero, n_zero, recomputed);
        return check_launch("rotation_certify_finish");
    }
    if (bf)
        launch_pdl(rot_certify_kernel<CQ_DTYPE_BF16>, grid, RQ_WARPS * 32, 0, st, v, x, Rt, n, d, eps_rel, codes, scales,
                   nonfinite, deq, tsum, zero, n_zero, recomputed);
    else
        launch_pdl(rot_certify_kernel<CQ_DTYPE_F32>, grid, RQ_WARPS * 32, 0, st, v, x, Rt, n, d, eps_rel, codes, scales,
                   nonfinite, deq, tsum, zero, n_zero, recomputed);
    return check_launch("rotation_certify");
}

// R (d, d) -> R^T, 32 x 32 tiles through shared memory.
__global__ void transpose_kernel(const float *__restrict__ R, int64_t d, float *__restrict__ Rt) {
    __shared__ float t[32][33];
    const int64_t bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y)
        if (by + i < d && bx + threadIdx.x < d) t[i][threadIdx.x] = R[(by + i) * d + bx + threadIdx.x];
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y)
        if (bx + i < d && by + threadIdx.x < d) Rt[(bx + i) * d + by + threadIdx.x] = t[threadIdx.x][i];
}

cq_status transpose_f32(const float *R, int64_t d, float *Rt, cudaStream_t st) {
    const dim3 grid((unsigned)ceil_div(d, 32), (unsigned)ceil_div(d, 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(R, d, Rt);
    return check_launch("rotation_transpose");
}

}  // namespace cq
