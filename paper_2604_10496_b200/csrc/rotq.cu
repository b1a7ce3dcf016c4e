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
    for (int64_t base = 0; base < nv; base += 32) {
        const int64_t j = base + lane;
        unsigned m = 0;
        if (j < nv) {
            const float4 a = v4[j];
            m = (pick(a.x) ? 1u : 0u) | (pick(a.y) ? 2u : 0u) | (pick(a.z) ? 4u : 0u) | (pick(a.w) ? 8u : 0u);
        }
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
    __syncwarp();
    return total;
}

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
    const int64_t nv = d / 4;

    // ---- 1. approximate max
    float mx = 0.0f;
    bool bad = false;
    for (int64_t j = lane; j < nv; j += 32) {
        const float4 a = v4[j];
        bad |= !isfinite(a.x) || !isfinite(a.y) || !isfinite(a.z) || !isfinite(a.w);
        mx = fmaxf(fmaxf(mx, fabsf(a.x)), fmaxf(fabsf(a.y), fmaxf(fabsf(a.z), fabsf(a.w))));
    }
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad) && lane == 0 && nonfinite != nullptr) atomicExch(nonfinite, 1);
    const float eps = eps_rel * mx;
    const float thr = mx > 0.0f ? mx - 2.0f * eps : INFINITY;  // an all-zero row has no candidates
    auto is_cand = [&](float a) { return fabsf(a) >= thr; };
    int n_chain = 0;

    // ---- fast path: one round of chains.  The exact max lies within eps of mx, so the scale lies in
    // [s_lo, s_hi]; an element whose code is the same at both ends of its value band under both
    // scales is settled whatever the exact scale, the others and the max candidates are recomputed.
    {
        const float s_lo = a4_scale(fmaxf(mx - eps, 0.0f)), s_hi = a4_scale(mx + eps);
        const float r_lo = 1.0f / s_lo, r_hi = 1.0f / s_hi;  // s_lo <= s <= s_hi
        auto picked = [&](float a) {
            if (is_cand(a)) return true;
            const float lo = a - eps, hi = a + eps;
            const float tmin = fminf(lo * r_lo, lo * r_hi), tmax = fmaxf(hi * r_lo, hi * r_hi);
            return rq_code_t(tmin - RQ_SLACK) != rq_code_t(tmax + RQ_SLACK);
        };
        const int total = rq_collect(v4, nv, lane, 0, idx, picked);
        if (total <= RQ_LIST) {
            rq_resolve<DT>(x, row, d, Rt, idx, val, total, lane);
            float mxe = 0.0f;
            for (int i = lane; i < total; i += 32)
                if (is_cand(v[row * d + idx[i]])) mxe = fmaxf(mxe, fabsf(val[i]));
            n_chain = total;
            mxe = warp_max(mxe);
            const float sc = a4_scale(mxe);  // quant.py:76-100 on the exact maximum
            const float rc = 1.0f / sc;
            if (lane == 0) scales[row] = sc;
            int8_t *crow = codes + row * d;
            float4 *drow = deq != nullptr ? reinterpret_cast<float4 *>(deq + row * d) : nullptr;
            int csum = 0, seen = 0;
            for (int64_t base = 0; base < nv; base += 32) {
                const int64_t j = base + lane;
                int8_t c[4] = {0, 0, 0, 0};
                unsigned m = 0;
                if (j < nv) {
                    const float4 a = v4[j];
                    const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        m |= picked(av[e]) ? 1u << e : 0u;
                        c[e] = (int8_t)rq_code_t(av[e] * rc);  // settled: equals a4_code(av[e], sc)
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
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (m >> e & 1u) c[e] = a4_code(val[pos++], sc);
                seen += __shfl_sync(0xffffffffu, incl, 31);
                if (j < nv) {
                    reinterpret_cast<char4 *>(crow)[j] = make_char4(c[0], c[1], c[2], c[3]);
                    csum += c[0] + c[1] + c[2] + c[3];
                    // dequantized value, rounded exactly as codes.astype(f32) * scales (model.py:379-381)
                    if (drow != nullptr)
                        drow[j] = make_float4(__fmul_rn((float)c[0], sc), __fmul_rn((float)c[1], sc),
                                              __fmul_rn((float)c[2], sc), __fmul_rn((float)c[3], sc));
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
            if (lane == 0) {
                if (tsum != nullptr) tsum[row] = csum;
                if (recomputed != nullptr) atomicAdd(recomputed, n_chain);
            }
            return;
        }
    }

    // ---- general path (more than RQ_LIST picked elements): the exact max over the candidates first,
    // in rounds, then the unsettled elements under the exact scale, in rounds
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

    // ---- 2. codes: settled where v_tc +- eps give one code, else from the exact chain value
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

// v (n, d) f32 from rot_gemm, x the layer input (dtype), Rt = R^T (d, d) f32.
cq_status rot_certify(const float *v, const void *x, int dtype, const float *Rt, int64_t n, int64_t d, int8_t *codes,
                      float *scales, int *nonfinite, float *deq, int32_t *tsum, int32_t *zero, int n_zero,
                      int *recomputed, cudaStream_t st) {
    if (n == 0) return CQ_OK;
    if (d % 8) {
        set_error("rotation: certified quantizer needs d_model % 8 == 0");
        return CQ_ERR_UNSUPPORTED;
    }
    const char *env = getenv("CQ_ROT_CERT_EPS");  // tests / experiments: the recompute band
    const float eps_rel = env ? (float)atof(env) : 1.5e-4f;
    const unsigned grid = (unsigned)ceil_div(n, RQ_WARPS);
    const size_t smem = 0;
    if (dtype == CQ_DTYPE_BF16)
        launch_pdl(rot_certify_kernel<CQ_DTYPE_BF16>, grid, RQ_WARPS * 32, smem, st, v, x, Rt, n, d, eps_rel, codes, scales,
                   nonfinite, deq, tsum, zero, n_zero, recomputed);
    else
        launch_pdl(rot_certify_kernel<CQ_DTYPE_F32>, grid, RQ_WARPS * 32, smem, st, v, x, Rt, n, d, eps_rel, codes, scales,
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
