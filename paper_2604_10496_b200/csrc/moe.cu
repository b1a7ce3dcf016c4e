// MoE layer operator: the MoE block of model.forward (model.py:377-404) on the
// device, stage by stage, all on the caller's stream with no host sync:
//
//   [rotation x@R] -> A4 quantize (quant.py:89-100) -> ordered router logits
//   -> top-k + counts -> permute into expert segments -> gather codes
//   -> grouped gate|up LUT GEMM with fused silu(a)*b  (model.py:392-396)
//   -> A4 re-quantize of the hidden               (model.py:397-398)
//   -> grouped down LUT GEMM                      (model.py:399)
//   -> weighted combine, experts ascending        (model.py:389-401)
//   [+ shared experts, weight 1 — builder-defined, SURVEY §8(a) a18]
#include <cooperative_groups.h>

#include "common.cuh"
#include "route_perm.cuh"

namespace cq {

// --- stage kernels defined in other units
cq_status quantize_a4(const void *, int, int64_t, int64_t, int8_t *, float *, int *, float *, cudaStream_t,
                      int32_t *tsum = nullptr, int32_t *zero = nullptr, int n_zero = 0);
cq_status router_logits(const int8_t *, const float *, const float *, const float *, int64_t, int64_t, int64_t,
                        float *, cudaStream_t);
cq_status router_fused(const float *, const float *, int64_t, int64_t, int64_t, float *, int32_t *, float *, int64_t,
                       cudaStream_t, bool *);
cq_status router_fused_quant(const void *, int, int8_t *, float *, int *, int32_t *, int32_t *, int, float *,
                             const float *, int64_t, int64_t, int64_t, float *, int32_t *, float *, int64_t,
                             cudaStream_t, bool *);
cq_status topk(const float *, int64_t, int64_t, int64_t, int32_t *, float *, int32_t *, int64_t, int64_t,
               cudaStream_t);
bool permute_counts_itself(int64_t n);
cq_status permute(const int32_t *, int32_t *, int64_t, int64_t, int64_t, int64_t, int32_t *,
                  int32_t *, int32_t *, int32_t *, cudaStream_t);
cq_status gather_rows(const int8_t *, const float *, const int32_t *, const int32_t *, int64_t, int64_t,
                      int64_t, int8_t *, float *, cudaStream_t);
cq_status lut_f32_grouped(const int8_t *, const float *, const int32_t *, int64_t, int64_t,
                          const uint8_t *, const float *, const uint8_t *, const float *, int64_t,
                          int64_t, int64_t, float *, cudaStream_t);
bool f32_path_ok(int64_t d_in, int64_t g);
cq_status ordered_lut(const int8_t *, const float *, const int32_t *, int64_t, int64_t, int64_t, const uint8_t *,
                      const float *, int64_t, int64_t, int64_t, float *, cudaStream_t);
cq_status ordered_matmul(const void *, int, const float *, int64_t, int64_t, int64_t, float *, cudaStream_t);
bool umma_ok(int64_t d_in, int64_t d_out, int64_t g);
cq_status lut_umma_grouped(const int8_t *, int8_t *, const float *, const int32_t *, int64_t, int64_t, int64_t,
                           const cq_expert_site *, float *, const cq_expert_site *, float *, int64_t, int64_t,
                           cudaStream_t, const UmmaIn &in = UmmaIn{});
int64_t umma_b_bytes(int64_t rows, int64_t d_in);
int32_t *umma_row_sums(int8_t *bbuf, int64_t rows, int64_t d_in);
int umma_geo_ck(int64_t rows, int64_t n_seg, int64_t d_in, int64_t d_out, int mats, int planes);
UmmaBOut umma_b_out(int8_t *bbuf, int64_t rows, int64_t d_in, int ck);
int64_t rot_tc_act_bytes(int64_t n, int64_t d);
const float *rot_tc_transposed(const void *prepared, int64_t d);
cq_status rot_certify(const float *v, const void *x, int dtype, const float *Rt, int64_t n, int64_t d, int8_t *codes,
                      float *scales, int *nonfinite, float *deq, int32_t *tsum, int32_t *zero, int n_zero,
                      int *recomputed, void *scratch, int64_t scratch_bytes, cudaStream_t st);
cq_status rot_tc_apply(const void *x, int dtype, int64_t n, int64_t d, const void *prepared, void *act, float *v,
                       cudaStream_t st);

// h = silu(a) * b (model.py:396) fused with the per-row A4 re-quantization of
// h (model.py:397-398, quant.py:89-100): pass 1 forms h in place of a and its
// max|h|; pass 2 writes the codes.  One CTA per row; same scale/rounding recipe
// as the input quantizer.
__global__ void __launch_bounds__(256) silu_quant_kernel(float *__restrict__ a, const float *__restrict__ b,
                                                          int64_t ff, int8_t *__restrict__ codes,
                                                          float *__restrict__ scales,
                                                          const int32_t *__restrict__ live,
                                                          int32_t *__restrict__ sums, int *__restrict__ nonfinite) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t row = blockIdx.x;
    if (live != nullptr && row >= *live) return;
    float *ar = a + row * ff;
    const float *br = b + row * ff;
    float mx = 0.0f;
    bool bad = false;
    for (int64_t j = threadIdx.x; j < ff; j += blockDim.x) {
        const float h = __fmul_rn(silu_fast(ar[j]), br[j]);
        ar[j] = h;
        mx = fmaxf(mx, fabsf(h));
        bad |= !(fabsf(h) <= FLT_MAX);
    }
    if (nonfinite != nullptr && __syncthreads_or(bad) && threadIdx.x == 0) atomicExch(nonfinite, 1);
    __shared__ float red[8];
    __shared__ float s_sh;
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
        float m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0) {
            s_sh = a4_scale(m);
            scales[row] = s_sh;
        }
    }
    __syncthreads();
    const float s = s_sh;
    int cs = 0;
    for (int64_t j = threadIdx.x; j < ff; j += blockDim.x) {
        const int8_t c = a4_code(ar[j], s);
        codes[row * ff + j] = c;
        cs += c;
    }
    if (sums != nullptr) {  // the down GEMM's unsigned-digit bias term (row_sums_kernel's value)
        const int t = block_sum_int(cs);
        if (threadIdx.x == 0) sums[row] = t;
    }
}

// Same, register-resident: 512 threads x V float4 cover the row (ff % 4 == 0,
// ff <= 8192 V), so a and b are read once with 16-byte loads and h never
// round-trips through memory before it is quantized.
template <int V>
__global__ void __launch_bounds__(512, V == 4 ? 4 : 1) silu_quant_vec_kernel(float *__restrict__ a, const float *__restrict__ b,
                                                              int64_t ff, int8_t *__restrict__ codes,
                                                              float *__restrict__ scales,
                                                              const int32_t *__restrict__ live,
                                                              int32_t *__restrict__ sums, int keep,
                                                              int *__restrict__ nonfinite, UmmaBOut bo) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    if (blockIdx.x == 0 && bo.zero != nullptr)  // the counters the B build would have zeroed
        for (int i = threadIdx.x; i < bo.n_zero; i += blockDim.x) bo.zero[i] = 0;
    const int64_t row = blockIdx.x;
    if (live != nullptr && row >= *live) return;
    float4 *ar = reinterpret_cast<float4 *>(a + row * ff);
    const float4 *br = reinterpret_cast<const float4 *>(b + row * ff);
    const int nv = (int)(ff >> 2);
    float4 h[V];
    uint32_t mb = 0;  // max |h| as bits: ordered like the floats, and inf / NaN (flagged) above every finite value
#pragma unroll
    for (int u = 0; u < V; ++u) {
        const int j = threadIdx.x + u * (int)blockDim.x;
        if (j < nv) {
            const float4 x = ar[j], y = br[j];
            h[u] = make_float4(__fmul_rn(silu_fast(x.x), y.x), __fmul_rn(silu_fast(x.y), y.y),
                               __fmul_rn(silu_fast(x.z), y.z), __fmul_rn(silu_fast(x.w), y.w));
            if (keep) ar[j] = h[u];  // h itself only for tracing (CQ_FLAG_KEEP_HIDDEN)
            mb = max(mb, abs_bits4(h[u]));
        }
    }
    if (nonfinite != nullptr && __syncthreads_or(mb >= 0x7f800000u) && threadIdx.x == 0) atomicExch(nonfinite, 1);
    __shared__ uint32_t red[16];
    __shared__ float s_sh;
    mb = __reduce_max_sync(0xffffffffu, mb);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mb;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
        m = __reduce_max_sync(0xffffffffu, m);
        if (threadIdx.x == 0) {
            s_sh = a4_scale(__uint_as_float(m));
            scales[row] = s_sh;
        }
    }
    __syncthreads();
    const float s = s_sh;
    const float rs = __frcp_rn(s);
    char4 *cr = codes != nullptr ? reinterpret_cast<char4 *>(codes + row * ff) : nullptr;
    int cs = 0;
#pragma unroll
    for (int u = 0; u < V; ++u) {
        const int j = threadIdx.x + u * (int)blockDim.x;
        if (j < nv) {
            const char4 c = make_char4(a4_code_rcp(h[u].x, s, rs), a4_code_rcp(h[u].y, s, rs), a4_code_rcp(h[u].z, s, rs),
                                       a4_code_rcp(h[u].w, s, rs));
            if (cr != nullptr) cr[j] = c;
            if (bo.dst != nullptr) *reinterpret_cast<char4 *>(bo.dst + bo.off(row, 4 * (int64_t)j)) = c;
            cs += c.x + c.y + c.z + c.w;
        }
    }
    if (sums != nullptr) {
        const int t = block_sum_int(cs);
        if (threadIdx.x == 0) sums[row] = t;
    }
}

// Few rows (decode: a row per route): one CTA per row leaves SMs idle and
// serialises each row's load -> max -> quantize.  Here a cluster of CL CTAs
// shares a row, each taking ff / CL columns; the row max is combined through
// distributed shared memory.  Same per-element math as silu_quant_vec_kernel.
template <int V, int CL>
__global__ void __launch_bounds__(256) silu_quant_cl_kernel(float *__restrict__ a, const float *__restrict__ b,
                                                             int64_t ff, int8_t *__restrict__ codes,
                                                             float *__restrict__ scales,
                                                             const int32_t *__restrict__ live,
                                                             int32_t *__restrict__ sums, int keep,
                                                             int *__restrict__ nonfinite, UmmaBOut bo) {
    namespace cg = cooperative_groups;
    griddep_wait();
    if (blockIdx.x == 0 && bo.zero != nullptr)  // the counters the B build would have zeroed
        for (int i = threadIdx.x; i < bo.n_zero; i += blockDim.x) bo.zero[i] = 0;
    const int64_t row = blockIdx.x / CL;
    if (live != nullptr && row >= *live) return;  // uniform over the cluster (one row)
    cg::cluster_group cluster = cg::this_cluster();
    const int part = (int)cluster.block_rank();
    const int64_t seg = ff / CL;
    float4 *ar = reinterpret_cast<float4 *>(a + row * ff + part * seg);
    const float4 *br = reinterpret_cast<const float4 *>(b + row * ff + part * seg);
    const int nv = (int)(seg >> 2);
    float4 h[V];
    uint32_t mb = 0;  // max |h| as bits (see silu_quant_vec_kernel)
#pragma unroll
    for (int u = 0; u < V; ++u) {
        const int j = threadIdx.x + u * 256;
        if (j < nv) {
            const float4 x = ar[j], y = br[j];
            h[u] = make_float4(__fmul_rn(silu_fast(x.x), y.x), __fmul_rn(silu_fast(x.y), y.y),
                               __fmul_rn(silu_fast(x.z), y.z), __fmul_rn(silu_fast(x.w), y.w));
            if (keep) ar[j] = h[u];  // h itself only for tracing (CQ_FLAG_KEEP_HIDDEN)
            mb = max(mb, abs_bits4(h[u]));
        }
    }
    if (nonfinite != nullptr && __syncthreads_or(mb >= 0x7f800000u) && threadIdx.x == 0) atomicExch(nonfinite, 1);
    __shared__ uint32_t red[8];
    __shared__ float part_max, s_sh;
    __shared__ int row_sum;  // rank 0's: the cluster's code sum
    if (part == 0 && threadIdx.x == 0) row_sum = 0;
    mb = __reduce_max_sync(0xffffffffu, mb);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mb;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t m = threadIdx.x < 8 ? red[threadIdx.x] : 0u;
        m = __reduce_max_sync(0xffffffffu, m);
        if (threadIdx.x == 0) part_max = __uint_as_float(m);
    }
    cluster.sync();
    if (threadIdx.x == 0) {
        float m = 0.0f;
#pragma unroll
        for (int r = 0; r < CL; ++r) m = fmaxf(m, *cluster.map_shared_rank(&part_max, r));
        s_sh = a4_scale(m);
        if (part == 0) scales[row] = s_sh;
    }
    // s_sh visible; no CTA leaves while its part_max may still be read (with sums:
    // the cluster barrier below, before any CTA exits)
    if (sums != nullptr)
        __syncthreads();
    else
        cluster.sync();
    const float s = s_sh;
    const float rs = __frcp_rn(s);
    char4 *cr = codes != nullptr ? reinterpret_cast<char4 *>(codes + row * ff + part * seg) : nullptr;
    int cs = 0;
#pragma unroll
    for (int u = 0; u < V; ++u) {
        const int j = threadIdx.x + u * 256;
        if (j < nv) {
            const char4 c = make_char4(a4_code_rcp(h[u].x, s, rs), a4_code_rcp(h[u].y, s, rs), a4_code_rcp(h[u].z, s, rs),
                                       a4_code_rcp(h[u].w, s, rs));
            if (cr != nullptr) cr[j] = c;
            if (bo.dst != nullptr)
                *reinterpret_cast<char4 *>(bo.dst + bo.off(row, part * seg + 4 * (int64_t)j)) = c;
            cs += c.x + c.y + c.z + c.w;
        }
    }
    if (sums != nullptr) {
        const int t = block_sum_int(cs);
        if (threadIdx.x == 0) atomicAdd(cluster.map_shared_rank(&row_sum, 0), t);
        cluster.sync();
        if (part == 0 && threadIdx.x == 0) sums[row] = row_sum;
    }
}

template <int CL>
static bool silu_quant_cluster(float *a, const float *b, int64_t rows, int64_t ff, int8_t *codes, float *scales,
                               const int32_t *live, int32_t *sums, int keep, int *nonfinite, const UmmaBOut &bo,
                               cudaStream_t st) {
    if (ff % (4 * CL)) return false;
    const int64_t v = ceil_div(ff / CL / 4, 256);
    const dim3 grid((unsigned)(rows * CL));
    switch (v) {
        case 1: launch_pdl_cluster(silu_quant_cl_kernel<1, CL>, grid, 256, 0, st, CL, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
        case 2: launch_pdl_cluster(silu_quant_cl_kernel<2, CL>, grid, 256, 0, st, CL, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
        case 3:
        case 4: launch_pdl_cluster(silu_quant_cl_kernel<4, CL>, grid, 256, 0, st, CL, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
        case 5: case 6: case 7:
        case 8: launch_pdl_cluster(silu_quant_cl_kernel<8, CL>, grid, 256, 0, st, CL, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
        default: return false;
    }
    return true;
}

static int vec_threads(int64_t ff, int v) {
    return (int)std::min<int64_t>(512, ceil_div(ceil_div(ff / 4, v), 32) * 32);
}

// The vector / cluster re-quantizers (which can write the B layout) cover the row.
static bool silu_b_ok(int64_t ff) { return ff % 4 == 0 && ceil_div(ff / 4, 512) <= 8; }

// `live` (device, nullable): rows at or past *live are skipped (EP slot bounds).
// sums (nullable): per-row code sums (the merged-layout GEMM's bias term).
// keep: also store h = silu(a) * b over a (fp32, read only by tracing); else a
// keeps the gate output and only the codes, scales and sums are written.
// nonfinite (nullable): set to 1 when some h is inf / NaN (the down site's DivergenceError).
// bo.dst: the codes go (also) straight into the down GEMM's B layout; codes may then be nullptr.
cq_status silu_quant(float *a, const float *b, int64_t rows, int64_t ff, int8_t *codes, float *scales,
                     const int32_t *live, cudaStream_t st, int32_t *sums, int keep, int *nonfinite,
                     const UmmaBOut &bo = UmmaBOut{}) {
    if (rows == 0) return CQ_OK;
    static int cl_env = -1;
    if (cl_env < 0) {
        const char *e = getenv("CQ_SILU_CLUSTER");
        cl_env = e ? atoi(e) : 1;
    }
    // about two CTAs per SM over the whole grid; long rows only (a cluster CTA keeps >= 256 float4)
    if (cl_env && ff >= 8192) {
        if (rows <= 74 && silu_quant_cluster<8>(a, b, rows, ff, codes, scales, live, sums, keep, nonfinite, bo, st)) return check_launch("silu_quant");
        if (rows > 74 && rows <= 148 && silu_quant_cluster<4>(a, b, rows, ff, codes, scales, live, sums, keep, nonfinite, bo, st))
            return check_launch("silu_quant");
        // (2-CTA clusters for 149-296 rows measured equal or slower than the CTA-per-row kernel)
    }
    // short rows (ff <= 2048) on CTAs of <= 128 threads (several float4 each): more rows in flight per SM
    // (DS 172 -> 140 us, QW 64 -> 53 us); long rows keep up to 512 (PH at 256: 158 -> 182 us).
    // CQ_SILU_THREADS overrides the short-row cap (experiments).
    static int max_thr = -1;
    if (max_thr < 0) {
        const char *e = getenv("CQ_SILU_THREADS");
        max_thr = e ? atoi(e) : 128;
    }
    const int64_t v = ceil_div(ff / 4, (ff <= 2048 ? max_thr : 512));
    if (ff % 4 == 0 && v <= 8) {
        switch (v) {
            case 1: {  // short rows: one float4 per thread, CTA sized to the row
                const int thr = (int)std::max<int64_t>(64, ceil_div(ff / 4, 32) * 32);
                launch_pdl(silu_quant_vec_kernel<1>, (unsigned)rows, thr, 0, st, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo);
                break;
            }
            // CTA sized to the row at V float4 per thread (PH ff = 6400: 416 threads instead of 512)
            case 2: launch_pdl(silu_quant_vec_kernel<2>, (unsigned)rows, vec_threads(ff, 2), 0, st, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
            case 3:
            case 4: launch_pdl(silu_quant_vec_kernel<4>, (unsigned)rows, vec_threads(ff, 4), 0, st, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
            default: launch_pdl(silu_quant_vec_kernel<8>, (unsigned)rows, vec_threads(ff, 8), 0, st, a, b, ff, codes, scales, live, sums, keep, nonfinite, bo); break;
        }
    } else {
        launch_pdl(silu_quant_kernel, (unsigned)rows, 256, 0, st, a, b, ff, codes, scales, live, sums, nonfinite);
    }
    return check_launch("silu_quant");
}

// h = silu(a) * b elementwise (model.py:396), in place into a.
__global__ void silu_mul_kernel(float *__restrict__ a, const float *__restrict__ b, int64_t count) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < count; x += (int64_t)gridDim.x * blockDim.x)
        a[x] = __fmul_rn(silu_f32(a[x]), b[x]);
}

// out[t, :] = ((0 + w_e1 f_e1) + w_e2 f_e2) + ...  with e ascending (model.py:401),
// then + add[t, :] (shared experts) when given.  grid (n, column blocks).
// 32 registers (8 CTAs of 256 per SM instead of 6): PH 38.5 -> 33.3 us, DS 101 -> 93.5, QW 53 -> 48.4.
__global__ void __launch_bounds__(256, 8)
    combine_kernel(const int32_t *__restrict__ selected, const float *__restrict__ weights,
                   const int32_t *__restrict__ inv, const float *__restrict__ fout, int64_t k, int64_t d,
                   const float *__restrict__ add, int n_add, int64_t add_stride, float *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t t = blockIdx.x;
    __shared__ int32_t pos_sh[16];
    __shared__ float w_sh[16];
    if (threadIdx.x < 32) {  // this token's routes in ascending expert order (ids are distinct): lane s
        const int lane = threadIdx.x;  // loads route s and places it at its rank among the k ids
        const bool on = lane < k;
        const int32_t ex = on ? __ldg(selected + t * k + lane) : INT32_MAX;
        const int32_t pos = on ? __ldg(inv + t * k + lane) : 0;
        const float w = on ? __ldg(weights + t * k + lane) : 0.0f;
        int rank = 0;
        for (int s = 0; s < k; ++s) rank += __shfl_sync(0xffffffffu, ex, s) < ex ? 1 : 0;
        if (on) {
            pos_sh[rank] = pos;
            w_sh[rank] = w;
        }
    }
    __syncthreads();
    const int kk = (int)k;
    if ((d & 3) == 0) {  // 16-byte rows: float4 per thread
        const int64_t d4 = d >> 2;
        const float4 *f4 = reinterpret_cast<const float4 *>(fout);
        for (int64_t j = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; j < d4; j += (int64_t)gridDim.y * blockDim.x) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s = 0; s < kk; ++s) {
                const float ws = w_sh[s];
                const float4 f = __ldg(f4 + (int64_t)pos_sh[s] * d4 + j);
                acc.x = __fadd_rn(acc.x, __fmul_rn(ws, f.x));
                acc.y = __fadd_rn(acc.y, __fmul_rn(ws, f.y));
                acc.z = __fadd_rn(acc.z, __fmul_rn(ws, f.z));
                acc.w = __fadd_rn(acc.w, __fmul_rn(ws, f.w));
            }
            for (int u = 0; u < n_add; ++u) {  // ((routed + add_0) + add_1) ...
                const float4 a4 = reinterpret_cast<const float4 *>(add + u * add_stride)[t * d4 + j];
                acc.x = __fadd_rn(acc.x, a4.x);
                acc.y = __fadd_rn(acc.y, a4.y);
                acc.z = __fadd_rn(acc.z, a4.z);
                acc.w = __fadd_rn(acc.w, a4.w);
            }
            reinterpret_cast<float4 *>(out)[t * d4 + j] = acc;
        }
        return;
    }
    for (int64_t j = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; j < d; j += (int64_t)gridDim.y * blockDim.x) {
        float acc = 0.0f;
        for (int s = 0; s < kk; ++s) acc = __fadd_rn(acc, __fmul_rn(w_sh[s], __ldg(fout + (int64_t)pos_sh[s] * d + j)));
        for (int u = 0; u < n_add; ++u) acc = __fadd_rn(acc, add[u * add_stride + t * d + j]);
        out[t * d + j] = acc;
    }
}

// ---------------------------------------------------------------------------
// workspace

int64_t workspace_layout(const cq_moe_desc *dsc, int64_t n, int64_t *off) {
    const int64_t d = dsc->d_model, ff = dsc->d_ff, E = dsc->n_experts, k = dsc->top_k;
    const int64_t R = n * k;
    const int64_t rows_sh = dsc->n_shared > 0 ? n : 0;
    // shared experts as extra segments of the routed launches: rows R + n_shared * n
    const bool merged = (dsc->flags & CQ_FLAG_SHARED_MERGED) && dsc->n_shared > 0;
    const int64_t Rh = merged ? R + dsc->n_shared * n : (R > rows_sh ? R : rows_sh);
    int64_t sz[CQ_WS_COUNT_] = {};
    sz[CQ_WS_CODES] = n * d;
    sz[CQ_WS_SCALES] = n * 4;
    sz[CQ_WS_LOGITS] = n * E * 4;
    sz[CQ_WS_SELECTED] = n * k * 4;
    sz[CQ_WS_WEIGHTS] = n * k * 4;
    sz[CQ_WS_COUNTS] = (E + 1) * 4;
    sz[CQ_WS_OFFSETS] = (E + 2 + (merged ? dsc->n_shared : 0)) * 4;
    sz[CQ_WS_PERM_TOKEN] = Rh * 4;
    sz[CQ_WS_PERM_SLOT] = R * 4;
    sz[CQ_WS_INV] = R * 4;
    sz[CQ_WS_CODES_PERM] = R * d;
    sz[CQ_WS_SCALES_PERM] = Rh * 4;  // the B build writes one scale per expert row
    sz[CQ_WS_HIDDEN] = Rh * ff * 4 * 2;  // h (or gate output a) | up output b
    sz[CQ_WS_HCODES] = Rh * ff;
    sz[CQ_WS_HSCALES] = Rh * 4;
    sz[CQ_WS_FOUT] = Rh * d * 4;
    sz[CQ_WS_ROTATED] = (dsc->rotation || dsc->rotation_tc) ? n * d * 4 : 0;
    sz[CQ_WS_SHARED] = dsc->n_shared * n * d * 4;  // one output per shared expert
    sz[CQ_WS_CODES_FRAG] = umma_b_bytes(Rh, d);     // >= the mma16 fragment size too
    sz[CQ_WS_HCODES_FRAG] = umma_b_bytes(Rh, ff);
    sz[CQ_WS_ROT_ACT] = dsc->rotation_tc ? rot_tc_act_bytes(n, d) : 0;
    sz[CQ_WS_TOK_SUMS] = n * 4;
    sz[CQ_WS_STATUS] = 4 * 4;
    sz[CQ_WS_SH_OFFSETS] = 2 * 4;
    int64_t pos = 0;
    for (int b = 0; b < CQ_WS_COUNT_; ++b) {
        if (off) off[b] = pos;
        pos += (sz[b] + 255) / 256 * 256;
    }
    return pos;
}

struct Ws {
    int8_t *codes;
    float *scales, *logits, *weights, *scales_perm, *hidden, *hscales, *fout, *rotated, *shared;
    int32_t *selected, *counts, *offsets, *perm_token, *perm_slot, *inv, *tok_sums;
    int *status;  // CQ_WS_STATUS: [0] layer input non-finite, [1] hidden (down input) non-finite
    int32_t *sh_offsets;
    int8_t *codes_perm, *hcodes;
    int8_t *codes_frag, *hcodes_frag;  // tcgen05 B-operand buffers
    void *rot_act;
};

Ws carve(void *base, const int64_t *o) {
    char *b = reinterpret_cast<char *>(base);
    Ws w;
    w.codes = reinterpret_cast<int8_t *>(b + o[CQ_WS_CODES]);
    w.scales = reinterpret_cast<float *>(b + o[CQ_WS_SCALES]);
    w.logits = reinterpret_cast<float *>(b + o[CQ_WS_LOGITS]);
    w.selected = reinterpret_cast<int32_t *>(b + o[CQ_WS_SELECTED]);
    w.weights = reinterpret_cast<float *>(b + o[CQ_WS_WEIGHTS]);
    w.counts = reinterpret_cast<int32_t *>(b + o[CQ_WS_COUNTS]);
    w.offsets = reinterpret_cast<int32_t *>(b + o[CQ_WS_OFFSETS]);
    w.perm_token = reinterpret_cast<int32_t *>(b + o[CQ_WS_PERM_TOKEN]);
    w.perm_slot = reinterpret_cast<int32_t *>(b + o[CQ_WS_PERM_SLOT]);
    w.inv = reinterpret_cast<int32_t *>(b + o[CQ_WS_INV]);
    w.tok_sums = reinterpret_cast<int32_t *>(b + o[CQ_WS_TOK_SUMS]);
    w.status = reinterpret_cast<int *>(b + o[CQ_WS_STATUS]);
    w.sh_offsets = reinterpret_cast<int32_t *>(b + o[CQ_WS_SH_OFFSETS]);
    w.codes_perm = reinterpret_cast<int8_t *>(b + o[CQ_WS_CODES_PERM]);
    w.scales_perm = reinterpret_cast<float *>(b + o[CQ_WS_SCALES_PERM]);
    w.hidden = reinterpret_cast<float *>(b + o[CQ_WS_HIDDEN]);
    w.hcodes = reinterpret_cast<int8_t *>(b + o[CQ_WS_HCODES]);
    w.hscales = reinterpret_cast<float *>(b + o[CQ_WS_HSCALES]);
    w.fout = reinterpret_cast<float *>(b + o[CQ_WS_FOUT]);
    w.rotated = reinterpret_cast<float *>(b + o[CQ_WS_ROTATED]);
    w.rot_act = b + o[CQ_WS_ROT_ACT];
    w.shared = reinterpret_cast<float *>(b + o[CQ_WS_SHARED]);
    w.codes_frag = reinterpret_cast<int8_t *>(b + o[CQ_WS_CODES_FRAG]);
    w.hcodes_frag = reinterpret_cast<int8_t *>(b + o[CQ_WS_HCODES_FRAG]);
    return w;
}

cq_status validate_desc(const cq_moe_desc *d) {
    if (d == nullptr || d->d_model < 1 || d->d_ff < 1 || d->n_experts < 1 || d->top_k < 1) {
        set_error("moe: bad descriptor dimensions");
        return CQ_ERR_SHAPE;
    }
    if (d->top_k > d->n_experts || d->top_k > 16) {
        set_error("moe: top_k must be <= n_experts and <= 16");
        return CQ_ERR_CONFIG;
    }
    if (d->expert_begin < 0 || d->n_local_experts < 0 || d->expert_begin + d->n_local_experts > d->n_experts) {
        set_error("moe: local expert range outside [0, n_experts)");
        return CQ_ERR_CONFIG;
    }
    const cq_expert_site *sites[3] = {&d->gate, &d->up, &d->down};
    const int64_t din[3] = {d->d_model, d->d_model, d->d_ff};
    for (int s = 0; s < 3; ++s) {
        const int64_t g = sites[s]->group_size;
        if (g < 1 || din[s] % g) {
            set_error("moe: group size does not divide the site's input dimension");
            return CQ_ERR_SHAPE;
        }
    }
    if (d->gate.group_size != d->up.group_size) {
        set_error("moe: gate and up must share a group size (fused kernel)");
        return CQ_ERR_CONFIG;
    }
    return CQ_OK;
}

int choose_path(const cq_moe_desc *d) {
    if (d->path != CQ_PATH_AUTO) return d->path;
    const bool tc = d->gate.tc_lut && d->up.tc_lut && d->down.tc_lut &&
                    umma_family(d->gate.tc_layout) == umma_family(d->up.tc_layout) &&
                    umma_family(d->up.tc_layout) == umma_family(d->down.tc_layout) &&
                    umma_ok(d->d_model, d->d_ff, d->gate.group_size) &&
                    umma_ok(d->d_ff, d->d_model, d->down.group_size);
    if (tc) return CQ_PATH_TC;
    if (f32_path_ok(d->d_model, d->gate.group_size) && f32_path_ok(d->d_ff, d->down.group_size))
        return CQ_PATH_F32;
    return CQ_PATH_ORDERED;
}

// Expert stage over segment rows (gate|up -> silu*b -> requant -> down).
cq_status run_experts(const cq_moe_desc *dsc, int path, const cq_expert_site &gate, const cq_expert_site &up,
                      const cq_expert_site &down, int64_t n_seg, int64_t seg_first, const int8_t *codes,
                      const float *scales, const int32_t *offsets, int64_t rows, float *hidden,
                      int8_t *hcodes, float *hscales, float *fout, int8_t *bbuf_in, int8_t *bbuf_h,
                      int *nonfinite, cudaStream_t st, cudaEvent_t *ev = nullptr, const UmmaIn &in = UmmaIn{}) {
    const int64_t d = dsc->d_model, ff = dsc->d_ff;
    if (rows == 0 || n_seg == 0) return CQ_OK;
    float *bout = hidden + rows * ff;  // up output (gate output / h in `hidden`)
    if (ev) cudaEventRecord(ev[0], st);
    if (path == CQ_PATH_TC) {
        // `in` may make the B build gather token rows (codes / scales per token, in.perm)
        CQ_TRY(lut_umma_grouped(codes, bbuf_in, scales, offsets, n_seg, seg_first, rows, &gate, hidden, &up, bout, d,
                                ff, st, in));
        if (ev) cudaEventRecord(ev[1], st);
        // the re-quantizer writes the down GEMM's row sums straight into its B buffer, and (vector / cluster
        // kernels) the codes in its tile layout: the down launch then has no B build.  The row-major codes
        // only for tracing (CQ_FLAG_KEEP_HIDDEN).
        UmmaIn hin;
        hin.sums_ready = true;
        int32_t *hsums = umma_row_sums(bbuf_h, rows, ff);
        const int keep = (dsc->flags & CQ_FLAG_KEEP_HIDDEN) != 0;
        UmmaBOut bo;
        if (silu_b_ok(ff)) {
            const int gck = umma_geo_ck(rows, n_seg, ff, d, 1, (int)down.tc_planes);  // < 0: prefill
            bo = umma_b_out(bbuf_h, rows, ff, gck < 0 ? -gck : gck);
            hin.b_ready = true;
        }
        CQ_TRY(silu_quant(hidden, bout, rows, ff, (keep || !hin.b_ready) ? hcodes : nullptr, hscales, offsets + n_seg,
                          st, hsums, keep, nonfinite, bo));
        if (ev) cudaEventRecord(ev[2], st);
        CQ_TRY(lut_umma_grouped(hcodes, bbuf_h, hscales, offsets, n_seg, seg_first, rows, &down, fout, nullptr,
                                nullptr, ff, d, st, hin));
        if (ev) cudaEventRecord(ev[3], st);
        return CQ_OK;
    }
    if (path == CQ_PATH_F32) {
        CQ_TRY(lut_f32_grouped(codes, scales, offsets, n_seg, seg_first, gate.ids, gate.centroids, up.ids,
                               up.centroids, d, ff, gate.group_size, hidden, st));
    } else {  // ordered: the reference's chains bit for bit (ordered.cu)
        CQ_TRY(ordered_lut(codes, scales, offsets, n_seg, seg_first, rows, gate.ids, gate.centroids, d, ff,
                           gate.group_size, hidden, st));
        CQ_TRY(ordered_lut(codes, scales, offsets, n_seg, seg_first, rows, up.ids, up.centroids, d, ff,
                           up.group_size, bout, st));
        launch_pdl(silu_mul_kernel, (unsigned)std::min<int64_t>(ceil_div(rows * ff, 256), 148 * 16), 256, 0, st,
                   hidden, (const float *)bout, rows * ff);
        CQ_TRY(check_launch("silu_mul"));
    }
    if (ev) cudaEventRecord(ev[1], st);
    CQ_TRY(quantize_a4(hidden, CQ_DTYPE_F32, rows, ff, hcodes, hscales, nonfinite, nullptr, st));
    if (ev) cudaEventRecord(ev[2], st);
    cq_status rc;
    if (path == CQ_PATH_F32)
        rc = lut_f32_grouped(hcodes, hscales, offsets, n_seg, seg_first, down.ids, down.centroids, nullptr, nullptr,
                             ff, d, down.group_size, fout, st);
    else
        rc = ordered_lut(hcodes, hscales, offsets, n_seg, seg_first, rows, down.ids, down.centroids, ff, d,
                         down.group_size, fout, st);
    if (ev) cudaEventRecord(ev[3], st);
    return rc;
}

// Shared experts as segments E .. E + n_shared - 1 of the routed launch (CQ_FLAG_SHARED_MERGED):
// every token, in order, after the R routed rows: perm[R + s*n + t] = t, offsets[E + 1 + s] =
// R + (s + 1) * n (offsets[E] = R: every route is local in cq_moe_forward).
__global__ void shared_segments_kernel(int32_t *perm, int32_t *offsets, int64_t n_exp, int64_t R, int64_t n,
                                       int64_t n_shared) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t total = n_shared * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x)
        perm[R + x] = (int32_t)(x % n);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int64_t sh = 0; sh < n_shared; ++sh) offsets[n_exp + 1 + sh] = (int32_t)(R + (sh + 1) * n);
}

__global__ void shared_offsets_kernel(int32_t *off, int64_t n_shared, int64_t n) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    for (int64_t s = 0; s <= n_shared; ++s) off[s] = (int32_t)(s * n);
}

// Builder-defined shared experts (not in the reference,
// SPEC.md:173): always-on experts of weight 1 over all n tokens of this rank,
// each run as one segment on the un-permuted layer-input codes into its own
// [n][d_model] slice of `out` (n_shared slices).
cq_status shared_experts(const cq_moe_desc *desc, int path, int64_t n, const Ws &w, float *out, cudaStream_t st) {
    if (desc->n_shared <= 0 || n == 0) return CQ_OK;
    launch_pdl(shared_offsets_kernel, 1, 1, 0, st, w.sh_offsets, (int64_t)1, n);
    CQ_TRY(check_launch("shared_offsets"));
    const int sp = (path == CQ_PATH_TC && desc->sh_gate.tc_lut == nullptr) ? CQ_PATH_F32 : path;
    for (int64_t s = 0; s < desc->n_shared; ++s)
        CQ_TRY(run_experts(desc, sp, desc->sh_gate, desc->sh_up, desc->sh_down, 1, s, w.codes, w.scales,
                           w.sh_offsets, n, w.hidden, w.hcodes, w.hscales, out + s * n * desc->d_model, w.codes_frag,
                           w.hcodes_frag, w.status + 1, st));
    return CQ_OK;
}

// gather = false: leave codes_perm / scales_perm unwritten (the tcgen05 expert
// stage gathers token rows itself, UmmaIn::perm).  deferred (nullable): at
// decode sizes, where the router launch also does the top-k (one expert group),
// stop there and set *deferred = 1: the permutation is the GEMM's B build's
// (UmmaIn::route); 0 = everything done here.

// Routing deferred to the B build (every B-build CTA derives the permutation itself): up to
// CQ_ROUTE_DEFER_MAX routes, past which it stops paying (MX: 128 routes 0.310 vs 0.311 ms deferred /
// separate, 256 equal, 512 0.468 vs 0.463, 1024 0.754 vs 0.726).
static bool route_deferrable(const cq_moe_desc *dsc, int64_t n) {
    static int64_t defer_max = -1;
    if (defer_max < 0) {
        const char *e = getenv("CQ_ROUTE_DEFER_MAX");
        defer_max = e ? atoll(e) : 256;
    }
    return n * dsc->top_k <= std::min<int64_t>(defer_max, RP_MAX_ROUTES) && dsc->n_local_experts <= RP_MAX_LOCAL &&
           dsc->top_k <= MAX_TOPK && dsc->top_k <= dsc->n_experts;
}

cq_status route(const cq_moe_desc *dsc, const void *x, int dtype, int64_t n, const Ws &w, cudaStream_t st,
                bool gather = true, int *deferred = nullptr) {
    const int64_t d = dsc->d_model;
    // the dequantized rows (router input) go to the fout buffer, unused until the down GEMM;
    // the quantizer also clears the route counts and the arrival counter (counts[E])
    if (dsc->rotation_tc != nullptr) {
        // tensor cores, bf16-split R (rotate_tc.cu), then the certified quantizer: the codes and scale of
        // the reference's ordered chain bit for bit (rotq.cu; recomputed elements counted in status[2])
        CQ_TRY(rot_tc_apply(x, dtype, n, d, dsc->rotation_tc, w.rot_act, w.rotated, st));
        CQ_TRY(rot_certify(w.rotated, x, dtype, rot_tc_transposed(dsc->rotation_tc, d), n, d, w.codes, w.scales,
                           w.status, w.fout, w.tok_sums, w.counts, (int)dsc->n_experts + 1, w.status + 2,
                           w.rot_act, rot_tc_act_bytes(n, d), st));
    } else {
        const void *qin = x;
        int qdt = dtype;
        if (deferred != nullptr && dsc->rotation == nullptr && route_deferrable(dsc, n)) {
            // decode: the quantizer runs inside the router launch (router_fused_quant), which saves a
            // launch and the dequantized rows' round trip through memory
            bool fused = false;
            CQ_TRY(router_fused_quant(x, dtype, w.codes, w.scales, w.status, w.tok_sums, w.counts,
                                      (int)dsc->n_experts + 1, w.fout, dsc->w_router, n, d, dsc->n_experts,
                                      w.logits, w.selected, w.weights, dsc->top_k, st, &fused));
            if (fused) {
                *deferred = 1;
                return CQ_OK;
            }
        }
        if (dsc->rotation != nullptr) {  // the reference's ordered chain (pipeline.py:516 -> _core.pyx:27-38)
            CQ_TRY(ordered_matmul(x, dtype, dsc->rotation, n, d, d, w.rotated, st));
            qin = w.rotated;
            qdt = CQ_DTYPE_F32;
        }
        CQ_TRY(quantize_a4(qin, qdt, n, d, w.codes, w.scales, w.status, w.fout, st, w.tok_sums, w.counts,
                           (int)dsc->n_experts + 1));
    }
    if (deferred != nullptr) {
        *deferred = 0;
        if (route_deferrable(dsc, n)) {
            bool fused = false;  // logits + top-k in one launch (one expert group)
            CQ_TRY(router_fused(w.fout, dsc->w_router, n, d, dsc->n_experts, w.logits, w.selected, w.weights,
                                dsc->top_k, st, &fused));
            if (fused) {
                *deferred = 1;
                return CQ_OK;
            }
        }
    }
    CQ_TRY(router_logits(w.codes, w.scales, w.fout, dsc->w_router, n, d, dsc->n_experts, w.logits, st));
    // the permutation counts the routes itself (no atomics in the top-k) unless routing stops at the top-k
    const bool perm_counts = !(dsc->flags & CQ_FLAG_SELECT_ONLY) && permute_counts_itself(n);
    CQ_TRY(topk(w.logits, n, dsc->n_experts, dsc->top_k, w.selected, w.weights, perm_counts ? nullptr : w.counts,
                dsc->expert_begin,
                dsc->n_local_experts, st));
    if (dsc->flags & CQ_FLAG_SELECT_ONLY) return CQ_OK;
    CQ_TRY(permute(w.selected, w.counts, n, dsc->top_k, dsc->expert_begin, dsc->n_local_experts, w.offsets,
                   w.perm_token, w.perm_slot, w.inv, st));
    if (!gather) return CQ_OK;
    return gather_rows(w.codes, w.scales, w.perm_token, w.offsets, dsc->n_local_experts, n * dsc->top_k, d,
                       w.codes_perm, w.scales_perm, st);
}

}  // namespace cq

using namespace cq;

extern "C" int64_t cq_moe_workspace(const cq_moe_desc *desc, int64_t n_tokens, int64_t *offsets_out) {
    if (desc == nullptr || n_tokens < 0) return -1;
    return workspace_layout(desc, n_tokens, offsets_out);
}

extern "C" cq_status cq_moe_route(const cq_moe_desc *desc, const void *x, int dtype, int64_t n_tokens,
                                  void *workspace, int64_t workspace_bytes, void *stream) {
    CQ_TRY(validate_desc(desc));
    int64_t off[CQ_WS_COUNT_];
    if (workspace_layout(desc, n_tokens, off) > workspace_bytes) {
        set_error("moe: workspace too small");
        return CQ_ERR_SHAPE;
    }
    if (n_tokens == 0) return CQ_OK;
    if (desc->flags & CQ_FLAG_SELECT_ONLY) {  // the fused decode router + top-k when it applies
        int fused = 0;
        return route(desc, x, dtype, n_tokens, carve(workspace, off), as_stream(stream), false, &fused);
    }
    return route(desc, x, dtype, n_tokens, carve(workspace, off), as_stream(stream));
}

extern "C" cq_status cq_moe_experts(const cq_moe_desc *desc, const int8_t *codes_perm, const float *scales_perm,
                                    const int32_t *offsets, int64_t rows, float *fout, void *workspace,
                                    int64_t workspace_bytes, void *stream) {
    CQ_TRY(validate_desc(desc));
    // the expert stage needs hidden/hcodes sized for `rows`; size the layout for rows/top_k tokens
    const int64_t n_equiv = ceil_div(rows, desc->top_k);
    int64_t off[CQ_WS_COUNT_];
    if (workspace_layout(desc, n_equiv, off) > workspace_bytes) {
        set_error("moe: workspace too small");
        return CQ_ERR_SHAPE;
    }
    Ws w = carve(workspace, off);
    return run_experts(desc, choose_path(desc), desc->gate, desc->up, desc->down, desc->n_local_experts, 0,
                       codes_perm, scales_perm, offsets, rows, w.hidden, w.hcodes, w.hscales, fout, w.codes_frag,
                       w.hcodes_frag, w.status + 1, as_stream(stream));
}

extern "C" cq_status cq_moe_profile_experts(const cq_moe_desc *desc, const int8_t *codes_perm,
                                            const float *scales_perm, const int32_t *offsets, int64_t rows, float *fout,
                                            void *workspace, int64_t workspace_bytes, int32_t iters,
                                            float *stage_ms_host, void *stream) {
    CQ_TRY(validate_desc(desc));
    const int64_t n_equiv = ceil_div(rows, desc->top_k);
    int64_t off[CQ_WS_COUNT_];
    if (workspace_layout(desc, n_equiv, off) > workspace_bytes) {
        set_error("moe: workspace too small");
        return CQ_ERR_SHAPE;
    }
    if (iters < 1) iters = 1;
    Ws w = carve(workspace, off);
    cudaStream_t st = as_stream(stream);
    cudaEvent_t ev[4];
    for (auto &e : ev) cudaEventCreate(&e);
    double acc[3] = {0, 0, 0};
    cq_status rc = CQ_OK;
    for (int i = 0; i < iters && rc == CQ_OK; ++i) {
        rc = run_experts(desc, choose_path(desc), desc->gate, desc->up, desc->down, desc->n_local_experts, 0,
                         codes_perm, scales_perm, offsets, rows, w.hidden, w.hcodes, w.hscales, fout, w.codes_frag,
                         w.hcodes_frag, nullptr, st, ev);
        cudaEventSynchronize(ev[3]);
        for (int k = 0; k < 3; ++k) {
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
            acc[k] += ms;
        }
    }
    for (auto &e : ev) cudaEventDestroy(e);
    for (int k = 0; k < 3; ++k) stage_ms_host[k] = (float)(acc[k] / iters);
    return rc;
}

// add (nullable): n_add buffers of [n_tokens][d_model], n_tokens * d_model apart, added to the
// routed sum in order.
static cq_status combine_n(const int32_t *selected, const float *weights, const int32_t *inv, const float *fout,
                           int64_t n_tokens, int64_t top_k, int64_t d_model, const float *add, int n_add, float *out,
                           void *stream) {
    if (n_tokens == 0) return CQ_OK;
    if (top_k < 1 || top_k > 16) {
        set_error("combine: top_k out of range");
        return CQ_ERR_CONFIG;
    }
    const int64_t cols = (d_model & 3) == 0 ? d_model / 4 : d_model;  // work items per token
    const int threads = (int)std::min<int64_t>(256, ceil_div(cols, 32) * 32);
    dim3 grid((unsigned)n_tokens, (unsigned)std::max<int64_t>(1, std::min<int64_t>(16, ceil_div(cols, threads))));
    launch_pdl(combine_kernel, grid, threads, 0, as_stream(stream), selected, weights, inv, fout, top_k, d_model, add,
               add ? n_add : 0, n_tokens * d_model, out);
    return check_launch("combine");
}

extern "C" cq_status cq_moe_combine(const int32_t *selected, const float *weights, const int32_t *inv,
                                    const float *fout, int64_t n_tokens, int64_t top_k, int64_t d_model,
                                    const float *add, int64_t n_add, float *out, void *stream) {
    if (n_add < 0 || (n_add > 0 && add == nullptr)) {
        set_error("combine: n_add buffers need a non-null add");
        return CQ_ERR_SHAPE;
    }
    return combine_n(selected, weights, inv, fout, n_tokens, top_k, d_model, add, (int)n_add, out, stream);
}

extern "C" cq_status cq_moe_shared_experts(const cq_moe_desc *desc, int64_t n_tokens, float *shared_out,
                                           void *workspace, int64_t workspace_bytes, void *stream) {
    CQ_TRY(validate_desc(desc));
    int64_t off[CQ_WS_COUNT_];
    if (workspace_layout(desc, n_tokens, off) > workspace_bytes) {
        set_error("moe: workspace too small");
        return CQ_ERR_SHAPE;
    }
    if (desc->n_shared > 0 && shared_out == nullptr) {
        set_error("moe: shared experts need an output buffer");
        return CQ_ERR_SHAPE;
    }
    return shared_experts(desc, choose_path(desc), n_tokens, carve(workspace, off), shared_out, as_stream(stream));
}

extern "C" cq_status cq_moe_forward(const cq_moe_desc *desc, const void *x, int dtype, int64_t n_tokens, float *out,
                                    void *workspace, int64_t workspace_bytes, void *stream) {
    CQ_TRY(validate_desc(desc));
    if (desc->expert_begin != 0 || desc->n_local_experts != desc->n_experts) {
        set_error("moe_forward runs all experts locally; use the EP driver for sharded experts");
        return CQ_ERR_CONFIG;
    }
    int64_t off[CQ_WS_COUNT_];
    if (workspace_layout(desc, n_tokens, off) > workspace_bytes) {
        set_error("moe: workspace too small");
        return CQ_ERR_SHAPE;
    }
    if (n_tokens == 0) return CQ_OK;
    cudaStream_t st = as_stream(stream);
    Ws w = carve(workspace, off);
    const int path = choose_path(desc);
    // tcgen05 layouts: the expert stage's B build gathers the token rows itself (no codes_perm)
    const bool umma = path == CQ_PATH_TC;
    int deferred = 0;
    const bool want_merged = umma && (desc->flags & CQ_FLAG_SHARED_MERGED) && desc->n_shared > 0;
    // merged shared segments need the explicit permutation (not the B build's route mode)
    CQ_TRY(route(desc, x, dtype, n_tokens, w, st, !umma, (umma && !want_merged) ? &deferred : nullptr));
    const bool merged = want_merged && !deferred;
    // builder-defined shared experts: extra segments of the routed launches when
    // merged, else separate launches first (they read only the layer-input codes, and the routed pass
    // after them leaves its own counts / hidden buffers for tracing)
    if (!merged) CQ_TRY(shared_experts(desc, path, n_tokens, w, w.shared, st));
    const int64_t R = n_tokens * desc->top_k;
    if (merged) {
        const int64_t ns = desc->n_shared, total = ns * n_tokens;
        launch_pdl(shared_segments_kernel, (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 8), 256, 0, st,
                   w.perm_token, w.offsets, desc->n_experts, R, n_tokens, ns);
        CQ_TRY(check_launch("shared_segments"));
        UmmaIn in;
        in.tok_sums = w.tok_sums;
        in.scales_out = w.scales_perm;
        in.perm = w.perm_token;
        CQ_TRY(run_experts(desc, path, desc->gate, desc->up, desc->down, desc->n_experts + ns, 0, w.codes, w.scales,
                           w.offsets, R + total, w.hidden, w.hcodes, w.hscales, w.fout, w.codes_frag, w.hcodes_frag,
                           w.status + 1, st, nullptr, in));
        // out = ((routed + sh_0) + sh_1) ..., the shared outputs are fout rows R + s * n + t
        return combine_n(w.selected, w.weights, w.inv, w.fout, n_tokens, desc->top_k, desc->d_model,
                         w.fout + R * desc->d_model, (int)ns, out, stream);
    }
    if (umma) {
        UmmaIn in;
        in.tok_sums = w.tok_sums;
        in.scales_out = w.scales_perm;
        if (deferred) {  // the B build derives the permutation and publishes it
            in.route.selected = w.selected;
            in.route.n_tok = n_tokens;
            in.route.k = (int)desc->top_k;
            in.route.local_begin = desc->expert_begin;
            in.route.n_local = (int)desc->n_local_experts;
            in.route.offsets = w.offsets;
            in.route.counts = w.counts;
            in.route.perm_token = w.perm_token;
            in.route.perm_slot = w.perm_slot;
            in.route.inv = w.inv;
        } else {
            in.perm = w.perm_token;
        }
        CQ_TRY(run_experts(desc, path, desc->gate, desc->up, desc->down, desc->n_experts, 0, w.codes, w.scales,
                           w.offsets, R, w.hidden, w.hcodes, w.hscales, w.fout, w.codes_frag, w.hcodes_frag,
                           w.status + 1, st, nullptr, in));
    } else {
        CQ_TRY(run_experts(desc, path, desc->gate, desc->up, desc->down, desc->n_experts, 0, w.codes_perm,
                           w.scales_perm, w.offsets, R, w.hidden, w.hcodes, w.hscales, w.fout, w.codes_frag,
                           w.hcodes_frag, w.status + 1, st));
    }
    // out = ((routed + sh_0) + sh_1) ..., the shared outputs added in order inside the combine pass
    return combine_n(w.selected, w.weights, w.inv, w.fout, n_tokens, desc->top_k, desc->d_model,
                     desc->n_shared > 0 ? w.shared : nullptr, (int)desc->n_shared, out, stream);
}
