// fp32 CUDA-core LUT GEMM / GEMV: the MoE layer's path="f32" expert stage.
//
// Same contract as _core.lut_gemm_f32 (kernels/_core.pyx:41-151): the product
// of centroid c = C[i, j/g, id[i,j]] and code q is exact-ish fp32 (FMA) and the
// per-token scale is applied once at the end.  Differences to the reference are
// accumulation order only (~1e-7 relative).
//
// Work split: one warp per output row, lanes split K eight columns at a time
// (one 32-bit word of packed ids per lane per step -> 128 B coalesced per row
// per warp), tokens in register tiles of T, warp-shuffle reduction at the end.
// Segments (offsets[s] .. offsets[s+1]) are the per-expert row ranges of the
// permuted token buffer; weights of segment s live at base + s * stride.
#include "common.cuh"

namespace cq {

constexpr int F32_WARPS = 8;
constexpr int F32_T = 8;

template <bool GLU>
__global__ void __launch_bounds__(F32_WARPS * 32) lut_f32_grouped_kernel(
    const int8_t *__restrict__ codes, const float *__restrict__ scales,
    const int32_t *__restrict__ offsets, int64_t seg_first,
    const uint8_t *__restrict__ ids_a, const float *__restrict__ cent_a,
    const uint8_t *__restrict__ ids_b, const float *__restrict__ cent_b,
    int64_t d_in, int64_t d_out, int64_t g, float *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t seg = blockIdx.y;
    const int64_t i = blockIdx.x * (int64_t)F32_WARPS + warp;
    const int64_t rb = offsets[seg], re = offsets[seg + 1];
    if (i >= d_out || rb >= re) return;
    const int64_t e = seg + seg_first;
    const int64_t row_bytes = d_in >> 1, n_groups = d_in / g;
    const uint8_t *ia = ids_a + (e * d_out + i) * row_bytes;
    const float *ca = cent_a + (e * d_out + i) * n_groups * 16;
    const uint8_t *ib = GLU ? ids_b + (e * d_out + i) * row_bytes : nullptr;
    const float *cb = GLU ? cent_b + (e * d_out + i) * n_groups * 16 : nullptr;

    for (int64_t t0 = rb; t0 < re; t0 += F32_T) {
        const int nt = (int)((re - t0) < F32_T ? (re - t0) : F32_T);
        float acc_a[F32_T], acc_b[F32_T];
#pragma unroll
        for (int u = 0; u < F32_T; ++u) acc_a[u] = acc_b[u] = 0.0f;
        for (int64_t k0 = lane * 8; k0 < d_in; k0 += 256) {
            const uint32_t wa = __ldg(reinterpret_cast<const uint32_t *>(ia + (k0 >> 1)));
            const float *ga = ca + (k0 / g) * 16;
            float cva[8], cvb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) cva[u] = __ldg(ga + ((wa >> (4 * u)) & 15));
            if (GLU) {
                const uint32_t wb = __ldg(reinterpret_cast<const uint32_t *>(ib + (k0 >> 1)));
                const float *gb = cb + (k0 / g) * 16;
#pragma unroll
                for (int u = 0; u < 8; ++u) cvb[u] = __ldg(gb + ((wb >> (4 * u)) & 15));
            }
#pragma unroll
            for (int tt = 0; tt < F32_T; ++tt) {
                if (tt < nt) {
                    const uint2 qv = __ldg(reinterpret_cast<const uint2 *>(codes + (t0 + tt) * d_in + k0));
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t word = u < 4 ? qv.x : qv.y;
                        const float q = (float)(int8_t)(word >> (8 * (u & 3)));
                        acc_a[tt] = fmaf(cva[u], q, acc_a[tt]);
                        if (GLU) acc_b[tt] = fmaf(cvb[u], q, acc_b[tt]);
                    }
                }
            }
        }
#pragma unroll
        for (int tt = 0; tt < F32_T; ++tt) {
            if (tt < nt) {
                const float sa = warp_sum(acc_a[tt]);
                const float sb = GLU ? warp_sum(acc_b[tt]) : 0.0f;
                if (lane == 0) {
                    const float s = __ldg(scales + t0 + tt);
                    const float a = __fmul_rn(s, sa);
                    out[(t0 + tt) * d_out + i] = GLU ? __fmul_rn(silu_f32(a), __fmul_rn(s, sb)) : a;
                }
            }
        }
    }
}

bool f32_path_ok(int64_t d_in, int64_t g) { return d_in % 8 == 0 && g % 8 == 0; }

// Grouped launch: n_seg segments whose weights start at expert seg_first.
cq_status lut_f32_grouped(const int8_t *codes, const float *scales, const int32_t *offsets,
                          int64_t n_seg, int64_t seg_first, const uint8_t *ids_a,
                          const float *cent_a, const uint8_t *ids_b, const float *cent_b,
                          int64_t d_in, int64_t d_out, int64_t g, float *out, cudaStream_t st) {
    if (n_seg == 0 || d_out == 0) return CQ_OK;
    dim3 grid((unsigned)ceil_div(d_out, F32_WARPS), (unsigned)n_seg);
    if (ids_b != nullptr)
        lut_f32_grouped_kernel<true><<<grid, F32_WARPS * 32, 0, st>>>(
            codes, scales, offsets, seg_first, ids_a, cent_a, ids_b, cent_b, d_in, d_out, g, out);
    else
        lut_f32_grouped_kernel<false><<<grid, F32_WARPS * 32, 0, st>>>(
            codes, scales, offsets, seg_first, ids_a, cent_a, nullptr, nullptr, d_in, d_out, g, out);
    return check_launch("lut_f32_grouped");
}

}  // namespace cq
