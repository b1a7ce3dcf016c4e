// One-time device re-layout of PackedClusteredWeights (lutgemm.py:53-87) for
// the tcgen05 LUT GEMM (lut_umma.cu), and the single-matrix tensor-core GEMM
// entry point.
//
// Digit planes.  Every weight row's centroids become integers
// m = rint(c / rowscale), |m| < 2^(7P-1), with one fp32 rowscale per row
// (row max / (2^(7P-1) - 1)).  m + 2^(7P-1) is written as P unsigned base-128
// digits (7 bits each, sign bit clear), one 16-entry byte table per (row,
// group, plane): the PRMT lookup of lut_umma.cu reads them with the packed ids
// as selectors.  3 planes keep 21 bits of the row max (gate / up, whose output
// is re-quantized), 2 planes 14 bits (down).
//
// Layouts written here (the ids are the same bytes, re-tiled):
//   tc_ids      [rows/128][d_in/128][kstep 4][row 128][16 B]
//   tc_lut      [rows/128][d_in/g][row 128][P][16]
//   tc_rowscale [rows]
#include "common.cuh"

namespace cq {

// rowscale[r] = max_c |C[r, c]| / mbound (1 for an all-zero row).
__global__ void rowscale_kernel(const float *__restrict__ cent, int64_t rows, int64_t per_row, double mbound,
                                float *__restrict__ rowscale) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const float *c = cent + row * per_row;
    float mx = 0.0f;
    for (int64_t i = threadIdx.x & 31; i < per_row; i += 32) mx = fmaxf(mx, fabsf(c[i]));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) rowscale[row] = mx > 0.0f ? (float)((double)mx / mbound) : 1.0f;
}

// One thread per (row, group): the P unsigned digit tables of its 16 centroids,
// straight into the 128-row tile layout.
__global__ void lut7_kernel(const float *__restrict__ cent, const float *__restrict__ rowscale, int64_t rows,
                            int64_t n_groups, int planes, int8_t *__restrict__ lut) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= rows * n_groups) return;
    const int64_t row = x / n_groups, grp = x - row * n_groups;
    const double s = (double)rowscale[row];
    const long long bias = 1LL << (7 * planes - 1), mb = bias - 1;
    int8_t *dst = lut + (((row / 128) * n_groups + grp) * 128 + row % 128) * planes * 16;
    for (int c = 0; c < 16; ++c) {
        long long m = llrint((double)cent[x * 16 + c] / s);
        m = m > mb ? mb : (m < -mb ? -mb : m);
        const long long u = m + bias;
        for (int p = 0; p < planes; ++p) dst[p * 16 + c] = (int8_t)((u >> (7 * p)) & 127);
    }
}

// ids (rows, d_in/2) -> [tile128][chunk][kstep][row][16 B] (the 16 packed bytes of
// a row's 32 columns are already 8 PRMT selectors, low nibble first).
__global__ void ids_umma_kernel(const uint8_t *__restrict__ ids, int64_t rows, int64_t d_in, uint4 *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t n_chunks = d_in / 128;
    const int64_t total = (rows / 128) * n_chunks * 4 * 128;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = x & 127, ks = (x >> 7) & 3, c = (x >> 9) % n_chunks, t = (x >> 9) / n_chunks;
        out[x] = *reinterpret_cast<const uint4 *>(ids + (t * 128 + r) * (d_in / 2) + c * 64 + ks * 16);
    }
}

bool umma_ok(int64_t d_in, int64_t d_out, int64_t g);
int64_t umma_b_bytes(int64_t rows, int64_t d_in);
cq_status lut_umma_grouped(const int8_t *, int8_t *, const float *, const int32_t *, int64_t, int64_t, int64_t,
                           const cq_expert_site *, float *, const cq_expert_site *, float *, int64_t, int64_t,
                           cudaStream_t, const UmmaIn &in = UmmaIn{});

cq_status lut8_prepare(const uint8_t *ids, const float *cent, int64_t rows, int64_t d_in, int64_t g, int64_t planes,
                       int64_t layout, uint8_t *tc_ids, int8_t *tc_lut, float *rowscale, cudaStream_t st) {
    if (planes != 2 && planes != 3) {
        set_error("lut8_prepare: planes must be 2 or 3");
        return CQ_ERR_CONFIG;
    }
    if (!umma_merged(layout)) {
        set_error("lut8_prepare: unknown layout (CQ_TC_UMMA128U or CQ_TC_UMMA128U8)");
        return CQ_ERR_CONFIG;
    }
    if (rows % 128 || !umma_ok(d_in, 128, g)) {
        set_error("lut8_prepare: needs rows % 128 == 0, d_in % 128 == 0, g % 128 == 0");
        return CQ_ERR_UNSUPPORTED;
    }
    if (rows == 0) return CQ_OK;
    const int64_t n_groups = d_in / g;
    const int64_t mb = (1LL << (7 * planes - 1)) - 1;
    rowscale_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(cent, rows, n_groups * 16, (double)mb, rowscale);
    CQ_TRY(check_launch("rowscale"));
    lut7_kernel<<<(unsigned)ceil_div(rows * n_groups, 128), 128, 0, st>>>(cent, rowscale, rows, n_groups, (int)planes,
                                                                        tc_lut);
    CQ_TRY(check_launch("lut7"));
    const int64_t total_ids = (rows / 128) * (d_in / 128) * 4 * 128;
    ids_umma_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total_ids, 256), 148 * 32), 256, 0, st>>>(
        ids, rows, d_in, reinterpret_cast<uint4 *>(tc_ids));
    return check_launch("ids_umma");
}

__global__ void tc_single_segment_kernel(int32_t *off, int64_t n) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    off[0] = 0;
    off[1] = (int32_t)n;
}

// single-matrix scratch: the B-operand buffer, then the 2-int segment table
static int64_t tc_gemm_ws(int64_t n, int64_t d_in) { return ceil_div(umma_b_bytes(n, d_in), 256) * 256 + 256; }

}  // namespace cq

using namespace cq;

extern "C" cq_status cq_lut8_prepare(const uint8_t *ids, const float *centroids, int64_t rows, int64_t d_in,
                                     int64_t g, int64_t planes, int64_t layout, uint8_t *tc_ids, int8_t *tc_lut,
                                     float *tc_rowscale, void *stream) {
    return lut8_prepare(ids, centroids, rows, d_in, g, planes, layout, tc_ids, tc_lut, tc_rowscale,
                        as_stream(stream));
}

extern "C" int64_t cq_lut_gemm_tc_workspace(int64_t n, int64_t d_in) {
    if (n < 0 || d_in < 0) return -1;
    return tc_gemm_ws(n, d_in);
}

extern "C" cq_status cq_lut_gemm_tc(const int8_t *codes, const float *scales, const uint8_t *tc_ids,
                                    const int8_t *tc_lut, const float *tc_rowscale, int64_t planes, int64_t layout,
                                    int64_t n, int64_t d_in, int64_t d_out, int64_t g, float *out, void *workspace,
                                    int64_t workspace_bytes, void *stream) {
    if (n < 0 || g < 1 || d_in % g) {
        set_error("group size does not divide the input dimension");
        return CQ_ERR_SHAPE;
    }
    if (n == 0 || d_out == 0) return CQ_OK;
    if (workspace == nullptr || workspace_bytes < tc_gemm_ws(n, d_in)) {
        set_error("lut_gemm_tc: workspace smaller than cq_lut_gemm_tc_workspace(n, d_in)");
        return CQ_ERR_SHAPE;
    }
    cudaStream_t st = as_stream(stream);
    cq_expert_site site{};
    site.group_size = g;
    site.tc_ids = tc_ids;
    site.tc_lut = tc_lut;
    site.tc_rowscale = tc_rowscale;
    site.tc_planes = planes;
    site.tc_layout = layout;
    int8_t *bbuf = reinterpret_cast<int8_t *>(workspace);
    int32_t *off = reinterpret_cast<int32_t *>(bbuf + tc_gemm_ws(n, d_in) - 256);
    launch_pdl(tc_single_segment_kernel, 1, 1, 0, st, off, n);
    CQ_TRY(check_launch("single_segment"));
    return lut_umma_grouped(codes, bbuf, scales, off, 1, 0, n, &site, out, nullptr, nullptr, d_in, d_out, st);
}
