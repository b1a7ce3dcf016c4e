// Ordered kernels that reproduce the reference's accumulation chains bit for
// bit (kernels/_core.pyx:27-38, 154-211).  They are the GPU-side oracle for
// full-size parity runs and the implementation of reference_gemm / matmul.
#include "common.cuh"

namespace cq {

// out[t,i] = s_t * (((0 + c*q_0) + c*q_1) + ...), j ascending; each warp owns
// one output row i (ids/centroids warp-uniform -> broadcast loads), lanes own
// 32 tokens; the token codes of a 64-column chunk are staged in smem.
constexpr int REF_ROWS = 8, REF_TOK = 32, REF_J = 64;

__global__ void __launch_bounds__(256) reference_gemm_kernel(
    const int8_t *__restrict__ codes, const float *__restrict__ scales,
    const uint8_t *__restrict__ ids, const float *__restrict__ cent, int64_t n, int64_t d_in,
    int64_t d_out, int64_t g, float *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int8_t tile[REF_J][REF_TOK];
    const int lane = threadIdx.x, wy = threadIdx.y;
    const int64_t t = blockIdx.x * (int64_t)REF_TOK + lane;
    const int64_t i = blockIdx.y * (int64_t)REF_ROWS + wy;
    const int64_t row_bytes = (d_in + 1) >> 1;
    const int64_t n_groups = d_in / g;
    const uint8_t *idrow = ids + (i < d_out ? i : 0) * row_bytes;
    const float *crow = cent + (i < d_out ? i : 0) * n_groups * 16;
    float acc = 0.0f;
    for (int64_t j0 = 0; j0 < d_in; j0 += REF_J) {
        __syncthreads();
        for (int e = wy * 32 + lane; e < REF_J * REF_TOK; e += 256) {
            const int tt = e / REF_J, jj = e % REF_J;
            const int64_t gt = blockIdx.x * (int64_t)REF_TOK + tt, gj = j0 + jj;
            tile[jj][tt] = (gt < n && gj < d_in) ? codes[gt * d_in + gj] : (int8_t)0;
        }
        __syncthreads();
        const int jn = (int)((d_in - j0) < REF_J ? (d_in - j0) : REF_J);
        for (int jj = 0; jj < jn; ++jj) {
            const int64_t j = j0 + jj;
            const uint8_t b = __ldg(idrow + (j >> 1));
            const int id = (j & 1) ? (b >> 4) : (b & 15);
            const float c = __ldg(crow + (j / g) * 16 + id);
            acc = __fadd_rn(acc, __fmul_rn(c, (float)tile[jj][lane]));
        }
    }
    if (t < n && i < d_out) out[t * d_out + i] = __fmul_rn(__ldg(scales + t), acc);
}

// out[m, c] = sum_k a[m,k] * b[k,c], k ascending, one rounding per op.
__global__ void matmul_ordered_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                      float *__restrict__ out, int64_t m, int64_t k, int64_t nc) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= m * nc) return;
    const int64_t r = idx / nc, c = idx - r * nc;
    const float *arow = a + r * k;
    float acc = 0.0f;
    for (int64_t kk = 0; kk < k; ++kk) acc = __fadd_rn(acc, __fmul_rn(__ldg(arow + kk), __ldg(b + kk * nc + c)));
    out[idx] = acc;
}

cq_status reference_gemm(const int8_t *codes, const float *scales, const uint8_t *ids,
                         const float *cent, int64_t n, int64_t d_in, int64_t d_out, int64_t g,
                         float *out, cudaStream_t st) {
    if (n == 0 || d_out == 0) return CQ_OK;
    if (d_in == 0) return cudaMemsetAsync(out, 0, n * d_out * 4, st) == cudaSuccess ? CQ_OK : CQ_ERR_CUDA;
    dim3 grid((unsigned)ceil_div(n, REF_TOK), (unsigned)ceil_div(d_out, REF_ROWS));
    reference_gemm_kernel<<<grid, dim3(32, REF_ROWS), 0, st>>>(codes, scales, ids, cent, n, d_in, d_out, g, out);
    return check_launch("reference_gemm");
}

cq_status validate_gemm(int64_t n, int64_t d_in, int64_t d_out, int64_t g) {
    if (n < 0 || d_in < 0 || d_out < 0) {
        set_error("gemm: negative shape");
        return CQ_ERR_SHAPE;
    }
    if (g < 1 || (d_in % g) != 0) {
        set_error("group size does not divide the input dimension");
        return CQ_ERR_SHAPE;
    }
    return CQ_OK;
}

}  // namespace cq

using namespace cq;

extern "C" cq_status cq_reference_gemm_f32(const int8_t *codes, const float *scales,
                                           const uint8_t *ids_packed, const float *centroids,
                                           int64_t n, int64_t d_in, int64_t d_out, int64_t g,
                                           float *out, void *stream) {
    CQ_TRY(validate_gemm(n, d_in, d_out, g));
    return reference_gemm(codes, scales, ids_packed, centroids, n, d_in, d_out, g, out, as_stream(stream));
}

extern "C" cq_status cq_matmul_f32(const float *a, const float *b, float *out, int64_t m, int64_t k,
                                   int64_t n, void *stream) {
    if (m < 0 || k < 0 || n < 0) {
        set_error("matmul: negative shape");
        return CQ_ERR_SHAPE;
    }
    if (m * n == 0) return CQ_OK;
    matmul_ordered_kernel<<<(unsigned)ceil_div(m * n, 256), 256, 0, as_stream(stream)>>>(a, b, out, m, k, n);
    return check_launch("matmul_ordered");
}
