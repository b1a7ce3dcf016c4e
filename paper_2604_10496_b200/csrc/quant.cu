// Per-token A4 quantization (quant.py:89-100) and nibble unpack
// (kernels/fallback.py:35-42), both bit-exact.
#include "common.cuh"

namespace cq {

template <int DT>
__device__ __forceinline__ float load_x(const void *x, int64_t idx) {
    if (DT == CQ_DTYPE_F32) return __ldg(reinterpret_cast<const float *>(x) + idx);
    return bf16_bits_to_f32(__ldg(reinterpret_cast<const uint16_t *>(x) + idx));
}

// One CTA per row.  Pass 1: max|x| (order-free, exact) + finiteness; pass 2:
// codes with the IEEE-division recipe of common.cuh (no fast math anywhere).
template <int DT>
__global__ void __launch_bounds__(256) quantize_a4_kernel(const void *__restrict__ x, int64_t d,
                                                          int8_t *__restrict__ codes,
                                                          float *__restrict__ scales,
                                                          int *__restrict__ nonfinite,
                                                          float *__restrict__ deq, int32_t *__restrict__ tsum,
                                                          int32_t *__restrict__ zero, int n_zero) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t row = blockIdx.x;
    if (row == 0)  // counters the next kernels accumulate into (route counts)
        for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
    const int64_t base = row * d;
    float mx = 0.0f;
    bool bad = false;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
        float v = load_x<DT>(x, base + j);
        bad |= !isfinite(v);
        mx = fmaxf(mx, fabsf(v));
    }
    __shared__ float red[8];
    __shared__ float s_sh;
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    if (nonfinite != nullptr && __syncthreads_or(bad) && threadIdx.x == 0) atomicExch(nonfinite, 1);
    __syncthreads();
    if (threadIdx.x < 32) {
        float m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0) {
            float s = a4_scale(m);
            s_sh = s;
            scales[row] = s;
        }
    }
    __syncthreads();
    const float s = s_sh;
    int csum = 0;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
        const int8_t c = a4_code(load_x<DT>(x, base + j), s);
        codes[base + j] = c;
        csum += c;
        // dequantized value, rounded exactly as codes.astype(f32) * scales (model.py:379-381)
        if (deq != nullptr) deq[base + j] = __fmul_rn((float)c, s);
    }
    if (tsum != nullptr) {  // sum of the row's codes (exact): the unsigned-digit bias term of the GEMM
        __shared__ int ired[8];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
        if ((threadIdx.x & 31) == 0) ired[threadIdx.x >> 5] = csum;
        __syncthreads();
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ired[w];
            tsum[row] = t;
        }
    }
}

// Same quantizer with the row held in registers (d % 4 == 0, d <= 8192): 256
// threads x V groups of 4 values, loaded once with 16-byte (fp32) / 8-byte
// (bf16) loads; codes, dequantized values and code sums as before.
// TH threads per row (256, or 128 for short rows: more rows in flight per SM).
template <int DT, int V, int TH = 256>
__global__ void __launch_bounds__(TH) quantize_a4_vec_kernel(const void *__restrict__ x, int64_t d,
                                                              int8_t *__restrict__ codes,
                                                              float *__restrict__ scales,
                                                              int *__restrict__ nonfinite,
                                                              float *__restrict__ deq, int32_t *__restrict__ tsum,
                                                              int32_t *__restrict__ zero, int n_zero) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t row = blockIdx.x;
    if (row == 0)
        for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
    const int nv = (int)(d >> 2);
    float h[V][4];
    float mx = 0.0f;
    bool bad = false;
#pragma unroll
    for (int u = 0; u < V; ++u) {
        const int j = threadIdx.x + u * TH;
        if (j < nv) {
            if (DT == CQ_DTYPE_F32) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(x) + row * nv + j);
                h[u][0] = v.x, h[u][1] = v.y, h[u][2] = v.z, h[u][3] = v.w;
            } else {
                const uint2 v = __ldg(reinterpret_cast<const uint2 *>(x) + row * nv + j);
                h[u][0] = __uint_as_float(v.x << 16), h[u][1] = __uint_as_float(v.x & 0xFFFF0000u);
                h[u][2] = __uint_as_float(v.y << 16), h[u][3] = __uint_as_float(v.y & 0xFFFF0000u);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bad |= !isfinite(h[u][q]);
                mx = fmaxf(mx, fabsf(h[u][q]));
            }
        }
    }
    __shared__ float red[8];
    __shared__ float s_sh;
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    if (nonfinite != nullptr && __syncthreads_or(bad) && threadIdx.x == 0) atomicExch(nonfinite, 1);
    __syncthreads();
    if (threadIdx.x < 32) {
        float m = threadIdx.x < TH / 32 ? red[threadIdx.x] : 0.0f;
        m = warp_max(m);
        if (threadIdx.x == 0) {
            const float sc = a4_scale(m);
            s_sh = sc;
            scales[row] = sc;
        }
    }
    __syncthreads();
    const float sc = s_sh;
    const float rs = __frcp_rn(sc);
    int csum = 0;
#pragma unroll
    for (int u = 0; u < V; ++u) {
        const int j = threadIdx.x + u * TH;
        if (j < nv) {
            const char4 c = make_char4(a4_code_rcp(h[u][0], sc, rs), a4_code_rcp(h[u][1], sc, rs),
                                       a4_code_rcp(h[u][2], sc, rs), a4_code_rcp(h[u][3], sc, rs));
            reinterpret_cast<char4 *>(codes + row * d)[j] = c;
            csum += c.x + c.y + c.z + c.w;
            // dequantized value, rounded exactly as codes.astype(f32) * scales (model.py:379-381)
            if (deq != nullptr)
                reinterpret_cast<float4 *>(deq + row * d)[j] =
                    make_float4(__fmul_rn((float)c.x, sc), __fmul_rn((float)c.y, sc), __fmul_rn((float)c.z, sc),
                                __fmul_rn((float)c.w, sc));
        }
    }
    if (tsum != nullptr) {
        const int t = block_sum_int(csum);
        if (threadIdx.x == 0) tsum[row] = t;
    }
}

__global__ void unpack_ids_kernel(const uint8_t *__restrict__ packed, int64_t rows, int64_t d_in,
                                  uint8_t *__restrict__ ids) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t row_bytes = (d_in + 1) >> 1;
    const int64_t total = rows * d_in;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / d_in, j = idx - r * d_in;
        const uint8_t b = packed[r * row_bytes + (j >> 1)];
        ids[idx] = (j & 1) ? (uint8_t)(b >> 4) : (uint8_t)(b & 15);
    }
}

// deq (nullable): also write code * scale as f32 (the router's input).
// tsum (nullable): per-row code sums.  zero[0..n_zero) is cleared by CTA 0.
cq_status quantize_a4(const void *x, int dtype, int64_t n, int64_t d, int8_t *codes, float *scales,
                      int *nonfinite_dev, float *deq, cudaStream_t st, int32_t *tsum, int32_t *zero, int n_zero) {
    if (n == 0) return CQ_OK;
    if (d % 4 == 0 && d <= 8 * 1024) {  // row in registers
        // short rows (d <= 2048) on 128-thread CTAs (more rows in flight per SM), else 256
        const bool small = d <= 2048;
        const int64_t v = ceil_div(d / 4, small ? 128 : 256);
#define CQ_QVEC(DT_, V_)                                                                                             \
    (small ? launch_pdl(quantize_a4_vec_kernel<DT_, V_, 128>, (unsigned)n, 128, 0, st, x, d, codes, scales,           \
                        nonfinite_dev, deq, tsum, zero, n_zero)                                                       \
           : launch_pdl(quantize_a4_vec_kernel<DT_, V_, 256>, (unsigned)n, 256, 0, st, x, d, codes, scales,           \
                        nonfinite_dev, deq, tsum, zero, n_zero))
        if (dtype == CQ_DTYPE_F32) {
            if (v == 1) CQ_QVEC(CQ_DTYPE_F32, 1); else if (v == 2) CQ_QVEC(CQ_DTYPE_F32, 2);
            else if (v <= 4) CQ_QVEC(CQ_DTYPE_F32, 4); else CQ_QVEC(CQ_DTYPE_F32, 8);
        } else {
            if (v == 1) CQ_QVEC(CQ_DTYPE_BF16, 1); else if (v == 2) CQ_QVEC(CQ_DTYPE_BF16, 2);
            else if (v <= 4) CQ_QVEC(CQ_DTYPE_BF16, 4); else CQ_QVEC(CQ_DTYPE_BF16, 8);
        }
#undef CQ_QVEC
        return check_launch("quantize_a4");
    }
    if (dtype == CQ_DTYPE_F32)
        launch_pdl(quantize_a4_kernel<CQ_DTYPE_F32>, (unsigned)n, 256, 0, st, x, d, codes, scales, nonfinite_dev, deq,
                   tsum, zero, n_zero);
    else
        launch_pdl(quantize_a4_kernel<CQ_DTYPE_BF16>, (unsigned)n, 256, 0, st, x, d, codes, scales, nonfinite_dev, deq,
                   tsum, zero, n_zero);
    return check_launch("quantize_a4");
}

}  // namespace cq

using namespace cq;

extern "C" cq_status cq_quantize_a4(const void *x, int dtype, int64_t n, int64_t d, int8_t *codes,
                                    float *scales, int32_t *nonfinite, void *stream) {
    if (n < 0 || d < 0) {
        set_error("quantize: negative shape");
        return CQ_ERR_SHAPE;
    }
    if (dtype != CQ_DTYPE_F32 && dtype != CQ_DTYPE_BF16) {
        set_error("quantize: dtype must be float32 or bfloat16");
        return CQ_ERR_SHAPE;
    }
    if (n == 0) return CQ_OK;
    if (d == 0) {  // empty rows: max over nothing -> reference errors; mirror as shape
        set_error("quantize: zero-width rows");
        return CQ_ERR_SHAPE;
    }
    // no host sync: a non-finite row sets *nonfinite (sticky), read by the caller at its next sync
    return quantize_a4(x, dtype, n, d, codes, scales, reinterpret_cast<int *>(nonfinite), nullptr, as_stream(stream),
                       nullptr, nullptr, 0);
}

extern "C" cq_status cq_unpack_ids(const uint8_t *packed, int64_t rows, int64_t d_in, uint8_t *ids,
                                   void *stream) {
    if (rows < 0 || d_in < 0) {
        set_error("unpack: negative shape");
        return CQ_ERR_SHAPE;
    }
    if (rows * d_in == 0) return CQ_OK;
    int64_t blocks = ceil_div(rows * d_in, 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    unpack_ids_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(packed, rows, d_in, ids);
    return check_launch("unpack_ids");
}
