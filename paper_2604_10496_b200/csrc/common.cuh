// Shared helpers for the cq_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cfloat>
#include <cstdio>
#include <string>
#include <utility>

#include "../../include/cq_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "cq_b200 targets sm_100a only"
#endif

namespace cq {

// Thread-local last error + a process-wide launch counter (cq_launch_count).
void set_error(const std::string &msg);
extern std::atomic<int64_t> g_launches;

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline cq_status check_launch(const char *what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return CQ_ERR_CUDA;
    }
    return CQ_OK;
}

#define CQ_TRY(expr)                         \
    do {                                     \
        cq_status _st = (expr);              \
        if (_st != CQ_OK) return _st;        \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// True the first time a call site asks for the current device (per-device one-time setup such
// as a kernel's dynamic shared-memory opt-in, which cudaFuncSetAttribute sets per device).
inline bool first_on_device(std::atomic<uint64_t> &seen) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    return (seen.fetch_or(bit) & bit) == 0;
}

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// quant.py:76-86 for float32: clear (bits-1)=3 low significand bits.
__device__ __forceinline__ float snap_scale(float s) {
    return __uint_as_float(__float_as_uint(s) & ~7u);
}

// quant.py:89-100 scale for one row with max|x| = mx (mx finite).
__device__ __forceinline__ float a4_scale(float mx) {
    float s = snap_scale(__fdiv_rn(mx, 7.0f));
    return mx == 0.0f ? 1.0f : s;
}

// round half away from zero (quant.py:69-73) then clip to [-8, 7].
__device__ __forceinline__ int8_t a4_code(float x, float s) {
    float r = roundf(__fdiv_rn(x, s));
    r = fminf(fmaxf(r, -8.0f), 7.0f);
    return static_cast<int8_t>(static_cast<int>(r));
}

// a4_code(x, s) given r = 1 / s (correctly rounded): t = x * r is within 2^-22 of x / s for
// |x / s| < 8 (the only range where a rounding boundary changes the clipped code), so roundf(t)
// equals roundf(x / s) unless x / s lies within 2^-19 of a half-integer; those (ties included)
// take the IEEE division.  Bit-exact with a4_code at a fraction of its instructions.
__device__ __forceinline__ int8_t a4_code_rcp(float x, float s, float r) {
    const float t = __fmul_rn(x, r);
    const float n = rintf(t);  // the nearest integer: roundf(t) except at half-integers
    // within 2^-19 of a half-integer <=> |t - n| > 0.5 - 2^-19 (t - n is exact); there roundf and
    // rintf may differ and t may differ from x / s: the IEEE division decides
    if (fabsf(t) < 8.0f && fabsf(t - n) > 0.5f - 0x1p-19f) return a4_code(x, s);
    return static_cast<int8_t>(min(max(__float2int_rn(n), -8), 7));
}

// model.py:233-237: x * sigmoid(x), sigmoid split at 0.
__device__ __forceinline__ float silu_f32(float x) {
    const bool pos = x >= 0.0f;
    const float ex = expf(pos ? -x : x);
    const float sig = pos ? __fdiv_rn(1.0f, __fadd_rn(1.0f, ex)) : __fdiv_rn(ex, __fadd_rn(1.0f, ex));
    return __fmul_rn(x, sig);
}

// Two IEEE-rounded fp32 products in one FMUL2 (sm_100): (a0 * b0, a1 * b1), each rounded like
// __fmul_rn.  The adds that consume them stay scalar __fadd_rn: ptxas keeps FMUL2 + FADD apart
// (a packed multiply-add pair would be contracted into FFMA2, one rounding).
__device__ __forceinline__ void fmul2_rn(float a0, float a1, float b0, float b1, float &c0, float &c1) {
    uint64_t a, b, c;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(c) : "l"(a), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}

// The tensor-core path's silu (silu|re-quantize kernels): the same function within a few ulp
// (fast exp2 + the hardware reciprocal of 1 + e^-|x| in [1, 2] instead of expf + IEEE division),
// a fraction of the instructions.  Its h is tolerance-checked against the ordered path, which keeps
// silu_f32.
__device__ __forceinline__ float silu_fast(float x) {
    const float ex = __expf(-fabsf(x));  // e^-|x| in (0, 1]
    float r;                             // sigmoid(|x|) = 1 / (1 + e^-|x|)
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(1.0f, ex)));
    return __fmul_rn(x, x >= 0.0f ? r : __fmul_rn(ex, r));
}

// max of |x|, |y|, |z|, |w| as bit patterns (non-negative floats order like their bits; inf and
// NaN come out >= 0x7f800000)
__device__ __forceinline__ uint32_t abs_bits4(float4 v) {
    const uint32_t a = __float_as_uint(v.x) & 0x7fffffffu, b = __float_as_uint(v.y) & 0x7fffffffu;
    const uint32_t c = __float_as_uint(v.z) & 0x7fffffffu, d = __float_as_uint(v.w) & 0x7fffffffu;
    return max(max(a, b), max(c, d));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Sum of v over the CTA (blockDim.x a multiple of 32), valid in thread 0.
__device__ __forceinline__ int block_sum_int(int v) {
    __shared__ int s_part[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w];
    return t;
}

}  // namespace cq

// ---------------------------------------------------------------------------
// Programmatic dependent launch: a kernel launched with launch_pdl may start
// (and run its prologue) while the previous kernel in the stream drains; it
// must call griddep_wait() before touching anything the previous kernel
// writes.  Under a normal launch griddep_wait() returns at once.  Disabled with
// CQ_PDL=0.
namespace cq {

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
    if (!pdl_enabled()) {
        kernel<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
        return cudaSuccess;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Route mode of the B build: the segment permutation is derived from the
// top-k in every CTA (route_perm.cuh); CTA 0 publishes it.
struct RoutePerm {
    const int32_t *selected = nullptr;  // [n_tok][k] global expert ids; nullptr = off
    int64_t n_tok = 0, local_begin = 0;
    int k = 0, n_local = 0;
    int32_t *offsets = nullptr, *counts = nullptr, *perm_token = nullptr, *perm_slot = nullptr, *inv = nullptr;
    __host__ __device__ bool on() const { return selected != nullptr; }
};

// Tensor-core layouts: UMMA128U8 is UMMA128U's data with every id < 8.
inline bool umma_merged(int64_t layout) { return layout == CQ_TC_UMMA128U || layout == CQ_TC_UMMA128U8; }
inline int64_t umma_family(int64_t layout) {
    return layout == CQ_TC_UMMA128U8 ? (int64_t)CQ_TC_UMMA128U : layout;
}

// Optional inputs of the tcgen05 grouped GEMM's B-operand build (lut_umma.cu).
struct UmmaIn {
    const int32_t *perm = nullptr;      // gather: segment row r reads codes[perm[r]] (codes per token)
    const int32_t *tok_sums = nullptr;  // gather / route: per-token code sums, gathered into the row sums
    float *scales_out = nullptr;        // gather / route: scales[perm[r]] lands here; the GEMM reads it
    bool sums_ready = false;            // otherwise: the row sums are already in the B buffer
    RoutePerm route;                    // route mode (implies the gather)
    bool b_ready = false;               // the B operand (tiles, row sums, zeroed counters) is built already
    bool gathers() const { return perm != nullptr || route.on(); }
};

// Where a re-quantizer writes its codes directly in the tcgen05 GEMM's B layout
// ([chunk CK][tile8][kstep][khalf][8 rows][16 B], lut_umma.cu's to_umma_b) and
// the counters that B build would have zeroed.  dst == nullptr: not used.
struct UmmaBOut {
    int8_t *dst = nullptr;
    int64_t tiles = 0;
    int ck = 128, ck_shift = 7;  // ck = 1 << ck_shift
    int32_t *zero = nullptr;
    int n_zero = 0;
    // byte offset of codes (row, col .. col + 3), col % 4 == 0:
    //   ((((c * tiles + row / 8) * (ck / 32) + ks) * 2 + khalf) * 8 + row % 8) * 16 + col % 16
    // with c = col / ck, ks = (col % ck) / 32, khalf = (col % 32) / 16, in shifts
    __device__ __forceinline__ int64_t off(int64_t row, int64_t col) const {
        const uint32_t cc = (uint32_t)col, c = cc >> ck_shift, r = cc & (uint32_t)(ck - 1);
        const uint32_t low = ((r >> 5) << 8) + ((r & 16u) << 3) + (((uint32_t)row & 7u) << 4) + (r & 15u);
        return (((int64_t)c * tiles + (row >> 3)) << (ck_shift + 3)) + low;
    }
};

// launch_pdl with a thread-block cluster of cluster_x CTAs along x.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      unsigned cluster_x, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster_x;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace cq
