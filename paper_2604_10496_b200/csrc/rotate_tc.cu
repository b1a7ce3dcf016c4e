// Online rotation v = x @ R (pipeline.py:516) on the tensor cores, at fp32
// accuracy: R is split once into three bf16 planes R = R0 + R1 + R2 (8 + 8 + 8
// significand bits), a bf16 activation x is exact in bf16, so
//   x R = x R0 + x R1 + x R2
// is one tcgen05 kind::f16 GEMM with K = 3 d and fp32 accumulation in TMEM.  An
// fp32 x is split the same way and the six largest products are kept
// (x0R0 + x0R1 + x1R0 + x0R2 + x1R1 + x2R0, dropping terms below 2^-24 relative).
//
// Operands use the canonical K-major no-swizzle UMMA layout of the LUT GEMM's
// activation tiles ([chunk 128 B][tile8][kstep 4][khalf 2][8 rows][16 B]): A =
// token rows, B = R^T rows (output columns).  CTA tile 128 tokens x 256 output
// columns, 4-deep smem ring of (A 16 KB, B 32 KB) chunks of 64 K-elements fed by
// bulk copies; warp 0 producer, warp 1 MMA issuer, warps 2-5 epilogue (one TMEM
// lane quarter each).
#include <cuda.h>  // CUtensorMap (the encode entry point comes from the runtime: no libcuda link)

#include "common.cuh"
#include "tc_ptx.cuh"

namespace cq {

namespace rt {
constexpr int BM = 128, BN = 256;          // CTA tile (tokens x output columns)
constexpr int KC = 64;                     // K elements per chunk (128 bytes of bf16)
constexpr int A_BYTES = BM * KC * 2;       // 16 KB
constexpr int B_BYTES = BN * KC * 2;       // 32 KB
constexpr int STAGES = 4;
constexpr int THREADS = 6 * 32;
}  // namespace rt

__device__ __forceinline__ uint16_t bf16_rn_bits(float x) {
    uint16_t r;
    asm("{\n\t.reg .b16 h;\n\tcvt.rn.bf16.f32 h, %1;\n\tmov.b16 %0, h;\n\t}" : "=h"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float bf16_bits_f32(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

// Three-way split: x = p0 + p1 + p2 (+ error below 2^-24 |x|), each a bf16.
__device__ __forceinline__ void split3(float x, uint16_t *p) {
    p[0] = bf16_rn_bits(x);
    const float r1 = __fsub_rn(x, bf16_bits_f32(p[0]));  // exact
    p[1] = bf16_rn_bits(r1);
    const float r2 = __fsub_rn(r1, bf16_bits_f32(p[1]));  // exact
    p[2] = bf16_rn_bits(r2);
}

// Index of the 16-byte piece x of the UMMA layout -> (row, first K element).
__device__ __forceinline__ void piece_coords(int64_t x, int64_t tiles, int64_t &row, int64_t &k0) {
    const int r = (int)(x & 7), kh = (int)((x >> 3) & 1), ks = (int)((x >> 4) & 3);
    const int64_t j = (x >> 6) % tiles, c = (x >> 6) / tiles;
    row = j * 8 + r;
    k0 = c * rt::KC + ks * 16 + kh * 8;
}

// R (d x d, row k, column n) -> three bf16 planes of R^T (rows n) in the UMMA layout.
__global__ void rot_split_r_kernel(const float *__restrict__ R, int64_t d, uint4 *__restrict__ planes) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t tiles = d / 8, per_plane = d * d / 8;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < per_plane; x += (int64_t)gridDim.x * blockDim.x) {
        int64_t n, k0;
        piece_coords(x, tiles, n, k0);
        uint16_t h[3][8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            uint16_t p[3];
            split3(__ldg(R + (k0 + e) * d + n), p);
            h[0][e] = p[0], h[1][e] = p[1], h[2][e] = p[2];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            uint4 v;
            v.x = h[q][0] | ((uint32_t)h[q][1] << 16);
            v.y = h[q][2] | ((uint32_t)h[q][3] << 16);
            v.z = h[q][4] | ((uint32_t)h[q][5] << 16);
            v.w = h[q][6] | ((uint32_t)h[q][7] << 16);
            planes[q * per_plane + x] = v;
        }
    }
}

// x (n x d, f32 or bf16) -> NP bf16 planes (1 for bf16 input: exact) in the
// UMMA layout, rows padded with zeros to `tiles` x 8.
template <int DT, int NP>
__global__ void rot_split_x_kernel(const void *__restrict__ x, int64_t n, int64_t d, int64_t tiles,
                                   uint4 *__restrict__ planes) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t per_plane = tiles * 8 * d / 8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_plane; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t row, k0;
        piece_coords(i, tiles, row, k0);
        uint16_t h[NP][8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (row >= n) {
#pragma unroll
                for (int q = 0; q < NP; ++q) h[q][e] = 0;
            } else if (DT == CQ_DTYPE_BF16) {
                h[0][e] = reinterpret_cast<const uint16_t *>(x)[row * d + k0 + e];
            } else {
                uint16_t p[3];
                split3(reinterpret_cast<const float *>(x)[row * d + k0 + e], p);
#pragma unroll
                for (int q = 0; q < NP; ++q) h[q][e] = p[q];
            }
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            uint4 v;
            v.x = h[q][0] | ((uint32_t)h[q][1] << 16);
            v.y = h[q][2] | ((uint32_t)h[q][3] << 16);
            v.z = h[q][4] | ((uint32_t)h[q][5] << 16);
            v.w = h[q][6] | ((uint32_t)h[q][7] << 16);
            planes[q * per_plane + i] = v;
        }
    }
}

// kind::f16 MMA, A and B from shared memory: D[tmem] (+)= A x B^T, 128 x N x 16, bf16 -> f32.
__device__ __forceinline__ void tc_mma_bf16_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t *v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}

// grid: (d / BN, ceil(n / BM)).  NPA: activation planes (1: bf16 input, 3: f32 input).  XT (bf16
// input): the A tiles come straight from the row-major x by TMA (xmap: [n][d] bf16, box 64 x 128,
// SWIZZLE_128B; rows past n read as zeros) instead of from planes re-laid out by rot_split_x.
template <int NPA, bool XT = false>
__global__ void __launch_bounds__(rt::THREADS, 1) rot_gemm_kernel(const uint8_t *__restrict__ xa, int64_t a_tiles,
                                                                   const uint8_t *__restrict__ rb, int64_t d,
                                                                   int64_t n, float *__restrict__ v, int npair,
                                                                   const __grid_constant__ CUtensorMap xmap) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    // (activation plane, R plane) products, largest first: x R0, x R1, x R2 for a bf16 x; for an
    // fp32 x the six terms of relative size >= 2^-16 (x0R0, x0R1, x1R0, x0R2, x1R1, x2R0).
    // npair: the leading pairs used (a bf16 x with npair = 2: R to 16 significand bits)
    const int NPAIR = npair;
    constexpr int PA1[3] = {0, 0, 0}, PB1[3] = {0, 1, 2};
    constexpr int PA3[6] = {0, 0, 1, 0, 1, 2}, PB3[6] = {0, 1, 0, 2, 1, 0};
    const int *PA = NPA == 1 ? PA1 : PA3, *PB = NPA == 1 ? PB1 : PB3;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full_bar[rt::STAGES], empty_bar[rt::STAGES], acc_bar;
    __shared__ uint32_t tmem_sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n0 = blockIdx.x * (int64_t)rt::BN, m0 = blockIdx.y * (int64_t)rt::BM;
    const int n_chunks = (int)(d / rt::KC), iters = NPAIR * n_chunks;
    const int64_t b_tiles = d / 8;
    const int64_t a_plane = a_tiles * 8 * d * 2, b_plane = d * d * 2;  // bytes per plane

    if (threadIdx.x == 0) {
        for (int s = 0; s < rt::STAGES; ++s) {
            u_bar_init(u_smem(&full_bar[s]), 1);
            u_bar_init(u_smem(&empty_bar[s]), 1);
        }
        u_bar_init(u_smem(&acc_bar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(u_smem(&tmem_sh)),
                     "r"(rt::BN)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_sh;
    const uint32_t stage0 = u_smem(smem);

    if (warp == 0) {
        // ---- producer: chunk c of pair p = (A plane, B plane)
        for (int it = 0; it < iters; ++it) {
            const int s = it % rt::STAGES, p = it / n_chunks, c = it - p * n_chunks;
            if (it >= rt::STAGES) u_bar_wait(u_smem(&empty_bar[s]), ((it / rt::STAGES) - 1) & 1);
            const uint32_t bar = u_smem(&full_bar[s]);
            const uint32_t dst = stage0 + s * (rt::A_BYTES + rt::B_BYTES);
            u_bar_expect_elect(bar, rt::A_BYTES + rt::B_BYTES);
            // A: 16 tile8 blocks of the token tile (1 KB each, contiguous); B: 32 of the column tile
            if constexpr (XT) {
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                    "[%4];\n\t}" ::"r"(dst),
                    "l"(&xmap), "r"(c * rt::KC), "r"((int)m0), "r"(bar)
                    : "memory");
            } else {
                u_bulk_elect(dst, xa + PA[p] * a_plane + ((int64_t)c * a_tiles + m0 / 8) * 1024, rt::A_BYTES, bar);
            }
            u_bulk_elect(dst + rt::A_BYTES, rb + PB[p] * b_plane + ((int64_t)c * b_tiles + n0 / 8) * 1024, rt::B_BYTES,
                         bar);
        }
    } else if (warp == 1) {
        // ---- MMA issuer: 4 k-steps of 16 per chunk, M=128, N=256
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(rt::BN >> 3) << 17) |
                               ((uint32_t)(rt::BM >> 4) << 24);
        for (int it = 0; it < iters; ++it) {
            const int s = it % rt::STAGES;
            u_bar_wait(u_smem(&full_bar[s]), (it / rt::STAGES) & 1);
            tc_fence_after();
            const uint32_t abase = stage0 + s * (rt::A_BYTES + rt::B_BYTES), bbase = abase + rt::A_BYTES;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                tc_mma_bf16_ss(tmem, XT ? smem_desc_sw128(abase + kk * 32) : smem_desc(abase + kk * 256, 128, 1024),
                               smem_desc(bbase + kk * 256, 128, 1024), idesc, (it > 0 || kk > 0) ? 1u : 0u);
            tc_commit_elect(u_smem(&empty_bar[s]));
        }
        tc_commit_elect(u_smem(&acc_bar));
    } else {
        // ---- epilogue: warp w reads TMEM lanes of quarter w % 4 (token rows), 32 columns at a time
        const int quarter = warp & 3;
        const int64_t row = m0 + quarter * 32 + lane;
        u_bar_wait(u_smem(&acc_bar), 0);
        tc_fence_after();
        for (int cb = 0; cb < rt::BN; cb += 32) {
            uint32_t r[32];
            tc_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)cb, r);
            tc_wait_ld();
            if (row < n) {
                float4 *o = reinterpret_cast<float4 *>(v + row * d + n0 + cb);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    o[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                       __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(rt::BN) : "memory");
    }
}

bool rot_tc_ok(int64_t d) { return d % rt::BN == 0 && d % rt::KC == 0; }

// R planes the bf16-activation rotation uses: 2 (R to 16 significand bits, the default) or 3 (R
// exact; CQ_ROT_PLANES=3).  Against the reference's ordered chain the 2-plane form is the more
// accurate one: its truncation (2^-17 relative per product) is far below the fp32 rounding of the
// TMEM accumulation, which it does over 2d instead of 3d products (tools/rot_err.py, PH, 3 seeds:
// max 2.07e-5 vs 2.55e-5 of the row max; the certified quantizer's band is 1.5e-4).
static int rot_planes() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CQ_ROT_PLANES");
        v = (e != nullptr && atoi(e) == 3) ? 3 : 2;
    }
    return v;
}

// prepared = [three bf16 planes of R^T in the UMMA layout: 3 d^2 * 2 B][R^T f32: d^2 * 4 B (the certified
// quantizer's ordered chains, rotq.cu)]
int64_t rot_tc_prepared_bytes(int64_t d) { return 3 * d * d * 2 + d * d * 4; }
const float *rot_tc_transposed(const void *prepared, int64_t d) {
    return reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(prepared) + 3 * d * d * 2);
}
cq_status transpose_f32(const float *R, int64_t d, float *Rt, cudaStream_t st);

// Activation planes for n tokens (f32 input needs 3, bf16 1; sized for 3).
int64_t rot_tc_act_bytes(int64_t n, int64_t d) { return 3 * ceil_div(n, rt::BM) * rt::BM * d * 2; }

cq_status rot_tc_prepare(const float *R, int64_t d, void *out, cudaStream_t st) {
    if (!rot_tc_ok(d)) {
        set_error("rotation: tensor-core path needs d_model % 256 == 0");
        return CQ_ERR_UNSUPPORTED;
    }
    rot_split_r_kernel<<<(unsigned)std::min<int64_t>(ceil_div(d * d / 8, 256), 148 * 16), 256, 0, st>>>(
        R, d, reinterpret_cast<uint4 *>(out));
    CQ_TRY(check_launch("rotation_prepare"));
    return transpose_f32(R, d, const_cast<float *>(rot_tc_transposed(out, d)), st);
}

// x [n][d] bf16 as a TMA tile map (box 64 columns x 128 rows, SWIZZLE_128B: the K-major operand
// layout with 128-byte rows).  The encoder is the driver's, reached through the runtime.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static bool x_tmap(CUtensorMap *m, const void *x, int64_t n, int64_t d) {
    static EncodeTiledFn fn = nullptr;
    if (fn == nullptr) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || f == nullptr)
            return false;
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    const cuuint32_t box[2] = {(cuuint32_t)rt::KC, (cuuint32_t)rt::BM};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(x), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// CQ_ROT_TMA=0: re-lay out x by rot_split_x instead of loading it by TMA (A/B)
static bool rot_tma_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CQ_ROT_TMA");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

cq_status rot_tc_apply(const void *x, int dtype, int64_t n, int64_t d, const void *prepared, void *act, float *v,
                       cudaStream_t st) {
    if (n == 0) return CQ_OK;
    const size_t smem = (size_t)rt::STAGES * (rt::A_BYTES + rt::B_BYTES);
    const dim3 grid((unsigned)(d / rt::BN), (unsigned)ceil_div(n, rt::BM));
    CUtensorMap xmap{};
    if (dtype == CQ_DTYPE_BF16 && rot_tma_enabled() && x_tmap(&xmap, x, n, d)) {
        cudaFuncSetAttribute(rot_gemm_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_pdl(rot_gemm_kernel<1, true>, grid, rt::THREADS, smem, st, (const uint8_t *)nullptr, (int64_t)0,
                   reinterpret_cast<const uint8_t *>(prepared), d, n, v, rot_planes(), xmap);
        return check_launch("rotation_gemm");
    }
    const int64_t tiles = ceil_div(n, rt::BM) * (rt::BM / 8);
    const int64_t pieces = tiles * 8 * d / 8;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(pieces, 256), 148 * 16);
    if (dtype == CQ_DTYPE_BF16)
        launch_pdl(rot_split_x_kernel<CQ_DTYPE_BF16, 1>, blocks, 256, 0, st, x, n, d, tiles, reinterpret_cast<uint4 *>(act));
    else
        launch_pdl(rot_split_x_kernel<CQ_DTYPE_F32, 3>, blocks, 256, 0, st, x, n, d, tiles, reinterpret_cast<uint4 *>(act));
    CQ_TRY(check_launch("rotation_split_x"));
    // the dynamic-smem opt-in is per device: set it on every launch (cheap next to the kernel)
    cudaFuncSetAttribute(rot_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(rot_gemm_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint8_t *a = reinterpret_cast<const uint8_t *>(act), *b = reinterpret_cast<const uint8_t *>(prepared);
    if (dtype == CQ_DTYPE_BF16)
        launch_pdl(rot_gemm_kernel<1>, grid, rt::THREADS, smem, st, a, tiles, b, d, n, v, rot_planes(), xmap);
    else
        launch_pdl(rot_gemm_kernel<3>, grid, rt::THREADS, smem, st, a, tiles, b, d, n, v, 6, xmap);
    return check_launch("rotation_gemm");
}

}  // namespace cq

using namespace cq;

extern "C" int64_t cq_rotation_prepared_bytes(int64_t d_model) { return rot_tc_prepared_bytes(d_model); }

extern "C" cq_status cq_rotation_prepare(const float *rotation, int64_t d_model, void *prepared, void *stream) {
    if (rotation == nullptr || prepared == nullptr || d_model <= 0) {
        set_error("rotation_prepare: null pointer or bad d_model");
        return CQ_ERR_SHAPE;
    }
    return rot_tc_prepare(rotation, d_model, prepared, as_stream(stream));
}
