// Ordered GEMMs: bit-exact restatements of the reference's accumulation chains
// (kernels/_core.pyx:27-38 matmul_f32; :41-151 lut_gemm_f32; :154-211
// reference_gemm_f32) on the CUDA cores.
//
//   out[r, c] = ((((0 + a[r,0] * b[0,c]) + a[r,1] * b[1,c]) + ...) + a[r,K-1] * b[K-1,c])
//
// one IEEE rounding per multiply and per add (__fmul_rn / __fadd_rn are never
// contracted into FMA), k strictly ascending; for the LUT GEMM b[k, c] is the
// centroid C[c, k/g, id[c, k]] and the row's token scale multiplies the chain
// once at the end (_core.pyx:110).  The table entry of the reference,
// T[id][q+8] = C_id * float(q) (lutgemm.py:45-50), is the same single fp32
// product, so the LUT and per-element forms are bitwise equal.
//
// Tiling.  Each output element is one sequential chain; the parallelism is
// over (row, column).  A CTA owns a TM x TN output tile, 256 threads each
// hold a (TM/16) x (TN/16) register tile of independent chains (16-64 chains
// per thread hide the 4-cycle FADD latency), and k advances in 32-wide chunks
// staged in shared memory: A as [TM][33] floats (conflict-free, broadcast
// reads), B as [32][TN] floats read as float4.  For the LUT B operand with
// 32 | g, a chunk lies inside one codebook group: the chunk's 16 packed id
// bytes per row and the group's 16 centroids per row are staged once, and the
// B tile is expanded from them in shared memory.
//
// Grouped form (the MoE ordered path): segment s covers rows offsets[s] ..
// offsets[s+1] and uses expert seg_first + s; CTAs are a flat list of
// (segment, row tile) found on the device from the offsets, so no host sync.
#include "common.cuh"

namespace cq {

enum { OA_I8 = 0, OA_F32 = 1, OA_BF16 = 2 };
enum { OB_LUT = 0, OB_LUT32 = 1, OB_DENSE = 2 };  // LUT32: the staged form (32 | K, 32 | g)

struct OrdArgs {
    const void *a;             // [rows][K]
    const float *a_scale;      // LUT: per-row token scale (applied once at the end); nullable
    const int32_t *offsets;    // segments [n_seg + 1]; nullptr = one segment of m rows
    int64_t m, n_seg, seg_first;
    const uint8_t *ids;        // LUT: [E][N][ceil(K/2)]
    const float *cent;         // LUT: [E][N][K/g][16]
    int64_t g;
    const float *bd;           // dense: [K][N]
    int64_t K, N;
    float *out;                // [rows][N]
};

constexpr int OKC = 32;  // k per chunk

template <int AK>
__device__ __forceinline__ float ord_a(const void *a, int64_t idx) {
    if (AK == OA_I8) return (float)reinterpret_cast<const int8_t *>(a)[idx];
    if (AK == OA_F32) return reinterpret_cast<const float *>(a)[idx];
    return bf16_bits_to_f32(reinterpret_cast<const uint16_t *>(a)[idx]);
}

template <int AK, int BK, int TM, int TN>
__global__ void __launch_bounds__(256) ordered_tile_kernel(OrdArgs p) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    constexpr int TMT = TM / 16, TNT = TN / 16;
    __shared__ __align__(16) float As[TM][OKC + 1];
    __shared__ __align__(16) float Bs[OKC][TN];
    __shared__ __align__(16) uint4 ids_s[BK == OB_LUT32 ? TN : 1];
    __shared__ float cent_s[BK == OB_LUT32 ? TN : 1][17];
    __shared__ int64_t seg_sh[3];

    // which (segment, row tile) this CTA is: warp 0 scans the segments' tile
    // counts 32 at a time (offsets are device data: no host sync)
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int64_t tile = blockIdx.x;
        if (p.offsets == nullptr) {
            if (lane == 0) {
                seg_sh[0] = tile * TM;
                seg_sh[1] = p.m;
                seg_sh[2] = 0;
            }
        } else {
            if (lane == 0) seg_sh[0] = seg_sh[1] = 0;  // past the last tile: no work
            int64_t before = 0;
            for (int64_t s0 = 0; s0 < p.n_seg; s0 += 32) {
                const int64_t s = s0 + lane;
                int64_t b = 0, en = 0;
                if (s < p.n_seg) {
                    b = p.offsets[s];
                    en = p.offsets[s + 1];
                }
                const int64_t nt = en > b ? (en - b + TM - 1) / TM : 0;
                int64_t incl = nt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int64_t excl = before + incl - nt;
                if (nt > 0 && tile >= excl && tile < excl + nt) {  // exactly one lane of one batch
                    seg_sh[0] = b + (tile - excl) * TM;
                    seg_sh[1] = en;
                    seg_sh[2] = p.seg_first + s;
                }
                before += __shfl_sync(0xffffffffu, incl, 31);
                if (tile < before) break;  // warp-uniform
            }
        }
    }
    __syncthreads();
    const int64_t m0 = seg_sh[0], re = seg_sh[1], e = seg_sh[2];
    if (m0 >= re) return;
    const int64_t n0 = (int64_t)blockIdx.y * TN;
    const int64_t K = p.K, N = p.N;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t row_bytes = (K + 1) >> 1, n_groups = K / p.g;

    float acc[TMT][TNT];
#pragma unroll
    for (int i = 0; i < TMT; ++i)
#pragma unroll
        for (int j = 0; j < TNT; ++j) acc[i][j] = 0.0f;

    for (int64_t k0 = 0; k0 < K; k0 += OKC) {
        // ---- A chunk: rows m0 .. m0+TM, columns k0 .. k0+32 (zero outside)
        for (int x = tid; x < TM * OKC; x += 256) {
            const int kk = x % OKC, mm = x / OKC;
            const int64_t r = m0 + mm, k = k0 + kk;
            As[mm][kk] = (r < re && k < K) ? ord_a<AK>(p.a, r * K + k) : 0.0f;
        }
        // ---- B chunk: [32][TN]
        if (BK == OB_DENSE) {
            for (int x = tid; x < OKC * TN; x += 256) {
                const int nn = x % TN, kk = x / TN;
                const int64_t c = n0 + nn, k = k0 + kk;
                Bs[kk][nn] = (c < N && k < K) ? __ldg(p.bd + k * N + c) : 0.0f;
            }
        } else if (BK == OB_LUT) {
            for (int x = tid; x < OKC * TN; x += 256) {
                const int nn = x % TN, kk = x / TN;
                const int64_t c = n0 + nn, k = k0 + kk;
                float v = 0.0f;
                if (c < N && k < K) {
                    const int64_t rr = e * N + c;
                    const uint8_t b = __ldg(p.ids + rr * row_bytes + (k >> 1));
                    const int id = (k & 1) ? (b >> 4) : (b & 15);
                    v = __ldg(p.cent + (rr * n_groups + k / p.g) * 16 + id);
                }
                Bs[kk][nn] = v;
            }
        } else {  // OB_LUT32: one group per chunk; stage its centroids when the group changes
            if (k0 % p.g == 0) {
                const int64_t grp = k0 / p.g;
                for (int x = tid; x < TN * 16; x += 256) {
                    const int nn = x >> 4, c = x & 15;
                    const int64_t col = n0 + nn;
                    cent_s[nn][c] = col < N ? __ldg(p.cent + ((e * N + col) * n_groups + grp) * 16 + c) : 0.0f;
                }
            }
            for (int x = tid; x < TN; x += 256) {
                const int64_t col = n0 + x;
                ids_s[x] = col < N ? __ldg(reinterpret_cast<const uint4 *>(p.ids + (e * N + col) * row_bytes + (k0 >> 1)))
                                   : make_uint4(0, 0, 0, 0);
            }
            __syncthreads();
            // 8 consecutive k of one column per step: one 32-bit word of ids
            for (int x = tid; x < TN * (OKC / 8); x += 256) {
                const int nn = x % TN, k8 = x / TN;
                const uint4 w4 = ids_s[nn];
                const uint32_t w = k8 == 0 ? w4.x : (k8 == 1 ? w4.y : (k8 == 2 ? w4.z : w4.w));
#pragma unroll
                for (int u = 0; u < 8; ++u) Bs[k8 * 8 + u][nn] = cent_s[nn][(w >> (4 * u)) & 15];
            }
        }
        __syncthreads();
        // ---- the chains: k ascending inside the chunk
#pragma unroll 4
        for (int kk = 0; kk < OKC; ++kk) {
            float a[TMT], b[TNT];
#pragma unroll
            for (int i = 0; i < TMT; ++i) a[i] = As[ty * TMT + i][kk];
#pragma unroll
            for (int j = 0; j < TNT; j += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(&Bs[kk][tx * TNT + j]);
                b[j] = v.x;
                b[j + 1] = v.y;
                b[j + 2] = v.z;
                b[j + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < TMT; ++i)
#pragma unroll
                for (int j = 0; j < TNT; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
        }
        __syncthreads();
    }
    // ---- epilogue: the token scale once (LUT), then store
#pragma unroll
    for (int i = 0; i < TMT; ++i) {
        const int64_t r = m0 + ty * TMT + i;
        if (r >= re) continue;
        const float s = p.a_scale != nullptr ? __ldg(p.a_scale + r) : 1.0f;
#pragma unroll
        for (int j = 0; j < TNT; ++j) {
            const int64_t c = n0 + tx * TNT + j;
            if (c < N) p.out[r * N + c] = p.a_scale != nullptr ? __fmul_rn(s, acc[i][j]) : acc[i][j];
        }
    }
}

// Two tile shapes: 64 x 128 (4 x 8 chains per thread) for many rows, 16 x 128
// (1 x 8) for decode-sized segments.
template <int AK, int BK>
static cq_status ordered_launch(const OrdArgs &p, int64_t rows_bound, bool small, cudaStream_t st) {
    const int64_t segs = p.offsets != nullptr ? p.n_seg : 1;
    if (small) {
        constexpr int TM = 16, TN = 128;
        dim3 grid((unsigned)(ceil_div(rows_bound, TM) + (p.offsets ? segs : 0)), (unsigned)ceil_div(p.N, TN));
        launch_pdl(ordered_tile_kernel<AK, BK, TM, TN>, grid, 256, 0, st, p);
    } else {
        constexpr int TM = 64, TN = 128;
        dim3 grid((unsigned)(ceil_div(rows_bound, TM) + (p.offsets ? segs : 0)), (unsigned)ceil_div(p.N, TN));
        launch_pdl(ordered_tile_kernel<AK, BK, TM, TN>, grid, 256, 0, st, p);
    }
    return check_launch("ordered_gemm");
}

// rows per segment (average) below which the 16-row tile wins
static bool ordered_small(int64_t rows_bound, int64_t segs) { return rows_bound <= 32 * (segs > 0 ? segs : 1); }

// LUT GEMM (int8 codes, 4- or 8-bit values) over segments; offsets == nullptr: one segment of rows_bound rows.
cq_status ordered_lut(const int8_t *codes, const float *scales, const int32_t *offsets, int64_t n_seg, int64_t seg_first,
                      int64_t rows_bound, const uint8_t *ids, const float *cent, int64_t d_in, int64_t d_out, int64_t g,
                      float *out, cudaStream_t st) {
    if (rows_bound == 0 || d_out == 0 || (offsets != nullptr && n_seg == 0)) return CQ_OK;
    if (d_in == 0) {  // every chain is the empty sum (+0), times the scale
        if (offsets != nullptr) {
            set_error("ordered GEMM: empty inner dimension in grouped form");
            return CQ_ERR_SHAPE;
        }
        return cudaMemsetAsync(out, 0, rows_bound * d_out * 4, st) == cudaSuccess ? CQ_OK : CQ_ERR_CUDA;
    }
    OrdArgs p{};
    p.a = codes;
    p.a_scale = scales;
    p.offsets = offsets;
    p.m = rows_bound;
    p.n_seg = n_seg;
    p.seg_first = seg_first;
    p.ids = ids;
    p.cent = cent;
    p.g = g;
    p.K = d_in;
    p.N = d_out;
    p.out = out;
    const bool small = ordered_small(rows_bound, offsets ? n_seg : 1);
    if (d_in % OKC == 0 && g % OKC == 0) return ordered_launch<OA_I8, OB_LUT32>(p, rows_bound, small, st);
    return ordered_launch<OA_I8, OB_LUT>(p, rows_bound, small, st);
}

// Dense ordered matmul out (m, n) = a (m, k) @ b (k, n); a float32 or bfloat16 (exact upcast).
cq_status ordered_matmul(const void *a, int dtype, const float *b, int64_t m, int64_t k, int64_t n, float *out,
                         cudaStream_t st) {
    if (m == 0 || n == 0) return CQ_OK;
    if (k == 0) return cudaMemsetAsync(out, 0, m * n * 4, st) == cudaSuccess ? CQ_OK : CQ_ERR_CUDA;
    OrdArgs p{};
    p.a = a;
    p.m = m;
    p.bd = b;
    p.K = k;
    p.N = n;
    p.out = out;
    p.g = 1;
    const bool small = m <= 32;
    if (dtype == CQ_DTYPE_BF16) return ordered_launch<OA_BF16, OB_DENSE>(p, m, small, st);
    return ordered_launch<OA_F32, OB_DENSE>(p, m, small, st);
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

// reference_gemm_f32 (_core.pyx:154-211) and lut_gemm_f32 (_core.pyx:41-151)
// compute the same chains, so both entry points are the same bit-exact kernel
// (the reference asserts lut_gemm == reference_gemm bytewise,
// tests/test_acceptance.py:358-387).
extern "C" cq_status cq_reference_gemm_f32(const int8_t *codes, const float *scales, const uint8_t *ids_packed,
                                           const float *centroids, int64_t n, int64_t d_in, int64_t d_out, int64_t g,
                                           float *out, void *stream) {
    CQ_TRY(validate_gemm(n, d_in, d_out, g));
    return ordered_lut(codes, scales, nullptr, 0, 0, n, ids_packed, centroids, d_in, d_out, g, out, as_stream(stream));
}

extern "C" cq_status cq_lut_gemm_f32(const int8_t *codes, const float *scales, const uint8_t *ids_packed,
                                     const float *centroids, int64_t n, int64_t d_in, int64_t d_out, int64_t g,
                                     float *out, void *stream) {
    CQ_TRY(validate_gemm(n, d_in, d_out, g));
    return ordered_lut(codes, scales, nullptr, 0, 0, n, ids_packed, centroids, d_in, d_out, g, out, as_stream(stream));
}

extern "C" cq_status cq_matmul_f32(const float *a, const float *b, float *out, int64_t m, int64_t k, int64_t n,
                                   void *stream) {
    if (m < 0 || k < 0 || n < 0) {
        set_error("matmul: negative shape");
        return CQ_ERR_SHAPE;
    }
    return ordered_matmul(a, CQ_DTYPE_F32, b, m, k, n, out, as_stream(stream));
}
