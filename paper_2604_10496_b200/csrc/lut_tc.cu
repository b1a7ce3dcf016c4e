// Tensor-core LUT GEMM: 16-entry codebooks expanded through PRMT byte lookups
// into int8 digit planes, multiplied against int8 activation codes on the
// tensor cores with exact int32 accumulation.
//
// Why digit planes.  The reference multiplies fp32 centroids by 4-bit codes
// (kernels/_core.pyx:41-151).  A bf16 centroid fails the layer tolerance (the
// down input is re-quantized to 4 bits), so every centroid of
// a weight row is written as an integer m = rint(c / rowscale) split into
// base-255 digits d_p in [-128, 126]:  c ~= rowscale * sum_p 255^p d_p.
// 3 planes keep 23 bits of the row max (gate/up, whose output is re-quantized),
// 2 planes 15 bits (down).  Codes are exact int8, so each plane's GEMM is an
// exact s8 x s8 -> s32 MMA and the planes are combined once in the epilogue.
//
// Why PRMT.  A (row, group) codebook is a 16-entry byte table per plane held
// in 4 registers.  `prmt.b32` selects 4 bytes out of 8 with one 4-bit
// selector per output byte — and four consecutive packed ids ARE such a
// selector (two ids per byte, low nibble first, lutgemm.py:111-116).  Ids 8..15
// set the selector's sign-replicate bit, so one PRMT against entries 0..7 and
// one against entries 8..15 (selector ^ 0x8888) each yield the right byte for
// their half and 0x00/0xFF "sign garbage" for the other half.  Both halves go
// through the MMA as separate K-slices (their sum is the lookup); the garbage
// is cancelled offline by pre-compensating each pair (a, a+8) of table
// entries (cq_lut8_prepare).  Cost: 2 PRMT per 4 weights per plane, no masks.
//
// Data path per warp: a 16-row weight tile streams through a private ring of
// cp.async.bulk stages (1 KB of fragment-ordered ids per 128 columns + the
// group's LUT block), completion on an mbarrier; activation codes come in
// mma.m16n8k32 B-fragment order straight from L1/L2; accumulators stay in
// registers (planes x 4 token tiles x 4).  Gate and up rows are computed by
// a warp pair and fused through shared memory into silu(a) * b.
#include "common.cuh"

namespace cq {

constexpr int TC_STAGES = 4;
constexpr int TC_CHUNK = 128;   // columns per stage
constexpr int TC_IDS = 1024;    // 16 rows x 128 columns x 4 bits
constexpr int TC_NT = 4;        // token tiles of 8 per pass
constexpr int TC_WARPS = 8;
constexpr int64_t TC_M3 = 126LL * (1 + 255 + 255 * 255) - 2;  // |m| bound, 3 planes
constexpr int64_t TC_M2 = 126LL * (1 + 255) - 1;              // |m| bound, 2 planes

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

__device__ __forceinline__ void mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---------------------------------------------------------------------------
// The GEMM.  P = digit planes of the streamed site(s); GLU = gate|up pair.

template <int P>
struct TcStage {
    static constexpr int LUT = 16 * P * 16;  // 16 rows x P planes x 16 entries
    static constexpr int B = TC_NT * 1024;    // activation fragments: NT tiles x 4 k32 x 32 lanes x 8 B
    static constexpr int BYTES = TC_IDS + LUT + B;
};

template <int P>
__device__ __forceinline__ double combine_planes(const int (&acc)[P][TC_NT][4], int nt, int r) {
    double s = (double)acc[P - 1][nt][r];
#pragma unroll
    for (int p = P - 2; p >= 0; --p) s = s * 255.0 + (double)acc[p][nt][r];
    return s;
}

template <int P, bool GLU>
__global__ void __launch_bounds__(TC_WARPS * 32) lut_tc_kernel(
    const uint2 *__restrict__ codes_frag, int64_t n_tiles, const float *__restrict__ scales,
    const int32_t *__restrict__ offsets, int64_t seg_first, const uint8_t *__restrict__ ids_a, const int8_t *__restrict__ lut_a,
    const float *__restrict__ rs_a, const uint8_t *__restrict__ ids_b, const int8_t *__restrict__ lut_b,
    const float *__restrict__ rs_b, int d_in, int d_out, int g, float *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    extern __shared__ __align__(128) uint8_t smem[];
    constexpr int SB = TcStage<P>::BYTES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g8 = lane >> 2, t4 = lane & 3;
    uint8_t *ring = smem + warp * TC_STAGES * SB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + TC_WARPS * TC_STAGES * SB) + warp * TC_STAGES;
    float *xbuf = reinterpret_cast<float *>(smem + TC_WARPS * TC_STAGES * SB + TC_WARPS * TC_STAGES * 8);

    const int tiles_per_cta = GLU ? TC_WARPS / 2 : TC_WARPS;
    const int rowtile = blockIdx.x * tiles_per_cta + (GLU ? (warp >> 1) : warp);
    const int mat = GLU ? (warp & 1) : 0;
    const int64_t seg = blockIdx.y;
    const int64_t rb = offsets[seg], re = offsets[seg + 1];
    if (rb >= re || rowtile * 16 >= d_out) return;  // uniform per warp pair

    const int64_t e = seg + seg_first;
    const int n_chunks = d_in / TC_CHUNK, cpg = g / TC_CHUNK;
    const int64_t tile_g = e * (d_out / 16) + rowtile;
    const uint8_t *ids = (mat ? ids_b : ids_a) + tile_g * (int64_t)n_chunks * TC_IDS;
    const int8_t *lut = (mat ? lut_b : lut_a) + tile_g * (int64_t)(d_in / g) * TcStage<P>::LUT;
    const float *rsp = (mat ? rs_b : rs_a) + e * (int64_t)d_out + rowtile * 16;
    const float rs0 = __ldg(rsp + g8), rs1 = __ldg(rsp + g8 + 8);

    if (lane == 0) {
        for (int s = 0; s < TC_STAGES; ++s) mbar_init(smem_addr(bars + s), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // one stage = 128 columns: fragment-ordered ids, the group's LUT block when
    // the chunk opens a group, and the ntc activation tiles of this chunk
    auto issue = [&](int chunk, int stage, int64_t j0, int ntc) {
        const uint32_t dst = smem_addr(ring + stage * SB);
        const uint32_t bar = smem_addr(bars + stage);
        const bool new_group = (chunk % cpg) == 0;
        mbar_expect_tx(bar, TC_IDS + (new_group ? TcStage<P>::LUT : 0) + ntc * 1024);
        bulk_g2s(dst, ids + (int64_t)chunk * TC_IDS, TC_IDS, bar);
        if (new_group) bulk_g2s(dst + TC_IDS, lut + (int64_t)(chunk / cpg) * TcStage<P>::LUT, TcStage<P>::LUT, bar);
        bulk_g2s(dst + TC_IDS + TcStage<P>::LUT, codes_frag + ((int64_t)chunk * n_tiles + j0) * 128, ntc * 1024, bar);
    };

    const int64_t j_first = rb >> 3, j_last = (re - 1) >> 3;
    uint32_t cnt = 0;  // chunks consumed by this warp (ring position + phase)
    for (int64_t j0 = j_first; j0 <= j_last; j0 += TC_NT) {
        const int ntc = (int)((j_last - j0 + 1) < TC_NT ? (j_last - j0 + 1) : TC_NT);
        int acc[P][TC_NT][4];
#pragma unroll
        for (int p = 0; p < P; ++p)
#pragma unroll
            for (int nt = 0; nt < TC_NT; ++nt)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[p][nt][r] = 0;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int c = 0; c < TC_STAGES && c < n_chunks; ++c) issue(c, (cnt + c) % TC_STAGES, j0, ntc);
        }
        uint4 L0[P], L1[P];  // LUT planes of rows g8 and g8 + 8
        for (int c = 0; c < n_chunks; ++c, ++cnt) {
            const int stage = cnt % TC_STAGES;
            mbar_wait(smem_addr(bars + stage), (cnt / TC_STAGES) & 1);
            const uint8_t *st = ring + stage * SB;
            if (c % cpg == 0) {
                const uint4 *lb = reinterpret_cast<const uint4 *>(st + TC_IDS);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    L0[p] = lb[g8 * P + p];
                    L1[p] = lb[(g8 + 8) * P + p];
                }
            }
            const uint4 h0 = reinterpret_cast<const uint4 *>(st)[lane];
            const uint4 h1 = reinterpret_cast<const uint4 *>(st)[32 + lane];
            const uint32_t wv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {
                const uint2 *bs = reinterpret_cast<const uint2 *>(st + TC_IDS + TcStage<P>::LUT);
                uint2 b[TC_NT];
#pragma unroll
                for (int nt = 0; nt < TC_NT; ++nt)
                    if (nt < ntc) b[nt] = bs[(nt * 4 + sub) * 32 + lane];
                const uint32_t w0 = wv[2 * sub], w1 = wv[2 * sub + 1];
                const uint32_t x0 = w0 ^ 0x88888888u, x1 = w1 ^ 0x88888888u;
                // selectors (low 16 bits used): a0 row g k-lo, a1 row g+8 k-lo, a2 row g k-hi, a3 row g+8 k-hi
                const uint32_t s0 = w0, s1 = __umulhi(w0, 0x10000u), s2 = w1, s3 = __umulhi(w1, 0x10000u);
                const uint32_t q0 = x0, q1 = __umulhi(x0, 0x10000u), q2 = x1, q3 = __umulhi(x1, 0x10000u);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const uint32_t pa0 = prmt(L0[p].x, L0[p].y, s0), pa1 = prmt(L1[p].x, L1[p].y, s1);
                    const uint32_t pa2 = prmt(L0[p].x, L0[p].y, s2), pa3 = prmt(L1[p].x, L1[p].y, s3);
                    const uint32_t qa0 = prmt(L0[p].z, L0[p].w, q0), qa1 = prmt(L1[p].z, L1[p].w, q1);
                    const uint32_t qa2 = prmt(L0[p].z, L0[p].w, q2), qa3 = prmt(L1[p].z, L1[p].w, q3);
#pragma unroll
                    for (int nt = 0; nt < TC_NT; ++nt)
                        if (nt < ntc) mma_s8(acc[p][nt], pa0, pa1, pa2, pa3, b[nt].x, b[nt].y);
#pragma unroll
                    for (int nt = 0; nt < TC_NT; ++nt)
                        if (nt < ntc) mma_s8(acc[p][nt], qa0, qa1, qa2, qa3, b[nt].x, b[nt].y);
                }
            }
            __syncwarp();
            if (lane == 0 && c + TC_STAGES < n_chunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(c + TC_STAGES, stage, j0, ntc);
            }
        }
        // ---- epilogue: rows (g8, g8+8) x tokens (2 t4, 2 t4 + 1) per token tile
        const int i0 = rowtile * 16 + g8;
        if (GLU) {
            float *xb = xbuf + (warp >> 1) * 16 * (TC_NT * 8);
            if (mat == 1) {
#pragma unroll
                for (int nt = 0; nt < TC_NT; ++nt)
                    if (nt < ntc)
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int64_t tok = (j0 + nt) * 8 + 2 * t4 + (r & 1);
                            const float sc = (tok >= rb && tok < re) ? __ldg(scales + tok) : 0.0f;
                            const float v = (float)(combine_planes<P>(acc, nt, r) * (double)(r < 2 ? rs0 : rs1));
                            xb[(g8 + (r >> 1) * 8) * (TC_NT * 8) + nt * 8 + 2 * t4 + (r & 1)] = __fmul_rn(v, sc);
                        }
            }
            named_bar(1 + (warp >> 1), 64);
            if (mat == 0) {
#pragma unroll
                for (int nt = 0; nt < TC_NT; ++nt)
                    if (nt < ntc)
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const int64_t tok = (j0 + nt) * 8 + 2 * t4 + (r & 1);
                            if (tok < rb || tok >= re) continue;
                            const float sc = __ldg(scales + tok);
                            const float a = __fmul_rn(
                                (float)(combine_planes<P>(acc, nt, r) * (double)(r < 2 ? rs0 : rs1)), sc);
                            const float bv = xb[(g8 + (r >> 1) * 8) * (TC_NT * 8) + nt * 8 + 2 * t4 + (r & 1)];
                            out[tok * d_out + i0 + (r >> 1) * 8] = __fmul_rn(silu_f32(a), bv);
                        }
            }
            named_bar(1 + (warp >> 1), 64);
        } else {
#pragma unroll
            for (int nt = 0; nt < TC_NT; ++nt)
                if (nt < ntc)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const int64_t tok = (j0 + nt) * 8 + 2 * t4 + (r & 1);
                        if (tok < rb || tok >= re) continue;
                        const float v = (float)(combine_planes<P>(acc, nt, r) * (double)(r < 2 ? rs0 : rs1));
                        out[tok * d_out + i0 + (r >> 1) * 8] = __fmul_rn(v, __ldg(scales + tok));
                    }
        }
    }
}

// codes (rows, K) row-major -> mma B-fragment order [chunk128][tile8][sub][lane]
// (8 B each): lane (g, t) of token tile j holds row 8j+g, columns
// 128c+32sub+4t..+3 and +16.  A stage's ntc consecutive tiles are one
// contiguous bulk copy.  Rows >= n are zero.
__global__ void to_frag_kernel(const int8_t *__restrict__ src, int64_t n, int64_t K, int64_t tiles,
                               uint2 *__restrict__ dst) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t total = (K / 128) * tiles * 128;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int lane = (int)(x & 31), sub = (int)((x >> 5) & 3);
        const int64_t j = (x >> 7) % tiles, chunk = (x >> 7) / tiles;
        const int64_t kc = chunk * 4 + sub;
        const int64_t row = j * 8 + (lane >> 2);
        uint2 v = make_uint2(0u, 0u);
        if (row < n) {
            const int8_t *p = src + row * K + kc * 32 + (lane & 3) * 4;
            v.x = *reinterpret_cast<const uint32_t *>(p);
            v.y = *reinterpret_cast<const uint32_t *>(p + 16);
        }
        dst[x] = v;
    }
}

// ---------------------------------------------------------------------------
// One-time preparation.

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

// One thread per (row, group): digits of the 16 centroids, then the
// sign-garbage compensation of every (a, a + 8) pair, per plane.
__global__ void lut8_kernel(const float *__restrict__ cent, const float *__restrict__ rowscale, int64_t rows,
                            int64_t n_groups, int planes, int64_t mbound, int8_t *__restrict__ lut) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= rows * n_groups) return;
    const int64_t row = x / n_groups, grp = x - row * n_groups;
    const double s = (double)rowscale[row];
    int dig[3][16];
    for (int c = 0; c < 16; ++c) {
        long long m = llrint((double)cent[x * 16 + c] / s);
        m = m > mbound ? mbound : (m < -mbound ? -mbound : m);
        for (int p = 0; p < planes; ++p) {
            long long d = ((m + 128) % 255 + 255) % 255 - 128;  // digit in [-128, 126]
            dig[p][c] = (int)d;
            m = (m - d) / 255;
        }
    }
    const int64_t tile = row / 16, r16 = row % 16;
    int8_t *dst = lut + ((tile * n_groups + grp) * 16 + r16) * planes * 16;
    for (int p = 0; p < planes; ++p) {
        for (int a = 0; a < 8; ++a) {
            const int ta = dig[p][a], tb = dig[p][a + 8];
            // find (xa, xb) with xa == (ta + xb < 0) and xb == (tb + xa < 0)
            int la = ta, lb = tb;
            for (int combo = 0; combo < 4; ++combo) {
                const int xa = combo & 1, xb = combo >> 1;
                la = ta + xb;
                lb = tb + xa;
                if ((la < 0) == (xa == 1) && (lb < 0) == (xb == 1)) break;
            }
            dst[p * 16 + a] = (int8_t)la;
            dst[p * 16 + a + 8] = (int8_t)lb;
        }
    }
}

// Unsigned variant for the tcgen05 kernel: m = rint(c / rowscale) in
// [-(2^(7P-1)-1), 2^(7P-1)-1] is stored biased, u = m + 2^(7P-1), as P base-128
// digits in [0, 127].  Every table byte then has its sign bit clear, so the
// sign-replicated half of each PRMT pair is exactly zero and the two halves
// merge with one OR; the bias returns in the epilogue as 2^(7P-1) * sum_j q_j.
__global__ void lut7_kernel(const float *__restrict__ cent, const float *__restrict__ rowscale, int64_t rows,
                            int64_t n_groups, int planes, int8_t *__restrict__ lut) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (x >= rows * n_groups) return;
    const int64_t row = x / n_groups, grp = x - row * n_groups;
    const double s = (double)rowscale[row];
    const long long bias = 1LL << (7 * planes - 1), mb = bias - 1;
    const int64_t tile = row / 16, r16 = row % 16;
    int8_t *dst = lut + ((tile * n_groups + grp) * 16 + r16) * planes * 16;
    for (int c = 0; c < 16; ++c) {
        long long m = llrint((double)cent[x * 16 + c] / s);
        m = m > mb ? mb : (m < -mb ? -mb : m);
        const long long u = m + bias;
        for (int p = 0; p < planes; ++p) dst[p * 16 + c] = (int8_t)((u >> (7 * p)) & 127);
    }
}

// ids (rows, d_in/2) -> [tile][chunk][h][lane][16 B]: lane (g, t), sub-chunk
// s = 2h + {0,1}: w0 = sel(g, 32s+4t) | sel(g+8, 32s+4t) << 16,
//                 w1 = sel(g, 32s+16+4t) | sel(g+8, 32s+16+4t) << 16,
// sel(r, k) = the 16-bit little-endian word at packed byte k/2 of row r.
__global__ void ids_frag_kernel(const uint8_t *__restrict__ ids, int64_t rows, int64_t d_in,
                                uint8_t *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t n_chunks = d_in / TC_CHUNK, row_bytes = d_in / 2;
    const int64_t total = (rows / 16) * n_chunks * 64;  // (h, lane) pairs
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int lane = (int)(x & 31), h = (int)((x >> 5) & 1);
        const int64_t chunk = (x >> 6) % n_chunks, tile = (x >> 6) / n_chunks;
        const int g = lane >> 2, t = lane & 3;
        const uint8_t *r0 = ids + (tile * 16 + g) * row_bytes, *r1 = ids + (tile * 16 + g + 8) * row_bytes;
        uint32_t w[4];
        for (int j = 0; j < 2; ++j) {
            const int64_t k_lo = chunk * TC_CHUNK + 32 * (2 * h + j) + 4 * t, k_hi = k_lo + 16;
            const uint32_t a = *reinterpret_cast<const uint16_t *>(r0 + k_lo / 2);
            const uint32_t b = *reinterpret_cast<const uint16_t *>(r1 + k_lo / 2);
            const uint32_t c = *reinterpret_cast<const uint16_t *>(r0 + k_hi / 2);
            const uint32_t d = *reinterpret_cast<const uint16_t *>(r1 + k_hi / 2);
            w[2 * j] = a | (b << 16);
            w[2 * j + 1] = c | (d << 16);
        }
        reinterpret_cast<uint4 *>(out)[x] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---------------------------------------------------------------------------
// host side

bool tc_path_ok(int64_t d_in, int64_t d_out, int64_t g) {
    return d_in % TC_CHUNK == 0 && g % TC_CHUNK == 0 && d_out % 16 == 0 && d_in <= (1 << 20);
}

template <int P, bool GLU>
size_t tc_smem() {
    return (size_t)TC_WARPS * TC_STAGES * TcStage<P>::BYTES + TC_WARPS * TC_STAGES * 8 +
           (GLU ? (TC_WARPS / 2) * 16 * TC_NT * 8 * sizeof(float) : 0);
}

template <int P, bool GLU>
cq_status launch_tc(const uint2 *frag, int64_t n_tiles, const float *scales, const int32_t *offsets, int64_t n_seg, int64_t seg_first,
                    const cq_expert_site *a, const cq_expert_site *b, int64_t d_in, int64_t d_out, float *out,
                    cudaStream_t st) {
    static bool attr = false;
    const size_t smem = tc_smem<P, GLU>();
    if (!attr) {
        cudaFuncSetAttribute(lut_tc_kernel<P, GLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int tiles_per_cta = GLU ? TC_WARPS / 2 : TC_WARPS;
    dim3 grid((unsigned)ceil_div(d_out / 16, tiles_per_cta), (unsigned)n_seg);
    lut_tc_kernel<P, GLU><<<grid, TC_WARPS * 32, smem, st>>>(
        frag, n_tiles, scales, offsets, seg_first, a->tc_ids, a->tc_lut, a->tc_rowscale, b ? b->tc_ids : nullptr,
        b ? b->tc_lut : nullptr, b ? b->tc_rowscale : nullptr, (int)d_in, (int)d_out, (int)a->group_size, out);
    return check_launch("lut_tc");
}

cq_status to_frag(const int8_t *codes, int64_t n, int64_t K, uint2 *frag, cudaStream_t st) {
    const int64_t tiles = ceil_div(n, 8);
    const int64_t total = tiles * (K / 128) * 128;
    if (total == 0) return CQ_OK;
    to_frag_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16), 256, 0, st>>>(codes, n, K, tiles,
                                                                                              frag);
    return check_launch("to_frag");
}

// Grouped launch over segments; `rows` = rows of the (row-major) codes buffer.
// The caller provides the fragment buffer (ceil(rows/8)*8 x d_in).
cq_status lut_tc_grouped_frag(const int8_t *codes, uint2 *frag, const float *scales, const int32_t *offsets,
                              int64_t n_seg, int64_t seg_first, int64_t rows, const cq_expert_site *a,
                              const cq_expert_site *b, int64_t d_in, int64_t d_out, float *out, cudaStream_t st) {
    if (rows == 0 || n_seg == 0) return CQ_OK;
    if (!tc_path_ok(d_in, d_out, a->group_size) || a->tc_lut == nullptr || (b && b->tc_lut == nullptr)) {
        set_error("tensor-core path: site not prepared or shape outside envelope");
        return CQ_ERR_UNSUPPORTED;
    }
    if (b && b->tc_planes != a->tc_planes) {
        set_error("tensor-core path: gate and up must have the same digit planes");
        return CQ_ERR_CONFIG;
    }
    CQ_TRY(to_frag(codes, rows, d_in, frag, st));
    const int64_t nt = ceil_div(rows, 8);
    const bool glu = b != nullptr;
    if (a->tc_planes == 3)
        return glu ? launch_tc<3, true>(frag, nt, scales, offsets, n_seg, seg_first, a, b, d_in, d_out, out, st)
                   : launch_tc<3, false>(frag, nt, scales, offsets, n_seg, seg_first, a, b, d_in, d_out, out, st);
    if (a->tc_planes == 2)
        return glu ? launch_tc<2, true>(frag, nt, scales, offsets, n_seg, seg_first, a, b, d_in, d_out, out, st)
                   : launch_tc<2, false>(frag, nt, scales, offsets, n_seg, seg_first, a, b, d_in, d_out, out, st);
    set_error("tensor-core path: planes must be 2 or 3");
    return CQ_ERR_CONFIG;
}

cq_status umma_prepare(const uint8_t *, const int8_t *, int64_t, int64_t, int64_t, int64_t, uint8_t *, int8_t *,
                       cudaStream_t);
cq_status lut_umma_grouped(const int8_t *, int8_t *, const float *, const int32_t *, int64_t, int64_t, int64_t,
                           const cq_expert_site *, float *, const cq_expert_site *, float *, int64_t, int64_t,
                           cudaStream_t, const UmmaIn &in = UmmaIn{});
bool umma_ok(int64_t d_in, int64_t d_out, int64_t g);
int64_t umma_b_bytes(int64_t rows, int64_t d_in);

cq_status lut8_prepare(const uint8_t *ids, const float *cent, int64_t rows, int64_t d_in, int64_t g, int64_t planes,
                       int64_t layout, uint8_t *tc_ids, int8_t *tc_lut, float *rowscale, cudaStream_t st) {
    if (planes != 2 && planes != 3) {
        set_error("lut8_prepare: planes must be 2 or 3");
        return CQ_ERR_CONFIG;
    }
    if (layout < CQ_TC_MMA16 || layout > CQ_TC_UMMA128U8) {
        set_error("lut8_prepare: unknown layout");
        return CQ_ERR_CONFIG;
    }
    if (rows % (layout == CQ_TC_MMA16 ? 16 : 128) || !tc_path_ok(d_in, 16, g)) {
        set_error("lut8_prepare: needs rows % 16 (mma16) / % 128 (umma128) == 0, d_in % 128 == 0, g % 128 == 0");
        return CQ_ERR_UNSUPPORTED;
    }
    if (rows == 0) return CQ_OK;
    const int64_t n_groups = d_in / g;
    const bool um = umma_merged(layout);  // unsigned base-128 digits (lut7_kernel)
    const int64_t mb = um ? (1LL << (7 * planes - 1)) - 1 : (planes == 3 ? TC_M3 : TC_M2);
    rowscale_kernel<<<(unsigned)ceil_div(rows, 8), 256, 0, st>>>(cent, rows, n_groups * 16,
                                                                 (double)mb, rowscale);
    CQ_TRY(check_launch("rowscale"));
    int8_t *lut16 = tc_lut;
    const bool relayout = layout == CQ_TC_UMMA128 || umma_merged(layout);
    if (relayout) {
        if (cudaMallocAsync(&lut16, rows * n_groups * planes * 16, st) != cudaSuccess) {
            set_error("lut8_prepare: scratch alloc failed");
            return CQ_ERR_CUDA;
        }
    }
    if (um) {
        lut7_kernel<<<(unsigned)ceil_div(rows * n_groups, 128), 128, 0, st>>>(cent, rowscale, rows, n_groups,
                                                                            (int)planes, lut16);
    } else {
        lut8_kernel<<<(unsigned)ceil_div(rows * n_groups, 128), 128, 0, st>>>(cent, rowscale, rows, n_groups,
                                                                            (int)planes, mb, lut16);
    }
    CQ_TRY(check_launch("lut8"));
    if (relayout) {
        cq_status rc = umma_prepare(ids, lut16, rows, d_in, g, planes, tc_ids, tc_lut, st);
        cudaFreeAsync(lut16, st);
        return rc;
    }
    const int64_t total = (rows / 16) * (d_in / TC_CHUNK) * 64;
    ids_frag_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 32), 256, 0, st>>>(ids, rows, d_in,
                                                                                                tc_ids);
    return check_launch("ids_frag");
}

}  // namespace cq

using namespace cq;

extern "C" cq_status cq_lut8_prepare(const uint8_t *ids, const float *centroids, int64_t rows, int64_t d_in,
                                     int64_t g, int64_t planes, int64_t layout, uint8_t *tc_ids, int8_t *tc_lut,
                                     float *tc_rowscale, void *stream) {
    return lut8_prepare(ids, centroids, rows, d_in, g, planes, layout, tc_ids, tc_lut, tc_rowscale,
                        as_stream(stream));
}

__global__ void tc_single_segment_kernel(int32_t *off, int64_t n) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    off[0] = 0;
    off[1] = (int32_t)n;
}

extern "C" cq_status cq_lut_gemm_tc(const int8_t *codes, const float *scales, const uint8_t *tc_ids,
                                    const int8_t *tc_lut, const float *tc_rowscale, int64_t planes, int64_t layout,
                                    int64_t n, int64_t d_in, int64_t d_out, int64_t g, float *out, void *stream) {
    if (n < 0 || g < 1 || d_in % g) {
        set_error("group size does not divide the input dimension");
        return CQ_ERR_SHAPE;
    }
    if (n == 0 || d_out == 0) return CQ_OK;
    cudaStream_t st = as_stream(stream);
    cq_expert_site site{};
    site.group_size = g;
    site.tc_ids = tc_ids;
    site.tc_lut = tc_lut;
    site.tc_rowscale = tc_rowscale;
    site.tc_planes = planes;
    site.tc_layout = layout;
    void *scratch = nullptr;
    const bool um = layout == CQ_TC_UMMA128 || umma_merged(layout);
    const int64_t frag_bytes = um ? umma_b_bytes(n, d_in) : ceil_div(n, 8) * 8 * d_in;
    if (cudaMallocAsync(&scratch, frag_bytes + 256, st) != cudaSuccess) {
        set_error("lut_gemm_tc: scratch alloc failed");
        return CQ_ERR_CUDA;
    }
    int32_t *off = reinterpret_cast<int32_t *>(reinterpret_cast<char *>(scratch) + frag_bytes);
    tc_single_segment_kernel<<<1, 1, 0, st>>>(off, n);
    cq_status rc = check_launch("single_segment");
    if (rc == CQ_OK && um)
        rc = lut_umma_grouped(codes, reinterpret_cast<int8_t *>(scratch), scales, off, 1, 0, n, &site, out, nullptr,
                              nullptr, d_in, d_out, st);
    else if (rc == CQ_OK)
        rc = lut_tc_grouped_frag(codes, reinterpret_cast<uint2 *>(scratch), scales, off, 1, 0, n, &site, nullptr, d_in,
                                 d_out, out, st);
    cudaFreeAsync(scratch, st);
    return rc;
}
