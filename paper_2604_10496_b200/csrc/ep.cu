// Expert parallelism, device side: the bookkeeping around
// the two exchanges of an EP MoE step, on the GPU, so a step needs at most one
// host read (the counts, in compact sizing) and in fixed sizing none at all
// (one CUDA graph holds the whole step).
//
// Rows.  A rank sends each peer rows of cq_ep_row_bytes(d, kr) bytes:
//   [codes][f32 scale][i32 m][(i32 e_j, f32 w_j) x kr][pad to 16 B]
// The codes are the token's A4 values in [-8, 7] — exact: quantization is per
// token and happens before routing (model.py:379) — as packed nibbles (d/2
// bytes, low nibble first, the reference's int4 format) when d % 32 == 0,
// else one byte each.  m routes of the token go to local experts e_0 < e_1 <
// ... of the receiving rank with receiver-side weights w_j.
//   * dedup (kr = min(top_k, experts per rank)): ONE row per (token, peer),
//     carrying all the token's routes to that peer and their route weights.
//     The receiver returns the per-row partial sum ((0 + w_0 f_0) + w_1 f_1)
//     ... (experts ascending) as one fp32 row; the source adds the partials
//     of its peers in ascending rank order.  Bytes per (token, peer): one code
//     row out, one fp32 row back, however many of the token's experts the peer
//     holds.  Differs from the single-GPU sum only by the association of the
//     fp32 adds across ranks (bitwise equal at world 1, and for every token
//     whose experts all live on one rank).
//   * exact (kr = 1): one row per route with w = 1; the receiver returns
//     f = 1 * f (exact) and the source applies the route weights in ascending
//     expert order — bitwise equal to the single-GPU layer for any world size.
//
// Sizing.  capacity > 0: every rank sends every peer exactly `capacity` rows
// (fixed slots; equal-split all_to_alls, no host read); empty rows carry m = 0
// and e = -1.  capacity == 0 (compact): rows to peer g are packed after the
// rows to peers < g; the per-peer row and route counts go first (one small
// all_to_all + one host read) and size exact all_to_all-v splits.
//
//   cq_ep_dispatch  routes -> send rows, per-peer counts, and per token the
//                   list of returned rows to add (src_slot / src_w).
//   cq_ep_group     received rows -> codes/scales grouped by local expert
//                   (stable in (row, j) order), offsets, route_pos.
//   cq_ep_partial   grouped expert outputs -> one returned fp32 row per
//                   received row.
//   cq_ep_combine   returned rows -> moe_sum (+ shared-expert outputs).
#include "common.cuh"

namespace cq {

constexpr int EP_THREADS = 1024;
constexpr int EP_MAX_BUCKETS = 256;
constexpr int EP_MAX_K = 16;

__host__ __device__ inline bool ep_packed(int64_t d) { return d % 32 == 0; }
__host__ __device__ inline int64_t ep_code_bytes(int64_t d) { return ep_packed(d) ? d / 2 : d; }
__host__ __device__ inline int64_t ep_header_bytes(int64_t kr) { return (8 + 8 * kr + 15) / 16 * 16; }
__host__ __device__ inline int64_t ep_row_bytes(int64_t d, int64_t kr) { return ep_code_bytes(d) + ep_header_bytes(kr); }

// Item i's bucket: p[(i / inner) * stride + (i % inner) * inner_stride]; negative = none.
struct KeySrc {
    const int32_t *p;
    int64_t stride;       // int32 words between rows
    int32_t inner;        // items per row
    int32_t inner_stride; // int32 words between items of a row
};

__device__ __forceinline__ int key_of(const KeySrc &k, int64_t i) {
    const int64_t r = i / k.inner;
    const int64_t j = i - r * k.inner;
    return k.p[r * k.stride + j * k.inner_stride];
}

// Stable bucket ranks in one block: rank[i] = #{j < i : bucket(j) == bucket(i)},
// counts[b * counts_stride], optional exclusive offsets[0..nb].  Warps match
// equal buckets (__match_any_sync); a per-(warp, bucket) table in shared memory
// carries the prefix across warps and chunks.
__global__ void __launch_bounds__(EP_THREADS) bucket_rank_kernel(KeySrc ks, int64_t n, int nb, int32_t *rank,
                                                                 int32_t *counts, int64_t counts_stride,
                                                                 int32_t *offsets) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    extern __shared__ int32_t sm[];
    int32_t *carry = sm;        // [nb]
    int32_t *wtab = sm + nb;    // [32][nb]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int b = tid; b < nb; b += EP_THREADS) carry[b] = 0;
    for (int64_t base = 0; base < n; base += EP_THREADS) {
        for (int x = tid; x < 32 * nb; x += EP_THREADS) wtab[x] = 0;
        __syncthreads();
        const int64_t i = base + tid;
        const int key = i < n ? key_of(ks, i) : -1;
        const unsigned m = __match_any_sync(0xffffffffu, key);
        const int lr = __popc(m & ((1u << lane) - 1u));
        if (key >= 0 && lr == 0) wtab[warp * nb + key] = __popc(m);
        __syncthreads();
        for (int b = tid; b < nb; b += EP_THREADS) {
            int acc = carry[b];
            for (int w = 0; w < 32; ++w) {
                const int t = wtab[w * nb + b];
                wtab[w * nb + b] = acc;
                acc += t;
            }
            carry[b] = acc;
        }
        __syncthreads();
        if (key >= 0) rank[i] = wtab[warp * nb + key] + lr;
        __syncthreads();
    }
    for (int b = tid; b < nb; b += EP_THREADS) counts[b * counts_stride] = carry[b];
    if (offsets != nullptr && tid == 0) {
        int acc = 0;
        for (int b = 0; b < nb; ++b) {
            offsets[b] = acc;
            acc += carry[b];
        }
        offsets[nb] = acc;
    }
}

cq_status bucket_rank(const KeySrc &ks, int64_t n, int nb, int32_t *rank, int32_t *counts, int64_t counts_stride,
                      int32_t *offsets, cudaStream_t st) {
    const size_t smem = (size_t)33 * nb * sizeof(int32_t);
    launch_pdl(bucket_rank_kernel, 1, EP_THREADS, smem, st, ks, n, nb, rank, counts, counts_stride, offsets);
    return check_launch("ep_bucket_rank");
}

// A token's routes in ascending expert order (its top-k ids are distinct).
__device__ __forceinline__ int sorted_routes(const int32_t *__restrict__ selected, const float *__restrict__ weights,
                                             int64_t t, int k, int32_t *e, float *w) {
    for (int s = 0; s < k; ++s) {
        e[s] = selected[t * k + s];
        w[s] = weights[t * k + s];
    }
    for (int a = 1; a < k; ++a)
        for (int b = a; b > 0 && e[b - 1] > e[b]; --b) {
            const int32_t te = e[b]; e[b] = e[b - 1]; e[b - 1] = te;
            const float tw = w[b]; w[b] = w[b - 1]; w[b - 1] = tw;
        }
    return k;
}

// One thread per token: the token's rows in ascending peer (dedup) or expert
// (exact) order -> rowkey[t*k + i] = peer (or -1 past the last row) and the
// source-side weight of returned row i (1 in dedup: the receiver weighs).
__global__ void ep_plan_kernel(const int32_t *__restrict__ selected, const float *__restrict__ weights, int64_t n,
                               int k, int per, int world, int dedup, int32_t *__restrict__ rowkey,
                               float *__restrict__ src_w, int32_t *__restrict__ src_slot, int32_t *counts,
                               int64_t counts_stride) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    if (blockIdx.x == 0)
        for (int g = threadIdx.x; g < world; g += blockDim.x) counts[g * counts_stride + 1] = 0;  // route counts
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        int32_t e[EP_MAX_K];
        float w[EP_MAX_K];
        sorted_routes(selected, weights, t, k, e, w);
        int rows = 0;
        for (int s = 0; s < k; ++s) {
            const int g = e[s] / per;
            if (dedup && s > 0 && g == e[s - 1] / per) continue;
            rowkey[t * k + rows] = g;
            src_w[t * k + rows] = dedup ? 1.0f : w[s];
            ++rows;
        }
        for (int i = rows; i < k; ++i) {
            rowkey[t * k + i] = -1;
            src_w[t * k + i] = 0.0f;
            src_slot[t * k + i] = -1;
        }
    }
}

// 8 int8 codes (two words) -> 8 nibbles, low first
__device__ __forceinline__ uint32_t nib_pack8(uint32_t a, uint32_t b) {
    uint32_t x = a & 0x0F0F0F0Fu, y = b & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    y = (y | (y >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    y = (y | (y >> 8)) & 0x0000FFFFu;
    return x | (y << 16);
}
// 4 nibbles (low 16 bits) -> 4 sign-extended int8 codes
__device__ __forceinline__ uint32_t nib_unpack4(uint32_t h) {
    uint32_t y = h & 0xFFFFu;
    y = (y | (y << 8)) & 0x00FF00FFu;
    y = (y | (y << 4)) & 0x0F0F0F0Fu;
    return __vsub4(y ^ 0x08080808u, 0x08080808u);  // per byte: (n ^ 8) - 8, no borrow across bytes
}

// Send rows.  Item (t, i) with rowkey >= 0 goes to slot base[peer] + rank; the
// thread of its last 16-byte piece writes the header, src_slot and the route
// count.  Fixed sizing also blanks the unused slots' headers.
__global__ void ep_pack_kernel(const int8_t *__restrict__ codes, const float *__restrict__ scales,
                               const int32_t *__restrict__ selected, const float *__restrict__ weights, int64_t n,
                               int k, int64_t d, int per, int kr, int dedup, int world,
                               const int32_t *__restrict__ rowkey, const int32_t *__restrict__ rank, int32_t *counts,
                               int64_t counts_stride, int64_t cap, uint8_t *__restrict__ send,
                               int32_t *__restrict__ src_slot) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int64_t base[EP_MAX_BUCKETS];
    if (threadIdx.x == 0) {
        int64_t acc = 0;
        for (int g = 0; g < world; ++g) {
            base[g] = cap > 0 ? (int64_t)g * cap : acc;
            acc += counts[g * counts_stride];
        }
    }
    __syncthreads();
    const int64_t cb = ep_code_bytes(d), cp = cb / 16, rb = cb + ep_header_bytes(kr);
    const int64_t pieces = cp + 1, total = n * k * pieces;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += stride) {
        const int64_t item = x / pieces, pc = x - item * pieces;
        const int g = rowkey[item];
        if (g < 0) continue;
        const int64_t t = item / k;
        const int64_t slot = base[g] + rank[item];
        uint8_t *row = send + slot * rb;
        if (pc < cp) {
            uint4 *out = reinterpret_cast<uint4 *>(row) + pc;
            if (ep_packed(d)) {  // 32 codes -> 16 bytes
                const uint4 *src = reinterpret_cast<const uint4 *>(codes + t * d) + 2 * pc;
                const uint4 u = src[0], v = src[1];
                *out = make_uint4(nib_pack8(u.x, u.y), nib_pack8(u.z, u.w), nib_pack8(v.x, v.y), nib_pack8(v.z, v.w));
            } else {
                *out = reinterpret_cast<const uint4 *>(codes + t * d)[pc];
            }
            continue;
        }
        int32_t e[EP_MAX_K];
        float w[EP_MAX_K];
        sorted_routes(selected, weights, t, k, e, w);
        int32_t *h = reinterpret_cast<int32_t *>(row + cb);
        int m = 0;
        if (dedup) {
            for (int s = 0; s < k; ++s)
                if (e[s] / per == g) {
                    h[2 + 2 * m] = e[s] - g * per;
                    h[3 + 2 * m] = __float_as_int(w[s]);
                    ++m;
                }
        } else {  // the i-th route in ascending expert order
            const int s = (int)(item - t * k);
            h[2] = e[s] - g * per;
            h[3] = __float_as_int(1.0f);
            m = 1;
        }
        for (int j = m; j < kr; ++j) {
            h[2 + 2 * j] = -1;
            h[3 + 2 * j] = 0;
        }
        for (int64_t z = 8 + 8 * (int64_t)kr; z < ep_header_bytes(kr); z += 4) h[z / 4] = 0;
        h[0] = __float_as_int(scales[t]);
        h[1] = m;
        src_slot[item] = (int32_t)slot;
        atomicAdd(counts + g * counts_stride + 1, m);
    }
    if (cap > 0) {  // fixed sizing: empty slots carry m = 0, e = -1
        const int64_t hw = ep_header_bytes(kr) / 4;
        for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < world * cap * hw; x += stride) {
            const int64_t s = x / hw, z = x - s * hw;
            const int64_t g = s / cap, p = s - g * cap;
            if (p < counts[g * counts_stride]) continue;
            int32_t *h = reinterpret_cast<int32_t *>(send + s * rb + cb);
            h[z] = (z >= 2 && z < 2 + 2 * kr && (z & 1) == 0) ? -1 : 0;
        }
    }
}

// Received routes -> grouped rows: pos = offsets[e] + rank[item]; route_pos[item] = pos (or -1).
__global__ void ep_group_kernel(const uint8_t *__restrict__ recv, int64_t rows, int64_t d, int kr,
                                const int32_t *__restrict__ rank, const int32_t *__restrict__ offsets,
                                int8_t *__restrict__ codes_perm, float *__restrict__ scales_perm,
                                int32_t *__restrict__ route_pos) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t cb = ep_code_bytes(d), cp = cb / 16, rb = cb + ep_header_bytes(kr);
    const int64_t pieces = cp + 1, total = rows * kr * pieces;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t item = x / pieces, pc = x - item * pieces;
        const int64_t r = item / kr, j = item - r * kr;
        const uint8_t *row = recv + r * rb;
        const int32_t *h = reinterpret_cast<const int32_t *>(row + cb);
        const int32_t e = h[2 + 2 * j];
        if (pc == cp) {
            const int64_t pos = e < 0 ? -1 : offsets[e] + rank[item];
            route_pos[item] = (int32_t)pos;
            if (e >= 0) scales_perm[pos] = __int_as_float(h[0]);
            continue;
        }
        if (e < 0) continue;
        const int64_t pos = offsets[e] + rank[item];
        const uint4 w = reinterpret_cast<const uint4 *>(row)[pc];
        if (ep_packed(d)) {  // 16 bytes -> 32 codes
            uint4 *dst = reinterpret_cast<uint4 *>(codes_perm + pos * d) + 2 * pc;
            dst[0] = make_uint4(nib_unpack4(w.x), nib_unpack4(w.x >> 16), nib_unpack4(w.y), nib_unpack4(w.y >> 16));
            dst[1] = make_uint4(nib_unpack4(w.z), nib_unpack4(w.z >> 16), nib_unpack4(w.w), nib_unpack4(w.w >> 16));
        } else {
            reinterpret_cast<uint4 *>(codes_perm + pos * d)[pc] = w;
        }
    }
}

// One returned row per received row: raw (exact sizing, m = 1, w = 1): f as is;
// else ((0 + w_0 f_0) + w_1 f_1) ... in j (= ascending expert) order.
__global__ void __launch_bounds__(256) ep_partial_kernel(const float4 *__restrict__ fout,
                                                         const int32_t *__restrict__ route_pos,
                                                         const uint8_t *__restrict__ recv, int64_t rows, int64_t d4,
                                                         int kr, int raw, float4 *__restrict__ back) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int32_t pos_sh[EP_MAX_K];
    __shared__ float w_sh[EP_MAX_K];
    __shared__ int m_sh;
    const int64_t cb = ep_code_bytes(d4 * 4), rb = cb + ep_header_bytes(kr);
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int32_t *h = reinterpret_cast<const int32_t *>(recv + r * rb + cb);
        if (threadIdx.x == 0) m_sh = h[1];
        if (threadIdx.x < kr) {
            pos_sh[threadIdx.x] = route_pos[r * kr + threadIdx.x];
            w_sh[threadIdx.x] = __int_as_float(h[3 + 2 * threadIdx.x]);
        }
        __syncthreads();
        const int m = m_sh;
        if (m > 0) {
            for (int64_t c = threadIdx.x; c < d4; c += blockDim.x) {
                float4 acc;
                if (raw) {
                    acc = fout[(int64_t)pos_sh[0] * d4 + c];
                } else {
                    acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int j = 0; j < m; ++j) {
                        const float ws = w_sh[j];
                        const float4 f = fout[(int64_t)pos_sh[j] * d4 + c];
                        acc.x = __fadd_rn(acc.x, __fmul_rn(ws, f.x));
                        acc.y = __fadd_rn(acc.y, __fmul_rn(ws, f.y));
                        acc.z = __fadd_rn(acc.z, __fmul_rn(ws, f.z));
                        acc.w = __fadd_rn(acc.w, __fmul_rn(ws, f.w));
                    }
                }
                back[r * d4 + c] = acc;
            }
        }
        __syncthreads();
    }
}

// out[t] = ((0 + c_0 ret[slot_0]) + c_1 ret[slot_1]) ... over the token's
// returned rows (slot -1 ends the list), then + add_0 + add_1 ... (shared experts).
__global__ void __launch_bounds__(256) ep_combine_kernel(const float4 *__restrict__ ret,
                                                         const int32_t *__restrict__ src_slot,
                                                         const float *__restrict__ src_w, int64_t n, int k,
                                                         int64_t d4, const float4 *__restrict__ add, int n_add,
                                                         int64_t add_stride4, float4 *__restrict__ out) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    __shared__ int32_t slot_sh[EP_MAX_K];
    __shared__ float w_sh[EP_MAX_K];
    for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
        if (threadIdx.x < k) {
            slot_sh[threadIdx.x] = src_slot[t * k + threadIdx.x];
            w_sh[threadIdx.x] = src_w[t * k + threadIdx.x];
        }
        __syncthreads();
        for (int64_t c = threadIdx.x; c < d4; c += blockDim.x) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int i = 0; i < k && slot_sh[i] >= 0; ++i) {
                const float ws = w_sh[i];
                const float4 f = ret[(int64_t)slot_sh[i] * d4 + c];
                acc.x = __fadd_rn(acc.x, __fmul_rn(ws, f.x));
                acc.y = __fadd_rn(acc.y, __fmul_rn(ws, f.y));
                acc.z = __fadd_rn(acc.z, __fmul_rn(ws, f.z));
                acc.w = __fadd_rn(acc.w, __fmul_rn(ws, f.w));
            }
            for (int u = 0; u < n_add; ++u) {
                const float4 a = add[u * add_stride4 + t * d4 + c];
                acc.x = __fadd_rn(acc.x, a.x);
                acc.y = __fadd_rn(acc.y, a.y);
                acc.z = __fadd_rn(acc.z, a.z);
                acc.w = __fadd_rn(acc.w, a.w);
            }
            out[t * d4 + c] = acc;
        }
        __syncthreads();
    }
}

struct EpDispatchScratch {
    int32_t *rowkey, *rank;
};
struct EpGroupScratch {
    int32_t *rank, *counts;
};

inline int64_t al64(int64_t x) { return ceil_div(std::max<int64_t>(x, 1), 64) * 64; }

}  // namespace cq

using namespace cq;

extern "C" int64_t cq_ep_row_bytes(int64_t d_model, int64_t routes_per_row) {
    return ep_row_bytes(d_model, routes_per_row);
}

extern "C" int64_t cq_ep_scratch_bytes(int64_t n_tokens, int64_t top_k, int64_t recv_rows, int64_t routes_per_row,
                                       int64_t n_local) {
    const int64_t disp = 2 * al64(n_tokens * top_k);
    const int64_t grp = al64(recv_rows * routes_per_row) + al64(n_local);
    return 4 * (std::max(disp, grp) + 64);
}

extern "C" cq_status cq_ep_dispatch(const int8_t *codes, const float *scales, const int32_t *selected,
                                    const float *weights, int64_t n_tokens, int64_t top_k, int64_t d_model,
                                    int64_t experts_per_rank, int32_t world, int32_t dedup, int64_t capacity,
                                    uint8_t *send, int32_t *counts, int64_t counts_stride, int32_t *src_slot,
                                    float *src_w, void *scratch, void *stream) {
    if (d_model <= 0 || d_model % 16 || top_k < 1 || top_k > EP_MAX_K || experts_per_rank < 1 || world < 1 ||
        world > EP_MAX_BUCKETS || counts_stride < 2 || n_tokens < 0) {
        set_error("ep_dispatch: need d_model % 16 == 0, 1 <= top_k <= 16, experts_per_rank >= 1, "
                  "1 <= world <= 256, counts_stride >= 2");
        return CQ_ERR_CONFIG;
    }
    const int64_t per_row = dedup ? 1 : std::min(top_k, experts_per_rank);  // rows per (token, peer)
    if (capacity < 0 || (capacity > 0 && capacity < n_tokens * per_row)) {
        set_error("ep_dispatch: capacity must be 0 (compact) or >= n_tokens (dedup) / "
                  "n_tokens * min(top_k, experts_per_rank) (exact)");
        return CQ_ERR_CONFIG;
    }
    cudaStream_t st = as_stream(stream);
    const int kr = dedup ? (int)std::min(top_k, experts_per_rank) : 1;
    int32_t *p = reinterpret_cast<int32_t *>(scratch);
    const int64_t items = n_tokens * top_k;
    EpDispatchScratch s{p, p + al64(items)};
    launch_pdl(ep_plan_kernel, (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_tokens, 256), 148 * 4)),
               256, 0, st, selected, weights, n_tokens, (int)top_k, (int)experts_per_rank, (int)world, (int)dedup,
               s.rowkey, src_w, src_slot, counts, counts_stride);
    CQ_TRY(check_launch("ep_plan"));
    CQ_TRY(bucket_rank({s.rowkey, 1, 1, 0}, items, world, s.rank, counts, counts_stride, nullptr, st));
    const int64_t pieces = ep_code_bytes(d_model) / 16 + 1;
    const int64_t work = std::max(items * pieces, capacity * world * (ep_header_bytes(kr) / 4));
    launch_pdl(ep_pack_kernel, (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, 256), 148 * 8)), 256,
               0, st, codes, scales, selected, weights, n_tokens, (int)top_k, d_model, (int)experts_per_rank, kr,
               (int)dedup, (int)world, (const int32_t *)s.rowkey, (const int32_t *)s.rank, counts, counts_stride,
               capacity, send, src_slot);
    return check_launch("ep_pack");
}

extern "C" cq_status cq_ep_group(const uint8_t *recv, int64_t rows, int64_t d_model, int64_t routes_per_row,
                                 int64_t n_local, int8_t *codes_perm, float *scales_perm, int32_t *offsets,
                                 int32_t *route_pos, void *scratch, void *stream) {
    if (d_model <= 0 || d_model % 16 || n_local < 1 || n_local > EP_MAX_BUCKETS || routes_per_row < 1 ||
        routes_per_row > EP_MAX_K || rows < 0) {
        set_error("ep_group: need d_model % 16 == 0, 1 <= n_local <= 256, 1 <= routes_per_row <= 16");
        return CQ_ERR_CONFIG;
    }
    cudaStream_t st = as_stream(stream);
    int32_t *p = reinterpret_cast<int32_t *>(scratch);
    const int64_t items = rows * routes_per_row;
    EpGroupScratch s{p, p + al64(items)};
    const int64_t cb = ep_code_bytes(d_model);  // header words after the codes: e_j at 2 + 2j
    const KeySrc ks{reinterpret_cast<const int32_t *>(recv + cb) + 2, ep_row_bytes(d_model, routes_per_row) / 4,
                    (int32_t)routes_per_row, 2};
    CQ_TRY(bucket_rank(ks, items, (int)n_local, s.rank, s.counts, 1, offsets, st));
    const int64_t total = items * (cb / 16 + 1);
    if (total == 0) return CQ_OK;
    launch_pdl(ep_group_kernel, (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 8), 256, 0, st, recv, rows,
               d_model, (int)routes_per_row, (const int32_t *)s.rank, (const int32_t *)offsets, codes_perm,
               scales_perm, route_pos);
    return check_launch("ep_group");
}

extern "C" cq_status cq_ep_partial(const float *fout, const int32_t *route_pos, const uint8_t *recv, int64_t rows,
                                   int64_t d_model, int64_t routes_per_row, int32_t raw, float *back, void *stream) {
    if (d_model <= 0 || d_model % 16 || routes_per_row < 1 || routes_per_row > EP_MAX_K || (raw && routes_per_row != 1)) {
        set_error("ep_partial: need d_model % 16 == 0, 1 <= routes_per_row <= 16 (1 when raw)");
        return CQ_ERR_CONFIG;
    }
    if (rows <= 0) return CQ_OK;
    launch_pdl(ep_partial_kernel, (unsigned)std::min<int64_t>(rows, 148 * 8), 128, 0, as_stream(stream),
               reinterpret_cast<const float4 *>(fout), route_pos, recv, rows, d_model / 4, (int)routes_per_row,
               (int)raw, reinterpret_cast<float4 *>(back));
    return check_launch("ep_partial");
}

extern "C" cq_status cq_ep_combine(const float *ret, const int32_t *src_slot, const float *src_w, int64_t n_tokens,
                                   int64_t top_k, int64_t d_model, const float *add, int64_t n_add, int64_t add_stride,
                                   float *out, void *stream) {
    if (d_model <= 0 || d_model % 4 || top_k < 1 || top_k > EP_MAX_K || n_add < 0 || (n_add > 0 && add == nullptr) ||
        add_stride % 4) {
        set_error("ep_combine: need d_model % 4 == 0, 1 <= top_k <= 16, add given when n_add > 0, add_stride % 4 == 0");
        return CQ_ERR_CONFIG;
    }
    if (n_tokens <= 0) return CQ_OK;
    launch_pdl(ep_combine_kernel, (unsigned)std::min<int64_t>(n_tokens, 148 * 8), 128, 0, as_stream(stream),
               reinterpret_cast<const float4 *>(ret), src_slot, src_w, n_tokens, (int)top_k, d_model / 4,
               reinterpret_cast<const float4 *>(add), (int)n_add, add_stride / 4, reinterpret_cast<float4 *>(out));
    return check_launch("ep_combine");
}
