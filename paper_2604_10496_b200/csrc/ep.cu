// Expert parallelism, device side: the bookkeeping around
// the two exchanges of an EP MoE step, done on the GPU so that one step has no
// host synchronisation and can be captured in a CUDA graph.
//
// Slots.  Every rank sends every peer a fixed block of `capacity` rows, so the
// exchanges are equal-split all_to_alls (or peer-memory copies).  A row is
// [codes][f32 scale][i32 local expert id][8 pad bytes]; unused slots carry
// expert id -1.  The codes are A4 values in [-8, 7], sent as packed nibbles
// (d_model / 2 bytes, low nibble first, the reference's int4 format) when
// d_model % 32 == 0, else one byte each.  capacity >= n_tokens * min(top_k,
// experts_per_rank) is enough for any routing (a token's top-k experts are
// distinct, so it sends at most min(k, per) routes to one rank).
//
//   cq_ep_dispatch  route (t, s) -> slot dst*capacity + rank, rank = stable
//                   order of the route among this rank's routes to dst
//                   ((t, s) order, as ep.plan_dispatch); packs the send rows
//                   and writes inv[t, s] = slot, the row the route's output
//                   comes back in, for cq_moe_combine.
//   cq_ep_group     received slots -> codes/scales grouped by local expert
//                   (stable in slot order) + offsets + slot_of_row.
//   cq_ep_scatter   grouped expert outputs -> slot order, for the return.
//
// Rows are computed independently by every expert kernel, so the grouping
// order does not change any bit of the result; stability just makes the
// buffers deterministic.
#include "common.cuh"

namespace cq {

constexpr int EP_THREADS = 1024;
constexpr int EP_MAX_BUCKETS = 256;

struct KeySrc {
    const int32_t *p;      // key word of item i at p[i * stride]
    int64_t stride;        // in int32 words
    int32_t div;           // bucket = word / div (negative word -> skipped)
};

__device__ __forceinline__ int bucket_of(const KeySrc &k, int64_t i) {
    const int32_t v = k.p[i * k.stride];
    return v < 0 ? -1 : v / k.div;
}

// Stable bucket ranks in one block: rank[i] = #{j < i : bucket(j) == bucket(i)},
// counts[b], optional exclusive offsets[0..nb] and slot_item[b*cap + rank] = i.
// Warps match equal buckets (__match_any_sync); a per-(warp, bucket) table in
// shared memory carries the prefix across warps and chunks.
__global__ void __launch_bounds__(EP_THREADS) bucket_rank_kernel(KeySrc ks, int64_t n, int nb, int32_t *rank,
                                                                 int32_t *counts, int32_t *offsets,
                                                                 int32_t *slot_item, int64_t cap) {
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
        const int key = i < n ? bucket_of(ks, i) : -1;
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
        if (key >= 0) {
            const int r = wtab[warp * nb + key] + lr;
            rank[i] = r;
            if (slot_item != nullptr) slot_item[key * cap + r] = (int32_t)i;
        }
        __syncthreads();
    }
    for (int b = tid; b < nb; b += EP_THREADS) counts[b] = carry[b];
    if (offsets != nullptr && tid == 0) {
        int acc = 0;
        for (int b = 0; b < nb; ++b) {
            offsets[b] = acc;
            acc += carry[b];
        }
        offsets[nb] = acc;
    }
}

cq_status bucket_rank(const KeySrc &ks, int64_t n, int nb, int32_t *rank, int32_t *counts, int32_t *offsets,
                      int32_t *slot_item, int64_t cap, cudaStream_t st) {
    const size_t smem = (size_t)33 * nb * sizeof(int32_t);
    bucket_rank_kernel<<<1, EP_THREADS, smem, st>>>(ks, n, nb, rank, counts, offsets, slot_item, cap);
    return check_launch("ep_bucket_rank");
}

// Send rows: slot s = (dst, p).  Filled slots copy the token's codes, scale
// and local expert id; empty slots get expert id -1.  Also inv[route] = slot.
__host__ __device__ inline bool ep_packed(int64_t d) { return d % 32 == 0; }
__host__ __device__ inline int64_t ep_code_bytes(int64_t d) { return ep_packed(d) ? d / 2 : d; }

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

__global__ void ep_pack_kernel(const int8_t *__restrict__ codes, const float *__restrict__ scales,
                               const int32_t *__restrict__ selected, const int32_t *__restrict__ rank, int64_t R,
                               int64_t k, int64_t d, int32_t per, const int32_t *__restrict__ counts,
                               const int32_t *__restrict__ slot_route, int64_t cap, int64_t slots,
                               uint8_t *__restrict__ send, int32_t *__restrict__ inv) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t cb = ep_code_bytes(d), cp = cb / 16;  // code pieces of 16 bytes
    const int64_t pieces = cp + 1, total = slots * pieces;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += stride) {
        const int64_t s = x / pieces, pc = x - s * pieces;
        const int64_t dst = s / cap, p = s - dst * cap;
        uint4 *out = reinterpret_cast<uint4 *>(send + s * (cb + 16)) + pc;
        if (p < counts[dst]) {
            const int32_t r = slot_route[s];
            const int64_t t = r / k;
            if (pc < cp) {
                if (ep_packed(d)) {  // 32 codes -> 16 bytes
                    const uint4 *src = reinterpret_cast<const uint4 *>(codes + t * d) + 2 * pc;
                    const uint4 u = src[0], v = src[1];
                    *out = make_uint4(nib_pack8(u.x, u.y), nib_pack8(u.z, u.w), nib_pack8(v.x, v.y),
                                      nib_pack8(v.z, v.w));
                } else {
                    *out = reinterpret_cast<const uint4 *>(codes + t * d)[pc];
                }
            } else {
                *out = make_uint4(__float_as_uint(scales[t]), (uint32_t)(selected[r] % per), 0u, 0u);
            }
        } else if (pc == cp) {
            *out = make_uint4(0u, 0xffffffffu, 0u, 0u);
        }
    }
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += stride)
        inv[r] = (selected[r] / per) * (int32_t)cap + rank[r];
}

// Received slots -> grouped rows: pos = offsets[e] + rank[slot].
__global__ void ep_group_kernel(const uint8_t *__restrict__ recv, int64_t slots, int64_t d,
                                const int32_t *__restrict__ rank, const int32_t *__restrict__ offsets,
                                int8_t *__restrict__ codes_perm, float *__restrict__ scales_perm,
                                int32_t *__restrict__ slot_of_row) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t cb = ep_code_bytes(d), pieces = cb / 16, total = slots * pieces;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = x / pieces, pc = x - s * pieces;
        const uint8_t *row = recv + s * (cb + 16);
        const int32_t e = *reinterpret_cast<const int32_t *>(row + cb + 4);
        if (e < 0) continue;
        const int64_t pos = offsets[e] + rank[s];
        const uint4 w = reinterpret_cast<const uint4 *>(row)[pc];
        if (ep_packed(d)) {  // 16 bytes -> 32 codes
            uint4 *dst = reinterpret_cast<uint4 *>(codes_perm + pos * d) + 2 * pc;
            dst[0] = make_uint4(nib_unpack4(w.x), nib_unpack4(w.x >> 16), nib_unpack4(w.y), nib_unpack4(w.y >> 16));
            dst[1] = make_uint4(nib_unpack4(w.z), nib_unpack4(w.z >> 16), nib_unpack4(w.w), nib_unpack4(w.w >> 16));
        } else {
            reinterpret_cast<uint4 *>(codes_perm + pos * d)[pc] = w;
        }
        if (pc == 0) {
            scales_perm[pos] = *reinterpret_cast<const float *>(row + cb);
            slot_of_row[pos] = (int32_t)s;
        }
    }
}

__global__ void ep_scatter_kernel(const float4 *__restrict__ fout, const int32_t *__restrict__ live,
                                  const int32_t *__restrict__ slot_of_row, int64_t rows_bound, int64_t d4,
                                  float4 *__restrict__ back) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t n = *live, total = (n < rows_bound ? n : rows_bound) * d4;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t pos = x / d4, c = x - pos * d4;
        back[(int64_t)slot_of_row[pos] * d4 + c] = fout[x];
    }
}

struct EpScratch {
    int32_t *rank, *counts, *slot_route;
};

EpScratch ep_carve(void *scratch, int64_t items, int64_t buckets) {
    int32_t *p = reinterpret_cast<int32_t *>(scratch);
    const int64_t a = ceil_div(items, 64) * 64, b = ceil_div(buckets, 64) * 64;
    return {p, p + a, p + a + b};
}

}  // namespace cq

using namespace cq;

extern "C" int64_t cq_ep_row_bytes(int64_t d_model) { return ep_code_bytes(d_model) + 16; }

extern "C" int64_t cq_ep_scratch_bytes(int64_t n_tokens, int64_t top_k, int32_t world, int64_t capacity,
                                       int64_t n_local) {
    const int64_t items = std::max<int64_t>(n_tokens * top_k, (int64_t)world * capacity);
    const int64_t buckets = std::max<int64_t>(world, n_local);
    return 4 * (ceil_div(items, 64) * 64 + ceil_div(buckets, 64) * 64 + (int64_t)world * capacity + 64);
}

extern "C" cq_status cq_ep_dispatch(const int8_t *codes, const float *scales, const int32_t *selected,
                                    int64_t n_tokens, int64_t top_k, int64_t d_model, int64_t experts_per_rank,
                                    int32_t world, int64_t capacity, uint8_t *send, int32_t *inv, void *scratch,
                                    void *stream) {
    if (d_model <= 0 || d_model % 16 || top_k < 1 || experts_per_rank < 1 || world < 1 || world > EP_MAX_BUCKETS) {
        set_error("ep_dispatch: need d_model % 16 == 0, top_k >= 1, experts_per_rank >= 1, 1 <= world <= 256");
        return CQ_ERR_CONFIG;
    }
    if (capacity < n_tokens * std::min(top_k, experts_per_rank)) {
        set_error("ep_dispatch: capacity < n_tokens * min(top_k, experts_per_rank)");
        return CQ_ERR_CONFIG;
    }
    cudaStream_t st = as_stream(stream);
    const int64_t R = n_tokens * top_k, slots = (int64_t)world * capacity;
    EpScratch s = ep_carve(scratch, std::max(R, slots), std::max<int64_t>(world, 1));
    if (R > 0) CQ_TRY(bucket_rank({selected, 1, (int32_t)experts_per_rank}, R, world, s.rank, s.counts, nullptr,
                                  s.slot_route, capacity, st));
    else if (cudaMemsetAsync(s.counts, 0, world * sizeof(int32_t), st) != cudaSuccess) {
        set_error("ep_dispatch: memset failed");
        return CQ_ERR_CUDA;
    }
    if (slots == 0) return CQ_OK;
    const int64_t total = slots * (d_model / 16 + 1);
    ep_pack_kernel<<<(unsigned)std::min<int64_t>(ceil_div(std::max(total, R), 256), 148 * 8), 256, 0, st>>>(
        codes, scales, selected, s.rank, R, top_k, d_model, (int32_t)experts_per_rank, s.counts, s.slot_route,
        capacity, slots, send, inv);
    return check_launch("ep_pack");
}

extern "C" cq_status cq_ep_group(const uint8_t *recv, int64_t slots, int64_t d_model, int64_t n_local,
                                 int8_t *codes_perm, float *scales_perm, int32_t *offsets, int32_t *slot_of_row,
                                 void *scratch, void *stream) {
    if (d_model <= 0 || d_model % 16 || n_local < 1 || n_local > EP_MAX_BUCKETS) {
        set_error("ep_group: need d_model % 16 == 0 and 1 <= n_local <= 256");
        return CQ_ERR_CONFIG;
    }
    cudaStream_t st = as_stream(stream);
    EpScratch s = ep_carve(scratch, std::max<int64_t>(slots, 1), n_local);
    const int64_t cb = ep_code_bytes(d_model);  // expert id after the codes and the scale
    const KeySrc ks{reinterpret_cast<const int32_t *>(recv + cb + 4), (cb + 16) / 4, 1};
    CQ_TRY(bucket_rank(ks, slots, (int)n_local, s.rank, s.counts, offsets, nullptr, 0, st));
    const int64_t total = slots * (d_model / 16);
    if (total == 0) return CQ_OK;
    ep_group_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 8), 256, 0, st>>>(
        recv, slots, d_model, s.rank, offsets, codes_perm, scales_perm, slot_of_row);
    return check_launch("ep_group");
}

extern "C" cq_status cq_ep_scatter(const float *fout, const int32_t *offsets, const int32_t *slot_of_row,
                                   int64_t n_local, int64_t rows_bound, int64_t d_model, float *back, void *stream) {
    if (d_model % 4) {
        set_error("ep_scatter: need d_model % 4 == 0");
        return CQ_ERR_CONFIG;
    }
    if (rows_bound == 0) return CQ_OK;
    const int64_t d4 = d_model / 4;
    ep_scatter_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows_bound * d4, 256), 148 * 8), 256, 0,
                        as_stream(stream)>>>(reinterpret_cast<const float4 *>(fout), offsets + n_local, slot_of_row,
                                             rows_bound, d4, reinterpret_cast<float4 *>(back));
    return check_launch("ep_scatter");
}
