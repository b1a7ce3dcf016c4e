/* cq_b200 — C ABI of the B200-native CodeQuant Stage-4 path (LUT MoE matmul).
 *
 * Plain pointers and sizes only.  Every pointer argument is DEVICE memory
 * unless its name ends in `_host`; `stream` is a cudaStream_t passed as void*.
 * Every entry point returns a cq_status; cq_last_error() gives the message.
 *
 * Each entry point replaces one reference interface (reference tree
 * /root/reference/pkg/src/codequant/, file:line):
 *
 *   cq_quantize_a4          quant.py:89-100        quantize_activations(x, QuantSpec(4))
 *   cq_unpack_ids           kernels/fallback.py:35-42  unpack_ids(ids_packed, d_in)
 *   cq_reference_gemm_f32   kernels/_core.pyx:154-211  reference_gemm_f32 (via
 *                           kernels/__init__.py:91-94, lutgemm.py:147-161)
 *   cq_lut_gemm_f32         kernels/_core.pyx:41-151   lut_gemm_f32 (via
 *                           kernels/__init__.py:86-88, lutgemm.py:133-144)
 *   cq_matmul_f32           kernels/_core.pyx:27-38    matmul_f32 (kernels/__init__.py:72-78)
 *   cq_route_topk           model.py:324-330 + 377-385 select_top_k on the router logits
 *   cq_moe_*                model.py:377-404       the MoE block of forward(), promoted to an
 *                                                  operator; the reference
 *                                                  has no such entry point.
 *   cq_lut8_prepare         (new) one-time device re-layout of PackedClusteredWeights for the
 *                           tensor-core path; consumes lutgemm.py:53-87 tensors unchanged.
 *   cq_lut_gemm_tc          (new) the tcgen05 LUT GEMM on prepared weights (lutgemm.py:133-144's
 *                           contract within the digit-plane representation error).
 *
 * Host synchronisation: no entry point synchronises the stream.  Errors the
 * reference raises from data (non-finite activations -> DivergenceError,
 * quant.py:93-94, model.py:307-309) are reported through caller-owned device
 * flags that the caller reads at its next sync.
 */
#ifndef CQ_B200_H
#define CQ_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define CQ_API __attribute__((visibility("default")))
#else
#define CQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CQ_OK = 0,
    CQ_ERR_SHAPE = 1,      /* -> ShapeError       (errors.py:12)  */
    CQ_ERR_CONFIG = 2,     /* -> ConfigError      (errors.py:20)  */
    CQ_ERR_DIVERGENCE = 3, /* -> DivergenceError  (errors.py:28)  */
    CQ_ERR_CUDA = 4,       /* -> RuntimeError (CUDA launch / device fault) */
    CQ_ERR_UNSUPPORTED = 5 /* -> ConfigError: shape outside a kernel's envelope */
} cq_status;

enum { CQ_DTYPE_F32 = 0, CQ_DTYPE_BF16 = 1 };

/* Last error message of the calling thread ("" when none). */
CQ_API const char *cq_last_error(void);
/* ABI version, bumped on any signature change. */
CQ_API int cq_abi_version(void);
/* Number of kernels this library launched so far (all entry points). */
CQ_API int64_t cq_launch_count(void);

/* Per-token symmetric 4-bit quantization, bit-exact with quant.py:89-100 for
 * float32 input (bf16 input is quantized as its exact float32 upcast).
 * x: (n, d) row-major, dtype CQ_DTYPE_*.  codes: (n, d) int8, scales: (n,) f32.
 * nonfinite (device int32, nullable): set to 1 when a row holds inf / NaN (the
 * reference's DivergenceError, quant.py:93-94); never cleared here. */
CQ_API cq_status cq_quantize_a4(const void *x, int dtype, int64_t n, int64_t d, int8_t *codes,
                         float *scales, int32_t *nonfinite, void *stream);

/* Low-nibble-first unpack, bit-exact: ids[r, 2m] = b & 15, ids[r, 2m+1] = b >> 4.
 * packed: (rows, ceil(d_in/2)) u8 -> ids: (rows, d_in) u8. */
CQ_API cq_status cq_unpack_ids(const uint8_t *packed, int64_t rows, int64_t d_in, uint8_t *ids,
                        void *stream);

/* Ordered per-element GEMM, BIT-EXACT with reference_gemm_f32 / lut_gemm_f32:
 * out[t,i] = s_t * (((0 + c(i,0)*q(t,0)) + c(i,1)*q(t,1)) + ...), fp32, no FMA.
 * codes (n, d_in) int8 (4- or 8-bit values), scales (n,), ids_packed
 * (d_out, ceil(d_in/2)), centroids (d_out, d_in/g, 16) f32, out (n, d_out) f32.
 * Any g >= 1 dividing d_in, any d_in (odd included). */
CQ_API cq_status cq_reference_gemm_f32(const int8_t *codes, const float *scales,
                                const uint8_t *ids_packed, const float *centroids, int64_t n,
                                int64_t d_in, int64_t d_out, int64_t g, float *out,
                                void *stream);

/* lut_gemm_f32 (_core.pyx:41-151): the reference's table entry T[id][q+8] =
 * C_id * float(q) is the same single fp32 product as reference_gemm's, and the
 * chains run in the same order, so this is the same BIT-EXACT computation as
 * cq_reference_gemm_f32 (acceptance #8, tests/test_acceptance.py:358-387). */
CQ_API cq_status cq_lut_gemm_f32(const int8_t *codes, const float *scales, const uint8_t *ids_packed,
                          const float *centroids, int64_t n, int64_t d_in, int64_t d_out,
                          int64_t g, float *out, void *stream);

/* Ordered fp32 matmul, bit-exact with _core.matmul_f32: out (m, n) = a (m, k) @ b (k, n),
 * k ascending, one rounding per multiply and per add. */
CQ_API cq_status cq_matmul_f32(const float *a, const float *b, float *out, int64_t m, int64_t k,
                        int64_t n, void *stream);

/* select_top_k (model.py:324-330) on fp32 logits (n, E): stable descending order,
 * ties -> lower expert id, weights = softmax over the selected logits.
 * selected (n, k) int32, weights (n, k) f32. */
CQ_API cq_status cq_route_topk(const float *logits, int64_t n, int64_t n_experts, int64_t top_k,
                        int32_t *selected, float *weights, void *stream);

/* ---------------------------------------------------------------------------
 * MoE layer operator (model.py:377-404).
 *
 * Expert weights are stacked per site: ids [E][d_out][d_in/2] u8 and centroids
 * [E][d_out][d_in/g][16] f32 — exactly PackedClusteredWeights (lutgemm.py:53-87)
 * of each expert laid end to end.  gate/up: d_in = d_model, d_out = d_ff;
 * down: d_in = d_ff, d_out = d_model.  Optional lut8 tensors (from
 * cq_lut8_prepare) enable the tensor-core path. */
typedef struct {
    const uint8_t *ids;        /* [E][d_out][d_in/2] */
    const float *centroids;    /* [E][d_out][d_in/g][16] */
    int64_t group_size;        /* g */
    /* tensor-core device layout (cq_lut8_prepare); NULL -> fp32 path */
    const uint8_t *tc_ids;     /* [E*d_out/16][d_in/128][1024] fragment-ordered nibbles (same bytes as ids) */
    const int8_t *tc_lut;      /* [E*d_out/16][d_in/g][16 rows][planes][16] int8 digit-plane LUTs */
    const float *tc_rowscale;  /* [E*d_out] */
    int64_t tc_planes;         /* 2 or 3 unsigned base-128 digit planes (3 where the output is re-quantized) */
    int64_t tc_layout;         /* CQ_TC_UMMA128U / CQ_TC_UMMA128U8 */
} cq_expert_site;

/* Tensor-core layouts (tcgen05 kernel, cq_lut8_prepare).  CQ_TC_UMMA128U8: the
   data of CQ_TC_UMMA128U, declared to have every id < 8 (codebooks with K <= 8,
   W3/W2): one PRMT per 4 operand bytes instead of three instructions.  The
   caller guarantees the ids; the preparation is identical.  (Values 0 and 1
   were the retired mma.sync and signed-digit layouts.) */
enum { CQ_TC_UMMA128U = 2, CQ_TC_UMMA128U8 = 3 };

typedef struct {
    int64_t d_model, d_ff, n_experts, top_k;
    int64_t n_local_experts;   /* experts held by this rank (== n_experts w/o EP) */
    int64_t expert_begin;      /* global id of the first local expert */
    const float *w_router;     /* [d_model][n_experts] f32 (full precision, pipeline.py:455-467) */
    const float *rotation;     /* optional online rotation R [d_model][d_model] f32, v = x @ R */
    cq_expert_site gate, up, down;
    int64_t n_shared;          /* builder-defined always-on experts (weight 1), stacked like the above */
    cq_expert_site sh_gate, sh_up, sh_down;
    int32_t path;              /* CQ_PATH_* */
    const void *rotation_tc;   /* optional: R prepared by cq_rotation_prepare (tensor-core rotation);
                                  NULL -> fp32 CUDA-core rotation of `rotation` */
    int64_t flags;             /* CQ_FLAG_* */
} cq_moe_desc;

/* CQ_FLAG_KEEP_HIDDEN: the tensor-core path also stores h = silu(a) * b in
   CQ_WS_HIDDEN (fp32) and its codes row-major in CQ_WS_HCODES (for tracing / parity
   checks).  Without it the expert stage writes the re-quantized h only into the down
   GEMM's operand tiles (CQ_WS_HCODES_FRAG) and CQ_WS_HSCALES, and CQ_WS_HIDDEN holds the
   gate output; the f32 and ordered paths always store h and its codes. */
enum { CQ_FLAG_KEEP_HIDDEN = 1 };
/* CQ_FLAG_SELECT_ONLY: cq_moe_route stops after the top-k (codes, scales, logits,
   selected, weights, tok_sums): no segment permutation or gathered codes (the
   expert-parallel driver plans its own rows). */
enum { CQ_FLAG_SELECT_ONLY = 2 };
/* CQ_FLAG_SHARED_MERGED: the tensor-core data of the shared experts (sh_gate/sh_up/sh_down)
   directly follows the routed experts' in gate/up/down (tc_ids, tc_lut, tc_rowscale), so
   cq_moe_forward runs them as extra segments of the routed grouped launches (all tokens each,
   weight 1) instead of separate launches.  Same per-row arithmetic, same results. */
enum { CQ_FLAG_SHARED_MERGED = 4 };

enum { CQ_PATH_AUTO = 0, CQ_PATH_F32 = 1, CQ_PATH_TC = 2, CQ_PATH_ORDERED = 3 };

/* Named scratch buffers inside the caller-provided workspace. */
enum {
    CQ_WS_CODES = 0,    /* int8 [n][d_model]   layer-input codes            */
    CQ_WS_SCALES,       /* f32  [n]                                          */
    CQ_WS_LOGITS,       /* f32  [n][E]         ordered router logits         */
    CQ_WS_SELECTED,     /* i32  [n][k]                                       */
    CQ_WS_WEIGHTS,      /* f32  [n][k]                                       */
    CQ_WS_COUNTS,       /* i32  [E+1]          routes per expert; [E] arrival counter */
    CQ_WS_OFFSETS,      /* i32  [E+1]          local expert segments         */
    CQ_WS_PERM_TOKEN,   /* i32  [n*k]                                        */
    CQ_WS_PERM_SLOT,    /* i32  [n*k]                                        */
    CQ_WS_INV,          /* i32  [n][k]         route -> segment row          */
    CQ_WS_CODES_PERM,   /* int8 [n*k][d_model] codes gathered per segment    */
    CQ_WS_SCALES_PERM,  /* f32  [n*k]                                        */
    CQ_WS_HIDDEN,       /* f32  [n*k][d_ff]    silu(a)*b (tc path: CQ_FLAG_KEEP_HIDDEN) */
    CQ_WS_HCODES,       /* int8 [n*k][d_ff]    re-quantized hidden           */
    CQ_WS_HSCALES,      /* f32  [n*k]                                        */
    CQ_WS_FOUT,         /* f32  [n*k][d_model] per-route down output         */
    CQ_WS_ROTATED,      /* f32  [n][d_model]   x @ R (online rotation only)  */
    CQ_WS_SHARED,       /* f32  [n_shared][n][d_model] per shared expert    */
    CQ_WS_CODES_FRAG,   /* int8 [ceil(n*k/8)*8][d_model] codes in mma-B fragment order */
    CQ_WS_HCODES_FRAG,  /* int8 [ceil(n*k/8)*8][d_ff]    hidden codes, fragment order  */
    CQ_WS_ROT_ACT,      /* bf16 [3][ceil(n/128)*128][d_model] rotation operand planes (rotation_tc) */
    CQ_WS_TOK_SUMS,     /* i32  [n]            per-token code sums (GEMM bias term) */
    CQ_WS_STATUS,       /* i32  [4]            sticky non-finite flags: [0] layer input (router / gate /
                                               up sites), [1] hidden (down input).  Zero it once when
                                               the workspace is created; the layer only sets it. */
    CQ_WS_SH_OFFSETS,   /* i32  [2]            shared-expert segment (0, n)                  */
    CQ_WS_COUNT_
};

/* Byte offsets of every CQ_WS_* buffer for n tokens; returns the total size. */
CQ_API int64_t cq_moe_workspace(const cq_moe_desc *desc, int64_t n_tokens, int64_t *offsets_out);

/* Full layer: x (n, d_model) dtype CQ_DTYPE_* -> out (n, d_model) f32 = moe_sum.
 * No host synchronisation; deterministic for a given path.  Non-finite values
 * set CQ_WS_STATUS (read it after a sync; the reference raises DivergenceError). */
CQ_API cq_status cq_moe_forward(const cq_moe_desc *desc, const void *x, int dtype, int64_t n_tokens,
                         float *out, void *workspace, int64_t workspace_bytes, void *stream);

/* The stages of cq_moe_forward, exposed for expert parallelism (the EP driver
 * runs routing on every rank, exchanges codes, and runs the expert stage on the
 * rank that owns the expert). */
CQ_API cq_status cq_moe_route(const cq_moe_desc *desc, const void *x, int dtype, int64_t n_tokens,
                       void *workspace, int64_t workspace_bytes, void *stream);
/* Grouped experts over segment rows: codes_perm (rows, d_model), scales_perm,
 * offsets (n_local+1) -> fout (rows, d_model).  `rows` is a host-known bound. */
CQ_API cq_status cq_moe_experts(const cq_moe_desc *desc, const int8_t *codes_perm,
                         const float *scales_perm, const int32_t *offsets, int64_t rows,
                         float *fout, void *workspace, int64_t workspace_bytes, void *stream);
/* Profiling: runs the expert stage `iters` times with CUDA events between its
 * kernels on `stream`; stage_ms_host[3] (host memory) receives the mean device
 * time of {gate|up GEMM (+ operand re-layout), silu*up + re-quantization, down GEMM}. */
CQ_API cq_status cq_moe_profile_experts(const cq_moe_desc *desc, const int8_t *codes_perm,
                                 const float *scales_perm, const int32_t *offsets, int64_t rows,
                                 float *fout, void *workspace, int64_t workspace_bytes,
                                 int32_t iters, float *stage_ms_host, void *stream);
/* Weighted combine in ascending expert order (model.py:389-401), then
 * out = ((routed + add_0) + add_1) ... over n_add buffers of [n_tokens][d_model]
 * laid end to end (shared-expert outputs; add may be NULL when n_add == 0). */
CQ_API cq_status cq_moe_combine(const int32_t *selected, const float *weights, const int32_t *inv,
                         const float *fout, int64_t n_tokens, int64_t top_k, int64_t d_model,
                         const float *add, int64_t n_add, float *out, void *stream);
/* The builder-defined shared experts (weight 1) of desc over the
 * n_tokens layer-input codes cq_moe_route left in the workspace:
 * shared_out [n_shared][n_tokens][d_model] f32.  Expert parallelism runs them on
 * every rank for its own tokens (they are replicated, no exchange). */
CQ_API cq_status cq_moe_shared_experts(const cq_moe_desc *desc, int64_t n_tokens, float *shared_out,
                                void *workspace, int64_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Expert parallelism, device-side planning (the reference has
 * no multi-GPU path — it evaluates every expert on every token, model.py:391-401
 * — so these serve the EP driver paper_2604_10496_b200/ep.py).  Experts
 * [r*per, (r+1)*per) live on rank r; the router weight and shared experts are
 * replicated.
 *
 * A rank sends each peer rows of cq_ep_row_bytes(d_model, kr) bytes:
 *   [codes][f32 scale][i32 m][(i32 e_j, f32 w_j) x kr][pad to 16 B]
 * codes as packed nibbles when d_model % 32 == 0 (else int8); m routes to the
 * peer's local experts e_0 < e_1 < ... (e = -1 past m).
 *   dedup != 0: one row per (token, peer) holding all its routes there,
 *     kr = min(top_k, experts_per_rank); the peer returns one fp32 partial sum
 *     per row (cq_ep_partial), the source adds them in ascending peer order.
 *   dedup == 0: one row per route, kr = 1, w = 1; the source applies the route
 *     weights: bitwise equal to cq_moe_forward for any world size.
 * capacity > 0: `capacity` rows per peer (fixed slots, equal-split exchanges,
 * no host read: a whole step fits one CUDA graph); >= n_tokens (dedup) or
 * n_tokens * min(top_k, experts_per_rank).  capacity == 0: compact, rows to
 * peer g follow the rows to peers < g (all_to_all-v sized by the counts). */
CQ_API int64_t cq_ep_row_bytes(int64_t d_model, int64_t routes_per_row);
/* Device scratch bytes for cq_ep_dispatch / cq_ep_group with these sizes. */
CQ_API int64_t cq_ep_scratch_bytes(int64_t n_tokens, int64_t top_k, int64_t recv_rows, int64_t routes_per_row,
                                   int64_t n_local);
/* codes (n, d) int8, scales (n,), selected (n, k) global expert ids, weights
 * (n, k) (cq_moe_route) -> send rows; counts[g*counts_stride + {0, 1}] = rows /
 * routes sent to peer g; per token the returned rows to add, in ascending peer
 * (dedup) or expert order: src_slot (n, k) (row index in the returned buffer,
 * -1 ends the list) and src_w (n, k) (1 in dedup mode). */
CQ_API cq_status cq_ep_dispatch(const int8_t *codes, const float *scales, const int32_t *selected,
                                const float *weights, int64_t n_tokens, int64_t top_k, int64_t d_model,
                                int64_t experts_per_rank, int32_t world, int32_t dedup, int64_t capacity,
                                uint8_t *send, int32_t *counts, int64_t counts_stride, int32_t *src_slot,
                                float *src_w, void *scratch, void *stream);
/* Received rows recv [rows] -> codes_perm / scales_perm grouped by local expert
 * (stable in (row, j) order), offsets (n_local+1), route_pos [rows][kr] (grouped
 * row of each route, -1 for none).  Pass rows * kr (or the exact route count) as
 * the row bound of cq_moe_experts. */
CQ_API cq_status cq_ep_group(const uint8_t *recv, int64_t rows, int64_t d_model, int64_t routes_per_row,
                             int64_t n_local, int8_t *codes_perm, float *scales_perm, int32_t *offsets,
                             int32_t *route_pos, void *scratch, void *stream);
/* Grouped expert outputs fout -> back [rows][d] f32, one returned row per
 * received row with m > 0: raw (dedup == 0): the route's output as is; else
 * ((0 + w_0 f_0) + w_1 f_1) ... in ascending expert order. */
CQ_API cq_status cq_ep_partial(const float *fout, const int32_t *route_pos, const uint8_t *recv, int64_t rows,
                               int64_t d_model, int64_t routes_per_row, int32_t raw, float *back, void *stream);
/* out[t] = ((0 + src_w[t,0] ret[src_slot[t,0]]) + ...) over the token's list,
 * then + add[u*add_stride + t*d] for u < n_add (shared-expert outputs, in order). */
CQ_API cq_status cq_ep_combine(const float *ret, const int32_t *src_slot, const float *src_w, int64_t n_tokens,
                               int64_t top_k, int64_t d_model, const float *add, int64_t n_add, int64_t add_stride,
                               float *out, void *stream);

/* Online rotation on the tensor cores (pipeline.py:516, v = x @ R) at fp32 accuracy:
 * R (d, d) f32 is split once into three bf16 planes of R^T in the UMMA operand layout
 * (`prepared`: cq_rotation_prepared_bytes(d) bytes); set cq_moe_desc.rotation_tc to it.
 * Requires d % 256 == 0. */
CQ_API int64_t cq_rotation_prepared_bytes(int64_t d_model);
CQ_API cq_status cq_rotation_prepare(const float *rotation, int64_t d_model, void *prepared, void *stream);

/* One-time re-layout of one stacked site (rows = E*d_out) for the tensor-core path:
 * every row's centroids become integers m = rint(c / rowscale), |m| < 2^(7P-1),
 * at one per-row scale, stored as P unsigned base-128 digit planes of 16-entry
 * byte LUTs (m + 2^(7P-1)); ids are re-tiled into 128-row k-step blocks (same
 * bytes).  tc_ids: d_in/2 bytes per row; tc_lut: rows * (d_in/g) * planes * 16;
 * tc_rowscale: rows floats.  Requires rows % 128 == 0, d_in % 128 == 0,
 * g % 128 == 0, planes in {2, 3}, layout CQ_TC_UMMA128U / _UMMA128U8. */
CQ_API cq_status cq_lut8_prepare(const uint8_t *ids, const float *centroids, int64_t rows,
                          int64_t d_in, int64_t g, int64_t planes, int64_t layout,
                          uint8_t *tc_ids, int8_t *tc_lut, float *tc_rowscale, void *stream);

/* Tensor-core LUT GEMM on prepared weights (one matrix): codes (n, d_in) int8
 * row-major (4- or 8-bit values), out (n, d_out) f32.  Same contract as
 * cq_lut_gemm_f32 within the digit-plane representation error (<= 2^-(7P-1) of
 * the row max per weight).  workspace: device scratch of at least
 * cq_lut_gemm_tc_workspace(n, d_in) bytes (no allocation inside). */
CQ_API int64_t cq_lut_gemm_tc_workspace(int64_t n, int64_t d_in);
CQ_API cq_status cq_lut_gemm_tc(const int8_t *codes, const float *scales, const uint8_t *tc_ids,
                         const int8_t *tc_lut, const float *tc_rowscale, int64_t planes,
                         int64_t layout, int64_t n, int64_t d_in, int64_t d_out, int64_t g,
                         float *out, void *workspace, int64_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CQ_B200_H */
