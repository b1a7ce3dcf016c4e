// tcgen05 LUT GEMM: codebook rows expanded by PRMT into int8 digit planes and
// written straight into TMEM as the MMA's A operand (kind::i8, A from TMEM),
// activation codes staged in shared memory by bulk copies as the B operand,
// exact int32 accumulators in TMEM.
//
// Numerics.  Each weight row's centroids are integers m = rint(c / rowscale)
// written as P int8 digit planes: 3 planes where the GEMM output is
// re-quantized (gate, up), 2 for down.  Codes are exact int8 and each plane's
// GEMM is an exact s8 x s8 -> s32 MMA; planes are combined in the epilogue.
//
// Lookup.  A (row, group) codebook plane is a 16-entry byte table in 4
// registers.  Four consecutive packed ids are exactly a `prmt.b32` selector
// (two ids per byte, low nibble first, lutgemm.py:111-116); ids 8..15 set the
// selector's sign-replicate bit, so prmt(entries 0..7, sel) and prmt(entries
// 8..15, sel ^ 0x8888) each give the right bytes for their half and a
// replicated sign byte for the other.  Digits are unsigned base 128, biased
// by 2^(7P-1) (CQ_TC_UMMA128U, lut7_kernel in prepare.cu): their sign bits are
// clear, so the replicated byte is 0 and the halves merge with one integer
// add (2 PRMT + 1 IMAD per 4 weights per plane, P MMAs per k-step); the bias
// returns in the epilogue as 2^(7P-1) * sum_j q[t,j].  CQ_TC_UMMA128U8 (every
// id < 8, codebooks with K <= 8) needs the first PRMT only.
//
// CTA = one 128-row weight tile of one expert matrix x token passes of <= 32
// tokens (MMA N = 16 or 32), warp-specialised, one CTA per SM (it owns all
// 512 TMEM columns):
//   warps 0-15 expanders, 4 warpgroups: warp w owns TMEM lane quarter w%4
//              (= 32 rows); warpgroup w/4 expands k-step w/4 of every
//              128-column chunk into its own A stages (tcgen05.st).  Four
//              warpgroups in flight hide the TMEM store latency.
//   warp 16    producer: cp.async.bulk of ids (8 KB per chunk), the group's LUT
//              block and the activation tile into an 8-deep smem ring.
//   warp 17    MMA issuer: the whole warp runs the loop converged and
//              elect.sync picks the issuing lane inside the asm (a divergent
//              `if (lane == 0)` issue costs ~200 cycles per MMA, converged
//              ~18: profiles/microbench/umma_probe.cu).  2P (or P) MMAs of
//              M=128, N=16|32, K=32 per k-step into P int32 accumulators.
// Epilogue: expanders tcgen05.ld the accumulators, combine the digits, scale
// by the row scale and the token scale, store fp32.
#include "common.cuh"
#include "route_perm.cuh"
#include "tc_ptx.cuh"

#include <cstdlib>

namespace cq {

#ifndef UM_CK
#define UM_CK 128  // measured: 64 (8 A stages, 2 per stream) loses to the per-chunk handshake cost
#endif
#ifndef UM_GS4  // chunk streams when >= 4 A stages fit (measured: 4 beats 2 double-buffered)
#define UM_GS4 4
#endif
#ifndef UM_PF2_GS  // chunk streams of the 2-plane prefill GEMM
#define UM_PF2_GS 2
#endif
#ifndef UM_SPLIT_AFREE  // data (full) and A-stage-free (afree) as separate barriers: 0 never, 1 always,
#define UM_SPLIT_AFREE 2  // 2: prefill geometry, 3 planes only (decode and the 2-plane down GEMM measured slower)
#endif
#ifndef UM_LAG  // chunks of data issued ahead of arming (smem ring = A stages + UM_LAG)
#define UM_LAG 4
#endif
#ifndef LAG_P2
#define LAG_P2 1
#endif
#ifndef UM_KGRP  // k-steps whose lookups all precede their TMEM stores
#define UM_KGRP 2
#endif
#ifndef LAG_P3
#define LAG_P3 1
#endif
namespace um {
constexpr int STAGES = 8;        // most A stages used
constexpr int WG = 4;            // expander warpgroups; warpgroup w expands k-step w of every chunk
constexpr int EXP_WARPS = 4 * WG, PROD_WARP = EXP_WARPS, MMA_WARP = EXP_WARPS + 1;
constexpr uint32_t TMEM_COLS = 512;
}  // namespace um

#ifndef UM_MMA_PER_PLANE  // merged layouts: one MMA warp per digit plane (own accumulator, own SMSP)
#define UM_MMA_PER_PLANE 1
#endif
// Warps of a CTA: the expanders, the producer, and NMMA MMA-issuing warps.  The
// MMA warp's issue rate (~55 cycles per tcgen05.mma, sharing an SMSP with 4
// expander warps) bounded the decode GEMM; with one warp per plane each issues
// a third (P = 3) of the MMAs from a different SMSP.  Planes accumulate into
// disjoint TMEM columns, so the warps never touch one accumulator concurrently.
template <int P>
struct UmWarps {
    static constexpr int NMMA = UM_MMA_PER_PLANE ? P : 1;
    static constexpr int WARPS = um::EXP_WARPS + 1 + NMMA;
    static constexpr int THREADS = WARPS * 32;
};

// Pass geometry: NT tokens per pass (MMA N), CK input columns per chunk.  Decode
// uses NT 32 / CK 128 (4 A stages of 4 k-steps); prefill NT 128 / CK 64 (the
// 3 x 128 accumulator columns leave room for 64-column A stages only), which
// expands each weight chunk once per 128 tokens instead of per 32.
template <int NT_, int CK_, int NACC_ = 1>
struct UmGeo {
    static constexpr int NT = NT_, CK = CK_;
    static constexpr int NACC = NACC_;         // accumulator buffers (2: unit u+1's MMAs run during u's epilogue)
    static constexpr int KS = CK / 32;         // MMA k-steps per chunk
    static constexpr int IDS = 128 * CK / 2;   // ids bytes per chunk: 128 rows x CK columns / 2
    static constexpr int BTILE = 8 * CK;       // activation bytes per 8-token tile per chunk
    static constexpr int NCB = NT / 32;        // epilogue column blocks per warpgroup
    static constexpr int PART_WORDS = 3 * NT * 128;  // int32 partial accumulators per slot (P <= 3)
};
using UmDecode = UmGeo<32, UM_CK>;
// prefill passes: 128 tokens, one accumulator (3 x 128 columns).  Measured (tools/gemm_stage.py, PH
// gate|up): 64-token passes with two accumulators 2228 us, 64 single 1933, 128 single 1187 — the
// expansion (PRMT, ALU pipe) bounds prefill too, so fewer tokens per expanded chunk loses.
#ifndef UM_PF_NT
#define UM_PF_NT 128
#endif
#ifndef UM_PF_NACC
#define UM_PF_NACC 1
#endif
using UmPrefill = UmGeo<UM_PF_NT, 64, UM_PF_NACC>;
// The 2-plane (down) prefill GEMM: its 2 x 128 accumulator columns leave room for four 128-column
// A stages, so it takes 128-column chunks (half the per-chunk handshakes of the 3-plane geometry):
// QW down 246 -> 228 us, PH 460 -> 373 us, DS 416 -> 391 us.
#ifndef UM_PF2_CK
#define UM_PF2_CK 128
#endif
using UmPrefill2 = UmGeo<UM_PF_NT, UM_PF2_CK, UM_PF_NACC>;

template <int P, class GEO>
struct UmStage {
    static constexpr int LUT = 128 * P * 16;
    static constexpr int B = (GEO::NT / 8) * GEO::BTILE;
    static constexpr int BYTES = GEO::IDS + LUT + B;
    static constexpr int SLICES = P;                             // MMA K-slices per k-step
    static constexpr int ACOLS = SLICES * 8;                     // TMEM columns per k-step
    static constexpr int CCOLS = GEO::KS * ACOLS;                // TMEM columns per A stage (one chunk)
    static constexpr int ACC1 = P * GEO::NT;                     // columns of one accumulator buffer
    static constexpr int ACC = ACC1 * GEO::NACC;                 // accumulator columns
    static constexpr int NCS = (um::TMEM_COLS - ACC) / CCOLS;    // A stages that fit in TMEM
    static_assert(NCS >= 1, "TMEM budget");
    // Chunk c uses smem stage and TMEM A stage c % NS (one ring).  full[s] for
    // chunk c means the producer refilled stage s, which it does only after the
    // MMAs of chunk c - NS completed (empty[s]), so the A stage is free too:
    // expanders wait on one barrier per chunk.  Chunk c is expanded by
    // stream c % GS; NS is a multiple of GS so every stage belongs to one
    // warpgroup, which consumes its phases in order (a stage shared by two
    // warpgroups would let one pass try_wait.parity on the other's older phase).
    // GS chunk streams: stream g expands the chunks c = g (mod GS); its WG / GS
    // warpgroups split each chunk's 4 k-steps.  Streams work on different
    // chunks (staggered waits, bookkeeping paid per GS k-steps) and each owns
    // NA / GS >= 2 A stages, so it expands chunk c + GS while the MMAs of c run.
    static constexpr int NA0 = NCS < um::STAGES ? NCS : um::STAGES;
    // (the 2-plane prefill GEMM with its four 128-column A stages: 2 streams + 2 stages of data lag
    //  beat 4 streams without lag: PH down 373 -> 354 us)
    static constexpr int GS = (GEO::NT == 128 && P == 2 && NA0 >= 4) ? UM_PF2_GS
                              : NA0 >= 4                             ? UM_GS4
                              : (NA0 >= 2 ? 2 : 1);
    static_assert(GEO::KS % (um::WG / GS) == 0, "a chunk's k-steps split evenly over a stream's warpgroups");
    static constexpr int NA = (NA0 / GS) * GS;
    // LAG > 0: NS = NA + LAG smem stages, so the producer issues chunk c's
    // copies as soon as the MMAs of chunk c - NS are done, LAG chunks before
    // A stage c % NA frees.  full[c % NS] then expects two arrivals: the
    // producer's arrive.expect_tx with the copies, and a tcgen05.commit the MMA
    // warp issues after chunk c - NA (fires when those MMAs, the last readers
    // of the A stage, complete).  full[] alone still means "data and A stage
    // ready", and the producer is out of the expanders' round trip.
    static constexpr int LAG_FIT = ((216 * 1024) / BYTES - NA) / GS * GS;  // most stages the smem holds
    static constexpr int LAG0 = (LAG_P2 && P == 2) || (LAG_P3 && P == 3) ? UM_LAG : 0;
    static constexpr int LAG = LAG0 < LAG_FIT ? LAG0 : LAG_FIT;
    static constexpr int NS = NA + LAG;
    static_assert(NS % GS == 0 && NA % GS == 0 && NS * BYTES <= 216 * 1024, "smem ring");
    static constexpr bool SPLIT_AFREE = UM_SPLIT_AFREE == 1 || (UM_SPLIT_AFREE == 2 && GEO::NT == 128 && P == 3);
};

// ---------------------------------------------------------------------------
// Work decomposition: persistent, data-parallel rounds + a stream-K tail.  A
// unit is one 128-row tile of one matrix for one pass of <= NTOK tokens of one
// segment; its d_in/128 chunks are iterations.  With G CTAs (one per SM),
// CTA b first runs whole units b, b+G, b+2G, ... (the order of a plain grid,
// so concurrent CTAs stream neighbouring tiles) for the full rounds; the R < G
// leftover units, which would otherwise form a mostly idle last wave, are
// split by iterations into equal contiguous ranges over the first G_t CTAs
// (>= MIN_ITERS chunks each).  A unit cut by a range boundary is finished by
// whichever of its CTAs arrives last on a per-unit counter: the others leave
// their int32 partial accumulators in `part`, the last one adds them before
// the epilogue.  Integer sums are exact, so the result does not depend on the
// split.  Every CTA pays the prologue and the pipeline fill once.
namespace um {
constexpr int MAX_SEG = 512;   // segments (experts) per launch, prefix table in smem
#ifndef UM_MIN_ITERS
#define UM_MIN_ITERS 8
#endif
constexpr int MIN_ITERS = UM_MIN_ITERS;   // fewest chunk iterations per CTA in the tail
#ifndef UM_TAIL_DIV  // tail ranges >= n_chunks / UM_TAIL_DIV (QW gate|up 465 -> 444 us, DS 987 -> 974 at 2)
#define UM_TAIL_DIV 2
#endif
}  // namespace um

struct UmWork {
    const int32_t *unit_pre;  // [n_seg + 1] units before segment s (smem)
    const int32_t *seg_off;   // [n_seg + 1] segment row offsets (smem copy of `offsets`)
    int n_rt, n_mat, n_chunks, G, Gt;
    int64_t n_units, full_rounds;
    int64_t T0, T;            // tail: iterations [T0, T0 + T)
    __device__ __forceinline__ int64_t tstart(int b) const { return T0 + (int64_t)b * T / Gt; }
    __device__ int owner(int64_t x) const {  // tail CTA whose range holds iteration x
        int b = (int)((x - T0) * Gt / T);
        while (b + 1 < Gt && tstart(b + 1) <= x) ++b;
        while (b > 0 && tstart(b) > x) --b;
        return b;
    }
};

// A CTA's sequence of (unit, first chunk, end chunk).
struct UmSeq {  // 32-bit: unit and iteration counts stay far below 2^31
    int u_next, full_left, t, te;
    __device__ __forceinline__ bool next(const UmWork &w, int &u, int &c0, int &c1) {
        if (full_left > 0) {
            u = u_next;
            u_next += w.G;
            --full_left;
            c0 = 0;
            c1 = w.n_chunks;
            return true;
        }
        if (t >= te) return false;
        u = t / w.n_chunks;
        c0 = t - u * w.n_chunks;
        c1 = (te - u * w.n_chunks) < w.n_chunks ? (te - u * w.n_chunks) : w.n_chunks;
        t = u * w.n_chunks + c1;
        return true;
    }
};

struct UmUnit {
    int64_t rb, re, j0, tile;
    int ntc, mat;
    int rt;
};

// unit u -> (segment, pass, matrix, row tile); `seg` walks forward (units are visited in order)
__device__ __forceinline__ UmUnit um_unit(const UmWork &w, int64_t seg_first, int u, int &seg, int tpp) {
    while (w.unit_pre[seg + 1] <= u) ++seg;
    UmUnit x;
    x.rb = w.seg_off[seg];
    x.re = w.seg_off[seg + 1];
    const int local = u - w.unit_pre[seg];
    const int per_pass = w.n_rt * w.n_mat;
    const int pass = local / per_pass, r = local - pass * per_pass;
    x.mat = r / w.n_rt;
    x.rt = r - x.mat * w.n_rt;
    const int64_t j_last = (x.re - 1) >> 3;
    x.j0 = (x.rb >> 3) + (int64_t)pass * tpp;
    const int64_t left = j_last - x.j0 + 1;
    x.ntc = (int)(left < tpp ? left : tpp);
    x.tile = (seg + seg_first) * w.n_rt + x.rt;
    return x;
}

// grid: (#SMs); n_mat = 2 computes gate (ids0 ... out0) and up (ids1 ... out1).
// NARROW (merged layout, every id < 8: codebooks with K <= 8): the 8 table
// bytes of entries 0..7 sit in L.x, L.y, so one PRMT yields 4 A bytes (no
// second PRMT over entries 8..15, no merge).
template <int P, class GEO, bool NARROW = false>
__global__ void __launch_bounds__(UmWarps<P>::THREADS, 1) lut_umma_kernel(
    const int8_t *__restrict__ bfrag, int64_t n_tiles, const float *__restrict__ scales,
    const int32_t *__restrict__ qsums, const int32_t *__restrict__ offsets, int n_seg, int64_t seg_first,
    const uint8_t *__restrict__ ids0, const int8_t *__restrict__ lut0, const float *__restrict__ rs0,
    float *__restrict__ out0, const uint8_t *__restrict__ ids1, const int8_t *__restrict__ lut1,
    const float *__restrict__ rs1, float *__restrict__ out1, int n_mat, int d_in, int d_out, int g,
    int32_t *__restrict__ part, int32_t *__restrict__ cnt) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    using S = UmStage<P, GEO>;
    constexpr int NMMA = UmWarps<P>::NMMA;
    constexpr int NA = S::NA, NS = S::NS, GS = S::GS, LAG = S::LAG;
    constexpr int WPS = um::WG / GS;  // warpgroups per stream
    constexpr int NT = GEO::NT, CK = GEO::CK, NCB = GEO::NCB;
    constexpr int TPP = NT / 8;       // token tiles per pass
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full_bar[NS], empty_bar[NS], afull_bar[NA], afree_bar[NA];
    __shared__ __align__(8) uint64_t accfull_bar[GEO::NACC], accempty_bar[GEO::NACC];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int32_t unit_pre[um::MAX_SEG + 1], seg_off[um::MAX_SEG + 1];
    // per expander warp and column block: 8 token scales, 8 row sums
    __shared__ __align__(16) uint32_t tok_sh[2][um::EXP_WARPS][NCB][16];  // [unit parity]
    __shared__ int last_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_chunks = d_in / CK, cpg = g / CK, n_groups = d_in / g;

    // units per segment -> prefix table (warp 0: a serial run per lane + shuffle scan)
    if (warp == 0) {
        const int per = (n_seg + 31) / 32;
        const int s0 = lane * per, s1 = min(n_seg, s0 + per);
        int run = 0;
        for (int s = s0; s < s1; ++s) {
            const int64_t rb = offsets[s], re = offsets[s + 1];
            const int np = rb < re ? (int)((((re - 1) >> 3) - (rb >> 3) + TPP) / TPP) : 0;
            run += np * (d_out / 128) * n_mat;
            unit_pre[s + 1] = run;
            seg_off[s] = (int32_t)rb;
            if (s == n_seg - 1) seg_off[n_seg] = (int32_t)re;
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        for (int s = s0; s < s1; ++s) unit_pre[s + 1] += incl - run;
        if (lane == 0) unit_pre[0] = 0;
    }
    __syncthreads();
    __shared__ UmWork W_sh;  // in smem: keeps the expanders' chunk loop clear of live descriptor registers
    UmWork &W = W_sh;
    W.unit_pre = unit_pre;
    W.seg_off = seg_off;
    W.n_rt = d_out / 128;
    W.n_mat = n_mat;
    W.n_chunks = n_chunks;
    W.G = gridDim.x;
    W.n_units = unit_pre[n_seg];
    W.full_rounds = W.n_units / W.G;
    W.T0 = W.full_rounds * W.G * n_chunks;
    W.T = (W.n_units - W.full_rounds * W.G) * n_chunks;
    {
        // tail ranges of at least max(MIN_ITERS, n_chunks / UM_TAIL_DIV) chunks: long units split over
        // fewer CTAs (fewer partial-sum exchanges)
        const int64_t mi = n_chunks / UM_TAIL_DIV > um::MIN_ITERS ? n_chunks / UM_TAIL_DIV : um::MIN_ITERS;
        const int64_t gt = W.T / mi > 0 ? W.T / mi : 1;
        W.Gt = (int)(gt < W.G ? gt : W.G);
    }
    const int cta = blockIdx.x;
    UmSeq seq0;
    seq0.u_next = cta;
    seq0.full_left = (int)W.full_rounds;
    seq0.t = W.T > 0 && cta < W.Gt ? (int)W.tstart(cta) : 0;
    seq0.te = W.T > 0 && cta < W.Gt ? (int)W.tstart(cta + 1) : 0;
    if (seq0.full_left == 0 && seq0.t >= seq0.te) return;  // CTA-uniform: no work
    const int first_tail_unit = seq0.t / n_chunks;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            u_bar_init(u_smem(&full_bar[s]), (LAG > 0 && !S::SPLIT_AFREE) ? 1 + NMMA : 1);
            u_bar_init(u_smem(&empty_bar[s]), NMMA);
        }
        for (int s = 0; s < NA; ++s) {
            u_bar_init(u_smem(&afull_bar[s]), 4 * WPS);  // the warps of one stream
            u_bar_init(u_smem(&afree_bar[s]), NMMA);      // SPLIT_AFREE: MMAs of the stage's last chunk done
        }
        // (splitting afull per chunk half, so the MMAs start earlier, measured slower: the extra
        //  tcgen05.wait::st mid-chunk costs more than the overlap gains)
        for (int b = 0; b < GEO::NACC; ++b) {
            u_bar_init(u_smem(&accfull_bar[b]), NMMA);
            u_bar_init(u_smem(&accempty_bar[b]), um::EXP_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(u_smem(&tmem_base_sh)),
                     "r"(um::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t a_col0 = (uint32_t)S::ACC;  // A stages follow the accumulators
    // shared-window addresses, computed once (slot s adds 8 * s / s * S::BYTES)
    // (volatile moves: ptxas would otherwise re-derive them from SR_CgaCtaId in every loop iteration)
    const uint32_t full_a = u_pin(u_smem(&full_bar[0])), empty_a = u_pin(u_smem(&empty_bar[0]));
    const uint32_t afull_a = u_pin(u_smem(&afull_bar[0])), stage_a = u_pin(u_smem(smem));
    const uint32_t afree_a = u_pin(u_smem(&afree_bar[0]));

    if (warp == um::PROD_WARP) {
        // ------------------------------------------------------------ producer (converged warp, elected lane)
        uint32_t k = 0;
        int seg = 0;
        UmSeq q = seq0;
        int u, c0, c1;
        while (q.next(W, u, c0, c1)) {
            const UmUnit x = um_unit(W, seg_first, u, seg, TPP);
            const uint8_t *ids = x.mat ? ids1 : ids0;
            const int8_t *lut = x.mat ? lut1 : lut0;
            const int ntc16 = (x.ntc + 1) & ~1;  // MMA N is a multiple of 16
            int grp = c0 / cpg, gc = c0 - grp * cpg;  // group and chunk-in-group, stepped without division
            for (int c = c0; c < c1; ++c, ++k) {
                const int s = k % NS;
                if (k >= NS) u_bar_wait(empty_a + 8 * s, ((k / NS) - 1) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const bool new_group = true;  // every chunk carries its LUT block: warpgroups take alternate chunks
                const uint32_t bar = full_a + 8 * s;
                const uint32_t dst = stage_a + s * S::BYTES;
                u_bar_expect_elect(bar, GEO::IDS + (new_group ? S::LUT : 0) + ntc16 * GEO::BTILE);
                if (LAG > 0 && !S::SPLIT_AFREE && (int)k < NA)
                    u_bar_arrive_cnt_elect(bar, NMMA);  // no chunk k - NA yet: stands in for its MMA commits
                u_bulk_elect(dst, ids + ((size_t)x.tile * n_chunks + c) * GEO::IDS, GEO::IDS, bar);
                if (new_group)
                    u_bulk_elect(dst + GEO::IDS, lut + ((size_t)x.tile * n_groups + grp) * S::LUT, S::LUT, bar);
                u_bulk_elect(dst + GEO::IDS + S::LUT, bfrag + ((size_t)c * n_tiles + x.j0) * GEO::BTILE,
                             ntc16 * GEO::BTILE, bar);
                if (++gc == cpg) {
                    gc = 0;
                    ++grp;
                }
            }
        }
    } else if (warp >= um::MMA_WARP && warp < um::MMA_WARP + NMMA) {
        // ------------------------------------------------------------ MMA issuer (converged warp, elected lane)
        uint32_t k = 0, nu = 0;
        int seg = 0;
        UmSeq q = seq0;
        int u, c0, c1;
#ifdef UM_EXP_TIMING
        long long m_acc = 0, m_af = 0, m_iss = 0, m_t0 = clock64();
#endif
        // The CTA allocates all 512 TMEM columns (one CTA per SM), so the base is column 0 of lane 0:
        // literal bases let ptxas keep the MMA operands in uniform registers.
        const uint32_t tm_u = tmem, stage_u = stage_a;
        for (; q.next(W, u, c0, c1); ++nu) {
            const UmUnit x = um_unit(W, seg_first, u, seg, TPP);
            const uint32_t idesc = idesc_i8(((x.ntc + 1) & ~1) * 8);
            const int c0u = c0, c1u = c1;
#ifdef UM_EXP_TIMING
            const long long ma = clock64();
#endif
            // accumulator buffer nu % NACC: free once the epilogue of unit nu - NACC has read it
            const uint32_t abuf = nu % GEO::NACC, dacc = tm_u + abuf * (uint32_t)S::ACC1;
            if (nu >= (uint32_t)GEO::NACC) u_bar_wait(u_smem(&accempty_bar[abuf]), ((nu / GEO::NACC) - 1) & 1);
#ifdef UM_EXP_TIMING
            m_acc += clock64() - ma;
#endif
            for (int c = c0u; c < c1u; ++c, ++k) {
                const int s = k % NS, sa = k % NA;
                const uint32_t bbase = stage_u + s * S::BYTES + GEO::IDS + S::LUT;
                const uint32_t abase = tm_u + a_col0 + (uint32_t)(sa * S::CCOLS);
                // afull implies full: every expander waited for the chunk's data
#ifdef UM_EXP_TIMING
                const long long mw = clock64();
#endif
                u_bar_wait(afull_a + 8 * sa, (k / NA) & 1);
#ifdef UM_EXP_TIMING
                const long long mi = clock64();
                m_af += mi - mw;
#endif
                tc_fence_after();
                // one asm block per chunk (B tile: [tile8][kstep][khalf][8 rows][16 B])
#ifndef UM_EXP_NO_MMA
                {
                    // lane-0 broadcasts of the operands: ptxas then converts each to a uniform register
                    // once per chunk (68 instead of 141 instructions per 12 MMAs)
                    const uint64_t bd = smem_desc(bbase, 128, GEO::BTILE);
                    if constexpr (NMMA > 1) {  // this warp's plane: accumulator columns p * NT, A columns p * 8
                        const uint32_t pl = (uint32_t)(warp - um::MMA_WARP);
                        tc_mma_plane<GEO::KS>(__shfl_sync(0xffffffffu, dacc + pl * NT, 0),
                                              __shfl_sync(0xffffffffu, abase + pl * 8, 0), (uint32_t)S::ACOLS,
                                              __shfl_sync(0xffffffffu, bd, 0), __shfl_sync(0xffffffffu, idesc, 0),
                                              c == c0u ? 0u : 1u);
                    } else {
                        tc_mma_chunk<GEO::KS, P>(__shfl_sync(0xffffffffu, dacc, 0), (uint32_t)NT,
                                                 __shfl_sync(0xffffffffu, abase, 0), __shfl_sync(0xffffffffu, bd, 0),
                                                 __shfl_sync(0xffffffffu, idesc, 0), c == c0u ? 0u : 1u);
                    }
                }
#endif
                tc_commit_elect(empty_a + 8 * s);  // frees the smem stage (and with LAG == 0 the A stage)
                if (S::SPLIT_AFREE)
                    tc_commit_elect(afree_a + 8 * sa);  // A stage free for chunk k + NA
                else if (LAG > 0)
                    tc_commit_elect(full_a + 8 * ((k + NA) % NS));  // A stage free for chunk k + NA
                if (c == c1u - 1) tc_commit_elect(u_smem(&accfull_bar[abuf]));
#ifdef UM_EXP_TIMING
                m_iss += clock64() - mi;
#endif
            }
        }
#ifdef UM_EXP_TIMING
        if (blockIdx.x == 0 && lane == 0)
            printf("mma warp %d chunks %u: afull-wait %lld issue %lld accempty-wait %lld total %lld\n", warp, k, m_af,
                   m_iss, m_acc, clock64() - m_t0);
#endif
    } else {
        // ------------------------------------------------------------ expanders
        const int wg = warp >> 2;
        constexpr int KSW = GEO::KS / WPS;  // k-steps per warpgroup and chunk
        const int stream = wg / WPS, ks0 = (wg % WPS) * KSW;  // chunks k = stream (mod GS), k-steps ks0..
        const int quarter = warp & 3;     // TMEM lane quarter = rows
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        const int cb = wg * 8;            // epilogue: token columns cb + 32 i .. + 7, i < NCB
        // KG k-steps are looked up before any of their tcgen05.st (a run of independent lookups, then a
        // burst of stores)
        constexpr int KG = (KSW % UM_KGRP == 0) ? UM_KGRP : 1;
        uint32_t k = 0, nu = 0;           // chunks and units this CTA has started
        int seg = 0, seg_e = 0;           // monotone segment cursors: unit starts / epilogues
        UmSeq q = seq0;
        // Where a unit's epilogue runs (measured per geometry, tools/gemm_stage.py):
        //   EPI 2, decode (one column block, TMEM released right after the load) and double-buffered
        //     accumulators (the next unit's MMAs use the other buffer): after this warpgroup
        //     has expanded its first chunk of the next unit (or at once when it has none), so that
        //     expansion overlaps the MMA drain of the finished unit (MX gate|up 208 -> 203 us);
        //   EPI 1, prefill with 2 planes: after the next unit's prologue, before its first chunk (the
        //     next unit's operand prefetch is in flight sooner; QW down 272 -> 255 us);
        //   EPI 0, prefill with 3 planes: at the end of the unit (deferral measured 7% slower: the next
        //     unit's MMAs wait longer for TMEM).
        constexpr int EPI = (NCB == 1 || GEO::NACC > 1) ? 2 : (P == 2 ? 1 : 0);
        bool pending = false;
        int pu = 0, pc0 = 0, pc1 = 0;
        float prs = 0.0f;
#ifdef UM_EXP_TIMING
        long long t_wait = 0, t_exp = 0, t_epi = 0, t_begin = clock64();
        int n_ch = 0;
#endif
        // ---- epilogue of unit pu (the (nu-1)-th).  Warpgroup wg owns token columns cb + 32 i (i < NCB).
        // newer: the next unit's token operands were prefetched after the pending unit's (one newer
        // cp.async group, left in flight)
        auto epilogue = [&](bool newer) {
#ifdef UM_EXP_TIMING
            const long long te0 = clock64();
#endif
            pending = false;
            const int slot = (nu - 1) & 1;
            const uint32_t pb = (nu - 1) % GEO::NACC;      // the pending unit's accumulator buffer
            const uint32_t acc_base = tmem + lane_addr + pb * (uint32_t)S::ACC1;
            u_bar_wait(u_smem(&accfull_bar[pb]), ((nu - 1) / GEO::NACC) & 1);
            tc_fence_after();
            const UmUnit x = um_unit(W, seg_first, pu, seg_e, TPP);
            const int n = ((x.ntc + 1) & ~1) * 8;
            const bool split = pc0 > 0 || pc1 < n_chunks;  // unit shared with neighbouring CTAs (stream-K tail)
            int bf = 0, bl = 0;
            if (split) {
                const int64_t ustart = (int64_t)pu * n_chunks;
                bf = W.owner(ustart);
                bl = W.owner(ustart + n_chunks - 1);
            }
            auto load_acc = [&](int cbi, int32_t (&acc)[P][8]) {
#pragma unroll
                for (int p = 0; p < P; ++p)
                    tc_ld8(acc_base + (uint32_t)(p * NT + cbi), reinterpret_cast<uint32_t *>(acc[p]));
                tc_wait_ld();
            };
            // the last CTA of a split unit adds the others' partials (exact int32)
            auto add_partials = [&](int cbi, int32_t (&acc)[P][8]) {
                __threadfence();
                for (int b2 = bf; b2 <= bl; ++b2) {
                    if (b2 == cta) continue;
                    const int64_t fu = W.tstart(b2) / n_chunks;
                    const int32_t *src = part + (size_t)(2 * b2 + (pu != fu ? 1 : 0)) * GEO::PART_WORDS;
#pragma unroll
                    for (int p = 0; p < P; ++p)
#pragma unroll
                        for (int c2 = 0; c2 < 8; ++c2) acc[p][c2] += __ldcg(src + (p * NT + cbi + c2) * 128 + row);
                }
            };
            auto publish = [&](int cbi, const int32_t (&acc)[P][8]) {
                int32_t *mine = part + (size_t)(2 * cta + (pu != first_tail_unit ? 1 : 0)) * GEO::PART_WORDS;
#pragma unroll
                for (int p = 0; p < P; ++p)
#pragma unroll
                    for (int c2 = 0; c2 < 8; ++c2) mine[(p * NT + cbi + c2) * 128 + row] = acc[p][c2];
            };
            auto arrive_last = [&]() -> bool {  // every expander thread: true on the unit's last CTA
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"r"(um::EXP_WARPS * 32) : "memory");
                if (threadIdx.x == 0) {
                    const int last = atomicAdd(cnt + bf, 1) == bl - bf;
                    if (last) cnt[bf] = 0;  // ready for the next launch
                    last_sh = last;
                }
                asm volatile("bar.sync 1, %0;" ::"r"(um::EXP_WARPS * 32) : "memory");
                return last_sh != 0;
            };
            auto store = [&](int ib, const int32_t (&acc)[P][8]) {
                const int cbi = cb + 32 * ib;
                float *out = x.mat ? out1 : out0;
                // the block's 8 token scales and code sums (smem, two vector loads each); entries of
                // tokens outside [rb, re) are stale and their results are never stored
                const float4 sa4 = *reinterpret_cast<const float4 *>(&tok_sh[slot][warp][ib][0]);
                const float4 sb4 = *reinterpret_cast<const float4 *>(&tok_sh[slot][warp][ib][4]);
                const int4 qa = *reinterpret_cast<const int4 *>(&tok_sh[slot][warp][ib][8]);
                const int4 qb = *reinterpret_cast<const int4 *>(&tok_sh[slot][warp][ib][12]);
                const float tscale[8] = {sa4.x, sa4.y, sa4.z, sa4.w, sb4.x, sb4.y, sb4.z, sb4.w};
                const int32_t tqsum[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
                float vv[8];
#pragma unroll
                for (int c2 = 0; c2 < 8; ++c2) {  // branch-free, so the 8 conversion chains overlap
                    // exact integer digit sum (|.| < 2^39) in int64, one conversion: the same double
                    // as summing converted planes, at a third of the fp64-pipe work
                    int64_t s64 = (int64_t)acc[P - 1][c2];
#pragma unroll
                    for (int p = P - 2; p >= 0; --p) s64 = s64 * 128 + (int64_t)acc[p][c2];
                    s64 -= (int64_t)tqsum[c2] << (7 * P - 1);
                    const double sum = (double)s64;
                    vv[c2] = __fmul_rn((float)(sum * (double)prs), tscale[c2]);
                }
                const int64_t tok0 = x.j0 * 8 + cbi;
                float *o = out + tok0 * d_out + (int64_t)x.rt * 128 + row;
                if (tok0 >= x.rb && tok0 + 8 <= x.re) {
#pragma unroll
                    for (int c2 = 0; c2 < 8; ++c2) o[(int64_t)c2 * d_out] = vv[c2];
                } else {
#pragma unroll
                    for (int c2 = 0; c2 < 8; ++c2)
                        if (tok0 + c2 >= x.rb && tok0 + c2 < x.re) o[(int64_t)c2 * d_out] = vv[c2];
                }
            };
            if constexpr (NCB == 1) {
                // one block: keep it in registers and release TMEM at once, so the MMAs of the next
                // unit overlap this epilogue
                int32_t acc[P][8];
                if (cb < n) load_acc(cb, acc);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) u_bar_arrive(u_smem(&accempty_bar[pb]));
                bool finish = true;
                if (split) {
                    if (cb < n) publish(cb, acc);
                    finish = arrive_last();
                    if (finish && cb < n) add_partials(cb, acc);
                }
                if (newer)
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                else
                    asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                if (finish && cb < n) store(0, acc);
            } else {
                // several blocks: read TMEM block by block, release it after the last
                bool finish = true;
                if (split) {
#pragma unroll 1
                    for (int ib = 0; ib < NCB; ++ib) {
                        if (cb + 32 * ib >= n) break;
                        int32_t acc[P][8];
                        load_acc(cb + 32 * ib, acc);
                        publish(cb + 32 * ib, acc);
                    }
                    finish = arrive_last();
                }
                if (newer)
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                else
                    asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                if (finish) {
#pragma unroll 1
                    for (int ib = 0; ib < NCB; ++ib) {
                        if (cb + 32 * ib >= n) break;
                        int32_t acc[P][8];
                        load_acc(cb + 32 * ib, acc);
                        if (split) add_partials(cb + 32 * ib, acc);
                        store(ib, acc);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) u_bar_arrive(u_smem(&accempty_bar[pb]));
            }
#ifdef UM_EXP_TIMING
            t_epi += clock64() - te0;
#endif
        };
        for (;;) {
            int u = 0, c0 = 0, c1 = 0;
            const bool has = q.next(W, u, c0, c1);
            float rscale = 0.0f;
            int first = 0, n_own = 0;
            if (has) {
                const UmUnit x = um_unit(W, seg_first, u, seg, TPP);
                rscale = __ldg((x.mat ? rs1 : rs0) + x.tile * 128 + row);
                // per-token epilogue operands: async copies into this warp's smem slots now, so their
                // latency hides under the unit's chunks (lanes 0-7 scales, 8-15 row sums)
#pragma unroll
                for (int i = 0; i < NCB; ++i)
                    if (lane < 16 && cb + 32 * i < ((x.ntc + 1) & ~1) * 8) {
                        const int64_t tok = x.j0 * 8 + cb + 32 * i + (lane & 7);
                        if (tok >= x.rb && tok < x.re)
                            cp_async4(&tok_sh[nu & 1][warp][i][lane],
                                      lane < 8 ? (const void *)(scales + tok) : (const void *)(qsums + tok));
                    }
                asm volatile("cp.async.commit_group;" ::: "memory");
                // this stream's chunks of the unit: those whose CTA-wide index k + (c - c0) = stream (mod GS)
                first = (stream - (int)(k % GS) + GS) % GS;
                n_own = c1 - c0 > first ? (c1 - c0 - first + GS - 1) / GS : 0;
            }
            for (int i = 0; i <= n_own; ++i) {
                if constexpr (EPI == 1) {
                    if (i == 0 && pending) epilogue(has);
                }
                if (i < n_own) {
                    // ---- expand chunk kc (k-steps ks0 .. ks0 + KSW - 1 of it, see UmStage)
                    const uint32_t kc = k + (uint32_t)(first + i * GS);
                    const int s = kc % NS, sa = kc % NA;
#ifdef UM_EXP_TIMING
                    const long long tw0 = clock64();
#endif
                    u_bar_wait(full_a + 8 * s, (kc / NS) & 1);
                    tc_fence_after();
#ifdef UM_EXP_TIMING
                    const long long tw1 = clock64();
                    t_wait += tw1 - tw0;
                    ++n_ch;
#endif
                    const uint8_t *st = smem + (size_t)s * S::BYTES;
                    uint4 L[P];
                    {
                        const uint4 *lb = reinterpret_cast<const uint4 *>(st + GEO::IDS) + row * P;
#pragma unroll
                        for (int p = 0; p < P; ++p) L[p] = lb[p];
                    }
                    const uint32_t abase0 = tmem + lane_addr + a_col0 + (uint32_t)(sa * S::CCOLS);
#ifdef UM_EXP_NO_EXPAND
                    if (false)
#endif
#pragma unroll
                    for (int kg = 0; kg < KSW; kg += KG) {
                        uint32_t v[KG][P][8];
#pragma unroll
                        for (int h = 0; h < KG; ++h) {
                            const int ks = ks0 + kg + h;
                            const uint4 w = reinterpret_cast<const uint4 *>(st)[ks * 128 + row];
                            const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
                            uint32_t sel[8], xsel[8];
#pragma unroll
                            for (int qq = 0; qq < 4; ++qq) {
                                const uint32_t xx = wv[qq] ^ 0x88888888u;
                                sel[2 * qq] = wv[qq];
                                sel[2 * qq + 1] = hi16(wv[qq]);
                                xsel[2 * qq] = xx;
                                xsel[2 * qq + 1] = hi16(xx);
                            }
#pragma unroll
                            for (int p = 0; p < P; ++p)
#pragma unroll
                                for (int cc = 0; cc < 8; ++cc)
                                    v[h][p][cc] = NARROW ? u_prmt(L[p].x, L[p].y, sel[cc])
                                                         : u_merge(u_prmt(L[p].x, L[p].y, sel[cc]),
                                                                   u_prmt(L[p].z, L[p].w, xsel[cc]));
                        }
                        if (S::SPLIT_AFREE && kg == 0) {
                            // the first k-steps expand into registers before the A stage is known free:
                            // the MMAs of this stage's previous chunk (kc - NA) overlap their PRMT work.  Pin
                            // the values: the PRMTs must run before the wait (register-only code may
                            // otherwise sink past the volatile barrier probe)
#pragma unroll
                            for (int h = 0; h < KG; ++h)
#pragma unroll
                                for (int p = 0; p < P; ++p)
#pragma unroll
                                    for (int cc = 0; cc < 8; ++cc) asm volatile("" : "+r"(v[h][p][cc]));
                            u_bar_wait(afree_a + 8 * sa, ((kc / NA) & 1) ^ 1);  // first use of a stage passes
                            tc_fence_after();
                        }
#pragma unroll
                        for (int h = 0; h < KG; ++h)
#pragma unroll
                            for (int p = 0; p < P; ++p)
                                tc_st8(abase0 + (uint32_t)((ks0 + kg + h) * S::ACOLS + p * 8), v[h][p]);
                    }
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) u_bar_arrive(afull_a + 8 * sa);
#ifdef UM_EXP_TIMING
                    t_exp += clock64() - tw1;
#endif
                }
                if constexpr (EPI == 2) {
                    if (i == 0 && pending) epilogue(has);
                }
            }
            if (!has) break;
            k += (uint32_t)(c1 - c0);
            pending = true;
            pu = u;
            pc0 = c0;
            pc1 = c1;
            prs = rscale;
            ++nu;
            if constexpr (EPI == 0) epilogue(false);
        }
#ifdef UM_EXP_TIMING
        if (blockIdx.x == 0 && lane == 0)
            printf("warp %2d chunks %d: full-wait %lld expand %lld epilogue %lld (cycles, total %lld)\n", warp, n_ch,
                   t_wait, t_exp, t_epi, clock64() - t_begin);
#endif
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(um::TMEM_COLS)
                     : "memory");
    }
}

// codes (rows, K) row-major -> [chunk CK][tile8][kstep KS][khalf2][8 rows][16 B],
// the canonical K-major no-swizzle UMMA B layout per k-step; rows >= n are zero.
// Also zeroes the GEMM's split-unit counters (zero[0..n_zero)).
// perm (nullable): gather form, segment row r < *live reads token row perm[r]
// of src, rows past *live are zero, and the per-row scale and code sum are
// gathered from the token arrays (gather_rows + row_sums without their launches).
// rp.selected (route mode): the permutation is derived here from the top-k
// (route_perm.cuh, every CTA in shared memory); CTA 0 publishes offsets,
// counts, perm_token, perm_slot and inv.  blockDim.x == TB_THREADS.
constexpr int TB_THREADS = 256;

// RM: 0 no route mode, 1 route mode (permutation of <= RP_MAX_LOCAL local experts).
template <int CK, int RM>
__global__ void __launch_bounds__(TB_THREADS) to_umma_b_kernel(
    const int8_t *__restrict__ src, int64_t n, int64_t K, int64_t tiles, uint4 *__restrict__ dst,
    int32_t *__restrict__ zero, int n_zero, const int32_t *__restrict__ perm, const int32_t *__restrict__ live,
    const float *__restrict__ tscales, float *__restrict__ scales_out, const int32_t *__restrict__ tsum,
    int32_t *__restrict__ sums, RoutePerm rp) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    constexpr int PIECES = 16 * (CK / 32);  // 16-byte pieces per tile-chunk: k-steps x 2 khalf x 8 rows
    const int64_t total = (K / CK) * tiles * PIECES;
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < n_zero; i += blockDim.x) zero[i] = 0;
    int64_t nrow;
    if (RM != 0) {
        extern __shared__ int32_t tb_sm[];  // [RP_MAX_LOCAL + 1] offsets | [n_tok * k] permutation
        int32_t *s_off = tb_sm, *s_perm = tb_sm + RP_MAX_LOCAL + 1;
        const bool pub = blockIdx.x == 0;
        route_permute<TB_THREADS>(rp.selected, rp.n_tok, rp.k, rp.local_begin, rp.n_local, s_off, s_perm,
                                           pub ? rp.perm_slot : nullptr, pub ? rp.inv : nullptr);
        nrow = s_off[rp.n_local];
        perm = s_perm;
        if (pub) {
            for (int64_t x = threadIdx.x; x < nrow; x += blockDim.x) rp.perm_token[x] = s_perm[x];
            for (int e = threadIdx.x; e <= rp.n_local; e += blockDim.x) {
                rp.offsets[e] = s_off[e];
                if (e < rp.n_local) rp.counts[e] = s_off[e + 1] - s_off[e];
            }
        }
    } else {
        nrow = perm != nullptr ? (int64_t)*live : n;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (perm != nullptr)
        for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nrow; x += stride) {
            const int32_t t = perm[x];
            scales_out[x] = tscales[t];
            if (sums != nullptr) sums[x] = tsum[t];
        }
    if (RM != 0) {  // decode: a 16-byte piece per thread over many CTAs, whose permutation phases overlap
        for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += stride) {
            const int r = (int)(x & 7), kh = (int)((x >> 3) & 1), ks = (int)((x >> 4) % (CK / 32));
            const int64_t j = (x / PIECES) % tiles, c = (x / PIECES) / tiles;
            const int64_t row = j * 8 + r;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (row < nrow)
                v = *reinterpret_cast<const uint4 *>(src + (int64_t)perm[row] * K + c * CK + ks * 32 + kh * 16);
            dst[x] = v;
        }
        return;
    }
    // a thread per (row, chunk): the row's CK bytes in CK / 16 loads in flight (DS 43.8 -> 41.5 us,
    // QW 24.1 -> 23.2 us against a piece per thread); a warp's 32 rows store 4 tiles' full
    // 128-byte lines per piece
    constexpr int NP = CK / 16;
    const int64_t rows8 = tiles * 8, units = (total / PIECES) * 8;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units; u += stride) {
        const int64_t row = u % rows8, c = u / rows8;
        uint4 v[NP];
        if (row < nrow) {
            const int64_t sr = perm != nullptr ? (int64_t)perm[row] : row;
            const uint4 *s = reinterpret_cast<const uint4 *>(src + sr * K + c * CK);
#pragma unroll
            for (int p = 0; p < NP; ++p) v[p] = s[p];
        } else {
#pragma unroll
            for (int p = 0; p < NP; ++p) v[p] = make_uint4(0, 0, 0, 0);
        }
        uint4 *d = dst + (c * tiles + row / 8) * PIECES + (row & 7);
#pragma unroll
        for (int p = 0; p < NP; ++p) d[p * 8] = v[p];  // piece p = (k-step p / 2, khalf p % 2)
    }
}

// sums[r] = sum_j codes[r, j] (exact int32): the bias term of the unsigned digits.
__global__ void row_sums_kernel(const int8_t *__restrict__ codes, int64_t n, int64_t K, int32_t *__restrict__ sums) {
    griddep_wait();  // PDL: inputs of the previous kernel are visible after this
    const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= n) return;
    const int8_t *r = codes + row * K;
    int32_t acc = 0;
    if ((K & 15) == 0) {
        for (int64_t j = (threadIdx.x & 31) * 16; j < K; j += 512) {
            const int4 v = *reinterpret_cast<const int4 *>(r + j);
            const int w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = __dp4a(w4[u], 0x01010101, acc);
        }
    } else {
        for (int64_t j = threadIdx.x & 31; j < K; j += 32) acc += r[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sums[row] = acc;
}

// ---------------------------------------------------------------------------
// host side

bool umma_ok(int64_t d_in, int64_t d_out, int64_t g) { return d_in % 128 == 0 && g % 128 == 0 && d_out % 128 == 0; }

template <int P, class GEO>
size_t umma_smem() {
    return (size_t)UmStage<P, GEO>::NS * UmStage<P, GEO>::BYTES;
}

template <int CK>
cq_status to_umma_b(const int8_t *codes, int64_t n, int64_t K, int64_t tiles, int8_t *dst, int32_t *sums,
                    int32_t *zero, int n_zero, const UmmaIn &in, const float *tscales, const int32_t *live,
                    cudaStream_t st) {
    const int64_t total = (K / CK) * tiles * 16 * (CK / 32);
    if (total == 0) return CQ_OK;
    const size_t smem = in.route.on() ? sizeof(int32_t) * (RP_MAX_LOCAL + 1 + in.route.n_tok * in.route.k) : 0;
    auto kern = in.route.on() ? to_umma_b_kernel<CK, 1> : to_umma_b_kernel<CK, 0>;
    const int64_t ctas = in.route.on() ? std::min<int64_t>(ceil_div(total, TB_THREADS), 148 * 16)
                                       : std::min<int64_t>(ceil_div(total / (CK / 16), TB_THREADS), 148 * 8);
    launch_pdl(kern, (unsigned)ctas, TB_THREADS, smem, st, codes, n, K, tiles, reinterpret_cast<uint4 *>(dst), zero,
               n_zero, in.perm, live, tscales, in.scales_out, in.tok_sums, in.gathers() ? sums : nullptr, in.route);
    CQ_TRY(check_launch("to_umma_b"));
    if (sums == nullptr || in.gathers() || in.sums_ready) return CQ_OK;
    launch_pdl(row_sums_kernel, (unsigned)ceil_div(n, 8), 256, 0, st, codes, n, K, sums);
    return check_launch("row_sums");
}

// Persistent grid: one CTA per SM (CQ_UMMA_GRID overrides, for experiments).
int umma_grid() {
    static int sms = 0;
    if (sms == 0) {
        const char *env = getenv("CQ_UMMA_GRID");
        if (env != nullptr) sms = atoi(env);
        int dev = 0;
        cudaGetDevice(&dev);
        if (sms <= 0 && (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0))
            sms = 148;
    }
    return sms;
}

// B buffer: umma_b_tiles(rows) tiles x d_in bytes (an N=16 MMA may read one
// tile past the end), then the int32 row sums, then the split-unit scratch:
// 2 partial-accumulator slots per CTA and one counter per CTA (256-byte aligned).
int64_t umma_b_tiles(int64_t rows) { return ceil_div(rows, 8) + 2; }
static int64_t umma_sums_off(int64_t rows, int64_t d_in) { return umma_b_tiles(rows) * 8 * d_in; }
static int64_t umma_part_off(int64_t rows, int64_t d_in) {
    return umma_sums_off(rows, d_in) + ceil_div(rows * 4, 256) * 256;
}
static int64_t umma_prefill_min() {  // CQ_UMMA_PREFILL_MIN overrides (experiments)
    static int64_t v = -1;
    if (v < 0) {
        const char *e = getenv("CQ_UMMA_PREFILL_MIN");
        v = e ? atoll(e) : 32;
    }
    return v;
}
// 128-token passes pay once the decode geometry's 32-token passes would repeat the expansion of a
// segment (measured whole layers, bench.py --batch, this round: at 32 rows per segment prefill wins
// by 5-12% (MX b=128, QW b=512, PH b=256), at 48-64 by 16-37% (DS b=512, MX b=256, PH b=512, QW
// b=1024); at 16-24 rows decode wins by 9-26%), and when the decode geometry would have many chunk
// iterations per CTA (small matrices stay fill-bound on it: a 2048x1536 expert at 96 rows 34 vs
// 23 us).  `rows` is a bound: expert parallelism passes its slot capacity (~2x the routed rows).
static bool umma_prefill(int64_t rows, int64_t n_seg, int64_t d_in, int64_t d_out, int mats) {
    if (rows < 64 || rows < umma_prefill_min() * n_seg) return false;  // the prefill scratch needs 64 rows
    const int64_t decode_iters = ceil_div(rows / n_seg, 32) * n_seg * (d_out / 128) * mats * (d_in / 128);
    return decode_iters >= 32LL * umma_grid();
}
// The scratch is sized for the largest geometry `rows` can select.
static int64_t umma_part_words(int64_t rows) {
    return rows >= 64 ? (UmPrefill::PART_WORDS > UmDecode::PART_WORDS ? UmPrefill::PART_WORDS : UmDecode::PART_WORDS)
                       : UmDecode::PART_WORDS;
}
static int64_t umma_cnt_off(int64_t rows, int64_t d_in) {
    return umma_part_off(rows, d_in) + (int64_t)2 * umma_grid() * umma_part_words(rows) * 4;
}
int64_t umma_b_bytes(int64_t rows, int64_t d_in) {
    return umma_cnt_off(rows, d_in) + ceil_div((int64_t)umma_grid() * 4, 256) * 256;
}

template <int P, class GEO, bool NARROW = false>
cq_status launch_umma(const int8_t *bfrag, int64_t n_tiles, const float *scales, const int32_t *sums,
                      const int32_t *offsets, int64_t n_seg, int64_t seg_first, const cq_expert_site *a, float *out_a,
                      const cq_expert_site *b, float *out_b, int64_t d_in, int64_t d_out, int32_t *part,
                      int32_t *cnt, cudaStream_t st) {
    // the dynamic-smem opt-in is per device: set it on every launch (cheap next to the kernel)
    const size_t smem = umma_smem<P, GEO>();
    cudaFuncSetAttribute(lut_umma_kernel<P, GEO, NARROW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(lut_umma_kernel<P, GEO, NARROW>, umma_grid(), UmWarps<P>::THREADS, smem, st,
        bfrag, n_tiles, scales, sums, offsets, (int)n_seg, seg_first, a->tc_ids, a->tc_lut, a->tc_rowscale, out_a,
        b ? b->tc_ids : nullptr, b ? b->tc_lut : nullptr, b ? b->tc_rowscale : nullptr, out_b, b ? 2 : 1, (int)d_in,
        (int)d_out, (int)a->group_size, part, cnt);
    return check_launch("lut_umma");
}

template <class GEO>
cq_status lut_umma_geo(const int8_t *codes, int8_t *bbuf, const float *scales, const int32_t *offsets, int64_t n_seg,
                       int64_t seg_first, int64_t rows, const cq_expert_site *a, float *out_a,
                       const cq_expert_site *b, float *out_b, int64_t d_in, int64_t d_out, const UmmaIn &in,
                       cudaStream_t st) {
    // narrow lookup only when every matrix of the launch has ids < 8 (the data is that of UMMA128U)
    const bool narrow = a->tc_layout == CQ_TC_UMMA128U8 && (b == nullptr || b->tc_layout == CQ_TC_UMMA128U8);
    const int64_t tiles = umma_b_tiles(rows);
    int32_t *sums = reinterpret_cast<int32_t *>(bbuf + umma_sums_off(rows, d_in));
    int32_t *part = reinterpret_cast<int32_t *>(bbuf + umma_part_off(rows, d_in));
    int32_t *cnt = reinterpret_cast<int32_t *>(bbuf + umma_cnt_off(rows, d_in));
    if (!in.b_ready)  // else the re-quantizer wrote the tiles, the row sums and zeroed cnt (umma_b_out)
        CQ_TRY(to_umma_b<GEO::CK>(codes, rows, d_in, tiles, bbuf, sums, cnt, umma_grid(), in, scales, offsets + n_seg,
                                  st));
    if (in.gathers()) scales = in.scales_out;  // per segment row from here on
#define CQ_UMMA(P_, N_)                                                                                        \
    launch_umma<P_, GEO, N_>(bbuf, tiles, scales, sums, offsets, n_seg, seg_first, a, out_a, b, out_b, d_in, d_out, \
                             part, cnt, st)
    if (narrow) {
        if (a->tc_planes == 3) return CQ_UMMA(3, true);
        if (a->tc_planes == 2) return CQ_UMMA(2, true);
    } else {
        if (a->tc_planes == 3) return CQ_UMMA(3, false);
        if (a->tc_planes == 2) return CQ_UMMA(2, false);
    }
#undef CQ_UMMA
    set_error("tcgen05 path: planes must be 2 or 3");
    return CQ_ERR_CONFIG;
}

// The geometry of a grouped launch, as its chunk width: prefill (128-token passes, merged layout
// only) when segments are long.  CQ_UMMA_GEOMETRY=prefill|decode forces one (tests; prefill needs
// rows >= 64 for its scratch).
int umma_geo_ck(int64_t rows, int64_t n_seg, int64_t d_in, int64_t d_out, int mats, int planes) {
    const char *geo = getenv("CQ_UMMA_GEOMETRY");
    const bool force_pf = geo != nullptr && geo[0] == 'p' && rows >= 64;
    const bool force_dc = (geo != nullptr && geo[0] == 'd') || getenv("CQ_UMMA_NO_PREFILL") != nullptr;
    if (!force_dc && (force_pf || umma_prefill(rows, n_seg, d_in, d_out, mats)))
        return planes == 2 ? -UmPrefill2::CK : -UmPrefill::CK;  // negative: the prefill geometry
    return UmDecode::CK;
}

// Where a producer of B codes writes them so the grouped launch over (rows, d_in) skips its B
// build (UmmaIn::b_ready): the tile layout for chunk width ck, and the split-unit counters to zero.
UmmaBOut umma_b_out(int8_t *bbuf, int64_t rows, int64_t d_in, int ck) {
    UmmaBOut o;
    o.dst = bbuf;
    o.tiles = umma_b_tiles(rows);
    o.ck = ck;
    o.ck_shift = __builtin_ctz((unsigned)ck);
    o.zero = reinterpret_cast<int32_t *>(bbuf + umma_cnt_off(rows, d_in));
    o.n_zero = umma_grid();
    return o;
}

// Grouped tcgen05 LUT GEMM over segments.  `bbuf` holds umma_b_bytes(rows,
// d_in) bytes.  With b != nullptr, computes two matrices (gate -> out_a,
// up -> out_b) in one launch.
cq_status lut_umma_grouped(const int8_t *codes, int8_t *bbuf, const float *scales, const int32_t *offsets,
                           int64_t n_seg, int64_t seg_first, int64_t rows, const cq_expert_site *a, float *out_a,
                           const cq_expert_site *b, float *out_b, int64_t d_in, int64_t d_out, cudaStream_t st,
                           const UmmaIn &in) {
    if (rows == 0 || n_seg == 0) return CQ_OK;
    if (!umma_ok(d_in, d_out, a->group_size) || a->tc_lut == nullptr || (b && b->tc_lut == nullptr) ||
        !umma_merged(a->tc_layout)) {
        set_error("tcgen05 path: site not prepared or shape outside envelope");
        return CQ_ERR_UNSUPPORTED;
    }
    if (b && (b->tc_planes != a->tc_planes || b->group_size != a->group_size)) {
        set_error("tcgen05 path: paired matrices must share planes and group size");
        return CQ_ERR_CONFIG;
    }
    if (b && umma_family(b->tc_layout) != umma_family(a->tc_layout)) {
        set_error("tcgen05 path: paired matrices must share the layout");
        return CQ_ERR_CONFIG;
    }
    if (n_seg > um::MAX_SEG) {
        set_error("tcgen05 path: at most 512 segments (experts) per launch");
        return CQ_ERR_UNSUPPORTED;
    }
    if (umma_geo_ck(rows, n_seg, d_in, d_out, b ? 2 : 1, (int)a->tc_planes) < 0) {
        if (a->tc_planes == 2 && UmPrefill2::CK != UmPrefill::CK)
            return lut_umma_geo<UmPrefill2>(codes, bbuf, scales, offsets, n_seg, seg_first, rows, a, out_a, b, out_b,
                                            d_in, d_out, in, st);
        return lut_umma_geo<UmPrefill>(codes, bbuf, scales, offsets, n_seg, seg_first, rows, a, out_a, b, out_b,
                                       d_in, d_out, in, st);
    }
    return lut_umma_geo<UmDecode>(codes, bbuf, scales, offsets, n_seg, seg_first, rows, a, out_a, b, out_b, d_in,
                                  d_out, in, st);
}

// Where the merged layout's int32 row sums live in a B buffer (silu_quant writes them directly).
int32_t *umma_row_sums(int8_t *bbuf, int64_t rows, int64_t d_in) {
    return reinterpret_cast<int32_t *>(bbuf + umma_sums_off(rows, d_in));
}

}  // namespace cq
