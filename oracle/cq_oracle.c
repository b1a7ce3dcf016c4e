/* CPU oracle, C restatement — TEST INFRASTRUCTURE ONLY.
 *
 * Restates the reference's native kernels (reference tree
 * pkg/src/codequant/kernels/_core.pyx) so full-size parity checks finish in
 * seconds.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load
 * this library; the product package never does.
 *
 * Build: oracle/Makefile  (gcc -O3 -ffp-contract=off: one rounding per
 * multiply and per add, exactly like the reference's setup.py:12).
 *
 *   cqo_lut_gemm_f32      <- _core.pyx:41-151 (lut_gemm_f32): per output row a
 *                            (group, id, code) product table, j ascending.
 *   cqo_reference_gemm_f32<- _core.pyx:154-211: centroid * float(code) per
 *                            element, same order (bitwise equal to the above).
 *   cqo_matmul_f32        <- _core.pyx:27-38: k ascending, no FMA.
 *   cqo_quantize_f32      <- quant.py:89-100 for float32 input.
 * Rows are split across POSIX threads; every output element has one writer,
 * so results do not depend on the thread count (kernels/compiled.py:1-6).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const int8_t *codes;
    const float *scales;
    const uint8_t *ids;
    const float *cent;
    int64_t n, d_in, d_out, g, row0, row1;
    float *out;
    int use_table;
} gemm_job;

static void *gemm_worker(void *arg) {
    gemm_job *jb = (gemm_job *)arg;
    const int64_t d_in = jb->d_in, g = jb->g, n = jb->n;
    const int64_t n_groups = d_in / g;
    const int64_t row_bytes = (d_in + 1) / 2;
    float *table = (float *)malloc((size_t)(n_groups > 0 ? n_groups : 1) * 256 * sizeof(float));
    uint8_t *ids_row = (uint8_t *)malloc((size_t)(d_in > 0 ? d_in : 1));
    for (int64_t i = jb->row0; i < jb->row1; ++i) {
        const uint8_t *src = jb->ids + i * row_bytes;
        for (int64_t j = 0; j < d_in; ++j)
            ids_row[j] = (j & 1) ? (uint8_t)(src[j >> 1] >> 4) : (uint8_t)(src[j >> 1] & 15);
        const float *crow = jb->cent + i * n_groups * 16;
        if (jb->use_table) {
            for (int64_t grp = 0; grp < n_groups; ++grp)
                for (int c = 0; c < 16; ++c)
                    for (int code = 0; code < 16; ++code)
                        table[grp * 256 + c * 16 + code] = crow[grp * 16 + c] * (float)(code - 8);
        }
        for (int64_t t = 0; t < n; ++t) {
            const int8_t *q = jb->codes + t * d_in;
            float acc = 0.0f;
            if (jb->use_table) {
                for (int64_t j = 0; j < d_in; ++j)
                    acc = acc + table[(j / g) * 256 + ids_row[j] * 16 + (q[j] + 8)];
            } else {
                for (int64_t j = 0; j < d_in; ++j)
                    acc = acc + crow[(j / g) * 16 + ids_row[j]] * (float)q[j];
            }
            jb->out[t * jb->d_out + i] = jb->scales[t] * acc;
        }
    }
    free(table);
    free(ids_row);
    return NULL;
}

static int run_gemm(const int8_t *codes, const float *scales, const uint8_t *ids,
                    const float *cent, int64_t n, int64_t d_in, int64_t d_out,
                    int64_t g, float *out, int threads, int use_table) {
    if (g < 1 || d_in % g) return 1;
    if (threads < 1) threads = 1;
    if (threads > d_out) threads = (int)(d_out > 0 ? d_out : 1);
    gemm_job jobs[256];
    pthread_t tids[256];
    if (threads > 256) threads = 256;
    int64_t per = (d_out + threads - 1) / threads;
    int launched = 0;
    for (int w = 0; w < threads; ++w) {
        int64_t r0 = w * per, r1 = r0 + per;
        if (r1 > d_out) r1 = d_out;
        if (r0 >= r1) break;
        jobs[w] = (gemm_job){codes, scales, ids, cent, n, d_in, d_out, g, r0, r1, out, use_table};
        if (threads == 1) { gemm_worker(&jobs[w]); continue; }
        pthread_create(&tids[w], NULL, gemm_worker, &jobs[w]);
        ++launched;
    }
    for (int w = 0; w < launched; ++w) pthread_join(tids[w], NULL);
    return 0;
}

int cqo_lut_gemm_f32(const int8_t *codes, const float *scales, const uint8_t *ids,
                     const float *cent, int64_t n, int64_t d_in, int64_t d_out,
                     int64_t g, float *out, int threads) {
    return run_gemm(codes, scales, ids, cent, n, d_in, d_out, g, out, threads, 1);
}

int cqo_reference_gemm_f32(const int8_t *codes, const float *scales, const uint8_t *ids,
                           const float *cent, int64_t n, int64_t d_in, int64_t d_out,
                           int64_t g, float *out, int threads) {
    return run_gemm(codes, scales, ids, cent, n, d_in, d_out, g, out, threads, 0);
}

typedef struct {
    const float *a, *b;
    float *out;
    int64_t k, n, row0, row1;
} mm_job;

static void *mm_worker(void *arg) {
    mm_job *jb = (mm_job *)arg;
    for (int64_t i = jb->row0; i < jb->row1; ++i) {
        float *o = jb->out + i * jb->n;
        for (int64_t j = 0; j < jb->n; ++j) o[j] = 0.0f;
        for (int64_t kk = 0; kk < jb->k; ++kk) {
            const float aik = jb->a[i * jb->k + kk];
            const float *brow = jb->b + kk * jb->n;
            for (int64_t j = 0; j < jb->n; ++j) o[j] = o[j] + aik * brow[j];
        }
    }
    return NULL;
}

/* _core.pyx:27-38: i-k-j, every out[i][j] an ordered chain over k (the j loop
 * vectorizes across independent outputs; -ffp-contract=off keeps mul and add
 * separate).  Rows split over `threads` POSIX threads (one writer per row). */
void cqo_matmul_f32(const float *a, const float *b, float *out, int64_t m, int64_t k, int64_t n, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads > m) threads = (int)(m > 0 ? m : 1);
    mm_job jobs[256];
    pthread_t tids[256];
    const int64_t per = (m + threads - 1) / threads;
    int launched = 0;
    for (int w = 0; w < threads; ++w) {
        int64_t r0 = w * per, r1 = r0 + per;
        if (r1 > m) r1 = m;
        if (r0 >= r1) break;
        jobs[w] = (mm_job){a, b, out, k, n, r0, r1};
        if (threads == 1) { mm_worker(&jobs[w]); continue; }
        pthread_create(&tids[w], NULL, mm_worker, &jobs[w]);
        ++launched;
    }
    for (int w = 0; w < launched; ++w) pthread_join(tids[w], NULL);
}

/* quant.py:89-100 for float32 rows: scale = snap(max|x| / 7), 1 for a zero
 * row; code = clip(round-half-away(x / scale), -8, 7). */
void cqo_quantize_f32(const float *x, int64_t n, int64_t d, int8_t *codes, float *scales) {
    for (int64_t t = 0; t < n; ++t) {
        const float *row = x + t * d;
        float mx = 0.0f;
        for (int64_t j = 0; j < d; ++j) {
            float a = fabsf(row[j]);
            if (a > mx) mx = a;
        }
        float s = mx / 7.0f;
        uint32_t bits;
        memcpy(&bits, &s, 4);
        bits &= ~7u;
        memcpy(&s, &bits, 4);
        if (mx == 0.0f) s = 1.0f;
        scales[t] = s;
        for (int64_t j = 0; j < d; ++j) {
            float r = roundf(row[j] / s);
            if (r > 7.0f) r = 7.0f;
            if (r < -8.0f) r = -8.0f;
            codes[t * d + j] = (int8_t)r;
        }
    }
}
