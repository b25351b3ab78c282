/*
 * ORACLE — test infrastructure only, NOT the product.
 *
 * Plain-C CPU restatement of the reference's CSR-dtANS decode and fused SpMV
 * (the Python package at /root/reference/pkg/src/csrdtans).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 *
 * Pinned: tests/test_oracle.py checks it against golden fixtures produced by
 * running the reference itself (tests/golden/make_golden.py): decode ==
 * the reference's decode_matrix, spmv bitwise == the reference's spmv.
 *
 * Semantics restated (production geometry W=2^32, K=4096, l=8, o=3, f=2):
 *   - per-slice 32-lane lockstep word consumption:
 *       container.py:370-521 (_decode_slice_range), event order
 *       container.py:254-280 (_event_grid), consume() container.py:406-413
 *   - unpack of 3 words into 8 12-bit slots: codec.py:148-162 and
 *       container.py:437-446 (slot 0 = low 12 bits of the LAST word)
 *   - escape payloads, low word first: container.py:459-470
 *   - mixed-radix accumulate (decremented radix d*bm1+d+dig) and the
 *       r >= W extract / load check: codec.py:127-145, container.py:478-494
 *   - unconditional load of word 2: container.py:495-497
 *   - consumption check: container.py:499-500 (CorruptStream)
 *   - per-row delta prefix sum, value bit reinterpretation:
 *       container.py:502-521
 *   - accumulation acc=+0.0; acc=fl(acc+fl(v*x)); out=fl(acc+y):
 *       container.py:534-551, sparse.py:330-353
 * Build with -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define SLICE 32
#define K_SLOTS 4096
#define L_SYM 8

typedef struct {
    int64_t rows, cols;
    int32_t precision; /* 4 or 8 */
    /* per-domain slot tables: domain 0 = column deltas, 1 = value bits */
    const uint64_t *sym[2];
    const uint8_t *digit[2];
    const uint8_t *bm1[2];
    const uint8_t *esc[2];
    const uint32_t *row_symbols;
    const uint64_t *directory; /* nslices + 1 */
    const uint32_t *stream;
    int64_t nwords;
} oracle_container;

enum { ORACLE_OK = 0, ORACLE_CORRUPT = 1, ORACLE_BADCOL = 2, ORACLE_NOMEM = 3 };

typedef unsigned __int128 u128;

/* Decode one slice.  For each lane writes symbols (padded grid, 8*nseg per
 * lane) into sym_out at lane offsets off[lane]. */
static int decode_slice(const oracle_container *c, int64_t s, uint64_t *sym_out,
                        const int64_t *off)
{
    int64_t row0 = s * SLICE;
    int nl = (int)((c->rows - row0) < SLICE ? (c->rows - row0) : SLICE);
    uint64_t cur = c->directory[s];
    uint64_t end = c->directory[s + 1];
    int64_t n[SLICE], nseg[SLICE];
    uint64_t w[3][SLICE];
    u128 d[SLICE], r[SLICE];
    int64_t max_nseg = 0;
    const int pw[2] = {1, c->precision / 4}; /* payload words per domain */

#define FETCH(dst)                                            \
    do {                                                      \
        if (cur >= (uint64_t)c->nwords) return ORACLE_CORRUPT; \
        (dst) = c->stream[cur++];                             \
    } while (0)

    for (int i = 0; i < nl; i++) {
        n[i] = c->row_symbols[row0 + i];
        nseg[i] = (n[i] + L_SYM - 1) / L_SYM;
        if (nseg[i] > max_nseg) max_nseg = nseg[i];
        d[i] = 0;
        r[i] = 1;
        w[0][i] = w[1][i] = w[2][i] = 0;
    }
    /* init events c = 0, 1, 2: every lane with n > 0 takes one word */
    for (int cp = 0; cp < 3; cp++)
        for (int i = 0; i < nl; i++)
            if (nseg[i] > 0) FETCH(w[cp][i]);

    for (int64_t j = 0; j < max_nseg; j++) {
        uint32_t slots[SLICE][L_SYM];
        uint64_t sym[SLICE][L_SYM];
        for (int i = 0; i < nl; i++) {
            if (j >= nseg[i]) continue;
            u128 num = ((u128)w[0][i] << 64) | ((u128)w[1][i] << 32) | (u128)w[2][i];
            for (int k = 0; k < L_SYM; k++) {
                slots[i][k] = (uint32_t)((num >> (12 * k)) & 0xFFF);
                sym[i][k] = c->sym[k & 1][slots[i][k]];
            }
        }
        /* payload event: lanes in order, escapes in k order, low word first */
        for (int i = 0; i < nl; i++) {
            if (j >= nseg[i]) continue;
            for (int k = 0; k < L_SYM; k++) {
                int dom = k & 1;
                if (!c->esc[dom][slots[i][k]]) continue;
                uint64_t val = 0;
                for (int q = 0; q < pw[dom]; q++) {
                    uint64_t wd;
                    FETCH(wd);
                    val |= wd << (32 * q);
                }
                sym[i][k] = val;
            }
            for (int k = 0; k < L_SYM; k++) sym_out[off[i] + j * L_SYM + k] = sym[i][k];
        }
        /* two conditional checks (groups {0..3}, {4..7}) */
        for (int g = 0; g < 2; g++) {
            for (int i = 0; i < nl; i++) {
                if (j + 1 >= nseg[i]) continue; /* last segment: no checks */
                for (int k = 4 * g; k < 4 * g + 4; k++) {
                    int dom = k & 1;
                    u128 bm1 = c->bm1[dom][slots[i][k]];
                    u128 dig = c->digit[dom][slots[i][k]];
                    d[i] = d[i] * bm1 + d[i] + dig;
                    r[i] = r[i] * bm1 + r[i];
                }
                if (r[i] >= ((u128)1 << 32)) {
                    w[g][i] = (uint64_t)(d[i] & 0xFFFFFFFFu);
                    d[i] >>= 32;
                    r[i] >>= 32;
                } else {
                    FETCH(w[g][i]);
                }
            }
        }
        /* unconditional load of word 2 */
        for (int i = 0; i < nl; i++)
            if (j + 1 < nseg[i]) FETCH(w[2][i]);
    }
#undef FETCH
    if (cur != end) return ORACLE_CORRUPT;
    return ORACLE_OK;
}

/* Per-slice scratch: padded symbol grid. */
typedef struct {
    uint64_t *buf;
    int64_t cap;
} scratch;

static int slice_grid(const oracle_container *c, int64_t s, scratch *sc,
                      int64_t off[SLICE], int *nl_out)
{
    int64_t row0 = s * SLICE;
    int nl = (int)((c->rows - row0) < SLICE ? (c->rows - row0) : SLICE);
    int64_t tot = 0;
    for (int i = 0; i < nl; i++) {
        off[i] = tot;
        tot += (((int64_t)c->row_symbols[row0 + i] + L_SYM - 1) / L_SYM) * L_SYM;
    }
    if (tot > sc->cap) {
        free(sc->buf);
        sc->cap = tot * 2;
        sc->buf = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)sc->cap);
        if (!sc->buf) return ORACLE_NOMEM;
    }
    *nl_out = nl;
    return decode_slice(c, s, sc->buf, off);
}

/* Full decode: row_nnz[rows], cols[nnz], valbits[nnz] (CSR order). */
int oracle_decode(const oracle_container *c, int64_t *row_nnz, int64_t *cols,
                  uint64_t *valbits)
{
    int64_t nslices = (c->rows + SLICE - 1) / SLICE;
    scratch sc = {NULL, 0};
    int64_t pos = 0;
    for (int64_t s = 0; s < nslices; s++) {
        int64_t off[SLICE];
        int nl;
        int rc = slice_grid(c, s, &sc, off, &nl);
        if (rc) { free(sc.buf); return rc; }
        for (int i = 0; i < nl; i++) {
            int64_t n = c->row_symbols[s * SLICE + i];
            int64_t col = 0;
            row_nnz[s * SLICE + i] = n / 2;
            for (int64_t q = 0; q + 1 < n; q += 2) {
                col += (int64_t)sc.buf[off[i] + q];
                cols[pos] = col;
                valbits[pos] = sc.buf[off[i] + q + 1];
                pos++;
            }
        }
    }
    free(sc.buf);
    return ORACLE_OK;
}

typedef struct {
    const oracle_container *c;
    const void *x, *y;
    void *out;
    int64_t s_lo, s_hi;
    int rc;
} job;

static void *spmv_range(void *arg)
{
    job *jb = (job *)arg;
    const oracle_container *c = jb->c;
    scratch sc = {NULL, 0};
    jb->rc = ORACLE_OK;
    for (int64_t s = jb->s_lo; s < jb->s_hi; s++) {
        int64_t off[SLICE];
        int nl;
        int rc = slice_grid(c, s, &sc, off, &nl);
        if (rc) { jb->rc = rc; break; }
        for (int i = 0; i < nl; i++) {
            int64_t row = s * SLICE + i;
            int64_t n = c->row_symbols[row];
            int64_t col = 0;
            if (c->precision == 8) {
                const double *x = (const double *)jb->x;
                double acc = 0.0;
                for (int64_t q = 0; q + 1 < n; q += 2) {
                    col += (int64_t)sc.buf[off[i] + q];
                    if (col < 0 || col >= c->cols) { jb->rc = ORACLE_BADCOL; goto done; }
                    double v;
                    memcpy(&v, &sc.buf[off[i] + q + 1], 8);
                    double p = v * x[col];
                    acc = acc + p;
                }
                ((double *)jb->out)[row] = acc + ((const double *)jb->y)[row];
            } else {
                const float *x = (const float *)jb->x;
                float acc = 0.0f;
                for (int64_t q = 0; q + 1 < n; q += 2) {
                    col += (int64_t)sc.buf[off[i] + q];
                    if (col < 0 || col >= c->cols) { jb->rc = ORACLE_BADCOL; goto done; }
                    uint32_t bits = (uint32_t)sc.buf[off[i] + q + 1];
                    float v;
                    memcpy(&v, &bits, 4);
                    float p = v * x[col];
                    acc = acc + p;
                }
                ((float *)jb->out)[row] = acc + ((const float *)jb->y)[row];
            }
        }
    }
done:
    free(sc.buf);
    return NULL;
}

/* y' = A x + y.  threads > 1 splits contiguous slice ranges (the reference's
 * ThreadPoolExecutor split, container.py:583-595); results do not depend on
 * the split. */
int oracle_spmv(const oracle_container *c, const void *x, const void *y, void *out,
                int threads)
{
    int64_t nslices = (c->rows + SLICE - 1) / SLICE;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads == 1 || nslices <= 1) {
        job jb = {c, x, y, out, 0, nslices, 0};
        spmv_range(&jb);
        return jb.rc;
    }
    pthread_t tid[256];
    job jobs[256];
    int64_t chunk = (nslices + threads - 1) / threads;
    int nt = 0;
    for (int64_t lo = 0; lo < nslices; lo += chunk) {
        int64_t hi = lo + chunk < nslices ? lo + chunk : nslices;
        jobs[nt] = (job){c, x, y, out, lo, hi, 0};
        pthread_create(&tid[nt], NULL, spmv_range, &jobs[nt]);
        nt++;
    }
    int rc = ORACLE_OK;
    for (int t = 0; t < nt; t++) {
        pthread_join(tid[t], NULL);
        if (jobs[t].rc && !rc) rc = jobs[t].rc;
    }
    return rc;
}
