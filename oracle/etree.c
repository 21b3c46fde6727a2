/*
 * etree.c -- the symmetric-pattern comparator: for a
 * structurally symmetric A, struct(L) is the Cholesky factor's structure,
 * which the elimination tree gives directly ("for symmetric matrices, the
 * elimination tree ... is used to compute the structure").
 *
 * TEST INFRASTRUCTURE ONLY (same rules as oracle.c).  It shares no code with
 * oracle.c (fill2 per row), gp.c (Gilbert-Peierls by columns) or the CUDA
 * path.
 *
 * Written out:
 *   etree (Liu): parent(k) = min { i > k : L(i,k) != 0 }, built row by row:
 *     for each A(i,k) != 0 with k < i, climb from k through the current
 *     ancestors (path-compressed) to its root r != i and set parent(r) = i;
 *   row subtree: L(i,:) = union over A(i,k) != 0, k < i, of the tree path
 *     k, parent(k), ... up to (excluding) i.
 * U = L^T plus the diagonal for a symmetric pattern (formed by the caller).
 * The pattern must be structurally symmetric (checked: returns -3 if not).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int cmp32e(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

static int has_entry(const int64_t *rowptr, const int32_t *colidx, int64_t i, int32_t j) {
    int64_t a = rowptr[i], b = rowptr[i + 1];
    while (a < b) {
        int64_t m = (a + b) / 2;
        if (colidx[m] == j) return 1;
        if (colidx[m] < j) a = m + 1; else b = m;
    }
    return 0;
}

typedef struct {
    int64_t n;
    const int64_t *rowptr;
    const int32_t *colidx;
    const int32_t *parent;
    int64_t r0, r1;          /* rows of this thread */
    int64_t *cnt;            /* [n] row counts (pass 1) */
    const int64_t *Lp;       /* row pointers (pass 2) */
    int32_t *Li;
    int pass;
} ejob_t;

static void *erows(void *p) {
    ejob_t *J = (ejob_t *)p;
    int32_t *mark = malloc((size_t)J->n * sizeof(int32_t));
    if (!mark) return (void *)1;
    for (int64_t v = 0; v < J->n; ++v) mark[v] = -1;
    for (int64_t i = J->r0; i < J->r1; ++i) {
        int64_t c = 0, o = J->pass == 2 ? J->Lp[i] : 0;
        mark[i] = (int32_t)i;
        for (int64_t e = J->rowptr[i]; e < J->rowptr[i + 1]; ++e) {
            int32_t k = J->colidx[e];
            if (k >= i) continue;
            while (mark[k] != i) {     /* the tree path k -> i */
                mark[k] = (int32_t)i;
                if (J->pass == 2) J->Li[o + c] = k;
                ++c;
                k = J->parent[k];
            }
        }
        if (J->pass == 1) J->cnt[i] = c;
        else qsort(J->Li + o, (size_t)c, sizeof(int32_t), cmp32e);
    }
    free(mark);
    return NULL;
}

/*
 * oracle_etree_rows(n, rowptr, colidx, nthreads, &Lp, &Li): L by rows
 * (strictly lower, ascending) of a structurally symmetric pattern.
 * Returns 0; -1 allocation failure; -2 bad arguments; -3 not symmetric.
 * The caller frees Lp / Li with oracle_free.
 */
int oracle_etree_rows(int64_t n, const int64_t *rowptr, const int32_t *colidx, int nthreads,
                      int64_t **Lp_out, int32_t **Li_out) {
    if (n < 0 || !rowptr || !colidx || !Lp_out || !Li_out) return -2;
    if (nthreads < 1) nthreads = 1;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (colidx[e] != i && !has_entry(rowptr, colidx, colidx[e], (int32_t)i)) return -3;
    int32_t *parent = malloc((size_t)(n ? n : 1) * sizeof(int32_t));
    int32_t *anc = malloc((size_t)(n ? n : 1) * sizeof(int32_t));
    int64_t *cnt = calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *Lp = malloc((size_t)(n + 1) * sizeof(int64_t));
    pthread_t *th = malloc((size_t)nthreads * sizeof(pthread_t));
    ejob_t *jobs = malloc((size_t)nthreads * sizeof(ejob_t));
    int rc = 0;
    if (!parent || !anc || !cnt || !Lp || !th || !jobs) { rc = -1; goto done; }
    for (int64_t i = 0; i < n; ++i) {
        parent[i] = -1;
        anc[i] = -1;
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
            int32_t r = colidx[e];
            if (r >= i) continue;
            while (anc[r] != -1 && anc[r] != i) {   /* climb, compressing to i */
                int32_t t = anc[r];
                anc[r] = (int32_t)i;
                r = t;
            }
            if (anc[r] == -1) { anc[r] = (int32_t)i; parent[r] = (int32_t)i; }
        }
    }
    for (int pass = 1; pass <= 2; ++pass) {
        int32_t *Li = NULL;
        if (pass == 2) {
            Lp[0] = 0;
            for (int64_t i = 0; i < n; ++i) Lp[i + 1] = Lp[i] + cnt[i];
            Li = malloc((size_t)(Lp[n] ? Lp[n] : 1) * sizeof(int32_t));
            if (!Li) { rc = -1; goto done; }
            *Li_out = Li;
        }
        for (int t = 0; t < nthreads; ++t) {
            jobs[t] = (ejob_t){n, rowptr, colidx, parent, n * t / nthreads, n * (t + 1) / nthreads,
                               cnt, Lp, Li, pass};
            if (pthread_create(&th[t], NULL, erows, &jobs[t])) { rc = -1; nthreads = t; break; }
        }
        for (int t = 0; t < nthreads; ++t) {
            void *res = NULL;
            pthread_join(th[t], &res);
            if (res) rc = -1;
        }
        if (rc) {
            if (pass == 2) { free(Li); *Li_out = NULL; }
            goto done;
        }
    }
    *Lp_out = Lp;
    Lp = NULL;
done:
    free(parent); free(anc); free(cnt); free(Lp); free(th); free(jobs);
    return rc;
}
