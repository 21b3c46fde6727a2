/*
 * gp.c -- a SECOND, independent CPU oracle: the Gilbert-Peierls symbolic
 * factorization, column by column.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as oracle.c).  It shares no code with
 * oracle.c (fill2 per row) nor with the CUDA path; the tests
 * cross-check the two oracles, so a mistake in one of them would have to be
 * repeated by a different algorithm on a different traversal graph.
 *
 * "this approach determines the nonzero structures column by column ... For
 * column k, it traverses the graph L(:,0:k-1)^T in a Depth-First Search
 * manner.  The vertex that is reachable by the vertices in column k results
 * in a fill-in at column k".  Written out (lower-triangular solve
 * L(:,0:k-1) x = A(:,k) with unit diagonal):
 *   struct(x) = every vertex reachable from struct(A(:,k)) in the directed
 *               graph with an edge j -> i for each L(i,j) != 0 (i > j),
 *               leaving only vertices j < k (whose columns are known);
 *   U(0:k, k)    = struct(x) restricted to rows <= k, plus the pivot (k, k);
 *   L(k+1:n, k)  = struct(x) restricted to rows > k.
 * The diagonal is implicit: A(k,k) is ignored, U(k,k) always present.
 * Outputs are column-compressed L (strictly lower) and U (upper incl.
 * diagonal), rows ascending within each column.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int cmp32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/*
 * oracle_gp(n, rowptr, colidx, ...):
 *   A given by rows (CSR); its columns are formed here (plain transpose).
 *   *Lp int64[n+1], *Li int32[...]: L by columns;  *Up, *Ui: U by columns.
 * Returns 0, -1 on allocation failure, -2 on bad arguments.  Caller frees the
 * four arrays with oracle_free.
 */
int oracle_gp(int64_t n, const int64_t *rowptr, const int32_t *colidx,
              int64_t **Lp_out, int32_t **Li_out, int64_t **Up_out, int32_t **Ui_out) {
    if (n <= 0 || !rowptr || !colidx) return -2;
    const int64_t nnz = rowptr[n];
    /* columns of A: cp / cr */
    int64_t *cp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int32_t *cr = (int32_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
    int64_t *at = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    /* L and U columns, grown as they are produced */
    int64_t *Lp = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    int64_t *Up = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    int64_t lcap = 1024, ucap = 1024, ln = 0, un = 0;
    int32_t *Li = (int32_t *)malloc((size_t)lcap * sizeof(int32_t));
    int32_t *Ui = (int32_t *)malloc((size_t)ucap * sizeof(int32_t));
    int32_t *mark = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *stack = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *xs = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int rc = 0;
    if (!cp || !cr || !at || !Lp || !Up || !Li || !Ui || !mark || !stack || !xs) { rc = -1; goto fail; }
    for (int64_t e = 0; e < nnz; ++e) {
        if (colidx[e] < 0 || colidx[e] >= n) { rc = -2; goto fail; }
        cp[colidx[e] + 1] += 1;
    }
    for (int64_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
    memcpy(at, cp, (size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) cr[at[colidx[e]]++] = (int32_t)i;
    for (int64_t v = 0; v < n; ++v) mark[v] = -1;
    Lp[0] = Up[0] = 0;
    for (int64_t k = 0; k < n; ++k) {
        /* reach of struct(A(:,k)) through the columns of L known so far */
        int64_t nx = 0, top = 0;
        for (int64_t e = cp[k]; e < cp[k + 1]; ++e) {
            const int32_t i = cr[e];
            if (i == k || mark[i] == k) continue;      /* the implicit diagonal */
            mark[i] = (int32_t)k;
            xs[nx++] = i;
            if (i < k) stack[top++] = i;               /* column i of L is known */
        }
        while (top > 0) {                              /* DFS */
            const int32_t j = stack[--top];
            for (int64_t e = Lp[j]; e < Lp[j + 1]; ++e) {
                const int32_t i = Li[e];               /* edge j -> i, L(i,j) != 0 */
                if (i == k || mark[i] == k) continue;
                mark[i] = (int32_t)k;
                xs[nx++] = i;
                if (i < k) stack[top++] = i;
            }
        }
        qsort(xs, (size_t)nx, sizeof(int32_t), cmp32);
        /* U(0:k, k): rows < k, then the pivot; L(k+1:n, k): rows > k */
        int64_t nu = 0;
        while (nu < nx && xs[nu] < k) ++nu;
        if (un + nu + 1 > ucap || ln + (nx - nu) > lcap) {
            while (un + nu + 1 > ucap) ucap *= 2;
            while (ln + (nx - nu) > lcap) lcap *= 2;
            int32_t *a = (int32_t *)realloc(Ui, (size_t)ucap * sizeof(int32_t));
            if (!a) { rc = -1; goto fail; }
            Ui = a;
            int32_t *b = (int32_t *)realloc(Li, (size_t)lcap * sizeof(int32_t));
            if (!b) { rc = -1; goto fail; }
            Li = b;
        }
        memcpy(Ui + un, xs, (size_t)nu * sizeof(int32_t));
        un += nu;
        Ui[un++] = (int32_t)k;
        memcpy(Li + ln, xs + nu, (size_t)(nx - nu) * sizeof(int32_t));
        ln += nx - nu;
        Up[k + 1] = un;
        Lp[k + 1] = ln;
    }
    *Lp_out = Lp; *Li_out = Li; *Up_out = Up; *Ui_out = Ui;
    free(cp); free(cr); free(at); free(mark); free(stack); free(xs);
    return 0;
fail:
    free(cp); free(cr); free(at); free(Lp); free(Up); free(Li); free(Ui);
    free(mark); free(stack); free(xs);
    return rc;
}
