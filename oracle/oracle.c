/*
 * oracle.c -- plain, slow, obviously-correct CPU symbolic LU factorization.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  It shares no code, header, table or helper with the CUDA path
 * (paper_2007_00840_b200/csrc); neither side includes the other.
 *
 * What it computes (PAPER.md = P):
 *   - struct(L+U) of a square pattern A with implicit nonzero diagonal
 *     (P:80-86): (i,j) is in L+U iff A(i,j) != 0 or there is a directed path
 *     i -> ... -> j in G(A) whose intermediate vertices are all < min(i,j)
 *     (fill-path theorem, Theorem thm:fill).
 *   - computed per row with Rose-Tarjan "fill2" (fig:alg_back(b)):
 *     thresholds are processed one at a time in increasing order, starting
 *     from the smallest; for each threshold t the vertices smaller than t
 *     that are connected to t are exhausted (a DFS through vertices < t);
 *     every vertex is visited once per row (fill(v) = src marking).
 *     Neighbours larger than the threshold are new entries of L(src,:) or
 *     U(src,:) and, if smaller than src, become later thresholds.
 *   - L = strictly lower part, U = upper part INCLUDING the diagonal
 *     (nnz(U(0,:)) = 3 in the worked example counts the pivot).
 *   - T3 supernodes (Definition def:T3): greedy left-to-right
 *     scan; row s joins the supernode that begins at leader r iff
 *     nnz(U(s,:)) = nnz(U(s-1,:)) - 1 and L(s,r) != 0; a row at a multiple
 *     of chunk_size always starts a new supernode (chunkSize = maximum
 *     supernode size; default 128).
 *
 * Rows are independent given the static G(A), so rows are spread
 * over POSIX threads (dynamic blocks of 64 rows, largest row ids first since
 * work grows with the source id).  No blocking, fusion or
 * reordering of a row's own arithmetic beyond fill2 itself.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n;
    const int64_t *rowptr;
    const int32_t *colidx;
    const int64_t *rows;   /* rows to compute */
    int64_t nrows;
    int64_t next_block;    /* shared cursor (from the end) */
    pthread_mutex_t lock;
    int32_t **Lrow, **Urow; /* per requested row, malloc'd */
    int64_t *Lcnt, *Ucnt;
    int64_t *visits;       /* per thread: sum of degrees of visited vertices */
    int failed;
} job_t;

typedef struct {
    job_t *job;
    int tid;
} targ_t;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* binary min-heap of int32 (the fill2 threshold priority queue) */
static void heap_push(int32_t *h, int64_t *sz, int32_t v) {
    int64_t i = (*sz)++;
    h[i] = v;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p] <= h[i]) break;
        int32_t t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}

static int32_t heap_pop(int32_t *h, int64_t *sz) {
    int32_t top = h[0];
    h[0] = h[--(*sz)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *sz && h[l] < h[m]) m = l;
        if (r < *sz && h[r] < h[m]) m = r;
        if (m == i) break;
        int32_t t = h[m]; h[m] = h[i]; h[i] = t;
        i = m;
    }
    return top;
}

/*
 * fill2 for one source row `src`.
 *   mark[v] == src  <=>  v already visited for this src   (fill(v) = src)
 *   S               =    columns of struct(L+U)(src,:) other than src
 * Returns the number of entries in S, or -1 on allocation failure.
 */
static int64_t fill2_row(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                         int32_t src, int32_t *mark, int32_t *heap,
                         int32_t *stack, int32_t **S, int64_t *Scap,
                         int64_t *visits) {
    int64_t ns = 0, hs = 0;
    (void)n;
#define S_ADD(v)                                                             \
    do {                                                                     \
        if (ns == *Scap) {                                                   \
            int64_t nc = *Scap ? 2 * *Scap : 1024;                           \
            int32_t *p = (int32_t *)realloc(*S, (size_t)nc * sizeof(int32_t)); \
            if (!p) return -1;                                               \
            *S = p; *Scap = nc;                                              \
        }                                                                    \
        (*S)[ns++] = (v);                                                    \
    } while (0)

    mark[src] = src;
    /* initialisation: the out-neighbours of src are in the structure; the
     * smaller ones are the first thresholds ("neighbors of src that
     * are smaller than src ... are inserted into frontierQueue") */
    *visits += rowptr[src + 1] - rowptr[src];
    for (int64_t e = rowptr[src]; e < rowptr[src + 1]; ++e) {
        int32_t w = colidx[e];
        if (w == src || mark[w] == src) continue;
        mark[w] = src;
        S_ADD(w);
        if (w < src) heap_push(heap, &hs, w);
    }
    /* one threshold at a time, smallest first ("starting from the
     * smallest one") */
    while (hs > 0) {
        int32_t t = heap_pop(heap, &hs);
        int64_t top = 0;
        stack[top++] = t;
        while (top > 0) {
            int32_t u = stack[--top];
            *visits += rowptr[u + 1] - rowptr[u];
            for (int64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
                int32_t w = colidx[e];
                if (mark[w] == src) continue;     /* visited once per src */
                mark[w] = src;
                if (w > t) {
                    /* every intermediate on src ~> t -> (vertices < t) -> w
                     * is <= t < min(src, w): Theorem thm:fill holds */
                    S_ADD(w);
                    if (w < src) heap_push(heap, &hs, w);  /* later threshold */
                } else {
                    /* w < t: reached with path maximum t > w, so (src,w) is
                     * not (yet) an entry; keep exhausting vertices < t */
                    stack[top++] = w;
                }
            }
        }
    }
#undef S_ADD
    return ns;
}

static void *worker(void *p) {
    targ_t *ta = (targ_t *)p;
    job_t *J = ta->job;
    int64_t n = J->n;
    int32_t *mark = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *heap = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *stack = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *S = NULL;
    int64_t Scap = 0, visits = 0;
    if (!mark || !heap || !stack) {
        pthread_mutex_lock(&J->lock); J->failed = 1; pthread_mutex_unlock(&J->lock);
        free(mark); free(heap); free(stack);
        return NULL;
    }
    for (int64_t v = 0; v < n; ++v) mark[v] = -1;
    for (;;) {
        int64_t hi;
        pthread_mutex_lock(&J->lock);
        hi = J->next_block;
        J->next_block = hi - 64;
        pthread_mutex_unlock(&J->lock);
        if (hi <= 0) break;
        int64_t lo = hi - 64 < 0 ? 0 : hi - 64;
        for (int64_t r = hi - 1; r >= lo; --r) {
            int32_t src = (int32_t)J->rows[r];
            int64_t ns = fill2_row(n, J->rowptr, J->colidx, src, mark, heap,
                                   stack, &S, &Scap, &visits);
            if (ns < 0) { J->failed = 1; continue; }
            qsort(S, (size_t)ns, sizeof(int32_t), cmp_i32);
            int64_t nl = 0;
            while (nl < ns && S[nl] < src) ++nl;
            int32_t *Lr = (int32_t *)malloc((size_t)(nl ? nl : 1) * sizeof(int32_t));
            int32_t *Ur = (int32_t *)malloc((size_t)(ns - nl + 1) * sizeof(int32_t));
            if (!Lr || !Ur) { J->failed = 1; free(Lr); free(Ur); continue; }
            memcpy(Lr, S, (size_t)nl * sizeof(int32_t));
            Ur[0] = src;  /* U carries the diagonal */
            memcpy(Ur + 1, S + nl, (size_t)(ns - nl) * sizeof(int32_t));
            J->Lrow[r] = Lr; J->Urow[r] = Ur;
            J->Lcnt[r] = nl; J->Ucnt[r] = ns - nl + 1;
        }
    }
    J->visits[ta->tid] = visits;
    free(S); free(mark); free(heap); free(stack);
    return NULL;
}

/*
 * oracle_rows: struct(L(i,:)) and struct(U(i,:)) for every i in rows[0..nrows).
 * Outputs (malloc'd, caller frees with oracle_free):
 *   *Lptr int64[nrows+1], *Lidx int32[...]  -- CSR over the requested rows
 *   *Uptr int64[nrows+1], *Uidx int32[...]  -- U includes the diagonal
 *   *visits = sum over rows of the degrees of visited vertices (work count)
 * Returns 0 on success, -1 on allocation failure, -2 on bad arguments.
 */
int oracle_rows(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                const int64_t *rows, int64_t nrows, int nthreads,
                int64_t **Lptr, int32_t **Lidx, int64_t **Uptr, int32_t **Uidx,
                int64_t *visits_out) {
    if (n <= 0 || !rowptr || !colidx || nrows < 0 || (nrows && !rows)) return -2;
    for (int64_t r = 0; r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= n) return -2;
    if (nthreads < 1) nthreads = 1;
    job_t J;
    memset(&J, 0, sizeof J);
    J.n = n; J.rowptr = rowptr; J.colidx = colidx; J.rows = rows; J.nrows = nrows;
    J.next_block = nrows;
    pthread_mutex_init(&J.lock, NULL);
    J.Lrow = (int32_t **)calloc((size_t)(nrows ? nrows : 1), sizeof(int32_t *));
    J.Urow = (int32_t **)calloc((size_t)(nrows ? nrows : 1), sizeof(int32_t *));
    J.Lcnt = (int64_t *)calloc((size_t)(nrows ? nrows : 1), sizeof(int64_t));
    J.Ucnt = (int64_t *)calloc((size_t)(nrows ? nrows : 1), sizeof(int64_t));
    J.visits = (int64_t *)calloc((size_t)nthreads, sizeof(int64_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    targ_t *ta = (targ_t *)calloc((size_t)nthreads, sizeof(targ_t));
    int rc = 0;
    if (!J.Lrow || !J.Urow || !J.Lcnt || !J.Ucnt || !J.visits || !th || !ta) { rc = -1; goto done; }
    for (int t = 0; t < nthreads; ++t) {
        ta[t].job = &J; ta[t].tid = t;
        pthread_create(&th[t], NULL, worker, &ta[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    if (J.failed) { rc = -1; goto done; }
    {
        int64_t *lp = (int64_t *)malloc((size_t)(nrows + 1) * sizeof(int64_t));
        int64_t *up = (int64_t *)malloc((size_t)(nrows + 1) * sizeof(int64_t));
        if (!lp || !up) { free(lp); free(up); rc = -1; goto done; }
        lp[0] = up[0] = 0;
        for (int64_t r = 0; r < nrows; ++r) {
            lp[r + 1] = lp[r] + J.Lcnt[r];
            up[r + 1] = up[r] + J.Ucnt[r];
        }
        int32_t *li = (int32_t *)malloc((size_t)(lp[nrows] ? lp[nrows] : 1) * sizeof(int32_t));
        int32_t *ui = (int32_t *)malloc((size_t)(up[nrows] ? up[nrows] : 1) * sizeof(int32_t));
        if (!li || !ui) { free(lp); free(up); free(li); free(ui); rc = -1; goto done; }
        for (int64_t r = 0; r < nrows; ++r) {
            memcpy(li + lp[r], J.Lrow[r], (size_t)J.Lcnt[r] * sizeof(int32_t));
            memcpy(ui + up[r], J.Urow[r], (size_t)J.Ucnt[r] * sizeof(int32_t));
        }
        *Lptr = lp; *Lidx = li; *Uptr = up; *Uidx = ui;
        int64_t v = 0;
        for (int t = 0; t < nthreads; ++t) v += J.visits[t];
        if (visits_out) *visits_out = v;
    }
done:
    for (int64_t r = 0; r < nrows; ++r) { free(J.Lrow[r]); free(J.Urow[r]); }
    free(J.Lrow); free(J.Urow); free(J.Lcnt); free(J.Ucnt); free(J.visits);
    free(th); free(ta);
    pthread_mutex_destroy(&J.lock);
    return rc;
}

/*
 * oracle_supernodes: T3 supernode partition of the consecutive rows
 * [row_begin, row_begin + nrows) by the greedy scan of Definition def:T3
 * (P:299-306), with a forced break at every row s with s % chunk_size == 0
 * (chunkSize = maximum supernode size) and at row_begin.
 *   Lptr/Lidx: CSR of L over those rows (sorted columns)
 *   Uptr:      row pointers of U over those rows (nnz(U(s,:)) incl. diagonal)
 *   sn_start:  out, int32[nrows+1] capacity; leading rows + sentinel row_end
 * Returns the number of supernodes, or -2 on bad arguments.
 */
int64_t oracle_supernodes(int64_t row_begin, int64_t nrows, const int64_t *Lptr,
                          const int32_t *Lidx, const int64_t *Uptr,
                          int64_t chunk_size, int32_t *sn_start) {
    if (nrows < 0 || chunk_size < 1 || !sn_start) return -2;
    int64_t ns = 0, r = -1;
    for (int64_t k = 0; k < nrows; ++k) {
        int64_t s = row_begin + k;
        int joins = 0;
        if (k > 0 && s % chunk_size != 0) {
            int64_t nnz_s = Uptr[k + 1] - Uptr[k];
            int64_t nnz_prev = Uptr[k] - Uptr[k - 1];
            if (nnz_s == nnz_prev - 1) {              /* requirement (i) */
                for (int64_t e = Lptr[k]; e < Lptr[k + 1]; ++e)
                    if (Lidx[e] == r) { joins = 1; break; }  /* (ii) L(s,r) != 0 */
            }
        }
        if (!joins) { r = s; sn_start[ns++] = (int32_t)s; }
    }
    sn_start[ns] = (int32_t)(row_begin + nrows);
    return ns;
}

void oracle_free(void *p) { free(p); }

/*
 * oracle_supernodes_cap: the cap-only variant of the T3 partition (SURVEY.md
 * §8(f) NEXT-3).  chunkSize is read only as "the size of the user defined
 * maximum supernode" (default 128 P:1011), without the forced break at
 * multiples of chunk_size: the greedy left-to-right scan of Definition def:T3
 * from row_begin, where row s joins the supernode of leader r iff
 *   s - r < cap                       (the supernode would not exceed cap rows)
 *   nnz(U(s,:)) = nnz(U(s-1,:)) - 1   (requirement (i))
 *   L(s, r) != 0                      (requirement (ii))
 * and otherwise starts a new supernode.  Arguments as oracle_supernodes.
 */
int64_t oracle_supernodes_cap(int64_t row_begin, int64_t nrows, const int64_t *Lptr,
                              const int32_t *Lidx, const int64_t *Uptr,
                              int64_t cap, int32_t *sn_start) {
    if (nrows < 0 || cap < 1 || !sn_start) return -2;
    int64_t ns = 0, r = -1;
    for (int64_t k = 0; k < nrows; ++k) {
        int64_t s = row_begin + k;
        int joins = 0;
        if (k > 0 && s - r < cap) {
            int64_t nnz_s = Uptr[k + 1] - Uptr[k];
            int64_t nnz_prev = Uptr[k] - Uptr[k - 1];
            if (nnz_s == nnz_prev - 1) {              /* requirement (i) */
                for (int64_t e = Lptr[k]; e < Lptr[k + 1]; ++e)
                    if (Lidx[e] == r) { joins = 1; break; }  /* (ii) L(s,r) != 0 */
            }
        }
        if (!joins) { r = s; sn_start[ns++] = (int32_t)s; }
    }
    sn_start[ns] = (int32_t)(row_begin + nrows);
    return ns;
}
