/*
 * gsofa.h -- C ABI of the B200-native gSoFa symbolic-factorization hot path.
 *
 * Problem (PAPER.md = P): "symbolic factorization is used to compute the
 * locations of the fill-ins for both L and U ... needed to allocate the
 * compressed sparse data structures for L and U".  For a square
 * sparsity pattern A with implicitly nonzero diagonal, entry (i,j)
 * of L+U is nonzero iff A(i,j) != 0 or there is a directed path i -> j in
 * G(A) whose intermediate vertices are all smaller than min(i,j) (fill-path
 * theorem, Theorem thm:fill).  The library finds, for every source
 * row, the L and U patterns with the paper's frontier-driven max-id
 * relaxation (sec:parallel) run for batches of concurrent sources
 * on the GPU, then detects T3 supernodes (Definition def:T3) with
 * the two-phase design.
 *
 * Everything here is plain C: pointers and sizes, no C++ or PyTorch types.
 * All entry points return an int status (0 = GSOFA_OK, negative = error);
 * on error no output object is produced (*out == NULL) and
 * gsofa_last_error_detail() describes the cause (thread-local).
 * There is no CPU fallback: every step of the factorization runs in the
 * library's sm_100a CUDA kernels; without a usable GPU calls fail with
 * GSOFA_ECUDA.
 */
#ifndef GSOFA_H
#define GSOFA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSOFA_VERSION 2

/* ---------------------------------------------------------- error codes -- */
#define GSOFA_OK            0
#define GSOFA_EINVAL       -1  /* bad argument: n <= 0, NULL pointer, bad opts,
                                  row_begin >= row_end, max_concurrent not a
                                  multiple of 32, a stitch tail that does not
                                  end at row_begin - 1 */
#define GSOFA_EBADCSR      -2  /* rowptr[0] != 0, rowptr decreasing, column out
                                  of [0,n), columns not strictly increasing in a
                                  row, nnz >= 2^31 */
#define GSOFA_ENOMEM       -3  /* device (or host output) allocation failed */
#define GSOFA_EINFEASIBLE  -4  /* memory budget below one 32-source group's
                                  footprint (the paper's "reduce the number of
                                  concurrent sources" cannot go lower) */
#define GSOFA_ECUDA        -5  /* any CUDA runtime error (no GPU, launch failure) */
#define GSOFA_EINTERNAL    -6  /* checked-mode invariant violated */

#define GSOFA_SCHEDULE_THRESHOLD 0
#define GSOFA_SCHEDULE_FIFO      1
#define GSOFA_SCHEDULE_AUTO      2
#define GSOFA_SCHEDULE_HEIGHT    3

/* Row interleave: the paper's source scheduling
 * across GPUs -- consecutive chunks of rows dealt round-robin to the
 * compute nodes and rows interleaved across the GPUs of a node to balance
 * the work (measured 1.6x and a further 3.3x there).  A
 * call with nparts > 1 computes only the units u = 0, 1, ... of unit_rows
 * rows, counted from row_begin, with u % nparts == part; its result holds
 * those rows in ascending order (local row k is the k-th of them).
 *   unit_rows a multiple of chunk_size: every unit starts a chunk, so the
 *     supernodes are unit-local and complete after the call;
 *   otherwise (finer interleave): the supernodes need the neighbouring
 *     rows of other parts -- nsuper is -1 after the call, and each part
 *     exports its per-row Def. def:T3 data (gsofa_result_rowinfo), the parts
 *     all-gather it and every part calls gsofa_supernodes_gathered.
 * nparts <= 1: no interleave (all rows of [row_begin, row_end)). */
typedef struct gsofa_interleave {
  int32_t nparts;     /* N: number of parts (GPUs) */
  int32_t part;       /* q in [0, N): this call's part */
  int32_t unit_rows;  /* U: rows per unit, a multiple of 32 */
  int32_t reserved;
} gsofa_interleave;

/* -------------------------------------------------------------- options -- */
typedef struct gsofa_opts {
  /* chunkSize = user-defined maximum supernode size; a supernode never crosses
   * a multiple of chunk_size ("chunkSize is identical to the size of the user
   * defined maximum supernode"; default 128).  >= 1. */
  int32_t chunk_size;
  /* #C, the number of concurrent sources per batch.  Multiple of
   * 32 (one 32-source slot group per warp lane set).  0 = automatic (the
   * largest batch the memory budget allows, capped at 65536). */
  int32_t max_concurrent;
  /* memory budget in bytes for the traversal arena.  0 = automatic
   * (about half of the free device memory). */
  int64_t mem_budget_bytes;
  /* 1 = "line 9.5" access order: test the structure before the atomicMin on
   * maxId.  Result-invariant; default 0 as in the paper. */
  int32_t fill_first;
  /* Processing order of the max-id relaxation (result-invariant; DESIGN.md
   * "Schedules"):
   *   GSOFA_SCHEDULE_THRESHOLD (0): frontier items in increasing newMaxId
   *     ("Dijkstra order"): no revisits, no grid-wide barriers;
   *     lockstep 32-source groups plus per-source solo warps.
   *   GSOFA_SCHEDULE_FIFO (1): the paper's order -- all frontiers of an
   *     iteration in parallel with revisits, one
   *     persistent grid-wide kernel per batch with epoch-encoded maxId
   *     labels.
   *   GSOFA_SCHEDULE_HEIGHT (3): the threshold order by elimination-tree
   *     height instead of vertex id: thresholds of one height have disjoint
   *     closures (they lie in disjoint subtrees of the etree of A + A^T,
   *     P:264), so a step expands all thresholds of one height at once;
   *     no revisits, |L(s,:)| steps per source become at most the tree
   *     height.  The plan computes the etree on the host (Liu's algorithm,
   *     O(nnz alpha)).
   *   GSOFA_SCHEDULE_AUTO (2, default): FIFO when the pattern is banded and
   *     dense (bandwidth <= n/8 and nnz >= 8n: few rounds, almost no
   *     revisits -- measured 1.3-2.9x faster there) and one batch of labels
   *     (min(rows, 65536) x n x 4 B) fits the memory budget of the call;
   *     threshold otherwise (ND orders, hubs: 15x the inspections in FIFO),
   *     and also when the FIFO plan turns out infeasible.  Within the
   *     threshold family, patterns with hub rows (largest row > 32x the
   *     mean row length) get the elimination tree computed on the host; the
   *     height order is taken when the last row's id-order chain exceeds 4x
   *     the tree height (C4's hubs), else id order.  The bandwidth and the
   *     largest row are measured by the CSR validation pass.
   *     gsofa_result.schedule reports the choice. */
  int32_t schedule;
  /* source rows [row_begin, row_end); row_end = -1 means n.  Any row_begin:
   * if it is not a multiple of chunk_size, the supernodes of the head rows
   * [row_begin, next multiple of chunk_size) are provisional (computed as if
   * row_begin started a block) until gsofa_supernode_stitch() is given the
   * predecessor range's tail; supernodes never cross a multiple of
   * chunk_size, so all later blocks are final. */
  int64_t row_begin, row_end;
  /* CUDA device ordinal used when the call creates its own context. */
  int32_t device;
  /* 1: result arrays are device pointers (cudaMalloc'd); 0: host (malloc). */
  int32_t outputs_on_device;
  /* cudaStream_t to run on (NULL = the context's own stream). */
  void *stream;
  /* 1 = checked mode: after the factorization a GPU
   * audit verifies every output row (L strictly lower and ascending, U
   * starting with the diagonal and ascending), pattern(A) within L+U, and
   * Definition def:T3 for every supernode row; a violation returns
   * GSOFA_EINTERNAL with the failed checks in gsofa_last_error_detail().
   * Costs one extra pass over the output; default 0. */
  int32_t checked;
  /* Supernode rule.  0 (default): forced break at
   * every multiple of chunk_size (chunks never share a supernode).
   * 1: cap-only -- chunk_size is only "the size of the user defined maximum
   * supernode": the greedy Def. def:T3 scan lets row s
   * join the block of leader r iff s - r < chunk_size and (i), (ii) hold,
   * so blocks may cross multiples of chunk_size.  A range's provisional head
   * blocks can then change up to the first row where the stitched scan meets
   * one of its own leaders (gsofa_supernode_stitch); the tail record's
   * leader carries the running block length (row - leader + 1). */
  int32_t sn_cap_only;
  /* row interleave (see gsofa_interleave); all zero = off.  Needs the
   * threshold family of schedules (AUTO then never picks FIFO), row_begin a
   * multiple of chunk_size and the forced-break supernode rule. */
  gsofa_interleave interleave;
} gsofa_opts;

/* ------------------------------------------------------------ statistics -- */
typedef struct gsofa_stats {
  int64_t edge_inspections;  /* (source, edge) relaxations performed, incl.
                                revisits (TEPS numerator) */
  int64_t frontier_items;    /* (vertex, 32-source group) work items expanded */
  int64_t item_edges;        /* (item, neighbour) pairs: adjacency entries read,
                                each touching one 32-source state word */
  int64_t rounds;            /* frontier levels (iterations) summed over
                                batches / groups */
  int64_t thresholds;        /* threshold steps (GSOFA_SCHEDULE_THRESHOLD) */
  int64_t batches;           /* source batches */
  int64_t max_batch;         /* largest #C used */
  int64_t kernel_launches;   /* CUDA kernels launched by this call */
  double ms_total;           /* device time of the whole call (CUDA events) */
  double ms_traverse;        /* seed + traversal kernels */
  double ms_extract;         /* row extraction (count + scan + write) */
  double ms_supernode;       /* supernode detection */
  double ms_transfer;        /* host<->device copies inside the call */
  /* R11: first-visit vs total work.  first_visits = (source, vertex)
   * pairs, vertex < source, whose maxId left "unvisited" (each such vertex is
   * expanded at least once); source_expansions = (source, vertex) frontier
   * expansions including revisits.  revisit factor = source_expansions /
   * first_visits: exactly 1 in threshold order (every reached vertex is
   * expanded once), > 1 in the paper's FIFO order.  Groups the lockstep
   * kernel abandons to the solo kernel count once (their redo). */
  int64_t first_visits;
  int64_t source_expansions;
  /* External frontier management (FIFO order): frontier queue
   * items written to pinned host memory because the HBM part of the queue
   * (1/8 of its worst case when the memory budget is short, else all of it)
   * was full.  0 when everything fit on the GPU. */
  int64_t frontier_spilled;
} gsofa_stats;

/* --------------------------------------------------------------- result -- */
typedef struct gsofa_result {
  int64_t n, row_begin, row_end;
  /* CSR over rows [row_begin, row_end) (row i at index i - row_begin);
   * L strictly lower (unit diagonal implicit), ascending columns */
  int64_t *L_rowptr;   /* [row_end - row_begin + 1], L_rowptr[0] = 0 */
  int32_t *L_colidx;   /* [nnz_L] */
  /* U upper triangle INCLUDING the diagonal (nnz(U(0,:)) = 3 in the worked
   * example counts the pivot), ascending columns; U(i,:)[0] == i */
  int64_t *U_rowptr;   /* [row_end - row_begin + 1] */
  int32_t *U_colidx;   /* [nnz_U] */
  /* T3 supernodes: leading rows ascending, then the sentinel row_end */
  int64_t nsuper;
  int32_t *sn_start;   /* [nsuper + 1] */
  int64_t nnz_L, nnz_U;
  int64_t nnz_A_offdiag;  /* off-diagonal nonzeros of A in the rows */
  int64_t fill_count;     /* nnz_L + (nnz_U - rows) - nnz_A_offdiag */
  int32_t on_device;      /* 1 if the arrays above are device pointers */
  int32_t device;
  gsofa_stats stats;
  int32_t schedule;       /* the schedule that ran (THRESHOLD or FIFO) */
  int32_t reserved;
  /* rows held: row_end - row_begin, or the rows of this part under a row
   * interleave (the arrays above are indexed by local row k; sn_start holds
   * global leading rows, its sentinel is one past the last row held) */
  int64_t rows;
  gsofa_interleave interleave;
} gsofa_result;

typedef struct gsofa_context gsofa_context;

/* Fill *o with the defaults above.  Returns GSOFA_EINVAL if o is NULL. */
int gsofa_default_opts(gsofa_opts *o);

/* A context owns the device arena (maxId labels, frontier queues and masks,
 * structure bitmaps: Table tab:complexity, allocated as "a big
 * chunk of memory"), its stream and the maxId epoch counter
 * (P:570-574), so that repeated calls neither reallocate nor re-initialise.
 * mem_budget_bytes = 0: automatic.  Not thread-safe: one context per thread. */
int gsofa_context_create(int32_t device, int64_t mem_budget_bytes, gsofa_context **ctx);
void gsofa_context_destroy(gsofa_context *ctx);

/*
 * gsofa_symbolic -- symbolic LU factorization of the n x n pattern
 * (rowptr, colidx) for source rows [opts->row_begin, opts->row_end).
 *
 *   ctx     context (NULL: a temporary one on opts->device)
 *   n       order of A (|V| of G(A)), 1 <= n < 2^31
 *   rowptr  int64[n+1] CSR row pointers, rowptr[0] = 0, nondecreasing
 *   colidx  int32[rowptr[n]] column indices, strictly increasing per row;
 *           diagonal entries are accepted and ignored (the diagonal is
 *           implicit)
 *   Inputs may be host or device pointers (detected with
 *   cudaPointerGetAttributes); they are borrowed read-only.
 *   opts    NULL = defaults
 *   out     receives a library-allocated result; release with
 *           gsofa_result_free().  The input must already be ordered
 *           (fill-reducing ordering is out of scope).
 */
int gsofa_symbolic(gsofa_context *ctx, int64_t n, const int64_t *rowptr,
                   const int32_t *colidx, const gsofa_opts *opts,
                   gsofa_result **out);

/* Tail record of a row range, exchanged between neighbouring ranges (the
 * multi-GPU supernode-boundary exchange): the range's last row, its nnz(U)
 * (diagonal included, R6) and the leading row of the supernode containing it. */
typedef struct gsofa_tail {
  int64_t row;
  int64_t nnzU;
  int64_t leader;
} gsofa_tail;

/*
 * gsofa_supernode_stitch -- supernode continuity across row ranges
 * (Definition def:T3; chunk rule P:640).
 *   r     a result of gsofa_symbolic over [row_begin, row_end); modified in
 *         place: sn_start / nsuper of the head rows [row_begin, next multiple
 *         of chunk_size) are recomputed by the greedy Def. def:T3 scan
 *         starting from *prev (row s joins the block of leader r iff
 *         nnz(U(s,:)) = nnz(U(s-1,:)) - 1 and L(s, r) != 0).  Blocks after
 *         that chunk boundary are unchanged.  With sn_cap_only the re-scan
 *         (also requiring s - r < chunk_size) runs until it starts a block at
 *         a row that already leads one (from there on the scans agree), or to
 *         row_end.  The scan runs in a CUDA kernel (host results are read
 *         through their pinned mapping).
 *   prev  tail of the range ending at row_begin - 1 (else GSOFA_EINVAL);
 *         NULL: row_begin truly starts a block (e.g. row_begin = 0), nothing
 *         changes.
 *   out   if not NULL, receives this range's tail (after stitching), to be
 *         passed to the next range.
 * Ranges must be stitched in increasing order.  Synchronous; a few hundred
 * bytes move.  Errors: GSOFA_EINVAL, GSOFA_ECUDA (r is left unchanged).
 */
int gsofa_supernode_stitch(gsofa_result *r, const gsofa_tail *prev, gsofa_tail *out);

/* Copies the result arrays into caller-owned buffers (host or device; any
 * NULL destination is skipped).  Sizes: L_rowptr/U_rowptr rows+1, L_colidx
 * nnz_L, U_colidx nnz_U, sn_start nsuper+1.  Synchronous.  Lets a binding
 * move results into its own allocations (e.g. framework tensors). */
int gsofa_result_copy(const gsofa_result *r, int64_t *L_rowptr, int32_t *L_colidx,
                      int64_t *U_rowptr, int32_t *U_colidx, int32_t *sn_start);

/*
 * gsofa_result_l_csc -- L of a result in compressed sparse COLUMN form
 * (SuperLU-style column storage; north_star "L and U patterns as CSR/CSC").
 *   r          a gsofa_symbolic result over rows [row_begin, row_end)
 *   on_device  1: the arrays are device memory (cudaMallocAsync), 0: host (malloc)
 *   col_ptr    receives int64[n+1]: column j's entries are row_idx[col_ptr[j] ..
 *              col_ptr[j+1]); columns span [0, n) (L(i,j) != 0 needs j < i)
 *   row_idx    receives int32[nnz_L]: the rows i in [row_begin, row_end) with
 *              L(i,j) != 0, ascending within each column
 * The caller owns both arrays: release them with gsofa_buffer_free(p, on_device).
 * Runs on the result's device: a stable radix sort of the (column, row) pairs
 * by column, then a binary search per column.  Errors: GSOFA_EINVAL,
 * GSOFA_ENOMEM, GSOFA_ECUDA (no arrays are returned).
 */
int gsofa_result_l_csc(const gsofa_result *r, int32_t on_device, int64_t **col_ptr,
                       int32_t **row_idx);
void gsofa_buffer_free(void *p, int32_t on_device);

/*
 * gsofa_result_supno -- the supernode partition in SuperLU's form: xsup is
 * r->sn_start itself (first row of each supernode, then the sentinel), and
 * supno[i - row_begin] = the index k of the supernode holding row i
 * (xsup[k] <= i < xsup[k+1]); numeric factorization codes index their
 * supernodal blocks by it.
 *   r          a gsofa_symbolic result (after any gsofa_supernode_stitch)
 *   on_device  1: *supno is device memory, 0: host (malloc)
 *   supno      receives int32[row_end - row_begin]; release with
 *              gsofa_buffer_free(p, on_device)
 * Runs on the result's device (one thread per supernode).  Errors:
 * GSOFA_EINVAL, GSOFA_ENOMEM, GSOFA_ECUDA.
 */
int gsofa_result_supno(const gsofa_result *r, int32_t on_device, int32_t **supno);

/*
 * gsofa_permute -- symmetric permutation B = P A P^T of a pattern, for applying
 * a fill-reducing ordering computed elsewhere (ordering itself is out of
 * scope): new vertex i is old vertex perm[i], so
 * B(i, j) != 0 iff A(perm[i], perm[j]) != 0.
 *   n, rowptr int64[n+1], colidx int32[nnz]   input CSR (columns ascending)
 *   perm      int32[n], a permutation of [0, n) (else GSOFA_EINVAL)
 *   out_rowptr int64[n+1], out_colidx int32[nnz]   caller-allocated output,
 *             columns ascending in every row
 * All five pointers host, or all device.  Runs on the current CUDA device
 * (one radix sort of (row, column) keys).  Synchronous.
 */
int gsofa_permute(int64_t n, const int64_t *rowptr, const int32_t *colidx, const int32_t *perm,
                  int64_t *out_rowptr, int32_t *out_colidx);

/*
 * gsofa_result_rowinfo -- what the supernode detection of the rows after this
 * part's rows needs from it (finer-than-chunk row interleave, see
 * gsofa_interleave): for each local row k (global row s):
 *   nnzU[k]              nnz(U(s,:)) including the diagonal (Def. def:T3 (i))
 *   lmask[k * W + d / 32] bit d % 32 set iff L(s, s - d) != 0, for
 *                        1 <= d <= s % chunk_size (candidate leaders inside
 *                        s's chunk, Def. def:T3 (ii)); W = (chunk_size + 31) / 32
 * Both arrays are caller-allocated DEVICE memory on the result's device
 * (int32[rows], uint32[rows * W]); r must be a device result.  One kernel on
 * the result's device, synchronous.  Errors: GSOFA_EINVAL, GSOFA_ECUDA.
 */
int gsofa_result_rowinfo(const gsofa_result *r, int32_t *nnzU, uint32_t *lmask);

/*
 * gsofa_supernodes_gathered -- the supernodes of an interleaved part from
 * every part's rowinfo (all-gathered, part-major: part p's local row k at
 * index p * stride + k of nnzU_all, and at (p * stride + k) * W of
 * lmask_all; device memory).  The greedy Def. def:T3 scan runs
 * once per chunk (forced break at every multiple of chunk_size) over
 * the rows of all parts; r keeps the leaders among its own rows: sn_start
 * and nsuper are written in place (the union over parts is the supernode
 * partition of [row_begin, row_end)).  Synchronous.  Errors: GSOFA_EINVAL
 * (r not interleaved, or not a device result), GSOFA_ECUDA.
 */
int gsofa_supernodes_gathered(gsofa_result *r, const int32_t *nnzU_all, const uint32_t *lmask_all,
                              int64_t stride);

/* Frees every array of r (host or device) and r itself.  NULL is a no-op. */
void gsofa_result_free(gsofa_result *r);

/*
 * gsofa_partition_rows -- split the source rows [0,n) into nparts contiguous
 * ranges of roughly equal estimated work, for running one range per GPU.
 * Work grows with the source id; the estimate for row s is the
 * degree sum over the subtree of s in the elimination tree of the symmetrised
 * pattern A + A^T (an upper bound of the vertices reachable from s through
 * smaller vertices; elimination tree).  Range starts are multiples of
 * `align` (1 = row-granular, the default of the multi-GPU layer, which then
 * stitches supernodes across ranges with gsofa_supernode_stitch; chunk_size
 * makes every range start a block).
 *   bounds: out int64[nparts+1], bounds[0] = 0, bounds[nparts] = n.
 * Host-only computation (no GPU needed); deterministic, so every rank
 * computes the same partition.
 */
int gsofa_partition_rows(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                         int32_t nparts, int32_t align, int64_t *bounds);

/*
 * gsofa_height_order -- plan step A2 of the height-ordered threshold schedule
 * (elimination tree; R18), the host pass
 * gsofa_symbolic runs for hub patterns: the elimination tree of the
 * symmetrised pattern A + A^T (Liu's algorithm, split over host threads:
 * GSOFA_HOST_THREADS, default the hardware threads for n >= 65536), each
 * vertex's height in it, and its position when the vertices are sorted by
 * (height, id).
 *   parent: out int32[n], -1 for roots     hgt: out int32[n]
 *   pos:    out int32[n], a permutation    (any of the three may be NULL)
 *   height: out, the tree height           last_row_chain: out, the number of
 *           vertices of the last row's subtree path union (|struct(L(n-1,:))|
 *           of A + A^T, the AUTO order choice's chain estimate); may be NULL
 * Host pointers only, borrowed; the same CSR rules as gsofa_symbolic (rowptr
 * monotone from 0, columns in [0,n) strictly increasing per row).  Errors:
 * GSOFA_EINVAL (bad arguments, device pointers), GSOFA_EBADCSR.
 */
int gsofa_height_order(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent,
                       int32_t *hgt, int32_t *pos, int64_t *height, int64_t *last_row_chain);

/* Static strings for an error code; thread-local detail of the last error. */
const char *gsofa_strerror(int code);
const char *gsofa_last_error_detail(void);
int gsofa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GSOFA_H */
