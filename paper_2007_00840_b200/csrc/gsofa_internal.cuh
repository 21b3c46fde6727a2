// gsofa_internal.cuh -- shared declarations of the CUDA path (sm_100a only).
//
// Device data layout for one batch of C = 32*G concurrent sources
// [s0, s0 + C):
//
//   lab [G][Vb][32] uint32  maxId labels, Vb = min(n, s0 + C): bubble removal
//                           at batch granularity.  Lane k of slot
//                           group g is source s0 + 32g + k, so one warp's 32
//                           labels of a vertex are one 128-byte line.
//                           Epoch-encoded: enc(m) = base + m + 1,
//                           m in [-1, n]; values from older epochs are larger
//                           than any current value and decode as "infinity".
//   fm  [2][G][Vb] uint32   frontier masks (bit k: (vertex, source k) is in the
//                           frontier of the current / next iteration); they
//                           replace frontierQueue+tracker (Table 2)
//   queue [2][cap] uint32   compacted (vertex << gbits | g) work items, one per
//                           (vertex, group) with a nonzero mask
//   is  [G][n] uint32       in-structure bitmaps: bit k of is[g][v] set iff
//                           (s0 + 32g + k, v) is an off-diagonal entry of L+U
//                           (the paper's fill(:))
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

namespace gsofa {

constexpr int kWarp = 32;

// The source rows of a call: [rb, re), or -- row interleave across GPUs, the
// paper's source scheduling -- only the
// units u = 0, 1, ... of U rows counted from rb with u % N == q.  Local row r
// (0 .. count-1, ascending) is global row row(r); groups of 32 local rows
// are 32 consecutive global rows (U is a multiple of 32).
struct RowMap {
  int32_t rb = 0, re = 0, N = 1, q = 0, U = 32;
  __host__ __device__ __forceinline__ int32_t row(int32_t r) const {
    if (N <= 1) return rb + r;
    const int32_t u = r / U;
    return rb + (u * N + q) * U + (r - u * U);
  }
  // host: number of local rows
  int64_t count() const {
    if (N <= 1) return (int64_t)re - rb;
    const int64_t len = (int64_t)re - rb, nu = (len + U - 1) / U;
    if (nu <= q) return 0;
    const int64_t mine = (nu - q + N - 1) / N;         // units q, q + N, ... < nu
    const int64_t last = q + (mine - 1) * N;            // my last unit
    return mine * U - (last == nu - 1 ? nu * U - len : 0);
  }
};
constexpr int kTraverseThreads = 512;   // 16 warps

struct BatchParams {
  const int32_t *rowptr;   // [n+1] (device, int32 offsets)
  const int32_t *colidx;   // [nnz]
  int32_t n;
  int32_t s0;              // first source of the batch
  int32_t s_end;           // one past the last valid source (<= row_end)
  int32_t G;               // slot groups (C = 32 G)
  int32_t gbits;           // bits for g in a queue item
  int32_t Vb;              // label rows per group
  uint32_t base;           // epoch base: enc(m) = base + m + 1
  uint32_t *lab;           // [G][Vb][32]
  uint32_t *fm0, *fm1;     // [G][Vb]
  uint32_t *q0, *q1;       // queues: items [0, qcap) in HBM ...
  uint32_t *qx0, *qx1;     // ... the rest in mapped host memory (external
                           // frontier; NULL when nothing spills)
  uint32_t qcap;
  uint32_t *qcount;        // [3] rotating item counters
  uint32_t *is;            // [G][n]
  unsigned long long *stats;  // [4]: items, edge inspections, rounds, pushes
};

// ---------------------------------------------------------------- kernels
// traverse.cu
cudaError_t launch_seed(const BatchParams &p, cudaStream_t st);
cudaError_t launch_traverse(const BatchParams &p, int fill_first, int grid_blocks,
                            cudaStream_t st);
int traverse_max_blocks(int device, int fill_first);

// threshold.cu (default schedule: increasing newMaxId, persistent streaming
// kernel, one 32-source group at a time per CTA)
struct StreamParams {
  const int32_t *rowptr;
  const int32_t *colidx;
  int32_t n, row_begin, row_end, ngroups, Vmax;
  RowMap map;                // local row -> global row (row interleave)
  int32_t nrows;             // local rows (= row_end - row_begin without interleave)
  uint32_t *ws;              // [slots][ws_words]
  size_t ws_words;
  uint32_t *is;              // [slots][is_words]: is[n] | isum[n/1024]
  size_t is_words;
  unsigned int *group_ctr;   // next fresh group (global counter, heaviest first)
  unsigned int *solo_ctr;    // next of the solo_top heaviest groups (solo kernel only)
  int32_t solo_top;          // groups ngroups-solo_top.. start on the solo kernel
  // heavy path: groups abandoned by the lockstep kernel after abort_cycles
  // are queued for the solo kernel (one warp per source)
  long long abort_cycles;    // 0: never abandon
  int32_t *hq;               // [ngroups] queued group ids
  unsigned int *hq_head, *hq_tail;
  int32_t *hq_ready;         // [ngroups] publication flags
  unsigned int *done;        // rows completed (both kernels)
  unsigned int *light_live;  // lockstep CTAs running (NULL: solo warps wait for `done`)
  unsigned long long *task_ctr;  // solo kernel: next dynamic source task
  uint32_t *hws;             // [solo slots = solo CTAs x warps][hws_words] per-source workspaces
  size_t hws_words;
  int32_t solo_ring;         // closure ring entries per solo slot (power of two)
  int32_t light_slots;       // is[] slots [0, light_slots) lockstep, then solo
  const int32_t *group_list; // optional explicit group ids (retry pass)
  int32_t list_len;
  int32_t *stage;            // staged rows: [L entries | diag | U entries]
  unsigned long long stage_cap;
  unsigned long long *stage_cursor;
  int64_t *row_off;          // [rows] staging offset (-1: not staged)
  int32_t *row_nL, *row_nU;  // [rows] counts (nU includes the diagonal)
  int32_t *failed;           // groups whose rows did not fit the staging area (each once)
  int32_t *failed_flag;      // [ngroups] 1 once a group is in `failed`
  int32_t *nfailed;
  unsigned long long *failed_need;
  unsigned long long *stats; // items, edges, levels, thresholds, pairs
  long long *group_trace;    // optional [ngroups][8]: steps, levels, items, cycles, ...
  long long *src_trace;      // optional [rows][4] (solo sources): start ns, end ns, steps, levels
  int *debug;                // optional dev checks
  // processing order of the solo kernel's thresholds (order.cu): hmode = 0:
  // increasing vertex id (one threshold per step); hmode = 1: increasing etree
  // height (all same-height thresholds of the window per step); threshold
  // bitmaps then indexed by position (vertices sorted by (height, id), npos = n)
  int32_t hmode;
  int32_t lmode;             // lockstep kernel: 0 = id order, 1 = height order (no solo kernel)
  int32_t lwarps;            // warps per lockstep CTA in height order (lock_warps)
  int32_t npos;
  int32_t wide;              // solo kernel shape: 0 = throughput (48 warps/SM), 1 = latency (4 batches)
  int64_t nnz;               // entries of colidx (the latency shape's bulk copies stay inside)
  const int4 *posrec;        // [n] per position: {vertex, rowptr, rowptr + 1, end of its
                             //     height's segment of positions}
  const int32_t *hgt;        // [n] etree height of a vertex
  const int32_t *pos;        // [n] vertex -> position
  const int32_t *ell;        // [8 n] ELL adjacency (id order, rows <= 8 entries), or NULL
  long long task_base;  // the solo kernel's first task (queue entry 32 x task_base)
  // solo slot layout: word offsets of its arrays (solo_layout)
  uint32_t so_pend, so_thr, so_rsum, so_tsum, so_is, so_isum, so_queue;
};
size_t stream_ws_words(int64_t Vmax, int64_t npos);
size_t stream_is_words(int64_t n);
// lock_h: the lockstep kernel in height order (heavy = 0; its slots then hold npos threshold bits)
int stream_max_blocks(int device, int64_t Vmax, int heavy, int64_t npos, bool wide, bool lock_h = false,
                      int lw = 16);
int lock_warps(int64_t groups, int sms, bool hubs);  // warps per lockstep CTA in height order
int stream_heavy_ratio();  // warps of a solo CTA / warps of a lockstep CTA
int stream_warps_per_cta();  // lockstep slots (one group per warp) per CTA
size_t solo_ws_words(int64_t Vmax, int64_t n, int64_t npos);  // per solo slot (one warp, one source)
size_t solo_layout(int64_t Vmax, int64_t n, int64_t npos, StreamParams *p);  // + offsets
int solo_warps_per_cta();
int solo_ring(int64_t Vmax);
int stream_light_per_sm_with_solo(int device, int64_t Vmax, int64_t npos, bool wide);
size_t stream_smem_bytes(int64_t Vmax, int64_t npos);  // dynamic smem: threshold-word summary
// order.cu (host): elimination tree of A + A^T and the height order
// last_row_subtree (optional): |struct(L(n-1,:))| of A + A^T
void etree_sym(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent,
               int64_t *last_row_subtree);
// the tree's shape, for the AUTO choice of the threshold order: its height
// (rounds of the last source in height order, at most) against the last
// row's structure size (its threshold steps in id order, about)
struct OrderShape {
  int64_t height = 0;
  int64_t last_row_chain = 0;
};
// etree heights, positions (sorted by (height, id)) and per position
// {vertex, rowptr, rowptr + 1, segment end} (int4 as four int32)
// scratch (transpose, tree, split) reused across calls; nullptr: per call
struct OrderScratch;
OrderScratch *order_scratch_new();
void order_scratch_free(OrderScratch *s);
const int32_t *order_scratch_parent(const OrderScratch *s);  // the tree of the last pass
OrderShape height_order(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *hgt,
                        int32_t *pos, int32_t *posrec, OrderScratch *scratch = nullptr);
cudaError_t launch_stream(const StreamParams &p, int grid, cudaStream_t st);
cudaError_t launch_solo(const StreamParams &p, int grid, cudaStream_t st);
cudaError_t launch_gather(const int32_t *stage, const int64_t *row_off, const int32_t *row_nL,
                          const int64_t *L_rowptr, const int64_t *U_rowptr, int rows,
                          int32_t *L_out, int32_t *U_out, cudaStream_t st);

// csc.cu: L (CSR over rows [row_begin, row_begin + rows)) -> CSC over columns
// [0, n): col_ptr[n+1], row_idx[nnz] (rows ascending per column); device arrays
cudaError_t l_rows_to_csc(const int64_t *L_rowptr, const int32_t *L_colidx, int64_t rows,
                          int64_t row_begin, int64_t n, int64_t nnz, int64_t *col_ptr,
                          int32_t *row_idx, cudaStream_t st);

// radix.cu: stable LSD radix sort (8-bit digits, 64-bit counts); the result
// is in the input or the tmp arrays (*result_in_tmp); hist scratch of
// radix_hist_bytes(grid) bytes
size_t radix_hist_bytes(int grid);
inline int radix_grid() { return 296; }  // 2 persistent 1024-thread CTAs per SM
cudaError_t radix_sort_pairs_u32(uint32_t *keys, int32_t *vals, uint32_t *keys_tmp, int32_t *vals_tmp,
                                 int64_t n, int key_bits, void *hist, int grid, cudaStream_t st,
                                 bool *result_in_tmp);
cudaError_t radix_sort_keys_u64(unsigned long long *keys, unsigned long long *keys_tmp, int64_t n,
                                int key_bits, void *hist, int grid, cudaStream_t st,
                                bool *result_in_tmp);

// csc.cu: symmetric permutation B = P A P^T of a pattern (device arrays)
cudaError_t launch_iperm(const int32_t *perm, int64_t n, int32_t *iperm, int *bad, cudaStream_t st);
cudaError_t launch_perm_degrees(const int64_t *rowptr, const int32_t *perm, int64_t n, int32_t *deg,
                                cudaStream_t st);
cudaError_t permute_pattern(const int64_t *rowptr, const int32_t *colidx, const int32_t *perm,
                            const int32_t *iperm, int64_t n, int64_t nnz, const int64_t *new_rowptr,
                            int32_t *new_colidx, cudaStream_t st);

// extract.cu
struct ExtractParams {
  const uint32_t *is_ro;
  uint32_t *is;
  int32_t n, s0, s_end, G, nchunks;  // nchunks = ceil(n / extract_sub_columns())
  uint32_t *cntL, *cntU;     // [G][nchunks][32] counts, then exclusive prefixes
  int64_t *rowL, *rowU;      // [C] row start offsets (relative to the batch)
  int64_t *totals;           // [2] batch totals (L, U incl. diagonal)
  int64_t *L_rowptr, *U_rowptr;  // global output row pointers (row_begin based)
  int32_t row_begin;
  int64_t baseL, baseU;      // global offsets of the batch's first row
  int32_t *L_out, *U_out;    // global colidx arrays
};
cudaError_t launch_extract_count(const ExtractParams &e, cudaStream_t st);
cudaError_t launch_extract_scan(const ExtractParams &e, cudaStream_t st);
cudaError_t launch_extract_write(const ExtractParams &e, cudaStream_t st);
int extract_sub_columns();  // columns per extraction warp unit

// supernode.cu + utilities
cudaError_t launch_validate(const int64_t *rowptr64, const int32_t *colidx, int64_t n,
                            int64_t nnz, int32_t *rowptr32, int *err_flag, unsigned int *bw,
                            cudaStream_t st);
cudaError_t launch_supno(const int32_t *sn_start, int64_t nsuper, int32_t row_begin, int32_t *supno,
                         cudaStream_t st);
cudaError_t launch_count_offdiag(const int32_t *rowptr, const int32_t *colidx, const RowMap &m,
                                 int32_t rows, unsigned long long *out, cudaStream_t st);
// flags: [3 rows] scratch; [0, rows) Phase-I bits, [rows, 2 rows) leaders,
// [2 rows, 3 rows) the cap-only successor table (free again on return)
cudaError_t launch_supernode_flags(const int64_t *L_rowptr, const int32_t *L_colidx,
                                   const int64_t *U_rowptr, const RowMap &m, int32_t rows,
                                   int32_t chunk, int32_t cap_only, int32_t *flags, cudaStream_t st);
// exclusive scans (int32 -> int32 / int32 -> int64); total -> *total
cudaError_t scan_exclusive_i32(const int32_t *in, int32_t *out, int64_t count, int32_t *total,
                               void *tmp, size_t tmp_bytes, cudaStream_t st);
cudaError_t scan_exclusive_i32_i64(const int32_t *in, int64_t *out, int64_t count, int64_t *total,
                                   void *tmp, size_t tmp_bytes, cudaStream_t st);
size_t scan_tmp_bytes(int64_t count);  // enough for either scan
cudaError_t launch_supernode_stitch(const int64_t *U_rowptr, const int64_t *L_rowptr,
                                    const int32_t *L_colidx, int32_t rb, int32_t he,
                                    int64_t prev_nnzU, int32_t prev_leader, const int32_t *sn_start,
                                    int64_t nsuper, int32_t *out, cudaStream_t st);
// cap-only rule: re-scan from rb until the scan starts a block at a row that
// already leads one (or row_end); out [3 + rows]: [0] new leaders, [1] old
// leaders below the meeting row, [2] the meeting row, [3..] the new leaders
cudaError_t launch_supernode_stitch_cap(const int64_t *U_rowptr, const int64_t *L_rowptr,
                                        const int32_t *L_colidx, int32_t rb, int32_t re, int32_t cap,
                                        int64_t prev_nnzU, int32_t prev_leader,
                                        const int32_t *sn_start, int64_t nsuper, int32_t *out,
                                        cudaStream_t st);
cudaError_t launch_audit(const int32_t *A_rowptr, const int32_t *A_colidx, const int64_t *L_rowptr,
                         const int32_t *L_colidx, const int64_t *U_rowptr, const int32_t *U_colidx,
                         const int32_t *sn_start, const int32_t *nsuper, const RowMap &m, int32_t rows,
                         int32_t n, int32_t chunk, int32_t cap_only, int *err, cudaStream_t st);
cudaError_t launch_rowinfo(const int64_t *L_rowptr, const int32_t *L_colidx, const int64_t *U_rowptr,
                          const RowMap &m, int32_t rows, int32_t chunk, int32_t *nnzU,
                          uint32_t *lmask, cudaStream_t st);
cudaError_t launch_supernode_gathered(const RowMap &m, int32_t chunk, const int32_t *nnzU_all,
                                      const uint32_t *lmask_all, int64_t stride, int32_t *leader,
                                      cudaStream_t st);
cudaError_t launch_supernode_scatter(const int32_t *flags, const int32_t *pos, const RowMap &m,
                                     int32_t rows, const int32_t *total, int32_t *sn_start,
                                     cudaStream_t st);

// ELL copy of the adjacency for the solo kernel's id order (rows <= 8
// entries): ell[8 v + j] = j-th neighbour of v, -1 padded
cudaError_t launch_ell_build(const int32_t *rowptr, const int32_t *colidx, int32_t n, int32_t *ell,
                             cudaStream_t st);

// ------------------------------------------------------------- helpers
// Row `lane` of a 32x32 bit matrix in, column `lane` out (bit j of the result
// = bit `lane` of row j): swap off-diagonal blocks at widths 16..1
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int j = 16 >> i;
    const uint32_t m = masks[i];
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// bits of a 32-column word below / above column d (d = source - first column):
// lm = columns < d (entries of L), um = columns > d (entries of U)
__device__ __forceinline__ void split_masks(int d, uint32_t &lm, uint32_t &um) {
  lm = d <= 0 ? 0u : (d >= 32 ? 0xFFFFFFFFu : ((1u << d) - 1u));
  um = d < 0 ? 0xFFFFFFFFu : (d >= 31 ? 0u : (0xFFFFFFFFu << (d + 1)));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace gsofa
