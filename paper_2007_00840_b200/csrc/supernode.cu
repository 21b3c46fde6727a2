// supernode.cu -- T3 supernode detection (Definition def:T3) with the
// paper's two-phase SIMT design, plus input validation, the
// off-diagonal count of A and a device-wide exclusive scan.
//
// Phase I (one thread per row): bit[s] = nnz(U(s,:)) == nnz(U(s-1,:)) - 1 and
//   s is not a chunk start (chunks of chunk_size rows never share a supernode,
//   P:640).  Rows with bit 0 are the Phase-I leaders ("queue" of P:609).
// Phase II (one thread per Phase-I leader): the leader r grows through the
//   following run of bit-1 rows while L(s, r) != 0 (binary search in the sorted
//   row s of L); a rejected row becomes a new leader and growth continues from
//   it ("continue this process until no supernode grows").  Runs
//   between Phase-I leaders are independent, which is the parallelism the
//   paper's first phase exposes.
#include <climits>

#include "gsofa_internal.cuh"

namespace gsofa {

namespace {
constexpr uint32_t kFull = 0xFFFFFFFFu;

// CSR checks + int64 -> int32 row pointers; with bw != NULL also the
// bandwidth max |i - j| of A (bw[0]) and the largest row length (bw[2]) for
// GSOFA_SCHEDULE_AUTO, taken only from rows that passed the row-pointer
// check, so a malformed rowptr never leads to a read outside colidx
__global__ void validate_kernel(const int64_t *rowptr64, const int32_t *colidx, int64_t n,
                                int64_t nnz, int32_t *rowptr32, int *err, unsigned int *bw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned int m = 0, dg = 0;
  if (i <= n) {
    const int64_t a = rowptr64[i];
    rowptr32[i] = (int32_t)a;
    if (i == 0 && a != 0) atomicOr(err, 1);
    if (i == n) {
      if (a != nnz) atomicOr(err, 1);
    } else {
      const int64_t b = rowptr64[i + 1];
      if (b < a || a < 0 || b > nnz) {
        atomicOr(err, 1);
      } else {
        dg = (unsigned int)(b - a > INT32_MAX ? INT32_MAX : b - a);
        int32_t prev = -1;
        for (int64_t e = a; e < b; ++e) {
          const int32_t c = colidx[e];
          if (c < 0 || c >= n) atomicOr(err, 2);
          if (c <= prev) atomicOr(err, 4);
          prev = c;
        }
        if (b > a) {  // columns ascend: the extremes are the first and last entries
          const int64_t d0 = i - (int64_t)colidx[a], d1 = (int64_t)colidx[b - 1] - i;
          int64_t d = d0 > d1 ? d0 : d1;
          if (d < 0) d = 0;
          if (d > INT32_MAX) d = INT32_MAX;
          m = (unsigned int)d;
        }
      }
    }
  }
  if (bw) {
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    dg = __reduce_max_sync(0xFFFFFFFFu, dg);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(bw, m);
    if ((threadIdx.x & 31) == 0 && dg) atomicMax(bw + 2, dg);
  }
}

__global__ void offdiag_kernel(const int32_t *rowptr, const int32_t *colidx, RowMap m,
                               int32_t rows, unsigned long long *out) {
  __shared__ unsigned long long ws[32];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (k < rows) {
    const int i = m.row(k);
    const int a = rowptr[i], b = rowptr[i + 1];
    c = (unsigned long long)(b - a);
    for (int e = a; e < b; ++e) c -= (colidx[e] == i);
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) c += __shfl_xor_sync(kFull, c, d);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    atomicAdd(out, t);
  }
}

__device__ __forceinline__ bool row_contains(const int32_t *cols, int64_t a, int64_t b,
                                             int32_t key) {
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    const int32_t v = cols[m];
    if (v == key) return true;
    if (v < key) a = m + 1;
    else b = m;
  }
  return false;
}

// Phase I: bit[k] = 1 iff row s = row_begin + k satisfies requirement (i)
// against s - 1 (and, under the forced-break rule, s is not a chunk start)
__global__ void sn_phase1_kernel(const int64_t *U_rowptr, RowMap m, int32_t rows,
                                 int32_t chunk, int32_t cap_only, int32_t *bit) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows) return;
  const int32_t s = m.row(k);
  int b = 0;
  // (interleaved rows: units start at multiples of chunk, so row k - 1 is
  // row s - 1 whenever s is not a chunk start)
  if (k != 0 && (cap_only || s % chunk != 0)) {
    const int64_t nu = U_rowptr[k + 1] - U_rowptr[k];
    const int64_t np = U_rowptr[k] - U_rowptr[k - 1];
    b = (nu == np - 1);
  }
  bit[k] = b;
}

// Phase II: each Phase-I leader grows through its run of bit-1 rows
__global__ void sn_phase2_kernel(const int64_t *L_rowptr, const int32_t *L_colidx, RowMap m,
                                 int32_t rows, const int32_t *bit, int32_t *leader) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows) return;
  if (bit[k]) return;  // not a Phase-I leader
  leader[k] = 1;
  int32_t r = m.row(k);  // (a run of bit-1 rows never leaves its unit)
  for (int kt = k + 1; kt < rows && bit[kt]; ++kt) {
    if (row_contains(L_colidx, L_rowptr[kt], L_rowptr[kt + 1], r)) {
      leader[kt] = 0;  // joins the supernode led by r (Def. def:T3 (ii))
    } else {
      leader[kt] = 1;  // rejected: starts a new supernode
      r = m.row(kt);
    }
  }
}

// Cap-only rule: chunk_size bounds the block size but
// forces no break, so a run of bit-1 rows may be longer than the cap and the
// greedy scan inside it is a chain of leaders.  Two steps keep the chain off
// the binary searches:
//   sn_next_kernel (one warp per row r as a would-be leader): nxt[r] = the
//     first row t in (r, r + cap] that cannot join r's block -- t = r + cap,
//     t = row_end, bit[t] = 0, or L(t, r) = 0 -- 32 candidate rows per probe;
//     also clears leader[r]
//   sn_walk_kernel (one thread per Phase-I leader, i.e. bit 0): follows
//     r -> nxt[r] through its run and marks every leader on the way; the
//     walk ends at the next Phase-I leader (that thread's run) or row_end.
__global__ void sn_next_kernel(const int64_t *L_rowptr, const int32_t *L_colidx, int32_t row_begin,
                               int32_t row_end, int32_t cap, const int32_t *bit, int32_t *nxt,
                               int32_t *leader) {
  const int lane = threadIdx.x & 31;
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int32_t rows = row_end - row_begin;
  if (k >= rows) return;
  const int32_t r = row_begin + (int32_t)k;
  const int32_t lim = (int32_t)min((int64_t)row_end, (int64_t)r + cap);
  int32_t res = lim;
  for (int32_t t0 = r + 1; t0 < lim; t0 += 32) {
    const int32_t t = t0 + lane;
    bool fail = false;
    if (t < lim) {
      const int kt = t - row_begin;
      fail = !bit[kt] || !row_contains(L_colidx, L_rowptr[kt], L_rowptr[kt + 1], r);
    }
    const uint32_t b = __ballot_sync(kFull, fail);
    if (b) {
      res = t0 + __ffs(b) - 1;
      break;
    }
  }
  if (lane == 0) {
    nxt[k] = res - row_begin;
    leader[k] = 0;
  }
}

__global__ void sn_walk_kernel(int32_t rows, const int32_t *bit, const int32_t *nxt,
                               int32_t *leader) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows || bit[k]) return;
  int32_t r = k;
  leader[r] = 1;
  for (;;) {
    const int32_t t = nxt[r];
    if (t >= rows || !bit[t]) break;  // the next run (its own thread) or the end
    leader[t] = 1;
    r = t;
  }
}

// Cap-only stitch: one warp re-runs the greedy scan over [rb, re) from the
// predecessor's tail, testing 32 rows per probe against the current leader r
// (t - r < cap, requirement (i) against row t - 1, L(t, r) != 0).  The first
// row that cannot join becomes a leader; if it already leads a provisional
// block the two scans agree from there on (same leader, same rows) and the
// re-scan stops.  out: [0] new leaders, [1] provisional leaders below the
// meeting row, [2] the meeting row, [3..] the new leaders.
__global__ void sn_stitch_cap_kernel(const int64_t *U_rowptr, const int64_t *L_rowptr,
                                     const int32_t *L_colidx, int32_t rb, int32_t re, int32_t cap,
                                     int64_t prev_nnzU, int32_t prev_leader,
                                     const int32_t *sn_start, int64_t nsuper, int32_t *out) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int32_t r = prev_leader, s = rb, meet = re;
  int nc = 0;
  while (s < re) {
    const int32_t t = s + lane;
    bool fail = false;
    if (t < re) {
      const int k = t - rb;
      const int64_t nu = U_rowptr[k + 1] - U_rowptr[k];
      const int64_t np = k == 0 ? prev_nnzU : U_rowptr[k] - U_rowptr[k - 1];
      fail = !((int64_t)t - r < cap && nu == np - 1 &&
               row_contains(L_colidx, L_rowptr[k], L_rowptr[k + 1], r));
    }
    const uint32_t b = __ballot_sync(kFull, fail);
    if (!b) {
      s += 32;
      continue;
    }
    const int32_t lead = s + __ffs(b) - 1;
    // does lead already start a provisional block?  (binary search)
    int64_t lo = 0, hi = nsuper;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (sn_start[m] < lead) lo = m + 1;
      else hi = m;
    }
    if (lo < nsuper && sn_start[lo] == lead) {
      meet = lead;
      break;
    }
    if (lane == 0) out[3 + nc] = lead;
    ++nc;
    r = lead;
    s = lead + 1;
  }
  if (lane == 0) {
    int64_t lo = 0, hi = nsuper;  // provisional leaders below meet
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (sn_start[m] < meet) lo = m + 1;
      else hi = m;
    }
    out[0] = nc;
    out[1] = (int32_t)lo;
    out[2] = meet;
  }
}

// ---- finer-than-chunk row interleave (gsofa_interleave): the parts
// exchange what Def. def:T3 needs about each row, then every part runs the
// greedy scan per chunk over all rows and keeps its own leaders.
// rowinfo (one thread per local row k, global row s): nnz(U(s,:)) and the
// mask of candidate leaders r = s - d inside s's chunk with L(s, r) != 0.
__global__ void rowinfo_kernel(const int64_t *L_rowptr, const int32_t *L_colidx,
                               const int64_t *U_rowptr, RowMap m, int32_t rows, int32_t chunk,
                               int32_t W, int32_t *nnzU, uint32_t *lmask) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows) return;
  const int32_t s = m.row(k), cs = s - s % chunk;
  nnzU[k] = (int32_t)(U_rowptr[k + 1] - U_rowptr[k]);
  uint32_t *mk = lmask + (size_t)k * W;
  for (int w = 0; w < W; ++w) mk[w] = 0u;
  int64_t a = L_rowptr[k], b = L_rowptr[k + 1];
  while (a < b) {  // first entry >= cs
    const int64_t mid = (a + b) >> 1;
    if (L_colidx[mid] < cs) a = mid + 1;
    else b = mid;
  }
  for (int64_t e = a; e < L_rowptr[k + 1]; ++e) {
    const int32_t d = s - L_colidx[e];  // 1 .. s - cs
    mk[d >> 5] |= 1u << (d & 31);
  }
}

// one thread per chunk: the greedy Def. def:T3 scan over the
// chunk's rows, wherever they live (part p = unit % N, local index from the
// unit); leader[local] for this part's rows
__global__ void sn_gathered_kernel(RowMap m, int32_t chunk, int32_t W, const int32_t *nnzU_all,
                                   const uint32_t *lmask_all, int64_t stride, int32_t *leader) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t cs64 = (int64_t)m.rb + c * chunk;
  if (cs64 >= m.re) return;
  const int32_t cs = (int32_t)cs64, ce = (int32_t)min((int64_t)m.re, cs64 + chunk);
  int32_t r = cs;
  int64_t pn = 0;
  for (int32_t s = cs; s < ce; ++s) {
    const int32_t off = s - m.rb, u = off / m.U;
    const int32_t part = u % m.N;
    const int64_t idx = (int64_t)part * stride + (int64_t)(u / m.N) * m.U + (off - u * m.U);
    const int64_t nu = nnzU_all[idx];
    bool join = false;
    if (s != cs) {
      const int32_t d = s - r;
      join = nu == pn - 1 && ((lmask_all[idx * W + (d >> 5)] >> (d & 31)) & 1u);
    }
    if (!join) r = s;
    if (part == m.q) leader[idx - (int64_t)part * stride] = join ? 0 : 1;
    pn = nu;
  }
}

// Supernode-boundary stitch (multi-range runs): the head rows [rb, he) of a
// range that starts inside a chunk were scanned as if rb started a block;
// re-run the greedy Def. def:T3 scan over them from the
// predecessor's tail (its last row's nnz(U) and the leader of its block).
// One thread: at most chunk_size - 1 rows.  out: [0] new head leaders,
// [1] old head leaders (sn_start entries < he), [2..] the new leaders.
__global__ void sn_stitch_kernel(const int64_t *U_rowptr, const int64_t *L_rowptr,
                                 const int32_t *L_colidx, int32_t rb, int32_t he, int64_t prev_nnzU,
                                 int32_t prev_leader, const int32_t *sn_start, int64_t nsuper,
                                 int32_t *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int32_t r = prev_leader;
  int64_t pn = prev_nnzU;
  int nc = 0;
  for (int32_t s = rb; s < he; ++s) {
    const int k = s - rb;
    const int64_t nu = U_rowptr[k + 1] - U_rowptr[k];
    // (i) nnz(U(s,:)) = nnz(U(s-1,:)) - 1 and (ii) L(s, r) != 0
    const bool join = nu == pn - 1 && row_contains(L_colidx, L_rowptr[k], L_rowptr[k + 1], r);
    if (!join) {
      r = s;
      out[2 + nc++] = s;
    }
    pn = nu;
  }
  int oc = 0;
  while (oc < nsuper && sn_start[oc] < he) ++oc;
  out[0] = nc;
  out[1] = oc;
}

// Checked mode (gsofa_opts.checked): audit of the finished
// structure, one warp per row s = row_begin + r.  Bits of *err:
//   1  an L row is not strictly increasing or not strictly below s
//   2  a U row does not start with s or is not strictly increasing above s
//   4  an entry of A is missing from L+U (pattern(A) must be a subset)
//   8  an interior supernode row violates Def. def:T3 against its leader
//  16  a leader (not a chunk start, not row_begin) could have joined the
//      previous block (the greedy scan would not have split there)
__global__ void audit_kernel(const int32_t *A_rowptr, const int32_t *A_colidx, const int64_t *L_rowptr,
                             const int32_t *L_colidx, const int64_t *U_rowptr, const int32_t *U_colidx,
                             const int32_t *sn_start, const int32_t *nsuper_p, RowMap m,
                             int32_t rows, int32_t n, int32_t chunk, int32_t cap_only, int *err) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int32_t s = m.row(r);
  const int64_t la = L_rowptr[r], lb = L_rowptr[r + 1], ua = U_rowptr[r], ub = U_rowptr[r + 1];
  int bad = 0;
  for (int64_t e = la + lane; e < lb; e += 32) {
    const int32_t c = L_colidx[e];
    if (c < 0 || c >= s || (e > la && L_colidx[e - 1] >= c)) bad |= 1;
  }
  if (ub <= ua || U_colidx[ua] != s) bad |= 2;
  for (int64_t e = ua + 1 + lane; e < ub; e += 32) {
    const int32_t c = U_colidx[e];
    if (c <= s || c >= n || U_colidx[e - 1] >= c) bad |= 2;
  }
  for (int32_t e = A_rowptr[s] + lane; e < A_rowptr[s + 1]; e += 32) {
    const int32_t c = A_colidx[e];
    if (c == s) continue;
    const bool found = c < s ? row_contains(L_colidx, la, lb, c) : row_contains(U_colidx, ua + 1, ub, c);
    if (!found) bad |= 4;
  }
  if (lane == 0 && nsuper_p) {  // (no supernodes yet: deferred to the exchange)
    // leader of s: the last sn_start entry <= s
    const int32_t ns = *nsuper_p;
    int32_t lo = 0, hi = ns;
    while (hi - lo > 1) {
      const int32_t m = (lo + hi) >> 1;
      if (sn_start[m] <= s) lo = m;
      else hi = m;
    }
    const int32_t lead = sn_start[lo];
    if (s != lead) {
      const int64_t nu = ub - ua, np = ua - U_rowptr[r - 1];
      const bool brk = cap_only ? s - lead >= chunk : s % chunk == 0;
      if (brk || nu != np - 1 || !row_contains(L_colidx, la, lb, lead)) bad |= 8;
    } else if (r != 0 && (cap_only || s % chunk != 0)) {
      int32_t lo2 = 0, hi2 = ns;  // leader of s - 1
      while (hi2 - lo2 > 1) {
        const int32_t m = (lo2 + hi2) >> 1;
        if (sn_start[m] <= s - 1) lo2 = m;
        else hi2 = m;
      }
      const int64_t nu = ub - ua, np = ua - U_rowptr[r - 1];
      const bool room = !cap_only || s - sn_start[lo2] < chunk;
      if (room && nu == np - 1 && row_contains(L_colidx, la, lb, sn_start[lo2])) bad |= 16;
    }
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (lane == 0 && bad) atomicOr(err, bad);
}

__global__ void sn_scatter_kernel(const int32_t *flags, const int32_t *pos, RowMap m, int32_t rows,
                                  const int32_t *total, int32_t *sn_start) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) sn_start[*total] = rows > 0 ? m.row(rows - 1) + 1 : m.rb;  // sentinel: after the last row
  if (k >= rows) return;
  if (flags[k]) sn_start[pos[k]] = m.row(k);
}

// ---- exclusive scan, 4096 items per block, recursive on block sums
constexpr int kScanThreads = 1024, kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kScanThreads) scan_tile_kernel(const Tin *in, Tout *out,
                                                                 int64_t count, Tout *sums) {
  __shared__ Tout ws[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)tid * kScanItems;
  Tout v[kScanItems];
  Tout t = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < count) ? (Tout)in[base + i] : (Tout)0;
    t += v[i];
  }
  Tout x = t;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Tout y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    Tout z = ws[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const Tout y = __shfl_up_sync(kFull, z, d);
      if (lane >= d) z += y;
    }
    ws[lane] = z;
  }
  __syncthreads();
  Tout run = x - t + (wid ? ws[wid - 1] : (Tout)0);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < count) out[base + i] = run;
    run += v[i];
  }
  if (tid == kScanThreads - 1) sums[blockIdx.x] = run;
}

template <typename T>
__global__ void scan_add_kernel(T *out, int64_t count, const T *offs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] += offs[i / kScanTile];
}

template <typename Tin, typename Tout>
cudaError_t scan_rec(const Tin *in, Tout *out, int64_t count, Tout *total, Tout *tmp,
                     cudaStream_t st) {
  const int64_t nb = (count + kScanTile - 1) / kScanTile;
  Tout *sums = tmp, *sums_scan = tmp + nb;
  scan_tile_kernel<Tin, Tout><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, count, sums);
  if (nb == 1) {
    cudaMemcpyAsync(total, sums, sizeof(Tout), cudaMemcpyDeviceToDevice, st);
    return cudaGetLastError();
  }
  cudaError_t e = scan_rec<Tout, Tout>(sums, sums_scan, nb, total, tmp + 2 * nb, st);
  if (e != cudaSuccess) return e;
  scan_add_kernel<Tout><<<(unsigned)((count + 255) / 256), 256, 0, st>>>(out, count, sums_scan);
  return cudaGetLastError();
}
}  // namespace

size_t scan_tmp_bytes(int64_t count) {
  size_t tot = 0;
  int64_t c = count;
  do {
    const int64_t nb = (c + kScanTile - 1) / kScanTile;
    tot += 2 * (size_t)nb;
    c = nb;
  } while (c > 1);
  return (tot + 16) * sizeof(int64_t);
}

cudaError_t scan_exclusive_i32(const int32_t *in, int32_t *out, int64_t count, int32_t *total,
                               void *tmp, size_t tmp_bytes, cudaStream_t st) {
  if (count <= 0) return cudaMemsetAsync(total, 0, sizeof(int32_t), st);
  if (tmp_bytes < scan_tmp_bytes(count)) return cudaErrorInvalidValue;
  return scan_rec<int32_t, int32_t>(in, out, count, total, (int32_t *)tmp, st);
}

cudaError_t scan_exclusive_i32_i64(const int32_t *in, int64_t *out, int64_t count, int64_t *total,
                                   void *tmp, size_t tmp_bytes, cudaStream_t st) {
  if (count <= 0) return cudaMemsetAsync(total, 0, sizeof(int64_t), st);
  if (tmp_bytes < scan_tmp_bytes(count)) return cudaErrorInvalidValue;
  return scan_rec<int32_t, int64_t>(in, out, count, total, (int64_t *)tmp, st);
}

// SuperLU-style supno (xsup = sn_start): supno[i - row_begin] = the index of
// the supernode holding row i, i.e. k with sn_start[k] <= i < sn_start[k+1];
// one thread per supernode writes its rows
__global__ void supno_kernel(const int32_t *sn_start, int64_t nsuper, int32_t row_begin,
                             int32_t *supno) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nsuper) return;
  for (int32_t i = sn_start[k]; i < sn_start[k + 1]; ++i) supno[i - row_begin] = (int32_t)k;
}

cudaError_t launch_supno(const int32_t *sn_start, int64_t nsuper, int32_t row_begin, int32_t *supno,
                         cudaStream_t st) {
  if (nsuper <= 0) return cudaSuccess;
  supno_kernel<<<(unsigned)((nsuper + 255) / 256), 256, 0, st>>>(sn_start, nsuper, row_begin, supno);
  return cudaGetLastError();
}

cudaError_t launch_validate(const int64_t *rowptr64, const int32_t *colidx, int64_t n,
                            int64_t nnz, int32_t *rowptr32, int *err_flag, unsigned int *bw,
                            cudaStream_t st) {
  validate_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(rowptr64, colidx, n, nnz,
                                                                   rowptr32, err_flag, bw);
  return cudaGetLastError();
}

cudaError_t launch_count_offdiag(const int32_t *rowptr, const int32_t *colidx, const RowMap &m,
                                 int32_t rows, unsigned long long *out, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  offdiag_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(rowptr, colidx, m, rows, out);
  return cudaGetLastError();
}

cudaError_t launch_supernode_flags(const int64_t *L_rowptr, const int32_t *L_colidx,
                                   const int64_t *U_rowptr, const RowMap &m, int32_t rows,
                                   int32_t chunk, int32_t cap_only, int32_t *flags, cudaStream_t st) {
  // flags has room for 3 * rows: [0, rows) = Phase-I bits, [rows, 2 rows) =
  // leaders, [2 rows, 3 rows) = cap-only successor table (cap-only rows are
  // never interleaved: m.row(k) = rb + k)
  if (rows <= 0) return cudaSuccess;
  const unsigned nb = (unsigned)((rows + 255) / 256);
  sn_phase1_kernel<<<nb, 256, 0, st>>>(U_rowptr, m, rows, chunk, cap_only, flags);
  if (cap_only) {
    sn_next_kernel<<<(unsigned)(((int64_t)rows * 32 + 255) / 256), 256, 0, st>>>(
        L_rowptr, L_colidx, m.rb, m.rb + rows, chunk, flags, flags + 2 * rows, flags + rows);
    sn_walk_kernel<<<nb, 256, 0, st>>>(rows, flags, flags + 2 * rows, flags + rows);
  } else {
    sn_phase2_kernel<<<nb, 256, 0, st>>>(L_rowptr, L_colidx, m, rows, flags, flags + rows);
  }
  return cudaGetLastError();
}

cudaError_t launch_supernode_scatter(const int32_t *flags, const int32_t *pos, const RowMap &m,
                                     int32_t rows, const int32_t *total, int32_t *sn_start,
                                     cudaStream_t st) {
  sn_scatter_kernel<<<(unsigned)((rows + 255) / 256 + 1), 256, 0, st>>>(flags, pos, m, rows, total,
                                                                        sn_start);
  return cudaGetLastError();
}

cudaError_t launch_supernode_stitch(const int64_t *U_rowptr, const int64_t *L_rowptr,
                                    const int32_t *L_colidx, int32_t rb, int32_t he,
                                    int64_t prev_nnzU, int32_t prev_leader, const int32_t *sn_start,
                                    int64_t nsuper, int32_t *out, cudaStream_t st) {
  sn_stitch_kernel<<<1, 32, 0, st>>>(U_rowptr, L_rowptr, L_colidx, rb, he, prev_nnzU, prev_leader,
                                     sn_start, nsuper, out);
  return cudaGetLastError();
}

cudaError_t launch_supernode_stitch_cap(const int64_t *U_rowptr, const int64_t *L_rowptr,
                                        const int32_t *L_colidx, int32_t rb, int32_t re, int32_t cap,
                                        int64_t prev_nnzU, int32_t prev_leader,
                                        const int32_t *sn_start, int64_t nsuper, int32_t *out,
                                        cudaStream_t st) {
  sn_stitch_cap_kernel<<<1, 32, 0, st>>>(U_rowptr, L_rowptr, L_colidx, rb, re, cap, prev_nnzU,
                                         prev_leader, sn_start, nsuper, out);
  return cudaGetLastError();
}

cudaError_t launch_rowinfo(const int64_t *L_rowptr, const int32_t *L_colidx, const int64_t *U_rowptr,
                          const RowMap &m, int32_t rows, int32_t chunk, int32_t *nnzU,
                          uint32_t *lmask, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  rowinfo_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(
      L_rowptr, L_colidx, U_rowptr, m, rows, chunk, (chunk + 31) / 32, nnzU, lmask);
  return cudaGetLastError();
}

cudaError_t launch_supernode_gathered(const RowMap &m, int32_t chunk, const int32_t *nnzU_all,
                                      const uint32_t *lmask_all, int64_t stride, int32_t *leader,
                                      cudaStream_t st) {
  const int64_t nch = ((int64_t)m.re - m.rb + chunk - 1) / chunk;
  if (nch <= 0) return cudaSuccess;
  sn_gathered_kernel<<<(unsigned)((nch + 127) / 128), 128, 0, st>>>(m, chunk, (chunk + 31) / 32,
                                                                    nnzU_all, lmask_all, stride, leader);
  return cudaGetLastError();
}

cudaError_t launch_audit(const int32_t *A_rowptr, const int32_t *A_colidx, const int64_t *L_rowptr,
                         const int32_t *L_colidx, const int64_t *U_rowptr, const int32_t *U_colidx,
                         const int32_t *sn_start, const int32_t *nsuper, const RowMap &m, int32_t rows,
                         int32_t n, int32_t chunk, int32_t cap_only, int *err, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  audit_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(A_rowptr, A_colidx, L_rowptr, L_colidx,
                                                           U_rowptr, U_colidx, sn_start, nsuper,
                                                           m, rows, n, chunk, cap_only, err);
  return cudaGetLastError();
}

}  // namespace gsofa
