// csc.cu -- L in compressed sparse column form (
// north_star: "L and U patterns as CSR/CSC").  SuperLU-style numeric
// factorization consumes L by columns; the traversal produces it by rows
// (one source row at a time), so this is a format conversion of the
// finished structure, not part of the traversal.
//
//   1. expand the row pointers: row[e] = row_begin + r for every entry e of row r
//   2. stable radix sort of (column, row) pairs by column (radix.cu, 64-bit
//      counts: C5's L has 2.2e9 entries): entries come in row-major order, so
//      the rows of each column stay ascending
//   3. col_ptr[j] = first position whose column is >= j (binary search)

#include "gsofa_internal.cuh"

namespace gsofa {
namespace {

__global__ void row_expand_kernel(const int64_t *L_rowptr, int64_t rows, int64_t row_begin,
                                  int32_t *row_of) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t a = L_rowptr[r], b = L_rowptr[r + 1];
  for (int64_t e = a + lane; e < b; e += 32) row_of[e] = (int32_t)(row_begin + r);
}

__global__ void colptr_kernel(const int32_t *cols, int64_t nnz, int64_t n, int64_t *col_ptr) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j > n) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (cols[m] < j) lo = m + 1;
    else hi = m;
  }
  col_ptr[j] = lo;
}

}  // namespace

cudaError_t l_rows_to_csc(const int64_t *L_rowptr, const int32_t *L_colidx, int64_t rows,
                          int64_t row_begin, int64_t n, int64_t nnz, int64_t *col_ptr,
                          int32_t *row_idx, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  uint32_t *ka = nullptr, *kb = nullptr;
  int32_t *vtmp = nullptr;
  void *hist = nullptr;
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
  const int passes = (bits + 7) / 8;
  const int grid = radix_grid();
  uint32_t *sorted = nullptr;
  if (nnz > 0) {
    if ((e = cudaMallocAsync((void **)&ka, (size_t)nnz * 4, st)) != cudaSuccess) goto done;
    if ((e = cudaMallocAsync((void **)&kb, (size_t)nnz * 4, st)) != cudaSuccess) goto done;
    if ((e = cudaMallocAsync((void **)&vtmp, (size_t)nnz * 4, st)) != cudaSuccess) goto done;
    if ((e = cudaMallocAsync(&hist, radix_hist_bytes(grid), st)) != cudaSuccess) goto done;
    if ((e = cudaMemcpyAsync(ka, L_colidx, (size_t)nnz * 4, cudaMemcpyDeviceToDevice, st)) !=
        cudaSuccess)
      goto done;
    {
      // the row values ping-pong between row_idx and vtmp: start where an
      // odd / even number of passes makes them end in row_idx
      int32_t *v0 = (passes & 1) ? vtmp : row_idx, *v1 = (passes & 1) ? row_idx : vtmp;
      row_expand_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(L_rowptr, rows, row_begin, v0);
      if ((e = cudaGetLastError()) != cudaSuccess) goto done;
      bool in_tmp = false;
      if ((e = radix_sort_pairs_u32(ka, v0, kb, v1, nnz, bits, hist, grid, st, &in_tmp)) !=
          cudaSuccess)
        goto done;
      sorted = in_tmp ? kb : ka;
    }
  }
  colptr_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>((const int32_t *)sorted, nnz, n,
                                                                 col_ptr);
  e = cudaGetLastError();
done:
  if (hist) cudaFreeAsync(hist, st);
  if (ka) cudaFreeAsync(ka, st);
  if (kb) cudaFreeAsync(kb, st);
  if (vtmp) cudaFreeAsync(vtmp, st);
  return e;
}

}  // namespace gsofa

// ------------------------------------------------------------------ permute
// B = P A P^T for the ordering perm (new vertex i = old vertex perm[i]):
// B(i, j) != 0 iff A(perm[i], perm[j]) != 0.  Entries become 64-bit keys
// (i << bits | iperm[col]); one radix sort (radix.cu) orders them by row,
// then column.
namespace gsofa {
namespace {

__global__ void iperm_kernel(const int32_t *perm, int64_t n, int32_t *iperm, int *bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t p = perm[i];
  if (p < 0 || p >= n) {
    atomicOr(bad, 1);
    return;
  }
  if (atomicExch(iperm + p, (int32_t)i) != -1) atomicOr(bad, 2);  // p listed twice
}

__global__ void perm_keys_kernel(const int64_t *rowptr, const int32_t *colidx, const int32_t *perm,
                                 const int32_t *iperm, int64_t n, const int64_t *new_rowptr,
                                 int bits, unsigned long long *keys) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const int32_t r = perm[i];
  const int64_t a = rowptr[r], b = rowptr[r + 1], o = new_rowptr[i];
  for (int64_t e = a + lane; e < b; e += 32)
    keys[o + (e - a)] = ((unsigned long long)i << bits) | (uint32_t)iperm[colidx[e]];
}

__global__ void perm_degree_kernel(const int64_t *rowptr, const int32_t *perm, int64_t n,
                                   int32_t *deg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) deg[i] = (int32_t)(rowptr[perm[i] + 1] - rowptr[perm[i]]);
}

__global__ void perm_split_kernel(const unsigned long long *keys, int64_t nnz, int bits,
                                  int32_t *colidx) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) colidx[e] = (int32_t)(keys[e] & ((1ull << bits) - 1ull));
}

}  // namespace

// all pointers device.  launch_iperm: inverse permutation and a check
// (*bad: 1 = entry out of range, 2 = duplicate); only if *bad == 0 may the
// caller go on with launch_perm_degrees, scan the degrees into new_rowptr
// and call permute_pattern.
cudaError_t launch_iperm(const int32_t *perm, int64_t n, int32_t *iperm, int *bad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(iperm, 0xFF, (size_t)n * 4, st);
  if (e != cudaSuccess) return e;
  iperm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(perm, n, iperm, bad);
  return cudaGetLastError();
}

cudaError_t launch_perm_degrees(const int64_t *rowptr, const int32_t *perm, int64_t n, int32_t *deg,
                                cudaStream_t st) {
  perm_degree_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rowptr, perm, n, deg);
  return cudaGetLastError();
}

cudaError_t permute_pattern(const int64_t *rowptr, const int32_t *colidx, const int32_t *perm,
                            const int32_t *iperm, int64_t n, int64_t nnz, const int64_t *new_rowptr,
                            int32_t *new_colidx, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  void *hist = nullptr;
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
  const int grid = radix_grid();
  bool in_tmp = false;
  if (nnz == 0) return cudaSuccess;
  if ((e = cudaMallocAsync((void **)&k0, (size_t)nnz * 8, st)) != cudaSuccess) goto done;
  if ((e = cudaMallocAsync((void **)&k1, (size_t)nnz * 8, st)) != cudaSuccess) goto done;
  if ((e = cudaMallocAsync(&hist, radix_hist_bytes(grid), st)) != cudaSuccess) goto done;
  perm_keys_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(rowptr, colidx, perm, iperm, n, new_rowptr,
                                                             bits, k0);
  if ((e = cudaGetLastError()) != cudaSuccess) goto done;
  // one sort of (row << bits | column) keys: 2 * bits key bits
  if ((e = radix_sort_keys_u64(k0, k1, nnz, 2 * bits, hist, grid, st, &in_tmp)) != cudaSuccess)
    goto done;
  perm_split_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(in_tmp ? k1 : k0, nnz, bits,
                                                                   new_colidx);
  e = cudaGetLastError();
done:
  if (hist) cudaFreeAsync(hist, st);
  if (k0) cudaFreeAsync(k0, st);
  if (k1) cudaFreeAsync(k1, st);
  return e;
}

}  // namespace gsofa
