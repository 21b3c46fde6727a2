// csc.cu -- L in compressed sparse column form (
// north_star: "L and U patterns as CSR/CSC").  SuperLU-style numeric
// factorization consumes L by columns; the traversal produces it by rows
// (one source row at a time), so this is a format conversion of the
// finished structure, not part of the traversal.
//
//   1. expand the row pointers: row[e] = row_begin + r for every entry e of row r
//   2. stable radix sort of (column, row) pairs by column (CUB): entries come in
//      row-major order, so the rows of each column stay ascending
//   3. col_ptr[j] = first position whose column is >= j (binary search)
#include <cub/device/device_radix_sort.cuh>

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
  int32_t *keys_in = nullptr, *keys_out = nullptr, *vals_in = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
  if (nnz > 0) {
    if ((e = cudaMallocAsync((void **)&keys_in, (size_t)nnz * 4, st)) != cudaSuccess) goto done;
    if ((e = cudaMallocAsync((void **)&keys_out, (size_t)nnz * 4, st)) != cudaSuccess) goto done;
    if ((e = cudaMallocAsync((void **)&vals_in, (size_t)nnz * 4, st)) != cudaSuccess) goto done;
    if ((e = cudaMemcpyAsync(keys_in, L_colidx, (size_t)nnz * 4, cudaMemcpyDeviceToDevice, st)) !=
        cudaSuccess)
      goto done;
    row_expand_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(L_rowptr, rows, row_begin, vals_in);
    if ((e = cudaGetLastError()) != cudaSuccess) goto done;
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, vals_in, row_idx,
                                             nnz, 0, bits, st)) != cudaSuccess)
      goto done;
    if ((e = cudaMallocAsync(&tmp, tmp_bytes, st)) != cudaSuccess) goto done;
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, row_idx, nnz,
                                             0, bits, st)) != cudaSuccess)
      goto done;
  }
  colptr_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(keys_out, nnz, n, col_ptr);
  e = cudaGetLastError();
done:
  if (tmp) cudaFreeAsync(tmp, st);
  if (keys_in) cudaFreeAsync(keys_in, st);
  if (keys_out) cudaFreeAsync(keys_out, st);
  if (vals_in) cudaFreeAsync(vals_in, st);
  return e;
}

}  // namespace gsofa

// ------------------------------------------------------------------ permute
// B = P A P^T for the ordering perm (new vertex i = old vertex perm[i]):
// B(i, j) != 0 iff A(perm[i], perm[j]) != 0.  Entries become 64-bit keys
// (i << 32 | iperm[col]); one radix sort orders them by row, then column.
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
                                 unsigned long long *keys) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const int32_t r = perm[i];
  const int64_t a = rowptr[r], b = rowptr[r + 1], o = new_rowptr[i];
  for (int64_t e = a + lane; e < b; e += 32)
    keys[o + (e - a)] = ((unsigned long long)i << 32) | (uint32_t)iperm[colidx[e]];
}

__global__ void perm_degree_kernel(const int64_t *rowptr, const int32_t *perm, int64_t n,
                                   int32_t *deg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) deg[i] = (int32_t)(rowptr[perm[i] + 1] - rowptr[perm[i]]);
}

__global__ void perm_split_kernel(const unsigned long long *keys, int64_t nnz, int32_t *colidx) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) colidx[e] = (int32_t)(keys[e] & 0xFFFFFFFFull);
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
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
  if (nnz == 0) return cudaSuccess;
  if ((e = cudaMallocAsync((void **)&k0, (size_t)nnz * 8, st)) != cudaSuccess) goto done;
  if ((e = cudaMallocAsync((void **)&k1, (size_t)nnz * 8, st)) != cudaSuccess) goto done;
  perm_keys_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(rowptr, colidx, perm, iperm, n, new_rowptr,
                                                             k0);
  if ((e = cudaGetLastError()) != cudaSuccess) goto done;
  // one sort over row (high word) and column (low word) bits
  if ((e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, nnz, 0, 32 + bits, st)) !=
      cudaSuccess)
    goto done;
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st)) != cudaSuccess) goto done;
  if ((e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, k0, k1, nnz, 0, 32 + bits, st)) != cudaSuccess)
    goto done;
  perm_split_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(k1, nnz, new_colidx);
  e = cudaGetLastError();
done:
  if (tmp) cudaFreeAsync(tmp, st);
  if (k0) cudaFreeAsync(k0, st);
  if (k1) cudaFreeAsync(k1, st);
  return e;
}

}  // namespace gsofa
