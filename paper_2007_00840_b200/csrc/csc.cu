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
