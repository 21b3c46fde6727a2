// radix.cu -- stable LSD radix sort of (key, value) pairs, 8-bit digits,
// 64-bit item counts.  Used for the format conversions of §8(f) NEXT-3/4
// (L by columns, symmetric permutation); not on the traversal path.
//
// One pass per 8-bit digit (stable counting sort):
//   1. count: each of G persistent CTAs owns one contiguous chunk of the
//      input and builds its digit histogram in shared memory;
//   2. offsets: an exclusive scan over (digit, CTA) in digit-major order
//      gives every CTA the global start of each digit for its chunk;
//   3. scatter: each CTA re-reads its chunk in order, 1024 items at a time;
//      within a warp, the items with the same digit are ranked by lane
//      (__match_any_sync), across the 32 warps by a per-(warp, digit) prefix
//      in shared memory; the CTA's running digit cursors advance per round.
//      Input order is kept among equal digits, so the passes compose into a
//      stable sort.
#include <cstdint>

#include "gsofa_internal.cuh"

namespace gsofa {
namespace {

constexpr int kRadixThreads = 1024;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kBins = 256;

template <typename K>
__device__ __forceinline__ int digit_of(K k, int shift) {
  return (int)((k >> shift) & (K)0xFF);
}

template <typename K>
__global__ void __launch_bounds__(kRadixThreads) radix_count_kernel(const K *keys, int64_t n,
                                                                    int64_t chunk, int shift,
                                                                    unsigned long long *hist) {
  __shared__ unsigned int h[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0u;
  __syncthreads();
  const int64_t a = (int64_t)blockIdx.x * chunk, b = min(n, a + chunk);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) atomicAdd(&h[digit_of(keys[i], shift)], 1u);
  __syncthreads();
  // digit-major: hist[d * G + cta]
  for (int d = threadIdx.x; d < kBins; d += blockDim.x)
    hist[(size_t)d * gridDim.x + blockIdx.x] = h[d];
}

// exclusive scan of the G * 256 counts in place (one CTA; G * 256 is small)
__global__ void __launch_bounds__(kRadixThreads) radix_offsets_kernel(unsigned long long *hist,
                                                                      int64_t m) {
  __shared__ unsigned long long part[kRadixThreads];
  const int64_t per = (m + blockDim.x - 1) / blockDim.x;
  const int64_t a = (int64_t)threadIdx.x * per, b = min(m, a + per);
  unsigned long long s = 0;
  for (int64_t i = a; i < b; ++i) s += hist[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const unsigned long long v = part[t];
      part[t] = acc;
      acc += v;
    }
  }
  __syncthreads();
  unsigned long long acc = part[threadIdx.x];
  for (int64_t i = a; i < b; ++i) {
    const unsigned long long v = hist[i];
    hist[i] = acc;
    acc += v;
  }
}

template <typename K, bool kVals>
__global__ void __launch_bounds__(kRadixThreads) radix_scatter_kernel(
    const K *keys, const int32_t *vals, int64_t n, int64_t chunk, int shift,
    const unsigned long long *hist, K *keys_out, int32_t *vals_out) {
  __shared__ unsigned long long cursor[kBins];
  __shared__ unsigned int wcnt[kRadixWarps][kBins];  // per-warp digit counts -> prefixes
  __shared__ unsigned int tot[kBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kBins; d += blockDim.x)
    cursor[d] = hist[(size_t)d * gridDim.x + blockIdx.x];
  const int64_t a = (int64_t)blockIdx.x * chunk, b = min(n, a + chunk);
  for (int64_t base = a; base < b; base += kRadixThreads) {
    for (int i = threadIdx.x; i < kRadixWarps * kBins; i += blockDim.x) (&wcnt[0][0])[i] = 0u;
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    const bool ok = i < b;
    K k = 0;
    int32_t v = 0;
    int d = kBins;  // items past the end take no digit
    if (ok) {
      k = keys[i];
      if (kVals) v = vals[i];
      d = digit_of(k, shift);
    }
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const int rank = __popc(peers & lanemask_lt());
    if (ok && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    // per digit: exclusive prefix over the warps, and the round's total
    for (int dd = threadIdx.x; dd < kBins; dd += blockDim.x) {
      unsigned int acc = 0;
      for (int w = 0; w < kRadixWarps; ++w) {
        const unsigned int c = wcnt[w][dd];
        wcnt[w][dd] = acc;
        acc += c;
      }
      tot[dd] = acc;
    }
    __syncthreads();
    if (ok) {
      const unsigned long long o = cursor[d] + wcnt[warp][d] + rank;
      keys_out[o] = k;
      if (kVals) vals_out[o] = v;
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < kBins; dd += blockDim.x) cursor[dd] += tot[dd];
  }
}

template <typename K, bool kVals>
cudaError_t radix_sort_impl(K *keys, int32_t *vals, K *keys_tmp, int32_t *vals_tmp, int64_t n,
                            int key_bits, unsigned long long *hist, int grid, cudaStream_t st,
                            bool *result_in_tmp) {
  const int64_t chunk = (n + grid - 1) / grid;
  K *ki = keys, *ko = keys_tmp;
  int32_t *vi = vals, *vo = vals_tmp;
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
    radix_count_kernel<K><<<grid, kRadixThreads, 0, st>>>(ki, n, chunk, shift, hist);
    radix_offsets_kernel<<<1, kRadixThreads, 0, st>>>(hist, (int64_t)grid * kBins);
    radix_scatter_kernel<K, kVals><<<grid, kRadixThreads, 0, st>>>(ki, vi, n, chunk, shift, hist,
                                                                    ko, vo);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    K *tk = ki;
    ki = ko;
    ko = tk;
    int32_t *tv = vi;
    vi = vo;
    vo = tv;
  }
  *result_in_tmp = passes & 1;
  return cudaSuccess;
}

}  // namespace

size_t radix_hist_bytes(int grid) { return (size_t)grid * kBins * sizeof(unsigned long long); }

// Sorts (keys, vals) by the low key_bits bits of the keys, stably.  Ping-pongs
// with the tmp arrays; *result_in_tmp tells which pair holds the result.
// hist: radix_hist_bytes(grid) bytes of device scratch.
cudaError_t radix_sort_pairs_u32(uint32_t *keys, int32_t *vals, uint32_t *keys_tmp, int32_t *vals_tmp,
                                 int64_t n, int key_bits, void *hist, int grid, cudaStream_t st,
                                 bool *result_in_tmp) {
  *result_in_tmp = false;
  if (n <= 0) return cudaSuccess;
  return radix_sort_impl<uint32_t, true>(keys, vals, keys_tmp, vals_tmp, n, key_bits,
                                         (unsigned long long *)hist, grid, st, result_in_tmp);
}

cudaError_t radix_sort_keys_u64(unsigned long long *keys, unsigned long long *keys_tmp, int64_t n,
                                int key_bits, void *hist, int grid, cudaStream_t st,
                                bool *result_in_tmp) {
  *result_in_tmp = false;
  if (n <= 0) return cudaSuccess;
  return radix_sort_impl<unsigned long long, false>(keys, nullptr, keys_tmp, nullptr, n, key_bits,
                                                    (unsigned long long *)hist, grid, st,
                                                    result_in_tmp);
}

}  // namespace gsofa
