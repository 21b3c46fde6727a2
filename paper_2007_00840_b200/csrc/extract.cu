// extract.cu -- turn the in-structure bitmaps of a batch into sorted CSR rows.
//
// is[g][v] bit k  <=>  (s0 + 32 g + k, v) is an off-diagonal entry of L+U.
// L(s,:) = { v < s : bit },  U(s,:) = { s } U { v > s : bit }   (DS-9; U carries
// the diagonal).  The paper appends entries into L(src,:)/U(src,:) as
// they are found; here rows come out sorted without a sort:
// a warp loads 32 consecutive bitmap words (one 128-byte line), transposes the
// 32x32 bit block with five shuffle-xor stages, and lane k then owns the
// membership of 32 consecutive columns for source k.
//
// Three launches per batch: count (per 2048-column sub-chunk and source),
// scan (per-source prefix over sub-chunks, then one block scans the sources),
// write (ascending column ids; zeroes the bitmap for the next batch).
#include "gsofa_internal.cuh"

namespace gsofa {

namespace {
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kSub = 2048;            // columns per warp unit
constexpr int kTilesPerSub = kSub / 32;
constexpr int kWarpsPerBlock = 4;



__global__ void __launch_bounds__(kWarpsPerBlock * 32) extract_count_kernel(ExtractParams e) {
  const int lane = threadIdx.x & 31;
  const int sub = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int g = blockIdx.y;
  if (sub >= e.nchunks) return;
  const int s = e.s0 + g * 32 + lane;
  const uint32_t *isg = e.is_ro + (size_t)g * e.n;
  uint32_t cl = 0, cu = 0;
  const int vb = sub * kSub;
  for (int t = 0; t < kTilesPerSub; ++t) {
    const int v0 = vb + t * 32;
    if (v0 >= e.n) break;
    const uint32_t x = (v0 + lane < e.n) ? __ldcg(isg + v0 + lane) : 0u;
    if (__ballot_sync(kFull, x != 0u) == 0u) continue;
    const uint32_t y = transpose32(x, lane);
    uint32_t lm, um;
    split_masks(s - v0, lm, um);
    cl += __popc(y & lm);
    cu += __popc(y & um);
  }
  const size_t o = ((size_t)g * e.nchunks + sub) * 32 + lane;
  e.cntL[o] = cl;
  e.cntU[o] = cu;
}

// per-source exclusive prefix over sub-chunks; totals into rowL/rowU (temporarily)
__global__ void extract_prefix_kernel(ExtractParams e, int C) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= C) return;
  const int g = slot >> 5, k = slot & 31;
  uint32_t aL = 0, aU = 0;
  for (int sub = 0; sub < e.nchunks; ++sub) {
    const size_t o = ((size_t)g * e.nchunks + sub) * 32 + k;
    const uint32_t l = e.cntL[o], u = e.cntU[o];
    e.cntL[o] = aL;
    e.cntU[o] = aU;
    aL += l;
    aU += u;
  }
  const bool valid = e.s0 + slot < e.s_end;
  e.rowL[slot] = valid ? (int64_t)aL : 0;
  e.rowU[slot] = valid ? (int64_t)aU + 1 : 0;  // + the diagonal
}

// one block: exclusive scan of the per-source totals -> row starts, rowptrs
__global__ void __launch_bounds__(1024) extract_rows_kernel(ExtractParams e, int C) {
  __shared__ int64_t wsL[32], wsU[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (C + 1023) / 1024;
  const int a = min(C, tid * per), b = min(C, a + per);
  int64_t sL = 0, sU = 0;
  for (int i = a; i < b; ++i) {
    sL += e.rowL[i];
    sU += e.rowU[i];
  }
  // block exclusive scan of (sL, sU)
  int64_t iL = sL, iU = sU;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t tL = __shfl_up_sync(kFull, iL, d), tU = __shfl_up_sync(kFull, iU, d);
    if (lane >= d) {
      iL += tL;
      iU += tU;
    }
  }
  if (lane == 31) {
    wsL[wid] = iL;
    wsU[wid] = iU;
  }
  __syncthreads();
  if (wid == 0) {
    int64_t xL = wsL[lane], xU = wsU[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t tL = __shfl_up_sync(kFull, xL, d), tU = __shfl_up_sync(kFull, xU, d);
      if (lane >= d) {
        xL += tL;
        xU += tU;
      }
    }
    wsL[lane] = xL;
    wsU[lane] = xU;
  }
  __syncthreads();
  int64_t offL = iL - sL + (wid ? wsL[wid - 1] : 0);
  int64_t offU = iU - sU + (wid ? wsU[wid - 1] : 0);
  for (int i = a; i < b; ++i) {
    const int64_t l = e.rowL[i], u = e.rowU[i];
    e.rowL[i] = offL;
    e.rowU[i] = offU;
    const int s = e.s0 + i;
    if (s < e.s_end) {
      e.L_rowptr[s - e.row_begin + 1] = e.baseL + offL + l;
      e.U_rowptr[s - e.row_begin + 1] = e.baseU + offU + u;
    }
    offL += l;
    offU += u;
  }
  if (tid == 1023) {
    e.totals[0] = offL;
    e.totals[1] = offU;
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) extract_write_kernel(ExtractParams e) {
  const int lane = threadIdx.x & 31;
  const int sub = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int g = blockIdx.y;
  if (sub >= e.nchunks) return;
  const int s = e.s0 + g * 32 + lane;
  uint32_t *isg = e.is + (size_t)g * e.n;
  const size_t o = ((size_t)g * e.nchunks + sub) * 32 + lane;
  const int slot = g * 32 + lane;
  const bool valid = s < e.s_end;
  int32_t *Lp = e.L_out + e.baseL + (valid ? e.rowL[slot] + e.cntL[o] : 0);
  int32_t *Up = e.U_out + e.baseU + (valid ? e.rowU[slot] + 1 + e.cntU[o] : 0);
  if (sub == 0 && valid) e.U_out[e.baseU + e.rowU[slot]] = s;  // diagonal first in U(s,:)
  const int vb = sub * kSub;
  for (int t = 0; t < kTilesPerSub; ++t) {
    const int v0 = vb + t * 32;
    if (v0 >= e.n) break;
    const uint32_t x = (v0 + lane < e.n) ? __ldcg(isg + v0 + lane) : 0u;
    if (__ballot_sync(kFull, x != 0u) == 0u) continue;
    if (x) isg[v0 + lane] = 0u;  // read-and-zero for the next batch
    const uint32_t y = transpose32(x, lane);
    uint32_t lm, um;
    split_masks(s - v0, lm, um);
    uint32_t yl = y & lm, yu = y & um;
    while (yl) {
      const int i = __ffs(yl) - 1;
      *Lp++ = v0 + i;
      yl &= yl - 1u;
    }
    while (yu) {
      const int i = __ffs(yu) - 1;
      *Up++ = v0 + i;
      yu &= yu - 1u;
    }
  }
}
}  // namespace

cudaError_t launch_extract_count(const ExtractParams &e, cudaStream_t st) {
  dim3 grid((e.nchunks + kWarpsPerBlock - 1) / kWarpsPerBlock, e.G);
  extract_count_kernel<<<grid, kWarpsPerBlock * 32, 0, st>>>(e);
  return cudaGetLastError();
}

cudaError_t launch_extract_scan(const ExtractParams &e, cudaStream_t st) {
  const int C = e.G * 32;
  extract_prefix_kernel<<<(C + 255) / 256, 256, 0, st>>>(e, C);
  extract_rows_kernel<<<1, 1024, 0, st>>>(e, C);
  return cudaGetLastError();
}

cudaError_t launch_extract_write(const ExtractParams &e, cudaStream_t st) {
  dim3 grid((e.nchunks + kWarpsPerBlock - 1) / kWarpsPerBlock, e.G);
  extract_write_kernel<<<grid, kWarpsPerBlock * 32, 0, st>>>(e);
  return cudaGetLastError();
}

int extract_sub_columns() { return kSub; }

}  // namespace gsofa
