// traverse.cu -- multi-source max-id relaxation (PAPER.md sec:parallel,
// P:514-598) for one batch of C = 32 G concurrent sources, sm_100a.
//
// Semantics (readings R2-R4, pinned by tests/test_relaxation_reading.py
// against the trace of P:547-551):
//   maxId(v) = min over discovered paths src ~> v of the largest intermediate
//   vertex.  Direct neighbours of src start at -1 (R3).  A frontier u
//   proposes newMaxId = max(maxId(u), u) (R2).  For a neighbour w of u:
//     w == src : skip (the diagonal is implicit)
//     w >  src : (src, w) is an entry of U(src,:)
//     w <  src : old = atomicMin(maxId(w), newMaxId)
//                if it lowered maxId(w) and w was not yet in the structure
//                (old > w): enqueue w for the next iteration, and if
//                newMaxId < w, (src, w) is a new fill of L(src,:)  (R4)
//   The traversal stops when no frontier remains.
//
// B200 design: one warp per (u, slot group g) frontier
// item; lane k is source s0 + 32 g + k, so the neighbour list of u is read
// once for 32 sources (coalesced 128-byte colidx loads) and the 32 labels of
// a neighbour are one 128-byte line (one coalesced atomicMin per lane).
// Frontier membership is a per-(g, v) bitmask; an item is pushed once, when
// its mask goes 0 -> nonzero (ballot + popc + warp-aggregated atomic enqueue,
// P:598).  All iterations of a batch run inside ONE persistent cooperative
// kernel separated by grid-wide barriers (no host round trips).
#include <cooperative_groups.h>

#include "gsofa_internal.cuh"

namespace cg = cooperative_groups;

namespace gsofa {

namespace {
constexpr uint32_t kFull = 0xFFFFFFFFu;

// queue slot i: the first qcap items live in HBM, the rest in mapped host
// memory (external frontier management)
__device__ __forceinline__ uint32_t q_load(const uint32_t *q, const uint32_t *qx, uint32_t qcap,
                                           uint32_t i) {
  return i < qcap ? __ldcg(q + i) : __ldcv(qx + (i - qcap));
}
__device__ __forceinline__ void q_store(uint32_t *q, uint32_t *qx, uint32_t qcap, uint32_t i,
                                        uint32_t v) {
  if (i < qcap) q[i] = v;
  else __stcg(qx + (i - qcap), v);
}

// Seed: every out-neighbour w != src of each source is in the structure;
// the smaller ones get maxId = -1 and form the first frontier.
__global__ void __launch_bounds__(256) seed_kernel(BatchParams p) {
  const int lane = threadIdx.x & 31;
  const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int s = p.s0 + slot;
  if (s >= p.s_end) return;
  const int g = slot >> 5, k = slot & 31;
  const uint32_t bit = 1u << k;
  const int beg = p.rowptr[s], end = p.rowptr[s + 1];
  uint32_t *isg = p.is + (size_t)g * p.n;
  uint32_t *labg = p.lab + (size_t)g * p.Vb * 32 + k;
  uint32_t *fmg = p.fm0 + (size_t)g * p.Vb;
  unsigned long long fv = 0;  // first visits of (s, w < s): the seeds
  for (int j = beg + lane; j < end; j += 32) {
    const int w = p.colidx[j];
    if (w == s) continue;
    fv += w < s;
    atomicOr(isg + w, bit);
    if (w < s) {
      labg[(size_t)w * 32] = p.base;  // enc(-1)
      if (atomicOr(fmg + w, bit) == 0u) {
        const uint32_t pos = atomicAdd(p.qcount, 1u);
        q_store(p.q0, p.qx0, p.qcap, pos, ((uint32_t)w << p.gbits) | (uint32_t)g);
      }
    }
  }
  fv = __reduce_add_sync(kFull, (unsigned)fv);
  if (lane == 0 && fv) atomicAdd(p.stats + 8, fv);
}

// coalesced 32-source label atomics a warp keeps in flight per item
#ifndef GSOFA_FIFO_INFLIGHT
#define GSOFA_FIFO_INFLIGHT 8  // measured: 4 -> 8 is C3 -6.5%; 16 spills
#endif
constexpr int kFifoInflight = GSOFA_FIFO_INFLIGHT;

template <bool kFillFirst>
__device__ __forceinline__ void expand_item(const BatchParams &p, uint32_t u, uint32_t g,
                                            uint32_t *fmc, uint32_t *fmn, uint32_t *nq,
                                            uint32_t *nqx, uint32_t *ncount, uint32_t *buf, int &nb,
                                            int lane, unsigned long long *wst,
                                            uint32_t &st_fv) {
  const size_t row = (size_t)g * p.Vb + u;
  uint32_t mask = 0;
  if (lane == 0) {
    mask = __ldcg(fmc + row);
    fmc[row] = 0u;  // only this warp touches fmc[row] in this iteration
  }
  mask = __shfl_sync(kFull, mask, 0);
  const bool act = (mask >> lane) & 1u;
  const int s = p.s0 + (int)(g << 5) + lane;
  // processing-time read of maxId(u) for the 32 sources (one 128-byte line)
  const uint32_t labu = __ldcg(p.lab + row * 32 + lane);
  const int c = max((int)(labu - p.base) - 1, (int)u);  // newMaxId, R2
  const uint32_t encc = p.base + (uint32_t)c + 1u;
  const int beg = __ldg(p.rowptr + u), end = __ldg(p.rowptr + u + 1);
  if (lane == 0) {
    // this warp's counters live in shared memory (registers are at the
    // 64-per-thread budget of 2 CTAs x 512 threads)
    wst[0] += 1;
    wst[1] += (unsigned long long)__popc(mask) * (unsigned long long)(end - beg);
    wst[2] += (unsigned long long)(end - beg);
    wst[3] += (unsigned long long)__popc(mask);
  }
  uint32_t *labg = p.lab + (size_t)g * p.Vb * 32 + lane;
  uint32_t *isg = p.is + (size_t)g * p.n;
  uint32_t *fmg = fmn + (size_t)g * p.Vb;
  for (int j0 = beg; j0 < end; j0 += 32) {
    const int cnt = min(32, end - j0);
    const int wl = lane < cnt ? __ldg(p.colidx + j0 + lane) : 0;
    uint32_t my_is = 0u, my_enq = 0u;
#pragma unroll 1
    for (int t = 0; t < cnt; t += kFifoInflight) {
      int w[kFifoInflight];
      uint32_t old[kFifoInflight];
      bool lo[kFifoInflight], up[kFifoInflight];
#pragma unroll
      for (int i = 0; i < kFifoInflight; ++i) {
        w[i] = __shfl_sync(kFull, wl, (t + i) & 31);
        const bool valid = (t + i) < cnt;
        lo[i] = act && valid && w[i] < s;
        up[i] = act && valid && w[i] > s;
        old[i] = 0xFFFFFFFFu;
        if (kFillFirst && lo[i]) {
          // "line 9.5": a vertex already in the structure always
          // proposes its own id, so do not lower its maxId
          if (__ldcg(labg + (size_t)w[i] * 32) < p.base + (uint32_t)w[i] + 1u) lo[i] = false;
        }
        if (lo[i]) old[i] = atomicMin(labg + (size_t)w[i] * 32, encc);  // line 10
      }
#pragma unroll
      for (int i = 0; i < kFifoInflight; ++i) {
        // first visit of (s, w): the old label is not of this batch's epoch
        // (values of the epoch are base .. base + n + 1)
        // (counted per lane, summed over the warp once at the end)
        st_fv += (lo[i] && old[i] > p.base + (uint32_t)p.n + 1u) ? 1u : 0u;
        const bool enq = lo[i] && encc < old[i] && old[i] > p.base + (uint32_t)w[i] + 1u;
        const bool fill = enq && c < w[i];
        const uint32_t ib = __ballot_sync(kFull, up[i] || fill);
        const uint32_t eb = __ballot_sync(kFull, enq);
        if (lane == t + i) {
          my_is = ib;
          my_enq = eb;
        }
      }
    }
    // lane j now owns neighbour j0 + j: structure bits and frontier bits
    if (my_is) atomicOr(isg + wl, my_is);  // no return value -> RED
    bool push = false;
    if (my_enq) push = atomicOr(fmg + wl, my_enq) == 0u;
    const uint32_t pb = __ballot_sync(kFull, push);
    if (pb) {
      if (push) buf[nb + __popc(pb & lanemask_lt())] = ((uint32_t)wl << p.gbits) | g;
      nb += __popc(pb);
      __syncwarp();
      if (nb >= 32) {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(ncount, 32u);
        b = __shfl_sync(kFull, b, 0);
        q_store(nq, nqx, p.qcap, b + lane, buf[lane]);
        __syncwarp();
        if (lane < nb - 32) buf[lane] = buf[32 + lane];
        __syncwarp();
        nb -= 32;
      }
    }
  }
}

template <bool kFillFirst>
__global__ void __launch_bounds__(kTraverseThreads, 2) traverse_kernel(BatchParams p) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t sbuf[kTraverseThreads / 32][64];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t gmask = (1u << p.gbits) - 1u;
  uint32_t *buf = sbuf[wib];
  // per warp: items, (source, edge) inspections, (item, neighbour) pairs,
  // source expansions
  __shared__ unsigned long long s_st[kTraverseThreads / 32][4];
  unsigned long long *wst = s_st[wib];
  if (lane < 4) wst[lane] = 0ull;
  __syncwarp();
  uint32_t st_fv = 0;  // this lane's first visits
  int round = 0;
  for (;; ++round) {
    const uint32_t *q = (round & 1) ? p.q1 : p.q0;
    uint32_t *nq = (round & 1) ? p.q0 : p.q1;
    const uint32_t *qx = (round & 1) ? p.qx1 : p.qx0;
    uint32_t *nqx = (round & 1) ? p.qx0 : p.qx1;
    uint32_t *fmc = (round & 1) ? p.fm1 : p.fm0;
    uint32_t *fmn = (round & 1) ? p.fm0 : p.fm1;
    uint32_t *ncount = p.qcount + (round + 1) % 3;
    const uint32_t qn = __ldcg(p.qcount + round % 3);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.qcount[(round + 2) % 3] = 0u;
      if (round == 0 && qn > p.qcap) atomicAdd(p.stats + 10, (unsigned long long)(qn - p.qcap));
    }
    uint32_t per = (qn + nw - 1) / nw;
    per = per < 1u ? 1u : (per > 32u ? 32u : per);
    int nb = 0;
    for (uint32_t b0 = gw * per; b0 < qn; b0 += nw * per) {
      const uint32_t cnt = min(per, qn - b0);
      const uint32_t my = lane < (int)cnt ? q_load(q, qx, p.qcap, b0 + lane) : 0u;
      for (uint32_t t = 0; t < cnt; ++t) {
        const uint32_t item = __shfl_sync(kFull, my, t);
        expand_item<kFillFirst>(p, item >> p.gbits, item & gmask, fmc, fmn, nq, nqx, ncount, buf,
                                nb, lane, wst, st_fv);
      }
    }
    if (nb > 0) {
      uint32_t b = 0;
      if (lane == 0) b = atomicAdd(ncount, (uint32_t)nb);
      b = __shfl_sync(kFull, b, 0);
      if (lane < nb) q_store(nq, nqx, p.qcap, b + lane, buf[lane]);
    }
    grid.sync();
    const uint32_t nn = __ldcg(ncount);
    // items of the next frontier that went to host memory
    if (blockIdx.x == 0 && threadIdx.x == 0 && nn > p.qcap)
      atomicAdd(p.stats + 10, (unsigned long long)(nn - p.qcap));
    if (nn == 0u) break;
  }
  unsigned long long fv = st_fv;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) fv += __shfl_xor_sync(kFull, fv, d);
  if (lane == 0 && wst[0]) {
    atomicAdd(p.stats + 0, wst[0]);
    atomicAdd(p.stats + 1, wst[1]);
    atomicAdd(p.stats + 4, wst[2]);
    atomicAdd(p.stats + 8, fv);
    atomicAdd(p.stats + 9, wst[3]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(p.stats + 2, (unsigned long long)(round + 1));
}
}  // namespace

cudaError_t launch_seed(const BatchParams &p, cudaStream_t st) {
  const int slots = p.s_end - p.s0;
  if (slots <= 0) return cudaSuccess;
  const int wpb = 256 / 32;
  seed_kernel<<<(slots + wpb - 1) / wpb, 256, 0, st>>>(p);
  return cudaGetLastError();
}

int traverse_max_blocks(int device, int fill_first) {
  int sms = 0, per = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  cudaError_t e = fill_first
      ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, traverse_kernel<true>, kTraverseThreads, 0)
      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, traverse_kernel<false>, kTraverseThreads, 0);
  if (e != cudaSuccess) return 0;
  return sms * per;
}

cudaError_t launch_traverse(const BatchParams &p, int fill_first, int grid_blocks,
                            cudaStream_t st) {
  BatchParams pp = p;
  void *args[] = {&pp};
  const void *fn = fill_first ? (const void *)traverse_kernel<true>
                              : (const void *)traverse_kernel<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid_blocks), dim3(kTraverseThreads), args, 0, st);
}

}  // namespace gsofa
