// threshold.cu -- the max-id relaxation (PAPER.md sec:parallel)
// scheduled in increasing newMaxId order, one CTA per 32-source slot group.
//
// Schedule: the paper relaxes all frontiers in
// parallel and accepts revisits; fill2 processes thresholds one
// at a time in increasing order and never revisits.  The relaxation is
// confluent (any order reaches the same maxId fixpoint), so the order is a
// scheduling choice.  On B200 the fine-grained parallelism comes from 32
// sources per warp lane set and from thousands of independent slot groups,
// not from relaxing one source out of order, so this kernel processes, per
// group, the frontier items in increasing newMaxId = T ("Dijkstra order",
// P:1038):
//   * thresholds T are the vertices that entered the structure (direct
//     neighbours get maxId = -1, R3, so newMaxId = max(-1, w) = w; fills get
//     maxId < w so newMaxId = w), visited in increasing id via a bitmap scan;
//   * the frontier of T is closed level by level (CTA barriers, no grid
//     barriers): every vertex w < T it reaches gets maxId = T and continues
//     with newMaxId = T; a vertex w > T (w < src) reached with T < w is a new
//     fill (R4) and a future threshold; w > src is an entry of U.
// In this order atomicMin(maxId(w), T) succeeds at most once per (source, w)
// -- the first T that reaches w is its final maxId -- so the 32 labels of a
// vertex collapse to one 32-bit "reached" mask and revisits vanish.
//
// Per group workspace (uint32 words): reached[Vb] | pend[Vb] | thr[Vb/32] |
// list0[Vb] | list1[Vb];  is[g][n] is the in-structure bitmap of extract.cu.
#include "gsofa_internal.cuh"

namespace gsofa {

namespace {
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kThrWarps = 4;
constexpr int kThrThreads = kThrWarps * 32;

// lanes k (sources s0g + k) with source > w, resp. source < w
__device__ __forceinline__ uint32_t lanes_above(int w, int s0g) {
  const int d = w - s0g;  // lane index of w
  if (d < 0) return kFull;
  if (d >= 31) return 0u;
  return kFull << (d + 1);
}
__device__ __forceinline__ uint32_t lanes_below(int w, int s0g) {
  const int d = w - s0g;
  if (d <= 0) return 0u;
  if (d >= 32) return kFull;
  return kFull >> (32 - d);
}

__global__ void __launch_bounds__(kThrThreads) threshold_kernel(ThrParams p) {
  const int g = blockIdx.x;
  const int s0g = p.s0 + 32 * g;
  if (s0g >= p.s_end) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsrc = min(32, p.s_end - s0g);
  const int Vb = p.Vb;
  const int tbw = (Vb + 31) >> 5;
  uint32_t *reached = p.ws + (size_t)g * p.ws_words;
  uint32_t *pend = reached + Vb;
  uint32_t *thr = pend + Vb;
  uint32_t *list0 = thr + tbw;
  uint32_t *list1 = list0 + Vb;
  uint32_t *isg = p.is + (size_t)g * p.n;
  const int32_t *__restrict__ rowptr = p.rowptr;
  const int32_t *__restrict__ colidx = p.colidx;

  __shared__ int s_T;
  __shared__ int s_qn[2];
  unsigned long long st_items = 0, st_edges = 0, st_pairs = 0, st_steps = 0, st_levels = 0;
  // XOR of atomic return values: consuming them forces the returning form
  // (ATOMG, the warp waits for completion at L2) instead of REDG.
  uint32_t sink = 0u;

  // ---- seed: out-neighbours of each source are in the
  // structure; the smaller ones are reached with maxId -1 -> thresholds
  for (int k = warp; k < nsrc; k += kThrWarps) {
    const int s = s0g + k;
    const uint32_t bit = 1u << k;
    const int beg = rowptr[s], end = rowptr[s + 1];
    for (int j = beg + lane; j < end; j += 32) {
      const int w = colidx[j];
      if (w == s) continue;
      atomicOr(isg + w, bit);
      if (w < s) {
        sink ^= atomicOr(reached + w, bit) ^ atomicOr(pend + w, bit) ^
                atomicOr(thr + (w >> 5), 1u << (w & 31));  // returning: see below
      }
    }
  }
  __syncthreads();

  int T = -1;
  int scan_word = 0;  // thr words below scan_word are known empty
  int max_list = 1;   // largest list length used (cleared at the end)
  for (;;) {
    // ---- next threshold: smallest set bit of thr above T (warp 0)
    if (warp == 0) {
      int nt = -1;
      const int start = T + 1;
      int wi = max(scan_word, start >> 5);
      bool first = true;
      while (wi < tbw) {
        const int idx = wi + lane;
        uint32_t x = idx < tbw ? __ldcg(thr + idx) : 0u;
        if (first && idx == (start >> 5)) x &= kFull << (start & 31);
        const uint32_t b = __ballot_sync(kFull, x != 0u);
        if (b) {
          const int l = __ffs(b) - 1;
          const uint32_t xl = __shfl_sync(kFull, x, l);
          nt = ((wi + l) << 5) + __ffs(xl) - 1;
          wi += l;
          break;
        }
        wi += 32;
        first = false;
      }
      if (lane == 0) {
        s_T = nt;
        if (nt >= 0) {
          list0[0] = (uint32_t)nt;
          s_qn[0] = 1;
          s_qn[1] = 0;
        }
      }
      scan_word = wi;
    }
    __syncthreads();
    T = s_T;
    if (T < 0) break;
    ++st_steps;
    // ---- close the frontier of T level by level (every item has newMaxId T)
    for (int lvl = 0;; ++lvl) {
      const int cur = lvl & 1, nxt = cur ^ 1;
      const uint32_t *cq = cur ? list1 : list0;
      uint32_t *nq = cur ? list0 : list1;
      const int qn = s_qn[cur];
      max_list = max(max_list, qn);
      __syncthreads();
      if (threadIdx.x == 0) s_qn[cur] = 0;
      ++st_levels;
      for (int b0 = warp * 32; b0 < qn; b0 += kThrThreads) {
        const int cnt = min(32, qn - b0);
        int u = 0, beg = 0, deg = 0;
        uint32_t mask = 0u;
        if (lane < cnt) {
          u = (int)cq[b0 + lane];
          mask = atomicExch(pend + u, 0u);  // lanes that expand u with newMaxId T
          if (mask) {
            beg = rowptr[u];
            deg = rowptr[u + 1] - beg;
          }
        }
        // load-balanced expansion of the (item, neighbour) pairs over lanes
        int incl = deg;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += y;
        }
        const int total = __shfl_sync(kFull, incl, 31);
        const int excl = incl - deg;
        st_items += mask != 0u;
        st_pairs += (unsigned long long)deg;
        st_edges += (unsigned long long)__popc(mask) * (unsigned long long)deg;
        for (int f0 = 0; f0 < total; f0 += 32) {
          const int f = f0 + lane;
          int o = 0;
#pragma unroll
          for (int step = 16; step >= 1; step >>= 1) {
            const int cand = o + step;
            const int e = __shfl_sync(kFull, excl, cand & 31);
            if (cand < 32 && e <= f) o = cand;
          }
          const int ob = __shfl_sync(kFull, beg, o);
          const int oe = __shfl_sync(kFull, excl, o);
          const uint32_t om = __shfl_sync(kFull, mask, o);
          bool push = false;
          int w = 0;
          if (f < total) {
            w = __ldg(colidx + ob + (f - oe));
            const uint32_t um = om & lanes_below(w, s0g);   // sources < w: U entry
            const uint32_t lm = om & lanes_above(w, s0g);   // sources > w: maxId(w)
            if (um) atomicOr(isg + w, um);
            if (lm) {
              // atomicMin(maxId(w), T) succeeds exactly for the lanes that
              // have not reached w yet (line 10)
              const uint32_t nw = lm & ~atomicOr(reached + w, lm);
              if (nw) {
                if (w > T) {
                  // newMaxId T < w: (src, w) is a fill of L (R4); w proposes
                  // newMaxId = w later, as a threshold.  pend/thr are read by
                  // other warps after the next barrier, so these are returning
                  // atomics whose results are consumed here (a fire-and-forget
                  // RED may still be in flight to L2 when the barrier opens).
                  atomicOr(isg + w, nw);
                  sink ^= atomicOr(pend + w, nw) ^ atomicOr(thr + (w >> 5), 1u << (w & 31));
                } else {
                  // w < T: maxId(w) = T, not in the structure, continue with T
                  push = atomicOr(pend + w, nw) == 0u;
                }
              }
            }
          }
          const uint32_t pb = __ballot_sync(kFull, push);
          if (pb) {
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_qn[nxt], __popc(pb));
            base = __shfl_sync(kFull, base, 0);
            if (push) nq[base + __popc(pb & lanemask_lt())] = (uint32_t)w;
          }
        }
      }
      __syncthreads();
      if (s_qn[nxt] == 0) break;
    }
  }
  // ---- reset the workspace: the next batch may lay groups out differently
  // (Vb changes), so every word this group wrote must be zero again --
  // reached and thr here, the used prefix of both lists, pend is already 0
  {
    for (int i = threadIdx.x; i < max_list; i += kThrThreads) {
      list0[i] = 0u;
      list1[i] = 0u;
    }
    uint4 *r4 = reinterpret_cast<uint4 *>(reached);
    const int n4 = Vb >> 2;
    for (int i = threadIdx.x; i < n4; i += kThrThreads) r4[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int i = (n4 << 2) + threadIdx.x; i < Vb; i += kThrThreads) reached[i] = 0u;
    for (int i = threadIdx.x; i < tbw; i += kThrThreads) thr[i] = 0u;
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    st_items += __shfl_xor_sync(kFull, st_items, d);
    st_edges += __shfl_xor_sync(kFull, st_edges, d);
    st_pairs += __shfl_xor_sync(kFull, st_pairs, d);
  }
  if (lane == 0) {
    atomicAdd(p.stats + 0, st_items);
    atomicAdd(p.stats + 1, st_edges);
    atomicAdd(p.stats + 4, st_pairs);
  }
  if (p.n < 0) p.stats[7] = sink;  // never true; keeps `sink` alive
  if (threadIdx.x == 0) {
    atomicAdd(p.stats + 2, st_levels);
    atomicAdd(p.stats + 3, st_steps);
  }
}
}  // namespace

size_t threshold_ws_words(int64_t Vb) {
  // reached + pend + list0 + list1 + thr, padded to 16 bytes
  const size_t w = 4 * (size_t)Vb + (size_t)((Vb + 31) / 32);
  return (w + 3) / 4 * 4;
}

cudaError_t launch_threshold(const ThrParams &p, cudaStream_t st) {
  if (p.s_end <= p.s0) return cudaSuccess;
  threshold_kernel<<<p.G, kThrThreads, 0, st>>>(p);
  return cudaGetLastError();
}

}  // namespace gsofa
