// threshold.cu -- the max-id relaxation (PAPER.md sec:parallel)
// scheduled in increasing newMaxId order, as ONE persistent streaming kernel:
// each CTA owns a workspace slot and repeatedly takes the next 32-source
// group (heaviest -- highest row ids -- first), traverses it,
// extracts its 32 rows into a staging area and resets what it touched.
//
// Schedule: the relaxation is confluent, so the order is a
// scheduling choice.  Per group, frontier items are processed in increasing
// newMaxId = T ("Dijkstra order"):
//   * thresholds T are the vertices that entered the structure (direct
//     neighbours get maxId -1 (R3), so newMaxId = max(-1, w) = w; fills get
//     maxId < w so newMaxId = w);
//   * the frontier of T is closed level by level with CTA barriers: every
//     vertex w < T it reaches gets maxId = T and continues with newMaxId = T;
//     a vertex T < w < src reached with T < w is a new fill (R4) and a later
//     threshold; w > src is an entry of U.
// In this order atomicMin(maxId(w), T) succeeds at most once per (source, w),
// so the 32 labels of a vertex collapse to one 32-bit "reached" mask and
// there are no revisits.
//
// Workspace slot (uint32 words, fixed layout per launch):
//   state[2*Vmax]  reached | pend interleaved per vertex (one 32 B sector)
//   thr[Vmax/32]   threshold bitmap          rsum[Vmax/1024] touched lines
//   list0[Vmax], list1[Vmax]                 frontier lists of a closure
//   is[n]          in-structure bits          isum[n/1024]   touched lines
// All of it is zero between groups; a group clears only the 32-vertex lines
// recorded in rsum/isum (first-touch tracking), never the whole slot.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "gsofa_internal.cuh"

namespace gsofa {

namespace {
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kLightWarps = 4;   // lockstep CTA: 32 sources share frontier items
constexpr int kSoloWarps = 16;   // solo CTA: independent warps, one source each

// lanes k (sources s0g + k) with source > w, resp. source < w
__device__ __forceinline__ uint32_t lanes_above(int w, int s0g) {
  const int d = w - s0g;
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



struct Slot {
  uint32_t *state, *thr, *rsum, *list0, *list1, *is, *isum;
  uint32_t *tsum;  // shared memory
};

// Next set bit of thr strictly above T (warp-cooperative), INT_MAX if none.
// tsum (shared memory) has one bit per thr word that is nonzero, so the scan
// touches at most two thr words however far the next threshold is.
__device__ __forceinline__ int scan_next(const uint32_t *thr, const uint32_t *tsum, int tbw, int T,
                                         int lane) {
  const int start = T + 1;
  const int wi = start >> 5;
  if (wi >= tbw) return INT_MAX;
  uint32_t x = 0u;
  if (lane == 0) x = __ldcg(thr + wi) & (kFull << (start & 31));
  x = __shfl_sync(kFull, x, 0);
  if (x) return (wi << 5) + __ffs(x) - 1;
  const int nw = wi + 1;  // first thr word to look for
  const int tsw = (tbw + 31) >> 5;
  for (int si = nw >> 5; si < tsw; si += 32) {
    const int idx = si + lane;
    uint32_t y = idx < tsw ? tsum[idx] : 0u;
    if (si == (nw >> 5) && lane == 0) y &= kFull << (nw & 31);
    const uint32_t b = __ballot_sync(kFull, y != 0u);
    if (b) {
      const int l = __ffs(b) - 1;
      const uint32_t yl = __shfl_sync(kFull, y, l);
      const int word = ((si + l) << 5) + __ffs(yl) - 1;
      const uint32_t z = __ldcg(thr + word);
      return (word << 5) + __ffs(z) - 1;
    }
  }
  return INT_MAX;
}

struct Counters {
  unsigned long long items, edges, pairs, levels, steps;
  unsigned long long fv, sx;  // first visits (source, w < source); (source, item) expansions
  uint32_t sink;
};

// release this thread's fire-and-forget reductions (REDs) before a barrier:
// after fence + bar.sync every thread of the CTA observes them
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

constexpr int kBatch = 4;  // 32-pair batches whose atomics a warp keeps in flight

// Expand up to 32 frontier items (one per lane; u < 0 = none) of the closure
// of threshold T.  Every item's newMaxId is T.  Pushes closure members into
// `nq` (count *nqn), records new fills in thr / tsum / *minfill.
// Only two atomics per (item, neighbour) pair return a value the warp waits
// for: the reached mask of w (line 10 of fig:alg) and, for w < T, the
// pend mask (enqueue test); both are issued for kBatch*32 pairs before any
// result is used.  Every other update is a RED, published by fence_gpu()
// before the next barrier.
// Height order (kH, lockstep): the step is every threshold of one etree
// height h (ids tmin = T .. tmax, union over the group's sources); a newly
// reached w < source is a fill iff w > tmax, or w > tmin and height(w) > h
// (order.cu), and its threshold bit sits at its position pos(w).
template <bool kH = false>
__device__ __forceinline__ void expand(const StreamParams &p, const Slot &sl, int s0g, int T,
                                       int u, uint32_t *nq, int *nqn, int *minfill, int lane,
                                       Counters &c, int tmax = 0, int hh = 0) {
  const int32_t *__restrict__ rowptr = p.rowptr;
  const int32_t *__restrict__ colidx = p.colidx;
  int beg = 0, deg = 0;
  uint32_t mask = 0u;
  if (u >= 0) {
    beg = __ldg(rowptr + u);
    deg = __ldg(rowptr + u + 1) - beg;
    mask = atomicExch(sl.state + 2 * u + 1, 0u);  // lanes that expand u (pend)
    if (!mask) deg = 0;
  }
  c.items += mask != 0u;
  c.sx += (unsigned long long)__popc(mask);
  c.pairs += (unsigned long long)deg;
  c.edges += (unsigned long long)__popc(mask) * (unsigned long long)deg;
  // load-balanced expansion of the (item, neighbour) pairs over the lanes
  int incl = deg;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  const int total = __shfl_sync(kFull, incl, 31);
  if (total == 0) return;
  const int excl = incl - deg;
  for (int f0 = 0; f0 < total; f0 += 32 * kBatch) {
    int w[kBatch];
    uint32_t lm[kBatch], ro[kBatch], io[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const int f = f0 + 32 * k + lane;
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
      w[k] = f < total ? __ldg(colidx + ob + (f - oe)) : 0;
      const uint32_t um = f < total ? om & lanes_below(w[k], s0g) : 0u;  // U entries
      lm[k] = f < total ? om & lanes_above(w[k], s0g) : 0u;             // maxId(w)
      // atomicMin(maxId(w), T) succeeds exactly for the lanes that have not
      // reached w yet (line 10); IS first-touch is detected from its
      // old value.  Both are issued now and consumed below.
      ro[k] = lm[k] ? atomicOr(sl.state + 2 * w[k], lm[k]) : kFull;
      io[k] = um ? atomicOr(sl.is + w[k], um) : kFull;
    }
    bool push[kBatch];
    uint32_t po[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      if (io[k] == 0u) atomicOr(sl.isum + (w[k] >> 10), 1u << ((w[k] >> 5) & 31));  // RED
      if (ro[k] == 0u) atomicOr(sl.rsum + (w[k] >> 10), 1u << ((w[k] >> 5) & 31));  // RED
      const uint32_t nw = lm[k] & ~ro[k];
      c.fv += (unsigned long long)__popc(nw);  // sources that reach w < source for the first time
      push[k] = false;
      po[k] = kFull;
      if (nw) {
        const bool fill = kH ? (w[k] > tmax || (w[k] > T && __ldg(p.hgt + w[k]) > hh)) : w[k] > T;
        if (fill) {
          // newMaxId T < w: (src, w) is a fill of L (R4); w proposes newMaxId
          // = w later, as a threshold (at its bitmap position q)
          const int q = kH ? __ldg(p.pos + w[k]) : w[k];
          atomicOr(sl.is + w[k], nw);                                           // RED
          atomicOr(sl.isum + (w[k] >> 10), 1u << ((w[k] >> 5) & 31));          // RED
          atomicOr(sl.state + 2 * w[k] + 1, nw);                                // RED
          atomicOr(sl.thr + (q >> 5), 1u << (q & 31));                          // RED
          atomicOr(sl.tsum + (q >> 10), 1u << ((q >> 5) & 31));                // smem
          atomicMin(minfill, q);                                                // smem
        } else {
          // w < T: maxId(w) = T, not in the structure: continue with T
          po[k] = atomicOr(sl.state + 2 * w[k] + 1, nw);
          push[k] = true;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      const bool ps = push[k] && po[k] == 0u;
      const uint32_t pb = __ballot_sync(kFull, ps);
      if (pb) {
        int base = 0;
        if (lane == 0) base = atomicAdd(nqn, __popc(pb));
        base = __shfl_sync(kFull, base, 0);
        if (ps) nq[base + __popc(pb & lanemask_lt())] = (uint32_t)w[k];
      }
    }
    if (f0 + 32 * kBatch >= total) break;
  }
}


// Extraction of a group's rows from its in-structure bitmap (touched lines
// only, ascending), staging reservation (one atomic per group) and write-out;
// zeroes the bitmap lines it reads.  All kWarps warps of the CTA take part.
// warp w owns isum words [w*q, (w+1)*q): its lines are ascending and all of
// them precede warp w+1's, so per-warp counts give the write offsets.
template <int kWarps, bool kWarpOnly = false>
__device__ __forceinline__ void stage_rows(const StreamParams &p, uint32_t *is, uint32_t *isum,
                                           int s0g, int nsrc, int g, int lane, int warp,
                                           uint32_t (*s_cnt)[2][32], long long *s_rowoff,
                                           int *s_nL, int *s_ok, bool write) {
  const int n = p.n;
  const int isw = (n + 1023) >> 10;
  const int q = (isw + kWarps - 1) / kWarps;
  const int wa = min(isw, warp * q), wb = min(isw, wa + q);
  const int s_lane = s0g + lane;
  if (write) {
    uint32_t cl = 0, cu = 0;
    for (int i = wa; i < wb; ++i) {
      uint32_t x = __ldcg(isum + i);
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1u;
        const int v0 = ((i << 5) + b) << 5;
        const uint32_t word = (v0 + lane < n) ? __ldcg(is + v0 + lane) : 0u;
        const uint32_t y = transpose32(word, lane);
        uint32_t lm, um;
        split_masks(s_lane - v0, lm, um);
        cl += __popc(y & lm);
        cu += __popc(y & um);
      }
    }
    s_cnt[warp][0][lane] = cl;
    s_cnt[warp][1][lane] = cu;
    if (kWarpOnly) __syncwarp(); else __syncthreads();
    if (warp == 0) {
      uint32_t nl = 0, nu = 0;
      for (int w2 = 0; w2 < kWarps; ++w2) {
        nl += s_cnt[w2][0][lane];
        nu += s_cnt[w2][1][lane];
      }
      const bool valid = lane < nsrc;
      if (valid) nu += 1;  // the diagonal
      const long long sz = valid ? (long long)nl + nu : 0;
      long long inc = sz;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(kFull, inc, d);
        if (lane >= d) inc += y;
      }
      const long long tot = __shfl_sync(kFull, inc, 31);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(p.stage_cursor, (unsigned long long)tot);
      base = __shfl_sync(kFull, base, 0);
      const bool ok = base + (unsigned long long)tot <= p.stage_cap;
      if (valid) {
        const long long off = (long long)base + inc - sz;
        s_rowoff[lane] = off;
        s_nL[lane] = (int)nl;
        const int r = 32 * g + lane;  // local row
        p.row_off[r] = ok ? off : -1;
        p.row_nL[r] = (int)nl;
        p.row_nU[r] = (int)nu;
        if (ok) p.stage[off + nl] = s_lane;  // U(s,:) starts with the diagonal
      }
      if (lane == 0) {
        *s_ok = ok;
        if (!ok) {
          if (atomicExch(p.failed_flag + g, 1) == 0) p.failed[atomicAdd(p.nfailed, 1)] = g;
          atomicAdd(p.failed_need, (unsigned long long)tot);
        }
      }
    }
    if (kWarpOnly) __syncwarp(); else __syncthreads();
  }
  const bool ok = write && *s_ok;
  long long pl = 0, pu = 0;
  if (ok)
    for (int w2 = 0; w2 < warp; ++w2) {
      pl += s_cnt[w2][0][lane];
      pu += s_cnt[w2][1][lane];
    }
  const bool valid = lane < nsrc;
  int32_t *Lp = p.stage + (valid && ok ? s_rowoff[lane] + pl : 0);
  int32_t *Up = p.stage + (valid && ok ? s_rowoff[lane] + s_nL[lane] + 1 + pu : 0);
  for (int i = wa; i < wb; ++i) {
    uint32_t x = __ldcg(isum + i);
    if (!x) continue;
    if (lane == 0) isum[i] = 0u;
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1u;
      const int v0 = ((i << 5) + b) << 5;
      const uint32_t word = (v0 + lane < n) ? __ldcg(is + v0 + lane) : 0u;
      if (v0 + lane < n) is[v0 + lane] = 0u;
      if (ok) {
        const uint32_t y = transpose32(word, lane);
        uint32_t lm, um;
        split_masks(s_lane - v0, lm, um);
        uint32_t yl = y & lm, yu = y & um;
        while (yl) {
          *Lp++ = v0 + __ffs(yl) - 1;
          yl &= yl - 1u;
        }
        while (yu) {
          *Up++ = v0 + __ffs(yu) - 1;
          yu &= yu - 1u;
        }
      }
    }
  }
}

// Lockstep kernel: the 32 sources of a group share frontier items (one bit
// each); a group that runs longer than p.abort_cycles is abandoned -- its
// slot is cleaned -- and handed to the solo kernel through the heavy queue.
// kH: etree-height order (order.cu) -- a step takes every threshold of one
// height (the group's union: the whole segment of positions), so a group is
// at most tree-height steps long and the 32 sources of hub / separator groups
// share their closures (C4); the threshold bitmap is indexed by position.
// kW warps per CTA: 4 in id order; height order takes 16 by default (one
// group's step spreads over more warps: a hub group is one CTA's work)
template <bool kH, int kW = kLightWarps>
__global__ void __launch_bounds__(kW * 32, 32 / kW) stream_kernel(StreamParams p) {
  constexpr int kWarps = kW;
  constexpr int kThreads = kWarps * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const int n = p.n, Vmax = p.Vmax;
  const int tbw_max = kH ? (p.npos + 31) >> 5 : (Vmax + 31) >> 5;
  const int rsw = (Vmax + 1023) >> 10;
  Slot sl;
  const size_t slot = blockIdx.x;
  sl.state = p.ws + slot * p.ws_words;
  sl.thr = sl.state + 2 * (size_t)Vmax;
  sl.rsum = sl.thr + tbw_max;
  sl.list0 = sl.rsum + rsw;
  sl.list1 = sl.list0 + Vmax;
  sl.is = p.is + slot * p.is_words;
  sl.isum = sl.is + n;
  extern __shared__ uint32_t s_tsum[];  // [(tbw_max + 31) / 32]
  sl.tsum = s_tsum;

  __shared__ int s_g, s_qn[3], s_scan[3], s_minfill[3];
  __shared__ uint32_t s_cnt[kWarps][2][32];
  __shared__ long long s_rowoff[32];
  __shared__ int s_nL[32];
  __shared__ int s_ok, s_abort;
  __shared__ int s_hs[4];  // kH step: segment end, height, tmin, tmax
  __shared__ int s_nx[3];  // kH: the scanned next threshold, its segment end and height
  Counters c = {0, 0, 0, 0, 0, 0, 0, 0u};
  // live lockstep CTAs: while any runs, it may still abandon a group to the
  // solo kernel's queue (idle solo warps wait only as long as that can happen)
  if (tid == 0 && p.light_live) atomicAdd(p.light_live, 1u);

  for (;;) {
    if (tid == 0) {
      // heaviest first: group ngroups-1-j is the j-th taken (work grows
      // with the source id)
      int gg = -1;
      const int j = (int)atomicAdd(p.group_ctr, 1u);
      if (p.group_list) {
        if (j < p.list_len) gg = p.group_list[j];
      } else if (j < p.ngroups - p.solo_top) {
        gg = p.ngroups - p.solo_top - 1 - j;  // the top solo_top go to the solo kernel
      }
      s_g = gg;
      s_abort = 0;
      s_qn[0] = s_qn[1] = s_qn[2] = 0;
      s_nx[0] = -1;
      for (int i = 0; i < 3; ++i) s_scan[i] = s_minfill[i] = INT_MAX;
    }
    __syncthreads();
    const int g = s_g;
    if (g < 0) break;
    const long long t_start = clock64();
    const unsigned long long st0 = c.steps, lv0 = c.levels, it0 = c.items, pr0 = c.pairs;
    const unsigned long long fv0 = c.fv, sx0 = c.sx;
    long long t_trav = 0, t_ext = 0;
    const int s0g = p.map.row(32 * g);  // the group's 32 rows are consecutive
    const int nsrc = min(32, p.nrows - 32 * g);
    const int Vb = min(n, s0g + nsrc);  // maxId only below the largest source
    const int tbw = kH ? tbw_max : (Vb + 31) >> 5;
    for (int i = tid; i < ((tbw + 31) >> 5); i += kThreads) s_tsum[i] = 0u;
    __syncthreads();

    // ---- seed: out-neighbours of each source are in the
    // structure; the smaller ones are reached with maxId -1 -> thresholds
    for (int k = warp; k < nsrc; k += kWarps) {
      const int s = s0g + k;
      const uint32_t bit = 1u << k;
      const int beg = __ldg(p.rowptr + s), end = __ldg(p.rowptr + s + 1);
      for (int j = beg + lane; j < end; j += 32) {
        const int w = __ldg(p.colidx + j);
        if (w == s) continue;
        atomicOr(sl.is + w, bit);                                     // RED
        atomicOr(sl.isum + (w >> 10), 1u << ((w >> 5) & 31));       // RED
        if (w < s) {
          c.fv += 1;                                                  // first visit of (s, w)
          atomicOr(sl.state + 2 * w, bit);                            // RED
          atomicOr(sl.rsum + (w >> 10), 1u << ((w >> 5) & 31));       // RED
          atomicOr(sl.state + 2 * w + 1, bit);                        // RED
          const int q = kH ? __ldg(p.pos + w) : w;                    // bitmap position
          atomicOr(sl.thr + (q >> 5), 1u << (q & 31));                // RED
          atomicOr(sl.tsum + (q >> 10), 1u << ((q >> 5) & 31));       // smem
        }
      }
    }
    fence_gpu();
    __syncthreads();
    if (warp == 0) {
      const int t0 = scan_next(sl.thr, sl.tsum, tbw, -1, lane);
      if (lane == 0) s_scan[0] = t0;
    }
    __syncthreads();

    // ---- thresholds in increasing order
    for (int step = 0;; ++step) {
      const int cur3 = step % 3, nx3 = (step + 1) % 3;
      const int T = min(s_scan[cur3], s_minfill[cur3]);
      if (T == INT_MAX) break;
      c.steps += 1;
      if (tid == 0) s_abort = p.abort_cycles > 0 && clock64() - t_start > p.abort_cycles;
      if (kH && tid == 0) {
        // the step: every threshold of height h = height(T), positions
        // [T, seg_end(h)); its record was usually prefetched with the scan
        // that found T (s_nx), else loaded now
        int lim, h;
        if (T == s_nx[0]) {
          lim = s_nx[1];
          h = s_nx[2];
        } else {
          const int4 r = __ldg(p.posrec + T);
          lim = r.w;
          h = __ldg(p.hgt + r.x);
        }
        s_hs[0] = lim;
        s_hs[1] = h;
        s_hs[2] = INT_MAX;
        s_hs[3] = -1;
      }
      __syncthreads();  // all threads are done with the previous step's s_qn / T
      if (s_abort) break;
      if (tid == 0) {
        s_scan[(step + 2) % 3] = INT_MAX;
        s_minfill[(step + 2) % 3] = INT_MAX;
      }
      int tmin = T, tmax = 0, hh = 0;
      if (kH) {
        // the step's thresholds (positions [T, lim), all final: fills are
        // ancestors, of greater height) become the first level's items (list1)
        const int lim = s_hs[0];
        const int w0 = T >> 5, w1 = (lim - 1) >> 5;
        int tmn = INT_MAX, tmx = -1;
        for (int si = (w0 >> 5) + warp; si <= (w1 >> 5); si += kWarps) {
          const int wi = (si << 5) + lane;
          uint32_t x = ((sl.tsum[si] >> lane) & 1u) && wi >= w0 && wi <= w1 ? __ldcg(sl.thr + wi) : 0u;
          if (wi == w0) x &= kFull << (T & 31);
          if (wi == w1 && (lim & 31)) x &= (1u << (lim & 31)) - 1u;
          for (;;) {
            const bool has = x != 0u;
            const uint32_t hb = __ballot_sync(kFull, has);
            if (!hb) break;
            int v = -1;
            if (has) {
              const int b = __ffs(x) - 1;
              x &= x - 1u;
              v = __ldg(&p.posrec[(wi << 5) + b].x);
              tmn = min(tmn, v);
              tmx = max(tmx, v);
            }
            int base = 0;
            if (lane == 0) base = atomicAdd(&s_qn[1], __popc(hb));
            base = __shfl_sync(kFull, base, 0);
            if (has) sl.list1[base + __popc(hb & lanemask_lt())] = (uint32_t)v;
          }
        }
        tmn = __reduce_min_sync(kFull, tmn);
        tmx = __reduce_max_sync(kFull, tmx);
        if (lane == 0 && tmx >= 0) {
          atomicMin(&s_hs[2], tmn);
          atomicMax(&s_hs[3], tmx);
        }
        __syncthreads();
        // the next threshold past the segment (this step's fills: s_minfill[nx3])
        // and its record, by the last warp (the one a small first level
        // leaves idle)
        if (warp == kWarps - 1) {
          const int nt = scan_next(sl.thr, sl.tsum, tbw, lim - 1, lane);
          if (lane == 0) {
            s_scan[nx3] = nt;
            if (nt != INT_MAX) {
              const int4 r = __ldg(p.posrec + nt);
              s_nx[1] = r.w;
              s_nx[2] = __ldg(p.hgt + r.x);
            }
            s_nx[0] = nt;
          }
        }
        tmin = s_hs[2];
        tmax = s_hs[3];
        hh = s_hs[1];
      } else {
        // level 0: warp 0 expands T itself; warp 1 finds the next threshold
        // above T in parallel (new fills of this step go to s_minfill[nx3])
        if (warp == 0) {
          expand(p, sl, s0g, T, lane == 0 ? T : -1, sl.list1, &s_qn[1], &s_minfill[nx3], lane, c);
        } else if (warp == 1) {
          const int nt = scan_next(sl.thr, sl.tsum, tbw, T, lane);
          if (lane == 0) s_scan[nx3] = nt;
        }
        __syncthreads();
      }
      c.levels += 1;
      // closure levels: every item has newMaxId T.  Levels only consume
      // returning atomics (reached, pend pushes); the REDs of this step
      // (fill pend / thr / is) are published before the next step's barrier.
      // One barrier per level: the item counts rotate over three words --
      // level l reads count l % 3, pushes into (l + 1) % 3 and clears
      // (l + 2) % 3, which every thread read at level l - 1 before its
      // barrier; the lists alternate (a level's barrier orders the reads of
      // one list before the next level's writes into it).
      for (int lvl = 1;; ++lvl) {
        const int cur = lvl & 1;
        const int qn = s_qn[lvl % 3];
        if (qn == 0) {
          fence_gpu();
          if (tid == 0) s_qn[0] = s_qn[1] = s_qn[2] = 0;  // (ordered by the next step's barrier)
          break;
        }
        const uint32_t *cq = cur ? sl.list1 : sl.list0;
        uint32_t *nq = cur ? sl.list0 : sl.list1;
        if (tid == 0) s_qn[(lvl + 2) % 3] = 0;
        c.levels += 1;
        for (int b0 = warp * 32; b0 < qn; b0 += kThreads) {
          const int u = (b0 + lane < qn) ? (int)cq[b0 + lane] : -1;
          expand<kH>(p, sl, s0g, tmin, u, nq, &s_qn[(lvl + 1) % 3], &s_minfill[nx3], lane, c, tmax, hh);
        }
        __syncthreads();
      }
    }

    __syncthreads();  // every thread's REDs were fenced at its last closure end
    const bool aborted = s_abort;
    t_trav = clock64();
    stage_rows<kWarps, false>(p, sl.is, sl.isum, s0g, nsrc, g, lane, warp, s_cnt, s_rowoff, s_nL, &s_ok,
                       !aborted);
    t_ext = clock64();
    __syncthreads();  // extraction done in every warp before the reset below
    // ---- reset the touched state lines (reached; pend is already 0) and thr
    {
      const int qr = (rsw + kWarps - 1) / kWarps;
      const int ra = min(rsw, warp * qr), rb = min(rsw, ra + qr);
      for (int i = ra; i < rb; ++i) {
        uint32_t x = __ldcg(sl.rsum + i);
        if (!x) continue;
        if (lane == 0) sl.rsum[i] = 0u;
        while (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1u;
          const int line = (i << 5) + b;
          reinterpret_cast<uint2 *>(sl.state)[(line << 5) + lane] = make_uint2(0u, 0u);
          if (!kH && lane == 0) sl.thr[line] = 0u;
        }
      }
      if (kH) {
        // threshold words sit at positions: the shared summary lists them
        for (int i = warp; i < ((tbw + 31) >> 5); i += kWarps)
          if ((sl.tsum[i] >> lane) & 1u) sl.thr[(i << 5) + lane] = 0u;
      }
    }
    // the clears above are plain stores; the next group's atomics on the same
    // words are performed at L2, so make the stores globally visible first
    __threadfence();
    if (aborted) {
      // the visit counters describe completed traversals only: the solo
      // kernel redoes this group from its seed
      c.fv = fv0;
      c.sx = sx0;
      // hand the group to the solo kernel (it restarts from the seed)
      __syncthreads();
      if (tid == 0) {
        const unsigned idx = atomicAdd(p.hq_tail, 1u);
        p.hq[idx] = g;
        __threadfence();
        atomicExch(p.hq_ready + idx, 1);
      }
    } else {
      if (p.group_trace && lane == 0) {
        long long *t = p.group_trace + 8 * (size_t)g;
        atomicAdd((unsigned long long *)&t[2], (unsigned long long)(c.items - it0));
        atomicAdd((unsigned long long *)&t[6], (unsigned long long)(c.pairs - pr0));
        if (warp == 0) {
          t[0] = (long long)(c.steps - st0);
          t[1] = (long long)(c.levels - lv0);
          t[3] = clock64() - t_start;
          t[4] = t_trav - t_start;
          t[5] = t_ext - t_trav;
          t[7] = 0;  // lockstep kernel
        }
      }
      if (tid == 0) atomicAdd(p.done, (unsigned)nsrc);  // rows completed
    }
    __syncthreads();
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    c.items += __shfl_xor_sync(kFull, c.items, d);
    c.edges += __shfl_xor_sync(kFull, c.edges, d);
    c.pairs += __shfl_xor_sync(kFull, c.pairs, d);
    c.fv += __shfl_xor_sync(kFull, c.fv, d);
    c.sx += __shfl_xor_sync(kFull, c.sx, d);
  }
  if (lane == 0) {
    atomicAdd(p.stats + 0, c.items);
    atomicAdd(p.stats + 1, c.edges);
    atomicAdd(p.stats + 4, c.pairs);
    atomicAdd(p.stats + 8, c.fv);
    atomicAdd(p.stats + 9, c.sx);
  }
  if (tid == 0) {
    atomicAdd(p.stats + 2, c.levels);
    atomicAdd(p.stats + 3, c.steps);
  }
  if (p.n < 0) p.stats[7] = c.sink;  // never true; keeps the returning atomics
  if (tid == 0 && p.light_live) {
    __threadfence();  // this CTA's queue pushes are visible before it leaves
    atomicSub(p.light_live, 1u);
  }
}

// ---------------------------------------------------------------- solo kernel
// Heavy sources (rows of top separators, hub rows): in threshold order the 32
// sources of such a group share few frontier items, and each is a long chain
// of |L(s,:)| threshold steps.  Here every warp runs ONE source on its own
// slot of per-source bitmaps (bit v of a word = vertex v), with no CTA
// barriers and no coupling to the other sources of its group:
//   * sources are tasks (queue entry e = t / 32, source k = t % 32); a warp's
//     first task is fixed so that the heaviest sources land on different SMs
//     (an SM's atomic issue rate, not latency alone, paces a chain when 32 of
//     them share it), later tasks come from a global counter;
//   * the queue holds groups: the top solo_top groups (pre-enqueued), groups
//     the lockstep kernel abandons, and fresh groups claimed by idle warps.
//
// Slot layout (uint32 words; all zero between sources):
//   reached[Vw] pend[Vw] thr[Vw]   bitmaps over [0, Vmax), Vw = Vmax/32
//   rsum[Vw/32] tsum[Vw/32]        touched reached words / nonzero thr words
//   is[nw] isum[nw/32]             in-structure bitmap over [0, n) + touched words
//   ring[R]                        closure overflow (vertex ids)
constexpr int kSoloQ = 64;  // shared-memory closure worklist entries per warp



__host__ __device__ inline size_t round4(size_t w) { return (w + 3) & ~(size_t)3; }

// A solo slot is one base pointer; the array offsets are recomputed from
// the launch parameters where they are used (fewer live registers: the
// kernel runs at the register budget of 32 warps per SM).
struct SoloSlot {
  uint32_t *base;
};

// slot offsets (in words) are computed on the host (solo_layout) and read
// from the kernel parameters: no per-use arithmetic, no registers
#define SL_REACHED (sl.base)
#define SL_PEND (sl.base + p.so_pend)
#define SL_THR (sl.base + p.so_thr)
#define SL_RSUM (sl.base + p.so_rsum)
#define SL_TSUM (sl.base + p.so_tsum)
#define SL_IS (sl.base + p.so_is)
#define SL_ISUM (sl.base + p.so_isum)
#define SL_QUEUE (sl.base + p.so_queue)
#define SL_QMASK (p.solo_ring - 1)

__device__ __forceinline__ SoloSlot solo_slot(const StreamParams &p, size_t slot) {
  return SoloSlot{p.hws + slot * p.hws_words};
}

__device__ __forceinline__ int solo_scan_next(const uint32_t *thr, const uint32_t *tsum, int tbw,
                                              int T, int lane) {
  const int start = T + 1;
  const int wi = start >> 5;
  if (wi >= tbw) return INT_MAX;
  uint32_t x = 0u;
  if (lane == 0) x = __ldcg(thr + wi) & (kFull << (start & 31));
  x = __shfl_sync(kFull, x, 0);
  if (x) return (wi << 5) + __ffs(x) - 1;
  const int nw = wi + 1;
  const int tsw = (tbw + 31) >> 5;
  for (int si = nw >> 5; si < tsw; si += 32) {
    const int idx = si + lane;
    uint32_t y = idx < tsw ? __ldcg(tsum + idx) : 0u;
    if (si == (nw >> 5) && lane == 0) y &= kFull << (nw & 31);
    const uint32_t b = __ballot_sync(kFull, y != 0u);
    if (b) {
      const int l = __ffs(b) - 1;
      const uint32_t yl = __shfl_sync(kFull, y, l);
      const int word = ((si + l) << 5) + __ffs(yl) - 1;
      const uint32_t z = __ldcg(thr + word);
      return (word << 5) + __ffs(z) - 1;
    }
  }
  return INT_MAX;
}

// Per-warp shared memory of the solo kernel.
//   win[32]   a window of 32 words (1024 vertices) of the threshold bitmap,
//             starting at word wb: thresholds found while the window covers
//             them are set here with shared-memory atomics, so finding the
//             next threshold costs no global round trip; thresholds beyond the
//             window go to the global bitmap + summary (REDs), published by
//             one fence when the window moves on
//   q*[kSoloQ] closure worklist: (w, rowptr[w], rowptr[w+1]); the row
//             pointers were loaded together with the atomic that reached w.
//             Overflow goes to the global ring (vertex only), then to pend.
// Reached-word cache (kC): a per-warp direct-mapped shared-memory table of
// reached-bitmap words known for the current source: {word index + 1, bits
// known set}.  Bits only get set during a source (the table is cleared when
// the next one starts), so a hit proves w was reached and its atomic can be
// skipped -- 78% of the (item, neighbour) atomics of C5 find w already
// reached (first visits 7.7e10 of 3.4e11 pairs).  Measured slower (C5 +7%,
// C2 +18%; profiles/r2/reached_cache_ab.txt): dev A/B only (GSOFA_RCACHE=1).
constexpr int kRC = 128;

struct SoloWarpSmem {
  uint32_t win[32];
  int qw[kSoloQ], qb[kSoloQ], qe[kSoloQ];
  uint32_t items, pairs, levels, steps;  // this source's counters (lane 0 updates)
  uint32_t fv;                           // first visits (vertices < s reached)
};

// Adjacency prefetch of the latency shape (kB > 1): when a closure member
// enters the shared-memory worklist its row pointers are already known, so
// its neighbour list is copied into shared memory right away with one bulk
// async copy (cp.async.bulk, completion on a per-slot mbarrier); when the item
// is expanded a level later its neighbours are read from shared memory, and
// the colidx round trip leaves the chain's critical path.  Lists that do not
// fit a 64-byte slot (with 16-byte alignment slack) are read from global
// memory as before.
// Measured slower (profiles/r2/tma_bulk_prefetch_ab.txt: 1.5-1.8x on C4/C5),
// so it is compiled only with -DGSOFA_ADJ_PREFETCH=1 (to reproduce the A/B).
#ifndef GSOFA_ADJ_PREFETCH
#define GSOFA_ADJ_PREFETCH 0
#endif
constexpr bool kAdjPrefetch = GSOFA_ADJ_PREFETCH != 0;
constexpr int kAdj = 16;  // ints per slot: the 16-byte-aligned span of <= 13 neighbours
struct alignas(128) SoloPF {
  int adj[kSoloQ][kAdj];
  unsigned long long bar[kSoloQ];
  uint32_t phase[kSoloQ / 32];  // per slot: parity of its next completion
};

__device__ __forceinline__ uint32_t smem_addr(const void *q) {
  return (uint32_t)__cvta_generic_to_shared(q);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void bulk_prefetch(int *dst, const int32_t *src, int bytes,
                                              unsigned long long *b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}

struct SoloQueue {
  int sh, st;      // shared-memory worklist head / tail (warp-uniform)
  int gh, gt;      // global ring head / tail
  bool spilled;    // items parked in pend
  int hold;        // slots below sh still being expanded (their prefetched lists are in use)
};

__device__ __forceinline__ uint32_t vbit(int v) { return 1u << (v & 31); }
// summary bit of word (v >> 5): word (v >> 10), bit ((v >> 5) & 31)
__device__ __forceinline__ void red_sum(uint32_t *sum, int v) {
  atomicOr(sum + (v >> 10), 1u << ((v >> 5) & 31));
}

// The thresholds of one step of source s, and how a newly reached w < s is
// classified.  Id order: one threshold T (tmin = tmax = T, h unused): a fill
// iff w > T, else a closure member.  Height order (order.cu): every
// threshold of one etree height h (ids tmin..tmax); a fill is an ancestor of
// one of them (so w > tmin) and a closure member a descendant (so w < tmax):
//   w > tmax -> fill,  w < tmin -> closure,  else fill iff height(w) > h
// (height(w) is loaded only for those in-between pairs).
struct SoloStep {
  int tmin, tmax, h;
};

// one closure item per lane into the worklist: shared memory, then the
// global ring, then parked in pend (push = this lane has an item)
// (pf: the latency shape's adjacency prefetch; qb's top bit marks a slot
// whose neighbour list is on its way to shared memory)
template <bool kPF>
__device__ __forceinline__ void solo_push(const StreamParams &p, const SoloSlot &sl,
                                          SoloWarpSmem &sw, SoloPF *pf, SoloQueue &Q, bool push,
                                          int wk, int rb, int re, int lane, uint32_t *ring,
                                          int rmask) {
  const uint32_t pb = __ballot_sync(kFull, push);
  if (!pb) return;
  const int pos = Q.st + __popc(pb & lanemask_lt());
  // (with prefetch, the slots of the items being expanded stay reserved:
  // their neighbour lists are read during this expansion)
  const bool in_s = pos - (Q.sh - (kPF ? Q.hold : 0)) < kSoloQ;
  if (push && in_s) {
    const int i = pos & (kSoloQ - 1);
    sw.qw[i] = wk;
    sw.qe[i] = re;
    if (kPF) {
      const int a = rb & ~3, e = (re + 3) & ~3;  // 16-byte aligned span
      const bool go = re > rb && e - a <= kAdj && e <= p.nnz;
      if (go) bulk_prefetch(pf->adj[i], p.colidx + a, (e - a) * 4, &pf->bar[i]);
      sw.qb[i] = go ? (rb | (int)0x80000000) : rb;
    } else {
      sw.qb[i] = rb;
    }
  }
  const uint32_t sb = __ballot_sync(kFull, push && in_s);
  Q.st += __popc(sb);
  const uint32_t gb = pb & ~sb;
  if (gb) {
    const int gpos = Q.gt + __popc(gb & lanemask_lt());
    const bool in_g = gpos - Q.gh <= rmask;
    if (push && !in_s) {
      if (in_g) ring[gpos & rmask] = (uint32_t)wk;
      else atomicOr(SL_PEND + (wk >> 5), vbit(wk));  // RED
    }
    Q.gt += __popc(__ballot_sync(kFull, push && !in_s && in_g));
    Q.spilled |= __ballot_sync(kFull, push && !in_s && !in_g) != 0u;
  }
}

// expand the closure items u (one per lane, -1 = none; beg/end = adjacency)
// of the current step t of source s.  Thresholds are kept at their bitmap
// position: the vertex id (id order) or pos(w) (height order, loaded for
// each new fill).
template <bool kH, int kB, bool kC = false>
__device__ __forceinline__ void solo_expand(const StreamParams &p, const SoloSlot &sl,
                                            SoloWarpSmem &sw, SoloPF *pf, int wb, SoloQueue &Q,
                                            int s, const SoloStep &t, int u, int beg, int end,
                                            int us, int lane, uint32_t *win, uint32_t *ring,
                                            int rmask, uint2 *rc = nullptr) {
  constexpr bool kPF = kB > 1 && kAdjPrefetch;  // us: this lane's prefetch slot (-1: none)
  const int deg = u >= 0 ? end - beg : 0;
  // fast path (every threshold's level 0, most closure levels of a chain):
  // one item in lane 0 with at most 32 neighbours -- lane j takes neighbour
  // j, no prefix scan or owner search on the chain's critical path
  const bool single = __ballot_sync(kFull, u >= 0) == 1u && __shfl_sync(kFull, deg, 0) <= 32;
  int incl = deg;
  if (!single) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += y;
    }
  }
  const int total = single ? __shfl_sync(kFull, deg, 0) : __shfl_sync(kFull, incl, 31);
  const int excl = incl - deg;
  {
    const uint32_t nitems = __popc(__ballot_sync(kFull, u >= 0));
    if (lane == 0) {
      sw.items += nitems;
      sw.pairs += (uint32_t)total;
      sw.levels += 1;
    }
  }
  // kB batches of 32 (item, neighbour) pairs are in flight at once:
  // all their colidx loads, then all their atomics, then the pushes
  for (int f0 = 0; f0 < total; f0 += 32 * kB) {
    int w[kB], rb[kB], re[kB], hw[kB], qw[kB];
    uint32_t ro[kB];
    const int nb = min(kB, (total - f0 + 31) >> 5);  // warp-uniform: skip empty batches
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      w[k] = s;
      if (k >= nb) continue;
      const int f = f0 + 32 * k + lane;
      if (single) {
        const int b0 = __shfl_sync(kFull, beg, 0);
        if (kPF) {
          const int s0 = __shfl_sync(kFull, us, 0);
          w[k] = f < total ? (s0 >= 0 ? pf->adj[s0][(b0 & 3) + f] : __ldg(p.colidx + b0 + f)) : s;
        } else {
          w[k] = f < total ? __ldg(p.colidx + b0 + f) : s;
        }
        continue;
      }
      int o = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int cand = o + step;
        const int e = __shfl_sync(kFull, excl, cand & 31);
        if (cand < 32 && e <= f) o = cand;
      }
      const int ob = __shfl_sync(kFull, beg, o);
      const int oe = __shfl_sync(kFull, excl, o);
      if (kPF) {
        const int os = __shfl_sync(kFull, us, o);
        w[k] = f < total ? (os >= 0 ? pf->adj[os][(ob & 3) + (f - oe)] : __ldg(p.colidx + ob + (f - oe)))
                         : s;
      } else {
        w[k] = f < total ? __ldg(p.colidx + ob + (f - oe)) : s;
      }
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      ro[k] = 1u;
      rb[k] = re[k] = 0;
      if (kH) {
        hw[k] = 0;
        qw[k] = w[k];
      }
      if (k >= nb) continue;
      const uint32_t bw = vbit(w[k]);
      // w > s: entry of U; w < s: atomicMin(maxId(w), T) succeeds
      // iff the source has not reached w yet (line 10 of fig:alg)
      bool known = false;
      if (kC && w[k] < s) {
        const uint2 e = rc[(w[k] >> 5) & (kRC - 1)];
        known = e.x == (uint32_t)(w[k] >> 5) + 1u && (e.y & bw);
      }
      ro[k] = w[k] < s && !known ? atomicOr(SL_REACHED + (w[k] >> 5), bw) : bw;
      if (w[k] > s) {
        // U entry: nothing waits for it -- two REDs (the summary bit is idempotent)
        atomicOr(SL_IS + (w[k] >> 5), bw);
        red_sum(SL_ISUM, w[k]);
      }
      // w < tmax may join the closure: its row pointers travel with the atomic
      if (w[k] < (kH ? t.tmax : t.tmin)) {  // (id order: the one threshold T = tmin)
        rb[k] = __ldg(p.rowptr + w[k]);
        re[k] = __ldg(p.rowptr + w[k] + 1);
      }
      if (kH && w[k] > t.tmin && w[k] < s) {
        // may be a fill: its threshold position travels with the atomic; between
        // the step's thresholds its height decides (height order)
        qw[k] = __ldg(p.pos + w[k]);
        if (w[k] < t.tmax) hw[k] = __ldg(p.hgt + w[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      if (k >= nb) continue;
      const int wk = w[k];
      const uint32_t bw = vbit(wk);
      if (kC && wk < s) rc[(wk >> 5) & (kRC - 1)] = make_uint2((uint32_t)(wk >> 5) + 1u, ro[k] | bw);
      bool push = false;
      if (!(ro[k] & bw)) {
        if (ro[k] == 0u) red_sum(SL_RSUM, wk);
        if (kH ? (wk > t.tmax || (wk > t.tmin && hw[k] > t.h)) : wk > t.tmin) {
          // fill of L(s,:) (R4); w becomes a threshold of this source
          atomicOr(SL_IS + (wk >> 5), bw);  // RED
          red_sum(SL_ISUM, wk);
          const int q = kH ? qw[k] : wk;  // its bitmap position
          const int d = (q >> 5) - wb;
          if (d < 32) {
            atomicOr(&win[d], vbit(q));  // smem (d >= 0: after the step's thresholds)
          } else {
            atomicOr(SL_THR + (q >> 5), vbit(q));  // RED
            red_sum(SL_TSUM, q);
          }
        } else {
          push = true;  // maxId(w) = T, not in the structure: continue with T
        }
      }
      solo_push<kPF>(p, sl, sw, pf, Q, push, wk, rb[k], re[k], lane, ring, rmask);
    }
  }
}

// ELL adjacency (id order, every row <= kEll entries): the neighbours of v
// are ell[kEll v .. kEll v + kEll), padded with -1, so a closure member's
// neighbour list depends on its id alone -- it is prefetched into L1 when
// the member is reached (in flight together with the reached atomic) and the
// next level reads it without waiting for row pointers.  Items map to lanes
// statically (4 items x 8 slots per 32-lane batch): no prefix sum or owner
// search.
constexpr int kEll = 8;

__device__ __forceinline__ void prefetch_l1(const void *q) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(q));
}

__device__ __forceinline__ void solo_expand_ell(const StreamParams &p, const SoloSlot &sl,
                                                SoloWarpSmem &sw, int wb, SoloQueue &Q, int s,
                                                int T, int u, int lane) {
  const int nitems = __popc(__ballot_sync(kFull, u >= 0));  // items sit in lanes 0 .. nitems-1
  uint32_t npairs = 0;
  for (int b0 = 0; b0 < nitems; b0 += 32 / kEll) {
    const int i = b0 + lane / kEll;
    const int ui = __shfl_sync(kFull, u, i & 31);
    int w = i < nitems ? __ldg(p.ell + (size_t)ui * kEll + (lane & (kEll - 1))) : -1;
    if (w < 0) w = s;  // padding: no pair
    npairs += __popc(__ballot_sync(kFull, w != s));
    const uint32_t bw = vbit(w);
    // w > s: entry of U; w < s: atomicMin(maxId(w), T) succeeds iff
    // the source has not reached w yet (line 10 of fig:alg)
    const uint32_t ro = w < s ? atomicOr(SL_REACHED + (w >> 5), bw) : bw;
    if (w > s) {
      atomicOr(SL_IS + (w >> 5), bw);  // RED
      red_sum(SL_ISUM, w);
    }
    if (w < T) prefetch_l1(p.ell + (size_t)w * kEll);  // a possible closure member
    bool push = false;
    if (!(ro & bw)) {
      if (ro == 0u) red_sum(SL_RSUM, w);
      if (w > T) {
        // fill of L(s,:) (R4); w becomes a threshold of this source
        atomicOr(SL_IS + (w >> 5), bw);  // RED
        red_sum(SL_ISUM, w);
        const int d = (w >> 5) - wb;
        if (d < 32) {
          atomicOr(&sw.win[d], bw);  // smem
        } else {
          atomicOr(SL_THR + (w >> 5), bw);  // RED
          red_sum(SL_TSUM, w);
        }
      } else {
        push = true;  // maxId(w) = T, not in the structure: continue with T
      }
    }
    solo_push<false>(p, sl, sw, nullptr, Q, push, w, -1, -1, lane, SL_QUEUE, SL_QMASK);
  }
  if (lane == 0) {
    sw.items += (uint32_t)nitems;
    sw.pairs += npairs;
    sw.levels += 1;
  }
}

// Next threshold of the source above T.  Inside the window: shared memory
// only.  Past it: publish this warp's global threshold REDs, scan the global
// bitmap (summary-guided) and load a new window at the found threshold.
__device__ __forceinline__ int solo_next_threshold(const uint32_t *thr, const uint32_t *tsum,
                                                   int tbw, int T, int &wb, uint32_t *win,
                                                   int lane) {
  if (wb >= 0) {
    const int d0 = (T + 1) >> 5;  // first candidate word
    const int rel = d0 - wb;
    if (rel < 32) {
      uint32_t x = lane >= rel ? win[lane] : 0u;
      if (lane == rel) x &= kFull << ((T + 1) & 31);
      const uint32_t b = __ballot_sync(kFull, x != 0u);
      if (b) {
        const int l = __ffs(b) - 1;
        const uint32_t xl = __shfl_sync(kFull, x, l);
        return ((wb + l) << 5) + __ffs(xl) - 1;
      }
    }
    T = max(T, ((wb + 32) << 5) - 1);  // the window holds nothing more
  }
  fence_gpu();  // this warp's global threshold REDs are visible to the scan
  __syncwarp();
  const int t = solo_scan_next(thr, tsum, tbw, T, lane);
  if (t == INT_MAX) return INT_MAX;
  wb = t >> 5;
  __syncwarp();
  win[lane] = wb + lane < tbw ? __ldcg(thr + wb + lane) : 0u;
  __syncwarp();
  return t;
}

// the max-id relaxation of source s in increasing threshold order -- by
// vertex id, or (kH) by etree height: the threshold bitmap is then indexed by
// position (vertices sorted by (height, id)) and a step takes every threshold
// of one height within the 32-word window (order.cu); the graph, reached and
// structure bitmaps stay in vertex ids (the ND order's locality)
template <bool kH, int kB, bool kE = false, bool kC = false>
__device__ __forceinline__ void solo_source(const StreamParams &p, const SoloSlot &sl, int s,
                                            int lane, SoloWarpSmem &sw, SoloPF *pf,
                                            uint2 *rc = nullptr) {
  if (kC) {
    // a new source: nothing is known reached yet
    for (int i = lane; i < kRC; i += 32) rc[i] = make_uint2(0u, 0u);
    __syncwarp();
  }
  constexpr bool kPF = kB > 1 && kAdjPrefetch;
  // threshold positions: below s (id order), anywhere in [0, n) (height order)
  const int tbw = kH ? (p.n + 31) >> 5 : (s + 31) >> 5;
  // seed: the out-neighbours of s are in the structure; the
  // smaller ones are reached with maxId -1 and are thresholds
  const int beg = __ldg(p.rowptr + s), end = __ldg(p.rowptr + s + 1);
  for (int j0 = beg; j0 < end; j0 += 32) {
    const int j = j0 + lane;
    const int w = j < end ? __ldg(p.colidx + j) : s;
    if (w == s) continue;
    const uint32_t bw = vbit(w);
    if (atomicOr(SL_IS + (w >> 5), bw) == 0u) red_sum(SL_ISUM, w);
    if (w < s) {
      if (atomicOr(SL_REACHED + (w >> 5), bw) == 0u) red_sum(SL_RSUM, w);
      const int q = kH ? __ldg(p.pos + w) : w;  // bitmap position
      atomicOr(SL_THR + (q >> 5), vbit(q));     // RED
      red_sum(SL_TSUM, q);
    }
  }
  __syncwarp();
  int wb = -1;  // no window yet
  int P = -1;   // the last threshold (position) taken
  for (;;) {
    P = solo_next_threshold(SL_THR, SL_TSUM, tbw, P, wb, sw.win, lane);
    if (P == INT_MAX) break;
    if (lane == 0) sw.steps += 1;
    SoloQueue Q = {0, 0, 0, 0, false, 0};
    int u = -1, ub = 0, ue = 0;
    SoloStep t;
    if (kH) {
      // the step: every threshold of h = height(P) in the window at or after
      // P, i.e. positions [P, min(seg_end(h), window end)); the first word's
      // items go to the lanes, the others to the worklist
      // {vertex, rowptr, rowptr + 1, end of its height's segment}: one load
      const int lim = min(__ldg(&p.posrec[P].w), (wb + 32) << 5);
      int tmin = INT_MAX, tmax = -1, hh = 0;
      for (int wi = P >> 5; (wi << 5) < lim; ++wi) {
        uint32_t x = sw.win[wi - wb];
        if (wi == (P >> 5)) x &= kFull << (P & 31);
        if (lim - (wi << 5) < 32) x &= (1u << (lim - (wi << 5))) - 1u;
        const bool has = (x >> lane) & 1u;
        int v = -1, vb = 0, ve = 0;
        if (has) {
          const int4 r = __ldg(p.posrec + (wi << 5) + lane);
          v = r.x;
          vb = r.y;
          ve = r.z;
          tmin = min(tmin, v);
          tmax = max(tmax, v);
          hh = __ldg(p.hgt + v);  // the step's height (used between tmin and tmax only)
        }
        if (wi == (P >> 5)) {
          // compact to the low lanes (the single-item fast path)
          const uint32_t b = __ballot_sync(kFull, has);
          const int src = __fns(b, 0, lane + 1) & 31;
          const int cu = __shfl_sync(kFull, v, src), cb = __shfl_sync(kFull, vb, src),
                    ce = __shfl_sync(kFull, ve, src);
          const bool ok = lane < __popc(b);
          u = ok ? cu : -1;
          ub = ok ? cb : 0;
          ue = ok ? ce : 0;
        } else {
          solo_push<kPF>(p, sl, sw, pf, Q, has, v, vb, ve, lane, SL_QUEUE, SL_QMASK);
        }
      }
      t.tmin = __reduce_min_sync(kFull, tmin);
      t.tmax = __reduce_max_sync(kFull, tmax);
      t.h = __reduce_max_sync(kFull, hh);
      P = lim - 1;  // the next step starts after these positions
    } else {
      t.tmin = P;  // the one threshold (tmax / h unused in id order)
      if (lane == 0) {
        u = P;
        if (!kE) {  // (ELL: the neighbour list needs no row pointers)
          ub = __ldg(p.rowptr + P);
          ue = __ldg(p.rowptr + P + 1);
        }
      }
    }
    // first visits (R11): every vertex newly reached below s is either a
    // closure member (pushed once, counted here per step) or a structure
    // member (a seed or a fill: |L(s,:)|, added when the row is staged)
    const int pushed0 = Q.st + Q.gt;  // the step's own thresholds queued above
    int us = -1;  // prefetch slot of this lane's item
    for (;;) {
      if (kE) solo_expand_ell(p, sl, sw, wb, Q, s, t.tmin, u, lane);
      else solo_expand<kH, kB, kC>(p, sl, sw, pf, wb, Q, s, t, u, ub, ue, us, lane, sw.win, SL_QUEUE, SL_QMASK, rc);
      __syncwarp();
      us = -1;
      if (kPF) Q.hold = 0;
      if (Q.sh < Q.st) {
        const int cnt = min(32, Q.st - Q.sh);
        if (kPF) Q.hold = cnt;
        u = -1;
        int i = 0;
        if (lane < cnt) {
          i = (Q.sh + lane) & (kSoloQ - 1);
          u = sw.qw[i];
          if (!kE) {
            ub = sw.qb[i];
            ue = sw.qe[i];
          }
          if (kPF && ub < 0) {
            // its neighbour list was prefetched: wait for the bytes, then
            // the slot's barrier is in its next phase
            ub &= 0x7FFFFFFF;
            us = i;
            mbar_wait(&pf->bar[i], (pf->phase[i >> 5] >> (i & 31)) & 1u);
            atomicXor(&pf->phase[i >> 5], 1u << (i & 31));
          }
        }
        Q.sh += cnt;
        __syncwarp();
        continue;
      }
      if (Q.gh >= Q.gt && Q.spilled) {
        // the ring overflowed during this closure: move parked items (pend
        // bits, all below tmax) back into the ring, as many as fit
        Q.spilled = false;
        __syncwarp();
        fence_gpu();
        const int pwords = ((kH ? t.tmax : t.tmin) + 31) >> 5;
        for (int w0 = 0; w0 < pwords && !Q.spilled; w0 += 32) {
          const int wi = w0 + lane;
          uint32_t x = wi < pwords ? __ldcg(SL_PEND + wi) : 0u;
          for (;;) {
            const bool has = x != 0u;
            const uint32_t hb = __ballot_sync(kFull, has);
            if (!hb) break;
            const int pos = Q.gt + __popc(hb & lanemask_lt());
            const bool fits = pos - Q.gh <= SL_QMASK;
            if (has && fits) {
              const int b = __ffs(x) - 1;
              x &= x - 1u;
              atomicAnd(SL_PEND + wi, ~(1u << b));  // RED (result unused)
              SL_QUEUE[pos & SL_QMASK] = (uint32_t)((wi << 5) + b);
            }
            Q.gt += __popc(__ballot_sync(kFull, has && fits));
            if (__ballot_sync(kFull, has && !fits)) {
              Q.spilled = true;  // still more parked: rescan after this batch drains
              break;
            }
          }
        }
        __syncwarp();
      }
      if (Q.gh >= Q.gt) {
        if (lane == 0) sw.fv += (uint32_t)(Q.st + Q.gt - pushed0);
        break;
      }
      const int cnt = min(32, Q.gt - Q.gh);
      u = lane < cnt ? (int)SL_QUEUE[(Q.gh + lane) & SL_QMASK] : -1;
      Q.gh += cnt;
      if (u >= 0 && !kE) {
        ub = __ldg(p.rowptr + u);
        ue = __ldg(p.rowptr + u + 1);
      }
    }
  }
}

// Row s from the per-source structure bitmap: L(s,:) = bits below s, U(s,:) =
// s then the bits above s, ascending; staged at one reservation; the bitmap
// words read are zeroed.  Returns false if the staging area was full.
__device__ __forceinline__ bool solo_stage_row(const StreamParams &p, const SoloSlot &sl, int s,
                                               int r, int g, int lane, SoloWarpSmem &sw) {
  const int ns = (((p.n + 31) >> 5) + 31) >> 5;
  // count pass: lane handles summary words i0 + lane (1024 vertices each)
  uint32_t cl = 0, cu = 0;
  for (int i0 = 0; i0 < ns; i0 += 32) {
    const int i = i0 + lane;
    uint32_t x = i < ns ? __ldcg(SL_ISUM + i) : 0u;
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1u;
      const int wi = (i << 5) + b, v0 = wi << 5;
      const uint32_t y = __ldcg(SL_IS + wi);
      const int d = s - v0;  // bits below d are < s, above d are > s
      const uint32_t lm = d <= 0 ? 0u : (d >= 32 ? kFull : ((1u << d) - 1u));
      const uint32_t um = d < 0 ? kFull : (d >= 31 ? 0u : (kFull << (d + 1)));
      cl += __popc(y & lm);
      cu += __popc(y & um);
    }
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    cl += __shfl_xor_sync(kFull, cl, d);
    cu += __shfl_xor_sync(kFull, cu, d);
  }
  const unsigned long long tot = (unsigned long long)cl + cu + 1;  // + the diagonal
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(p.stage_cursor, tot);
  base = __shfl_sync(kFull, base, 0);
  const bool ok = base + tot <= p.stage_cap;
  if (lane == 0) {
    p.row_off[r] = ok ? (long long)base : -1;
    p.row_nL[r] = (int)cl;
    sw.fv += cl;  // the seeds and fills below s: first visits too
    p.row_nU[r] = (int)cu + 1;
    if (ok) {
      p.stage[base + cl] = s;  // U(s,:) starts with the diagonal
    } else {
      // the retry pass re-runs the whole group: ask for room for all of it
      if (atomicExch(p.failed_flag + g, 1) == 0) p.failed[atomicAdd(p.nfailed, 1)] = g;
      atomicAdd(p.failed_need, tot * 32ull);
    }
  }
  // write pass (zeroes what it reads): per summary word, lanes in ascending order
  long long pl = (long long)base, pu = (long long)base + cl + 1;
  for (int i0 = 0; i0 < ns; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t x0 = i < ns ? __ldcg(SL_ISUM + i) : 0u;
    if (!__ballot_sync(kFull, x0 != 0u)) continue;
    if (x0) SL_ISUM[i] = 0u;
    uint32_t nl = 0, nu = 0;
    for (uint32_t x = x0; x;) {
      const int b = __ffs(x) - 1;
      x &= x - 1u;
      const int wi = (i << 5) + b, v0 = wi << 5;
      const uint32_t y = __ldcg(SL_IS + wi);
      const int d = s - v0;
      const uint32_t lm = d <= 0 ? 0u : (d >= 32 ? kFull : ((1u << d) - 1u));
      const uint32_t um = d < 0 ? kFull : (d >= 31 ? 0u : (kFull << (d + 1)));
      nl += __popc(y & lm);
      nu += __popc(y & um);
    }
    uint32_t el = nl, eu = nu;  // inclusive prefix over lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t a = __shfl_up_sync(kFull, el, d), bb = __shfl_up_sync(kFull, eu, d);
      if (lane >= d) {
        el += a;
        eu += bb;
      }
    }
    long long ol = pl + el - nl, ou = pu + eu - nu;
    for (uint32_t x = x0; x;) {
      const int b = __ffs(x) - 1;
      x &= x - 1u;
      const int wi = (i << 5) + b, v0 = wi << 5;
      uint32_t y = __ldcg(SL_IS + wi);
      SL_IS[wi] = 0u;
      if (!ok) continue;
      while (y) {
        const int v = v0 + __ffs(y) - 1;
        y &= y - 1u;
        if (v < s) p.stage[ol++] = v;
        else p.stage[ou++] = v;
      }
    }
    pl += __shfl_sync(kFull, el, 31);
    pu += __shfl_sync(kFull, eu, 31);
  }
  return ok;
}

// Two shapes: kB = 1: 48 warps per SM (40 registers, one
// 32-pair batch in flight per warp) -- the throughput shape, measured best
// against 32 warps / 64 registers and 64 warps / 32 registers when sources
// outnumber warps; kB = 4 ("wide"): 32 warps per SM, a level's first 128
// pairs in flight at once -- the latency shape for chain-bound sources (few
// heavy sources: C4's hub rows, the top-separator ranges of a multi-GPU split)
template <bool kH, int kB, bool kE = false, bool kC = false>
__global__ void __launch_bounds__(kSoloWarps * 32, kB == 1 ? 48 / kSoloWarps : 32 / kSoloWarps)
    solo_kernel(StreamParams p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rows = p.nrows;
  const size_t slot = (size_t)blockIdx.x * kSoloWarps + warp;
  const SoloSlot sl = solo_slot(p, slot);
  const int Vs = (int)(p.so_tsum - p.so_rsum);  // reached-word summary words
  __shared__ SoloWarpSmem s_sw[kSoloWarps];
  SoloWarpSmem &sw = s_sw[warp];
  __shared__ uint2 s_rc[kC ? kSoloWarps * kRC : 1];  // reached-word caches (kC)
  uint2 *rc = kC ? s_rc + warp * kRC : nullptr;
  extern __shared__ __align__(128) unsigned char s_dyn[];  // latency shape: SoloPF per warp
  SoloPF *pf = nullptr;
  if (kB > 1 && kAdjPrefetch) {
    pf = reinterpret_cast<SoloPF *>(s_dyn) + warp;
    for (int i = lane; i < kSoloQ; i += 32) mbar_init(&pf->bar[i]);
    if (lane < kSoloQ / 32) pf->phase[lane] = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (lane == 0) sw.items = sw.pairs = sw.levels = sw.steps = sw.fv = 0u;
  __syncwarp();
  // first task: warp-major over the grid, so consecutive (heaviest) sources
  // start on different SMs; then the global task counter
  long long t = (long long)warp * gridDim.x + blockIdx.x + p.task_base;
  const long long t_static = (long long)kSoloWarps * gridDim.x + p.task_base;
  for (bool first = true;; first = false) {
    if (!first) {
      if (lane == 0) t = t_static + (long long)atomicAdd(p.task_ctr, 1ull);
      t = __shfl_sync(kFull, t, 0);
    }
    const unsigned e = (unsigned)(t >> 5);
    const int k = (int)(t & 31);
    int g = -1;
    if (lane == 0) {
      for (;;) {
        if (e < *(volatile unsigned *)p.hq_tail) {
          while (*(volatile int *)(p.hq_ready + e) == 0) __nanosleep(200);
          g = *(volatile int *)(p.hq + e);
          break;
        }
        // entry e does not exist yet: claim a fresh group (heaviest first)
        // and queue it, unless every row is done
        const int nfresh = p.ngroups - p.solo_top;
        if (*(volatile unsigned *)p.group_ctr < (unsigned)nfresh) {
          const int j = (int)atomicAdd(p.group_ctr, 1u);
          if (j < nfresh) {
            const unsigned idx = atomicAdd(p.hq_tail, 1u);
            p.hq[idx] = nfresh - 1 - j;
            __threadfence();
            atomicExch(p.hq_ready + idx, 1);
            continue;
          }
        }
        if (*(volatile unsigned *)p.done >= (unsigned)rows) break;
        // no lockstep CTA left to abandon a group and every fresh group
        // claimed: entry e can no longer appear, so this warp is done (idle
        // polling took ~40% of issue slots in chain-bound tails, ncu)
        if (p.light_live && *(volatile unsigned *)p.light_live == 0u &&
            *(volatile unsigned *)p.group_ctr >= (unsigned)nfresh) {
          __threadfence();
          if (e >= *(volatile unsigned *)p.hq_tail) break;
          continue;
        }
        __nanosleep(2000);
      }
    }
    g = __shfl_sync(kFull, g, 0);
    if (g < 0) break;
    const int r = 32 * g + k;  // local row
    if (r >= rows) continue;   // tail of the last group
    const int s = p.map.row(r);
    if (p.src_trace && lane == 0) {
      // dev trace (GSOFA_SRC_TRACE): start / end ns, steps, levels of this source
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      p.src_trace[4 * (size_t)r] = (long long)t0;
    }
    solo_source<kH, kB, kE, kC>(p, sl, s, lane, sw, pf, rc);
    if (p.src_trace && lane == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      long long *tr = p.src_trace + 4 * (size_t)r;
      tr[1] = (long long)t1;
      tr[2] = sw.steps;
      tr[3] = sw.levels;
    }
    fence_gpu();  // this warp's REDs are visible to its extraction
    __syncwarp();
    solo_stage_row(p, sl, s, r, g, lane, sw);
    // reset the touched words: reached | pend (| thr in id order, where a
    // threshold bit sits in the word of its reached bit), and the summaries
    for (int i0 = 0; i0 < Vs; i0 += 32) {
      const int i = i0 + lane;
      uint32_t x = i < Vs ? __ldcg(SL_RSUM + i) : 0u;
      if (x) {
        SL_RSUM[i] = 0u;
        if (!kH) SL_TSUM[i] = 0u;
      }
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1u;
        const int wi = (i << 5) + b;
        SL_REACHED[wi] = 0u;
        SL_PEND[wi] = 0u;
        if (!kH) SL_THR[wi] = 0u;
      }
    }
    if (kH) {
      // height order: threshold bits sit at positions; the summary lists the
      // global words written (window bits never reach global memory)
      const int Ts = (int)(p.so_is - p.so_tsum);
      for (int i0 = 0; i0 < Ts; i0 += 32) {
        const int i = i0 + lane;
        uint32_t x = i < Ts ? __ldcg(SL_TSUM + i) : 0u;
        if (x) SL_TSUM[i] = 0u;
        while (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1u;
          SL_THR[(i << 5) + b] = 0u;
        }
      }
    }
    // the clears are plain stores; the next source's atomics act at L2
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      atomicAdd(p.stats + 0, (unsigned long long)sw.items);
      atomicAdd(p.stats + 1, (unsigned long long)sw.pairs);  // solo: one source per item
      atomicAdd(p.stats + 4, (unsigned long long)sw.pairs);
      atomicAdd(p.stats + 2, (unsigned long long)sw.levels);
      atomicAdd(p.stats + 3, (unsigned long long)sw.steps);
      atomicAdd(p.stats + 8, (unsigned long long)sw.fv);
      atomicAdd(p.stats + 9, (unsigned long long)sw.items);  // solo: items are per source
      atomicAdd(p.done, 1u);
      sw.items = sw.pairs = sw.levels = sw.steps = sw.fv = 0u;
    }
    __syncwarp();
  }
}


// copies each staged row into the final CSR arrays (warp per row)
__global__ void gather_kernel(const int32_t *stage, const int64_t *row_off, const int32_t *row_nL,
                              const int64_t *L_rowptr, const int64_t *U_rowptr, int rows,
                              int32_t *L_out, int32_t *U_out) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t off = row_off[r];
  const int nl = row_nL[r];
  const int64_t lo = L_rowptr[r], uo = U_rowptr[r];
  const int nu = (int)(U_rowptr[r + 1] - uo);
  for (int i = lane; i < nl; i += 32) L_out[lo + i] = stage[off + i];
  for (int i = lane; i < nu; i += 32) U_out[uo + i] = stage[off + nl + i];
}
}  // namespace

// npos > 0: height order (threshold bitmap over npos positions)
size_t stream_ws_words(int64_t Vmax, int64_t npos) {
  const int64_t tb = npos > 0 ? npos : Vmax;
  const size_t w = 2 * (size_t)Vmax + (size_t)((tb + 31) / 32) + (size_t)((Vmax + 1023) / 1024) +
                   2 * (size_t)Vmax;
  return (w + 7) / 8 * 8;
}

size_t stream_is_words(int64_t n) {
  const size_t w = (size_t)n + (size_t)((n + 1023) / 1024);
  return (w + 7) / 8 * 8;
}

size_t stream_smem_bytes(int64_t Vmax, int64_t npos) {
  const int64_t tb = npos > 0 ? npos : Vmax;
  return (size_t)((((tb + 31) / 32) + 31) / 32) * 4;
}

// kernel instances of the two threshold orders (kH = height order)
// warps per lockstep CTA in height order: 32 when every group of the call
// gets its own SM at once (a hub group is one CTA's work: C4's hub rank
// 324 -> 238 ms vs 16 warps); else 16 for hub patterns (C4 whole: 368 ms vs
// 556 with 8 warps -- its hub groups are long) and 8 otherwise (more groups
// in flight: C5 2,260 vs 2,369 ms with 16, 3,816 with 4, 3,687 with 32);
// GSOFA_LOCK_WARPS = 4 / 8 / 16 / 32 forces it (dev A/B)
int lock_warps(int64_t groups, int sms, bool hubs) {
  if (const char *e = std::getenv("GSOFA_LOCK_WARPS")) {
    const int w = atoi(e);
    if (w == 4 || w == 8 || w == 16 || w == 32) return w;
  }
  if (groups <= (int64_t)sms) return 32;
  return hubs ? 16 : 8;
}
const void *stream_fn(bool h, int lw) {
  if (!h) return (const void *)stream_kernel<false>;
  switch (lw) {
    case 4: return (const void *)stream_kernel<true, 4>;
    case 8: return (const void *)stream_kernel<true, 8>;
    case 32: return (const void *)stream_kernel<true, 32>;
    default: return (const void *)stream_kernel<true, 16>;
  }
}

const void *solo_fn(bool h, bool wide) {
  if (wide) return h ? (const void *)solo_kernel<true, 4> : (const void *)solo_kernel<false, 4>;
  return h ? (const void *)solo_kernel<true, 1> : (const void *)solo_kernel<false, 1>;
}

// dynamic shared memory of the solo kernel: the latency shape's prefetch slots
size_t solo_dyn_smem(bool wide) { return wide && kAdjPrefetch ? sizeof(SoloPF) * kSoloWarps : 0; }

int stream_max_blocks(int device, int64_t Vmax, int heavy, int64_t npos, bool wide, bool lock_h, int lw) {
  int sms = 0, per = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  cudaError_t e;
  const bool h = heavy ? npos > 0 : lock_h;
  if (heavy) {
    const size_t dyn = solo_dyn_smem(wide);
    if (dyn && cudaFuncSetAttribute(solo_fn(h, wide), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)dyn) != cudaSuccess)
      return 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, solo_fn(h, wide), kSoloWarps * 32, dyn);
  } else {
    const size_t smem = stream_smem_bytes(Vmax, lock_h ? npos : 0);  // lockstep: id or height order
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(stream_fn(h, lw), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stream_fn(h, lw), (h ? lw : kLightWarps) * 32, smem);
  }
  if (e != cudaSuccess) return 0;
  return sms * per;
}

int stream_heavy_ratio() { return kSoloWarps / kLightWarps; }

int stream_warps_per_cta() { return 1; }  // slots are CTAs

// lockstep CTAs that still fit on an SM next to one solo CTA
int stream_light_per_sm_with_solo(int device, int64_t Vmax, int64_t npos, bool wide) {
  cudaFuncAttributes fs, fl;
  const bool h = npos > 0;
  if (cudaFuncGetAttributes(&fs, solo_fn(h, wide)) != cudaSuccess ||
      cudaFuncGetAttributes(&fl, stream_fn(false, kLightWarps)) != cudaSuccess)  // next to a solo CTA: id order
    return 0;
  int regs = 0, warps = 0, smem_sm = 0;
  cudaDeviceGetAttribute(&regs, cudaDevAttrMaxRegistersPerMultiprocessor, device);
  cudaDeviceGetAttribute(&warps, cudaDevAttrMaxThreadsPerMultiProcessor, device);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  warps /= 32;
  const int solo_regs = ((fs.numRegs * 32 + 255) / 256 * 256) * kSoloWarps;
  const int light_regs = ((fl.numRegs * 32 + 255) / 256 * 256) * kLightWarps;
  const int by_regs = (regs - solo_regs) / light_regs;
  const int by_warps = (warps - kSoloWarps) / kLightWarps;
  const size_t light_smem = fl.sharedSizeBytes + stream_smem_bytes(Vmax, 0) + 1024;
  const int by_smem =
      (int)((smem_sm - fs.sharedSizeBytes - solo_dyn_smem(wide) - 1024) / light_smem);
  return std::max(0, std::min(std::min(by_regs, by_warps), by_smem));
}

// closure ring entries per solo slot: a power of two; GSOFA_SOLO_RING (dev /
// tests) forces a smaller one to exercise the pend-bitmap spill
int solo_ring(int64_t Vmax) {
  int r = 1024;
  while (r < 16384 && r < Vmax) r <<= 1;
  if (const char *e = std::getenv("GSOFA_SOLO_RING")) {
    const int f = atoi(e);
    if (f >= 32 && (f & (f - 1)) == 0) r = std::min(r, f);
  }
  return r;
}

// solo slot layout (words): reached, pend [Vw] (bitmaps over [0, Vmax));
// thr [Tw] (over vertices, or positions in height order); rsum [Vs], tsum
// [Ts] (summaries: one bit per word); is [nw], isum [ns] (structure over
// [0, n)); the closure ring.  npos > 0: height order.  Returns the total.
size_t solo_layout(int64_t Vmax, int64_t n, int64_t npos, StreamParams *p) {
  // reached / pend over vertex ids [0, Vmax); thr over ids [0, Vmax) or
  // positions [0, npos) (height order)
  const size_t Vw = round4((size_t)((Vmax + 31) / 32)), Vs = round4((Vw + 31) / 32);
  const size_t Tw = npos > 0 ? round4((size_t)((npos + 31) / 32)) : Vw, Ts = round4((Tw + 31) / 32);
  const size_t nw = round4((size_t)((n + 31) / 32)), ns = round4((nw + 31) / 32);
  if (p) {
    p->so_pend = (uint32_t)Vw;
    p->so_thr = (uint32_t)(2 * Vw);
    p->so_rsum = (uint32_t)(2 * Vw + Tw);
    p->so_tsum = p->so_rsum + (uint32_t)Vs;
    p->so_is = p->so_tsum + (uint32_t)Ts;
    p->so_isum = p->so_is + (uint32_t)nw;
    p->so_queue = p->so_isum + (uint32_t)ns;
  }
  const size_t w = 2 * Vw + Tw + Vs + Ts + nw + ns + (size_t)solo_ring(Vmax);
  return (w + 7) / 8 * 8;
}

size_t solo_ws_words(int64_t Vmax, int64_t n, int64_t npos) { return solo_layout(Vmax, n, npos, nullptr); }

int solo_warps_per_cta() { return kSoloWarps; }

cudaError_t launch_stream(const StreamParams &p, int grid, cudaStream_t st) {
  if (grid <= 0) return cudaSuccess;
  const bool h = p.lmode != 0;
  const size_t smem = stream_smem_bytes(p.Vmax, h ? p.npos : 0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(stream_fn(h, p.lwarps), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (!h) {
    stream_kernel<false><<<grid, kLightWarps * 32, smem, st>>>(p);
  } else {
    switch (p.lwarps) {
      case 4: stream_kernel<true, 4><<<grid, 4 * 32, smem, st>>>(p); break;
      case 8: stream_kernel<true, 8><<<grid, 8 * 32, smem, st>>>(p); break;
      case 32: stream_kernel<true, 32><<<grid, 32 * 32, smem, st>>>(p); break;
      default: stream_kernel<true, 16><<<grid, 16 * 32, smem, st>>>(p); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_solo(const StreamParams &p, int grid, cudaStream_t st) {
  if (grid <= 0) return cudaSuccess;
  if (p.wide) {
    const size_t dyn = solo_dyn_smem(true);
    if (dyn) {
      cudaError_t e = cudaFuncSetAttribute(solo_fn(p.hmode, true),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return e;
    }
    if (p.hmode) solo_kernel<true, 4><<<grid, kSoloWarps * 32, dyn, st>>>(p);
    else solo_kernel<false, 4><<<grid, kSoloWarps * 32, dyn, st>>>(p);
  } else {
    if (p.hmode) solo_kernel<true, 1><<<grid, kSoloWarps * 32, 0, st>>>(p);
    else if (p.ell) solo_kernel<false, 1, true><<<grid, kSoloWarps * 32, 0, st>>>(p);
    else if (std::getenv("GSOFA_RCACHE") && atoi(std::getenv("GSOFA_RCACHE")) != 0)  // A/B
      solo_kernel<false, 1, false, true><<<grid, kSoloWarps * 32, 0, st>>>(p);
    else solo_kernel<false, 1><<<grid, kSoloWarps * 32, 0, st>>>(p);
  }
  return cudaGetLastError();
}

cudaError_t launch_gather(const int32_t *stage, const int64_t *row_off, const int32_t *row_nL,
                          const int64_t *L_rowptr, const int64_t *U_rowptr, int rows,
                          int32_t *L_out, int32_t *U_out, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  gather_kernel<<<(rows + 7) / 8, 256, 0, st>>>(stage, row_off, row_nL, L_rowptr, U_rowptr, rows,
                                                L_out, U_out);
  return cudaGetLastError();
}

namespace {
__global__ void ell_build_kernel(const int32_t *rowptr, const int32_t *colidx, int32_t n,
                                 int32_t *ell) {
  const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int32_t a = rowptr[v], d = rowptr[v + 1] - a;
  int r[kEll];
#pragma unroll
  for (int j = 0; j < kEll; ++j) r[j] = j < d ? colidx[a + j] : -1;
  int4 *o = reinterpret_cast<int4 *>(ell + (size_t)v * kEll);
  o[0] = make_int4(r[0], r[1], r[2], r[3]);
  o[1] = make_int4(r[4], r[5], r[6], r[7]);
}
}  // namespace

cudaError_t launch_ell_build(const int32_t *rowptr, const int32_t *colidx, int32_t n, int32_t *ell,
                             cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ell_build_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rowptr, colidx, n, ell);
  return cudaGetLastError();
}

}  // namespace gsofa
