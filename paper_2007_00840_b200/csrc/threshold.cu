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
#include <climits>

#include "gsofa_internal.cuh"

namespace gsofa {

namespace {
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kLightWarps = 4;   // CTA of the light kernel (most groups)
constexpr int kHeavyWarps = 16;  // CTA of the heavy kernel (the heaviest groups)

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

__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int j = 16 >> i;
    const uint32_t m = masks[i];
    const uint32_t y = __shfl_xor_sync(kFull, x, j);
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
  }
  return x;
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
__device__ __forceinline__ void expand(const StreamParams &p, const Slot &sl, int s0g, int T,
                                       int u, uint32_t *nq, int *nqn, int *minfill, int lane,
                                       Counters &c) {
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
      push[k] = false;
      po[k] = kFull;
      if (nw) {
        if (w[k] > T) {
          // newMaxId T < w: (src, w) is a fill of L (R4); w proposes newMaxId
          // = w later, as a threshold
          atomicOr(sl.is + w[k], nw);                                           // RED
          atomicOr(sl.isum + (w[k] >> 10), 1u << ((w[k] >> 5) & 31));          // RED
          atomicOr(sl.state + 2 * w[k] + 1, nw);                                // RED
          atomicOr(sl.thr + (w[k] >> 5), 1u << (w[k] & 31));                    // RED
          atomicOr(sl.tsum + (w[k] >> 10), 1u << ((w[k] >> 5) & 31));          // smem
          atomicMin(minfill, w[k]);                                             // smem
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

__device__ __forceinline__ void split_masks(int d, uint32_t &lm, uint32_t &um) {
  lm = d <= 0 ? 0u : (d >= 32 ? kFull : ((1u << d) - 1u));
  um = d < 0 ? kFull : (d >= 31 ? 0u : (kFull << (d + 1)));
}

template <int kWarps>
__global__ void __launch_bounds__(kWarps * 32, kWarps == kLightWarps ? 8 : 2)
    stream_kernel(StreamParams p, int slot_base, int heavy) {
  constexpr int kThreads = kWarps * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const int n = p.n, Vmax = p.Vmax;
  const int tbw_max = (Vmax + 31) >> 5;
  const int rsw = (Vmax + 1023) >> 10;
  const int isw = (n + 1023) >> 10;
  Slot sl;
  const size_t slot = (size_t)slot_base + blockIdx.x;
  sl.state = p.ws + slot * p.ws_words;
  sl.thr = sl.state + 2 * (size_t)Vmax;
  sl.rsum = sl.thr + tbw_max;
  sl.list0 = sl.rsum + rsw;
  sl.list1 = sl.list0 + Vmax;
  sl.is = p.is + slot * p.is_words;
  sl.isum = sl.is + n;
  extern __shared__ uint32_t s_tsum[];  // [(tbw_max + 31) / 32]
  sl.tsum = s_tsum;

  __shared__ int s_g, s_qn[2], s_scan[3], s_minfill[3];
  __shared__ uint32_t s_cnt[kWarps][2][32];
  __shared__ long long s_rowoff[32];
  __shared__ int s_nL[32];
  __shared__ int s_ok;
  Counters c = {0, 0, 0, 0, 0, 0u};

  for (;;) {
    if (tid == 0) {
      // heaviest first: group ngroups-1-j is the j-th taken; the heavy kernel
      // owns the first n_heavy of them, then helps with the rest
      int gg = -1;
      if (p.group_list) {
        const int j = (int)atomicAdd(p.group_ctr, 1u);
        if (j < p.list_len) gg = p.group_list[j];
      } else {
        if (heavy) {
          const int j = (int)atomicAdd(p.ctr_heavy, 1u);
          if (j < p.n_heavy) gg = p.ngroups - 1 - j;
        }
        if (gg < 0) {
          const int j = (int)atomicAdd(p.group_ctr, 1u) + p.n_heavy;
          if (j < p.ngroups) gg = p.ngroups - 1 - j;
        }
      }
      s_g = gg;
      s_qn[0] = s_qn[1] = 0;
      for (int i = 0; i < 3; ++i) s_scan[i] = s_minfill[i] = INT_MAX;
    }
    __syncthreads();
    const int g = s_g;
    if (g < 0) break;
    const long long t_start = clock64();
    const unsigned long long st0 = c.steps, lv0 = c.levels, it0 = c.items, pr0 = c.pairs;
    long long t_trav = 0, t_ext = 0;
    const int s0g = p.row_begin + 32 * g;
    const int nsrc = min(32, p.row_end - s0g);
    const int Vb = min(n, s0g + nsrc);  // maxId only below the largest source
    const int tbw = (Vb + 31) >> 5;
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
          atomicOr(sl.state + 2 * w, bit);                            // RED
          atomicOr(sl.rsum + (w >> 10), 1u << ((w >> 5) & 31));       // RED
          atomicOr(sl.state + 2 * w + 1, bit);                        // RED
          atomicOr(sl.thr + (w >> 5), 1u << (w & 31));                // RED
          atomicOr(sl.tsum + (w >> 10), 1u << ((w >> 5) & 31));       // smem
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
      __syncthreads();  // all threads are done with the previous step's s_qn / T
      if (tid == 0) {
        s_scan[(step + 2) % 3] = INT_MAX;
        s_minfill[(step + 2) % 3] = INT_MAX;
      }
      // level 0: warp 0 expands T itself; warp 1 finds the next threshold
      // above T in parallel (new fills of this step go to s_minfill[nx3])
      if (warp == 0) {
        expand(p, sl, s0g, T, lane == 0 ? T : -1, sl.list1, &s_qn[1], &s_minfill[nx3], lane, c);
      } else if (warp == 1) {
        const int nt = scan_next(sl.thr, sl.tsum, tbw, T, lane);
        if (lane == 0) s_scan[nx3] = nt;
      }
      __syncthreads();
      c.levels += 1;
      // closure levels: every item has newMaxId T.  Levels only consume
      // returning atomics (reached, pend pushes); the REDs of this step
      // (fill pend / thr / is) are published before the next step's barrier.
      for (int lvl = 1;; ++lvl) {
        const int cur = lvl & 1, nxt = cur ^ 1;
        const int qn = s_qn[cur];
        if (qn == 0) {
          fence_gpu();
          break;
        }
        const uint32_t *cq = cur ? sl.list1 : sl.list0;
        uint32_t *nq = cur ? sl.list0 : sl.list1;
        __syncthreads();
        if (tid == 0) s_qn[cur] = 0;
        c.levels += 1;
        for (int b0 = warp * 32; b0 < qn; b0 += kThreads) {
          const int u = (b0 + lane < qn) ? (int)cq[b0 + lane] : -1;
          expand(p, sl, s0g, T, u, nq, &s_qn[nxt], &s_minfill[nx3], lane, c);
        }
        __syncthreads();
      }
    }

    __syncthreads();  // every thread's REDs were fenced at its last closure end
    t_trav = clock64();
    // ---- extraction of the group's rows (touched IS lines, ascending)
    // warp w owns isum words [w*q, (w+1)*q): its lines are ascending and all
    // of them precede warp w+1's, so per-warp counts give the write offsets
    const int q = (isw + kWarps - 1) / kWarps;
    const int wa = min(isw, warp * q), wb = min(isw, wa + q);
    const int s_lane = s0g + lane;
    uint32_t cl = 0, cu = 0;
    for (int i = wa; i < wb; ++i) {
      uint32_t x = __ldcg(sl.isum + i);
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1u;
        const int v0 = ((i << 5) + b) << 5;
        const uint32_t word = (v0 + lane < n) ? __ldcg(sl.is + v0 + lane) : 0u;
        const uint32_t y = transpose32(word, lane);
        uint32_t lm, um;
        split_masks(s_lane - v0, lm, um);
        cl += __popc(y & lm);
        cu += __popc(y & um);
      }
    }
    s_cnt[warp][0][lane] = cl;
    s_cnt[warp][1][lane] = cu;
    __syncthreads();
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
        const int r = s_lane - p.row_begin;
        p.row_off[r] = ok ? off : -1;
        p.row_nL[r] = (int)nl;
        p.row_nU[r] = (int)nu;
        if (ok) p.stage[off + nl] = s_lane;  // U(s,:) starts with the diagonal
      }
      if (lane == 0) {
        s_ok = ok;
        if (!ok) {
          p.failed[atomicAdd(p.nfailed, 1)] = g;
          atomicAdd(p.failed_need, (unsigned long long)tot);
        }
      }
    }
    __syncthreads();
    {
      const bool ok = s_ok;
      long long pl = 0, pu = 0;
      for (int w2 = 0; w2 < warp; ++w2) {
        pl += s_cnt[w2][0][lane];
        pu += s_cnt[w2][1][lane];
      }
      const bool valid = lane < nsrc;
      int32_t *Lp = p.stage + (valid && ok ? s_rowoff[lane] + pl : 0);
      int32_t *Up = p.stage + (valid && ok ? s_rowoff[lane] + s_nL[lane] + 1 + pu : 0);
      for (int i = wa; i < wb; ++i) {
        uint32_t x = __ldcg(sl.isum + i);
        if (!x) continue;
        if (lane == 0) sl.isum[i] = 0u;
        while (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1u;
          const int v0 = ((i << 5) + b) << 5;
          const uint32_t word = (v0 + lane < n) ? __ldcg(sl.is + v0 + lane) : 0u;
          if (v0 + lane < n) sl.is[v0 + lane] = 0u;
          const uint32_t y = transpose32(word, lane);
          if (ok) {
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
    t_ext = clock64();
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
          if (lane == 0) sl.thr[line] = 0u;
        }
      }
    }
    // the clears above are plain stores; the next group's atomics on the same
    // words are performed at L2, so make the stores globally visible first
    __threadfence();
    if (p.group_trace && lane == 0) {
      long long *t = p.group_trace + 8 * (size_t)g;
      // per-warp item / pair counts are summed over the warps' lane 0
      atomicAdd((unsigned long long *)&t[2], (unsigned long long)(c.items - it0));
      atomicAdd((unsigned long long *)&t[6], (unsigned long long)(c.pairs - pr0));
      if (warp == 0) {
        t[0] = (long long)(c.steps - st0);
        t[1] = (long long)(c.levels - lv0);
        t[3] = clock64() - t_start;
        t[4] = t_trav - t_start;
        t[5] = t_ext - t_trav;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    c.items += __shfl_xor_sync(kFull, c.items, d);
    c.edges += __shfl_xor_sync(kFull, c.edges, d);
    c.pairs += __shfl_xor_sync(kFull, c.pairs, d);
  }
  if (lane == 0) {
    atomicAdd(p.stats + 0, c.items);
    atomicAdd(p.stats + 1, c.edges);
    atomicAdd(p.stats + 4, c.pairs);
  }
  if (tid == 0) {
    atomicAdd(p.stats + 2, c.levels);
    atomicAdd(p.stats + 3, c.steps);
  }
  if (p.n < 0) p.stats[7] = c.sink;  // never true; keeps the returning atomics
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

size_t stream_ws_words(int64_t Vmax) {
  const size_t w = 2 * (size_t)Vmax + (size_t)((Vmax + 31) / 32) + (size_t)((Vmax + 1023) / 1024) +
                   2 * (size_t)Vmax;
  return (w + 7) / 8 * 8;
}

size_t stream_is_words(int64_t n) {
  const size_t w = (size_t)n + (size_t)((n + 1023) / 1024);
  return (w + 7) / 8 * 8;
}

size_t stream_smem_bytes(int64_t Vmax) {
  return (size_t)((((Vmax + 31) / 32) + 31) / 32) * 4;
}

template <int W>
int max_blocks_t(int device, int64_t Vmax) {
  int sms = 0, per = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  const size_t smem = stream_smem_bytes(Vmax);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(stream_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stream_kernel<W>, W * 32, smem) != cudaSuccess)
    return 0;
  return sms * per;
}

int stream_max_blocks(int device, int64_t Vmax, int heavy) {
  return heavy ? max_blocks_t<kHeavyWarps>(device, Vmax) : max_blocks_t<kLightWarps>(device, Vmax);
}

int stream_heavy_ratio() { return kHeavyWarps / kLightWarps; }

cudaError_t launch_stream(const StreamParams &p, int grid, int heavy, int slot_base, cudaStream_t st) {
  if (grid <= 0) return cudaSuccess;
  const size_t smem = stream_smem_bytes(p.Vmax);
  if (heavy) {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(stream_kernel<kHeavyWarps>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    stream_kernel<kHeavyWarps><<<grid, kHeavyWarps * 32, smem, st>>>(p, slot_base, 1);
  } else {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(stream_kernel<kLightWarps>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    stream_kernel<kLightWarps><<<grid, kLightWarps * 32, smem, st>>>(p, slot_base, 0);
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

}  // namespace gsofa
