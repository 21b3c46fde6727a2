// order.cu -- the processing order of the threshold schedule (plan step A2).
//
// The relaxation is confluent: any order that expands a threshold only after
// every threshold whose closure can reach into its own has the same result
// (R16, R18).  Increasing vertex id (fill2) is one such
// order; it makes a source a chain of |L(s,:)| threshold steps.  The
// elimination tree of the symmetrised pattern A + A^T gives a much
// shorter one:
//   * the closure of threshold T (vertices < T reached from T through
//     unreached vertices < T) lies in the subtree of T: it is connected to T
//     in G(A+A^T) restricted to {0..T}, and that connected component is the
//     subtree of T;
//   * a vertex w > T adjacent to that subtree is an ancestor of T, so every
//     fill a closure finds is an ancestor of its threshold;
//   * hence thresholds that are not ancestor-related have disjoint closures,
//     and processing them by increasing etree HEIGHT (one round per height,
//     all thresholds of a round together) is exact, with no revisits: a
//     vertex newly reached in the round of height h is a fill iff its height
//     exceeds h, otherwise it joins the closure (it is a descendant).
// Rounds per source drop from |L(s,:)| to at most the tree height (C4's
// hub rows: 577k -> 4.2k; C5's top separator rows: ~1.5x).
//
// The solo kernel keeps the graph and its reached / structure bitmaps in
// vertex ids (the nested-dissection order's locality) and only its threshold
// bitmap in POSITIONS: vertices sorted by (height, id), so a forward scan
// meets thresholds by increasing height.  A step takes every threshold of one
// height in its window; with tmin / tmax their smallest / largest id, a newly
// reached w is a fill if w > tmax (a descendant of a threshold is smaller than
// it), a closure member if w < tmin (an ancestor is larger), and otherwise by
// height(w) > h -- one lookup for those in-between edges only.
//
// Host code ("int32 parent[n] ... from the etree of
// A+A^T, O(nnz alpha)"): Liu's algorithm with path compression, run on
// several host threads.  The tree is on the solo kernel's critical path
// (C4: ~190 ms single-threaded, of a 420 ms call), so the pass is split:
//   * transpose of the upper part (rows x < u with A(x,u) != 0, by u) with
//     atomic counters -- the order inside a column does not matter to Liu;
//   * lo(u) = the smallest neighbour of u in A + A^T (u if none below), and
//     P(a) = the first u >= a with lo(u) < a: the range [a, P(a)) has no
//     edge to [0, a), so Liu over it needs no state below a (an ND subtree
//     and the subtrees/separators that follow it on the same side);
//   * phase 1: T chunks [a_j, a_j+1) with a_j chosen where P reaches far;
//     thread j runs Liu over its independent prefix [a_j, p_j),
//     p_j = min(P(a_j), a_j+1) -- no vertex of another prefix is touched;
//   * phase 2: one thread runs Liu over the rest ([p_j, a_j+1) for every
//     j) in increasing order.  A vertex u there sees, below u, exactly the
//     state sequential Liu has at time u: prefixes below u are complete and
//     prefixes above u only linked vertices above u among themselves.
// Heights and the (height, id) positions follow the same split.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "gsofa_internal.cuh"

namespace gsofa {

struct OrderScratch {
  std::vector<int32_t> cp, cr, anc, parent, lo, P, nxt, hist;
  std::vector<int64_t> at;
};

OrderScratch *order_scratch_new() { return new OrderScratch(); }
void order_scratch_free(OrderScratch *s) { delete s; }
const int32_t *order_scratch_parent(const OrderScratch *s) { return s->parent.data(); }

namespace {

// host threads of the pass: GSOFA_HOST_THREADS if set (also for small n:
// tests), else the hardware threads for n >= 64k
int host_threads(int64_t n) {
  if (const char *e = std::getenv("GSOFA_HOST_THREADS"))
    return (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)atoi(e), 32, std::max<int64_t>(n / 4, 1)}));
  if (n < (1 << 16)) return 1;
  return std::max(1, std::min((int)std::thread::hardware_concurrency(), 32));
}

template <class F>
void par(int T, F &&f) {
  if (T <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve((size_t)T - 1);
  for (int j = 1; j < T; ++j) th.emplace_back(f, j);
  f(0);
  for (auto &t : th) t.join();
}

template <class V>
void fit(V &v, size_t n) {
  if (v.size() < n) v.resize(n);
}

// one Liu step: link the roots of u's lower neighbours (row u of A and
// column u of A, i.e. bucket u of the upper transpose) under u
inline void liu_step(int32_t u, const int64_t *rowptr, const int32_t *colidx, const int32_t *cp,
                     const int32_t *cr, int32_t *anc, int32_t *parent) {
  parent[u] = -1;
  anc[u] = -1;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t e0 = pass ? cp[u] : rowptr[u], e1 = pass ? cp[u + 1] : rowptr[u + 1];
    const int32_t *I = pass ? cr : colidx;
    for (int64_t e = e0; e < e1; ++e) {
      int32_t k = I[e];
      if (k >= u) {
        if (pass) continue;
        break;  // row entries ascend: the rest is >= u
      }
      while (k != -1 && k != u) {
        const int32_t nx = anc[k];
        anc[k] = u;
        if (nx == -1) parent[k] = u;
        k = nx;
      }
    }
  }
}

}  // namespace

// Elimination tree of A + A^T (parent[v] = -1 for roots) from the CSR of A
// (columns ascending within a row, as validated); see the header comment.
// Also fills the split (a[j], p[j]) used, for the height pass.
static double ord_now() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void etree_par(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent,
                      int64_t *last_row_subtree, OrderScratch &S, int T, std::vector<int64_t> &a,
                      std::vector<int64_t> &pe) {
  fit(S.cp, (size_t)n + 1);
  fit(S.anc, (size_t)n);
  fit(S.lo, (size_t)n);
  int32_t *cp = S.cp.data();
  int32_t *anc = S.anc.data(), *lo = S.lo.data();
  const double t0 = ord_now();
  // upper transpose: count, scan, scatter (atomic cursors)
  std::memset(cp, 0, ((size_t)n + 1) * sizeof(int32_t));
  par(T, [&](int j) {
    const int64_t r0 = n * j / T, r1 = n * (j + 1) / T;
    for (int64_t x = r0; x < r1; ++x)
      for (int64_t e = rowptr[x + 1] - 1; e >= rowptr[x]; --e) {
        const int32_t u = colidx[e];
        if (u <= x) break;  // ascending: the rest is <= x
        __atomic_fetch_add(cp + u + 1, 1, __ATOMIC_RELAXED);
      }
  });
  for (int64_t i = 0; i < n; ++i) cp[i + 1] += cp[i];
  fit(S.cr, (size_t)std::max<int32_t>(cp[n], 1));
  fit(S.at, (size_t)n);
  int32_t *cr = S.cr.data();
  int64_t *at = S.at.data();
  for (int64_t i = 0; i < n; ++i) at[i] = cp[i];
  par(T, [&](int j) {
    const int64_t r0 = n * j / T, r1 = n * (j + 1) / T;
    for (int64_t x = r0; x < r1; ++x)
      for (int64_t e = rowptr[x + 1] - 1; e >= rowptr[x]; --e) {
        const int32_t u = colidx[e];
        if (u <= x) break;
        cr[__atomic_fetch_add(at + u, (int64_t)1, __ATOMIC_RELAXED)] = (int32_t)x;
      }
  });
  const double t1 = ord_now();
  // chunk starts: a[0] = 0 and, for T > 1, the start in each window that
  // reaches furthest without an edge below it
  a.assign((size_t)T + 1, n);
  pe.assign((size_t)T, n);
  a[0] = 0;
  if (T > 1) {
    par(T, [&](int j) {
      const int64_t r0 = n * j / T, r1 = n * (j + 1) / T;
      for (int64_t u = r0; u < r1; ++u) {
        int32_t m = (int32_t)u;
        if (rowptr[u + 1] > rowptr[u]) m = std::min(m, colidx[rowptr[u]]);
        for (int32_t e = cp[u]; e < cp[u + 1]; ++e) m = std::min(m, cr[e]);
        lo[u] = m;
      }
    });
    // P(a) = min{u >= a : lo(u) < a}, needed only inside the window
    // [t_j - n/2T, t_j + n/2T) around each target t_j = j n / T and only up
    // to the cap a + n/T: per window (in parallel), u increasing from the
    // window start claims the still unclaimed a of the window in
    // (lo(u), u]; nxt skips claimed ones (path halving)
    fit(S.P, (size_t)n);
    fit(S.nxt, (size_t)n + T);
    int32_t *P = S.P.data(), *nx = S.nxt.data();
    const int64_t half = std::max<int64_t>(1, n / (2 * T)), cap = std::max<int64_t>(1, n / T);
    par(T - 1, [&](int jj) {
      const int j = jj + 1;
      const int64_t t = n * j / T;
      const int64_t w0 = std::max<int64_t>(1, t - half), w1 = std::min(n, t + half);
      if (w0 >= w1) return;
      int32_t *q = nx + w0 + jj;  // this window's skip links: q[x - w0], x in [w0, w1]
      for (int64_t x = w0; x <= w1; ++x) q[x - w0] = (int32_t)x;
      for (int64_t x = w0; x < w1; ++x) P[x] = (int32_t)n;
      auto find = [&](int32_t x) {
        while (q[x - w0] != x) {
          q[x - w0] = q[q[x - w0] - w0];
          x = q[x - w0];
        }
        return x;
      };
      // (past the next chunk's furthest possible start: P beyond it does not matter)
      const int64_t u1 = std::min(n, n * (j + 1) / T + half + 1);
      for (int64_t u = w0; u < u1; ++u) {
        if (lo[u] >= u) continue;
        const int64_t lo_a = std::max<int64_t>(lo[u] + 1, w0);
        if (lo_a >= w1) continue;
        for (int32_t x = find((int32_t)lo_a); x <= u && x < w1; x = find(x)) {
          P[x] = (int32_t)u;
          q[x - w0] = x + 1;
        }
      }
    });
    for (int j = 1; j < T; ++j) {
      const int64_t t = n * j / T;
      const int64_t w0 = std::max(a[j - 1] + 1, std::max<int64_t>(1, t - half)), w1 = std::min(n, t + half);
      int64_t best = std::max(a[j - 1] + 1, std::min(t, n - 1)), gain = -1;
      for (int64_t c = w0; c < w1; ++c) {
        const int64_t g = std::min<int64_t>(P[c], c + cap) - c;
        if (g > gain) {
          gain = g;
          best = c;
        }
      }
      a[j] = std::min<int64_t>(best, n);
    }
    // P is known inside the windows (a_j, j >= 1, lies in one) up to the
    // cap; a[0] = 0 has no vertex below it
    for (int j = 0; j < T; ++j) {
      int64_t r = n;
      if (j > 0) {
        const int64_t t = n * j / T;
        const bool in_w = a[j] >= std::max<int64_t>(1, t - half) && a[j] < std::min(n, t + half);
        r = in_w ? (int64_t)P[a[j]] : a[j];  // (outside: no independent prefix)
      }
      pe[j] = std::max(a[j], std::min(r, a[j + 1]));
    }
  }
  // phase 1: independent prefixes in parallel; phase 2: the rest in order
  if (std::getenv("GSOFA_ORDER_DEBUG")) {
    int64_t p1 = 0;
    for (int j = 0; j < T; ++j) p1 += pe[j] - a[j];
    std::fprintf(stderr, "[order] T=%d phase-1 vertices %lld of %lld  transpose %.1f ms split %.1f ms\n", T,
                 (long long)p1, (long long)n, t1 - t0, ord_now() - t1);
  }
  const double t2 = ord_now();
  par(T, [&](int j) {
    for (int64_t u = a[j]; u < pe[j]; ++u) liu_step((int32_t)u, rowptr, colidx, cp, cr, anc, parent);
  });
  for (int j = 0; j < T; ++j)
    for (int64_t u = pe[j]; u < a[j + 1]; ++u) liu_step((int32_t)u, rowptr, colidx, cp, cr, anc, parent);
  if (std::getenv("GSOFA_ORDER_DEBUG")) std::fprintf(stderr, "[order] liu %.1f ms\n", ord_now() - t2);
  if (last_row_subtree && n > 0) {
    // |struct(L(n-1,:))| of A + A^T: the row subtree of the last row, i.e.
    // every vertex on a tree path from one of its lower neighbours up to it
    // (anc is reused as the visited mark)
    const int64_t s = n - 1;
    int64_t cnt = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int64_t e0 = pass ? cp[s] : rowptr[s], e1 = pass ? cp[s + 1] : rowptr[s + 1];
      const int32_t *I = pass ? cr : colidx;
      for (int64_t e = e0; e < e1; ++e)
        for (int32_t k = I[e]; k != -1 && k < s && anc[k] != -2; k = parent[k]) {
          anc[k] = -2;
          ++cnt;
        }
    }
    *last_row_subtree = cnt;
  }
}

void etree_sym(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent,
               int64_t *last_row_subtree) {
  OrderScratch S;
  std::vector<int64_t> a, pe;
  etree_par(n, rowptr, colidx, parent, last_row_subtree, S, host_threads(n), a, pe);
}

// Height order of the vertices (see the header comment), into caller
// arrays: hgt[n] (etree height), pos[n] (vertex -> position, sorted by
// (height, id)), posrec[4n] (per position: vertex, rowptr[v], rowptr[v+1],
// the end of v's height segment of positions).
OrderShape height_order(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *hgt,
                        int32_t *pos, int32_t *posrec, OrderScratch *scratch) {
  OrderScratch local;
  OrderScratch &S = scratch ? *scratch : local;
  const int T = host_threads(n);
  fit(S.parent, (size_t)n);
  int32_t *parent = S.parent.data();
  OrderShape shape;
  std::vector<int64_t> a, pe;
  etree_par(n, rowptr, colidx, parent, &shape.last_row_chain, S, T, a, pe);
  // heights (parents are larger): inside each prefix in parallel (a prefix
  // vertex's parent is in its prefix or in the phase-2 rest), then the
  // prefix roots' parents and the rest in increasing order
  par(T, [&](int j) {
    for (int64_t v = a[j]; v < pe[j]; ++v) hgt[v] = 0;
    for (int64_t v = pe[j]; v < a[j + 1]; ++v) hgt[v] = 0;
    for (int64_t v = a[j]; v < pe[j]; ++v) {
      const int32_t q = parent[v];
      if (q >= 0 && q < pe[j]) hgt[q] = std::max(hgt[q], hgt[v] + 1);
    }
  });
  for (int j = 0; j < T; ++j)
    for (int64_t v = a[j]; v < pe[j]; ++v) {
      const int32_t q = parent[v];
      if (q >= pe[j]) hgt[q] = std::max(hgt[q], hgt[v] + 1);
    }
  for (int j = 0; j < T; ++j)
    for (int64_t v = pe[j]; v < a[j + 1]; ++v) {
      const int32_t q = parent[v];
      if (q >= 0) hgt[q] = std::max(hgt[q], hgt[v] + 1);
    }
  int32_t H = 0;
  for (int64_t v = 0; v < n; ++v) H = std::max(H, hgt[v]);
  // positions: stable counting sort by height over T vertex ranges
  // (per-range histograms; one range when the tree is tall)
  const int Tp = (int64_t)(H + 1) * T <= n / 4 ? T : 1;
  const size_t hb = (size_t)H + 2;
  fit(S.hist, hb * (size_t)Tp);
  int32_t *hist = S.hist.data();
  par(Tp, [&](int j) {
    int32_t *h = hist + hb * (size_t)j;
    std::fill(h, h + hb, 0);
    for (int64_t v = n * j / Tp, v1 = n * (j + 1) / Tp; v < v1; ++v) h[hgt[v]] += 1;
  });
  std::vector<int64_t> seg(hb, 0);  // seg[k + 1]: end of height k's segment
  {
    int64_t run = 0;
    for (int32_t k = 0; k <= H; ++k) {
      for (int j = 0; j < Tp; ++j) {
        const int32_t c = hist[hb * (size_t)j + k];
        hist[hb * (size_t)j + k] = (int32_t)run;  // this range's first position of height k
        run += c;
      }
      seg[(size_t)k + 1] = run;
    }
  }
  par(Tp, [&](int j) {
    int32_t *h = hist + hb * (size_t)j;
    for (int64_t v = n * j / Tp, v1 = n * (j + 1) / Tp; v < v1; ++v) {
      const int64_t q = h[hgt[v]]++;
      pos[v] = (int32_t)q;
      posrec[4 * q + 0] = (int32_t)v;
      posrec[4 * q + 1] = (int32_t)rowptr[v];
      posrec[4 * q + 2] = (int32_t)rowptr[v + 1];
      posrec[4 * q + 3] = (int32_t)seg[(size_t)hgt[v] + 1];
    }
  });
  shape.height = H;
  return shape;
}

}  // namespace gsofa
