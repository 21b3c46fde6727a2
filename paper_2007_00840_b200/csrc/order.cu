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
// A+A^T, O(nnz alpha)"): Liu's algorithm with path compression.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "gsofa_internal.cuh"

namespace gsofa {

// Elimination tree of A + A^T (parent[v] = -1 for roots) from the CSR of A.
// Row u's lower entries of A and of A^T (column u of A) are the edges
// (x, u), x < u, of the symmetrised graph; each links the root of x's
// current tree under u (Liu's algorithm; `anc` compresses paths).
void etree_sym(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent,
               int64_t *last_row_subtree) {
  const int64_t nnz = rowptr[n];
  // lower entries of column u of A, i.e. rows x < u with A(x, u) != 0
  std::vector<int64_t> cp(n + 1, 0);
  for (int64_t e = 0; e < nnz; ++e) cp[colidx[e] + 1] += 1;
  for (int64_t i = 0; i < n; ++i) cp[i + 1] += cp[i];
  std::vector<int32_t> cr((size_t)std::max<int64_t>(nnz, 1));
  {
    std::vector<int64_t> at(cp.begin(), cp.end() - 1);
    for (int64_t x = 0; x < n; ++x)
      for (int64_t e = rowptr[x]; e < rowptr[x + 1]; ++e) cr[at[colidx[e]]++] = (int32_t)x;
  }
  std::vector<int32_t> anc((size_t)n);
  for (int64_t u = 0; u < n; ++u) {
    parent[u] = -1;
    anc[u] = -1;
    for (int pass = 0; pass < 2; ++pass) {
      const int64_t *P = pass ? cp.data() : rowptr;
      const int32_t *I = pass ? cr.data() : colidx;
      for (int64_t e = P[u]; e < P[u + 1]; ++e) {
        int32_t k = I[e];
        if (k >= u) {
          if (pass) break;  // column entries ascend: the rest is >= u
          continue;
        }
        while (k != -1 && k != (int32_t)u) {
          const int32_t nx = anc[k];
          anc[k] = (int32_t)u;
          if (nx == -1) parent[k] = (int32_t)u;
          k = nx;
        }
      }
    }
  }
  if (last_row_subtree && n > 0) {
    // |struct(L(n-1,:))| of A + A^T: the row subtree of the last row, i.e.
    // every vertex on a tree path from one of its lower neighbours up to it
    // (anc is reused as the visited mark)
    const int64_t s = n - 1;
    int64_t cnt = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int64_t *P = pass ? cp.data() : rowptr;
      const int32_t *I = pass ? cr.data() : colidx;
      for (int64_t e = P[s]; e < P[s + 1]; ++e)
        for (int32_t k = I[e]; k != -1 && k < s && anc[k] != -2; k = parent[k]) {
          anc[k] = -2;
          ++cnt;
        }
    }
    *last_row_subtree = cnt;
  }
}

// Height order of the vertices (see the header comment), into caller
// arrays: hgt[n] (etree height), pos[n] (vertex -> position, sorted by
// (height, id)), posrec[4n] (per position: vertex, rowptr[v], rowptr[v+1],
// the end of v's height segment of positions).
OrderShape height_order(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *hgt,
                        int32_t *pos, int32_t *posrec) {
  std::vector<int32_t> parent((size_t)n);
  OrderShape shape;
  etree_sym(n, rowptr, colidx, parent.data(), &shape.last_row_chain);
  int32_t H = 0;
  for (int64_t v = 0; v < n; ++v) hgt[v] = 0;
  for (int64_t v = 0; v < n; ++v) {  // parents are larger: one ascending pass
    if (parent[v] >= 0) hgt[parent[v]] = std::max(hgt[parent[v]], hgt[v] + 1);
    H = std::max(H, hgt[v]);
  }
  std::vector<int64_t> seg((size_t)H + 2, 0);
  for (int64_t v = 0; v < n; ++v) seg[hgt[v] + 1] += 1;
  for (int32_t k = 0; k <= H; ++k) seg[k + 1] += seg[k];
  std::vector<int64_t> at(seg.begin(), seg.end() - 1);
  for (int64_t v = 0; v < n; ++v) {
    const int64_t q = at[hgt[v]]++;
    pos[v] = (int32_t)q;
    posrec[4 * q + 0] = (int32_t)v;
    posrec[4 * q + 1] = (int32_t)rowptr[v];
    posrec[4 * q + 2] = (int32_t)rowptr[v + 1];
    posrec[4 * q + 3] = (int32_t)seg[hgt[v] + 1];
  }
  shape.height = H;
  return shape;
}

}  // namespace gsofa
