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
// The solo kernel runs this order in POSITION space: vertices sorted by
// (height, id), each height's segment starting at a multiple of 32 (a bitmap
// word never mixes two heights), and the graph relabelled to positions.  All
// tests of the traversal become position comparisons against segment
// bounds, with no per-edge lookups (threshold.cu, solo_expand<true>):
//   * a neighbour of a vertex of subtree(s) is in subtree(s) (height below
//     s's: position < seg[h(s)]), s itself, or an ancestor of s (an entry of
//     U, position >= seg[h(s)+1]) -- so "w < s" is "pos(w) < seg[h(s)]";
//   * in the round of height h a newly reached vertex is a fill iff
//     pos(w) >= seg[h+1], a closure member iff pos(w) < seg[h].
// Rows are still written in vertex ids (the structure bitmap stays in id
// space; vert[] maps a position back when a bit is set).
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
void etree_sym(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent) {
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
}

// Height order of the vertices (see the header comment).  Outputs:
//   pos[n]        vertex -> position (sorted by (height, id))
//   vert[npos]    position -> vertex (-1 in padding)
//   wkey[npos/32] bitmap word -> height of its positions
//   seg[H+2]      height h occupies positions [seg[h], seg[h+1]) (padding at the end)
// Returns npos (a multiple of 32).
int64_t height_order(int64_t n, const int64_t *rowptr, const int32_t *colidx,
                     std::vector<int32_t> &pos, std::vector<int32_t> &vert,
                     std::vector<int32_t> &wkey, std::vector<int32_t> &seg) {
  std::vector<int32_t> parent((size_t)n), h((size_t)n, 0);
  etree_sym(n, rowptr, colidx, parent.data());
  int32_t H = 0;
  for (int64_t v = 0; v < n; ++v) {  // parents are larger: one ascending pass
    if (parent[v] >= 0) h[parent[v]] = std::max(h[parent[v]], h[v] + 1);
    H = std::max(H, h[v]);
  }
  std::vector<int64_t> cnt((size_t)H + 1, 0);
  for (int64_t v = 0; v < n; ++v) cnt[h[v]] += 1;
  seg.assign((size_t)H + 2, 0);
  int64_t acc = 0;
  for (int32_t k = 0; k <= H; ++k) {
    seg[k] = (int32_t)acc;
    acc += (cnt[k] + 31) / 32 * 32;  // each height's segment starts a bitmap word
  }
  seg[H + 1] = (int32_t)acc;
  const int64_t npos = std::max<int64_t>(acc, 32);
  vert.assign((size_t)npos, -1);
  wkey.assign((size_t)(npos / 32), 0);
  pos.resize((size_t)n);
  std::vector<int64_t> at(seg.begin(), seg.end() - 1);
  for (int64_t v = 0; v < n; ++v) {
    const int64_t p = at[h[v]]++;
    vert[p] = (int32_t)v;
    wkey[p >> 5] = h[v];
    pos[v] = (int32_t)p;
  }
  return npos;
}

namespace {
__global__ void relabel_degree_kernel(const int32_t *rowptr, const int32_t *pos, int64_t n,
                                      int32_t *degP) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) degP[pos[v]] = rowptr[v + 1] - rowptr[v];
}

// warp per row: row pos(v) of the relabelled graph = positions of v's neighbours
__global__ void relabel_scatter_kernel(const int32_t *rowptr, const int32_t *colidx,
                                       const int32_t *pos, int64_t n, const int32_t *rowptrP,
                                       int32_t *colidxP) {
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= n) return;
  const int a = rowptr[v], b = rowptr[v + 1];
  const int o = rowptrP[pos[v]];
  for (int e = a + lane; e < b; e += 32) colidxP[o + (e - a)] = __ldg(pos + colidx[e]);
}
}  // namespace

cudaError_t launch_relabel(const int32_t *rowptr, const int32_t *colidx, const int32_t *pos,
                           int64_t n, int64_t npos, int32_t *rowptrP, int32_t *colidxP,
                           void *tmp, size_t tmp_bytes, cudaStream_t st) {
  // degrees by position (padding rows empty) -> row pointers -> columns
  cudaError_t e = cudaMemsetAsync(rowptrP, 0, (size_t)(npos + 1) * sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  int32_t *deg = (int32_t *)tmp;
  const size_t deg_bytes = ((size_t)npos * 4 + 255) / 256 * 256;
  if (tmp_bytes < deg_bytes + scan_tmp_bytes(npos)) return cudaErrorInvalidValue;
  e = cudaMemsetAsync(deg, 0, (size_t)npos * 4, st);
  if (e != cudaSuccess) return e;
  relabel_degree_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rowptr, pos, n, deg);
  e = scan_exclusive_i32(deg, rowptrP, npos, rowptrP + npos, (char *)tmp + deg_bytes,
                         tmp_bytes - deg_bytes, st);
  if (e != cudaSuccess) return e;
  relabel_scatter_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(rowptr, colidx, pos, n,
                                                                        rowptrP, colidxP);
  return cudaGetLastError();
}

size_t relabel_tmp_bytes(int64_t npos) {
  return ((size_t)npos * 4 + 255) / 256 * 256 + scan_tmp_bytes(npos);
}

}  // namespace gsofa
