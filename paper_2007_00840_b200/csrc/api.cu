// api.cu -- the C ABI of include/gsofa.h: context/arena management, input
// upload + validation, batch planning under a memory budget, the per-batch
// pipeline (seed -> persistent traversal -> extraction), supernode detection
// and output assembly.  Host code only orchestrates: every step that touches
// the matrix or the result runs in the kernels of traverse.cu, extract.cu and
// supernode.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/gsofa.h"
#include "gsofa_internal.cuh"

namespace gsofa {
int extract_sub_columns();
}

namespace {

thread_local char g_detail[512] = "";

void set_detail(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_detail, sizeof g_detail, fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what) {
  set_detail("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  if (e == cudaErrorMemoryAllocation) return GSOFA_ENOMEM;
  return GSOFA_ECUDA;
}

#define CK(call)                                        \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) {                            \
      rc = cuda_fail(e_, #call);                        \
      goto fail;                                        \
    }                                                   \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

// Pinned host block for host-side results, shared by a context (its pool)
// and by the results that point into it; freed when the last owner lets go.
struct HostBlock {
  char *p = nullptr;
  size_t cap = 0;
  int refs = 0;
  bool in_use = false;  // handed to a live result
};

void host_block_release(HostBlock *b) {
  if (b && --b->refs == 0) {
    if (b->p) cudaFreeHost(b->p);
    delete b;
  }
}

// a result and its bookkeeping; the public struct is the first member
struct ResultImpl {
  gsofa_result r;
  HostBlock *block;  // pinned host storage of the arrays (host results)
  int32_t chunk_size;  // of the call (supernode stitch); sn_start has room for rows+1
  int32_t cap_only;    // supernode rule of the call (gsofa_opts.sn_cap_only)
};

// ------------------------------------------------------------------ context
struct Plan {
  int64_t Cmax, Gmax;
  int gbits;
  size_t work_bytes, is_words, cnt_words;
  int64_t nsub;
  size_t total;
  // FIFO: the queues hold 1 / 2^qfl of their worst case in HBM; the rest
  // goes to pinned host memory (external frontier management)
  int qfl = 0;
  // streaming (threshold) schedule
  int64_t slots = 0, heavy = 0, light = 0, Vmax = 0;
  size_t ws_words = 0, slot_is_words = 0, hws_words = 0;
};

struct gsofa_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // heavy-group kernel runs here, concurrently
  int64_t budget = 0;        // requested budget (0 = auto)
  // arena (one cudaMalloc, carved in fixed regions)
  char *arena = nullptr;
  size_t arena_bytes = 0;
  // arena layout key
  int64_t key_n = -1;
  int64_t Cmax = 0, Gmax = 0;
  int gbits = 0;
  size_t work_bytes = 0, is_words = 0;
  int qfl = 0;               // FIFO queue fraction in HBM: 1 / 2^qfl (Plan::qfl)
  int work_state = 0;        // WorkState
  uint64_t layout_sig = 0;   // streaming slot layout of the last call (Vmax, ws_words)
  int stream_blocks = 0;     // resident CTAs of the streaming kernel
  int sms = 0, clock_khz = 0;  // device attributes, queried once (clock rate can be slow to query)
  unsigned int *bw_dev = nullptr;  // bandwidth scratch (GSOFA_SCHEDULE_AUTO)
  // last plan and its key: repeated calls on the same problem skip the
  // free-memory query and the occupancy queries, and keep the arena layout
  Plan plan_cache;
  int64_t plan_key[7] = {-1, -1, -1, -1, -1, -1, -1};
  int32_t *stage = nullptr;  // staging area for streamed rows (grow-only)
  size_t stage_cap = 0;
  uint32_t *work = nullptr, *is = nullptr;
  uint32_t *cntL = nullptr, *cntU = nullptr;
  int64_t *rowL = nullptr, *rowU = nullptr, *totals = nullptr;
  uint32_t *qcount = nullptr;
  unsigned long long *stats = nullptr;
  int *err = nullptr;
  int64_t nsub = 0;
  uint32_t floor = 0xFFFFFFFFu;  // lowest maxId value ever written (epoch floor)
  int max_blocks[2] = {0, 0};
  // input staging (grow-only)
  int64_t *in_rowptr = nullptr;
  int32_t *in_colidx = nullptr, *rowptr32 = nullptr;
  size_t in_rowptr_cap = 0, in_colidx_cap = 0, rowptr32_cap = 0;
  int64_t *h_small = nullptr;  // pinned host scratch
  // height order (order.cu): per-position records | heights | positions,
  // one grow-only buffer
  int32_t *ord_buf = nullptr;
  size_t ord_cap = 0;
  // ... their host side: the tree pass's scratch, and one grow-only pinned
  // block for the order arrays and (device inputs) the host copy of the CSR
  gsofa::OrderScratch *ord_scratch = nullptr;
  char *ord_pin = nullptr;
  size_t ord_pin_cap = 0;
  // ELL copy of the adjacency (solo kernel, id order, rows <= 8 entries)
  int32_t *ell = nullptr;
  size_t ell_cap = 0;
  HostBlock *hpool = nullptr;  // pinned storage reused by host-side results
  // external frontier (FIFO queue overflow) in mapped pinned host memory,
  // grow-only; spill_dev is its device address
  uint32_t *spill = nullptr, *spill_dev = nullptr;
  size_t spill_cap = 0;  // words
};

namespace {

void release_arena(gsofa_context *c) {
  if (c->arena) cudaFree(c->arena);
  c->arena = nullptr;
  c->arena_bytes = 0;
  c->key_n = -1;
}



size_t small_bytes(int64_t Cmax) {
  return (size_t)Cmax * 2 * sizeof(int64_t) + 64 + 64 + 64 + 256;
}

// Traversal working set of a batch of C sources whose labels cover Vb
// vertices (Table tab:complexity, after bubble removal):
//   FIFO:      maxId labels C*Vb*4 B + 2 frontier masks (G*Vb words each) +
//              2 queues (G*Vb words each, of which 1 / 2^qfl in HBM)
//   threshold: per 32-source group reached/pend/list0/list1 (Vb words each)
//              + a threshold bitmap (Vb/32 words)
size_t work_need(int schedule, int64_t C, int64_t Vb, int qfl = 0) {
  const int64_t G = C / 32;
  if (schedule == GSOFA_SCHEDULE_FIFO)
    return (size_t)C * Vb * 4 + (size_t)G * Vb * 8 + (((size_t)G * Vb) >> qfl) * 8;
  return (size_t)G * gsofa::stream_ws_words(Vb, 0) * 4;
}

// FIFO keeps its label region apart from masks/queues so that every label
// cell only ever holds epoch-encoded values (P:573 requires stale values to
// decode as "uninitialised").  Per (group, vertex) cell: 128 B of labels,
// 8 B of masks, 8 / 2^qfl B of queues in HBM.
size_t fifo_label_bytes(size_t work, int qfl) {
  return (size_t)((double)work * 128.0 / (136.0 + 8.0 / (double)(1 << qfl))) / 512 * 512;
}
// mask capacity (words per mask array) and HBM queue capacity (items per queue)
void fifo_caps(size_t work, int qfl, size_t &Qm, size_t &Qq) {
  const size_t lab = fifo_label_bytes(work, qfl);
  Qm = (size_t)((double)(work - lab) / (8.0 + 8.0 / (double)(1 << qfl)));
  Qq = Qm >> qfl;
}

bool make_plan(int schedule, int64_t n, int64_t rows, int64_t vb_max, int64_t cmax_req,
               int64_t budget, Plan &p) {
  const int64_t sub = gsofa::extract_sub_columns();
  // external frontier management first, then fewer concurrent sources
  // (P:780-784): when the budget cannot hold the whole batch with its full
  // queues, only 1/8 of each queue stays in HBM (the paper measured peak
  // frontier usage up to 25% and far less on average, Table tab:FQ_usage)
  int qfl = 0;
  if (schedule == GSOFA_SCHEDULE_FIFO) {
    const int64_t C0 = std::max<int64_t>(32, round_up(std::min<int64_t>(cmax_req, round_up(rows, 32)), 32));
    const int64_t G0 = C0 / 32;
    const size_t full = work_need(schedule, C0, vb_max) + (size_t)G0 * n * 4 +
                        2 * (size_t)G0 * ceil_div(n, sub) * 32 * 4 + small_bytes(C0) + 8192 + 4096;
    if ((int64_t)full > budget) qfl = 3;
    if (const char *e = std::getenv("GSOFA_FRONTIER_FRAC_LOG")) qfl = std::max(0, std::min(20, atoi(e)));
  }
  int64_t Cmax = std::min<int64_t>(cmax_req, round_up(rows, 32));
  Cmax = std::max<int64_t>(32, round_up(Cmax, 32));
  for (; Cmax >= 32; Cmax = (Cmax / 2 / 32) * 32) {
    const int64_t G = Cmax / 32;
    int gb = 0;
    while ((int64_t(1) << gb) < G) ++gb;
    if (schedule == GSOFA_SCHEDULE_FIFO && ((uint64_t)n << gb) > 0xFFFFFFFFull) continue;
    const int64_t nsub = ceil_div(n, sub);
    const size_t is_words = (size_t)G * n;
    const size_t cnt_words = (size_t)G * nsub * 32;
    const size_t fixed = is_words * 4 + 2 * cnt_words * 4 + small_bytes(Cmax) + 8192;
    const size_t need_max = work_need(schedule, Cmax, vb_max, qfl) + 4096;
    const size_t need_min = work_need(schedule, 32, vb_max, qfl) + 4096;
    if ((int64_t)(fixed + need_min) > budget) continue;
    size_t work = std::min<size_t>(need_max, (size_t)budget - fixed);
    work = (work + 4095) / 4096 * 4096;
    p.Cmax = Cmax;
    p.Gmax = G;
    p.gbits = gb;
    p.qfl = qfl;
    p.work_bytes = work;
    p.is_words = is_words;
    p.cnt_words = cnt_words;
    p.nsub = nsub;
    p.total = work + is_words * 4 + 2 * cnt_words * 4 + small_bytes(Cmax) + 4096 + 12 * 256;
    return true;
  }
  return false;
}

// Streaming schedule: one workspace slot per resident CTA, each slot holding
// one 32-source group at a time: reached/pend/lists over Vmax vertices (bubble
// removal: no maxId state above the largest source) plus an n-word
// structure bitmap.  The number of slots is what the budget allows
// ("reduce the number of concurrent sources"), at most the resident
// CTA count and the number of groups.
// Streaming schedule: one workspace slot per resident CTA.  Lockstep slots
// (4-warp CTAs, one 32-source group at a time, shared frontier items) and
// solo slots (32-warp CTAs, one warp per source, for the heavy groups the
// lockstep kernel hands over).  No maxId state above the largest source
// (bubble removal).  Slot counts follow the residency of both kernels
// sharing the SMs and the memory budget ("reduce the number of concurrent
// sources").
// npos > 0: height order (threshold bitmaps over npos positions, order.cu)
bool make_plan_stream(int64_t n, int64_t rows, int64_t Vmax, int64_t budget, int device, Plan &p,
                      int64_t npos, bool wide, bool lock_h = false, int lw = 16) {
  // the lockstep kernel runs id order (its slots do not depend on npos), or
  // height order alone (lock_h: threshold bits over npos positions, no solo)
  const int64_t lnpos = lock_h ? npos : 0;
  if (gsofa::stream_smem_bytes(Vmax, lnpos) > 200 * 1024) return false;
  const size_t ws = gsofa::stream_ws_words(Vmax, lnpos), isw = gsofa::stream_is_words(n);
  const size_t hws = gsofa::solo_ws_words(Vmax, n, npos);
  const int64_t spc = gsofa::solo_warps_per_cta();
  const size_t per_light = (ws + isw) * 4, per_heavy = hws * 4 * (size_t)spc;  // per solo CTA
  const size_t fixed = small_bytes(32) + 8192;
  if (budget <= (int64_t)(fixed + per_light)) return false;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t ngroups = ceil_div(rows, 32);
  const int64_t wpc = gsofa::stream_warps_per_cta();  // lockstep slots (warps) per CTA
  const int64_t res_light = gsofa::stream_max_blocks(device, Vmax, 0, npos, wide, lock_h, lw) * wpc;
  const int64_t res_heavy = gsofa::stream_max_blocks(device, Vmax, 1, npos, wide);
  if (res_light < 1) return false;
  // solo CTAs: one per SM is resident next to the lockstep CTAs from the
  // start; more become resident as lockstep CTAs finish (the grid is
  // deliberately larger than the first wave), up to the kernel's residency
  // heavy sources are spread warp-major over at least one CTA per SM: a
  // chain is paced by its SM's atomic issue rate, not by latency alone
  int64_t heavy = std::min<int64_t>(std::max<int64_t>(res_heavy, (int64_t)sms),
                                    std::max<int64_t>((int64_t)sms, ceil_div(rows, spc)));
  (void)res_heavy;
  if (const char *e = std::getenv("GSOFA_SOLO_CTAS")) heavy = std::min<int64_t>(heavy, atoll(e));
  heavy = std::max<int64_t>(0, std::min<int64_t>(heavy, (int64_t)(((size_t)budget - fixed) / 2 / per_heavy)));
  if (lock_h) heavy = 0;  // every group runs lockstep in height order
  int64_t light = heavy > 0 ? (int64_t)sms * gsofa::stream_light_per_sm_with_solo(device, Vmax, npos, wide) * wpc
                            : res_light;
  if (res_heavy < 1) heavy = 0;
  light = std::min<int64_t>(light, res_light);
  if (const char *e = std::getenv("GSOFA_LIGHT_CTAS")) light = std::min<int64_t>(light, atoll(e));
  light = std::min<int64_t>(light, (int64_t)(((size_t)budget - fixed - heavy * per_heavy) / per_light));
  light = std::max<int64_t>(1, std::min<int64_t>(light, ngroups));
  if ((size_t)light * per_light + (size_t)heavy * per_heavy + fixed > (size_t)budget) return false;
  p.Cmax = 32;
  p.Gmax = 1;
  p.gbits = 0;
  p.slots = light + heavy;
  p.heavy = heavy;
  p.light = light;
  p.Vmax = Vmax;
  p.ws_words = ws;
  p.hws_words = hws;
  p.slot_is_words = isw;
  p.work_bytes = (size_t)light * ws * 4 + (size_t)heavy * per_heavy;
  p.is_words = (size_t)light * isw;  // solo slots keep their bitmap in hws
  p.cnt_words = 0;
  p.nsub = 0;
  p.total = p.work_bytes + p.is_words * 4 + small_bytes(32) + 4096 + 12 * 256;
  return true;
}

// largest multiple of 32 <= cap whose working set fits `work` bytes
int64_t fit_batch(int schedule, int64_t n, int64_t s0, int64_t cap, size_t work, int qfl) {
  int64_t lo = 0, hi = cap / 32;  // in groups
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    const int64_t C = mid * 32;
    const int64_t vb = std::min<int64_t>(n, s0 + C);
    size_t need = work_need(schedule, C, vb, qfl);
    if (schedule == GSOFA_SCHEDULE_FIFO) {
      // labels and masks must fit; the queues overflow into host memory
      size_t Qm, Qq;
      fifo_caps(work, qfl, Qm, Qq);
      need = ((size_t)C * vb * 4 > fifo_label_bytes(work, qfl) || (size_t)(C / 32) * vb > Qm) ? work + 1 : 0;
    }
    if (need <= work) lo = mid;
    else hi = mid - 1;
  }
  return lo * 32;
}

enum WorkState { kWorkZero = 0, kWorkFifo = 1, kWorkDirty = 2 };

int ensure_arena(gsofa_context *c, int64_t n, const Plan &p, cudaStream_t st) {
  int rc = GSOFA_OK;
  if (c->arena && c->key_n == n && c->Cmax == p.Cmax && c->work_bytes == p.work_bytes &&
      c->is_words == p.is_words && c->qfl == p.qfl)
    return rc;
  release_arena(c);
  {
    cudaError_t e = cudaMalloc((void **)&c->arena, p.total);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c->arena = nullptr;
      set_detail("arena cudaMalloc(%zu bytes) failed: %s", p.total, cudaGetErrorString(e));
      return GSOFA_ENOMEM;
    }
  }
  c->arena_bytes = p.total;
  {
    char *q = c->arena;
    auto carve = [&](size_t bytes) {
      char *r = q;
      q += (bytes + 255) / 256 * 256;
      return r;
    };
    c->work = (uint32_t *)carve(p.work_bytes);
    c->is = (uint32_t *)carve(p.is_words * 4);
    c->cntL = (uint32_t *)carve(p.cnt_words * 4);
    c->cntU = (uint32_t *)carve(p.cnt_words * 4);
    c->rowL = (int64_t *)carve(p.Cmax * 8);
    c->rowU = (int64_t *)carve(p.Cmax * 8);
    c->totals = (int64_t *)carve(64);
    c->qcount = (uint32_t *)carve(64);
    c->stats = (unsigned long long *)carve(128);
    c->err = (int *)carve(64);
  }
  c->key_n = n;
  c->Cmax = p.Cmax;
  c->Gmax = p.Gmax;
  c->gbits = p.gbits;
  c->work_bytes = p.work_bytes;
  c->is_words = p.is_words;
  c->qfl = p.qfl;
  c->nsub = p.nsub;
  c->layout_sig = 0;
  CK(cudaMemsetAsync(c->work, 0, p.work_bytes, st));
  CK(cudaMemsetAsync(c->is, 0, p.is_words * 4, st));
  c->work_state = kWorkZero;
  c->floor = 0xFFFFFFFFu;
  return rc;
fail:
  release_arena(c);
  return rc;
}

// Bring the work region into the state a schedule expects.
int prepare_work(gsofa_context *c, int schedule, cudaStream_t st) {
  int rc = GSOFA_OK;
  if (schedule == GSOFA_SCHEDULE_FIFO) {
    if (c->work_state != kWorkFifo) {
      const size_t lab = fifo_label_bytes(c->work_bytes, c->qfl);
      CK(cudaMemsetAsync(c->work, 0xFF, lab, st));                    // labels: above every epoch
      CK(cudaMemsetAsync((char *)c->work + lab, 0, c->work_bytes - lab, st));  // masks, queues
      c->floor = 0xFFFFFFFFu;
      c->work_state = kWorkFifo;
    }
  } else if (c->work_state != kWorkZero) {
    CK(cudaMemsetAsync(c->work, 0, c->work_bytes, st));
    c->work_state = kWorkZero;
  }
  return rc;
fail:
  c->work_state = kWorkDirty;
  return rc;
}

template <typename T>
int grow_device(T **buf, size_t *cap, size_t need, cudaStream_t st) {
  if (*cap >= need) return GSOFA_OK;
  size_t nc = std::max(need, *cap * 2);
  T *nb = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&nb, nc * sizeof(T), st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_detail("output cudaMallocAsync(%zu bytes) failed: %s", nc * sizeof(T), cudaGetErrorString(e));
    return GSOFA_ENOMEM;
  }
  if (*buf) {
    if (*cap) cudaMemcpyAsync(nb, *buf, *cap * sizeof(T), cudaMemcpyDeviceToDevice, st);
    cudaFreeAsync(*buf, st);
  }
  *buf = nb;
  *cap = nc;
  return GSOFA_OK;
}

// gsofa_partition_rows cost exponent: cost(s) = work(s)^alpha.  With many
// ranks, the ranks holding the top separator are bound by their longest
// chains rather than their total work, so heavy rows are weighted slightly
// below their work.  With few ranks the top rank is throughput-bound and
// alpha = 1 balances best.  Measured with scripts/scaling_emulation.py: C5 at
// 8 ranks max rank 685 -> 633 ms (alpha 0.94), but at 2 ranks 1.82x -> 1.61x.
double part_alpha(int nparts) {
  if (nparts <= 4) return 1.0;
  if (nparts >= 8) return 0.94;
  return 1.0 - 0.015 * (nparts - 4);
}

int64_t auto_budget(int device) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  (void)device;
  return (int64_t)(fr * 0.5);
}

}  // namespace

extern "C" {

int gsofa_version(void) { return GSOFA_VERSION; }

const char *gsofa_strerror(int code) {
  switch (code) {
    case GSOFA_OK: return "ok";
    case GSOFA_EINVAL: return "invalid argument";
    case GSOFA_EBADCSR: return "malformed CSR input";
    case GSOFA_ENOMEM: return "out of memory";
    case GSOFA_EINFEASIBLE: return "memory budget below one 32-source group";
    case GSOFA_ECUDA: return "CUDA error";
    case GSOFA_EINTERNAL: return "internal invariant violated";
    default: return "unknown error";
  }
}

const char *gsofa_last_error_detail(void) { return g_detail; }

int gsofa_default_opts(gsofa_opts *o) {
  if (!o) return GSOFA_EINVAL;
  std::memset(o, 0, sizeof *o);
  o->chunk_size = 128;
  o->max_concurrent = 0;
  o->mem_budget_bytes = 0;
  o->fill_first = 0;
  o->schedule = GSOFA_SCHEDULE_AUTO;
  o->row_begin = 0;
  o->row_end = -1;
  o->device = 0;
  o->outputs_on_device = 1;
  o->stream = nullptr;
  o->checked = 0;
  return GSOFA_OK;
}

int gsofa_context_create(int32_t device, int64_t mem_budget_bytes, gsofa_context **out) {
  if (!out) return GSOFA_EINVAL;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_detail("no CUDA device available (%s)", cudaGetErrorString(e));
    return GSOFA_ECUDA;
  }
  if (device < 0 || device >= ndev || mem_budget_bytes < 0) {
    set_detail("bad device %d or budget", device);
    return GSOFA_EINVAL;
  }
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  gsofa_context *c = new (std::nothrow) gsofa_context();
  if (!c) return GSOFA_ENOMEM;
  c->device = device;
  c->budget = mem_budget_bytes;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaStreamCreate");
  }
  e = cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaStreamDestroy(c->stream);
    delete c;
    return cuda_fail(e, "cudaStreamCreate");
  }
  e = cudaMallocHost((void **)&c->h_small, 64 * sizeof(int64_t));
  if (e != cudaSuccess) {
    cudaStreamDestroy(c->stream);
    delete c;
    return cuda_fail(e, "cudaMallocHost");
  }
  // keep stream-ordered output allocations cached between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  c->stream_blocks = gsofa::stream_max_blocks(device, 1 << 20, 0, 0, false);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->clock_khz, cudaDevAttrClockRate, device);
  c->max_blocks[0] = gsofa::traverse_max_blocks(device, 0);
  c->max_blocks[1] = gsofa::traverse_max_blocks(device, 1);
  if (c->max_blocks[0] <= 0 || c->max_blocks[1] <= 0 || c->stream_blocks <= 0) {
    cudaFreeHost(c->h_small);
    cudaStreamDestroy(c->stream);
    delete c;
    set_detail("traversal kernel cannot be made resident (occupancy 0)");
    return GSOFA_ECUDA;
  }
  *out = c;
  return GSOFA_OK;
}

void gsofa_context_destroy(gsofa_context *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  release_arena(c);
  if (c->in_rowptr) cudaFree(c->in_rowptr);
  if (c->in_colidx) cudaFree(c->in_colidx);
  if (c->rowptr32) cudaFree(c->rowptr32);
  if (c->bw_dev) cudaFree(c->bw_dev);
  if (c->stage) cudaFree(c->stage);
  if (c->ord_buf) cudaFree(c->ord_buf);
  if (c->ord_pin) cudaFreeHost(c->ord_pin);
  gsofa::order_scratch_free(c->ord_scratch);
  if (c->ell) cudaFree(c->ell);
  if (c->h_small) cudaFreeHost(c->h_small);
  if (c->spill) cudaFreeHost(c->spill);
  host_block_release(c->hpool);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  delete c;
}

int gsofa_result_l_csc(const gsofa_result *r, int32_t on_device, int64_t **col_ptr,
                       int32_t **row_idx) {
  if (!r || !col_ptr || !row_idx) {
    set_detail("NULL argument to gsofa_result_l_csc");
    return GSOFA_EINVAL;
  }
  *col_ptr = nullptr;
  *row_idx = nullptr;
  if (r->interleave.nparts > 1) {
    set_detail("gsofa_result_l_csc: an interleaved part's rows are not a range");
    return GSOFA_EINVAL;
  }
  cudaError_t e = cudaSetDevice(r->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const int64_t n = r->n, rows = r->row_end - r->row_begin, nnz = r->nnz_L;
  int64_t *d_rp = nullptr, *d_cp = nullptr;
  int32_t *d_ci = nullptr, *d_ri = nullptr;
  bool own_in = false;
  int rc = GSOFA_OK;
  cudaStream_t st = nullptr;
  auto dev_alloc = [&](void **p, size_t b) { return cudaMallocAsync(p, std::max<size_t>(b, 4), st); };
  if (r->on_device) {
    d_rp = r->L_rowptr;
    d_ci = r->L_colidx;
  } else {
    own_in = true;
    if ((e = dev_alloc((void **)&d_rp, (size_t)(rows + 1) * 8)) != cudaSuccess ||
        (e = dev_alloc((void **)&d_ci, (size_t)nnz * 4)) != cudaSuccess)
      goto cuda_err;
    if ((e = cudaMemcpyAsync(d_rp, r->L_rowptr, (size_t)(rows + 1) * 8, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess ||
        (nnz && (e = cudaMemcpyAsync(d_ci, r->L_colidx, (size_t)nnz * 4, cudaMemcpyHostToDevice, st)) !=
                    cudaSuccess))
      goto cuda_err;
  }
  if ((e = dev_alloc((void **)&d_cp, (size_t)(n + 1) * 8)) != cudaSuccess ||
      (e = dev_alloc((void **)&d_ri, (size_t)nnz * 4)) != cudaSuccess)
    goto cuda_err;
  if ((e = gsofa::l_rows_to_csc(d_rp, d_ci, rows, r->row_begin, n, nnz, d_cp, d_ri, st)) != cudaSuccess)
    goto cuda_err;
  if (on_device) {
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) goto cuda_err;
    *col_ptr = d_cp;
    *row_idx = d_ri;
    d_cp = nullptr;
    d_ri = nullptr;
  } else {
    int64_t *h_cp = (int64_t *)std::malloc((size_t)(n + 1) * 8);
    int32_t *h_ri = (int32_t *)std::malloc(std::max<size_t>((size_t)nnz * 4, 4));
    if (!h_cp || !h_ri) {
      std::free(h_cp);
      std::free(h_ri);
      set_detail("host allocation for L in CSC failed");
      rc = GSOFA_ENOMEM;
      goto done;
    }
    e = cudaMemcpyAsync(h_cp, d_cp, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(h_ri, d_ri, (size_t)nnz * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      std::free(h_cp);
      std::free(h_ri);
      goto cuda_err;
    }
    *col_ptr = h_cp;
    *row_idx = h_ri;
  }
  goto done;
cuda_err:
  rc = cuda_fail(e, "gsofa_result_l_csc");
done:
  if (own_in) {
    if (d_rp) cudaFreeAsync(d_rp, st);
    if (d_ci) cudaFreeAsync(d_ci, st);
  }
  if (d_cp) cudaFreeAsync(d_cp, st);
  if (d_ri) cudaFreeAsync(d_ri, st);
  cudaStreamSynchronize(st);
  return rc;
}

int gsofa_permute(int64_t n, const int64_t *rowptr, const int32_t *colidx, const int32_t *perm,
                  int64_t *out_rowptr, int32_t *out_colidx) {
  if (n <= 0 || n >= (int64_t(1) << 31) || !rowptr || !colidx || !perm || !out_rowptr || !out_colidx) {
    set_detail("bad arguments to gsofa_permute");
    return GSOFA_EINVAL;
  }
  cudaStream_t st = nullptr;
  const bool dev = is_device_ptr(rowptr);
  if (dev != is_device_ptr(colidx) || dev != is_device_ptr(perm) || dev != is_device_ptr(out_rowptr) ||
      dev != is_device_ptr(out_colidx)) {
    set_detail("gsofa_permute: pointers must all be host or all be device");
    return GSOFA_EINVAL;
  }
  int64_t nnz = 0;
  cudaError_t e = cudaSuccess;
  if (dev) {
    if ((e = cudaMemcpy(&nnz, rowptr + n, 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
      return cuda_fail(e, "gsofa_permute");
  } else {
    nnz = rowptr[n];
  }
  if (nnz < 0 || nnz >= (int64_t(1) << 31)) {
    set_detail("gsofa_permute: nnz=%lld out of range", (long long)nnz);
    return GSOFA_EBADCSR;
  }
  int64_t *d_rp = nullptr, *d_nrp = nullptr;
  int32_t *d_ci = nullptr, *d_perm = nullptr, *d_nci = nullptr, *d_iperm = nullptr, *d_deg = nullptr;
  int *d_bad = nullptr;
  void *tmp = nullptr;
  int rc = GSOFA_OK, bad = 0;
  const size_t tmpb = gsofa::scan_tmp_bytes(n);
  auto A = [&](void **p, size_t b) { return cudaMallocAsync(p, std::max<size_t>(b, 8), st); };
  if ((e = A((void **)&d_iperm, (size_t)n * 4)) != cudaSuccess || (e = A((void **)&d_deg, (size_t)n * 4)) != cudaSuccess ||
      (e = A((void **)&d_bad, 64)) != cudaSuccess || (e = A(&tmp, tmpb)) != cudaSuccess)
    goto cuda_err;
  if (dev) {
    d_rp = const_cast<int64_t *>(rowptr);
    d_ci = const_cast<int32_t *>(colidx);
    d_perm = const_cast<int32_t *>(perm);
    d_nrp = out_rowptr;
    d_nci = out_colidx;
  } else {
    if ((e = A((void **)&d_rp, (size_t)(n + 1) * 8)) != cudaSuccess || (e = A((void **)&d_ci, (size_t)nnz * 4)) != cudaSuccess ||
        (e = A((void **)&d_perm, (size_t)n * 4)) != cudaSuccess || (e = A((void **)&d_nrp, (size_t)(n + 1) * 8)) != cudaSuccess ||
        (e = A((void **)&d_nci, (size_t)nnz * 4)) != cudaSuccess)
      goto cuda_err;
    if ((e = cudaMemcpyAsync(d_rp, rowptr, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (nnz && (e = cudaMemcpyAsync(d_ci, colidx, (size_t)nnz * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) ||
        (e = cudaMemcpyAsync(d_perm, perm, (size_t)n * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      goto cuda_err;
  }
  if ((e = cudaMemsetAsync(d_bad, 0, 64, st)) != cudaSuccess) goto cuda_err;
  if ((e = gsofa::launch_iperm(d_perm, n, d_iperm, d_bad, st)) != cudaSuccess) goto cuda_err;
  if ((e = cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost)) != cudaSuccess) goto cuda_err;
  if (bad) {
    set_detail("gsofa_permute: perm is not a permutation of [0, n)%s%s", (bad & 1) ? " (entry out of range)" : "",
               (bad & 2) ? " (duplicate entry)" : "");
    rc = GSOFA_EINVAL;
    goto done;
  }
  if ((e = gsofa::launch_perm_degrees(d_rp, d_perm, n, d_deg, st)) != cudaSuccess ||
      (e = gsofa::scan_exclusive_i32_i64(d_deg, d_nrp, n, d_nrp + n, tmp, tmpb, st)) != cudaSuccess ||
      (e = gsofa::permute_pattern(d_rp, d_ci, d_perm, d_iperm, n, nnz, d_nrp, d_nci, st)) != cudaSuccess)
    goto cuda_err;
  if (!dev) {
    if ((e = cudaMemcpyAsync(out_rowptr, d_nrp, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (nnz && (e = cudaMemcpyAsync(out_colidx, d_nci, (size_t)nnz * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess))
      goto cuda_err;
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) goto cuda_err;
  goto done;
cuda_err:
  rc = cuda_fail(e, "gsofa_permute");
done:
  if (!dev) {
    for (void *p : {(void *)d_rp, (void *)d_ci, (void *)d_perm, (void *)d_nrp, (void *)d_nci})
      if (p) cudaFreeAsync(p, st);
  }
  for (void *p : {(void *)d_iperm, (void *)d_deg, (void *)d_bad, tmp})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  return rc;
}

int gsofa_result_supno(const gsofa_result *r, int32_t on_device, int32_t **supno) {
  if (!r || !supno) {
    set_detail("NULL argument to gsofa_result_supno");
    return GSOFA_EINVAL;
  }
  *supno = nullptr;
  if (r->interleave.nparts > 1) {
    set_detail("gsofa_result_supno: an interleaved part's rows are not a range");
    return GSOFA_EINVAL;
  }
  cudaError_t e = cudaSetDevice(r->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const int64_t rows = r->row_end - r->row_begin;
  int32_t *d_sn = nullptr, *d_out = nullptr;
  cudaStream_t st = nullptr;
  if (r->on_device) {
    d_sn = r->sn_start;
  } else {
    if ((e = cudaMallocAsync((void **)&d_sn, (size_t)(r->nsuper + 1) * 4, st)) != cudaSuccess)
      return cuda_fail(e, "cudaMallocAsync");
    if ((e = cudaMemcpyAsync(d_sn, r->sn_start, (size_t)(r->nsuper + 1) * 4, cudaMemcpyHostToDevice,
                             st)) != cudaSuccess) {
      cudaFreeAsync(d_sn, st);
      return cuda_fail(e, "cudaMemcpyAsync");
    }
  }
  if ((e = cudaMallocAsync((void **)&d_out, (size_t)std::max<int64_t>(rows, 1) * 4, st)) == cudaSuccess)
    e = gsofa::launch_supno(d_sn, r->nsuper, (int32_t)r->row_begin, d_out, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (!r->on_device) cudaFreeAsync(d_sn, st);
  if (e != cudaSuccess) {
    if (d_out) cudaFreeAsync(d_out, st);
    cudaStreamSynchronize(st);
    return cuda_fail(e, "supno");
  }
  if (on_device) {
    *supno = d_out;
    return GSOFA_OK;
  }
  int32_t *h = (int32_t *)std::malloc((size_t)std::max<int64_t>(rows, 1) * 4);
  if (!h) {
    cudaFreeAsync(d_out, st);
    cudaStreamSynchronize(st);
    set_detail("host allocation for supno failed");
    return GSOFA_ENOMEM;
  }
  e = cudaMemcpy(h, d_out, (size_t)rows * 4, cudaMemcpyDeviceToHost);
  cudaFreeAsync(d_out, st);
  cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    std::free(h);
    return cuda_fail(e, "cudaMemcpy");
  }
  *supno = h;
  return GSOFA_OK;
}

void gsofa_buffer_free(void *p, int32_t on_device) {
  if (!p) return;
  if (on_device) {
    cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
  } else {
    std::free(p);
  }
}

int gsofa_result_copy(const gsofa_result *r, int64_t *L_rowptr, int32_t *L_colidx,
                      int64_t *U_rowptr, int32_t *U_colidx, int32_t *sn_start) {
  if (!r) {
    set_detail("result is NULL");
    return GSOFA_EINVAL;
  }
  if (r->on_device) {
    cudaError_t e = cudaSetDevice(r->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  }
  const int64_t rows = r->rows;
  struct {
    void *dst;
    const void *src;
    size_t bytes;
  } cp[5] = {{L_rowptr, r->L_rowptr, (size_t)(rows + 1) * 8},
             {L_colidx, r->L_colidx, (size_t)r->nnz_L * 4},
             {U_rowptr, r->U_rowptr, (size_t)(rows + 1) * 8},
             {U_colidx, r->U_colidx, (size_t)r->nnz_U * 4},
             {sn_start, r->sn_start, (size_t)(r->nsuper + 1) * 4}};
  for (auto &c : cp) {
    if (!c.dst || !c.bytes) continue;
    if (r->on_device || is_device_ptr(c.dst)) {
      cudaError_t e = cudaMemcpy(c.dst, c.src, c.bytes, cudaMemcpyDefault);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(result)");
    } else {
      std::memcpy(c.dst, c.src, c.bytes);
    }
  }
  return GSOFA_OK;
}

namespace {
gsofa::RowMap result_map(const gsofa_result *r) {
  gsofa::RowMap m;
  m.rb = (int32_t)r->row_begin;
  m.re = (int32_t)r->row_end;
  if (r->interleave.nparts > 1) {
    m.N = r->interleave.nparts;
    m.q = r->interleave.part;
    m.U = r->interleave.unit_rows;
  }
  return m;
}
}  // namespace

int gsofa_result_rowinfo(const gsofa_result *r, int32_t *nnzU, uint32_t *lmask) {
  if (!r || !nnzU || !lmask || !r->on_device) {
    set_detail("gsofa_result_rowinfo: NULL argument or a host result");
    return GSOFA_EINVAL;
  }
  cudaError_t e = cudaSetDevice(r->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const int32_t chunk = reinterpret_cast<const ResultImpl *>(r)->chunk_size;
  e = gsofa::launch_rowinfo(r->L_rowptr, r->L_colidx, r->U_rowptr, result_map(r), (int32_t)r->rows,
                            chunk, nnzU, lmask, nullptr);
  if (e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
  return e == cudaSuccess ? GSOFA_OK : cuda_fail(e, "gsofa_result_rowinfo");
}

int gsofa_supernodes_gathered(gsofa_result *r, const int32_t *nnzU_all, const uint32_t *lmask_all,
                              int64_t stride) {
  if (!r || !nnzU_all || !lmask_all || !r->on_device || r->interleave.nparts <= 1 ||
      stride < r->rows) {
    set_detail("gsofa_supernodes_gathered: needs an interleaved device result and stride >= rows");
    return GSOFA_EINVAL;
  }
  cudaError_t e = cudaSetDevice(r->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const int32_t chunk = reinterpret_cast<const ResultImpl *>(r)->chunk_size;
  const int64_t rows = r->rows;
  const gsofa::RowMap m = result_map(r);
  cudaStream_t st = nullptr;
  const size_t tmpb = gsofa::scan_tmp_bytes(rows);
  char *scr = nullptr;
  if ((e = cudaMallocAsync((void **)&scr, (size_t)rows * 8 + 64 + tmpb, st)) != cudaSuccess)
    return cuda_fail(e, "cudaMallocAsync");
  int32_t *leader = (int32_t *)scr, *pos = leader + rows, *total = pos + rows;
  void *tmp = scr + (size_t)rows * 8 + 64;
  int32_t ns = 0;
  e = gsofa::launch_supernode_gathered(m, chunk, nnzU_all, lmask_all, stride, leader, st);
  if (e == cudaSuccess) e = gsofa::scan_exclusive_i32(leader, pos, rows, total, tmp, tmpb, st);
  if (e == cudaSuccess) e = gsofa::launch_supernode_scatter(leader, pos, m, (int32_t)rows, total, r->sn_start, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&ns, total, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(scr, st);
  if (e != cudaSuccess) return cuda_fail(e, "gsofa_supernodes_gathered");
  r->nsuper = ns;
  return GSOFA_OK;
}

void gsofa_result_free(gsofa_result *r) {
  if (!r) return;
  ResultImpl *impl = reinterpret_cast<ResultImpl *>(r);
  void *ptrs[5] = {r->L_rowptr, r->L_colidx, r->U_rowptr, r->U_colidx, r->sn_start};
  if (r->on_device) {
    // the arrays came from the device's stream-ordered pool (cudaMallocAsync):
    // hand them back to it (no cudaFree: that would unmap the pages and the
    // next call would pay for mapping them again)
    cudaSetDevice(r->device);
    for (void *p : ptrs)
      if (p) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
  } else if (impl->block) {
    impl->block->in_use = false;
    host_block_release(impl->block);
  } else {
    for (void *p : ptrs) std::free(p);
  }
  std::free(impl);
}

int gsofa_supernode_stitch(gsofa_result *r, const gsofa_tail *prev, gsofa_tail *out) {
  if (!r) {
    set_detail("result is NULL");
    return GSOFA_EINVAL;
  }
  ResultImpl *impl = reinterpret_cast<ResultImpl *>(r);
  const int64_t rb = r->row_begin, re = r->row_end, rows = re - rb;
  if (r->interleave.nparts > 1) {
    set_detail("gsofa_supernode_stitch: interleaved parts use gsofa_supernodes_gathered");
    return GSOFA_EINVAL;
  }
  const int32_t chunk = impl->chunk_size;
  if (prev && (prev->row != rb - 1 || prev->leader < 0 || prev->leader > prev->row || prev->nnzU < 1)) {
    set_detail("stitch tail {row %lld, nnzU %lld, leader %lld} does not precede row_begin %lld",
               (long long)prev->row, (long long)prev->nnzU, (long long)prev->leader, (long long)rb);
    return GSOFA_EINVAL;
  }
  cudaError_t e = cudaSetDevice(r->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const bool cap = impl->cap_only != 0;
  if (prev && (cap || rb % chunk != 0)) {
    // provisional head blocks: re-scan from the predecessor's tail -- over
    // [rb, next chunk start) under the forced-break rule, until the scan
    // meets a provisional leader under the cap-only rule
    const int64_t he = std::min<int64_t>(re, (rb / chunk + 1) * chunk);
    const int64_t cap_out = cap ? rows + 3 : chunk + 2;
    int32_t *d_out = nullptr;
    if ((e = cudaMalloc((void **)&d_out, (size_t)cap_out * 4)) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc(stitch)");
    int32_t hdr[3] = {0, 0, 0};
    if (cap) {
      e = gsofa::launch_supernode_stitch_cap(r->U_rowptr, r->L_rowptr, r->L_colidx, (int32_t)rb,
                                             (int32_t)re, chunk, prev->nnzU, (int32_t)prev->leader,
                                             r->sn_start, r->nsuper, d_out, nullptr);
      if (e == cudaSuccess) e = cudaMemcpy(hdr, d_out, 12, cudaMemcpyDeviceToHost);
    } else {
      e = gsofa::launch_supernode_stitch(r->U_rowptr, r->L_rowptr, r->L_colidx, (int32_t)rb,
                                         (int32_t)he, prev->nnzU, (int32_t)prev->leader, r->sn_start,
                                         r->nsuper, d_out, nullptr);
      if (e == cudaSuccess) e = cudaMemcpy(hdr, d_out, 8, cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess) {
      cudaFree(d_out);
      return cuda_fail(e, "supernode stitch");
    }
    const int64_t nc = hdr[0], oc = hdr[1], tail = r->nsuper + 1 - oc;  // tail incl. the sentinel
    const int32_t *d_new = d_out + (cap ? 3 : 2);                        // the new head leaders
    if (r->on_device) {
      if (nc != oc && tail > 0) {
        int32_t *tmp = nullptr;
        e = cudaMalloc((void **)&tmp, (size_t)tail * 4);
        if (e == cudaSuccess) e = cudaMemcpy(tmp, r->sn_start + oc, (size_t)tail * 4, cudaMemcpyDeviceToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(r->sn_start + nc, tmp, (size_t)tail * 4, cudaMemcpyDeviceToDevice);
        cudaFree(tmp);
      }
      if (e == cudaSuccess && nc)
        e = cudaMemcpy(r->sn_start, d_new, (size_t)nc * 4, cudaMemcpyDeviceToDevice);
    } else {
      std::memmove(r->sn_start + nc, r->sn_start + oc, (size_t)tail * 4);
      if (nc) e = cudaMemcpy(r->sn_start, d_new, (size_t)nc * 4, cudaMemcpyDeviceToHost);
    }
    cudaFree(d_out);
    if (e != cudaSuccess) return cuda_fail(e, "supernode stitch copy");
    r->nsuper += nc - oc;
  }
  if (out) {
    int64_t up[2] = {0, 0};
    int32_t lead = 0;
    e = cudaMemcpy(up, r->U_rowptr + rows - 1, 16, cudaMemcpyDefault);
    if (e == cudaSuccess && r->nsuper > 0)
      e = cudaMemcpy(&lead, r->sn_start + r->nsuper - 1, 4, cudaMemcpyDefault);
    if (e != cudaSuccess) return cuda_fail(e, "stitch tail");
    out->row = re - 1;
    out->nnzU = up[1] - up[0];
    // every row joined the predecessor's block: its leader carries on
    out->leader = r->nsuper > 0 ? lead : prev->leader;
  }
  return GSOFA_OK;
}

// A2 host pass (order.cu): the elimination tree of A + A^T, heights and
// (height, id) positions into the context's pinned block (posrec | hgt | pos,
// 6n int32), from host inputs or a host copy of device inputs (made on s).
static cudaError_t host_height_order(gsofa_context *c, int64_t n, int64_t nnz, bool in_dev,
                                     const int64_t *rowptr, const int32_t *colidx, cudaStream_t s,
                                     gsofa::OrderShape *shape) {
  const size_t ob = ((size_t)n * 6 * 4 + 15) & ~(size_t)15;
  const size_t need = ob + (in_dev ? ((size_t)n + 1) * 8 + (size_t)std::max<int64_t>(nnz, 1) * 4 : 0);
  cudaError_t e;
  if (c->ord_pin_cap < need) {
    if (c->ord_pin) cudaFreeHost(c->ord_pin);
    c->ord_pin = nullptr;
    c->ord_pin_cap = 0;
    if ((e = cudaMallocHost((void **)&c->ord_pin, need)) != cudaSuccess) return e;
    c->ord_pin_cap = need;
  }
  if (!c->ord_scratch) c->ord_scratch = gsofa::order_scratch_new();
  int32_t *ord_host = (int32_t *)c->ord_pin;
  const int64_t *rp_h = rowptr;
  const int32_t *ci_h = colidx;
  if (in_dev) {
    int64_t *hrp = (int64_t *)(c->ord_pin + ob);
    int32_t *hci = (int32_t *)(c->ord_pin + ob + ((size_t)n + 1) * 8);
    if ((e = cudaMemcpyAsync(hrp, rowptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if (nnz && (e = cudaMemcpyAsync(hci, colidx, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    rp_h = hrp;
    ci_h = hci;
  }
  auto now_ms = [] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t0 = now_ms();
  *shape = gsofa::height_order(n, rp_h, ci_h, ord_host + 4 * n, ord_host + 5 * n, ord_host, c->ord_scratch);
  if (std::getenv("GSOFA_TIMELINE")) std::fprintf(stderr, "[timeline] host height order %.3f ms\n", now_ms() - t0);
  return cudaSuccess;
}

int gsofa_symbolic(gsofa_context *ctx, int64_t n, const int64_t *rowptr, const int32_t *colidx,
                   const gsofa_opts *opts_in, gsofa_result **out) {
  if (!out) {
    set_detail("out is NULL");
    return GSOFA_EINVAL;
  }
  *out = nullptr;
  gsofa_opts o;
  if (opts_in) o = *opts_in;
  else gsofa_default_opts(&o);
  if (n <= 0 || n >= (int64_t(1) << 31) || !rowptr || !colidx) {
    set_detail("bad n=%lld or NULL input", (long long)n);
    return GSOFA_EINVAL;
  }
  if (o.row_end < 0) o.row_end = n;
  if (o.chunk_size < 1 || o.row_begin < 0 || o.row_end > n || o.row_begin >= o.row_end ||
      o.max_concurrent < 0 || o.max_concurrent % 32 != 0 ||
      o.mem_budget_bytes < 0 || o.schedule < 0 || o.schedule > GSOFA_SCHEDULE_HEIGHT ||
      o.sn_cap_only < 0 || o.sn_cap_only > 1) {
    set_detail("bad opts: chunk=%d rows=[%lld,%lld) C=%d budget=%lld", o.chunk_size,
               (long long)o.row_begin, (long long)o.row_end, o.max_concurrent,
               (long long)o.mem_budget_bytes);
    return GSOFA_EINVAL;
  }
  // row interleave (gsofa_interleave): the units of this part
  gsofa::RowMap rmap;
  rmap.rb = (int32_t)o.row_begin;
  rmap.re = (int32_t)o.row_end;
  const bool ilv = o.interleave.nparts > 1;
  if (ilv) {
    const gsofa_interleave &iv = o.interleave;
    if (iv.part < 0 || iv.part >= iv.nparts || iv.unit_rows < 32 || iv.unit_rows % 32 != 0 ||
        o.sn_cap_only || o.schedule == GSOFA_SCHEDULE_FIFO || o.row_begin % o.chunk_size != 0) {
      set_detail("bad interleave: parts=%d part=%d unit_rows=%d (multiple of 32; threshold "
                 "schedules, forced-break supernodes, row_begin a multiple of chunk_size)",
                 iv.nparts, iv.part, iv.unit_rows);
      return GSOFA_EINVAL;
    }
    rmap.N = iv.nparts;
    rmap.q = iv.part;
    rmap.U = iv.unit_rows;
    if (rmap.count() < 1) {
      set_detail("interleave part %d of %d holds no rows of [%lld, %lld)", iv.part, iv.nparts,
                 (long long)o.row_begin, (long long)o.row_end);
      return GSOFA_EINVAL;
    }
  }
  // finer than a chunk: supernodes wait for the parts' exchange
  const bool sn_deferred = ilv && o.interleave.unit_rows % o.chunk_size != 0;
  bool own_ctx = false;
  int rc = GSOFA_OK;
  if (!ctx) {
    rc = gsofa_context_create(o.device, o.mem_budget_bytes, &ctx);
    if (rc != GSOFA_OK) return rc;
    own_ctx = true;
  }
  gsofa_context *c = ctx;
  cudaStream_t st = o.stream ? (cudaStream_t)o.stream : c->stream;
  gsofa_result *res = nullptr;
  int64_t *Lrp = nullptr, *Urp = nullptr;
  int32_t *Lci = nullptr, *Uci = nullptr, *sn = nullptr;
  size_t Lcap = 0, Ucap = 0;
  int32_t *sn_scratch = nullptr;
  void *scan_tmp = nullptr;
  void *stream_scratch = nullptr;
  std::vector<cudaEvent_t> evs;
  std::vector<int> ev_line;  // source line of each event (GSOFA_TIMELINE dev dump)
  int64_t launches = 0;
  std::vector<double> ev_host;  // host clock at each event record (GSOFA_TIMELINE)
  auto ev_at = [&](int line) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    evs.push_back(e);
    ev_line.push_back(line);
    ev_host.push_back(std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now().time_since_epoch()).count());
    return (int)evs.size() - 1;
  };
#define ev() ev_at(__LINE__)
  const int64_t rb = o.row_begin, re = o.row_end, rows = rmap.count();
  int64_t nnz = 0;
  bool in_dev;
  const int64_t *d_rowptr64;
  const int32_t *d_colidx;
  int e_start, e_up, e_sn0, e_sn1, e_end;
  std::vector<std::pair<int, int>> e_trav, e_ext;
  int64_t baseL = 0, baseU = 0, nbatches = 0, maxC = 0;
  Plan plan;
  bool auto_fifo = false;
  unsigned int maxdeg = 0;  // largest row of A (validation pass)
  int64_t ord_npos = 0;  // > 0: height order possible (threshold bitmaps sized for n positions)
  bool auto_order = false;  // AUTO: pick the threshold order from the tree's shape
  bool auto_hubs = false;   // AUTO: the pattern has hub rows
  bool lock_h = false;      // height order in the lockstep kernel (no solo kernel)
  int lock_w = 16;          // ... its warps per CTA
  // solo kernel shape: the latency shape (4 pair batches in
  // flight, 32 warps/SM) when the call's sources fit one wave of its slots --
  // the chain-bound ranks of a multi-GPU split (C2's top ranks: 61 -> 57 ms;
  // two waves of long chains lose: C5's 4,922-row top range 645 -> 860 ms);
  // GSOFA_SOLO_WIDE=0/1 forces a shape (dev A/B)
  const bool solo_wide = std::getenv("GSOFA_SOLO_WIDE") ? atoi(std::getenv("GSOFA_SOLO_WIDE")) != 0
                                                        : rows <= 32 * (int64_t)std::max(c->sms, 1);

  CK(cudaSetDevice(c->device));
  e_start = ev();
  // ---------------------------------------------------- A1: residency
  in_dev = is_device_ptr(rowptr);
  if (in_dev != is_device_ptr(colidx) && n > 0) {
    // mixed is allowed only if colidx is empty-ish; require same kind
    set_detail("rowptr and colidx must both be host or both be device pointers");
    rc = GSOFA_EINVAL;
    goto fail;
  }
  if (in_dev) {
    CK(cudaMemcpyAsync(c->h_small, rowptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    nnz = c->h_small[0];
  } else {
    nnz = rowptr[n];
  }
  if (nnz < 0 || nnz >= (int64_t(1) << 31)) {
    set_detail("nnz=%lld out of range [0, 2^31)", (long long)nnz);
    rc = GSOFA_EBADCSR;
    goto fail;
  }
  if (in_dev) {
    d_rowptr64 = rowptr;
    d_colidx = colidx;
  } else {
    if ((rc = grow_device(&c->in_rowptr, &c->in_rowptr_cap, (size_t)n + 1, st)) != GSOFA_OK) goto fail;
    if ((rc = grow_device(&c->in_colidx, &c->in_colidx_cap, (size_t)std::max<int64_t>(nnz, 1), st)) != GSOFA_OK) goto fail;
    CK(cudaMemcpyAsync(c->in_rowptr, rowptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (nnz) CK(cudaMemcpyAsync(c->in_colidx, colidx, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    d_rowptr64 = c->in_rowptr;
    d_colidx = c->in_colidx;
  }
  e_up = ev();
  // ---------------------------------------------------- A1: validation
  // CSR checks (GSOFA_EBADCSR) and int32 row pointers, before anything else
  // reads the input; the same pass measures the bandwidth for AUTO
  if ((rc = grow_device(&c->rowptr32, &c->rowptr32_cap, (size_t)n + 1, st)) != GSOFA_OK) goto fail;
  if (!c->bw_dev) CK(cudaMalloc((void **)&c->bw_dev, 64));
  CK(cudaMemsetAsync(c->bw_dev, 0, 12, st));  // [0] bandwidth, [1] error flags, [2] max degree
  CK(gsofa::launch_validate(d_rowptr64, d_colidx, n, nnz, c->rowptr32, (int *)(c->bw_dev + 1),
                            c->bw_dev, st));
  ++launches;
  CK(cudaMemcpyAsync(c->h_small, c->bw_dev, 12, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (const int f = ((int *)c->h_small)[1]) {
    set_detail("CSR check failed:%s%s%s", (f & 1) ? " bad rowptr" : "",
               (f & 2) ? " column out of range" : "", (f & 4) ? " columns not strictly increasing" : "");
    rc = GSOFA_EBADCSR;
    goto fail;
  }
  maxdeg = ((unsigned int *)c->h_small)[2];  // largest row of A
  if (o.schedule == GSOFA_SCHEDULE_AUTO) {
    // banded and dense -> the paper's FIFO order (few rounds, no revisits);
    // otherwise threshold order (DESIGN.md §8 "Schedule").  FIFO also needs
    // one batch of maxId labels (sources x vertices x 4 B) to fit the budget
    // the plan will use: FIFO in many small batches loses its edge.
    const unsigned int bw = ((unsigned int *)c->h_small)[0];
    auto_fifo = (int64_t)bw * 8 <= n && nnz >= 8 * n && !ilv;
    if (auto_fifo) {
      int64_t budget = o.mem_budget_bytes ? o.mem_budget_bytes : c->budget;
      if (!budget) budget = auto_budget(c->device) + (int64_t)c->arena_bytes;
      const double labels = (double)std::min<int64_t>(rows, 65536) * (double)n * 4.0;
      auto_fifo = labels <= (double)budget;
    }
    o.schedule = auto_fifo ? GSOFA_SCHEDULE_FIFO : GSOFA_SCHEDULE_THRESHOLD;
    // threshold family: the solo kernel's order (id or etree height) is
    // chosen once the tree is known (below).  The tree is a host pass
    // (O(nnz alpha) plus a copy of A) on the solo kernel's critical path, so
    // it is computed only for patterns with hub rows (largest row > 32x the
    // mean), where height order was measured to win (C4: 1.19 s -> 0.45 s);
    // on grids it would only delay the solo kernel (C5: ~5%)
    const int64_t mean = std::max<int64_t>(1, nnz / std::max<int64_t>(1, n));
    auto_hubs = (int64_t)maxdeg > 32 * mean;
    // large patterns (n >= 2^20) factorized whole take the height order in
    // the lockstep kernel too: the sources of a group share their closures
    // (C5: 3,386 -> 2,389 ms; C2 at n = 262k stays faster in id order, 125 vs
    // 165 ms).  Row ranges of a multi-GPU split keep id order: their
    // chain-bound top ranks were slower in height order (C5 8-way: 1,102 vs
    // 631 ms on one of them)
    auto_order = !auto_fifo && (auto_hubs || (n >= (int64_t(1) << 20) && rows == n));
  }
  // ---------------------------------------------------- A2: height order
  // positions are a permutation of [0, n): the plan does not depend on the
  // tree, which is computed on the host while the lockstep kernel runs
  if (o.schedule == GSOFA_SCHEDULE_HEIGHT || auto_order) {
    ord_npos = n;
    if ((rc = grow_device(&c->ord_buf, &c->ord_cap, (size_t)n * 6, st)) != GSOFA_OK) goto fail;
    if (!std::getenv("GSOFA_HEIGHT_SOLO")) {
      // height order in the LOCKSTEP kernel (default): a group's steps are the
      // union of its sources' heights (<= the tree height), and the 32 hub /
      // separator sources of a group share their closures (C4's top groups:
      // 10-15x fewer pairs than 32 solo sources, union steps ~ one source's),
      // so every group runs lockstep and no solo kernel is launched.  The tree
      // is needed before the launch: computed here, on the host.
      // GSOFA_HEIGHT_SOLO=1 keeps the solo kernel's height order (dev A/B).
      gsofa::OrderShape shape;
      CK(host_height_order(c, n, nnz, in_dev, rowptr, colidx, st, &shape));
      bool use_h = true;
      if (auto_order) {
        // AUTO: large patterns always; hub patterns when the last row's
        // id-order chain (about |L(n-1,:)| threshold steps) is far longer
        // than the tree is high (C4's hub rows: 577k vs 4.2k)
        use_h = !auto_hubs || shape.last_row_chain > 4 * shape.height;
        o.schedule = use_h ? GSOFA_SCHEDULE_HEIGHT : GSOFA_SCHEDULE_THRESHOLD;
        auto_order = false;
      }
      if (use_h) {
        lock_h = true;
        const int64_t mean = std::max<int64_t>(1, nnz / std::max<int64_t>(1, n));
        lock_w = gsofa::lock_warps(ceil_div(rows, 32), c->sms, (int64_t)maxdeg > 32 * mean);
        CK(cudaMemcpyAsync(c->ord_buf, c->ord_pin, (size_t)n * 6 * 4, cudaMemcpyHostToDevice, st));
      } else {
        ord_npos = 0;
      }
    }
  }
  // ---------------------------------------------------- plan + arena
  {
    const int64_t cmax_req =
        o.max_concurrent ? o.max_concurrent : 65536;  // FIFO: one batch when it fits (C3 -6% vs 16k)
    const int64_t budget_req = o.mem_budget_bytes ? o.mem_budget_bytes : c->budget;
    int64_t key[7] = {o.schedule, n, rb, re ^ ((int64_t)rmap.q << 32) ^ ((int64_t)rmap.N << 40),
                      budget_req, cmax_req, ord_npos * 256 + lock_w * 4 + solo_wide * 2 + lock_h};
    bool ok = true;
    if (std::equal(key, key + 7, c->plan_key)) {
      plan = c->plan_cache;
    } else {
      int64_t budget = budget_req;
      if (!budget) budget = auto_budget(c->device) + (int64_t)c->arena_bytes;
      const int64_t vb_max = std::min<int64_t>(n, re + 32);
      ok = o.schedule == GSOFA_SCHEDULE_FIFO
               ? make_plan(o.schedule, n, rows, vb_max, cmax_req, budget, plan)
               : make_plan_stream(n, rows, std::min<int64_t>(n, re), budget, c->device, plan,
                                  ord_npos, solo_wide, lock_h, lock_w);
      if (!ok && auto_fifo) {
        // AUTO picked FIFO but its smallest batch does not fit: threshold
        // order needs far less memory per source (no maxId labels)
        o.schedule = GSOFA_SCHEDULE_THRESHOLD;
        key[0] = o.schedule;
        ok = make_plan_stream(n, rows, std::min<int64_t>(n, re), budget, c->device, plan, 0, solo_wide);
      }
      if (ok && !std::getenv("GSOFA_LIGHT_CTAS") && !std::getenv("GSOFA_SOLO_CTAS") &&
          !std::getenv("GSOFA_SOLO_RING") && !std::getenv("GSOFA_FRONTIER_FRAC_LOG")) {
        c->plan_cache = plan;
        std::copy(key, key + 7, c->plan_key);
      }
    }
    const int64_t budget = budget_req;  // (for the message below; 0 = automatic)
    if (!ok) {
      set_detail("budget %lld B cannot hold one 32-source group for n=%lld", (long long)budget,
                 (long long)n);
      rc = GSOFA_EINFEASIBLE;
      goto fail;
    }
  }
  if ((rc = ensure_arena(c, n, plan, st)) != GSOFA_OK) goto fail;
  if (o.schedule != GSOFA_SCHEDULE_FIFO) {
    // the slot layout (Vmax, ws_words) moved: list garbage could now sit
    // under state words, so start from an all-zero work region
    const uint64_t sig = ((uint64_t)plan.Vmax << 32) ^ (uint64_t)plan.ws_words ^
                         ((uint64_t)plan.light << 48) ^ ((uint64_t)plan.heavy << 40) ^
                         ((uint64_t)plan.hws_words << 8) ^ ((uint64_t)ord_npos << 20);
    if (c->layout_sig != sig && c->work_state == kWorkZero && c->layout_sig != 0) c->work_state = kWorkDirty;
    c->layout_sig = sig;
  }
  if ((rc = prepare_work(c, o.schedule, st)) != GSOFA_OK) goto fail;
  ev();
  CK(cudaMemsetAsync(c->stats, 0, 16 * sizeof(unsigned long long), st));
  // ---------------------------------------------------- outputs
  {
    cudaError_t e1 = cudaMallocAsync((void **)&Lrp, (rows + 1) * sizeof(int64_t), st);
    cudaError_t e2 = cudaMallocAsync((void **)&Urp, (rows + 1) * sizeof(int64_t), st);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      cudaGetLastError();
      set_detail("output row pointer allocation failed");
      rc = GSOFA_ENOMEM;
      goto fail;
    }
    CK(cudaMemsetAsync(Lrp, 0, sizeof(int64_t), st));
    CK(cudaMemsetAsync(Urp, 0, sizeof(int64_t), st));
    if (o.schedule == GSOFA_SCHEDULE_FIFO) {
      const size_t guess = (size_t)std::max<int64_t>(1024, 4 * (nnz + n) * rows / n);
      if ((rc = grow_device(&Lci, &Lcap, guess, st)) != GSOFA_OK) goto fail;
      if ((rc = grow_device(&Uci, &Ucap, guess, st)) != GSOFA_OK) goto fail;
    }
  }
  if (o.schedule != GSOFA_SCHEDULE_FIFO) {
    // ---------------------------------------------- streaming threshold schedule
    const int64_t ngroups = ceil_div(rows, 32);
    int64_t *row_off = nullptr;
    int32_t *row_nL = nullptr, *row_nU = nullptr, *failed = nullptr, *grp = nullptr;
    int32_t *hq = nullptr, *hq_ready = nullptr, *gflag = nullptr;
    {
      cudaError_t e1 = cudaMallocAsync((void **)&stream_scratch,
                                       (size_t)rows * 16 + (size_t)ngroups * 20 + 256, st);
      if (e1 != cudaSuccess) {
        cudaGetLastError();
        set_detail("row scratch allocation failed");
        rc = GSOFA_ENOMEM;
        goto fail;
      }
      char *q = (char *)stream_scratch;
      row_off = (int64_t *)q;
      row_nL = (int32_t *)(q + (size_t)rows * 8);
      row_nU = row_nL + rows;
      failed = row_nU + rows;
      grp = failed + ngroups;
      hq = grp + ngroups;
      hq_ready = hq + ngroups;
      gflag = hq_ready + ngroups;  // per group: already in the failed list
      CK(cudaMemsetAsync(hq_ready, 0, (size_t)ngroups * 8, st));  // hq_ready + gflag
    }
    ev();
    if (c->stage_cap == 0) {
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      size_t want = std::max<size_t>((size_t)1 << 24, (size_t)(fr * 0.3) / 4);
      // dev / tests: a small initial staging area exercises the overflow retry
      if (const char *e = std::getenv("GSOFA_STAGE_CAP")) want = std::max<size_t>(1024, atoll(e));
      if ((rc = grow_device(&c->stage, &c->stage_cap, want, st)) != GSOFA_OK) goto fail;
    }
    unsigned int *group_ctr = c->qcount;
    int32_t *nfailed = (int32_t *)(c->qcount + 1);
    unsigned long long *cursor = (unsigned long long *)c->totals;
    unsigned long long *failed_need = cursor + 1;
    // qcount: [0] group_ctr, [1] nfailed, [2] hq_head, [3] hq_tail, [4] done,
    // [5] solo_ctr, [6..7] task_ctr, [8] live lockstep CTAs
    // [9] unused
    CK(cudaMemsetAsync(c->qcount, 0, 40, st));
    CK(cudaMemsetAsync(c->totals, 0, 16, st));
    gsofa::StreamParams sp;
    sp.rowptr = c->rowptr32;
    sp.colidx = d_colidx;
    sp.n = (int32_t)n;
    sp.row_begin = (int32_t)rb;
    sp.row_end = (int32_t)re;
    sp.map = rmap;
    sp.nrows = (int32_t)rows;
    sp.ngroups = (int32_t)ngroups;
    sp.Vmax = (int32_t)plan.Vmax;
    sp.ws = c->work;
    sp.ws_words = plan.ws_words;
    sp.is = c->is;
    sp.is_words = plan.slot_is_words;
    sp.group_ctr = group_ctr;
    sp.solo_ctr = c->qcount + 5;
    sp.solo_top = 0;
    sp.group_list = nullptr;
    sp.list_len = 0;
    sp.stage = c->stage;
    sp.stage_cap = c->stage_cap;
    sp.stage_cursor = cursor;
    sp.row_off = row_off;
    sp.row_nL = row_nL;
    sp.row_nU = row_nU;
    sp.failed = failed;
    sp.failed_flag = gflag;
    sp.nfailed = nfailed;
    sp.failed_need = failed_need;
    sp.stats = c->stats;
    sp.group_trace = nullptr;
    sp.src_trace = nullptr;
    sp.ell = nullptr;
    sp.task_base = 0;
    const char *src_trace_path = std::getenv("GSOFA_SRC_TRACE");  // dev: per-source trace dump
    if (src_trace_path) {
      if (cudaMallocAsync((void **)&sp.src_trace, (size_t)rows * 32, st) != cudaSuccess) {
        cudaGetLastError();
        sp.src_trace = nullptr;
      } else {
        cudaMemsetAsync(sp.src_trace, 0, (size_t)rows * 32, st);
      }
    }
    sp.debug = nullptr;
    if (std::getenv("GSOFA_CHECK_CLEAN")) {
      cudaMallocAsync((void **)&sp.debug, 256, st);
      cudaMemsetAsync(sp.debug, 0, 256, st);
    }
    const char *trace_path = std::getenv("GSOFA_GROUP_TRACE");  // dev: per-group trace dump
    if (trace_path) {
      if (cudaMallocAsync((void **)&sp.group_trace, (size_t)ngroups * 64, st) != cudaSuccess) {
        cudaGetLastError();
        sp.group_trace = nullptr;
      } else {
        cudaMemsetAsync(sp.group_trace, 0, (size_t)ngroups * 64, st);
      }
    }
    sp.hq = hq;
    sp.hq_ready = hq_ready;
    sp.hq_head = c->qcount + 2;
    sp.hq_tail = c->qcount + 3;
    sp.done = c->qcount + 4;
    sp.light_live = c->qcount + 8;  // zeroed with qcount[0..8] below
    sp.task_ctr = (unsigned long long *)(c->qcount + 6);  // qcount[6..7]
    sp.hws = c->work + (size_t)plan.light * plan.ws_words;
    sp.hws_words = plan.hws_words;
    sp.solo_ring = gsofa::solo_ring(plan.Vmax);
    sp.light_slots = (int32_t)plan.light;
    sp.abort_cycles = 0;
    gsofa::solo_layout(plan.Vmax, n, ord_npos, &sp);
    sp.hmode = o.schedule == GSOFA_SCHEDULE_HEIGHT && !lock_h;  // AUTO: decided at the solo launch
    sp.lmode = lock_h;
    sp.lwarps = lock_w;
    sp.wide = solo_wide;
    sp.nnz = nnz;
    sp.npos = (int32_t)ord_npos;
    sp.posrec = reinterpret_cast<const int4 *>(c->ord_buf);  // 16-byte aligned (buffer start)
    sp.hgt = c->ord_buf + 4 * n;
    sp.pos = c->ord_buf + 5 * n;
    sp.ell = nullptr;
    if (maxdeg <= 8 && !sp.wide && !sp.hmode && std::getenv("GSOFA_ELL") && atoi(std::getenv("GSOFA_ELL")) != 0) {
      // dev A/B (GSOFA_ELL=1): id-order solo sources read neighbour lists from
      // an ELL copy (every row fits 8 entries) -- one dependent round trip
      // less per closure level, but measured slower (C5 3.41 -> 3.61 s, top
      // range 4.4 -> 4.6 us per level: the reached atomic, not the list
      // load, is the wait; profiles/r2/ell_ab.txt), so off by default
      if ((rc = grow_device(&c->ell, &c->ell_cap, (size_t)n * 8, st)) != GSOFA_OK) goto fail;
      CK(gsofa::launch_ell_build(c->rowptr32, d_colidx, (int32_t)n, c->ell, st));
      ++launches;
      sp.ell = c->ell;
    }
    if (plan.heavy > 0) {
      // the heaviest groups (top separator / hub rows) start on
      // the solo kernel: one per first-wave solo CTA (one per SM)
      int64_t top = std::min<int64_t>(plan.heavy, c->sms);
      if (const char *e = std::getenv("GSOFA_SOLO_TOP")) top = std::min<int64_t>(plan.heavy, atoll(e));
      sp.solo_top = (int32_t)std::min<int64_t>(top, ngroups);
      ev();
      // the solo_top heaviest groups are queued for the solo kernel up front
      if (sp.solo_top > 0) {
        std::vector<int32_t> hv((size_t)sp.solo_top * 2);
        for (int32_t i = 0; i < sp.solo_top; ++i) {
          hv[i] = (int32_t)ngroups - 1 - i;
          hv[sp.solo_top + i] = 1;
        }
        const uint32_t tail = (uint32_t)sp.solo_top;
        CK(cudaMemcpyAsync(hq, hv.data(), (size_t)sp.solo_top * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(hq_ready, hv.data() + sp.solo_top, (size_t)sp.solo_top * 4,
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(sp.hq_tail, &tail, 4, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));  // hv is a host temporary
      }
      double ms = 5.0;
      if (const char *e = std::getenv("GSOFA_ABORT_MS")) ms = atof(e);
      const int khz = c->clock_khz;
      sp.abort_cycles = (long long)(ms * (double)khz);
    }
    int64_t grid = plan.light;
    for (int pass = 0;; ++pass) {
      const int et0 = ev();
      if (pass == 0 && plan.heavy > 0) {
        // solo kernel (32-warp CTAs) on the second stream, concurrently with
        // the lockstep kernel; it serves the heavy queue until all are done
        cudaEvent_t ea, eb;
        CK(cudaEventCreateWithFlags(&ea, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&eb, cudaEventDisableTiming));
        CK(cudaEventRecord(ea, st));
        CK(gsofa::launch_stream(sp, (int)ceil_div(grid, gsofa::stream_warps_per_cta()), st));  // lockstep first
        CK(cudaStreamWaitEvent(c->stream2, ea, 0));
        if (ord_npos > 0) {
          // A2, height order: the elimination tree of A + A^T, heights and
          // (height, id) positions on the host (order.cu; SURVEY §8(a) A2,
          // O(nnz alpha)), while the lockstep kernel -- id order, no tree
          // needed -- runs; then up to the solo kernel's stream
          gsofa::OrderShape shape;
          CK(host_height_order(c, n, nnz, in_dev, rowptr, colidx, c->stream2, &shape));
          int32_t *ord_host = (int32_t *)c->ord_pin;
          if (auto_order) {
            // AUTO: height order when the last row's id-order chain (about
            // |L(n-1,:)| threshold steps) is far longer than the tree is
            // high (its rounds in height order) -- C4's hub rows: 577k vs
            // 4.2k; 3D grids: 58k vs 38k keep id order, which is faster per
            // step.  The chain-bound pattern also takes the latency shape.
            const bool use_h = shape.last_row_chain > 4 * shape.height;
            sp.hmode = use_h;
            if (!std::getenv("GSOFA_SOLO_WIDE")) sp.wide = use_h || solo_wide;
            o.schedule = use_h ? GSOFA_SCHEDULE_HEIGHT : GSOFA_SCHEDULE_THRESHOLD;
          }
          if (sp.hmode)
            CK(cudaMemcpyAsync(c->ord_buf, ord_host, (size_t)n * 6 * 4, cudaMemcpyHostToDevice, c->stream2));
        }
        // the solo kernel's first tasks are static per CTA, so every CTA of
        // its grid must be able to become resident: AUTO may have switched
        // the order / shape after the plan, so clamp to the residency of the
        // variant actually launched
        int64_t hgrid = plan.heavy;
        const int64_t hres =
            gsofa::stream_max_blocks(c->device, plan.Vmax, 1, sp.hmode ? ord_npos : 0, sp.wide);
        if (hres > 0) hgrid = std::min<int64_t>(hgrid, hres);
        sp.task_base = 0;
        CK(gsofa::launch_solo(sp, (int)hgrid, c->stream2));
        CK(cudaEventRecord(eb, c->stream2));
        CK(cudaStreamWaitEvent(st, eb, 0));
        cudaEventDestroy(ea);
        cudaEventDestroy(eb);
        launches += 2;
      } else {
        CK(gsofa::launch_stream(sp, (int)ceil_div(std::max<int64_t>(grid, 1), gsofa::stream_warps_per_cta()),
                                st));
        ++launches;
      }
      e_trav.push_back({et0, ev()});
      CK(cudaMemcpyAsync(c->h_small, c->totals, 16, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(c->h_small + 2, c->qcount, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      const unsigned long long used = (unsigned long long)c->h_small[0];
      const unsigned long long need = (unsigned long long)c->h_small[1];
      const int nf = (int)((uint32_t)(c->h_small[2] >> 32));
      if (nf == 0) break;
      if (pass > 4) {
        set_detail("staging retries did not converge");
        rc = GSOFA_EINTERNAL;
        goto fail;
      }
      // rows of nf groups did not fit: grow the staging area (keeping what is
      // there) and re-run just those groups
      if ((rc = grow_device(&c->stage, &c->stage_cap, (size_t)(used + need + (need >> 3) + 1024),
                            st)) != GSOFA_OK)
        goto fail;
      CK(cudaMemcpyAsync(grp, failed, (size_t)nf * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemsetAsync(gflag, 0, (size_t)ngroups * 4, st));
      CK(cudaMemsetAsync(c->qcount, 0, 8, st));
      CK(cudaMemsetAsync(failed_need, 0, 8, st));
      sp.stage = c->stage;
      sp.stage_cap = c->stage_cap;
      sp.group_list = grp;
      sp.list_len = nf;
      grid = std::min<int64_t>(plan.light, nf);
      sp.abort_cycles = 0;  // retries run on the lockstep kernel alone
      sp.solo_top = 0;
    }
    if (sp.src_trace) {
      std::vector<long long> h((size_t)rows * 4);
      cudaMemcpyAsync(h.data(), sp.src_trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (FILE *f = std::fopen(src_trace_path, "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
      }
      cudaFreeAsync(sp.src_trace, st);
    }
    if (sp.group_trace) {
      std::vector<long long> h((size_t)ngroups * 8);
      cudaMemcpyAsync(h.data(), sp.group_trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (FILE *f = std::fopen(trace_path, "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
      }
      cudaFreeAsync(sp.group_trace, st);
    }
    if (std::getenv("GSOFA_CHECK_CLEAN")) {
      // dev: every state word must be zero again after the traversal
      // (lists / queues excepted); report the first offenders per array
      cudaStreamSynchronize(st);
      std::vector<uint32_t> hw(c->work_bytes / 4), hi(c->is_words);
      cudaMemcpy(hw.data(), c->work, c->work_bytes, cudaMemcpyDeviceToHost);
      cudaMemcpy(hi.data(), c->is, c->is_words * 4, cudaMemcpyDeviceToHost);
      const size_t Vm = plan.Vmax, tbw = (Vm + 31) / 32, rsw = (Vm + 1023) / 1024;
      int reported = 0;
      for (int64_t sl = 0; sl < plan.light && reported < 8; ++sl) {
        const uint32_t *b = hw.data() + sl * plan.ws_words;
        for (size_t i = 0; i < 2 * Vm + tbw + rsw && reported < 8; ++i)
          if (b[i]) {
            std::fprintf(stderr, "[dirty] light slot %lld word %zu (%s) = %08x\n", (long long)sl, i,
                         i < 2 * Vm ? "state" : (i < 2 * Vm + tbw ? "thr" : "rsum"), b[i]);
            ++reported;
          }
      }
      {
        const size_t live = sp.so_queue;  // everything but the ring
        const int64_t nslots = plan.heavy * gsofa::solo_warps_per_cta();
        for (int64_t sl = 0; sl < nslots && reported < 16; ++sl) {
          const uint32_t *b = hw.data() + plan.light * plan.ws_words + sl * plan.hws_words;
          for (size_t i = 0; i < live && reported < 16; ++i)
            if (b[i]) {
              std::fprintf(stderr, "[dirty] solo slot %lld word %zu = %08x\n", (long long)sl, i, b[i]);
              ++reported;
            }
        }
      }
      for (size_t i = 0; i < hi.size() && reported < 24; ++i)
        if (hi[i]) {
          std::fprintf(stderr, "[dirty] is slot %zu word %zu = %08x\n", i / plan.slot_is_words,
                       i % plan.slot_is_words, hi[i]);
          ++reported;
        }
      std::fprintf(stderr, "[dirty] check done, %d reported\n", reported);
      if (sp.debug) {
        int hd[33];
        cudaMemcpy(hd, sp.debug, sizeof hd, cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "[solo-check] %d groups left reached bits\n", hd[0]);
        for (int i = 0; i < std::min(hd[0], 8); ++i)
          std::fprintf(stderr, "  g=%d vertex=%d val=%08x kind/cta=%d\n", hd[1 + 4 * i],
                       hd[2 + 4 * i], hd[3 + 4 * i], hd[4 + 4 * i]);
      }
    }
    // row pointers (int64: C5 has > 2^31 entries) and the final CSR gather
    {
      const int ex0 = ev();
      const size_t tmpb = gsofa::scan_tmp_bytes(rows);
      cudaError_t e1 = cudaMallocAsync(&scan_tmp, tmpb, st);
      if (e1 != cudaSuccess) {
        cudaGetLastError();
        set_detail("scan scratch allocation failed");
        rc = GSOFA_ENOMEM;
        goto fail;
      }
      CK(gsofa::scan_exclusive_i32_i64(row_nL, Lrp, rows, Lrp + rows, scan_tmp, tmpb, st));
      CK(gsofa::scan_exclusive_i32_i64(row_nU, Urp, rows, Urp + rows, scan_tmp, tmpb, st));
      launches += 4;
      CK(cudaMemcpyAsync(c->h_small, Lrp + rows, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(c->h_small + 1, Urp + rows, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      baseL = c->h_small[0];
      baseU = c->h_small[1];
      if ((rc = grow_device(&Lci, &Lcap, (size_t)std::max<int64_t>(baseL, 1), st)) != GSOFA_OK) goto fail;
      if ((rc = grow_device(&Uci, &Ucap, (size_t)std::max<int64_t>(baseU, 1), st)) != GSOFA_OK) goto fail;
      CK(gsofa::launch_gather(c->stage, row_off, row_nL, Lrp, Urp, (int)rows, Lci, Uci, st));
      ++launches;
      e_ext.push_back({ex0, ev()});
      cudaFreeAsync(scan_tmp, st);
      scan_tmp = nullptr;
    }
    nbatches = 1;
    maxC = 32 * std::min<int64_t>(plan.slots, ngroups);  // concurrent sources
  }
  // ---------------------------------------------------- batches (FIFO)
  for (int64_t s0 = rb; o.schedule == GSOFA_SCHEDULE_FIFO && s0 < re;) {
    // #C for this batch: the largest multiple of 32 whose bubble-removed
    // working set fits the work region ("dynamic space allocation",
    // P:768-778; "reduce the number of concurrent sources")
    const int64_t C = fit_batch(o.schedule, n, s0, std::min<int64_t>(c->Cmax, round_up(re - s0, 32)),
                                c->work_bytes, c->qfl);
    if (C < 32) {
      set_detail("work region too small for a 32-source group at s0=%lld", (long long)s0);
      rc = GSOFA_EINFEASIBLE;
      goto fail;
    }
    const int64_t G = C / 32;
    const int64_t vb = std::min<int64_t>(n, s0 + C);
    const int32_t s_end = (int32_t)std::min<int64_t>(re, s0 + C);
    const int et0 = ev();
    if (o.schedule == GSOFA_SCHEDULE_FIFO) {
      // epoch: a fresh value range below every value written so far
      if (c->floor < (uint32_t)(n + 2) + 1u) {
        CK(cudaMemsetAsync(c->work, 0xFF, fifo_label_bytes(c->work_bytes, c->qfl), st));
        c->floor = 0xFFFFFFFFu;
      }
      const uint32_t base = c->floor - (uint32_t)(n + 2);
      c->floor = base;
      // masks and queues at FIXED offsets (capacity Qm words per mask, Qq
      // items per queue in HBM): a mask array must never land on memory a
      // previous batch used as a queue
      const size_t lab_b = fifo_label_bytes(c->work_bytes, c->qfl);
      size_t Qm, Qq;
      fifo_caps(c->work_bytes, c->qfl, Qm, Qq);
      uint32_t *fmq = (uint32_t *)((char *)c->work + lab_b);
      // external frontier: queue items past Qq go to mapped pinned host
      // memory, at most G * vb - Qq per queue
      const size_t ext = (size_t)G * vb > Qq ? (size_t)G * vb - Qq : 0;
      if (ext && 2 * ext > c->spill_cap) {
        CK(cudaStreamSynchronize(st));
        if (c->spill) cudaFreeHost(c->spill);
        c->spill = c->spill_dev = nullptr;
        c->spill_cap = 0;
        cudaError_t e2 = cudaHostAlloc((void **)&c->spill, 2 * ext * 4, cudaHostAllocMapped);
        if (e2 == cudaSuccess) e2 = cudaHostGetDevicePointer((void **)&c->spill_dev, c->spill, 0);
        if (e2 != cudaSuccess) {
          cudaGetLastError();
          set_detail("external frontier: cudaHostAlloc(%zu bytes) failed", 2 * ext * 4);
          rc = GSOFA_ENOMEM;
          goto fail;
        }
        c->spill_cap = 2 * ext;
      }
      gsofa::BatchParams bp;
      bp.rowptr = c->rowptr32;
      bp.colidx = d_colidx;
      bp.n = (int32_t)n;
      bp.s0 = (int32_t)s0;
      bp.s_end = s_end;
      bp.G = (int32_t)G;
      bp.gbits = c->gbits;
      bp.Vb = (int32_t)vb;
      bp.base = base;
      bp.lab = c->work;
      bp.fm0 = fmq;
      bp.fm1 = fmq + Qm;
      bp.q0 = fmq + 2 * Qm;
      bp.q1 = fmq + 2 * Qm + Qq;
      bp.qcap = (uint32_t)std::min<size_t>(Qq, (size_t)G * vb);
      bp.qx0 = ext ? c->spill_dev : nullptr;
      bp.qx1 = ext ? c->spill_dev + ext : nullptr;
      bp.qcount = c->qcount;
      bp.is = c->is;
      bp.stats = c->stats;
      CK(cudaMemsetAsync(c->qcount, 0, 3 * sizeof(uint32_t), st));
      CK(gsofa::launch_seed(bp, st));
      CK(gsofa::launch_traverse(bp, o.fill_first ? 1 : 0, c->max_blocks[o.fill_first ? 1 : 0], st));
      launches += 2;
    }
    const int et1 = ev();
    e_trav.push_back({et0, et1});

    gsofa::ExtractParams ep;
    ep.is_ro = c->is;
    ep.is = c->is;
    ep.n = (int32_t)n;
    ep.s0 = (int32_t)s0;
    ep.s_end = s_end;
    ep.G = (int32_t)G;
    ep.nchunks = (int32_t)c->nsub;
    ep.cntL = c->cntL;
    ep.cntU = c->cntU;
    ep.rowL = c->rowL;
    ep.rowU = c->rowU;
    ep.totals = c->totals;
    ep.L_rowptr = Lrp;
    ep.U_rowptr = Urp;
    ep.row_begin = (int32_t)rb;
    ep.baseL = baseL;
    ep.baseU = baseU;
    ep.L_out = nullptr;
    ep.U_out = nullptr;
    CK(gsofa::launch_extract_count(ep, st));
    CK(gsofa::launch_extract_scan(ep, st));
    launches += 3;
    CK(cudaMemcpyAsync(c->h_small, c->totals, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    {
      const int64_t tL = c->h_small[0], tU = c->h_small[1];
      if ((rc = grow_device(&Lci, &Lcap, (size_t)(baseL + tL), st)) != GSOFA_OK) goto fail;
      if ((rc = grow_device(&Uci, &Ucap, (size_t)(baseU + tU), st)) != GSOFA_OK) goto fail;
      ep.L_out = Lci;
      ep.U_out = Uci;
      CK(gsofa::launch_extract_write(ep, st));
      ++launches;
      baseL += tL;
      baseU += tU;
    }
    e_ext.push_back({et1, ev()});
    ++nbatches;
    maxC = std::max(maxC, C);
    s0 += C;
  }
  // ---------------------------------------------------- supernodes (A8)
  e_sn0 = ev();
  {
    const size_t tmpb = gsofa::scan_tmp_bytes(rows);
    cudaError_t e1 = cudaMallocAsync((void **)&sn_scratch, (size_t)rows * 3 * sizeof(int32_t) + 64, st);
    cudaError_t e2 = cudaMallocAsync(&scan_tmp, tmpb, st);
    cudaError_t e3 = cudaMallocAsync((void **)&sn, (size_t)(rows + 1) * sizeof(int32_t), st);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      cudaGetLastError();
      set_detail("supernode scratch allocation failed");
      rc = GSOFA_ENOMEM;
      goto fail;
    }
    int32_t *flags = sn_scratch;                 // [2 rows]: Phase-I bits, leaders
    int32_t *pos = sn_scratch + 2 * rows;        // [rows]
    int32_t *total = (int32_t *)c->totals + 4;   // scratch int
    if (!sn_deferred)
      CK(gsofa::launch_supernode_flags(Lrp, Lci, Urp, rmap, (int32_t)rows, o.chunk_size,
                                       o.sn_cap_only, flags, st));
    else  // no leaders yet (gsofa_supernodes_gathered); the sentinel only
      CK(cudaMemsetAsync(flags + rows, 0, (size_t)rows * 4, st));
    CK(gsofa::scan_exclusive_i32(flags + rows, pos, rows, total, scan_tmp, tmpb, st));
    CK(gsofa::launch_supernode_scatter(flags + rows, pos, rmap, (int32_t)rows, total, sn, st));
    launches += 4;
    unsigned long long *offd = c->stats + 5;
    CK(gsofa::launch_count_offdiag(c->rowptr32, d_colidx, rmap, (int32_t)rows, offd, st));
    ++launches;
  }
  e_sn1 = ev();
  if (o.checked) {
    // ---------------------------------------------------- checked mode
    CK(cudaMemsetAsync(c->err, 0, sizeof(int), st));
    if (const char *inj = std::getenv("GSOFA_AUDIT_INJECT")) {
      // tests only: corrupt one output entry to show the audit catches it
      const int32_t v = (int32_t)n - 1;
      if (inj[0] == 'L' && baseL > 0) CK(cudaMemcpyAsync(Lci, &v, 4, cudaMemcpyHostToDevice, st));
      if (inj[0] == 'U' && baseU > 0) CK(cudaMemsetAsync(Uci, 0xFF, 4, st));
      CK(cudaStreamSynchronize(st));
    }
    CK(gsofa::launch_audit(c->rowptr32, d_colidx, Lrp, Lci, Urp, Uci, sn,
                           sn_deferred ? nullptr : (int32_t *)c->totals + 4, rmap, (int32_t)rows,
                           (int32_t)n, o.chunk_size, o.sn_cap_only, c->err, st));
    ++launches;
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (bad) {
      set_detail("checked mode: output invariants violated (bits %d:%s%s%s%s%s)", bad,
                 (bad & 1) ? " L-row order" : "", (bad & 2) ? " U-row order" : "",
                 (bad & 4) ? " A not within L+U" : "", (bad & 8) ? " supernode Def. T3" : "",
                 (bad & 16) ? " supernode maximality" : "");
      rc = GSOFA_EINTERNAL;
      goto fail;
    }
  }
  // ---------------------------------------------------- result
  res = (gsofa_result *)std::calloc(1, sizeof(ResultImpl));
  if (!res) {
    rc = GSOFA_ENOMEM;
    goto fail;
  }
  CK(cudaMemcpyAsync(c->h_small, c->stats, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->h_small + 16, (int32_t *)c->totals + 4, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  {
    const unsigned long long *hs = (const unsigned long long *)c->h_small;
    res->n = n;
    res->row_begin = rb;
    res->row_end = re;
    res->nnz_L = baseL;
    res->nnz_U = baseU;
    res->nsuper = sn_deferred ? -1 : *(int32_t *)(c->h_small + 16);
    res->rows = rows;
    res->interleave = ilv ? o.interleave : gsofa_interleave{0, 0, 0, 0};
    res->nnz_A_offdiag = (int64_t)hs[5];
    res->fill_count = baseL + (baseU - rows) - res->nnz_A_offdiag;
    res->device = c->device;
    res->schedule = o.schedule;
    reinterpret_cast<ResultImpl *>(res)->chunk_size = o.chunk_size;
    reinterpret_cast<ResultImpl *>(res)->cap_only = o.sn_cap_only;
    res->stats.frontier_items = (int64_t)hs[0];
    res->stats.edge_inspections = (int64_t)hs[1];
    res->stats.rounds = (int64_t)hs[2];
    res->stats.thresholds = (int64_t)hs[3];
    res->stats.item_edges = (int64_t)hs[4];
    res->stats.first_visits = (int64_t)hs[8];
    res->stats.source_expansions = (int64_t)hs[9];
    res->stats.frontier_spilled = (int64_t)hs[10];
    res->stats.batches = nbatches;
    res->stats.max_batch = maxC;
    res->stats.kernel_launches = launches;
  }
  if (o.outputs_on_device) {
    res->on_device = 1;
    res->L_rowptr = Lrp;
    res->U_rowptr = Urp;
    res->L_colidx = Lci;
    res->U_colidx = Uci;
    res->sn_start = sn;
    Lrp = Urp = nullptr;
    Lci = Uci = sn = nullptr;
  } else {
    res->on_device = 0;
    const size_t nl = (size_t)res->nnz_L, nu = (size_t)res->nnz_U, ns = (size_t)res->nsuper + 1;
    // pinned host storage (fast D2H), reused from the context pool when the
    // previous host result has been freed
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t need = al((rows + 1) * 8) * 2 + al(std::max<size_t>(nl, 1) * 4) +
                        al(std::max<size_t>(nu, 1) * 4) + al((rows + 1) * 4);  // sn_start: room for a stitch
    HostBlock *blk = c->hpool;
    if (!blk || blk->in_use || blk->cap < need) {
      if (blk && !blk->in_use) {  // too small: drop it
        host_block_release(blk);
        c->hpool = blk = nullptr;
      }
      HostBlock *nb = new (std::nothrow) HostBlock();
      if (!nb || cudaMallocHost((void **)&nb->p, need + need / 8) != cudaSuccess) {
        cudaGetLastError();
        delete nb;
        set_detail("pinned host output allocation failed");
        rc = GSOFA_ENOMEM;
        goto fail;
      }
      nb->cap = need + need / 8;
      nb->refs = 1;  // the result's reference
      if (!c->hpool) {
        c->hpool = nb;
        nb->refs = 2;  // + the pool's
      }
      blk = nb;
    } else {
      blk->refs += 1;
    }
    blk->in_use = true;
    reinterpret_cast<ResultImpl *>(res)->block = blk;
    {
      char *q = blk->p;
      res->L_rowptr = (int64_t *)q;
      q += al((rows + 1) * 8);
      res->U_rowptr = (int64_t *)q;
      q += al((rows + 1) * 8);
      res->L_colidx = (int32_t *)q;
      q += al(std::max<size_t>(nl, 1) * 4);
      res->U_colidx = (int32_t *)q;
      q += al(std::max<size_t>(nu, 1) * 4);
      res->sn_start = (int32_t *)q;
    }
    const int eh0 = ev();
    CK(cudaMemcpyAsync(res->L_rowptr, Lrp, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(res->U_rowptr, Urp, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    if (nl) CK(cudaMemcpyAsync(res->L_colidx, Lci, nl * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (nu) CK(cudaMemcpyAsync(res->U_colidx, Uci, nu * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(res->sn_start, sn, ns * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    const int eh1 = ev();
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, evs[eh0], evs[eh1]);
    res->stats.ms_transfer += ms;
  }
  e_end = ev();
  CK(cudaStreamSynchronize(st));
  {
    float ms = 0;
    cudaEventElapsedTime(&ms, evs[e_start], evs[e_end]);
    res->stats.ms_total = ms;
    if (!in_dev) {
      cudaEventElapsedTime(&ms, evs[e_start], evs[e_up]);
      res->stats.ms_transfer += ms;
    }
    for (auto &p : e_trav) {
      cudaEventElapsedTime(&ms, evs[p.first], evs[p.second]);
      res->stats.ms_traverse += ms;
    }
    for (auto &p : e_ext) {
      cudaEventElapsedTime(&ms, evs[p.first], evs[p.second]);
      res->stats.ms_extract += ms;
    }
    cudaEventElapsedTime(&ms, evs[e_sn0], evs[e_sn1]);
    res->stats.ms_supernode = ms;
    if (std::getenv("GSOFA_TIMELINE"))
      for (size_t i = 1; i < evs.size(); ++i) {
        cudaEventElapsedTime(&ms, evs[i - 1], evs[i]);
        std::fprintf(stderr, "[timeline] api.cu:%d -> api.cu:%d  gpu %.3f ms  host %.3f ms\n", ev_line[i - 1],
                     ev_line[i], ms, ev_host[i] - ev_host[i - 1]);
      }
  }
#undef ev
  if (sn_scratch) cudaFreeAsync(sn_scratch, st);
  if (scan_tmp) cudaFreeAsync(scan_tmp, st);
  if (stream_scratch) cudaFreeAsync(stream_scratch, st);
  if (Lrp) cudaFreeAsync(Lrp, st);
  if (Urp) cudaFreeAsync(Urp, st);
  if (Lci) cudaFreeAsync(Lci, st);
  if (Uci) cudaFreeAsync(Uci, st);
  if (sn) cudaFreeAsync(sn, st);
  cudaStreamSynchronize(st);
  for (auto e : evs) cudaEventDestroy(e);
  if (own_ctx) gsofa_context_destroy(c);
  *out = res;
  return GSOFA_OK;

fail:
  cudaStreamSynchronize(st);
  cudaGetLastError();
  if (sn_scratch) cudaFree(sn_scratch);
  if (scan_tmp) cudaFree(scan_tmp);
  if (stream_scratch) cudaFree(stream_scratch);
  if (Lrp) cudaFree(Lrp);
  if (Urp) cudaFree(Urp);
  if (Lci) cudaFree(Lci);
  if (Uci) cudaFree(Uci);
  if (sn) cudaFree(sn);
  if (res) {
    ResultImpl *impl = reinterpret_cast<ResultImpl *>(res);
    if (impl->block) {
      impl->block->in_use = false;
      host_block_release(impl->block);
    }
    std::free(res);
  }
  for (auto e : evs) cudaEventDestroy(e);
  // a failed batch may leave masks/bitmaps dirty: force re-initialisation
  release_arena(c);
  if (own_ctx) gsofa_context_destroy(c);
  return rc;
}

// ------------------------------------------------------------ partitioning
int gsofa_partition_rows(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t nparts,
                         int32_t align, int64_t *bounds) {
  if (n <= 0 || !rowptr || !colidx || nparts < 1 || align < 1 || !bounds) {
    set_detail("bad arguments to gsofa_partition_rows");
    return GSOFA_EINVAL;
  }
  if (is_device_ptr(rowptr) || is_device_ptr(colidx)) {
    set_detail("gsofa_partition_rows takes host pointers");
    return GSOFA_EINVAL;
  }
  const int64_t nnz = rowptr[n];
  // the loops below index colidx through rowptr: check it first (the same
  // row-pointer rules as the GPU validation)
  if (rowptr[0] != 0 || nnz < 0 || nnz >= (int64_t(1) << 31)) {
    set_detail("bad rowptr (rowptr[0] != 0 or nnz out of range)");
    return GSOFA_EBADCSR;
  }
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i] || rowptr[i + 1] > nnz) {
      set_detail("bad rowptr at row %lld", (long long)i);
      return GSOFA_EBADCSR;
    }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t cix = colidx[e];
      if (cix < 0 || cix >= n || (e > rowptr[i] && cix <= colidx[e - 1])) {
        set_detail("column out of range or not strictly increasing in row %lld", (long long)i);
        return GSOFA_EBADCSR;
      }
    }
  // elimination tree of A + A^T (Liu, with path compression; order.cu)
  std::vector<int32_t> parent(n, -1);
  gsofa::etree_sym(n, rowptr, colidx, parent.data(), nullptr);
  // work(s) ~ sum of out-degrees over the subtree of s (vertices reachable from
  // s through smaller ids are inside it; work grows with s)
  std::vector<double> w(n);
  for (int64_t v = 0; v < n; ++v) w[v] = 1.0 + (double)(rowptr[v + 1] - rowptr[v]);
  for (int64_t v = 0; v < n; ++v)
    if (parent[v] >= 0) w[parent[v]] += w[v];
  // cost(s) = work(s)^alpha; GSOFA_PART_ALPHA overrides (dev calibration)
  double alpha = part_alpha(nparts);
  if (const char *e = std::getenv("GSOFA_PART_ALPHA")) alpha = atof(e);
  std::vector<double> pre(n + 1, 0.0);
  for (int64_t v = 0; v < n; ++v) pre[v + 1] = pre[v] + (alpha == 1.0 ? w[v] : std::pow(w[v], alpha));
  bounds[0] = 0;
  for (int32_t p = 1; p < nparts; ++p) {
    const double target = pre[n] * p / nparts;
    int64_t s = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
    s = std::min<int64_t>(n, std::max<int64_t>(bounds[p - 1], (s + align / 2) / align * align));
    bounds[p] = s;
  }
  bounds[nparts] = n;
  return GSOFA_OK;
}

// ----------------------------------------------------- height order (A2)
int gsofa_height_order(int64_t n, const int64_t *rowptr, const int32_t *colidx, int32_t *parent,
                       int32_t *hgt, int32_t *pos, int64_t *height, int64_t *last_row_chain) {
  if (n <= 0 || n >= (int64_t(1) << 31) || !rowptr || !colidx) {
    set_detail("bad arguments to gsofa_height_order");
    return GSOFA_EINVAL;
  }
  if (is_device_ptr(rowptr) || is_device_ptr(colidx)) {
    set_detail("gsofa_height_order takes host pointers");
    return GSOFA_EINVAL;
  }
  const int64_t nnz = rowptr[n];
  if (rowptr[0] != 0 || nnz < 0 || nnz >= (int64_t(1) << 31)) {
    set_detail("bad rowptr (rowptr[0] != 0 or nnz out of range)");
    return GSOFA_EBADCSR;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (rowptr[i + 1] < rowptr[i] || rowptr[i + 1] > nnz) {
      set_detail("bad rowptr at row %lld", (long long)i);
      return GSOFA_EBADCSR;
    }
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t cix = colidx[e];
      if (cix < 0 || cix >= n || (e > rowptr[i] && cix <= colidx[e - 1])) {
        set_detail("column out of range or not strictly increasing in row %lld", (long long)i);
        return GSOFA_EBADCSR;
      }
    }
  }
  std::vector<int32_t> buf((size_t)n * 6);
  gsofa::OrderScratch *sc = gsofa::order_scratch_new();
  const gsofa::OrderShape sh =
      gsofa::height_order(n, rowptr, colidx, buf.data() + 4 * n, buf.data() + 5 * n, buf.data(), sc);
  if (parent) std::memcpy(parent, gsofa::order_scratch_parent(sc), (size_t)n * 4);
  gsofa::order_scratch_free(sc);
  if (hgt) std::memcpy(hgt, buf.data() + 4 * n, (size_t)n * 4);
  if (pos) std::memcpy(pos, buf.data() + 5 * n, (size_t)n * 4);
  if (height) *height = sh.height;
  if (last_row_chain) *last_row_chain = sh.last_row_chain;
  return GSOFA_OK;
}

}  // extern "C"
