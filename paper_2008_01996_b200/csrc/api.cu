// C-ABI of libkhb200 (declared in include/khb200.h).
#ifndef KH_DEFAULT_LANES
#define KH_DEFAULT_LANES 2
#endif
#ifndef KH_DEFAULT_SOLVE_LANES
#define KH_DEFAULT_SOLVE_LANES 2
#endif
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/khb200.h"
#include "kernels.h"
#include "symbolic.h"

struct kh_symbolic {
  kh::Symbolic S;
  // launch schedule derived from S (built once per analysis: kh_plan_bytes
  // and kh_plan_create of the same symbolic share it), keyed by the schedule
  // environment knobs
  mutable std::mutex sched_mu;
  mutable std::shared_ptr<const void> sched;
  mutable std::string sched_key;
};

static std::atomic<long long> g_launches{0};
void kh_note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaError_t kh_smem_optin(const void* kernel, int bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(kernel, dev);
  const auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[key] = bytes;
  return e;
}

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(KH_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Makes the plan's device current for one ABI call and restores the
// caller's current device afterwards (the caller's torch state is untouched).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

#define KH_CUDA(call)                                        \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);      \
  } while (0)

constexpr int32_t kDefaultLeaf = 24;
// fronts with m <= kClassMax[c] use the register-resident kernels; the rest
// ("large", class kSmallClasses) the level-synchronous DMMA kernels
constexpr int kSmallClasses = 6;
#ifndef KH_CLASS4
#define KH_CLASS4 96
#endif
constexpr int32_t kClassMax[kSmallClasses] = {32, 40, 48, 64, KH_CLASS4, 128};
#ifndef KH_WARP_CLASSES
#define KH_WARP_CLASSES 7
#endif
// the warp-per-front solve kernels take every class up to m <= 128 (R = 1, 2,
// 2, 2, 3, 4 rows per lane); c3 solve with the classes up to 64 / 96 / 128:
// 4.37 / 4.17 / 4.12 ms (the rest goes through the CTA kernels)
#ifndef KH_SOLVE_SMALL_CLASSES
#define KH_SOLVE_SMALL_CLASSES 6
#endif
constexpr int kSolveSmallClasses = KH_SOLVE_SMALL_CLASSES;  // classes with warp-per-front solves
constexpr int kClsStride = kSmallClasses + 2;
constexpr int32_t kAbsmaxBlocks = 64;
constexpr int32_t kResidualBlocks = 1184;  // 8 x 148 SMs

template <class T>
cudaError_t upload(T** dst, const T* src, size_t count) {
  *dst = nullptr;
  if (count == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dst), count * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

}  // namespace

struct kh_plan {
  int device = 0;
  int64_t n = 0, nnz = 0, max_batch = 0, slots = 0;
  int32_t nf = 0, max_p = 0, max_m = 0;
  std::vector<int32_t> level_off;  // levels d -> [level_off[d], level_off[d+1]) in level_fronts
  // kClsStride per level: starts of the front classes (m <= 32, 40, 48, 64, 96, 128, large)
  // relative to level_off[d], plus the end
  std::vector<int32_t> cls_off;
  const int32_t* classes(int32_t d) const { return cls_off.data() + kClsStride * d; }
  std::vector<int32_t> task_off;   // Schur-update tasks of level d: [task_off[d], task_off[d+1])
  // per level and warp-solve class: largest lower panel (the class's shared-memory size)
  std::vector<int32_t> small_panel_max;
  // per level: largest lower panel and m among the other fronts when they all
  // fit the bulk-copy staged solve kernels' shared memory (else 0)
  std::vector<int32_t> mid_panel_max, mid_m_max;
  std::vector<int32_t> big_m_max;  // per level: largest m among the fronts with m > 64 (streamed solves' stage size)
  int32_t* tasks = nullptr;        // device (front, tile row, tile col) triples
  // large-front schedule: per level an assembly list and per 32-wide pivot
  // block the diag / left-looking / TRSM lists (offsets into btasks, int32s)
  struct SuperBlock {  // one 64-pivot super-block of a level's large fronts: task lists in btasks
    int32_t piv_off, piv_n, trsm_off, trsm_n, upd_off, upd_n;
  };
  struct BigLevel {
    int32_t asm_off, asm_n;
    int32_t sb_off, nsb;  // 64-pivot super-blocks (sbinfo): pivot block, panel TRSM, panel update
  };
  std::vector<SuperBlock> sbinfo;
  double2* minv = nullptr;     // [max_batch][minv_size]: B images of a level's pivot blocks (pivot_block_kernel)
  int64_t minv_size = 1;
  std::vector<BigLevel> big;
  int32_t* btasks = nullptr;
  char* owned = nullptr;           // workspace allocated by the plan (null if caller-provided)
  // side streams: the fused-front kernels of a level run there (one stream
  // per size class, so the classes overlap each other's tails), concurrently
  // with the large-front kernels on the caller's stream; levels are joined
  // Shift lanes: a batch of shifts is split into n_lanes contiguous groups,
  // each walking the tree on its own stream set (lane 0's main stream is the
  // caller's): one lane's latency-bound kernels (pivot blocks, narrow-level
  // solves, level tails) overlap the other lanes' throughput-bound ones.
  struct Lane {
    cudaStream_t main = nullptr;  // lanes >= 1 (owned); lane 0 runs on the caller's stream
    cudaStream_t side[kSmallClasses] = {};
    cudaEvent_t ev_main = nullptr, ev_side[kSmallClasses] = {};
    cudaEvent_t ev_fwd = nullptr;   // large fronts' panels final (fused forward sweep may start)
    cudaEvent_t ev_done = nullptr;  // the lane's work is queued up to here (joined by the caller's stream)
  };
  static constexpr int kMaxLanes = 4;
  Lane lane[kMaxLanes];
  int factor_lanes = 1, solve_lanes = 1;
  // batches with fewer (front, shift) pairs than this run in one lane: on small
  // problems (c1: 16 shifts of a 15 x 15 mesh) a second lane only doubles the launches
  int64_t lane_min_work = 200000;
  int lanes_for(int configured, int64_t nshift) const { return nshift * nf >= lane_min_work ? configured : 1; }
  cudaEvent_t ev_fork = nullptr;
  // optional per-level timing of the factorization (kh_plan_set_level_timing):
  // lvl_ev[i] recorded on the caller's stream before level depth - i and at the end
  bool level_timing = false;
  std::vector<cudaEvent_t> lvl_ev;
  int32_t depth = 0;
  int64_t panel_total = 0, upd_size[2] = {0, 0}, rupd_size[2] = {0, 0};
  // device
  KhDevFront* fronts = nullptr;
  KhDevFront* lf_fronts = nullptr;
  KhKid* kids = nullptr;
  int32_t *child_list = nullptr, *relind = nullptr, *cmap = nullptr, *orig_dst = nullptr, *level_fronts = nullptr;
  int32_t* wdst = nullptr;  // originals' slots in the warp-front kernels' dense image
  // per small class: register-resident warp kernel tile count (0: shared-memory kernel)
  int warp_mt[kSmallClasses] = {};
  int n_fused = kSmallClasses;  // classes [0, n_fused) use the fused per-front factor kernels, the rest the large-front path
  int64_t *urows = nullptr, *orig_src = nullptr, *perm = nullptr, *indptr = nullptr, *indices = nullptr;
  double *mv = nullptr, *av = nullptr;
  double *om = nullptr, *oa = nullptr;  // values in front-original order (gathered on the device)
  int64_t n_orig = 0;
  double2* panels = nullptr;
  double2* upd[2] = {nullptr, nullptr};
  double2* rupd[2] = {nullptr, nullptr};
  double2* y = nullptr;
  double2* lam = nullptr;
  double* minpiv_work = nullptr;  // [max_batch][nf]
  double* absmax_work = nullptr;  // [max_batch][kAbsmaxBlocks]
  double* minpiv = nullptr;       // [slots]
  double* absmax = nullptr;       // [slots]
  double* resid_part = nullptr;   // [2][kResidualBlocks]

  KhTree tree() const {
    KhTree T;
    T.fronts = fronts;
    T.lf_fronts = lf_fronts;
    T.lf_base = level_fronts;
    T.kids = kids;
    T.child_list = child_list;
    T.relind = relind;
    T.cmap = cmap;
    T.urows = urows;
    T.orig_src = orig_src;
    T.orig_dst = orig_dst;
    T.mv = mv;
    T.av = av;
    T.om = om;
    T.oa = oa;
    T.nf = nf;
    T.n = n;
    T.panel_total = panel_total;
    return T;
  }
};

namespace {

void plan_release(kh_plan* p) {
  if (p->owned) cudaFree(p->owned);
  p->owned = nullptr;
  for (cudaEvent_t e : p->lvl_ev) cudaEventDestroy(e);
  p->lvl_ev.clear();
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  p->ev_fork = nullptr;
  for (kh_plan::Lane& L : p->lane) {
    for (cudaEvent_t* e : {&L.ev_main, &L.ev_fwd, &L.ev_done}) {
      if (*e) cudaEventDestroy(*e);
      *e = nullptr;
    }
    for (int c = 0; c < kSmallClasses; ++c) {
      if (L.ev_side[c]) cudaEventDestroy(L.ev_side[c]);
      if (L.side[c]) cudaStreamDestroy(L.side[c]);
      L.ev_side[c] = nullptr;
      L.side[c] = nullptr;
    }
    if (L.main) cudaStreamDestroy(L.main);
    L.main = nullptr;
  }
}

cudaError_t lane_create(kh_plan::Lane& L, bool own_main) {
  cudaError_t e = cudaSuccess;
  if (own_main) e = cudaStreamCreateWithFlags(&L.main, cudaStreamNonBlocking);
  for (int c = 0; c < kSmallClasses; ++c) {
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&L.side[c], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&L.ev_side[c], cudaEventDisableTiming);
  }
  for (cudaEvent_t* ev : {&L.ev_main, &L.ev_fwd, &L.ev_done})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  return e;
}

int env_lanes(const char* name, int dflt) {
  const char* v = std::getenv(name);
  const int n = v ? std::atoi(v) : dflt;
  return std::min(std::max(n, 1), kh_plan::kMaxLanes);
}

// fork: the side streams start after the work queued so far on `st`
cudaError_t fork_side(kh_plan::Lane& L, cudaStream_t st) {
  cudaError_t e = cudaEventRecord(L.ev_main, st);
  for (int c = 0; c < kSmallClasses && e == cudaSuccess; ++c) e = cudaStreamWaitEvent(L.side[c], L.ev_main, 0);
  return e;
}

// join every way: the next level on any stream sees this level's results
cudaError_t join_side(kh_plan::Lane& L, cudaStream_t st) {
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < kSmallClasses && e == cudaSuccess; ++c) e = cudaEventRecord(L.ev_side[c], L.side[c]);
  for (int c = 0; c < kSmallClasses && e == cudaSuccess; ++c) e = cudaStreamWaitEvent(st, L.ev_side[c], 0);
  if (e == cudaSuccess) e = cudaEventRecord(L.ev_main, st);
  for (int c = 0; c < kSmallClasses && e == cudaSuccess; ++c) e = cudaStreamWaitEvent(L.side[c], L.ev_main, 0);
  return e;
}

// One contiguous group of a batch's shifts and the streams it runs on.
struct LaneRun {
  kh_plan::Lane* L;
  cudaStream_t st;
  int64_t off;  // first shift of the group inside the batch (index into the per-batch work buffers)
  int32_t ns;
};

// Split ns shifts into at most `lanes` groups (multiples of 4 shifts: the
// register-resident front kernels put four shifts of a front in one CTA) and
// fork the extra lanes' streams off the caller's.
cudaError_t lanes_begin(kh_plan* p, int lanes, int32_t ns, cudaStream_t st, std::vector<LaneRun>& runs) {
  int32_t per = (ns + lanes - 1) / lanes;
  per = (per + 3) & ~3;
  runs.clear();
  for (int32_t off = 0, l = 0; off < ns; off += per, ++l)
    runs.push_back({&p->lane[l], l == 0 ? st : p->lane[l].main, off, std::min(per, ns - off)});
  cudaError_t e = cudaSuccess;
  if (runs.size() > 1) {
    e = cudaEventRecord(p->ev_fork, st);
    for (size_t l = 1; l < runs.size() && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(runs[l].st, p->ev_fork, 0);
  }
  for (size_t l = 0; l < runs.size() && e == cudaSuccess; ++l) e = fork_side(*runs[l].L, runs[l].st);
  return e;
}

// The caller's stream waits for the extra lanes.
cudaError_t lanes_end(cudaStream_t st, std::vector<LaneRun>& runs) {
  cudaError_t e = cudaSuccess;
  for (size_t l = 1; l < runs.size() && e == cudaSuccess; ++l) {
    e = cudaEventRecord(runs[l].L->ev_done, runs[l].st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, runs[l].L->ev_done, 0);
  }
  return e;
}

}  // namespace

extern "C" {

int kh_version(void) { return 1; }

int64_t kh_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* kh_status_string(int status) {
  switch (status) {
    case KH_OK: return "ok";
    case KH_ERR_DIMENSION: return "dimension mismatch";
    case KH_ERR_SINGULAR: return "singular matrix";
    case KH_ERR_INVALID: return "invalid usage";
    case KH_ERR_CUDA: return "CUDA error";
    case KH_ERR_NOMEM: return "out of device memory";
    default: return "unknown status";
  }
}

const char* kh_last_error(void) { return g_last_error.c_str(); }

namespace {
// per-thread, per-device scratch for plan-free reductions
cudaError_t scratch(double** out) {
  static thread_local double* part[64] = {nullptr};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!part[dev]) {
    e = cudaMalloc(&part[dev], 2 * kResidualBlocks * sizeof(double));
    if (e != cudaSuccess) return e;
  }
  *out = part[dev];
  return cudaSuccess;
}
}  // namespace

extern "C" int kh_dgemm_dd(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double* C_hi, double* C_lo, int64_t ldc, void* stream) {
  if ((m > 0 && n > 0) && (!A || !B || !C_hi || !C_lo)) return fail(KH_ERR_INVALID, "null argument");
  if (lda < m || ldb < k || ldc < m) return fail(KH_ERR_DIMENSION, "leading dimension too small");
  KH_CUDA(kh_launch_dgemm_dd(m, n, k, A, lda, B, ldb, C_hi, C_lo, ldc, static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

extern "C" int kh_csr_pair_residual_dd(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                       const double* m_vals, const double* a_vals, const double* Y1, int64_t ldy1,
                                       const double* Y2hi, const double* Y2lo, int64_t ldy2, const double* F,
                                       int64_t ldf, double* R, int64_t ldr, double* norms2, void* stream) {
  if (!indptr || !Y1 || !Y2hi || !Y2lo || !F || !norms2) return fail(KH_ERR_INVALID, "null argument");
  if (ldy1 < n || ldy2 < n || ldf < n || (R && ldr < n)) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = nullptr;
  KH_CUDA(scratch(&part));
  KH_CUDA(kh_launch_pair_residual_dd(n, nt, indptr, indices, m_vals, a_vals, Y1, ldy1, Y2hi, Y2lo, ldy2, F, ldf, R,
                                     ldr, part, kResidualBlocks, st));
  KH_CUDA(kh_launch_rowreduce(part, kResidualBlocks, 2, 0, norms2, st));
  return KH_OK;
}

extern "C" int kh_csr_pair_residual(int64_t n, int64_t nt, const int64_t* indptr, const int64_t* indices,
                                    const double* m_vals, const double* a_vals, const double* Y, int64_t ldy,
                                    const double* F, int64_t ldf, double* R, int64_t ldr, double* norms2,
                                    void* stream) {
  if (!indptr || !Y || !F || !norms2) return fail(KH_ERR_INVALID, "null argument");
  if (ldy < n || ldf < n || (R && ldr < n)) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = nullptr;
  KH_CUDA(scratch(&part));
  KH_CUDA(kh_launch_pair_residual(n, nt, indptr, indices, m_vals, a_vals, Y, ldy, F, ldf, R, ldr, part,
                                  kResidualBlocks, st));
  KH_CUDA(kh_launch_rowreduce(part, kResidualBlocks, 2, 0, norms2, st));
  return KH_OK;
}

extern "C" int kh_daxpy(int64_t n, double alpha, const double* x, double* y, void* stream) {
  if (n > 0 && (!x || !y)) return fail(KH_ERR_INVALID, "null argument");
  KH_CUDA(kh_launch_daxpy(n, alpha, x, y, static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

extern "C" int kh_sumsq(const double* x, int64_t n, double* out, void* stream) {
  if (!out || (n > 0 && !x)) return fail(KH_ERR_INVALID, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = nullptr;
  KH_CUDA(scratch(&part));
  KH_CUDA(kh_launch_sumsq(x, n, part, kResidualBlocks, st));
  KH_CUDA(kh_launch_rowreduce(part, kResidualBlocks, 1, 0, out, st));
  return KH_OK;
}

int kh_set_device(int device) {
  KH_CUDA(cudaSetDevice(device));
  return KH_OK;
}

int kh_stream_sync(void* stream) {
  KH_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

int kh_analyze(int64_t n, const int64_t* indptr, const int64_t* indices, int32_t leaf_size, kh_symbolic** out) {
  if (!out || (n > 0 && (!indptr || !indices))) return fail(KH_ERR_INVALID, "null argument");
  if (n < 0) return fail(KH_ERR_DIMENSION, "negative dimension");
  kh_symbolic* s = new kh_symbolic();
  std::string err = kh::analyze(n, indptr, indices, leaf_size > 0 ? leaf_size : kDefaultLeaf, s->S);
  if (!err.empty()) {
    delete s;
    return fail(KH_ERR_DIMENSION, err);
  }
  *out = s;
  return KH_OK;
}

int kh_analyze_union(int64_t n, const int64_t* indptr1, const int64_t* indices1, const int64_t* indptr2,
                     const int64_t* indices2, int32_t leaf_size, kh_symbolic** out) {
  if (!out || (n > 0 && (!indptr1 || !indices1 || !indptr2 || !indices2))) return fail(KH_ERR_INVALID, "null argument");
  if (n < 0) return fail(KH_ERR_DIMENSION, "negative dimension");
  // row-wise union of the two patterns (merge of sorted rows; rows that are
  // not sorted are concatenated and left to kh_analyze's symmetrization)
  std::vector<int64_t> ptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + (indptr1[i + 1] - indptr1[i]) + (indptr2[i + 1] - indptr2[i]);
  std::vector<int64_t> idx(ptr[n]);
  std::vector<int64_t> len(n);
  auto merge_rows = [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      const int64_t *a = indices1 + indptr1[i], *ae = indices1 + indptr1[i + 1];
      const int64_t *b = indices2 + indptr2[i], *be = indices2 + indptr2[i + 1];
      int64_t* o = idx.data() + ptr[i];
      const bool sorted = std::is_sorted(a, ae) && std::is_sorted(b, be);
      if (sorted) {
        int64_t* e = std::set_union(a, ae, b, be, o);
        len[i] = std::unique(o, e) - o;
      } else {
        int64_t* e = std::copy(b, be, std::copy(a, ae, o));
        len[i] = e - o;
      }
    }
  };
  const int nth = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < 4096 || nth == 1) {
    merge_rows(0, n);
  } else {
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(merge_rows, n * t / nth, n * (t + 1) / nth);
    merge_rows(0, n / nth);
    for (auto& x : th) x.join();
  }
  // compact
  std::vector<int64_t> cptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) cptr[i + 1] = cptr[i] + len[i];
  std::vector<int64_t> cidx(cptr[n]);
  for (int64_t i = 0; i < n; ++i) std::copy(idx.begin() + ptr[i], idx.begin() + ptr[i] + len[i], cidx.begin() + cptr[i]);
  return kh_analyze(n, cptr.data(), cidx.data(), leaf_size, out);
}

int kh_symbolic_stats_get(const kh_symbolic* s, kh_symbolic_stats* o) {
  if (!s || !o) return fail(KH_ERR_INVALID, "null argument");
  const kh::Symbolic& S = s->S;
  std::memset(o, 0, sizeof(*o));
  o->n = S.n;
  o->nnz = S.nnz;
  o->n_fronts = (int64_t)S.fronts.size();
  o->max_front = S.max_front;
  for (const auto& F : S.fronts) o->max_pivots = std::max<int64_t>(o->max_pivots, F.p);
  o->depth = S.max_depth;
  o->factor_nnz = S.factor_nnz;
  o->panel_entries = S.panel_total;
  o->upd_entries = S.upd_size[0] + S.upd_size[1] + S.rupd_size[0] + S.rupd_size[1] + S.n;
  o->leaf_size = S.leaf_size;
  o->flops = S.flops;
  return KH_OK;
}

int kh_symbolic_perm(const kh_symbolic* s, int64_t* perm) {
  if (!s || (!perm && s->S.n)) return fail(KH_ERR_INVALID, "null argument");
  std::copy(s->S.perm.begin(), s->S.perm.end(), perm);
  return KH_OK;
}

int kh_symbolic_fronts(const kh_symbolic* s, int64_t* first, int32_t* npiv, int32_t* nupd, int32_t* parent,
                       int32_t* depth) {
  if (!s) return fail(KH_ERR_INVALID, "null argument");
  const auto& Fs = s->S.fronts;
  for (size_t f = 0; f < Fs.size(); ++f) {
    if (first) first[f] = Fs[f].first;
    if (npiv) npiv[f] = Fs[f].p;
    if (nupd) nupd[f] = Fs[f].q;
    if (parent) parent[f] = Fs[f].parent;
    if (depth) depth[f] = Fs[f].depth;
  }
  return KH_OK;
}

int kh_align_values(int64_t n, const int64_t* pat_indptr, const int64_t* pat_indices, const int64_t* indptr,
                    const int64_t* indices, const double* vals, double* out) {
  if (n < 0 || (n > 0 && (!pat_indptr || !indptr))) return fail(KH_ERR_INVALID, "null argument");
  for (int64_t i = 0; i < n; ++i) {
    int64_t q = pat_indptr[i];
    const int64_t qe = pat_indptr[i + 1];
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
      const int64_t j = indices[e];
      while (q < qe && pat_indices[q] < j) out[q++] = 0.0;
      if (q == qe || pat_indices[q] != j) return fail(KH_ERR_DIMENSION, "matrix has entries outside the analyzed pattern");
      out[q++] = vals[e];
    }
    while (q < qe) out[q++] = 0.0;
  }
  return KH_OK;
}

int kh_symbolic_pattern(const kh_symbolic* s, int64_t* indptr, int64_t* indices) {
  if (!s || !indptr || (s->S.nnz && !indices)) return fail(KH_ERR_INVALID, "null argument");
  std::memcpy(indptr, s->S.pat_ptr.data(), sizeof(int64_t) * s->S.pat_ptr.size());
  if (s->S.nnz) std::memcpy(indices, s->S.pat_idx.data(), sizeof(int64_t) * s->S.nnz);
  return KH_OK;
}

int kh_symbolic_rows(const kh_symbolic* s, int64_t* rows) {
  if (!s || (!rows && !s->S.urows.empty())) return fail(KH_ERR_INVALID, "null argument");
  std::copy(s->S.urows.begin(), s->S.urows.end(), rows);
  return KH_OK;
}

void kh_symbolic_free(kh_symbolic* s) { delete s; }

}  // extern "C"

namespace {

// Host-side launch schedule derived from the analysis: fronts grouped per
// level and kernel class, Schur tiles and the large-front block lists.
// shared-memory budget (complex entries: panel + front vector) of the
// bulk-copy staged solve kernels for fronts with m > 64 (c3: 4500-8000 give
// 39.47 ms/step, 13000 -- one 208 KB CTA per SM on depth 6 -- 41.5, off 39.74)
#ifndef KH_MID_MAX_ENTRIES
#define KH_MID_MAX_ENTRIES 8000
#endif

struct Sched {
  std::vector<int32_t> small_panel_max, mid_panel_max, mid_m_max, big_m_max;
  std::vector<KhDevFront> df, lf_df;
  std::vector<KhKid> kids;
  std::vector<int32_t> orig_dst;  // device copy: packed offsets for the fused-front classes
  std::vector<int32_t> wdst;      // warp-front image slots (-1 outside the warp classes)
  int warp_mt[kSmallClasses] = {};
  int n_fused = kSmallClasses;  // classes factored by the fused per-front kernels (KH_SMALL_MAX)
  std::vector<int32_t> lf, level_off, cls_off, tasks, task_off, bt;
  std::vector<kh_plan::BigLevel> big;
  std::vector<kh_plan::SuperBlock> sbinfo;
  int32_t max_p = 0, max_m = 0;
  int64_t minv_size = 1;
};

void build_schedule(const kh::Symbolic& S, Sched& X) {
  const int32_t nf = (int32_t)S.fronts.size();
  X.df.resize(nf);
  for (int32_t f = 0; f < nf; ++f) {
    const kh::Front& F = S.fronts[f];
    KhDevFront& D = X.df[f];
    D.first = F.first;
    D.p = F.p;
    D.q = F.q;
    D.panel_off = F.panel_off;
    D.upd_off = F.upd_off;
    D.rupd_off = F.rupd_off;
    D.orig_begin = F.orig_begin;
    D.orig_end = F.orig_end;
    D.rows_begin = F.rows_begin;
    D.child_begin = S.child_ptr[f];
    D.child_end = S.child_ptr[f + 1];
    D.cmap_begin = F.cmap_begin;
    D.depth = F.depth;
    D.pad = 0;
    X.max_p = std::max(X.max_p, F.p);
    X.max_m = std::max(X.max_m, F.m());
  }
  // KH_SMALL_MAX caps the register/shared-memory small-front classes
  // (0 disables them, for A/B measurements)
  // default 96: the m <= 128 fused class measured slower than the large-front
  // super-block path for those fronts (c3 factorization 21.07 -> 20.70 ms)
  int small_max = 96;
  if (const char* env = std::getenv("KH_SMALL_MAX")) small_max = std::atoi(env);
  // Front lists are always ordered by the size classes (the solves pick their
  // kernels by class); the first n_fused classes are factored by the fused
  // per-front kernels, the rest by the large-front path
  int n_fused = 0;
  while (n_fused < kSmallClasses && kClassMax[n_fused] <= small_max) ++n_fused;
  X.n_fused = n_fused;
  auto front_class = [&](int32_t m) {
    for (int c = 0; c < kSmallClasses; ++c)
      if (m <= kClassMax[c]) return c;
    return kSmallClasses;  // m > 128
  };
  // originals of fused fronts address the packed block-column layout directly
  X.orig_dst = S.orig_dst;
  for (int32_t f = 0; f < nf; ++f) {
    const kh::Front& F = S.fronts[f];
    const int32_t m = F.m();
    if (front_class(m) >= n_fused) continue;
    for (int64_t e = F.orig_begin; e < F.orig_end; ++e) {
      const int32_t d = X.orig_dst[e], c = d / m, r = d - c * m;
      X.orig_dst[e] = kh_packed_col_base(m, c) + r;
    }
  }
  // register-resident warp kernels for the classes m <= 32 and m <= 48
  // (KH_WARP_CLASSES: bit c enables class c; default 0b111: m <= 32, 40, 48)
  int warp_mask = KH_WARP_CLASSES;
  if (const char* env = std::getenv("KH_WARP_CLASSES")) warp_mask = std::atoi(env);
  for (int c = 0; c < kSmallClasses; ++c)
    X.warp_mt[c] = ((warp_mask >> c) & 1) && kClassMax[c] <= 48 && c < n_fused ? kClassMax[c] / 8 : 0;
  X.wdst.assign(S.orig_dst.size(), -1);
  for (int32_t f = 0; f < nf; ++f) {
    const kh::Front& F = S.fronts[f];
    const int32_t m = F.m(), c = front_class(m);
    if (c >= n_fused || !X.warp_mt[c]) continue;
    for (int64_t e = F.orig_begin; e < F.orig_end; ++e) {
      const int32_t d = S.orig_dst[e], cc = d / m, r = d - cc * m;
      X.wdst[e] = kh_warp_front_slot(m, F.p, r, cc);
    }
  }
  X.level_off.push_back(0);
  for (const auto& lev : S.levels) {
    const int32_t base = (int32_t)X.lf.size();
    for (int c = 0; c <= kSmallClasses; ++c) {
      X.cls_off.push_back((int32_t)X.lf.size() - base);
      for (int32_t f : lev)
        if (front_class(S.fronts[f].m()) == c) X.lf.push_back(f);
    }
    X.cls_off.push_back((int32_t)X.lf.size() - base);
    X.level_off.push_back((int32_t)X.lf.size());
  }
  for (const auto& lev : S.levels) {
    // per class: the solve kernels of a class are launched with that class's
    // largest panel as shared memory (occupancy of the small classes)
    int32_t mx[kSolveSmallClasses];
    for (int c = 0; c < kSolveSmallClasses; ++c) mx[c] = 1;
    for (int32_t f : lev) {
      const kh::Front& F = S.fronts[f];
      const int c = front_class(F.m());
      if (c < kSolveSmallClasses) mx[c] = std::max<int32_t>(mx[c], F.p * F.m() - F.p * (F.p - 1) / 2);
    }
    for (int c = 0; c < kSolveSmallClasses; ++c) X.small_panel_max.push_back(mx[c]);
    int32_t pm = 0, mm = 0;
    for (int32_t f : lev) {
      const kh::Front& F = S.fronts[f];
      if (front_class(F.m()) >= kSolveSmallClasses) {
        pm = std::max<int32_t>(pm, F.p * F.m() - F.p * (F.p - 1) / 2);
        mm = std::max<int32_t>(mm, F.m());
      }
    }
    const bool fits = pm > 0 && pm + mm <= KH_MID_MAX_ENTRIES;
    X.mid_panel_max.push_back(fits ? pm : 0);
    X.mid_m_max.push_back(fits ? mm : 0);
    X.big_m_max.push_back(mm);
  }
  X.lf_df.resize(X.lf.size());
  for (size_t i = 0; i < X.lf.size(); ++i) {
    X.lf_df[i] = X.df[X.lf[i]];
    X.lf_df[i].pad = X.lf[i];
  }
  X.kids.resize(S.child_list.size());
  for (size_t j = 0; j < S.child_list.size(); ++j) {
    const kh::Front& C = S.fronts[S.child_list[j]];
    X.kids[j] = {C.upd_off, C.rows_begin, C.rupd_off, C.cmap_begin, C.q, 0};
  }
  X.task_off.push_back(0);
  for (size_t d = 0; d < S.levels.size(); ++d) {
    const int32_t first_large = X.level_off[d] + X.cls_off[kClsStride * d + n_fused];
    std::vector<int32_t> large(X.lf.begin() + first_large, X.lf.begin() + X.level_off[d + 1]);
    // Schur-update tasks: lower 64x64 tiles of U
    for (int32_t f : large) {
      const int32_t nt = (S.fronts[f].q + 63) / 64;
      for (int32_t jt = 0; jt < nt; ++jt)
        for (int32_t it = jt; it < nt; ++it) X.tasks.insert(X.tasks.end(), {f, it, jt});
    }
    X.task_off.push_back((int32_t)(X.tasks.size() / 3));
    kh_plan::BigLevel L{};
    L.asm_off = (int32_t)X.bt.size();
    auto img_tiles = [](int32_t p) { const int64_t pt = (p + 7) / 8; return pt * (pt + 1) / 2; };
    for (int32_t f : large) {
      const kh::Front& F = S.fronts[f];
      // (front, chunk start, originals range of the chunk): the originals of
      // a front are sorted by destination, so each chunk's range is found
      // here once instead of by a binary search in every CTA
      int64_t e = F.orig_begin;
      for (int32_t idx0 = 0; idx0 < F.m() * F.p; idx0 += KH_ASM_CHUNK) {
        const int32_t end = std::min(F.m() * F.p, idx0 + KH_ASM_CHUNK);
        while (e < F.orig_end && S.orig_dst[e] < idx0) ++e;
        const int64_t lo = e;
        while (e < F.orig_end && S.orig_dst[e] < end) ++e;
        X.bt.insert(X.bt.end(), {f, idx0, (int32_t)lo, (int32_t)e});
      }
    }
    L.asm_n = ((int32_t)X.bt.size() - L.asm_off) / 4;
    // super-block sbi (pivots c0 = 64 sbi .. c0 + w): pivot block (front, image
    // offset) -> TRSM of the rows below (front, row, offset) -> right-looking
    // update of the later pivot columns (front, row tile, column tile)
    constexpr int32_t SB = kh_piv_max();
    int32_t nsb = 0;
    for (int32_t f : large)
      nsb = std::max(nsb, (S.fronts[f].p + SB - 1) / SB);
    L.sb_off = (int32_t)X.sbinfo.size();
    L.nsb = nsb;
    for (int32_t sbi = 0; sbi < nsb; ++sbi) {
      const int32_t c0 = SB * sbi;
      kh_plan::SuperBlock K{};
      int64_t off = 0;
      K.piv_off = (int32_t)X.bt.size();
      for (int32_t f : large)
        if (S.fronts[f].p > c0) {
          X.bt.insert(X.bt.end(), {f, (int32_t)off});
          off += 64 * img_tiles(std::min(SB, S.fronts[f].p - c0));
        }
      K.piv_n = ((int32_t)X.bt.size() - K.piv_off) / 2;
      X.minv_size = std::max(X.minv_size, off);
      off = 0;
      K.trsm_off = (int32_t)X.bt.size();
      for (int32_t f : large) {
        const kh::Front& F = S.fronts[f];
        if (F.p <= c0) continue;
        const int32_t w = std::min(SB, F.p - c0);
        for (int32_t i0 = c0 + w; i0 < F.m(); i0 += 64) X.bt.insert(X.bt.end(), {f, i0, (int32_t)off});
        off += 64 * img_tiles(w);
      }
      K.trsm_n = ((int32_t)X.bt.size() - K.trsm_off) / 3;
      K.upd_off = (int32_t)X.bt.size();
      for (int32_t f : large) {
        const kh::Front& F = S.fronts[f];
        if (F.p <= c0 + SB) continue;
        for (int32_t j0 = c0 + SB; j0 < F.p; j0 += 64)
          for (int32_t i0 = j0; i0 < F.m(); i0 += 64) X.bt.insert(X.bt.end(), {f, i0, j0});
      }
      K.upd_n = ((int32_t)X.bt.size() - K.upd_off) / 3;
      X.sbinfo.push_back(K);
    }
    X.big.push_back(L);
  }
}

// Sub-allocator over one device workspace (256-byte aligned pieces). With a
// null base it only measures, so the same code computes the workspace size.
struct Carver {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  void take(T** out, size_t count) {
    off = (off + 255) & ~size_t(255);
    *out = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += std::max<size_t>(count * sizeof(T), 16);
  }
};

void carve(kh_plan* p, const kh::Symbolic& S, const Sched& X, Carver& C) {
  C.take(&p->fronts, X.df.size());
  C.take(&p->child_list, S.child_list.size());
  C.take(&p->relind, S.relind.size());
  C.take(&p->cmap, S.cmap.size());
  C.take(&p->urows, S.urows.size());
  C.take(&p->orig_src, S.orig_src.size());
  C.take(&p->orig_dst, S.orig_dst.size());
  C.take(&p->wdst, X.wdst.size());
  C.take(&p->level_fronts, X.lf.size());
  C.take(&p->lf_fronts, X.lf_df.size());
  C.take(&p->kids, X.kids.size());
  C.take(&p->tasks, X.tasks.size());
  C.take(&p->btasks, X.bt.size());
  C.take(&p->perm, (size_t)S.n);
  C.take(&p->indptr, (size_t)S.n + 1);
  C.take(&p->indices, (size_t)S.nnz);
  C.take(&p->mv, (size_t)S.nnz);
  C.take(&p->av, (size_t)S.nnz);
  C.take(&p->om, S.orig_src.size());
  C.take(&p->oa, S.orig_src.size());
  C.take(&p->panels, (size_t)(p->slots * S.panel_total));
  for (int k = 0; k < 2; ++k) {
    C.take(&p->upd[k], (size_t)(p->max_batch * p->upd_size[k]));
    C.take(&p->rupd[k], (size_t)(p->max_batch * p->rupd_size[k]));
  }
  C.take(&p->y, (size_t)(p->max_batch * S.n));
  C.take(&p->minv, (size_t)(p->max_batch * p->minv_size));
  C.take(&p->lam, (size_t)p->max_batch);
  C.take(&p->minpiv_work, (size_t)(p->max_batch * (int64_t)X.df.size()));
  C.take(&p->absmax_work, (size_t)(p->max_batch * kAbsmaxBlocks));
  C.take(&p->minpiv, (size_t)p->slots);
  C.take(&p->absmax, (size_t)p->slots);
  C.take(&p->resid_part, (size_t)(2 * kResidualBlocks));
}

void plan_sizes(kh_plan* p, const kh::Symbolic& S, int64_t max_batch, int64_t slots) {
  p->n = S.n;
  p->nnz = S.nnz;
  p->max_batch = max_batch;
  p->slots = slots;
  p->nf = (int32_t)S.fronts.size();
  p->depth = S.max_depth;
  p->panel_total = S.panel_total;
  for (int k = 0; k < 2; ++k) {
    p->upd_size[k] = std::max<int64_t>(S.upd_size[k], 1);
    p->rupd_size[k] = std::max<int64_t>(S.rupd_size[k], 1);
  }
}

// The symbolic's schedule, built on first use (thread-safe).
std::shared_ptr<const Sched> schedule_of(const kh_symbolic* s) {
  std::string key;
  for (const char* v : {"KH_SMALL_MAX", "KH_WARP_CLASSES"}) {
    const char* e = std::getenv(v);
    key += e ? e : "-";
    key += ';';
  }
  std::lock_guard<std::mutex> lock(s->sched_mu);
  if (!s->sched || s->sched_key != key) {
    auto X = std::make_shared<Sched>();
    build_schedule(s->S, *X);
    s->sched = X;
    s->sched_key = key;
  }
  return std::static_pointer_cast<const Sched>(s->sched);
}

}  // namespace

extern "C" {

int kh_plan_bytes(const kh_symbolic* s, int64_t max_batch, int64_t factor_slots, int64_t* bytes) {
  if (!s || !bytes) return fail(KH_ERR_INVALID, "null argument");
  kh_plan tmp;
  const Sched& X = *schedule_of(s);
  plan_sizes(&tmp, s->S, max_batch, factor_slots);
  tmp.minv_size = X.minv_size;
  Carver C;
  carve(&tmp, s->S, X, C);
  *bytes = (int64_t)C.off;
  return KH_OK;
}

int kh_plan_create(const kh_symbolic* s, int device, const int64_t* indptr, const int64_t* indices,
                   const double* m_vals, const double* a_vals, int64_t max_batch, int64_t factor_slots,
                   void* workspace, int64_t workspace_bytes, kh_plan** out) {
  if (!s || !out || !indptr || (s->S.nnz && (!indices || !m_vals || !a_vals)))
    return fail(KH_ERR_INVALID, "null argument");
  if (max_batch < 1 || factor_slots < max_batch) return fail(KH_ERR_INVALID, "need factor_slots >= max_batch >= 1");
  const kh::Symbolic& S = s->S;
  if (indptr[S.n] != S.nnz) return fail(KH_ERR_DIMENSION, "CSR does not match the analyzed pattern");
  if (S.orig_dst.size() >= (size_t)INT32_MAX)  // assembly tasks carry int32 originals ranges
    return fail(KH_ERR_DIMENSION, "too many original entries for one plan (>= 2^31)");
  DeviceGuard dev_guard(device);
  KH_CUDA(dev_guard.err);
  kh_plan* p = new kh_plan();
  p->device = device;
  plan_sizes(p, S, max_batch, factor_slots);
  const std::shared_ptr<const Sched> Xp = schedule_of(s);
  const Sched& X = *Xp;
  p->max_p = X.max_p;
  p->max_m = X.max_m;
  p->level_off = X.level_off;
  p->cls_off = X.cls_off;
  p->task_off = X.task_off;
  p->small_panel_max = X.small_panel_max;
  p->mid_panel_max = X.mid_panel_max;
  p->mid_m_max = X.mid_m_max;
  p->big_m_max = X.big_m_max;
  for (int c = 0; c < kSmallClasses; ++c) p->warp_mt[c] = X.warp_mt[c];
  p->n_fused = X.n_fused;
  p->big = X.big;
  p->sbinfo = X.sbinfo;
  p->minv_size = X.minv_size;
  Carver measure;
  carve(p, S, X, measure);
  cudaError_t e = cudaSuccess;
  Carver C;
  if (workspace) {
    if (workspace_bytes < (int64_t)measure.off) {
      delete p;
      return fail(KH_ERR_INVALID, "workspace smaller than kh_plan_bytes()");
    }
    C.base = static_cast<char*>(workspace);
  } else {
    e = cudaMalloc(reinterpret_cast<void**>(&p->owned), measure.off);
    C.base = p->owned;
  }
  p->factor_lanes = env_lanes("KH_LANES", KH_DEFAULT_LANES);
  p->solve_lanes = env_lanes("KH_SOLVE_LANES", KH_DEFAULT_SOLVE_LANES);
  if (const char* v = std::getenv("KH_LANES_MIN_WORK")) p->lane_min_work = std::atoll(v);
  for (int l = 0; l < std::max(p->factor_lanes, p->solve_lanes) && e == cudaSuccess; ++l)
    e = lane_create(p->lane[l], l > 0);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) {
    carve(p, S, X, C);
    auto up = [&](void* dst, const void* src, size_t bytes) {
      if (e == cudaSuccess && bytes) e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    };
    up(p->fronts, X.df.data(), X.df.size() * sizeof(KhDevFront));
    up(p->child_list, S.child_list.data(), S.child_list.size() * 4);
    up(p->relind, S.relind.data(), S.relind.size() * 4);
    up(p->cmap, S.cmap.data(), S.cmap.size() * 4);
    up(p->urows, S.urows.data(), S.urows.size() * 8);
    up(p->orig_src, S.orig_src.data(), S.orig_src.size() * 8);
    up(p->orig_dst, X.orig_dst.data(), X.orig_dst.size() * 4);
    up(p->wdst, X.wdst.data(), X.wdst.size() * 4);
    up(p->level_fronts, X.lf.data(), X.lf.size() * 4);
    up(p->lf_fronts, X.lf_df.data(), X.lf_df.size() * sizeof(KhDevFront));
    up(p->kids, X.kids.data(), X.kids.size() * sizeof(KhKid));
    up(p->tasks, X.tasks.data(), X.tasks.size() * 4);
    up(p->btasks, X.bt.data(), X.bt.size() * 4);
    up(p->perm, S.perm.data(), S.perm.size() * 8);
    up(p->indptr, indptr, ((size_t)S.n + 1) * 8);
    up(p->indices, indices, (size_t)S.nnz * 8);
    up(p->mv, m_vals, (size_t)S.nnz * 8);
    up(p->av, a_vals, (size_t)S.nnz * 8);
    p->n_orig = (int64_t)S.orig_src.size();
    if (e == cudaSuccess) e = kh_launch_gather_orig(p->n_orig, p->orig_src, p->mv, p->av, p->om, p->oa, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    plan_release(p);
    delete p;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? KH_ERR_NOMEM : KH_ERR_CUDA,
                std::string("kh_plan_create: ") + cudaGetErrorString(e));
  }
  *out = p;
  return KH_OK;
}

int kh_plan_set_values(kh_plan* p, const double* m_vals, const double* a_vals) {
  if (!p || (p->nnz && (!m_vals || !a_vals))) return fail(KH_ERR_INVALID, "null argument");
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  KH_CUDA(cudaMemcpy(p->mv, m_vals, p->nnz * 8, cudaMemcpyHostToDevice));
  KH_CUDA(cudaMemcpy(p->av, a_vals, p->nnz * 8, cudaMemcpyHostToDevice));
  KH_CUDA(kh_launch_gather_orig(p->n_orig, p->orig_src, p->mv, p->av, p->om, p->oa, 0));
  KH_CUDA(cudaDeviceSynchronize());
  return KH_OK;
}

namespace {

// Factor the batch; with `fwd`, also the forward sweep of the solve for the
// rhs already gathered into p->y (fused into the small-front kernels, the
// large fronts' forward kernels launched right after their level).
int factor_impl(kh_plan* p, int64_t slot0, int64_t nshift, const double* lambda_ri, cudaStream_t st, bool fwd) {
  KH_CUDA(cudaMemcpyAsync(p->lam, lambda_ri, nshift * 16, cudaMemcpyHostToDevice, st));
  const KhTree T = p->tree();
  if (p->level_timing && p->lvl_ev.size() < (size_t)p->depth + 2) {
    for (size_t i = p->lvl_ev.size(); i < (size_t)p->depth + 2; ++i) {
      cudaEvent_t e;
      KH_CUDA(cudaEventCreate(&e));
      p->lvl_ev.push_back(e);
    }
  }
  // per-level timing describes the single-lane schedule (levels of different lanes overlap otherwise)
  std::vector<LaneRun> runs;
  KH_CUDA(lanes_begin(p, p->level_timing ? 1 : p->lanes_for(p->factor_lanes, nshift), (int32_t)nshift, st, runs));
  for (int32_t d = p->depth; d >= 0; --d) {
    if (p->level_timing) KH_CUDA(cudaEventRecord(p->lvl_ev[p->depth - d], st));
    const int32_t* lev = p->level_fronts + p->level_off[d];
    const int32_t* co = p->classes(d);
    const int64_t sc = p->upd_size[d & 1], sch = p->upd_size[(d + 1) & 1];
    const int64_t rs = p->rupd_size[d & 1], rsh = p->rupd_size[(d + 1) & 1];
    const kh_plan::BigLevel& B = p->big[d];
    for (const LaneRun& R : runs) {
      kh_plan::Lane& L = *R.L;
      const int32_t ns = R.ns;
      double2* panels = p->panels + (slot0 + R.off) * p->panel_total;
      double2 *uc = p->upd[d & 1] + R.off * sc, *uch = p->upd[(d + 1) & 1] + R.off * sch;
      const double2* lam = p->lam + R.off;
      double* minpiv = p->minpiv_work + R.off * p->nf;
      double2* minv = p->minv + R.off * p->minv_size;
      const KhFwd fw{p->y + R.off * p->n, p->rupd[d & 1] + R.off * rs, rs, p->rupd[(d + 1) & 1] + R.off * rsh, rsh};
      for (int c = 0; c < p->n_fused; ++c) {
        if (p->warp_mt[c] && !fwd)
          KH_CUDA(kh_launch_warp_front(p->warp_mt[c], T, lev + co[c], co[c + 1] - co[c], ns, lam, panels, uc, sc, uch,
                                       sch, minpiv, p->wdst, L.side[c]));
        else
          KH_CUDA(kh_launch_factor_small(kClassMax[c], T, lev + co[c], co[c + 1] - co[c], ns, lam, panels, uc, sc,
                                         uch, sch, minpiv, L.side[c], fwd ? &fw : nullptr));
      }
      KH_CUDA(kh_launch_big_assemble(T, p->btasks + B.asm_off, B.asm_n, ns, lam, panels, uch, sch, R.st));
      for (int32_t sbi = 0; sbi < B.nsb; ++sbi) {
        const kh_plan::SuperBlock& K = p->sbinfo[B.sb_off + sbi];
        const int c0 = kh_piv_max() * sbi;
        KH_CUDA(kh_launch_pivot_block(T, p->btasks + K.piv_off, K.piv_n, c0, ns, panels, minpiv, minv, p->minv_size,
                                      R.st));
        KH_CUDA(kh_launch_panel_solve(T, p->btasks + K.trsm_off, K.trsm_n, c0, ns, panels, minv, p->minv_size, R.st));
        KH_CUDA(kh_launch_panel_update(T, p->btasks + K.upd_off, K.upd_n, c0, ns, panels, R.st));
      }
      if (fwd) {  // the level's large fronts: panels are final after their trsm;
                  // their forward sweep runs on a side stream beside the Schur kernel
        KH_CUDA(cudaEventRecord(L.ev_fwd, R.st));
        KH_CUDA(cudaStreamWaitEvent(L.side[0], L.ev_fwd, 0));
        KH_CUDA(kh_launch_fwd_level(T, lev + co[p->n_fused], co[kSmallClasses + 1] - co[p->n_fused], ns,
                                    p->max_m, panels, fw.y, fw.ru_cur, fw.ru_stride_cur, fw.ru_child,
                                    fw.ru_stride_child, L.side[0], 0, 0, p->big_m_max[d]));
      }
      KH_CUDA(kh_launch_schur(T, p->tasks + 3 * p->task_off[d], p->task_off[d + 1] - p->task_off[d], ns, panels, uc,
                              sc, uch, sch, R.st));
      KH_CUDA(join_side(L, R.st));
    }
  }
  KH_CUDA(lanes_end(st, runs));
  if (p->level_timing) KH_CUDA(cudaEventRecord(p->lvl_ev[p->depth + 1], st));
  KH_CUDA(kh_launch_rowreduce(p->minpiv_work, p->nf, (int32_t)nshift, 1, p->minpiv + slot0, st));
  KH_CUDA(kh_launch_shift_absmax_nnz(p->mv, p->av, p->nnz, (int32_t)nshift, p->lam, p->absmax_work,
                                     kAbsmaxBlocks, st));
  KH_CUDA(kh_launch_rowreduce(p->absmax_work, kAbsmaxBlocks, (int32_t)nshift, 2, p->absmax + slot0, st));
  return KH_OK;
}

int check_batch(kh_plan* p, int64_t slot0, int64_t nshift) {
  if (nshift < 0 || nshift > p->max_batch || slot0 < 0 || slot0 + nshift > p->slots)
    return fail(KH_ERR_INVALID, "shift batch outside the plan's slots");
  return KH_OK;
}

// one level of the forward / backward sweep for one lane's shifts
int solve_fwd_level(kh_plan* p, const KhTree& T, const LaneRun& R, int64_t slot0, int32_t d) {
  constexpr int L = kSolveSmallClasses;  // fronts with m <= 64 use the warp-per-front kernels, the rest the CTA ones
  const double2* panels = p->panels + (slot0 + R.off) * p->panel_total;
  double2* y = p->y + R.off * p->n;
  const int32_t* lev = p->level_fronts + p->level_off[d];
  const int32_t* co = p->classes(d);
  const int64_t sc = p->rupd_size[d & 1], sch = p->rupd_size[(d + 1) & 1];
  double2 *rc = p->rupd[d & 1] + R.off * sc, *rch = p->rupd[(d + 1) & 1] + R.off * sch;
  for (int c = 0; c < L; ++c)  // one launch per class (its own shared-memory size), on its own side stream
    KH_CUDA(kh_launch_fwd_small(T, lev + co[c], co[c + 1] - co[c], R.ns, panels, y, rc, sc, rch, sch,
                                p->small_panel_max[L * d + c], R.L->side[c], kClassMax[c]));
  KH_CUDA(kh_launch_fwd_level(T, lev + co[L], co[kSmallClasses + 1] - co[L], R.ns, p->max_m, panels, y, rc, sc, rch,
                              sch, R.st, p->mid_panel_max[d], p->mid_m_max[d], p->big_m_max[d]));
  KH_CUDA(join_side(*R.L, R.st));
  return KH_OK;
}

int solve_bwd_level(kh_plan* p, const KhTree& T, const LaneRun& R, int64_t slot0, int32_t d) {
  constexpr int L = kSolveSmallClasses;
  const double2* panels = p->panels + (slot0 + R.off) * p->panel_total;
  double2* y = p->y + R.off * p->n;
  const int32_t* lev = p->level_fronts + p->level_off[d];
  const int32_t* co = p->classes(d);
  for (int c = 0; c < L; ++c)
    KH_CUDA(kh_launch_bwd_small(T, lev + co[c], co[c + 1] - co[c], R.ns, panels, y, p->small_panel_max[L * d + c],
                                R.L->side[c], kClassMax[c]));
  KH_CUDA(kh_launch_bwd_level(T, lev + co[L], co[kSmallClasses + 1] - co[L], R.ns, p->max_p, p->max_m, panels, y,
                              R.st, p->mid_panel_max[d], p->mid_m_max[d], p->big_m_max[d]));
  KH_CUDA(join_side(*R.L, R.st));
  return KH_OK;
}

// backward sweep from p->y (forward-solved) and the scatter to x
int solve_bwd_impl(kh_plan* p, int64_t slot0, int32_t ns, double* x_re, double* x_im, int64_t ldx, cudaStream_t st) {
  const KhTree T = p->tree();
  std::vector<LaneRun> runs;
  KH_CUDA(lanes_begin(p, p->lanes_for(p->solve_lanes, ns), ns, st, runs));
  for (int32_t d = 0; d <= p->depth; ++d)
    for (const LaneRun& R : runs)
      if (int rc = solve_bwd_level(p, T, R, slot0, d)) return rc;
  KH_CUDA(lanes_end(st, runs));
  KH_CUDA(kh_launch_scatter_sol(p->n, ns, p->perm, p->y, x_re, x_im, ldx, st));
  return KH_OK;
}

}  // namespace

int kh_plan_factor(kh_plan* p, int64_t slot0, int64_t nshift, const double* lambda_ri, void* stream) {
  if (!p || (nshift > 0 && !lambda_ri)) return fail(KH_ERR_INVALID, "null argument");
  if (check_batch(p, slot0, nshift) != KH_OK) return KH_ERR_INVALID;
  if (nshift == 0) return KH_OK;
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  return factor_impl(p, slot0, nshift, lambda_ri, static_cast<cudaStream_t>(stream), false);
}

int kh_plan_factor_fwd(kh_plan* p, int64_t slot0, int64_t nshift, const double* lambda_ri, const double* b_re,
                       const double* b_im, int64_t ldb, void* stream) {
  if (!p || (nshift > 0 && (!lambda_ri || !b_re))) return fail(KH_ERR_INVALID, "null argument");
  if (check_batch(p, slot0, nshift) != KH_OK) return KH_ERR_INVALID;
  if (ldb < p->n) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  if (nshift == 0 || p->n == 0) return KH_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  KH_CUDA(kh_launch_gather_rhs(p->n, (int32_t)nshift, p->perm, b_re, b_im, ldb, p->y, st));
  return factor_impl(p, slot0, nshift, lambda_ri, st, true);
}

int kh_plan_solve_bwd(kh_plan* p, int64_t slot0, int64_t nshift, double* x_re, double* x_im, int64_t ldx,
                      void* stream) {
  if (!p || (nshift > 0 && !x_re)) return fail(KH_ERR_INVALID, "null argument");
  if (check_batch(p, slot0, nshift) != KH_OK) return KH_ERR_INVALID;
  if (ldx < p->n) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  if (nshift == 0 || p->n == 0) return KH_OK;
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  return solve_bwd_impl(p, slot0, (int32_t)nshift, x_re, x_im, ldx, static_cast<cudaStream_t>(stream));
}

int kh_plan_factor_solve(kh_plan* p, int64_t slot0, int64_t nshift, const double* lambda_ri, const double* b_re,
                         const double* b_im, int64_t ldb, double* x_re, double* x_im, int64_t ldx, void* stream) {
  if (!p || (nshift > 0 && (!lambda_ri || !b_re || !x_re))) return fail(KH_ERR_INVALID, "null argument");
  if (ldx < p->n) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  const int rc = kh_plan_factor_fwd(p, slot0, nshift, lambda_ri, b_re, b_im, ldb, stream);
  if (rc != KH_OK) return rc;
  return kh_plan_solve_bwd(p, slot0, nshift, x_re, x_im, ldx, stream);
}

int kh_plan_factor_storage(const kh_plan* p, void** panels, int64_t* panel_total) {
  if (!p || !panels || !panel_total) return fail(KH_ERR_INVALID, "null argument");
  *panels = p->panels;
  *panel_total = p->panel_total;
  return KH_OK;
}

int kh_plan_set_level_timing(kh_plan* p, int32_t on) {
  if (!p) return fail(KH_ERR_INVALID, "null argument");
  p->level_timing = on != 0;
  return KH_OK;
}

int kh_plan_level_times(kh_plan* p, float* ms, int32_t n_levels) {
  if (!p || !ms) return fail(KH_ERR_INVALID, "null argument");
  if (n_levels != p->depth + 1) return fail(KH_ERR_DIMENSION, "n_levels must be the tree depth + 1");
  if (!p->level_timing || p->lvl_ev.size() < (size_t)p->depth + 2)
    return fail(KH_ERR_INVALID, "level timing was not enabled for the last factorization");
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  KH_CUDA(cudaEventSynchronize(p->lvl_ev[p->depth + 1]));
  for (int32_t i = 0; i <= p->depth; ++i) {
    float t = 0.f;
    KH_CUDA(cudaEventElapsedTime(&t, p->lvl_ev[i], p->lvl_ev[i + 1]));
    ms[p->depth - i] = t;  // index by depth (0 = root)
  }
  return KH_OK;
}

int kh_plan_pivot_check(kh_plan* p, int64_t slot0, int64_t nshift, double rel_threshold, void* stream,
                        int64_t* first_bad, double* worst_ratio) {
  if (!p) return fail(KH_ERR_INVALID, "null argument");
  if (nshift < 0 || slot0 < 0 || slot0 + nshift > p->slots) return fail(KH_ERR_INVALID, "slots out of range");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  std::vector<double> mp(nshift), am(nshift);
  if (nshift) {
    KH_CUDA(cudaMemcpyAsync(mp.data(), p->minpiv + slot0, nshift * 8, cudaMemcpyDeviceToHost, st));
    KH_CUDA(cudaMemcpyAsync(am.data(), p->absmax + slot0, nshift * 8, cudaMemcpyDeviceToHost, st));
  }
  KH_CUDA(cudaStreamSynchronize(st));
  int64_t bad = -1;
  double worst = INFINITY;
  for (int64_t s = 0; s < nshift; ++s) {
    double ratio = am[s] > 0.0 ? mp[s] / am[s] : 0.0;
    if (!(mp[s] >= 0.0) || !std::isfinite(mp[s])) ratio = -1.0;
    worst = std::min(worst, ratio);
    if (bad < 0 && (am[s] == 0.0 || !(ratio >= rel_threshold))) bad = s;
  }
  if (first_bad) *first_bad = bad;
  if (worst_ratio) *worst_ratio = worst;
  if (bad >= 0) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "pivot %.3e below threshold %.3e (shift %lld)", mp[bad] < 0 ? NAN : mp[bad],
                  rel_threshold * am[bad], (long long)bad);
    return fail(KH_ERR_SINGULAR, buf);
  }
  return KH_OK;
}

int kh_plan_solve(kh_plan* p, int64_t slot0, int64_t nshift, const double* b_re, const double* b_im, int64_t ldb,
                  double* x_re, double* x_im, int64_t ldx, void* stream) {
  if (!p || (nshift > 0 && (!b_re || !x_re))) return fail(KH_ERR_INVALID, "null argument");
  if (nshift < 0 || nshift > p->max_batch || slot0 < 0 || slot0 + nshift > p->slots)
    return fail(KH_ERR_INVALID, "shift batch outside the plan's slots");
  if (ldb < p->n || ldx < p->n) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  if (nshift == 0 || p->n == 0) return KH_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  const KhTree T = p->tree();
  const int32_t ns = (int32_t)nshift;
  KH_CUDA(kh_launch_gather_rhs(p->n, ns, p->perm, b_re, b_im, ldb, p->y, st));
  // each lane runs its forward sweep and goes straight into its backward sweep
  std::vector<LaneRun> runs;
  KH_CUDA(lanes_begin(p, p->lanes_for(p->solve_lanes, ns), ns, st, runs));
  for (int32_t d = p->depth; d >= 0; --d)
    for (const LaneRun& R : runs)
      if (int rc = solve_fwd_level(p, T, R, slot0, d)) return rc;
  for (int32_t d = 0; d <= p->depth; ++d)
    for (const LaneRun& R : runs)
      if (int rc = solve_bwd_level(p, T, R, slot0, d)) return rc;
  KH_CUDA(lanes_end(st, runs));
  KH_CUDA(kh_launch_scatter_sol(p->n, ns, p->perm, p->y, x_re, x_im, ldx, st));
  return KH_OK;
}

int kh_plan_residual_scale(kh_plan* p, int64_t nt, const double* Y, int64_t ldy, const double* F, int64_t ldf,
                           double* norms2, void* stream) {
  if (!p || !Y || !F || !norms2) return fail(KH_ERR_INVALID, "null argument");
  if (ldy < p->n || ldf < p->n) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  KH_CUDA(kh_launch_residual_scale(p->n, nt, p->indptr, p->indices, p->mv, p->av, Y, ldy, F, ldf, p->resid_part,
                                   kResidualBlocks, st));
  KH_CUDA(kh_launch_rowreduce(p->resid_part, kResidualBlocks, 2, 0, norms2, st));
  return KH_OK;
}

int kh_plan_residual_dd(kh_plan* p, int64_t nt, const double* Y1, int64_t ldy1, const double* Y2hi,
                        const double* Y2lo, int64_t ldy2, const double* F, int64_t ldf, double* R, int64_t ldr,
                        double* norms2, void* stream) {
  if (!p || !Y1 || !Y2hi || !Y2lo || !F || !norms2) return fail(KH_ERR_INVALID, "null argument");
  if (ldy1 < p->n || ldy2 < p->n || ldf < p->n || (R && ldr < p->n))
    return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  KH_CUDA(kh_launch_pair_residual_dd(p->n, nt, p->indptr, p->indices, p->mv, p->av, Y1, ldy1, Y2hi, Y2lo, ldy2, F,
                                     ldf, R, ldr, p->resid_part, kResidualBlocks, st));
  KH_CUDA(kh_launch_rowreduce(p->resid_part, kResidualBlocks, 2, 0, norms2, st));
  return KH_OK;
}

int kh_plan_residual(kh_plan* p, int64_t nt, const double* Y, int64_t ldy, const double* F, int64_t ldf, double* R,
                     int64_t ldr, double* norms2, void* stream) {
  if (!p || !Y || !F || !norms2) return fail(KH_ERR_INVALID, "null argument");
  if (ldy < p->n || ldf < p->n || (R && ldr < p->n)) return fail(KH_ERR_DIMENSION, "leading dimension smaller than n");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DeviceGuard dev_guard(p->device);
  KH_CUDA(dev_guard.err);
  KH_CUDA(kh_launch_pair_residual(p->n, nt, p->indptr, p->indices, p->mv, p->av, Y, ldy, F, ldf, R, ldr,
                                  p->resid_part, kResidualBlocks, st));
  KH_CUDA(kh_launch_rowreduce(p->resid_part, kResidualBlocks, 2, 0, norms2, st));
  return KH_OK;
}

void kh_plan_free(kh_plan* p) {
  if (!p) return;
  DeviceGuard dev_guard(p->device);
  plan_release(p);
  delete p;
}

int kh_dgemm(int64_t m, int64_t n, int64_t k, double alpha, const double* A, int64_t lda, const double* B,
             int64_t ldb, double beta, double* C, int64_t ldc, void* stream) {
  if (m < 0 || n < 0 || k < 0) return fail(KH_ERR_DIMENSION, "negative GEMM dimension");
  if ((m > 0 && lda < m) || (k > 0 && ldb < k) || (m > 0 && ldc < m))
    return fail(KH_ERR_DIMENSION, "GEMM leading dimension too small");
  if (m && n && (!C || (k && (!A || !B)))) return fail(KH_ERR_INVALID, "null GEMM operand");
  KH_CUDA(kh_launch_dgemm(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

int kh_dgemm_rowscatter(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* const* dst, int32_t parts, int64_t rows_per_part, int64_t ld_dst, void* stream) {
  if (m < 0 || n < 0 || k < 0 || parts < 1 || rows_per_part < 1) return fail(KH_ERR_DIMENSION, "bad scatter shape");
  if ((int64_t)parts * rows_per_part < m) return fail(KH_ERR_DIMENSION, "parts do not cover the rows");
  if ((m > 0 && lda < m) || (k > 0 && ldb < k) || ld_dst < rows_per_part)
    return fail(KH_ERR_DIMENSION, "GEMM leading dimension too small");
  if (m && n && (!dst || (k && (!A || !B)))) return fail(KH_ERR_INVALID, "null GEMM operand");
  KH_CUDA(kh_launch_dgemm_rowscatter(m, n, k, A, lda, B, ldb, dst, rows_per_part, ld_dst,
                                     static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

int kh_sum_parts(int32_t parts, const double* slots, int64_t part_elems, double* out, void* stream) {
  if (parts < 1 || part_elems < 0) return fail(KH_ERR_DIMENSION, "bad part count");
  if (part_elems && (!slots || !out)) return fail(KH_ERR_INVALID, "null argument");
  KH_CUDA(kh_launch_sum_parts(parts, slots, part_elems, out, static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

int kh_ht_workspace_bytes(int32_t degree, int64_t n_cells, int64_t* bytes) {
  if ((degree != 1 && degree != 2) || n_cells < 1 || degree * n_cells > (1 << 20))
    return fail(KH_ERR_DIMENSION, "H_T assembly: degree must be 1 or 2 and n_cells >= 1");
  if (!bytes) return fail(KH_ERR_INVALID, "null argument");
  const int nr = (int)(degree * n_cells);
  *bytes = (int64_t)sizeof(double) * kh_ht::workspace_doubles(nr, (int)n_cells, kh_ht::chunk(nr));
  return KH_OK;
}

int kh_ht_assemble(int32_t degree, int64_t n_cells, const double* nodes, int64_t j_max, double* A, double* M,
                   double* C, void* workspace, int64_t workspace_bytes, void* stream) {
  int64_t need = 0;
  int st = kh_ht_workspace_bytes(degree, n_cells, &need);
  if (st != KH_OK) return st;
  if (j_max < 0) return fail(KH_ERR_DIMENSION, "j_max must be >= 0");
  if (!nodes || !A || !M || !C || !workspace) return fail(KH_ERR_INVALID, "null argument");
  if (workspace_bytes < need) return fail(KH_ERR_DIMENSION, "H_T workspace too small");
  double T = 0.0;
  KH_CUDA(cudaMemcpy(&T, nodes + n_cells, sizeof(double), cudaMemcpyDeviceToHost));
  if (!(T > 0.0)) return fail(KH_ERR_INVALID, "nodes must end at T > 0");
  const int nr = (int)(degree * n_cells);
  KH_CUDA(kh_ht::assemble(degree, (int)n_cells, nodes, T, j_max, kh_ht::chunk(nr), A, M, C,
                          static_cast<double*>(workspace), static_cast<cudaStream_t>(stream)));
  return KH_OK;
}

int kh_ipc_handle(const void* dev_ptr, void* handle, int64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(KH_ERR_INVALID, "null argument");
  // the handle names the whole allocation and opens at its base: report
  // where dev_ptr sits inside it (caching allocators sub-allocate)
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  KH_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(KH_ERR_CUDA, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (reinterpret_cast<GetRange>(fn)(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
    return fail(KH_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  KH_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &h, sizeof h);
  *offset = (int64_t)(reinterpret_cast<unsigned long long>(dev_ptr) - base);
  return KH_OK;
}

int kh_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(KH_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  KH_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return KH_OK;
}

int kh_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(KH_ERR_INVALID, "null argument");
  KH_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return KH_OK;
}

}  // extern "C"
