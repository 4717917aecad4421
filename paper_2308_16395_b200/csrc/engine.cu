// Host side of the B200 streaming ST-HOSVD engine and its C ABI (include/tsg.h).
//
// The handle owns the streaming state in HBM in the reference's layouts
// (SURVEY A19): factors U_k (N_k x R_k, column-major, ld N_k, capacity N_k
// columns), core and right factor Q as n x r slabs (core colexicographic
// R_0 x .. x R_{d-2} x r == v_tensor's buffer, streaming.cpp:19-35), the
// streaming factor ("left") row-major n_d x capr, and a device control block
// holding ledgers, ranks and per-slice scalars. The steady-state update
// (no basis growth) is enqueued with exactly one host synchronisation: after
// the mode projections, to learn whether a non-streaming basis must grow.
// Growth (rare) and stream_init run host-orchestrated on the same kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>
#include <limits>
#include <cstdio>

#include "../../include/tsg.h"
#include "kernels.cuh"

using namespace tsg;

namespace {

struct TsgError : std::runtime_error {
  int code;
  TsgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw TsgError(code, msg); }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(TSG_EDEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

thread_local std::string g_free_err;

long long prod(const long long* d, int n) {
  long long p = 1;
  for (int i = 0; i < n; ++i) p *= d[i];
  return p;
}

}  // namespace

struct tsg_stream {
  int device = 0;
  int flags = 0;
  cudaStream_t st = nullptr;
  std::string err;

  // dims (host mirror; exact)
  int d = 0;
  double tau = 0.0;
  long long N[kMaxD] = {0};
  long long R[kMaxD] = {0};
  long long n_d = 0;
  long long insertions_host = 0;
  int r_host = 0;  // streaming rank as of the last synchronisation
  int capr = 0;
  long long cap_rows = 0;
  long long slice_elems = 0;
  bool initialized = false;

  // device state
  double* U[kMaxD] = {nullptr};
  double *core = nullptr, *core2 = nullptr, *Q = nullptr, *Q2 = nullptr;
  long long qcap = 0;  // doubles per Q/core buffer
  double *sigma = nullptr, *sigma2 = nullptr;
  double *left = nullptr, *left2 = nullptr;
  double* slice = nullptr;   // device staging for host slices
  double* slice_b = nullptr; // second caller-visible slice buffer
  double *w0 = nullptr, *w1 = nullptr, *w2 = nullptr;
  double* ebuf = nullptr;
  double* kbuf = nullptr;
  double* evec = nullptr;
  double* partial = nullptr;
  long long partial_cap = 0;
  double* ipart = nullptr;
  long long ipart_cap = 0;
  double* pgram = nullptr;
  double* inner = nullptr;
  unsigned* tile_ctr = nullptr;  // dynamic tile-scheduler counters
  unsigned* tail_done = nullptr;  // fused tail arrival counter
  double* isvd_hand = nullptr;    // grid insertion handoff
  unsigned* isvd_gsync = nullptr; // grid insertion epoch / flag / arrivals
  double* upad[kMaxD] = {nullptr};  // pre-padded U_k images (proj_dmma smem layout)
  long long upad_R[kMaxD] = {0};    // rank the image was built for
  unsigned ctr_next = 0;
  Ctrl* ctrl = nullptr;
  Ctrl* ctrl_h = nullptr;
  // two-stage pipeline: projections of slice t+1 (stream st) overlap the
  // ISVD of slice t (stream si); per-parity decision slots and work buffers
  cudaStream_t si = nullptr;
  cudaStream_t sc = nullptr;     // host-to-device copies (overlap with compute)
  cudaStream_t s2 = nullptr;     // trailing modes + decision (overlap the next mode 0)
  // kNP slices in flight: projections of slice t+1 and t+2 may run while the
  // insertion of slice t does (per-slot buffers, decisions, events)
  static constexpr int kNP = 3;
  cudaEvent_t ev_m0[kNP] = {};
  cudaEvent_t ev_h2d[kNP] = {};
  bool ev_h2d_valid[kNP] = {};
  SliceCtl* slots = nullptr;     // device [kNP]
  SliceCtl* slots_h = nullptr;   // pinned mirror [kNP]
  double* pw[kNP][2] = {};
  long long pipe_elems = 0;
  cudaEvent_t ev_proj[kNP] = {}, ev_isvd[kNP] = {};
  bool ev_isvd_valid[kNP] = {};
  long long upd_count = 0;
  // Host-mapped channels (no copy calls on the per-slice path): decisions
  // published by decide_kernel, the projection input pointer per parity, and
  // the per-insertion record ring.
  SliceCtl* hslot = nullptr;              // mapped [kNP]
  SliceCtl* hslot_d = nullptr;
  unsigned long long* seq_dev = nullptr;  // device [kNP] decision counters
  unsigned long long seq_expect[kNP] = {};
  RecRing* ring_h = nullptr;              // mapped (published by the tail kernels)
  RecRing* ring_d = nullptr;              // device alias of ring_h
  RecRing* ring_dev = nullptr;            // device ring the insertion kernels write
  unsigned long long* ring_pub = nullptr; // device: records copied to ring_h
  RecRing ring_shadow{};                  // host copy of ring_dev at a forced drain
  unsigned long long rec_read = 0;        // records consumed by the host
  struct Pending {
    int mask;
    double wall;
  };
  std::vector<Pending> pending;  // issued insertions not yet drained, oldest first
  int r_exact = 0;               // streaming rank after the last drained insertion
  Ctrl last_ctrl{};              // control snapshot of the last drained insertion
  bool have_last_ctrl = false;
  int drift_pending = 0;
  std::vector<tsg_slice_metrics> metrics;

  // CUDA graphs of the per-slice fast path, one per buffer/pointer set
  struct GraphEntry {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;
    cudaGraphNode_t xnode = nullptr;  // kernel node reading the slice
    cudaKernelNodeParams kp{};
    ProjArgs pa;
  };
  cudaGraphNode_t cap_xnode = nullptr;
  unsigned long long* tail_clk = nullptr;  // TSG_TAIL_CLK debug stamps
  void dump_tail_clk() {
    if (!tail_clk) return;
    std::vector<unsigned long long> h(16 * kMaxGrid + 8);
    cudaMemcpy(h.data(), tail_clk, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ULL;
    int nb = 0;
    for (int b = 0; b < kMaxGrid; ++b)
      if (h[b * 16]) {
        t0 = std::min(t0, h[b * 16]);
        nb = b + 1;
      }
    for (int i = 0; i < 16; ++i) {
      unsigned long long lo = ~0ULL, hi = 0;
      for (int b = 0; b < nb; ++b)
        if (h[b * 16 + i] >= t0) {
          lo = std::min(lo, h[b * 16 + i]);
          hi = std::max(hi, h[b * 16 + i]);
        }
      if (hi) std::fprintf(stderr, "tail stamp %2d: min %8.2f us  max %8.2f us\n", i, (lo - t0) * 1e-3, (hi - t0) * 1e-3);
    }
    const unsigned long long* cs = h.data() + 16 * kMaxGrid;
    if (cs[0] && cs[3])
      std::fprintf(stderr, "tail last CTA (cycles): arrive->last %llu, reduce %llu, decide+publish %llu\n",
                   cs[1] - cs[0], cs[2] - cs[1], cs[3] - cs[2]);
  }
  std::map<std::vector<long long>, GraphEntry> graphs;
  bool use_graphs = std::getenv("TSG_NO_GRAPH") == nullptr;
  void clear_graphs() {
    if (graphs.empty()) return;
    sync();
    for (auto& kv : graphs) {
      cudaGraphExecDestroy(kv.second.exec);
      cudaGraphDestroy(kv.second.graph);
    }
    graphs.clear();
  }
  // Run `body(capturing)` on stream s_, from a cached graph when enabled;
  // `x` re-points the captured slice-reading kernel node.
  template <class F>
  void run(const std::vector<long long>& key, cudaStream_t s_, F&& body,
           const double* x = nullptr) {
    if (!use_graphs) {
      body(false);
      return;
    }
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      if (graphs.size() >= 64) clear_graphs();
      GraphEntry g;
      const long long l0 = g_launches;
      cap_xnode = nullptr;
      const auto cap_t0 = std::chrono::steady_clock::now();
      ck(cudaStreamBeginCapture(s_, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
      try {
        body(true);
      } catch (...) {
        cudaGraph_t tmp = nullptr;
        cudaStreamEndCapture(s_, &tmp);
        if (tmp) cudaGraphDestroy(tmp);
        throw;
      }
      ck(cudaStreamEndCapture(s_, &g.graph), "cudaStreamEndCapture");
      const cudaError_t e = cudaGraphInstantiate(&g.exec, g.graph, 0);
      if (e != cudaSuccess) cudaGraphDestroy(g.graph);
      ck(e, "cudaGraphInstantiate");
      g.launches = g_launches - l0;
      g_launches = l0;
      if (x && cap_xnode) {
        ck(cudaGraphKernelNodeGetParams(cap_xnode, &g.kp), "kernel node params");
        std::memcpy(&g.pa, g.kp.kernelParams[0], sizeof(ProjArgs));
        g.xnode = cap_xnode;
      } else if (x) {
        fail(TSG_EDEVICE, "graph capture: slice-reading kernel node not found");
      }
      it = graphs.emplace(key, g).first;
      if (growth_clk) {
        gclk[6] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - cap_t0).count();
        ++gcnt[6];
      }
    }
    GraphEntry& ge = it->second;
    if (ge.xnode && ge.pa.x != x) {
      ge.pa.x = x;
      void* args[1] = {&ge.pa};
      cudaKernelNodeParams kp = ge.kp;
      kp.kernelParams = args;
      kp.extra = nullptr;
      ck(cudaGraphExecKernelNodeSetParams(ge.exec, ge.xnode, &kp), "graph node update");
    }
    ck(cudaGraphLaunch(ge.exec, s_), "cudaGraphLaunch");
    g_launches += it->second.launches;
  }
  void wait_ev(cudaStream_t s_, cudaEvent_t e, bool cap) {
    ck(cudaStreamWaitEvent(s_, e, cap ? cudaEventWaitExternal : 0), "cudaStreamWaitEvent");
  }
  void record_ev(cudaEvent_t e, cudaStream_t s_, bool cap) {
    ck(cudaEventRecordWithFlags(e, s_, cap ? cudaEventRecordExternal : 0), "cudaEventRecord");
  }

  // Spin on a host-mapped flag; surfaces device faults and lost results.
  template <class Pred>
  void spin(Pred ready, const char* what) {
    for (unsigned it = 1;; ++it) {
      if (ready()) return;
      if ((it & 255) == 0) {
        const cudaError_t e1 = cudaStreamQuery(st), e2 = cudaStreamQuery(si), e3 = cudaStreamQuery(s2);
        if (e1 != cudaSuccess && e1 != cudaErrorNotReady) ck(e1, what);
        if (e2 != cudaSuccess && e2 != cudaErrorNotReady) ck(e2, what);
        if (e3 != cudaSuccess && e3 != cudaErrorNotReady) ck(e3, what);
        if (e1 == cudaSuccess && e2 == cudaSuccess && e3 == cudaSuccess) {
          std::atomic_thread_fence(std::memory_order_seq_cst);
          if (ready()) return;
          fail(TSG_EDEVICE, std::string(what) + ": device result was never published");
        }
      }
    }
  }
  unsigned long long rec_done() const {
    return *reinterpret_cast<const volatile unsigned long long*>(&ring_h->done);
  }
  // Wait for the decision of the last projection launched on parity `par`.
  SliceCtl wait_slot(int par) {
    const volatile unsigned long long* q = &hslot[par].seq;
    spin([&] { return *q == seq_expect[par]; }, "slice decision");
    std::atomic_thread_fence(std::memory_order_acquire);
    return hslot[par];
  }

  // phase profiling (TSG_PROFILE): per-slice event sets, reused every
  // kProfSets slices (by then the slice's work has long completed)
  static constexpr int kProfSets = 6;  // a multiple of kNP and of the 2-buffer ping-pong (bounded graph keys)
  cudaEvent_t pev[kProfSets][5] = {};
  bool pev_live[kProfSets] = {};
  int cur_q = -1;  // event set of the slice being enqueued (-1: none)
  double prof[6] = {0, 0, 0, 0, 0, 0};
  bool profiling() const { return flags & (TSG_PROFILE | TSG_PROFILE_MODE0); }
  // TSG_PROFILE_MODE0: only the mode-0 kernel's events (stream st); the
  // tail / insertion streams — the slice period's critical path — carry none
  bool prof_m0_only() const { return !(flags & TSG_PROFILE); }
  void ev_mark(int i, cudaStream_t s_, bool cap) {
    if (!profiling() || cur_q < 0) return;
    if (prof_m0_only() && i > 1) return;
    record_ev(pev[cur_q][i], s_, cap);
  }
  void resolve_prof(int q) {
    if (!pev_live[q]) return;
    pev_live[q] = false;
    if (prof_m0_only()) {
      ck(cudaEventSynchronize(pev[q][1]), "cudaEventSynchronize");
      float a = 0.f;
      cudaEventElapsedTime(&a, pev[q][0], pev[q][1]);
      prof[0] += 1;
      prof[1] += a;
      prof[5] += 1;
      return;
    }
    ck(cudaEventSynchronize(pev[q][4]), "cudaEventSynchronize");
    float a = 0.f, b = 0.f, c = 0.f, g = 0.f;
    cudaEventElapsedTime(&a, pev[q][0], pev[q][1]);
    cudaEventElapsedTime(&b, pev[q][1], pev[q][2]);
    cudaEventElapsedTime(&g, pev[q][2], pev[q][3]);
    cudaEventElapsedTime(&c, pev[q][3], pev[q][4]);
    prof[0] += 1;
    prof[1] += a;
    prof[2] += b;
    prof[3] += c;
    prof[4] += g;
    prof[5] += 1;
    if (tl_base && timeline.size() < 100000) {
      std::array<float, 5> row{};
      for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&row[i], tl_base, pev[q][i]);
      timeline.push_back(row);
    }
  }
  // per-slice timeline (TSG_PROFILE): event times of mode-0 start / end, tail
  // end (decision), insertion start / end, relative to the last profile reset
  cudaEvent_t tl_base = nullptr;
  std::vector<std::array<float, 5>> timeline;
  void reset_timeline() {
    if (!tl_base) ck(cudaEventCreate(&tl_base), "event");
    ck(cudaEventRecord(tl_base, st), "cudaEventRecord");
    ck(cudaEventSynchronize(tl_base), "cudaEventSynchronize");
    timeline.clear();
  }
  void resolve_all() {
    for (int q = 0; q < kProfSets; ++q) resolve_prof(q);
  }

  long long cur_bytes = 0, peak_bytes = 0;
  std::vector<std::pair<void*, long long>> allocs;
  long long launches_at_create = 0;

  // TSG_GROWTH_CLK=1: host wall-clock breakdown of the slow path (stderr)
  bool growth_clk = std::getenv("TSG_GROWTH_CLK") != nullptr;
  double gclk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long gcnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::chrono::steady_clock::time_point gt0;
  void gtic() {
    if (growth_clk) {
      sync();
      gt0 = std::chrono::steady_clock::now();
    }
  }
  void gtoc(int i) {
    if (!growth_clk) return;
    sync();
    gclk[i] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - gt0).count();
    ++gcnt[i];
    gt0 = std::chrono::steady_clock::now();
  }
  void gdump() {
    if (!growth_clk) return;
    static const char* nm[8] = {"rebuild-proj", "residual", "gram+eig", "finish(carried,pad,concat)",
                                "re-decide", "insert", "graph-capture", "slow-path total"};
    for (int i = 0; i < 8; ++i)
      if (gcnt[i])
        std::fprintf(stderr, "growth clk: %-28s x%5lld  %9.3f ms total  %8.3f ms avg\n", nm[i], gcnt[i],
                     gclk[i], gclk[i] / gcnt[i]);
  }

  // ------------------------------------------------------------ memory
  // Freed blocks up to kPoolBlockMax are kept (by capacity) and handed out
  // again: the growth path allocates the same temporaries for every basis
  // growth, and cudaMalloc / cudaFree cost 0.1-1 ms each and synchronise the
  // device. dfree() drains the engine's streams before it caches a block
  // (what cudaFree's implicit synchronisation guaranteed before).
  static constexpr long long kPoolBlockMax = 256LL << 20;
  static constexpr long long kPoolTotalMax = 2048LL << 20;
  std::multimap<long long, void*> pool;  // capacity in bytes -> block
  std::map<void*, long long> pool_cap;   // every live or pooled block: its capacity
  long long pool_bytes = 0;
  void pool_flush() {
    for (auto& kv : pool) {
      pool_cap.erase(kv.second);
      cudaFree(kv.second);
    }
    pool.clear();
    pool_bytes = 0;
  }
  double* dalloc(long long n_doubles) {
    if (n_doubles <= 0) n_doubles = 1;
    const long long bytes = n_doubles * (long long)sizeof(double);
    void* p = nullptr;
    auto it = pool.lower_bound(bytes);
    if (it != pool.end() && it->first <= bytes + bytes / 4 + 4096) {
      p = it->second;
      pool_bytes -= it->first;
      pool.erase(it);
    } else {
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e == cudaErrorMemoryAllocation && !pool.empty()) {
        cudaGetLastError();
        pool_flush();
        e = cudaMalloc(&p, bytes);
      }
      ck(e, "cudaMalloc");
      pool_cap[p] = bytes;
    }
    allocs.emplace_back(p, bytes);
    cur_bytes += bytes;
    peak_bytes = std::max(peak_bytes, cur_bytes);
    return static_cast<double*>(p);
  }
  // State buffers (Q, core, ...) are read up to a rank hint past the columns
  // ever written: pooled memory is not zero, so they start cleared.
  double* dalloc_zero(long long n_doubles) {
    double* p = dalloc(n_doubles);
    ck(cudaMemsetAsync(p, 0, sizeof(double) * (size_t)(n_doubles > 0 ? n_doubles : 1), st), "memset");
    return p;
  }
  void dfree(void* p) {
    if (!p) return;
    for (size_t i = 0; i < allocs.size(); ++i)
      if (allocs[i].first == p) {
        cur_bytes -= allocs[i].second;
        allocs.erase(allocs.begin() + i);
        break;
      }
    auto c = pool_cap.find(p);
    if (c != pool_cap.end() && c->second <= kPoolBlockMax &&
        pool_bytes + c->second <= kPoolTotalMax && st && si) {
      if (sc) cudaStreamSynchronize(sc);
      if (s2) cudaStreamSynchronize(s2);
      cudaStreamSynchronize(si);
      cudaStreamSynchronize(st);
      pool.emplace(c->second, p);
      pool_bytes += c->second;
      return;
    }
    if (c != pool_cap.end()) pool_cap.erase(c);
    cudaFree(p);
  }
  void free_all() {
    gdump();
    for (int i = 0; i < 8; ++i) gclk[i] = 0, gcnt[i] = 0;
    if (st) cudaStreamSynchronize(st);
    if (si) cudaStreamSynchronize(si);
    if (sc) cudaStreamSynchronize(sc);
    if (s2) cudaStreamSynchronize(s2);
    for (auto& a : allocs) cudaFree(a.first);
    allocs.clear();
    for (auto& kv : pool) cudaFree(kv.second);
    pool.clear();
    pool_cap.clear();
    pool_bytes = 0;
    cur_bytes = 0;
    for (auto& kv : graphs) {
      cudaGraphExecDestroy(kv.second.exec);
      cudaGraphDestroy(kv.second.graph);
    }
    graphs.clear();
    if (ctrl_h) cudaFreeHost(ctrl_h);
    if (slots_h) cudaFreeHost(slots_h);
    if (hslot) cudaFreeHost(hslot);
    if (ring_h) cudaFreeHost(ring_h);
    ctrl_h = nullptr;
    slots_h = nullptr;
    hslot = nullptr;
    ring_h = nullptr;
    ring_d = nullptr;
  }

  // all streams
  void sync() {
    if (sc) ck(cudaStreamSynchronize(sc), "cudaStreamSynchronize");
    if (s2) ck(cudaStreamSynchronize(s2), "cudaStreamSynchronize");
    ck(cudaStreamSynchronize(si), "cudaStreamSynchronize");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  }
  // TSG_DEBUG_SYNC=1: synchronise and check after each orchestration step.
  bool debug_sync = std::getenv("TSG_DEBUG_SYNC") != nullptr;
  void dbg(const char* where) {
    if (!debug_sync) return;
    ck(cudaStreamSynchronize(st), where);
    ck(cudaGetLastError(), where);
  }

  void pull_ctrl() {
    ck(cudaStreamSynchronize(si), "cudaStreamSynchronize");
    ck(cudaMemcpyAsync(ctrl_h, ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "ctrl D2H");
    sync();
    ck(cudaGetLastError(), "kernel");
    if (profiling()) resolve_all();
  }
  // this slice's decision record (projection stream only)
  void pull_slot(int par) {
    ck(cudaMemcpyAsync(slots_h + par, slots + par, sizeof(SliceCtl), cudaMemcpyDeviceToHost, st),
       "slot D2H");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    ck(cudaGetLastError(), "kernel");
  }
  void push_ctrl() {
    ck(cudaMemcpyAsync(ctrl, ctrl_h, sizeof(Ctrl), cudaMemcpyHostToDevice, st), "ctrl H2D");
  }

  long long n_rows() const { return prod(R, d - 1); }
  // partial-sum layout: per-mode pairs from the projection kernels, then the
  // fused tail's per-CTA partials
  static constexpr long long kTailPart = 2LL * kMaxGrid * (kMaxD + 1);
  static constexpr long long kPartStride = kTailPart + (long long)kMaxD * kMaxGrid + 64;
  DecideArgs last_da[kNP];  // partial layout of the last captured leading-mode pass
  bool use_tail = std::getenv("TSG_NO_TAIL") == nullptr;
  // Mode-0 slice loads carry an L2 evict-first hint: the insertion chain
  // (the slice period's bound) then keeps Q, core and the streaming factor in
  // L2 while the next slices stream through (C2: insertion 58 -> 52 us,
  // 15.5 k -> 17.1 k slices/s, same-box A/B). TSG_EVICT_FIRST=0 disables.
  bool evict_first = [] {
    const char* e = std::getenv("TSG_EVICT_FIRST");
    return e ? std::atoi(e) != 0 : true;
  }();
  // First mode handled by the fused tail kernel (d-1: none; the tail then
  // only decides): trailing modes with small inputs.
  int tail_start() const {
    int m = d - 1;
    for (int k = d - 2; k >= 1; --k) {
      long long in = 1;
      for (int j = 0; j < d - 1; ++j) in *= (j < k ? R[j] : N[j]);
      if (!tail_eligible(N[k], R[k]) || in > (2LL << 20)) break;
      m = k;
    }
    return m;
  }

  // --------------------------------------------------------- buffers
  // Partials for every mode plus one spare region, allocated once so that
  // pointers captured by enqueued kernels stay valid.
  void ensure_partial(long long n) {
    const long long need = std::max(n, kNP * kPartStride);
    if (need <= partial_cap) return;
    if (partial) sync();
    dfree(partial);
    partial_cap = need;
    partial = dalloc(partial_cap);
  }
  void ensure_isvd_buffers() {
    // capr must leave room for r+1 columns after the insertion
    const long long need_ip = (296LL * (capr + 1)) * 2 + 296 + 2 * 148 * 8 + 64;
    if (need_ip > ipart_cap) {
      dfree(ipart);
      ipart_cap = need_ip;
      ipart = dalloc(ipart_cap);
    }
  }
  void grow_capr(int new_capr) {
    // Q / core hold n x capr; left holds cap_rows x capr; sigma capr
    const long long n = n_rows();
    sync();
    double* nq = dalloc_zero(n * new_capr);
    double* nc = dalloc_zero(n * new_capr);
    double* nq2 = dalloc_zero(n * new_capr);
    double* nc2 = dalloc_zero(n * new_capr);
    ck(cudaMemcpyAsync(nq, Q, sizeof(double) * n * capr, cudaMemcpyDeviceToDevice, st), "grow");
    ck(cudaMemcpyAsync(nc, core, sizeof(double) * n * capr, cudaMemcpyDeviceToDevice, st), "grow");
    double* nl = dalloc(cap_rows * new_capr);
    double* nl2 = dalloc(cap_rows * new_capr);
    ck(cudaMemset2DAsync(nl, new_capr * sizeof(double), 0, new_capr * sizeof(double), cap_rows, st), "memset");
    ck(cudaMemcpy2DAsync(nl, new_capr * sizeof(double), left, capr * sizeof(double),
                         capr * sizeof(double), cap_rows, cudaMemcpyDeviceToDevice, st), "grow left");
    double* ns = dalloc(new_capr + 1);
    double* ns2 = dalloc(new_capr + 1);
    ck(cudaMemcpyAsync(ns, sigma, sizeof(double) * capr, cudaMemcpyDeviceToDevice, st), "grow");
    double* npg = dalloc((long long)new_capr * new_capr);
    double* nin = dalloc(isvd_inner_scratch(new_capr));
    sync();
    dfree(Q); dfree(Q2); dfree(core); dfree(core2); dfree(left); dfree(left2);
    dfree(sigma); dfree(sigma2); dfree(pgram); dfree(inner);
    Q = nq; Q2 = nq2; core = nc; core2 = nc2; left = nl; left2 = nl2;
    sigma = ns; sigma2 = ns2; pgram = npg; inner = nin;
    capr = new_capr;
    qcap = n * new_capr;
    ensure_isvd_buffers();
  }
  void grow_rows(long long need) {
    if (need <= cap_rows) return;
    long long nr = std::max(need, cap_rows * 2);
    double* nl = dalloc(nr * capr);
    double* nl2 = dalloc(nr * capr);
    ck(cudaMemsetAsync(nl, 0, sizeof(double) * nr * capr, st), "memset");
    ck(cudaMemcpyAsync(nl, left, sizeof(double) * cap_rows * capr, cudaMemcpyDeviceToDevice, st), "grow rows");
    sync();
    dfree(left); dfree(left2);
    left = nl; left2 = nl2;
    cap_rows = nr;
  }

  // ---------------------------------------------------- metrics drain
  // Retire published insertions in order (all issued ones when `force`).
  // Records reach the host two ways: published into the mapped ring by the
  // tail kernels of later slices (non-forced drains read that), or copied
  // from the device ring after a synchronisation (forced drains).
  void drain(bool force = true) {
    if (pending.empty()) return;
    const unsigned long long target = rec_read + pending.size();
    const RecRing* src = ring_h;
    unsigned long long done;
    if (force) {
      sync();
      ck(cudaMemcpy(&ring_shadow, ring_dev, sizeof(RecRing), cudaMemcpyDeviceToHost), "record copy");
      src = &ring_shadow;
      done = ring_shadow.done;
      if (done < target) fail(TSG_EDEVICE, "insertion record: device result was never published");
    } else {
      done = rec_done();
      std::atomic_thread_fence(std::memory_order_acquire);
    }
    while (rec_read < done && !pending.empty()) {
      const int pos = (int)(rec_read % kRecRing);
      const Metrics m = src->rec[pos];
      const Ctrl cs = src->ctrl[pos];
      const Pending p = pending.front();
      tsg_slice_metrics o;
      std::memset(&o, 0, sizeof o);
      o.slice_index = m.slice_index;
      for (int k = 0; k < d; ++k) o.ranks[k] = m.ranks[k];
      o.slice_norm = m.slice_norm;
      o.projected_norm = m.projected_norm;
      o.error_estimate = m.error_estimate;
      for (int k = 0; k + 1 < d; ++k) o.mode_residuals[k] = m.mode_residuals[k];
      o.expanded_mask = p.mask;
      o.peak_bytes = peak_bytes;
      o.wall_ms = p.wall;
      o.trunc_margin = m.trunc_margin;
      o.jacobi_sweeps = m.sweeps;
      metrics.push_back(o);
      r_exact = cs.r;
      last_ctrl = cs;
      have_last_ctrl = true;
      if (cs.status != 0) drift_pending = cs.status;
      ++rec_read;
      pending.erase(pending.begin());
    }
  }
  // Room in the record ring for one more insertion.
  void reserve_record() {
    if (pending.size() + 2 >= (size_t)kRecRing) drain(true);
  }

  void check_status() {
    if (drift_pending) {
      const int code = drift_pending;
      drift_pending = 0;
      if (code == 2)
        fail(TSG_EDRIFT,
             "streaming state invariant violated: core no longer matches the ISVD factorization");
      fail(TSG_EOTHER, "device numerical failure");
    }
    if (ctrl_h->status == 2)
      fail(TSG_EDRIFT,
           "streaming state invariant violated: core no longer matches the ISVD factorization");
    if (ctrl_h->status != 0) fail(TSG_EOTHER, "device numerical failure");
  }

  // ---------------------------------------------------- mode subspace
  struct Sub {
    double* basis = nullptr;  // rows x rank (ld rows)
    double* evals = nullptr;  // >= rows entries
    long long rank = 0;
    double disc = 0.0;
    std::vector<double*> owned;
  };
  void release(Sub& s) {
    for (double* p : s.owned) dfree(p);
    s.owned.clear();
  }

  // Gram route of mode_subspace from a formed Gram matrix (sthosvd.cpp:61-75):
  // eigensolve, truncation against delta, basis = leading eigenvectors. The
  // sharded growth calls it on the all-reduced sum of the ranks' partial Grams.
  void subspace_from_gram(Sub& s, const double* g, long long rows, double delta,
                          long long* rk_d = nullptr) {
    if (!rk_d) {
      rk_d = reinterpret_cast<long long*>(dalloc(2));
      s.owned.push_back(reinterpret_cast<double*>(rk_d));
    }
    double* disc_d = reinterpret_cast<double*>(rk_d) + 1;
    double* ev = dalloc(rows);
    s.owned.push_back(ev);
    if (tri_eig_applicable((int)rows)) {
      // n >= 96: tridiagonal route — all eigenvalues for the truncation rule,
      // then only the retained eigenvectors (tridiag_eig.cu)
      const int max_rank = tri_eig_max_rank((int)rows);
      double* twork = dalloc(tri_eig_work_doubles((int)rows, max_rank));
      s.owned.push_back(twork);
      if (launch_tri_eigvals(g, (int)rows, ev, twork, st)) {
        launch_truncate(ev, (int)rows, delta, 0, rk_d, disc_d, st);
        long long hr[2];
        ck(cudaMemcpyAsync(hr, rk_d, 16, cudaMemcpyDeviceToHost, st), "rank D2H");
        sync();
        ck(cudaGetLastError(), "mode_subspace");
        if (hr[0] <= max_rank) {
          s.rank = hr[0];
          std::memcpy(&s.disc, &hr[1], 8);
          double* vec = dalloc(rows * std::max(s.rank, 1LL));
          s.owned.push_back(vec);
          launch_tri_eigvecs((int)rows, (int)s.rank, twork, vec, st);
          // callers may read the basis from another stream: complete it here
          sync();
          ck(cudaGetLastError(), "mode_subspace eigenvectors");
          s.basis = vec;
          s.evals = ev;
          return;
        }
      }
      // (no cooperative launch, or most of the spectrum retained: Jacobi)
    }
    double* work = dalloc(3 * rows * rows + 512);
    double* vec = dalloc(rows * rows);
    s.owned.insert(s.owned.end(), {work, vec});
    launch_sym_eig(g, (int)rows, ev, vec, work, nullptr, st);
    launch_truncate(ev, (int)rows, delta, 0, rk_d, disc_d, st);
    long long hr[2];
    ck(cudaMemcpyAsync(hr, rk_d, 16, cudaMemcpyDeviceToHost, st), "rank D2H");
    sync();
    ck(cudaGetLastError(), "mode_subspace");
    s.rank = hr[0];
    std::memcpy(&s.disc, &hr[1], 8);
    s.basis = vec;
    s.evals = ev;
  }

  // mode_subspace (sthosvd.cpp:39-92) on a device tensor.
  Sub mode_subspace(const double* t, const long long* dims, int order, int mode, double delta) {
    Sub s;
    const long long rows = dims[mode];
    const long long size = prod(dims, order);
    const long long cols = rows == 0 ? 0 : size / rows;
    if (rows <= 0) fail(TSG_EINVAL, "mode_subspace: empty mode");
    ModeView v{prod(dims, mode), rows, prod(dims + mode + 1, order - mode - 1)};
    const double* A = t;
    if (mode != 0) {
      double* a = dalloc(size);
      s.owned.push_back(a);
      launch_unfold(t, v, a, st);
      A = a;
    }
    long long* rk_d = reinterpret_cast<long long*>(dalloc(2));
    s.owned.push_back(reinterpret_cast<double*>(rk_d));
    double* disc_d = reinterpret_cast<double*>(rk_d) + 1;
    if (rows <= cols) {
      double* g = dalloc(rows * rows);
      const int splits = gram_splits((int)rows, cols);
      double* part = dalloc((long long)splits * rows * rows);
      s.owned.insert(s.owned.end(), {g, part});
      launch_gram(A, (int)rows, cols, g, part, st);
      subspace_from_gram(s, g, rows, delta, rk_d);
      return s;
    }
    // thin route
    double* g = dalloc(cols * cols);
    double* work = dalloc(3 * cols * cols + 512);
    double* vec = dalloc(cols * cols);
    double* ev = dalloc(rows);
    s.owned.insert(s.owned.end(), {g, work, vec, ev});
    ck(cudaMemsetAsync(ev, 0, sizeof(double) * rows, st), "memset");
    launch_gram_t(A, rows, (int)cols, g, st);
    launch_sym_eig(g, (int)cols, ev, vec, work, nullptr, st);
    launch_truncate(ev, (int)cols, delta, 1, rk_d, disc_d, st);
    long long hr[2];
    ck(cudaMemcpyAsync(hr, rk_d, 16, cudaMemcpyDeviceToHost, st), "rank D2H");
    sync();
    ck(cudaGetLastError(), "mode_subspace");
    s.rank = hr[0];
    std::memcpy(&s.disc, &hr[1], 8);
    double* basis = dalloc(rows * std::max(s.rank, 1LL));
    s.owned.push_back(basis);
    launch_gemm_nn(A, rows, vec, cols, basis, rows, rows, (int)s.rank, (int)cols, st);
    launch_scale_cols_invsqrt(basis, rows, rows, (int)s.rank, ev, st);
    launch_mgs(basis, rows, rows, (int)s.rank, st);
    // callers copy the basis out on another stream: complete it here
    sync();
    ck(cudaGetLastError(), "mode_subspace");
    s.basis = basis;
    s.evals = ev;
    return s;
  }

  // ------------------------------------------------------- projection
  // Projection of y (dims yd, order d-1) along `mode`: P into out,
  // partials into `part`; returns partial count.
  // Pre-padded U image and tile counters (allocated outside graph capture).
  void prep_proj(int mode) {
    if (upad_R[mode] != R[mode]) {
      dfree(upad[mode]);
      upad[mode] = dalloc(upad_size(N[mode], (int)R[mode]));
      launch_pad_u(U[mode], N[mode], (int)R[mode], upad[mode], st);
      upad_R[mode] = R[mode];
    }
    if (!tile_ctr) tile_ctr = reinterpret_cast<unsigned*>(dalloc(kMaxD * 2));
    if (!tail_done) {
      tail_done = reinterpret_cast<unsigned*>(dalloc((kNP + 1) / 2));
      ck(cudaMemsetAsync(tail_done, 0, 8 * ((kNP + 1) / 2), st), "memset");
      ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    }
  }
  int project(const double* y, const long long* yd, int mode, double* out, double* part,
              double* e = nullptr) {
    ProjArgs a;
    a.x = y;
    a.v = ModeView{prod(yd, mode), yd[mode], prod(yd + mode + 1, d - 2 - mode)};
    a.u = U[mode];
    a.R = (int)R[mode];
    a.p = out;
    a.e = e;
    a.partial = part;
    a.residual = 1;
    a.stream_in = (mode == 0 && y != w0 && y != w1 && y != w2) ? (evict_first ? 2 : 1) : 0;
    prep_proj(mode);
    a.upad = upad[mode];
    if (shard_world > 0) {
      // sharded: static tile order, so the partial sums (and every decision
      // and ledger derived from them) are bitwise identical on all ranks
      a.tile_counter = nullptr;
    } else {
      a.tile_counter = tile_ctr + (ctr_next++ % (kMaxD * 4));
      ck(cudaMemsetAsync(a.tile_counter, 0, sizeof(unsigned), st), "memset");
    }
    return launch_project(a, st);
  }

  // Grow U_k by the residual's dominant directions (streaming.cpp:142-151).
  // y: mode input tensor (dims yd); p: its projection; result written to
  // `dst` (concat of p and the carried coefficients), yd updated.
  void expand_mode(const double* y, long long* yd, int mode, double delta, double* p,
                   double* dst) {
    gtic();
    expand_residual(y, yd, mode, p);
    gtoc(1);
    Sub s = mode_subspace(ebuf, yd, d - 1, mode, delta);
    dbg("expand: mode_subspace");
    gtoc(2);
    expand_finish(yd, mode, s, p, dst);
    gtoc(3);
  }
  // First half: P = U^T Y into p, residual E = Y - U P into ebuf.
  void expand_residual(const double* y, const long long* yd, int mode, double* p) {
    if (!ebuf) ebuf = dalloc(slice_elems);
    if (!kbuf) kbuf = dalloc(slice_elems);
    dbg("expand: entry");
    project(y, yd, mode, p, partial + 2LL * kMaxGrid * kMaxD, ebuf);
    dbg("expand: residual");
  }
  // Second half, from the subspace W of the residual: carried = W^T E,
  // U <- [U W], core / Q padded, ledger, dst = concat(P, carried). On a
  // sharded rank y / p / ebuf are the local parts and the state updates run
  // identically on every rank.
  void expand_finish(long long* yd, int mode, Sub& s, double* p, double* dst) {
    ModeView v{prod(yd, mode), yd[mode], prod(yd + mode + 1, d - 2 - mode)};
    const long long g = s.rank;
    if (R[mode] + g > N[mode]) fail(TSG_EOTHER, "expansion exceeds the mode size");
    // carried = W^T E (streaming.cpp:145)
    ProjArgs a;
    a.x = ebuf;
    a.v = v;
    a.u = s.basis;
    a.R = (int)g;
    a.p = kbuf;
    a.e = nullptr;
    a.partial = nullptr;
    a.residual = 0;
    launch_project(a, st);
    dbg("expand: carried");
    // U_k <- [U_k W] (old columns untouched)
    {
      const cudaError_t e = cudaMemcpyAsync(U[mode] + R[mode] * N[mode], s.basis,
                                            sizeof(double) * N[mode] * g, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "hcat: %s (mode %d R %lld N %lld g %lld basis %p U %p rows %lld)",
                      cudaGetErrorString(e), mode, R[mode], N[mode], g, (void*)s.basis,
                      (void*)U[mode], yd[mode]);
        fail(TSG_EDEVICE, buf);
      }
    }
    // pad core and v (= Q) along mode (tensor.cpp:168-184)
    long long cd[kMaxD];
    for (int k = 0; k + 1 < d; ++k) cd[k] = R[k];
    const int r = ctrl_h->r;
    cd[d - 1] = r;
    ModeView cv{prod(cd, mode), R[mode], prod(cd + mode + 1, d - 1 - mode)};
    const long long n_new = n_rows() / R[mode] * (R[mode] + g);
    const long long new_qcap = n_new * capr;
    // The out-of-place pad lands in the idle ping-pong buffers when they are
    // large enough (no allocation per growth); otherwise all four buffers are
    // re-allocated with room for further growth.
    const bool in_spare = new_qcap <= qcap;
    const long long alloc_qcap = in_spare ? qcap : 2 * new_qcap;
    double* nq = in_spare ? Q2 : dalloc_zero(alloc_qcap);
    double* nc = in_spare ? core2 : dalloc_zero(alloc_qcap);
    launch_pad(Q, cv, g, nq, st);
    launch_pad(core, cv, g, nc, st);
    double* nq2 = in_spare ? Q : dalloc_zero(alloc_qcap);
    double* nc2 = in_spare ? core : dalloc_zero(alloc_qcap);
    // ledger (streaming.cpp:150)
    double* dd = dalloc(1);
    ck(cudaMemcpyAsync(dd, &s.disc, 8, cudaMemcpyHostToDevice, st), "disc");
    launch_ledger_add_nonstream(ctrl, dd, st);
    // y <- concat_k(P, carried)
    launch_concat(p, kbuf, v.left, R[mode], g, v.right, dst, st);
    dbg("expand: concat");
    sync();
    dfree(dd);
    if (!in_spare) {
      dfree(Q); dfree(Q2); dfree(core); dfree(core2);
    }
    Q = nq; Q2 = nq2; core = nc; core2 = nc2;
    qcap = alloc_qcap;
    if (e_alloc_n() < n_new) {
      dfree(evec);
      evec = dalloc(2 * n_new);
      evec_n = 2 * n_new;
    }
    release(s);
    R[mode] += g;
    yd[mode] = R[mode];
  }
  long long evec_n = 0;
  long long e_alloc_n() const { return evec_n; }

  // ---------------------------------------------------------- update
  // A work buffer that is none of `avoid` (three rotate; slices never
  // overwrite the caller's input).
  double* pick(const double* a0, const double* a1) {
    for (double* b : {w0, w1, w2})
      if (b != a0 && b != a1) return b;
    return nullptr;
  }

  // Work buffers of the pipelined path: two per slice parity, sized for the
  // largest projected tensor (the output of mode 0).
  void ensure_pipe() {
    long long need = 1;
    for (int k = 0; k + 1 < d; ++k) need *= (k == 0 ? R[0] : N[k]);
    if (need <= pipe_elems) return;
    sync();
    // room for the leading basis to grow by half again (capped at its mode
    // size) before the next re-allocation
    long long room = need / std::max(1LL, R[0]) * std::min(N[0], R[0] + std::max(8LL, R[0] / 2));
    room = std::max(room, need);
    for (auto& set : pw)
      for (auto& b : set) {
        dfree(b);
        b = dalloc(room);
      }
    pipe_elems = room;
  }

  // Enqueue the ISVD insertion + core rotation for the slice whose projected
  // tensor is `b` and whose decisions are in slot `par`, on stream `s_`
  // (the ISVD stream, from a cached graph, on the fast path; `st` eagerly
  // after a slow path).
  void enqueue_isvd(const double* b, int par, int mask, cudaStream_t s_, bool commit,
                    std::chrono::steady_clock::time_point t0) {
    drain(false);
    int r_ub = r_exact + (int)pending.size();
    if (r_ub + 1 > capr) {
      sync();
      drain(true);
      r_ub = r_exact;
      if (r_ub + 1 > capr) grow_capr(std::max(capr + 16, (r_ub + 1 + 7) / 8 * 8 + 8));
    }
    if (n_d + 1 > cap_rows) {
      sync();
      grow_rows(n_d + 1);
    }
    const long long n = n_rows();
    if (evec_n < n) {
      sync();
      dfree(evec);
      evec = dalloc(n);
      evec_n = n;
    }
    reserve_record();
    IsvdBufs B;
    std::memset(&B, 0, sizeof B);
    B.ctrl = ctrl;
    B.slot = slots + par;
    B.b = b;
    B.q = Q;
    B.qn = Q2;
    B.c = core;
    B.cn = core2;
    B.e = evec;
    B.sigma = sigma;
    B.sigma_new = sigma2;
    B.left = left;
    B.left_new = left2;
    B.pgram = pgram;
    B.inner = inner;
    B.partial = ipart;
    B.hand = isvd_hand;
    B.gsync = isvd_gsync;
    B.ring = ring_dev;
    B.n = n;
    B.cap_rows = cap_rows;
    B.capr = capr;
    B.order = d;
    static const int rpad = std::getenv("TSG_RHINT_PAD") ? std::atoi(std::getenv("TSG_RHINT_PAD")) : 0;
    // The hint is an upper bound of the rank the kernel will find (it selects
    // the register-bound template and the Q columns staged). On the graph
    // path it is part of the key: the count of undrained insertions wobbles
    // between 1 and kNP with the record ring's publication lag, which made
    // new (slot, hint) pairs — each a 1-3 ms capture — appear long after the
    // warm-up. The pipelined engine therefore rounds it up to the steady
    // bound r + kNP + 1 (arithmetic is RMAX-invariant, see DESIGN).
    int r_key = r_ub;
    if (s_ == si && (flags & TSG_ASYNC)) {
      r_key = std::max(r_ub, r_exact + kNP + 1);
      // ... and up to the next template bound, so that a streaming rank that
      // creeps up one by one (config 5: 8 -> 36) re-captures the insertion
      // graphs at ~10 bounds instead of at every rank
      static const int bounds[] = {8, 12, 14, 16, 20, 24, 31, 39, 47, 63, 95, 127};
      for (int bnd : bounds)
        if (r_key <= bnd) {
          r_key = bnd;
          break;
        }
    }
    B.r_hint = std::min(r_key + rpad, capr - 1);
    B.commit_modes = commit ? d - 1 : 0;  // ledger commit fused into the insertion
    for (int k = 0; k + 1 < d; ++k) B.spatial_ranks[k] = R[k];
    const bool graph = (s_ == si);
    const int q = mask == 0 ? cur_q : -1;
    const bool reorth = reorth_every > 0 && (insertions_host + 1) % reorth_every == 0;
    auto body = [&](bool cap) {
      const int saved = cur_q;
      cur_q = q;
      if (s_ != st) wait_ev(s_, ev_proj[par], cap);
      ev_mark(3, s_, cap);
      launch_isvd(B, s_);
      if (reorth) launch_reorth(ctrl, B.left_new, capr, B.qn, n, s_);
      ev_mark(4, s_, cap);
      record_ev(ev_isvd[par], s_, cap);
      cur_q = saved;
    };
    if (graph) {
      std::vector<long long> key = {1, par, commit, (long long)(uintptr_t)b,
                                    (long long)(uintptr_t)Q, (long long)(uintptr_t)Q2,
                                    (long long)(uintptr_t)core, (long long)(uintptr_t)core2,
                                    (long long)(uintptr_t)sigma, (long long)(uintptr_t)sigma2,
                                    (long long)(uintptr_t)left, (long long)(uintptr_t)left2,
                                    (long long)(uintptr_t)evec, (long long)(uintptr_t)pgram,
                                    (long long)(uintptr_t)inner, (long long)(uintptr_t)ipart,
                                    (long long)(uintptr_t)isvd_hand, (long long)(uintptr_t)isvd_gsync,
                                    n, cap_rows, capr, B.r_hint, d, prof_m0_only() ? -1 : q,
                                    reorth ? 1 : 0};
      for (int k = 0; k + 1 < d; ++k) key.push_back(R[k]);
      run(key, s_, body);
    } else {
      body(false);
    }
    if (q >= 0 && profiling()) pev_live[q] = true;
    ev_isvd_valid[par] = true;
    std::swap(Q, Q2);
    std::swap(core, core2);
    std::swap(sigma, sigma2);
    std::swap(left, left2);
    ++n_d;
    ++insertions_host;
    pending.push_back(Pending{mask, std::chrono::duration<double, std::milli>(
                                        std::chrono::steady_clock::now() - t0).count()});
  }

  // A slice whose projections are enqueued but whose decision (basis growth,
  // zero slice) has not been acted on yet.
  struct Pend {
    int par = 0;
    int q = -1;                 // profiling event set
    const double* y = nullptr;  // device input (caller buffer or staging)
    const double* b = nullptr;  // projected tensor
    std::chrono::steady_clock::time_point t0;
  };
  // Slices whose projections are enqueued and whose decisions are not acted
  // on yet, oldest first. The pipelined engine keeps kDefer of them: the host
  // enqueues the projections of slice t+2 BEFORE it waits for the decision of
  // slice t, so the projection stream always holds queued work (with one
  // deferred slice the period was (decision latency + host turnaround) / 2).
  static constexpr int kDefer = kNP - 1;
  std::vector<Pend> deferred;
  // Act on the oldest deferred slices until at most `keep` remain; when a slow
  // path ran (bases may have grown), the younger ones are projected again.
  void settle(size_t keep) {
    while (deferred.size() > keep) {
      Pend p = deferred.front();
      deferred.erase(deferred.begin());
      if (complete(p))
        for (Pend& q : deferred) enqueue_proj(q.y, q);
    }
  }
  double* stage[kNP] = {};  // host-slice staging per slot

  // Mode projections + decision of one slice on `st` (a cached graph: the
  // input pointer is read by the mode-0 kernel from mapped memory; the
  // decision is published to mapped memory with a sequence number).
  void enqueue_proj(const double* y, Pend& p) {
    const int par = p.par;
    ensure_pipe();
    ensure_partial(1);
    for (int k = 0; k + 1 < d; ++k) prep_proj(k);
    if (p.q >= 0 && profiling()) resolve_prof(p.q);
    const int m0 = use_tail ? tail_start() : d - 1;
    double* part = partial + par * kPartStride;  // per parity: slices t, t+1 overlap
    // leading (large) modes on st; with the fused tail, the trailing modes and
    // the decision run on s2 so that they overlap the next slice's mode 0
    auto mbody = [&](bool cap) {
      const int saved = cur_q;
      cur_q = p.q;
      wait_ev(st, ev_isvd[par], cap);  // buffers + slot last read by the insertion kNP slices ago
      wait_ev(st, ev_h2d[par], cap);   // staged host slice
      long long yd[kMaxD];
      for (int k = 0; k + 1 < d; ++k) yd[k] = N[k];
      DecideArgs& da = last_da[par];
      std::memset(&da, 0, sizeof da);
      da.slot = slots + par;
      da.host_slot = hslot_d + par;
      da.seq_counter = seq_dev + par;
      da.ring_dev = ring_dev;
      da.ring_host = ring_d;
      da.ring_pub = ring_pub;
      da.nmodes = d - 1;
      da.tau = tau;
      da.order = d;
      da.partial = part;
      const double* cur = y;
      int off = 0;
      for (int k = 0; k < m0; ++k) {
        double* out = pw[par][k & 1];
        da.off[k] = off;
        if (k == 0) ev_mark(0, st, cap);
        da.cnt[k] = project(cur, yd, k, out, part + off);
        if (k == 0 && cap) {
          // the mode-0 kernel node: its input pointer is re-pointed per launch
          cudaStreamCaptureStatus cs;
          const cudaGraphNode_t* deps = nullptr;
          size_t nd = 0;
          ck(cudaStreamGetCaptureInfo(st, &cs, nullptr, nullptr, &deps, &nd), "capture info");
          cap_xnode = nd == 1 ? deps[0] : nullptr;
        }
        if (k == 0) ev_mark(1, st, cap);
        off += 2 * da.cnt[k];
        yd[k] = R[k];
        cur = out;
      }
      da.first_mode = 0;
      if (!use_tail) {
        launch_decide(da, st);
        ev_mark(2, st, cap);
        record_ev(ev_proj[par], st, cap);
      } else {
        record_ev(ev_m0[par], st, cap);
      }
      cur_q = saved;
    };
    auto tbody = [&](bool cap) {
      const int saved = cur_q;
      cur_q = p.q;
      wait_ev(s2, ev_m0[par], cap);
      TailArgs ta;
      std::memset(&ta, 0, sizeof ta);
      ta.x = pw[par][(m0 - 1) & 1];
      for (int k = m0; k + 1 < d; ++k) {
        ta.out[k] = pw[par][k & 1];
        ta.u[k] = U[k];
        ta.N[k] = N[k];
        ta.R[k] = (int)R[k];
        ta.left[k] = prod(R, k);
        ta.right[k] = prod(N + k + 1, d - 2 - k);
      }
      ta.m0 = m0;
      ta.m1 = d - 1;
      ta.part = part + kTailPart;
      ta.done = tail_done + par;
      ta.da = last_da[par];
      if (std::getenv("TSG_TAIL_CLK")) {
        if (!tail_clk) {
          tail_clk = reinterpret_cast<unsigned long long*>(dalloc(16 * kMaxGrid + 8));
          cudaMemset(tail_clk, 0, (16 * kMaxGrid + 8) * 8);
        }
        ta.clk = tail_clk;
      }
      if (launch_tail(ta, s2) < 0) fail(TSG_EDEVICE, "fused tail kernel launch failed");
      ev_mark(2, s2, cap);
      record_ev(ev_proj[par], s2, cap);
      cur_q = saved;
    };
    std::vector<long long> key = {0, par, d, m0, (long long)(uintptr_t)pw[par][0],
                                  (long long)(uintptr_t)pw[par][1], (long long)(uintptr_t)partial,
                                  (long long)(uintptr_t)tile_ctr, profiling() ? p.q : -1};
    for (int k = 0; k + 1 < d; ++k) {
      key.push_back((long long)(uintptr_t)U[k]);
      key.push_back((long long)(uintptr_t)upad[k]);
      key.push_back(R[k]);
      key.push_back(N[k]);
    }
    ++seq_expect[par];
    run(key, st, mbody, y);
    if (use_tail) {
      key[0] = 2;
      run(key, s2, tbody);
    }
    p.y = y;
    p.b = d >= 2 ? pw[par][(d - 2) & 1] : nullptr;
  }

  // Act on a slice's decision. Returns true when the slow path ran (the
  // non-streaming bases may have grown, so later projections must be redone).
  bool complete(Pend& p) {
    const SliceCtl sc = wait_slot(p.par);
    if (sc.zero_slice || sc.expand_mode >= 0) {
      if (p.q >= 0) pev_live[p.q] = false;
      update_slow(p.y, p.par, p.t0);
      return true;
    }
    const int saved = cur_q;
    cur_q = p.q;
    enqueue_isvd(p.b, p.par, 0, si, true, p.t0);
    cur_q = saved;
    return false;
  }

  void update(const double* y_in, int mem_kind) {
    if (!initialized) fail(TSG_EINVAL, "stream_update: state not initialised");
    Pend cur;
    cur.t0 = std::chrono::steady_clock::now();
    cur.q = profiling() ? (int)(upd_count % kProfSets) : -1;
    cur.par = (int)(upd_count++ % kNP);
    const double* y = y_in;
    const bool misaligned = (reinterpret_cast<uintptr_t>(y_in) & 15) != 0;
    if (mem_kind == TSG_MEM_HOST || misaligned) {
      // copy engine stream: the H2D of slice t overlaps compute of slice t-1;
      // staging[par] is free once the projections that read it are done
      if (!stage[cur.par]) stage[cur.par] = dalloc(slice_elems);
      // staging[par] is free once the mode-0 pass that read it is done
      ck(cudaStreamWaitEvent(sc, use_tail ? ev_m0[cur.par] : ev_proj[cur.par], 0),
         "cudaStreamWaitEvent");
      ck(cudaMemcpyAsync(stage[cur.par], y_in, sizeof(double) * slice_elems,
                         mem_kind == TSG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                         sc), "slice copy");
      ck(cudaEventRecord(ev_h2d[cur.par], sc), "cudaEventRecord");
      ev_h2d_valid[cur.par] = true;
      y = stage[cur.par];
      // the caller's previous host slice has been consumed once its copy ends
      const int pp = (cur.par + kNP - 1) % kNP;
      if (ev_h2d_valid[pp]) ck(cudaEventSynchronize(ev_h2d[pp]), "h2d sync");
    }
    // enqueue this slice first, then settle the previous one: the projection
    // stream never waits on the host
    enqueue_proj(y, cur);
    deferred.push_back(cur);
    if (flags & TSG_ASYNC) {
      settle(kDefer);
      drain(false);
    } else {
      settle(0);
      drain(true);
      if (have_last_ctrl && pending.empty()) {
        *ctrl_h = last_ctrl;  // the device block as the last insertion left it
        ck(cudaGetLastError(), "kernel");
      } else {
        pull_ctrl();
      }
      check_status();
    }
  }

  // Zero slice or basis growth: serialise both streams and run the
  // host-orchestrated path (streaming.cpp:171-185, 140-151).
  void update_slow(const double* y, int par, std::chrono::steady_clock::time_point t0) {
    sync();
    const auto s0 = std::chrono::steady_clock::now();
    drain(true);
    pull_ctrl();
    const SliceCtl sc = hslot[par];
    if (sc.zero_slice) {
      zero_slice_path(par, t0);
      return;
    }
    long long yd[kMaxD];
    for (int k = 0; k + 1 < d; ++k) yd[k] = N[k];
    run_growth(y, yd, 0, sc.expand_mode, sc.delta, par, t0);
    if (growth_clk) {
      sync();
      gclk[7] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s0).count();
      ++gcnt[7];
    }
  }

  // streaming.cpp:171-185: a zero left row and a metrics record.
  void zero_slice_path(int par, std::chrono::steady_clock::time_point t0) {
    {
      launch_commit_modes(ctrl, slots + par, 0, 0, 1, st);
      if (n_d + 1 > cap_rows) grow_rows(n_d + 1);
      reserve_record();
      long long sp[kMaxD] = {0};
      for (int k = 0; k + 1 < d; ++k) sp[k] = R[k];
      launch_zero_slice(ctrl, slots + par, left, capr, ring_dev, d, sp, st);
      ck(cudaEventRecord(ev_isvd[par], st), "cudaEventRecord");
      ev_isvd_valid[par] = true;
      ++n_d;
      pending.push_back(Pending{0, std::chrono::duration<double, std::milli>(
                                       std::chrono::steady_clock::now() - t0).count()});
    }
  }

  // Basis growth (streaming.cpp:140-151) starting from `base_in`, the input
  // of mode m0_in with dims yd_in: rebuild the input of mode `em` (the first
  // mode whose residual exceeds delta), grow it, continue with the grown
  // tensor, then insert. Slot `par` holds the slice's decision record.
  // `commit_lo` / `with_total` / `mask0`: the sharded engine enters here after
  // local modes [0, commit_lo) were committed (and some of them grown) already.
  void run_growth(const double* base_in, const long long* yd_in, int m0_in, int em, double delta,
                  int par, std::chrono::steady_clock::time_point t0, int commit_lo = 0,
                  int with_total = 1, int mask0 = 0) {
    long long yd[kMaxD];
    for (int k = 0; k + 1 < d; ++k) yd[k] = yd_in[k];
    DecideArgs da;
    std::memset(&da, 0, sizeof da);
    da.slot = slots + par;
    da.nmodes = d - 1;
    da.tau = tau;
    da.order = d;
    da.partial = partial;
    const double* base = base_in;
    int m0 = m0_in, mask = mask0;
    launch_commit_modes(ctrl, slots + par, commit_lo, em, with_total, st);
    const double* b = nullptr;
    while (true) {
      // rebuild the input of mode em from `base` (same kernels, same data)
      gtic();
      const double* cur = base;
      for (int k = m0; k < em; ++k) {
        double* out = pick(cur, base);
        project(cur, yd, k, out, partial + 2LL * kMaxGrid * kMaxD);
        yd[k] = R[k];
        cur = out;
      }
      gtoc(0);
      double* pbuf = pick(cur, base);
      double* dst = pick(cur, pbuf);
      expand_mode(cur, yd, em, delta, pbuf, dst);
      mask |= 1 << em;
      base = dst;
      m0 = em + 1;
      if (m0 == d - 1) {
        b = base;
        break;
      }
      // speculatively project the remaining modes, decide once
      long long ydk[kMaxD];
      std::memcpy(ydk, yd, sizeof yd);
      const double* c2 = base;
      int off = 0;
      for (int k = m0; k + 1 < d; ++k) {
        double* out = pick(c2, base);
        da.off[k] = off;
        da.cnt[k] = project(c2, ydk, k, out, partial + off);
        off += 2 * da.cnt[k];
        ydk[k] = R[k];
        c2 = out;
      }
      da.first_mode = m0;
      launch_decide(da, st);
      pull_slot(par);
      gtoc(4);
      em = slots_h[par].expand_mode;
      if (em < 0) {
        launch_commit_modes(ctrl, slots + par, m0, d - 1, 0, st);
        b = c2;
        break;
      }
      launch_commit_modes(ctrl, slots + par, m0, em, 0, st);
    }
    pull_ctrl();
    r_exact = ctrl_h->r;
    gtic();
    ensure_pipe();
    enqueue_isvd(b, par, mask, st, false, t0);
    ck(cudaEventRecord(ev_proj[par], st), "cudaEventRecord");
    gtoc(5);
  }

  // ------------------------------------------------------ sharded update
  // SURVEY §8(e). Rank `shard_rank` of `shard_world` holds rows
  // [shard_lo[g], shard_lo[g] + shard_n[g]) of ONE spatial mode s of every
  // slice (tsg_shard_setup_mode; default: the largest spatial mode, the last
  // one on ties), as a dense tensor N_0 x .. x n_g x .. x N_{d-2}. Modes
  // 0..s-1 are projected on the local slab; the per-slice exchange is ONE
  // allgather of [partial norm pairs of the local modes | local part of the
  // input of mode s] (the compressed tensor R_0..R_{s-1} x n_g x N_{s+1}..).
  // Mode s onwards, the decision and the insertion then run redundantly on
  // the identical assembled bytes, so all ranks hold bitwise-identical states
  // without a factor broadcast.
  // Basis growth at a local mode k < s: every rank forms the N_k x N_k Gram of
  // ITS part of the residual, ONE all-reduce sums the partial Grams
  // (N_k^2 doubles; identical bytes on every rank), the eigensolve and the
  // truncation run redundantly, and K = W^T E, the concat and the remaining
  // local modes stay local (sthosvd.cpp:45-59, streaming.cpp:142-151 split
  // over the ranks). The thin route (N_k > columns, tiny tensors only) falls
  // back to gathering the mode's input.
  // The host fulfils each exchange (NCCL over NVLink, or any other transport)
  // between tsg_shard_begin and tsg_shard_continue.
  int shard_world = 0, shard_rank = 0, shard_mode = -1;
  long long shard_lo[kMaxShards] = {0}, shard_n[kMaxShards] = {0};
  double *sh_send = nullptr, *sh_recv = nullptr, *sh_z = nullptr, *sh_stage = nullptr;
  double *sh_loc = nullptr, *sh_p = nullptr, *sh_gpart = nullptr, *sh_unf = nullptr;
  long long sh_send_cap = 0, sh_recv_cap = 0, sh_stage_cap = 0, sh_loc_cap = 0, sh_p_cap = 0,
            sh_gpart_cap = 0, sh_unf_cap = 0;
  const double* sh_y = nullptr;     // this slice's local slab (device)
  const double* sh_base = nullptr;  // local input of mode sh_m0 (the slab, or the grown local tensor)
  int sh_m0 = 0;                    // first local mode not yet settled for this slice
  int sh_mask = 0;                  // modes grown so far for this slice
  bool sh_total_done = false;       // the slice's ||y||^2 is booked
  // 0 idle, 1 compressed-tensor gather, 2 growth-mode input gather (thin
  // route), 3 partial-Gram all-reduce
  int sh_phase = 0;
  int sh_em = -1, sh_header = 0;
  long long sh_count = 0;
  long long sh_yd[kMaxD] = {0};     // local dims of the tensor behind sh_p / ebuf (phase 3)
  std::chrono::steady_clock::time_point sh_t0;

  void shard_setup(int rank, int world, int mode, const long long* bounds) {
    if (!initialized) fail(TSG_EINVAL, "shard_setup: state not initialised");
    if (world < 1 || world > kMaxShards || rank < 0 || rank >= world)
      fail(TSG_EINVAL, "shard_setup: bad rank / world size");
    if (mode < -1 || mode > d - 2) fail(TSG_EINVAL, "shard_setup: the shard mode must be a spatial mode");
    if (mode < 0) {
      mode = 0;
      for (int k = 1; k + 1 < d; ++k)
        if (N[k] >= N[mode]) mode = k;  // largest spatial mode, the last one on ties
    }
    const long long ns = N[mode];
    if (bounds[0] != 0 || bounds[world] != ns)
      fail(TSG_EINVAL, "shard_setup: bounds must cover [0, N_s) of the shard mode");
    for (int g = 0; g < world; ++g)
      if (bounds[g + 1] <= bounds[g]) fail(TSG_EINVAL, "shard_setup: every rank needs >= 1 row");
    flush();
    shard_world = world;
    shard_rank = rank;
    shard_mode = mode;
    for (int g = 0; g < world; ++g) {
      shard_lo[g] = bounds[g];
      shard_n[g] = bounds[g + 1] - bounds[g];
    }
    if (!sh_z) sh_z = dalloc(slice_elems);
  }
  long long shard_max_n() const {
    long long m = 0;
    for (int g = 0; g < shard_world; ++g) m = std::max(m, shard_n[g]);
    return m;
  }
  void shard_buffers(long long count, long long recv_count) {
    if (count > sh_send_cap) {
      dfree(sh_send);
      sh_send = dalloc(count);
      sh_send_cap = count;
    }
    if (recv_count > sh_recv_cap) {
      dfree(sh_recv);
      sh_recv = dalloc(recv_count);
      sh_recv_cap = recv_count;
    }
  }
  void ensure_buf(double*& buf, long long& cap, long long need) {
    if (need <= cap) return;
    dfree(buf);
    buf = dalloc(need);
    cap = need;
  }
  // Local dims of the tensor that enters local mode `m` (modes < m compressed).
  void shard_local_dims(int m, long long* yd) const {
    for (int k = 0; k + 1 < d; ++k) yd[k] = k < m ? R[k] : N[k];
    yd[shard_mode] = shard_n[shard_rank];
  }
  // Elements per shard-mode row of the input of mode `m` (m <= s): what one
  // row of a rank's block carries in an exchange of that tensor.
  long long shard_row_elems(int m) const {
    long long e = 1;
    for (int k = 0; k + 1 < d; ++k)
      if (k != shard_mode) e *= k < m ? R[k] : N[k];
    return e;
  }
  // Project the local tensor `base` (the input of local mode m_begin) through
  // modes [m_begin, m_end); the last output (base itself when the range is
  // empty) lands in sh_send + header, the partial pairs of those modes (when
  // header > 0) in sh_send[0, 2 (m_end - m_begin)).
  void shard_local_pass(const double* base, int m_begin, int m_end, int header) {
    long long yd[kMaxD];
    shard_local_dims(m_begin, yd);
    ShardPairs sp;
    std::memset(&sp, 0, sizeof sp);
    sp.partial = partial;
    sp.nmodes = m_end - m_begin;
    const double* cur = base;
    int off = 0;
    for (int k = m_begin; k < m_end; ++k) {
      double* out = (k == m_end - 1) ? sh_send + header : pick(cur, base);
      sp.off[k - m_begin] = off;
      sp.cnt[k - m_begin] = project(cur, yd, k, out, partial + off);
      off += 2 * sp.cnt[k - m_begin];
      yd[k] = R[k];
      cur = out;
    }
    if (m_end == m_begin)
      ck(cudaMemcpyAsync(sh_send + header, base, sizeof(double) * prod(yd, d - 1),
                         cudaMemcpyDeviceToDevice, st), "slab copy");
    if (header > 0) launch_shard_pack_pairs(sp, sh_send, st);
  }
  // The request is returned as soon as the local pass is enqueued: the
  // caller's collective must run on tsg_cuda_stream(h) (or after a sync).
  void shard_request(tsg_exchange* ex, int op) {
    ck(cudaGetLastError(), "shard local pass");
    ex->pending = 1;
    ex->op = op;
    ex->count = sh_count;
    ex->send = sh_send;
    ex->recv = sh_recv;
  }
  // `in_flight`: the slice took the fast path and its insertion is only
  // enqueued — the call returns without a synchronisation, the record
  // arrives through the mapped ring (published by a later slice's decision
  // kernel) and the host work of the next slice overlaps this insertion.
  void shard_done(tsg_exchange* ex, bool in_flight = false) {
    sh_phase = 0;
    if (in_flight) {
      drain(false);
    } else {
      drain(true);
      if (have_last_ctrl && pending.empty()) {
        *ctrl_h = last_ctrl;
        ck(cudaGetLastError(), "kernel");
      } else {
        pull_ctrl();
      }
      r_exact = ctrl_h->r;
    }
    ex->pending = 0;
    ex->op = TSG_XCHG_ALLGATHER;
    ex->count = 0;
    ex->send = ex->recv = nullptr;
    check_status();
  }
  // Phase 1 request: local modes [sh_m0, s) of sh_base, then the allgather of
  // [pairs of those modes | compressed local tensor].
  void shard_request_compressed(tsg_exchange* ex) {
    const int s = shard_mode;
    sh_header = 2 * (s - sh_m0);
    sh_count = (sh_header + shard_row_elems(s) * shard_max_n() + 1) / 2 * 2;
    shard_buffers(sh_count, sh_count * shard_world);
    shard_local_pass(sh_base, sh_m0, s, sh_header);
    sh_phase = 1;
    shard_request(ex, TSG_XCHG_ALLGATHER);
  }

  void shard_begin(const double* slab, int mem_kind, tsg_exchange* ex) {
    if (!initialized) fail(TSG_EINVAL, "stream_update: state not initialised");
    if (shard_world == 0) fail(TSG_EINVAL, "tsg_shard_begin: call tsg_shard_setup first");
    if (sh_phase != 0) fail(TSG_EINVAL, "tsg_shard_begin: the previous slice's exchange is pending");
    if (!deferred.empty()) flush();  // a preceding async tsg_update
    sh_t0 = std::chrono::steady_clock::now();
    const long long le = slice_elems / N[shard_mode] * shard_n[shard_rank];
    const bool misaligned = (reinterpret_cast<uintptr_t>(slab) & 15) != 0;
    if (mem_kind == TSG_MEM_HOST || misaligned) {
      ensure_buf(sh_stage, sh_stage_cap, le);
      ck(cudaMemcpyAsync(sh_stage, slab, sizeof(double) * le,
                         mem_kind == TSG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                         st), "slab copy");
      sh_y = sh_stage;
    } else {
      sh_y = slab;
    }
    sh_base = sh_y;
    sh_m0 = 0;
    sh_mask = 0;
    sh_total_done = false;
    shard_request_compressed(ex);
  }

  ShardLayout shard_layout() const {
    ShardLayout L;
    std::memset(&L, 0, sizeof L);
    L.world = shard_world;
    L.count = sh_count;
    L.ns = N[shard_mode];
    for (int g = 0; g < shard_world; ++g) {
      L.lo[g] = shard_lo[g];
      L.nloc[g] = shard_n[g];
    }
    return L;
  }

  // Local-mode growth, first half: the local residual of mode em and its
  // partial Gram; the all-reduce request.
  void shard_growth_request(int em, tsg_exchange* ex) {
    const long long rows = N[em];
    long long yd[kMaxD];
    shard_local_dims(sh_m0, yd);
    const double* cur = sh_base;
    for (int k = sh_m0; k < em; ++k) {
      double* out = pick(cur, sh_base);
      project(cur, yd, k, out, partial + 2LL * kMaxGrid * kMaxD);
      yd[k] = R[k];
      cur = out;
    }
    const long long size = prod(yd, d - 1);
    ensure_buf(sh_p, sh_p_cap, size / rows * std::max(R[em], 1LL));
    expand_residual(cur, yd, em, sh_p);  // P_loc -> sh_p, E_loc -> ebuf
    std::memcpy(sh_yd, yd, sizeof yd);
    const long long cols = size / rows;
    const double* A = ebuf;
    if (em != 0) {
      ensure_buf(sh_unf, sh_unf_cap, size);
      ModeView v{prod(yd, em), rows, prod(yd + em + 1, d - 2 - em)};
      launch_unfold(ebuf, v, sh_unf, st);
      A = sh_unf;
    }
    sh_count = (rows * rows + 1) / 2 * 2;
    shard_buffers(sh_count, sh_count);
    const int splits = gram_splits((int)rows, cols);
    ensure_buf(sh_gpart, sh_gpart_cap, (long long)splits * rows * rows);
    if (sh_count > rows * rows)
      ck(cudaMemsetAsync(sh_send + rows * rows, 0, sizeof(double), st), "memset");
    launch_gram(A, (int)rows, cols, sh_send, sh_gpart, st);
    sh_em = em;
    sh_phase = 3;
    shard_request(ex, TSG_XCHG_ALLREDUCE_SUM);
  }

  void shard_continue(tsg_exchange* ex) {
    if (sh_phase == 0) fail(TSG_EINVAL, "tsg_shard_continue: no exchange pending");
    const int s = shard_mode, G = shard_world;
    long long yd[kMaxD];
    if (sh_phase == 3) {
      // the summed Gram of the residual: subspace, then everything local
      const int em = sh_em;
      pull_ctrl();
      Sub sub;
      subspace_from_gram(sub, sh_recv, N[em], slots_h[0].delta);
      long long ydl[kMaxD];
      std::memcpy(ydl, sh_yd, sizeof ydl);
      const long long grown = prod(ydl, d - 1) / N[em] * (R[em] + sub.rank);
      ensure_buf(sh_loc, sh_loc_cap, grown);
      // sh_base may be sh_loc itself (a second local growth): the concat
      // reads only sh_p and kbuf
      expand_finish(ydl, em, sub, sh_p, sh_loc);
      sh_mask |= 1 << em;
      sh_base = sh_loc;
      sh_m0 = em + 1;
      shard_request_compressed(ex);
      return;
    }
    if (sh_phase == 2) {
      // thin route: the gathered input of the growing mode, grown redundantly
      const int em = sh_em;
      ShardLayout L = shard_layout();
      L.header = 0;
      L.inner = 1;
      for (int k = 0; k < s; ++k) L.inner *= k < em ? R[k] : N[k];
      L.outer = prod(N + s + 1, d - 2 - s);
      launch_shard_unpack(L, sh_recv, sh_z, nullptr, st);
      for (int k = 0; k + 1 < d; ++k) yd[k] = k < em ? R[k] : N[k];
      pull_ctrl();
      run_growth(sh_z, yd, em, em, slots_h[0].delta, 0, sh_t0, em, 0, sh_mask);
      shard_done(ex);
      return;
    }
    // phase 1: assemble the input of mode s and the per-rank pairs of the
    // local modes [m0, s) (into the decision's partial area, rank order)
    const int m0 = sh_m0;
    ShardLayout L = shard_layout();
    L.header = sh_header;
    L.inner = prod(R, s);
    L.outer = prod(N + s + 1, d - 2 - s);
    launch_shard_unpack(L, sh_recv, sh_z, partial, st);
    for (int k = 0; k + 1 < d; ++k) yd[k] = k < s ? R[k] : N[k];
    DecideArgs da;
    std::memset(&da, 0, sizeof da);
    da.slot = slots;
    da.nmodes = d - 1;
    da.tau = tau;
    da.order = d;
    da.partial = partial;
    da.first_mode = m0;
    int off = 2 * G * (s - m0);
    for (int k = m0; k < s; ++k) {
      da.off[k] = 2 * G * (k - m0);
      da.cnt[k] = G;
    }
    long long ydk[kMaxD];
    std::memcpy(ydk, yd, sizeof yd);
    const double* cur = sh_z;
    for (int k = s; k + 1 < d; ++k) {
      double* out = pick(cur, sh_z);
      da.off[k] = off;
      da.cnt[k] = project(cur, ydk, k, out, partial + off);
      off += 2 * da.cnt[k];
      ydk[k] = R[k];
      cur = out;
    }
    SliceCtl sc;
    if (m0 == 0) {
      // the decision comes back through the mapped slot (a spin, no copy
      // call); the same kernel publishes the records of completed insertions
      da.host_slot = hslot_d;
      da.seq_counter = seq_dev;
      da.ring_dev = ring_dev;
      da.ring_host = ring_d;
      da.ring_pub = ring_pub;
      ++seq_expect[0];
      launch_decide(da, st);
      sc = wait_slot(0);
      slots_h[0] = sc;  // the growth paths read the slice's delta from here
    } else {
      // after a local growth: the remaining modes against the slice's delta
      launch_decide(da, st);
      pull_slot(0);
      sc = slots_h[0];
    }
    const int with_total = sh_total_done ? 0 : 1;
    if (sc.zero_slice) {
      zero_slice_path(0, sh_t0);
    } else if (sc.expand_mode < 0) {
      if (m0 == 0) {
        enqueue_isvd(cur, 0, 0, st, true, sh_t0);
        shard_done(ex, /*in_flight=*/true);
        return;
      } else {
        launch_commit_modes(ctrl, slots, m0, d - 1, with_total, st);
        pull_ctrl();
        r_exact = ctrl_h->r;
        ensure_pipe();
        enqueue_isvd(cur, 0, sh_mask, st, false, sh_t0);
      }
    } else if (sc.expand_mode >= s) {
      pull_ctrl();
      run_growth(sh_z, yd, s, sc.expand_mode, sc.delta, 0, sh_t0, m0, with_total, sh_mask);
    } else {
      // growth at a local mode
      const int em = sc.expand_mode;
      launch_commit_modes(ctrl, slots, m0, em, with_total, st);
      sh_total_done = true;
      const long long cols_full = slice_elems_at(em) / N[em];
      if (N[em] <= cols_full) {
        shard_growth_request(em, ex);
      } else {
        // thin route (rows > columns): gather that mode's input instead
        sh_em = em;
        sh_count = (shard_row_elems(em) * shard_max_n() + 1) / 2 * 2;
        shard_buffers(sh_count, sh_count * shard_world);
        shard_local_pass(sh_base, sh_m0, em, 0);
        sh_phase = 2;
        shard_request(ex, TSG_XCHG_ALLGATHER);
      }
      return;
    }
    shard_done(ex);
  }
  // Elements of the full input tensor of mode m (modes < m compressed).
  long long slice_elems_at(int m) const {
    long long e = 1;
    for (int k = 0; k + 1 < d; ++k) e *= k < m ? R[k] : N[k];
    return e;
  }

  void flush() {
    settle(0);
    sync();
    drain(true);
    pull_ctrl();
    r_exact = ctrl_h->r;
    dump_tail_clk();
    check_status();
  }

  // ------------------------------------------------------------ init
  void init(const double* x, int order, const long long* dims, double t, int mem_kind) {
    if (order < 2) fail(TSG_EINVAL, "stream_init: need at least one non-streaming mode");
    if (order > kMaxD) fail(TSG_EINVAL, "stream_init: order exceeds TSG_MAXD");
    for (int k = 0; k < order; ++k)
      if (dims[k] <= 0) fail(TSG_EINVAL, "stream_init: dims must be positive");
    reset_state();
    d = order;
    tau = t;
    const long long size = prod(dims, order);
    // a device batch is read in place (never written): no second copy of what
    // may be the largest buffer of the run (config 4: 72.5 GB)
    const bool own_x = !(mem_kind == TSG_MEM_DEVICE && (reinterpret_cast<uintptr_t>(x) & 15) == 0);
    double* X = const_cast<double*>(x);
    if (own_x) {
      X = dalloc(size);
      ck(cudaMemcpyAsync(X, x, sizeof(double) * size,
                         mem_kind == TSG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                         st), "init H2D");
    }
    auto drop_x = [&] {
      if (own_x) dfree(X);
    };
    double* nrm = dalloc(1 + 1024);
    launch_sumsq(X, size, nrm, nrm + 1, st);
    double xsq = 0.0;
    ck(cudaMemcpyAsync(&xsq, nrm, 8, cudaMemcpyDeviceToHost, st), "norm D2H");
    sync();
    ck(cudaGetLastError(), "init norm");
    dfree(nrm);
    if (std::sqrt(xsq) == 0.0) {
      drop_x();
      fail(TSG_EINVAL, "stream_init: initial batch must be nonzero to seed a factorization");
    }
    if (!(t > 0.0 && t < 1.0)) {
      drop_x();
      fail(TSG_EINVAL, "sthosvd: tau must lie in (0, 1)");
    }
    // sthosvd (sthosvd.cpp:94-133)
    const double delta = t * std::sqrt(xsq) / std::sqrt((double)order);
    long long cd[kMaxD];
    for (int k = 0; k < order; ++k) cd[k] = dims[k];
    double* coreT = X;
    double discarded = 0.0;
    Sub last;
    double* left_cm = nullptr;
    for (int k = 0; k < order; ++k) {
      Sub s = mode_subspace(coreT, cd, order, k, delta);
      const long long rk = s.rank;
      ModeView v{prod(cd, k), cd[k], prod(cd + k + 1, order - k - 1)};
      double* nc = dalloc(v.left * rk * v.right);
      ProjArgs a;
      a.x = coreT;
      a.v = v;
      a.u = s.basis;
      a.R = (int)rk;
      a.p = nc;
      a.e = nullptr;
      a.partial = nullptr;
      a.residual = 0;
      launch_project(a, st);
      if (k < order - 1) {
        N[k] = dims[k];
        R[k] = rk;
        U[k] = dalloc(N[k] * N[k]);
        ck(cudaMemcpyAsync(U[k], s.basis, sizeof(double) * N[k] * rk, cudaMemcpyDeviceToDevice, st),
           "factor");
      } else {
        left_cm = dalloc(dims[k] * rk);
        ck(cudaMemcpyAsync(left_cm, s.basis, sizeof(double) * dims[k] * rk,
                           cudaMemcpyDeviceToDevice, st), "left");
      }
      discarded += s.disc;
      sync();
      if (coreT != X) dfree(coreT);
      else drop_x();
      coreT = nc;
      cd[k] = rk;
      if (k == order - 1) {
        last = s;
      } else {
        release(s);
      }
    }
    const int r = (int)cd[order - 1];
    const long long n = prod(cd, order - 1);
    n_d = dims[order - 1];
    slice_elems = prod(dims, order - 1);
    capr = std::max(16, (2 * r + 8 + 7) / 8 * 8);
    if (cfg_capr > 0) capr = std::max<int>(capr, (int)cfg_capr);
    cap_rows = std::max<long long>(cfg_rows > 0 ? cfg_rows : 0, std::max(256LL, 2 * n_d));
    qcap = n * capr;
    Q = dalloc_zero(qcap);
    Q2 = dalloc_zero(qcap);
    core = dalloc_zero(qcap);
    core2 = dalloc_zero(qcap);
    sigma = dalloc(capr + 1);
    sigma2 = dalloc(capr + 1);
    left = dalloc(cap_rows * capr);
    left2 = dalloc(cap_rows * capr);
    ck(cudaMemsetAsync(left, 0, sizeof(double) * cap_rows * capr, st), "memset");
    pgram = dalloc((long long)capr * capr);
    inner = dalloc(isvd_inner_scratch(capr));
    slice = dalloc(slice_elems);
    slice_b = dalloc(slice_elems);
    w0 = dalloc(slice_elems);
    w1 = dalloc(slice_elems);
    w2 = dalloc(slice_elems);
    evec = dalloc(n);
    evec_n = n;
    ensure_isvd_buffers();
    ensure_partial(0);
    ck(cudaMemcpyAsync(core, coreT, sizeof(double) * n * r, cudaMemcpyDeviceToDevice, st), "core");
    launch_init_isvd(ctrl, coreT, n, r, last.evals, Q, sigma, left_cm, n_d, left, capr, st);
    // isvd_init validation (isvd.cpp:139-153)
    double* od = dalloc(2);
    launch_orth_defect(left_cm, n_d, n_d, r, od, st);
    launch_orth_defect(Q, n, n, r, od + 1, st);
    std::memset(ctrl_h, 0, sizeof(Ctrl));
    ctrl_h->squared_error = discarded;
    ctrl_h->total_input_sq = xsq;
    ctrl_h->nonstream_discarded_sq = 0.0;
    ctrl_h->r = r;
    ctrl_h->n_d = n_d;
    push_ctrl();
    launch_coupling_check(ctrl, core, Q, sigma, n, r, nullptr, st);
    double defects[2];
    std::vector<double> sv(r);
    ck(cudaMemcpyAsync(defects, od, 16, cudaMemcpyDeviceToHost, st), "defect");
    ck(cudaMemcpyAsync(sv.data(), sigma, 8 * r, cudaMemcpyDeviceToHost, st), "sigma");
    pull_ctrl();
    dfree(od);
    dfree(coreT);
    dfree(left_cm);
    release(last);
    for (int k = order - 1; k < kMaxD; ++k) R[k] = 0;
    r_host = r;
    r_exact = r;
    if (defects[0] > 1e-6) fail(TSG_EINVAL, "isvd_init: left factor not orthonormal");
    if (defects[1] > 1e-6) fail(TSG_EINVAL, "isvd_init: right factor not orthonormal");
    for (int j = 0; j < r; ++j) {
      if (!(sv[j] > 0.0)) fail(TSG_EINVAL, "isvd_init: singular values must be positive");
      if (j > 0 && sv[j] > sv[j - 1]) fail(TSG_EINVAL, "isvd_init: singular values must descend");
    }
    if (!(discarded >= 0.0)) fail(TSG_EINVAL, "isvd_init: initial squared error must be nonnegative");
    check_status();
    initialized = true;
  }

  long long cfg_capr = 0, cfg_rows = 0;
  // ISVDOptions::reorthogonalize_every (isvd.hpp:62-67): MGS of both factors
  // after every K-th insertion (isvd.cpp:243-248); 0 = off (reference default)
  long long reorth_every = 0;

  void reset_state() {
    free_all();
    for (int k = 0; k < kMaxD; ++k) U[k] = nullptr;
    core = core2 = Q = Q2 = sigma = sigma2 = left = left2 = nullptr;
    slice = slice_b = w0 = w1 = w2 = ebuf = kbuf = evec = partial = ipart = pgram = inner = nullptr;
    tile_ctr = nullptr;
    tail_done = nullptr;
    isvd_hand = nullptr;
    isvd_gsync = nullptr;
    for (int k = 0; k < kMaxD; ++k) {
      upad[k] = nullptr;
      upad_R[k] = 0;
    }
    for (auto& p : stage) p = nullptr;
    sh_send = sh_recv = sh_z = sh_stage = nullptr;
    sh_send_cap = sh_recv_cap = sh_stage_cap = 0;
    shard_world = 0;
    sh_phase = 0;
    sh_loc = sh_p = sh_gpart = sh_unf = nullptr;
    sh_loc_cap = sh_p_cap = sh_gpart_cap = sh_unf_cap = 0;
    deferred.clear();
    partial_cap = ipart_cap = 0;
    evec_n = 0;
    metrics.clear();
    pending.clear();
    rec_read = 0;
    have_last_ctrl = false;
    for (auto& l : pev_live) l = false;
    for (auto& q : seq_expect) q = 0;
    r_exact = 0;
    drift_pending = 0;
    upd_count = 0;
    for (auto& v : ev_isvd_valid) v = false;
    pipe_elems = 0;
    for (auto& set : pw)
      for (auto& b : set) b = nullptr;
    initialized = false;
    n_d = 0;
    insertions_host = 0;
    if (!si) ck(cudaStreamCreateWithFlags(&si, cudaStreamNonBlocking), "cudaStreamCreate");
    if (!sc) ck(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking), "cudaStreamCreate");
    if (!s2) ck(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking), "cudaStreamCreate");
    for (int i = 0; i < kNP; ++i)
      if (!ev_m0[i]) ck(cudaEventCreateWithFlags(&ev_m0[i], cudaEventDisableTiming), "event");
    for (int i = 0; i < kNP; ++i) {
      if (!ev_h2d[i]) ck(cudaEventCreateWithFlags(&ev_h2d[i], cudaEventDisableTiming), "event");
      ev_h2d_valid[i] = false;
    }
    for (int i = 0; i < kNP; ++i) {
      if (!ev_proj[i]) ck(cudaEventCreateWithFlags(&ev_proj[i], cudaEventDisableTiming), "event");
      if (!ev_isvd[i]) ck(cudaEventCreateWithFlags(&ev_isvd[i], cudaEventDisableTiming), "event");
    }
    for (auto& set : pev)
      for (auto& e : set)
        if (!e) ck(cudaEventCreate(&e), "event");
    // every cross-stream event starts recorded, so graph wait nodes are valid
    for (int i = 0; i < kNP; ++i) {
      ck(cudaEventRecord(ev_h2d[i], st), "cudaEventRecord");
      ck(cudaEventRecord(ev_proj[i], st), "cudaEventRecord");
      ck(cudaEventRecord(ev_isvd[i], st), "cudaEventRecord");
      ck(cudaEventRecord(ev_m0[i], st), "cudaEventRecord");
    }
    ctrl = reinterpret_cast<Ctrl*>(dalloc((sizeof(Ctrl) + 7) / 8));
    ck(cudaMallocHost(&ctrl_h, sizeof(Ctrl)), "cudaMallocHost");
    std::memset(ctrl_h, 0, sizeof(Ctrl));
    push_ctrl();
    slots = reinterpret_cast<SliceCtl*>(dalloc(kNP * ((sizeof(SliceCtl) + 7) / 8)));
    ck(cudaMallocHost(&slots_h, kNP * sizeof(SliceCtl)), "cudaMallocHost");
    std::memset(slots_h, 0, kNP * sizeof(SliceCtl));
    ck(cudaHostAlloc(&hslot, kNP * sizeof(SliceCtl), cudaHostAllocMapped), "cudaHostAlloc");
    std::memset(hslot, 0, kNP * sizeof(SliceCtl));
    ck(cudaHostAlloc(&ring_h, sizeof(RecRing), cudaHostAllocMapped), "cudaHostAlloc");
    std::memset(ring_h, 0, sizeof(RecRing));
    void* dp = nullptr;
    ck(cudaHostGetDevicePointer(&dp, hslot, 0), "cudaHostGetDevicePointer");
    hslot_d = static_cast<SliceCtl*>(dp);
    ck(cudaHostGetDevicePointer(&dp, ring_h, 0), "cudaHostGetDevicePointer");
    ring_d = static_cast<RecRing*>(dp);
    ring_dev = reinterpret_cast<RecRing*>(dalloc((sizeof(RecRing) + 7) / 8));
    ck(cudaMemsetAsync(ring_dev, 0, sizeof(RecRing), st), "memset");
    ring_pub = reinterpret_cast<unsigned long long*>(dalloc(1));
    ck(cudaMemsetAsync(ring_pub, 0, 8, st), "memset");
    seq_dev = reinterpret_cast<unsigned long long*>(dalloc(kNP));
    ck(cudaMemsetAsync(seq_dev, 0, kNP * sizeof(unsigned long long), st), "memset");
    // grid-insertion handoff + handshake words (zeroed before any insertion)
    isvd_hand = dalloc(kHandDoubles);
    isvd_gsync = reinterpret_cast<unsigned*>(dalloc(2));
    ck(cudaMemsetAsync(isvd_gsync, 0, 16, st), "memset");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  }

  void destroy_streams() {
    for (int i = 0; i < kNP; ++i) {
      if (ev_proj[i]) cudaEventDestroy(ev_proj[i]);
      if (ev_isvd[i]) cudaEventDestroy(ev_isvd[i]);
    }
    for (auto& set : pev)
      for (auto& e : set)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < kNP; ++i)
      if (ev_h2d[i]) cudaEventDestroy(ev_h2d[i]);
    for (int i = 0; i < kNP; ++i)
      if (ev_m0[i]) cudaEventDestroy(ev_m0[i]);
    if (si) cudaStreamDestroy(si);
    if (sc) cudaStreamDestroy(sc);
    if (s2) cudaStreamDestroy(s2);
    si = nullptr;
    sc = nullptr;
    s2 = nullptr;
  }

  // ------------------------------------------------------ export/import
  void query(tsg_dims* o) {
    flush();
    std::memset(o, 0, sizeof *o);
    o->order = d;
    o->n_d = ctrl_h->n_d;
    o->rank = ctrl_h->r;
    o->insertions = ctrl_h->insertions;
    for (int k = 0; k + 1 < d; ++k) {
      o->core_dims[k] = R[k];
      o->slice_dims[k] = N[k];
    }
    o->core_dims[d - 1] = ctrl_h->r;
    o->tau = tau;
    o->squared_error = ctrl_h->squared_error;
    o->total_input_sq = ctrl_h->total_input_sq;
    o->nonstream_discarded_sq = ctrl_h->nonstream_discarded_sq;
  }

  void export_state(double* hcore, double* factors, double* hsigma, double* hleft, double* hright) {
    flush();
    const int r = ctrl_h->r;
    const long long n = n_rows();
    const long long nd = ctrl_h->n_d;
    if (hcore) ck(cudaMemcpy(hcore, core, sizeof(double) * n * r, cudaMemcpyDeviceToHost), "export");
    if (hright) ck(cudaMemcpy(hright, Q, sizeof(double) * n * r, cudaMemcpyDeviceToHost), "export");
    if (hsigma) ck(cudaMemcpy(hsigma, sigma, sizeof(double) * r, cudaMemcpyDeviceToHost), "export");
    if (factors) {
      long long off = 0;
      for (int k = 0; k + 1 < d; ++k) {
        ck(cudaMemcpy(factors + off, U[k], sizeof(double) * N[k] * R[k], cudaMemcpyDeviceToHost),
           "export");
        off += N[k] * R[k];
      }
    }
    if (hleft) {
      std::vector<double> rm(std::max<long long>(nd * capr, 1));
      ck(cudaMemcpy(rm.data(), left, sizeof(double) * nd * capr, cudaMemcpyDeviceToHost), "export");
      for (long long i = 0; i < nd; ++i)
        for (int j = 0; j < r; ++j) hleft[i + j * nd] = rm[i * capr + j];
    }
  }

  void import_state(const tsg_dims* dm, const double* hcore, const double* factors,
                    const double* hsigma, const double* hleft, const double* hright) {
    const int order = dm->order;
    if (order < 2 || order > kMaxD) fail(TSG_EINVAL, "assemble_streaming_state: need d >= 2");
    reset_state();
    d = order;
    tau = dm->tau;
    for (int k = 0; k + 1 < d; ++k) {
      N[k] = dm->slice_dims[k];
      R[k] = dm->core_dims[k];
      if (R[k] > N[k] || R[k] <= 0) fail(TSG_EINVAL, "assemble_streaming_state: bad ranks");
    }
    const int r = (int)dm->core_dims[d - 1];
    const long long n = n_rows();
    n_d = dm->n_d;
    slice_elems = prod(N, d - 1);
    capr = std::max(16, (2 * r + 8 + 7) / 8 * 8);
    cap_rows = std::max(256LL, 2 * n_d);
    qcap = n * capr;
    Q = dalloc_zero(qcap); Q2 = dalloc_zero(qcap); core = dalloc_zero(qcap); core2 = dalloc_zero(qcap);
    sigma = dalloc(capr + 1); sigma2 = dalloc(capr + 1);
    left = dalloc(cap_rows * capr); left2 = dalloc(cap_rows * capr);
    pgram = dalloc((long long)capr * capr);
    inner = dalloc(isvd_inner_scratch(capr));
    slice = dalloc(slice_elems); slice_b = dalloc(slice_elems);
    w0 = dalloc(slice_elems); w1 = dalloc(slice_elems); w2 = dalloc(slice_elems);
    evec = dalloc(n);
    evec_n = n;
    ensure_isvd_buffers();
    ensure_partial(0);
    long long off = 0;
    for (int k = 0; k + 1 < d; ++k) {
      U[k] = dalloc(N[k] * N[k]);
      ck(cudaMemcpy(U[k], factors + off, sizeof(double) * N[k] * R[k], cudaMemcpyHostToDevice), "import");
      off += N[k] * R[k];
    }
    ck(cudaMemcpy(core, hcore, sizeof(double) * n * r, cudaMemcpyHostToDevice), "import");
    ck(cudaMemcpy(Q, hright, sizeof(double) * n * r, cudaMemcpyHostToDevice), "import");
    ck(cudaMemcpy(sigma, hsigma, sizeof(double) * r, cudaMemcpyHostToDevice), "import");
    std::vector<double> rm(cap_rows * capr, 0.0);
    for (long long i = 0; i < n_d; ++i)
      for (int j = 0; j < r; ++j) rm[i * capr + j] = hleft[i + j * n_d];
    ck(cudaMemcpy(left, rm.data(), sizeof(double) * cap_rows * capr, cudaMemcpyHostToDevice), "import");
    std::memset(ctrl_h, 0, sizeof(Ctrl));
    ctrl_h->squared_error = dm->squared_error;
    ctrl_h->total_input_sq = dm->total_input_sq;
    ctrl_h->nonstream_discarded_sq = dm->nonstream_discarded_sq;
    ctrl_h->r = r;
    ctrl_h->n_d = n_d;
    ctrl_h->insertions = dm->insertions;
    push_ctrl();
    launch_coupling_check(ctrl, core, Q, sigma, n, r, nullptr, st);
    pull_ctrl();
    r_host = r;
    r_exact = r;
    check_status();
    initialized = true;
  }

  // ------------------------------------------------------ reconstruction
  // Slices [t0, t0 + count) of full_model() (streaming.hpp:48-49) into the
  // device buffer `out` (colexicographic N_0 x .. x N_{d-2} x count).
  void reconstruct_dev(long long t0, long long count, double* out) {
    flush();
    const long long nd = ctrl_h->n_d;
    if (t0 < 0 || count < 0 || t0 + count > nd)
      fail(TSG_EINVAL, "reconstruct: slice range outside [0, n_d)");
    if (count == 0) return;
    const int r = ctrl_h->r;
    const long long n = n_rows();
    long long dims[kMaxD];
    for (int k = 0; k + 1 < d; ++k) dims[k] = R[k];
    const long long total = slice_elems * count;
    double* a = dalloc(total);
    double* b = dalloc(total);
    launch_recon_core(core, n, r, left, capr, t0, count, a, st);
    double* cur = a;
    for (int k = 0; k + 1 < d; ++k) {
      const long long lft = prod(dims, k);
      const long long rgt = prod(dims + k + 1, d - 2 - k) * count;
      double* dst = (k + 2 == d) ? out : (cur == a ? b : a);
      launch_recon_expand(cur, lft, (int)R[k], rgt, U[k], N[k], dst, st);
      dims[k] = N[k];
      cur = dst;
    }
    ck(cudaStreamSynchronize(st), "reconstruct");
    ck(cudaGetLastError(), "reconstruct");
    dfree(a);
    dfree(b);
  }
  void reconstruct(long long t0, long long count, double* out, int mem_kind) {
    if (mem_kind == TSG_MEM_DEVICE) {
      reconstruct_dev(t0, count, out);
      return;
    }
    double* tmp = dalloc(std::max(1LL, slice_elems * count));
    reconstruct_dev(t0, count, tmp);
    ck(cudaMemcpy(out, tmp, sizeof(double) * slice_elems * count, cudaMemcpyDeviceToHost), "D2H");
    dfree(tmp);
  }
  // ||x - X||^2 and ||x||^2 over slices [t0, t0 + count) of full_model()
  // (relative_error, sthosvd.cpp:148-160, accumulated per slice range).
  void error_sums(const double* x, long long t0, long long count, int mem_kind, double* num_sq,
                  double* den_sq) {
    const long long total = slice_elems * count;
    double* rec = dalloc(std::max(1LL, total));
    reconstruct_dev(t0, count, rec);
    const double* xd = x;
    double* xc = nullptr;
    if (mem_kind == TSG_MEM_HOST) {
      xc = dalloc(std::max(1LL, total));
      ck(cudaMemcpy(xc, x, sizeof(double) * total, cudaMemcpyHostToDevice), "H2D");
      xd = xc;
    }
    double* part = dalloc(4 * kNumSMs + 2);
    double hs[2] = {0.0, 0.0};
    if (total > 0) {
      launch_diff_sumsq(xd, rec, total, part, part + 4 * kNumSMs, st);
      ck(cudaMemcpyAsync(hs, part + 4 * kNumSMs, 16, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "error sums");
    }
    *num_sq = hs[0];
    *den_sq = hs[1];
    dfree(part);
    if (xc) dfree(xc);
    dfree(rec);
  }

  // process_nonstreaming_mode (streaming.cpp:126-155) on a host tensor.
  // add_row (isvd.hpp:110-111, isvd.cpp:163-250) on the device state, with
  // the core rotation stream_update applies around it (streaming.cpp:199-222):
  // b = vec(projected slice), n = prod R_k entries; abs_tol is the explicit
  // truncation threshold; slice_sq (>= 0) is booked into total_input_sq.
  // stream_update == process_nonstreaming_mode for every mode + this call.
  void add_row(const double* b_in, int mem_kind, double abs_tol, double slice_sq,
               tsg_add_row_result* out) {
    if (!initialized) fail(TSG_EINVAL, "add_row: state not initialised");
    if (!(abs_tol >= 0.0) || !(slice_sq >= 0.0)) fail(TSG_EINVAL, "add_row: negative threshold or norm");
    flush();
    const long long n = n_rows();
    double* bd = w0;  // >= slice_elems >= n doubles
    ck(cudaMemcpyAsync(bd, b_in, sizeof(double) * n,
                       mem_kind == TSG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st),
       "row copy");
    SliceCtl sc;
    std::memset(&sc, 0, sizeof sc);
    sc.slice_sq = slice_sq;
    sc.delta = abs_tol;
    sc.expand_mode = -1;
    slots_h[0] = sc;
    ck(cudaMemcpyAsync(slots, slots_h, sizeof(SliceCtl), cudaMemcpyHostToDevice, st), "slot H2D");
    launch_commit_modes(ctrl, slots, 0, 0, 1, st);  // total_input_sq += slice_sq
    const int r_old = ctrl_h->r;
    r_exact = r_old;
    ensure_pipe();
    enqueue_isvd(bd, 0, 0, st, false, std::chrono::steady_clock::now());
    sync();
    drain(true);
    pull_ctrl();
    r_exact = ctrl_h->r;
    if (out) {
      out->r_old = r_old;
      out->r_new = ctrl_h->r;
      out->degenerate = ctrl_h->degenerate;
      out->added_error_sq = ctrl_h->added_error_sq;
    }
    check_status();
  }

  double process_mode(const double* y_h, const long long* ydims, int mode, double delta,
                      double* y_out, long long cap, long long* ydims_out) {
    if (mode < 0 || mode >= d - 1) fail(TSG_EINVAL, "process_mode: mode out of range");
    if (ydims[mode] != N[mode]) fail(TSG_EINVAL, "process_mode: shape mismatch");
    flush();
    long long yd[kMaxD];
    for (int k = 0; k + 1 < d; ++k) yd[k] = ydims[k];
    const long long size = prod(yd, d - 1);
    double* yb = dalloc(size);
    double* pb = dalloc(size);
    double* cb = dalloc(size + prod(yd, d - 1) / std::max(1LL, yd[mode]) * N[mode]);
    ck(cudaMemcpyAsync(yb, y_h, sizeof(double) * size, cudaMemcpyHostToDevice, st), "y H2D");
    ensure_partial(2 * 148 + 16);
    DecideArgs da;
    std::memset(&da, 0, sizeof da);
    da.slot = slots;
    da.nmodes = mode + 1;
    da.tau = tau;
    da.order = d;
    da.partial = partial;
    da.off[mode] = 0;
    da.cnt[mode] = project(yb, yd, mode, pb, partial);
    da.first_mode = mode;
    da.keep_delta = 1;  // the caller's delta (streaming.hpp:69-70), also for mode 0
    slots_h[0].delta = delta;
    ck(cudaMemcpyAsync(&slots[0].delta, &slots_h[0].delta, 8, cudaMemcpyHostToDevice, st), "delta");
    launch_decide(da, st);
    pull_slot(0);
    const double res = std::sqrt(slots_h[0].res_sq[mode]);
    const double* out = pb;
    if (slots_h[0].expand_mode < 0) {
      launch_commit_modes(ctrl, slots, mode, mode + 1, 0, st);
      yd[mode] = R[mode];
    } else {
      // sized for yd[mode] <= N[mode]
      if (!ebuf || slice_elems < size) {
        if (size > slice_elems) fail(TSG_EINVAL, "process_mode: tensor larger than a slice");
      }
      expand_mode(yb, yd, mode, delta, pb, cb);
      out = cb;
    }
    const long long osz = prod(yd, d - 1);
    if (osz > cap) fail(TSG_EINVAL, "process_mode: output capacity");
    ck(cudaMemcpyAsync(y_out, out, sizeof(double) * osz, cudaMemcpyDeviceToHost, st), "y D2H");
    sync();
    for (int k = 0; k + 1 < d; ++k) ydims_out[k] = yd[k];
    dfree(yb);
    dfree(pb);
    dfree(cb);
    pull_ctrl();
    return res;
  }
};

// ===================================================================== C ABI
namespace {

template <class F>
int guarded(tsg_stream* h, F&& f) {
  try {
    if (h) ck(cudaSetDevice(h->device), "cudaSetDevice");
    f();
    return TSG_OK;
  } catch (const TsgError& e) {
    (h ? h->err : g_free_err) = e.what();
    cudaGetLastError();  // clear a non-sticky error so later calls start clean
    return e.code;
  } catch (const std::bad_alloc&) {
    (h ? h->err : g_free_err) = "host allocation failed";
    return TSG_EOTHER;
  } catch (const std::exception& e) {
    (h ? h->err : g_free_err) = e.what();
    return TSG_EOTHER;
  }
}

// A scratch handle for the handle-less building blocks.
struct Scratch {
  cudaStream_t st = nullptr;
  std::vector<void*> ptrs;
  Scratch() { ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream"); }
  ~Scratch() {
    for (void* p : ptrs) cudaFree(p);
    if (st) cudaStreamDestroy(st);
  }
  double* alloc(long long n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, sizeof(double) * std::max(1LL, n)), "cudaMalloc");
    ptrs.push_back(p);
    return static_cast<double*>(p);
  }
  double* up(const double* h, long long n) {
    double* p = alloc(n);
    ck(cudaMemcpyAsync(p, h, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
    return p;
  }
  void down(double* h, const double* p, long long n) {
    ck(cudaMemcpyAsync(h, p, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
  }
  void sync() {
    ck(cudaStreamSynchronize(st), "sync");
    ck(cudaGetLastError(), "kernel");
  }
};

}  // namespace

extern "C" {

int tsg_create(const tsg_config* cfg, tsg_stream** out) {
  *out = nullptr;
  tsg_stream* h = new (std::nothrow) tsg_stream();
  if (!h) return TSG_EOTHER;
  if (cfg) {
    h->device = cfg->device;
    h->flags = cfg->flags;
    h->cfg_capr = cfg->rank_capacity;
    h->cfg_rows = cfg->row_capacity;
    if (cfg->reorthogonalize_every < 0) {
      g_free_err = "reorthogonalize_every must be nonnegative";
      delete h;
      return TSG_EINVAL;
    }
    h->reorth_every = cfg->reorthogonalize_every;
  }
  int st = guarded(h, [&] {
    int n = 0;
    ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (h->device < 0 || h->device >= n) fail(TSG_EDEVICE, "no such CUDA device");
    ck(cudaSetDevice(h->device), "cudaSetDevice");
    // a BLOCKING stream: the engine's reads of a caller's device slice are
    // ordered after work the caller queued on the legacy default stream (where
    // torch, cudaMemcpy and most producers write it) with no per-call API cost
    ck(cudaStreamCreate(&h->st), "cudaStreamCreate");
    h->launches_at_create = g_launches;
  });
  if (st) {
    g_free_err = h->err;
    delete h;
    return st;
  }
  *out = h;
  return TSG_OK;
}

void tsg_destroy(tsg_stream* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  h->free_all();
  h->destroy_streams();
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

const char* tsg_last_error(const tsg_stream* h) { return h ? h->err.c_str() : g_free_err.c_str(); }

int tsg_init(tsg_stream* h, const double* x, int32_t order, const int64_t* dims, double tau,
             int32_t mem_kind) {
  return guarded(h, [&] {
    long long dd[kMaxD];
    if (order > kMaxD || order < 0) fail(TSG_EINVAL, "stream_init: bad order");
    for (int k = 0; k < order; ++k) dd[k] = dims[k];
    h->init(x, order, dd, tau, mem_kind);
  });
}

int tsg_update(tsg_stream* h, const double* slice, int32_t mem_kind) {
  return guarded(h, [&] { h->update(slice, mem_kind); });
}

int tsg_reconstruct(tsg_stream* h, int64_t t0, int64_t count, double* out, int32_t mem_kind) {
  return guarded(h, [&] {
    if (!out && count > 0) fail(TSG_EINVAL, "reconstruct: null output");
    h->reconstruct(t0, count, out, mem_kind);
  });
}

int tsg_error_sums(tsg_stream* h, const double* x, int64_t t0, int64_t count, int32_t mem_kind,
                   double* num_sq, double* den_sq) {
  return guarded(h, [&] {
    if ((!x && count > 0) || !num_sq || !den_sq) fail(TSG_EINVAL, "relative_error: null argument");
    h->flush();
    if (t0 < 0 || count < 0 || t0 + count > h->ctrl_h->n_d)
      fail(TSG_EINVAL, "relative_error: slice range outside [0, n_d)");
    h->error_sums(x, t0, count, mem_kind, num_sq, den_sq);
  });
}

int tsg_shard_setup(tsg_stream* h, int32_t rank, int32_t world, const int64_t* bounds) {
  return tsg_shard_setup_mode(h, rank, world, -1, bounds);
}

int tsg_shard_setup_mode(tsg_stream* h, int32_t rank, int32_t world, int32_t mode,
                         const int64_t* bounds) {
  return guarded(h, [&] {
    if (!bounds) fail(TSG_EINVAL, "tsg_shard_setup: bounds must not be null");
    if (world < 1 || world > kMaxShards) fail(TSG_EINVAL, "tsg_shard_setup: bad world size");
    std::vector<long long> b(bounds, bounds + world + 1);
    h->shard_setup(rank, world, mode, b.data());
  });
}

int tsg_shard_begin(tsg_stream* h, const double* slab, int32_t mem_kind, tsg_exchange* ex) {
  const int rc = guarded(h, [&] {
    if (!ex) fail(TSG_EINVAL, "tsg_shard_begin: exchange descriptor must not be null");
    h->shard_begin(slab, mem_kind, ex);
  });
  if (rc != TSG_OK) h->sh_phase = 0;  // a failed slice leaves no exchange pending
  return rc;
}

int tsg_shard_continue(tsg_stream* h, tsg_exchange* ex) {
  const int rc = guarded(h, [&] {
    if (!ex) fail(TSG_EINVAL, "tsg_shard_continue: exchange descriptor must not be null");
    h->shard_continue(ex);
  });
  if (rc != TSG_OK) h->sh_phase = 0;  // a failed slice leaves no exchange pending
  return rc;
}

int tsg_synchronize(tsg_stream* h) {
  return guarded(h, [&] {
    if (h->initialized) h->flush();
    else h->sync();
  });
}

int tsg_process_mode(tsg_stream* h, const double* y, const int64_t* ydims, int32_t mode,
                     double delta, double* y_out, int64_t y_out_cap, int64_t* ydims_out,
                     double* res) {
  return guarded(h, [&] {
    long long yd[kMaxD], od[kMaxD];
    for (int k = 0; k + 1 < h->d; ++k) yd[k] = ydims[k];
    *res = h->process_mode(y, yd, mode, delta, y_out, y_out_cap, od);
    for (int k = 0; k + 1 < h->d; ++k) ydims_out[k] = od[k];
  });
}

int tsg_add_row(tsg_stream* h, const double* b, int32_t mem_kind, double abs_tol,
                double slice_norm_sq, tsg_add_row_result* out) {
  return guarded(h, [&] {
    if (!b) fail(TSG_EINVAL, "tsg_add_row: row must not be null");
    h->add_row(b, mem_kind, abs_tol, slice_norm_sq, out);
  });
}

int tsg_query(tsg_stream* h, tsg_dims* out) {
  return guarded(h, [&] {
    if (!h->initialized) fail(TSG_EINVAL, "state not initialised");
    h->query(out);
  });
}

int tsg_export_state(tsg_stream* h, double* core, double* factors, double* sigma, double* left,
                     double* right) {
  return guarded(h, [&] {
    if (!h->initialized) fail(TSG_EINVAL, "state not initialised");
    h->export_state(core, factors, sigma, left, right);
  });
}

int tsg_import_state(tsg_stream* h, const tsg_dims* dims, const double* core,
                     const double* factors, const double* sigma, const double* left,
                     const double* right) {
  return guarded(h, [&] { h->import_state(dims, core, factors, sigma, left, right); });
}

// ---- TUCKCKPT v1 checkpoints (reference io.cpp:268-423): the streaming
// state as the reference's save_checkpoint writes it, little-endian:
//   "TUCKCKPT", u32 version = 1, u32 d, u64 dims[d] (N_0..N_{d-2}, n_d),
//   u64 ranks[d], f64 tau, u64 mode_order[d] (identity), u32 has_isvd = 1,
//   f64 core, f64 factors k < d-1 (column-major N_k x R_k), f64 sigma[r],
//   f64 left (n_d x r, column-major = streaming_factor()), f64 right
//   (n x r), f64 squared_error, total_input_sq, nonstream_discarded_sq,
//   u64 n_d.
// Written to path.tmp and renamed into place (io.cpp:151-191); loading runs
// load_checkpoint's validation, then from_checkpoint = isvd_init +
// assemble_streaming_state (coupling re-checked by the import).
}  // extern "C"
namespace ckpt {
constexpr char kMagic[8] = {'T', 'U', 'C', 'K', 'C', 'K', 'P', 'T'};
constexpr uint32_t kVersion = 1;
constexpr std::size_t kMaxOrder = 64;
[[noreturn]] void io_fail(const char* path, const std::string& msg, const char* status) {
  fail(TSG_EIO, std::string(path) + ": " + msg + " (" + status + ")");
}
struct Reader {
  FILE* f;
  const char* path;
  void exact(void* dst, std::size_t n) {
    if (std::fread(dst, 1, n, f) != n) {
      if (std::ferror(f)) io_fail(path, "read failed", "io failure");
      io_fail(path, "file ends before the declared payload", "truncated");
    }
  }
  template <class T>
  T scalar() {
    T v;
    exact(&v, sizeof v);
    return v;  // little-endian host (x86-64 / aarch64)
  }
};
}  // namespace ckpt
extern "C" {

int tsg_save_checkpoint(tsg_stream* h, const char* path) {
  return guarded(h, [&] {
    if (!h->initialized) fail(TSG_EINVAL, "state not initialised");
    if (!path) fail(TSG_EINVAL, "save_checkpoint: null path");
    tsg_dims dm;
    h->query(&dm);
    const int d = dm.order;
    const long long r = dm.rank;
    long long n = 1, core_n = 1, fac_n = 0;
    for (int k = 0; k + 1 < d; ++k) {
      n *= dm.core_dims[k];
      fac_n += dm.slice_dims[k] * dm.core_dims[k];
    }
    for (int k = 0; k < d; ++k) core_n *= dm.core_dims[k];
    std::vector<double> core(std::max(core_n, 1LL)), fac(std::max(fac_n, 1LL)), sig(std::max(r, 1LL)),
        left(std::max(dm.n_d * r, 1LL)), right(std::max(n * r, 1LL));
    h->export_state(core.data(), fac.data(), sig.data(), left.data(), right.data());
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) ckpt::io_fail(path, "cannot open for writing", "io failure");
    bool ok = true;
    auto put = [&](const void* p, std::size_t bytes) {
      if (ok && bytes && std::fwrite(p, 1, bytes, f) != bytes) ok = false;
    };
    auto u32 = [&](uint32_t v) { put(&v, 4); };
    auto u64 = [&](uint64_t v) { put(&v, 8); };
    auto f64 = [&](double v) { put(&v, 8); };
    put(ckpt::kMagic, 8);
    u32(ckpt::kVersion);
    u32((uint32_t)d);
    for (int k = 0; k + 1 < d; ++k) u64((uint64_t)dm.slice_dims[k]);
    u64((uint64_t)dm.n_d);
    for (int k = 0; k < d; ++k) u64((uint64_t)dm.core_dims[k]);
    f64(dm.tau);
    for (int k = 0; k < d; ++k) u64((uint64_t)k);
    u32(1u);
    put(core.data(), sizeof(double) * core_n);
    put(fac.data(), sizeof(double) * fac_n);
    put(sig.data(), sizeof(double) * r);
    put(left.data(), sizeof(double) * dm.n_d * r);
    put(right.data(), sizeof(double) * n * r);
    f64(dm.squared_error);
    f64(dm.total_input_sq);
    f64(dm.nonstream_discarded_sq);
    u64((uint64_t)dm.n_d);
    if (std::fflush(f) != 0) ok = false;
    if (std::fclose(f) != 0) ok = false;
    if (!ok) {
      std::remove(tmp.c_str());
      ckpt::io_fail(path, "write failed", "io failure");
    }
    if (std::rename(tmp.c_str(), path) != 0) {
      std::remove(tmp.c_str());
      ckpt::io_fail(path, "rename failed", "io failure");
    }
  });
}

int tsg_load_checkpoint(tsg_stream* h, const char* path) {
  return guarded(h, [&] {
    if (!path) fail(TSG_EINVAL, "load_checkpoint: null path");
    FILE* f = std::fopen(path, "rb");
    if (!f) ckpt::io_fail(path, "cannot open for reading", "io failure");
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    ckpt::Reader rd{f, path};
    char magic[8];
    rd.exact(magic, 8);
    if (std::memcmp(magic, ckpt::kMagic, 8) != 0) ckpt::io_fail(path, "not a model/checkpoint file", "bad magic");
    const uint32_t ver = rd.scalar<uint32_t>();
    if (ver != ckpt::kVersion) ckpt::io_fail(path, "unsupported format version " + std::to_string(ver), "bad version");
    const uint32_t d = rd.scalar<uint32_t>();
    if (d == 0 || d > ckpt::kMaxOrder)
      ckpt::io_fail(path, "unreasonable model order " + std::to_string(d), "shape mismatch");
    std::vector<uint64_t> dims(d), ranks(d), order(d);
    for (auto& v : dims) v = rd.scalar<uint64_t>();
    for (auto& v : ranks) v = rd.scalar<uint64_t>();
    const double tau = rd.scalar<double>();
    for (auto& v : order) v = rd.scalar<uint64_t>();
    const uint32_t has_isvd = rd.scalar<uint32_t>();
    if (has_isvd > 1) ckpt::io_fail(path, "invalid streaming flag", "shape mismatch");
    auto product = [&](const std::vector<uint64_t>& v) {
      uint64_t p = 1;
      for (uint64_t x : v) {
        if (x == 0 || x > std::numeric_limits<uint64_t>::max() / p)
          ckpt::io_fail(path, "dimension list has a zero or overflowing entry", "shape mismatch");
        p *= x;
      }
      return p;
    };
    const uint64_t core_n = product(ranks);
    product(dims);
    if (!(tau > 0.0 && tau < 1.0)) ckpt::io_fail(path, "stored tolerance outside (0, 1)", "shape mismatch");
    {
      std::vector<bool> seen(d, false);
      for (uint64_t m : order) {
        if (m >= d || seen[m]) ckpt::io_fail(path, "mode order is not a permutation", "shape mismatch");
        seen[m] = true;
      }
    }
    for (uint32_t k = 0; k < d; ++k)
      if (ranks[k] > dims[k]) ckpt::io_fail(path, "stored rank exceeds the matching dimension", "shape mismatch");
    if (has_isvd && d < 2) ckpt::io_fail(path, "streaming checkpoint needs at least two modes", "shape mismatch");
    // from_checkpoint (io.cpp:414-423): only streaming checkpoints resume
    if (!has_isvd) fail(TSG_EINVAL, "checkpoint holds a batch model, not a resumable stream");
    if ((int)d > TSG_MAXD) fail(TSG_EINVAL, "checkpoint order exceeds TSG_MAXD");
    uint64_t width = 1;
    for (uint32_t k = 0; k + 1 < d; ++k) width *= ranks[k];
    const uint64_t r = ranks[d - 1];
    uint64_t fac_n = 0;
    for (uint32_t k = 0; k + 1 < d; ++k) fac_n += dims[k] * ranks[k];
    const uint64_t need = core_n + fac_n + r + dims[d - 1] * r + width * r + 3;
    {
      // reject short files before allocating the payload (require_payload)
      const long here = std::ftell(f);
      std::fseek(f, 0, SEEK_END);
      const long end = std::ftell(f);
      std::fseek(f, here, SEEK_SET);
      if (here < 0 || end < 0 || (uint64_t)(end - here) < need * 8 + 8)
        ckpt::io_fail(path, "file ends before the declared payload", "truncated");
    }
    std::vector<double> core(core_n), fac(std::max<uint64_t>(fac_n, 1)), sig(std::max<uint64_t>(r, 1)),
        left(std::max<uint64_t>(dims[d - 1] * r, 1)), right(std::max<uint64_t>(width * r, 1));
    rd.exact(core.data(), 8 * core_n);
    rd.exact(fac.data(), 8 * fac_n);
    rd.exact(sig.data(), 8 * r);
    rd.exact(left.data(), 8 * dims[d - 1] * r);
    rd.exact(right.data(), 8 * width * r);
    tsg_dims dm;
    std::memset(&dm, 0, sizeof dm);
    dm.order = (int32_t)d;
    dm.squared_error = rd.scalar<double>();
    dm.total_input_sq = rd.scalar<double>();
    dm.nonstream_discarded_sq = rd.scalar<double>();
    const uint64_t nd = rd.scalar<uint64_t>();
    if (nd != dims[d - 1])
      ckpt::io_fail(path, "slice count does not match the streaming factor height", "shape mismatch");
    dm.n_d = (int64_t)nd;
    dm.rank = (int64_t)r;
    dm.insertions = 0;  // isvd_init starts a fresh insertion count
    dm.tau = tau;
    for (uint32_t k = 0; k < d; ++k) dm.core_dims[k] = (int64_t)ranks[k];
    for (uint32_t k = 0; k + 1 < d; ++k) dm.slice_dims[k] = (int64_t)dims[k];
    h->import_state(&dm, core.data(), fac.data(), sig.data(), left.data(), right.data());
  });
}

double tsg_estimate_relative_error(tsg_stream* h) {
  double out = 0.0;
  guarded(h, [&] {
    h->flush();
    const Ctrl& c = *h->ctrl_h;
    if (c.total_input_sq <= 0.0) return;
    out = std::sqrt(std::max(c.squared_error + c.nonstream_discarded_sq, 0.0) / c.total_input_sq);
  });
  return out;
}

int64_t tsg_metrics_count(tsg_stream* h) {
  int64_t n = -1;
  guarded(h, [&] {
    h->drain();
    n = (int64_t)h->metrics.size();
  });
  return n;
}

int tsg_metrics_at(tsg_stream* h, int64_t i, tsg_slice_metrics* out) {
  return guarded(h, [&] {
    h->drain();
    if (i < 0 || i >= (int64_t)h->metrics.size()) fail(TSG_EINVAL, "metrics index out of range");
    *out = h->metrics[(size_t)i];
  });
}

int tsg_last_metrics(tsg_stream* h, tsg_slice_metrics* out) {
  return guarded(h, [&] {
    h->drain();
    if (h->metrics.empty()) fail(TSG_EINVAL, "no metrics recorded");
    *out = h->metrics.back();
  });
}

int tsg_profile(tsg_stream* h, double* out, int32_t n, int32_t reset) {
  return guarded(h, [&] {
    h->sync();
    h->resolve_all();
    for (int i = 0; i < n && i < 6; ++i) out[i] = h->prof[i];
    if (reset) {
      for (double& v : h->prof) v = 0.0;
      if (h->profiling()) h->reset_timeline();
    }
  });
}

int64_t tsg_profile_timeline(tsg_stream* h, double* out, int64_t cap) {
  int64_t n = 0;
  const int st = guarded(h, [&] {
    h->sync();
    h->resolve_all();
    for (const auto& row : h->timeline) {
      if (n >= cap) break;
      for (int i = 0; i < 5; ++i) out[5 * n + i] = row[i];
      ++n;
    }
  });
  return st == TSG_OK ? n : -1;
}

int tsg_measure_fp64_peaks(int32_t device, double* dmma_tflops, double* dfma_tflops) {
  const int st = tsg::measure_fp64_peaks(device, dmma_tflops, dfma_tflops);
  if (st) g_free_err = "fp64 peak measurement failed";
  return st;
}

int tsg_debug_isvd_clocks(int64_t* out) { return tsg::read_isvd_clocks(reinterpret_cast<long long*>(out)); }

// Profiling harness: time `reps` launches of the fused projection on device
// buffers (x: left*n*right, u: n x R column-major, p: left*R*right).
int tsg_debug_project(const double* x, int64_t left, int64_t n, int64_t right, const double* u,
                      int32_t R, double* p, int32_t flags, int32_t reps, double* ms_out) {
  return guarded(nullptr, [&] {
    cudaStream_t st;
    ck(cudaStreamCreate(&st), "stream");
    double* part = nullptr;
    double* up = nullptr;
    unsigned* ctr = nullptr;
    ck(cudaMalloc(&part, sizeof(double) * 2 * kMaxGrid), "malloc");
    ck(cudaMalloc(&up, sizeof(double) * tsg::upad_size(n, R)), "malloc");
    ck(cudaMalloc(&ctr, sizeof(unsigned) * 64), "malloc");
    tsg::launch_pad_u(u, n, R, up, st);
    ProjArgs a;
    a.x = x;
    a.v = ModeView{left, n, right};
    a.u = u;
    a.R = R;
    a.p = p;
    a.partial = part;
    a.residual = (flags & 1) ? 0 : 1;
    a.stream_in = left == 1 ? 1 : 0;
    a.upad = up;
    a.debug_skip = flags & 7;
    // TMA mode-0 kernel profiling switches: 64 stream only; 128 / 256 / 512 skip
    // the cross-warp reduction / phase 2 / phase 1 (results then meaningless)
    a.karg1 = (flags & 64) ? 7 : ((((flags >> 7) & 7) << 3) | (((flags >> 10) & 1) << 6));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < reps + 2; ++i) {
      if (i == 2) cudaEventRecord(e0, st);
      cudaMemsetAsync(ctr + (i % 64), 0, sizeof(unsigned), st);
      a.tile_counter = ctr + (i % 64);
      launch_project(a, st);
    }
    cudaEventRecord(e1, st);
    ck(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = ms / reps;
    cudaFree(part);
    cudaFree(up);
    cudaFree(ctr);
    cudaStreamDestroy(st);
    ck(cudaGetLastError(), "kernel");
  });
}

int64_t tsg_readback_bytes_per_update(void) {
  return (int64_t)(sizeof(Ctrl) + sizeof(Metrics) + sizeof(SliceCtl));
}

int64_t tsg_kernel_launches(tsg_stream* h) { return h ? g_launches - h->launches_at_create : g_launches; }

void* tsg_cuda_stream(tsg_stream* h) { return h ? (void*)h->st : nullptr; }

double* tsg_slice_buffer(tsg_stream* h, int32_t which) {
  if (!h || !h->initialized) return nullptr;
  return which ? h->slice_b : h->slice;
}

int tsg_sym_eig_desc(int64_t n, const double* g, double* evals, double* evecs) {
  return guarded(nullptr, [&] {
    double max_abs = 0.0, max_asym = 0.0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        max_abs = std::max(max_abs, std::fabs(g[i + j * n]));
        max_asym = std::max(max_asym, std::fabs(g[i + j * n] - g[j + i * n]));
      }
    if (max_asym > 1e-10 * std::max(max_abs, 1e-300))
      fail(TSG_EINVAL, "sym_eig_desc: matrix is not symmetric");
    if (n == 0) return;
    Scratch s;
    double* dg = s.up(g, n * n);
    double* ev = s.alloc(n);
    double* vec = s.alloc(n * n);
    double* work = s.alloc(3 * n * n + 512);
    launch_sym_eig(dg, (int)n, ev, vec, work, nullptr, s.st);
    s.down(evals, ev, n);
    s.down(evecs, vec, n * n);
    s.sync();
  });
}

int tsg_small_svd_truncated(int64_t m, int64_t n, const double* a, double thr, double* left,
                            double* sigma, double* right, int64_t* rank, double* disc) {
  // small_svd_truncated (linalg.cpp:210-259) from the device building blocks
  return guarded(nullptr, [&] {
    if (thr < 0.0) fail(TSG_EINVAL, "small_svd_truncated: threshold must be nonnegative");
    *rank = 0;
    *disc = 0.0;
    if (m == 0 || n == 0) return;
    Scratch s;
    double* da = s.up(a, m * n);
    double* g = s.alloc(n * n);
    double* ev = s.alloc(n);
    double* vec = s.alloc(n * n);
    double* work = s.alloc(3 * n * n + 512);
    double* rk = s.alloc(2);
    launch_gram_t(da, m, (int)n, g, s.st);
    launch_sym_eig(g, (int)n, ev, vec, work, nullptr, s.st);
    double lam0 = 0.0;
    s.down(&lam0, ev, 1);
    s.sync();
    if (std::sqrt(lam0) == 0.0) return;
    launch_truncate(ev, (int)n, thr, 1, reinterpret_cast<long long*>(rk), rk + 1, s.st);
    long long hr[2];
    ck(cudaMemcpyAsync(hr, rk, 16, cudaMemcpyDeviceToHost, s.st), "D2H");
    s.sync();
    const long long r = hr[0];
    std::memcpy(disc, &hr[1], 8);
    *rank = r;
    double* lf = s.alloc(m * r);
    launch_gemm_nn(da, m, vec, n, lf, m, m, (int)r, (int)n, s.st);
    launch_scale_cols_invsqrt(lf, m, m, (int)r, ev, s.st);
    launch_mgs(lf, m, m, (int)r, s.st);
    std::vector<double> lam(r);
    s.down(lam.data(), ev, r);
    s.down(right, vec, n * r);
    s.down(left, lf, m * r);
    s.sync();
    for (long long j = 0; j < r; ++j) sigma[j] = std::sqrt(lam[j]);
  });
}

int tsg_mode_subspace(const double* t, int32_t order, const int64_t* dims, int32_t mode,
                      double delta, double* basis, int64_t* rank, double* evals, double* disc) {
  tsg_stream tmp;
  return guarded(nullptr, [&] {
    ck(cudaStreamCreateWithFlags(&tmp.st, cudaStreamNonBlocking), "stream");
    long long dd[kMaxD];
    for (int k = 0; k < order; ++k) dd[k] = dims[k];
    const long long size = prod(dd, order);
    double* dt = tmp.dalloc(size);
    ck(cudaMemcpy(dt, t, sizeof(double) * size, cudaMemcpyHostToDevice), "H2D");
    auto s = tmp.mode_subspace(dt, dd, order, mode, delta);
    *rank = s.rank;
    *disc = s.disc;
    const long long rows = dd[mode];
    ck(cudaMemcpy(basis, s.basis, sizeof(double) * rows * s.rank, cudaMemcpyDeviceToHost), "D2H");
    ck(cudaMemcpy(evals, s.evals, sizeof(double) * rows, cudaMemcpyDeviceToHost), "D2H");
    tmp.release(s);
    tmp.free_all();
    cudaStreamDestroy(tmp.st);
    tmp.st = nullptr;
  });
}

int tsg_ttm(const double* t, int32_t order, const int64_t* dims, int32_t mode, const double* a,
            int64_t a_rows, int64_t a_cols, int32_t transpose_a, double* out) {
  return guarded(nullptr, [&] {
    long long dd[kMaxD];
    for (int k = 0; k < order; ++k) dd[k] = dims[k];
    const long long contracted = transpose_a ? a_rows : a_cols;
    if (mode < 0 || mode >= order) fail(TSG_EINVAL, "mode index out of range for tensor order");
    if (contracted != dd[mode]) fail(TSG_EINVAL, "ttm: matrix does not match mode size");
    const long long produced = transpose_a ? a_cols : a_rows;
    Scratch s;
    const long long size = prod(dd, order);
    double* dt = s.up(t, size);
    // P = U^T X with U = a (transpose_a) or a^T materialised
    std::vector<double> u(a_rows * a_cols);
    if (transpose_a) {
      std::memcpy(u.data(), a, sizeof(double) * a_rows * a_cols);
    } else {
      for (long long i = 0; i < a_rows; ++i)
        for (long long j = 0; j < a_cols; ++j) u[j + i * a_cols] = a[i + j * a_rows];
    }
    double* du = s.up(u.data(), a_rows * a_cols);
    const long long osz = size / std::max(1LL, dd[mode]) * produced;
    double* dout = s.alloc(osz);
    ProjArgs pa;
    pa.x = dt;
    pa.v = ModeView{prod(dd, mode), dd[mode], prod(dd + mode + 1, order - mode - 1)};
    pa.u = du;
    pa.R = (int)produced;
    pa.p = dout;
    pa.e = nullptr;
    pa.partial = nullptr;
    pa.residual = 0;
    if (osz > 0 && size > 0) launch_project(pa, s.st);
    s.down(out, dout, osz);
    s.sync();
  });
}

}  // extern "C"
