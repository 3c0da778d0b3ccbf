// api.cu — the C ABI of libwbpr.so (declared in include/wbpr.h): argument
// validation, workspace carving, launch orchestration and error mapping.
// Each solve: K-BUILD kernels (A1) -> one cooperative persistent kernel (A2-A7)
// -> extraction kernels (A8) -> one stream synchronisation.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "wbpr.h"
#include "internal.h"
#include "kernels.h"

using namespace wbpr;

namespace {

thread_local std::string g_err;

wbpr_status fail(wbpr_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

#define CK(call)                                                                                      \
  do {                                                                                                \
    cudaError_t _e = (call);                                                                          \
    if (_e != cudaSuccess) {                                                                          \
      return fail(WBPR_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));                    \
    }                                                                                                 \
  } while (0)

struct DevInfo {
  int num_sms = 0;
  int occ[2] = {0, 0};
};

std::mutex g_mu;
std::unordered_map<int, DevInfo> g_dev;
std::unordered_map<const void*, wbpr_residual> g_views;
struct TraceInfo { const void* ptr; int rounds; int warps; };
std::unordered_map<const void*, TraceInfo> g_traces;

wbpr_status dev_info(DevInfo& out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) { out = it->second; return WBPR_OK; }
  DevInfo d;
  CK(cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev));
  d.occ[0] = solve_max_blocks_per_sm(0, kSolveThreads);
  d.occ[1] = solve_max_blocks_per_sm(1, kSolveThreads);
  CK(cudaGetLastError());
  g_dev[dev] = d;
  out = d;
  return WBPR_OK;
}

__global__ void k_init_ctrl(Ctrl* c) {
  int* p = reinterpret_cast<int*>(c);
  for (size_t i = threadIdx.x; i < sizeof(Ctrl) / sizeof(int); i += blockDim.x) p[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) c->bad_edge = LLONG_MAX;
}

__global__ void k_terms(uint8_t* term, const long long* s, const long long* t, int k) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) {
    term[s[i]] = kSource;
    term[t[i]] = kSink;
  }
}

template <typename T> T* at(void* ws, size_t off) { return reinterpret_cast<T*>(static_cast<char*>(ws) + off); }

constexpr int64_t kSlotsPerCta = 32768;   // auto grid size for small graphs

struct Ws {
  Layout L;
  void* base;
  Ctrl* ctrl;
};

// Pinned staging for the small host <-> device copies of a call (terminals, instance ranges,
// group descriptors, the control record, per-instance results).  Pageable copies are staged
// by the driver and can serialise with other streams' transfers, which would stop one
// caller thread's large H2D from overlapping another thread's kernels.  One buffer per host
// thread; every call synchronises its stream before returning, so a region is never reused
// while a copy from / to it is in flight.  The first allocation covers every group descriptor
// and a few thousand instances; a larger request allocates a bigger buffer and RETIRES the old
// one (kept until the thread exits): cudaFreeHost synchronises the whole device and would
// stall other threads' streams in the middle of their solves.
struct PinnedScratch {
  char* p = nullptr;
  size_t cap = 0;
  std::vector<char*> retired;
  ~PinnedScratch() {
    if (p) cudaFreeHost(p);
    for (char* r : retired) cudaFreeHost(r);
  }
  char* get(size_t n) {
    if (n > cap) {
      const size_t want = std::max<size_t>(n, sizeof(GroupDesc) * kMaxGroups + sizeof(Ctrl) + (size_t(1) << 17));
      char* q = nullptr;
      if (cudaHostAlloc(reinterpret_cast<void**>(&q), want, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;   // callers fall back to pageable copies
      }
      if (p) retired.push_back(p);
      p = q;
      cap = want;
    }
    return p;
  }
};
thread_local PinnedScratch g_pin;

// device -> host through the pinned scratch at byte offset `at` (synchronous)
wbpr_status read_ctrl(const Ctrl* d, Ctrl& h, cudaStream_t st) {
  char* b = g_pin.get(sizeof(Ctrl));
  if (!b) {
    CK(cudaMemcpyAsync(&h, d, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return WBPR_OK;
  }
  CK(cudaMemcpyAsync(b, d, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  memcpy(&h, b, sizeof(Ctrl));
  return WBPR_OK;
}

// host -> device of a small array through pinned memory (offset `at` of the call's upload area)
cudaError_t upload(void* dst, const void* src, size_t bytes, size_t at, cudaStream_t st) {
  char* b = g_pin.get(at + bytes);
  if (!b) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  memcpy(b + at, src, bytes);
  return cudaMemcpyAsync(dst, b + at, bytes, cudaMemcpyHostToDevice, st);
}

wbpr_options resolve(const wbpr_options* o) {
  wbpr_options r;
  wbpr_default_options(&r);
  if (o) r = *o;
  if (!(r.gr_beta > 0.f)) r.gr_beta = 0.5f;
  if (r.timeout_ms <= 0) r.timeout_ms = 120000;
  if (r.gr_gamma < 0.f) r.gr_gamma = 1.0f;
  return r;
}

// A1 for one workspace.  BCSR: no host synchronisation after validation (M stays on
// the device and is read after the solve); RCSR: Mf is read back (the reverse sort
// needs the longest reverse segment).  `ro,col,cap` are device pointers.
wbpr_status build_residual(const Ws& W, const int64_t* ro, const int32_t* col, const int32_t* cap, int layout,
                           int num_sms, const int64_t* d_vbase, int k, int& Mf, int64_t& selfloops,
                           int64_t& bad_edge, cudaStream_t st) {
  const Layout& L = W.L;
  BuildArgs a{};
  a.n = L.n; a.m = L.m; a.layout = layout; a.num_sms = num_sms;
  a.ro = ro; a.col = col; a.cap = cap; a.ctrl = W.ctrl;
  a.deg = at<int>(W.base, L.deg); a.cursor = at<int>(W.base, L.cursor);
  a.soff = at<int>(W.base, L.soff); a.off = at<int>(W.base, L.off); a.roff = at<int>(W.base, L.roff);
  a.scan_part = at<int>(W.base, L.scan_part); a.q0 = at<int>(W.base, L.q0);
  a.keys = at<uint64_t>(W.base, L.regA); a.tmp = at<uint64_t>(W.base, L.regB);
  a.arc = at<int2>(W.base, L.regC);
  a.mate = at<int>(W.base, L.regB);
  a.cap0 = at<int>(W.base, L.regB + L.bcap0);
  a.rarc = at<int2>(W.base, L.regC + 8 * (size_t)L.m);
  a.bcf = at<int>(W.base, L.regB);
  a.vbase = d_vbase; a.k = k;
  a.rsoff = at<int>(W.base, L.rsoff);
  a.need = at<uint8_t>(W.base, L.deact);
  a.q1 = at<int>(W.base, L.q1);
  a.mtasks = at<int2>(W.base, L.hc0);
  a.mheads = at<int>(W.base, L.hc1);
  a.ine = at<int>(W.base, L.regA + 4 * (size_t)L.m);
  a.src = at<int>(W.base, L.regA + 8 * (size_t)L.m);
  a.inslot = at<int>(W.base, L.regA + 8 * (size_t)L.m);
  a.outslot = at<int>(W.base, L.regD);
  a.seg = at<int2>(W.base, L.seg);

  build_validate(a, st);
  CK(cudaGetLastError());
  Ctrl c;
  wbpr_status s = read_ctrl(W.ctrl, c, st);
  if (s) return s;
  selfloops = c.selfloops;
  bad_edge = c.bad_edge == LLONG_MAX ? -1 : c.bad_edge;
  if (c.bad_rows) return fail(WBPR_EINVAL, "row_offsets are not a valid CSR offset array");
  if (bad_edge >= 0)
    return fail(WBPR_EINVAL, "edge " + std::to_string(bad_edge) +
                                 " has a column outside its instance's range or a negative capacity");
  a.maxlen = c.maxlen;
  a.maxlen_out = c.maxlen_out;
  a.any_unsorted = c.any_unsorted;
  if (layout == WBPR_LAYOUT_BCSR) {
    a.H = 2 * L.m - c.selfloops;
    build_bcsr_merge(a, st);
    build_bcsr_mate(a, st);
    CK(cudaGetLastError());
    Mf = -1;   // on the device
  } else {
    a.H = L.m;
    build_rcsr_forward(a, st);
    CK(cudaGetLastError());
    s = read_ctrl(W.ctrl, c, st);
    if (s) return s;
    if (c.overflow == 1) return fail(WBPR_EOVERFLOW, "merged capacity exceeds INT32_MAX");
    Mf = c.M;
    build_rcsr_reverse_counts(a, Mf, st);
    CK(cudaGetLastError());
    s = read_ctrl(W.ctrl, c, st);
    if (s) return s;
    build_rcsr_reverse(a, Mf, c.maxlen, st);
    CK(cudaGetLastError());
  }
  return WBPR_OK;
}

void register_view(const Ws& W, int layout, int M, int Mf) {
  const Layout& L = W.L;
  wbpr_residual v{};
  v.layout = layout;
  v.n = L.n; v.M = M; v.Mf = Mf;
  v.off = at<int>(W.base, L.off);
  v.arc = at<int>(W.base, L.regC);
  v.cap0 = at<int>(W.base, L.regB + L.bcap0);
  if (layout == WBPR_LAYOUT_BCSR) {
    v.off = nullptr;                       // gapped layout: segments by seg[u] = {begin, end}
    v.seg = at<int32_t>(W.base, L.seg);
    v.M = 2 * L.m;                         // extent of the slot space (arc/mate/cap0 length)
    v.mate = at<int>(W.base, L.regB);
  } else {
    v.roff = at<int>(W.base, L.roff);
    v.rarc = at<int>(W.base, L.regC + 8 * (size_t)L.m);
    v.bcf = at<int>(W.base, L.regB);
  }
  v.e = at<int64_t>(W.base, L.e);
  v.h = at<int32_t>(W.base, L.h);
  std::lock_guard<std::mutex> lk(g_mu);
  g_views[W.base] = v;
}

wbpr_status check_graph_args(const wbpr_csr* g) {
  if (!g) return fail(WBPR_EINVAL, "graph is NULL");
  if (g->n < 2) return fail(WBPR_EINVAL, "n must be >= 2");
  if (g->n >= INT32_MAX) return fail(WBPR_EOVERFLOW, "n must be < 2^31");
  if (g->m < 0) return fail(WBPR_EINVAL, "m must be >= 0");
  if (2 * g->m >= INT32_MAX) return fail(WBPR_EOVERFLOW, "2*m must be < 2^31");
  if (!g->row_offsets || (g->m > 0 && (!g->col || !g->cap))) return fail(WBPR_EINVAL, "NULL CSR array");
  return WBPR_OK;
}

// Every error return after work was enqueued on the stream synchronises it first (the
// persistent kernel may still be writing the caller's workspace).
struct SyncOnExit {
  cudaStream_t st;
  bool armed = false;
  ~SyncOnExit() { if (armed) { cudaStreamSynchronize(st); cudaGetLastError(); } }
};

struct Events {
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  ~Events() { for (auto& e : ev) if (e) cudaEventDestroy(e); }
  cudaError_t create() {
    for (auto& e : ev) { cudaError_t r = cudaEventCreate(&e); if (r) return r; }
    return cudaSuccess;
  }
};

// The one-CTA fused path (tiny.cu) for a tiny single BCSR instance: one launch, the result
// record back through the pinned scratch, one synchronisation.
wbpr_status solve_tiny(const wbpr_csr* g, int64_t s_v, int64_t t_v, const wbpr_options& opt, const Ws& W,
                       uint32_t* bitmap, int64_t* flow_out, int64_t* cut_out, wbpr_stats* stats, cudaStream_t st) {
  const Layout& L = W.L;
  void* ws = W.base;
  const int64_t n = g->n, m = g->m;
  const long long launches0 = launch_count();
  Events E;
  CK(E.create());
  SyncOnExit guard{st};
  guard.armed = true;
  CK(cudaEventRecord(E.ev[0], st));
  const int64_t* ro = g->row_offsets;
  const int32_t* col = g->col;
  const int32_t* cap = g->cap;
  if (g->on_host) {
    CK(cudaMemcpyAsync(at<int64_t>(ws, L.in_row), ro, 8 * (n + 1), cudaMemcpyHostToDevice, st));
    if (m > 0) {
      CK(cudaMemcpyAsync(at<int32_t>(ws, L.in_col), col, 4 * m, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(at<int32_t>(ws, L.in_cap), cap, 4 * m, cudaMemcpyHostToDevice, st));
    }
    ro = at<int64_t>(ws, L.in_row);
    col = at<int32_t>(ws, L.in_col);
    cap = at<int32_t>(ws, L.in_cap);
  }
  uint32_t* dbm = bitmap;
  if (bitmap && g->on_host) dbm = reinterpret_cast<uint32_t*>(at<int>(ws, L.q0));
  TinyArgs a{};
  a.ro = ro; a.col = col; a.cap = cap;
  a.n = (int)n; a.m = (int)m; a.s = (int)s_v; a.t = (int)t_v;
  a.seg = at<int2>(ws, L.seg); a.arc = at<int2>(ws, L.regC); a.mate = at<int>(ws, L.regB);
  a.cap0 = at<int>(ws, L.regB + L.bcap0);
  a.h = at<int>(ws, L.h); a.e = at<long long>(ws, L.e);
  a.bitmap = dbm;
  a.flow = at<long long>(ws, L.inst_flow); a.cut = at<long long>(ws, L.inst_cut);
  a.ctrl = W.ctrl;
  a.gr_beta = opt.gr_beta;
  a.max_rounds = opt.max_rounds > 0 ? opt.max_rounds : 10 * n + 1000;
  a.deadline_ns_rel = (unsigned long long)opt.timeout_ms * 1000000ull;
  CK(launch_tiny(a, st));
  CK(cudaEventRecord(E.ev[1], st));
  char* pin = g_pin.get(sizeof(Ctrl) + 16 + 64);
  Ctrl c;
  long long F = 0, Cc = 0;
  if (pin) {
    CK(cudaMemcpyAsync(pin, W.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pin + sizeof(Ctrl), a.flow, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pin + sizeof(Ctrl) + 8, a.cut, 8, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(&c, W.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&F, a.flow, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&Cc, a.cut, 8, cudaMemcpyDeviceToHost, st));
  }
  if (bitmap && g->on_host) CK(cudaMemcpyAsync(bitmap, dbm, 4 * ((n + 31) / 32), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(E.ev[2], st));
  CK(cudaStreamSynchronize(st));
  guard.armed = false;
  if (pin) { memcpy(&c, pin, sizeof(Ctrl)); memcpy(&F, pin + sizeof(Ctrl), 8); memcpy(&Cc, pin + sizeof(Ctrl) + 8, 8); }
  const int64_t bad_edge = c.bad_edge == LLONG_MAX ? -1 : c.bad_edge;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->n = n; stats->m = m; stats->bad_edge_index = bad_edge;
    stats->tiny_path = 1;
  }
  if (c.bad_rows) return fail(WBPR_EINVAL, "row_offsets are not a valid CSR offset array");
  if (bad_edge >= 0)
    return fail(WBPR_EINVAL, "edge " + std::to_string(bad_edge) +
                                 " has a column outside its instance's range or a negative capacity");
  register_view(W, WBPR_LAYOUT_BCSR, c.M, c.M);
  if (c.overflow) return fail(WBPR_EOVERFLOW, "merged capacity exceeds INT32_MAX");
  if (flow_out) flow_out[0] = F;
  if (cut_out) cut_out[0] = Cc;
  if (stats) {
    stats->flow_value = F;
    stats->cut_capacity = Cc;
    stats->M = c.M;
    stats->rounds = c.stats[ST_ROUNDS];
    stats->global_relabels = c.stats[ST_GRS];
    stats->bfs_levels = c.stats[ST_BFS_LEVELS];
    stats->pushes = c.stats[ST_PUSHES];
    stats->relabels = c.stats[ST_RELABELS];
    stats->arcs_scanned = c.stats[ST_ARCS];
    stats->bfs_arcs_scanned = c.stats[ST_BFS_ARCS];
    stats->self_loops_ignored = c.selfloops;
    stats->excess_total = c.excess_total;
    float ms = 0;
    cudaEventElapsedTime(&ms, E.ev[0], E.ev[1]);
    stats->total_ms = ms;
    stats->build_ms = (float)((double)c.phase_ns[PK_NONE] / 1e6);
    if (stats->build_ms > ms) stats->build_ms = ms;
    stats->solve_ms = ms - stats->build_ms;
    cudaEventElapsedTime(&ms, E.ev[1], E.ev[2]); stats->extract_ms = ms;
    stats->grid_blocks = 1;
    stats->block_threads = 1024;
    for (int i = 0; i < kPhBuckets; ++i) { stats->phase_ns[i] = c.phase_ns[i]; stats->phase_count[i] = c.phase_cnt[i]; }
    stats->kernel_launches = launch_count() - launches0;
  }
  if (c.status == DS_NOTCONVERGED) return fail(WBPR_ENOTCONVERGED, "round cap exceeded");
  if (c.abort || c.status == DS_TIMEOUT) return fail(WBPR_ENOTCONVERGED, "device watchdog timeout");
  if (F != Cc) return fail(WBPR_EINTERNAL, "certificate failed: cut capacity != flow value");
  if (F != c.excess_total) return fail(WBPR_EINTERNAL, "Excess_total bookkeeping disagrees with e(t)");
  return WBPR_OK;
}

// Shared driver of single and batch solves.
wbpr_status solve_impl(const wbpr_csr* g, int k, const int64_t* vbase_h, const int64_t* s_h, const int64_t* t_h,
                       const wbpr_options* opt_in, void* ws, size_t ws_bytes, uint32_t* bitmap, int64_t* flow_out,
                       int64_t* cut_out, wbpr_stats* stats, cudaStream_t st, bool build_only) {
  wbpr_status s = check_graph_args(g);
  if (s) return s;
  wbpr_options opt = resolve(opt_in);
  if (opt.layout != WBPR_LAYOUT_BCSR && opt.layout != WBPR_LAYOUT_RCSR) return fail(WBPR_EINVAL, "unknown layout");
  if (opt.schedule != 0 && opt.schedule != 1) return fail(WBPR_EINVAL, "unknown schedule");
  const int64_t n = g->n, m = g->m;
  if (k < 1 || k > kMaxInst) return fail(WBPR_EINVAL, "instance count out of range");
  if (vbase_h[0] != 0 || vbase_h[k] != n) return fail(WBPR_EINVAL, "vbase must start at 0 and end at n");
  for (int i = 0; i < k; ++i) {
    if (vbase_h[i + 1] <= vbase_h[i]) return fail(WBPR_EINVAL, "vbase must be increasing");
    if (s_h[i] < vbase_h[i] || s_h[i] >= vbase_h[i + 1] || t_h[i] < vbase_h[i] || t_h[i] >= vbase_h[i + 1])
      return fail(WBPR_EINVAL, "terminal out of its instance range");
    if (s_h[i] == t_h[i]) return fail(WBPR_EINVAL, "s == t");
  }
  if (!ws) return fail(WBPR_EINVAL, "workspace is NULL");
  Ws W;
  W.L = make_layout(n, m, k, opt.layout, opt.trace_rounds);
  if (ws_bytes < W.L.total)
    return fail(WBPR_ENOMEM, "workspace too small: need " + std::to_string(W.L.total) + " bytes");
  W.base = ws;
  W.ctrl = at<Ctrl>(ws, W.L.ctrl);
  DevInfo di;
  s = dev_info(di);
  if (s) return s;
  const Layout& L = W.L;

  if (opt.batch_groups < 0) return fail(WBPR_EINVAL, "batch_groups must be >= 0");
  if (opt.debug_stop < 0) return fail(WBPR_EINVAL, "debug_stop must be >= 0");
  if (opt.debug_stop > 0 && (k != 1 || opt.phase2 || opt.schedule != 0))
    return fail(WBPR_EINVAL, "debug_stop needs a single-instance vertex-centric phase-1 solve");
  if (opt.tiny_mode == 0 && k == 1 && !build_only && opt.layout == WBPR_LAYOUT_BCSR && opt.schedule == 0 &&
      !opt.phase2 && opt.trace_rounds <= 0 && opt.gap_mode == 0 && opt.push_mode == 1 && opt.debug_stop == 0 &&
      opt.grid_blocks == 0 && opt.bfs_mode == 1 && !opt.l2_persist && tiny_fits(n, m))
    return solve_tiny(g, s_h[0], t_h[0], opt, W, bitmap, flow_out, cut_out, stats, st);
  const long long launches0 = launch_count();
  Events E;
  CK(E.create());
  SyncOnExit guard{st};
  guard.armed = true;
  CK(cudaEventRecord(E.ev[0], st));

  const int64_t* ro = g->row_offsets;
  const int32_t* col = g->col;
  const int32_t* cap = g->cap;
  if (g->on_host) {
    CK(cudaMemcpyAsync(at<int64_t>(ws, L.in_row), ro, 8 * (n + 1), cudaMemcpyHostToDevice, st));
    if (m > 0) {
      CK(cudaMemcpyAsync(at<int32_t>(ws, L.in_col), col, 4 * m, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(at<int32_t>(ws, L.in_cap), cap, 4 * m, cudaMemcpyHostToDevice, st));
    }
    ro = at<int64_t>(ws, L.in_row);
    col = at<int32_t>(ws, L.in_col);
    cap = at<int32_t>(ws, L.in_cap);
  }
  { k_init_ctrl<<<1, 256, 0, st>>>(W.ctrl); note_launch(); }
  long long* d_s = at<long long>(ws, L.inst_s);
  long long* d_t = at<long long>(ws, L.inst_t);
  int64_t* d_vb = at<int64_t>(ws, L.vbase);
  // (pinned upload area: [s | t | vbase | group descriptors]; read_ctrl's download uses the
  //  start of the buffer only after the stream synchronised)
  const size_t up_s = 0, up_t = 8 * (size_t)k, up_vb = 16 * (size_t)k, up_gd = 24 * (size_t)k + 8;
  g_pin.get(up_gd + sizeof(GroupDesc) * (size_t)kMaxGroups + sizeof(Ctrl) + 16 * (size_t)k + 64);
  CK(upload(d_s, s_h, 8 * k, up_s, st));
  CK(upload(d_t, t_h, 8 * k, up_t, st));
  CK(upload(d_vb, vbase_h, 8 * (k + 1), up_vb, st));
  uint8_t* term = at<uint8_t>(ws, L.term);
  CK(cudaMemsetAsync(term, 0, n, st));
  { k_terms<<<(k + 255) / 256, 256, 0, st>>>(term, d_s, d_t, k); note_launch(); }
  CK(cudaGetLastError());

  int Mf = 0;
  int64_t selfloops = 0, bad_edge = -1;
  s = build_residual(W, ro, col, cap, opt.layout, di.num_sms, d_vb, k, Mf, selfloops, bad_edge, st);
  if (stats) { memset(stats, 0, sizeof(*stats)); stats->bad_edge_index = bad_edge; stats->n = n; stats->m = m; }
  if (s) return s;
  CK(cudaEventRecord(E.ev[1], st));
  if (build_only) {
    Ctrl cb;
    s = read_ctrl(W.ctrl, cb, st);
    if (s) return s;
    const int M = opt.layout == WBPR_LAYOUT_BCSR ? cb.M : 2 * Mf;
    register_view(W, opt.layout, M, opt.layout == WBPR_LAYOUT_BCSR ? cb.M : Mf);
    if (cb.overflow == 1) return fail(WBPR_EOVERFLOW, "merged capacity exceeds INT32_MAX");
    if (cb.overflow == 2) return fail(WBPR_EINTERNAL, "reverse arc not found while building mate[]");
    if (stats) {
      stats->M = M; stats->self_loops_ignored = selfloops;
      float ms = 0; cudaEventElapsedTime(&ms, E.ev[0], E.ev[1]); stats->build_ms = ms; stats->total_ms = ms;
      stats->kernel_launches = launch_count() - launches0;
    }
    return WBPR_OK;
  }

  SolveParams P{};
  P.ctrl = W.ctrl;
  P.n = (int)n; P.k = k; P.layout = opt.layout; P.M = 0; P.Mf = Mf;
  P.off = at<int>(ws, L.off);
  P.seg = at<int2>(ws, L.seg);
  P.arc = at<int2>(ws, L.regC);
  P.mate = at<int>(ws, L.regB);
  P.roff = at<int>(ws, L.roff);
  P.rarc = at<int2>(ws, L.regC + 8 * (size_t)m);
  P.bcf = at<int>(ws, L.regB);
  P.h = at<int>(ws, L.h);
  P.e = at<long long>(ws, L.e);
  P.term = term;
  P.deact = at<uint8_t>(ws, L.deact);
  P.q[0] = at<int>(ws, L.q0); P.q[1] = at<int>(ws, L.q1);
  P.hq[0] = at<HugeRec>(ws, L.hq0); P.hq[1] = at<HugeRec>(ws, L.hq1);
  P.hc[0] = at<int2>(ws, L.hc0); P.hc[1] = at<int2>(ws, L.hc1);
  P.hist = at<int>(ws, L.hist);
  P.aring = at<int2>(ws, L.aring);
  P.inq = at<int>(ws, L.inq);
  P.hs = at<int2>(ws, L.hs);
  P.src = d_s; P.snk = d_t;
  P.max_rounds = opt.max_rounds > 0 ? opt.max_rounds : 10 * n + 1000;
  P.gr_beta = opt.gr_beta;
  P.gap_mode = opt.gap_mode;
  P.push_mode = opt.push_mode;
  P.bfs_mode = opt.bfs_mode;
  P.small_mode = opt.small_mode;
  P.schedule = opt.schedule;
  P.phase2 = opt.phase2;
  P.trace_rounds = opt.trace_rounds > 0 ? opt.trace_rounds : 0;
  P.trace = P.trace_rounds ? at<TraceRec>(ws, L.trace) : nullptr;
  P.h1 = at<int>(ws, L.h1);
  P.gr_gamma = opt.gr_gamma;
  P.deadline_ns_rel = (unsigned long long)opt.timeout_ms * 1000000ull;
  P.debug_stop = opt.debug_stop;
  int occ = di.occ[opt.layout];
  if (occ < 1) return fail(WBPR_ECUDA, "solve kernel cannot be resident on this device");
  int blocks = di.num_sms * occ;
  if (opt.grid_blocks > 0 && opt.grid_blocks < blocks) blocks = opt.grid_blocks;
  else if (opt.grid_blocks == 0) {
    // auto: tiny graphs are phase-latency bound and a grid barrier over 296 CTAs costs more
    // than the work of a phase: one CTA up to kSlotsPerCta residual slots (C1), one CTA per
    // 2048 slots below the full grid (measured on C1, R-MAT-14, 128^2 grids, profiles/r1)
    const int64_t slots = n + 2 * m;
    const int64_t want = slots <= kSlotsPerCta ? 1 : slots / 2048 + 1;
    if (want < blocks) blocks = (int)want;
  }

  // ---- solver groups (A10): independent instances get disjoint CTA groups of the
  // persistent grid, sized by their edge counts, each with its own barrier and state
  std::vector<GroupDesc> groups;
  {
    int G = 1;
    if (k > 1) {
      G = opt.batch_groups > 0 ? opt.batch_groups : 1;
      G = std::max(1, std::min(G, std::min(k, std::min(blocks, kMaxGroups))));
    }
    std::vector<int64_t> eoff(k + 1, 0);
    if (G > 1) {
      // edge offsets at the instance boundaries: row_offsets[vbase[i]]
      if (g->on_host) {
        for (int i = 0; i <= k; ++i) eoff[i] = g->row_offsets[vbase_h[i]];
      } else {
        for (int i = 0; i <= k; ++i)
          CK(cudaMemcpyAsync(&eoff[i], ro + vbase_h[i], 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
    }
    const int64_t mtot = std::max<int64_t>(1, eoff[k] - eoff[0]);
    // contiguous instance ranges with balanced edge counts
    std::vector<int> cut(G + 1, 0);
    cut[G] = k;
    for (int gi = 1; gi < G; ++gi) {
      int64_t target = eoff[0] + mtot * gi / G;
      int i = cut[gi - 1] + 1;
      while (i < k - (G - gi) && eoff[i] < target) ++i;
      cut[gi] = i;
    }
    // CTAs proportional to edges, at least one per group
    std::vector<int> nbg(G, 1);
    int left = blocks - G;
    std::vector<std::pair<double, int>> rem;
    for (int gi = 0; gi < G; ++gi) {
      double share = (G == 1) ? blocks : (double)left * (double)(eoff[cut[gi + 1]] - eoff[cut[gi]]) / (double)mtot;
      int add = G == 1 ? blocks - 1 : (int)share;
      nbg[gi] += add;
      rem.push_back({share - add, gi});
    }
    int used = 0;
    for (int gi = 0; gi < G; ++gi) used += nbg[gi];
    std::sort(rem.begin(), rem.end(), [](auto& a, auto& b) { return a.first > b.first; });
    for (int r = 0; used < blocks && r < (int)rem.size(); ++r, ++used) nbg[rem[r].second]++;
    int b0 = 0;
    int64_t hub0 = 0;
    for (int gi = 0; gi < G; ++gi) {
      GroupDesc d{};
      d.b0 = b0; d.nb = nbg[gi]; d.i0 = cut[gi]; d.i1 = cut[gi + 1];
      d.vlo = (int)vbase_h[d.i0]; d.vhi = (int)vbase_h[d.i1]; d.hub0 = (int)hub0;
      const int64_t mg = G == 1 ? m : eoff[d.i1] - eoff[d.i0];
      hub0 += 2 * mg / kMinChunk + 64;
      b0 += d.nb;
      groups.push_back(d);
    }
    blocks = b0;
    CK(upload(at<GroupDesc>(ws, L.gdesc), groups.data(), sizeof(GroupDesc) * groups.size(), up_gd, st));
    CK(cudaMemsetAsync(at<GroupCtrl>(ws, L.gctrl), 0, sizeof(GroupCtrl) * groups.size(), st));
    P.groups = at<GroupDesc>(ws, L.gdesc);
    P.gctrl = at<GroupCtrl>(ws, L.gctrl);
    P.ngroups = (int)groups.size();
    if (P.ngroups > 1) {
      P.trace = nullptr; P.trace_rounds = 0;
      P.gap_mode = 0;   // the online gap histogram is indexed by height: one solver only
    }
  }
  // Keep the label array h[] (the random-gather target of every scan and BFS step)
  // resident in L2: a persisting access-policy window over h for the solve launch.
  bool window = false;
  {
    int dev = 0, maxp = 0, maxw = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    size_t hb = sizeof(int) * (size_t)n;
    if (maxp > 0 && maxw > 0 && opt.l2_persist) {
      size_t lim = std::min((size_t)maxp, hb);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
      cudaStreamAttrValue v{};
      v.accessPolicyWindow.base_ptr = P.h;
      v.accessPolicyWindow.num_bytes = std::min((size_t)maxw, hb);
      v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)lim / (float)v.accessPolicyWindow.num_bytes);
      v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      window = cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
      cudaGetLastError();
    }
  }
  if (P.trace) CK(cudaMemsetAsync(P.trace, 0, sizeof(TraceRec) * (size_t)kTraceWarps * P.trace_rounds, st));
  CK(launch_solve(P, blocks, kSolveThreads, st));
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_traces[ws] = TraceInfo{P.trace, P.trace_rounds, blocks * (kSolveThreads / 32)};
  }
  if (window) {
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    cudaGetLastError();
  }
  CK(cudaEventRecord(E.ev[2], st));

  // the cut bitmap is always built (in queue scratch when the caller wants none or wants it on
  // the host): the certificate looks the sides up in it (n/8 bytes instead of the labels);
  // q0 holds the exported AVQ of debug_stop solves, so a bitmap nobody asked for goes to q1
  uint32_t* dbm = bitmap;
  if (bitmap && g->on_host) dbm = reinterpret_cast<uint32_t*>(at<int>(ws, L.q0));
  if (!bitmap) dbm = reinterpret_cast<uint32_t*>(at<int>(ws, L.q1));
  long long* d_flow = at<long long>(ws, L.inst_flow);
  long long* d_cut = at<long long>(ws, L.inst_cut);
  {
    SolveParams PX = P;
    if (opt.phase2) PX.h = P.h1;   // the cut comes from the phase-1 labels
    extract_results(PX, ro, col, cap, m, dbm, d_vb, k, d_flow, d_cut, di.num_sms, st);
  }
  CK(cudaGetLastError());
  std::vector<long long> hf(k), hc(k);
  // results through the pinned scratch (its upload area is free once the uploads completed,
  // which the stream order guarantees before these copies run)
  char* pin = g_pin.get(sizeof(Ctrl) + 16 * (size_t)k + 64);
  Ctrl c;
  if (pin) {
    CK(cudaMemcpyAsync(pin + sizeof(Ctrl), d_flow, 8 * k, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pin + sizeof(Ctrl) + 8 * k, d_cut, 8 * k, cudaMemcpyDeviceToHost, st));
  } else {
    CK(cudaMemcpyAsync(hf.data(), d_flow, 8 * k, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), d_cut, 8 * k, cudaMemcpyDeviceToHost, st));
  }
  if (bitmap && g->on_host)
    CK(cudaMemcpyAsync(bitmap, dbm, 4 * ((n + 31) / 32), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(E.ev[3], st));
  if (pin) CK(cudaMemcpyAsync(pin, W.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  else CK(cudaMemcpyAsync(&c, W.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  guard.armed = false;
  if (pin) {
    memcpy(&c, pin, sizeof(Ctrl));
    memcpy(hf.data(), pin + sizeof(Ctrl), 8 * k);
    memcpy(hc.data(), pin + sizeof(Ctrl) + 8 * k, 8 * k);
  }

  const int M = opt.layout == WBPR_LAYOUT_BCSR ? c.M : 2 * Mf;
  register_view(W, opt.layout, M, opt.layout == WBPR_LAYOUT_BCSR ? c.M : Mf);
  if (opt.debug_stop > 0) {
    std::lock_guard<std::mutex> lk(g_mu);
    wbpr_residual& v = g_views[W.base];
    v.avq = at<int32_t>(ws, L.q0);
    v.avq_len = (int64_t)c.dbg_qn + c.dbg_hn;
    v.excess_total = c.excess_total;
  }
  if (c.overflow == 1) return fail(WBPR_EOVERFLOW, "merged capacity exceeds INT32_MAX");
  if (c.overflow == 2) return fail(WBPR_EINTERNAL, "reverse arc not found while building mate[]");
  long long F = 0, C = 0;
  bool cert = true;
  for (int i = 0; i < k; ++i) {
    F += hf[i]; C += hc[i];
    if (hf[i] != hc[i]) cert = false;
    if (flow_out) flow_out[i] = hf[i];
    if (cut_out) cut_out[i] = hc[i];
  }
  if (stats) {
    stats->flow_value = F;
    stats->cut_capacity = C;
    stats->M = M;
    stats->rounds = c.stats[ST_ROUNDS];
    stats->global_relabels = c.stats[ST_GRS];
    stats->bfs_levels = c.stats[ST_BFS_LEVELS];
    stats->pushes = c.stats[ST_PUSHES];
    stats->relabels = c.stats[ST_RELABELS];
    stats->arcs_scanned = c.stats[ST_ARCS];
    stats->bfs_arcs_scanned = c.stats[ST_BFS_ARCS];
    stats->compaction_candidates = c.stats[ST_CAND];
    stats->avq_total = c.stats[ST_AVQ];
    stats->gap_lifts = c.stats[ST_GAPLIFT];
    stats->self_loops_ignored = selfloops;
    stats->excess_total = c.excess_total;
    float ms;
    cudaEventElapsedTime(&ms, E.ev[0], E.ev[1]); stats->build_ms = ms;
    cudaEventElapsedTime(&ms, E.ev[1], E.ev[2]); stats->solve_ms = ms;
    cudaEventElapsedTime(&ms, E.ev[2], E.ev[3]); stats->extract_ms = ms;
    cudaEventElapsedTime(&ms, E.ev[0], E.ev[3]); stats->total_ms = ms;
    stats->grid_blocks = blocks;
    stats->block_threads = kSolveThreads;
    stats->kernel_launches = launch_count() - launches0;
    stats->t_barrier_ns = c.stats[ST_COUNT - 3];
    stats->t_flush_ns = c.stats[ST_COUNT - 2];
    stats->t_round_ns = c.stats[ST_COUNT - 1];
    for (int i = 0; i < kPhBuckets; ++i) { stats->phase_ns[i] = c.phase_ns[i]; stats->phase_count[i] = c.phase_cnt[i]; }
    stats->bfs_arcs_bottom_up = c.stats[ST_BFS_BU];
  }
  if (c.status == DS_NOTCONVERGED) return fail(WBPR_ENOTCONVERGED, "round cap exceeded");
  if (c.abort) return fail(WBPR_ENOTCONVERGED, "device watchdog timeout");
  if (opt.debug_stop > 0) return WBPR_OK;   // stopped mid-solve: no certificate (wbpr.h)
  if (!cert) return fail(WBPR_EINTERNAL, "certificate failed: cut capacity != flow value");
  // Paper's termination identity: e(s) + e(t) >= Excess_total at the end.
  if (F != c.excess_total) return fail(WBPR_EINTERNAL, "Excess_total bookkeeping disagrees with e(t)");
  return WBPR_OK;
}

}  // namespace

extern "C" {

wbpr_status wbpr_default_options(wbpr_options* opt) {
  if (!opt) return fail(WBPR_EINVAL, "NULL options");
  memset(opt, 0, sizeof(*opt));
  opt->layout = WBPR_LAYOUT_BCSR;
  opt->gr_beta = 0.5f;
  opt->gap_mode = 0;
  opt->max_rounds = 0;
  opt->grid_blocks = 0;
  opt->timeout_ms = 120000;
  opt->push_mode = 1;
  opt->gr_gamma = 1.0f;
  opt->l2_persist = 0;
  opt->bfs_mode = 1;
  opt->small_mode = 1;
  opt->batch_groups = 0;
  return WBPR_OK;
}

wbpr_status wbpr_workspace_size(int64_t n, int64_t m, int32_t k, const wbpr_options* opt, size_t* bytes) {
  if (!bytes) return fail(WBPR_EINVAL, "NULL bytes");
  if (n < 2 || m < 0 || k < 1) return fail(WBPR_EINVAL, "bad sizes");
  if (n >= INT32_MAX || 2 * m >= INT32_MAX) return fail(WBPR_EOVERFLOW, "size beyond int32 indexing");
  wbpr_options o = resolve(opt);
  *bytes = make_layout(n, m, k, o.layout, o.trace_rounds).total;
  return WBPR_OK;
}

wbpr_status wbpr_maxflow_solve(const wbpr_csr* g, int64_t s, int64_t t, const wbpr_options* opt, void* workspace,
                               size_t ws_bytes, uint32_t* cut_bitmap, wbpr_stats* stats, void* stream) {
  if (!g) return fail(WBPR_EINVAL, "graph is NULL");
  if (s < 0 || t < 0 || s >= g->n || t >= g->n) return fail(WBPR_EINVAL, "s or t out of range");
  if (s == t) return fail(WBPR_EINVAL, "s == t");
  int64_t vb[2] = {0, g->n};
  return solve_impl(g, 1, vb, &s, &t, opt, workspace, ws_bytes, cut_bitmap, nullptr, nullptr, stats,
                    (cudaStream_t)stream, false);
}

wbpr_status wbpr_maxflow_solve_batch(const wbpr_csr* g, int32_t k, const int64_t* vbase, const int64_t* s,
                                     const int64_t* t, const wbpr_options* opt, void* workspace, size_t ws_bytes,
                                     uint32_t* cut_bitmap, int64_t* flow_out, int64_t* cutcap_out, wbpr_stats* stats,
                                     void* stream) {
  if (!vbase || !s || !t) return fail(WBPR_EINVAL, "NULL batch arrays");
  return solve_impl(g, k, vbase, s, t, opt, workspace, ws_bytes, cut_bitmap, flow_out, cutcap_out, stats,
                    (cudaStream_t)stream, false);
}

wbpr_status wbpr_build_residual(const wbpr_csr* g, const wbpr_options* opt, void* workspace, size_t ws_bytes,
                                wbpr_stats* stats, void* stream) {
  if (!g) return fail(WBPR_EINVAL, "graph is NULL");
  int64_t vb[2] = {0, g->n};
  int64_t s = 0, t = g->n - 1;
  return solve_impl(g, 1, vb, &s, &t, opt, workspace, ws_bytes, nullptr, nullptr, nullptr, stats,
                    (cudaStream_t)stream, true);
}

wbpr_status wbpr_bipartite_workspace_size(int64_t nL, int64_t nR, int64_t E, const wbpr_options* opt, size_t* bytes) {
  if (nL < 0 || nR < 0 || E < 0) return fail(WBPR_EINVAL, "bad sizes");
  return wbpr_workspace_size(nL + nR + 2, nL + E + nR, 1, opt, bytes);
}

wbpr_status wbpr_bipartite_match(int64_t nL, int64_t nR, int64_t E, const int32_t* l, const int32_t* r,
                                 const wbpr_options* opt_in, void* workspace, size_t ws_bytes, int32_t* match_of_left,
                                 int64_t* size_out, wbpr_stats* stats, void* stream) {
  if (nL < 0 || nR < 0 || E < 0) return fail(WBPR_EINVAL, "bad sizes");
  if (E > 0 && (!l || !r)) return fail(WBPR_EINVAL, "NULL edge arrays");
  if (!workspace) return fail(WBPR_EINVAL, "workspace is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  wbpr_options opt = resolve(opt_in);
  const int64_t n = nL + nR + 2, m = nL + E + nR;
  if (2 * m >= INT32_MAX || n >= INT32_MAX) return fail(WBPR_EOVERFLOW, "size beyond int32 indexing");
  Layout L = make_layout(n, m, 1, opt.layout, opt.trace_rounds);
  if (ws_bytes < L.total) return fail(WBPR_ENOMEM, "workspace too small: need " + std::to_string(L.total) + " bytes");
  DevInfo di;
  wbpr_status s = dev_info(di);
  if (s) return s;
  Ctrl* ctrl = at<Ctrl>(workspace, L.ctrl);
  int* deg = at<int>(workspace, L.deg);
  int* cursor = at<int>(workspace, L.cursor);
  int64_t* ro = at<int64_t>(workspace, L.in_row);
  int32_t* col = at<int32_t>(workspace, L.in_col);
  int32_t* cap = at<int32_t>(workspace, L.in_cap);
  { k_init_ctrl<<<1, 256, 0, st>>>(ctrl); note_launch(); }
  bip_validate(nL, nR, E, l, r, deg, cursor, ctrl, di.num_sms, st);
  CK(cudaGetLastError());
  Ctrl c;
  s = read_ctrl(ctrl, c, st);
  if (s) return s;
  if (c.bad_edge != LLONG_MAX) {
    if (stats) { memset(stats, 0, sizeof(*stats)); stats->bad_edge_index = c.bad_edge; }
    return fail(WBPR_EINVAL, "edge " + std::to_string(c.bad_edge) + " has an id outside its side");
  }
  bip_build(nL, nR, E, l, r, ro, col, cap, deg, cursor, at<int>(workspace, L.scan_part), di.num_sms, st);
  CK(cudaGetLastError());
  wbpr_csr g{n, m, ro, col, cap, 0};
  int64_t vb[2] = {0, n};
  int64_t sv = 0, tv = n - 1;
  int64_t F = 0;
  s = solve_impl(&g, 1, vb, &sv, &tv, &opt, workspace, ws_bytes, nullptr, &F, nullptr, stats, st, false);
  if (s) return s;
  SolveParams P{};
  P.layout = opt.layout;
  P.off = at<int>(workspace, L.off);
  P.seg = at<int2>(workspace, L.seg);
  P.arc = at<int2>(workspace, L.regC);
  P.roff = at<int>(workspace, L.roff);
  P.rarc = at<int2>(workspace, L.regC + 8 * (size_t)m);
  P.bcf = at<int>(workspace, L.regB);
  if (match_of_left && nL > 0) {
    bip_extract(P, nL, nR, match_of_left, di.num_sms, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
  }
  if (size_out) *size_out = F;
  return WBPR_OK;
}

wbpr_status wbpr_residual_view(const void* workspace, wbpr_residual* view) {
  if (!workspace || !view) return fail(WBPR_EINVAL, "NULL argument");
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_views.find(workspace);
  if (it == g_views.end()) return fail(WBPR_EINVAL, "no residual has been built in this workspace");
  *view = it->second;
  return WBPR_OK;
}

wbpr_status wbpr_trace_view(const void* workspace, const void** records, int64_t* rounds, int32_t* warps) {
  if (!workspace || !records || !rounds || !warps) return fail(WBPR_EINVAL, "NULL argument");
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_traces.find(workspace);
  if (it == g_traces.end() || !it->second.ptr) return fail(WBPR_EINVAL, "no traced solve in this workspace");
  *records = it->second.ptr;
  *rounds = it->second.rounds;
  *warps = it->second.warps;
  return WBPR_OK;
}

wbpr_status wbpr_barrier_cost(int32_t grid_blocks, int32_t iters, double* ns_per_phase, void* stream) {
  if (!ns_per_phase || iters < 1) return fail(WBPR_EINVAL, "bad arguments");
  DevInfo di;
  wbpr_status s = dev_info(di);
  if (s) return s;
  int blocks = di.num_sms * std::max(1, di.occ[0]);
  if (grid_blocks > 0 && grid_blocks < blocks) blocks = grid_blocks;
  CK(barrier_probe(blocks, iters, ns_per_phase, (cudaStream_t)stream));
  return WBPR_OK;
}

const char* wbpr_status_string(wbpr_status st) {
  switch (st) {
    case WBPR_OK: return "WBPR_OK";
    case WBPR_EINVAL: return "WBPR_EINVAL";
    case WBPR_EOVERFLOW: return "WBPR_EOVERFLOW";
    case WBPR_ENOMEM: return "WBPR_ENOMEM";
    case WBPR_ECUDA: return "WBPR_ECUDA";
    case WBPR_ENOTCONVERGED: return "WBPR_ENOTCONVERGED";
    case WBPR_EINTERNAL: return "WBPR_EINTERNAL";
    case WBPR_ENOTIMPL: return "WBPR_ENOTIMPL";
    default: return "WBPR_UNKNOWN";
  }
}

const char* wbpr_last_error(void) { return g_err.c_str(); }

const char* wbpr_version(void) { return "wbpr 0.1 sm_100a"; }

}  // extern "C"
