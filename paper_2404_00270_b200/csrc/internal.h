// internal.h — workspace layout and device control block shared by the host
// orchestration (api.cu) and the kernels.  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace wbpr {

#ifndef WBPR_CHUNK
#define WBPR_CHUNK 1024
#endif
constexpr int kChunk = WBPR_CHUNK; // slots per warp task of a BFS level; vertices with more slots are "huge"
#ifndef WBPR_RCHUNK
#define WBPR_RCHUNK 512   // measured: 512 best on C5 (1024 / 256 slower or equal)
#endif
constexpr int kRChunk = WBPR_RCHUNK;   // slots per warp task of a push/relabel round
constexpr int kMinChunk = kChunk < kRChunk ? kChunk : kRChunk;
constexpr int kSortTile = 4096;    // CTA shared-memory sort tile (64-bit keys)
constexpr int kScanTile = 4096;    // elements per scan tile
constexpr int kMaxInst = 1 << 20;  // batch instances

// Vertex terminal flags (term[v])
constexpr uint8_t kSource = 1;
constexpr uint8_t kSink = 2;

// Per-phase counters, triple-buffered by phase parity (see solve.cu).
struct Ring {
  int qn;                   // appended normal queue entries
  int hn;                   // appended huge vertices
  int hc;                   // appended huge chunk tasks
  unsigned work;            // relabel work (slots scanned by relabels), saturating
  int kind;                 // PhaseKind of the phase that used this slot
  unsigned fedges;          // BFS: residual slots of the vertices appended to the next frontier
  int maxdeg;               // largest degree among the appended vertices
  int pad;
};

// What the last CTA to arrive at a grid barrier publishes for everyone (one 16-B
// release store; waiters poll it with 16-B acquire loads).
struct __align__(16) Bcast {
  unsigned gen;
  int qn;
  int hc;
  unsigned flags;   // bit 0: a global relabel is due; bit 1: next BFS level bottom-up;
                    // bit 2: run the next phases in the small-frontier CTA mode;
                    // bit 3: an online gap was found (lift phase before the next round)
};

enum PhaseKind { PK_NONE = 0, PK_ROUND = 1, PK_GR_RESET = 2, PK_BFS = 3, PK_COMPACT = 4, PK_PREFLOW = 5, PK_GAP = 6,
                 PK_ABFS = 7 };
// phase-time buckets (Ctrl::phase_ns / phase_cnt): the PhaseKinds, plus
constexpr int kPhBfsUp = 8;     // bottom-up BFS levels (PK_BFS counts the top-down ones)
constexpr int kPhSmall = 9;     // small-frontier CTA-mode spans (CTA 0 alone)
constexpr int kPhBuckets = 10;

// Global-relabel policy state, written only by the last CTA to arrive at a barrier.
struct GrPolicy {
  unsigned long long work_since_gr;
  unsigned long long t_gr_start;
  unsigned long long t_after_gr;
  unsigned long long gr_time;
  unsigned long long bfs_seen_edges;   // slots of the vertices labelled so far in this GR
  unsigned long long prev_reached;     // slots labelled by the previous GR (0 = none yet)
  unsigned long long t_release;        // globaltimer at the last barrier release (phase timing)
  int bfs_bottom_up;                   // direction of the current BFS level
  int bfs_bottom_up_prev;              // direction of the BFS level now running (phase timing)
};

// Huge-vertex record for one round: chunk tasks fold their partial minima into
// `best` and the last chunk (done == nchunks) performs the push or relabel.
struct HugeRec {
  unsigned long long best;  // (h << 32) | slot
  long long spent;          // discharge: excess reserved by the chunks
  long long pushed;         // discharge: excess actually pushed by the chunks
  int u;
  int nchunks;
  int done;
  int pad;
};

enum StatIdx {
  ST_ROUNDS = 0, ST_GRS, ST_BFS_LEVELS, ST_PUSHES, ST_RELABELS, ST_ARCS, ST_BFS_ARCS,
  ST_CAND, ST_AVQ, ST_GAPLIFT, ST_SMALL_PHASES, ST_SMALL_ENTRIES,
  ST_BFS_BU,   // residual slots read by bottom-up BFS levels (ST_BFS_ARCS counts both directions)
  ST_COUNT = 16
};

enum DevStatus { DS_OK = 0, DS_NOTCONVERGED = 1, DS_TIMEOUT = 2, DS_INTERNAL = 3 };

// Hand-off record of the small-frontier mode (CTA 0 runs phases alone; the other
// CTAs wait on `epoch` and resume the grid loop from this state).
struct Resume {
  unsigned epoch;
  int state;        // next main-loop state
  int qn, hc;       // counts of the queue the next phase reads
  int cur, fb, level;
  int flags;        // Bcast flags for the resumed phase (bit 3: gap lift pending)
  long long rounds;
};

// Per-group solver state (A10): every solver group (one instance, several instances,
// or the whole batch) has its own barrier, phase counters, GR policy and hand-off record.
struct GroupCtrl {
  GridBarrier bar;
  int pad_bar[2];
  Bcast bc;
  Ring ring[3];
  GrPolicy pol;
  Resume res;
  int small_hn, small_hc;  // huge appends made in the small mode
  int gap_level;           // online gap: lowest emptied level seen since the last check (A6)
  int gap_pending;         // the gap level the next lift phase uses
  int nhs;                 // entries of the static huge-chunk list
  int pad[3];
  // asynchronous GR continuation (bfs_mode 3): ring head / tail / pending entries, each on
  // its own 128-B line
  int aq_head[32];
  int aq_tail[32];
  int aq_pending[32];
};

// Host-computed partition of the persistent grid into solver groups.
struct GroupDesc {
  int b0, nb;     // CTAs [b0, b0 + nb)
  int i0, i1;     // instances [i0, i1)
  int vlo, vhi;   // vertices [vlo, vhi)
  int hub0;       // offset of the group's slice of the huge-vertex arrays
  int pad;
};
constexpr int kMaxGroups = 1024;

// Device control block at the start of the workspace.
struct Ctrl {
  int abort;
  int status;
  long long excess_total;
  long long stats[ST_COUNT];
  // build info
  long long bad_edge;     // first offending edge index (min), LLONG_MAX if none
  int bad_rows;           // row offsets malformed
  int overflow;           // merged capacity > INT32_MAX
  int maxlen;             // longest build segment
  int M;                  // residual slots (BCSR) / forward arcs (RCSR)
  int Mr;                 // RCSR reverse entries
  int selfloops;
  int hub_chunks;         // build scratch counter
  int sort_items;         // build scratch counter
  int sort_items_med;     // build scratch counter
  int mlist_w, mlist_c;   // build: vertices merged by a warp / by a CTA
  int maxlen_out;         // build: longest input row
  int any_unsorted;       // build: some input row is not column-sorted (else the row sort is skipped)
  int bigcap;             // build: some merged BCSR capacity exceeds INT32_MAX / 2 (pair-sum check needed)
  int dbg_qn, dbg_hn;     // debug_stop: AVQ entries / hub vertices exported after the stopping GR
  long long phase_ns[kPhBuckets];    // solve: barrier-release-to-release time per phase kind
  long long phase_cnt[kPhBuckets];
};

// Per-warp workload trace record (NEXT #3): one per warp per traced round.
struct TraceRec {
  int round, warp;
  unsigned busy_ns;   // time from the round's start to the warp finishing its tasks
  int tasks;          // queue tasks (VC) / active vertices (TC) the warp processed
  int slots, pushes, relabels, schedule;
};
constexpr int kTraceWarps = 16384;   // trace capacity per round (>= any persistent grid)

// Byte offsets of every region of a workspace (all 256-B aligned).
struct Layout {
  int64_t n, m, k, H;       // H = 2m half-arcs (BCSR) ; RCSR uses m + m
  int32_t layout;
  size_t ctrl, inst_s, inst_t, inst_flow, inst_cut, vbase;
  size_t in_row, in_col, in_cap;           // staging copy of a host CSR
  size_t h, e, term, deact, deg, cursor, off, soff, roff, rsoff, h1, seg;
  size_t q0, q1, hq0, hq1, hc0, hc1, hist, hs, aring, inq;
  size_t scan_part;
  size_t regA, regB, regC;                 // build / residual regions
  size_t regD;                             // BCSR build: slot of every out-half-arc (4m B)
  size_t trace;                            // per-warp trace records
  size_t gdesc, gctrl;                     // solver groups
  size_t bcap0;                            // offset inside regB of cap0
  size_t total;
};

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

inline Layout make_layout(int64_t n, int64_t m, int64_t k, int32_t layout, int32_t trace_rounds = 0) {
  Layout L{};
  L.n = n; L.m = m; L.k = k; L.layout = layout;
  L.H = 2 * m;
  const int64_t H = L.H;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
  L.ctrl = take(sizeof(Ctrl));
  L.inst_s = take(8 * k); L.inst_t = take(8 * k); L.inst_flow = take(8 * k); L.inst_cut = take(8 * k);
  L.vbase = take(8 * (k + 1));
  L.in_row = take(8 * (n + 1)); L.in_col = take(4 * m + 4); L.in_cap = take(4 * m + 4);
  L.h = take(4 * n); L.e = take(8 * n); L.term = take(n); L.deact = take(n); L.h1 = take(4 * n);
  L.deg = take(4 * n + 4); L.cursor = take(4 * n + 4);
  L.off = take(4 * (n + 1)); L.soff = take(4 * (n + 1)); L.roff = take(4 * (n + 1)); L.rsoff = take(4 * (n + 1));
  L.seg = take(8 * n + 8);   // BCSR: {begin, end} of every vertex segment (gapped layout)
  L.q0 = take(4 * n + 4); L.q1 = take(4 * n + 4);
  int64_t hub = H / kMinChunk + 64 * (k + 1);   // per-group slices (+64 slack each)
  L.hq0 = take(sizeof(HugeRec) * hub); L.hq1 = take(sizeof(HugeRec) * hub);
  L.hc0 = take(8 * (2 * hub + 64)); L.hc1 = take(8 * (2 * hub + 64));
  L.hist = take(4 * (n + 2));
  L.aring = take(8 * (n + 1)); L.inq = take(4 * (n + 1));   // asynchronous GR ring + in-queue flags
  L.hs = take(8 * (2 * hub + 64));
  L.scan_part = take(4 * ((H + 2 + n) / kScanTile + 64));
  L.regA = take(8 * H + 8);
  L.regB = take(8 * H + 1024);
  L.bcap0 = align_up(4 * H + 260);
  L.regC = take(8 * H + 8);
  L.regD = take(layout == 0 ? 4 * m + 8 : 8);
  L.trace = take(sizeof(TraceRec) * (size_t)kTraceWarps * (size_t)(trace_rounds > 0 ? trace_rounds : 0) + 32);
  L.gdesc = take(sizeof(GroupDesc) * kMaxGroups);
  L.gctrl = take(sizeof(GroupCtrl) * kMaxGroups);
  L.total = o;
  return L;
}

// One-CTA fused path for tiny single instances (tiny.cu): limits and launch arguments.
constexpr int kTinyN = 2048;     // vertices
constexpr int kTinyS = 16384;    // half-arcs (2m)
struct TinyArgs {
  const int64_t* ro; const int32_t* col; const int32_t* cap;   // input CSR (device)
  int n, m, s, t;
  int2* seg; int2* arc; int* mate; int* cap0;                  // BCSR in the workspace (residual view)
  int* h; long long* e;
  uint32_t* bitmap;                                            // nullptr: no bitmap
  long long* flow; long long* cut;                             // per-instance results [1]
  Ctrl* ctrl;
  float gr_beta;
  long long max_rounds;
  unsigned long long deadline_ns_rel;
};

// Launch parameters of the persistent solve kernel.
struct SolveParams {
  Ctrl* ctrl;
  int n;                 // vertices (union)
  int k;                 // instances
  int layout;
  int M, Mf;             // slots (BCSR) / forward arcs (RCSR)
  const int* off;        // RCSR forward offsets
  const int2* seg;       // BCSR {begin, end} per vertex (segments may be followed by gaps)
  int2* arc;             // {col, cf}
  const int* mate;       // BCSR
  const int* roff;       // RCSR reverse offsets
  const int2* rarc;      // RCSR {col, fidx}
  int* bcf;              // RCSR backward cf
  int* h;
  long long* e;
  uint8_t* term;
  uint8_t* deact;
  int* h1;               // phase-1 labels (the cut) saved before phase 2
  int phase2;
  TraceRec* trace;       // NEXT #3 per-warp trace (nullptr = off)
  int trace_rounds;
  const GroupDesc* groups;   // solver groups (sorted by b0)
  GroupCtrl* gctrl;
  int ngroups;
  int* q[2];
  HugeRec* hq[2];
  int2* hc[2];
  int* hist;
  int2* aring;           // asynchronous GR: ring cells {seq, vertex} (slice [vlo, vhi) per group)
  int* inq;              // asynchronous GR: 1 while the vertex is queued
  int2* hs;              // static (vertex, chunk) list of all vertices with > kChunk slots
  const long long* src; // sources [k]
  const long long* snk; // sinks [k]
  long long max_rounds;
  float gr_beta;         // GR when relabel work since the last GR >= gr_beta * (n + M)
  float gr_gamma;        // GR when round time since the last GR >= gr_gamma * (last GR time)
  int gap_mode;
  int push_mode;         // 0: one push to the lowest neighbour (Alg. 2); 1: warp-parallel discharge
  int bfs_mode;          // 0: top-down only; 1: direction-optimizing; 2: bottom-up after level 0
  int small_mode;        // 1: phases with small queues run in CTA 0 alone (thread per vertex)
  int schedule;          // 0: vertex-centric (AVQ + warp per vertex, Alg. 2); 1: thread-centric sweeps (Alg. 1)
  unsigned long long deadline_ns_rel;
  int debug_stop;        // > 0: stop right after the compaction that follows the debug_stop-th
                         // global relabel and export the AVQ (tests of the GR labels / AVQ)
};

}  // namespace wbpr
