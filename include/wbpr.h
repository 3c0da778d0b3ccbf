/*
 * wbpr.h — C ABI of libwbpr.so, the B200 (sm_100a) hot path of WBPR
 * ("Engineering A Workload-balanced Push-Relabel Algorithm for Massive Graphs
 * on GPUs", arXiv 2404.00270; PAPER.md in the reference tree).
 *
 * The library solves maximum flow / minimum cut (§2.1) with
 * the vertex-centric lock-free push-relabel loop of Alg. 1 and
 * Alg. 2 over the bidirectional / reversed CSR residual layouts of
 * §3.2, entirely on the device:
 *   A1 residual construction  (BCSR/RCSR; in-lists by segmented sort, reverse-arc index
 *                              from the edge ids carried through the merge)
 *   A2 preflow                (Alg. 1 Step 0)
 *   A3 active-vertex queue    (Alg. 2 lines 1-5)
 *   A4 push/relabel           (Alg. 1 lines 9-21 with the relaxed rule P:187-189,
 *                              one warp per active vertex)
 *   A5 global relabel + termination, A6 gap heuristic
 *   A7 device-resident loop   (one cooperative persistent kernel; no host polling)
 *   A8 flow value e(t) and the canonical min-cut bitmap
 *   A9 bipartite matching wrapper, A10 batches of disjoint instances.
 *
 * Conventions (all entry points):
 *   - Every call returns wbpr_status (0 = OK, < 0 = error) and never aborts the
 *     process.  wbpr_last_error() returns a message for the last failure on the
 *     calling thread.
 *   - Synchronous: work is enqueued on `stream` (a cudaStream_t passed as void*,
 *     NULL = legacy default stream) and results are valid on return.  A BCSR solve
 *     synchronises the stream twice: once after the validation kernels (so a
 *     malformed graph is reported before construction) and once at the end; RCSR
 *     adds two more (its reverse sort is sized from device counts), batch_groups > 1
 *     one more.  On every error return after work was enqueued the stream is
 *     synchronised first, so the caller may free or reuse the workspace at once.
 *   - Host staging: small copies (terminals, instance ranges, results) go through a
 *     per-thread pinned buffer that only grows (never freed while the thread lives),
 *     so a solve never calls cudaFreeHost.
 *   - Ownership: inputs are never written; the workspace is caller-allocated
 *     device memory of at least wbpr_*_workspace_size() bytes (256-B aligned);
 *     the library performs no cudaMalloc inside a solve.  One workspace serves
 *     one solve at a time.
 *   - Limits: vertex ids are int32 (n < 2^31); residual slots M < 2^31 and
 *     2*m < 2^31; capacities are non-negative int32; flows are int64.
 *   - Input rules: self-loops are ignored (counted); parallel edges are summed;
 *     antiparallel edges share one arc pair in BCSR and stay distinct in RCSR;
 *     zero capacities are allowed; rows may list their edges in any order.
 *   - Bitmap: bit v lives in word v>>5 at bit position v&31 (LSB first);
 *     padding bits >= n are 0; bit v = 1 <=> v is on the source side S*, where
 *     S* = V \ {v : v reaches t in the final residual graph} (unique, §8(c)).
 */
#ifndef WBPR_H
#define WBPR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t wbpr_status;
#define WBPR_OK 0
#define WBPR_EINVAL (-1)        /* bad argument or malformed graph (see stats.bad_edge_index) */
#define WBPR_EOVERFLOW (-2)     /* merged capacity > INT32_MAX, or M / 2m >= 2^31 */
#define WBPR_ENOMEM (-3)        /* workspace too small */
#define WBPR_ECUDA (-4)         /* a CUDA runtime error; message in wbpr_last_error() */
#define WBPR_ENOTCONVERGED (-5) /* round cap or watchdog timeout exceeded */
#define WBPR_EINTERNAL (-6)     /* device certificate failed: cut capacity != e(t) */
#define WBPR_ENOTIMPL (-7)

/* Input graph in CSR form.  Edge i of row u is (u, col[i], cap[i]),
 * i in [row_offsets[u], row_offsets[u+1]).  on_host = 0: the three arrays are
 * DEVICE pointers; on_host = 1: HOST pointers (copied into the workspace inside
 * the call, host->device time included in the call). */
typedef struct wbpr_csr {
  int64_t n;                  /* number of vertices, >= 2           */
  int64_t m;                  /* number of edges, >= 0              */
  const int64_t* row_offsets; /* [n+1], row_offsets[0]=0, [n]=m      */
  const int32_t* col;         /* [m], 0 <= col < n                   */
  const int32_t* cap;         /* [m], >= 0                           */
  int32_t on_host;
} wbpr_csr;

#define WBPR_LAYOUT_BCSR 0
#define WBPR_LAYOUT_RCSR 1

typedef struct wbpr_options {
  int32_t layout;        /* WBPR_LAYOUT_BCSR (default) or WBPR_LAYOUT_RCSR     */
  float gr_beta;         /* global relabel when relabel work since the last GR exceeds
                            gr_beta * (n + M) slots, or when the queue empties (P:178,
                            P:374; reading §8(c) #8).  <= 0 -> default 0.5             */
  int32_t gap_mode;      /* 0: gap by exact GR only; 1: + online height histogram (A6) */
  int64_t max_rounds;    /* push/relabel round cap, 0 -> 10*n + 1000             */
  int32_t grid_blocks;   /* persistent grid size, 0 -> all co-resident CTAs             */
  int32_t timeout_ms;    /* device watchdog, 0 -> 120000                                 */
  int32_t push_mode;     /* 0: one push per active vertex per round to its lowest residual
                            neighbour (Alg. 2); 1: warp-parallel discharge: every
                            admissible arc (h(v) < h(u)) of the vertex gets a share of e(u) in
                            the same round (a deviation)                          */
  float gr_gamma;        /* also GR when the time spent in rounds since the last GR reaches
                            gr_gamma x the duration of that GR (balances the two; 0 = off);
                            < 0 -> default 1.0                                               */
  int32_t l2_persist;    /* 1: persisting L2 access-policy window over the label
                            array h[] for the solve launch (sets the context's persisting-L2
                            limit); 0 (default): off                                                */
  int32_t bfs_mode;      /* global-relabel BFS: 0 top-down only; 1 (default) direction-
                            optimizing (bottom-up levels while the frontier is large);
                            2 bottom-up from the first level (testing); 3 direction-optimizing,
                            and a GR deeper than 32 levels continues as an asynchronous
                            label-correcting BFS (one shared work ring, no level barriers;
                            converges to the same exact distances; measured ~2x slower than
                            the level-synchronous BFS on grids - ring contention - so not
                            the default)                                                     */
  int32_t small_mode;    /* 1 (default): phases whose queue fits one CTA (<= 512 vertices of
                            <= 8 slots) run in CTA 0 alone, one thread per vertex, with
                            block barriers instead of grid barriers; 0: off                 */
  int32_t schedule;      /* 0 (default): vertex-centric - active-vertex queue, one warp per
                            active vertex (Alg. 2, the paper's method); 1: thread-centric -
                            every sweep one thread per vertex tests activity and scans the
                            residual arcs serially (Alg. 1 Step 1, the paper's baseline)     */
  int32_t phase2;        /* 1: after the maximum preflow, return the stranded excess to the
                            sources on the device (same loop, terminal roles swapped) so the
                            residual state is a true flow; 0 (default): stop
                            at the maximum preflow (flow value and cut are final there)     */
  int32_t trace_rounds;  /* > 0: record one per-warp workload record (busy time, tasks, slots,
                            pushes, relabels) for each of the first trace_rounds grid rounds
                            (§4.3 Fig. 3; NEXT #3); the workspace grows
                            by trace_rounds x 16384 x 32 B; read with wbpr_trace_view()     */
  int32_t batch_groups;  /* batch solves (A10): number of independent solver groups the
                            persistent grid is split into (contiguous instance ranges, CTAs
                            proportional to edges, each with its own barrier, queues and GR
                            policy); 0 or 1 (default) = one solver for the whole disjoint
                            union (it shares the grid dynamically: on C5 the groups' static
                            CTA shares leave the easy groups' CTAs idle behind the hardest
                            instance, profiles/r1)                                           */
  int32_t debug_stop;    /* testing (single instance, phase 1): > 0 stops the solve right after
                            the active-vertex compaction that follows the debug_stop-th global
                            relabel.  h[] then holds that GR's exact labels (distance to t in
                            G_f, unreached = n), e[] the excess, and the residual
                            view exposes the compacted AVQ (Alg. 2 l.1-4).  The
                            flow value is not final and the certificate is not checked.
                            0 (default): off                                                 */
  int32_t tiny_mode;     /* 0 (default): a single BCSR instance with n <= 2048 vertices and
                            2m <= 16384 half-arcs (C1-sized) runs the whole path - A1
                            construction, preflow, rounds, global relabels, extraction - in ONE
                            launch of ONE CTA with the residual graph in shared memory
                            (tiny.cu); launch- and barrier-latency, not work, bounds such
                            instances.  Same readings and results; options that need the
                            persistent kernel (RCSR, thread-centric, phase 2, traces, online
                            gap, push_mode 0, debug_stop, grid_blocks > 0, bfs_mode != 1,
                            l2_persist) use it instead.
                            1: always the multi-kernel path                                  */
} wbpr_options;

typedef struct wbpr_stats {
  int64_t flow_value;        /* e(t) (sum over instances for a batch)                  */
  int64_t cut_capacity;      /* sum of c over input edges S* -> V\S*                   */
  int64_t n, m, M;           /* vertices, input edges, residual slots                  */
  int64_t rounds;            /* push/relabel rounds (Alg. 2 iterations)                */
  int64_t global_relabels;
  int64_t bfs_levels;        /* BFS levels over all global relabels                    */
  int64_t pushes, relabels;
  int64_t arcs_scanned;      /* residual slots read by push/relabel scans              */
  int64_t bfs_arcs_scanned;  /* residual slots read by global-relabel BFS              */
  int64_t compaction_candidates; /* vertices examined by full AVQ compactions          */
  int64_t avq_total;         /* sum of |AVQ| over rounds                                */
  int64_t gap_lifts;         /* vertices lifted by the online gap heuristic            */
  int64_t self_loops_ignored;
  int64_t bad_edge_index;    /* first offending edge for EINVAL, else -1               */
  int64_t excess_total;      /* Excess_total at termination              */
  float build_ms, solve_ms, extract_ms, total_ms; /* CUDA-event times on `stream`       */
  int32_t grid_blocks, block_threads;
  int64_t kernel_launches;   /* kernels this call launched (all of them this library's own) */
  int64_t t_barrier_ns, t_flush_ns, t_round_ns; /* CTA 0 time in grid barriers / queue flushes /
                                                   round task loops (globaltimer)             */
  int64_t phase_ns[10];      /* solve time by phase kind, barrier release to release
                                (globaltimer): 0 init, 1 push/relabel rounds, 2 GR label
                                reset, 3 top-down BFS levels, 4 compactions, 5 preflow,
                                6 gap lifts, 7 asynchronous GR continuation, 8 bottom-up
                                BFS levels, 9 small-frontier spans                          */
  int64_t phase_count[10];   /* phases per kind (small-frontier: phases run in CTA mode)  */
  int64_t bfs_arcs_bottom_up; /* the part of bfs_arcs_scanned read by bottom-up levels (a
                                 slot's own {col, cf} + h[col]: 12 B); the rest are top-down
                                 in-arcs (col, mate, cf[mate], h: 16 B) - DESIGN.md §5      */
  int64_t tiny_path;         /* 1: this call ran the one-CTA fused path (tiny_mode)        */
} wbpr_stats;

/* Fill *opt with the defaults above. */
wbpr_status wbpr_default_options(wbpr_options* opt);

/* Bytes of device workspace a solve of a graph with n vertices and m edges needs
 * (k instances for a batch; k = 1 otherwise). */
wbpr_status wbpr_workspace_size(int64_t n, int64_t m, int32_t k, const wbpr_options* opt, size_t* bytes);

/*
 * wbpr_maxflow_solve — maximum flow value and canonical minimum cut of (g, s, t).
 *   cut_bitmap: ceil(n/32) uint32 words, DEVICE (or HOST when g->on_host), caller-owned,
 *               may be NULL.
 *   stats:      HOST, may be NULL.
 * Errors: EINVAL (n < 2, s == t, s/t out of range, cap < 0, col out of range, bad
 * row offsets), EOVERFLOW, ENOMEM, ECUDA, ENOTCONVERGED, EINTERNAL.
 */
wbpr_status wbpr_maxflow_solve(const wbpr_csr* g, int64_t s, int64_t t, const wbpr_options* opt,
                               void* workspace, size_t ws_bytes, uint32_t* cut_bitmap,
                               wbpr_stats* stats, void* stream);

/*
 * wbpr_maxflow_solve_batch — k independent instances given as one disjoint-union
 * CSR: instance i owns vertices [vbase[i], vbase[i+1]) and has terminals s[i], t[i]
 * (HOST arrays).  Edges crossing instance ranges -> EINVAL.  flow_out / cutcap_out:
 * HOST int64[k].  cut_bitmap covers the union graph (instance i = bits
 * [vbase[i], vbase[i+1])).  All instances advance in the same rounds.
 */
wbpr_status wbpr_maxflow_solve_batch(const wbpr_csr* g, int32_t k, const int64_t* vbase,
                                     const int64_t* s, const int64_t* t, const wbpr_options* opt,
                                     void* workspace, size_t ws_bytes, uint32_t* cut_bitmap,
                                     int64_t* flow_out, int64_t* cutcap_out, wbpr_stats* stats,
                                     void* stream);

/* Workspace for wbpr_bipartite_match. */
wbpr_status wbpr_bipartite_workspace_size(int64_t nL, int64_t nR, int64_t E, const wbpr_options* opt,
                                          size_t* bytes);

/*
 * wbpr_bipartite_match — maximum bipartite matching as maximum flow: the
 * network is built on the device with s = 0, left l -> 1+l, right r -> 1+nL+r,
 * t = nL+nR+1, unit capacities; duplicate (l, r) pairs are merged.
 *   l, r:           DEVICE int32[E], 0 <= l < nL, 0 <= r < nR.
 *   match_of_left:  DEVICE int32[nL], written: the matched right id or -1.
 *   size_out:       HOST, the matching size (= max flow value).
 */
wbpr_status wbpr_bipartite_match(int64_t nL, int64_t nR, int64_t E, const int32_t* l, const int32_t* r,
                                 const wbpr_options* opt, void* workspace, size_t ws_bytes,
                                 int32_t* match_of_left, int64_t* size_out, wbpr_stats* stats,
                                 void* stream);

/* Debug/test view of the residual state left in a workspace by the last solve.
 * All pointers are DEVICE pointers into the workspace.  BCSR (gapped): vertex u's
 * segment is slots [seg[2u], seg[2u+1]) of arc/mate/cap0, which span M = 2m slots;
 * segments appear in vertex order and the slots between one segment's end and the next
 * one's begin are unused (they absorb the merged parallel / antiparallel half-arcs, so
 * no counting pass is needed; off = NULL).  arc[p] = {col, cf}; mate[p] = slot of the
 * reverse arc.  RCSR: foff/farc/cap0 (forward), roff/rarc (rarc[q] = {col, flow_idx}),
 * bcf (backward cf per forward arc).  e = excess (int64[n]), h = heights (int32[n],
 * >= n means source side). */
typedef struct wbpr_residual {
  int32_t layout;
  int64_t n, M, Mf;
  const int32_t* off;   /* RCSR forward offsets [n+1]; BCSR: NULL (see seg) */
  const int32_t* arc;   /* int2 pairs: BCSR [M] / RCSR forward [Mf] */
  const int32_t* mate;  /* BCSR [M] */
  const int32_t* cap0;  /* initial cf: BCSR [M] / RCSR forward [Mf] */
  const int32_t* roff;  /* RCSR [n+1] */
  const int32_t* rarc;  /* RCSR int2 [Mf] */
  const int32_t* bcf;   /* RCSR [Mf] */
  const int64_t* e;
  const int32_t* h;
  const int32_t* seg;   /* BCSR: int2 {begin, end} per vertex [n] (gapped segments) */
  const int32_t* avq;   /* debug_stop solves: the compacted active-vertex queue [avq_len]
                           (normal entries, then one entry per hub vertex); else NULL */
  int64_t avq_len;
  int64_t excess_total; /* Excess_total after the last compaction          */
} wbpr_residual;
wbpr_status wbpr_residual_view(const void* workspace, wbpr_residual* view);

/* Construction only (A1): builds the residual layout of g into the workspace
 * and returns; wbpr_residual_view() then exposes it.  Used by the layout parity
 * tests (bit-exact against the definition). */
wbpr_status wbpr_build_residual(const wbpr_csr* g, const wbpr_options* opt, void* workspace,
                                size_t ws_bytes, wbpr_stats* stats, void* stream);

/* Per-warp workload trace of the last solve in `workspace` (when trace_rounds > 0):
 * *records = DEVICE pointer to 32-B records {int round, int warp, uint32 busy_ns, int tasks,
 * int slots, int pushes, int relabels, int schedule} laid out [round][warp];
 * *rounds = traced rounds, *warps = warps of the persistent grid. */
wbpr_status wbpr_trace_view(const void* workspace, const void** records, int64_t* rounds, int32_t* warps);

/* Measurement helper (not part of a solve): the device time of one EMPTY grid-synchronous
 * phase of the persistent solve kernel - the same barrier protocol (one acq_rel arrival per
 * CTA, last-arriver bookkeeping, one 16-B release store, acquire polling) with no work in
 * between, on grid_blocks co-resident CTAs (0 = the full persistent grid), averaged over
 * `iters` phases.  phases x this cost is the latency floor of a solve (the paper's
 * synchronisation overhead on small / long-path graphs).
 * Synchronises `stream`; may allocate 8 B of device memory.  Errors: EINVAL, ECUDA. */
wbpr_status wbpr_barrier_cost(int32_t grid_blocks, int32_t iters, double* ns_per_phase, void* stream);

const char* wbpr_status_string(wbpr_status st);
const char* wbpr_last_error(void);
/* Library version string, e.g. "wbpr 0.1 sm_100a". */
const char* wbpr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WBPR_H */
