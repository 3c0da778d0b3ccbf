// solve.cu — A2-A7: preflow, global relabel + termination, active-vertex queue
// compaction and the vertex-centric push/relabel rounds, as ONE cooperative
// persistent kernel (no host polling; the host synchronises once at the end).
//
// Paper mapping:
//   preflow                      Alg. 1 Step 0
//   outer loop / termination     Alg. 1 P:84 "while e(s)+e(t) < Excess_total", decided only
//                                right after an exact global relabel
//   global relabel               P:108-109: backward BFS from the sink in G_f,
//                                unreached -> |V| (the exact gap); P:182 Excess_total update
//   AVQ scan (compaction)        Alg. 2 lines 1-4, P:343-349 (warp ballot + prefix + one atomic)
//   grid_sync between phases     Alg. 2 line 5
//   tile per active vertex       Alg. 2 "first/second level parallelism": one warp
//                                (tile = warp) per AVQ entry; vertices with more than
//                                kChunk slots are split over several warps (workload balance,
//                                §2.4 Eq. 1)
//   min-height neighbour         Alg. 1 lines 10-13 (reading §8(c) #1: min over cf>0 arcs),
//                                warp min-reduction with redux.sync
//   push / relabel               Alg. 1 lines 14-21 with the relaxed rule h(u) > h(v')
//                                (P:187-189), delegated to lane 0
//   early break                  AVQ empty -> global relabel
//
// After round 1 (exact GR) the next AVQ is produced by the round itself: a vertex is
// appended exactly once, by its own warp if it stays active, or by the warp whose push
// raised its excess from 0 (atomics on e make this unique) — a sparse compaction that
// replaces the paper's full |V| rescan in every iteration (§8(a) A3).
#include <climits>
#include <cstdlib>

#include "internal.h"
#include "kernels.h"

namespace wbpr {

constexpr int kWarps = kSolveThreads / 32;
constexpr int kBufCap = 256;     // per-warp append staging (ints)
constexpr int kBufFlush = 224;
constexpr unsigned kInf = 0xffffffffu;

// ------------------------------------------------------------------ layouts
struct Seg {
  int fb, fe;  // forward (BCSR: the whole segment)
  int rb, re;  // RCSR reverse entries
  __device__ int deg() const { return (fe - fb) + (re - rb); }
};

struct BcsrOps {
  const int2* segs; int2* arc; const int* mate;   // segs[u] = {begin, end} (gapped layout)
  unsigned long long pf = 0;   // L2 evict_first policy for streamed arrays
  __device__ void init() { pf = policy_evict_first(); }
  __device__ Seg seg(int u) const { const int2 b = __ldg(segs + u); Seg s; s.fb = b.x; s.fe = b.y; s.rb = s.re = 0; return s; }
  __device__ int degree(int u) const { const int2 b = __ldg(segs + u); return b.y - b.x; }
  // residual out-arc #i of u: u -> col with residual capacity cf, identified by slot
  __device__ void out_arc(const Seg& s, int i, int& col, int& cf, int& slot) const {
    slot = s.fb + i;
    int2 a = ld_cg_hint(arc + slot, pf);
    col = a.x; cf = a.y;
  }
  // residual in-arc #i of w: col -> w with capacity cf(col -> w)
  __device__ void in_arc(const Seg& s, int i, int& col, int& cf) const {
    int p = s.fb + i;
    col = ld_nc_hint(&arc[p].x, pf);
    cf = ld_cg(&arc[ld_nc_hint(mate + p, pf)].y);
  }
  // the same in-arc in two steps (top-down BFS): the neighbour and a key, then c_f(col -> w)
  // only for neighbours still unlabelled (most in-arcs of later levels point at labelled
  // vertices, so their c_f[mate] gather is skipped)
  __device__ void in_arc_col(const Seg& s, int i, int& col, int& key) const {
    const int p = s.fb + i;
    col = ld_nc_hint(&arc[p].x, pf);
    key = ld_nc_hint(mate + p, pf);
  }
  __device__ int in_cf(int key) const { return ld_cg(&arc[key].y); }
  __device__ void col_cf_of_slot(int slot, int& col, int& cf) const {
    int2 a = ld_cg(arc + slot); col = a.x; cf = a.y;
  }
  // out-arcs b0 .. b0+7 of a segment with five 16-B loads (two arcs each, aligned down) instead
  // of eight 8-B ones: one thread scanning its own segment issues fewer L1 wavefronts
  static constexpr bool kVec8 = true;
  __device__ void arcs8(const Seg& s, int b0, int d, int (&col)[8], int (&cf)[8]) const {
    const int first = s.fb + b0;
    const int a = first & ~1;
    const bool odd = (first & 1) != 0;
    int4 w[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int p = a + 2 * q;
      w[q] = p < s.fe ? ld_cg_hint(reinterpret_cast<const int4*>(arc + p), pf) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // arc j + odd of the window: even -> (x, y) of w[(j+odd)/2], odd -> (z, w)
      const int4 e0 = w[j >> 1], e1 = w[(j + 1) >> 1];
      const int c0 = (j & 1) ? e0.z : e0.x, f0 = (j & 1) ? e0.w : e0.y;      // arc j       (odd == 0)
      const int c1 = (j & 1) ? e1.x : e0.z, f1 = (j & 1) ? e1.y : e0.w;      // arc j + 1   (odd == 1)
      col[j] = odd ? c1 : c0;
      cf[j] = b0 + j < d ? (odd ? f1 : f0) : 0;
    }
  }
  __device__ void push(int slot, int d) const {
    atomicAdd(&arc[slot].y, -d);
    atomicAdd(&arc[__ldg(mate + slot)].y, d);
  }
  // the reverse-arc lookup of a push, loadable ahead of the push (latency-bound phases)
  __device__ int aux(int slot) const { return ld_nc_hint(mate + slot, pf); }
  __device__ void push_aux(int slot, int ax, int d) const {
    atomicAdd(&arc[slot].y, -d);
    atomicAdd(&arc[ax].y, d);
  }
  __device__ void saturate(int slot, int d) const { push(slot, d); }
};

struct RcsrOps {
  static constexpr bool kVec8 = false;
  __device__ void arcs8(const Seg&, int, int, int (&)[8], int (&)[8]) const {}
  const int* foff; int2* farc; const int* roff; const int2* rarc; int* bcf; int Mf;
  unsigned long long pf = 0;
  __device__ void init() { pf = policy_evict_first(); }
  __device__ Seg seg(int u) const {
    Seg s; s.fb = __ldg(foff + u); s.fe = __ldg(foff + u + 1); s.rb = __ldg(roff + u); s.re = __ldg(roff + u + 1);
    return s;
  }
  __device__ int degree(int u) const {
    return (__ldg(foff + u + 1) - __ldg(foff + u)) + (__ldg(roff + u + 1) - __ldg(roff + u));
  }
  __device__ void out_arc(const Seg& s, int i, int& col, int& cf, int& slot) const {
    int df = s.fe - s.fb;
    if (i < df) {
      slot = s.fb + i;
      int2 a = ld_cg_hint(farc + slot, pf);
      col = a.x; cf = a.y;
    } else {
      int q = s.rb + (i - df);
      int2 r = ld_nc_hint(rarc + q, pf);   // {col, flow_idx}
      col = r.x;
      cf = ld_cg(bcf + r.y);               // backward cf: flow on col -> u that can return
      slot = Mf + q;
    }
  }
  __device__ void in_arc(const Seg& s, int i, int& col, int& cf) const {
    int df = s.fe - s.fb;
    if (i < df) {                          // w -> col forward: col -> w is its backward arc
      int p = s.fb + i;
      col = ld_nc_hint(&farc[p].x, pf);
      cf = ld_cg(bcf + p);
    } else {                               // col -> w forward arc f
      int2 r = ld_nc_hint(rarc + s.rb + (i - df), pf);
      col = r.x;
      cf = ld_cg(&farc[r.y].y);
    }
  }
  __device__ void in_arc_col(const Seg& s, int i, int& col, int& key) const {
    const int df = s.fe - s.fb;
    if (i < df) { const int p = s.fb + i; col = ld_nc_hint(&farc[p].x, pf); key = ~p; }   // c_f = bcf[p]
    else { const int2 r = ld_nc_hint(rarc + s.rb + (i - df), pf); col = r.x; key = r.y; }  // c_f = farc[f].y
  }
  __device__ int in_cf(int key) const { return key < 0 ? ld_cg(bcf + ~key) : ld_cg(&farc[key].y); }
  __device__ void col_cf_of_slot(int slot, int& col, int& cf) const {
    if (slot < Mf) { int2 a = ld_cg(farc + slot); col = a.x; cf = a.y; }
    else { int2 r = __ldg(rarc + (slot - Mf)); col = r.x; cf = ld_cg(bcf + r.y); }
  }
  __device__ void push(int slot, int d) const {
    if (slot < Mf) { atomicAdd(&farc[slot].y, -d); atomicAdd(bcf + slot, d); }
    else { int f = __ldg(&rarc[slot - Mf].y); atomicAdd(bcf + f, -d); atomicAdd(&farc[f].y, d); }
  }
  __device__ int aux(int slot) const { return slot < Mf ? slot : __ldg(&rarc[slot - Mf].y); }
  __device__ void push_aux(int slot, int ax, int d) const {
    if (slot < Mf) { atomicAdd(&farc[slot].y, -d); atomicAdd(bcf + slot, d); }
    else { atomicAdd(bcf + ax, -d); atomicAdd(&farc[ax].y, d); }
  }
};

// ------------------------------------------------------------------ grid barrier
// Arrival: one acq_rel atomic per CTA.  The last CTA to arrive reads the counters
// the finished phase accumulated, zeroes the ring slot the phase after next will
// use, and publishes {generation, counts} with ONE 16-B release store; waiters poll
// that word with 16-B acquire loads, so the counts arrive together with the
// release (no extra round trip after the barrier).  Waiters give up at the
// watchdog deadline or when another CTA aborted (never hangs the device).
WBPR_DEV unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
WBPR_DEV uint4 ld_acquire_v4(const Bcast* p) {
  uint4 r;
  asm volatile("ld.acquire.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}
WBPR_DEV void st_release_v4(Bcast* p, uint4 v) {
  asm volatile("st.release.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

#ifndef WBPR_TD_LAZY
#define WBPR_TD_LAZY 1   // top-down BFS: c_f(col -> w) loaded only for unlabelled neighbours
#endif
constexpr int kSmallCap = 2048;   // small-frontier mode: shared-memory queue capacity
#ifndef WBPR_SMALL_MAX
#define WBPR_SMALL_MAX 512
#endif
constexpr int kSmallMax = WBPR_SMALL_MAX;   // small-frontier mode: queues up to this size (one pass of 512 threads)
#ifndef WBPR_SMALL_DEG
#define WBPR_SMALL_DEG 8
#endif
constexpr int kSmallDeg = WBPR_SMALL_DEG;   // small-frontier mode: largest degree processed by one thread
#ifndef WBPR_SB
#define WBPR_SB 4
#endif
constexpr int kSB = WBPR_SB;      // small-frontier mode: slots loaded per batch (independent loads)
constexpr int kGapBins = 256;     // online gap: shared-memory bins for the lowest levels
#ifndef WBPR_BUT
#define WBPR_BUT 32
#endif
constexpr int kBuThread = WBPR_BUT; // bottom-up BFS: vertices up to this many slots are scanned by one thread
#ifndef WBPR_BUB
#define WBPR_BUB 8
#endif
#ifndef WBPR_BU_ALPHA
#define WBPR_BU_ALPHA 7   // measured (3 x 20-step A/B, tools/sweep_bu.sh): C5 solve 11.4 -> 9.9 ms, C1 0.74 -> 0.58 ms,
#endif                    // C3 / C3h equal, C4 +0.5 ms (14 was the previous default; 4 and 1 no better)
#ifndef WBPR_BU_BETA
#define WBPR_BU_BETA 24
#endif
constexpr int kBuAlpha = WBPR_BU_ALPHA;   // go bottom-up when frontier slots * alpha > slots not yet labelled (Beamer)
constexpr int kBuBeta = WBPR_BU_BETA;     // back to top-down when the frontier holds < n / beta vertices
constexpr int kBuB = WBPR_BUB;    // bottom-up BFS: slots loaded per batch (independent loads)
// neighbour-label gathers: L2-only (default) or L1-allocating
#ifndef WBPR_H_L1
#define WBPR_H_L1 0   // measured: L1-allocating label gathers gave no gain (B200, C5/C3/C4)
#endif
__device__ __forceinline__ int ld_h(const int* p, unsigned long long pol) {
  return WBPR_H_L1 ? ld_ca_hint(p, pol) : ld_cg_hint(p, pol);
}
constexpr int kAsyncLevel = 32;   // bfs_mode 3: a GR deeper than this continues asynchronously
#ifndef WBPR_ASYNC_WARPS
#define WBPR_ASYNC_WARPS 128         // warps taking part in the asynchronous GR continuation (best of 128/512/2048)
#endif
#ifndef WBPR_TDT
#define WBPR_TDT 8
#endif
constexpr int kTdThread = WBPR_TDT; // top-down BFS: frontier vertices up to this many slots are scanned by one thread
constexpr int kTdPack = 4;        // top-down BFS: pack 32 frontier entries per warp when |frontier| >= kTdPack x warps
#ifndef WBPR_RU
#define WBPR_RU 4
#endif
constexpr int kRU = WBPR_RU;
constexpr int kRThr = 64;         // rounds: vertices up to this many slots are discharged by one thread ...
constexpr int kRThrPack = 4;      // ... when the queue holds at least kRThrPack x warps entries      // push/relabel discharge: 32-slot groups loaded per iteration

struct SharedState {
  int buf[kWarps][kBufCap];
  int wsum[kWarps];
  int wmaxdeg[kWarps];
  unsigned long long wsum64[kWarps];
  int base;
  int abort;
  Bcast bc;           // counts of the phase that just finished
  int gbin[kGapBins];  // low levels of the height histogram (online gap, A6)
  // small-frontier mode
  int sq[2][kSmallCap];
  int s_n, s_maxdeg, s_huge, s_exit;
  unsigned long long s_work;
};

// ------------------------------------------------------------------ warp append buffers
// terminal flags change between the phases (phase 2 swaps them): plain coherent loads
__device__ __forceinline__ uint8_t ld_term(const uint8_t* p) {
  unsigned short v;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return (uint8_t)v;
}

struct QueueOut {   // next-queue destination
  int* q; int* qn;
  HugeRec* hq; int2* hc; int* hn; int* hc_cnt;
  int* md;           // largest appended degree (Ring::maxdeg)
};

__device__ __forceinline__ unsigned lanemask_lt() { unsigned r; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r)); return r; }

__device__ __forceinline__ void warp_flush(SharedState& S, int& cnt, const QueueOut& out) {
  int lane = lane_id(), w = warp_id();
  __syncwarp();
  int base = 0;
  if (lane == 0) base = atomicAdd(out.qn, cnt);
  base = __shfl_sync(FULL, base, 0);
  for (int i = lane; i < cnt; i += 32) st_cg(out.q + base + i, S.buf[w][i]);
  __syncwarp();
  cnt = 0;
}

// all lanes call; lanes with pred append val (warp ballot + prefix; AVQ append)
__device__ __forceinline__ void warp_append(SharedState& S, int& cnt, bool pred, int val, const QueueOut& out,
                                            int dg) {
  unsigned b = __ballot_sync(FULL, pred);
  if (!b) return;
  int w = warp_id();
  unsigned md = __reduce_max_sync(FULL, pred ? (unsigned)dg : 0u);
  if (lane_id() == 0 && (int)md > S.wmaxdeg[w]) S.wmaxdeg[w] = (int)md;
  if (pred) S.buf[w][cnt + __popc(b & lanemask_lt())] = val;
  cnt += __popc(b);
  if (cnt >= kBufFlush) warp_flush(S, cnt, out);
}

// a vertex with more than kChunk slots becomes nchunks warp tasks (single lane)
__device__ __forceinline__ void huge_append(int u, int deg, const QueueOut& out, int chunk) {
  int nch = (deg + chunk - 1) / chunk;
  int hi = atomicAdd(out.hn, 1);
  int c0 = atomicAdd(out.hc_cnt, nch);
  HugeRec r; r.best = ~0ull; r.spent = 0; r.pushed = 0; r.u = u; r.nchunks = nch; r.done = 0; r.pad = 0;
  out.hq[hi] = r;
  for (int j = 0; j < nch; ++j) out.hc[c0 + j] = make_int2(hi, j);
}

// ------------------------------------------------------------------ the kernel
__device__ __forceinline__ void block_flush_all(SharedState& S, int& cnt, const QueueOut& out) {
  // block-aggregated final flush: one global atomic per CTA
  int lane = lane_id(), w = warp_id();
  if (lane == 0) S.wsum[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0, md = 0;
    for (int i = 0; i < kWarps; ++i) {
      int c = S.wsum[i]; S.wsum[i] = tot; tot += c;
      md = max(md, S.wmaxdeg[i]); S.wmaxdeg[i] = 0;
    }
    S.base = tot ? atomicAdd(out.qn, tot) : 0;
    if (md && out.md) atomicMax(out.md, md);
  }
  __syncthreads();
  int base = S.base + S.wsum[w];
  for (int i = lane; i < cnt; i += 32) st_cg(out.q + base + i, S.buf[w][i]);
  cnt = 0;
}

__device__ __forceinline__ unsigned long long block_sum_u64(SharedState& S, unsigned long long v) {
  v = warp_sum(v);
  if (lane_id() == 0) S.wsum64[warp_id()] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) t += S.wsum64[i];
  __syncthreads();
  return t;  // thread 0
}

template <class Ops, int MINB>
__global__ void __launch_bounds__(kSolveThreads, MINB) k_solve(const SolveParams P, const Ops ops_in) {
  __shared__ SharedState S;
  Ops ops = ops_in;
  ops.init();
  const unsigned long long pl = policy_evict_last();   // keep h[] in L2
  Ctrl* C = P.ctrl;
  const int N = P.n;                 // |V| of the union: the label bound (h >= N: inactive)
  // ---- solver group of this CTA (A10 batches): CTAs [b0, b0+nb) run an independent
  // solver over instances [I0, I1) = vertices [VLO, VHI) with their own barrier, counters,
  // queues and GR policy; a single instance is one group spanning the whole grid
  int gid = 0;
  {
    int lo = 0, hi = P.ngroups;
    while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (P.groups[mid].b0 <= (int)blockIdx.x) lo = mid; else hi = mid; }
    gid = lo;
  }
  const GroupDesc GD = P.groups[gid];
  GroupCtrl* GC = P.gctrl + gid;
  const int brank = (int)blockIdx.x - GD.b0;   // CTA rank inside the group
  const unsigned nb = (unsigned)GD.nb;
  const int VLO = GD.vlo, VHI = GD.vhi, I0 = GD.i0, KI = GD.i1 - GD.i0;
  int* const Q[2] = {P.q[0] + VLO, P.q[1] + VLO};
  HugeRec* const HQ[2] = {P.hq[0] + GD.hub0, P.hq[1] + GD.hub0};
  int2* const HC[2] = {P.hc[0] + 2 * GD.hub0, P.hc[1] + 2 * GD.hub0};
  int2* const HS = P.hs + 2 * GD.hub0;
  const int Mslots = P.layout == 0 ? (__ldg(&P.seg[VHI - 1].y) - __ldg(&P.seg[VLO].x))
                                   : 2 * (__ldg(P.off + VHI) - __ldg(P.off + VLO));
  const unsigned long long gr_threshold =
      (unsigned long long)((double)P.gr_beta * (double)((long long)(VHI - VLO) + (long long)Mslots)) + 1;
  const int lane = lane_id(), w = warp_id();
  const int gwarp = brank * kWarps + w;
  const int nwarps = (int)nb * kWarps;
  long long l_rounds = 0, l_grs = 0, l_levels = 0;   // thread 0 of CTA rank 0: per-group counts
  unsigned gen = 0;
  int ph = 0;
  const unsigned long long deadline = globaltimer() + P.deadline_ns_rel;
  // per-warp statistics (registers; lane 0 holds the counts)
  long long st_push = 0, st_relabel = 0, st_arcs = 0, st_bfs_arcs = 0, st_cand = 0;
  int cnt = 0;  // this warp's staged appends (lane-uniform)

  auto ring = [&](int p) -> Ring* { return &GC->ring[p % 3]; };
  auto out_for = [&](int buf) {
    QueueOut o;
    Ring* r = ring(ph);
    o.q = Q[buf]; o.qn = &r->qn;
    o.hq = HQ[buf]; o.hc = HC[buf]; o.hn = &r->hn; o.hc_cnt = &r->hc;
    o.md = &r->maxdeg;
    return o;
  };
  unsigned long long t_sync = 0, t_flush = 0, t_round = 0;
  auto gsync = [&]() -> bool {
    const unsigned long long ts0 = (brank == 0 && threadIdx.x == 0) ? globaltimer() : 0;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = gen + 1;
      int ab = 0;
      uint4 b;
      // (a two-level arrival - 16 sub-counters - measured no faster on B200: the arrival
      // atomics are not the bottleneck of a phase)
      if (atom_add_acqrel(&GC->bar.count, 1u) == nb - 1) {
        GC->bar.count = 0;
        Ring* r = ring(ph);
        // the whole phase record and the abort word in one round trip
        const int4 r0 = ld_cg(reinterpret_cast<const int4*>(r));
        const int4 r1 = ld_cg(reinterpret_cast<const int4*>(r) + 1);
        const int abort_now = ld_volatile(&C->abort);
        const int qn = r0.x, rhn = r0.y, hc = r0.z, kind = r1.x, rmaxdeg = r1.z;
        const unsigned rwork = (unsigned)r0.w, rfedges = (unsigned)r1.y;
        const unsigned long long now = globaltimer();
        GrPolicy& G = GC->pol;
        unsigned flags = 0;
        if (kind == PK_ROUND) {
          atomicAdd((unsigned long long*)&C->stats[ST_AVQ], (unsigned long long)(qn + rhn));
          G.work_since_gr += rwork;
          // GR policy (reading §8(c) #8): queue empty, relabel work above
          // beta (n + M), or time spent in rounds since the last GR above gamma x its cost
          bool due = qn + hc == 0 || G.work_since_gr >= gr_threshold ||
                     (P.gr_gamma > 0.f && (double)(now - G.t_after_gr) >= (double)P.gr_gamma * (double)G.gr_time);
          if (due) { flags = 1; G.t_gr_start = now; }
          else if (P.gap_mode) {
            const int gl = ld_cg(&GC->gap_level);
            if (gl < N) { flags |= 8; GC->gap_pending = gl; GC->gap_level = N; }
          }
        } else if (kind == PK_PREFLOW) {
          G.t_gr_start = now;
        } else if (kind == PK_GR_RESET || kind == PK_BFS) {
          // direction-optimizing BFS (Beamer): bottom-up while the frontier's slots
          // exceed 1/14 of the slots not yet labelled; back to top-down when the
          // frontier holds fewer than n/24 vertices
          const unsigned long long fe = rfedges;
          if (kind == PK_GR_RESET) { G.bfs_seen_edges = 0; G.bfs_bottom_up = 0; }
          G.bfs_seen_edges += fe;
          // slots still to be labelled: bounded by what the previous GR reached (vertices cut
          // off from the sinks stay unreachable, N5), so large unreachable regions do not
          // pull the BFS into bottom-up scans that can never find a parent
          unsigned long long Mtot = (unsigned long long)Mslots;
          if (G.prev_reached && G.prev_reached < Mtot) Mtot = G.prev_reached;
          const unsigned long long rest = Mtot > G.bfs_seen_edges ? Mtot - G.bfs_seen_edges : 0;
          if (!G.bfs_bottom_up) G.bfs_bottom_up = P.bfs_mode != 0 && fe * (unsigned long long)kBuAlpha > rest;
          else G.bfs_bottom_up = (long long)qn * kBuBeta >= (long long)(VHI - VLO);
          if (P.bfs_mode == 2) G.bfs_bottom_up = 1;
          if (G.bfs_bottom_up) flags |= 2;
          // bfs_mode 3: a deep GR continues as the asynchronous label-correcting BFS
          if (P.bfs_mode == 3 && kind == PK_BFS && r1.w + 1 >= kAsyncLevel && qn + hc > 0) flags |= 32;
        } else if (kind == PK_COMPACT) {
          GC->gap_level = N;
          G.prev_reached = G.bfs_seen_edges;
          G.gr_time = now - G.t_gr_start;
          G.t_after_gr = now;
          G.work_since_gr = 0;
        }
        // small-frontier mode for the next phase: a round or a top-down BFS level whose
        // queue fits one CTA (no hub tasks, every queued vertex <= kSmallDeg slots)
        {
          int next = 0;
          if (kind == PK_ROUND) next = (flags & 1) ? 0 : 1;
          else if (kind == PK_GR_RESET || kind == PK_BFS) next = (qn + hc > 0 && !(flags & 2)) ? 2 : 0;
          else if (kind == PK_COMPACT) next = (qn + hc > 0) ? 1 : 0;
          const int md = rmaxdeg;
          if (P.small_mode && P.schedule == 0 && next && hc == 0 && qn > 0 && qn <= kSmallMax && md <= kSmallDeg) flags |= 4;
        }
        {   // phase timing: release of the previous barrier -> this release, by phase kind
          int bk = (kind == PK_BFS && G.bfs_bottom_up_prev) ? kPhBfsUp : kind;
          if (bk >= 0 && bk < kPhBuckets && G.t_release) {
            atomicAdd((unsigned long long*)&C->phase_ns[bk], now - G.t_release);
            atomicAdd((unsigned long long*)&C->phase_cnt[bk], 1ull);
          }
          G.bfs_bottom_up_prev = (flags & 2) ? 1 : 0;
          G.t_release = now;
        }
        if (abort_now) flags |= 16;
        if (rmaxdeg <= kRThr) flags |= 64;   // every queued vertex is small: rounds may use the thread mode
        b.x = target;
        b.y = (unsigned)qn;
        b.z = (unsigned)hc;
        b.w = flags;
        Ring* z = ring(ph + 1);
        reinterpret_cast<int4*>(z)[0] = make_int4(0, 0, 0, 0);
        reinterpret_cast<int4*>(z)[1] = make_int4(0, 0, 0, 0);
        st_release_v4(&GC->bc, b);
      } else {
        unsigned ns = 0;
        while (true) {
          b = ld_acquire_v4(&GC->bc);
          if (b.x == target) break;
          if (ld_volatile(&C->abort)) { ab = 1; break; }
          if (globaltimer() > deadline) { atomicExch(&C->abort, 1); ab = 1; break; }
          if (ns) __nanosleep(ns);
          ns = ns ? (ns < 128 ? ns * 2 : 128) : 16;
        }
      }
      if (!ab) ab = (b.w & 16) != 0;   // the last arriver saw the abort word
      S.abort = ab;
      S.bc.qn = (int)b.y; S.bc.hc = (int)b.z; S.bc.flags = b.w;
    }
    ++gen;
    ++ph;
    __syncthreads();
    if (brank == 0 && threadIdx.x == 0) t_sync += globaltimer() - ts0;
    return S.abort == 0;
  };

  // targets of the global relabel: the sinks (phase 1) / the sources (phase 2)
  const long long* SNK = P.snk + I0;
  // ---------------------------------------------------------------- init
  if (brank == 0 && threadIdx.x == 0) GC->gap_level = N;
  {   // 4 independent vertices per thread and iteration (memory-level parallelism)
    const int stride = nb * blockDim.x;
    for (int v0 = VLO + brank * blockDim.x + threadIdx.x; v0 < VHI; v0 += 4 * stride) {
      int dgq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) dgq[q] = v0 + q * stride < VHI ? ops.degree(v0 + q * stride) : 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int v = v0 + q * stride;
        if (v >= VHI) continue;
        st_cg(P.e + v, 0ll);
        P.deact[v] = 0;
        // static chunk list of the vertices with > kChunk slots (bottom-up BFS splits them)
        const int dg = dgq[q];
        if (dg > kChunk) {
          int nch = (dg + kChunk - 1) / kChunk;
          int t0 = atomicAdd(&GC->nhs, nch);
          for (int j = 0; j < nch; ++j) HS[t0 + j] = make_int2(v, j);
        }
      }
    }
  }
  if (!gsync()) return;

  // ---------------------------------------------------------------- preflow (Alg. 1 Step 0)
  {
    unsigned long long exc = 0;
    for (int i = I0; i < I0 + KI; ++i) {
      int s = (int)P.src[i];
      Seg sg = ops.seg(s);
      int d = sg.deg();
      for (int j = brank * blockDim.x + threadIdx.x; j < d; j += nb * blockDim.x) {
        int col, cf, slot;
        ops.out_arc(sg, j, col, cf, slot);
        if (cf > 0) {   // c_f(s,v) <- 0, c_f(v,s) <- c(s,v), e(v) <- c(s,v)
          ops.push(slot, cf);
          atomicAdd((unsigned long long*)(P.e + col), (unsigned long long)cf);
          exc += (unsigned long long)cf;
        }
      }
    }
    unsigned long long t = block_sum_u64(S, exc);
    if (threadIdx.x == 0 && t) atomicAdd((unsigned long long*)&C->excess_total, t);
    if (brank == 0 && threadIdx.x == 0) ring(ph)->kind = PK_PREFLOW;
  }
  if (!gsync()) return;


  // ---------------------------------------------------------------- small-frontier mode helpers
  // CTA 0 alone, one THREAD per queued vertex (<= kSmallDeg slots, 8-slot batches of
  // independent loads), queues in shared memory, __syncthreads instead of grid barriers.
  // online gap (A6): height histogram updated at every relabel; a level that empties
  // is recorded and lifted at the next round boundary (a heuristic under relaxed labels,
  // corrected by the next exact GR; never used for termination or Excess_total)
  auto gap_relabel = [&](int old, int nh) {
    if (!P.gap_mode) return;
    if (old < N) {
      int prev = atomicSub(P.hist + old, 1);
      if (prev == 1) atomicMin(&GC->gap_level, old);
    }
    if (nh < N) atomicAdd(P.hist + nh, 1);
  };
  // per-warp workload trace (NEXT #3, §4.3 / Fig. 3): one record per warp per traced round
  long long trace_round = 0;
  auto trace_begin = [&](unsigned long long& t0, long long& a0, long long& p0, long long& r0, int& n0) {
    t0 = globaltimer(); a0 = st_arcs; p0 = st_push; r0 = st_relabel; n0 = 0;
  };
  auto trace_end = [&](unsigned long long t0, long long a0, long long p0, long long r0, int ntasks) {
    if (!P.trace || trace_round >= P.trace_rounds) return;
    unsigned long long t1 = globaltimer();
    long long da = warp_sum(st_arcs - a0), dp = warp_sum(st_push - p0), dr = warp_sum(st_relabel - r0);
    if (lane_id() == 0) {
      TraceRec r;
      r.round = (int)trace_round; r.warp = gwarp; r.busy_ns = (unsigned)(t1 - t0); r.tasks = ntasks;
      r.slots = (int)da; r.pushes = (int)dp; r.relabels = (int)dr; r.schedule = P.schedule;
      P.trace[(long long)trace_round * nwarps + gwarp] = r;
    }
  };
  int sa = 0, sdst = 0;   // shared-memory queue being read; global queue buffer being written
  auto small_append = [&](int v, int dg, int chunk) {   // chunk: kChunk (BFS) / kRChunk (rounds)
    if (dg > chunk) {
      QueueOut ho;
      ho.q = nullptr; ho.qn = nullptr; ho.md = nullptr;
      ho.hq = HQ[sdst]; ho.hc = HC[sdst]; ho.hn = &GC->small_hn; ho.hc_cnt = &GC->small_hc;
      huge_append(v, dg, ho, chunk);
      S.s_huge = 1;
      return;
    }
    int pos = atomicAdd(&S.s_n, 1);
    st_cg(Q[sdst] + pos, v);                 // complete copy in global memory (grid resume)
    if (pos < kSmallCap) S.sq[sa ^ 1][pos] = v;
    atomicMax(&S.s_maxdeg, dg);
  };
  // tc = true: thread-centric sweep (Alg. 1 Step 1, NEXT #1) - no queue appends
  unsigned long long tc_work = 0;
  auto small_round_vertex = [&](int u, bool tc) {
    Seg sg = ops.seg(u);
    const int d = sg.deg();
    const int hu = ld_cg(P.h + u);
    const long long eu = ld_cg(P.e + u);
    if (hu >= N) return;   // lifted by the gap heuristic: inactive until the next GR
    unsigned long long best = ~0ull;
    int bcf = 0, bcol = 0;
    long long budget = eu, pushed = 0;
    for (int b0 = 0; b0 < d; b0 += kSB) {
      int col[kSB], cf[kSB], slot[kSB], hv[kSB];
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        cf[j] = 0; col[j] = 0; slot[j] = 0;
        if (b0 + j < d) ops.out_arc(sg, b0 + j, col[j], cf[j], slot[j]);
      }
      // everything a push needs is loaded together with the labels (one round trip)
      int dgc[kSB], axc[kSB];
      uint8_t tmc[kSB];
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        const bool pre = P.push_mode != 0 && cf[j] > 0;
        hv[j] = cf[j] > 0 ? ld_h(P.h + col[j], pl) : INT_MAX;
        dgc[j] = pre ? ops.degree(col[j]) : 0;
        axc[j] = pre ? ops.aux(slot[j]) : 0;
        tmc[j] = pre ? ld_term(P.term + col[j]) : 1;
      }
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        if (cf[j] > 0) {
          unsigned long long cand = ((unsigned long long)(unsigned)hv[j] << 32) | (unsigned)slot[j];
          if (cand < best) { best = cand; bcf = cf[j]; bcol = col[j]; }
        }
      }
      if (P.push_mode != 0) {
#pragma unroll
        for (int j = 0; j < kSB; ++j) {
          if (cf[j] > 0 && hv[j] < hu && budget > 0) {
            int dd = (int)(budget < (long long)cf[j] ? budget : (long long)cf[j]);
            int dgv = dgc[j];
            ops.push_aux(slot[j], axc[j], dd);
            long long old_v = (long long)atomicAdd((unsigned long long*)(P.e + col[j]), (unsigned long long)dd);
            if (!tc && old_v == 0 && tmc[j] == 0) small_append(col[j], dgv, kRChunk);
            budget -= dd;
            pushed += dd;
            ++st_push;
          }
        }
        if (budget <= 0) break;
      }
    }
    st_arcs += d;
    const unsigned hmin = (unsigned)(best >> 32);
    if (P.push_mode == 0 && best != ~0ull && (int)hmin < hu && bcf > 0) {
      int dd = (int)(eu < (long long)bcf ? eu : (long long)bcf);
      int dgv = ops.degree(bcol);
      ops.push((int)(best & 0xffffffffu), dd);
      long long old_u = (long long)atomicAdd((unsigned long long*)(P.e + u), (unsigned long long)(-(long long)dd));
      long long old_v = (long long)atomicAdd((unsigned long long*)(P.e + bcol), (unsigned long long)dd);
      if (!tc && old_u - dd > 0) small_append(u, d, kRChunk);
      if (!tc && old_v == 0 && ld_term(P.term + bcol) == 0) small_append(bcol, dgv, kRChunk);
      ++st_push;
    } else if (P.push_mode != 0 && pushed > 0) {
      long long old_u = (long long)atomicAdd((unsigned long long*)(P.e + u), (unsigned long long)(-pushed));
      if (!tc && old_u - pushed > 0) small_append(u, d, kRChunk);
    } else {
      int nh = (best == ~0ull || (int)hmin >= N - 1) ? N : (int)hmin + 1;
      st_cg(P.h + u, nh);
      gap_relabel(hu, nh);
      if (!tc && nh < N) small_append(u, d, kRChunk);
      if (tc) tc_work += (unsigned long long)d + 1;
      else atomicAdd(&S.s_work, (unsigned long long)d + 1);
      ++st_relabel;
    }
  };
  auto small_bfs_vertex = [&](int wv, int lvl) {
    Seg sg = ops.seg(wv);
    const int d = sg.deg();
    for (int b0 = 0; b0 < d; b0 += kSB) {
      int u[kSB], cf[kSB], hu8[kSB];
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        cf[j] = 0; u[j] = 0;
        if (b0 + j < d) ops.in_arc(sg, b0 + j, u[j], cf[j]);
      }
      // labels and degrees loaded with the residual capacities (one round trip; the graphs
      // that reach the small mode are latency-bound)
      int dgu[kSB];
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        hu8[j] = b0 + j < d ? ld_h(P.h + u[j], pl) : -1;
        dgu[j] = b0 + j < d ? ops.degree(u[j]) : 0;
      }
#pragma unroll
      for (int j = 0; j < kSB; ++j)
        if (cf[j] > 0 && hu8[j] == N && atomicCAS(P.h + u[j], N, lvl + 1) == N) small_append(u[j], dgu[j], kChunk);
    }
    st_bfs_arcs += d;
  };

  // bottom-up BFS, one warp over slots [lo, hi) of a vertex: is there an out-arc with
  // c_f > 0 into the current level?  kRU groups of 32 slots per iteration (all arc loads,
  // then all label gathers), early exit per iteration.  All lanes call; warp-uniform result.
  int level = 0;
  auto bu_warp_scan = [&](const Seg& sg, int lo, int hi, int& scanned) -> bool {
    for (int b = lo; b < hi; b += 32 * kRU) {
      int col[kRU], cf[kRU];
#pragma unroll
      for (int j = 0; j < kRU; ++j) {
        const int i = b + j * 32 + lane;
        col[j] = 0; cf[j] = 0;
        if (i < hi) { int slot; ops.out_arc(sg, i, col[j], cf[j], slot); }
      }
      bool ok = false;
#pragma unroll
      for (int j = 0; j < kRU; ++j) ok |= cf[j] > 0 && ld_h(P.h + col[j], pl) == level;
      scanned += min(32 * kRU, hi - b);
      if (__ballot_sync(FULL, ok)) return true;
    }
    return false;
  };
  // top-down BFS, one warp over in-arcs [lo, hi) of frontier vertex w: label every
  // unlabelled u with c_f(u, w) > 0 (CAS; first finder appends u).  kRU groups per
  // iteration: in-arc loads, then the c_f / label gathers, then the CASes, then the appends.
  auto td_warp_scan = [&](const Seg& sg, int lo, int hi, const QueueOut& o, unsigned& fedges) {
    for (int b = lo; b < hi; b += 32 * kRU) {
      int u[kRU], cf[kRU], hu[kRU];
#if WBPR_TD_LAZY
      int mk[kRU];
#pragma unroll
      for (int j = 0; j < kRU; ++j) {
        const int i = b + j * 32 + lane;
        u[j] = 0; mk[j] = 0;
        if (i < hi) ops.in_arc_col(sg, i, u[j], mk[j]);
      }
#pragma unroll
      for (int j = 0; j < kRU; ++j) hu[j] = (b + j * 32 + lane < hi) ? ld_h(P.h + u[j], pl) : -1;
#pragma unroll
      for (int j = 0; j < kRU; ++j) cf[j] = hu[j] == N ? ops.in_cf(mk[j]) : 0;   // only unlabelled neighbours
#else
#pragma unroll
      for (int j = 0; j < kRU; ++j) {
        const int i = b + j * 32 + lane;
        u[j] = 0; cf[j] = 0;
        if (i < hi) ops.in_arc(sg, i, u[j], cf[j]);
      }
#pragma unroll
      for (int j = 0; j < kRU; ++j) hu[j] = (b + j * 32 + lane < hi) ? ld_h(P.h + u[j], pl) : -1;   // with c_f (parallel)
#endif
      bool found[kRU];
#pragma unroll
      for (int j = 0; j < kRU; ++j)   // sinks 0, sources N+1: never N; level(u) = level(w) + 1
        found[j] = cf[j] > 0 && hu[j] == N && atomicCAS(P.h + u[j], N, level + 1) == N;
      int dg[kRU];
#pragma unroll
      for (int j = 0; j < kRU; ++j) dg[j] = found[j] ? ops.degree(u[j]) : 0;
#pragma unroll
      for (int j = 0; j < kRU; ++j) {
        if (!__ballot_sync(FULL, found[j])) continue;
        unsigned fsum = warp_sum((unsigned)dg[j]);
        if (lane == 0) fedges += fsum;
        const bool huge = found[j] && dg[j] > kChunk;
        if (huge) huge_append(u[j], dg[j], o, kChunk);
        warp_append(S, cnt, found[j] && !huge, u[j], o, dg[j]);
      }
    }
  };

  enum { S_GR = 0, S_BFS = 1, S_COMPACT = 2, S_ROUND = 3, S_DONE = 4, S_ABFS = 5 };
  int phase = 1;          // 2: return the stranded excess to the sources (NEXT #2)
  bool converged = false; // phase ended by an exact GR with no active vertex
  long long rounds = 0;
  int cur = 0, fb = 0;
  int state = S_GR;
  unsigned small_epoch = 0;
  int grs_done = 0;       // global relabels started by this group (every thread; debug_stop)

  while (true) {
  while (state != S_DONE) {
    if (state == S_ROUND && (S.bc.flags & 8)) {   // (TC sweeps skip lifted vertices by h >= n)
      // ------------------------------------------------------------ gap lift (A6)
      const int sqn = S.bc.qn, shc = S.bc.hc;
      const int gl = ld_cg(&GC->gap_pending);
      unsigned long long lifted = 0;
      for (int v = VLO + brank * blockDim.x + threadIdx.x; v < VHI; v += nb * blockDim.x) {
        int hv = ld_cg(P.h + v);
        if (hv > gl && hv < N) {
          st_cg(P.h + v, N);
          atomicSub(P.hist + hv, 1);
          ++lifted;
        }
      }
      unsigned long long t = block_sum_u64(S, lifted);
      if (threadIdx.x == 0 && t) atomicAdd((unsigned long long*)&C->stats[ST_GAPLIFT], t);
      if (brank == 0 && threadIdx.x == 0) ring(ph)->kind = PK_GAP;
      if (!gsync()) return;
      if (threadIdx.x == 0) { S.bc.qn = sqn; S.bc.hc = shc; S.bc.flags = 0; }
      __syncthreads();
      continue;
    }
    if (S.bc.flags & 4) {
      // ------------------------------------------------------------ small-frontier mode
      if (brank == 0) {
        int qa = S.bc.qn;
        const int* gsrc = (state == S_BFS) ? Q[fb] : Q[cur];
        for (int i = threadIdx.x; i < qa; i += blockDim.x) S.sq[0][i] = ld_cg(gsrc + i);
        // thread 0 keeps the GR-policy state and counters in registers while CTA 0 runs alone
        unsigned long long g_work = 0, g_after = 0, g_grtime = 0;
        long long c_rounds = 0, c_avq = 0, c_levels = 0, c_phases = 0;
        if (threadIdx.x == 0) {
          GC->small_hn = 0; GC->small_hc = 0; atomicAdd((unsigned long long*)&C->stats[ST_SMALL_ENTRIES], 1ull);
          g_work = GC->pol.work_since_gr; g_after = GC->pol.t_after_gr; g_grtime = GC->pol.gr_time;
        }
        sa = 0;
        int code = 0, nn = 0;
        __syncthreads();
        while (true) {
          // (s_exit is not reset here: thread 0 writes it every phase between the two barriers
          // below, and a reset here would race with the other threads' read of the previous one)
          if (threadIdx.x == 0) { S.s_n = 0; S.s_maxdeg = 0; S.s_huge = 0; S.s_work = 0; }
          sdst = (state == S_BFS) ? (fb ^ 1) : (cur ^ 1);
          __syncthreads();
          if (state == S_BFS) {
            for (int i = threadIdx.x; i < qa; i += blockDim.x) small_bfs_vertex(S.sq[sa][i], level);
          } else {
            if (threadIdx.x == 0) { ++c_rounds; c_avq += qa; }
            for (int i = threadIdx.x; i < qa; i += blockDim.x) small_round_vertex(S.sq[sa][i], false);
          }
          __syncthreads();
          nn = S.s_n;
          if (state == S_BFS) { fb ^= 1; ++level; } else { cur ^= 1; ++rounds; }
          if (threadIdx.x == 0) {
            ++c_phases;
            int ex = 0;
            const unsigned long long now = globaltimer();
            const bool spill = nn > kSmallMax || S.s_maxdeg > kSmallDeg || S.s_huge;
            if (state == S_BFS) {
              ++c_levels;
              if (nn == 0 && !S.s_huge) ex = 2;
              else if (spill || (P.bfs_mode == 3 && level + 1 >= kAsyncLevel)) ex = 1;
            } else {
              g_work += S.s_work;
              bool due = (nn == 0 && !S.s_huge) || g_work >= gr_threshold ||
                         (P.gr_gamma > 0.f && (double)(now - g_after) >= (double)P.gr_gamma * (double)g_grtime);
              if (due) { GC->pol.t_gr_start = now; ex = 3; }
              else if (rounds >= P.max_rounds) { C->status = DS_NOTCONVERGED; ex = 4; }
              else if (P.gap_mode && ld_cg(&GC->gap_level) < N) {
                GC->gap_pending = GC->gap_level; GC->gap_level = N; ex = 6;
              }
              else if (spill) ex = 1;
            }
            // (the abort word costs a dependent L2 round trip: polled every 64 phases)
            if (!ex && (now > deadline || ((c_phases & 63) == 0 && ld_volatile(&C->abort)))) { atomicExch(&C->abort, 1); ex = 5; }
            S.s_exit = ex;
          }
          __syncthreads();
          code = S.s_exit;
          if (code) break;
          qa = nn;
          sa ^= 1;
        }
        if (code == 2) state = S_COMPACT;
        else if (code == 3) state = S_GR;
        else if (code == 4 || code == 5) state = S_DONE;
        if (threadIdx.x == 0) {
          GC->pol.work_since_gr = g_work;
          l_rounds += c_rounds; l_levels += c_levels;
          atomicAdd((unsigned long long*)&C->stats[ST_AVQ], (unsigned long long)c_avq);
          atomicAdd((unsigned long long*)&C->stats[ST_SMALL_PHASES], (unsigned long long)c_phases);
          {
            const unsigned long long now = globaltimer();
            if (GC->pol.t_release) {
              atomicAdd((unsigned long long*)&C->phase_ns[kPhSmall], now - GC->pol.t_release);
              atomicAdd((unsigned long long*)&C->phase_cnt[kPhSmall], (unsigned long long)c_phases);
            }
            GC->pol.t_release = now;
          }
          Resume& R = GC->res;
          R.state = state; R.qn = nn; R.hc = GC->small_hc; R.cur = cur; R.fb = fb; R.level = level;
          R.rounds = rounds;
          R.flags = code == 6 ? 8 : 0;
          __threadfence();
          atomicAdd(&R.epoch, 1u);
          S.bc.qn = nn; S.bc.hc = GC->small_hc; S.bc.flags = code == 6 ? 8 : 0;
          S.abort = code == 5;
        }
        ++small_epoch;
        __syncthreads();
        if (S.abort) return;
      } else {
        if (threadIdx.x == 0) {
          const unsigned target = small_epoch + 1;
          int ab = 0;
          unsigned ns = 32;
          while (ld_acquire(&GC->res.epoch) != target) {
            if (ld_volatile(&C->abort)) { ab = 1; break; }
            if (globaltimer() > deadline) { atomicExch(&C->abort, 1); ab = 1; break; }
            __nanosleep(ns);
            if (ns < 256) ns <<= 1;
          }
          Resume& R = GC->res;
          S.bc.qn = ld_cg(&R.qn); S.bc.hc = ld_cg(&R.hc); S.bc.flags = (unsigned)ld_cg(&R.flags);
          S.s_n = ld_cg(&R.state); S.s_maxdeg = ld_cg(&R.cur); S.s_huge = ld_cg(&R.fb); S.s_exit = ld_cg(&R.level);
          S.s_work = (unsigned long long)ld_cg(&R.rounds);
          S.abort = ab;
        }
        __syncthreads();
        if (S.abort) return;
        state = S.s_n; cur = S.s_maxdeg; fb = S.s_huge; level = S.s_exit; rounds = (long long)S.s_work;
        ++small_epoch;
        __syncthreads();
      }
      continue;
    }

    if (state == S_GR) {
      ++grs_done;
      // ------------------------------------------------------------ global relabel
      // reset labels: sinks 0, everything else |V| (= unreached); frontier <- sinks
      {   // 4 independent vertices per thread and iteration (memory-level parallelism)
        const int stride = nb * blockDim.x;
        for (int v0 = VLO + brank * blockDim.x + threadIdx.x; v0 < VHI; v0 += 4 * stride) {
          uint8_t tv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) tv[q] = v0 + q * stride < VHI ? ld_term(P.term + v0 + q * stride) : 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int v = v0 + q * stride;
            if (v < VHI) {
              st_cg(P.h + v, (tv[q] & kSink) ? 0 : ((tv[q] & kSource) ? N + 1 : N));
              if (P.gap_mode) st_cg(P.hist + v, 0);
            }
          }
        }
      }
      if (brank == 0) {
        QueueOut o = out_for(0);
        for (int base = w * 32; base < KI; base += kWarps * 32) {
          int i = base + lane;
          int t = i < KI ? (int)SNK[i] : 0;
          int dg = i < KI ? ops.degree(t) : 0;
          bool huge = i < KI && dg > kChunk;
          if (huge) huge_append(t, dg, o, kChunk);
          warp_append(S, cnt, i < KI && !huge, t, o, dg);
          unsigned fsum = warp_sum((unsigned)dg);
          if (lane == 0 && fsum) atomicAdd(&ring(ph)->fedges, fsum);
        }
        block_flush_all(S, cnt, o);
        if (threadIdx.x == 0) { ++l_grs; ring(ph)->kind = PK_GR_RESET; }
      }
      if (!gsync()) return;
      state = S_BFS;
      fb = 0;
      level = 0;
      continue;
    }

    if (state == S_BFS && (S.bc.flags & 32)) { state = S_ABFS; continue; }

    if (state == S_ABFS) {
      // ------------------------------------------------------------ asynchronous GR continuation
      // (bfs_mode 3, a GR deeper than kAsyncLevel levels).  The labels set so far are exact BFS
      // distances and the frontier holds level `level`.  From here a label-correcting BFS runs
      // over one bounded MPMC ring (cells {seq, v}: enqueue at position p waits for seq == p and
      // writes p + 1, dequeue waits for p + 1 and frees the cell with p + cap) with no level
      // barriers: a dequeued vertex w relaxes every residual in-arc u -> w,
      // h(u) <- min(h(u), h(w) + 1), re-queueing u when it improves (in-queue flag: at most one
      // ring entry per vertex, so cap = |group| cells suffice).  When nothing is pending, every
      // label is its exact distance again (the Bellman-Ford fixed point over unit arcs), so the
      // compaction, Excess_total and termination read the same labels as after the
      // level-synchronous BFS.
      const int fq = S.bc.qn, fh = S.bc.hc;     // the frontier (level `level`)
      const int cap = VHI - VLO;
      int2* const aring = P.aring + VLO;
      for (int i = brank * blockDim.x + threadIdx.x; i < cap; i += nb * blockDim.x) {
        st_cg_v2(aring + i, make_int2(i, 0));
        st_cg(P.inq + VLO + i, 0);
      }
      if (brank == 0 && threadIdx.x == 0) {
        GC->aq_head[0] = 0; GC->aq_tail[0] = 0; GC->aq_pending[0] = 0; ring(ph)->kind = PK_ABFS;
      }
      if (!gsync()) return;
      // warp-collective enqueue of the lanes with pred (pending counted before the entries
      // become visible, so pending == 0 means no entry queued and no vertex being processed)
      auto aq_push = [&](bool pred, int v) {
        const unsigned b = __ballot_sync(FULL, pred);
        if (!b) return;
        int base = 0;
        if (lane == 0) {
          atomicAdd(&GC->aq_pending[0], __popc(b));
          base = atomicAdd(&GC->aq_tail[0], __popc(b));
        }
        base = __shfl_sync(FULL, base, 0);
        __syncwarp();
        if (pred) {
          const int pos = base + __popc(b & lanemask_lt());
          int2* const cell = aring + (pos % cap);
          unsigned spins = 0;
          bool ok = true;
          while (ld_acquire_v2(cell).x != pos) {   // (the watchdog / abort word is polled here too)
            __nanosleep(20);
            if ((++spins & 255u) == 0 && (globaltimer() > deadline || ld_volatile(&C->abort))) {
              atomicExch(&C->abort, 1);
              ok = false;
              break;
            }
          }
          if (ok) st_release_v2(cell, make_int2(pos + 1, v));
        }
      };
      // seed: the frontier (normal entries and hub vertices, chunk 0 of each)
      for (int t = gwarp * 32 + lane; t - lane < fq; t += nwarps * 32) {
        const bool p = t < fq;
        const int v = p ? ld_cg(Q[fb] + t) : 0;
        if (p) st_cg(P.inq + v, 1);
        aq_push(p, v);
      }
      for (int t = gwarp * 32 + lane; t - lane < fh; t += nwarps * 32) {
        bool p = false;
        int v = 0;
        if (t < fh) {
          const int2 c = ld_cg(HC[fb] + t);
          if (c.y == 0) { p = true; v = ld_cg(&HQ[fb][c.x].u); st_cg(P.inq + v, 1); }
        }
        aq_push(p, v);
      }
      if (brank == 0 && threadIdx.x == 0) ring(ph)->kind = PK_ABFS;
      if (!gsync()) return;
      // the asynchronous loop: warps take up to 32 produced entries at a time (only the first
      // kAsyncWarps warps take part: idle pollers would contend with the working ones)
      unsigned idle_ns = 32;
      while (gwarp < WBPR_ASYNC_WARPS) {
        int base = 0, got = 0;
        if (lane == 0) {
          while (true) {
            const int h0 = ld_volatile(&GC->aq_head[0]);
            const int t0 = ld_volatile(&GC->aq_tail[0]);
            if (h0 >= t0) break;
            const int k = min(32, t0 - h0);
            if (atomicCAS(&GC->aq_head[0], h0, h0 + k) == h0) { base = h0; got = k; break; }
          }
        }
        base = __shfl_sync(FULL, base, 0);
        got = __shfl_sync(FULL, got, 0);
        if (got == 0) {
          int stop = 0;
          if (lane == 0) {
            stop = ld_volatile(&GC->aq_pending[0]) == 0;
            if (!stop && (globaltimer() > deadline || ld_volatile(&C->abort))) { atomicExch(&C->abort, 1); stop = 1; }
          }
          if (__shfl_sync(FULL, stop, 0)) break;
          __nanosleep(idle_ns);
          if (idle_ns < 1024) idle_ns <<= 1;
          continue;
        }
        idle_ns = 32;
        int w = -1;
        if (lane < got) {
          const int pos = base + lane;
          int2* const cell = aring + (pos % cap);
          int2 c = ld_acquire_v2(cell);
          unsigned spins = 0;
          bool ok = true;
          while (c.x != pos + 1) {
            __nanosleep(20);
            c = ld_acquire_v2(cell);
            if ((++spins & 255u) == 0 && c.x != pos + 1 && (globaltimer() > deadline || ld_volatile(&C->abort))) {
              atomicExch(&C->abort, 1);
              ok = false;
              break;
            }
          }
          if (ok) {
            w = c.y;
            st_release_v2(cell, make_int2(pos + cap, 0));
            atom_exch_acquire(P.inq + w, 0);   // dequeued: a later improvement of h(w) re-queues it
          }
        }
        const int hw = w >= 0 ? ld_cg(P.h + w) : 0;
        Seg sw;
        sw.fb = sw.fe = sw.rb = sw.re = 0;
        int dw = 0;
        if (w >= 0) { sw = ops.seg(w); dw = sw.deg(); }
        auto relax = [&](bool ok, int u, int cf, int hsrc) -> bool {   // true: u improved and must be queued
          if (!ok || cf <= 0) return false;
          const int nl = hsrc + 1;
          if (ld_term(P.term + u) != 0 || ld_cg(P.h + u) <= nl) return false;
          if (atomicMin(P.h + u, nl) <= nl) return false;
          return atom_or_release(P.inq + u, 1) == 0;
        };
        // vertices with <= kTdThread slots: one thread each; larger ones: the whole warp
        const bool thr = w >= 0 && dw <= kTdThread;
        if (thr) st_bfs_arcs += dw;
        for (int b0 = 0; __any_sync(FULL, thr && b0 < dw); b0 += kBuB) {
          int u[kBuB], cf[kBuB];
#pragma unroll
          for (int j = 0; j < kBuB; ++j) {
            u[j] = 0; cf[j] = 0;
            if (thr && b0 + j < dw) ops.in_arc(sw, b0 + j, u[j], cf[j]);
          }
#pragma unroll
          for (int j = 0; j < kBuB; ++j) aq_push(relax(thr && b0 + j < dw, u[j], cf[j], hw), u[j]);
        }
        unsigned todo = __ballot_sync(FULL, w >= 0 && !thr);
        while (todo) {
          const int j = __ffs(todo) - 1;
          todo &= todo - 1;
          Seg sg;
          sg.fb = __shfl_sync(FULL, sw.fb, j); sg.fe = __shfl_sync(FULL, sw.fe, j);
          sg.rb = __shfl_sync(FULL, sw.rb, j); sg.re = __shfl_sync(FULL, sw.re, j);
          const int hj = __shfl_sync(FULL, hw, j);
          const int d = sg.deg();
          if (lane == 0) st_bfs_arcs += d;
          for (int b = 0; b < d; b += 32) {
            int u = 0, cf = 0;
            if (b + lane < d) ops.in_arc(sg, b + lane, u, cf);
            aq_push(relax(b + lane < d, u, cf, hj), u);
          }
        }
        __syncwarp();
        if (lane == 0) atomicAdd(&GC->aq_pending[0], -got);   // after this warp's pushes
      }
      if (brank == 0 && threadIdx.x == 0) { ++l_levels; ring(ph)->kind = PK_ABFS; }
      if (!gsync()) return;
      state = S_COMPACT;
      continue;
    }

    if (state == S_BFS) {
      int qn = S.bc.qn, hc = S.bc.hc;
      if (qn + hc == 0) { state = S_COMPACT; continue; }
      {
        QueueOut o = out_for(fb ^ 1);
        unsigned fedges = 0;   // lane 0: slots of the vertices this warp appended
        if (!(S.bc.flags & 2)) {
          // ---- top-down: frontier vertex w, in-arcs u -> w with c_f > 0
          const int* qf = Q[fb];
          const HugeRec* hqf = HQ[fb];
          const int2* hcf = HC[fb];
          // frontier entries 32 per warp iteration: vertices with <= kBuThread slots are
          // scanned by one THREAD each (kBuB in-arcs per batch, independent loads), larger
          // ones by the whole warp (td_warp_scan), hub chunks one warp per chunk task
          // (packing 32 entries per warp pays only when the frontier outnumbers the warps)
          const int per = qn >= nwarps * kTdPack ? 32 : 1;
          // (the frontier entries of a warp's next iteration are loaded one iteration ahead)
          const bool ldr = per == 32 || lane == 0;
          int wv_next = (gwarp * per + (per == 32 ? lane : 0) < qn && ldr) ? ld_cg(qf + gwarp * per + (per == 32 ? lane : 0)) : 0;
          for (int base = gwarp * per; base < qn; base += nwarps * per) {
            const int tk = base + (per == 32 ? lane : 0);
            int wv = 0, dw = 0;
            Seg sw;
            const int wv_cur = wv_next;
            if (tk + nwarps * per < qn && ldr) wv_next = ld_cg(qf + tk + nwarps * per);
            if (tk < qn && ldr) { wv = wv_cur; sw = ops.seg(wv); dw = sw.deg(); }
            const bool thr = per == 32 && tk < qn && dw <= kTdThread;
            const int dthr = thr ? dw : 0;
            if (thr) st_bfs_arcs += dw;   // per-thread partial (block-summed at the end)
            for (int b0 = 0; __any_sync(FULL, b0 < dthr); b0 += kBuB) {
              int u[kBuB], cf[kBuB];
              // (16-B vector loads of the in-arcs, as the bottom-up scan does for out-arcs, were
              //  measured slower here: the c_f gathers dominate and the selects cost issue slots)
              int hu[kBuB];
#if WBPR_TD_LAZY
              int mk[kBuB];
#pragma unroll
              for (int j = 0; j < kBuB; ++j) {
                u[j] = 0; mk[j] = 0;
                if (b0 + j < dthr) ops.in_arc_col(sw, b0 + j, u[j], mk[j]);
              }
#pragma unroll
              for (int j = 0; j < kBuB; ++j) hu[j] = (b0 + j < dthr) ? ld_h(P.h + u[j], pl) : -1;
#pragma unroll
              for (int j = 0; j < kBuB; ++j) cf[j] = hu[j] == N ? ops.in_cf(mk[j]) : 0;   // only unlabelled neighbours
#else
#pragma unroll
              for (int j = 0; j < kBuB; ++j) {
                u[j] = 0; cf[j] = 0;
                if (b0 + j < dthr) ops.in_arc(sw, b0 + j, u[j], cf[j]);
              }
#pragma unroll
              for (int j = 0; j < kBuB; ++j) hu[j] = (b0 + j < dthr) ? ld_h(P.h + u[j], pl) : -1;   // with c_f (parallel)
#endif
              bool found[kBuB];
#pragma unroll
              for (int j = 0; j < kBuB; ++j) found[j] = cf[j] > 0 && hu[j] == N && atomicCAS(P.h + u[j], N, level + 1) == N;
              int dg[kBuB];
#pragma unroll
              for (int j = 0; j < kBuB; ++j) dg[j] = found[j] ? ops.degree(u[j]) : 0;
#pragma unroll
              for (int j = 0; j < kBuB; ++j) {
                if (!__ballot_sync(FULL, found[j])) continue;
                unsigned fsum = warp_sum((unsigned)dg[j]);
                if (lane == 0) fedges += fsum;
                const bool huge = found[j] && dg[j] > kChunk;
                if (huge) huge_append(u[j], dg[j], o, kChunk);
                warp_append(S, cnt, found[j] && !huge, u[j], o, dg[j]);
              }
            }
            unsigned todo = __ballot_sync(FULL, tk < qn && !thr && (per == 32 || lane == 0));
            while (todo) {
              const int j = __ffs(todo) - 1;
              todo &= todo - 1;
              const int wj = __shfl_sync(FULL, wv, j);
              Seg sg = ops.seg(wj);
              const int d = sg.deg();
              if (lane == 0) st_bfs_arcs += d;
              td_warp_scan(sg, 0, d, o, fedges);
            }
          }
          for (int t = gwarp; t < hc; t += nwarps) {
            int2 c = ld_cg(hcf + t);
            const int wv = ld_cg(&hqf[c.x].u);
            Seg sg = ops.seg(wv);
            const int lo = c.y * kChunk, hi = min(sg.deg(), lo + kChunk);
            if (lane == 0) st_bfs_arcs += hi - lo;
            td_warp_scan(sg, lo, hi, o, fedges);
          }
        } else {
          // ---- bottom-up: every unlabelled vertex v looks for an out-arc v -> w with
          // c_f > 0 and level(w) = level (early exit per 32-slot group)
          unsigned long long bu = 0;   // slots read by this level (12 B each, §5; top-down 16 B)
          // the label / frozen flag of the next 32-vertex group are loaded one iteration ahead
          int nbase = VLO + gwarp * 32;
          int hv_next = nbase + lane < VHI ? ld_cg_hint(P.h + nbase + lane, pl) : -1;
          uint8_t fz_next = nbase + lane < VHI ? ld_term(P.deact + nbase + lane) : 1;
          for (int base = nbase; base < VHI; base += nwarps * 32) {
            int v = base + lane;
            const int hv = hv_next;
            const uint8_t fz = fz_next;
            {
              const int nv = base + nwarps * 32 + lane;
              hv_next = nv < VHI ? ld_cg_hint(P.h + nv, pl) : -1;
              fz_next = nv < VHI ? ld_term(P.deact + nv) : 1;
            }
            // low-degree vertices (<= kBuThread slots, the bulk of a power-law graph): one
            // THREAD per vertex, kBuB independent arc loads then kBuB label gathers per batch
            // (early exit per batch); larger ones below, one warp per vertex
            bool self_hit = false;
            int dself = 0;
            Seg sv;
            sv.fb = sv.fe = sv.rb = sv.re = 0;
            const bool unl = hv == N && !(phase == 1 && fz);   // frozen: never reachable
            if (unl) { sv = ops.seg(v); dself = sv.deg(); }
            const bool thr = unl && dself <= kBuThread;
            if (thr) {
              int scanned = 0;
              for (int b0 = 0; b0 < dself && !self_hit; b0 += kBuB) {
                int col[kBuB], cf[kBuB];
                if constexpr (Ops::kVec8 && kBuB == 8) {
                  ops.arcs8(sv, b0, dself, col, cf);
                } else {
#pragma unroll
                  for (int j = 0; j < kBuB; ++j) {
                    col[j] = 0; cf[j] = 0;
                    if (b0 + j < dself) { int slot; ops.out_arc(sv, b0 + j, col[j], cf[j], slot); }
                  }
                }
                int hl[kBuB];
#pragma unroll
                for (int j = 0; j < kBuB; ++j) hl[j] = cf[j] > 0 ? ld_h(P.h + col[j], pl) : -1;
#pragma unroll
                for (int j = 0; j < kBuB; ++j) self_hit |= hl[j] == level;
                scanned += min(kBuB, dself - b0);
              }
              bu += scanned;   // per-thread partial; summed over the block at the end
              if (self_hit) st_cg(P.h + v, level + 1);
            }
            unsigned todo = __ballot_sync(FULL, unl && !thr);
            unsigned found_mask = __ballot_sync(FULL, self_hit);
            while (todo) {
              int j = __ffs(todo) - 1;
              todo &= todo - 1;
              int vv = base + j;
              Seg sg;                               // lane j loaded it above
              sg.fb = __shfl_sync(FULL, sv.fb, j); sg.fe = __shfl_sync(FULL, sv.fe, j);
              sg.rb = __shfl_sync(FULL, sv.rb, j); sg.re = __shfl_sync(FULL, sv.re, j);
              int d = sg.deg();
              if (d > kChunk) continue;            // hubs: static chunk tasks below
              int scanned = 0;
              const bool hit = bu_warp_scan(sg, 0, d, scanned);
              if (lane == 0) bu += scanned;
              if (hit) {
                found_mask |= 1u << j;
                if (lane == 0) st_cg(P.h + vv, level + 1);
              }
            }
            bool found = (found_mask >> lane) & 1u;
            int dg = found ? dself : 0;   // (dself = deg(v) for every unlabelled lane)
            unsigned fsum = warp_sum((unsigned)dg);
            if (lane == 0) fedges += fsum;
            warp_append(S, cnt, found, v, o, dg);
          }
          // unlabelled hubs: one warp per 1024-slot chunk, first finder labels (CAS)
          const int nhs = ld_cg(&GC->nhs);
          for (int t = gwarp; t < nhs; t += nwarps) {
            int2 hsk = ld_cg(HS + t);
            int vv = hsk.x;
            if (ld_cg_hint(P.h + vv, pl) != N || (phase == 1 && ld_term(P.deact + vv))) continue;
            Seg sg = ops.seg(vv);
            int lo2 = hsk.y * kChunk, hi2 = min(sg.deg(), lo2 + kChunk);
            int scanned = 0;
            const bool hit = bu_warp_scan(sg, lo2, hi2, scanned);
            if (lane == 0) {
              bu += scanned;
              if (hit && atomicCAS(P.h + vv, N, level + 1) == N) {
                huge_append(vv, sg.deg(), o, kChunk);
                fedges += sg.deg();
              }
            }
          }
          st_bfs_arcs += bu;
          const unsigned long long tb = block_sum_u64(S, bu);
          if (threadIdx.x == 0 && tb) atomicAdd((unsigned long long*)&C->stats[ST_BFS_BU], tb);
        }
        {
          unsigned long long t = block_sum_u64(S, (unsigned long long)fedges);
          if (threadIdx.x == 0 && t) atomicAdd(&ring(ph)->fedges, (unsigned)t);
        }
        block_flush_all(S, cnt, o);
        if (brank == 0 && threadIdx.x == 0) { ++l_levels; ring(ph)->kind = PK_BFS; ring(ph)->pad = level; }
      }
      if (!gsync()) return;
      fb ^= 1;
      ++level;
      continue;
    }

    if (state == S_COMPACT) {
      // ------------------------------------------------------------ full compaction (Alg. 2 l.1-4)
      // + Excess_total bookkeeping for vertices the GR found unable to reach a sink
      {
        QueueOut o = out_for(0);
        unsigned long long dropped = 0;
        if (P.gap_mode) {
          for (int i = threadIdx.x; i < kGapBins; i += blockDim.x) S.gbin[i] = 0;
          __syncthreads();
        }
        uint8_t c_tv = 1, c_fz = 1;
        int c_hv = N;
        long long c_ev = 0;
        {
          const int v0 = VLO + brank * blockDim.x + w * 32 + lane;
          if (v0 < VHI) { c_tv = ld_term(P.term + v0); c_hv = ld_cg(P.h + v0); c_ev = ld_cg(P.e + v0); c_fz = ld_term(P.deact + v0); }
        }
        for (int base = VLO + brank * blockDim.x + w * 32; base < VHI; base += nb * blockDim.x) {
          int v = base + lane;
          bool act = false, huge = false;
          int dg = 0;
          if (P.gap_mode && v < VHI) {
            int hv0 = ld_cg(P.h + v);
            if (hv0 < kGapBins) atomicAdd(&S.gbin[hv0], 1);
            else if (hv0 < N) atomicAdd(P.hist + hv0, 1);
          }
          // terminal flag, label, excess and frozen flag: loaded one iteration ahead
          const uint8_t tv = c_tv, fz = c_fz;
          const int hv = c_hv;
          const long long ev = c_ev;
          {
            const int nv = v + nb * blockDim.x;
            c_tv = 1; c_fz = 1; c_hv = N; c_ev = 0;
            if (nv < VHI) { c_tv = ld_term(P.term + nv); c_hv = ld_cg(P.h + nv); c_ev = ld_cg(P.e + nv); c_fz = ld_term(P.deact + nv); }
          }
          if (tv == 0) {
            if (hv < N) {
              if (ev > 0) {
                act = true;
                dg = ops.degree(v);
                huge = dg > kRChunk;
              }
            } else if (phase == 1 && !fz) {
              // v cannot reach a sink: it stays so for the rest of phase 1 (the set is closed,
              // §8(c) N5) - frozen: its excess leaves Excess_total once and later
              // bottom-up BFS levels skip it
              P.deact[v] = 1;
              if (ev > 0) dropped += (unsigned long long)ev;
            }
          }
          if (lane == 0) st_cand += min(32, VHI - base);
          if (huge) huge_append(v, dg, o, kRChunk);
          warp_append(S, cnt, act && !huge, v, o, dg);
        }
        block_flush_all(S, cnt, o);
        unsigned long long t = block_sum_u64(S, dropped);
        if (threadIdx.x == 0 && t) atomicAdd((unsigned long long*)&C->excess_total, (unsigned long long)(-(long long)t));
        if (brank == 0 && threadIdx.x == 0) ring(ph)->kind = PK_COMPACT;
        if (P.gap_mode)
          for (int i = threadIdx.x; i < kGapBins && i < N; i += blockDim.x)
            if (S.gbin[i]) atomicAdd(P.hist + i, S.gbin[i]);
      }
      if (!gsync()) return;
      cur = 0;
      // termination: right after an exact GR, no active vertex <=> e(s)+e(t) >= Excess_total
      state = (S.bc.qn + S.bc.hc == 0) ? S_DONE : S_ROUND;
      if (state == S_DONE) converged = true;
      if (P.debug_stop > 0 && grs_done >= P.debug_stop) {
        // debug_stop: export the AVQ the compaction just built (entries, then one entry per hub
        // vertex) and stop with the exact labels of this GR in h[] (tests of A3 / A5)
        if (brank == 0) {
          const int qn = S.bc.qn, hc = S.bc.hc;
          for (int t = threadIdx.x; t < hc; t += blockDim.x) {
            const int2 c = ld_cg(HC[0] + t);
            if (c.y == 0) st_cg(Q[0] + qn + atomicAdd(&C->dbg_hn, 1), ld_cg(&HQ[0][c.x].u));
          }
          if (threadIdx.x == 0) C->dbg_qn = qn;
        }
        state = S_DONE;
      }
      continue;
    }

    if (P.schedule == 1) {
      // ------------------------------------------------------------ thread-centric sweep
      // Alg. 1 Step 1: every thread tests its vertices for activity and scans
      // their residual arcs serially (NEXT #1: the paper's comparison baseline)
      if (brank == 0 && threadIdx.x == 0) { ++l_rounds; ring(ph)->kind = PK_ROUND; }
      unsigned long long active = 0;
      tc_work = 0;
      unsigned long long tt0; long long ta0, tp0, tr0c; int tn0;
      trace_begin(tt0, ta0, tp0, tr0c, tn0);
      for (int v = VLO + brank * blockDim.x + threadIdx.x; v < VHI; v += nb * blockDim.x) {
        if (ld_cg(P.e + v) > 0 && ld_term(P.term + v) == 0 && ld_cg(P.h + v) < N) {
          ++active;
          small_round_vertex(v, true);
        }
      }
      trace_end(tt0, ta0, tp0, tr0c, (int)warp_sum((int)active));
      ++trace_round;
      if (lane == 0) st_cand += 0;
      unsigned long long ta = block_sum_u64(S, active);
      unsigned long long tw = block_sum_u64(S, tc_work);
      if (threadIdx.x == 0) {
        if (ta) atomicAdd(&ring(ph)->qn, (int)ta);   // "queue" size = active vertices found
        if (tw) atomicAdd(&ring(ph)->work, (unsigned)(tw < 0x7fffffffull ? tw : 0x7fffffffull));
      }
      if (!gsync()) return;
      ++rounds;
      if (rounds >= P.max_rounds) {
        if (brank == 0 && threadIdx.x == 0) { C->status = DS_NOTCONVERGED; }
        state = S_DONE;
        continue;
      }
      if (S.bc.flags & 1) state = S_GR;
      continue;
    }

    // -------------------------------------------------------------- one push/relabel round
    {
      const unsigned long long tr0 = (brank == 0 && threadIdx.x == 0) ? globaltimer() : 0;
      const int qn = S.bc.qn, hc = S.bc.hc;
      if (brank == 0 && threadIdx.x == 0) {
        ++l_rounds;
        ring(ph)->kind = PK_ROUND;
      }
      QueueOut o = out_for(cur ^ 1);
      const int* qc = Q[cur];
      HugeRec* hqc = HQ[cur];
      const int2* hcc = HC[cur];
      unsigned long long work = 0;
      const int total = qn + hc;
      unsigned long long tt0; long long ta0, tp0, tr0c; int tn0;
      trace_begin(tt0, ta0, tp0, tr0c, tn0);
      // thread-serial discharge of vertex u (<= kRThr slots) by one lane: the same semantics as
      // the warp discharge below (pushes to every admissible arc in slot order, budget split,
      // relabel to min + 1 only when none is admissible); appends are warp-collective
      auto thread_discharge = [&](bool thr, int u, const Seg& sg, int d, int hu, long long eu, const QueueOut& oq,
                                  unsigned long long& wk) {
        unsigned long long best = ~0ull;
        long long budget = eu, pushed = 0;
        int scanned = 0;
        for (int b0 = 0; __any_sync(FULL, thr && b0 < d && budget > 0); b0 += 8) {
          const bool act = thr && b0 < d && budget > 0;
          int col[8], cf[8], sl[8];
          if constexpr (Ops::kVec8) {
            if (act) ops.arcs8(sg, b0, d, col, cf);
            else {
#pragma unroll
              for (int j = 0; j < 8; ++j) { col[j] = 0; cf[j] = 0; }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) sl[j] = sg.fb + b0 + j;
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              col[j] = 0; cf[j] = 0; sl[j] = 0;
              if (act && b0 + j < d) ops.out_arc(sg, b0 + j, col[j], cf[j], sl[j]);
            }
          }
          if (act) scanned += min(8, d - b0);
          int hv[8], ax[8], dg[8];
          uint8_t tm[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            hv[j] = cf[j] > 0 ? ld_h(P.h + col[j], pl) : INT_MAX;
            ax[j] = cf[j] > 0 ? ops.aux(sl[j]) : 0;
            dg[j] = cf[j] > 0 ? ops.degree(col[j]) : 0;
            tm[j] = cf[j] > 0 ? ld_term(P.term + col[j]) : 1;
          }
          bool app[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            app[j] = false;
            if (cf[j] > 0) {
              const unsigned long long cand = ((unsigned long long)(unsigned)hv[j] << 32) | (unsigned)sl[j];
              if (cand < best) best = cand;
            }
            if (cf[j] > 0 && hv[j] < hu && budget > 0) {
              const int dd = (int)(budget < (long long)cf[j] ? budget : (long long)cf[j]);
              ops.push_aux(sl[j], ax[j], dd);
              const long long old_v = (long long)atomicAdd((unsigned long long*)(P.e + col[j]), (unsigned long long)dd);
              app[j] = old_v == 0 && tm[j] == 0;
              budget -= dd;
              pushed += dd;
              ++st_push;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool hg = app[j] && dg[j] > kRChunk;
            if (hg) huge_append(col[j], dg[j], oq, kRChunk);
            warp_append(S, cnt, app[j] && !hg, col[j], oq, dg[j]);
          }
        }
        st_arcs += scanned;
        bool app_u = false;
        if (thr) {
          if (pushed > 0) {
            const long long old_u = (long long)atomicAdd((unsigned long long*)(P.e + u), (unsigned long long)(-pushed));
            app_u = old_u - pushed > 0;
          } else {
            const unsigned hmin = (unsigned)(best >> 32);
            const int nh = (best == ~0ull || (int)hmin >= N - 1) ? N : (int)hmin + 1;
            st_cg(P.h + u, nh);
            gap_relabel(hu, nh);
            app_u = nh < N;
            wk += (unsigned long long)d + 1;
            ++st_relabel;
          }
        }
        warp_append(S, cnt, app_u, u, oq, d);
      };
      // one task: vertex u, or chunk [lo, lo + kRChunk) of hub record hidx (the whole warp)
      auto run_task = [&](int u, int lo, int hidx) {
        // independent loads issued together: segment bounds, h(u), e(u)
        Seg sg = ops.seg(u);
        const int hu = ld_cg(P.h + u);
        const long long eu = ld_cg(P.e + u);
        if (hu >= N) return;     // lifted by the gap heuristic: inactive until the next GR
        int hi;
        if (hidx < 0) { lo = 0; hi = sg.deg(); } else { hi = min(sg.deg(), lo + kRChunk); }
        if (lane == 0) st_arcs += hi - lo;

        unsigned long long best = ~0ull;   // (h, slot) minimum over residual arcs (Alg. 1 l.10-13)
        int bcf = 0, bcol = 0;
        long long pushed = 0;              // discharge: excess moved by this warp
        if (P.push_mode == 0) {
          // ---- second-level parallelism: lanes scan the residual arcs
#pragma unroll 2
          for (int i = lo + lane; i < hi; i += 32) {
            int col, cf, slot;
            ops.out_arc(sg, i, col, cf, slot);
            if (cf > 0) {
              unsigned hv = (unsigned)ld_h(P.h + col, pl);
              unsigned long long cand = ((unsigned long long)hv << 32) | (unsigned)slot;
              if (cand < best) { best = cand; bcf = cf; bcol = col; }
            }
          }
        } else {
          // ---- warp-parallel discharge: every admissible arc (h(v) < h(u), relaxed rule
          // P:187-189) of this 32-slot group receives part of the remaining budget, split
          // by an exclusive prefix sum of the residual capacities in slot order.
          long long snap = eu;             // lower bound of e(u) (only u's warps decrease it)
          long long budget = eu;           // normal task: local budget
          // kRU groups of 32 slots per iteration: all arc loads, then all label gathers,
          // then the pushes, then the appends, so each dependent memory step is paid once
          // per 32*kRU slots instead of once per 32 (memory-level parallelism)
          for (int b0 = lo; b0 < hi; b0 += 32 * kRU) {
            int col[kRU], cf[kRU], slot[kRU], hv[kRU];
#pragma unroll
            for (int j = 0; j < kRU; ++j) {
              const int i = b0 + j * 32 + lane;
              col[j] = 0; cf[j] = 0; slot[j] = 0;
              if (i < hi) ops.out_arc(sg, i, col[j], cf[j], slot[j]);
            }
#pragma unroll
            for (int j = 0; j < kRU; ++j) hv[j] = cf[j] > 0 ? ld_h(P.h + col[j], pl) : INT_MAX;
            // a task of <= 32 slots (road-like / matching graphs: latency-bound rounds) loads the
            // reverse-arc lookup, terminal flag and degree of every residual arc together with
            // the labels, so a push costs no further dependent round trips
            const bool shortt = hi - lo <= 32;
            int ax0 = 0, dg0 = 0;
            uint8_t tm0 = 1;
            if (shortt && cf[0] > 0) { ax0 = ops.aux(slot[0]); dg0 = ops.degree(col[0]); tm0 = ld_term(P.term + col[0]); }
            long long want = 0;            // admissible capacity of the whole super-group
            unsigned amask = 0;            // groups with an admissible arc
#pragma unroll
            for (int j = 0; j < kRU; ++j) {
              if (cf[j] > 0) {
                unsigned long long cand = ((unsigned long long)(unsigned)hv[j] << 32) | (unsigned)slot[j];
                if (cand < best) { best = cand; bcf = cf[j]; bcol = col[j]; }
              }
              const bool adm = cf[j] > 0 && hv[j] < hu;
              if (__ballot_sync(FULL, adm)) amask |= 1u << j;
              want += adm ? (long long)cf[j] : 0;
            }
            if (!amask) continue;
            want = warp_sum(want);
            long long avail;
            if (hidx < 0) {
              avail = budget;
            } else {
              long long got = 0;
              if (lane == 0) got = (long long)atomicAdd((unsigned long long*)&hqc[hidx].spent, (unsigned long long)want);
              got = __shfl_sync(FULL, got, 0);
              avail = snap - got;
              if (avail < 0) avail = 0;
            }
            // split avail over the admissible arcs in slot order (group-major, then lane)
            long long before = 0;          // admissible capacity of the earlier groups
            long long oldv[kRU];
#pragma unroll
            for (int j = 0; j < kRU; ++j) {
              oldv[j] = -1;
              if (!((amask >> j) & 1u)) continue;
              const bool adm = cf[j] > 0 && hv[j] < hu;
              const long long c = adm ? cf[j] : 0;
              long long incl = c;
#pragma unroll
              for (int o2 = 1; o2 < 32; o2 <<= 1) {
                long long y = __shfl_up_sync(FULL, incl, o2);
                if (lane >= o2) incl += y;
              }
              const long long excl = before + incl - c;
              before += __shfl_sync(FULL, incl, 31);
              const long long d = adm ? (avail - excl < c ? avail - excl : c) : 0;
              if (d > 0) {
                if (shortt && j == 0) ops.push_aux(slot[0], ax0, (int)d);
                else ops.push(slot[j], (int)d);
                oldv[j] = (long long)atomicAdd((unsigned long long*)(P.e + col[j]), (unsigned long long)d);
                ++st_push;
              }
            }
            const long long used = want < avail ? want : avail;
            pushed += used;
            budget -= used;
            // a push that raised e(v) from 0 appends v (exactly once, atomics on e)
            bool app[kRU];
#pragma unroll
            for (int j = 0; j < kRU; ++j)
              app[j] = oldv[j] == 0 && ((shortt && j == 0) ? tm0 == 0 : ld_term(P.term + col[j]) == 0);
            int dgv[kRU];
#pragma unroll
            for (int j = 0; j < kRU; ++j) dgv[j] = app[j] ? ((shortt && j == 0) ? dg0 : ops.degree(col[j])) : 0;
#pragma unroll
            for (int j = 0; j < kRU; ++j) {
              if (!((amask >> j) & 1u)) continue;
              const bool hugev = app[j] && dgv[j] > kRChunk;
              if (hugev) huge_append(col[j], dgv[j], o, kRChunk);
              warp_append(S, cnt, app[j] && !hugev, col[j], o, dgv[j]);
            }
            if (hidx < 0 && budget <= 0) break;
          }
        }
        // warp minimum (redux.sync) of the (h, slot) candidates
        unsigned hmin = __reduce_min_sync(FULL, (unsigned)(best >> 32));
        unsigned smin = __reduce_min_sync(FULL, (unsigned)(best >> 32) == hmin ? (unsigned)best : kInf);
        unsigned long long wbest = ((unsigned long long)hmin << 32) | smin;
        unsigned owner = __ballot_sync(FULL, best == wbest && best != ~0ull);
        int src_lane = owner ? __ffs(owner) - 1 : 0;
        int cfv = __shfl_sync(FULL, bcf, src_lane);
        int colv = __shfl_sync(FULL, bcol, src_lane);
        if (hidx >= 0) {
          // fold this chunk into the vertex record; the last chunk finalizes
          int last = 0;
          if (lane == 0) {
            if (wbest != ~0ull) atomicMin(&hqc[hidx].best, wbest);
            if (pushed) atomicAdd((unsigned long long*)&hqc[hidx].pushed, (unsigned long long)pushed);
            __threadfence();
            int nch = ld_cg(&hqc[hidx].nchunks);
            last = (atomicAdd(&hqc[hidx].done, 1) == nch - 1);
            if (last) {
              __threadfence();
              wbest = ld_cg(&hqc[hidx].best);
              pushed = ld_cg(&hqc[hidx].pushed);
              if (wbest != ~0ull) ops.col_cf_of_slot((int)(wbest & 0xffffffffu), colv, cfv);
            }
          }
          if (!__shfl_sync(FULL, last, 0)) return;
          wbest = __shfl_sync(FULL, wbest, 0);
          colv = __shfl_sync(FULL, colv, 0);
          cfv = __shfl_sync(FULL, cfv, 0);
          pushed = __shfl_sync(FULL, pushed, 0);
          hmin = (unsigned)(wbest >> 32);
        }
        // delegated lane 0: push or relabel
        int app_u = -1, app_v = -1, dgu = 0, dgv = 0;
        if (lane == 0) {
          if (P.push_mode == 0 && hmin != kInf && (int)hmin < hu && cfv > 0) {
            // push: d = min(e(u), c_f(u,v')) (Alg. 1 line 15), four atomics (lines 16-19)
            const int dv = ops.degree(colv);
            int d = (int)(eu < (long long)cfv ? eu : (long long)cfv);
            int slot = (int)(wbest & 0xffffffffu);
            ops.push(slot, d);
            long long old_u = (long long)atomicAdd((unsigned long long*)(P.e + u), (unsigned long long)(-(long long)d));
            long long old_v = (long long)atomicAdd((unsigned long long*)(P.e + colv), (unsigned long long)d);
            if (old_u - d > 0) { app_u = u; dgu = sg.deg(); }
            if (old_v == 0 && ld_term(P.term + colv) == 0) { app_v = colv; dgv = dv; }
            ++st_push;
          } else if (P.push_mode != 0 && pushed > 0) {
            long long old_u = (long long)atomicAdd((unsigned long long*)(P.e + u), (unsigned long long)(-pushed));
            if (old_u - pushed > 0) { app_u = u; dgu = sg.deg(); }
          } else {
            // relabel: h(u) <- h' + 1 (Alg. 1 line 21); >= |V| deactivates
            int nh = (hmin == kInf || (int)hmin >= N - 1) ? N : (int)hmin + 1;
            st_cg(P.h + u, nh);
            gap_relabel(hu, nh);
            if (nh < N) { app_u = u; dgu = sg.deg(); }
            work += (unsigned long long)sg.deg() + 1;
            ++st_relabel;
          }
          if (app_u >= 0 && dgu > kRChunk) { huge_append(app_u, dgu, o, kRChunk); app_u = -1; }
          if (app_v >= 0 && dgv > kRChunk) { huge_append(app_v, dgv, o, kRChunk); app_v = -1; }
        }
        warp_append(S, cnt, lane == 0 && app_u >= 0, app_u, o, dgu);
        warp_append(S, cnt, lane == 0 && app_v >= 0, app_v, o, dgv);
      };
      // many active vertices (e.g. the first rounds of a matching, ~10^6 of them): 32 queue
      // entries per warp, those with <= kRThr slots discharged by one THREAD each (8-slot
      // batches, all loads of a batch in flight together), the rest by the whole warp
      // (only when no queued vertex has more than kRThr slots: a warp that met big vertices among
      //  its 32 entries would run them one after another - skewed graphs keep the warp mode)
      const bool thread_mode = P.push_mode != 0 && qn >= nwarps * kRThrPack && hc == 0 && (S.bc.flags & 64);
      if (thread_mode) {
        for (int t = gwarp; t < hc; t += nwarps) {
          ++tn0;
          const int2 c = ld_cg(hcc + t);
          run_task(ld_cg(&hqc[c.x].u), c.y * kRChunk, c.x);
        }
        for (int base = gwarp * 32; base < qn; base += nwarps * 32) {
          ++tn0;
          const int tk = base + lane;
          const int u = tk < qn ? ld_cg(qc + tk) : -1;
          Seg sg;
          sg.fb = sg.fe = sg.rb = sg.re = 0;
          int hu = N;
          long long eu = 0;
          if (u >= 0) { sg = ops.seg(u); hu = ld_cg(P.h + u); eu = ld_cg(P.e + u); }
          const int d = sg.deg();
          const bool thr = u >= 0 && hu < N && d <= kRThr;
          thread_discharge(thr, u, sg, d, hu, eu, o, work);
          unsigned todo = __ballot_sync(FULL, u >= 0 && hu < N && !thr);
          while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            run_task(__shfl_sync(FULL, u, j), 0, -1);
          }
        }
      } else {
      // the queue entry of a warp's next task is loaded while the current one runs
      int u_next = gwarp < qn ? ld_cg(qc + gwarp) : 0;
      for (int tk = gwarp; tk < total; tk += nwarps) {
        ++tn0;
        int u, lo = 0, hidx = -1;
        if (tk < qn) {
          u = u_next;
          if (tk + nwarps < qn) u_next = ld_cg(qc + tk + nwarps);
        } else {
          int2 c = ld_cg(hcc + (tk - qn));
          hidx = c.x;
          lo = c.y * kRChunk;
          u = ld_cg(&hqc[hidx].u);
        }
        run_task(u, lo, hidx);
      }
      }
      trace_end(tt0, ta0, tp0, tr0c, tn0);
      ++trace_round;
      const unsigned long long tf0 = (brank == 0 && threadIdx.x == 0) ? globaltimer() : 0;
      block_flush_all(S, cnt, o);
      unsigned long long t = block_sum_u64(S, work);
      if (threadIdx.x == 0 && t) atomicAdd(&ring(ph)->work, (unsigned)(t < 0x7fffffffull ? t : 0x7fffffffull));
      if (brank == 0 && threadIdx.x == 0) { t_flush += globaltimer() - tf0; t_round += tf0 - tr0; }
      if (!gsync()) return;
      cur ^= 1;
      ++rounds;
      if (rounds >= P.max_rounds) {
        if (brank == 0 && threadIdx.x == 0) { C->status = DS_NOTCONVERGED; }
        state = S_DONE;
        continue;
      }
      // early break / periodic GR, decided by the barrier's last arriver
      if (S.bc.flags & 1) state = S_GR;
    }
  }
  // ---------------------------------------------------------------- phase 2 (NEXT #2)
  // The maximum preflow is final: e(t) = F and the labels give S*.  Save them, swap the
  // terminal roles and run the same loop toward the sources, which returns every
  // stranded unit of excess to s through the residual arcs (a true flow).
  if (phase == 1 && P.phase2 && converged) {
    for (int v = VLO + brank * blockDim.x + threadIdx.x; v < VHI; v += nb * blockDim.x) {
      st_cg(P.h1 + v, ld_cg(P.h + v));
      uint8_t tv = P.term[v];
      P.term[v] = (uint8_t)(((tv & kSource) ? kSink : 0) | ((tv & kSink) ? kSource : 0));
    }
    SNK = P.src + I0;
    phase = 2;
    converged = false;
    state = S_GR;
    if (!gsync()) return;
    continue;
  }
  break;
  }

  // ---------------------------------------------------------------- statistics
  if (brank == 0 && threadIdx.x == 0) {   // rounds / GRs / levels: max over the groups
    atomicMax((unsigned long long*)&C->stats[ST_ROUNDS], (unsigned long long)l_rounds);
    atomicMax((unsigned long long*)&C->stats[ST_GRS], (unsigned long long)l_grs);
    atomicMax((unsigned long long*)&C->stats[ST_BFS_LEVELS], (unsigned long long)l_levels);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    C->stats[ST_COUNT - 3] = (long long)t_sync;
    C->stats[ST_COUNT - 2] = (long long)t_flush;
    C->stats[ST_COUNT - 1] = (long long)t_round;
  }
  {
    long long v[5] = {st_push, st_relabel, st_arcs, st_bfs_arcs, st_cand};
    int idx[5] = {ST_PUSHES, ST_RELABELS, ST_ARCS, ST_BFS_ARCS, ST_CAND};
    for (int i = 0; i < 5; ++i) {
      unsigned long long t = block_sum_u64(S, (unsigned long long)v[i]);
      if (threadIdx.x == 0 && t) atomicAdd((unsigned long long*)&C->stats[idx[i]], t);
    }
  }
}

// ------------------------------------------------------------------ barrier-latency probe
// The cost of one EMPTY grid-synchronous phase of k_solve (the latency floor of the
// phase-bound workloads): the same arrival (one acq_rel atomic per
// CTA), last-arriver bookkeeping (two 16-B ring loads + the abort word, one 16-B release
// store) and acquire polling, with no work between barriers.  Same CTA size, co-resident grid.
__device__ GroupCtrl g_probe_gc;
__device__ int g_probe_abort;
__global__ void __launch_bounds__(kSolveThreads, 1) k_barrier_probe(int iters, unsigned long long* out_ns) {
  __shared__ uint4 sb;
  GroupCtrl* GC = &g_probe_gc;
  const unsigned nb = gridDim.x;
  const unsigned long long t0 = globaltimer();
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)it + 1;
      uint4 b;
      if (atom_add_acqrel(&GC->bar.count, 1u) == nb - 1) {
        GC->bar.count = 0;
        Ring* r = &GC->ring[it % 3];
        const int4 r0 = ld_cg(reinterpret_cast<const int4*>(r));
        const int4 r1 = ld_cg(reinterpret_cast<const int4*>(r) + 1);
        const int ab = ld_volatile(&g_probe_abort);
        b = make_uint4(target, (unsigned)(r0.x + r1.x), (unsigned)ab, 0u);
        st_release_v4(&GC->bc, b);
      } else {
        unsigned ns = 0;
        do {
          b = ld_acquire_v4(&GC->bc);
          if (b.x == target) break;
          if (ns) __nanosleep(ns);
          ns = ns ? (ns < 128 ? ns * 2 : 128) : 16;
        } while (true);
      }
      sb = b;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out_ns = globaltimer() - t0;
}

cudaError_t barrier_probe(int blocks, int iters, double* ns_per_barrier, cudaStream_t st) {
  GroupCtrl z{};
  cudaError_t e = cudaMemcpyToSymbolAsync(g_probe_gc, &z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  if (e) return e;
  unsigned long long* d = nullptr;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), st))) return e;
  void* args[] = {(void*)&iters, (void*)&d};
  note_launch();
  e = cudaLaunchCooperativeKernel((const void*)k_barrier_probe, dim3(blocks), dim3(kSolveThreads), args, 0, st);
  unsigned long long ns = 0;
  if (!e) e = cudaMemcpyAsync(&ns, d, sizeof(ns), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (!e) e = cudaStreamSynchronize(st);
  if (!e) *ns_per_barrier = (double)ns / (double)(iters > 0 ? iters : 1);
  return e;
}

// ------------------------------------------------------------------ host launch
// Two register budgets: MINB = 2 (64 registers, 2 CTAs / 32 warps per SM, some spills) and
// MINB = 1 (128 registers, 1 CTA / 16 warps per SM, no spills).  WBPR_SOLVE_MINB picks one
// (default kSolveMinBlocks).
static int solve_minb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("WBPR_SOLVE_MINB");
    v = (e && (e[0] == '1' || e[0] == '2')) ? e[0] - '0' : kSolveMinBlocks;
  }
  return v;
}

template <class Ops> static const void* solve_fn() {
  return solve_minb() == 1 ? (const void*)k_solve<Ops, 1> : (const void*)k_solve<Ops, kSolveMinBlocks>;
}

int solve_max_blocks_per_sm(int layout, int threads) {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, layout == 0 ? solve_fn<BcsrOps>() : solve_fn<RcsrOps>(), threads, 0);
  return b;
}

cudaError_t launch_solve(const SolveParams& p, int blocks, int threads, cudaStream_t st) {
  note_launch();
  if (p.layout == 0) {
    BcsrOps o{p.seg, p.arc, p.mate};
    void* args[] = {(void*)&p, (void*)&o};
    return cudaLaunchCooperativeKernel(solve_fn<BcsrOps>(), dim3(blocks), dim3(threads), args, 0, st);
  } else {
    RcsrOps o{p.off, p.arc, p.roff, p.rarc, p.bcf, p.Mf};
    void* args[] = {(void*)&p, (void*)&o};
    return cudaLaunchCooperativeKernel(solve_fn<RcsrOps>(), dim3(blocks), dim3(threads), args, 0, st);
  }
}

}  // namespace wbpr
