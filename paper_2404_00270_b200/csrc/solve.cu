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
  const int* off; int2* arc; const int* mate;
  __device__ Seg seg(int u) const { Seg s; s.fb = __ldg(off + u); s.fe = __ldg(off + u + 1); s.rb = s.re = 0; return s; }
  __device__ int degree(int u) const { return __ldg(off + u + 1) - __ldg(off + u); }
  // residual out-arc #i of u: u -> col with residual capacity cf, identified by slot
  __device__ void out_arc(const Seg& s, int i, int& col, int& cf, int& slot) const {
    slot = s.fb + i;
    int2 a = ld_cg(arc + slot);
    col = a.x; cf = a.y;
  }
  // residual in-arc #i of w: col -> w with capacity cf(col -> w)
  __device__ void in_arc(const Seg& s, int i, int& col, int& cf) const {
    int p = s.fb + i;
    col = __ldg(&arc[p].x);
    cf = ld_cg(&arc[__ldg(mate + p)].y);
  }
  __device__ void col_cf_of_slot(int slot, int& col, int& cf) const {
    int2 a = ld_cg(arc + slot); col = a.x; cf = a.y;
  }
  __device__ void push(int slot, int d) const {
    atomicAdd(&arc[slot].y, -d);
    atomicAdd(&arc[__ldg(mate + slot)].y, d);
  }
  __device__ void saturate(int slot, int d) const { push(slot, d); }
};

struct RcsrOps {
  const int* foff; int2* farc; const int* roff; const int2* rarc; int* bcf; int Mf;
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
      int2 a = ld_cg(farc + slot);
      col = a.x; cf = a.y;
    } else {
      int q = s.rb + (i - df);
      int2 r = __ldg(rarc + q);            // {col, flow_idx}
      col = r.x;
      cf = ld_cg(bcf + r.y);               // backward cf: flow on col -> u that can return
      slot = Mf + q;
    }
  }
  __device__ void in_arc(const Seg& s, int i, int& col, int& cf) const {
    int df = s.fe - s.fb;
    if (i < df) {                          // w -> col forward: col -> w is its backward arc
      int p = s.fb + i;
      col = __ldg(&farc[p].x);
      cf = ld_cg(bcf + p);
    } else {                               // col -> w forward arc f
      int2 r = __ldg(rarc + s.rb + (i - df));
      col = r.x;
      cf = ld_cg(&farc[r.y].y);
    }
  }
  __device__ void col_cf_of_slot(int slot, int& col, int& cf) const {
    if (slot < Mf) { int2 a = ld_cg(farc + slot); col = a.x; cf = a.y; }
    else { int2 r = __ldg(rarc + (slot - Mf)); col = r.x; cf = ld_cg(bcf + r.y); }
  }
  __device__ void push(int slot, int d) const {
    if (slot < Mf) { atomicAdd(&farc[slot].y, -d); atomicAdd(bcf + slot, d); }
    else { int f = __ldg(&rarc[slot - Mf].y); atomicAdd(bcf + f, -d); atomicAdd(&farc[f].y, d); }
  }
};

// ------------------------------------------------------------------ warp append buffers
struct SharedState {
  int buf[kWarps][kBufCap];
  int cnt[kWarps];
  int wsum[kWarps];
  unsigned long long wsum64[kWarps];
  int base;
  Ring ring;          // post-barrier broadcast of the finalized ring slot
};

struct QueueOut {   // next-queue destination
  int* q; int* qn;
  HugeRec* hq; int2* hc; int* hn; int* hc_cnt;
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
__device__ __forceinline__ void warp_append(SharedState& S, int& cnt, bool pred, int val, const QueueOut& out) {
  unsigned b = __ballot_sync(FULL, pred);
  if (!b) return;
  int w = warp_id();
  if (pred) S.buf[w][cnt + __popc(b & lanemask_lt())] = val;
  cnt += __popc(b);
  if (cnt >= kBufFlush) warp_flush(S, cnt, out);
}

// a vertex with more than kChunk slots becomes nchunks warp tasks (single lane)
__device__ __forceinline__ void huge_append(int u, int deg, const QueueOut& out) {
  int nch = (deg + kChunk - 1) / kChunk;
  int hi = atomicAdd(out.hn, 1);
  int c0 = atomicAdd(out.hc_cnt, nch);
  HugeRec r; r.best = ~0ull; r.u = u; r.nchunks = nch; r.done = 0; r.pad = 0;
  out.hq[hi] = r;
  for (int j = 0; j < nch; ++j) out.hc[c0 + j] = make_int2(hi, j);
}

// ------------------------------------------------------------------ the kernel
template <class Ops>
struct Solver {
  const SolveParams& P;
  Ops ops;
  __device__ Solver(const SolveParams& p, const Ops& o) : P(p), ops(o) {}
};

template <class Ops>
__device__ __forceinline__ void block_flush_all(SharedState& S, int& cnt, const QueueOut& out) {
  // block-aggregated final flush: one global atomic per CTA
  int lane = lane_id(), w = warp_id();
  if (lane == 0) S.wsum[w] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kWarps; ++i) { int c = S.wsum[i]; S.wsum[i] = tot; tot += c; }
    S.base = tot ? atomicAdd(out.qn, tot) : 0;
  }
  __syncthreads();
  int base = S.base + S.wsum[w];
  for (int i = lane; i < cnt; i += 32) st_cg(out.q + base + i, S.buf[w][i]);
  cnt = 0;
  __syncthreads();
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

template <class Ops>
__global__ void __launch_bounds__(kSolveThreads) k_solve(const SolveParams P, const Ops ops) {
  __shared__ SharedState S;
  Ctrl* C = P.ctrl;
  const int N = P.n;
  const unsigned nb = gridDim.x;
  const int lane = lane_id(), w = warp_id();
  const int gwarp = blockIdx.x * kWarps + w;
  const int nwarps = gridDim.x * kWarps;
  unsigned gen = 0;
  int ph = 0;
  const unsigned long long deadline = globaltimer() + P.deadline_ns_rel;
  // per-warp statistics (registers)
  long long st_push = 0, st_relabel = 0, st_arcs = 0, st_bfs_arcs = 0, st_cand = 0;
  int cnt = 0;  // this warp's staged appends (lane-uniform)

  auto ring = [&](int p) -> Ring* { return &C->ring[((p % 3) + 3) % 3]; };
  auto out_for = [&](int buf) {
    QueueOut o;
    o.q = P.q[buf]; o.qn = &ring(ph)->qn;
    o.hq = P.hq[buf]; o.hc = P.hc[buf]; o.hn = &ring(ph)->hn; o.hc_cnt = &ring(ph)->hc;
    return o;
  };
  // barrier + ring rotation + broadcast of the finalized counters
  auto gsync = [&]() -> bool {
    bool ok = grid_sync(&C->bar, nb, gen, &C->abort, deadline);
    ++ph;
    if (threadIdx.x == 0) {
      Ring* r = ring(ph - 1);
      S.ring.work = ld_cg(&r->work);
      S.ring.qn = ld_cg(&r->qn);
      S.ring.hn = ld_cg(&r->hn);
      S.ring.hc = ld_cg(&r->hc);
      if (blockIdx.x == 0) {
        Ring* z = ring(ph + 1);
        z->work = 0; z->qn = 0; z->hn = 0; z->hc = 0;
      }
    }
    __syncthreads();
    return ok;
  };

  // ---------------------------------------------------------------- init
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += nb * blockDim.x) {
    st_cg(P.e + v, 0ll);
    P.deact[v] = 0;
  }
  if (!gsync()) return;

  // ---------------------------------------------------------------- preflow (Alg. 1 Step 0)
  {
    unsigned long long exc = 0;
    for (int i = 0; i < P.k; ++i) {
      int s = (int)P.src[i];
      Seg sg = ops.seg(s);
      int d = sg.deg();
      for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += nb * blockDim.x) {
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
  }
  if (!gsync()) return;

  long long rounds = 0;
  unsigned long long work_since_gr = 0;
  int cur = 0;          // queue buffer holding the current AVQ
  bool need_gr = true;
  bool done = false;

  while (!done) {
    if (need_gr) {
      // ------------------------------------------------------------ global relabel
      // reset labels: sinks 0, everything else |V| (= unreached); frontier <- sinks
      for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += nb * blockDim.x)
        st_cg(P.h + v, (__ldg(P.term + v) & kSink) ? 0 : N);
      if (blockIdx.x == 0) {
        QueueOut o = out_for(0);
        for (int base = w * 32; base < P.k; base += kWarps * 32) {
          int i = base + lane;
          int t = i < P.k ? (int)P.snk[i] : 0;
          int dg = i < P.k ? ops.degree(t) : 0;
          bool huge = i < P.k && dg > kChunk;
          if (huge) huge_append(t, dg, o);
          warp_append(S, cnt, i < P.k && !huge, t, o);
        }
        block_flush_all<Ops>(S, cnt, o);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) C->stats[ST_GRS]++;
      if (!gsync()) return;
      int fb = 0, level = 0;
      while (true) {
        int qn = S.ring.qn, hc = S.ring.hc;
        if (qn + hc == 0) break;
        QueueOut o = out_for(fb ^ 1);
        const int* qf = P.q[fb];
        const HugeRec* hqf = P.hq[fb];
        const int2* hcf = P.hc[fb];
        int total = qn + hc;
        for (int tk = gwarp; tk < total; tk += nwarps) {
          int wv, lo, hi;
          Seg sg;
          if (tk < qn) {
            wv = ld_cg(qf + tk);
            sg = ops.seg(wv); lo = 0; hi = sg.deg();
          } else {
            int2 c = ld_cg(hcf + (tk - qn));
            wv = ld_cg(&hqf[c.x].u);
            sg = ops.seg(wv);
            lo = c.y * kChunk; hi = min(sg.deg(), lo + kChunk);
          }
          st_bfs_arcs += hi - lo;
          for (int b = lo; b < hi; b += 32) {
            int i = b + lane;
            bool found = false;
            int u = 0, dg = 0;
            if (i < hi) {
              int cf;
              ops.in_arc(sg, i, u, cf);
              if (cf > 0 && __ldg(P.term + u) == 0 && ld_cg(P.h + u) == N) {
                if (atomicCAS(P.h + u, N, level + 1) == N) {   // level(u) = level(w) + 1
                  found = true;
                  dg = ops.degree(u);
                }
              }
            }
            bool huge = found && dg > kChunk;
            if (huge) huge_append(u, dg, o);
            warp_append(S, cnt, found && !huge, u, o);
          }
        }
        block_flush_all<Ops>(S, cnt, o);
        if (blockIdx.x == 0 && threadIdx.x == 0) C->stats[ST_BFS_LEVELS]++;
        if (!gsync()) return;
        fb ^= 1;
        ++level;
      }
      // ------------------------------------------------------------ full compaction (Alg. 2 l.1-4)
      // + Excess_total bookkeeping for vertices the GR found unable to reach a sink
      {
        QueueOut o = out_for(0);
        unsigned long long dropped = 0;
        for (int base = blockIdx.x * blockDim.x + w * 32; base < N; base += nb * blockDim.x) {
          int v = base + lane;
          bool act = false, huge = false;
          int dg = 0;
          if (v < N) {
            long long ev = ld_cg(P.e + v);
            if (ev > 0 && __ldg(P.term + v) == 0) {
              int hv = ld_cg(P.h + v);
              if (hv < N) {
                act = true;
                dg = ops.degree(v);
                huge = dg > kChunk;
              } else if (!P.deact[v]) {
                P.deact[v] = 1;
                dropped += (unsigned long long)ev;
              }
            }
          }
          st_cand += min(32, N - base);
          if (huge) huge_append(v, dg, o);
          warp_append(S, cnt, act && !huge, v, o);
        }
        block_flush_all<Ops>(S, cnt, o);
        unsigned long long t = block_sum_u64(S, dropped);
        if (threadIdx.x == 0 && t) atomicAdd((unsigned long long*)&C->excess_total, (unsigned long long)(-(long long)t));
      }
      if (!gsync()) return;
      cur = 0;
      work_since_gr = 0;
      need_gr = false;
      // termination: right after an exact GR, no active vertex <=> e(s)+e(t) >= Excess_total
      if (S.ring.qn + S.ring.hn == 0) { done = true; break; }
    }

    // -------------------------------------------------------------- one push/relabel round
    {
      int qn = S.ring.qn, hc = S.ring.hc;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        C->stats[ST_ROUNDS]++;
        C->stats[ST_AVQ] += qn + S.ring.hn;
      }
      QueueOut o = out_for(cur ^ 1);
      const int* qc = P.q[cur];
      HugeRec* hqc = P.hq[cur];
      const int2* hcc = P.hc[cur];
      unsigned long long work = 0;
      int total = qn + hc;
      for (int tk = gwarp; tk < total; tk += nwarps) {
        int u, lo, hi, hidx = -1;
        Seg sg;
        if (tk < qn) {
          u = ld_cg(qc + tk);
          sg = ops.seg(u); lo = 0; hi = sg.deg();
        } else {
          int2 c = ld_cg(hcc + (tk - qn));
          hidx = c.x;
          u = ld_cg(&hqc[hidx].u);
          sg = ops.seg(u);
          lo = c.y * kChunk; hi = min(sg.deg(), lo + kChunk);
        }
        st_arcs += hi - lo;
        // second-level parallelism: lanes scan the residual arcs, keep (h, slot) minimum
        unsigned long long best = ~0ull;
        int bcf = 0, bcol = 0;
#pragma unroll 2
        for (int i = lo + lane; i < hi; i += 32) {
          int col, cf, slot;
          ops.out_arc(sg, i, col, cf, slot);
          if (cf > 0) {
            unsigned hv = (unsigned)ld_cg(P.h + col);
            unsigned long long cand = ((unsigned long long)hv << 32) | (unsigned)slot;
            if (cand < best) { best = cand; bcf = cf; bcol = col; }
          }
        }
        unsigned hmin = __reduce_min_sync(FULL, (unsigned)(best >> 32));
        unsigned smin = __reduce_min_sync(FULL, (unsigned)(best >> 32) == hmin ? (unsigned)best : kInf);
        unsigned long long wbest = ((unsigned long long)hmin << 32) | smin;
        unsigned owner = __ballot_sync(FULL, best == wbest && best != ~0ull);
        int src_lane = owner ? __ffs(owner) - 1 : 0;
        int cfv = __shfl_sync(FULL, bcf, src_lane);
        int colv = __shfl_sync(FULL, bcol, src_lane);
        bool finalize = true;
        if (hidx >= 0) {
          // fold this chunk's minimum into the vertex record; the last chunk finalizes
          int last = 0;
          if (lane == 0) {
            if (wbest != ~0ull) atomicMin(&hqc[hidx].best, wbest);
            __threadfence();
            int nch = ld_cg(&hqc[hidx].nchunks);
            last = (atomicAdd(&hqc[hidx].done, 1) == nch - 1);
            if (last) {
              __threadfence();
              wbest = ld_cg(&hqc[hidx].best);
              if (wbest != ~0ull) ops.col_cf_of_slot((int)(wbest & 0xffffffffu), colv, cfv);
            }
          }
          finalize = __shfl_sync(FULL, last, 0);
          wbest = __shfl_sync(FULL, wbest, 0);
          colv = __shfl_sync(FULL, colv, 0);
          cfv = __shfl_sync(FULL, cfv, 0);
          hmin = (unsigned)(wbest >> 32);
        }
        if (!finalize) continue;
        // delegated lane 0: push or relabel
        int app_u = -1, app_v = -1, dgu = 0, dgv = 0;
        if (lane == 0) {
          int hu = ld_cg(P.h + u);
          long long eu = ld_cg(P.e + u);
          if (hmin != kInf && (int)hmin < hu && cfv > 0) {
            // push: d = min(e(u), c_f(u,v')) (Alg. 1 line 15), four atomics (lines 16-19)
            int d = (int)(eu < (long long)cfv ? eu : (long long)cfv);
            int slot = (int)(wbest & 0xffffffffu);
            ops.push(slot, d);
            long long old_u = (long long)atomicAdd((unsigned long long*)(P.e + u), (unsigned long long)(-(long long)d));
            long long old_v = (long long)atomicAdd((unsigned long long*)(P.e + colv), (unsigned long long)d);
            if (old_u - d > 0) { app_u = u; dgu = sg.deg(); }
            if (old_v == 0 && __ldg(P.term + colv) == 0) { app_v = colv; dgv = ops.degree(colv); }
            ++st_push;
          } else {
            // relabel: h(u) <- h' + 1 (Alg. 1 line 21); >= |V| deactivates
            int nh = (hmin == kInf || (int)hmin >= N - 1) ? N : (int)hmin + 1;
            st_cg(P.h + u, nh);
            if (nh < N) { app_u = u; dgu = sg.deg(); }
            work += (unsigned long long)sg.deg() + 1;
            ++st_relabel;
          }
          if (app_u >= 0 && dgu > kChunk) { huge_append(app_u, dgu, o); app_u = -1; }
          if (app_v >= 0 && dgv > kChunk) { huge_append(app_v, dgv, o); app_v = -1; }
        }
        warp_append(S, cnt, lane == 0 && app_u >= 0, app_u, o);
        warp_append(S, cnt, lane == 0 && app_v >= 0, app_v, o);
      }
      block_flush_all<Ops>(S, cnt, o);
      unsigned long long t = block_sum_u64(S, work);
      if (threadIdx.x == 0 && t) atomicAdd(&ring(ph)->work, t);
      if (!gsync()) return;
      cur ^= 1;
      ++rounds;
      work_since_gr += S.ring.work;
      if (rounds >= P.max_rounds) {
        if (blockIdx.x == 0 && threadIdx.x == 0) { C->status = DS_NOTCONVERGED; }
        break;
      }
      // early break / periodic GR (reading §8(c) #8)
      if (S.ring.qn + S.ring.hn == 0 || work_since_gr >= P.gr_threshold) need_gr = true;
    }
  }

  // ---------------------------------------------------------------- statistics
  {
    long long v[5] = {st_push, st_relabel, st_arcs, st_bfs_arcs, st_cand};
    int idx[5] = {ST_PUSHES, ST_RELABELS, ST_ARCS, ST_BFS_ARCS, ST_CAND};
    for (int i = 0; i < 5; ++i) {
      unsigned long long t = block_sum_u64(S, (unsigned long long)v[i]);
      if (threadIdx.x == 0 && t) atomicAdd((unsigned long long*)&C->stats[idx[i]], t);
    }
  }
}

// ------------------------------------------------------------------ host launch
int solve_max_blocks_per_sm(int layout, int threads) {
  int b = 0;
  if (layout == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_solve<BcsrOps>, threads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_solve<RcsrOps>, threads, 0);
  return b;
}

cudaError_t launch_solve(const SolveParams& p, int blocks, int threads, cudaStream_t st) {
  if (p.layout == 0) {
    BcsrOps o{p.off, p.arc, p.mate};
    void* args[] = {(void*)&p, (void*)&o};
    return cudaLaunchCooperativeKernel((void*)k_solve<BcsrOps>, dim3(blocks), dim3(threads), args, 0, st);
  } else {
    RcsrOps o{p.off, p.arc, p.roff, p.rarc, p.bcf, p.Mf};
    void* args[] = {(void*)&p, (void*)&o};
    return cudaLaunchCooperativeKernel((void*)k_solve<RcsrOps>, dim3(blocks), dim3(threads), args, 0, st);
  }
}

}  // namespace wbpr
