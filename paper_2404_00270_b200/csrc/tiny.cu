// tiny.cu — the whole path (A1-A8) in ONE launch of ONE CTA, for tiny single instances
// (C1-sized: n <= kTinyN vertices, 2m <= kTinyS half-arcs).
//
// Such instances are bound by launch and synchronisation latency, not by work: the
// multi-kernel construction plus the persistent solve cost ~25 launches, a host
// synchronisation after validation and a grid barrier per phase.  Here every step runs in
// one CTA with block barriers and the residual graph in shared memory:
//   A1  BCSR: the 2m half-arcs keyed (owner, column, half-arc id) are sorted by one block
//       bitonic sort; runs of equal (owner, column) merge into one slot (parallel edges
//       summed, an antiparallel pair = one arc pair); mate[] pairs the two halves of
//       every input edge (the paper's backward-arc search, becomes one lookup).
//       The layout is written to the workspace in the standard BCSR form (dense segments),
//       so wbpr_residual_view works as after the multi-kernel path.
//   A2  preflow (Alg. 1 Step 0); A5 exact GR (reverse BFS from t, P:108-109,
//       P:178-182) right after it and whenever the active queue empties or the relabel work
//       reaches gr_beta (n + M); unreachable vertices leave Excess_total once;
//   A3/A4 rounds: active-vertex compaction, one warp per active vertex, lowest-label scan,
//       push (push_mode 1: every admissible arc gets a share) or relabel
//       (Alg. 2, readings §8(c) #1-#3);
//   A8  flow = e(t), bitmap [h >= n], certificate cut capacity over the input edges.
// Same readings and results (F, cut capacity, canonical S*) as the multi-kernel path;
// the trajectory differs (one CTA), which no result depends on (§8(c) N6).
#include <climits>

#include "internal.h"
#include "kernels.h"

namespace wbpr {

constexpr int kTinyThreads = 1024;
constexpr int kTinyWarps = kTinyThreads / 32;
constexpr int kTinyIt = kTinyS / kTinyThreads;   // sort keys per thread
static_assert(kTinyIt == 16 && (kTinyS & (kTinyS - 1)) == 0, "register-blocked bitonic sort layout");
constexpr int kTinyThr = 64;   // vertices up to this many slots are handled by one thread
constexpr int kTinyWarpMode = 4 * kTinyWarps;   // ... unless the queue is this small (warps then)
// padded key index: one spare element per 16, so the blocked sort layout (16 consecutive keys
// per thread) does not put all lanes of a warp on the same shared-memory bank
__device__ __forceinline__ int kx(int i) { return i + (i >> 4); }

struct TinySmem {
  union {
    unsigned long long keys[kTinyS + kTinyS / 16];   // build: sorted half-arc keys (padded, kx())
    struct {
      int cf[kTinyS];                         // solve: residual capacity per slot
      uint16_t col[kTinyS];                   // column per slot
      uint16_t mate[kTinyS];                  // reverse slot
    } r;
  };
  union {
    uint16_t slotof[kTinyS];                  // build: slot of every half-arc id
    struct {
      long long e[kTinyN];                    // solve: excess
      uint16_t q[2][kTinyN];                  // solve: active queue / BFS frontier
      uint8_t deact[kTinyN];                  // solve: excess already dropped from Excess_total
    } s;
  };
  int segb[kTinyN + 1];                       // segment of v = [segb[v], segb[v + 1])
  int h[kTinyN];                              // labels
  int scan[kTinyWarps];
  long long red[kTinyWarps];
  int qn[2];
  unsigned work;
  long long excess_total;
  int flag;
};

// block-wide exclusive scan of one int per thread; *total = the sum
__device__ __forceinline__ int tiny_scan(int v, TinySmem& S, int* total) {
  const int lane = lane_id(), w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(FULL, x, o); if (lane >= o) x += y; }
  if (lane == 31) S.scan[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = S.scan[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(FULL, t, o); if (lane >= o) t += y; }
    S.scan[lane] = t;
  }
  __syncthreads();
  const int before = w ? S.scan[w - 1] : 0;
  *total = S.scan[kTinyWarps - 1];
  __syncthreads();
  return before + x - v;
}

// Sorts keys[b, b + c) (c <= 32 R) with one warp: R keys per lane (blocked), bitonic with
// ~0 padding in registers; partners within a lane unrolled, across lanes by shuffles.
template <int R>
__device__ __forceinline__ void tiny_warp_sort(TinySmem& S, int b, int c, int lane) {
  unsigned long long x[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { const int i = lane * R + r; x[r] = i < c ? S.keys[kx(b + i)] : ~0ull; }
  int P = 32 * R;
  while (P / 2 >= c && P > 2) P >>= 1;   // (the smallest power of two >= c, at least 2)
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < R) {
#pragma unroll
        for (int J = R / 2; J > 0; J >>= 1) {
          if (J > j) continue;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int pr = r ^ J;
            if (pr > r) {
              const bool up = ((lane * R + r) & k) == 0;
              const unsigned long long a0 = x[r], a1 = x[pr];
              if ((a0 > a1) == up) { x[r] = a1; x[pr] = a0; }
            }
          }
        }
        break;
      }
      const int tj = j / R;
      const bool lower = (lane & tj) == 0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const unsigned long long o = __shfl_xor_sync(FULL, x[r], tj);
        const bool up = ((lane * R + r) & k) == 0;
        const bool keep_min = lower == up;
        x[r] = keep_min ? (x[r] < o ? x[r] : o) : (x[r] > o ? x[r] : o);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) { const int i = lane * R + r; if (i < c) S.keys[kx(b + i)] = x[r]; }
}

__device__ __forceinline__ long long tiny_sum(long long v, TinySmem& S) {
  v = warp_sum(v);
  if (lane_id() == 0) S.red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = 0;
  for (int i = 0; i < kTinyWarps; ++i) t += S.red[i];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kTinyThreads, 1) k_tiny(TinyArgs A) {
  extern __shared__ __align__(16) unsigned char traw[];
  TinySmem& S = *reinterpret_cast<TinySmem*>(traw);
  const int tid = threadIdx.x, lane = lane_id(), w = tid >> 5;
  const int n = A.n, m = A.m, N = n, s = A.s, t = A.t;
  Ctrl* C = A.ctrl;
  const unsigned long long t0 = globaltimer();
  const unsigned long long deadline = t0 + A.deadline_ns_rel;
  // ---------------------------------------------------------------- A1: validate
  {   // the control block (the multi-kernel path's k_init_ctrl)
    int* cp = reinterpret_cast<int*>(C);
    for (int i = tid; i < (int)(sizeof(Ctrl) / sizeof(int)); i += kTinyThreads) cp[i] = 0;
  }
  if (tid == 0) { S.flag = 0; S.work = 0; S.excess_total = 0; }
  __syncthreads();
  if (tid == 0) C->bad_edge = LLONG_MAX;
  // row offsets into shared memory (n + 1 entries: segb holds them during the build)
  for (int u = tid; u <= n; u += kTinyThreads) {
    const long long a = A.ro[u];
    const bool bad = a < 0 || a > m || (u == 0 && a != 0) || (u == n && a != m) || (u > 0 && A.ro[u - 1] > a);
    if (bad) atomicExch(&S.flag, 1);
    S.segb[u] = (int)a;
  }
  __syncthreads();
  if (S.flag) { if (tid == 0) C->bad_rows = 1; return; }
  // half-arc keys: ((owner * 2^11 + column) << 20) | id, id = 2e (out half) / 2e + 1 (in
  // half); self-loop halves are ~0 (they sort last in their owner's bucket and get no slot).
  // Buckets: owner v's out halves (its CSR row) then its in halves, at B0[v] (exclusive
  // prefix of outdeg + indeg); each bucket is then sorted on its own, so the whole key array
  // ends up sorted by (owner, column, id).
  int* B0 = reinterpret_cast<int*>(S.slotof);   // [n + 1] (slotof is written later)
  for (int v = tid; v < n; v += kTinyThreads) S.h[v] = 0;
  __syncthreads();
  int loops = 0;
  for (int e = tid; e < m; e += kTinyThreads) {
    const int v = A.col[e], c = A.cap[e];
    if (v < 0 || v >= n || c < 0) {
      atomicMin((unsigned long long*)&C->bad_edge, (unsigned long long)e);
      S.flag = 2;
      continue;
    }
    atomicAdd(&S.h[v], 1);   // in-degree (self-loops included: their in half sits in v's bucket)
  }
  __syncthreads();
  if (S.flag) return;        // EINVAL: C->bad_edge holds the first offending edge
  {
    const int per = (n + kTinyThreads - 1) / kTinyThreads;   // <= 2
    int loc[2], sum = 0;
    for (int r = 0; r < per; ++r) {
      const int v = tid * per + r;
      loc[r] = v < n ? S.segb[v + 1] - S.segb[v] + S.h[v] : 0;
      sum += loc[r];
    }
    int tot;
    int pre = tiny_scan(sum, S, &tot);
    for (int r = 0; r < per; ++r) {
      const int v = tid * per + r;
      if (v < n) { B0[v] = pre; pre += loc[r]; }
    }
    if (tid == 0) B0[n] = tot;
  }
  for (int v = tid; v < n; v += kTinyThreads) S.h[v] = 0;   // in-half cursors
  __syncthreads();
  for (int e = tid; e < m; e += kTinyThreads) {
    int lo = 0, hi = n;   // owner: largest u with ro[u] <= e
    while (hi - lo > 1) { const int md = (lo + hi) >> 1; if (S.segb[md] <= e) lo = md; else hi = md; }
    const int u = lo, v = A.col[e];
    const bool loop = v == u;
    loops += loop;
    S.keys[kx(B0[u] + (e - S.segb[u]))] = loop ? ~0ull : ((unsigned long long)(u * kTinyN + v) << 20) | (unsigned)(2 * e);
    const int q = B0[v] + (S.segb[v + 1] - S.segb[v]) + atomicAdd(&S.h[v], 1);
    S.keys[kx(q)] = loop ? ~0ull : ((unsigned long long)(v * kTinyN + u) << 20) | (unsigned)(2 * e + 1);
  }
  loops = (int)tiny_sum(loops, S);   // (ends with a barrier)
  if (tid == 0) C->selfloops = loops;
  // ---------------------------------------------------------------- A1: bucket sorts
  // one warp per bucket of <= 128 keys (registers + shuffles); larger buckets (hubs) by the
  // whole block afterwards
  if (tid == 0) S.qn[0] = 0;
  __syncthreads();
  for (int v = w; v < n; v += kTinyWarps) {
    const int b = B0[v], c = B0[v + 1] - b;
    if (c <= 1) continue;
    if (c <= 32) tiny_warp_sort<1>(S, b, c, lane);
    else if (c <= 64) tiny_warp_sort<2>(S, b, c, lane);
    else if (c <= 128) tiny_warp_sort<4>(S, b, c, lane);
    else if (lane == 0) S.s.q[0][atomicAdd(&S.qn[0], 1)] = (uint16_t)v;   // (q aliases nothing in use)
  }
  __syncthreads();
  for (int h_ = 0; h_ < S.qn[0]; ++h_) {
    const int v = S.s.q[0][h_];
    const int b = B0[v], c = B0[v + 1] - b;
    int P = 1;
    while (P < c) P <<= 1;
    // bitonic sort with every merge ascending ("flip" first step): the virtual +inf keys at
    // indices >= c never move, so the bucket sorts in place without padding
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < P / 2; i += kTinyThreads) {
          const int lo = 2 * i - (i & (j - 1));
          const int hi = j == (k >> 1) ? (lo | (k - 1)) - (lo & (k - 1)) : lo + j;   // flip / half-cleaner
          if (hi < c) {
            const unsigned long long x0 = S.keys[kx(b + lo)], x1 = S.keys[kx(b + hi)];
            if (x0 > x1) { S.keys[kx(b + lo)] = x1; S.keys[kx(b + hi)] = x0; }
          }
        }
        __syncthreads();
      }
  }
  // ---------------------------------------------------------------- A1: merge runs into slots
  constexpr int IT = kTinyS / kTinyThreads;
  int hf[IT], cnt = 0;
  const int valid_end = 2 * m;
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const int i = tid * IT + r;
    int hd = 0;
    if (i < valid_end) {
      const unsigned long long k = S.keys[kx(i)];
      hd = k != ~0ull && (i == 0 || (S.keys[kx(i - 1)] >> 20) != (k >> 20));
    }
    hf[r] = hd;
    cnt += hd;
  }
  int M;
  int run = tiny_scan(cnt, S, &M);   // heads before this thread's first element
  // per-owner slot counts -> dense segments (segb reused: row offsets are no longer needed)
  for (int u = tid; u <= n; u += kTinyThreads) S.segb[u] = 0;
  __syncthreads();
  int overflow = 0;
  int capr[IT];   // capacities of this thread's own half-arcs, loaded up front (independent loads)
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const int i = tid * IT + r;
    const unsigned long long k = i < valid_end ? S.keys[kx(i)] : ~0ull;
    capr[r] = k != ~0ull ? __ldg(A.cap + ((int)(k & 0xfffffu) >> 1)) : 0;
  }
#pragma unroll
  for (int r = 0; r < IT; ++r) {
    const int i = tid * IT + r;
    run += hf[r];
    if (i >= valid_end) continue;
    const unsigned long long k = S.keys[kx(i)];
    if (k == ~0ull) continue;
    const int slot = run - 1;
    S.slotof[(int)(k & 0xfffffu)] = (uint16_t)slot;
    if (hf[r]) {
      const int oc = (int)(k >> 20), u = oc / kTinyN, v = oc % kTinyN;
      atomicAdd(&S.segb[u + 1], 1);
      long long fw = 0, bw = 0;   // c(u -> v) (out halves), c(v -> u) (in halves)
      if (k & 1) bw += capr[r]; else fw += capr[r];
      // the rest of the run (parallel / antiparallel halves: rare)
      for (int q = i + 1; q < valid_end && (S.keys[kx(q)] >> 20) == (unsigned long long)oc; ++q) {
        const int id = (int)(S.keys[kx(q)] & 0xfffffu);
        const long long c = __ldg(A.cap + (id >> 1));
        if (id & 1) bw += c; else fw += c;
      }
      // a pair's two residual capacities always sum to fw + bw (a push moves d between them)
      if (fw > INT_MAX || bw > INT_MAX || fw + bw > INT_MAX) overflow = 1;
      A.arc[slot] = make_int2(v, (int)(fw > INT_MAX ? INT_MAX : fw));
      A.cap0[slot] = (int)(fw > INT_MAX ? INT_MAX : fw);
    }
  }
  if (overflow) atomicExch(&C->overflow, 1);
  __syncthreads();
  {   // exclusive scan of the per-owner counts (segb[u + 1] held u's count)
    const int per = (n + 1 + kTinyThreads - 1) / kTinyThreads;   // <= 3
    int loc[3], sum = 0;
    for (int r = 0; r < per; ++r) {
      const int u = tid * per + r;
      loc[r] = u <= n ? S.segb[u] : 0;
      sum += loc[r];
    }
    int tot;
    int pre = tiny_scan(sum, S, &tot);
    for (int r = 0; r < per; ++r) {
      const int u = tid * per + r;
      pre += loc[r];
      if (u <= n) S.segb[u] = pre;
    }
  }
  __syncthreads();
  for (int u = tid; u < n; u += kTinyThreads) A.seg[u] = make_int2(S.segb[u], S.segb[u + 1]);
  // mate: the two halves of every input edge, found through the sorted keys (self-loop halves
  // have no slot; parallel edges write the same pair)
  for (int i = tid; i < valid_end; i += kTinyThreads) {
    const unsigned long long k = S.keys[kx(i)];
    if (k == ~0ull || (k & 1u)) continue;           // out halves only
    const int id = (int)(k & 0xfffffu);
    const int p = S.slotof[id], q = S.slotof[id + 1];
    A.mate[p] = q;
    A.mate[q] = p;
  }
  if (tid == 0) C->M = M;
  __syncthreads();
  if (ld_cg(&C->overflow)) return;
  // ---------------------------------------------------------------- solve state in smem
  for (int p = tid; p < M; p += kTinyThreads) {
    const int2 a = ld_cg(A.arc + p);
    S.r.col[p] = (uint16_t)a.x;
    S.r.cf[p] = a.y;
    S.r.mate[p] = (uint16_t)ld_cg(A.mate + p);
  }
  for (int v = tid; v < n; v += kTinyThreads) {
    S.h[v] = v == s ? N + 1 : 0;
    S.s.e[v] = 0;
    S.s.deact[v] = 0;
  }
  __syncthreads();
  const unsigned long long t_build = globaltimer();
  // ---------------------------------------------------------------- A2: preflow
  {
    long long d_sum = 0;
    for (int p = S.segb[s] + tid; p < S.segb[s + 1]; p += kTinyThreads) {
      const int d = S.r.cf[p];
      if (d <= 0) continue;
      S.r.cf[p] = 0;
      atomicAdd(&S.r.cf[S.r.mate[p]], d);
      atomicAdd((unsigned long long*)&S.s.e[S.r.col[p]], (unsigned long long)d);
      d_sum += d;
    }
    d_sum = tiny_sum(d_sum, S);
    if (tid == 0) S.excess_total = d_sum;
  }
  __syncthreads();
  const unsigned gr_threshold = (unsigned)((double)A.gr_beta * (double)(n + M)) + 1u;
  long long rounds = 0, grs = 0, levels = 0;
  long long tot_push = 0, tot_rel = 0, tot_arcs = 0, tot_bfs = 0;
  unsigned long long t_bfs = 0, t_epi = 0, t_rnd = 0, tq = 0;   // (thread 0: phase times)
  int status = DS_OK;
  while (true) {
    // ------------------------------------------------------------ A5: exact global relabel
    if (tid == 0) tq = globaltimer();
    for (int v = tid; v < n; v += kTinyThreads) S.h[v] = v == t ? 0 : (v == s ? N + 1 : N);
    if (tid == 0) { S.s.q[0][0] = (uint16_t)t; S.qn[0] = 1; S.qn[1] = 0; S.work = 0; }
    __syncthreads();
    int cur = 0, level = 0;
    while (S.qn[cur] > 0) {
      const int qa = S.qn[cur];
      long long arcs = 0;
      // frontier vertices with <= kTinyThr slots: one THREAD each while the frontier is large;
      // a small frontier (latency-bound) and large vertices: one warp each
      const int thr_max = qa > kTinyWarpMode ? kTinyThr : 0;
      for (int j = tid; j < qa; j += kTinyThreads) {
        const int x = S.s.q[cur][j];
        const int b = S.segb[x], e_ = S.segb[x + 1];
        if (e_ - b > thr_max) continue;
        arcs += e_ - b;
        for (int p = b; p < e_; ++p) {
          const int u = S.r.col[p];
          // residual in-arc u -> x: c_f(u, x) = cf[mate[p]]
          // (labels are written with atomics: concurrent plain reads of them are the
          // algorithm's benign races, never a torn or lost value)
          if (S.h[u] == N && S.r.cf[S.r.mate[p]] > 0) atomicCAS(&S.h[u], N, level + 1);
        }
      }
      for (int j = w; j < qa; j += kTinyWarps) {
        const int x = S.s.q[cur][j];
        const int b = S.segb[x], e_ = S.segb[x + 1];
        if (e_ - b <= thr_max) continue;
        for (int p = b + lane; p < e_; p += 32) {
          const int u = S.r.col[p];
          ++arcs;
          if (S.h[u] == N && S.r.cf[S.r.mate[p]] > 0) atomicCAS(&S.h[u], N, level + 1);
        }
      }
      tot_bfs += arcs;   // (per-thread; summed once at the end)
      __syncwarp();
      __syncthreads();
      // next frontier = the vertices labelled level + 1 (a compaction over n with one
      // shared atomic per warp, instead of one contended append per discovered vertex)
      if (tid == 0) { S.qn[cur] = 0; ++levels; }
      for (int v0 = 0; v0 < n; v0 += kTinyThreads) {
        const int v = v0 + tid;
        const bool nf = v < n && S.h[v] == level + 1;
        const unsigned bm = __ballot_sync(FULL, nf);
        int base = 0;
        if (lane == 0 && bm) base = atomicAdd(&S.qn[cur ^ 1], __popc(bm));
        base = __shfl_sync(FULL, base, 0);
        if (nf) S.s.q[cur ^ 1][base + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)v;
      }
      cur ^= 1;
      ++level;
      __syncthreads();
    }
    ++grs;
    if (tid == 0) { const unsigned long long x = globaltimer(); t_bfs += x - tq; tq = x; }
    // unreachable vertices holding excess leave Excess_total once (N5); then the
    // active set: termination right after an exact GR (N6)
    {
      long long drop = 0;
      int act = 0;
      for (int v = tid; v < n; v += kTinyThreads) {
        if (v == s || v == t) continue;
        const long long ev = S.s.e[v];
        if (ev <= 0) continue;
        if (S.h[v] >= N) { if (!S.s.deact[v]) { S.s.deact[v] = 1; drop += ev; } }
        else ++act;
      }
      drop = tiny_sum(drop, S);
      act = (int)tiny_sum(act, S);
      if (tid == 0) { S.excess_total -= drop; const unsigned long long x = globaltimer(); t_epi += x - tq; tq = x; }
      if (act == 0) break;
    }
    // ------------------------------------------------------------ A3/A4: rounds
    bool gr_due = false;
    while (!gr_due) {
      if (tid == 0) S.qn[0] = 0;
      __syncthreads();
      for (int v0 = 0; v0 < n; v0 += kTinyThreads) {   // warp-aggregated appends
        const int v = v0 + tid;
        const bool act = v < n && v != s && v != t && S.s.e[v] > 0 && S.h[v] < N;
        const unsigned bm = __ballot_sync(FULL, act);
        int base = 0;
        if (lane == 0 && bm) base = atomicAdd(&S.qn[0], __popc(bm));
        base = __shfl_sync(FULL, base, 0);
        if (act) S.s.q[0][base + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)v;
      }
      __syncwarp();
      __syncthreads();
      const int qa = S.qn[0];
      __syncthreads();      // (everyone has read qa before the GR below rewrites S.qn)
      if (qa == 0) break;   // queue empty: exact GR decides termination
      long long pushes = 0, relabels = 0, arcs = 0;
      // active vertices with <= kTinyThr slots: one THREAD each (the same push / relabel
      // semantics as the warp form below: lowest residual label, then shares of e(u) over the
      // admissible arcs in slot order, or a relabel)
      const int thr_max = qa > kTinyWarpMode ? kTinyThr : 0;   // (small queue: warps, see BFS)
      for (int j = tid; j < qa; j += kTinyThreads) {
        const int u = S.s.q[0][j];
        const int b = S.segb[u], e_ = S.segb[u + 1];
        if (e_ - b > thr_max) continue;
        const int hu = S.h[u];
        unsigned long long best = ~0ull;
        bool adm = false;
        for (int p = b; p < e_; ++p) {
          if (S.r.cf[p] <= 0) continue;
          const int hv = S.h[S.r.col[p]];
          best = min(best, ((unsigned long long)(unsigned)hv << 32) | (unsigned)p);
          adm |= hv < hu;
        }
        arcs += e_ - b;
        if (adm) {
          long long left = S.s.e[u], sent = 0;
          for (int p = b; p < e_ && left > 0; ++p) {
            const int c = S.r.cf[p];
            if (c <= 0) continue;
            const int v = S.r.col[p];
            if (S.h[v] >= hu) continue;
            const int d = (int)(left < c ? left : c);
            atomicSub(&S.r.cf[p], d);
            atomicAdd(&S.r.cf[S.r.mate[p]], d);
            atomicAdd((unsigned long long*)&S.s.e[v], (unsigned long long)d);
            left -= d; sent += d; ++pushes;
          }
          if (sent) atomicAdd((unsigned long long*)&S.s.e[u], (unsigned long long)(-sent));
        } else {
          atomicExch(&S.h[u], best == ~0ull ? N : min(N, (int)(best >> 32) + 1));
          ++relabels;
          atomicAdd(&S.work, (unsigned)(e_ - b));
        }
      }
      for (int j = w; j < qa; j += kTinyWarps) {
        const int u = S.s.q[0][j];
        const int b = S.segb[u], e_ = S.segb[u + 1];
        if (e_ - b <= thr_max) continue;
        const int hu = S.h[u];
        // pass 1: lowest label over residual arcs (ties: smallest slot), any admissible arc
        unsigned long long best = ~0ull;
        bool adm = false;
        for (int p = b + lane; p < e_; p += 32) {
          const int c = S.r.cf[p];
          if (c <= 0) continue;
          const int hv = S.h[S.r.col[p]];
          best = min(best, ((unsigned long long)(unsigned)hv << 32) | (unsigned)p);
          adm |= hv < hu;
        }
        if (lane == 0) arcs += e_ - b;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(FULL, best, o));
        adm = __any_sync(FULL, adm);
        if (adm) {
          // push: e(u) shared over the admissible arcs in slot order (push_mode 1)
          long long left = __shfl_sync(FULL, S.s.e[u], 0);   // a lower bound (only u decreases it, N1)
          long long sent = 0;
          for (int p0 = b; p0 < e_ && left > 0; p0 += 32) {
            const int p = p0 + lane;
            int c = 0;
            if (p < e_) { c = S.r.cf[p]; if (c > 0 && S.h[S.r.col[p]] >= hu) c = 0; }
            // inclusive prefix of the admissible capacities in slot order
            long long x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) { const long long y = __shfl_up_sync(FULL, x, o); if (lane >= o) x += y; }
            const long long before = x - c;
            long long d = left - before;
            d = d < 0 ? 0 : (d > c ? c : d);
            if (d > 0) {
              const int v = S.r.col[p];
              atomicSub(&S.r.cf[p], (int)d);
              atomicAdd(&S.r.cf[S.r.mate[p]], (int)d);
              atomicAdd((unsigned long long*)&S.s.e[v], (unsigned long long)d);
              ++pushes;
              sent += d;
            }
            left -= __shfl_sync(FULL, x, 31);
          }
          sent = warp_sum(sent);
          if (lane == 0 && sent) atomicAdd((unsigned long long*)&S.s.e[u], (unsigned long long)(-sent));
        } else if (lane == 0) {
          // relabel to the lowest residual neighbour + 1 (no residual arc: unreachable, n)
          atomicExch(&S.h[u], best == ~0ull ? N : min(N, (int)(best >> 32) + 1));
          ++relabels;
          atomicAdd(&S.work, (unsigned)(e_ - b));
        }
      }
      tot_push += pushes; tot_rel += relabels; tot_arcs += arcs;   // (per-thread; summed at the end)
      __syncwarp();
      ++rounds;
      if (tid == 0) {
        const unsigned long long x = globaltimer();
        t_rnd += x - tq; tq = x;
        S.flag = rounds >= A.max_rounds ? DS_NOTCONVERGED : (x > deadline ? DS_TIMEOUT : DS_OK);
      }
      __syncthreads();
      status = S.flag;
      gr_due = S.work >= gr_threshold;
      __syncthreads();   // (S.flag / S.work are rewritten next round)
      if (status != DS_OK) break;
    }
    if (status != DS_OK) break;
  }
  // ---------------------------------------------------------------- A8: results
  for (int p = tid; p < M; p += kTinyThreads) A.arc[p].y = S.r.cf[p];
  for (int v = tid; v < n; v += kTinyThreads) { A.h[v] = S.h[v]; A.e[v] = S.s.e[v]; }
  for (int base = w * 32; base < ((n + 31) & ~31); base += kTinyThreads) {
    const int v = base + lane;
    const unsigned bits = __ballot_sync(FULL, v < n && S.h[v] >= N);
    if (lane == 0 && A.bitmap) A.bitmap[base >> 5] = bits;
  }
  long long cut = 0;
  for (int u = w; u < n; u += kTinyWarps) {
    if (S.h[u] < N) continue;
    for (long long i = A.ro[u] + lane; i < A.ro[u + 1]; i += 32) {
      const int v = A.col[i];
      if (v != u && S.h[v] < N) cut += A.cap[i];
    }
  }
  cut = tiny_sum(cut, S);
  tot_push = tiny_sum(tot_push, S);
  tot_rel = tiny_sum(tot_rel, S);
  tot_arcs = tiny_sum(tot_arcs, S);
  tot_bfs = tiny_sum(tot_bfs, S);
  if (tid == 0) {
    A.flow[0] = S.s.e[t];
    A.cut[0] = cut;
    C->excess_total = S.excess_total;
    C->status = status;
    if (status == DS_TIMEOUT) C->abort = 1;
    C->stats[ST_ROUNDS] = rounds;
    C->stats[ST_GRS] = grs;
    C->stats[ST_BFS_LEVELS] = levels;
    C->stats[ST_PUSHES] = tot_push;
    C->stats[ST_RELABELS] = tot_rel;
    C->stats[ST_ARCS] = tot_arcs;
    C->stats[ST_BFS_ARCS] = tot_bfs;
    C->phase_ns[PK_NONE] = (long long)(t_build - t0);   // build time (host reports build_ms)
    C->phase_ns[PK_ROUND] = (long long)t_rnd; C->phase_cnt[PK_ROUND] = rounds;
    C->phase_ns[PK_BFS] = (long long)t_bfs; C->phase_cnt[PK_BFS] = levels;
    C->phase_ns[PK_COMPACT] = (long long)t_epi; C->phase_cnt[PK_COMPACT] = grs;
  }
}

bool tiny_fits(int64_t n, int64_t m) { return n <= kTinyN && 2 * m <= kTinyS && n >= 2; }

cudaError_t launch_tiny(const TinyArgs& a, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(k_tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TinySmem));
  if (e != cudaSuccess) return e;
  k_tiny<<<1, kTinyThreads, sizeof(TinySmem), st>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace wbpr
