// merge.cu — BCSR construction (A1) by merging two sorted lists per vertex.
//
// seg(x) of the BCSR (§3.2) is the column-sorted union of x's
// out-arcs (its input CSR row, cap c) and its in-arcs (the transposed edges,
// residual capacity 0).  Instead of sorting the concatenation:
//   * out-rows are taken in input order and sorted only where the input row is not
//     already column-sorted (detected per row while the 64-bit keys are written);
//   * in-lists carry the 32-bit INDEX e of the input edge (its capacity is always 0),
//     scattered by a histogram + atomic cursor and sorted with the 32-bit segmented sort
//     (sorting by e orders an in-list by source, rows being stored in vertex order);
//     k_in_resolve then writes the source u = src[e] beside e;
//   * one merge pass writes {col, cf = sum of caps} and cap0 (parallel edges and
//     antiparallel pairs collapse) into a GAPPED layout: seg(x) starts at
//     outdeg-prefix(x) + indeg-prefix(x), an upper bound of the distinct columns before
//     x, so no counting pass or offset scan is needed; seg[x] = {begin, end};
//   * the merge records the slot of every out-half-arc (outslot[e]) and of every in-list
//     entry (inslot[t]); mate[] is then one lookup per input edge (build.cu k_mate) -
//     the paper's backward-arc binary search is never run.
// Merge classes: <= kMergeThreadMax (12) elements: one thread, sequential two-pointer merge;
// <= 8192: one warp, merge path advanced 32 outputs at a time with the 32-element
// windows of both lists held in registers (co-rank by shuffles); larger: split into
// 4096-output warp tasks whose starts come from a global co-rank search (their counts
// come from a counting pass over those hub vertices only).
#include <climits>

#include "internal.h"
#include "kernels.h"

namespace wbpr {

constexpr uint64_t kSentKey = ~0ull;
constexpr uint32_t kInf = 0xffffffffu;
#ifndef WBPR_MERGE_TMAX
#define WBPR_MERGE_TMAX 12   // measured (profiles/r2/ab_merge_tmax.txt): 32 -> 16 -> 12: C5 build 20.64 -> 20.49 ms, C4 4.23 -> 4.04 ms
#endif
constexpr int kMergeThreadMax = WBPR_MERGE_TMAX;
constexpr int kMergeWarpMax = 8192;
constexpr int kMergeChunk = 4096;

__device__ __forceinline__ uint32_t kcol(uint64_t k) { return (uint32_t)(k >> 32); }
__device__ __forceinline__ long long kcap(uint64_t k) { return (long long)(uint32_t)(k & 0xffffffffu); }

__device__ __forceinline__ int row_of64(const int64_t* __restrict__ ro, int64_t n, int64_t i) {
  int64_t lo = 0, hi = n;
  while (hi - lo > 1) { int64_t mid = (lo + hi) >> 1; if (__ldg(ro + mid) <= i) lo = mid; else hi = mid; }
  return (int)lo;
}

// in-list scatter: the out-half-arc at sorted row position e (edge u -> v, u != v)
// lands in v's in-list as the 32-bit edge index e (sorting the in-list by e orders it by
// the source u, since rows are stored in vertex order); k_in_resolve then turns e into
// u and keeps e beside it, so the merge can pair both half-arcs of the edge (mate[]).
// One warp per kScatChunk consecutive edges as rows of 32 (coalesced loads); the
// kScatRows cursor atomics of a lane are issued back to back; the cursors start at the
// in-list offsets, so an atomic returns the absolute position.
constexpr int kScatRows = 8;
constexpr int kScatChunk = 32 * kScatRows * 8;
__global__ void __launch_bounds__(256) k_inscatter(const uint64_t* __restrict__ outk, int64_t m, int* cursor,
                                                   uint32_t* inkeys) {
  const int lane = lane_id();
  const int64_t E0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * kScatChunk;
  if (E0 >= m) return;
  const int64_t E1 = E0 + kScatChunk < m ? E0 + kScatChunk : m;
  for (int64_t eb = E0; eb < E1; eb += 32 * kScatRows) {
    uint64_t k[kScatRows];
#pragma unroll
    for (int r = 0; r < kScatRows; ++r) {
      const int64_t i = eb + r * 32 + lane;
      k[r] = i < E1 ? __ldg(outk + i) : kSentKey;
    }
    int q[kScatRows];
#pragma unroll
    for (int r = 0; r < kScatRows; ++r) q[r] = k[r] != kSentKey ? atomicAdd(cursor + kcol(k[r]), 1) : -1;
#pragma unroll
    for (int r = 0; r < kScatRows; ++r)
      if (q[r] >= 0) inkeys[q[r]] = (uint32_t)(eb + r * 32 + lane);
  }
}

// in-list entries: edge index e -> (source u = src[e] in place, e kept in ine[])
__global__ void __launch_bounds__(256) k_in_resolve(uint32_t* ink, int* ine, const int* __restrict__ src,
                                                    const int* __restrict__ rsoff, int n) {
  const int total = __ldg(rsoff + n);
  const int base = blockIdx.x * blockDim.x * 4 + threadIdx.x;
  uint32_t e[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) { const int q = base + r * blockDim.x; e[r] = q < total ? ink[q] : 0u; }
  int u[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) u[r] = base + r * (int)blockDim.x < total ? __ldg(src + e[r]) : 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int q = base + r * blockDim.x;
    if (q < total) { ine[q] = (int)e[r]; ink[q] = (uint32_t)u[r]; }
  }
}

struct MergeArgs {
  const int* ooff;          // out-list offsets (int32 copy of row_offsets), n+1
  const uint64_t* outk;     // sorted out keys (col << 32 | cap), self-loops = kSentKey (last)
  const int* ioff;          // in-list offsets, n+1
  const uint32_t* ink;      // sorted in-list source ids
  int n;
  int* mdeg;                // chunk class: distinct columns per vertex (pass 0)
  int2* seg;                // pass 1 output: {begin, end} of every vertex segment
  int2* arc;                // pass 1 output
  int* cap0;
  int* outslot;             // pass 1 output: slot of every out-half-arc (by sorted row position)
  int* inslot;              // pass 1 output: slot of every in-list entry (by in-list position)
  int* wlist;               // vertices for the warp class
  int2* tasks;              // (vertex, chunk) tasks of the chunked class (> kMergeWarpMax)
  int* chunk_heads;         // distinct columns found by each chunk task
  Ctrl* ctrl;
};

__device__ __forceinline__ void emit(const MergeArgs& a, int slot, uint32_t c, long long sum) {
  if (sum > INT_MAX) { atomicExch(&a.ctrl->overflow, 1); sum = INT_MAX; }
  // a pair u->v / v->u shares one arc pair whose cf values always sum to cap0[p] + cap0[mate]
  // (a push moves d from one to the other): flag big capacities so k_mate checks that sum
  if (sum > (INT_MAX >> 1)) a.ctrl->bigcap = 1;
  a.arc[slot] = make_int2((int)c, (int)sum);
  a.cap0[slot] = (int)sum;
}

// PASS 0: classification only (warp-class list, chunk tasks); PASS 1: merge of the
// thread class (<= kMergeThreadMax elements, one thread per vertex)
template <int PASS>
__global__ void __launch_bounds__(256) k_merge_thread(MergeArgs a) {
  const int lane = lane_id();
  long long msum = 0;   // slots written by this thread (ctrl->M)
  for (int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < a.n; base += gridDim.x * blockDim.x) {
    int x = base + lane;
    int ob = 0, lo = 0, ib = 0, li = 0;
    if (x < a.n) {
      ob = __ldg(a.ooff + x); lo = __ldg(a.ooff + x + 1) - ob;
      ib = __ldg(a.ioff + x); li = __ldg(a.ioff + x + 1) - ib;
    }
    bool big = x < a.n && lo + li > kMergeThreadMax;
    if (PASS == 0) {
      bool wl = big && lo + li <= kMergeWarpMax, cl = big && !wl;
      unsigned bw = __ballot_sync(FULL, wl);
      int pw = 0;
      if (lane == 0 && bw) pw = atomicAdd(&a.ctrl->mlist_w, __popc(bw));
      pw = __shfl_sync(FULL, pw, 0);
      unsigned lt = (1u << lane) - 1u;
      if (wl) a.wlist[pw + __popc(bw & lt)] = x;
      if (cl) {   // split into kMergeChunk-output tasks (rare: hubs)
        int nch = (lo + li + kMergeChunk - 1) / kMergeChunk;
        int t0 = atomicAdd(&a.ctrl->mlist_c, nch);
        for (int c = 0; c < nch; ++c) a.tasks[t0 + c] = make_int2(x, c);
        a.mdeg[x] = 0;
      }
    }
    if (PASS == 0 || x >= a.n || big) continue;
    // gapped layout: seg(x) starts at ooff[x] + ioff[x] (the sum of both list lengths
    // before x bounds the distinct columns before x), so no counting pass is needed
    int i = 0, j = 0, r = 0;
    const int slot0 = ob + ib;
    // two-pointer merge; each element is loaded once, one element ahead of its use in each
    // list (a consumed head's successor is already in flight)
    uint64_t ka = lo > 0 ? a.outk[ob] : kSentKey;
    uint64_t ka2 = lo > 1 ? a.outk[ob + 1] : kSentKey;
    uint32_t kb = li > 0 ? a.ink[ib] : kInf;
    uint32_t kb2 = li > 1 ? a.ink[ib + 1] : kInf;
    while (true) {
      uint32_t ca = kcol(ka);
      const uint32_t c = ca < kb ? ca : kb;
      if (c == kInf) break;
      long long sum = 0;
      while (ca == c) {
        sum += kcap(ka);
        if (PASS == 1) a.outslot[ob + i] = slot0 + r;
        ++i;
        ka = ka2;
        ka2 = i + 1 < lo ? a.outk[ob + i + 1] : kSentKey;
        ca = kcol(ka);
      }
      while (kb == c) {
        if (PASS == 1) a.inslot[ib + j] = slot0 + r;
        ++j;
        kb = kb2;
        kb2 = j + 1 < li ? a.ink[ib + j + 1] : kInf;
      }
      if (PASS == 1) emit(a, slot0 + r, c, sum);
      ++r;
    }
    a.seg[x] = make_int2(slot0, slot0 + r);
    // unused slots after the segment (merged duplicates, self-loops) are zeroed: the solver's
    // 16-B vector loads may cover them (values masked, but never uninitialised)
    if (PASS == 1)
      for (int g = slot0 + r; g < slot0 + lo + li; ++g) a.arc[g] = make_int2(0, 0);
    msum += r;
  }
  if (PASS == 1) {
    msum = warp_sum(msum);
    if (lane == 0 && msum) atomicAdd(&a.ctrl->M, (int)msum);
  }
}

// One warp walks output positions [k0, k1) of the merge of Out (lo) and In (li),
// starting at list positions (i0, j0) with the previous output column prev.
// PASS 0: returns the number of distinct-column heads; PASS 1: also writes them at
// slot base + rank.
template <int PASS>
__device__ __forceinline__ int warp_merge_range(const MergeArgs& a, int ob, int lo, int ib, int li, int i0, int j0,
                                                int k0, int k1, uint32_t prev, int slot_base) {
  const int lane = lane_id();
  int heads = 0;
  // register windows: 32 out-keys (column and capacity) and 32 in-list sources; the next
  // window is loaded as soon as this one's consumption is known, before its stores
  uint64_t ak = (k0 < k1 && i0 + lane < lo) ? a.outk[ob + i0 + lane] : kSentKey;
  uint32_t bv = (k0 < k1 && j0 + lane < li) ? a.ink[ib + j0 + lane] : kInf;
  for (int produced = k0; produced < k1; produced += 32) {
    const uint32_t av = kcol(ak);
    int la = lo - i0 < 32 ? lo - i0 : 32;
    int lb = li - j0 < 32 ? li - j0 : 32;
    if (la < 0) la = 0;
    if (lb < 0) lb = 0;
    // co-rank of output k = lane inside the two register windows (A wins ties)
    int k = lane;
    int rlo = k - lb > 0 ? k - lb : 0, rhi = k < la ? k : la;
#pragma unroll
    for (int it = 0; it < 6; ++it) {
      int mid = (rlo + rhi) >> 1;
      int bidx = k - mid - 1;
      uint32_t Am = __shfl_sync(FULL, av, mid & 31);
      uint32_t Bm = __shfl_sync(FULL, bv, (bidx < 0 ? 0 : bidx) & 31);
      if (rlo < rhi) {
        if (Am <= Bm) rlo = mid + 1; else rhi = mid;
      }
    }
    int i = rlo, j = k - rlo;
    uint32_t Ai = __shfl_sync(FULL, av, i & 31);
    uint32_t Bj = __shfl_sync(FULL, bv, j & 31);
    const uint64_t Aki = __shfl_sync(FULL, ak, i & 31);            // A[i] with its capacity
    const uint32_t Ai1 = __shfl_sync(FULL, av, (i + 1) & 31);      // A[i + 1] (parallel edge?)
    bool takeA = j >= lb || (i < la && Ai <= Bj);
    uint32_t c = takeA ? Ai : Bj;
    bool valid = produced + lane < k1 && c != kInf;
    uint32_t pc = __shfl_up_sync(FULL, c, 1);
    if (lane == 0) pc = prev;
    bool head = valid && c != pc;
    unsigned hm = __ballot_sync(FULL, head);
    const int nA = __shfl_sync(FULL, i + (takeA ? 1 : 0), 31);
    const uint32_t last = __shfl_sync(FULL, c, 31);
    const int i0n = i0 + nA, j0n = j0 + 32 - nA;
    uint64_t akn = kSentKey;
    uint32_t bvn = kInf;
    if (produced + 32 < k1) {   // (warp-uniform)
      akn = i0n + lane < lo ? a.outk[ob + i0n + lane] : kSentKey;
      bvn = j0n + lane < li ? a.ink[ib + j0n + lane] : kInf;
    }
    if (PASS == 1 && valid) {
      // slot of this output's run: the last head at or before this lane (a run without a
      // head in this window continues the previous window's last slot)
      const int slot = slot_base + heads + __popc(hm & (((1u << lane) - 1u) | (1u << lane))) - 1;
      if (takeA) a.outslot[ob + i0 + i] = slot;
      else a.inslot[ib + j0 + j] = slot;
    }
    if (PASS == 1 && head) {
      long long sum = 0;
      if (takeA) {
        sum = kcap(Aki);
        // parallel edges: the run continues past A[i] (rare; from global memory)
        if (i + 1 >= la || Ai1 == c)
          for (int q = i0 + i + 1; q < lo; ++q) {
            uint64_t kk = a.outk[ob + q];
            if (kcol(kk) != c) break;
            sum += kcap(kk);
          }
      }
      emit(a, slot_base + heads + __popc(hm & ((1u << lane) - 1u)), c, sum);
    }
    heads += __popc(hm);
    prev = last;
    i0 = i0n;
    j0 = j0n;
    ak = akn;
    bv = bvn;
  }
  return heads;
}

#ifndef WBPR_MERGE_PF
#define WBPR_MERGE_PF 1   // measured: C5 build 21.3 -> 21.0 ms, C3 +0.08 ms, C4 equal
#endif
__global__ void __launch_bounds__(256) k_merge_warp(MergeArgs a) {
  const int cnt = a.ctrl->mlist_w;
  const int lane = lane_id();
  long long msum = 0;   // slots written by this warp (ctrl->M)
  int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
#if WBPR_MERGE_PF
  // software pipeline over the grid-stride loop (a C5 vertex is about one 32-wide window): the
  // vertex id two tasks ahead and the list offsets one task ahead are in flight during a merge
  int x1 = wg < cnt ? a.wlist[wg] : 0;
  int x2 = wg + nw < cnt ? a.wlist[wg + nw] : 0;
  int ob1 = 0, oe1 = 0, ib1 = 0, ie1 = 0;
  if (wg < cnt) { ob1 = __ldg(a.ooff + x1); oe1 = __ldg(a.ooff + x1 + 1); ib1 = __ldg(a.ioff + x1); ie1 = __ldg(a.ioff + x1 + 1); }
  for (int it = wg; it < cnt; it += nw) {
    const int x = x1, ob = ob1, lo = oe1 - ob1, ib = ib1, li = ie1 - ib1;
    x1 = x2;
    x2 = it + 2 * nw < cnt ? a.wlist[it + 2 * nw] : 0;
    if (it + nw < cnt) { ob1 = __ldg(a.ooff + x1); oe1 = __ldg(a.ooff + x1 + 1); ib1 = __ldg(a.ioff + x1); ie1 = __ldg(a.ioff + x1 + 1); }
#else
  for (int it = wg; it < cnt; it += nw) {
    int x = a.wlist[it];
    int ob = __ldg(a.ooff + x), lo = __ldg(a.ooff + x + 1) - ob;
    int ib = __ldg(a.ioff + x), li = __ldg(a.ioff + x + 1) - ib;
#endif
    const int base = ob + ib;   // gapped layout (see k_merge_thread)
    int h = warp_merge_range<1>(a, ob, lo, ib, li, 0, 0, 0, lo + li, kInf, base);
    if (lane == 0) a.seg[x] = make_int2(base, base + h);
    msum += h;
    for (int g = base + h + lane; g < base + lo + li; g += 32) a.arc[g] = make_int2(0, 0);   // unused tail
  }
  // one slot-count atomic per warp, not per vertex (millions of same-address atomics serialise)
  if (lane == 0 && msum) atomicAdd(&a.ctrl->M, (int)msum);
}

// global co-rank on the full lists (Out compared by column)
__device__ __forceinline__ int co_rank_lists(int k, const uint64_t* A, int la, const uint32_t* B, int lb) {
  int lo = k - lb > 0 ? k - lb : 0, hi = k < la ? k : la;
  while (lo < hi) {
    int i = (lo + hi) >> 1;
    if (kcol(A[i]) <= B[k - i - 1]) lo = i + 1; else hi = i;
  }
  return lo;
}

// Chunked class: one warp per (vertex, chunk) task of kMergeChunk outputs; the
// chunk's start in both lists is found by a global co-rank search.
template <int PASS>
__global__ void __launch_bounds__(256) k_merge_chunk(MergeArgs a) {
  const int cnt = a.ctrl->mlist_c;
  const int lane = lane_id();
  int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = wg; t < cnt; t += nw) {
    int2 tk = a.tasks[t];
    int x = tk.x, c = tk.y;
    int ob = __ldg(a.ooff + x), lo = __ldg(a.ooff + x + 1) - ob;
    int ib = __ldg(a.ioff + x), li = __ldg(a.ioff + x + 1) - ib;
    int total = lo + li;
    int k0 = c * kMergeChunk;
    int k1 = k0 + kMergeChunk < total ? k0 + kMergeChunk : total;
    int i0 = co_rank_lists(k0, a.outk + ob, lo, a.ink + ib, li);
    int j0 = k0 - i0;
    uint32_t prev = kInf;
    if (k0 > 0) {
      uint32_t pa = i0 > 0 ? kcol(a.outk[ob + i0 - 1]) : 0u;
      uint32_t pb = j0 > 0 ? a.ink[ib + j0 - 1] : 0u;
      prev = pa > pb ? pa : pb;
    }
    if (PASS == 0) {
      int h = warp_merge_range<0>(a, ob, lo, ib, li, i0, j0, k0, k1, prev, 0);
      if (lane == 0) {
        a.chunk_heads[t] = h;
        atomicAdd(a.mdeg + x, h);
      }
    } else {
      int before = 0;
      for (int q = lane; q < c; q += 32) before += a.chunk_heads[t - c + q];
      before = warp_sum(before);
      const int base = ob + ib;   // gapped layout (see k_merge_thread)
      warp_merge_range<1>(a, ob, lo, ib, li, i0, j0, k0, k1, prev, base + before);
      if (c == 0) {
        const int d = __ldg(a.mdeg + x);
        if (lane == 0) {
          a.seg[x] = make_int2(base, base + d);
          atomicAdd(&a.ctrl->M, d);
        }
        for (int g = base + d + lane; g < base + total; g += 32) a.arc[g] = make_int2(0, 0);   // unused tail
      }
    }
  }
}

static unsigned gridcap(int64_t items, int threads, int num_sms, int per_sm) {
  int64_t b = (items + threads - 1) / threads;
  if (b > (int64_t)num_sms * per_sm) b = (int64_t)num_sms * per_sm;
  return (unsigned)(b < 1 ? 1 : b);
}

// Build BCSR from the validated input (BuildArgs: deg = in-degrees, maxlen = max
// in-degree, maxlen_out = max out-degree).
void build_bcsr_merge(const BuildArgs& a, cudaStream_t st) {
  const int T = 256;
  const int64_t n = a.n, m = a.m;
  // in-list offsets; out-list offsets (int32 copy of the input row offsets)
  cudaMemcpyAsync(a.rsoff, a.deg, sizeof(int) * n, cudaMemcpyDeviceToDevice, st);
  exclusive_scan(a.rsoff, n, a.scan_part, st);
  { k_ro_to_i32_ext(a.ro, n, a.soff, a.num_sms, st); }
  uint64_t* outk = a.tmp;                                     // region B [0, 8m)
  uint32_t* ink = reinterpret_cast<uint32_t*>(a.keys);        // region A [0, 4m)
  uint32_t* itmp = ink + m;                                   // region A [4m, 8m)
  uint64_t* otmp = reinterpret_cast<uint64_t*>(a.arc);        // region C [0, 8m)
  int2* items = a.arc + m;                                    // region C [8m, 12m)
  int2* items_med = a.arc + m + m / 2 + 1;                    // region C [12m, 16m)
  // out-keys, their sortedness flags and the edge owners (src) were written by the
  // validation pass (k_edges); rows not column-sorted are sorted first, so that the in-list
  // entries can name out-half-arcs by their sorted position
  if (a.any_unsorted)   // (validation found every row column-sorted: nothing to sort)
    segmented_sort_filtered(outk, otmp, a.soff, (int)n, a.maxlen_out, a.need, a.ctrl, items, items_med, a.q0,
                            a.num_sms, st);
  cudaMemcpyAsync(a.cursor, a.rsoff, sizeof(int) * n, cudaMemcpyDeviceToDevice, st);
  if (m > 0) {
    const int64_t sthreads = (m + kScatChunk - 1) / kScatChunk * 32;
    { k_inscatter<<<(unsigned)((sthreads + T - 1) / T), T, 0, st>>>(outk, m, a.cursor, ink); note_launch(); }
  }
  segmented_sort32(ink, itmp, a.rsoff, (int)n, a.maxlen, a.ctrl, items, items_med, a.q0, a.num_sms, st);
  if (m > 0) { k_in_resolve<<<(unsigned)((m + 1023) / 1024), T, 0, st>>>(ink, a.ine, a.src, a.rsoff, (int)n); note_launch(); }
  MergeArgs ma;
  ma.ooff = a.soff; ma.outk = outk; ma.ioff = a.rsoff; ma.ink = ink; ma.n = (int)n;
  ma.mdeg = a.deg; ma.seg = a.seg; ma.arc = a.arc; ma.cap0 = a.cap0;
  ma.outslot = a.outslot; ma.inslot = a.inslot;
  ma.wlist = a.q0; ma.tasks = a.mtasks; ma.chunk_heads = a.mheads; ma.ctrl = a.ctrl;
  cudaMemsetAsync(&a.ctrl->mlist_w, 0, 2 * sizeof(int), st);
  cudaMemsetAsync(&a.ctrl->M, 0, sizeof(int), st);
  { k_merge_thread<0><<<gridcap(n, T, a.num_sms, 16), T, 0, st>>>(ma); note_launch(); }   // classify
  { k_merge_chunk<0><<<a.num_sms * 4, T, 0, st>>>(ma); note_launch(); }                  // hub chunk counts
  { k_merge_thread<1><<<gridcap(n, T, a.num_sms, 16), T, 0, st>>>(ma); note_launch(); }
  { k_merge_warp<<<a.num_sms * 16, T, 0, st>>>(ma); note_launch(); }
  { k_merge_chunk<1><<<a.num_sms * 4, T, 0, st>>>(ma); note_launch(); }
}

}  // namespace wbpr
