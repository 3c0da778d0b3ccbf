// build.cu — K-BUILD (A1): device-side construction of the residual layouts of
// PAPER.md §3.2 (Fig. 2):
//   BCSR  one merged, column-sorted segment per vertex with its in- and out-arcs
//         (gapped: segments in vertex order, unused slots between them,
//         seg[u] = {begin, end}) plus mate[p] = slot of the reverse arc: the paper's
//         per-push binary search replaced by edge identities carried
//         through the construction (reading §8(c) #12; merge.cu, k_mate below).
//   RCSR  forward CSR + reversed CSR whose entries carry flow_idx.
// Readings: parallel edges summed, antiparallel pairs share one BCSR arc
// pair, self-loops dropped and counted, zero-capacity pairs kept.
#include <climits>

#include "internal.h"
#include "kernels.h"

namespace wbpr {

constexpr uint64_t kSent = ~0ull;  // self-loop / invalid half-arc: sorts last, never a head

__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ ro, int64_t n, int64_t i) {
  // largest u with ro[u] <= i  (ro non-decreasing, ro[0] = 0)
  int64_t lo = 0, hi = n;  // answer in [0, n)
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(ro + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int row_of32(const int* __restrict__ off, int n, int i) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}

// Row-offset sanity + raw out-degrees (self-loops included as sentinel slots).
__global__ void k_rows(const int64_t* __restrict__ ro, int64_t n, int64_t m, int* deg, Ctrl* ctrl, int write_deg) {
  int mx = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = ro[u], b = ro[u + 1];
    bool bad = a > b || a < 0 || b > m || (u == 0 && a != 0) || (u == n - 1 && b != m);
    if (bad) atomicExch(&ctrl->bad_rows, 1);
    int d = bad ? 0 : (int)(b - a);
    if (write_deg) deg[u] = d;
    mx = max(mx, d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  if (lane_id() == 0) atomicMax(&ctrl->maxlen_out, mx);
}

constexpr int kEdgesPerThread = 8;

// Validation + in-degree histogram, fused with the 64-bit row keys (col << 32 | cap,
// self-loops = all ones) and the per-row "not column-sorted" flags the construction needs.
// One warp per kEdgeChunk consecutive edges as rows of 32 (coalesced loads and key
// stores; owners by warp_owner; the previous key of lane 0 is carried across rows).
constexpr int kEdgeRows = 8;
constexpr int kEdgeChunk = 32 * kEdgeRows * 8;
__global__ void __launch_bounds__(256) k_edges(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                                               const int32_t* __restrict__ cap, int64_t n, int64_t m, int* indeg,
                                               Ctrl* ctrl, int count_in, const int64_t* __restrict__ vbase, int k,
                                               uint64_t* keys, uint8_t* need, int* src) {
  const int lane = lane_id();
  const int64_t E0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * kEdgeChunk;
  if (E0 >= m) return;
  const int64_t E1 = E0 + kEdgeChunk < m ? E0 + kEdgeChunk : m;
  int ucur = (int)row_of(ro, n, E0);
  // carry: owner and key of edge eb - 1 (the edge before lane 0's)
  int cu = -1;
  uint64_t ck = 0;
  if (E0 > 0) {
    cu = (int)row_of(ro, n, E0 - 1);
    const int pv = __ldg(col + E0 - 1);
    ck = (pv == cu) ? kSent : (((uint64_t)(uint32_t)pv << 32) | (uint32_t)__ldg(cap + E0 - 1));
  }
  int64_t ilo = 0, ihi = k > 1 ? 0 : n;   // instance [ilo, ihi) of the lane's current owner (A10)
  int loops = 0;
  for (int64_t eb = E0; eb < E1; eb += 32) {
    const int64_t i = eb + lane;
    const bool ok = i < E1;
    const int u = warp_owner(ro, (int)n, ucur, ok ? i : E1 - 1);
    ucur = __shfl_sync(FULL, u, 31);
    const int v = ok ? __ldg(col + i) : 0;
    const int c = ok ? __ldg(cap + i) : 0;
    const uint64_t key = (v == u) ? kSent : (((uint64_t)(uint32_t)v << 32) | (uint32_t)c);
    const int pu0 = __shfl_up_sync(FULL, u, 1);
    const uint64_t pk0 = __shfl_up_sync(FULL, key, 1);
    const int pu = lane == 0 ? cu : pu0;
    const uint64_t pk = lane == 0 ? ck : pk0;
    cu = __shfl_sync(FULL, u, 31);
    ck = __shfl_sync(FULL, key, 31);
    if (!ok) continue;
    keys[i] = key;
    if (src) src[i] = u;
    if (pu == u && key < pk) { need[u] = 1; ctrl->any_unsorted = 1; }
    if (k > 1 && (u < ilo || u >= ihi)) {
      int a = 0, b = k;
      while (b - a > 1) { int mid = (a + b) >> 1; if (__ldg(vbase + mid) <= u) a = mid; else b = mid; }
      ilo = __ldg(vbase + a); ihi = __ldg(vbase + a + 1);
    }
    if (v < ilo || v >= ihi || c < 0) {
      atomicMin((unsigned long long*)&ctrl->bad_edge, (unsigned long long)i);
      continue;
    }
    if (v == u) { ++loops; continue; }
    if (count_in) atomicAdd(indeg + v, 1);
  }
  loops = warp_sum(loops);
  if (lane == 0 && loops) atomicAdd(&ctrl->selfloops, loops);
}

__global__ void k_maxlen(const int* __restrict__ deg, int64_t n, Ctrl* ctrl) {
  int mx = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, deg[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  if (lane_id() == 0) atomicMax(&ctrl->maxlen, mx);
}

__global__ void k_ro_to_i32(const int64_t* __restrict__ ro, int64_t n, int* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int)ro[i];
}

// flags[soff[x]] = 1 for non-empty segments (row starts).
__global__ void k_rowstarts(const int* __restrict__ soff, int64_t n, int* flags) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    if (soff[x] < soff[x + 1]) flags[soff[x]] = 1;
}

// head(j) = key is real and (j starts its row or its column differs from j-1)
__global__ void k_heads(const uint64_t* __restrict__ keys, int64_t H, int* flags) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < H; j += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = keys[j];
    int f;
    if (k == kSent) f = 0;
    else if (flags[j]) f = 1;
    else f = (uint32_t)(k >> 32) != (uint32_t)(keys[j - 1] >> 32);
    flags[j] = f;
  }
}

// new offsets: off[x] = scan[soff[x]]
__global__ void k_newoff(const int* __restrict__ soff, const int* __restrict__ scan, int64_t n, int* off) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n; x += (int64_t)gridDim.x * blockDim.x)
    off[x] = scan[soff[x]];
}

// Merge each run of equal columns into one slot: cf = sum of capacities
// (parallel edges summed).  Overflow beyond INT32_MAX is reported.
__global__ void k_merge_write(const uint64_t* __restrict__ keys, int64_t H, const int* __restrict__ scan,
                              int2* arc, int* cap0, Ctrl* ctrl) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < H; j += (int64_t)gridDim.x * blockDim.x) {
    int slot = scan[j];
    if (scan[j + 1] == slot) continue;  // not a head
    uint64_t k = keys[j];
    uint32_t c = (uint32_t)(k >> 32);
    long long sum = (long long)(uint32_t)(k & 0xffffffffu);
    for (int64_t q = j + 1; q < H; ++q) {
      if (scan[q + 1] != scan[q]) break;  // next head
      uint64_t kq = keys[q];
      if (kq == kSent) break;
      sum += (long long)(uint32_t)(kq & 0xffffffffu);
    }
    if (sum > INT_MAX) { atomicExch(&ctrl->overflow, 1); sum = INT_MAX; }
    arc[slot] = make_int2((int)c, (int)sum);
    if (cap0) cap0[slot] = (int)sum;
  }
}

// mate[] from the edge identities carried through the construction (merge.cu): the
// in-list entry t of input edge e = ine[t] = (u -> x) sits at slot q = inslot[t] of seg(x)
// and pairs with the slot p = outslot[e] of e's out-half-arc in seg(u) — the paper's
// backward-arc binary search replaced by one lookup per input edge.  Pairs
// with arcs in both directions (and parallel edges) are written more than once, always
// with the same values; every slot is written by itself or by its partner.
constexpr int kMatePerThread = 4;
__global__ void __launch_bounds__(256) k_mate(const int* __restrict__ ine, const int* __restrict__ inslot,
                                              const int* __restrict__ outslot, const int* __restrict__ rsoff, int n,
                                              int* mate, const int* __restrict__ cap0, Ctrl* ctrl) {
  const int total = __ldg(rsoff + n);   // in-list entries
  const int base = blockIdx.x * blockDim.x * kMatePerThread + threadIdx.x;
  int e[kMatePerThread], q[kMatePerThread];
#pragma unroll
  for (int r = 0; r < kMatePerThread; ++r) {
    const int t = base + r * blockDim.x;
    e[r] = t < total ? __ldg(ine + t) : -1;
    q[r] = t < total ? __ldg(inslot + t) : -1;
  }
  int p[kMatePerThread];
#pragma unroll
  for (int r = 0; r < kMatePerThread; ++r) p[r] = e[r] >= 0 ? __ldg(outslot + e[r]) : -1;
#pragma unroll
  for (int r = 0; r < kMatePerThread; ++r)
    if (p[r] >= 0) { mate[q[r]] = p[r]; mate[p[r]] = q[r]; }
  // the pair's residual capacities sum to cap0[p] + cap0[q] forever (a push moves d between
  // them): beyond INT32_MAX the int32 cf would wrap, so report EOVERFLOW.  Only checked when
  // the merge saw a capacity above INT32_MAX / 2 (otherwise no pair can exceed it).
  if (ld_cg(&ctrl->bigcap)) {
#pragma unroll
    for (int r = 0; r < kMatePerThread; ++r)
      if (p[r] >= 0 && (long long)__ldg(cap0 + p[r]) + (long long)__ldg(cap0 + q[r]) > INT_MAX)
        atomicExch(&ctrl->overflow, 1);
  }
}

// RCSR reverse in-degree over forward arcs
__global__ void k_rdeg(const int2* __restrict__ farc, int Mf, int* rdeg) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < Mf; p += gridDim.x * blockDim.x)
    atomicAdd(rdeg + farc[p].x, 1);
}

// RCSR reverse scatter: forward arc p = (u -> v) lands in v's reverse segment
// with key (u, p); u distinct per segment after the merge, so keys are unique.
__global__ void k_scatter_rev(const int* __restrict__ foff, const int2* __restrict__ farc, int n, int Mf,
                              const int* __restrict__ roff, int* cursor, uint64_t* keys) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t p0 = t * kEdgesPerThread;
  if (p0 >= Mf) return;
  int u = row_of32(foff, n, (int)p0);
  int p1 = (int)(p0 + kEdgesPerThread < (int64_t)Mf ? p0 + kEdgesPerThread : (int64_t)Mf);
  for (int p = (int)p0; p < p1; ++p) {
    while (__ldg(foff + u + 1) <= p) ++u;
    int v = farc[p].x;
    int q = roff[v] + atomicAdd(cursor + v, 1);
    keys[q] = ((uint64_t)(uint32_t)u << 32) | (uint32_t)p;
  }
}

__global__ void k_write_rarc(const uint64_t* __restrict__ keys, int Mf, int2* rarc, int* bcf) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Mf; q += gridDim.x * blockDim.x) {
    uint64_t k = keys[q];
    rarc[q] = make_int2((int)(k >> 32), (int)(k & 0xffffffffu));
    bcf[q] = 0;   // backward cf of forward arc q (indexed by forward arc)
  }
}

// ------------------------------------------------------------------ host side
static unsigned grid_for(int64_t items, int threads, int num_sms, int per_sm = 16) {
  int64_t b = (items + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}
static unsigned grid_exact(int64_t items, int threads) {
  int64_t b = (items + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : b);
}

// Phase 1 of the build: validation and segment lengths.  Leaves seg lengths in
// deg[] and fills ctrl->{bad_edge, bad_rows, selfloops, maxlen}.
void build_validate(const BuildArgs& a, cudaStream_t st) {
  const int T = 256;
  // BCSR: deg[] = in-degrees (out-rows come straight from the input); RCSR: deg[] = out-degrees
  if (a.layout == 0) cudaMemsetAsync(a.deg, 0, sizeof(int) * a.n, st);
  { k_rows<<<grid_for(a.n, T, a.num_sms), T, 0, st>>>(a.ro, a.n, a.m, a.deg, a.ctrl, a.layout != 0); note_launch(); }
  int64_t threads = (a.m + kEdgeChunk - 1) / kEdgeChunk * 32;
  // row keys go to region B (BCSR merge build) / region A (RCSR forward sort)
  cudaMemsetAsync(a.need, 0, a.n, st);
  if (a.m > 0)
    { k_edges<<<grid_exact(threads, T), T, 0, st>>>(a.ro, a.col, a.cap, a.n, a.m, a.deg, a.ctrl,
                                                   a.layout == 0 ? 1 : 0, a.vbase, a.k,
                                                   a.layout == 0 ? a.tmp : a.keys, a.need,
                                                   a.layout == 0 ? a.src : nullptr); note_launch(); }
  { k_maxlen<<<grid_for(a.n, T, a.num_sms), T, 0, st>>>(a.deg, a.n, a.ctrl); note_launch(); }
}

void build_bcsr_mate(const BuildArgs& a, cudaStream_t st) {
  const int T = 256;
  // one thread per kMatePerThread in-list entries (rsoff[n] of them; m bounds it)
  const int64_t per_block = (int64_t)T * kMatePerThread;
  if (a.m > 0) { k_mate<<<(unsigned)((a.m + per_block - 1) / per_block), T, 0, st>>>(a.ine, a.inslot, a.outslot, a.rsoff, (int)a.n, a.mate, a.cap0, a.ctrl); note_launch(); }
}

void k_ro_to_i32_ext(const int64_t* ro, int64_t n, int* out, int num_sms, cudaStream_t st) {
  { k_ro_to_i32<<<grid_for(n + 1, 256, num_sms), 256, 0, st>>>(ro, n, out); note_launch(); }
}

void build_rcsr_forward(const BuildArgs& a, cudaStream_t st) {
  const int T = 256;
  const int64_t n = a.n, m = a.m;
  { k_ro_to_i32<<<grid_for(n + 1, T, a.num_sms), T, 0, st>>>(a.ro, n, a.soff); note_launch(); }
  // rows already column-sorted in the input are not sorted again (keys + flags from k_edges)
  segmented_sort_filtered(a.keys, a.tmp, a.soff, (int)n, a.maxlen, a.need, a.ctrl, a.arc, a.arc + a.H / 2, a.q0,
                          a.num_sms, st);
  int* flags = (int*)a.tmp;
  cudaMemsetAsync(flags, 0, sizeof(int) * (m + 1), st);
  { k_rowstarts<<<grid_for(n, T, a.num_sms), T, 0, st>>>(a.soff, n, flags); note_launch(); }
  if (m > 0) { k_heads<<<grid_for(m, T, a.num_sms, 32), T, 0, st>>>(a.keys, m, flags); note_launch(); }
  exclusive_scan(flags, m, a.scan_part, st);
  { k_newoff<<<grid_for(n + 1, T, a.num_sms), T, 0, st>>>(a.soff, flags, n, a.off); note_launch(); }
  if (m > 0) { k_merge_write<<<grid_for(m, T, a.num_sms, 32), T, 0, st>>>(a.keys, m, flags, a.arc, a.cap0, a.ctrl); note_launch(); }
  cudaMemcpyAsync(&a.ctrl->M, flags + m, sizeof(int), cudaMemcpyDeviceToDevice, st);
}

// Reverse CSR over the Mf merged forward arcs; needs the max reverse segment
// length (host-known after a sync) for the sort.
void build_rcsr_reverse_counts(const BuildArgs& a, int Mf, cudaStream_t st) {
  const int T = 256;
  cudaMemsetAsync(a.deg, 0, sizeof(int) * a.n, st);
  if (Mf > 0) { k_rdeg<<<grid_for(Mf, T, a.num_sms, 32), T, 0, st>>>(a.arc, Mf, a.deg); note_launch(); }
  cudaMemsetAsync(&a.ctrl->maxlen, 0, sizeof(int), st);
  { k_maxlen<<<grid_for(a.n, T, a.num_sms), T, 0, st>>>(a.deg, a.n, a.ctrl); note_launch(); }
  cudaMemcpyAsync(a.roff, a.deg, sizeof(int) * a.n, cudaMemcpyDeviceToDevice, st);
  exclusive_scan(a.roff, a.n, a.scan_part, st);
}

void build_rcsr_reverse(const BuildArgs& a, int Mf, int maxlen, cudaStream_t st) {
  const int T = 256;
  cudaMemsetAsync(a.cursor, 0, sizeof(int) * a.n, st);
  int64_t threads = ((int64_t)Mf + kEdgesPerThread - 1) / kEdgesPerThread;
  if (Mf > 0)
    { k_scatter_rev<<<grid_exact(threads, T), T, 0, st>>>(a.off, a.arc, (int)a.n, Mf, a.roff, a.cursor, a.keys); note_launch(); }
  segmented_sort(a.keys, a.tmp, a.roff, (int)a.n, maxlen, a.ctrl, a.rarc, a.rarc + a.m / 2, a.q0, a.num_sms, st);
  if (Mf > 0) { k_write_rarc<<<grid_for(Mf, T, a.num_sms, 32), T, 0, st>>>(a.keys, Mf, a.rarc, a.bcf); note_launch(); }
}

}  // namespace wbpr
