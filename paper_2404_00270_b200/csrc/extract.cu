// extract.cu — A8: results after the final exact global relabel.
//   flow_i   = e(t_i)                         (Alg. 1 output)
//   bitmap   bit v = [h(v) >= |V|]            (after the final exact GR this is the
//                                             set that cannot reach a sink = S*)
//   cutcap_i = sum of c(u,v) over INPUT edges with u in S*, v not in S*, per instance
//              (the device certificate: must equal flow_i by max-flow/min-cut duality,
//              P:120-127)
#include "internal.h"
#include "kernels.h"

namespace wbpr {

__global__ void k_bitmap(const int* __restrict__ h, int n, int N, uint32_t* bitmap) {
  int nwords = (n + 31) >> 5;
  for (int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < nwords * 32;
       base += gridDim.x * blockDim.x) {
    int v = base + lane_id();
    bool in_s = v < n && ld_cg(h + v) >= N;
    unsigned b = __ballot_sync(FULL, in_s);
    if (lane_id() == 0) bitmap[base >> 5] = b;
  }
}

// One warp per kCutChunk consecutive input edges as rows of 32 (coalesced col/cap loads,
// owners by warp_owner); the side of v is looked up only for edges leaving S*, in the cut
// bitmap when there is one (n/8 bytes: L1/L2-resident, where h is 4n bytes of random gathers).
constexpr int kCutChunk = 32 * 64;
__device__ __forceinline__ bool in_s(const uint32_t* __restrict__ bm, const int* __restrict__ h, int N, int v) {
  return bm ? ((__ldg(bm + (v >> 5)) >> (v & 31)) & 1u) != 0 : ld_cg(h + v) >= N;
}
__global__ void __launch_bounds__(256) k_cutcap(const int64_t* __restrict__ ro, const int32_t* __restrict__ col,
                                                const int32_t* __restrict__ cap, int64_t n, int64_t m,
                                                const int* __restrict__ h, int N, const uint32_t* __restrict__ bm,
                                                const int64_t* __restrict__ vbase, int k, long long* cut) {
  const int lane = lane_id();
  const int64_t E0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * kCutChunk;
  if (E0 >= m) return;
  const int64_t E1 = E0 + kCutChunk < m ? E0 + kCutChunk : m;
  int64_t lo = 0, hi = n;
  while (hi - lo > 1) { int64_t mid = (lo + hi) >> 1; if (__ldg(ro + mid) <= E0) lo = mid; else hi = mid; }
  int ucur = (int)lo;
  int inst = -1;           // instance of the lane's accumulator
  int64_t ilo = 0, ihi = 0;
  long long acc = 0;
  for (int64_t eb = E0; eb < E1; eb += 32) {
    const int64_t i = eb + lane;
    const bool ok = i < E1;
    const int u = warp_owner(ro, (int)n, ucur, ok ? i : E1 - 1);
    ucur = __shfl_sync(FULL, u, 31);
    if (!ok) continue;
    if (!in_s(bm, h, N, u)) continue;      // u not in S*: the edge is not cut (skips col/cap)
    const int v = __ldg(col + i);
    const int c = __ldg(cap + i);
    if (!in_s(bm, h, N, v)) {
      if (u < ilo || u >= ihi) {
        if (acc) atomicAdd((unsigned long long*)(cut + inst), (unsigned long long)acc);
        acc = 0;
        int a = 0, b = k;
        while (b - a > 1) { int mid = (a + b) >> 1; if (__ldg(vbase + mid) <= u) a = mid; else b = mid; }
        inst = a; ilo = __ldg(vbase + a); ihi = __ldg(vbase + a + 1);
      }
      acc += c;
    }
  }
  if (acc) atomicAdd((unsigned long long*)(cut + inst), (unsigned long long)acc);
}

__global__ void k_flows(const long long* __restrict__ e, const long long* __restrict__ snk, int k, long long* flow) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
    flow[i] = ld_cg(e + snk[i]);
}

void extract_results(const SolveParams& p, const int64_t* ro, const int32_t* col, const int32_t* cap,
                     int64_t m, uint32_t* bitmap, const int64_t* vbase, int k, long long* inst_flow,
                     long long* inst_cut, int num_sms, cudaStream_t st) {
  const int T = 256;
  if (bitmap) {
    int64_t words = (p.n + 31) / 32;
    int64_t blocks = (words * 32 + T - 1) / T;
    if (blocks > num_sms * 16) blocks = num_sms * 16;
    { k_bitmap<<<(unsigned)blocks, T, 0, st>>>(p.h, p.n, p.n, bitmap); note_launch(); }
  }
  cudaMemsetAsync(inst_cut, 0, sizeof(long long) * k, st);
  if (m > 0) {
    int64_t threads = (m + kCutChunk - 1) / kCutChunk * 32;
    { k_cutcap<<<(unsigned)((threads + T - 1) / T), T, 0, st>>>(ro, col, cap, p.n, m, p.h, p.n, bitmap, vbase, k, inst_cut); note_launch(); }
  }
  { k_flows<<<(k + T - 1) / T, T, 0, st>>>(p.e, p.snk, k, inst_flow); note_launch(); }
}

}  // namespace wbpr
