// scan.cu — device-wide exclusive prefix sum over int32 (three-pass: tile
// reduce, scan of tile sums, tile scan + offset).  Used by construction (A1)
// for segment offsets and for the merge of duplicate columns.
#include "internal.h"
#include "kernels.h"

#include <atomic>

namespace wbpr {

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

constexpr int kScanThreads = 256;
constexpr int kScanItems = kScanTile / kScanThreads;  // 16

__device__ __forceinline__ int block_excl_scan(int v, int* smem, int* total) {
  // inclusive warp scan
  int lane = lane_id(), w = warp_id();
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[w] = x;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    int s = lane < nw ? smem[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) smem[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  int base = w > 0 ? smem[w - 1] : 0;
  *total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return base + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const int* __restrict__ a, int64_t N, int* part) {
  __shared__ int sm[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t j = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (j < N) s += a[j];
  }
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) k_scan_partials(int* part, int64_t ntiles) {
  __shared__ int sm[32];
  int64_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  int64_t lo = threadIdx.x * per, hi = lo + per < ntiles ? lo + per : ntiles;
  int s = 0;
  for (int64_t i = lo; i < hi; ++i) s += part[i];
  int tot;
  int ex = block_excl_scan(s, sm, &tot);
  for (int64_t i = lo; i < hi; ++i) { int v = part[i]; part[i] = ex; ex += v; }
  if (threadIdx.x == 0) part[ntiles] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(int* a, int64_t N, const int* __restrict__ part,
                                                           int64_t ntiles) {
  __shared__ int sm[32];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t j = base + i;
    v[i] = j < N ? a[j] : 0;
    s += v[i];
  }
  int tot;
  int ex = block_excl_scan(s, sm, &tot) + part[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t j = base + i;
    if (j < N) a[j] = ex;
    ex += v[i];
  }
  if (blockIdx.x == ntiles - 1 && threadIdx.x == 0) a[N] = part[ntiles];
}

// Exclusive scan of a[0..N) in place; a[N] receives the total.  part needs
// ceil(N/4096)+1 ints.
void exclusive_scan(int* a, int64_t N, int* part, cudaStream_t st) {
  if (N <= 0) {
    cudaMemsetAsync(a, 0, sizeof(int), st);
    return;
  }
  int64_t ntiles = (N + kScanTile - 1) / kScanTile;
  { k_scan_reduce<<<(unsigned)ntiles, kScanThreads, 0, st>>>(a, N, part); note_launch(); }
  { k_scan_partials<<<1, 1024, 0, st>>>(part, ntiles); note_launch(); }
  { k_scan_down<<<(unsigned)ntiles, kScanThreads, 0, st>>>(a, N, part, ntiles); note_launch(); }
}

}  // namespace wbpr
