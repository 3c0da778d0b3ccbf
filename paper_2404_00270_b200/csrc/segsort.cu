// segsort.cu — hand-written segmented sort (32- or 64-bit keys) for residual
// construction (A1).  BCSR needs every vertex segment sorted by column (PAPER.md
// §3.2, "sort the column list in ascending order by vertex ID") so that
// duplicate columns become adjacent (merge) and the reverse arc can be located
// by binary search once, into mate[].
//
// Segment classes (lengths from 1 to ~1.6e5 at R-MAT scale 22):
//   len <= 32         one warp per segment, rank sort in registers (32 shuffles)
//   32 < len <= 1024  one warp per segment (<= 512 for 64-bit keys), register bitonic
//                     network sized to the length (2..32 keys per lane; shuffles for the
//                     cross-lane stages, no shared memory, no barriers)
//   ... len <= 4096   one 512-thread CTA: each warp sorts a 256-key chunk in
//                     registers, then merge-path passes in shared memory
//   len > 4096        4096-key chunks sorted as above, then log2(len/4096) merge
//                     passes in global memory (co-rank search, 8 outputs per thread),
//                     ping-ponging between keys and tmp.
// An optional per-segment `need` flag skips segments known to be sorted already.
#include "internal.h"
#include "kernels.h"

namespace wbpr {

constexpr int kTileThreads = 512;
constexpr int kMedLen = 256;   // warp register sort up to this length
constexpr int kWarpMergeMax = 1024;   // warp chunk-sort + shared-memory merge up to this length (32-bit keys)

template <typename K> __device__ __forceinline__ K key_max() { return (K)~(K)0; }

template <typename K>
__global__ void __launch_bounds__(256) k_sort_warp(K* keys, const int* __restrict__ off, int nseg,
                                                   const uint8_t* __restrict__ need) {
  // each warp screens 32 consecutive segments with one ballot, then rank-sorts the ones
  // with 2..32 keys (and a set `need` flag) one after the other
  int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = lane_id();
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int base = wg * 32; base < nseg; base += nw * 32) {
    int sgi = base + lane;
    int beg = 0, len = 0;
    if (sgi < nseg && (!need || need[sgi])) { beg = off[sgi]; len = off[sgi + 1] - beg; }
    // segments of <= 8 / <= 16 keys: 4 / 2 at a time, one 8- / 16-lane group each (rank
    // sort over the group's lanes: 8 / 16 shuffles per key instead of 32)
    unsigned t8 = __ballot_sync(FULL, len >= 2 && len <= 8);
    while (t8) {
      int jg[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) { jg[g] = t8 ? __ffs(t8) - 1 : -1; t8 &= t8 ? t8 - 1 : 0u; }
      const int g = lane >> 3, sub = lane & 7;
      const int j = g == 0 ? jg[0] : g == 1 ? jg[1] : g == 2 ? jg[2] : jg[3];
      const int b = __shfl_sync(FULL, beg, j < 0 ? 0 : j), l0 = __shfl_sync(FULL, len, j < 0 ? 0 : j);
      const int l = j < 0 ? 0 : l0;
      K k = sub < l ? keys[b + sub] : key_max<K>();
      int rank = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        K o = __shfl_sync(FULL, k, q, 8);
        rank += (o < k) || (o == k && q < sub);
      }
      __syncwarp();
      if (sub < l) keys[b + rank] = k;
    }
    unsigned t16 = __ballot_sync(FULL, len > 8 && len <= 16);
    while (t16) {
      const int j0 = __ffs(t16) - 1;
      t16 &= t16 - 1;
      const int j1 = t16 ? __ffs(t16) - 1 : -1;
      if (t16) t16 &= t16 - 1;
      const int sub = lane & 15;
      const int j = lane < 16 ? j0 : j1;
      const int b = __shfl_sync(FULL, beg, j < 0 ? 0 : j), l0 = __shfl_sync(FULL, len, j < 0 ? 0 : j);
      const int l = j < 0 ? 0 : l0;
      K k = sub < l ? keys[b + sub] : key_max<K>();
      int rank = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        K o = __shfl_sync(FULL, k, q, 16);
        rank += (o < k) || (o == k && q < sub);
      }
      __syncwarp();
      if (sub < l) keys[b + rank] = k;
    }
    unsigned todo = __ballot_sync(FULL, len > 16 && len <= 32);
    while (todo) {
      int j = __ffs(todo) - 1;
      todo &= todo - 1;
      int b = __shfl_sync(FULL, beg, j), l = __shfl_sync(FULL, len, j);
      K k = lane < l ? keys[b + lane] : key_max<K>();
      int rank = 0;
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        K o = __shfl_sync(FULL, k, q);
        rank += (o < k) || (o == k && q < lane);
      }
      __syncwarp();
      if (lane < l) keys[b + rank] = k;
    }
  }
}

// Bitonic network over P = 32*NR keys held by one warp as r[j] = element j*32 + lane.
template <typename K, int NR>
__device__ __forceinline__ void warp_bitonic(K (&r)[NR], int lane) {
  constexpr int P = 32 * NR;
#pragma unroll
  for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= 32) {
        const int dj = jj >> 5;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          if ((j & dj) == 0) {
            const bool up = ((j * 32 + lane) & k) == 0;
            K a = r[j], b = r[j | dj];
            if ((a > b) == up) { r[j] = b; r[j | dj] = a; }
          }
        }
      } else {
        const bool lower = (lane & jj) == 0;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          K o = __shfl_xor_sync(FULL, r[j], jj);
          const bool up = ((j * 32 + lane) & k) == 0;
          K mn = r[j] < o ? r[j] : o, mx = r[j] < o ? o : r[j];
          r[j] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

template <typename K, int NR>
__device__ __forceinline__ void warp_sort_segment(K* keys, int beg, int len, int lane) {
  K r[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    int e = j * 32 + lane;
    r[j] = e < len ? keys[beg + e] : key_max<K>();
  }
  warp_bitonic<K, NR>(r, lane);
#pragma unroll
  for (int j = 0; j < NR; ++j) {
    int e = j * 32 + lane;
    if (e < len) keys[beg + e] = r[j];
  }
}

// Longest segment sorted by one warp (32-bit keys: <= 1024 keys as 256-key register
// bitonic chunks merged in warp-private shared memory; 64-bit keys: <= 256 in registers).
// Longer segments go to the CTA tile sort, whose merge passes need several warps to pay off.
template <typename K> constexpr int warp_sort_max() { return sizeof(K) == 4 ? kWarpMergeMax : kMedLen; }

template <typename K>
__global__ void __launch_bounds__(256) k_sort_med(K* keys, const int2* __restrict__ items, const int* count) {
  const int nitems = *count;
  int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int nw = (gridDim.x * blockDim.x) >> 5;
  int lane = lane_id();
  for (int it = wg; it < nitems; it += nw) {
    int2 item = items[it];
    if (item.y > kMedLen) continue;   // (32-bit keys) k_sort_wm
    if (item.y <= 64) warp_sort_segment<K, 2>(keys, item.x, item.y, lane);
    else if (item.y <= 128) warp_sort_segment<K, 4>(keys, item.x, item.y, lane);
    else warp_sort_segment<K, 8>(keys, item.x, item.y, lane);
  }
}

// Enumerate sort items: 32 < len <= 256 -> warp items; 256 < len <= tile -> CTA item;
// longer segments -> ceil(len/tile) CTA chunk items and the `big` list.
// (medium items are appended with one atomic per warp: they are numerous, and same-address
// atomics from every thread serialise)
__global__ void k_sort_items(const int* __restrict__ off, int nseg, const uint8_t* __restrict__ need,
                             int2* items, int2* items_med, int* big, Ctrl* ctrl, int medmax) {
  const int lane = lane_id();
  for (int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < nseg; base += gridDim.x * blockDim.x) {
    const int sgi = base + lane;
    int beg = 0, len = 0;
    if (sgi < nseg && (!need || need[sgi])) { beg = off[sgi]; len = off[sgi + 1] - beg; }
    const bool med = len > 32 && len <= medmax;
    const unsigned bm = __ballot_sync(FULL, med);
    int pm = 0;
    if (lane == 0 && bm) pm = atomicAdd(&ctrl->sort_items_med, __popc(bm));
    pm = __shfl_sync(FULL, pm, 0);
    if (med) items_med[pm + __popc(bm & ((1u << lane) - 1u))] = make_int2(beg, len);
    if (len <= medmax) continue;
    int nit = (len + kSortTile - 1) / kSortTile;
    int idx = atomicAdd(&ctrl->sort_items, nit);
    for (int c = 0; c < nit; ++c) {
      int s = beg + c * kSortTile;
      int l = min(kSortTile, beg + len - s);
      items[idx + c] = make_int2(s, l);
    }
    if (nit > 1) big[atomicAdd(&ctrl->hub_chunks, 1)] = sgi;
  }
}

// Smallest i in [max(0,k-lb), min(k,la)] with A[i] > B[k-i-1] (A wins ties): the
// number of outputs among the first k that come from A.
template <typename K>
__device__ __forceinline__ int co_rank(int k, const K* A, int la, const K* B, int lb) {
  int lo = k - lb > 0 ? k - lb : 0, hi = k < la ? k : la;
  while (lo < hi) {
    int i = (lo + hi) >> 1;
    if (A[i] <= B[k - i - 1]) lo = i + 1; else hi = i;
  }
  return lo;
}

// 256 < len <= kWarpMergeMax (32-bit keys): one warp sorts the 256-key chunks of the
// segment (padded to a power of two) with the register bitonic network, then merges them
// pairwise in its own shared memory (merge path: each lane emits a run of consecutive
// outputs from its co-rank) and writes the result back coalesced.
__global__ void __launch_bounds__(256) k_sort_wm(uint32_t* keys, const int2* __restrict__ items, const int* count) {
  extern __shared__ __align__(16) uint32_t wsm[];
  uint32_t* const A0 = wsm + warp_id() * 2 * kWarpMergeMax;
  uint32_t* const B0 = A0 + kWarpMergeMax;
  const int nitems = *count;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int lane = lane_id();
  for (int it = wg; it < nitems; it += nw) {
    const int2 item = items[it];
    const int beg = item.x, len = item.y;
    if (len <= kMedLen) continue;      // k_sort_med
    const int total = len <= 512 ? 512 : kWarpMergeMax;
    for (int c = 0; c < total / kMedLen; ++c) {
      uint32_t r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = c * kMedLen + j * 32 + lane;
        r[j] = e < len ? keys[beg + e] : 0xffffffffu;
      }
      warp_bitonic<uint32_t, 8>(r, lane);
#pragma unroll
      for (int j = 0; j < 8; ++j) A0[c * kMedLen + j * 32 + lane] = r[j];
    }
    __syncwarp();
    uint32_t* src = A0;
    uint32_t* dst = B0;
    const int per = total / 32;
    for (int wd = kMedLen; wd < total; wd <<= 1) {
      const int kk = lane * per;
      const int pair0 = kk / (2 * wd) * (2 * wd);
      const uint32_t* SA = src + pair0;
      const uint32_t* SB = SA + wd;
      const int k = kk - pair0;
      int i = co_rank<uint32_t>(k, SA, wd, SB, wd);
      int j = k - i;
      for (int q = 0; q < per; ++q) {
        const bool takeA = j >= wd || (i < wd && SA[i] <= SB[j]);
        dst[kk + q] = takeA ? SA[i++] : SB[j++];
      }
      __syncwarp();
      uint32_t* t = src; src = dst; dst = t;
    }
    for (int e = lane; e < len; e += 32) keys[beg + e] = src[e];
    __syncwarp();
  }
}

template <typename K>
__global__ void __launch_bounds__(kTileThreads) k_sort_tile(K* keys, const int2* __restrict__ items,
                                                             const int* count) {
  extern __shared__ __align__(16) unsigned char smraw[];
  K* A = reinterpret_cast<K*>(smraw);
  K* B = A + kSortTile;
  const int nitems = *count;
  const int lane = lane_id(), w = warp_id();
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    int2 item = items[it];
    const int beg = item.x, len = item.y;
    const int nc = (len + kMedLen - 1) / kMedLen;          // 256-key chunks
    if (w < nc) {
      K r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int e = w * kMedLen + j * 32 + lane;
        r[j] = e < len ? keys[beg + e] : key_max<K>();
      }
      warp_bitonic<K, 8>(r, lane);
#pragma unroll
      for (int j = 0; j < 8; ++j) A[w * kMedLen + j * 32 + lane] = r[j];
    }
    __syncthreads();
    const int total = nc * kMedLen;
    K* src = A;
    K* dst = B;
    for (int wd = kMedLen; wd < total; wd <<= 1) {
      for (int kk = threadIdx.x * 8; kk < total; kk += blockDim.x * 8) {
        int pair0 = kk / (2 * wd) * (2 * wd);
        int la = min(wd, total - pair0);
        int lb = min(wd, total - pair0 - la);
        if (lb < 0) lb = 0;
        const K* SA = src + pair0;
        const K* SB = SA + la;
        int k = kk - pair0;
        int i = co_rank<K>(k, SA, la, SB, lb);
        int j = k - i;
        int outn = min(8, la + lb - k);
        for (int q = 0; q < outn; ++q) {
          bool takeA = j >= lb || (i < la && SA[i] <= SB[j]);
          dst[kk + q] = takeA ? SA[i++] : SB[j++];
        }
      }
      __syncthreads();
      K* t = src; src = dst; dst = t;
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) keys[beg + i] = src[i];
    __syncthreads();
  }
}

// One merge pass of width w over every big segment (one CTA per segment).
// One merge pass of width w over every big segment: one CTA per segment when there are
// many, else every segment in turn by the whole grid (a 2^20-entry hub list would
// otherwise be merged by a single CTA).  Each thread emits 8 outputs from its co-rank.
template <typename K>
__device__ __forceinline__ void merge_pass_task(const K* __restrict__ src, K* dst, int beg, int len, int w, int tk) {
  int kk = tk << 3;
  int pair0 = kk / (2 * w) * (2 * w);
  int la = min(w, len - pair0);
  int lb = min(w, len - pair0 - la);
  if (lb < 0) lb = 0;
  const K* A = src + beg + pair0;
  const K* B = A + la;
  int k = kk - pair0;
  int i = co_rank<K>(k, A, la, B, lb);
  int j = k - i;
  int outn = min(8, la + lb - k);
  K* O = dst + beg + kk;
  for (int q = 0; q < outn; ++q) {
    bool takeA = j >= lb || (i < la && A[i] <= B[j]);
    O[q] = takeA ? A[i++] : B[j++];
  }
}

template <typename K>
__global__ void __launch_bounds__(256) k_merge_pass(const K* __restrict__ src, K* dst, const int* __restrict__ off,
                                                    const int* __restrict__ big, const int* count, int w) {
  const int nbig = *count;
  if (nbig >= (int)gridDim.x / 4) {
    for (int bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
      int sgi = big[bi];
      int beg = off[sgi], len = off[sgi + 1] - beg;
      int ntask = (len + 7) >> 3;
      for (int tk = threadIdx.x; tk < ntask; tk += blockDim.x) merge_pass_task<K>(src, dst, beg, len, w, tk);
    }
  } else {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
    for (int bi = 0; bi < nbig; ++bi) {
      int sgi = big[bi];
      int beg = off[sgi], len = off[sgi + 1] - beg;
      int ntask = (len + 7) >> 3;
      for (int tk = gt; tk < ntask; tk += T) merge_pass_task<K>(src, dst, beg, len, w, tk);
    }
  }
}

template <typename K>
__global__ void __launch_bounds__(256) k_copy_big(const K* __restrict__ src, K* dst, const int* __restrict__ off,
                                                  const int* __restrict__ big, const int* count) {
  const int nbig = *count;
  if (nbig >= (int)gridDim.x / 4) {   // many big segments: one CTA each
    for (int bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
      int sgi = big[bi];
      int beg = off[sgi], len = off[sgi + 1] - beg;
      for (int i = threadIdx.x; i < len; i += blockDim.x) dst[beg + i] = src[beg + i];
    }
    return;
  }
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  for (int bi = 0; bi < nbig; ++bi) {   // few (hub) segments: the whole grid on each
    int sgi = big[bi];
    int beg = off[sgi], len = off[sgi + 1] - beg;
    for (int i = gt; i < len; i += T) dst[beg + i] = src[beg + i];
  }
}

template <typename K>
void segmented_sort_t(K* keys, K* tmp, const int* off, int nseg, int maxlen, const uint8_t* need, Ctrl* ctrl,
                      int2* items, int2* items_med, int* big, int num_sms, cudaStream_t st) {
  if (nseg <= 0 || maxlen < 2) return;
  cudaMemsetAsync(&ctrl->sort_items, 0, sizeof(int), st);
  cudaMemsetAsync(&ctrl->sort_items_med, 0, sizeof(int), st);
  cudaMemsetAsync(&ctrl->hub_chunks, 0, sizeof(int), st);
  {
    int64_t blocks = ((int64_t)nseg + 255) / 256;
    if (blocks > (int64_t)num_sms * 32) blocks = (int64_t)num_sms * 32;
    { k_sort_warp<K><<<(unsigned)blocks, 256, 0, st>>>(keys, off, nseg, need); note_launch(); }
  }
  if (maxlen <= 32) return;
  {
    int64_t blocks = (nseg + 255) / 256;
    if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
    { k_sort_items<<<(unsigned)blocks, 256, 0, st>>>(off, nseg, need, items, items_med, big, ctrl, warp_sort_max<K>()); note_launch(); }
  }
  { k_sort_med<K><<<num_sms * 16, 256, 0, st>>>(keys, items_med, &ctrl->sort_items_med); note_launch(); }
  if constexpr (sizeof(K) == 4) {
    if (maxlen > kMedLen) {
      const int smem = 8 * 2 * kWarpMergeMax * (int)sizeof(uint32_t);
      cudaFuncSetAttribute(k_sort_wm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      k_sort_wm<<<num_sms * 3, 256, smem, st>>>(reinterpret_cast<uint32_t*>(keys), items_med, &ctrl->sort_items_med);
      note_launch();
    }
  }
  if (maxlen <= warp_sort_max<K>()) return;
  {
    const int smem = 2 * kSortTile * (int)sizeof(K);
    cudaFuncSetAttribute(k_sort_tile<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int per_sm = sizeof(K) == 8 ? 3 : 6;
    k_sort_tile<K><<<num_sms * per_sm, kTileThreads, smem, st>>>(keys, items, &ctrl->sort_items);
    note_launch();
  }
  if (maxlen <= kSortTile) return;
  const K* src = keys;
  K* dst = tmp;
  int passes = 0;
  for (int w = kSortTile; w < maxlen; w <<= 1) {
    { k_merge_pass<K><<<num_sms * 8, 256, 0, st>>>(src, dst, off, big, &ctrl->hub_chunks, w); note_launch(); }
    const K* t = src; src = dst; dst = const_cast<K*>(t);
    ++passes;
  }
  if (passes & 1) { k_copy_big<K><<<num_sms * 8, 256, 0, st>>>(tmp, keys, off, big, &ctrl->hub_chunks); note_launch(); }
}

void segmented_sort(uint64_t* keys, uint64_t* tmp, const int* off, int nseg, int maxlen, Ctrl* ctrl,
                    int2* items, int2* items_med, int* big, int num_sms, cudaStream_t st) {
  segmented_sort_t<uint64_t>(keys, tmp, off, nseg, maxlen, nullptr, ctrl, items, items_med, big, num_sms, st);
}
void segmented_sort_filtered(uint64_t* keys, uint64_t* tmp, const int* off, int nseg, int maxlen,
                             const uint8_t* need, Ctrl* ctrl, int2* items, int2* items_med, int* big, int num_sms,
                             cudaStream_t st) {
  segmented_sort_t<uint64_t>(keys, tmp, off, nseg, maxlen, need, ctrl, items, items_med, big, num_sms, st);
}
void segmented_sort32(uint32_t* keys, uint32_t* tmp, const int* off, int nseg, int maxlen, Ctrl* ctrl, int2* items,
                      int2* items_med, int* big, int num_sms, cudaStream_t st) {
  segmented_sort_t<uint32_t>(keys, tmp, off, nseg, maxlen, nullptr, ctrl, items, items_med, big, num_sms, st);
}

}  // namespace wbpr
