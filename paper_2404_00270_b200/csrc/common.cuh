// common.cuh — device helpers shared by the WBPR sm_100a kernels.
//
// Memory-model notes (B200, sm_100a):
//  * The persistent solve kernel crosses grid barriers; L1 is not coherent across
//    SMs, so every MUTABLE array (cf, e, h, queues, counters) is read with
//    ld.global.cg / ld.relaxed.gpu (served by L2), never through L1.
//  * Immutable arrays (offsets, columns in a separate array, mate, terminal flags)
//    go through the read-only path (ld.global.nc).
#pragma once
#include <climits>
#include <cstdint>
#include <cuda_runtime.h>

#define WBPR_HOSTDEV __host__ __device__ __forceinline__
#define WBPR_DEV __device__ __forceinline__

namespace wbpr {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarp = 32;

// ----------------------------------------------------------------- loads / stores
WBPR_DEV int ld_cg(const int* p) { int v; asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
WBPR_DEV unsigned ld_cg(const unsigned* p) { unsigned v; asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
WBPR_DEV long long ld_cg(const long long* p) { long long v; asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p)); return v; }
WBPR_DEV unsigned long long ld_cg(const unsigned long long* p) { unsigned long long v; asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p)); return v; }
WBPR_DEV int2 ld_cg(const int2* p) { int2 v; asm volatile("ld.global.cg.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p)); return v; }
WBPR_DEV int4 ld_cg(const int4* p) { int4 v; asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)); return v; }
WBPR_DEV void st_cg(int* p, int v) { asm volatile("st.global.cg.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
WBPR_DEV void st_cg(long long* p, long long v) { asm volatile("st.global.cg.s64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }

WBPR_DEV int2 ld_acquire_v2(const int2* p) {
  int2 v; asm volatile("ld.acquire.gpu.global.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory"); return v;
}
WBPR_DEV void st_release_v2(int2* p, int2 v) {
  asm volatile("st.release.gpu.global.v2.s32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
}
WBPR_DEV void st_cg_v2(int2* p, int2 v) {
  asm volatile("st.global.cg.v2.s32 [%0], {%1,%2};" :: "l"(p), "r"(v.x), "r"(v.y) : "memory");
}
WBPR_DEV int atom_or_release(int* p, int v) {
  int o; asm volatile("atom.release.gpu.global.or.b32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o;
}
WBPR_DEV int atom_exch_acquire(int* p, int v) {
  int o; asm volatile("atom.acquire.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory"); return o;
}
WBPR_DEV unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
WBPR_DEV int ld_volatile(const int* p) { int v; asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }

template <typename T> WBPR_DEV T ld_nc(const T* p) { return __ldg(p); }

// L2 eviction-priority hints (createpolicy + .L2::cache_hint): streamed arrays (arcs,
// mate, queues) are loaded evict_first so they do not push the label array h[] (the
// random-gather target, a few MB to ~70 MB) out of the 126 MB L2.
WBPR_DEV unsigned long long policy_evict_first() {
  unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
WBPR_DEV unsigned long long policy_evict_last() {
  unsigned long long p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
WBPR_DEV int2 ld_cg_hint(const int2* p, unsigned long long pol) {
  int2 v; asm volatile("ld.global.cg.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol)); return v;
}
WBPR_DEV int4 ld_cg_hint(const int4* p, unsigned long long pol) {
  int4 v; asm volatile("ld.global.cg.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol)); return v;
}
WBPR_DEV int ld_cg_hint(const int* p, unsigned long long pol) {
  int v; asm volatile("ld.global.cg.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v;
}
// L1-allocating load with an L2 hint, for gathers of neighbour labels h[v] (a few hot
// vertices are read by many warps of an SM).  L1 is not coherent across SMs, but every
// grid barrier of the solve kernel ends with an acquire (CCTL.IVALL invalidates the SM's
// L1), so a cached label is never older than the current phase; inside a phase a stale
// label is one of the interleavings the lock-free algorithm already admits.
WBPR_DEV int ld_ca_hint(const int* p, unsigned long long pol) {
  int v; asm volatile("ld.global.ca.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v;
}
WBPR_DEV int ld_nc_hint(const int* p, unsigned long long pol) {
  int v; asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol)); return v;
}
WBPR_DEV int4 ld_nc_hint(const int4* p, unsigned long long pol) {
  int4 v; asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol)); return v;
}
WBPR_DEV int2 ld_nc_hint(const int2* p, unsigned long long pol) {
  int2 v; asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol)); return v;
}

WBPR_DEV unsigned long long globaltimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

// ----------------------------------------------------------------- warp helpers
WBPR_DEV int lane_id() { return threadIdx.x & 31; }
WBPR_DEV int warp_id() { return threadIdx.x >> 5; }

template <typename T> WBPR_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Owner row of position p in a CSR-like offset array, for a warp walking a row of 32
// consecutive positions: `base` (warp-uniform) is the owner of the row's first position,
// i.e. off[base] <= first < off[base + 1].  Each lane returns the u with
// off[u] <= p < off[u + 1] (p < off[n]); one coalesced load of 32 offsets plus a 5-step
// shuffle search per 32 vertex boundaries crossed (instead of a log2(n)-deep binary
// search per thread).  All lanes must call.
template <typename T>
WBPR_DEV int warp_owner(const T* __restrict__ off, int n, int base, long long p) {
  const int lane = threadIdx.x & 31;
  int owner = -1;
  while (true) {
    const int k = base + 1 + lane;
    const long long wv = k <= n ? (long long)__ldg(off + k) : LLONG_MAX;
    const long long w31 = __shfl_sync(FULL, wv, 31);
    int c = 0;   // number of window entries <= p (entries are non-decreasing)
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const long long v = __shfl_sync(FULL, wv, c + s - 1);
      if (v <= p) c += s;
    }
    if (c == 31 && w31 <= p) c = 32;
    if (owner < 0 && c < 32) owner = base + c;
    if (!__ballot_sync(FULL, owner < 0)) break;
    base += 32;
  }
  return owner;
}

// ----------------------------------------------------------------- block reductions
template <typename T> __device__ T block_sum(T v, T* smem /* >= 32 */) {
  v = warp_sum(v);
  __syncthreads();
  if (lane_id() == 0) smem[warp_id()] = v;
  __syncthreads();
  T r = 0;
  if (warp_id() == 0) {
    r = (lane_id() < (int)(blockDim.x >> 5)) ? smem[lane_id()] : T(0);
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// ----------------------------------------------------------------- grid barrier
// Arrival counter of the software grid barrier of the persistent solve kernel
// (protocol in solve.cu).
struct GridBarrier {
  unsigned count;
  unsigned gen;
};

}  // namespace wbpr
