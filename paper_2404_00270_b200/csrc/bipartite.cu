// bipartite.cu — A9: maximum bipartite matching as maximum flow (§4.1
// P:433, "the super-source and super-sink connect to two groups of vertices").
// Network ids per SPEC S:304: s = 0, left l -> 1+l, right r -> 1+nL+r,
// t = nL+nR+1, unit capacities; built directly on the device as the CSR the
// max-flow path consumes.  After the solve, right vertex x with saturated x -> t
// takes the lowest-id left vertex whose flow into x is 1 (the other incoming
// units are stranded preflow on the source side).  Every left vertex has net
// outflow <= 1, so the pairs form a matching whose size is e(t).
#include "internal.h"
#include "kernels.h"

namespace wbpr {

__global__ void k_bip_hist(const int32_t* __restrict__ l, const int32_t* __restrict__ r, int64_t E, int64_t nL,
                           int64_t nR, int* deg, Ctrl* ctrl) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    int a = l[i], b = r[i];
    if (a < 0 || a >= nL || b < 0 || b >= nR) {
      atomicMin((unsigned long long*)&ctrl->bad_edge, (unsigned long long)i);
      continue;
    }
    atomicAdd(deg + a, 1);
  }
}

__global__ void k_bip_rows(const int* __restrict__ lscan, int64_t nL, int64_t nR, int64_t E, int64_t* ro) {
  int64_t n = nL + nR + 2;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n; x += (int64_t)gridDim.x * blockDim.x) {
    int64_t v;
    if (x == 0) v = 0;
    else if (x <= nL) v = nL + lscan[x - 1];                 // rows 1..nL start after s's row
    else if (x <= nL + nR + 1) v = nL + E + (x - 1 - nL);    // right rows: one edge each
    else v = nL + E + nR;                                    // row of t (empty) / end
    ro[x] = v;
  }
}

__global__ void k_bip_scatter(const int32_t* __restrict__ l, const int32_t* __restrict__ r, int64_t E, int64_t nL,
                              int64_t nR, const int* __restrict__ lscan, int* cursor, int32_t* col, int32_t* cap) {
  int64_t t = nL + nR + 1;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nL; i += stride) {
    col[i] = (int32_t)(1 + i); cap[i] = 1;                   // s -> l
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += stride) {
    int a = l[i], b = r[i];
    int64_t pos = nL + lscan[a] + atomicAdd(cursor + a, 1);
    col[pos] = (int32_t)(1 + nL + b); cap[pos] = 1;          // l -> r
  }
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nR; j += stride) {
    col[nL + E + j] = (int32_t)t; cap[nL + E + j] = 1;       // r -> t
  }
}

__global__ void k_bip_extract_bcsr(const int2* __restrict__ seg, const int2* __restrict__ arc, int64_t nL, int64_t nR,
                                   int32_t* match) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nR; j += (int64_t)gridDim.x * blockDim.x) {
    int x = (int)(1 + nL + j);
    int b = seg[x].x, e = seg[x].y;
    if (e <= b) continue;
    int2 last = ld_cg(arc + e - 1);                        // column t sorts last
    if (last.x != (int)(nL + nR + 1) || last.y != 0) continue;   // x -> t not saturated
    for (int p = b; p < e - 1; ++p) {
      int2 a = ld_cg(arc + p);                             // x -> l residual = flow on l -> x
      if (a.y >= 1) { match[a.x - 1] = (int32_t)j; break; }
    }
  }
}

__global__ void k_bip_extract_rcsr(const int* __restrict__ foff, const int2* __restrict__ farc,
                                   const int* __restrict__ roff, const int2* __restrict__ rarc,
                                   const int* __restrict__ bcf, int64_t nL, int64_t nR, int32_t* match) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nR; j += (int64_t)gridDim.x * blockDim.x) {
    int x = (int)(1 + nL + j);
    int fb = foff[x], fe = foff[x + 1];
    if (fe <= fb) continue;
    int2 a = ld_cg(farc + fb);                             // the single forward arc x -> t
    if (a.y != 0) continue;
    for (int q = roff[x]; q < roff[x + 1]; ++q) {           // l -> x forward arcs, sorted by l
      int2 rq = rarc[q];
      if (ld_cg(bcf + rq.y) >= 1) { match[rq.x - 1] = (int32_t)j; break; }
    }
  }
}

void bip_extract(const SolveParams& p, int64_t nL, int64_t nR, int32_t* match_of_left, int num_sms,
                 cudaStream_t st) {
  const int T = 256;
  cudaMemsetAsync(match_of_left, 0xff, sizeof(int32_t) * nL, st);
  unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nR + T - 1) / T, num_sms * 32));
  if (nR <= 0) return;
  if (p.layout == 0) { k_bip_extract_bcsr<<<g, T, 0, st>>>(p.seg, p.arc, nL, nR, match_of_left); note_launch(); }
  else { k_bip_extract_rcsr<<<g, T, 0, st>>>(p.off, p.arc, p.roff, p.rarc, p.bcf, nL, nR, match_of_left); note_launch(); }
}

// Validation + left-degree histogram (first offending edge lands in ctrl->bad_edge).
void bip_validate(int64_t nL, int64_t nR, int64_t E, const int32_t* l, const int32_t* r, int* deg, int* cursor,
                  Ctrl* ctrl, int num_sms, cudaStream_t st) {
  const int T = 256;
  cudaMemsetAsync(deg, 0, sizeof(int) * (nL + 1), st);
  cudaMemsetAsync(cursor, 0, sizeof(int) * (nL + 1), st);
  unsigned gE = (unsigned)std::max<int64_t>(1, std::min<int64_t>((E + T - 1) / T, num_sms * 32));
  if (E > 0) { k_bip_hist<<<gE, T, 0, st>>>(l, r, E, nL, nR, deg, ctrl); note_launch(); }
}

// Network CSR (after a successful validation).
void bip_build(int64_t nL, int64_t nR, int64_t E, const int32_t* l, const int32_t* r, int64_t* ro, int32_t* col,
               int32_t* cap, int* deg, int* cursor, int* scan_part, int num_sms, cudaStream_t st) {
  const int T = 256;
  exclusive_scan(deg, nL, scan_part, st);   // deg[nL] = E
  int64_t n = nL + nR + 2;
  unsigned gN = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 1 + T - 1) / T, num_sms * 32));
  { k_bip_rows<<<gN, T, 0, st>>>(deg, nL, nR, E, ro); note_launch(); }
  int64_t mx = std::max(std::max(nL, nR), E);
  unsigned gS = (unsigned)std::max<int64_t>(1, std::min<int64_t>((mx + T - 1) / T, num_sms * 32));
  { k_bip_scatter<<<gS, T, 0, st>>>(l, r, E, nL, nR, deg, cursor, col, cap); note_launch(); }
}

}  // namespace wbpr
