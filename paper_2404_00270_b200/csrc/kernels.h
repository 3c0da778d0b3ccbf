// kernels.h — host-callable launch wrappers of the WBPR kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.h"

namespace wbpr {

// number of kernels this library launched (process-wide; bench's gpu_launches)
void note_launch();
long long launch_count();

void exclusive_scan(int* a, int64_t N, int* part, cudaStream_t st);

void segmented_sort(uint64_t* keys, uint64_t* tmp, const int* off, int nseg, int maxlen, Ctrl* ctrl,
                    int2* items, int2* items_med, int* big, int num_sms, cudaStream_t st);
void segmented_sort_filtered(uint64_t* keys, uint64_t* tmp, const int* off, int nseg, int maxlen,
                             const uint8_t* need, Ctrl* ctrl, int2* items, int2* items_med, int* big, int num_sms,
                             cudaStream_t st);
void segmented_sort32(uint32_t* keys, uint32_t* tmp, const int* off, int nseg, int maxlen, Ctrl* ctrl, int2* items,
                      int2* items_med, int* big, int num_sms, cudaStream_t st);
void k_ro_to_i32_ext(const int64_t* ro, int64_t n, int* out, int num_sms, cudaStream_t st);

struct BuildArgs {
  int64_t n, m, H;
  int32_t layout;
  int num_sms;
  const int64_t* ro;
  const int32_t* col;
  const int32_t* cap;
  Ctrl* ctrl;
  int* deg;
  int* cursor;
  int* soff;
  int* off;
  int* roff;
  int* scan_part;
  int* q0;
  uint64_t* keys;  // region A
  uint64_t* tmp;   // region B
  int2* arc;       // region C
  int* mate;       // region B (after the merge)
  int* cap0;       // region B + bcap0
  int2* rarc;      // region C + 8m (RCSR)
  int* bcf;        // region B (RCSR)
  int maxlen;
  const int64_t* vbase;  // batch instance ranges (device), k entries + 1
  int k;
  int* src;              // BCSR build: owner row of every input edge (region A + 8m; dead after the in-list resolve)
  int* ine;              // BCSR build: input-edge index of every in-list entry (region A + 4m)
  int* inslot;           // BCSR build: merged slot of every in-list entry (region A + 8m; src is dead by then)
  int* outslot;          // BCSR build: per out-half-arc (sorted row position), its merged slot (region D)
  int2* seg;             // BCSR: {begin, end} of every vertex segment
  int any_unsorted;      // BCSR: some input row needs sorting (host copy of the validation flag)
  int* rsoff;            // BCSR merge build: in-list offsets
  uint8_t* need;         // BCSR merge build: per-row "not sorted" flags
  int* q1;
  int2* mtasks;          // BCSR merge build: chunk tasks of hub vertices
  int* mheads;
  int maxlen_out;
};

void build_validate(const BuildArgs& a, cudaStream_t st);
void build_bcsr_mate(const BuildArgs& a, cudaStream_t st);
void build_bcsr_merge(const BuildArgs& a, cudaStream_t st);
void build_rcsr_forward(const BuildArgs& a, cudaStream_t st);
void build_rcsr_reverse_counts(const BuildArgs& a, int Mf, cudaStream_t st);
void build_rcsr_reverse(const BuildArgs& a, int Mf, int maxlen, cudaStream_t st);

// solve.cu
int solve_max_blocks_per_sm(int layout, int threads);
cudaError_t launch_solve(const SolveParams& p, int blocks, int threads, cudaStream_t st);
cudaError_t barrier_probe(int blocks, int iters, double* ns_per_barrier, cudaStream_t st);
#ifndef WBPR_SOLVE_THREADS
#define WBPR_SOLVE_THREADS 512
#endif
#ifndef WBPR_SOLVE_MINB_DEFAULT
#define WBPR_SOLVE_MINB_DEFAULT 2
#endif
constexpr int kSolveThreads = WBPR_SOLVE_THREADS;
constexpr int kSolveMinBlocks = WBPR_SOLVE_MINB_DEFAULT;   // default register budget of k_solve (see solve.cu)

// extract.cu
void extract_results(const SolveParams& p, const int64_t* ro, const int32_t* col, const int32_t* cap,
                     int64_t m, uint32_t* bitmap, const int64_t* vbase, int k, long long* inst_flow,
                     long long* inst_cut, int num_sms, cudaStream_t st);

// bipartite.cu
void bip_validate(int64_t nL, int64_t nR, int64_t E, const int32_t* l, const int32_t* r, int* deg, int* cursor,
                  Ctrl* ctrl, int num_sms, cudaStream_t st);
void bip_build(int64_t nL, int64_t nR, int64_t E, const int32_t* l, const int32_t* r, int64_t* ro, int32_t* col,
               int32_t* cap, int* deg, int* cursor, int* scan_part, int num_sms, cudaStream_t st);
void bip_extract(const SolveParams& p, int64_t nL, int64_t nR, int32_t* match_of_left, int num_sms,
                 cudaStream_t st);

// tiny.cu: the whole path in one launch of one CTA (tiny single instances)
bool tiny_fits(int64_t n, int64_t m);
cudaError_t launch_tiny(const TinyArgs& a, cudaStream_t st);

}  // namespace wbpr
