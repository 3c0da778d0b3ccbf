/*
 * synth/gen.c — seeded synthetic input generators for the WBPR hot path.
 *
 * This module holds NO max-flow arithmetic.  It only draws graphs with the
 * shapes of the paper's workloads (§4.1: power-law
 * SNAP/DIMACS graphs, 20 BFS-chosen s/t pairs behind a super-source and a
 * super-sink, KONECT bipartite graphs) and of BASELINE.json configs C1-C5
 * (recipe in DESIGN.md "Input recipe").  Both the oracle (oracle/) and the
 * CUDA path consume the same arrays produced here; neither imports the other.
 *
 * Every random draw comes from a counter-based splitmix64 stream
 * (value = mix(seed, stream, counter)), so results are independent of
 * thread count and call order.
 *
 * Output format everywhere: an edge list (src i32[m], dst i32[m], cap i32[m])
 * which the Python side turns into CSR; generators that need an intermediate
 * edge count return it through *m_out and write into caller buffers sized by
 * a preceding "_count" call or a caller-provided upper bound.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Threads of the OpenMP regions (the draws are counter-based: results never depend on it).
 * torchrun exports OMP_NUM_THREADS=1 to every rank; the bench sets its share of the cores. */
void synth_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* counter-based draw: stream id separates purposes (edges, caps, perm, ...) */
static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return mix64(mix64(seed * 0xD1B54A32D192ED03ull + stream) ^ (ctr * 0x9E3779B97F4A7C15ull));
}
uint64_t synth_draw(uint64_t seed, uint64_t stream, uint64_t ctr) { return draw(seed, stream, ctr); }

enum { ST_EDGE = 1, ST_CAP = 2, ST_PERM = 3, ST_START = 4, ST_PICK = 5, ST_SHUF = 6 };

static inline int32_t cap_1_100(uint64_t seed, uint64_t i) {
  return (int32_t)(1 + draw(seed, ST_CAP, i) % 100);
}

/* ---------- LSD radix sort of uint64 keys (for dedupe) ---------- */
static void radix_sort_u64(uint64_t* a, int64_t n, int key_bits) {
  if (n <= 1) return;
  uint64_t* tmp = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  int passes = (key_bits + 15) / 16;
  for (int ps = 0; ps < passes; ++ps) {
    int sh = 16 * ps;
    int64_t* cnt = (int64_t*)calloc(65536, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[(a[i] >> sh) & 0xFFFF]++;
    int64_t sum = 0;
    for (int b = 0; b < 65536; ++b) { int64_t c = cnt[b]; cnt[b] = sum; sum += c; }
    for (int64_t i = 0; i < n; ++i) tmp[cnt[(a[i] >> sh) & 0xFFFF]++] = a[i];
    memcpy(a, tmp, (size_t)n * sizeof(uint64_t));
    free(cnt);
  }
  free(tmp);
}

static int bits_for(int64_t n) { int b = 1; while (((int64_t)1 << b) < n) ++b; return b; }

/* ---------- C1: uniform random distinct ordered pairs u != v ---------- */
/* Rejection sampling with an open-addressing hash set; pairs kept in draw order. */
int64_t synth_random_pairs(int32_t n, int64_t m, uint64_t seed,
                           int32_t* src, int32_t* dst, int32_t* cap) {
  if (n < 2) return 0;
  int64_t maxm = (int64_t)n * (n - 1);
  if (m > maxm) m = maxm;
  int64_t hsz = 1; while (hsz < 4 * m + 16) hsz <<= 1;
  uint64_t* hs = (uint64_t*)malloc((size_t)hsz * sizeof(uint64_t));
  for (int64_t i = 0; i < hsz; ++i) hs[i] = ~0ull;
  int64_t k = 0; uint64_t ctr = 0;
  while (k < m) {
    uint64_t x = draw(seed, ST_EDGE, ctr++);
    int32_t u = (int32_t)((x & 0xFFFFFFFFull) % (uint64_t)n);
    int32_t v = (int32_t)((x >> 32) % (uint64_t)n);
    if (u == v) continue;
    uint64_t key = ((uint64_t)u << 32) | (uint32_t)v;
    uint64_t h = mix64(key) & (uint64_t)(hsz - 1);
    int dup = 0;
    while (hs[h] != ~0ull) { if (hs[h] == key) { dup = 1; break; } h = (h + 1) & (uint64_t)(hsz - 1); }
    if (dup) continue;
    hs[h] = key;
    src[k] = u; dst[k] = v; cap[k] = cap_1_100(seed, (uint64_t)k);
    ++k;
  }
  free(hs);
  return k;
}

/* ---------- C2: W x H 4-neighbour grid with border super-terminals ---------- */
/* id = y*W + x; S = W*H (-> every x=0 vertex), T = W*H+1 (<- every x=W-1 vertex).
 * cap_mode 0: unit caps on grid arcs; 1: U[1,100] i.i.d. per directed arc.
 * Super-arc caps = incident-capacity sums (S:382 reading; never binding).
 * Edge count = 2*(W-1)*H + 2*W*(H-1) + 2*H. Returns the count. */
int64_t synth_grid_count(int32_t W, int32_t H) {
  return 2ll * (W - 1) * H + 2ll * W * (H - 1) + 2ll * H;
}
int64_t synth_grid(int32_t W, int32_t H, int32_t cap_mode, uint64_t seed,
                   int32_t* src, int32_t* dst, int32_t* cap) {
  int64_t k = 0;
  int32_t N = W * H, S = N, T = N + 1;
  /* grid arcs in (y, x, dir) order; directed arc index k drives the cap stream */
  static const int dx[4] = {1, -1, 0, 0}, dy[4] = {0, 0, 1, -1};
  for (int32_t y = 0; y < H; ++y)
    for (int32_t x = 0; x < W; ++x)
      for (int d = 0; d < 4; ++d) {
        int32_t X = x + dx[d], Y = y + dy[d];
        if (X < 0 || X >= W || Y < 0 || Y >= H) continue;
        src[k] = y * W + x; dst[k] = Y * W + X;
        cap[k] = cap_mode ? cap_1_100(seed, (uint64_t)k) : 1;
        ++k;
      }
  int64_t kg = k;
  /* out-cap sums for x=0 vertices, in-cap sums for x=W-1 vertices */
  int64_t* outc = (int64_t*)calloc((size_t)N, sizeof(int64_t));
  int64_t* inc = (int64_t*)calloc((size_t)N, sizeof(int64_t));
  for (int64_t i = 0; i < kg; ++i) { outc[src[i]] += cap[i]; inc[dst[i]] += cap[i]; }
  for (int32_t y = 0; y < H; ++y) {
    int32_t v = y * W;
    src[k] = S; dst[k] = v; cap[k] = (int32_t)outc[v]; ++k;
  }
  for (int32_t y = 0; y < H; ++y) {
    int32_t v = y * W + (W - 1);
    src[k] = v; dst[k] = T; cap[k] = (int32_t)inc[v]; ++k;
  }
  free(outc); free(inc);
  return k;
}

/* ---------- R-MAT (Graph500 A,B,C,D = 0.57,0.19,0.19,0.05) ---------- */
/* Generates 2^scale * edgefactor raw edges, drops self-loops, collapses
 * duplicates, applies a Fisher-Yates vertex permutation, then draws caps
 * U[1,100] in sorted-unique order.  src/dst must hold 2^scale*edgefactor.
 * Returns the unique edge count; edges come out sorted by (perm src, perm dst)
 * only up to the permutation — i.e. sorted by original ids. */
int64_t synth_rmat(int32_t scale, int32_t edgefactor, uint64_t seed,
                   int32_t* src, int32_t* dst, int32_t* cap) {
  int64_t n = (int64_t)1 << scale;
  int64_t M = n * edgefactor;
  uint64_t* keys = (uint64_t*)malloc((size_t)M * sizeof(uint64_t));
  /* thresholds on a 32-bit uniform */
  const uint64_t tA = (uint64_t)(0.57 * 4294967296.0);
  const uint64_t tB = (uint64_t)(0.76 * 4294967296.0);
  const uint64_t tC = (uint64_t)(0.95 * 4294967296.0);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < M; ++e) {
    uint64_t u = 0, v = 0;
    for (int lvl = 0; lvl < scale; ++lvl) {
      uint64_t r = draw(seed, ST_EDGE, (uint64_t)e * 64 + (uint64_t)lvl) & 0xFFFFFFFFull;
      u <<= 1; v <<= 1;
      if (r < tA) { }
      else if (r < tB) { v |= 1; }
      else if (r < tC) { u |= 1; }
      else { u |= 1; v |= 1; }
    }
    keys[e] = (u << 32) | v;
  }
  /* permutation */
  int32_t* perm = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)(draw(seed, ST_PERM, (uint64_t)i) % (uint64_t)(i + 1));
    int32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
  }
  /* apply permutation before dedupe so output is sorted by permuted ids */
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < M; ++e) {
    uint64_t u = keys[e] >> 32, v = keys[e] & 0xFFFFFFFFull;
    keys[e] = ((uint64_t)perm[u] << 32) | (uint64_t)perm[v];
  }
  free(perm);
  radix_sort_u64(keys, M, 32 + bits_for(n));
  int64_t k = 0;
  uint64_t prev = ~0ull;
  for (int64_t e = 0; e < M; ++e) {
    uint64_t key = keys[e];
    if (key == prev) continue;
    prev = key;
    int32_t u = (int32_t)(key >> 32), v = (int32_t)(key & 0xFFFFFFFFull);
    if (u == v) continue;
    src[k] = u; dst[k] = v; ++k;
  }
  free(keys);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) cap[i] = cap_1_100(seed, (uint64_t)i);
  return k;
}

/* ---------- bipartite: nE uniform (l, r) draws, duplicates collapsed ---------- */
int64_t synth_bipartite(int32_t nL, int32_t nR, int64_t nE, uint64_t seed,
                        int32_t* l_out, int32_t* r_out) {
  uint64_t* keys = (uint64_t*)malloc((size_t)nE * sizeof(uint64_t));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < nE; ++e) {
    uint64_t x = draw(seed, ST_EDGE, (uint64_t)e);
    uint64_t l = (x & 0xFFFFFFFFull) % (uint64_t)nL;
    uint64_t r = (x >> 32) % (uint64_t)nR;
    keys[e] = (l << 32) | r;
  }
  radix_sort_u64(keys, nE, 32 + bits_for(nL));
  int64_t k = 0; uint64_t prev = ~0ull;
  for (int64_t e = 0; e < nE; ++e) {
    if (keys[e] == prev) continue;
    prev = keys[e];
    l_out[k] = (int32_t)(keys[e] >> 32); r_out[k] = (int32_t)(keys[e] & 0xFFFFFFFFull); ++k;
  }
  free(keys);
  return k;
}

/* ---------- terminal selection helpers over a CSR (row_off i64, col i32) ---------- */
static int32_t uf_find(int32_t* p, int32_t x) {
  while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
  return x;
}

/* forward BFS from `start`; returns depth (max level) and writes the list of
 * deepest-level vertices count into *ndeep and their ids into deep[] (cap n). */
static int32_t bfs_depth(int32_t n, const int64_t* ro, const int32_t* col, int32_t start,
                         int32_t* lvl, int32_t* queue, int32_t* deep, int64_t* ndeep) {
  for (int32_t i = 0; i < n; ++i) lvl[i] = -1;
  int64_t qh = 0, qt = 0;
  queue[qt++] = start; lvl[start] = 0;
  int32_t maxd = 0;
  while (qh < qt) {
    int32_t u = queue[qh++];
    for (int64_t p = ro[u]; p < ro[u + 1]; ++p) {
      int32_t v = col[p];
      if (lvl[v] < 0) { lvl[v] = lvl[u] + 1; if (lvl[v] > maxd) maxd = lvl[v]; queue[qt++] = v; }
    }
  }
  int64_t nd = 0;
  for (int64_t i = 0; i < qt; ++i) if (lvl[queue[i]] == maxd) deep[nd++] = queue[i];
  *ndeep = nd;
  return maxd;
}

/* Paper rule (reading in DESIGN.md): draw `nstarts` seeded starts with
 * out-degree > 0 in the largest weakly connected component; forward BFS from each;
 * target = a deepest-level vertex chosen by a seeded draw; keep pairs whose depth
 * is in the top quartile; greedily take `k` pairs ordered by (-depth, start id)
 * with all 2k endpoints distinct, relaxing to lower depths if needed.
 * Writes sources[k], sinks[k]; returns the number of pairs found. */
int32_t synth_select_pairs(int32_t n, const int64_t* ro, const int32_t* col, int32_t k,
                           int32_t nstarts, uint64_t seed, int32_t* sources, int32_t* sinks) {
  int64_t m = ro[n];
  int32_t* par = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  for (int32_t i = 0; i < n; ++i) par[i] = i;
  for (int32_t u = 0; u < n; ++u)
    for (int64_t p = ro[u]; p < ro[u + 1]; ++p) {
      int32_t a = uf_find(par, u), b = uf_find(par, col[p]);
      if (a != b) { if (a < b) par[b] = a; else par[a] = b; }
    }
  int32_t* csize = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  int32_t best = 0;
  for (int32_t i = 0; i < n; ++i) { int32_t r = uf_find(par, i); csize[r]++; }
  for (int32_t i = 0; i < n; ++i) if (csize[i] > csize[best]) best = i;
  (void)m;
  /* draw starts */
  int32_t* starts = (int32_t*)malloc((size_t)nstarts * sizeof(int32_t));
  int32_t ns = 0; uint64_t ctr = 0;
  uint64_t limit = (uint64_t)nstarts * 1000 + 100000;
  while (ns < nstarts && ctr < limit) {
    int32_t v = (int32_t)(draw(seed, ST_START, ctr++) % (uint64_t)n);
    if (ro[v + 1] == ro[v] || uf_find(par, v) != best) continue;
    int dup = 0;
    for (int32_t j = 0; j < ns; ++j) if (starts[j] == v) { dup = 1; break; }
    if (!dup) starts[ns++] = v;
  }
  int32_t* depth = (int32_t*)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int32_t));
  int32_t* target = (int32_t*)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int32_t));
#pragma omp parallel
  {
    int32_t* lvl = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* q = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    int32_t* deep = (int32_t*)malloc((size_t)n * sizeof(int32_t));
#pragma omp for schedule(dynamic, 1)
    for (int32_t i = 0; i < ns; ++i) {
      int64_t nd = 0;
      depth[i] = bfs_depth(n, ro, col, starts[i], lvl, q, deep, &nd);
      target[i] = nd > 0 ? deep[draw(seed, ST_PICK, (uint64_t)starts[i]) % (uint64_t)nd] : starts[i];
    }
    free(lvl); free(q); free(deep);
  }
  /* order by (-depth, start id) */
  int32_t* ord = (int32_t*)malloc((size_t)(ns > 0 ? ns : 1) * sizeof(int32_t));
  for (int32_t i = 0; i < ns; ++i) ord[i] = i;
  for (int32_t i = 1; i < ns; ++i) {           /* insertion sort: ns is small */
    int32_t x = ord[i], j = i - 1;
    while (j >= 0 && (depth[ord[j]] < depth[x] ||
                      (depth[ord[j]] == depth[x] && starts[ord[j]] > starts[x]))) {
      ord[j + 1] = ord[j]; --j;
    }
    ord[j + 1] = x;
  }
  /* 75th percentile threshold of depths */
  int32_t thr = ns > 0 ? depth[ord[(ns - 1) / 4]] : 0;
  unsigned char* used = (unsigned char*)calloc((size_t)n, 1);
  int32_t got = 0;
  for (int pass = 0; pass < 2 && got < k; ++pass)
    for (int32_t ii = 0; ii < ns && got < k; ++ii) {
      int32_t i = ord[ii];
      if (pass == 0 && depth[i] < thr) continue;
      if (pass == 1 && depth[i] >= thr) continue;
      int32_t a = starts[i], b = target[i];
      if (a == b || used[a] || used[b]) continue;
      used[a] = used[b] = 1;
      sources[got] = a; sinks[got] = b; ++got;
    }
  free(used); free(ord); free(depth); free(target); free(starts); free(csize); free(par);
  return got;
}

/* hub20 stress rule: sources = top-k out-degree vertices (ties: smaller id);
 * sinks = top-k in-degree vertices excluding the sources. */
int32_t synth_select_hubs(int32_t n, const int64_t* ro, const int32_t* col, int32_t k,
                          int32_t* sources, int32_t* sinks) {
  int64_t* indeg = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  for (int64_t p = 0; p < ro[n]; ++p) indeg[col[p]]++;
  unsigned char* used = (unsigned char*)calloc((size_t)n, 1);
  for (int32_t j = 0; j < k; ++j) {
    int32_t b = -1; int64_t bd = -1;
    for (int32_t v = 0; v < n; ++v) {
      int64_t d = ro[v + 1] - ro[v];
      if (!used[v] && d > bd) { bd = d; b = v; }
    }
    used[b] = 1; sources[j] = b;
  }
  for (int32_t j = 0; j < k; ++j) {
    int32_t b = -1; int64_t bd = -1;
    for (int32_t v = 0; v < n; ++v)
      if (!used[v] && indeg[v] > bd) { bd = indeg[v]; b = v; }
    used[b] = 1; sinks[j] = b;
  }
  free(indeg); free(used);
  return k;
}

/* Seeded Fisher-Yates shuffle of positions [lo, hi) of three parallel arrays:
 * used by tests to present CSR rows in arbitrary order (the boundary accepts any
 * order within a row). */
void synth_shuffle_rows(int64_t n, const int64_t* ro, int32_t* col, int32_t* cap, uint64_t seed) {
  for (int64_t u = 0; u < n; ++u) {
    int64_t lo = ro[u], hi = ro[u + 1];
    for (int64_t i = hi - 1; i > lo; --i) {
      int64_t j = lo + (int64_t)(draw(seed, ST_SHUF, (uint64_t)i) % (uint64_t)(i - lo + 1));
      int32_t t = col[i]; col[i] = col[j]; col[j] = t;
      t = cap[i]; cap[i] = cap[j]; cap[j] = t;
    }
  }
}

/* ---------- DIMACS-shaped generators (NEXT #4; structure decoded in SURVEY E1) ---------- */
/* Washington random level graph: L levels of W vertices, each vertex -> `deg` random
 * vertices of the next level, caps U[1, capmax]; S = L*W -> level 0, level L-1 -> T = L*W+1
 * (super caps = incident sums).  Edge count = (L-1)*W*deg + 2*W. */
int64_t synth_rlg_count(int32_t L, int32_t W, int32_t deg) { return (int64_t)(L - 1) * W * deg + 2ll * W; }
int64_t synth_rlg(int32_t L, int32_t W, int32_t deg, int32_t capmax, uint64_t seed,
                  int32_t* src, int32_t* dst, int32_t* cap) {
  int64_t k = 0;
  int32_t N = L * W;
  for (int32_t l = 0; l + 1 < L; ++l)
    for (int32_t x = 0; x < W; ++x)
      for (int32_t d = 0; d < deg; ++d) {
        uint64_t r = draw(seed, ST_EDGE, (uint64_t)k);
        src[k] = l * W + x;
        dst[k] = (l + 1) * W + (int32_t)(r % (uint64_t)W);
        cap[k] = (int32_t)(1 + draw(seed, ST_CAP, (uint64_t)k) % (uint64_t)capmax);
        ++k;
      }
  int64_t kin = k;
  int64_t* outc = (int64_t*)calloc((size_t)N, sizeof(int64_t));
  int64_t* inc = (int64_t*)calloc((size_t)N, sizeof(int64_t));
  for (int64_t i = 0; i < kin; ++i) { outc[src[i]] += cap[i]; inc[dst[i]] += cap[i]; }
  for (int32_t x = 0; x < W; ++x) { src[k] = N; dst[k] = x; cap[k] = (int32_t)(outc[x] ? outc[x] : 1); ++k; }
  for (int32_t x = 0; x < W; ++x) {
    int32_t v = (L - 1) * W + x;
    src[k] = v; dst[k] = N + 1; cap[k] = (int32_t)(inc[v] ? inc[v] : 1); ++k;
  }
  free(outc); free(inc);
  return k;
}

/* Genrmf (Goldfarb-Grigoriadis): b frames of a x a grids; in-frame 4-neighbour arcs (both
 * directions) with cap c2*a*a; frame i -> frame i+1 through a seeded permutation with caps
 * U[c1, c2]; s = vertex 0 of frame 0, t = last vertex of frame b-1.
 * Edge count = 4*a*(a-1)*b + a*a*(b-1). */
int64_t synth_genrmf_count(int32_t a, int32_t b) { return 4ll * a * (a - 1) * b + (int64_t)a * a * (b - 1); }
int64_t synth_genrmf(int32_t a, int32_t b, int32_t c1, int32_t c2, uint64_t seed,
                     int32_t* src, int32_t* dst, int32_t* cap) {
  int64_t k = 0;
  int32_t A = a * a;
  int32_t big = c2 * a * a;
  static const int dx[4] = {1, -1, 0, 0}, dy[4] = {0, 0, 1, -1};
  for (int32_t f = 0; f < b; ++f)
    for (int32_t y = 0; y < a; ++y)
      for (int32_t x = 0; x < a; ++x)
        for (int d = 0; d < 4; ++d) {
          int32_t X = x + dx[d], Y = y + dy[d];
          if (X < 0 || X >= a || Y < 0 || Y >= a) continue;
          src[k] = f * A + y * a + x; dst[k] = f * A + Y * a + X; cap[k] = big; ++k;
        }
  int32_t* perm = (int32_t*)malloc((size_t)A * sizeof(int32_t));
  for (int32_t f = 0; f + 1 < b; ++f) {
    for (int32_t i = 0; i < A; ++i) perm[i] = i;
    for (int32_t i = A - 1; i > 0; --i) {
      int32_t j = (int32_t)(draw(seed, ST_PERM, (uint64_t)f * A + i) % (uint64_t)(i + 1));
      int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    for (int32_t i = 0; i < A; ++i) {
      src[k] = f * A + i; dst[k] = (f + 1) * A + perm[i];
      cap[k] = c1 + (int32_t)(draw(seed, ST_CAP, (uint64_t)k) % (uint64_t)(c2 - c1 + 1));
      ++k;
    }
  }
  free(perm);
  return k;
}
