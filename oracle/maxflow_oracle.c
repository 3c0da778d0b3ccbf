/*
 * oracle/maxflow_oracle.c — CPU ORACLE for the WBPR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2404_00270_b200/csrc) and neither side imports the other.
 *
 * What it computes (§2.1):
 *   F*   = max s-t flow value = min cut capacity (textbook duality),
 *   S*   = V \ {v : v reaches t in the residual graph G_f} (canonical cut side),
 *   cut  = sum of c(u,v) over input edges with u in S*, v not in S*,
 *   f[i] = a valid flow on every input edge (after phase 2).
 *
 * Algorithm: the generic push-relabel method as the paper states it
 * (§2.2): preflow ("pushes flow from the source to all
 * its neighbor vertices as much as possible"), push iff h(u) = h(v)+1 (P:160,
 * the EXACT rule, not the GPU's relaxed one), relabel h(u) <- min h(v) + 1 over
 * residual arcs, deactivation at h >= |V|, run in FIFO order with
 * a current-arc pointer, plus
 *   - the gap heuristic (north_star; not in the paper): when no vertex below
 *     |V| has height g any more, every vertex with g < h < |V| is lifted to |V|;
 *   - optional global relabel: exact reverse BFS from the
 *     sink in G_f, unreached vertices get |V|.
 * Phase 2 returns stranded excess to s by running the
 * same discharge loop with s as the target, giving a true flow.
 *
 * Representation: input edge i = (u,v,c), u != v, becomes
 * arc 2i = u->v with residual capacity c and arc 2i+1 = v->u with residual
 * capacity 0; arc a's reverse is a^1.  No merging of parallel or antiparallel
 * edges (deliberately different from the CUDA path's BCSR merge).  Self-loops
 * carry no flow and are left out of the adjacency lists.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n, m;
  int64_t s, t;
  /* arcs */
  int32_t* head;      /* head[a] : vertex the arc points to            */
  int64_t* rc;        /* rc[a]   : residual capacity c_f of arc a      */
  /* adjacency: arcs leaving v are adj[first[v] .. first[v+1]) */
  int64_t* first;
  int64_t* adj;
  /* push-relabel state */
  int64_t* e;         /* excess e(v)  */
  int64_t* h;         /* height h(v)  */
  int64_t* cur;       /* current-arc pointer          */
  int64_t* cnt;       /* cnt[k] = #vertices with h == k, k < n (for the gap test) */
  int64_t* queue;     /* FIFO ring of active vertices */
  uint8_t* inq;
  int64_t qh, qt, qn;
  int64_t* bfsq;
  /* stats */
  int64_t pushes, relabels, grs, gaps, relabels_since_gr;
} pr_t;

static void q_push(pr_t* g, int64_t v) {
  if (g->inq[v]) return;
  g->inq[v] = 1;
  g->queue[g->qt] = v;
  g->qt = (g->qt + 1) % (g->n + 1);
  g->qn++;
}
static int64_t q_pop(pr_t* g) {
  int64_t v = g->queue[g->qh];
  g->qh = (g->qh + 1) % (g->n + 1);
  g->qn--;
  g->inq[v] = 0;
  return v;
}

/* Reverse BFS from `target` in G_f: level(target) = 0, and u gets level k+1 if
 * an arc u->w has c_f > 0 and level(w) = k.  The vertex `blocked` is never
 * expanded.  Unreached vertices get n.  ("backward breadth-first search
 * (BFS) from the sink"; unreached -> |V| is SURVEY §8(c) reading #7.) */
static void reverse_bfs(pr_t* g, int64_t target, int64_t blocked, int64_t* level) {
  int64_t n = g->n;
  for (int64_t v = 0; v < n; ++v) level[v] = n;
  int64_t qh = 0, qt = 0;
  level[target] = 0;
  g->bfsq[qt++] = target;
  while (qh < qt) {
    int64_t w = g->bfsq[qh++];
    for (int64_t k = g->first[w]; k < g->first[w + 1]; ++k) {
      int64_t a = g->adj[k];          /* a = w -> u */
      int64_t u = g->head[a];
      /* residual arc u -> w is the reverse arc a^1 */
      if (g->rc[a ^ 1] > 0 && level[u] == n && u != blocked && u != target) {
        level[u] = level[w] + 1;
        g->bfsq[qt++] = u;
      }
    }
  }
}

/* Global relabel toward `target`; rebuilds cnt[] and the FIFO queue. */
static void global_relabel(pr_t* g, int64_t target, int64_t blocked) {
  int64_t n = g->n;
  reverse_bfs(g, target, blocked, g->h);
  g->h[blocked] = n;
  for (int64_t k = 0; k < n; ++k) g->cnt[k] = 0;
  for (int64_t v = 0; v < n; ++v) if (g->h[v] < n) g->cnt[g->h[v]]++;
  g->qh = g->qt = g->qn = 0;
  for (int64_t v = 0; v < n; ++v) g->inq[v] = 0;
  for (int64_t v = 0; v < n; ++v) {
    g->cur[v] = g->first[v];
    if (v != target && v != blocked && g->e[v] > 0 && g->h[v] < n) q_push(g, v);
  }
  g->grs++;
  g->relabels_since_gr = 0;
}

/* Relabel: h(u) <- 1 + min{ h(v) : (u,v) in E_f }, capped at n
 * (a vertex at height >= |V| is deactivated).  Then the gap test. */
static void relabel(pr_t* g, int64_t u, int use_gap) {
  int64_t n = g->n;
  int64_t old = g->h[u];
  int64_t mn = n;                       /* no residual arc -> deactivate */
  for (int64_t k = g->first[u]; k < g->first[u + 1]; ++k) {
    int64_t a = g->adj[k];
    if (g->rc[a] > 0 && g->h[g->head[a]] < mn) mn = g->h[g->head[a]];
  }
  int64_t nh = mn + 1 < n ? mn + 1 : n;
  g->h[u] = nh;
  g->cur[u] = g->first[u];
  g->relabels++;
  g->relabels_since_gr++;
  if (old < n) g->cnt[old]--;
  if (nh < n) g->cnt[nh]++;
  /* gap heuristic: no vertex left at height `old` -> nothing above it reaches the target */
  if (use_gap && old < n && g->cnt[old] == 0) {
    int lifted = 0;
    for (int64_t v = 0; v < n; ++v)
      if (g->h[v] > old && g->h[v] < n) { g->cnt[g->h[v]]--; g->h[v] = n; lifted = 1; }
    if (lifted) g->gaps++;
  }
}

/* Push (P:95-101 with the exact admissibility of P:160): delta = min(e(u), c_f(a)). */
static void push(pr_t* g, int64_t u, int64_t a, int64_t target, int64_t blocked) {
  int64_t v = g->head[a];
  int64_t d = g->e[u] < g->rc[a] ? g->e[u] : g->rc[a];
  g->rc[a] -= d;
  g->rc[a ^ 1] += d;
  g->e[u] -= d;
  g->e[v] += d;
  g->pushes++;
  if (v != target && v != blocked && g->h[v] < g->n) q_push(g, v);
}

/* FIFO discharge loop toward `target`; `blocked` is the other terminal. */
static void run_fifo(pr_t* g, int64_t target, int64_t blocked, int use_gr, int use_gap) {
  int64_t n = g->n;
  while (g->qn > 0) {
    int64_t u = q_pop(g);
    if (u == target || u == blocked) continue;
    while (g->e[u] > 0 && g->h[u] < n) {
      if (g->cur[u] == g->first[u + 1]) {
        relabel(g, u, use_gap);
        continue;
      }
      int64_t a = g->adj[g->cur[u]];
      if (g->rc[a] > 0 && g->h[u] == g->h[g->head[a]] + 1) push(g, u, a, target, blocked);
      else g->cur[u]++;
    }
    if (use_gr && g->relabels_since_gr >= n) global_relabel(g, target, blocked);
  }
}

/*
 * oracle_maxflow — returns 0 on success, -1 on invalid input, -2 on allocation failure.
 *   in_S (n bytes, may be NULL):   1 iff v is in S* (cannot reach t in G_f).
 *   edge_flow (m, may be NULL):    per-input-edge flow after phase 2 (strict flow).
 *   stats (6, may be NULL):        pushes, relabels, global relabels, gaps (phase 1),
 *                                  pushes (phase 2), relabels (phase 2).
 */
int oracle_maxflow(int64_t n, int64_t m, const int64_t* row_off, const int32_t* col, const int32_t* cap,
                   int64_t s, int64_t t, int32_t use_gr, int32_t use_gap, int32_t phase2,
                   int64_t* flow_out, int64_t* cutcap_out, uint8_t* in_S, int64_t* edge_flow,
                   int64_t* stats) {
  if (n < 2 || s < 0 || t < 0 || s >= n || t >= n || s == t || m < 0) return -1;
  for (int64_t u = 0; u < n; ++u)
    if (row_off[u] > row_off[u + 1]) return -1;
  if (row_off[0] != 0 || row_off[n] != m) return -1;
  for (int64_t i = 0; i < m; ++i)
    if (col[i] < 0 || col[i] >= n || cap[i] < 0) return -1;

  pr_t G; memset(&G, 0, sizeof(G));
  pr_t* g = &G;
  g->n = n; g->m = m; g->s = s; g->t = t;
  g->head = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
  g->rc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  g->first = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
  g->adj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  g->e = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  g->h = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  g->cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  g->cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  g->queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  g->inq = (uint8_t*)calloc((size_t)n, 1);
  g->bfsq = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* tail = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  if (!g->head || !g->rc || !g->first || !g->adj || !g->e || !g->h || !g->cur || !g->cnt ||
      !g->queue || !g->inq || !g->bfsq || !tail) return -2;

  /* ingest: arc 2i = u->v (cap c), arc 2i+1 = v->u (cap 0) */
  for (int64_t u = 0; u < n; ++u)
    for (int64_t i = row_off[u]; i < row_off[u + 1]; ++i) {
      int64_t v = col[i];
      g->head[2 * i] = (int32_t)v;     tail[2 * i] = u;     g->rc[2 * i] = cap[i];
      g->head[2 * i + 1] = (int32_t)u; tail[2 * i + 1] = v; g->rc[2 * i + 1] = 0;
      if (u != v) { g->first[u + 1]++; g->first[v + 1]++; }
    }
  for (int64_t v = 0; v < n; ++v) g->first[v + 1] += g->first[v];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t v = 0; v < n; ++v) fill[v] = g->first[v];
    for (int64_t a = 0; a < 2 * m; ++a) {
      if (g->head[a] == tail[a]) continue;     /* self-loop: no residual arcs */
      g->adj[fill[tail[a]]++] = a;
    }
    free(fill);
  }

  /* Step 0, preflow (Alg. 1): h(s) = |V|, saturate every arc out of s. */
  for (int64_t v = 0; v < n; ++v) g->h[v] = 0;
  g->h[s] = n;
  for (int64_t k = g->first[s]; k < g->first[s + 1]; ++k) {
    int64_t a = g->adj[k];
    int64_t d = g->rc[a];
    if (d <= 0) continue;
    g->rc[a] = 0;
    g->rc[a ^ 1] += d;
    g->e[g->head[a]] += d;
  }
  g->e[s] = 0;   /* e(s) is not tracked as negative; only e(v), v != s, matters */

  if (use_gr) {
    global_relabel(g, t, s);
  } else {
    for (int64_t k = 0; k < n; ++k) g->cnt[k] = 0;
    for (int64_t v = 0; v < n; ++v) if (g->h[v] < n) g->cnt[g->h[v]]++;
    for (int64_t v = 0; v < n; ++v) {
      g->cur[v] = g->first[v];
      if (v != s && v != t && g->e[v] > 0) q_push(g, v);
    }
  }
  /* Phase 1: discharge until no active vertex remains ("until there are no
   * remaining active vertices"). */
  run_fifo(g, t, s, use_gr, use_gap);
  int64_t F = g->e[t];
  int64_t p1_pushes = g->pushes, p1_relabels = g->relabels, p1_grs = g->grs, p1_gaps = g->gaps;

  /* S* = V \ {v reaches t in G_f}: a fresh reverse BFS that ignores the labels. */
  int64_t* lvl = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  reverse_bfs(g, t, -1, lvl);
  uint8_t* S = (uint8_t*)malloc((size_t)n);
  for (int64_t v = 0; v < n; ++v) S[v] = (lvl[v] == n) ? 1 : 0;
  free(lvl);

  /* cut capacity over the INPUT edges (P:120-127 definition) */
  int64_t cut = 0;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t i = row_off[u]; i < row_off[u + 1]; ++i)
      if (S[u] && !S[col[i]]) cut += cap[i];

  /* Phase 2: return stranded excess to s (target = s, blocked = t). */
  if (phase2) {
    g->pushes = g->relabels = 0;
    g->h[t] = n;
    global_relabel(g, s, t);
    run_fifo(g, s, t, 1, use_gap);
  }
  if (edge_flow)
    for (int64_t i = 0; i < m; ++i)
      edge_flow[i] = (tail[2 * i] == g->head[2 * i]) ? 0 : (int64_t)cap[i] - g->rc[2 * i];

  if (flow_out) *flow_out = F;
  if (cutcap_out) *cutcap_out = cut;
  if (in_S) memcpy(in_S, S, (size_t)n);
  if (stats) {
    stats[0] = p1_pushes; stats[1] = p1_relabels; stats[2] = p1_grs; stats[3] = p1_gaps;
    stats[4] = phase2 ? g->pushes : 0; stats[5] = phase2 ? g->relabels : 0;
  }
  free(S); free(tail);
  free(g->head); free(g->rc); free(g->first); free(g->adj); free(g->e); free(g->h);
  free(g->cur); free(g->cnt); free(g->queue); free(g->inq); free(g->bfsq);
  return 0;
}

/*
 * oracle_initial_state — Step 0 of Alg. 1 followed by one exact global
 * relabel on the resulting residual graph, exposed for the worked
 * examples of SPEC S:155-157 / S:215 and for the CUDA path's initial-label parity.
 *   excess_out (n):  e(v) right after the preflow;      *excess_total_out = sum c(s,v)
 *   level_out  (n):  reverse-BFS distance to t in G_f after the preflow; unreached = n;
 *                    s is never expanded and keeps n.
 *   level0_out (n, may be NULL): the same BFS on the graph BEFORE the preflow
 *                    (all arcs at full capacity; s included).
 */
int oracle_initial_state(int64_t n, int64_t m, const int64_t* row_off, const int32_t* col,
                         const int32_t* cap, int64_t s, int64_t t, int64_t* excess_out,
                         int64_t* excess_total_out, int64_t* level_out, int64_t* level0_out) {
  if (n < 2 || s < 0 || t < 0 || s >= n || t >= n || s == t) return -1;
  pr_t G; memset(&G, 0, sizeof(G));
  pr_t* g = &G;
  g->n = n; g->m = m;
  g->head = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * m + 1));
  g->rc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  g->first = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
  g->adj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  g->bfsq = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* tail = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * m + 1));
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t i = row_off[u]; i < row_off[u + 1]; ++i) {
      int64_t v = col[i];
      g->head[2 * i] = (int32_t)v;     tail[2 * i] = u;     g->rc[2 * i] = cap[i];
      g->head[2 * i + 1] = (int32_t)u; tail[2 * i + 1] = v; g->rc[2 * i + 1] = 0;
      if (u != v) { g->first[u + 1]++; g->first[v + 1]++; }
    }
  for (int64_t v = 0; v < n; ++v) g->first[v + 1] += g->first[v];
  for (int64_t v = 0; v < n; ++v) fill[v] = g->first[v];
  for (int64_t a = 0; a < 2 * m; ++a)
    if (g->head[a] != tail[a]) g->adj[fill[tail[a]]++] = a;
  if (level0_out) reverse_bfs(g, t, -1, level0_out);
  for (int64_t v = 0; v < n; ++v) excess_out[v] = 0;
  int64_t tot = 0;
  for (int64_t k = g->first[s]; k < g->first[s + 1]; ++k) {
    int64_t a = g->adj[k];
    int64_t d = g->rc[a];
    if (d <= 0) continue;
    g->rc[a] = 0; g->rc[a ^ 1] += d;
    excess_out[g->head[a]] += d;
    tot += d;
  }
  excess_out[s] = 0;
  *excess_total_out = tot;
  reverse_bfs(g, t, s, level_out);
  level_out[s] = n;
  free(fill); free(tail); free(g->head); free(g->rc); free(g->first); free(g->adj); free(g->bfsq);
  return 0;
}
