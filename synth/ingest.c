/*
 * synth/ingest.c — readers for the paper's on-disk workloads (§4.1, P:427-434;
 * SPEC.md "ingest" module): DIMACS max-flow files (the Washington / Genrmf
 * networks of Table 1), SNAP edge lists (Table 1 R0-R10; unit
 * capacities per the Table 1 caption) and KONECT bipartite edge lists (Table 2).
 *
 * Like gen.c this module holds NO max-flow arithmetic: it turns text into edge lists that
 * both the oracle and the CUDA path consume (the Python side builds the CSR).  Every
 * reader fills an ingest_result whose arrays are malloc'd here and released by
 * ingest_free(); ids come out 0-based.
 *
 * Grammars (all readers accept CRLF line ends and trailing whitespace):
 *   DIMACS  `c ...` comments; one `p max N M`; `n ID s` / `n ID t`; `a U V CAP` (1-based)
 *   SNAP    `#` comments; `u v` per line, arbitrary non-negative ids, remapped densely in
 *           order of first appearance; self-loops dropped; duplicates merged with
 *           their capacities summed
 *   KONECT  `%` comments (the second header line `% E L R` gives the side sizes when
 *           present); `l r [weight [time]]` per line, 1-based per side; weights ignored;
 *           duplicates collapsed
 * Errors are returned as negative codes with the offending 1-based line in err_line.
 */
#include <ctype.h>
#include <errno.h>
#include <fcntl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

enum {
  ING_OK = 0,
  ING_EIO = -1,           /* cannot open / read the file */
  ING_ENOPROBLEM = -2,    /* DIMACS: no `p max` line */
  ING_ENOTERMINAL = -3,   /* DIMACS: no source or no sink designated */
  ING_EMALFORMED = -4,    /* a line that does not parse (err_line) */
  ING_ERANGE = -5,        /* vertex id outside the declared range (err_line) */
  ING_ECAP = -6,          /* capacity negative or above INT32_MAX (err_line) */
  ING_ENOMEM = -7,
};

typedef struct {
  int64_t n, m;              /* vertices, edges written to src/dst/cap */
  int32_t *src, *dst, *cap;  /* malloc'd, 0-based ids */
  int64_t s, t;              /* DIMACS terminals (0-based), else -1 */
  int64_t nL, nR;            /* KONECT side sizes */
  int64_t declared_m;        /* DIMACS problem line arc count / KONECT header E, else -1 */
  int64_t self_loops;        /* SNAP self-loops dropped */
  int64_t duplicates;        /* SNAP / KONECT duplicate lines merged */
  int64_t err_line;          /* 1-based line of the error, 0 if none */
} ingest_result;

void ingest_free(ingest_result* r) {
  free(r->src); free(r->dst); free(r->cap);
  r->src = r->dst = r->cap = NULL;
}

/* ---- file mapping and a line cursor ---- */
typedef struct { const char *p, *end; void* map; size_t len; int64_t line; } cursor;

static int map_file(const char* path, cursor* c) {
  memset(c, 0, sizeof(*c));
  int fd = open(path, O_RDONLY);
  if (fd < 0) return ING_EIO;
  struct stat st;
  if (fstat(fd, &st) != 0) { close(fd); return ING_EIO; }
  c->len = (size_t)st.st_size;
  if (c->len > 0) {
    c->map = mmap(NULL, c->len, PROT_READ, MAP_PRIVATE, fd, 0);
    if (c->map == MAP_FAILED) { close(fd); c->map = NULL; return ING_EIO; }
    madvise(c->map, c->len, MADV_SEQUENTIAL);
  }
  close(fd);
  c->p = (const char*)c->map;
  c->end = c->p + c->len;
  return ING_OK;
}
static void unmap_file(cursor* c) { if (c->map) munmap(c->map, c->len); c->map = NULL; }

/* next line as [*b, *e) without the line end; returns 0 at EOF */
static int next_line(cursor* c, const char** b, const char** e) {
  if (c->p >= c->end) return 0;
  const char* s = c->p;
  const char* nl = memchr(s, '\n', (size_t)(c->end - s));
  const char* le = nl ? nl : c->end;
  c->p = nl ? nl + 1 : c->end;
  while (le > s && (le[-1] == '\r' || le[-1] == ' ' || le[-1] == '\t')) --le;
  while (s < le && (*s == ' ' || *s == '\t')) ++s;
  *b = s; *e = le;
  c->line++;
  return 1;
}
static int parse_i64(const char** p, const char* e, int64_t* out) {
  const char* s = *p;
  while (s < e && (*s == ' ' || *s == '\t')) ++s;
  int neg = 0;
  if (s < e && (*s == '-' || *s == '+')) { neg = *s == '-'; ++s; }
  if (s >= e || !isdigit((unsigned char)*s)) return 0;
  int64_t v = 0;
  while (s < e && isdigit((unsigned char)*s)) {
    if (v > (INT64_MAX - 9) / 10) return 0;
    v = v * 10 + (*s - '0');
    ++s;
  }
  if (s < e && !(*s == ' ' || *s == '\t')) return 0;   /* e.g. "12x" or "1.5" */
  *out = neg ? -v : v;
  *p = s;
  return 1;
}
/* skip a numeric-looking token (KONECT weights may be floats) */
static int skip_token(const char** p, const char* e) {
  const char* s = *p;
  while (s < e && (*s == ' ' || *s == '\t')) ++s;
  if (s >= e) return 0;
  while (s < e && !(*s == ' ' || *s == '\t')) ++s;
  *p = s;
  return 1;
}
static int at_end(const char* p, const char* e) {
  while (p < e && (*p == ' ' || *p == '\t')) ++p;
  return p == e;
}

/* growable edge arrays */
typedef struct { int32_t *a, *b, *c; int64_t n, capn; } edges;
static int push_edge(edges* E, int64_t u, int64_t v, int64_t w) {
  if (E->n == E->capn) {
    int64_t nc = E->capn ? E->capn * 2 : 1 << 16;
    int32_t* a = (int32_t*)realloc(E->a, (size_t)nc * 4);
    if (!a) return ING_ENOMEM;
    E->a = a;
    int32_t* b = (int32_t*)realloc(E->b, (size_t)nc * 4);
    if (!b) return ING_ENOMEM;
    E->b = b;
    if (w >= 0 || E->c) {
      int32_t* c = (int32_t*)realloc(E->c, (size_t)nc * 4);
      if (!c) return ING_ENOMEM;
      E->c = c;
    }
    E->capn = nc;
  }
  E->a[E->n] = (int32_t)u;
  E->b[E->n] = (int32_t)v;
  if (E->c) E->c[E->n] = (int32_t)w;
  E->n++;
  return ING_OK;
}
static void free_edges(edges* E) { free(E->a); free(E->b); free(E->c); memset(E, 0, sizeof(*E)); }

/* ------------------------------------------------------------------ DIMACS max-flow */
int32_t ingest_dimacs(const char* path, ingest_result* r) {
  memset(r, 0, sizeof(*r));
  r->s = r->t = -1; r->declared_m = -1; r->nL = r->nR = -1;
  cursor c;
  int rc = map_file(path, &c);
  if (rc) return rc;
  edges E = {0};
  int64_t n = -1;
  const char *b, *e;
  rc = ING_OK;
  while (rc == ING_OK && next_line(&c, &b, &e)) {
    if (b == e || *b == 'c') continue;
    const char* p = b + 1;
    if (*b == 'p') {
      while (p < e && (*p == ' ' || *p == '\t')) ++p;
      if (e - p < 3 || strncmp(p, "max", 3) != 0 || n >= 0) { rc = ING_EMALFORMED; break; }
      p += 3;
      int64_t N, M;
      if (!parse_i64(&p, e, &N) || !parse_i64(&p, e, &M) || !at_end(p, e) || N < 0 || M < 0 || N > INT32_MAX) {
        rc = ING_EMALFORMED; break;
      }
      n = N; r->declared_m = M;
    } else if (*b == 'n') {
      int64_t id;
      if (n < 0 || !parse_i64(&p, e, &id)) { rc = n < 0 ? ING_ENOPROBLEM : ING_EMALFORMED; break; }
      while (p < e && (*p == ' ' || *p == '\t')) ++p;
      if (p + 1 != e || (*p != 's' && *p != 't')) { rc = ING_EMALFORMED; break; }
      if (id < 1 || id > n) { rc = ING_ERANGE; break; }
      if (*p == 's') r->s = id - 1; else r->t = id - 1;
    } else if (*b == 'a') {
      int64_t u, v, w;
      if (n < 0) { rc = ING_ENOPROBLEM; break; }
      if (!parse_i64(&p, e, &u) || !parse_i64(&p, e, &v) || !parse_i64(&p, e, &w) || !at_end(p, e)) {
        rc = ING_EMALFORMED; break;
      }
      if (u < 1 || u > n || v < 1 || v > n) { rc = ING_ERANGE; break; }
      if (w < 0 || w > INT32_MAX) { rc = ING_ECAP; break; }
      rc = push_edge(&E, u - 1, v - 1, w);
      if (E.c == NULL && rc == ING_OK) rc = ING_ENOMEM;
    } else {
      rc = ING_EMALFORMED;
    }
  }
  if (rc != ING_OK) r->err_line = c.line;
  unmap_file(&c);
  if (rc == ING_OK && n < 0) rc = ING_ENOPROBLEM;
  if (rc == ING_OK && (r->s < 0 || r->t < 0)) rc = ING_ENOTERMINAL;
  if (rc != ING_OK) { free_edges(&E); return rc; }
  r->n = n; r->m = E.n;
  r->src = E.a; r->dst = E.b; r->cap = E.c;
  return ING_OK;
}

/* ---- open-addressing map: int64 id -> dense int32 (first appearance) ---- */
typedef struct { int64_t* key; int32_t* val; int64_t mask, size; } idmap;
static uint64_t hmix(uint64_t z) {
  z ^= z >> 33; z *= 0xff51afd7ed558ccdull; z ^= z >> 33; z *= 0xc4ceb9fe1a85ec53ull; z ^= z >> 33;
  return z;
}
static int idmap_init(idmap* h, int64_t cap) {
  int64_t sz = 1024;
  while (sz < 2 * cap) sz <<= 1;
  h->key = (int64_t*)malloc((size_t)sz * 8);
  h->val = (int32_t*)malloc((size_t)sz * 4);
  if (!h->key || !h->val) return ING_ENOMEM;
  memset(h->key, 0xff, (size_t)sz * 8);   /* -1 = empty (ids are non-negative) */
  h->mask = sz - 1; h->size = 0;
  return ING_OK;
}
static int idmap_grow(idmap* h) {
  idmap g;
  if (idmap_init(&g, (h->mask + 1)) != ING_OK) return ING_ENOMEM;
  for (int64_t i = 0; i <= h->mask; ++i)
    if (h->key[i] >= 0) {
      int64_t j = (int64_t)(hmix((uint64_t)h->key[i]) & (uint64_t)g.mask);
      while (g.key[j] >= 0) j = (j + 1) & g.mask;
      g.key[j] = h->key[i]; g.val[j] = h->val[i];
    }
  g.size = h->size;
  free(h->key); free(h->val);
  *h = g;
  return ING_OK;
}
/* returns the dense id, or -1 on allocation failure / more than INT32_MAX ids */
static int64_t idmap_get(idmap* h, int64_t id) {
  if (2 * (h->size + 1) > h->mask + 1 && idmap_grow(h) != ING_OK) return -1;
  int64_t j = (int64_t)(hmix((uint64_t)id) & (uint64_t)h->mask);
  while (h->key[j] >= 0) {
    if (h->key[j] == id) return h->val[j];
    j = (j + 1) & h->mask;
  }
  if (h->size >= INT32_MAX) return -1;
  h->key[j] = id; h->val[j] = (int32_t)h->size;
  return h->size++;
}
static void idmap_free(idmap* h) { free(h->key); free(h->val); }

/* LSD radix sort of (key, payload) by 64-bit key */
static int sort_pairs(uint64_t* k, int32_t* v, int64_t n, int bits) {
  if (n <= 1) return ING_OK;
  uint64_t* tk = (uint64_t*)malloc((size_t)n * 8);
  int32_t* tv = v ? (int32_t*)malloc((size_t)n * 4) : NULL;
  int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
  if (!tk || (v && !tv) || !cnt) { free(tk); free(tv); free(cnt); return ING_ENOMEM; }
  for (int sh = 0; sh < bits; sh += 16) {
    memset(cnt, 0, 65536 * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) cnt[(k[i] >> sh) & 0xffff]++;
    int64_t s = 0;
    for (int d = 0; d < 65536; ++d) { int64_t x = cnt[d]; cnt[d] = s; s += x; }
    for (int64_t i = 0; i < n; ++i) {
      int64_t q = cnt[(k[i] >> sh) & 0xffff]++;
      tk[q] = k[i];
      if (v) tv[q] = v[i];
    }
    memcpy(k, tk, (size_t)n * 8);
    if (v) memcpy(v, tv, (size_t)n * 4);
  }
  free(tk); free(tv); free(cnt);
  return ING_OK;
}
static int bits_of(int64_t n) { int b = 1; while (b < 63 && ((int64_t)1 << b) < n) ++b; return b; }

/* ------------------------------------------------------------------ SNAP edge list */
int32_t ingest_snap(const char* path, int32_t default_cap, ingest_result* r) {
  memset(r, 0, sizeof(*r));
  r->s = r->t = -1; r->declared_m = -1; r->nL = r->nR = -1;
  if (default_cap < 0) return ING_ECAP;
  cursor c;
  int rc = map_file(path, &c);
  if (rc) return rc;
  idmap H;
  if (idmap_init(&H, 1 << 16) != ING_OK) { unmap_file(&c); return ING_ENOMEM; }
  edges E = {0};
  const char *b, *e;
  while (rc == ING_OK && next_line(&c, &b, &e)) {
    if (b == e || *b == '#' || *b == '%') continue;
    const char* p = b;
    int64_t u, v;
    if (!parse_i64(&p, e, &u) || !parse_i64(&p, e, &v) || !at_end(p, e)) { rc = ING_EMALFORMED; break; }
    if (u < 0 || v < 0) { rc = ING_ERANGE; break; }
    int64_t du = idmap_get(&H, u), dv = idmap_get(&H, v);
    if (du < 0 || dv < 0) { rc = ING_ENOMEM; break; }
    if (du == dv) { r->self_loops++; continue; }
    rc = push_edge(&E, du, dv, -1);
  }
  if (rc != ING_OK) r->err_line = c.line;
  unmap_file(&c);
  const int64_t n = H.size;
  idmap_free(&H);
  if (rc != ING_OK) { free_edges(&E); return rc; }
  /* duplicates merged, capacities summed: sort by (u, v), sum runs */
  const int64_t m0 = E.n;
  uint64_t* key = (uint64_t*)malloc((size_t)(m0 > 0 ? m0 : 1) * 8);
  if (!key) { free_edges(&E); return ING_ENOMEM; }
  for (int64_t i = 0; i < m0; ++i) key[i] = ((uint64_t)(uint32_t)E.a[i] << 32) | (uint32_t)E.b[i];
  free_edges(&E);
  rc = sort_pairs(key, NULL, m0, 32 + bits_of(n));
  if (rc != ING_OK) { free(key); return rc; }
  int64_t m = 0;
  for (int64_t i = 0; i < m0; ++i) if (i == 0 || key[i] != key[i - 1]) ++m;
  r->src = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * 4);
  r->dst = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * 4);
  r->cap = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * 4);
  if (!r->src || !r->dst || !r->cap) { free(key); ingest_free(r); return ING_ENOMEM; }
  int64_t j = -1;
  for (int64_t i = 0; i < m0; ++i) {
    if (i == 0 || key[i] != key[i - 1]) {
      ++j;
      r->src[j] = (int32_t)(key[i] >> 32);
      r->dst[j] = (int32_t)(key[i] & 0xffffffffu);
      r->cap[j] = default_cap;
    } else {
      r->duplicates++;
      if ((int64_t)r->cap[j] + default_cap > INT32_MAX) { free(key); ingest_free(r); return ING_ECAP; }
      r->cap[j] += default_cap;
    }
  }
  free(key);
  r->n = n; r->m = m;
  return ING_OK;
}

/* ------------------------------------------------------------------ KONECT bipartite */
int32_t ingest_konect(const char* path, ingest_result* r) {
  memset(r, 0, sizeof(*r));
  r->s = r->t = -1; r->declared_m = -1;
  cursor c;
  int rc = map_file(path, &c);
  if (rc) return rc;
  edges E = {0};
  int64_t nL = 0, nR = 0, hdrL = 0, hdrR = 0;
  int headers = 0;
  const char *b, *e;
  while (rc == ING_OK && next_line(&c, &b, &e)) {
    if (b == e) continue;
    if (*b == '%' || *b == '#') {
      /* KONECT's second header line: "% E L R" */
      if (*b == '%' && ++headers == 2) {
        const char* p = b + 1;
        int64_t x, y, z;
        if (parse_i64(&p, e, &x) && parse_i64(&p, e, &y) && parse_i64(&p, e, &z) && x >= 0 && y >= 0 && z >= 0) {
          r->declared_m = x; hdrL = y; hdrR = z;
        }
      }
      continue;
    }
    const char* p = b;
    int64_t l, q;
    if (!parse_i64(&p, e, &l) || !parse_i64(&p, e, &q)) { rc = ING_EMALFORMED; break; }
    while (skip_token(&p, e)) {}   /* weight / timestamp columns are ignored */
    if (l < 1 || q < 1 || l > INT32_MAX || q > INT32_MAX) { rc = ING_ERANGE; break; }
    if (l > nL) nL = l;
    if (q > nR) nR = q;
    rc = push_edge(&E, l - 1, q - 1, -1);
  }
  if (rc != ING_OK) r->err_line = c.line;
  unmap_file(&c);
  if (rc != ING_OK) { free_edges(&E); return rc; }
  if (hdrL > nL) nL = hdrL;
  if (hdrR > nR) nR = hdrR;
  const int64_t m0 = E.n;
  uint64_t* key = (uint64_t*)malloc((size_t)(m0 > 0 ? m0 : 1) * 8);
  if (!key) { free_edges(&E); return ING_ENOMEM; }
  for (int64_t i = 0; i < m0; ++i) key[i] = ((uint64_t)(uint32_t)E.a[i] << 32) | (uint32_t)E.b[i];
  free_edges(&E);
  rc = sort_pairs(key, NULL, m0, 32 + bits_of(nL));
  if (rc != ING_OK) { free(key); return rc; }
  int64_t m = 0;
  for (int64_t i = 0; i < m0; ++i) if (i == 0 || key[i] != key[i - 1]) ++m;
  r->src = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * 4);
  r->dst = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * 4);
  if (!r->src || !r->dst) { free(key); ingest_free(r); return ING_ENOMEM; }
  int64_t j = 0;
  for (int64_t i = 0; i < m0; ++i) {
    if (i > 0 && key[i] == key[i - 1]) { r->duplicates++; continue; }
    r->src[j] = (int32_t)(key[i] >> 32);
    r->dst[j] = (int32_t)(key[i] & 0xffffffffu);
    ++j;
  }
  free(key);
  r->nL = nL; r->nR = nR; r->n = nL + nR; r->m = m;
  return ING_OK;
}
