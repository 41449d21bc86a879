/*
 * synth.c — seeded synthetic inputs for Batched SpMM (arXiv 1903.11409).
 *
 * This module ONLY draws inputs. It holds none of the method's arithmetic
 * (no products, no scans used by the method, no sorting of COO entries): it
 * is shared by the oracle side (oracle/, tests) and the CUDA side (bench,
 * GPU tests) exactly so that both see the same bytes.
 * "Input recipe".
 *
 * Generators:
 *   G-rand(dim, d)   — PAPER.md:340 ("randomly generated sparse matrices are
 *                      square. The row size (dim) and nnz/row are parameterized"):
 *                      dim x dim, every row has exactly d distinct columns drawn
 *                      uniformly without replacement; diagonal not forced.
 *   G-mix            — PAPER.md:429 (batch with mixed dim and nnz/row): per graph
 *                      dim ~ U{dmin..dmax}, d ~ U{dlo..dhi}, then G-rand(dim, d).
 *   G-mol(nmin,nmax) — molecule-like (Tox21-shaped, max dim 50;
 *                      north_star 20-60 nodes): random spanning tree with
 *                      valence cap 4, floor(n/10) ring-closing edges, symmetric,
 *                      plus self-loops a_uu = 1.
 *
 * Determinism: graph i draws from its own splitmix64 streams keyed by
 * (seed, i, stream), so any contiguous range [i0, i1) can be regenerated
 * alone (multi-GPU ranks) and results never depend on the thread count.
 * Streams: 0 = structure, 1 = A values, 2 = B values, 3 = COO shuffle.
 *
 * Values: A and B ~ U[-1, 1) on the 2^-23 grid (exact in fp32); integer
 * variant (reading R3): A in {1, 2}, B in {-8..8}.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SYN_RAND 0
#define SYN_MOL 1
#define SYN_MIX 2

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
typedef struct { uint64_t s; } rng_t;
static inline uint64_t rng_next(rng_t* r) {
  r->s += 0x9E3779B97F4A7C15ull;
  return mix64(r->s);
}
static inline rng_t rng_for(uint64_t seed, int64_t graph, int stream) {
  rng_t r;
  r.s = mix64(seed ^ mix64((uint64_t)graph * 8ull + (uint64_t)stream + 0x5851F42D4C957F2Dull));
  return r;
}
/* uniform integer in [0, m), m >= 1 (Lemire multiply-shift on the top 32 bits) */
static inline uint32_t rng_below(rng_t* r, uint32_t m) {
  return (uint32_t)(((rng_next(r) >> 32) * (uint64_t)m) >> 32);
}
/* uniform in [-1, 1) on the 2^-23 grid: exactly representable in fp32 */
static inline float rng_pm1(rng_t* r) {
  int32_t v = (int32_t)(rng_next(r) >> 40) - (1 << 23);
  return (float)v * (1.0f / 8388608.0f);
}

/* ---- per-graph structure (CSR rows with sorted local columns) ---------- */
typedef struct {
  int n;
  int cap_nnz;
  int nnz;
  int32_t* rp;  /* n+1 */
  int32_t* col; /* nnz */
  int cap_n;
  /* scratch */
  int32_t* deg;
  int32_t* nb; /* n*4 */
  uint8_t* mark;
} graph_t;

static void g_reserve(graph_t* g, int n, int nnz) {
  if (n + 1 > g->cap_n) {
    g->cap_n = 2 * (n + 1);
    g->rp = (int32_t*)realloc(g->rp, sizeof(int32_t) * g->cap_n);
    g->deg = (int32_t*)realloc(g->deg, sizeof(int32_t) * g->cap_n);
    g->nb = (int32_t*)realloc(g->nb, sizeof(int32_t) * 4 * g->cap_n);
    g->mark = (uint8_t*)realloc(g->mark, g->cap_n);
  }
  if (nnz > g->cap_nnz) {
    g->cap_nnz = 2 * nnz;
    g->col = (int32_t*)realloc(g->col, sizeof(int32_t) * g->cap_nnz);
  }
}
static void g_free(graph_t* g) {
  free(g->rp); free(g->col); free(g->deg); free(g->nb); free(g->mark);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* exactly d distinct uniform columns per row (rejection against a mark array) */
static void gen_rand(graph_t* g, rng_t* r, int dim, int d) {
  if (d > dim) d = dim;
  g_reserve(g, dim, dim * d);
  g->n = dim;
  memset(g->mark, 0, dim);
  int e = 0;
  for (int row = 0; row < dim; ++row) {
    g->rp[row] = e;
    for (int j = 0; j < d; ++j) {
      int c;
      do { c = (int)rng_below(r, (uint32_t)dim); } while (g->mark[c]);
      g->mark[c] = 1;
      g->col[e + j] = c;
    }
    for (int j = 0; j < d; ++j) g->mark[g->col[e + j]] = 0;
    qsort(g->col + e, d, sizeof(int32_t), cmp_i32);
    e += d;
  }
  g->rp[dim] = e;
  g->nnz = e;
}

static int adjacent(const graph_t* g, int u, int v) {
  for (int j = 0; j < g->deg[u]; ++j)
    if (g->nb[4 * u + j] == v) return 1;
  return 0;
}
static void add_edge(graph_t* g, int u, int v) {
  g->nb[4 * u + g->deg[u]++] = v;
  g->nb[4 * v + g->deg[v]++] = u;
}

static void gen_mol(graph_t* g, rng_t* r, int nmin, int nmax) {
  int n = nmin + (int)rng_below(r, (uint32_t)(nmax - nmin + 1));
  g_reserve(g, n, 5 * n);
  g->n = n;
  for (int v = 0; v < n; ++v) g->deg[v] = 0;
  /* spanning tree: v attaches to a uniform earlier node with degree < 4 */
  for (int v = 1; v < n; ++v) {
    int u = -1;
    for (int tries = 0; tries < 16; ++tries) {
      int c = (int)rng_below(r, (uint32_t)v);
      if (g->deg[c] < 4) { u = c; break; }
    }
    if (u < 0)
      for (int c = 0; c < v; ++c)
        if (g->deg[c] < 4) { u = c; break; }
    add_edge(g, u, v);
  }
  /* floor(n/10) ring-closing edges between non-adjacent nodes of degree < 4 */
  int rings = n / 10;
  for (int k = 0; k < rings; ++k) {
    for (int tries = 0; tries < 8; ++tries) {
      int a = (int)rng_below(r, (uint32_t)n), b = (int)rng_below(r, (uint32_t)n);
      if (a == b || g->deg[a] >= 4 || g->deg[b] >= 4 || adjacent(g, a, b)) continue;
      add_edge(g, a, b);
      break;
    }
  }
  /* rows: self-loop + neighbours, sorted */
  int e = 0;
  for (int v = 0; v < n; ++v) {
    g->rp[v] = e;
    g->col[e] = v;
    for (int j = 0; j < g->deg[v]; ++j) g->col[e + 1 + j] = g->nb[4 * v + j];
    qsort(g->col + e, 1 + g->deg[v], sizeof(int32_t), cmp_i32);
    e += 1 + g->deg[v];
  }
  g->rp[n] = e;
  g->nnz = e;
}

static void gen_graph(graph_t* g, int kind, const int* p, uint64_t seed, int64_t i) {
  rng_t r = rng_for(seed, i, 0);
  if (kind == SYN_RAND) {
    gen_rand(g, &r, p[0], p[1]);
  } else if (kind == SYN_MOL) {
    gen_mol(g, &r, p[0], p[1]);
  } else {
    int dim = p[0] + (int)rng_below(&r, (uint32_t)(p[1] - p[0] + 1));
    int d = p[2] + (int)rng_below(&r, (uint32_t)(p[3] - p[2] + 1));
    gen_rand(g, &r, dim, d);
  }
}

/* ---- exported API --------------------------------------------------------
 * kind/params: SYN_RAND (dim, d), SYN_MOL (nmin, nmax), SYN_MIX (dmin, dmax, dlo, dhi).
 * All "off" arrays are local to the range [i0, i1): off[0] = 0.               */

int synth_counts(int kind, const int* params, uint64_t seed, int64_t i0, int64_t i1,
                 int32_t* n_out, int32_t* nnz_out) {
  if (i1 < i0 || !params) return 1;
  int64_t cnt = i1 - i0;
#pragma omp parallel
  {
    graph_t g;
    memset(&g, 0, sizeof(g));
#pragma omp for schedule(dynamic, 256)
    for (int64_t j = 0; j < cnt; ++j) {
      gen_graph(&g, kind, params, seed, i0 + j);
      n_out[j] = g.n;
      nnz_out[j] = g.nnz;
    }
    g_free(&g);
  }
  return 0;
}

/* row_off/nnz_off: [cnt+1] local prefix sums of the counts (computed by the
 * caller with plain integer adds); row_ptr gets ABSOLUTE (range-local)
 * positions, col LOCAL column ids, vals the A values. */
int synth_fill_csr(int kind, const int* params, uint64_t seed, int64_t i0, int64_t i1,
                   const int64_t* row_off, const int64_t* nnz_off, int32_t* row_ptr,
                   int32_t* col, float* vals, int int_valued) {
  if (i1 < i0 || !params) return 1;
  int64_t cnt = i1 - i0;
#pragma omp parallel
  {
    graph_t g;
    memset(&g, 0, sizeof(g));
#pragma omp for schedule(dynamic, 256)
    for (int64_t j = 0; j < cnt; ++j) {
      gen_graph(&g, kind, params, seed, i0 + j);
      int64_t g0 = row_off[j], z0 = nnz_off[j];
      for (int r = 0; r < g.n; ++r) row_ptr[g0 + r] = (int32_t)(z0 + g.rp[r]);
      rng_t rv = rng_for(seed, i0 + j, 1);
      for (int e = 0; e < g.nnz; ++e) {
        col[z0 + e] = g.col[e];
        vals[z0 + e] = int_valued ? (float)(1 + (int)rng_below(&rv, 2)) : rng_pm1(&rv);
      }
    }
    g_free(&g);
  }
  if (cnt > 0) row_ptr[row_off[cnt]] = (int32_t)nnz_off[cnt];
  else row_ptr[0] = 0;
  return 0;
}

/* B rows of graph i (n_i x k, row-major with leading dimension ld >= k);
 * columns [k, ld) are left untouched. */
int synth_fill_dense(uint64_t seed, int64_t i0, int64_t i1, const int64_t* row_off,
                     int k, int64_t ld, float* B, int int_valued) {
  if (i1 < i0 || k < 0 || ld < k) return 1;
  int64_t cnt = i1 - i0;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t j = 0; j < cnt; ++j) {
    rng_t r = rng_for(seed, i0 + j, 2);
    for (int64_t row = row_off[j]; row < row_off[j + 1]; ++row) {
      float* dst = B + row * ld;
      for (int c = 0; c < k; ++c)
        dst[c] = int_valued ? (float)((int)rng_below(&r, 17) - 8) : rng_pm1(&r);
    }
  }
  return 0;
}

/* SparseTensor (COO) view: each graph's CSR entries, Fisher-Yates shuffled
 * ("non-zero elements are not sorted").  idx is interleaved
 * (row, col) pairs as in TF SparseTensor. */
int synth_shuffle_coo(uint64_t seed, int64_t i0, int64_t i1, const int64_t* row_off,
                      const int64_t* nnz_off, const int32_t* row_ptr, const int32_t* col,
                      const float* vals, int32_t* idx_out, float* vals_out) {
  if (i1 < i0) return 1;
  int64_t cnt = i1 - i0;
#pragma omp parallel
  {
    int64_t cap = 0;
    int32_t* perm = NULL;
#pragma omp for schedule(dynamic, 64)
    for (int64_t j = 0; j < cnt; ++j) {
      int64_t z0 = nnz_off[j], m = nnz_off[j + 1] - z0;
      if (m > cap) { cap = 2 * m; perm = (int32_t*)realloc(perm, sizeof(int32_t) * cap); }
      for (int64_t e = 0; e < m; ++e) perm[e] = (int32_t)e;
      rng_t r = rng_for(seed, i0 + j, 3);
      for (int64_t e = m - 1; e > 0; --e) {
        int64_t s = (int64_t)rng_below(&r, (uint32_t)(e + 1));
        int32_t t = perm[e]; perm[e] = perm[s]; perm[s] = t;
      }
      int64_t nrows = row_off[j + 1] - row_off[j];
      /* place: slot q takes CSR entry perm[q] */
      for (int64_t q = 0; q < m; ++q) {
        int64_t src = z0 + perm[q];
        /* find row of src by binary search over this graph's row_ptr */
        int64_t lo = 0, hi = nrows; /* row_ptr[g0+lo] <= src < row_ptr[g0+hi] */
        while (hi - lo > 1) {
          int64_t mid = (lo + hi) / 2;
          if (row_ptr[row_off[j] + mid] <= src) lo = mid; else hi = mid;
        }
        idx_out[2 * (z0 + q)] = (int32_t)lo;
        idx_out[2 * (z0 + q) + 1] = col[src];
        vals_out[z0 + q] = vals[src];
      }
    }
    free(perm);
  }
  return 0;
}
