/*
 * oracle.c — CPU restatement of the reference algorithms on the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package
 * (paper_2201_02789_b200/) may import, link or call this; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * use it, and only as the checker / the timed CPU baseline.
 *
 * Each function restates the reference's serial (No-CDP) variant, which the
 * reference itself uses as ground truth (bench/harness.py:57-62):
 *   oracle_bfs         BFS_NOCDP main + _bfs_drive  bench/benchmarks.py:122-168
 *   oracle_sssp        SSSP_NOCDP main + relax + _sssp_drive  :184-195,225-270
 *   oracle_manylaunch  MANYLAUNCH_NOCDP main        :303-332
 * and the builder-defined apps the reference lacks (parity unpinned by the
 * reference):
 *   oracle_tc          exact triangle count over a degree-oriented CSR+
 *   oracle_bt          Bezier tessellation, fp64 vertices, fp32 counts
 *   oracle_gc          greedy colouring in Jones-Plassmann (LLF) priority order
 *   oracle_mst         Kruskal minimum spanning forest in (weight, eid) order
 *   oracle_sp          survey propagation sweeps on a k-SAT factor graph
 *
 * Parallel versions (nthreads > 1) use the same atomics the reference's
 * kernels use; outputs are schedule-invariant (benchmarks.py:10-15), so any
 * thread count gives the same bytes.  Integer arithmetic wraps at 32 bits
 * like the reference's (sim/compile.py:36-37, sim/machine.py:35-40).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define UNREACHED (1 << 30) /* bench/graphs.py:29 */

static int nthr(int t) { return t > 0 ? t : omp_get_max_threads(); }

static inline int32_t wrap_add(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}

/* Returns the number of host launches (levels including the final
 * no-change pass), or -1 if more than n+1 levels were needed. */
long oracle_bfs(const int32_t* rowptr, const int32_t* col, int32_t n,
                int32_t src, int32_t* dist, int32_t* counts, int nthreads) {
  const int nt = nthr(nthreads);
  for (int32_t i = 0; i < n; ++i) {
    dist[i] = UNREACHED;
    counts[i] = 0;
  }
  dist[src] = 0;
  for (long level = 0; level <= n; ++level) {
    int changed = 0;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 256) reduction(| : changed)
    for (int32_t u = 0; u < n; ++u) {
      if (__atomic_load_n(&dist[u], __ATOMIC_RELAXED) != level) continue;
      const int32_t start = rowptr[u];
      const int32_t deg = rowptr[u + 1] - start;
      for (int32_t e = 0; e < deg; ++e) {
        const int32_t v = col[start + e];
        __atomic_fetch_add(&counts[v], 1, __ATOMIC_RELAXED);
        int32_t expect = UNREACHED;
        if (__atomic_compare_exchange_n(&dist[v], &expect, (int32_t)level + 1,
                                        0, __ATOMIC_RELAXED, __ATOMIC_RELAXED))
          changed = 1;
      }
    }
    if (!changed) return level + 1;
  }
  return -1;
}

/* Bellman-Ford rounds; returns rounds executed or -1 past n+1 rounds. */
long oracle_sssp(const int32_t* rowptr, const int32_t* col,
                 const int32_t* weight, int32_t n, int32_t src, int32_t* dist,
                 int nthreads) {
  const int nt = nthr(nthreads);
  for (int32_t i = 0; i < n; ++i) dist[i] = UNREACHED;
  dist[src] = 0;
  for (long round = 0; round <= n; ++round) {
    int changed = 0;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 256) reduction(| : changed)
    for (int32_t u = 0; u < n; ++u) {
      const int32_t du = __atomic_load_n(&dist[u], __ATOMIC_RELAXED);
      if (!(du < UNREACHED)) continue;
      const int32_t start = rowptr[u];
      const int32_t deg = rowptr[u + 1] - start;
      for (int32_t e = 0; e < deg; ++e) {
        const int32_t v = col[start + e];
        const int32_t alt = wrap_add(du, weight[start + e]);
        /* relax(): CAS loop lowering dist[v] (benchmarks.py:184-195) */
        int32_t cur = __atomic_load_n(&dist[v], __ATOMIC_RELAXED);
        while (alt < cur) {
          if (__atomic_compare_exchange_n(&dist[v], &cur, alt, 0,
                                          __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
            changed = 1;
            break;
          }
        }
      }
    }
    if (!changed) return round + 1;
  }
  return -1;
}

void oracle_manylaunch(const int32_t* sizes, int32_t n, int32_t* out,
                       int32_t* total, int nthreads) {
  const int nt = nthr(nthreads);
  int32_t tot = 0;
  memset(out, 0, sizeof(int32_t) * (size_t)n);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 256)
  for (int32_t i = 0; i < n; ++i) {
    const int32_t s = sizes[i];
    int32_t acc = 0, cnt = 0;
    for (int32_t j = 0; j < s; ++j) {
      acc = wrap_add(acc, j + 1);
      cnt = wrap_add(cnt, 1);
    }
    out[i] = acc;
    __atomic_fetch_add(&tot, cnt, __ATOMIC_RELAXED);
  }
  *total = tot;
}

/* sorted-merge intersection size */
static int64_t merge_count(const int32_t* a, int64_t na, const int32_t* b,
                           int64_t nb) {
  int64_t i = 0, j = 0, c = 0;
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (a[i] > b[j]) ++j;
    else { ++c; ++i; ++j; }
  }
  return c;
}

/* triangles = sum over oriented edges (u,v) in [lo,hi) of |N+(u) ∩ N+(v)| */
uint64_t oracle_tc(const int32_t* rowptr, const int32_t* col, int32_t n,
                   int64_t lo, int64_t hi, int nthreads) {
  const int nt = nthr(nthreads);
  uint64_t total = 0;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64) reduction(+ : total)
  for (int32_t u = 0; u < n; ++u) {
    int64_t b = rowptr[u], e = rowptr[u + 1];
    if (b < lo) b = lo;
    if (e > hi) e = hi;
    for (int64_t k = b; k < e; ++k) {
      const int32_t v = col[k];
      total += (uint64_t)merge_count(col + rowptr[u], rowptr[u + 1] - rowptr[u],
                                     col + rowptr[v], rowptr[v + 1] - rowptr[v]);
    }
  }
  return total;
}

/* Vertex count per curve, fp32 round-to-nearest with no contraction (built
 * with -ffp-contract=off), identical to the device computation. */
static int32_t tess_count(const float* p, float scale, int32_t max_tess) {
  volatile float mx = 0.5f * (p[0] + p[4]);
  volatile float my = 0.5f * (p[1] + p[5]);
  volatile float dx = p[2] - mx, dy = p[3] - my;
  volatile float lx = p[4] - p[0], ly = p[5] - p[1];
  volatile float dxx = dx * dx, dyy = dy * dy, lxx = lx * lx, lyy = ly * ly;
  volatile float num = sqrtf(dxx + dyy);
  volatile float den = sqrtf(lxx + lyy);
  volatile float q = num / den;
  volatile float t = q * scale;
  int32_t nt = t < (float)max_tess ? (int32_t)t : max_tess;
  return nt < 4 ? 4 : nt;
}

/* ntess[c]; canonical offsets[c] = exclusive prefix; verts[2*V] in fp64.
 * Returns total vertex count (call with verts == NULL to size). */
int64_t oracle_bt(const float* cp, int32_t ncurves, int32_t max_tess,
                  float scale, int32_t* ntess, int64_t* offsets, double* verts,
                  int nthreads) {
  const int nt_ = nthr(nthreads);
  int64_t acc = 0;
  for (int32_t c = 0; c < ncurves; ++c) {
    ntess[c] = tess_count(cp + 6 * (int64_t)c, scale, max_tess);
    offsets[c] = acc;
    acc += ntess[c];
  }
  if (!verts) return acc;
#pragma omp parallel for num_threads(nt_) schedule(dynamic, 64)
  for (int32_t c = 0; c < ncurves; ++c) {
    const float* p = cp + 6 * (int64_t)c;
    const int32_t nt = ntess[c];
    for (int32_t i = 0; i < nt; ++i) {
      const double t = (double)i / (double)(nt - 1);
      const double s = 1.0 - t;
      double* o = verts + 2 * (offsets[c] + i);
      o[0] = s * s * p[0] + 2.0 * s * t * p[2] + t * t * p[4];
      o[1] = s * s * p[1] + 2.0 * s * t * p[3] + t * t * p[5];
    }
  }
  return acc;
}

/* ---- graph colouring (north-star app; no reference implementation) ------
 * Sequential greedy colouring in decreasing priority key(v) =
 * (floor(log2(deg v + 1)) : 5 bits, high 27 bits of hash32(v), v : 32 bits)
 * (largest-log-degree-first, hash tie-break): each vertex takes the smallest
 * colour unused by its already-coloured (= higher-priority) neighbours.
 * Independent restatement of what the Jones-Plassmann rounds on the device
 * must produce. */
static uint64_t gc_key(int32_t v, int32_t deg) {
  uint32_t x = (uint32_t)v * 0x9E3779B1u;
  x ^= x >> 16;
  x *= 0x85EBCA6Bu;
  x ^= x >> 13;
  x *= 0xC2B2AE35u;
  x ^= x >> 16;
  uint32_t lg = 0;
  for (uint32_t d = (uint32_t)deg + 1u; d > 1u; d >>= 1) ++lg;
  return ((uint64_t)lg << 59) | ((uint64_t)(x >> 5) << 32) | (uint32_t)v;
}

static int gc_cmp_desc(const void* a, const void* b) {
  const uint64_t ka = *(const uint64_t*)a, kb = *(const uint64_t*)b;
  return ka < kb ? 1 : (ka > kb ? -1 : 0);
}

/* returns the number of colours used, or -1 on allocation failure */
int32_t oracle_gc(const int32_t* rowptr, const int32_t* col, int32_t n,
                  int32_t* color) {
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
  int32_t maxdeg = 0;
  for (int32_t u = 0; u < n; ++u) {
    keys[u] = gc_key(u, rowptr[u + 1] - rowptr[u]);
    color[u] = -1;
    if (rowptr[u + 1] - rowptr[u] > maxdeg) maxdeg = rowptr[u + 1] - rowptr[u];
  }
  int32_t* stamp = (int32_t*)calloc((size_t)maxdeg + 2, sizeof(int32_t));
  if (!keys || !stamp) {
    free(keys);
    free(stamp);
    return -1;
  }
  qsort(keys, (size_t)n, sizeof(uint64_t), gc_cmp_desc);
  int32_t ncolors = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t u = (int32_t)(keys[i] & 0xffffffffu);
    const int32_t deg = rowptr[u + 1] - rowptr[u];
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      const int32_t c = color[col[e]];
      if (c >= 0 && c <= deg) stamp[c] = i + 1;
    }
    int32_t c = 0;
    while (stamp[c] == i + 1) ++c;
    color[u] = c;
    if (c + 1 > ncolors) ncolors = c + 1;
  }
  free(keys);
  free(stamp);
  return ncolors;
}

/* ---- minimum spanning forest: MSTF / MSTV (no reference
 * implementation) ------------------------------------------------------------
 * Kruskal over the canonical slots (eid[e] == e) in increasing key =
 * (weight, eid) with a union-find: under that strict total order the minimum
 * spanning forest is unique, so it must equal the device's Boruvka forest
 * edge for edge.  in_mst[m] gets 1 at each forest edge's canonical slot.
 * Returns the number of forest edges (-1 on allocation failure). */
static uint64_t mst_key(int32_t w, int32_t e) {
  return ((uint64_t)((uint32_t)w ^ 0x80000000u) << 32) | (uint32_t)e;
}

static int u64_cmp(const void* a, const void* b) {
  const uint64_t ka = *(const uint64_t*)a, kb = *(const uint64_t*)b;
  return ka < kb ? -1 : (ka > kb ? 1 : 0);
}

static int32_t uf_find(int32_t* parent, int32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}

int64_t oracle_mst(const int32_t* rowptr, const int32_t* col,
                   const int32_t* weight, const int32_t* eid, int32_t n,
                   int64_t m, uint8_t* in_mst, int64_t* total_weight) {
  int64_t k = 0;
  for (int64_t e = 0; e < m; ++e) k += eid[e] == e;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(k ? k : 1));
  int32_t* src = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  if (!keys || !src || !parent) {
    free(keys);
    free(src);
    free(parent);
    return -1;
  }
  for (int32_t u = 0; u < n; ++u) {
    parent[u] = u;
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) src[e] = u;
  }
  k = 0;
  for (int64_t e = 0; e < m; ++e) {
    in_mst[e] = 0;
    if (eid[e] == e) keys[k++] = mst_key(weight[e], (int32_t)e);
  }
  qsort(keys, (size_t)k, sizeof(uint64_t), u64_cmp);
  int64_t nedges = 0, total = 0;
  for (int64_t i = 0; i < k; ++i) {
    const int32_t e = (int32_t)(keys[i] & 0xffffffffu);
    const int32_t a = uf_find(parent, src[e]), b = uf_find(parent, col[e]);
    if (a == b) continue;
    parent[a < b ? b : a] = a < b ? a : b;
    in_mst[e] = 1;
    total += weight[e];
    ++nedges;
  }
  *total_weight = total;
  free(keys);
  free(src);
  free(parent);
  return nedges;
}

/* ---- survey propagation on random k-SAT (no reference
 * implementation) -------------------------------------------------------------
 * Synchronous sweeps in the Braunstein-Mezard-Zecchina form: per variable the
 * products P_s = prod (1 - eta) over its positive / negative occurrences
 * (zero factors counted apart), then per edge (a, i)
 *   eta'[a,i] = prod_{j in a, j != i} Pu / (Pu + Ps + P0),
 *   S = P_s(j) / (1 - eta[a,j]), U = P_-s(j), Pu = (1-U)S, Ps = (1-S)U, P0 = SU.
 * fp64 arithmetic and surveys (no contraction: -ffp-contract=off), products
 * in ascending occurrence order.  Stops when max |eta' - eta| <= eps or after
 * max_sweeps; then the biases W+ / W- of every variable.  Returns sweeps. */
typedef struct {
  double p[2];
  int32_t z[2];
} sp_prod;

static void sp_var_pass(int32_t nvars, const int32_t* occ_row,
                        const int32_t* occ, const int32_t* lits,
                        const double* eta, sp_prod* prod, int nt) {
  /* one thread per variable, its occurrences in CSR order: the same
   * products whatever the thread count */
#pragma omp parallel for num_threads(nt) schedule(static, 1024)
  for (int32_t i = 0; i < nvars; ++i) {
    sp_prod q = {{1.0, 1.0}, {0, 0}};
    for (int32_t t = occ_row[i]; t < occ_row[i + 1]; ++t) {
      const int32_t e = occ[t];
      const int neg = lits[e] & 1;
      const double f = 1.0 - eta[e];
      if (f == 0.0)
        q.z[neg] += 1;
      else
        q.p[neg] *= f;
    }
    prod[i] = q;
  }
}

static double sp_ratio(const sp_prod* q, int neg, double eta_e) {
  const double f = 1.0 - eta_e;
  double S;
  if (f == 0.0)
    S = q->z[neg] - 1 == 0 ? q->p[neg] : 0.0;
  else
    S = q->z[neg] == 0 ? q->p[neg] / f : 0.0;
  const double U = q->z[neg ^ 1] == 0 ? q->p[neg ^ 1] : 0.0;
  const double pu = (1.0 - U) * S;
  const double ps = (1.0 - S) * U;
  const double p0 = S * U;
  const double den = (pu + ps) + p0;
  return den > 0.0 ? pu / den : 0.0;
}

/* double -> float rounded towards +inf (the device's __double2float_ru) */
static float sp_f32_up(double x) {
  float f = (float)x;
  if ((double)f < x) f = nextafterf(f, INFINITY);
  return f;
}

int32_t oracle_sp(const int32_t* lits, int32_t k, int32_t nclauses,
                  const int32_t* occ_row, const int32_t* occ, int32_t nvars,
                  const double* eta0, int32_t max_sweeps, float eps,
                  double* eta, float* wpos, float* wneg, float* last_delta,
                  int nthreads) {
  const int nt = nthr(nthreads);
  const int64_t ne = (int64_t)nclauses * k;
  sp_prod* prod = (sp_prod*)malloc(sizeof(sp_prod) * (size_t)(nvars ? nvars : 1));
  double* nxt = (double*)malloc(sizeof(double) * (size_t)(ne ? ne : 1));
  if (!prod || !nxt) {
    free(prod);
    free(nxt);
    return -1;
  }
  memcpy(eta, eta0, sizeof(double) * (size_t)ne);
  int32_t sweeps = 0;
  float delta = 0.f;
  while (sweeps < max_sweeps) {
    sp_var_pass(nvars, occ_row, occ, lits, eta, prod, nt);
    delta = 0.f;
    /* one thread per clause (synchronous sweep: reads eta, writes nxt) */
#pragma omp parallel for num_threads(nt) schedule(static, 1024) reduction(max : delta)
    for (int32_t a = 0; a < nclauses; ++a) {
      const int64_t base = (int64_t)a * k;
      for (int32_t t = 0; t < k; ++t) {
        double v = 1.0;
        for (int32_t j = 0; j < k; ++j) {
          if (j == t) continue;
          const int32_t l = lits[base + j];
          v *= sp_ratio(&prod[l >> 1], l & 1, eta[base + j]);
        }
        const float d = sp_f32_up(fabs(v - eta[base + t]));
        if (d > delta) delta = d;
        nxt[base + t] = v;
      }
    }
    memcpy(eta, nxt, sizeof(double) * (size_t)ne);
    ++sweeps;
    if (delta <= eps) break;
  }
  sp_var_pass(nvars, occ_row, occ, lits, eta, prod, nt);
  for (int32_t i = 0; i < nvars; ++i) {
    const double pp = prod[i].z[0] == 0 ? prod[i].p[0] : 0.0;
    const double pn = prod[i].z[1] == 0 ? prod[i].p[1] : 0.0;
    const double ip = (1.0 - pp) * pn, in = (1.0 - pn) * pp, i0 = pp * pn;
    const double den = (ip + in) + i0;
    wpos[i] = den > 0.0 ? (float)(ip / den) : 0.f;
    wneg[i] = den > 0.0 ? (float)(in / den) : 0.f;
  }
  if (last_delta) *last_delta = delta;
  free(prod);
  free(nxt);
  return sweeps;
}

/* ------------------------------------------------------------------------
 * RMAT generator (builder-defined input of BASELINE configs 3-5; the
 * reference has none).  Restates the product generator
 * (paper_2201_02789_b200/csrc/gen.cpp) independently so the reference arm and
 * the RMAT-26 parity check never load the product library: Graph500
 * quadrants (.57, .19, .19, .05) drawn bit by bit from the top level down,
 * each level's draw a 32-bit half of splitmix64(key ^ (16 e + level / 2)),
 * key = splitmix64(seed ^ "RMAT"); multi-edges and self-loops kept; rows
 * ascending when sort_rows (the BFS outputs do not depend on the row order,
 * so the RMAT-26 check may skip the sort).
 * ------------------------------------------------------------------------ */
static uint64_t sm64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static void rmat_pair(uint64_t key, int64_t e, int scale, int32_t* s,
                      int32_t* d) {
  /* quadrant thresholds floor(p * 2^32) for the cumulative a, a+b, a+b+c */
  const uint64_t ta = 2448131358ull, tab = 3264175144ull,
                 tabc = 4080218931ull;
  uint32_t src = 0, dst = 0;
  uint64_t h = 0;
  for (int l = 0; l < scale; ++l) {
    if (!(l & 1)) h = sm64(key ^ ((uint64_t)e * 16u + (uint64_t)(l / 2)));
    const uint64_t r = (l & 1) ? (h >> 32) : (h & 0xffffffffull);
    /* a: (0,0)  b: (0,1)  c: (1,0)  d: (1,1) */
    const uint32_t row_bit = r >= tab;
    const uint32_t col_bit = (r >= ta && r < tab) || r >= tabc;
    src = src * 2u + row_bit;
    dst = dst * 2u + col_bit;
  }
  *s = (int32_t)src;
  *d = (int32_t)dst;
}

static int i32_cmp(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

static void sort_row(int32_t* a, int64_t k) {
  if (k > 24) {
    qsort(a, (size_t)k, sizeof(int32_t), i32_cmp);
    return;
  }
  for (int64_t i = 1; i < k; ++i) { /* insertion sort for short rows */
    const int32_t x = a[i];
    int64_t j = i - 1;
    while (j >= 0 && a[j] > x) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = x;
  }
}

/* rowptr int32[2^scale + 1], col int32[edge_factor * 2^scale]; 0 or -1 */
int oracle_rmat_csr(int32_t scale, int32_t edge_factor, uint64_t seed,
                    int32_t* rowptr, int32_t* col, int sort_rows,
                    int nthreads) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
  const int64_t n = (int64_t)1 << scale, m = (int64_t)edge_factor * n;
  if (m > 0x7fffffffLL) return -1;
  const uint64_t key = sm64(seed ^ 0x524D4154ull);
  const int nt = nthr(nthreads);
  int64_t* fill = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!fill) return -1;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int32_t s, d;
    rmat_pair(key, e, scale, &s, &d);
    __atomic_fetch_add(&fill[s], 1, __ATOMIC_RELAXED);
  }
  int64_t run = 0;
  for (int64_t u = 0; u < n; ++u) { /* exclusive scan -> row starts */
    rowptr[u] = (int32_t)run;
    const int64_t c = fill[u];
    fill[u] = run;
    run += c;
  }
  rowptr[n] = (int32_t)run;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int32_t s, d;
    rmat_pair(key, e, scale, &s, &d);
    col[__atomic_fetch_add(&fill[s], 1, __ATOMIC_RELAXED)] = d;
  }
  free(fill);
  if (sort_rows) {
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
    for (int64_t u = 0; u < n; ++u)
      sort_row(col + rowptr[u], (int64_t)rowptr[u + 1] - rowptr[u]);
  }
  return 0;
}
