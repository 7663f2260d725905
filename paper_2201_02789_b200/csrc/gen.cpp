// gen.cpp — host-side input generation for the BASELINE configs that the
// reference has no generator for.
//
// RMAT: Graph500 quadrant probabilities (a, b, c, d) = (.57, .19, .19, .05),
// n = 2^scale vertices, m = edge_factor * n directed edges, no permutation,
// multi-edges and self-loops kept (the reference CSR keeps both too,
// bench/graphs.py:117-128), rows sorted ascending.  Randomness is a
// counter-based 64-bit mix of (seed, edge, level), so the graph is the same
// for any thread count and on any host; the quadrant draw compares 32-bit
// integers against integer thresholds (no floating point).
#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/dynpar.h"

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// floor(p * 2^32) for p = .57, .57+.19, .57+.19+.19
constexpr uint64_t kA = 2448131358ull;
constexpr uint64_t kAB = 3264175144ull;
constexpr uint64_t kABC = 4080218931ull;

inline void rmat_edge(uint64_t key, int64_t e, int scale, int32_t* src,
                      int32_t* dst) {
  uint32_t s = 0, d = 0;
  uint64_t h = 0;
  for (int l = 0; l < scale; ++l) {
    uint32_t r;
    if ((l & 1) == 0) {
      h = mix64(key ^ ((uint64_t)e * 16 + (uint64_t)(l >> 1)));
      r = (uint32_t)h;
    } else {
      r = (uint32_t)(h >> 32);
    }
    const uint32_t sb = r >= kAB;                   // quadrants c, d
    const uint32_t db = (r >= kA && r < kAB) || r >= kABC;  // b, d
    s = (s << 1) | sb;
    d = (d << 1) | db;
  }
  *src = (int32_t)s;
  *dst = (int32_t)d;
}

int threads_of(int32_t nthreads) {
  return nthreads > 0 ? nthreads : omp_get_max_threads();
}

}  // namespace

extern "C" {

int dp_rmat_csr(int32_t scale, int32_t edge_factor, uint64_t seed,
                int32_t* rowptr, int32_t* col, int32_t nthreads) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return DP_ERR_INVALID;
  const int64_t n = (int64_t)1 << scale;
  const int64_t m = (int64_t)edge_factor * n;
  if (m > 0x7fffffffLL) return DP_ERR_INVALID;  // int32 rowptr
  const uint64_t key = mix64(seed ^ 0x524D4154ull /* "RMAT" */);
  const int nt = threads_of(nthreads);
  std::vector<int32_t> cursor(n + 1, 0);
  // pass 1: out-degrees
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int32_t s, d;
    rmat_edge(key, e, scale, &s, &d);
    __atomic_fetch_add(&cursor[s + 1], 1, __ATOMIC_RELAXED);
  }
  rowptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) rowptr[i + 1] = rowptr[i] + cursor[i + 1];
  std::memcpy(cursor.data(), rowptr, sizeof(int32_t) * n);
  // pass 2: scatter targets, then sort each row (order-independent result)
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int32_t s, d;
    rmat_edge(key, e, scale, &s, &d);
    const int32_t pos = __atomic_fetch_add(&cursor[s], 1, __ATOMIC_RELAXED);
    col[pos] = d;
  }
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; ++u) std::sort(col + rowptr[u], col + rowptr[u + 1]);
  return 0;
}

int dp_rmat_csr_part(int32_t scale, int32_t edge_factor, uint64_t seed,
                     int32_t nparts, int32_t part, int32_t* rowptr_p,
                     int32_t* col_p, int64_t col_capacity, int64_t* m_p,
                     int32_t nthreads) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || nparts < 1 || part < 0 ||
      part >= nparts || !rowptr_p || !m_p)
    return DP_ERR_INVALID;
  const int64_t n = (int64_t)1 << scale;
  const int64_t m = (int64_t)edge_factor * n;
  const int64_t np_ = (n - part + nparts - 1) / nparts;  // owned: v % P == p
  const uint64_t key = mix64(seed ^ 0x524D4154ull);
  const int nt = threads_of(nthreads);
  std::vector<int64_t> cursor(np_ + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int32_t s, d;
    rmat_edge(key, e, scale, &s, &d);
    if (s % nparts == part)
      __atomic_fetch_add(&cursor[s / nparts + 1], 1, __ATOMIC_RELAXED);
  }
  int64_t acc = 0;
  rowptr_p[0] = 0;
  for (int64_t i = 0; i < np_; ++i) {
    acc += cursor[i + 1];
    if (acc > 0x7fffffffLL) return DP_ERR_INVALID;
    rowptr_p[i + 1] = (int32_t)acc;
  }
  *m_p = acc;
  if (!col_p) return 0;  // sizing call
  if (col_capacity < acc) return DP_ERR_INVALID;
  for (int64_t i = 0; i < np_; ++i) cursor[i] = rowptr_p[i];
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    int32_t s, d;
    rmat_edge(key, e, scale, &s, &d);
    if (s % nparts == part)
      col_p[__atomic_fetch_add(&cursor[s / nparts], 1, __ATOMIC_RELAXED)] = d;
  }
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1024)
  for (int64_t u = 0; u < np_; ++u)
    std::sort(col_p + rowptr_p[u], col_p + rowptr_p[u + 1]);
  return 0;
}

int dp_tc_orient(const int32_t* rowptr, const int32_t* col, int32_t n,
                 int32_t** rowptr_plus, int32_t** col_plus, int64_t* m_plus,
                 int32_t nthreads) {
  if (n < 0 || !rowptr_plus || !col_plus || !m_plus) return DP_ERR_INVALID;
  const int nt = threads_of(nthreads);
  // 1) symmetric adjacency without self-loops (duplicates still present)
  std::vector<int64_t> sp(n + 1, 0);
  std::vector<int64_t> cur(n + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u)
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      const int32_t v = col[e];
      if (v == u) continue;
      __atomic_fetch_add(&cur[u + 1], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&cur[v + 1], 1, __ATOMIC_RELAXED);
    }
  for (int64_t i = 0; i < n; ++i) sp[i + 1] = sp[i] + cur[i + 1];
  std::vector<int32_t> sym(sp[n]);
  for (int64_t i = 0; i < n; ++i) cur[i] = sp[i];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u)
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      const int32_t v = col[e];
      if (v == u) continue;
      sym[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
      sym[__atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED)] = (int32_t)u;
    }
  // 2) sort + dedup each row -> simple undirected degree
  std::vector<int32_t> deg(n, 0);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; ++u) {
    int32_t* b = sym.data() + sp[u];
    int32_t* e = sym.data() + sp[u + 1];
    std::sort(b, e);
    deg[u] = (int32_t)(std::unique(b, e) - b);
  }
  // 3) relabel by degree rank: rank(u) = position of u in ascending
  //    (deg u, u) order; the output vertex r = rank(u) keeps the edges to
  //    the higher-ranked neighbours, u -> v iff (deg u, u) < (deg v, v), now
  //    simply r(u) < r(v).  Rows ascending in the new ids, so the out-list
  //    of u past v's slot is exactly {w in N+(u) : w > v}, the only part
  //    that can close a triangle (u, v, w) at v -- TcApp probes that suffix.
  //    The triangle count is that of the input graph.
  std::vector<int32_t> order(n), rank(n);
  for (int64_t u = 0; u < n; ++u) order[u] = (int32_t)u;
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return deg[a] < deg[b] || (deg[a] == deg[b] && a < b);
  });
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = 0; i < n; ++i) rank[order[i]] = (int32_t)i;
  std::vector<int64_t> op(n + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u) {
    int64_t c = 0;
    for (int64_t i = sp[u]; i < sp[u] + deg[u]; ++i) c += rank[sym[i]] > rank[u];
    op[rank[u] + 1] = c;
  }
  for (int64_t i = 0; i < n; ++i) op[i + 1] += op[i];
  if (op[n] > 0x7fffffffLL) return DP_ERR_INVALID;
  int32_t* rp = (int32_t*)std::malloc(sizeof(int32_t) * (n + 1));
  int32_t* cp = (int32_t*)std::malloc(sizeof(int32_t) * std::max<int64_t>(op[n], 1));
  if (!rp || !cp) {
    std::free(rp);
    std::free(cp);
    return DP_ERR_INVALID;
  }
  for (int64_t i = 0; i <= n; ++i) rp[i] = (int32_t)op[i];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u) {
    const int32_t ru = rank[u];
    int64_t o = op[ru];
    for (int64_t i = sp[u]; i < sp[u] + deg[u]; ++i)
      if (rank[sym[i]] > ru) cp[o++] = rank[sym[i]];
    std::sort(cp + op[ru], cp + o);
  }
  *rowptr_plus = rp;
  *col_plus = cp;
  *m_plus = op[n];
  return 0;
}

int dp_symmetrize(const int32_t* rowptr, const int32_t* col, int32_t n,
                  int32_t** rowptr_s, int32_t** col_s, int64_t* m_s,
                  int32_t nthreads) {
  if (n < 0 || !rowptr_s || !col_s || !m_s) return DP_ERR_INVALID;
  const int nt = threads_of(nthreads);
  std::vector<int64_t> cur(n + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u)
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      const int32_t v = col[e];
      if (v == u) continue;
      __atomic_fetch_add(&cur[u + 1], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&cur[v + 1], 1, __ATOMIC_RELAXED);
    }
  std::vector<int64_t> sp(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) sp[i + 1] = sp[i] + cur[i + 1];
  std::vector<int32_t> sym(std::max<int64_t>(sp[n], 1));
  for (int64_t i = 0; i < n; ++i) cur[i] = sp[i];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u)
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      const int32_t v = col[e];
      if (v == u) continue;
      sym[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
      sym[__atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED)] = (int32_t)u;
    }
  std::vector<int64_t> deg(n + 1, 0);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; ++u) {
    int32_t* b = sym.data() + sp[u];
    int32_t* e = sym.data() + sp[u + 1];
    std::sort(b, e);
    deg[u + 1] = std::unique(b, e) - b;
  }
  for (int64_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
  if (deg[n] > 0x7fffffffLL) return DP_ERR_INVALID;
  int32_t* rp = (int32_t*)std::malloc(sizeof(int32_t) * (n + 1));
  int32_t* cp = (int32_t*)std::malloc(sizeof(int32_t) * std::max<int64_t>(deg[n], 1));
  if (!rp || !cp) {
    std::free(rp);
    std::free(cp);
    return DP_ERR_INVALID;
  }
  for (int64_t i = 0; i <= n; ++i) rp[i] = (int32_t)deg[i];
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096)
  for (int64_t u = 0; u < n; ++u)
    std::memcpy(cp + deg[u], sym.data() + sp[u],
                sizeof(int32_t) * (deg[u + 1] - deg[u]));
  *rowptr_s = rp;
  *col_s = cp;
  *m_s = deg[n];
  return 0;
}

// For a symmetric CSR with sorted rows and no duplicates: mirror[e] = the
// slot of (v, u) for the slot e of (u, v).  Returns DP_ERR_INVALID if some
// reverse edge is missing (the graph is not symmetric).
int dp_edge_mirror(const int32_t* rowptr, const int32_t* col, int32_t n,
                   int32_t* mirror, int32_t nthreads) {
  if (n < 0 || !mirror) return DP_ERR_INVALID;
  const int nt = threads_of(nthreads);
  int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4096) reduction(| : bad)
  for (int64_t u = 0; u < n; ++u)
    for (int32_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      const int32_t v = col[e];
      const int32_t* b = col + rowptr[v];
      const int32_t* f = col + rowptr[v + 1];
      const int32_t* p = std::lower_bound(b, f, (int32_t)u);
      if (p == f || *p != u) {
        bad = 1;
        mirror[e] = -1;
      } else {
        mirror[e] = (int32_t)(p - col);
      }
    }
  return bad ? DP_ERR_INVALID : 0;
}

void dp_free(void* p) { std::free(p); }

}  // extern "C"
