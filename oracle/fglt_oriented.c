/*
 * fglt_oriented.c — TEST INFRASTRUCTURE ONLY (parity checker for the sizes
 * the reference's own O(W) passes cannot reach, i.e. config 4 = R-MAT 23).
 *
 * Degree-oriented CPU restatements of the four W-cost terms of the
 * reference hot path. Each produces exactly the quantity the reference
 * function produces (the identities are SURVEY App. A; tests/test_oracle_pin.py
 * pins every function here bit-exact to the UNMODIFIED reference, oracle/_ref,
 * on R-MAT <= 14, SBM and RGG samples):
 *
 *   fglt_oriented_c3   C3 (nnz, aligned with ci) and c3
 *                      = proj/src/kernels.cpp:41-89 (compute_c3_C3)
 *   fglt_oriented_c4   c4 = kernels.cpp:109-147 (compute_c4_d14, c4 part);
 *                      d14 from C3: d14(i) = sum_{k in N(i)} C(C3(i,k),2)
 *   fglt_oriented_d13  d13(i) = sum over triangles {i,j,k} of (C3(j,k)-1)
 *                      = kernels.cpp:207-232 (compute_d13)
 *   fglt_oriented_d15  #4-cliques through i = kernels.cpp:234-288
 *
 * Method (NOT the reference's sparse-accumulator algorithm): vertices are
 * ranked by (degree, id) and the graph is relabelled by rank, so
 * N+(u) = the suffix of row u above u. Every triangle is listed once at its
 * lowest vertex u as an edge (x, y) inside S = N+(u) (marker array);
 * 4-cliques through u are the triangles of G[S] (bitmaps, popcount per G[S]
 * edge, credited to both ends); 4-cycles are counted once at their highest
 * vertex u by wedge counting L[w] = #{v < u : v ~ u, v ~ w}, w < u.
 * OpenMP, dynamic schedule, 64-bit atomics for cross-row credits.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef int64_t i64;
typedef int32_t i32;
typedef uint32_t u32;

typedef struct {
  i64 n;
  i64 *rp;   /* relabelled CSR, rows sorted ascending */
  i32 *ci;
  i32 *perm; /* perm[r] = original id of rank r */
  i32 *inv;  /* inv[v] = rank of original v */
} ranked_t;

static int cmp_i32(const void *a, const void *b) {
  i32 x = *(const i32 *)a, y = *(const i32 *)b;
  return (x > y) - (x < y);
}

static int cmp_key(const void *a, const void *b) {
  u64 x = *(const u64 *)a, y = *(const u64 *)b;
  return (x > y) - (x < y);
}

static void ranked_build(const i32 *rp, const i32 *ci, i64 n, ranked_t *g) {
  g->n = n;
  u64 *key = (u64 *)malloc(sizeof(u64) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(static)
  for (i64 v = 0; v < n; ++v) key[v] = ((u64)(rp[v + 1] - rp[v]) << 32) | (u64)v;
  qsort(key, (size_t)n, sizeof(u64), cmp_key);
  g->perm = (i32 *)malloc(sizeof(i32) * (size_t)(n > 0 ? n : 1));
  g->inv = (i32 *)malloc(sizeof(i32) * (size_t)(n > 0 ? n : 1));
  for (i64 r = 0; r < n; ++r) {
    g->perm[r] = (i32)(key[r] & 0xffffffffu);
    g->inv[g->perm[r]] = (i32)r;
  }
  free(key);
  g->rp = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
  g->rp[0] = 0;
  for (i64 r = 0; r < n; ++r) {
    i32 v = g->perm[r];
    g->rp[r + 1] = g->rp[r] + (rp[v + 1] - rp[v]);
  }
  g->ci = (i32 *)malloc(sizeof(i32) * (size_t)(g->rp[n] > 0 ? g->rp[n] : 1));
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 r = 0; r < n; ++r) {
    i32 v = g->perm[r];
    i64 w = g->rp[r];
    for (i64 a = rp[v]; a < rp[v + 1]; ++a) g->ci[w++] = g->inv[ci[a]];
    qsort(g->ci + g->rp[r], (size_t)(g->rp[r + 1] - g->rp[r]), sizeof(i32), cmp_i32);
  }
}

static void ranked_free(ranked_t *g) {
  free(g->rp); free(g->ci); free(g->perm); free(g->inv);
}

/* first position in row u holding an id > u */
static inline i64 up_start(const ranked_t *g, i64 u) {
  i64 lo = g->rp[u], hi = g->rp[u + 1];
  while (lo < hi) {
    i64 mid = lo + (hi - lo) / 2;
    if (g->ci[mid] <= (i32)u) lo = mid + 1; else hi = mid;
  }
  return lo;
}

static inline i64 find_pos(const i32 *ci, i64 lo, i64 hi, i32 key) {
  while (lo < hi) {
    i64 mid = lo + (hi - lo) / 2;
    if (ci[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

static inline void add64(u64 *p, u64 v) { if (v) __atomic_fetch_add(p, v, __ATOMIC_RELAXED); }

/* Triangle listing at the lowest vertex. For each triangle (u < x < y) the
 * callback gets the relabelled CSR positions of (u,x), (u,y), (x,y). */
#define FOR_TRIANGLES(G, UP, IDX, BODY)                                         \
  for (i64 u_ = 0; u_ < (G)->n; ++u_) {                                         \
    const i64 s0_ = (UP)[u_], s1_ = (G)->rp[u_ + 1];                           \
    if (s1_ - s0_ < 2) continue;                                                \
    for (i64 a_ = s0_; a_ < s1_; ++a_) (IDX)[(G)->ci[a_]] = a_;                 \
    for (i64 a_ = s0_; a_ < s1_; ++a_) {                                        \
      const i32 x_ = (G)->ci[a_];                                               \
      for (i64 b_ = (UP)[x_]; b_ < (G)->rp[x_ + 1]; ++b_) {                     \
        const i64 c_ = (IDX)[(G)->ci[b_]];                                      \
        if (c_ < 0) continue;                                                   \
        BODY(u_, a_, c_, b_)                                                    \
      }                                                                         \
    }                                                                           \
    for (i64 a_ = s0_; a_ < s1_; ++a_) (IDX)[(G)->ci[a_]] = -1;                 \
  }

static i64 *up_starts(const ranked_t *g) {
  i64 *up = (i64 *)malloc(sizeof(i64) * (size_t)(g->n > 0 ? g->n : 1));
#pragma omp parallel for schedule(static)
  for (i64 u = 0; u < g->n; ++u) up[u] = up_start(g, u);
  return up;
}

/* relabelled per-edge triangle counts (both orientations filled) */
static u32 *ranked_C3(const ranked_t *g, const i64 *up) {
  const i64 nnz = g->rp[g->n];
  u32 *C = (u32 *)calloc((size_t)(nnz > 0 ? nnz : 1), sizeof(u32));
#pragma omp parallel
  {
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)(g->n > 0 ? g->n : 1));
    for (i64 v = 0; v < g->n; ++v) idx[v] = -1;
#define C3_BODY(U, PUX, PUY, PXY)                              \
  __atomic_fetch_add(&C[PUX], 1u, __ATOMIC_RELAXED);           \
  __atomic_fetch_add(&C[PUY], 1u, __ATOMIC_RELAXED);           \
  __atomic_fetch_add(&C[PXY], 1u, __ATOMIC_RELAXED);
#pragma omp for schedule(dynamic, 64)
    FOR_TRIANGLES(g, up, idx, C3_BODY)
#undef C3_BODY
    free(idx);
  }
  /* mirror the canonical (upper) entries into the lower halves */
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 u = 0; u < g->n; ++u)
    for (i64 a = up[u]; a < g->rp[u + 1]; ++a) {
      const i32 x = g->ci[a];
      C[find_pos(g->ci, g->rp[x], up[x], (i32)u)] = C[a];
    }
  return C;
}

/* C3 (u64, aligned with the ORIGINAL ci) and c3 = row sum / 2 */
void fglt_oriented_c3(const i32 *rp, const i32 *ci, i64 n, u64 *c3, u64 *C3) {
  ranked_t g;
  ranked_build(rp, ci, n, &g);
  i64 *up = up_starts(&g);
  u32 *C = ranked_C3(&g, up);
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 v = 0; v < n; ++v) {
    const i64 r = g.inv[v];
    u64 s = 0;
    for (i64 k = rp[v]; k < rp[v + 1]; ++k) {
      const i64 p = find_pos(g.ci, g.rp[r], g.rp[r + 1], g.inv[ci[k]]);
      C3[k] = C[p];
      s += C[p];
    }
    c3[v] = s / 2;
  }
  free(C); free(up);
  ranked_free(&g);
}

/* d13(i) = sum over triangles {i,j,k} of (C3(j,k) - 1); C3 aligned with ci */
void fglt_oriented_d13(const i32 *rp, const i32 *ci, i64 n, const u64 *C3o, u64 *d13) {
  ranked_t g;
  ranked_build(rp, ci, n, &g);
  i64 *up = up_starts(&g);
  const i64 nnz = g.rp[n];
  u32 *C = (u32 *)malloc(sizeof(u32) * (size_t)(nnz > 0 ? nnz : 1));
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 v = 0; v < n; ++v) {
    const i64 r = g.inv[v];
    for (i64 k = rp[v]; k < rp[v + 1]; ++k)
      C[find_pos(g.ci, g.rp[r], g.rp[r + 1], g.inv[ci[k]])] = (u32)C3o[k];
  }
  u64 *acc = (u64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u64));
#pragma omp parallel
  {
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    for (i64 v = 0; v < n; ++v) idx[v] = -1;
#define D13_BODY(U, PUX, PUY, PXY)                 \
  add64(&acc[U], (u64)C[PXY] - 1);                 \
  add64(&acc[g.ci[PUX]], (u64)C[PUY] - 1);         \
  add64(&acc[g.ci[PUY]], (u64)C[PUX] - 1);
#pragma omp for schedule(dynamic, 64)
    FOR_TRIANGLES((&g), up, idx, D13_BODY)
#undef D13_BODY
    free(idx);
  }
#pragma omp parallel for schedule(static)
  for (i64 v = 0; v < n; ++v) d13[v] = acc[g.inv[v]];
  free(acc); free(C); free(up);
  ranked_free(&g);
}

/* c4 = #4-cycles through each vertex; d14 from C3 (aligned with ci).
 * Returns the reference's accumulator touch count, W - 2m. */
u64 fglt_oriented_c4_d14(const i32 *rp, const i32 *ci, i64 n, const u64 *C3o, u64 *c4,
                         u64 *d14) {
  ranked_t g;
  ranked_build(rp, ci, n, &g);
  u64 *acc = (u64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u64));
#pragma omp parallel
  {
    u32 *L = (u32 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u32));
    i32 *touched = (i32 *)malloc(sizeof(i32) * (size_t)(n > 0 ? n : 1));
#pragma omp for schedule(dynamic, 32)
    for (i64 u = 0; u < n; ++u) {
      i64 nt = 0;
      for (i64 a = g.rp[u]; a < g.rp[u + 1] && g.ci[a] < (i32)u; ++a) {
        const i32 v = g.ci[a];
        for (i64 b = g.rp[v]; b < g.rp[v + 1] && g.ci[b] < (i32)u; ++b) {
          const i32 w = g.ci[b];
          if (L[w]++ == 0) touched[nt++] = w;
        }
      }
      u64 cu = 0;
      for (i64 t = 0; t < nt; ++t) {
        const u64 l = L[touched[t]];
        const u64 c = l * (l - 1) / 2;
        cu += c;
        add64(&acc[touched[t]], c);
      }
      for (i64 a = g.rp[u]; a < g.rp[u + 1] && g.ci[a] < (i32)u; ++a) {
        const i32 v = g.ci[a];
        u64 s = 0;
        for (i64 b = g.rp[v]; b < g.rp[v + 1] && g.ci[b] < (i32)u; ++b) s += L[g.ci[b]] - 1;
        add64(&acc[v], s);
      }
      add64(&acc[u], cu);
      for (i64 t = 0; t < nt; ++t) L[touched[t]] = 0;
    }
    free(L); free(touched);
  }
  u64 W = 0, m2 = 0;
#pragma omp parallel for schedule(static) reduction(+ : W, m2)
  for (i64 v = 0; v < n; ++v) {
    c4[v] = acc[g.inv[v]];
    u64 s = 0;
    for (i64 k = rp[v]; k < rp[v + 1]; ++k) s += C3o[k] * (C3o[k] - (C3o[k] ? 1 : 0)) / 2;
    d14[v] = s;
    const u64 d = (u64)(rp[v + 1] - rp[v]);
    W += d * d;
    m2 += d;
  }
  free(acc);
  ranked_free(&g);
  return W - m2;
}

/* #4-cliques through each vertex: per root u, the triangles of G[N+(u)] from
 * adjacency bitmaps; each G[S] edge (a,b) adds popcount(row a & row b) to
 * both ends (every triangle of G[S] then credits each member twice). */
void fglt_oriented_d15(const i32 *rp, const i32 *ci, i64 n, u64 *d15) {
  ranked_t g;
  ranked_build(rp, ci, n, &g);
  i64 *up = up_starts(&g);
  i64 smax = 0;
  for (i64 u = 0; u < n; ++u) if (g.rp[u + 1] - up[u] > smax) smax = g.rp[u + 1] - up[u];
  u64 *acc = (u64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u64));
#pragma omp parallel
  {
    i64 *idx = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    for (i64 v = 0; v < n; ++v) idx[v] = -1;
    const i64 words = (smax + 63) / 64;
    u64 *bm = (u64 *)calloc((size_t)(smax > 0 ? smax : 1) * (size_t)(words > 0 ? words : 1), 8);
    u64 *t2 = (u64 *)calloc((size_t)(smax > 0 ? smax : 1), 8);
#pragma omp for schedule(dynamic, 16)
    for (i64 u = 0; u < n; ++u) {
      const i64 s0 = up[u], s = g.rp[u + 1] - s0;
      if (s < 3) continue;
      const i64 wd = (s + 63) / 64;
      for (i64 a = 0; a < s; ++a) idx[g.ci[s0 + a]] = a;
      int any = 0;
      for (i64 a = 0; a < s; ++a) {
        const i32 x = g.ci[s0 + a];
        for (i64 b = up[x]; b < g.rp[x + 1]; ++b) {
          const i64 c = idx[g.ci[b]];
          if (c < 0) continue;
          bm[a * wd + (c >> 6)] |= 1ull << (c & 63);
          bm[c * wd + (a >> 6)] |= 1ull << (a & 63);
          any = 1;
        }
      }
      if (any) {
        u64 tot = 0;
        for (i64 a = 0; a < s; ++a) {
          const u64 *ra = bm + a * wd;
          for (i64 w = (a + 1) >> 6; w < wd; ++w) {
            u64 bits = ra[w];
            if (w == ((a + 1) >> 6)) bits &= ~0ull << ((a + 1) & 63);
            while (bits) {
              const i64 b = w * 64 + __builtin_ctzll(bits);
              bits &= bits - 1;
              const u64 *rb = bm + b * wd;
              u64 p = 0;
              for (i64 k = 0; k < wd; ++k) p += (u64)__builtin_popcountll(ra[k] & rb[k]);
              t2[a] += p;
              t2[b] += p;
              tot += p;
            }
          }
        }
        for (i64 a = 0; a < s; ++a) {
          add64(&acc[g.ci[s0 + a]], t2[a] / 2);
          t2[a] = 0;
        }
        add64(&acc[u], tot / 3);
        memset(bm, 0, sizeof(u64) * (size_t)(s * wd));
      }
      for (i64 a = 0; a < s; ++a) idx[g.ci[s0 + a]] = -1;
    }
    free(idx); free(bm); free(t2);
  }
#pragma omp parallel for schedule(static)
  for (i64 v = 0; v < n; ++v) d15[v] = acc[g.inv[v]];
  free(acc); free(up);
  ranked_free(&g);
}
