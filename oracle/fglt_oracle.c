/*
 * fglt_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C, CPU restatement of the reference Fast Graphlet Transform hot
 * path (arxiv 2007.11111, reference tree /root/reference/proj). It is linked
 * into oracle/liboracle.so and loaded ONLY by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg, always as the checker, never as the thing
 * measured or shipped. The product path (paper_2007_11111_b200) never loads it.
 *
 * Pinning: tests/test_oracle_pin.py checks every function here against the
 * golden vectors the reference's own tests hold (Fig. 2 tables,
 * proj/tests/testutil.hpp:40-62; per-kernel KATs, proj/tests/test_kernels.cpp)
 * and against the compiled reference itself (oracle/_ref/libfglt_ref.so built
 * from the unmodified sources by oracle/Makefile).
 *
 * Arithmetic contract (proj/include/graphlet/types.hpp:59-94): all counts are
 * uint64; `sat_sub` is the rectified difference; the overflow-checked sites
 * are exactly the reference's `checked_add/checked_mul/choose2/choose3`
 * sites; everything else wraps mod 2^64 as unchecked C++ uint64 does.
 *
 * Error semantics: the reference throws the first exception raised; with one
 * thread that is the lowest vertex of the first failing column in fill order
 * (proj/src/kernels.cpp:384-412), then the lowest vertex of net_from_raw's
 * walk (proj/src/conversion.cpp:88-113). This restatement reports exactly
 * that (deterministic for any OpenMP thread count).
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

enum { OK = 0, E_STRUCT = 2, E_OVERFLOW = 3, E_INCONSIST = 4, E_NOMEM = 6 };

/* ---------------------------------------------------------------- arithmetic
 * proj/include/graphlet/types.hpp:59-94 */
static inline u64 sat_sub(u64 a, u64 b) { return a > b ? a - b : 0; }
/* Returns 1 on overflow (reference: throws OverflowError). */
static inline int add_ov(u64 a, u64 b, u64 *r) { return __builtin_add_overflow(a, b, r); }
static inline int mul_ov(u64 a, u64 b, u64 *r) { return __builtin_mul_overflow(a, b, r); }
/* choose2: checked d*(d-1), then /2 (types.hpp:84-88) */
static inline int choose2_ov(u64 d, u64 *r) {
  if (d < 2) { *r = 0; return 0; }
  u64 t;
  if (mul_ov(d, d - 1, &t)) return 1;
  *r = t / 2;
  return 0;
}
/* choose3: unchecked d(d-1)/2, checked *(d-2), then /3 (types.hpp:91-94) */
static inline int choose3_ov(u64 d, u64 *r) {
  if (d < 3) { *r = 0; return 0; }
  u64 t;
  if (mul_ov(d * (d - 1) / 2, d - 2, &t)) return 1;
  *r = t / 3;
  return 0;
}

/* ----------------------------------------------------------- error tracking
 * A failure is ordered by (stage, vertex); the smallest wins, matching the
 * single-threaded reference. `graphlet` is whatever the reference would name
 * for that vertex. */
typedef struct {
  u64 key; /* (stage << 40) | vertex ; UINT64_MAX = none */
  int code;
  int graphlet;
} err_t;

static void err_init(err_t *e) { e->key = UINT64_MAX; e->code = OK; e->graphlet = -1; }
static void err_offer(err_t *e, int stage, i64 v, int code, int graphlet) {
  u64 key = ((u64)stage << 40) | (u64)v;
#pragma omp critical(fglt_oracle_err)
  {
    if (key < e->key) { e->key = key; e->code = code; e->graphlet = graphlet; }
  }
}

/* ------------------------------------------------------------------- kernels */

/* p1 = A e (proj/src/graph.cpp:251-256) */
void fglt_oracle_p1(const i32 *rp, i64 n, u64 *p1) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) p1[i] = (u64)(rp[i + 1] - rp[i]);
}

/* p2(i) = sat_sub(sum_{j in N(i)} p1[j], p1[i]) (proj/src/kernels.cpp:26-39) */
void fglt_oracle_p2(const i32 *rp, const i32 *ci, i64 n, const u64 *p1, u64 *p2) {
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 i = 0; i < n; ++i) {
    u64 acc = 0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) acc += p1[ci[k]];
    p2[i] = sat_sub(acc, p1[i]);
  }
}

/* fglt_oriented.c */
void fglt_oriented_c3(const i32 *rp, const i32 *ci, i64 n, u64 *c3, u64 *C3);
void fglt_oriented_d13(const i32 *rp, const i32 *ci, i64 n, const u64 *C3, u64 *d13);
u64 fglt_oriented_c4_d14(const i32 *rp, const i32 *ci, i64 n, const u64 *C3, u64 *c4, u64 *d14);
void fglt_oriented_d15(const i32 *rp, const i32 *ci, i64 n, u64 *d15);

static i64 lower_bound_i32(const i32 *a, i64 lo, i64 hi, i32 key) {
  while (lo < hi) {
    i64 mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* C3(i,j) = |N(i) ∩ N(j)| on the adjacency pattern by sorted merge for each
 * edge i<j, mirrored into (j,i); c3 = row sum / 2
 * (proj/src/kernels.cpp:41-89). C3 is aligned with ci (nnz entries). */
void fglt_oracle_c3(const i32 *rp, const i32 *ci, i64 n, u64 *c3, u64 *C3) {
#pragma omp parallel for schedule(dynamic, 64)
  for (i64 i = 0; i < n; ++i) {
    for (i64 a = rp[i]; a < rp[i + 1]; ++a) {
      i32 j = ci[a];
      if (j < i) continue;
      i64 x = rp[i], xe = rp[i + 1], y = rp[j], ye = rp[j + 1];
      u64 common = 0;
      while (x < xe && y < ye) {
        if (ci[x] == ci[y]) { ++common; ++x; ++y; }
        else if (ci[x] < ci[y]) ++x;
        else ++y;
      }
      C3[a] = common;
      C3[lower_bound_i32(ci, rp[j], rp[j + 1], (i32)i)] = common;
    }
  }
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) {
    u64 s = 0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) s += C3[k];
    c3[i] = s / 2;
  }
}

/* p3(i) = sat_sub(sum_j p2[j], p1*sat_sub(p1,1) + 2 c3) (kernels.cpp:91-107) */
void fglt_oracle_p3(const i32 *rp, const i32 *ci, i64 n, const u64 *p1,
                    const u64 *p2, const u64 *c3, u64 *p3) {
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 i = 0; i < n; ++i) {
    u64 walk = 0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) walk += p2[ci[k]];
    p3[i] = sat_sub(walk, p1[i] * sat_sub(p1[i], 1) + 2 * c3[i]);
  }
}

/* Fused two-path-row pass: the row P2(i,·) is accumulated in a dense
 * per-thread scratch with a touched list; c4 = sum_k C(P2(i,k),2) over all k,
 * d14 = the same sum restricted to k in N(i); touches = number of adds
 * (proj/src/kernels.cpp:109-147). Returns total touches. */
u64 fglt_oracle_c4_d14(const i32 *rp, const i32 *ci, i64 n, u64 *c4, u64 *d14) {
  u64 touches = 0;
#pragma omp parallel reduction(+ : touches)
  {
    u64 *val = (u64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u64));
    i32 *touched = (i32 *)malloc(sizeof(i32) * (size_t)(n > 0 ? n : 1));
    uint32_t *mark = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    uint32_t epoch = 0;
#pragma omp for schedule(dynamic, 16)
    for (i64 i = 0; i < n; ++i) {
      i64 nt = 0;
      for (i64 a = rp[i]; a < rp[i + 1]; ++a) {
        i32 j = ci[a];
        for (i64 b = rp[j]; b < rp[j + 1]; ++b) {
          i32 k = ci[b];
          if (k == i) continue;
          ++touches;
          if (val[k] == 0) touched[nt++] = k;
          val[k] += 1;
        }
      }
      ++epoch;
      for (i64 a = rp[i]; a < rp[i + 1]; ++a) mark[ci[a]] = epoch;
      u64 c4i = 0, d14i = 0;
      for (i64 t = 0; t < nt; ++t) {
        i32 k = touched[t];
        u64 v = val[k];
        u64 pairs = v * (v - 1) / 2;
        c4i += pairs;
        if (mark[k] == epoch) d14i += pairs;
        val[k] = 0;
      }
      c4[i] = c4i;
      d14[i] = d14i;
    }
    free(val); free(touched); free(mark);
  }
  return touches;
}

/* d13(i) = (1/2) sum_{j in N(i)} sum_{k in N(j) ∩ N(i)} sat_sub(C3(j,k),1)
 * (proj/src/kernels.cpp:207-232) */
void fglt_oracle_d13(const i32 *rp, const i32 *ci, i64 n, const u64 *C3, u64 *d13) {
#pragma omp parallel
  {
    uint32_t *mark = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    uint32_t epoch = 0;
#pragma omp for schedule(dynamic, 16)
    for (i64 i = 0; i < n; ++i) {
      ++epoch;
      for (i64 a = rp[i]; a < rp[i + 1]; ++a) mark[ci[a]] = epoch;
      u64 total = 0;
      for (i64 a = rp[i]; a < rp[i + 1]; ++a) {
        i32 j = ci[a];
        for (i64 b = rp[j]; b < rp[j + 1]; ++b)
          if (mark[ci[b]] == epoch) total += sat_sub(C3[b], 1);
      }
      d13[i] = total / 2;
    }
    free(mark);
  }
}

/* d15: per edge i<j, q = N(i) ∩ N(j); t = number of ordered adjacent pairs in
 * q; add t to i and j; d15 = sum / 6 (proj/src/kernels.cpp:234-288). Exact
 * but pathological on power-law graphs (it is the reference's own cost). */
void fglt_oracle_d15_ref_algorithm(const i32 *rp, const i32 *ci, i64 n, u64 *d15) {
  memset(d15, 0, sizeof(u64) * (size_t)n);
#pragma omp parallel
  {
    u64 *sums = (u64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u64));
    uint32_t *mi = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    uint32_t *mq = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    i32 *q = (i32 *)malloc(sizeof(i32) * (size_t)(n > 0 ? n : 1));
    uint32_t ei = 0, eq = 0;
#pragma omp for schedule(dynamic, 16)
    for (i64 i = 0; i < n; ++i) {
      ++ei;
      for (i64 a = rp[i]; a < rp[i + 1]; ++a) mi[ci[a]] = ei;
      for (i64 a = rp[i]; a < rp[i + 1]; ++a) {
        i32 j = ci[a];
        if (j <= i) continue;
        i64 nq = 0;
        for (i64 b = rp[j]; b < rp[j + 1]; ++b)
          if (mi[ci[b]] == ei) q[nq++] = ci[b];
        if (nq < 2) continue;
        ++eq;
        for (i64 t = 0; t < nq; ++t) mq[q[t]] = eq;
        u64 t2 = 0;
        for (i64 t = 0; t < nq; ++t) {
          i32 k = q[t];
          if ((i64)(rp[k + 1] - rp[k]) <= nq) {
            for (i64 b = rp[k]; b < rp[k + 1]; ++b)
              if (mq[ci[b]] == eq) ++t2;
          } else {
            for (i64 s = 0; s < nq; ++s) {
              i32 l = q[s];
              if (l == k) continue;
              i64 p = lower_bound_i32(ci, rp[k], rp[k + 1], l);
              if (p < rp[k + 1] && ci[p] == l) ++t2;
            }
          }
        }
        sums[i] += t2;
        sums[j] += t2;
      }
    }
#pragma omp critical(fglt_oracle_d15)
    for (i64 v = 0; v < n; ++v) d15[v] += sums[v];
    free(sums); free(mi); free(mq); free(q);
  }
  for (i64 v = 0; v < n; ++v) d15[v] /= 6;
}

/* Independent per-vertex 4-clique counter (NOT the reference's algorithm):
 * orient every edge from lower to higher (degree, id); for each vertex u and
 * each out-neighbour v, W = N+(u) ∩ N+(v); every edge inside W closes one K4,
 * credited to its four vertices. Pinned bit-exact against the reference's
 * compute_d15 (tests/test_oracle_pin.py) and used for d15 parity where the
 * reference's own algorithm is out of reach. */
static inline int fwd(const i32 *rp, i32 a, i32 b) {
  i32 da = rp[a + 1] - rp[a], db = rp[b + 1] - rp[b];
  return da < db || (da == db && a < b);
}
void fglt_oracle_d15_oriented(const i32 *rp, const i32 *ci, i64 n, u64 *d15) {
  /* forward adjacency, sorted by id */
  i64 *orp = (i64 *)malloc(sizeof(i64) * (size_t)(n + 1));
  orp[0] = 0;
  for (i64 u = 0; u < n; ++u) {
    i64 c = 0;
    for (i64 a = rp[u]; a < rp[u + 1]; ++a) c += fwd(rp, (i32)u, ci[a]);
    orp[u + 1] = orp[u] + c;
  }
  i32 *oci = (i32 *)malloc(sizeof(i32) * (size_t)(orp[n] > 0 ? orp[n] : 1));
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 u = 0; u < n; ++u) {
    i64 w = orp[u];
    for (i64 a = rp[u]; a < rp[u + 1]; ++a)
      if (fwd(rp, (i32)u, ci[a])) oci[w++] = ci[a];
  }
  memset(d15, 0, sizeof(u64) * (size_t)n);
#pragma omp parallel
  {
    u64 *loc = (u64 *)calloc((size_t)(n > 0 ? n : 1), sizeof(u64));
    uint32_t *mw = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    uint32_t *mu = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    i32 *W = (i32 *)malloc(sizeof(i32) * (size_t)(n > 0 ? n : 1));
    uint32_t eu = 0, ew = 0;
#pragma omp for schedule(dynamic, 8)
    for (i64 u = 0; u < n; ++u) {
      ++eu;
      for (i64 a = orp[u]; a < orp[u + 1]; ++a) mu[oci[a]] = eu;
      u64 ku = 0;
      for (i64 a = orp[u]; a < orp[u + 1]; ++a) {
        i32 v = oci[a];
        i64 nw = 0;
        ++ew;
        for (i64 b = orp[v]; b < orp[v + 1]; ++b)
          if (mu[oci[b]] == eu) { W[nw++] = oci[b]; mw[oci[b]] = ew; }
        u64 kv = 0;
        for (i64 t = 0; t < nw; ++t) {
          i32 w = W[t];
          for (i64 b = orp[w]; b < orp[w + 1]; ++b) {
            i32 x = oci[b];
            if (mw[x] == ew) { ++kv; loc[w] += 1; loc[x] += 1; }
          }
        }
        ku += kv;
        loc[v] += kv;
      }
      loc[u] += ku;
    }
#pragma omp critical(fglt_oracle_k4)
    for (i64 v = 0; v < n; ++v) d15[v] += loc[v];
    free(loc); free(mw); free(mu); free(W);
  }
  free(orp); free(oci);
}

/* d7(i) = sum_j choose2(sat_sub(p1[j],1)), checked (kernels.cpp:149-163) */
static void d7_into(const i32 *rp, const i32 *ci, i64 n, const u64 *p1, u64 *d7,
                    err_t *err, int stage) {
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 i = 0; i < n; ++i) {
    u64 acc = 0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
      u64 c;
      if (choose2_ov(sat_sub(p1[ci[k]], 1), &c) || add_ov(acc, c, &acc)) {
        err_offer(err, stage, i, E_OVERFLOW, 7);
        break;
      }
    }
    d7[i] = acc;
  }
}

/* d9 = sat_sub(sum_j c3[j] (checked), 2c3); d10 = sum_j C3(i,j)*sat_sub(p1[j],2)
 * (checked); d11 = sat_sub(p1,2)*c3 (checked) (kernels.cpp:176-205) */
static void dippers_into(const i32 *rp, const i32 *ci, i64 n, const u64 *p1,
                         const u64 *c3, const u64 *C3, u64 *d9, u64 *d10,
                         u64 *d11, err_t *err, int stage) {
#pragma omp parallel for schedule(dynamic, 256)
  for (i64 i = 0; i < n; ++i) {
    u64 nt = 0, base = 0;
    int bad = 0;
    for (i64 k = rp[i]; k < rp[i + 1] && !bad; ++k) {
      i32 j = ci[k];
      if (add_ov(nt, c3[j], &nt)) { err_offer(err, stage, i, E_OVERFLOW, 9); bad = 1; break; }
      u64 t;
      if (mul_ov(C3[k], sat_sub(p1[j], 2), &t) || add_ov(base, t, &base)) {
        err_offer(err, stage, i, E_OVERFLOW, 10); bad = 1; break;
      }
    }
    if (bad) continue;
    d9[i] = sat_sub(nt, 2 * c3[i]);
    d10[i] = base;
    if (mul_ov(sat_sub(p1[i], 2), c3[i], &d11[i])) err_offer(err, stage, i, E_OVERFLOW, 11);
  }
}

/* ---------------------------------------------------------------- conversion
 * U16, rows = raw graphlet, cols = net graphlet: PAPER.md Table 2 as encoded
 * in proj/src/conversion.cpp:14-32 (restated here). */
static const unsigned char U16[16][16] = {
    {1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {0, 0, 1, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {0, 0, 0, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
    {0, 0, 0, 0, 0, 1, 0, 0, 0, 2, 1, 0, 2, 4, 2, 6},
    {0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 1, 2, 2, 2, 4, 6},
    {0, 0, 0, 0, 0, 0, 0, 1, 0, 1, 1, 0, 0, 2, 1, 3},
    {0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 1, 1},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 2, 0, 3},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 2, 2, 6},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 2, 3},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 3},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 3},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 3},
    {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1},
};

void fglt_oracle_u16(uint64_t *out256) {
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 16; ++c) out256[r * 16 + c] = U16[r][c];
}

static int ids_of(uint32_t mask, int *ids) {
  mask |= 3u; /* {0,1} always present (proj/src/dictionary.cpp:38-50) */
  int k = 0;
  for (int i = 0; i < 16; ++i)
    if (mask & (1u << i)) ids[k++] = i;
  return k;
}

/* Per-vertex exact back-substitution with U(s,s) (conversion.cpp:80-116).
 * raw/net are n x k row-major. */
static void net_into(const u64 *raw, u64 *net, i64 n, const int *ids, int k,
                     int lenient, err_t *err, int stage) {
#pragma omp parallel for schedule(static)
  for (i64 v = 0; v < n; ++v) {
    const u64 *in = raw + (size_t)v * k;
    u64 *out = net + (size_t)v * k;
    for (int r = k - 1; r >= 0; --r) {
      u64 absorbed = 0;
      int bad = 0;
      for (int c = r + 1; c < k; ++c) {
        u64 coef = U16[ids[r]][ids[c]], t;
        if (!coef) continue;
        if (mul_ov(coef, out[c], &t) || add_ov(absorbed, t, &absorbed)) {
          err_offer(err, stage, v, E_OVERFLOW, ids[r]);
          bad = 1;
          break;
        }
      }
      if (bad) break;
      if (absorbed > in[r]) {
        if (!lenient) { err_offer(err, stage, v, E_INCONSIST, ids[r]); break; }
        out[r] = 0;
      } else {
        out[r] = in[r] - absorbed;
      }
    }
  }
}

void fglt_oracle_net_from_raw(const u64 *raw, u64 *net, i64 n, uint32_t dict_mask,
                              int lenient, int32_t *err_graphlet, int64_t *err_vertex,
                              int *code) {
  int ids[16];
  int k = ids_of(dict_mask, ids);
  err_t err;
  err_init(&err);
  net_into(raw, net, n, ids, k, lenient, &err, 0);
  *code = err.code;
  if (err.code) { *err_graphlet = err.graphlet; *err_vertex = (i64)(err.key & ((1ull << 40) - 1)); }
}

/* ------------------------------------------------------------ full transform
 * Plan (proj/src/dictionary.cpp:143-158) then column fill
 * (proj/src/kernels.cpp:384-412), then net (proj/src/transform.cpp:9-26).
 * d15_mode: 0 = the reference's own algorithm, 1 = the independent oriented
 * K4 counter (pinned equal; used at sizes the former cannot reach), 2 = every
 * W-cost term (C3, c4/d14, d13, d15) from the degree-oriented restatements of
 * fglt_oriented.c (pinned equal; the only mode that finishes at R-MAT 23).
 * Returns 0 or the reference CLI exit class (tools/glt.cpp:17-21). */
int fglt_oracle_transform(const i32 *rp, const i32 *ci, i64 n, uint32_t dict_mask,
                          int lenient, int d15_mode, u64 *raw, u64 *net,
                          int32_t *err_graphlet, int64_t *err_vertex,
                          u64 *touches_out) {
  int ids[16], pos[16];
  int k = ids_of(dict_mask, ids);
  const int oriented = d15_mode == 2;
  uint32_t m = 0;
  for (int i = 0; i < 16; ++i) pos[i] = -1;
  for (int t = 0; t < k; ++t) { pos[ids[t]] = t; m |= 1u << ids[t]; }
#define HAS(id) ((m >> (id)) & 1u)
#define ANY(mask) ((m & (mask)) != 0)
  const i64 nnz = rp[n];
  size_t nv = (size_t)(n > 0 ? n : 1);
  u64 *p1 = calloc(nv, 8), *p2 = calloc(nv, 8), *p3 = calloc(nv, 8), *c3 = calloc(nv, 8);
  u64 *c4 = calloc(nv, 8), *d14 = calloc(nv, 8), *d13 = calloc(nv, 8), *d15 = calloc(nv, 8);
  u64 *d7 = calloc(nv, 8), *d9 = calloc(nv, 8), *d10 = calloc(nv, 8), *d11 = calloc(nv, 8);
  u64 *C3 = calloc((size_t)(nnz > 0 ? nnz : 1), 8);
  err_t err;
  err_init(&err);
  if (touches_out) *touches_out = 0;

  fglt_oracle_p1(rp, n, p1);
  const uint32_t tri_cols =
      (1u << 4) | (1u << 5) | (1u << 6) | (1u << 9) | (1u << 10) | (1u << 11) | (1u << 13);
  if (oriented) {
    if (ANY(tri_cols | (1u << 14))) fglt_oriented_c3(rp, ci, n, c3, C3);
  } else if (ANY(tri_cols)) {
    fglt_oracle_c3(rp, ci, n, c3, C3);
  }
  if (ANY((1u << 2) | (1u << 5) | (1u << 6))) fglt_oracle_p2(rp, ci, n, p1, p2);
  if (HAS(5)) fglt_oracle_p3(rp, ci, n, p1, p2, c3, p3);
  if (ANY((1u << 12) | (1u << 14))) {
    u64 t = oriented ? fglt_oriented_c4_d14(rp, ci, n, C3, c4, d14)
                     : fglt_oracle_c4_d14(rp, ci, n, c4, d14);
    if (touches_out) *touches_out = t;
  }
  if (HAS(13)) {
    if (oriented) fglt_oriented_d13(rp, ci, n, C3, d13);
    else fglt_oracle_d13(rp, ci, n, C3, d13);
  }
  if (HAS(15)) {
    if (oriented) fglt_oriented_d15(rp, ci, n, d15);
    else if (d15_mode) fglt_oracle_d15_oriented(rp, ci, n, d15);
    else fglt_oracle_d15_ref_algorithm(rp, ci, n, d15);
  }

  /* column fill, in the reference's order; stage numbers order the errors */
  if (HAS(3)) {
#pragma omp parallel for schedule(static)
    for (i64 v = 0; v < n; ++v) {
      u64 r;
      if (choose2_ov(p1[v], &r)) err_offer(&err, 1, v, E_OVERFLOW, 3);
    }
  }
  if (HAS(6)) {
#pragma omp parallel for schedule(static)
    for (i64 v = 0; v < n; ++v) {
      u64 r;
      if (mul_ov(p2[v], sat_sub(p1[v], 1), &r)) err_offer(&err, 2, v, E_OVERFLOW, 6);
    }
  }
  if (HAS(7)) d7_into(rp, ci, n, p1, d7, &err, 3);
  if (HAS(8)) {
#pragma omp parallel for schedule(static)
    for (i64 v = 0; v < n; ++v) {
      u64 r;
      if (choose3_ov(p1[v], &r)) err_offer(&err, 4, v, E_OVERFLOW, 8);
    }
  }
  if (ANY((1u << 9) | (1u << 10) | (1u << 11)))
    dippers_into(rp, ci, n, p1, c3, C3, d9, d10, d11, &err, 5);

  int code = OK;
  if (err.code == OK) {
#pragma omp parallel for schedule(static)
    for (i64 v = 0; v < n; ++v) {
      u64 col[16], r;
      col[0] = 1;
      col[1] = p1[v];
      col[2] = p2[v];
      col[3] = choose2_ov(p1[v], &r) ? 0 : r;
      col[4] = c3[v];
      col[5] = p3[v];
      col[6] = sat_sub(p2[v] * sat_sub(p1[v], 1), 2 * c3[v]);
      col[7] = d7[v];
      col[8] = choose3_ov(p1[v], &r) ? 0 : r;
      col[9] = d9[v];
      col[10] = d10[v];
      col[11] = d11[v];
      col[12] = c4[v];
      col[13] = d13[v];
      col[14] = d14[v];
      col[15] = d15[v];
      for (int t = 0; t < k; ++t) raw[(size_t)v * k + t] = col[ids[t]];
    }
    net_into(raw, net, n, ids, k, lenient, &err, 6);
  }
  code = err.code;
  if (code) {
    *err_graphlet = err.graphlet;
    *err_vertex = (i64)(err.key & ((1ull << 40) - 1));
  }
  free(p1); free(p2); free(p3); free(c3); free(c4); free(d14); free(d13); free(d15);
  free(d7); free(d9); free(d10); free(d11); free(C3);
  (void)pos;
  return code;
#undef HAS
#undef ANY
}

/* Whole-graph figures for the roofline model: W = sum_v d_v^2,
 * d_max. */
void fglt_oracle_graph_stats(const i32 *rp, i64 n, u64 *W, u64 *dmax) {
  u64 w = 0, dm = 0;
#pragma omp parallel for reduction(+ : w) reduction(max : dm)
  for (i64 v = 0; v < n; ++v) {
    u64 d = (u64)(rp[v + 1] - rp[v]);
    w += d * d;
    if (d > dm) dm = d;
  }
  *W = w;
  *dmax = dm;
}

int fglt_oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
