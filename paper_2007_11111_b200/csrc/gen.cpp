// Seeded synthetic workload generators for the five BASELINE.json configs and
// the host-side CSR sanitiser. Host C++ (OpenMP); no CUDA.
//
// Every generator emits an undirected edge sample that goes through
// fglt_build_csr32 (symmetrise, drop self-loops, dedupe, sorted rows), the
// same sanitising contract as the reference's build_adjacency
// (proj/src/graph.cpp:192-249). The CSR is canonical, so any correct builder
// (this one, the GPU ingest kernel, the reference's) yields identical bytes.
//
// Randomness: er_graph reproduces the reference's own test generator exactly
// (std::mt19937_64 + std::bernoulli_distribution over u<v in lexicographic
// order, proj/tests/testutil.hpp:90-99), which pins config 1. The large
// configs use a counter-based splitmix64 stream so that generation is
// embarrassingly parallel and identical for any thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// Counter-based stream: value #ctr of stream (seed, tag).
inline uint64_t rnd(uint64_t seed, uint64_t tag, uint64_t ctr) {
  return mix64(mix64(seed * 0x9e3779b97f4a7c15ULL + tag) + ctr * 0x9e3779b97f4a7c15ULL);
}
inline double unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

struct Edges {
  std::vector<int64_t> u, v;
};

}  // namespace

extern "C" {

// ----------------------------------------------------------------- CSR build
// Sanitise an undirected sample into a symmetric CSR with strictly increasing
// rows and no diagonal. rp_out holds n+1 entries, ci_out at least 2*ne
// (an upper bound on nnz). Returns nnz.
int64_t fglt_build_csr32(const int64_t* eu, const int64_t* ev, int64_t ne,
                         int64_t n, int32_t* rp_out, int32_t* ci_out,
                         int64_t* self_loops, int64_t* dup_merged) {
  std::vector<int64_t> cnt((size_t)n + 1, 0);
  std::atomic<int64_t> loops{0};
  {
    std::vector<std::atomic<int64_t>> c((size_t)n);
    for (auto& x : c) x.store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < ne; ++k) {
      if (eu[k] == ev[k]) { loops.fetch_add(1, std::memory_order_relaxed); continue; }
      c[eu[k]].fetch_add(1, std::memory_order_relaxed);
      c[ev[k]].fetch_add(1, std::memory_order_relaxed);
    }
    for (int64_t i = 0; i < n; ++i) cnt[i + 1] = cnt[i] + c[i].load();
  }
  std::vector<int32_t> tmp((size_t)cnt[n]);
  {
    std::vector<std::atomic<int64_t>> fill((size_t)n);
    for (int64_t i = 0; i < n; ++i) fill[i].store(cnt[i], std::memory_order_relaxed);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < ne; ++k) {
      int64_t a = eu[k], b = ev[k];
      if (a == b) continue;
      tmp[fill[a].fetch_add(1, std::memory_order_relaxed)] = (int32_t)b;
      tmp[fill[b].fetch_add(1, std::memory_order_relaxed)] = (int32_t)a;
    }
  }
  std::vector<int64_t> deg((size_t)n, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    int32_t* b = tmp.data() + cnt[i];
    int32_t* e = tmp.data() + cnt[i + 1];
    std::sort(b, e);
    deg[i] = std::unique(b, e) - b;
  }
  rp_out[0] = 0;
  for (int64_t i = 0; i < n; ++i) rp_out[i + 1] = rp_out[i] + (int32_t)deg[i];
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i)
    std::memcpy(ci_out + rp_out[i], tmp.data() + cnt[i], (size_t)deg[i] * 4);
  if (self_loops) *self_loops = loops.load();
  if (dup_merged) *dup_merged = (cnt[n] - (int64_t)rp_out[n]) / 2;
  return (int64_t)rp_out[n];
}

// ------------------------------------------------------------- generators
// Each returns the number of sampled undirected pairs; call with eu==nullptr
// to size, then again to fill.

// Config 1: the reference's er_graph (proj/tests/testutil.hpp:90-99).
int64_t fglt_gen_er(int64_t n, double p, uint64_t seed, int64_t* eu, int64_t* ev) {
  std::mt19937_64 rng(seed);
  std::bernoulli_distribution coin(p);
  int64_t k = 0;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t v = u + 1; v < n; ++v)
      if (coin(rng)) {
        if (eu) { eu[k] = u; ev[k] = v; }
        ++k;
      }
  return k;
}

// Configs 3/4: R-MAT, 2^scale vertices, edge_factor * 2^scale samples, per
// level quadrant probabilities (a, b, c, 1-a-b-c), no noise.
int64_t fglt_gen_rmat(int scale, int edge_factor, double a, double b, double c,
                      uint64_t seed, int64_t* eu, int64_t* ev) {
  const int64_t ne = (int64_t)edge_factor << scale;
  if (!eu) return ne;
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < ne; ++k) {
    int64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      double r = unit(rnd(seed, 0x524d4154, (uint64_t)k * (uint64_t)scale + (uint64_t)l));
      int ub = 0, vb = 0;
      if (r < a) {
      } else if (r < ab) {
        vb = 1;
      } else if (r < abc) {
        ub = 1;
      } else {
        ub = 1; vb = 1;
      }
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    eu[k] = u;
    ev[k] = v;
  }
  return ne;
}

// Config 2: random geometric graph, n points iid U[0,1)^2, radius chosen for
// the target average degree (r = sqrt(avg_deg / (pi n))), then vertices
// relabelled by a seeded random permutation.
int64_t fglt_gen_rgg(int64_t n, double avg_deg, uint64_t seed, int64_t* eu, int64_t* ev) {
  const double r = std::sqrt(avg_deg / (M_PI * (double)n));
  const int64_t g = std::max<int64_t>(1, (int64_t)std::floor(1.0 / r));
  std::vector<double> x((size_t)n), y((size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    x[i] = unit(rnd(seed, 0x52474758, (uint64_t)i));
    y[i] = unit(rnd(seed, 0x52474759, (uint64_t)i));
  }
  // random relabel: sort ids by a hash key (a seeded uniform permutation)
  std::vector<std::pair<uint64_t, int64_t>> key((size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) key[i] = {rnd(seed, 0x5045524d, (uint64_t)i), i};
  std::sort(key.begin(), key.end());
  std::vector<int64_t> label((size_t)n);
  for (int64_t i = 0; i < n; ++i) label[key[i].second] = i;
  // grid bucketing
  std::vector<int64_t> cell((size_t)n), start((size_t)(g * g + 1), 0), order((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t cx = std::min<int64_t>(g - 1, (int64_t)(x[i] * g));
    int64_t cy = std::min<int64_t>(g - 1, (int64_t)(y[i] * g));
    cell[i] = cy * g + cx;
    start[cell[i] + 1]++;
  }
  for (int64_t c = 0; c < g * g; ++c) start[c + 1] += start[c];
  {
    std::vector<int64_t> f(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < n; ++i) order[f[cell[i]]++] = i;
  }
  const double r2 = r * r;
  // count per point, then fill (pairs i<j by id within distance)
  std::vector<int64_t> cnt((size_t)n + 1, 0);
  auto visit = [&](int64_t i, auto&& emit) {
    int64_t cx = cell[i] % g, cy = cell[i] / g;
    for (int64_t dy = -1; dy <= 1; ++dy)
      for (int64_t dx = -1; dx <= 1; ++dx) {
        int64_t nx = cx + dx, ny = cy + dy;
        if (nx < 0 || ny < 0 || nx >= g || ny >= g) continue;
        int64_t c = ny * g + nx;
        for (int64_t t = start[c]; t < start[c + 1]; ++t) {
          int64_t j = order[t];
          if (j <= i) continue;
          double ddx = x[i] - x[j], ddy = y[i] - y[j];
          if (ddx * ddx + ddy * ddy < r2) emit(j);
        }
      }
  };
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    visit(i, [&](int64_t) { ++c; });
    cnt[i + 1] = c;
  }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  if (!eu) return cnt[n];
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) {
    int64_t w = cnt[i];
    visit(i, [&](int64_t j) {
      eu[w] = label[i];
      ev[w] = label[j];
      ++w;
    });
  }
  return cnt[n];
}

// Config 5: planted-community SBM: `blocks` blocks of `bs` vertices, each
// intra-block pair with probability p_in, plus cross_factor*n uniformly random
// cross-block pairs.
int64_t fglt_gen_sbm(int64_t blocks, int64_t bs, double p_in, double cross_factor,
                     uint64_t seed, int64_t* eu, int64_t* ev) {
  const int64_t n = blocks * bs;
  const int64_t pairs_per_block = bs * (bs - 1) / 2;
  std::vector<int64_t> cnt((size_t)blocks + 1, 0);
  auto intra = [&](int64_t b, auto&& emit) {
    int64_t t = 0;
    for (int64_t i = 0; i < bs; ++i)
      for (int64_t j = i + 1; j < bs; ++j, ++t)
        if (unit(rnd(seed, 0x53424d30, (uint64_t)(b * pairs_per_block + t))) < p_in)
          emit(b * bs + i, b * bs + j);
  };
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < blocks; ++b) {
    int64_t c = 0;
    intra(b, [&](int64_t, int64_t) { ++c; });
    cnt[b + 1] = c;
  }
  for (int64_t b = 0; b < blocks; ++b) cnt[b + 1] += cnt[b];
  const int64_t ncross = (int64_t)std::llround(cross_factor * (double)n);
  if (!eu) return cnt[blocks] + ncross;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < blocks; ++b) {
    int64_t w = cnt[b];
    intra(b, [&](int64_t i, int64_t j) { eu[w] = i; ev[w] = j; ++w; });
  }
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < ncross; ++k) {
    int64_t u = (int64_t)(rnd(seed, 0x53424d31, (uint64_t)k) % (uint64_t)n);
    int64_t v = (int64_t)(rnd(seed, 0x53424d32, (uint64_t)k) % (uint64_t)(n - bs));
    int64_t b0 = (u / bs) * bs;
    if (v >= b0) v += bs;  // skip u's own block
    eu[cnt[blocks] + k] = u;
    ev[cnt[blocks] + k] = v;
  }
  return cnt[blocks] + ncross;
}

}  // extern "C"
