// fglt_device.cuh — sm_100a kernels of the B200-native FGlT hot path.
//
// Every kernel works on the DEGREE-RELABELLED graph: vertices are renumbered
// by (degree, original id) ascending, rows re-sorted. With that labelling the
// edge orientation "low rank -> high rank" used by all enumeration kernels is
// a plain id comparison: N+(u) is the suffix of row u after `split[u]`, N-(u)
// the prefix. `mir[p]` maps every CSR position (u, v) to the position of
// (v, u), so the canonical (u<v) slot of each undirected edge is reachable
// from both rows without searching. All counting is integer and every
// cross-thread accumulation is a commutative integer atomic, so results are
// bit-identical for any schedule, grid size or number of GPUs.
//
// Quantities (reference formulas, proj/src/kernels.cpp):
//   p1 = d, p2 = sum_j d_j - d                          (:26-39)
//   C3(i,j) = |N(i) ∩ N(j)|, c3 = sum_j C3 / 2          (:41-89)
//   p3 = sum_j p2_j - (d(d-1) + 2 c3)   [rectified]     (:91-107)
//   c4 = #4-cycles through i, d14 = sum_j C(C3(i,j),2)  (:109-147)
//   d7, d9, d10, d11                                    (:149-205)
//   d13 = sum_{triangles {i,j,k}} (C3(j,k) - 1)         (:207-232)
//   d15 = #4-cliques through i                          (:234-288)
#pragma once

#include <cstdint>

// Device bounds checks of the hot kernels' indexed accesses (shared-memory
// tiles, triangle-list records, cursors, table rows): compiled in with
// -DFGLT_DEBUG_BOUNDS (tools/build_variant.sh checked -DFGLT_DEBUG_BOUNDS);
// a violation prints and abandons the offending thread's work, so the
// parity check of the same run fails too. Off in the product build.
#ifdef FGLT_DEBUG_BOUNDS
#include <cstdio>
#define FGLT_BOUNDS(cond, tag, a, b)                                                   \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("FGLT bounds %s: %lld %lld (block %d thread %d)\n", tag, (long long)(a),   \
             (long long)(b), blockIdx.x, threadIdx.x);                                 \
      return;                                                                          \
    }                                                                                  \
  } while (0)
#else
#define FGLT_BOUNDS(cond, tag, a, b) do { } while (0)
#endif

namespace fglt {

typedef unsigned long long u64;
typedef unsigned int u32;

constexpr int kWarp = 32;

__device__ __forceinline__ int lower_bound_i32(const int* __restrict__ a, int lo,
                                               int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int lower_bound_smem(const int* a, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__device__ __forceinline__ u64 group_sum_u64(u64 v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
  return v;
}

__device__ __forceinline__ u64 sat_sub(u64 a, u64 b) { return a > b ? a - b : 0ull; }

// Exact 64-bit accumulation in shared memory from native 32-bit atomics: the
// low word wraps, its carry goes to the high word. Little-endian [lo, hi], so
// the pair reads back as one u64 after a barrier. (A 64-bit shared atomicAdd
// compiles to a CAS spin loop, ATOMS.CAST.SPIN.64, which lost updates under
// contention in our kernels — see DESIGN.md.)
__device__ __forceinline__ void smem_add_u64(u64* addr, u64 v) {
  u32* w = reinterpret_cast<u32*>(addr);
  const u32 vl = (u32)v;
  const u32 vh = (u32)(v >> 32);
  const u32 old = atomicAdd(w, vl);
  const u32 carry = (u32)(old + vl < old);
  if (vh + carry) atomicAdd(w + 1, vh + carry);
}

// ------------------------------------------------- warp segment flattening
// A warp holds one segment per lane (start, len). flat_prefix computes the
// exclusive offsets and the total; flat_row maps a flattened element index k
// to the lane (row) owning it with a 5-step shuffle search over the offsets
// (the largest r with off[r] <= k; empty rows are skipped automatically).
// Consumers then stream the batch's elements with all 32 lanes busy and
// independent loads (no data-dependent loop exits).
__device__ __forceinline__ int flat_prefix(int len, int* total) {
  const int lane = threadIdx.x & 31;
  int incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  *total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - len;
}

__device__ __forceinline__ int flat_row(int off, int k) {
  int r = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int o = __shfl_sync(0xffffffffu, off, r + s);
    if (o <= k) r += s;
  }
  return r;
}

// Segmented sum across the warp of values whose rows are nondecreasing in the
// lane index: returns, in the LAST lane of each run of equal `row`, the run's
// total and sets *tail there.
__device__ __forceinline__ u64 seg_sum_runs(int row, u64 v, bool* tail) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 t = __shfl_up_sync(0xffffffffu, v, o);
    const int tr = __shfl_up_sync(0xffffffffu, row, o);
    if (lane >= o && tr == row) v += t;
  }
  const int nr = __shfl_down_sync(0xffffffffu, row, 1);
  *tail = (lane == 31) || (nr != row);
  return v;
}

// ---------------------------------------------------------------- root bins
struct BinThr {
  u64 thr[8];
  int nbins;
};
struct BinBases {
  int base[9];
};

__device__ __forceinline__ int bin_of(u64 x, const BinThr& T) {
  if (x == 0) return -1;  // key 0 roots are dropped
  int b = 0;
  while (b + 1 < T.nbins && x > T.thr[b]) ++b;
  return b;
}

// all 32 lanes call it (b = -1: nothing to count)
__device__ __forceinline__ void bin_tally(int b, int nbins, int& acc) {
  const int lane = threadIdx.x & 31;
  for (int q = 0; q < nbins; ++q) {
    const unsigned m = __ballot_sync(0xffffffffu, b == q);
    if (lane == q) acc += __popc(m);
  }
}

__device__ __forceinline__ void bin_tally_flush(int acc, int nbins, int* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  if (lane < nbins && acc) atomicAdd(counts + lane, acc);
}

// ------------------------------------------------------------ preprocessing

// key = degree << 32 | id : sorting these gives the relabelling order.
// Vertices of degree <= 1 lie on no triangle or cycle: they are ranked LAST
// (bit 31 of the degree field), so the enumeration id range [0, n_active)
// holds only vertices of degree >= 2 and the 4-cycle tiles shrink with it.
// Rank order of the relabel: degree ascending with degree <= 1 vertices last
// (degree 0 before 1), ties by id. As a STABLE sort of the ids by one int key
// (CUB radix sort is stable): key = d for d >= 2, n + d below (d <= n - 1,
// so every leaf key is above every active one).
// Low-skew graphs (d_max <= flat_dmax, read from the device-side graph stats:
// no host round trip): every active vertex gets the same key, so the active
// ids keep the caller's order (and whatever locality it has: the SBM's
// communities are contiguous) and only the leaves move to the end. With
// degrees this small the orientation by id costs about the same enumeration
// work as the orientation by degree.
__global__ void k_degree_keys(const int* __restrict__ rp, int n, int* __restrict__ keys,
                              int* __restrict__ ids, const u64* __restrict__ stats,
                              u64 flat_dmax) {
  const bool flat = stats[1] <= flat_dmax;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int d = rp[i + 1] - rp[i];
    keys[i] = d >= 2 ? (flat ? 2 : d) : n + d;
    ids[i] = i;
  }
}

// sorted_ids may BE perm (the degree sort's id buffers are (split, perm)): no
// __restrict__ on the two; each thread reads its entry before writing it.
__global__ void k_perm(const int* sorted_ids, const int* __restrict__ rp, int n, int* perm,
                       int* __restrict__ inv, int* __restrict__ ndeg) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int old = sorted_ids[r];
    perm[r] = old;
    inv[old] = r;
    ndeg[r] = rp[old + 1] - rp[old];
  }
}

// Warp per new row r: the relabelled neighbours of the old row (unsorted) and
// the row id of each. The array is r-major, so a STABLE sort of these pairs
// by neighbour id lists, for every vertex y, its neighbours r in ascending
// order: the transpose of a symmetric graph is the graph itself, so that sort
// yields the sorted relabelled CSR (a 20-bit key sort instead of a sort of
// every row).
// Active rows [0, n_active) have non-decreasing degree after the relabel, so
// the long ones are the contiguous range [first_long_row, n_active).
__device__ __forceinline__ int first_long_row(const int* __restrict__ nrp, int nact, int thr) {
  int lo = 0, hi = nact;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (nrp[mid + 1] - nrp[mid] > thr) hi = mid; else lo = mid + 1;
  }
  return lo;
}

constexpr int kLongRow = 1024;  // rows longer than this get a whole block

template <int G>  // lanes per short row (from the mean degree)
__global__ void k_fill_rows(const int* __restrict__ rp, const int* __restrict__ ci,
                            const int* __restrict__ perm, const int* __restrict__ inv,
                            const int* __restrict__ nrp, int n,
                            const unsigned long long* __restrict__ nact_p,
                            int* __restrict__ out, int* __restrict__ row_of) {
  const int nact = (int)*nact_p;
  const int fl = first_long_row(nrp, nact, kLongRow);
  for (int r = fl + blockIdx.x; r < nact; r += gridDim.x) {  // block per long row
    const int o = perm[r];
    const int b = rp[o], e = rp[o + 1], w = nrp[r];
    for (int p = b + threadIdx.x; p < e; p += blockDim.x) {
      out[w + (p - b)] = inv[ci[p]];
      row_of[w + (p - b)] = r;
    }
  }
  const int lane = threadIdx.x & (G - 1);
  const int groups = (gridDim.x * blockDim.x) / G;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) / G; r < n; r += groups) {
    if (r >= fl && r < nact) continue;
    const int o = perm[r];
    const int b = rp[o], e = rp[o + 1], w = nrp[r];
    for (int p = b + lane; p < e; p += G) {
      out[w + (p - b)] = inv[ci[p]];
      row_of[w + (p - b)] = r;
    }
  }
}

// split[r] = first position of row r holding a neighbour > r.
__global__ void k_split(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                        const unsigned long long* __restrict__ nact_p, int* __restrict__ split,
                        int* __restrict__ send, unsigned long long* __restrict__ maxout) {
  // split[r]: first neighbour > r; send[r]: first neighbour >= n_active (the
  // pendant/isolated tail). N+(r) restricted to active vertices is
  // [split[r], send[r]); vertices >= n_active are never enumeration roots.
  const int nact = (int)*nact_p;
  unsigned long long mo = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int s = lower_bound_i32(ci, rp[r], rp[r + 1], r);
    const int e = r < nact ? lower_bound_i32(ci, s, rp[r + 1], nact) : s;
    split[r] = s;
    send[r] = e;
    mo = max(mo, (unsigned long long)(e - s));
  }
  // one atomic per warp: every thread hitting the same word serialises
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, o));
  if ((threadIdx.x & 31) == 0 && mo) atomicMax(maxout, mo);
}

// Low-degree graphs (binary searches are short): G lanes per row; for each
// canonical position p (row r, v = ci[p] > r) find the mirror position q of
// r in row v (a prefix entry) and record both.
template <int G>  // lanes per row (from the mean degree)
__global__ void k_mirror(const int* __restrict__ rp, const int* __restrict__ ci,
                         const int* __restrict__ split, const int* __restrict__ send, int n,
                         int* __restrict__ mir) {
  // canonical edges between active vertices only: edges to the pendant tail
  // carry no triangles (their C3 stays 0 in both slots)
  const int lane = threadIdx.x & (G - 1);
  const int groups = (gridDim.x * blockDim.x) / G;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) / G; r < n; r += groups) {
    const int s = split[r], e = send[r];
    for (int p = s + lane; p < e; p += G) {
      const int v = ci[p];
      const int q = lower_bound_i32(ci, rp[v], split[v], r);
      mir[p] = q;
      mir[q] = p;
    }
  }
}

// Low-degree graphs (d_max <= G * K): the relabelled row r is built AND sorted
// by its own G lanes in registers — K elements per lane, each element's rank
// = the number of row elements below it (ties by position, so a malformed
// row with repeats still lands in distinct slots) — and written straight to
// its sorted slot: one read of the input row, one write of the new row, no
// global sort and no (row, key) scratch arrays. The same lanes count the
// neighbours below r and below n_active: split[r], send[r] and max |N+(r)|
// (k_split's outputs).
template <int G, int K>
__global__ void __launch_bounds__(256)
k_fill_sort(const int* __restrict__ rp, const int* __restrict__ ci, const int* __restrict__ perm,
            const int* __restrict__ inv, const int* __restrict__ nrp, int n,
            const unsigned long long* __restrict__ nact_p, int* __restrict__ out,
            int* __restrict__ split, int* __restrict__ send,
            unsigned long long* __restrict__ maxout) {
  const int nact = (int)*nact_p;
  const int lane = threadIdx.x & (G - 1);
  const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
  const int groups = (gridDim.x * blockDim.x) / G;
  const int g0 = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int rounds = (n + groups - 1) / groups;
  unsigned long long mo = 0;
  for (int it = 0; it < rounds; ++it) {  // warp-uniform trip count (group shuffles)
    const int r = g0 + it * groups;
    int d = 0, b = 0, w = 0;
    if (r < n) {
      const int o = perm[r];
      b = rp[o];
      d = rp[o + 1] - b;
      w = nrp[r];
    }
    int x[K], rank[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int i = lane + k * G;
      x[k] = i < d ? inv[__ldg(ci + b + i)] : 0x7fffffff;
      rank[k] = 0;
    }
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      if (kk * G < d) {  // group-uniform
#pragma unroll
        for (int l = 0; l < G; ++l) {
          const int y = __shfl_sync(gmask, x[kk], l, G);
#pragma unroll
          for (int k = 0; k < K; ++k)
            rank[k] += (y < x[k]) || (y == x[k] && (kk < k || (kk == k && l < lane)));
        }
      }
    }
    int below = 0, act = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (lane + k * G < d) {
        out[w + rank[k]] = x[k];
        below += x[k] < r;
        act += x[k] < nact;
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      below += __shfl_xor_sync(gmask, below, o, G);
      act += __shfl_xor_sync(gmask, act, o, G);
    }
    if (r < n && lane == 0) {
      const int s = w + below;
      const int e = r < nact ? w + act : s;
      split[r] = s;
      send[r] = e;
      mo = max(mo, (unsigned long long)(e - s));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, o));
  if ((threadIdx.x & 31) == 0 && mo) atomicMax(maxout, mo);
}

// a[i] = i and k[i] = src[i]: the (key, value) input of the mirror transpose
// sort (the sort consumes its key buffer, so the graph's column array is
// copied, not handed over).
__global__ void k_iota_copy(int* __restrict__ a, int* __restrict__ k, const int* __restrict__ src,
                            long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    a[i] = (int)i;
    k[i] = src[i];
  }
}

__global__ void k_iota(int* __restrict__ a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = (int)i;
}

// ------------------------------------------------------------------ sweeps
// Per-row sweeps. Each is a functor: elem() folds one CSR entry into NV
// accumulators, fin() writes the row. Rows of degree <= kSweepBig go G lanes
// per row (k_rows_group); longer rows, listed once by k_list_big_rows, get a
// whole block each (k_rows_block), so one hub row never serialises a group.
constexpr int kSweepBig = 1024;
constexpr int kSweepBlock = 256;

__global__ void k_list_big_rows(const int* __restrict__ rp, int n, int* __restrict__ list,
                                int* __restrict__ count) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    if (rp[r + 1] - rp[r] > kSweepBig) list[atomicAdd(count, 1)] = r;
}

// Rows r = r0 + i * rstep (multi-GPU: rank `r0` of `rstep` takes every
// rstep-th row, an even share of every degree range; 0 / 1 = all rows).
template <int G, class F>
__global__ void k_rows_group(F f, const int* __restrict__ rp, int n, int r0, int rstep) {
  const int lane = threadIdx.x & (G - 1);
  const int groups = (gridDim.x * blockDim.x) / G;
  const int g0 = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int mine_n = n > r0 ? (n - r0 + rstep - 1) / rstep : 0;
  const int rounds = (mine_n + groups - 1) / groups;
  for (int it = 0; it < rounds; ++it) {  // warp-uniform trip count (group shuffles)
    const int i = g0 + it * groups;
    const int r = i < mine_n ? r0 + i * rstep : n;
    u64 acc[F::NV] = {};
    bool mine = false;
    if (r < n) {
      const int b = rp[r], e = rp[r + 1];
      mine = e - b <= kSweepBig;
      if (mine)
        for (int p = b + lane; p < e; p += G) f.elem(r, p, acc);
    }
#pragma unroll
    for (int k = 0; k < F::NV; ++k) acc[k] = group_sum_u64<G>(acc[k]);
    if (mine && lane == 0) f.fin(r, acc);
  }
}

template <class F>
__global__ void __launch_bounds__(kSweepBlock)
k_rows_block(F f, const int* __restrict__ rp, const int* __restrict__ list,
             const int* __restrict__ count, int r0, int rstep) {
  __shared__ u64 part[F::NV][kSweepBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nb = *count;
  for (int i = blockIdx.x; i < nb; i += gridDim.x) {
    const int r = list[i];
    if (rstep > 1 && r % rstep != r0) continue;  // block-uniform
    u64 acc[F::NV] = {};
    for (int p = rp[r] + threadIdx.x; p < rp[r + 1]; p += kSweepBlock) f.elem(r, p, acc);
#pragma unroll
    for (int k = 0; k < F::NV; ++k) {
      const u64 v = warp_sum_u64(acc[k]);
      if (lane == 0) part[k][wid] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < F::NV; ++k) {
        u64 t = 0;
        for (int w = 0; w < kSweepBlock / 32; ++w) t += part[k][w];
        acc[k] = t;
      }
      f.fin(r, acc);
    }
    __syncthreads();
  }
}

// Sweep A: p2 = sum_j d_j - d  (compute_p2, kernels.cpp:26-39);
// d7 = sum_j C(d_j - 1, 2) (compute_d7, kernels.cpp:149-163).
struct SweepA {
  static constexpr int NV = 2;
  const int* rp;
  const int* ci;
  u64* p2;
  u64* d7;
  __device__ void elem(int, int p, u64 (&acc)[NV]) const {
    const int j = ci[p];
    const u64 dj = (u64)(rp[j + 1] - rp[j]);
    acc[0] += dj;
    const u64 t = dj - 1;  // dj >= 1 for a neighbour
    acc[1] += t < 2 ? 0ull : t * (t - 1) / 2;
  }
  __device__ void fin(int r, const u64 (&acc)[NV]) const {
    const u64 d = (u64)(rp[r + 1] - rp[r]);
    if (p2) p2[r] = sat_sub(acc[0], d);
    if (d7) d7[r] = acc[1];
  }
};

// The triangle pass (per-edge C3, and 4-cliques) is root-centric: see
// k_roots_warp / k_roots_block<kC3=true> in fglt_roots.cuh.

// Copy canonical C3 values into their mirror slots so rows read contiguously
// (per-kernel API only): row r's canonical slots are [split[r], send[r]).
__global__ void k_c3_mirror(const int* __restrict__ split, const int* __restrict__ send,
                            const int* __restrict__ mir, int nact, u32* __restrict__ C3f) {
  const int lane = threadIdx.x & 7;
  const int groups = (gridDim.x * blockDim.x) >> 3;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 3; r < nact; r += groups)
    for (int p = split[r] + lane; p < send[r]; p += 8) C3f[mir[p]] = C3f[p];
}

// c3 = sum C3 / 2; d14 = sum C(C3,2); d10 = sum C3 * (d_j - 2)+;
// p3 = sum p2_j - (d(d-1) + 2 c3) rectified   (kernels.cpp:91-107, :176-205)
// Sweep B: c3 = sum C3 / 2; d14 = sum C(C3,2); d10 = sum C3 * (d_j - 2)+;
// p3 = sum p2_j - (d(d-1) + 2 c3) rectified   (kernels.cpp:91-107, :176-205)
// C3f holds each edge's count at its canonical slot only (row min(u,v)'s
// suffix, where the triangle pass adds); a lower neighbour j < r reads it
// through mir. Rows r >= n_active (degree <= 1) have no triangles: their
// slots stay 0 and have no mirror entry.
struct SweepB {
  static constexpr int NV = 4;
  const int* rp;
  const int* ci;
  const u32* C3f;
  const int* mir;
  int nact;
  const u64* p2;
  u64* c3;
  u64* d14;
  u64* d10;
  u64* p3;
  __device__ void elem(int r, int p, u64 (&acc)[NV]) const {
    const int j = ci[p];
    const u64 c = C3f[j < r && r < nact ? mir[p] : p];
    acc[0] += c;
    acc[1] += c * (c - (c > 0)) / 2;
    const u64 dj = (u64)(rp[j + 1] - rp[j]);
    acc[2] += c * (dj > 2 ? dj - 2 : 0ull);
    if (p2) acc[3] += p2[j];
  }
  __device__ void fin(int r, const u64 (&acc)[NV]) const {
    const u64 d = (u64)(rp[r + 1] - rp[r]);
    const u64 c3v = acc[0] / 2;
    c3[r] = c3v;
    if (d14) d14[r] = acc[1];
    if (d10) d10[r] = acc[2];
    if (p3) p3[r] = sat_sub(acc[3], d * (d > 0 ? d - 1 : 0ull) + 2 * c3v);
  }
};

// Sweep C: d9 = sum_j c3_j - 2 c3, rectified (kernels.cpp:194-199)
struct SweepC {
  static constexpr int NV = 1;
  const int* ci;
  const u64* c3;
  u64* d9;
  __device__ void elem(int, int p, u64 (&acc)[NV]) const { acc[0] += c3[ci[p]]; }
  __device__ void fin(int r, const u64 (&acc)[NV]) const { d9[r] = sat_sub(acc[0], 2 * c3[r]); }
};

}  // namespace fglt
