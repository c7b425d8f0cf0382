// fglt_roots.cuh — root-centric enumeration kernels (4-cycles, diamonds,
// 4-cliques) and the fused raw->net epilogue. See fglt_device.cuh for the
// labelling conventions.
#pragma once

#include "fglt_device.cuh"
#include "fglt_tables.h"


namespace fglt {

// =============================================================== 4-cycles
// Every 4-cycle has a unique highest vertex u; its opposite vertex w < u and
// both middle vertices v, v' < u. For a root u, L[w] counts wedges u-v-w with
// v in N-(u) and w in N(v), w < u (the prefix of row v up to the mirror
// position of u). Then, exactly (the per-vertex form of the reference's
// c4 = sum_k C(P2(i,k),2), kernels.cpp:109-147):
//   c4[u] += sum_w C(L[w],2);  c4[w] += C(L[w],2);  c4[v] += sum_{w} (L[w]-1)
// The accumulator L lives in shared memory: a per-warp or per-block open
// addressing table for light roots, dense 48K-entry tiles of the w range for
// heavy roots.

// wc(u) = number of wedges rooted at u: sum over v in N-(u) of the prefix of
// row v below u, whose end is the mirror position of u. A row functor
// (k_rows_group / k_rows_block); pendant/isolated vertices root nothing.
struct RootWork {
  static constexpr int NV = 1;
  const int* rp;
  const int* ci;
  const int* split;
  const int* mir;
  int nact;
  u64* wc;
  __device__ void elem(int r, int p, u64 (&acc)[NV]) const {
    if (r < nact && p < split[r]) acc[0] += (u64)(mir[p] - rp[ci[p]]);
  }
  __device__ void fin(int r, const u64 (&acc)[NV]) const { wc[r] = acc[0]; }
};

// tw(u) = triangle-probe work of u (sum of |N+(x)| over x in N+(u), plus
// |N+(u)|); used only to cut root ranges of equal work across ranks.
template <int G>
__global__ void k_probe_work(const int* __restrict__ split, const int* __restrict__ send,
                             const int* __restrict__ ci, int n,
                             const unsigned long long* __restrict__ nact_p,
                             u64* __restrict__ tw) {
  const int nact = (int)*nact_p;
  const int lane = threadIdx.x & (G - 1);
  const int groups = (gridDim.x * blockDim.x) / G;
  const int g0 = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int rounds = (n + groups - 1) / groups;
  for (int it = 0; it < rounds; ++it) {
    const int u = g0 + it * groups;
    u64 t = 0;
    if (u < nact)
      for (int p = split[u] + lane; p < send[u]; p += G) {
        const int x = ci[p];
        t += (u64)(send[x] - split[x]);
      }
    t = group_sum_u64<G>(t);
    if (u < n && lane == 0) tw[u] = u < nact ? t + (u64)(send[u] - split[u]) : 0;
  }
}

__device__ __forceinline__ u32 hash_slot(int w, int logcap) {
  return ((u32)w * 0x9E3779B1u) >> (32 - logcap);
}

__device__ __forceinline__ void hash_insert(int* keys, u32* vals, int logcap, int w) {
  const u32 mask = (1u << logcap) - 1;
  u32 h = hash_slot(w, logcap);
  while (true) {
    const int k = atomicCAS(keys + h, -1, w);
    if (k == -1 || k == w) { atomicAdd(vals + h, 1u); return; }
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ u32 hash_get(const int* keys, const u32* vals, int logcap, int w) {
  const u32 mask = (1u << logcap) - 1;
  u32 h = hash_slot(w, logcap);
  while (true) {
    const int k = keys[h];
    if (k == w) return vals[h];
    if (k == -1) return 0;
    h = (h + 1) & mask;
  }
}

// Warp per root; a 2^LOGCAP-slot table per warp in shared memory.
// Lookup that also claims the slot: bit 31 of the count marks "C(L,2) already
// emitted for this target"; *first is true for exactly one caller per slot.
__device__ __forceinline__ u32 hash_get_claim(const int* keys, u32* vals, int logcap, int w,
                                              bool* first) {
  const u32 mask = (1u << logcap) - 1;
  u32 h = hash_slot(w, logcap);
  while (true) {
    const int k = keys[h];
    if (k == w) {
      const u32 old = atomicOr(vals + h, 0x80000000u);
      *first = !(old & 0x80000000u);
      return old & 0x7fffffffu;
    }
    h = (h + 1) & mask;
  }
}

// Warp per root (wc <= 256): a table of 2^hlog <= 2^LOGCAP slots sized to the
// root; the rows of N-(u) are walked 32 at a time with segment flattening so
// every lane streams one wedge per step.
// Class-1 roots with at most kC4Tiny wedges (most roots of low-degree graphs,
// e.g. RGG's ~2-5): thread per root, the wedge targets in registers (static
// indexing via shift insertion), L[w] by pairwise equality. No shared table to
// clear and no warp-wide bookkeeping per root; k_c4_warp skips these roots.
#ifndef FGLT_C4_TINY
#define FGLT_C4_TINY 16
#endif
constexpr int kC4Tiny = FGLT_C4_TINY;
__global__ void __launch_bounds__(256) k_c4_tiny(const int* __restrict__ rp,
                                                 const int* __restrict__ ci,
                                                 const int* __restrict__ split,
                                                 const int* __restrict__ mir,
                                                 const int* __restrict__ roots, int nroots,
                                                 const u64* __restrict__ wcv,
                                                 u64* __restrict__ c4) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nroots; k += gridDim.x * blockDim.x) {
    const int u = roots[k];
    int wl[kC4Tiny], vl[kC4Tiny];
#pragma unroll
    for (int i = 0; i < kC4Tiny; ++i) wl[i] = -1 - i;  // distinct sentinels never match
    int cnt = 0;
    const int b = rp[u], s = split[u];
    for (int q = b; q < s; ++q) {
      const int v = ci[q];
      const int e = mir[q];
      for (int p = rp[v]; p < e; ++p) {
        const int w = __ldg(ci + p);
#pragma unroll
        for (int i = kC4Tiny - 1; i > 0; --i) {
          wl[i] = wl[i - 1];
          vl[i] = vl[i - 1];
        }
        wl[0] = w;
        vl[0] = v;
        ++cnt;
      }
    }
    u64 cu = 0;
#pragma unroll
    for (int i = 0; i < kC4Tiny; ++i) {
      if (i >= cnt) break;
      u32 L = 0;
      bool first = true;
#pragma unroll
      for (int j = 0; j < kC4Tiny; ++j) {
        const bool eq = wl[j] == wl[i];
        L += eq;
        first &= !(eq && j < i);
      }
      if (L >= 2) {
        if (first) {
          const u64 c = (u64)L * (L - 1) / 2;
          cu += c;
          atomicAdd(c4 + wl[i], c);
        }
        atomicAdd(c4 + vl[i], (u64)(L - 1));
      }
    }
    if (cu) atomicAdd(c4 + u, cu);
  }
}

template <int LOGCAP>
__global__ void k_c4_warp(const int* __restrict__ rp, const int* __restrict__ ci,
                          const int* __restrict__ split, const int* __restrict__ mir,
                          const int* __restrict__ roots, int nroots, const u64* __restrict__ wcv,
                          u64* __restrict__ c4) {
  constexpr int CAP = 1 << LOGCAP;
  constexpr int PER_WARP = CAP * 2 + 100;  // keys, vals, base[32], off[33], rowsum[32], pad (16 B)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int* keys = reinterpret_cast<int*>(smem_raw) + wib * PER_WARP;
  u32* vals = reinterpret_cast<u32*>(keys + CAP);
  int* fbase = reinterpret_cast<int*>(vals + CAP);
  int* foff = fbase + 32;
  u32* rs = reinterpret_cast<u32*>(foff + 33);
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nroots; k += warps) {
    const int u = roots[k];
    int hlog = 5;
    while (hlog < LOGCAP && ((u64)1 << hlog) < 2 * wcv[u]) ++hlog;
    const int cap = 1 << hlog;
    {
      uint4* k4 = reinterpret_cast<uint4*>(keys);
      uint4* v4 = reinterpret_cast<uint4*>(vals);
      for (int i = lane; i < (cap >> 2); i += 32) {
        k4[i] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
        v4[i] = make_uint4(0, 0, 0, 0);
      }
    }
    rs[lane] = 0;
    __syncwarp();
    const int b = rp[u], s = split[u];
    for (int q0 = b; q0 < s; q0 += 32) {
      const int q = q0 + lane;
      int st = 0, len = 0;
      if (q < s) {
        st = rp[ci[q]];
        len = mir[q] - st;
      }
      int T;
      const int off = flat_prefix(len, &T);
      fbase[lane] = st - off;
      foff[lane] = off;
      if (lane == 0) foff[32] = T;
      __syncwarp();
      int r = 0;
      for (int kk = lane; kk < T; kk += 128) {  // 4 independent loads in flight
        int w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int kj = kk + 32 * j;
          w[j] = -1;
          if (kj < T) {
            while (foff[r + 1] <= kj) ++r;
            w[j] = __ldg(ci + fbase[r] + kj);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (w[j] >= 0) hash_insert(keys, vals, hlog, w[j]);
      }
      __syncwarp();
    }
    u64 acc = 0;  // sum_w C(L[w],2), emitted by the first visitor of each target
    for (int q0 = b; q0 < s; q0 += 32) {
      const int q = q0 + lane;
      int st = 0, len = 0;
      if (q < s) {
        st = rp[ci[q]];
        len = mir[q] - st;
      }
      int T;
      const int off = flat_prefix(len, &T);
      fbase[lane] = st - off;
      foff[lane] = off;
      if (lane == 0) foff[32] = T;
      __syncwarp();
      int r = 0, cr = 0;
      u32 part = 0;
      for (int kk = lane; kk < T; kk += 128) {  // 4 independent loads in flight
        int w[4], rr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int kj = kk + 32 * j;
          w[j] = -1;
          if (kj < T) {
            while (foff[r + 1] <= kj) ++r;
            rr[j] = r;
            w[j] = __ldg(ci + fbase[r] + kj);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (w[j] < 0) break;
          if (rr[j] != cr) {
            if (part) atomicAdd(rs + cr, part);
            part = 0;
            cr = rr[j];
          }
          bool first;
          const u32 l = hash_get_claim(keys, vals, hlog, w[j], &first);
          if (first && l >= 2) {
            const u64 cc = (u64)l * (l - 1) / 2;
            acc += cc;
            atomicAdd(c4 + w[j], cc);
          }
          part += l - 1;
        }
      }
      if (part) atomicAdd(rs + cr, part);
      __syncwarp();
      if (q < s && rs[lane]) atomicAdd(c4 + ci[q], (u64)rs[lane]);
      rs[lane] = 0;
      __syncwarp();
    }
    acc = warp_sum_u64(acc);
    if (lane == 0 && acc) atomicAdd(c4 + u, acc);
    __syncwarp();
  }
}

__device__ __forceinline__ u64 block_sum_u64(u64 v, u64* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_u64(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  u64 t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < nw ? red[threadIdx.x] : 0ull;
    t = warp_sum_u64(t);
  }
  return t;  // valid in thread 0
}

// Cost-model classes for roots with wc(u) > 0 (k_c4_class):
//   9 thread per root (k_c4_tiny)        wc <= kC4Tiny
//   1 warp table, 512 slots              wc <= 256
//   8 small block table (128 threads, 1024 slots), wc <= 512
//   2 small block table (128 threads, 2048 slots), wc <= 1024
//   3 small block table (128 threads, <= 4096 slots), wc <= 2048
//   4 block table, P hash-partition passes over the wedges, P = ceil(wc/12288)
//   5 dense tiles, 16-bit packed counters (|N-(u)| < 65536), 96K ids per tile
//   6 dense tiles, 32-bit counters, 48K ids per tile
// Class 4 vs 5/6 is chosen per root by the cheaper of the two modelled costs.
#ifndef FGLT_C4B_LOG
#define FGLT_C4B_LOG 14
#define FGLT_C4B_THREADS 1024
#endif
#ifndef FGLT_HASH_WEIGHT
// hash-pass cost vs the big-tile dense cost. Measured after the dense kernel's
// lane-row rewrite (four-cycle phase, ms; R-MAT 20 / R-MAT 23): 1: 17.6 / 357,
// 2: 16.3 / 357, 4: 16.1 / 351, 8: 16.2 / 360, 16: 16.5 / 383, never hash:
// 16.2 / 383
#define FGLT_HASH_WEIGHT 4
#endif
#ifndef FGLT_HASH_WEIGHT_S
#define FGLT_HASH_WEIGHT_S FGLT_HASH_WEIGHT  // ... vs the small-tile dense cost
#endif
#ifndef FGLT_TILE_FIXED
#define FGLT_TILE_FIXED 2048  // per-tile fixed cost (barriers, setup) in the cost model
#endif
constexpr int kC4HashLog = FGLT_C4B_LOG;    // 16384 slots (keys + counts = 128 KB)
constexpr int kC4SmallLog = 12;             // 4096 slots (32 KB)
constexpr u64 kC4HashFill = 3ull << (kC4HashLog - 2);  // distinct targets per pass (LF 0.75)
#ifndef FGLT_DENSE_THREADS
#define FGLT_DENSE_THREADS 1024
#define FGLT_DENSE_TILE_BYTES 196608
#endif
// Two dense configurations, chosen per root by the cost model: big tiles
// (one 1024-thread block per SM, 192 KB) for roots whose rows pay a per-tile
// setup (large |N-(u)| x tiles), small tiles (two 512-thread blocks per SM,
// 96 KB each, so one block's tile barriers overlap the other's work) else.
constexpr int kC4DenseThreads = FGLT_DENSE_THREADS;     // big: one block per SM
constexpr int kC4TileBytes = FGLT_DENSE_TILE_BYTES;     // big: counter tile (192 KB)
constexpr int kC4DenseThreadsS = 512;                   // small: two blocks per SM
#ifndef FGLT_TILE_BYTES_S
#define FGLT_TILE_BYTES_S 98304
#endif
constexpr int kC4TileBytesS = FGLT_TILE_BYTES_S;        // small: 96 KB tiles
#ifndef FGLT_ROW_TILE
#define FGLT_ROW_TILE 1  // cost of one row's segment setup per tile, in wedges
#endif
#ifndef FGLT_SMALL_MAX_TILES
#define FGLT_SMALL_MAX_TILES 8
#endif
#ifndef FGLT_SMALL_EFF
#define FGLT_SMALL_EFF 85  // small-tile cost, percent of the modelled (better latency hiding)
#endif
constexpr int kC4Tile16 = kC4TileBytes / 2; // ids per packed tile
constexpr int kC4Tile32 = kC4TileBytes / 4; // ids per 32-bit tile
#ifndef FGLT_C4_LONG
#define FGLT_C4_LONG 16
#endif
constexpr int kC4Long = FGLT_C4_LONG;       // rows at least this long: flattened batches
#ifndef FGLT_GIANT
#define FGLT_GIANT 512
#endif
constexpr int kC4GiantPerTile = FGLT_GIANT;  // rows expected to put this many wedges in a tile: warp per row
#ifndef FGLT_GIANT_BIG
#define FGLT_GIANT_BIG FGLT_GIANT  // the same for the big-tile (1024-thread) kernel
#endif
constexpr int kC4GiantPerTileBig = FGLT_GIANT_BIG;
#ifndef FGLT_PROBE_NOCUT
#define FGLT_PROBE_NOCUT 0  // probe lists up to this long are probed whole (no cut search)
#endif
#ifndef FGLT_PROBE_NOCUT_WARP
#define FGLT_PROBE_NOCUT_WARP 0  // the same for warp roots (|S| <= 32)
#endif
#ifndef FGLT_PAIR_W
#define FGLT_PAIR_W 1   // relative cost of one hub-row pair test ...
#define FGLT_PROBE_W 3  // ... and of one probed element (members choose the cheaper path)
#endif
#ifndef FGLT_QUADS
#define FGLT_QUADS 2
#endif
#ifndef FGLT_ROOTS_LANE_MEMBER
#define FGLT_ROOTS_LANE_MEMBER 0  // root probes: thread per member instead of block-flattened quads
#endif
#ifndef FGLT_BATCH_LANE_ROW
#define FGLT_BATCH_LANE_ROW 1  // dense long-row batches: lane per row instead of flattened quads
#endif
#ifndef FGLT_BATCH_G
#define FGLT_BATCH_G 2  // lanes per row in lane-row batches (1, 2, 4, 8)
#endif
#ifndef FGLT_BATCH_MASKED
#define FGLT_BATCH_MASKED 0  // lane-row batches over aligned quads with masked ends: every load of a round issued up front
#endif
constexpr int kBatchG = FGLT_BATCH_LANE_ROW ? FGLT_BATCH_G : 1;
constexpr int kBatchRows = 32 / kBatchG;
constexpr int kQuadsInFlight = FGLT_QUADS;          // 16-byte loads in flight per lane (dense batches)
#ifndef FGLT_ROOTS_QUADS
#define FGLT_ROOTS_QUADS 1  // the same for the triangle pass (k_roots_block): 1 keeps it at 64 registers (2: 80), R-MAT 23 triangles 234 -> 215 ms
#endif
constexpr int kRootsQuads = FGLT_ROOTS_QUADS;
constexpr int kC4BlockThreads = FGLT_C4B_THREADS;  // class-4 block (one 128 KB table per SM)

// Dense tiles use counters as narrow as the target's degree allows: L[w] <=
// deg(w) (each wedge into w has a distinct middle vertex v in N(w)), and the
// active ids are in ascending degree, so ids [0, b4) (degree <= 15) get 4-bit
// counters, [b4, b8) (degree <= 255) 8-bit, [b8, b16) (degree <= 65535)
// 16-bit and the few ids above b16 32-bit ones. Tiles never straddle a band:
// a tile of T bytes holds 2T ids in the 4-bit band, T in the 8-bit band, T/2
// in the 16-bit band and T/4 above (the host builds the same boundaries).
// Roots u <= b16 never meet a 32-bit band (PACK kernels).
__host__ __device__ inline void dense_span(u64 u, u64 b4, u64 b8, u64 b16, u64 tile_bytes,
                                           u64* tiles, u64* bytes) {
  const u64 nib = u < b4 ? u : b4;
  const u64 byt = u > b4 ? (u < b8 ? u : b8) - b4 : 0;
  const u64 sht = u > b8 ? (u < b16 ? u : b16) - b8 : 0;
  const u64 rest = u > b16 ? u - b16 : 0;
  const u64 t4 = 2 * tile_bytes, t8 = tile_bytes, t16 = tile_bytes / 2, t32 = tile_bytes / 4;
  *tiles = (nib + t4 - 1) / t4 + (byt + t8 - 1) / t8 + (sht + t16 - 1) / t16 + (rest + t32 - 1) / t32;
  *bytes = (nib + 1) / 2 + byt + 2 * sht + 4 * rest;
}

__global__ void k_c4_class(const int* __restrict__ rp, const int* __restrict__ split,
                           const u64* __restrict__ wc, int u0, int u1, int b4, int b8, int b16,
                           u32* __restrict__ cls, u32* __restrict__ parts, int force_cls,
                           int force_parts, unsigned long long* __restrict__ class_wedges,
                           int* __restrict__ bin_counts) {
  // class_wedges[0] += wedges of the dense-tile roots (classes 5/6/7),
  // class_wedges[1] += all wedges (the 4-cycle phases' work units);
  // bin_counts[c - 1] += roots of class c (k_bin's list sizes)
  unsigned long long dense_w = 0, all_w = 0;
  int tally = 0;
  const int lane_ = threadIdx.x & 31;
  for (int ub = u0 + blockIdx.x * blockDim.x + threadIdx.x - lane_; ub < u1;
       ub += gridDim.x * blockDim.x) {
    const int u = ub + lane_;
    const bool valid = u < u1;  // warp-uniform trip count: idle lanes still vote below
    const u64 w = valid ? wc[u] : 0;
    u64 c = 0, P = 1;
    if (w == 0) {
      c = 0;
    } else if (w <= (u64)kC4Tiny) {
      c = 9;  // thread per root (k_c4_tiny)
    } else if (w <= 256) {
      c = 1;
    } else if (w <= 512) {
      c = 8;  // 128-thread block, 1024-slot table (twice the blocks per SM of class 2)
    } else if (w <= 1024) {
      c = 2;
    } else if (w <= 2048) {
      c = 3;
    } else {
      const u64 nq = (u64)(split[u] - rp[u]);
      P = (w + kC4HashFill - 1) / kC4HashFill;
      const u64 cost_base = P * (w + (1ull << kC4HashLog)) + w;
      const u64 cost_hash = FGLT_HASH_WEIGHT * cost_base;
      const u64 cost_hash_s = FGLT_HASH_WEIGHT_S * cost_base;
      const bool pack = u <= b16;  // no 32-bit band below u
      u64 tiles, bytes, tiles_s, bytes_s;
      dense_span((u64)u, (u64)b4, (u64)b8, (u64)b16, kC4TileBytes, &tiles, &bytes);
      dense_span((u64)u, (u64)b4, (u64)b8, (u64)b16, kC4TileBytesS, &tiles_s, &bytes_s);
      const u64 cost_dense = bytes / 8 + tiles * (FGLT_TILE_FIXED + FGLT_ROW_TILE * nq) + 2 * w;
      // small tiles only for roots that need few of them: with many tiles per
      // root the per-tile row setup and tail imbalance outweigh the overlap
      // (measured: R-MAT 20, <= 6 tiles, small wins 15%; R-MAT 23, up to 34
      // tiles, small loses 17%)
      const u64 cost_small =
          tiles_s > FGLT_SMALL_MAX_TILES
              ? ~0ull
              : (bytes_s / 8 + tiles_s * (FGLT_TILE_FIXED / 2 + FGLT_ROW_TILE * nq) + 2 * w) *
                    FGLT_SMALL_EFF / 100;
      if (cost_hash <= cost_dense && (!pack || cost_hash_s <= cost_small)) c = 4;
      else if (!pack) c = 6;
      else c = cost_small < cost_dense ? 7 : 5;
    }
    if (force_cls > 0 && w > 0) {  // test hook: route every root to one path
      const u64 nq = (u64)(split[u] - rp[u]);
      // external numbering: 2 hash passes, 3 packed tiles, 4 32-bit tiles,
      // 5 small packed tiles
      c = force_cls == 5 ? 7 : (u64)force_cls + 2;
      if ((c == 5 || c == 7) && u > b16) c = 6;
      if (c == 4) {
        P = (w + kC4HashFill - 1) / kC4HashFill;
        if (force_parts > 0) P = (u64)force_parts;
      }
    }
    if (valid) {
      cls[u] = (u32)c;
      parts[u] = (u32)P;  // P <= wc / 12288 + 1 < 2^32 (wc < 2^45: nnz < 2^31 rows of < 2^31)
    }
    all_w += w;
    if (c >= 5 && c <= 7) dense_w += w;
    bin_tally((int)c - 1, 9, tally);
  }
  bin_tally_flush(tally, 9, bin_counts);
  dense_w = warp_sum_u64(dense_w);
  all_w = warp_sum_u64(all_w);
  if ((threadIdx.x & 31) == 0) {
    if (dense_w) atomicAdd(class_wedges, dense_w);
    if (all_w) atomicAdd(class_wedges + 1, all_w);
  }
}

// Block per root, P hash-partition passes: pass `part` inserts only targets w
// with part_of(w) == part, so every pass fits the table. G lanes per row.
__device__ __forceinline__ u32 part_of(int w, u32 P) {
  return (u32)(((u64)(((u32)w * 0x85EBCA6Bu) ^ ((u32)w >> 13)) * P) >> 32);
}

// Block per root with a shared hash table of 2^hlog slots sized to the
// root (hlog <= max_log); P hash-partition passes when the distinct targets
// could exceed the table. G lanes per row; trip counts are warp-uniform
// because the group reductions shuffle the full warp.
template <int G>
__global__ void
k_c4_hashp(const int* __restrict__ rp, const int* __restrict__ ci,
           const int* __restrict__ split, const int* __restrict__ mir,
           const int* __restrict__ roots, int nroots, const u64* __restrict__ wcv,
           const u32* __restrict__ parts, int max_log, int* __restrict__ next_root,
           u64* __restrict__ c4) {
  // roots are sorted by work (largest first) and handed out dynamically
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ u64 red[32];
  const int maxcap = 1 << max_log;
  int* keys = reinterpret_cast<int*>(smem_raw);
  u32* vals = reinterpret_cast<u32*>(keys + maxcap);
  const int gl = threadIdx.x & (G - 1);
  const int gid = threadIdx.x / G, ngroups = blockDim.x / G;
  __shared__ int s_root;
  while (true) {
    if (threadIdx.x == 0) s_root = atomicAdd(next_root, 1);
    __syncthreads();
    const int k = s_root;
    if (k >= nroots) break;
    const int u = roots[k];
    const u32 P = parts[u];
    const u64 per_pass = (wcv[u] + P - 1) / P;
    int hlog = 6;
    while (hlog < max_log && ((u64)1 << hlog) < 2 * per_pass) ++hlog;
    const int cap = 1 << hlog;
    const int b = rp[u], s = split[u];
    const int rounds = (s - b + ngroups - 1) / ngroups;
    u64 acc = 0;
    for (u32 part = 0; part < P; ++part) {
      for (int i = threadIdx.x; i < cap; i += blockDim.x) { keys[i] = -1; vals[i] = 0; }
      __syncthreads();
      for (int q = b + gid; q < s; q += ngroups) {
        const int v = ci[q];
        const int end = mir[q];
        for (int p = rp[v] + gl; p < end; p += G) {
          const int w = __ldg(ci + p);
          if (P == 1 || part_of(w, P) == part) hash_insert(keys, vals, hlog, w);
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < cap; i += blockDim.x) {
        const u32 l = vals[i];
        if (l >= 2) {
          const u64 c = (u64)l * (l - 1) / 2;
          acc += c;
          atomicAdd(c4 + keys[i], c);
        }
      }
      for (int it = 0; it < rounds; ++it) {
        const int q = b + gid + it * ngroups;
        u64 sv = 0;
        int v = -1;
        if (q < s) {
          v = ci[q];
          const int end = mir[q];
          for (int p = rp[v] + gl; p < end; p += G) {
            const int w = __ldg(ci + p);
            if (P == 1 || part_of(w, P) == part) sv += hash_get(keys, vals, hlog, w) - 1;
          }
        }
        sv = group_sum_u64<G>(sv);
        if (gl == 0 && sv) atomicAdd(c4 + v, sv);
      }
      __syncthreads();
    }
    acc = block_sum_u64(acc, red);
    if (threadIdx.x == 0 && acc) atomicAdd(c4 + u, acc);
    __syncthreads();
  }
}

// Block per heavy root; the w range [0,u) is swept in dense shared-memory
// tiles (PACK: two 16-bit counters per word, valid since L[w] <= |N-(u)| <
// 65536). Each row keeps a cursor across tiles, so every wedge is read exactly
// twice (count, attribution). Rows are split at the first one of length >=
// kC4Long (rows of N-(u) are in ascending degree): short rows thread-per-row,
// long rows warp-cooperative.
// First index in [lo, hi) with a[i] >= key, found by the whole warp with a
// 32-ary search (one coalesced probe round per factor of 32). Warp-uniform.
__device__ __forceinline__ int warp_lower_bound(const int* __restrict__ a, int lo, int hi,
                                                int key) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) >> 5;
    const int pos = lo + step * (lane + 1) - 1;
    const bool less = pos < hi && __ldg(a + pos) < key;
    const int c = __popc(__ballot_sync(0xffffffffu, less));
    lo += c * step;
    hi = min(hi, lo + step);
  }
  const int pos = lo + lane;
  const bool less = pos < hi && __ldg(a + pos) < key;
  return lo + __popc(__ballot_sync(0xffffffffu, less));
}

// f(a[i]) for i in [st, se) by the whole warp: scalar head/tail, 16-byte
// vector body (two vectors in flight per lane).
template <class F>
__device__ __forceinline__ void warp_for_each(const int* __restrict__ a, int st, int se, F&& f) {
  const int lane = threadIdx.x & 31;
  const int a0 = min(se, (st + 3) & ~3);
  const int a1 = max(a0, se & ~3);
  if (st + lane < a0) f(__ldg(a + st + lane));
  int p = a0 + 4 * lane;
  for (; p + 128 < a1; p += 256) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(a + p));
    const int4 y = __ldg(reinterpret_cast<const int4*>(a + p + 128));
    f(x.x); f(x.y); f(x.z); f(x.w);
    f(y.x); f(y.y); f(y.z); f(y.w);
  }
  if (p < a1) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(a + p));
    f(x.x); f(x.y); f(x.z); f(x.w);
  }
  if (a1 + lane < se) f(__ldg(a + a1 + lane));
}

// Block-wide flattening of one segment per thread: writes exclusive offsets
// (g_off[0..nthreads], g_off[nthreads] = total) and per-row element bases
// g_st[r] = start - off; returns the total. Contains __syncthreads.
struct NoReserve {
  __device__ void operator()(int) const {}
};

// R(total) is called by one thread between the second and third barrier, so
// whatever it writes to shared memory is visible to the block on return.
template <class R = NoReserve>
__device__ __forceinline__ int block_flatten(int len, int start, int* g_off, int* g_st,
                                             int* wtot, R reserve = R()) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wtot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int x = lane < nw ? wtot[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < nw) wtot[lane] = xi - x;  // exclusive warp base
    if (lane == 31) {
      g_off[blockDim.x] = xi;
      reserve(xi);
    }
  }
  __syncthreads();
  const int off = wtot[wid] + incl - len;
  g_off[threadIdx.x] = off;
  g_st[threadIdx.x] = start - off;
  __syncthreads();
  return g_off[blockDim.x];
}

// Row of flattened element k: the largest r with g_off[r] <= k.
__device__ __forceinline__ int upper_row(const int* g_off, int k, int n) {
  int lo = 0, hi = n;  // invariant: g_off[lo] <= k (k >= 0 = g_off[0])
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (g_off[mid] <= k) lo = mid; else hi = mid;
  }
  return lo;
}

// Block per root, hash table in shared memory, P hash-partition passes.
// The rows of N-(u) are flattened block-wide over 16-byte quads of ci, in
// chunks of NT rows; each warp owns an equal contiguous share of the quads
// (one binary search per lane to find its first row, then a forward walk), so
// a root's work is balanced across all warps with no per-row serial loops.
template <int NT, bool LANEROW = false>
__global__ void __launch_bounds__(NT)
k_c4_block(const int* __restrict__ rp, const int* __restrict__ ci,
           const int* __restrict__ split, const int* __restrict__ mir,
           const int* __restrict__ roots, int nroots, const u64* __restrict__ wcv,
           const u32* __restrict__ parts, int max_log, int* __restrict__ next_root,
           u64* __restrict__ c4) {
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ u64 red[32];
  __shared__ int g_off[NT + 1];  // quad offsets of the chunk's rows
  __shared__ int g_st[NT];       // quad k of row r is ci quad g_st[r] + k
  __shared__ int g_sa[NT], g_sb[NT];  // row element range [sa, sb)
  __shared__ u64 rowsum[NT];
  __shared__ int wtot[32];
  __shared__ int s_root;
  const int maxcap = 1 << max_log;
  int* keys = reinterpret_cast<int*>(smem_raw);
  u32* vals = reinterpret_cast<u32*>(keys + maxcap);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  rowsum[threadIdx.x] = 0;
  while (true) {
    if (threadIdx.x == 0) s_root = atomicAdd(next_root, 1);
    __syncthreads();
    const int k = s_root;
    if (k >= nroots) break;
    const int u = roots[k];
    const u32 P = parts[u];
    const u64 per_pass = (wcv[u] + P - 1) / P;
    int hlog = 6;
    while (hlog < max_log && ((u64)1 << hlog) < 2 * per_pass) ++hlog;
    const int cap = 1 << hlog;
    const int b = rp[u], s = split[u];
    u64 acc = 0;
    // flatten rows [c0, c0 + NT) of N-(u); returns the quad count
    auto flatten = [&](int c0) -> int {
      const int q = c0 + threadIdx.x;
      int st = 0, se = 0;
      if (q < s) {
        st = rp[ci[q]];
        se = mir[q];
      }
      const int qa = st >> 2;
      const int nqd = se > st ? ((se + 3) >> 2) - qa : 0;
      g_sa[threadIdx.x] = st;
      g_sb[threadIdx.x] = se;
      return block_flatten(nqd, qa, g_off, g_st, wtot);  // g_st = qa - off
    };
    // visit every wedge target of the chunk: f(row, w)
    auto sweep_quads = [&](int T, auto&& f) {
      const int per = (T + NW - 1) / NW;
      const int k0 = wid * per, k1 = min(T, k0 + per);
      if (k0 + lane >= k1) return;
      int r = upper_row(g_off, k0 + lane, NT);
      for (int kk = k0 + lane; kk < k1; kk += 32 * kQuadsInFlight) {
        int4 v[kQuadsInFlight];
        int lt[kQuadsInFlight], ht[kQuadsInFlight], rr[kQuadsInFlight];
#pragma unroll
        for (int j = 0; j < kQuadsInFlight; ++j) {
          const int kj = kk + 32 * j;
          lt[j] = 4;
          ht[j] = 0;
          rr[j] = r;
          if (kj < k1) {
            while (g_off[r + 1] <= kj) ++r;
            rr[j] = r;
            const int e0 = (g_st[r] + kj) << 2;
            v[j] = __ldg(reinterpret_cast<const int4*>(ci + e0));
            lt[j] = g_sa[r] - e0;
            ht[j] = g_sb[r] - e0;
          }
        }
#pragma unroll
        for (int j = 0; j < kQuadsInFlight; ++j) {
          if (lt[j] <= 0 && ht[j] > 0) f(rr[j], v[j].x);
          if (lt[j] <= 1 && ht[j] > 1) f(rr[j], v[j].y);
          if (lt[j] <= 2 && ht[j] > 2) f(rr[j], v[j].z);
          if (lt[j] <= 3 && ht[j] > 3) f(rr[j], v[j].w);
        }
      }
    };
    for (u32 part = 0; part < P; ++part) {
      {
        uint4* k4 = reinterpret_cast<uint4*>(keys);
        uint4* v4 = reinterpret_cast<uint4*>(vals);
        for (int i = threadIdx.x; i < (cap >> 2); i += NT) {
          k4[i] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
          v4[i] = make_uint4(0, 0, 0, 0);
        }
      }
      // LANEROW (the <= 2048-wedge classes, whose rows have similar degree):
      // rows of a chunk in lane groups: G = the largest power of two with
      // rows x G <= NT lanes per row, each group streaming its row's
      // segment (16-byte loads at stride G) — no per-quad row search/masks
      auto group_stream = [&](int c0, auto&& f) {
        const int nrows = min(NT, s - c0);
        int G = 1;
        while (G < 32 && nrows * (G * 2) <= NT) G *= 2;
        const int row = threadIdx.x / G, sub = threadIdx.x & (G - 1);
        const int q = c0 + row;
        if (row < nrows) {
          const int st = rp[ci[q]], se = mir[q];
          if (se > st) {
            const int a0 = min(se, (st + 3) & ~3), a1 = max(a0, se & ~3);
            for (int p = st + sub; p < a0; p += G) f(__ldg(ci + p));
            for (int p = a0 + 4 * sub; p < a1; p += 4 * G) {
              const int4 x = __ldg(reinterpret_cast<const int4*>(ci + p));
              f(x.x); f(x.y); f(x.z); f(x.w);
            }
            for (int p = a1 + sub; p < se; p += G) f(__ldg(ci + p));
          }
        }
        return G;
      };
      if (LANEROW) {
        __syncthreads();  // the clear before any insert
        for (int c0 = b; c0 < s; c0 += NT)
          group_stream(c0, [&](int w) {
            if (P == 1 || part_of(w, P) == part) hash_insert(keys, vals, hlog, w);
          });
        __syncthreads();
      } else {
        // count pass (block_flatten's barriers order the clear before inserts)
        for (int c0 = b; c0 < s; c0 += NT) {
          const int T = flatten(c0);
          sweep_quads(T, [&](int, int w) {
            if (P == 1 || part_of(w, P) == part) hash_insert(keys, vals, hlog, w);
          });
          __syncthreads();
        }
      }
      for (int i = threadIdx.x; i < cap; i += NT) {
        const u32 l = vals[i];
        if (l >= 2) {
          const u64 c = (u64)l * (l - 1) / 2;
          acc += c;
          atomicAdd(c4 + keys[i], c);
        }
      }
      // attribution pass: c4[v] += sum_w (L[w] - 1)
      if (LANEROW)
      for (int c0 = b; c0 < s; c0 += NT) {
        u64 sv = 0;
        const int G = group_stream(c0, [&](int w) {
          if (P == 1 || part_of(w, P) == part) sv += hash_get(keys, vals, hlog, w) - 1;
        });
        for (int o = G / 2; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
        const int row = threadIdx.x / G;
        if ((threadIdx.x & (G - 1)) == 0 && c0 + row < s && sv) atomicAdd(c4 + ci[c0 + row], sv);
      }
      else
      for (int c0 = b; c0 < s; c0 += NT) {
        const int T = flatten(c0);
        int cr = -1;
        u64 part_sum = 0;
        sweep_quads(T, [&](int r, int w) {
          if (P == 1 || part_of(w, P) == part) {
            if (r != cr) {
              if (part_sum) smem_add_u64(rowsum + cr, part_sum);
              part_sum = 0;
              cr = r;
            }
            part_sum += hash_get(keys, vals, hlog, w) - 1;
          }
        });
        if (part_sum) smem_add_u64(rowsum + cr, part_sum);
        __syncthreads();
        const int q = c0 + threadIdx.x;
        if (q < s && rowsum[threadIdx.x]) atomicAdd(c4 + ci[q], rowsum[threadIdx.x]);
        rowsum[threadIdx.x] = 0;
      }
      __syncthreads();
    }
    acc = block_sum_u64(acc, red);
    if (threadIdx.x == 0 && acc) atomicAdd(c4 + u, acc);
    __syncthreads();
  }
}

// Absolute tile boundaries of the active rows, shared by every dense root:
// bnd[k * nact + v] = first position in N(v) with id >= tb[k] (k = 0..K-1,
// tb = the banded tile starts). A row's segment in a tile is then two
// independent loads instead of a dependent binary search per (root, row, tile).
__global__ void k_tile_bounds(const int* __restrict__ rp, const int* __restrict__ ci, int nact,
                              int K, const int* __restrict__ tb, int* __restrict__ bnd) {
  const long long total = (long long)K * nact;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i / nact);
    const int v = (int)(i - (long long)k * nact);
    bnd[i] = k == 0 ? rp[v] : lower_bound_i32(ci, rp[v], rp[v + 1], tb[k]);
  }
}

// Degree bands of the active range (ids ascending in degree): out[0] = first
// id with degree > 15, out[1] > 255, out[2] > 65535.
__global__ void k_degree_bands(const int* __restrict__ rp, int nact, int* __restrict__ out) {
  if (threadIdx.x >= 3 || blockIdx.x) return;
  const int lim = threadIdx.x == 0 ? 15 : threadIdx.x == 1 ? 255 : 65535;
  int lo = 0, hi = nact;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rp[mid + 1] - rp[mid] <= lim) lo = mid + 1; else hi = mid;
  }
  out[threadIdx.x] = lo;
}

// Optional phase timers for the dense kernel (profiling builds only,
// -DFGLT_DENSE_PROF): per-warp clock deltas summed over the grid and printed
// by the last block. Phases: 0 zero, 1 count work, 2 count barrier, 3 sweep,
// 4 attribution work, 5 attribution barrier, 6 root setup.
#ifdef FGLT_DENSE_PROF
__device__ unsigned long long g_dense_prof[16];
__device__ unsigned int g_dense_done;
#define DPROF_MARK(k)                                                       \
  do {                                                                      \
    const long long _t = clock64();                                         \
    if (lane == 0) atomicAdd(g_dense_prof + (k), (unsigned long long)(_t - _pt)); \
    _pt = _t;                                                               \
  } while (0)
#else
#define DPROF_MARK(k) do {} while (0)
#endif

template <bool PACK, int NT, bool SPLIT = false>
__global__ void __launch_bounds__(NT, 1024 / NT)
k_c4_dense(const int* __restrict__ rp, const int* __restrict__ ci,
           const int* __restrict__ split, const int* __restrict__ mir,
           const int* __restrict__ roots, int nroots, int* __restrict__ cursor,
           long long cursor_stride, const int* __restrict__ bnd, long long bnd_stride,
           const int* __restrict__ tb, int b4, int b8, int b16, int* __restrict__ next_root,
           u64* __restrict__ c4, int split_kt_arg) {
  // roots are sorted by work (largest first) and handed out dynamically; with
  // SPLIT (requires bnd) the work items are (root, tile) pairs, item
  // k * split_kt + t, so a few huge roots spread over all SMs
  const int split_kt = SPLIT ? split_kt_arg : 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ u64 red[32];
  // per-warp flattening tables of the quad-flattened batches (unused, and
  // reduced to one row, in lane-row mode: more shared memory for the tiles)
  constexpr int NW = FGLT_BATCH_LANE_ROW ? 1 : NT / 32;
  __shared__ u64 rsum[NW][32];
  __shared__ int bst_all[NW][32];
  __shared__ int boff_all[NW][33];
  __shared__ int bsa_all[NW][32];  // per-batch row [start, end) in ci
  __shared__ int bsb_all[NW][32];
  __shared__ int next_batch[2];
  __shared__ int next_giant[2];
  u32* L = reinterpret_cast<u32*>(smem_raw);
  int* cur = cursor + (long long)blockIdx.x * 2 * cursor_stride;
  int* segend = cur + cursor_stride;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64* rs = rsum[wid % NW];
  int* bst = bst_all[wid % NW];
  int* boff = boff_all[wid % NW];
  int* bsa = bsa_all[wid % NW];
  int* bsb = bsb_all[wid % NW];
  // counters of the current tile: 2^sh per 32-bit word, 32 >> sh bits each
  int sh = 0;
  constexpr int kTileWords = (NT == kC4DenseThreadsS ? kC4TileBytesS : kC4TileBytes) / 4;
  auto inc = [&](int off) {
    FGLT_BOUNDS(off >= 0 && (off >> sh) < kTileWords, "c4 tile inc", off, sh);
    atomicAdd(L + (off >> sh), 1u << ((off & ((1 << sh) - 1)) << (5 - sh)));
  };
  auto get = [&](int off) -> u32 {
    FGLT_BOUNDS(off >= 0 && (off >> sh) < kTileWords, "c4 tile get", off, sh);
    const u32 x = L[off >> sh] >> ((off & ((1 << sh) - 1)) << (5 - sh));
    return sh ? x & ((1u << (32 >> sh)) - 1u) : x;
  };
  rs[lane] = 0;
#ifdef FGLT_DENSE_PROF
  long long _pt = clock64();
#endif
  __shared__ int s_root;
  while (true) {
    if (threadIdx.x == 0) s_root = atomicAdd(next_root, 1);
    __syncthreads();
    const int item = s_root;
    const int k = split_kt ? item / split_kt : item;
    if (k >= nroots) break;
    const int t_only = split_kt ? item % split_kt : 0;
    const int u = roots[k];
    if (split_kt && t_only > 0 && tb[t_only] >= u) {  // root has no such tile
      __syncthreads();
      continue;
    }
    const int b = rp[u], nq = split[u] - b;
    // first long row (rows in N-(u) have nondecreasing degree)
    int lo_q = 0, hi_q = nq;
    while (lo_q < hi_q) {
      const int mid = (lo_q + hi_q) >> 1;
      const int v = ci[b + mid];
      if (rp[v + 1] - rp[v] < kC4Long) lo_q = mid + 1; else hi_q = mid;
    }
    const int qs = lo_q;
    // giant rows: expected >= 512 elements per tile -> warp per row
    int ntiles = 0;
    while (tb[ntiles] < u) ++ntiles;
    const int giant_deg =
        max(kC4Long, (NT == kC4DenseThreadsS ? kC4GiantPerTile : kC4GiantPerTileBig) * ntiles);
    hi_q = nq;
    while (lo_q < hi_q) {
      const int mid = (lo_q + hi_q) >> 1;
      const int v = ci[b + mid];
      if (rp[v + 1] - rp[v] < giant_deg) lo_q = mid + 1; else hi_q = mid;
    }
    const int qg = lo_q;
    // batches of kBatchRows long rows (kBatchG lanes per row in lane-row mode)
    const int nb = (qg - qs + kBatchRows - 1) / kBatchRows;
    // short rows walk with per-row cursors across the tiles; a split item
    // (one tile of a root) takes their segments from the tile boundaries
    if (!split_kt)
      for (int q = threadIdx.x; q < nq; q += blockDim.x) cur[q] = rp[ci[b + q]];
    u64 acc = 0;
    const int t_end = split_kt ? t_only + 1 : ntiles;
    for (int t = split_kt ? t_only : 0; t < t_end; ++t) {
      const int lo = tb[t], hi = min(tb[t + 1], u);
      sh = lo < b4 ? 3 : lo < b8 ? 2 : lo < b16 ? 1 : 0;  // PACK roots never reach b16
      const int words = (hi - lo + (1 << sh) - 1) >> sh;
      const long long kb_lo = t, kb_hi = t + 1;
      {
        uint4* L4 = reinterpret_cast<uint4*>(L);
        const int n4 = (words + 3) >> 2;
        DPROF_MARK(6);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) L4[i] = make_uint4(0, 0, 0, 0);
      }
      if (threadIdx.x == 0) {
        next_batch[0] = next_batch[1] = 0;
        next_giant[0] = next_giant[1] = 0;
      }
      __syncthreads();
      DPROF_MARK(0);
      // ---- count pass: giant rows (warp per row, 16-byte loads, largest
      // first), then long-row batches, then short rows
      while (true) {
        int gi = 0;
        if (lane == 0) gi = atomicAdd(next_giant, 1);
        gi = __shfl_sync(0xffffffffu, gi, 0);
        const int q = nq - 1 - gi;
        if (q < qg) break;
        const int em = mir[b + q];
        int st, se;
        if (bnd) {
          const int v = ci[b + q];
          st = bnd[kb_lo * bnd_stride + v];
          se = hi >= u ? em : min(em, bnd[kb_hi * bnd_stride + v]);
          if (lane == 0) cur[q] = st;
        } else {
          st = cur[q];
          se = hi >= u ? em : warp_lower_bound(ci, st, em, hi);
        }
        if (lane == 0) segend[q] = se;
        warp_for_each(ci, st, se, [&](int w) { inc(w - lo); });
      }
      DPROF_MARK(7);
      for (int q = threadIdx.x; q < qs; q += blockDim.x) {
        const int end = mir[b + q];
        if (split_kt) {  // segment from the tile boundaries
          const int v = ci[b + q];
          const int st = bnd[kb_lo * bnd_stride + v];
          const int se = hi >= u ? end : min(end, bnd[kb_hi * bnd_stride + v]);
          for (int p = st; p < se; ++p) inc(ci[p] - lo);
          continue;
        }
        for (int p = cur[q]; p < end; ++p) {
          const int w = ci[p];
          if (w >= hi) break;
          inc(w - lo);
        }
      }
      DPROF_MARK(8);
      while (true) {
        int bt = 0;
        if (lane == 0) bt = atomicAdd(next_batch, 1);
        bt = __shfl_sync(0xffffffffu, bt, 0);
        if (bt >= nb) break;
        bt = nb - 1 - bt;  // largest rows first
        const int q = qs + bt * kBatchRows + lane / kBatchG;
        const bool valid = q < qg;
        int st = 0, se = 0;
        if (valid) {
          const int em = mir[b + q];
          if (bnd) {
            const int v = ci[b + q];
            st = bnd[kb_lo * bnd_stride + v];
            se = hi >= u ? em : min(em, bnd[kb_hi * bnd_stride + v]);
          } else {
            st = cur[q];
            se = hi >= u ? em : lower_bound_i32(ci, st, em, hi);
          }
        }
        // a row's lanes all read the old cursor before any of them writes
        __syncwarp();
        if (valid && (lane & (kBatchG - 1)) == 0) {
          cur[q] = st;
          segend[q] = se;
        }
#if FGLT_BATCH_LANE_ROW
        // lane per row: the batch's rows are consecutive in N-(u), so their
        // degrees (and tile segments) are similar; each lane streams its own
        // segment with 16-byte loads, no flattening bookkeeping per quad
#if FGLT_BATCH_MASKED
        if (se > st) {
          // aligned quads [st >> 2, (se + 3) >> 2) at stride kBatchG; elements
          // outside [st, se) masked; a round's loads are all issued before use
          const int sub = lane & (kBatchG - 1);
          const int4* q4 = reinterpret_cast<const int4*>(ci);
          const int qe = (se + 3) >> 2;
          const u32 len = (u32)(se - st);
          for (int k = (st >> 2) + sub; k < qe; k += kBatchG * kQuadsInFlight) {
            int4 x[kQuadsInFlight];
#pragma unroll
            for (int j = 0; j < kQuadsInFlight; ++j)
              if (k + j * kBatchG < qe) x[j] = __ldg(q4 + k + j * kBatchG);
#pragma unroll
            for (int j = 0; j < kQuadsInFlight; ++j) {
              const int kj = k + j * kBatchG;
              if (kj < qe) {
                const int d = (kj << 2) - st;  // segment position of the quad's first element
                if ((u32)d < len) inc(x[j].x - lo);
                if ((u32)(d + 1) < len) inc(x[j].y - lo);
                if ((u32)(d + 2) < len) inc(x[j].z - lo);
                if ((u32)(d + 3) < len) inc(x[j].w - lo);
              }
            }
          }
        }
        continue;
#endif
        if (se > st) {
          const int sub = lane & (kBatchG - 1);
          const int a0 = min(se, (st + 3) & ~3), a1 = max(a0, se & ~3);
          for (int p = st + sub; p < a0; p += kBatchG) inc(__ldg(ci + p) - lo);
          int p = a0 + 4 * sub;
          for (; p + 4 * kBatchG < a1; p += 8 * kBatchG) {
            const int4 x = __ldg(reinterpret_cast<const int4*>(ci + p));
            const int4 y = __ldg(reinterpret_cast<const int4*>(ci + p + 4 * kBatchG));
            inc(x.x - lo); inc(x.y - lo); inc(x.z - lo); inc(x.w - lo);
            inc(y.x - lo); inc(y.y - lo); inc(y.z - lo); inc(y.w - lo);
          }
          if (p < a1) {
            const int4 x = __ldg(reinterpret_cast<const int4*>(ci + p));
            inc(x.x - lo); inc(x.y - lo); inc(x.z - lo); inc(x.w - lo);
          }
          for (int pt = a1 + sub; pt < se; pt += kBatchG) inc(__ldg(ci + pt) - lo);
        }
        continue;
#endif
        // flattened over 16-byte quads of ci: quad k of row r is ci[4 (bst[r] + k)]
        // + 0..3, elements outside [st, se) masked
        const int qa = st >> 2;
        const int nqd = se > st ? ((se + 3) >> 2) - qa : 0;
        int T;
        const int off = flat_prefix(nqd, &T);
        bst[lane] = qa - off;
        boff[lane] = off;
        bsa[lane] = st;
        bsb[lane] = se;
        if (lane == 0) boff[32] = T;
        __syncwarp();
        int r = 0;
        for (int kk = lane; kk < T; kk += 32 * kQuadsInFlight) {
          int4 v[kQuadsInFlight];
          int lt[kQuadsInFlight], ht[kQuadsInFlight];
#pragma unroll
          for (int j = 0; j < kQuadsInFlight; ++j) {
            const int kj = kk + 32 * j;
            lt[j] = 4;
            ht[j] = 0;
            if (kj < T) {
              while (boff[r + 1] <= kj) ++r;
              const int e0 = (bst[r] + kj) << 2;
              v[j] = __ldg(reinterpret_cast<const int4*>(ci + e0));
              lt[j] = bsa[r] - e0;
              ht[j] = bsb[r] - e0;
            }
          }
#pragma unroll
          for (int j = 0; j < kQuadsInFlight; ++j) {
            if (lt[j] <= 0 && ht[j] > 0) inc(v[j].x - lo);
            if (lt[j] <= 1 && ht[j] > 1) inc(v[j].y - lo);
            if (lt[j] <= 2 && ht[j] > 2) inc(v[j].z - lo);
            if (lt[j] <= 3 && ht[j] > 3) inc(v[j].w - lo);
          }
        }
        __syncwarp();
      }
      DPROF_MARK(1);
      __syncthreads();
      DPROF_MARK(2);
      {
        // 16-byte sweep; words past the tile end were zeroed with the tile
        const uint4* L4 = reinterpret_cast<const uint4*>(L);
        const int n4 = (words + 3) >> 2;
        // some counter >= 2 in the word
        const u32 ge2 = sh == 3 ? 0xeeeeeeeeu : sh == 2 ? 0xfefefefeu : sh == 1 ? 0xfffefffeu
                                                                              : 0xfffffffeu;
        const int bits = 32 >> sh;
        const u32 vmask = sh ? (1u << bits) - 1u : 0xffffffffu;
        for (int i4 = threadIdx.x; i4 < n4; i4 += blockDim.x) {
          const uint4 v = L4[i4];
          if (((v.x | v.y | v.z | v.w) & ge2) == 0) continue;
          const u32 xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            u32 x = xs[j];
            if ((x & ge2) == 0) continue;
            const int base = lo + ((4 * i4 + j) << sh);
            // one flag bit at the low end of every counter >= 2, visited by ffs
            u32 f = sh == 0 ? 1u : 0u;
            if (sh) {
              u32 hi = x & ge2;  // bits above each counter's lowest
#pragma unroll
              for (int t = 1; t < 16; t <<= 1)
                if (t < bits) hi |= hi >> t;
              f = hi & (ge2 >> 1) & ~(ge2 >> 1 & ge2);  // keep each counter's low bit
            }
            while (f) {
              const int b = __ffs(f) - 1;
              f &= f - 1;
              const u32 l = (x >> b) & vmask;
              const u64 c = (u64)l * (l - 1) / 2;
              acc += c;
              atomicAdd(c4 + base + (b >> (5 - sh)), c);
            }
          }
        }
      }
      DPROF_MARK(3);
      // ---- attribution pass: c4[v] += sum (L[w] - 1); cursors advance
      while (true) {
        int gi = 0;
        if (lane == 0) gi = atomicAdd(next_giant + 1, 1);
        gi = __shfl_sync(0xffffffffu, gi, 0);
        const int q = nq - 1 - gi;
        if (q < qg) break;
        const int st = cur[q];
        const int se = segend[q];
        u64 sv = 0;
        warp_for_each(ci, st, se, [&](int w) { sv += get(w - lo) - 1; });
        sv = warp_sum_u64(sv);
        if (lane == 0) {
          if (sv) atomicAdd(c4 + ci[b + q], sv);
          cur[q] = se;
        }
      }
      DPROF_MARK(9);
      for (int q = threadIdx.x; q < qs; q += blockDim.x) {
        const int end = mir[b + q];
        u64 sv = 0;
        if (split_kt) {
          const int v = ci[b + q];
          const int st = bnd[kb_lo * bnd_stride + v];
          const int se = hi >= u ? end : min(end, bnd[kb_hi * bnd_stride + v]);
          for (int p = st; p < se; ++p) sv += get(ci[p] - lo) - 1;
        } else {
          int p = cur[q];
          for (; p < end; ++p) {
            const int w = ci[p];
            if (w >= hi) break;
            sv += get(w - lo) - 1;
          }
          cur[q] = p;
        }
        if (sv) atomicAdd(c4 + ci[b + q], sv);
      }
      DPROF_MARK(10);
      while (true) {
        int bt = 0;
        if (lane == 0) bt = atomicAdd(next_batch + 1, 1);
        bt = __shfl_sync(0xffffffffu, bt, 0);
        if (bt >= nb) break;
        bt = nb - 1 - bt;  // largest rows first
        const int q = qs + bt * kBatchRows + lane / kBatchG;
        const bool valid = q < qg;
        const int st = valid ? cur[q] : 0;
        const int se = valid ? segend[q] : 0;
#if FGLT_BATCH_LANE_ROW
        {
          const int sub = lane & (kBatchG - 1);
          u64 sv = 0;
          typename std::conditional<PACK, u32, u64>::type ps = 0;
#if FGLT_BATCH_MASKED
          if (se > st) {
            const int4* q4 = reinterpret_cast<const int4*>(ci);
            const int qe = (se + 3) >> 2;
            const u32 len = (u32)(se - st);
            for (int k = (st >> 2) + sub; k < qe; k += kBatchG * kQuadsInFlight) {
              int4 x[kQuadsInFlight];
#pragma unroll
              for (int j = 0; j < kQuadsInFlight; ++j)
                if (k + j * kBatchG < qe) x[j] = __ldg(q4 + k + j * kBatchG);
#pragma unroll
              for (int j = 0; j < kQuadsInFlight; ++j) {
                const int kj = k + j * kBatchG;
                if (kj < qe) {
                  const int d = (kj << 2) - st;
                  if ((u32)d < len) ps += get(x[j].x - lo) - 1;
                  if ((u32)(d + 1) < len) ps += get(x[j].y - lo) - 1;
                  if ((u32)(d + 2) < len) ps += get(x[j].z - lo) - 1;
                  if ((u32)(d + 3) < len) ps += get(x[j].w - lo) - 1;
                }
              }
              if (PACK) { sv += ps; ps = 0; }
            }
          }
#else
          if (se > st) {
            const int a0 = min(se, (st + 3) & ~3), a1 = max(a0, se & ~3);
            for (int p = st + sub; p < a0; p += kBatchG) ps += get(__ldg(ci + p) - lo) - 1;
            int p = a0 + 4 * sub;
            for (; p + 4 * kBatchG < a1; p += 8 * kBatchG) {
              const int4 x = __ldg(reinterpret_cast<const int4*>(ci + p));
              const int4 y = __ldg(reinterpret_cast<const int4*>(ci + p + 4 * kBatchG));
              ps += get(x.x - lo) + get(x.y - lo) + get(x.z - lo) + get(x.w - lo) - 4;
              ps += get(y.x - lo) + get(y.y - lo) + get(y.z - lo) + get(y.w - lo) - 4;
              if (PACK) { sv += ps; ps = 0; }
            }
            if (p < a1) {
              const int4 x = __ldg(reinterpret_cast<const int4*>(ci + p));
              ps += get(x.x - lo) + get(x.y - lo) + get(x.z - lo) + get(x.w - lo) - 4;
            }
            for (int pt = a1 + sub; pt < se; pt += kBatchG) ps += get(__ldg(ci + pt) - lo) - 1;
          }
#endif
          sv += ps;
#pragma unroll
          for (int o = kBatchG / 2; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
          if (valid && sub == 0) {
            if (sv) atomicAdd(c4 + ci[b + q], sv);
            cur[q] = se;
          }
        }
        continue;
#endif
        const int qa = st >> 2;
        const int nqd = se > st ? ((se + 3) >> 2) - qa : 0;
        int T;
        const int off = flat_prefix(nqd, &T);
        bst[lane] = qa - off;
        boff[lane] = off;
        bsa[lane] = st;
        bsb[lane] = se;
        if (lane == 0) boff[32] = T;
        __syncwarp();
        int r = 0, cr = 0;
        u64 part = 0;
        for (int kk = lane; kk < T; kk += 32 * kQuadsInFlight) {
          int4 v[kQuadsInFlight];
          int lt[kQuadsInFlight], ht[kQuadsInFlight], rr[kQuadsInFlight];
#pragma unroll
          for (int j = 0; j < kQuadsInFlight; ++j) {
            const int kj = kk + 32 * j;
            lt[j] = 4;
            ht[j] = 0;
            rr[j] = r;
            if (kj < T) {
              while (boff[r + 1] <= kj) ++r;
              rr[j] = r;
              const int e0 = (bst[r] + kj) << 2;
              v[j] = __ldg(reinterpret_cast<const int4*>(ci + e0));
              lt[j] = bsa[r] - e0;
              ht[j] = bsb[r] - e0;
            }
          }
#pragma unroll
          for (int j = 0; j < kQuadsInFlight; ++j) {
            if (ht[j] <= 0) break;
            // PACK counters are < 2^16, so four of them fit 32 bits
            typename std::conditional<PACK, u32, u64>::type ps = 0;
            if (lt[j] <= 0) ps += get(v[j].x - lo) - 1;
            if (lt[j] <= 1 && ht[j] > 1) ps += get(v[j].y - lo) - 1;
            if (lt[j] <= 2 && ht[j] > 2) ps += get(v[j].z - lo) - 1;
            if (ht[j] > 3) ps += get(v[j].w - lo) - 1;
            if (rr[j] != cr) {
              if (part) smem_add_u64(rs + cr, part);
              part = 0;
              cr = rr[j];
            }
            part += ps;
          }
        }
        if (part) smem_add_u64(rs + cr, part);
        __syncwarp();
        if (valid) {
          if (rs[lane]) atomicAdd(c4 + ci[b + q], rs[lane]);
          cur[q] = se;
        }
        rs[lane] = 0;
        __syncwarp();
      }
      DPROF_MARK(4);
      __syncthreads();
      DPROF_MARK(5);
    }
    acc = block_sum_u64(acc, red);
    if (threadIdx.x == 0 && acc) atomicAdd(c4 + u, acc);
    __syncthreads();
  }
#ifdef FGLT_DENSE_PROF
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&g_dense_done, 1u) == gridDim.x - 1) {
    unsigned long long t = 0;
    for (int k = 0; k < 11; ++k) t += g_dense_prof[k];
    printf("dense phases (warp-cycles %%): zero %.1f | count: giant %.1f short %.1f batch %.1f bar %.1f | sweep %.1f | attr: giant %.1f short %.1f batch %.1f bar %.1f | setup %.1f\n",
           100.0 * g_dense_prof[0] / t, 100.0 * g_dense_prof[7] / t, 100.0 * g_dense_prof[8] / t,
           100.0 * g_dense_prof[1] / t, 100.0 * g_dense_prof[2] / t, 100.0 * g_dense_prof[3] / t,
           100.0 * g_dense_prof[9] / t, 100.0 * g_dense_prof[10] / t, 100.0 * g_dense_prof[4] / t,
           100.0 * g_dense_prof[5] / t, 100.0 * g_dense_prof[6] / t);
    for (int k = 0; k < 16; ++k) g_dense_prof[k] = 0;
    g_dense_done = 0;
  }
#endif
}

// ================================================== diamonds and 4-cliques
// Root u, S = N+(u) (sorted, ids > u). A probe of N+(x) for x = S[a] against
// S[a+1..] finds every triangle {u, x, y} whose lowest vertex is u exactly
// once. Per triangle (paper D4 term; reference compute_d13, kernels.cpp:
// 207-232, restated as sum over triangles of (C3(opposite edge) - 1)):
//   d13[u] += C3(x,y)-1, d13[x] += C3(u,y)-1, d13[y] += C3(u,x)-1.
// The same probe sets the bit (a,b) of the induced subgraph G[S] (a bitmap
// row per member). Every 4-clique has a unique lowest vertex u and is a
// triangle of G[S]; for member a, t_a = (1/2) sum_{b in row a}
// popc(row_a & row_b) is the number of G[S]-triangles through a, so
// d15[S[a]] += t_a and d15[u] += sum_a t_a / 3 (reference compute_d15,
// kernels.cpp:234-288, same counts).

// ---- triangle list. The triangle pass of block roots (|S| > 32) records
// every triangle {u, S[a], S[b]} it finds as (a | b << 16, CSR position of
// (S[a], S[b])) in a device pool, in per-root pieces; the diamond pass then
// reads the list (k_diamond_list) instead of probing again. A block reserves
// pool space for a probe/pair phase up front (an upper bound: one record per
// probed element or pair test), returns the unused tail after the phase and
// publishes the phase's records as one piece. Roots whose records did not fit
// (pool or piece table exhausted, or |S| > kTriListMaxS) are flagged and keep
// the probing diamond pass; pieces of flagged roots are ignored.
constexpr int kTriListMaxS = 8192;              // member ids fit 16 bits, sD fits smem
constexpr unsigned long long kTriListChunk = 1ull << 13;  // records per pool grab (64 KB)

struct TriPiece {
  unsigned long long start;  // first record
  int u;                     // root
  unsigned count;            // records
};

// Warp roots (|S| <= 32) append into per-warp chunks of kTriListWarpChunk
// records instead of pieces: a header record (0x80000000 | count, root) then
// the root's records; a chunk directory entry is written when the warp
// retires the chunk.
constexpr unsigned kTriListWarpChunk = 4096;

struct TriChunk {
  unsigned long long start;
  unsigned used;
  unsigned pad;
};

struct TriList {
  uint2* rec = nullptr;                 // nullptr: no list
  unsigned long long cap = 0;           // pool records
  unsigned long long* top = nullptr;    // pool bump pointer
  TriPiece* pieces = nullptr;
  unsigned* npieces = nullptr;
  unsigned pieces_cap = 0;
  unsigned char* fail = nullptr;        // per root: 1 = not (fully) listed
  TriChunk* chunks = nullptr;           // warp-root chunk directory
  unsigned* nchunks = nullptr;
  unsigned chunks_cap = 0;
};

// Thread per root for |S| <= tiny_s <= kRootsTiny (most roots of low-degree
// graphs: RGG's mean |N+(u)| is 1.5; the host enables it when d_max is small,
// since on power-law graphs the members' probe lists are long and a thread
// walking them serially loses to the warp): S, the sums and G[S] (8 x 8 bits)
// live in registers (static indexing only); the same per-triangle updates as
// k_roots_warp. Tiny roots never use the triangle list: the diamond pass
// re-probes them with this kernel (kD13), and k_roots_warp skips them in
// both passes.
#ifndef FGLT_ROOTS_TINY
#define FGLT_ROOTS_TINY 8
#endif
constexpr int kRootsTiny = FGLT_ROOTS_TINY;
static_assert(kRootsTiny <= 8, "G[S] rows are 8-bit fields of one u64");
template <bool kC3, bool kD13, bool kD15>
__global__ void __launch_bounds__(256) k_roots_tiny(const int* __restrict__ rp,
                                                    const int* __restrict__ ci,
                                                    const int* __restrict__ split,
                                                    const int* __restrict__ send,
                                                    u32* __restrict__ C3f,
                                                    const int* __restrict__ roots, int nroots,
                                                    u64* __restrict__ d13, u64* __restrict__ d15) {
  // roots: the tiny bin, |N+(u)| <= kRootsTiny
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nroots; k += gridDim.x * blockDim.x) {
    const int u = roots[k];
    const int s0 = split[u];
    const int s = send[u] - s0;
    int S[kRootsTiny];
    u32 cu[kRootsTiny];  // kD13: C3(u, S[a]); kC3: triangles on edge (u, S[a])
    u64 da[kRootsTiny];  // kD13: d13 partial of S[a]
#pragma unroll
    for (int a = 0; a < kRootsTiny; ++a) {
      S[a] = a < s ? __ldg(ci + s0 + a) : -1;
      cu[a] = kD13 && a < s ? C3f[s0 + a] : 0u;
      da[a] = 0;
    }
    const int smax = __ldg(ci + s0 + s - 1);
    u64 g = 0;  // G[S]: bit 8a + b
    u64 tu = 0;
#pragma unroll
    for (int a = 0; a + 1 < kRootsTiny; ++a) {
      if (a + 1 >= s) break;
      const int x = S[a];
      const int e = rp[x + 1];
      for (int p = split[x]; p < e; ++p) {
        const int y = __ldg(ci + p);
        if (y > smax) break;
        int bi = -1;
#pragma unroll
        for (int b = a + 1; b < kRootsTiny; ++b)
          if (S[b] == y) bi = b;
        if (bi < 0) continue;
        // triangle {u, S[a], S[bi]}; (S[a], S[bi]) is CSR slot p
        if (kD15) g |= (1ull << (8 * a + bi)) | (1ull << (8 * bi + a));
        if (kC3) {
          atomicAdd(C3f + p, 1u);
          ++cu[a];
#pragma unroll
          for (int b = a + 1; b < kRootsTiny; ++b) cu[b] += b == bi;
        }
        if (kD13) {
          tu += (u64)__ldg(C3f + p) - 1;
          u32 cb = 0;
#pragma unroll
          for (int b = a + 1; b < kRootsTiny; ++b) {
            if (b == bi) {
              cb = cu[b];
              da[b] += (u64)cu[a] - 1;
            }
          }
          da[a] += (u64)cb - 1;
        }
      }
    }
    u64 tot = 0;
#pragma unroll
    for (int a = 0; a < kRootsTiny; ++a) {
      if (a >= s) break;
      if (kC3 && cu[a]) atomicAdd(C3f + s0 + a, cu[a]);
      if (kD13 && da[a]) atomicAdd(d13 + S[a], da[a]);
      if (kD15) {
        const u32 row = (u32)(g >> (8 * a)) & 0xffu;
        u32 t = 0;
#pragma unroll
        for (int b = 0; b < kRootsTiny; ++b)
          if (row >> b & 1u) t += __popc(row & ((u32)(g >> (8 * b)) & 0xffu));
        if (t / 2) atomicAdd(d15 + S[a], (u64)(t / 2));
        tot += t / 2;
      }
    }
    if (kD13 && tu) atomicAdd(d13 + u, tu);
    if (kD15 && tot) atomicAdd(d15 + u, tot / 3);
  }
}

// Warp per root, |S| <= 32: rows are single words.
constexpr int kRootsWarpInts = 32 * 5 + 33 + 1;  // sS, sC, rows, fbase, foff(33), fsplit, wcnt
template <bool kC3, bool kD13, bool kD15>
__global__ void __launch_bounds__(256, 8) k_roots_warp(const int* __restrict__ rp, const int* __restrict__ ci,
                             const int* __restrict__ split, const int* __restrict__ send,
                             u32* __restrict__ C3f,
                             const int* __restrict__ roots, int nroots,
                             u64* __restrict__ d13, u64* __restrict__ d15,
                             const unsigned long long* __restrict__ hub,
                             const int* __restrict__ hub_base, int hb, int hub_force,
                             TriList tl) {
  // kC3: per-edge triangle counts (atomics into C3f) — the triangle pass.
  // kD13: diamonds from the final C3 — a later pass (needs complete C3).
  // Members that are hubs may test their pairs against the hub rows instead
  // of probing (see k_roots_block).
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  u64* sD = reinterpret_cast<u64*>(smem_raw) + wib * 32;
  int* sS = reinterpret_cast<int*>(reinterpret_cast<u64*>(smem_raw) + (blockDim.x >> 5) * 32) +
            wib * kRootsWarpInts;
  u32* sC = reinterpret_cast<u32*>(sS + 32);
  u32* rows = sC + 32;
  int* fbase = reinterpret_cast<int*>(rows + 32);  // per-warp flattening tables
  int* foff = fbase + 32;                           // 33 entries
  int* fsplit = foff + 33;                          // pair rows: split[S[a]]
  unsigned* wcnt = reinterpret_cast<unsigned*>(fsplit + 32);  // records of the current root
  const int warps = (gridDim.x * blockDim.x) >> 5;
  // this warp's triangle-list chunk [cb, ce), write cursor wt (warp-uniform)
  unsigned long long cb = 0, ce = 0, wt = 0;
  bool wfail = !(kC3 && tl.rec);
  auto retire = [&]() {
    if (wt > cb && lane == 0) {
      const unsigned ci_ = atomicAdd(tl.nchunks, 1u);
      if (ci_ < tl.chunks_cap) tl.chunks[ci_] = TriChunk{cb, (unsigned)(wt - cb), 0u};
    }
  };
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nroots; k += warps) {
    const int u = roots[k];
    if (kD13 && tl.rec && !tl.fail[u]) continue;  // listed: k_diamond_wlist handles it
    const int s0 = split[u];
    const int s = send[u] - s0;
    // reserve room for a header and up to C(s,2) records of this root
    bool listing = false;
    if (kC3 && tl.rec) {
      const unsigned long long need = 1 + (unsigned long long)s * (s - 1) / 2;
      if (!wfail && ce - wt < need) {
        retire();
        unsigned long long st0 = 0;
        if (lane == 0) st0 = atomicAdd(tl.top, (unsigned long long)kTriListWarpChunk);
        st0 = __shfl_sync(0xffffffffu, st0, 0);
        if (st0 + kTriListWarpChunk > tl.cap) {
          wfail = true;
          cb = ce = wt = 0;
        } else {
          cb = wt = st0;
          ce = st0 + kTriListWarpChunk;
        }
      }
      listing = !wfail;
      if (lane == 0) {
        *wcnt = 0;
        if (!listing) tl.fail[u] = 1;
      }
    }
    if (lane < s) {
      sS[lane] = ci[s0 + lane];
      if (kD13) sC[lane] = C3f[s0 + lane];
    }
    if (kC3) sC[lane] = 0;
    sD[lane] = 0;
    rows[lane] = 0;
    __syncwarp();
    const int smax = sS[s - 1];
    const bool narrow = (u64)s * (u64)(rp[u + 1] - rp[u]) < (1ull << 32);
    u64 tu = 0;
    // Flatten the probe lists N+(S[a]) (cut at max S) of all members: lane a
    // sets up its segment, then every lane streams one element per step.
    int st = 0, len = 0, x = 0;
    bool pairs = false;
    if (lane + 1 < s) {
      x = sS[lane];
      st = split[x];
      const int full = rp[x + 1];  // short lists: probe whole, skip the dependent search
      len = (full - st <= FGLT_PROBE_NOCUT_WARP ? full : lower_bound_i32(ci, st, full, smax + 1)) - st;
      pairs = hub != nullptr && x >= hb &&
              (hub_force || (s - 1 - lane) * FGLT_PAIR_W < len * FGLT_PROBE_W);
      if (pairs) len = 0;
    }
    int T;
    const int off = flat_prefix(len, &T);
    fbase[lane] = st - off;
    foff[lane] = off;
    if (lane == 0) foff[32] = T;
    __syncwarp();
    int r = 0, cr = 0;
    u64 da = 0;
    u32 na = 0;
    for (int kk = lane; kk < T; kk += 32) {
      while (foff[r + 1] <= kk) ++r;
      if (r != cr) {  // flush the per-member partials of row cr
        if (kC3 && na) atomicAdd(sC + cr, na);
        if (kD13 && da) smem_add_u64(sD + cr, da);
        na = 0;
        da = 0;
        cr = r;
      }
      const int p = fbase[r] + kk;
      const int y = __ldg(ci + p);
      const int bi = lower_bound_smem(sS, r + 1, s, y);
      if (bi < s && sS[bi] == y) {
        if (kD15) {
          atomicOr(rows + r, 1u << bi);
          atomicOr(rows + bi, 1u << r);
        }
        if (kC3) {
          atomicAdd(C3f + p, 1u);
          atomicAdd(sC + bi, 1u);
          ++na;
          if (listing) {
            const unsigned m = __activemask();
            const int leader = __ffs(m) - 1;
            unsigned base = 0;
            if (lane == leader) base = atomicAdd(wcnt, (unsigned)__popc(m));
            base = __shfl_sync(m, base, leader);
            tl.rec[wt + 1 + base + __popc(m & ((1u << lane) - 1u))] =
                make_uint2((u32)r | ((u32)bi << 16), (u32)p);
          }
        }
        if (kD13) {
          tu += (u64)__ldg(C3f + p) - 1;
          da += (u64)sC[bi] - 1;
          if (narrow) atomicAdd(reinterpret_cast<u32*>(sD + bi), sC[r] - 1);
          else smem_add_u64(sD + bi, (u64)sC[r] - 1);
        }
      }
    }
    if (kC3 && na) atomicAdd(sC + cr, na);
    if (kD13 && da) smem_add_u64(sD + cr, da);
    __syncwarp();
    if (hub != nullptr && __any_sync(0xffffffffu, pairs)) {
      // pair rows: member a tests S[a+1..s) against its hub row
      int T2;
      const int off2 = flat_prefix(pairs ? s - 1 - lane : 0, &T2);
      fbase[lane] = pairs ? hub_base[x - hb] : 0;
      foff[lane] = off2;
      fsplit[lane] = st;
      if (lane == 0) foff[32] = T2;
      __syncwarp();
      r = 0;
      cr = 0;
      na = 0;
      da = 0;
      for (int kk = lane; kk < T2; kk += 32) {
        while (foff[r + 1] <= kk) ++r;
        if (r != cr) {
          if (kC3 && na) atomicAdd(sC + cr, na);
          if (kD13 && da) smem_add_u64(sD + cr, da);
          na = 0;
          da = 0;
          cr = r;
        }
        const int bi = r + 1 + (kk - foff[r]);
        const int o = sS[bi] - sS[r] - 1;
        const unsigned long long wv = __ldg(hub + fbase[r] + (o >> 5));
        const u32 bits = (u32)wv;
        if ((bits >> (o & 31)) & 1u) {
          const int p = fsplit[r] + (int)(wv >> 32) + __popc(bits & ((1u << (o & 31)) - 1u));
          if (kD15) {
            atomicOr(rows + r, 1u << bi);
            atomicOr(rows + bi, 1u << r);
          }
          if (kC3) {
            atomicAdd(C3f + p, 1u);
            atomicAdd(sC + bi, 1u);
            ++na;
            if (listing) {
              const unsigned m = __activemask();
              const int leader = __ffs(m) - 1;
              unsigned base = 0;
              if (lane == leader) base = atomicAdd(wcnt, (unsigned)__popc(m));
              base = __shfl_sync(m, base, leader);
              tl.rec[wt + 1 + base + __popc(m & ((1u << lane) - 1u))] =
                  make_uint2((u32)r | ((u32)bi << 16), (u32)p);
            }
          }
          if (kD13) {
            tu += (u64)__ldg(C3f + p) - 1;
            da += (u64)sC[bi] - 1;
            if (narrow) atomicAdd(reinterpret_cast<u32*>(sD + bi), sC[r] - 1);
            else smem_add_u64(sD + bi, (u64)sC[r] - 1);
          }
        }
      }
      if (kC3 && na) atomicAdd(sC + cr, na);
      if (kD13 && da) smem_add_u64(sD + cr, da);
      __syncwarp();
    }
    if (kC3 && listing) {  // close the root's records with their header
      __syncwarp();
      const unsigned cnt = *wcnt;
      if (cnt) {
        FGLT_BOUNDS(wt + cnt < ce && ce <= tl.cap, "trilist warp chunk", wt + cnt, ce);
        if (lane == 0) tl.rec[wt] = make_uint2(0x80000000u | cnt, (u32)u);
        wt += 1 + cnt;
      }
    }
    if (kC3 && lane < s && sC[lane]) atomicAdd(C3f + s0 + lane, sC[lane]);
    if (kD13) {
      if (lane < s && sD[lane]) atomicAdd(d13 + sS[lane], sD[lane]);
      tu = warp_sum_u64(tu);
      if (lane == 0 && tu) atomicAdd(d13 + u, tu);
    }
    if (kD15) {
      u64 ta = 0;
      if (lane < s) {
        const u32 row = rows[lane];
        u32 bits = row;
        u32 t = 0;
        while (bits) {
          const int bb = __ffs(bits) - 1;
          bits &= bits - 1;
          t += __popc(row & rows[bb]);
        }
        ta = t / 2;
        if (ta) atomicAdd(d15 + sS[lane], ta);
      }
      ta = warp_sum_u64(ta);
      if (lane == 0 && ta) atomicAdd(d15 + u, ta / 3);
    }
    __syncwarp();
  }
  if (kC3 && tl.rec) retire();
}

// Block per root, |S| > 32. Shared-memory layout (host computes the same
// sizes, roots_smem_bytes): sD u64[s_cap] | sS int[s_cap] | sC u32[s_cap] |
// hash keys int[hcap] | hash idx u16[hcap] | per-warp pair lists u16[nw x s_cap]
// | bitmap u32[s_cap x stride_cap]. With kGlobal the bitmap, hash and lists
// live in the block's slice of a global slab instead (rare, very large S).
// Bitmap rows use the bitmap_stride() stride so lanes reading different rows at the
// same word index spread over banks.
// G[S] bitmap row stride in 32-bit words: rows hold whole 64-bit words (for
// 64-bit popcounts) and an odd number of them, so lanes reading different
// rows at the same index spread over the banks.
__host__ __device__ inline int bitmap_stride(int nw) { return 2 * (((nw + 1) >> 1) | 1); }

struct RootsLayout {
  int s_cap, hcap, hlog, nwarps, stride_cap;
  __host__ __device__ size_t bytes_core() const {  // always in smem
    return (size_t)s_cap * (8 + 4 + 4);
  }
  __host__ __device__ size_t bytes_aux() const {  // smem or slab
    size_t h = (size_t)hcap * 4 + (((size_t)hcap * 2 + 15) & ~(size_t)15);
    size_t l = (((size_t)nwarps * s_cap * 2) + 15) & ~(size_t)15;
    return h + l + (size_t)s_cap * stride_cap * 4;
  }
};

__device__ __forceinline__ int s_hash_find(const int* keys, const unsigned short* idx, int hlog,
                                           int y) {
  const u32 mask = (1u << hlog) - 1;
  u32 h = ((u32)y * 0x9E3779B1u) >> (32 - hlog);
  while (true) {
    const int k = keys[h];
    if (k == y) return idx[h];
    if (k < 0) return -1;
    h = (h + 1) & mask;
  }
}

// ---- hub rows. The R highest-ranked active vertices [hb, n_active) (the
// highest-degree ones, after the relabel) get a packed adjacency row over the
// ids above them: for x = hb + i, word k of row i covers ids x+1+32k ..
// x+32+32k; low 32 bits = adjacency, high 32 bits = number of N+(x) entries
// before the word (so the CSR position of (x, y) is split[x] + high +
// popc(low below y)). Rows are ceil((R-1-i)/32) words, packed back to back.
#ifndef FGLT_HUB_MAX
#define FGLT_HUB_MAX 49152
#define FGLT_HUB_MIN_DEG 128
#endif
#ifndef FGLT_ROOT_HASH_FACTOR
#define FGLT_ROOT_HASH_FACTOR 4  // root hash slots >= this x |S|
#endif
constexpr int kHubMax = FGLT_HUB_MAX;  // R cap: R^2/8 bytes of rows (288 MB at 48K)
constexpr int kHubMinDegree = FGLT_HUB_MIN_DEG;  // hub rows only when the R-th largest degree reaches this

__global__ void k_hub_words(int R, int* __restrict__ w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= R; i += gridDim.x * blockDim.x)
    w[i] = i < R ? (R - 1 - i + 31) >> 5 : 0;
}

// Warp per hub row (hub_base = exclusive scan of k_hub_words).
__global__ void k_hub_rows(const int* __restrict__ ci, const int* __restrict__ split,
                           const int* __restrict__ send, int hb, int R,
                           const int* __restrict__ hub_base, unsigned long long* __restrict__ hub) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < R; i += warps) {
    const int x = hb + i;
    const int base = hub_base[i], nw = hub_base[i + 1] - base;
    const int st = split[x], en = send[x];  // N+(x): ids in (x, n_active)
    for (int k = lane; k < nw; k += 32) {
      const int before = lower_bound_i32(ci, st, en, x + 1 + 32 * k) - st;
      hub[base + k] = (unsigned long long)before << 32;
    }
    __syncwarp();
    for (int j = st + lane; j < en; j += 32) {
      const int o = ci[j] - x - 1;
      atomicOr(reinterpret_cast<unsigned*>(hub + base + (o >> 5)), 1u << (o & 31));
    }
  }
}

#ifndef FGLT_K4_THREAD_NW
#define FGLT_K4_THREAD_NW 16  // G[S] rows of at most this many words: thread-per-member 4-cliques
#endif
#ifndef FGLT_ROOTS_THREADS
#define FGLT_ROOTS_THREADS 256
#endif
constexpr int kRootsThreads = FGLT_ROOTS_THREADS;  // block threads for |S| > 256 (smaller bins: 64, 128)
#ifndef FGLT_PAIRS_IN_FLIGHT
#define FGLT_PAIRS_IN_FLIGHT 4
#endif
constexpr int kPairsInFlight = FGLT_PAIRS_IN_FLIGHT;  // hub-row words in flight per lane

// (Measured and dropped: a minimum-blocks launch bound capping the 64/128-
// thread bins at 48/40/32 registers spills, R-MAT 20 triangles 11.7 -> 14.3/
// 15.2/16.0 ms; even a bound of (NT, 1) changes the allocation to 86
// registers and loses the 64-register occupancy: keep plain (NT).)
template <bool kC3, bool kD13, bool kD15, bool kGlobal, int NT>
__global__ void __launch_bounds__(NT)
k_roots_block(const int* __restrict__ rp, const int* __restrict__ ci,
              const int* __restrict__ split, const int* __restrict__ send,
              u32* __restrict__ C3f,
              const int* __restrict__ roots, int nroots, RootsLayout L,
              unsigned char* __restrict__ slab, long long slab_stride,
              int* __restrict__ next_root, u64* __restrict__ d13, u64* __restrict__ d15,
              const unsigned long long* __restrict__ hub, const int* __restrict__ hub_base,
              int hb, int hub_force, TriList tl) {
  // roots sorted by |S| (largest first), handed out dynamically
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ u64 red[32];
  __shared__ int next_item[2];
  constexpr int NWB = NT / 32;
  __shared__ int f_off[NT + 1], f_st[NT];  // probe / pair flattening
  __shared__ int f_sa[NT], f_sb[NT], f_hb[NT];
  __shared__ int f_wtot[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64* sD = reinterpret_cast<u64*>(smem_raw);
  int* sS = reinterpret_cast<int*>(sD + L.s_cap);
  u32* sC = reinterpret_cast<u32*>(sS + L.s_cap);
  unsigned char* aux = kGlobal ? slab + (long long)blockIdx.x * slab_stride
                               : reinterpret_cast<unsigned char*>(sC + L.s_cap);
  int* hkeys = reinterpret_cast<int*>(aux);
  unsigned short* hidx = reinterpret_cast<unsigned short*>(hkeys + L.hcap);
  unsigned short* lists = reinterpret_cast<unsigned short*>(
      aux + (size_t)L.hcap * 4 + ((((size_t)L.hcap * 2) + 15) & ~(size_t)15));
  u32* bm = reinterpret_cast<u32*>(
      reinterpret_cast<unsigned char*>(lists) +
      ((((size_t)L.nwarps * L.s_cap * 2) + 15) & ~(size_t)15));
  unsigned short* mylist = lists + (size_t)wid * L.s_cap;

  __shared__ int s_root;
  // triangle list state (kC3 with tl.rec): this block's pool reservation
  // [s_tb, s_te), records of the current phase, and the root's failure flag
  __shared__ unsigned long long s_tb, s_te;
  __shared__ unsigned s_tc;
  __shared__ int s_tfail;
  if (threadIdx.x == 0) {
    s_tb = s_te = 0;
    s_tc = 0;
  }
  while (true) {
    if (threadIdx.x == 0) s_root = atomicAdd(next_root, 1);
    __syncthreads();
    const int k = s_root;
    if (k >= nroots) break;
    const int u = roots[k];
    if (kD13 && tl.rec && !tl.fail[u]) {  // listed: k_diamond_list handles it
      __syncthreads();
      continue;
    }
    const int s0 = split[u];
    const int s = send[u] - s0;
    if (kC3 && tl.rec && threadIdx.x == 0) s_tfail = s > kTriListMaxS;
    const int nw = (s + 31) >> 5;
    const int stride = bitmap_stride(nw);
    const int nw64 = (nw + 1) >> 1;
    int hlog = 6;
    while ((1 << hlog) < FGLT_ROOT_HASH_FACTOR * s) ++hlog;
    const int hcap = 1 << hlog;
    FGLT_BOUNDS(s <= L.s_cap, "s", s, L.s_cap);
    FGLT_BOUNDS(hlog <= L.hlog, "hlog", hlog, L.hlog);
    FGLT_BOUNDS(stride <= L.stride_cap, "stride", stride, L.stride_cap);
    for (int a = threadIdx.x; a < s; a += blockDim.x) {
      sS[a] = ci[s0 + a];
      if (kD13) { sC[a] = C3f[s0 + a]; sD[a] = 0; }
      if (kD15) sD[a] = 0;  // sK (u32 view), see below
      if (kC3) sC[a] = 0;  // per-(u, S[a]) triangle counts
    }
    for (int i = threadIdx.x; i < hcap; i += blockDim.x) hkeys[i] = -1;
    if (kD15)
      for (long long i = threadIdx.x; i < (long long)s * stride; i += blockDim.x) bm[i] = 0;
    if (threadIdx.x == 0) { next_item[0] = 0; next_item[1] = 0; }
    __syncthreads();
    for (int a = threadIdx.x; a < s; a += blockDim.x) {
      const int y = sS[a];
      u32 h = ((u32)y * 0x9E3779B1u) >> (32 - hlog);
      while (atomicCAS(hkeys + h, -1, y) != -1) h = (h + 1) & (hcap - 1);
      hidx[h] = (unsigned short)a;
    }
    __syncthreads();
    const int smax = sS[s - 1];
    // sD[b] sums C3(u, .) - 1 < deg(u) over < s triangles: 32 bits suffice
    // (no carry) when s * deg(u) < 2^32
    const bool narrow = (u64)s * (u64)(rp[u + 1] - rp[u]) < (1ull << 32);
    u64 tu = 0;
    // ---- every triangle {u, S[a], S[b]} with a < b, once, found from
    // member a by one of two means, chosen per member:
    //   probe: N+(S[a]) cut at max S, flattened block-wide over 16-byte quads
    //          of ci and looked up in the hash of S;
    //   pairs: S[a] is a hub (id >= hb): test S[b], b > a, against the
    //          packed adjacency row of S[a] (k_hub_rows), which also gives the
    //          CSR position of (S[a], S[b]) by a popcount rank.
    // Per-row partials (na, da) are flushed when a lane's row changes.
    int cr = -1;
    u32 ca = 0, na = 0;
    u64 da = 0;
    auto flush = [&](int c0) {
      if (cr < 0) return;
      if (kC3 && na) atomicAdd(sC + c0 + cr, na);
      if (kD13 && da) smem_add_u64(sD + c0 + cr, da);
      cr = -1;
    };
    auto to_row = [&](int c0, int r) {
      if (r != cr) {
        flush(c0);
        cr = r;
        na = 0;
        da = 0;
        if (kD13) ca = sC[c0 + r];
      }
    };
    auto hit = [&](int a, int bi, int p) {
      if (kD15) {
        atomicOr(bm + (long long)a * stride + (bi >> 5), 1u << (bi & 31));
        atomicOr(bm + (long long)bi * stride + (a >> 5), 1u << (a & 31));
      }
      if (kC3) {
        atomicAdd(C3f + p, 1u);
        atomicAdd(sC + bi, 1u);
        ++na;
        if (tl.rec && !s_tfail) {  // warp-aggregated append to the phase's reservation
          const unsigned m = __activemask();
          const int leader = __ffs(m) - 1;
          unsigned base = 0;
          if (lane == leader) base = atomicAdd(&s_tc, (unsigned)__popc(m));
          base = __shfl_sync(m, base, leader);
          const unsigned idx = base + __popc(m & ((1u << lane) - 1u));
          FGLT_BOUNDS(s_tb + idx < s_te && s_te <= tl.cap, "trilist block rec", s_tb + idx, s_te);
          tl.rec[s_tb + idx] = make_uint2((u32)a | ((u32)bi << 16), (u32)p);
        }
      }
      if (kD13) {
        tu += (u64)__ldg(C3f + p) - 1;
        da += (u64)sC[bi] - 1;
        if (narrow) atomicAdd(reinterpret_cast<u32*>(sD + bi), ca - 1);
        else smem_add_u64(sD + bi, (u64)ca - 1);
      }
    };
    // reserve room for at most `bound` records of the next phase (one thread,
    // inside block_flatten) / publish the phase's records as a piece (after
    // the phase's trailing barrier)
    auto tl_reserve = [&](unsigned long long bound) {
      if (!(kC3 && tl.rec)) return;
      s_tc = 0;
      if (!s_tfail && bound > 0 && s_te - s_tb < bound) {
        const unsigned long long grab = bound > kTriListChunk ? bound : kTriListChunk;
        const unsigned long long st = atomicAdd(tl.top, grab);
        if (st + grab > tl.cap) {
          s_tfail = 1;
        } else {
          s_tb = st;
          s_te = st + grab;
        }
      }
    };
    auto tl_publish = [&]() {
      if (!(kC3 && tl.rec) || threadIdx.x != 0 || s_tfail || s_tc == 0) return;
      const unsigned pi = atomicAdd(tl.npieces, 1u);
      if (pi < tl.pieces_cap) {
        tl.pieces[pi] = TriPiece{s_tb, u, s_tc};
        s_tb += s_tc;
      } else {
        s_tfail = 1;
      }
    };
    for (int c0 = 0; c0 + 1 < s; c0 += NT) {
      const int a_me = c0 + threadIdx.x;
      int x = 0, st = 0, se = 0;
      bool pairs = false;
      if (a_me + 1 < s) {
        x = sS[a_me];
        st = split[x];
        const int full = rp[x + 1];  // short lists: probe whole, skip the dependent search
        se = full - st <= FGLT_PROBE_NOCUT ? full : lower_bound_i32(ci, st, full, smax + 1);
        pairs = hub != nullptr && x >= hb &&
                (hub_force || (s - 1 - a_me) * FGLT_PAIR_W < (se - st) * FGLT_PROBE_W);
      }
      // probe rows
      {
        const int qa = st >> 2;
        const int nqd = (!pairs && se > st) ? ((se + 3) >> 2) - qa : 0;
        f_sa[threadIdx.x] = st;
        f_sb[threadIdx.x] = se;
        block_flatten(nqd, qa, f_off, f_st, f_wtot,
                      [&](int T) { tl_reserve(4ull * (unsigned long long)T); });
      }
#if FGLT_ROOTS_LANE_MEMBER
      if (!pairs && se > st) {  // thread per member: stream its own probe list
        to_row(c0, threadIdx.x);
        auto one = [&](int pp, int y) {
          const int bi = s_hash_find(hkeys, hidx, hlog, y);
          if (bi >= 0) hit(a_me, bi, pp);
        };
        int p = st;
        for (; p < se && (p & 3); ++p) one(p, __ldg(ci + p));
        for (; p + 4 <= se; p += 4) {
          const int4 x = __ldg(reinterpret_cast<const int4*>(ci + p));
          one(p, x.x); one(p + 1, x.y); one(p + 2, x.z); one(p + 3, x.w);
        }
        for (; p < se; ++p) one(p, __ldg(ci + p));
        flush(c0);
      }
      if (false)
#endif
      {
        const int T = f_off[NT];
        const int per = (T + NWB - 1) / NWB;
        const int k0 = wid * per, k1 = min(T, k0 + per);
        if (k0 + lane < k1) {
          int r = upper_row(f_off, k0 + lane, NT);
          for (int kk = k0 + lane; kk < k1; kk += 32 * kRootsQuads) {
            int4 v[kRootsQuads];
            int lt[kRootsQuads], ht[kRootsQuads], rr[kRootsQuads], e0[kRootsQuads];
#pragma unroll
            for (int j = 0; j < kRootsQuads; ++j) {
              const int kj = kk + 32 * j;
              lt[j] = 4;
              ht[j] = 0;
              rr[j] = r;
              e0[j] = 0;
              if (kj < k1) {
                while (f_off[r + 1] <= kj) ++r;
                rr[j] = r;
                e0[j] = (f_st[r] + kj) << 2;
                v[j] = __ldg(reinterpret_cast<const int4*>(ci + e0[j]));
                lt[j] = f_sa[r] - e0[j];
                ht[j] = f_sb[r] - e0[j];
              }
            }
#pragma unroll
            for (int j = 0; j < kRootsQuads; ++j) {
              if (ht[j] <= 0) break;
              to_row(c0, rr[j]);
              const int a = c0 + rr[j];
              const int ys[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                if (t < lt[j] || t >= ht[j]) continue;
                const int bi = s_hash_find(hkeys, hidx, hlog, ys[t]);
                FGLT_BOUNDS(bi < s && (bi < 0 || bi > a), "bi", bi, a);
                if (bi >= 0) hit(a, bi, e0[j] + t);
              }
            }
          }
          flush(c0);
        }
      }
      // barrier (f_* are rewritten below) that also tells whether any member
      // of this chunk takes the hub-row pair path
      const int any_pairs = __syncthreads_or(pairs ? 1 : 0);
      tl_publish();
      if (hub == nullptr || !any_pairs) continue;
      // pair rows
      {
        f_sa[threadIdx.x] = x;
        f_sb[threadIdx.x] = st;
        f_hb[threadIdx.x] = pairs ? hub_base[x - hb] : 0;
        block_flatten(pairs ? s - 1 - a_me : 0, 0, f_off, f_st, f_wtot,
                      [&](int T) { tl_reserve((unsigned long long)T); });
      }
      {
        const int T = f_off[NT];
        const int per = (T + NWB - 1) / NWB;
        const int k0 = wid * per, k1 = min(T, k0 + per);
        if (k0 + lane < k1) {
          int r = upper_row(f_off, k0 + lane, NT);
          for (int kk = k0 + lane; kk < k1; kk += 32 * kPairsInFlight) {
            unsigned long long wv[kPairsInFlight];
            int rr[kPairsInFlight], bb[kPairsInFlight], ob[kPairsInFlight];
#pragma unroll
            for (int j = 0; j < kPairsInFlight; ++j) {
              const int kj = kk + 32 * j;
              rr[j] = -1;
              if (kj < k1) {
                while (f_off[r + 1] <= kj) ++r;
                rr[j] = r;
                bb[j] = c0 + r + 1 + (kj - f_off[r]);
                const int o = sS[bb[j]] - f_sa[r] - 1;
                ob[j] = o & 31;
                wv[j] = __ldg(hub + f_hb[r] + (o >> 5));
              }
            }
#pragma unroll
            for (int j = 0; j < kPairsInFlight; ++j) {
              if (rr[j] < 0) break;
              const u32 bits = (u32)wv[j];
              if (!((bits >> ob[j]) & 1u)) continue;
              to_row(c0, rr[j]);
              const int pos = f_sb[rr[j]] + (int)(wv[j] >> 32) + __popc(bits & ((1u << ob[j]) - 1u));
              hit(c0 + rr[j], bb[j], pos);
            }
          }
          flush(c0);
        }
      }
      __syncthreads();
      tl_publish();
    }
    __syncthreads();
    if (kC3 && tl.rec && threadIdx.x == 0 && s_tfail) tl.fail[u] = 1;
    if (kC3)
      for (int a = threadIdx.x; a < s; a += blockDim.x)
        if (sC[a]) atomicAdd(C3f + s0 + a, sC[a]);
    if (kD13) {
      for (int a = threadIdx.x; a < s; a += blockDim.x)
        if (sD[a]) atomicAdd(d13 + sS[a], sD[a]);
      tu = block_sum_u64(tu, red);
      if (threadIdx.x == 0 && tu) atomicAdd(d13 + u, tu);
    }
    if (kD15) {
      // Each G[S] edge (a, b), a < b, once: c_ab = popc(row_a & row_b) is the
      // number of G[S]-triangles on it and is credited to both ends, so
      // sK[a] = sum_{b in row a} c_ab = 2 t_a (t_a = G[S]-triangles through a).
      u32* sK = reinterpret_cast<u32*>(sD);
      if (nw <= FGLT_K4_THREAD_NW) {
        // small S: thread per member, its row in registers; each G[S] edge
        // (a, b > a) popcounted once and credited to both ends
        for (int a = threadIdx.x; a + 1 < s; a += NT) {
          const u32* ra = bm + (long long)a * stride;
          const u64* ra64 = reinterpret_cast<const u64*>(ra);
          u64 r[FGLT_K4_THREAD_NW / 2];
#pragma unroll
          for (int t = 0; t < FGLT_K4_THREAD_NW / 2; ++t) r[t] = t < nw64 ? ra64[t] : 0ull;
          const int j0 = (a + 1) >> 5;
          u32 acc = 0;
          for (int j = j0; j < nw; ++j) {
            u32 w = ra[j] & (j == j0 ? ~0u << ((a + 1) & 31) : ~0u);
            while (w) {
              const int bb = (j << 5) + __ffs(w) - 1;
              w &= w - 1;
              const u64* rb = reinterpret_cast<const u64*>(bm + (long long)bb * stride);
              u32 c = 0;
#pragma unroll
              for (int t = 0; t < FGLT_K4_THREAD_NW / 2; ++t)
                if (t < nw64) c += __popcll(r[t] & rb[t]);
              if (c) {
                acc += c;
                atomicAdd(sK + bb, c);
              }
            }
          }
          if (acc) atomicAdd(sK + a, acc);
        }
      } else
      while (true) {
        int a = 0;
        if (lane == 0) a = atomicAdd(next_item + 1, 1);
        a = __shfl_sync(0xffffffffu, a, 0);
        if (a + 1 >= s) break;
        const u32* ra = bm + (long long)a * stride;
        const int j0 = (a + 1) >> 5;
        const u32 m0 = ~0u << ((a + 1) & 31);  // bits > a in word j0
        u32 acc = 0;
        if (nw <= 8) {
          // lane l takes bit l of each nonzero word
          for (int j = j0; j < nw; ++j) {
            const u32 w = ra[j] & (j == j0 ? m0 : ~0u);
            if (w == 0) continue;
            if ((w >> lane) & 1u) {
              const int bb = (j << 5) + lane;
              const u64* rb = reinterpret_cast<const u64*>(bm + (long long)bb * stride);
              const u64* ra64 = reinterpret_cast<const u64*>(ra);
              u32 c = 0;
              for (int t = 0; t < nw64; ++t) c += __popcll(ra64[t] & rb[t]);
              if (c) {
                acc += c;
                atomicAdd(sK + bb, c);
              }
            }
          }
        } else {
          // extract the neighbours b > a of a, then lanes over them
          int written = 0;
          for (int jb = j0; jb < nw; jb += 32) {
            const int j = jb + lane;
            u32 w = j < nw ? ra[j] & (j == j0 ? m0 : ~0u) : 0u;
            const int c = __popc(w);
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += t;
            }
            int off = written + incl - c;
            while (w) {
              mylist[off++] = (unsigned short)((j << 5) + __ffs(w) - 1);
              w &= w - 1;
            }
            written += __shfl_sync(0xffffffffu, incl, 31);
          }
          __syncwarp();
          FGLT_BOUNDS(written <= s, "written", written, s);
          for (int i = lane; i < written; i += 32) {
            const int bb = mylist[i];
            FGLT_BOUNDS(bb > a && bb < s, "list", bb, s);
            const u64* rb = reinterpret_cast<const u64*>(bm + (long long)bb * stride);
            const u64* ra64 = reinterpret_cast<const u64*>(ra);
            u32 c = 0;
            for (int t = 0; t < nw64; ++t) c += __popcll(ra64[t] & rb[t]);
            if (c) {
              acc += c;
              atomicAdd(sK + bb, c);
            }
          }
          __syncwarp();
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0 && acc) atomicAdd(sK + a, acc);
      }
      __syncthreads();
      u64 tot = 0;
      for (int a = threadIdx.x; a < s; a += blockDim.x) {
        const u32 ta = sK[a] >> 1;
        if (ta) {
          atomicAdd(d15 + sS[a], (u64)ta);
          tot += ta;
        }
      }
      tot = block_sum_u64(tot, red);
      if (threadIdx.x == 0 && tot) atomicAdd(d15 + u, tot / 3);
    }
    __syncthreads();
  }
}

// Diamonds from the triangle list (the kD13 terms of k_roots_block, see
// above): block per piece, per-member partial sums in shared memory.
#ifndef FGLT_DLIST_UNROLL
#define FGLT_DLIST_UNROLL 1  // measured at R-MAT 20 (diamond rows, ms): 1: 2.5, 2: 2.5, 4: 2.9, 8: 3.4 (L2 gather rate, not latency)
#endif
constexpr int kDlistUnroll = FGLT_DLIST_UNROLL;
template <int NT>
__global__ void __launch_bounds__(NT)
k_diamond_list(const TriPiece* __restrict__ pieces, const unsigned* __restrict__ npieces,
               unsigned pieces_cap, const uint2* __restrict__ rec, const int* __restrict__ rp,
               const int* __restrict__ ci, const int* __restrict__ split,
               const int* __restrict__ send, const u32* __restrict__ C3f,
               const unsigned char* __restrict__ fail, int* __restrict__ next,
               u64* __restrict__ d13) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* sD = reinterpret_cast<u64*>(smem_raw);
  __shared__ u64 red[32];
  __shared__ int s_item;
  const unsigned np = min(*npieces, pieces_cap);
  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(next, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= (int)np) break;
    const TriPiece pc = pieces[it];
    const int u = pc.u;
    if (fail[u]) {
      __syncthreads();
      continue;
    }
    const int s0 = split[u];
    const int s = send[u] - s0;
    for (int a = threadIdx.x; a < s; a += NT) sD[a] = 0;
    __syncthreads();
    const bool narrow = (u64)s * (u64)(rp[u + 1] - rp[u]) < (1ull << 32);
    u64 tu = 0;
    const uint2* r = rec + pc.start;
    // kDlistUnroll records per thread and round: the records, then their three
    // count gathers, are all issued before the first shared add
    for (unsigned i0 = threadIdx.x; i0 < pc.count; i0 += kDlistUnroll * NT) {
      uint2 x[kDlistUnroll];
      u32 ca[kDlistUnroll], cb[kDlistUnroll], cp[kDlistUnroll];
#pragma unroll
      for (int j = 0; j < kDlistUnroll; ++j) {
        const unsigned i = i0 + j * NT;
        x[j] = i < pc.count ? r[i] : make_uint2(0xffffffffu, 0u);
      }
#pragma unroll
      for (int j = 0; j < kDlistUnroll; ++j) {
        if (x[j].x == 0xffffffffu) continue;  // a == b == 0xffff never occurs (a < b)
        ca[j] = __ldg(C3f + s0 + (int)(x[j].x & 0xffffu));
        cb[j] = __ldg(C3f + s0 + (int)(x[j].x >> 16));
        cp[j] = __ldg(C3f + x[j].y);
      }
#pragma unroll
      for (int j = 0; j < kDlistUnroll; ++j) {
        if (x[j].x == 0xffffffffu) continue;
        const int a = (int)(x[j].x & 0xffffu), b = (int)(x[j].x >> 16);
        tu += (u64)cp[j] - 1;
        if (narrow) {
          atomicAdd(reinterpret_cast<u32*>(sD + a), cb[j] - 1);
          atomicAdd(reinterpret_cast<u32*>(sD + b), ca[j] - 1);
        } else {
          smem_add_u64(sD + a, (u64)cb[j] - 1);
          smem_add_u64(sD + b, (u64)ca[j] - 1);
        }
      }
    }
    __syncthreads();
    for (int a = threadIdx.x; a < s; a += NT)
      if (sD[a]) atomicAdd(d13 + ci[s0 + a], sD[a]);
    tu = block_sum_u64(tu, red);
    if (threadIdx.x == 0 && tu) atomicAdd(d13 + u, tu);
    __syncthreads();
  }
}

// Diamonds of the listed warp roots: warp per chunk, root by root (header,
// then its records, one per lane), per-member sums in shared memory.
__global__ void __launch_bounds__(256)
k_diamond_wlist(const TriChunk* __restrict__ chunks, const unsigned* __restrict__ nchunks,
                unsigned chunks_cap, const uint2* __restrict__ rec, const int* __restrict__ rp,
                const int* __restrict__ ci, const int* __restrict__ split,
                const int* __restrict__ send, const u32* __restrict__ C3f,
                u64* __restrict__ d13) {
  __shared__ u64 sDall[8][32];
  __shared__ u32 sCall[8][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  u64* sD = sDall[wib];
  u32* sC = sCall[wib];
  const unsigned nc = min(*nchunks, chunks_cap);
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (unsigned k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nc; k += warps) {
    const TriChunk ch = chunks[k];
    unsigned long long pos = ch.start;
    const unsigned long long end = ch.start + ch.used;
    while (pos < end) {
      const uint2 h = rec[pos];
      const unsigned cnt = h.x & 0x7fffffffu;
      const int u = (int)h.y;
      const int s0 = split[u];
      const int s = send[u] - s0;
      sD[lane] = 0;
      sC[lane] = lane < s ? C3f[s0 + lane] : 0u;
      __syncwarp();
      const bool narrow = (u64)s * (u64)(rp[u + 1] - rp[u]) < (1ull << 32);
      u64 tu = 0;
      for (unsigned i = lane; i < cnt; i += 32) {
        const uint2 x = rec[pos + 1 + i];
        const int a = (int)(x.x & 0xffffu), b = (int)(x.x >> 16);
        tu += (u64)__ldg(C3f + x.y) - 1;
        if (narrow) {
          atomicAdd(reinterpret_cast<u32*>(sD + a), sC[b] - 1);
          atomicAdd(reinterpret_cast<u32*>(sD + b), sC[a] - 1);
        } else {
          smem_add_u64(sD + a, (u64)sC[b] - 1);
          smem_add_u64(sD + b, (u64)sC[a] - 1);
        }
      }
      __syncwarp();
      if (lane < s && sD[lane]) atomicAdd(d13 + ci[s0 + lane], sD[lane]);
      tu = warp_sum_u64(tu);
      if (lane == 0 && tu) atomicAdd(d13 + u, tu);
      __syncwarp();
      pos += 1 + cnt;
    }
  }
}

// Sum over roots u in [u0, u1) with 2 <= |N+(u)| <= kTriListMaxS of
// C(|N+(u)|, 2) (+1 header for warp roots): an upper bound of the records.
#ifndef FGLT_TL_TIGHT
#define FGLT_TL_TIGHT 1
#endif
__global__ void k_trilist_bound(const int* __restrict__ split, const int* __restrict__ send,
                                const int* __restrict__ ci, int u0, int u1,
                                unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int u = u0 + blockIdx.x * blockDim.x + threadIdx.x; u < u1; u += gridDim.x * blockDim.x) {
    const unsigned long long s = (unsigned long long)(send[u] - split[u]);
    if (s >= 2 && s <= (unsigned long long)kTriListMaxS) {
      unsigned long long b = s * (s - 1) / 2;
#if FGLT_TL_TIGHT
      // a triangle {u, S[a], y} (y > S[a]) is found from member a as y in
      // N+(S[a]) ∩ S[a+1..]: at most min(|N+(S[a])|, s - 1 - a) of them
      unsigned long long o = 0;
      const int s0 = split[u];
      for (int a = 0; a < (int)s && o < b; ++a) {
        const int x = ci[s0 + a];
        const unsigned long long out = (unsigned long long)(send[x] - split[x]);
        const unsigned long long rest = s - 1 - (unsigned long long)a;
        o += out < rest ? out : rest;
      }
      b = o < b ? o : b;
#endif
      acc += b + (s <= 32);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// =============================================================== epilogue
// Column fill (kernels.cpp:384-412) + exact raw->net back-substitution with
// U(s,s) (conversion.cpp:80-116), one thread per ORIGINAL vertex, rows written
// in original order. Checked sites follow the reference; the first failure in
// (fill stage, vertex) order is reported through an atomicMin on
//   key = stage << 40 | vertex << 8 | code << 4 | graphlet.
struct DictInfo {
  int k;
  int ids[16];
  unsigned mask;
  int ntail[16];          // per dictionary position r, number of tail entries
  int tail_col[16][16];   // positions c > r with U[ids[r]][ids[c]] != 0
  unsigned long long tail_coef[16][16];  // U(s,s) or a caller's ConversionMatrix
};

__device__ __forceinline__ bool mul_ov(u64 a, u64 b, u64* r) {
  *r = a * b;
  return __umul64hi(a, b) != 0ull;
}
__device__ __forceinline__ bool add_ov(u64 a, u64 b, u64* r) {
  *r = a + b;
  return *r < a;
}

// U16 coefficients: fglt_tables.h (one definition for host and device).
using fglt_tables::u16_coef;

struct EpilogueIn {
  const int* rp;   // graph the vectors are indexed by (relabelled or original)
  const int* inv;  // original id -> row of that graph; null = identity
  const u64 *p2, *p3, *c3, *d7, *d9, *d10, *d14, *c4, *d13, *d15;
};

__device__ __forceinline__ void offer_err(u64* err, int stage, long long v, int code, int g) {
  const u64 key = ((u64)stage << 40) | ((u64)v << 8) | ((u64)code << 4) | (u64)g;
  atomicMin(err, key);
}

// One vertex's raw columns (kernels.cpp:384-412) and their exact net
// back-substitution (conversion.cpp:80-116); v = ORIGINAL id (error order),
// r = its row in the vector arrays.
__device__ __forceinline__ void epi_row_full(const EpilogueIn& in, const DictInfo& D, int v, int r,
                                        int lenient, bool want_net, u64* __restrict__ err,
                                        u64 (&rw)[16], u64 (&nt)[16]) {
  const int k = D.k;
  const unsigned m = D.mask;
  const u64 d = (u64)(in.rp[r + 1] - in.rp[r]);
  u64 col[16];
  u64 t;
  col[0] = 1;
  col[1] = d;
  col[2] = (m & (1u << 2) || m & (1u << 5) || m & (1u << 6)) && in.p2 ? in.p2[r] : 0;
  // col 3: choose2(p1), checked (types.hpp:84-88)
  col[3] = 0;
  if (m & (1u << 3) && d >= 2) {
    if (mul_ov(d, d - 1, &t)) offer_err(err, 1, v, 0, 3);
    col[3] = t / 2;
  }
  const u64 c3v = in.c3 ? in.c3[r] : 0;
  col[4] = c3v;
  col[5] = in.p3 ? in.p3[r] : 0;
  col[6] = 0;
  if (m & (1u << 6)) {
    if (mul_ov(col[2], sat_sub(d, 1), &t)) offer_err(err, 2, v, 0, 6);
    col[6] = sat_sub(t, 2 * c3v);
  }
  col[7] = in.d7 ? in.d7[r] : 0;
  col[8] = 0;
  if (m & (1u << 8) && d >= 3) {  // choose3: unchecked d(d-1)/2, checked *(d-2)
    if (mul_ov(d * (d - 1) / 2, d - 2, &t)) offer_err(err, 4, v, 0, 8);
    col[8] = t / 3;
  }
  col[9] = in.d9 ? in.d9[r] : 0;
  col[10] = in.d10 ? in.d10[r] : 0;
  col[11] = 0;
  if (m & ((1u << 9) | (1u << 10) | (1u << 11))) {
    if (mul_ov(sat_sub(d, 2), c3v, &t)) offer_err(err, 5, v, 0, 11);
    col[11] = t;
  }
  col[12] = in.c4 ? in.c4[r] : 0;
  col[13] = in.d13 ? in.d13[r] : 0;
  col[14] = in.d14 ? in.d14[r] : 0;
  col[15] = in.d15 ? in.d15[r] : 0;
  // full dictionary: identity column map and the constant U16, fully
  // unrolled with no data-dependent control flow. Every row is computed; the
  // reported failure is the first one of the reference's downward walk (the
  // highest failing row: rows below it only see values the walk never
  // produces).
#pragma unroll
  for (int i = 0; i < 16; ++i) rw[i] = col[i];
  if (!want_net) {
#pragma unroll
    for (int i = 0; i < 16; ++i) nt[i] = 0;
    return;
  }
  int bad_r = -1, bad_code = 0;
#pragma unroll
  for (int rr = 15; rr >= 0; --rr) {
    u64 absorbed = 0;
    bool ov = false;
#pragma unroll
    for (int cc = rr + 1; cc < 16; ++cc) {
      if (u16_coef(rr, cc) == 0) continue;
      u64 prod;
      ov |= mul_ov((u64)u16_coef(rr, cc), nt[cc], &prod);
      ov |= add_ov(absorbed, prod, &absorbed);
    }
    const bool neg = absorbed > rw[rr];
    nt[rr] = neg ? 0ull : rw[rr] - absorbed;
    if (bad_r < 0 && (ov || (neg && !lenient))) {
      bad_r = rr;
      bad_code = ov ? 0 : 1;
    }
  }
  if (bad_r >= 0) offer_err(err, 6, v, bad_code, bad_r);
}

__device__ __forceinline__ void epi_row(const EpilogueIn& in, const DictInfo& D, int v, int r,
                                        int lenient, bool want_net, u64* __restrict__ err,
                                        u64 (&rw)[16], u64 (&nt)[16]) {
  const int k = D.k;
  const unsigned m = D.mask;
  const u64 d = (u64)(in.rp[r + 1] - in.rp[r]);
  u64 col[16];
  u64 t;
  col[0] = 1;
  col[1] = d;
  col[2] = (m & (1u << 2) || m & (1u << 5) || m & (1u << 6)) && in.p2 ? in.p2[r] : 0;
  // col 3: choose2(p1), checked (types.hpp:84-88)
  col[3] = 0;
  if (m & (1u << 3) && d >= 2) {
    if (mul_ov(d, d - 1, &t)) offer_err(err, 1, v, 0, 3);
    col[3] = t / 2;
  }
  const u64 c3v = in.c3 ? in.c3[r] : 0;
  col[4] = c3v;
  col[5] = in.p3 ? in.p3[r] : 0;
  col[6] = 0;
  if (m & (1u << 6)) {
    if (mul_ov(col[2], sat_sub(d, 1), &t)) offer_err(err, 2, v, 0, 6);
    col[6] = sat_sub(t, 2 * c3v);
  }
  col[7] = in.d7 ? in.d7[r] : 0;
  col[8] = 0;
  if (m & (1u << 8) && d >= 3) {  // choose3: unchecked d(d-1)/2, checked *(d-2)
    if (mul_ov(d * (d - 1) / 2, d - 2, &t)) offer_err(err, 4, v, 0, 8);
    col[8] = t / 3;
  }
  col[9] = in.d9 ? in.d9[r] : 0;
  col[10] = in.d10 ? in.d10[r] : 0;
  col[11] = 0;
  if (m & ((1u << 9) | (1u << 10) | (1u << 11))) {
    if (mul_ov(sat_sub(d, 2), c3v, &t)) offer_err(err, 5, v, 0, 11);
    col[11] = t;
  }
  col[12] = in.c4 ? in.c4[r] : 0;
  col[13] = in.d13 ? in.d13[r] : 0;
  col[14] = in.d14 ? in.d14[r] : 0;
  col[15] = in.d15 ? in.d15[r] : 0;
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (i < k) rw[i] = col[D.ids[i]];
  bool stop = !want_net;  // raw only: the conversion never runs
  for (int rr = k - 1; rr >= 0; --rr) {
    u64 absorbed = 0;
    nt[rr] = 0;
    if (stop) continue;
    for (int j = 0; j < D.ntail[rr]; ++j) {
      u64 prod;
      if (mul_ov((u64)D.tail_coef[rr][j], nt[D.tail_col[rr][j]], &prod) ||
          add_ov(absorbed, prod, &absorbed)) {
        offer_err(err, 6, v, 0, D.ids[rr]);
        stop = true;
        break;
      }
    }
    if (stop) continue;
    if (absorbed > rw[rr]) {
      if (!lenient) {
        offer_err(err, 6, v, 1, D.ids[rr]);
        stop = true;
        continue;
      }
      nt[rr] = 0;
    } else {
      nt[rr] = rw[rr] - absorbed;
    }
  }
}

constexpr int kEpilogueThreads = 128;

__global__ void __launch_bounds__(kEpilogueThreads) k_epilogue(EpilogueIn in, const DictInfo* __restrict__ dict, int v0, int v1,
                           int lenient, u64* __restrict__ raw, u64* __restrict__ net,
                           u64* __restrict__ err) {
  __shared__ DictInfo D;
  // rows are staged here and written out coalesced (a thread's own row is
  // 128 B: direct stores would touch 32 lines per warp instruction)
  __shared__ u64 stage[kEpilogueThreads * 17];
  if (threadIdx.x == 0) D = *dict;
  __syncthreads();
  const int k = D.k;
  const int stride = k | 1;  // odd row stride: conflict-free 8-byte staging
  const unsigned m = D.mask;
  for (int vb = v0 + blockIdx.x * blockDim.x; vb < v1; vb += gridDim.x * blockDim.x) {
    const int v = vb + threadIdx.x;
    const int nrows = min((int)blockDim.x, v1 - vb);
    auto store_rows = [&](const u64* vals, u64* out) {
      __syncthreads();
      if (v < v1)
        for (int i = 0; i < k; ++i) stage[threadIdx.x * stride + i] = vals[i];
      __syncthreads();
      u64* o = out + (long long)(vb - v0) * k;
      for (int i = threadIdx.x; i < nrows * k; i += blockDim.x) {
        const int row = i / k;
        o[i] = stage[row * stride + (i - row * k)];
      }
    };
    u64 rw[16], nt[16];
    if (v < v1) {
    const int r = in.inv ? in.inv[v] : v;
    epi_row(in, D, v, r, lenient, net != nullptr, err, rw, nt);
    }
    if (raw) store_rows(rw, raw);
    if (net) store_rows(nt, net);
  }
}

// Whole-table variant (rows [0, n)): walks the vector rows r in order (every
// vector read coalesced) and writes each row to its original id perm[r] as
// whole 16-byte units (a full 128-byte line per table when k = 16).
// Full dictionary, 16-byte aligned tables: a warp stages its 32 rows in
// shared memory and writes every table row as one coalesced 128-byte line
// (8 lanes x 16 bytes, 4 rows per store instruction) instead of 32 scattered
// 16-byte pieces per instruction.
constexpr int kEpiStride = 17;  // u64 per staged row: odd, so lanes' rows spread over banks
__device__ __forceinline__ void epi_store_lines(const u64* __restrict__ st, int lane, int base,
                                                int n, int v_lane, u64* __restrict__ table) {
  const int c = lane & 7;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int j = it * 4 + (lane >> 3);
    const int vj = __shfl_sync(0xffffffffu, v_lane, j);
    if (base + j < n) {
      const u64* src = st + j * kEpiStride + 2 * c;
      *reinterpret_cast<ulonglong2*>(table + (long long)vj * 16 + 2 * c) =
          make_ulonglong2(src[0], src[1]);
    }
  }
}

// Full-dictionary row of vertex v (vector row r) computed straight into the
// staging row `row` (shared memory): raw columns (kernels.cpp:384-412), and
// after the raw line is stored, the net back substitution IN PLACE (row r of
// U16 only reads net entries c > r, already overwritten) — no 32-u64 register
// arrays, so the kernel runs at high occupancy.
__device__ __forceinline__ void epi_raw_into(const EpilogueIn& in, int v, int r, u64* err,
                                             u64* __restrict__ row) {
  const u64 d = (u64)(in.rp[r + 1] - in.rp[r]);
  u64 t;
  row[0] = 1;
  row[1] = d;
  const u64 p2 = in.p2 ? in.p2[r] : 0;
  row[2] = p2;
  u64 c2 = 0;
  if (d >= 2) {
    if (mul_ov(d, d - 1, &t)) offer_err(err, 1, v, 0, 3);
    c2 = t / 2;
  }
  row[3] = c2;
  const u64 c3v = in.c3 ? in.c3[r] : 0;
  row[4] = c3v;
  row[5] = in.p3 ? in.p3[r] : 0;
  if (mul_ov(p2, sat_sub(d, 1), &t)) offer_err(err, 2, v, 0, 6);
  row[6] = sat_sub(t, 2 * c3v);
  row[7] = in.d7 ? in.d7[r] : 0;
  u64 c8 = 0;
  if (d >= 3) {  // choose3: unchecked d(d-1)/2, checked *(d-2)
    if (mul_ov(d * (d - 1) / 2, d - 2, &t)) offer_err(err, 4, v, 0, 8);
    c8 = t / 3;
  }
  row[8] = c8;
  row[9] = in.d9 ? in.d9[r] : 0;
  row[10] = in.d10 ? in.d10[r] : 0;
  if (mul_ov(sat_sub(d, 2), c3v, &t)) offer_err(err, 5, v, 0, 11);
  row[11] = t;
  row[12] = in.c4 ? in.c4[r] : 0;
  row[13] = in.d13 ? in.d13[r] : 0;
  row[14] = in.d14 ? in.d14[r] : 0;
  row[15] = in.d15 ? in.d15[r] : 0;
}

__device__ __forceinline__ void epi_net_in_place(int v, int lenient, u64* err,
                                                 u64* __restrict__ row) {
  int bad_r = -1, bad_code = 0;
#pragma unroll
  for (int rr = 15; rr >= 0; --rr) {
    u64 absorbed = 0;
    bool ov = false;
#pragma unroll
    for (int cc = rr + 1; cc < 16; ++cc) {
      if (u16_coef(rr, cc) == 0) continue;
      u64 prod;
      ov |= mul_ov((u64)u16_coef(rr, cc), row[cc], &prod);
      ov |= add_ov(absorbed, prod, &absorbed);
    }
    const u64 x = row[rr];
    const bool neg = absorbed > x;
    row[rr] = neg ? 0ull : x - absorbed;
    if (bad_r < 0 && (ov || (neg && !lenient))) {
      bad_r = rr;
      bad_code = ov ? 0 : 1;
    }
  }
  if (bad_r >= 0) offer_err(err, 6, v, bad_code, bad_r);
}

// Full dictionary, 16-byte aligned tables (the common case): a warp stages
// its 32 rows in shared memory, writes every table row as one coalesced
// 128-byte line, and converts raw -> net in place between the two stores.
// Few live registers: 12 blocks of 128 threads per SM.
__global__ void __launch_bounds__(kEpilogueThreads, 12) k_epilogue_lines(
    EpilogueIn in, const int* __restrict__ perm, int n, int lenient, u64* __restrict__ raw,
    u64* __restrict__ net, u64* __restrict__ err) {
  __shared__ u64 stage[kEpilogueThreads / 32][32 * kEpiStride];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64* sr = stage[wid];
  u64* mine = sr + lane * kEpiStride;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) << 5; base < n;
       base += warps << 5) {
    const int r = base + lane;
    int v = 0;
    if (r < n) {
      v = perm[r];
      epi_raw_into(in, v, r, err, mine);
    }
    __syncwarp();
    if (raw) epi_store_lines(sr, lane, base, n, v, raw);
    __syncwarp();
    if (net) {
      if (r < n) epi_net_in_place(v, lenient, err, mine);
      __syncwarp();
      epi_store_lines(sr, lane, base, n, v, net);
      __syncwarp();
    }
  }
}

template <bool kFull>
__global__ void __launch_bounds__(kEpilogueThreads) k_epilogue_rank(
    EpilogueIn in, const int* __restrict__ perm, const DictInfo* __restrict__ dict, int n,
    int lenient, u64* __restrict__ raw, u64* __restrict__ net, u64* __restrict__ err) {
  __shared__ DictInfo D;
  if (threadIdx.x == 0) D = *dict;
  __syncthreads();
  const int k = D.k;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const int v = perm[r];
    const long long o = (long long)v * k;
    if (kFull) {  // full dictionary: all tables in registers, 16-byte stores
      u64 rw[16], nt[16];
      epi_row_full(in, D, v, r, lenient, net != nullptr, err, rw, nt);
      if (((reinterpret_cast<unsigned long long>(raw) |
            reinterpret_cast<unsigned long long>(net)) & 15ull) == 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          if (raw) *reinterpret_cast<ulonglong2*>(raw + o + i) = make_ulonglong2(rw[i], rw[i + 1]);
          if (net) *reinterpret_cast<ulonglong2*>(net + o + i) = make_ulonglong2(nt[i], nt[i + 1]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (raw) raw[o + i] = rw[i];
          if (net) net[o + i] = nt[i];
        }
      }
      continue;
    }
    u64 rw[16], nt[16];
    epi_row(in, D, v, r, lenient, net != nullptr, err, rw, nt);
    const bool vec = (k & 1) == 0 &&
                     ((reinterpret_cast<unsigned long long>(raw) |
                       reinterpret_cast<unsigned long long>(net)) & 15ull) == 0;
    if (vec) {
      if (raw)
        for (int i = 0; i < k; i += 2)
          *reinterpret_cast<ulonglong2*>(raw + o + i) = make_ulonglong2(rw[i], rw[i + 1]);
      if (net)
        for (int i = 0; i < k; i += 2)
          *reinterpret_cast<ulonglong2*>(net + o + i) = make_ulonglong2(nt[i], nt[i + 1]);
    } else {
      if (raw)
        for (int i = 0; i < k; ++i) raw[o + i] = rw[i];
      if (net)
        for (int i = 0; i < k; ++i) net[o + i] = nt[i];
    }
  }
}

// Stand-alone net_from_raw over a given raw table (conversion.cpp:80-116).
__global__ void k_net_only(const u64* __restrict__ raw, const DictInfo* __restrict__ dict,
                           long long n, int lenient, u64* __restrict__ net, u64* __restrict__ err) {
  __shared__ DictInfo D;
  if (threadIdx.x == 0) D = *dict;
  __syncthreads();
  const int k = D.k;
  for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    u64 nt[16];
    bool stop = false;
    for (int rr = k - 1; rr >= 0; --rr) {
      u64 absorbed = 0;
      nt[rr] = 0;
      if (stop) continue;
      for (int j = 0; j < D.ntail[rr]; ++j) {
        u64 prod;
        if (mul_ov((u64)D.tail_coef[rr][j], nt[D.tail_col[rr][j]], &prod) ||
            add_ov(absorbed, prod, &absorbed)) {
          offer_err(err, 6, v, 0, D.ids[rr]);
          stop = true;
          break;
        }
      }
      if (stop) continue;
      const u64 x = raw[v * k + rr];
      if (absorbed > x) {
        if (!lenient) { offer_err(err, 6, v, 1, D.ids[rr]); stop = true; continue; }
        nt[rr] = 0;
      } else {
        nt[rr] = x - absorbed;
      }
    }
    for (int i = 0; i < k; ++i) net[v * k + i] = nt[i];
  }
}

// W = sum d^2, d_max (stats and the roofline model).
__global__ void k_graph_stats(const int* __restrict__ rp, int n, u64* __restrict__ out) {
  // out[0] W = sum d^2, out[1] d_max, out[3] n_active (#vertices of degree >= 2)
  u64 w = 0, dm = 0, act = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 d = (u64)(rp[i + 1] - rp[i]);
    w += d * d;
    dm = d > dm ? d : dm;
    act += d >= 2;
  }
  w = warp_sum_u64(w);
  act = warp_sum_u64(act);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 x = __shfl_xor_sync(0xffffffffu, dm, o);
    dm = x > dm ? x : dm;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, w);
    atomicMax(out + 1, dm);
    if (act) atomicAdd(out + 3, act);
  }
}

// Bin roots into compact work lists. The kernel that computes the keys also
// tallies the bins (bin_tally: lane q of a warp accumulates bin q, one atomic
// per warp and bin at the end), so the lists are sized exactly: one array of
// (#binned roots) ints per binning instead of one n-int list per bin.
// lists[base[b] ..] gets the roots of bin b (order within a bin is arbitrary)
__global__ void k_bin(const u32* __restrict__ key, int u0, int u1, BinThr T, BinBases B,
                      int* __restrict__ cursors, int* __restrict__ list) {
  // warp-aggregated: one atomic per (warp, bin) instead of one per root
  const int lane = threadIdx.x & 31;
  const int span = u1 - u0;
  const int stride = gridDim.x * blockDim.x;
  for (int i0 = (blockIdx.x * blockDim.x + threadIdx.x) - lane; i0 < span; i0 += stride) {
    const int i = i0 + lane;
    const int b = i < span ? bin_of(key[u0 + i], T) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, b);
    if (b >= 0) {
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(cursors + b, __popc(peers));
      base = __shfl_sync(peers, base, leader);
      const int rank = __popc(peers & ((1u << lane) - 1));
      list[B.base[b] + base + rank] = u0 + i;
    }
  }
}

}  // namespace fglt
