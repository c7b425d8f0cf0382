// fglt_ingest.cuh — device CSR ingest: the sanitising
// contract of build_adjacency (proj/src/graph.cpp:192-249) on the GPU.
// Each undirected pair becomes packed 64-bit keys (row << 32 | col), mirrored
// when symmetrising; self-loops and padding become the sentinel ~0, which
// sorts last. One CUB radix sort + unique give sorted, deduplicated rows; row
// offsets come from the boundaries of the sorted key array.
#pragma once

#include "fglt_device.cuh"

namespace fglt {

// flags[0] = negative id seen, flags[1] = self-loops, flags[2] = max id,
// flags[3] = input index of the first self-loop (init ~0; the reference
// reports the first one in input order, graph.cpp:207-209)
__global__ void k_ingest_scan(const long long* __restrict__ eu, const long long* __restrict__ ev,
                              long long ne, u64* __restrict__ flags) {
  long long mx = -1;
  u64 loops = 0, neg = 0, first = ~0ull;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ne;
       i += (long long)gridDim.x * blockDim.x) {
    const long long u = eu[i], v = ev[i];
    neg |= (u < 0) | (v < 0);
    if (u == v) {
      ++loops;
      if ((u64)i < first) first = (u64)i;
    }
    mx = max(mx, max(u, v));
  }
  if (first != ~0ull) atomicMin(flags + 3, first);
  loops = warp_sum_u64(loops);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    neg |= __shfl_xor_sync(0xffffffffu, neg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (neg) atomicOr(flags, 1ull);
    if (loops) atomicAdd(flags + 1, loops);
    if (mx >= 0) atomicMax(flags + 2, (u64)mx);
  }
}

__global__ void k_ingest_keys(const long long* __restrict__ eu, const long long* __restrict__ ev,
                              long long ne, int mirror, u64* __restrict__ keys) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ne;
       i += (long long)gridDim.x * blockDim.x) {
    const u64 u = (u64)eu[i], v = (u64)ev[i];
    const bool loop = u == v;
    keys[2 * i] = loop ? ~0ull : (u << 32) | v;
    keys[2 * i + 1] = (loop || !mirror) ? ~0ull : (v << 32) | u;
  }
}

// row_ptr from sorted keys: element i opens rows (row(i-1), row(i)].
__global__ void k_ingest_rows(const u64* __restrict__ keys, long long nnz, int n,
                              int* __restrict__ rp, int* __restrict__ ci) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i <= nnz;
       i += (long long)gridDim.x * blockDim.x) {
    const int row = i < nnz ? (int)(keys[i] >> 32) : n;
    const int prev = i > 0 ? (int)(keys[i - 1] >> 32) : -1;
    for (int r = prev + 1; r <= row; ++r) rp[r] = (int)i;
    if (i < nnz) ci[i] = (int)(keys[i] & 0xffffffffull);
  }
}

// Symmetry check (symmetrize off): every (u, v) needs (v, u).
__global__ void k_ingest_symmetric(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                                   u64* __restrict__ bad) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    for (int p = rp[u]; p < rp[u + 1]; ++p) {
      const int v = ci[p];
      const int q = lower_bound_i32(ci, rp[v], rp[v + 1], u);
      if (q >= rp[v + 1] || ci[q] != u) {
        atomicMin(bad, ((u64)(unsigned)u << 32) | (unsigned)v);
        break;
      }
    }
}

}  // namespace fglt
