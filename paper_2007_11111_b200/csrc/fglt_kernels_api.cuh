// fglt_kernels_api.cuh — device kernels behind the reference's public
// per-kernel functions (proj/include/graphlet/kernels.hpp:43-98,
// src/kernels.cpp:26-288): compute_p2, compute_p3, compute_d7, compute_d8,
// compute_d9_d10_d11, the per-edge C3 in ORIGINAL CSR positions for
// compute_c3_C3, and compute_d13 for a caller-supplied C3.
//
// These take the caller's vectors as given (p1 need not be the degree
// vector), walk the ORIGINAL int32 CSR, and reproduce the reference's
// arithmetic site by site: unchecked sums wrap mod 2^64, checked sites raise
// OverflowError(graphlet, vertex). One thread per vertex walks its row in
// the reference's loop order, so the first failing site of a vertex is the
// reference's; across vertices the lowest vertex is reported (the reference's
// parallel_for reports whichever worker throws first; with one thread, the
// lowest vertex). The error word is the context's d_small[0] (atomicMin of
// vertex << 8 | graphlet, the epilogue's encoding with stage 0).
#pragma once

namespace fglt {

__device__ __forceinline__ void api_fail(u64* errw, int g, long long v) {
  atomicMin(reinterpret_cast<unsigned long long*>(errw),
            ((unsigned long long)v << 8) | (unsigned long long)g);
}

// checked helpers (types.hpp:59-94 of the reference): return false on overflow
__device__ __forceinline__ bool ck_add(u64 a, u64 b, u64* r) {
  *r = a + b;
  return *r >= a;
}
__device__ __forceinline__ bool ck_mul(u64 a, u64 b, u64* r) {
  *r = a * b;
  return a == 0 || __umul64hi(a, b) == 0;
}
__device__ __forceinline__ bool ck_choose2(u64 d, u64* r) {
  if (d < 2) { *r = 0; return true; }
  u64 x;
  if (!ck_mul(d, d - 1, &x)) return false;
  *r = x / 2;
  return true;
}
__device__ __forceinline__ bool ck_choose3(u64 d, u64* r) {
  if (d < 3) { *r = 0; return true; }
  u64 x;
  if (!ck_mul(d * (d - 1) / 2, d - 2, &x)) return false;
  *r = x / 3;
  return true;
}

// compute_p2 (kernels.cpp:26-39): p2[i] = sat_sub(sum_{j in N(i)} p1[j], p1[i])
__global__ void k_api_p2(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                         const u64* __restrict__ p1, u64* __restrict__ p2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 acc = 0;
    for (int e = rp[i]; e < rp[i + 1]; ++e) acc += p1[ci[e]];
    p2[i] = sat_sub(acc, p1[i]);
  }
}

// compute_p3 (kernels.cpp:91-107)
__global__ void k_api_p3(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                         const u64* __restrict__ p1, const u64* __restrict__ p2,
                         const u64* __restrict__ c3, u64* __restrict__ p3) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 walk = 0;
    for (int e = rp[i]; e < rp[i + 1]; ++e) walk += p2[ci[e]];
    const u64 back = p1[i] * sat_sub(p1[i], 1) + 2 * c3[i];
    p3[i] = sat_sub(walk, back);
  }
}

// compute_d7 (kernels.cpp:149-163): checked choose2 and sum, graphlet 7
__global__ void k_api_d7(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                         const u64* __restrict__ p1, u64* __restrict__ d7, u64* errw) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 acc = 0;
    bool ok = true;
    for (int e = rp[i]; e < rp[i + 1] && ok; ++e) {
      u64 c;
      ok = ck_choose2(sat_sub(p1[ci[e]], 1), &c) && ck_add(acc, c, &acc);
    }
    if (!ok) api_fail(errw, 7, i);
    d7[i] = acc;
  }
}

// compute_d8 (kernels.cpp:165-174): checked choose3, graphlet 8
__global__ void k_api_d8(int n, const u64* __restrict__ p1, u64* __restrict__ d8, u64* errw) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 r = 0;
    if (!ck_choose3(p1[i], &r)) api_fail(errw, 8, i);
    d8[i] = r;
  }
}

// compute_d9_d10_d11 (kernels.cpp:176-205): per neighbour, the graphlet-9
// sum is checked before the graphlet-10 product and sum; d11 after the row.
__global__ void k_api_d9_11(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                            const u64* __restrict__ p1, const u64* __restrict__ c3,
                            const u64* __restrict__ C3, u64* __restrict__ d9,
                            u64* __restrict__ d10, u64* __restrict__ d11, u64* errw) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    u64 nt = 0, base = 0;
    int bad = 0;
    for (int e = rp[i]; e < rp[i + 1] && !bad; ++e) {
      const int j = ci[e];
      if (!ck_add(nt, c3[j], &nt)) { bad = 9; break; }
      u64 t;
      if (!ck_mul(C3[e], sat_sub(p1[j], 2), &t) || !ck_add(base, t, &base)) bad = 10;
    }
    u64 x11 = 0;
    if (!bad && !ck_mul(sat_sub(p1[i], 2), c3[i], &x11)) bad = 11;
    if (bad) api_fail(errw, bad, i);
    d9[i] = sat_sub(nt, 2 * c3[i]);
    d10[i] = base;
    d11[i] = x11;
  }
}

// Per-edge C3 in ORIGINAL positions from the relabelled pipeline's C3f:
// original slot (i, j) is relabelled slot (inv[i], inv[j]), found by a binary
// search of the relabelled row. Warp per original row.
__global__ void k_api_map_c3(const int* __restrict__ orp, const int* __restrict__ oci, int n,
                             const int* __restrict__ inv, const int* __restrict__ rrp,
                             const int* __restrict__ rci, const u32* __restrict__ C3f,
                             const u64* __restrict__ c3r, u64* __restrict__ C3, u64* __restrict__ c3) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int r = inv[i];
    const int b = rrp[r], e = rrp[r + 1];
    for (int p = orp[i] + lane; p < orp[i + 1]; p += 32) {
      const int t = inv[oci[p]];
      const int q = lower_bound_i32(rci, b, e, t);
      C3[p] = C3f[q];
    }
    if (lane == 0) c3[i] = c3r[r];
  }
}

// Number of slots where a != b (a: caller's uint64 C3, b: device C3).
__global__ void k_api_diff(const u64* __restrict__ a, const u64* __restrict__ b, long long cnt,
                           unsigned long long* __restrict__ ndiff) {
  unsigned long long d = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt;
       i += (long long)gridDim.x * blockDim.x)
    d += a[i] != b[i];
  d = __reduce_add_sync(0xffffffffu, (unsigned)d);
  if ((threadIdx.x & 31) == 0 && d) atomicAdd(ndiff, d);
}

// compute_d13 for an arbitrary caller C3 (kernels.cpp:207-232):
// d13[i] = (1/2) sum_{j in N(i)} sum_{k in N(j) cap N(i)} sat_sub(C3(j,k), 1),
// C3(j,k) read from row j. Warp per row i; lanes over the members of N(j),
// membership in N(i) by binary search of row i. Unchecked, as the reference.
__global__ void k_api_d13(const int* __restrict__ rp, const int* __restrict__ ci, int n,
                          const u64* __restrict__ C3, u64* __restrict__ d13) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int bi = rp[i], ei = rp[i + 1];
    u64 tot = 0;
    for (int e = bi; e < ei; ++e) {
      const int j = ci[e];
      for (int p = rp[j] + lane; p < rp[j + 1]; p += 32) {
        const int k = ci[p];
        const int q = lower_bound_i32(ci, bi, ei, k);
        if (q < ei && ci[q] == k) tot += sat_sub(C3[p], 1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) d13[i] = tot / 2;
  }
}

// out[i] = v[inv[i]]: a relabelled per-vertex vector in original order.
__global__ void k_api_gather(const u64* __restrict__ v, const int* __restrict__ inv, int n,
                             u64* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = v[inv[i]];
}

}  // namespace fglt
