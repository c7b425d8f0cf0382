// Root cause of the round-1 "lost updates" in the d13 shared accumulators
// (DESIGN.md §4): the diamond pass added into the same shared u64 counter
// both with a 64-bit atomicAdd (which sm_100a compiles to a CAS spin loop,
// ATOMS.CAST.SPIN.64) and — on its `narrow` path — with a 32-bit atomicAdd
// on the counter's low word. Mixed-size atomics on overlapping locations are
// not atomic with respect to each other (PTX memory model: atomicity is only
// defined between operations on the same location and size). This test
// counts increments for three disciplines on hot shared counters:
//   A  64-bit atomicAdd only                    (same size: exact)
//   B  64-bit atomicAdd + 32-bit on the low word (mixed: may lose updates)
//   C  smem_add_u64 (two 32-bit atomics + carry) + 32-bit on the low word
//      (same size everywhere: exact — the fix)
// Dev tool: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_mixed microbench_mixed_atomics.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned u32;

__device__ __forceinline__ void smem_add_u64(u64* addr, u64 v) {
  u32* w = reinterpret_cast<u32*>(addr);
  const u32 vl = (u32)v, vh = (u32)(v >> 32);
  const u32 old = atomicAdd(w, vl);
  const u32 carry = (u32)(old + vl < old);
  if (vh + carry) atomicAdd(w + 1, vh + carry);
}

template <int MODE>
__global__ void k_mixed(int iters, int slots, u64* out) {
  extern __shared__ u64 S[];
  for (int i = threadIdx.x; i < slots; i += blockDim.x) S[i] = 0;
  __syncthreads();
  unsigned x = blockIdx.x * 7919u + threadIdx.x * 104729u + 1u;
  for (int i = 0; i < iters; ++i) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    u64* p = S + (x % (unsigned)slots);
    const bool narrow = (threadIdx.x & 1) != 0;  // half the threads take the 32-bit path
    if (MODE == 0) atomicAdd(p, 1ull);
    else if (MODE == 1) {
      if (narrow) atomicAdd(reinterpret_cast<u32*>(p), 1u);
      else atomicAdd(p, 1ull);
    } else {
      if (narrow) atomicAdd(reinterpret_cast<u32*>(p), 1u);
      else smem_add_u64(p, 1ull);
    }
  }
  __syncthreads();
  u64 s = 0;
  for (int i = threadIdx.x; i < slots; i += blockDim.x) s += S[i];
  atomicAdd(out, s);
}

template <int MODE>
u64 run(int blocks, int threads, int iters, int slots) {
  u64* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  k_mixed<MODE><<<blocks, threads, slots * 8>>>(iters, slots, d);
  u64 h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

int main() {
  const int blocks = 148 * 2, threads = 512, iters = 2000;
  const u64 expect = (u64)blocks * threads * iters;
  const char* names[3] = {"A 64-bit only", "B 64-bit + 32-bit low word (mixed)", "C smem_add_u64 + 32-bit low word"};
  for (int slots : {8, 64, 1024}) {
    const u64 got[3] = {run<0>(blocks, threads, iters, slots), run<1>(blocks, threads, iters, slots),
                        run<2>(blocks, threads, iters, slots)};
    for (int m = 0; m < 3; ++m)
      std::printf("slots %5d  %-38s increments %llu of %llu  lost %lld\n", slots, names[m], got[m],
                  expect, (long long)(expect - got[m]));
  }
  return 0;
}
