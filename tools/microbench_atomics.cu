// Microbenchmark: throughput of random-address counter increments through
// (a) local shared-memory atomics, (b) DSMEM atomics across an 8-CTA cluster,
// (c) global RED.ADD into an L2-resident array, (d) global random reads.
// Dev tool: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_atomics.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned hsh(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}

__global__ void k_smem(int iters, unsigned range, unsigned* out) {
  extern __shared__ unsigned L[];
  for (unsigned i = threadIdx.x; i < range; i += blockDim.x) L[i] = 0;
  __syncthreads();
  unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    s = hsh(s + i);
    atomicAdd(L + (s % range), 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = L[0];
}

__global__ void __cluster_dims__(8, 1, 1) k_dsmem(int iters, unsigned range, unsigned* out) {
  extern __shared__ unsigned L[];
  cg::cluster_group cl = cg::this_cluster();
  for (unsigned i = threadIdx.x; i < range; i += blockDim.x) L[i] = 0;
  cl.sync();
  unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    s = hsh(s + i);
    unsigned owner = s & 7;
    unsigned* remote = cl.map_shared_rank(L, owner);
    atomicAdd(remote + ((s >> 3) % range), 1u);
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = L[0];
}

// cluster of 2: every CTA adds into either half of the pair's combined
// counters (its own or its partner's shared memory), like a dense tile split
// over two SMs
__global__ void __cluster_dims__(2, 1, 1) k_dsmem2(int iters, unsigned range, unsigned* out) {
  extern __shared__ unsigned L[];
  cg::cluster_group cl = cg::this_cluster();
  for (unsigned i = threadIdx.x; i < range; i += blockDim.x) L[i] = 0;
  cl.sync();
  unsigned* mine = L;
  unsigned* other = cl.map_shared_rank(L, cl.block_rank() ^ 1);
  unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    s = hsh(s + i);
    atomicAdd(((s & 1) ? other : mine) + ((s >> 1) % range), 1u);
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = L[0];
}

__global__ void k_red(int iters, unsigned range, unsigned* arr) {
  unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    s = hsh(s + i);
    atomicAdd(arr + (s % range), 1u);
  }
}

__global__ void k_read(int iters, unsigned range, const unsigned* arr, unsigned* out) {
  unsigned s = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    s = hsh(s + i);
    acc += __ldg(arr + (s % range));
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  cudaMalloc(&out, 1 << 20);
  unsigned* arr;
  cudaMalloc(&arr, 1ull << 30);
  cudaMemset(arr, 0, 1ull << 30);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2048, threads = 1024;
  const unsigned range = 48 * 1024;
  auto time = [&](const char* name, auto launch, double ops) {
    launch();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-40s %8.3f ms  %8.2f Gops/s  %s\n", name, ms, ops / ms / 1e6, cudaGetErrorString(e));
  };
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, range * 4);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, range * 4);
  double ops = (double)sms * threads * iters;
  time("smem atomicAdd (48K u32/CTA)", [&] { k_smem<<<sms, threads, range * 4>>>(iters, range, out); }, ops);
  cudaFuncSetAttribute(k_dsmem2, cudaFuncAttributeMaxDynamicSharedMemorySize, range * 4);
  time("dsmem atomicAdd (cluster 2, half remote)",
       [&] { k_dsmem2<<<(sms / 2) * 2, threads, range * 4>>>(iters, range, out); },
       (double)((sms / 2) * 2) * threads * iters);
  int g8 = (sms / 8) * 8;
  time("dsmem atomicAdd (cluster 8)", [&] { k_dsmem<<<g8, threads, range * 4>>>(iters, range, out); },
       (double)g8 * threads * iters);
  for (unsigned mb : {4u, 16u, 64u, 256u, 1024u}) {
    unsigned r = mb * 262144u;
    char name[64];
    snprintf(name, 64, "global RED.ADD range %u MB", mb);
    time(name, [&] { k_red<<<sms * 2, threads>>>(iters / 2, r, arr); }, (double)sms * 2 * threads * iters / 2);
    snprintf(name, 64, "global random LDG range %u MB", mb);
    time(name, [&] { k_read<<<sms * 2, threads>>>(iters / 2, r, arr, out); }, (double)sms * 2 * threads * iters / 2);
  }
  return 0;
}
