// Microbenchmark: does an LDS issued after in-flight cp.async (LDGSTS) wait for them?
// mode 0: loop { 4x cp.async 16B (random rows, L2/HBM) }; mode 1: + LDS of an unrelated smem
// word whose value feeds the next iteration's addresses (dependent chain, like the gather's
// index rows); mode 2: LDS only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldsorder ldsorder.cu && ./ldsorder
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const uint4* __restrict__ src, int64_t nrows, int iters, unsigned long long* out) {
  __shared__ __align__(16) uint4 buf[128 * 4];
  __shared__ int idx[256];
  const int t = threadIdx.x;
  idx[t] = (t * 7919) & 255;
  __syncthreads();
  uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&buf[t * 4]));
  int j = t;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    if (MODE != 2) {
      const uint4* s = src + ((static_cast<int64_t>(j) * 2654435761ull + i * 40503ull) % nrows) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + q * 16), "l"(s + q) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 6;" ::: "memory");  // keep <= 6 groups in flight
    }
    if (MODE != 0) j = idx[(j + i) & 255];  // dependent LDS
    else j = (j * 5 + 1) & 255;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (t == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (j == -1) out[1] = 0;
}

int main() {
  const int64_t nrows = 1 << 20;  // 64 MB of rows
  uint4* src;
  cudaMalloc(&src, nrows * 64);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  const int iters = 4000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<296, 128>>>(src, nrows, iters, d);
      if (mode == 1) k<1><<<296, 128>>>(src, nrows, iters, d);
      if (mode == 2) k<2><<<296, 128>>>(src, nrows, iters, d);
      cudaDeviceSynchronize();
    }
    unsigned long long ns;
    cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %.1f ns/iter (%s)\n", mode, mode == 0 ? "cp.async only" : (mode == 1 ? "cp.async + dependent LDS" : "LDS only"),
           double(ns) / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
