// Microbenchmark: producer/consumer mbarrier ring with no payload, to measure the per-stage
// handshake floor (mbarrier arrive / try_wait, tcgen05.commit) on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring ring.cu && ./ring
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}

// mode 0: consumer arrives on empty with mbarrier.arrive; mode 1: consumer uses tcgen05.commit
// producers: P threads (all arrive on full, count P)
template <int MODE>
__global__ void ring(int iters, int S, int P, unsigned long long* out) {
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { init(&full[s], P); init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (MODE == 1 && warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x < P) {
    int st = 0; uint32_t ph = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
      wait(&empty[st], ph ^ 1);
      arrive(&full[st]);
      if (MODE == 2 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        out[1 + (i & 1023)] = t;
      }
      if (++st == S) { st = 0; ph ^= 1; }
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  } else if (warp == 4 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait(&full[st], ph);
      if (MODE != 1) arrive(&empty[st]); else commit(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  if (MODE == 1 && warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tslot));
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 1100);
  const int iters = 20000;
  for (int mode = 0; mode < 3; ++mode)
    for (int P : {1, 128})
      for (int S : {4, 9}) {
        for (int grid : {1, 296}) {
          if (mode == 0) ring<0><<<grid, 160>>>(iters, S, P, d);
          else if (mode == 1) ring<1><<<grid, 160>>>(iters, S, P, d);
          else ring<2><<<grid, 160>>>(iters, S, P, d);
          cudaDeviceSynchronize();
          unsigned long long ns; cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
          printf("mode=%s P=%3d S=%d grid=%3d: %.1f ns/stage (%s)\n", mode == 1 ? "tc_commit" : (mode == 2 ? "arrive+gtimer" : "arrive  "), P, S, grid,
                 double(ns) / iters, cudaGetErrorString(cudaGetLastError()));
        }
      }
  return 0;
}
