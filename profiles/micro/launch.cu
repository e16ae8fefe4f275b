// Fixed cost of a fused-conv-shaped launch on B200 (profiles/micro): back-to-back launches of
// near-empty kernels with the fused kernel's launch shape (296 CTAs x 288 threads), adding one
// ingredient at a time -- 113 KB dynamic shared memory, TMEM alloc/dealloc, mbarrier init, an
// alternating small kernel with a different shared-memory carveout, PDL -- timed with CUDA
// events over 200 launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch launch.cu && ./launch
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <bool TMEM, bool BAR>
__global__ void __launch_bounds__(288, 2) k_empty(int* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ unsigned slot;
  __shared__ unsigned long long bars[16];
  if (BAR && threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(129));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TMEM && threadIdx.x / 32 == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = static_cast<int>(reinterpret_cast<size_t>(smem) & 1);
  __syncthreads();
  if (TMEM && threadIdx.x / 32 == 8)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(256) : "memory");
}

__global__ void k_small(int* out) {
  __shared__ int s[512];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (out && threadIdx.x == 0 && blockIdx.x == 0) out[1] = s[5];
}

template <class K>
float run(K kern, size_t smem, bool pdl, bool alternate, int* out, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(296);
  cfg.blockDim = dim3(288);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  for (int w = 0; w < 20; ++w) cudaLaunchKernelEx(&cfg, kern, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 200;
  cudaEventRecord(a, st);
  const auto h0 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i) {
    cudaLaunchKernelEx(&cfg, kern, out);
    if (alternate) k_small<<<148, 256, 0, st>>>(out);
  }
  const double host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count() / N;
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  std::printf("   [host enqueue %.2f us per iteration] ", host_us);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / N;
}

int main() {
  int* out;
  cudaMalloc(&out, 64);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const size_t big = 113 * 1024;
  for (auto f : {k_empty<false, false>, k_empty<true, false>, k_empty<true, true>}) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  std::printf("us per launch (296 CTAs x 288 threads, 200 back to back)\n");
  std::printf("empty, 0 smem                 %6.2f\n", run(k_empty<false, false>, 0, false, false, out, st));
  std::printf("empty, 113 KB smem            %6.2f\n", run(k_empty<false, false>, big, false, false, out, st));
  std::printf("+ TMEM alloc                  %6.2f\n", run(k_empty<true, false>, big, false, false, out, st));
  std::printf("+ mbarrier init               %6.2f\n", run(k_empty<true, true>, big, false, false, out, st));
  std::printf("+ PDL                         %6.2f\n", run(k_empty<true, true>, big, true, false, out, st));
  std::printf("alternating with a small kernel (pair):\n");
  std::printf("  no PDL                      %6.2f\n", run(k_empty<true, true>, big, false, true, out, st));
  std::printf("  PDL                         %6.2f\n", run(k_empty<true, true>, big, true, true, out, st));
  std::printf("  small kernel alone          %6.2f\n", run(k_small, 0, false, false, out, st));
  return 0;
}
