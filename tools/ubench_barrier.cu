// Grid-barrier micro-benchmark: G co-resident CTAs x `iters` barriers (stm::grid_barrier).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2202_10042_b200/csrc tools/ubench_barrier.cu -o /tmp/ub
#include <cstdio>
#include <cuda_runtime.h>
#include "fs1_stream.cuh"
using namespace fs1;

__global__ void kbar(unsigned* bar, int iters, int variant) {
  unsigned gen = 0;
  for (int i = 0; i < iters; ++i) {
    if (variant == 0) {
      stm::grid_barrier(bar, gridDim.x, gen);
    } else {  // release/acquire only (no __threadfence, no proxy fences)
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned target = (gen + 1) * gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        while (stm::ld_acquire(bar) < target) {
        }
      }
      ++gen;
      __syncthreads();
    }
  }
}

int main() {
  unsigned* bar;
  cudaMalloc(&bar, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {1, 2}) {
    for (int variant : {0, 1}) {
      const int G = sms * per, iters = 2000;
      cudaMemset(bar, 0, 8);
      void* args[] = {&bar, (void*)&iters, &variant};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel((void*)kbar, G, 256, args, 0, 0);  // warm-up
      cudaMemset(bar, 0, 8);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)kbar, G, 256, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("G %d variant %d: %.3f us per barrier (%s)\n", G, variant, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
