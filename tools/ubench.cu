// Pipe-throughput micro-benchmark for the ALU rooflines in bench.py / DESIGN.md §6:
// MUFU rcp.approx.f32, MUFU ex2.approx.f32, MUFU lg2.approx.f32, FFMA, DFMA,
// MUFU rcp.approx.ftz.f64 (RCP64H seed) and the IEEE fp64 reciprocal __drcp_rn.
//
// Every thread runs 8 independent dependency chains; each operation consumes the
// previous result of its chain, so nothing can be folded or hoisted, and every chain's
// final value is stored.  The MUFU ops are inline PTX behind asm volatile.  The rate
// per SM per clock divides the event-timed throughput by (SMs x the SM clock measured
// inside the kernel from clock64 against %globaltimer), so it does not assume any
// occupancy.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int OP>
__global__ void kern(float* out, double* outd, int iters, float m, float c, double md, double cd,
                     unsigned long long* clk) {
  float a[8];
  double d[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = 1.0f + threadIdx.x * 1e-3f + i;
    d[i] = a[i];
  }
  const long long c0 = clock64();
  const unsigned long long g0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // rcp is an involution: ptxas folds rcp(rcp(x)) pairs, so each step adds c (FMA pipe)
      if (OP == 0) asm volatile("rcp.approx.ftz.f32 %0, %0;\n\tadd.ftz.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(c));
      if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 2) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 3) a[i] = fmaf(a[i], m, c);
      if (OP == 4) d[i] = fma(d[i], md, cd);
      if (OP == 5) asm volatile("rcp.approx.ftz.f64 %0, %0;\n\tadd.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(cd));
      if (OP == 6) d[i] = __drcp_rn(d[i]);
    }
  }
  const long long c1 = clock64();
  const unsigned long long g1 = gtimer();
  float s = 0;
  double sd = 0;
  for (int i = 0; i < 8; ++i) {
    s += a[i];
    sd += d[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    clk[0] = (unsigned long long)(c1 - c0);
    clk[1] = g1 - g0;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int T = 256, B = sms * 8;
  float* o;
  double* od;
  unsigned long long* clk;
  cudaMalloc(&o, (size_t)B * T * 4);
  cudaMalloc(&od, (size_t)B * T * 8);
  cudaMalloc(&clk, 16);
  const char* names[] = {"MUFU.RCP f32", "MUFU.EX2 f32", "MUFU.LG2 f32", "FFMA",
                         "DFMA", "MUFU.RCP64H f64", "__drcp_rn f64"};
  const int iters[] = {4096, 4096, 4096, 16384, 2048, 1024, 256};
  void (*ks[])(float*, double*, int, float, float, double, double, unsigned long long*) = {
      kern<0>, kern<1>, kern<2>, kern<3>, kern<4>, kern<5>, kern<6>};
  printf("%d SMs, %d CTAs x %d threads, 8 chains per thread\n", sms, B, T);
  printf("%-16s %12s %10s %14s %10s\n", "op", "ops/s", "SM MHz", "ops/clk/SM", "ms");
  for (int k = 0; k < 7; ++k) {
    ks[k]<<<B, T>>>(o, od, 16, 0.999f, 1e-3f, 0.999, 1e-3, clk);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", names[k], cudaGetErrorString(e));
      return 1;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ks[k]<<<B, T>>>(o, od, iters[k], 0.999f, 1e-3f, 0.999, 1e-3, clk);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("%s: launch failed\n", names[k]);
      return 1;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c[2];
    cudaMemcpy(c, clk, 16, cudaMemcpyDeviceToHost);
    const double mhz = (double)c[0] / (double)c[1] * 1e3;
    const double ops = (double)B * T * iters[k] * 8;
    const double rate = ops / (ms * 1e-3);
    printf("%-16s %12.4e %10.0f %14.2f %10.3f\n", names[k], rate, mhz, rate / (sms * mhz * 1e6), ms);
  }
  return 0;
}
