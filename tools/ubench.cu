// Pipe-throughput microbenchmark (per SM per clock) for the ALU roofline of the
// persistent kernel: MUFU rcp.approx.f32, FFMA (register form), DFMA, DRCP-based
// fp64 division.  Each thread runs 8 independent chains; 148*k CTAs of 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void kern(float* out, double* outd, int iters, long long* cyc) {
  float a[8]; double d[8];
  for (int i = 0; i < 8; ++i) { a[i] = 1.0f + threadIdx.x * 1e-3f + i; d[i] = a[i]; }
  const float m = 0.999f, c = 1e-3f; const double md = 0.999, cd = 1e-3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[i])); a[i] = r; }
      if (OP == 1) a[i] = fmaf(a[i], m, c);
      if (OP == 2) d[i] = fma(d[i], md, cd);
      if (OP == 3) d[i] = __drcp_rn(d[i]);
      if (OP == 4) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[i])); a[i] = r * 1e-3f; }
    }
  }
  long long t1 = clock64();
  float s = 0; double sd = 0;
  for (int i = 0; i < 8; ++i) { s += a[i]; sd += d[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s; outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int T = 256, B = sms * 8, iters = 4096;
  float* o; double* od; long long* cyc;
  cudaMalloc(&o, B * T * 4); cudaMalloc(&od, B * T * 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"MUFU.RCP f32", "FFMA reg", "DFMA", "DRCP_rn f64", "MUFU.EX2 f32"};
  void (*ks[])(float*, double*, int, long long*) = {kern<0>, kern<1>, kern<2>, kern<3>, kern<4>};
  for (int k = 0; k < 5; ++k) {
    ks[k]<<<B, T>>>(o, od, 16, cyc);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    ks[k]<<<B, T>>>(o, od, iters, cyc);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = (double)B * T * iters * 8;
    // per-SM per-clock from the CTA-0 cycle count (8 CTAs/SM resident at 256 thr)
    double per_clk = (double)T * 8 * iters * 8 / (double)c;
    printf("%-14s %.3e ops/s  %.1f ops/clk/SM (clock64 of CTA 0)  %.3f ms\n", names[k], ops / (ms * 1e-3), per_clk, ms);
  }
  return 0;
}
