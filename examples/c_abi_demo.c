/* c_abi_demo.c — the FS-1 library used from plain C through include/fs1.h (no Python,
 * no PyTorch): plan, solve one batch of histogram pairs on the GPU, read the results.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c -L paper_2202_10042_b200 -lfs1 \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2202_10042_b200 -o c_abi_demo
 *   ./c_abi_demo [n] [batch] [iterations]
 *
 * Inputs: pair p has a = normalised 1 + 0.5 sin(2 pi (p+1) x), b = its mirror image, on
 * [0, 1] with h = 1/n (cell centres).  Prints each pair's transport cost, marginal error,
 * iterations and flags (Algorithm 1).
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "fs1.h"

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));             \
      return 2;                                                            \
    }                                                                      \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1024;
  const int batch = argc > 2 ? atoi(argv[2]) : 4;
  const int itr = argc > 3 ? atoi(argv[3]) : 200;
  const double pi = 3.14159265358979323846;
  double* a = (double*)malloc(sizeof(double) * n * batch);
  double* b = (double*)malloc(sizeof(double) * n * batch);
  for (int p = 0; p < batch; ++p) {
    double sa = 0, sb = 0;
    for (int i = 0; i < n; ++i) {
      const double x = (i + 0.5) / n;
      a[p * n + i] = 1.0 + 0.5 * sin(2 * pi * (p + 1) * x);
      b[p * n + i] = 1.0 + 0.5 * sin(2 * pi * (p + 1) * (1.0 - x));
      sa += a[p * n + i];
      sb += b[p * n + i];
    }
    for (int i = 0; i < n; ++i) { a[p * n + i] /= sa; b[p * n + i] /= sb; }
  }
  fs1_desc d = {0};
  d.ndim = 1; d.n = n; d.m = 1; d.h1 = 1.0 / n; d.eps = 1e-2; d.batch = batch;
  d.dtype = FS1_F64; d.domain = FS1_LOG; d.itr_max = itr; d.tol = 0.0; d.check_interval = 1;
  fs1_plan_t* plan = NULL;
  size_t ws_bytes = 0;
  fs1_status s = fs1_plan(&d, 0, &plan, &ws_bytes);
  if (s != FS1_OK) { fprintf(stderr, "fs1_plan: %s\n", fs1_status_string(s)); return 1; }
  fs1_plan_info_t info;
  fs1_plan_info(plan, &info);
  const size_t vb = sizeof(double) * n * batch;
  double *da, *db, *du, *dv, *derr, *dcost;
  int *diters, *dflags;
  void* dws = NULL;
  CK(cudaMalloc((void**)&da, vb)); CK(cudaMalloc((void**)&db, vb));
  CK(cudaMalloc((void**)&du, vb)); CK(cudaMalloc((void**)&dv, vb));
  CK(cudaMalloc((void**)&derr, sizeof(double) * batch)); CK(cudaMalloc((void**)&dcost, sizeof(double) * batch));
  CK(cudaMalloc((void**)&diters, sizeof(int) * batch)); CK(cudaMalloc((void**)&dflags, sizeof(int) * batch));
  if (ws_bytes) CK(cudaMalloc(&dws, ws_bytes));
  /* the log domain with linear weights (input_is_log = 0) */
  CK(cudaMemcpy(da, a, vb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b, vb, cudaMemcpyHostToDevice));
  s = fs1_solve(plan, da, db, du, dv, diters, derr, dflags, dcost, dws, NULL);
  if (s != FS1_OK) { fprintf(stderr, "fs1_solve: %s\n", fs1_status_string(s)); return 1; }
  CK(cudaDeviceSynchronize());
  double* cost = (double*)malloc(sizeof(double) * batch);
  double* err = (double*)malloc(sizeof(double) * batch);
  int* iters = (int*)malloc(sizeof(int) * batch);
  int* flags = (int*)malloc(sizeof(int) * batch);
  CK(cudaMemcpy(cost, dcost, sizeof(double) * batch, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(err, derr, sizeof(double) * batch, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(iters, diters, sizeof(int) * batch, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(flags, dflags, sizeof(int) * batch, cudaMemcpyDeviceToHost));
  printf("kernel %s abi %d\n", info.kernel, fs1_abi_version());
  for (int p = 0; p < batch; ++p)
    printf("pair %d cost %.17g err %.17g iters %d flags %d\n", p, cost[p], err[p], iters[p], flags[p]);
  fs1_plan_destroy(plan);
  cudaFree(da); cudaFree(db); cudaFree(du); cudaFree(dv); cudaFree(derr); cudaFree(dcost);
  cudaFree(diters); cudaFree(dflags); if (dws) cudaFree(dws);
  free(a); free(b); free(cost); free(err); free(iters); free(flags);
  return 0;
}
