// fs1_extra.cu — the steps either side of the loop:
//  * k_dual: the dual objective of Eq. (2.3) at a state, from the state
//    and one kernel apply S = K psi (scaling) / log K e^G (log) done by fs1_apply:
//      D = eps (sum_{a>0} a F + sum_{b>0} b G - sum_kl gamma_kl) + eps (sum a + sum b) / 2,
//      sum_kl gamma_kl = sum_k phi_k (K psi)_k  = sum_k e^{F_k + S_k}
//    (F = log phi, G = log psi; one CTA per problem, fixed-order fp64 reduction).
//  * k_rescale: the warm start between eps-scaling stages, F <- F eps_{k-1} / eps_k
//    (the dual potentials f = eps F held fixed), elementwise in the plan dtype.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"

namespace fs1 {
namespace extra {

template <class T>
__global__ void k_dual(const T* a, const T* b, const T* u, const T* v, const T* s, long long size, double eps,
                       int logd, int input_is_log, double* out) {
  __shared__ double red[32];
  const long long p = blockIdx.x;
  const T* ap = a + p * size;
  const T* bp = b + p * size;
  const T* up = u + p * size;
  const T* vp = v + p * size;
  const T* sp = s + p * size;
  double fa = 0.0, gb = 0.0, gam = 0.0, ma = 0.0, mb = 0.0;
  for (long long k = threadIdx.x; k < size; k += blockDim.x) {
    double wa = (double)ap[k], wb = (double)bp[k];
    if (input_is_log) {
      wa = exp(wa);
      wb = exp(wb);
    }
    double F, G, g;
    if (logd) {
      F = (double)up[k];
      G = (double)vp[k];
      g = exp(F + (double)sp[k]);
    } else {
      F = log((double)up[k]);
      G = log((double)vp[k]);
      g = (double)up[k] * (double)sp[k];
    }
    if (wa > 0.0) fa = fma(wa, F, fa);
    if (wb > 0.0) gb = fma(wb, G, gb);
    gam += g;
    ma += wa;
    mb += wb;
  }
  double vals[5] = {fa, gb, gam, ma, mb};
  double tot[5];
  for (int q = 0; q < 5; ++q) {
    double x = warp_sum(vals[q]);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    tot[q] = t;
  }
  if (threadIdx.x == 0) out[p] = eps * (tot[0] + tot[1] - tot[2]) + eps * (tot[3] + tot[4]) * 0.5;
}

template <class T>
__global__ void k_rescale(T* u, T* v, long long count, double ratio) {
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (long long)gridDim.x * blockDim.x) {
    u[k] = (T)((double)u[k] * ratio);
    v[k] = (T)((double)v[k] * ratio);
  }
}

}  // namespace extra

cudaError_t launch_dual(int dtype, const void* a, const void* b, const void* u, const void* v, const void* s,
                        long long batch, long long size, double eps, int logd, int input_is_log, double* out,
                        cudaStream_t st) {
  if (dtype == 1)
    extra::k_dual<double><<<(unsigned)batch, 256, 0, st>>>((const double*)a, (const double*)b, (const double*)u,
                                                          (const double*)v, (const double*)s, size, eps, logd,
                                                          input_is_log, out);
  else
    extra::k_dual<float><<<(unsigned)batch, 256, 0, st>>>((const float*)a, (const float*)b, (const float*)u,
                                                         (const float*)v, (const float*)s, size, eps, logd,
                                                         input_is_log, out);
  return cudaGetLastError();
}

cudaError_t launch_rescale(int dtype, void* u, void* v, long long count, double ratio, cudaStream_t st) {
  const int blocks = (int)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
  if (dtype == 1)
    extra::k_rescale<double><<<blocks, 256, 0, st>>>((double*)u, (double*)v, count, ratio);
  else
    extra::k_rescale<float><<<blocks, 256, 0, st>>>((float*)u, (float*)v, count, ratio);
  return cudaGetLastError();
}

}  // namespace fs1
