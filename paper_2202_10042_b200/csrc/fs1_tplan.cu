// fs1_tplan.cu — materialise the transport plan gamma = diag(phi) K diag(psi)
// (Eq. 2.4 and the plan comparisons of Tables 1-4, column 5) for
// small problems.  One thread per entry, grid-stride:
//   gamma_ij = exp(F_i + G_j - c |i - j|)           (log domain: F, G logs)
//   gamma_ij = phi_i lambda^{|i-j|} psi_j            (scaling domain, formed as
//              exp(log phi_i + log psi_j - c |i-j|) so that lambda^{|i-j|} never
//              underflows alone, Remark 3.3)
// in fp64 and rounded once to the plan dtype.  1D index (i, j); 2D problems use the
// column-major flat index k = j2 n + i2 on both sides and the l1 distance.
// k_entries: single entries at index triples for problems of any size (fs1_plan_entries).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

namespace fs1 {

template <class T>
__global__ void k_tplan(const T* u, const T* v, T* g, long long batch, long long n, long long m, double c1,
                        double c2, int logd) {
  const long long nm = n * m;
  const long long total = batch * nm * nm;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = t / (nm * nm), r = t % (nm * nm);
    const long long k = r / nm, l = r % nm;  // source point k (phi side), target point l (psi side)
    const long long ki = k % n, kj = k / n, li = l % n, lj = l / n;
    const double d = c1 * (double)llabs(ki - li) + c2 * (double)llabs(kj - lj);
    const double a = (double)u[p * nm + k], b = (double)v[p * nm + l];
    double val;
    if (logd) val = exp(a + b - d);
    else val = (a > 0.0 && b > 0.0) ? exp(log(a) + log(b) - d) : 0.0;
    g[t] = (T)val;
  }
}

cudaError_t launch_tplan(int dtype, const void* u, const void* v, void* g, long long batch, long long n, long long m,
                         double c1, double c2, int logd, cudaStream_t st) {
  const long long total = batch * n * m * n * m;
  const int threads = 256;
  const long long blocks = std::min<long long>((total + threads - 1) / threads, 148LL * 32);
  if (dtype == 0)
    k_tplan<float><<<(unsigned)blocks, threads, 0, st>>>((const float*)u, (const float*)v, (float*)g, batch, n, m, c1,
                                                         c2, logd);
  else
    k_tplan<double><<<(unsigned)blocks, threads, 0, st>>>((const double*)u, (const double*)v, (double*)g, batch, n, m,
                                                          c1, c2, logd);
  return cudaGetLastError();
}

// Entries at index triples (fs1_plan_entries): one thread per triple, the same formula
// for any size and dimension (3D: flat index (z m + j) n + i), fp64 output; a triple
// outside the ranges gives NaN.
template <class T>
__global__ void k_entries(const T* u, const T* v, const long long* idx, long long count, double* out,
                          long long batch, long long n, long long m, long long l, double c1, double c2, double c3,
                          int logd) {
  const long long size = n * m * l;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    const long long p = idx[3 * t], k = idx[3 * t + 1], q = idx[3 * t + 2];
    if (p < 0 || p >= batch || k < 0 || k >= size || q < 0 || q >= size) {
      out[t] = NAN;
      continue;
    }
    const long long ki = k % n, kj = (k / n) % m, kz = k / (n * m);
    const long long qi = q % n, qj = (q / n) % m, qz = q / (n * m);
    const double d = c1 * (double)llabs(ki - qi) + c2 * (double)llabs(kj - qj) + c3 * (double)llabs(kz - qz);
    const double a = (double)u[p * size + k], b = (double)v[p * size + q];
    double val;
    if (logd) val = exp(a + b - d);
    else val = (a > 0.0 && b > 0.0) ? exp(log(a) + log(b) - d) : 0.0;
    out[t] = val;
  }
}

cudaError_t launch_entries(int dtype, const void* u, const void* v, const long long* idx, long long count,
                           double* out, long long batch, long long n, long long m, long long l, double c1, double c2,
                           double c3, int logd, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const int threads = 256;
  const long long blocks = std::min<long long>((count + threads - 1) / threads, 148LL * 16);
  if (dtype == 0)
    k_entries<float><<<(unsigned)blocks, threads, 0, st>>>((const float*)u, (const float*)v, idx, count, out, batch,
                                                           n, m, l, c1, c2, c3, logd);
  else
    k_entries<double><<<(unsigned)blocks, threads, 0, st>>>((const double*)u, (const double*)v, idx, count, out,
                                                            batch, n, m, l, c1, c2, c3, logd);
  return cudaGetLastError();
}

}  // namespace fs1
