// fs1_sep2d64.cu — K5: Algorithm 2 in fp64, scaling domain, for
// batches of small 2D problems (the paper's 2D random-distribution workload E3,
// N x N up to 160 x 160, h1 = h2 = 1, eps = 0.01, so lambda =
// e^{-100}, which fp32 cannot hold and the fp32 log-domain kernels K3 / K3w refuse).
//
// One CTA per problem for the whole solve.  Every K x is the paper's separable form
// K = T_M(lambda2) (x) T_N(lambda1): a pass along axis 1 (K0 on
// every column) then a pass along axis 2, and
// each 1D line apply is Eq. "recursion" run sequentially by ONE
// THREAD per line, exactly as the paper writes it (no scan):
//   r_1 = x_1, r_{k+1} = lambda r_k + x_{k+1};  s_N = 0, s_k = lambda (s_{k+1} + x_{k+1});
//   (K x)_k = r_k + s_k.
// The axis-2 pass is fused with the update y = tgt / (K x) (Alg. 2 lines 7 / 12) and,
// on check iterations, the marginal error (line 2).  Arrays are column-major (k =
// j n + i): the axis-2 pass (thread per row i) reads consecutive
// addresses across a warp; the axis-1 pass walks each column through L1.  The state
// (phi, psi) lives in the caller's u, v; the axis-1 result in the workspace.  The
// return line is sum phi . [(W1 (x) K2) + (K1 (x) W2)] psi with the
// weighted (Jordan-block) line apply W x = h (P' + Q'), P'_{k+1} = lambda (P'_k + p_k),
// Q'_k = lambda (Q'_{k+1} + t_{k+1}) (R7).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"
#include "fs1_dispatch.h"
#include "fs1_params.h"

namespace fs1 {
namespace s64 {

constexpr int FLAG_CONVERGED = 1, FLAG_NONFINITE = 2, FLAG_ITR_MAX = 4;

// Sequential sweeps over a line of len points at stride st (the paper's recursions are
// sequential; the loads are not): U loads are issued ahead into registers so a thread
// keeps U memory requests in flight instead of one dependent miss per step.
constexpr int U8 = 8;


// axis 1: T[:, j] = K1 x[:, j] for every column j (weighted: W1, i.e. h (P' + Q'))
template <bool WEIGHTED>
__device__ __forceinline__ void col_pass(const double* __restrict__ x, double* __restrict__ T, int n, int m,
                                         double lam, double h) {
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double* xc = x + (size_t)j * n;
    double* tc = T + (size_t)j * n;
    if (!WEIGHTED) {
      // forward: r_1 = x_1, r_{i+1} = lam r_i + x_{i+1}  (staged in tc)
      double r = 0.0;
      for (int i0 = 0; i0 < n; i0 += U8) {
        double xv[U8];
#pragma unroll
        for (int u = 0; u < U8; ++u) xv[u] = (i0 + u < n) ? xc[i0 + u] : 0.0;
#pragma unroll
        for (int u = 0; u < U8; ++u)
          if (i0 + u < n) {
            r = (i0 + u == 0) ? xv[u] : fma(lam, r, xv[u]);
            tc[i0 + u] = r;
          }
      }
      // backward: s_N = 0, s_i = lam (s_{i+1} + x_{i+1});  K x = r + s
      double s = 0.0, xn = xc[n - 1];
      for (int i1 = n - 2; i1 >= 0; i1 -= U8) {
        double xv[U8], rv[U8];
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int i = i1 - u;
          xv[u] = i >= 0 ? xc[i] : 0.0;
          rv[u] = i >= 0 ? tc[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int i = i1 - u;
          if (i >= 0) {
            s = lam * (s + xn);
            tc[i] = rv[u] + s;
            xn = xv[u];
          }
        }
      }
    } else {
      double p = xc[0], P = 0.0;
      tc[0] = 0.0;
      for (int i = 1; i < n; ++i) {
        P = lam * (P + p);
        p = fma(lam, p, xc[i]);
        tc[i] = P;
      }
      double t = xc[n - 1], Q = 0.0;
      tc[n - 1] *= h;
      for (int i = n - 2; i >= 0; --i) {
        Q = lam * (Q + t);
        t = fma(lam, t, xc[i]);
        tc[i] = h * (tc[i] + Q);
      }
    }
  }
}

// axis 2 for every row i of T (thread per row): k = K2 T[i, :] (weighted: W2), then
//   UPD:   y = tgt / k, [CHECK: err += |yold k - tgt|], written to y (r staged in y)
//   DOT:   acc += sum_j phi[i, j] k_j   (the cost)
//   APPLY: y = k
template <int MODE>
__device__ __forceinline__ void row_pass(const double* __restrict__ T, const double* __restrict__ tgt,
                                         const double* __restrict__ yold, double* __restrict__ y,
                                         const double* __restrict__ phi, int n, int m, double lam, double h,
                                         double& acc, int& bad) {
  constexpr int UPD = 1, CHECK = 2, DOT = 4, APPLY = 8, WEIGHTED = 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (MODE & WEIGHTED) {
      double p = T[i], P = 0.0, t, Q = 0.0;
      double a = 0.0;  // phi_1 P'_1 with P'_1 = 0
      for (int j = 1; j < m; ++j) {
        P = lam * (P + p);
        p = fma(lam, p, T[(size_t)j * n + i]);
        a = fma(phi[(size_t)j * n + i], P, a);
      }
      t = T[(size_t)(m - 1) * n + i];
      for (int j = m - 2; j >= 0; --j) {
        Q = lam * (Q + t);
        t = fma(lam, t, T[(size_t)j * n + i]);
        a = fma(phi[(size_t)j * n + i], Q, a);
      }
      acc = fma(h, a, acc);
      continue;
    }
    double r = T[i];
    if (!(MODE & DOT)) {
      double* st = y;  // forward values r_j staged in y, overwritten by the backward sweep
      for (int j0 = 0; j0 < m; j0 += U8) {
        double tv[U8];
#pragma unroll
        for (int u = 0; u < U8; ++u) tv[u] = (j0 + u < m) ? T[(size_t)(j0 + u) * n + i] : 0.0;
#pragma unroll
        for (int u = 0; u < U8; ++u)
          if (j0 + u < m) {
            r = (j0 + u == 0) ? tv[u] : fma(lam, r, tv[u]);
            st[(size_t)(j0 + u) * n + i] = r;
          }
      }
      double s = 0.0;
      for (int j1 = m - 1; j1 >= 0; j1 -= U8) {
        double tv[U8], rv[U8], gv[U8], ov[U8];
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int j = j1 - u;
          const size_t k = (size_t)(j >= 0 ? j : 0) * n + i;
          tv[u] = j >= 0 ? T[k] : 0.0;
          rv[u] = j >= 0 ? st[k] : 0.0;
          gv[u] = ((MODE & UPD) && j >= 0) ? tgt[k] : 0.0;
          ov[u] = ((MODE & CHECK) && j >= 0) ? yold[k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int j = j1 - u;
          if (j < 0) break;
          const size_t k = (size_t)j * n + i;
          const double kx = rv[u] + s;
          s = lam * (s + tv[u]);
          if (MODE & UPD) {
            const double out = gv[u] / kx;
            if (MODE & CHECK) acc += fabs(ov[u] * kx - gv[u]);
            bad |= !isfinite(out);
            st[k] = out;
          } else {
            st[k] = kx;
          }
        }
      }
    } else {
      // forward: sum_j phi_j r_j; backward: sum_j phi_j s_j
      double a = phi[i] * r;
      for (int j = 1; j < m; ++j) {
        r = fma(lam, r, T[(size_t)j * n + i]);
        a = fma(phi[(size_t)j * n + i], r, a);
      }
      double s = 0.0;
      for (int j = m - 2; j >= 0; --j) {
        s = lam * (s + T[(size_t)(j + 1) * n + i]);
        a = fma(phi[(size_t)j * n + i], s, a);
      }
      acc += a;
    }
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  __syncthreads();
  return s;
}

__global__ void fs1_sep2d64_kernel(const __grid_constant__ Sep2d64Params P) {
  __shared__ double red[32];
  const int n = P.n, m = P.m;
  const size_t nm = (size_t)n * m;
  const long long pb = blockIdx.x;
  double* T = P.ws + (size_t)pb * 2 * nm;
  double* Y = T + nm;
  const double* a = P.a + pb * nm;
  const double* b = P.b + pb * nm;
  double* U = P.u + pb * nm;
  double* V = P.v + pb * nm;
  int bad = 0;
  double dummy = 0.0;
  if (P.mode == 2) {  // apply: y = K x
    col_pass<false>(P.x + pb * nm, T, n, m, P.lam1, P.h1);
    __syncthreads();
    row_pass<8>(T, nullptr, nullptr, P.y + pb * nm, nullptr, n, m, P.lam2, P.h2, dummy, bad);
    return;
  }
  if (P.mode == 0) {
    // line 1: phi = psi = 1/(N M), or the caller's warm start
    if (!P.warm) {
      const double init = 1.0 / (double)nm;
      for (size_t k = threadIdx.x; k < nm; k += blockDim.x) {
        U[k] = init;
        V[k] = init;
      }
    }
    __syncthreads();
    const bool use_tol = P.tol > 0.0;
    int l = 0, flag = 0;
    double errv = NAN;
    while (true) {
      const bool check = (l >= P.itr_max) || (use_tol && (l % P.check_interval) == 0);
      // lines 2-7: psi = b ./ (K phi)  (K symmetric: K^T phi = K phi)
      col_pass<false>(U, T, n, m, P.lam1, P.h1);
      __syncthreads();
      bad = 0;
      if (check) {
        double e = 0.0;
        row_pass<1 | 2>(T, b, V, Y, nullptr, n, m, P.lam2, P.h2, e, bad);
        errv = block_sum(e, red);
        if (l >= P.itr_max || errv <= P.tol) {
          flag = (use_tol && errv <= P.tol) ? FLAG_CONVERGED : FLAG_ITR_MAX;
          break;
        }
        for (size_t k = threadIdx.x; k < nm; k += blockDim.x) V[k] = Y[k];
      } else {
        row_pass<1>(T, b, nullptr, V, nullptr, n, m, P.lam2, P.h2, dummy, bad);
      }
      __syncthreads();
      // lines 8-12: phi = a ./ (K psi)
      col_pass<false>(V, T, n, m, P.lam1, P.h1);
      __syncthreads();
      row_pass<1>(T, a, nullptr, U, nullptr, n, m, P.lam2, P.h2, dummy, bad);
      ++l;  // line 13
      if (__syncthreads_or(bad)) {
        flag = FLAG_NONFINITE;
        errv = NAN;
        break;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (P.iters) P.iters[pb] = l;
      if (P.err) P.err[pb] = errv;
      if (P.flags) P.flags[pb] = flag;
    }
    if (flag == FLAG_NONFINITE) {
      if (threadIdx.x == 0 && P.cost) P.cost[pb] = NAN;
      return;
    }
  }
  if (!P.cost) return;
  // line 14: phi . (W1 (x) K2) psi + phi . (K1 (x) W2) psi
  double acc = 0.0;
  col_pass<true>(V, T, n, m, P.lam1, P.h1);
  __syncthreads();
  row_pass<4>(T, nullptr, nullptr, nullptr, U, n, m, P.lam2, P.h2, acc, bad);
  __syncthreads();
  col_pass<false>(V, T, n, m, P.lam1, P.h1);
  __syncthreads();
  row_pass<16>(T, nullptr, nullptr, nullptr, U, n, m, P.lam2, P.h2, acc, bad);
  const double cost = block_sum(acc, red);
  if (threadIdx.x == 0) P.cost[pb] = cost;
}

}  // namespace s64

cudaError_t launch_sep2d64(const Sep2d64Params& P, long long batch, int threads, cudaStream_t st) {
  s64::fs1_sep2d64_kernel<<<(unsigned)batch, threads, 0, st>>>(P);
  return cudaGetLastError();
}

}  // namespace fs1
