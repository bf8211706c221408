// fs1_sep2d64.cu — K5: Algorithm 2 in fp64, scaling domain, for
// batches of small 2D problems and its 3D extension ("can be easily
// extended to high-dimensional cases"): the paper's 2D random-distribution workload
// E3 (N x N up to 160 x 160, h1 = h2 = 1, eps = 0.01, so lambda =
// e^{-100}, which fp32 cannot hold and the fp32 log-domain kernels K3 / K3w refuse).
//
// One CTA per problem for the whole solve.  Every K x is the separable form
// K = T_L(lambda3) (x) T_M(lambda2) (x) T_N(lambda1) (PAPER.md:255-280 for two axes):
// a pass along axis 1 (K0 on every column), then axis 2
// (PAPER.md:300-312), then axis 3 in 3D, and each 1D line apply is Eq. "recursion"
// run sequentially by ONE THREAD per line, exactly as the paper
// writes it (no scan):
//   r_1 = x_1, r_{k+1} = lambda r_k + x_{k+1};  s_N = 0, s_k = lambda (s_{k+1} + x_{k+1});
//   (K x)_k = r_k + s_k.
// The last axis's pass is fused with the update y = tgt / (K x) (Alg. 2 lines 7 / 12)
// and, on check iterations, the marginal error (line 2).  Arrays are column-major
// (flat index (z M + j) N + i, PAPER.md:244-255 extended): lines of axis 2 and 3 read
// consecutive addresses across a warp; axis-1 lines walk their column through L1.
// Loads are issued 8 deep into registers ahead of the recursion.  The state (phi,
// psi) lives in the caller's u, v; the intermediate passes in the workspace.  The
// return line (extended) is sum over axes a of phi . (K..W_a..K) psi
// with the weighted (Jordan-block) line apply W x = h (P' + Q'), P'_{k+1} =
// lambda (P'_k + p_k), Q'_k = lambda (Q'_{k+1} + t_{k+1}) (R7).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"
#include "fs1_dispatch.h"
#include "fs1_params.h"

namespace fs1 {
namespace s64 {

constexpr int FLAG_CONVERGED = 1, FLAG_NONFINITE = 2, FLAG_ITR_MAX = 4;
constexpr int U8 = 8;  // loads in flight per thread ahead of the sequential recursion

// pass modes (what happens to the line result k = K x or W x)
constexpr int STORE = 0, UPD = 1, CHECK = 2, DOT = 4;

struct Geo {
  int n, m, l;  // points along axes 1, 2, 3 (l = 1 in 2D)
};

// lines of axis `ax`: count, length, point stride, and the base offset of line `q`
__device__ __forceinline__ long long nlines(const Geo& g, int ax) {
  return ax == 0 ? (long long)g.m * g.l : ax == 1 ? (long long)g.n * g.l : (long long)g.n * g.m;
}
__device__ __forceinline__ int llen(const Geo& g, int ax) { return ax == 0 ? g.n : ax == 1 ? g.m : g.l; }
__device__ __forceinline__ long long lstride(const Geo& g, int ax) {
  return ax == 0 ? 1 : ax == 1 ? (long long)g.n : (long long)g.n * g.m;
}
__device__ __forceinline__ long long lbase(const Geo& g, int ax, long long q) {
  if (ax == 0) return q * g.n;                                     // q = z M + j
  if (ax == 1) return (q / g.n) * (long long)g.n * g.m + q % g.n;  // q = z N + i
  return q;                                                        // q = j N + i
}

// One pass of 1D line applies along axis `ax` (thread per line).  WEIGHTED: the
// distance-weighted apply W x = h (P' + Q') instead of K x.  MODE as above; UPD /
// CHECK read tgt / yold, DOT accumulates sum phi . k into acc.
template <bool WEIGHTED, int MODE>
__device__ __forceinline__ void line_pass(const Geo& g, int ax, const double* __restrict__ x,
                                          double* __restrict__ y, const double* __restrict__ tgt,
                                          const double* __restrict__ yold, const double* __restrict__ phi,
                                          double lam, double h, double& acc, int& bad) {
  const long long L = nlines(g, ax);
  const int n = llen(g, ax);
  const long long st = lstride(g, ax);
  for (long long q = threadIdx.x; q < L; q += blockDim.x) {
    const long long b0 = lbase(g, ax, q);
    auto at = [&](int k) { return b0 + (long long)k * st; };
    if (!WEIGHTED) {
      // forward: r staged in y (DOT: accumulate phi . r directly, no staging)
      double r = 0.0;
      double a = 0.0;
      for (int k0 = 0; k0 < n; k0 += U8) {
        double xv[U8], pv[U8];
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          xv[u] = (k0 + u < n) ? x[at(k0 + u)] : 0.0;
          pv[u] = ((MODE & DOT) && k0 + u < n) ? phi[at(k0 + u)] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U8; ++u)
          if (k0 + u < n) {
            r = (k0 + u == 0) ? xv[u] : fma(lam, r, xv[u]);
            if (MODE & DOT) a = fma(pv[u], r, a);
            else y[at(k0 + u)] = r;
          }
      }
      // backward: s_n = 0, s_k = lam (s_{k+1} + x_{k+1}); K x = r + s
      double s = 0.0, xn = 0.0;
      for (int k1 = n - 1; k1 >= 0; k1 -= U8) {
        double xv[U8], rv[U8], gv[U8], ov[U8], pv[U8];
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int k = k1 - u;
          const long long o = at(k >= 0 ? k : 0);
          xv[u] = k >= 0 ? x[o] : 0.0;
          rv[u] = (!(MODE & DOT) && k >= 0) ? y[o] : 0.0;
          gv[u] = ((MODE & UPD) && k >= 0) ? tgt[o] : 0.0;
          ov[u] = ((MODE & CHECK) && k >= 0) ? yold[o] : 0.0;
          pv[u] = ((MODE & DOT) && k >= 0) ? phi[o] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int k = k1 - u;
          if (k < 0) break;
          if (k < n - 1) s = lam * (s + xn);  // xn = x_{k+1}
          xn = xv[u];
          if (MODE & DOT) {
            a = fma(pv[u], s, a);
            continue;
          }
          const long long o = at(k);
          const double kx = rv[u] + s;
          if (MODE & UPD) {
            const double out = gv[u] / kx;
            if (MODE & CHECK) acc += fabs(ov[u] * kx - gv[u]);
            bad |= !isfinite(out);
            y[o] = out;
          } else {
            y[o] = kx;
          }
        }
      }
      if (MODE & DOT) acc += a;
    } else {
      // weighted: P'_1 = 0, P'_{k+1} = lam (P'_k + p_k); Q'_n = 0, Q'_k = lam (Q'_{k+1} + t_{k+1})
      double p = x[at(0)], P = 0.0;
      double a = 0.0;
      if (!(MODE & DOT)) y[at(0)] = 0.0;
      for (int k = 1; k < n; ++k) {
        P = lam * (P + p);
        p = fma(lam, p, x[at(k)]);
        if (MODE & DOT) a = fma(phi[at(k)], P, a);
        else y[at(k)] = P;
      }
      double t = x[at(n - 1)], Q = 0.0;
      if (!(MODE & DOT)) y[at(n - 1)] *= h;
      for (int k = n - 2; k >= 0; --k) {
        Q = lam * (Q + t);
        t = fma(lam, t, x[at(k)]);
        if (MODE & DOT) a = fma(phi[at(k)], Q, a);
        else y[at(k)] = h * (y[at(k)] + Q);
      }
      if (MODE & DOT) acc = fma(h, a, acc);
    }
  }
}

// ---- 2D problems whose intermediate fits shared memory (n m <= SMEM_NM): the axis-1
// result T lives in shared memory (columns padded to n + 1 doubles: the column pass's
// threads hit distinct banks) and the axis-2 pass stages its forward values there too,
// so both sweeps run at shared-memory latency; only x, the targets and y touch global
// memory (loads issued 8 deep ahead).
constexpr int SMEM_NM = 13600;  // (n + 1) m + n m doubles <= 227 KB

// axis 1: T[j (n+1) + i] = (K1 x[:, j])_i, thread per column j (x from global memory,
// loads issued 8 deep; copying x into shared memory first measured slower)
__device__ __forceinline__ void col_pass_s(const double* __restrict__ x, double* T, int n, int m, double lam) {
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const double* xc = x + (size_t)j * n;
    double* tc = T + (size_t)j * (n + 1);
    double r = 0.0;
    for (int k0 = 0; k0 < n; k0 += U8) {
      double xv[U8];
#pragma unroll
      for (int u = 0; u < U8; ++u) xv[u] = (k0 + u < n) ? xc[k0 + u] : 0.0;
#pragma unroll
      for (int u = 0; u < U8; ++u)
        if (k0 + u < n) {
          r = (k0 + u == 0) ? xv[u] : fma(lam, r, xv[u]);
          tc[k0 + u] = r;
        }
    }
    double s = 0.0, xn = 0.0;
    for (int k1 = n - 1; k1 >= 0; k1 -= U8) {
      double xv[U8];
#pragma unroll
      for (int u = 0; u < U8; ++u) xv[u] = (k1 - u >= 0) ? xc[k1 - u] : 0.0;
#pragma unroll
      for (int u = 0; u < U8; ++u) {
        const int k = k1 - u;
        if (k < 0) break;
        if (k < n - 1) s = lam * (s + xn);
        xn = xv[u];
        tc[k] += s;
      }
    }
  }
}

// axis 2 fused with the update: y[:, ] = tgt / (K2 T[i, :]) per row i (thread per row);
// forward values staged in Rs[j n + i]; CHECK: acc += |yold k - tgt|
template <bool CHECK>
__device__ __forceinline__ void row_pass_s(const double* T, double* Rs, const double* __restrict__ tgt,
                                           const double* __restrict__ yold, double* __restrict__ y, int n, int m,
                                           double lam, double& acc, int& bad) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double r = 0.0;
    for (int j = 0; j < m; ++j) {
      const double t = T[(size_t)j * (n + 1) + i];
      r = (j == 0) ? t : fma(lam, r, t);
      Rs[(size_t)j * n + i] = r;
    }
    double s = 0.0;
    for (int j1 = m - 1; j1 >= 0; j1 -= U8) {
      double gv[U8], ov[U8];
#pragma unroll
      for (int u = 0; u < U8; ++u) {
        const int j = j1 - u;
        const size_t o = (size_t)(j >= 0 ? j : 0) * n + i;
        gv[u] = j >= 0 ? tgt[o] : 0.0;
        ov[u] = (CHECK && j >= 0) ? yold[o] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U8; ++u) {
        const int j = j1 - u;
        if (j < 0) break;
        const size_t o = (size_t)j * n + i;
        if (j < m - 1) s = lam * (s + T[(size_t)(j + 1) * (n + 1) + i]);
        const double kx = Rs[o] + s;
        const double out = gv[u] / kx;
        if (CHECK) acc += fabs(ov[u] * kx - gv[u]);
        bad |= !isfinite(out);
        y[o] = out;
      }
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

// K x over all axes into dst (the last axis with MODE: UPD / CHECK write y, STORE
// writes dst); the intermediate passes ping-pong through T1 / T2.
template <int MODE>
__device__ __forceinline__ void apply_all(const Geo& g, int nax, const Sep2d64Params& P, const double* x,
                                          double* dst, const double* tgt, const double* yold, double* T1,
                                          double* T2, double& acc, int& bad) {
  const double lam[3] = {P.lam1, P.lam2, P.lam3};
  const double* src = x;
  double* bufs[2] = {T1, T2};
  for (int ax = 0; ax < nax - 1; ++ax) {
    double* o = bufs[ax & 1];
    line_pass<false, STORE>(g, ax, src, o, nullptr, nullptr, nullptr, lam[ax], 0.0, acc, bad);
    __syncthreads();
    src = o;
  }
  line_pass<false, MODE>(g, nax - 1, src, dst, tgt, yold, nullptr, lam[nax - 1], 0.0, acc, bad);
}

// return line: sum over axes w of phi . (K .. W_w .. K) psi
__device__ __forceinline__ double cost_all(const Geo& g, int nax, const Sep2d64Params& P, const double* phi,
                                           const double* psi, double* T1, double* T2, double* red) {
  const double lam[3] = {P.lam1, P.lam2, P.lam3}, hh[3] = {P.h1, P.h2, P.h3};
  double acc = 0.0;
  int bad = 0;
  double* bufs[2] = {T1, T2};
  for (int w = 0; w < nax; ++w) {
    const double* src = psi;
    for (int ax = 0; ax < nax - 1; ++ax) {
      double* o = bufs[ax & 1];
      if (ax == w) line_pass<true, STORE>(g, ax, src, o, nullptr, nullptr, nullptr, lam[ax], hh[ax], acc, bad);
      else line_pass<false, STORE>(g, ax, src, o, nullptr, nullptr, nullptr, lam[ax], hh[ax], acc, bad);
      __syncthreads();
      src = o;
    }
    const int ax = nax - 1;
    if (ax == w) line_pass<true, DOT>(g, ax, src, nullptr, nullptr, nullptr, phi, lam[ax], hh[ax], acc, bad);
    else line_pass<false, DOT>(g, ax, src, nullptr, nullptr, nullptr, phi, lam[ax], hh[ax], acc, bad);
    __syncthreads();
  }
  return block_sum(acc, red);
}

__global__ void __launch_bounds__(512) fs1_sep2d64_kernel(const __grid_constant__ Sep2d64Params P) {
  __shared__ double red[32];
  const Geo g{P.n, P.m, P.l};
  const int nax = P.l > 1 ? 3 : 2;
  const size_t nm = (size_t)P.n * P.m * P.l;
  const long long pb = blockIdx.x;
  double* T1 = P.ws + (size_t)pb * 3 * nm;
  double* T2 = T1 + nm;
  double* Y = T2 + nm;
  const double* a = P.a + pb * nm;
  const double* b = P.b + pb * nm;
  double* U = P.u + pb * nm;
  double* V = P.v + pb * nm;
  int bad = 0;
  double dummy = 0.0;
  if (P.mode == 2) {  // apply: y = K x
    apply_all<STORE>(g, nax, P, P.x + pb * nm, P.y + pb * nm, nullptr, nullptr, T1, T2, dummy, bad);
    return;
  }
  if (P.mode == 0) {
    // line 1: phi = psi = 1/(N M L), or the caller's warm start
    if (!P.warm) {
      const double init = 1.0 / (double)nm;
      for (size_t k = threadIdx.x; k < nm; k += blockDim.x) {
        U[k] = init;
        V[k] = init;
      }
    }
    __syncthreads();
    const bool use_tol = P.tol > 0.0;
    int it = 0, flag = 0;
    double errv = NAN;
    extern __shared__ double sst[];
    const bool staged = nax == 2 && P.staged;
    double* sT = sst;                                      // [(n + 1) m]
    double* sR = sst + (size_t)(P.n + 1) * P.m;             // [n m]: the axis-2 staging
    while (true) {
      const bool check = (it >= P.itr_max) || (use_tol && (it % P.check_interval) == 0);
      bad = 0;
      if (staged) {
        // lines 2-7 and 8-12 with the intermediate in shared memory
        col_pass_s(U, sT, P.n, P.m, P.lam1);
        __syncthreads();
        if (check) {
          double e = 0.0;
          row_pass_s<true>(sT, sR, b, V, Y, P.n, P.m, P.lam2, e, bad);
          errv = block_sum(e, red);
          if (it >= P.itr_max || errv <= P.tol) {
            flag = (use_tol && errv <= P.tol) ? FLAG_CONVERGED : FLAG_ITR_MAX;
            break;
          }
          for (size_t k = threadIdx.x; k < nm; k += blockDim.x) V[k] = Y[k];
        } else {
          double e = 0.0;
          row_pass_s<false>(sT, sR, b, nullptr, V, P.n, P.m, P.lam2, e, bad);
        }
        __syncthreads();
        col_pass_s(V, sT, P.n, P.m, P.lam1);
        __syncthreads();
        {
          double e = 0.0;
          row_pass_s<false>(sT, sR, a, nullptr, U, P.n, P.m, P.lam2, e, bad);
        }
        ++it;
        if (__syncthreads_or(bad)) {
          flag = FLAG_NONFINITE;
          errv = NAN;
          break;
        }
        continue;
      }
      // lines 2-7: psi = b ./ (K phi)  (K symmetric: K^T phi = K phi)
      if (check) {
        double e = 0.0;
        apply_all<UPD | CHECK>(g, nax, P, U, Y, b, V, T1, T2, e, bad);
        errv = block_sum(e, red);
        if (it >= P.itr_max || errv <= P.tol) {
          flag = (use_tol && errv <= P.tol) ? FLAG_CONVERGED : FLAG_ITR_MAX;
          break;
        }
        for (size_t k = threadIdx.x; k < nm; k += blockDim.x) V[k] = Y[k];
      } else {
        apply_all<UPD>(g, nax, P, U, V, b, nullptr, T1, T2, dummy, bad);
      }
      __syncthreads();
      // lines 8-12: phi = a ./ (K psi)
      apply_all<UPD>(g, nax, P, V, U, a, nullptr, T1, T2, dummy, bad);
      ++it;  // line 13
      if (__syncthreads_or(bad)) {
        flag = FLAG_NONFINITE;
        errv = NAN;
        break;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (P.iters) P.iters[pb] = it;
      if (P.err) P.err[pb] = errv;
      if (P.flags) P.flags[pb] = flag;
    }
    if (flag == FLAG_NONFINITE) {
      if (threadIdx.x == 0 && P.cost) P.cost[pb] = NAN;
      return;
    }
  }
  if (!P.cost) return;
  const double cost = cost_all(g, nax, P, U, V, T1, T2, red);
  if (threadIdx.x == 0) P.cost[pb] = cost;
}

// ---------------------------------------------------------------------------------
// K5w: the same 2D solve with G LANES per line (G = 1 .. 32, 32 / G lines per warp): lane
// q of a segment owns the E contiguous points [q E, q E + E) of a line of up to G E,
// and the line apply is a chunked scan (lane Horner aggregates, a log2(G)-level segment
// scan of the affine maps y -> lambda^L y + c, both recursions from the exact carries)
// instead of one thread walking the whole line (G = 1: exactly that).  The scan
// multipliers lambda^{E 2^k} are formed on the host as two factors (each >= sqrt of
// the power) so that an underflow of the power alone cannot zero a carry that is still
// representable (Remark 3.3; lambda = e^{-100} at E3).

template <int G, int E>
__device__ __forceinline__ void seg_line_apply(const double (&x)[E], double (&y)[E], double lam,
                                               const double* lvA, const double* lvB, int q) {
  double f = 0.0, g = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) f = fma(lam, f, x[e]);           // forward value at the chunk end
#pragma unroll
  for (int e = E - 1; e >= 0; --e) g = fma(lam, g, x[e]);      // backward value at the chunk start
  double cf = 0.0, cb = 0.0;
  if constexpr (G > 1) {
#pragma unroll
    for (int k = 0; (1 << k) < G; ++k) {
      const int d = 1 << k;
      const double up = __shfl_up_sync(FULL, f, d, G), dn = __shfl_down_sync(FULL, g, d, G);
      if (q >= d) f = fma(up * lvA[k], lvB[k], f);
      if (q + d < G) g = fma(dn * lvA[k], lvB[k], g);
    }
    cf = __shfl_up_sync(FULL, f, 1, G);
    cb = __shfl_down_sync(FULL, g, 1, G);
    if (q == 0) cf = 0.0;
    if (q == G - 1) cb = 0.0;
  }
  // forward recursion r_k = lam r_{k-1} + x_k from the exact carry
  double p = cf;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    p = fma(lam, p, x[e]);
    y[e] = p;
  }
  // backward: t_k = x_k + lam t_{k+1} (inclusive), K x = r_k + lam t_{k+1}
  double t = cb;
#pragma unroll
  for (int e = E - 1; e >= 0; --e) {
    const double kx = fma(lam, t, y[e]);
    t = fma(lam, t, x[e]);
    y[e] = kx;
  }
}

// Internal layouts of K5w (workspace): every line padded to a multiple of lcm(E, 4)
// doubles, so that a lane's E points are aligned 16 / 32-byte vectors inside the line
// and rows start 32-byte aligned.  Row layout: [i ldm + j] (axis 2 contiguous); column
// layout: [j ldn + i] (axis 1 contiguous, the layout of the interface's u, v, a, b).
__host__ __device__ constexpr int w_padw(int E) { return E % 4 == 0 ? E : (E % 2 == 0 ? 2 * E : 4 * E); }
__host__ __device__ inline int w_ld(int len, int E) { return (len + w_padw(E) - 1) / w_padw(E) * w_padw(E); }
// shared-memory stage of one round of transposed line results: RL lines x SP points,
// SP = ld + 2 or + 4 (>= a whole chunk row; even: 16-byte aligned rows; = 2 mod 4: the
// column-wise readout of consecutive rows spreads over the banks)
__host__ __device__ inline int w_sp(int L, int E) {
  const int ld = w_ld(L, E);
  return ld % 4 == 0 ? ld + 2 : ld + 4;
}

// lane's chunk (E doubles from `line`; all inside the padded line).  The pads of
// every internal line hold zeros (written once, never overwritten), so nothing masks
// the chunk and nothing waits on the load until the recursion consumes it.
template <int E>
__device__ __forceinline__ void vload(double (&x)[E], const double* __restrict__ p, bool valid) {
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = 0.0;
  if (valid) {
    if constexpr (E % 4 == 0) {
#pragma unroll
      for (int q = 0; q < E / 4; ++q)
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                     : "=d"(x[4 * q]), "=d"(x[4 * q + 1]), "=d"(x[4 * q + 2]), "=d"(x[4 * q + 3])
                     : "l"(p + 4 * q));
    } else {
#pragma unroll
      for (int q = 0; q < E / 2; ++q)
        asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(x[2 * q]), "=d"(x[2 * q + 1]) : "l"(p + 2 * q));
    }
  }
}

template <int E>
__device__ __forceinline__ void vstore(double* __restrict__ p, const double (&x)[E]) {
  if constexpr (E % 4 == 0) {
#pragma unroll
    for (int q = 0; q < E / 4; ++q)
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * q), "d"(x[4 * q]), "d"(x[4 * q + 1]),
                   "d"(x[4 * q + 2]), "d"(x[4 * q + 3])
                   : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < E / 2; ++q)
      asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p + 2 * q), "d"(x[2 * q]), "d"(x[2 * q + 1]) : "memory");
  }
}

// line 7 / 12: t / k as a reciprocal estimate, one Newton step and a residual correction
// (< 1 ulp).  The IEEE '/' takes its slow path whenever any lane's operands leave a
// narrow exponent window, which E3's potentials (2^-925 .. 2^908 at 160^2) do in every
// warp; it remains for denominators outside 2^-1000 .. 2^1000 (and zero / non-finite
// ones), where the estimate's flush to zero would differ.
__device__ __forceinline__ double upd_div(double t, double k) {
  const double ak = fabs(k);
  return (ak > 0x1p-1000 && ak < 0x1p1000) ? Tr<double>::div<true>(t, k) : t / k;
}

// One half of Algorithm 2 on the `count` lines (length len, padded ld) of one axis,
// fused with the first axis of the next half (K = K1 (x) K2 is separable and the two
// axes commute):
//   kz         = K_this z    (the lambda-recursions of line r of Tin, which already
//                             holds K_other of the other potential),
//   y_new      = tgt / kz                               (line 7 / line 12),
//   Tout       = K_this y_new, transposed                (the next half's first axis),
//   MODE CHECK: acc += |y_old kz - tgt|                  (line 2's marginal error).
// MODE PRO (prologue): Tout = K_this Tin, transposed, nothing else.  y_new is stored
// only when `store` (the state is needed: before a check, see the kernel).
// Lines go in rounds of RL = NW 32 / G (one per segment); a round's Tout lines are
// staged in shared memory and written out column-wise by the whole CTA (RL consecutive
// doubles per point: coalesced), one barrier per round with the stage double-buffered.
// The next line's Tin loads are in flight while this one is scanned.
constexpr int W_PRO = 0, W_UPD = 1, W_CHECK = 2;

template <int G, int E, int MODE>
__device__ __forceinline__ void half_pass(const double* __restrict__ Tin, const double* __restrict__ tgt,
                                          const double* __restrict__ yold, double* __restrict__ ynew, bool store,
                                          double* __restrict__ Tout, int len, int ld, int count, int ldo,
                                          double lam, const double* lvA, const double* lvB, double* stage, int sp,
                                          int seg, int q, int nw, double& acc, int& bad) {
  const int RL = nw * (32 / G);
  const int k0 = q * E;               // this lane's first point on its line
  const bool chunk = k0 < ld;         // the chunk lies inside the padded line
  double v[E];
  if (MODE != W_CHECK) vload<E>(v, Tin + (size_t)seg * ld + k0, chunk && seg < count);
  int buf = 0;
  for (int r0 = 0; r0 < count; r0 += RL, buf ^= 1) {
    const int r = r0 + seg;
    const bool live = r < count;
    double* st = stage + (size_t)buf * RL * sp;
    const size_t base = (size_t)r * ld + k0;
    double nv[E], kz[E];
    double tg[E];
    if (MODE != W_PRO) vload<E>(tg, tgt + base, chunk && live);
    // (check passes, rare, load their lines one at a time: the old psi takes the
    // registers of the prefetch)
    if (MODE == W_CHECK) vload<E>(v, Tin + base, chunk && live);
    else vload<E>(nv, Tin + base + (size_t)RL * ld, chunk && r + RL < count);
    seg_line_apply<G, E>(v, kz, lam, lvA, lvB, q);
    if (MODE != W_PRO) {
      if (MODE == W_CHECK) {
        double yo[E];
        vload<E>(yo, yold + base, chunk && live);
#pragma unroll
        for (int e = 0; e < E; ++e) acc += fabs(yo[e] * kz[e] - tg[e]);  // pads, dead lines: 0 kz - 0
      }
      // line 7 / 12 (upd_div) with the range test hoisted: one warp-uniform branch per
      // line; pads and dead lines divide 0 / 1.  Non-finite test on sum(out) / 16
      // (positive terms: any inf or NaN survives, finite ones cannot overflow)
      bool inr = true;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (!live || k0 + e >= len) kz[e] = 1.0;
        const double ak = fabs(kz[e]);
        inr &= ak > 0x1p-1000 && ak < 0x1p1000;
      }
      if (__all_sync(FULL, inr)) {
#pragma unroll
        for (int e = 0; e < E; ++e) tg[e] = Tr<double>::div<true>(tg[e], kz[e]);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) tg[e] = upd_div(tg[e], kz[e]);
      }
      double chk = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) chk = fma(tg[e], 0.0625, chk);
      bad |= !isfinite(chk);
      if (store && chunk && live) vstore<E>(ynew + base, tg);
      seg_line_apply<G, E>(tg, kz, lam, lvA, lvB, q);
    }
    // stage row `seg`: this line's Tout values, lane chunk as 16-byte vectors
    if (live && k0 < len) {
      double2* srow = reinterpret_cast<double2*>(st + (size_t)seg * sp + k0);
#pragma unroll
      for (int h = 0; h < E / 2; ++h) srow[h] = make_double2(kz[2 * h], kz[2 * h + 1]);
    }
    if (MODE != W_CHECK) {
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = nv[e];
    }
    __syncthreads();
    // write-out: Tout[k ldo + r0 + w] = stage[w][k], nr <= RL consecutive doubles per
    // point k, four per thread as one 32-byte store (ldo and r0 are multiples of 4);
    // thread t takes (k, group) = divmod(t, NQ), then steps by the block size
    const int nr = count - r0 < RL ? count - r0 : RL;
    const int NQ = (nr + 3) >> 2, T = nw * 32;
    const int dk = T / NQ, dg = T - dk * NQ;
    int k = threadIdx.x / NQ, g = threadIdx.x - k * NQ;
    for (; k < len;) {
      const int w = 4 * g;
      const double* sc = st + (size_t)w * sp + k;
      double* o = Tout + (size_t)k * ldo + r0 + w;
      if (w + 4 <= nr) {
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(o), "d"(sc[0]), "d"(sc[sp]), "d"(sc[2 * sp]),
                     "d"(sc[3 * sp])
                     : "memory");
      } else {
        for (int h = 0; w + h < nr; ++h) o[h] = sc[(size_t)h * sp];
      }
      k += dk;
      g += dg;
      if (g >= NQ) {
        g -= NQ;
        ++k;
      }
    }
  }
}

// 2D fp64 solve, one CTA per problem (K5w).  The loop keeps only the two intermediates
// (TR, TC) and the targets live; phi and psi are stored only on the iterations whose
// state a check can return (the iteration before every check, i.e. before
// l = itr_max and, with tol > 0, before every check_interval-th one).  A problem that
// turns non-finite replays from the last stored state with every iteration stored, so
// it too returns the state at which it stopped (fs1.h).
template <int G, int E, int NT>
__global__ void __launch_bounds__(NT) fs1_sep2d64w_kernel(const __grid_constant__ Sep2d64Params P) {
  const int NW = blockDim.x >> 5, BT = blockDim.x;  // launched with <= NT threads
  __shared__ double red[32];
  extern __shared__ __align__(16) double stage[];
  const int n = P.n, m = P.m;
  const int ldn = w_ld(n, E), ldm = w_ld(m, E);
  const size_t nm = (size_t)n * m;
  const size_t szR = (size_t)n * ldm, szC = (size_t)m * ldn;
  const long long pb = blockIdx.x;
  // workspace (4 row-layout + 3 column-layout buffers per problem): TR, TC the
  // intermediates; psi in row layout (ping-pong: a check iteration that stops keeps
  // the psi of the last completed iteration); b in row layout; a and phi in column
  // layout (padded copies of the interface's arrays)
  double* TR = P.ws + (size_t)pb * (4 * szR + 3 * szC);
  double* Vc = TR + szR;
  double* Vn = Vc + szR;
  double* bR = Vn + szR;
  double* TC = bR + szR;
  double* aC = TC + szC;
  double* UC = aC + szC;
  const double* a = P.a + pb * nm;
  const double* b = P.b + pb * nm;
  double* U = P.u + pb * nm;
  double* V = P.v + pb * nm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = warp * (32 / G) + lane / G, q = lane % G;  // line slot in a round, lane in the line
  const int sp = w_sp(n > m ? n : m, E);
  {
    // zero the pads (and everything else) of all seven buffers, then fill
    double2* z = reinterpret_cast<double2*>(TR);
    const size_t nz = (4 * szR + 3 * szC) / 2;
    for (size_t k = threadIdx.x; k < nz; k += BT) z[k] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double init = 1.0 / (double)nm;
  for (size_t k = threadIdx.x; k < nm; k += BT) {
    const size_t j = k / n, i = k - j * n;  // interface index k = j n + i
    UC[j * ldn + i] = P.warm ? U[k] : init;
    aC[j * ldn + i] = a[k];
    Vc[i * ldm + j] = P.warm ? V[k] : init;
    bR[i * ldm + j] = b[k];
  }
  __syncthreads();
  const bool use_tol = P.tol > 0.0;
  auto is_check = [&](int l) { return l >= P.itr_max || (use_tol && (l % P.check_interval) == 0); };
  int it = 0, flag = 0, last = 0, bad = 0;
  bool store_all = false;
  double errv = NAN;
  bool prologue = true;
  while (true) {
    if (prologue) {
      // TR = K1 phi (axis 1 on the columns of phi, stored transposed)
      double e0 = 0.0;
      half_pass<G, E, W_PRO>(UC, nullptr, nullptr, nullptr, false, TR, n, ldn, m, ldm, P.lam1, P.wA1, P.wB1,
                                 stage, sp, seg, q, NW, e0, bad);
      __syncthreads();
      prologue = false;
    }
    const bool check = is_check(it);
    const bool store = store_all || is_check(it + 1);
    bad = 0;
    // lines 2-7 on the rows: psi = b / K2 TR, TC = K2 psi
    if (check) {
      double e = 0.0;
      half_pass<G, E, W_CHECK>(TR, bR, Vc, Vn, store, TC, m, ldm, n, ldn, P.lam2, P.wA2, P.wB2, stage, sp,
                                   seg, q, NW, e, bad);
      errv = block_sum(e, red);
      if (it >= P.itr_max || errv <= P.tol) {
        flag = (use_tol && errv <= P.tol) ? FLAG_CONVERGED : FLAG_ITR_MAX;
        break;  // phi, psi in UC, Vc: the state of the last completed iteration
      }
    } else {
      double e = 0.0;
      half_pass<G, E, W_UPD>(TR, bR, nullptr, Vn, store, TC, m, ldm, n, ldn, P.lam2, P.wA2, P.wB2, stage, sp,
                                 seg, q, NW, e, bad);
    }
    if (store) {
      double* t = Vc;
      Vc = Vn;
      Vn = t;
    }
    __syncthreads();
    // lines 8-12 on the columns: phi = a / K1 TC, TR = K1 phi
    {
      double e = 0.0;
      half_pass<G, E, W_UPD>(TC, aC, nullptr, UC, store, TR, n, ldn, m, ldm, P.lam1, P.wA1, P.wB1, stage, sp,
                                 seg, q, NW, e, bad);
    }
    ++it;  // line 13
    if (__syncthreads_or(bad)) {
      if (!store_all) {
        // replay from the stored state of iteration `last`, storing every iteration
        store_all = true;
        it = last;
        prologue = true;
        continue;
      }
      flag = FLAG_NONFINITE;
      errv = NAN;
      break;
    }
    if (store) last = it;
  }
  __syncthreads();
  // phi and psi back to the interface layout
  for (size_t k = threadIdx.x; k < nm; k += BT) {
    const size_t j = k / n, i = k - j * n;
    U[k] = UC[j * ldn + i];
    V[k] = Vc[i * ldm + j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (P.iters) P.iters[pb] = it;
    if (P.err) P.err[pb] = errv;
    if (P.flags) P.flags[pb] = flag;
  }
  if (flag == FLAG_NONFINITE) {
    if (threadIdx.x == 0 && P.cost) P.cost[pb] = NAN;
    return;
  }
  if (!P.cost) return;
  const Geo g{P.n, P.m, 1};
  const double cost = cost_all(g, 2, P, U, V, TR, TC, red);
  if (threadIdx.x == 0) P.cost[pb] = cost;
}

// the instantiated (G, E) pairs; a plan picks the cheapest that covers max(n, m)
// (NT: the launch bound, the most threads a plan may launch: 384 keeps E = 10 free of
// spills)
struct WVar {
  int G, E, NT;
};
constexpr WVar W_VARS[] = {{1, 10, 384}, {2, 10, 384}, {4, 10, 384}, {8, 10, 384}, {16, 10, 384}, {32, 8, 512}};

}  // namespace s64

// K5w variant for a 2D problem: 1 + the index into W_VARS of the pair (G lanes per line,
// E points per lane) with G E >= max(n, m) and the fewest instructions per line under
// the count model (6 E + 12 log2 G + 20) G / 32 (a Horner / recursion step per point,
// a scan level per doubling of G, spread over the 32 / G lines a warp carries); 0: no
// variant covers the problem.
int sep2d64w_chunk(long long n, long long m) {
  const long long L = n > m ? n : m;
  int best = 0;
  double bc = 0.0;
  for (int i = 0; i < (int)(sizeof(s64::W_VARS) / sizeof(s64::W_VARS[0])); ++i) {
    const int G = s64::W_VARS[i].G, E = s64::W_VARS[i].E;
    if ((long long)G * E < L) continue;
    int lg = 0;
    while ((1 << lg) < G) ++lg;
    const double c = (6.0 * E + 12.0 * lg + 20.0) * G / 32.0;
    if (!best || c < bc) {
      best = i + 1;
      bc = c;
    }
  }
  return best;
}

void sep2d64w_geom(int var, int* G, int* E) {
  *G = s64::W_VARS[var - 1].G;
  *E = s64::W_VARS[var - 1].E;
}

size_t sep2d64w_workspace(long long n, long long m, int var) {
  const int E = s64::W_VARS[var - 1].E;
  const size_t ldn = (size_t)s64::w_ld((int)n, E), ldm = (size_t)s64::w_ld((int)m, E);
  return (4 * (size_t)n * ldm + 3 * (size_t)m * ldn) * sizeof(double);
}

// threads for a K5w launch: the fewest warps (>= 4) that reach the smallest number of
// rounds (RL = warps x 32 / G lines per round) over the two half-passes
int sep2d64w_threads(long long n, long long m, int var) {
  const int G = s64::W_VARS[var - 1].G, maxw = s64::W_VARS[var - 1].NT / 32;
  auto rounds = [&](int nw) {
    const long long RL = (long long)nw * (32 / G);
    return (n + RL - 1) / RL + (m + RL - 1) / RL;
  };
  const long long best = rounds(maxw);
  int nw = 4 < maxw ? 4 : maxw;
  while (nw < maxw && rounds(nw) > best) ++nw;
  return nw * 32;
}

size_t sep2d64w_smem(long long n, long long m, int var, int threads) {
  const int G = s64::W_VARS[var - 1].G, E = s64::W_VARS[var - 1].E;
  const int RL = threads / 32 * (32 / G);
  return (size_t)2 * RL * s64::w_sp((int)(n > m ? n : m), E) * sizeof(double);
}

#define FS1_W_KERNEL(i) s64::fs1_sep2d64w_kernel<s64::W_VARS[i].G, s64::W_VARS[i].E, s64::W_VARS[i].NT>

const void* sep2d64w_fn(int var) {
  switch (var) {
    case 1: return (const void*)&FS1_W_KERNEL(0);
    case 2: return (const void*)&FS1_W_KERNEL(1);
    case 3: return (const void*)&FS1_W_KERNEL(2);
    case 4: return (const void*)&FS1_W_KERNEL(3);
    case 5: return (const void*)&FS1_W_KERNEL(4);
    case 6: return (const void*)&FS1_W_KERNEL(5);
    default: return nullptr;
  }
}

cudaError_t launch_sep2d64w(const Sep2d64Params& P, long long batch, int var, int threads, cudaStream_t st) {
  const size_t smem = sep2d64w_smem(P.n, P.m, var, threads);
  const dim3 grid((unsigned)batch), block(threads);
  switch (var) {
    case 1: FS1_W_KERNEL(0)<<<grid, block, smem, st>>>(P); break;
    case 2: FS1_W_KERNEL(1)<<<grid, block, smem, st>>>(P); break;
    case 3: FS1_W_KERNEL(2)<<<grid, block, smem, st>>>(P); break;
    case 4: FS1_W_KERNEL(3)<<<grid, block, smem, st>>>(P); break;
    case 5: FS1_W_KERNEL(4)<<<grid, block, smem, st>>>(P); break;
    case 6: FS1_W_KERNEL(5)<<<grid, block, smem, st>>>(P); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

size_t sep2d64_smem(long long n, long long m, int ndim) {
  if (ndim != 2 || (n + 1) * m > s64::SMEM_NM) return 0;
  return (size_t)((n + 1) * m + n * m) * sizeof(double);
}

const void* sep2d64_fn() { return (const void*)&s64::fs1_sep2d64_kernel; }

cudaError_t launch_sep2d64(const Sep2d64Params& P, long long batch, int threads, cudaStream_t st) {
  const size_t smem = P.staged ? sep2d64_smem(P.n, P.m, P.l > 1 ? 3 : 2) : 0;
  s64::fs1_sep2d64_kernel<<<(unsigned)batch, threads, smem, st>>>(P);
  return cudaGetLastError();
}

}  // namespace fs1
