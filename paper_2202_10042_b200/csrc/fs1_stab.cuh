// fs1_stab.cuh — K4: the paper's own log-domain-stabilised FS-1 (Remark 2.1 +
// Remark 3.2) for batches of 1D problems, fp64,
// one CTA per problem for the whole solve.
//
// State per problem: the absorbed potentials A = alpha/eps, B = beta/eps and the
// scalings phi, psi, so that gamma = diag(e^A phi) K diag(e^B psi).  Between
// absorptions the rescaled kernel K~ = diag(e^A) K diag(e^B) is applied by the
// variable-coefficient recursions of Remark 3.2 (read with alpha <- alpha + eps ln
// phi, R8; own = B on the psi side, A on the phi side):
//
//   r_k = f_k r_{k-1} + w_k x_k,          f_k = lambda e^{own_k - own_{k-1}}     (line 5 / 10)
//   u_k = g_k u_{k+1} + w_k x_k,          g_k = lambda e^{own_k - own_{k+1}}
//   (K~ x)_k = r_k + g_k u_{k+1}          (s_k = g_k u_{k+1}: line 6 / 11)
//   w_k = e^{A_k + B_k}
//
// Multiply-only between absorptions: the coefficient arrays f, g (per side) and w
// are formed once per absorption (exp of neighbour differences, as printed) and
// kept in the workspace (L2-resident), the state in shared memory.  On the GPU
// each recursion is a chunked scan of affine maps y -> M y + C: per-thread chunk
// aggregates (M a product of E coefficients), a warp shuffle scan and a cross-warp
// fold in extended range (so a product of many coefficients never over/underflows
// on its own: Remark 3.3's concern), then both recursions from the exact carries
// fused with the update y = target / (K~ x) and the marginal error.  Absorption
// (Remark 2.1): after a full iteration, if max(|phi|_inf, |psi|_inf) > tau, then
// A += ln phi, B += ln psi, phi = psi = 1 and the coefficients are re-formed.
// The return line is the Jordan-block pair scan
//   (p, P)_k = (f_k p_{k-1} + w_k psi_k, f_k (P_{k-1} + p_{k-1})),
//   (u, Q)_k = (g_k u_{k+1} + w_k psi_k, g_k (Q_{k+1} + u_{k+1}))      (own = A)
// with cost = h sum_k phi_k (P_k + Q_k) = sum_ij phi_i K~_ij psi_j |i-j| h.
//
// Layout: thread t owns points k = t E + e (e < E); every per-point array (shared
// and workspace) is stored [e][t] (index e T + t) so warp accesses coalesce.
#pragma once
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"
#include "fs1_params.h"

namespace fs1 {
namespace stab {

// unroll depth of the three half-step passes (the loads of the coefficient arrays go to
// L2: deeper unrolling keeps more of them in flight)
#ifndef FS1_STAB_UNROLL
#define FS1_STAB_UNROLL 16
#endif
#define FS1_STAB_STR2(x) #x
#define FS1_STAB_STR(x) FS1_STAB_STR2(unroll x)
#define FS1_STAB_UNROLL_STR FS1_STAB_STR(FS1_STAB_UNROLL)

enum { WA = 0, WB, WW, WFA, WGA, WFB, WGB, WTA, WTB, WN };  // workspace arrays per problem
constexpr int FS1F_CONVERGED = 1, FS1F_NONFINITE = 2, FS1F_ITR_MAX = 4;

// The workspace arrays are written and read by the same CTA only: plain (L1-coherent
// for the CTA) loads, never the non-coherent or L1-bypassing paths.
__device__ __forceinline__ double ld_(const double* p) { return *p; }

// line 7 / 12's quotient: a reciprocal estimate with one Newton step and a residual
// correction (< 1 ulp) where the denominator lies in 2^-1000 .. 2^1000, the IEEE '/'
// otherwise (zero, non-finite or extreme denominators keep its exact semantics)
#ifndef FS1_STAB_NDIV
#define FS1_STAB_NDIV 1
#endif
__device__ __forceinline__ double sdiv(double t, double k) {
  if (!FS1_STAB_NDIV) return t / k;
  const double ak = fabs(k);
  return (ak > 0x1p-1000 && ak < 0x1p1000) ? Tr<double>::div<true>(t, k) : t / k;
}

// an extended-range value as a double (overflow -> inf, underflow -> 0)
__device__ __forceinline__ double er_val(ER<double> x) {
  return x.e > 1023 ? INFINITY : er_rel(x, 0);
}

__device__ __forceinline__ ER<double> er1() { return ER<double>{1.0, 0}; }
__device__ __forceinline__ ER<double> erd(double x) { return er_norm<double>(x, 0); }  // x >= 0
__device__ __forceinline__ ER<double> erfma(ER<double> a, ER<double> b, ER<double> c) {
  return er_add(er_mul(a, b), c);
}

// y -> M y + C
struct Aff {
  ER<double> M, C;
};
__device__ __forceinline__ Aff ident(Aff*) { return Aff{er1(), er_zero<double>()}; }
__device__ __forceinline__ Aff compose(Aff L, Aff E) {  // L after E
  return Aff{er_mul(L.M, E.M), erfma(L.M, E.C, L.C)};
}
// branch-free keep-or-replace of a map at a scan level (an `if (lane >= d) x = ...`
// around the extended-range compose compiled to a divergent branch at every level)
__device__ __forceinline__ ER<double> er_sel(bool p, ER<double> a, ER<double> b) {
  return ER<double>{p ? a.m : b.m, p ? a.e : b.e};
}
__device__ __forceinline__ Aff msel(bool p, Aff a, Aff b) { return Aff{er_sel(p, a.M, b.M), er_sel(p, a.C, b.C)}; }
__device__ __forceinline__ Aff shfl_up_m(Aff x, int d) { return Aff{shfl_up_er(x.M, d), shfl_up_er(x.C, d)}; }
__device__ __forceinline__ Aff shfl_down_m(Aff x, int d) { return Aff{shfl_down_er(x.M, d), shfl_down_er(x.C, d)}; }
__device__ __forceinline__ Aff shfl_idx_m(Aff x, int s) { return Aff{shfl_idx_er(x.M, s), shfl_idx_er(x.C, s)}; }

// (p, P) -> (a p + c1, b p + a P + c2): the Jordan-block maps of the cost scan
struct Jor {
  ER<double> a, b, c1, c2;
};
__device__ __forceinline__ Jor ident(Jor*) { return Jor{er1(), er_zero<double>(), er_zero<double>(), er_zero<double>()}; }
__device__ __forceinline__ Jor compose(Jor L, Jor E) {
  return Jor{er_mul(L.a, E.a), er_add(er_mul(L.a, E.b), er_mul(L.b, E.a)), erfma(L.a, E.c1, L.c1),
             er_add(er_add(er_mul(L.b, E.c1), er_mul(L.a, E.c2)), L.c2)};
}
__device__ __forceinline__ Jor msel(bool p, Jor a, Jor b) {
  return Jor{er_sel(p, a.a, b.a), er_sel(p, a.b, b.b), er_sel(p, a.c1, b.c1), er_sel(p, a.c2, b.c2)};
}
__device__ __forceinline__ Jor shfl_up_m(Jor x, int d) {
  return Jor{shfl_up_er(x.a, d), shfl_up_er(x.b, d), shfl_up_er(x.c1, d), shfl_up_er(x.c2, d)};
}
__device__ __forceinline__ Jor shfl_down_m(Jor x, int d) {
  return Jor{shfl_down_er(x.a, d), shfl_down_er(x.b, d), shfl_down_er(x.c1, d), shfl_down_er(x.c2, d)};
}

// Exclusive scan over the CTA's threads of per-thread chunk maps, FWD: the composite
// of the chunks of threads < t (in order), else of threads > t (right to left).
// Deterministic (fixed trees and orders).  `sm` holds W maps; the caller synchronises
// before the next use of sm.
template <class Map, int W, bool FWD>
__device__ __forceinline__ Map block_scan_excl(Map x, Map* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Map y = FWD ? shfl_up_m(x, d) : shfl_down_m(x, d);
    x = msel(FWD ? lane >= d : lane + d < 32, compose(x, y), x);
  }
  if (lane == (FWD ? 31 : 0)) sm[warp] = x;
  __syncthreads();
  Map cw = ident((Map*)nullptr);
  if (FWD) {
    for (int w = 0; w < warp; ++w) cw = compose(sm[w], cw);
  } else {
    for (int w = W - 1; w > warp; --w) cw = compose(sm[w], cw);
  }
  Map ex = FWD ? shfl_up_m(x, 1) : shfl_down_m(x, 1);
  if (lane == (FWD ? 0 : 31)) ex = ident((Map*)nullptr);
  return compose(ex, cw);
}

// Both directions of the half-step's affine-map scan with one block barrier: warp
// inclusive scans (forward up, backward down), the warp totals through shared memory,
// then every warp scans the W totals across its lanes (lane j <-> warp j, shuffle
// levels instead of a serial fold) and takes the composite of the warps before /
// after it.  Returns the exclusive maps of this thread's chunk.  Deterministic.
template <int W>
__device__ __forceinline__ void block_scan2(Aff xf, Aff xb, Aff* sm, Aff& ef, Aff& eb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Aff yf = shfl_up_m(xf, d);
    const Aff yb = shfl_down_m(xb, d);
    xf = msel(lane >= d, compose(xf, yf), xf);
    xb = msel(lane + d < 32, compose(xb, yb), xb);
  }
  if (lane == 31) sm[warp] = xf;
  if (lane == 0) sm[W + warp] = xb;
  __syncthreads();
  // lanes j < W hold warp j's totals; inclusive scans across them
  Aff wf = lane < W ? sm[lane] : ident((Aff*)nullptr);
  Aff wb = lane < W ? sm[W + lane] : ident((Aff*)nullptr);
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    const Aff yf = shfl_up_m(wf, d);
    const Aff yb = shfl_down_m(wb, d);
    wf = msel(lane >= d, compose(wf, yf), wf);
    wb = msel(lane + d < W, compose(wb, yb), wb);
  }
  // composite of the warps before (after) this one: lane warp-1 (warp+1) of the scans
  Aff cwf = shfl_idx_m(wf, warp > 0 ? warp - 1 : 0);
  Aff cwb = shfl_idx_m(wb, warp + 1 < W ? warp + 1 : 0);
  if (warp == 0) cwf = ident((Aff*)nullptr);
  if (warp == W - 1) cwb = ident((Aff*)nullptr);
  Aff xef = shfl_up_m(xf, 1), xeb = shfl_down_m(xb, 1);
  if (lane == 0) xef = ident((Aff*)nullptr);
  if (lane == 31) xeb = ident((Aff*)nullptr);
  ef = compose(xef, cwf);
  eb = compose(xeb, cwb);
}

__device__ __forceinline__ double block_sum(double v, double* red, int W) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < W; ++w) s += red[w];
  return s;
}

__device__ __forceinline__ double block_max(double v, double* red, int W) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < W; ++w) s = fmax(s, red[w]);
  return s;
}

// One half-step y = tgt ./ (K~ x) (lines 3-7 or 8-12 with Remark 3.2's recursions).
// CHECK: also the marginal error sum |y_old (K~ x) - tgt| (line 2); the new y goes to
// R (the caller commits it once the check has not stopped the loop), else to ys.
template <int E, int W, bool CHECK>
__device__ __forceinline__ void half(long long n, const double* xs, double* ys, double* R, const double* wv,
                                     const double* fv, const double* gv, const double* tv, Aff* sm,
                                     double& errp) {
  constexpr int T = 32 * W;
  const int t = threadIdx.x;
  // pass 1: the chunk's forward / backward maps.  The products M of the chunk's E
  // coefficients are formed in plain fp64 (no extended-range step per point) unless one
  // leaves [2^-960, 2^960] — then the chunk recomputes them in extended range, so no
  // product of many coefficients ever under/overflows on its own (Remark 3.3).
  double mf = 1.0, mb = 1.0;
  double Cf = 0.0, Cb = 0.0;
_Pragma(FS1_STAB_UNROLL_STR)
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    const double f = ld_(fv + i), g = ld_(gv + E * T - T - e * T + t);
    const double xf = ld_(wv + i) * xs[i];
    const int j = (E - 1 - e) * T + t;
    Cf = fma(f, Cf, xf);
    Cb = fma(g, Cb, ld_(wv + j) * xs[j]);
    mf *= f;
    mb *= g;
  }
  ER<double> Mf, Mb;
  const double LO = 0x1p-960, HI = 0x1p960;
  if ((mf == 0.0 || (mf >= LO && mf <= HI)) && (mb == 0.0 || (mb >= LO && mb <= HI))) {
    Mf = erd(mf);
    Mb = erd(mb);
  } else {
    Mf = er1();
    Mb = er1();
    for (int e = 0; e < E; ++e) {
      Mf = er_mul(Mf, erd(ld_(fv + e * T + t)));
      Mb = er_mul(Mb, erd(ld_(gv + e * T + t)));
    }
  }
  // carries: r just before this chunk, u just after it (both from zero at the ends)
  Aff cf, cb;
  block_scan2<W>(Aff{Mf, er_norm<double>(fabs(Cf), 0)}, Aff{Mb, er_norm<double>(fabs(Cb), 0)}, sm, cf, cb);
  double r = er_val(cf.C);
  double u = er_val(cb.C);
  // pass 2: the forward recursion r_k
_Pragma(FS1_STAB_UNROLL_STR)
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    r = fma(ld_(fv + i), r, ld_(wv + i) * xs[i]);
    R[i] = r;
  }
  // pass 3: backward recursion fused with the update
_Pragma(FS1_STAB_UNROLL_STR)
  for (int e = E - 1; e >= 0; --e) {
    const int i = e * T + t;
    const long long k = (long long)t * E + e;
    const double g = ld_(gv + i);
    const double su = g * u;            // s_k = g_k u_{k+1}
    const double kx = R[i] + su;        // (K~ x)_k = r_k + s_k
    u = su + ld_(wv + i) * xs[i];    // u_k = s_k + w_k x_k
    const double tg = ld_(tv + i);
    const double y = k < n ? sdiv(tg, kx) : 0.0;
    if (CHECK) {
      if (k < n) errp += fabs(ys[i] * kx - tg);
      R[i] = y;
    } else {
      ys[i] = y;
    }
  }
}

// Re-form the coefficient arrays from A, B (Remark 3.2's factors, as printed):
// w_k = e^{A_k + B_k}; f^A_k = lambda e^{A_k - A_{k-1}} (k >= 1); g^A_k = lambda
// e^{A_k - A_{k+1}} (k <= n-2); the same with B; 0 at the ends and on padding.
template <int E, int W>
__device__ __forceinline__ void form_coeffs(long long n, double lam, double* ws) {
  constexpr int T = 32 * W;
  const long long P = (long long)T * E;
  const int t = threadIdx.x;
  double* A = ws + WA * P;
  double* B = ws + WB * P;
  auto at = [&](long long k) { return (int)((k % E) * T + k / E); };
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    const long long k = (long long)t * E + e;
    double w = 0.0, fa = 0.0, ga = 0.0, fb = 0.0, gb = 0.0;
    if (k < n) {
      const double a = A[i], b = B[i];
      w = exp(a + b);
      if (k >= 1) {
        const int j = at(k - 1);
        fa = lam * exp(a - A[j]);
        fb = lam * exp(b - B[j]);
      }
      if (k + 1 < n) {
        const int j = at(k + 1);
        ga = lam * exp(a - A[j]);
        gb = lam * exp(b - B[j]);
      }
    }
    ws[WW * P + i] = w;
    ws[WFA * P + i] = fa;
    ws[WGA * P + i] = ga;
    ws[WFB * P + i] = fb;
    ws[WGB * P + i] = gb;
  }
}

// Return line on the state (A, B, phi, psi): the pair scans above.
template <int E, int W>
__device__ __forceinline__ double cost_stab(long long n, double h, const double* phi, const double* psi,
                                            const double* ws, Jor* sj, double* red) {
  constexpr int T = 32 * W;
  const long long P = (long long)T * E;
  const int t = threadIdx.x;
  const double* wv = ws + WW * P;
  const double* fv = ws + WFA * P;
  const double* gv = ws + WGA * P;
  // chunk maps: element k maps (p, P) -> (f p + x^, f (P + p)), i.e. a = b = f, c1 = x^
  Jor jf = ident((Jor*)nullptr), jb = ident((Jor*)nullptr);
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    const ER<double> f = erd(ld_(fv + i));
    const ER<double> x = erd(ld_(wv + i) * psi[i]);
    jf = compose(Jor{f, f, x, er_zero<double>()}, jf);
  }
  for (int e = E - 1; e >= 0; --e) {
    const int i = e * T + t;
    const ER<double> g = erd(ld_(gv + i));
    const ER<double> x = erd(ld_(wv + i) * psi[i]);
    jb = compose(Jor{g, g, x, er_zero<double>()}, jb);
  }
  const Jor cf = block_scan_excl<Jor, W, true>(jf, sj);
  __syncthreads();
  const Jor cb = block_scan_excl<Jor, W, false>(jb, sj);
  double p = er_val(cf.c1), Pp = er_val(cf.c2);
  double acc = 0.0;
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    const double f = ld_(fv + i);
    Pp = f * (Pp + p);
    p = fma(f, p, ld_(wv + i) * psi[i]);
    acc = fma(phi[i], Pp, acc);
  }
  double u = er_val(cb.c1), Q = er_val(cb.c2);
  for (int e = E - 1; e >= 0; --e) {
    const int i = e * T + t;
    const double g = ld_(gv + i);
    Q = g * (Q + u);
    u = fma(g, u, ld_(wv + i) * psi[i]);
    acc = fma(phi[i], Q, acc);
  }
  return h * block_sum(acc, red, W);
}

template <int E, int W>
__global__ void __launch_bounds__(32 * W, 1) fs1_stab_solve(const __grid_constant__ StabParams SP) {
  constexpr int T = 32 * W;
  constexpr long long P = (long long)T * E;
  extern __shared__ __align__(16) unsigned char smem[];
  double* phi = reinterpret_cast<double*>(smem);
  double* psi = phi + P;
  double* R = psi + P;
  double* red = R + P;                                   // 32 doubles
  Jor* sj = reinterpret_cast<Jor*>(red + 32);            // W maps (also used as Aff scratch)
  Aff* sm = reinterpret_cast<Aff*>(sj);

  const int t = threadIdx.x;
  const long long pb = blockIdx.x;
  const long long n = SP.n;
  double* ws = SP.ws + pb * (long long)WN * P;
  const double* a = reinterpret_cast<const double*>(SP.a) + pb * n;
  const double* b = reinterpret_cast<const double*>(SP.b) + pb * n;
  double* F = reinterpret_cast<double*>(SP.u) + pb * n;
  double* G = reinterpret_cast<double*>(SP.v) + pb * n;

  if (SP.mode == 1) {
    // the return line alone on a given state (F, G) = (alpha/eps, beta/eps), phi = psi = 1
    for (int e = 0; e < E; ++e) {
      const int i = e * T + t;
      const long long k = (long long)t * E + e;
      const bool ok = k < n;
      ws[WA * P + i] = ok ? F[k] : 0.0;
      ws[WB * P + i] = ok ? G[k] : 0.0;
      phi[i] = ok ? 1.0 : 0.0;
      psi[i] = ok ? 1.0 : 0.0;
    }
    __syncthreads();
    form_coeffs<E, W>(n, SP.lam, ws);
    __syncthreads();
    const double cost = cost_stab<E, W>(n, SP.h, phi, psi, ws, sj, red);
    if (t == 0 && SP.cost) SP.cost[pb] = cost;
    return;
  }
  // line 1: phi = psi = 1/N, alpha = beta = 0; targets (linear weights) to the workspace
  const double init = 1.0 / (double)n;
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    const long long k = (long long)t * E + e;
    const bool ok = k < n;
    double ta = 0.0, tb = 0.0;
    if (ok) {
      ta = SP.input_is_log ? exp(a[k]) : a[k];
      tb = SP.input_is_log ? exp(b[k]) : b[k];
    }
    ws[WTA * P + i] = ta;
    ws[WTB * P + i] = tb;
    ws[WA * P + i] = 0.0;
    ws[WB * P + i] = 0.0;
    phi[i] = ok ? init : 0.0;
    psi[i] = ok ? init : 0.0;
  }
  __syncthreads();
  form_coeffs<E, W>(n, SP.lam, ws);
  __syncthreads();

  const bool use_tol = SP.tol > 0.0;
  int l = 0, flag = 0;
  double errv = NAN;
  while (true) {
    const bool check = (l >= SP.itr_max) || (use_tol && (l % SP.check_interval) == 0);
    // ---- lines 2-7 (own = B): psi = b ./ (K~^T phi)
    if (check) {
      double ep = 0.0;
      half<E, W, true>(n, phi, psi, R, ws + WW * P, ws + WFB * P, ws + WGB * P, ws + WTB * P, sm, ep);
      errv = block_sum(ep, red, W);
      if (l >= SP.itr_max || errv <= SP.tol) {
        flag = (use_tol && errv <= SP.tol) ? FS1F_CONVERGED : FS1F_ITR_MAX;
        break;
      }
      for (int e = 0; e < E; ++e) psi[e * T + t] = R[e * T + t];
    } else {
      double ep = 0.0;
      half<E, W, false>(n, phi, psi, R, ws + WW * P, ws + WFB * P, ws + WGB * P, ws + WTB * P, sm, ep);
    }
    __syncthreads();
    // ---- lines 8-12 (own = A): phi = a ./ (K~ psi)
    {
      double ep = 0.0;
      half<E, W, false>(n, psi, phi, R, ws + WW * P, ws + WFA * P, ws + WGA * P, ws + WTA * P, sm, ep);
    }
    __syncthreads();
    ++l;  // line 13
    // non-finite state: abnormal termination; else Remark 2.1's test
    double mx = 0.0;
    int bad = 0;
    for (int e = 0; e < E; ++e) {
      const int i = e * T + t;
      const double x = phi[i], y = psi[i];
      if (!isfinite(x) || !isfinite(y)) bad = 1;
      mx = fmax(mx, fmax(fabs(x), fabs(y)));
    }
    if (__syncthreads_or(bad)) {
      flag = FS1F_NONFINITE;
      errv = NAN;
      break;
    }
    if (block_max(mx, red, W) > SP.tau) {
      // absorption: alpha += eps ln phi, beta += eps ln psi (kept divided by eps), phi = psi = 1
      for (int e = 0; e < E; ++e) {
        const int i = e * T + t;
        const long long k = (long long)t * E + e;
        if (k < n) {
          ws[WA * P + i] += log(phi[i]);
          ws[WB * P + i] += log(psi[i]);
          phi[i] = 1.0;
          psi[i] = 1.0;
        }
      }
      __syncthreads();
      form_coeffs<E, W>(n, SP.lam, ws);
    }
    __syncthreads();
  }
  __syncthreads();
  double cost = NAN;
  if (flag != FS1F_NONFINITE) cost = cost_stab<E, W>(n, SP.h, phi, psi, ws, sj, red);
  // outputs: F = A + ln phi, G = B + ln psi
  for (int e = 0; e < E; ++e) {
    const int i = e * T + t;
    const long long k = (long long)t * E + e;
    if (k < n) {
      F[k] = ws[WA * P + i] + log(phi[i]);
      G[k] = ws[WB * P + i] + log(psi[i]);
    }
  }
  if (t == 0) {
    if (SP.iters) SP.iters[pb] = l;
    if (SP.err) SP.err[pb] = errv;
    if (SP.flags) SP.flags[pb] = flag;
    if (SP.cost) SP.cost[pb] = cost;
  }
}

}  // namespace stab
}  // namespace fs1
