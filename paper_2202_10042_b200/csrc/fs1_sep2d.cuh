// fs1_sep2d.cuh — K3: the separable 2D FS-1 kernel (fp32, log domain; config C4,
// 2048 x 2048).
//
// Algorithm 2 on an n x m grid with the block-Toeplitz kernel
// K = T_M(lambda2) (x) T_N(lambda1): every K x is a pass of
// 1D applies along axis 1 (the paper's K0 on every column) and
// a pass along axis 2 (the lambda2 recursion across columns).
//
// B200 design: one cooperative persistent launch for the whole solve.  Both
// passes always run on CONTIGUOUS lines: the first pass of a half-step writes its
// result transposed (8 lines are staged in shared memory and leave as 32-byte
// rows), so the second pass again reads contiguous lines.  The state therefore
// alternates layouts: F = log phi is kept column-major (the user's layout,
// PAPER.md:244-255), G = log psi row-major (transposed); targets are stored in
// the layout of the pass that consumes them (log a column-major, log b
// row-major).  Each line is one CTA-wide chunked scan (256 threads x 8 points,
// the persistent kernel's extended-range carries, fs1_persist.cuh); inside a
// thread chunk the arithmetic is linear fp32 relative to the chunk's binary
// exponent, with one MUFU ex2 per point in and one lg2 out per pass (the
// chunk-relative log scheme of SURVEY.md §7 hard part 3).  Grid-wide barriers
// separate the passes (4 per iteration).
#pragma once
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"
#include "fs1_params.h"
#include "fs1_persist.cuh"
#include "fs1_stream.cuh"

namespace fs1 {
namespace sep {

constexpr int E = 8;
constexpr int W = 8;
constexpr int NT = 32 * W;
constexpr int LMAX = E * NT;  // longest line (2048)
constexpr int TL = 8;         // lines staged per transposed write
constexpr float LOG2E_F = 1.4426950408889634f;
constexpr float LN2_F = 0.6931471805599453f;
using PS = Persist<float, E, W, true>;

struct Smem {
  float* stage;  // [TL][LMAX]
  double* xm;    // [4][W]
  int* xi;       // [4][W]
  double* red;   // [64]
  int* ired;     // [64]
};
constexpr size_t OFF_XM = (size_t)TL * LMAX * 4;
constexpr size_t OFF_XI = OFF_XM + 4 * W * 8;
constexpr size_t OFF_RED = OFF_XI + 4 * W * 4;
constexpr size_t OFF_IRED = OFF_RED + 64 * 8;
constexpr size_t SMEM = OFF_IRED + 64 * 4;

__device__ __forceinline__ float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2f(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

struct Ctx {
  int tid, lane, warp, r;
  int par;
  unsigned gen;
  Smem s;
};

// Load this thread's chunk of a log line into mantissas relative to 2^oe
// (oe = floor(max log2), one ex2 per point).
__device__ __forceinline__ void load_log_chunk(const float* xg, int len, int tid, float (&m)[E], int& oe,
                                               int& nv) {
  const int g0 = tid * E;
  nv = max(0, min(E, len - g0));
  float X[E];
#pragma unroll
  for (int e = 0; e < E; ++e) X[e] = (e < nv) ? __ldcg(xg + g0 + e) : -INFINITY;
  float M = -INFINITY;
#pragma unroll
  for (int e = 0; e < E; ++e) M = fmaxf(M, X[e]);
  if (M == -INFINITY) {
    oe = ZE;
#pragma unroll
    for (int e = 0; e < E; ++e) m[e] = 0.f;
  } else if (!(M < INFINITY)) {
    oe = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) m[e] = NAN;
  } else {
    oe = (int)floorf(M * LOG2E_F);
    const float o = (float)oe;
#pragma unroll
    for (int e = 0; e < E; ++e) m[e] = (X[e] == -INFINITY) ? 0.f : ex2f(fmaf(X[e], LOG2E_F, -o));
  }
}

// log K e^x along one line (lambda, tables of Pa): Y[e] for this thread's chunk.
__device__ __forceinline__ void line_logK(Ctx& c, const PersistParams& Pa, const float* xg, int len,
                                          float (&Y)[E], int& nv) {
  float m[E];
  int oe;
  load_log_chunk(xg, len, c.tid, m, oe, nv);
  const float lam = (float)Pa.lam;
  float f = 0.f, g = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    f = fmaf(lam, f, m[e]);
    g = fmaf(lam, g, m[E - 1 - e]);
  }
  ER<double> CF, CB;
  PS::carries_er(f, g, oe, CF, CB, Pa, c.s.xm, c.s.xi, c.par, c.lane, c.warp,
                 ER<double>{Pa.lanem[c.lane], Pa.lanee[c.lane]},
                 ER<double>{Pa.lanem[31 - c.lane], Pa.lanee[31 - c.lane]});
  c.par ^= 1;
  const int xeff = (f > 0.f) ? oe : ZE;
  int R = max(xeff, max(CF.e, CB.e));
  if (R == ZE) R = 0;
  const float s = Tr<float>::pow2(max(oe - R, -1000));
  const float cf = (float)er_rel(CF, R), cb = (float)er_rel(CB, R);
  float pf[E];
  float p = cf;
#pragma unroll
  for (int e = 0; e < E; ++e) { p = fmaf(lam, p, m[e] * s); pf[e] = p; }
  float tn = cb;
  const float Rf = (float)R;
#pragma unroll
  for (int e = E - 1; e >= 0; --e) {
    const float kx = fmaf(lam, tn, pf[e]);
    tn = fmaf(lam, tn, m[e] * s);
    Y[e] = (lg2f(kx) + Rf) * LN2_F;
  }
}

// Pass A: lines of `in` (nlines x len, contiguous lines) -> log K e^x written
// transposed into `out` (len x nlines).
__device__ __forceinline__ void pass_transposed(Ctx& c, const PersistParams& Pa, const float* in, int nlines,
                                                int len, float* out, int G) {
  const int ngroups = (nlines + TL - 1) / TL;
  for (int grp = c.r; grp < ngroups; grp += G) {
    for (int k = 0; k < TL; ++k) {
      const int line = grp * TL + k;
      if (line >= nlines) break;  // uniform
      float Y[E];
      int nv;
      line_logK(c, Pa, in + (size_t)line * len, len, Y, nv);
      float* st = c.s.stage + (size_t)k * LMAX + c.tid * E;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e < nv) st[e] = Y[e];
    }
    __syncthreads();
    const int l0 = grp * TL;
    const int nk = min(TL, nlines - l0);
    const bool vec = (nk == TL) && ((nlines & 7) == 0);
    for (int pos = c.tid; pos < len; pos += NT) {
      float v[TL];
#pragma unroll
      for (int k = 0; k < TL; ++k) v[k] = c.s.stage[(size_t)k * LMAX + pos];
      float* o = out + (size_t)pos * nlines + l0;
      if (vec) {
        reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(o)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
        for (int k = 0; k < nk; ++k) o[k] = v[k];
      }
    }
    __syncthreads();
  }
}

// Pass B: lines of `in` -> y = LT - log K e^x in the same layout (the update of
// PAPER.md:330/334), or y = log K e^x when LT == nullptr (apply).  CHECK adds
// sum |e^{yold + log K e^x} - e^{LT}| (the marginal error).
template <bool CHECK, bool WRITE>
__device__ __forceinline__ void pass_update(Ctx& c, const PersistParams& Pa, const float* in, int nlines,
                                            int len, const float* LT, const float* yold, float* y, int G,
                                            double& errsum, int& bad) {
  for (int line = c.r; line < nlines; line += G) {
    float Y[E];
    int nv;
    const size_t off = (size_t)line * len;
    line_logK(c, Pa, in + off, len, Y, nv);
    const int g0 = c.tid * E;
    double ep = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e < nv) {
        const float lt = LT ? __ldcg(LT + off + g0 + e) : 0.f;
        if (CHECK) {
          const float yo = __ldcg(yold + off + g0 + e);
          const float a = ex2f((yo + Y[e]) * LOG2E_F);
          const float b = (lt == -INFINITY) ? 0.f : ex2f(lt * LOG2E_F);
          ep += fabs((double)a - (double)b);
        }
        if (WRITE) {
          float v;
          if (LT) v = (lt == -INFINITY) ? -INFINITY : lt - Y[e];
          else v = Y[e];
          if (v != v || v == INFINITY) bad = 1;
          y[off + g0 + e] = v;
        }
      }
    }
    if (CHECK) {
      // deterministic block sum of this line's error, accumulated in line order
      ep = warp_sum(ep);
      if (c.lane == 0) c.s.red[c.warp] = ep;
      __syncthreads();
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) s += c.s.red[w];
      errsum += s;
      __syncthreads();
    }
  }
}

// Elementwise log / transpose phases (prologue and epilogue).
// out (cols x rows) = f(in (rows x cols))^T through 32 x 32 shared tiles.
__device__ __forceinline__ void transpose_phase(Ctx& c, const float* in, int rows, int cols, float* out,
                                                bool to_log, int G) {
  float* t = c.s.stage;  // [32][33]
  const int tr = (rows + 31) / 32, tc = (cols + 31) / 32;
  const int tx = c.tid & 31, ty = c.tid >> 5;  // 32 x 8
  for (int tile = c.r; tile < tr * tc; tile += G) {
    const int r0 = (tile / tc) * 32, c0 = (tile % tc) * 32;
    for (int k = ty; k < 32; k += 8) {
      const int rr = r0 + k, cc = c0 + tx;
      float v = 0.f;
      if (rr < rows && cc < cols) {
        v = __ldcg(in + (size_t)rr * cols + cc);
        if (to_log) v = logf(v);
      }
      t[k * 33 + tx] = v;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
      const int cc = c0 + k, rr = r0 + tx;
      if (rr < rows && cc < cols) out[(size_t)cc * rows + rr] = t[tx * 33 + k];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void map_phase(Ctx& c, const float* in, size_t cnt, float* out, int mode, float cst,
                                          int G) {
  // mode 0: copy, 1: log, 2: constant
  for (size_t k = (size_t)c.r * NT + c.tid; k < cnt; k += (size_t)G * NT) {
    float v = cst;
    if (mode != 2) {
      v = __ldcg(in + k);
      if (mode == 1) v = logf(v);
    }
    out[k] = v;
  }
}

// One line of the return line: sum_k y_k (W x)_k with x, y log lines,
// W the distance-weighted kernel of this axis (h, lambda of Pa).
__device__ __forceinline__ double line_cost(Ctx& c, const PersistParams& Pa, const float* xg, const float* yg,
                                            int len) {
  using Vt = float4;
  Vt* sx = reinterpret_cast<Vt*>(c.s.stage);
  Vt* sy = reinterpret_cast<Vt*>(c.s.stage + LMAX);
  float m[E];
  int xe, ye, nv;
  load_log_chunk(xg, len, c.tid, m, xe, nv);
  PS::sts(sx, c.tid, m);
  load_log_chunk(yg, len, c.tid, m, ye, nv);
  PS::sts(sy, c.tid, m);
  __syncthreads();
  const double cp = cost_pass<float, E, W, true>(Pa, sx, xe, sy, ye, c.tid, c.lane, c.warp, c.s.xm, c.s.xi);
  double s = warp_sum(cp);
  __syncthreads();
  if (c.lane == 0) c.s.red[c.warp] = s;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < W; ++w) t += c.s.red[w];
  __syncthreads();
  return t;
}

// Sum over CTAs of one value per CTA (slot k of part), identical on every CTA.
__device__ __forceinline__ double grid_sum(Ctx& c, const Sep2dParams& P, double mine, int slot, int& flag,
                                           int myflag) {
  if (c.tid == 0) {
    P.part[(size_t)slot * P.G + c.r] = mine;
    P.flagp[(size_t)slot * P.G + c.r] = myflag;
  }
  stm::grid_barrier(P.bar, P.G, c.gen);
  if (c.warp == 0) {
    double s = 0.0;
    int f = 0;
    for (int k = c.lane; k < P.G; k += 32) {
      s += __ldcg(P.part + (size_t)slot * P.G + k);
      f |= __ldcg(P.flagp + (size_t)slot * P.G + k);
    }
    s = warp_sum(s);
    f = __reduce_or_sync(FULL, (unsigned)f);
    if (c.lane == 0) { c.s.red[32] = s; c.s.ired[32] = f; }
  }
  __syncthreads();
  const double r = c.s.red[32];
  flag = c.s.ired[32];
  __syncthreads();
  return r;
}

#ifdef FS1_SEP2D_KERNEL_TU  // defined once, in fs1_sep2d.cu
__global__ void __launch_bounds__(NT, 1) fs1_sep2d_kernel(const __grid_constant__ Sep2dParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  Ctx c;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  c.r = blockIdx.x;
  c.par = 0;
  c.gen = 0;
  c.s.stage = reinterpret_cast<float*>(smem);
  c.s.xm = reinterpret_cast<double*>(smem + OFF_XM);
  c.s.xi = reinterpret_cast<int*>(smem + OFF_XI);
  c.s.red = reinterpret_cast<double*>(smem + OFF_RED);
  c.s.ired = reinterpret_cast<int*>(smem + OFF_IRED);
  const int n = P.n, m = P.m, G = P.G;
  const size_t nm = (size_t)n * m;
  const float* A = reinterpret_cast<const float*>(P.a);
  const float* B = reinterpret_cast<const float*>(P.b);
  float* U = reinterpret_cast<float*>(P.u);
  float* V = reinterpret_cast<float*>(P.v);
  int flag = 0;

  if (P.mode == 1) {  // apply: y = log K e^x (column-major in and out)
    const float* X = reinterpret_cast<const float*>(P.x);
    float* Y = reinterpret_cast<float*>(P.y);
    pass_transposed(c, P.ax1, X, m, n, P.Z, G);  // columns along axis 1 -> row-major
    stm::grid_barrier(P.bar, G, c.gen);
    pass_transposed(c, P.ax2, P.Z, n, m, Y, G);  // rows along axis 2 -> column-major
    return;
  }
  if (P.mode == 2) {  // cost of (u, v) given column-major logs
    transpose_phase(c, V, m, n, P.Gt0, false, G);  // v (cols of length n) -> row-major
    stm::grid_barrier(P.bar, G, c.gen);
  } else {
    // ---- prologue: log a (col-major), (log b)^T (row-major), phi0 / psi0
    map_phase(c, A, nm, P.LA, P.input_is_log ? 0 : 1, 0.f, G);
    transpose_phase(c, B, m, n, P.LBt, !P.input_is_log, G);
    const float init = -logf((float)n) - logf((float)m);
    if (!P.warm) {
      map_phase(c, nullptr, nm, U, 2, init, G);
      map_phase(c, nullptr, nm, P.Gt0, 2, init, G);
    } else {
      transpose_phase(c, V, m, n, P.Gt0, false, G);
    }
    stm::grid_barrier(P.bar, G, c.gen);
  }

  int l = 0, qi = 0;
  double errv = NAN;
  if (P.mode == 0) {
    const bool use_tol = P.tol > 0.0;
    while (true) {
      const bool check = (l >= P.itr_max) || (use_tol && (l % P.check_interval) == 0);
      const bool last = l >= P.itr_max;
      float* Gi = qi ? P.Gt1 : P.Gt0;
      float* Go = qi ? P.Gt0 : P.Gt1;
      // ---- psi half-step (Alg. 2 lines 3-7): K1 on columns of F, transposed; then K2
      // along rows fused with G = log b - log K e^F
      pass_transposed(c, P.ax1, U, m, n, P.Z, G);
      stm::grid_barrier(P.bar, G, c.gen);
      double es = 0.0;
      int bad = 0;
      if (!check) pass_update<false, true>(c, P.ax2, P.Z, n, m, P.LBt, nullptr, Go, G, es, bad);
      else if (!last) pass_update<true, true>(c, P.ax2, P.Z, n, m, P.LBt, Gi, Go, G, es, bad);
      else pass_update<true, false>(c, P.ax2, P.Z, n, m, P.LBt, Gi, Go, G, es, bad);
      bad = __syncthreads_or(bad);
      int f;
      const double e = grid_sum(c, P, es, 0, f, bad);
      if (check) {
        errv = e;
        if (last || errv <= P.tol) {
          flag = (use_tol && errv <= P.tol) ? 1 : 4;
          break;
        }
      }
      qi ^= 1;  // psi^(l+1) is now current
      if (f) { ++l; flag = 2; break; }
      // ---- phi half-step (lines 8-12): K2 along rows of G, transposed; then K1 along
      // columns fused with F = log a - log K e^G
      pass_transposed(c, P.ax2, Go, n, m, P.Z, G);
      stm::grid_barrier(P.bar, G, c.gen);
      bad = 0;
      pass_update<false, true>(c, P.ax1, P.Z, m, n, P.LA, nullptr, U, G, es, bad);
      bad = __syncthreads_or(bad);
      grid_sum(c, P, 0.0, 1, f, bad);
      ++l;  // line 13
      if (f) { flag = 2; break; }
    }
  }
  float* Gf = (P.mode == 2) ? P.Gt0 : (qi ? P.Gt1 : P.Gt0);
  float* Gs = (P.mode == 2) ? P.Gt1 : (qi ? P.Gt0 : P.Gt1);
  double cost = NAN;
  if (flag != 2) {
    // ---- return line: sum phi (W1 (x) K2) psi + sum psi (K1 (x) W2) phi
    pass_transposed(c, P.ax2, Gf, n, m, P.Z, G);  // K2 along rows of psi -> column-major
    pass_transposed(c, P.ax1, U, m, n, Gs, G);    // K1 along columns of phi -> row-major
    stm::grid_barrier(P.bar, G, c.gen);
    double s = 0.0;
    for (int j = c.r; j < m; j += G) s += line_cost(c, P.ax1, P.Z + (size_t)j * n, U + (size_t)j * n, n);
    for (int i = c.r; i < n; i += G) s += line_cost(c, P.ax2, Gs + (size_t)i * m, Gf + (size_t)i * m, m);
    int f;
    cost = grid_sum(c, P, s, 2, f, 0);
  } else {
    errv = NAN;
  }
  if (P.mode == 2) {
    if (c.r == 0 && c.tid == 0 && P.cost) P.cost[0] = cost;
    return;
  }
  // ---- outputs: F is already in u (column-major); v = G transposed back
  transpose_phase(c, Gf, n, m, V, false, G);
  if (c.r == 0 && c.tid == 0) {
    if (P.iters) P.iters[0] = l;
    if (P.err) P.err[0] = errv;
    if (P.flags) P.flags[0] = flag;
    if (P.cost) P.cost[0] = cost;
  }
}

#endif  // FS1_SEP2D_KERNEL_TU

}  // namespace sep
}  // namespace fs1
