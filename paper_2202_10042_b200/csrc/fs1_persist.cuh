// fs1_persist.cuh — the persistent one-CTA-per-problem FS-1 kernel (sm_100a).
//
// One CTA owns one problem (one histogram pair) for the whole solve
// (Algorithm 1).  Thread t owns the E consecutive grid
// points [tE, tE+E); phi and psi live in registers (the 64-point fp32 chunks: one
// array shared by both, ONE below), a and b in swizzled shared memory, for all
// iterations.  Every K x (Eq. 3.1) is evaluated as the paper's
// forward and backward first-order recursions (Eq. "recursion")
// run as a chunked associative scan of the affine maps y -> lambda^L y + c:
//   1. per thread: the chunk aggregates f = p at the chunk end and g = t at the
//      chunk start, from zero carries (Horner, 1 FMA per point per direction);
//   2. warp: Hillis-Steele scan of the aggregates over lanes (5 shuffle levels),
//      multipliers lambda^{E 2^k}; CTA: warp totals through shared memory;
//   3. per thread: the two recursions again from the exact carries, fused with
//      the update psi = b ./ (p + q) (q_k = lam t_{k+1}).
// Steps 1 and 3 run as NCH interleaved sub-chains per thread chunk (ILP).
// The marginal error and the return-line cost (PAPER.md:163,
// O(N) Jordan-block scan, R7) are fused into the same passes.
//
// LOGD = true is the log domain: phi, psi are mantissas with one binary
// exponent per thread chunk (ER form), renormalised every half-step — the
// absorption of Remark 2.1 / 3.2 in exact powers
// of two; carries between chunks are ER numbers.
#pragma once
#include <math.h>

#include <type_traits>

#include "fs1_common.cuh"
#include "fs1_params.h"

namespace fs1 {

constexpr int NF_EVERY = 16;
#ifndef FS1_NOSC
#define FS1_NOSC 16
#endif
#ifndef FS1_NCH
#define FS1_NCH 4
#endif
#ifndef FS1_NEWTON_WARPS
#define FS1_NEWTON_WARPS 4
#endif
#ifndef FS1_ONE
#define FS1_ONE 1
#endif
// resident warps per SM the one-array fp32 variants size their registers for
#ifndef FS1_ONE_W64
#define FS1_ONE_W64 12
#endif
constexpr int NOSC = FS1_NOSC;  // renormalisation skipped while |kexp| <= NOSC (LOGD)  // non-finite detection interval of multi-warp CTAs
constexpr int FS1_NONFINITE_FLAG = 2;
constexpr double LN2 = 0.69314718055994530942;

// ONE: the 64-point fp32 variants hold a single state vector in registers.  A half-step reads
// x into the array, overwrites it with the forward recursion p and recovers
// x_k = p_k - lam p_{k-1} in the backward recursion, so phi and psi share one register
// array (the other one lives only as the next half-step's input).  The vector a
// check compares against (psi^(l)) and the state a stopping check
// returns (phi^(l)) are stashed as raw mantissas in the output buffers u, v when a
// loop top may need them; no third shared array (sK).  Halving the register state
// raises the resident problems per SM (C5: 4 -> 6 CTAs, smem-bound by a and b).
// Only the 64-point fp32 chunks use it: the 32-point ones already hold 16 warps per SM
// with both vectors, and the recovery's extra FMA per point made C2 slower (2.33 ->
// 2.57 ms; C5 47.3 -> 40.4 ms).
// the guarded renormalisation skip also in the one-array 64-point chunks: measured
// slower (C5 39.6 -> 42.3 ms: the second copy of the backward loop), off
#ifndef FS1_SKIP64
#define FS1_SKIP64 0
#endif
#ifndef FS1_ONE_MINE
#define FS1_ONE_MINE 64
#endif
#ifndef FS1_ONE_W32
#define FS1_ONE_W32 28
#endif
template <class T, int E> constexpr bool persist_one() { return FS1_ONE && sizeof(T) == 4 && E >= FS1_ONE_MINE; }

template <class T, int E, int WARPS, bool LOGD> struct Persist {
  using Tt = Tr<T>;
  using Vt = typename Tt::V;
  static constexpr int VEC = Tt::VEC;
  static constexpr int V = E / VEC;
  static constexpr int NT = 32 * WARPS;
  static constexpr bool ONE = persist_one<T, E>();
  // fp64 quotient by Newton refinement in the small-CTA variants (latency-bound: one
  // or a few problems), by the correctly rounded reciprocal in the 8-32-warp ones
  static constexpr bool NEWTON = (WARPS <= FS1_NEWTON_WARPS);
  static_assert(E % VEC == 0, "E must be a multiple of the vector width");

  // shared memory layout (bytes): a, b mantissas [, y_old of a check (two-array mode)]
  static constexpr size_t ARR = (size_t)NT * V * sizeof(Vt);
  static constexpr size_t OFF_XM = (ONE ? 2 : 3) * ARR;              // [2 par][2 dir][WARPS] double
  static constexpr size_t OFF_XE = OFF_XM + 4 * WARPS * sizeof(double);  // [2][2][WARPS] int
  static constexpr size_t OFF_RED = OFF_XE + 4 * WARPS * sizeof(int);    // [2][WARPS] double
  static constexpr size_t OFF_INT = OFF_RED + 2 * WARPS * sizeof(double);  // [2][WARPS] int
  static constexpr size_t OFF_LPM = (OFF_INT + 2 * WARPS * sizeof(int) + 15) & ~(size_t)15;  // [32] double
  static constexpr size_t OFF_LPE = OFF_LPM + 64 * sizeof(double);                          // [32] int
  // multi-warp CTAs: the lane powers lambda^{E l} (log: ER; scaling: the two factors
  // laneA, laneB at [0, 32) and [32, 64)) live in shared memory,
  // read lane-indexed where the cross-warp carries use them (held in registers they were
  // re-read from the parameter bank with lane-divergent addresses on every half-step)
  static constexpr size_t SMEM = OFF_LPE + 32 * sizeof(int);

  // vector j of thread t at s[j * NT + t]: consecutive threads read consecutive 16-byte
  // words (conflict-free) and every access is one base register plus an immediate offset
  __device__ __forceinline__ static int vidx(int tid, int j) { return j * NT + tid; }
  __device__ __forceinline__ static void lds(const Vt* s, int tid, T (&o)[E]) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      Vt v = s[vidx(tid, j)];
      Tt::unpack(v, &o[j * VEC]);
    }
  }
  __device__ __forceinline__ static void sts(Vt* s, int tid, const T (&o)[E]) {
#pragma unroll
    for (int j = 0; j < V; ++j) s[vidx(tid, j)] = Tt::pack(&o[j * VEC]);
  }
  __device__ __forceinline__ static T lds1(const Vt* s, int tid, int e) {  // one element
    const T* p = reinterpret_cast<const T*>(s);
    return p[vidx(tid, e / VEC) * VEC + (e % VEC)];
  }

  // ---------------------------------------------------------------- block sums
  __device__ __forceinline__ static double block_sum(double v, double* red, int par, int lane,
                                                     int warp) {
    v = warp_sum(v);
    if constexpr (WARPS == 1) {
      return v;
    } else {
      if (lane == 0) red[par * WARPS + warp] = v;
      __syncthreads();
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) s += red[par * WARPS + w];
      return s;
    }
  }
  __device__ __forceinline__ static int block_min(int v, int* ired, int par, int lane, int warp) {
    v = warp_min(v);
    if constexpr (WARPS == 1) {
      return v;
    } else {
      if (lane == 0) ired[par * WARPS + warp] = v;
      __syncthreads();
      int s = ired[par * WARPS];
#pragma unroll
      for (int w = 1; w < WARPS; ++w) s = min(s, ired[par * WARPS + w]);
      return s;
    }
  }

  // ------------------------------------------------------- carries, scaling domain
  // f: forward aggregate of this chunk, g: backward aggregate (zero carries in).
  // out: cf = p just before the chunk, cb = t just after it (exclusive scan).
  __device__ __forceinline__ static void carries_lin(T f, T g, T& cf, T& cb,
                                                     const PersistParams& P, double* xm, int par,
                                                     int lane, int warp, T lA, T lB, T rA, T rB) {
    T F = f, G = g;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int d = 1 << k;
      T up = __shfl_up_sync(FULL, F, d);
      T dn = __shfl_down_sync(FULL, G, d);
      const T A = (T)P.lvA[k], B = (T)P.lvB[k];
      if (lane >= d) F = fma(up * A, B, F);
      if (lane + d < 32) G = fma(dn * A, B, G);
    }
    cf = __shfl_up_sync(FULL, F, 1);
    cb = __shfl_down_sync(FULL, G, 1);
    if (lane == 0) cf = T(0);
    if (lane == 31) cb = T(0);
    if constexpr (WARPS > 1) {
      double* wf = xm + (par * 2 + 0) * WARPS;
      double* wg = xm + (par * 2 + 1) * WARPS;
      if (lane == 31) wf[warp] = (double)F;
      if (lane == 0) wg[warp] = (double)G;
      __syncthreads();
      const T wA = (T)P.wA, wB = (T)P.wB;
      T CF = T(0), CG = T(0);
#pragma unroll
      for (int w = 0; w < WARPS; ++w)
        if (w < warp) CF = fma(CF * wA, wB, (T)wf[w]);
#pragma unroll
      for (int w = WARPS - 1; w >= 0; --w)
        if (w > warp) CG = fma(CG * wA, wB, (T)wg[w]);
      cf = fma(CF * lA, lB, cf);
      cb = fma(CG * rA, rB, cb);
    }
  }

  // ------------------------------------------------------- carries, log domain (ER)
  __device__ __forceinline__ static void carries_er(T f, T g, int xe, ER<double>& cf,
                                                    ER<double>& cb, const PersistParams& P,
                                                    double* xm, int* xi, int par, int lane,
                                                    int warp, ER<double> lP, ER<double> rP) {
    ER<T> Fa = er_norm<T>(f, xe), Ga = er_norm<T>(g, xe);
    const int Rw = warp_max(max(Fa.e, Ga.e));
    double F = (double)Fa.m * pow2d(Fa.e - Rw);
    double G = (double)Ga.m * pow2d(Ga.e - Rw);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      F = scan_up(F, 1u << k, P.lvd[k]);
      G = scan_down(G, 1u << k, P.lvd[k]);
    }
    const double cfd = prev_or0(F);
    const double cbd = next_or0(G);
    cf = er_norm<double>(cfd, Rw);
    cb = er_norm<double>(cbd, Rw);
    if constexpr (WARPS > 1) {
      double* wfm = xm + (par * 2 + 0) * WARPS;
      double* wgm = xm + (par * 2 + 1) * WARPS;
      int* wfe = xi + (par * 2 + 0) * WARPS;
      int* wge = xi + (par * 2 + 1) * WARPS;
      if (lane == 31) {
        ER<double> t = er_norm<double>(F, Rw);
        wfm[warp] = t.m;
        wfe[warp] = t.e;
      }
      if (lane == 0) {
        ER<double> t = er_norm<double>(G, Rw);
        wgm[warp] = t.m;
        wge[warp] = t.e;
      }
      __syncthreads();
      const ER<double> LW{P.lvm[5], P.lve[5]};
      ER<double> CF = er_zero<double>(), CG = er_zero<double>();
#pragma unroll
      for (int w = 0; w < WARPS; ++w)
        if (w < warp) CF = er_add(er_mul(CF, LW), ER<double>{wfm[w], wfe[w]});
#pragma unroll
      for (int w = WARPS - 1; w >= 0; --w)
        if (w > warp) CG = er_add(er_mul(CG, LW), ER<double>{wgm[w], wge[w]});
      // warp-uniform skips of the zero contributions (warp 0 has no warp to its left,
      // the last none to its right): bit-identical, adding an ER zero returns cf / cb
      if (warp > 0) cf = er_add(cf, er_mul(CF, lP));
      if (warp < WARPS - 1) cb = er_add(cb, er_mul(CG, rP));
    }
  }
  // the same with the lane powers read from a lane-indexed shared table where they are
  // used (K1: held in registers they were re-read from the parameter bank with
  // lane-divergent addresses on every half-step)
  __device__ __forceinline__ static void carries_er(T f, T g, int xe, ER<double>& cf, ER<double>& cb,
                                                    const PersistParams& P, double* xm, int* xi, int par,
                                                    int lane, int warp, const double* lpm, const int* lpe) {
    if constexpr (WARPS > 1)
      carries_er(f, g, xe, cf, cb, P, xm, xi, par, lane, warp, ER<double>{lpm[lane], lpe[lane]},
                 ER<double>{lpm[31 - lane], lpe[31 - lane]});
    else
      carries_er(f, g, xe, cf, cb, P, xm, xi, par, lane, warp, er_zero<double>(), er_zero<double>());
  }
};

// ---------------------------------------------------------------------------------------
// One half-step x -> y = tgt ./ (K x) on the chunk of this thread.
//   CHECK: also computes the error terms |y_old (K x) - tgt| (y keeps y_old, kx is
//          left in y and y_old saved in sK; the caller finishes with finish()).
// Returns through refs: new y exponent (LOGD), R and kexp for finish().
template <class T, int E, int WARPS, bool LOGD> struct Half {
  using PS = Persist<T, E, WARPS, LOGD>;
  using Tt = Tr<T>;
  using Vt = typename Tt::V;

  struct Ctx {
    int tid, lane, warp, nv;
    T lam, lamS;  // lambda, lambda^S (S = E / NCH: one sub-chain run)
    const double* lab;       // scaling: lane powers laneA[32], laneB[32] (shared memory)
    const double* lpm;       // log: lane powers lambda^{E l} (shared memory)
    const int* lpe;
    double* xm;
    int* xi;
    const T* yold;           // ONE: this chunk's stashed y_old (global) for a check
  };
  static constexpr bool ONE = PS::ONE;

  // Sub-chains of a thread chunk (ILP): the chunk is split into NCH runs of S = E/NCH
  // points whose recursions run interleaved; run c enters with the carry
  // lam^S (carry of run c-1) + (run c-1's aggregate).  S stays a multiple of the
  // shared-memory vector width.
  static constexpr int NCH = (E / PS::VEC >= 8 && FS1_NCH >= 8) ? 8
                             : (E / PS::VEC >= 4 && FS1_NCH >= 4) ? 4 : ((E / PS::VEC >= 2 && FS1_NCH >= 2) ? 2 : 1);
  static constexpr int S = E / NCH;

  // 3. the recursions from the exact carries (fq: forward run aggregates, gq: backward)
  template <bool CHECK, bool MASK, bool SLOW>
  __device__ __forceinline__ static double passes(const Ctx& c, const T (&x)[E], T (&y)[E], int ye,
                                                  const Vt* tgt, int te, Vt* sK, T cf, T cb, T s,
                                                  const T (&fq)[NCH], const T (&gq)[NCH], int R,
                                                  int& kexp_out) {
    constexpr int VEC = PS::VEC;
    const T lam = c.lam, lS = c.lamS;
    auto xs = [&](int e) { return SLOW ? x[e] * s : x[e]; };

    // 3a. forward recursion p_k = lam p_{k-1} + x_k (Alg. 1 line 5 / 10)
    T p[NCH];
    p[0] = cf;
#pragma unroll
    for (int r = 1; r < NCH; ++r) p[r] = fma(lS, p[r - 1], SLOW ? fq[r - 1] * s : fq[r - 1]);
    T p0[NCH];  // ONE: p just before each run (recovers the run's first x)
#pragma unroll
    for (int r = 0; r < NCH; ++r) p0[r] = p[r];
#pragma unroll
    for (int e = 0; e < S; ++e) {
#pragma unroll
      for (int r = 0; r < NCH; ++r) {
        p[r] = fma(lam, p[r], xs(r * S + e));
        y[r * S + e] = p[r];
      }
    }

    // 3b. backward recursion t_k = lam t_{k+1} + x_k, K x = p + lam t_{k+1} (line 6 / 11),
    //     fused with the update y = tgt / Kx (line 7 / 12)
    T t[NCH];
    t[NCH - 1] = cb;
#pragma unroll
    for (int r = NCH - 2; r >= 0; --r) t[r] = fma(lS, t[r + 1], SLOW ? gq[r + 1] * s : gq[r + 1]);
    double errp = 0.0;
    T sc = T(1);
    int kexp = 0;
    T errs = T(1);
    if constexpr (CHECK && LOGD) errs = Tt::pow2(max(min(ye + R - te, 120), -120));
    // the exponent of K x at the chunk's last point renormalises y (LOGD)
    if constexpr (LOGD) kexp = Tt::expo(fma(lam, t[NCH - 1], y[E - 1]));
    auto back = [&](auto sc_on) {
      constexpr bool SC = decltype(sc_on)::value;
      T tv[NCH][VEC], yo[NCH][VEC];
      (void)yo;
      (void)SC;
#pragma unroll
      for (int i = 0; i < S; ++i) {
        if (i % VEC == 0) {
#pragma unroll
          for (int r = 0; r < NCH; ++r) {
            const int e = r * S + S - 1 - i;
            Tt::unpack(tgt[PS::vidx(c.tid, e / VEC)], tv[r]);
            if constexpr (CHECK && !ONE) Tt::unpack(sK[PS::vidx(c.tid, e / VEC)], yo[r]);
            if constexpr (CHECK && ONE) {
#pragma unroll
              for (int q = 0; q < VEC; ++q) {
                const int eq = (e / VEC) * VEC + q;
                yo[r][q] = (!MASK || eq < c.nv) ? c.yold[eq] : T(0);
              }
            }
          }
        }
        T kx[NCH];
#pragma unroll
        for (int rr = 0; rr < NCH; ++rr) {
          const int r = NCH - 1 - rr;
          const int e = r * S + S - 1 - i;
          kx[r] = fma(lam, t[r], y[e]);
          if constexpr (ONE) {
            // x_e = p_e - lam p_{e-1}: y[e - 1] still holds p (written after this read)
            const T pm = (i == S - 1) ? p0[r] : y[e - 1];
            t[r] = fma(lam, t[r], fma(-lam, pm, y[e]));
          } else {
            t[r] = fma(lam, t[r], xs(e));
          }
        }
#pragma unroll
        for (int r = 0; r < NCH; ++r) {
          const int e = r * S + S - 1 - i;
          const int q = e % VEC;
          if constexpr (CHECK) {
            y[e] = kx[r];
            if (!MASK || e < c.nv) errp += (double)fabs(fma(yo[r][q] * errs, kx[r], -tv[r][q]));
          } else {
            T v;
            if constexpr (LOGD && SC) v = Tt::template div<PS::NEWTON>(tv[r][q] * sc, kx[r]);
            else v = Tt::template div<PS::NEWTON>(tv[r][q], kx[r]);
            if (MASK && e >= c.nv) v = T(0);
            y[e] = v;
          }
        }
      }
    };
    if constexpr (LOGD && !CHECK && (sizeof(T) * E <= 128 || (FS1_SKIP64 && ONE))) {
      // (only for chunks whose two state vectors leave registers to spare: the second
      // copy of the loop costs the 64-element float variant more than it saves)
      // The renormalisation is an exact power of two: skip its multiply when every chunk
      // of the warp is already within 2^+-NOSC of it (y's exponent then keeps the offset).
      if (__all_sync(FULL, kexp >= -NOSC && kexp <= NOSC)) {
        kexp = 0;
        back(std::false_type{});
      } else {
        sc = Tt::pow2(kexp);
        back(std::true_type{});
      }
    } else {
      if constexpr (LOGD) sc = Tt::pow2(kexp);
      back(std::true_type{});
    }
    kexp_out = kexp;
    return errp;
  }

  // Returns the per-thread error partial (CHECK) in fp64, units of 1; acc receives the
  // sum of the chunk aggregates of x (non-finite iff some x of the chunk is).
  template <bool CHECK, bool MASK>
  __device__ __forceinline__ static double run(const Ctx& c, const PersistParams& P, const T (&x)[E],
                                               int xe, T (&y)[E], int& ye, const Vt* tgt, int te,
                                               Vt* sK, int par, T& acc, int& R_out, int& k_out) {
    const T lam = c.lam, lS = c.lamS;
    // 1. chunk aggregates (Horner; Eq. recursion with zero carries), 2 NCH independent
    //    chains over the runs: fq[r] forward at the run end, gq[r] backward at its start
    T fq[NCH], gq[NCH];
#pragma unroll
    for (int r = 0; r < NCH; ++r) fq[r] = gq[r] = T(0);
#pragma unroll
    for (int e = 0; e < S; ++e) {
#pragma unroll
      for (int r = 0; r < NCH; ++r) {
        fq[r] = fma(lam, fq[r], x[r * S + e]);
        gq[r] = fma(lam, gq[r], x[r * S + S - 1 - e]);
      }
    }
    T f = fq[0], g = gq[NCH - 1];
#pragma unroll
    for (int r = 1; r < NCH; ++r) f = fma(lS, f, fq[r]);
#pragma unroll
    for (int r = NCH - 2; r >= 0; --r) g = fma(lS, g, gq[r]);
    acc = f + g;  // non-finite input detection (x >= 0: inf and NaN propagate)

    // 2. carries
    T cf, cb, s = T(1);
    int R = 0;
    bool slow = false;
    if constexpr (!LOGD) {
      PS::carries_lin(f, g, cf, cb, P, c.xm, par, c.lane, c.warp, (T)c.lab[c.lane], (T)c.lab[32 + c.lane],
                      (T)c.lab[31 - c.lane], (T)c.lab[63 - c.lane]);
    } else if constexpr (WARPS == 1) {
      // one warp: the ER carries of carries_er() in plain doubles relative to the warp's
      // largest chunk exponent Rw; exact exponents only where the slow-path test needs them
      const int xeff = (f > T(0)) ? xe : ZE;
      const int Rw = warp_max(xeff);
      const double si = pow2d(xe - Rw);
      double F = (double)f * si, G = (double)g * si;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        F = scan_up(F, 1u << k, P.lvd[k]);
        G = scan_down(G, 1u << k, P.lvd[k]);
      }
      const double cfd = prev_or0(F), cbd = next_or0(G);
      const int ecf = (cfd > 0.0) ? Rw + Tr<double>::expo(cfd) : ZE;
      const int ecb = (cbd > 0.0) ? Rw + Tr<double>::expo(cbd) : ZE;
      R = xeff;
      slow = (ecf - xeff > Tt::LIM) || (ecb - xeff > Tt::LIM) || (Rw - xeff > 1000);
      if (slow) {
        R = max(R, max(ecf, ecb));
        s = Tt::pow2(max(xe - R, -1000));
        const double so = pow2d(Rw - R);
        cf = (T)(cfd * so);
        cb = (T)(cbd * so);
      } else {
        const double so = pow2d(Rw - xe);
        cf = (T)(cfd * so);
        cb = (T)(cbd * so);
      }
    } else {
      ER<double> CF, CB;
      PS::carries_er(f, g, xe, CF, CB, P, c.xm, c.xi, par, c.lane, c.warp, c.lpm, c.lpe);
      const int xeff = (f > T(0)) ? xe : ZE;
      R = xeff;
      slow = (CF.e - xeff > Tt::LIM) || (CB.e - xeff > Tt::LIM);
      if (slow) {
        R = max(CF.e, CB.e);
        s = Tt::pow2(max(xe - R, -1000));
      }
      cf = (T)er_rel(CF, R);
      cb = (T)er_rel(CB, R);
    }

    if constexpr (CHECK && !ONE) PS::sts(sK, c.tid, y);  // keep y_old (ONE: stashed already)
    double errp;
    int kexp;
    if (!LOGD || !slow) errp = passes<CHECK, MASK, false>(c, x, y, ye, tgt, te, sK, cf, cb, s, fq, gq, R, kexp);
    else errp = passes<CHECK, MASK, true>(c, x, y, ye, tgt, te, sK, cf, cb, s, fq, gq, R, kexp);
    if constexpr (LOGD) {
      if constexpr (CHECK) errp *= pow2d(te);
      if (!CHECK) ye = (te == ZE) ? ZE : te - R - kexp;
    }
    R_out = R;
    k_out = kexp;
    return errp;
  }

  // After a CHECK half-step that continues: y (holding Kx) -> tgt / Kx.
  template <bool MASK>
  __device__ __forceinline__ static void finish(const Ctx& c, T (&y)[E], int& ye, const Vt* tgt,
                                                int te, int R, int kexp) {
    const T sc = LOGD ? Tt::pow2(kexp) : T(1);
#pragma unroll
    for (int j = 0; j < PS::V; ++j) {
      T tv[PS::VEC];
      Tt::unpack(tgt[PS::vidx(c.tid, j)], tv);
#pragma unroll
      for (int r = 0; r < PS::VEC; ++r) {
        const int e = j * PS::VEC + r;
        T val = Tt::template div<PS::NEWTON>(tv[r] * sc, y[e]);
        if (MASK && e >= c.nv) val = T(0);
        y[e] = val;
      }
    }
    if constexpr (LOGD) ye = (te == ZE) ? ZE : te - R - kexp;
  }

  // After a CHECK half-step that stops: restore y_old.
  __device__ __forceinline__ static void restore(const Ctx& c, T (&y)[E], const Vt* sK) {
    PS::lds(sK, c.tid, y);
  }
};

// ONE: raw mantissas of one thread chunk to / from a global stash (rare: loop tops
// that may check; same thread writes and reads)
template <class T, int E>
__device__ __forceinline__ void stash_store(T* g, int nv, const T (&x)[E]) {
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e < nv) g[e] = x[e];
}
template <class T, int E>
__device__ __forceinline__ void stash_load(const T* g, int nv, T (&x)[E]) {
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = (e < nv) ? g[e] : T(0);
}


// ---------------------------------------------------------------------------------------
// Helpers to bring a chunk of global data into (mantissa, exponent) form.
template <class T, int E, bool LOGD>
__device__ __forceinline__ void load_chunk(const T* g, long long n, long long g0, int nv,
                                           bool is_log, T (&o)[E], int& oe) {
  if constexpr (!LOGD) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const T v = (e < nv) ? g[g0 + e] : T(0);
      o[e] = (e < nv) ? (is_log ? (T)exp((double)v) : v) : T(0);
    }
    oe = 0;
  } else {
    if (is_log) {  // o = exp(l - oe ln2), oe = floor(max l / ln2)
      double M = -INFINITY;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e < nv) M = fmax(M, (double)g[g0 + e]);
      if (!(M > -INFINITY) || !isfinite(M)) {
        oe = ZE;
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = T(0);
        if (M == INFINITY) {  // +inf weight: propagate a NaN so the problem flags NONFINITE
#pragma unroll
          for (int e = 0; e < E; ++e) o[e] = (T)NAN;
        }
      } else {
        oe = (int)floor(M / LN2);
#pragma unroll
        for (int e = 0; e < E; ++e)
          o[e] = (e < nv) ? (T)exp((double)g[g0 + e] - (double)oe * LN2) : T(0);
      }
    } else {
      double M = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (e < nv) M = fmax(M, (double)g[g0 + e]);
      if (!(M > 0.0)) {
        oe = ZE;
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = T(0);
      } else {
        oe = Tr<double>::expo(M);
        const double sc = pow2d(-oe);
#pragma unroll
        for (int e = 0; e < E; ++e) o[e] = (e < nv) ? (T)((double)g[g0 + e] * sc) : T(0);
      }
    }
  }
}

template <class T, int E, bool LOGD>
__device__ __forceinline__ void store_chunk(T* g, long long g0, int nv, const T (&x)[E], int xe) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (e < nv) {
      if constexpr (LOGD) g[g0 + e] = (T)(log((double)x[e]) + (double)xe * LN2);
      else g[g0 + e] = x[e];
    }
  }
}

// ---------------------------------------------------------------------------------------
// Cost pass (return line PAPER.md:163): sum_j psi_j (W phi)_j with
// (W x)_k = h sum_j |k-j| lambda^{|k-j|} x_j evaluated by the Jordan-block recursions
// P'_k = lam (P'_{k-1} + p_{k-1}), Q'_k = lam (Q'_{k+1} + t_{k+1}) (R7),
// as a chunked scan of the pairs (p, P') / (t, Q') in fp64 with ER carries.
template <class T, int E, int WARPS, bool LOGD>
__device__ double cost_pass(const PersistParams& P, const typename Tr<T>::V* sx, int xe,
                            const typename Tr<T>::V* sy, int ye, int tid, int lane, int warp,
                            double* xm, int* xi) {
  using PS = Persist<T, E, WARPS, LOGD>;
  const double lam = P.lam;
  auto x = [&](int e) { return (double)PS::lds1(sx, tid, e); };
  auto y = [&](int e) { return (double)PS::lds1(sy, tid, e); };
  // local aggregates from zero state
  double p = 0, Pp = 0, t = 0, Q = 0;
#pragma unroll 1
  for (int e = 0; e < E; ++e) { Pp = lam * (Pp + p); p = fma(lam, p, x(e)); }
#pragma unroll 1
  for (int e = E - 1; e >= 0; --e) { Q = lam * (Q + t); t = fma(lam, t, x(e)); }
  const int e0 = LOGD ? xe : 0;
  ER<double> ap = er_norm<double>(p, e0), aP = er_norm<double>(Pp, e0);
  ER<double> bt = er_norm<double>(t, e0), bQ = er_norm<double>(Q, e0);
  // combine(A left, B right of span L): p = l^L A.p + B.p ; P = l^L (A.P + L A.p) + B.P
  auto comb = [](ER<double>& Ap, ER<double>& AP, ER<double> Bp, ER<double> BP, ER<double> LL,
                 double L) {
    ER<double> np = er_add(er_mul(Ap, LL), Bp);
    ER<double> nP = er_add(er_mul(er_add(AP, er_scale(Ap, L)), LL), BP);
    Ap = np;
    AP = nP;
  };
  // intra-warp inclusive scans (forward over lanes for (p,P), backward for (t,Q))
  ER<double> Fp = ap, FP = aP, Gt = bt, GQ = bQ;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int d = 1 << k;
    const ER<double> LL{P.lvm[k], P.lve[k]};
    const double L = (double)E * d;
    ER<double> up = shfl_up_er(Fp, d), uP = shfl_up_er(FP, d);
    ER<double> dt = shfl_down_er(Gt, d), dQ = shfl_down_er(GQ, d);
    if (lane >= d) {  // left = up (earlier), right = own (span d chunks)
      ER<double> np = up, nP = uP;
      comb(np, nP, Fp, FP, LL, L);
      Fp = np;
      FP = nP;
    }
    if (lane + d < 32) {
      ER<double> nt = dt, nQ = dQ;
      comb(nt, nQ, Gt, GQ, LL, L);
      Gt = nt;
      GQ = nQ;
    }
  }
  ER<double> cp = shfl_up_er(Fp, 1), cP = shfl_up_er(FP, 1);
  ER<double> ct = shfl_down_er(Gt, 1), cQ = shfl_down_er(GQ, 1);
  if (lane == 0) { cp = er_zero<double>(); cP = er_zero<double>(); }
  if (lane == 31) { ct = er_zero<double>(); cQ = er_zero<double>(); }
  if constexpr (WARPS > 1) {
    // warp totals -> shared, serial fold over warps (span 32E), fix-up per lane (span lane E)
    __syncthreads();
    double* m = xm;  // reuse: [4][WARPS]
    int* ex = xi;
    if (lane == 31) { m[0 * WARPS + warp] = Fp.m; ex[0 * WARPS + warp] = Fp.e;
                      m[1 * WARPS + warp] = FP.m; ex[1 * WARPS + warp] = FP.e; }
    if (lane == 0) { m[2 * WARPS + warp] = Gt.m; ex[2 * WARPS + warp] = Gt.e;
                     m[3 * WARPS + warp] = GQ.m; ex[3 * WARPS + warp] = GQ.e; }
    __syncthreads();
    const ER<double> LW{P.lvm[5], P.lve[5]};
    const double LWL = 32.0 * E;
    ER<double> Cp = er_zero<double>(), CP = er_zero<double>();
    ER<double> Ct = er_zero<double>(), CQ = er_zero<double>();
    for (int w = 0; w < warp; ++w)
      comb(Cp, CP, ER<double>{m[0 * WARPS + w], ex[0 * WARPS + w]},
           ER<double>{m[1 * WARPS + w], ex[1 * WARPS + w]}, LW, LWL);
    for (int w = WARPS - 1; w > warp; --w)
      comb(Ct, CQ, ER<double>{m[2 * WARPS + w], ex[2 * WARPS + w]},
           ER<double>{m[3 * WARPS + w], ex[3 * WARPS + w]}, LW, LWL);
    // carry into lane = combine(warp carry, intra-warp exclusive of span lane*E)
    comb(Cp, CP, cp, cP, ER<double>{P.lanem[lane], P.lanee[lane]}, (double)E * lane);
    comb(Ct, CQ, ct, cQ, ER<double>{P.lanem[31 - lane], P.lanee[31 - lane]},
         (double)E * (31 - lane));
    cp = Cp; cP = CP; ct = Ct; cQ = CQ;
    __syncthreads();
  }
  // in-chunk passes relative to R, accumulating sum_e y_e P'_e and sum_e y_e Q'_e
  int R = max(max(cp.e, cP.e), max(ct.e, cQ.e));
  R = max(R, (p > 0.0 || t > 0.0) ? e0 : ZE);
  const double s = pow2d(max(e0 - R, -1100));
  double pr = er_rel(cp, R), Pr = er_rel(cP, R), tr = er_rel(ct, R), Qr = er_rel(cQ, R);
  double acc = 0.0;
#pragma unroll 1
  for (int e = 0; e < E; ++e) {
    Pr = lam * (Pr + pr);
    pr = fma(lam, pr, x(e) * s);
    acc = fma(y(e), Pr, acc);
  }
#pragma unroll 1
  for (int e = E - 1; e >= 0; --e) {
    Qr = lam * (Qr + tr);
    tr = fma(lam, tr, x(e) * s);
    acc = fma(y(e), Qr, acc);
  }
  const int yexp = LOGD ? ye : 0;
  return (acc == 0.0) ? 0.0 : acc * pow2d(max(min(R + yexp, 1023), -1100)) * P.h;
}

// ---------------------------------------------------------------------------------------
// resident CTAs the register budget is sized for: 16 warps per SM, 8 when the chunk
// state (2 E values of T per thread) needs more than 128 registers
// (ONE: one E-vector per thread; 12 warps, the bound the shared a, b of N = 4096 set)
template <class T, int E, int WARPS> constexpr int persist_minb() {
  const int warps = persist_one<T, E>() ? (E >= 64 ? FS1_ONE_W64 : E >= 32 ? FS1_ONE_W32 : 16)
                                       : ((sizeof(T) * E >= 256) ? 8 : 16);
  return warps / WARPS > 0 ? warps / WARPS : 1;
}

// The solve of the one-array variants (ONE): Algorithm 1 with a
// single register array A that holds phi between half-steps and psi inside an
// iteration.  u, v double as the stashes of phi^(l) and psi^(l) (raw mantissas, same
// thread) for the loop tops that may check; the results overwrite them at the end.
template <class T, int E, int WARPS, bool LOGD>
__device__ __forceinline__ void persist_solve_one(const PersistParams& P, typename Half<T, E, WARPS, LOGD>::Ctx& c,
                                                  typename Tr<T>::V* sA, typename Tr<T>::V* sB, double* xm,
                                                  int* xi, double* red, int* ired, long long base, long long g0,
                                                  bool full) {
  using PS = Persist<T, E, WARPS, LOGD>;
  using H = Half<T, E, WARPS, LOGD>;
  const long long n = P.n;
  const long long pid = blockIdx.x;
  T* const ug = reinterpret_cast<T*>(P.u) + base;
  T* const vg = reinterpret_cast<T*>(P.v) + base;
  T* const su = ug + g0;  // stash of phi^(l)
  T* const sv = vg + g0;  // stash of psi^(l)
  T A[E];
  int ae, be, pe = 0, qe = 0;
  double err = NAN, cost = NAN;
  int l = 0, flag = 0, par = 0;
  int ue = 0, ve = 0;  // exponents of the stashed phi, psi
  // fs1_cost (write_uv = 0): the loop top l = itr_max = 0 on the given state, u and v
  // untouched: the return line only (err is not reported)
  const bool cost_only = !P.write_uv;
  if (cost_only) {
    load_chunk<T, E, LOGD>(ug, n, g0, c.nv, LOGD, A, ue);
    PS::sts(sA, c.tid, A);
    load_chunk<T, E, LOGD>(vg, n, g0, c.nv, LOGD, A, ve);
    PS::sts(sB, c.tid, A);
    flag = 4;
  } else {
    load_chunk<T, E, LOGD>(reinterpret_cast<const T*>(P.a) + base, n, g0, c.nv, P.input_is_log, A, ae);
    PS::sts(sA, c.tid, A);
    load_chunk<T, E, LOGD>(reinterpret_cast<const T*>(P.b) + base, n, g0, c.nv, P.input_is_log, A, be);
    PS::sts(sB, c.tid, A);
    // ---- initial scalings or the caller's: psi^(0) to its stash (the first
    // loop top may check on it), phi^(0) into A
    if (P.warm) {
      load_chunk<T, E, LOGD>(vg, n, g0, c.nv, LOGD, A, qe);
      stash_store<T, E>(sv, c.nv, A);
      load_chunk<T, E, LOGD>(ug, n, g0, c.nv, LOGD, A, pe);
    } else {
      const double inv = 1.0 / (double)n;
      T m0;
      int e0;
      if constexpr (LOGD) { m0 = (T)Tr<double>::mant(inv); e0 = Tr<double>::expo(inv); }
      else { m0 = (T)inv; e0 = 0; }
#pragma unroll
      for (int e = 0; e < E; ++e) A[e] = (e < c.nv) ? m0 : T(0);
      pe = qe = e0;
      stash_store<T, E>(sv, c.nv, A);
    }
    ue = pe;
    ve = qe;
    c.yold = sv;
    __syncthreads();

    int firstbad = 0x7fffffff;
    const int itr_max = P.itr_max;
    const bool use_tol = P.tol > 0.0;
    const int ci = P.check_interval;
    // (captures by value: a reference capture would take the kernel parameter's address
    // and move it to local memory)
    auto is_check = [=](int k) { return (k >= itr_max) || (use_tol && (k % ci) == 0); };
    while (true) {
      const bool check = is_check(l);
      T accx = T(0), accy = T(0);
      int R, kx;
      if (check) {
        // line 2: err = sum |psi^(l) (K^T phi^(l)) - b|; phi^(l) stashed first (a stop returns it)
        stash_store<T, E>(su, c.nv, A);
        ue = pe;
        double ep = full ? H::template run<true, false>(c, P, A, pe, A, ve, sB, be, nullptr, par, accx, R, kx)
                         : H::template run<true, true>(c, P, A, pe, A, ve, sB, be, nullptr, par, accx, R, kx);
        par ^= 1;
        if (!isfinite((double)accx)) firstbad = min(firstbad, l);
        err = PS::block_sum(ep, red, par, c.lane, c.warp);
        int fb;
        if constexpr (WARPS > 1) fb = PS::block_min(firstbad, ired, par, c.lane, c.warp);
        else fb = warp_min(firstbad);
        if (fb != 0x7fffffff) { l = fb; flag = FS1_NONFINITE_FLAG; break; }
        if (l >= itr_max || err <= P.tol) {
          flag = (use_tol && err <= P.tol) ? 1 : 4;
          break;
        }
        if (full) H::template finish<false>(c, A, qe, sB, be, R, kx);
        else H::template finish<true>(c, A, qe, sB, be, R, kx);
      } else {
        // lines 3-7: psi = b ./ (K^T phi)
        if (full) H::template run<false, false>(c, P, A, pe, A, qe, sB, be, nullptr, par, accx, R, kx);
        else H::template run<false, true>(c, P, A, pe, A, qe, sB, be, nullptr, par, accx, R, kx);
        par ^= 1;
      }
      if (is_check(l + 1)) {  // the next loop top compares against psi^(l+1)
        stash_store<T, E>(sv, c.nv, A);
        ve = qe;
      }
      // lines 8-12: phi = a ./ (K psi)
      if (full) H::template run<false, false>(c, P, A, qe, A, pe, sA, ae, nullptr, par, accy, R, kx);
      else H::template run<false, true>(c, P, A, qe, A, pe, sA, ae, nullptr, par, accy, R, kx);
      par ^= 1;
      if (!isfinite((double)accx)) firstbad = min(firstbad, l);
      else if (!isfinite((double)accy)) firstbad = min(firstbad, l + 1);
      ++l;  // line 13
      if constexpr (WARPS == 1) {
        if (__any_sync(FULL, firstbad != 0x7fffffff)) {
          l = warp_min(firstbad);
          flag = FS1_NONFINITE_FLAG;
          break;
        }
      } else {
        if ((l % NF_EVERY) == 0) {
          par ^= 1;
          const int fb = PS::block_min(firstbad, ired, par, c.lane, c.warp);
          if (fb != 0x7fffffff) { l = fb; flag = FS1_NONFINITE_FLAG; break; }
        }
      }
    }

  }  // !cost_only

  // ---- outputs: the state of the stopping loop top from the stashes
  if (flag != FS1_NONFINITE_FLAG) {
    par ^= 1;
    __syncthreads();  // a, b are no longer needed: their shared arrays take phi, psi
    if (!cost_only) {
      stash_load<T, E>(su, c.nv, A);
      PS::sts(sA, c.tid, A);
      stash_load<T, E>(sv, c.nv, A);
      PS::sts(sB, c.tid, A);
    }
    const double cp = cost_pass<T, E, WARPS, LOGD>(P, sA, ue, sB, ve, c.tid, c.lane, c.warp, xm, xi);
    cost = PS::block_sum(cp, red, par, c.lane, c.warp);
    if (!cost_only) {
      PS::lds(sA, c.tid, A);
      store_chunk<T, E, LOGD>(ug, g0, c.nv, A, ue);
      PS::lds(sB, c.tid, A);
      store_chunk<T, E, LOGD>(vg, g0, c.nv, A, ve);
    }
  } else {
    err = NAN;
    store_chunk<T, E, LOGD>(ug, g0, c.nv, A, pe);  // the non-finite state; v holds no result
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (e < c.nv) sv[e] = (T)NAN;
  }
  if (c.tid == 0) {
    if (P.iters) P.iters[pid] = l;
    if (P.err) P.err[pid] = err;
    if (P.flags) P.flags[pid] = flag;
    if (P.cost) P.cost[pid] = cost;
  }
}

template <class T, int E, int WARPS, bool LOGD>
__global__ void __launch_bounds__(32 * WARPS, (persist_minb<T, E, WARPS>())) fs1_persist_solve(const PersistParams P) {
  using PS = Persist<T, E, WARPS, LOGD>;
  using H = Half<T, E, WARPS, LOGD>;
  using Vt = typename PS::Vt;
  extern __shared__ __align__(16) unsigned char smem[];
  Vt* sA = reinterpret_cast<Vt*>(smem);
  Vt* sB = reinterpret_cast<Vt*>(smem + PS::ARR);
  Vt* sK = reinterpret_cast<Vt*>(smem + 2 * PS::ARR);
  double* xm = reinterpret_cast<double*>(smem + PS::OFF_XM);
  int* xi = reinterpret_cast<int*>(smem + PS::OFF_XE);
  double* red = reinterpret_cast<double*>(smem + PS::OFF_RED);
  int* ired = reinterpret_cast<int*>(smem + PS::OFF_INT);

  const long long pid = blockIdx.x;
  const long long n = P.n;
  const long long base = pid * n;
  typename H::Ctx c;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  const long long g0 = (long long)c.tid * E;
  c.nv = (int)max(0LL, min((long long)E, n - g0));
  c.lam = (T)P.lam;
  {
    double l = 1.0;  // lambda^S by stepwise multiplication (Remark 3.3)
    for (int k = 0; k < H::S; ++k) l *= P.lam;
    c.lamS = (T)l;
  }
  c.xm = xm;
  c.xi = xi;
  if constexpr (!LOGD) {
    double* lab = reinterpret_cast<double*>(smem + PS::OFF_LPM);
    if (c.tid < 32) {
      lab[c.tid] = P.laneA[c.tid];
      lab[32 + c.tid] = P.laneB[c.tid];
    }
    c.lab = lab;
  } else {
    double* lpm = reinterpret_cast<double*>(smem + PS::OFF_LPM);
    int* lpe = reinterpret_cast<int*>(smem + PS::OFF_LPE);
    if (c.tid < 32) {
      lpm[c.tid] = P.lanem[c.tid];
      lpe[c.tid] = P.lanee[c.tid];
    }
    c.lpm = lpm;
    c.lpe = lpe;
  }
  // warp-uniform: the masked and unmasked paths contain different barriers
  const bool full = __all_sync(FULL, c.nv == E);
  if constexpr (PS::ONE) {
    persist_solve_one<T, E, WARPS, LOGD>(P, c, sA, sB, xm, xi, red, ired, base, g0, full);
    return;
  }

  // ---- inputs into shared memory (mantissas) and registers (chunk exponents)
  T phi[E], psi[E];
  int ae, be, pe = 0, qe = 0;
  {
    const T* ga = reinterpret_cast<const T*>(P.a) + base;
    const T* gb = reinterpret_cast<const T*>(P.b) + base;
    load_chunk<T, E, LOGD>(ga, n, g0, c.nv, P.input_is_log, phi, ae);
    PS::sts(sA, c.tid, phi);
    load_chunk<T, E, LOGD>(gb, n, g0, c.nv, P.input_is_log, psi, be);
    PS::sts(sB, c.tid, psi);
  }
  // ---- initial scalings: phi0 = psi0 = 1/N or caller-given (warm start)
  if (P.warm) {
    load_chunk<T, E, LOGD>(reinterpret_cast<const T*>(P.u) + base, n, g0, c.nv, LOGD, phi, pe);
    load_chunk<T, E, LOGD>(reinterpret_cast<const T*>(P.v) + base, n, g0, c.nv, LOGD, psi, qe);
  } else {
    const double inv = 1.0 / (double)n;
    T m0;
    int e0;
    if constexpr (LOGD) { m0 = (T)Tr<double>::mant(inv); e0 = Tr<double>::expo(inv); }
    else { m0 = (T)inv; e0 = 0; }
#pragma unroll
    for (int e = 0; e < E; ++e) { phi[e] = (e < c.nv) ? m0 : T(0); psi[e] = phi[e]; }
    pe = qe = e0;
  }
  __syncthreads();

  // ---- Algorithm 1 loop
  int l = 0, flag = 0, par = 0;
  double err = NAN;
  int firstbad = 0x7fffffff;
  const int itr_max = P.itr_max;
  const bool use_tol = P.tol > 0.0;
  while (true) {
    const bool check = (l >= itr_max) || (use_tol && (l % P.check_interval) == 0);
    T accx = T(0), accy = T(0);
    int R, kx;
    if (check) {
      // line 2: err = sum |psi (K^T phi) - b| with phi^(l), psi^(l)
      double ep = full ? H::template run<true, false>(c, P, phi, pe, psi, qe, sB, be, sK, par, accx, R, kx)
                       : H::template run<true, true>(c, P, phi, pe, psi, qe, sB, be, sK, par, accx, R, kx);
      par ^= 1;
      if (!isfinite((double)accx)) firstbad = min(firstbad, l);
      err = PS::block_sum(ep, red, par, c.lane, c.warp);
      int fb;
      if constexpr (WARPS > 1) fb = PS::block_min(firstbad, ired, par, c.lane, c.warp);
      else fb = warp_min(firstbad);
      if (fb != 0x7fffffff) { l = fb; flag = FS1_NONFINITE_FLAG; break; }
      if (l >= itr_max || err <= P.tol) {
        H::restore(c, psi, sK);
        flag = (use_tol && err <= P.tol) ? 1 : 4;
        break;
      }
      if (full) H::template finish<false>(c, psi, qe, sB, be, R, kx);
      else H::template finish<true>(c, psi, qe, sB, be, R, kx);
    } else {
      // lines 3-7: psi = b ./ (K^T phi)
      if (full) H::template run<false, false>(c, P, phi, pe, psi, qe, sB, be, sK, par, accx, R, kx);
      else H::template run<false, true>(c, P, phi, pe, psi, qe, sB, be, sK, par, accx, R, kx);
      par ^= 1;
    }
    // lines 8-12: phi = a ./ (K psi)
    if (full) H::template run<false, false>(c, P, psi, qe, phi, pe, sA, ae, sK, par, accy, R, kx);
    else H::template run<false, true>(c, P, psi, qe, phi, pe, sA, ae, sK, par, accy, R, kx);
    par ^= 1;
    // non-finite state: phi^(l) seen by the psi half-step, psi^(l+1) by
    // the phi half-step; the problem stops with the iteration count of the first one.
    if (!isfinite((double)accx)) firstbad = min(firstbad, l);
    else if (!isfinite((double)accy)) firstbad = min(firstbad, l + 1);
    ++l;  // line 13
    if constexpr (WARPS == 1) {
      if (__any_sync(FULL, firstbad != 0x7fffffff)) {
        l = warp_min(firstbad);
        flag = FS1_NONFINITE_FLAG;
        break;
      }
    } else {
      if ((l % NF_EVERY) == 0) {
        par ^= 1;
        const int fb = PS::block_min(firstbad, ired, par, c.lane, c.warp);
        if (fb != 0x7fffffff) { l = fb; flag = FS1_NONFINITE_FLAG; break; }
      }
    }
  }

  // ---- outputs
  double cost = NAN;
  if (flag != FS1_NONFINITE_FLAG) {
    par ^= 1;
    __syncthreads();  // a, b are no longer needed: their shared arrays take phi, psi
    PS::sts(sA, c.tid, phi);
    PS::sts(sB, c.tid, psi);
    const double cp = cost_pass<T, E, WARPS, LOGD>(P, sA, pe, sB, qe, c.tid, c.lane, c.warp, xm, xi);
    cost = PS::block_sum(cp, red, par, c.lane, c.warp);
  } else {
    err = NAN;
  }
  if (P.write_uv) {
    store_chunk<T, E, LOGD>(reinterpret_cast<T*>(P.u) + base, g0, c.nv, phi, pe);
    store_chunk<T, E, LOGD>(reinterpret_cast<T*>(P.v) + base, g0, c.nv, psi, qe);
  }
  if (c.tid == 0) {
    if (P.iters) P.iters[pid] = l;
    if (P.err) P.err[pid] = err;
    if (P.flags) P.flags[pid] = flag;
    if (P.cost) P.cost[pid] = cost;
  }
}

// ---------------------------------------------------------------------------------------
// y = K x (scaling) or y = log K e^x (log) for every problem: the kernel apply alone.
template <class T, int E, int WARPS, bool LOGD>
__global__ void __launch_bounds__(32 * WARPS) fs1_persist_apply(const PersistParams P, const T* x,
                                                                T* y) {
  using PS = Persist<T, E, WARPS, LOGD>;
  using Tt = Tr<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  double* xm = reinterpret_cast<double*>(smem + PS::OFF_XM);
  int* xi = reinterpret_cast<int*>(smem + PS::OFF_XE);
  const long long pid = blockIdx.x;
  const long long n = P.n;
  const long long base = pid * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long g0 = (long long)tid * E;
  const int nv = (int)max(0LL, min((long long)E, n - g0));
  const T lam = (T)P.lam;
  T v[E];
  int ve;
  load_chunk<T, E, LOGD>(x + base, n, g0, nv, LOGD, v, ve);
  T f = T(0), g = T(0);
#pragma unroll
  for (int e = 0; e < E; ++e) f = fma(lam, f, v[e]);
#pragma unroll
  for (int e = E - 1; e >= 0; --e) g = fma(lam, g, v[e]);
  T cf, cb, s = T(1);
  int R = 0;
  if constexpr (!LOGD) {
    PS::carries_lin(f, g, cf, cb, P, xm, 0, lane, warp, (T)P.laneA[lane], (T)P.laneB[lane],
                    (T)P.laneA[31 - lane], (T)P.laneB[31 - lane]);
  } else {
    ER<double> CF, CB;
    double* lpm = reinterpret_cast<double*>(smem + PS::OFF_LPM);
    int* lpe = reinterpret_cast<int*>(smem + PS::OFF_LPE);
    if (tid < 32) {
      lpm[tid] = P.lanem[tid];
      lpe[tid] = P.lanee[tid];
    }
    __syncthreads();
    PS::carries_er(f, g, ve, CF, CB, P, xm, xi, 0, lane, warp, lpm, lpe);
    const int xeff = (f > T(0)) ? ve : ZE;
    R = max(xeff, max(CF.e, CB.e));
    s = Tt::pow2(max(ve - R, -1000));
    cf = (T)er_rel(CF, R);
    cb = (T)er_rel(CB, R);
  }
  T pp[E];
  T p = cf;
#pragma unroll
  for (int e = 0; e < E; ++e) { p = fma(lam, p, v[e] * s); pp[e] = p; }
  T tn = cb;
#pragma unroll
  for (int e = E - 1; e >= 0; --e) {
    const T kx = fma(lam, tn, pp[e]);
    tn = fma(lam, tn, v[e] * s);
    pp[e] = kx;
  }
  store_chunk<T, E, LOGD>(y + base, g0, nv, pp, R);
}

}  // namespace fs1
