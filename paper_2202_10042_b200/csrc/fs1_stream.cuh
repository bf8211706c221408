// fs1_stream.cuh — K2: the multi-CTA HBM-streaming FS-1 kernel for one large 1D
// problem (fp64, log domain; N = 2^24).
//
// The whole solve (Algorithm 1) is ONE cooperative launch of G
// co-resident CTAs (one per SM).  CTA r owns the contiguous tile range
// [T0_r, T1_r) of 256-point tiles for every vector and every half-step, so the
// per-tile scan tables and tile exponents of the vectors it produces stay in its
// shared memory; only 2 extended-range words per CTA cross the grid per
// half-step.  One half-step x -> y = tgt ./ (K x) (Alg. 1 lines 3-7 / 8-12):
//
//  [A] after the grid barrier: the other CTAs' range totals of x, one per thread,
//      decayed and summed (fixed order) into this range's external forward /
//      backward carries; every tile's full
//      carries = local exclusive carries (made by this CTA when it produced x)
//      + lambda^{256 i} x external carry;
//  [B] each warp streams its tiles: 1D TMA bulk copies (cp.async.bulk, mbarrier
//      complete_tx) of x and tgt into a private S-stage shared-memory ring, a
//      conflict-free XOR-swizzled read into registers (8 points per lane; zero excessive
//      shared wavefronts in ncu's source view, profiles/r02/r02z_bank_conflicts_c3.txt), lane
//      Horner aggregates, a 5-level warp shuffle scan, the forward and backward
//      recursions of Eq. "recursion" from the exact carries,
//      y = tgt * rcp(p + lambda t), one exact power-of-two renormalisation of the
//      output tile, the output tile's totals (one weighted warp reduction each), and a
//      TMA bulk store of y;
//  [C] a block scan of the produced tiles' totals gives their local exclusive
//      carries (kept for the next half-step) and this range's totals, which are
//      published before the grid barrier.
//
// Per update the kernel reads x, tgt and writes y once per half-step: 48 B per
// grid-point update in fp64 (+8 B on check iterations for psi^(l)), the
// algorithmic minimum of SURVEY.md §8(d).  Values are mantissas with one binary
// exponent per tile: the log domain costs one exp per point at
// load and one log at store per solve, none per iteration.
#pragma once
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"
#include "fs1_params.h"

namespace fs1 {
namespace stm {

constexpr int E = 8;                // points per lane
constexpr int TILE = 32 * E;        // points per warp tile
constexpr int TBYTES = TILE * 8;    // bytes per fp64 tile
constexpr int LIM = 600;            // carries up to 2^LIM above a tile keep the tile's exponent
constexpr int MODE_SOLVE = 0, MODE_APPLY = 1, MODE_COST = 2;
constexpr double LN2_HI = 6.93147180369123816490e-01;  // Cody-Waite split of ln 2
constexpr double LN2_LO = 1.90821492927058770002e-10;
constexpr double INV_LN2 = 1.44269504088896338700e+00;

// ------------------------------------------------------------------ shared layout
struct Layout {
  size_t stage, mbar, pwm, pwd, pwe, ax, bx, px, qx0, qx1, pfm, pbm, pfe, pbe, qfm, qbm, qfe, qbe, cfr,
      cbr, rr, errt, redm, rede, dpm, dpe, tza, tzb, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }

__host__ __device__ inline Layout layout(int NW, int S, int ntmax, int G) {
  Layout L;
  size_t o = 0;
  const size_t nt = (size_t)ntmax + 1;
  L.stage = o; o = al16(o + (size_t)NW * S * 2 * TBYTES);
  L.mbar = o;  o = al16(o + (size_t)NW * S * 8);
  L.dpm = o;   o = al16(o + (size_t)G * 8);
  L.dpe = o;   o = al16(o + (size_t)G * 4);
  L.tza = o;   o = al16(o + nt);
  L.tzb = o;   o = al16(o + nt);
  L.pwm = o;   o = al16(o + nt * 8);
  L.pwd = o;   o = al16(o + nt * 8);
  L.pfm = o;   o = al16(o + nt * 8);
  L.pbm = o;   o = al16(o + nt * 8);
  L.qfm = o;   o = al16(o + nt * 8);
  L.qbm = o;   o = al16(o + nt * 8);
  L.cfr = o;   o = al16(o + nt * 8);
  L.cbr = o;   o = al16(o + nt * 8);
  L.errt = o;  o = al16(o + nt * 8);
  L.redm = o;  o = al16(o + 16 * 64 * 8);
  L.pwe = o;   o = al16(o + nt * 4);
  L.ax = o;    o = al16(o + nt * 4);
  L.bx = o;    o = al16(o + nt * 4);
  L.px = o;    o = al16(o + nt * 4);
  L.qx0 = o;   o = al16(o + nt * 4);
  L.qx1 = o;   o = al16(o + nt * 4);
  L.pfe = o;   o = al16(o + nt * 4);
  L.pbe = o;   o = al16(o + nt * 4);
  L.qfe = o;   o = al16(o + nt * 4);
  L.qbe = o;   o = al16(o + nt * 4);
  L.rr = o;    o = al16(o + nt * 4);
  L.rede = o;  o = al16(o + 16 * 64 * 4);
  L.total = o;
  return L;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(b))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// scan_up / scan_down / prev_or0 / next_or0: fs1_common.cuh
__device__ __forceinline__ double fdiv(double t, double x) {
  // t / x without branches: hardware reciprocal estimate r (relative error e, |e| <=
  // 2^-23), refined as r (1 + e + e^2) (relative error O(e^3), below an ulp), times t:
  // a quotient within ~1.5 ulp (x = 0 or non-finite -> non-finite).  The residual
  // correction of the quotient (< 1 ulp) was measured 2% slower at C3 for no parity
  // change (3e-14 norm-wise either way, profiles/r02/golden_errors.txt).
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  r = fma(r, fma(e, e, e), r);
  return t * r;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#ifndef FS1_GB_NOTF
#define FS1_GB_NOTF 0
#endif
// Grid-wide barrier of the co-resident CTAs (the cooperative launch guarantees
// residency): one release-add per CTA on a monotonic counter, then an acquire
// spin until it reaches G x (barriers so far).  bar[0] must be 0 at launch.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned G, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_async();
#if !FS1_GB_NOTF
    __threadfence();
#endif
    const unsigned target = (gen + 1) * G;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (ld_acquire(bar) < target) {
    }
    fence_async();
  }
  ++gen;
  __syncthreads();
}

// ------------------------------------------------------------------ swizzled tiles
// Lane l owns points [8l, 8l+8) of a tile = 4 double2 chunks.  Every internal
// vector (workspace mantissas of a, b, phi, psi) stores chunk j of lane l at
// 16-byte slot 4l + (j ^ sw(l)), sw = (l>>1)&3, in global AND shared memory (the
// TMA copies are verbatim).  Instruction j of a warp then touches slots
// 4l + (j ^ sw): the 8 lanes of a 128-bit phase hit 8 distinct bank groups
// (conflict-free) and registers come out in natural order with no selects.
__device__ __forceinline__ int swz(int lane) { return (lane >> 1) & 3; }
__device__ __forceinline__ void lds_tile(const double* base, int lane, double (&v)[E]) {
  const int sw = swz(lane);
  const double2* p = reinterpret_cast<const double2*>(base) + lane * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 t = p[j ^ sw];
    v[2 * j] = t.x;
    v[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ void sts_tile(double* base, int lane, const double (&v)[E]) {
  const int sw = swz(lane);
  double2* p = reinterpret_cast<double2*>(base) + lane * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j ^ sw] = make_double2(v[2 * j], v[2 * j + 1]);
}
// the same permuted layout from / to global memory (prologue, epilogue, cost, check)
__device__ __forceinline__ void ldg_tile(const double* g, int lane, double (&v)[E]) {
  const int sw = swz(lane);
  const double2* p = reinterpret_cast<const double2*>(g) + lane * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 t = __ldcg(p + (j ^ sw));
    v[2 * j] = t.x;
    v[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ void stg_tile(double* g, int lane, const double (&v)[E]) {
  const int sw = swz(lane);
  double2* p = reinterpret_cast<double2*>(g) + lane * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) p[j ^ sw] = make_double2(v[2 * j], v[2 * j + 1]);
}

// ------------------------------------------------------------------ context
struct Ctx {
  int tid, lane, warp, NT, NW;
  int r, T0, nt;
  double* stage;
  uint64_t* mbar;
  double* dpm;          // lambda^{256 d_k}: distance from range k to this range (ext carries)
  int* dpe;
  unsigned char* tzA;   // tile of a / b has a zero (or padding) entry
  unsigned char* tzB;
  double* pwm;
  double* pwd;  // lambda^{256 k} as a plain double (0 once it underflows)
  int* pwe;
  int* AX;
  int* BX;
  int* PX;
  int* QX0;
  int* QX1;
  double *PFm, *PBm, *QFm, *QBm;
  int *PFe, *PBe, *QFe, *QBe;
  double* cfr;
  double* cbr;
  int* Rr;
  double* errt;
  double* redm;
  int* rede;
  unsigned phase;
  unsigned gen;
};

__device__ __forceinline__ ER<double> pw(const Ctx& c, int k) { return ER<double>{c.pwm[k], c.pwe[k]}; }
__device__ __forceinline__ ER<double> er_fma(ER<double> a, ER<double> b, ER<double> d) {
  return er_add(er_mul(a, b), d);
}
// lambda^{256 k} for any k by binary decomposition (host-formed lambda^{256 2^j})
__device__ __forceinline__ ER<double> pow_tiles(const StreamParams& P, long long k) {
  ER<double> r{1.0, 0};
  for (int j = 0; j < 20 && k; ++j, k >>= 1)
    if (k & 1) r = er_mul(r, ER<double>{P.t2m[j], P.t2e[j]});
  return r;
}
__device__ __forceinline__ long long range_T0(const StreamParams& P, int r) {
  return (long long)r * P.ntiles / P.G;
}
__device__ __forceinline__ ER<double> warp_er_sum(ER<double> a) {
  const int M = warp_max(a.m > 0.0 ? a.e : ZE);
  double s = (a.m > 0.0) ? a.m * pow2d(max(a.e - M, -1100)) : 0.0;
  s = warp_sum(s);
  return er_norm<double>(s, M);
}
__device__ __forceinline__ int expo_d(double m) { return Tr<double>::expo(m); }

// ---------------------------------------------------------------- tile aggregates
// Lane Horner aggregates and the warp scan of a tile held 8 points per lane.
// Returns the inclusive scans: Fi (forward, lane 31 = tile total at the tile end),
// Gi (backward, lane 0 = tile total at the tile start).
__device__ __forceinline__ void tile_scan_lanes(const StreamParams& P, int lane, const double (&v)[E],
                                                double& Fi, double& Gi) {
  const double lam = P.lam;
  double f = 0.0, g = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    f = fma(lam, f, v[e]);
    g = fma(lam, g, v[E - 1 - e]);
  }
  Fi = f;
  Gi = g;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    Fi = scan_up(Fi, 1u << k, P.lvd[k]);
    Gi = scan_down(Gi, 1u << k, P.lvd[k]);
  }
}

// Tile totals only (no per-lane prefixes): forward total at the tile end
// sum_l lambda^{8(31-l)} f_l and backward total at the tile start sum_l lambda^{8l} g_l
// (f_l, g_l the lane aggregates), by one weighted butterfly reduction each; every lane
// gets both totals.  lp = lambda^{8 lane}, rp = lambda^{8(31-lane)}.
#ifndef FS1_K2_REDTOT
#define FS1_K2_REDTOT 1
#endif
#ifndef FS1_K2_SELHOIST
#define FS1_K2_SELHOIST 1
#endif
__device__ __forceinline__ void tile_totals_lanes(const StreamParams& P, double lp, double rp, const double (&v)[E],
                                                  double& Ft, double& Gt) {
  const double lam = P.lam;
  double f = 0.0, g = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    f = fma(lam, f, v[e]);
    g = fma(lam, g, v[E - 1 - e]);
  }
  f *= rp;
  g *= lp;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    f += __shfl_xor_sync(FULL, f, d);
    g += __shfl_xor_sync(FULL, g, d);
  }
  Ft = f;
  Gt = g;
}

// Store the tile totals of a produced tile (exponent Y) into the table at i.
__device__ __forceinline__ void put_totals(int lane, double Fi, double Gi, int Y, double* Fm, int* Fe,
                                           double* Bm, int* Be, int i) {
  if (lane == 31) {
    const ER<double> t = er_norm<double>(Fi, Y);
    Fm[i] = t.m;
    Fe[i] = t.e;
  }
  if (lane == 0) {
    const ER<double> t = er_norm<double>(Gi, Y);
    Bm[i] = t.m;
    Be[i] = t.e;
  }
}

// ---------------------------------------------------------------- block tile scan
// In: F/B hold per-tile totals (forward at the tile end, backward at the tile start).
// Out (in place): exclusive local carries CFloc_i = sum_{i'<i} lambda^{256(i-1-i')} FT_i',
// CBloc_i = sum_{i'>i} lambda^{256(i'-i-1)} GT_i'; returns the range totals.
__device__ __forceinline__ void block_tile_scan_er(Ctx& c, double* Fm, int* Fe, double* Bm, int* Be,
                                                   ER<double>& totF, ER<double>& totB) {
  const int nt = c.nt, NT = c.NT, lane = c.lane, warp = c.warp;
  const int q = (nt + NT - 1) / NT;
  const int i0 = min(nt, c.tid * q), i1 = min(nt, i0 + q);
  const ER<double> L1 = pw(c, 1);
  ER<double> f = er_zero<double>(), g = er_zero<double>();
  for (int i = i0; i < i1; ++i) f = er_fma(f, L1, ER<double>{Fm[i], Fe[i]});
  for (int i = i1 - 1; i >= i0; --i) g = er_fma(g, L1, ER<double>{Bm[i], Be[i]});
  int sF = i1 - i0, sG = i1 - i0;
  ER<double> F = f, G = g;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const ER<double> uf = shfl_up_er(F, d);
    const int us = __shfl_up_sync(FULL, sF, d);
    const ER<double> dg = shfl_down_er(G, d);
    const int ds = __shfl_down_sync(FULL, sG, d);
    if (lane >= d) { F = er_fma(uf, pw(c, sF), F); sF += us; }
    if (lane + d < 32) { G = er_fma(dg, pw(c, sG), G); sG += ds; }
  }
  ER<double> eF = shfl_up_er(F, 1);
  int esF = __shfl_up_sync(FULL, sF, 1);
  ER<double> eG = shfl_down_er(G, 1);
  int esG = __shfl_down_sync(FULL, sG, 1);
  if (lane == 0) { eF = er_zero<double>(); esF = 0; }
  if (lane == 31) { eG = er_zero<double>(); esG = 0; }
  double* wFm = c.redm;
  double* wGm = c.redm + 64;
  int* wFe = c.rede;
  int* wGe = c.rede + 64;
  int* wFs = c.rede + 128;
  int* wGs = c.rede + 192;
  __syncthreads();  // scratch reuse
  if (lane == 31) { wFm[warp] = F.m; wFe[warp] = F.e; wFs[warp] = sF; }
  if (lane == 0) { wGm[warp] = G.m; wGe[warp] = G.e; wGs[warp] = sG; }
  __syncthreads();
  ER<double> cw = er_zero<double>(), cg = er_zero<double>();
  for (int w = 0; w < warp; ++w) cw = er_fma(cw, pw(c, wFs[w]), ER<double>{wFm[w], wFe[w]});
  for (int w = c.NW - 1; w > warp; --w) cg = er_fma(cg, pw(c, wGs[w]), ER<double>{wGm[w], wGe[w]});
  ER<double> cf = er_fma(cw, pw(c, esF), eF);
  ER<double> cb = er_fma(cg, pw(c, esG), eG);
  for (int i = i0; i < i1; ++i) {
    const ER<double> t{Fm[i], Fe[i]};
    Fm[i] = cf.m; Fe[i] = cf.e;
    cf = er_fma(cf, L1, t);
  }
  for (int i = i1 - 1; i >= i0; --i) {
    const ER<double> t{Bm[i], Be[i]};
    Bm[i] = cb.m; Be[i] = cb.e;
    cb = er_fma(cb, L1, t);
  }
  __syncthreads();
  if (c.tid == NT - 1) { wFm[0] = cf.m; wFe[0] = cf.e; }
  if (c.tid == 0) { wGm[0] = cb.m; wGe[0] = cb.e; }
  __syncthreads();
  totF = ER<double>{wFm[0], wFe[0]};
  totB = ER<double>{wGm[0], wGe[0]};
  __syncthreads();
}

// The same scan in plain fp64 relative to 2^M (M = the largest tile exponent of the
// range) when every nonzero total lies within 2^900 of it — always so at C3 — and in
// extended range otherwise.  Contributions that underflow relative to 2^M are below
// 2^-122 of every tile they reach.
__device__ __forceinline__ void block_tile_scan(Ctx& c, double* Fm, int* Fe, double* Bm, int* Be, ER<double>& totF,
                                                ER<double>& totB) {
  const int nt = c.nt, NT = c.NT, lane = c.lane, warp = c.warp;
  int mx = ZE, mn = 0x7fffffff;
  for (int i = c.tid; i < nt; i += NT) {
    if (Fm[i] > 0.0) { mx = max(mx, Fe[i]); mn = min(mn, Fe[i]); }
    if (Bm[i] > 0.0) { mx = max(mx, Be[i]); mn = min(mn, Be[i]); }
  }
  mx = warp_max(mx);
  mn = warp_min(mn);
  int* wi = c.rede + 384;  // (callers enter after a block synchronisation)
  if (lane == 0) { wi[warp] = mx; wi[32 + warp] = mn; }
  __syncthreads();
  mx = warp_max(lane < c.NW ? wi[lane] : ZE);
  mn = warp_min(lane < c.NW ? wi[32 + lane] : 0x7fffffff);
  if (mx != ZE && mn < mx - 900) {
    block_tile_scan_er(c, Fm, Fe, Bm, Be, totF, totB);
    return;
  }
  const int M = (mx == ZE) ? 0 : mx;
  const int q = (nt + NT - 1) / NT;
  const int i0 = min(nt, c.tid * q), i1 = min(nt, i0 + q);
  const double L1 = c.pwd[1];
  double f = 0.0, g = 0.0;
  for (int i = i0; i < i1; ++i) f = fma(f, L1, Fm[i] * pow2d(max(Fe[i] - M, -1100)));
  for (int i = i1 - 1; i >= i0; --i) g = fma(g, L1, Bm[i] * pow2d(max(Be[i] - M, -1100)));
  int sF = i1 - i0, sG = i1 - i0;
  double F = f, G = g;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double uf = __shfl_up_sync(FULL, F, d);
    const int us = __shfl_up_sync(FULL, sF, d);
    const double dg = __shfl_down_sync(FULL, G, d);
    const int ds = __shfl_down_sync(FULL, sG, d);
    if (lane >= d) { F = fma(uf, c.pwd[sF], F); sF += us; }
    if (lane + d < 32) { G = fma(dg, c.pwd[sG], G); sG += ds; }
  }
  double eF = __shfl_up_sync(FULL, F, 1);
  int esF = __shfl_up_sync(FULL, sF, 1);
  double eG = __shfl_down_sync(FULL, G, 1);
  int esG = __shfl_down_sync(FULL, sG, 1);
  if (lane == 0) { eF = 0.0; esF = 0; }
  if (lane == 31) { eG = 0.0; esG = 0; }
  double* wF = c.redm;
  double* wG = c.redm + 64;
  int* wFs = c.rede + 128;
  int* wGs = c.rede + 192;
  if (lane == 31) { wF[warp] = F; wFs[warp] = sF; }
  if (lane == 0) { wG[warp] = G; wGs[warp] = sG; }
  __syncthreads();
  // carries from the other warps: every warp scans the NW warp totals across its lanes
  // (lane j <-> warp j; 5 shuffle levels instead of a serial loop over the warps)
  double xF = 0.0, xG = 0.0;
  int xsF = 0, xsG = 0;
  if (lane < c.NW) { xF = wF[lane]; xsF = wFs[lane]; xG = wG[lane]; xsG = wGs[lane]; }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    if (d >= c.NW) break;
    const double uf = __shfl_up_sync(FULL, xF, d);
    const int us = __shfl_up_sync(FULL, xsF, d);
    const double dg = __shfl_down_sync(FULL, xG, d);
    const int ds = __shfl_down_sync(FULL, xsG, d);
    if (lane >= d) { xF = fma(uf, c.pwd[xsF], xF); xsF += us; }
    if (lane + d < 32) { xG = fma(dg, c.pwd[xsG], xG); xsG += ds; }
  }
  // exclusive: the warps before (after) this one
  const double cw = warp > 0 ? __shfl_sync(FULL, xF, warp - 1) : 0.0;
  const double cg = warp + 1 < c.NW ? __shfl_sync(FULL, xG, warp + 1) : 0.0;
  double cf = fma(cw, c.pwd[esF], eF);
  double cb = fma(cg, c.pwd[esG], eG);
  for (int i = i0; i < i1; ++i) {
    const double t = Fm[i] * pow2d(max(Fe[i] - M, -1100));
    const ER<double> o = er_norm<double>(cf, M);
    Fm[i] = o.m; Fe[i] = o.e;
    cf = fma(cf, L1, t);
  }
  for (int i = i1 - 1; i >= i0; --i) {
    const double t = Bm[i] * pow2d(max(Be[i] - M, -1100));
    const ER<double> o = er_norm<double>(cb, M);
    Bm[i] = o.m; Be[i] = o.e;
    cb = fma(cb, L1, t);
  }
  // range totals: the forward one is the inclusive value at the last warp's end (every
  // warp has it: lane NW-1 of the cross-warp scan), the backward one at warp 0's start
  totF = er_norm<double>(__shfl_sync(FULL, xF, c.NW - 1), M);
  totB = er_norm<double>(__shfl_sync(FULL, xG, 0), M);
}

// Deterministic block sum (fixed tree) of per-tile ER values vm/ve[0..nt).
__device__ __forceinline__ ER<double> block_er_sum(Ctx& c, const double* vm, const int* ve) {
  const int nt = c.nt, NT = c.NT;
  const int q = (nt + NT - 1) / NT;
  const int i0 = min(nt, c.tid * q), i1 = min(nt, i0 + q);
  ER<double> s = er_zero<double>();
  for (int i = i0; i < i1; ++i) s = er_add(s, ER<double>{vm[i], ve[i]});
  s = warp_er_sum(s);
  __syncthreads();
  if (c.lane == 0) { c.redm[c.warp] = s.m; c.rede[c.warp] = s.e; }
  __syncthreads();
  ER<double> t = er_zero<double>();
  for (int w = 0; w < c.NW; ++w) t = er_add(t, ER<double>{c.redm[w], c.rede[w]});
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------- external carries
// Warp 0: the other ranges' totals (slot par), each decayed by the precomputed
// lambda^{256 d_k} to this range's boundary, summed in a fixed order.
constexpr int GLANE = 8;  // ranges per lane in the warp-0 folds (G <= 256, checked by the plan)
// Every thread decays at most one other range's totals (range k = tid, G <= NT); the
// per-warp sums are folded by warp 0 in warp order (fixed order: deterministic).
__device__ __forceinline__ void ext_carries_cta(Ctx& c, const StreamParams& P, int par, double* wm, int* we) {
  const double* gt = P.gtot + (size_t)par * P.G * 4;
  const int* ge = P.gtote + (size_t)par * P.G * 4;
  ER<double> f = er_zero<double>(), b = er_zero<double>();
  const int k = c.tid;
  if (k < P.G && k != c.r) {
    const ER<double> dp{c.dpm[k], c.dpe[k]};
    if (k < c.r) f = er_mul(dp, ER<double>{__ldcg(gt + 4 * k), __ldcg(ge + 4 * k)});
    else b = er_mul(dp, ER<double>{__ldcg(gt + 4 * k + 1), __ldcg(ge + 4 * k + 1)});
  }
  f = warp_er_sum(f);
  b = warp_er_sum(b);
  if (c.lane == 0) {
    wm[2 * c.warp] = f.m; we[2 * c.warp] = f.e;
    wm[2 * c.warp + 1] = b.m; we[2 * c.warp + 1] = b.e;
  }
}
// tiles between range k and this range r (the decay distance of k's total)
__device__ __forceinline__ long long range_gap(const StreamParams& P, int k, int r) {
  return k < r ? range_T0(P, r) - range_T0(P, k + 1) : range_T0(P, k) - range_T0(P, r + 1);
}

// [A]: full per-tile carries of the consumed vector x (tables F/B, exponents Xx).
__device__ __forceinline__ void tile_carries(Ctx& c, const StreamParams& P, int par, const double* Fm, const int* Fe,
                             const double* Bm, const int* Be, const int* Xx, unsigned long long* td = nullptr) {
  ext_carries_cta(c, P, par, c.redm + 64, c.rede + 64);
  __syncthreads();
  if (td) td[4] = gtimer();
  if (c.warp == 0) {
    ER<double> F = er_zero<double>(), B = er_zero<double>();
    if (c.lane < c.NW) {
      F = ER<double>{c.redm[64 + 2 * c.lane], c.rede[64 + 2 * c.lane]};
      B = ER<double>{c.redm[64 + 2 * c.lane + 1], c.rede[64 + 2 * c.lane + 1]};
    }
    F = warp_er_sum(F);
    B = warp_er_sum(B);
    if (c.lane == 0) {
      c.redm[0] = F.m; c.rede[0] = F.e;
      c.redm[1] = B.m; c.rede[1] = B.e;
    }
  }
  __syncthreads();
  if (td) td[5] = gtimer();
  const ER<double> CFx{c.redm[0], c.rede[0]}, CBx{c.redm[1], c.rede[1]};
  for (int i = c.tid; i < c.nt; i += c.NT) {
    const ER<double> CF = er_fma(pw(c, i), CFx, ER<double>{Fm[i], Fe[i]});
    const ER<double> CB = er_fma(pw(c, c.nt - 1 - i), CBx, ER<double>{Bm[i], Be[i]});
    const int X = Xx[i];
    int R = X;
    if (X == ZE || CF.e - X > LIM || CB.e - X > LIM) R = max(CF.e, CB.e);
    if (R == ZE) R = 0;
    c.cfr[i] = er_rel(CF, R);
    c.cbr[i] = er_rel(CB, R);
    c.Rr[i] = R;
  }
  __syncthreads();
}

// After the grid barrier: thread k reads range k's published (totals, error share, flag)
// of slot `par` (all loads in flight at once) and decays the other ranges' totals by the
// precomputed lambda^{256 d_k}; per-warp partial sums go through shared memory (one block
// synchronisation); then every warp folds them in the same fixed order (identical values
// in all warps: the external carries, the error sum, the OR of the flags) and forms the
// full carries of its own tiles of the consumed vector (tables F/B hold its local
// exclusive carries, Xx its tile exponents) for the next stream_half, with no second
// block synchronisation.
__device__ __forceinline__ void warp_step_in(Ctx& c, const StreamParams& P, int par, const double* Fm, const int* Fe,
                                             const double* Bm, const int* Be, const int* Xx, double& err,
                                             int& flag) {
  const double* gt = P.gtot + (size_t)par * P.G * 4;
  const int* ge = P.gtote + (size_t)par * P.G * 4;
  ER<double> f = er_zero<double>(), b = er_zero<double>();
  double es = 0.0;
  int fl = 0;
  const int k = c.tid;
  if (k < P.G) {
    es = __ldcg(gt + 4 * k + 2);
    fl = __ldcg(ge + 4 * k + 2);
    if (k != c.r) {
      const ER<double> dp{c.dpm[k], c.dpe[k]};
      if (k < c.r) f = er_mul(dp, ER<double>{__ldcg(gt + 4 * k), __ldcg(ge + 4 * k)});
      else b = er_mul(dp, ER<double>{__ldcg(gt + 4 * k + 1), __ldcg(ge + 4 * k + 1)});
    }
  }
  f = warp_er_sum(f);
  b = warp_er_sum(b);
  es = warp_sum(es);
  fl = __reduce_or_sync(FULL, (unsigned)fl);
  double* wm = c.redm + 700;  // scratch used by nothing else in the solve loop
  int* we = c.rede + 700;
  if (c.lane == 0) {
    wm[3 * c.warp] = f.m; we[3 * c.warp] = f.e;
    wm[3 * c.warp + 1] = b.m; we[3 * c.warp + 1] = b.e;
    wm[3 * c.warp + 2] = es; we[3 * c.warp + 2] = fl;
  }
  __syncthreads();
  // lane j takes warp j's partials; fixed-tree warp sums (the same in every warp)
  ER<double> xf = er_zero<double>(), xb = er_zero<double>();
  double xs = 0.0;
  int xl = 0;
  if (c.lane < c.NW) {
    const int j = c.lane;
    xf = ER<double>{wm[3 * j], we[3 * j]};
    xb = ER<double>{wm[3 * j + 1], we[3 * j + 1]};
    xs = wm[3 * j + 2];
    xl = we[3 * j + 2];
  }
  const ER<double> CFx = warp_er_sum(xf), CBx = warp_er_sum(xb);
  err = warp_sum(xs);
  flag = __reduce_or_sync(FULL, (unsigned)xl);
  // full carries of this warp's tiles: lambda^{256 i} CFx + local exclusive carry (and
  // the backward mirror), formed directly relative to the tile's reference exponent R
  // in plain fp64 (integer exponent arithmetic, no extended-range normalisation): the
  // two terms are m 2^e with m < 4; R = the tile exponent X unless an upper bound of a
  // carry's exponent exceeds X + LIM (then R = that bound).
  const bool fz = !(CFx.m > 0.0), bz = !(CBx.m > 0.0);
  for (int i = c.warp + c.lane * c.NW; i < c.nt; i += 32 * c.NW) {
    const int j = c.nt - 1 - i;
    const double fa = c.pwm[i] * CFx.m, ba = c.pwm[j] * CBx.m;
    const int efa = fz ? ZE : c.pwe[i] + CFx.e, eba = bz ? ZE : c.pwe[j] + CBx.e;
    const double fb = Fm[i], bb = Bm[i];
    const int efb = fb > 0.0 ? Fe[i] : ZE, ebb = bb > 0.0 ? Be[i] : ZE;
    const int EF = max(efa, efb), EB = max(eba, ebb);
    const int X = Xx[i];
    int R = X;
    if (X == ZE || EF + 2 - X > LIM || EB + 2 - X > LIM) R = max(EF, EB) + 2;
    if (R <= ZE + 2) R = 0;
    c.cfr[i] = fa * pow2d(max(efa - R, -1100)) + fb * pow2d(max(efb - R, -1100));
    c.cbr[i] = ba * pow2d(max(eba - R, -1100)) + bb * pow2d(max(ebb - R, -1100));
    c.Rr[i] = R;
  }
  __syncwarp();
}

// ---------------------------------------------------------------- streamed half-step
struct HalfArgs {
  const double* xg;  // consumed mantissas
  const int* Xx;     // consumed tile exponents
  const double* tg;  // target mantissas (a or b)
  const int* Xt;
  const double* og;  // psi^(l) for the check (CHECK)
  const int* Xo;
  double* yg;        // produced mantissas (WRITE)
  int* Xy;
  double *yFm, *yBm;
  int *yFe, *yBe;
  const unsigned char* tz;  // per-tile "target has a zero entry" flags
};

// DIV: y = tgt / Kx (solve) else y = Kx (apply); CHECK: accumulate the marginal
// error sum |psi_old (Kx) - tgt| per tile; WRITE: produce y.
// Each warp streams the tiles i = warp, warp + NW, ... of this range through its
// S-stage ring; y overwrites x in the stage and leaves by TMA bulk store; a stage
// is refilled (S - 1 tiles ahead) once the store of its previous tile has read it.
// Prefetch: `pre` = the first S-1 tiles of this half-step were already issued by the
// previous call; (nx, nt_) != null = issue the next half-step's first S-1 tiles
// (x = the y this warp just produced, target nt_) before the grid barrier.
template <int NW, int S, bool DIV, bool CHECK, bool WRITE>
__device__ __forceinline__ void stream_half(Ctx& c, const StreamParams& P, const HalfArgs& A, int& nonfinite,
                                            bool pre = false, const double* nx = nullptr,
                                            const double* ntg = nullptr) {
  const int lane = c.lane, w = c.warp;
  const long long gbase = (long long)c.T0 * TILE;
  double* stg = c.stage + (size_t)w * S * 2 * TILE;
  uint64_t* mb = c.mbar + w * S;
  constexpr bool LOADT = DIV || CHECK;
  const double lam = P.lam;
  const double lp = P.lanepow[lane], rp = P.lanepow[31 - lane];

  auto issue = [&](int k) {  // lane 0
    const int i = w + k * NW;
    if (i >= c.nt) return;
    const int s = k % S;
    mbar_expect_tx(&mb[s], LOADT ? 2 * TBYTES : TBYTES);
    bulk_g2s(stg + (s * 2) * TILE, A.xg + gbase + (long long)i * TILE, TBYTES, &mb[s]);
    if (LOADT) bulk_g2s(stg + (s * 2 + 1) * TILE, A.tg + gbase + (long long)i * TILE, TBYTES, &mb[s]);
  };
  if (lane == 0 && !pre) {
    fence_async();
#pragma unroll
    for (int k = 0; k < S - 1; ++k) issue(k);
  }
  int bad = 0;
  int k = 0;
  for (int i = w; i < c.nt; i += NW, ++k) {
    const int s = k % S;
    double* xs = stg + (s * 2) * TILE;
    mbar_wait(&mb[s], (c.phase >> s) & 1u);
    c.phase ^= (1u << s);
    double xv[E], tv[E];
    lds_tile(xs, lane, xv);
    if (LOADT) lds_tile(xs + TILE, lane, tv);
    double ov[E];
    if (CHECK) ldg_tile(A.og + gbase + (long long)i * TILE, lane, ov);

    const int X = A.Xx[i];
    const int R = c.Rr[i];
    if (X != R) {  // carries far above the tile: compute relative to 2^R (warp-uniform)
      const double sc = pow2d(max(X - R, -1100));
#pragma unroll
      for (int e = 0; e < E; ++e) xv[e] *= sc;
    }
    // carries into this lane's chunk: intra-tile exclusive scan + decayed tile carries
    double Fi, Gi;
    tile_scan_lanes(P, lane, xv, Fi, Gi);
    const double cf = fma(lp, c.cfr[i], prev_or0(Fi));
    const double cb = fma(rp, c.cbr[i], next_or0(Gi));
    // forward recursion p_k = lam p_{k-1} + x_k (Alg. 1 line 5 / 10)
    double pf[E];
    double p = cf;
#pragma unroll
    for (int e = 0; e < E; ++e) { p = fma(lam, p, xv[e]); pf[e] = p; }
    // backward recursion t_k = lam t_{k+1} + x_k, K x = p + lam t_{k+1} (line 6 / 11),
    // fused with the update y = tgt / (K x) (line 7 / 12); y overwrites tv
    double tn = cb;
    double errp = 0.0;
    double sce = 0.0;
    if (CHECK) sce = pow2d(min(max(A.Xo[i] + R - A.Xt[i], -1100), 1000));
    const bool guard = DIV && A.tz[i];  // zero targets: y = 0 exactly (warp-uniform)
    unsigned zm = 0;  // FS1_K2_SELHOIST: the zero targets of a guarded tile, zeroed after the loop
    if (FS1_K2_SELHOIST && guard) {
#pragma unroll
      for (int e = 0; e < E; ++e) zm |= (unsigned)!(tv[e] > 0.0) << e;
    }
#pragma unroll
    for (int e = E - 1; e >= 0; --e) {
      const double kx = fma(lam, tn, pf[e]);
      tn = fma(lam, tn, xv[e]);
      if (CHECK) errp += fabs(fma(ov[e] * sce, kx, -tv[e]));
      if (WRITE) {
        if (DIV) {
          // branch-free: the quotient always, a select for the zero targets of a guarded
          // tile (the nested conditional compiled to two branches and two copies of the
          // division per point)
          const double q = fdiv(tv[e], kx);
          tv[e] = FS1_K2_SELHOIST ? q : ((guard && !(tv[e] > 0.0)) ? 0.0 : q);
        }
        else tv[e] = kx;
      }
    }
    if (FS1_K2_SELHOIST && DIV && WRITE && guard) {  // warp-uniform, rare
#pragma unroll
      for (int e = 0; e < E; ++e)
        if ((zm >> e) & 1u) tv[e] = 0.0;
    }
    if (CHECK) {
      const double es = warp_sum(errp);
      if (lane == 0) c.errt[i] = ldexp(es, A.Xt[i]);
    }
    if (WRITE) {
      // exact power-of-two renormalisation of the output tile: the largest high word
      // of the (non-negative) doubles gives the tile's top binary exponent
      int hm = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) hm = max(hm, __double2hiint(tv[e]));
      hm = warp_max(hm);
      const int base = DIV ? (A.Xt[i] == ZE ? ZE : A.Xt[i] - R) : R;
      int Y = ZE;
      if (hm >= 0x00100000 && base != ZE) {
        const int M = min(max((hm >> 20) - 1023, -1020), 1020);
        const double sc = pow2d(-M);
#pragma unroll
        for (int e = 0; e < E; ++e) tv[e] *= sc;
        Y = base + M;
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) tv[e] = 0.0;
      }
      double FiY, GiY;
      if (FS1_K2_REDTOT) tile_totals_lanes(P, lp, rp, tv, FiY, GiY);
      else tile_scan_lanes(P, lane, tv, FiY, GiY);
      if (!isfinite(FiY + GiY)) bad = 1;
      put_totals(lane, FiY, GiY, Y, A.yFm, A.yFe, A.yBm, A.yBe, i);
      if (lane == 0) A.Xy[i] = Y;
      // y overwrites x in this stage (each lane rewrites only the chunks it read)
      sts_tile(xs, lane, tv);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(A.yg + gbase + (long long)i * TILE, xs, TBYTES);
        bulk_commit();
      }
    } else {
      __syncwarp();
    }
    if (lane == 0) {
      // refill the previous tile's stage once its store has read it
      if (WRITE) bulk_wait_read1();
      issue(k + S - 1);
    }
  }
  if (WRITE && lane == 0) bulk_wait_all();
  if (nx && lane == 0) {  // next half-step: same tiles of this warp, stages 0..S-2
    fence_async();
#pragma unroll
    for (int k2 = 0; k2 < S - 1; ++k2) {
      const int i = w + k2 * NW;
      if (i >= c.nt) break;
      mbar_expect_tx(&mb[k2], 2 * TBYTES);
      bulk_g2s(stg + (k2 * 2) * TILE, nx + gbase + (long long)i * TILE, TBYTES, &mb[k2]);
      bulk_g2s(stg + (k2 * 2 + 1) * TILE, ntg + gbase + (long long)i * TILE, TBYTES, &mb[k2]);
    }
  }
  if (__any_sync(FULL, bad)) nonfinite = 1;
}

// Wait out prefetched loads that will not be consumed (the solve stops).
template <int NW, int S>
__device__ __forceinline__ void drain_prefetch(Ctx& c) {
  uint64_t* mb = c.mbar + c.warp * S;
  for (int k = 0; k < S - 1; ++k) {
    if (c.warp + k * NW >= c.nt) break;
    mbar_wait(&mb[k], (c.phase >> k) & 1u);
    c.phase ^= (1u << k);
  }
}

// ---------------------------------------------------------------- prologue/epilogue
// Convert a user vector (linear, log, or the constant init) of tile i into
// mantissas + tile exponent, write the mantissas, return them in registers.
__device__ __forceinline__ void to_tile(const Ctx& c, const StreamParams& P, const double* src, int kind, double init,
                        double* dst, int i, double (&m)[E], int& X) {
  // kind: 0 linear, 1 log, 2 constant init
  const int lane = c.lane;
  const long long g0 = ((long long)c.T0 + i) * TILE + lane * E;
  double v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool ok = g0 + e < P.n;
    if (kind == 2) v[e] = ok ? init : 0.0;
    else v[e] = ok ? __ldcg(src + g0 + e) : (kind == 1 ? -INFINITY : 0.0);
  }
  if (kind == 1) {
    double M = -INFINITY;
#pragma unroll
    for (int e = 0; e < E; ++e) M = fmax(M, v[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(FULL, M, o));
    if (M == -INFINITY) {
      X = ZE;
#pragma unroll
      for (int e = 0; e < E; ++e) m[e] = 0.0;
    } else if (!isfinite(M)) {
      X = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) m[e] = NAN;
    } else {
      X = (int)floor(M * INV_LN2);
      const double xh = (double)X * LN2_HI, xl = (double)X * LN2_LO;
#pragma unroll
      for (int e = 0; e < E; ++e) m[e] = (v[e] == -INFINITY) ? 0.0 : exp((v[e] - xh) - xl);
    }
  } else {
    double M = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) M = fmax(M, v[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(FULL, M, o));
    if (!(M > 0.0)) {
      X = ZE;
#pragma unroll
      for (int e = 0; e < E; ++e) m[e] = 0.0;
    } else {
      X = expo_d(M);
      const double s1 = pow2d(-(X / 2)), s2 = pow2d(-(X - X / 2));
#pragma unroll
      for (int e = 0; e < E; ++e) m[e] = (v[e] * s1) * s2;
    }
  }
  stg_tile(dst + ((long long)c.T0 + i) * TILE, lane, m);
}

__device__ __forceinline__ void from_tile(const Ctx& c, const StreamParams& P, const double* srcm, int X, bool logd,
                          double* dst, int i) {
  const int lane = c.lane;
  double m[E];
  ldg_tile(srcm + ((long long)c.T0 + i) * TILE, lane, m);
  const long long g0 = ((long long)c.T0 + i) * TILE + lane * E;
  const double xh = (double)X * LN2_HI, xl = (double)X * LN2_LO;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (g0 + e < P.n) {
      double o;
      if (logd) o = (m[e] > 0.0 && X != ZE) ? (log(m[e]) + xl) + xh : (m[e] == 0.0 ? -INFINITY : NAN);
      else o = (X == ZE) ? 0.0 : ldexp(m[e], X);
      dst[g0 + e] = o;
    }
  }
}

// Convert a user vector into a state buffer with its tile exponents and scan totals.
__device__ __forceinline__ void load_vector(Ctx& c, const StreamParams& P, const double* src, int kind, double init,
                            double* dst, int* Xt, double* Fm, int* Fe, double* Bm, int* Be,
                            unsigned char* tz = nullptr) {
  for (int i = c.warp; i < c.nt; i += c.NW) {
    double m[E];
    int X;
    to_tile(c, P, src, kind, init, dst, i, m, X);
    if (c.lane == 0) Xt[i] = X;
    if (tz) {
      bool z = false;
#pragma unroll
      for (int e = 0; e < E; ++e) z |= !(m[e] > 0.0);
      z = __any_sync(FULL, z);
      if (c.lane == 0) tz[i] = z ? 1 : 0;
    }
    if (Fm) {
      double Fi, Gi;
      tile_scan_lanes(P, c.lane, m, Fi, Gi);
      put_totals(c.lane, Fi, Gi, X, Fm, Fe, Bm, Be, i);
    }
  }
}

// ---------------------------------------------------------------- cost phase
// Return line: h sum_k phi_k (P'_k + Q'_k) with the Jordan-block
// recursions P'_k = lam (P'_{k-1} + p_{k-1}), Q'_k = lam (Q'_{k+1} + t_{k+1}) over psi
// (R7), as a grid-wide scan of the pairs (p, P') and (t, Q').
struct Pair {
  ER<double> a, b;  // (p, P') or (t, Q')
};
// combine(A left/near, B right/far) over span L (points) of the far part: forward
// (p, P'): p = l^L pA + pB, P' = l^L (P'A + L pA) + P'B; backward is the mirror image.
__device__ __forceinline__ Pair pcomb(Pair A, Pair B, ER<double> lL, double L) {
  Pair r;
  r.a = er_fma(A.a, lL, B.a);
  r.b = er_fma(er_add(A.b, er_scale(A.a, L)), lL, B.b);
  return r;
}
__device__ __forceinline__ Pair pzero() { return Pair{er_zero<double>(), er_zero<double>()}; }
__device__ __forceinline__ Pair shfl_up_pair(Pair x, int d) { return Pair{shfl_up_er(x.a, d), shfl_up_er(x.b, d)}; }
__device__ __forceinline__ Pair shfl_down_pair(Pair x, int d) {
  return Pair{shfl_down_er(x.a, d), shfl_down_er(x.b, d)};
}

// lane-level Jordan aggregates and warp scans in plain fp64 relative to the tile exponent
__device__ __forceinline__ void jordan_lanes(const StreamParams& P, int lane, const double (&v)[E],
                                             double& fp, double& fP, double& bt, double& bQ) {
  const double lam = P.lam;
  double p = 0, Pp = 0, t = 0, Q = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) { Pp = lam * (Pp + p); p = fma(lam, p, v[e]); }
#pragma unroll
  for (int e = E - 1; e >= 0; --e) { Q = lam * (Q + t); t = fma(lam, t, v[e]); }
  fp = p; fP = Pp; bt = t; bQ = Q;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int d = 1 << k;
    const double L = (double)(E << k), l = P.lvd[k];
    const double up = __shfl_up_sync(FULL, fp, d), uP = __shfl_up_sync(FULL, fP, d);
    const double dt = __shfl_down_sync(FULL, bt, d), dQ = __shfl_down_sync(FULL, bQ, d);
    if (lane >= d) { fP = fma(l, fma(L, up, uP), fP); fp = fma(l, up, fp); }
    if (lane + d < 32) { bQ = fma(l, fma(L, dt, dQ), bQ); bt = fma(l, dt, bt); }
  }
}

__device__ __forceinline__ void block_pair_scan(Ctx& c, double* Am, int* Ae, double* A2m, int* A2e, double* Bm, int* Be,
                                double* B2m, int* B2e, Pair& totF, Pair& totB) {
  const int nt = c.nt, NT = c.NT, lane = c.lane, warp = c.warp;
  const int q = (nt + NT - 1) / NT;
  const int i0 = min(nt, c.tid * q), i1 = min(nt, i0 + q);
  const ER<double> L1 = pw(c, 1);
  Pair f = pzero(), g = pzero();
  for (int i = i0; i < i1; ++i)
    f = pcomb(f, Pair{ER<double>{Am[i], Ae[i]}, ER<double>{A2m[i], A2e[i]}}, L1, (double)TILE);
  for (int i = i1 - 1; i >= i0; --i)
    g = pcomb(g, Pair{ER<double>{Bm[i], Be[i]}, ER<double>{B2m[i], B2e[i]}}, L1, (double)TILE);
  int sF = i1 - i0, sG = i1 - i0;
  Pair F = f, G = g;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Pair uf = shfl_up_pair(F, d);
    const int us = __shfl_up_sync(FULL, sF, d);
    const Pair dg = shfl_down_pair(G, d);
    const int ds = __shfl_down_sync(FULL, sG, d);
    if (lane >= d) { F = pcomb(uf, F, pw(c, sF), (double)TILE * sF); sF += us; }
    if (lane + d < 32) { G = pcomb(dg, G, pw(c, sG), (double)TILE * sG); sG += ds; }
  }
  Pair eF = shfl_up_pair(F, 1), eG = shfl_down_pair(G, 1);
  int esF = __shfl_up_sync(FULL, sF, 1), esG = __shfl_down_sync(FULL, sG, 1);
  if (lane == 0) { eF = pzero(); esF = 0; }
  if (lane == 31) { eG = pzero(); esG = 0; }
  double* wm = c.redm;  // [4][64]
  int* we = c.rede;     // [4][64] + spans [2][64] at 256
  __syncthreads();
  if (lane == 31) {
    wm[warp] = F.a.m; we[warp] = F.a.e; wm[64 + warp] = F.b.m; we[64 + warp] = F.b.e;
    we[256 + warp] = sF;
  }
  if (lane == 0) {
    wm[128 + warp] = G.a.m; we[128 + warp] = G.a.e; wm[192 + warp] = G.b.m; we[192 + warp] = G.b.e;
    we[320 + warp] = sG;
  }
  __syncthreads();
  Pair cw = pzero(), cg = pzero();
  for (int w = 0; w < warp; ++w)
    cw = pcomb(cw, Pair{ER<double>{wm[w], we[w]}, ER<double>{wm[64 + w], we[64 + w]}}, pw(c, we[256 + w]),
               (double)TILE * we[256 + w]);
  for (int w = c.NW - 1; w > warp; --w)
    cg = pcomb(cg, Pair{ER<double>{wm[128 + w], we[128 + w]}, ER<double>{wm[192 + w], we[192 + w]}},
               pw(c, we[320 + w]), (double)TILE * we[320 + w]);
  Pair cf = pcomb(cw, eF, pw(c, esF), (double)TILE * esF);
  Pair cb = pcomb(cg, eG, pw(c, esG), (double)TILE * esG);
  for (int i = i0; i < i1; ++i) {
    const Pair t{ER<double>{Am[i], Ae[i]}, ER<double>{A2m[i], A2e[i]}};
    Am[i] = cf.a.m; Ae[i] = cf.a.e; A2m[i] = cf.b.m; A2e[i] = cf.b.e;
    cf = pcomb(cf, t, L1, (double)TILE);
  }
  for (int i = i1 - 1; i >= i0; --i) {
    const Pair t{ER<double>{Bm[i], Be[i]}, ER<double>{B2m[i], B2e[i]}};
    Bm[i] = cb.a.m; Be[i] = cb.a.e; B2m[i] = cb.b.m; B2e[i] = cb.b.e;
    cb = pcomb(cb, t, L1, (double)TILE);
  }
  __syncthreads();
  if (c.tid == NT - 1) { wm[0] = cf.a.m; we[0] = cf.a.e; wm[1] = cf.b.m; we[1] = cf.b.e; }
  if (c.tid == 0) { wm[2] = cb.a.m; we[2] = cb.a.e; wm[3] = cb.b.m; we[3] = cb.b.e; }
  __syncthreads();
  totF = Pair{ER<double>{wm[0], we[0]}, ER<double>{wm[1], we[1]}};
  totB = Pair{ER<double>{wm[2], we[2]}, ER<double>{wm[3], we[3]}};
  __syncthreads();
}

// cost of the state (Pm, Xp) = phi, (Qm, Xq) = psi; returns the value on every CTA.
template <int NW>
__device__ __forceinline__ double cost_phase(Ctx& c, const StreamParams& P, const double* Pm, const int* Xp,
                             const double* Qm, const int* Xq) {
  const int lane = c.lane;
  // tables: forward (p, P') in PF/PB, backward (t, Q') in QF/QB
  double *Am = c.PFm, *A2m = c.PBm, *Bm = c.QFm, *B2m = c.QBm;
  int *Ae = c.PFe, *A2e = c.PBe, *Be = c.QFe, *B2e = c.QBe;
  for (int i = c.warp; i < c.nt; i += NW) {
    double v[E];
    ldg_tile(Qm + ((long long)c.T0 + i) * TILE, lane, v);
    double fp, fP, bt, bQ;
    jordan_lanes(P, lane, v, fp, fP, bt, bQ);
    const int X = Xq[i];
    if (lane == 31) {
      ER<double> t = er_norm<double>(fp, X); Am[i] = t.m; Ae[i] = t.e;
      t = er_norm<double>(fP, X); A2m[i] = t.m; A2e[i] = t.e;
    }
    if (lane == 0) {
      ER<double> t = er_norm<double>(bt, X); Bm[i] = t.m; Be[i] = t.e;
      t = er_norm<double>(bQ, X); B2m[i] = t.m; B2e[i] = t.e;
    }
  }
  __syncthreads();
  Pair tF, tB;
  block_pair_scan(c, Am, Ae, A2m, A2e, Bm, Be, B2m, B2e, tF, tB);
  if (c.tid == 0) {
    double* g = P.gtot2 + (size_t)c.r * 8;
    int* ge = P.gtot2e + (size_t)c.r * 8;
    g[0] = tF.a.m; ge[0] = tF.a.e; g[1] = tF.b.m; ge[1] = tF.b.e;
    g[2] = tB.a.m; ge[2] = tB.a.e; g[3] = tB.b.m; ge[3] = tB.b.e;
  }
  grid_barrier(P.bar, P.G, c.gen);
  // external pair carries (warp 0): every other range's totals advanced over the gap
  // to this range (precomputed lambda^{256 d}), summed component-wise
  if (c.warp == 0) {
    Pair ef = pzero(), eb = pzero();
    for (int k = lane; k < P.G; k += 32) {
      if (k == c.r) continue;
      const double* g = P.gtot2 + (size_t)k * 8;
      const int* ge = P.gtot2e + (size_t)k * 8;
      const ER<double> dp{c.dpm[k], c.dpe[k]};
      const double L = (double)TILE * (double)range_gap(P, k, c.r);
      if (k < c.r) {
        const Pair t = pcomb(Pair{ER<double>{__ldcg(g), __ldcg(ge)}, ER<double>{__ldcg(g + 1), __ldcg(ge + 1)}},
                             pzero(), dp, L);
        ef.a = er_add(ef.a, t.a);
        ef.b = er_add(ef.b, t.b);
      } else {
        const Pair t = pcomb(Pair{ER<double>{__ldcg(g + 2), __ldcg(ge + 2)}, ER<double>{__ldcg(g + 3), __ldcg(ge + 3)}},
                             pzero(), dp, L);
        eb.a = er_add(eb.a, t.a);
        eb.b = er_add(eb.b, t.b);
      }
    }
    ef.a = warp_er_sum(ef.a);
    ef.b = warp_er_sum(ef.b);
    eb.a = warp_er_sum(eb.a);
    eb.b = warp_er_sum(eb.b);
    if (lane == 0) {
      c.redm[500] = ef.a.m; c.rede[500] = ef.a.e; c.redm[501] = ef.b.m; c.rede[501] = ef.b.e;
      c.redm[502] = eb.a.m; c.rede[502] = eb.a.e; c.redm[503] = eb.b.m; c.rede[503] = eb.b.e;
    }
  }
  __syncthreads();
  const Pair EF{ER<double>{c.redm[500], c.rede[500]}, ER<double>{c.redm[501], c.rede[501]}};
  const Pair EB{ER<double>{c.redm[502], c.rede[502]}, ER<double>{c.redm[503], c.rede[503]}};
  // full per-tile carries relative to R (in place: A/A2 <- forward, B/B2 <- backward)
  for (int i = c.tid; i < c.nt; i += c.NT) {
    const Pair cf = pcomb(EF, Pair{ER<double>{Am[i], Ae[i]}, ER<double>{A2m[i], A2e[i]}}, pw(c, i),
                          (double)TILE * i);
    const int sb = c.nt - 1 - i;
    const Pair cb = pcomb(EB, Pair{ER<double>{Bm[i], Be[i]}, ER<double>{B2m[i], B2e[i]}}, pw(c, sb),
                          (double)TILE * sb);
    const int X = Xq[i];
    const int mx = max(max(cf.a.e, cf.b.e), max(cb.a.e, cb.b.e));
    int R = X;
    if (X == ZE || mx - X > LIM) R = mx;
    if (R == ZE) R = 0;
    Am[i] = er_rel(cf.a, R); A2m[i] = er_rel(cf.b, R);
    Bm[i] = er_rel(cb.a, R); B2m[i] = er_rel(cb.b, R);
    c.Rr[i] = R;
  }
  __syncthreads();
  // per-tile weighted dot sum_k phi_k (P'_k + Q'_k)
  const double lam = P.lam;
  for (int i = c.warp; i < c.nt; i += NW) {
    double v[E], ph[E];
    ldg_tile(Qm + ((long long)c.T0 + i) * TILE, lane, v);
    ldg_tile(Pm + ((long long)c.T0 + i) * TILE, lane, ph);
    const int X = Xq[i], R = c.Rr[i];
    if (X != R) {
      const double sc = pow2d(max(X - R, -1100));
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] *= sc;
    }
    double fp, fP, bt, bQ;
    jordan_lanes(P, lane, v, fp, fP, bt, bQ);
    // lane-exclusive values
    double xp = __shfl_up_sync(FULL, fp, 1), xP = __shfl_up_sync(FULL, fP, 1);
    double xt = __shfl_down_sync(FULL, bt, 1), xQ = __shfl_down_sync(FULL, bQ, 1);
    if (lane == 0) { xp = 0; xP = 0; }
    if (lane == 31) { xt = 0; xQ = 0; }
    // combine with the tile carries over span 8 lane (forward) / 8 (31 - lane) (backward)
    const double Lf = (double)(E * lane), Lb = (double)(E * (31 - lane));
    const double lf = P.lanepow[lane], lb = P.lanepow[31 - lane];
    const double cp = Am[i], cP = A2m[i], ct = Bm[i], cQ = B2m[i];
    double p = fma(lf, cp, xp), Pp = fma(lf, fma(Lf, cp, cP), xP);
    double t = fma(lb, ct, xt), Q = fma(lb, fma(Lb, ct, cQ), xQ);
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) { Pp = lam * (Pp + p); p = fma(lam, p, v[e]); acc = fma(ph[e], Pp, acc); }
#pragma unroll
    for (int e = E - 1; e >= 0; --e) { Q = lam * (Q + t); t = fma(lam, t, v[e]); acc = fma(ph[e], Q, acc); }
    const double s = warp_sum(acc);
    if (lane == 0) {
      const ER<double> t2 = (Xp[i] == ZE) ? er_zero<double>() : er_norm<double>(s, R + Xp[i]);
      c.errt[i] = t2.m;
      c.Rr[i] = t2.e;
    }
  }
  __syncthreads();
  const ER<double> tot = block_er_sum(c, c.errt, c.Rr);
  if (c.tid == 0) {
    P.gtot2[(size_t)c.r * 8 + 4] = tot.m;
    P.gtot2e[(size_t)c.r * 8 + 4] = tot.e;
  }
  grid_barrier(P.bar, P.G, c.gen);
  // every CTA folds the G partials in the same fixed order
  ER<double> s = er_zero<double>();
  for (int k = lane; k < P.G; k += 32)
    s = er_add(s, ER<double>{__ldcg(P.gtot2 + (size_t)k * 8 + 4), __ldcg(P.gtot2e + (size_t)k * 8 + 4)});
  s = warp_er_sum(s);
  return (s.m == 0.0) ? 0.0 : ldexp(s.m, s.e) * P.h;
}

// ---------------------------------------------------------------- publish / read
__device__ __forceinline__ void publish(Ctx& c, const StreamParams& P, int slot, ER<double> F, ER<double> B, double errs,
                        int flag) {
  if (c.tid == 0) {
    double* g = P.gtot + ((size_t)slot * P.G + c.r) * 4;
    int* ge = P.gtote + ((size_t)slot * P.G + c.r) * 4;
    g[0] = F.m; ge[0] = F.e;
    g[1] = B.m; ge[1] = B.e;
    g[2] = errs; ge[2] = flag;
  }
}
// totals over ranges of slot: error sum (fixed order) and OR of flags (warp 0 result
// broadcast through shared memory)
__device__ __forceinline__ void read_slot(Ctx& c, const StreamParams& P, int slot, double& err, int& flag) {
  if (c.warp == 0) {
    double v[GLANE];
    int fl[GLANE];
#pragma unroll
    for (int j = 0; j < GLANE; ++j) {  // all loads first, then the fixed-order sum
      const int k = c.lane + 32 * j;
      v[j] = 0.0;
      fl[j] = 0;
      if (k < P.G) {
        v[j] = __ldcg(P.gtot + ((size_t)slot * P.G + k) * 4 + 2);
        fl[j] = __ldcg(P.gtote + ((size_t)slot * P.G + k) * 4 + 2);
      }
    }
    double s = 0.0;
    int f = 0;
#pragma unroll
    for (int j = 0; j < GLANE; ++j) {
      s += v[j];
      f |= fl[j];
    }
    s = warp_sum(s);
    f = __reduce_or_sync(FULL, (unsigned)f);
    if (c.lane == 0) { c.redm[510] = s; c.rede[510] = f; }
  }
  __syncthreads();
  err = c.redm[510];
  flag = c.rede[510];
  __syncthreads();
}

// ---------------------------------------------------------------- the kernel
template <int NW, int S>
__global__ void __launch_bounds__(32 * NW, 1) fs1_stream_kernel(const __grid_constant__ StreamParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  Ctx c;
  c.NW = NW;
  c.NT = 32 * NW;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  c.r = blockIdx.x;
  c.T0 = (int)range_T0(P, c.r);
  c.nt = (int)(range_T0(P, c.r + 1) - c.T0);
  const Layout L = layout(NW, S, P.ntmax, P.G);
  c.stage = reinterpret_cast<double*>(smem + L.stage);
  c.mbar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  c.dpm = reinterpret_cast<double*>(smem + L.dpm);
  c.dpe = reinterpret_cast<int*>(smem + L.dpe);
  c.tzA = smem + L.tza;
  c.tzB = smem + L.tzb;
  c.pwm = reinterpret_cast<double*>(smem + L.pwm);
  c.pwd = reinterpret_cast<double*>(smem + L.pwd);
  c.pwe = reinterpret_cast<int*>(smem + L.pwe);
  c.AX = reinterpret_cast<int*>(smem + L.ax);
  c.BX = reinterpret_cast<int*>(smem + L.bx);
  c.PX = reinterpret_cast<int*>(smem + L.px);
  c.QX0 = reinterpret_cast<int*>(smem + L.qx0);
  c.QX1 = reinterpret_cast<int*>(smem + L.qx1);
  c.PFm = reinterpret_cast<double*>(smem + L.pfm);
  c.PBm = reinterpret_cast<double*>(smem + L.pbm);
  c.QFm = reinterpret_cast<double*>(smem + L.qfm);
  c.QBm = reinterpret_cast<double*>(smem + L.qbm);
  c.PFe = reinterpret_cast<int*>(smem + L.pfe);
  c.PBe = reinterpret_cast<int*>(smem + L.pbe);
  c.QFe = reinterpret_cast<int*>(smem + L.qfe);
  c.QBe = reinterpret_cast<int*>(smem + L.qbe);
  c.cfr = reinterpret_cast<double*>(smem + L.cfr);
  c.cbr = reinterpret_cast<double*>(smem + L.cbr);
  c.Rr = reinterpret_cast<int*>(smem + L.rr);
  c.errt = reinterpret_cast<double*>(smem + L.errt);
  c.redm = reinterpret_cast<double*>(smem + L.redm);
  c.rede = reinterpret_cast<int*>(smem + L.rede);
  c.phase = 0;
  c.gen = 0;

  if (c.lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&c.mbar[c.warp * S + s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int k = c.tid; k <= P.ntmax; k += c.NT) {
    const ER<double> t = pow_tiles(P, k);
    c.pwm[k] = t.m;
    c.pwe[k] = t.e;
    c.pwd[k] = er_rel(t, 0);
  }
  for (int k = c.tid; k < P.G; k += c.NT) {  // decay from range k to this range
    const ER<double> t = (k == c.r) ? er_zero<double>() : pow_tiles(P, range_gap(P, k, c.r));
    c.dpm[k] = t.m;
    c.dpe[k] = t.e;
  }
  for (int i = c.tid; i < c.nt; i += c.NT) c.errt[i] = 0.0;
  __syncthreads();

  const double* dA = reinterpret_cast<const double*>(P.a);
  const double* dB = reinterpret_cast<const double*>(P.b);
  double* dU = reinterpret_cast<double*>(P.u);
  double* dV = reinterpret_cast<double*>(P.v);
  int nonfinite = 0;

  if (P.mode == MODE_APPLY) {
    load_vector(c, P, reinterpret_cast<const double*>(P.x), P.logd ? 1 : 0, 0.0, P.Pm, c.PX, c.PFm, c.PFe,
                c.PBm, c.PBe);
    __syncthreads();
    ER<double> tF, tB;
    block_tile_scan(c, c.PFm, c.PFe, c.PBm, c.PBe, tF, tB);
    publish(c, P, 0, tF, tB, 0.0, 0);
    grid_barrier(P.bar, P.G, c.gen);
    tile_carries(c, P, 0, c.PFm, c.PFe, c.PBm, c.PBe, c.PX);
    HalfArgs A{P.Pm, c.PX, nullptr, nullptr, nullptr, nullptr, P.Qm0, c.QX0,
               c.QFm, c.QBm, c.QFe, c.QBe, nullptr};
    stream_half<NW, S, false, false, true>(c, P, A, nonfinite);
    __syncthreads();
    fence_async();
    __syncthreads();
    for (int i = c.warp; i < c.nt; i += NW)
      from_tile(c, P, P.Qm0, c.QX0[i], P.logd, reinterpret_cast<double*>(P.y), i);
    return;
  }
  if (P.mode == MODE_COST) {
    load_vector(c, P, dU, P.logd ? 1 : 0, 0.0, P.Pm, c.PX, nullptr, nullptr, nullptr, nullptr);
    load_vector(c, P, dV, P.logd ? 1 : 0, 0.0, P.Qm0, c.QX0, nullptr, nullptr, nullptr, nullptr);
    __syncthreads();
    const double cost = cost_phase<NW>(c, P, P.Pm, c.PX, P.Qm0, c.QX0);
    if (c.r == 0 && c.tid == 0 && P.cost) P.cost[0] = cost;
    return;
  }

  // ---------------- solve (Algorithm 1)
  const int kin = P.input_is_log ? 1 : 0;
  load_vector(c, P, dA, kin, 0.0, P.Am, c.AX, nullptr, nullptr, nullptr, nullptr, c.tzA);
  load_vector(c, P, dB, kin, 0.0, P.Bm, c.BX, nullptr, nullptr, nullptr, nullptr, c.tzB);
  const double init = 1.0 / (double)P.n;  // phi0 = psi0 = 1/N
  load_vector(c, P, dU, P.warm ? 1 : 2, init, P.Pm, c.PX, c.PFm, c.PFe, c.PBm, c.PBe);
  load_vector(c, P, dV, P.warm ? 1 : 2, init, P.Qm0, c.QX0, nullptr, nullptr, nullptr, nullptr);
  __syncthreads();
  int par = 0;
  {
    ER<double> tF, tB;
    block_tile_scan(c, c.PFm, c.PFe, c.PBm, c.PBe, tF, tB);
    publish(c, P, par, tF, tB, 0.0, 0);
    grid_barrier(P.bar, P.G, c.gen);
  }
  const bool use_tol = P.tol > 0.0;
  int l = 0, qi = 0, flag = 0;
  bool pre = false;
  double errv = NAN;
  {
    double e;
    int f;
    warp_step_in(c, P, par, c.PFm, c.PFe, c.PBm, c.PBe, c.PX, e, f);
  }
  while (true) {
    const bool check = (l >= P.itr_max) || (use_tol && (l % P.check_interval) == 0);
    const bool last = l >= P.itr_max;
    // ---- lines 2-7: psi = b ./ (K^T phi), with the marginal error on check iterations
    unsigned long long* td = (P.tdbg && c.tid == 0 && l < 64) ? P.tdbg + ((size_t)c.r * 64 + l) * 8 : nullptr;
    if (td) td[0] = gtimer();
    const int qo = check ? (qi ^ 1) : qi;  // a checking step keeps psi^(l) in Qm[qi]
    double* Qi = qi ? P.Qm1 : P.Qm0;
    int* QXi = qi ? c.QX1 : c.QX0;
    double* Qo = qo ? P.Qm1 : P.Qm0;
    int* QXo = qo ? c.QX1 : c.QX0;
    HalfArgs A{P.Pm, c.PX, P.Bm, c.BX, Qi, QXi, Qo, QXo, c.QFm, c.QBm, c.QFe, c.QBe, c.tzB};
    nonfinite = 0;
    // a non-checking psi step is always followed by the phi step: prefetch its tiles
    if (!check) stream_half<NW, S, true, false, true>(c, P, A, nonfinite, pre, Qo, P.Am);
    else if (!last) stream_half<NW, S, true, true, true>(c, P, A, nonfinite, pre);
    else stream_half<NW, S, true, true, false>(c, P, A, nonfinite, pre);
    pre = !check;
    __syncthreads();
    if (td) td[1] = gtimer();
    if (td) td[2] = gtimer();
    {
      ER<double> tF = er_zero<double>(), tB = er_zero<double>();
      if (!last) block_tile_scan(c, c.QFm, c.QFe, c.QBm, c.QBe, tF, tB);
      if (td) td[5] = gtimer();
      double es = 0.0;
      if (check) {
        // deterministic per-range error sum
        const int q = (c.nt + c.NT - 1) / c.NT;
        const int i0 = min(c.nt, c.tid * q), i1 = min(c.nt, i0 + q);
        double sm = 0.0;
        for (int i = i0; i < i1; ++i) sm += c.errt[i];
        sm = warp_sum(sm);
        __syncthreads();
        if (c.lane == 0) c.redm[c.warp] = sm;
        __syncthreads();
        for (int w = 0; w < NW; ++w) es += c.redm[w];
        __syncthreads();
      }
      const int nf = __syncthreads_or(nonfinite);
      if (td) td[6] = gtimer();
      publish(c, P, par ^ 1, tF, tB, es, nf);
      if (td) td[3] = gtimer();
      grid_barrier(P.bar, P.G, c.gen);
      if (td) td[7] = gtimer();
      par ^= 1;
    }
    {
      double e;
      int f;
      // err / flags of this step and the carries of psi for the phi step (which reads
      // Qm[qo]: on a check that continues, qi flips to qo)
      warp_step_in(c, P, par, c.QFm, c.QFe, c.QBm, c.QBe, QXo, e, f);
      if (td) td[4] = gtimer();
      if (check) {
        errv = e;
        if (last || errv <= P.tol) {
          flag = (use_tol && errv <= P.tol) ? 1 : 4;
          break;
        }
        qi ^= 1;
      }
      if (f) {
        if (pre) drain_prefetch<NW, S>(c);
        ++l; flag = 2; break;
      }
    }
    // ---- lines 8-12: phi = a ./ (K psi)
    double* Qc = qi ? P.Qm1 : P.Qm0;
    int* QXc = qi ? c.QX1 : c.QX0;
    HalfArgs B{Qc, QXc, P.Am, c.AX, nullptr, nullptr, P.Pm, c.PX, c.PFm, c.PBm, c.PFe, c.PBe, c.tzA};
    nonfinite = 0;
    stream_half<NW, S, true, false, true>(c, P, B, nonfinite, pre, P.Pm, P.Bm);
    pre = true;  // the next psi step reads phi (just written) and b
    __syncthreads();
    {
      ER<double> tF, tB;
      block_tile_scan(c, c.PFm, c.PFe, c.PBm, c.PBe, tF, tB);
      const int nf = __syncthreads_or(nonfinite);
      publish(c, P, par ^ 1, tF, tB, 0.0, nf);
      grid_barrier(P.bar, P.G, c.gen);
      par ^= 1;
      double e;
      int f;
      warp_step_in(c, P, par, c.PFm, c.PFe, c.PBm, c.PBe, c.PX, e, f);
      ++l;  // line 13
      if (f) {
        drain_prefetch<NW, S>(c);
        flag = 2; break;
      }
    }
  }
  double* Qf = qi ? P.Qm1 : P.Qm0;
  int* QXf = qi ? c.QX1 : c.QX0;
  double cost = NAN;
  if (flag != 2) cost = cost_phase<NW>(c, P, P.Pm, c.PX, Qf, QXf);
  else errv = NAN;
  // outputs: F = log phi, G = log psi
  for (int i = c.warp; i < c.nt; i += NW) {
    from_tile(c, P, P.Pm, c.PX[i], true, dU, i);
    from_tile(c, P, Qf, QXf[i], true, dV, i);
  }
  if (c.r == 0 && c.tid == 0) {
    if (P.iters) P.iters[0] = l;
    if (P.err) P.err[0] = errv;
    if (P.flags) P.flags[0] = flag;
    if (P.cost) P.cost[0] = cost;
  }
}

}  // namespace stm
}  // namespace fs1
