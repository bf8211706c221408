// fs1_shard.cuh — K2s: one 1D FS-1 problem sharded over ranks (GPUs) by contiguous
// segments of whole 256-point tiles.
//
// Every K x of Algorithm 1 is the forward and backward recursion
// of Eq. "recursion" over the WHOLE grid, so a segment needs, per
// half-step, the recursion values entering it from the left (forward) and from the
// right (backward).  These depend on the other segments only through their totals:
// the forward total at a segment's end and the backward total at its start (2
// extended-range fp64 numbers per rank).  One half-step on rank r is therefore
//
//   [exchange]  all ranks' totals of x (4 doubles each, one all-gather over NVLink);
//   k_half      per tile: full carries = local exclusive tile carry (k_scan of the
//               previous call) + the other ranks' totals decayed over the gap; the
//               lane scan, both recursions, the update y = tgt / K x (PAPER.md:154 /
//               160), the marginal error on check iterations, an exact
//               power-of-two renormalisation of the tile, and y's tile totals;
//   k_scan      one CTA scans the tile totals of y: local exclusive carries for the
//               next half-step and the rank's totals of y (the next exchange).
//
// The state is mantissas with one binary exponent per tile (the log domain of
// DESIGN.md §5.3), fp64.  The return line runs the Jordan-block pair
// recursion (R7) the same way with 8-double pair totals per rank.
#pragma once
#include <math.h>
#include <stdint.h>

#include "fs1_common.cuh"
#include "fs1_params.h"
#include "fs1_stream.cuh"

namespace fs1 {
namespace shd {

constexpr int E = 8;
constexpr int TILE = 256;
constexpr int NW = 8;               // warps per CTA of the tile kernels
constexpr int LIM = 600;            // carries up to 2^LIM above a tile keep its exponent
constexpr int SCAN_NT = 1024;       // threads of the tile-scan CTA
constexpr double LN2 = 0.69314718055994530942;

// lambda^{256 k} (k >= 0 tiles) by binary decomposition of host-formed powers
__device__ __forceinline__ ER<double> powt(const ShardParams& P, long long k) {
  ER<double> r{1.0, 0};
  for (int j = 0; j < 40 && k; ++j, k >>= 1)
    if (k & 1) r = er_mul(r, ER<double>{P.t2m[j], P.t2e[j]});
  return r;
}
__device__ __forceinline__ ER<double> er_fma(ER<double> a, ER<double> b, ER<double> d) {
  return er_add(er_mul(a, b), d);
}

// Natural-order tile access: lane l holds points [8l, 8l+8) of the tile.  Loads go
// through L1 (each lane's 64-byte chunk is two sectors read by four 16-byte loads:
// L1 keeps the second load of each sector from going to L2 again).
__device__ __forceinline__ void ld_tile(const double* g, int lane, double (&v)[E]) {
  const double2* p = reinterpret_cast<const double2*>(g + lane * E);
#pragma unroll
  for (int j = 0; j < E / 2; ++j) {
    const double2 t = __ldca(p + j);
    v[2 * j] = t.x;
    v[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ void st_tile(double* g, int lane, const double (&v)[E]) {
  double2* p = reinterpret_cast<double2*>(g + lane * E);
#pragma unroll
  for (int j = 0; j < E / 2; ++j) p[j] = make_double2(v[2 * j], v[2 * j + 1]);
}

// lane Horner aggregates + 5-level warp scan (fp64 relative to the tile exponent):
// Fi = forward inclusive (lane 31: tile total at its end), Gi = backward inclusive
// (lane 0: tile total at its start)
__device__ __forceinline__ void lane_scan(const ShardParams& P, const double (&v)[E], double& Fi, double& Gi) {
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

// tile totals only (as K2's tile_totals_lanes): forward sum_l lambda^{8(31-l)} f_l at the
// tile end, backward sum_l lambda^{8l} g_l at its start, on every lane (lp = lambda^{8 lane},
// rp = lambda^{8(31-lane)})
__device__ __forceinline__ void lane_tot(const ShardParams& P, double lp, double rp, const double (&v)[E],
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

__device__ __forceinline__ void put_tot(const ShardParams& P, int lane, double Fi, double Gi, int X, int i,
                                        double* Fm, int* Fe, double* Bm, int* Be) {
  if (lane == 31) {
    const ER<double> t = er_norm<double>(Fi, X);
    Fm[i] = t.m;
    Fe[i] = t.e;
  }
  if (lane == 0) {
    const ER<double> t = er_norm<double>(Gi, X);
    Bm[i] = t.m;
    Be[i] = t.e;
  }
}

// ------------------------------------------------------------------ k_load
// Segment vector -> tiles of mantissas with one exponent per tile (+ tile totals).
// kind 0: linear weights, 1: log-weights, 2: the constant `init`.
__global__ void __launch_bounds__(32 * NW) k_load(const ShardParams P, const double* src, int kind, double init,
                                                  double* m, int* X, unsigned char* tz, double* Fm, int* Fe,
                                                  double* Bm, int* Be) {
  const int lane = threadIdx.x & 31;
  const long long wg = (long long)blockIdx.x * NW + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * NW;
  for (long long i = wg; i < P.T; i += nwarps) {
    double v[E];
    bool zero = false;
    double M = kind == 1 ? -INFINITY : 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const long long q = i * TILE + lane * E + e;  // segment point
      const bool valid = P.lo + q < P.n && q < P.len;
      double w = kind == 1 ? -INFINITY : 0.0;
      if (valid) w = kind == 2 ? init : __ldcg(src + q);
      v[e] = w;
      zero |= !valid || (kind == 1 ? !(w > -INFINITY) : !(w > 0.0));
      M = fmax(M, w);
    }
    double Mw = M;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mw = fmax(Mw, __shfl_xor_sync(FULL, Mw, o));
    int Xt;
    if (kind == 1) {
      if (!(Mw > -INFINITY)) {
        Xt = ZE;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = 0.0;
      } else if (!(Mw < INFINITY)) {  // +inf / NaN weight: poison (NONFINITE)
        Xt = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = NAN;
      } else {
        Xt = (int)floor(Mw / LN2);
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = exp(v[e] - (double)Xt * LN2);
      }
    } else {
      if (!(Mw > 0.0)) {
        Xt = ZE;
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = 0.0;
      } else {
        Xt = Tr<double>::expo(Mw);
        const double s = pow2d(-Xt);
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] *= s;
      }
    }
    st_tile(m + i * TILE, lane, v);
    if (lane == 0) X[i] = Xt;
    if (tz) {
      const unsigned any = __any_sync(FULL, zero);
      if (lane == 0) tz[i] = (unsigned char)any;
    }
    if (Fm) {
      double Fi, Gi;
      lane_scan(P, v, Fi, Gi);
      put_tot(P, lane, Fi, Gi, Xt, (int)i, Fm, Fe, Bm, Be);
    }
  }
}

// ------------------------------------------------------------------ scans
// Powers of the per-element multiplier L = lambda^{256 s}: table pw[j] = L^{2^j}
// (j < 32), powers by binary decomposition.
struct PowTab {
  const double* m;   // L^{2^j}, j < 32
  const int* e;
  const double* dm;  // optional direct table L^k, k < dn (shared memory)
  const int* de;
  int dn;
};
__device__ __forceinline__ ER<double> tpow(PowTab t, long long k) {
  if (k < t.dn) return ER<double>{t.dm[k], t.de[k]};
  ER<double> r{1.0, 0};
  for (int j = 0; j < 32 && k; ++j, k >>= 1)
    if (k & 1) r = er_mul(r, ER<double>{t.m[j], t.e[j]});
  return r;
}
constexpr int TBMAX = 512;  // tiles per block (the direct power table of k_half)

// Warp-level inclusive scans of (F, span) forward and (G, span) backward with
// multipliers tpow(span) (Hillis-Steele, 5 levels).
__device__ __forceinline__ void warp_pair_scan(PowTab t, int lane, ER<double>& F, int& sF, ER<double>& G,
                                               int& sG) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const ER<double> uf = shfl_up_er(F, d);
    const int us = __shfl_up_sync(FULL, sF, d);
    const ER<double> dg = shfl_down_er(G, d);
    const int ds = __shfl_down_sync(FULL, sG, d);
    // combined on every lane, kept by selects (branch-free scan levels)
    const ER<double> Fn = er_fma(uf, tpow(t, sF), F), Gn = er_fma(dg, tpow(t, sG), G);
    const bool tf = lane >= d, tb = lane + d < 32;
    F = ER<double>{tf ? Fn.m : F.m, tf ? Fn.e : F.e};
    sF += tf ? us : 0;
    G = ER<double>{tb ? Gn.m : G.m, tb ? Gn.e : G.e};
    sG += tb ? ds : 0;
  }
}

// One CTA (NTH threads): exclusive local carries over n elements in place,
//   CF_i = sum_{i'<i} L^{i-1-i'} F_i',  CB_i = sum_{i'>i} L^{i'-i-1} B_i'
// (L = lambda^{256 s}, s = tiles per element: 1 for tiles, TB for blocks), and the
// totals {F at the end, B at the start}.  Only the last element may be shorter
// (s_last tiles): no carry into an element crosses it, only the forward total does
// (and the backward total when n = 1), so the lane / warp combines use the uniform
// span and the per-element steps the element's own.  The per-warp totals are scanned
// by warp 0 (5 levels), not folded serially.
template <int NTH>
__device__ __forceinline__ void cta_scan(PowTab t, ER<double> Ll, int n, double* Fm, int* Fe, double* Bm, int* Be,
                                         ER<double>& totF, ER<double>& totB) {
  constexpr int NWP = NTH / 32;
  __shared__ double wFm[NWP], wGm[NWP];
  __shared__ int wFe[NWP], wGe[NWP], wFs[NWP], wGs[NWP];
  __shared__ double tm[2];
  __shared__ int te[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = (n + NTH - 1) / NTH;
  const int i0 = min(n, tid * q), i1 = min(n, i0 + q);
  const ER<double> L1{t.m[0], t.e[0]};
  ER<double> f = er_zero<double>(), g = er_zero<double>();
  for (int i = i0; i < i1; ++i) f = er_fma(f, L1, ER<double>{Fm[i], Fe[i]});
  for (int i = i1 - 1; i >= i0; --i) g = er_fma(g, L1, ER<double>{Bm[i], Be[i]});
  int sF = i1 - i0, sG = i1 - i0;
  ER<double> F = f, G = g;
  warp_pair_scan(t, lane, F, sF, G, sG);
  ER<double> eF = shfl_up_er(F, 1);
  int esF = __shfl_up_sync(FULL, sF, 1);
  ER<double> eG = shfl_down_er(G, 1);
  int esG = __shfl_down_sync(FULL, sG, 1);
  if (lane == 0) { eF = er_zero<double>(); esF = 0; }
  if (lane == 31) { eG = er_zero<double>(); esG = 0; }
  if (lane == 31) { wFm[warp] = F.m; wFe[warp] = F.e; wFs[warp] = sF; }
  if (lane == 0) { wGm[warp] = G.m; wGe[warp] = G.e; wGs[warp] = sG; }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the warp totals
    ER<double> A = er_zero<double>(), C = er_zero<double>();
    int sa = 0, sc = 0;
    if (lane < NWP) {
      A = ER<double>{wFm[lane], wFe[lane]}; sa = wFs[lane];
      C = ER<double>{wGm[lane], wGe[lane]}; sc = wGs[lane];
    }
    warp_pair_scan(t, lane, A, sa, C, sc);
    ER<double> xa = shfl_up_er(A, 1), xc = shfl_down_er(C, 1);
    if (lane == 0) xa = er_zero<double>();
    if (lane == 31 || lane + 1 >= NWP) xc = er_zero<double>();
    __syncwarp();
    if (lane < NWP) {
      wFm[lane] = xa.m; wFe[lane] = xa.e;
      wGm[lane] = xc.m; wGe[lane] = xc.e;
    }
  }
  __syncthreads();
  ER<double> cf = er_fma(ER<double>{wFm[warp], wFe[warp]}, tpow(t, esF), eF);
  ER<double> cb = er_fma(ER<double>{wGm[warp], wGe[warp]}, tpow(t, esG), eG);
  for (int i = i0; i < i1; ++i) {
    const ER<double> v{Fm[i], Fe[i]};
    Fm[i] = cf.m; Fe[i] = cf.e;
    cf = er_fma(cf, (i == n - 1) ? Ll : L1, v);
  }
  for (int i = i1 - 1; i >= i0; --i) {
    const ER<double> v{Bm[i], Be[i]};
    Bm[i] = cb.m; Be[i] = cb.e;
    cb = er_fma(cb, (i == n - 1) ? Ll : L1, v);
  }
  if (n == 0) {
    if (tid == 0) { tm[0] = tm[1] = 0.0; te[0] = te[1] = ZE; }
  } else {
    if (i0 < n && i1 == n) { tm[0] = cf.m; te[0] = cf.e; }  // owner of the last element
    if (tid == 0) { tm[1] = cb.m; te[1] = cb.e; }
  }
  __syncthreads();
  totF = ER<double>{tm[0], te[0]};
  totB = ER<double>{tm[1], te[1]};
  __syncthreads();
}

// Block level: CTA b scans its block's tile totals in place (in-block exclusive
// carries) and writes the block totals {F end, B start} to BF/BB[b].
struct BlockIO {
  double *Fm, *Bm;   // tile totals -> in-block exclusive carries
  int *Fe, *Be;
  double *BFm, *BBm; // [nblocks] block totals -> block carries (k_scan_blocks)
  int *BFe, *BBe;
};
__device__ __forceinline__ void block_totals(const ShardParams& P, const BlockIO& bi, PowTab tiles) {
  const int b = blockIdx.x;
  const int t0 = b * P.TB, n = min(P.T, t0 + P.TB) - t0;
  ER<double> tF, tB;
  cta_scan<32 * NW>(tiles, ER<double>{P.t2m[0], P.t2e[0]}, n, bi.Fm + t0, bi.Fe + t0, bi.Bm + t0, bi.Be + t0, tF, tB);
  if (threadIdx.x == 0) {
    bi.BFm[b] = tF.m; bi.BFe[b] = tF.e;
    bi.BBm[b] = tB.m; bi.BBe[b] = tB.e;
  }
}
__global__ void __launch_bounds__(32 * NW) k_block_scan(const ShardParams P, const BlockIO bi) {
  block_totals(P, bi, PowTab{P.t2m, P.t2e, nullptr, nullptr, 0});
}

// ---------------------------------------------------------------- fused exchange
// Mailbox of a rank (device memory its peers write through NVLink):
//   double tot[2][world][4]  totals of production e in slot e & 1, one row per rank
//   u32 flag[world]          flag[k] = the last production rank k delivered here
//   u32 epoch                this rank's own production counter
// Producer (k_scan_blocks, one thread): e = ++epoch; row `rank` of slot e & 1 in every
// mailbox, one system-scope fence, then flag[rank] = e in every mailbox (release).
// Consumer (k_box_wait, one warp, lane k = rank k): wait for flag[k] >= e (its own
// epoch: the ranks produce in lock step), one fence (acquire); then k_half reads row
// k of slot e & 1.  Two slots suffice:
// a rank produces e + 2 only after consuming e + 1, i.e. after every rank produced
// e + 1, i.e. after every rank finished consuming e.
__device__ __forceinline__ unsigned* box_flags(double* box, int world) {
  return reinterpret_cast<unsigned*>(box + 8 * world);
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// one system-scope fence per side: data stores -> fence -> flag stores (release
// pattern); flag loads -> fence -> data loads (acquire pattern)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void box_publish(const ShardParams& P, const double (&t)[4]) {
  unsigned* ep = box_flags(P.box[P.rank], P.world) + P.world;
  const unsigned e = __ldcg(ep) + 1u;
  *ep = e;
  const int slot = e & 1;
  for (int p = 0; p < P.world; ++p) {
    double* dst = P.box[p] + ((size_t)slot * P.world + P.rank) * 4;
    dst[0] = t[0]; dst[1] = t[1]; dst[2] = t[2]; dst[3] = t[3];
  }
  fence_acq_rel_sys();
  for (int p = 0; p < P.world; ++p) st_relaxed_sys(box_flags(P.box[p], P.world) + P.rank, e);
}
// Consumer side, one warp ahead of k_half (lane k = rank k): wait until every rank
// delivered this rank's epoch e, then one system-scope fence (acquire pattern).  The
// kernel boundary orders k_half's reads of the slot after it.  (Waiting inside the
// producing kernel would save this launch but deadlocks the lock-stepped ranks of
// one device, whose producers run one after another on one stream.)
__global__ void k_box_wait(const ShardParams P) {
  const unsigned* fl = box_flags(P.box[P.rank], P.world);
  const unsigned e = __ldcg(fl + P.world);
  for (int k = threadIdx.x; k < P.world; k += 32)
    while (ld_relaxed_sys(fl + k) < e) {
    }
  fence_acq_rel_sys();
}
__device__ __forceinline__ const double* box_slot(const ShardParams& P) {
  const unsigned e = __ldcg(box_flags(P.box[P.rank], P.world) + P.world);
  return P.box[P.rank] + (size_t)(e & 1) * P.world * 4;
}

// One CTA over the blocks: exclusive block carries in place and the rank's totals
// {F at the segment end, B at its start} -> tot[0..3] (m, e as doubles).
__global__ void __launch_bounds__(SCAN_NT) k_scan_blocks(const ShardParams P, const BlockIO bi, double* tot) {
  __shared__ double pm[32];
  __shared__ int pe[32];
  if (threadIdx.x == 0) {  // (lambda^{256 TB})^{2^j} by repeated squaring
    ER<double> x = powt(P, P.TB);
    for (int j = 0; j < 32; ++j) {
      pm[j] = x.m; pe[j] = x.e;
      x = er_mul(x, x);
    }
  }
  __syncthreads();
  ER<double> tF, tB;
  const ER<double> Ll = powt(P, P.T - (long long)(P.nblk - 1) * P.TB);
  cta_scan<SCAN_NT>(PowTab{pm, pe, nullptr, nullptr, 0}, Ll, P.nblk, bi.BFm, bi.BFe, bi.BBm, bi.BBe, tF, tB);
  if (threadIdx.x == 0) {
    const double t[4] = {tF.m, (double)tF.e, tB.m, (double)tB.e};
    if (tot) { tot[0] = t[0]; tot[1] = t[1]; tot[2] = t[2]; tot[3] = t[3]; }
    if (P.fused) box_publish(P, t);
  }
}

// Decay of the other ranks' totals to this segment: lane k of warp 0 takes rank k
// (forward from ranks k < r over the tiles between k's end and this segment's start,
// backward from ranks k > r), then a fixed-order warp sum.  allT = [world][4]
// {F m, F e, B m, B e}; world <= 32 per pass of the lane loop.
__device__ __forceinline__ void ext_carries(const ShardParams& P, const double* allT, int lane, ER<double>& EF,
                                            ER<double>& EB) {
  ER<double> f = er_zero<double>(), b = er_zero<double>();
  for (int k = lane; k < P.world; k += 32) {
    if (k == P.rank) continue;
    const long long T0k = (long long)k * P.Ttot / P.world, T1k = (long long)(k + 1) * P.Ttot / P.world;
    if (k < P.rank) {
      const ER<double> t{__ldcg(allT + 4 * k), (int)__ldcg(allT + 4 * k + 1)};
      f = er_add(f, er_mul(powt(P, P.T0 - T1k), t));
    } else {
      const ER<double> t{__ldcg(allT + 4 * k + 2), (int)__ldcg(allT + 4 * k + 3)};
      b = er_add(b, er_mul(powt(P, T0k - (P.T0 + P.T)), t));
    }
  }
  EF = stm::warp_er_sum(f);
  EB = stm::warp_er_sum(b);
}

// ------------------------------------------------------------------ k_half
struct HalfIO {
  const double* xm; const int* xX;                 // x (consumed): mantissas, tile exponents
  const double* CFm; const int* CFe;               // x's in-block exclusive tile carries
  const double* CBm; const int* CBe;
  const double* BCFm; const int* BCFe;             // x's block carries (k_scan_blocks)
  const double* BCBm; const int* BCBe;
  BlockIO yb;                                      // y's tile totals -> in-block carries, block totals
  const double* tm; const int* tX; const unsigned char* tz;  // target a or b
  const double* om; const int* oX;                 // psi^(l) (check)
  double* ym; int* yX;                             // y (produced)
  const double* allT;                              // [world][4] totals of x
  double* part;                                    // [gridDim] error partials
  int* flag;                                       // [2]: non-finite seen, first iteration
  int l;                                           // iteration (for the non-finite record);
                                                   // < 0: read it from flag[2] (graph replays)
};

template <bool CHECK, bool WRITE>
__global__ void __launch_bounds__(32 * NW) k_half(const ShardParams P, const HalfIO io) {
  __shared__ double sEm[2];
  __shared__ int sEe[2];
  __shared__ double werr[NW];
  __shared__ double pwm[TBMAX + 1];  // lambda^{256 k}, k <= TB (this block's tile spans)
  __shared__ int pwe[TBMAX + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k <= P.TB; k += blockDim.x) {
    const ER<double> t = powt(P, k);
    pwm[k] = t.m;
    pwe[k] = t.e;
  }
  if (warp == 0) {
    ER<double> EF, EB;
    const double* allT = P.fused ? box_slot(P) : io.allT;
    ext_carries(P, allT, lane, EF, EB);
    if (lane == 0) { sEm[0] = EF.m; sEe[0] = EF.e; sEm[1] = EB.m; sEe[1] = EB.e; }
  }
  __syncthreads();
  const PowTab tiles{P.t2m, P.t2e, pwm, pwe, P.TB + 1};
  const ER<double> EF{sEm[0], sEe[0]}, EB{sEm[1], sEe[1]};
  const double lam = P.lam;
  const double lp = P.lanepow[lane], rp = P.lanepow[31 - lane];
  double errw = 0.0;
  int bad = 0;
  // this CTA's block of tiles [t0, t1): the carries entering it (block carries of this
  // rank + the other ranks' totals decayed over the tiles before / after the block)
  const int blk = blockIdx.x;
  const int t0 = blk * P.TB, t1 = min(P.T, t0 + P.TB);
  const ER<double> CFb = er_fma(powt(P, t0), EF, ER<double>{io.BCFm[blk], io.BCFe[blk]});
  const ER<double> CBb = er_fma(powt(P, P.T - t1), EB, ER<double>{io.BCBm[blk], io.BCBe[blk]});
  for (int i = t0 + warp; i < t1; i += NW) {
    // full carries of tile i relative to its reference exponent R
    const ER<double> CF = er_fma(tpow(tiles, i - t0), CFb, ER<double>{io.CFm[i], io.CFe[i]});
    const ER<double> CB = er_fma(tpow(tiles, t1 - 1 - i), CBb, ER<double>{io.CBm[i], io.CBe[i]});
    const int X = io.xX[i];
    int R = X;
    if (X == ZE || CF.e - X > LIM || CB.e - X > LIM) R = max(CF.e, CB.e);
    if (R == ZE) R = 0;
    const double cfr = er_rel(CF, R), cbr = er_rel(CB, R);
    double xv[E], tv[E];
    ld_tile(io.xm + (size_t)i * TILE, lane, xv);
    ld_tile(io.tm + (size_t)i * TILE, lane, tv);
    if (X != R) {
      const double sc = pow2d(max(X - R, -1100));
#pragma unroll
      for (int e = 0; e < E; ++e) xv[e] *= sc;
    }
    double Fi, Gi;
    lane_scan(P, xv, Fi, Gi);
    const double cf = fma(lp, cfr, prev_or0(Fi));
    const double cb = fma(rp, cbr, next_or0(Gi));
    // forward p_k = lam p_{k-1} + x_k; backward t_k = lam t_{k+1} + x_k, K x = p + lam t_{k+1}
    double pf[E];
    double p = cf;
#pragma unroll
    for (int e = 0; e < E; ++e) { p = fma(lam, p, xv[e]); pf[e] = p; }
    double ov[E];
    double sce = 0.0;
    if (CHECK) {
      ld_tile(io.om + (size_t)i * TILE, lane, ov);
      sce = pow2d(min(max(io.oX[i] + R - io.tX[i], -1100), 1000));
    }
    const int Xt = io.tX[i];
    const bool guard = io.tz[i];
    unsigned zm = 0;  // zero targets of a guarded tile (warp-uniform test), zeroed after the loop
    if (WRITE && guard) {
#pragma unroll
      for (int e = 0; e < E; ++e) zm |= (unsigned)!(tv[e] > 0.0) << e;
    }
    double tn = cb, errp = 0.0;
#pragma unroll
    for (int e = E - 1; e >= 0; --e) {
      const double kx = fma(lam, tn, pf[e]);
      tn = fma(lam, tn, xv[e]);
      if (CHECK) errp += fabs(fma(ov[e] * sce, kx, -tv[e]));
      if (WRITE) tv[e] = stm::fdiv(tv[e], kx);  // branch-free (as K2's update)
    }
    if (WRITE && guard) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if ((zm >> e) & 1u) tv[e] = 0.0;
    }
    if (CHECK) {
      const double es = warp_sum(errp);
      errw += (Xt == ZE) ? 0.0 : ldexp(es, Xt);
    }
    if (WRITE) {
      // exact power-of-two renormalisation of the produced tile
      int hm = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) hm = max(hm, __double2hiint(tv[e]));
      hm = warp_max(hm);
      const int base = (Xt == ZE) ? ZE : Xt - R;
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
      lane_tot(P, lp, rp, tv, FiY, GiY);
      if (!isfinite(FiY + GiY)) bad = 1;
      put_tot(P, lane, FiY, GiY, Y, i, io.yb.Fm, io.yb.Fe, io.yb.Bm, io.yb.Be);
      st_tile(io.ym + (size_t)i * TILE, lane, tv);
      if (lane == 0) io.yX[i] = Y;
    }
  }
  if (CHECK) {
    if (lane == 0) werr[warp] = errw;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += werr[w];
      io.part[blockIdx.x] = s;
    }
  }
  if (WRITE) {  // y's tiles of this block: in-block exclusive carries and block totals
    __syncthreads();
    block_totals(P, io.yb, tiles);
  }
  if (__any_sync(FULL, bad) && lane == 0) {
    atomicOr(&io.flag[0], 1);
    atomicMin(&io.flag[1], io.l >= 0 ? io.l : io.flag[2]);
  }
}

__global__ void k_init_flag(int* flag) {
  flag[0] = 0;
  flag[1] = 0x7fffffff;
  flag[2] = 1;  // device iteration counter l + 1 (advanced by k_tick)
}
// advance the device iteration counter (one per iteration, after the phi half-step)
__global__ void k_tick(int* flag) { flag[2] += 1; }

// deterministic sum of the per-CTA partials (fixed order) -> out[0]; out[1] = the first
// iteration whose state was non-finite (0: none)
__global__ void k_reduce(const double* part, int nparts, const int* flag, double* out) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < nparts; ++k) s += part[k];
    out[0] = s;
    out[1] = flag[0] ? (double)flag[1] : 0.0;
  }
}

// ------------------------------------------------------------------ cost (Jordan pairs)
struct Pair {
  ER<double> a, b;
};
// pair state (p, P') after a span of L points with multiplier lL = lam^L: left A then right B
__device__ __forceinline__ Pair pcomb(Pair A, Pair B, ER<double> lL, double L) {
  return Pair{er_add(er_mul(A.a, lL), B.a), er_add(er_mul(er_add(A.b, er_scale(A.a, L)), lL), B.b)};
}
__device__ __forceinline__ Pair pzero() { return Pair{er_zero<double>(), er_zero<double>()}; }

// lane pair aggregates (relative): forward (p, P') at the chunk end, backward (t, Q') at
// its start, then warp scans in ER form: inclusive (forward over lanes, backward).
__device__ __forceinline__ void jordan_tile(const ShardParams& P, int lane, const double (&v)[E], int X,
                                            Pair& fwd, Pair& bwd) {
  const double lam = P.lam;
  double p = 0, Pp = 0, t = 0, Q = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) { Pp = lam * (Pp + p); p = fma(lam, p, v[e]); }
#pragma unroll
  for (int e = E - 1; e >= 0; --e) { Q = lam * (Q + t); t = fma(lam, t, v[e]); }
  fwd = Pair{er_norm<double>(p, X), er_norm<double>(Pp, X)};
  bwd = Pair{er_norm<double>(t, X), er_norm<double>(Q, X)};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int d = 1 << k;
    const ER<double> LL{P.lvm8[k], P.lve8[k]};
    const double L = (double)E * d;
    const Pair up{shfl_up_er(fwd.a, d), shfl_up_er(fwd.b, d)};
    const Pair dn{shfl_down_er(bwd.a, d), shfl_down_er(bwd.b, d)};
    if (lane >= d) fwd = pcomb(up, fwd, LL, L);
    if (lane + d < 32) bwd = pcomb(dn, bwd, LL, L);
  }
}

// per tile of psi: the tile pair totals (forward at the end, backward at the start)
__global__ void __launch_bounds__(32 * NW) k_cost_tiles(const ShardParams P, const double* qm, const int* qX,
                                                        double* Jm, int* Je) {
  const int lane = threadIdx.x & 31;
  const long long wg = (long long)blockIdx.x * NW + (threadIdx.x >> 5);
  const long long nwarps = (long long)gridDim.x * NW;
  for (long long i = wg; i < P.T; i += nwarps) {
    double v[E];
    ld_tile(qm + i * TILE, lane, v);
    Pair f, b;
    jordan_tile(P, lane, v, qX[i], f, b);
    if (lane == 31) { Jm[4 * i] = f.a.m; Je[4 * i] = f.a.e; Jm[4 * i + 1] = f.b.m; Je[4 * i + 1] = f.b.e; }
    if (lane == 0) { Jm[4 * i + 2] = b.a.m; Je[4 * i + 2] = b.a.e; Jm[4 * i + 3] = b.b.m; Je[4 * i + 3] = b.b.e; }
  }
}

// one CTA: exclusive local pair carries per tile (in place) + segment pair totals
// tot8 = {p m, p e, P' m, P' e (end); t m, t e, Q' m, Q' e (start)}
__global__ void __launch_bounds__(SCAN_NT) k_cost_scan(const ShardParams P, double* Jm, int* Je, double* tot8) {
  __shared__ double sm[32][4];
  __shared__ int se[32][4], ss[32][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = SCAN_NT / 32;
  const int T = P.T;
  const int q = (T + SCAN_NT - 1) / SCAN_NT;
  const int i0 = min(T, tid * q), i1 = min(T, i0 + q);
  const ER<double> L1{P.t2m[0], P.t2e[0]};
  const double LT = (double)TILE;
  auto ld = [&](int i, int k) { return ER<double>{Jm[4 * i + k], Je[4 * i + k]}; };
  Pair f = pzero(), g = pzero();
  for (int i = i0; i < i1; ++i) f = pcomb(f, Pair{ld(i, 0), ld(i, 1)}, L1, LT);
  for (int i = i1 - 1; i >= i0; --i) g = pcomb(g, Pair{ld(i, 2), ld(i, 3)}, L1, LT);
  int sF = i1 - i0, sG = i1 - i0;
  Pair F = f, G = g;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Pair uf{shfl_up_er(F.a, d), shfl_up_er(F.b, d)};
    const int us = __shfl_up_sync(FULL, sF, d);
    const Pair dg{shfl_down_er(G.a, d), shfl_down_er(G.b, d)};
    const int ds = __shfl_down_sync(FULL, sG, d);
    if (lane >= d) { F = pcomb(uf, F, powt(P, sF), LT * sF); sF += us; }
    if (lane + d < 32) { G = pcomb(dg, G, powt(P, sG), LT * sG); sG += ds; }
  }
  Pair eF{shfl_up_er(F.a, 1), shfl_up_er(F.b, 1)};
  int esF = __shfl_up_sync(FULL, sF, 1);
  Pair eG{shfl_down_er(G.a, 1), shfl_down_er(G.b, 1)};
  int esG = __shfl_down_sync(FULL, sG, 1);
  if (lane == 0) { eF = pzero(); esF = 0; }
  if (lane == 31) { eG = pzero(); esG = 0; }
  if (lane == 31) { sm[warp][0] = F.a.m; se[warp][0] = F.a.e; sm[warp][1] = F.b.m; se[warp][1] = F.b.e; ss[warp][0] = sF; }
  if (lane == 0) { sm[warp][2] = G.a.m; se[warp][2] = G.a.e; sm[warp][3] = G.b.m; se[warp][3] = G.b.e; ss[warp][1] = sG; }
  __syncthreads();
  Pair cw = pzero(), cg = pzero();
  for (int w = 0; w < warp; ++w)
    cw = pcomb(cw, Pair{ER<double>{sm[w][0], se[w][0]}, ER<double>{sm[w][1], se[w][1]}}, powt(P, ss[w][0]),
               LT * ss[w][0]);
  for (int w = nwarp - 1; w > warp; --w)
    cg = pcomb(cg, Pair{ER<double>{sm[w][2], se[w][2]}, ER<double>{sm[w][3], se[w][3]}}, powt(P, ss[w][1]),
               LT * ss[w][1]);
  Pair cf = pcomb(cw, eF, powt(P, esF), LT * esF);
  Pair cb = pcomb(cg, eG, powt(P, esG), LT * esG);
  for (int i = i0; i < i1; ++i) {
    const Pair t{ld(i, 0), ld(i, 1)};
    Jm[4 * i] = cf.a.m; Je[4 * i] = cf.a.e; Jm[4 * i + 1] = cf.b.m; Je[4 * i + 1] = cf.b.e;
    cf = pcomb(cf, t, L1, LT);
  }
  for (int i = i1 - 1; i >= i0; --i) {
    const Pair t{ld(i, 2), ld(i, 3)};
    Jm[4 * i + 2] = cb.a.m; Je[4 * i + 2] = cb.a.e; Jm[4 * i + 3] = cb.b.m; Je[4 * i + 3] = cb.b.e;
    cb = pcomb(cb, t, L1, LT);
  }
  if (tid == SCAN_NT - 1) {
    tot8[0] = cf.a.m; tot8[1] = cf.a.e; tot8[2] = cf.b.m; tot8[3] = cf.b.e;
  }
  if (tid == 0) {
    tot8[4] = cb.a.m; tot8[5] = cb.a.e; tot8[6] = cb.b.m; tot8[7] = cb.b.e;
  }
}

// per tile: sum_k phi_k (P'_k + Q'_k) with the full pair carries (local + other ranks),
// per-CTA partials (ER) -> part / parte
__global__ void __launch_bounds__(32 * NW) k_cost_dot(const ShardParams P, const double* qm, const int* qX,
                                                      const double* pm, const int* pX, const double* Jm,
                                                      const int* Je, const double* all8, double* part,
                                                      int* parte) {
  __shared__ Pair sE[2];
  __shared__ double wm[NW];
  __shared__ int we[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double LT = (double)TILE;
  if (threadIdx.x == 0) {
    // fold the other ranks' pair totals in order: forward k = 0..r-1 (each followed by
    // its gap to the next segment), backward k = world-1..r+1
    Pair ef = pzero(), eb = pzero();
    for (int k = 0; k < P.rank; ++k) {
      const long long T0k = (long long)k * P.Ttot / P.world, T1k = (long long)(k + 1) * P.Ttot / P.world;
      const Pair t{ER<double>{all8[8 * k], (int)all8[8 * k + 1]}, ER<double>{all8[8 * k + 2], (int)all8[8 * k + 3]}};
      ef = pcomb(ef, t, powt(P, T1k - T0k), LT * (double)(T1k - T0k));
    }
    for (int k = P.world - 1; k > P.rank; --k) {
      const long long T0k = (long long)k * P.Ttot / P.world, T1k = (long long)(k + 1) * P.Ttot / P.world;
      const Pair t{ER<double>{all8[8 * k + 4], (int)all8[8 * k + 5]}, ER<double>{all8[8 * k + 6], (int)all8[8 * k + 7]}};
      eb = pcomb(eb, t, powt(P, T1k - T0k), LT * (double)(T1k - T0k));
    }
    sE[0] = ef;
    sE[1] = eb;
  }
  __syncthreads();
  const Pair EF = sE[0], EB = sE[1];
  const double lam = P.lam;
  ER<double> accw = er_zero<double>();
  const long long wg = (long long)blockIdx.x * NW + warp;
  const long long nwarps = (long long)gridDim.x * NW;
  for (long long i = wg; i < P.T; i += nwarps) {
    auto ld = [&](int k) { return ER<double>{Jm[4 * i + k], Je[4 * i + k]}; };
    const Pair cf = pcomb(EF, Pair{ld(0), ld(1)}, powt(P, i), LT * (double)i);
    const Pair cb = pcomb(EB, Pair{ld(2), ld(3)}, powt(P, P.T - 1 - i), LT * (double)(P.T - 1 - i));
    const int X = qX[i];
    const int mx = max(max(cf.a.e, cf.b.e), max(cb.a.e, cb.b.e));
    int R = X;
    if (X == ZE || mx - X > LIM) R = mx;
    if (R == ZE) R = 0;
    double v[E], ph[E];
    ld_tile(qm + i * TILE, lane, v);
    ld_tile(pm + i * TILE, lane, ph);
    if (X != R) {
      const double sc = pow2d(max(X - R, -1100));
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] *= sc;
    }
    // lane-exclusive pair carries inside the tile (relative to 2^R)
    double fp = 0, fP = 0, bt = 0, bQ = 0;
    {
      double p = 0, Pp = 0, t = 0, Q = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) { Pp = lam * (Pp + p); p = fma(lam, p, v[e]); }
#pragma unroll
      for (int e = E - 1; e >= 0; --e) { Q = lam * (Q + t); t = fma(lam, t, v[e]); }
      fp = p; fP = Pp; bt = t; bQ = Q;
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int d = 1 << k;
        const double LL = P.lvd[k], L = (double)E * d;
        const double up = __shfl_up_sync(FULL, fp, d), uP = __shfl_up_sync(FULL, fP, d);
        const double dt = __shfl_down_sync(FULL, bt, d), dQ = __shfl_down_sync(FULL, bQ, d);
        if (lane >= d) { fP = fma(LL, fma(L, up, uP), fP); fp = fma(LL, up, fp); }
        if (lane + d < 32) { bQ = fma(LL, fma(L, dt, dQ), bQ); bt = fma(LL, dt, bt); }
      }
    }
    double xp = __shfl_up_sync(FULL, fp, 1), xP = __shfl_up_sync(FULL, fP, 1);
    double xt = __shfl_down_sync(FULL, bt, 1), xQ = __shfl_down_sync(FULL, bQ, 1);
    if (lane == 0) { xp = 0; xP = 0; }
    if (lane == 31) { xt = 0; xQ = 0; }
    const double Lf = (double)(E * lane), Lb = (double)(E * (31 - lane));
    const double lf = P.lanepow[lane], lb = P.lanepow[31 - lane];
    const double cp = er_rel(cf.a, R), cP = er_rel(cf.b, R), ct = er_rel(cb.a, R), cQ = er_rel(cb.b, R);
    double p = fma(lf, cp, xp), Pp = fma(lf, fma(Lf, cp, cP), xP);
    double t = fma(lb, ct, xt), Q = fma(lb, fma(Lb, ct, cQ), xQ);
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) { Pp = lam * (Pp + p); p = fma(lam, p, v[e]); acc = fma(ph[e], Pp, acc); }
#pragma unroll
    for (int e = E - 1; e >= 0; --e) { Q = lam * (Q + t); t = fma(lam, t, v[e]); acc = fma(ph[e], Q, acc); }
    const double s = warp_sum(acc);
    if (pX[i] != ZE) accw = er_add(accw, er_norm<double>(s, R + pX[i]));
  }
  if (lane == 0) { wm[warp] = accw.m; we[warp] = accw.e; }
  __syncthreads();
  if (threadIdx.x == 0) {
    ER<double> s = er_zero<double>();
    for (int w = 0; w < NW; ++w) s = er_add(s, ER<double>{wm[w], we[w]});
    part[blockIdx.x] = s.m;
    parte[blockIdx.x] = s.e;
  }
}

// cost partial of this rank: h * sum of the per-CTA ER partials (fixed order)
__global__ void k_cost_reduce(const ShardParams P, const double* part, const int* parte, int nparts, double* out) {
  if (threadIdx.x == 0) {
    ER<double> s = er_zero<double>();
    for (int k = 0; k < nparts; ++k) s = er_add(s, ER<double>{part[k], parte[k]});
    out[0] = (s.m == 0.0) ? 0.0 : ldexp(s.m, s.e) * P.h;
  }
}

// ------------------------------------------------------------------ k_store
// F = log phi or G = log psi of the segment's valid points.
__global__ void __launch_bounds__(32 * NW) k_store(const ShardParams P, const double* m, const int* X, double* out) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q = k; q < P.len && P.lo + q < P.n; q += stride) {
    const int Xt = X[q / TILE];
    const double v = m[q];
    out[q] = (v > 0.0 && Xt != ZE) ? log(v) + (double)Xt * LN2 : (v == 0.0 ? -INFINITY : NAN);
  }
}

}  // namespace shd
}  // namespace fs1
