// fs1_sep2dw.cuh — K3w: the warp-per-line separable 2D FS-1 solve (fp32, log domain;
// config C4, 2048 x 2048).
//
// Algorithm 2 with K = T_M(lambda2) (x) T_N(lambda1)
// (PAPER.md:255-280): every K x is a pass of 1D applies along axis 1 (K0 on every
// column) and a pass along axis 2.  Each 1D
// line apply is the forward / backward recursion of Eq. "recursion"
// (PAPER.md:129-137), run by ONE WARP per line as a chunked scan: lane l owns the E
// consecutive points [lE, lE+E) of a line of up to 32 E points.
//
// Layout.  Every internal array is a set of lines of LP = 32 E floats stored in the
// lane-chunk-permuted order: the 8-float run j of lane l's chunk sits at run slot
// 32 j + l, so a warp loads its whole line with E/8 fully coalesced 1 KiB
// 256-bit loads and every lane ends up with its own chunk in registers (no
// shared-memory staging), and the 8 lines of a group land as one 32-byte sector
// per position in the transposed write.  Padding points (index >= line length)
// hold -inf.
//
// Passes.  Two fused passes per iteration, each one grid barrier:
//   R (lines = rows i, along axis 2):  k = K2 e^{Z1_i}  (Z1 = log K1 phi, transposed)
//       [check: err += sum |e^{G_old + log k} - b|]
//       psi_i = b_i / k as linear mantissas          (psi update)
//       [G_i = log b_i - log k stored only where a loop top may stop on it]
//       Z2 = log K2 psi_i, written transposed        (first pass of the phi half-step)
//   C (lines = columns j, along axis 1):  phi_j = a_j / K1 e^{Z2_j}
//       Z1 = log K1 phi_j, written transposed        (first pass of the next psi half-step)
// The fused second apply reuses the freshly updated line from registers, so each
// point is read and written twice per iteration instead of four times, and there
// are 2 grid barriers per iteration instead of 4.  Transposed writes go through a
// per-CTA shared stage of W = 8 lines so that each position leaves as one sector.
//
// Arithmetic (the chunk-relative log scheme): the first apply of a
// pass converts the lane's chunk, m_e = 2^(X_e log2 e - oe) with oe = floor(max X
// log2 e) (one MUFU ex2 per point), the recursions run linearly in fp32 relative to
// 2^oe, the update is one MUFU rcp per point against the target's mantissas, the
// second apply runs on those linear values directly, and the pass leaves through one
// MUFU lg2 per point (3 MUFU per point per pass).  Chunk totals cross lanes as
// extended-range fp32 numbers (mantissa in [1,2), int exponent) in a 5-level warp
// shuffle scan with multipliers lambda^{E 2^k} formed on the host (Remark 3.3).
// In-lane work runs as 2-4 independent chains (ILP): the chunk halves get their own
// carries from the half aggregates.
#pragma once
#include <math.h>
#include <stdint.h>

#include "fs1_sep2d.cuh"

namespace fs1 {
namespace sepw {

// per-phase timestamps of pass R at iteration 5 (tools/phase_sep.py) only in probe builds
// (tools/variant.sh probe -DFS1_K3W_PROBE=1)
#ifndef FS1_K3W_PROBE
#define FS1_K3W_PROBE 0
#endif
#ifndef FS1_K3W_LATE_TMA
#define FS1_K3W_LATE_TMA 1
#endif
// the next pass's first target line is fetched by TMA at the end of a pass (the stage is
// free once the transposed write is out), so it lands during the grid barrier
#ifndef FS1_K3W_PREFETCH
#define FS1_K3W_PREFETCH 0
#endif
// fused passes test the updated line for NaN / +inf through the second apply's chunk
// aggregates instead of point by point
#ifndef FS1_K3W_AGGNF
#define FS1_K3W_AGGNF 1
#endif
constexpr int W = 8;        // warps = lines per CTA group
constexpr int NT = 32 * W;
constexpr int LIMF = 60;    // carries up to 2^60 above a chunk keep its exponent
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

template <int E> struct Cfg {
  static constexpr int LP = 32 * E;             // padded line length (floats)
  static constexpr int Q = E / 4;               // float4 per lane chunk
  static constexpr int SROW = E + 4;            // stage floats per lane chunk (padded)
  static constexpr int SLINE = 32 * SROW;       // stage floats per line (>= LP)
  static constexpr size_t STAGE = (size_t)W * SLINE * 4;
  static constexpr size_t STAGE_ALL = STAGE > (size_t)sep::OFF_XM ? STAGE : (size_t)sep::OFF_XM;
  static constexpr size_t LINEB = (size_t)LP * 4;
  static constexpr size_t OFF_MBAR = STAGE_ALL;                // [W][2] mbarriers
  static constexpr size_t OFF_XM = OFF_MBAR + W * 2 * 8;
  static constexpr size_t OFF_XI = OFF_XM + 4 * sep::W * 8;
  static constexpr size_t OFF_RED = OFF_XI + 4 * sep::W * 4;
  static constexpr size_t OFF_IRED = OFF_RED + 64 * 8;
  static constexpr size_t SMEM = OFF_IRED + 64 * 4;
};

// position of point q of a line in the permuted layout: 8-float run j of lane l's chunk
// sits at run slot 32 j + l (one 32-byte sector)
template <int E> __device__ __forceinline__ int pidx(int q) {
  const int l = q / E, e = q - l * E;
  return ((e >> 3) * 32 + l) * 8 + (e & 7);
}
// point of permuted slot k
template <int E> __device__ __forceinline__ int pinv(int k) {
  const int j8 = k >> 3, l = j8 & 31, e = (j8 >> 5) * 8 + (k & 7);
  return l * E + e;
}

// 256-bit global accesses (LDG/STG.E.ENL2.256): one full sector per lane
__device__ __forceinline__ void ldg8(const float* p, float* v) {
  asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void stg8(float* p, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

// ------------------------------------------------------------ extended-range fp32
struct ERf {
  float m;
  int e;
};
__device__ __forceinline__ float p2f(int d) {  // exact 2^d, 0 below 2^-126
  d = min(d, 127);
  return d >= -126 ? __uint_as_float((unsigned)(d + 127) << 23) : 0.f;
}
__device__ __forceinline__ ERf ern(float x, int e) {  // normalise x 2^e (x >= 0, normal or 0)
  // selects, no branch (a branch here made every scan level of line_apply_lin divergent)
  const unsigned u = __float_as_uint(x);
  const bool pos = x > 0.f;
  ERf r;
  r.e = pos ? e + (int)((u >> 23) & 0xffu) - 127 : ZE;
  r.m = pos ? __uint_as_float((u & 0x807fffffu) | 0x3f800000u) : 0.f;
  return r;
}
__device__ __forceinline__ ERf era(ERf a, ERf b) {
  const int e = max(a.e, b.e);
  return ern(fmaf(a.m, p2f(a.e - e), b.m * p2f(b.e - e)), e);
}
__device__ __forceinline__ ERf erm(ERf a, float bm, int be) { return ern(a.m * bm, a.e + be); }

// Per-axis scan tables (host-formed, Remark 3.3), read straight from the
// __grid_constant__ parameter block (constant-bank operands, no registers).
using AxT = Sep2dParams::WAx;

// ------------------------------------------------------------ one line apply
// Natural logs X of this lane's chunk -> mantissas relative to 2^oe, oe = floor(max X
// log2 e) (one MUFU ex2 per point); an all -inf chunk gives zeros and oe = ZE.
template <int E>
__device__ __forceinline__ int prep_log(float (&A)[E]) {
  float M = -INFINITY;
#pragma unroll
  for (int e = 0; e < E; ++e) M = fmaxf(M, A[e]);
  int oe;
  if (M == -INFINITY) {
    oe = ZE;
#pragma unroll
    for (int e = 0; e < E; ++e) A[e] = 0.f;
  } else if (!(M < INFINITY)) {  // +inf weight: poison the chunk (the problem flags NONFINITE)
    oe = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) A[e] = NAN;
  } else {
    oe = (int)floorf(M * LOG2E);
    const float o = (float)oe;
#pragma unroll
    for (int e = 0; e < E; ++e) A[e] = sep::ex2f(fmaf(A[e], LOG2E, -o));
  }
  return oe;
}

// A: this lane's chunk as linear mantissas relative to 2^oe (oe = ZE: zero chunk).
// On return A[e] = (K x)_e relative to 2^R (linear fp32), R returned.
// nf (optional): set when this lane's chunk holds a NaN or +inf (its aggregates are then
// non-finite: the chains only add non-negative terms), the update's non-finite test
template <int E>
__device__ __forceinline__ int line_apply_lin(float (&A)[E], int oe, const AxT& T, int lane,
                                              int* nf = nullptr) {
  constexpr int H = E / 2;
  // chunk aggregates (Horner, zero carries), 4 independent chains over the halves
  const float lam = T.lam, lH = T.lamH;
  float f0 = 0.f, f1 = 0.f, g0 = 0.f, g1 = 0.f;
#pragma unroll
  for (int e = 0; e < H; ++e) {
    f0 = fmaf(lam, f0, A[e]);
    f1 = fmaf(lam, f1, A[H + e]);
    g0 = fmaf(lam, g0, A[H - 1 - e]);
    g1 = fmaf(lam, g1, A[E - 1 - e]);
  }
  const float fa = fmaf(lH, f0, f1), ga = fmaf(lH, g1, g0);
  if (nf) *nf |= !(fa + ga < INFINITY);
  ERf F = ern(fa, oe);  // forward total at the chunk end
  ERf B = ern(ga, oe);  // backward total at the chunk start
  // warp inclusive scans of the affine maps y -> lambda^{E d} y + c (Hillis-Steele)
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int d = 1 << k;
    const ERf up{__shfl_up_sync(FULL, F.m, d), __shfl_up_sync(FULL, F.e, d)};
    const ERf dn{__shfl_down_sync(FULL, B.m, d), __shfl_down_sync(FULL, B.e, d)};
    // combined on every lane, kept by a select (branch-free: the lanes below d / above
    // 31 - d would otherwise diverge at every level)
    const ERf Fn = era(erm(up, T.Lm[k], T.Le[k]), F);
    const ERf Bn = era(erm(dn, T.Lm[k], T.Le[k]), B);
    const bool tf = lane >= d, tb = lane + d < 32;
    F.m = tf ? Fn.m : F.m;
    F.e = tf ? Fn.e : F.e;
    B.m = tb ? Bn.m : B.m;
    B.e = tb ? Bn.e : B.e;
  }
  ERf cf{__shfl_up_sync(FULL, F.m, 1), __shfl_up_sync(FULL, F.e, 1)};
  ERf cb{__shfl_down_sync(FULL, B.m, 1), __shfl_down_sync(FULL, B.e, 1)};
  if (lane == 0) cf = ERf{0.f, ZE};
  if (lane == 31) cb = ERf{0.f, ZE};
  // reference exponent of the chunk: its own, unless the carries dwarf it
  int R = oe;
  if (oe == ZE || cf.e - oe > LIMF || cb.e - oe > LIMF) {
    R = max(cf.e, cb.e);
    if (R == ZE) R = (oe == ZE) ? 0 : oe;
    const float s = (oe == ZE) ? 0.f : p2f(oe - R);
#pragma unroll
    for (int e = 0; e < E; ++e) A[e] *= s;
    f0 *= s;
    g1 *= s;
  }
  const float cfr = cf.m * p2f(cf.e - R), cbr = cb.m * p2f(cb.e - R);
  // forward recursion p_k = lam p_{k-1} + x_k (Alg. 2 lines 4 / 9), two chains
  const float q0 = fmaf(lH, cfr, f0);  // p at the end of the first half
  float p = cfr, q = q0;
#pragma unroll
  for (int e = 0; e < H; ++e) {
    p = fmaf(lam, p, A[e]);
    A[e] = p;
    q = fmaf(lam, q, A[H + e]);
    A[H + e] = q;
  }
  // backward recursion t_k = lam t_{k+1} + x_k and K x = p + lam t_{k+1} (lines 5 / 10),
  // two chains; x_k = p_k - lam p_{k-1} is recovered from the stored forward values
  float ta = cbr, tb = fmaf(lH, cbr, g1);
#pragma unroll
  for (int i = 0; i < H; ++i) {
    const int ea = E - 1 - i, eb = H - 1 - i;
    const float xa = fmaf(-lam, (ea == H) ? q0 : A[ea - 1], A[ea]);
    const float ka = fmaf(lam, ta, A[ea]);
    ta = fmaf(lam, ta, xa);
    A[ea] = ka;
    const float xb = fmaf(-lam, (eb == 0) ? cfr : A[eb - 1], A[eb]);
    const float kb = fmaf(lam, tb, A[eb]);
    tb = fmaf(lam, tb, xb);
    A[eb] = kb;
  }
  return R;
}

// A: natural logs of this lane's chunk (padding -inf) -> (K e^X)_e relative to 2^R.
template <int E>
__device__ __forceinline__ int line_apply(float (&A)[E], const AxT& T, int lane) {
  const int oe = prep_log<E>(A);
  return line_apply_lin<E>(A, oe, T, lane);
}

template <int E>
__device__ __forceinline__ void load_line(const float* line, int lane, float (&A)[E]) {
#pragma unroll
  for (int j = 0; j < E / 8; ++j) ldg8(line + (j * 32 + lane) * 8, &A[8 * j]);
}
template <int E>
__device__ __forceinline__ void store_line(float* line, int lane, const float (&A)[E]) {
#pragma unroll
  for (int j = 0; j < E / 8; ++j) stg8(line + (j * 32 + lane) * 8, &A[8 * j]);
}

// MODE bits of a fused pass
constexpr int UPD = 1, WR = 2, CHK = 4, FUSE = 8;

// Per-warp TMA state: X line and target (+ G_old) line buffers with one mbarrier each.
struct WarpIO {
  float* ts;       // target line: aliases this warp's stage region (free until the FUSE output)
  uint64_t* mb;    // [2]: (unused), target
  unsigned ph0, ph1;  // parity of the next wait on mb[0] / mb[1]
  int pre;            // the first target line of the next pass is already in flight (warp-uniform)
};

// One fused pass over `nlines` lines of length `len` (axis tables T):
//   UPD:  k = K e^{X} (linear, relative to 2^R); the update y = tgt / k (PAPER.md:154 /
//         160) as linear mantissas  s = tm * rcp(k) with chunk exponent tx - R, where
//         (tm, tx) are the target's mantissas and per-lane-chunk exponents; [CHK] the
//         marginal error sum |e^{Yold + log k} - e^{LT}|; [WR] the state
//         y = LT - log k stored as logs into Yout (only where a loop top may stop on it).
//   FUSE: Z = log K y (y = X when !UPD), written transposed into Zout (lines =
//         positions 0..len-1, points = this pass's line indices).
// The target mantissa line arrives by a 1D TMA bulk copy issued when the warp takes
// the line, so the update reads it from shared memory.  Target entries below 2^-126 of
// their chunk's largest flush to 0 in s; within the chunk span (c E <= 40 nats) their
// contribution to every K y is below fp32 resolution, and the stored state (WR) comes
// from the exact log form.
template <int E, int MODE>
__device__ __forceinline__ void fused_pass(sep::Ctx& c, WarpIO& io, const AxT& T, const float* X,
                                           const float* TM, const int* TX, const float* LT,
                                           const float* Yold, float* Yout, float* Zout, int nlines,
                                           int len, int G, double& errsum, int& bad,
                                           unsigned long long* td = nullptr, const float* TMn = nullptr,
                                           int nln = 0) {
  using C = Cfg<E>;
  const int lane = c.lane, w = c.warp;
  const int ngroups = (nlines + W - 1) / W;
  float* stage = c.s.stage;
  int gi = 0;
  for (int grp = c.r; grp < ngroups; grp += G, ++gi) {
    unsigned long long* t = (FS1_K3W_PROBE && td && lane == 0 && gi < 2) ? td + (((size_t)c.r * W + w) * 2 + gi) * 8 : nullptr;
    if (t) t[0] = stm::gtimer();
    const int line = grp * W + w;
    float A[E];
    if (line < nlines) {
      const size_t off = (size_t)line * C::LP;
      // the target line arrives by TMA; issued once this warp's X line has landed, so the
      // two 16 MB bursts of a pass (every warp's X, then every warp's target) share L2
      // bandwidth with the first apply instead of with each other
      const bool pre = gi == 0 && io.pre;  // issued at the end of the previous pass
      io.pre = 0;
      auto issue_target = [&]() {
        if ((MODE & UPD) && lane == 0 && !pre) {
          stm::fence_async_smem();
          stm::mbar_expect_tx(&io.mb[1], (unsigned)C::LINEB);
          stm::bulk_g2s(io.ts, TM + off, (unsigned)C::LINEB, &io.mb[1]);
        }
      };
      if (!FS1_K3W_LATE_TMA) issue_target();
      load_line<E>(X + off, lane, A);  // E/8 coalesced 256-bit loads, all in flight at once
      if (t) t[1] = stm::gtimer() + (A[0] == 12345.f);
      int oe2 = 0;
      if (MODE & UPD) {
        const int oe1 = prep_log<E>(A);
        if (FS1_K3W_LATE_TMA) issue_target();
        const int R = line_apply_lin<E>(A, oe1, T, lane);
        if (t) t[2] = stm::gtimer() + (R == 12345);
        const int tx = TX[(size_t)line * 32 + lane];
        oe2 = (tx == ZE) ? ZE : tx - R;
        const float Rl = (float)R * LN2;
        double ep = 0.0;
        stm::mbar_wait(&io.mb[1], io.ph1);
        io.ph1 ^= 1u;
        if (t) t[3] = stm::gtimer();
        const float4* tm4 = reinterpret_cast<const float4*>(io.ts);
        int b = 0;
#pragma unroll
        for (int j = 0; j < E / 8; ++j) {
          if ((j & 1) == 0) __syncwarp();  // bounds the hoisting of the shared loads (registers)
          const float4 m0 = tm4[(j * 32 + lane) * 2], m1 = tm4[(j * 32 + lane) * 2 + 1];
          const float tmv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
          float lt[8], yo[8], ys[8];
          if (MODE & (CHK | WR)) ldg8(LT + off + (j * 32 + lane) * 8, lt);  // rare passes only
          if (MODE & CHK) ldg8(Yold + off + (j * 32 + lane) * 8, yo);
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const int e = 8 * j + r;
            const float k = A[e];
            if (MODE & (CHK | WR)) {
              const float Y = fmaf(sep::lg2f(k), LN2, Rl);
              if (MODE & CHK) {
                const float ea = sep::ex2f((yo[r] + Y) * LOG2E);
                const float eb = (lt[r] == -INFINITY) ? 0.f : sep::ex2f(lt[r] * LOG2E);
                ep += fabs((double)ea - (double)eb);
              }
              ys[r] = (lt[r] == -INFINITY) ? -INFINITY : lt[r] - Y;
              if (MODE & WR) b |= (ys[r] != ys[r]) | (ys[r] == INFINITY);
            }
            const float v = tmv[r] * Tr<float>::rcp(k);
            if (!(FS1_K3W_AGGNF && (MODE & FUSE))) b |= (v != v) | (v == INFINITY);
            A[e] = v;
          }
          if (MODE & WR) stg8(Yout + off + (j * 32 + lane) * 8, ys);
        }
        if (b) bad = 1;
        if (MODE & CHK) {
          ep = warp_sum(ep);
          if (lane == 0) c.s.red[w] = ep;
        }
      }
      if (t) t[4] = stm::gtimer() + (A[1] == 12345.f);
      if (MODE & FUSE) {
        int nf = 0;
        const int R2 = (MODE & UPD) ? line_apply_lin<E>(A, oe2, T, lane, FS1_K3W_AGGNF ? &nf : nullptr)
                                    : line_apply<E>(A, T, lane);
        if (FS1_K3W_AGGNF && (MODE & UPD) && nf) bad = 1;
        if (t) t[5] = stm::gtimer() + (R2 == 12345);
        const float Rl2 = (float)R2 * LN2;
        __syncwarp();  // every lane has read its target chunk (the stage aliases it)
        float4* st = reinterpret_cast<float4*>(stage + (size_t)w * C::SLINE + lane * C::SROW);
#pragma unroll
        for (int j = 0; j < E / 4; ++j)
          st[j] = make_float4(fmaf(sep::lg2f(A[4 * j]), LN2, Rl2), fmaf(sep::lg2f(A[4 * j + 1]), LN2, Rl2),
                              fmaf(sep::lg2f(A[4 * j + 2]), LN2, Rl2), fmaf(sep::lg2f(A[4 * j + 3]), LN2, Rl2));
      }
    } else {
      if ((MODE & CHK) && lane == 0) c.s.red[w] = 0.0;
      if (MODE & FUSE) {
        float4* st = reinterpret_cast<float4*>(stage + (size_t)w * C::SLINE + lane * C::SROW);
#pragma unroll
        for (int j = 0; j < E / 4; ++j) st[j] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
    }
    if ((MODE & (CHK | FUSE)) == 0) {
      __syncwarp();
      continue;
    }
    __syncthreads();
    if (t) t[6] = stm::gtimer();
    if (MODE & CHK) {  // line errors in line order (deterministic)
      if (c.tid == 0) {
        double s = 0.0;
        for (int k = 0; k < W; ++k) s += c.s.red[k];
        errsum += s;
      }
    }
    if (MODE & FUSE) {
      // position p of these W lines -> consumer line p, points grp W .. grp W + W - 1
      const int q0 = grp * W, lc = q0 / E, e0 = q0 - lc * E;  // same lane chunk (E >= 8)
      for (int p = c.tid; p < len; p += NT) {
        const int sp = (p / E) * C::SROW + (p % E);
        float v[W];
#pragma unroll
        for (int k = 0; k < W; ++k) v[k] = stage[(size_t)k * C::SLINE + sp];
        stg8(Zout + (size_t)p * C::LP + ((e0 >> 3) * 32 + lc) * 8, v);
      }
    }
    __syncthreads();
    if (t) t[7] = stm::gtimer();
    if (FS1_K3W_PREFETCH && TMn && grp + G >= ngroups) {
      // this warp's first line of the next pass (same group index c.r): its target line
      // goes into the now free stage region while the CTA waits at the grid barrier
      const int nl = c.r * W + w;
      if (nl < nln) {
        if (lane == 0) {
          stm::fence_async_smem();
          stm::mbar_expect_tx(&io.mb[1], (unsigned)C::LINEB);
          stm::bulk_g2s(io.ts, TMn + (size_t)nl * C::LP, (unsigned)C::LINEB, &io.mb[1]);
        }
        io.pre = 1;
      }
    }
  }
}

// Prologue: target logs (permuted lines) -> linear mantissas relative to one exponent
// per lane chunk (the update's numerator), exponents to X[line * 32 + lane].
template <int E>
__device__ __forceinline__ void to_mantissa(const sep::Ctx& c, const float* Lg, int nlines, float* M, int* X,
                                            int G) {
  using C = Cfg<E>;
  for (int line = c.r * W + c.warp; line < nlines; line += G * W) {
    float A[E];
    load_line<E>(Lg + (size_t)line * C::LP, c.lane, A);
    const int oe = prep_log<E>(A);
    store_line<E>(M + (size_t)line * C::LP, c.lane, A);
    X[(size_t)line * 32 + c.lane] = oe;
  }
}

// ------------------------------------------------------------ layout conversions
// dst (permuted lines, `lines` x LP) <- src natural: point q of line l is
// src[l * ls + q * qs] (f applied), padding -inf.  mode 0 copy, 1 log, 2 constant.
template <int E>
__device__ __forceinline__ void to_perm(const sep::Ctx& c, const float* src, long long ls, long long qs, int lines,
                                        int len, float* dst, int mode, float cst, int G) {
  using C = Cfg<E>;
  const size_t tot = (size_t)lines * C::LP;
  for (size_t k = (size_t)c.r * NT + c.tid; k < tot; k += (size_t)G * NT) {
    const int l = (int)(k / C::LP), s = (int)(k % C::LP);
    const int q = pinv<E>(s);
    float v = -INFINITY;
    if (q < len) {
      if (mode == 2) {
        v = cst;
      } else {
        v = __ldcg(src + (size_t)l * ls + (size_t)q * qs);
        if (mode == 1) v = logf(v);
      }
    }
    dst[k] = v;
  }
}
// natural dst[l * ls + q] <- permuted src line l point q (q < len)
template <int E>
__device__ __forceinline__ void from_perm(const sep::Ctx& c, const float* src, int lines, int len, float* dst,
                                          int G) {
  using C = Cfg<E>;
  const size_t tot = (size_t)lines * len;
  for (size_t k = (size_t)c.r * NT + c.tid; k < tot; k += (size_t)G * NT) {
    const int l = (int)(k / len), q = (int)(k % len);
    dst[k] = __ldcg(src + (size_t)l * C::LP + pidx<E>(q));
  }
}
__device__ __forceinline__ void fill(const sep::Ctx& c, float* dst, size_t cnt, float v, int G) {
  for (size_t k = (size_t)c.r * NT + c.tid; k < cnt; k += (size_t)G * NT) dst[k] = v;
}

// Grid barrier that also ORs one flag over the CTAs (non-check passes: no error sum).
// bar[1] is a sticky word (zeroed at launch with the barrier counter).
// FS1_K3W_FLAG64: bar[0] (counter) and bar[1] (flag word) are one aligned 8-byte pair and
// the spinning thread reads both with one 64-bit acquire load.  A CTA's OR precedes its
// release-add, so the load that sees the last arrival also sees every OR: no second L2
// round trip for the flag, and (called right after the caller's __syncthreads_or, with a
// block-uniform myflag) one block barrier per pass instead of four.
#ifndef FS1_K3W_FLAG64
#define FS1_K3W_FLAG64 1
#endif
// FS1_K3W_NOTF >= 1: no fence.proxy.async / __threadfence before the arrival (the pass's
// writes are generic-proxy stores, ordered by the block barrier and the red's own release,
// which is cumulative over the CTA).  2: no fence.proxy.async after the spin either: the only
// async-proxy (TMA) reads of the loop fetch the mantissa lines AM / BM, written once before
// the fully fenced stm::grid_barrier that precedes the loop; everything a pass produces is
// read back by generic ld.global.cg.
#ifndef FS1_K3W_NOTF
#define FS1_K3W_NOTF 2
#endif
__device__ __forceinline__ int grid_flag(sep::Ctx& c, const Sep2dParams& P, int myflag) {
#if FS1_K3W_FLAG64
  if (c.tid == 0) {
    if (myflag) atomicOr(&P.bar[1], 1u);
#if !FS1_K3W_NOTF
    stm::fence_async();
    __threadfence();
#endif
    const unsigned target = (c.gen + 1) * (unsigned)P.G;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bar) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(P.bar) : "memory");
    } while ((unsigned)v < target);
#if FS1_K3W_NOTF < 2
    stm::fence_async();
#endif
    c.s.ired[33] = (int)(v >> 32);
  }
  ++c.gen;
  __syncthreads();
  // the next write of ired[33] follows the next pass's block barriers: no trailing barrier
  return c.s.ired[33];
#else
  if (c.tid == 0 && myflag) atomicOr(&P.bar[1], 1u);
  stm::grid_barrier(P.bar, P.G, c.gen);
  if (c.tid == 0) c.s.ired[33] = (int)stm::ld_acquire(&P.bar[1]);
  __syncthreads();
  const int f = c.s.ired[33];
  __syncthreads();
  return f;
#endif
}

// ------------------------------------------------------------ the kernel (solve only)
template <int E, int MINB>
__global__ void __launch_bounds__(NT, MINB) fs1_sep2dw_kernel(const __grid_constant__ Sep2dParams P) {
  using C = Cfg<E>;
  extern __shared__ __align__(128) unsigned char smem[];
  sep::Ctx c;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  c.r = blockIdx.x;
  c.par = 0;
  c.gen = 0;
  c.s.stage = reinterpret_cast<float*>(smem);
  c.s.xm = reinterpret_cast<double*>(smem + C::OFF_XM);
  c.s.xi = reinterpret_cast<int*>(smem + C::OFF_XI);
  c.s.red = reinterpret_cast<double*>(smem + C::OFF_RED);
  c.s.ired = reinterpret_cast<int*>(smem + C::OFF_IRED);
  WarpIO io;
  io.ts = c.s.stage + (size_t)c.warp * C::SLINE;
  io.mb = reinterpret_cast<uint64_t*>(smem + C::OFF_MBAR) + 2 * c.warp;
  io.ph0 = io.ph1 = 0;
  io.pre = 0;
  if (c.lane == 0) {
    stm::mbar_init(&io.mb[0], 1);
    stm::mbar_init(&io.mb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int n = P.n, m = P.m, G = P.G;
  const float* A = reinterpret_cast<const float*>(P.a);
  const float* Bv = reinterpret_cast<const float*>(P.b);
  float* U = reinterpret_cast<float*>(P.u);
  float* V = reinterpret_cast<float*>(P.v);
  const AxT& T1 = P.wax[0];
  const AxT& T2 = P.wax[1];
  // permuted state: LA, F columns (m lines of n points); LBt, G rows (n lines of m);
  // Z1 rows (K1 phi, transposed), Z2 columns (K2 psi, transposed)
  float* LA = P.LA;
  float* LBt = P.LBt;
  float* Fp = P.Fp;
  float* Z1 = P.Z;
  float* Z2 = P.Z2;

  // ---- prologue: log a, (log b)^T, phi0 = psi0 = 1/(N M)
  const int li = P.input_is_log ? 0 : 1;
  to_perm<E>(c, A, n, 1, m, n, LA, li, 0.f, G);
  to_perm<E>(c, Bv, 1, n, n, m, LBt, li, 0.f, G);
  const float init = -logf((float)n) - logf((float)m);
  if (!P.warm) {
    to_perm<E>(c, nullptr, 0, 0, m, n, Fp, 2, init, G);
    to_perm<E>(c, nullptr, 0, 0, n, m, P.Gt0, 2, init, G);
  } else {
    to_perm<E>(c, U, n, 1, m, n, Fp, 0, 0.f, G);
    to_perm<E>(c, V, 1, n, n, m, P.Gt0, 0, 0.f, G);
  }
  fill(c, Z1, (size_t)n * C::LP, -INFINITY, G);
  fill(c, Z2, (size_t)m * C::LP, -INFINITY, G);
  stm::grid_barrier(P.bar, G, c.gen);
  // the update's numerators a, b as mantissas + per-lane-chunk exponents
  float* AM = P.AMp;
  float* BM = P.BMp;
  int* AX = P.AXe;
  int* BX = P.BXe;
  to_mantissa<E>(c, LA, m, AM, AX, G);
  to_mantissa<E>(c, LBt, n, BM, BX, G);
  double dummy = 0.0;
  int bad = 0;
  // Z1 = K1 on the columns of F, transposed
  fused_pass<E, FUSE>(c, io, T1, Fp, nullptr, nullptr, nullptr, nullptr, nullptr, Z1, m, n, G, dummy, bad);
  stm::grid_barrier(P.bar, G, c.gen);

  int l = 0, qi = 0, flag = 0;
  double errv = NAN;
  const bool use_tol = P.tol > 0.0;
  // the loop top checks at l >= itr_max, or every check_interval iterations with tol > 0
  auto is_check = [&](int k) { return (k >= P.itr_max) || (use_tol && (k % P.check_interval) == 0); };
  while (true) {
    const bool check = is_check(l);
    const bool last = l >= P.itr_max;
    // F^(l+1), G^(l+1) are stored only when the next loop top can stop on them (a check
    // reads psi^(l+1) and may return the state); otherwise they live in registers only
    // long enough to produce the next pass's input (Z1, Z2).
    const bool keep = is_check(l + 1);
    float* Gi = qi ? P.Gt1 : P.Gt0;
    float* Go = qi ? P.Gt0 : P.Gt1;
    double es = 0.0;
    bad = 0;
    // ---- pass R: psi half-step (Alg. 2 lines 3-7) + first pass of the phi half-step
    // (a check pass may stop the loop: no prefetch for the pass after it)
    if (last) fused_pass<E, UPD | CHK>(c, io, T2, Z1, BM, BX, LBt, Gi, Go, Z2, n, m, G, es, bad);
    else if (check && keep)
      fused_pass<E, UPD | WR | CHK | FUSE>(c, io, T2, Z1, BM, BX, LBt, Gi, Go, Z2, n, m, G, es, bad);
    else if (check) fused_pass<E, UPD | CHK | FUSE>(c, io, T2, Z1, BM, BX, LBt, Gi, Go, Z2, n, m, G, es, bad);
    else if (keep)
      fused_pass<E, UPD | WR | FUSE>(c, io, T2, Z1, BM, BX, LBt, nullptr, Go, Z2, n, m, G, es, bad, nullptr, AM, m);
    else fused_pass<E, UPD | FUSE>(c, io, T2, Z1, BM, BX, LBt, nullptr, Go, Z2, n, m, G, es, bad,
                                   (P.tdbg && l == 5) ? P.tdbg : nullptr, AM, m);
    bad = __syncthreads_or(bad);
    int f;
    double e = 0.0;
    if (check) e = sep::grid_sum(c, P, es, 0, f, bad);
    else f = grid_flag(c, P, bad);
    if (P.tdbg && l == 5 && c.tid == 0) P.tdbg[(size_t)G * W * 16 + c.r] = stm::gtimer();
    if (check) {
      errv = e;
      if (last || errv <= P.tol) {
        flag = (use_tol && errv <= P.tol) ? 1 : 4;
        break;
      }
    }
    if (keep) qi ^= 1;  // psi^(l+1) is the stored state
    if (f) { ++l; flag = 2; break; }
    // ---- pass C: phi half-step (lines 8-12) + first pass of the next psi half-step
    bad = 0;
    // the next R pass always runs (unless a flag stops the loop, drained below)
    if (keep) fused_pass<E, UPD | WR | FUSE>(c, io, T1, Z2, AM, AX, LA, nullptr, Fp, Z1, m, n, G, es, bad, nullptr, BM, n);
    else fused_pass<E, UPD | FUSE>(c, io, T1, Z2, AM, AX, LA, nullptr, Fp, Z1, m, n, G, es, bad, nullptr, BM, n);
    bad = __syncthreads_or(bad);
    f = grid_flag(c, P, bad);
    ++l;  // line 13
    if (f) { flag = 2; break; }
  }

  if (io.pre) {  // a prefetched target line nobody consumed (a flag stopped the loop)
    stm::mbar_wait(&io.mb[1], io.ph1);
    io.ph1 ^= 1u;
    io.pre = 0;
  }
  __syncthreads();

  // ---- outputs in the user layout: F column-major into u, G row-major natural (for the
  // cost) into the LA buffer, then transposed into v (column-major)
  float* Gc = qi ? P.Gt1 : P.Gt0;
  float* Gnat = LA;
  from_perm<E>(c, Fp, m, n, U, G);
  from_perm<E>(c, Gc, n, m, Gnat, G);
  stm::grid_barrier(P.bar, G, c.gen);
  double cost = NAN;
  if (flag != 2) {
    // return line on the CTA-line machinery: phi (W1 (x) K2) psi + psi (K1 (x) W2) phi
    float* Zc = Z1;   // K2 along rows of psi -> column-major (natural)
    float* Gs = Z2;   // K1 along columns of phi -> row-major (natural)
    sep::pass_transposed(c, P.ax2, Gnat, n, m, Zc, G);
    sep::pass_transposed(c, P.ax1, U, m, n, Gs, G);
    stm::grid_barrier(P.bar, G, c.gen);
    double s = 0.0;
    for (int j = c.r; j < m; j += G) s += sep::line_cost(c, P.ax1, Zc + (size_t)j * n, U + (size_t)j * n, n);
    for (int i = c.r; i < n; i += G) s += sep::line_cost(c, P.ax2, Gs + (size_t)i * m, Gnat + (size_t)i * m, m);
    int f;
    cost = sep::grid_sum(c, P, s, 2, f, 0);
  } else {
    errv = NAN;
  }
  sep::transpose_phase(c, Gnat, n, m, V, false, G);
  if (c.r == 0 && c.tid == 0) {
    if (P.iters) P.iters[0] = l;
    if (P.err) P.err[0] = errv;
    if (P.flags) P.flags[0] = flag;
    if (P.cost) P.cost[0] = cost;
  }
}

}  // namespace sepw
}  // namespace fs1
