// fs1_common.cuh — device helpers shared by the FS-1 kernels (sm_100a).
//
// * Tr<T>      : per-dtype bit tricks (exact powers of two, exponent extraction,
//                reciprocal) used by the chunk-exponent ("extended range")
//                representation of the log domain.
// * ER<T>      : extended-range number m * 2^e, m in [1,2) or 0.  It carries the
//                scan carries between chunks of the log-domain kernels so that a
//                carry lambda^L * x never underflows in isolation (Remark 3.3,
//                "stepwise multiplication of lambda").
// * warp/block reductions (deterministic trees, no float atomics).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fs1 {

constexpr unsigned FULL = 0xffffffffu;
constexpr int ZE = -(1 << 28);  // exponent of an ER zero

template <class T> struct Tr;

template <> struct Tr<float> {
  using V = float4;
  static constexpr int VEC = 4;
  static constexpr int LIM = 60;  // carries up to 2^LIM above a chunk stay in the fast path
  __device__ __forceinline__ static float pow2(int d) {  // exact 2^d, 0 below 2^-126
    d = min(d, 127);
    return d >= -126 ? __uint_as_float((unsigned)(d + 127) << 23) : 0.f;
  }
  __device__ __forceinline__ static int expo(float m) {  // unbiased exponent of a normal m
    return (int)((__float_as_uint(m) >> 23) & 0xffu) - 127;
  }
  __device__ __forceinline__ static float mant(float m) {  // m with exponent 0 -> [1,2)
    return __uint_as_float((__float_as_uint(m) & 0x807fffffu) | 0x3f800000u);
  }
  __device__ __forceinline__ static float rcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
  template <bool NEWTON = false>
  __device__ __forceinline__ static float div(float t, float x) { return t * rcp(x); }
  __device__ __forceinline__ static void unpack(const V& v, float* o) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  __device__ __forceinline__ static V pack(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
};

template <> struct Tr<double> {
  using V = double2;
  static constexpr int VEC = 2;
  static constexpr int LIM = 600;
  __device__ __forceinline__ static double pow2(int d) {
    d = min(d, 1023);
    return d >= -1022 ? __longlong_as_double((long long)(d + 1023) << 52) : 0.0;
  }
  __device__ __forceinline__ static int expo(double m) {
    return (int)((__double_as_longlong(m) >> 52) & 0x7ff) - 1023;
  }
  __device__ __forceinline__ static double mant(double m) {
    return __longlong_as_double((__double_as_longlong(m) & 0x800fffffffffffffLL) |
                                0x3ff0000000000000LL);
  }
  __device__ __forceinline__ static double rcp(double x) { return __drcp_rn(x); }
  // t / x two ways.  NEWTON: reciprocal estimate, one Newton step, one residual
  // correction of the quotient (< 1 ulp, no branch; x = 0 or non-finite ->
  // non-finite): the shorter dependency chain, faster where latency binds (one
  // problem on a few warps: C1 1.47 -> 1.26 ms).  Otherwise t * rcp.rn(x): fewer fp64
  // pipe operations, faster where throughput binds (E1/E2: 3.5%).
  template <bool NEWTON = false>
  __device__ __forceinline__ static double div(double t, double x) {
    if constexpr (NEWTON) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
      const double e = fma(-x, r, 1.0);
      r = fma(r, e, r);
      const double q = t * r;
      return fma(r, fma(-x, q, t), q);
    } else {
      return t * __drcp_rn(x);
    }
  }
  __device__ __forceinline__ static void unpack(const V& v, double* o) { o[0] = v.x; o[1] = v.y; }
  __device__ __forceinline__ static V pack(const double* o) { return make_double2(o[0], o[1]); }
};

__device__ __forceinline__ double pow2d(int d) { return Tr<double>::pow2(d); }

template <class T> struct ER {
  T m;
  int e;
};

template <class T> __device__ __forceinline__ ER<T> er_zero() { return ER<T>{T(0), ZE}; }

// normalise m * 2^e (m >= 0 finite, normal or zero)
template <class T> __device__ __forceinline__ ER<T> er_norm(T m, int e) {
  ER<T> r;
  bool z = !(m > T(0));
  r.m = z ? T(0) : Tr<T>::mant(m);
  r.e = z ? ZE : e + Tr<T>::expo(m);
  return r;
}

template <class T> __device__ __forceinline__ ER<T> er_add(ER<T> a, ER<T> b) {
  int e = max(a.e, b.e);
  T m = a.m * Tr<T>::pow2(a.e - e) + b.m * Tr<T>::pow2(b.e - e);
  return er_norm<T>(m, e);
}

template <class T> __device__ __forceinline__ ER<T> er_mul(ER<T> a, ER<T> b) {
  return er_norm<T>(a.m * b.m, a.e + b.e);
}

template <class T> __device__ __forceinline__ ER<T> er_scale(ER<T> a, T s) {  // s > 0 plain
  return er_norm<T>(a.m * s, a.e);
}

// value relative to 2^R as double (flushes below 2^-1022)
template <class T> __device__ __forceinline__ double er_rel(ER<T> a, int R) {
  return (double)a.m * pow2d(a.e - R);
}

template <class T> __device__ __forceinline__ ER<T> shfl_up_er(ER<T> a, int d) {
  ER<T> r;
  r.m = __shfl_up_sync(FULL, a.m, d);
  r.e = __shfl_up_sync(FULL, a.e, d);
  return r;
}
template <class T> __device__ __forceinline__ ER<T> shfl_down_er(ER<T> a, int d) {
  ER<T> r;
  r.m = __shfl_down_sync(FULL, a.m, d);
  r.e = __shfl_down_sync(FULL, a.e, d);
  return r;
}

template <class T> __device__ __forceinline__ ER<T> shfl_idx_er(ER<T> a, int src) {
  ER<T> r;
  r.m = __shfl_sync(FULL, a.m, src);
  r.e = __shfl_sync(FULL, a.e, src);
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
// one REDUX.SYNC instruction each (instead of a 5-level shuffle tree)
__device__ __forceinline__ int warp_max(int v) { return __reduce_max_sync(FULL, v); }
__device__ __forceinline__ int warp_min(int v) { return __reduce_min_sync(FULL, v); }

// Warp scan step without selects: the shuffle's in-range predicate guards the FMA.
// up:   v + m * v[lane - d]  (lane >= d), else v
// down: v + m * v[lane + d]  (lane + d < 32), else v
#ifndef FS1_SCAN_SELM
#define FS1_SCAN_SELM 1
#endif
#if FS1_SCAN_SELM
// Variant: the shuffle's predicate selects the multiplier (m or 0) and one FMA updates v in
// place (out-of-range lanes get their own value back, times 0).
__device__ __forceinline__ double scan_up(double v, unsigned d, double m) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, a, b;\n\t.reg .f64 s, mm;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "shfl.sync.up.b32 a|p, lo, %1, 0, -1;\n\t"
      "shfl.sync.up.b32 b, hi, %1, 0, -1;\n\t"
      "mov.b64 s, {a, b};\n\t"
      "selp.f64 mm, %2, 0d0000000000000000, p;\n\t"
      "fma.rn.f64 %0, mm, s, %0;\n\t}"
      : "+d"(v)
      : "r"(d), "d"(m));
  return v;
}
__device__ __forceinline__ double scan_down(double v, unsigned d, double m) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, a, b;\n\t.reg .f64 s, mm;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "shfl.sync.down.b32 a|p, lo, %1, 31, -1;\n\t"
      "shfl.sync.down.b32 b, hi, %1, 31, -1;\n\t"
      "mov.b64 s, {a, b};\n\t"
      "selp.f64 mm, %2, 0d0000000000000000, p;\n\t"
      "fma.rn.f64 %0, mm, s, %0;\n\t}"
      : "+d"(v)
      : "r"(d), "d"(m));
  return v;
}
#else
__device__ __forceinline__ double scan_up(double v, unsigned d, double m) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, a, b;\n\t.reg .f64 s;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "shfl.sync.up.b32 a|p, lo, %1, 0, -1;\n\t"
      "shfl.sync.up.b32 b, hi, %1, 0, -1;\n\t"
      "mov.b64 s, {a, b};\n\t"
      "@p fma.rn.f64 %0, %2, s, %0;\n\t}"
      : "+d"(v)
      : "r"(d), "d"(m));
  return v;
}
__device__ __forceinline__ double scan_down(double v, unsigned d, double m) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, a, b;\n\t.reg .f64 s;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "shfl.sync.down.b32 a|p, lo, %1, 31, -1;\n\t"
      "shfl.sync.down.b32 b, hi, %1, 31, -1;\n\t"
      "mov.b64 s, {a, b};\n\t"
      "@p fma.rn.f64 %0, %2, s, %0;\n\t}"
      : "+d"(v)
      : "r"(d), "d"(m));
  return v;
}
#endif
// exclusive neighbours: v[lane-1] (0 at lane 0) and v[lane+1] (0 at lane 31)
__device__ __forceinline__ double prev_or0(double v) {
  double r = 0.0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, a, b;\n\t"
      "mov.b64 {lo, hi}, %1;\n\t"
      "shfl.sync.up.b32 a|p, lo, 1, 0, -1;\n\t"
      "shfl.sync.up.b32 b, hi, 1, 0, -1;\n\t"
      "@p mov.b64 %0, {a, b};\n\t}"
      : "+d"(r)
      : "d"(v));
  return r;
}
__device__ __forceinline__ double next_or0(double v) {
  double r = 0.0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, a, b;\n\t"
      "mov.b64 {lo, hi}, %1;\n\t"
      "shfl.sync.down.b32 a|p, lo, 1, 31, -1;\n\t"
      "shfl.sync.down.b32 b, hi, 1, 31, -1;\n\t"
      "@p mov.b64 %0, {a, b};\n\t}"
      : "+d"(r)
      : "d"(v));
  return r;
}
}  // namespace fs1
