// fs1_params.h — host/device parameter blocks of the FS-1 kernels (internal).
#pragma once
#include <stdint.h>

namespace fs1 {

// Persistent one-CTA-per-problem kernel (K1 in SURVEY.md §2.2).
// Scan multipliers are lambda^L for the spans L the kernel combines; they are
// formed on the host in fp64 by stepwise multiplication / exact exponent split
// (Remark 3.3) and never as exp(-L h/eps) in the kernel dtype.
struct PersistParams {
  const void* a;
  const void* b;
  void* u;
  void* v;
  int32_t* iters;
  double* err;
  int32_t* flags;
  double* cost;
  long long n;       // grid points per problem
  long long batch;
  double lam;        // lambda = e^{-h/eps}
  double h;
  double tol;
  int itr_max;
  int check_interval;
  int warm;          // u, v hold the initial state
  int input_is_log;  // a, b hold log-weights
  int write_uv;      // write the final state back to u, v
  double* dbg;       // optional per-half-step trace (debug builds of the tests only)
  // scaling domain: lambda^{E 2^k} = lvA[k] * lvB[k] (two factors: an underflow of the
  // power alone cannot zero a carry that is still representable, Remark 3.3)
  double lvA[5], lvB[5];
  double wA, wB;                 // lambda^{32 E}
  double laneA[32], laneB[32];   // lambda^{E l}
  // log domain (extended range): plain fp64 lambda^{E 2^k} for the warp scan, and
  // ER<double> (mantissa, exponent) forms of lambda^{E 2^k}, lambda^{32E}, lambda^{E l}
  double lvd[5];
  double lvm[6];
  int lve[6];
  double lanem[32];
  int lanee[32];
};

}  // namespace fs1
