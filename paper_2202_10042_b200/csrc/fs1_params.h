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
  double lamH;       // lambda^{E/2}: carry between the two halves of a thread chunk (ILP)
  double h;
  double tol;
  int itr_max;
  int check_interval;
  int warm;          // u, v hold the initial state
  int input_is_log;  // a, b hold log-weights
  int write_uv;      // write the final state back to u, v
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


// Multi-CTA HBM-streaming kernel (K2 in SURVEY.md §2.2), fp64, one problem per launch.
// The state lives in the workspace as mantissas with one binary exponent per 256-point
// tile; tile exponents and scan tables stay in shared memory of
// the CTA that owns the tile range for the whole solve.
struct StreamParams {
  const void* a;     // [n] histograms (fp64; log-weights when input_is_log)
  const void* b;
  void* u;           // [n] out (in when warm): F = log phi (or phi for the apply/scaling views)
  void* v;
  int32_t* iters;
  double* err;
  int32_t* flags;
  double* cost;
  const void* x;     // apply: input  [n]
  void* y;           // apply: output [n]
  double* Am;        // workspace mantissas [npad]
  double* Bm;
  double* Pm;        // phi state
  double* Qm0;       // psi state, ping-pong pair (check iterations keep psi^(l))
  double* Qm1;
  double* gtot;      // [2 parity][G][4]: forward total m, backward total m, err, cost
  int* gtote;        // [2 parity][G][4]: forward total e, backward total e, flag, cost e
  double* gtot2;     // [G][8] cost-phase range totals (p, P', t, Q') m
  int* gtot2e;       // [G][8]
  unsigned* bar;     // grid barrier {count, generation}
  unsigned long long* tdbg;  // optional phase timestamps (test-only), [G][64 half-steps][8]
  long long n;
  long long npad;    // ntiles * 256
  int ntiles;
  int G;             // CTAs (co-resident)
  int ntmax;         // max tiles per CTA
  double lam;
  double h;
  double tol;
  int itr_max;
  int check_interval;
  int warm;
  int input_is_log;
  int mode;          // 0 solve, 1 apply, 2 cost
  int logd;          // 1: u, v, x, y are logs; 0: linear
  double lvd[5];     // lambda^{8 * 2^k}
  double lanepow[32];  // lambda^{8 l}
  double t2m[20];    // lambda^{256 * 2^j} as mantissa in [1,2) ...
  int t2e[20];       // ... and binary exponent (Remark 3.3: never formed alone in fp64)
};

// Separable 2D kernel (K3 in SURVEY.md §2.2), fp32 log domain, one problem per launch.
struct Sep2dParams {
  PersistParams ax1;  // scan tables of axis 1 (lambda1 = e^{-h1/eps}, h1), E = 8
  PersistParams ax2;  // axis 2 (lambda2, h2)
  const void* a;      // [n*m] column-major (log-weights when input_is_log)
  const void* b;
  void* u;            // [n*m] F = log phi, column-major (state, in place)
  void* v;            // [n*m] G = log psi, column-major (written at exit)
  int32_t* iters;
  double* err;
  int32_t* flags;
  double* cost;
  const void* x;      // apply input / output (column-major logs)
  void* y;
  float* LA;          // [n*m] log a, column-major
  float* LBt;         // [m*n] log b, row-major (transposed)
  float* Gt0;         // [m*n] G, row-major, ping-pong pair
  float* Gt1;
  float* Z;           // [n*m] pass scratch
  float* Z2;          // K3w: [m][LP] second transposed scratch (permuted lines)
  float* Fp;          // K3w: [m][LP] F state (permuted lines)
  float* AMp;         // K3w: [m][LP] a as mantissas per lane chunk (permuted lines)
  float* BMp;         // K3w: [n][LP] b (row lines)
  int* AXe;           // K3w: [m][32] exponents of the lane chunks of a
  int* BXe;           // K3w: [n][32]
  double* part;       // [3][G] per-CTA partial sums
  int* flagp;         // [3][G]
  unsigned* bar;
  int n, m, G;
  double tol;
  int itr_max, check_interval, warm, input_is_log, mode;
  // K3w (warp-per-line solve): chunk E (0 = CTA-line kernel K3), per-axis scan tables
  int wE;
  unsigned long long* tdbg;  // optional phase timestamps (test-only): [G][W][2 groups][8]
  struct WAx {
    float lam, lamH;  // lambda_k, lambda_k^{E/2}
    float Lm[5];      // lambda_k^{E 2^j} = Lm 2^Le (Remark 3.3)
    int Le[5];
  } wax[2];
};

// One 1D problem sharded over ranks by contiguous whole-tile segments (K2s,
// fs1_shard.cuh), fp64 log domain.  Per-rank scalars and tables; the workspace
// pointers live in the host plan and are passed per launch.
#ifndef FS1_SHARD_MAXW
#define FS1_SHARD_MAXW 16  // ranks of a fused (mailbox) exchange
#endif
struct ShardParams {
  long long n;       // global points N
  long long lo;      // first global point of this segment (multiple of 256)
  long long len;     // segment points (T * 256; the last segment's tail past N is padding)
  long long T0;      // global index of the first tile
  long long Ttot;    // global tiles
  int T;             // tiles of this segment
  int TB, nblk;      // tiles per block (one CTA of the tile kernels), blocks
  int world, rank;
  double lam, h;
  double lvd[5];       // lambda^{8 2^k}
  double lvm8[5];      // ... as (mantissa, exponent)
  int lve8[5];
  double lanepow[32];  // lambda^{8 l}
  double t2m[40];      // lambda^{256 2^j} = t2m 2^t2e (Remark 3.3)
  int t2e[40];
  // Fused exchange (fs1_shard_set_mailboxes): every rank's mailbox, box[rank] = own,
  // peers' through NVLink peer / IPC mappings; fused = 0: totals come from all_tot.
  int fused;
  double* box[FS1_SHARD_MAXW];
};

}  // namespace fs1

namespace fs1 {

// K4: the paper's stabilised FS-1 (Remark 2.1 + 3.2), fp64, one CTA per problem.
struct StabParams {
  const void* a;     // [batch][n] histograms (linear; log-weights when input_is_log)
  const void* b;
  void* u;           // [batch][n] out: F = alpha/eps + ln phi
  void* v;           //               G = beta/eps + ln psi
  int32_t* iters;
  double* err;
  int32_t* flags;
  double* cost;
  double* ws;        // [batch][9][T E] workspace (fs1_stab.cuh WN arrays)
  long long n;
  double lam;        // lambda = e^{-h/eps}
  double h;
  double tol;
  double tau;        // absorption threshold (Remark 2.1)
  int itr_max;
  int check_interval;
  int input_is_log;
  int mode;          // 0 solve; 1 cost of the given (u, v) = (F, G)
};

}  // namespace fs1

namespace fs1 {

// K5: Algorithm 2 (and its 3D extension) in fp64, scaling domain, one CTA per problem
// (fs1_sep2d64.cu).
struct Sep2d64Params {
  const double* a;   // [batch][n m] column-major histograms
  const double* b;
  double* u;         // [batch][n m] phi (in when warm)
  double* v;         //              psi
  int32_t* iters;
  double* err;
  int32_t* flags;
  double* cost;
  const double* x;   // apply: input / output
  double* y;
  double* ws;        // [batch][3][n m l]
  int n, m, l;       // l = 1 in 2D
  double lam1, lam2, lam3, h1, h2, h3, tol;
  int itr_max, check_interval, warm;
  int mode;          // 0 solve, 1 cost, 2 apply
  int staged;        // 2D with n m <= SMEM_NM: the intermediate lives in shared memory
  int wE;            // > 0: the warp-per-line variant K5w with chunk E (2D, max(n, m) <= 32 E)
  double wA1[5], wB1[5], wA2[5], wB2[5];  // K5w: lambda^{E 2^k} per axis as two factors
};

}  // namespace fs1
