/* fs1.h — C ABI of the B200-native FS-1 hot path (libfs1.so).
 *
 * FS-1 (Liao, Chen, Wang, Bai, Jin, Wu; arXiv 2202.10042) solves the
 * entropy-regularised Wasserstein-1 problem on a uniform grid,
 *
 *   min_gamma  sum_ij gamma_ij |i-j| h + eps gamma_ij ln gamma_ij       PAPER.md:69-75, Eq. (2.3)
 *   s.t. sum_j gamma_ij = a_i, sum_i gamma_ij = b_j,
 *
 * by Sinkhorn's iteration gamma = diag(phi) K diag(psi), K_ij = lambda^{|i-j|},
 * lambda = e^{-h/eps}
 *
 *   psi <- b ./ (K^T phi),   phi <- a ./ (K psi)          (psi first)
 *
 * where every K x is evaluated in O(N) by a forward and a backward
 * first-order recursion (Eq. "recursion"; Algorithm 1,
 * PAPER.md:141-165).  In 2D (Algorithm 2) the kernel is the
 * block-Toeplitz K = T_M(lambda2) (x) T_N(lambda1) and the cost is
 * |i1-i2| h1 + |j1-j2| h2.
 *
 * Notation map: the paper's histograms u, v are this ABI's
 * a, b; the paper's scalings phi, psi are this ABI's u, v.
 *
 * Conventions common to every entry point
 *  - Every data pointer is a DEVICE pointer owned by the caller; the library
 *    never allocates, frees or synchronises inside fs1_solve / fs1_cost /
 *    fs1_apply; every call is asynchronous on `stream` (a cudaStream_t,
 *    passed as void*, NULL = legacy default stream).
 *  - Batched layout: `batch` independent problems, each `n*m*l` contiguous
 *    values of the plan's dtype, problem-major: x[p*(n*m*l) + k].
 *    2D arrays are flattened column-major, k = j*n + i, i along axis 1 (h1),
 *    j along axis 2 (h2)
 *    3D (the extension of PAPER.md:314): k = (z*m + j)*n + i, z along axis 3 (h3).
 *  - Call-level errors are returned synchronously before any launch (only
 *    argument, shape and support problems are detected; data is not
 *    validated).  Per-problem outcomes go to device arrays.
 *  - The library holds no global mutable state; a plan is immutable after
 *    fs1_plan and may be shared by threads and streams; concurrent calls
 *    need distinct workspaces.
 */
#ifndef FS1_H
#define FS1_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS1_ABI_VERSION 2

typedef enum {
  FS1_OK = 0,
  FS1_ERR_ARG = 1,          /* NULL pointer, batch < 1, n < 1, m < 1, itr_max < 0, tol < 0, ... */
  FS1_ERR_EPS = 2,          /* eps <= 0 or h <= 0 or non-finite (SPEC's NonPositiveEpsilon)     */
  FS1_ERR_UNSUPPORTED = 3,  /* dtype / domain / size combination with no kernel                 */
  FS1_ERR_CUDA = 4,         /* a CUDA runtime error (launch failure, no device, ...)           */
  FS1_ERR_WORKSPACE = 5     /* workspace NULL or misaligned while the plan needs one           */
} fs1_status;

typedef enum { FS1_F32 = 0, FS1_F64 = 1 } fs1_dtype;

/* FS1_SCALING: u, v hold phi, psi; the plain (unstabilised) iteration of
 *              Algorithm 1; overflow terminates the problem (NONFINITE),
 *              as the paper's unstabilised runs do.
 * FS1_LOG:     u, v hold F = log phi, G = log psi.  Internally the kernels
 *              keep phi, psi as mantissas with one binary exponent per chunk
 *              of consecutive grid points, i.e. the absorption of Remark 2.1
 *              / Remark 3.2 carried out every
 *              half-step in exact powers of two.  It never
 *              overflows and matches the log-sum-exp iteration of the
 *              north star to rounding.
 * FS1_STABILIZED: the paper's own log-domain stabilisation (Remark 2.1 +
 *              Remark 3.2): the scaling-domain
 *              iteration on the rescaled kernel diag(e^{alpha/eps}) K
 *              diag(e^{beta/eps}) evaluated by the variable-coefficient
 *              recursions of Remark 3.2, with the absorption alpha += eps ln phi,
 *              beta += eps ln psi, phi = psi = 1 whenever max(|phi|, |psi|) >
 *              desc.tau after a full iteration (R8, R29, R30).  u, v hold
 *              F = alpha/eps + ln phi, G = beta/eps + ln psi (as FS1_LOG).  1D, fp64,
 *              n <= FS1_MAX_STAB, no warm start; fs1_apply is unsupported.       */
typedef enum { FS1_SCALING = 0, FS1_LOG = 1, FS1_STABILIZED = 2 } fs1_domain;
#define FS1_MAX_STAB 8192

/* per-problem flags (bit set) */
#define FS1_FLAG_CONVERGED 1  /* stopped because err <= tol (tol > 0)               */
#define FS1_FLAG_NONFINITE 2  /* phi or psi became non-finite ("terminates abnormally") */
#define FS1_FLAG_ITR_MAX 4    /* stopped at itr_max                                  */

typedef struct {
  int32_t ndim;          /* 1, 2 or 3 (3D: the separable extension PAPER.md:314 names; fp64
                            scaling domain, the K5 kernel)                                    */
  int64_t n;             /* points along axis 1 (>= 1)                                         */
  int64_t m;             /* points along axis 2 (1 for ndim == 1)                             */
  double h1, h2;         /* grid spacings (> 0); h2 ignored when ndim == 1                   */
  double eps;            /* regularisation epsilon (> 0)                                      */
  int64_t batch;         /* number of independent problems (>= 1)                             */
  fs1_dtype dtype;       /* element type of a, b, u, v                                        */
  fs1_domain domain;     /* see above                                                         */
  int32_t input_is_log;  /* FS1_LOG only: a, b hold log-weights (may be -inf)                */
  int32_t itr_max;       /* iteration cap (>= 0)                                              */
  double tol;            /* >= 0; stop when the marginal error <= tol;
                            0 = fixed iterations (the paper's §5 protocol)     */
  int32_t check_interval;/* >= 1: the error is evaluated when l % check_interval == 0       */
  int32_t warm_start;    /* 1: u, v hold the initial phi, psi (LOG: F, G); 0: 1/(n m)        */
  double tau;            /* FS1_STABILIZED: absorption threshold (> 1; 0 selects 1e10, the
                            reading of the unstated tau, R30); ignored otherwise   */
  int64_t l;             /* ndim == 3: points along axis 3 (>= 1); 0 or 1 otherwise         */
  double h3;             /* ndim == 3: axis-3 spacing (> 0); ignored otherwise              */
} fs1_desc;

typedef struct fs1_plan_s fs1_plan_t;

typedef struct {
  char kernel[48];       /* name of the kernel family chosen                                  */
  int32_t chunk;         /* grid points per thread (E)                                        */
  int32_t threads;       /* threads per CTA                                                   */
  int32_t ctas_per_problem;
  int64_t grid;          /* CTAs launched by fs1_solve                                        */
  size_t smem_bytes;     /* dynamic shared memory per CTA                                     */
  size_t workspace_bytes;
} fs1_plan_info_t;

/* fs1_plan — validate `desc`, choose a kernel, size the workspace.
 *   desc      : problem description (copied).
 *   device    : CUDA device ordinal the plan will run on.
 *   out       : receives the plan (free with fs1_plan_destroy).
 *   workspace_bytes : receives the device workspace fs1_solve / fs1_cost need
 *               (may be 0; pass a buffer of at least this size, 256-byte aligned).
 * Kernel choice: 1D problems that fit one CTA -> the persistent
 * one-CTA-per-problem kernel; larger 1D problems -> the multi-CTA HBM-streaming scan
 * kernel; 2D fp32 log -> the separable warp-per-line kernel; 2D and 3D fp64 scaling ->
 * the one-CTA-per-problem line kernel; FS1_STABILIZED -> the stabilised kernel.
 * Log domain range limits: a persistent chunk of E points needs
 * c E <= 40 (fp32) / 300 (fp64) and c 32 E <= 650 with c = h/eps; fs1_solve on a
 * streaming plan (fp64 log) needs c (min(n, 256) - 1) <= 600 and returns FS1_ERR_UNSUPPORTED
 * otherwise (fs1_apply has no such limit: its range is that of the data).
 * Returns FS1_ERR_ARG / FS1_ERR_EPS / FS1_ERR_UNSUPPORTED / FS1_ERR_CUDA.    */
fs1_status fs1_plan(const fs1_desc* desc, int device, fs1_plan_t** out, size_t* workspace_bytes);

/* fs1_solve — run Algorithm 1 (ndim 1) or Algorithm 2 (ndim 2) on every problem.
 *   a, b   : [batch][n*m] source / target histograms (paper's u, v), dtype of the plan;
 *            linear weights (> 0 in the scaling domain), or log-weights when
 *            desc.input_is_log (LOG domain).  Read only.
 *   u, v   : [batch][n*m] out (in, if warm_start): SCALING -> phi, psi;
 *            LOG -> F = log phi, G = log psi.  On return they hold the state
 *            (phi^(l), psi^(l)) at which the loop stopped;
 *            the kernels may use them as scratch during the solve, and a NONFINITE
 *            problem's u, v hold no defined state.
 *   iters  : [batch] int32, l at exit (number of completed iterations).
 *   err    : [batch] fp64, sum_i |psi_i (K^T phi)_i - b_i| evaluated on the exit
 *            state (PAPER.md:148 and §5's termination rule).
 *   flags  : [batch] int32, FS1_FLAG_* bits.
 *   cost   : [batch] fp64 or NULL; the return line
 *            sum_ij phi_i psi_j lambda^{|i-j|} |i-j| h (2D :339),
 *            evaluated in O(N) on the exit state.
 *   workspace : device buffer of fs1_plan's size (may be NULL if that size is 0).
 *   stream : cudaStream_t.
 * Problems are independent; a NONFINITE problem stops alone.                    */
fs1_status fs1_solve(const fs1_plan_t* plan, const void* a, const void* b, void* u, void* v,
                     int32_t* iters, double* err, int32_t* flags, double* cost,
                     void* workspace, void* stream);

/* fs1_cost — the return line alone, on caller-given u, v (same layout and
 * domain as fs1_solve's outputs).  cost: [batch] fp64.                          */
fs1_status fs1_cost(const fs1_plan_t* plan, const void* u, const void* v, double* cost,
                    void* workspace, void* stream);

/* fs1_apply — y = K x for each of the batch vectors (Eq. 3.1 / Eq. 4.x evaluated by
 * the recursion of PAPER.md:129-137 / 2D :300-309).  SCALING: x, y linear;
 * LOG: x, y are logs (y = log K e^x).  The kernel-level entry point used by the
 * parity tests.  x, y: [batch][n*m], must not alias.                             */
fs1_status fs1_apply(const fs1_plan_t* plan, const void* x, void* y, void* workspace, void* stream);

/* fs1_transport_plan — materialise gamma = diag(phi) K diag(psi) (
 * the plans compared in Tables 1-4, column 5) for problems of at most
 * FS1_MAX_TPLAN points (n*m): gamma[p][k][l] = phi_k lambda^{dist(k,l)} psi_l with
 * k, l flat indices (2D: column-major, l1 distance in cells weighted by h1, h2),
 * formed as exp(F_k + G_l - dist/eps) in fp64 and rounded once to the plan dtype.
 *   u, v  : [batch][n*m] state as fs1_solve returns it (LOG: F, G; SCALING: phi, psi).
 *   gamma : [batch][n*m][n*m], caller-owned, the plan dtype.
 * Errors: FS1_ERR_ARG (NULL), FS1_ERR_UNSUPPORTED (n*m > FS1_MAX_TPLAN).          */
#define FS1_MAX_TPLAN 8192
fs1_status fs1_transport_plan(const fs1_plan_t* plan, const void* u, const void* v, void* gamma, void* stream);

/* fs1_plan_entries — individual entries of the transport plan gamma = diag(phi) K diag(psi)
 * (gamma_ij = e^{-1/2-alpha_i/eps} K_ij e^{-1/2-beta_j/eps}; SPEC's
 * plan_entry) at caller-given index triples, for problems of any size and dimension
 * (no FS1_MAX_TPLAN limit: nothing N^2 is formed):
 *   gamma = exp(F_k + G_l - dist(k, l) / eps) in fp64, dist the l1 grid distance
 *   (1D h1 |k - l|; 2D / 3D per axis of the column-major flat indices (z m + j) n + i,
 *   weighted by h1, h2, h3); SCALING: F = log phi, G = log psi (phi_k = 0 or psi_l = 0
 *   gives 0); LOG / STABILIZED: u, v hold F, G.
 *   u, v  : [batch][size] state as fs1_solve returns it (device, plan dtype).
 *   idx   : [count][3] int64 (problem p, source flat index k, target flat index l), device.
 *   out   : [count] fp64, device, caller-owned.  count may be 0.
 * Errors: FS1_ERR_ARG (NULL plan, or NULL pointers with count > 0, or count < 0).  A
 * triple outside [0, batch) x [0, size)^2 writes NaN to its slot (not an error code:
 * the entries are computed asynchronously on `stream`).                            */
fs1_status fs1_plan_entries(const fs1_plan_t* plan, const void* u, const void* v, const int64_t* idx,
                            long long count, double* out, void* stream);

/* fs1_dual — the dual objective of the entropic problem Eq. (2.3) at the
 * state (u, v) as fs1_solve returns it:
 *   D = eps (sum_k a_k F_k + sum_l b_l G_l - sum_kl gamma_kl) + eps (sum a + sum b) / 2,
 *   gamma_kl = e^{F_k + G_l} K_kl,  F = log phi, G = log psi  (terms with zero weight count 0).
 * max D = W_eps (strong duality) and D <= the objective of every feasible plan; every
 * Sinkhorn half-step maximises D over one block.  One kernel apply (as fs1_apply) into
 * `scratch` ([batch][n*m] of the plan dtype, caller-owned) and one reduction.
 *   a, b : as for fs1_solve;  dual : [batch] fp64.
 * Errors: FS1_ERR_ARG, FS1_ERR_UNSUPPORTED (FS1_STABILIZED, or no apply for the plan).     */
fs1_status fs1_dual(const fs1_plan_t* plan, const void* a, const void* b, const void* u, const void* v,
                    void* scratch, double* dual, void* workspace, void* stream);

/* eps-scaling continuation (the slow convergence at small eps that
 * PAPER.md:529 names): Algorithm 1 / 2 at eps_k = max(eps, eps0 factor^k), k = 0, 1, ...,
 * each stage warm-started from the previous one with the dual potentials f = eps F,
 * g = eps G held fixed (F <- F eps_{k-1} / eps_k); intermediate stages run `stage_iters`
 * fixed iterations, the last (eps_k = desc->eps) desc->itr_max / tol / check_interval.
 * FS1_LOG only.  Outputs are the last stage's (iters counts its iterations only).
 * fs1_eps_scaling_plan returns the number of stages and the workspace the calls need;
 * the library creates and destroys one plan per stage on the host (no device allocation).
 * Errors: FS1_ERR_ARG (factor not in (0,1), eps0 < eps, ...), FS1_ERR_UNSUPPORTED,
 * FS1_ERR_WORKSPACE (workspace_bytes too small).                                            */
fs1_status fs1_eps_scaling_plan(const fs1_desc* desc, int device, double eps0, double factor, int32_t* stages,
                                size_t* workspace_bytes);
fs1_status fs1_solve_eps_scaling(const fs1_desc* desc, int device, double eps0, double factor, int32_t stage_iters,
                                 const void* a, const void* b, void* u, void* v, int32_t* iters, double* err,
                                 int32_t* flags, double* cost, void* workspace, size_t workspace_bytes,
                                 void* stream);

fs1_status fs1_plan_info(const fs1_plan_t* plan, fs1_plan_info_t* info);
void fs1_plan_destroy(fs1_plan_t* plan);
const char* fs1_status_string(fs1_status s);
int fs1_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FS1_H */
