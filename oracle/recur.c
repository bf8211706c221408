/* FS-1 ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * The paper's O(N) kernel apply written out literally, in plain sequential C,
 * fp64.  Used by the oracle where the dense O(N^2) apply is infeasible
 * (N = 2^24, 2048 x 2048).  Validated against the dense apply in
 * tests/test_oracle_apply.py wherever both run.
 *
 *  fs1o_sweep_scaling : Eq. (recursion), i.e. Algorithm 1
 *                       lines 3-6:
 *                         r_1 = x_1, r_{i+1} = lam r_i + x_{i+1}
 *                         s_N = 0,   s_{N-i} = lam (s_{N-i+1} + x_{N-i+1})
 *                         y = r + s
 *  fs1o_sweep_log     : the same two sweeps in log-sum-exp form
 *                       (BASELINE.json north_star), c = h/eps:
 *                         R_1 = X_1, R_{i+1} = logaddexp(R_i - c, X_{i+1})
 *                         S_N = -inf, S_{N-i} = -c + logaddexp(S_{N-i+1}, X_{N-i+1})
 *                         Y = logaddexp(R, S)
 *  fs1o_wsweep_log    : log of the distance-weighted apply whose bilinear form
 *                       is Algorithm 1's return line:
 *                       (W x)_k = sum_j |k-j| h lam^{|k-j|} x_j, from
 *                         P'_1 = 0, P'_{k+1} = lam (P'_k + p_k)   (p = inclusive forward sum)
 *                         Q'_N = 0, Q'_k = lam (Q'_{k+1} + t_{k+1}) (t = inclusive backward sum)
 *                       (W x)_k = h (P'_k + Q'_k).  SURVEY.md §8(c) Q7 / DESIGN.md R7.
 *
 * Precision: the log-sum-exp sweeps accumulate in x87 extended precision
 * (long double, 64-bit significand).  In fp64 the sequential LSE recursion
 * drifts by ~ulp(|R|) per step over its memory 1/(1 - lambda): at config 3
 * (|F| ~ 1e4, 1/(1-lambda) ~ 1700) that is ~2e-9 relative in e^R, above the
 * 1e-10 parity gate it has to certify (R24).  The recursion itself is
 * unchanged; only its accumulator is wider.  Results are rounded to fp64.
 *
 * Every routine works on `lines` independent lines of `n` points with element
 * stride `stride` and line stride `lstride` (2D: axis 1 = columns, contiguous;
 * axis 2 = rows, stride N; PAPER.md:244-255 column-major flattening).
 * Lines are independent (PAPER.md:282-312 applies K0 column by column), so the
 * loop over lines may run in parallel; arithmetic within a line is sequential.
 */
#include <math.h>
#include <stdlib.h>

typedef long double ld;

static ld lae(ld a, ld b) {                        /* log(e^a + e^b), extended */
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  ld m = a > b ? a : b;
  return m + log1pl(expl(-fabsl(a - b)));
}

void fs1o_sweep_scaling(const double* x, long n, long stride, long lines, long lstride,
                        double lam, double* y) {
#pragma omp parallel for schedule(static)
  for (long l = 0; l < lines; ++l) {
    const double* xl = x + l * lstride;
    double* yl = y + l * lstride;
    double* r = (double*)malloc(sizeof(double) * n);
    double* s = (double*)malloc(sizeof(double) * n);
    r[0] = xl[0];
    s[n - 1] = 0.0;
    for (long i = 1; i <= n - 1; ++i) {              /* for i = 1 : N-1 (1-based) */
      r[i] = lam * r[i - 1] + xl[i * stride];        /* r_{i+1} = lam r_i + x_{i+1} */
      long k = n - 1 - i;                            /* 0-based index of s_{N-i}    */
      s[k] = lam * (s[k + 1] + xl[(k + 1) * stride]);/* s_{N-i} = lam(s_{N-i+1}+x_{N-i+1}) */
    }
    for (long i = 0; i < n; ++i) yl[i * stride] = r[i] + s[i];
    free(r);
    free(s);
  }
}

/* The two sweeps of one line are independent of each other (lines 5 and 6 of
 * Algorithm 1 read only x), so they are written as two loops; for a single line
 * (config 3) they run on two threads.  Each sweep is still sequential and its
 * arithmetic is unchanged. */
static void fwd_log(const double* xl, long n, long stride, ld C, ld* r) {
  r[0] = xl[0];
  for (long i = 1; i <= n - 1; ++i) r[i] = lae(r[i - 1] - C, (ld)xl[i * stride]);
}

static void bwd_log(const double* xl, long n, long stride, ld C, ld* s) {
  s[n - 1] = -INFINITY;
  for (long i = 1; i <= n - 1; ++i) {
    long k = n - 1 - i;
    s[k] = -C + lae(s[k + 1], (ld)xl[(k + 1) * stride]);
  }
}

void fs1o_sweep_log(const double* X, long n, long stride, long lines, long lstride,
                    double c, double* Y) {
  const ld C = (ld)c;
  if (lines == 1) {
    ld* r = (ld*)malloc(sizeof(ld) * n);
    ld* s = (ld*)malloc(sizeof(ld) * n);
#pragma omp parallel sections num_threads(2)
    {
#pragma omp section
      fwd_log(X, n, stride, C, r);
#pragma omp section
      bwd_log(X, n, stride, C, s);
    }
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) Y[i * stride] = (double)lae(r[i], s[i]);
    free(r);
    free(s);
    return;
  }
#pragma omp parallel for schedule(static)
  for (long l = 0; l < lines; ++l) {
    const double* xl = X + l * lstride;
    double* yl = Y + l * lstride;
    ld* r = (ld*)malloc(sizeof(ld) * n);
    ld* s = (ld*)malloc(sizeof(ld) * n);
    fwd_log(xl, n, stride, C, r);
    bwd_log(xl, n, stride, C, s);
    for (long i = 0; i < n; ++i) yl[i * stride] = (double)lae(r[i], s[i]);
    free(r);
    free(s);
  }
}

/* The weighted sweeps of one line: (p, P') forward and (t, Q') backward are independent
 * of each other; for a single line (config 3's cost) they run on two threads, each
 * still sequential with unchanged arithmetic. */
static void wfwd_log(const double* xl, long n, long stride, ld C, ld* p, ld* P) {
  p[0] = xl[0];
  for (long i = 1; i < n; ++i) p[i] = lae(p[i - 1] - C, (ld)xl[i * stride]);
  P[0] = -INFINITY;
  for (long i = 1; i < n; ++i) P[i] = -C + lae(P[i - 1], p[i - 1]);
}

static void wbwd_log(const double* xl, long n, long stride, ld C, ld* t, ld* Q) {
  t[n - 1] = xl[(n - 1) * stride];
  for (long i = n - 2; i >= 0; --i) t[i] = lae(t[i + 1] - C, (ld)xl[i * stride]);
  Q[n - 1] = -INFINITY;
  for (long i = n - 2; i >= 0; --i) Q[i] = -C + lae(Q[i + 1], t[i + 1]);
}

void fs1o_wsweep_log(const double* X, long n, long stride, long lines, long lstride,
                     double c, double h, double* Y) {
  const ld C = (ld)c;
  const ld lh = logl((ld)h);
  if (lines == 1) {
    ld* p = (ld*)malloc(sizeof(ld) * n);   /* log inclusive forward sums  */
    ld* t = (ld*)malloc(sizeof(ld) * n);   /* log inclusive backward sums */
    ld* P = (ld*)malloc(sizeof(ld) * n);   /* log P'                       */
    ld* Q = (ld*)malloc(sizeof(ld) * n);   /* log Q'                       */
#pragma omp parallel sections num_threads(2)
    {
#pragma omp section
      wfwd_log(X, n, stride, C, p, P);
#pragma omp section
      wbwd_log(X, n, stride, C, t, Q);
    }
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) Y[i * stride] = (double)(lh + lae(P[i], Q[i]));
    free(p);
    free(t);
    free(P);
    free(Q);
    return;
  }
#pragma omp parallel for schedule(static)
  for (long l = 0; l < lines; ++l) {
    const double* xl = X + l * lstride;
    double* yl = Y + l * lstride;
    ld* p = (ld*)malloc(sizeof(ld) * n);
    ld* t = (ld*)malloc(sizeof(ld) * n);
    ld* P = (ld*)malloc(sizeof(ld) * n);
    ld* Q = (ld*)malloc(sizeof(ld) * n);
    wfwd_log(xl, n, stride, C, p, P);
    wbwd_log(xl, n, stride, C, t, Q);
    for (long i = 0; i < n; ++i) yl[i * stride] = (double)(lh + lae(P[i], Q[i]));
    free(p);
    free(t);
    free(P);
    free(Q);
  }
}

/* sum_k exp(A_k + B_k) over n entries, in fp64 (cost and error reductions). */
double fs1o_sum_exp2(const double* A, const double* B, long n) {
  ld s = 0.0L;
  for (long i = 0; i < n; ++i) {
    ld v = (ld)A[i] + (ld)B[i];
    if (v != -INFINITY) s += expl(v);
  }
  return (double)s;
}

/* fs1o_stab_sweep : Remark 3.2's replacement lines, the
 *                   paper's log-domain-stabilised recursion, in plain fp64.
 *   With the absorbed potentials read as alpha <- alpha + eps ln phi (DESIGN.md
 *   R8) and passed divided by eps (own = beta/eps, other = alpha/eps for lines
 *   5-6, the psi half-step; own = alpha/eps, other = beta/eps for lines 10-11,
 *   the phi half-step):
 *     r_1     = e^{other_1 + own_1} x_1                       (line 3, rescaled: R29)
 *     r_{i+1} = lam e^{own_{i+1} - own_i} r_i + e^{other_{i+1} + own_{i+1}} x_{i+1}     (line 5 / 10)
 *     s_N     = 0
 *     s_{N-i} = lam e^{own_{N-i} - own_{N-i+1}} (s_{N-i+1} + e^{other_{N-i+1} + own_{N-i+1}} x_{N-i+1})
 *                                                                                      (line 6 / 11)
 *     y = r + s  (= diag(e^own) K diag(e^other) x, the rescaled kernel of Remark 2.1)
 * Each factor is formed exactly as printed: lam * exp(difference), exp(sum). */
void fs1o_stab_sweep(const double* x, const double* own, const double* other, long n, double lam,
                     double* y) {
  double* r = (double*)malloc(sizeof(double) * n);
  double* s = (double*)malloc(sizeof(double) * n);
  r[0] = exp(other[0] + own[0]) * x[0];
  s[n - 1] = 0.0;
  for (long i = 1; i <= n - 1; ++i) {            /* for i = 1 : N-1 (1-based) */
    r[i] = lam * exp(own[i] - own[i - 1]) * r[i - 1] + exp(other[i] + own[i]) * x[i];
    long k = n - 1 - i;                          /* 0-based index of s_{N-i} */
    s[k] = lam * exp(own[k] - own[k + 1]) * (s[k + 1] + exp(other[k + 1] + own[k + 1]) * x[k + 1]);
  }
  for (long i = 0; i < n; ++i) y[i] = r[i] + s[i];
  free(r);
  free(s);
}
