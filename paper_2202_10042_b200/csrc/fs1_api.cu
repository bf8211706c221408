// fs1_api.cu — the C ABI of include/fs1.h: plan validation, kernel choice,
// scan-multiplier tables and launches.  No device allocation, no synchronisation.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>

#include "../../include/fs1.h"
#include "fs1_dispatch.h"
#include "fs1_params.h"

using namespace fs1;

struct fs1_plan_s {
  fs1_desc d;
  int device;
  int kind;  // 0 persistent
  const PersistEntry* pe;
  PersistParams base;  // multipliers + scalars; pointers filled per call
  const StreamEntry* se;
  StreamParams sbase;  // K2: scalars + multiplier tables; pointers filled per call
  Sep2dParams tbase;   // K3
  const StabEntry* ke = nullptr;  // K4 stabilised kernel
  StabParams kbase;
  Sep2d64Params dbase;            // K5 fp64 2D kernel
  int threads = 0;
  int grid;            // K2 / K3: co-resident CTAs
  const Sep2dwEntry* sw = nullptr;  // K3w solve kernel (nullptr: K3)
  int gridw = 0;                    // K3w co-resident CTAs
  size_t smem;         // dynamic shared memory per CTA (>= the kernel's need; sized for occupancy)
  size_t ws;
  fs1_plan_info_t info;
};

namespace {

constexpr int KIND_PERSIST = 0;
constexpr int KIND_STREAM = 1;
constexpr int KIND_SEP2D = 2;
constexpr int KIND_STAB = 3;
constexpr int KIND_SEP64 = 4;
void er_pow(long double c, long double L, double* m, int* e);
void fill_persist_tables(PersistParams& P, double c, int E);
constexpr int TILE = 256;

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// workspace of the streaming kernel: 5 mantissa vectors + grid scratch
struct StreamWs {
  size_t Am, Bm, Pm, Qm0, Qm1, gtot, gtote, gtot2, gtot2e, bar, total;
};
StreamWs stream_ws(long long npad, int G) {
  StreamWs w;
  size_t o = 0;
  const size_t v = al256((size_t)npad * 8);
  w.Am = o; o += v;
  w.Bm = o; o += v;
  w.Pm = o; o += v;
  w.Qm0 = o; o += v;
  w.Qm1 = o; o += v;
  w.gtot = o; o += al256((size_t)2 * G * 4 * 8);
  w.gtote = o; o += al256((size_t)2 * G * 4 * 4);
  w.gtot2 = o; o += al256((size_t)G * 8 * 8);
  w.gtot2e = o; o += al256((size_t)G * 8 * 4);
  w.bar = o; o += 256;
  w.total = o;
  return w;
}

void fill_stream_tables(StreamParams& P, double c) {
  const long double C = (long double)c;
  for (int k = 0; k < 5; ++k) P.lvd[k] = (double)expl(-C * (long double)(8 << k));
  for (int l = 0; l < 32; ++l) P.lanepow[l] = (double)expl(-C * (long double)(8 * l));
  for (int j = 0; j < 20; ++j) er_pow(C, (long double)TILE * (long double)(1LL << j), &P.t2m[j], &P.t2e[j]);
}

// Plan the K2 streaming kernel: G = SMs (one CTA per SM), the deepest TMA ring that
// fits next to the per-tile tables.
fs1_status plan_stream(fs1_plan_s* p, int device, int variant) {
  const fs1_desc& d = p->d;
  if (d.ndim != 1 || d.dtype != FS1_F64) return FS1_ERR_UNSUPPORTED;
  int sms = 0, optin = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return FS1_ERR_CUDA;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess)
    return FS1_ERR_CUDA;
  const long long ntiles = (d.n + TILE - 1) / TILE;
  if (ntiles > (1LL << 30)) return FS1_ERR_UNSUPPORTED;

  const int G = (int)std::min<long long>(std::min(sms, 256), ntiles);  // one range per thread in the folds
  const int ntmax = (int)((ntiles + G - 1) / G);
  int cnt = 0;
  const StreamEntry* tab = stream_table(&cnt);
  const StreamEntry* best = nullptr;
  size_t smem = 0;
  for (int i = 0; i < cnt; ++i) {
    if (variant >= 0 && i != variant) continue;
    if (32 * tab[i].NW < G) continue;  // ext_carries_cta: one range per thread
    const size_t need = stream_smem(tab[i].NW, tab[i].S, ntmax, G);
    if (need <= (size_t)optin) { best = &tab[i]; smem = need; break; }
  }
  if (!best) return FS1_ERR_UNSUPPORTED;
  if (cudaFuncSetAttribute(best->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return FS1_ERR_CUDA;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, best->fn, 32 * best->NW, smem) != cudaSuccess)
    return FS1_ERR_CUDA;
  if (occ < 1) return FS1_ERR_UNSUPPORTED;
  p->kind = KIND_STREAM;
  p->se = best;
  p->grid = G;
  p->smem = smem;
  StreamParams& P = p->sbase;
  memset(&P, 0, sizeof(P));
  P.n = d.n;
  P.npad = ntiles * TILE;
  P.ntiles = (int)ntiles;
  P.G = G;
  P.ntmax = ntmax;
  P.lam = exp(-d.h1 / d.eps);
  P.h = d.h1;
  P.tol = d.tol;
  P.itr_max = d.itr_max;
  P.check_interval = d.check_interval;
  P.warm = d.warm_start;
  P.input_is_log = d.domain == FS1_LOG ? d.input_is_log : 0;
  P.logd = d.domain == FS1_LOG;
  fill_stream_tables(P, d.h1 / d.eps);
  p->ws = stream_ws(P.npad, G).total;
  snprintf(p->info.kernel, sizeof(p->info.kernel), "stream_f64_%s_NW%d_S%d", P.logd ? "log" : "scaling",
           best->NW, best->S);
  p->info.chunk = 8;
  p->info.threads = 32 * best->NW;
  p->info.ctas_per_problem = G;
  p->info.grid = G;
  p->info.smem_bytes = smem;
  p->info.workspace_bytes = p->ws;
  return FS1_OK;
}

StreamParams stream_params(const fs1_plan_s* p, void* ws) {
  StreamParams P = p->sbase;
  const StreamWs w = stream_ws(P.npad, P.G);
  char* b = (char*)ws;
  P.Am = (double*)(b + w.Am);
  P.Bm = (double*)(b + w.Bm);
  P.Pm = (double*)(b + w.Pm);
  P.Qm0 = (double*)(b + w.Qm0);
  P.Qm1 = (double*)(b + w.Qm1);
  P.gtot = (double*)(b + w.gtot);
  P.gtote = (int*)(b + w.gtote);
  P.gtot2 = (double*)(b + w.gtot2);
  P.gtot2e = (int*)(b + w.gtot2e);
  P.bar = (unsigned*)(b + w.bar);
  return P;
}

// K3 / K3w workspace: log a, (log b)^T, G ping-pong, two pass scratches, F (K3w), fp32
// arrays of max(n m, lines x LP) floats each, + per-CTA partials and the barrier
struct SepWs {
  size_t LA, LBt, Gt0, Gt1, Z, Z2, Fp, AM, BM, AX, BX, part, flagp, bar, total;
};
SepWs sep_ws(size_t nm, size_t nperm, int G) {
  SepWs w;
  size_t o = 0;
  const size_t v = al256(std::max(nm, nperm) * 4);
  w.LA = o; o += v;
  w.LBt = o; o += v;
  w.Gt0 = o; o += v;
  w.Gt1 = o; o += v;
  w.Z = o; o += v;
  w.Z2 = o; o += nperm ? v : 0;
  w.Fp = o; o += nperm ? v : 0;
  w.AM = o; o += nperm ? v : 0;
  w.BM = o; o += nperm ? v : 0;
  const size_t vx = nperm ? al256(nperm / 2) : 0;  // >= [lines][32] ints (nperm = lines x 32 E, E >= 8)
  w.AX = o; o += vx;
  w.BX = o; o += vx;
  w.part = o; o += al256((size_t)3 * G * 8);
  w.flagp = o; o += al256((size_t)3 * G * 4);
  w.bar = o; o += 256;
  w.total = o;
  return w;
}
size_t sep_nperm(const Sep2dParams& P) {
  return P.wE ? (size_t)std::max(P.n, P.m) * 32 * P.wE : 0;
}

fs1_status plan_sep2d(fs1_plan_s* p, int device, int force) {
  const fs1_desc& d = p->d;
  if (d.dtype != FS1_F32 || d.domain != FS1_LOG) return FS1_ERR_UNSUPPORTED;
  if (d.n > sep2d_lmax() || d.m > sep2d_lmax() || d.n * d.m > (1LL << 31)) return FS1_ERR_UNSUPPORTED;
  const double c1 = d.h1 / d.eps, c2 = d.h2 / d.eps;
  if (c1 * 8 > 40.0 || c2 * 8 > 40.0) return FS1_ERR_UNSUPPORTED;  // chunk span
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return FS1_ERR_CUDA;
  if (cudaFuncSetAttribute(sep2d_fn(), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sep2d_smem()) !=
      cudaSuccess)
    return FS1_ERR_CUDA;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sep2d_fn(), 256, sep2d_smem()) != cudaSuccess)
    return FS1_ERR_CUDA;
  if (occ < 1) return FS1_ERR_UNSUPPORTED;
  const long long lines = std::max(d.n, d.m);
  const int G = (int)std::min<long long>((long long)sms * occ, std::max<long long>(1, lines));
  p->kind = KIND_SEP2D;
  p->grid = G;
  p->smem = sep2d_smem();
  Sep2dParams& P = p->tbase;
  memset(&P, 0, sizeof(P));
  fill_persist_tables(P.ax1, c1, 8);
  fill_persist_tables(P.ax2, c2, 8);
  P.ax1.lam = exp(-c1); P.ax1.h = d.h1;
  P.ax2.lam = exp(-c2); P.ax2.h = d.h2;
  P.n = (int)d.n;
  P.m = (int)d.m;
  P.G = G;
  P.tol = d.tol;
  P.itr_max = d.itr_max;
  P.check_interval = d.check_interval;
  P.warm = d.warm_start;
  P.input_is_log = d.input_is_log;
  snprintf(p->info.kernel, sizeof(p->info.kernel), "sep2d_f32_log_E8_W8");
  p->info.chunk = 8;
  p->info.threads = 256;
  p->info.ctas_per_problem = G;
  p->info.grid = G;
  // K3w (warp-per-line solve): the smallest chunk E whose 32 E covers both axes and
  // whose span c E stays within the fp32 chunk range
  P.wE = 0;
  p->sw = nullptr;
  if (force != 3) {
    int cnt = 0;
    const Sep2dwEntry* tab = sep2dw_table(&cnt);
    for (int i = 0; i < cnt; ++i) {
      const int E = tab[i].E;
      if (force >= 20 && i != force - 20) continue;
      if (32LL * E < std::max(d.n, d.m) || c1 * E > 40.0 || c2 * E > 40.0) continue;
      if (p->sw) continue;
      if (cudaFuncSetAttribute(tab[i].fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tab[i].smem) !=
          cudaSuccess)
        return FS1_ERR_CUDA;
      int o2 = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, tab[i].fn, 256, tab[i].smem) != cudaSuccess)
        return FS1_ERR_CUDA;
      if (o2 < 1) continue;
      p->sw = &tab[i];
      const long long groups = (std::max(d.n, d.m) + 7) / 8;
      p->gridw = (int)std::min<long long>((long long)sms * o2, groups);
    }
    if (p->sw) {
      const int E = p->sw->E;
      P.wE = E;
      const double cs[2] = {c1, c2};
      for (int ax = 0; ax < 2; ++ax) {
        const long double C = (long double)cs[ax];
        P.wax[ax].lam = (float)expl(-C);
        P.wax[ax].lamH = (float)expl(-C * (long double)(E / 2));
        for (int k = 0; k < 5; ++k) {
          double m;
          er_pow(C, (long double)E * (1 << k), &m, &P.wax[ax].Le[k]);
          P.wax[ax].Lm[k] = (float)m;
          if (P.wax[ax].Lm[k] >= 2.0f) { P.wax[ax].Lm[k] *= 0.5f; P.wax[ax].Le[k] += 1; }
        }
      }
      snprintf(p->info.kernel, sizeof(p->info.kernel), "sep2dw_f32_log_E%d_W8_B%d", E, p->sw->minb);
      p->info.chunk = E;
      p->info.ctas_per_problem = p->gridw;
      p->info.grid = p->gridw;
      p->info.smem_bytes = p->sw->smem;
    }
  }
  p->ws = sep_ws((size_t)d.n * d.m, sep_nperm(P), std::max(G, p->gridw)).total;
  if (!p->sw) p->info.smem_bytes = p->smem;
  p->info.workspace_bytes = p->ws;
  return FS1_OK;
}

Sep2dParams sep_params(const fs1_plan_s* p, void* ws) {
  Sep2dParams P = p->tbase;
  const SepWs w = sep_ws((size_t)P.n * P.m, sep_nperm(P), std::max(P.G, p->gridw));
  char* b = (char*)ws;
  P.LA = (float*)(b + w.LA);
  P.LBt = (float*)(b + w.LBt);
  P.Gt0 = (float*)(b + w.Gt0);
  P.Gt1 = (float*)(b + w.Gt1);
  P.Z = (float*)(b + w.Z);
  P.Z2 = P.wE ? (float*)(b + w.Z2) : nullptr;
  P.Fp = P.wE ? (float*)(b + w.Fp) : nullptr;
  P.AMp = P.wE ? (float*)(b + w.AM) : nullptr;
  P.BMp = P.wE ? (float*)(b + w.BM) : nullptr;
  P.AXe = P.wE ? (int*)(b + w.AX) : nullptr;
  P.BXe = P.wE ? (int*)(b + w.BX) : nullptr;
  P.part = (double*)(b + w.part);
  P.flagp = (int*)(b + w.flagp);
  P.bar = (unsigned*)(b + w.bar);
  return P;
}

fs1_status launch_sep(const fs1_plan_s* p, Sep2dParams& P, cudaStream_t st) {
  if (cudaMemsetAsync(P.bar, 0, 2 * sizeof(unsigned), st) != cudaSuccess) return FS1_ERR_CUDA;
  if (P.mode == 0 && p->sw) {  // solve: the warp-per-line kernel K3w
    P.G = p->gridw;
    return p->sw->launch(P, p->gridw, st) == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  return launch_sep2d(P, p->grid, st) == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status launch_stream(const fs1_plan_s* p, StreamParams& P, cudaStream_t st) {
  if (cudaMemsetAsync(P.bar, 0, 2 * sizeof(unsigned), st) != cudaSuccess) return FS1_ERR_CUDA;
  const cudaError_t e = p->se->launch(P, p->grid, p->smem, st);
  return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

// lambda^L as (mantissa in [1,2), exponent), from log2(lambda^L) = -L c / ln 2 in long double.
void er_pow(long double c, long double L, double* m, int* e) {
  if (L == 0) {
    *m = 1.0;
    *e = 0;
    return;
  }
  long double x = -L * c / logl(2.0L);
  long double f = floorl(x);
  *m = (double)exp2l(x - f);
  *e = (int)f;
  if (*m >= 2.0) { *m *= 0.5; *e += 1; }
}

double powl_d(long double c, long double L) { return (double)expl(-c * L); }

void fill_persist_tables(PersistParams& P, double c, int E) {
  const long double C = (long double)c;
  P.lamH = powl_d(C, (long double)(E / 2));
  for (int k = 0; k < 5; ++k) {
    const long double L = (long double)E * (1 << k);
    P.lvA[k] = powl_d(C, ceill(L / 2));
    P.lvB[k] = powl_d(C, floorl(L / 2));
    P.lvd[k] = powl_d(C, L);
    er_pow(C, L, &P.lvm[k], &P.lve[k]);
  }
  er_pow(C, 32.0L * E, &P.lvm[5], &P.lve[5]);
  P.wA = powl_d(C, 16.0L * E);
  P.wB = powl_d(C, 16.0L * E);
  for (int l = 0; l < 32; ++l) {
    const long double L = (long double)E * l;
    P.laneA[l] = powl_d(C, ceill(L / 2));
    P.laneB[l] = powl_d(C, floorl(L / 2));
    er_pow(C, L, &P.lanem[l], &P.lanee[l]);
  }
}

// Dynamic shared memory of a persistent-kernel plan: the instantiation's own need.
// (Padding it to trade resident CTAs for an even last wave was measured slower: the
// kernel is latency-bound, so the extra resident warps of a full first wave win —
// C2 2.86 -> 2.65 ms without the padding.)
cudaError_t size_persist_smem(const PersistEntry* pe, long long batch, int device, size_t* out) {
  (void)batch;
  (void)device;
  int occ = 0;
  cudaError_t e = cudaFuncSetAttribute(pe->solve_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pe->smem);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pe->solve_fn, 32 * pe->W, pe->smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  *out = pe->smem;
  return cudaSuccess;
}

}  // namespace

// serialises get/set-device around attribute and occupancy queries (also fs1_shard.cu)
std::mutex g_attr_mu;

extern "C" {

int fs1_abi_version(void) { return FS1_ABI_VERSION; }

const char* fs1_status_string(fs1_status s) {
  switch (s) {
    case FS1_OK: return "FS1_OK";
    case FS1_ERR_ARG: return "FS1_ERR_ARG: invalid argument";
    case FS1_ERR_EPS: return "FS1_ERR_EPS: eps and h must be finite and > 0";
    case FS1_ERR_UNSUPPORTED: return "FS1_ERR_UNSUPPORTED: no kernel for this dtype/domain/size";
    case FS1_ERR_CUDA: return "FS1_ERR_CUDA: CUDA runtime error";
    case FS1_ERR_WORKSPACE: return "FS1_ERR_WORKSPACE: workspace missing or misaligned";
  }
  return "FS1_?: unknown status";
}

static fs1_status plan_impl(const fs1_desc* desc, int device, int force, fs1_plan_t** out,
                            size_t* workspace_bytes) {
  if (!desc || !out) return FS1_ERR_ARG;
  *out = nullptr;
  const fs1_desc& d = *desc;
  if (d.ndim != 1 && d.ndim != 2 && d.ndim != 3) return FS1_ERR_ARG;
  if (d.ndim == 3 ? d.l < 1 : (d.l != 0 && d.l != 1)) return FS1_ERR_ARG;
  if (d.ndim == 3 && (!(d.h3 > 0.0) || !isfinite(d.h3))) return FS1_ERR_EPS;
  if (d.n < 1 || d.m < 1 || d.batch < 1 || d.itr_max < 0 || d.check_interval < 1) return FS1_ERR_ARG;
  if (!(d.tol >= 0.0) || !isfinite(d.tol)) return FS1_ERR_ARG;
  if (d.ndim == 1 && d.m != 1) return FS1_ERR_ARG;
  if (d.dtype != FS1_F32 && d.dtype != FS1_F64) return FS1_ERR_ARG;
  if (d.domain != FS1_SCALING && d.domain != FS1_LOG && d.domain != FS1_STABILIZED) return FS1_ERR_ARG;
  if (d.domain == FS1_STABILIZED && !(d.tau == 0.0 || (d.tau > 1.0 && isfinite(d.tau)))) return FS1_ERR_ARG;
  if (!(d.eps > 0.0) || !isfinite(d.eps) || !(d.h1 > 0.0) || !isfinite(d.h1)) return FS1_ERR_EPS;
  if (d.ndim >= 2 && (!(d.h2 > 0.0) || !isfinite(d.h2))) return FS1_ERR_EPS;
  if (d.batch > 0x7fffffffLL) return FS1_ERR_UNSUPPORTED;

  fs1_plan_s* p = new (std::nothrow) fs1_plan_s();
  if (!p) return FS1_ERR_ARG;
  p->d = d;
  p->device = device;
  const bool logd = d.domain == FS1_LOG;
  const double c = d.h1 / d.eps;

  if (d.domain == FS1_STABILIZED) {
    // K4: the paper's stabilised FS-1 (Remark 2.1 + 3.2), one CTA per problem
    if (d.ndim != 1 || d.dtype != FS1_F64 || d.warm_start || d.n > FS1_MAX_STAB) {
      delete p;
      return FS1_ERR_UNSUPPORTED;
    }
    int cnt = 0;
    const StabEntry* tab = stab_table(&cnt);
    const StabEntry* best = nullptr;
    for (int i = 0; i < cnt; ++i)
      if (32LL * tab[i].W * tab[i].E >= d.n && (!best || 32 * tab[i].W * tab[i].E < 32 * best->W * best->E))
        best = &tab[i];
    if (!best) { delete p; return FS1_ERR_UNSUPPORTED; }
    {
      std::lock_guard<std::mutex> lk(g_attr_mu);
      int cur = 0;
      if (cudaGetDevice(&cur) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      if (cur != device && cudaSetDevice(device) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      const cudaError_t e =
          cudaFuncSetAttribute(best->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best->smem());
      if (cur != device) cudaSetDevice(cur);
      if (e != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
    }
    p->kind = KIND_STAB;
    p->ke = best;
    StabParams& K = p->kbase;
    memset(&K, 0, sizeof(K));
    K.n = d.n;
    K.lam = exp(-c);
    K.h = d.h1;
    K.tol = d.tol;
    K.tau = d.tau == 0.0 ? 1e10 : d.tau;
    K.itr_max = d.itr_max;
    K.check_interval = d.check_interval;
    K.input_is_log = d.input_is_log;
    const long long P = 32LL * best->W * best->E;
    p->ws = al256((size_t)d.batch * 9 * P * 8);
    p->smem = best->smem();
    snprintf(p->info.kernel, sizeof(p->info.kernel), "stab_f64_E%d_W%d", best->E, best->W);
    p->info.chunk = best->E;
    p->info.threads = 32 * best->W;
    p->info.ctas_per_problem = 1;
    p->info.grid = d.batch;
    p->info.smem_bytes = p->smem;
    p->info.workspace_bytes = p->ws;
  } else if (d.ndim == 3 || (d.ndim == 2 && d.dtype == FS1_F64)) {
    // K5: Algorithm 2 (and its 3D extension) in fp64 (scaling domain), one CTA per
    // problem, a thread per line
    const long long L3 = d.ndim == 3 ? d.l : 1;
    if (d.dtype != FS1_F64 || d.domain != FS1_SCALING || d.n * d.m * L3 > (1LL << 28)) {
      delete p;
      return FS1_ERR_UNSUPPORTED;
    }
    p->kind = KIND_SEP64;
    Sep2d64Params& D = p->dbase;
    memset(&D, 0, sizeof(D));
    D.n = (int)d.n;
    D.m = (int)d.m;
    D.l = (int)L3;
    D.lam1 = exp(-d.h1 / d.eps);
    D.lam2 = exp(-d.h2 / d.eps);
    D.lam3 = d.ndim == 3 ? exp(-d.h3 / d.eps) : 0.0;
    D.h1 = d.h1;
    D.h2 = d.h2;
    D.h3 = d.ndim == 3 ? d.h3 : 0.0;
    D.tol = d.tol;
    D.itr_max = d.itr_max;
    D.check_interval = d.check_interval;
    D.warm = d.warm_start;
    // a thread per line of the busiest axis (2D: max(n, m); 3D: max(m l, n l, n m)), at most
    // 512 (the kernel's launch bound)
    const long long lines = d.ndim == 3 ? std::max<long long>(std::max<long long>(d.m * L3, d.n * L3), d.n * d.m)
                                        : std::max<long long>(d.n, d.m);
    p->threads = (int)std::min<long long>(512, ((lines + 31) / 32) * 32);
    // 2D problems whose lines fit a warp (G E <= 256 points): K5w, G lanes per line with
    // a chunked scan (test-only kind 5 keeps the thread-per-line kernel)
    const int wE = d.ndim == 2 && force != 5 ? sep2d64w_chunk(d.n, d.m) : 0;
    int wG = 0, wEp = 0;
    if (wE) {
      D.wE = wE;
      sep2d64w_geom(wE, &wG, &wEp);
      const long double cc[2] = {(long double)d.h1 / (long double)d.eps, (long double)d.h2 / (long double)d.eps};
      for (int k = 0; k < 5; ++k) {
        const long double L = (long double)wEp * (long double)(1 << k);
        const long double La = ceill(L / 2), Lb = floorl(L / 2);
        D.wA1[k] = (double)expl(-cc[0] * La);
        D.wB1[k] = (double)expl(-cc[0] * Lb);
        D.wA2[k] = (double)expl(-cc[1] * La);
        D.wB2[k] = (double)expl(-cc[1] * Lb);
      }
    }
    // K5w's transposition stage (fs1_sep2d64.cu); else small 2D problems: the
    // intermediate in shared memory
    if (wE) p->threads = sep2d64w_threads(d.n, d.m, wE);
    const size_t ssm = wE ? sep2d64w_smem(d.n, d.m, wE, p->threads) : sep2d64_smem(d.n, d.m, d.ndim);
    if (ssm > (wE ? 48 * 1024 : 0)) {
      std::lock_guard<std::mutex> lk(g_attr_mu);
      int cur = 0;
      if (cudaGetDevice(&cur) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      if (cur != device && cudaSetDevice(device) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      const cudaError_t e = cudaFuncSetAttribute(wE ? sep2d64w_fn(wE) : sep2d64_fn(),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm);
      if (cur != device) cudaSetDevice(cur);
      if (e != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      if (!wE) D.staged = 1;
    }
    p->ws = al256(wE ? (size_t)d.batch * sep2d64w_workspace(d.n, d.m, wE)
                     : (size_t)d.batch * 3 * (size_t)d.n * (size_t)d.m * (size_t)L3 * 8);
    p->smem = 0;
    if (wE) snprintf(p->info.kernel, sizeof(p->info.kernel), "sep2d64w_f64_scaling_G%dE%d", wG, wEp);
    else snprintf(p->info.kernel, sizeof(p->info.kernel), d.ndim == 3 ? "sep3d64_f64_scaling" : "sep2d64_f64_scaling");
    p->info.chunk = 1;
    p->info.threads = p->threads;
    p->info.ctas_per_problem = 1;
    p->info.grid = d.batch;
    p->info.smem_bytes = 0;
    p->info.workspace_bytes = p->ws;
  } else if (d.ndim == 1 && (force == 2 || (force >= 10 && force < 20))) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
    if (cur != device && cudaSetDevice(device) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
    const fs1_status st = plan_stream(p, device, (force >= 10 && force < 20) ? force - 10 : -1);
    if (cur != device) cudaSetDevice(cur);
    if (st != FS1_OK) { delete p; return st; }
  } else if (d.ndim == 1) {
    // persistent kernel: the smallest (E, W) instantiation whose 32 W E covers n
    const PersistEntry* (*tables[3])(int*) = {nullptr, nullptr, nullptr};
    if (d.dtype == FS1_F32) {
      if (logd) { tables[0] = persist_table_f32l; tables[1] = persist_table_f32l2; }
      else tables[0] = persist_table_f32s;
    } else {
      tables[0] = logd ? persist_table_f64l : persist_table_f64s;
    }
    const PersistEntry* best = nullptr;
    for (int ti = 0; ti < 3 && tables[ti]; ++ti) {
     int cnt = 0;
     const PersistEntry* tab = tables[ti](&cnt);
     for (int i = 0; i < cnt; ++i) {
      const PersistEntry& e = tab[i];
      if (e.logd != logd) continue;
      if (force >= 30 && force < 100 && e.W != force - 30) continue;  // test-only: warps per CTA
      if (force >= 100 && force < 200 && e.E != force - 100) continue;  // test-only: chunk E
      const long long cap = 32LL * e.W * e.E;
      if (cap < d.n) continue;
      if (logd) {
        // mantissa range per chunk and exactness of the fp64 warp scan
        const double lim_chunk = d.dtype == FS1_F32 ? 40.0 : 300.0;
        if (c * e.E > lim_chunk || c * e.E * 32.0 > 650.0) continue;
      }
      if (!best || cap < 32LL * best->W * best->E ||
          (cap == 32LL * best->W * best->E && e.W < best->W))
        best = &e;
     }
    }
    if (!best) {
      // too large for one CTA: the multi-CTA streaming kernel (fp64)
      if (force == 1) { delete p; return FS1_ERR_UNSUPPORTED; }
      std::lock_guard<std::mutex> lk(g_attr_mu);
      int cur = 0;
      if (cudaGetDevice(&cur) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      if (cur != device && cudaSetDevice(device) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      const fs1_status st = plan_stream(p, device, -1);
      if (cur != device) cudaSetDevice(cur);
      if (st != FS1_OK) { delete p; return st; }
      if (workspace_bytes) *workspace_bytes = p->ws;
      *out = p;
      return FS1_OK;
    }
    p->kind = KIND_PERSIST;
    p->pe = best;
    memset(&p->base, 0, sizeof(p->base));
    p->base.n = d.n;
    p->base.batch = d.batch;
    p->base.lam = exp(-c);
    p->base.h = d.h1;
    p->base.tol = d.tol;
    p->base.itr_max = d.itr_max;
    p->base.check_interval = d.check_interval;
    p->base.warm = d.warm_start;
    p->base.input_is_log = logd ? d.input_is_log : 0;
    p->base.write_uv = 1;
    fill_persist_tables(p->base, c, best->E);
    {
      std::lock_guard<std::mutex> lk(g_attr_mu);
      int cur = 0;
      if (cudaGetDevice(&cur) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      if (cur != device && cudaSetDevice(device) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
      cudaError_t e = size_persist_smem(best, d.batch, device, &p->smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(best->apply_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)best->smem);
      if (cur != device) cudaSetDevice(cur);
      if (e != cudaSuccess) {
        delete p;
        return FS1_ERR_CUDA;
      }
    }
    p->ws = 0;
    snprintf(p->info.kernel, sizeof(p->info.kernel), "persist_%s_%s_E%d_W%d",
             d.dtype == FS1_F32 ? "f32" : "f64", logd ? "log" : "scaling", best->E, best->W);
    p->info.chunk = best->E;
    p->info.threads = 32 * best->W;
    p->info.ctas_per_problem = 1;
    p->info.grid = d.batch;
    p->info.smem_bytes = p->smem;
    p->info.workspace_bytes = 0;
  } else {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
    if (cur != device && cudaSetDevice(device) != cudaSuccess) { delete p; return FS1_ERR_CUDA; }
    const fs1_status st = plan_sep2d(p, device, force);
    if (cur != device) cudaSetDevice(cur);
    if (st != FS1_OK) { delete p; return st; }
  }
  if (workspace_bytes) *workspace_bytes = p->ws;
  *out = p;
  return FS1_OK;
}

fs1_status fs1_plan(const fs1_desc* desc, int device, fs1_plan_t** out, size_t* workspace_bytes) {
  return plan_impl(desc, device, 0, out, workspace_bytes);
}

// test-only (not in include/fs1.h): plan with a forced kernel family so the parity
// tests reach every kernel at small sizes and the benchmarks can compare
// instantiations.  kind: 1 persistent (K1); 2 streaming (K2); 5 the 2D fp64 kernel K5
// with a thread per line (not its warp-per-line variant K5w); 10 + i streaming
// instantiation i; 3 2D CTA-line kernel (K3); 20 + i 2D warp-line instantiation i
// (K3w); 30 + W persistent with W warps per CTA; 100 + E persistent with chunk E.
fs1_status fs1__plan_kind(const fs1_desc* desc, int device, int kind, fs1_plan_t** out,
                          size_t* workspace_bytes) {
  return plan_impl(desc, device, kind, out, workspace_bytes);
}

// test-only (not in include/fs1.h): phase timestamps of the streaming kernel,
// buf = [grid][64][4] u64 (globaltimer ns at: barrier exit, carries ready, stream
// done, totals published) for the first 64 psi half-steps.
fs1_status fs1__set_stream_timers(fs1_plan_t* plan, unsigned long long* buf) {
  if (!plan) return FS1_ERR_ARG;
  plan->sbase.tdbg = buf;
  return FS1_OK;
}

// test-only: phase timestamps of the 2D warp-line kernel at iteration 5, pass R:
// buf = [grid][8 warps][2 groups][8] u64 + [grid] barrier exits.
fs1_status fs1__set_sep_timers(fs1_plan_t* plan, unsigned long long* buf) {
  if (!plan) return FS1_ERR_ARG;
  plan->tbase.tdbg = buf;
  return FS1_OK;
}

fs1_status fs1_plan_info(const fs1_plan_t* plan, fs1_plan_info_t* info) {
  if (!plan || !info) return FS1_ERR_ARG;
  *info = plan->info;
  return FS1_OK;
}

void fs1_plan_destroy(fs1_plan_t* plan) { delete plan; }

fs1_status fs1_solve(const fs1_plan_t* plan, const void* a, const void* b, void* u, void* v,
                     int32_t* iters, double* err, int32_t* flags, double* cost, void* workspace,
                     void* stream) {
  if (!plan || !a || !b || !u || !v) return FS1_ERR_ARG;
  if (plan->ws && (!workspace || ((uintptr_t)workspace & 255))) return FS1_ERR_WORKSPACE;
  if (plan->kind == KIND_PERSIST) {
    PersistParams P = plan->base;
    P.a = a; P.b = b; P.u = u; P.v = v;
    P.iters = iters; P.err = err; P.flags = flags; P.cost = cost;
    cudaError_t e = plan->pe->launch_solve(P, plan->d.batch, plan->smem, (cudaStream_t)stream);
    return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_SEP64) {
    Sep2d64Params P = plan->dbase;
    P.a = (const double*)a; P.b = (const double*)b; P.u = (double*)u; P.v = (double*)v;
    P.iters = iters; P.err = err; P.flags = flags; P.cost = cost;
    P.ws = (double*)workspace;
    P.mode = 0;
    const cudaError_t e = P.wE ? launch_sep2d64w(P, plan->d.batch, P.wE, plan->threads, (cudaStream_t)stream)
                               : launch_sep2d64(P, plan->d.batch, plan->threads, (cudaStream_t)stream);
    return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_STAB) {
    StabParams P = plan->kbase;
    P.a = a; P.b = b; P.u = u; P.v = v;
    P.iters = iters; P.err = err; P.flags = flags; P.cost = cost;
    P.ws = (double*)workspace;
    P.mode = 0;
    return plan->ke->launch(P, plan->d.batch, (cudaStream_t)stream) == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_SEP2D) {
    const long long nm = plan->d.n * plan->d.m;
    for (long long k = 0; k < plan->d.batch; ++k) {
      Sep2dParams P = sep_params(plan, workspace);
      P.a = (const float*)a + k * nm; P.b = (const float*)b + k * nm;
      P.u = (float*)u + k * nm; P.v = (float*)v + k * nm;
      P.iters = iters ? iters + k : nullptr; P.err = err ? err + k : nullptr;
      P.flags = flags ? flags + k : nullptr; P.cost = cost ? cost + k : nullptr;
      P.mode = 0;
      const fs1_status st = launch_sep(plan, P, (cudaStream_t)stream);
      if (st != FS1_OK) return st;
    }
    return FS1_OK;
  }
  if (plan->kind == KIND_STREAM) {
    if (plan->d.domain != FS1_LOG) return FS1_ERR_UNSUPPORTED;
    // one binary exponent per 256-point tile holds a tile of the potentials in fp64
    // only if they can vary by at most c x 256 <= 600 nats across it: Sinkhorn's
    // potentials are c-Lipschitz up to log a, log b (R25); a tile spans
    // min(n, 256) - 1 cells
    if (plan->d.h1 / plan->d.eps * (double)(std::min<long long>(plan->d.n, TILE) - 1) > 600.0)
      return FS1_ERR_UNSUPPORTED;
    // one cooperative launch per problem, in order on the stream (shared workspace)
    for (long long k = 0; k < plan->d.batch; ++k) {
      StreamParams P = stream_params(plan, workspace);
      const long long o = k * plan->d.n;
      P.a = (const double*)a + o; P.b = (const double*)b + o;
      P.u = (double*)u + o; P.v = (double*)v + o;
      P.iters = iters ? iters + k : nullptr; P.err = err ? err + k : nullptr;
      P.flags = flags ? flags + k : nullptr; P.cost = cost ? cost + k : nullptr;
      P.mode = 0;
      const fs1_status st = launch_stream(plan, P, (cudaStream_t)stream);
      if (st != FS1_OK) return st;
    }
    return FS1_OK;
  }
  return FS1_ERR_UNSUPPORTED;
}

fs1_status fs1_cost(const fs1_plan_t* plan, const void* u, const void* v, double* cost,
                    void* workspace, void* stream) {
  if (!plan || !u || !v || !cost) return FS1_ERR_ARG;
  if (plan->ws && (!workspace || ((uintptr_t)workspace & 255))) return FS1_ERR_WORKSPACE;
  if (plan->kind == KIND_PERSIST) {
    // The loop top with l = itr_max = 0 on the given state: evaluates err and the
    // return line, leaves u, v untouched.  a = b = u (never read for the cost).
    PersistParams P = plan->base;
    P.itr_max = 0;
    P.tol = 0.0;
    P.warm = 1;
    P.write_uv = 0;
    P.input_is_log = plan->d.domain == FS1_LOG;
    P.a = u; P.b = v; P.u = const_cast<void*>(u); P.v = const_cast<void*>(v);
    P.iters = nullptr; P.err = nullptr; P.flags = nullptr; P.cost = cost;
    cudaError_t e = plan->pe->launch_solve(P, plan->d.batch, plan->smem, (cudaStream_t)stream);
    return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_SEP2D) {
    const long long nm = plan->d.n * plan->d.m;
    for (long long k = 0; k < plan->d.batch; ++k) {
      Sep2dParams P = sep_params(plan, workspace);
      P.u = (float*)const_cast<void*>(u) + k * nm; P.v = (float*)const_cast<void*>(v) + k * nm;
      P.cost = cost + k;
      P.mode = 2;
      const fs1_status st = launch_sep(plan, P, (cudaStream_t)stream);
      if (st != FS1_OK) return st;
    }
    return FS1_OK;
  }
  if (plan->kind == KIND_STREAM) {
    for (long long k = 0; k < plan->d.batch; ++k) {
      StreamParams P = stream_params(plan, workspace);
      const long long o = k * plan->d.n;
      P.u = (double*)const_cast<void*>(u) + o; P.v = (double*)const_cast<void*>(v) + o;
      P.cost = cost + k;
      P.mode = 2;
      const fs1_status st = launch_stream(plan, P, (cudaStream_t)stream);
      if (st != FS1_OK) return st;
    }
    return FS1_OK;
  }
  if (plan->kind == KIND_SEP64) {
    Sep2d64Params P = plan->dbase;
    P.u = (double*)const_cast<void*>(u); P.v = (double*)const_cast<void*>(v);
    P.cost = cost;
    P.ws = (double*)workspace;
    P.mode = 1;
    return launch_sep2d64(P, plan->d.batch, plan->threads, (cudaStream_t)stream) == cudaSuccess ? FS1_OK
                                                                                            : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_STAB) {
    // the return line on (alpha/eps, beta/eps) = (F, G), phi = psi = 1 (an absorbed state)
    StabParams P = plan->kbase;
    P.u = const_cast<void*>(u); P.v = const_cast<void*>(v);
    P.cost = cost;
    P.ws = (double*)workspace;
    P.mode = 1;
    return plan->ke->launch(P, plan->d.batch, (cudaStream_t)stream) == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  return FS1_ERR_UNSUPPORTED;
}

fs1_status fs1_transport_plan(const fs1_plan_t* plan, const void* u, const void* v, void* gamma, void* stream) {
  if (!plan || !u || !v || !gamma) return FS1_ERR_ARG;
  const fs1_desc& d = plan->d;
  if (d.ndim == 3 || d.n * d.m > FS1_MAX_TPLAN) return FS1_ERR_UNSUPPORTED;
  const double c1 = d.h1 / d.eps, c2 = d.ndim == 2 ? d.h2 / d.eps : 0.0;
  const cudaError_t e = launch_tplan(d.dtype == FS1_F64 ? 1 : 0, u, v, gamma, d.batch, d.n, d.m, c1, c2,
                                     d.domain != FS1_SCALING ? 1 : 0, (cudaStream_t)stream);
  return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_plan_entries(const fs1_plan_t* plan, const void* u, const void* v, const int64_t* idx,
                            long long count, double* out, void* stream) {
  if (!plan || count < 0) return FS1_ERR_ARG;
  if (count == 0) return FS1_OK;
  if (!u || !v || !idx || !out) return FS1_ERR_ARG;
  const fs1_desc& d = plan->d;
  const double c1 = d.h1 / d.eps, c2 = d.ndim >= 2 ? d.h2 / d.eps : 0.0, c3 = d.ndim == 3 ? d.h3 / d.eps : 0.0;
  const long long l = d.ndim == 3 ? d.l : 1;
  const cudaError_t e = launch_entries(d.dtype == FS1_F64 ? 1 : 0, u, v, (const long long*)idx, count, out, d.batch,
                                       d.n, d.m, l, c1, c2, c3, d.domain != FS1_SCALING ? 1 : 0, (cudaStream_t)stream);
  return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_apply(const fs1_plan_t* plan, const void* x, void* y, void* workspace, void* stream) {
  if (!plan || !x || !y || x == y) return FS1_ERR_ARG;
  if (plan->ws && (!workspace || ((uintptr_t)workspace & 255))) return FS1_ERR_WORKSPACE;
  if (plan->kind == KIND_PERSIST) {
    cudaError_t e = plan->pe->launch_apply(plan->base, x, y, plan->d.batch, (cudaStream_t)stream);
    return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_SEP64) {
    Sep2d64Params P = plan->dbase;
    P.x = (const double*)x; P.y = (double*)y;
    P.ws = (double*)workspace;
    P.mode = 2;
    return launch_sep2d64(P, plan->d.batch, plan->threads, (cudaStream_t)stream) == cudaSuccess ? FS1_OK
                                                                                            : FS1_ERR_CUDA;
  }
  if (plan->kind == KIND_SEP2D) {
    const long long nm = plan->d.n * plan->d.m;
    for (long long k = 0; k < plan->d.batch; ++k) {
      Sep2dParams P = sep_params(plan, workspace);
      P.x = (const float*)x + k * nm; P.y = (float*)y + k * nm;
      P.mode = 1;
      const fs1_status st = launch_sep(plan, P, (cudaStream_t)stream);
      if (st != FS1_OK) return st;
    }
    return FS1_OK;
  }
  if (plan->kind == KIND_STREAM) {
    for (long long k = 0; k < plan->d.batch; ++k) {
      StreamParams P = stream_params(plan, workspace);
      const long long o = k * plan->d.n;
      P.x = (const double*)x + o; P.y = (double*)y + o;
      P.mode = 1;
      const fs1_status st = launch_stream(plan, P, (cudaStream_t)stream);
      if (st != FS1_OK) return st;
    }
    return FS1_OK;
  }
  return FS1_ERR_UNSUPPORTED;
}

fs1_status fs1_dual(const fs1_plan_t* plan, const void* a, const void* b, const void* u, const void* v,
                    void* scratch, double* dual, void* workspace, void* stream) {
  if (!plan || !a || !b || !u || !v || !scratch || !dual) return FS1_ERR_ARG;
  if (plan->d.domain == FS1_STABILIZED) return FS1_ERR_UNSUPPORTED;
  // S = K psi (scaling) / log K e^G (log): the kernel apply of the plan
  const fs1_status st = fs1_apply(plan, v, scratch, workspace, stream);
  if (st != FS1_OK) return st;
  const fs1_desc& d = plan->d;
  const long long size = d.n * d.m * (d.ndim == 3 ? d.l : 1);
  const cudaError_t e = launch_dual(d.dtype == FS1_F64 ? 1 : 0, a, b, u, v, scratch, d.batch, size, d.eps,
                                    d.domain == FS1_LOG ? 1 : 0, d.domain == FS1_LOG ? d.input_is_log : 0, dual,
                                    (cudaStream_t)stream);
  return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

// the eps-scaling schedule: eps_k = max(eps, eps0 factor^k) (oracle/sinkhorn.py eps_schedule)
static int eps_schedule(double eps, double eps0, double factor, double* out, int cap) {
  int k = 0;
  double e = eps0;
  while (e > eps * (1.0 + 1e-12) && k < cap - 1) {
    if (out) out[k] = e;
    ++k;
    e *= factor;
  }
  if (out) out[k] = eps;
  return k + 1;
}

static fs1_status eps_scaling_check(const fs1_desc* desc, double eps0, double factor) {
  if (!desc) return FS1_ERR_ARG;
  if (desc->domain != FS1_LOG) return FS1_ERR_UNSUPPORTED;
  if (!(factor > 0.0 && factor < 1.0) || !(eps0 >= desc->eps) || !isfinite(eps0)) return FS1_ERR_ARG;
  if (eps_schedule(desc->eps, eps0, factor, nullptr, 4096) >= 4096) return FS1_ERR_ARG;
  return FS1_OK;
}

fs1_status fs1_eps_scaling_plan(const fs1_desc* desc, int device, double eps0, double factor, int32_t* stages,
                                size_t* workspace_bytes) {
  fs1_status st = eps_scaling_check(desc, eps0, factor);
  if (st != FS1_OK) return st;
  static thread_local double sched[4096];
  const int ns = eps_schedule(desc->eps, eps0, factor, sched, 4096);
  size_t mx = 0;
  for (int k = 0; k < ns; ++k) {
    fs1_desc dk = *desc;
    dk.eps = sched[k];
    fs1_plan_t* p = nullptr;
    size_t ws = 0;
    st = fs1_plan(&dk, device, &p, &ws);
    if (st != FS1_OK) return st;
    fs1_plan_destroy(p);
    mx = std::max(mx, ws);
  }
  if (stages) *stages = ns;
  if (workspace_bytes) *workspace_bytes = mx;
  return FS1_OK;
}

fs1_status fs1_solve_eps_scaling(const fs1_desc* desc, int device, double eps0, double factor, int32_t stage_iters,
                                 const void* a, const void* b, void* u, void* v, int32_t* iters, double* err,
                                 int32_t* flags, double* cost, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  fs1_status st = eps_scaling_check(desc, eps0, factor);
  if (st != FS1_OK) return st;
  if (stage_iters < 0 || !a || !b || !u || !v) return FS1_ERR_ARG;
  static thread_local double sched[4096];
  const int ns = eps_schedule(desc->eps, eps0, factor, sched, 4096);
  for (int k = 0; k < ns; ++k) {
    const bool final = k == ns - 1;
    fs1_desc dk = *desc;
    dk.eps = sched[k];
    dk.itr_max = final ? desc->itr_max : stage_iters;
    dk.tol = final ? desc->tol : 0.0;
    dk.warm_start = (k > 0 || desc->warm_start) ? 1 : 0;
    fs1_plan_t* p = nullptr;
    size_t ws = 0;
    st = fs1_plan(&dk, device, &p, &ws);
    if (st != FS1_OK) return st;
    if (ws > workspace_bytes || (ws && !workspace)) {
      fs1_plan_destroy(p);
      return FS1_ERR_WORKSPACE;
    }
    if (k > 0) {
      // the previous stage's dual potentials f = eps F, g = eps G carried to this eps
      const cudaError_t e = launch_rescale(desc->dtype == FS1_F64 ? 1 : 0, u, v, desc->batch * desc->n * desc->m,
                                           sched[k - 1] / sched[k], (cudaStream_t)stream);
      if (e != cudaSuccess) {
        fs1_plan_destroy(p);
        return FS1_ERR_CUDA;
      }
    }
    st = fs1_solve(p, a, b, u, v, iters, err, flags, final ? cost : nullptr, workspace, stream);
    fs1_plan_destroy(p);  // launches captured their parameters by value
    if (st != FS1_OK) return st;
  }
  return FS1_OK;
}

}  // extern "C"
