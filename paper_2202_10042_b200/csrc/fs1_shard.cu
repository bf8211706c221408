// fs1_shard.cu — C ABI of include/fs1_shard.h: plans, workspace layout and launches
// of the sharded single-problem kernels (fs1_shard.cuh).
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>

#include "../../include/fs1_shard.h"
#include "fs1_shard.cuh"

extern std::mutex g_attr_mu;  // fs1_api.cu: serialises get/set-device around attribute queries

using namespace fs1;

namespace {

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

void er_pow_l(long double c, long double L, double* m, int* e) {
  if (L == 0) {
    *m = 1.0;
    *e = 0;
    return;
  }
  const long double x = -L * c / logl(2.0L);
  const long double f = floorl(x);
  *m = (double)exp2l(x - f);
  *e = (int)f;
  if (*m >= 2.0) { *m *= 0.5; *e += 1; }
}

// workspace layout of one rank
struct Ws {
  size_t Am, Bm, Pm, Q0, Q1, AX, BX, PX, QX0, QX1, tzA, tzB;
  size_t Fm[2], Bmt[2], Fe[2], Be[2];     // tile totals / in-block carries, two sets
  size_t BFm[2], BBm[2], BFe[2], BBe[2];  // block totals / block carries, two sets
  size_t Jm, Je, part, parte, flag, total;
};
Ws ws_layout(long long T, int grid) {
  Ws w;
  size_t o = 0;
  const size_t vd = al256((size_t)T * shd::TILE * 8), ti = al256((size_t)T * 4), td = al256((size_t)T * 8);
  w.Am = o; o += vd; w.Bm = o; o += vd; w.Pm = o; o += vd; w.Q0 = o; o += vd; w.Q1 = o; o += vd;
  w.AX = o; o += ti; w.BX = o; o += ti; w.PX = o; o += ti; w.QX0 = o; o += ti; w.QX1 = o; o += ti;
  w.tzA = o; o += al256((size_t)T); w.tzB = o; o += al256((size_t)T);
  for (int k = 0; k < 2; ++k) {
    w.Fm[k] = o; o += td; w.Bmt[k] = o; o += td; w.Fe[k] = o; o += ti; w.Be[k] = o; o += ti;
  }
  const size_t bd = al256((size_t)grid * 8), bi = al256((size_t)grid * 4);
  for (int k = 0; k < 2; ++k) {
    w.BFm[k] = o; o += bd; w.BBm[k] = o; o += bd; w.BFe[k] = o; o += bi; w.BBe[k] = o; o += bi;
  }
  w.Jm = o; o += 4 * td; w.Je = o; o += 4 * ti;
  w.part = o; o += al256((size_t)grid * 8);
  w.parte = o; o += al256((size_t)grid * 4);
  w.flag = o; o += 256;
  w.total = o;
  return w;
}

}  // namespace

struct fs1_shard_s {
  fs1_desc d;
  int device;
  int grid;  // CTAs of the tile kernels
  ShardParams P;
  Ws w;
};

template <class T> static T* at(void* ws, size_t off) { return reinterpret_cast<T*>((char*)ws + off); }

static shd::BlockIO block_io(const Ws& w, void* ws, int set) {
  shd::BlockIO b;
  b.Fm = at<double>(ws, w.Fm[set]); b.Fe = at<int>(ws, w.Fe[set]);
  b.Bm = at<double>(ws, w.Bmt[set]); b.Be = at<int>(ws, w.Be[set]);
  b.BFm = at<double>(ws, w.BFm[set]); b.BFe = at<int>(ws, w.BFe[set]);
  b.BBm = at<double>(ws, w.BBm[set]); b.BBe = at<int>(ws, w.BBe[set]);
  return b;
}

extern "C" {

fs1_status fs1_shard_plan(const fs1_desc* desc, int world, int rank, int device, fs1_shard_t** out,
                          size_t* workspace_bytes, int64_t* seg_lo, int64_t* seg_len) {
  if (!desc || !out) return FS1_ERR_ARG;
  const fs1_desc& d = *desc;
  if (world < 1 || rank < 0 || rank >= world || d.batch != 1 || d.warm_start || d.n < 1 || d.itr_max < 0 ||
      d.tol < 0 || d.check_interval < 1)
    return FS1_ERR_ARG;
  if (!(d.eps > 0) || !(d.h1 > 0) || !isfinite(d.eps) || !isfinite(d.h1)) return FS1_ERR_EPS;
  if (d.ndim != 1 || d.m != 1 || d.dtype != FS1_F64 || d.domain != FS1_LOG) return FS1_ERR_UNSUPPORTED;
  const double c = d.h1 / d.eps;
  if (c * (double)(std::min<long long>(d.n, shd::TILE) - 1) > 600.0) return FS1_ERR_UNSUPPORTED;
  const long long Ttot = (d.n + shd::TILE - 1) / shd::TILE;
  const long long T0 = (long long)rank * Ttot / world, T1 = (long long)(rank + 1) * Ttot / world;
  if (T1 <= T0 || T1 - T0 > INT_MAX / shd::TILE) return FS1_ERR_ARG;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return FS1_ERR_CUDA;
  fs1_shard_s* s = new (std::nothrow) fs1_shard_s();
  if (!s) return FS1_ERR_CUDA;
  s->d = d;
  s->device = device;
  ShardParams& P = s->P;
  memset(&P, 0, sizeof(P));
  P.n = d.n;
  P.T0 = T0;
  P.T = (int)(T1 - T0);
  P.Ttot = Ttot;
  P.lo = T0 * shd::TILE;
  P.len = (long long)P.T * shd::TILE;
  P.world = world;
  P.rank = rank;
  P.lam = exp(-c);
  P.h = d.h1;
  const long double C = (long double)c;
  for (int k = 0; k < 5; ++k) {
    P.lvd[k] = (double)expl(-C * (long double)(8 << k));
    er_pow_l(C, (long double)(8 << k), &P.lvm8[k], &P.lve8[k]);
  }
  for (int l = 0; l < 32; ++l) P.lanepow[l] = (double)expl(-C * (long double)(8 * l));
  for (int j = 0; j < 40; ++j) er_pow_l(C, (long double)shd::TILE * ldexpl(1.0L, j), &P.t2m[j], &P.t2e[j]);
  // blocks of TB tiles, one CTA each (about 4 per SM): the tile kernels' work units and
  // the first level of the two-level tile scan
  // resident CTAs of the half-step kernel per SM (registers), one block each: a single
  // balanced wave over the SMs
  int occ = 0;
  {
    // the occupancy query runs on the current device: make it `device` for the query
    // (the same guard fs1_plan uses, fs1_api.cu)
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e == cudaSuccess && cur != device) e = cudaSetDevice(device);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)&shd::k_half<false, true>, 32 * shd::NW, 0);
    if (cur >= 0 && cur != device) cudaSetDevice(cur);
    if (e != cudaSuccess) {
      delete s;
      return FS1_ERR_CUDA;
    }
  }
  occ = std::max(1, occ);
  P.TB = std::max(shd::NW, (int)((P.T + (long long)occ * sms - 1) / ((long long)occ * sms)));
  if (P.TB > shd::TBMAX) P.TB = shd::TBMAX;
  P.nblk = (P.T + P.TB - 1) / P.TB;
  s->grid = P.nblk;
  s->w = ws_layout(P.T, s->grid);
  if (workspace_bytes) *workspace_bytes = s->w.total;
  if (seg_lo) *seg_lo = P.lo;
  if (seg_len) *seg_len = std::min<long long>(P.len, d.n - P.lo);
  *out = s;
  return FS1_OK;
}

fs1_status fs1_shard_init(const fs1_shard_t* s, const void* a_seg, const void* b_seg, double* tot4, void* ws,
                          void* stream) {
  if (!s || !a_seg || !b_seg || !tot4 || !ws || ((uintptr_t)ws & 255)) return FS1_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const ShardParams& P = s->P;
  const Ws& w = s->w;
  const int kin = s->d.input_is_log ? 1 : 0;
  shd::k_init_flag<<<1, 1, 0, st>>>(at<int>(ws, w.flag));
  const dim3 g(s->grid), b(32 * shd::NW);
  shd::k_load<<<g, b, 0, st>>>(P, (const double*)a_seg, kin, 0.0, at<double>(ws, w.Am), at<int>(ws, w.AX),
                               at<unsigned char>(ws, w.tzA), nullptr, nullptr, nullptr, nullptr);
  shd::k_load<<<g, b, 0, st>>>(P, (const double*)b_seg, kin, 0.0, at<double>(ws, w.Bm), at<int>(ws, w.BX),
                               at<unsigned char>(ws, w.tzB), nullptr, nullptr, nullptr, nullptr);
  const double init = 1.0 / (double)P.n;  // phi0 = psi0 = 1/N
  shd::k_load<<<g, b, 0, st>>>(P, nullptr, 2, init, at<double>(ws, w.Pm), at<int>(ws, w.PX), nullptr,
                               at<double>(ws, w.Fm[0]), at<int>(ws, w.Fe[0]), at<double>(ws, w.Bmt[0]),
                               at<int>(ws, w.Be[0]));
  shd::k_load<<<g, b, 0, st>>>(P, nullptr, 2, init, at<double>(ws, w.Q0), at<int>(ws, w.QX0), nullptr, nullptr,
                               nullptr, nullptr, nullptr);
  const shd::BlockIO b0 = block_io(w, ws, 0);
  shd::k_block_scan<<<s->grid, 32 * shd::NW, 0, st>>>(P, b0);
  shd::k_scan_blocks<<<1, shd::SCAN_NT, 0, st>>>(P, b0, tot4);
  return cudaGetLastError() == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_half(const fs1_shard_t* s, int which, int hs, int check, int write, int l1, int psi_in,
                          int psi_out, const double* all_tot, double* tot4, double* errflag, void* ws,
                          void* stream) {
  if (!s || (!all_tot && !s->P.fused) || !ws || ((uintptr_t)ws & 255) || (which != 0 && which != 1) || hs < 0 ||
      (psi_in & ~1) || (psi_out & ~1) || (write && !tot4) || (check && !errflag))
    return FS1_ERR_ARG;
  if (which == 1 && check) return FS1_ERR_ARG;  // the check rides on the psi half-step (R3)
  cudaStream_t st = (cudaStream_t)stream;
  const ShardParams& P = s->P;
  const Ws& w = s->w;
  const int si = hs & 1, so = si ^ 1;
  const size_t Qoff[2] = {w.Q0, w.Q1}, QXoff[2] = {w.QX0, w.QX1};
  shd::HalfIO io;
  memset(&io, 0, sizeof(io));
  const shd::BlockIO bx = block_io(w, ws, si);
  io.CFm = bx.Fm; io.CFe = bx.Fe; io.CBm = bx.Bm; io.CBe = bx.Be;
  io.BCFm = bx.BFm; io.BCFe = bx.BFe; io.BCBm = bx.BBm; io.BCBe = bx.BBe;
  io.yb = block_io(w, ws, so);
  io.allT = all_tot;
  io.part = at<double>(ws, w.part);
  io.flag = at<int>(ws, w.flag);
  io.l = l1;
  if (which == 0) {  // psi = b ./ (K^T phi)
    io.xm = at<double>(ws, w.Pm); io.xX = at<int>(ws, w.PX);
    io.tm = at<double>(ws, w.Bm); io.tX = at<int>(ws, w.BX); io.tz = at<unsigned char>(ws, w.tzB);
    io.om = at<double>(ws, Qoff[psi_in]); io.oX = at<int>(ws, QXoff[psi_in]);
    io.ym = at<double>(ws, Qoff[psi_out]); io.yX = at<int>(ws, QXoff[psi_out]);
  } else {           // phi = a ./ (K psi)
    io.xm = at<double>(ws, Qoff[psi_in]); io.xX = at<int>(ws, QXoff[psi_in]);
    io.tm = at<double>(ws, w.Am); io.tX = at<int>(ws, w.AX); io.tz = at<unsigned char>(ws, w.tzA);
    io.ym = at<double>(ws, w.Pm); io.yX = at<int>(ws, w.PX);
  }
  if (check && write && which == 0 && psi_in == psi_out) return FS1_ERR_ARG;  // psi^(l) must survive
  const dim3 g(s->grid), b(32 * shd::NW);
  if (P.fused) shd::k_box_wait<<<1, 32, 0, st>>>(P);
  if (check && write) shd::k_half<true, true><<<g, b, 0, st>>>(P, io);
  else if (check) shd::k_half<true, false><<<g, b, 0, st>>>(P, io);
  else if (write) shd::k_half<false, true><<<g, b, 0, st>>>(P, io);
  if (write) shd::k_scan_blocks<<<1, shd::SCAN_NT, 0, st>>>(P, io.yb, tot4);
  if (l1 < 0 && which == 1) shd::k_tick<<<1, 1, 0, st>>>(io.flag);  // device counter mode
  if (check) shd::k_reduce<<<1, 32, 0, st>>>(io.part, s->grid, io.flag, errflag);
  return cudaGetLastError() == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_cost_totals(const fs1_shard_t* s, int psi, double* tot8, void* ws, void* stream) {
  if (!s || !tot8 || !ws || ((uintptr_t)ws & 255) || (psi & ~1)) return FS1_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const Ws& w = s->w;
  const size_t Qoff[2] = {w.Q0, w.Q1}, QXoff[2] = {w.QX0, w.QX1};
  shd::k_cost_tiles<<<s->grid, 32 * shd::NW, 0, st>>>(s->P, at<double>(ws, Qoff[psi]), at<int>(ws, QXoff[psi]),
                                                      at<double>(ws, w.Jm), at<int>(ws, w.Je));
  shd::k_cost_scan<<<1, shd::SCAN_NT, 0, st>>>(s->P, at<double>(ws, w.Jm), at<int>(ws, w.Je), tot8);
  return cudaGetLastError() == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_finish(const fs1_shard_t* s, int psi, const double* all_tot8, void* u_seg, void* v_seg,
                            double* cost_partial, void* ws, void* stream) {
  if (!s || !ws || ((uintptr_t)ws & 255) || (psi & ~1) || !u_seg || !v_seg) return FS1_ERR_ARG;
  if (cost_partial && !all_tot8) return FS1_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const Ws& w = s->w;
  const size_t Qoff[2] = {w.Q0, w.Q1}, QXoff[2] = {w.QX0, w.QX1};
  if (cost_partial) {
    shd::k_cost_dot<<<s->grid, 32 * shd::NW, 0, st>>>(s->P, at<double>(ws, Qoff[psi]), at<int>(ws, QXoff[psi]),
                                                      at<double>(ws, w.Pm), at<int>(ws, w.PX), at<double>(ws, w.Jm),
                                                      at<int>(ws, w.Je), all_tot8, at<double>(ws, w.part),
                                                      at<int>(ws, w.parte));
    shd::k_cost_reduce<<<1, 32, 0, st>>>(s->P, at<double>(ws, w.part), at<int>(ws, w.parte), s->grid, cost_partial);
  }
  shd::k_store<<<s->grid, 32 * shd::NW, 0, st>>>(s->P, at<double>(ws, w.Pm), at<int>(ws, w.PX), (double*)u_seg);
  shd::k_store<<<s->grid, 32 * shd::NW, 0, st>>>(s->P, at<double>(ws, Qoff[psi]), at<int>(ws, QXoff[psi]),
                                                 (double*)v_seg);
  return cudaGetLastError() == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

size_t fs1_shard_mailbox_bytes(int world) {
  if (world < 1 || world > FS1_SHARD_MAXW) return 0;
  return al256((size_t)world * 8 * sizeof(double) + ((size_t)world + 1) * sizeof(unsigned));
}

fs1_status fs1_shard_mailbox_alloc(int world, int device, void** box, void* ipc_handle) {
  const size_t bytes = fs1_shard_mailbox_bytes(world);
  if (!bytes || !box) return FS1_ERR_ARG;
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) return FS1_ERR_CUDA;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && ipc_handle) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, p);
    if (e == cudaSuccess) memcpy(ipc_handle, &h, sizeof(h));
  }
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (p) cudaFree(p);
    return FS1_ERR_CUDA;
  }
  *box = p;
  return FS1_OK;
}

fs1_status fs1_shard_mailbox_open(const void* ipc_handle, int device, void** box) {
  if (!ipc_handle || !box) return FS1_ERR_ARG;
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess) return FS1_ERR_CUDA;
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(box, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(prev);
  return e == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_mailbox_close(void* box) {
  if (!box) return FS1_ERR_ARG;
  return cudaIpcCloseMemHandle(box) == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_mailbox_free(void* box) {
  if (!box) return FS1_ERR_ARG;
  return cudaFree(box) == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_set_mailboxes(fs1_shard_t* s, void* const* boxes) {
  if (!s) return FS1_ERR_ARG;
  ShardParams& P = s->P;
  if (!boxes) {
    P.fused = 0;
    memset(P.box, 0, sizeof(P.box));
    return FS1_OK;
  }
  if (P.world > FS1_SHARD_MAXW) return FS1_ERR_ARG;
  for (int k = 0; k < P.world; ++k)
    if (!boxes[k]) return FS1_ERR_ARG;
  for (int k = 0; k < P.world; ++k) P.box[k] = static_cast<double*>(boxes[k]);
  P.fused = 1;
  return FS1_OK;
}

// Loop-top decision of Algorithm 1 line 2 over every rank's errflag row
// ([world][2] in rank order): err = the rank-ordered sum of the error partials (a fixed
// order, the same on every rank), the first non-finite iteration = the smallest positive
// record; out = {err, flag (0 continue, 1 CONVERGED, 2 NONFINITE, 4 ITR_MAX), l at stop}.
__global__ void k_shard_decide(const double* all, int world, int l, int itr_max, double tol, double* out) {
  double err = 0.0;
  double bad = 0.0;
  for (int k = 0; k < world; ++k) {
    err += all[2 * k];
    const double f = all[2 * k + 1];
    if (f > 0.0 && (bad == 0.0 || f < bad)) bad = f;
  }
  const bool use_tol = tol > 0.0;
  double flag = 0.0, lstop = (double)l;
  if (bad > 0.0) {
    flag = 2.0;  // "terminates abnormally"
    lstop = bad;
  } else if (l >= itr_max || err <= tol) {
    flag = (use_tol && err <= tol) ? 1.0 : 4.0;
  }
  out[0] = err;
  out[1] = flag;
  out[2] = lstop;
  out[3] = 0.0;
}

// rank-ordered sum of column `col` of a [world][stride] row set (the cost partials)
__global__ void k_shard_sum(const double* all, int world, int stride, int col, double* out) {
  double sacc = 0.0;
  for (int k = 0; k < world; ++k) sacc += all[(size_t)k * stride + col];
  out[0] = sacc;
}

fs1_status fs1_shard_decide(const fs1_shard_t* s, const double* all_errflag, int l, double* out4, void* stream) {
  if (!s || !all_errflag || !out4 || l < 0) return FS1_ERR_ARG;
  k_shard_decide<<<1, 1, 0, (cudaStream_t)stream>>>(all_errflag, s->P.world, l, s->d.itr_max, s->d.tol, out4);
  return cudaGetLastError() == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

fs1_status fs1_shard_sum(const fs1_shard_t* s, const double* rows, int stride, int col, double* out,
                         void* stream) {
  if (!s || !rows || !out || stride < 1 || col < 0 || col >= stride) return FS1_ERR_ARG;
  k_shard_sum<<<1, 1, 0, (cudaStream_t)stream>>>(rows, s->P.world, stride, col, out);
  return cudaGetLastError() == cudaSuccess ? FS1_OK : FS1_ERR_CUDA;
}

void fs1_shard_destroy(fs1_shard_t* s) { delete s; }

}  // extern "C"
