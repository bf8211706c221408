// fs1_dispatch.h — kernel registry (internal).
#pragma once
#include <cuda_runtime.h>

#include "fs1_params.h"

namespace fs1 {

struct PersistEntry {
  int dtype;  // 0 f32, 1 f64
  bool logd;
  int E, W;
  size_t smem;
  const void* solve_fn;
  const void* apply_fn;
  cudaError_t (*launch_solve)(const PersistParams&, long long grid, size_t smem, cudaStream_t);
  cudaError_t (*launch_apply)(const PersistParams&, const void* x, void* y, long long grid,
                              cudaStream_t);
};

// tables defined in fs1_persist_*.cu
const PersistEntry* persist_table_f32s(int* count);
const PersistEntry* persist_table_f32l(int* count);
const PersistEntry* persist_table_f32l2(int* count);
const PersistEntry* persist_table_f64s(int* count);
const PersistEntry* persist_table_f64l(int* count);

// K2 streaming kernel (fs1_stream.cu)
struct StreamEntry {
  int NW, S;
  const void* fn;
  cudaError_t (*launch)(const StreamParams&, int grid, size_t smem, cudaStream_t);
};
const StreamEntry* stream_table(int* count);
size_t stream_smem(int NW, int S, int ntmax, int G);

// K3 separable 2D kernel (fs1_sep2d.cu)
cudaError_t launch_sep2d(const Sep2dParams& P, int grid, cudaStream_t st);
const void* sep2d_fn();
size_t sep2d_smem();
int sep2d_lmax();

// K3w warp-per-line separable 2D solve (fs1_sep2dw.cu), E in {8, 16, 32, 64}
struct Sep2dwEntry {
  int E, minb;
  const void* fn;
  size_t smem;
  cudaError_t (*launch)(const Sep2dParams&, int grid, cudaStream_t);
};
const Sep2dwEntry* sep2dw_table(int* count);

// K4 stabilised FS-1 (fs1_stab.cu): one CTA of 32 W threads per problem, E points each
struct StabEntry {
  int E, W;
  const void* fn;
  size_t (*smem)();
  cudaError_t (*launch)(const StabParams&, long long batch, cudaStream_t);
};
const StabEntry* stab_table(int* count);

// K5 fp64 scaling-domain 2D solve, one CTA per problem (fs1_sep2d64.cu)
cudaError_t launch_sep2d64(const Sep2d64Params& P, long long batch, int threads, cudaStream_t st);
size_t sep2d64_smem(long long n, long long m, int ndim);  // dynamic shared memory of the staged 2D path (0: none)
int sep2d64w_chunk(long long n, long long m);             // K5w variant for a 2D problem (0: none)
void sep2d64w_geom(int var, int* G, int* E);               // lanes per line, points per lane
cudaError_t launch_sep2d64w(const Sep2d64Params& P, long long batch, int var, int threads, cudaStream_t st);
int sep2d64w_threads(long long n, long long m, int var);       // K5w block size
size_t sep2d64w_workspace(long long n, long long m, int var);  // K5w workspace bytes per problem
size_t sep2d64w_smem(long long n, long long m, int var, int threads);  // K5w dynamic shared memory
const void* sep2d64w_fn(int var);
const void* sep2d64_fn();

// dual objective and eps-scaling warm start (fs1_extra.cu)
cudaError_t launch_dual(int dtype, const void* a, const void* b, const void* u, const void* v, const void* s,
                        long long batch, long long size, double eps, int logd, int input_is_log, double* out,
                        cudaStream_t st);
cudaError_t launch_rescale(int dtype, void* u, void* v, long long count, double ratio, cudaStream_t st);

// transport-plan materialisation (fs1_tplan.cu)
cudaError_t launch_tplan(int dtype, const void* u, const void* v, void* g, long long batch, long long n, long long m,
                         double c1, double c2, int logd, cudaStream_t st);
cudaError_t launch_entries(int dtype, const void* u, const void* v, const long long* idx, long long count,
                           double* out, long long batch, long long n, long long m, long long l, double c1, double c2,
                           double c3, int logd, cudaStream_t st);

}  // namespace fs1
