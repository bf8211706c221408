// fs1_sep2d.cu — cooperative launch of the K3 separable 2D kernel.
#include <cuda_runtime.h>

#include "fs1_dispatch.h"
#define FS1_SEP2D_KERNEL_TU
#include "fs1_sep2d.cuh"

namespace fs1 {

cudaError_t launch_sep2d(const Sep2dParams& P, int grid, cudaStream_t st) {
  void* args[] = {const_cast<Sep2dParams*>(&P)};
  return cudaLaunchCooperativeKernel((const void*)&sep::fs1_sep2d_kernel, dim3(grid), dim3(sep::NT), args,
                                     sep::SMEM, st);
}
const void* sep2d_fn() { return (const void*)&sep::fs1_sep2d_kernel; }
size_t sep2d_smem() { return sep::SMEM; }
int sep2d_lmax() { return sep::LMAX; }

}  // namespace fs1
