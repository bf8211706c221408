// fs1_sep2dw.cu — cooperative launches of the K3w warp-per-line separable 2D solve.
#include <cuda_runtime.h>

#include "fs1_dispatch.h"
#include "fs1_sep2dw.cuh"

namespace fs1 {

template <int E>
cudaError_t launch_sep2dw_t(const Sep2dParams& P, int grid, cudaStream_t st) {
  void* args[] = {const_cast<Sep2dParams*>(&P)};
  return cudaLaunchCooperativeKernel((const void*)&sepw::fs1_sep2dw_kernel<E>, dim3(grid), dim3(sepw::NT),
                                     args, sepw::Cfg<E>::SMEM, st);
}

static const Sep2dwEntry kSepw[] = {
    {8, (const void*)&sepw::fs1_sep2dw_kernel<8>, sepw::Cfg<8>::SMEM, &launch_sep2dw_t<8>},
    {16, (const void*)&sepw::fs1_sep2dw_kernel<16>, sepw::Cfg<16>::SMEM, &launch_sep2dw_t<16>},
    {32, (const void*)&sepw::fs1_sep2dw_kernel<32>, sepw::Cfg<32>::SMEM, &launch_sep2dw_t<32>},
    {64, (const void*)&sepw::fs1_sep2dw_kernel<64>, sepw::Cfg<64>::SMEM, &launch_sep2dw_t<64>},
};
const Sep2dwEntry* sep2dw_table(int* count) {
  *count = (int)(sizeof(kSepw) / sizeof(kSepw[0]));
  return kSepw;
}

}  // namespace fs1
