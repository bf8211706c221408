// fs1_sep2dw.cu — cooperative launches of the K3w warp-per-line separable 2D solve.
#include <cuda_runtime.h>

#include "fs1_dispatch.h"
#include "fs1_sep2dw.cuh"

namespace fs1 {

template <int E, int MINB>
cudaError_t launch_sep2dw_t(const Sep2dParams& P, int grid, cudaStream_t st) {
  void* args[] = {const_cast<Sep2dParams*>(&P)};
  return cudaLaunchCooperativeKernel((const void*)&sepw::fs1_sep2dw_kernel<E, MINB>, dim3(grid),
                                     dim3(sepw::NT), args, sepw::Cfg<E>::SMEM, st);
}
#define FS1_SEPW(E, MINB) \
  { E, MINB, (const void*)&sepw::fs1_sep2dw_kernel<E, MINB>, sepw::Cfg<E>::SMEM, &launch_sep2dw_t<E, MINB> }

// auto choice: the first entry (in order) whose 32 E covers both axes; a second
// E = 64 build with one CTA per SM (255 registers, no spills) is selectable by the
// test-only plan override 20 + index.
static const Sep2dwEntry kSepw[] = {
    FS1_SEPW(8, 2), FS1_SEPW(16, 2), FS1_SEPW(32, 2), FS1_SEPW(64, 2), FS1_SEPW(64, 1),
};
const Sep2dwEntry* sep2dw_table(int* count) {
  *count = (int)(sizeof(kSepw) / sizeof(kSepw[0]));
  return kSepw;
}

}  // namespace fs1
