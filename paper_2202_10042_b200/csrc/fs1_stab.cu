// fs1_stab.cu — instantiations and launch of K4, the stabilised FS-1 kernel.
#include <cuda_runtime.h>

#include "fs1_dispatch.h"
#include "fs1_stab.cuh"

namespace fs1 {

template <int E, int W>
static size_t stab_smem_t() {
  // phi, psi, R (T E doubles each) + 32 reduction slots + W Jordan maps
  return (size_t)3 * 32 * W * E * 8 + 32 * 8 + (size_t)W * sizeof(stab::Jor);
}

template <int E, int W>
static cudaError_t launch_stab_t(const StabParams& P, long long batch, cudaStream_t st) {
  // (fs1_plan set the dynamic shared memory attribute on the plan's device)
  stab::fs1_stab_solve<E, W><<<(unsigned)batch, 32 * W, stab_smem_t<E, W>(), st>>>(P);
  return cudaGetLastError();
}

#define FS1_STAB_ENTRY(E, W) \
  StabEntry { E, W, (const void*)&stab::fs1_stab_solve<E, W>, &stab_smem_t<E, W>, &launch_stab_t<E, W> }

static const StabEntry kStab[] = {
    FS1_STAB_ENTRY(4, 4),   //   512 points
    FS1_STAB_ENTRY(8, 4),   //  1024
    FS1_STAB_ENTRY(8, 8),   //  2048
    FS1_STAB_ENTRY(8, 16),  //  4096
    FS1_STAB_ENTRY(16, 16), //  8192
};

const StabEntry* stab_table(int* count) {
  *count = (int)(sizeof(kStab) / sizeof(kStab[0]));
  return kStab;
}

}  // namespace fs1
