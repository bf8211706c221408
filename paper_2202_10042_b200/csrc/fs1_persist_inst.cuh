// fs1_persist_inst.cuh — explicit instantiation helpers for the persistent kernel.
#pragma once
#include "fs1_dispatch.h"
#include "fs1_persist.cuh"

namespace fs1 {

template <class T, int E, int W, bool L>
cudaError_t launch_solve_t(const PersistParams& P, long long grid, size_t smem, cudaStream_t st) {
  fs1_persist_solve<T, E, W, L><<<(unsigned)grid, 32 * W, smem, st>>>(P);
  return cudaGetLastError();
}
template <class T, int E, int W, bool L>
cudaError_t launch_apply_t(const PersistParams& P, const void* x, void* y, long long grid,
                           cudaStream_t st) {
  using PS = Persist<T, E, W, L>;
  fs1_persist_apply<T, E, W, L><<<(unsigned)grid, 32 * W, PS::SMEM, st>>>(
      P, reinterpret_cast<const T*>(x), reinterpret_cast<T*>(y));
  return cudaGetLastError();
}

#define FS1_PERSIST_ENTRY(T, DT, E, W, L)                                                  \
  PersistEntry {                                                                           \
    DT, L, E, W, Persist<T, E, W, L>::SMEM, (const void*)&fs1_persist_solve<T, E, W, L>,   \
        (const void*)&fs1_persist_apply<T, E, W, L>, &launch_solve_t<T, E, W, L>,           \
        &launch_apply_t<T, E, W, L>                                                        \
  }

}  // namespace fs1
