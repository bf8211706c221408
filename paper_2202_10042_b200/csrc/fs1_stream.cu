// fs1_stream.cu — instantiations and cooperative launch of the K2 streaming kernel.
#include <cuda_runtime.h>

#include "fs1_dispatch.h"
#include "fs1_stream.cuh"

namespace fs1 {

template <int NW, int S>
static cudaError_t launch_stream_t(const StreamParams& P, int grid, size_t smem, cudaStream_t st) {
  void* args[] = {const_cast<StreamParams*>(&P)};
  return cudaLaunchCooperativeKernel((const void*)&stm::fs1_stream_kernel<NW, S>, dim3(grid), dim3(32 * NW),
                                     args, smem, st);
}

#define FS1_STREAM_ENTRY(NW, S) \
  StreamEntry { NW, S, (const void*)&stm::fs1_stream_kernel<NW, S>, &launch_stream_t<NW, S> }

static const StreamEntry kStream[] = {
    FS1_STREAM_ENTRY(12, 3),   // measured fastest at C3 (88 us per half-step; 16x2: 95 us)
    FS1_STREAM_ENTRY(16, 2),
    FS1_STREAM_ENTRY(8, 4),
    FS1_STREAM_ENTRY(8, 2),
};

const StreamEntry* stream_table(int* count) {
  *count = (int)(sizeof(kStream) / sizeof(kStream[0]));
  return kStream;
}

size_t stream_smem(int NW, int S, int ntmax, int G) { return stm::layout(NW, S, ntmax, G).total; }

}  // namespace fs1
