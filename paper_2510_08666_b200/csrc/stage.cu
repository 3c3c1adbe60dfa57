// Host-buffer staging for dinfer_step_host (the e2e path): zero-copy copies
// between pinned host memory (mapped into the device address space) and the
// step's device buffers, as kernels rather than copy-engine transfers, so they
// join the step's programmatic-dependent-launch chain:
//   stage-in  (host -> device: hidden block + packed small state) triggers its
//             dependents first, so K12 / K1 stream W while the PCIe reads land
//             (the W stream does not depend on the inputs);
//   stage-out (device -> host: packed small state) is launched behind K34 and
//             writes straight into the caller-visible pinned block.
// Pure data movement; no arithmetic of the method.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace dinfer {
namespace {

constexpr int kStageThreads = 256;

__global__ void __launch_bounds__(kStageThreads)
    stage_copy_kernel(const uint4* src0, uint4* dst0, long n0, const uint4* src1, uint4* dst1, long n1, int in) {
  if (in) grid_dep_launch_dependents();  // the next kernel may prefetch its weights under the copy
  grid_dep_wait();                       // the buffers are free (the previous kernel is complete)
  const long tid = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  const long nt = static_cast<long>(gridDim.x) * blockDim.x;
  // all of a thread's loads issued before its stores (PCIe round trips overlap)
  constexpr int kU = 4;
  for (long j0 = tid; j0 < n0 + n1; j0 += nt * kU) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long j = j0 + u * nt;
      if (j < n0) v[u] = __ldcv(src0 + j);
      else if (j < n0 + n1) v[u] = __ldcv(src1 + (j - n0));
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long j = j0 + u * nt;
      if (j < n0) dst0[j] = v[u];
      else if (j < n0 + n1) dst1[j - n0] = v[u];
    }
  }
  if (!in) {
    __threadfence_system();  // host-visible before the stream reports completion
    grid_dep_launch_dependents();
  }
}

}  // namespace

cudaError_t launch_stage_copy(const void* src0, void* dst0, size_t bytes0, const void* src1, void* dst1,
                              size_t bytes1, bool in, cudaStream_t st, bool pdl) {
  const long n0 = static_cast<long>(bytes0 / 16), n1 = static_cast<long>(bytes1 / 16);
  const long units = (n0 + n1 + 3) / 4;
  const int grid = static_cast<int>(std::min<long>(148, std::max<long>(1, (units + kStageThreads - 1) / kStageThreads)));
  return launch_ex(stage_copy_kernel, dim3(grid), dim3(kStageThreads), 0, st, pdl, static_cast<const uint4*>(src0),
                   static_cast<uint4*>(dst0), n0, static_cast<const uint4*>(src1), static_cast<uint4*>(dst1), n1,
                   in ? 1 : 0);
}

}  // namespace dinfer
