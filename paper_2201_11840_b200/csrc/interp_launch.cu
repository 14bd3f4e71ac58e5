// Kernel dispatch: picks the interpreter instantiation for (datatype, reduction, protocol).
// The instantiations live in interp_k_*.cu (one translation unit per reduction, compiled in
// parallel); the kernel itself is in interp.cuh.
#include <cuda_runtime.h>

#include "devplan.hpp"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);
KernelFn interp_kernel_copy(bool ll);
KernelFn interp_kernel_sum(int dtype, bool ll);
KernelFn interp_kernel_prod(int dtype, bool ll);
KernelFn interp_kernel_max(int dtype, bool ll);
KernelFn interp_kernel_min(int dtype, bool ll);

// dtype: ncclDataType_t; redop: ncclRedOp_t or -1 for copy-only programs.
KernelFn interp_kernel(int dtype, int redop, bool ll) {
  switch (redop) {
    case -1: return interp_kernel_copy(ll);
    case 0: return interp_kernel_sum(dtype, ll);
    case 1: return interp_kernel_prod(dtype, ll);
    case 2: return interp_kernel_max(dtype, ll);
    case 3: return interp_kernel_min(dtype, ll);
    default: return nullptr;
  }
}

cudaError_t interp_launch(KernelFn fn, const LaunchArgs& args, int grid, cudaStream_t stream) {
  void* params[] = {const_cast<LaunchArgs*>(&args)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(kThreads), params, 0, stream);
}

int interp_blocks_per_sm(KernelFn fn) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reinterpret_cast<const void*>(fn), kThreads, 0) != cudaSuccess) return 0;
  return n;
}

}  // namespace gc3
