// Kernel dispatch: picks the interpreter instantiation for (datatype, reduction, protocol).
// The instantiations live in interp_k_*.cu (one translation unit per reduction, compiled in
// parallel); the kernel itself is in interp.cuh.
#include <cuda_runtime.h>

#include <mutex>
#include <set>

#include "devplan.hpp"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);
KernelFn interp_kernel_copy(int proto);
KernelFn interp_kernel_copy_wq();
KernelFn interp_kernel_sum(int dtype, int proto);
KernelFn interp_kernel_prod(int dtype, int proto);
KernelFn interp_kernel_max(int dtype, int proto);
KernelFn interp_kernel_min(int dtype, int proto);
KernelFn interp_kernel_copy_df();
KernelFn interp_kernel_sum_df(int dtype);
KernelFn interp_kernel_prod_df(int dtype);
KernelFn interp_kernel_max_df(int dtype);
KernelFn interp_kernel_min_df(int dtype);

constexpr int kMaxDynamicSmem = 220 << 10;  // TMA staging budget per block (runtime smem_kb <= 220)

KernelFn interp_kernel_wq(int redop) { return redop == -1 ? interp_kernel_copy_wq() : nullptr; }

// dataflow kernel (Simple protocol, every rank of the program in the launch)
KernelFn interp_kernel_df(int dtype, int redop) {
  switch (redop) {
    case -1: return interp_kernel_copy_df();
    case 0: return interp_kernel_sum_df(dtype);
    case 1: return interp_kernel_prod_df(dtype);
    case 2: return interp_kernel_max_df(dtype);
    case 3: return interp_kernel_min_df(dtype);
    default: return nullptr;
  }
}

// dtype: ncclDataType_t; redop: ncclRedOp_t or -1 for copy-only programs; ll: kProtoSimple / kProtoLL / kProtoLL128.
KernelFn interp_kernel(int dtype, int redop, int ll) {
  switch (redop) {
    case -1: return interp_kernel_copy(ll);
    case 0: return interp_kernel_sum(dtype, ll);
    case 1: return interp_kernel_prod(dtype, ll);
    case 2: return interp_kernel_max(dtype, ll);
    case 3: return interp_kernel_min(dtype, ll);
    default: return nullptr;
  }
}

static cudaError_t allow_smem(KernelFn fn) {
  static std::mutex mu;
  static std::set<std::pair<int, KernelFn>> done;  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, fn})) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynamicSmem);
  if (e == cudaSuccess) done.insert({dev, fn});
  return e;
}

cudaError_t interp_launch(KernelFn fn, const LaunchArgs& args, int grid, size_t smem, cudaStream_t stream) {
  const cudaError_t e = allow_smem(fn);
  if (e != cudaSuccess) return e;
  void* params[] = {const_cast<LaunchArgs*>(&args)};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(kThreads), params, smem, stream);
}

int interp_blocks_per_sm(KernelFn fn, size_t smem) {
  if (allow_smem(fn) != cudaSuccess) return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, reinterpret_cast<const void*>(fn), kThreads, smem) != cudaSuccess) return 0;
  return n;
}

}  // namespace gc3
