// Interpreter instantiation for copy-only programs (AllGather / AllToAll IRs; see interp.cuh).
#include "interp.cuh"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);

KernelFn interp_kernel_copy(bool ll) { return ll ? dev::interp<dev::RedNone, true> : dev::interp<dev::RedNone, false>; }
KernelFn interp_kernel_copy_wq() { return dev::interp_wq_kernel<dev::RedNone>; }

}  // namespace gc3
