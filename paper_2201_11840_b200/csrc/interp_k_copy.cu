// Interpreter instantiation for copy-only programs (AllGather / AllToAll IRs; see interp.cuh).
#include "interp.cuh"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);

KernelFn interp_kernel_copy(int proto) {
  return proto == kProtoLL128 ? dev::interp<dev::RedNone, kProtoLL128>
         : proto == kProtoLL  ? dev::interp<dev::RedNone, kProtoLL>
                              : dev::interp<dev::RedNone, kProtoSimple>;
}
KernelFn interp_kernel_copy_wq() { return dev::interp_wq_kernel<dev::RedNone>; }
KernelFn interp_kernel_copy_df() { return dev::interp_df_kernel<dev::RedNone>; }

}  // namespace gc3
