// Dataflow-kernel instantiations for the prod reduction over every ncclDataType_t (see interp.cuh):
// the dataflow kernel (interp_df_kernel, Simple protocol).
#include "interp.cuh"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);

template <class R>
static KernelFn pick_df() {
  return dev::interp_df_kernel<R>;
}

#define GC3_BY_DTYPE(EXPR)                                   \
  switch (dtype) {                                           \
    case 0: { using R = dev::RedInt<int8_t, OP>; EXPR; }     \
    case 1: { using R = dev::RedInt<uint8_t, OP>; EXPR; }    \
    case 2: { using R = dev::RedInt<int32_t, OP>; EXPR; }    \
    case 3: { using R = dev::RedInt<uint32_t, OP>; EXPR; }   \
    case 4: { using R = dev::RedInt<int64_t, OP>; EXPR; }    \
    case 5: { using R = dev::RedInt<uint64_t, OP>; EXPR; }   \
    case 6: { using R = dev::RedHalf<false, OP>; EXPR; }     \
    case 7: { using R = dev::RedFloat<float, OP>; EXPR; }    \
    case 8: { using R = dev::RedFloat<double, OP>; EXPR; }   \
    case 9: { using R = dev::RedHalf<true, OP>; EXPR; }      \
    default: return nullptr;                                 \
  }

KernelFn interp_kernel_prod_df(int dtype) {
  constexpr int OP = dev::kProd;
  GC3_BY_DTYPE(return pick_df<R>())
}

}  // namespace gc3
