// Interpreter instantiations for the min reduction over every ncclDataType_t (see interp.cuh):
// the static-lane interpreter per protocol (the dataflow kernel is in interp_k_min_df.cu).
#include "interp.cuh"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);

template <class R>
static KernelFn pick(int proto) {
  return proto == kProtoLL128 ? dev::interp<R, kProtoLL128> : proto == kProtoLL ? dev::interp<R, kProtoLL> : dev::interp<R, kProtoSimple>;
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

KernelFn interp_kernel_min(int dtype, int proto) {
  constexpr int OP = dev::kMin;
  GC3_BY_DTYPE(return pick<R>(proto))
}

}  // namespace gc3
