// Interpreter instantiations for the sum reduction over every ncclDataType_t (see interp.cuh).
#include "interp.cuh"

namespace gc3 {

using KernelFn = void (*)(LaunchArgs);

template <class R>
static KernelFn pick(int proto) {
  return proto == kProtoLL128 ? dev::interp<R, kProtoLL128> : proto == kProtoLL ? dev::interp<R, kProtoLL> : dev::interp<R, kProtoSimple>;
}

KernelFn interp_kernel_sum(int dtype, int ll) {
  constexpr int OP = dev::kSum;
  switch (dtype) {
    case 0: return pick<dev::RedInt<int8_t, OP>>(ll);
    case 1: return pick<dev::RedInt<uint8_t, OP>>(ll);
    case 2: return pick<dev::RedInt<int32_t, OP>>(ll);
    case 3: return pick<dev::RedInt<uint32_t, OP>>(ll);
    case 4: return pick<dev::RedInt<int64_t, OP>>(ll);
    case 5: return pick<dev::RedInt<uint64_t, OP>>(ll);
    case 6: return pick<dev::RedHalf<false, OP>>(ll);
    case 7: return pick<dev::RedFloat<float, OP>>(ll);
    case 8: return pick<dev::RedFloat<double, OP>>(ll);
    case 9: return pick<dev::RedHalf<true, OP>>(ll);
    default: return nullptr;
  }
}

}  // namespace gc3
