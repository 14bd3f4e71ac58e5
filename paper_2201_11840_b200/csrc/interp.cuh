// GC3-IR interpreter for sm_100a.
//
// One persistent launch per device executes every IR thread block of every rank hosted on that
// device (all thread blocks co-resident, cooperative launch). IR thread block b
// is replicated over `lanes` CUDA blocks; lane l owns tiles l, l+lanes, ... of every chunk, and
// has its own FIFOs and semaphores, so lanes never synchronise with each other. Within a lane the
// loop structure is the paper's: tiles outermost, instructions in order,
//   wait deps -> wait FIFO -> fused transfer (+reduction) -> publish FIFO / semaphore.
//
// Protocols:
//   Simple: payload stored with 128-bit vector stores into the receiver's FIFO slot, then one
//           release store of the slot counter (`head`); the receiver acquires it.
//   LL:     every 8 payload bytes travel in a 16-byte line {d0, flag, d1, flag} written with one
//           128-bit store; the receiver polls the flags, no fences on the data path.
// In both, the receiver returns the slot with a release store of `tail` into sender memory.
//
// Reductions are fused into the transfer (rrc / rrcs / rrs / reduce): no separate elementwise
// kernel exists. Arithmetic is the oracle's (oracle/gc3_oracle.c gc3o_reduce): f16/bf16 go
// through f32 and are rounded to nearest even, integers wrap, max/min select.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "devplan.hpp"

#ifndef GC3_UNROLL
#define GC3_UNROLL 4
#endif
#ifndef GC3_UNROLL_COPY
#define GC3_UNROLL_COPY 8
#endif
#ifndef GC3_MINBLOCKS
#define GC3_MINBLOCKS 1
#endif
#ifndef GC3_LL_BATCH  // LL lines in flight per thread
#define GC3_LL_BATCH 1
#endif
#ifndef GC3_TAIL_UNROLL  // vectors in flight per thread in the predicated tail of a data move
#define GC3_TAIL_UNROLL 1
#endif
#ifndef GC3_MOVE_NOINLINE  // compile the data mover once per reduction instead of at every op site
#define GC3_MOVE_NOINLINE 0
#endif
#if GC3_MOVE_NOINLINE
#define GC3_MOVE_ATTR __noinline__
#else
#define GC3_MOVE_ATTR
#endif

namespace gc3 {
namespace dev {

// ------------------------------------------------------------------ memory-model primitives
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel(bool sys) {
  if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v, bool sys) {
  if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// data loads bypass L1: the lines may have been written by other SMs/GPUs during this launch
__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_cg8(const void* p) {
  uint2 v;
  asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vec(uint4* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_vec8(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
// LL lines: strong (relaxed) 128-bit accesses at the scope of the peers (.gpu for same-device
// loopback ranks: STRONG.GPU stays in L2; .sys across GPUs)
__device__ __forceinline__ uint4 ld_line(const uint4* p, bool sys) {
  uint4 v;
  if (sys)
    asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_line(uint4* p, uint4 v, bool sys) {
  if (sys) asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// ------------------------------------------------------------------ arithmetic
__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
__device__ __forceinline__ uint16_t f32_to_bf16(float f) {  // RNE, NaN -> 0x7fff (oracle rule)
  uint32_t x = __float_as_uint(f);
  if ((x & 0x7f800000u) == 0x7f800000u && (x & 0x7fffffu)) return 0x7fff;
  x += 0x7fffu + ((x >> 16) & 1u);
  return static_cast<uint16_t>(x >> 16);
}
__device__ __forceinline__ float f16_to_f32(uint16_t h) {
  float f;
  asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
  return f;
}
__device__ __forceinline__ uint16_t f32_to_f16(float f) {  // RNE, NaN -> 0x7fff (oracle rule)
  if (f != f) return 0x7fff;
  uint16_t h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f));
  return h;
}
__device__ __forceinline__ float canon(float x) { return x != x ? __uint_as_float(0x7fffffffu) : x; }
__device__ __forceinline__ double canon(double x) { return x != x ? __longlong_as_double(0x7fffffffffffffffll) : x; }

enum RedOp { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };

template <typename T, int OP>
struct IntOp {
  __device__ static T apply(T a, T b) {
    using U = typename std::make_unsigned<T>::type;
    if (OP == kSum) return static_cast<T>(static_cast<U>(a) + static_cast<U>(b));
    if (OP == kProd) return static_cast<T>(static_cast<U>(a) * static_cast<U>(b));
    if (OP == kMax) return a > b ? a : b;
    return a < b ? a : b;
  }
};
template <typename F, int OP>
__device__ __forceinline__ F float_apply(F a, F b) {
  if (OP == kSum) return canon(a + b);
  if (OP == kProd) return canon(a * b);
  if (OP == kMax) return a != a ? b : (b != b ? a : (a > b ? a : b));
  return a != a ? b : (b != b ? a : (a < b ? a : b));
}

// Element-wise reduction functor over raw storage. kEsize = element bytes.
// kBulkAdd: the L2 can apply this reduction to a bulk copy bit-exactly (cp.reduce.async.bulk .add):
// 1 u32, 2 u64 (wrapping integer sums), 3 bf16, 4 f16 (.noftz), 5 f32 (round to nearest even; measured
// to keep subnormals and to give the oracle's NaN/inf bits: test_large_sums_with_special_values); 0 none
template <typename T, int OP>
struct RedInt {
  static constexpr int kEsize = sizeof(T);
  static constexpr bool kReduce = true;
  static constexpr int kBulkAdd = OP == kSum ? (sizeof(T) == 4 ? 1 : (sizeof(T) == 8 ? 2 : 0)) : 0;
  __device__ static void elem(const char* a, const char* b, char* o) {
    *reinterpret_cast<T*>(o) = IntOp<T, OP>::apply(*reinterpret_cast<const T*>(a), *reinterpret_cast<const T*>(b));
  }
  template <typename V>
  __device__ static V vec(V a, V b) {
    V r;
    const T* x = reinterpret_cast<const T*>(&a);
    const T* y = reinterpret_cast<const T*>(&b);
    T* z = reinterpret_cast<T*>(&r);
#pragma unroll
    for (int i = 0; i < static_cast<int>(sizeof(V) / sizeof(T)); ++i) z[i] = IntOp<T, OP>::apply(x[i], y[i]);
    return r;
  }
};
#ifndef GC3_F32_BULKADD  // f32 sums through the L2 too (subnormals kept: measured by the tests)
#define GC3_F32_BULKADD 1
#endif
template <typename F, int OP>
struct RedFloat {
  static constexpr int kEsize = sizeof(F);
  static constexpr bool kReduce = true;
  static constexpr int kBulkAdd = GC3_F32_BULKADD && OP == kSum && sizeof(F) == 4 ? 5 : 0;
  __device__ static void elem(const char* a, const char* b, char* o) {
    *reinterpret_cast<F*>(o) = float_apply<F, OP>(*reinterpret_cast<const F*>(a), *reinterpret_cast<const F*>(b));
  }
  template <typename V>
  __device__ static V vec(V a, V b) {
    V r;
    const F* x = reinterpret_cast<const F*>(&a);
    const F* y = reinterpret_cast<const F*>(&b);
    F* z = reinterpret_cast<F*>(&r);
#pragma unroll
    for (int i = 0; i < static_cast<int>(sizeof(V) / sizeof(F)); ++i) z[i] = float_apply<F, OP>(x[i], y[i]);
    return r;
  }
};
template <bool BF, int OP>
struct RedHalf {
  static constexpr int kEsize = 2;
  static constexpr bool kReduce = true;
  static constexpr int kBulkAdd = OP == kSum ? (BF ? 3 : 4) : 0;
  __device__ static uint16_t one(uint16_t a, uint16_t b) {
    const float p = BF ? bf16_to_f32(a) : f16_to_f32(a);
    const float q = BF ? bf16_to_f32(b) : f16_to_f32(b);
    if (OP == kMax || OP == kMin) {  // select keeps the operand bits
      const bool take_b = p != p ? true : (q != q ? false : (OP == kMax ? !(p > q) : !(p < q)));
      return take_b ? b : a;
    }
    const float r = float_apply<float, OP>(p, q);
    return BF ? f32_to_bf16(r) : f32_to_f16(r);
  }
  __device__ static void elem(const char* a, const char* b, char* o) {
    *reinterpret_cast<uint16_t*>(o) = one(*reinterpret_cast<const uint16_t*>(a), *reinterpret_cast<const uint16_t*>(b));
  }
  template <typename V>
  __device__ static V vec(V a, V b) {
    V r;
    const uint16_t* x = reinterpret_cast<const uint16_t*>(&a);
    const uint16_t* y = reinterpret_cast<const uint16_t*>(&b);
    uint16_t* z = reinterpret_cast<uint16_t*>(&r);
#pragma unroll
    for (int i = 0; i < static_cast<int>(sizeof(V) / 2); ++i) z[i] = one(x[i], y[i]);
    return r;
  }
};
// Copy-only programs (AllGather / AllToAll IRs): byte granularity, never reduces.
struct RedNone {
  static constexpr int kEsize = 1;
  static constexpr bool kReduce = false;
  static constexpr int kBulkAdd = 0;
  __device__ static void elem(const char* a, const char*, char* o) { *o = *a; }
  template <typename V>
  __device__ static V vec(V a, V) {
    return a;
  }
};

// ------------------------------------------------------------------ data movers
// Executed by the `n` threads of one unit; `t` is the thread's index in the unit.
// out0 (and out1 if non-null) = RED ? R(in0, in1) : in0, over nbytes. All pointers 16B aligned
// takes the 128-bit path; the ragged remainder (and misaligned segments) go element-wise.
template <class R, bool RED, bool TWO>
__device__ __forceinline__ void move_vec(const uint4* a, const uint4* b, uint4* o0, uint4* o1, int64_t nvec, int t, int n) {
  constexpr int U = R::kReduce ? GC3_UNROLL : GC3_UNROLL_COPY;  // 128-bit loads in flight per thread
  int64_t i = t;
  for (; i + (U - 1) * n < nvec; i += U * n) {
    uint4 x[U], y[U];
#pragma unroll
    for (int k = 0; k < U; ++k) x[k] = ld_cg(a + i + k * n);
    if (RED) {
#pragma unroll
      for (int k = 0; k < U; ++k) y[k] = ld_cg(b + i + k * n);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint4 v = RED ? R::template vec<uint4>(x[k], y[k]) : x[k];
      st_vec(o0 + i + k * n, v);
      if (TWO) st_vec(o1 + i + k * n, v);
    }
  }
  // the rest (< U vectors per thread) in predicated passes of T: a small tile costs one or two
  // memory round trips instead of one per vector
  constexpr int T = U < GC3_TAIL_UNROLL ? U : GC3_TAIL_UNROLL;
  for (; i < nvec; i += T * n) {
    uint4 x[T], y[T];
#pragma unroll
    for (int k = 0; k < T; ++k)
      if (i + k * n < nvec) x[k] = ld_cg(a + i + k * n);
    if (RED) {
#pragma unroll
      for (int k = 0; k < T; ++k)
        if (i + k * n < nvec) y[k] = ld_cg(b + i + k * n);
    }
#pragma unroll
    for (int k = 0; k < T; ++k) {
      if (i + k * n < nvec) {
        const uint4 v = RED ? R::template vec<uint4>(x[k], y[k]) : x[k];
        st_vec(o0 + i + k * n, v);
        if (TWO) st_vec(o1 + i + k * n, v);
      }
    }
  }
}

template <class R>
__device__ __forceinline__ void move_elems(const char* a, const char* b, char* o0, char* o1, int64_t nbytes, bool red, int t, int n) {
  constexpr int E = R::kEsize;
  for (int64_t i = t * static_cast<int64_t>(E); i < nbytes; i += static_cast<int64_t>(n) * E) {
    char tmp[E];
    if (red) R::elem(a + i, b + i, tmp);
    else
      for (int k = 0; k < E; ++k) tmp[k] = a[i + k];
    for (int k = 0; k < E; ++k) o0[i + k] = tmp[k];
    if (o1)
      for (int k = 0; k < E; ++k) o1[i + k] = tmp[k];
  }
}

template <class R>
__device__ GC3_MOVE_ATTR void move(const char* a, const char* b, char* o0, char* o1, int64_t nbytes, int t, int n) {
  if (nbytes <= 0) return;
  if (!o0) {
    o0 = o1;
    o1 = nullptr;
  }
  const bool red = R::kReduce && b != nullptr;
  const uintptr_t align = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(o0) |
                          (b ? reinterpret_cast<uintptr_t>(b) : 0) | (o1 ? reinterpret_cast<uintptr_t>(o1) : 0);
  int64_t done = 0;
  if ((align & 15) == 0) {
    const int64_t nvec = nbytes >> 4;
    const uint4* va = reinterpret_cast<const uint4*>(a);
    const uint4* vb = reinterpret_cast<const uint4*>(b);
    uint4* v0 = reinterpret_cast<uint4*>(o0);
    uint4* v1 = reinterpret_cast<uint4*>(o1);
    if (red) {
      if (o1) move_vec<R, true, true>(va, vb, v0, v1, nvec, t, n);
      else move_vec<R, true, false>(va, vb, v0, v1, nvec, t, n);
    } else {
      if (o1) move_vec<R, false, true>(va, vb, v0, v1, nvec, t, n);
      else move_vec<R, false, false>(va, vb, v0, v1, nvec, t, n);
    }
    done = nvec << 4;
  }
  if (done < nbytes)
    move_elems<R>(a + done, b ? b + done : nullptr, o0 + done, o1 ? o1 + done : nullptr, nbytes - done, red, t, n);
}

// ------------------------------------------------------------------ TMA bulk copies
// Pure-copy ops (send, recv, copy, rcs) on the Simple protocol move through shared memory with the
// Tensor Memory Accelerator's 1-D bulk engine: one thread keeps `stages` x kStageBytes in flight
// (cp.async.bulk global->shared, completion on an mbarrier; cp.async.bulk shared->global as bulk
// groups), so the unit's bandwidth no longer depends on registers or resident warps.
constexpr int kStageBytes = 16 << 10;  // largest stage (LaunchArgs::stage_bytes picks <= this)
constexpr int kMaxStages = 8;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load_plain(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// every span this runtime bulk-loads is read once (inputs, pulled spans, forwarded spans, FIFO slots):
// with a policy (L2 evict_first) the lines make room for data still to be read
__device__ __forceinline__ void bulk_load_hint(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  if (pol) bulk_load_hint(smem, gmem, bytes, bar, pol);
  else bulk_load_plain(smem, gmem, bytes, bar);
}
__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gmem, const void* smem, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem), "r"(smem_addr(smem)),
               "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_vec_hint(uint4* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
template <int K>
__device__ __forceinline__ void bulk_reduce_add(void* gmem, const void* smem, uint32_t bytes) {
  if (K == 1)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)), "r"(bytes) : "memory");
  if (K == 2)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)), "r"(bytes) : "memory");
  if (K == 3)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.noftz.bf16 [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)), "r"(bytes) : "memory");
  if (K == 4)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.noftz.f16 [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)), "r"(bytes) : "memory");
  if (K == 5)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gmem), "r"(smem_addr(smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Ops whose data movement is a plain copy (no reduction); recv with the message already in place
// moves nothing.
__device__ __forceinline__ bool is_tma_copy(int op, bool in_direct) {
  return op == kOpSend || op == kOpCopy || op == kOpRcs || (op == kOpRecv && !in_direct);
}

// Per-unit bulk-copy pipeline state (lives in thread 0 of the unit).
struct Tma {
  char* stage;    // stages x sb bytes of shared memory
  int sb;         // bytes per stage (a multiple of 1 KiB, <= kStageBytes)
  uint64_t* bar;  // one mbarrier per stage
  int stages;
  uint32_t* seq;  // (shared) pieces issued so far: stage = seq % stages, parity = (seq / stages) & 1;
                  // written by thread 0 at the end of an op, read by the unit's threads in a later one
  uint64_t pol;     // L2 policy for the stores of the current op (0: none)
  uint64_t pol_rd;  // L2 policy for the bulk loads (0: none)
};

// Copies `count` segments of `nbytes` (segment j: a + j*sa -> o0 + j*s0 [, o1 + j*s1]).
// Called by thread 0 of the unit; returns after every store has completed (async-proxy writes
// ordered for the generic proxy by the caller's fence.proxy.async).
// K > 0: the stores are L2 reductions (o0 += piece, see kBulkAdd) instead of copies
template <int K = 0>
static __device__ void tma_copy(Tma& m, const char* a, int64_t sa, char* o0, int64_t s0, char* o1, int64_t s1, int64_t nbytes,
                         int count) {
  const int SB = m.sb;
  const int64_t per_seg = (nbytes + SB - 1) / SB;
  const int64_t total = per_seg * count;
  auto piece = [&](int64_t p, const char*& src, char*& d0, char*& d1, uint32_t& bytes) {
    const int64_t j = p / per_seg, k = p - j * per_seg;
    const int64_t off = k * SB;
    bytes = static_cast<uint32_t>(min(static_cast<int64_t>(SB), nbytes - off));
    src = a + j * sa + off;
    d0 = o0 + j * s0 + off;
    d1 = o1 ? o1 + j * s1 + off : nullptr;
  };
  const uint32_t base = *m.seq;
  const int64_t prime = min(static_cast<int64_t>(m.stages), total);
  for (int64_t p = 0; p < prime; ++p) {
    const char* src;
    char *d0, *d1;
    uint32_t bytes;
    piece(p, src, d0, d1, bytes);
    const uint32_t g = base + static_cast<uint32_t>(p);
    uint64_t* bar = m.bar + g % m.stages;
    mbar_expect_tx(bar, bytes);
    bulk_load(m.stage + static_cast<size_t>(g % m.stages) * SB, src, bytes, bar, m.pol_rd);
  }
  for (int64_t p = 0; p < total; ++p) {
    const char* src;
    char *d0, *d1;
    uint32_t bytes;
    piece(p, src, d0, d1, bytes);
    const uint32_t g = base + static_cast<uint32_t>(p);
    char* sm = m.stage + static_cast<size_t>(g % m.stages) * SB;
    mbar_wait(m.bar + g % m.stages, (g / m.stages) & 1);
    if (K) {
      bulk_reduce_add<K>(d0, sm, bytes);
    } else if (m.pol) {
      bulk_store_hint(d0, sm, bytes, m.pol);
      if (d1) bulk_store_hint(d1, sm, bytes, m.pol);
    } else {
      bulk_store(d0, sm, bytes);
      if (d1) bulk_store(d1, sm, bytes);
    }
    bulk_commit();
    // refill the previous piece's stage once its store has read it: the store just issued stays in
    // flight (wait_group.read 1), so loads and stores overlap instead of alternating
    const int64_t rp = m.stages > 1 ? p - 1 : p, np = rp + m.stages;
    if (rp >= 0 && np < total) {
      if (m.stages > 1) bulk_wait_read_1();
      else bulk_wait_read_all();  // one stage: it is the one just stored
      const uint32_t rg = base + static_cast<uint32_t>(rp);
      const char* nsrc;
      char *n0, *n1;
      uint32_t nbytes_p;
      piece(np, nsrc, n0, n1, nbytes_p);
      uint64_t* bar = m.bar + rg % m.stages;
      mbar_expect_tx(bar, nbytes_p);
      bulk_load(m.stage + static_cast<size_t>(rg % m.stages) * SB, nsrc, nbytes_p, bar, m.pol_rd);
    }
  }
  bulk_wait_all();
  *m.seq = base + static_cast<uint32_t>(total);
}

__device__ __forceinline__ void unit_sync(int uw, int bar_id, int n);
// Streams through the bulk engine: the operand(s) of every piece (half a stage each when reducing)
// are brought into shared memory by cp.async.bulk, `stages` pieces in flight per unit regardless of
// registers; every thread of the unit then combines its 16-byte vectors from shared memory (R::vec,
// operand order a (op) b exactly as the register path) and stores the result with st.global to o0
// [and o1]. Stores leave from registers, so a stage is free as soon as it has been read: loads keep
// (almost) every stage in flight, unlike bulk stores that hold their stage until they have read it.
// Segment j: a + j*sa [, b + j*sb] -> o0 + j*s0 [, o1 + j*s1], nbytes each (all 16-byte aligned).
template <class R, bool RED>
__device__ void tma_stream(Tma& m, const char* a, int64_t sa, const char* b, int64_t sb, char* o0, int64_t s0, char* o1,
                           int64_t s1, int64_t nbytes, int count, int t, int n, int uw, int bar_id) {
  const int SB = m.sb;
  const int P = RED ? SB / 2 : SB;  // bytes of one operand per piece
  const int64_t per_seg = (nbytes + P - 1) / P;
  const int64_t total = per_seg * count;
  auto piece = [&](int64_t p, int64_t& j, int64_t& off, uint32_t& bytes) {
    j = p / per_seg;
    off = (p - j * per_seg) * P;
    bytes = static_cast<uint32_t>(min(static_cast<int64_t>(P), nbytes - off));
  };
  const uint32_t base = *m.seq;
  auto issue = [&](int64_t p) {  // thread 0: the operands of piece p into its stage
    int64_t j, off;
    uint32_t bytes;
    piece(p, j, off, bytes);
    const uint32_t g = base + static_cast<uint32_t>(p);
    char* st = m.stage + static_cast<size_t>(g % m.stages) * SB;
    uint64_t* bar = m.bar + g % m.stages;
    mbar_expect_tx(bar, RED ? 2 * bytes : bytes);
    bulk_load(st, a + j * sa + off, bytes, bar, m.pol_rd);
    if (RED) bulk_load(st + P, b + j * sb + off, bytes, bar, m.pol_rd);
  };
  if (t == 0) {
    fence_proxy_async_global();  // generic-proxy acquires (deps, flags) -> async-proxy reads
    for (int64_t p = 0; p < min(static_cast<int64_t>(m.stages), total); ++p) issue(p);
  }
  for (int64_t p = 0; p < total; ++p) {
    int64_t j, off;
    uint32_t bytes;
    piece(p, j, off, bytes);
    const uint32_t g = base + static_cast<uint32_t>(p);
    const char* st = m.stage + static_cast<size_t>(g % m.stages) * SB;
    mbar_wait(m.bar + g % m.stages, (g / m.stages) & 1);
    const uint4* x = reinterpret_cast<const uint4*>(st);
    const uint4* y = reinterpret_cast<const uint4*>(st + P);
    uint4* d0 = reinterpret_cast<uint4*>(o0 + j * s0 + off);
    uint4* d1 = o1 ? reinterpret_cast<uint4*>(o1 + j * s1 + off) : nullptr;
    for (int v = t; v < static_cast<int>(bytes >> 4); v += n) {
      const uint4 r = RED ? R::template vec<uint4>(x[v], y[v]) : x[v];
      if (m.pol) {
        st_vec_hint(d0 + v, r, m.pol);
        if (d1) st_vec_hint(d1 + v, r, m.pol);
      } else {
        st_vec(d0 + v, r);
        if (d1) st_vec(d1 + v, r);
      }
    }
    unit_sync(uw, bar_id, n);  // the stage is consumed (stores issued from registers): refill it
    if (t == 0 && p + m.stages < total) issue(p + m.stages);
  }
  if (t == 0) *m.seq = base + static_cast<uint32_t>(total);
}

// ------------------------------------------------------------------ launch prologue
// Every rank's buffers of the launch, staged in shared memory once per block: one strided copy
// straight from the parameter bank (the kernels take LaunchArgs as __grid_constant__, so indexing
// it dynamically neither copies it to local memory nor unrolls into a per-thread branch table —
// the unrolled form compiled to ~80 KB of divergent code whose instruction-cache misses cost
// ~9 us at the first barrier of every launch; ncu, profiles/r02bc_prologue.md).
__device__ __forceinline__ void stage_bufs(const LaunchArgs& a, char** s_bufs) {
  char* const* flat = &a.bufs[0][0];
  for (int i = threadIdx.x; i < kMaxLocalRanks * kBufs; i += blockDim.x) s_bufs[i] = flat[i];
}

// The semaphore / progress tag of this launch. Read from device memory (not a kernel argument) so
// a launch captured in a CUDA graph gets a new epoch at every replay: every block reads the counter
// once, and the last block to do so advances it for the next launch (launches of a device are
// serialised, so the next one starts after every block of this one has read it).
__device__ __forceinline__ uint64_t launch_epoch(uint64_t* epoch_ptr, int32_t* epoch_ctr, uint64_t fallback) {
  if (!epoch_ptr) return fallback;
  uint64_t e;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(e) : "l"(epoch_ptr) : "memory");
  if (atomicAdd(epoch_ctr, 1) == static_cast<int>(gridDim.x) - 1) {
    *epoch_ctr = 0;
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(epoch_ptr), "l"(e + 1) : "memory");
  }
  return e;
}

// ------------------------------------------------------------------ watchdog
// Everything here is passed by value (a small struct the spin loops keep in registers).
struct Ctx {
  int32_t* abort_flag;
  uint64_t* err_info;
  uint64_t timeout_ns;
  int rank_slot, tbi, step;
  int64_t tile;
};

static __device__ __noinline__ void raise_timeout(const Ctx c, int what) {
  if (atomicCAS(c.abort_flag, 0, 1) == 0 && c.err_info) {
    volatile uint64_t* e = c.err_info;
    e[1] = static_cast<uint64_t>(c.rank_slot);
    e[2] = static_cast<uint64_t>(c.tbi);
    e[3] = static_cast<uint64_t>(c.step);
    e[4] = static_cast<uint64_t>(c.tile);
    e[5] = static_cast<uint64_t>(what);
    __threadfence_system();
    e[0] = 1;  // code: watchdog timeout
  }
}

// Spins until *p >= target; false if the launch was aborted. Polls with relaxed loads (an acquire
// load would invalidate L1 on every iteration); once the flag is reached, one acquire load of it
// (the flag only grows, so it still satisfies the target) synchronises with the publisher's
// release pattern. A load rather than a fence: fence.acq_rel would also wait for this thread's own
// outstanding stores (the previous op's flag stores) to be acknowledged — one L2 round trip per op
// on the critical path (C1 80.6 -> 75.9 us, profiles/r02be_trace.txt).
__device__ __forceinline__ bool wait_geq(const uint64_t* p, uint64_t target, bool sys, const Ctx& c, int what) {
  if (ld_acquire(p, sys) >= target) return true;
  const uint64_t start = globaltimer();
  for (int n = 0;; ++n) {
    if (ld_relaxed(p, sys) >= target) {
      ld_acquire(p, sys);
      return true;
    }
    if ((n & 255) == 255) {
      if (*reinterpret_cast<volatile int*>(c.abort_flag)) return false;
      if (c.timeout_ns && globaltimer() - start > c.timeout_ns) {
        raise_timeout(c, what);
        return false;
      }
    }
  }
}

__device__ __forceinline__ bool is_recv(int op) {
  return op == kOpRecv || op == kOpRrc || op == kOpRcs || op == kOpRrcs || op == kOpRrs;
}
__device__ __forceinline__ bool is_send(int op) { return op == kOpSend || op == kOpRcs || op == kOpRrcs || op == kOpRrs; }

// ------------------------------------------------------------------ LL op body
// Lines of the incoming/outgoing message are distributed over the unit's threads; every thread
// polls the flags of its own lines only. The incoming message comes from inl (LL lines), inp (pulled
// from the sender's span; its head flag was acquired before the op) or is in place (direct) or
// absent; the outgoing one goes to outl (LL lines), outd (direct, plain stores) or nowhere (pulled).
template <class R>
__device__ bool ll_op(int opcode, int count, char* src0, const char* srcr0, char* dst0, int64_t chunk_bytes, int64_t tbytes, const uint4* inl,
                      const char* inp, uint4* outl, char* outd, uint32_t in_flag, uint32_t out_flag, bool sys, const Ctx& c,
                      int t, int n) {
  constexpr int U = GC3_LL_BATCH;  // lines in flight per thread: their loads are issued together, then polled
  const int64_t lines_per_seg = tbytes >> 3;
  const int64_t nlines = lines_per_seg * count;
  const bool send = is_send(opcode);
  // ops that read their local span: send, rrc, rrcs, rrs, and rcs whose message is already in place
  const bool reads_src = opcode == kOpSend || opcode == kOpRrc || opcode == kOpRrcs || opcode == kOpRrs ||
                         (opcode == kOpRcs && !inl && !inp);
  for (int64_t k0 = t; k0 < nlines; k0 += static_cast<int64_t>(U) * n) {
    uint4 l[U];
    uint2 own[U];
    int64_t off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + static_cast<int64_t>(u) * n;
      if (k >= nlines) continue;
      const int64_t j = k / lines_per_seg;
      off[u] = ((k - j * lines_per_seg) << 3) + j * chunk_bytes;
      if (inl) l[u] = ld_line(inl + k, sys);
      if (inp) {  // pulled: the sender's span, laid out like the local one
        const uint2 m = ld_cg8(inp + off[u]);
        l[u] = make_uint4(m.x, in_flag, m.y, in_flag);
      }
      if (reads_src) own[u] = ld_cg8((opcode == kOpRcs ? src0 : srcr0) + off[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + static_cast<int64_t>(u) * n;
      if (k >= nlines || !inl) continue;
      if (l[u].y != in_flag || l[u].w != in_flag) {
        const uint64_t start = globaltimer();
        for (int it = 0;; ++it) {
          l[u] = ld_line(inl + k, sys);
          if (l[u].y == in_flag && l[u].w == in_flag) break;
          if ((it & 255) == 255) {
            if (*reinterpret_cast<volatile int*>(c.abort_flag)) return false;
            if (c.timeout_ns && globaltimer() - start > c.timeout_ns) {
              raise_timeout(c, 4);
              return false;
            }
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = k0 + static_cast<int64_t>(u) * n;
      if (k >= nlines) continue;
      const bool has_msg = inl || inp;
      const uint2 msg = has_msg ? make_uint2(l[u].x, l[u].z) : make_uint2(0, 0);
      char* src = src0 + off[u];
      char* dst = dst0 + off[u];
      uint2 v;
      switch (opcode) {
        case kOpSend: v = own[u]; break;
        case kOpRecv:
          if (has_msg) st_vec8(dst, msg);
          continue;
        case kOpRrc: st_vec8(dst, R::template vec<uint2>(own[u], msg)); continue;
        case kOpRcs:
          if (has_msg) {
            v = msg;
            st_vec8(src, v);
          } else {
            v = own[u];  // direct: the message is already in the local span
          }
          break;
        case kOpRrcs: v = R::template vec<uint2>(own[u], msg); st_vec8(src, v); break;
        case kOpRrs: v = R::template vec<uint2>(own[u], msg); break;
        default: continue;
      }
      if (send) {
        if (outl) st_line(outl + k, make_uint4(v.x, out_flag, v.y, out_flag), sys);
        else if (outd) st_vec8(outd + off[u], v);
      }
    }
  }
  return true;
}

// ------------------------------------------------------------------ LL128 op body
// LL128 (NCCL's 128-byte-line protocol): a message travels as 128-byte lines of
// 15 payload words (8 bytes each) and one 8-byte flag word, the 64-bit message sequence number.
// Eight consecutive threads of a warp own one line and write it with one 16-byte store each (the
// eighth thread carries the flag in its upper half), so a warp-wide store puts whole lines in one
// memory transaction; a receiver whose eight threads load the line together and see the flag has
// the whole payload. Lines whose flag does not match yet are re-loaded by their eight threads
// together. 120 of every 128 bytes are payload (LL: 8 of 16); no fences on the data path.
// Line k of the message is segment k / lps, payload words (k % lps) * 15 ... + 14 of that segment.
#ifndef GC3_LL128_BATCH  // lines in flight per 8-thread group
#define GC3_LL128_BATCH 2
#endif
constexpr int kLL128Words = 15;
__device__ __forceinline__ uint64_t ll128_flag(const uint4& v) { return (static_cast<uint64_t>(v.w) << 32) | v.z; }

template <class R>
__device__ bool ll128_op(int opcode, int count, char* src0, const char* srcr0, char* dst0, int64_t chunk_bytes, int64_t tbytes,
                         const uint4* inl, uint4* outl, uint64_t in_flag, uint64_t out_flag, bool sys, const Ctx& c, int t, int n) {
  constexpr int U = GC3_LL128_BATCH;
  const int64_t words = tbytes >> 3;
  const int64_t lps = (words + kLL128Words - 1) / kLL128Words;
  const int64_t nlines = lps * count;
  const bool send = is_send(opcode);
  // ops that read their local span: send, rrc, rrcs, rrs, and rcs whose message is already in place
  const bool reads_src = opcode == kOpSend || opcode == kOpRrc || opcode == kOpRrcs || opcode == kOpRrs || (opcode == kOpRcs && !inl);
  const int lt = t & 31, g = lt >> 3, j8 = lt & 7;
  const int w = t >> 5, nw = n >> 5;
  const bool flag_thread = j8 == 7;
  const int mywords = flag_thread ? 1 : 2;  // payload words of this thread in its line
  const int64_t step = static_cast<int64_t>(nw) * 4 * U;
  for (int64_t kb = static_cast<int64_t>(w) * 4 * U; kb < nlines; kb += step) {
    uint4 l[U];
    uint2 own[U][2];
    int64_t off[U];
    int nv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = kb + u * 4 + g;  // a warp covers 4 consecutive lines per u: 512 contiguous bytes
      nv[u] = -1;
      off[u] = 0;
      if (k >= nlines) continue;
      const int64_t seg = k / lps, line = k - seg * lps;
      const int64_t wi = line * kLL128Words + 2 * j8;
      const int64_t left = words - wi;
      nv[u] = left <= 0 ? 0 : (left < mywords ? static_cast<int>(left) : mywords);
      off[u] = seg * chunk_bytes + wi * 8;
      if (inl) l[u] = ld_line(inl + k * 8 + j8, sys);
      if (reads_src) {
        const char* s = (opcode == kOpRcs ? src0 : srcr0) + off[u];
        if (nv[u] > 0) own[u][0] = ld_cg8(s);
        if (nv[u] > 1) own[u][1] = ld_cg8(s + 8);
      }
    }
    if (inl) {
      const uint64_t start = globaltimer();
      for (int it = 0;; ++it) {
        bool bad[U], any = false;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bad[u] = nv[u] >= 0 && flag_thread && ll128_flag(l[u]) != in_flag;
          any = any || bad[u];
        }
        if (!__any_sync(0xffffffffu, any)) break;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          // the line's eight threads re-load it together (one transaction)
          if (__shfl_sync(0xffffffffu, bad[u], lt | 7)) l[u] = ld_line(inl + (kb + u * 4 + g) * 8 + j8, sys);
        }
        if ((it & 255) == 255) {
          if (*reinterpret_cast<volatile int*>(c.abort_flag)) return false;
          if (c.timeout_ns && globaltimer() - start > c.timeout_ns) {
            raise_timeout(c, 4);
            return false;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (nv[u] < 0) continue;  // the whole 8-thread group is past the end
      const uint2 msg[2] = {make_uint2(l[u].x, l[u].y), make_uint2(l[u].z, l[u].w)};
      char* src = src0 + off[u];
      char* dst = dst0 + off[u];
      uint2 v[2] = {make_uint2(0, 0), make_uint2(0, 0)};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i >= nv[u]) break;
        switch (opcode) {
          case kOpSend: v[i] = own[u][i]; break;
          case kOpRecv:
            if (inl) st_vec8(dst + 8 * i, msg[i]);
            break;
          case kOpRrc: st_vec8(dst + 8 * i, R::template vec<uint2>(own[u][i], msg[i])); break;
          case kOpRcs:
            if (inl) {
              v[i] = msg[i];
              st_vec8(src + 8 * i, v[i]);
            } else {
              v[i] = own[u][i];
            }
            break;
          case kOpRrcs:
            v[i] = R::template vec<uint2>(own[u][i], msg[i]);
            st_vec8(src + 8 * i, v[i]);
            break;
          case kOpRrs: v[i] = R::template vec<uint2>(own[u][i], msg[i]); break;
          default: break;
        }
      }
      if (send && outl) {
        const uint4 line = flag_thread ? make_uint4(v[0].x, v[0].y, static_cast<uint32_t>(out_flag), static_cast<uint32_t>(out_flag >> 32))
                                       : make_uint4(v[0].x, v[0].y, v[1].x, v[1].y);
        st_line(outl + (kb + u * 4 + g) * 8 + j8, line, sys);
      }
    }
  }
  return true;
}

// The data movement of one op on one tile (Simple transports): staged reductions, bulk copies or
// the register path. `in` is the incoming message (FIFO slot or pulled span; segment j at
// + j * in_stride; null when already in place or absent), `out` the outgoing one (FIFO slot or the
// receiver's span; null when pulled or absent). Reads of the op's spans go through srcr / dstr.
#ifndef GC3_TRANSFER_NOINLINE
#define GC3_TRANSFER_NOINLINE 0
#endif
#if GC3_TRANSFER_NOINLINE
#define GC3_TRANSFER_ATTR __noinline__
#else
#define GC3_TRANSFER_ATTR __forceinline__
#endif
template <class R>
__device__ GC3_TRANSFER_ATTR void transfer(const DevOp& op, bool in_d, char* src, char* dst, const char* srcr, const char* dstr,
                                         const char* in, int64_t in_stride, char* out, int64_t out_stride, int64_t tbytes,
                                         int64_t chunk_bytes, int tma_ops, Tma& tma, int t, int n, int uw, int bar_id,
                                         int64_t tma_min) {
  // small transfers take the register path: one round trip, no bulk-engine setup latency
  if (tbytes * op.count < tma_min) tma_ops = 0;
  if (R::kBulkAdd && (tma_ops & 8) && tma.stages > 0 && in && !out && srcr == src &&
      (op.opcode == kOpRrcs || (op.opcode == kOpRrc && dst == src)) &&
      ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(in) | static_cast<uintptr_t>(tbytes) |
        static_cast<uintptr_t>(chunk_bytes) | static_cast<uintptr_t>(in_stride)) & 15) == 0) {
    // in-place sum: the message streams through shared memory and the L2 adds it into the local
    // span (cp.reduce.async.bulk); the SM never loads the local operand
    if (t == 0 && tbytes > 0) {
      fence_proxy_async_global();
      tma_copy<R::kBulkAdd>(tma, in, in_stride, src, chunk_bytes, nullptr, 0, tbytes, op.count);
      fence_proxy_async_global();
    }
  } else if (R::kReduce && (tma_ops & 2) && tma.stages >= 2 && in &&
             (op.opcode == kOpRrc || op.opcode == kOpRrcs || op.opcode == kOpRrs) &&
             ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(srcr) | reinterpret_cast<uintptr_t>(dst) |
               reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out) | static_cast<uintptr_t>(tbytes) |
               static_cast<uintptr_t>(chunk_bytes) | static_cast<uintptr_t>(in_stride)) & 15) == 0) {
    // staged reduction: local operand (op.src read) (op) message, both through shared memory
    switch (op.opcode) {
      case kOpRrc: tma_stream<R, true>(tma, srcr, chunk_bytes, in, in_stride, dst, chunk_bytes, nullptr, 0, tbytes, op.count, t, n, uw, bar_id); break;
      case kOpRrcs: tma_stream<R, true>(tma, srcr, chunk_bytes, in, in_stride, src, chunk_bytes, out, out_stride, tbytes, op.count, t, n, uw, bar_id); break;
      case kOpRrs:
        if (out) tma_stream<R, true>(tma, srcr, chunk_bytes, in, in_stride, out, out_stride, nullptr, 0, tbytes, op.count, t, n, uw, bar_id);
        break;
      default: break;
    }
  } else if ((tma_ops & 1) && tma.stages > 0 && is_tma_copy(op.opcode, in_d) &&
             ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(in) |
               reinterpret_cast<uintptr_t>(out) | static_cast<uintptr_t>(tbytes) | static_cast<uintptr_t>(chunk_bytes)) & 15) == 0) {
    if (tma_ops & 4) {  // bulk loads, stores from registers by the whole unit
      switch (op.opcode) {
        case kOpSend:
          if (out) tma_stream<R, false>(tma, srcr, chunk_bytes, nullptr, 0, out, out_stride, nullptr, 0, tbytes, op.count, t, n, uw, bar_id);
          break;
        case kOpRecv: tma_stream<R, false>(tma, in, in_stride, nullptr, 0, dst, chunk_bytes, nullptr, 0, tbytes, op.count, t, n, uw, bar_id); break;
        case kOpCopy: tma_stream<R, false>(tma, srcr, chunk_bytes, nullptr, 0, dst, chunk_bytes, nullptr, 0, tbytes, op.count, t, n, uw, bar_id); break;
        case kOpRcs:
          if (!in_d) tma_stream<R, false>(tma, in, in_stride, nullptr, 0, src, chunk_bytes, out, out_stride, tbytes, op.count, t, n, uw, bar_id);
          else if (out) tma_stream<R, false>(tma, src, chunk_bytes, nullptr, 0, out, out_stride, nullptr, 0, tbytes, op.count, t, n, uw, bar_id);
          break;
        default: break;
      }
    } else if (t == 0 && tbytes > 0) {  // one thread drives the bulk engine; the unit waits at the barrier
      fence_proxy_async_global();  // generic-proxy acquires above -> async-proxy reads
      switch (op.opcode) {
        case kOpSend:
          if (out) tma_copy(tma, srcr, chunk_bytes, out, out_stride, nullptr, 0, tbytes, op.count);
          break;
        case kOpRecv: tma_copy(tma, in, in_stride, dst, chunk_bytes, nullptr, 0, tbytes, op.count); break;
        case kOpCopy: tma_copy(tma, srcr, chunk_bytes, dst, chunk_bytes, nullptr, 0, tbytes, op.count); break;
        case kOpRcs:
          if (!in_d) tma_copy(tma, in, in_stride, src, chunk_bytes, out, out_stride, tbytes, op.count);
          else if (out) tma_copy(tma, src, chunk_bytes, out, out_stride, nullptr, 0, tbytes, op.count);
          break;
        default: break;
      }
      fence_proxy_async_global();  // async-proxy writes -> the generic release below
    }
  } else {
    for (int j = 0; j < op.count; ++j) {
      char* sj = src + j * chunk_bytes;
      char* dj = dst + j * chunk_bytes;
      const char* sr = srcr + j * chunk_bytes;
      const char* dr = dstr + j * chunk_bytes;
      const char* mi = in ? in + j * in_stride : nullptr;
      char* mo = out ? out + j * out_stride : nullptr;
      switch (op.opcode) {
        case kOpSend:
          if (mo) move<R>(sr, nullptr, mo, nullptr, tbytes, t, n);
          break;
        case kOpRecv:
          if (mi) move<R>(mi, nullptr, dj, nullptr, tbytes, t, n);
          break;
        case kOpCopy: move<R>(sr, nullptr, dj, nullptr, tbytes, t, n); break;
        case kOpReduce: move<R>(dr, sr, dj, nullptr, tbytes, t, n); break;
        case kOpRrc: move<R>(sr, mi, dj, nullptr, tbytes, t, n); break;
        case kOpRcs:
          if (mi) move<R>(mi, nullptr, sj, mo, tbytes, t, n);
          else if (mo) move<R>(sj, nullptr, mo, nullptr, tbytes, t, n);
          break;
        case kOpRrcs: move<R>(sr, mi, sj, mo, tbytes, t, n); break;
        case kOpRrs: move<R>(sr, mi, nullptr, mo, tbytes, t, n); break;
        default: break;
      }
    }
  }
}

// Clipped tiles (ragged AllReduce on the caller's buffer): the rank block holds `clip` elements, chunk
// k covers elements [k * chunk_elems, (k + 1) * chunk_elems) of it, so the tile of an op on chunk k
// is cut at the block's end (possibly to nothing: the op then only synchronises). 0: no clipping.
__device__ __forceinline__ int64_t clip_tile(int64_t clip, int64_t chunk_elems, int chunk, int64_t t0, int64_t tlen) {
  if (clip <= 0) return tlen;
  const int64_t v = clip - static_cast<int64_t>(chunk) * chunk_elems - t0;
  return v <= 0 ? 0 : min(v, tlen);
}

// ------------------------------------------------------------------ the interpreter
// A "unit" of `unit_warps` warps interprets one (IR thread block, lane): for each tile of the lane,
// for each op in order:
//   (1) wait: deps on other thread blocks' semaphores, a free outgoing FIFO slot,
//       a posted incoming message -- polled in parallel by different threads of the unit;
//   (2) move: the unit's threads move the op's bytes, the reduction fused into the transfer;
//   (3) publish: after a unit barrier, thread 0 fences and posts the slot counter, frees the
//       incoming slot and sets the semaphore.
// A CUDA block holds kThreads/32/unit_warps units, so small units give many independent pipelines
// (a thread block's tiles are serial inside one lane; concurrency comes from lanes).
// Units sync with __syncwarp (1 warp) or a per-unit named barrier (bar.sync id, n).
__device__ __forceinline__ bool unit_and(bool p, int uw, int bar_id, int n) {
  if (uw == 1) return __all_sync(0xffffffffu, p);
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbar.red.and.pred q, %2, %3, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r) : "r"(static_cast<int>(p)), "r"(bar_id), "r"(n) : "memory");
  return r != 0;
}
__device__ __forceinline__ void unit_sync(int uw, int bar_id, int n) {
  if (uw == 1) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(n) : "memory");
}

// Work-queue mode (programs whose messages are all direct or pulled, Simple protocol, every rank in
// this launch). A work item is one (thread block, tile): the unit that claims it runs all of the
// thread block's ops on that tile in order. Units claim items from one counter in tile-major order
// (item = tile * ntbs + thread block), so a unit never idles while any work is left, whatever the
// phase structure of the program. Deps and message deps wait on a per-(thread block, tile) progress
// word; every dependency of an item is on the same tile, and with at least ntbs co-resident units all
// items of a tile are claimed before any unit can block on one of them: no deadlock.
#ifndef GC3_WQ_NOINLINE
#define GC3_WQ_NOINLINE 0
#endif
#if GC3_WQ_NOINLINE
#define GC3_WQ_ATTR __noinline__
#else
#define GC3_WQ_ATTR
#endif
struct WqArgs {  // the launch arguments the work queue reads (by value: no local copy of LaunchArgs)
  const DevTb* tbs;
  const DevOp* ops;
  const DevDep* deps;
  int32_t* wq_next;
  const int32_t* wq_order;
  uint64_t* prog;
  int32_t* abort_flag;
  uint64_t* err_info;
  uint64_t timeout_ns;
  int64_t chunk_elems, tile_elems, ntiles;
  uint64_t epoch;
  int ntbs, tma_ops;
  int64_t tma_min;
};

template <class R>
__device__ GC3_WQ_ATTR void interp_wq(const WqArgs a, char* const* s_bufs, Tma& tma, uint64_t pol_last, int t, int n, int uw, int uib,
                          int bar_id) {
  __shared__ int s_item[kThreads / 32];
  const int64_t chunk_elems = a.chunk_elems, tile_elems = a.tile_elems, ntiles = a.ntiles;
  const int64_t chunk_bytes = chunk_elems * R::kEsize;
  const int64_t nitems = ntiles * a.ntbs;
  const uint64_t tag = a.epoch << 32;
  for (;;) {
    if (t == 0) s_item[uib] = static_cast<int>(atomicAdd(a.wq_next, 1));
    unit_sync(uw, bar_id, n);
    const int64_t claim = s_item[uib];
    if (claim >= nitems) return;
    const int64_t item = a.wq_order ? a.wq_order[claim] : claim;
    const int tbi = static_cast<int>(item % a.ntbs);
    const int64_t tile = item / a.ntbs;
    const DevTb tb = a.tbs[tbi];
    char* const* const mine = s_bufs + kBufs * tb.rank_slot;
    char* const* const peer = s_bufs + kBufs * (tb.peer_slot >= 0 ? tb.peer_slot : 0);
    char* const* const rpeer = s_bufs + kBufs * (tb.recv_slot >= 0 ? tb.recv_slot : 0);
    const DevOp* const ops = a.ops + tb.op_begin;
    const int64_t t0 = tile * tile_elems;
    const int64_t tbytes = min(tile_elems, chunk_elems - t0) * R::kEsize;
    const int64_t t0_bytes = t0 * R::kEsize;
    Ctx c{a.abort_flag, a.err_info, a.timeout_ns, tb.rank_slot, tbi, 0, tile};
    for (int s = 0; s < tb.nops; ++s) {
      const DevOp op = ops[s];
      c.step = s;
      tma.pol = op.hot ? pol_last : 0;
      bool ok = true;
      for (int d = t; d < op.ndeps; d += n) {  // deps and message deps: same tile, progress words
        const DevDep dd = a.deps[op.dep_begin + d];
        ok = ok && wait_geq(a.prog + static_cast<int64_t>(dd.tbi) * ntiles + tile, tag | static_cast<uint64_t>(dd.step + 1), false, c, 1);
      }
      if (!unit_and(ok, uw, bar_id, n)) return;
      const bool in_d = (op.direct & kInDirect) != 0, in_p = (op.direct & kInPull) != 0;
      const bool out_d = (op.direct & kOutDirect) != 0;
      char* src = mine[op.src_buf] + op.src_off * chunk_bytes + t0_bytes;
      char* dst = mine[op.dst_buf] + op.dst_off * chunk_bytes + t0_bytes;
      const char* srcr = mine[op.src_rbuf] + op.src_off * chunk_bytes + t0_bytes;
      const char* dstr = mine[op.dst_rbuf] + op.dst_off * chunk_bytes + t0_bytes;
      const char* in = in_p ? rpeer[op.in_buf] + op.in_off * chunk_bytes + t0_bytes : nullptr;
      char* out = out_d ? peer[op.dst_buf] + op.dst_off * chunk_bytes + t0_bytes : nullptr;
      transfer<R>(op, in_d, src, dst, srcr, dstr, in, chunk_bytes, out, chunk_bytes, tbytes, chunk_bytes, a.tma_ops, tma, t, n, uw,
                  bar_id, a.tma_min);
      if (!unit_and(true, uw, bar_id, n)) return;
      if (t == 0 && (op.has_dep || (op.direct & kPubSem))) {
        fence_acq_rel(false);
        st_relaxed(a.prog + static_cast<int64_t>(tbi) * ntiles + tile, tag | static_cast<uint64_t>(s + 1), false);
      }
    }
    unit_sync(uw, bar_id, n);  // s_item is rewritten by thread 0 next
  }
}

template <class R, int P>
__global__ void __launch_bounds__(kThreads, GC3_MINBLOCKS) interp(const __grid_constant__ LaunchArgs a) {
  // every rank's buffers of this launch, staged in shared memory once: ops index them by rank slot
  // and buffer id (a dynamically indexed kernel parameter would be copied to local memory)
  __shared__ char* s_bufs[kMaxLocalRanks * kBufs];
  __shared__ uint64_t s_epoch;
  stage_bufs(a, s_bufs);
  if (threadIdx.x == kThreads - 1) s_epoch = launch_epoch(a.epoch_ptr, a.epoch_ctr, a.epoch);
  __syncthreads();
  const int uw = a.unit_warps;
  const int n = uw * 32;                         // threads per unit
  const int uib = threadIdx.x / n;               // unit in this block
  const int t = threadIdx.x - uib * n;           // thread in unit
  const int unit = blockIdx.x * (kThreads / n) + uib;
  const int L0 = a.lanes;  // base lanes; thread block i runs L0 x mult_i lanes
  if (unit >= a.weight * L0) return;  // a whole unit leaves together
  const int bar_id = 1 + uib;
  // TMA staging: a.tma_stages x a.stage_bytes of dynamic shared memory per unit, one mbarrier each
  extern __shared__ __align__(128) char s_stage[];
  __shared__ uint64_t s_bar[kThreads / 32][kMaxStages];
  __shared__ uint32_t s_seq[kThreads / 32];
  Tma tma{s_stage + static_cast<size_t>(uib) * a.tma_stages * a.stage_bytes, a.stage_bytes, s_bar[uib], a.tma_stages, &s_seq[uib], 0,
          (a.l2hint & 2) ? l2_evict_first_policy() : 0};
  const uint64_t pol_last = l2_evict_last_policy();
  if (t == 0) s_seq[uib] = 0;
  if (t == 0 && a.tma_stages > 0) {
    for (int s = 0; s < a.tma_stages; ++s) mbar_init(&s_bar[uib][s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // unit -> thread block: thread block i owns units [L0 * unit_base_i, L0 * (unit_base_i + mult_i))
  // (uniform launches run every thread block on the base lanes)
  int tbi = 0;
  if (a.uniform) {
    tbi = unit / L0;
  } else {
    for (int lo = 0, hi = a.ntbs - 1; lo < hi;) {
      const int mid = (lo + hi + 1) / 2;
      if (a.tbs[mid].unit_base * L0 <= unit) lo = mid;
      else hi = mid - 1;
      tbi = lo;
    }
  }
  const DevTb tb = a.tbs[tbi];
  const int lanes = a.uniform ? L0 : L0 * tb.mult;
  const int lane = a.uniform ? unit - tbi * L0 : unit - tb.unit_base * L0;
  // scope per thread block: .sys fences and flags only where a connection reaches another GPU
  const bool sys = a.sys_scope != 0 && tb.sys != 0;
  const int tma_ops = sys ? (a.tma_ops & a.tma_sys_ops) : a.tma_ops;
  const bool has_in = tb.chan_in >= 0, has_out = tb.chan_out >= 0;
  const int64_t chunk_elems = a.chunk_elems, tile_elems = a.tile_elems, ntiles = a.ntiles;
  const int64_t chunk_bytes = chunk_elems * R::kEsize;
  const uint64_t slots = static_cast<uint64_t>(a.slots);
  const uint64_t epoch = s_epoch;
  char* const* const mine = s_bufs + kBufs * tb.rank_slot;                            // this rank's buffers
  char* const* const peer = s_bufs + kBufs * (tb.peer_slot >= 0 ? tb.peer_slot : 0);  // send peer's (direct)
  char* const* const rpeer = s_bufs + kBufs * (tb.recv_slot >= 0 ? tb.recv_slot : 0); // receive peer's (pull)
  const DevChan* const cin = has_in ? a.chans + tb.chan_in + lane : nullptr;
  const DevChan* const cout = has_out ? a.chans + tb.chan_out + lane : nullptr;
  uint64_t rcvd = has_in ? *cin->mine : 0;
  uint64_t sent = has_out ? *cout->mine : 0;
  uint64_t* const sems = a.sems;
  const DevOp* const ops = a.ops + tb.op_begin;
  // the op list is re-read every tile: bring it into L1 once, while the first waits are pending
  for (int i = t; i * 128 < tb.nops * static_cast<int>(sizeof(DevOp)); i += n)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const char*>(ops) + i * 128));
  Ctx c{a.abort_flag, a.err_info, a.timeout_ns, tb.rank_slot, tbi, 0, 0};
  uint64_t* const trace = a.trace;
  const int trace_ops = a.trace_ops;
  auto stamp = [&](int qq, int k) {
    if (trace && qq < trace_ops) trace[(static_cast<int64_t>(unit) * trace_ops + qq) * 4 + k] = globaltimer();
  };

  // Execution order inside the lane: groups of G tiles, op-major within a group (op s of every tile
  // of the group, then op s+1). Tiles are position-independent instances of the program, and every
  // thread block uses the same order, so the k-th send still meets the k-th receive on each
  // connection; a group lets the lane's tiles pipeline through multi-hop chains (the planner checks
  // the order is deadlock-free at this FIFO depth). G = 1 is the paper's tile-major loop.
  const int nops = tb.nops;
  const int64_t my_tiles = ntiles > lane ? (ntiles - 1 - lane) / lanes + 1 : 0;
  const int G = a.group > 0 ? a.group : 1;
  int q = 0;  // position in the lane's (tile, op) order; semaphores publish q + 1
  for (int64_t g0 = 0; g0 < my_tiles; g0 += G) {
    const int gsize = static_cast<int>(min(static_cast<int64_t>(G), my_tiles - g0));
    for (int s = 0; s < nops; ++s)
    for (int jj = 0; jj < gsize; ++jj, ++q) {
      const int64_t i_tile = g0 + jj;
      const int64_t tile = lane + i_tile * lanes;
      // tile geometry: n_head small tiles, n_big big tiles, small tiles to the end of the chunk
      const int64_t nhb = a.n_head + a.n_big;
      const int64_t t0 = tile < a.n_head ? tile * a.small_elems
                         : tile < nhb    ? a.n_head * a.small_elems + (tile - a.n_head) * tile_elems
                                         : a.n_head * a.small_elems + a.n_big * tile_elems + (tile - nhb) * a.small_elems;
      const int64_t tlen = tile < a.n_head || tile >= nhb ? a.small_elems : tile_elems;
      const int64_t t0_bytes = t0 * R::kEsize;
      c.tile = tile;
      const DevOp op = ops[s];
      const int64_t tbytes = clip_tile(a.clip_elems, chunk_elems, op.src_off, t0, min(tlen, chunk_elems - t0)) * R::kEsize;
      tma.pol = op.hot ? pol_last : 0;
      const bool recv = is_recv(op.opcode), send = is_send(op.opcode);
      const int tr = op.direct & a.transports;
      const bool in_d = (tr & kInDirect) != 0, out_d = (tr & kOutDirect) != 0;
      const bool in_p = (tr & kInPull) != 0, out_p = (tr & kOutPull) != 0;
      const bool in_fifo = recv && !in_d && !in_p, out_fifo = send && !out_d && !out_p;
      const bool ll_in = P != kProtoSimple && in_fifo, ll_out = P != kProtoSimple && out_fifo;
      c.step = s;
      if (t == 0) stamp(q, 0);
      // (1) preconditions, polled in parallel
      bool ok = true;
      if (t == 0 && out_fifo) ok = wait_geq(cout->tail, sent + 1 > slots ? sent + 1 - slots : 0, sys, c, 2);
      // direct / pulled receives wait on their sender's semaphore (the trailing message dep)
      if (t == 1 && recv && !ll_in && !(tr & kMsgDep)) ok = wait_geq(cin->head, rcvd + 1, sys, c, 3);
      const int ndeps = op.ndeps - ((tr & kMsgDep) ? 0 : op.nmsg);
      for (int d = t - 2; d >= 0 && d < ndeps; d += n - 2) {
        const DevDep dd = a.deps[op.dep_begin + d];
        // the depended-on thread block may run a different lane count: find the lane that owns this
        // tile there and the tile's position in that lane's order
        const int ld_lanes = a.uniform ? L0 : L0 * dd.mult;
        const int dl = static_cast<int>(tile % ld_lanes);
        const int64_t di = tile / ld_lanes;
        const int64_t dn = (ntiles - 1 - dl) / ld_lanes + 1;
        const int64_t dg0 = di / G * G;
        const int64_t dgs = min(static_cast<int64_t>(G), dn - dg0);
        const uint64_t target = (epoch << 32) | static_cast<uint64_t>(dg0 * dd.nops + static_cast<int64_t>(dd.step) * dgs + (di - dg0) + 1);
        ok = ok && wait_geq(sems + dd.sem + dl, target, false, c, 1);
      }
      if (!unit_and(ok, uw, bar_id, n)) return;
      if (t == 0) stamp(q, 1);

      // (2) the transfer, with the reduction fused in. The incoming message is read from `in`
      // (FIFO slot, or the sender's span when pulled; segment j at + j * in_stride) unless it is
      // already in place; the outgoing one is written to `out` (FIFO slot, or the receiver's span
      // when direct) unless it is pulled from this rank's span.
      char* src = mine[op.src_buf] + op.src_off * chunk_bytes + t0_bytes;
      char* dst = mine[op.dst_buf] + op.dst_off * chunk_bytes + t0_bytes;
      // where the spans are read from: the caller's const buffer for first reads of an in-place IR
      const char* srcr = mine[op.src_rbuf] + op.src_off * chunk_bytes + t0_bytes;
      const char* dstr = mine[op.dst_rbuf] + op.dst_off * chunk_bytes + t0_bytes;
      const char* in = nullptr;
      int64_t in_stride = tbytes;
      if (in_fifo) in = cin->fifo[P] + static_cast<int64_t>(rcvd % slots) * cin->slot_bytes[P];
      if (in_p) {
        in = rpeer[op.in_buf] + op.in_off * chunk_bytes + t0_bytes;
        in_stride = chunk_bytes;
      }
      char* out = nullptr;
      int64_t out_stride = tbytes;
      if (out_fifo) out = cout->fifo[P] + static_cast<int64_t>(sent % slots) * cout->slot_bytes[P];
      if (out_d) {
        out = peer[op.dst_buf] + op.dst_off * chunk_bytes + t0_bytes;
        out_stride = chunk_bytes;
      }
      if ((ll_in || ll_out) && P == kProtoLL128) {
        ok = ll128_op<R>(op.opcode, op.count, src, srcr, dst, chunk_bytes, tbytes, ll_in ? reinterpret_cast<const uint4*>(in) : nullptr,
                         ll_out ? reinterpret_cast<uint4*>(out) : nullptr, rcvd + 1, sent + 1, sys, c, t, n);
      } else if (ll_in || ll_out) {
        ok = ll_op<R>(op.opcode, op.count, src, srcr, dst, chunk_bytes, tbytes, ll_in ? reinterpret_cast<const uint4*>(in) : nullptr,
                      in_p ? in : nullptr, ll_out ? reinterpret_cast<uint4*>(out) : nullptr, out_d ? out : nullptr,
                      static_cast<uint32_t>(rcvd + 1), static_cast<uint32_t>(sent + 1), sys, c, t, n);
      } else {
        transfer<R>(op, in_d, src, dst, srcr, dstr, in, in_stride, out, out_stride, tbytes, chunk_bytes, tma_ops, tma, t, n, uw,
                    bar_id, a.tma_min);
      }
      if (t == 0) stamp(q, 2);
      if (!unit_and(ok, uw, bar_id, n)) return;
      if (a.discard && in_fifo && !ll_in) {
        // the consumed slot is dead until the sender refills it: drop its lines from L2 so they are
        // never written back to HBM (the FIFO round trip stays on chip when the consumer is prompt)
        const int64_t used = static_cast<int64_t>(op.count) * tbytes;
        for (int64_t off = static_cast<int64_t>(t) * 128; off + 128 <= used; off += static_cast<int64_t>(n) * 128)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(in + off) : "memory");
        unit_sync(uw, bar_id, n);
      }

      // (3) publish: slot posted / slot freed / semaphore
      if (t == 0) {
        // one scoped fence orders the unit's data (gathered by the barrier above) before all
        // three flag stores: a release pattern per flag without a fence per store. An LL receive
        // returns its slot without one: its loads have returned (their data was used above) and
        // it stored nothing another party reads through this flag.
        // connections without FIFO messages keep no counters
        const bool pub_head = send && !ll_out && !(tr & kNoCtrOut), pub_tail = recv && !(tr & kNoCtrIn);
        const bool pub_sem = op.has_dep || (tr & kPubSem);
        if (pub_head || (pub_tail && !ll_in) || pub_sem) fence_acq_rel(sys);
        if (pub_head) st_relaxed(cout->head, sent + 1, sys);
        if (pub_tail) st_relaxed(cin->tail, rcvd + 1, sys);
        if (pub_sem) st_relaxed(sems + tb.sem + lane, (epoch << 32) | static_cast<uint64_t>(q + 1), false);
        stamp(q, 3);
      }
      if (send && !(tr & kNoCtrOut)) ++sent;
      if (recv && !(tr & kNoCtrIn)) ++rcvd;
    }
  }
  if (t == 0) {  // persistent FIFO counters for the next launch
    if (has_in) *cin->mine = rcvd;
    if (has_out) *cout->mine = sent;
  }
}

// Work-queue entry point (copy-only programs; see interp_wq). A separate kernel, so the static-lane
// interpreter's register allocation is unaffected.
template <class R>
__global__ void __launch_bounds__(kThreads, GC3_MINBLOCKS) interp_wq_kernel(const __grid_constant__ LaunchArgs a) {
  __shared__ char* s_bufs[kMaxLocalRanks * kBufs];
  __shared__ uint64_t s_epoch;
  stage_bufs(a, s_bufs);
  if (threadIdx.x == kThreads - 1) s_epoch = launch_epoch(a.epoch_ptr, a.epoch_ctr, a.epoch);
  __syncthreads();
  const int uw = a.unit_warps;
  const int n = uw * 32;
  const int uib = threadIdx.x / n;
  const int t = threadIdx.x - uib * n;
  const int bar_id = 1 + uib;
  extern __shared__ __align__(128) char s_stage[];
  __shared__ uint64_t s_bar[kThreads / 32][kMaxStages];
  __shared__ uint32_t s_seq[kThreads / 32];
  Tma tma{s_stage + static_cast<size_t>(uib) * a.tma_stages * a.stage_bytes, a.stage_bytes, s_bar[uib], a.tma_stages, &s_seq[uib], 0,
          0};  // (evict_first loads measured 2% slower on the AllToAll family)
  const uint64_t pol_last = l2_evict_last_policy();
  if (t == 0) s_seq[uib] = 0;
  if (t == 0 && a.tma_stages > 0) {
    for (int s = 0; s < a.tma_stages; ++s) mbar_init(&s_bar[uib][s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unit_sync(uw, bar_id, n);
  const WqArgs w{a.tbs, a.ops, a.deps, a.wq_next, a.wq_order, a.prog, a.abort_flag, a.err_info, a.timeout_ns,
                 a.chunk_elems, a.tile_elems, a.ntiles, s_epoch, a.ntbs, a.tma_ops, a.tma_min};
  interp_wq<R>(w, s_bufs, tma, pol_last, t, n, uw, uib, bar_id);
}

// ------------------------------------------------------------------ dataflow execution
// Programs whose ranks all run in this launch (Simple protocol) can execute as a dataflow graph:
// a work item is (node, tile), a node being one op of one thread block, and it is claimed only when
// every predecessor of the node in the happens-before graph (the previous op of its thread block,
// its declared deps -- PAPER.md:424, 431-433 -- and the sender of its message) has finished that
// tile. Units never block on a dependency: whatever is ready is what runs, so chains of dependent
// hops (ring / hierarchical AllReduce, ReduceScatter, AllGather) pipeline across tiles without idle
// units, and a producer's output is consumed while it is still in L2.
// Tiles are position-disjoint instances of the program (every op maps byte x of a chunk to byte x
// of a chunk), so the per-tile graphs are independent and any linear extension of each is a valid
// execution. Messages are direct, pulled (as in the static interpreter) or mailed: written by the
// sender into a per-message mailbox span and read from there by the receiver.
// Scheduling: a unit that completes an item's last predecessor runs that item next itself (its
// continuation: the data it just produced is still in L2); further items it makes ready go to a
// ready queue. A unit without a continuation takes the next root item (nodes without predecessors,
// tile-major), else claims the next queue position (atomicAdd: positions are filled in push order)
// and waits until a unit fills it or every item has run. Only ready items are ever pushed and a
// running item never waits, so some claimed position is always filled while items remain: no
// deadlock. Predecessor counters and queue slots are reset by their consumer, so the tables are
// zero at every launch without a memset (only the four counters are).
__device__ __forceinline__ int32_t ld_relaxed32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_acquire32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed32(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// one acq_rel read-modify-write: releases this unit's data (gathered by the barrier before it) and,
// for the last predecessor to arrive, acquires every earlier predecessor's release (their RMWs
// extend one release sequence on the counter) — a fence, an atomic and a second fence before
__device__ __forceinline__ int32_t atom_add_acq_rel32(int32_t* p, int32_t v) {
  int32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release32(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <class R>
__global__ void __launch_bounds__(kThreads, GC3_MINBLOCKS) interp_df_kernel(const __grid_constant__ LaunchArgs a) {
  __shared__ char* s_bufs[kMaxLocalRanks * kBufs];
  stage_bufs(a, s_bufs);
  __syncthreads();
  const int uw = a.unit_warps;
  const int n = uw * 32;
  const int uib = threadIdx.x / n;
  const int t = threadIdx.x - uib * n;
  const int bar_id = 1 + uib;
  extern __shared__ __align__(128) char s_stage[];
  __shared__ uint64_t s_bar[kThreads / 32][kMaxStages];
  __shared__ uint32_t s_seq[kThreads / 32];
  __shared__ int64_t s_item[kThreads / 32];
  Tma tma{s_stage + static_cast<size_t>(uib) * a.tma_stages * a.stage_bytes, a.stage_bytes, s_bar[uib], a.tma_stages, &s_seq[uib], 0,
          (a.l2hint & 2) ? l2_evict_first_policy() : 0};
  const uint64_t pol_last = l2_evict_last_policy();
  if (t == 0) s_seq[uib] = 0;
  if (t == 0 && a.tma_stages > 0) {
    for (int s = 0; s < a.tma_stages; ++s) mbar_init(&s_bar[uib][s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unit_sync(uw, bar_id, n);
  const int64_t chunk_elems = a.chunk_elems, tile_elems = a.tile_elems, ntiles = a.ntiles;
  const int64_t chunk_bytes = chunk_elems * R::kEsize;
  const int64_t nn = a.df_n;
  const int64_t total = nn * ntiles;
  const int64_t nroot_items = static_cast<int64_t>(a.df_nroots) * ntiles;
  uint64_t* const trace = a.trace;
  // counters (zeroed before the launch), one 128-byte line each: root items claimed, queue pushes,
  // queue pops, items finished
  int32_t* const roots_ctr = a.df_ctr;
  int32_t* const push_ctr = a.df_ctr + 32;
  int32_t* const pop_ctr = a.df_ctr + 64;
  int32_t* const done_ctr = a.df_ctr + 96;
  __shared__ int64_t s_cont[kThreads / 32];
  int64_t cont = -1;  // (thread 0) the ready successor this unit runs next
  for (;;) {
    if (t == 0) {
      const uint64_t t_claim = trace ? globaltimer() : 0;
      int64_t item = cont;
      cont = -1;
      // work, in this order: a continuation (depth first: the producer's data is still in L2), the
      // next root item (tile-major), the next position of the ready queue (waited on until a unit
      // fills it; positions are taken with atomicAdd, never retried)
      if (item < 0) {
        // tiles in flight are bounded by df_window (0: unbounded): a root of tile t starts only
        // once the finished items amount to tile t - window's worth, so producers' spans are still
        // in L2 when their consumers run. Finished items only grow, and with no item running every
        // older tile's remaining items are ready, so the window never blocks the last work.
        const int32_t r0 = ld_relaxed32(roots_ctr);
        const bool open = r0 < nroot_items &&
                          (a.df_window <= 0 || r0 / a.df_nroots < a.df_window + ld_relaxed32(done_ctr) / nn);
        if (open) {
          const int64_t idx = atomicAdd(roots_ctr, 1);
          if (idx < nroot_items) item = (idx / a.df_nroots) * nn + a.df_roots[idx % a.df_nroots];
        }
      }
      if (item < 0) {
        const int32_t q = atomicAdd(pop_ctr, 1);
        int32_t* slot = a.df_q + q;
        Ctx c{a.abort_flag, a.err_info, a.timeout_ns, 0, -1, 0, q};
        const uint64_t start = globaltimer();
        for (int it = 0;; ++it) {
          const int32_t v = ld_relaxed32(slot);
          if (v != 0) {
            ld_acquire32(slot);  // acquire: the producers' data (released before the push) is visible
            st_relaxed32(slot, 0);
            item = v - 1;
            break;
          }
          if ((it & 15) == 15) {
            if (ld_relaxed32(done_ctr) >= total) break;  // every item has run: this position stays empty
            if (*reinterpret_cast<volatile int*>(a.abort_flag)) break;
            if (c.timeout_ns && globaltimer() - start > c.timeout_ns) {
              raise_timeout(c, 5);
              break;
            }
          }
        }
      }
      if (trace && item >= 0) {
        trace[item * 4 + 0] = t_claim;
        trace[item * 4 + 1] = globaltimer();
      }
      s_item[uib] = item;
      s_cont[uib] = -1;
    }
    unit_sync(uw, bar_id, n);
    const int64_t item = s_item[uib];
    if (item < 0) return;
    const int64_t tile = item / nn;
    const int u = static_cast<int>(item - tile * nn);
    const DfNode nd = a.df_nodes[u];  // one 64-byte line: op, transports, peers, successors
    const DevOp& op = nd.op;
    char* const* const mine = s_bufs + kBufs * nd.rank_slot;
    char* const* const peer = s_bufs + kBufs * (nd.peer_slot >= 0 ? nd.peer_slot : 0);
    char* const* const rpeer = s_bufs + kBufs * (nd.recv_slot >= 0 ? nd.recv_slot : 0);
    const int64_t t0 = tile * tile_elems;
    const int64_t tbytes = clip_tile(a.clip_elems, chunk_elems, op.src_off, t0, min(tile_elems, chunk_elems - t0)) * R::kEsize;
    const int64_t t0_bytes = t0 * R::kEsize;
    tma.pol = op.hot ? pol_last : 0;
    const bool in_d = (op.direct & kInDirect) != 0, in_p = (op.direct & kInPull) != 0;
    const bool out_d = (op.direct & kOutDirect) != 0;
    char* src = mine[op.src_buf] + op.src_off * chunk_bytes + t0_bytes;
    char* dst = mine[op.dst_buf] + op.dst_off * chunk_bytes + t0_bytes;
    const char* srcr = mine[op.src_rbuf] + op.src_off * chunk_bytes + t0_bytes;
    const char* dstr = mine[op.dst_rbuf] + op.dst_off * chunk_bytes + t0_bytes;
    const char* in = nd.in_mail >= 0 ? a.mail + nd.in_mail * chunk_bytes + t0_bytes
                     : in_p          ? rpeer[op.in_buf] + op.in_off * chunk_bytes + t0_bytes
                                     : nullptr;
    char* out = nd.out_mail >= 0 ? a.mail + nd.out_mail * chunk_bytes + t0_bytes
                : out_d          ? peer[op.dst_buf] + op.dst_off * chunk_bytes + t0_bytes
                                 : nullptr;
    transfer<R>(op, in_d, src, dst, srcr, dstr, in, chunk_bytes, out, chunk_bytes, tbytes, chunk_bytes, a.tma_ops, tma, t, n, uw, bar_id,
                a.tma_min);
    unit_sync(uw, bar_id, n);
    if (trace && t == 0) trace[item * 4 + 2] = globaltimer();
    if (a.discard && nd.in_mail >= 0 && ((reinterpret_cast<uintptr_t>(in) | static_cast<uintptr_t>(chunk_bytes)) & 127) == 0) {
      // the mailbox span is dead once read: drop its (whole, 128-byte aligned) lines from L2 so
      // they are never written back
      for (int j = 0; j < op.count; ++j)
        for (int64_t off = static_cast<int64_t>(t) * 128; off + 128 <= tbytes; off += static_cast<int64_t>(n) * 128)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(in + j * chunk_bytes + off) : "memory");
    }
    // publish, one successor per thread: release the unit's data (gathered by the barrier above),
    // count the predecessor in; the last one makes the item ready. Successors 0..31 are counted by
    // warp 0 and the lowest-index ready one becomes this unit's continuation (the runtime lists
    // message receivers first: they read what this item just produced, still in L2); every other
    // ready item goes to the queue
    auto count_in = [&](int k) -> int64_t {
      const DfSucc sc = a.df_succ[nd.succ + k];
      // a successor with this item as its only predecessor is ready now: no counter (its push is a
      // release store; a continuation stays on this unit)
      if (sc.indeg == 1) return tile * nn + sc.node;
      int32_t* cnt = a.df_cnt + tile * nn + sc.node;
      if (a.df_policy & 2) {
        fence_acq_rel(false);
        if (atomicAdd(cnt, 1) + 1 != sc.indeg) return -1;
        __threadfence();  // acquire the other predecessors' releases (read through the counter)
      } else if (atom_add_acq_rel32(cnt, 1) + 1 != sc.indeg) {
        return -1;
      }
      return tile * nn + sc.node;  // its counter (df_cnt[ready]) is reset after the push
    };
    // a ready item's counter is reset for the next launch only after its push: the push's release
    // would otherwise wait for the reset store to be acknowledged
    auto push = [&](int64_t ready) {
      const int32_t pos = atomicAdd(push_ctr, 1);
      st_release32(a.df_q + pos, static_cast<int32_t>(ready) + 1);
      a.df_cnt[ready] = 0;
    };
    if (t < 32) {
      const int64_t ready = t < nd.nsucc ? count_in(t) : -1;
      const unsigned ready_mask = __ballot_sync(0xffffffffu, ready >= 0);
      if (ready >= 0) {
        if ((a.df_policy & 1) && t == __ffs(ready_mask) - 1) {
          s_cont[uib] = ready;
          a.df_cnt[ready] = 0;
        } else {
          push(ready);
        }
      }
    }
    for (int k = t < 32 ? t + n : t; k < nd.nsucc; k += n) {
      const int64_t ready = count_in(k);
      if (ready >= 0) push(ready);
    }
    unit_sync(uw, bar_id, n);
    if (t == 0) {
      cont = s_cont[uib];
      atomicAdd(done_ctr, 1);
    }
    if (trace && t == 0) trace[item * 4 + 3] = globaltimer();
  }
}

}  // namespace dev

}  // namespace gc3
