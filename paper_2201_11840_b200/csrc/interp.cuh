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
#define GC3_MINBLOCKS 2
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
__device__ __forceinline__ uint4 ld_volatile_line(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_line(uint4* p, uint4 v) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
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
template <typename T, int OP>
struct RedInt {
  static constexpr int kEsize = sizeof(T);
  static constexpr bool kReduce = true;
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
template <typename F, int OP>
struct RedFloat {
  static constexpr int kEsize = sizeof(F);
  static constexpr bool kReduce = true;
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
  __device__ static void elem(const char* a, const char*, char* o) { *o = *a; }
  template <typename V>
  __device__ static V vec(V a, V) {
    return a;
  }
};

// ------------------------------------------------------------------ data movers
// Executed by the data warps only: thread `t` of `n` data threads.
// out0 (and out1 if non-null) = RED ? R(in0, in1) : in0, over nbytes. All pointers 16B aligned
// takes the 128-bit path; the ragged remainder (and misaligned segments) go element-wise.
constexpr int kDataThreads = kThreads - 32;

template <class R, bool RED, bool TWO>
__device__ __forceinline__ void move_vec(const uint4* a, const uint4* b, uint4* o0, uint4* o1, int64_t nvec, int t) {
  constexpr int U = R::kReduce ? GC3_UNROLL : GC3_UNROLL_COPY;  // 128-bit loads in flight per thread
  constexpr int N = kDataThreads;
  int64_t i = t;
  for (; i + (U - 1) * N < nvec; i += U * N) {
    uint4 x[U], y[U];
#pragma unroll
    for (int k = 0; k < U; ++k) x[k] = ld_cg(a + i + k * N);
    if (RED) {
#pragma unroll
      for (int k = 0; k < U; ++k) y[k] = ld_cg(b + i + k * N);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint4 v = RED ? R::template vec<uint4>(x[k], y[k]) : x[k];
      st_vec(o0 + i + k * N, v);
      if (TWO) st_vec(o1 + i + k * N, v);
    }
  }
  for (; i < nvec; i += N) {
    const uint4 x = ld_cg(a + i);
    const uint4 v = RED ? R::template vec<uint4>(x, ld_cg(b + i)) : x;
    st_vec(o0 + i, v);
    if (TWO) st_vec(o1 + i, v);
  }
}

template <class R>
__device__ __forceinline__ void move_elems(const char* a, const char* b, char* o0, char* o1, int64_t nbytes, bool red, int t) {
  constexpr int E = R::kEsize;
  for (int64_t i = t * static_cast<int64_t>(E); i < nbytes; i += static_cast<int64_t>(kDataThreads) * E) {
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
__device__ void move(const char* a, const char* b, char* o0, char* o1, int64_t nbytes, int t) {
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
      if (o1) move_vec<R, true, true>(va, vb, v0, v1, nvec, t);
      else move_vec<R, true, false>(va, vb, v0, v1, nvec, t);
    } else {
      if (o1) move_vec<R, false, true>(va, vb, v0, v1, nvec, t);
      else move_vec<R, false, false>(va, vb, v0, v1, nvec, t);
    }
    done = nvec << 4;
  }
  if (done < nbytes)
    move_elems<R>(a + done, b ? b + done : nullptr, o0 + done, o1 ? o1 + done : nullptr, nbytes - done, red, t);
}

// ------------------------------------------------------------------ watchdog
// Everything here is passed by value: taking the address of a kernel parameter would force the
// whole LaunchArgs into local memory.
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

__device__ __forceinline__ bool is_recv(int op) {
  return op == kOpRecv || op == kOpRrc || op == kOpRcs || op == kOpRrcs || op == kOpRrs;
}
__device__ __forceinline__ bool is_send(int op) { return op == kOpSend || op == kOpRcs || op == kOpRrcs || op == kOpRrs; }

// ------------------------------------------------------------------ LL op body (data warps)
// Lines of the incoming/outgoing message are distributed over the data threads; every thread
// polls the flags of its own lines only. inl == nullptr: the incoming message is in place (direct)
// or absent; outl == nullptr: the outgoing message goes to outd (direct, plain stores) or is absent.
template <class R>
__device__ void ll_op(int opcode, int count, char* src0, char* dst0, int64_t chunk_bytes, int64_t tbytes, const uint4* inl,
                      uint4* outl, char* outd, uint32_t in_flag, uint32_t out_flag, const Ctx& c, int t) {
  const int64_t lines_per_seg = tbytes >> 3;
  const int64_t nlines = lines_per_seg * count;
  const bool send = is_send(opcode);
  for (int64_t k = t; k < nlines; k += kDataThreads) {
    const int j = static_cast<int>(k / lines_per_seg);
    const int64_t off = ((k - j * lines_per_seg) << 3) + j * chunk_bytes;
    char* src = src0 + off;
    char* dst = dst0 + off;
    uint2 msg = make_uint2(0, 0);
    if (inl) {
      uint4 l = ld_volatile_line(inl + k);
      if (l.y != in_flag || l.w != in_flag) {
        const uint64_t start = globaltimer();
        for (int n = 0;; ++n) {
          l = ld_volatile_line(inl + k);
          if (l.y == in_flag && l.w == in_flag) break;
          if ((n & 255) == 255) {
            if (*reinterpret_cast<volatile int*>(c.abort_flag)) return;  // the control warp exits the launch
            if (c.timeout_ns && globaltimer() - start > c.timeout_ns) {
              raise_timeout(c, 4);
              return;
            }
          }
        }
      }
      msg = make_uint2(l.x, l.z);
    }
    uint2 v;
    switch (opcode) {
      case kOpSend: v = ld_cg8(src); break;
      case kOpRecv:
        if (inl) st_vec8(dst, msg);
        continue;
      case kOpRrc: st_vec8(dst, R::template vec<uint2>(ld_cg8(src), msg)); continue;
      case kOpRcs:
        if (inl) {
          v = msg;
          st_vec8(src, v);
        } else {
          v = ld_cg8(src);  // direct: the message is already in the local span
        }
        break;
      case kOpRrcs: v = R::template vec<uint2>(ld_cg8(src), msg); st_vec8(src, v); break;
      case kOpRrs: v = R::template vec<uint2>(ld_cg8(src), msg); break;
      default: continue;
    }
    if (send) {
      if (outl) st_volatile_line(outl + k, make_uint4(v.x, out_flag, v.y, out_flag));
      else st_vec8(outd + off, v);
    }
  }
}

// ------------------------------------------------------------------ the interpreter
// Warp-specialised execution of one (IR thread block, lane) per CUDA block:
//   * warp 0 (control) walks the (tile, op) sequence: it waits for each op's preconditions
//     (deps, FIFO credit, posted message), describes the op's data movement in a shared-memory
//     descriptor, and publishes the op (FIFO head / tail, semaphore) once the data warps are done;
//   * warps 1.. (data) execute descriptors: vectorised moves with the reduction fused in, or LL
//     line traffic.
// Descriptors are double-buffered. While the data warps move op k, the control warp already polls
// op k+1's preconditions, but it publishes op k as soon as op k's data is done (never after
// blocking on op k+1, which could depend on op k's publication). A named barrier hands a
// descriptor to the data warps; a shared counter reports completion. Ops are separated: the data
// warps start a descriptor only after the previous one completed block-wide.
struct Desc {
  const char* a;
  const char* b;
  char* o0;
  char* o1;
  int64_t sa, sb, s0, s1;  // per-segment strides
  int64_t nbytes;          // per segment
  // LL
  char* src;
  char* dst;
  const uint4* inl;
  uint4* outl;
  char* outd;
  int64_t chunk_bytes;
  uint32_t in_flag, out_flag;
  int32_t count;
  int32_t opcode;
  int32_t kind;  // 1 vector move, 2 LL, 3 exit
  int32_t step;
  int64_t tile;
};

__device__ __forceinline__ void bar_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kThreads) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kThreads) : "memory"); }

template <class R, bool LL>
__global__ void __launch_bounds__(kThreads, GC3_MINBLOCKS) interp(const LaunchArgs a) {
  __shared__ Desc s_desc[2];
  __shared__ unsigned s_done[2];
  const int lanes = a.lanes;
  const int lane = blockIdx.x % lanes;
  const int tbi = blockIdx.x / lanes;
  if (threadIdx.x < 2) s_done[threadIdx.x] = 0;
  __syncthreads();

  if (threadIdx.x >= 32) {  // ---------------- data warps
    const int t = threadIdx.x - 32;
    const Ctx c{a.abort_flag, a.err_info, a.timeout_ns, 0, tbi, 0, 0};
    for (int n = 0;; ++n) {
      bar_sync(1 + (n & 1));
      const Desc& d = s_desc[n & 1];
      const int kind = d.kind;
      if (kind == 3) return;
      if (kind == 2) {
        Ctx cc = c;
        cc.step = d.step;
        cc.tile = d.tile;
        ll_op<R>(d.opcode, d.count, d.src, d.dst, d.chunk_bytes, d.nbytes, d.inl, d.outl, d.outd, d.in_flag, d.out_flag, cc, t);
      } else {
        const char* pa = d.a;
        const char* pb = d.b;
        char* p0 = d.o0;
        char* p1 = d.o1;
        for (int j = 0; j < d.count; ++j) {
          move<R>(pa, pb, p0, p1, d.nbytes, t);
          pa += d.sa;
          if (pb) pb += d.sb;
          if (p0) p0 += d.s0;
          if (p1) p1 += d.s1;
        }
      }
      // release this warp's stores at CTA scope; the control warp's scoped fence is cumulative
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        unsigned prev;
        asm volatile("atom.release.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(prev) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(&s_done[n & 1]))) : "memory");
      }
    }
  }

  // ---------------- control warp
  const int wl = threadIdx.x;
  const DevTb tb = a.tbs[tbi];
  const bool sys = a.sys_scope != 0;
  const bool has_in = tb.chan_in >= 0, has_out = tb.chan_out >= 0;
  const int64_t chunk_elems = a.chunk_elems, tile_elems = a.tile_elems, ntiles = a.ntiles;
  const int64_t chunk_bytes = chunk_elems * R::kEsize;
  const uint64_t slots = static_cast<uint64_t>(a.slots);
  const uint64_t epoch = a.epoch;
  // this rank's buffers and the send peer's (direct writes), selected with constant indices (a
  // dynamically indexed kernel parameter would be copied to local memory)
  char* buf[3] = {nullptr, nullptr, nullptr};
  char* peer[3] = {nullptr, nullptr, nullptr};
#pragma unroll
  for (int i = 0; i < kMaxLocalRanks; ++i) {
    if (i == tb.rank_slot) {
      buf[0] = a.bufs[i][0];
      buf[1] = a.bufs[i][1];
      buf[2] = a.bufs[i][2];
    }
    if (i == tb.peer_slot) {
      peer[0] = a.bufs[i][0];
      peer[1] = a.bufs[i][1];
      peer[2] = a.bufs[i][2];
    }
  }
  DevChan cin{}, cout{};
  if (has_in) cin = a.chans[tb.chan_in + lane];
  if (has_out) cout = a.chans[tb.chan_out + lane];
  uint64_t rcvd = has_in ? *cin.mine : 0;
  uint64_t sent = has_out ? *cout.mine : 0;
  uint64_t* const sems = a.sems;
  uint64_t* const my_sem = sems + tb.sem + lane;
  const DevOp* const ops = a.ops + tb.op_begin;
  const DevDep* const deps = a.deps;
  Ctx c{a.abort_flag, a.err_info, a.timeout_ns, tb.rank_slot, tbi, 0, 0};
  uint64_t* const trace = a.trace;
  const int trace_ops = a.trace_ops;
  auto stamp = [&](int qq, int k) {
    if (trace && qq < trace_ops && wl == 0) trace[(static_cast<int64_t>(blockIdx.x) * trace_ops + qq) * 4 + k] = globaltimer();
  };
  const int nops = tb.nops;
  const int my_tiles = ntiles > lane ? static_cast<int>((ntiles - 1 - lane) / lanes + 1) : 0;
  const int total = my_tiles * nops;

  // one non-blocking poll of op q's preconditions (one flag per lane); true when all hold
  bool pend_send = false, pend_recv = false;  // the in-flight op will advance sent / rcvd
  auto poll = [&](int q) -> bool {
    const int s = q % nops;
    const int64_t it = q / nops;
    const DevOp op = ops[s];
    const bool recv = is_recv(op.opcode), send = is_send(op.opcode);
    const bool in_d = (op.direct & kInDirect) != 0, out_d = (op.direct & kOutDirect) != 0;
    bool ok = true;
    // counters as they will be once the in-flight op is published
    const uint64_t sent_q = sent + (pend_send ? 1 : 0), rcvd_q = rcvd + (pend_recv ? 1 : 0);
    if (wl == 0 && send && !out_d) ok = ld_relaxed(cout.tail, sys) + slots >= sent_q + 1;
    if (wl == 1 && recv && !(LL && !in_d)) ok = ld_relaxed(cin.head, sys) >= rcvd_q + 1;
    for (int d = wl - 2; d >= 0 && d < op.ndeps; d += 30) {
      const DevDep dd = deps[op.dep_begin + d];
      ok = ok && ld_relaxed(sems + dd.sem + lane, false) >= ((epoch << 32) | static_cast<uint64_t>(it * dd.nops + dd.step + 1));
    }
    return __all_sync(0xffffffffu, ok);
  };
  auto aborted = [&]() { return *reinterpret_cast<volatile int*>(a.abort_flag) != 0; };

  int posted = 0;            // descriptors handed to the data warps
  int pending = -1;          // op whose data is in flight (published when done), -1 if none
  bool pending_data = false;
  uint64_t wait_start = 0;
  bool pre_ok = false;
  for (int q = 0; q <= total; ++q) {
    // wait for op q's preconditions while completing op `pending`
    pre_ok = q == total;
    if (!pre_ok) {
      c.step = q % nops;
      c.tile = lane + static_cast<int64_t>(q / nops) * lanes;
      stamp(q, 0);
    }
    wait_start = 0;
    for (int n = 0;; ++n) {
      if (!pre_ok) pre_ok = poll(q);
      if (pending >= 0) {
        const bool done = !pending_data || *reinterpret_cast<volatile unsigned*>(&s_done[(posted - 1) & 1]) == kThreads / 32 - 1;
        if (done) {
          // publish op `pending`: slot posted / slot freed / semaphore
          const int ps = pending % nops;
          const DevOp pop = ops[ps];
          const bool precv = is_recv(pop.opcode), psend = is_send(pop.opcode);
          const bool pin_d = (pop.direct & kInDirect) != 0, pout_d = (pop.direct & kOutDirect) != 0;
          const bool pll_out = LL && psend && !pout_d;
          stamp(pending, 2);
          if (wl == 0) {
            if (pending_data) s_done[(posted - 1) & 1] = 0;
            fence_acq_rel(sys);
            if (psend && !pll_out) st_release(cout.head, sent + 1, sys);
            if (precv) st_release(cin.tail, rcvd + 1, sys);
            if (pop.has_dep)
              st_release(my_sem, (epoch << 32) | static_cast<uint64_t>((pending / nops) * nops + ps + 1), false);
            if (pending + 1 == total) {  // persistent FIFO counters for the next launch
              if (has_in) *cin.mine = rcvd + (precv ? 1 : 0);
              if (has_out) *cout.mine = sent + (psend ? 1 : 0);
            }
          }
          (void)pin_d;
          stamp(pending, 3);
          if (psend) ++sent;
          if (precv) ++rcvd;
          pending = -1;
          pend_send = pend_recv = false;
          __syncwarp();
        }
      }
      if (pre_ok && pending < 0) break;
      if ((n & 63) == 63) {
        if (aborted()) break;
        if (a.timeout_ns) {
          const uint64_t now = globaltimer();
          if (!wait_start) wait_start = now;
          else if (now - wait_start > a.timeout_ns) {
            if (wl == 0) raise_timeout(c, pending >= 0 ? 5 : 1);
            break;
          }
        }
      }
    }
    if (!(pre_ok && pending < 0) || q == total) break;
    fence_acq_rel(sys);  // acquire what the polled flags published
    stamp(q, 1);

    // describe op q's data movement
    const int s = q % nops;
    const int64_t tile = lane + static_cast<int64_t>(q / nops) * lanes;
    const int64_t t0 = tile * tile_elems;
    const int64_t tlen = min(tile_elems, chunk_elems - t0);
    const int64_t tbytes = tlen * R::kEsize;
    const int64_t t0_bytes = t0 * R::kEsize;
    const DevOp op = ops[s];
    const bool recv = is_recv(op.opcode), send = is_send(op.opcode);
    const bool in_d = (op.direct & kInDirect) != 0, out_d = (op.direct & kOutDirect) != 0;
    const bool ll_in = LL && recv && !in_d, ll_out = LL && send && !out_d;
    auto sel = [](int b, char* const* v) { return b == 0 ? v[0] : (b == 1 ? v[1] : v[2]); };
    char* src = sel(op.src_buf, buf) + op.src_off * chunk_bytes + t0_bytes;
    char* dst = sel(op.dst_buf, buf) + op.dst_off * chunk_bytes + t0_bytes;
    char* peer_dst = out_d ? sel(op.dst_buf, peer) + op.dst_off * chunk_bytes + t0_bytes : nullptr;
    const char* in = recv && !in_d ? cin.fifo + static_cast<int64_t>(rcvd % slots) * cin.slot_bytes : nullptr;
    char* out = send && !out_d ? cout.fifo + static_cast<int64_t>(sent % slots) * cout.slot_bytes : nullptr;
    int kind = 1;
    const char *pa = nullptr, *pb = nullptr;
    char *p0 = nullptr, *p1 = nullptr;
    int64_t sa = chunk_bytes, sb = tbytes, s0 = chunk_bytes, s1 = tbytes;
    char* mo = out_d ? peer_dst : out;
    const int64_t smo = out_d ? chunk_bytes : tbytes;
    if (ll_in || ll_out) {
      kind = 2;
    } else {
      switch (op.opcode) {
        case kOpSend: pa = src; p0 = mo; s0 = smo; break;
        case kOpRecv:
          if (in_d) kind = 0;
          else { pa = in; sa = tbytes; p0 = dst; }
          break;
        case kOpCopy: pa = src; p0 = dst; break;
        case kOpReduce: pa = dst; pb = src; sb = chunk_bytes; p0 = dst; break;
        case kOpRrc: pa = src; pb = in; p0 = dst; break;
        case kOpRcs:
          if (in_d) { pa = src; p0 = mo; s0 = smo; }
          else { pa = in; sa = tbytes; p0 = src; p1 = mo; s1 = smo; }
          break;
        case kOpRrcs: pa = src; pb = in; p0 = src; p1 = mo; s1 = smo; break;
        case kOpRrs: pa = src; pb = in; p0 = mo; s0 = smo; break;
        default: kind = 0; break;
      }
      if (tbytes <= 0) kind = 0;
    }
    if (kind != 0) {
      if (wl == 0) {
        Desc& d = s_desc[posted & 1];
        d.a = pa;
        d.b = pb;
        d.o0 = p0;
        d.o1 = p1;
        d.sa = sa;
        d.sb = sb;
        d.s0 = s0;
        d.s1 = s1;
        d.nbytes = tbytes;
        d.src = src;
        d.dst = dst;
        d.inl = ll_in ? reinterpret_cast<const uint4*>(in) : nullptr;
        d.outl = ll_out ? reinterpret_cast<uint4*>(out) : nullptr;
        d.outd = peer_dst;
        d.chunk_bytes = chunk_bytes;
        d.in_flag = static_cast<uint32_t>(rcvd + 1);
        d.out_flag = static_cast<uint32_t>(sent + 1);
        d.count = op.count;
        d.opcode = op.opcode;
        d.kind = kind;
        d.step = s;
        d.tile = tile;
      }
      __syncwarp();
      bar_arrive(1 + (posted & 1));
      ++posted;
    }
    pending = q;
    pend_send = send;
    pend_recv = recv;
    pending_data = kind != 0;
  }
  // release the data warps
  if (wl == 0) s_desc[posted & 1].kind = 3;
  __syncwarp();
  bar_arrive(1 + (posted & 1));
}

}  // namespace dev

}  // namespace gc3
