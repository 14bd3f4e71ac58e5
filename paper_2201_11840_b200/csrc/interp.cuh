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
// out0 (and out1 if non-null) = RED ? R(in0, in1) : in0, over nbytes. All pointers 16B aligned
// takes the 128-bit path; the ragged remainder (and misaligned segments) go element-wise.
template <class R, bool RED, bool TWO>
__device__ __forceinline__ void move_vec(const uint4* a, const uint4* b, uint4* o0, uint4* o1, int64_t nvec) {
  constexpr int U = R::kReduce ? GC3_UNROLL : GC3_UNROLL_COPY;  // 128-bit loads in flight per thread
  int64_t i = threadIdx.x;
  for (; i + (U - 1) * kThreads < nvec; i += U * kThreads) {
    uint4 x[U], y[U];
#pragma unroll
    for (int k = 0; k < U; ++k) x[k] = ld_cg(a + i + k * kThreads);
    if (RED) {
#pragma unroll
      for (int k = 0; k < U; ++k) y[k] = ld_cg(b + i + k * kThreads);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint4 v = RED ? R::template vec<uint4>(x[k], y[k]) : x[k];
      st_vec(o0 + i + k * kThreads, v);
      if (TWO) st_vec(o1 + i + k * kThreads, v);
    }
  }
  for (; i < nvec; i += kThreads) {
    const uint4 x = ld_cg(a + i);
    const uint4 v = RED ? R::template vec<uint4>(x, ld_cg(b + i)) : x;
    st_vec(o0 + i, v);
    if (TWO) st_vec(o1 + i, v);
  }
}

template <class R>
__device__ __forceinline__ void move_elems(const char* a, const char* b, char* o0, char* o1, int64_t nbytes, bool red) {
  constexpr int E = R::kEsize;
  for (int64_t i = threadIdx.x * static_cast<int64_t>(E); i < nbytes; i += static_cast<int64_t>(kThreads) * E) {
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
__device__ void move(const char* a, const char* b, char* o0, char* o1, int64_t nbytes) {
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
      if (o1) move_vec<R, true, true>(va, vb, v0, v1, nvec);
      else move_vec<R, true, false>(va, vb, v0, v1, nvec);
    } else {
      if (o1) move_vec<R, false, true>(va, vb, v0, v1, nvec);
      else move_vec<R, false, false>(va, vb, v0, v1, nvec);
    }
    done = nvec << 4;
  }
  if (done < nbytes)
    move_elems<R>(a + done, b ? b + done : nullptr, o0 + done, o1 ? o1 + done : nullptr, nbytes - done, red);
}

// LL: one 16-byte line carries 8 payload bytes as {d0, flag, d1, flag}.
template <class R>
__device__ __forceinline__ uint2 red8(uint2 x, uint2 y) {
  return R::template vec<uint2>(x, y);
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

// Spins until *p >= target; false if the launch was aborted. Polls with relaxed loads (an acquire
// load would invalidate L1 on every iteration) and acquires once with a fence when satisfied.
__device__ __forceinline__ bool wait_geq(const uint64_t* p, uint64_t target, bool sys, const Ctx& c, int what) {
  if (ld_relaxed(p, sys) >= target) {
    fence_acq_rel(sys);
    return true;
  }
  const uint64_t start = globaltimer();
  for (int n = 0;; ++n) {
    if (ld_relaxed(p, sys) >= target) {
      fence_acq_rel(sys);
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

__device__ __forceinline__ char* pick_buf(int b, char* in, char* out, char* sc) { return b == 0 ? in : (b == 1 ? out : sc); }

// ------------------------------------------------------------------ LL op body
// Lines of the incoming/outgoing message are distributed over threads; every thread polls the
// flags of its own lines only.
// inl == nullptr: the incoming message is in place (direct) or absent; outl == nullptr: the
// outgoing message goes to outd (direct, plain stores) or is absent.
template <class R>
__device__ bool ll_op(const DevOp op, char* src0, char* dst0, int64_t chunk_bytes, int64_t tbytes, const uint4* inl, uint4* outl,
                      char* outd, uint32_t in_flag, uint32_t out_flag, const Ctx& c) {
  const int64_t lines_per_seg = tbytes >> 3;
  const int64_t nlines = lines_per_seg * op.count;
  const bool send = is_send(op.opcode);
  for (int64_t k = threadIdx.x; k < nlines; k += kThreads) {
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
            if (*reinterpret_cast<volatile int*>(c.abort_flag)) return false;
            if (c.timeout_ns && globaltimer() - start > c.timeout_ns) {
              raise_timeout(c, 4);
              return false;
            }
          }
        }
      }
      msg = make_uint2(l.x, l.z);
    }
    uint2 v;
    switch (op.opcode) {
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
  return true;
}

// ------------------------------------------------------------------ the interpreter
// Warp-asynchronous execution of one (IR thread block, lane): every warp walks the same
// (tile, op) sequence and moves its share of each op's bytes; there is no block-wide barrier in
// the op loop. Each warp waits for the op's preconditions itself (deps, FIFO credit, posted
// message), fences its own stores, and arrives on a per-op shared-memory counter; the last warp
// to arrive publishes the op (FIFO head / tail, semaphore). Warps may therefore overlap the loads
// of op k+1 with the stores of op k. Thread->byte mapping is identical for every op, so a warp
// always re-reads what it wrote itself (sequential semantics inside the thread block hold per
// thread). A drift bound keeps warps within kDrift ops of the last published op.
constexpr int kWarps = kThreads / 32;
constexpr int kRing = 16;
constexpr int kDrift = 6;

template <class R, bool LL>
__global__ void __launch_bounds__(kThreads, GC3_MINBLOCKS) interp(const LaunchArgs a) {
  const int lanes = a.lanes;
  const int lane = blockIdx.x % lanes;
  const int tbi = blockIdx.x / lanes;
  const DevTb tb = a.tbs[tbi];
  const bool sys = a.sys_scope != 0;
  const bool has_in = tb.chan_in >= 0, has_out = tb.chan_out >= 0;
  const int64_t chunk_elems = a.chunk_elems, tile_elems = a.tile_elems, ntiles = a.ntiles;
  const int64_t chunk_bytes = chunk_elems * R::kEsize;
  const uint64_t slots = static_cast<uint64_t>(a.slots);
  const uint64_t epoch = a.epoch;
  const int wid = threadIdx.x >> 5, wl = threadIdx.x & 31;
  // this block's rank buffers: select with constant indices (no dynamic param-space indexing)
  char *b_in = nullptr, *b_out = nullptr, *b_sc = nullptr;
  char *p_in = nullptr, *p_out = nullptr, *p_sc = nullptr;  // send peer's buffers (direct writes)
#pragma unroll
  for (int i = 0; i < kMaxLocalRanks; ++i) {
    if (i == tb.rank_slot) {
      b_in = a.bufs[i][0];
      b_out = a.bufs[i][1];
      b_sc = a.bufs[i][2];
    }
    if (i == tb.peer_slot) {
      p_in = a.bufs[i][0];
      p_out = a.bufs[i][1];
      p_sc = a.bufs[i][2];
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
  __shared__ unsigned s_arrive[kRing];
  __shared__ volatile int s_posted;  // ops published so far
  __shared__ volatile int s_abort;
  if (threadIdx.x < kRing) s_arrive[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    s_posted = 0;
    s_abort = 0;
  }
  __syncthreads();

  // event log (gc3SetConfig "trace"): per op {start, preconditions met, warp 0 data done, published}
  uint64_t* const trace = a.trace;
  const int trace_ops = a.trace_ops;
  auto stamp = [&](int qq, int k) {
    if (trace && qq < trace_ops) trace[(static_cast<int64_t>(blockIdx.x) * trace_ops + qq) * 4 + k] = globaltimer();
  };
  const int my_tiles = ntiles > lane ? static_cast<int>((ntiles - 1 - lane) / lanes + 1) : 0;
  const int total_ops = my_tiles * tb.nops;
  int q = 0;  // op sequence number within this block
  int64_t iter = 0;
  for (int64_t tile = lane; tile < ntiles; tile += lanes, ++iter) {
    const int64_t t0 = tile * tile_elems;
    const int64_t tlen = min(tile_elems, chunk_elems - t0);
    const int64_t tbytes = tlen * R::kEsize;
    const int64_t t0_bytes = t0 * R::kEsize;
    c.tile = tile;
    for (int s = 0; s < tb.nops; ++s, ++q) {
      const DevOp op = ops[s];
      const bool recv = is_recv(op.opcode), send = is_send(op.opcode);
      c.step = s;
      // drift bound (also keeps the arrival ring from wrapping onto an unpublished op)
      if (q - s_posted > kDrift) {
        while (q - s_posted > kDrift) {
          if (s_abort || *reinterpret_cast<volatile int*>(c.abort_flag)) return;
        }
      }
      // (1) preconditions, per warp: deps, a free outgoing slot, a posted message
      if (threadIdx.x == 0) stamp(q, 0);
      bool ok = true;
      for (int d = wl; d < op.ndeps; d += 32) {
        const DevDep dd = deps[op.dep_begin + d];
        const uint64_t target = (epoch << 32) | static_cast<uint64_t>(iter * dd.nops + dd.step + 1);
        ok = ok && wait_geq(sems + dd.sem + lane, target, false, c, 1);
      }
      const bool in_d = (op.direct & kInDirect) != 0, out_d = (op.direct & kOutDirect) != 0;
      const bool ll_in = LL && recv && !in_d, ll_out = LL && send && !out_d;  // LL lines carry the payload
      if (wl == 0 && send && !out_d) ok = wait_geq(cout.tail, sent + 1 > slots ? sent + 1 - slots : 0, sys, c, 2);
      if (wl == 1 && recv && !ll_in) ok = wait_geq(cin.head, rcvd + 1, sys, c, 3);
      if (!__all_sync(0xffffffffu, ok)) {
        s_abort = 1;
        return;
      }
      __syncwarp();  // orders the other lanes' data accesses after lanes 0/1's acquires
      if (threadIdx.x == 0) stamp(q, 1);

      // (2) this warp's share of the transfer, with the reduction fused in
      char* src = pick_buf(op.src_buf, b_in, b_out, b_sc) + op.src_off * chunk_bytes + t0_bytes;
      char* dst = pick_buf(op.dst_buf, b_in, b_out, b_sc) + op.dst_off * chunk_bytes + t0_bytes;
      const int64_t slot_in = static_cast<int64_t>(rcvd % slots) * cin.slot_bytes;
      const int64_t slot_out = static_cast<int64_t>(sent % slots) * cout.slot_bytes;
      // a direct outgoing message lands in the receiver's own span (the send op's dst fields name it,
      // lowering.hpp:71); a direct incoming one is already in this rank's write span
      char* peer_dst = out_d ? pick_buf(op.dst_buf, p_in, p_out, p_sc) + op.dst_off * chunk_bytes + t0_bytes : nullptr;
      if (ll_in || ll_out) {
        const uint4* inl = ll_in ? reinterpret_cast<const uint4*>(cin.fifo + slot_in) : nullptr;
        uint4* outl = ll_out ? reinterpret_cast<uint4*>(cout.fifo + slot_out) : nullptr;
        ok = ll_op<R>(op, src, dst, chunk_bytes, tbytes, inl, outl, peer_dst, static_cast<uint32_t>(rcvd + 1),
                      static_cast<uint32_t>(sent + 1), c);
        if (!__all_sync(0xffffffffu, ok)) {
          s_abort = 1;
          return;
        }
      } else {
        const char* in = recv && !in_d ? cin.fifo + slot_in : nullptr;
        char* out = send && !out_d ? cout.fifo + slot_out : nullptr;
        for (int j = 0; j < op.count; ++j) {
          char* sj = src + j * chunk_bytes;
          char* dj = dst + j * chunk_bytes;
          const char* mi = in ? in + j * tbytes : nullptr;
          char* mo = out_d ? peer_dst + j * chunk_bytes : (out ? out + j * tbytes : nullptr);
          switch (op.opcode) {
            case kOpSend: move<R>(sj, nullptr, mo, nullptr, tbytes); break;
            case kOpRecv:
              if (!in_d) move<R>(mi, nullptr, dj, nullptr, tbytes);
              break;
            case kOpCopy: move<R>(sj, nullptr, dj, nullptr, tbytes); break;
            case kOpReduce: move<R>(dj, sj, dj, nullptr, tbytes); break;
            case kOpRrc: move<R>(sj, mi, dj, nullptr, tbytes); break;
            case kOpRcs:
              if (in_d) move<R>(sj, nullptr, mo, nullptr, tbytes);
              else move<R>(mi, nullptr, sj, mo, tbytes);
              break;
            case kOpRrcs: move<R>(sj, mi, sj, mo, tbytes); break;
            case kOpRrs: move<R>(sj, mi, nullptr, mo, tbytes); break;
            default: break;
          }
        }
      }

      // (3) arrive; the last warp publishes: slot posted / slot freed / semaphore
      const bool publishes = (send && !ll_out) || recv || op.has_dep;
      if (threadIdx.x == 0) stamp(q, 2);
      // every warp releases its stores at CTA scope; the publisher's gpu/sys-scope release is
      // cumulative over what it acquired through the arrival counter (PTX causality order)
      __syncwarp();
      if (wl == 0) {
        unsigned prev;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(prev) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(&s_arrive[q % kRing]))) : "memory");
        if (prev == kWarps - 1) {
          s_arrive[q % kRing] = 0;
          if (publishes) fence_acq_rel(sys);
          if (send && !ll_out) st_release(cout.head, sent + 1, sys);
          if (recv) st_release(cin.tail, rcvd + 1, sys);
          if (op.has_dep) st_release(my_sem, (epoch << 32) | static_cast<uint64_t>(iter * tb.nops + s + 1), false);
          if (q + 1 == total_ops) {  // persistent FIFO counters for the next launch
            if (has_in) *cin.mine = rcvd + (recv ? 1 : 0);
            if (has_out) *cout.mine = sent + (send ? 1 : 0);
          }
          stamp(q, 3);
          __threadfence_block();
          s_posted = q + 1;
        }
      }
      if (send) ++sent;
      if (recv) ++rcvd;
    }
  }
}

}  // namespace dev

}  // namespace gc3
