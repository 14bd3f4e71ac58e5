/*
 * gc3_oracle.c — CPU restatement of the GC3-IR interpreter.  TEST INFRASTRUCTURE ONLY.
 * See gc3_oracle.h for the contract, the reference citations and the parity status.
 */
#include "gc3_oracle.h"

#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ncclDataType_t / ncclRedOp_t numbering (nccl.h:260-290) */
enum { T_I8 = 0, T_U8, T_I32, T_U32, T_I64, T_U64, T_F16, T_F32, T_F64, T_BF16 };
enum { OP_SUM = 0, OP_PROD, OP_MAX, OP_MIN };

static int receives(int op) { return op == GC3O_RECV || op == GC3O_RRC || op == GC3O_RCS || op == GC3O_RRCS || op == GC3O_RRS; }
static int sends(int op) { return op == GC3O_SEND || op == GC3O_RCS || op == GC3O_RRCS || op == GC3O_RRS; }

static void set_err(char* err, size_t n, const char* fmt, ...) {
  if (!err || !n) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, n, fmt, ap);
  va_end(ap);
}

size_t gc3o_dtype_size(int dtype) {
  switch (dtype) {
    case T_I8: case T_U8: return 1;
    case T_F16: case T_BF16: return 2;
    case T_I32: case T_U32: case T_F32: return 4;
    case T_I64: case T_U64: case T_F64: return 8;
    default: return 0;
  }
}

/* ---- arithmetic ------------------------------------------------------------------------ */
/* Canonical NaNs: the device returns 0x7fffffff for any f32 arithmetic NaN; the restatement
 * canonicalises the same way so NaN-carrying inputs stay bit-exact. */
static float canon_f32(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7f800000u) == 0x7f800000u && (x & 0x7fffffu)) x = 0x7fffffffu;
  memcpy(&f, &x, 4);
  return f;
}
static double canon_f64(double d) {
  uint64_t x;
  memcpy(&x, &d, 8);
  if ((x & 0x7ff0000000000000ull) == 0x7ff0000000000000ull && (x & 0xfffffffffffffull)) x = 0x7fffffffffffffffull;
  memcpy(&d, &x, 8);
  return d;
}
static float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000) << 16, exp = (h >> 10) & 0x1f, mant = h & 0x3ff, x;
  if (exp == 0x1f) x = sign | 0x7f800000u | (mant << 13);
  else if (exp == 0) {
    if (mant == 0) x = sign;
    else { /* subnormal: normalise */
      int e = -1;
      do { mant <<= 1; e++; } while (!(mant & 0x400));
      x = sign | ((uint32_t)(127 - 15 - e) << 23) | ((mant & 0x3ff) << 13);
    }
  } else x = sign | ((exp + 112) << 23) | (mant << 13);
  float f;
  memcpy(&f, &x, 4);
  return f;
}
static uint16_t f32_to_f16(float f) { /* round to nearest even, NaN -> 0x7fff */
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000, exp = (x >> 23) & 0xff, mant = x & 0x7fffff;
  if (exp == 0xff) return mant ? 0x7fff : (uint16_t)(sign | 0x7c00);
  if (exp <= 112) { /* result subnormal or zero: value = m * 2^(exp-150), unit 2^-24 */
    if (exp < 102) return (uint16_t)sign;
    uint32_t m = mant | 0x800000u, shift = 126 - exp, q = m >> shift, rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1))) q++;
    return (uint16_t)(sign | q);
  }
  uint32_t q = ((exp - 112) << 10) | (mant >> 13), rem = mant & 0x1fff;
  if (rem > 0x1000 || (rem == 0x1000 && (q & 1))) q++;
  if (q >= 0x7c00) q = 0x7c00;
  return (uint16_t)(sign | q);
}
static float bf16_to_f32(uint16_t h) {
  uint32_t x = (uint32_t)h << 16;
  float f;
  memcpy(&f, &x, 4);
  return f;
}
static uint16_t f32_to_bf16(float f) { /* round to nearest even, NaN -> 0x7fff */
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7f800000u) == 0x7f800000u && (x & 0x7fffffu)) return 0x7fff;
  x += 0x7fffu + ((x >> 16) & 1);
  return (uint16_t)(x >> 16);
}

/* max/min select the non-NaN operand; on equality (incl. -0 == +0) they return b. */
#define FMAX(a, b) ((a) != (a) ? (b) : (b) != (b) ? (a) : ((a) > (b) ? (a) : (b)))
#define FMIN(a, b) ((a) != (a) ? (b) : (b) != (b) ? (a) : ((a) < (b) ? (a) : (b)))
#define IMAX(a, b) ((a) > (b) ? (a) : (b))
#define IMIN(a, b) ((a) < (b) ? (a) : (b))

#define INT_LOOP(T, UT)                                                              \
  {                                                                                  \
    T* x = (T*)a;                                                                    \
    const T* y = (const T*)b;                                                        \
    for (size_t i = 0; i < n; i++) {                                                 \
      switch (redop) {                                                               \
        case OP_SUM: x[i] = (T)((UT)x[i] + (UT)y[i]); break;                         \
        case OP_PROD: x[i] = (T)((UT)x[i] * (UT)y[i]); break;                        \
        case OP_MAX: x[i] = IMAX(x[i], y[i]); break;                                 \
        default: x[i] = IMIN(x[i], y[i]); break;                                     \
      }                                                                              \
    }                                                                                \
    return 0;                                                                        \
  }

static float f32op(float p, float q, int redop) {
  switch (redop) {
    case OP_SUM: return canon_f32(p + q);
    case OP_PROD: return canon_f32(p * q);
    case OP_MAX: return FMAX(p, q);
    default: return FMIN(p, q);
  }
}

int gc3o_reduce(void* a, const void* b, size_t n, int dtype, int redop) {
  if (redop < OP_SUM || redop > OP_MIN) return -1;
  switch (dtype) {
    case T_I8: INT_LOOP(int8_t, uint8_t)
    case T_U8: INT_LOOP(uint8_t, uint8_t)
    case T_I32: INT_LOOP(int32_t, uint32_t)
    case T_U32: INT_LOOP(uint32_t, uint32_t)
    case T_I64: INT_LOOP(int64_t, uint64_t)
    case T_U64: INT_LOOP(uint64_t, uint64_t)
    case T_F32: {
      float* x = (float*)a;
      const float* y = (const float*)b;
      for (size_t i = 0; i < n; i++) x[i] = f32op(x[i], y[i], redop);
      return 0;
    }
    case T_F64: {
      double* x = (double*)a;
      const double* y = (const double*)b;
      for (size_t i = 0; i < n; i++) {
        double p = x[i], q = y[i];
        switch (redop) {
          case OP_SUM: x[i] = canon_f64(p + q); break;
          case OP_PROD: x[i] = canon_f64(p * q); break;
          case OP_MAX: x[i] = FMAX(p, q); break;
          default: x[i] = FMIN(p, q); break;
        }
      }
      return 0;
    }
    case T_F16: case T_BF16: {
      uint16_t* x = (uint16_t*)a;
      const uint16_t* y = (const uint16_t*)b;
      const int bf = dtype == T_BF16;
      for (size_t i = 0; i < n; i++) {
        float p = bf ? bf16_to_f32(x[i]) : f16_to_f32(x[i]);
        float q = bf ? bf16_to_f32(y[i]) : f16_to_f32(y[i]);
        if (redop == OP_MAX || redop == OP_MIN) { /* select: keep the original bits */
          int pn = p != p, qn = q != q;
          int take_b = pn ? 1 : qn ? 0 : (redop == OP_MAX ? !(p > q) : !(p < q));
          x[i] = take_b ? y[i] : x[i];
        } else {
          float r = f32op(p, q, redop);
          x[i] = bf ? f32_to_bf16(r) : f32_to_f16(r);
        }
      }
      return 0;
    }
    default: return -1;
  }
}

/* ---- program bookkeeping --------------------------------------------------------------- */
typedef struct {
  int src, dst, ch;
} conn_key;

typedef struct {
  const gc3o_program* p;
  char* const* bufs;
  size_t chunk_elems, esize, tile_elems, ntiles;
  int dtype, redop;
  int nconn, dry;
  int* conn_in;  /* per tb: incoming connection index or -1 */
  int* conn_out; /* per tb: outgoing connection index or -1 */
  int* tb_base;  /* per rank: index of its first tb */
  int* tb_count; /* per rank */
} ctx_t;

static int find_conn(conn_key* keys, int* n, int src, int dst, int ch) {
  for (int i = 0; i < *n; i++)
    if (keys[i].src == src && keys[i].dst == dst && keys[i].ch == ch) return i;
  keys[*n].src = src;
  keys[*n].dst = dst;
  keys[*n].ch = ch;
  return (*n)++;
}

static int ctx_init(ctx_t* c, const gc3o_program* p, void* const* bufs, size_t chunk_elems, int dtype, int redop,
                    size_t tile_elems, char* err, size_t errlen) {
  memset(c, 0, sizeof(*c));
  c->p = p;
  c->bufs = (char* const*)bufs;
  c->chunk_elems = chunk_elems;
  c->esize = gc3o_dtype_size(dtype);
  c->dtype = dtype;
  c->redop = redop;
  if (!c->esize) { set_err(err, errlen, "unsupported dtype %d", dtype); return -1; }
  c->tile_elems = (tile_elems == 0 || tile_elems > chunk_elems) ? chunk_elems : tile_elems;
  c->ntiles = chunk_elems == 0 ? 0 : (chunk_elems + c->tile_elems - 1) / c->tile_elems;
  c->conn_in = malloc(sizeof(int) * (p->ntbs + 1));
  c->conn_out = malloc(sizeof(int) * (p->ntbs + 1));
  c->tb_base = calloc(p->nranks + 1, sizeof(int));
  c->tb_count = calloc(p->nranks + 1, sizeof(int));
  conn_key* keys = malloc(sizeof(conn_key) * (2 * p->ntbs + 1));
  for (int t = 0; t < p->ntbs; t++) {
    const gc3o_tb* tb = &p->tbs[t];
    if (tb->rank < 0 || tb->rank >= p->nranks) { set_err(err, errlen, "tb %d: bad rank", t); free(keys); return -1; }
    if (c->tb_count[tb->rank]++ == 0) c->tb_base[tb->rank] = t;
    c->conn_out[t] = tb->send_peer >= 0 ? find_conn(keys, &c->nconn, tb->rank, tb->send_peer, tb->channel) : -1;
    c->conn_in[t] = tb->recv_peer >= 0 ? find_conn(keys, &c->nconn, tb->recv_peer, tb->rank, tb->channel) : -1;
  }
  free(keys);
  for (int t = 0; t < p->ntbs; t++) {
    const gc3o_tb* tb = &p->tbs[t];
    for (int s = 0; s < tb->nops; s++) {
      const gc3o_op* op = &p->ops[tb->first_op + s];
      if (sends(op->opcode) && c->conn_out[t] < 0) { set_err(err, errlen, "rank %d tb %d step %d sends without a send peer", tb->rank, t, s); return -1; }
      if (receives(op->opcode) && c->conn_in[t] < 0) { set_err(err, errlen, "rank %d tb %d step %d receives without a receive peer", tb->rank, t, s); return -1; }
      for (int d = 0; d < op->ndeps; d++)
        if (op->dep_tb[d] < 0 || op->dep_tb[d] >= c->tb_count[tb->rank]) { set_err(err, errlen, "rank %d tb %d step %d: bad dep", tb->rank, t, s); return -1; }
      if (op->count < 1 && op->opcode != GC3O_NOP) { set_err(err, errlen, "count < 1"); return -1; }
      const int bufs_ok = op->src_buf >= 0 && op->src_buf < 3 && op->dst_buf >= 0 && op->dst_buf < 3;
      if (!bufs_ok) { set_err(err, errlen, "bad buffer"); return -1; }
      if (op->opcode != GC3O_NOP) {
        /* span checks for the spans the op touches locally (ir.hpp:388-389) */
        if (op->src_off < 0 || op->src_off + op->count > p->nchunks[op->src_buf] || op->dst_off < 0 || op->dst_off + op->count > p->nchunks[op->dst_buf]) {
          set_err(err, errlen, "rank %d tb %d step %d: span out of range", tb->rank, t, s);
          return -1;
        }
      }
    }
  }
  return 0;
}

static void ctx_free(ctx_t* c) {
  free(c->conn_in);
  free(c->conn_out);
  free(c->tb_base);
  free(c->tb_count);
}

/* address of tile t of chunk (off + j) in rank r's buffer b */
static char* tile_ptr(const ctx_t* c, int r, int b, int chunk, size_t t) {
  return c->bufs[r * 3 + b] + ((size_t)chunk * c->chunk_elems + t * c->tile_elems) * c->esize;
}
static size_t tile_len(const ctx_t* c, size_t t) {
  size_t beg = t * c->tile_elems;
  return beg >= c->chunk_elems ? 0 : (c->chunk_elems - beg < c->tile_elems ? c->chunk_elems - beg : c->tile_elems);
}

/*
 * Applies one op on tile t.  `in` is the incoming message (count tiles back to back), `out` the
 * outgoing message buffer.  Semantics: SURVEY.md Appendix B / lowering.hpp:68-77, 96-119.
 */
static void apply_op(const ctx_t* c, int r, const gc3o_op* op, size_t t, const char* in, char* out) {
  if (c->dry) return;
  const size_t len = tile_len(c, t), bytes = len * c->esize;
  for (int j = 0; j < op->count; j++) {
    char* src = tile_ptr(c, r, op->src_buf, op->src_off + j, t);
    char* dst = tile_ptr(c, r, op->dst_buf, op->dst_off + j, t);
    const char* msg = in ? in + j * bytes : NULL;
    char* o = out ? out + j * bytes : NULL;
    switch (op->opcode) {
      case GC3O_SEND: memcpy(o, src, bytes); break;
      case GC3O_RECV: memcpy(dst, msg, bytes); break;
      case GC3O_COPY: memmove(dst, src, bytes); break;
      case GC3O_REDUCE: gc3o_reduce(dst, src, len, c->dtype, c->redop); break;
      case GC3O_RRC: /* dst = src (+) msg; the compiler emits src == dst (lowering.hpp:277) */
        if (dst != src) memmove(dst, src, bytes);
        gc3o_reduce(dst, msg, len, c->dtype, c->redop);
        break;
      case GC3O_RCS: memcpy(src, msg, bytes); memcpy(o, msg, bytes); break;
      case GC3O_RRCS: gc3o_reduce(src, msg, len, c->dtype, c->redop); memcpy(o, src, bytes); break;
      case GC3O_RRS: memcpy(o, src, bytes); gc3o_reduce(o, msg, len, c->dtype, c->redop); break;
      default: break;
    }
  }
}

/* ---- single-threaded modes --------------------------------------------------------------- */
typedef struct msg_s {
  struct msg_s* next;
  char data[];
} msg_t;
typedef struct {
  msg_t *head, *tail;
  int len;
} queue_t;

static uint64_t splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static int run_serial(ctx_t* c, int randomized, uint64_t seed, int slots, char* err, size_t errlen) {
  const gc3o_program* p = c->p;
  const int nt = p->ntbs;
  int* pc = calloc(nt, sizeof(int));
  size_t* tile = calloc(nt, sizeof(size_t));
  int64_t* sem = malloc(sizeof(int64_t) * nt); /* progress = tile * nops + step */
  queue_t* q = calloc(c->nconn + 1, sizeof(queue_t));
  int* runnable = malloc(sizeof(int) * (nt + 1));
  for (int t = 0; t < nt; t++) sem[t] = -1;
  const size_t ntiles = randomized ? c->ntiles : (c->chunk_elems ? 1 : 0);
  if (!randomized) { c->tile_elems = c->chunk_elems; }
  int rc = GC3O_OK;
  for (;;) {
    int nrun = 0, all_done = 1;
    for (int t = 0; t < nt; t++) {
      const gc3o_tb* tb = &p->tbs[t];
      if (tile[t] >= ntiles || tb->nops == 0) continue;
      all_done = 0;
      const gc3o_op* op = &p->ops[tb->first_op + pc[t]];
      int ok = 1;
      for (int d = 0; d < op->ndeps && ok; d++) {
        const int dt = c->tb_base[tb->rank] + op->dep_tb[d];
        const int64_t need = (int64_t)tile[t] * p->tbs[dt].nops + op->dep_step[d];
        if (sem[dt] < need) ok = 0;
      }
      if (ok && receives(op->opcode) && q[c->conn_in[t]].len == 0) ok = 0;
      if (ok && randomized && sends(op->opcode) && q[c->conn_out[t]].len >= slots) ok = 0;
      if (ok) runnable[nrun++] = t;
    }
    if (all_done) break;
    if (nrun == 0) {
      char buf[512];
      size_t off = 0;
      for (int t = 0; t < nt && off < sizeof(buf) - 40; t++)
        if (tile[t] < ntiles && p->tbs[t].nops)
          off += snprintf(buf + off, sizeof(buf) - off, " r%d.tb%d@t%zu.s%d", p->tbs[t].rank, t - c->tb_base[p->tbs[t].rank], tile[t], pc[t]);
      set_err(err, errlen, "deadlock: blocked%s", buf);
      rc = GC3O_DEADLOCK;
      break;
    }
    /* deterministic: run every runnable tb once per sweep in order; randomized: pick one */
    const int picks = randomized ? 1 : nrun;
    for (int k = 0; k < picks; k++) {
      const int t = randomized ? runnable[splitmix(&seed) % (uint64_t)nrun] : runnable[k];
      const gc3o_tb* tb = &p->tbs[t];
      const gc3o_op* op = &p->ops[tb->first_op + pc[t]];
      if (!randomized && k > 0) { /* re-check readiness: earlier picks this sweep may not matter, but queues may have changed */
        if (receives(op->opcode) && q[c->conn_in[t]].len == 0) continue;
      }
      const size_t bytes = tile_len(c, tile[t]) * c->esize * (size_t)op->count;
      msg_t* in = NULL;
      msg_t* out = NULL;
      if (receives(op->opcode)) {
        queue_t* qi = &q[c->conn_in[t]];
        in = qi->head;
        qi->head = in->next;
        if (!qi->head) qi->tail = NULL;
        qi->len--;
      }
      if (sends(op->opcode)) out = malloc(sizeof(msg_t) + (c->dry ? 0 : bytes) + 1);
      apply_op(c, tb->rank, op, tile[t], in ? in->data : NULL, out ? out->data : NULL);
      free(in);
      if (out) {
        queue_t* qo = &q[c->conn_out[t]];
        out->next = NULL;
        if (qo->tail) qo->tail->next = out; else qo->head = out;
        qo->tail = out;
        qo->len++;
      }
      sem[t] = (int64_t)tile[t] * tb->nops + pc[t];
      if (++pc[t] == tb->nops) { pc[t] = 0; tile[t]++; }
    }
  }
  for (int i = 0; i < c->nconn; i++) {
    while (q[i].head) { msg_t* m = q[i].head; q[i].head = m->next; free(m); }
  }
  free(pc); free(tile); free(sem); free(q); free(runnable);
  return rc;
}

/* ---- threaded mode (CPU baseline) -------------------------------------------------------- */
typedef struct {
  pthread_mutex_t mu;
  pthread_cond_t cv;
  char** slot;       /* s slot buffers */
  size_t head, tail; /* messages produced / consumed */
} tconn_t;

#include <time.h>
/* waits on cv for at most 20 ms; returns 1 once the global deadline passed or abort was raised */
static int timed_wait(pthread_cond_t* cv, pthread_mutex_t* mu, volatile int* abort_flag, const struct timespec* deadline) {
  struct timespec now, until;
  clock_gettime(CLOCK_REALTIME, &now);
  if (*abort_flag) return 1;
  if (now.tv_sec > deadline->tv_sec || (now.tv_sec == deadline->tv_sec && now.tv_nsec >= deadline->tv_nsec)) {
    *abort_flag = 1;
    return 1;
  }
  until = now;
  until.tv_nsec += 20 * 1000 * 1000;
  if (until.tv_nsec >= 1000000000L) { until.tv_sec++; until.tv_nsec -= 1000000000L; }
  pthread_cond_timedwait(cv, mu, &until);
  return *abort_flag;
}

typedef struct {
  ctx_t* c;
  tconn_t* conns;
  int slots;
  volatile int64_t* sem;
  pthread_mutex_t* sem_mu;
  pthread_cond_t* sem_cv;
  int t;
  volatile int* abort_flag;
  const struct timespec* deadline;
} targ_t;

static void* tb_thread(void* arg) {
  targ_t* a = (targ_t*)arg;
  ctx_t* c = a->c;
  const gc3o_program* p = c->p;
  const gc3o_tb* tb = &p->tbs[a->t];
  const int r = tb->rank;
  tconn_t* in = tb->recv_peer >= 0 ? &a->conns[c->conn_in[a->t]] : NULL;
  tconn_t* out = tb->send_peer >= 0 ? &a->conns[c->conn_out[a->t]] : NULL;
  for (size_t t = 0; t < c->ntiles; t++) {
    for (int s = 0; s < tb->nops; s++) {
      const gc3o_op* op = &p->ops[tb->first_op + s];
      if (op->ndeps) {
        pthread_mutex_lock(a->sem_mu);
        for (int d = 0; d < op->ndeps; d++) {
          const int dt = c->tb_base[r] + op->dep_tb[d];
          const int64_t need = (int64_t)t * p->tbs[dt].nops + op->dep_step[d];
          while (a->sem[dt] < need && !timed_wait(a->sem_cv, a->sem_mu, a->abort_flag, a->deadline)) {}
        }
        pthread_mutex_unlock(a->sem_mu);
      }
      const char* inmsg = NULL;
      char* outmsg = NULL;
      size_t in_idx = 0, out_idx = 0;
      if (receives(op->opcode)) {
        pthread_mutex_lock(&in->mu);
        while (in->head == in->tail && !timed_wait(&in->cv, &in->mu, a->abort_flag, a->deadline)) {}
        in_idx = in->tail;
        pthread_mutex_unlock(&in->mu);
        inmsg = in->slot[in_idx % a->slots];
      }
      if (sends(op->opcode)) {
        pthread_mutex_lock(&out->mu);
        while (out->head - out->tail >= (size_t)a->slots && !timed_wait(&out->cv, &out->mu, a->abort_flag, a->deadline)) {}
        out_idx = out->head;
        pthread_mutex_unlock(&out->mu);
        outmsg = out->slot[out_idx % a->slots];
      }
      if (*a->abort_flag) return NULL;
      apply_op(c, r, op, t, inmsg, outmsg);
      if (receives(op->opcode)) {
        pthread_mutex_lock(&in->mu);
        in->tail++;
        pthread_cond_broadcast(&in->cv);
        pthread_mutex_unlock(&in->mu);
      }
      if (sends(op->opcode)) {
        pthread_mutex_lock(&out->mu);
        out->head++;
        pthread_cond_broadcast(&out->cv);
        pthread_mutex_unlock(&out->mu);
      }
      if (op->has_dep) {
        pthread_mutex_lock(a->sem_mu);
        a->sem[a->t] = (int64_t)t * tb->nops + s;
        pthread_cond_broadcast(a->sem_cv);
        pthread_mutex_unlock(a->sem_mu);
      }
    }
  }
  return NULL;
}

static int run_threaded(ctx_t* c, int slots, char* err, size_t errlen) {
  const gc3o_program* p = c->p;
  int maxcount = 1;
  for (int t = 0; t < p->ntbs; t++)
    for (int s = 0; s < p->tbs[t].nops; s++)
      if (p->ops[p->tbs[t].first_op + s].count > maxcount) maxcount = p->ops[p->tbs[t].first_op + s].count;
  const size_t slot_bytes = (size_t)maxcount * c->tile_elems * c->esize + 1;
  tconn_t* conns = calloc(c->nconn + 1, sizeof(tconn_t));
  for (int i = 0; i < c->nconn; i++) {
    pthread_mutex_init(&conns[i].mu, NULL);
    pthread_cond_init(&conns[i].cv, NULL);
    conns[i].slot = malloc(sizeof(char*) * slots);
    for (int k = 0; k < slots; k++) conns[i].slot[k] = malloc(slot_bytes);
  }
  volatile int64_t* sem = malloc(sizeof(int64_t) * (p->ntbs + 1));
  for (int t = 0; t < p->ntbs; t++) sem[t] = -1;
  pthread_mutex_t sem_mu = PTHREAD_MUTEX_INITIALIZER;
  pthread_cond_t sem_cv = PTHREAD_COND_INITIALIZER;
  volatile int abort_flag = 0;
  struct timespec deadline;
  clock_gettime(CLOCK_REALTIME, &deadline);
  deadline.tv_sec += 120;
  pthread_t* th = malloc(sizeof(pthread_t) * (p->ntbs + 1));
  targ_t* args = malloc(sizeof(targ_t) * (p->ntbs + 1));
  int rc = GC3O_OK;
  for (int t = 0; t < p->ntbs; t++) {
    args[t] = (targ_t){c, conns, slots, sem, &sem_mu, &sem_cv, t, &abort_flag, &deadline};
    if (pthread_create(&th[t], NULL, tb_thread, &args[t])) {
      set_err(err, errlen, "pthread_create failed");
      abort_flag = 1;
      rc = GC3O_ERROR;
      for (int u = 0; u < t; u++) pthread_join(th[u], NULL);
      goto done;
    }
  }
  for (int t = 0; t < p->ntbs; t++) pthread_join(th[t], NULL);
  if (abort_flag) {
    set_err(err, errlen, "threaded run timed out (deadlock or > 120 s)");
    rc = GC3O_DEADLOCK;
  }
done:
  for (int i = 0; i < c->nconn; i++) {
    for (int k = 0; k < slots; k++) free(conns[i].slot[k]);
    free(conns[i].slot);
    pthread_mutex_destroy(&conns[i].mu);
    pthread_cond_destroy(&conns[i].cv);
  }
  free(conns);
  free((void*)sem);
  free(th);
  free(args);
  return rc;
}

/* ---- race detection ("happens-before race detection over (rank, buffer,
 * index) slots", "vector clocks over block steps, comm edges, and semaphore edges") ------------
 * One dry deterministic run: every thread block carries a vector clock (ops completed per thread
 * block); a message carries its sender's clock (comm edge, k-th send -> k-th receive), a dep joins
 * the clock the depended-on op published (semaphore edge).  Every local access of a chunk slot is
 * checked against the slot's last write and the reads since: two accesses conflict when at least
 * one writes and neither clock has seen the other.  In-place programs alias output onto input
 * (core.hpp:167-170). */
typedef struct {
  int tb, clk, step; /* accessor, its own clock after the op (1-based op count), its step */
} acc_t;
typedef struct {
  acc_t w;      /* last write (tb < 0: none) */
  acc_t* rd;    /* reads since the last write */
  int nrd, cap;
} slot_t;

static void race_add(gc3o_race* out, int max, int* n, const gc3o_program* p, const ctx_t* c, int rank, int buf, int idx,
                     acc_t a, acc_t b, int kind) {
  if (*n < max && out) {
    gc3o_race* r = &out[*n];
    r->rank = rank, r->buf = buf, r->index = idx, r->kind = kind;
    r->tb_a = a.tb - c->tb_base[rank], r->step_a = a.step;
    r->tb_b = b.tb - c->tb_base[rank], r->step_b = b.step;
  }
  (*n)++;
  (void)p;
}

int gc3o_races(const gc3o_program* p, gc3o_race* out, int max, char* err, size_t errlen) {
  ctx_t c;
  if (err && errlen) err[0] = 0;
  if (ctx_init(&c, p, NULL, 1, 7 /* f32: dry run */, 0, 0, err, errlen)) { ctx_free(&c); return -1; }
  const int nt = p->ntbs;
  int nops = 0;
  for (int t = 0; t < nt; t++) nops += p->tbs[t].nops;
  int* vc = calloc((size_t)nt * nt, sizeof(int));                  /* current clock per tb */
  int* snap = calloc((size_t)(nops + 1) * nt, sizeof(int));        /* clock after every op */
  int* pc = calloc(nt, sizeof(int));
  /* per connection: FIFO of sender clocks (unbounded, k-th send -> k-th receive) */
  int** fifo = calloc(c.nconn + 1, sizeof(int*));
  int* fhead = calloc(c.nconn + 1, sizeof(int));
  int* ftail = calloc(c.nconn + 1, sizeof(int));
  int* fcap = calloc(c.nconn + 1, sizeof(int));
  /* slots: per rank, buffers 0..2 x nchunks */
  const int nslot_rank = p->nchunks[0] + p->nchunks[1] + p->nchunks[2];
  slot_t* slots = calloc((size_t)p->nranks * nslot_rank + 1, sizeof(slot_t));
  for (int i = 0; i < p->nranks * nslot_rank; i++) slots[i].w.tb = -1;
  int nraces = 0, rc = 0;
  for (;;) {
    int progress = 0, all_done = 1;
    for (int t = 0; t < nt; t++) {
      const gc3o_tb* tb = &p->tbs[t];
      if (pc[t] >= tb->nops) continue;
      all_done = 0;
      const gc3o_op* op = &p->ops[tb->first_op + pc[t]];
      int ok = 1;
      for (int d = 0; d < op->ndeps && ok; d++) {
        const int dt = c.tb_base[tb->rank] + op->dep_tb[d];
        if (pc[dt] <= op->dep_step[d]) ok = 0;
      }
      if (ok && receives(op->opcode) && fhead[c.conn_in[t]] == ftail[c.conn_in[t]]) ok = 0;
      if (!ok) continue;
      int* me = vc + (size_t)t * nt;
      for (int d = 0; d < op->ndeps; d++) { /* semaphore edge */
        const int dt = c.tb_base[tb->rank] + op->dep_tb[d];
        const int* s = snap + (size_t)(p->tbs[dt].first_op + op->dep_step[d]) * nt;
        for (int k = 0; k < nt; k++) if (s[k] > me[k]) me[k] = s[k];
      }
      if (receives(op->opcode)) { /* comm edge */
        const int ci = c.conn_in[t];
        const int* s = fifo[ci] + (size_t)fhead[ci]++ * nt;
        for (int k = 0; k < nt; k++) if (s[k] > me[k]) me[k] = s[k];
      }
      me[t] = pc[t] + 1;
      /* local accesses (lowering.hpp:96-119): reads first, then writes */
      int rb[2] = {-1, -1}, ro[2] = {0, 0}, wb = -1, wo = 0, nr = 0;
      switch (op->opcode) {
        case GC3O_SEND: case GC3O_RRS: rb[nr] = op->src_buf, ro[nr++] = op->src_off; break;
        case GC3O_RECV: wb = op->dst_buf, wo = op->dst_off; break;
        case GC3O_COPY: case GC3O_RRC: rb[nr] = op->src_buf, ro[nr++] = op->src_off; wb = op->dst_buf, wo = op->dst_off; break;
        case GC3O_REDUCE:
          rb[nr] = op->src_buf, ro[nr++] = op->src_off;
          rb[nr] = op->dst_buf, ro[nr++] = op->dst_off;
          wb = op->dst_buf, wo = op->dst_off;
          break;
        case GC3O_RCS: wb = op->src_buf, wo = op->src_off; break;
        case GC3O_RRCS: rb[nr] = op->src_buf, ro[nr++] = op->src_off; wb = op->src_buf, wo = op->src_off; break;
        default: break;
      }
      const acc_t cur = {t, me[t], pc[t]};
      for (int i = 0; i <= nr; i++) {
        const int is_write = i == nr;
        const int b = is_write ? wb : rb[i];
        const int off = is_write ? wo : ro[i];
        if (b < 0) continue;
        const int sb = (p->inplace && b == GC3O_OUTPUT) ? GC3O_INPUT : b;
        const int base = sb == 0 ? 0 : sb == 1 ? p->nchunks[0] : p->nchunks[0] + p->nchunks[1];
        for (int j = 0; j < op->count; j++) {
          slot_t* s = &slots[(size_t)tb->rank * nslot_rank + base + off + j];
          if (s->w.tb >= 0 && s->w.tb != t && me[s->w.tb] < s->w.clk)
            race_add(out, max, &nraces, p, &c, tb->rank, sb, off + j, s->w, cur, is_write ? 0 : 1);
          if (is_write) {
            for (int k = 0; k < s->nrd; k++)
              if (s->rd[k].tb != t && me[s->rd[k].tb] < s->rd[k].clk)
                race_add(out, max, &nraces, p, &c, tb->rank, sb, off + j, s->rd[k], cur, 2);
            s->w = cur;
            s->nrd = 0;
          } else {
            if (s->nrd == s->cap) {
              s->cap = s->cap ? 2 * s->cap : 4;
              s->rd = realloc(s->rd, sizeof(acc_t) * s->cap);
            }
            s->rd[s->nrd++] = cur;
          }
        }
      }
      if (sends(op->opcode)) {
        const int co = c.conn_out[t];
        if (ftail[co] == fcap[co]) {
          fcap[co] = fcap[co] ? 2 * fcap[co] : 8;
          fifo[co] = realloc(fifo[co], sizeof(int) * (size_t)fcap[co] * nt);
        }
        memcpy(fifo[co] + (size_t)ftail[co]++ * nt, me, sizeof(int) * nt);
      }
      memcpy(snap + (size_t)(tb->first_op + pc[t]) * nt, me, sizeof(int) * nt);
      pc[t]++;
      progress = 1;
    }
    if (all_done) break;
    if (!progress) {
      set_err(err, errlen, "deadlock: the program cannot complete, races undetermined");
      rc = -1;
      break;
    }
  }
  for (int i = 0; i < p->nranks * nslot_rank; i++) free(slots[i].rd);
  for (int i = 0; i < c.nconn; i++) free(fifo[i]);
  free(slots); free(fifo); free(fhead); free(ftail); free(fcap); free(vc); free(snap); free(pc);
  ctx_free(&c);
  return rc < 0 ? rc : nraces;
}

int gc3o_run(const gc3o_program* p, void* const* bufs, size_t chunk_elems, int dtype, int redop,
             int mode, uint64_t seed, int slots, size_t tile_elems, char* err, size_t errlen) {
  ctx_t c;
  if (err && errlen) err[0] = 0;
  if (redop < OP_SUM || redop > OP_MIN) { set_err(err, errlen, "unsupported redop %d", redop); return GC3O_ERROR; }
  if (ctx_init(&c, p, bufs, chunk_elems, dtype, redop, tile_elems, err, errlen)) { ctx_free(&c); return GC3O_ERROR; }
  if (slots < 1) slots = 1;
  int rc;
  if (mode == GC3O_THREADED) {
    /* a deadlocking IR would hang the threads: screen it with the randomized simulation first
     * at the same capacity and tiling (fused ops atomic, as the threads implement them) */
    c.dry = 1;
    rc = run_serial(&c, 1, seed, slots, err, errlen);
    c.dry = 0;
    if (rc == GC3O_OK) rc = run_threaded(&c, slots, err, errlen);
  } else {
    rc = run_serial(&c, mode == GC3O_RANDOM, seed, slots, err, errlen);
  }
  ctx_free(&c);
  return rc;
}
