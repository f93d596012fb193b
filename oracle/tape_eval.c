/*
 * TEST INFRASTRUCTURE — the parity checker, never the product path.
 *
 * A plain-C restatement of the reference CPU executor's tape semantics
 * (staircase `run_tape`), used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg to check the CUDA backend.  Nothing under
 * paper_2307_16080_b200/ may link or call this file.
 *
 * Reference semantics restated here (file:line into /root/reference/pkg/src/staircase):
 *   opcode numbering and operand layout ........ interp/tape.py:20-45
 *   dispatch loop (tally[op] += 1 per instr) .... interp/_evalpy.py:81-232
 *   LOAD/STORE row-major offset + bounds check .. interp/_evalpy.py:90-114
 *   integer store wrap .......................... interp/_evalpy.py:108-110, interp/buffer.py:22-24
 *   BINF in double, f32 results rounded per op .. interp/_evalpy.py:115-127, interp/_evalcy.pyx:122-136
 *   BINI two's-complement wrap .................. interp/_evalpy.py:128-138
 *   loops: test (+1 bookkeeping), next, step<=0 . interp/_evalpy.py:139-163
 *   CMPF / CMPI predicates ...................... interp/_evalpy.py:168-199
 *   CAST index_cast (i32 wrap) .................. interp/_evalpy.py:200-202
 *   PARALLEL row-major product, +1 per point .... interp/_evalpy.py:235-273
 *   CALL / RETURN ............................... interp/_evalpy.py:216-226
 *   LAUNCH bx,by,bz,tx,ty,tz (+1 per thread) .... interp/_evalpy.py:303-331
 *   GPUID ........................................ interp/_evalpy.py:228-230
 *
 * Compiled with -O2 -ffp-contract=off so every f32/f64 operation is a
 * separately rounded IEEE operation, exactly like the reference.
 *
 * Encoding (built by oracle/encode.py): a program is a list of tapes; each
 * tape is a list of instructions; each instruction is a variable-length run
 * of int64 words starting with the opcode.  ins_off[t][pc] gives the word
 * offset of instruction pc of tape t.  Registers are 64-bit slots holding
 * either an int64 or a double (the instruction decides which).  Memref
 * registers hold an index into the buffer table.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  CONST = 0, BINF = 1, BINI = 2, CMPF = 3, CMPI = 4, CAST = 5, LOAD = 6,
  STORE = 7, ALLOC = 8, DEALLOC = 9, LOOP_INIT_S = 10, LOOP_INIT_A = 11,
  LOOP_TEST_R = 12, LOOP_TEST_I = 13, LOOP_NEXT_R = 14, LOOP_NEXT_I = 15,
  JUMP = 16, IF_FALSE = 17, PARALLEL = 18, CALL = 19, RETURN = 20,
  LAUNCH = 21, GPUID = 22, RETURN_GPU = 23, N_OPCODES = 24
};

/* dtype codes: 0 f32, 1 f64, 2 i32, 3 i64 */
typedef struct {
  void *data;
  int64_t dtype;
  int64_t rank;
  int64_t shape[8];
  int64_t strides[8];
} orc_buf;

typedef union {
  int64_t i;
  double f;
} slot;

typedef struct {
  const int64_t *words;     /* all instruction words, all tapes */
  const int64_t *tape_info; /* per tape: [first_ins, n_ins, n_regs, ...] */
  const int64_t *ins_off;   /* per global instruction index: word offset */
  orc_buf *bufs;            /* buffer table (args first, allocs appended) */
  int64_t n_bufs, cap_bufs;
  int64_t *tally;           /* N_OPCODES + 1 */
  int64_t gpu_emulated;
  int64_t gpu_ids[6];
  int64_t have_gpu_ids;
  /* error report */
  int64_t err;              /* 0 ok, 1 OOB, 2 InvalidBound, 3 ModeUnsupported */
  int64_t err_a, err_b, err_c, err_d; /* OOB: idx, extent, buf, loc; launch: loc */
} orc_machine;

#define TAPE_FIRST(m, t) ((m)->tape_info[4 * (t) + 0])
#define TAPE_NINS(m, t) ((m)->tape_info[4 * (t) + 1])
#define TAPE_NREGS(m, t) ((m)->tape_info[4 * (t) + 2])

static int64_t wrap_i32(int64_t v) { return (int64_t)(int32_t)(uint32_t)(uint64_t)v; }

static int64_t elem_size(int64_t dtype) { return (dtype == 1 || dtype == 3) ? 8 : 4; }

/* Returns pointer to the instruction words of instruction pc of tape t. */
static const int64_t *ins_at(orc_machine *m, int64_t t, int64_t pc) {
  return m->words + m->ins_off[TAPE_FIRST(m, t) + pc];
}

static int run_tape(orc_machine *m, int64_t t, slot *regs, slot *rets, int64_t *n_rets);

/* Row-major offset with the per-dimension bounds check of _evalpy.py:90-97. */
static int offset_of(orc_machine *m, const orc_buf *b, int64_t bufno, const int64_t *idx,
                     int64_t rank, slot *regs, int64_t loc, int64_t *off_out) {
  int64_t off = 0;
  for (int64_t k = 0; k < rank; ++k) {
    int64_t i = regs[idx[k]].i;
    if (i < 0 || i >= b->shape[k]) {
      m->err = 1;
      m->err_a = i;
      m->err_b = b->shape[k];
      m->err_c = bufno;
      m->err_d = loc;
      return -1;
    }
    off += i * b->strides[k];
  }
  *off_out = off;
  return 0;
}

static int64_t new_buffer(orc_machine *m, const int64_t *shape, int64_t rank, int64_t dtype) {
  if (m->n_bufs == m->cap_bufs) {
    int64_t cap = m->cap_bufs ? m->cap_bufs * 2 : 16;
    orc_buf *nb = (orc_buf *)malloc(sizeof(orc_buf) * cap);
    if (m->n_bufs) memcpy(nb, m->bufs, sizeof(orc_buf) * m->n_bufs);
    /* the caller-owned initial table is never freed here */
    m->bufs = nb;
    m->cap_bufs = cap;
  }
  orc_buf *b = &m->bufs[m->n_bufs];
  int64_t size = 1;
  b->rank = rank;
  b->dtype = dtype;
  for (int64_t k = 0; k < rank; ++k) {
    b->shape[k] = shape[k];
    size *= shape[k];
  }
  int64_t s = 1;
  for (int64_t k = rank - 1; k >= 0; --k) {
    b->strides[k] = s;
    s *= shape[k];
  }
  b->data = calloc((size_t)size, (size_t)elem_size(dtype));
  return m->n_bufs++;
}

/* PARALLEL: iterate the row-major product of the ranges, one bookkeeping
 * count per point, sub-register file seeded from captures once and reused
 * across points (_evalpy.py:244-273). */
static int run_parallel(orc_machine *m, const int64_t *w, slot *regs) {
  int64_t sub = w[1], nd = w[2];
  const int64_t *lbr = w + 3, *ubr = w + 3 + nd, *str = w + 3 + 2 * nd;
  int64_t ncap = w[3 + 3 * nd];
  const int64_t *caps = w + 4 + 3 * nd; /* pairs outer,inner */
  const int64_t *index_regs = caps + 2 * ncap;
  int64_t lb[8], ub[8], st[8], cur[8];
  for (int64_t d = 0; d < nd; ++d) {
    lb[d] = regs[lbr[d]].i;
    ub[d] = regs[ubr[d]].i;
    st[d] = regs[str[d]].i;
    if (st[d] <= 0) {
      m->err = 2;
      return -1;
    }
  }
  for (int64_t d = 0; d < nd; ++d)
    if (lb[d] >= ub[d]) return 0; /* empty product */
  int64_t nregs = TAPE_NREGS(m, sub);
  slot *sr = (slot *)calloc((size_t)(nregs ? nregs : 1), sizeof(slot));
  for (int64_t c = 0; c < ncap; ++c) sr[caps[2 * c + 1]] = regs[caps[2 * c]];
  for (int64_t d = 0; d < nd; ++d) cur[d] = lb[d];
  int rc = 0;
  for (;;) {
    for (int64_t d = 0; d < nd; ++d) sr[index_regs[d]].i = cur[d];
    m->tally[N_OPCODES] += 1;
    int64_t nr = 0;
    rc = run_tape(m, sub, sr, NULL, &nr);
    if (rc) break;
    int64_t d = nd - 1;
    for (; d >= 0; --d) {
      cur[d] += st[d];
      if (cur[d] < ub[d]) break;
      cur[d] = lb[d];
    }
    if (d < 0) break;
  }
  free(sr);
  return rc;
}

/* LAUNCH: gpu_emulated only; six nested host loops, fresh kernel register
 * file per thread (_evalpy.py:303-331). */
static int run_launch(orc_machine *m, const int64_t *w, slot *regs) {
  int64_t kern = w[1];
  int64_t nargs = w[8];
  const int64_t *args = w + 9;
  int64_t loc = w[9 + nargs];
  if (!m->gpu_emulated) {
    m->err = 3;
    m->err_d = loc;
    return -1;
  }
  int64_t g[3], b[3];
  for (int d = 0; d < 3; ++d) {
    g[d] = regs[w[2 + d]].i;
    b[d] = regs[w[5 + d]].i;
  }
  /* kernel arg registers are the first tape_info extras */
  int64_t nregs = TAPE_NREGS(m, kern);
  const int64_t *arg_regs = m->words + m->tape_info[4 * kern + 3];
  int64_t saved_have = m->have_gpu_ids, saved[6];
  memcpy(saved, m->gpu_ids, sizeof(saved));
  slot *kr = (slot *)malloc(sizeof(slot) * (size_t)(nregs ? nregs : 1));
  int rc = 0;
  for (int64_t bx = 0; bx < g[0] && !rc; ++bx)
    for (int64_t by = 0; by < g[1] && !rc; ++by)
      for (int64_t bz = 0; bz < g[2] && !rc; ++bz)
        for (int64_t tx = 0; tx < b[0] && !rc; ++tx)
          for (int64_t ty = 0; ty < b[1] && !rc; ++ty)
            for (int64_t tz = 0; tz < b[2] && !rc; ++tz) {
              m->gpu_ids[0] = bx; m->gpu_ids[1] = by; m->gpu_ids[2] = bz;
              m->gpu_ids[3] = tx; m->gpu_ids[4] = ty; m->gpu_ids[5] = tz;
              m->have_gpu_ids = 1;
              m->tally[N_OPCODES] += 1;
              memset(kr, 0, sizeof(slot) * (size_t)(nregs ? nregs : 1));
              for (int64_t a = 0; a < nargs; ++a) kr[arg_regs[a]] = regs[args[a]];
              int64_t nr = 0;
              rc = run_tape(m, kern, kr, NULL, &nr);
            }
  free(kr);
  memcpy(m->gpu_ids, saved, sizeof(saved));
  m->have_gpu_ids = saved_have;
  return rc;
}

static int run_tape(orc_machine *m, int64_t t, slot *regs, slot *rets, int64_t *n_rets) {
  int64_t n = TAPE_NINS(m, t);
  int64_t pc = 0;
  while (pc < n) {
    const int64_t *w = ins_at(m, t, pc);
    int64_t op = w[0];
    m->tally[op] += 1;
    switch (op) {
      case LOAD: { /* [op, dst, buf, rank, idx..., loc] */
        int64_t bufno = regs[w[2]].i, rank = w[3], off;
        orc_buf *b = &m->bufs[bufno];
        if (offset_of(m, b, bufno, w + 4, rank, regs, w[4 + rank], &off)) return -1;
        switch (b->dtype) {
          case 0: regs[w[1]].f = (double)((float *)b->data)[off]; break;
          case 1: regs[w[1]].f = ((double *)b->data)[off]; break;
          case 2: regs[w[1]].i = (int64_t)((int32_t *)b->data)[off]; break;
          default: regs[w[1]].i = ((int64_t *)b->data)[off]; break;
        }
        break;
      }
      case STORE: { /* [op, src, buf, rank, idx..., loc] */
        int64_t bufno = regs[w[2]].i, rank = w[3], off;
        orc_buf *b = &m->bufs[bufno];
        if (offset_of(m, b, bufno, w + 4, rank, regs, w[4 + rank], &off)) return -1;
        switch (b->dtype) {
          case 0: ((float *)b->data)[off] = (float)regs[w[1]].f; break;
          case 1: ((double *)b->data)[off] = regs[w[1]].f; break;
          case 2: ((int32_t *)b->data)[off] = (int32_t)wrap_i32(regs[w[1]].i); break;
          default: ((int64_t *)b->data)[off] = regs[w[1]].i; break;
        }
        break;
      }
      case BINF: { /* [op, dst, fop, a, b, is_f32] */
        double a = regs[w[3]].f, b = regs[w[4]].f, r;
        switch (w[2]) {
          case 0: r = a + b; break;
          case 1: r = a - b; break;
          case 2: r = a * b; break;
          default: r = a / b; break; /* IEEE: matches _fdiv incl. x/0 */
        }
        if (w[5]) r = (double)(float)r;
        regs[w[1]].f = r;
        break;
      }
      case BINI: { /* [op, dst, iop, a, b, is_i32] */
        uint64_t a = (uint64_t)regs[w[3]].i, b = (uint64_t)regs[w[4]].i, r;
        switch (w[2]) {
          case 0: r = a + b; break;
          case 1: r = a - b; break;
          default: r = a * b; break;
        }
        regs[w[1]].i = w[5] ? wrap_i32((int64_t)r) : (int64_t)r;
        break;
      }
      case LOOP_TEST_R:
        if (regs[w[1]].i >= regs[w[2]].i) {
          pc = w[3];
          continue;
        }
        m->tally[N_OPCODES] += 1;
        break;
      case LOOP_TEST_I:
        if (regs[w[1]].i >= w[2]) {
          pc = w[3];
          continue;
        }
        m->tally[N_OPCODES] += 1;
        break;
      case LOOP_NEXT_R: {
        int64_t step = regs[w[2]].i;
        if (step <= 0) {
          m->err = 2;
          return -1;
        }
        regs[w[1]].i += step;
        pc = w[3];
        continue;
      }
      case LOOP_NEXT_I:
        regs[w[1]].i += w[2];
        pc = w[3];
        continue;
      case LOOP_INIT_S: regs[w[1]] = regs[w[2]]; break;
      case LOOP_INIT_A: regs[w[1]].i = w[2]; break;
      case CONST: /* [op, dst, kind(0 int/1 float), bits] */
        if (w[2]) memcpy(&regs[w[1]].f, &w[3], 8);
        else regs[w[1]].i = w[3];
        break;
      case CMPF: {
        double a = regs[w[3]].f, b = regs[w[4]].f;
        int64_t r;
        switch (w[2]) {
          case 0: r = a == b; break;
          case 1: r = (a == a) && (b == b) && (a != b); break;
          case 2: r = a < b; break;
          case 3: r = a <= b; break;
          case 4: r = a > b; break;
          default: r = a >= b; break;
        }
        regs[w[1]].i = r;
        break;
      }
      case CMPI: {
        int64_t a = regs[w[3]].i, b = regs[w[4]].i, r;
        switch (w[2]) {
          case 0: r = a == b; break;
          case 1: r = a != b; break;
          case 2: r = a < b; break;
          case 3: r = a <= b; break;
          case 4: r = a > b; break;
          default: r = a >= b; break;
        }
        regs[w[1]].i = r;
        break;
      }
      case CAST: /* [op, dst, src, to_i32] */
        regs[w[1]].i = w[3] ? wrap_i32(regs[w[2]].i) : regs[w[2]].i;
        break;
      case IF_FALSE:
        if (!regs[w[1]].i) {
          pc = w[2];
          continue;
        }
        break;
      case JUMP:
        pc = w[1];
        continue;
      case ALLOC: /* [op, dst, dtype, rank, shape...] */
        regs[w[1]].i = new_buffer(m, w + 4, w[3], w[2]);
        break;
      case DEALLOC:
        break;
      case PARALLEL:
        if (run_parallel(m, w, regs)) return -1;
        break;
      case CALL: { /* [op, callee, nargs, args..., ndst, dsts...] */
        int64_t callee = w[1], nargs = w[2];
        const int64_t *args = w + 3;
        int64_t ndst = w[3 + nargs];
        const int64_t *dsts = w + 4 + nargs;
        int64_t nregs = TAPE_NREGS(m, callee);
        const int64_t *arg_regs = m->words + m->tape_info[4 * callee + 3];
        slot *cr = (slot *)calloc((size_t)(nregs ? nregs : 1), sizeof(slot));
        for (int64_t a = 0; a < nargs; ++a) cr[arg_regs[a]] = regs[args[a]];
        slot rv[16];
        int64_t nr = 0;
        int rc = run_tape(m, callee, cr, rv, &nr);
        free(cr);
        if (rc) return -1;
        for (int64_t d = 0; d < ndst && d < nr; ++d) regs[dsts[d]] = rv[d];
        break;
      }
      case RETURN:
      case RETURN_GPU: { /* [op, n, srcs...] */
        int64_t nr = w[1];
        if (rets)
          for (int64_t k = 0; k < nr && k < 16; ++k) rets[k] = regs[w[2 + k]];
        *n_rets = nr;
        return 0;
      }
      case LAUNCH:
        if (run_launch(m, w, regs)) return -1;
        break;
      case GPUID: /* [op, dst, dim, is_thread] */
        regs[w[1]].i = m->gpu_ids[w[2] + (w[3] ? 3 : 0)];
        break;
      default:
        return -1;
    }
    pc += 1;
  }
  *n_rets = -1; /* fell off the end: no RETURN (body tapes) */
  return 0;
}

/*
 * Entry point.  regs: the entry tape's register file, pre-seeded with
 * argument values (memref args hold buffer-table indices).  On return,
 * rets[0..n_rets) hold the RETURN operands.  bufs/n_bufs: the buffer
 * table; buffers created by ALLOC are appended and reported through
 * out_bufs / out_n_bufs (the caller frees them with orc_free_buffers).
 * status[0] = error code, status[1..4] = error payload.
 */
int orc_run(const int64_t *words, const int64_t *tape_info, const int64_t *ins_off,
            int64_t entry, orc_buf *bufs, int64_t n_bufs, slot *regs, slot *rets,
            int64_t *n_rets, int64_t *tally, int64_t gpu_emulated, int64_t *status,
            orc_buf **out_bufs, int64_t *out_n_bufs) {
  orc_machine m;
  memset(&m, 0, sizeof(m));
  m.words = words;
  m.tape_info = tape_info;
  m.ins_off = ins_off;
  m.bufs = bufs;
  m.n_bufs = n_bufs;
  m.cap_bufs = n_bufs;
  m.tally = tally;
  m.gpu_emulated = gpu_emulated;
  int rc = run_tape(&m, entry, regs, rets, n_rets);
  status[0] = m.err;
  status[1] = m.err_a;
  status[2] = m.err_b;
  status[3] = m.err_c;
  status[4] = m.err_d;
  *out_bufs = m.bufs;
  *out_n_bufs = m.n_bufs;
  return rc ? -1 : 0;
}

void orc_free_table(orc_buf *table, orc_buf *initial, int64_t first_alloc, int64_t n) {
  for (int64_t k = first_alloc; k < n; ++k) free(table[k].data);
  if (table != initial) free(table);
}
