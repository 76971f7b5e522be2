/* gevo_plan.h -- the launch-plan format the host lowering hands to libgevo.
 *
 * A plan is one flat blob per generation:
 *   gevo_plan_header | gevo_instr[n_instr] | gevo_prog[n_prog] | double consts[n_const]
 * Each gevo_prog is one individual (one mutated program): index ranges into
 * the instruction table for its @train_step (step 0 and up to two more
 * layouts of its weights, which can differ only in operand layouts) and its
 * @forward, plus its arena size.
 *
 * Scratch is two-tier: values small enough live in the CTA's shared memory
 * (GEVO_BUF_SMEM, reused by liveness), the rest in the individual's HBM arena
 * (GEVO_BUF_ARENA); a value produced by one instruction and consumed by the
 * next therefore never round-trips through L2 unless it is large.
 *
 * Every device element is one 64-bit word (f32 of the dialect is computed as
 * float64 exactly like the reference, ir.py:33-37; i32 -> int64; i1 -> int64
 * 0/1).  Operands address a buffer (see GEVO_BUF_*) at an element offset with
 * per-dimension element strides; views (transpose, broadcast_in_dim, slice,
 * view-reshape) never become instructions -- they are folded into strides,
 * exactly the numpy views the reference interpreter passes around
 * (interpreter.py:118-153).
 */
#ifndef GEVO_PLAN_H
#define GEVO_PLAN_H
#include <stdint.h>

#define GEVO_PLAN_MAGIC 0x47455650u /* "GEVP" */
#define GEVO_PLAN_VERSION 2
#define GEVO_MAXR 6        /* max tensor rank */
#define GEVO_MAXP 8        /* max function params / returns */

/* buffer ids */
enum {
  GEVO_BUF_ARENA = 0,               /* per-individual scratch */
  GEVO_BUF_CONST = 1,               /* per-individual constant pool */
  GEVO_BUF_PARAM0 = 2,              /* params 0..7 -> ids 2..9 */
  GEVO_BUF_OUT0 = 2 + GEVO_MAXP,    /* returns 0..7 -> ids 10..17 */
  GEVO_BUF_SMEM = 2 + 2 * GEVO_MAXP, /* per-individual scratch in shared memory */
  GEVO_NBUF = 3 + 2 * GEVO_MAXP
};

/* element kinds */
enum { GEVO_K_F64 = 0, GEVO_K_I64 = 1, GEVO_K_I1 = 2 };

/* instruction classes (interpreter.py:78-185) */
enum {
  GEVO_OP_UNARY = 1,   /* sub: GEVO_U_* */
  GEVO_OP_BINARY = 2,  /* sub: GEVO_B_* */
  GEVO_OP_SELECT = 3,
  GEVO_OP_REDUCE = 4,  /* sub: GEVO_R_*; aux[0]=L, aux[1]=stride along axis */
  GEVO_OP_DOT = 5,     /* sub: GEVO_D_* for columns < aux[1]; aux[2] for the
                          rest; aux[0]=K */
  GEVO_OP_PAD = 6,     /* aux[d]=low[d], aux2[d]=input extent[d] */
  GEVO_OP_EXT = 7,     /* continuation record of the preceding DOT: a fused
                          elementwise epilogue (see below) */
  GEVO_OP_TAPSUM = 8   /* f64 sum of products: v = in0*in1, then v = v + x_t*y_t
                          for taps t = 1 .. aux2[5]-1, each product and sum
                          rounded on its own; (x_t, y_t) are the operands of
                          the aux2[4] EXT records that follow, 3 per record.
                          All x share in[0]'s strides, all y in[1]'s.
                          aux2[3] = M <= 3 epilogue micro-ops applied before
                          the store: aux[m] = GEVO_B_* | left << 4, operand m
                          = EXT operand 2*(taps-1) + m (its own strides). */
};

/* Dot epilogues.  A DOT whose aux2[0] = E > 0 is followed by E GEVO_OP_EXT
 * records.  Together they describe up to 4*E micro-ops applied, in order, to
 * every output element before it is stored to the DOT's `out` operand:
 *   ext.in[0..2]   extra operands, addressed with the output (i, j) index;
 *   ext.aux[0..5], ext.aux2[0..5]: four micro-ops of three words each:
 *     w0 = class | sub << 4 | kin << 8 | kout << 12   (class: UNARY, BINARY,
 *          SELECT as above)
 *     w1 = src_a | src_b << 8,  w2 = src_c
 *   sources: 0 = the dot value, 1 + 3*e + k = operand k of ext record e,
 *            64 + m = result of micro-op m.  The last micro-op is stored.
 * Each micro-op rounds exactly like the standalone instruction it replaces,
 * so fusion never changes a result bit. */
#define GEVO_EPI_SRC_OP 64
enum { GEVO_U_NEG = 0, GEVO_U_EXP, GEVO_U_LOG, GEVO_U_COPY, GEVO_U_CVT };
enum {
  GEVO_B_ADD = 0, GEVO_B_SUB, GEVO_B_MUL, GEVO_B_DIV, GEVO_B_MAX,
  GEVO_B_EQ, GEVO_B_NE, GEVO_B_LT, GEVO_B_LE, GEVO_B_GT, GEVO_B_GE
};
/* summation orders reproduced from numpy */
enum { GEVO_R_SUM_PAIRWISE = 0, GEVO_R_SUM_SEQ = 1, GEVO_R_MAX = 2 };
enum {
  GEVO_D_FMA_CHAIN = 0,   /* acc = fma(a_k, b_k, acc), k ascending, acc0 = 0 */
  GEVO_D_ACC8_TREE = 1,   /* 8 lane accumulators (k mod 8), pairwise tree */
  GEVO_D_SEQ_NOFMA = 2,   /* numpy's own loop: acc += a_k * b_k (rounded) */
  GEVO_D_ACC8_TAIL = 3    /* 8 lanes over k < K&~7, tree, then fma tail */
};

typedef struct {
  int32_t buf;
  int32_t off;
  int32_t st[GEVO_MAXR];
} gevo_operand;                       /* 32 bytes */

typedef struct {
  int32_t op, sub, kout, kin;
  int32_t rank, n;                    /* output rank, element count */
  int32_t shp[GEVO_MAXR];             /* output shape */
  int32_t aux[GEVO_MAXR];
  int32_t aux2[GEVO_MAXR];
  gevo_operand out;                   /* out.st: the numpy layout of the result */
  gevo_operand in[3];
} gevo_instr;                         /* 224 bytes */

/* gevo_prog.flags */
/* bits 0..1: which program each training step runs.  The weights' numpy
 * layouts can change from step to step (a mutated train_step may return a
 * transposed or broadcast view), and every program is lowered for the
 * layouts it reads; the lowering follows the layouts to their cycle
 * (plan.lower_variant) and a variant whose cycle does not fit these four is
 * refused (plan.UnsupportedVariant), never approximated.  Step 0 always runs
 * train0 (C-ordered initial weights). */
#define GEVO_SCHED_MASK 3
#define GEVO_SCHED_STEADY1 0          /* steps >= 1: train1 */
#define GEVO_SCHED_STEADY2 1          /* step 1: train1; steps >= 2: train2 */
#define GEVO_SCHED_ALT01 2            /* steps >= 1: odd -> train1, even -> train0 */
#define GEVO_SCHED_ALT12 3            /* steps >= 1: odd -> train1, even -> train2 */
#define GEVO_FLAG_ALTERNATE GEVO_SCHED_ALT01   /* (plan version 1 name) */
/* In-place weights (training, GEVO_SCHED_STEADY1 only): bit w of
 * (flags >> GEVO_FLAG_INPLACE_SHIFT) & 0x3F set means weight w is updated in
 * place by train1 -- it lives in block 0 of the individual's weight
 * ping-pong from step 0 on (step 0 reads the shared initial weights and
 * writes block 0; later steps read and write block 0).  The lowering proves
 * it safe (plan.inplace_weights): one instruction writes the return, reading
 * the parameter only at the words it overwrites, and nothing after it reads
 * the parameter.  Halves the weights' HBM/L2 footprint (w1: 200 KB). */
#define GEVO_FLAG_INPLACE_SHIFT 2
#define GEVO_FLAG_INPLACE(f) (((f) >> GEVO_FLAG_INPLACE_SHIFT) & 0x3F)
/* Score parts (prediction mode only): an individual's scored batches are
 * independent (fitness.py:361-368), so n_parts programs may share one
 * result_slot, part j scoring batches j, j + n_parts, ...  gevo_eval merges
 * them into results[result_slot] with integer sums (bit-exact). */
#define GEVO_FLAG_PART_SHIFT 8        /* bits 8..19: this program's part */
#define GEVO_FLAG_NPARTS_SHIFT 20     /* bits 20..30: parts of its individual (0 = 1) */
#define GEVO_FLAG_PART(f) (((f) >> GEVO_FLAG_PART_SHIFT) & 0xFFF)
#define GEVO_FLAG_NPARTS(f) ((((f) >> GEVO_FLAG_NPARTS_SHIFT) & 0x7FF) ? (((f) >> GEVO_FLAG_NPARTS_SHIFT) & 0x7FF) : 1)

typedef struct {
  int32_t train0, train0_n;           /* @train_step, step 0 */
  int32_t train1, train1_n;           /* @train_step, steps >= 1 */
  int32_t fwd, fwd_n;                 /* @forward */
  int32_t const_off;                  /* element offset into the const pool */
  int32_t result_slot;                /* where this individual's result goes */
  int64_t arena_off;                  /* element offset of [arena|w0|w1] */
  int32_t arena_elems;                /* scratch elements (before weights) */
  int32_t flags;
  int32_t param_off[GEVO_MAXP];       /* exec-once: offsets into params blob */
  int32_t out_off[GEVO_MAXP];         /* exec-once: offsets into outs blob */
  int32_t train2, train2_n;           /* @train_step for a third layout (GEVO_SCHED_*) */
} gevo_prog;                          /* 120 bytes */

typedef struct {
  uint32_t magic, version;
  int32_t n_instr, n_prog, n_const;
  int32_t weight_elems;               /* per-individual weight block */
  int32_t n_weights;                  /* weight arrays (returns of train_step) */
  int32_t wofs[GEVO_MAXP];            /* offsets of each weight in the block */
  int32_t max_arena;                  /* largest arena_elems of any prog */
  int32_t max_smem;                   /* largest shared-memory scratch (elements) */
  int64_t total_elems;                /* device elements for all individuals */
} gevo_plan_header;                   /* 80 bytes */

#endif
