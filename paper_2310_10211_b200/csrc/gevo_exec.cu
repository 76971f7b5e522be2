// gevo_exec.cu -- the population executor: one CTA runs one individual's
// whole fitness evaluation (600 train steps + scoring) inside ONE launch.
//
// Replaces, per individual, the reference hot loop
//   for step in range(steps): weights = plan.run(weights + [xb, yb])
//   (fitness.py:344-349 -> interpreter.py:219-225)
// and the scorer (fitness.py:355-369).  The variant program is an
// instruction table (include/gevo_plan.h) walked by all threads of the CTA
// with a CTA barrier between instructions; weights ping-pong between two
// per-individual HBM blocks so a step never overwrites its own inputs (the
// reference may return a parameter unchanged, genome.py:471-478).
#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
// This file is compiled twice (build.py): GEVO_TC_MODE 0 is the float64
// parity executor; GEVO_TC_MODE 1 (gevo_exec_tc.cu) is the same executor
// with every f64 DOT on tcgen05 (dot_tc.cuh), as separate kernels and
// launchers (`*_tc`).  Keeping the tensor-core path out of the float64
// build keeps its register allocation: adding the dot_tc call to the one
// kernel raised the spills of every DMMA dot path and cost ~30 % of the
// parity mode's speed (measured).
#ifndef GEVO_TC_MODE
#define GEVO_TC_MODE 0
#endif
#if GEVO_TC_MODE
#define GEVO_KNAME(x) x##_tc
#else
#define GEVO_KNAME(x) x
#endif
#include "gevo_plan.h"
#include "exec_core.cuh"
#include "exp_np.cuh"
#include "gevo_exec.cuh"

namespace gevo {

constexpr int kThreads = 256;   // 8 warps; 2 CTAs/SM (128 registers)
#ifndef GEVO_MIN_BLOCKS
#define GEVO_MIN_BLOCKS 2   // CTAs per SM the register budget is sized for
#endif
constexpr int kInstrCache = 64;   // instructions staged in shared memory

// a dot's fused elementwise epilogue, decoded once per instruction into
// shared memory (gevo_plan.h, "Dot epilogues")
constexpr int kEpiOps = 8, kEpiExt = 6;
constexpr int kEpiPre = 2;   // epilogue operands prefetched per output element
struct EpiDev {
  int nops;
  int op[kEpiOps][4];          // class, sub, kin, kout
  int src[kEpiOps][3];
  int next;                    // extra operands actually read
  int fast;                    // 0 generic, 1 f64 binary chain, 2 select
  int fsub[kEpiOps];           // fast chain: binary sub-op per micro-op
  int fleft[kEpiOps];          // fast chain: dot value is the left operand
  const double* ptr[kEpiExt];  // operand base + offset
  int64_t st0[kEpiExt], st1[kEpiExt];
};

// tensor-core (tcgen05, tf32 mode) state of a CTA: TMEM columns and the
// two staging mbarriers (dot_tc.cuh)
struct TcState {
  uint32_t tmem;
  uint32_t ph;                        // bit b: parity of the next wait on stage b
  uint32_t pending;                   // bit b: a commit on stage b not yet waited for
  uint32_t tph;                       // bit b: parity of the next TMA wait on stage b
  __align__(8) uint64_t mbar[2];      // MMA commits (stage free again)
  __align__(8) uint64_t tbar[2];      // TMA transactions (stage's A chunk landed)
  const void* tmap;                   // the launch's tensor map (param space), or null
  const double* tx64;                 // the f64 x it mirrors
  int64_t trows;
  int tcols;
};

struct Shared {
  double* base[GEVO_NBUF];
  int flag;
  int wrong;
  EpiDev epi;
  int tc_on;                          // DOTs on tcgen05 (GEVO_B200_DTYPE=tf32)
  TcState tc;
  unsigned long long* prof;           // nullable: profile counters (dot_tc phases)
};

__device__ __forceinline__ double* opptr(const Shared& S, const gevo_operand& o) {
  return S.base[o.buf];
}

// ---------------------------------------------------------------------------
// elementwise (UNARY / BINARY / SELECT)
//
// The op is resolved once per instruction into a functor; the element loop
// is then specialised per functor and per addressing class: every operand
// linear/scalar (index math free) or some operand strided (unravel).  Each
// thread keeps kEwUnroll independent elements in flight for memory-level
// parallelism.
// ---------------------------------------------------------------------------
constexpr int kEwUnroll = 4;

struct FAdd { __device__ double operator()(double a, double b, double) const { return __dadd_rn(a, b); } };
struct FSub { __device__ double operator()(double a, double b, double) const { return __dsub_rn(a, b); } };
struct FMul { __device__ double operator()(double a, double b, double) const { return __dmul_rn(a, b); } };
struct FDiv { __device__ double operator()(double a, double b, double) const { return __ddiv_rn(a, b); } };
struct FMax { __device__ double operator()(double a, double b, double) const { return np_fmax(a, b); } };
struct FGt { __device__ double operator()(double a, double b, double) const { return as_w(a > b); } };
struct FNeg { __device__ double operator()(double a, double, double) const { return -a; } };
struct FExp { __device__ double operator()(double a, double, double) const { return exp_np(a); } };
struct FCopy { __device__ double operator()(double a, double, double) const { return a; } };
struct FSel { __device__ double operator()(double p, double t, double f) const { return as_i64(p) != 0 ? t : f; } };
struct FBinGeneric {   // any kind / compare: runtime sub
  int sub, kin;
  __device__ double operator()(double a, double b, double) const { return apply_binary(sub, kin, a, b); }
};
struct FUnGeneric {
  int sub, kin, kout;
  __device__ double operator()(double a, double, double) const { return apply_unary(sub, kin, kout, a); }
};

// One elementwise instruction, read straight from the (shared-memory cached)
// record: addressing per operand from aux2 (AM_LINEAR / AM_SCALAR: address
// off + i*step; otherwise rank <= 2 walked as (row, col) incrementally, or a
// generic unravel).  One out-of-line instance per functor.
template <int NIN, class F>
__device__ __noinline__ void ew_instr(const Shared& S, const gevo_instr& I, F f) {
  const int n = I.n;
  const gevo_operand* ops[4] = {&I.out, &I.in[0], &I.in[1], &I.in[2]};
  double* out = S.base[I.out.buf];
  const double* in0 = S.base[I.in[0].buf];
  const double* in1 = NIN > 1 ? S.base[I.in[1].buf] : in0;
  const double* in2 = NIN > 2 ? S.base[I.in[2].buf] : in0;
  int off[4], step[4];
  bool strided = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int am = k <= NIN ? I.aux2[k] : AM_SCALAR;
    off[k] = k <= NIN ? ops[k]->off : 0;
    step[k] = am == AM_LINEAR ? 1 : 0;
    strided |= am == AM_STRIDED;
  }
  if (!strided) {
    for (int base = threadIdx.x; base < n; base += kEwUnroll * kThreads) {
      double a[kEwUnroll], b[kEwUnroll], c[kEwUnroll];
#pragma unroll
      for (int u = 0; u < kEwUnroll; ++u) {
        const int i = base + u * kThreads;
        if (i < n) {
          a[u] = in0[off[1] + i * step[1]];
          if (NIN > 1) b[u] = in1[off[2] + i * step[2]];
          if (NIN > 2) c[u] = in2[off[3] + i * step[3]];
        }
      }
#pragma unroll
      for (int u = 0; u < kEwUnroll; ++u) {
        const int i = base + u * kThreads;
        if (i < n) out[off[0] + i * step[0]] = f(a[u], NIN > 1 ? b[u] : 0.0, NIN > 2 ? c[u] : 0.0);
      }
    }
    return;
  }
  const int rank = I.rank;
  if (rank <= 2) {
    int sr[4], sc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      sr[k] = k <= NIN && rank == 2 ? ops[k]->st[0] : 0;
      sc[k] = k <= NIN && rank >= 1 ? ops[k]->st[rank - 1] : 0;
    }
    const int C = rank == 2 ? I.shp[1] : (rank == 1 ? I.shp[0] : 1);
    const int q = kThreads / C, rm = kThreads - q * C;
    int r = threadIdx.x / C, c = threadIdx.x - r * C;
    for (int base = threadIdx.x; base < n; base += kEwUnroll * kThreads) {
      double a[kEwUnroll], b[kEwUnroll], x[kEwUnroll];
      int ao[kEwUnroll];
#pragma unroll
      for (int u = 0; u < kEwUnroll; ++u) {
        if (base + u * kThreads < n) {
          ao[u] = off[0] + r * sr[0] + c * sc[0];
          a[u] = in0[off[1] + r * sr[1] + c * sc[1]];
          if (NIN > 1) b[u] = in1[off[2] + r * sr[2] + c * sc[2]];
          if (NIN > 2) x[u] = in2[off[3] + r * sr[3] + c * sc[3]];
        }
        c += rm;
        r += q;
        if (c >= C) { c -= C; ++r; }
      }
#pragma unroll
      for (int u = 0; u < kEwUnroll; ++u)
        if (base + u * kThreads < n) out[ao[u]] = f(a[u], NIN > 1 ? b[u] : 0.0, NIN > 2 ? x[u] : 0.0);
    }
    return;
  }
  // rank 3..6: the thread's multi-index advances by kThreads in the shape's
  // mixed radix (digit add with carry) -- no division per element
  int idx[GEVO_MAXR], dig[GEVO_MAXR], shp[GEVO_MAXR], st[4][GEVO_MAXR];
  unravel(threadIdx.x, rank, I.shp, idx);
  unravel(kThreads, rank, I.shp, dig);
  // strides and shape into registers: stores through `out` may alias the
  // (shared-memory) instruction record, which would force reloads
#pragma unroll
  for (int d = 0; d < GEVO_MAXR; ++d) {
    shp[d] = I.shp[d];
#pragma unroll
    for (int k = 0; k < 4; ++k) st[k][d] = k <= NIN ? ops[k]->st[d] : 0;
  }
  constexpr int U = 4;
  for (int base = threadIdx.x; base < n; base += U * kThreads) {
    int ao[U];
    double a[U], b[U], c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * kThreads < n) {
        int ad[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          int v = off[k];
          if (k <= NIN) {
#pragma unroll
            for (int d = 0; d < GEVO_MAXR; ++d)
              if (d < rank) v += idx[d] * st[k][d];
          }
          ad[k] = v;
        }
        ao[u] = ad[0];
        a[u] = in0[ad[1]];
        if (NIN > 1) b[u] = in1[ad[2]];
        if (NIN > 2) c[u] = in2[ad[3]];
      }
      int carry = 0;
#pragma unroll
      for (int d = GEVO_MAXR - 1; d >= 0; --d) {
        if (d < rank) {
          int v = idx[d] + dig[d] + carry;
          carry = v >= shp[d];
          idx[d] = carry ? v - shp[d] : v;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * kThreads < n) out[ao[u]] = f(a[u], NIN > 1 ? b[u] : 0.0, NIN > 2 ? c[u] : 0.0);
  }
}

__device__ __forceinline__ void run_elementwise(const Shared& S, const gevo_instr& I) {
  const int op = I.op, kin = I.kin, sub = I.sub;
  if (op == GEVO_OP_SELECT) { ew_instr<3>(S, I, FSel()); return; }
  if (op == GEVO_OP_UNARY) {
    if (sub == GEVO_U_COPY) { ew_instr<1>(S, I, FCopy()); return; }
    if (kin == GEVO_K_F64 && sub == GEVO_U_EXP) { ew_instr<1>(S, I, FExp()); return; }
    if (kin == GEVO_K_F64 && sub == GEVO_U_NEG) { ew_instr<1>(S, I, FNeg()); return; }
    ew_instr<1>(S, I, FUnGeneric{sub, kin, I.kout});
    return;
  }
  if (kin == GEVO_K_F64) {
    switch (sub) {
      case GEVO_B_ADD: ew_instr<2>(S, I, FAdd()); return;
      case GEVO_B_SUB: ew_instr<2>(S, I, FSub()); return;
      case GEVO_B_MUL: ew_instr<2>(S, I, FMul()); return;
      case GEVO_B_DIV: ew_instr<2>(S, I, FDiv()); return;
      case GEVO_B_MAX: ew_instr<2>(S, I, FMax()); return;
      case GEVO_B_GT: ew_instr<2>(S, I, FGt()); return;
    }
  }
  ew_instr<2>(S, I, FBinGeneric{sub, kin});
}

__device__ __noinline__ void run_pad(const Shared& S, const gevo_instr& I) {
  double* out = opptr(S, I.out);
  const double* in = opptr(S, I.in[0]);
  const double pv = opptr(S, I.in[1])[I.in[1].off];
  if (I.rank <= 2) {
    // (r, c) walked incrementally; rank 1 is one row
    const bool two = I.rank == 2;
    const int C = two ? I.shp[1] : (I.rank == 1 ? I.shp[0] : 1);
    const int lo0 = two ? I.aux[0] : 0, lo1 = I.rank >= 1 ? I.aux[I.rank - 1] : 0;
    const int ex0 = two ? I.aux2[0] : 1, ex1 = I.rank >= 1 ? I.aux2[I.rank - 1] : 1;
    const int is0 = two ? I.in[0].st[0] : 0, is1 = I.rank >= 1 ? I.in[0].st[I.rank - 1] : 0;
    const int os0 = two ? I.out.st[0] : 0, os1 = I.rank >= 1 ? I.out.st[I.rank - 1] : 0;
    const int q = kThreads / C, rm = kThreads - q * C;
    int r = threadIdx.x / C, c = threadIdx.x - (threadIdx.x / C) * C;
    for (int i = threadIdx.x; i < I.n; i += kThreads) {
      const int j0 = r - lo0, j1 = c - lo1;
      const bool inside = j0 >= 0 && j0 < ex0 && j1 >= 0 && j1 < ex1;
      out[I.out.off + r * os0 + c * os1] = inside ? in[I.in[0].off + j0 * is0 + j1 * is1] : pv;
      c += rm;
      r += q;
      if (c >= C) { c -= C; ++r; }
    }
    return;
  }
  int idx[GEVO_MAXR], dig[GEVO_MAXR], shp[GEVO_MAXR], lo[GEVO_MAXR], ex[GEVO_MAXR], is[GEVO_MAXR],
      os[GEVO_MAXR];
  const int rank = I.rank, n = I.n, ioff = I.in[0].off, ooff = I.out.off;
  unravel(threadIdx.x, rank, I.shp, idx);
  unravel(kThreads, rank, I.shp, dig);
#pragma unroll
  for (int d = 0; d < GEVO_MAXR; ++d) {   // registers (stores may alias the record)
    shp[d] = I.shp[d];
    lo[d] = I.aux[d];
    ex[d] = I.aux2[d];
    is[d] = I.in[0].st[d];
    os[d] = I.out.st[d];
  }
  // U elements per thread in flight: the loads of all U first, then the stores
  constexpr int U = 4;
  for (int base = threadIdx.x; base < n; base += U * kThreads) {
    int dsts[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool inside = true;
      int src = ioff, dst = ooff;
#pragma unroll
      for (int d = 0; d < GEVO_MAXR; ++d) {
        if (d < rank) {
          const int j = idx[d] - lo[d];
          inside = inside && j >= 0 && j < ex[d];
          src += j * is[d];
          dst += idx[d] * os[d];
        }
      }
      dsts[u] = dst;
      v[u] = pv;
      if (inside && base + u * kThreads < n) v[u] = in[src];
      int carry = 0;
#pragma unroll
      for (int d = GEVO_MAXR - 1; d >= 0; --d) {
        if (d < rank) {
          const int w = idx[d] + dig[d] + carry;
          carry = w >= shp[d];
          idx[d] = carry ? w - shp[d] : w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * kThreads < n) out[dsts[u]] = v[u];
  }
}

__device__ __noinline__ void run_reduce(const Shared& S, const gevo_instr& I) {
  double* out = opptr(S, I.out);
  const double* in = opptr(S, I.in[0]);
  // the record's fields into registers (stores may alias it)
  const int L = I.aux[0], n = I.n, rank = I.rank, kin = I.kin, sub = I.sub;
  const int64_t rs = I.aux[1];
  int shp[GEVO_MAXR], ist[GEVO_MAXR], ost[GEVO_MAXR];
#pragma unroll
  for (int d = 0; d < GEVO_MAXR; ++d) {
    shp[d] = I.shp[d];
    ist[d] = I.in[0].st[d];
    ost[d] = I.out.st[d];
  }
  const int ioff = I.in[0].off, ooff = I.out.off;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int idx[GEVO_MAXR];
    unravel(i, rank, shp, idx);
    int src = ioff, dst = ooff;
#pragma unroll
    for (int d = 0; d < GEVO_MAXR; ++d) {
      if (d < rank) {
        src += idx[d] * ist[d];
        dst += idx[d] * ost[d];
      }
    }
    const double* p = in + src;
    double r;
    if (kin == GEVO_K_F64) {
      if (sub == GEVO_R_MAX) {
        r = p[0];
        for (int k = 1; k < L; ++k) r = np_fmax(r, p[k * rs]);
      } else if (sub == GEVO_R_SUM_PAIRWISE) {
        r = pairwise_sum(p, L, rs);
      } else {
        r = 0.0;
        for (int k = 0; k < L; ++k) r = __dadd_rn(r, p[k * rs]);
      }
    } else {
      int64_t v;
      if (sub == GEVO_R_MAX) {
        v = as_i64(p[0]);
        for (int k = 1; k < L; ++k) { int64_t x = as_i64(p[k * rs]); v = x > v ? x : v; }
      } else {
        uint64_t acc = 0;
        for (int k = 0; k < L; ++k) acc += (uint64_t)as_i64(p[k * rs]);
        v = (int64_t)acc;
      }
      r = as_w(v);
    }
    out[dst] = r;
  }
}

// fused dot epilogues (the DOT itself: dot_staged.cuh)

// decode the EXT records following a DOT (thread 0; caller syncs)
__device__ void decode_epilogue(Shared& S, const gevo_instr* ext, int n_ext, int nops) {
  EpiDev& e = S.epi;
  e.nops = nops;
  int used = 0;
  for (int m = 0; m < nops; ++m) {
    const gevo_instr& X = ext[m >> 2];
    const int q = m & 3;
    const int w0 = q < 2 ? X.aux[3 * q] : X.aux2[3 * q - 6];
    const int w1 = q < 2 ? X.aux[3 * q + 1] : X.aux2[3 * q - 5];
    const int w2 = q < 2 ? X.aux[3 * q + 2] : X.aux2[3 * q - 4];
    e.op[m][0] = w0 & 15;
    e.op[m][1] = (w0 >> 4) & 15;
    e.op[m][2] = (w0 >> 8) & 15;
    e.op[m][3] = (w0 >> 12) & 15;
    e.src[m][0] = w1 & 255;
    e.src[m][1] = (w1 >> 8) & 255;
    e.src[m][2] = w2;
    const int nsrc = e.op[m][0] == GEVO_OP_UNARY ? 1 : (e.op[m][0] == GEVO_OP_BINARY ? 2 : 3);
    for (int k = 0; k < nsrc; ++k)
      if (e.src[m][k] >= 1 && e.src[m][k] < GEVO_EPI_SRC_OP) used = max(used, e.src[m][k]);
  }
  e.next = used;
  // fast paths: (1) each micro-op is an f64 add/sub/mul/div/max of the
  // running value with ext operand m (in order); (2) one select(ext0, v, ext1)
  // or select(ext0, ext1, v)
  bool chain = nops <= kEpiPre;
  for (int m = 0; m < nops && chain; ++m) {
    const int prev = m == 0 ? 0 : GEVO_EPI_SRC_OP + m - 1;
    chain = e.op[m][0] == GEVO_OP_BINARY && e.op[m][2] == GEVO_K_F64 && e.op[m][1] <= GEVO_B_MAX;
    if (chain && e.src[m][0] == prev && e.src[m][1] == m + 1) e.fleft[m] = 1;
    else if (chain && e.src[m][1] == prev && e.src[m][0] == m + 1) e.fleft[m] = 0;
    else chain = false;
    e.fsub[m] = e.op[m][1];
  }
  e.fast = chain ? 1 : 0;
  if (!chain && nops == 1 && e.op[0][0] == GEVO_OP_SELECT && e.src[0][0] == 1 &&
      ((e.src[0][1] == 0 && e.src[0][2] == 2) || (e.src[0][1] == 2 && e.src[0][2] == 0))) {
    e.fast = 2;
    e.fleft[0] = e.src[0][1] == 0;   // dot value is the "then" branch
  }
  for (int x = 0; x < kEpiExt; ++x) {
    if (x < 3 * n_ext) {
      const gevo_operand& o = ext[x / 3].in[x % 3];
      e.ptr[x] = S.base[o.buf] + o.off;
      e.st0[x] = o.st[0];
      e.st1[x] = o.st[1];
    } else {
      e.ptr[x] = nullptr;
    }
  }
}

// prefetch the first kEpiPre epilogue operands of output (r, c) into ev[]
__device__ __forceinline__ void epi_fetch(const EpiDev& e, int64_t r, int64_t c, double* ev) {
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x)
    ev[x] = x < e.next ? e.ptr[x][r * e.st0[x] + c * e.st1[x]] : 0.0;
}

__device__ __forceinline__ double bin_f64(int sub, double a, double b) {
  switch (sub) {
    case GEVO_B_ADD: return __dadd_rn(a, b);
    case GEVO_B_SUB: return __dsub_rn(a, b);
    case GEVO_B_MUL: return __dmul_rn(a, b);
    case GEVO_B_DIV: return __ddiv_rn(a, b);
    default: return np_fmax(a, b);
  }
}

// generic epilogue: any micro-op sequence (kept out of line so the dot's
// hot loops do not carry its registers)
__device__ __noinline__ double epilogue_generic(const EpiDev& e, const double* ev, double v,
                                                int64_t r, int64_t c) {
  double vals[kEpiOps + 1];
  vals[0] = v;
  for (int m = 0; m < e.nops; ++m) {
    double a[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int s = e.src[m][k];
      if (s == 0) a[k] = vals[0];
      else if (s >= GEVO_EPI_SRC_OP) a[k] = vals[1 + s - GEVO_EPI_SRC_OP];
      else if (s == 1) a[k] = ev[0];
      else if (s == 2) a[k] = ev[1];
      else a[k] = e.ptr[s - 1][r * e.st0[s - 1] + c * e.st1[s - 1]];
    }
    const int cls = e.op[m][0];
    double res;
    if (cls == GEVO_OP_UNARY) res = apply_unary(e.op[m][1], e.op[m][2], e.op[m][3], a[0]);
    else if (cls == GEVO_OP_BINARY) res = apply_binary(e.op[m][1], e.op[m][2], a[0], a[1]);
    else res = as_i64(a[0]) != 0 ? a[1] : a[2];
    vals[m + 1] = res;
  }
  return vals[e.nops];
}

// epilogue kinds the dot kernels are specialised for
enum { EK_NONE = 0, EK_CHAIN = 1, EK_SELECT = 2, EK_GENERIC = 3 };

// apply the decoded epilogue to dot value v at (r, c); operands below
// kEpiPre come prefetched in ev[], the rest are loaded here
template <int EK>
__device__ __forceinline__ double epilogue_k(const EpiDev& e, const double* ev, double v,
                                             int64_t r, int64_t c) {
  if (EK == EK_NONE) return v;
  if (EK == EK_CHAIN) {
#pragma unroll
    for (int m = 0; m < kEpiPre; ++m)
      if (m < e.nops) v = e.fleft[m] ? bin_f64(e.fsub[m], v, ev[m]) : bin_f64(e.fsub[m], ev[m], v);
    return v;
  }
  if (EK == EK_SELECT) {
    const bool p = as_i64(ev[0]) != 0;
    return e.fleft[0] ? (p ? v : ev[1]) : (p ? ev[1] : v);
  }
  return epilogue_generic(e, ev, v, r, c);
}

__device__ __forceinline__ double epilogue(const EpiDev& e, const double* ev, double v,
                                           int64_t r, int64_t c) {
  if (e.fast == 1) return epilogue_k<EK_CHAIN>(e, ev, v, r, c);
  if (e.fast == 2) return epilogue_k<EK_SELECT>(e, ev, v, r, c);
  return epilogue_generic(e, ev, v, r, c);
}

// An elementwise instruction with a fused chain (lowering.fuse_ew_chains):
// the instruction's own op, then the decoded micro-ops on each element, one
// store.  rank <= 2; element i = (r, c) of the output, operands addressed by
// their (r, c) strides (rank 1: one row).  EXT records follow the
// instruction (aux2[4] of them, aux2[5] micro-ops).
// fast form: an f64 binary op followed by <= 2 f64 binary micro-ops, micro-op
// m combining the running value with EXT operand m + 1 (b1 - lr * g and the
// like).  Every thread decodes the one EXT record into registers: no
// shared-memory decode, no extra barrier.  Returns false for any other chain.
__device__ __forceinline__ bool ew_chain_fast(const Shared& S, const gevo_instr& I) {
  const int nops = I.aux2[5];
  if (I.op != GEVO_OP_BINARY || I.kin != GEVO_K_F64 || I.sub > GEVO_B_MAX || nops > 2)
    return false;
  const gevo_instr& X = (&I)[1];
  int fsub[2] = {0, 0}, fleft[2] = {0, 0};
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    if (m >= nops) break;
    const int w0 = X.aux[3 * m], w1 = X.aux[3 * m + 1];
    const int cls = w0 & 15, sub = (w0 >> 4) & 15, kin = (w0 >> 8) & 15;
    const int s0 = w1 & 255, s1 = (w1 >> 8) & 255;
    const int prev = m == 0 ? 0 : GEVO_EPI_SRC_OP + m - 1;
    if (cls != GEVO_OP_BINARY || kin != GEVO_K_F64 || sub > GEVO_B_MAX) return false;
    if (s0 == prev && s1 == m + 1) fleft[m] = 1;
    else if (s1 == prev && s0 == m + 1) fleft[m] = 0;
    else return false;
    fsub[m] = sub;
  }
  const int n = I.n, rank = I.rank, sub = I.sub;
  const int C = rank == 2 ? I.shp[1] : (rank == 1 ? I.shp[0] : 1);
  auto st0 = [&](const gevo_operand& o) { return rank == 2 ? o.st[0] : 0; };
  auto st1 = [&](const gevo_operand& o) { return rank == 2 ? o.st[1] : (rank == 1 ? o.st[0] : 0); };
  double* out = S.base[I.out.buf] + I.out.off;
  const double* a = S.base[I.in[0].buf] + I.in[0].off;
  const double* b = S.base[I.in[1].buf] + I.in[1].off;
  const int o0 = st0(I.out), o1 = st1(I.out), a0 = st0(I.in[0]), a1 = st1(I.in[0]);
  const int b0 = st0(I.in[1]), b1 = st1(I.in[1]);
  // EXT operands are (r, c) views already (lowering._as2d)
  const double* e0 = S.base[X.in[0].buf] + X.in[0].off;
  const double* e1 = nops > 1 ? S.base[X.in[1].buf] + X.in[1].off : e0;
  const int e00 = X.in[0].st[0], e01 = X.in[0].st[1];
  const int e10 = nops > 1 ? X.in[1].st[0] : 0, e11 = nops > 1 ? X.in[1].st[1] : 0;
  for (int i = threadIdx.x; i < n; i += kThreads) {
    const int r = i / C, c = i - r * C;
    const double x0 = e0[r * e00 + c * e01];
    const double x1 = nops > 1 ? e1[r * e10 + c * e11] : 0.0;
    double v = bin_f64(sub, a[r * a0 + c * a1], b[r * b0 + c * b1]);
    v = fleft[0] ? bin_f64(fsub[0], v, x0) : bin_f64(fsub[0], x0, v);
    if (nops > 1) v = fleft[1] ? bin_f64(fsub[1], v, x1) : bin_f64(fsub[1], x1, v);
    out[r * o0 + c * o1] = v;
  }
  return true;
}

// rank 3..6 chains (always the fast form, lowering._fast_form): the output's
// multi-index advances by kThreads in mixed radix (as ew_instr's N-d walk) and
// every operand -- the op's two inputs and the EXT operands -- is addressed by
// its own full strides.
//
// Channel form: when every operand is C-ordered, a scalar, or a last-dim
// (per-channel) broadcast -- the CNN's folded batch norm, x * scale[c] +
// bias[c] then max(., 0) -- element i is at i, at 0, or at i mod C, and the
// walk is a running channel index instead of the N-d digits.
__device__ __forceinline__ int chan_kind(const gevo_operand& o, const gevo_instr& I) {
  int cst = 1;
  bool lin = true, scal = true, chan = true;
  for (int d = I.rank - 1; d >= 0; --d) {
    const int e = I.shp[d], st = o.st[d];
    if (e != 1) {
      lin &= st == cst;
      scal &= st == 0;
      chan &= d == I.rank - 1 ? st == 1 : st == 0;
    }
    cst *= e;
  }
  return lin ? 0 : (scal ? 1 : (chan ? 2 : -1));
}

__device__ __noinline__ bool ew_chain_chan(const Shared& S, const gevo_instr& I, const int* fsub,
                                           const int* fleft) {
  const gevo_instr& X = (&I)[1];
  const int nops = I.aux2[5], n = I.n, sub = I.sub, C = I.shp[I.rank - 1];
  const gevo_operand* ops[5] = {&I.out, &I.in[0], &I.in[1], &X.in[0], &X.in[1]};
  int kind[5];
  const double* p[5];
  for (int k = 0; k < 5; ++k) {
    const bool used = k < 3 || k - 3 < nops;
    kind[k] = used ? chan_kind(*ops[k], I) : 1;
    if (kind[k] < 0 || (k == 0 && kind[k] != 0)) return false;
    p[k] = S.base[ops[k]->buf] + (used ? ops[k]->off : 0);
  }
  double* out = S.base[I.out.buf] + I.out.off;
  constexpr int U = 2;
  int c0 = threadIdx.x % C;
  const int c1 = kThreads % C, cstep = (U * kThreads) % C;
  for (int base = threadIdx.x; base < n; base += U * kThreads) {
    double a[U], b[U], x0[U], x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * kThreads;
      int c = c0 + u * c1;
      if (c >= C) c -= C;
      int ad[5];
#pragma unroll
      for (int k = 1; k < 5; ++k) ad[k] = kind[k] == 0 ? i : (kind[k] == 2 ? c : 0);
      if (i < n) {
        a[u] = p[1][ad[1]];
        b[u] = p[2][ad[2]];
        x0[u] = p[3][ad[3]];
        x1[u] = nops > 1 ? p[4][ad[4]] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * kThreads;
      if (i < n) {
        double v = bin_f64(sub, a[u], b[u]);
        v = fleft[0] ? bin_f64(fsub[0], v, x0[u]) : bin_f64(fsub[0], x0[u], v);
        if (nops > 1) v = fleft[1] ? bin_f64(fsub[1], v, x1[u]) : bin_f64(fsub[1], x1[u], v);
        out[i] = v;
      }
    }
    c0 += cstep;
    if (c0 >= C) c0 -= C;
  }
  return true;
}

__device__ __noinline__ void ew_chain_nd(const Shared& S, const gevo_instr& I) {
  const gevo_instr& X = (&I)[1];
  const int nops = I.aux2[5], n = I.n, rank = I.rank, sub = I.sub;
  int fsub[2] = {0, 0}, fleft[2] = {1, 1};
  for (int m = 0; m < nops; ++m) {
    const int w0 = X.aux[3 * m], w1 = X.aux[3 * m + 1];
    fsub[m] = (w0 >> 4) & 15;
    fleft[m] = (w1 & 255) == (m == 0 ? 0 : GEVO_EPI_SRC_OP + m - 1);
  }
  if (ew_chain_chan(S, I, fsub, fleft)) return;
  const gevo_operand* ops[5] = {&I.out, &I.in[0], &I.in[1], &X.in[0], &X.in[1]};
  double* p[5];
  // the 5 operands' strides live in shared memory (broadcast reads): in
  // registers they spill
  __shared__ int st[5][GEVO_MAXR];
  int shp[GEVO_MAXR], idx[GEVO_MAXR], dig[GEVO_MAXR];
  if (threadIdx.x < 5 * GEVO_MAXR) {
    const int k = threadIdx.x / GEVO_MAXR, d = threadIdx.x % GEVO_MAXR;
    st[k][d] = (k < 3 || k - 3 < nops) && d < rank ? ops[k]->st[d] : 0;
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const bool used = k < 3 || k - 3 < nops;
    p[k] = S.base[ops[k]->buf] + (used ? ops[k]->off : 0);
  }
#pragma unroll
  for (int d = 0; d < GEVO_MAXR; ++d) shp[d] = I.shp[d];
  __syncthreads();
  unravel(threadIdx.x, rank, I.shp, idx);
  unravel(kThreads, rank, I.shp, dig);
  // U elements per thread in flight: all loads first, then the math and
  // the stores (memory-level parallelism, as ew_instr)
  constexpr int U = 2;
  for (int base = threadIdx.x; base < n; base += U * kThreads) {
    int ao[U];
    double a[U], b[U], x0[U], x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * kThreads < n) {
        int ad[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          int v = 0;
#pragma unroll
          for (int d = 0; d < GEVO_MAXR; ++d)
            if (d < rank) v += idx[d] * st[k][d];
          ad[k] = v;
        }
        ao[u] = ad[0];
        a[u] = p[1][ad[1]];
        b[u] = p[2][ad[2]];
        x0[u] = p[3][ad[3]];
        x1[u] = nops > 1 ? p[4][ad[4]] : 0.0;
      }
      int carry = 0;
#pragma unroll
      for (int d = GEVO_MAXR - 1; d >= 0; --d) {
        if (d < rank) {
          const int w = idx[d] + dig[d] + carry;
          carry = w >= shp[d];
          idx[d] = carry ? w - shp[d] : w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * kThreads < n) {
        double v = bin_f64(sub, a[u], b[u]);
        v = fleft[0] ? bin_f64(fsub[0], v, x0[u]) : bin_f64(fsub[0], x0[u], v);
        if (nops > 1) v = fleft[1] ? bin_f64(fsub[1], v, x1[u]) : bin_f64(fsub[1], x1[u], v);
        p[0][ao[u]] = v;
      }
    }
  }
}

__device__ __noinline__ void run_ew_chain(Shared& S, const gevo_instr& I) {
  if (I.rank > 2) {
    ew_chain_nd(S, I);
    return;
  }
  if (ew_chain_fast(S, I)) return;
  if (threadIdx.x == 0) decode_epilogue(S, &I + 1, I.aux2[4], I.aux2[5]);
  __syncthreads();
  const EpiDev& e = S.epi;
  const int n = I.n, rank = I.rank, op = I.op, sub = I.sub, kin = I.kin, kout = I.kout;
  const int C = rank == 2 ? I.shp[1] : (rank == 1 ? I.shp[0] : 1);
  const gevo_operand* ops[4] = {&I.out, &I.in[0], &I.in[1], &I.in[2]};
  const int nin = op == GEVO_OP_UNARY ? 1 : (op == GEVO_OP_BINARY ? 2 : 3);
  double* p[4];
  int s0[4], s1[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const gevo_operand& o = *ops[k];
    const bool used = k <= nin;
    p[k] = used ? S.base[o.buf] + o.off : S.base[0];
    s0[k] = used && rank == 2 ? o.st[0] : 0;
    s1[k] = used ? (rank == 2 ? o.st[1] : (rank == 1 ? o.st[0] : 0)) : 0;
  }
  for (int i = threadIdx.x; i < n; i += kThreads) {
    const int r = i / C, c = i - r * C;
    const double a = p[1][r * s0[1] + c * s1[1]];
    const double b = nin > 1 ? p[2][r * s0[2] + c * s1[2]] : 0.0;
    const double x = nin > 2 ? p[3][r * s0[3] + c * s1[3]] : 0.0;
    double v;
    if (op == GEVO_OP_UNARY) v = apply_unary(sub, kin, kout, a);
    else if (op == GEVO_OP_BINARY) v = apply_binary(sub, kin, a, b);
    else v = as_i64(a) != 0 ? b : x;
    double ev[kEpiPre];
    epi_fetch(e, r, c, ev);
    p[0][r * s0[0] + c * s1[0]] = epilogue(e, ev, v, r, c);
  }
}

}  // namespace gevo
#include "dot_staged.cuh"
#if GEVO_TC_MODE
#include "dot_tc.cuh"
#endif
namespace gevo {

__device__ __noinline__ void run_dot(Shared& S, const gevo_instr& I, double* stage) {
  const int n_ext = I.aux2[0];
  const EpiDev* epi = nullptr;
  if (n_ext > 0) {
    if (threadIdx.x == 0) decode_epilogue(S, &I + 1, n_ext, I.aux2[1]);
    __syncthreads();
    epi = &S.epi;
  }
  DotArgs d;
  d.A = opptr(S, I.in[0]) + I.in[0].off;
  d.B = opptr(S, I.in[1]) + I.in[1].off;
  d.sam = I.in[0].st[0];
  d.sak = I.in[0].st[1];
  d.sbk = I.in[1].st[0];
  d.sbn = I.in[1].st[1];
  d.a_smem = I.in[0].buf == GEVO_BUF_SMEM;
  d.b_smem = I.in[1].buf == GEVO_BUF_SMEM;
  d.out = opptr(S, I.out) + I.out.off;
  d.som = I.out.st[0];
  d.son = I.out.st[1];
  d.M = I.shp[0];
  d.K = I.aux[0];
  const int N = I.shp[1];
  const bool integer = I.kin != GEVO_K_F64;
#if GEVO_TC_MODE
  if (!integer) {                     // reduced-precision mode: every f64 dot on tcgen05
    if (S.tc_on == 2) dot_tc<true>(S.tc, d, 0, N, epi, stage, S.prof);   // bf16
    else dot_tc<false>(S.tc, d, 0, N, epi, stage, S.prof);            // tf32
    return;
  }
#endif
  const int split = integer ? N : min(I.aux[1], N);
  d.xrow = 1 << 30;
  dot_columns(d, 0, split, I.sub, integer, stage, epi);
  // aux[3] = 1 + first row of the edge corner (0: none), columns >= split
  if (I.aux[3] > 0) d.xrow = I.aux[3] - 1;
  dot_columns(d, split, N, I.aux[2], integer, stage, epi);
}

// GEVO_OP_TAPSUM (lowering.fuse_tap_sums; the CNN's depthwise 3x3): per
// output element, v = x0*y0, then v = v + xt*yt for each further tap, with
// the multiply and add roundings of the instructions it replaces.  The taps
// share their x strides and their y strides, so one N-d walk gives every
// tap's offset; the tap base pointers are read from shared memory.
constexpr int kTapMax = 9;
__device__ __noinline__ void run_tapsum(Shared& S, const gevo_instr& I) {
  const int ntap = I.aux2[5], n = I.n, rank = I.rank;
  __shared__ const double* tx[kTapMax];
  __shared__ const double* ty[kTapMax];
  __shared__ int sx[GEVO_MAXR], sy[GEVO_MAXR], so[GEVO_MAXR];
  // epilogue micro-ops (aux2[3] of them, <= 3): sub | left << 4 in aux[m],
  // operand m = EXT operand 2 * (ntap - 1) + m
  constexpr int kTapEpi = 3;
  const int nm = I.aux2[3];
  __shared__ const double* mp[kTapEpi];
  __shared__ int mst[kTapEpi][GEVO_MAXR];
  if (threadIdx.x >= 32 && threadIdx.x < 32 + kTapEpi * GEVO_MAXR) {
    const int m = (threadIdx.x - 32) / GEVO_MAXR, d = (threadIdx.x - 32) % GEVO_MAXR;
    const int e = 2 * (ntap - 1) + m;
    const gevo_operand& W = (&I)[1 + e / 3].in[e % 3];
    if (m < nm) {
      mst[m][d] = d < rank ? W.st[d] : 0;
      if (d == 0) mp[m] = S.base[W.buf] + W.off;
    } else {
      mst[m][d] = 0;
    }
  }
  if (threadIdx.x < ntap) {
    const int t = threadIdx.x;
    const int ex = 2 * (t - 1), ey = ex + 1;      // operand index among the EXT records
    const gevo_operand& X = t == 0 ? I.in[0] : (&I)[1 + ex / 3].in[ex % 3];
    const gevo_operand& Y = t == 0 ? I.in[1] : (&I)[1 + ey / 3].in[ey % 3];
    tx[t] = S.base[X.buf] + X.off;
    ty[t] = S.base[Y.buf] + Y.off;
  }
  if (threadIdx.x < GEVO_MAXR) {
    const int d = threadIdx.x;
    sx[d] = d < rank ? I.in[0].st[d] : 0;
    sy[d] = d < rank ? I.in[1].st[d] : 0;
    so[d] = d < rank ? I.out.st[d] : 0;
  }
  double* out = S.base[I.out.buf] + I.out.off;
  int idx[GEVO_MAXR], dig[GEVO_MAXR], shp[GEVO_MAXR];
#pragma unroll
  for (int d = 0; d < GEVO_MAXR; ++d) shp[d] = I.shp[d];
  unravel(threadIdx.x, rank, I.shp, idx);
  unravel(kThreads, rank, I.shp, dig);
  __syncthreads();
  int msub[kTapEpi], mleft[kTapEpi];
#pragma unroll
  for (int m = 0; m < kTapEpi; ++m) {
    msub[m] = I.aux[m] & 15;
    mleft[m] = (I.aux[m] >> 4) & 1;
  }
  constexpr int U = 2;
  for (int base = threadIdx.x; base < n; base += U * kThreads) {
    int ax[U], ay[U], ao[U], am[U][kTapEpi];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int a = 0, b = 0, c = 0, w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
      for (int d = 0; d < GEVO_MAXR; ++d)
        if (d < rank) {
          a += idx[d] * sx[d];
          b += idx[d] * sy[d];
          c += idx[d] * so[d];
          if (nm > 0) w0 += idx[d] * mst[0][d];
          if (nm > 1) w1 += idx[d] * mst[1][d];
          if (nm > 2) w2 += idx[d] * mst[2][d];
        }
      ax[u] = a;
      ay[u] = b;
      ao[u] = c;
      am[u][0] = w0;
      am[u][1] = w1;
      am[u][2] = w2;
      int carry = 0;
#pragma unroll
      for (int d = GEVO_MAXR - 1; d >= 0; --d) {
        if (d < rank) {
          const int w = idx[d] + dig[d] + carry;
          carry = w >= shp[d];
          idx[d] = carry ? w - shp[d] : w;
        }
      }
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = base + u * kThreads < n ? __dmul_rn(tx[0][ax[u]], ty[0][ay[u]]) : 0.0;
    for (int t = 1; t < ntap; ++t) {
      const double* px = tx[t];
      const double* py = ty[t];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (base + u * kThreads < n) v[u] = __dadd_rn(v[u], __dmul_rn(px[ax[u]], py[ay[u]]));
    }
#pragma unroll
    for (int m = 0; m < kTapEpi; ++m) {
      if (m < nm) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (base + u * kThreads < n) {
            const double w = mp[m][am[u][m]];
            v[u] = mleft[m] ? bin_f64(msub[m], v[u], w) : bin_f64(msub[m], w, v[u]);
          }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (base + u * kThreads < n) out[ao[u]] = v[u];
  }
}

// profile slot of an instruction: op class x sub-op x size bucket
__device__ __forceinline__ int prof_slot(const gevo_instr& I) {
  const int big = I.n >= 4096 ? 1 : 0;
  return ((I.op & 7) * 16 + (I.sub & 15)) * 2 + big;
}

__device__ __noinline__ void run_instrs(Shared& S, const gevo_instr* ins, int n, double* stage,
                           unsigned long long* prof) {
  long long t0 = 0;
  if (prof && threadIdx.x == 0) t0 = clock64();
  for (int k = 0; k < n; ++k) {
    const gevo_instr& I = ins[k];
    // small f64 binary ops with linear/scalar operands (most of a step's
    // non-dot instructions): inline, no call
    if (I.op == GEVO_OP_BINARY && I.kin == GEVO_K_F64 && I.sub <= GEVO_B_MAX && I.n <= 2 * kThreads &&
        I.aux2[0] != AM_STRIDED && I.aux2[1] != AM_STRIDED && I.aux2[2] != AM_STRIDED &&
        I.aux2[4] == 0) {
      const int n_ = I.n, sub = I.sub;
      const int so = I.aux2[0] == AM_LINEAR, sa = I.aux2[1] == AM_LINEAR, sb = I.aux2[2] == AM_LINEAR;
      double* o = S.base[I.out.buf] + I.out.off;
      const double* a = S.base[I.in[0].buf] + I.in[0].off;
      const double* b = S.base[I.in[1].buf] + I.in[1].off;
      const int i0 = threadIdx.x, i1 = threadIdx.x + kThreads;
      const bool h0 = i0 < n_, h1 = i1 < n_;
      double a0 = 0.0, b0 = 0.0, a1 = 0.0, b1 = 0.0;
      if (h0) { a0 = a[i0 * sa]; b0 = b[i0 * sb]; }
      if (h1) { a1 = a[i1 * sa]; b1 = b[i1 * sb]; }
      double r0, r1;
      switch (sub) {
        case GEVO_B_ADD: r0 = __dadd_rn(a0, b0); r1 = __dadd_rn(a1, b1); break;
        case GEVO_B_SUB: r0 = __dsub_rn(a0, b0); r1 = __dsub_rn(a1, b1); break;
        case GEVO_B_MUL: r0 = __dmul_rn(a0, b0); r1 = __dmul_rn(a1, b1); break;
        case GEVO_B_DIV: r0 = __ddiv_rn(a0, b0); r1 = __ddiv_rn(a1, b1); break;
        default: r0 = np_fmax(a0, b0); r1 = np_fmax(a1, b1); break;
      }
      if (h0) o[i0 * so] = r0;
      if (h1) o[i1 * so] = r1;
    } else switch (I.op) {
      case GEVO_OP_UNARY:
      case GEVO_OP_BINARY:
      case GEVO_OP_SELECT:
        if (I.aux2[4] > 0) {
          run_ew_chain(S, I);
          k += I.aux2[4];
        } else {
          run_elementwise(S, I);
        }
        break;
      case GEVO_OP_REDUCE: run_reduce(S, I); break;
      case GEVO_OP_TAPSUM: run_tapsum(S, I); k += I.aux2[4]; break;
      case GEVO_OP_DOT: run_dot(S, I, stage); k += I.aux2[0]; break;
      case GEVO_OP_PAD: run_pad(S, I); break;
    }
    __syncthreads();
    if (prof && threadIdx.x == 0) {
      const long long t1 = clock64();
      const int slot = prof_slot(I);
      atomicAdd(prof + 2 * slot, (unsigned long long)(t1 - t0));
      atomicAdd(prof + 2 * slot + 1, 1ULL);
      t0 = t1;
    }
  }
}

// stage a function's instructions in shared memory when they fit
__device__ const gevo_instr* stage(gevo_instr* cache, const gevo_instr* g, int n) {
  if (n > kInstrCache) return g;
  const int words = n * (int)(sizeof(gevo_instr) / 4);
  const int* src = reinterpret_cast<const int*>(g);
  int* dst = reinterpret_cast<int*>(cache);
  for (int w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
  __syncthreads();
  return cache;
}

// every weight finite: weight i at (inplace bit i ? blk0 : cur) + wofs[i]
// (its extent runs to the next weight's offset; padding words stay zero)
__device__ bool weights_finite(const double* blk0, const double* cur, int inplace, const int32_t* wofs,
                               int nw, int elems) {
  int bad = 0;
  for (int w = 0; w < nw; ++w) {
    const double* b = ((inplace >> w) & 1) ? blk0 : cur;
    const int lo = w == 0 ? 0 : wofs[w], hi = w + 1 < nw ? wofs[w + 1] : elems;
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) bad |= !isfinite(b[i]);
  }
  return !__syncthreads_or(bad);
}

__device__ bool all_finite(const double* w, int n) {
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) bad |= !isfinite(w[i]);
  return !__syncthreads_or(bad);
}

__global__ void __launch_bounds__(kThreads, GEVO_MIN_BLOCKS)
GEVO_KNAME(eval_kernel)(const __grid_constant__ EvalArgs args) {
  __shared__ Shared S;
  __shared__ gevo_instr cache[kInstrCache];
  extern __shared__ double dyn_smem[];
  double* dstage = dyn_smem;                // dot staging tiles
  double* smem_arena = dyn_smem + kStageElems;
  const gevo_prog P = args.progs[blockIdx.x];
  if (threadIdx.x == 0) {
    S.tc_on = GEVO_TC_MODE ? args.tc : 0;
    S.prof = args.prof;
    S.tc.tmap = args.tma_x64 ? static_cast<const void*>(args.tma_map) : nullptr;
    S.tc.tx64 = args.tma_x64;
    S.tc.trows = args.tma_rows;
    S.tc.tcols = args.tma_cols;
  }
  __syncthreads();
#if GEVO_TC_MODE
  tc_setup(S.tc);
#endif
#ifdef GEVO_DOT_TIMING
  if (threadIdx.x == 0) g_dot_prof = args.prof;
#endif
  double* ind = args.arena + P.arena_off;
  const int wsz = (args.weight_elems + 15) & ~15;
  const int psz = (args.probs_elems + 15) & ~15;
  double* scratch = ind;
  double* probs = ind + P.arena_elems;
  // weight blocks: in the launch's weight region when the host gave one (all
  // block 0s contiguous -- the in-place weights' home -- so one L2 persisting
  // window covers them; gevo_abi.cu), else after the individual's scratch
  double* wbuf[2] = {probs + psz, probs + psz + wsz};
  if (args.wreg) {
    wbuf[0] = args.wreg + (int64_t)blockIdx.x * wsz;
    wbuf[1] = args.wreg + (int64_t)(args.n_prog + blockIdx.x) * wsz;
  }
  const double* consts = args.consts + P.const_off;
  const int nw = args.n_weights;
  int status = GEVO_STATUS_OK;
  int steps_run = 0;
  const long long t_start = clock64();
  unsigned long long g_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));

  const double* final_w = args.init_weights;
  // weights updated in place (GEVO_FLAG_INPLACE): they live in block 0
  const int inplace = (args.mode == GEVO_MODE_TRAIN && args.steps > 0 &&
                       (P.flags & GEVO_SCHED_MASK) == GEVO_SCHED_STEADY1) ? GEVO_FLAG_INPLACE(P.flags) : 0;
  if (args.mode == GEVO_MODE_TRAIN && args.steps > 0) {
    // A step stores each returned weight in its numpy layout; a broadcast
    // (stride-0) or otherwise compact return covers only part of its slot.
    // Zero both ping-pong blocks first so the uncovered words -- not part of
    // any weight -- are finite for the whole-block checks below.  The two
    // blocks are not adjacent in the launch's weight region (all block 0s,
    // then all block 1s): zero each on its own, never a neighbour's.
    for (int i = threadIdx.x; i < wsz; i += blockDim.x) {
      wbuf[0][i] = 0.0;
      wbuf[1][i] = 0.0;
    }
    __syncthreads();
    const gevo_instr* t0 = stage(cache, args.instrs + P.train0, P.train0_n);
    const gevo_instr* cur = t0;
    const int check = args.check_every > 0 ? args.check_every : 1;
    // step 0 reads C-ordered weights (train0); later steps read the layout
    // the previous step stored, so the program follows the layout cycle
    // (gevo_plan.h GEVO_SCHED_*): train1 for every s >= 1; train1 on odd and
    // train0 on even steps (C <-> L0); train1 at step 1 then train2; train1
    // on odd and train2 on even steps >= 2 (L0 <-> L1)
    const int sched = P.flags & GEVO_SCHED_MASK;
    const int pstart[3] = {P.train0, P.train1, P.train2};
    const int plen[3] = {P.train0_n, P.train1_n, P.train2_n};
    int pid = 0;
    for (int s = 0; s < args.steps; ++s) {
      int want = 0;
      if (s > 0) {
        switch (sched) {
          case GEVO_SCHED_STEADY1: want = 1; break;
          case GEVO_SCHED_STEADY2: want = s == 1 ? 1 : 2; break;
          case GEVO_SCHED_ALT01: want = (s & 1) ? 1 : 0; break;
          default: want = (s & 1) ? 1 : 2; break;
        }
      }
      if (want != pid) {
        if (pstart[want] != pstart[pid]) {
          __syncthreads();
          cur = stage(cache, args.instrs + pstart[want], plen[want]);
        }
        pid = want;
      }
      const double* win = (s == 0) ? args.init_weights : wbuf[s & 1];
      double* wout = wbuf[(s + 1) & 1];
      // in-place weights live in block 0 (read from it from step 1 on)
      const double* win_ip = (s == 0) ? args.init_weights : wbuf[0];
      const int b = s % args.train_nb;
      if (threadIdx.x == 0) {
        S.base[GEVO_BUF_ARENA] = scratch;
        S.base[GEVO_BUF_SMEM] = smem_arena;
        S.base[GEVO_BUF_CONST] = const_cast<double*>(consts);
        for (int i = 0; i < nw; ++i) {
          const bool ip = (inplace >> i) & 1;
          S.base[GEVO_BUF_PARAM0 + i] = const_cast<double*>(ip ? win_ip : win) + args.wofs[i];
          S.base[GEVO_BUF_OUT0 + i] = (ip ? wbuf[0] : wout) + args.wofs[i];
        }
        S.base[GEVO_BUF_PARAM0 + nw] = const_cast<double*>(args.train_x) + (int64_t)b * args.x_elems;
        S.base[GEVO_BUF_PARAM0 + nw + 1] = const_cast<double*>(args.train_y) + (int64_t)b * args.y_elems;
      }
      __syncthreads();
      run_instrs(S, cur, plen[pid], dstage, args.prof);
      steps_run = s + 1;
      if ((s + 1) % check == 0 &&
          !(inplace ? weights_finite(wbuf[0], wout, inplace, args.wofs, nw, args.weight_elems)
                    : all_finite(wout, args.weight_elems))) {
        status = GEVO_STATUS_NONFINITE_WEIGHTS;
        break;
      }
    }
    final_w = wbuf[args.steps & 1];
    if (status == GEVO_STATUS_OK &&
        !(inplace ? weights_finite(wbuf[0], final_w, inplace, args.wofs, nw, args.weight_elems)
                  : all_finite(final_w, args.weight_elems)))
      status = GEVO_STATUS_NONFINITE_WEIGHTS;
    __syncthreads();
  }

  int64_t wrong = 0, total = 0;
  if (status == GEVO_STATUS_OK) {
    const gevo_instr* fw = stage(cache, args.instrs + P.fwd, P.fwd_n);
    const int B = args.batch, C = args.classes;
    // score parts (prediction mode): this program scores every n_parts-th batch
    const int part = args.mode == GEVO_MODE_TRAIN ? 0 : GEVO_FLAG_PART(P.flags);
    const int parts = args.mode == GEVO_MODE_TRAIN ? 1 : GEVO_FLAG_NPARTS(P.flags);
    for (int b = part; b < args.score_nb; b += parts) {
      if (threadIdx.x == 0) {
        S.base[GEVO_BUF_ARENA] = scratch;
        S.base[GEVO_BUF_SMEM] = smem_arena;
        S.base[GEVO_BUF_CONST] = const_cast<double*>(consts);
        for (int i = 0; i < nw; ++i)
          S.base[GEVO_BUF_PARAM0 + i] = const_cast<double*>(((inplace >> i) & 1) ? wbuf[0] : final_w) + args.wofs[i];
        S.base[GEVO_BUF_PARAM0 + nw] = const_cast<double*>(args.score_x) + (int64_t)b * args.x_elems;
        S.base[GEVO_BUF_OUT0] = probs;
        S.wrong = 0;
      }
      __syncthreads();
      run_instrs(S, fw, P.fwd_n, dstage, args.prof);
      if (!all_finite(probs, B * C)) { status = GEVO_STATUS_NONFINITE_PROBS; break; }
      // first-max argmax per row (np.argmax) vs label
      for (int r = threadIdx.x; r < B; r += blockDim.x) {
        const double* row = probs + (int64_t)r * C;
        int arg = 0;
        double best = row[0];
        for (int c = 1; c < C; ++c) if (row[c] > best) { best = row[c]; arg = c; }
        if (arg != args.score_labels[(int64_t)b * B + r]) atomicAdd(&S.wrong, 1);
      }
      __syncthreads();
      wrong += S.wrong;
      total += B;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    gevo_result* R = args.results + blockIdx.x;   // per program; gevo_eval merges by result_slot
    R->wrong = status == GEVO_STATUS_OK ? wrong : 0;
    R->total = status == GEVO_STATUS_OK ? total : 0;
    R->status = status;
    R->steps_run = steps_run;
    R->cycles = clock64() - t_start;
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    R->t0_ns = (int64_t)g_start;
    R->t1_ns = (int64_t)g_end;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    R->smid = (int32_t)smid;
  }
  if (args.final_weights != nullptr) {
    double* dst = args.final_weights + (int64_t)P.result_slot * args.weight_elems;
    for (int w = 0; w < nw; ++w) {
      const double* b = ((inplace >> w) & 1) ? wbuf[0] : final_w;
      const int lo = w == 0 ? 0 : args.wofs[w], hi = w + 1 < nw ? args.wofs[w + 1] : args.weight_elems;
      for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) dst[i] = b[i];
    }
  }
#if GEVO_TC_MODE
  tc_teardown(S.tc);
#endif
}

// run one function once per prog with explicit params (tests, tools)
__global__ void __launch_bounds__(kThreads, GEVO_MIN_BLOCKS)
GEVO_KNAME(exec_once_kernel)(OnceArgs args) {
  __shared__ Shared S;
  __shared__ gevo_instr cache[kInstrCache];
  extern __shared__ double dyn_smem[];
  double* dstage = dyn_smem;                // dot staging tiles
  double* smem_arena = dyn_smem + kStageElems;
  const gevo_prog P = args.progs[blockIdx.x];
  if (threadIdx.x == 0) {
    S.tc_on = GEVO_TC_MODE ? args.tc : 0;
    S.prof = nullptr;
    S.base[GEVO_BUF_ARENA] = args.arena + P.arena_off;
    S.base[GEVO_BUF_SMEM] = smem_arena;
    S.base[GEVO_BUF_CONST] = const_cast<double*>(args.consts) + P.const_off;
    for (int i = 0; i < GEVO_MAXP; ++i) {
      S.base[GEVO_BUF_PARAM0 + i] = const_cast<double*>(args.params) + P.param_off[i];
      S.base[GEVO_BUF_OUT0 + i] = args.outs + P.out_off[i];
    }
  }
  __syncthreads();
#if GEVO_TC_MODE
  if (threadIdx.x == 0) S.tc.tmap = nullptr;
  tc_setup(S.tc);
#endif
  const gevo_instr* ins = stage(cache, args.instrs + P.train0, P.train0_n);
  run_instrs(S, ins, P.train0_n, dstage, nullptr);
#if GEVO_TC_MODE
  tc_teardown(S.tc);
#endif
}

// The dynamic shared-memory ceiling is a per-function attribute shared by
// every context (and host thread) of the process: raise it once to the
// opt-in maximum instead of per launch, so two contexts launching
// concurrently with different plan sizes cannot lower it under each other.
template <class K>
static void raise_smem_ceiling(K kernel) {
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [&] {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kernel);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  });
}

void GEVO_KNAME(launch_eval)(const EvalArgs& a, int n_prog, cudaStream_t st) {
  const size_t smem = (size_t)(a.smem_elems + kStageElems) * sizeof(double);
  raise_smem_ceiling(GEVO_KNAME(eval_kernel));
  GEVO_KNAME(eval_kernel)<<<n_prog, kThreads, smem, st>>>(a);
}

void GEVO_KNAME(launch_once)(const OnceArgs& a, int n_prog, cudaStream_t st) {
  const size_t smem = (size_t)(a.smem_elems + kStageElems) * sizeof(double);
  raise_smem_ceiling(GEVO_KNAME(exec_once_kernel));
  GEVO_KNAME(exec_once_kernel)<<<n_prog, kThreads, smem, st>>>(a);
}

}  // namespace gevo
