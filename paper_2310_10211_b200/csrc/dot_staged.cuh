// dot_staged.cuh -- the executor's DOT: every summation order the reference
// can produce (lowering.dot_modes), fed through a shared-memory pipeline.
//
// Replaces `v[i] @ v[j]` (interpreter.py:114-116): numpy -> OpenBLAS dgemm
// for blasable f64 operands, numpy's own loop otherwise.  Orders:
//   FMA_CHAIN  one fma chain per output, k ascending     -> DMMA m8n8k4
//   ACC8_TREE  8 chains (k mod 8) + fixed pairwise tree   -> DMMA per chain
//   ACC8_TAIL  ACC8 over k < K&~7, tree, fma tail         -> DMMA + scalar tail
//   SEQ_NOFMA  acc = acc + a*b, two roundings             -> scalar DMUL/DADD
//   integer    wrapping int64 multiply-add                -> scalar
// DMMA m8n8k4 was probed bit-identical to four chained fma() in k order
// (tests/tools/dmma_probe2.cu), so a k-ordered DMMA sequence reproduces a
// single-accumulator chain exactly; ACC8 chains get their own accumulator
// tiles, the k values of chain j are gathered into one DMMA by a k
// permutation applied while staging.
//
// Pipeline: the output is cut into panels (<= 32 x 32); each (panel, 32-k
// chunk) is one stage: an A tile plus a second tile -- the B chunk, or, when
// all of B fits one persistent tile, a full-matrix epilogue operand (e.g. w1
// in w1 - lr * x^T.d) -- copied with cp.async kDotStages deep.  Each thread
// precomputes its copy plan (source/smem offsets) once per instruction:
// 16-byte copies along the operand's unit-stride axis when lines are
// contiguous and aligned, 8-byte gathers for any other strides, synchronous
// copies from the shared-memory arena.  Tile rows are padded to 36 doubles so
// DMMA fragment reads are bank-conflict free in either orientation.
// (A TMA bulk-copy ring -- one cp.async.bulk per 256-byte line, mbarrier
// full/empty -- measured 2.3x slower than this ring on B200; see
// profiles/r01_dot_experiments.md.)
#pragma once
#include <stdint.h>
#include "gevo_plan.h"

namespace gevo {

constexpr int kKC = 32;              // k per chunk
constexpr int kPanel = 32;           // panel rows / cols
constexpr int kTS = 36;              // padded tile row (doubles)
constexpr int kTileElems = kPanel * kTS;
constexpr int kDotStages = 3;
// 3 stages x (A tile + second tile) + one persistent B tile
constexpr int kStageElems = (kDotStages * 2 + 1) * kTileElems;   // 8064 doubles

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
// 16 bytes, of which `bytes` (8 or 16) are read and the rest zero-filled
__device__ __forceinline__ void cp_async16(uint32_t dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int kDotThreads = kThreads;          // the executor's CTA
constexpr int kDotWarps = kDotThreads / 32;

constexpr int kVecPasses = 512 / kDotThreads;   // 16-byte copies per thread per tile
constexpr int kGatherPasses = 1024 / kDotThreads;

// One operand staged as 32 x 32 tiles: element (r, k) -> smem r*rs + pos(k)*ks
// with (rs, ks) = (kTS, 1) when k is the line axis ("k-major") else (1, kTS).
// Copies run along the line axis (the operand's unit-stride axis when it has
// one).  Thread t's copy i covers cross index x0(t) + i*xs at line index
// f(t): 16-byte lines (x0 = t>>4, f = 2*(t&15)) or 8-byte gathers (x0 = t>>5,
// f = t&31).  Kept compact: this is live across the whole dot.
enum { CP_GATHER = 0, CP_VEC = 1, CP_SMEM = 2 };
struct CopyPlan {      // uniform across the CTA: lives in shared memory
  const double* p;     // element (0, 0) of the operand
  int sr, sk;          // element strides along r (m or n) and k
  int so;              // source step between a thread's copies
  int flags;           // bits 0-1 mode, bit 2 k-major, bit 3 ACC8 permutation
  int cross, along;
};

__device__ __forceinline__ int cp_mode(const CopyPlan& c) { return c.flags & 3; }
__device__ __forceinline__ bool cp_kmajor(const CopyPlan& c) { return (c.flags >> 2) & 1; }
__device__ __forceinline__ int cp_rs(const CopyPlan& c) { return cp_kmajor(c) ? kTS : 1; }
__device__ __forceinline__ int cp_ks(const CopyPlan& c) { return cp_kmajor(c) ? 1 : kTS; }

__device__ __forceinline__ void plan_init(CopyPlan& c, const double* p, int sr, int sk, bool smem, bool perm) {
  c.p = p;
  c.sr = sr;
  c.sk = sk;
  const int ar = sr < 0 ? -sr : sr, ak = sk < 0 ? -sk : sk;
  // lines along k when k is the (non-broadcast) contiguous axis
  const bool kmajor = ak != 0 && (ar == 0 || ak <= ar);
  const int cross = kmajor ? sr : sk, along = kmajor ? sk : sr;
  const bool aligned = ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (cross & 1) == 0;
  const int mode = smem ? CP_SMEM : ((!perm && along == 1 && aligned) ? CP_VEC : CP_GATHER);
  c.flags = mode | (kmajor ? 4 : 0) | (perm ? 8 : 0);
  const int xs = mode == CP_VEC ? kDotThreads / 16 : kDotWarps;
  c.so = xs * cross;
  c.cross = cross;
  c.along = along;
}

// thread's source offset of its first copy
__device__ __forceinline__ int plan_o0(const CopyPlan& c) {
  const int t = threadIdx.x;
  const bool vec = (c.flags & 3) == CP_VEC;
  const int x0 = vec ? t >> 4 : t >> 5;
  const int f = vec ? (t & 15) * 2 : t & 31;
  return x0 * c.cross + f * c.along;
}

// stage the tile at (r0, k0) with nr x nk valid elements into smem `dst`
__device__ __forceinline__ void stage(uint32_t dst, const CopyPlan& c, int o0, int r0, int nr, int k0, int nk) {
  const bool kmajor = cp_kmajor(c);
  const int mode = cp_mode(c);
  const int nx = kmajor ? nr : nk, nf = kmajor ? nk : nr;
  const int t = threadIdx.x;
  const double* src = c.p + ((int64_t)r0 * c.sr + (int64_t)k0 * c.sk + o0);
  if (mode == CP_VEC) {
    const int x0 = t >> 4, f = (t & 15) * 2;
    if (f >= nf) return;
    const int bytes = nf - f >= 2 ? 16 : 8;
    const uint32_t d = dst + 8u * (x0 * kTS + f);
#pragma unroll
    for (int i = 0; i < kVecPasses; ++i)
      if (x0 + (kDotThreads / 16) * i < nx) cp_async16(d + 8u * ((kDotThreads / 16) * kTS) * i, src + i * c.so, bytes);
    return;
  }
  const int x0 = t >> 5, f = t & 31;
  if (f >= nf) return;
  const bool perm = (c.flags >> 3) & 1;
  const int rs = kmajor ? kTS : 1, ks = kmajor ? 1 : kTS;
#pragma unroll
  for (int i = 0; i < kGatherPasses; ++i) {
    const int x = x0 + kDotWarps * i;
    if (x < nx) {
      const int rr = kmajor ? x : f, kk = kmajor ? f : x;
      const int pk = perm ? (((kk & 7) << 2) | (kk >> 3)) : kk;
      const uint32_t d = dst + 8u * (rr * rs + pk * ks);
      if (mode == CP_GATHER) cp_async8(d, src + i * c.so);
      else *reinterpret_cast<double*>(__cvta_shared_to_generic(d)) = src[i * c.so];
    }
  }
}

// Epilogue (fused elementwise consumers of the dot, gevo_plan.h): the fast
// kinds keep their operand descriptors in registers; each of the first
// kEpiPre operands is a scalar, the panel's staged tile, or a direct load.
enum { ES_SCALAR = 0, ES_TILE = 1, ES_DIRECT = 2 };
struct EpiR {
  int nops;
  int src[kEpiPre], fsub[kEpiPre], fleft[kEpiPre];
  double sval[kEpiPre];
  const double* ptr[kEpiPre];
  int st0[kEpiPre], st1[kEpiPre];
  int tile;            // operand index staged with the panel (-1: none)
};

__device__ __forceinline__ void epi_init(EpiR& R, const EpiDev* e, bool tile_free) {
  R.nops = e ? e->nops : 0;
  R.tile = -1;
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x) {
    R.src[x] = ES_DIRECT;
    R.sval[x] = 0.0;
    R.fsub[x] = e ? e->fsub[x] : 0;
    R.fleft[x] = e ? e->fleft[x] : 0;
    R.ptr[x] = e ? e->ptr[x] : nullptr;
    R.st0[x] = e ? (int)e->st0[x] : 0;
    R.st1[x] = e ? (int)e->st1[x] : 0;
    if (e && e->fast && x < e->next) {
      if (R.st0[x] == 0 && R.st1[x] == 0) {
        R.src[x] = ES_SCALAR;
        R.sval[x] = R.ptr[x][0];
      } else if (tile_free && R.tile < 0 && R.st0[x] != 0 && R.st1[x] != 0 && !__isShared(R.ptr[x])) {
        R.src[x] = ES_TILE;
        R.tile = x;
      }
    }
  }
}

__device__ __forceinline__ double epi_operand(const EpiR& R, int x, const double* Es, int ers, int eks,
                                              int m, int n, int mm, int nn) {
  if (R.src[x] == ES_SCALAR) return R.sval[x];
  if (R.src[x] == ES_TILE) return Es[mm * ers + nn * eks];
  return R.ptr[x][(int64_t)m * R.st0[x] + (int64_t)n * R.st1[x]];
}

// the epilogue of output (m, n) (panel-local (mm, nn)) applied to dot value v
template <int EK>
__device__ __forceinline__ double epi_apply(const EpiR& R, const EpiDev* epi, const double* Es, int ers,
                                            int eks, double v, int m, int n, int mm, int nn) {
  if (EK == EK_NONE) return v;
  if (EK == EK_CHAIN) {
#pragma unroll
    for (int x = 0; x < kEpiPre; ++x) {
      if (x < R.nops) {
        const double o = epi_operand(R, x, Es, ers, eks, m, n, mm, nn);
        v = R.fleft[x] ? bin_f64(R.fsub[x], v, o) : bin_f64(R.fsub[x], o, v);
      }
    }
    return v;
  }
  if (EK == EK_SELECT) {
    const bool p = as_i64(epi_operand(R, 0, Es, ers, eks, m, n, mm, nn)) != 0;
    const double o = epi_operand(R, 1, Es, ers, eks, m, n, mm, nn);
    return R.fleft[0] ? (p ? v : o) : (p ? o : v);
  }
  double ev[kEpiPre];
  epi_fetch(*epi, m, n, ev);
  return epilogue_generic(*epi, ev, v, m, n);
}

struct DotArgs {
  const double* A;
  const double* B;
  int sam, sak, sbk, sbn;
  bool a_smem, b_smem;
  double* out;
  int som, son;
  int M, K;
  int xrow;     // ACC8 outputs in rows >= xrow reduce their lanes in the
                // AVX-512 order (OpenBLAS edge kernels for the m % 4 rows)
};

// the 8 lane chains of output h (lane j in acc[2j + h]) folded to one value:
// the pairwise tree ((0+1)+(2+3))+((4+5)+(6+7)) of the full-width kernels, or
// (avx) the _mm512_reduce_add_pd order ((0+4)+(2+6))+((1+5)+(3+7)) of the
// OpenBLAS edge kernels (lowering.dot_modes)
__device__ __forceinline__ double lane_tree(const double* acc, int h, bool avx) {
  const double l0 = acc[h], l1 = acc[2 + h], l2 = acc[4 + h], l3 = acc[6 + h];
  const double l4 = acc[8 + h], l5 = acc[10 + h], l6 = acc[12 + h], l7 = acc[14 + h];
  if (avx)
    return __dadd_rn(__dadd_rn(__dadd_rn(l0, l4), __dadd_rn(l2, l6)),
                     __dadd_rn(__dadd_rn(l1, l5), __dadd_rn(l3, l7)));
  return __dadd_rn(__dadd_rn(__dadd_rn(l0, l1), __dadd_rn(l2, l3)),
                   __dadd_rn(__dadd_rn(l4, l5), __dadd_rn(l6, l7)));
}

// Panel epilogue + store (all threads): the panel's raw dot values sit in
// the C tile (row-major, stride kCS); thread t handles elements
// e = t + kDotThreads*u of the 32 x 32 panel, (i, j) = (e >> 5, e & 31), so
// consecutive threads store consecutive output columns.  EK is uniform.
constexpr int kCS = 33;
constexpr int kEmitPer = 1024 / kDotThreads;   // panel elements per thread

template <int EK>
__device__ __forceinline__ void dot_emit_panel(const double* Cs, const double* Es, const EpiR& Rs, int ers, int eks,
                                            const EpiDev* epi, double* out, int som, int son, int m0, int n0,
                                            int pm, int pn) {
  double v[kEmitPer];
  bool in[kEmitPer];
#pragma unroll
  for (int u = 0; u < kEmitPer; ++u) {
    const int e = threadIdx.x + u * kDotThreads;
    const int i = e >> 5, j = e & 31;
    in[u] = i < pm && j < pn;
    v[u] = in[u] ? Cs[i * kCS + j] : 0.0;
  }
  if (EK == EK_CHAIN || EK == EK_SELECT) {
    const EpiR R = Rs;                 // registers; uniform decisions below
    const int nx = EK == EK_SELECT ? 2 : R.nops;
    double o[kEpiPre][kEmitPer];
#pragma unroll
    for (int x = 0; x < kEpiPre; ++x) {
      if (x < nx) {
        const int src = R.src[x];
        if (src == ES_SCALAR) {
#pragma unroll
          for (int u = 0; u < kEmitPer; ++u) o[x][u] = R.sval[x];
        } else if (src == ES_TILE) {
#pragma unroll
          for (int u = 0; u < kEmitPer; ++u) {
            const int e = threadIdx.x + u * kDotThreads;
            o[x][u] = in[u] ? Es[(e >> 5) * ers + (e & 31) * eks] : 0.0;
          }
        } else {
          const double* pp = R.ptr[x] + (int64_t)m0 * R.st0[x] + (int64_t)n0 * R.st1[x];
#pragma unroll
          for (int u = 0; u < kEmitPer; ++u) {
            const int e = threadIdx.x + u * kDotThreads;
            o[x][u] = in[u] ? pp[(int64_t)(e >> 5) * R.st0[x] + (int64_t)(e & 31) * R.st1[x]] : 0.0;
          }
        }
      }
    }
    if (EK == EK_SELECT) {
#pragma unroll
      for (int u = 0; u < kEmitPer; ++u) {
        const bool p = as_i64(o[0][u]) != 0;
        v[u] = R.fleft[0] ? (p ? v[u] : o[1][u]) : (p ? o[1][u] : v[u]);
      }
    } else {
#pragma unroll
      for (int x = 0; x < kEpiPre; ++x) {
        if (x < nx) {
          const bool left = R.fleft[x];
#define GEVO_EMIT_OP(EXPR)                                                  \
  _Pragma("unroll") for (int u = 0; u < kEmitPer; ++u) {                    \
    const double a = left ? v[u] : o[x][u], b = left ? o[x][u] : v[u];     \
    v[u] = (EXPR);                                                          \
  }
          switch (R.fsub[x]) {   // warp-uniform: one dispatch per micro-op
            case GEVO_B_ADD: GEVO_EMIT_OP(__dadd_rn(a, b)); break;
            case GEVO_B_SUB: GEVO_EMIT_OP(__dsub_rn(a, b)); break;
            case GEVO_B_MUL: GEVO_EMIT_OP(__dmul_rn(a, b)); break;
            case GEVO_B_DIV: GEVO_EMIT_OP(__ddiv_rn(a, b)); break;
            default: GEVO_EMIT_OP(np_fmax(a, b)); break;
          }
#undef GEVO_EMIT_OP
        }
      }
    }
  } else if (EK == EK_GENERIC) {
#pragma unroll
    for (int u = 0; u < kEmitPer; ++u) {
      if (in[u]) {
        const int e = threadIdx.x + u * kDotThreads;
        const int m = m0 + (e >> 5), n = n0 + (e & 31);
        double ev[kEpiPre];
        epi_fetch(*epi, m, n, ev);
        v[u] = epilogue_generic(*epi, ev, v[u], m, n);
      }
    }
  }
  double* ob = out + (int64_t)m0 * som + (int64_t)n0 * son;
#pragma unroll
  for (int u = 0; u < kEmitPer; ++u) {
    const int e = threadIdx.x + u * kDotThreads;
    if (in[u]) ob[(int64_t)(e >> 5) * som + (int64_t)(e & 31) * son] = v[u];
  }
}

template <int EK>
__device__ __forceinline__ void dot_emit_dispatch(int ek, const double* Cs, const double* Es, const EpiR& R,
                                                  int ers, int eks, const EpiDev* epi, double* out, int som,
                                                  int son, int m0, int n0, int pm, int pn) {
  switch (ek) {
    case EK_NONE: dot_emit_panel<EK_NONE>(Cs, Es, R, ers, eks, epi, out, som, son, m0, n0, pm, pn); break;
    case EK_CHAIN: dot_emit_panel<EK_CHAIN>(Cs, Es, R, ers, eks, epi, out, som, son, m0, n0, pm, pn); break;
    case EK_SELECT: dot_emit_panel<EK_SELECT>(Cs, Es, R, ers, eks, epi, out, som, son, m0, n0, pm, pn); break;
    default: dot_emit_panel<EK_GENERIC>(Cs, Es, R, ers, eks, epi, out, som, son, m0, n0, pm, pn); break;
  }
}

// KIND: 0 FMA_CHAIN (DMMA; warp = 8 x 16 strip of a 32 x 32 panel), 1 ACC8
// (DMMA; warp = one 8 x 8 tile x 8 chains; panels 32 x 16), 2 SEQ_NOFMA,
// 3 integer (scalar; thread = 4 outputs of a 32 x 32 panel).  Output columns
// [col0, col1).  After a panel's last chunk its values go to the C tile (the
// slot's A region) and dot_emit_panel applies the epilogue and stores.
template <int KIND>
__device__ __forceinline__ void dot_pipeline(const DotArgs& dref, int col0, int col1, int mode, double* stage_buf,
                                             const EpiDev* epi) {
  static_assert(kDotWarps == 8, "dot tiling assumes 8 warps");
  const DotArgs d = dref;   // registers: stores through d.out must not alias it
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  constexpr int PN = KIND == 1 ? 16 : kPanel;   // ACC8 panels are 32 x 16
  constexpr bool perm = KIND == 1;
  const int M = d.M, K = d.K;
  const int ncols = col1 - col0;
  const int npc = (ncols + PN - 1) / PN;
  const int nch = (K + kKC - 1) / kKC;
  const int total = ((M + kPanel - 1) / kPanel) * npc * nch;
  const int ek = !epi ? EK_NONE : (epi->fast == 1 ? EK_CHAIN : (epi->fast == 2 ? EK_SELECT : EK_GENERIC));
  // all of B in one persistent tile: staged once; each stage's second tile
  // is then free for a full-matrix epilogue operand
  const bool bpersist = nch == 1 && npc == 1;
  // uniform per-instruction state in shared memory (registers go to the
  // accumulators and the per-thread copy offsets)
  __shared__ EpiR R;
  __shared__ CopyPlan pa_, pb_, pe_;
  if (threadIdx.x == 0) {
    epi_init(R, ek == EK_CHAIN || ek == EK_SELECT ? epi : nullptr, bpersist);
    plan_init(pa_, d.A, d.sam, d.sak, d.a_smem, perm);
    plan_init(pb_, d.B, d.sbn, d.sbk, d.b_smem, perm);
    if (R.tile >= 0) plan_init(pe_, R.ptr[R.tile], R.st0[R.tile], R.st1[R.tile], false, false);
  }
  __syncthreads();
  const bool etile = R.tile >= 0;
  const int oa = plan_o0(pa_), ob = plan_o0(pb_), oe = etile ? plan_o0(pe_) : 0;
  const uint32_t ring = smem_u32(stage_buf);
  double* Bp = stage_buf + kDotStages * 2 * kTileElems;

  if (bpersist) stage(smem_u32(Bp), pb_, ob, col0, ncols, 0, K);
  int lc = 0, lm0 = 0, ln0 = col0;     // load-side cursor: chunk, panel origin
  auto load_next = [&](int slot) {
    const uint32_t As = ring + 8u * (slot * 2 * kTileElems);
    const uint32_t Xs = As + 8u * kTileElems;
    const int k0 = lc * kKC;
    const int nk = min(kKC, K - k0), pm = min(kPanel, M - lm0), pn = min(PN, col1 - ln0);
    stage(As, pa_, oa, lm0, pm, k0, nk);
    if (!bpersist) stage(Xs, pb_, ob, ln0, pn, k0, nk);
    else if (etile) stage(Xs, pe_, oe, lm0, pm, ln0, pn);
    if (++lc == nch) {
      lc = 0;
      ln0 += PN;
      if (ln0 >= col1) { ln0 = col0; lm0 += kPanel; }
    }
  };
#pragma unroll 1
  for (int s = 0; s < kDotStages - 1; ++s) {
    if (s < total) load_next(s);
    cp_async_commit();
  }

  constexpr int NACC = KIND == 1 ? 16 : 4;
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  const int rb = warp >> 1;
  const int cb0 = KIND == 1 ? (warp & 1) : (warp & 1) * 2;
  const int ars = cp_rs(pa_), aks = cp_ks(pa_), brs = cp_rs(pb_), bks = cp_ks(pb_);
  const int lm = rb * 8 + g;          // lane's panel row (DMMA kinds)
  const int ln = cb0 * 8 + 2 * t4;    // lane's first panel column
  int c = 0, m0 = 0, n0 = col0;       // compute-side cursor
  int slot = 0, lslot = kDotStages - 1;

#pragma unroll 1
  for (int s = 0; s < total; ++s) {
    if (s + kDotStages - 1 < total) load_next(lslot);
    cp_async_commit();
    cp_async_wait<kDotStages - 1>();
    __syncthreads();
    const int k0 = c * kKC;
    const int nk = min(kKC, K - k0);
    const bool last = c == nch - 1;
    double* As = stage_buf + slot * 2 * kTileElems;
    // a persistent B tile holds every k (nch == 1); a streamed one this chunk's
    const double* Bs = bpersist ? Bp : As + kTileElems;
    const int pm = min(kPanel, M - m0), pn = min(PN, col1 - n0);
    double* Cs = As;                    // C tile (after the A tile is consumed)

    if (KIND == 0) {
      const bool act0 = rb * 8 < pm && cb0 * 8 < pn;
      const bool act1 = act0 && (cb0 + 1) * 8 < pn;
      if (act0) {
        const double* pa = As + lm * ars + t4 * aks;
        const double* pb0 = Bs + (cb0 * 8 + g) * brs + t4 * bks;
        const double* pb1 = pb0 + 8 * brs;
        const int nq = nk >> 2;
        const int qa = 4 * aks, qb = 4 * bks;
        if (nq == 8 && act1) {
          double fa[8], fb0[8], fb1[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            fa[q] = pa[q * qa];
            fb0[q] = pb0[q * qb];
            fb1[q] = pb1[q * qb];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            dmma884(acc[0], acc[1], fa[q], fb0[q]);
            dmma884(acc[2], acc[3], fa[q], fb1[q]);
          }
        } else {
#pragma unroll 1
          for (int q = 0; q < nq; ++q) {
            const double a = pa[q * qa];
            dmma884(acc[0], acc[1], a, pb0[q * qb]);
            if (act1) dmma884(acc[2], acc[3], a, pb1[q * qb]);
          }
          // k tail (K % 4), last chunk only: scalar fma on this lane's outputs
#pragma unroll 1
          for (int kk = nq * 4; kk < nk; ++kk) {
            const double a = As[lm * ars + kk * aks];
            acc[0] = fma(a, Bs[ln * brs + kk * bks], acc[0]);
            acc[1] = fma(a, Bs[(ln + 1) * brs + kk * bks], acc[1]);
            if (act1) {
              acc[2] = fma(a, Bs[(ln + 8) * brs + kk * bks], acc[2]);
              acc[3] = fma(a, Bs[(ln + 9) * brs + kk * bks], acc[3]);
            }
          }
        }
      }
      if (last) {
        __syncthreads();                // every warp is done reading A
        if (act0) {
          Cs[lm * kCS + ln] = acc[0];
          Cs[lm * kCS + ln + 1] = acc[1];
          Cs[lm * kCS + ln + 8] = acc[2];
          Cs[lm * kCS + ln + 9] = acc[3];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = 0.0;
      }
    } else if (KIND == 1) {
      const int kmain = (mode == GEVO_D_ACC8_TAIL) ? (K & ~7) : K;
      const bool act = rb * 8 < pm && cb0 * 8 < pn;
      double r0 = 0.0, r1 = 0.0;
      if (act) {
        const double* pa = As + lm * ars + t4 * aks;
        const double* pb = Bs + (cb0 * 8 + g) * brs + t4 * bks;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (k0 + j + 24 < kmain) {
            // chain j's four k (j, j+8, j+16, j+24) sit at positions 4j..4j+3
            dmma884(acc[2 * j], acc[2 * j + 1], pa[4 * j * aks], pb[4 * j * bks]);
          } else {
#pragma unroll 1
            for (int t = 0; t < 4; ++t) {
              const int kk = j + 8 * t;
              if (k0 + kk >= kmain) break;
              const int pk = 4 * j + t;
              const double a = As[lm * ars + pk * aks];
              acc[2 * j] = fma(a, Bs[ln * brs + pk * bks], acc[2 * j]);
              acc[2 * j + 1] = fma(a, Bs[(ln + 1) * brs + pk * bks], acc[2 * j + 1]);
            }
          }
        }
        if (last) {
          const bool avx = m0 + lm >= d.xrow;
          r0 = lane_tree(acc, 0, avx);
          r1 = lane_tree(acc, 1, avx);
#pragma unroll 1
          for (int kk = kmain - k0; kk < nk; ++kk) {     // ACC8_TAIL: k >= K&~7
            const int pk = ((kk & 7) << 2) | (kk >> 3);
            const double a = As[lm * ars + pk * aks];
            r0 = fma(a, Bs[ln * brs + pk * bks], r0);
            r1 = fma(a, Bs[(ln + 1) * brs + pk * bks], r1);
          }
        }
      }
      if (last) {
        __syncthreads();
        if (act) {
          Cs[lm * kCS + ln] = r0;
          Cs[lm * kCS + ln + 1] = r1;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.0;
      }
    } else {
      // scalar (KIND 2 f64 no-FMA, KIND 3 integer): thread owns outputs
      // o = tid + kDotThreads u of the 32 x 32 panel
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int o = threadIdx.x + u * kDotThreads;
        const int mm = o >> 5, nn = o & 31;
        if (mm < pm && nn < pn) {
          const double* pa = As + mm * ars;
          const double* pb = Bs + nn * brs;
          double v = acc[u];
          if (KIND == 2) {
#pragma unroll 1
            for (int kk = 0; kk < nk; ++kk) v = __dadd_rn(v, __dmul_rn(pa[kk * aks], pb[kk * bks]));
          } else {
            uint64_t w = (uint64_t)as_i64(v);
#pragma unroll 1
            for (int kk = 0; kk < nk; ++kk)
              w += (uint64_t)as_i64(pa[kk * aks]) * (uint64_t)as_i64(pb[kk * bks]);
            v = as_w((int64_t)w);
          }
          acc[u] = v;
        }
      }
      if (last) {
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o = threadIdx.x + u * kDotThreads;
          Cs[(o >> 5) * kCS + (o & 31)] = acc[u];
          acc[u] = 0.0;
        }
      }
    }
    if (last) {
      __syncthreads();                  // C tile complete
      const int ers = etile ? cp_rs(pe_) : 0, eks = etile ? cp_ks(pe_) : 0;
      dot_emit_dispatch<0>(ek, Cs, As + kTileElems, R, ers, eks, epi, d.out, d.som, d.son, m0, n0, pm, pn);
    }
    if (++c == nch) {
      c = 0;
      n0 += PN;
      if (n0 >= col1) { n0 = col0; m0 += kPanel; }
    }
    slot = slot + 1 == kDotStages ? 0 : slot + 1;
    lslot = lslot + 1 == kDotStages ? 0 : lslot + 1;
    __syncthreads();   // buffer `slot` is refilled next iteration
  }
  cp_async_wait<0>();
}

template <int KIND>
__device__ __noinline__ void dot_run(const DotArgs& d, int col0, int col1, int mode, double* stage_buf,
                                     const EpiDev* epi) {
  dot_pipeline<KIND>(d, col0, col1, mode, stage_buf, epi);
}


// ---------------------------------------------------------------------------
// Fast paths for the two dot shapes that dominate the workloads (FMA chain,
// every staged operand made of whole 16-byte-aligned lines):
//   KSTREAM  one <= 32 x 32 output panel, K streamed in 32-k chunks
//            (x . w1, K = 784: the forward pass)
//   PANELS   K <= 32 and <= 32 columns: B staged once, the rows streamed in
//            32-row panels, each with its full-matrix epilogue operand
//            (x^T . delta fused with w1 - lr * (.): the weight update)
// Each thread keeps running source pointers for its two 16-byte copies per
// operand tile, so a stage costs a handful of instructions.
struct VecCopy {
  const double* p0;    // thread's copy 0 at the current stage
  int64_t so;          // copy 1 = copy 0 + so
  int64_t adv;         // advance per stage
  uint32_t d0;         // smem byte offset of copy 0 within a tile
  int line0, f;        // cross (line) index of copy 0, element index along the line
  bool kmaj;           // lines run along k (rows of the tile are r)
};

__device__ __forceinline__ void vec_init(VecCopy& v, const double* p, int sr, int sk, int adv_elems) {
  const int ar = sr < 0 ? -sr : sr, ak = sk < 0 ? -sk : sk;
  v.kmaj = ak != 0 && (ar == 0 || ak <= ar);
  const int cross = v.kmaj ? sr : sk;
  const int t = threadIdx.x;
  v.line0 = t >> 4;
  v.f = (t & 15) * 2;
  v.p0 = p + (int64_t)v.line0 * cross + v.f;
  v.so = (int64_t)16 * cross;
  v.adv = adv_elems;
  v.d0 = 8u * (v.line0 * kTS + v.f);
}

__device__ __forceinline__ bool vec_ok(const double* p, int sr, int sk, int rext, int kext) {
  const int ar = sr < 0 ? -sr : sr, ak = sk < 0 ? -sk : sk;
  const bool kmaj = ak != 0 && (ar == 0 || ak <= ar);
  const int cross = kmaj ? sr : sk, along = kmaj ? sk : sr;
  return along == 1 && (cross & 1) == 0 && ((reinterpret_cast<uintptr_t>(p) & 15) == 0) &&
         ((kmaj ? kext : rext) & 1) == 0;
}

// issue one tile (nr x nk valid) of a VecCopy operand into smem tile `tile`
__device__ __forceinline__ void vec_stage(const VecCopy& v, uint32_t tile, int nr, int nk) {
  const int nline = v.kmaj ? nr : nk, nlen = v.kmaj ? nk : nr;
  if (v.f >= nlen) return;
  const int bytes = nlen - v.f >= 2 ? 16 : 8;
  if (v.line0 < nline) cp_async16(tile + v.d0, v.p0, bytes);
  if (v.line0 + 16 < nline) cp_async16(tile + v.d0 + 8u * 16 * kTS, v.p0 + v.so, bytes);
}

#ifdef GEVO_DOT_TIMING
// diagnostics build only: per-phase cycles of dot_fast into profile slots of
// the unused op class 0 (phase p -> slot 2p)
__device__ unsigned long long* g_dot_prof;
#define GEVO_TSTAMP(v) long long v = 0; if (threadIdx.x == 0) v = clock64();
#define GEVO_TACC(p, a, b) if (threadIdx.x == 0 && g_dot_prof) { atomicAdd(g_dot_prof + 4 * (p), (unsigned long long)((b) - (a))); atomicAdd(g_dot_prof + 4 * (p) + 1, 1ULL); }
#else
#define GEVO_TSTAMP(v)
#define GEVO_TACC(p, a, b)
#endif

// One staged operand of dot_fast: whole aligned lines through a running
// pointer (two 16-byte copies per thread per tile: lines t>>4 and t>>4 + 16 at
// element 2*(t&15)), or, for any other strides / shared-memory sources, the
// generic CopyPlan (kept in shared memory) with a (r0, k0) cursor.  Kept
// small: it is live across the whole dot.
struct Feed {
  const double* p;     // vec: thread's copy 0 at the current stage
  int so;              // vec: copy 1 = copy 0 + so
  int adv;             // vec: advance per stage (elements)
  int o0, r0, k0;      // generic: thread offset and tile origin
  int flags;           // bit 0 vec, bit 1 lines along k
};

__device__ __forceinline__ int feed_rs(const Feed& f) { return (f.flags & 2) ? kTS : 1; }
__device__ __forceinline__ int feed_ks(const Feed& f) { return (f.flags & 2) ? 1 : kTS; }

__device__ __forceinline__ void feed_init(Feed& f, CopyPlan& cp, const double* p, int sr, int sk, bool smem,
                                          int r0, int k0, int adv, int rext, int kext) {
  const bool vec = !smem && vec_ok(p, sr, sk, rext, kext);
  if (vec) {
    const int ar = sr < 0 ? -sr : sr, ak = sk < 0 ? -sk : sk;
    const bool kmaj = ak != 0 && (ar == 0 || ak <= ar);
    const int cross = kmaj ? sr : sk;
    const int t = threadIdx.x;
    f.p = p + (int64_t)r0 * sr + (int64_t)k0 * sk + (int64_t)(t >> 4) * cross + (t & 15) * 2;
    f.so = 16 * cross;
    f.adv = adv;
    f.flags = 1 | (kmaj ? 2 : 0);
  } else {
    if (threadIdx.x == 0) plan_init(cp, p, sr, sk, smem, false);
    __syncthreads();
    f.o0 = plan_o0(cp);
    f.flags = cp_kmajor(cp) ? 2 : 0;
  }
  f.r0 = r0;
  f.k0 = k0;
}

// stage the next tile (nr x nk valid); the generic cursor moves by (DR, DK)
template <int DR, int DK>
__device__ __forceinline__ void feed_stage(Feed& f, const CopyPlan& cp, uint32_t tile, int nr, int nk) {
  if (f.flags & 1) {
    const bool kmaj = f.flags & 2;
    const int nline = kmaj ? nr : nk, nlen = kmaj ? nk : nr;
    const int t = threadIdx.x, line0 = t >> 4, e = (t & 15) * 2;
    if (e < nlen) {
      const int bytes = nlen - e >= 2 ? 16 : 8;
      const uint32_t d0 = tile + 8u * (line0 * kTS + e);
      if (line0 < nline) cp_async16(d0, f.p, bytes);
      if (line0 + 16 < nline) cp_async16(d0 + 8u * 16 * kTS, f.p + f.so, bytes);
    }
    f.p += f.adv;
  } else {
    stage(tile, cp, f.o0, f.r0, nr, f.k0, nk);
    f.r0 += DR;
    f.k0 += DK;
  }
}


// Fast epilogue on one lane's four DMMA outputs (row m; panel-local row mm;
// columns nn, nn+1, nn+8, nn+9 of the piece starting at col0).  Operand
// sources and op codes are warp-uniform: one dispatch per micro-op.
__device__ __forceinline__ void epi_lane4(const EpiR& Rs, int ek, const double* Es, int ers, int eks,
                                          double* v, int m, int col0, int mm, int nn, int ncols) {
  if (ek == EK_NONE) return;
  // the whole descriptor in registers first (independent shared loads),
  // then uniform decisions
  int nops = Rs.nops, src[kEpiPre], fsub[kEpiPre], fleft[kEpiPre], st0[kEpiPre], st1[kEpiPre];
  double sval[kEpiPre];
  const double* ptr[kEpiPre];
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x) {
    src[x] = Rs.src[x];
    fsub[x] = Rs.fsub[x];
    fleft[x] = Rs.fleft[x];
    sval[x] = Rs.sval[x];
    ptr[x] = Rs.ptr[x];
    st0[x] = Rs.st0[x];
    st1[x] = Rs.st1[x];
  }
  const int nx = ek == EK_SELECT ? 2 : nops;
  double o[kEpiPre][4];
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x) {
    if (x < nx) {
      if (src[x] == ES_SCALAR) {
#pragma unroll
        for (int h = 0; h < 4; ++h) o[x][h] = sval[x];
      } else if (src[x] == ES_TILE) {
        const double* e = Es + mm * ers + nn * eks;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = (h >> 1) * 8 + (h & 1);
          o[x][h] = nn + c < ncols ? e[c * eks] : 0.0;
        }
      } else {
        const double* e = ptr[x] + (int64_t)m * st0[x] + (int64_t)(col0 + nn) * st1[x];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = (h >> 1) * 8 + (h & 1);
          o[x][h] = nn + c < ncols ? e[(int64_t)c * st1[x]] : 0.0;
        }
      }
    }
  }
  if (ek == EK_SELECT) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const bool p = as_i64(o[0][h]) != 0;
      v[h] = fleft[0] ? (p ? v[h] : o[1][h]) : (p ? o[1][h] : v[h]);
    }
    return;
  }
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x) {
    if (x < nx) {
      const bool left = fleft[x];
#define GEVO_LANE_OP(EXPR)                                                  \
  _Pragma("unroll") for (int h = 0; h < 4; ++h) {                           \
    const double a = left ? v[h] : o[x][h], b = left ? o[x][h] : v[h];     \
    v[h] = (EXPR);                                                          \
  }
      switch (fsub[x]) {
        case GEVO_B_ADD: GEVO_LANE_OP(__dadd_rn(a, b)); break;
        case GEVO_B_SUB: GEVO_LANE_OP(__dsub_rn(a, b)); break;
        case GEVO_B_MUL: GEVO_LANE_OP(__dmul_rn(a, b)); break;
        case GEVO_B_DIV: GEVO_LANE_OP(__ddiv_rn(a, b)); break;
        default: GEVO_LANE_OP(np_fmax(a, b)); break;
      }
#undef GEVO_LANE_OP
    }
  }
}

// Lean variant of dot_fast for the hot case: FMA chain, every operand whole
// aligned lines (VecCopy only; nothing else live across the loop).
template <bool PANELS>
__device__ __noinline__ void dot_fast_vec(const DotArgs& dref, int col0, int col1, double* stage_buf,
                                      const EpiDev* epi) {
  const DotArgs d = dref;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int M = d.M, K = d.K, ncols = col1 - col0;
  const int ek = !epi ? EK_NONE : (epi->fast == 1 ? EK_CHAIN : (epi->fast == 2 ? EK_SELECT : EK_GENERIC));
  __shared__ EpiR R;
  if (threadIdx.x == 0) epi_init(R, ek == EK_CHAIN || ek == EK_SELECT ? epi : nullptr, PANELS);
  __syncthreads();
  const bool etile = PANELS && R.tile >= 0;
  const int total = PANELS ? (M + kPanel - 1) / kPanel : (K + kKC - 1) / kKC;
  const uint32_t ring = smem_u32(stage_buf);
  double* Bp = stage_buf + kDotStages * 2 * kTileElems;

  VecCopy va, vx;        // A; second tile: B chunk (KSTREAM) or epilogue operand (PANELS)
  int brs, bks;
  if (PANELS) {
    vec_init(va, d.A + (int64_t)col0 * 0, d.sam, d.sak, 32 * d.sam);
    if (etile) vec_init(vx, R.ptr[R.tile] + (int64_t)col0 * R.st1[R.tile], R.st0[R.tile], R.st1[R.tile],
                        32 * R.st0[R.tile]);
    // B (K x ncols) once, any layout
    CopyPlan pb;
    plan_init(pb, d.B + (int64_t)col0 * d.sbn, d.sbn, d.sbk, d.b_smem, false);
    stage(smem_u32(Bp), pb, plan_o0(pb), 0, ncols, 0, K);
    brs = cp_rs(pb);
    bks = cp_ks(pb);
  } else {
    vec_init(va, d.A, d.sam, d.sak, 32 * d.sak);
    vec_init(vx, d.B + (int64_t)col0 * d.sbn, d.sbn, d.sbk, 32 * d.sbk);
    brs = vx.kmaj ? kTS : 1;
    bks = vx.kmaj ? 1 : kTS;
  }
  const int ars = va.kmaj ? kTS : 1, aks = va.kmaj ? 1 : kTS;
  const int ers = vx.kmaj ? kTS : 1, eks = vx.kmaj ? 1 : kTS;

  // stage i covers rows [32i, ..) (PANELS) or k [32i, ..) (KSTREAM)
  auto load = [&](int i, int slot) {
    const uint32_t As = ring + 8u * (slot * 2 * kTileElems);
    if (PANELS) {
      const int pm = min(kPanel, M - i * kPanel);
      vec_stage(va, As, pm, K);
      if (etile) vec_stage(vx, As + 8u * kTileElems, pm, ncols);
    } else {
      const int nk = min(kKC, K - i * kKC);
      vec_stage(va, As, M, nk);
      vec_stage(vx, As + 8u * kTileElems, ncols, nk);
    }
    va.p0 += va.adv;
    vx.p0 += vx.adv;
  };
#pragma unroll 1
  for (int i = 0; i < kDotStages - 1; ++i) {
    if (i < total) load(i, i);
    cp_async_commit();
  }
  const int rb = warp >> 1, cb0 = (warp & 1) * 2;
  const int lm = rb * 8 + g, ln = cb0 * 8 + 2 * t4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int slot = 0, lslot = kDotStages - 1;
#pragma unroll 1
  for (int s = 0; s < total; ++s) {
    GEVO_TSTAMP(ta)
    GEVO_TSTAMP(tl)
    // stage s was committed one iteration ago (or in the prologue); the
    // next load is issued after this stage's DMMAs so it overlaps them
    cp_async_wait<kDotStages - 2>();
    __syncthreads();
    GEVO_TSTAMP(tb)
    GEVO_TACC(1, ta, tl)
    GEVO_TACC(2, tl, tb)
    double* As = stage_buf + slot * 2 * kTileElems;
    const double* Bs = PANELS ? Bp : As + kTileElems;
    const int pm = PANELS ? min(kPanel, M - s * kPanel) : M;
    const int nk = PANELS ? K : min(kKC, K - s * kKC);
    const bool last = PANELS || s == total - 1;
    const bool act0 = rb * 8 < pm && cb0 * 8 < ncols;
    const bool act1 = act0 && (cb0 + 1) * 8 < ncols;
    if (act0) {
      const double* pa = As + lm * ars + t4 * aks;
      const double* pb0 = Bs + (cb0 * 8 + g) * brs + t4 * bks;
      const double* pb1 = pb0 + 8 * brs;
      const int nq = nk >> 2;
      const int qa = 4 * aks, qb = 4 * bks;
      if (nq == 8 && act1) {
        // all 24 fragments first (one LDS latency), then 16 back-to-back DMMAs
        double fa[8], fb0[8], fb1[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          fa[q] = pa[q * qa];
          fb0[q] = pb0[q * qb];
          fb1[q] = pb1[q * qb];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          dmma884(acc[0], acc[1], fa[q], fb0[q]);
          dmma884(acc[2], acc[3], fa[q], fb1[q]);
        }
      } else {
#pragma unroll 1
        for (int q = 0; q < nq; ++q) {
          const double a = pa[q * qa];
          dmma884(acc[0], acc[1], a, pb0[q * qb]);
          if (act1) dmma884(acc[2], acc[3], a, pb1[q * qb]);
        }
#pragma unroll 1
        for (int kk = nq * 4; kk < nk; ++kk) {
          const double a = As[lm * ars + kk * aks];
          acc[0] = fma(a, Bs[ln * brs + kk * bks], acc[0]);
          acc[1] = fma(a, Bs[(ln + 1) * brs + kk * bks], acc[1]);
          if (act1) {
            acc[2] = fma(a, Bs[(ln + 8) * brs + kk * bks], acc[2]);
            acc[3] = fma(a, Bs[(ln + 9) * brs + kk * bks], acc[3]);
          }
        }
      }
    }
    if (s + kDotStages - 1 < total) load(s + kDotStages - 1, lslot);
    cp_async_commit();
    GEVO_TSTAMP(tc)
    GEVO_TACC(3, tb, tc)
    if (last && ek != EK_GENERIC) {
      // epilogue on the accumulators: the lane holds row lm, columns ln, ln+1
      // (tile 0) and ln+8, ln+9 (tile 1); one warp-uniform dispatch per
      // micro-op for all four values
      GEVO_TSTAMP(te0)
      GEVO_TACC(4, tc, te0)
      if (act0 && lm < pm) {
        const int m = (PANELS ? s * kPanel : 0) + lm;
        const double* Es = As + kTileElems;
        epi_lane4(R, ek, Es, ers, eks, acc, m, col0, lm, ln, ncols);
        double* orow = d.out + (int64_t)m * d.som + (int64_t)(col0 + ln) * d.son;
        const int64_t s1 = d.son, s8 = 8 * d.son;
        if (ln < ncols) orow[0] = acc[0];
        if (ln + 1 < ncols) orow[s1] = acc[1];
        if (act1 && ln + 8 < ncols) orow[s8] = acc[2];
        if (act1 && ln + 9 < ncols) orow[s8 + s1] = acc[3];
      }
      acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
      GEVO_TSTAMP(te1)
      GEVO_TACC(5, te0, te1)
    } else if (last) {
      __syncthreads();                // A consumed: its region becomes the C tile
      double* Cs = As;
      if (act0) {
        Cs[lm * kCS + ln] = acc[0];
        Cs[lm * kCS + ln + 1] = acc[1];
        Cs[lm * kCS + ln + 8] = acc[2];
        Cs[lm * kCS + ln + 9] = acc[3];
      }
      acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
      __syncthreads();
      const int m0 = PANELS ? s * kPanel : 0;
      GEVO_TSTAMP(te0)
      GEVO_TACC(4, tc, te0)
      dot_emit_dispatch<0>(ek, Cs, As + kTileElems, R, ers, eks, epi, d.out, d.som, d.son, m0, col0, pm, ncols);
      GEVO_TSTAMP(te1)
      GEVO_TACC(5, te0, te1)
    }
    slot = slot + 1 == kDotStages ? 0 : slot + 1;
    lslot = lslot + 1 == kDotStages ? 0 : lslot + 1;
    GEVO_TSTAMP(tf0)
    __syncthreads();
    GEVO_TSTAMP(tf1)
    GEVO_TACC(6, tf0, tf1)
  }
  cp_async_wait<0>();
}


// Weight-update shape (K <= 32, B persistent, 32-row panels, FMA chain, fast
// epilogue), software-pipelined: the DMMAs of panel s are issued before the
// epilogue of panel s-1 runs, so the tensor pipe works while the previous
// panel's operands are combined and stored.  The epilogue operands of a panel
// are copied to registers right after its DMMAs issue (the ring slot holding
// its full-matrix operand is refilled two panels later).
__device__ __forceinline__ void epi_load4(const EpiR& R, int ek, const double* Es, int ers, int eks, int m,
                                          int col0, int mm, int nn, int ncols, double (*o)[4]) {
  const int nx = ek == EK_SELECT ? 2 : R.nops;
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x) {
    if (x < nx) {
      const int src = R.src[x];
      if (src == ES_SCALAR) {
        const double sv = R.sval[x];
#pragma unroll
        for (int h = 0; h < 4; ++h) o[x][h] = sv;
      } else if (src == ES_TILE) {
        const double* e = Es + mm * ers + nn * eks;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = (h >> 1) * 8 + (h & 1);
          o[x][h] = nn + c < ncols ? e[c * eks] : 0.0;
        }
      } else {
        const int s1 = R.st1[x];
        const double* e = R.ptr[x] + (int64_t)m * R.st0[x] + (int64_t)(col0 + nn) * s1;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = (h >> 1) * 8 + (h & 1);
          o[x][h] = nn + c < ncols ? e[(int64_t)c * s1] : 0.0;
        }
      }
    }
  }
}

__device__ __forceinline__ void epi_apply4(const EpiR& R, int ek, double* v, const double (*o)[4]) {
  if (ek == EK_NONE) return;
  if (ek == EK_SELECT) {
    const bool left = R.fleft[0];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const bool p = as_i64(o[0][h]) != 0;
      v[h] = left ? (p ? v[h] : o[1][h]) : (p ? o[1][h] : v[h]);
    }
    return;
  }
  const int nx = R.nops;
#pragma unroll
  for (int x = 0; x < kEpiPre; ++x) {
    if (x < nx) {
      const bool left = R.fleft[x];
#define GEVO_PIPE_OP(EXPR)                                                  \
  _Pragma("unroll") for (int h = 0; h < 4; ++h) {                           \
    const double a = left ? v[h] : o[x][h], b = left ? o[x][h] : v[h];     \
    v[h] = (EXPR);                                                          \
  }
      switch (R.fsub[x]) {
        case GEVO_B_ADD: GEVO_PIPE_OP(__dadd_rn(a, b)); break;
        case GEVO_B_SUB: GEVO_PIPE_OP(__dsub_rn(a, b)); break;
        case GEVO_B_MUL: GEVO_PIPE_OP(__dmul_rn(a, b)); break;
        case GEVO_B_DIV: GEVO_PIPE_OP(__ddiv_rn(a, b)); break;
        default: GEVO_PIPE_OP(np_fmax(a, b)); break;
      }
#undef GEVO_PIPE_OP
    }
  }
}

__device__ __noinline__ void dot_panels_pipe(const DotArgs& dref, int col0, int col1, double* stage_buf,
                                             const EpiDev* epi) {
  const DotArgs d = dref;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int M = d.M, K = d.K, ncols = col1 - col0;
  const int ek = !epi ? EK_NONE : (epi->fast == 1 ? EK_CHAIN : EK_SELECT);
  __shared__ EpiR R;
  if (threadIdx.x == 0) epi_init(R, ek == EK_NONE ? nullptr : epi, true);
  __syncthreads();
  const bool etile = R.tile >= 0;
  const int total = (M + kPanel - 1) / kPanel;
  const uint32_t ring = smem_u32(stage_buf);
  double* Bp = stage_buf + kDotStages * 2 * kTileElems;
  VecCopy va, vx;
  vec_init(va, d.A, d.sam, d.sak, 32 * d.sam);
  if (etile) vec_init(vx, R.ptr[R.tile] + (int64_t)col0 * R.st1[R.tile], R.st0[R.tile], R.st1[R.tile],
                      32 * R.st0[R.tile]);
  else vx.kmaj = true;
  {
    CopyPlan pb;
    plan_init(pb, d.B + (int64_t)col0 * d.sbn, d.sbn, d.sbk, d.b_smem, false);
    stage(smem_u32(Bp), pb, plan_o0(pb), 0, ncols, 0, K);
  }
  const int brs = (d.b_smem || !(abs(d.sbk) != 0 && (d.sbn == 0 || abs(d.sbk) <= abs(d.sbn)))) ? 1 : kTS;
  // (B's smem layout as plan_init chose it: k-major iff k is the contiguous axis)
  const bool bkmaj = abs(d.sbk) != 0 && (d.sbn == 0 || abs(d.sbk) <= abs(d.sbn));
  const int brs2 = bkmaj ? kTS : 1, bks = bkmaj ? 1 : kTS;
  (void)brs;
  const int ars = va.kmaj ? kTS : 1, aks = va.kmaj ? 1 : kTS;
  const int ers = vx.kmaj ? kTS : 1, eks = vx.kmaj ? 1 : kTS;
  auto load = [&](int slot, int i) {
    const uint32_t As = ring + 8u * (slot * 2 * kTileElems);
    const int pm = min(kPanel, M - i * kPanel);
    vec_stage(va, As, pm, K);
    if (etile) vec_stage(vx, As + 8u * kTileElems, pm, ncols);
    va.p0 += va.adv;
    vx.p0 += vx.adv;
  };
  load(0, 0);
  cp_async_commit();
  if (total > 1) load(1, 1);
  cp_async_commit();

  const int rb = warp >> 1, cb0 = (warp & 1) * 2;
  const int lm = rb * 8 + g, ln = cb0 * 8 + 2 * t4;
  const bool c0 = cb0 * 8 < ncols, c1 = (cb0 + 1) * 8 < ncols;
  const int nq = K >> 2;
  const double* pb0 = Bp + (cb0 * 8 + g) * brs2 + t4 * bks;
  const double* pb1 = pb0 + 8 * brs2;
  double accA[4], accB[4], eo[kEpiPre][4];
  int slot = 0, lslot = 2;
  bool pend = false;
  int pm_prev = 0, m0_prev = 0;

  // one panel's DMMAs (into acc) with its K tail
  auto mma_panel = [&](double* acc, const double* As, int pm) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = 0.0;
    if (!(c0 && rb * 8 < pm)) return;
    const double* pa = As + lm * ars + t4 * aks;
    const int qa = 4 * aks, qb = 4 * bks;
    if (nq == 8 && c1) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double a = pa[q * qa];
        dmma884(acc[0], acc[1], a, pb0[q * qb]);
        dmma884(acc[2], acc[3], a, pb1[q * qb]);
      }
    } else {
      for (int q = 0; q < nq; ++q) {
        const double a = pa[q * qa];
        dmma884(acc[0], acc[1], a, pb0[q * qb]);
        if (c1) dmma884(acc[2], acc[3], a, pb1[q * qb]);
      }
      for (int kk = nq * 4; kk < K; ++kk) {
        const double a = As[lm * ars + kk * aks];
        acc[0] = fma(a, Bp[ln * brs2 + kk * bks], acc[0]);
        acc[1] = fma(a, Bp[(ln + 1) * brs2 + kk * bks], acc[1]);
        if (c1) {
          acc[2] = fma(a, Bp[(ln + 8) * brs2 + kk * bks], acc[2]);
          acc[3] = fma(a, Bp[(ln + 9) * brs2 + kk * bks], acc[3]);
        }
      }
    }
  };
  auto emit_panel = [&](double* acc, int m0, int pm) {
    if (!(c0 && lm < pm)) return;
    const int m = m0 + lm;
    epi_apply4(R, ek, acc, eo);
    double* orow = d.out + (int64_t)m * d.som + (int64_t)(col0 + ln) * d.son;
    const int64_t s1 = d.son, s8 = 8 * d.son;
    if (ln < ncols) orow[0] = acc[0];
    if (ln + 1 < ncols) orow[s1] = acc[1];
    if (c1 && ln + 8 < ncols) orow[s8] = acc[2];
    if (c1 && ln + 9 < ncols) orow[s8 + s1] = acc[3];
  };
  auto stage_body = [&](double* cur, double* prev, int s) {
    cp_async_wait<1>();                       // panel s (committed an iteration ago)
    __syncthreads();
    double* As = stage_buf + slot * 2 * kTileElems;
    const int pm = min(kPanel, M - s * kPanel);
    mma_panel(cur, As, pm);                   // tensor pipe busy ...
    if (s + 2 < total) load(lslot, s + 2);    // ... while panel s+2 is fetched
    cp_async_commit();
    if (pend) emit_panel(prev, m0_prev, pm_prev);   // ... while panel s-1 is finished
    if (ek != EK_NONE && c0 && lm < pm)
      epi_load4(R, ek, As + kTileElems, ers, eks, s * kPanel + lm, col0, lm, ln, ncols, eo);
    pend = true;
    pm_prev = pm;
    m0_prev = s * kPanel;
    slot = slot == 2 ? 0 : slot + 1;
    lslot = lslot == 2 ? 0 : lslot + 1;
    __syncthreads();
  };
#pragma unroll 1
  for (int s = 0; s < total; s += 2) {
    stage_body(accA, accB, s);
    if (s + 1 < total) stage_body(accB, accA, s + 1);
  }
  if (pend) emit_panel((total & 1) ? accA : accB, m0_prev, pm_prev);
  cp_async_wait<0>();
  __syncthreads();
}

// CK: 0 FMA_CHAIN, 1 ACC8 (8 lane chains (k mod 8) per output, each on its
// own DMMA accumulator tile, chain j's four k of a chunk (j, j+8, j+16, j+24)
// read from the unpermuted tile with stride 8; warp = an 8x16 strip, two
// tiles x 8 chains, so a 32-column piece is one pass), 2 SEQ_NOFMA, 3 integer (scalar; thread = 4 outputs of the panel).
template <bool PANELS, int CK>
__device__ __noinline__ void dot_fast(const DotArgs& dref, int col0, int col1, double* stage_buf,
                                      const EpiDev* epi, int mode) {
  constexpr bool ACC8 = CK == 1;
  constexpr bool SCALAR = CK >= 2;
  const DotArgs d = dref;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int M = d.M, K = d.K, ncols = col1 - col0;
  const int ek = !epi ? EK_NONE : (epi->fast == 1 ? EK_CHAIN : (epi->fast == 2 ? EK_SELECT : EK_GENERIC));
  __shared__ EpiR R;
  __shared__ CopyPlan cpa, cpx, cpb;
  if (threadIdx.x == 0) epi_init(R, ek == EK_CHAIN || ek == EK_SELECT ? epi : nullptr, PANELS);
  __syncthreads();
  const bool etile = PANELS && R.tile >= 0;
  const int total = PANELS ? (M + kPanel - 1) / kPanel : (K + kKC - 1) / kKC;
  const uint32_t ring = smem_u32(stage_buf);
  double* Bp = stage_buf + kDotStages * 2 * kTileElems;

  // A; the second tile (B chunk for KSTREAM, epilogue operand for PANELS)
  Feed fa, fx;
  int brs, bks;
  if (PANELS) {
    feed_init(fa, cpa, d.A, d.sam, d.sak, d.a_smem, 0, 0, kPanel * d.sam, M, K);
    if (etile)
      feed_init(fx, cpx, R.ptr[R.tile], R.st0[R.tile], R.st1[R.tile], false, 0, col0, kPanel * R.st0[R.tile],
                M, ncols);
    else
      fx.flags = 3;
    // B (K x ncols) once, any layout
    if (threadIdx.x == 0) plan_init(cpb, d.B + (int64_t)col0 * d.sbn, d.sbn, d.sbk, d.b_smem, false);
    __syncthreads();
    stage(smem_u32(Bp), cpb, plan_o0(cpb), 0, ncols, 0, K);
    brs = cp_rs(cpb);
    bks = cp_ks(cpb);
  } else {
    feed_init(fa, cpa, d.A, d.sam, d.sak, d.a_smem, 0, 0, kKC * d.sak, M, K);
    feed_init(fx, cpx, d.B, d.sbn, d.sbk, d.b_smem, col0, 0, kKC * d.sbk, ncols, K);
    brs = feed_rs(fx);
    bks = feed_ks(fx);
  }
  const int ars = feed_rs(fa), aks = feed_ks(fa);
  const int ers = feed_rs(fx), eks = feed_ks(fx);

  // stage i covers rows [32i, ..) (PANELS) or k [32i, ..) (KSTREAM)
  auto load = [&](int i, int slot) {
    const uint32_t As = ring + 8u * (slot * 2 * kTileElems);
    if (PANELS) {
      const int pm = min(kPanel, M - i * kPanel);
      feed_stage<kPanel, 0>(fa, cpa, As, pm, K);
      if (etile) feed_stage<kPanel, 0>(fx, cpx, As + 8u * kTileElems, pm, ncols);
    } else {
      const int nk = min(kKC, K - i * kKC);
      feed_stage<0, kKC>(fa, cpa, As, M, nk);
      feed_stage<0, kKC>(fx, cpx, As + 8u * kTileElems, ncols, nk);
    }
  };
#pragma unroll 1
  for (int i = 0; i < kDotStages - 1; ++i) {
    if (i < total) load(i, i);
    cp_async_commit();
  }
  const int rb = warp >> 1, cb0 = (warp & 1) * 2;      // warp = 8 x 16 strip (two tiles)
  const int lm = rb * 8 + g, ln = cb0 * 8 + 2 * t4;
  const int kmain = (ACC8 && mode == GEVO_D_ACC8_TAIL) ? (K & ~7) : K;
  constexpr int NACC = ACC8 ? 32 : 4;                  // ACC8: 2 tiles x 8 chains x 2
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  int slot = 0, lslot = kDotStages - 1;
#pragma unroll 1
  for (int s = 0; s < total; ++s) {
    GEVO_TSTAMP(ta)
    if (s + kDotStages - 1 < total) load(s + kDotStages - 1, lslot);
    cp_async_commit();
    GEVO_TSTAMP(tl)
    cp_async_wait<kDotStages - 1>();
    __syncthreads();
    GEVO_TSTAMP(tb)
    GEVO_TACC(1, ta, tl)
    GEVO_TACC(2, tl, tb)
    double* As = stage_buf + slot * 2 * kTileElems;
    const double* Bs = PANELS ? Bp : As + kTileElems;
    const int pm = PANELS ? min(kPanel, M - s * kPanel) : M;
    const int nk = PANELS ? K : min(kKC, K - s * kKC);    const bool last = PANELS || s == total - 1;
    const bool act0 = !SCALAR && rb * 8 < pm && cb0 * 8 < ncols;
    const bool act1 = act0 && (cb0 + 1) * 8 < ncols;
    if (SCALAR) {
      // the thread's 4 outputs (rows mm + 8u, column nn) advance together so
      // their 4 dependent chains overlap; invalid rows compute garbage that is
      // never stored
      const int mm = threadIdx.x >> 5, nn = threadIdx.x & 31;
      const double* pa = As + mm * ars;
      const double* pb = Bs + nn * brs;
      const int ra = 8 * ars;
      if (CK == 2) {
#pragma unroll 4
        for (int kk = 0; kk < nk; ++kk) {
          const double b = pb[kk * bks];
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[u] = __dadd_rn(acc[u], __dmul_rn(pa[u * ra + kk * aks], b));
        }
      } else {
#pragma unroll 4
        for (int kk = 0; kk < nk; ++kk) {
          const uint64_t b = (uint64_t)as_i64(pb[kk * bks]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            acc[u] = as_w((int64_t)((uint64_t)as_i64(acc[u]) + (uint64_t)as_i64(pa[u * ra + kk * aks]) * b));
        }
      }
    }
    if (ACC8 && act0) {
      const int k0 = PANELS ? 0 : s * kKC;
      const double* pa = As + lm * ars + 8 * t4 * aks;
      const double* pb = Bs + (cb0 * 8 + g) * brs + 8 * t4 * bks;
      const double* pb1 = pb + 8 * brs;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (k0 + j + 24 < kmain) {
          const double a = pa[j * aks];
          dmma884(acc[2 * j], acc[2 * j + 1], a, pb[j * bks]);
          if (act1) dmma884(acc[16 + 2 * j], acc[17 + 2 * j], a, pb1[j * bks]);
        } else {
#pragma unroll 1
          for (int t = 0; t < 4; ++t) {
            const int kk = j + 8 * t;
            if (k0 + kk >= kmain) break;
            const double a = As[lm * ars + kk * aks];
            acc[2 * j] = fma(a, Bs[ln * brs + kk * bks], acc[2 * j]);
            acc[2 * j + 1] = fma(a, Bs[(ln + 1) * brs + kk * bks], acc[2 * j + 1]);
            if (act1) {
              acc[16 + 2 * j] = fma(a, Bs[(ln + 8) * brs + kk * bks], acc[16 + 2 * j]);
              acc[17 + 2 * j] = fma(a, Bs[(ln + 9) * brs + kk * bks], acc[17 + 2 * j]);
            }
          }
        }
      }
      if (last) {
        // pairwise lane tree, then (ACC8_TAIL) the fma tail over k >= K&~7
        const bool avx = (PANELS ? s * kPanel : 0) + lm >= d.xrow;
        double r0 = lane_tree(acc, 0, avx);
        double r1 = lane_tree(acc, 1, avx);
        double r2 = lane_tree(acc + 16, 0, avx);
        double r3 = lane_tree(acc + 16, 1, avx);
#pragma unroll 1
        for (int kk = kmain - k0; kk < nk; ++kk) {
          const double a = As[lm * ars + kk * aks];
          r0 = fma(a, Bs[ln * brs + kk * bks], r0);
          r1 = fma(a, Bs[(ln + 1) * brs + kk * bks], r1);
          if (act1) {
            r2 = fma(a, Bs[(ln + 8) * brs + kk * bks], r2);
            r3 = fma(a, Bs[(ln + 9) * brs + kk * bks], r3);
          }
        }
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
        acc[0] = r0;
        acc[1] = r1;
        acc[2] = r2;
        acc[3] = r3;
      }
    } else if (!ACC8 && act0) {
      const double* pa = As + lm * ars + t4 * aks;
      const double* pb0 = Bs + (cb0 * 8 + g) * brs + t4 * bks;
      const double* pb1 = pb0 + 8 * brs;
      const int nq = nk >> 2;
      const int qa = 4 * aks, qb = 4 * bks;
      if (nq == 8 && act1) {
        // all 24 fragments first (one LDS latency), then 16 back-to-back DMMAs
        double fa[8], fb0[8], fb1[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          fa[q] = pa[q * qa];
          fb0[q] = pb0[q * qb];
          fb1[q] = pb1[q * qb];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          dmma884(acc[0], acc[1], fa[q], fb0[q]);
          dmma884(acc[2], acc[3], fa[q], fb1[q]);
        }
      } else {
#pragma unroll 1
        for (int q = 0; q < nq; ++q) {
          const double a = pa[q * qa];
          dmma884(acc[0], acc[1], a, pb0[q * qb]);
          if (act1) dmma884(acc[2], acc[3], a, pb1[q * qb]);
        }
#pragma unroll 1
        for (int kk = nq * 4; kk < nk; ++kk) {
          const double a = As[lm * ars + kk * aks];
          acc[0] = fma(a, Bs[ln * brs + kk * bks], acc[0]);
          acc[1] = fma(a, Bs[(ln + 1) * brs + kk * bks], acc[1]);
          if (act1) {
            acc[2] = fma(a, Bs[(ln + 8) * brs + kk * bks], acc[2]);
            acc[3] = fma(a, Bs[(ln + 9) * brs + kk * bks], acc[3]);
          }
        }
      }
    }
    GEVO_TSTAMP(tc)
    GEVO_TACC(3, tb, tc)
    if (last) {
      __syncthreads();                // A consumed: its region becomes the C tile
      double* Cs = As;
      if (SCALAR) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o = threadIdx.x + u * kDotThreads;
          Cs[(o >> 5) * kCS + (o & 31)] = acc[u];
        }
      } else if (act0) {
        Cs[lm * kCS + ln] = acc[0];
        Cs[lm * kCS + ln + 1] = acc[1];
        if (!ACC8 || act1) {
          Cs[lm * kCS + ln + 8] = acc[2];
          Cs[lm * kCS + ln + 9] = acc[3];
        }
      }
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
      __syncthreads();
      const int m0 = PANELS ? s * kPanel : 0;
      GEVO_TSTAMP(te0)
      GEVO_TACC(4, tc, te0)
      dot_emit_dispatch<0>(ek, Cs, As + kTileElems, R, ers, eks, epi, d.out, d.som, d.son, m0, col0, pm, ncols);
      GEVO_TSTAMP(te1)
      GEVO_TACC(5, te0, te1)
    }
    slot = slot + 1 == kDotStages ? 0 : slot + 1;
    lslot = lslot + 1 == kDotStages ? 0 : lslot + 1;
    GEVO_TSTAMP(tf0)
    __syncthreads();
    GEVO_TSTAMP(tf1)
    GEVO_TACC(6, tf0, tf1)
  }
  cp_async_wait<0>();
}


// ---------------------------------------------------------------------------
// Tiny dots (M, N, K <= 32: the hidden/output-layer dots of the MLP step):
// no staging -- each lane reads its DMMA fragments straight from the
// operands (shared-memory arena or global) and applies the epilogue to its
// own outputs.  FMA: warp = 8x16 strip (two tiles); ACC8: warp = one 8x8
// tile with its 8 lane chains.
template <bool ACC8, int EK>
__device__ __noinline__ void dot_tiny(const DotArgs& dref, int col0, int col1, const EpiDev* epi,
                                      const EpiR& R, int mode) {
  const DotArgs d = dref;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int M = d.M, K = d.K, ncols = col1 - col0;
  const int rb = warp >> 1, cb0 = ACC8 ? (warp & 1) : (warp & 1) * 2;
  if (rb * 8 >= M || cb0 * 8 >= ncols) return;
  const int ntile = ACC8 ? 1 : ((cb0 + 1) * 8 < ncols ? 2 : 1);
  const int m = rb * 8 + g;
  const int mc = min(m, M - 1);                        // clamped (valid) row for loads
  double acc[ACC8 ? 16 : 4];
#pragma unroll
  for (int i = 0; i < (ACC8 ? 16 : 4); ++i) acc[i] = 0.0;
  const double* arow = d.A + (int64_t)mc * d.sam;
  int bcol[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) bcol[t] = col0 + min((cb0 + t) * 8 + g, ncols - 1);
  if (!ACC8) {
    const int nq = K >> 2;
#pragma unroll 8
    for (int q = 0; q < nq; ++q) {
      const int k = 4 * q + t4;
      const double a = arow[(int64_t)k * d.sak];
      dmma884(acc[0], acc[1], a, d.B[(int64_t)k * d.sbk + (int64_t)bcol[0] * d.sbn]);
      if (ntile > 1) dmma884(acc[2], acc[3], a, d.B[(int64_t)k * d.sbk + (int64_t)bcol[1] * d.sbn]);
    }
    for (int k = nq * 4; k < K; ++k) {                 // k tail: scalar fma chain
      const double a = arow[(int64_t)k * d.sak];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int nn = (h >> 1) * 8 + 2 * t4 + (h & 1);
        if ((h < 2 || ntile > 1) && cb0 * 8 + nn < ncols)
          acc[h] = fma(a, d.B[(int64_t)k * d.sbk + (int64_t)(col0 + cb0 * 8 + nn) * d.sbn], acc[h]);
      }
    }
  } else {
    const int kmain = mode == GEVO_D_ACC8_TAIL ? (K & ~7) : K;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      for (int k0 = 0; k0 < kmain; k0 += 32) {
        if (k0 + j + 24 < kmain) {
          const int k = k0 + j + 8 * t4;
          dmma884(acc[2 * j], acc[2 * j + 1], arow[(int64_t)k * d.sak],
                  d.B[(int64_t)k * d.sbk + (int64_t)bcol[0] * d.sbn]);
        } else {
          for (int t = 0; t < 4; ++t) {
            const int k = k0 + j + 8 * t;
            if (k >= kmain) break;
            const double a = arow[(int64_t)k * d.sak];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int nn = cb0 * 8 + 2 * t4 + h;
              if (nn < ncols)
                acc[2 * j + h] = fma(a, d.B[(int64_t)k * d.sbk + (int64_t)(col0 + nn) * d.sbn], acc[2 * j + h]);
            }
          }
        }
      }
    }
    double r[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      r[h] = lane_tree(acc, h, m >= d.xrow);
      const int nn = cb0 * 8 + 2 * t4 + h;
      for (int k = kmain; k < K; ++k)                  // ACC8_TAIL
        if (nn < ncols)
          r[h] = fma(arow[(int64_t)k * d.sak], d.B[(int64_t)k * d.sbk + (int64_t)(col0 + nn) * d.sbn], r[h]);
    }
    acc[0] = r[0];
    acc[1] = r[1];
  }
  if (m >= M) return;
  double* orow = d.out + (int64_t)m * d.som;
#pragma unroll
  for (int h = 0; h < (ACC8 ? 2 : 4); ++h) {
    const int nn = cb0 * 8 + (h >> 1) * 8 + 2 * t4 + (h & 1);
    if ((h < 2 || ntile > 1) && nn < ncols) {
      const int n = col0 + nn;
      double v = acc[h];
      if (EK == EK_CHAIN) {
#pragma unroll
        for (int x = 0; x < kEpiPre; ++x) {
          if (x < R.nops) {
            const double o = R.src[x] == ES_SCALAR ? R.sval[x]
                                                   : R.ptr[x][(int64_t)m * R.st0[x] + (int64_t)n * R.st1[x]];
            v = R.fleft[x] ? bin_f64(R.fsub[x], v, o) : bin_f64(R.fsub[x], o, v);
          }
        }
      } else if (EK == EK_SELECT) {
        const double o0 = R.src[0] == ES_SCALAR ? R.sval[0]
                                                : R.ptr[0][(int64_t)m * R.st0[0] + (int64_t)n * R.st1[0]];
        const double o1 = R.src[1] == ES_SCALAR ? R.sval[1]
                                                : R.ptr[1][(int64_t)m * R.st0[1] + (int64_t)n * R.st1[1]];
        const bool p = as_i64(o0) != 0;
        v = R.fleft[0] ? (p ? v : o1) : (p ? o1 : v);
      } else if (EK == EK_GENERIC) {
        double ev[kEpiPre];
        epi_fetch(*epi, m, n, ev);
        v = epilogue_generic(*epi, ev, v, m, n);
      }
      orow[(int64_t)n * d.son] = v;
    }
  }
}

__device__ __forceinline__ void dot_tiny_dispatch(const DotArgs& d, int col0, int col1, const EpiDev* epi,
                                                  bool acc8, int mode) {
  __shared__ EpiR R;
  const int ek = !epi ? EK_NONE : (epi->fast == 1 ? EK_CHAIN : (epi->fast == 2 ? EK_SELECT : EK_GENERIC));
  if (threadIdx.x == 0) epi_init(R, ek == EK_CHAIN || ek == EK_SELECT ? epi : nullptr, false);
  __syncthreads();
#define GEVO_TINY(A8)                                                         \
  switch (ek) {                                                               \
    case EK_NONE: dot_tiny<A8, EK_NONE>(d, col0, col1, epi, R, mode); break;  \
    case EK_CHAIN: dot_tiny<A8, EK_CHAIN>(d, col0, col1, epi, R, mode); break; \
    case EK_SELECT: dot_tiny<A8, EK_SELECT>(d, col0, col1, epi, R, mode); break; \
    default: dot_tiny<A8, EK_GENERIC>(d, col0, col1, epi, R, mode); break;     \
  }
  if (acc8) { GEVO_TINY(true) } else { GEVO_TINY(false) }
#undef GEVO_TINY
  __syncthreads();
}

// PANELS needs its tile-staged epilogue operand (the first full-matrix one,
// see epi_init) to be made of whole aligned lines
__device__ __forceinline__ bool dot_etile_ok(const EpiDev* e, int ncols, int M) {
  for (int x = 0; x < kEpiPre && x < e->next; ++x) {
    if ((e->st0[x] == 0 && e->st1[x] == 0) || e->st0[x] == 0 || e->st1[x] == 0 || __isShared(e->ptr[x])) continue;
    return vec_ok(e->ptr[x], (int)e->st0[x], (int)e->st1[x], M, ncols);
  }
  return true;
}

// columns [col0, col1) of a DOT in summation order `mode`
__device__ __forceinline__ void dot_columns(const DotArgs& d, int col0, int col1, int mode, bool integer,
                                            double* stage_buf, const EpiDev* epi) {
  if (col0 >= col1) return;
  // fast paths (one <= 32-row panel with K streamed, or K <= 32 with rows
  // streamed), in column pieces of <= 32; the general
  // pipeline otherwise
  const int ck = integer ? 3 : (mode == GEVO_D_SEQ_NOFMA ? 2 : (mode == GEVO_D_FMA_CHAIN ? 0 : 1));
  const int width = kPanel;
  if (ck <= 1 && d.M <= kPanel && d.K <= kKC && col1 - col0 <= (ck == 1 ? 16 : kPanel)) {
    dot_tiny_dispatch(d, col0, col1, epi, ck == 1, mode);
    return;
  }
  const bool kstream = d.M <= kPanel && d.K > kKC;
  const bool panels = d.K <= kKC && (!epi || epi->fast == 0 || dot_etile_ok(epi, col1 - col0, d.M));
  if (kstream || panels) {
    for (int c = col0; c < col1; c += width) {
      const int c1 = min(c + width, col1);
      if (ck == 0 && !d.a_smem && vec_ok(d.A, d.sam, d.sak, d.M, d.K) &&
          (kstream ? (!d.b_smem && vec_ok(d.B + (int64_t)c * d.sbn, d.sbn, d.sbk, c1 - c, d.K)) : true)) {
        if (kstream) dot_fast_vec<false>(d, c, c1, stage_buf, epi);
        else if (!epi || epi->fast != 0) dot_panels_pipe(d, c, c1, stage_buf, epi);
        else dot_fast_vec<true>(d, c, c1, stage_buf, epi);
        continue;
      }
      if (kstream) {
        switch (ck) {
          case 0: dot_fast<false, 0>(d, c, c1, stage_buf, epi, mode); break;
          case 1: dot_fast<false, 1>(d, c, c1, stage_buf, epi, mode); break;
          case 2: dot_fast<false, 2>(d, c, c1, stage_buf, epi, mode); break;
          default: dot_fast<false, 3>(d, c, c1, stage_buf, epi, mode); break;
        }
      } else {
        switch (ck) {
          case 0: dot_fast<true, 0>(d, c, c1, stage_buf, epi, mode); break;
          case 1: dot_fast<true, 1>(d, c, c1, stage_buf, epi, mode); break;
          case 2: dot_fast<true, 2>(d, c, c1, stage_buf, epi, mode); break;
          default: dot_fast<true, 3>(d, c, c1, stage_buf, epi, mode); break;
        }
      }
    }
    return;
  }
  switch (ck) {
    case 0: dot_run<0>(d, col0, col1, mode, stage_buf, epi); break;
    case 1: dot_run<1>(d, col0, col1, mode, stage_buf, epi); break;
    case 2: dot_run<2>(d, col0, col1, mode, stage_buf, epi); break;
    default: dot_run<3>(d, col0, col1, mode, stage_buf, epi); break;
  }
}

}  // namespace gevo
