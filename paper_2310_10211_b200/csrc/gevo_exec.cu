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
#include "gevo_plan.h"
#include "exec_core.cuh"
#include "exp_np.cuh"
#include "gevo_exec.cuh"

namespace gevo {

constexpr int kThreads = 256;
constexpr int kInstrCache = 80;   // instructions staged in shared memory

struct Shared {
  double* base[GEVO_NBUF];
  int flag;
  int wrong;
};

__device__ __forceinline__ double* opptr(const Shared& S, const gevo_operand& o) {
  return S.base[o.buf];
}

// elementwise (UNARY / BINARY / SELECT) over the output shape
__device__ void run_elementwise(const Shared& S, const gevo_instr& I) {
  const int n = I.n;
  const int rank = I.rank;
  double* out = opptr(S, I.out);
  const double* in0 = opptr(S, I.in[0]);
  const double* in1 = I.op >= GEVO_OP_BINARY ? opptr(S, I.in[1]) : nullptr;
  const double* in2 = I.op == GEVO_OP_SELECT ? opptr(S, I.in[2]) : nullptr;
  const int am_out = I.aux2[0], am0 = I.aux2[1], am1 = I.aux2[2], am2 = I.aux2[3];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int idx[GEVO_MAXR];
    if (am_out == AM_STRIDED || am0 == AM_STRIDED || am1 == AM_STRIDED || am2 == AM_STRIDED)
      unravel(i, rank, I.shp, idx);
    auto ad = [&](const gevo_operand& o, int am) -> int64_t {
      if (am == AM_LINEAR) return o.off + i;
      if (am == AM_SCALAR) return o.off;
      return addr(o, idx, rank);
    };
    double a = in0[ad(I.in[0], am0)];
    double r;
    if (I.op == GEVO_OP_UNARY) {
      r = apply_unary(I.sub, I.kin, I.kout, a);
    } else if (I.op == GEVO_OP_BINARY) {
      r = apply_binary(I.sub, I.kin, a, in1[ad(I.in[1], am1)]);
    } else {
      r = as_i64(a) != 0 ? in1[ad(I.in[1], am1)] : in2[ad(I.in[2], am2)];
    }
    out[ad(I.out, am_out)] = r;
  }
}

__device__ void run_pad(const Shared& S, const gevo_instr& I) {
  double* out = opptr(S, I.out);
  const double* in = opptr(S, I.in[0]);
  const double pv = opptr(S, I.in[1])[I.in[1].off];
  for (int i = threadIdx.x; i < I.n; i += blockDim.x) {
    int idx[GEVO_MAXR];
    unravel(i, I.rank, I.shp, idx);
    bool inside = true;
    int64_t src = I.in[0].off;
#pragma unroll
    for (int d = 0; d < GEVO_MAXR; ++d) {
      if (d < I.rank) {
        int j = idx[d] - I.aux[d];
        inside = inside && j >= 0 && j < I.aux2[d];
        src += (int64_t)j * I.in[0].st[d];
      }
    }
    out[addr(I.out, idx, I.rank)] = inside ? in[src] : pv;
  }
}

__device__ void run_reduce(const Shared& S, const gevo_instr& I) {
  double* out = opptr(S, I.out);
  const double* in = opptr(S, I.in[0]);
  const int L = I.aux[0];
  const int64_t rs = I.aux[1];
  for (int i = threadIdx.x; i < I.n; i += blockDim.x) {
    int idx[GEVO_MAXR];
    unravel(i, I.rank, I.shp, idx);
    const double* p = in + addr(I.in[0], idx, I.rank);
    double r;
    if (I.kin == GEVO_K_F64) {
      if (I.sub == GEVO_R_MAX) {
        r = p[0];
        for (int k = 1; k < L; ++k) r = np_fmax(r, p[k * rs]);
      } else if (I.sub == GEVO_R_SUM_PAIRWISE) {
        r = pairwise_sum(p, L, rs);
      } else {
        r = 0.0;
        for (int k = 0; k < L; ++k) r = __dadd_rn(r, p[k * rs]);
      }
    } else {
      int64_t v;
      if (I.sub == GEVO_R_MAX) {
        v = as_i64(p[0]);
        for (int k = 1; k < L; ++k) { int64_t x = as_i64(p[k * rs]); v = x > v ? x : v; }
      } else {
        uint64_t acc = 0;
        for (int k = 0; k < L; ++k) acc += (uint64_t)as_i64(p[k * rs]);
        v = (int64_t)acc;
      }
      r = as_w(v);
    }
    out[addr(I.out, idx, I.rank)] = r;
  }
}

__device__ __forceinline__ double dot_elem(int mode, const double* a, int64_t sa,
                                           const double* b, int64_t sb, int K) {
  if (mode == GEVO_D_FMA_CHAIN) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc = fma(a[k * sa], b[k * sb], acc);
    return acc;
  }
  if (mode == GEVO_D_SEQ_NOFMA) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k * sa], b[k * sb]));
    return acc;
  }
  // 8 lane accumulators over k, then the pairwise lane tree
  double l[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) l[j] = 0.0;
  int kmain = (mode == GEVO_D_ACC8_TAIL) ? (K & ~7) : K;
  for (int k = 0; k < kmain; ++k) l[k & 7] = fma(a[k * sa], b[k * sb], l[k & 7]);
  double r = __dadd_rn(__dadd_rn(__dadd_rn(l[0], l[1]), __dadd_rn(l[2], l[3])),
                       __dadd_rn(__dadd_rn(l[4], l[5]), __dadd_rn(l[6], l[7])));
  for (int k = kmain; k < K; ++k) r = fma(a[k * sa], b[k * sb], r);
  return r;
}

// D(8x8) += A(8x4) B(4x8) on the FP64 tensor path.  Probed on B200:
// bit-identical to four chained fma() in k order (tests/tools/dmma_probe.cu),
// so an 8x8 tile accumulated over k0 = 0, 4, 8, ... reproduces the
// reference's single-accumulator FMA chain (OpenBLAS dgemm kernels) exactly.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// FMA-chain dot over output columns [0, ncols): one warp owns an 8x16 strip
// (two 8x8 tiles sharing the A fragment) for the whole K range -- never a
// split-K, which would change the summation order.
__device__ void dot_fma_dmma(const gevo_instr& I, double* out, const double* A,
                             const double* B, int ncols) {
  const int M = I.shp[0], K = I.aux[0];
  const int64_t sam = I.in[0].st[0], sak = I.in[0].st[1];
  const int64_t sbk = I.in[1].st[0], sbn = I.in[1].st[1];
  const int64_t som = I.out.st[0], son = I.out.st[1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int tm = (M + 7) >> 3, tn2 = (ncols + 15) >> 4;
  const int K4 = K & ~3;
  A += I.in[0].off;
  B += I.in[1].off;
  for (int tile = warp; tile < tm * tn2; tile += nwarp) {
    const int ti = tile / tn2, tj = tile - ti * tn2;
    const int i = ti * 8 + g;                 // A-fragment row of this lane
    const int j0 = tj * 16 + g, j1 = j0 + 8;  // B-fragment columns of this lane
    const bool vi = i < M, v0 = j0 < ncols, v1 = j1 < ncols;
    const double* pa = A + (vi ? i : 0) * sam + t4 * sak;
    const double* pb0 = B + (v0 ? j0 : 0) * sbn + t4 * sbk;
    const double* pb1 = B + (v1 ? j1 : 0) * sbn + t4 * sbk;
    const int64_t ska = 4 * sak, skb = 4 * sbk;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < K4; k0 += 4) {
      const double a = vi ? *pa : 0.0;
      const double b0 = v0 ? *pb0 : 0.0;
      const double b1 = v1 ? *pb1 : 0.0;
      dmma884(c00, c01, a, b0);
      dmma884(c10, c11, a, b1);
      pa += ska;
      pb0 += skb;
      pb1 += skb;
    }
    // D fragment: row ti*8+g, columns tj*16 + {2t4, 2t4+1} and +8
    const int r = ti * 8 + g;
    const int cA = tj * 16 + 2 * t4, cB = cA + 8;
    if (K4 < K && r < M) {                    // k tail, same chain order
      const double* ar = A + r * sam;
      for (int k = K4; k < K; ++k) {
        const double a = ar[k * sak];
        const double* bk = B + k * sbk;
        if (cA < ncols) c00 = fma(a, bk[cA * sbn], c00);
        if (cA + 1 < ncols) c01 = fma(a, bk[(cA + 1) * sbn], c01);
        if (cB < ncols) c10 = fma(a, bk[cB * sbn], c10);
        if (cB + 1 < ncols) c11 = fma(a, bk[(cB + 1) * sbn], c11);
      }
    }
    if (r < M) {
      double* o = out + I.out.off + r * som;
      if (cA < ncols) o[cA * son] = c00;
      if (cA + 1 < ncols) o[(cA + 1) * son] = c01;
      if (cB < ncols) o[cB * son] = c10;
      if (cB + 1 < ncols) o[(cB + 1) * son] = c11;
    }
  }
}

__device__ void run_dot(const Shared& S, const gevo_instr& I) {
  double* out = opptr(S, I.out);
  const double* A = opptr(S, I.in[0]);
  const double* B = opptr(S, I.in[1]);
  const int M = I.shp[0], N = I.shp[1], K = I.aux[0];
  int split = I.aux[1];
  const int64_t sam = I.in[0].st[0], sak = I.in[0].st[1];
  const int64_t sbk = I.in[1].st[0], sbn = I.in[1].st[1];
  const bool f = I.kin == GEVO_K_F64;
  int first = 0;  // columns [0, first) done on the tensor path
  if (f && I.sub == GEVO_D_FMA_CHAIN && split > 0) {
    dot_fma_dmma(I, out, A, B, split);
    first = split;
    if (first >= N) return;
  }
  const int span = N - first;
  for (int e = threadIdx.x; e < M * span; e += blockDim.x) {
    int i = e / span, j = first + (e - i * span);
    const double* a = A + I.in[0].off + i * sam;
    const double* b = B + I.in[1].off + j * sbn;
    double r;
    if (f) {
      r = dot_elem(j < split ? I.sub : I.aux[2], a, sak, b, sbk, K);
    } else {
      uint64_t acc = 0;
      for (int k = 0; k < K; ++k)
        acc += (uint64_t)as_i64(a[k * sak]) * (uint64_t)as_i64(b[k * sbk]);
      r = as_w((int64_t)acc);
    }
    out[I.out.off + (int64_t)i * I.out.st[0] + (int64_t)j * I.out.st[1]] = r;
  }
}

__device__ void run_instrs(const Shared& S, const gevo_instr* ins, int n) {
  for (int k = 0; k < n; ++k) {
    const gevo_instr& I = ins[k];
    switch (I.op) {
      case GEVO_OP_UNARY:
      case GEVO_OP_BINARY:
      case GEVO_OP_SELECT: run_elementwise(S, I); break;
      case GEVO_OP_REDUCE: run_reduce(S, I); break;
      case GEVO_OP_DOT: run_dot(S, I); break;
      case GEVO_OP_PAD: run_pad(S, I); break;
    }
    __syncthreads();
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

__device__ bool all_finite(const double* w, int n) {
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) bad |= !isfinite(w[i]);
  return !__syncthreads_or(bad);
}

__global__ void __launch_bounds__(kThreads)
eval_kernel(EvalArgs args) {
  __shared__ Shared S;
  __shared__ gevo_instr cache[kInstrCache];
  const gevo_prog P = args.progs[blockIdx.x];
  double* ind = args.arena + P.arena_off;
  const int wsz = (args.weight_elems + 15) & ~15;
  const int psz = (args.probs_elems + 15) & ~15;
  double* scratch = ind;
  double* probs = ind + P.arena_elems;
  double* wbuf[2] = {probs + psz, probs + psz + wsz};
  const double* consts = args.consts + P.const_off;
  const int nw = args.n_weights;
  int status = GEVO_STATUS_OK;
  int steps_run = 0;

  const double* final_w = args.init_weights;
  if (args.mode == GEVO_MODE_TRAIN && args.steps > 0) {
    const gevo_instr* t0 = stage(cache, args.instrs + P.train0, P.train0_n);
    const gevo_instr* cur = t0;
    const int check = args.check_every > 0 ? args.check_every : 1;
    for (int s = 0; s < args.steps; ++s) {
      if (s == 1 && P.train1 != P.train0) {
        __syncthreads();
        cur = stage(cache, args.instrs + P.train1, P.train1_n);
      }
      const double* win = (s == 0) ? args.init_weights : wbuf[s & 1];
      double* wout = wbuf[(s + 1) & 1];
      const int b = s % args.train_nb;
      if (threadIdx.x == 0) {
        S.base[GEVO_BUF_ARENA] = scratch;
        S.base[GEVO_BUF_CONST] = const_cast<double*>(consts);
        for (int i = 0; i < nw; ++i) {
          S.base[GEVO_BUF_PARAM0 + i] = const_cast<double*>(win) + args.wofs[i];
          S.base[GEVO_BUF_OUT0 + i] = wout + args.wofs[i];
        }
        S.base[GEVO_BUF_PARAM0 + nw] = const_cast<double*>(args.train_x) + (int64_t)b * args.x_elems;
        S.base[GEVO_BUF_PARAM0 + nw + 1] = const_cast<double*>(args.train_y) + (int64_t)b * args.y_elems;
      }
      __syncthreads();
      run_instrs(S, cur, (s == 0) ? P.train0_n : P.train1_n);
      steps_run = s + 1;
      if ((s + 1) % check == 0 && !all_finite(wout, args.weight_elems)) {
        status = GEVO_STATUS_NONFINITE_WEIGHTS;
        break;
      }
    }
    final_w = wbuf[args.steps & 1];
    if (status == GEVO_STATUS_OK && !all_finite(final_w, args.weight_elems))
      status = GEVO_STATUS_NONFINITE_WEIGHTS;
    __syncthreads();
  }

  int64_t wrong = 0, total = 0;
  if (status == GEVO_STATUS_OK) {
    const gevo_instr* fw = stage(cache, args.instrs + P.fwd, P.fwd_n);
    const int B = args.batch, C = args.classes;
    for (int b = 0; b < args.score_nb; ++b) {
      if (threadIdx.x == 0) {
        S.base[GEVO_BUF_ARENA] = scratch;
        S.base[GEVO_BUF_CONST] = const_cast<double*>(consts);
        for (int i = 0; i < nw; ++i)
          S.base[GEVO_BUF_PARAM0 + i] = const_cast<double*>(final_w) + args.wofs[i];
        S.base[GEVO_BUF_PARAM0 + nw] = const_cast<double*>(args.score_x) + (int64_t)b * args.x_elems;
        S.base[GEVO_BUF_OUT0] = probs;
        S.wrong = 0;
      }
      __syncthreads();
      run_instrs(S, fw, P.fwd_n);
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
    gevo_result* R = args.results + P.result_slot;
    R->wrong = status == GEVO_STATUS_OK ? wrong : 0;
    R->total = status == GEVO_STATUS_OK ? total : 0;
    R->status = status;
    R->steps_run = steps_run;
  }
  if (args.final_weights != nullptr) {
    double* dst = args.final_weights + (int64_t)P.result_slot * args.weight_elems;
    for (int i = threadIdx.x; i < args.weight_elems; i += blockDim.x) dst[i] = final_w[i];
  }
}

// run one function once per prog with explicit params (tests, tools)
__global__ void __launch_bounds__(kThreads)
exec_once_kernel(OnceArgs args) {
  __shared__ Shared S;
  __shared__ gevo_instr cache[kInstrCache];
  const gevo_prog P = args.progs[blockIdx.x];
  if (threadIdx.x == 0) {
    S.base[GEVO_BUF_ARENA] = args.arena + P.arena_off;
    S.base[GEVO_BUF_CONST] = const_cast<double*>(args.consts) + P.const_off;
    for (int i = 0; i < GEVO_MAXP; ++i) {
      S.base[GEVO_BUF_PARAM0 + i] = const_cast<double*>(args.params) + P.param_off[i];
      S.base[GEVO_BUF_OUT0 + i] = args.outs + P.out_off[i];
    }
  }
  __syncthreads();
  const gevo_instr* ins = stage(cache, args.instrs + P.train0, P.train0_n);
  run_instrs(S, ins, P.train0_n);
}

void launch_eval(const EvalArgs& a, int n_prog, cudaStream_t st) {
  eval_kernel<<<n_prog, kThreads, 0, st>>>(a);
}

void launch_once(const OnceArgs& a, int n_prog, cudaStream_t st) {
  exec_once_kernel<<<n_prog, kThreads, 0, st>>>(a);
}

}  // namespace gevo
