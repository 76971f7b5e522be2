// dot_tc.cuh -- the DOT on the 5th-generation tensor cores (tcgen05, kind::tf32):
// the executor's reduced-precision mode (GEVO_B200_DTYPE=tf32).
//
// The parity mode (default) computes every dot in float64 in the reference's
// own summation order on DMMA (dot_staged.cuh): tcgen05 has no f64 kind.  In
// tf32 mode a DOT's operands are rounded to tf32 (cvt.rna), multiplied on
// tcgen05.mma with fp32 accumulation in tensor memory, and the result is
// widened back to float64 for the fused epilogue and every other op, which
// stay float64.  Fitness then differs from the reference's by the tf32
// product error; bench.py reports the exact-match rate and the tolerance.
//
// Per 128 x 64 output tile (64 fp32 columns of TMEM, allocated once per
// CTA): K is walked in 32-wide chunks through two shared-memory stages.  When
// A is a 32-row batch of the training split's x -- the operand every
// individual shares -- its chunks come by TMA from one fp32 mirror of the
// split (a tensor map per launch, gevo_abi.cu); the CTA's threads stage the
// rest.  The
// CTA's threads stage a chunk -- A rows and B columns, f64 -> tf32 -- in the
// K-major no-swizzle canonical layout (8-row x 16-byte core matrices: LBO =
// 128 B between the two core matrices of one MMA's K = 8, SBO = 1 KB between
// 8-row groups); one elected thread issues the chunk's four MMAs and commits
// them to the stage's mbarrier, which the threads wait on before refilling
// that stage (so staging chunk c+1 overlaps the MMAs of chunk c).  Rows of
// the A tile past M are never staged: the MMA reads whatever lies there and
// writes those products to TMEM lanes that are never read.  The epilogue
// warps read their rows with tcgen05.ld.32x32b (warp w: lanes 32(w%4)..,
// column half w/4), apply the fused micro-ops in float64 and store.
#pragma once
#include <stdint.h>

namespace gevo {

constexpr int kTcCols = 64;           // TMEM columns per CTA (fp32 accumulator): N per tile
constexpr int kTcKC = 32;             // K per staged chunk
constexpr uint32_t kTcSBO = (kTcKC / 4) * 128;   // bytes between 8-row groups (tf32)
constexpr uint32_t kTcLBO = 128;                 // bytes between K core matrices
constexpr uint32_t kTcTileA = 16 * kTcSBO;       // a 128-row A tile (16 KB; bf16 uses half)
constexpr uint32_t kTcTileB = (kTcCols / 8) * kTcSBO;   // a 64-column B tile (8 KB)

// per element type: bytes per element, elements per 16-byte core-matrix row,
// SBO (bytes between 8-row groups of a KC-wide chunk), K of one MMA
template <bool BF> struct TcFmt {
  static constexpr int ES = BF ? 2 : 4;
  static constexpr int EPC = 16 / ES;
  static constexpr uint32_t SBO = (kTcKC / EPC) * 128;
  static constexpr int MMA_K = BF ? 16 : 8;
};

__device__ __forceinline__ uint64_t tc_desc(uint32_t addr, uint32_t sbo = kTcSBO) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((kTcLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100); SWIZZLE_NONE
  return d;
}

// D f32; A, B tf32 (format 2, kind::tf32) or bf16 (format 1, kind::f16); K-major
__device__ __forceinline__ uint32_t tc_idesc(int M, int N, bool bf = false) {
  const uint32_t f = bf ? 1u : 2u;
  return (1u << 4) | (f << 7) | (f << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t bf16_bits(double x) {
  unsigned short h;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"((float)x));
  return h;
}

__device__ __forceinline__ uint32_t tf32_bits(double x) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"((float)x));
  return t;
}

__device__ __forceinline__ void tc_wait(uint32_t mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(mbar), "r"(phase) : "memory");
}

// CTA-wide setup / teardown (TcState, gevo_exec.cu): tc_setup at kernel
// start, tc_teardown at the end
__device__ __forceinline__ void tc_setup(TcState& T) {
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&T.mbar[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&T.tbar[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    T.ph = 0;
    T.pending = 0;
    T.tph = 0;
    if (T.tmap) asm volatile("prefetch.tensormap [%0];" ::"l"(T.tmap) : "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&T.tmem)), "n"(kTcCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_teardown(TcState& T) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(T.tmem), "n"(kTcCols));
}

// all threads: wait for the commit on stage b if one is pending
__device__ __forceinline__ void tc_drain(TcState& T, int b, uint32_t& ph, uint32_t& pending) {
  if ((pending >> b) & 1) {
    tc_wait(smem_u32(&T.mbar[b]), (ph >> b) & 1);
    ph ^= 1u << b;
    pending &= ~(1u << b);
  }
}

// TMA (cp.async.bulk.tensor) of one 8-row x 4-column fp32 box of the
// mirrored x -- exactly one core matrix of the canonical layout -- into smem
// `dst`, completing on mbarrier `bar`
__device__ __forceinline__ void tma_box(uint32_t dst, const void* map, int col, int row, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(col), "r"(row), "r"(bar) : "memory");
}

// columns [col0, col1) of the DOT, every row, on tcgen05 (tf32 operands, fp32
// accumulation); the epilogue (if any) is applied in float64.
// profile mode: thread 0 adds phase cycles to slots 240.. (op class 7 of
// tests/tools/op_profile.py): 0 wait for a stage, 1 stage + fence + barrier,
// 2 MMA issue + commit, 3 wait for the accumulator, 4 TMEM read + epilogue
__device__ __forceinline__ void tc_tick(unsigned long long* prof, int ph, long long& t) {
  if (prof && threadIdx.x == 0) {
    const long long n = clock64();
    atomicAdd(prof + 2 * (240 + ph), (unsigned long long)(n - t));
    atomicAdd(prof + 2 * (240 + ph) + 1, 1ULL);
    t = n;
  }
}

template <bool BF>
__device__ __noinline__ void dot_tc(TcState& T, const DotArgs& dref, int col0, int col1, const EpiDev* epi,
                                    double* stage_buf, unsigned long long* prof) {
  using F = TcFmt<BF>;
  const DotArgs d = dref;            // registers, not the caller's stack frame
  long long tt = clock64();
  const int M = d.M, K = d.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // TMA destinations need 128-byte alignment: round the staging base up
  // (48 KB of the 63 KB buffer are used, so the slack fits)
  uint8_t* sm = reinterpret_cast<uint8_t*>(stage_buf);
  sm += (128u - (smem_u32(sm) & 127u)) & 127u;
  // stage b: B tile at b * kTcTileB, A tile at 2 * kTcTileB + b * kTcTileA
  // (48 KB of the 63 KB staging buffer; an A tile's unstaged row groups are
  // read by the MMA and land in TMEM lanes nobody reads)
  const uint32_t sbase = smem_u32(sm);
  uint32_t ph = T.ph, pending = T.pending;
  const int nch = (K + kTcKC - 1) / kTcKC;
  for (int m0 = 0; m0 < M; m0 += 128) {
    const int mt = min(128, M - m0);
    for (int n0 = col0; n0 < col1; n0 += kTcCols) {
      const int nt = min(kTcCols, col1 - n0);
      const int ntp = (nt + 15) & ~15;
      const uint32_t idesc = tc_idesc(128, ntp, BF);
      // staging slots: A 16 per thread of the 128 x 32 chunk, B 8 of the
      // 64 x 32 chunk, consecutive threads along each operand's unit-stride
      // axis; each batch of 8 slots has all its loads in flight before any
      // is converted and stored (no registers held across chunks: the
      // function runs under the kernel's 128-register cap)
      const bool a_kfast = d.sak == 1 || d.sam != 1;
      const bool b_nfast = d.sbn == 1 || d.sbk != 1;
      const int am0 = a_kfast ? (tid >> 5) : (tid & 127), ak0 = a_kfast ? (tid & 31) : (tid >> 7);
      const int amd = a_kfast ? 8 : 0, akd = a_kfast ? 0 : 2;
      const int bn0 = b_nfast ? (tid & 63) : (tid >> 5), bk0 = b_nfast ? (tid >> 6) : (tid & 31);
      const int bnd = b_nfast ? 0 : 8, bkd = b_nfast ? 4 : 0;
      const double* pa = d.A + (int64_t)(m0 + am0) * d.sam + (int64_t)ak0 * d.sak;
      const double* pb = d.B + (int64_t)bk0 * d.sbk + (int64_t)(n0 + bn0) * d.sbn;
      const int64_t sa_u = (int64_t)amd * d.sam + (int64_t)akd * d.sak;
      const int64_t sb_u = (int64_t)bkd * d.sbk + (int64_t)bnd * d.sbn;
      // A from the shared batch x: TMA boxes of its fp32 mirror, one per
      // core matrix (8 rows x 4 columns), issued by one thread per chunk
      int trow0 = -1;
      if (!BF && T.tmap && mt == 32 && d.sak == 1 && d.sam == T.tcols && d.A >= T.tx64) {
        const int64_t off = (d.A + (int64_t)m0 * d.sam) - T.tx64;
        if (off < T.trows * (int64_t)T.tcols && off % T.tcols == 0 && (off / T.tcols) % 8 == 0 &&
            off / T.tcols + 32 <= T.trows)
          trow0 = (int)(off / T.tcols);
      }
      const bool tma_a = trow0 >= 0;
      const int na = tma_a ? 0 : (a_kfast ? max(0, min(16, (mt - am0 + 7) / 8)) : 16);   // A slots, rows < mt
      for (int c = 0; c < nch; ++c) {
        const int b = c & 1, k0 = c * kTcKC;
        tc_drain(T, b, ph, pending);       // the MMAs that read stage b are done
        tc_tick(prof, 0, tt);
        if (tma_a && tid == 0) {
          const uint32_t bar = smem_u32(&T.tbar[b]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(32 * kTcKC * 4)
                       : "memory");
          const uint32_t a0 = sbase + 2 * kTcTileB + b * kTcTileA;
#pragma unroll
          for (int rg = 0; rg < 4; ++rg)
#pragma unroll
            for (int cg = 0; cg < kTcKC / 4; ++cg)
              tma_box(a0 + rg * kTcSBO + cg * kTcLBO, T.tmap, k0 + cg * 4, trow0 + rg * 8, bar);
        }
        uint8_t* As = sm + 2 * kTcTileB + b * kTcTileA;
        uint8_t* Bs = sm + b * kTcTileB;
        const double* pac = pa + (int64_t)k0 * d.sak;
        const double* pbc = pb + (int64_t)k0 * d.sbk;
        for (int u0 = 0; u0 < 24; u0 += 8) {
          if (u0 < 16 && u0 >= na) continue;
          double v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int u = u0 + j;
            v[j] = 0.0;
            if (u < 16) {
              const int m = am0 + u * amd, k = k0 + ak0 + u * akd;
              if (m < mt && k < K) v[j] = pac[u * sa_u];
            } else {
              const int n = bn0 + (u - 16) * bnd, k = k0 + bk0 + (u - 16) * bkd;
              if (n < nt && k < K) v[j] = pbc[(u - 16) * sb_u];
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int u = u0 + j;
            if (u < 16) {
              const int m = am0 + u * amd, k = ak0 + u * akd;
              if (m < mt) {
                const uint32_t o = (m >> 3) * F::SBO + (k / F::EPC) * kTcLBO + (m & 7) * 16 + (k % F::EPC) * F::ES;
                if (BF) *reinterpret_cast<unsigned short*>(As + o) = (unsigned short)bf16_bits(v[j]);
                else *reinterpret_cast<uint32_t*>(As + o) = tf32_bits(v[j]);
              }
            } else {
              const int n = bn0 + (u - 16) * bnd, k = bk0 + (u - 16) * bkd;
              if (n < ntp) {
                const uint32_t o = (n >> 3) * F::SBO + (k / F::EPC) * kTcLBO + (n & 7) * 16 + (k % F::EPC) * F::ES;
                if (BF) *reinterpret_cast<unsigned short*>(Bs + o) = (unsigned short)bf16_bits(v[j]);
                else *reinterpret_cast<uint32_t*>(Bs + o) = tf32_bits(v[j]);
              }
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        tc_tick(prof, 1, tt);
        if (tid == 0) {
          if (tma_a) {                     // the chunk's A boxes have landed
            tc_wait(smem_u32(&T.tbar[b]), (T.tph >> b) & 1);
            T.tph ^= 1u << b;
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = sbase + 2 * kTcTileB + b * kTcTileA, b0 = sbase + b * kTcTileB;
#pragma unroll
          for (int kk = 0; kk < kTcKC / F::MMA_K; ++kk) {
            const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
            const uint64_t da = tc_desc(a0 + kk * 2 * kTcLBO, F::SBO), db = tc_desc(b0 + kk * 2 * kTcLBO, F::SBO);
            if (BF)
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(T.tmem),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc));
            else
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(T.tmem),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(smem_u32(&T.mbar[b])) : "memory");
        }
        pending |= 1u << b;
        tc_tick(prof, 2, tt);
      }
      // the accumulator is complete once every commit has arrived
      tc_drain(T, 0, ph, pending);
      tc_drain(T, 1, ph, pending);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      tc_tick(prof, 3, tt);
      // epilogue: the accumulator goes TMEM -> registers -> a float tile in
      // the (now idle) staging buffer, so the float64 epilogue and the stores
      // walk the output row-major, coalesced.  Warp w reads lanes
      // 32(w%4)+lane (its rows), the column half w/4.
      float* Cs = reinterpret_cast<float*>(stage_buf);
      constexpr int kCS = kTcCols + 1;
      {
        const int row = (warp & 3) * 32 + lane;
        const int half = ntp / 2, cbeg = (warp >> 2) * half;
        const uint32_t taddr = T.tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)cbeg;
        for (int j0 = 0; j0 < half; j0 += 8) {
          uint32_t v[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                         "=r"(v[7])
                       : "r"(taddr + j0));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 8; ++u) Cs[row * kCS + cbeg + j0 + u] = __uint_as_float(v[u]);
        }
      }
      __syncthreads();
      // thread t: column t % 64, rows t / 64 + 4 r; four rows in flight
      {
        const int c = tid & 63, r0 = tid >> 6;
        const int n = n0 + c;
        if (c < nt) {
          for (int rb = r0; rb < mt; rb += 16) {
            double ev[4][kEpiPre], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int r = rb + 4 * u;
              if (r < mt) {
                x[u] = (double)Cs[r * kCS + c];
                if (epi) epi_fetch(*epi, m0 + r, n, ev[u]);
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int r = rb + 4 * u;
              if (r < mt) {
                double y = x[u];
                if (epi) y = epilogue(*epi, ev[u], y, m0 + r, n);
                d.out[(int64_t)(m0 + r) * d.som + (int64_t)n * d.son] = y;
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();                    // TMEM free for the next tile's MMAs
      tc_tick(prof, 4, tt);
    }
  }
  if (tid == 0) {
    T.ph = ph;
    T.pending = pending;
  }
  __syncthreads();
}

}  // namespace gevo
