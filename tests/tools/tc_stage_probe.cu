// tc_stage_probe.cu -- hardware probe (tool): the staging pattern of dot_tc
// in isolation.  NB CTAs (2 per SM) each stream a 32 x 784 A (shared) and
// their own 784 x 32 B (f64, global) through 32-wide k chunks: loads ->
// tf32 -> canonical smem tiles -> (optionally) 4 tcgen05 MMAs per chunk.
// Prints cycles per chunk of each phase, to separate memory latency from the
// interpreter's surroundings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_stage_probe tests/tools/tc_stage_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t tf32_bits(double x) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"((float)x));
  return t;
}
__device__ __forceinline__ uint64_t tc_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <bool MMA>
__global__ void __launch_bounds__(256, 2) probe(const double* A, const double* B, int K, unsigned long long* cyc,
                                                 float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint32_t tmem;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x;
  const double* Bi = B + (size_t)blockIdx.x * K * 32;
  if (MMA) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  long long t_ld = 0, t_st = 0, t_sync = 0, t_mma = 0;
  uint32_t phase = 0;
  const int ak = tid & 31, am = tid >> 5;          // A: 4 slots (rows am + 8u, u < 4)
  const int bn = tid & 31, bk = tid >> 5;          // B: 4 slots (k = bk + 8u)
  float acc = 0.f;
  for (int k0 = 0; k0 < K; k0 += 32) {
    long long t0 = clock64();
    double va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      va[u] = A[(am + 8 * u) * K + k0 + ak];
      vb[u] = Bi[(k0 + bk + 8 * u) * 32 + bn];
    }
    // force arrival before timing the stores
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += (float)va[u] + (float)vb[u];
    long long t1 = clock64();
    const int b = (k0 / 32) & 1;
    uint8_t* As = sm + 16384 + b * 16384;
    uint8_t* Bs = sm + b * 8192;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int m = am + 8 * u, k = ak;
      *reinterpret_cast<uint32_t*>(As + (m >> 3) * 1024 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4) = tf32_bits(va[u]);
      const int n = bn, kk = bk + 8 * u;
      *reinterpret_cast<uint32_t*>(Bs + (n >> 3) * 1024 + (kk >> 2) * 128 + (n & 7) * 16 + (kk & 3) * 4) = tf32_bits(vb[u]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    long long t2 = clock64();
    __syncthreads();
    long long t3 = clock64();
    if (MMA) {
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (4u << 17) | (8u << 24);
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t accf = (k0 > 0 || kk > 0) ? 1u : 0u;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                       "l"(tc_desc(a0 + kk * 256)), "l"(tc_desc(b0 + kk * 256)), "r"(idesc), "r"(accf));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(smem_u32(&mbar)) : "memory");
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase) : "memory");
      phase ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    long long t4 = clock64();
    t_ld += t1 - t0;
    t_st += t2 - t1;
    t_sync += t3 - t2;
    t_mma += t4 - t3;
  }
  if (tid == 0) {
    atomicAdd(cyc + 0, (unsigned long long)t_ld);
    atomicAdd(cyc + 1, (unsigned long long)t_st);
    atomicAdd(cyc + 2, (unsigned long long)t_sync);
    atomicAdd(cyc + 3, (unsigned long long)t_mma);
  }
  out[blockIdx.x * 256 + tid] = acc;
  if (MMA) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
  }
}

int main() {
  const int K = 784, NB = 296;
  double *A, *B;
  float* out;
  unsigned long long* cyc;
  CK(cudaMalloc(&A, 32 * K * 8));
  CK(cudaMalloc(&B, (size_t)NB * K * 32 * 8));
  CK(cudaMalloc(&out, NB * 256 * 4));
  CK(cudaMalloc(&cyc, 64));
  CK(cudaMemset(A, 0, 32 * K * 8));
  CK(cudaMemset(B, 0, (size_t)NB * K * 32 * 8));
  const int smem = 48 * 1024;
  CK(cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int mma = 0; mma < 2; ++mma)
    for (int nb : {2, NB}) {
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaMemset(cyc, 0, 64));
        if (mma) probe<true><<<nb, 256, smem>>>(A, B, K, cyc, out);
        else probe<false><<<nb, 256, smem>>>(A, B, K, cyc, out);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
      }
      unsigned long long h[4];
      CK(cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost));
      const double ch = (double)nb * ((K + 31) / 32);
      printf("mma=%d CTAs=%3d  per chunk: loads %.0f  stores+fence %.0f  barrier %.0f  mma+wait %.0f cycles\n", mma, nb,
             h[0] / ch, h[1] / ch, h[2] / ch, h[3] / ch);
    }
  return 0;
}
