// tc_probe.cu -- hardware probe (tool) for the tcgen05 tf32 path: one CTA
// computes C[128 x N] = A[128 x K] . B[K x N] with tcgen05.mma kind::tf32,
// operands staged by the threads into the K-major no-swizzle canonical
// layout, accumulator in TMEM read back with tcgen05.ld.32x32b; checked
// against a host fp64 product of the tf32-rounded operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tests/tools/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                  // version (sm_100)
  return d;                                // base offset 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)                         // D f32
       | (2u << 7) | (2u << 10)            // A, B tf32
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

template <int N, int K>
__global__ void probe(const float* A, const float* B, float* C, int reps, long long* cyc) {
  extern __shared__ __align__(128) uint8_t sm[];
  float* As = reinterpret_cast<float*>(sm);                 // 128 x K
  float* Bs = As + 128 * K;                                  // N x K
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t SBO = (K / 4) * 128, LBO = 128;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const uint32_t off = (m / 8) * SBO + (k / 4) * LBO + (m % 8) * 16 + (k % 4) * 4;
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(A[i]));
    *reinterpret_cast<uint32_t*>(sm + off) = t;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int k = i / N, n = i % N;                         // B row-major [K][N]
    const uint32_t off = (n / 8) * SBO + (k / 4) * LBO + (n % 8) * 16 + (k % 4) * 4;
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(B[i]));
    *reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(Bs) + off) = t;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_addr(&tmem_base)), "n"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t a0 = smem_addr(As), b0 = smem_addr(Bs);
  constexpr uint32_t idesc = idesc_tf32(128, N);
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int r = 0; r < reps; ++r) {
    if (tid == 0) {
#pragma unroll
      for (int kk = 0; kk < K / 8; ++kk) {
        const uint64_t da = smem_desc(a0 + kk * 256, LBO, SBO);
        const uint64_t db = smem_desc(b0 + kk * 256, LBO, SBO);
        const uint32_t acc = kk > 0 ? 1u : 0u;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   :: "r"(smem_addr(&mbar)) : "memory");
    }
    // all threads wait for the MMAs
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
                 :: "r"(smem_addr(&mbar)), "r"(phase) : "memory");
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  long long t1 = clock64();
  if (warp < 4) {
    uint32_t v[N];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
    for (int c = 0; c < N; c += 8) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[c]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]), "=r"(v[c + 4]),
                     "=r"(v[c + 5]), "=r"(v[c + 6]), "=r"(v[c + 7])
                   : "r"(taddr + c));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = warp * 32 + lane;
#pragma unroll
    for (int c = 0; c < N; ++c) C[m * N + c] = __uint_as_float(v[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(N < 32 ? 32 : N));
  if (tid == 0) *cyc = t1 - t0;
}

static float tf32r(float x) {   // round to nearest, ties away (cvt.rna.tf32)
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

template <int N, int K>
int run(int reps) {
  std::vector<float> A(128 * K), B(K * N), C(128 * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX) * 2 - 1;
  for (auto& x : B) x = (rand() / (float)RAND_MAX) * 2 - 1;
  float *dA, *dB, *dC;
  long long* dcyc;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dC, C.size() * 4));
  CK(cudaMalloc(&dcyc, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  const int smem = (128 + N) * K * 4;
  CK(cudaFuncSetAttribute(probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<N, K><<<1, 128, smem>>>(dA, dB, dC, reps, dcyc);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  long long cyc;
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)tf32r(A[m * K + k]) * (double)tf32r(B[k * N + n]);
      maxerr = fmax(maxerr, fabs(s - C[m * N + n]));
    }
  printf("N=%d K=%d max|err| %.3e  (C[0]=%f)  %lld cycles for %d reps (%.1f cyc/MMA-set)\n", N, K, maxerr,
         C[0], cyc, reps, (double)cyc / reps);
  return maxerr < 1e-3 ? 0 : 1;
}

int main() {
  int bad = 0;
  bad |= run<32, 32>(1);
  bad |= run<32, 64>(1);
  bad |= run<64, 32>(1);
  bad |= run<32, 32>(100);
  printf(bad ? "FAIL\n" : "OK\n");
  return bad;
}
