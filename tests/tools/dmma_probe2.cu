// Probe (tool): FP64 tensor-core shapes on sm_100a.
//  (1) layout check with exact small-integer data, (2) rounding order: is
//  each shape bit-identical to a single fma chain in ascending k?  (3)
//  dependent-chain latency and per-SM throughput of each shape, and DFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/p tests/tools/dmma_probe2.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#define MMA884(d0, d1, a, b)                                                             \
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" \
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b))
#define MMA1684(c, a0, a1, b0)                                                            \
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b0))
#define MMA1688(c, a, b)                                                                  \
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])                         \
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]))
#define MMA16816(c, a, b)                                                                 \
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])                         \
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), \
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]))

// C[16x8] = A[16xK] B[Kx8]; A row-major (lda K), B row-major (ldb 8); one warp
template <int SHAPE>
__global__ void gemm_mma(const double* A, const double* B, double* C, int K) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double c[4] = {0, 0, 0, 0};
  if (SHAPE == 4) {
    for (int k0 = 0; k0 < K; k0 += 4) {
      double a0 = A[g * K + k0 + t], a1 = A[(g + 8) * K + k0 + t], b0 = B[(k0 + t) * 8 + g];
      MMA1684(c, a0, a1, b0);
    }
  } else if (SHAPE == 8) {
    for (int k0 = 0; k0 < K; k0 += 8) {
      double a[4] = {A[g * K + k0 + t], A[(g + 8) * K + k0 + t], A[g * K + k0 + t + 4], A[(g + 8) * K + k0 + t + 4]};
      double b[2] = {B[(k0 + t) * 8 + g], B[(k0 + t + 4) * 8 + g]};
      MMA1688(c, a, b);
    }
  } else if (SHAPE == 16) {
    for (int k0 = 0; k0 < K; k0 += 16) {
      double a[8], b[4];
      for (int i = 0; i < 4; ++i) {
        a[2 * i] = A[g * K + k0 + t + 4 * i];
        a[2 * i + 1] = A[(g + 8) * K + k0 + t + 4 * i];
        b[i] = B[(k0 + t + 4 * i) * 8 + g];
      }
      MMA16816(c, a, b);
    }
  } else {   // m8n8k4 twice (rows 0-7, 8-15)
    for (int k0 = 0; k0 < K; k0 += 4) {
      double a0 = A[g * K + k0 + t], a1 = A[(g + 8) * K + k0 + t], b0 = B[(k0 + t) * 8 + g];
      MMA884(c[0], c[1], a0, b0);
      MMA884(c[2], c[3], a1, b0);
    }
  }
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

__global__ void gemm_fma(const double* A, const double* B, double* C, int K) {
  int i = threadIdx.x >> 3, j = threadIdx.x & 7;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) acc = fma(A[i * K + k], B[k * 8 + j], acc);
  C[i * 8 + j] = acc;
}

template <int SHAPE, int CHAINS>
__global__ void timing(double* out, int iters, long long* cyc) {
  const int lane = threadIdx.x & 31;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = (lane + i) * 1e-3;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
  double c[CHAINS][4] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < CHAINS; ++u) {
      if (SHAPE == 0) MMA884(c[u][0], c[u][1], a[0], b[0]);
      if (SHAPE == 4) MMA1684(c[u], a[0], a[1], b[0]);
      if (SHAPE == 8) MMA1688(c[u], a, b);
      if (SHAPE == 16) MMA16816(c[u], a, b);
      if (SHAPE == 1) c[u][0] = fma(a[0], b[0], c[u][0]);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < CHAINS; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

static double rnd() { return (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 12 - 6); }

template <int SHAPE, int CHAINS>
void time_one(const char* name, double* o, long long* cyc, double fl_per_mma) {
  const int iters = 4000;
  // latency: one warp, CHAINS chains
  timing<SHAPE, CHAINS><<<1, 32>>>(o, iters, cyc);
  cudaDeviceSynchronize();
  double lat = (double)*cyc / iters;   // cycles per iteration of CHAINS independent ops
  // throughput: 148 SMs x 16 warps
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  timing<SHAPE, CHAINS><<<148 * 2, 256>>>(o, iters, cyc);
  cudaEventRecord(e0);
  timing<SHAPE, CHAINS><<<148 * 2, 256>>>(o, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)iters * CHAINS * (148 * 2 * 8);  // warp-level ops
  if (SHAPE == 1) ops *= 32;
  printf("%-10s chains=%d: %.1f cycles/iter (1 warp)  -> throughput %.2f TFLOP/s over 148 SMs\n",
         name, CHAINS, lat, ops * fl_per_mma / ms / 1e9);
}

int main() {
  const int K = 784;
  double *A, *B, *C1, *C2, *o;
  long long* cyc;
  cudaMallocManaged(&A, 16 * K * 8); cudaMallocManaged(&B, K * 8 * 8);
  cudaMallocManaged(&C1, 128 * 8); cudaMallocManaged(&C2, 128 * 8);
  cudaMallocManaged(&o, 148 * 2 * 256 * 8); cudaMallocManaged(&cyc, 8);
  const char* names[4] = {"m8n8k4x2", "m16n8k4", "m16n8k8", "m16n8k16"};
  for (int s = 0; s < 4; ++s) {
    long bad_exact = 0, bad = 0, tot = 0;
    srand(1);
    for (int trial = 0; trial < 100; ++trial) {
      bool exact = trial < 10;   // small integers: layout check, any order exact
      for (int i = 0; i < 16 * K; ++i) A[i] = exact ? (rand() % 7 - 3) : rnd();
      for (int i = 0; i < 8 * K; ++i) B[i] = exact ? (rand() % 7 - 3) : rnd();
      if (s == 0) gemm_mma<0><<<1, 32>>>(A, B, C1, K);
      if (s == 1) gemm_mma<4><<<1, 32>>>(A, B, C1, K);
      if (s == 2) gemm_mma<8><<<1, 32>>>(A, B, C1, K);
      if (s == 3) gemm_mma<16><<<1, 32>>>(A, B, C1, K);
      gemm_fma<<<1, 128>>>(A, B, C2, K);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", names[s], cudaGetErrorString(e)); return 1; }
      for (int i = 0; i < 128; ++i) {
        if (exact) bad_exact += (C1[i] != C2[i]);
        else { bad += (C1[i] != C2[i]); ++tot; }
      }
    }
    printf("%-10s layout mismatches (exact data) %ld; vs ascending fma chain: %ld / %ld differ\n",
           names[s], bad_exact, bad, tot);
  }
  time_one<0, 1>("m8n8k4", o, cyc, 512);
  time_one<0, 4>("m8n8k4", o, cyc, 512);
  time_one<0, 8>("m8n8k4", o, cyc, 512);
  time_one<4, 1>("m16n8k4", o, cyc, 1024);
  time_one<4, 4>("m16n8k4", o, cyc, 1024);
  time_one<8, 1>("m16n8k8", o, cyc, 2048);
  time_one<8, 4>("m16n8k8", o, cyc, 2048);
  time_one<16, 1>("m16n8k16", o, cyc, 4096);
  time_one<16, 4>("m16n8k16", o, cyc, 4096);
  time_one<1, 1>("dfma", o, cyc, 2);
  time_one<1, 8>("dfma", o, cyc, 2);
  return 0;
}
