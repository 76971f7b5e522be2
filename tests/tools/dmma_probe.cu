// Probe (tool): does mma.sync.m8n8k4.f64 round like 4 chained fma()s in k
// order?  And DFMA vs DMMA throughput on one SM.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// C[8x8] = A[8xK] B[Kx8], one warp; A row-major, B row-major (K x 8)
__global__ void gemm_dmma(const double* A, const double* B, double* C, int K) {
  int lane = threadIdx.x;
  int g = lane >> 2, t = lane & 3;          // groupID, threadID_in_group
  double c0 = 0.0, c1 = 0.0;
  for (int k0 = 0; k0 < K; k0 += 4) {
    double a = A[g * K + k0 + t];           // A frag: row g, col t
    double b = B[(k0 + t) * 8 + g];         // B frag (col-major 4x8): row t, col g
    dmma(c0, c1, a, b, c0, c1);
  }
  C[g * 8 + 2 * t] = c0;                    // D frag: row g, cols 2t, 2t+1
  C[g * 8 + 2 * t + 1] = c1;
}

__global__ void gemm_fma(const double* A, const double* B, double* C, int K) {
  int i = threadIdx.x >> 3, j = threadIdx.x & 7;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) acc = fma(A[i * K + k], B[k * 8 + j], acc);
  C[i * 8 + j] = acc;
}

__global__ void tput_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma(c[u][0], c[u][1], a, b, c[u][0], c[u][1]);
  double s = 0;
  for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void tput_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[8] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) c[u] = fma(a, b, c[u]);
  double s = 0;
  for (int u = 0; u < 8; ++u) s += c[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int K = 784;
  double *A, *B, *C1, *C2, *o;
  cudaMallocManaged(&A, 8 * K * 8); cudaMallocManaged(&B, K * 8 * 8);
  cudaMallocManaged(&C1, 64 * 8); cudaMallocManaged(&C2, 64 * 8);
  cudaMallocManaged(&o, 148 * 1024 * 8);
  long bad = 0, tot = 0;
  srand(1);
  for (int trial = 0; trial < 200; ++trial) {
    for (int i = 0; i < 8 * K; ++i) A[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 12 - 6);
    for (int i = 0; i < 8 * K; ++i) B[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 12 - 6);
    gemm_dmma<<<1, 32>>>(A, B, C1, K);
    gemm_fma<<<1, 64>>>(A, B, C2, K);
    cudaDeviceSynchronize();
    for (int i = 0; i < 64; ++i) { bad += (C1[i] != C2[i]); ++tot; }
  }
  printf("dmma vs fma-chain mismatches: %ld / %ld\n", bad, tot);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); tput_dmma<<<148, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * 8 * iters * (148 * 256 / 32);
    printf("DMMA: %.2f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0); tput_dfma<<<148, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * iters * 148.0 * 256;
    printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  return 0;
}
