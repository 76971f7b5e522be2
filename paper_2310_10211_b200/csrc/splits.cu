// splits.cu -- dataset bytes decoded into device splits.
//
// The reference reads pixels as uint8 and scales them on the host:
//   read_idx_images   datasets.py:33-45   u8.astype(float64) / 255.0
//   load_dataset      datasets.py:187-192 (synthetic digits, same scaling)
//   whole_batches     datasets.py:149-162 (one-hot y, labels; partial
//                                          trailing batch dropped)
// Here the raw bytes cross PCIe (1 B per pixel instead of 8) and the
// scaling, the one-hot rows and the label widening run on the device.
// x = __ddiv_rn(double(u8), 255.0) is the IEEE quotient numpy computes, so
// the decoded split is bit-identical to the reference's float64 array.
//
// CIFAR-10 binary records ([label u8][C planes of side*side u8], channel
// planes in R, G, B order) are decoded to the NHWC rows the CNN workload
// reads (cnn.py), label byte included.
//
// All kernels are HBM-bound streaming passes: grid = 4 x SMs CTAs of 256
// threads, grid-stride, each thread moving 4 pixels per iteration (one
// 32-bit load, two 16-byte stores) on the flat path.
#include <cuda_runtime.h>
#include <stdint.h>
#include "gevo_exec.cuh"

namespace gevo {

__global__ void __launch_bounds__(256) decode_u8_kernel(const uint8_t* __restrict__ px,
                                                        int64_t count, double* __restrict__ x) {
  const int64_t quads = count >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < quads; q += stride) {
    const uchar4 v = reinterpret_cast<const uchar4*>(px)[q];
    double2 a, b;
    a.x = __ddiv_rn((double)v.x, 255.0);
    a.y = __ddiv_rn((double)v.y, 255.0);
    b.x = __ddiv_rn((double)v.z, 255.0);
    b.y = __ddiv_rn((double)v.w, 255.0);
    reinterpret_cast<double2*>(x)[2 * q] = a;
    reinterpret_cast<double2*>(x)[2 * q + 1] = b;
  }
  // tail (count % 4) by the first threads
  const int64_t t = (quads << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < count && t >= (quads << 2)) x[t] = __ddiv_rn((double)px[t], 255.0);
}

// CIFAR records -> NHWC doubles; one thread per output pixel, consecutive
// threads write consecutive doubles and read from the C planes
__global__ void __launch_bounds__(256) decode_cifar_kernel(const uint8_t* __restrict__ rec,
                                                           int64_t rows, int C, int HW,
                                                           double* __restrict__ x,
                                                           int64_t* __restrict__ labels) {
  const int64_t rec_bytes = 1 + (int64_t)C * HW;
  const int64_t per_row = (int64_t)C * HW;
  const int64_t count = rows * per_row;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < count; o += stride) {
    const int64_t r = o / per_row;
    const int rem = (int)(o - r * per_row);
    const int p = rem / C, c = rem - p * C;          // NHWC: pixel p, channel c
    x[o] = __ddiv_rn((double)rec[r * rec_bytes + 1 + (int64_t)c * HW + p], 255.0);
  }
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += stride)
    labels[r] = rec[r * rec_bytes];
}

// one-hot rows (datasets.py:158-159) from device labels
__global__ void __launch_bounds__(256) one_hot_kernel(const int64_t* __restrict__ labels,
                                                      int64_t rows, int classes,
                                                      double* __restrict__ y) {
  const int64_t count = rows * classes;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    const int64_t r = i / classes;
    y[i] = labels[r] == (int64_t)(i - r * classes) ? 1.0 : 0.0;
  }
}

static int grid_for(int64_t work, int sms) {
  const int64_t want = (work + 255) / 256;
  const int64_t cap = (int64_t)sms * 4;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

// the tf32 mode's copy of a split's x (the operand TMA feeds to tcgen05):
// each value rounded to tf32 exactly as the CTA-staged operands are
// (cvt.rna of the fp32 value), stored as fp32 bits with the low 13 zero
__global__ void __launch_bounds__(256) to_f32_kernel(const double* __restrict__ x, int64_t n,
                                                     float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"((float)x[i]));
    y[i] = __uint_as_float(t);
  }
}

void launch_to_f32(const double* x, int64_t n, float* y, int sms, cudaStream_t st) {
  if (n <= 0) return;
  to_f32_kernel<<<grid_for(n, sms), 256, 0, st>>>(x, n, y);
}

void launch_decode_u8(const uint8_t* px, int64_t count, double* x, int sms, cudaStream_t st) {
  if (count <= 0) return;
  decode_u8_kernel<<<grid_for((count + 3) / 4, sms), 256, 0, st>>>(px, count, x);
}

void launch_decode_cifar(const uint8_t* rec, int64_t rows, int C, int HW, double* x,
                         int64_t* labels, int sms, cudaStream_t st) {
  if (rows <= 0) return;
  decode_cifar_kernel<<<grid_for(rows * C * HW, sms), 256, 0, st>>>(rec, rows, C, HW, x, labels);
}

void launch_one_hot(const int64_t* labels, int64_t rows, int classes, double* y, int sms,
                    cudaStream_t st) {
  if (rows <= 0) return;
  one_hot_kernel<<<grid_for(rows * classes, sms), 256, 0, st>>>(labels, rows, classes, y);
}

}  // namespace gevo
