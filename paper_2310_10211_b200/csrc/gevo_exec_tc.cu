// gevo_exec_tc.cu -- the executor's reduced-precision build: gevo_exec.cu
// with every f64 DOT on the tcgen05 tensor cores (dot_tc.cuh), compiled as
// its own module in namespace gevo_tc (kernels eval_kernel_tc /
// exec_once_kernel_tc) and reached from gevo_abi.cu through the two C
// launchers below when GEVO_B200_DTYPE=tf32.  EvalArgs / OnceArgs have the
// same layout in both namespaces (one header, gevo_exec.cuh).
#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
#define gevo gevo_tc
#define GEVO_TC_MODE 1
#include "gevo_exec.cu"
#undef gevo

extern "C" void gevo_internal_launch_eval_tc(const void* a, int n_prog, cudaStream_t st) {
  gevo_tc::launch_eval_tc(*static_cast<const gevo_tc::EvalArgs*>(a), n_prog, st);
}
extern "C" void gevo_internal_launch_once_tc(const void* a, int n_prog, cudaStream_t st) {
  gevo_tc::launch_once_tc(*static_cast<const gevo_tc::OnceArgs*>(a), n_prog, st);
}
