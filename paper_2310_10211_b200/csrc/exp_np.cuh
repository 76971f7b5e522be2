// exp_np.cuh -- float64 exp used for the dialect's `exponential`.
// The reference evaluates np.exp (interpreter.py:106-108).  This is the
// placeholder: CUDA's correctly-rounded-in-most-cases exp.
#pragma once
namespace gevo {
__device__ __forceinline__ double exp_np(double x) { return exp(x); }
}  // namespace gevo
