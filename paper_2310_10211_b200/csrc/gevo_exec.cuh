// gevo_exec.cuh -- internal launch interfaces of the executor.
#pragma once
#include <cuda_runtime.h>
#include "gevo.h"

namespace gevo {

struct EvalArgs {
  const gevo_instr* instrs;
  const gevo_prog* progs;
  const double* consts;
  double* arena;
  int32_t wofs[GEVO_MAXP];
  int n_weights, weight_elems, probs_elems;
  int mode, steps, check_every;
  const double* init_weights;
  const double* train_x;
  const double* train_y;
  int train_nb;
  const double* score_x;
  const int64_t* score_labels;
  int score_nb;
  int batch, classes;
  int64_t x_elems, y_elems;   // per batch
  gevo_result* results;
  double* final_weights;      // nullable
  int smem_elems;             // shared-memory scratch tier per CTA
  unsigned long long* prof;   // nullable: per-instruction-class cycles
  int tc;                     // 1: DOTs on tcgen05 in tf32 (GEVO_B200_DTYPE=tf32)
  double* wreg;               // nullable: weight blocks of all programs, block 0 of
                              // program i at wreg + i*wsz, block 1 at wreg + (n + i)*wsz
  int n_prog;                 // programs of the launch (wreg's block-1 offset)
  // tf32 mode: the training split's x as fp32 under a TMA tensor map; a dot
  // whose A operand is a batch of that x (row-major, 32 rows) has its A
  // chunks loaded by cp.async.bulk.tensor instead of the CTA's threads
  const double* tma_x64;      // nullable: the f64 x the map mirrors
  int64_t tma_rows;
  int tma_cols;
  alignas(64) unsigned char tma_map[128];   // CUtensorMap (opaque)
};

struct OnceArgs {
  const gevo_instr* instrs;
  const gevo_prog* progs;
  const double* consts;
  double* arena;
  const double* params;
  double* outs;
  int smem_elems;
  int tc;                     // as EvalArgs::tc
};

void launch_eval(const EvalArgs& a, int n_prog, cudaStream_t st);
void launch_once(const OnceArgs& a, int n_prog, cudaStream_t st);
// (namespace gevo_tc, the tf32 build: gevo_exec_tc.cu wraps these two)
void launch_eval_tc(const EvalArgs& a, int n_prog, cudaStream_t st);
void launch_once_tc(const OnceArgs& a, int n_prog, cudaStream_t st);

// NSGA-II (nsga2.cu)
struct NsArgs {
  int n, keep;
  int one_front;      // all points form a single front (crowding only)
  const double* c;
  const double* e;
  int32_t* rank;      // [n]
  double* crowd;      // [n]
  int32_t* order;     // [n] points grouped by front
  int32_t* fstart;    // [n+1]
  int32_t* nfronts;   // [1]
  int32_t* chosen;    // [keep] or null
  int32_t* count;     // scratch [n]
  int32_t* ord0;      // scratch [n] front-local order along axis 0
  int32_t* ord1;      // scratch [n] front-local order along axis 1
  int32_t* front_of_pos;  // scratch [n]
};

void launch_nsga2(const NsArgs& a, cudaStream_t st);

// Archive merge and hypervolume (nsga2.cu)
struct ArchArgs {
  int n;
  const double* c;
  const double* e;
  int32_t* keep;      // [n] kept indices in order
  int32_t* n_keep;    // [1]
};

struct HvArgs {
  int n;
  const double* c;
  const double* e;
  double ref_c, ref_e;
  double* sc;         // scratch [n] inside points in sweep order
  double* se;         // scratch [n]
  double* area;       // scratch [n] step areas
  int32_t* flag;      // scratch [n] the point steps the ceiling down
  double* out;        // [1]
};

void launch_archive_merge(const ArchArgs& a, cudaStream_t st);

// dataset bytes -> split arrays (splits.cu)
void launch_decode_u8(const uint8_t* px, int64_t count, double* x, int sms, cudaStream_t st);
void launch_to_f32(const double* x, int64_t n, float* y, int sms, cudaStream_t st);
void launch_decode_cifar(const uint8_t* rec, int64_t rows, int C, int HW, double* x,
                         int64_t* labels, int sms, cudaStream_t st);
void launch_one_hot(const int64_t* labels, int64_t rows, int classes, double* y, int sms,
                    cudaStream_t st);
void launch_hypervolume(const HvArgs& a, cudaStream_t st);

}  // namespace gevo
