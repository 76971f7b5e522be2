/* gevo.h -- C ABI of libgevo, the B200 fitness evaluator for GEVO-ML.
 *
 * The reference evaluates one patched program at a time on the CPU through
 * Python objects.  libgevo evaluates a whole generation per call.  Each
 * entry point names the reference interface it replaces:
 *
 *   gevo_create / gevo_destroy   -- (no reference analogue: owns a device,
 *                                   a stream and all device memory)
 *   gevo_upload_split            -- SplitView.whole_batches
 *                                   (pkg/src/evotir/datasets.py:149-162),
 *                                   uploaded once instead of per evaluation
 *   gevo_upload_split_u8         -- read_idx_images / load_dataset scaling
 *                                   (datasets.py:33-45,187-192) +
 *                                   whole_batches: raw pixel bytes decoded
 *                                   on the device
 *   gevo_upload_split_cifar      -- (new, CNN workload A24) CIFAR-10 binary
 *                                   records decoded to NHWC on the device
 *   gevo_download_split          -- (no analogue: reads a split back)
 *   gevo_upload_weights          -- module.constants[w1,b1,w2,b2]
 *                                   (fitness.py:341, fitness.py:388)
 *   gevo_eval                    -- evaluate() for a list of variants
 *                                   (fitness.py:372-393, holdout_report
 *                                   fitness.py:396-426), i.e. the body of
 *                                   _Evaluator.__call__ (search.py:257-273)
 *   gevo_exec_once               -- ExecPlan.run on explicit inputs
 *                                   (interpreter.py:219-225, eval_op :272)
 *   gevo_nsga2_rank              -- rank_population (search.py:143-150):
 *                                   nondominated_sort :96-120 +
 *                                   crowding_distance :123-140
 *   gevo_nsga2_crowding          -- crowding_distance (search.py:123-140)
 *   gevo_nsga2_select            -- select_survivors (search.py:163-179)
 *   gevo_archive_merge           -- Archive.offer (search.py:208-228) for a
 *                                   batch of offers with new keys
 *   gevo_hypervolume             -- hypervolume (search.py:182-195)
 *   gevo_comm_unique_id /        -- (no reference analogue: the reference is
 *   gevo_comm_init /                single-process) one NCCL communicator per
 *   gevo_allgather /                context; ONE all-gather of fixed-size
 *   gevo_comm_destroy               fitness records per generation after each
 *                                   rank evaluated its shard of the fresh
 *                                   patches of _Evaluator.__call__
 *                                   (search.py:257-273), SURVEY.md §8(e)
 *   gevo_last_error              -- (Python exceptions in the reference)
 *   gevo_profile                 -- (no analogue: per-instruction-class
 *                                   cycle counters for diagnostics)
 *   gevo_last_kernel_ms          -- (no analogue: device time of the last
 *                                   gevo_eval launch, CUDA events on the
 *                                   context's stream)
 *   gevo_span_ms                 -- (no analogue: device span of a
 *                                   generation split over two contexts)
 *   gevo_range_push /            -- (no analogue: the reference has only
 *   gevo_range_pop                  wall time, search.py:342,396) NVTX
 *                                   ranges for nsys / ncu timelines
 *
 * Conventions: every call returns 0 on success and a negative GEVO_E_* code
 * on failure (then gevo_last_error explains); no C++ exception crosses the
 * ABI.  The caller owns host buffers; the context owns device memory.  One
 * context per device, used by one host thread at a time.  Results are
 * deterministic: no floating-point atomics anywhere.
 * The launch-plan format consumed by gevo_eval is in gevo_plan.h.
 */
#ifndef GEVO_H
#define GEVO_H
#include <stddef.h>
#include <stdint.h>
#include "gevo_plan.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gevo_ctx gevo_ctx;

enum {
  GEVO_OK = 0,
  GEVO_E_ARG = -1,      /* bad argument / malformed plan */
  GEVO_E_CUDA = -2,     /* CUDA runtime failure */
  GEVO_E_NOSPLIT = -3,  /* split id not uploaded */
  GEVO_E_STATE = -4,    /* weights not uploaded, ... */
  GEVO_E_COMM = -5      /* NCCL unavailable or failed */
};

/* per-individual status: the reference's failure encodings (fitness.py:
 * 347-351 blow-up -> error 1.0; 364-365 non-finite probabilities -> 1.0) */
enum {
  GEVO_STATUS_OK = 0,
  GEVO_STATUS_NONFINITE_WEIGHTS = 1,
  GEVO_STATUS_NONFINITE_PROBS = 2,
  GEVO_STATUS_EXEC_ERROR = 3
};

enum { GEVO_MODE_TRAIN = 0, GEVO_MODE_PREDICT = 1 };

typedef struct {
  int64_t wrong;      /* misclassified examples (0 unless status OK) */
  int64_t total;      /* scored examples (0 unless status OK) */
  int32_t status;     /* GEVO_STATUS_* */
  int32_t steps_run;  /* training steps executed before an early exit */
  int64_t cycles;     /* SM clock cycles this individual's CTA ran (diagnostics:
                         load balance, stragglers) */
  int64_t t0_ns, t1_ns; /* global timer at the CTA's start and end (ns) */
  int32_t smid;       /* SM the CTA ran on */
  int32_t pad;
} gevo_result;

typedef struct {
  int32_t mode;          /* GEVO_MODE_TRAIN | GEVO_MODE_PREDICT */
  int32_t steps;         /* WorkloadConfig.steps (fitness.py:61) */
  int32_t check_every;   /* WorkloadConfig.finite_check_every */
  int32_t train_split;   /* split whose batches train (search) */
  int32_t score_split;   /* split scored by @forward (search or holdout) */
  int32_t want_weights;  /* copy final weights out (n_ind * weight_elems) */
} gevo_eval_desc;

int gevo_create(int device, gevo_ctx** out);
int gevo_destroy(gevo_ctx* ctx);
const char* gevo_last_error(gevo_ctx* ctx);

/* x: n x features row-major float64; labels: n int64.  Keeps the whole
 * batches (partial trailing batch dropped) with one-hot targets. */
int gevo_upload_split(gevo_ctx* ctx, int split_id, const double* x, int64_t n,
                      int features, const int64_t* labels, int classes,
                      int batch);

/* Same split from raw pixel bytes (n x features uint8): x = u8 / 255.0 is
 * computed on the device, bit-identical to u8.astype(float64) / 255.0
 * (datasets.py:44,192). */
int gevo_upload_split_u8(gevo_ctx* ctx, int split_id, const uint8_t* pixels,
                         int64_t n, int features, const int64_t* labels,
                         int classes, int batch);

/* CIFAR-10 binary records, each [label u8][channels planes of side*side u8];
 * decoded on the device to NHWC rows x = u8 / 255.0 (features =
 * side*side*channels) plus labels and one-hot targets. */
int gevo_upload_split_cifar(gevo_ctx* ctx, int split_id, const uint8_t* records,
                            int64_t n, int channels, int side, int classes,
                            int batch);

/* Copy a split's device arrays back (any pointer may be NULL); *rows = the
 * number of rows kept (whole batches). */
int gevo_download_split(gevo_ctx* ctx, int split_id, double* x, double* y,
                        int64_t* labels, int64_t* rows);

/* concatenated initial (training) or frozen (prediction) weight arrays,
 * C order, in @train_step return order */
int gevo_upload_weights(gevo_ctx* ctx, const double* w, int64_t n_elems);

/* One launch over the plan's programs.  results[prog.result_slot] receives
 * each individual's record (the caller sizes `results` for header.n_prog
 * records); programs that share a slot are the score parts of one
 * prediction-mode individual (GEVO_FLAG_PART) and are merged here. */
int gevo_eval(gevo_ctx* ctx, const void* plan, size_t plan_bytes,
              const gevo_eval_desc* desc, gevo_result* results,
              double* final_weights);

/* run prog.train0 once per prog: params from `params` (prog.param_off),
 * returns into `outs` (prog.out_off); 64-bit words */
int gevo_exec_once(gevo_ctx* ctx, const void* plan, size_t plan_bytes,
                   const double* params, size_t param_words, double* outs,
                   size_t out_words);

/* rank[i], crowding[i] for every point; front_of_order lists point indices
 * front by front (front 0 in index order, later fronts ascending, as
 * nondominated_sort returns them); front_start[f] indexes it (n_fronts+1
 * entries).  Bit-exact with search.py:96-150. */
int gevo_nsga2_rank(gevo_ctx* ctx, const double* cost, const double* error,
                    int n, int32_t* rank, double* crowding,
                    int32_t* front_order, int32_t* front_start,
                    int32_t* n_fronts);

/* Archive.offer (search.py:208-228) of a whole batch: points 0..n-1 are the
 * archive entries in order followed by the batch's valid offers in offer
 * order, all with keys that are not in the archive and not repeated in the
 * batch (the caller splits a batch at a repeated key; search.py:211).
 * keep[0..*n_keep) = indices of the resulting entries, in archive order;
 * identical to offering the batch one point at a time.  keep holds n ints. */
int gevo_archive_merge(gevo_ctx* ctx, const double* cost, const double* error,
                       int n, int32_t* keep, int32_t* n_keep);

/* hypervolume(points, ref) (search.py:182-195), bit-identical */
int gevo_hypervolume(gevo_ctx* ctx, const double* cost, const double* error,
                     int n, double ref_cost, double ref_error, double* out);

/* crowding_distance (search.py:123-140) of points taken as ONE front
 * (ties on an axis break by position) */
int gevo_nsga2_crowding(gevo_ctx* ctx, const double* cost, const double* error,
                        int n, double* crowding);

/* indices chosen by select_survivors(pool, keep) in survivor order, plus the
 * rank/crowding it assigns (search.py:163-179) */
int gevo_nsga2_select(gevo_ctx* ctx, const double* cost, const double* error,
                      int n, int keep, int32_t* chosen, int32_t* rank,
                      double* crowding);

/* instruction-class profile (diagnostics): with enable != 0 the following
 * gevo_eval calls accumulate, per class (op*16+sub)*2+big, the CTA cycles
 * spent and the count, into GEVO_PROFILE_SLOTS (cycles, count) pairs; `out`
 * (n int64, may be null) receives the last accumulation. */
#define GEVO_PROFILE_SLOTS 256
int gevo_profile(gevo_ctx* ctx, int enable, int64_t* out, int n);

/* device milliseconds of the evaluation kernel of the last gevo_eval */
int gevo_last_kernel_ms(gevo_ctx* ctx, double* ms);

/* device milliseconds from the start of `first`'s last gevo_eval to the end
 * of the later of the two contexts' last gevo_eval (one generation split in
 * two halves over two contexts/streams of the same device) */
int gevo_span_ms(gevo_ctx* first, gevo_ctx* second, double* ms);

/* NCCL plumbing for population sharding (NCCL is dlopen'ed on first use).
 * gevo_comm_unique_id writes an ncclUniqueId (128 bytes; len >= 128) that
 * rank 0 creates and every rank passes to gevo_comm_init.  gevo_allgather
 * copies `bytes` from host `send`, all-gathers them over the context's
 * communicator on its stream (NVLink/NVSwitch between the GPUs of a node)
 * and writes world * bytes, rank-major, to host `recv`. */
int gevo_comm_unique_id(void* out, size_t len);
int gevo_comm_init(gevo_ctx* ctx, int rank, int world, const void* uid, size_t len);
int gevo_allgather(gevo_ctx* ctx, const void* send, size_t bytes, void* recv);
int gevo_comm_destroy(gevo_ctx* ctx);

/* NVTX ranges (header-only NVTX 3: free unless a tool such as nsys or ncu
 * --nvtx is attached).  The library itself marks gevo_eval (plan upload,
 * launch + wait), gevo_exec_once, the NSGA-II / archive / hypervolume calls
 * and gevo_allgather; the host pushes one range per generation and chunk.
 * Ranges nest per calling thread. */
int gevo_range_push(const char* name);
int gevo_range_pop(void);

/* device and build info, e.g. "NVIDIA B200 sm_100 148 SMs" */
int gevo_device_info(gevo_ctx* ctx, char* buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif
