// gevo_abi.cu -- the C ABI of libgevo (declared in include/gevo.h).
//
// Owns the device, one stream, the resident dataset splits, the shared
// initial weights and the growable device arena; validates plans; no C++
// exception crosses the boundary.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <mutex>
#include <string>
#include <vector>
#include "gevo.h"
#include "gevo_exec.cuh"

using namespace gevo;

namespace {

// one NVTX range for the lifetime of a scope (NVTX 3 is header-only: a
// push/pop costs a branch unless a tool is attached)
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

struct Split {
  double* x = nullptr;         // [nb, B, F]
  double* y = nullptr;         // [nb, B, C] one-hot
  int64_t* labels = nullptr;   // [nb, B]
  int nb = 0, batch = 0, features = 0, classes = 0;
};

// Device buffer that grows on demand.  Growth is stream-ordered
// (cudaFreeAsync / cudaMallocAsync on the owning context's stream): a plain
// cudaFree synchronises the whole device, which serialised the two halves of
// a generation running on two contexts whenever a buffer grew.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes, cudaStream_t st) {
    if (bytes <= cap) return 0;
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    cap = 0;
    size_t want = bytes + bytes / 4 + 256;
    if (cudaMallocAsync(&p, want, st) != cudaSuccess) return -1;
    cap = want;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// the tcgen05 executor build (gevo_exec_tc.cu, its own module: tf32 and bf16)
extern "C" void gevo_internal_launch_eval_tc(const void* a, int n_prog, cudaStream_t st);
extern "C" void gevo_internal_launch_once_tc(const void* a, int n_prog, cudaStream_t st);

// The DOT arithmetic (GEVO_B200_DTYPE): "f64" (default) -- float64 in the
// reference's summation orders on DMMA, bit-exact; "tf32" -- tcgen05 tensor
// cores with tf32 operands and fp32 accumulation (dot_tc.cuh); "bf16" -- the
// same with bf16 operands (kind::f16).  The last two are reduced-precision
// modes whose fitness is reported against the reference, not gated.
// -1: unknown value.
int tc_mode() {
  const char* v = getenv("GEVO_B200_DTYPE");
  if (!v || !*v || !strcmp(v, "f64")) return 0;
  if (!strcmp(v, "tf32")) return 1;
  if (!strcmp(v, "bf16")) return 2;
  return -1;
}

}  // namespace

struct gevo_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  Split splits[4];
  double* weights = nullptr;
  int64_t weight_elems = 0;
  DevBuf plan, arena, results, finalw, params, outs, ns;
  DevBuf wreg;                       // training: every program's weight blocks (L2 window)
  DevBuf x32;                        // tf32 mode: fp32 mirror of the training split's x
  void* window_base = nullptr;       // the stream's current L2 access window
  size_t window_bytes = 0;
  bool persist_limit_set = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  bool profile = false;
  DevBuf prof;
  ncclComm_t comm = nullptr;   // gevo_comm_init: the population all-gather
  int comm_rank = 0, comm_world = 1;
  DevBuf gather;
};

static int fail(gevo_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

static int cuda_fail(gevo_ctx* c, cudaError_t e, const char* what) {
  return fail(c, GEVO_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                              \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr);  \
  } while (0)

namespace {

struct PlanView {
  const gevo_plan_header* h;
  size_t instr_off, prog_off, const_off;
};

int parse_plan(gevo_ctx* ctx, const void* plan, size_t bytes, PlanView* v) {
  if (!plan || bytes < sizeof(gevo_plan_header))
    return fail(ctx, GEVO_E_ARG, "plan blob too small");
  const gevo_plan_header* h = static_cast<const gevo_plan_header*>(plan);
  if (h->magic != GEVO_PLAN_MAGIC || h->version != GEVO_PLAN_VERSION)
    return fail(ctx, GEVO_E_ARG, "bad plan magic/version");
  if (h->n_instr < 0 || h->n_prog < 0 || h->n_const < 0 || h->total_elems < 0)
    return fail(ctx, GEVO_E_ARG, "negative plan counts");
  if (h->max_smem < 0 || h->max_smem > 24576)
    return fail(ctx, GEVO_E_ARG, "shared-memory scratch exceeds 192 KB");
  size_t need = sizeof(gevo_plan_header) + (size_t)h->n_instr * sizeof(gevo_instr) +
                (size_t)h->n_prog * sizeof(gevo_prog) + (size_t)h->n_const * 8;
  if (need != bytes) return fail(ctx, GEVO_E_ARG, "plan size mismatch");
  v->h = h;
  v->instr_off = sizeof(gevo_plan_header);
  v->prog_off = v->instr_off + (size_t)h->n_instr * sizeof(gevo_instr);
  v->const_off = v->prog_off + (size_t)h->n_prog * sizeof(gevo_prog);
  // host-side validation of every instruction range
  const gevo_prog* progs = reinterpret_cast<const gevo_prog*>(
      static_cast<const char*>(plan) + v->prog_off);
  for (int i = 0; i < h->n_prog; ++i) {
    const gevo_prog& p = progs[i];
    auto ok = [&](int o, int n) { return o >= 0 && n >= 0 && o + n <= h->n_instr; };
    if (!ok(p.train0, p.train0_n) || !ok(p.train1, p.train1_n) || !ok(p.train2, p.train2_n) ||
        !ok(p.fwd, p.fwd_n))
      return fail(ctx, GEVO_E_ARG, "prog instruction range out of bounds");
    if (p.arena_off < 0 || p.arena_off > h->total_elems)
      return fail(ctx, GEVO_E_ARG, "prog arena offset out of bounds");
    if (p.result_slot < 0 || p.result_slot >= h->n_prog)
      return fail(ctx, GEVO_E_ARG, "prog result slot out of bounds");
    if (GEVO_FLAG_PART(p.flags) >= GEVO_FLAG_NPARTS(p.flags))
      return fail(ctx, GEVO_E_ARG, "prog score part out of range");
  }
  return 0;
}

int upload_plan(gevo_ctx* ctx, const void* plan, size_t bytes, const PlanView& v,
                const gevo_instr** di, const gevo_prog** dp, const double** dc) {
  if (ctx->plan.ensure(bytes + 16, ctx->stream)) return fail(ctx, GEVO_E_CUDA, "plan alloc failed");
  CK(cudaMemcpyAsync(ctx->plan.p, plan, bytes, cudaMemcpyHostToDevice, ctx->stream));
  char* base = static_cast<char*>(ctx->plan.p);
  *di = reinterpret_cast<const gevo_instr*>(base + v.instr_off);
  *dp = reinterpret_cast<const gevo_prog*>(base + v.prog_off);
  *dc = reinterpret_cast<const double*>(base + v.const_off);
  return 0;
}

// per-program records -> results[result_slot]: a whole individual is copied;
// score parts add their integer counts, a non-finite part makes the whole
// individual non-finite (the reference stops at its first non-finite batch
// and returns error 1.0 whichever batch it was), timings span the parts
void merge_results(const gevo_prog* progs, int n_prog, const gevo_result* per_prog, gevo_result* out) {
  std::vector<uint8_t> done((size_t)n_prog, 0);
  for (int i = 0; i < n_prog; ++i) {
    const int s = progs[i].result_slot;
    const gevo_result& r = per_prog[i];
    gevo_result& o = out[s];
    if (!done[s]) { o = r; done[s] = 1; continue; }
    if (o.status == GEVO_STATUS_OK && r.status == GEVO_STATUS_OK) {
      o.wrong += r.wrong;
      o.total += r.total;
    } else if (o.status == GEVO_STATUS_OK) {
      o.status = r.status;
      o.wrong = o.total = 0;
    }
    o.steps_run = r.steps_run > o.steps_run ? r.steps_run : o.steps_run;
    o.cycles = r.cycles > o.cycles ? r.cycles : o.cycles;
    o.t0_ns = r.t0_ns < o.t0_ns ? r.t0_ns : o.t0_ns;
    o.t1_ns = r.t1_ns > o.t1_ns ? r.t1_ns : o.t1_ns;
    if (GEVO_FLAG_PART(progs[i].flags) == 0) o.smid = r.smid;
  }
}

}  // namespace

extern "C" {

int gevo_create(int device, gevo_ctx** out) {
  if (!out) return GEVO_E_ARG;
  *out = nullptr;
  gevo_ctx* ctx = new (std::nothrow) gevo_ctx();
  if (!ctx) return GEVO_E_ARG;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
  if (e != cudaSuccess) {
    // keep the context so the caller can read the error
    ctx->err = std::string("cuda init: ") + cudaGetErrorString(e);
    *out = ctx;
    return GEVO_E_CUDA;
  }
  *out = ctx;
  return GEVO_OK;
}

int gevo_destroy(gevo_ctx* ctx) {
  if (!ctx) return GEVO_E_ARG;
  cudaSetDevice(ctx->device);
  for (auto& s : ctx->splits) {
    cudaFree(s.x);
    cudaFree(s.y);
    cudaFree(s.labels);
  }
  cudaFree(ctx->weights);
  ctx->plan.release();
  ctx->arena.release();
  ctx->results.release();
  ctx->finalw.release();
  ctx->params.release();
  ctx->outs.release();
  ctx->ns.release();
  ctx->gather.release();
  ctx->wreg.release();
  ctx->x32.release();
  gevo_comm_destroy(ctx);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return GEVO_OK;
}

const char* gevo_last_error(gevo_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

int gevo_device_info(gevo_ctx* ctx, char* buf, size_t len) {
  if (!ctx || !buf || !len) return GEVO_E_ARG;
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, ctx->device));
  snprintf(buf, len, "%s sm_%d%d %d SMs", p.name, p.major, p.minor, p.multiProcessorCount);
  return GEVO_OK;
}

int gevo_upload_split(gevo_ctx* ctx, int split_id, const double* x, int64_t n,
                      int features, const int64_t* labels, int classes, int batch) {
  if (!ctx) return GEVO_E_ARG;
  if (split_id < 0 || split_id >= 4 || !x || !labels || n < 0 || features <= 0 ||
      classes <= 0 || batch <= 0)
    return fail(ctx, GEVO_E_ARG, "bad split arguments");
  CK(cudaSetDevice(ctx->device));
  Split& s = ctx->splits[split_id];
  cudaFree(s.x);
  cudaFree(s.y);
  cudaFree(s.labels);
  s = Split();
  const int nb = (int)(n / batch);
  const int64_t rows = (int64_t)nb * batch;
  for (int64_t i = 0; i < rows; ++i)
    if (labels[i] < 0 || labels[i] >= classes)
      return fail(ctx, GEVO_E_ARG, "label out of range");
  std::vector<double> y((size_t)rows * classes, 0.0);
  for (int64_t i = 0; i < rows; ++i) y[(size_t)i * classes + labels[i]] = 1.0;
  if (rows > 0) {
    CK(cudaMalloc(&s.x, rows * features * sizeof(double)));
    CK(cudaMalloc(&s.y, rows * classes * sizeof(double)));
    CK(cudaMalloc(&s.labels, rows * sizeof(int64_t)));
    CK(cudaMemcpy(s.x, x, rows * features * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.y, y.data(), rows * classes * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.labels, labels, rows * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  s.nb = nb;
  s.batch = batch;
  s.features = features;
  s.classes = classes;
  return GEVO_OK;
}

// a split's device arrays for nb whole batches (frees the previous ones)
static int alloc_split(gevo_ctx* ctx, int split_id, int64_t n, int features, int classes,
                       int batch, Split** out) {
  Split& s = ctx->splits[split_id];
  cudaFree(s.x);
  cudaFree(s.y);
  cudaFree(s.labels);
  s = Split();
  const int nb = (int)(n / batch);
  const int64_t rows = (int64_t)nb * batch;
  if (rows > 0) {
    CK(cudaMalloc(&s.x, rows * features * sizeof(double)));
    CK(cudaMalloc(&s.y, rows * classes * sizeof(double)));
    CK(cudaMalloc(&s.labels, rows * sizeof(int64_t)));
  }
  s.nb = nb;
  s.batch = batch;
  s.features = features;
  s.classes = classes;
  *out = &s;
  return GEVO_OK;
}

static int device_sms(gevo_ctx* ctx) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess)
    sms = 148;
  return sms;
}

int gevo_upload_split_u8(gevo_ctx* ctx, int split_id, const uint8_t* pixels, int64_t n,
                         int features, const int64_t* labels, int classes, int batch) {
  if (!ctx) return GEVO_E_ARG;
  if (split_id < 0 || split_id >= 4 || !pixels || !labels || n < 0 || features <= 0 ||
      classes <= 0 || batch <= 0)
    return fail(ctx, GEVO_E_ARG, "bad split arguments");
  CK(cudaSetDevice(ctx->device));
  const int64_t rows = (n / batch) * batch;
  for (int64_t i = 0; i < rows; ++i)
    if (labels[i] < 0 || labels[i] >= classes) return fail(ctx, GEVO_E_ARG, "label out of range");
  Split* s = nullptr;
  int rc = alloc_split(ctx, split_id, n, features, classes, batch, &s);
  if (rc) return rc;
  if (rows == 0) return GEVO_OK;
  const int64_t count = rows * features;
  uint8_t* raw = nullptr;
  CK(cudaMalloc(&raw, count));
  CK(cudaMemcpyAsync(raw, pixels, count, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(s->labels, labels, rows * sizeof(int64_t), cudaMemcpyHostToDevice,
                     ctx->stream));
  const int sms = device_sms(ctx);
  launch_decode_u8(raw, count, s->x, sms, ctx->stream);
  launch_one_hot(s->labels, rows, classes, s->y, sms, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(raw);
  return GEVO_OK;
}

int gevo_upload_split_cifar(gevo_ctx* ctx, int split_id, const uint8_t* records, int64_t n,
                            int channels, int side, int classes, int batch) {
  if (!ctx) return GEVO_E_ARG;
  if (split_id < 0 || split_id >= 4 || !records || n < 0 || channels <= 0 || side <= 0 ||
      classes <= 0 || batch <= 0)
    return fail(ctx, GEVO_E_ARG, "bad split arguments");
  CK(cudaSetDevice(ctx->device));
  const int HW = side * side;
  const int64_t rec_bytes = 1 + (int64_t)channels * HW;
  const int64_t rows = (n / batch) * batch;
  for (int64_t i = 0; i < rows; ++i)
    if (records[i * rec_bytes] >= classes) return fail(ctx, GEVO_E_ARG, "label out of range");
  Split* s = nullptr;
  int rc = alloc_split(ctx, split_id, n, channels * HW, classes, batch, &s);
  if (rc) return rc;
  if (rows == 0) return GEVO_OK;
  uint8_t* raw = nullptr;
  CK(cudaMalloc(&raw, rows * rec_bytes));
  CK(cudaMemcpyAsync(raw, records, rows * rec_bytes, cudaMemcpyHostToDevice, ctx->stream));
  const int sms = device_sms(ctx);
  launch_decode_cifar(raw, rows, channels, HW, s->x, s->labels, sms, ctx->stream);
  launch_one_hot(s->labels, rows, classes, s->y, sms, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(raw);
  return GEVO_OK;
}

int gevo_download_split(gevo_ctx* ctx, int split_id, double* x, double* y, int64_t* labels,
                        int64_t* rows) {
  if (!ctx) return GEVO_E_ARG;
  if (split_id < 0 || split_id >= 4 || !rows) return fail(ctx, GEVO_E_ARG, "bad split id");
  CK(cudaSetDevice(ctx->device));
  const Split& s = ctx->splits[split_id];
  const int64_t r = (int64_t)s.nb * s.batch;
  *rows = r;
  if (r == 0) return GEVO_OK;
  if (x) CK(cudaMemcpy(x, s.x, r * s.features * sizeof(double), cudaMemcpyDeviceToHost));
  if (y) CK(cudaMemcpy(y, s.y, r * s.classes * sizeof(double), cudaMemcpyDeviceToHost));
  if (labels) CK(cudaMemcpy(labels, s.labels, r * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return GEVO_OK;
}

int gevo_upload_weights(gevo_ctx* ctx, const double* w, int64_t n_elems) {
  if (!ctx) return GEVO_E_ARG;
  if (!w || n_elems <= 0) return fail(ctx, GEVO_E_ARG, "bad weights");
  CK(cudaSetDevice(ctx->device));
  cudaFree(ctx->weights);
  ctx->weights = nullptr;
  CK(cudaMalloc(&ctx->weights, n_elems * sizeof(double)));
  CK(cudaMemcpy(ctx->weights, w, n_elems * sizeof(double), cudaMemcpyHostToDevice));
  ctx->weight_elems = n_elems;
  return GEVO_OK;
}

int gevo_eval(gevo_ctx* ctx, const void* plan, size_t plan_bytes,
              const gevo_eval_desc* desc, gevo_result* results, double* final_weights) {
  Range nvtx_range("gevo_eval");
  if (!ctx) return GEVO_E_ARG;
  if (!desc || !results) return fail(ctx, GEVO_E_ARG, "null desc/results");
  CK(cudaSetDevice(ctx->device));
  PlanView v;
  int rc = parse_plan(ctx, plan, plan_bytes, &v);
  if (rc) return rc;
  const gevo_plan_header* h = v.h;
  if (h->n_prog == 0) return GEVO_OK;
  if (!ctx->weights) return fail(ctx, GEVO_E_STATE, "weights not uploaded");
  if (h->weight_elems != ctx->weight_elems)
    return fail(ctx, GEVO_E_ARG, "plan weight block does not match uploaded weights");
  if (desc->score_split < 0 || desc->score_split >= 4 || !ctx->splits[desc->score_split].x)
    return fail(ctx, GEVO_E_NOSPLIT, "score split not uploaded");
  const Split& sc = ctx->splits[desc->score_split];
  const Split* tr = nullptr;
  if (desc->mode == GEVO_MODE_TRAIN) {
    if (desc->train_split < 0 || desc->train_split >= 4 || !ctx->splits[desc->train_split].x)
      return fail(ctx, GEVO_E_NOSPLIT, "train split not uploaded");
    tr = &ctx->splits[desc->train_split];
    if (tr->batch != sc.batch || tr->features != sc.features || tr->classes != sc.classes)
      return fail(ctx, GEVO_E_ARG, "train/score split shapes differ");
    if (desc->steps < 0) return fail(ctx, GEVO_E_ARG, "negative steps");
  } else if (desc->mode != GEVO_MODE_PREDICT) {
    return fail(ctx, GEVO_E_ARG, "bad mode");
  }
  if (h->n_weights < 0 || h->n_weights > GEVO_MAXP - 2)
    return fail(ctx, GEVO_E_ARG, "bad weight count");

  // score parts: every result slot needs each of its n_parts programs once;
  // training programs are never split (their steps are sequential)
  const gevo_prog* hp = reinterpret_cast<const gevo_prog*>(static_cast<const char*>(plan) + v.prog_off);
  {
    std::vector<int32_t> nparts(h->n_prog, 0);
    std::vector<uint8_t> seen;
    bool split = false;
    for (int i = 0; i < h->n_prog; ++i) split |= GEVO_FLAG_NPARTS(hp[i].flags) > 1;
    if (split && desc->mode == GEVO_MODE_TRAIN)
      return fail(ctx, GEVO_E_ARG, "score parts in a training plan");
    for (int i = 0; i < h->n_prog; ++i) {
      const int slot = hp[i].result_slot, np = GEVO_FLAG_NPARTS(hp[i].flags);
      if (nparts[slot] == 0) nparts[slot] = np;
      else if (nparts[slot] != np) return fail(ctx, GEVO_E_ARG, "inconsistent score parts");
    }
    std::vector<int64_t> first(h->n_prog, 0);
    int64_t cells = 0;
    for (int s = 0; s < h->n_prog; ++s) { first[s] = cells; cells += nparts[s]; }
    seen.assign((size_t)cells, 0);
    for (int i = 0; i < h->n_prog; ++i) {
      uint8_t& c = seen[(size_t)(first[hp[i].result_slot] + GEVO_FLAG_PART(hp[i].flags))];
      if (c) return fail(ctx, GEVO_E_ARG, "duplicate result slot / score part");
      c = 1;
    }
    for (int64_t c = 0; c < cells; ++c)
      if (!seen[(size_t)c]) return fail(ctx, GEVO_E_ARG, "result slot missing a score part");
  }

  const gevo_instr* di;
  const gevo_prog* dp;
  const double* dc;
  {
    Range r("plan upload");
    rc = upload_plan(ctx, plan, plan_bytes, v, &di, &dp, &dc);
  }
  if (rc) return rc;
  if (ctx->arena.ensure((size_t)h->total_elems * sizeof(double) + 64, ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "arena alloc failed");
  if (ctx->results.ensure((size_t)h->n_prog * sizeof(gevo_result), ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "results alloc failed");
  if (final_weights &&
      ctx->finalw.ensure((size_t)h->n_prog * h->weight_elems * sizeof(double) + 8, ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "final weight alloc failed");

  EvalArgs a;
  memset(&a, 0, sizeof(a));
  a.instrs = di;
  a.progs = dp;
  a.consts = dc;
  a.arena = static_cast<double*>(ctx->arena.p);
  // diagnostics: GEVO_POISON=1 fills every individual's arena (scratch,
  // probs, weight ping-pong) with NaN before the launch, so a read of memory
  // no instruction wrote shows up as a wrong result instead of stale data
  if (getenv("GEVO_POISON"))
    CK(cudaMemsetAsync(ctx->arena.p, 0xFF, (size_t)h->total_elems * sizeof(double), ctx->stream));
  for (int i = 0; i < GEVO_MAXP; ++i) a.wofs[i] = h->wofs[i];
  a.n_weights = h->n_weights;
  a.weight_elems = h->weight_elems;
  a.probs_elems = sc.batch * sc.classes;
  a.mode = desc->mode;
  a.steps = desc->steps;
  a.check_every = desc->check_every;
  a.init_weights = ctx->weights;
  if (tr) {
    a.train_x = tr->x;
    a.train_y = tr->y;
    a.train_nb = tr->nb;
  }
  a.score_x = sc.x;
  a.score_labels = sc.labels;
  a.score_nb = sc.nb;
  a.batch = sc.batch;
  a.classes = sc.classes;
  a.x_elems = (int64_t)sc.batch * sc.features;
  a.y_elems = (int64_t)sc.batch * sc.classes;
  a.results = static_cast<gevo_result*>(ctx->results.p);
  a.final_weights = final_weights ? static_cast<double*>(ctx->finalw.p) : nullptr;
  a.smem_elems = h->max_smem;
  a.tc = tc_mode();
  if (a.tc < 0) return fail(ctx, GEVO_E_ARG, "GEVO_B200_DTYPE must be f64, tf32 or bf16");
  a.prof = nullptr;
  if (ctx->profile) {
    if (ctx->prof.ensure(GEVO_PROFILE_SLOTS * 2 * 8, ctx->stream)) return fail(ctx, GEVO_E_CUDA, "profile alloc");
    CK(cudaMemsetAsync(ctx->prof.p, 0, GEVO_PROFILE_SLOTS * 2 * 8, ctx->stream));
    a.prof = static_cast<unsigned long long*>(ctx->prof.p);
  }
  if (a.mode == GEVO_MODE_TRAIN && a.train_nb == 0 && a.steps > 0)
    return fail(ctx, GEVO_E_ARG, "train split has no whole batch");
  // tf32 mode, training: an fp32 mirror of the training split's x and a TMA
  // tensor map over it (8 x 4 boxes = one canonical core matrix each), so the
  // tcgen05 dots take their shared A operand by cp.async.bulk.tensor
  // (dot_tc.cuh).  GEVO_B200_TMA=0 stages it with the threads instead.
  if (a.tc == 1 && a.mode == GEVO_MODE_TRAIN && tr && tr->x && tr->features % 4 == 0) {
    const char* et = getenv("GEVO_B200_TMA");
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      cudaGetLastError();
    }
    const int64_t rows = (int64_t)tr->nb * tr->batch, cols = tr->features;
    if ((!et || atoi(et) != 0) && encode && rows > 0) {
      if (ctx->x32.ensure((size_t)(rows * cols) * sizeof(float), ctx->stream))
        return fail(ctx, GEVO_E_CUDA, "x32 alloc failed");
      launch_to_f32(tr->x, rows * cols, static_cast<float*>(ctx->x32.p), device_sms(ctx), ctx->stream);
      CUtensorMap map;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
      cuuint32_t box[2] = {4, 8};
      cuuint32_t estr[2] = {1, 1};
      if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ctx->x32.p, dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
        static_assert(sizeof(map) == sizeof(a.tma_map), "CUtensorMap size");
        memcpy(a.tma_map, &map, sizeof map);
        a.tma_x64 = tr->x;
        a.tma_rows = rows;
        a.tma_cols = (int)cols;
      }
    }
  }
  // Training: the weight blocks move to one region, all block 0s first.
  // Block 0 is where in-place weights live for the whole launch (w1: 200 KB
  // per individual, read twice and written once per step), so one L2
  // persisting access window can cover exactly the hot weights
  // (GEVO_B200_L2WINDOW=1; off by default: +1 % on the bench's one launch of
  // 256, but -30 % on the recorded 512 x 50 run's many smaller launches
  // alternating between two contexts, profiles/r02_experiments.md).  The window stays on the context's stream; the
  // blocks are zeroed at every launch start, so lines left persisting hold no
  // input of the next launch.
  if (a.mode == GEVO_MODE_TRAIN && a.steps > 0) {
    const size_t wsz = (size_t)((h->weight_elems + 15) & ~15);
    const size_t bytes = 2 * wsz * (size_t)h->n_prog * sizeof(double);
    if (ctx->wreg.ensure(bytes, ctx->stream)) return fail(ctx, GEVO_E_CUDA, "weight region alloc failed");
    a.wreg = static_cast<double*>(ctx->wreg.p);
    a.n_prog = h->n_prog;
    if (getenv("GEVO_POISON"))          // the weight region too (see the arena's poison)
      CK(cudaMemsetAsync(ctx->wreg.p, 0xFF, bytes, ctx->stream));
    const char* ew = getenv("GEVO_B200_L2WINDOW");
    if (ew && atoi(ew) != 0) {
      int max_persist = 0, max_window = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
      const size_t hot = wsz * (size_t)h->n_prog * sizeof(double);
      const size_t nbytes = hot < (size_t)max_window ? hot : (size_t)max_window;
      if (max_persist > 0 && max_window > 0 &&
          (ctx->window_base != ctx->wreg.p || ctx->window_bytes != nbytes)) {
        if (!ctx->persist_limit_set) {      // device-wide, once per context
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
          ctx->persist_limit_set = true;
        }
        cudaStreamAttrValue v;
        memset(&v, 0, sizeof v);
        v.accessPolicyWindow.base_ptr = ctx->wreg.p;
        v.accessPolicyWindow.num_bytes = hot < (size_t)max_window ? hot : (size_t)max_window;
        const double ratio = (double)max_persist / (double)v.accessPolicyWindow.num_bytes;
        v.accessPolicyWindow.hitRatio = ratio < 1.0 ? (float)ratio : 1.0f;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        if (cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess) {
          ctx->window_base = ctx->wreg.p;
          ctx->window_bytes = nbytes;
        }
        cudaGetLastError();
      }
    }
  }
  Range launch_range(a.tc ? "eval_kernel_tc launch + wait" : "eval_kernel launch + wait");
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  if (a.tc) gevo_internal_launch_eval_tc(&a, h->n_prog, ctx->stream);
  else launch_eval(a, h->n_prog, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  std::vector<gevo_result> per_prog((size_t)h->n_prog);
  CK(cudaMemcpyAsync(per_prog.data(), ctx->results.p, (size_t)h->n_prog * sizeof(gevo_result),
                     cudaMemcpyDeviceToHost, ctx->stream));
  if (final_weights)
    CK(cudaMemcpyAsync(final_weights, ctx->finalw.p,
                       (size_t)h->n_prog * h->weight_elems * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  merge_results(hp, h->n_prog, per_prog.data(), results);
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->last_ms = ms;
  return GEVO_OK;
}

int gevo_range_push(const char* name) {
  if (!name) return GEVO_E_ARG;
  nvtxRangePushA(name);
  return GEVO_OK;
}

int gevo_range_pop(void) {
  nvtxRangePop();
  return GEVO_OK;
}

int gevo_profile(gevo_ctx* ctx, int enable, int64_t* out, int n) {
  if (!ctx) return GEVO_E_ARG;
  ctx->profile = enable != 0;
  if (out && n > 0) {
    if (!ctx->prof.p) { memset(out, 0, (size_t)n * 8); return GEVO_OK; }
    const int k = n < GEVO_PROFILE_SLOTS * 2 ? n : GEVO_PROFILE_SLOTS * 2;
    CK(cudaMemcpy(out, ctx->prof.p, (size_t)k * 8, cudaMemcpyDeviceToHost));
  }
  return GEVO_OK;
}

int gevo_last_kernel_ms(gevo_ctx* ctx, double* ms) {
  if (!ctx || !ms) return GEVO_E_ARG;
  *ms = ctx->last_ms;
  return GEVO_OK;
}

int gevo_span_ms(gevo_ctx* first, gevo_ctx* second, double* ms) {
  if (!first || !second || !ms) return GEVO_E_ARG;
  gevo_ctx* ctx = first;   // CK reports into the first context
  if (first->device != second->device) return fail(ctx, GEVO_E_ARG, "contexts on different devices");
  CK(cudaSetDevice(first->device));
  float a = 0.f, b = 0.f;
  CK(cudaEventElapsedTime(&a, first->ev0, first->ev1));
  CK(cudaEventElapsedTime(&b, first->ev0, second->ev1));
  *ms = a > b ? a : b;
  return GEVO_OK;
}

int gevo_exec_once(gevo_ctx* ctx, const void* plan, size_t plan_bytes, const double* params,
                   size_t param_words, double* outs, size_t out_words) {
  Range nvtx_range("gevo_exec_once");
  if (!ctx) return GEVO_E_ARG;
  if (!params || !outs) return fail(ctx, GEVO_E_ARG, "null params/outs");
  CK(cudaSetDevice(ctx->device));
  PlanView v;
  int rc = parse_plan(ctx, plan, plan_bytes, &v);
  if (rc) return rc;
  const gevo_plan_header* h = v.h;
  if (h->n_prog == 0) return GEVO_OK;
  const gevo_instr* di;
  const gevo_prog* dp;
  const double* dc;
  rc = upload_plan(ctx, plan, plan_bytes, v, &di, &dp, &dc);
  if (rc) return rc;
  if (ctx->arena.ensure((size_t)h->total_elems * sizeof(double) + 64, ctx->stream) ||
      ctx->params.ensure(param_words * 8 + 8, ctx->stream) || ctx->outs.ensure(out_words * 8 + 8, ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "exec-once alloc failed");
  CK(cudaMemcpyAsync(ctx->params.p, params, param_words * 8, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemsetAsync(ctx->outs.p, 0, out_words * 8, ctx->stream));
  OnceArgs a;
  a.instrs = di;
  a.progs = dp;
  a.consts = dc;
  a.arena = static_cast<double*>(ctx->arena.p);
  a.params = static_cast<const double*>(ctx->params.p);
  a.outs = static_cast<double*>(ctx->outs.p);
  a.tc = tc_mode();
  if (a.tc < 0) return fail(ctx, GEVO_E_ARG, "GEVO_B200_DTYPE must be f64, tf32 or bf16");
  a.smem_elems = h->max_smem;
  if (a.tc) gevo_internal_launch_once_tc(&a, h->n_prog, ctx->stream);
  else launch_once(a, h->n_prog, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(outs, ctx->outs.p, out_words * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return GEVO_OK;
}

static int nsga2_common(gevo_ctx* ctx, const double* cost, const double* error, int n,
                        int keep, int32_t* chosen, int32_t* rank, double* crowding,
                        int32_t* front_order, int32_t* front_start, int32_t* n_fronts,
                        int one_front = 0) {
  if (!ctx) return GEVO_E_ARG;
  if (n < 0 || !cost || !error) return fail(ctx, GEVO_E_ARG, "bad nsga2 arguments");
  if (n == 0) {
    if (n_fronts) *n_fronts = 0;
    if (front_start) front_start[0] = 0;
    return GEVO_OK;
  }
  CK(cudaSetDevice(ctx->device));
  // layout: c[n] e[n] crowd[n] | rank order fstart(n+1) nf count ord0 ord1 fop chosen
  size_t dbl = 3 * (size_t)n * 8;
  size_t ints = (size_t)(8 * n + 2 + (keep > 0 ? keep : 0)) * 4;
  if (ctx->ns.ensure(dbl + ints + 64, ctx->stream)) return fail(ctx, GEVO_E_CUDA, "nsga2 alloc failed");
  double* d = static_cast<double*>(ctx->ns.p);
  int32_t* iv = reinterpret_cast<int32_t*>(d + 3 * (size_t)n);
  NsArgs a;
  a.n = n;
  a.keep = keep;
  a.one_front = one_front;
  a.c = d;
  a.e = d + n;
  a.crowd = d + 2 * (size_t)n;
  a.rank = iv;
  a.order = iv + n;
  a.fstart = iv + 2 * n;
  a.nfronts = iv + 3 * n + 1;
  a.count = iv + 3 * n + 2;
  a.ord0 = iv + 4 * n + 2;
  a.ord1 = iv + 5 * n + 2;
  a.front_of_pos = iv + 6 * n + 2;
  a.chosen = chosen ? iv + 7 * n + 2 : nullptr;
  CK(cudaMemcpyAsync(d, cost, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d + n, error, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  launch_nsga2(a, ctx->stream);
  CK(cudaGetLastError());
  int32_t nf = 0;
  CK(cudaMemcpyAsync(&nf, a.nfronts, 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (rank) CK(cudaMemcpyAsync(rank, a.rank, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (crowding)
    CK(cudaMemcpyAsync(crowding, a.crowd, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (front_order)
    CK(cudaMemcpyAsync(front_order, a.order, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (front_start)
    CK(cudaMemcpy(front_start, a.fstart, (size_t)(nf + 1) * 4, cudaMemcpyDeviceToHost));
  if (chosen && keep > 0)
    CK(cudaMemcpy(chosen, a.chosen, (size_t)keep * 4, cudaMemcpyDeviceToHost));
  if (n_fronts) *n_fronts = nf;
  return GEVO_OK;
}

int gevo_archive_merge(gevo_ctx* ctx, const double* cost, const double* error, int n,
                       int32_t* keep, int32_t* n_keep) {
  Range nvtx_range("gevo_archive_merge");
  if (!ctx) return GEVO_E_ARG;
  if (n < 0 || (n > 0 && (!cost || !error || !keep)) || !n_keep)
    return fail(ctx, GEVO_E_ARG, "bad archive_merge arguments");
  *n_keep = 0;
  if (n == 0) return GEVO_OK;
  CK(cudaSetDevice(ctx->device));
  if (ctx->ns.ensure(2 * (size_t)n * 8 + ((size_t)n + 2) * 4 + 64, ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "archive alloc failed");
  double* d = static_cast<double*>(ctx->ns.p);
  int32_t* iv = reinterpret_cast<int32_t*>(d + 2 * (size_t)n);
  ArchArgs a;
  a.n = n;
  a.c = d;
  a.e = d + n;
  a.keep = iv;
  a.n_keep = iv + n;
  CK(cudaMemcpyAsync(d, cost, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d + n, error, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  launch_archive_merge(a, ctx->stream);
  CK(cudaGetLastError());
  int32_t k = 0;
  CK(cudaMemcpyAsync(&k, a.n_keep, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (k < 0 || k > n) return fail(ctx, GEVO_E_CUDA, "archive merge returned a bad count");
  if (k) CK(cudaMemcpy(keep, a.keep, (size_t)k * 4, cudaMemcpyDeviceToHost));
  *n_keep = k;
  return GEVO_OK;
}

int gevo_hypervolume(gevo_ctx* ctx, const double* cost, const double* error, int n,
                     double ref_cost, double ref_error, double* out) {
  Range nvtx_range("gevo_hypervolume");
  if (!ctx) return GEVO_E_ARG;
  if (n < 0 || (n > 0 && (!cost || !error)) || !out)
    return fail(ctx, GEVO_E_ARG, "bad hypervolume arguments");
  *out = 0.0;
  if (n == 0) return GEVO_OK;
  CK(cudaSetDevice(ctx->device));
  if (ctx->ns.ensure((5 * (size_t)n + 1) * 8 + (size_t)n * 4 + 64, ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "hypervolume alloc failed");
  double* d = static_cast<double*>(ctx->ns.p);
  HvArgs a;
  a.n = n;
  a.c = d;
  a.e = d + n;
  a.sc = d + 2 * (size_t)n;
  a.se = d + 3 * (size_t)n;
  a.area = d + 4 * (size_t)n;
  a.out = d + 5 * (size_t)n;
  a.flag = reinterpret_cast<int32_t*>(d + 5 * (size_t)n + 1);
  a.ref_c = ref_cost;
  a.ref_e = ref_error;
  CK(cudaMemcpyAsync(d, cost, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d + n, error, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  launch_hypervolume(a, ctx->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, a.out, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return GEVO_OK;
}

int gevo_nsga2_rank(gevo_ctx* ctx, const double* cost, const double* error, int n,
                    int32_t* rank, double* crowding, int32_t* front_order,
                    int32_t* front_start, int32_t* n_fronts) {
  Range nvtx_range("gevo_nsga2_rank");
  return nsga2_common(ctx, cost, error, n, 0, nullptr, rank, crowding, front_order,
                      front_start, n_fronts);
}

int gevo_nsga2_crowding(gevo_ctx* ctx, const double* cost, const double* error, int n,
                        double* crowding) {
  Range nvtx_range("gevo_nsga2_crowding");
  return nsga2_common(ctx, cost, error, n, 0, nullptr, nullptr, crowding, nullptr, nullptr,
                      nullptr, 1);
}

int gevo_nsga2_select(gevo_ctx* ctx, const double* cost, const double* error, int n,
                      int keep, int32_t* chosen, int32_t* rank, double* crowding) {
  Range nvtx_range("gevo_nsga2_select");
  if (keep < 0 || keep > n) return fail(ctx, GEVO_E_ARG, "keep out of range");
  return nsga2_common(ctx, cost, error, n, keep, chosen, rank, crowding, nullptr, nullptr,
                      nullptr);
}


// ---------------------------------------------------------------------------
// Population all-gather over NCCL: NCCL is opened at run
// time (dlopen "libnccl.so.2"), so the library loads on hosts without it and
// only the multi-GPU entry points need it.
// ---------------------------------------------------------------------------
}  // extern "C"

namespace {
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    api.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("cannot open libnccl.so.2: ") + dlerror();
      return;
    }
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy &&
             api.errorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

int nccl_fail(gevo_ctx* c, ncclResult_t r, const char* what) {
  return fail(c, GEVO_E_COMM, std::string(what) + ": " + nccl().errorString(r));
}
}  // namespace

extern "C" {

int gevo_comm_unique_id(void* out, size_t len) {
  if (!out || len < sizeof(ncclUniqueId)) return GEVO_E_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return GEVO_E_COMM;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != ncclSuccess) return GEVO_E_COMM;
  memcpy(out, &id, sizeof(id));
  return GEVO_OK;
}

int gevo_comm_init(gevo_ctx* ctx, int rank, int world, const void* uid, size_t len) {
  if (!ctx) return GEVO_E_ARG;
  if (world < 1 || rank < 0 || rank >= world || !uid || len < sizeof(ncclUniqueId))
    return fail(ctx, GEVO_E_ARG, "bad communicator arguments");
  NcclApi& api = nccl();
  if (!api.ok) return fail(ctx, GEVO_E_COMM, api.why);
  CK(cudaSetDevice(ctx->device));
  gevo_comm_destroy(ctx);
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = api.commInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommInitRank");
  ctx->comm = comm;
  ctx->comm_rank = rank;
  ctx->comm_world = world;
  return GEVO_OK;
}

int gevo_comm_destroy(gevo_ctx* ctx) {
  if (!ctx) return GEVO_E_ARG;
  if (ctx->comm) {
    nccl().commDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ctx->comm_rank = 0;
  ctx->comm_world = 1;
  return GEVO_OK;
}

int gevo_allgather(gevo_ctx* ctx, const void* send, size_t bytes, void* recv) {
  Range nvtx_range("gevo_allgather");
  if (!ctx) return GEVO_E_ARG;
  if (!ctx->comm) return fail(ctx, GEVO_E_STATE, "gevo_comm_init has not been called");
  if ((!send || !recv) && bytes) return fail(ctx, GEVO_E_ARG, "null buffer");
  CK(cudaSetDevice(ctx->device));
  const size_t total = bytes * (size_t)ctx->comm_world;
  if (ctx->gather.ensure(bytes + total + 16, ctx->stream))
    return fail(ctx, GEVO_E_CUDA, "gather alloc failed");
  char* dsend = static_cast<char*>(ctx->gather.p);
  char* drecv = dsend + ((bytes + 15) & ~size_t(15));
  CK(cudaMemcpyAsync(dsend, send, bytes, cudaMemcpyHostToDevice, ctx->stream));
  ncclResult_t r = nccl().allGather(dsend, drecv, bytes, ncclUint8, ctx->comm, ctx->stream);
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclAllGather");
  CK(cudaMemcpyAsync(recv, drecv, total, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return GEVO_OK;
}

}  // extern "C"
