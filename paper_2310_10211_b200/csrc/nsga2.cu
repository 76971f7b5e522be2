// nsga2.cu -- NSGA-II ranking, crowding and survivor selection on the GPU.
//
// Bit-exact restatement of pkg/src/evotir/search.py:
//   dominates          :91-93   (minimisation; equal points never dominate)
//   nondominated_sort  :96-120  (front 0 in index order, later fronts sorted;
//                                 membership = peeling by dominator counts)
//   crowding_distance  :123-140 (per axis: order by (value, index); both ends
//                                 set to inf BEFORE the degenerate-axis skip;
//                                 interior += (next - prev) / span, axis 0
//                                 then axis 1, one IEEE rounding each)
//   select_survivors   :163-179 (whole fronts, then the partial front by
//                                 (-crowding, index))
//   hypervolume        :182-195 and the Archive merge :208-228 (below)
// One CTA of 1024 threads; O(n^2) dominance work spread over the CTA, all
// sorts are counting sorts on unique (key, index) pairs, no float atomics.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include "gevo_exec.cuh"

namespace gevo {

constexpr int kNsThreads = 1024;

__device__ __forceinline__ bool dom(double ac, double ae, double bc, double be) {
  return ac <= bc && ae <= be && (ac < bc || ae < be);
}



// block-wide exclusive scan of 0/1 flags (kNsThreads threads, one item each)
__device__ int block_scan(int v, int* tmp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < (kNsThreads / 32) ? tmp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    tmp[lane] = w;
  }
  __syncthreads();
  int excl = x - v + (warp > 0 ? tmp[warp - 1] : 0);
  *total = tmp[kNsThreads / 32 - 1];
  __syncthreads();
  return excl;
}

__global__ void __launch_bounds__(kNsThreads) nsga2_kernel(NsArgs a) {
  __shared__ int tmp[32];
  __shared__ int s_nf, s_off;
  const int n = a.n;
  const double* C = a.c;
  const double* E = a.e;
  if (a.one_front) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      a.count[j] = 0;
      a.rank[j] = -1;
    }
    __syncthreads();
  }
  // 1. dominator counts
  for (int j = threadIdx.x; j < n && !a.one_front; j += blockDim.x) {
    int cnt = 0;
    const double cj = C[j], ej = E[j];
    for (int i = 0; i < n; ++i) cnt += dom(C[i], E[i], cj, ej);
    a.count[j] = cnt;
    a.rank[j] = -1;
  }
  if (threadIdx.x == 0) { s_nf = 0; s_off = 0; }
  __syncthreads();
  // 2. peel fronts: members in ascending index order
  for (;;) {
    const int f = s_nf;
    const int base = s_off;
    int added = 0;
    for (int j0 = 0; j0 < n; j0 += blockDim.x) {
      int j = j0 + threadIdx.x;
      int flag = (j < n && a.rank[j] == -1 && a.count[j] == 0) ? 1 : 0;
      int total;
      int pos = block_scan(flag, tmp, &total);
      if (flag) a.order[base + added + pos] = j;
      added += total;
    }
    if (added == 0) break;
    for (int k = threadIdx.x; k < added; k += blockDim.x) a.rank[a.order[base + k]] = f;
    __syncthreads();
    // remove this front's dominance from the rest
    for (int j = threadIdx.x; j < n && !a.one_front; j += blockDim.x) {
      if (a.rank[j] != -1) continue;
      int d = 0;
      const double cj = C[j], ej = E[j];
      for (int k = 0; k < added; ++k) {
        int i = a.order[base + k];
        d += dom(C[i], E[i], cj, ej);
      }
      a.count[j] -= d;
    }
    if (threadIdx.x == 0) {
      a.fstart[f] = base;
      s_nf = f + 1;
      s_off = base + added;
    }
    __syncthreads();
  }
  const int nf = s_nf;
  if (threadIdx.x == 0) { a.fstart[nf] = n; *a.nfronts = nf; }
  __syncthreads();
  // 3. front-local orders along each axis by (value, index)
  for (int k = threadIdx.x; k < n; k += blockDim.x) a.front_of_pos[k] = a.rank[a.order[k]];
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const int f = a.rank[p];
    const int fs = a.fstart[f], fe = a.fstart[f + 1];
    int p0 = 0, p1 = 0;
    for (int k = fs; k < fe; ++k) {
      int q = a.order[k];
      p0 += (C[q] < C[p]) || (C[q] == C[p] && q < p);
      p1 += (E[q] < E[p]) || (E[q] == E[p] && q < p);
    }
    a.ord0[fs + p0] = p;
    a.ord1[fs + p1] = p;
  }
  __syncthreads();
  // 4. crowding, replaying the reference's operation order per point
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int f = a.front_of_pos[k];
    const int fs = a.fstart[f], fe = a.fstart[f + 1];
    const int len = fe - fs;
    if (len <= 2) { a.crowd[a.ord0[k]] = INFINITY; continue; }
    // the point at axis-0 position k
    const int p = a.ord0[k];
    double d = 0.0;
    {
      const double lo = C[a.ord0[fs]], hi = C[a.ord0[fe - 1]];
      if (k == fs || k == fe - 1) d = INFINITY;
      else if (!(hi == lo || hi == INFINITY || lo == INFINITY))
        d = __dadd_rn(d, __ddiv_rn(__dsub_rn(C[a.ord0[k + 1]], C[a.ord0[k - 1]]),
                                   __dsub_rn(hi, lo)));
    }
    // its axis-1 position
    int k1 = fs;
    while (a.ord1[k1] != p) ++k1;
    {
      const double lo = E[a.ord1[fs]], hi = E[a.ord1[fe - 1]];
      if (k1 == fs || k1 == fe - 1) d = INFINITY;
      else if (!(hi == lo || hi == INFINITY || lo == INFINITY))
        d = __dadd_rn(d, __ddiv_rn(__dsub_rn(E[a.ord1[k1 + 1]], E[a.ord1[k1 - 1]]),
                                   __dsub_rn(hi, lo)));
    }
    a.crowd[p] = d;
  }
  __syncthreads();
  // 5. survivors
  if (a.chosen == nullptr) return;
  const int keep = a.keep;
  int fstar = 0, taken = 0;
  while (fstar < nf && taken + (a.fstart[fstar + 1] - a.fstart[fstar]) <= keep) {
    taken += a.fstart[fstar + 1] - a.fstart[fstar];
    ++fstar;
  }
  for (int k = threadIdx.x; k < taken; k += blockDim.x) a.chosen[k] = a.order[k];
  if (fstar < nf && taken < keep) {
    const int fs = a.fstart[fstar], fe = a.fstart[fstar + 1];
    for (int k = fs + threadIdx.x; k < fe; k += blockDim.x) {
      const int p = a.order[k];
      const double dp = a.crowd[p];
      int pos = 0;
      for (int m = fs; m < fe; ++m) {
        const int q = a.order[m];
        const double dq = a.crowd[q];
        pos += (dq > dp) || (dq == dp && q < p);
      }
      if (taken + pos < keep) a.chosen[taken + pos] = p;
    }
  }
}

void launch_nsga2(const NsArgs& a, cudaStream_t st) {
  nsga2_kernel<<<1, kNsThreads, 0, st>>>(a);
}

// ---------------------------------------------------------------------------
// Archive merge (search.py:208-228, batched).  Points 0..n_old-1 are the
// archive entries in order, the rest one batch of valid offers in offer
// order whose keys are all new (the host splits batches at key repeats).
// Offering them one by one keeps exactly the points that nothing in the
// list dominates and that no EARLIER point equals (an equal or dominating
// point reaching the archive first blocks it; anything that later evicts
// that blocker dominates it too), in list order -- which is the order
// `kept + [new]` leaves them in.  O(n^2) compares over the CTA, order kept
// by a block scan.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNsThreads) archive_merge_kernel(ArchArgs a) {
  __shared__ int tmp[32];
  const int n = a.n;
  const double* C = a.c;
  const double* E = a.e;
  int base = 0;
  for (int j0 = 0; j0 < n; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    int keep = 0;
    if (j < n) {
      const double cj = C[j], ej = E[j];
      keep = 1;
      for (int i = 0; i < n; ++i) {
        const double ci = C[i], ei = E[i];
        if (dom(ci, ei, cj, ej) || (i < j && ci == cj && ei == ej)) { keep = 0; break; }
      }
    }
    int total;
    const int pos = block_scan(keep, tmp, &total);
    if (keep) a.keep[base + pos] = j;
    base += total;
  }
  if (threadIdx.x == 0) *a.n_keep = base;
}

// block-wide exclusive running minimum (kNsThreads threads, one item each);
// min is exact, so any association gives the sequential result
__device__ double block_min_scan(double v, double init, double* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x = v;
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = fmin(x, y);
  }
  if (lane == 31) tmp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    double w = lane < (kNsThreads / 32) ? tmp[lane] : INFINITY;
    for (int o = 1; o < 32; o <<= 1) {
      double y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = fmin(w, y);
    }
    tmp[lane] = w;
  }
  __syncthreads();
  double excl = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) excl = INFINITY;
  if (warp > 0) excl = fmin(excl, tmp[warp - 1]);
  excl = fmin(excl, init);
  __syncthreads();
  return excl;
}

// ---------------------------------------------------------------------------
// Hypervolume (search.py:182-195).  The points strictly inside the corner
// are placed in (cost, error) order by counting (ties by index, as the
// stable sort leaves them).  The running ceiling before each point is an
// exclusive min-scan, and each step's area is one IEEE subtract/subtract/
// multiply.  One thread then adds the stepping points' areas in sweep order,
// as the reference's `total +=` does.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNsThreads) hypervolume_kernel(HvArgs a) {
  __shared__ int tmp[32];
  __shared__ double dtmp[32];
  const int n = a.n;
  const double* C = a.c;
  const double* E = a.e;
  const double r0 = a.ref_c, r1 = a.ref_e;
  int m = 0;
  // 1. inside points, counted into sweep positions
  for (int j0 = 0; j0 < n; j0 += blockDim.x) {
    const int p = j0 + threadIdx.x;
    int in = 0;
    double cp = 0, ep = 0;
    if (p < n) {
      cp = C[p];
      ep = E[p];
      in = cp < r0 && ep < r1;
    }
    int total;
    block_scan(in, tmp, &total);
    m += total;
    if (!in) continue;
    int pos = 0;
    for (int q = 0; q < n; ++q) {
      const double cq = C[q], eq = E[q];
      if (!(cq < r0 && eq < r1)) continue;
      pos += cq < cp || (cq == cp && (eq < ep || (eq == ep && q < p)));
    }
    a.sc[pos] = cp;
    a.se[pos] = ep;
  }
  __syncthreads();
  // 2. ceiling before each position and the step areas
  double ceil_carry = r1;
  for (int k0 = 0; k0 < m; k0 += blockDim.x) {
    const int k = k0 + threadIdx.x;
    const double e = k < m ? a.se[k] : INFINITY;
    const double ceil = block_min_scan(e, ceil_carry, dtmp);
    if (k < m) {
      const bool step = e < ceil;
      a.area[k] = step ? __dmul_rn(__dsub_rn(r0, a.sc[k]), __dsub_rn(ceil, e)) : 0.0;
      a.flag[k] = step;
    }
    // carry = min over this chunk, via the last thread's inclusive value
    if (threadIdx.x == blockDim.x - 1) dtmp[0] = fmin(ceil, e);
    __syncthreads();
    ceil_carry = dtmp[0];
    __syncthreads();
  }
  // 3. the sequential sum
  if (threadIdx.x == 0) {
    double total = 0.0;
    for (int k = 0; k < m; ++k)
      if (a.flag[k]) total = __dadd_rn(total, a.area[k]);
    *a.out = total;
  }
}

void launch_archive_merge(const ArchArgs& a, cudaStream_t st) {
  archive_merge_kernel<<<1, kNsThreads, 0, st>>>(a);
}

void launch_hypervolume(const HvArgs& a, cudaStream_t st) {
  hypervolume_kernel<<<1, kNsThreads, 0, st>>>(a);
}

}  // namespace gevo
