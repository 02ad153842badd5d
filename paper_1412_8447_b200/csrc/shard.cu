// shard.cu -- column-sharded CPQR across GPUs (one process per GPU) and the
// NCCL plumbing of the column-sharded entry points (SURVEY.md section 8e,
// north_star: "each GPU computes its slice of the norm/pivot updates, NCCL
// selects the global pivot, the Householder reflector is broadcast").
//
// Semantics are cpqr.hpp:48-85 exactly as the single-GPU kernels implement
// them; only the owner of a column changes.  Rank g owns the columns
// [off_g, off_g + n_g) of the short-wide working matrix (the sketch Y, or C^T
// for the row ID).  Per step s, ONE collective carries both the pivot choice
// and the reflector:
//
//   every rank stages its local candidate (largest downdated norm^2 among its
//   active columns, ties -> lowest logical position; header + the column)
//   -> ncclAllGather of the N candidates
//   -> every rank picks the same winner from the same bytes (max norm^2, then
//      lowest logical position: the reference's strict '>' first-maximum
//      scan), builds the Householder reflector from the winner's column with
//      a fixed-order reduction (bitwise identical on every rank), applies it
//      to its own columns, downdates / recomputes their norms, relabels the
//      column at logical position s (the reference's swap), and stages its
//      next candidate.
//
// No rank ever holds the whole working matrix.  Swaps are logical (the
// single-GPU panel kernel does the same): a column keeps its slot and carries
// its logical position; the full permutation and the top k rows of the R
// factor in logical order are assembled once at the end by a scatter and an
// all-reduce-sum with exactly one non-zero contribution per entry (exact).
//
// Every column's arithmetic is independent of which rank or CTA owns it, so
// pivots, R and the coefficients are bitwise identical for every shard count
// (tested: N = 1 through the NCCL path on the GPU, N = 2 over gloo for the
// host protocol in tests/test_distributed.py).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace lrb {

// ---------------------------------------------------------------- NCCL (run-time bound)
// The library does not link NCCL: the process's libnccl.so.2 (torch's bundled
// one when torch is loaded, else the system's) is bound on first use.
namespace {
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      api.error = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather || !api.AllReduce ||
        !api.GetErrorString)
      api.error = "libnccl.so.2 lacks a required symbol";
  });
  if (!api.error.empty()) throw NcclError(api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl_api().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id.internal) == 128, "NCCL unique id size");
  memcpy(out, id.internal, 128);
}

void* nccl_comm_init(const unsigned char id[128], int nranks, int rank) {
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ncclComm_t comm = nullptr;
  nccl_check(nccl_api().CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  return comm;
}

void nccl_comm_destroy(void* comm) {
  if (comm) nccl_api().CommDestroy(static_cast<ncclComm_t>(comm));
}

// Without a communicator (a single unsharded rank) the collectives are local
// copies; with one attached they always go through NCCL, also for 1 rank.
void ShardComm::all_gather_bytes(const void* send, void* recv, size_t bytes, cudaStream_t st) const {
  if (!comm) {
    if (send != recv) LRB_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, st));
    return;
  }
  nccl_check(nccl_api().AllGather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(comm), st),
             "ncclAllGather");
}

void ShardComm::all_reduce_sum(double* buf, size_t count, cudaStream_t st) const {
  if (!comm || count == 0) return;
  nccl_check(nccl_api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), st),
             "ncclAllReduce");
}

void ShardComm::all_reduce_sum(int64_t* buf, size_t count, cudaStream_t st) const {
  if (!comm || count == 0) return;
  nccl_check(nccl_api().AllReduce(buf, buf, count, ncclInt64, ncclSum, static_cast<ncclComm_t>(comm), st),
             "ncclAllReduce");
}

void ShardComm::all_reduce_max(double* buf, size_t count, cudaStream_t st) const {
  if (!comm || count == 0) return;
  nccl_check(nccl_api().AllReduce(buf, buf, count, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm), st),
             "ncclAllReduce");
}

// ---------------------------------------------------------------- sharded CPQR kernels
namespace {

constexpr int kShT = 256;          // threads per CTA
constexpr int kShW = kShT / 32;    // warps per CTA
constexpr int kShHdr = 4;          // candidate header: norm^2, logical position, global column, valid
constexpr int kShMaxRanks = 64;

__device__ __forceinline__ bool sh_better(double v1, long long p1, double v2, long long p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

// fixed-order CTA sum, every thread gets the result
__device__ double sh_cta_sum(double x, double* sh) {
  x = warp_sum(x);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[w] = x;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < kShW; ++i) t += sh[i];
  __syncthreads();
  return t;
}

struct ShardArgs {
  double* W;          // m x n_loc, ld (working matrix, in place)
  int64_t ld, m, n_loc, off, k;
  double* nrm;        // running norm^2 (-inf: pivoted)
  double* nrmx;       // norm^2 at the last exact evaluation
  long long* pos;     // logical position of each owned column
  double* part_v;     // per-CTA argmax partials
  long long* part_p;  // (logical position << 32) | local column
  unsigned int* counter;
  double* cand;        // this rank's candidate: header + m doubles
  const double* cand_all;  // gathered candidates [nranks][kShHdr + m]
  int nranks;
  double* rdiag;       // [k] diagonal of R at each step (sign fix)
  long long* rpos;     // [k] logical position the winner held
  int* flags;          // [0]: non-finite input
  unsigned long long* recomputes;
};

// Per-CTA argmax (value, key) -> partials; the last CTA to finish reduces them
// in CTA order and stages the rank's candidate (header + the column).
__device__ void stage_candidate(const ShardArgs& a, double bv, long long bp) {
  __shared__ double sv[kShW];
  __shared__ long long sp[kShW];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long op = __shfl_xor_sync(0xffffffffu, bp, o);
    if (sh_better(ov, op, bv, bp)) { bv = ov; bp = op; }
  }
  if (lane == 0) { sv[w] = bv; sp[w] = bp; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double cv = sv[0];
    long long cp = sp[0];
    for (int i = 1; i < kShW; ++i)
      if (sh_better(sv[i], sp[i], cv, cp)) { cv = sv[i]; cp = sp[i]; }
    a.part_v[blockIdx.x] = cv;
    a.part_p[blockIdx.x] = cp;
    __threadfence();  // this CTA's column updates and partial before the count
    last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double gv;
  __shared__ long long gp;
  if (threadIdx.x == 0) {
    double cv = __ldcg(a.part_v);
    long long cp = __ldcg(a.part_p);
    for (unsigned i = 1; i < gridDim.x; ++i) {
      const double v = __ldcg(a.part_v + i);
      const long long p = __ldcg(a.part_p + i);
      if (sh_better(v, p, cv, cp)) { cv = v; cp = p; }
    }
    gv = cv;
    gp = cp;
    *a.counter = 0;  // ready for the next launch (stream order)
  }
  __syncthreads();
  const bool valid = gv != -INFINITY && gp != LLONG_MAX;
  const int64_t j = valid ? (gp & 0xffffffffll) : 0;
  if (threadIdx.x == 0) {
    a.cand[0] = valid ? gv : -INFINITY;
    a.cand[1] = valid ? (double)(gp >> 32) : 0.0;
    a.cand[2] = valid ? (double)(a.off + j) : -1.0;
    a.cand[3] = valid ? 1.0 : 0.0;
  }
  if (valid)
    for (int64_t i = threadIdx.x; i < a.m; i += blockDim.x) a.cand[kShHdr + i] = __ldcg(a.W + j * a.ld + i);
}

__global__ void __launch_bounds__(kShT) shard_init_kernel(ShardArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double bv = -INFINITY;
  long long bp = LLONG_MAX;
  for (int64_t j = gw; j < a.n_loc; j += nw) {
    const double* col = a.W + j * a.ld;
    double acc = 0.0;
    bool fin = true;
    for (int64_t i = lane; i < a.m; i += 32) {
      const double x = col[i];
      fin &= isfinite(x);
      acc += x * x;
    }
    acc = warp_sum(acc);
    if (!__all_sync(0xffffffffu, fin) && lane == 0) atomicOr(a.flags, 1);
    const long long p = a.off + j;
    if (lane == 0) {
      a.nrm[j] = acc;
      a.nrmx[j] = acc;
      a.pos[j] = p;
    }
    const long long key = (p << 32) | j;
    if (sh_better(acc, key, bv, bp)) { bv = acc; bp = key; }
  }
  stage_candidate(a, bv, bp);
}

// Step s: winner from the gathered candidates, reflector, apply to the owned
// columns, downdate / recompute, relabel, next candidate.
__global__ void __launch_bounds__(kShT) shard_step_kernel(ShardArgs a, int64_t s) {
  extern __shared__ double vv[];  // the winner's reflector, rows s..m-1
  __shared__ double red[kShW];
  __shared__ int win;
  const int lane = threadIdx.x & 31;
  const int64_t m = a.m;
  const int64_t cand_sz = kShHdr + m;
  if (threadIdx.x == 0) {
    int w = -1;
    double bv = -INFINITY;
    long long bp = LLONG_MAX;
    for (int r = 0; r < a.nranks; ++r) {
      const double* h = a.cand_all + (int64_t)r * cand_sz;
      if (h[3] == 0.0) continue;
      const double v = h[0];
      const long long p = (long long)h[1];
      if (w < 0 || sh_better(v, p, bv, bp)) { w = r; bv = v; bp = p; }
    }
    win = w;
  }
  __syncthreads();
  if (win < 0) return;  // fewer active columns than steps: nothing left to factor
  const double* wc = a.cand_all + (int64_t)win * cand_sz;
  const long long wpos = (long long)wc[1];
  const long long wcol = (long long)wc[2];
  // reflector (cpqr.hpp:59-66): alpha = x_s, beta = -sign(alpha)|x|, tau = (beta - alpha)/beta,
  // v = x / (alpha - beta) below the diagonal
  double cn2 = 0.0;
  for (int64_t i = s + threadIdx.x; i < m; i += blockDim.x) {
    const double x = wc[kShHdr + i];
    vv[i - s] = x;
    cn2 += x * x;
  }
  cn2 = sh_cta_sum(cn2, red);
  const double alpha = vv[0];
  const double colnorm = sqrt(cn2);
  const bool apply = colnorm > 0.0;
  const double beta = apply ? (alpha >= 0.0 ? -colnorm : colnorm) : alpha;
  const double tau = apply ? (beta - alpha) / beta : 0.0;
  if (apply) {
    const double scale = alpha - beta;
    for (int64_t i = s + 1 + threadIdx.x; i < m; i += blockDim.x) vv[i - s] = vv[i - s] / scale;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    vv[0] = 1.0;
    if (blockIdx.x == 0) {
      a.rdiag[s] = beta;
      a.rpos[s] = wpos;
    }
  }
  __syncthreads();

  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double bv = -INFINITY;
  long long bp = LLONG_MAX;
  unsigned long long rec = 0;
  for (int64_t j = gw; j < a.n_loc; j += nw) {
    const double nr0 = a.nrm[j];
    if (nr0 == -INFINITY) continue;  // pivoted at an earlier step
    double* col = a.W + j * a.ld;
    if (a.off + j == wcol) {  // the pivot: keep its reflector (R diagonal + v below)
      if (apply)
        for (int64_t i = s + lane; i < m; i += 32) col[i] = (i == s) ? beta : vv[i - s];
      if (lane == 0) {
        a.nrm[j] = -INFINITY;
        a.pos[j] = s;
      }
      continue;
    }
    long long p = a.pos[j];
    if (p == s) p = wpos;  // the reference's swap: the column at position s takes the pivot's position
    if (apply) {
      double dot = 0.0;
      for (int64_t i = s + lane; i < m; i += 32) dot += col[i] * vv[i - s];
      dot = warp_sum(dot);
      for (int64_t i = s + lane; i < m; i += 32) col[i] -= (tau * vv[i - s]) * dot;
    }
    __syncwarp();
    const double xs = col[s];
    double nr = nr0 - xs * xs;
    double nx = a.nrmx[j];
    if (nr < 1e-6 * nx) {  // cpqr.hpp:78-84: exact recompute below the threshold
      double acc = 0.0;
      for (int64_t i = s + 1 + lane; i < m; i += 32) acc += col[i] * col[i];
      nr = warp_sum(acc);
      nx = nr;
      ++rec;
    }
    if (lane == 0) {
      a.nrm[j] = nr;
      a.nrmx[j] = nx;
      a.pos[j] = p;
    }
    const long long key = (p << 32) | j;
    if (sh_better(nr, key, bv, bp)) { bv = nr; bp = key; }
  }
  if (lane == 0 && rec) atomicAdd(a.recomputes, rec);
  stage_candidate(a, bv, bp);
}

// Assembly: perm[pos] = global column; S(0:krows, pos) = top rows of each owned
// column with the sign fix of cpqr.hpp:105-112 (rows whose R diagonal is
// negative are negated; a pivot column's entries below its diagonal are the
// reflector and read as zero).  Both targets are zeroed by the caller and
// all-reduce-summed afterwards.
__global__ void shard_scatter_kernel(const double* __restrict__ W, int64_t ld, int64_t n_loc, int64_t off,
                                     int64_t steps, int64_t krows, const long long* __restrict__ pos,
                                     const double* __restrict__ rdiag, int64_t* __restrict__ perm,
                                     double* __restrict__ S, int64_t lds) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = gw; j < n_loc; j += nw) {
    const long long p = pos[j];
    if (lane == 0) perm[p] = off + j;
    for (int64_t i = lane; i < krows; i += 32) {
      double v = (p < steps && i > p) ? 0.0 : W[j * ld + i];
      if (rdiag[i] < 0.0) v = -v;
      S[p * lds + i] = v;
    }
  }
}

int shard_grid(int64_t n_loc) {
  const int64_t need = (n_loc + kShW - 1) / kShW;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, 4 * (int64_t)num_sms()));
}


__global__ void owned_index_kernel(const int64_t* perm, int64_t k, int64_t off, int64_t n_loc, int64_t* idx) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= k) return;
  const int64_t g = perm[l];
  idx[l] = (g >= off && g < off + n_loc) ? g - off : -1;
}
__global__ void inverse_perm_kernel(const int64_t* perm, int64_t n, int64_t* inv) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < n) inv[perm[l]] = l;
}
// B (k x n_loc, ld k): column j = the row of basis() (id.hpp:21-30) of global
// column off + j: e_l for logical position l < k, else coeff(:, l - k)
__global__ void basis_rows_kernel(const int64_t* inv, int64_t off, int64_t n_loc, int64_t k, const double* coeff,
                                  int64_t ldc, double* B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * n_loc) return;
  const int64_t j = e / k, i = e % k;
  const int64_t l = inv[off + j];
  B[j * k + i] = l < k ? (i == l ? 1.0 : 0.0) : coeff[(l - k) * ldc + i];
}

}  // namespace

void owned_index(const int64_t* perm, int64_t k, int64_t off, int64_t n_loc, int64_t* idx, cudaStream_t st) {
  owned_index_kernel<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(perm, k, off, n_loc, idx);
  LRB_CHECK_LAUNCH();
}
void inverse_perm(const int64_t* perm, int64_t n, int64_t* inv, cudaStream_t st) {
  inverse_perm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(perm, n, inv);
  LRB_CHECK_LAUNCH();
}
void basis_rows(const int64_t* inv, int64_t off, int64_t n_loc, int64_t k, const double* coeff, int64_t ldc,
                double* B, cudaStream_t st) {
  basis_rows_kernel<<<(unsigned)((k * n_loc + 255) / 256), 256, 0, st>>>(inv, off, n_loc, k, coeff, ldc, B);
  LRB_CHECK_LAUNCH();
}

// Device state of one shard of the sharded CPQR, carved from `base`.
namespace {
struct ShardState {
  ShardArgs a{};
  int G = 1;
  double* cand_all = nullptr;
};

size_t shard_state_bytes(int64_t m, int64_t n_loc, int64_t k, int nranks, int G) {
  const size_t nl = (size_t)std::max<int64_t>(n_loc, 1);
  const int64_t cand_sz = kShHdr + m;
  return sizeof(double) * (2 * nl + G + (size_t)cand_sz * (1 + nranks) + k) + sizeof(long long) * (nl + G + k) +
         16 * 16;
}

ShardState shard_state(uint8_t* base, int64_t m, int64_t n_loc, int64_t off, double* W, int64_t ld, int64_t k,
                       int nranks, double* cand_all_shared, int* d_flags, long long* d_recomputes) {
  ShardState st;
  st.G = shard_grid(std::max<int64_t>(n_loc, 1));
  const size_t nl = (size_t)std::max<int64_t>(n_loc, 1);
  const int64_t cand_sz = kShHdr + m;
  auto take = [&](size_t b) {
    uint8_t* p = base;
    base += (b + 15) / 16 * 16;
    return p;
  };
  ShardArgs& a = st.a;
  a.W = W;
  a.ld = ld;
  a.m = m;
  a.n_loc = n_loc;
  a.off = off;
  a.k = k;
  a.nrm = reinterpret_cast<double*>(take(sizeof(double) * nl));
  a.nrmx = reinterpret_cast<double*>(take(sizeof(double) * nl));
  a.pos = reinterpret_cast<long long*>(take(sizeof(long long) * nl));
  a.part_v = reinterpret_cast<double*>(take(sizeof(double) * st.G));
  a.part_p = reinterpret_cast<long long*>(take(sizeof(long long) * st.G));
  a.cand = reinterpret_cast<double*>(take(sizeof(double) * cand_sz));
  double* own_all = reinterpret_cast<double*>(take(sizeof(double) * cand_sz * nranks));
  st.cand_all = cand_all_shared ? cand_all_shared : own_all;
  a.cand_all = st.cand_all;
  a.nranks = nranks;
  a.rdiag = reinterpret_cast<double*>(take(sizeof(double) * k));
  a.rpos = reinterpret_cast<long long*>(take(sizeof(long long) * k));
  a.counter = reinterpret_cast<unsigned int*>(take(16));
  a.flags = d_flags;
  a.recomputes = reinterpret_cast<unsigned long long*>(d_recomputes);
  return st;
}

void shard_begin(const ShardState& st, cudaStream_t s) {
  LRB_CUDA(cudaMemsetAsync(st.a.counter, 0, 16, s));
  if (st.a.n_loc > 0) {
    shard_init_kernel<<<st.G, kShT, 0, s>>>(st.a);
    LRB_CHECK_LAUNCH();
  } else {  // an empty shard still takes part in every exchange
    const double empty_hdr[kShHdr] = {-INFINITY, 0.0, -1.0, 0.0};
    LRB_CUDA(cudaMemcpyAsync(st.a.cand, empty_hdr, sizeof(empty_hdr), cudaMemcpyHostToDevice, s));
    LRB_CUDA(cudaStreamSynchronize(s));  // empty_hdr is a host stack array
  }
}

void shard_step(const ShardState& st, int64_t step, cudaStream_t s) {
  shard_step_kernel<<<st.G, kShT, sizeof(double) * (size_t)st.a.m, s>>>(st.a, step);
  LRB_CHECK_LAUNCH();
}

void shard_scatter(const ShardState& st, int64_t* perm, double* S, int64_t lds, int64_t krows, cudaStream_t s) {
  if (st.a.n_loc > 0) {
    shard_scatter_kernel<<<st.G, kShT, 0, s>>>(st.a.W, st.a.ld, st.a.n_loc, st.a.off, st.a.k, krows, st.a.pos,
                                               st.a.rdiag, perm, S, lds);
    LRB_CHECK_LAUNCH();
  }
}
}  // namespace

// Column-sharded CPQR of the local block W (m x n_loc, ld; overwritten) for
// `steps` steps; outputs replicated on every rank: perm (n_total) and the
// sign-fixed top `krows` rows of R in logical column order (S, ld lds).
void cpqr_sharded(Workspace& ws, const ShardComm& comm, int64_t m, int64_t n_loc, int64_t off, int64_t n_total,
                  double* W, int64_t ld, int64_t steps, int64_t krows, int64_t* perm, double* S, int64_t lds,
                  int* d_flags, long long* d_recomputes, cudaStream_t st) {
  if (comm.nranks > kShMaxRanks) throw std::runtime_error("cpqr_sharded: too many ranks");
  const int G = shard_grid(std::max<int64_t>(n_loc, 1));
  uint8_t* base = static_cast<uint8_t*>(ws.get(WsSlot::kShard, shard_state_bytes(m, n_loc, steps, comm.nranks, G)));
  const ShardState sh = shard_state(base, m, n_loc, off, W, ld, steps, comm.nranks, nullptr, d_flags, d_recomputes);
  shard_begin(sh, st);
  for (int64_t s = 0; s < steps; ++s) {
    comm.all_gather_bytes(sh.a.cand, sh.cand_all, sizeof(double) * (kShHdr + m), st);
    shard_step(sh, s, st);
  }
  LRB_CUDA(cudaMemsetAsync(perm, 0, sizeof(int64_t) * n_total, st));
  LRB_CUDA(cudaMemsetAsync(S, 0, sizeof(double) * (size_t)lds * n_total, st));
  shard_scatter(sh, perm, S, lds, krows, st);
  comm.all_reduce_sum(perm, (size_t)n_total, st);
  comm.all_reduce_sum(S, (size_t)lds * n_total, st);
}

// The same protocol for `nshards` column blocks of ONE matrix in one process
// (a test vehicle for the multi-rank logic on a single GPU): each step the
// shards' candidates are copied into one gathered buffer, then every shard's
// step kernel runs -- in sequence on one stream, no kernel waits on another.
void cpqr_sharded_emulated(Workspace& ws, int nshards, int64_t m, int64_t n, double* W, int64_t ld, int64_t steps,
                           int64_t krows, int64_t* perm, double* S, int64_t lds, int* d_flags,
                           long long* d_recomputes, cudaStream_t st) {
  if (nshards < 1 || nshards > kShMaxRanks) throw std::runtime_error("cpqr_sharded_emulated: bad shard count");
  const int64_t cand_sz = kShHdr + m;
  std::vector<ShardState> sh;
  std::vector<size_t> offs;
  size_t total = 0;
  for (int r = 0; r < nshards; ++r) {
    const int64_t lo = n * r / nshards, nl = n * (r + 1) / nshards - lo;
    offs.push_back(total);
    total += shard_state_bytes(m, nl, steps, nshards, shard_grid(std::max<int64_t>(nl, 1)));
  }
  total += sizeof(double) * cand_sz * nshards + 16;
  uint8_t* base = static_cast<uint8_t*>(ws.get(WsSlot::kShard, total));
  double* cand_all = reinterpret_cast<double*>(base + (total - sizeof(double) * cand_sz * nshards - 16));
  for (int r = 0; r < nshards; ++r) {
    const int64_t lo = n * r / nshards, nl = n * (r + 1) / nshards - lo;
    sh.push_back(shard_state(base + offs[r], m, nl, lo, W + lo * ld, ld, steps, nshards, cand_all, d_flags,
                             d_recomputes));
    shard_begin(sh.back(), st);
  }
  for (int64_t s = 0; s < steps; ++s) {
    for (int r = 0; r < nshards; ++r)
      LRB_CUDA(cudaMemcpyAsync(cand_all + r * cand_sz, sh[r].a.cand, sizeof(double) * cand_sz,
                               cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < nshards; ++r) shard_step(sh[r], s, st);
  }
  LRB_CUDA(cudaMemsetAsync(perm, 0, sizeof(int64_t) * n, st));
  LRB_CUDA(cudaMemsetAsync(S, 0, sizeof(double) * (size_t)lds * n, st));
  for (int r = 0; r < nshards; ++r) shard_scatter(sh[r], perm, S, lds, krows, st);
}

}  // namespace lrb
