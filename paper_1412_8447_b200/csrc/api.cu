// api.cu -- the C ABI (include/lowrank_b200.h) and the host orchestration of
// the ID / CUR pipeline over the sm_100a kernels.  Every entry point mirrors
// one template of the reference library (cited per function) in argument
// meaning, validation order and error class; the arithmetic runs on the GPU
// only (no CPU fallback: a missing device is LR_ECUDA).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <optional>
#include <vector>

#include <cuda.h>

#include "../../include/lowrank_b200.h"
#include "common.cuh"
#include "kernels.h"

using namespace lrb;

namespace {

thread_local std::string g_err;
thread_local int64_t g_sing = -1;

struct LrError {
  int code;
  std::string msg;
  int64_t index;
};
[[noreturn]] void fail(int code, const std::string& msg, int64_t index = -1) { throw LrError{code, msg, index}; }

void arena_close();

template <typename F>
int guard(F&& f) {
  struct Close {
    ~Close() { arena_close(); }
  } close_arena;
  try {
    f();
    return LR_OK;
  } catch (const LrError& e) {
    g_err = e.msg;
    if (e.code == LR_ESINGULAR) g_sing = e.index;
    return e.code;
  } catch (const CudaError& e) {
    g_err = e.what();
    return LR_ECUDA;
  } catch (const NcclError& e) {
    g_err = e.what();
    return LR_ENCCL;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return LR_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LR_ERUNTIME;
  }
}

inline int64_t even(int64_t x) { return x + (x & 1); }

// Per-context call arena: every DBuf of a public call on the context's stream
// is a bump allocation in one grow-only device block, reset at the next call
// (stream order makes the reuse safe; switching streams synchronises the old
// one).  Re-allocating multi-GB temporaries from the stream-ordered pool every
// call fragmented it and made some calls map fresh memory (~100 ms).
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0, overflow = 0, want = 0;
  cudaStream_t st = nullptr;
  bool active = false;
};
thread_local Arena* tl_arena = nullptr;

// stream-ordered device buffer: from the call arena, else the default pool
template <typename T>
struct DBuf {
  T* p = nullptr;
  cudaStream_t st = nullptr;
  bool from_arena = false;
  DBuf() = default;
  DBuf(size_t n, cudaStream_t s) : st(s) {
    const size_t bytes = sizeof(T) * std::max<size_t>(n, 1);
    Arena* ar = tl_arena;
    if (ar && ar->active && s == ar->st) {
      const size_t off = (ar->used + 255) & ~size_t(255);
      if (off + bytes <= ar->cap) {
        p = reinterpret_cast<T*>(ar->base + off);
        ar->used = off + bytes;
        from_arena = true;
        return;
      }
      ar->overflow += bytes + 256;  // grow the arena before the next call
    }
    LRB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, s));
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), st(o.st), from_arena(o.from_arena) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    reset();
    p = o.p;
    st = o.st;
    from_arena = o.from_arena;
    o.p = nullptr;
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() {
    if (p && !from_arena) cudaFreeAsync(p, st);
    p = nullptr;
  }
  operator T*() const { return p; }
};

}  // namespace

struct lr_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t st = nullptr;
  Workspace ws;
  int* h_flags = nullptr;  // pinned
  double* h_scal = nullptr;
  long long* h_ll = nullptr;
  lr_stats stats{};
  // stage timing with CUDA events on the context stream (lr_ctx_enable_timing)
  bool timing = false;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  std::vector<std::pair<std::string, double>> stage_ms;
  std::vector<std::pair<std::string, long long>> stage_count;
  // contraction engine for the two A-sized GEMMs (lr_ctx_set_gemm_mode)
  int gemm_mode = LR_GEMM_DMMA;
  // Ozaki residue planes of A, kept for the duration of one CUR call so the
  // sketch and the A^T Q contraction split A once (OzakiScope)
  bool oz_cache_on = false;
  bool oz_pinned = false;  // lr_ctx_cache_operand: the cache outlives single calls
  const double* pin_src = nullptr;
  int64_t pin_K = 0, pin_cols = 0, pin_ld = 0;
  const double* oz_src = nullptr;
  int64_t oz_K = 0, oz_cols = 0, oz_ld = 0;
  lrb::OzakiOperand oz_op;
  // auxiliary streams of the host-pointer entry points: host->device upload
  // of A (overlapped with the sketch) and device->host of finished factors
  cudaStream_t up_st = nullptr, down_st = nullptr;
  cudaStream_t side_st = nullptr;  // second chain of independent small factorizations (cholqr2_pair)
  Workspace ws_side;               // its scratch (split-K partials, Cholesky panels)
  Arena arena;
  // two disjoint SM partitions (green contexts) for the concurrent CUR tail
  // SMs of the concurrent CUR tail's row-ID partition (lr_ctx_set_concurrent_tail):
  // -1 automatic, 0 sequential tail, > 0 that many
  int tail_sms = -1;
  struct SmSplit {
    bool tried = false, ok = false;
    int want = 0;        // partition size the green contexts were built for
    int n1 = 0, n2 = 0;  // SMs of partition 1 (row ID chain) / 2 (A^T Q_c chain)
    CUgreenCtx g1 = nullptr, g2 = nullptr;
    CUstream s1 = nullptr, s2 = nullptr;
  } split;
  // communicator of the column-sharded entry points (lr_ctx_attach_comm)
  lrb::ShardComm comm;
  // > 0 (no communicator): the sharded CPQRs run as that many column blocks in
  // this process (lr_ctx_set_shard_emulation, a single-GPU test vehicle)
  int emu_shards = 0;
};

namespace {

// Small device -> host reads of control values (flags, norms) go through a
// one-warp kernel into the context's mapped pinned words instead of
// cudaMemcpyAsync: a copy would queue on the copy engine behind the
// megabyte-sized factor downloads in flight on the download stream.
void d2h_mapped(lr_ctx* c, void* h, const void* d, size_t bytes) { copy_bytes_mapped(h, d, bytes, c->st); }

// Close the interval since the previous mark and label it `stage`.
void mark(lr_ctx* c, const char* stage) {
  if (!c->timing) return;
  static const bool host_trace = getenv("LRB_MARK_HOST") != nullptr;
  if (host_trace) {  // host-side timeline of the marks (diagnostic)
    static const auto h0 = std::chrono::steady_clock::now();
    fprintf(stderr, "mark %-16s host %10.3f ms\n", stage,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
  }
  cudaEvent_t e;
  LRB_CUDA(cudaEventCreate(&e));
  LRB_CUDA(cudaEventRecord(e, c->st));
  c->marks.emplace_back(stage, e);
}

void flush_marks(lr_ctx* c) {
  if (c->marks.empty()) return;
  LRB_CUDA(cudaStreamSynchronize(c->st));
  for (size_t i = 1; i < c->marks.size(); ++i) {
    const std::string& name = c->marks[i].first;
    if (name == "begin") continue;
    float ms = 0.f;
    LRB_CUDA(cudaEventElapsedTime(&ms, c->marks[i - 1].second, c->marks[i].second));
    bool found = false;
    for (size_t j = 0; j < c->stage_ms.size(); ++j)
      if (c->stage_ms[j].first == name) {
        c->stage_ms[j].second += ms;
        c->stage_count[j].second += 1;
        found = true;
      }
    if (!found) {
      c->stage_ms.emplace_back(name, ms);
      c->stage_count.emplace_back(name, 1);
    }
  }
  for (auto& m : c->marks) cudaEventDestroy(m.second);
  c->marks.clear();
}

// ---------------------------------------------------------------- helpers
void sync(lr_ctx* c) { LRB_CUDA(cudaStreamSynchronize(c->st)); }

void require_nonempty(int64_t m, int64_t n, const char* who) {
  if (m < 1 || n < 1) fail(LR_EINVAL, std::string(who) + ": matrix must be nonempty");
}
void require_rank_in_range(int64_t k, int64_t rows, int64_t cols, const char* who) {
  if (k < 1 || k > std::min(rows, cols))
    fail(LR_EINVAL, std::string(who) + ": rank " + std::to_string(k) + " out of range for " + std::to_string(rows) +
                        "x" + std::to_string(cols) + " matrix");
}
void require_sample_count(int64_t ell, int64_t rows, const char* who) {
  if (ell < 1 || ell > rows)
    fail(LR_EINVAL, std::string(who) + ": sample count " + std::to_string(ell) + " out of range for " +
                        std::to_string(rows) + " rows");
}
void require_ld(int64_t rows, int64_t ld, const char* who) {
  if (ld < std::max<int64_t>(rows, 1)) fail(LR_EINVAL, std::string(who) + ": leading dimension smaller than rows");
}

bool device_all_finite(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda) {
  DBuf<int> f(1, c->st);
  LRB_CUDA(cudaMemsetAsync(f.p, 0, sizeof(int), c->st));
  check_finite(m, n, a, lda, f, c->st);
  d2h_mapped(c, c->h_flags, f.p, sizeof(int));
  sync(c);
  return c->h_flags[0] == 0;
}

// GEMM wrapper: pads misaligned operands (TMA needs 16B-aligned base and ld)
void gemm(lr_ctx* c, int64_t M, int64_t N, int64_t K, const double* P, int64_t ldp, const double* Q, int64_t ldq,
          double* out, int64_t ldo, double alpha = 1.0, double beta = 0.0, int splits = -1, bool upper = false,
          int tri = 0) {
  auto ok = [](const double* p, int64_t ld) { return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0); };
  DBuf<double> pp, qq;
  if (!ok(P, ldp)) {
    const int64_t l = even(K);
    pp = DBuf<double>((size_t)l * M, c->st);
    copy_matrix(K, M, P, ldp, pp, l, c->st);
    P = pp;
    ldp = l;
  }
  if (!ok(Q, ldq)) {
    const int64_t l = even(K);
    qq = DBuf<double>((size_t)l * N, c->st);
    copy_matrix(K, N, Q, ldq, qq, l, c->st);
    Q = qq;
    ldq = l;
  }
  gemm_tn(c->ws, (int)M, (int)N, (int)K, P, ldp, Q, ldq, out, ldo, alpha, beta, splits, c->st, upper, tri);
}

// ---------------------------------------------------------------- A-sized contractions
// Ozaki-II emulation applies while K fits exact int32 accumulation; beyond
// that (and in the default mode) the DMMA GEMM runs.
constexpr int64_t kOzakiMaxK = int64_t(1) << 17;

// Residue planes of X (K x cols, K-contiguous) in grow-only workspace slots
// (a 68.7 GB plane set re-allocated from the stream pool every call fragments
// it; persistent slots keep steady-state calls allocation-free).  `cacheable`
// operands (A of the current CUR call) are split once and reused while an
// OzakiScope is open; `tmp_slot` 0/1 picks the slots of the other operand.
const OzakiOperand* ozaki_operand(lr_ctx* c, int64_t K, int64_t cols, const double* X, int64_t ldx, bool cacheable,
                                  int tmp_slot, OzakiOperand& out, int beta_override = 0) {
  const int beta = beta_override > 0 ? beta_override : ozaki_beta(K);
  if (cacheable) {  // the input matrix: kOzA slot, reused while an OzakiScope is open
    if (c->oz_cache_on && c->oz_src == X && c->oz_K == K && c->oz_cols == cols && c->oz_ld == ldx)
      return &c->oz_op;
    c->oz_src = nullptr;
    int8_t* pl = static_cast<int8_t*>(c->ws.try_get(WsSlot::kOzA, ozaki_plane_bytes(K, cols)));
    if (!pl) return nullptr;  // no room for the planes: the caller runs the DMMA GEMM
    c->oz_op.planes = pl;
    c->oz_op.shift = static_cast<int*>(c->ws.get(WsSlot::kOzAShift, sizeof(int) * (size_t)cols));
    c->oz_op.unsigned_res = K <= kOzakiMaxKUnsigned;  // A: the cheap u8 split (its partner stays s8)
    ozaki_split(K, cols, X, ldx, beta, c->oz_op, c->st);
    c->oz_src = c->oz_cache_on ? X : nullptr;
    c->oz_K = K;
    c->oz_cols = cols;
    c->oz_ld = ldx;
    return &c->oz_op;
  }
  out.planes = static_cast<int8_t*>(c->ws.try_get(tmp_slot ? WsSlot::kOzQ : WsSlot::kOzP, ozaki_plane_bytes(K, cols)));
  if (!out.planes) return nullptr;
  out.shift = static_cast<int*>(c->ws.get(tmp_slot ? WsSlot::kOzQShift : WsSlot::kOzPShift, sizeof(int) * (size_t)cols));
  out.unsigned_res = false;
  ozaki_split(K, cols, X, ldx, beta, out, c->st);
  return &out;
}

// out (M x N) = P^T Q where P or Q is the input matrix A (`a_side` 0: P, 1: Q)
void gemm_a(lr_ctx* c, int64_t M, int64_t N, int64_t K, const double* P, int64_t ldp, const double* Q, int64_t ldq,
            double* out, int64_t ldo, int a_side) {
  if (c->gemm_mode != LR_GEMM_OZAKI_INT8 || K > kOzakiMaxK) {
    gemm(c, M, N, K, P, ldp, Q, ldq, out, ldo);
    return;
  }
  if (a_side < 0 && c->oz_pinned) {  // a caller-pinned matrix (lr_ctx_cache_operand) keeps its planes
    if (P == c->pin_src && K == c->pin_K && M == c->pin_cols && ldp == c->pin_ld) a_side = 0;
    else if (Q == c->pin_src && K == c->pin_K && N == c->pin_cols && ldq == c->pin_ld) a_side = 1;
  }
  OzakiOperand op, oq;
  const OzakiOperand* Po = ozaki_operand(c, K, M, P, ldp, a_side == 0, 0, op);
  const OzakiOperand* Qo = Po ? ozaki_operand(c, K, N, Q, ldq, a_side == 1, 1, oq) : nullptr;
  if (!Po || !Qo) {  // residue planes do not fit next to the caller's data: FP64 DMMA
    gemm(c, M, N, K, P, ldp, Q, ldq, out, ldo);
    return;
  }
  mark(c, "ozaki_split");
  ozaki_gemm_tn(c->ws, *Po, *Qo, M, N, out, ldo, 1.0, 0.0, c->st);
}

// Scope of one CUR call: A's residue planes live until it closes.
struct OzakiScope {
  lr_ctx* c;
  explicit OzakiScope(lr_ctx* cc) : c(cc) { c->oz_cache_on = true; }
  ~OzakiScope() {
    if (c->oz_pinned) {  // a pinned operand's planes stay valid across calls; any other
      // matrix split during this call (e.g. a CUR input that is not the pinned one,
      // or upload_sketch's call-local copy) must not be matched by address later
      if (c->oz_src != c->pin_src) c->oz_src = nullptr;
      return;
    }
    c->oz_cache_on = false;
    c->oz_src = nullptr;  // the planes stay allocated in the workspace for the next call
  }
};

// ---------------------------------------------------------------- CPQR
// In-place CPQR of a working matrix W (ld even, 16B aligned).  Throws the
// reference's non-finite error for `who`.
// Working-matrix leading dimension for CPQR: heights <= 512 are padded to a
// multiple of 64 with zero rows (the predicate-free fast path of cpqr.cu).
inline int64_t work_ld(int64_t m) { return m <= 512 ? ((m + 63) / 64) * 64 : even(m); }
inline bool work_padded(int64_t m, int64_t ld) { return m <= 512 && ld == work_ld(m); }
void zero_pad_rows(lr_ctx* c, double* W, int64_t m, int64_t ld, int64_t n) {
  if (ld > m && n > 0)
    LRB_CUDA(cudaMemset2DAsync(W + m, ld * sizeof(double), 0, (ld - m) * sizeof(double), n, c->st));
}

void cpqr_core(lr_ctx* c, int64_t m, int64_t n, double* W, int64_t ldw, int64_t k, int64_t* piv, double* tau,
               const char* who, bool padded = false, bool nopivot = false) {
  DBuf<int> flags(1, c->st);
  DBuf<long long> rec(1, c->st);
  LRB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), c->st));
  LRB_CUDA(cudaMemsetAsync(rec.p, 0, sizeof(long long), c->st));
  cpqr_inplace(c->ws, m, n, W, ldw, k, piv, tau, flags, rec, padded, c->st, nopivot);
  d2h_mapped(c, c->h_flags, flags.p, sizeof(int));
  d2h_mapped(c, c->h_ll, rec.p, sizeof(long long));
  sync(c);
  if (c->h_flags[0]) fail(LR_EINVAL, std::string(who) + ": matrix has non-finite entries");
  c->stats.cpqr_steps += k;
  c->stats.norm_recomputes += c->h_ll[0];
}

// ---------------------------------------------------------------- triangular solve
void pinv_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double thr, double* out, int64_t ldo);

// solve.hpp:104-145 on device.  s11 upper part (+ diagonal) is used; when
// `check_inputs` the reference's validation (finite, strictly-lower zero) runs.
void solve_core(lr_ctx* c, int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12, int64_t ld12,
                const lr_solve_strategy& strat, double* t, int64_t ldt, bool check_inputs) {
  if (check_inputs) {
    DBuf<int> fl(2, c->st);
    LRB_CUDA(cudaMemsetAsync(fl.p, 0, 2 * sizeof(int), c->st));
    check_upper_triangular(k, s11, ld11, fl, c->st);
    check_finite(k, nc, s12, ld12, fl.p + 1, c->st);
    d2h_mapped(c, c->h_flags, fl.p, 2 * sizeof(int));
    sync(c);
    if (c->h_flags[1]) fail(LR_EINVAL, "stabilized_coeff_solve: non-finite entries");
    if (c->h_flags[0]) fail(LR_EINVAL, "stabilized_coeff_solve: block is not upper triangular");
  }
  c->stats.solve_escalated = 0;
  if (nc == 0) return;
  int kind = strat.kind;
  if (kind == LR_SOLVE_BACKSUB && strat.escalate) {
    DBuf<double> mm(2, c->st);
    diag_absminmax(k, s11, ld11, mm, c->st);
    d2h_mapped(c, c->h_scal, mm.p, 2 * sizeof(double));
    sync(c);
    const double dmax = c->h_scal[0], dmin = c->h_scal[1];
    if (dmax == 0.0 || dmin == 0.0 || dmax / dmin > 1e10) kind = LR_SOLVE_PINV;
  }
  if (kind == LR_SOLVE_BACKSUB) {
    DBuf<double> Mt((size_t)k * k, c->st);
    DBuf<int> zr(k, c->st);
    // no diagonal at or below the zeroing tolerance (known from the escalation
    // check): M = S11^-1 exactly, by the blocked inverse; otherwise the
    // back-substitution operator with its zeroed rows (solve.hpp:62-89)
    const bool no_zero_rows = strat.escalate && k > 64 && c->h_scal[1] > strat.threshold * c->h_scal[0];
    if (no_zero_rows) {
      DBuf<double> M((size_t)k * k, c->st);
      tri_upper_inverse_blocked(k, s11, ld11, M, k, c->st);
      transpose_matrix(k, k, M, k, Mt, k, c->st);
    } else {
      backsub_operator_t(k, s11, ld11, strat.threshold, Mt, zr, c->st);
    }
    gemm(c, k, nc, k, Mt, k, s12, ld12, t, ldt, 1.0, 0.0, -1, false, kTriP);  // M upper triangular
    if (!strat.escalate) {  // allow_singularity_error (solve.hpp:75-83)
      std::vector<int> hz(k);
      LRB_CUDA(cudaMemcpyAsync(hz.data(), zr.p, sizeof(int) * k, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      bool any = false;
      for (int z : hz) any |= z != 0;
      if (any) {
        DBuf<double> res(k, c->st), part(4 * num_sms() + 4, c->st), smax(1, c->st);
        max_abs(k, nc, s12, ld12, part, smax, c->st);
        backsub_residual_rows(k, nc, s11, ld11, s12, ld12, t, ldt, hz.data(), res, c->st);
        std::vector<double> hres(k);
        double rhs_scale = 0.0;
        LRB_CUDA(cudaMemcpyAsync(hres.data(), res.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c->st));
        LRB_CUDA(cudaMemcpyAsync(&rhs_scale, smax.p, sizeof(double), cudaMemcpyDeviceToHost, c->st));
        sync(c);
        for (int64_t i = k - 1; i >= 0; --i)
          if (hz[i] && hres[i] > strat.threshold * rhs_scale)
            fail(LR_ESINGULAR,
                 "stabilized_coeff_solve: zero diagonal with inconsistent right-hand side at index " +
                     std::to_string(i),
                 i);
      }
    }
    return;
  }
  if (kind == LR_SOLVE_PINV) {
    c->stats.solve_escalated = 1;
    // clean upper-triangular copy (the working matrix carries reflectors below the diagonal)
    DBuf<double> s((size_t)k * k, c->st), sp((size_t)k * k, c->st), spt((size_t)k * k, c->st);
    copy_upper(k, s11, ld11, s, k, c->st);
    pinv_core(c, k, k, s, k, strat.threshold, sp, k);
    transpose_matrix(k, k, sp, k, spt, k, c->st);
    gemm(c, k, nc, k, spt, k, s12, ld12, t, ldt);
    return;
  }
  // Tikhonov (solve.hpp:133-142): (S11^T S11 + ridge^2 I) T = S11^T S12, solved
  // by Cholesky on the GPU; when the normal matrix is singular (ridge = 0 and a
  // rank-deficient S11) the Cholesky breaks down and the reference's own
  // method runs instead: conjugate gradients per column to 1e-28 relative
  // residual, leaving on a non-positive curvature (solve.hpp:37-57).
  DBuf<double> s((size_t)k * k, c->st), rhs((size_t)k * nc, c->st);
  copy_upper(k, s11, ld11, s, k, c->st);
  DBuf<double> nm((size_t)k * k, c->st), eye((size_t)k * k, c->st);
  {
    std::vector<double> he((size_t)k * k, 0.0);
    for (int64_t i = 0; i < k; ++i) he[i + i * k] = strat.ridge * strat.ridge;
    LRB_CUDA(cudaMemcpyAsync(nm.p, he.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice, c->st));
    sync(c);
  }
  gemm(c, k, k, k, s, k, s, k, nm, k, 1.0, 1.0);  // nm = S^T S + ridge^2 I
  gemm(c, k, nc, k, s, k, s12, ld12, rhs, k);     // rhs = S^T S12
  copy_matrix(k, k, nm, k, eye, k, c->st);
  DBuf<int> info(1, c->st);
  cholesky_upper(c->ws, k, eye, k, info, c->st);
  d2h_mapped(c, c->h_flags, info.p, sizeof(int));
  sync(c);
  if (c->h_flags[0] == 0) {
    DBuf<double> ri((size_t)k * k, c->st), rit((size_t)k * k, c->st), y((size_t)k * nc, c->st);
    tri_upper_inverse(k, eye, k, ri, k, c->st);
    transpose_matrix(k, k, ri, k, rit, k, c->st);
    gemm(c, k, nc, k, ri, k, rhs, k, y, k);     // y = R^-T rhs
    gemm(c, k, nc, k, rit, k, y, k, t, ldt);    // t = R^-1 y
    return;
  }
  const int64_t ldk = even(k);
  DBuf<double> nme((size_t)ldk * k, c->st), x((size_t)ldk * nc, c->st), r((size_t)ldk * nc, c->st),
      d((size_t)ldk * nc, c->st), nd((size_t)ldk * nc, c->st), state((size_t)3 * nc, c->st);
  DBuf<int> act(1, c->st);
  copy_matrix(k, k, nm, k, nme, ldk, c->st);
  cg_init(k, nc, ldk, rhs, k, x, r, d, state, c->st);
  const int64_t max_iters = 8 * k + 16;
  for (int64_t it = 0; it < max_iters; ++it) {
    gemm(c, k, nc, k, nme, ldk, d, ldk, nd, ldk);  // nd = normal d (normal symmetric)
    LRB_CUDA(cudaMemsetAsync(act.p, 0, sizeof(int), c->st));
    cg_step(k, nc, ldk, nd, x, r, d, state, act, c->st);
    if ((it & 7) == 7 || it + 1 == max_iters) {
      d2h_mapped(c, c->h_flags, act.p, sizeof(int));
      sync(c);
      if (c->h_flags[0] == 0) break;
    }
  }
  copy_matrix(k, nc, x, ldk, t, ldt, c->st);
}

// ---------------------------------------------------------------- SVD / pinv
void svd_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma, double* v) {
  const bool transposed = m < n;
  if (!transposed) {
    if (!jacobi_svd(c->ws, m, n, a, lda, u, sigma, v, c->st))
      fail(LR_ECONVERGE, "svd: one-sided Jacobi did not converge within 60 sweeps for " + std::to_string(m) + "x" +
                             std::to_string(n) + " input");
    return;
  }
  DBuf<double> at((size_t)n * m, c->st);
  transpose_matrix(m, n, a, lda, at, n, c->st);
  // svd of a^T (n x m): ub (n x m), vb (m x m); swap (svd.hpp:181)
  if (!jacobi_svd(c->ws, n, m, at, n, v, sigma, u, c->st))
    fail(LR_ECONVERGE, "svd: one-sided Jacobi did not converge within 60 sweeps for " + std::to_string(m) + "x" +
                           std::to_string(n) + " input");
}

// out (n x m) = V_r diag(1/s) U_r^T with rank r = #{s >= thr * s_1}
void pinv_svd_path(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double thr, double* out,
                   int64_t ldo) {
  const int64_t r = std::min(m, n);
  DBuf<double> u((size_t)m * r, c->st), s(r, c->st), v((size_t)n * r, c->st);
  svd_core(c, m, n, a, lda, u, s, v);
  std::vector<double> hs(r);
  LRB_CUDA(cudaMemcpyAsync(hs.data(), s.p, sizeof(double) * r, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  int64_t rank = 0;
  if (hs[0] != 0.0)
    while (rank < r && hs[rank] >= thr * hs[0]) ++rank;
  if (rank == 0) {
    for (int64_t j = 0; j < m; ++j) LRB_CUDA(cudaMemsetAsync(out + j * ldo, 0, sizeof(double) * n, c->st));
    return;
  }
  // P = (V_r D)^T (rank x n), Q = U_r^T (rank x m); out = P^T Q
  std::vector<double> inv(rank);
  for (int64_t l = 0; l < rank; ++l) inv[l] = 1.0 / hs[l];
  DBuf<double> vd((size_t)n * rank, c->st), P((size_t)even(rank) * n, c->st), Q((size_t)even(rank) * m, c->st);
  copy_matrix(n, rank, v, n, vd, n, c->st);
  for (int64_t l = 0; l < rank; ++l) scale_matrix((int)n, 1, vd.p + l * n, n, inv[l], c->st);
  transpose_matrix(n, rank, vd, n, P, even(rank), c->st);
  transpose_matrix(m, rank, u, m, Q, even(rank), c->st);
  gemm(c, n, m, rank, P, even(rank), Q, even(rank), out, ldo);
}

// Largest ||R||_F ||R^-1||_F for which a pseudoinverse with relative cutoff
// thr (svd.hpp:193-207: keep sigma_i >= thr sigma_1) provably truncates
// nothing: ||R||_F >= sigma_1 and ||R^-1||_F >= 1/sigma_min, so a bound below
// 1/thr gives sigma_min > thr sigma_1.  1e7 caps it for the CholeskyQR2
// accuracy argument (cond^2 eps of the first Gram matrix well below 1).
double fast_cond_limit(double thr) { return std::min(1e7, 1.0 / thr); }

// CholeskyQR2 of a tall X (rows x k, ld) given also X^T (k x rows, ldt):
// R (k x k upper) with X = Q R, Rinv = R^-1.  Returns false when the Gram
// factorisation breaks down or cond bound ||R||_F ||R^-1||_F >= max_cond.
bool cholqr2(lr_ctx* c, int64_t rows, int64_t k, const double* X, int64_t ldx, const double* Xt, int64_t ldxt,
             double* R, double* Rinv, double max_cond = 1e7) {
  DBuf<double> G((size_t)k * k, c->st), R1inv((size_t)k * k, c->st), Q1((size_t)even(rows) * k, c->st);
  DBuf<int> info(2, c->st);
  gemm(c, k, k, rows, X, ldx, X, ldx, G, k, 1.0, 0.0, -1, true);  // G1 = X^T X (upper tiles)
  cholesky_upper(c->ws, k, G, k, info, c->st);  // G <- R1
  d2h_mapped(c, c->h_flags, info.p, sizeof(int));
  sync(c);
  if (c->h_flags[0] != 0) return false;
  tri_upper_inverse_blocked(k, G, k, R1inv, k, c->st);
  gemm(c, rows, k, k, Xt, ldxt, R1inv, k, Q1, even(rows), 1.0, 0.0, -1, false, kTriQ);  // Q1 = X R1^-1
  DBuf<double> G2((size_t)k * k, c->st), R2t((size_t)k * k, c->st);
  gemm(c, k, k, rows, Q1, even(rows), Q1, even(rows), G2, k, 1.0, 0.0, -1, true);  // G2 = Q1^T Q1
  cholesky_upper(c->ws, k, G2, k, info.p + 1, c->st);
  d2h_mapped(c, c->h_flags + 1, info.p + 1, sizeof(int));
  sync(c);
  if (c->h_flags[1] != 0) return false;
  // R = R2 R1: R(i,j) = sum_l R2(i,l) R1(l,j) -> P = R2^T
  transpose_matrix(k, k, G2, k, R2t, k, c->st);
  gemm(c, k, k, k, R2t, k, G, k, R, k);
  tri_upper_inverse_blocked(k, R, k, Rinv, k, c->st);
  DBuf<double> part(4 * num_sms() + 4, c->st), f(2, c->st);
  frob2(k, k, R, k, part, f, c->st);
  frob2(k, k, Rinv, k, part, f.p + 1, c->st);
  d2h_mapped(c, c->h_scal, f.p, 2 * sizeof(double));
  sync(c);
  const double cond_bound = std::sqrt(c->h_scal[0]) * std::sqrt(c->h_scal[1]);
  return std::isfinite(cond_bound) && cond_bound < max_cond;
}

cudaStream_t aux_stream(cudaStream_t& s);

// Two independent CholeskyQR2 factorizations (cholqr2 above) interleaved on
// two streams: each is a chain of latency-bound small kernels (Gram GEMM,
// blocked Cholesky, triangular inverse) with host reads of the Cholesky info
// and the condition bound; phase by phase the two chains run concurrently and
// share those synchronisation points (three instead of six).
struct Chol2Job {
  int64_t rows, k;
  const double* X;
  int64_t ldx;
  const double* Xt;
  int64_t ldxt;
  double* R;
  double* Rinv;
  double max_cond;
  bool ok;
};
void cholqr2_pair(lr_ctx* c, Chol2Job& j0, Chol2Job& j1) {
  cudaStream_t S[2] = {c->st, aux_stream(c->side_st)};
  Chol2Job* J[2] = {&j0, &j1};
  DBuf<double> G[2], R1inv[2], Q1[2], G2[2], R2t[2], part[2], f[2];
  DBuf<int> info(4, c->st);
  for (int i = 0; i < 2; ++i) {
    const int64_t k = J[i]->k, rows = J[i]->rows;
    G[i] = DBuf<double>((size_t)k * k, c->st);
    R1inv[i] = DBuf<double>((size_t)k * k, c->st);
    Q1[i] = DBuf<double>((size_t)even(rows) * k, c->st);
    G2[i] = DBuf<double>((size_t)k * k, c->st);
    R2t[i] = DBuf<double>((size_t)k * k, c->st);
    part[i] = DBuf<double>(4 * num_sms() + 4, c->st);
    f[i] = DBuf<double>(2, c->st);
    J[i]->ok = false;
  }
  cudaEvent_t fork = nullptr;
  LRB_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  LRB_CUDA(cudaEventRecord(fork, S[0]));  // the buffers above (and the jobs' inputs) are ordered on S[0]
  LRB_CUDA(cudaStreamWaitEvent(S[1], fork, 0));
  cudaEventDestroy(fork);
  // Declared after the buffers, so it runs first on every exit (an exception
  // included): S[0] waits for the side chain before any buffer is released.
  struct Join {
    cudaStream_t main, side;
    ~Join() {
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
      cudaEventRecord(e, side);
      cudaStreamWaitEvent(main, e, 0);
      cudaEventDestroy(e);
    }
  } join{S[0], S[1]};
  cudaStream_t main_st = c->st;
  // the side chain runs with its own stream AND its own workspace (the GEMM's
  // split-K partials and the Cholesky panels live in workspace slots)
  auto on = [&](int i, const std::function<void()>& fn) {
    c->st = S[i];
    if (i == 1) c->ws.swap(c->ws_side);
    auto restore = [&] {
      if (i == 1) c->ws.swap(c->ws_side);
      c->st = main_st;
    };
    try {
      fn();
    } catch (...) {
      restore();
      throw;
    }
    restore();
  };
  auto sync_both = [&] {
    LRB_CUDA(cudaStreamSynchronize(S[0]));
    LRB_CUDA(cudaStreamSynchronize(S[1]));
  };
  // phase 1: G1 = X^T X (upper tiles), R1 = chol(G1)
  for (int i = 0; i < 2; ++i)
    on(i, [&] {
      const Chol2Job& j = *J[i];
      gemm(c, j.k, j.k, j.rows, j.X, j.ldx, j.X, j.ldx, G[i], j.k, 1.0, 0.0, -1, true);
      cholesky_upper(c->ws, j.k, G[i], j.k, info.p + i, c->st);
      copy_bytes_mapped(c->h_flags + i, info.p + i, sizeof(int), c->st);
    });
  sync_both();
  bool ok[2] = {c->h_flags[0] == 0, c->h_flags[1] == 0};
  // phase 2: Q1 = X R1^-1, G2 = Q1^T Q1, R2 = chol(G2)
  for (int i = 0; i < 2; ++i)
    if (ok[i])
      on(i, [&] {
        const Chol2Job& j = *J[i];
        tri_upper_inverse_blocked(j.k, G[i], j.k, R1inv[i], j.k, c->st);
        gemm(c, j.rows, j.k, j.k, j.Xt, j.ldxt, R1inv[i], j.k, Q1[i], even(j.rows), 1.0, 0.0, -1, false, kTriQ);
        gemm(c, j.k, j.k, j.rows, Q1[i], even(j.rows), Q1[i], even(j.rows), G2[i], j.k, 1.0, 0.0, -1, true);
        cholesky_upper(c->ws, j.k, G2[i], j.k, info.p + 2 + i, c->st);
        copy_bytes_mapped(c->h_flags + 2 + i, info.p + 2 + i, sizeof(int), c->st);
      });
  sync_both();
  for (int i = 0; i < 2; ++i) ok[i] = ok[i] && c->h_flags[2 + i] == 0;
  // phase 3: R = R2 R1, R^-1, ||R||_F ||R^-1||_F
  for (int i = 0; i < 2; ++i)
    if (ok[i])
      on(i, [&] {
        const Chol2Job& j = *J[i];
        transpose_matrix(j.k, j.k, G2[i], j.k, R2t[i], j.k, c->st);
        gemm(c, j.k, j.k, j.k, R2t[i], j.k, G[i], j.k, j.R, j.k);
        tri_upper_inverse_blocked(j.k, j.R, j.k, j.Rinv, j.k, c->st);
        frob2(j.k, j.k, j.R, j.k, part[i], f[i], c->st);
        frob2(j.k, j.k, j.Rinv, j.k, part[i], f[i].p + 1, c->st);
        copy_bytes_mapped(c->h_scal + 2 * i, f[i].p, 2 * sizeof(double), c->st);
      });
  sync_both();
  for (int i = 0; i < 2; ++i) {
    if (!ok[i]) continue;
    const double cb = std::sqrt(c->h_scal[2 * i]) * std::sqrt(c->h_scal[2 * i + 1]);
    J[i]->ok = std::isfinite(cb) && cb < J[i]->max_cond;
  }
}

void pinv_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double thr, double* out, int64_t ldo) {
  if (!(thr > 0.0 && thr < 1.0)) fail(LR_EINVAL, "pinv: threshold must lie in (0,1)");
  require_nonempty(m, n, "svd");
  if (!device_all_finite(c, m, n, a, lda)) fail(LR_EINVAL, "svd: matrix has non-finite entries");
  // fast path on the tall orientation when provably no singular value is truncated
  const bool tall = m >= n;
  const int64_t rows = tall ? m : n, k = tall ? n : m;
  if (rows >= 2 * k && k >= 8) {
    DBuf<double> X((size_t)even(rows) * k, c->st), Xt((size_t)even(k) * rows, c->st);
    if (tall) {
      copy_matrix(m, n, a, lda, X, even(rows), c->st);
      transpose_matrix(m, n, a, lda, Xt, even(k), c->st);
    } else {
      transpose_matrix(m, n, a, lda, X, even(rows), c->st);
      copy_matrix(m, n, a, lda, Xt, even(k), c->st);
    }
    DBuf<double> R((size_t)k * k, c->st), Ri((size_t)k * k, c->st);
    if (cholqr2(c, rows, k, X, even(rows), Xt, even(k), R, Ri, fast_cond_limit(thr))) {
      // X^+ = R^-1 R^-T X^T (k x rows).  Qt = R^-T X^T: Qt(l,j) = sum_t Ri(t,l) Xt(t,j)
      DBuf<double> Qt((size_t)even(k) * rows, c->st), Rit((size_t)k * k, c->st);
      gemm(c, k, rows, k, Ri, k, Xt, even(k), Qt, even(k));
      transpose_matrix(k, k, Ri, k, Rit, k, c->st);
      if (tall) {
        gemm(c, k, rows, k, Rit, k, Qt, even(k), out, ldo);  // out (n x m) = R^-1 Qt
      } else {
        DBuf<double> xp((size_t)k * rows, c->st);
        gemm(c, k, rows, k, Rit, k, Qt, even(k), xp, k);  // pinv(a^T) (m x n)
        transpose_matrix(k, rows, xp, k, out, ldo, c->st);
      }
      c->stats.pinv_fast_path = 1;
      return;
    }
  }
  c->stats.pinv_fast_path = 0;
  pinv_svd_path(c, m, n, a, lda, thr, out, ldo);
}

// ---------------------------------------------------------------- pipelines
struct ColumnIdDev {
  DBuf<double> W;  // working matrix after CPQR (k rows of s in its top)
  int64_t ldw = 0;
};

// id.hpp:91-105 on a working copy; pivots/coeff device pointers
void id_column_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                    const lr_solve_strategy& strat, int64_t* piv, double* coeff, int64_t ldc) {
  require_rank_in_range(k, m, n, "id_column");
  require_nonempty(m, n, "cpqr_partial");
  const int64_t ldw = work_ld(m);
  DBuf<double> W((size_t)ldw * n, c->st), tau(k, c->st);
  zero_pad_rows(c, W, m, ldw, n);
  copy_matrix(m, n, a, lda, W, ldw, c->st);
  cpqr_core(c, m, n, W, ldw, k, piv, tau, "cpqr_partial", work_padded(m, ldw));
  solve_core(c, k, n - k, W, ldw, W.p + k * ldw, ldw, strat, coeff, ldc, false);
}

// sketch.hpp:67-78 into y (ell x n, ldy); a must be validated by the caller
// rng.hpp:14-62 on the host (SRFT row sampling)
uint64_t host_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t host_stream_value(uint64_t seed, uint64_t index) { return host_mix64(seed + (index + 1) * 0x9E3779B97F4A7C15ULL); }
uint64_t host_derive_seed(uint64_t seed, uint64_t tag) { return host_stream_value(seed, tag ^ 0xD1B54A32D192ED03ULL); }
// CounterRng::sample_without_replacement (partial Fisher-Yates), rng.hpp:53-62
std::vector<int64_t> sample_without_replacement(uint64_t seed, int64_t population, int64_t count) {
  std::vector<int64_t> pool((size_t)population);
  for (int64_t i = 0; i < population; ++i) pool[(size_t)i] = i;
  uint64_t next = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t j = i + (int64_t)(host_stream_value(seed, next++) % (uint64_t)(population - i));
    std::swap(pool[(size_t)i], pool[(size_t)j]);
  }
  pool.resize((size_t)count);
  return pool;
}

// Omega^T (m x ell, ld m) of the sketch kind: Gaussian (rng.hpp:74-94) or the
// SRFT operator (sketch.hpp:84-100; the reference applies it through a fast
// Hartley transform when m is a power of two -- same operator, the GPU
// contracts with it on the tensor cores like the Gaussian one)
void sketch_operator_t(lr_ctx* c, int64_t m, int64_t ell, int kind, uint64_t seed, double* omt) {
  if (kind == LR_SKETCH_SRFT) {
    const std::vector<int64_t> rows = sample_without_replacement(host_derive_seed(seed, 2), m, ell);
    DBuf<int64_t> dr(ell, c->st);
    LRB_CUDA(cudaMemcpyAsync(dr.p, rows.data(), sizeof(int64_t) * ell, cudaMemcpyHostToDevice, c->st));
    srft_operator_t(m, ell, host_derive_seed(seed, 1), dr, omt, m, c->st);
    sync(c);  // rows (host vector) must outlive the copy
  } else {
    gaussian_matrix(ell, m, seed, omt, m, true, c->st);
  }
}

// sketch.hpp:137-141: for a row count that is not a power of two the
// reference forms the SRFT sample as the plain dense product operator * A;
// that product is reproduced with its exact arithmetic (ascending k, no FMA),
// the power-of-two (fast Hartley) case is contracted on the tensor cores
inline bool srft_dense_fallback(int kind, int64_t m) { return kind == LR_SKETCH_SRFT && (m & (m - 1)) != 0; }

void sketch_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed,
                 double* y, int64_t ldy, int kind = LR_SKETCH_GAUSSIAN) {
  DBuf<double> omt((size_t)m * even(ell), c->st);
  // Omega^T (m x ell): element (i,j) of Omega stored at omt[j + i*m]
  sketch_operator_t(c, m, ell, kind, seed, omt);
  mark(c, "omega");
  if (srft_dense_fallback(kind, m))
    gemm_tn_ordered((int)ell, (int)n, (int)m, omt, m, a, lda, y, ldy, c->st);
  else
    gemm_a(c, ell, n, m, omt, m, a, lda, y, ldy, 1);
  mark(c, "sketch_gemm");
}

// svd.hpp:216-235 orth_rows on the transposed sample: an orthonormal basis Q
// (rows x r, ld ldq) of the columns of X (rows x k, ld ldx), rank-trimmed like
// the reference's Householder QR (trailing |R_ii| <= max|R_ii| eps max(rows, k)
// dropped).  CholeskyQR2 when it is provably safe (cond bound < 1e7, hence full
// rank), else the unpivoted Householder QR of cpqr.cu.  Q may differ from the
// reference's by column signs, which leave the power sketch's row space, every
// pivot and T unchanged.  Returns r.
int64_t orth_cols_core(lr_ctx* c, int64_t rows, int64_t k, const double* X, int64_t ldx, double* Q, int64_t ldq) {
  require_nonempty(rows, k, "orth_rows");
  if (!device_all_finite(c, rows, k, X, ldx)) fail(LR_EINVAL, "orth_rows: matrix has non-finite entries");
  if (rows >= 2 * k) {
    DBuf<double> Xt((size_t)even(k) * rows, c->st), R((size_t)k * k, c->st), Ri((size_t)k * k, c->st);
    transpose_matrix(rows, k, X, ldx, Xt, even(k), c->st);
    if (cholqr2(c, rows, k, X, ldx, Xt, even(k), R, Ri)) {
      gemm(c, rows, k, k, Xt, even(k), Ri, k, Q, ldq, 1.0, 0.0, -1, false, kTriQ);  // Q = X R^-1
      return k;
    }
  }
  const int64_t rmax = std::min(rows, k), ldw = even(rows);
  DBuf<double> W((size_t)ldw * k, c->st), tau(rmax, c->st), d(rmax, c->st), Qf((size_t)ldw * rmax, c->st);
  DBuf<int64_t> piv(k, c->st);
  copy_matrix(rows, k, X, ldx, W, ldw, c->st);
  cpqr_core(c, rows, k, W, ldw, rmax, piv, tau, "orth_rows", false, true);
  // |R_ii| -> host, trailing trim
  LRB_CUDA(cudaMemcpy2DAsync(d.p, sizeof(double), W.p, (ldw + 1) * sizeof(double), sizeof(double), rmax,
                             cudaMemcpyDeviceToDevice, c->st));
  std::vector<double> h(rmax);
  LRB_CUDA(cudaMemcpyAsync(h.data(), d.p, sizeof(double) * rmax, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  double dmax = 0.0;
  for (double v : h) dmax = std::max(dmax, std::fabs(v));
  const double tol = dmax * 2.220446049250313e-16 * (double)std::max(rows, k);
  int64_t r = rmax;
  while (r > 0 && std::fabs(h[r - 1]) <= tol) --r;
  if (r > 0) {
    cpqr_form_q(rows, k, W, ldw, rmax, tau, Qf, ldw, c->st);
    copy_matrix(rows, r, Qf, ldw, Q, ldq, c->st);
  }
  return r;
}

// sketch.hpp:148-164 power rounds on the sample Y (rows x n, ld ldy):
// Z^T = A Y^T (A^T materialised once so both products are K-contiguous),
// Y = Z A (the input matrix's contraction: Ozaki or DMMA per the context).
// Returns the new sample in Yb (ld work_ld(rows), zero padded); *rows updated.
//
// On the INT8 engine with A's residue planes cached (the sketch split them), Z^T = A Y^T contracts
// over A's columns, the index A's planes are scaled along: with x_ij = rint(a_ij 2^s_j) the
// integers behind the planes, A Y^T = X (diag(2^-s) Y^T) exactly, so the column scales are folded
// into Y^T's rows, that product's right operand is split along its own columns as usual, and A's
// planes enter the tcgen05 GEMM as the M-major operand (ozaki_gemm_a_cols).  No A^T is formed
// (34 GB at C4) and the round's 2 l m n flops leave the DMMA pipe.  The rounding differs from the
// TN products': A is rounded to beta bits relative to its COLUMN maxima (a columnwise backward
// error of 2^-beta), Y^T's scaled rows relative to their column maxima.
bool power_zt_int8(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t rows, const double* Ym,
                   int64_t ldym, double* Zt, int64_t ldz) {
  static const bool off = getenv("LRB_POWER_INT8") && atoi(getenv("LRB_POWER_INT8")) == 0;
  if (off || c->gemm_mode != LR_GEMM_OZAKI_INT8 || !c->oz_cache_on || c->oz_src != a || c->oz_K != m ||
      c->oz_cols != n || c->oz_ld != lda || n > kOzakiMaxK || (c->oz_op.unsigned_res && n > kOzakiMaxKUnsigned))
    return false;
  const int bq = ozaki_partner_beta(n, c->oz_op.beta);
  if (bq < 40) return false;  // too few bits left for the partner (n much larger than m)
  DBuf<double> Ys((size_t)even(n) * rows, c->st);
  ozaki_fold_scales(n, rows, Ym, ldym, c->oz_op.shift, Ys, even(n), c->st);
  OzakiOperand oq;
  const OzakiOperand* Qo = ozaki_operand(c, n, rows, Ys, even(n), false, 1, oq, bq);
  if (!Qo) return false;
  DBuf<int> zero((size_t)m, c->st);
  LRB_CUDA(cudaMemsetAsync(zero.p, 0, sizeof(int) * (size_t)m, c->st));
  mark(c, "ozaki_split");
  ozaki_gemm_a_cols(c->ws, c->oz_op, *Qo, rows, Zt, ldz, zero, c->st);
  return true;
}

void power_rounds_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int q, bool reorth,
                       DBuf<double>& Yb, int64_t& ldy, int64_t& rows) {
  const int64_t ldat = even(n);
  DBuf<double> At;  // A^T (n x m), formed only when a round takes the DMMA path
  for (int round = 0; round < q; ++round) {
    DBuf<double> Yt((size_t)ldat * rows, c->st), Qy;
    transpose_matrix(rows, n, Yb, ldy, Yt, ldat, c->st);  // Y^T: n x rows
    const double* Ym = Yt;
    if (reorth) {
      Qy = DBuf<double>((size_t)ldat * rows, c->st);
      rows = orth_cols_core(c, n, rows, Yt, ldat, Qy, ldat);
      Ym = Qy;
    }
    if (rows < 1) fail(LR_ERUNTIME, "randomized_id: sample rank collapsed below target rank");
    mark(c, "power_orth");
    DBuf<double> Zt((size_t)even(m) * rows, c->st), Qz;
    if (!power_zt_int8(c, m, n, a, lda, rows, Ym, ldat, Zt, even(m))) {
      if (!At.p) {
        At = DBuf<double>((size_t)ldat * m, c->st);
        transpose_matrix(m, n, a, lda, At, ldat, c->st);
        mark(c, "power_transpose_a");
      }
      gemm(c, m, rows, n, At, ldat, Ym, ldat, Zt, even(m));  // Z^T = A Y^T (m x rows)
    }
    mark(c, "power_zt_gemm");
    const double* Zm = Zt;
    if (reorth) {
      Qz = DBuf<double>((size_t)even(m) * rows, c->st);
      rows = orth_cols_core(c, m, rows, Zt, even(m), Qz, even(m));
      Zm = Qz;
    }
    mark(c, "power_orth");
    if (rows < 1) fail(LR_ERUNTIME, "randomized_id: sample rank collapsed below target rank");
    ldy = work_ld(rows);
    Yb = DBuf<double>((size_t)ldy * n, c->st);
    zero_pad_rows(c, Yb, rows, ldy, n);
    gemm_a(c, rows, n, m, Zm, even(m), a, lda, Yb, ldy, 1);  // Y = Z A (rows x n)
    mark(c, "power_y_gemm");
  }
}

// sketch.hpp:200-223 argument checks (before any work)
int64_t check_randomized_id(int64_t m, int64_t n, int64_t k, const lr_sketch_config& cfg) {
  require_rank_in_range(k, m, n, "randomized_id");
  if (cfg.kind != LR_SKETCH_GAUSSIAN && cfg.kind != LR_SKETCH_SRFT)
    fail(LR_EINVAL, "randomized_id: unknown sketch kind");
  if (cfg.power < 0) fail(LR_EINVAL, "sketch_power: q must be nonnegative");
  // SketchConfig::sample_count, sketch.hpp:29-32
  const int64_t ell = cfg.kind == LR_SKETCH_GAUSSIAN ? k + cfg.oversample
                                                      : (cfg.srft_samples > 0 ? cfg.srft_samples : 2 * k);
  if (ell < k) fail(LR_EINVAL, "build_sample: sample count below target rank");
  const char* who = cfg.kind == LR_SKETCH_GAUSSIAN ? "sketch_gaussian" : "sketch_srft";
  require_nonempty(m, n, who);
  require_sample_count(ell, m, who);
  return ell;
}

// sketch.hpp:200-223.  Ypre: the sample Y (ell x n, ld work_ld(ell), zero
// padded) already formed by the caller (the pipelined upload), else sketched here.
void randomized_id_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                        const lr_sketch_config& cfg, const lr_solve_strategy& strat, int64_t* piv, double* coeff,
                        int64_t ldc, double* Ypre = nullptr) {
  int64_t ell = check_randomized_id(m, n, k, cfg);
  int64_t ldy = work_ld(ell);
  // power rounds contract A 1 + 2q times: keep its residue planes for the whole call
  // (a CUR caller has its own scope open already)
  std::optional<OzakiScope> planes_scope;
  if (cfg.power > 0 && !c->oz_cache_on) planes_scope.emplace(c);
  DBuf<double> Yb;
  double* Y = Ypre;
  if (!Y) {
    Yb = DBuf<double>((size_t)ldy * n, c->st);
    Y = Yb;
    zero_pad_rows(c, Y, ell, ldy, n);
    sketch_core(c, m, n, a, lda, ell, cfg.seed, Y, ldy, cfg.kind);
  }
  if (cfg.power > 0) {  // sketch.hpp:148-164 (the caller's pre-sketched Y only for q = 0)
    if (Ypre) fail(LR_ERUNTIME, "randomized_id: power rounds need the library-owned sample");
    power_rounds_core(c, m, n, a, lda, cfg.power, cfg.reorthonormalize != 0, Yb, ldy, ell);
    Y = Yb;
  }
  const int64_t steps = std::min(ell, n);  // cpqr_full
  if (steps < k) fail(LR_ERUNTIME, "randomized_id: sample rank collapsed below target rank");
  DBuf<double> tau(steps, c->st);
  try {
    cpqr_core(c, ell, n, Y, ldy, steps, piv, tau, "cpqr_partial", work_padded(ell, ldy));
  } catch (const LrError& e) {
    // Y is non-finite: distinguish a non-finite A (sketch_gaussian's check) from overflow in Y
    if (e.code == LR_EINVAL && !device_all_finite(c, m, n, a, lda))
      fail(LR_EINVAL, std::string(cfg.kind == LR_SKETCH_SRFT ? "sketch_srft" : "sketch_gaussian") +
                          ": matrix has non-finite entries");
    throw;
  }
  mark(c, "cpqr_sample");
  solve_core(c, k, n - k, Y, ldy, Y + k * ldy, ldy, strat, coeff, ldc, false);
  mark(c, "coeff_solve_col");
}

// id.hpp:124-134: row ID of C = A(:, J) (full rank) + skeleton
void tsid_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const int64_t* col_piv,
               const lr_solve_strategy& strat, int64_t* row_piv, double* row_coeff, int64_t ldrc, double* skeleton,
               double* C_out /* m x k or null */, double* Ct_keep /* k x m (ld even(k)) or null */) {
  (void)n;
  DBuf<double> Cb;
  double* C = C_out;
  if (!C) {
    Cb = DBuf<double>((size_t)m * k, c->st);
    C = Cb;
  }
  if (a) gather_columns(m, k, a, lda, col_piv, C, m, c->st);  // a == null: C_out already holds C
  const int64_t ldct = work_ld(k);
  DBuf<double> Ct((size_t)ldct * m, c->st);
  zero_pad_rows(c, Ct, k, ldct, m);
  transpose_matrix(m, k, C, m, Ct, ldct, c->st);
  if (Ct_keep) copy_matrix(k, m, Ct, ldct, Ct_keep, even(k), c->st);
  // id_row(c, k) = id_column(c^T, k) (id.hpp:109-119)
  require_rank_in_range(k, k, m, "id_column");
  DBuf<double> tau(k, c->st);
  mark(c, "gather_c");
  cpqr_core(c, k, m, Ct, ldct, k, row_piv, tau, "cpqr_partial", work_padded(k, ldct));
  mark(c, "cpqr_ct");
  solve_core(c, k, m - k, Ct, ldct, Ct.p + k * ldct, ldct, strat, row_coeff, ldrc, false);
  if (skeleton) gather_rows(k, k, C, m, row_piv, skeleton, k, c->st);
  mark(c, "coeff_solve_row");
}

// cur.hpp:23-34 / lowrank_main.cpp:215 given skeleton index sets
// Xt (n x k, ld ldxt) = A^T Q for Q (m x k, ld ldq): the one place U touches A
using ApplyAt = std::function<void(const double* Q, int64_t ldq, double* Xt, int64_t ldxt)>;

// U of the CUR from its skeletons C (m x k, ld m) and R (k x n, ld k):
// cur.hpp:30 (u_mode LR_U_VT_RPINV) or lowrank_main.cpp:215 (LR_U_CPINV_A_RPINV)
void u_core(lr_ctx* c, int64_t m, int64_t n, int64_t k, const double* C, const double* R, const int64_t* col_piv,
            const double* col_coeff, int64_t ldcc, double thr, int u_mode, double* U,
            const double* Ct_in /* k x m ld even(k), may be null */, const ApplyAt& apply_at) {
  if (!(thr > 0.0 && thr < 1.0)) fail(LR_EINVAL, "pinv: threshold must lie in (0,1)");
  const int64_t ldk = even(k);
  DBuf<double> Ctb;
  const double* Ct = Ct_in;
  if (!Ct) {
    Ctb = DBuf<double>((size_t)ldk * m, c->st);
    transpose_matrix(m, k, C, m, Ctb, ldk, c->st);
    Ct = Ctb;
  }
  DBuf<double> Rt((size_t)even(n) * k, c->st), Rk((size_t)ldk * n, c->st);
  transpose_matrix(k, n, R, k, Rt, even(n), c->st);
  copy_matrix(k, n, R, k, Rk, ldk, c->st);  // R with an even leading dimension for TMA
  DBuf<double> Sr((size_t)k * k, c->st), Sri((size_t)k * k, c->st);
  mark(c, "gather_r");
  c->stats.pinv_fast_path = 0;
  c->stats.concurrent_tail = 0;
  if (u_mode == LR_U_CPINV_A_RPINV) {
    DBuf<double> Rc((size_t)k * k, c->st), Rci((size_t)k * k, c->st);
    DBuf<double> Cm((size_t)even(m) * k, c->st);
    copy_matrix(m, k, C, m, Cm, even(m), c->st);
    // R^T = Qr Sr and C = Qc Rc are independent: both CholeskyQR2 chains at once
    Chol2Job jr{n, k, Rt, even(n), Rk, ldk, Sr, Sri, fast_cond_limit(thr), false};
    Chol2Job jc{m, k, Cm, even(m), Ct, ldk, Rc, Rci, fast_cond_limit(thr), false};
    cholqr2_pair(c, jr, jc);
    const bool r_ok = jr.ok, c_ok = jc.ok;
    mark(c, "cholqr2_rc");
    if (c_ok && r_ok) {
      c->stats.pinv_fast_path = 1;
      // C = Qc Rc, R^T = Qr Sr  =>  U = C^+ A R^+ = Rc^-1 (Qc^T A Qr) Sr^-T.
      // The big contraction uses the orthonormal Qc (not C): applying Rc^-1
      // to C^T A would square cond(C) in the least-squares error.
      DBuf<double> Qc((size_t)even(m) * k, c->st), Qr((size_t)even(n) * k, c->st);
      gemm(c, m, k, k, Ct, ldk, Rci, k, Qc, even(m), 1.0, 0.0, -1, false, kTriQ);            // Qc = C Rc^-1  (m x k)
      gemm(c, n, k, k, Rk, ldk, Sri, k, Qr, even(n), 1.0, 0.0, -1, false, kTriQ);            // Qr = R^T Sr^-1 (n x k)
      DBuf<double> Xt((size_t)even(n) * k, c->st), W((size_t)k * k, c->st);
      mark(c, "form_q");
      apply_at(Qc, even(m), Xt, even(n));                        // X^T = A^T Qc  (n x k)
      mark(c, "ctA_gemm");
      gemm(c, k, k, n, Xt, even(n), Qr, even(n), W, k);          // W = Qc^T A Qr
      DBuf<double> t1((size_t)k * k, c->st), tt((size_t)k * k, c->st), st((size_t)k * k, c->st);
      transpose_matrix(k, k, Rci, k, tt, k, c->st);
      gemm(c, k, k, k, tt, k, W, k, t1, k);                      // t1 = Rc^-1 W
      transpose_matrix(k, k, t1, k, tt, k, c->st);
      transpose_matrix(k, k, Sri, k, st, k, c->st);
      gemm(c, k, k, k, tt, k, st, k, U, k);                      // U = t1 Sr^-T
      mark(c, "u_small");
      return;
    }
    // general path: explicit truncated pseudoinverses (SVD route when ill-conditioned)
    DBuf<double> Cp((size_t)k * m, c->st), Rp((size_t)n * k, c->st);
    pinv_core(c, m, k, C, m, thr, Cp, k);
    pinv_core(c, k, n, R, k, thr, Rp, n);
    // (Cp A) Rp: X^T = A^T Cp^T (n x k) then U = X Rp
    DBuf<double> Cpt((size_t)even(m) * k, c->st), Xt((size_t)even(n) * k, c->st);
    transpose_matrix(k, m, Cp, k, Cpt, even(m), c->st);
    apply_at(Cpt, even(m), Xt, even(n));
    DBuf<double> Rpe((size_t)even(n) * k, c->st);
    copy_matrix(n, k, Rp, n, Rpe, even(n), c->st);
    gemm(c, k, k, n, Xt, even(n), Rpe, even(n), U, k);
    return;
  }
  // u = basis()^T pinv(r) (cur.hpp:30) = R+^T(:, J_skel)^T + coeff R+(J_res, :)
  const bool r_ok = cholqr2(c, n, k, Rt, even(n), Rk, ldk, Sr, Sri, fast_cond_limit(thr));
  mark(c, "cholqr2_r");
  DBuf<double> Rpt((size_t)ldk * n, c->st);  // R+^T (k x n)
  if (r_ok) {
    c->stats.pinv_fast_path = 1;
    DBuf<double> Qrt((size_t)ldk * n, c->st), Srit((size_t)k * k, c->st);
    gemm(c, k, n, k, Sri, k, Rk, ldk, Qrt, ldk);  // Qr^T = Sr^-T R
    transpose_matrix(k, k, Sri, k, Srit, k, c->st);
    gemm(c, k, n, k, Srit, k, Qrt, ldk, Rpt, ldk);  // R+^T = Sr^-1 Qr^T
  } else {
    DBuf<double> Rp((size_t)n * k, c->st);
    pinv_core(c, k, n, R, k, thr, Rp, n);
    transpose_matrix(n, k, Rp, n, Rpt, ldk, c->st);
  }
  // G = R+^T(:, J): columns permuted by the column pivots
  DBuf<double> G((size_t)ldk * n, c->st);
  DBuf<int64_t> pv(n, c->st);
  // col_piv holds the full permutation (n entries)
  gather_columns(k, n, Rpt, ldk, col_piv, G, ldk, c->st);
  // U^T = G_skel + G_res coeff^T -> U^T(b,a) = sum_l G_res^T(l,b) coeff^T(l,a)
  const int64_t nr = n - k;
  DBuf<double> Ut((size_t)k * k, c->st);
  copy_matrix(k, k, G, ldk, Ut, k, c->st);
  if (nr > 0) {
    DBuf<double> Grt((size_t)even(nr) * k, c->st), cft((size_t)even(nr) * k, c->st);
    transpose_matrix(k, nr, G.p + k * ldk, ldk, Grt, even(nr), c->st);
    transpose_matrix(k, nr, col_coeff, ldcc, cft, even(nr), c->st);
    gemm(c, k, k, nr, Grt, even(nr), cft, even(nr), Ut, k, 1.0, 1.0);
  }
  transpose_matrix(k, k, Ut, k, U, k, c->st);
}

// ---------------------------------------------------------------- concurrent CUR tail
// After C = A(:, J) the tail of the randomized CUR is two independent chains:
//   (1) row ID of C (CPQR of C^T, k steps, latency-bound) -> R = A(I, :) ->
//       CholeskyQR2 of R^T -> Q_r
//   (2) Q_c = C R_c^-1 -> X^T = A^T Q_c (the second A-sized contraction,
//       tensor-bound)
// joined by U = R_c^-1 (X^T ... Q_r) S_r^-T.  They run concurrently on two
// disjoint SM partitions (green contexts; CUDA driver API through the
// runtime's entry points), each chain's grids sized to its partition
// (g_sm_budget).  Same kernels, same arithmetic, same results as the
// sequential tsid_core + cur_core; LRB_CUR_SPLIT=<SMs of chain 1> enables it
// (default off, see sm_split).
namespace {
template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
}  // namespace

void release_sm_split(lr_ctx* c) {
  auto& sp = c->split;
  using StreamDestroy = CUresult (*)(CUstream);
  using GreenDestroy = CUresult (*)(CUgreenCtx);
  auto sdestroy = driver_fn<StreamDestroy>("cuStreamDestroy");
  auto gdestroy = driver_fn<GreenDestroy>("cuGreenCtxDestroy");
  if (sdestroy) {
    if (sp.s1) sdestroy(sp.s1);
    if (sp.s2) sdestroy(sp.s2);
  }
  if (gdestroy) {
    if (sp.g1) gdestroy(sp.g1);
    if (sp.g2) gdestroy(sp.g2);
  }
  sp = lr_ctx::SmSplit{};
}

// SMs for the row-ID chain of the concurrent tail, 0 = sequential tail.
// Automatic choice (measured at C4 on the Ozaki engine with the bound-pruned
// CPQR, profiles/r02_cur_split_sweep.jsonl: 123.2 ms sequential, 119.9-120.4 ms
// with 32-48 SMs; with the retry-driven CPQR threshold 40 SMs lead 48 by ~1 ms,
// profiles/r02_cur_split_p_sweep.log): 40 SMs when A^T Q_c runs on the INT8 engine, both
// dimensions are >= 32768 and A has at least 2^31 entries.  On the DMMA engine the A^T Q_c GEMM is 5x longer
// than the row ID, and a static partition would slow it for its whole length.
int tail_sms_wanted(lr_ctx* c, int64_t m, int64_t n, bool host_entry) {
  if (c->tail_sms >= 0) return c->tail_sms;
  if (const char* e = getenv("LRB_CUR_SPLIT")) return std::max(0, atoi(e));
  // under an injected profiler (ncu sets NV_COMPUTE_PROFILER_PERFWORKS_DIR and
  // NV_NSIGHT_INJECTION_* in the child, nsys CUDA_INJECTION64_PATH) the automatic schedule
  // stays sequential: ncu cannot replay kernels launched into green contexts ("Failed to
  // prepare kernel for profiling"), and it serialises launches anyway
  static const bool injected = getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") != nullptr ||
                               getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||
                               getenv("CUDA_INJECTION64_PATH") != nullptr;
  if (injected) return 0;
  // other shapes (profiles/r02_cur_split_shapes.jsonl): 32768 x 65536 74.7 -> 70.6 ms, 65536 x 32768
  // 74.3 -> 72.9, 49152^2 (k = 300) 62.3 -> 61.4, but 32768^2 46.8 -> 47.3: on from 2^31 entries
  // the row ID works on m columns whatever n is, the GEMM chain scales with m n: a tall A
  // (65536 x 32768: 72.9 ms sequential, P = 40: 74.8, 48: 71.6, 56: 69.3, 64: 69.2, 72: 71.6)
  // wants the larger row-ID partition
  if (!(c->gemm_mode == LR_GEMM_OZAKI_INT8 && m >= 32768 && n >= 32768 && m * n >= (int64_t(1) << 31))) return 0;
  if (m > n && n < 49152) return 56;
  // host-pointer entry: the row-ID chain's results (row pivots, row T, R) are downloaded as they
  // become final, so that chain gates the end of the call: 48 SMs (e2e 0.6823-0.6829 s against
  // 0.6845-0.6869 s with 40, which is ~1 ms ahead on the device-resident entry)
  return host_entry ? 48 : 40;
}

bool sm_split(lr_ctx* c, int want) {
  auto& sp = c->split;
  if (want <= 0) return false;
  if (sp.tried && sp.want == want) return sp.ok;
  if (sp.tried) {  // another partition size: rebuild the green contexts
    LRB_CUDA(cudaStreamSynchronize(c->st));
    release_sm_split(c);
  }
  sp.tried = true;
  sp.want = want;
  using DeviceGet = CUresult (*)(CUdevice*, int);
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                             unsigned int);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
  using GreenCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
  using GreenStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
  auto device_get = driver_fn<DeviceGet>("cuDeviceGet");
  auto get_res = driver_fn<GetRes>("cuDeviceGetDevResource");
  auto split = driver_fn<Split>("cuDevSmResourceSplitByCount");
  auto gen = driver_fn<GenDesc>("cuDevResourceGenerateDesc");
  auto gcreate = driver_fn<GreenCreate>("cuGreenCtxCreate");
  auto gstream = driver_fn<GreenStream>("cuGreenCtxStreamCreate");
  if (!device_get || !get_res || !split || !gen || !gcreate || !gstream) return false;
  CUdevice dev;
  CUdevResource all{}, part[1], rest{};
  unsigned nb = 1;
  CUdevResourceDesc d1, d2;
  if (device_get(&dev, c->device) != CUDA_SUCCESS || get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      split(part, &nb, &all, &rest, 0, (unsigned)want) != CUDA_SUCCESS || nb != 1 ||
      gen(&d1, &part[0], 1) != CUDA_SUCCESS || gen(&d2, &rest, 1) != CUDA_SUCCESS ||
      gcreate(&sp.g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      gcreate(&sp.g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      gstream(&sp.s1, sp.g1, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
      gstream(&sp.s2, sp.g2, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    release_sm_split(c);
    sp.tried = true;
    sp.want = want;
    return false;
  }
  sp.n1 = (int)part[0].sm.smCount;
  sp.n2 = (int)rest.sm.smCount;
  sp.ok = sp.n1 >= 8 && sp.n2 >= 8;
  return sp.ok;
}

// Enqueue on a partition stream: the context stream, the call arena's stream
// and the grid budget follow it; timing marks pause (intervals across streams
// mean nothing).  The stream first waits for everything enqueued so far.
struct OnPartition {
  lr_ctx* c;
  cudaStream_t prev_st, prev_ar;
  int prev_budget;
  bool prev_timing;
  OnPartition(lr_ctx* cc, CUstream s, int sms, cudaEvent_t fork) : c(cc) {
    prev_st = c->st;
    prev_ar = c->arena.st;
    prev_budget = g_sm_budget;
    prev_timing = c->timing;
    LRB_CUDA(cudaStreamWaitEvent((cudaStream_t)s, fork, 0));
    c->st = (cudaStream_t)s;
    c->arena.st = (cudaStream_t)s;
    g_sm_budget = sms;
    c->timing = false;
  }
  ~OnPartition() {
    c->st = prev_st;
    c->arena.st = prev_ar;
    g_sm_budget = prev_budget;
    c->timing = prev_timing;
  }
};

cudaEvent_t record_event(cudaStream_t s) {
  cudaEvent_t e;
  LRB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  LRB_CUDA(cudaEventRecord(e, s));
  return e;
}

bool split_applies(lr_ctx* c, int64_t m, int64_t n, int64_t k, int u_mode, bool host_entry = false) {
  return u_mode == LR_U_CPINV_A_RPINV && m >= 16384 && n >= 16384 && k > 192 && k <= 512 &&
         sm_split(c, tail_sms_wanted(c, m, n, host_entry));
}

// tsid_core + cur_core (u_mode LR_U_CPINV_A_RPINV) with the two chains
// concurrent.  on_rows: row pivots / row coefficients / skeleton are final
// (called with c->st = chain 1's stream); on_r: R is final (same).
void tsid_cur_split(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                    const int64_t* col_piv, const double* col_coeff, int64_t ldcc, const lr_solve_strategy& strat,
                    int64_t* row_piv, double* row_coeff, int64_t ldrc, double* skeleton, double thr, double* C,
                    double* U, double* R, const std::function<void()>& on_rows, const std::function<void()>& on_r) {
  if (!(thr > 0.0 && thr < 1.0)) fail(LR_EINVAL, "pinv: threshold must lie in (0,1)");
  c->stats.concurrent_tail = 0;
  const int64_t ldk = even(k), ldct = work_ld(k);
  gather_columns(m, k, a, lda, col_piv, C, m, c->st);
  DBuf<double> Ctp((size_t)ldct * m, c->st), Ct((size_t)ldk * m, c->st);
  zero_pad_rows(c, Ctp, k, ldct, m);
  transpose_matrix(m, k, C, m, Ctp, ldct, c->st);
  copy_matrix(k, m, Ctp, ldct, Ct, ldk, c->st);
  require_rank_in_range(k, k, m, "id_column");
  mark(c, "gather_c");
  DBuf<double> Rc((size_t)k * k, c->st), Rci((size_t)k * k, c->st), Cm((size_t)even(m) * k, c->st);
  copy_matrix(m, k, C, m, Cm, even(m), c->st);
  const bool c_ok = cholqr2(c, m, k, Cm, even(m), Ct, ldk, Rc, Rci, fast_cond_limit(thr));
  mark(c, "cholqr2_c");
  DBuf<double> Qc((size_t)even(m) * k, c->st), Xt((size_t)even(n) * k, c->st);
  DBuf<double> tau(k, c->st), Rt((size_t)even(n) * k, c->st), Rk((size_t)ldk * n, c->st);
  DBuf<double> Sr((size_t)k * k, c->st), Sri((size_t)k * k, c->st), Qr((size_t)even(n) * k, c->st);
  cudaEvent_t fork = record_event(c->st);
  cudaEvent_t done2 = nullptr, done1 = nullptr;
  const auto& sp = c->split;
  // Declared after the buffers, so it runs first when chain 1 throws (e.g. a
  // SingularityError from its coefficient solve): the main stream waits for
  // both partition streams before any buffer above is released in its order.
  struct JoinChains {
    cudaStream_t main, s1, s2;
    cudaEvent_t* ev[3];
    ~JoinChains() {
      for (cudaStream_t s : {s1, s2}) {
        if (!s || s == main) continue;
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) continue;
        cudaEventRecord(e, s);
        cudaStreamWaitEvent(main, e, 0);
        cudaEventDestroy(e);
      }
      for (cudaEvent_t* e : ev)
        if (*e) {
          cudaEventDestroy(*e);
          *e = nullptr;
        }
    }
  } join{c->st, sp.s1, sp.s2, {&fork, &done1, &done2}};
  if (c_ok) {  // chain 2 first: it has no host synchronisation, so it is fully enqueued before chain 1 blocks
    OnPartition on(c, sp.s2, sp.n2, fork);
    gemm(c, m, k, k, Ct, ldk, Rci, k, Qc, even(m), 1.0, 0.0, -1, false, kTriQ);         // Qc = C Rc^-1
    gemm_a(c, n, k, m, a, lda, Qc, even(m), Xt, even(n), 0);  // X^T = A^T Qc
    done2 = record_event(c->st);
  }
  bool r_ok = false;
  // CholeskyQR2 of R^T: DMMA GEMMs that scale with the SM count, so by default
  // they run after the join on the whole GPU and chain 1 keeps only the
  // latency-bound row ID (LRB_CUR_SPLIT_LATE_R=0: inside chain 1's partition)
  static const bool late_r = !(getenv("LRB_CUR_SPLIT_LATE_R") && atoi(getenv("LRB_CUR_SPLIT_LATE_R")) == 0);
  auto factor_r = [&] {
    transpose_matrix(k, n, R, k, Rt, even(n), c->st);
    copy_matrix(k, n, R, k, Rk, ldk, c->st);
    r_ok = cholqr2(c, n, k, Rt, even(n), Rk, ldk, Sr, Sri, fast_cond_limit(thr));
    if (r_ok) gemm(c, n, k, k, Rk, ldk, Sri, k, Qr, even(n), 1.0, 0.0, -1, false, kTriQ);  // Qr = R^T Sr^-1
  };
  {
    OnPartition on(c, sp.s1, sp.n1, fork);
    cpqr_core(c, k, m, Ctp, ldct, k, row_piv, tau, "cpqr_partial", work_padded(k, ldct));
    solve_core(c, k, m - k, Ctp, ldct, Ctp.p + k * ldct, ldct, strat, row_coeff, ldrc, false);
    if (skeleton) gather_rows(k, k, C, m, row_piv, skeleton, k, c->st);
    on_rows();
    gather_rows(k, n, a, lda, row_piv, R, k, c->st);
    on_r();
    if (!late_r) factor_r();
    done1 = record_event(c->st);
  }
  LRB_CUDA(cudaStreamWaitEvent(c->st, done1, 0));
  if (done2) LRB_CUDA(cudaStreamWaitEvent(c->st, done2, 0));
  if (late_r) factor_r();
  mark(c, "tsid_ctA_split");
  if (!(c_ok && r_ok)) {  // rare: the general U path, sequentially
    u_core(c, m, n, k, C, R, col_piv, col_coeff, ldcc, thr, LR_U_CPINV_A_RPINV, U, Ct,
           [&](const double* Q, int64_t ldq, double* X, int64_t ldx) { gemm_a(c, n, k, m, a, lda, Q, ldq, X, ldx, 0); });
    return;
  }
  c->stats.pinv_fast_path = 1;
  c->stats.concurrent_tail = 1;
  DBuf<double> W((size_t)k * k, c->st), t1((size_t)k * k, c->st), tt((size_t)k * k, c->st),
      st((size_t)k * k, c->st);
  gemm(c, k, k, n, Xt, even(n), Qr, even(n), W, k);  // W = Qc^T A Qr
  transpose_matrix(k, k, Rci, k, tt, k, c->st);
  gemm(c, k, k, k, tt, k, W, k, t1, k);              // t1 = Rc^-1 W
  transpose_matrix(k, k, t1, k, tt, k, c->st);
  transpose_matrix(k, k, Sri, k, st, k, c->st);
  gemm(c, k, k, k, tt, k, st, k, U, k);              // U = t1 Sr^-T
  mark(c, "u_small");
}

// cur.hpp:23-34 / lowrank_main.cpp:215 on a dense A given the skeleton index sets
void cur_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const int64_t* col_piv,
              const double* col_coeff, int64_t ldcc, const int64_t* row_piv, double thr, int u_mode, double* C,
              double* U, double* R, const double* Ct_in /* k x m ld even(k), may be null */,
              const std::function<void()>& on_r = {} /* R is final (e.g. start its download) */) {
  if (!(thr > 0.0 && thr < 1.0)) fail(LR_EINVAL, "pinv: threshold must lie in (0,1)");
  gather_columns(m, k, a, lda, col_piv, C, m, c->st);
  gather_rows(k, n, a, lda, row_piv, R, k, c->st);
  if (on_r) on_r();
  u_core(c, m, n, k, C, R, col_piv, col_coeff, ldcc, thr, u_mode, U, Ct_in,
         [&](const double* Q, int64_t ldq, double* Xt, int64_t ldxt) {
           gemm_a(c, n, k, m, a, lda, Q, ldq, Xt, ldxt, 0);
         });
}

void error_core(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const double* C,
                const double* U, const double* R, double* out_host) {
  const int64_t ldk = even(k);
  DBuf<double> Ut((size_t)ldk * k, c->st), Rk((size_t)ldk * n, c->st), UR((size_t)ldk * n, c->st),
      Ct((size_t)ldk * m, c->st);
  transpose_matrix(k, k, U, k, Ut, ldk, c->st);
  copy_matrix(k, n, R, k, Rk, ldk, c->st);
  gemm(c, k, n, k, Ut, ldk, Rk, ldk, UR, ldk);  // UR = U R
  transpose_matrix(m, k, C, m, Ct, ldk, c->st);
  const int tiles = gemm_tn_grid_ctas((int)m, (int)n);
  DBuf<double> part(std::max(tiles, 4 * num_sms()) + 4, c->st), res(2, c->st);
  int np = 0;
  const double* A = a;
  DBuf<double> Apad;
  gemm_tn_resid_sq(c->ws, (int)m, (int)n, (int)k, Ct, ldk, UR, ldk, A, lda, part, &np, c->st);
  sum_partials(part, np, res, c->st);
  frob2(m, n, a, lda, part, res.p + 1, c->st);
  LRB_CUDA(cudaMemcpyAsync(out_host, res.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  out_host[0] = std::sqrt(out_host[0]);
  out_host[1] = std::sqrt(out_host[1]);
}

// host <-> device staging helpers for the plain (host-pointer) entry points
DBuf<double> to_dev(lr_ctx* c, int64_t m, int64_t n, const double* h, int64_t ld, int64_t* ld_out) {
  const int64_t l = even(m);
  DBuf<double> d((size_t)l * n, c->st);
  LRB_CUDA(cudaMemcpy2DAsync(d.p, l * sizeof(double), h, ld * sizeof(double), m * sizeof(double), n,
                             cudaMemcpyHostToDevice, c->st));
  *ld_out = l;
  return d;
}
void to_host(lr_ctx* c, int64_t m, int64_t n, const double* d, int64_t ldd, double* h, int64_t ldh) {
  if (!h || m <= 0 || n <= 0) return;
  LRB_CUDA(cudaMemcpy2DAsync(h, ldh * sizeof(double), d, ldd * sizeof(double), m * sizeof(double), n,
                             cudaMemcpyDeviceToHost, c->st));
}
void idx_to_host(lr_ctx* c, int64_t n, const int64_t* d, int64_t* h) {
  if (h && n > 0) LRB_CUDA(cudaMemcpyAsync(h, d, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->st));
}

cudaStream_t aux_stream(cudaStream_t& s) {
  if (!s) LRB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

bool is_pinned(const void* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Host -> device upload of A (m x n, lda) into d (ld l) in column chunks on
// the upload stream, with the sketch Y = Omega A of each chunk issued on the
// compute stream as soon as that chunk has landed: the PCIe transfer hides
// the sketch (and, on the Ozaki engine, the residue split of A, which is kept
// in the context's cache for the A^T Q contraction of the same call).
void upload_sketch(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double* d, int64_t l, int64_t ell,
                   uint64_t seed, double* Y, int64_t ldy, int kind) {
  cudaStream_t up = aux_stream(c->up_st);
  DBuf<double> omt((size_t)m * even(ell), c->st);
  sketch_operator_t(c, m, ell, kind, seed, omt);
  const bool ordered = srft_dense_fallback(kind, m);
  bool oz = !ordered && c->gemm_mode == LR_GEMM_OZAKI_INT8 && m <= kOzakiMaxK;
  OzakiOperand om;
  int8_t* aplanes = nullptr;
  if (oz) {
    // the cached operand of A, filled chunk by chunk (DMMA when the planes do not fit)
    aplanes = static_cast<int8_t*>(c->ws.try_get(WsSlot::kOzA, ozaki_plane_bytes(m, n)));
    oz = aplanes != nullptr && ozaki_operand(c, m, ell, omt, m, false, 0, om) != nullptr;
  }
  if (oz) {
    c->oz_op.planes = aplanes;
    c->oz_op.shift = static_cast<int*>(c->ws.get(WsSlot::kOzAShift, sizeof(int) * (size_t)n));
    c->oz_op.K = m;
    c->oz_op.cols = n;
    c->oz_op.ld = (m + 15) / 16 * 16;
    c->oz_op.plane_stride = c->oz_op.ld * n;
    c->oz_op.beta = ozaki_beta(m);
    c->oz_op.unsigned_res = m <= kOzakiMaxKUnsigned;
    c->oz_src = d;
    c->oz_K = m;
    c->oz_cols = n;
    c->oz_ld = l;
  }
  mark(c, "omega");
  // ~8 chunks, whole 512-column tiles of the INT8 GEMM; the last full chunk
  // is cut into halving pieces so that the sketch left after the final
  // transfer (the only part not hidden behind PCIe) is one small piece
  const int64_t chunk = std::max<int64_t>(512, ((n + 7) / 8 + 511) / 512 * 512);
  std::vector<int64_t> pieces;
  for (int64_t o = 0; o < n; o += chunk) pieces.push_back(std::min(chunk, n - o));
  int64_t last = pieces.back();
  pieces.pop_back();
  while (last > 1024) {
    const int64_t h = ((last / 2) + 511) / 512 * 512;
    pieces.push_back(h);
    last -= h;
  }
  pieces.push_back(last);
  cudaEvent_t ready;
  LRB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  cudaEvent_t start;
  LRB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  LRB_CUDA(cudaEventRecord(start, c->st));  // d is allocated on the compute stream
  LRB_CUDA(cudaStreamWaitEvent(up, start, 0));
  int64_t off = 0;
  for (const int64_t nc : pieces) {
    LRB_CUDA(cudaMemcpy2DAsync(d + off * l, l * sizeof(double), a + off * lda, lda * sizeof(double),
                               m * sizeof(double), nc, cudaMemcpyHostToDevice, up));
    LRB_CUDA(cudaEventRecord(ready, up));
    LRB_CUDA(cudaStreamWaitEvent(c->st, ready, 0));
    if (oz) {
      const OzakiOperand view = ozaki_cols(c->oz_op, off, nc);
      ozaki_split_into(d + off * l, l, view, c->st);
      ozaki_gemm_tn(c->ws, om, view, ell, nc, Y + off * ldy, ldy, 1.0, 0.0, c->st);
    } else if (ordered) {
      gemm_tn_ordered((int)ell, (int)nc, (int)m, omt, m, d + off * l, l, Y + off * ldy, ldy, c->st);
    } else {
      gemm(c, ell, nc, m, omt, m, d + off * l, l, Y + off * ldy, ldy);
    }
    off += nc;
  }
  cudaEventDestroy(ready);
  cudaEventDestroy(start);
  mark(c, "upload_sketch");
}

// Device -> host copies of finished factors.  Pinned destinations are copied
// on the download stream as soon as their producer has run (overlapping the
// rest of the pipeline); pageable ones are copied at the end on the compute
// stream.  The destructor orders the compute stream after every download, so
// the stream-ordered frees of the device buffers cannot overtake a copy.
struct Downloads {
  lr_ctx* c;
  std::vector<std::function<void()>> deferred;
  bool used = false;
  explicit Downloads(lr_ctx* cc) : c(cc) {}
  void mat(int64_t m, int64_t n, const double* dsrc, int64_t ldd, double* h, int64_t ldh) {
    if (!h || m <= 0 || n <= 0) return;
    if (is_pinned(h)) {
      issue([=](cudaStream_t s) {
        LRB_CUDA(cudaMemcpy2DAsync(h, ldh * sizeof(double), dsrc, ldd * sizeof(double), m * sizeof(double), n,
                                   cudaMemcpyDeviceToHost, s));
      });
    } else {
      deferred.push_back([=] { to_host(c, m, n, dsrc, ldd, h, ldh); });
    }
  }
  void idx(int64_t n, const int64_t* dsrc, int64_t* h) {
    if (!h || n <= 0) return;
    if (is_pinned(h)) {
      issue([=](cudaStream_t s) {
        LRB_CUDA(cudaMemcpyAsync(h, dsrc, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
      });
    } else {
      deferred.push_back([=] { idx_to_host(c, n, dsrc, h); });
    }
  }
  template <class F>
  void issue(F f) {
    cudaStream_t s = aux_stream(c->down_st);
    cudaEvent_t e;
    LRB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    LRB_CUDA(cudaEventRecord(e, c->st));
    LRB_CUDA(cudaStreamWaitEvent(s, e, 0));
    cudaEventDestroy(e);
    f(s);
    used = true;
  }
  void finish() {
    for (auto& f : deferred) f();
    deferred.clear();
  }
  ~Downloads() {
    if (!used) return;
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(e, c->down_st);
      cudaStreamWaitEvent(c->st, e, 0);
      cudaEventDestroy(e);
    }
  }
};

lr_ctx* checked(lr_ctx* c) {
  if (!c) fail(LR_EINVAL, "null lr_ctx");
  LRB_CUDA(cudaSetDevice(c->device));
  // open the call arena (grown to the previous calls' high-water mark)
  Arena& ar = c->arena;
  if (!ar.active) {
    if (ar.want > ar.cap) {
      LRB_CUDA(cudaDeviceSynchronize());
      if (ar.base) LRB_CUDA(cudaFree(ar.base));
      ar.base = nullptr;
      ar.cap = 0;
      const size_t bytes = (ar.want + ar.want / 8 + (64u << 20)) & ~size_t((2u << 20) - 1);
      if (cudaMalloc(reinterpret_cast<void**>(&ar.base), bytes) == cudaSuccess) {
        ar.cap = bytes;
      } else {
        cudaGetLastError();  // no room: this call allocates from the pool
        ar.base = nullptr;
        ar.want = 0;
      }
    }
    ar.used = 0;
    ar.overflow = 0;
    ar.st = c->st;
    ar.active = true;
    tl_arena = &ar;
  }
  return c;
}

void arena_close() {
  Arena* ar = tl_arena;
  if (!ar) return;
  ar->want = std::max(ar->want, ar->used + ar->overflow);
  ar->active = false;
  tl_arena = nullptr;
}

// ---------------------------------------------------------------- column-sharded pipeline (multi-GPU)
// One process per GPU, rank g owning the column block A(:, off_g : off_g + n_g)
// (SURVEY.md section 8e).  Every decision that ends a call (non-finite input,
// escalation, CholeskyQR2 acceptance, singularity) is taken on replicated,
// all-reduced data, so all ranks take it together and no rank is left waiting
// in a collective.
// all ranks agree on a flag (max over ranks)
bool any_rank(lr_ctx* c, bool local) {
  if (!c->comm.comm) return local;
  DBuf<double> f(1, c->st);
  const double v = local ? 1.0 : 0.0;
  LRB_CUDA(cudaMemcpyAsync(f.p, &v, sizeof(double), cudaMemcpyHostToDevice, c->st));
  c->comm.all_reduce_max(f, 1, c->st);
  d2h_mapped(c, c->h_scal, f.p, sizeof(double));
  sync(c);
  return c->h_scal[0] != 0.0;
}

// cpqr.hpp:32-114 on the column-sharded short-wide matrix a (m x n_loc, this
// rank's columns [off, off + n_loc) of m x n_total), `steps` steps; replicated
// perm (n_total) and the sign-fixed top `krows` rows of R in logical order
// (S, krows x n_total, ld krows).
void cpqr_sharded_core(lr_ctx* c, int64_t m, int64_t n_loc, int64_t off, int64_t n_total, const double* a,
                       int64_t lda, int64_t steps, int64_t krows, int64_t* perm, double* S, const char* who,
                       int emulate_shards = 0) {
  require_nonempty(m, n_total, who);
  require_rank_in_range(steps, m, n_total, who);
  const int64_t ldw = even(m);
  DBuf<double> W((size_t)ldw * std::max<int64_t>(n_loc, 1), c->st);
  if (n_loc > 0) copy_matrix(m, n_loc, a, lda, W, ldw, c->st);
  DBuf<int> flags(1, c->st);
  DBuf<long long> rec(1, c->st);
  LRB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), c->st));
  LRB_CUDA(cudaMemsetAsync(rec.p, 0, sizeof(long long), c->st));
  if (emulate_shards > 0)
    cpqr_sharded_emulated(c->ws, emulate_shards, m, n_total, W, ldw, steps, krows, perm, S, krows, flags, rec, c->st);
  else
    cpqr_sharded(c->ws, c->comm, m, n_loc, off, n_total, W, ldw, steps, krows, perm, S, krows, flags, rec, c->st);
  c->comm.all_reduce_sum(reinterpret_cast<int64_t*>(rec.p), 1, c->st);
  d2h_mapped(c, c->h_flags, flags.p, sizeof(int));
  d2h_mapped(c, c->h_ll, rec.p, sizeof(long long));
  sync(c);
  if (any_rank(c, c->h_flags[0] != 0)) fail(LR_EINVAL, std::string(who) + ": matrix has non-finite entries");
  c->stats.cpqr_steps += steps;
  c->stats.norm_recomputes += c->h_ll[0];
}

// sketch.hpp:227-234 (+ lowrank_main.cpp:215 for u_mode LR_U_CPINV_A_RPINV)
// on the column-sharded A.  Replicated outputs: col_pivots (n), row_pivots
// (m), C (m x k), U, col_coeff (k x (n-k)), row_coeff (k x (m-k)), skeleton;
// R_loc (k x n_loc) is this rank's block of R.
void randomized_cur_sharded_core(lr_ctx* c, int64_t m, int64_t n_loc, int64_t off, int64_t n, const double* a,
                                 int64_t lda, int64_t k, const lr_sketch_config& cfg, const lr_solve_strategy& strat,
                                 double thr, int u_mode, int64_t* col_piv, int64_t* row_piv, double* C, double* U,
                                 double* R_loc, double* col_coeff, double* row_coeff, double* skeleton,
                                 const double* Ypre = nullptr, int64_t ldy_pre = 0) {
  const ShardComm& cm = c->comm;
  if (!(thr > 0.0 && thr < 1.0)) fail(LR_EINVAL, "pinv: threshold must lie in (0,1)");
  if (cfg.kind != LR_SKETCH_GAUSSIAN || cfg.power != 0)
    fail(LR_EUNSUPPORTED, "randomized_cur (column-sharded): Gaussian sketch with q = 0 only");
  if (u_mode != LR_U_VT_RPINV && u_mode != LR_U_CPINV_A_RPINV) fail(LR_EINVAL, "randomized_cur: unknown u_mode");
  if (off < 0 || n_loc < 0 || off + n_loc > n) fail(LR_EINVAL, "randomized_cur (column-sharded): bad column block");
  const int64_t ell = check_randomized_id(m, n, k, cfg);
  if (any_rank(c, n_loc > 0 && !device_all_finite(c, m, n_loc, a, lda)))
    fail(LR_EINVAL, "sketch_gaussian: matrix has non-finite entries");
  mark(c, "begin");
  OzakiScope scope(c);  // the shard's residue planes serve the sketch and A^T Q_c
  const int64_t ldk = even(k);
  // (1) Y_g = Omega A_g (Omega from the counter stream: identical on every rank);
  // Ypre: already formed by the caller (the pipelined host upload)
  int64_t ldy = even(ell);
  DBuf<double> Yb;
  const double* Y = Ypre;
  if (Ypre) {
    ldy = ldy_pre;
  } else {
    Yb = DBuf<double>((size_t)ldy * std::max<int64_t>(n_loc, 1), c->st);
    if (n_loc > 0) sketch_core(c, m, n_loc, a, lda, ell, cfg.seed, Yb, ldy);
    Y = Yb;
  }
  // (2) CPQR(Y), ell steps, sharded; T = S11^-1 S12 on the replicated top k rows
  DBuf<double> S1((size_t)k * n, c->st);
  const int emu = c->comm.comm ? 0 : c->emu_shards;
  cpqr_sharded_core(c, ell, n_loc, off, n, Y, ldy, std::min(ell, n), k, col_piv, S1, "cpqr_partial", emu);
  mark(c, "cpqr_sample");
  solve_core(c, k, n - k, S1, k, S1.p + k * k, k, strat, col_coeff, k, false);
  mark(c, "coeff_solve_col");
  // (3) C = A(:, J): owners gather, all-reduce-sum (one non-zero term per entry)
  {
    DBuf<int64_t> idx(k, c->st);
    owned_index(col_piv, k, off, n_loc, idx, c->st);
    gather_columns(m, k, a, lda, idx, C, m, c->st);
    cm.all_reduce_sum(C, (size_t)m * k, c->st);
  }
  mark(c, "gather_c");
  // (4) row ID: CPQR of C^T sharded by row blocks of C, k steps
  const int64_t r0 = m * cm.rank / cm.nranks, m_loc = m * (cm.rank + 1) / cm.nranks - r0;
  {
    DBuf<double> Ct_loc((size_t)ldk * std::max<int64_t>(m_loc, 1), c->st), S1r((size_t)k * m, c->st);
    if (m_loc > 0) transpose_matrix(m_loc, k, C + r0, m, Ct_loc, ldk, c->st);
    cpqr_sharded_core(c, k, m_loc, r0, m, Ct_loc, ldk, k, k, row_piv, S1r, "cpqr_partial", emu);
    mark(c, "cpqr_ct");
    solve_core(c, k, m - k, S1r, k, S1r.p + k * k, k, strat, row_coeff, k, false);
    if (skeleton) gather_rows(k, k, C, m, row_piv, skeleton, k, c->st);
    mark(c, "coeff_solve_row");
  }
  // (5) R_g = A_g(I, :)
  if (n_loc > 0) gather_rows(k, n_loc, a, lda, row_piv, R_loc, k, c->st);
  mark(c, "gather_r");
  // (6) U.  C = Qc Rc (replicated CholeskyQR2); R^T = Qr Sr by CholeskyQR2 with
  // all-reduced Gram matrices over the column blocks
  const int64_t nl = std::max<int64_t>(n_loc, 1), ldn = even(nl);
  DBuf<double> Rt((size_t)ldn * k, c->st), Rk((size_t)ldk * nl, c->st);
  LRB_CUDA(cudaMemsetAsync(Rt.p, 0, sizeof(double) * ldn * k, c->st));
  LRB_CUDA(cudaMemsetAsync(Rk.p, 0, sizeof(double) * ldk * nl, c->st));
  if (n_loc > 0) {
    transpose_matrix(k, n_loc, R_loc, k, Rt, ldn, c->st);
    copy_matrix(k, n_loc, R_loc, k, Rk, ldk, c->st);
  }
  DBuf<double> G((size_t)k * k, c->st), S1i((size_t)k * k, c->st), Q1((size_t)ldn * k, c->st);
  DBuf<double> G2((size_t)k * k, c->st), S2t((size_t)k * k, c->st), Sr((size_t)k * k, c->st),
      Sri((size_t)k * k, c->st);
  DBuf<int> info(2, c->st);
  bool r_ok = true;
  gemm(c, k, k, nl, Rt, ldn, Rt, ldn, G, k);  // R_g R_g^T
  cm.all_reduce_sum(G, (size_t)k * k, c->st);
  cholesky_upper(c->ws, k, G, k, info, c->st);
  d2h_mapped(c, c->h_flags, info.p, sizeof(int));
  sync(c);
  r_ok = c->h_flags[0] == 0;
  if (r_ok) {
    tri_upper_inverse_blocked(k, G, k, S1i, k, c->st);
    gemm(c, nl, k, k, Rk, ldk, S1i, k, Q1, ldn, 1.0, 0.0, -1, false, kTriQ);  // Q1_g = R_g^T S1^-1
    gemm(c, k, k, nl, Q1, ldn, Q1, ldn, G2, k);
    cm.all_reduce_sum(G2, (size_t)k * k, c->st);
    cholesky_upper(c->ws, k, G2, k, info.p + 1, c->st);
    d2h_mapped(c, c->h_flags + 1, info.p + 1, sizeof(int));
    sync(c);
    r_ok = c->h_flags[1] == 0;
  }
  if (r_ok) {
    transpose_matrix(k, k, G2, k, S2t, k, c->st);
    gemm(c, k, k, k, S2t, k, G, k, Sr, k);  // Sr = S2 S1
    tri_upper_inverse_blocked(k, Sr, k, Sri, k, c->st);
    DBuf<double> part(4 * num_sms() + 4, c->st), f(2, c->st);
    frob2(k, k, Sr, k, part, f, c->st);
    frob2(k, k, Sri, k, part, f.p + 1, c->st);
    d2h_mapped(c, c->h_scal, f.p, 2 * sizeof(double));
    sync(c);
    const double cb = std::sqrt(c->h_scal[0]) * std::sqrt(c->h_scal[1]);
    r_ok = std::isfinite(cb) && cb < fast_cond_limit(thr);
  }
  mark(c, "cholqr2_r");
  // local rows of R^+ (n_loc x k, ld ldn): Qr_g Sr^-T on the fast path
  // (R^T = Qr Sr => R^+ = Qr Sr^-T), else rows of the truncated pseudoinverse of
  // the all-gathered R (svd.hpp:193-207, Jacobi route)
  DBuf<double> Rp_loc((size_t)ldn * k, c->st);
  LRB_CUDA(cudaMemsetAsync(Rp_loc.p, 0, sizeof(double) * ldn * k, c->st));
  DBuf<double> Qr;
  if (r_ok) {
    Qr = DBuf<double>((size_t)ldn * k, c->st);
    gemm(c, nl, k, k, Rk, ldk, Sri, k, Qr, ldn, 1.0, 0.0, -1, false, kTriQ);  // Qr_g = R_g^T Sr^-1
  } else {
    DBuf<double> Rfull((size_t)k * n, c->st), Rp((size_t)n * k, c->st);
    LRB_CUDA(cudaMemsetAsync(Rfull.p, 0, sizeof(double) * k * n, c->st));
    if (n_loc > 0) copy_matrix(k, n_loc, R_loc, k, Rfull.p + off * k, k, c->st);
    cm.all_reduce_sum(Rfull, (size_t)k * n, c->st);
    pinv_core(c, k, n, Rfull, k, thr, Rp, n);
    if (n_loc > 0) copy_matrix(n_loc, k, Rp.p + off, n, Rp_loc, ldn, c->st);
  }
  auto rp_from_qr = [&] {
    DBuf<double> srt((size_t)k * k, c->st), Qrt((size_t)ldk * nl, c->st);
    transpose_matrix(k, k, Sri, k, srt, k, c->st);
    transpose_matrix(nl, k, Qr, ldn, Qrt, ldk, c->st);
    gemm(c, nl, k, k, Qrt, ldk, srt, k, Rp_loc, ldn);  // R^+_g = Qr_g Sr^-T
  };
  if (u_mode == LR_U_CPINV_A_RPINV) {
    DBuf<double> Ct((size_t)ldk * m, c->st), Cm((size_t)even(m) * k, c->st), Rc((size_t)k * k, c->st),
        Rci((size_t)k * k, c->st);
    transpose_matrix(m, k, C, m, Ct, ldk, c->st);
    copy_matrix(m, k, C, m, Cm, even(m), c->st);
    const bool c_ok = cholqr2(c, m, k, Cm, even(m), Ct, ldk, Rc, Rci, fast_cond_limit(thr));
    mark(c, "cholqr2_c");
    DBuf<double> Xt((size_t)ldn * k, c->st), W((size_t)k * k, c->st);
    LRB_CUDA(cudaMemsetAsync(Xt.p, 0, sizeof(double) * ldn * k, c->st));
    if (c_ok && r_ok) {
      c->stats.pinv_fast_path = 1;
      // U = Rc^-1 (Qc^T A Qr) Sr^-T with W = sum_g (A_g^T Qc)^T Qr_g
      DBuf<double> Qc((size_t)even(m) * k, c->st);
      gemm(c, m, k, k, Ct, ldk, Rci, k, Qc, even(m), 1.0, 0.0, -1, false, kTriQ);  // Qc = C Rc^-1
      mark(c, "form_q");
      if (n_loc > 0) gemm_a(c, nl, k, m, a, lda, Qc, even(m), Xt, ldn, 0);       // X_g^T = A_g^T Qc
      mark(c, "ctA_gemm");
      gemm(c, k, k, nl, Xt, ldn, Qr, ldn, W, k);
      cm.all_reduce_sum(W, (size_t)k * k, c->st);
      DBuf<double> t1((size_t)k * k, c->st), tt((size_t)k * k, c->st), st2((size_t)k * k, c->st);
      transpose_matrix(k, k, Rci, k, tt, k, c->st);
      gemm(c, k, k, k, tt, k, W, k, t1, k);  // Rc^-1 W
      transpose_matrix(k, k, t1, k, tt, k, c->st);
      transpose_matrix(k, k, Sri, k, st2, k, c->st);
      gemm(c, k, k, k, tt, k, st2, k, U, k);  // (Rc^-1 W) Sr^-T
    } else {
      // U = sum_g (C^+ A_g) R^+_g with the replicated truncated C^+ (Jacobi route)
      c->stats.pinv_fast_path = 0;
      if (r_ok) rp_from_qr();
      DBuf<double> Cp((size_t)k * m, c->st), Cpt((size_t)even(m) * k, c->st);
      pinv_core(c, m, k, C, m, thr, Cp, k);
      transpose_matrix(k, m, Cp, k, Cpt, even(m), c->st);
      if (n_loc > 0) gemm_a(c, nl, k, m, a, lda, Cpt, even(m), Xt, ldn, 0);  // X_g^T = A_g^T C^+T
      mark(c, "ctA_gemm");
      gemm(c, k, k, nl, Xt, ldn, Rp_loc, ldn, U, k);
      cm.all_reduce_sum(U, (size_t)k * k, c->st);
    }
  } else {
    // u = basis()^T R^+ (cur.hpp:30) = sum_g B_g R^+_g, B_g = the basis rows of the owned columns
    if (r_ok) rp_from_qr();
    c->stats.pinv_fast_path = r_ok ? 1 : 0;
    DBuf<int64_t> inv(n, c->st);
    inverse_perm(col_piv, n, inv, c->st);
    DBuf<double> B((size_t)k * nl, c->st), Bt((size_t)ldn * k, c->st);
    LRB_CUDA(cudaMemsetAsync(Bt.p, 0, sizeof(double) * ldn * k, c->st));
    if (n_loc > 0) {
      basis_rows(inv, off, n_loc, k, col_coeff, k, B, c->st);
      transpose_matrix(k, n_loc, B, k, Bt, ldn, c->st);
    }
    gemm(c, k, k, nl, Bt, ldn, Rp_loc, ldn, U, k);  // U = B_g R^+_g
    cm.all_reduce_sum(U, (size_t)k * k, c->st);
  }
  mark(c, "u_small");
}

// ---------------------------------------------------------------- verifiers (verify.hpp:14-166) at scale
// The reference evaluates every spectral norm as sigma_1 of a full Jacobi SVD
// of the materialised m x n residual (svd.hpp:185-189, verify.hpp:39-124).
// Here the residuals stay operators (E = A - X Y applied to blocks of
// vectors through A, A^T, X, Y) and sigma_1 comes from a block Krylov
// iteration on E^T E: a seeded Gaussian start block, every Krylov block made
// orthonormal against the basis (block Gram-Schmidt twice, then CholeskyQR2 /
// Householder), Ritz value sigma_1 = sqrt(lambda_max(Z^T Z)) with Z = E K over
// the whole basis (Jacobi SVD of the small Gram matrix).  It increases
// monotonically to sigma_1(E) and stops when two consecutive values agree to
// 1e-14 relative or the basis is exhausted.
using BlockOp = std::function<void(int64_t r, const double* in, int64_t ldi, double* out, int64_t ldo)>;

double krylov_sigma1(lr_ctx* c, int64_t rows, int64_t cols, const BlockOp& E, const BlockOp& Et, uint64_t seed,
                     int64_t b = 32, int qmax = 12) {
  const int64_t cap = std::min<int64_t>((int64_t)(qmax + 1) * b, std::min(rows, cols));
  if (cap < 1) return 0.0;
  b = std::min(b, cap);
  const int64_t ldk = even(cols), ldz = even(rows), ldkt = even(cap);
  DBuf<double> K((size_t)ldk * cap, c->st), Kt((size_t)ldkt * cols, c->st), Z((size_t)ldz * cap, c->st);
  DBuf<double> blk((size_t)ldk * b, c->st), H((size_t)ldkt * b, c->st), part(4 * num_sms() + 4, c->st),
      nrm(2, c->st);
  gaussian_matrix(cols, b, seed, blk, ldk, false, c->st);
  int64_t nb = 0;
  double prev = -1.0, est = 0.0;
  for (int it = 0; it <= qmax && nb < cap; ++it) {
    const int64_t r0 = std::min(b, cap - nb);
    // block Gram-Schmidt (twice) against the basis; a block that vanishes
    // against it means the Krylov space is exhausted
    frob2(cols, r0, blk, ldk, part, nrm, c->st);
    for (int pass = 0; pass < 2 && nb > 0; ++pass) {
      gemm(c, nb, r0, cols, K, ldk, blk, ldk, H, ldkt);                  // H = K^T blk
      gemm(c, cols, r0, nb, Kt, ldkt, H, ldkt, blk, ldk, -1.0, 1.0);      // blk -= K H
    }
    frob2(cols, r0, blk, ldk, part, nrm.p + 1, c->st);
    d2h_mapped(c, c->h_scal, nrm.p, 2 * sizeof(double));
    sync(c);
    if (!(c->h_scal[1] > 1e-24 * c->h_scal[0]) || c->h_scal[1] == 0.0) break;
    const int64_t r = orth_cols_core(c, cols, r0, blk, ldk, K.p + nb * ldk, ldk);
    if (r < 1) break;
    transpose_matrix(cols, r, K.p + nb * ldk, ldk, Kt.p + nb, ldkt, c->st);
    E(r, K.p + nb * ldk, ldk, Z.p + nb * ldz, ldz);  // Z(:, new) = E K(:, new)
    const int64_t nb_new = nb + r;
    DBuf<double> G((size_t)nb_new * nb_new, c->st), u((size_t)nb_new * nb_new, c->st), s(nb_new, c->st),
        v((size_t)nb_new * nb_new, c->st);
    gemm(c, nb_new, nb_new, rows, Z, ldz, Z, ldz, G, nb_new);  // Z^T Z
    svd_core(c, nb_new, nb_new, G, nb_new, u, s, v);
    d2h_mapped(c, c->h_scal, s.p, sizeof(double));
    sync(c);
    est = std::sqrt(std::max(0.0, c->h_scal[0]));
    if (prev >= 0.0 && std::abs(est - prev) <= 1e-14 * est) break;
    prev = est;
    // next block: E^T E applied to the newest block
    Et(r, Z.p + nb * ldz, ldz, blk, ldk);
    nb = nb_new;
    if (r < b) break;
  }
  return est;
}

// E = A - X Y (X m x k, Y k x n; k = 0: E = A) as a block operator.  At is A^T
// (n x m, ld ldat): the column-major A serves E^T U = A^T U - Y^T (X^T U)
// directly and At serves E V = A V - X (Y V) on the same GEMM.
struct ResidualOp {
  lr_ctx* c;
  int64_t m, n, k;
  const double *A, *At, *X, *Xt, *Y, *Yt;
  int64_t lda, ldat, ldx, ldxt, ldy, ldyt;
  void apply(int64_t r, const double* V, int64_t ldv, double* out, int64_t ldo) const {
    gemm(c, m, r, n, At, ldat, V, ldv, out, ldo);  // A V
    if (k > 0) {
      DBuf<double> t((size_t)k * r, c->st);
      gemm(c, k, r, n, Yt, ldyt, V, ldv, t, k);            // Y V
      gemm(c, m, r, k, Xt, ldxt, t, k, out, ldo, -1.0, 1.0);  // -= X (Y V)
    }
  }
  void apply_t(int64_t r, const double* U, int64_t ldu, double* out, int64_t ldo) const {
    gemm(c, n, r, m, A, lda, U, ldu, out, ldo);  // A^T U
    if (k > 0) {
      DBuf<double> t((size_t)k * r, c->st);
      gemm(c, k, r, m, X, ldx, U, ldu, t, k);               // X^T U
      gemm(c, n, r, k, Y, ldy, t, k, out, ldo, -1.0, 1.0);  // -= Y^T (X^T U)
    }
  }
};

// the transposes a ResidualOp needs, owned
struct ResidualBufs {
  DBuf<double> Xt, Yt;
};
ResidualOp residual_op(lr_ctx* c, int64_t m, int64_t n, const double* A, int64_t lda, const double* At,
                       int64_t ldat, int64_t k, const double* X, int64_t ldx, const double* Y, int64_t ldy,
                       ResidualBufs& bufs) {
  ResidualOp op{c, m, n, k, A, At, X, nullptr, Y, nullptr, lda, ldat, ldx, even(k), ldy, even(n)};
  if (k > 0) {
    bufs.Xt = DBuf<double>((size_t)even(k) * m, c->st);
    bufs.Yt = DBuf<double>((size_t)even(n) * k, c->st);
    transpose_matrix(m, k, X, ldx, bufs.Xt, even(k), c->st);
    transpose_matrix(k, n, Y, ldy, bufs.Yt, even(n), c->st);
    op.Xt = bufs.Xt;
    op.Yt = bufs.Yt;
  }
  return op;
}

double op_sigma1(lr_ctx* c, const ResidualOp& op, uint64_t seed) {
  return krylov_sigma1(
      c, op.m, op.n, [&](int64_t r, const double* i, int64_t li, double* o, int64_t lo) { op.apply(r, i, li, o, lo); },
      [&](int64_t r, const double* i, int64_t li, double* o, int64_t lo) { op.apply_t(r, i, li, o, lo); }, seed);
}

// ||A - X Y||_F by the fused residual GEMM (never forms X Y)
double residual_frob(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const double* X,
                     int64_t ldx, const double* Y, int64_t ldy) {
  DBuf<double> part(4 * num_sms() + 4, c->st), res(2, c->st);
  if (k == 0) {
    frob2(m, n, a, lda, part, res, c->st);
  } else {
    const int64_t ldk = even(k);
    DBuf<double> Xt((size_t)ldk * m, c->st), Yk((size_t)ldk * n, c->st);
    transpose_matrix(m, k, X, ldx, Xt, ldk, c->st);
    copy_matrix(k, n, Y, ldy, Yk, ldk, c->st);
    const int tiles = gemm_tn_grid_ctas((int)m, (int)n);
    DBuf<double> parts(std::max(tiles, 4 * num_sms()) + 4, c->st);
    int np = 0;
    gemm_tn_resid_sq(c->ws, (int)m, (int)n, (int)k, Xt, ldk, Yk, ldk, a, lda, parts, &np, c->st);
    sum_partials(parts, np, res, c->st);
  }
  d2h_mapped(c, c->h_scal, res.p, sizeof(double));
  sync(c);
  return std::sqrt(c->h_scal[0]);
}

// the pieces of the verifiers: A^T, C = A(:, J), V^T = basis()^T (k x n), R = A(I, :), W^T (k x m)
struct VerifyParts {
  DBuf<double> At, C, Vt, R, Wt, W;
};
void basis_t(lr_ctx* c, int64_t n, int64_t k, const int64_t* piv, const double* coeff, int64_t ldc, double* out) {
  DBuf<int64_t> inv(n, c->st);
  inverse_perm(piv, n, inv, c->st);
  basis_rows(inv, 0, n, k, coeff, ldc, out, c->st);  // out (k x n): column j = basis() row j
}
// ||T||_2 of a k x nc coefficient block (ld ldt): sqrt(lambda_max(T T^T)) (Jacobi SVD of the k x k Gram)
double coeff_norm2(lr_ctx* c, int64_t k, int64_t nc, const double* t, int64_t ldt) {
  if (nc == 0) return 0.0;
  DBuf<double> Tt((size_t)even(nc) * k, c->st), G((size_t)k * k, c->st), u((size_t)k * k, c->st), s(k, c->st),
      v((size_t)k * k, c->st);
  transpose_matrix(k, nc, t, ldt, Tt, even(nc), c->st);
  gemm(c, k, k, nc, Tt, even(nc), Tt, even(nc), G, k);
  svd_core(c, k, k, G, k, u, s, v);
  d2h_mapped(c, c->h_scal, s.p, sizeof(double));
  sync(c);
  return std::sqrt(std::max(0.0, c->h_scal[0]));
}

constexpr uint64_t kVerifySeed = 0x5eed1412ull;

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* lr_last_error(void) { return g_err.c_str(); }
int64_t lr_last_singular_index(void) { return g_sing; }

lr_solve_strategy lr_solve_strategy_default(void) { return {LR_SOLVE_BACKSUB, 1e-12, 0.0, 1}; }
lr_sketch_config lr_sketch_config_default(void) { return {LR_SKETCH_GAUSSIAN, 10, 0, 0, 1, 0}; }

int lr_ctx_create(lr_ctx** out, int device) {
  return guard([&] {
    if (!out) fail(LR_EINVAL, "lr_ctx_create: null output");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
      throw CudaError("lr_ctx_create: no CUDA device " + std::to_string(device));
    cudaDeviceProp prop;
    LRB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError("lr_ctx_create: sm_100 (B200) device required");
    LRB_CUDA(cudaSetDevice(device));
    auto* c = new lr_ctx();
    c->device = device;
    LRB_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->st = c->own;
    LRB_CUDA(cudaMallocHost(&c->h_flags, 64));
    LRB_CUDA(cudaMallocHost(&c->h_scal, 64));
    LRB_CUDA(cudaMallocHost(&c->h_ll, 64));
    cudaMemPool_t pool;
    LRB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    LRB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = c;
  });
}

int lr_ctx_destroy(lr_ctx* c) {
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    cudaDeviceSynchronize();
    c->ws.release_all();
    c->ws_side.release_all();
    if (c->arena.base) cudaFree(c->arena.base);
    cudaFreeHost(c->h_flags);
    cudaFreeHost(c->h_scal);
    cudaFreeHost(c->h_ll);
    if (c->up_st) cudaStreamDestroy(c->up_st);
    if (c->down_st) cudaStreamDestroy(c->down_st);
    if (c->side_st) cudaStreamDestroy(c->side_st);
    release_sm_split(c);
    nccl_comm_destroy(c->comm.comm);
    cudaStreamDestroy(c->own);
    delete c;
  });
}

int lr_ctx_set_stream(lr_ctx* c, void* s) {
  // NULL is the CUDA legacy default stream (what torch reports for its default stream)
  return guard([&] {
    const cudaStream_t ns = s ? static_cast<cudaStream_t>(s) : cudaStreamLegacy;
    // the call arena is reused in stream order: finish the old stream's work first
    if (checked(c)->st != ns) LRB_CUDA(cudaStreamSynchronize(c->st));
    c->st = ns;
  });
}
int lr_ctx_set_gemm_mode(lr_ctx* c, int mode) {
  return guard([&] {
    checked(c);
    if (mode != LR_GEMM_DMMA && mode != LR_GEMM_OZAKI_INT8) fail(LR_EINVAL, "set_gemm_mode: unknown mode");
    c->gemm_mode = mode;
  });
}
int lr_ctx_get_gemm_mode(lr_ctx* c) { return c ? c->gemm_mode : -1; }
int lr_ctx_set_concurrent_tail(lr_ctx* c, int sms) {
  return guard([&] {
    checked(c);
    if (sms < -1) fail(LR_EINVAL, "set_concurrent_tail: sms must be -1 (automatic), 0 (off) or an SM count");
    c->tail_sms = sms;
  });
}
int lr_ctx_cache_operand(lr_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "cache_operand");
    require_ld(m, lda, "cache_operand");
    c->oz_pinned = true;
    c->oz_cache_on = true;
    if (c->pin_src != a || c->pin_K != m || c->pin_cols != n || c->pin_ld != lda) c->oz_src = nullptr;
    c->pin_src = a;
    c->pin_K = m;
    c->pin_cols = n;
    c->pin_ld = lda;
  });
}
// frees the grow-only workspace (Ozaki residue planes, CPQR state, ...) and the
// call arena; the next call grows them again
int lr_ctx_release_workspace(lr_ctx* c) {
  return guard([&] {
    checked(c);
    LRB_CUDA(cudaStreamSynchronize(c->st));
    if (c->side_st) LRB_CUDA(cudaStreamSynchronize(c->side_st));
    c->ws.release_all();
    c->ws_side.release_all();
    c->oz_src = nullptr;
    c->oz_pinned = false;
    c->oz_cache_on = false;
    c->pin_src = nullptr;
    if (c->arena.base) {
      LRB_CUDA(cudaFree(c->arena.base));
      c->arena.base = nullptr;
      c->arena.cap = c->arena.used = c->arena.overflow = c->arena.want = 0;
    }
  });
}
int lr_ctx_clear_operand_cache(lr_ctx* c) {
  return guard([&] {
    checked(c);
    c->oz_pinned = false;
    c->oz_cache_on = false;
    c->oz_src = nullptr;
    c->pin_src = nullptr;
  });
}
int lr_ctx_use_own_stream(lr_ctx* c) {
  return guard([&] {
    if (checked(c)->st != c->own) LRB_CUDA(cudaStreamSynchronize(c->st));
    c->st = c->own;
  });
}
int lr_ctx_get_stats(lr_ctx* c, lr_stats* out) {
  return guard([&] { *out = checked(c)->stats; });
}
int lr_ctx_synchronize(lr_ctx* c) {
  return guard([&] { sync(checked(c)); });
}

// rng.hpp:74-94
int lr_gaussian_matrix_d(lr_ctx* c, int64_t rows, int64_t cols, uint64_t seed, double* out, int64_t ldo) {
  return guard([&] {
    checked(c);
    if (rows < 1 || cols < 1) fail(LR_EINVAL, "gaussian_matrix: dimensions must be positive");
    gaussian_matrix(rows, cols, seed, out, ldo, false, c->st);
  });
}
int lr_gaussian_matrix(lr_ctx* c, int64_t rows, int64_t cols, uint64_t seed, double* out) {
  return guard([&] {
    checked(c);
    if (rows < 1 || cols < 1) fail(LR_EINVAL, "gaussian_matrix: dimensions must be positive");
    DBuf<double> d((size_t)rows * cols, c->st);
    gaussian_matrix(rows, cols, seed, d, rows, false, c->st);
    to_host(c, rows, cols, d, rows, out, rows);
    sync(c);
  });
}

// sketch.hpp:67-78
int lr_sketch_gaussian_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed,
                         double* y, int64_t ldy) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "sketch_gaussian");
    require_ld(m, lda, "sketch_gaussian");
    if (!device_all_finite(c, m, n, a, lda)) fail(LR_EINVAL, "sketch_gaussian: matrix has non-finite entries");
    require_sample_count(ell, m, "sketch_gaussian");
    sketch_core(c, m, n, a, lda, ell, seed, y, ldy);
  });
}
int lr_sketch_gaussian(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed,
                       double* y) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "sketch_gaussian");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    if (!device_all_finite(c, m, n, d, l)) fail(LR_EINVAL, "sketch_gaussian: matrix has non-finite entries");
    require_sample_count(ell, m, "sketch_gaussian");
    DBuf<double> yd((size_t)ell * n, c->st);
    sketch_core(c, m, n, d, l, ell, seed, yd, ell);
    to_host(c, ell, n, yd, ell, y, ell);
    sync(c);
  });
}

// sketch.hpp:84-100 srft_operator: out (ell x m, ld ell), host
int lr_srft_operator(lr_ctx* c, int64_t m, int64_t ell, uint64_t seed, double* out) {
  return guard([&] {
    checked(c);
    require_sample_count(ell, m, "srft_operator");
    DBuf<double> omt((size_t)m * ell, c->st), om((size_t)ell * m, c->st);
    sketch_operator_t(c, m, ell, LR_SKETCH_SRFT, seed, omt);
    transpose_matrix(m, ell, omt, m, om, ell, c->st);
    to_host(c, ell, m, om, ell, out, ell);
    sync(c);
  });
}

// svd.hpp:216-235 orth_rows: out (first *r rows of ell x n, ld ell), host
int lr_orth_rows(lr_ctx* c, int64_t ell, int64_t n, const double* y, int64_t ldy, double* out, int64_t* r) {
  return guard([&] {
    checked(c);
    require_nonempty(ell, n, "orth_rows");
    int64_t l;
    DBuf<double> d = to_dev(c, ell, n, y, ldy, &l);
    const int64_t ldn = even(n);
    DBuf<double> Yt((size_t)ldn * ell, c->st), Q((size_t)ldn * ell, c->st), Qt((size_t)ell * n, c->st);
    transpose_matrix(ell, n, d, l, Yt, ldn, c->st);
    const int64_t rr = orth_cols_core(c, n, ell, Yt, ldn, Q, ldn);
    if (rr > 0) {
      transpose_matrix(n, rr, Q, ldn, Qt, rr, c->st);
      to_host(c, rr, n, Qt, rr, out, ell);
    }
    sync(c);
    *r = rr;
  });
}

// sketch.hpp:238-254 randomized_svd: u (m x k), sigma (k), v (n x k), all host
int lr_randomized_svd(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_sketch_config cfg,
                      double* u, double* sigma, double* v) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "randomized_svd");
    require_rank_in_range(k, m, n, "randomized_svd");
    int64_t ell = check_randomized_id(m, n, k, cfg);
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    int64_t ldy = work_ld(ell);
    DBuf<double> Y((size_t)ldy * n, c->st);
    zero_pad_rows(c, Y, ell, ldy, n);
    sketch_core(c, m, n, d, l, ell, cfg.seed, Y, ldy, cfg.kind);
    if (cfg.power > 0) power_rounds_core(c, m, n, d, l, cfg.power, cfg.reorthonormalize != 0, Y, ldy, ell);
    // q = orth_rows(y): Q_y = q^T (n x r)
    const int64_t ldn = even(n);
    DBuf<double> Yt((size_t)ldn * ell, c->st), Qy((size_t)ldn * ell, c->st);
    transpose_matrix(ell, n, Y, ldy, Yt, ldn, c->st);
    const int64_t r = orth_cols_core(c, n, ell, Yt, ldn, Qy, ldn);
    if (r < k) fail(LR_ERUNTIME, "randomized_svd: sample rank collapsed below target rank");
    // projected = a q^T (m x r) = (A^T)^T Q_y with A^T materialised (K = n contiguous)
    DBuf<double> At((size_t)ldn * m, c->st), Pm((size_t)even(m) * r, c->st);
    transpose_matrix(m, n, d, l, At, ldn, c->st);
    gemm(c, m, r, n, At, ldn, Qy, ldn, Pm, even(m));
    const int64_t rr = std::min(m, r);
    DBuf<double> su((size_t)m * rr, c->st), ss(rr, c->st), sv((size_t)r * rr, c->st);
    svd_core(c, m, r, Pm, even(m), su, ss, sv);
    // v = q^T small.v(:, :k): out (n x k) = P^T Q with P = Q_y^T (r x n), Q = small.v (r x k)
    DBuf<double> Qyt((size_t)even(r) * n, c->st), vd((size_t)n * k, c->st);
    transpose_matrix(n, r, Qy, ldn, Qyt, even(r), c->st);
    gemm(c, n, k, r, Qyt, even(r), sv, r, vd, n);
    to_host(c, m, k, su, m, u, m);
    to_host(c, k, 1, ss, k, sigma, k);
    to_host(c, n, k, vd, n, v, n);
    sync(c);
  });
}

// sketch.hpp:110-143: y (ell x n, ld ell)
int lr_sketch_srft(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, uint64_t seed,
                   double* y) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "sketch_srft");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    if (!device_all_finite(c, m, n, d, l)) fail(LR_EINVAL, "sketch_srft: matrix has non-finite entries");
    require_sample_count(ell, m, "sketch_srft");
    DBuf<double> yd((size_t)ell * n, c->st);
    sketch_core(c, m, n, d, l, ell, seed, yd, ell, LR_SKETCH_SRFT);
    to_host(c, ell, n, yd, ell, y, ell);
    sync(c);
  });
}

// sketch.hpp:148-164: y (ell x n, ld ell; first *rows rows valid)
int lr_sketch_power(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t ell, int q, int reorth,
                    uint64_t seed, double* y, int64_t* rows) {
  return guard([&] {
    checked(c);
    if (q < 0) fail(LR_EINVAL, "sketch_power: q must be nonnegative");
    require_nonempty(m, n, "sketch_gaussian");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    if (!device_all_finite(c, m, n, d, l)) fail(LR_EINVAL, "sketch_gaussian: matrix has non-finite entries");
    require_sample_count(ell, m, "sketch_gaussian");
    int64_t ldy = work_ld(ell), r = ell;
    DBuf<double> yd((size_t)ldy * n, c->st);
    zero_pad_rows(c, yd, ell, ldy, n);
    sketch_core(c, m, n, d, l, ell, seed, yd, ldy);
    if (q > 0) power_rounds_core(c, m, n, d, l, q, reorth != 0, yd, ldy, r);
    to_host(c, r, n, yd, ldy, y, ell);
    sync(c);
    *rows = r;
  });
}

// cpqr.hpp:32-114
int lr_cpqr_partial_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, double* q, double* s,
                      int64_t* pivots) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "cpqr_partial");
    if (!device_all_finite(c, m, n, a, lda)) fail(LR_EINVAL, "cpqr_partial: matrix has non-finite entries");
    require_rank_in_range(k, m, n, "cpqr_partial");
    const int64_t ldw = work_ld(m);
    DBuf<double> W((size_t)ldw * n, c->st), tau(k, c->st);
    zero_pad_rows(c, W, m, ldw, n);
    copy_matrix(m, n, a, lda, W, ldw, c->st);
    cpqr_core(c, m, n, W, ldw, k, pivots, tau, "cpqr_partial", work_padded(m, ldw));
    cpqr_extract_s(m, n, W, ldw, k, s, k, c->st);
    if (q) cpqr_form_q(m, n, W, ldw, k, tau, q, m, c->st);
  });
}
int lr_cpqr_partial(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, double* q, double* s,
                    int64_t* pivots) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "cpqr_partial");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    if (!device_all_finite(c, m, n, d, l)) fail(LR_EINVAL, "cpqr_partial: matrix has non-finite entries");
    require_rank_in_range(k, m, n, "cpqr_partial");
    DBuf<double> tau(k, c->st), sd((size_t)k * n, c->st), qd(q ? (size_t)m * k : 1, c->st);
    DBuf<int64_t> pd(n, c->st);
    const int64_t lw = work_ld(m);
    DBuf<double> W((size_t)lw * n, c->st);
    zero_pad_rows(c, W, m, lw, n);
    copy_matrix(m, n, d, l, W, lw, c->st);
    cpqr_core(c, m, n, W, lw, k, pd, tau, "cpqr_partial", work_padded(m, lw));
    cpqr_extract_s(m, n, W, lw, k, sd, k, c->st);
    if (q) cpqr_form_q(m, n, W, lw, k, tau, qd, m, c->st);
    to_host(c, k, n, sd, k, s, k);
    if (q) to_host(c, m, k, qd, m, q, m);
    idx_to_host(c, n, pd, pivots);
    sync(c);
  });
}
int lr_cpqr_full(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double* q, double* s,
                 int64_t* pivots) {
  if (m < 1 || n < 1) {
    g_err = "cpqr_full: matrix must be nonempty";
    return LR_EINVAL;
  }
  return lr_cpqr_partial(c, m, n, a, lda, std::min(m, n), q, s, pivots);
}

// solve.hpp:104-145
int lr_stabilized_coeff_solve(lr_ctx* c, int64_t k, int64_t nc, const double* s11, int64_t ld11, const double* s12,
                              int64_t ld12, lr_solve_strategy strat, double* t) {
  return guard([&] {
    checked(c);
    if (k < 0 || nc < 0) fail(LR_EINVAL, "stabilized_coeff_solve: row count mismatch");
    if (k == 0) return;
    int64_t l11, l12 = even(k);
    DBuf<double> d11 = to_dev(c, k, k, s11, ld11, &l11);
    DBuf<double> d12 = nc > 0 ? to_dev(c, k, nc, s12, ld12, &l12) : DBuf<double>(1, c->st);
    DBuf<double> td((size_t)k * std::max<int64_t>(nc, 1), c->st);
    solve_core(c, k, nc, d11, l11, d12, l12, strat, td, k, true);
    to_host(c, k, nc, td, k, t, k);
    sync(c);
  });
}

// svd.hpp:132-183 / 193-207
int lr_svd(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double* u, double* sigma, double* v) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "svd");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    if (!device_all_finite(c, m, n, d, l)) fail(LR_EINVAL, "svd: matrix has non-finite entries");
    const int64_t r = std::min(m, n);
    DBuf<double> ud((size_t)m * r, c->st), sd(r, c->st), vd((size_t)n * r, c->st);
    svd_core(c, m, n, d, l, ud, sd, vd);
    to_host(c, m, r, ud, m, u, m);
    to_host(c, r, 1, sd, r, sigma, r);
    to_host(c, n, r, vd, n, v, n);
    sync(c);
  });
}
int lr_pinv(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double thr, double* out) {
  return guard([&] {
    checked(c);
    if (!(thr > 0.0 && thr < 1.0)) fail(LR_EINVAL, "pinv: threshold must lie in (0,1)");
    require_nonempty(m, n, "svd");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<double> od((size_t)n * m, c->st);
    pinv_core(c, m, n, d, l, thr, od, n);
    to_host(c, n, m, od, n, out, n);
    sync(c);
  });
}

// id.hpp:91-119
int lr_id_column(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_solve_strategy strat,
                 int64_t* pivots, double* coeff) {
  return guard([&] {
    checked(c);
    require_rank_in_range(k, m, n, "id_column");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<int64_t> pd(n, c->st);
    DBuf<double> cd((size_t)k * std::max<int64_t>(n - k, 1), c->st);
    id_column_core(c, m, n, d, l, k, strat, pd, cd, k);
    idx_to_host(c, n, pd, pivots);
    to_host(c, k, n - k, cd, k, coeff, k);
    sync(c);
  });
}
int lr_id_column_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                   lr_solve_strategy strat, int64_t* pivots, double* coeff) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "id_column");
    id_column_core(c, m, n, a, lda, k, strat, pivots, coeff, k);
  });
}
int lr_id_row(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_solve_strategy strat,
              int64_t* pivots, double* coeff) {
  return guard([&] {
    checked(c);
    require_rank_in_range(k, n, m, "id_column");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    const int64_t lt = even(n);
    DBuf<double> dt((size_t)lt * m, c->st);
    transpose_matrix(m, n, d, l, dt, lt, c->st);
    DBuf<int64_t> pd(m, c->st);
    DBuf<double> cd((size_t)k * std::max<int64_t>(m - k, 1), c->st);
    id_column_core(c, n, m, dt, lt, k, strat, pd, cd, k);
    idx_to_host(c, m, pd, pivots);
    to_host(c, k, m - k, cd, k, coeff, k);
    sync(c);
  });
}

// sketch.hpp:200-223
int lr_randomized_id_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       lr_sketch_config cfg, lr_solve_strategy strat, int64_t* pivots, double* coeff) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "randomized_id");
    randomized_id_core(c, m, n, a, lda, k, cfg, strat, pivots, coeff, k);
  });
}
int lr_randomized_id(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_sketch_config cfg,
                     lr_solve_strategy strat, int64_t* pivots, double* coeff) {
  return guard([&] {
    checked(c);
    require_rank_in_range(k, m, n, "randomized_id");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<int64_t> pd(n, c->st);
    DBuf<double> cd((size_t)k * std::max<int64_t>(n - k, 1), c->st);
    randomized_id_core(c, m, n, d, l, k, cfg, strat, pd, cd, k);
    idx_to_host(c, n, pd, pivots);
    to_host(c, k, n - k, cd, k, coeff, k);
    sync(c);
  });
}

// id.hpp:124-134
int lr_tsid_from_column_id(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                           const int64_t* col_pivots, lr_solve_strategy strat, int64_t* row_pivots, double* row_coeff,
                           double* skeleton) {
  return guard([&] {
    checked(c);
    if (k < 1 || k > std::min(m, n)) require_rank_in_range(k, k, m, "id_column");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<int64_t> cp(n, c->st), rp(m, c->st);
    LRB_CUDA(cudaMemcpyAsync(cp.p, col_pivots, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->st));
    DBuf<double> rc((size_t)k * std::max<int64_t>(m - k, 1), c->st), sk((size_t)k * k, c->st);
    tsid_core(c, m, n, d, l, k, cp, strat, rp, rc, k, sk, nullptr, nullptr);
    idx_to_host(c, m, rp, row_pivots);
    to_host(c, k, m - k, rc, k, row_coeff, k);
    to_host(c, k, k, sk, k, skeleton, k);
    sync(c);
  });
}

// cur.hpp:23-34, lowrank_main.cpp:210-215
int lr_cur_from_two_sided(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                          const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots, double thr,
                          int u_mode, double* C, double* U, double* R) {
  return guard([&] {
    checked(c);
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<int64_t> cp(n, c->st), rp(m, c->st);
    LRB_CUDA(cudaMemcpyAsync(cp.p, col_pivots, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->st));
    LRB_CUDA(cudaMemcpyAsync(rp.p, row_pivots, sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->st));
    int64_t lcc = k;
    DBuf<double> cc = n > k ? to_dev(c, k, n - k, col_coeff, k, &lcc) : DBuf<double>(1, c->st);
    DBuf<double> Cd((size_t)m * k, c->st), Ud((size_t)k * k, c->st), Rd((size_t)k * n, c->st);
    cur_core(c, m, n, d, l, k, cp, cc, lcc, rp, thr, u_mode, Cd, Ud, Rd, nullptr);
    to_host(c, m, k, Cd, m, C, m);
    to_host(c, k, k, Ud, k, U, k);
    to_host(c, k, n, Rd, k, R, k);
    sync(c);
  });
}

// sketch.hpp:227-234 (+ lowrank_main.cpp:215 when u_mode == LR_U_CPINV_A_RPINV)
int lr_randomized_cur_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                        lr_sketch_config cfg, lr_solve_strategy strat, double thr, int u_mode, int64_t* col_pivots,
                        int64_t* row_pivots, double* C, double* U, double* R, double* col_coeff, double* row_coeff,
                        double* skeleton) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "randomized_cur");
    DBuf<double> cc, rc;
    if (!col_coeff) {
      cc = DBuf<double>((size_t)k * std::max<int64_t>(n - k, 1), c->st);
      col_coeff = cc;
    }
    if (!row_coeff) {
      rc = DBuf<double>((size_t)k * std::max<int64_t>(m - k, 1), c->st);
      row_coeff = rc;
    }
    mark(c, "begin");
    OzakiScope scope(c);
    randomized_id_core(c, m, n, a, lda, k, cfg, strat, col_pivots, col_coeff, k);
    if (split_applies(c, m, n, k, u_mode)) {
      tsid_cur_split(c, m, n, a, lda, k, col_pivots, col_coeff, k, strat, row_pivots, row_coeff, k, skeleton, thr, C,
                     U, R, [] {}, [] {});
      return;
    }
    DBuf<double> Ct((size_t)even(k) * m, c->st);
    tsid_core(c, m, n, a, lda, k, col_pivots, strat, row_pivots, row_coeff, k, skeleton, C, Ct);
    cur_core(c, m, n, a, lda, k, col_pivots, col_coeff, k, row_pivots, thr, u_mode, C, U, R, Ct);
  });
}
int lr_randomized_cur(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_sketch_config cfg,
                      lr_solve_strategy strat, double thr, int u_mode, int64_t* col_pivots, int64_t* row_pivots,
                      double* C, double* U, double* R, double* col_coeff, double* row_coeff, double* skeleton) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "randomized_cur");
    const int64_t ell = check_randomized_id(m, n, k, cfg);
    const int64_t l = even(m);
    DBuf<double> d((size_t)l * n, c->st);
    DBuf<int64_t> cp(n, c->st), rp(m, c->st);
    DBuf<double> Cd((size_t)m * k, c->st), Ud((size_t)k * k, c->st), Rd((size_t)k * n, c->st),
        ccd((size_t)k * std::max<int64_t>(n - k, 1), c->st), rcd((size_t)k * std::max<int64_t>(m - k, 1), c->st),
        skd((size_t)k * k, c->st);
    const int64_t ldy = work_ld(ell);
    DBuf<double> Y((size_t)ldy * n, c->st);
    zero_pad_rows(c, Y, ell, ldy, n);
    {
      Downloads down(c);  // declared after the buffers it reads: drains first
      OzakiScope scope(c);
      mark(c, "begin");
      if (cfg.power == 0) {
        upload_sketch(c, m, n, a, lda, d, l, ell, cfg.seed, Y, ldy, cfg.kind);
        randomized_id_core(c, m, n, d, l, k, cfg, strat, cp, ccd, k, Y);
      } else {
        LRB_CUDA(cudaMemcpy2DAsync(d.p, l * sizeof(double), a, lda * sizeof(double), m * sizeof(double), n,
                                   cudaMemcpyHostToDevice, c->st));
        randomized_id_core(c, m, n, d, l, k, cfg, strat, cp, ccd, k);
      }
      down.idx(n, cp, col_pivots);
      down.mat(k, n - k, ccd, k, col_coeff, k);
      auto rows_done = [&] {
        down.idx(m, rp, row_pivots);
        down.mat(m, k, Cd, m, C, m);
        down.mat(k, m - k, rcd, k, row_coeff, k);
        down.mat(k, k, skd, k, skeleton, k);
      };
      if (split_applies(c, m, n, k, u_mode, true)) {
        tsid_cur_split(c, m, n, d, l, k, cp, ccd, k, strat, rp, rcd, k, skd, thr, Cd, Ud, Rd, rows_done,
                       [&] { down.mat(k, n, Rd, k, R, k); });
        down.mat(k, k, Ud, k, U, k);
      } else {
        DBuf<double> Ct((size_t)even(k) * m, c->st);
        tsid_core(c, m, n, d, l, k, cp, strat, rp, rcd, k, skd, Cd, Ct);
        rows_done();
        cur_core(c, m, n, d, l, k, cp, ccd, k, rp, thr, u_mode, Cd, Ud, Rd, Ct,
                 [&] { down.mat(k, n, Rd, k, R, k); });
        down.mat(k, k, Ud, k, U, k);
      }
      down.finish();
    }
    sync(c);
  });
}

// cur.hpp:37-42 cur_id(a, k): id_two_sided -> cur_from_two_sided
int lr_cur_id_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_solve_strategy strat,
                double thr, int u_mode, int64_t* col_pivots, int64_t* row_pivots, double* C, double* U, double* R,
                double* col_coeff, double* row_coeff, double* skeleton) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "cur_id");
    DBuf<double> cc, rc;
    if (!col_coeff) {
      cc = DBuf<double>((size_t)k * std::max<int64_t>(n - k, 1), c->st);
      col_coeff = cc;
    }
    if (!row_coeff) {
      rc = DBuf<double>((size_t)k * std::max<int64_t>(m - k, 1), c->st);
      row_coeff = rc;
    }
    id_column_core(c, m, n, a, lda, k, strat, col_pivots, col_coeff, k);
    DBuf<double> Ct((size_t)even(k) * m, c->st);
    tsid_core(c, m, n, a, lda, k, col_pivots, strat, row_pivots, row_coeff, k, skeleton, C, Ct);
    cur_core(c, m, n, a, lda, k, col_pivots, col_coeff, k, row_pivots, thr, u_mode, C, U, R, Ct);
  });
}
int lr_cur_id(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, lr_solve_strategy strat,
              double thr, int u_mode, int64_t* col_pivots, int64_t* row_pivots, double* C, double* U, double* R,
              double* col_coeff, double* row_coeff, double* skeleton) {
  return guard([&] {
    checked(c);
    require_rank_in_range(k, m, n, "id_column");
    int64_t l;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<int64_t> cp(n, c->st), rp(m, c->st);
    DBuf<double> Cd((size_t)m * k, c->st), Ud((size_t)k * k, c->st), Rd((size_t)k * n, c->st),
        ccd((size_t)k * std::max<int64_t>(n - k, 1), c->st), rcd((size_t)k * std::max<int64_t>(m - k, 1), c->st),
        skd((size_t)k * k, c->st);
    id_column_core(c, m, n, d, l, k, strat, cp, ccd, k);
    DBuf<double> Ct((size_t)even(k) * m, c->st);
    tsid_core(c, m, n, d, l, k, cp, strat, rp, rcd, k, skd, Cd, Ct);
    cur_core(c, m, n, d, l, k, cp, ccd, k, rp, thr, u_mode, Cd, Ud, Rd, Ct);
    idx_to_host(c, n, cp, col_pivots);
    idx_to_host(c, m, rp, row_pivots);
    to_host(c, m, k, Cd, m, C, m);
    to_host(c, k, k, Ud, k, U, k);
    to_host(c, k, n, Rd, k, R, k);
    to_host(c, k, n - k, ccd, k, col_coeff, k);
    to_host(c, k, m - k, rcd, k, row_coeff, k);
    to_host(c, k, k, skd, k, skeleton, k);
    sync(c);
  });
}

int lr_cur_error_fro_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const double* C,
                       const double* U, const double* R, double* out) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "cur_error_fro");
    if (lda % 2 != 0 || reinterpret_cast<uintptr_t>(a) % 16 != 0) {
      const int64_t l = even(m);
      DBuf<double> ap((size_t)l * n, c->st);
      copy_matrix(m, n, a, lda, ap, l, c->st);
      error_core(c, m, n, ap, l, k, C, U, R, out);
      return;
    }
    error_core(c, m, n, a, lda, k, C, U, R, out);
  });
}
int lr_cur_error_fro(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const double* C,
                     const double* U, const double* R, double* out) {
  return guard([&] {
    checked(c);
    int64_t l, lc, lu, lr;
    DBuf<double> d = to_dev(c, m, n, a, lda, &l);
    DBuf<double> Cd = to_dev(c, m, k, C, m, &lc);
    DBuf<double> Ud = to_dev(c, k, k, U, k, &lu);
    DBuf<double> Rd = to_dev(c, k, n, R, k, &lr);
    // error_core expects C (ld m), U (ld k), R (ld k)
    DBuf<double> Cc((size_t)m * k, c->st), Uc((size_t)k * k, c->st), Rc((size_t)k * n, c->st);
    copy_matrix(m, k, Cd, lc, Cc, m, c->st);
    copy_matrix(k, k, Ud, lu, Uc, k, c->st);
    copy_matrix(k, n, Rd, lr, Rc, k, c->st);
    error_core(c, m, n, d, l, k, Cc, Uc, Rc, out);
  });
}

int lr_ctx_enable_timing(lr_ctx* c, int on) {
  return guard([&] {
    checked(c);
    flush_marks(c);
    c->timing = on != 0;
  });
}

int lr_ctx_stage_report(lr_ctx* c, char* buf, int64_t buflen) {
  return guard([&] {
    checked(c);
    flush_marks(c);
    std::string s = "{";
    for (size_t i = 0; i < c->stage_ms.size(); ++i) {
      if (i) s += ", ";
      char tmp[160];
      snprintf(tmp, sizeof tmp, "\"%s\": {\"ms\": %.6f, \"count\": %lld}", c->stage_ms[i].first.c_str(),
               c->stage_ms[i].second, c->stage_count[i].second);
      s += tmp;
    }
    s += "}";
    if (buf && buflen > 0) {
      strncpy(buf, s.c_str(), (size_t)buflen - 1);
      buf[buflen - 1] = 0;
    }
  });
}

int lr_ctx_reset_stats(lr_ctx* c) {
  return guard([&] {
    checked(c);
    flush_marks(c);
    c->stage_ms.clear();
    c->stage_count.clear();
    c->stats = lr_stats{};
  });
}

long long lr_kernel_launches(void) { return (long long)lrb::g_kernel_launches; }

// ---------------------------------------------------------------- sparse CUR (BASELINE config 5)
// sketch.hpp:227-234 + lowrank_main.cpp:215 on a CSR matrix: the dense
// contractions with A become SpMMs; C = A(:, J) and R = A(I, :) come back as
// sparse extracts (CSC / CSR, capacity nnz each).  The reference has no sparse
// path (core.hpp:14-17): semantics are those of the dense algorithm applied to
// the densified matrix.
int lr_randomized_cur_csr_d(lr_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                            const int64_t* col_idx, const double* val, int64_t k, lr_sketch_config cfg,
                            lr_solve_strategy strat, double thr, int u_mode, int64_t* col_pivots, int64_t* row_pivots,
                            double* U, int64_t* c_col_ptr, int64_t* c_row_idx, double* c_val, int64_t* r_row_ptr,
                            int64_t* r_col_idx, double* r_val, double* col_coeff, double* row_coeff,
                            double* skeleton) {
  return guard([&] {
    checked(c);
    require_rank_in_range(k, m, n, "randomized_id");
    if (cfg.kind != LR_SKETCH_GAUSSIAN || cfg.power != 0)
      fail(LR_EUNSUPPORTED, "randomized_id: only the Gaussian sketch with power 0 runs on the B200 path");
    const int64_t ell = k + cfg.oversample;
    if (ell < k) fail(LR_EINVAL, "build_sample: sample count below target rank");
    if (nnz > 0 && !device_all_finite(c, nnz, 1, val, std::max<int64_t>(nnz, 1)))
      fail(LR_EINVAL, "sketch_gaussian: matrix has non-finite entries");
    require_sample_count(ell, m, "sketch_gaussian");
    mark(c, "begin");
    DBuf<int64_t> colp(n + 1, c->st), rowi(std::max<int64_t>(nnz, 1), c->st);
    DBuf<double> cv(std::max<int64_t>(nnz, 1), c->st);
    csr_to_csc(m, n, nnz, row_ptr, col_idx, val, colp, rowi, cv, c->st);
    mark(c, "csr_to_csc");
    // Y = Omega A (SpMM), Omega l x m column-major
    DBuf<double> om((size_t)ell * m, c->st);
    gaussian_matrix(ell, m, cfg.seed, om, ell, false, c->st);
    const int64_t ldy = work_ld(ell);
    DBuf<double> Y((size_t)ldy * n, c->st);
    zero_pad_rows(c, Y, ell, ldy, n);
    spmm_csc(ell, n, om, ell, colp, rowi, cv, Y, ldy, c->st);
    mark(c, "sketch_spmm");
    const int64_t steps = std::min(ell, n);
    DBuf<double> tau(steps, c->st), cc, rc;
    if (!col_coeff) {
      cc = DBuf<double>((size_t)k * std::max<int64_t>(n - k, 1), c->st);
      col_coeff = cc;
    }
    if (!row_coeff) {
      rc = DBuf<double>((size_t)k * std::max<int64_t>(m - k, 1), c->st);
      row_coeff = rc;
    }
    cpqr_core(c, ell, n, Y, ldy, steps, col_pivots, tau, "cpqr_partial", work_padded(ell, ldy));
    mark(c, "cpqr_sample");
    solve_core(c, k, n - k, Y, ldy, Y.p + k * ldy, ldy, strat, col_coeff, k, false);
    mark(c, "coeff_solve_col");
    // C = A(:, J) (CSC extract + dense copy), row ID of C
    sparse_select(k, colp, rowi, cv, col_pivots, c_col_ptr, c_row_idx, c_val, c->st);
    DBuf<double> Cd((size_t)m * k, c->st), Ct((size_t)even(k) * m, c->st);
    sparse_scatter_cols(m, k, c_col_ptr, c_row_idx, c_val, Cd, m, c->st);
    tsid_core(c, m, k, nullptr, m, k, nullptr, strat, row_pivots, row_coeff, k, skeleton, Cd, Ct);
    // R = A(I, :) (CSR extract + dense copy)
    sparse_select(k, row_ptr, col_idx, val, row_pivots, r_row_ptr, r_col_idx, r_val, c->st);
    DBuf<double> Rd((size_t)k * n, c->st);
    sparse_scatter_rows(k, n, r_row_ptr, r_col_idx, r_val, Rd, k, c->st);
    u_core(c, m, n, k, Cd, Rd, col_pivots, col_coeff, k, thr, u_mode, U, Ct,
           [&](const double* Q, int64_t ldq, double* Xt, int64_t ldxt) {
             // X^T = A^T Q  <=>  X = Q^T A (k x n): SpMM with Q^T as the dense operand
             DBuf<double> Qt((size_t)k * m, c->st), X((size_t)k * n, c->st);
             mark(c, "at_alloc");
             transpose_matrix(m, k, Q, ldq, Qt, k, c->st);
             mark(c, "at_transpose_q");
             spmm_csc(k, n, Qt, k, colp, rowi, cv, X, k, c->st);
             mark(c, "at_spmm");
             transpose_matrix(k, n, X, k, Xt, ldxt, c->st);
             mark(c, "at_transpose_x");
           });
    mark(c, "u_sparse");
  });
}

// ||A - C U R||_F and ||A||_F for CSR A with C (CSC extract, m x k) and R (CSR
// extract, k x n): ||A||^2 - 2 <A, CUR> + ||CUR||^2, where <A, CUR> only needs
// CUR at A's nonzeros (an SpMM) and ||CUR||^2 = <(CU)^T CU, R R^T> (k x k).
int lr_cur_error_fro_csr_d(lr_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* row_ptr,
                           const int64_t* col_idx, const double* val, int64_t k, const int64_t* c_col_ptr,
                           const int64_t* c_row_idx, const double* c_val, const double* U, const int64_t* r_row_ptr,
                           const int64_t* r_col_idx, const double* r_val, double* out) {
  return guard([&] {
    checked(c);
    const int64_t ldk = even(k);
    DBuf<int64_t> colp(n + 1, c->st), rowi(std::max<int64_t>(nnz, 1), c->st);
    DBuf<double> cv(std::max<int64_t>(nnz, 1), c->st);
    csr_to_csc(m, n, nnz, row_ptr, col_idx, val, colp, rowi, cv, c->st);
    DBuf<double> Cd((size_t)m * k, c->st), Ct((size_t)ldk * m, c->st), Rd((size_t)ldk * n, c->st),
        Rt((size_t)even(n) * k, c->st), CU((size_t)even(m) * k, c->st), CUt((size_t)k * m, c->st),
        Z((size_t)k * n, c->st), G1((size_t)k * k, c->st), G2((size_t)k * k, c->st);
    sparse_scatter_cols(m, k, c_col_ptr, c_row_idx, c_val, Cd, m, c->st);
    sparse_scatter_rows(k, n, r_row_ptr, r_col_idx, r_val, Rd, ldk, c->st);
    transpose_matrix(m, k, Cd, m, Ct, ldk, c->st);
    gemm(c, m, k, k, Ct, ldk, U, k, CU, even(m));  // CU = C U
    transpose_matrix(m, k, CU, even(m), CUt, k, c->st);
    spmm_csc(k, n, CUt, k, colp, rowi, cv, Z, k, c->st);  // Z = (CU)^T A
    transpose_matrix(k, n, Rd, ldk, Rt, even(n), c->st);
    gemm(c, k, k, m, CU, even(m), CU, even(m), G1, k);    // (CU)^T CU
    gemm(c, k, k, n, Rt, even(n), Rt, even(n), G2, k);    // R R^T
    DBuf<double> part(4096 + 8, c->st), res(3, c->st);
    int np = 0;
    dot_sum(std::max<int64_t>(nnz, 1), 1, val, std::max<int64_t>(nnz, 1), val, std::max<int64_t>(nnz, 1), part, &np,
            c->st);
    sum_partials(part, np, res, c->st);
    dot_sum(k, n, Z, k, Rd, ldk, part, &np, c->st);
    sum_partials(part, np, res.p + 1, c->st);
    dot_sum(k, k, G1, k, G2, k, part, &np, c->st);
    sum_partials(part, np, res.p + 2, c->st);
    double h[3];
    LRB_CUDA(cudaMemcpyAsync(h, res.p, sizeof h, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    const double a2 = nnz > 0 ? h[0] : 0.0;
    const double e2 = a2 - 2.0 * h[1] + h[2];
    out[0] = std::sqrt(std::max(e2, 0.0));
    out[1] = std::sqrt(a2);
  });
}

// ---------------------------------------------------------------- shard primitives (distributed.py)
// randomized_id's second half (sketch.hpp:210-221) on a sample y (ell x n).
int lr_id_from_sample_d(lr_ctx* c, int64_t ell, int64_t n, const double* y, int64_t ldy, int64_t k,
                        lr_solve_strategy strat, int64_t* pivots, double* coeff) {
  return guard([&] {
    checked(c);
    require_nonempty(ell, n, "cpqr_partial");
    const int64_t steps = std::min(ell, n);
    if (k < 1 || steps < k) fail(LR_ERUNTIME, "randomized_id: sample rank collapsed below target rank");
    const int64_t lw = work_ld(ell);
    DBuf<double> W((size_t)lw * n, c->st), tau(steps, c->st);
    zero_pad_rows(c, W, ell, lw, n);
    copy_matrix(ell, n, y, ldy, W, lw, c->st);
    mark(c, "sample_exchange");  // since the previous stage: the caller's all-gather of Y (sharded protocol)
    cpqr_core(c, ell, n, W, lw, steps, pivots, tau, "cpqr_partial", work_padded(ell, lw));
    mark(c, "cpqr_sample");
    solve_core(c, k, n - k, W, lw, W.p + k * lw, lw, strat, coeff, k, false);
    mark(c, "coeff_solve_col");
  });
}

// id.hpp:124-134 given the column skeleton c = A(:, J) (m x k, ld ldc)
int lr_tsid_from_skeleton_columns_d(lr_ctx* c, int64_t m, int64_t k, const double* cs, int64_t ldc,
                                    lr_solve_strategy strat, int64_t* row_pivots, double* row_coeff,
                                    double* skeleton) {
  return guard([&] {
    checked(c);
    require_rank_in_range(k, k, m, "id_column");
    DBuf<double> C((size_t)m * k, c->st);
    copy_matrix(m, k, cs, ldc, C, m, c->st);
    tsid_core(c, m, k, nullptr, m, k, nullptr, strat, row_pivots, row_coeff, k, skeleton, C, nullptr);
  });
}

// core.hpp:70-76 (idx[j] < 0 gathers a zero column: masked gather for shard assembly)
int lr_gather_columns_d(lr_ctx* c, int64_t m, int64_t k, const double* a, int64_t lda, const int64_t* idx, double* out,
                        int64_t ldo) {
  return guard([&] { gather_columns(m, k, a, lda, idx, out, ldo, checked(c)->st); });
}
// core.hpp:79-85
int lr_gather_rows_d(lr_ctx* c, int64_t k, int64_t n, const double* a, int64_t lda, const int64_t* idx, double* out,
                     int64_t ldo) {
  return guard([&] { gather_rows(k, n, a, lda, idx, out, ldo, checked(c)->st); });
}

// G = R^T R in place (upper R); LR_ERUNTIME if G is not numerically SPD
int lr_cholesky_upper_d(lr_ctx* c, int64_t k, double* g, int64_t ldg) {
  return guard([&] {
    checked(c);
    DBuf<int> info(1, c->st);
    cholesky_upper(c->ws, k, g, ldg, info, c->st);
    d2h_mapped(c, c->h_flags, info.p, sizeof(int));
    sync(c);
    if (c->h_flags[0]) fail(LR_ERUNTIME, "cholesky: leading minor " + std::to_string(c->h_flags[0]) + " not positive");
  });
}

int lr_transpose_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, double* out, int64_t ldo) {
  return guard([&] { transpose_matrix(m, n, a, lda, out, ldo, checked(c)->st); });
}

int lr_tri_upper_inverse_d(lr_ctx* c, int64_t k, const double* r, int64_t ldr, double* rinv, int64_t ldi) {
  return guard([&] { tri_upper_inverse(k, r, ldr, rinv, ldi, checked(c)->st); });
}

// CholeskyQR2 of a tall x (rows x k): r (k x k upper), rinv; *ok = 0 when the
// factorisation broke down or cond bound >= 1e7 (caller falls back to SVD).
int lr_cholqr2_d(lr_ctx* c, int64_t rows, int64_t k, const double* x, int64_t ldx, double* r, double* rinv, int* ok) {
  return guard([&] {
    checked(c);
    DBuf<double> X((size_t)even(rows) * k, c->st), Xt((size_t)even(k) * rows, c->st);
    copy_matrix(rows, k, x, ldx, X, even(rows), c->st);
    transpose_matrix(rows, k, x, ldx, Xt, even(k), c->st);
    *ok = cholqr2(c, rows, k, X, even(rows), Xt, even(k), r, rinv) ? 1 : 0;
  });
}

int lr_gemm_tn_d(lr_ctx* c, int64_t M, int64_t N, int64_t K, const double* P, int64_t ldp, const double* Q,
                 int64_t ldq, double* out, int64_t ldo) {
  return guard([&] {
    checked(c);
    if (M < 1 || N < 1 || K < 1) fail(LR_EINVAL, "gemm_tn: dimensions must be positive");
    // in the Ozaki mode both operands are split (no A cache outside a CUR call)
    gemm_a(c, M, N, K, P, ldp, Q, ldq, out, ldo, -1);
  });
}

// ---- io.hpp:197-233 binary matrices straight to / from device memory
namespace {
constexpr int64_t kIoBlockBytes = 64ll << 20;  // row block per transfer (page-locked, double-buffered)
struct PinnedPair {
  double* h[2] = {nullptr, nullptr};
  ~PinnedPair() {
    for (double* p : h)
      if (p) cudaFreeHost(p);
  }
};
}  // namespace

int lr_read_matrix_binary_d(lr_ctx* c, const char* path, int64_t* rows, int64_t* cols, double* out, int64_t ldo) {
  return guard([&] {
    checked(c);
    const std::string p = path ? path : "";
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(p.c_str(), "rb"), std::fclose);
    if (!f) fail(LR_EPARSE, p + ":0: cannot open file");
    int64_t dims[2] = {0, 0};
    if (std::fread(dims, sizeof(int64_t), 2, f.get()) != 2 || dims[0] < 1 || dims[1] < 1)
      fail(LR_EPARSE, p + ":0: invalid binary matrix header");
    const int64_t m = dims[0], n = dims[1];
    if (rows) *rows = m;
    if (cols) *cols = n;
    if (!out) return;
    require_ld(m, ldo, "read_matrix_binary");
    // row blocks of rb rows (row-major rb x n = column-major n x rb, ld n)
    const int64_t rb = std::max<int64_t>(1, std::min<int64_t>(m, kIoBlockBytes / (8 * n)));
    PinnedPair hb;
    for (auto& h : hb.h) LRB_CUDA(cudaMallocHost(&h, sizeof(double) * (size_t)rb * n));
    DBuf<double> db0((size_t)rb * n, c->st), db1((size_t)rb * n, c->st);
    double* db[2] = {db0.p, db1.p};
    cudaStream_t up = aux_stream(c->up_st);
    cudaEvent_t copied[2], used[2];
    for (int b = 0; b < 2; ++b) {
      LRB_CUDA(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
      LRB_CUDA(cudaEventCreateWithFlags(&used[b], cudaEventDisableTiming));
      LRB_CUDA(cudaEventRecord(used[b], c->st));
    }
    struct Ev {
      cudaEvent_t* e;
      ~Ev() {
        for (int b = 0; b < 4; ++b) cudaEventDestroy(e[b]);
      }
    };
    cudaEvent_t all[4] = {copied[0], copied[1], used[0], used[1]};
    Ev ev{all};
    // runs before the buffers above are released, on every exit: no copy or
    // transpose may still touch them
    struct Drain {
      cudaStream_t a, b;
      ~Drain() {
        cudaStreamSynchronize(a);
        cudaStreamSynchronize(b);
      }
    } drain{up, c->st};
    int64_t blk = 0;
    for (int64_t i0 = 0; i0 < m; i0 += rb, ++blk) {
      const int b = (int)(blk & 1);
      const int64_t r = std::min(rb, m - i0);
      LRB_CUDA(cudaEventSynchronize(copied[b]));  // the host buffer's previous upload is done
      if (std::fread(hb.h[b], sizeof(double), (size_t)(r * n), f.get()) != (size_t)(r * n))
        fail(LR_EPARSE, p + ":0: truncated binary matrix payload");
      LRB_CUDA(cudaStreamWaitEvent(up, used[b], 0));  // the device buffer's previous transpose is done
      LRB_CUDA(cudaMemcpyAsync(db[b], hb.h[b], sizeof(double) * (size_t)(r * n), cudaMemcpyHostToDevice, up));
      LRB_CUDA(cudaEventRecord(copied[b], up));
      LRB_CUDA(cudaStreamWaitEvent(c->st, copied[b], 0));
      transpose_matrix(n, r, db[b], n, out + i0, ldo, c->st);  // rows i0 .. i0 + r - 1, column-major
      LRB_CUDA(cudaEventRecord(used[b], c->st));
    }
    sync(c);
  });
}

int lr_write_matrix_binary_d(lr_ctx* c, const char* path, int64_t m, int64_t n, const double* a, int64_t lda) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "write_matrix_binary");
    require_ld(m, lda, "write_matrix_binary");
    const std::string p = path ? path : "";
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(p.c_str(), "wb"), std::fclose);
    if (!f) fail(LR_ERUNTIME, "write_matrix_binary: cannot open " + p);
    const int64_t dims[2] = {m, n};
    if (std::fwrite(dims, sizeof(int64_t), 2, f.get()) != 2) fail(LR_ERUNTIME, "write_matrix_binary: write failed for " + p);
    const int64_t rb = std::max<int64_t>(1, std::min<int64_t>(m, kIoBlockBytes / (8 * n)));
    PinnedPair hb;
    for (auto& h : hb.h) LRB_CUDA(cudaMallocHost(&h, sizeof(double) * (size_t)rb * n));
    DBuf<double> db((size_t)rb * n, c->st);
    int64_t blk = 0;
    for (int64_t i0 = 0; i0 < m; i0 += rb, ++blk) {
      const int b = (int)(blk & 1);
      const int64_t r = std::min(rb, m - i0);
      transpose_matrix(r, n, a + i0, lda, db, n, c->st);  // rows i0.. -> row-major block
      LRB_CUDA(cudaMemcpyAsync(hb.h[b], db.p, sizeof(double) * (size_t)(r * n), cudaMemcpyDeviceToHost, c->st));
      sync(c);
      if (std::fwrite(hb.h[b], sizeof(double), (size_t)(r * n), f.get()) != (size_t)(r * n))
        fail(LR_ERUNTIME, "write_matrix_binary: write failed for " + p);
    }
  });
}

// C (m x n) = A (m x k) B (k x n), column-major: the reconstructions of
// id.hpp:143-159 / cur.hpp:77-80 on the GPU (the drop-in header and the Python
// mirror route their products here instead of a host GEMM)
int lr_gemm_d(lr_ctx* c, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, const double* b, int64_t ldb,
              double* out, int64_t ldo) {
  return guard([&] {
    checked(c);
    if (m < 1 || n < 1 || k < 1) fail(LR_EINVAL, "gemm: dimensions must be positive");
    require_ld(m, lda, "gemm");
    require_ld(k, ldb, "gemm");
    require_ld(m, ldo, "gemm");
    DBuf<double> at((size_t)even(k) * m, c->st);
    transpose_matrix(m, k, a, lda, at, even(k), c->st);
    gemm(c, m, n, k, at, even(k), b, ldb, out, ldo);
  });
}
int lr_gemm(lr_ctx* c, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, const double* b, int64_t ldb,
            double* out, int64_t ldo) {
  return guard([&] {
    checked(c);
    if (m < 1 || n < 1 || k < 1) fail(LR_EINVAL, "gemm: dimensions must be positive");
    int64_t la, lb;
    DBuf<double> da = to_dev(c, m, k, a, lda, &la), db = to_dev(c, k, n, b, ldb, &lb);
    DBuf<double> at((size_t)even(k) * m, c->st), dc((size_t)m * n, c->st);
    transpose_matrix(m, k, da, la, at, even(k), c->st);
    gemm(c, m, n, k, at, even(k), db, lb, dc, m);
    to_host(c, m, n, dc, m, out, ldo);
    sync(c);
  });
}

// ---- column-sharded entry points (one process per GPU)
int lr_nccl_get_unique_id(unsigned char* id) {
  return guard([&] {
    if (!id) fail(LR_EINVAL, "nccl_get_unique_id: null buffer");
    nccl_unique_id(id);
  });
}
int lr_ctx_attach_comm(lr_ctx* c, const unsigned char* id, int nranks, int rank) {
  return guard([&] {
    checked(c);
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) fail(LR_EINVAL, "attach_comm: bad unique id, size or rank");
    if (c->comm.comm) nccl_comm_destroy(c->comm.comm);
    c->comm = ShardComm{};
    ShardComm sc;
    sc.comm = nccl_comm_init(id, nranks, rank);
    sc.nranks = nranks;
    sc.rank = rank;
    c->comm = sc;
  });
}
int lr_ctx_detach_comm(lr_ctx* c) {
  return guard([&] {
    checked(c);
    LRB_CUDA(cudaStreamSynchronize(c->st));
    nccl_comm_destroy(c->comm.comm);
    c->comm = ShardComm{};
  });
}
int lr_ctx_comm_info(lr_ctx* c, int* nranks, int* rank) {
  return guard([&] {
    checked(c);
    if (nranks) *nranks = c->comm.nranks;
    if (rank) *rank = c->comm.rank;
  });
}
// host pointers: this rank's block uploads in column chunks with the sketch of
// each chunk issued as it lands (upload_sketch), then the sharded pipeline;
// the replicated factors and the rank's R block come back to host memory
int lr_randomized_cur_sharded(lr_ctx* c, int64_t m, int64_t n_local, int64_t col_offset, int64_t n_total,
                              const double* a_local, int64_t lda, int64_t k, lr_sketch_config cfg,
                              lr_solve_strategy strat, double thr, int u_mode, int64_t* col_pivots,
                              int64_t* row_pivots, double* C, double* U, double* r_local, double* col_coeff,
                              double* row_coeff, double* skeleton) {
  return guard([&] {
    checked(c);
    if (n_local < 1) fail(LR_EINVAL, "randomized_cur (column-sharded, host): empty column block");
    require_ld(m, lda, "randomized_cur");
    const int64_t ell = check_randomized_id(m, n_total, k, cfg);
    if (cfg.kind != LR_SKETCH_GAUSSIAN || cfg.power != 0)
      fail(LR_EUNSUPPORTED, "randomized_cur (column-sharded): Gaussian sketch with q = 0 only");
    const int64_t l = even(m), ldy = even(ell);
    DBuf<double> d((size_t)l * n_local, c->st), Y((size_t)ldy * n_local, c->st);
    DBuf<int64_t> cp(n_total, c->st), rp(m, c->st);
    DBuf<double> Cd((size_t)m * k, c->st), Ud((size_t)k * k, c->st), Rd((size_t)k * n_local, c->st),
        ccd((size_t)k * std::max<int64_t>(n_total - k, 1), c->st),
        rcd((size_t)k * std::max<int64_t>(m - k, 1), c->st), skd((size_t)k * k, c->st);
    OzakiScope scope(c);
    upload_sketch(c, m, n_local, a_local, lda, d, l, ell, cfg.seed, Y, ldy, cfg.kind);
    randomized_cur_sharded_core(c, m, n_local, col_offset, n_total, d, l, k, cfg, strat, thr, u_mode, cp, rp, Cd,
                                Ud, Rd, ccd, rcd, skd, Y, ldy);
    idx_to_host(c, n_total, cp, col_pivots);
    idx_to_host(c, m, rp, row_pivots);
    to_host(c, m, k, Cd, m, C, m);
    to_host(c, k, k, Ud, k, U, k);
    to_host(c, k, n_local, Rd, k, r_local, k);
    if (col_coeff) to_host(c, k, n_total - k, ccd, k, col_coeff, k);
    if (row_coeff) to_host(c, k, m - k, rcd, k, row_coeff, k);
    if (skeleton) to_host(c, k, k, skd, k, skeleton, k);
    sync(c);
  });
}
int lr_cpqr_sharded_d(lr_ctx* c, int64_t m, int64_t n_local, int64_t col_offset, int64_t n_total,
                      const double* a_local, int64_t lda, int64_t k, int64_t* pivots, double* s) {
  return guard([&] {
    checked(c);
    if (n_local > 0) require_ld(m, lda, "cpqr_partial");
    if (col_offset < 0 || n_local < 0 || col_offset + n_local > n_total)
      fail(LR_EINVAL, "cpqr_partial (column-sharded): bad column block");
    cpqr_sharded_core(c, m, n_local, col_offset, n_total, a_local, lda, k, k, pivots, s, "cpqr_partial",
                      c->comm.comm ? 0 : c->emu_shards);
  });
}
int lr_ctx_set_shard_emulation(lr_ctx* c, int nshards) {
  return guard([&] {
    checked(c);
    if (nshards < 0 || nshards > 64) fail(LR_EINVAL, "set_shard_emulation: 0..64 shards");
    c->emu_shards = nshards;
  });
}
int lr_randomized_cur_sharded_d(lr_ctx* c, int64_t m, int64_t n_local, int64_t col_offset, int64_t n_total,
                                const double* a_local, int64_t lda, int64_t k, lr_sketch_config cfg,
                                lr_solve_strategy strat, double thr, int u_mode, int64_t* col_pivots,
                                int64_t* row_pivots, double* C, double* U, double* r_local, double* col_coeff,
                                double* row_coeff, double* skeleton) {
  return guard([&] {
    checked(c);
    if (n_local > 0) require_ld(m, lda, "randomized_cur");
    DBuf<double> cc, rc;
    if (!col_coeff) {
      cc = DBuf<double>((size_t)k * std::max<int64_t>(n_total - k, 1), c->st);
      col_coeff = cc;
    }
    if (!row_coeff) {
      rc = DBuf<double>((size_t)k * std::max<int64_t>(m - k, 1), c->st);
      row_coeff = rc;
    }
    randomized_cur_sharded_core(c, m, n_local, col_offset, n_total, a_local, lda, k, cfg, strat, thr, u_mode,
                                col_pivots, row_pivots, C, U, r_local, col_coeff, row_coeff, skeleton);
  });
}


// ---- verifiers at scale (verify.hpp:14-166; spectral norms by block Krylov on the residual operators)
int lr_residual_norms_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const double* x,
                        int64_t ldx, const double* y, int64_t ldy, double* spectral, double* frobenius) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "spectral_norm");
    require_ld(m, lda, "spectral_norm");
    if (k < 0 || k > std::min(m, n)) fail(LR_EINVAL, "residual_norms: rank out of range");
    if (spectral) {
      DBuf<double> At((size_t)even(n) * m, c->st);
      transpose_matrix(m, n, a, lda, At, even(n), c->st);
      ResidualBufs rb;
      const ResidualOp op = residual_op(c, m, n, a, lda, At, even(n), k, x, ldx, y, ldy, rb);
      *spectral = op_sigma1(c, op, kVerifySeed);
    }
    if (frobenius) *frobenius = residual_frob(c, m, n, a, lda, k, x, ldx, y, ldy);
  });
}

int lr_error_report_lowrank_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                              const double* x, int64_t ldx, const double* y, int64_t ldy, lr_error_report* out) {
  return guard([&] {
    checked(c);
    require_nonempty(m, n, "error_report");
    require_ld(m, lda, "error_report");
    if (!out) fail(LR_EINVAL, "error_report: null report");
    DBuf<double> At((size_t)even(n) * m, c->st);
    transpose_matrix(m, n, a, lda, At, even(n), c->st);
    ResidualBufs r0, r1;
    const double a2 = op_sigma1(c, residual_op(c, m, n, a, lda, At, even(n), 0, nullptr, 1, nullptr, 1, r0),
                                kVerifySeed);
    const double af = residual_frob(c, m, n, a, lda, 0, nullptr, 1, nullptr, 1);
    lr_error_report rep{};
    rep.abs_spectral = op_sigma1(c, residual_op(c, m, n, a, lda, At, even(n), k, x, ldx, y, ldy, r1), kVerifySeed);
    rep.abs_frob = residual_frob(c, m, n, a, lda, k, x, ldx, y, ldy);
    if (af == 0.0) {  // verify.hpp:41-44
      rep.rel_is_absolute = 1;
      rep.rel_spectral = rep.abs_spectral;
      rep.rel_frob = rep.abs_frob;
    } else {
      rep.rel_spectral = rep.abs_spectral / a2;
      rep.rel_frob = rep.abs_frob / af;
    }
    *out = rep;
  });
}

namespace {
// C = A(:, J), V^T, R = A(I, :), W, (C U) and A^T for the verifiers
struct VerifyInputs {
  DBuf<double> At, C, Ct, Vt, R, Wt, W, CU;
};
void verify_inputs(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k, const int64_t* col_piv,
                   const double* col_coeff, const int64_t* row_piv, const double* row_coeff, const double* u,
                   VerifyInputs& v) {
  v.At = DBuf<double>((size_t)even(n) * m, c->st);
  transpose_matrix(m, n, a, lda, v.At, even(n), c->st);
  v.C = DBuf<double>((size_t)m * k, c->st);
  gather_columns(m, k, a, lda, col_piv, v.C, m, c->st);
  v.Vt = DBuf<double>((size_t)k * n, c->st);
  basis_t(c, n, k, col_piv, col_coeff, k, v.Vt);
  if (row_piv) {
    v.R = DBuf<double>((size_t)k * n, c->st);
    gather_rows(k, n, a, lda, row_piv, v.R, k, c->st);
  }
  if (row_piv && row_coeff) {
    v.Wt = DBuf<double>((size_t)k * m, c->st);
    basis_t(c, m, k, row_piv, row_coeff, k, v.Wt);
    v.W = DBuf<double>((size_t)m * k, c->st);
    transpose_matrix(k, m, v.Wt, k, v.W, m, c->st);
  }
  if (u) {  // reconstruct(cur) = (C U) R  (cur.hpp:77-80)
    v.Ct = DBuf<double>((size_t)even(k) * m, c->st);
    transpose_matrix(m, k, v.C, m, v.Ct, even(k), c->st);
    v.CU = DBuf<double>((size_t)m * k, c->st);
    gemm(c, m, k, k, v.Ct, even(k), u, k, v.CU, m);
  }
}
}  // namespace

int lr_verify_lemma1_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots,
                       const double* row_coeff, const double* u, lr_lemma1_report* out) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "verify_lemma1");
    require_rank_in_range(k, m, n, "verify_lemma1");
    if (!out) fail(LR_EINVAL, "verify_lemma1: null report");
    VerifyInputs v;
    verify_inputs(c, m, n, a, lda, k, col_pivots, col_coeff, row_pivots, row_coeff, u, v);
    ResidualBufs b0, b1, b2;
    lr_lemma1_report rep{};
    rep.e_norm = op_sigma1(c, residual_op(c, m, n, a, lda, v.At, even(n), k, v.C, m, v.Vt, k, b0), kVerifySeed);
    rep.etilde_norm = op_sigma1(c, residual_op(c, m, n, a, lda, v.At, even(n), k, v.W, m, v.R, k, b1), kVerifySeed);
    rep.lhs = op_sigma1(c, residual_op(c, m, n, a, lda, v.At, even(n), k, v.CU, m, v.R, k, b2), kVerifySeed);
    rep.rhs = rep.e_norm + rep.etilde_norm;
    rep.holds = rep.lhs <= rep.rhs * (1.0 + 1e-8);  // verify.hpp:77-78
    *out = rep;
  });
}

int lr_verify_lemma2_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                       const int64_t* col_pivots, const double* col_coeff, const int64_t* row_pivots,
                       const double* row_coeff, lr_lemma2_report* out) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "verify_lemma2");
    require_rank_in_range(k, m, n, "verify_lemma2");
    if (!out) fail(LR_EINVAL, "verify_lemma2: null report");
    VerifyInputs v;
    verify_inputs(c, m, n, a, lda, k, col_pivots, col_coeff, row_pivots, row_coeff, nullptr, v);
    const int64_t mr = m - k, ldr = even(std::max<int64_t>(mr, 1));
    ResidualBufs be, bw;
    const ResidualOp e = residual_op(c, m, n, a, lda, v.At, even(n), k, v.C, m, v.Vt, k, be);
    const ResidualOp w = residual_op(c, m, n, a, lda, v.At, even(n), k, v.W, m, v.R, k, bw);
    lr_lemma2_report rep{};
    rep.e_norm = op_sigma1(c, e, kVerifySeed);
    rep.etilde_norm = op_sigma1(c, w, kVerifySeed);
    // the permuted stack [0; F E] (verify.hpp:108-117) as an operator: rows I(l), l >= k,
    // take E(I(l), :) - T(:, l-k)^T E(I_skel, :); the skeleton rows are zero
    DBuf<double> Tt((size_t)ldr * k, c->st);
    if (mr > 0) transpose_matrix(k, mr, row_coeff, k, Tt, ldr, c->st);
    auto stack = [&](int64_t r, double* x, int64_t ldx, double* o, int64_t ldo) {  // o = S x (m x r)
      DBuf<double> sk((size_t)k * r, c->st), rs((size_t)ldr * r, c->st);
      gather_rows(k, r, x, ldx, row_pivots, sk, k, c->st);
      if (mr > 0) {
        gather_rows(mr, r, x, ldx, row_pivots + k, rs, ldr, c->st);
        gemm(c, mr, r, k, row_coeff, k, sk, k, rs, ldr, -1.0, 1.0);
      }
      scatter_stack(m, r, k, row_pivots, nullptr, 0, rs, ldr, o, ldo, c->st);
    };
    auto stack_t = [&](int64_t r, const double* x, int64_t ldx, double* o, int64_t ldo) {  // o = S^T x
      DBuf<double> rs((size_t)ldr * r, c->st), top((size_t)k * r, c->st);
      LRB_CUDA(cudaMemsetAsync(top.p, 0, sizeof(double) * k * r, c->st));
      if (mr > 0) {
        gather_rows(mr, r, x, ldx, row_pivots + k, rs, ldr, c->st);
        gemm(c, k, r, mr, Tt, ldr, rs, ldr, top, k, -1.0, 0.0);
      }
      scatter_stack(m, r, k, row_pivots, top, k, rs, ldr, o, ldo, c->st);
    };
    const int64_t ldm = even(m);
    rep.fe_norm = krylov_sigma1(
        c, m, n,
        [&](int64_t r, const double* in, int64_t li, double* o, int64_t lo) {
          DBuf<double> t((size_t)ldm * r, c->st);
          e.apply(r, in, li, t, ldm);
          stack(r, t, ldm, o, lo);
        },
        [&](int64_t r, const double* in, int64_t li, double* o, int64_t lo) {
          DBuf<double> t((size_t)ldm * r, c->st);
          stack_t(r, in, li, t, ldm);
          e.apply_t(r, t, ldm, o, lo);
        },
        kVerifySeed);
    // entrywise gap of the two paths: direct - stack = -(C(I_res,:) - T^T C(I_skel,:)) V^T on
    // the residual rows and 0 on the skeleton rows; its largest entry, by column blocks
    rep.entry_diff = 0.0;
    if (mr > 0) {
      DBuf<double> Csk((size_t)k * k, c->st), D((size_t)ldr * k, c->st), Dt((size_t)even(k) * mr, c->st);
      gather_rows(k, k, v.C, m, row_pivots, Csk, k, c->st);
      gather_rows(mr, k, v.C, m, row_pivots + k, D, ldr, c->st);
      gemm(c, mr, k, k, row_coeff, k, Csk, k, D, ldr, -1.0, 1.0);
      transpose_matrix(mr, k, D, ldr, Dt, even(k), c->st);
      DBuf<double> Vk((size_t)even(k) * n, c->st);
      copy_matrix(k, n, v.Vt, k, Vk, even(k), c->st);
      const int64_t nb = 2048;
      DBuf<double> blk((size_t)ldr * nb, c->st), part(4 * num_sms() + 4, c->st), mx(1, c->st);
      double emax = 0.0;
      for (int64_t j0 = 0; j0 < n; j0 += nb) {
        const int64_t w2 = std::min(nb, n - j0);
        gemm(c, mr, w2, k, Dt, even(k), Vk.p + j0 * even(k), even(k), blk, ldr);
        max_abs(mr, w2, blk, ldr, part, mx, c->st);
        d2h_mapped(c, c->h_scal, mx.p, sizeof(double));
        sync(c);
        emax = std::max(emax, c->h_scal[0]);
      }
      rep.entry_diff = emax;
    }
    rep.t_norm = mr > 0 ? coeff_norm2(c, k, mr, row_coeff, k) : 0.0;
    rep.bound_rhs = (1.0 + rep.t_norm) * rep.e_norm;
    const double scale = std::max(rep.etilde_norm, rep.fe_norm);
    const double af = residual_frob(c, m, n, a, lda, 0, nullptr, 1, nullptr, 1);
    rep.holds = std::abs(rep.etilde_norm - rep.fe_norm) <= 1e-8 * scale || scale <= 1e-12 * af;  // verify.hpp:126-127
    rep.bound_holds = rep.etilde_norm <= rep.bound_rhs * (1.0 + 1e-8);
    *out = rep;
  });
}

int lr_verify_corollary_d(lr_ctx* c, int64_t m, int64_t n, const double* a, int64_t lda, int64_t k,
                          const int64_t* col_pivots, const double* col_coeff, const double* u, lr_solve_strategy strat,
                          lr_corollary_report* out) {
  return guard([&] {
    checked(c);
    require_ld(m, lda, "verify_corollary");
    require_rank_in_range(k, m, n, "verify_corollary");
    if (!out) fail(LR_EINVAL, "verify_corollary: null report");
    // the row skeletonization of C recomputed (verify.hpp:148: id_row(skeleton_columns(a, col_id), k))
    DBuf<int64_t> rp(m, c->st);
    DBuf<double> rcf((size_t)k * std::max<int64_t>(m - k, 1), c->st), Cb((size_t)m * k, c->st);
    tsid_core(c, m, n, a, lda, k, col_pivots, strat, rp, rcf, k, nullptr, Cb, nullptr);
    VerifyInputs v;
    verify_inputs(c, m, n, a, lda, k, col_pivots, col_coeff, rp, nullptr, u, v);
    ResidualBufs b0, b1;
    lr_corollary_report rep{};
    rep.t_norm = m > k ? coeff_norm2(c, k, m - k, rcf, k) : 0.0;
    rep.e_norm = op_sigma1(c, residual_op(c, m, n, a, lda, v.At, even(n), k, v.C, m, v.Vt, k, b0), kVerifySeed);
    rep.lhs = op_sigma1(c, residual_op(c, m, n, a, lda, v.At, even(n), k, v.CU, m, v.R, k, b1), kVerifySeed);
    rep.bound = (2.0 + rep.t_norm) * rep.e_norm;
    rep.ceiling = 2.0 * std::sqrt((double)k * (double)(m - k));
    rep.holds = rep.lhs <= rep.bound * (1.0 + 1e-8);
    *out = rep;
  });
}

}  // extern "C"
