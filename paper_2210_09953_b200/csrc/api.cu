// api.cu -- C ABI (include/rcholqr.h): plan/workspace management, argument validation, the launch
// sequence of Algorithm 2 and the multi-GPU all-reduce.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <unordered_set>
#include <vector>
#include "internal.cuh"
#include "rcholqr.h"

using namespace rcq;

// ---------------------------------------------------------------------------------------------
// NCCL, loaded lazily (a single-GPU plan never touches it).
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  const char* env = getenv("RCHOLQR_NCCL_LIB");
  void* h = nullptr;
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy;
  return g_nccl.ok;
}
}  // namespace

// ---------------------------------------------------------------------------------------------
// SRHT sampled rows (reading A23), computed on the host at plan creation: a host
// Philox4x32-10 (Salmon et al. SC'11; the device generator is theta.cuh's philox_at).
namespace {
void host_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed, uint32_t out[4]) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint32_t c[4] = {c0, c1, c2, c3};
  for (int round = 0; round < 10; ++round) {
    if (round) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0; c[1] = (uint32_t)p1; c[2] = n2; c[3] = (uint32_t)p0;
  }
  for (int t = 0; t < 4; ++t) out[t] = c[t];
}
// s_r = (w1 << 32 | w0) mod 2^48 of Philox(ctr = (r, 0, a, 7)), a advancing past duplicates
std::vector<uint64_t> srht_rows_host(uint64_t seed, int k) {
  std::vector<uint64_t> s((size_t)k);
  std::unordered_set<uint64_t> seen;
  for (int r = 0; r < k; ++r)
    for (uint32_t a = 0;; ++a) {
      uint32_t w[4];
      host_philox((uint32_t)r, 0u, a, 7u, seed, w);
      const uint64_t v = (((uint64_t)w[1] << 32) | w[0]) & ((1ull << 48) - 1);
      if (seen.insert(v).second) { s[(size_t)r] = v; break; }
    }
  return s;
}
}  // namespace

// Which tall-solve kernels serve n columns of dtype (the plan's n, or Alg. 7's rank r).
struct SolvePlan {
  TrsmLaunch tr{};
  int pairs = 0, stream_tb = 0;
  bool solve_tc = false;
  bool mstream = false;   // 128 < n <= 256: warp-pair substitution with M streamed per column block
};

struct rcholqr_plan_s {
  rcholqr_desc d;
  int sms = 0;
  size_t smem_optin = 0;
  SketchLaunch sk{};
  // tall-solve kernels for n columns: TrsmLaunch tr (R^{-1} GEMM); pairs > 0: warp-pair blocked
  // substitution with this many pairs per CTA; stream_tb > 0: streamed blocked substitution (fp64,
  // n > 256) with this block width; solve_tc: fp32 X, n <= 128, tcgen05 digit solve (solve_tc.cu)
  SolvePlan sp{};
  void* xdig = nullptr;     // pre-split X digit planes of the tcgen05 Gaussian sketch (grown on demand)
  // RCholeskyQR2 (rcqr2.cu): Gram partials, A, Cholesky work, R', R1, and Q1 (grown on demand)
  int gram_splits = 0;
  double* gpart = nullptr; double* gA = nullptr; double* gW = nullptr; double* gRp = nullptr; double* gR1 = nullptr;
  void* q1buf = nullptr; size_t q1_bytes = 0;
  // reduced RCholeskyQR (Alg. 5): the (k + l)-row sketch [P; Y] and its partials (grown on demand)
  int red_l = 0;
  SketchLaunch red_sk{};
  double* red_part = nullptr; double* red_partc = nullptr; double* red_P = nullptr;
  // rank-revealing RCholeskyQR (Alg. 7), allocated on first use: [P; colsq] (k + 1) x n, P D^{-1},
  // the pivoting workspace, P(:, perm), R, R11^{-1}, the compact R11, d, column partials, scalars
  double* rr_buf = nullptr; double* rr_Pn = nullptr; double* rr_A = nullptr; double* rr_Pg = nullptr;
  uint64_t* srht_d = nullptr;   // SRHT: the k sampled Hadamard rows
  double* rr_R = nullptr; double* rr_W = nullptr; double* rr_R11 = nullptr; double* rr_d = nullptr;
  double* rr_cpart = nullptr; double* rr_cspart = nullptr; double* rr_sd = nullptr; int* rr_si = nullptr; int* rr_perm = nullptr;
  int* rr_qst = nullptr; int rr_splits = 0;
  void* rr_xr = nullptr; size_t rr_xr_bytes = 0;
  size_t xdig_bytes = 0;
  void* qws = nullptr;      // its W-digit workspace
  double* tbuf = nullptr;   // [m_local][stream_tb] T_J workspace of the streamed solve
  size_t tbuf_elems = 0;
  int qr_kind = 0;
  double* qr_ws = nullptr;   // blocked Householder workspace (kQrBlocked)
  double* part = nullptr;   // [splits][k][n] per-CTA sketch partials (running sums)
  double* partc = nullptr;  // [splits][k][n] their TwoSum compensations (Gaussian sketch)
  double* P = nullptr;      // [k][n] reduced sketch
  double* W = nullptr;      // [n][n] R^{-1}
  double* Awork = nullptr;  // [n][k] column-major Householder workspace (reflectors)
  double* diag = nullptr;   // [2n] raw pivots (sign before normalisation), then reflector heads v0
  double* tau = nullptr;    // [n] reflector scalings
  double* Rtmp = nullptr;   // [n][n] R when the caller does not want one
  int* status_d = nullptr;
  int* flag_d = nullptr;    // tensor-core sketch overflow flag (selects the guarded fallback kernel)
  int* flag_seen_d = nullptr;   // set by the reduction when that flag was raised (rcholqr_last_path)
  unsigned path = 0;        // RCHOLQR_PATH_* bits of the current / last call
  int* status_h = nullptr;  // pinned
  // factor_host staging
  void* xbuf = nullptr; void* qbuf = nullptr; size_t xq_bytes = 0;
  double* rbuf = nullptr; double* sbuf = nullptr;
  // rcholqr_factor_graph: the captured kernel chain of one argument tuple
  struct GraphKey {
    const void* X = nullptr; int64_t m = -1, ro = 0, ldx = 0; void* Q = nullptr; int64_t ldq = 0;
    double* R = nullptr; double* S = nullptr;
    // the plan's lazily grown workspaces the chain reads (a later, larger call frees and reallocates them:
    // a graph captured before that must not be replayed)
    const void* xdig = nullptr; const void* tbuf = nullptr;
    bool operator==(const GraphKey& o) const {
      return X == o.X && m == o.m && ro == o.ro && ldx == o.ldx && Q == o.Q && ldq == o.ldq && R == o.R && S == o.S &&
             xdig == o.xdig && tbuf == o.tbuf;
    }
  } gkey;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;   // capture stream (capture on the legacy default stream is not allowed)
  unsigned gpath = 0;               // path bits of the captured chain
  bool timing = false;
  cudaEvent_t ev[7] = {};
  float last_ms[6] = {0, 0, 0, 0, 0, 0};
  bool have_timing = false;
};

namespace {
size_t esize(int dtype) { return dtype == RCHOLQR_F64 ? 8 : 4; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// internal: no native column-major kernel for this plan / alignment (rcholqr_factor_colmajor then takes the adapter)
constexpr rcholqr_status RCHOLQR_E_UNSUPPORTED_INTERNAL = (rcholqr_status)100;

rcholqr_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return RCHOLQR_OK;
  if (getenv("RCHOLQR_DEBUG")) fprintf(stderr, "rcholqr: CUDA error: %s\n", cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return RCHOLQR_E_NOMEM;
  return RCHOLQR_E_CUDA;
}
#define CU(x)                                        \
  do {                                               \
    cudaError_t _e = (x);                            \
    if (_e != cudaSuccess) return cuda_status(_e);   \
  } while (0)

rcholqr_status validate_desc(const rcholqr_desc* d) {
  if (!d) return RCHOLQR_E_INVALID;
  if (d->dtype != RCHOLQR_F64 && d->dtype != RCHOLQR_F32) return RCHOLQR_E_INVALID;
  if (d->sketch != RCHOLQR_GAUSSIAN && d->sketch != RCHOLQR_SPARSE_SIGN && d->sketch != RCHOLQR_RADEMACHER &&
      d->sketch != RCHOLQR_SRHT)
    return RCHOLQR_E_INVALID;
  if (d->n < 1 || d->k < d->n) return RCHOLQR_E_SHAPE;
  if (d->sketch == RCHOLQR_SPARSE_SIGN &&
      (d->nnz_per_col < 1 || d->nnz_per_col > d->k || d->k % d->nnz_per_col != 0))
    return RCHOLQR_E_SHAPE;
  if ((int64_t)d->k * d->n > (int64_t)1 << 28) return RCHOLQR_E_SHAPE;
  return RCHOLQR_OK;
}

bool overlaps(const void* a, size_t abytes, const void* b, size_t bbytes) {
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + bbytes && pb < pa + abytes;
}

size_t span_bytes(int64_t rows, int64_t ld, int n, size_t es) {
  return rows <= 0 ? 0 : (size_t)((rows - 1) * ld + n) * es;
}

rcholqr_status status_from_word(int w) {
  if (w & kStNonfinite) return RCHOLQR_E_NONFINITE;
  if (w & kStSingular) return RCHOLQR_E_SINGULAR;
  return RCHOLQR_OK;
}

rcholqr_status check_factor_args(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx,
                                 const void* Q, int64_t ldq) {
  if (!p) return RCHOLQR_E_INVALID;
  const int n = p->d.n;
  if (m < 0 || ro < 0 || ldx < n || ldq < n) return RCHOLQR_E_INVALID;
  if (m > 0 && (!X || !Q)) return RCHOLQR_E_INVALID;
  const size_t es = esize(p->d.dtype);
  if (m > 0 && overlaps(X, span_bytes(m, ldx, n, es), Q, span_bytes(m, ldq, n, es))) return RCHOLQR_E_INVALID;
  return RCHOLQR_OK;
}

// Step 1 (+ the all-reduce).  By default the plan's k-row sketch; Alg. 5 passes its own launch `L` of
// `k` rows (partials part/partc), with rows >= k_first scaled as extractor rows, and may defer the
// all-reduce (allreduce = false) to sum [P; Y] at once.
rcholqr_status do_sketch(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, double* P,
                         cudaStream_t st, const SketchLaunch* Lp = nullptr, int k = 0, double* part = nullptr,
                         double* partc = nullptr, int k_first = 0, bool allreduce = true, double* cs_part = nullptr,
                         double* cs_out = nullptr, bool* cs_done = nullptr, bool colmajor = false) {
  if (cs_done) *cs_done = false;
  const auto& d = p->d;
  const SketchLaunch& L = Lp ? *Lp : p->sk;
  if (!Lp) { k = d.k; part = p->part; partc = p->partc; }
  const bool timed = p->timing && allreduce;
  if (m > 0) {
    if (timed) cudaEventRecord(p->ev[0], st);
    if (L.tc && L.kind < kSketchSparse) {   // grow the pre-split digit workspace (capped)
      const size_t need = gauss_tcp_chunk_workspace(m, d.n, d.dtype, L.tc_splits);
      if (need > p->xdig_bytes) {
        cudaFree(p->xdig);
        p->xdig = nullptr; p->xdig_bytes = 0;
        if (cudaMalloc(&p->xdig, need) == cudaSuccess) p->xdig_bytes = need;
        else cudaGetLastError();   // not enough memory: the in-kernel split is used instead
      }
    }
    const cudaError_t se = launch_sketch(L, X, d.dtype, m, d.n, ldx, ro, k, d.nnz_per_col, d.seed, part, partc, P,
                                         p->status_d, p->flag_d, p->xdig, p->xdig_bytes, st, timed ? p->ev[1] : nullptr,
                                         k_first, &p->path, p->flag_seen_d, cs_part, cs_out, cs_done, colmajor);
    if (colmajor && se == cudaErrorNotSupported) return RCHOLQR_E_UNSUPPORTED_INTERNAL;
    CU(se);
  } else {
    if (timed) { cudaEventRecord(p->ev[0], st); cudaEventRecord(p->ev[1], st); }
    CU(cudaMemsetAsync(P, 0, sizeof(double) * (size_t)k * d.n, st));
  }
  if (timed) cudaEventRecord(p->ev[2], st);
  if (d.nccl_comm && allreduce) {
    if (!nccl_load()) return RCHOLQR_E_NCCL;
    ncclResult_t r = g_nccl.AllReduce(P, P, (size_t)k * d.n, ncclFloat64, ncclSum, (ncclComm_t)d.nccl_comm, st);
    if (r != ncclSuccess) return RCHOLQR_E_NCCL;
  }
  if (timed) cudaEventRecord(p->ev[3], st);
  return RCHOLQR_OK;
}

// n <= 128: warp-pair blocked substitution (or the tcgen05 digit solve for fp32 X); 128 < n <= 256:
// streamed-M substitution; fp64 n > 256: column-block GEMMs; fp32 n > 256: the R^{-1} GEMM kernel.
SolvePlan plan_solve(int n, int dtype, size_t smem_optin) {
  SolvePlan s;
  s.tr = plan_trsm(n, dtype, smem_optin);
  s.pairs = trsm_pair_count(n, smem_optin);
  s.mstream = s.pairs == 0 && trsm_mstream_applicable(n, smem_optin);
  if (s.pairs == 0 && !s.mstream && dtype == RCHOLQR_F64) s.stream_tb = n < 512 ? 64 : 128;
  s.solve_tc = solve_tc_applicable(dtype, n);
  return s;
}

// Step 3: triangular prep + tall solve (the kernels plan_solve picked).  `n_cols`
// > 0 solves with that many columns (R n_cols x n_cols) instead of the plan's n.
// colmajor: X and Q column-major -- only the tcgen05 digit solve reads and writes that layout (else
// RCHOLQR_E_UNSUPPORTED_INTERNAL: the caller takes the layout adapter).
rcholqr_status solve(rcholqr_plan p, const void* X, int64_t m, int64_t ldx, const double* R, void* Q, int64_t ldq,
                     cudaStream_t st, bool timed, int n_cols = 0, bool colmajor = false) {
  const int n = n_cols > 0 ? n_cols : p->d.n;
  SolvePlan sp_own;
  if (n_cols > 0) sp_own = plan_solve(n, p->d.dtype, p->smem_optin);
  const SolvePlan& sp = n_cols > 0 ? sp_own : p->sp;
  if (sp.solve_tc && m > 0 && solve_tc_supported(X, m, ldx, Q, ldq)) {
    CU(launch_tri_inverse(R, n, p->W, p->status_d, st));
    if (timed && p->timing) cudaEventRecord(p->ev[5], st);
    const cudaError_t e = launch_solve_tc(p->W, n, (const float*)X, m, ldx, (float*)Q, ldq, p->qws, p->status_d,
                                          p->sms, st, colmajor);
    if (e == cudaSuccess) { p->path |= kPathSolveTC; return RCHOLQR_OK; }
    if (e != cudaErrorNotSupported) return cuda_status(e);
  }
  if (colmajor) return RCHOLQR_E_UNSUPPORTED_INTERNAL;
  if (m > 0) p->path |= kPathSolveDmma;
  if (sp.mstream) {
    CU(launch_tri_prep_blocked(R, n, p->W, p->status_d, st));
    if (timed && p->timing) cudaEventRecord(p->ev[5], st);
    if (m > 0) CU(launch_trsm_mstream(X, p->d.dtype, m, n, ldx, p->W, Q, ldq, p->status_d, p->sms, st));
  } else if (sp.stream_tb > 0) {
    // blocked substitution by column blocks of width tb, each = 2 fp64 DMMA GEMM launches
    const int tb = sp.stream_tb, npad = (n + 7) / 8 * 8;
    CU(launch_tri_prep_blocked(R, n, p->W, p->status_d, st, tb, npad));
    if (timed && p->timing) cudaEventRecord(p->ev[5], st);
    if (m > 0) {
      const size_t need = (size_t)m * tb;
      if (need > p->tbuf_elems) {
        cudaFree(p->tbuf);
        p->tbuf = nullptr; p->tbuf_elems = 0;
        CU(cudaMalloc(&p->tbuf, sizeof(double) * need));
        p->tbuf_elems = need;
      }
      const double* Xd = (const double*)X;
      double* Qd = (double*)Q;
      for (int Jb = 0; Jb < n; Jb += tb) {
        const int bw = std::min(tb, n - Jb);
        // T_J = X_J + Q_{<J} (-R_{<J,J})
        CU(launch_gemm_f64(Qd, ldq, p->W + Jb, npad, Xd + Jb, ldx, p->tbuf, tb, m, bw, Jb, false, p->status_d, st));
        // Q_J = T_J Winv_JJ
        CU(launch_gemm_f64(p->tbuf, tb, p->W + (size_t)Jb * npad + Jb, npad, nullptr, 0, Qd + Jb, ldq, m, bw, bw, true,
                           p->status_d, st));
      }
    }
  } else if (sp.pairs > 0) {
    CU(launch_tri_prep_blocked(R, n, p->W, p->status_d, st));
    if (timed && p->timing) cudaEventRecord(p->ev[5], st);
    if (m > 0) CU(launch_trsm_pairs(sp.pairs, X, p->d.dtype, m, n, ldx, p->W, Q, ldq, p->status_d, p->sms, st));
  } else {
    CU(launch_tri_inverse(R, n, p->W, p->status_d, st));
    if (timed && p->timing) cudaEventRecord(p->ev[5], st);
    if (m > 0) CU(launch_trsm(sp.tr, X, p->d.dtype, m, n, ldx, p->W, Q, ldq, p->status_d, st));
  }
  return RCHOLQR_OK;
}

rcholqr_status read_status(rcholqr_plan p, cudaStream_t st) {
  CU(cudaMemcpyAsync(p->status_h, p->status_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (p->timing) {
    const int pairs[6][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}};
    for (int t = 0; t < 6; ++t) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p->ev[pairs[t][0]], p->ev[pairs[t][1]]) != cudaSuccess) ms = -1.f;
      p->last_ms[t] = ms;
    }
    p->have_timing = true;
  }
  return status_from_word(*p->status_h);
}
}  // namespace

// ---------------------------------------------------------------------------------------------
extern "C" {

#ifdef RCHOLQR_ABLATION
// ablation builds only (not declared in include/rcholqr.h): copy CTA 0's event timeline of the last traced
// kernel (which = 0: tcgen05 solve, 1: sparse tcgen05 sketch) to the host and clear it
int32_t rcholqr_trace_read(int32_t which, void* host, size_t bytes) {
  if (bytes < sizeof(long long) * rcq::kTraceRoles * rcq::kTraceTiles * rcq::kTraceEvents) return -1;
  return which == 0 ? rcq::trace_read_solve(host) : rcq::trace_read_sketch(host);
}
#endif

int32_t rcholqr_version(void) { return RCHOLQR_VERSION; }

const char* rcholqr_strerror(rcholqr_status s) {
  switch (s) {
    case RCHOLQR_OK: return "ok";
    case RCHOLQR_E_INVALID: return "invalid argument";
    case RCHOLQR_E_SHAPE: return "invalid shape (need n >= 1, k >= n, sparse: k % nnz == 0)";
    case RCHOLQR_E_NONFINITE: return "sketch contains NaN/Inf";
    case RCHOLQR_E_SINGULAR: return "R has a zero or non-finite pivot (X not numerically full rank)";
    case RCHOLQR_E_CUDA: return "CUDA error";
    case RCHOLQR_E_NCCL: return "NCCL unavailable or collective failed";
    case RCHOLQR_E_NOMEM: return "out of memory";
  }
  return "unknown status";
}

rcholqr_status rcholqr_create(const rcholqr_desc* desc, rcholqr_plan* out) {
  if (!out) return RCHOLQR_E_INVALID;
  *out = nullptr;
  rcholqr_status vs = validate_desc(desc);
  if (vs != RCHOLQR_OK) return vs;
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (desc->device < 0 || desc->device >= ndev) return RCHOLQR_E_INVALID;
  DeviceGuard dg(desc->device);
  rcholqr_plan p = new (std::nothrow) rcholqr_plan_s();
  if (!p) return RCHOLQR_E_NOMEM;
  p->d = *desc;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, desc->device);
  if (e != cudaSuccess) { delete p; return cuda_status(e); }
  p->sms = prop.multiProcessorCount;
  p->smem_optin = prop.sharedMemPerBlockOptin;
  const int k = desc->k, n = desc->n;
  p->sk = plan_sketch(k, n, desc->dtype, desc->sketch, desc->nnz_per_col, p->sms, p->smem_optin);
  p->sp = plan_solve(n, desc->dtype, p->smem_optin);
  p->qr_kind = plan_qr(k, n, p->smem_optin);
  const size_t kn = (size_t)k * n, nn = (size_t)((n + 7) / 8 * 8) * ((n + 7) / 8 * 8);
  bool okalloc = cudaMalloc(&p->part, sizeof(double) * kn * p->sk.max_splits()) == cudaSuccess &&
                 cudaMalloc(&p->partc, sizeof(double) * kn * p->sk.max_splits()) == cudaSuccess &&
                 cudaMalloc(&p->flag_d, sizeof(int)) == cudaSuccess &&
                 cudaMalloc(&p->qws, solve_tc_workspace()) == cudaSuccess &&
                 (p->qr_kind != kQrBlocked || cudaMalloc(&p->qr_ws, qr_blocked_workspace(k, n)) == cudaSuccess) &&
                 cudaMalloc(&p->P, sizeof(double) * kn) == cudaSuccess &&
                 cudaMalloc(&p->W, sizeof(double) * nn) == cudaSuccess &&
                 cudaMalloc(&p->Awork, sizeof(double) * kn) == cudaSuccess &&
                 cudaMalloc(&p->diag, sizeof(double) * 2 * n) == cudaSuccess &&
                 cudaMalloc(&p->tau, sizeof(double) * n) == cudaSuccess &&
                 cudaMalloc(&p->Rtmp, sizeof(double) * nn) == cudaSuccess &&
                 cudaMalloc(&p->status_d, 2 * sizeof(int)) == cudaSuccess &&   // [status, flag_seen]
                 cudaMallocHost(&p->status_h, sizeof(int)) == cudaSuccess;
  if (okalloc) {
    p->flag_seen_d = p->status_d + 1;
    for (int t = 0; t < 7 && okalloc; ++t) okalloc = cudaEventCreate(&p->ev[t]) == cudaSuccess;
  }
  if (!okalloc) {
    cudaGetLastError();
    rcholqr_destroy(p);
    return RCHOLQR_E_NOMEM;
  }
  if (desc->sketch == RCHOLQR_SRHT) {
    const std::vector<uint64_t> rows = srht_rows_host(desc->seed, k);
    if (cudaMalloc(&p->srht_d, sizeof(uint64_t) * (size_t)k) != cudaSuccess ||
        cudaMemcpy(p->srht_d, rows.data(), sizeof(uint64_t) * (size_t)k, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      rcholqr_destroy(p);
      return RCHOLQR_E_NOMEM;
    }
    p->sk.srht_s = p->srht_d;
  }
  cudaMemset(p->status_d, 0, 2 * sizeof(int));
  *p->status_h = 0;
  *out = p;
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_destroy(rcholqr_plan p) {
  if (!p) return RCHOLQR_OK;
  DeviceGuard dg(p->d.device);
  cudaFree(p->part); cudaFree(p->partc); cudaFree(p->P); cudaFree(p->W); cudaFree(p->Awork); cudaFree(p->diag); cudaFree(p->tau);
  cudaFree(p->Rtmp); cudaFree(p->status_d); cudaFree(p->flag_d); cudaFree(p->qws); cudaFree(p->xdig); cudaFree(p->qr_ws);
  cudaFree(p->gpart); cudaFree(p->gA); cudaFree(p->gW); cudaFree(p->gRp); cudaFree(p->gR1); cudaFree(p->q1buf);
  cudaFree(p->red_part); cudaFree(p->red_partc); cudaFree(p->red_P);
  cudaFree(p->rr_buf); cudaFree(p->rr_Pn); cudaFree(p->rr_A); cudaFree(p->rr_Pg); cudaFree(p->rr_R); cudaFree(p->rr_W);
  cudaFree(p->rr_R11); cudaFree(p->rr_d); cudaFree(p->rr_cpart); cudaFree(p->rr_cspart); cudaFree(p->rr_sd); cudaFree(p->rr_si);
  cudaFree(p->rr_perm); cudaFree(p->rr_qst); cudaFree(p->rr_xr); cudaFree(p->srht_d);
  if (p->status_h) cudaFreeHost(p->status_h);
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  if (p->gstream) cudaStreamDestroy(p->gstream);
  cudaFree(p->xbuf); cudaFree(p->qbuf); cudaFree(p->rbuf); cudaFree(p->sbuf); cudaFree(p->tbuf);
  for (int t = 0; t < 7; ++t)
    if (p->ev[t]) cudaEventDestroy(p->ev[t]);
  delete p;
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_factor_async(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, void* Q,
                                    int64_t ldq, double* R, double* S, void* stream) {
  rcholqr_status a = check_factor_args(p, X, m, ro, ldx, Q, ldq);
  if (a != RCHOLQR_OK) return a;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = p->d.k, n = p->d.n;
  double* Rout = R ? R : p->Rtmp;
  p->path = 0;   // a new call: clear the path bits and the device status / overflow-seen words
  CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
  rcholqr_status s = do_sketch(p, X, m, ro, ldx, p->P, st);
  if (s != RCHOLQR_OK) return s;
  CU(launch_qr(p->qr_kind, p->P, k, n, Rout, p->Awork, p->diag, p->tau, p->qr_ws, p->status_d, st));
  if (S) CU(launch_form_s(p->Awork, p->tau, p->diag, k, n, S, p->status_d, st));
  if (p->timing) cudaEventRecord(p->ev[4], st);
  rcholqr_status s2 = solve(p, X, m, ldx, Rout, Q, ldq, st, true);
  if (s2 != RCHOLQR_OK) return s2;
  if (p->timing) cudaEventRecord(p->ev[6], st);
  return RCHOLQR_OK;
}

// Launch-bound problems (C1: 10^4 x 20, a few microseconds of work per kernel; PAPER.md:163 expects the small
// steps to "not have much impact"): the whole chain -- status memset, sketch, reduction, small QR, triangular
// prep, solve -- is captured once per argument tuple into a CUDA graph and replayed with ONE launch.
rcholqr_status rcholqr_factor_graph(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, void* Q,
                                    int64_t ldq, double* R, double* S, void* stream) {
  rcholqr_status a = check_factor_args(p, X, m, ro, ldx, Q, ldq);
  if (a != RCHOLQR_OK) return a;
  if (p->d.nccl_comm || p->timing)   // collective / event-timed chains are launched directly
    return rcholqr_factor_async(p, X, m, ro, ldx, Q, ldq, R, S, stream);
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  rcholqr_plan_s::GraphKey key;
  key.X = X; key.m = m; key.ro = ro; key.ldx = ldx; key.Q = Q; key.ldq = ldq; key.R = R; key.S = S;
  key.xdig = p->xdig; key.tbuf = p->tbuf;
  if (p->gexec && key == p->gkey) {
    p->path = p->gpath;
    CU(cudaGraphLaunch(p->gexec, st));
    return RCHOLQR_OK;
  }
  // new arguments: this call runs directly (it also sizes every lazily grown workspace, so the capture
  // below allocates nothing), then the same chain is captured for the calls that follow
  if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
  rcholqr_status s = rcholqr_factor_async(p, X, m, ro, ldx, Q, ldq, R, S, stream);
  if (s != RCHOLQR_OK) return s;
  const unsigned path = p->path;
  if (!p->gstream) CU(cudaStreamCreateWithFlags(&p->gstream, cudaStreamNonBlocking));
  CU(cudaStreamSynchronize(st));   // the capture pass re-issues (does not run) the chain; keep it off the live buffers' timeline
  if (cudaStreamBeginCapture(p->gstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) { cudaGetLastError(); return RCHOLQR_OK; }
  const rcholqr_status cs = rcholqr_factor_async(p, X, m, ro, ldx, Q, ldq, R, S, p->gstream);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(p->gstream, &g);
  p->path = path;
  if (cs == RCHOLQR_OK && ce == cudaSuccess && g && cudaGraphInstantiate(&p->gexec, g, 0) == cudaSuccess) {
    key.xdig = p->xdig; key.tbuf = p->tbuf;      // as the direct run above left them
    p->gkey = key;
    p->gpath = path;
  } else {
    cudaGetLastError();          // not capturable here: later calls keep launching directly
    p->gexec = nullptr;
  }
  if (g) cudaGraphDestroy(g);
  return RCHOLQR_OK;
}

// Gram / Cholesky workspace of Alg. 3 and RRRCholeskyQR2 (n x n each; the partials hold the most
// splits any column count <= n uses), allocated on first use.
static bool ensure_gram(rcholqr_plan p) {
  if (p->gA) return true;
  const int n = p->d.n;
  const size_t nn = (size_t)n * n;
  p->gram_splits = gram_splits(n, p->sms);
  size_t part_elems = nn * (size_t)p->gram_splits;
  for (int r = 1; r <= n; r = r < 128 ? 128 : n + 1)     // n <= 128 uses the most splits (4 per SM)
    part_elems = std::max(part_elems, (size_t)r * r * (size_t)gram_splits(std::min(r, n), p->sms));
  bool ok = cudaMalloc(&p->gpart, sizeof(double) * part_elems) == cudaSuccess &&
            cudaMalloc(&p->gA, sizeof(double) * nn) == cudaSuccess &&
            cudaMalloc(&p->gW, sizeof(double) * nn) == cudaSuccess &&
            cudaMalloc(&p->gRp, sizeof(double) * nn) == cudaSuccess &&
            cudaMalloc(&p->gR1, sizeof(double) * nn) == cudaSuccess;
  if (!ok) { cudaGetLastError(); return false; }
  return true;
}

rcholqr_status rcholqr_factor2(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, void* Q,
                               int64_t ldq, double* R, double* Rprime, int32_t implicit, void* stream) {
  rcholqr_status a = check_factor_args(p, X, m, ro, ldx, Q, ldq);
  if (a != RCHOLQR_OK) return a;
  if (!R || (implicit && !Rprime)) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int n = p->d.n;
  const size_t nn = (size_t)n * n, es = esize(p->d.dtype);
  if (!ensure_gram(p)) return RCHOLQR_E_NOMEM;
  // Q1: the caller's Q (implicit form) or a plan-owned buffer (explicit form; Q must not alias it)
  void* Q1 = Q;
  int64_t ldq1 = ldq;
  if (!implicit && m > 0) {
    const size_t need = (size_t)m * n * es;
    if (need > p->q1_bytes) {
      cudaFree(p->q1buf);
      p->q1buf = nullptr; p->q1_bytes = 0;
      CU(cudaMalloc(&p->q1buf, need));
      p->q1_bytes = need;
    }
    Q1 = p->q1buf;
    ldq1 = n;
  }
  // 1. RCholeskyQR (Alg. 2): Q1, R1
  rcholqr_status s = rcholqr_factor_async(p, X, m, ro, ldx, Q1, ldq1, p->gR1, nullptr, stream);
  if (s != RCHOLQR_OK) return s;
  // 2. A = Q1^T Q1 (+ all-reduce)
  if (m > 0) CU(launch_gram(Q1, p->d.dtype, m, n, ldq1, p->gram_splits, p->gpart, p->gA, p->status_d, st));
  else CU(cudaMemsetAsync(p->gA, 0, sizeof(double) * nn, st));
  if (p->d.nccl_comm) {
    if (!nccl_load()) return RCHOLQR_E_NCCL;
    if (g_nccl.AllReduce(p->gA, p->gA, nn, ncclFloat64, ncclSum, (ncclComm_t)p->d.nccl_comm, st) != ncclSuccess)
      return RCHOLQR_E_NCCL;
  }
  // 3. R' = chol(A), R = R' R1
  double* Rp = Rprime ? Rprime : p->gRp;
  CU(launch_cholesky(p->gA, n, p->gW, Rp, p->status_d, st));
  CU(launch_trmm_upper(Rp, p->gR1, n, R, p->status_d, st));
  // 4. Q = Q1 R'^{-1} (explicit form)
  if (!implicit) {
    rcholqr_status s2 = solve(p, Q1, m, ldq1, Rp, Q, ldq, st, false);
    if (s2 != RCHOLQR_OK) return s2;
  }
  return read_status(p, st);
}

rcholqr_status rcholqr_factor_reduced(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, int32_t l,
                                      double* Z, double* R, double* S, double* Y, void* stream) {
  if (!p || !Z || l < 1 || m < 0 || ro < 0 || ldx < p->d.n || (m > 0 && !X)) return RCHOLQR_E_INVALID;
  const int k = p->d.k, n = p->d.n;
  const bool gauss = p->d.sketch == RCHOLQR_GAUSSIAN;
  if ((int64_t)(k + (int64_t)l) * n > (int64_t)1 << 28) return RCHOLQR_E_SHAPE;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  if (p->red_l != l) {   // the (k + l)-row launch (Gaussian Theta) or the l-row extractor launch (sparse Theta)
    cudaFree(p->red_part); cudaFree(p->red_partc); cudaFree(p->red_P);
    p->red_part = p->red_partc = p->red_P = nullptr;
    p->red_l = 0;
    p->red_sk = plan_sketch(gauss ? k + l : l, n, p->d.dtype, RCHOLQR_GAUSSIAN, p->d.nnz_per_col, p->sms, p->smem_optin);
    const size_t rows = gauss ? (size_t)(k + l) : (size_t)l;
    const size_t elems = rows * n * p->red_sk.max_splits();
    bool ok = cudaMalloc(&p->red_part, sizeof(double) * elems) == cudaSuccess &&
              cudaMalloc(&p->red_partc, sizeof(double) * elems) == cudaSuccess &&
              cudaMalloc(&p->red_P, sizeof(double) * (size_t)(k + l) * n) == cudaSuccess;
    if (!ok) { cudaGetLastError(); return RCHOLQR_E_NOMEM; }
    p->red_l = l;
  }
  double* P = p->red_P;
  double* Yd = p->red_P + (size_t)k * n;
  double* Rout = R ? R : p->Rtmp;
  p->path = 0;   // a new call: clear the path bits and the device status / overflow-seen words
  CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
  // 1. P = Theta X, Y = L X: one (k + l)-row pass for a Gaussian Theta, else the sparse sketch and the
  //    l-row Gaussian extract; one all-reduce of [P; Y] either way
  rcholqr_status s;
  const bool t = p->timing;
  if (gauss) {   // (library events as for rcholqr_factor: sketch | reduce | all-reduce | QR | - | Z)
    s = do_sketch(p, X, m, ro, ldx, P, st, &p->red_sk, k + l, p->red_part, p->red_partc, k, true);
  } else {       // events: both passes (sparse P, Gaussian Y, their reductions) | - | all-reduce
    if (t) cudaEventRecord(p->ev[0], st);
    p->timing = false;
    s = do_sketch(p, X, m, ro, ldx, P, st, &p->sk, k, p->part, p->partc, 0, false);
    if (s == RCHOLQR_OK) s = do_sketch(p, X, m, ro, ldx, Yd, st, &p->red_sk, l, p->red_part, p->red_partc, 0, false);
    p->timing = t;
    if (t) { cudaEventRecord(p->ev[1], st); cudaEventRecord(p->ev[2], st); }
    if (s == RCHOLQR_OK && p->d.nccl_comm) {
      if (!nccl_load()) s = RCHOLQR_E_NCCL;
      else if (g_nccl.AllReduce(P, P, (size_t)(k + l) * n, ncclFloat64, ncclSum, (ncclComm_t)p->d.nccl_comm, st) !=
               ncclSuccess)
        s = RCHOLQR_E_NCCL;
    }
    if (t) cudaEventRecord(p->ev[3], st);
  }
  if (s != RCHOLQR_OK) { p->timing = t; return s; }
  // 2. [S, R] = QR(P)
  cudaError_t e = launch_qr(p->qr_kind, P, k, n, Rout, p->Awork, p->diag, p->tau, p->qr_ws, p->status_d, st);
  if (e == cudaSuccess && S) e = launch_form_s(p->Awork, p->tau, p->diag, k, n, S, p->status_d, st);
  if (p->timing) { cudaEventRecord(p->ev[4], st); cudaEventRecord(p->ev[5], st); }
  // 3. Z = Y R^{-1}
  if (e == cudaSuccess) e = launch_rowsub(Yd, l, n, Rout, Z, p->status_d, st);
  if (p->timing) cudaEventRecord(p->ev[6], st);
  if (e == cudaSuccess && Y) e = cudaMemcpyAsync(Y, Yd, sizeof(double) * (size_t)l * n, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) { p->timing = t; return cuda_status(e); }
  rcholqr_status r = read_status(p, st);
  p->timing = t;
  return r;
}

rcholqr_status rcholqr_factor_rr(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, double tau,
                                 double f, int32_t rank_fixed, void* Q, int64_t ldq, double* R, int32_t* perm,
                                 double* D, double* S, int32_t* rank_out, int32_t* swaps_out, void* stream) {
  rcholqr_status a = check_factor_args(p, X, m, ro, ldx, Q, ldq);
  if (a != RCHOLQR_OK) return a;
  if (!R || !perm || !rank_out || !(f > 1.0) || !(tau >= 0.0) || !std::isfinite(tau) || rank_fixed < 0)
    return RCHOLQR_E_INVALID;
  const int k = p->d.k, n = p->d.n;
  if (n > 1024) return RCHOLQR_E_SHAPE;                      // the pivoting kernel's norm arrays
  const size_t kn = (size_t)k * n, nn = (size_t)n * n, es = esize(p->d.dtype);
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  if (!p->rr_buf) {
    p->rr_splits = colsq_splits(n, p->sms);
    bool ok = cudaMalloc(&p->rr_buf, sizeof(double) * (kn + n)) == cudaSuccess &&
              cudaMalloc(&p->rr_Pn, sizeof(double) * kn) == cudaSuccess &&
              cudaMalloc(&p->rr_A, sizeof(double) * kn) == cudaSuccess &&
              cudaMalloc(&p->rr_Pg, sizeof(double) * kn) == cudaSuccess &&
              cudaMalloc(&p->rr_R, sizeof(double) * nn) == cudaSuccess &&
              cudaMalloc(&p->rr_W, sizeof(double) * nn) == cudaSuccess &&
              cudaMalloc(&p->rr_R11, sizeof(double) * nn) == cudaSuccess &&
              cudaMalloc(&p->rr_d, sizeof(double) * n) == cudaSuccess &&
              cudaMalloc(&p->rr_cpart, sizeof(double) * n * p->rr_splits) == cudaSuccess &&
              cudaMalloc(&p->rr_cspart, sizeof(double) * n * kXdigSplitBlocks) == cudaSuccess &&
              cudaMalloc(&p->rr_sd, sizeof(double) * 2) == cudaSuccess &&
              cudaMalloc(&p->rr_si, sizeof(int) * 2) == cudaSuccess &&
              cudaMalloc(&p->rr_perm, sizeof(int) * n) == cudaSuccess &&
              cudaMalloc(&p->rr_qst, sizeof(int)) == cudaSuccess;
    if (!ok) { cudaGetLastError(); return RCHOLQR_E_NOMEM; }
  }
  const bool t = p->timing;
  p->timing = false;
  struct Restore { rcholqr_plan p; bool t; ~Restore() { p->timing = t; } } restore{p, t};
  p->path = 0;   // a new call: clear the path bits and the device status / overflow-seen words
  CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
  // library events: sketch | column norms | all-reduce | RRQR (incl. host decisions) | gather | solve
  if (t) cudaEventRecord(p->ev[0], st);
  // 1. P = Theta X and the column sums of squares, all-reduced together as [P; colsq]
  //    (D "along with P <- Theta X in step 1 during the same pass": the pre-split Gaussian path sums
  //    the squares in its digit-split kernel; the other sketch paths fall back to one colsq pass over X)
  bool cs_fused = false;
  rcholqr_status s = do_sketch(p, X, m, ro, ldx, p->rr_buf, st, nullptr, 0, nullptr, nullptr, 0, false, p->rr_cspart,
                               p->rr_buf + kn, &cs_fused);
  if (s != RCHOLQR_OK) return s;
  if (t) cudaEventRecord(p->ev[1], st);
  if (cs_fused) p->path |= RCHOLQR_PATH_COLSQ_FUSED;
  else if (m > 0) CU(launch_colsq(X, p->d.dtype, m, n, ldx, p->rr_splits, p->rr_cpart, p->rr_buf + kn, p->status_d, st));
  else CU(cudaMemsetAsync(p->rr_buf + kn, 0, sizeof(double) * n, st));
  if (t) cudaEventRecord(p->ev[2], st);
  if (p->d.nccl_comm) {
    if (!nccl_load()) return RCHOLQR_E_NCCL;
    if (g_nccl.AllReduce(p->rr_buf, p->rr_buf, kn + n, ncclFloat64, ncclSum, (ncclComm_t)p->d.nccl_comm, st) !=
        ncclSuccess)
      return RCHOLQR_E_NCCL;
  }
  if (t) cudaEventRecord(p->ev[3], st);
  // (a non-finite P is caught by the final status read: every later kernel honours the status word)
  // P <- P D^{-1}; column pivoting picks Pi
  CU(launch_rr_normalize(p->rr_buf, k, n, p->rr_Pn, p->rr_d, st));
  CU(launch_qrcp(p->rr_Pn, k, n, p->rr_A, p->rr_perm, st));
  std::vector<int> hperm(n);
  // 2.-3. R of P(:, Pi) (the Householder kernels of Alg. 2), the rank rule, Gu-Eisenstat swaps
  int r = 0, swaps = 0;
  for (int pass = 0;; ++pass) {
    CU(launch_rr_gather(p->rr_Pn, k, n, p->rr_perm, p->rr_Pg, st));
    CU(cudaMemsetAsync(p->rr_qst, 0, sizeof(int), st));   // zero pivots beyond the rank are expected
    CU(launch_qr(p->qr_kind, p->rr_Pg, k, n, p->rr_R, p->Awork, p->diag, p->tau, p->qr_ws, p->rr_qst, st));
    if (pass == 0) {   // one host round trip: the permutation and the rank
      CU(launch_rank(p->rr_R, n, tau, rank_fixed, p->rr_si, p->rr_sd, st));
      CU(cudaMemcpyAsync(hperm.data(), p->rr_perm, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(&r, p->rr_si, sizeof(int), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
    }
    if (r == 0 || r == n || pass >= 64) break;
    double rho2 = 0.0;
    int flat = 0;
    CU(launch_strong(p->rr_R, n, r, p->rr_W, p->rr_sd + 1, p->rr_si + 1, st));
    CU(cudaMemcpyAsync(&rho2, p->rr_sd + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(&flat, p->rr_si + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (!(rho2 > f * f) || flat < 0 || flat >= r * (n - r)) break;
    const int bi = flat / (n - r), bj = flat % (n - r);
    std::swap(hperm[bi], hperm[r + bj]);
    CU(cudaMemcpyAsync(p->rr_perm, hperm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
    ++swaps;
  }
  *rank_out = r;
  if (swaps_out) *swaps_out = swaps;
  CU(cudaMemcpyAsync(perm, p->rr_perm, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
  if (D) CU(cudaMemcpyAsync(D, p->rr_d, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (S) CU(launch_form_s(p->Awork, p->tau, p->diag, k, n, S, p->rr_qst, st));
  if (r == 0) {   // rank 0: E_SINGULAR, unless the sketch (or D) was non-finite -- then that is the diagnosis
    CU(cudaMemsetAsync(R, 0, sizeof(double) * nn, st));
    const rcholqr_status s0 = read_status(p, st);
    return s0 == RCHOLQR_E_NONFINITE ? s0 : RCHOLQR_E_SINGULAR;
  }
  // R <- R(1:r, :) Pi^T D Pi;  4. Q = (X Pi(:, 1:r)) R11^{-1}
  CU(launch_rr_finalize(p->rr_R, n, r, p->rr_d, p->rr_perm, R, p->rr_R11, st));
  if (t) cudaEventRecord(p->ev[4], st);
  if (m > 0) {
    const size_t need = (size_t)m * r * es;
    if (need > p->rr_xr_bytes) {
      cudaFree(p->rr_xr);
      p->rr_xr = nullptr; p->rr_xr_bytes = 0;
      CU(cudaMalloc(&p->rr_xr, need));
      p->rr_xr_bytes = need;
    }
    CU(launch_gather_x(X, p->d.dtype, m, ldx, p->rr_perm, r, p->rr_xr, p->sms, st));
    if (t) cudaEventRecord(p->ev[5], st);
    CU(launch_check_diag(p->rr_R11, r, p->status_d, st));
    s = solve(p, p->rr_xr, m, r, p->rr_R11, Q, ldq, st, false, r);
    if (s != RCHOLQR_OK) return s;
  } else if (t) {
    cudaEventRecord(p->ev[5], st);
  }
  if (t) cudaEventRecord(p->ev[6], st);
  p->timing = t;
  return read_status(p, st);
}

rcholqr_status rcholqr_factor_rr2(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, double tau,
                                  double f, int32_t rank_fixed, void* Q, int64_t ldq, double* R, double* Rprime,
                                  int32_t* perm, double* D, int32_t* rank_out, int32_t* swaps_out, void* stream) {
  rcholqr_status a = check_factor_args(p, X, m, ro, ldx, Q, ldq);
  if (a != RCHOLQR_OK) return a;
  if (!R || !perm || !rank_out) return RCHOLQR_E_INVALID;
  const int n = p->d.n;
  const size_t es = esize(p->d.dtype);
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  if (!ensure_gram(p)) return RCHOLQR_E_NOMEM;
  if (m > 0) {                                                 // Q1: plan-owned m x n (first r columns used)
    const size_t need = (size_t)m * n * es;
    if (need > p->q1_bytes) {
      cudaFree(p->q1buf);
      p->q1buf = nullptr; p->q1_bytes = 0;
      CU(cudaMalloc(&p->q1buf, need));
      p->q1_bytes = need;
    }
  }
  // 1. Alg. 7: Q1 (m x r), R1 (r x n), perm, r
  int32_t r = 0;
  rcholqr_status s = rcholqr_factor_rr(p, X, m, ro, ldx, tau, f, rank_fixed, m > 0 ? p->q1buf : Q, n, p->gR1, perm, D,
                                       nullptr, &r, swaps_out, stream);
  *rank_out = r;
  if (s != RCHOLQR_OK) return s;
  // 2. A = Q1^T Q1 (r x r, + all-reduce); 3. R' = chol(A), R = R' R1; 4. Q = Q1 R'^{-1}
  CU(cudaMemsetAsync(p->status_d, 0, sizeof(int), st));
  if (m > 0) CU(launch_gram(p->q1buf, p->d.dtype, m, r, n, gram_splits(r, p->sms), p->gpart, p->gA, p->status_d, st));
  else CU(cudaMemsetAsync(p->gA, 0, sizeof(double) * (size_t)r * r, st));
  if (p->d.nccl_comm) {
    if (!nccl_load()) return RCHOLQR_E_NCCL;
    if (g_nccl.AllReduce(p->gA, p->gA, (size_t)r * r, ncclFloat64, ncclSum, (ncclComm_t)p->d.nccl_comm, st) !=
        ncclSuccess)
      return RCHOLQR_E_NCCL;
  }
  double* Rp = Rprime ? Rprime : p->gRp;
  CU(launch_cholesky(p->gA, r, p->gW, Rp, p->status_d, st));
  CU(launch_trmm_trap(Rp, r, p->gR1, n, R, p->status_d, st));
  if (m > 0) {
    s = solve(p, p->q1buf, m, n, Rp, Q, ldq, st, false, r);
    if (s != RCHOLQR_OK) return s;
  }
  const bool t = p->timing;
  p->timing = false;
  rcholqr_status rs = read_status(p, st);
  p->timing = t;
  return rs;
}

rcholqr_status rcholqr_factor_colmajor(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, void* Q,
                                       int64_t ldq, double* R, double* S, void* stream) {
  if (!p || m < 0 || ro < 0 || ldx < std::max<int64_t>(m, 1) || ldq < std::max<int64_t>(m, 1) ||
      (m > 0 && (!X || !Q)))
    return RCHOLQR_E_INVALID;
  const int n = p->d.n;
  const size_t es = esize(p->d.dtype);
  if (m > 0 && overlaps(X, span_bytes(n, ldx, (int)m, es), Q, span_bytes(n, ldq, (int)m, es))) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  // Native path (column-wise storage keeps the sketch a single pass): the tcgen05 sketch (sparse-sign /
  // Rademacher / SRHT E tile, or the pre-split Gaussian) and the tcgen05 digit solve read X and write Q column-major
  // through their tensor maps -- no transposes, the same two reads of X and one write of Q as the row-major
  // path.  It needs fp32 X with n <= 128 (the digit solve) and 16-byte aligned bases and column pitches; if a
  // sketch kernel raises its headroom-overflow flag (the guarded fallbacks are row-major kernels) or a kernel
  // is not applicable, the call is redone through the layout adapter below.
  if (m > 0 && p->sp.solve_tc && solve_tc_supported(X, m, ldx, Q, ldq) && !getenv("RCHOLQR_COLMAJOR_ADAPTER")) {
    const int k = p->d.k;
    double* Rout = R ? R : p->Rtmp;
    p->path = 0;
    CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
    rcholqr_status s = do_sketch(p, X, m, ro, ldx, p->P, st, nullptr, 0, nullptr, nullptr, 0, true, nullptr, nullptr,
                                 nullptr, true);
    if (s == RCHOLQR_OK) {
      CU(launch_qr(p->qr_kind, p->P, k, n, Rout, p->Awork, p->diag, p->tau, p->qr_ws, p->status_d, st));
      if (S) CU(launch_form_s(p->Awork, p->tau, p->diag, k, n, S, p->status_d, st));
      if (p->timing) cudaEventRecord(p->ev[4], st);
      s = solve(p, X, m, ldx, Rout, Q, ldq, st, true, 0, true);
      if (s == RCHOLQR_OK) {
        if (p->timing) cudaEventRecord(p->ev[6], st);
        int words[2] = {0, 0};                                       // [status, sketch overflow seen]
        CU(cudaMemcpyAsync(words, p->status_d, sizeof(words), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (!words[1]) {
          p->path |= kPathColmajorNative;
          return read_status(p, st);
        }
      }
    }
    if (s != RCHOLQR_OK && s != RCHOLQR_E_UNSUPPORTED_INTERNAL) return s;
  }
  const size_t need = (size_t)std::max<int64_t>(m, 1) * n * es;   // row-major staging of X and Q
  if (need > p->xq_bytes) {
    cudaFree(p->xbuf); cudaFree(p->qbuf);
    p->xbuf = p->qbuf = nullptr; p->xq_bytes = 0;
    CU(cudaMalloc(&p->xbuf, need));
    CU(cudaMalloc(&p->qbuf, need));
    p->xq_bytes = need;
  }
  // X (n columns of length m, ld ldx) -> row-major m x n; the row-major path; Q back to column-major
  CU(launch_transpose(X, n, m, ldx, p->xbuf, n, es, st));
  rcholqr_status s = rcholqr_factor_async(p, p->xbuf, m, ro, n, p->qbuf, n, R, S, stream);
  if (s != RCHOLQR_OK) return s;
  CU(launch_transpose(p->qbuf, m, n, n, Q, ldq, es, st));
  return rcholqr_query_status(p, stream);
}

rcholqr_status rcholqr_query_status(rcholqr_plan p, void* stream) {
  if (!p) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  return read_status(p, (cudaStream_t)stream);
}

rcholqr_status rcholqr_factor(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, void* Q,
                              int64_t ldq, double* R, double* S, void* stream) {
  rcholqr_status s = rcholqr_factor_async(p, X, m, ro, ldx, Q, ldq, R, S, stream);
  if (s != RCHOLQR_OK) return s;
  return rcholqr_query_status(p, stream);
}

rcholqr_status rcholqr_factor_host(rcholqr_plan p, const void* Xh, int64_t m, int64_t ro, int64_t ldx, void* Qh,
                                   int64_t ldq, double* Rh, double* Sh, void* stream) {
  if (!p || !Rh) return RCHOLQR_E_INVALID;
  const int n = p->d.n, k = p->d.k;
  if (m < 0 || ldx < n || ldq < n || (m > 0 && (!Xh || !Qh))) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t es = esize(p->d.dtype);
  const size_t need = (size_t)std::max<int64_t>(m, 1) * n * es;
  if (need > p->xq_bytes) {
    cudaFree(p->xbuf); cudaFree(p->qbuf);
    p->xbuf = p->qbuf = nullptr; p->xq_bytes = 0;
    CU(cudaMalloc(&p->xbuf, need));
    CU(cudaMalloc(&p->qbuf, need));
    p->xq_bytes = need;
  }
  if (!p->rbuf) CU(cudaMalloc(&p->rbuf, sizeof(double) * (size_t)n * n));
  if (Sh && !p->sbuf) CU(cudaMalloc(&p->sbuf, sizeof(double) * (size_t)k * n));
  if (m > 0 && ldx == n) CU(cudaMemcpyAsync(p->xbuf, Xh, (size_t)m * n * es, cudaMemcpyHostToDevice, st));
  else if (m > 0) CU(cudaMemcpy2DAsync(p->xbuf, n * es, Xh, ldx * es, n * es, m, cudaMemcpyHostToDevice, st));
  rcholqr_status s = rcholqr_factor_async(p, p->xbuf, m, ro, n, p->qbuf, n, p->rbuf, Sh ? p->sbuf : nullptr, st);
  if (s != RCHOLQR_OK) return s;
  if (m > 0 && ldq == n) CU(cudaMemcpyAsync(Qh, p->qbuf, (size_t)m * n * es, cudaMemcpyDeviceToHost, st));
  else if (m > 0) CU(cudaMemcpy2DAsync(Qh, ldq * es, p->qbuf, n * es, n * es, m, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(Rh, p->rbuf, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToHost, st));
  if (Sh) CU(cudaMemcpyAsync(Sh, p->sbuf, sizeof(double) * (size_t)k * n, cudaMemcpyDeviceToHost, st));
  return read_status(p, st);
}

rcholqr_status rcholqr_sketch(rcholqr_plan p, const void* X, int64_t m, int64_t ro, int64_t ldx, double* P,
                              void* stream) {
  if (!p || !P || m < 0 || ro < 0 || ldx < p->d.n || (m > 0 && !X)) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  p->path = 0;   // a new call: clear the path bits and the device status / overflow-seen words
  CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
  rcholqr_status s = do_sketch(p, X, m, ro, ldx, P, st);
  if (s != RCHOLQR_OK) return s;
  const bool t = p->timing;
  p->timing = false;
  s = read_status(p, st);
  p->timing = t;
  return s;
}

rcholqr_status rcholqr_small_qr(rcholqr_plan p, const double* P, double* R, double* S, void* stream) {
  if (!p || !P || !R) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int k = p->d.k, n = p->d.n;
  p->path = 0;   // a new call: clear the path bits and the device status / overflow-seen words
  CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
  CU(launch_qr(p->qr_kind, P, k, n, R, p->Awork, p->diag, p->tau, p->qr_ws, p->status_d, st));
  if (S) CU(launch_form_s(p->Awork, p->tau, p->diag, k, n, S, p->status_d, st));
  const bool t = p->timing;
  p->timing = false;
  rcholqr_status s = read_status(p, st);
  p->timing = t;
  return s;
}

rcholqr_status rcholqr_tri_solve(rcholqr_plan p, const void* X, int64_t m, int64_t ldx, const double* R, void* Q,
                                 int64_t ldq, void* stream) {
  rcholqr_status a = check_factor_args(p, X, m, 0, ldx, Q, ldq);
  if (a != RCHOLQR_OK) return a;
  if (!R) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  const int n = p->d.n;
  p->path = 0;   // a new call: clear the path bits and the device status / overflow-seen words
  CU(cudaMemsetAsync(p->status_d, 0, 2 * sizeof(int), st));
  CU(launch_check_diag(R, n, p->status_d, st));
  rcholqr_status s2 = solve(p, X, m, ldx, R, Q, ldq, st, false);
  if (s2 != RCHOLQR_OK) return s2;
  const bool t = p->timing;
  p->timing = false;
  rcholqr_status s = read_status(p, st);
  p->timing = t;
  return s;
}

rcholqr_status rcholqr_theta_export(uint64_t seed, int32_t k, int32_t sketch, int32_t zeta, int64_t ro, int64_t m,
                                    float* Z, int32_t* rows, int8_t* signs, void* stream) {
  if (k < 1 || m < 0 || ro < 0) return RCHOLQR_E_INVALID;
  if (sketch != RCHOLQR_GAUSSIAN && sketch != RCHOLQR_SPARSE_SIGN && sketch != RCHOLQR_RADEMACHER &&
      sketch != RCHOLQR_SRHT)
    return RCHOLQR_E_INVALID;
  if (sketch == RCHOLQR_SPARSE_SIGN && (zeta < 1 || zeta > k || k % zeta != 0)) return RCHOLQR_E_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t* sd = nullptr;
  if (sketch == RCHOLQR_SRHT) {
    const std::vector<uint64_t> rows_h = srht_rows_host(seed, k);
    CU(cudaMalloc(&sd, sizeof(uint64_t) * (size_t)k));
    CU(cudaMemcpy(sd, rows_h.data(), sizeof(uint64_t) * (size_t)k, cudaMemcpyHostToDevice));
  }
  cudaError_t e = launch_theta_export(seed, k, sketch, zeta, ro, m, Z, rows, signs, st, sd);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(sd);
  CU(e);
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) return RCHOLQR_E_INVALID;
  if (!nccl_load()) return RCHOLQR_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return RCHOLQR_E_NCCL;
  memcpy(id_out, &id, 128);
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return RCHOLQR_E_INVALID;
  *comm = nullptr;
  if (!nccl_load()) return RCHOLQR_E_NCCL;
  DeviceGuard dg(device);
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t c = nullptr;
  if (g_nccl.CommInitRank(&c, nranks, uid, rank) != ncclSuccess) return RCHOLQR_E_NCCL;
  *comm = (void*)c;
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_comm_destroy(void* comm) {
  if (!comm) return RCHOLQR_OK;
  if (!nccl_load()) return RCHOLQR_E_NCCL;
  return g_nccl.CommDestroy((ncclComm_t)comm) == ncclSuccess ? RCHOLQR_OK : RCHOLQR_E_NCCL;
}

int32_t rcholqr_launches_per_factor(rcholqr_plan p, int64_t m) {
  if (!p) return -1;
  // Our kernels per factor (without S), assuming 16-byte aligned X/Q so the tensor-core paths run;
  // memsets and the NCCL all-reduce are not counted.
  //   sketch: [tcgen05 sketch +] the CUDA-core kernel (its guarded fallback, exits at once) + reduce
  //   QR: 1 | triangular prep (blocked prep or R^{-1}): 1 | solve: tcgen05 (W-digit prep + solve) = 2,
  //   streamed fp64 GEMMs = 2 per column block, else 1.
  const bool gauss_tc = p->sk.tc && 2.0 * p->d.k * (double)m * p->d.n >= gauss_tc_min_work();
  const bool tc_sketch = p->sk.sp_tc || (p->sk.kind < kSketchSparse && (gauss_tc || p->sk.rad_tc));
  int sketch_launches = (tc_sketch ? 2 : 1) + 1;
  if (p->sk.fwht) sketch_launches = (p->d.k + 1023) / 1024 + 1;   // SRHT transform launches (no guarded fallback) + reduce
  if (tc_sketch && p->sk.kind < kSketchSparse && gauss_tc && m > 0) {   // pre-split: (column maxima + digit planes + sketch) per chunk
    const size_t cap = gauss_tcp_chunk_workspace(m, p->d.n, p->d.dtype, p->sk.tc_splits);
    int64_t chunk = m;
    while (chunk > 32 && gauss_tcp_workspace(chunk, p->d.n, p->d.dtype, p->sk.tc_splits) > cap) chunk = (chunk + 1) / 2;
    const int64_t chunks = (m + chunk - 1) / chunk;
    sketch_launches += (int)(3 * chunks - 1);
  }
  int solve_launches = 1;
  if (p->sp.solve_tc) solve_launches = 2;
  else if (p->sp.stream_tb > 0) solve_launches = 2 * ((p->d.n + p->sp.stream_tb - 1) / p->sp.stream_tb);
  int qr_launches = 1;
  if (p->qr_kind == kQrBlocked) {   // copy + per panel (panel kernel + 3 GEMMs, the last panel 1) + finalize
    const int panels = (p->d.n + 31) / 32;
    qr_launches = 2 + panels + 3 * (panels - 1);
  }
  return (m > 0 ? sketch_launches : 0) + qr_launches + 1 + (m > 0 ? solve_launches : 0);
}

rcholqr_status rcholqr_last_path(rcholqr_plan p, uint32_t* out, void* stream) {
  if (!p || !out) return RCHOLQR_E_INVALID;
  DeviceGuard dg(p->d.device);
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(p->status_h, p->flag_seen_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  *out = p->path | (*p->status_h ? kPathSketchFallback : 0u);
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_set_timing(rcholqr_plan p, int32_t enable) {
  if (!p) return RCHOLQR_E_INVALID;
  p->timing = enable != 0;
  return RCHOLQR_OK;
}

rcholqr_status rcholqr_last_timings(rcholqr_plan p, float out_ms[6]) {
  if (!p || !out_ms) return RCHOLQR_E_INVALID;
  for (int t = 0; t < 6; ++t) out_ms[t] = p->have_timing ? p->last_ms[t] : -1.f;
  return RCHOLQR_OK;
}

}  // extern "C"
