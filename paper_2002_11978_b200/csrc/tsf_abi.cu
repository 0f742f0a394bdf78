// C ABI of the tsfrac B200 engine: plans, tables, dispatch, native march.
// Declarations and reference mapping: include/tsfrac_b200.h.
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tsfrac_b200.h"
#include "tsf_dispatch.h"
#include "tsf_large_api.h"
#include "tsf_soe.cuh"
#include "tsf_dids.cuh"

using namespace tsf;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(TSF_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));     \
  } while (0)

int ilog2_host(long x) {
  int r = 0;
  while ((1L << r) < x) ++r;
  return r;
}
bool is_pow2(long x) { return x > 0 && (x & (x - 1)) == 0; }


}  // namespace

namespace tsf {
int report_cuda(cudaError_t e, const char* what) {
  return fail(TSF_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}
int report_error(int code, const char* msg) { return fail(code, "%s", msg); }

bool graph_mode() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_SOLVE_GRAPH");
    v = (s && s[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// BiCGSTAB takes the even channel of each Toeplitz product from the Strang
// solve's stored spectrum (tsf_filters.cuh filt_strang_tab); TSF_SPEC_REUSE=0
// restores the recomputed forward transform (A/B measurement).
bool spec_reuse() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_SPEC_REUSE");
    v = (s && s[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Half-length transform engine of the Strang-preconditioned BiCGSTAB level
// solve (tsf_half.cuh); TSF_HALF=0 restores the full-length phase kernels.
bool half_mode() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_HALF");
    v = (s && s[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool fuse_vt() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_FUSE_VT");
    v = (s && s[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int persist_h_max_b() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_PERSIST_MAX_B");
    v = s ? atoi(s) : 0x7fffffff;   // every batch (0: the phase kernels in a graph)
  }
  return v;
}

int solve_groups(int B) {
  static int env = -2;
  if (env == -2) {
    const char* s = getenv("TSF_SOLVE_GROUPS");
    env = s ? atoi(s) : -1;
  }
  int g = env > 0 ? env : (B >= 1024 ? 4 : 1);
  if (g > kMaxSolveGroups) g = kMaxSolveGroups;
  if (g > B) g = B > 0 ? B : 1;
  // groups of ceil(B/g) instances: drop the empty trailing groups (B = 5,
  // g = 4 -> 2 per group -> 3 groups; B = 9, g = 4 -> 3 groups of 3)
  if (B > 0) {
    const int bg = (B + g - 1) / g;
    g = (B + bg - 1) / bg;
  }
  return g;
}

SolveGraphs::~SolveGraphs() {
  for (auto& a : slot)
    for (auto& b : a)
      for (auto& g : b) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
      }
}

// two-level twiddle table of W_N (tsf_fft.cuh tw_get): padded [W^j, j < 64]
// then padded [W^(64 i), i < max(1, N/64)], computed in long double
std::vector<double2> twiddle_table(int N) {
  const long double two_pi = 6.283185307179586476925286766559005768L;
  auto w = [&](long e) {
    long double a = two_pi * (long double)(e % N) / (long double)N;
    return make_double2((double)cosl(a), (double)-sinl(a));
  };
  std::vector<double2> t(tw_table_elems(N), make_double2(0.0, 0.0));
  for (int j = 0; j < 64; ++j) t[tw_lo_slot(j)] = w(j);
  for (int i = 0; i < tw_hi_count(N); ++i) t[kTwLo + tw_lo_slot(i)] = w(64L * i);
  return t;
}
// Explicit per-pass twiddles of the length-N transform (FftPlan<N, 8>
// ptw_off layout): pass p >= 1 of radix R = 2^lr(p) after NS = 8^p points
// holds W_{NS R}^{k m} at off(p) + (m-1) NS + k.
std::vector<double2> pass_twiddles(int N) {
  const long double two_pi = 6.283185307179586476925286766559005768L;
  int logn = 0;
  while ((1 << logn) < N) ++logn;
  const int npass = (logn + 2) / 3;
  std::vector<double2> t;
  for (int p = 1; p < npass; ++p) {
    const int lr = p < npass - 1 ? 3 : logn - 3 * (npass - 1);
    const long R = 1L << lr, NS = 1L << (3 * p);
    for (long m = 1; m < R; ++m)
      for (long k = 0; k < NS; ++k) {
        const long double a = two_pi * (long double)((k * m) % (NS * R)) / (long double)(NS * R);
        t.push_back(make_double2((double)cosl(a), (double)-sinl(a)));
      }
  }
  if (t.empty()) t.push_back(make_double2(1.0, 0.0));
  return t;
}
}  // namespace tsf

struct tsf_plan {
  int n = 0;
  int L = 0;
  int log_L = 0;
  int has_pc = 0;
  int device = 0;
  double2* tw = nullptr;   // W_L^e
  double2* mvS = nullptr;  // (S_{2k}, S_{2k+1}) / L, even part of the symbol
  double2* pclam = nullptr;  // (lam_k, lam_{n-k})
  double2* ptw = nullptr;    // per-pass twiddles of the length-L/2 transform
  int layout = 0;            // 1: 64 x 64 engine (permuted tables / workspaces)
  int vs = 0;                // per-instance stride of the workspace vectors
  // Krylov workspaces [cap][n] x 6
  int cap = 0;
  double* ws = nullptr;
  int* ist = nullptr;       // [0] = active-instance counter
  double* dst = nullptr;
  KState* kst = nullptr;    // per-instance Krylov scalars
  int* h_active = nullptr;  // pinned host mirror of the counter
  LargePlan* large = nullptr;  // n > 4096: four-step engine (tsf_large.cu)
  SolveGraphs* graphs = nullptr;  // graph-mode level solves (tsf_dispatch_impl.cuh)
  FilterTables tables() const {
    FilterTables t{tw, mvS, pclam};
    t.ptw = ptw;
    return t;
  }
};

// ------------------------------------------------------------- dispatch
namespace {

template <template <int> class F, int LOG = kMinLogL>
struct ForLog {
  template <typename... A>
  static int run(int log, A&&... args) {
    if (log == LOG) return F<LOG>::call(static_cast<A&&>(args)...);
    if constexpr (LOG < kMaxLogL) return ForLog<F, LOG + 1>::run(log, static_cast<A&&>(args)...);
    return fail(TSF_E_UNSUPPORTED, "transform size 2^%d not built", log);
  }
};

template <int LOG>
struct MatvecF {
  template <typename... A>
  static int call(A... a) { return Dispatch<LOG>::matvec(a...); }
};
template <int LOG>
struct PrecondF {
  template <typename... A>
  static int call(A... a) { return Dispatch<LOG>::precond(a...); }
};
template <int LOG>
struct LayoutF {
  static int call() { return Dispatch<LOG>::layout(); }
};
template <int LOG>
struct SolveF {
  template <typename... A>
  static int call(A... a) { return Dispatch<LOG>::solve(a...); }
};
template <int LOG>
struct FftF {
  template <typename... A>
  static int call(A... a) { return Dispatch<LOG>::fft(a...); }
};
template <int LOG>
struct HalfDebugF {
  template <typename... A>
  static int call(A... a) { return Dispatch<LOG>::half_debug(a...); }
};


constexpr int kWsVectors = 11;
int ensure_reserved(tsf_plan* p, int B) {
  if (p->large) {
    const int rc = large_reserve(p->large, B);
    if (rc == TSF_SUCCESS) p->cap = p->large->cap;
    return rc;
  }
  if (B <= p->cap) return TSF_SUCCESS;
  if (p->ws) cudaFree(p->ws);
  if (p->ist) cudaFree(p->ist);
  if (p->dst) cudaFree(p->dst);
  if (p->kst) cudaFree(p->kst);
  p->ws = nullptr;
  p->ist = nullptr;
  p->dst = nullptr;
  p->kst = nullptr;
  p->cap = 0;
  CK(cudaSetDevice(p->device));
  // 11 vectors [B][vs] (r p v ph s sh t kwork pspec r0w xw) + the Strang
  // spectra of the last preconditioner output (hspec): half spectra
  // [B][L/4+1] complex, full [B][L/2] complex for the 64 x 64 engine
  const size_t hs = p->layout ? (size_t)p->L : (size_t)(p->L / 2 + 2);
  CK(cudaMalloc(&p->ws, sizeof(double) * ((size_t)B * p->vs * kWsVectors + (size_t)B * hs)));
  CK(cudaMalloc(&p->ist, sizeof(int) * (size_t)B * 2));
  CK(cudaMalloc(&p->dst, sizeof(double) * (size_t)B));
  CK(cudaMalloc(&p->kst, sizeof(KState) * (size_t)B));
  if (!p->h_active) CK(cudaHostAlloc(&p->h_active, sizeof(int), cudaHostAllocDefault));
  p->cap = B;
  return TSF_SUCCESS;
}

}  // namespace

// Every plan entry point runs on the plan's device and restores the caller's
// current device on return (ctypes callers and Plan.__del__ may run with
// any device current).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ======================================================================
extern "C" {

int tsf_abi_version(void) { return TSF_ABI_VERSION; }

const char* tsf_last_error(void) { return g_err.c_str(); }

int tsf_plan_create(tsf_plan** out, int n, int L, const double* symbol_re, const double* lam,
                    int device) {
  if (!out) return fail(TSF_E_INVALID, "plan pointer is NULL");
  *out = nullptr;
  if (n < 1) return fail(TSF_E_INVALID, "n must be >= 1, got %d", n);
  if (!is_pow2(L) || L < 2 * n - 1 || L < 32)
    return fail(TSF_E_INVALID, "L=%d must be a power of two >= max(2n-1, 32)", L);
  if (!symbol_re) return fail(TSF_E_INVALID, "symbol is NULL");
  const int lg = ilog2_host(L);
  DeviceGuard dg(device);
  if (lg > kMaxLogL) {
    // four-step engine: transform length L/2 = 2^13..2^24, any n with 2n-1 <= L
    if (lam && !(is_pow2(n) && L == 2 * n))
      return fail(TSF_E_UNSUPPORTED,
                  "Strang tables need a power-of-two n with L = 2n (n=%d, L=%d)", n, L);
    tsf_plan* p = new tsf_plan();
    p->n = n;
    p->L = L;
    p->log_L = lg;
    p->device = device;
    p->has_pc = lam != nullptr;
    p->large = new LargePlan();
    const int rc = large_plan_init(p->large, n, L, symbol_re, lam, device);
    if (rc) {
      tsf_plan_destroy(p);
      return rc;
    }
    *out = p;
    return TSF_SUCCESS;
  }
  if (lg < kMinLogL)
    return fail(TSF_E_UNSUPPORTED, "embedding L=%d below 32", L);
  if (lam && !(is_pow2(n) && n >= 16 && L == 2 * n))
    return fail(TSF_E_UNSUPPORTED, "Strang preconditioner needs pow2 n >= 16 with L = 2n (n=%d, L=%d)", n, L);
  tsf_plan* p = new tsf_plan();
  p->n = n;
  p->L = L;
  p->log_L = lg;
  p->device = device;
  p->has_pc = lam != nullptr;
  auto cleanup = [&](int rc) {
    tsf_plan_destroy(p);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) return cleanup(fail(TSF_E_CUDA, "cudaSetDevice(%d)", device));
  p->layout = ForLog<LayoutF>::run(lg);
  p->vs = p->layout ? L / 2 : n;
  // twiddles W_L^e: modulation of the odd-bin half; the length-N transforms use stride 2
  std::vector<double2> tw = twiddle_table(L);
  // The reference keeps Re IFFT(S . FFT(pad x)) (toeplitz.py:62-63): its
  // effective symbol is the even part of S.  1/L of the inverse folded in;
  // stored as (S_{2k}, S_{2k+1}) for the even / odd output-bin halves.
  auto Ssym = [&](int k) -> double {
    return (double)(0.5L * ((long double)symbol_re[k] + (long double)symbol_re[(L - k) % L]) /
                    (long double)L);
  };
  std::vector<double2> S(L / 2);
  for (int k = 0; k < L / 2; ++k) S[k] = make_double2(Ssym(2 * k), Ssym(2 * k + 1));
  std::vector<double2> pl;
  if (lam) {
    pl.resize(n);
    for (int k = 0; k < n; ++k) pl[k] = make_double2(lam[k], lam[(n - k) % n]);
  }
  if (p->layout) {
    // 64 x 64 engine: bin oidx(t, c) stored at position spos(t, c)
    // (tsf_fft64.cuh), so a warp's table loads are contiguous
    const int N = L / 2, T = N / 8;
    auto permute = [&](std::vector<double2>& v) {
      if (v.empty()) return;
      std::vector<double2> w(v.size());
      for (int t = 0; t < T; ++t)
        for (int c = 0; c < 8; ++c) w[t + c * T] = v[oidx<4096>(t, c)];
      v.swap(w);
    };
    permute(S);
    permute(pl);
  }
  auto up = [&](auto** d, const auto& h) -> int {
    if (h.empty()) return TSF_SUCCESS;
    CK(cudaMalloc(d, h.size() * sizeof(h[0])));
    CK(cudaMemcpy(*d, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice));
    return TSF_SUCCESS;
  };
  int rc;
  std::vector<double2> ptw = pass_twiddles(L / 2);
  if ((rc = up(&p->tw, tw)) || (rc = up(&p->mvS, S)) || (rc = up(&p->pclam, pl)) ||
      (rc = up(&p->ptw, ptw)))
    return cleanup(rc);
  *out = p;
  return TSF_SUCCESS;
}

int tsf_plan_destroy(tsf_plan* p) {
  if (!p) return TSF_SUCCESS;
  DeviceGuard dg(p->device);
  if (p->large) {
    large_plan_free(p->large);
    delete p->large;
  }
  delete p->graphs;
  cudaFree(p->tw);
  cudaFree(p->mvS);
  cudaFree(p->pclam);
  cudaFree(p->ptw);
  cudaFree(p->ws);
  cudaFree(p->ist);
  cudaFree(p->dst);
  cudaFree(p->kst);
  if (p->h_active) cudaFreeHost(p->h_active);
  delete p;
  return TSF_SUCCESS;
}

int tsf_plan_info(const tsf_plan* p, int64_t* o) {
  if (!p || !o) return fail(TSF_E_INVALID, "NULL argument");
  o[0] = p->n;
  o[1] = p->L;
  o[2] = p->L / 16;
  o[3] = p->has_pc;
  o[4] = p->cap;
  return TSF_SUCCESS;
}

int tsf_plan_reserve(tsf_plan* p, int B) {
  if (!p || B < 1) return fail(TSF_E_INVALID, "bad plan or batch");
  DeviceGuard dg(p->device);
  return ensure_reserved(p, B);
}

int tsf_toeplitz_matvec(tsf_plan* p, int B, const double* x, double* y, const double* kappa,
                        double shift, void* stream) {
  if (!p || !x || !y || B < 0) return fail(TSF_E_INVALID, "bad argument");
  if (B == 0) return TSF_SUCCESS;
  DeviceGuard dg(p->device);
  if (p->large) return large_matvec(p->large, B, x, y, kappa, shift, (cudaStream_t)stream);
  return ForLog<MatvecF>::run(p->log_L, p->n, p->tables(), B, x, y, kappa, shift,
                              (cudaStream_t)stream);
}

int tsf_precond_solve(tsf_plan* p, int B, const double* v, double* z, double shift,
                      double kbar, const double* kbar_dev, void* stream) {
  if (!p || !v || !z || B < 0) return fail(TSF_E_INVALID, "bad argument");
  if (!p->has_pc) return fail(TSF_E_UNSUPPORTED, "plan has no Strang preconditioner (non-pow2 n)");
  if (B == 0) return TSF_SUCCESS;
  DeviceGuard dg(p->device);
  if (p->large)
    return large_precond(p->large, B, v, z, shift, kbar, kbar_dev, (cudaStream_t)stream);
  return ForLog<PrecondF>::run(p->log_L, p->n, p->tables(), B, v, z, shift, kbar, kbar_dev,
                               (cudaStream_t)stream);
}

static int solve_impl(tsf_plan* p, int B, int method, int pc, KrylovArgs& a, cudaStream_t st) {
  if (pc == 1 && !p->has_pc) return fail(TSF_E_UNSUPPORTED, "plan has no Strang preconditioner");
  if (pc == 2 && (p->large || p->layout))
    return fail(TSF_E_UNSUPPORTED, "circulant-column preconditioner needs the single-CTA "
                                   "Stockham engine (n <= 4096)");
  DeviceGuard dg(p->device);
  if (p->large) {
    if (a.soe_epilogue) return fail(TSF_E_UNSUPPORTED, "fused SOE epilogue needs n <= 4096");
    a.n = p->n;
    a.B = B;
    return large_solve(p->large, B, method, pc, a, st);
  }
  int rc = ensure_reserved(p, B);
  if (rc) return rc;
  const size_t vn = (size_t)p->cap * p->vs;
  a.n = p->n;
  a.B = B;
  a.vs = p->vs;
  a.r = p->ws;
  a.p = p->ws + vn;
  a.v = p->ws + 2 * vn;
  a.ph = p->ws + 3 * vn;
  a.s = p->ws + 4 * vn;
  a.sh = p->ws + 5 * vn;
  a.t = p->ws + 6 * vn;
  a.pspec = p->ws + 8 * vn;
  a.hspec = spec_reuse() ? reinterpret_cast<double2*>(p->ws + kWsVectors * vn) : nullptr;
  if (p->layout) {
    a.r0w = p->ws + 9 * vn;
    a.xw = p->ws + 10 * vn;
    a.kwork = p->ws + 7 * vn;   // internal layout (the caller's kwork has stride n)
  } else {
    a.r0w = a.rhs;
    a.xw = a.x;
  }
  a.kst = p->kst;
  a.active = p->ist;
  a.h_active = p->h_active;
  if (!a.kwork) a.kwork = p->ws + 7 * vn;
  a.tab = p->tables();
  if (a.max_iters <= 0) a.max_iters = 10 * p->n;
  if (!a.soe_epilogue) {
    // graph mode (the fused SOE epilogue keeps the host-driven loop)
    if (!p->graphs) p->graphs = new SolveGraphs();
    a.graphs = p->graphs;
  }
  return ForLog<SolveF>::run(p->log_L, B, method, pc, (const KrylovArgs&)a, st);
}

int tsf_krylov_solve(tsf_plan* p, int B, int method, int precond, const double* rhs, double* x,
                     const double* kappa, double shift, double kappa_bar, double tol, int max_iters, int* iters,
                     double* relres, int* status, void* stream) {
  if (!p || !rhs || !x || !kappa || !iters || !relres || !status || B < 0)
    return fail(TSF_E_INVALID, "bad argument");
  if (method != 0 && method != 1) return fail(TSF_E_INVALID, "method must be 0 or 1");
  if (B == 0) return TSF_SUCCESS;
  KrylovArgs a{};
  a.rhs = rhs;
  a.x = x;
  a.kappa = kappa;
  a.shift = shift;
  a.kbar = kappa_bar;
  a.tol = tol;
  a.max_iters = max_iters;
  a.iters = iters;
  a.relres = relres;
  a.status = status;
  return solve_impl(p, B, method, precond, a, (cudaStream_t)stream);
}

int tsf_krylov_solve_circ(tsf_plan* p, int B, int method, const double* rhs, double* x,
                          const double* kappa, double shift, const double* pc_spec,
                          int64_t pc_stride, double tol, int max_iters, int* iters,
                          double* relres, int* status, void* stream) {
  if (!p || !rhs || !x || !kappa || !pc_spec || !iters || !relres || !status || B < 0)
    return fail(TSF_E_INVALID, "bad argument");
  if (method != 0 && method != 1) return fail(TSF_E_INVALID, "method must be 0 or 1");
  if (pc_stride != 0 && pc_stride < p->L / 2)
    return fail(TSF_E_INVALID, "pc_stride must be 0 or >= L/2");
  if (B == 0) return TSF_SUCCESS;
  KrylovArgs a{};
  a.rhs = rhs;
  a.x = x;
  a.kappa = kappa;
  a.shift = shift;
  a.kbar = 1.0;   // unused by the circulant-column preconditioner
  a.tol = tol;
  a.max_iters = max_iters;
  a.iters = iters;
  a.relres = relres;
  a.status = status;
  a.pcS = reinterpret_cast<const double2*>(pc_spec);
  a.pcS_stride = (long)pc_stride;
  return solve_impl(p, B, method, 2, a, (cudaStream_t)stream);
}

static int soe_launch(int B, SoeArgs& s, cudaStream_t st) {
  if (B == 0) return TSF_SUCCESS;
  const int chunks = (s.n + 2 * kSoeThreads - 1) / (2 * kSoeThreads);
  const int smem = 3 * s.nexp * (int)sizeof(double);
  if (smem > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_soe_push_rhs<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  k_soe_push_rhs<8><<<(unsigned)B * chunks, kSoeThreads, smem, st>>>(s);
  CK(cudaGetLastError());
  return TSF_SUCCESS;
}

int tsf_l1_history_rhs(int B, int n, int rows, const double* hist, int64_t inst_stride,
                       const double* w, double c0, double G, const double* f, double* rhs,
                       void* stream) {
  if (B < 0 || n < 1 || rows < 1) return fail(TSF_E_INVALID, "bad argument");
  if (!hist || !f || !rhs || (rows > 1 && !w)) return fail(TSF_E_INVALID, "NULL pointer");
  if (inst_stride < (int64_t)rows * n && B > 1)
    return fail(TSF_E_INVALID, "instance stride smaller than rows*n");
  if (!(G > 0.0)) return fail(TSF_E_INVALID, "G must be > 0");
  if (B == 0) return TSF_SUCCESS;
  const dim3 grid((unsigned)((n + kDidsCols - 1) / kDidsCols), (unsigned)B);
  k_l1_history_rhs<<<grid, dim3(kDidsCols, kDidsGroups), 0, (cudaStream_t)stream>>>(
      n, rows, hist, (long)inst_stride, w, c0, G, f, rhs);
  CK(cudaGetLastError());
  return TSF_SUCCESS;
}

int tsf_soe_push_rhs(int B, int n, int nexp, double* W, const double* u,
                     const double* uprev, double tau_push, const double* decay,
                     const double* coef, const double* hcoef, int do_push, int w_zero,
                     int do_rhs, double a_next, double G, const double* f, double* rhs,
                     void* stream) {
  if (B < 0 || n < 1 || nexp < 1) return fail(TSF_E_INVALID, "bad argument");
  if (do_push && (!uprev || !u || !decay || !coef || !(tau_push > 0.0)))
    return fail(TSF_E_INVALID, "push needs u, uprev, decay, coef and tau_push > 0");
  if (!w_zero && !W) return fail(TSF_E_INVALID, "W is NULL");
  if (do_rhs && (!u || !hcoef || !rhs)) return fail(TSF_E_INVALID, "rhs needs u, hcoef, rhs");
  SoeArgs s{};
  s.n = n;
  s.nexp = nexp;
  s.W = W;
  s.u = u;
  s.uprev = uprev;
  s.tau_push = tau_push;
  s.decay = decay;
  s.coef = coef;
  s.hcoef = hcoef;
  s.do_push = do_push;
  s.w_zero = w_zero;
  s.do_rhs = do_rhs;
  s.a_next = a_next;
  s.G = G;
  s.nf = 0;
  s.f = f;
  s.rhs = rhs;
  return soe_launch(B, s, (cudaStream_t)stream);
}

int tsf_fids_march(tsf_plan* p, const tsf_march* d, void* stream) {
  if (!p || !d) return fail(TSF_E_INVALID, "NULL argument");
  DeviceGuard dg(p->device);
  const int B = d->B, M = d->M, nexp = d->nexp, n = p->n;
  if (B < 1 || M < 1 || nexp < 1) return fail(TSF_E_INVALID, "bad B/M/nexp");
  if (d->m_begin < 1 || d->m_end < d->m_begin || d->m_end > M + 1)
    return fail(TSF_E_INVALID, "bad level range [%d, %d)", d->m_begin, d->m_end);
  if (d->kappa.nmodes < 1 || d->kappa.nmodes > kMaxModes || d->source.nmodes < 0 ||
      d->source.nmodes > 4)
    return fail(TSF_E_INVALID, "kappa needs 1..4 modes, source 0..4");
  if (!d->u_buf0 || !d->u_buf1 || !d->W || !d->rhs || !d->soe_tab || !d->iters ||
      !d->relres || !d->status || !d->shift || !d->a_mm || !d->tau)
    return fail(TSF_E_INVALID, "NULL buffer in march descriptor");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_reserved(p, B);
  if (rc) return rc;
  double* ubuf[2] = {d->u_buf0, d->u_buf1};
  const size_t vn = (size_t)B * n;
  auto rec = [&](int m, int k) -> int {
    if (d->events) CK(cudaEventRecord((cudaEvent_t)d->events[3 * (m - d->m_begin) + k], st));
    return TSF_SUCCESS;
  };
  // per-level SOE/RHS arguments: push of level `pm` (pm = 0: none) + history
  // term and RHS of level `rm` (rm > M: none)
  auto soe_args = [&](int pm, int rm) {
    SoeArgs s{};
    s.n = n;
    s.nexp = nexp;
    s.W = d->W;
    s.u = ubuf[(rm - 1) & 1];  // u^{rm-1} == u^{pm}
    s.uprev = ubuf[rm & 1];    // u^{rm-2}
    s.do_push = pm >= 1;
    s.w_zero = (rm == 1) || (pm == 1);  // W^{0} = 0
    if (pm >= 1) {
      const double* tab = d->soe_tab + (size_t)(pm - 1) * 3 * nexp;
      s.tau_push = d->tau[pm - 1];
      s.decay = tab;
      s.coef = tab + nexp;
    }
    s.do_rhs = rm <= M;
    if (s.do_rhs) {
      s.hcoef = d->soe_tab + (size_t)(rm - 1) * 3 * nexp + 2 * nexp;
      s.a_next = d->a_mm[rm - 1];
      s.nf = d->source.nmodes;
      s.fmodes = d->source.modes ? d->source.modes + (size_t)rm * d->source.t_stride : nullptr;
      s.fq_stride = d->source.q_stride;
      s.fb_stride = d->source.b_stride;
      for (int q = 0; q < s.nf; ++q) s.fcoef[q] = d->source.coef[(size_t)rm * s.nf + q];
    }
    s.G = d->G;
    s.f = nullptr;
    s.rhs = d->rhs;
    return s;
  };
  // TSF_FUSE_SOE=1: each converged instance's CTA streams its own W rows at
  // the end of its solve (push of level m + RHS of level m+1).  Measured
  // slower on configs[2] (the 512-thread solve CTA holds the whole register
  // file, so the streaming cannot overlap transform work on that SM), hence
  // off by default: one SOE kernel per level.
  const char* fz = getenv("TSF_FUSE_SOE");
  const int K = d->soe_block;
  const bool blocked = K > 1;
  if (blocked && (K > kSoeMaxBlock || !d->soe_alpha || !d->soe_beta || !d->soe_ring))
    return fail(TSF_E_INVALID, "blocked SOE needs soe_block <= %d, soe_alpha, soe_beta, soe_ring",
                kSoeMaxBlock);
  const bool fuse = fz && fz[0] == '1' && !p->large && !blocked;
  double* du_ring = blocked ? d->soe_ring : nullptr;
  double* g_ring = blocked ? d->soe_ring + (size_t)K * vn : nullptr;
  // block pass at base mb: W^{mb-ka} -> W^{mb} (ka pushes), history terms of
  // levels mb+1 .. mb+kn, RHS of level mb+1
  auto block_pass = [&](int mb, int ka, int kn) -> int {
    SoeBlockArgs b{};
    b.n = n;
    b.nexp = nexp;
    b.B = B;
    b.W = d->W;
    b.u_cur = ubuf[mb & 1];
    b.u_prev = ubuf[(mb + 1) & 1];
    b.tau_cur = mb >= 1 ? d->tau[mb - 1] : 0.0;
    b.du_ring = du_ring;
    b.K = K;
    b.mb = mb;
    b.ka = ka;
    b.w_zero = (mb - ka) == 0;
    b.push_tab = d->soe_tab;
    b.kn = kn;
    b.alpha = d->soe_alpha;
    b.g_ring = g_ring;
    if (kn >= 1) {
      const int rm = mb + 1;
      b.a_next = d->a_mm[rm - 1];
      b.nf = d->source.nmodes;
      b.fmodes = d->source.modes ? d->source.modes + (size_t)rm * d->source.t_stride : nullptr;
      b.fq_stride = d->source.q_stride;
      b.fb_stride = d->source.b_stride;
      for (int q = 0; q < b.nf; ++q) b.fcoef[q] = d->source.coef[(size_t)rm * b.nf + q];
    }
    b.G = d->G;
    b.rhs = d->rhs;
    const int chunks = (n + 2 * kSoeThreads - 1) / (2 * kSoeThreads);
    const int smem = (2 * ka + kn) * nexp * (int)sizeof(double);
    // register arrays sized by the block length (K <= 8: ~90 registers, 5 CTAs/SM)
    auto go = [&](auto kern) -> int {
      if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kern<<<(unsigned)B * chunks, kSoeThreads, smem, st>>>(b);
      CK(cudaGetLastError());
      return TSF_SUCCESS;
    };
    if (ka == K && kn == K && (n & 1) == 0 && (K == 4 || K == 8 || K == 16)) {
      const int fsm = ((K + K / 2) * nexp + kSoeRing * kSoeThreads) * (int)sizeof(double2);
      auto gof = [&](auto kern) -> int {
        if (fsm > 48 * 1024)
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm));
        kern<<<(unsigned)B * chunks, kSoeThreads, fsm, st>>>(b);
        CK(cudaGetLastError());
        return TSF_SUCCESS;
      };
      const bool wz = b.w_zero != 0;
      if (K == 4) return wz ? gof(k_soe_block_full<4, true>) : gof(k_soe_block_full<4, false>);
      if (K == 8) {
        static const int pd = getenv("TSF_SOE_PD") ? atoi(getenv("TSF_SOE_PD")) : 0;
        if (!wz && pd == 0) return gof(k_soe_block_full<8, false, 0>);
        return wz ? gof(k_soe_block_full<8, true>) : gof(k_soe_block_full<8, false>);
      }
      return wz ? gof(k_soe_block_full<16, true>) : gof(k_soe_block_full<16, false>);
    }
    if (K <= 4) return go(k_soe_block<4>);
    if (K <= 8) return go(k_soe_block<8>);
    return go(k_soe_block<kSoeMaxBlock>);
  };
  auto level_rhs = [&](int m, int mb) -> int {
    SoeLevelArgs l{};
    l.n = n;
    l.B = B;
    l.K = K;
    l.m = m;
    l.mb = mb;
    l.u1 = ubuf[(m - 1) & 1];
    l.u2 = ubuf[m & 1];
    l.tau1 = d->tau[m - 2];
    l.du_ring = du_ring;
    l.g_ring = g_ring;
    for (int q = 0; q < m - 1 - mb; ++q) l.beta[q] = d->soe_beta[(size_t)(m - 1) * 16 + q];
    l.a_m = d->a_mm[m - 1];
    l.G = d->G;
    l.nf = d->source.nmodes;
    l.fmodes = d->source.modes ? d->source.modes + (size_t)m * d->source.t_stride : nullptr;
    l.fq_stride = d->source.q_stride;
    l.fb_stride = d->source.b_stride;
    for (int q = 0; q < l.nf; ++q) l.fcoef[q] = d->source.coef[(size_t)m * l.nf + q];
    l.rhs = d->rhs;
    const dim3 grid((unsigned)((n + 511) / 512), (unsigned)B);
    k_soe_level<<<grid, 256, 0, st>>>(l);
    CK(cudaGetLastError());
    return TSF_SUCCESS;
  };
  for (int m = d->m_begin; m < d->m_end; ++m) {
    if ((rc = rec(m, 0))) return rc;
    if (blocked) {
      const int mb = ((m - 1) / K) * K;
      if (m - 1 == mb) {
        if ((rc = block_pass(mb, mb == 0 ? 0 : K, std::min(K, M - mb)))) return rc;
      } else if ((rc = level_rhs(m, mb))) {
        return rc;
      }
    } else if (m == 1 || !fuse) {
      // push of level m-1 (fused with the history term) + RHS of level m
      SoeArgs s = soe_args(m - 1, m);
      if ((rc = soe_launch(B, s, st))) return rc;
    }
    if ((rc = rec(m, 1))) return rc;
    // ---- level solve -> u^m into ubuf[m & 1]; each converged instance then
    // streams its own W rows: push of level m, history term + RHS of level m+1
    KrylovArgs a{};
    a.rhs = d->rhs;
    a.x = ubuf[m & 1];
    a.kappa = nullptr;
    a.kmodes = d->kappa.modes + (size_t)m * d->kappa.t_stride;
    a.kq_stride = d->kappa.q_stride;
    a.kb_stride = d->kappa.b_stride;
    a.nk = d->kappa.nmodes;
    for (int q = 0; q < a.nk; ++q) a.kcoef[q] = d->kappa.coef[(size_t)m * a.nk + q];
    a.kwork = d->kwork;
    a.shift = d->shift[m - 1];
    a.tol = d->tol;
    a.max_iters = d->max_iters;
    a.iters = d->iters + (size_t)(m - 1) * B;
    a.relres = d->relres + (size_t)(m - 1) * B;
    a.status = d->status + (size_t)(m - 1) * B;
    a.soe = soe_args(m, m + 1);
    a.soe_epilogue = fuse ? 1 : 0;
    if ((rc = solve_impl(p, B, d->method, d->precond, a, st))) return rc;
    if ((rc = rec(m, 2))) return rc;
    if (d->hist && d->hist_B > 0) {
      CK(cudaMemcpyAsync(d->hist + (size_t)m * d->hist_B * n, ubuf[m & 1],
                         sizeof(double) * (size_t)d->hist_B * n, cudaMemcpyDeviceToDevice, st));
    }
  }
  if (!fuse && d->m_end == M + 1 && d->m_begin <= M) {
    // final push of level M (scheme.py:290 runs after every level)
    if (blocked) {
      const int mbl = ((M - 1) / K) * K;   // base of level M's block
      if ((rc = block_pass(M, M - mbl, 0))) return rc;
    } else {
      SoeArgs s = soe_args(M, M + 1);
      if ((rc = soe_launch(B, s, st))) return rc;
    }
  }
  (void)vn;
  return TSF_SUCCESS;
}

int tsf_fft_debug(int N, int inverse, int B, const double* in, double* out, void* stream) {
  if (!is_pow2(N) || N < 16 || N > 4096 || B < 1 || !in || !out)
    return fail(TSF_E_INVALID, "bad FFT debug arguments");
  const int lg = ilog2_host(N) + 1;  // Dispatch<LOG> transforms N = 2^(LOG-1)
  static double2* dtw[kMaxLogL + 2] = {};
  if (!dtw[lg]) {
    std::vector<double2> t = twiddle_table(N);
    CK(cudaMalloc(&dtw[lg], t.size() * sizeof(double2)));
    CK(cudaMemcpy(dtw[lg], t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice));
  }
  return ForLog<FftF>::run(lg, inverse, B, (const double2*)in, (double2*)out,
                           (const double2*)dtw[lg], (cudaStream_t)stream);
}

int tsf_half_debug(tsf_plan* p, int mode, int B, const double* x, const double* aux, double shift,
                   double* hs, double* out, void* stream) {
  if (!p || !x || !aux || !hs || !out || B < 1 || (mode != 0 && mode != 1))
    return fail(TSF_E_INVALID, "bad half-engine debug arguments");
  if (p->large || p->layout || !p->has_pc || p->n * 2 != p->L)
    return fail(TSF_E_UNSUPPORTED, "half-length engine needs a power-of-two n <= 4096");
  DeviceGuard dg(p->device);
  const int rc = ForLog<HalfDebugF>::run(p->log_L, mode, B, x, aux, shift, (double2*)hs, out,
                                         p->tables(), (cudaStream_t)stream);
  if (rc == -1) return fail(TSF_E_UNSUPPORTED, "half-length engine not built for this size");
  return rc;
}

}  // extern "C"
