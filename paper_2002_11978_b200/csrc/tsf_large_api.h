// Host interface of the large-n engine (tsf_large.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "tsf_large.cuh"

namespace tsf {

// shared with tsf_abi.cu: sets tsf_last_error() and returns `code`
int report_error(int code, const char* msg);
// two-level twiddle table of W_N (layout: tsf_fft.cuh tw_get)
std::vector<double2> twiddle_table(int N);

// Graph-mode iteration loop of one (method, preconditioner): a conditional
// WHILE node whose body is one captured Krylov iteration (the launch chain of
// Runner::bicg_iteration / cg_iteration) plus the loop test.  Later solves
// re-capture the chain into a scratch graph and copy its kernel parameters
// into the instantiated body node by node (the chain's shape never changes).
struct LargeLoopGraph {
  bool built = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond{};
  std::vector<cudaGraphNode_t> body;   // body kernel nodes in chain order
};

struct LargePlan {
  int n = 0, nt = 0, N1 = 0, N2 = 0, np = 0;   // vector length n <= transform length nt
  int ncol_cta = 0;            // column CTAs per instance (partial-sum count)
  int has_pc = 0;
  int device = 0;
  double lam_min = 0.0;       // min_k lam_k (preconditioner positivity test)
  LargeTables lt{};
  double2* tables = nullptr;  // one allocation for every table
  // workspaces, sized for `cap` instances
  int cap = 0;
  double* ws = nullptr;       // 8 vectors [cap][n] + Strang spectrum [cap][nt]
  double2* Z = nullptr;       // [2][cap][n] (two transform channels)
  double* part = nullptr;     // [cap][4][np]
  LState* st = nullptr;       // [cap]
  int* active = nullptr;
  int* h_active = nullptr;
  cudaStream_t cap_stream = nullptr;   // graph capture (non-blocking)
  LargeLoopGraph loops[2][2][4];       // [method][pc][few-CTA column kernels + 2 * half-length engine]
  // half-length engine (tsf_hlarge.cuh): power-of-two n >= 2^14 with Strang tables
  int half = 0;
  int ncol_cta_h = 0;
  HalfGeom hg{};
};

// embedding L a power of two in [2^14, 2^25] with 2n-1 <= L (vectors of length n are
// zero-padded to the transform length L/2); symbol_re: L reals; lam: n reals (n = L/2) or null
int large_plan_init(LargePlan* lp, int n, int L, const double* symbol_re, const double* lam,
                    int device);
void large_plan_free(LargePlan* lp);
int large_reserve(LargePlan* lp, int B);

int large_matvec(LargePlan* lp, int B, const double* x, double* y, const double* kappa,
                 double shift, cudaStream_t st);
int large_precond(LargePlan* lp, int B, const double* v, double* z, double shift, double kbar,
                  const double* kbar_dev, cudaStream_t st);
// Level solve: kappa given [B][n] (kappa != null) or separable modes (KrylovArgs fields);
// method 0 = BiCGSTAB (CG: TSF_E_UNSUPPORTED for now)
int large_solve(LargePlan* lp, int B, int method, int pc, const KrylovArgs& a, cudaStream_t st);

}  // namespace tsf
