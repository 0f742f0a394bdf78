// Per-size dispatch of the single-CTA engine.  The bodies live in
// tsf_dispatch_impl.cuh and are explicitly instantiated one size per
// translation unit (gen/inst_L*.cu) so the build parallelises.
#pragma once

#include "tsf_kernels.cuh"

namespace tsf {

constexpr int kMinLogL = 5;   // L = 32
constexpr int kMaxLogL = 13;  // L = 8192 (n <= 4096 single-CTA engine)

// sets tsf_last_error() and returns TSF_E_CUDA (defined in tsf_abi.cu)
int report_cuda(cudaError_t e, const char* what);

// Instantiated level-solve graphs of one plan (graph mode): one slot per
// (transform size, preconditioner, method).  Built on first use; later
// solves only rewrite the kernel-node parameters and relaunch.
// A level-solve graph: `groups` independent branches (contiguous instance
// groups), each  set -> begin -> WHILE(active_g > 0) { a ; b ; test }.
constexpr int kMaxSolveGroups = 8;
struct SolveGraph {
  bool built = false;
  bool half = false;   // built from the half-length kernels (tsf_half.cuh)
  int groups = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond[kMaxSolveGroups]{};
  cudaGraphNode_t n_set[kMaxSolveGroups]{}, n_begin[kMaxSolveGroups]{}, n_a[kMaxSolveGroups]{},
      n_b[kMaxSolveGroups]{}, n_c[kMaxSolveGroups]{};
};
int solve_groups(int B);  // TSF_SOLVE_GROUPS (default: 4 for B >= 1024, else 1)
struct SolveGraphs {
  SolveGraph slot[kMaxLogL + 1][3][2];  // [log L][pc: none / Strang / circulant column][cg]
  ~SolveGraphs();
};
bool graph_mode();  // TSF_SOLVE_GRAPH (default 1)
bool spec_reuse();  // TSF_SPEC_REUSE (default 1)
bool fuse_vt();     // TSF_FUSE_VT (default 0): both BiCGSTAB phases of an iteration in one kernel
int persist_h_max_b();   // TSF_PERSIST_MAX_B (default: no limit): largest batch the half-length
                         // engine solves with one persistent kernel per instance (0: phase kernels)
bool half_mode();   // TSF_HALF (default 1): half-length transform engine, tsf_half.cuh

template <int LOG>
struct Dispatch {
  static int matvec(int n, const FilterTables& t, int B, const double* x, double* y,
                    const double* kappa, double shift, cudaStream_t st);
  static int precond(int n, const FilterTables& t, int B, const double* v, double* z,
                     double shift, double kbar, const double* kbar_dev, cudaStream_t st);
  static int solve(int B, int method, int pc, const KrylovArgs& a, cudaStream_t st);
  static int fft(int inverse, int B, const double2* in, double2* out, const double2* tw,
                 cudaStream_t st);
  // 1: the 64 x 64 engine (tsf_fft64.cuh) — plan tables and workspace
  // vectors in the permuted internal layout, per-instance stride N
  static int layout();
  // building blocks of the half-length engine alone (tests): -1 = not built for this size
  static int half_debug(int mode, int B, const double* x, const double* aux_in, double shift,
                        double2* hs, double* out, const FilterTables& t, cudaStream_t st);
};

#define TSF_EXTERN_DISPATCH(L) extern template struct Dispatch<L>;
TSF_EXTERN_DISPATCH(5)
TSF_EXTERN_DISPATCH(6)
TSF_EXTERN_DISPATCH(7)
TSF_EXTERN_DISPATCH(8)
TSF_EXTERN_DISPATCH(9)
TSF_EXTERN_DISPATCH(10)
TSF_EXTERN_DISPATCH(11)
TSF_EXTERN_DISPATCH(12)
TSF_EXTERN_DISPATCH(13)

}  // namespace tsf
