// Kernel launch bodies of Dispatch<LOG> (see tsf_dispatch.h); LOG = log2(L),
// the per-instance transform length is N = L/2.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "tsf_dispatch.h"
#include "tsf_half.cuh"

namespace tsf {

inline int launch_error(cudaError_t e) {
  return e == cudaSuccess ? 0 : report_cuda(e, "kernel launch");
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename K>
inline cudaError_t prep_kernel(K kernel, int smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

template <int LOG>
int Dispatch<LOG>::matvec(int n, const FilterTables& t, int B, const double* x, double* y,
                          const double* kappa, double shift, cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  using S = KShape<N>;
  if constexpr (half_ok<N>()) {
    if (half_mode() && n == N && aligned16(x) && aligned16(y) && (!kappa || aligned16(kappa))) {
      auto kh = k_toeplitz_apply_h<N>;
      cudaError_t eh = prep_kernel(kh, HShape<N>::SMEM);
      if (eh != cudaSuccess) return launch_error(eh);
      kh<<<B, HShape<N>::BLOCK, HShape<N>::SMEM, st>>>(x, y, kappa, shift, t);
      return launch_error(cudaGetLastError());
    }
  }
  auto k = k_toeplitz_apply<N>;
  cudaError_t e = prep_kernel(k, S::SMEM);
  if (e != cudaSuccess) return launch_error(e);
  k<<<B, S::BLOCK, S::SMEM, st>>>(n, x, y, kappa, shift, t);
  return launch_error(cudaGetLastError());
}

template <int LOG>
int Dispatch<LOG>::precond(int n, const FilterTables& t, int B, const double* v, double* z,
                           double shift, double kbar, const double* kbar_dev, cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  using S = KShape<N>;
  if constexpr (half_ok<N>()) {
    if (half_mode() && n == N && aligned16(v) && aligned16(z)) {
      auto kh = k_strang_apply_h<N>;
      cudaError_t eh = prep_kernel(kh, HShape<N>::SMEM);
      if (eh != cudaSuccess) return launch_error(eh);
      kh<<<B, HShape<N>::BLOCK, HShape<N>::SMEM, st>>>(v, z, shift, kbar, kbar_dev, t);
      return launch_error(cudaGetLastError());
    }
  }
  auto k = k_strang_apply<N>;
  cudaError_t e = prep_kernel(k, S::SMEM);
  if (e != cudaSuccess) return launch_error(e);
  k<<<B, S::BLOCK, S::SMEM, st>>>(n, v, z, shift, kbar, kbar_dev, t);
  return launch_error(cudaGetLastError());
}

// Host driver of one level solve for B instances: begin kernel, then the
// iteration kernels in chunks of kChunk iterations; after each chunk the
// device count of unfinished instances is read back (one small D2H copy and
// a stream sync per chunk).  Finished instances' CTAs return immediately, so
// the overshoot costs at most kChunk-1 near-empty launch pairs.
// TSF_SOLVE_PERSIST=1 selects the persistent per-instance kernel (one launch
// per level solve) instead of the host-driven phase kernels.
inline bool persist_mode() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_SOLVE_PERSIST");
    v = (s && s[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Graph mode: the whole level solve is ONE graph launch —
//   set(active = B) -> begin -> WHILE(active > 0) { v-phase ; t-phase ; test }
// (PCG: one iteration kernel in the body).  No host round trip, no chunk
// overshoot; the graph is instantiated once per plan and size/method, and
// later solves rewrite the kernel-node parameters in place
// (cudaGraphExecKernelNodeSetParams, body nodes included).
template <typename K>
cudaKernelNodeParams knode(K kernel, dim3 grid, dim3 block, int smem, void** args) {
  cudaKernelNodeParams p{};
  p.func = reinterpret_cast<void*>(kernel);
  p.gridDim = grid;
  p.blockDim = block;
  p.sharedMemBytes = smem;
  p.kernelParams = args;
  return p;
}

// Instance group [o, o + Bg) of a level solve: every per-instance pointer
// offset, its own active counter (a.active + g).
inline KrylovArgs group_args(const KrylovArgs& a, int N, bool full_spec, int o, int Bg, int g) {
  KrylovArgs r = a;
  const long vo = (long)o * a.n;    // caller vectors
  const long wo = (long)o * a.vs;   // workspace vectors
  r.B = Bg;
  r.rhs = a.rhs + vo;
  r.x = a.x + vo;
  r.r0w = a.r0w == a.rhs ? r.rhs : a.r0w + wo;
  r.xw = a.xw == a.x ? r.x : a.xw + wo;
  if (a.kappa) r.kappa = a.kappa + vo;
  if (a.kmodes) r.kmodes = a.kmodes + (long)o * a.kb_stride;
  if (a.kwork) r.kwork = a.kwork + wo;
  r.r = a.r + wo;
  r.p = a.p + wo;
  r.v = a.v + wo;
  r.ph = a.ph + wo;
  r.s = a.s + wo;
  r.sh = a.sh + wo;
  r.t = a.t + wo;
  if (a.pspec) r.pspec = a.pspec + wo;
  if (a.hspec) r.hspec = a.hspec + (long)o * (full_spec ? N : N / 2 + 1);
  r.kst = a.kst + o;
  r.active = a.active + g;
  r.iters = a.iters + o;
  r.relres = a.relres + o;
  r.status = a.status + o;
  return r;
}

// Half-length transform engine (tsf_half.cuh): Strang-preconditioned BiCGSTAB
// with the spectrum reuse on a power-of-two grid, 16-byte aligned vectors.
template <int N, int PC, bool CG>
bool use_half(const KrylovArgs& a) {
  if constexpr (PC == 1 && !CG && half_ok<N>()) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return half_mode() && a.hspec && !a.soe_epilogue && a.n == N && a.vs == N && al(a.rhs) &&
           al(a.x) &&
           (a.kappa ? al(a.kappa)
                    : (al(a.kmodes) && al(a.kwork) && a.kq_stride % 2 == 0 && a.kb_stride % 2 == 0));
  } else {
    return false;
  }
}
using SolveKernel = void (*)(KrylovArgs, KState*, int*);
template <int N, int PC, bool CG>
struct SolveKernels {
  SolveKernel kb, kv, kt, kc;
  int block, smem;
  bool one = CG;   // one kernel per iteration (PCG, or the fused BiCGSTAB phases)
  explicit SolveKernels(bool half) {
    kb = k_solve_begin<N, PC, CG>;
    kv = k_bicg_v<N, PC>;
    kt = k_bicg_t<N, PC>;
    kc = k_cg_iter<N, PC>;
    block = KShape<N>::BLOCK;
    smem = KShape<N>::SMEM;
    if constexpr (PC == 1 && !CG && half_ok<N>()) {
      if (half) {
        kb = k_solve_begin_h<N>;
        kv = fuse_vt() ? k_bicg_h<N, 3> : k_bicg_h<N, 1>;
        kt = k_bicg_h<N, 2>;
        one = fuse_vt();
        block = HShape<N>::BLOCK;
        smem = HShape<N>::SMEM;
      }
    }
  }
};

// The level solve as one graph launch of G independent branches over
// contiguous instance groups.  With one branch, the level's tail (a few
// slow instances, ~30-40 us per phase launch) leaves the GPU nearly idle;
// with G branches the other groups' full launches fill it (measured on
// configs[2] with G separate marches on G streams: 3.7% faster at G = 4,
// tools/group_probe.py).  Each group's instances are computed exactly as
// with one branch (per-instance CTAs), so results do not depend on G.
template <int N, int PC, bool CG>
int solve_graph(int B, const KrylovArgs& a_in, cudaStream_t st) {
  constexpr int LOG = ilog2(2 * N);
  SolveGraphs* cache = static_cast<SolveGraphs*>(a_in.graphs);
  SolveGraph& G = cache->slot[LOG][PC][CG ? 1 : 0];
  const int ng = solve_groups(B);
  const int bg = (B + ng - 1) / ng;
  const bool half = use_half<N, PC, CG>(a_in);
  const SolveKernels<N, PC, CG> K(half);
  cudaError_t e;
  if (G.built && (G.groups != ng || G.half != half)) {
    cudaGraphExecDestroy(G.exec);
    cudaGraphDestroy(G.graph);
    G = SolveGraph{};
  }
  const SolveKernel kb = K.kb, kv = K.kv, kt = K.kt, kc = K.kc;
  if (!G.built) {
    if ((e = prep_kernel(kb, K.smem)) != cudaSuccess) return launch_error(e);
    if ((e = prep_kernel(CG ? kc : kv, K.smem)) != cudaSuccess) return launch_error(e);
    if (!K.one && (e = prep_kernel(kt, K.smem)) != cudaSuccess) return launch_error(e);
    if ((e = cudaGraphCreate(&G.graph, 0)) != cudaSuccess) return launch_error(e);
    G.groups = ng;
    G.half = half;
  }
  for (int g = 0; g < ng; ++g) {
    const int o = g * bg;
    const int Bg = std::min(bg, B - o);
    KrylovArgs a = group_args(a_in, N, use64<N>(), o, Bg, g);
    KState* kst = a.kst;
    int* active = a.active;
    int bval = Bg;
    void* set_args[] = {&active, &bval};
    void* k_args[] = {&a, &kst, &active};
    const cudaKernelNodeParams p_set = knode(k_set_int, dim3(1), dim3(1), 0, set_args);
    const cudaKernelNodeParams p_begin = knode(kb, dim3(Bg), dim3(K.block), K.smem, k_args);
    const cudaKernelNodeParams p_a = CG ? knode(kc, dim3(Bg), dim3(K.block), K.smem, k_args)
                                        : knode(kv, dim3(Bg), dim3(K.block), K.smem, k_args);
    const cudaKernelNodeParams p_b = knode(kt, dim3(Bg), dim3(K.block), K.smem, k_args);
    // the loop test reads the group's active counter, which moves when the
    // plan's workspaces grow (ensure_reserved): its node is rewritten too
    cudaGraphConditionalHandle h = G.cond[g];
    void* c_args[] = {&h, &active};
    if (!G.built) {
      if ((e = cudaGraphConditionalHandleCreate(&G.cond[g], G.graph, 1,
                                                cudaGraphCondAssignDefault)) != cudaSuccess)
        return launch_error(e);
      if ((e = cudaGraphAddKernelNode(&G.n_set[g], G.graph, nullptr, 0, &p_set)) != cudaSuccess)
        return launch_error(e);
      if ((e = cudaGraphAddKernelNode(&G.n_begin[g], G.graph, &G.n_set[g], 1, &p_begin)) !=
          cudaSuccess)
        return launch_error(e);
      cudaGraphNodeParams cp{};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = G.cond[g];
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t n_loop;
      if ((e = cudaGraphAddNode(&n_loop, G.graph, &G.n_begin[g], 1, &cp)) != cudaSuccess)
        return launch_error(e);
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      if ((e = cudaGraphAddKernelNode(&G.n_a[g], body, nullptr, 0, &p_a)) != cudaSuccess)
        return launch_error(e);
      cudaGraphNode_t last = G.n_a[g];
      if (!K.one) {
        if ((e = cudaGraphAddKernelNode(&G.n_b[g], body, &G.n_a[g], 1, &p_b)) != cudaSuccess)
          return launch_error(e);
        last = G.n_b[g];
      }
      h = G.cond[g];
      const cudaKernelNodeParams p_c = knode(k_loop_cond, dim3(1), dim3(1), 0, c_args);
      if ((e = cudaGraphAddKernelNode(&G.n_c[g], body, &last, 1, &p_c)) != cudaSuccess)
        return launch_error(e);
    } else {
      if ((e = cudaGraphExecKernelNodeSetParams(G.exec, G.n_set[g], &p_set)) != cudaSuccess ||
          (e = cudaGraphExecKernelNodeSetParams(G.exec, G.n_begin[g], &p_begin)) != cudaSuccess ||
          (e = cudaGraphExecKernelNodeSetParams(G.exec, G.n_a[g], &p_a)) != cudaSuccess ||
          (!K.one && (e = cudaGraphExecKernelNodeSetParams(G.exec, G.n_b[g], &p_b)) != cudaSuccess))
        return launch_error(e);
      const cudaKernelNodeParams p_c = knode(k_loop_cond, dim3(1), dim3(1), 0, c_args);
      if ((e = cudaGraphExecKernelNodeSetParams(G.exec, G.n_c[g], &p_c)) != cudaSuccess)
        return launch_error(e);
    }
  }
  if (!G.built) {
    if ((e = cudaGraphInstantiate(&G.exec, G.graph, 0)) != cudaSuccess) return launch_error(e);
    G.built = true;
  }
  return launch_error(cudaGraphLaunch(G.exec, st));
}

template <int N, int PC, bool CG>
int solve_t(int B, const KrylovArgs& a, cudaStream_t st) {
  using S = KShape<N>;
  constexpr int kChunk = 4;
  cudaError_t e;
  if constexpr (PC == 1 && !CG && half_ok<N>()) {
    // small batches (one CTA per SM at most): the whole solve in one kernel
    if (B <= persist_h_max_b() && use_half<N, PC, CG>(a)) {
      // TSF_PERSIST_CTAS=2: the register-capped instantiation (two CTAs per SM)
      static const bool two = [] {
        const char* s = getenv("TSF_PERSIST_CTAS");
        return s && s[0] == '2';
      }();
      // batches of at most one CTA per SM keep every vector that fits on chip
      static const int sms = [] {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
          n = 148;
        return n;
      }();
      const bool full = !two && B <= sms && HPersist<N>::NV > 3;
      SolveKernel kp = two    ? k_krylov_persist_h<N, (HShape<N>::MIN_BLOCKS > 1 ? HShape<N>::MIN_BLOCKS : 1), false>
                       : full ? k_krylov_persist_h<N, 1, true>
                              : k_krylov_persist_h<N, 1, false>;
      const int smem = two ? HShape<N>::SMEM : full ? HPersist<N>::BYTES : HPersist<N>::bytes(HPersist<N>::NV >= 3 ? 3 : 0);
      if ((e = prep_kernel(kp, smem)) != cudaSuccess) return launch_error(e);
      k_set_int<<<1, 1, 0, st>>>(a.active, B);
      kp<<<B, HShape<N>::BLOCK, smem, st>>>(a, a.kst, a.active);
      return launch_error(cudaGetLastError());
    }
  }
  if (a.graphs && graph_mode() && !persist_mode()) return solve_graph<N, PC, CG>(B, a, st);
  if (persist_mode()) {
    auto kp = k_krylov_persist<N, PC, CG>;
    if ((e = prep_kernel(kp, S::SMEM)) != cudaSuccess) return launch_error(e);
    k_set_int<<<1, 1, 0, st>>>(a.active, B);
    kp<<<B, S::BLOCK, S::SMEM, st>>>(a, a.kst, a.active);
    return launch_error(cudaGetLastError());
  }
  const SolveKernels<N, PC, CG> K(use_half<N, PC, CG>(a));
  const SolveKernel kb = K.kb, kv = K.kv, kt = K.kt, kc = K.kc;
  if ((e = prep_kernel(kb, K.smem)) != cudaSuccess) return launch_error(e);
  if (!CG) {
    if ((e = prep_kernel(kv, K.smem)) != cudaSuccess) return launch_error(e);
    if (!K.one && (e = prep_kernel(kt, K.smem)) != cudaSuccess) return launch_error(e);
  } else if ((e = prep_kernel(kc, K.smem)) != cudaSuccess) {
    return launch_error(e);
  }
  k_set_int<<<1, 1, 0, st>>>(a.active, B);
  kb<<<B, K.block, K.smem, st>>>(a, a.kst, a.active);
  if ((e = cudaGetLastError()) != cudaSuccess) return launch_error(e);
  for (int it = 0; it < a.max_iters; it += kChunk) {
    for (int k = 0; k < kChunk && it + k < a.max_iters; ++k) {
      if (!CG) {
        kv<<<B, K.block, K.smem, st>>>(a, a.kst, a.active);
        if (!K.one) kt<<<B, K.block, K.smem, st>>>(a, a.kst, a.active);
      } else {
        kc<<<B, K.block, K.smem, st>>>(a, a.kst, a.active);
      }
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return launch_error(e);
    if ((e = cudaMemcpyAsync(a.h_active, a.active, sizeof(int), cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
      return launch_error(e);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return launch_error(e);
    if (*a.h_active <= 0) break;
  }
  return 0;
}

template <int LOG>
int Dispatch<LOG>::solve(int B, int method, int pc, const KrylovArgs& a, cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  if (method == 0) {
    if (pc == 2) return solve_t<N, 2, false>(B, a, st);
    return pc ? solve_t<N, 1, false>(B, a, st) : solve_t<N, 0, false>(B, a, st);
  }
  if (pc == 2) return solve_t<N, 2, true>(B, a, st);
  return pc ? solve_t<N, 1, true>(B, a, st) : solve_t<N, 0, true>(B, a, st);
}

template <int LOG>
int Dispatch<LOG>::half_debug(int mode, int B, const double* x, const double* aux_in, double shift,
                              double2* hs, double* out, const FilterTables& t, cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  if constexpr (half_ok<N>()) {
    auto k = k_half_debug<N>;
    cudaError_t e = prep_kernel(k, HShape<N>::SMEM);
    if (e != cudaSuccess) return launch_error(e);
    k<<<B, HShape<N>::BLOCK, HShape<N>::SMEM, st>>>(mode, x, aux_in, shift, hs, out, t);
    return launch_error(cudaGetLastError());
  } else {
    return -1;
  }
}

template <int LOG>
int Dispatch<LOG>::layout() {
  return use64<(1 << (LOG - 1))>() ? 1 : 0;
}

template <int LOG>
int Dispatch<LOG>::fft(int inverse, int B, const double2* in, double2* out, const double2* tw,
                       cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  using S = KShape<N>;
  constexpr int E = FShape<N>::E;
  constexpr int smem = use64<N>() ? f64::kBytes
                                  : (kFftInPlace ? 1 : 2) * FftPlan<N, E>::SMEM_ELEMS * 16 +
                                        tw_table_elems(N) * 16;
  cudaError_t e;
  if (inverse) {
    auto k = k_fft_debug<N, E, true>;
    if ((e = prep_kernel(k, smem)) != cudaSuccess) return launch_error(e);
    k<<<B, S::BLOCK, smem, st>>>(in, out, tw, 0);
  } else {
    auto k = k_fft_debug<N, E, false>;
    if ((e = prep_kernel(k, smem)) != cudaSuccess) return launch_error(e);
    k<<<B, S::BLOCK, smem, st>>>(in, out, tw, 0);
  }
  return launch_error(cudaGetLastError());
}

}  // namespace tsf
