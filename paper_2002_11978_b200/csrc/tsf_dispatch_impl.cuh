// Kernel launch bodies of Dispatch<LOG> (see tsf_dispatch.h); LOG = log2(L),
// the per-instance transform length is N = L/2.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

#include "tsf_dispatch.h"

namespace tsf {

inline int launch_error(cudaError_t e) {
  return e == cudaSuccess ? 0 : report_cuda(e, "kernel launch");
}

template <typename K>
inline cudaError_t prep_kernel(K kernel, int smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

template <int LOG>
int Dispatch<LOG>::matvec(int n, const FilterTables& t, int B, const double* x, double* y,
                          const double* kappa, double shift, cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  using S = KShape<N>;
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

template <int N, int PC, bool CG>
int solve_t(int B, const KrylovArgs& a, cudaStream_t st) {
  using S = KShape<N>;
  constexpr int kChunk = 4;
  cudaError_t e;
  if (persist_mode()) {
    auto kp = k_krylov_persist<N, PC, CG>;
    if ((e = prep_kernel(kp, S::SMEM)) != cudaSuccess) return launch_error(e);
    k_set_int<<<1, 1, 0, st>>>(a.active, B);
    kp<<<B, S::BLOCK, S::SMEM, st>>>(a, a.kst, a.active);
    return launch_error(cudaGetLastError());
  }
  auto kb = k_solve_begin<N, PC, CG>;
  if ((e = prep_kernel(kb, S::SMEM)) != cudaSuccess) return launch_error(e);
  auto kv = k_bicg_v<N, PC>;
  auto kt = k_bicg_t<N, PC>;
  auto kc = k_cg_iter<N, PC>;
  if (!CG) {
    if ((e = prep_kernel(kv, S::SMEM)) != cudaSuccess) return launch_error(e);
    if ((e = prep_kernel(kt, S::SMEM)) != cudaSuccess) return launch_error(e);
  } else if ((e = prep_kernel(kc, S::SMEM)) != cudaSuccess) {
    return launch_error(e);
  }
  k_set_int<<<1, 1, 0, st>>>(a.active, B);
  kb<<<B, S::BLOCK, S::SMEM, st>>>(a, a.kst, a.active);
  if ((e = cudaGetLastError()) != cudaSuccess) return launch_error(e);
  for (int it = 0; it < a.max_iters; it += kChunk) {
    for (int k = 0; k < kChunk && it + k < a.max_iters; ++k) {
      if (!CG) {
        kv<<<B, S::BLOCK, S::SMEM, st>>>(a, a.kst, a.active);
        kt<<<B, S::BLOCK, S::SMEM, st>>>(a, a.kst, a.active);
      } else {
        kc<<<B, S::BLOCK, S::SMEM, st>>>(a, a.kst, a.active);
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
  if (method == 0) return pc ? solve_t<N, 1, false>(B, a, st) : solve_t<N, 0, false>(B, a, st);
  return pc ? solve_t<N, 1, true>(B, a, st) : solve_t<N, 0, true>(B, a, st);
}

template <int LOG>
int Dispatch<LOG>::fft(int inverse, int B, const double2* in, double2* out, const double2* tw,
                       cudaStream_t st) {
  constexpr int N = 1 << (LOG - 1);
  using S = KShape<N>;
  constexpr int E = FShape<N>::E;
  constexpr int smem = (kFftInPlace ? 1 : 2) * FftPlan<N, E>::SMEM_ELEMS * 16 + tw_table_elems(N) * 16;
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
