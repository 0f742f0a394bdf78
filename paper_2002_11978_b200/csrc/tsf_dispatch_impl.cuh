// Kernel launch bodies of Dispatch<LOG> (see tsf_dispatch.h); LOG = log2(L),
// the per-instance transform length is N = L/2.
#pragma once

#include <cuda_runtime.h>

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
  cudaError_t e = prep_kernel(k, S::FFT_BYTES);
  if (e != cudaSuccess) return launch_error(e);
  k<<<B, S::BLOCK, S::FFT_BYTES, st>>>(n, v, z, shift, kbar, kbar_dev, t);
  return launch_error(cudaGetLastError());
}

template <int N, int PC, bool CG>
int solve_t(int B, const KrylovArgs& a, cudaStream_t st) {
  using S = KShape<N>;
  auto k = k_krylov_solve<N, PC, CG>;
  cudaError_t e = prep_kernel(k, S::SMEM);
  if (e != cudaSuccess) return launch_error(e);
  k<<<B, S::BLOCK, S::SMEM, st>>>(a);
  return launch_error(cudaGetLastError());
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
  constexpr int smem = FftPlan<N, 16>::SMEM_ELEMS * 16;
  cudaError_t e;
  if (inverse) {
    auto k = k_fft_debug<N, 16, true>;
    if ((e = prep_kernel(k, smem)) != cudaSuccess) return launch_error(e);
    k<<<B, S::BLOCK, smem, st>>>(in, out, tw, 0);
  } else {
    auto k = k_fft_debug<N, 16, false>;
    if ((e = prep_kernel(k, smem)) != cudaSuccess) return launch_error(e);
    k<<<B, S::BLOCK, smem, st>>>(in, out, tw, 0);
  }
  return launch_error(cudaGetLastError());
}

}  // namespace tsf
