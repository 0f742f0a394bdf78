// Launch bodies of LargeDispatch<LOG> (tsf_large.cuh); explicitly
// instantiated one size per translation unit (gen/large_L*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstring>

#include "tsf_dispatch.h"
#include "tsf_large.cuh"
#include "tsf_hlarge.cuh"

namespace tsf {

int report_error(int code, const char* msg);   // tsf_abi.cu

inline int large_launch_error(cudaError_t e) {
  return e == cudaSuccess ? 0 : report_cuda(e, "large-n kernel launch");
}

template <typename K>
inline cudaError_t large_prep(K kernel, int smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// TMA tile loads (tsf_tma.cuh) apply when the vectors are exact N1 x N2
// views (n = nt: power-of-two n) and a G-column row segment is >= 16 bytes
template <int N1>
inline bool col_tma_ok(const LargeArgs& a, int which) {
  return (tma_mode() & which) && a.n == a.nt && LCol<N1>::G * 8 >= 16;
}

template <int LOG>
int LargeDispatch<LOG>::col_fwd(const LargeArgs& a, const double* src, int in_mode,
                                cudaStream_t st) {
  constexpr int N1 = 1 << LOG;
  using S = LCol<N1>;
  const dim3 grid(a.nt / N1 / S::G, a.B);
  ColMaps cm;
  memset(&cm, 0, sizeof(cm));
  if (col_tma_ok<N1>(a, 1)) {
    const int N2 = (int)(a.nt / N1);
    const double* vs[3] = {src, nullptr, nullptr};
    int nv = 1;
    if (in_mode == CI_PUPD) {
      vs[0] = a.r; vs[1] = a.p; vs[2] = a.v; nv = 3;
    } else if (in_mode == CI_SUPD) {
      vs[0] = a.r; vs[1] = a.v; nv = 2;
    }
    int rc = 0;
    for (int q = 0; q < nv && !rc; ++q)
      rc = tma_map_vector(&cm.v[q], vs[q], a.n, N1, N2, a.B, S::G);
    if (rc) return rc;
    cm.nv = nv;
    cm.use = 1;
  }
  auto k = few_ctas((long)grid.x * grid.y) ? k_lcol_fwd<N1, 1> : k_lcol_fwd<N1>;
  static cudaError_t prep = large_prep(k_lcol_fwd<N1>, S::SMEM);
  static cudaError_t prep1 = large_prep(k_lcol_fwd<N1, 1>, S::SMEM);
  if (prep != cudaSuccess) return large_launch_error(prep);
  if (prep1 != cudaSuccess) return large_launch_error(prep1);
  launch_pdl(k, grid, S::BLOCK, S::SMEM, st, a, src, in_mode, cm);
  return large_launch_error(cudaGetLastError());
}

template <int LOG>
int LargeDispatch<LOG>::row(const LargeArgs& a, int spec_mode, cudaStream_t st) {
  constexpr int N2 = 1 << LOG;
  using S = LRow<N2>;
  // short rows (N2 <= 128: n = 8192) — at N2 = 256 (configs[1]) measured no
  // faster than k_lrow, which stays (profiles/r01c_summary.md)
  if constexpr (S::T < 32) {
    constexpr int IT = 64 / S::T;
    constexpr int smem = (IT * 2 * FftPlan<N2, S::E>::SMEM_ELEMS + tw_table_elems(N2)) * 16;
    auto ks = k_lrow_small<N2>;
    static cudaError_t prep_s = large_prep(ks, smem);
    if (prep_s != cudaSuccess) return large_launch_error(prep_s);
    const int items = (int)(a.nt / N2) * (spec_mode == RS_APPLY ? 2 : 1);
    launch_pdl(ks, dim3((items + IT - 1) / IT, a.B), 64, smem, st, a, spec_mode);
    return large_launch_error(cudaGetLastError());
  }
  auto k = k_lrow<N2>;
  static cudaError_t prep = large_prep(k, S::SMEM);
  if (prep != cudaSuccess) return large_launch_error(prep);
  launch_pdl(k, dim3(a.nt / N2, a.B), S::BLOCK, S::SMEM, st, a, spec_mode);
  return large_launch_error(cudaGetLastError());
}

template <int LOG>
int LargeDispatch<LOG>::col_inv(const LargeArgs& a, double* dst, int out_mode, const double* xin,
                                const double* w1, int pslot, cudaStream_t st) {
  constexpr int N1 = 1 << LOG;
  using S = LCol<N1>;
  const dim3 grid(a.nt / N1 / S::G, a.B);
  ColMaps cm;
  memset(&cm, 0, sizeof(cm));
  if (col_tma_ok<N1>(a, 2)) {
    const int rc = tma_map_z(&cm.z, a.Z, N1, (int)(a.nt / N1), a.B, S::G);
    if (rc) return rc;
    cm.use = 1;
  }
  const int smem = S::SMEM;
  auto k = few_ctas((long)grid.x * grid.y) ? k_lcol_inv<N1, 1> : k_lcol_inv<N1>;
  static cudaError_t prep = large_prep(k_lcol_inv<N1>, S::SMEM);
  static cudaError_t prep1 = large_prep(k_lcol_inv<N1, 1>, S::SMEM);
  if (prep != cudaSuccess) return large_launch_error(prep);
  if (prep1 != cudaSuccess) return large_launch_error(prep1);
  launch_pdl(k, grid, S::BLOCK, smem, st, a, dst, out_mode, xin, w1, pslot, cm);
  return large_launch_error(cudaGetLastError());
}

template <int LOG>
int LargeDispatch<LOG>::hcol_fwd(const LargeArgs& a, const double* src, int in_mode,
                                 cudaStream_t st) {
  constexpr int N1 = 1 << LOG;
  using S = LCol<N1>;
  const dim3 grid(a.hg.N2 / S::G, a.B);
  ColMaps cm;
  memset(&cm, 0, sizeof(cm));
  // packed [N1 x G] operand tiles (16-byte words) by TMA: the vector as
  // {2 N2, N1, B} doubles, boxes of 2 G doubles
  if ((tma_half_mode() & 1) && in_mode != HF_ODD && N1 <= 2048 &&
      !few_ctas((long)grid.x * grid.y)) {
    const double* vs[2] = {src, nullptr};
    int nv = 1;
    if (in_mode == HF_PUPD) {
      vs[0] = a.p; vs[1] = a.v; nv = 2;
    } else if (in_mode == HF_SUPD) {
      vs[0] = a.r; vs[1] = a.v; nv = 2;
    }
    int rc = 0;
    for (int q = 0; q < nv && !rc; ++q)
      rc = tma_map_vector(&cm.v[q], vs[q], a.n, N1, 2 * a.hg.N2, a.B, 2 * S::G);
    if (rc) return rc;
    cm.nv = nv;
    cm.use = 1;
  }
  auto k = k_hcol_fwd<N1>;
  static cudaError_t prep = large_prep(k, S::SMEM);
  if (prep != cudaSuccess) return large_launch_error(prep);
  launch_pdl(k, grid, S::BLOCK, S::SMEM, st, a, src, in_mode, cm);
  return large_launch_error(cudaGetLastError());
}

template <int LOG>
int LargeDispatch<LOG>::hrow_strang(const LargeArgs& a, int mode, cudaStream_t st) {
  constexpr int N2 = 1 << LOG;
  if constexpr (HRow<N2>::OK) {
    using S = HRow<N2>;
    auto k = k_hrow_strang<N2>;
    static cudaError_t prep = large_prep(k, S::SMEM);
    if (prep != cudaSuccess) return large_launch_error(prep);
    launch_pdl(k, dim3(a.hg.N1 / 2 / S::NP, a.B), S::BLOCK, S::SMEM, st, a, mode);
    return large_launch_error(cudaGetLastError());
  } else {
    return report_error(-3, "half-length row pairs need 64 <= N2 <= 2048");
  }
}

template <int LOG>
int LargeDispatch<LOG>::hrow_mv(const LargeArgs& a, cudaStream_t st) {
  constexpr int N2 = 1 << LOG;
  if constexpr (HRow<N2>::OK) {
    using S = LRow<N2>;
    auto k = k_hrow_mv<N2>;
    static cudaError_t prep = large_prep(k, S::SMEM);
    if (prep != cudaSuccess) return large_launch_error(prep);
    launch_pdl(k, dim3(a.hg.N1, a.B), S::BLOCK, S::SMEM, st, a);
    return large_launch_error(cudaGetLastError());
  } else {
    return report_error(-3, "half-length rows need 64 <= N2 <= 2048");
  }
}

template <int LOG>
int LargeDispatch<LOG>::hcol_inv(const LargeArgs& a, double* dst, int out_mode, double* dst1,
                                 const double* xin, const double* ye, const double* w1, int pslot,
                                 cudaStream_t st) {
  constexpr int N1 = 1 << LOG;
  using S = LCol<N1>;
  const dim3 grid(a.hg.N2 / S::G, a.B, (out_mode == HO_PACK && dst1) ? 2 : 1);
  ColMaps cm;
  memset(&cm, 0, sizeof(cm));
  if ((tma_half_mode() & 2) && N1 <= 2048 && !few_ctas((long)grid.x * grid.y)) {
    const int rc = tma_map_z(&cm.z, a.Z, N1, a.hg.N2, a.B, S::G);
    if (rc) return rc;
    cm.use = 1;
  }
  auto k = k_hcol_inv<N1>;
  static cudaError_t prep = large_prep(k, S::SMEM);
  if (prep != cudaSuccess) return large_launch_error(prep);
  launch_pdl(k, grid, S::BLOCK, S::SMEM, st, a, dst, out_mode, dst1, xin, ye, w1, pslot, cm);
  return large_launch_error(cudaGetLastError());
}

template <int LOG>
int LargeDispatch<LOG>::col_group() {
  return LCol<1 << LOG>::G;
}

}  // namespace tsf
