// Direct L1 history right-hand side of the DIDS scheme (run_dids,
// scheme.py:184-233, the history term at scheme.py:213-216):
//
//   rhs_i = ( f_i + (a_1/G) u^0_i ) + ( sum_{k=1}^{m-1} (a_{k+1} - a_k) u^k_i ) / G
//
// with a = l1_weights(mesh, gamma, m).a (mesh.py:53-80, computed on the host
// exactly as the reference does) and G = Gamma(1-gamma).  The sum is the
// reference's `np.diff(a) @ hist[1:m]` (an OpenBLAS GEMV): O(m n) HBM reads
// per level, streamed once.  Layout: thread (x, y) of a 32 x 8 CTA owns
// column i = 32*blockIdx.x + x and sums rows k = 1 + y, 1 + y + 8, ... (each
// warp reads one contiguous 256-byte row segment per step); the 8 row-group
// partials are combined in a fixed order (deterministic).  The first term
// keeps numpy's rounding (no FMA contraction: f + c0*h0 in two roundings).
#pragma once

#include "tsf_common.cuh"

namespace tsf {

constexpr int kDidsCols = 32;
constexpr int kDidsGroups = 8;

__global__ void __launch_bounds__(kDidsCols * kDidsGroups)
k_l1_history_rhs(int n, int rows, const double* __restrict__ hist, long inst_stride,
                 const double* __restrict__ w, double c0, double G,
                 const double* __restrict__ f, double* __restrict__ rhs) {
  __shared__ double part[kDidsGroups][kDidsCols];
  const int i = blockIdx.x * kDidsCols + threadIdx.x;
  const int b = blockIdx.y;
  const double* h = hist + (long)b * inst_stride;
  double s = 0.0;
  if (i < n) {
    for (int k = 1 + threadIdx.y; k < rows; k += kDidsGroups) s = fma(w[k - 1], h[(long)k * n + i], s);
  }
  part[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && i < n) {
    double acc = part[0][threadIdx.x];
#pragma unroll
    for (int g = 1; g < kDidsGroups; ++g) acc += part[g][threadIdx.x];
    const long o = (long)b * n + i;
    const double t = __dadd_rn(f[o], __dmul_rn(c0, h[i]));
    rhs[o] = rows > 1 ? __dadd_rn(t, __ddiv_rn(acc, G)) : t;
  }
}

}  // namespace tsf
