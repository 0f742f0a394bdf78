// Large-n engine (n = N1*N2 > 4096, power of two): four-step transforms
// through L2/HBM, one CTA per column or row of the N1 x N2 view.
//
// A length-N filter  y = IFFT_N( S . FFT_N(x) )  is three kernels:
//   col_fwd : per column t2, x[N2 t1 + t2] (t1 < N1) -> FFT_N1 -> * W_N^{t2 k1}
//             -> Z[k1][t2]                      (input prologue: load / modulate /
//                                                 Krylov vector update)
//   row     : per row k1, FFT_N2 over Z[k1][.] -> * S[k1 + N1 k2] -> IFFT_N2
//             (S stored permuted as [k1][k2])
//   col_inv : per column t2, Z[.][t2] * conj(W_N^{t2 k1}) -> IFFT_N1 -> y at
//             j = N2 t1 + t2                   (epilogue: store / combine /
//                                                 operator / dot partials)
// The matvec uses the same even/odd-bin split as the single-CTA engine
// (tsf_filters.cuh): two length-n filters, the odd one on x_j W_L^j.
// Reductions are deterministic: per-CTA partials [B][4][N2] reduced in fixed
// order by one-thread-per-instance scalar kernels, which also hold the
// reference's BiCGSTAB/PCG control flow (krylov.py:43-153).
#pragma once

#include "tsf_kernels.cuh"

namespace tsf {

struct LargeTables {
  const double2* tw1;   // two-level W_N1 table (column transforms)
  const double2* tw2;   // two-level W_N2 table (row transforms)
  const double2* twN;   // two-level W_N table (N = n): inter-pass twiddles
  const double2* twL;   // two-level W_L table (L = 2n), modulation of the odd half
  const double2* sEO;   // [k1][k2] -> (S_{2k}, S_{2k+1}) / L at k = k1 + N1 k2
  const double2* lamP;  // [k1][k2] -> (lam_k, lam_{n-k}) at k = k1 + N1 k2 (Strang)
};

// BiCGSTAB / PCG per-instance control (scalar kernels)
enum LMode : int { LM_ACTIVE = 0, LM_EARLY = 1, LM_DONE = 2 };

struct LState {
  double rho, rho_new, alpha, omega, nrm0, rnorm, snorm, kbar, rz;
  int it, mode;
};

// Column prologues
enum ColIn : int {
  CI_LOAD = 0,     // z = x
  CI_MOD = 1,      // z = x_j W_L^j
  CI_PUPD = 2,     // p = r + beta (p - omega v) (or r0 at it 1); store p; z = p
  CI_SUPD = 3,     // s = r - alpha v; store s; ||s||^2 partial; z = s
};
// Column epilogues
enum ColOut : int {
  CO_REAL = 0,     // y_j = Re z   (store)
  CO_COMBINE = 1,  // y_j = d x_j + kappa_j (ye_j + Re(conj(w_j) z)) ; dot partials
};
// Row spectra
enum RowSpec : int { RS_EVEN = 0, RS_ODD = 1, RS_STRANG = 2 };

struct LargeArgs {
  int n, B;
  LargeTables lt;
  double2* Z;          // [B][N] transform work array
  double* ye;          // [B][N] even-half result
  double* part;        // [B][4][NP] partial sums (NP = max(N1, N2))
  int np;
  LState* st;          // [B]
  // Krylov vectors [B][n]
  const double* r0;
  double* x;
  double* r;
  double* p;
  double* v;
  double* ph;
  double* s;
  double* sh;
  double* t;
  const double* kappa;  // level diffusivity [B][n] (null: plain Toeplitz product)
  double* pspec;       // [B][N] permuted Strang spectrum S_k / n
  double shift;
  double tol;
  int max_iters;
  int* iters;
  double* relres;
  int* status;
  int* active;
};

TSF_D bool inst_skip(const LargeArgs& a, int b) { return a.st[b].mode != LM_ACTIVE; }

// two-level table lookup straight from global memory (L1/L2 resident)
TSF_D double2 tw_get_g(const double2* tw, long e) {
  return cmul(ldt(&tw[kTwLo + (e >> 6)]), ldt(&tw[tw_lo_slot((int)(e & 63))]));
}

template <int NT>
TSF_D void stage_tw(double2* dst, const double2* src) {
  for (int i = threadIdx.x; i < tw_table_elems(NT); i += blockDim.x) dst[i] = ldt(&src[i]);
}

// ------------------------------------------------------------ col_fwd
template <int N1>
__global__ void __launch_bounds__(FShape<N1>::T < 32 ? 32 : FShape<N1>::T)
k_lcol_fwd(LargeArgs a, const double* __restrict__ src, int in_mode, int real_input) {
  const int N2 = a.n / N1;
  const long N = a.n;
  constexpr int E = FShape<N1>::E;
  constexpr int T = FShape<N1>::T;
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  const int t2 = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  if (a.st && inst_skip(a, b)) return;
  double2* tw1 = sm + 2 * FftPlan<N1, E>::SMEM_ELEMS;
  stage_tw<N1>(tw1, a.lt.tw1);
  const long off = (long)b * a.n;
  const bool own = tid < T;
  double xr[E];
  double2 z[E];
  double part = 0.0;
  const LState stv = a.st ? a.st[b] : LState{};
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int t1 = tid + c * T;
      const long j = (long)N2 * t1 + t2;
      double val;
      if (in_mode == CI_PUPD) {
        if (stv.it == 1) {
          val = a.r0[off + j];
        } else {
          const double beta = (stv.rho_new / stv.rho) * (stv.alpha / stv.omega);
          val = a.r[off + j] + beta * (a.p[off + j] - stv.omega * a.v[off + j]);
        }
        a.p[off + j] = val;
      } else if (in_mode == CI_SUPD) {
        const double* rc = (stv.it == 1) ? a.r0 : a.r;
        val = rc[off + j] - stv.alpha * a.v[off + j];
        a.s[off + j] = val;
        part = fma(val, val, part);
      } else {
        val = src[off + j];
      }
      xr[c] = val;
      if (!real_input) z[c] = cscale(tw_get_g(a.lt.twL, j), val);  // x_j W_L^j
    }
  }
  if (in_mode == CI_SUPD) {
    part = block_sum1(part, red);
    if (tid == 0) a.part[((long)b * 4 + 2) * a.np + t2] = part;
  }
  if (real_input) block_fft_real<N1, E>(xr, z, sm, tw1, 0);
  else block_fft<N1, E, false>(z, sm, tw1, 0);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k1 = tid + c * T;
      const double2 w = tw_get_g(a.lt.twN, ((long)t2 * k1) % N);
      a.Z[(long)b * N + (long)k1 * N2 + t2] = cmul(z[c], w);
    }
  }
}

// ------------------------------------------------------------ row
template <int N2>
__global__ void __launch_bounds__(FShape<N2>::T < 32 ? 32 : FShape<N2>::T)
k_lrow(LargeArgs a, int spec_mode) {
  const long N = a.n;
  constexpr int E = FShape<N2>::E;
  constexpr int T = FShape<N2>::T;
  extern __shared__ double2 sm[];
  const int k1 = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  if (a.st && inst_skip(a, b)) return;
  double2* tw2 = sm + 2 * FftPlan<N2, E>::SMEM_ELEMS;
  stage_tw<N2>(tw2, a.lt.tw2);
  const bool own = tid < T;
  double2* row = a.Z + (long)b * N + (long)k1 * N2;
  double2 z[E];
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = row[tid + c * T];
  }
  block_fft<N2, E, false>(z, sm, tw2, 0);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long idx = (long)k1 * N2 + tid + c * T;   // bin k1 + N1 k2
      double s;
      if (spec_mode == RS_EVEN) s = ldt(&a.lt.sEO[idx]).x;
      else if (spec_mode == RS_ODD) s = ldt(&a.lt.sEO[idx]).y;
      else s = a.pspec[(long)b * N + idx];
      z[c] = cscale(z[c], s);
    }
  }
  block_fft<N2, E, true>(z, sm, tw2, 0);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) row[tid + c * T] = z[c];
  }
}

// ------------------------------------------------------------ col_inv
template <int N1>
__global__ void __launch_bounds__(FShape<N1>::T < 32 ? 32 : FShape<N1>::T)
k_lcol_inv(LargeArgs a, double* __restrict__ dst, int out_mode, const double* __restrict__ xin,
           const double* __restrict__ w1, int pslot) {
  const int N2 = a.n / N1;
  const long N = a.n;
  constexpr int E = FShape<N1>::E;
  constexpr int T = FShape<N1>::T;
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  const int t2 = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  if (a.st && inst_skip(a, b)) return;
  double2* tw1 = sm + 2 * FftPlan<N1, E>::SMEM_ELEMS;
  stage_tw<N1>(tw1, a.lt.tw1);
  const long off = (long)b * a.n;
  const bool own = tid < T;
  double2 z[E];
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k1 = tid + c * T;
      const double2 w = tw_get_g(a.lt.twN, ((long)t2 * k1) % N);
      z[c] = cmulc(a.Z[(long)b * N + (long)k1 * N2 + t2], w);
    }
  }
  block_fft<N1, E, true>(z, sm, tw1, 0);
  Vals<2> pr;
  pr.v[0] = pr.v[1] = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int t1 = tid + c * T;
      const long j = (long)N2 * t1 + t2;
      if (out_mode == CO_REAL) {
        dst[off + j] = z[c].x;
      } else {
        const double2 w = tw_get_g(a.lt.twL, j);
        const double ax = a.ye[off + j] + fma(z[c].x, w.x, z[c].y * w.y);
        const double y = a.kappa ? fma(a.shift, xin[off + j], a.kappa[off + j] * ax) : ax;
        dst[off + j] = y;
        pr.v[0] = fma(y, y, pr.v[0]);
        if (w1) pr.v[1] = fma(y, w1[off + j], pr.v[1]);
      }
    }
  }
  if (out_mode == CO_COMBINE && pslot >= 0) {
    pr = block_sum<2>(pr, red);
    if (tid == 0) {
      a.part[((long)b * 4 + pslot) * a.np + t2] = pr.v[0];
      a.part[((long)b * 4 + pslot + 1) * a.np + t2] = pr.v[1];
    }
  }
}

// Per-size launchers (bodies in tsf_large_impl.cuh, one TU per size:
// gen/large_L*.cu).  LOG = log2 of the column (N1) or row (N2) length.
constexpr int kLargeMinLog = 6;   // N1 >= 64
constexpr int kLargeMaxLog = 12;  // N1, N2 <= 4096  ->  n <= 2^24

template <int LOG>
struct LargeDispatch {
  static int col_fwd(const LargeArgs& a, const double* src, int in_mode, int real_input,
                     cudaStream_t st);
  static int row(const LargeArgs& a, int spec_mode, cudaStream_t st);
  static int col_inv(const LargeArgs& a, double* dst, int out_mode, const double* xin,
                     const double* w1, int pslot, cudaStream_t st);
};

#define TSF_EXTERN_LARGE(L) extern template struct LargeDispatch<L>;
TSF_EXTERN_LARGE(6)
TSF_EXTERN_LARGE(7)
TSF_EXTERN_LARGE(8)
TSF_EXTERN_LARGE(9)
TSF_EXTERN_LARGE(10)
TSF_EXTERN_LARGE(11)
TSF_EXTERN_LARGE(12)

}  // namespace tsf
