// Real, even circulant filters applied to real data with full complex FFTs.
//
// Both operators on the hot path multiply by a real, even spectrum:
//   * Toeplitz matvec  A x = first_n( Re IFFT_L( S . FFT_L(pad_L x) ) ),
//     S = FFT of the even circulant embedding of A's first column
//     (toeplitz.py:34-63);
//   * Strang solve     P^{-1} v = Re IFFT_n( FFT_n(v) / (d + kbar lam) )
//     (toeplitz.py:101-136), lam real and even.
// Exactly like the reference, each is ONE complex transform pair on the real
// data (imaginary part zero) followed by taking the real part.  The cheaper
// real-packed variant (two reals per complex point, half-length transforms)
// was implemented first and measured: its rounding errors alias bin k with
// bin k+L/2, and at the Krylov tolerance 1e-12 that biased BiCGSTAB by +0.5
// iterations per level against the reference, so the hot
// path keeps the full transforms.
//
// Ownership (tsf_fft.cuh): a CTA has T = L/16 owning threads; thread tid
// owns the real entries j = tid + c*T, c < 8, of every vector (j < L/2 >= n),
// which are exactly the nonzero inputs / needed outputs of the length-L
// transform (slots c < 8 of E = 16) and all slots of the length-n Strang
// transform (E = 8, pow2 n = L/2).
//
// The reference keeps the REAL part of the inverse, which makes its
// effective filters the even parts of S and of 1/total; those are formed
// explicitly (host side for S, per bin for 1/total): numpy's lam is even only
// up to rounding of size eps*max(lam), which is large relative to total at
// low frequencies where 1/total peaks.
#pragma once

#include "tsf_fft.cuh"

namespace tsf {

struct FilterTables {
  const double2* tw;    // W_L^e, e < L
  const double* mvS;    // even part of the Toeplitz symbol / L, k < L
  const double2* pclam; // (lam_k, lam_{n-k}), k < n   (pow2 n = L/2 only)
};

TSF_D double ld_real(const double* __restrict__ base, int n, int j) {
  return j < n ? base[j] : 0.0;
}
TSF_D void st_real(double* __restrict__ base, int n, int j, double v) {
  if (j < n) base[j] = v;
}

// y = A x for the owned entries io[c] (j = tid + c*T); L = 16*T.
template <int L>
TSF_D void toeplitz_filter(double (&io)[8], double2* sm, const FilterTables& t) {
  constexpr int T = L / 16;
  double2 z[16];
#pragma unroll
  for (int c = 0; c < 8; ++c) z[c] = make_double2(io[c], 0.0);
#pragma unroll
  for (int c = 8; c < 16; ++c) z[c] = make_double2(0.0, 0.0);
  block_fft<L, 16, false>(z, sm, t.tw, 0);
  if (threadIdx.x < T) {
#pragma unroll
    for (int c = 0; c < 16; ++c) z[c] = cscale(z[c], __ldg(&t.mvS[threadIdx.x + c * T]));
  }
  block_fft<L, 16, true>(z, sm, t.tw, 0);
#pragma unroll
  for (int c = 0; c < 8; ++c) io[c] = z[c].x;
}

// z = P^{-1} v, P = d I + kbar s(A); n = L/2 (power of two).
template <int L>
TSF_D void strang_filter(double (&io)[8], double2* sm, const FilterTables& t, double d,
                         double kbar) {
  constexpr int N = L / 2;
  constexpr int T = N / 8;
  constexpr double inv_n = 1.0 / N;
  double2 z[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) z[c] = make_double2(io[c], 0.0);
  block_fft<N, 8, false>(z, sm, t.tw, 1);
  if (threadIdx.x < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 lam = __ldg(&t.pclam[threadIdx.x + c * T]);
      const double s = 0.5 * (1.0 / (d + kbar * lam.x) + 1.0 / (d + kbar * lam.y));
      z[c] = cscale(z[c], s * inv_n);
    }
  }
  block_fft<N, 8, true>(z, sm, t.tw, 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) io[c] = z[c].x;
}

}  // namespace tsf
