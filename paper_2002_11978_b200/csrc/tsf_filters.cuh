// Real-even circulant filters on real data packed two-per-complex.
//
// Both operators on the hot path are "multiply by a real, even spectrum":
//   * the Toeplitz matvec A x = first_n( IFFT_L( S . FFT_L(pad_L x) ) ),
//     S = FFT of the even circulant embedding (toeplitz.py:34-63);
//   * the Strang preconditioner P^{-1} v = IFFT_n( FFT_n(v) / (d + kbar lam) )
//     (toeplitz.py:101-136), lam real and even.
// A length-2N real filter is done with ONE length-N complex FFT pair:
//   z_j = x_{2j} + i x_{2j+1},  Z = FFT_N(z),
//   Z'_k = a_k Z_k + i b_k conj(Z_{N-k}),  z' = IFFT_N(Z'),
//   a_k = P_k - Q_k sin(th_k), b_k = Q_k cos(th_k), th_k = 2 pi k / 2N,
//   P_k = (S_k + S_{k+N})/2, Q_k = (S_k - S_{k+N})/2,
// and y_{2j} + i y_{2j+1} = z'_j (the 1/N of the inverse is folded into
// a_k, b_k).  Derivation in DESIGN.md §3.
//
// Slot convention (see tsf_fft.cuh): thread tid owns complex slots
// j = tid + c*T, c < 16 for the matvec transform (N_mv = L/2 points) and
// c < 8 for the preconditioner transform (N_pc = n/2 points, pow2 n), so a
// real vector is held as 8 double2 per thread: x2[c] = (x[2j], x[2j+1]).
#pragma once

#include "tsf_fft.cuh"

namespace tsf {

struct FilterTables {
  const double2* tw;     // W_{N_mv}^e, e < N_mv
  const double2* mvab;   // (a_k, b_k) of the Toeplitz symbol, k < N_mv (1/N_mv folded)
  const double2* pclam;  // (lam_k, lam_{k+N_pc}), k < N_pc
  const double2* pcsc;   // (sin th_k, cos th_k), th_k = 2 pi k / n, k < N_pc
};

// Load/store of the owned pairs of a real vector of length n (any n).
TSF_D double2 ld_pair(const double* __restrict__ base, int n, int j) {
  const int i = 2 * j;
  if (i + 1 < n) {
    if ((n & 1) == 0) return *reinterpret_cast<const double2*>(base + i);
    return make_double2(base[i], base[i + 1]);
  }
  if (i < n) return make_double2(base[i], 0.0);
  return make_double2(0.0, 0.0);
}
TSF_D void st_pair(double* __restrict__ base, int n, int j, double2 v) {
  const int i = 2 * j;
  if (i + 1 < n) {
    if ((n & 1) == 0) {
      *reinterpret_cast<double2*>(base + i) = v;
    } else {
      base[i] = v.x;
      base[i + 1] = v.y;
    }
  } else if (i < n) {
    base[i] = v.x;
  }
}

// After a forward transform the owned spectrum is in z[]; exchange with the
// mirrored bin N-k through shared memory and apply Z'_k = a Z_k + i b conj(Z_{N-k}).
// ABF(k) returns (a_k, b_k).
template <int N, int E, typename ABF>
TSF_D void apply_even_filter(double2 (&z)[E], double2* sm, ABF abf) {
  using PL = FftPlan<N, E>;
  const int tid = threadIdx.x;
  const bool own = tid < PL::T;
  __syncthreads();
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) sm[PL::pad(tid + c * PL::T)] = z[c];
  }
  __syncthreads();
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k = tid + c * PL::T;
      const double2 zm = sm[PL::pad((N - k) & (N - 1))];
      const double2 ab = abf(k);
      const double2 zk = z[c];
      z[c] = make_double2(fma(ab.x, zk.x, ab.y * zm.y), fma(ab.x, zk.y, ab.y * zm.x));
    }
  }
}

// y = A x (Toeplitz matvec through the embedding of length L = 2*NMV).
// io[c], c < 8: in = x pairs, out = (A x) pairs.
template <int NMV>
TSF_D void toeplitz_filter(double2 (&io)[8], double2* sm, const FilterTables& t) {
  double2 z[16];
#pragma unroll
  for (int c = 0; c < 8; ++c) z[c] = io[c];
#pragma unroll
  for (int c = 8; c < 16; ++c) z[c] = make_double2(0.0, 0.0);
  block_fft<NMV, 16, false>(z, sm, t.tw, 0);
  apply_even_filter<NMV, 16>(z, sm, [&](int k) { return __ldg(&t.mvab[k]); });
  block_fft<NMV, 16, true>(z, sm, t.tw, 0);
#pragma unroll
  for (int c = 0; c < 8; ++c) io[c] = z[c];
}

// z = P^{-1} v with P = d I + kbar s(A), pow2 n = NMV (N_pc = NMV/2).
template <int NMV>
TSF_D void strang_filter(double2 (&io)[8], double2* sm, const FilterTables& t, double d,
                         double kbar) {
  constexpr int NPC = NMV / 2;
  const double half_inv = 0.5 / NPC;
  block_fft<NPC, 8, false>(io, sm, t.tw, 1);
  apply_even_filter<NPC, 8>(io, sm, [&](int k) {
    const double2 lam = __ldg(&t.pclam[k]);
    const double2 sc = __ldg(&t.pcsc[k]);
    const double s1 = 1.0 / (d + kbar * lam.x);
    const double s2 = 1.0 / (d + kbar * lam.y);
    const double P = (s1 + s2) * half_inv;
    const double Q = (s1 - s2) * half_inv;
    return make_double2(fma(-Q, sc.x, P), Q * sc.y);
  });
  block_fft<NPC, 8, true>(io, sm, t.tw, 1);
}

}  // namespace tsf
