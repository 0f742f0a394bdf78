// Real, even circulant filters applied to real data with complex FFTs of
// length N = L/2 (one CTA, shared memory).
//
// Both operators on the hot path multiply by a real, even spectrum:
//   * Toeplitz matvec  A x = first_n( Re IFFT_L( S . FFT_L(pad_L x) ) ),
//     S = FFT of the even circulant embedding of A's first column
//     (toeplitz.py:34-63);
//   * Strang solve     P^{-1} v = Re IFFT_n( FFT_n(v) / (d + kbar lam) )
//     (toeplitz.py:101-136), lam real and even.
//
// Matvec.  x is zero beyond n <= N = L/2, so one radix-2 DIF step splits the
// length-L transform into two length-N ones (even / odd output bins):
//   X_{2k}   = FFT_N(x)_k,            X_{2k+1} = FFT_N(x_j w_j)_k,  w_j = W_L^j
//   y_j = (1/L) [ IFFT_N(S_{2k} X_{2k})_j + conj(w_j) IFFT_N(S_{2k+1} X_{2k+1})_j ],
// and the real part is kept, as the reference does.  Each half is a full
// complex transform of the data (imaginary part zero or the modulation) —
// NOT the cheaper two-reals-per-complex packing: that variant was built and
// measured first, and its rounding errors alias bin k onto bin k+N, which at
// the Krylov tolerance 1e-12 biased BiCGSTAB by +0.5 iterations per level
// against the reference.  The split keeps the shared-memory
// footprint at N complex points (64 KB for n = 4096).
//
// Effective spectra are the EVEN parts of S and 1/total, which is what the
// reference's Re(...) keeps: numpy's FFTs of even sequences are even only up
// to rounding of size eps*max, large relative to 1/total at low frequency.
//
// Ownership (tsf_fft.cuh): T = N/E owning threads; thread tid owns the real
// entries j = tid + c*T, c < E, of every vector (covering j < N, n <= N).
#pragma once

#include "tsf_fft.cuh"
#include "tsf_fft64.cuh"

namespace tsf {

struct FilterTables {
  const double2* tw;    // two-level W_L table (tsf_fft.cuh tw_get); kernels stage it in smem
  const double2* mvS;   // (S_{2k}, S_{2k+1}) / L, even part of the symbol, k < N
  const double2* pclam; // (lam_k, lam_{n-k}), k < n   (pow2 n = N only)
  const double* ps = nullptr;  // the instance's staged Strang spectrum (shared memory) or null
  const double2* ptw = nullptr;  // per-pass twiddles of the length-N transform (TSF_PASS_TW)
};

TSF_D double ld_real(const double* __restrict__ base, int n, int j) {
  return j < n ? base[j] : 0.0;
}
TSF_D void st_real(double* __restrict__ base, int n, int j, double v) {
  if (j < n) base[j] = v;
}

// elements (complex slots) per owning thread
constexpr int kE = TSF_KE;

template <int N>
struct FShape {
  // 8 slots: one transform needs ~93 registers; 16 slots (radix-16, three
  // passes at N = 4096) need ~166 and spill under the 128-register cap of
  // 512-thread CTAs (measured)
  static constexpr int E = kE;
  static constexpr int T = N / E;
};

// Shared-memory plan of the single-CTA kernels:
//   transform buffer(s) | real staging vector (N doubles) | twiddle table |
//   [symbol table mvS, N double2] | [instance Strang spectrum, N doubles]
// With TSF_STAGE_TABLES=1 the two tables are staged (cp.async at kernel
// start, landing while the first transform runs) when they fit without
// lowering the CTAs per SM.  Measured slower on configs[2] (35.1 / 36.5 ms
// per level vs 33.1 ms, ping-pong / in-place): the bigger carve-out costs the
// L1 the streaming vectors use, so it is off by default.
#ifndef TSF_STAGE_TABLES
#define TSF_STAGE_TABLES 0
#endif
constexpr int kSmemCap = 227 * 1024;       // dynamic shared memory per CTA
constexpr int kSmemPerSM = 228 * 1024;
template <int N>
struct FStage {
  static constexpr int FFT_BYTES =
      use64<N>() ? f64::kBytes : (kFftInPlace ? 1 : 2) * FftPlan<N, kE>::SMEM_ELEMS * 16;
  static constexpr int TW_BYTES = tw_table_elems(2 * N) * 16;
  static constexpr int PTW_BYTES = kPassTw        ? FftPlan<N, kE>::PTW_ELEMS * 16
                                   : kPassTwSmall ? FftPlan<N, kE>::PTWS_ELEMS * 16
                                                  : 0;
  static constexpr int BASE = FFT_BYTES + N * 8 + TW_BYTES + PTW_BYTES;
  static constexpr int BLOCK = (N / kE) < 32 ? 32 : (N / kE);
  static constexpr int REG_CTAS = (65536 / (BLOCK * 128)) < 1 ? 1 : 65536 / (BLOCK * 128);
  static constexpr int occ(int bytes) { return kSmemPerSM / (bytes + 1024 + 1024); }
  static constexpr int OCC0 = occ(BASE) < REG_CTAS ? occ(BASE) : REG_CTAS;
  static constexpr bool PS = TSF_STAGE_TABLES && BASE + N * 8 <= kSmemCap && occ(BASE + N * 8) >= OCC0;
  static constexpr bool MV = PS && BASE + N * 24 <= kSmemCap && occ(BASE + N * 24) >= OCC0;
  static constexpr int SMEM = BASE + (PS ? N * 8 : 0) + (MV ? N * 16 : 0);
};

// twiddle-table argument of the filters' transforms (tsf_fft.cuh SmallTw)
TSF_D auto xtw(const FilterTables& t) {
  if constexpr (kPassTwSmall) return SmallTw{t.ptw};
  else return t.ptw;
}

template <int N>
TSF_D double2 mv_spec(const FilterTables& t, int k) {
  if constexpr (FStage<N>::MV) return t.mvS[k];   // staged in shared memory
  else return ldt(&t.mvS[k]);
}

// The filters' transforms: the 64 x 64 engine (tsf_fft64.cuh) at N = 4096,
// the radix-8 Stockham engine (tsf_fft.cuh) otherwise.  Slot c of thread t
// holds index oidx<N>(t, c) in both domains.
template <int N, bool INV, class Hook = NoHook>
TSF_D void xfft(double2 (&v)[FShape<N>::E], double2* sm, const FilterTables& t,
                const Hook& hook = Hook{}) {
  if constexpr (use64<N>()) fft64<INV>(v, sm, hook);
  else block_fft<N, FShape<N>::E, INV>(v, sm, t.tw, 1, xtw(t), hook);
}
template <int N, class Hook = NoHook>
TSF_D void xfft_real(const double (&x)[FShape<N>::E], double2 (&v)[FShape<N>::E], double2* sm,
                     const FilterTables& t, const Hook& hook = Hook{}) {
  if constexpr (use64<N>()) fft64_real(x, v, sm, hook);
  else block_fft_real<N, FShape<N>::E>(x, v, sm, t.tw, 1, xtw(t), hook);
}

// even output bins: z <- IFFT_N( S_even . FFT_N(x) ) for real x; caller keeps Re(z)
template <int N, class Hook = NoHook>
TSF_D void filt_even(const double (&x)[FShape<N>::E], double2 (&z)[FShape<N>::E], double2* sm,
                     const FilterTables& t, const Hook& inv_hook = Hook{}) {
  constexpr int T = FShape<N>::T;
  constexpr int E = FShape<N>::E;
  const bool own = threadIdx.x < T;
  double se[E];
  xfft_real<N>(x, z, sm, t, [&] {
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) se[c] = mv_spec<N>(t, spos<N>(threadIdx.x, c)).x;
    }
  });
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = cscale(z[c], se[c]);
  }
  xfft<N, true>(z, sm, t, inv_hook);
}

// odd output bins: z (already modulated by w_j) <- IFFT_N( S_odd . FFT_N(z) );
// caller keeps Re(conj(w_j) z_j)
// inv_hook: the caller's loads for after the inverse transform (tsf_fft.cuh
// NoHook / hook_pass)
template <int N, class Hook = NoHook>
TSF_D void filt_odd(double2 (&z)[FShape<N>::E], double2* sm, const FilterTables& t,
                    const Hook& inv_hook = Hook{}) {
  constexpr int T = FShape<N>::T;
  constexpr int E = FShape<N>::E;
  const bool own = threadIdx.x < T;
  double so[E];
  xfft<N, false>(z, sm, t, [&] {
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) so[c] = mv_spec<N>(t, spos<N>(threadIdx.x, c)).y;
    }
  });
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = cscale(z[c], so[c]);
  }
  xfft<N, true>(z, sm, t, inv_hook);
}

// Strang: z <- IFFT_n( FFT_n(x) . Ssym / n ) for real x, n = N; caller keeps Re(z)
template <int N>
TSF_D void filt_strang(const double (&x)[FShape<N>::E], double2 (&z)[FShape<N>::E], double2* sm,
                       const FilterTables& t, double d, double kbar) {
  constexpr int T = FShape<N>::T;
  constexpr int E = FShape<N>::E;
  constexpr double inv_n = 1.0 / N;
  xfft_real<N>(x, z, sm, t);
  if (threadIdx.x < T) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const double2 lam = ldt(&t.pclam[spos<N>(threadIdx.x, c)]);
      const double s = 0.5 * (rcp_pos(d + kbar * lam.x) + rcp_pos(d + kbar * lam.y));
      z[c] = cscale(z[c], s * inv_n);
    }
  }
  xfft<N, true>(z, sm, t);
}

// Strang with a precomputed per-instance spectrum spec[k] = S_k / n (the level
// solve forms it once per level in k_solve_begin instead of two reciprocals
// per bin in every application).
//
// hs != null: also write the filtered spectrum's bins k <= N/2 to hs.  With
// x_hat = Re IFFT(z) the Strang output, FFT_N(x_hat) = N Herm(z) exactly (the
// real part of an inverse transform is the inverse transform of the
// spectrum's Hermitian part), so the next Toeplitz product of x_hat takes its
// even-bin channel from hs (filt_even_spec) instead of transforming x_hat
// again: 5 transforms per BiCGSTAB half-iteration instead of 6.  Checked on
// the CPU against the reference's iteration counts (tools/pair_probe.py
// family): no bias, unlike any pairing of two real vectors
// into one complex transform.
template <int N>
TSF_D void filt_strang_tab(const double (&x)[FShape<N>::E], double2 (&z)[FShape<N>::E], double2* sm,
                           const FilterTables& t, const double* __restrict__ spec,
                           double2* __restrict__ hs = nullptr) {
  constexpr int T = FShape<N>::T;
  constexpr int E = FShape<N>::E;
  double sp[E];
  const bool own = threadIdx.x < T;
  xfft_real<N>(x, z, sm, t, [&] {
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) sp[c] = spec[spos<N>(threadIdx.x, c)];
    }
  });
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k = oidx<N>(threadIdx.x, c);
      z[c] = cscale(z[c], sp[c]);
      if constexpr (use64<N>()) {
        if (hs) hs[spos<N>(threadIdx.x, c)] = z[c];   // full spectrum, stored permuted
      } else {
        if (hs && k <= N / 2) hs[k] = z[c];
      }
    }
  }
  xfft<N, true>(z, sm, t);
}

// even output bins of the Toeplitz product from a stored half spectrum:
// z <- IFFT_N( S_even . N Herm(hs) ); caller keeps Re(z).  Equals filt_even
// of x_hat = Re IFFT_N(hs) without its forward transform.
template <int N>
TSF_D void load_even_spec(const double2* hs, const FilterTables& t, double2 (&z)[FShape<N>::E]) {
  constexpr int T = FShape<N>::T;
  constexpr int E = FShape<N>::E;
  if (threadIdx.x < T) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k = oidx<N>(threadIdx.x, c);
      double2 h;
      if constexpr (use64<N>()) h = hs[spos<N>(threadIdx.x, c)];
      else h = k <= N / 2 ? hs[k] : cconj(hs[N - k]);
      z[c] = cscale(h, mv_spec<N>(t, spos<N>(threadIdx.x, c)).x * N);  // N S/L: exact (pow2 N)
    }
  }
}
template <int N, class Hook = NoHook>
TSF_D void filt_even_spec(const double2* hs, double2 (&z)[FShape<N>::E], double2* sm,
                          const FilterTables& t, const Hook& inv_hook = Hook{}) {
  load_even_spec<N>(hs, t, z);
  xfft<N, true>(z, sm, t, inv_hook);
}

// w_j = W_L^j for the owned slots
TSF_D double2 modulation(const FilterTables& t, int j) { return tw_get(t.tw, j); }

// Copy the two-level twiddle table of the length-L = 2N embedding into
// shared memory at `dst` (the first transform's leading barrier publishes
// it) and start the asynchronous copies of the staged tables (FStage; the
// transforms' inter-pass barriers wait for them, tsf_fft.cuh fft_rec).
// `ps_src`: the instance's Strang spectrum to stage, or null.
template <int N>
TSF_D FilterTables stage_tables(const FilterTables& g, double2* dst, const double* ps_src = nullptr) {
  constexpr int NT = tw_table_elems(2 * N);
  for (int i = threadIdx.x; i < NT; i += blockDim.x) dst[i] = ldt(&g.tw[i]);
  if constexpr (use64<N>()) {
    // the transform region starts FFT_BYTES + N doubles before dst (kernel
    // layout: transform | real staging vector | twiddle table | ...)
    stage_fft64_tables(reinterpret_cast<double2*>(reinterpret_cast<char*>(dst) -
                                                  FStage<N>::FFT_BYTES - N * 8));
  }
  FilterTables t = g;
  t.tw = dst;
  double2* next = dst + NT;
  if constexpr (kPassTwSmall) {
    constexpr int NP = FftPlan<N, kE>::PTWS_ELEMS;
    for (int i = threadIdx.x; i < NP; i += blockDim.x) next[i] = ldt(&g.ptw[i]);
    t.ptw = next;   // the plan always builds the table (tsf_abi.cu pass_twiddles)
    next += NP;
  }
  if constexpr (kPassTw) {
    constexpr int NP = FftPlan<N, kE>::PTW_ELEMS;
    if (g.ptw) {
      for (int i = threadIdx.x; i < NP; i += blockDim.x) cp_async16(&next[i], &g.ptw[i]);
      t.ptw = next;
    }
    next += NP;
  }
  if constexpr (FStage<N>::MV) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) cp_async16(&next[i], &g.mvS[i]);
    t.mvS = next;
    next += N;
  }
  if constexpr (FStage<N>::PS) {
    if (ps_src) {
      double* ps = reinterpret_cast<double*>(next);
      for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) cp_async16(&ps[i], &ps_src[i]);
      t.ps = ps;
    }
  }
  if constexpr (kAsyncStaging) cp_async_commit();
  return t;
}

}  // namespace tsf
