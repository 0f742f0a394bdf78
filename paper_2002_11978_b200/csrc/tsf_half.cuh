// Half-length transform engine of the Strang-preconditioned BiCGSTAB level
// solve (power-of-two n = N, 512 <= N <= 4096).
//
// Every transform of a level solve (scheme.py:120-143, krylov.py:88-153,
// toeplitz.py:51-63 and 131-136) acts on real data, or on the odd bins of a
// real sequence, so each runs as ONE complex transform of length H = N/2:
//
//  * Strang solve of a real vector u: z_m = u_{2m} + i u_{2m+1}, Z = FFT_H(z),
//    split step  P_k = E_k + W_N^k O_k,  E = (Z_k + conj Z_{H-k})/2,
//    O = -i (Z_k - conj Z_{H-k})/2  (k = 0..H; the thread owning bin k gets
//    Z_{H-k} through one shared-memory mirror exchange and forms both P_k and
//    conj(P_{H-k}) = E_k - W_N^k O_k), filter Q = P . S/n, inverse pre-step
//    Z'_k = (Q_k + conj Q_{H-k}) + i conj(W_N^k)(Q_k - conj Q_{H-k}),
//    IFFT_H(Z')_m = q_{2m} + i q_{2m+1}.
//  * Toeplitz product, even bins: spectrum N Herm(Q) of the Strang output is
//    already known (tsf_filters.cuh filt_strang_tab), so only the pre-step
//    and one inverse transform.
//  * Toeplitz product, odd bins: X_{4m+1} = FFT_H[ W_L^j (x_j - i x_{j+H}) ]_m
//    exactly (DIF step; the bins 4m+3 are the conjugate mirrors of a real
//    sequence), g = IFFT_H(S_{4m+1} X_{4m+1}),
//    y_j = 2 Re(conj(w_j) g_j),  y_{j+H} = -2 Im(conj(w_j) g_j).
//
// Five length-H transforms per BiCGSTAB half-iteration instead of five of
// length N: half the FP64 and shared-memory work, and a 256-thread CTA per
// instance at N = 4096, so two CTAs share an SM and overlap each other's
// barrier phases.  Parity: the odd-bin channel is the pruned complex
// transform (same rounding structure), the packed forward transform only
// feeds the preconditioner, and the packed inverse has the error of a complex
// inverse; tools/half_probe.py measures the reference's iteration counts
// under this arithmetic on the CPU (identical +-1 statistics to the
// full-length structure), DESIGN.md §3.8.
//
// Real-vector ownership: thread t owns the 16 reals (2m, 2m+1), m = t + c T,
// c < 8 (one 16-byte access per slot) for every elementwise step; the odd
// channel reads x at (m, m+H) and returns its result through the shared
// staging vector.
#pragma once

#include "tsf_kernels.cuh"

#ifndef TSF_HALF
#define TSF_HALF 1
#endif
// Two ncu-driven changes, measured and NOT adopted (configs[2]
// level solve, one box): an unpadded mirror-exchange buffer removes the
// kernel's only bank conflicts (2-way on the descending mirror reads, 2% of
// its wavefronts) but ran 17.25 -> 17.38 ms; loading 2 / 4 slots of the x
// update before their stores removes eight serialised memory latencies (11%
// of the t-phase's stall samples) but ran 17.36 / 18.00 ms — with two CTAs
// per SM the other CTA already fills those stalls, and the extra live
// registers cost more elsewhere.
#ifndef TSF_H_XB_PAD
#define TSF_H_XB_PAD 1      // 0: unpadded mirror exchange
#endif
#ifndef TSF_H_XUPD_CHUNK
#define TSF_H_XUPD_CHUNK 1  // slots of the x update loaded before their stores (1, 2, 4, 8)
#endif

namespace tsf {

template <int N>
struct HShape {
  static constexpr int H = N / 2;
  static constexpr int E = 8;
  static constexpr int T = H / E;
  static constexpr int BLOCK = T < 32 ? 32 : T;
  using PL = FftPlan<(H < 8 ? 8 : H), E>;
  static constexpr int FFT_BYTES = 2 * PL::SMEM_ELEMS * 16;
  static constexpr int TW_BYTES = tw_table_elems(2 * N) * 16;
  // transform buffers | real staging vector (N doubles) | twiddle table
  static constexpr int SMEM = FFT_BYTES + N * 8 + TW_BYTES;
  static constexpr int MIN_BLOCKS = BLOCK >= 512 ? 1 : 512 / BLOCK;  // <= 128 registers
};

template <int N>
constexpr bool half_ok() {
  return TSF_HALF && N >= 512 && !use64<N>() && !kFftInPlace && kE == 8 && !kAsyncStaging &&
         !kPassTw && !kPassTwSmall;
}

template <int N>
TSF_D const double2* stage_tw_half(const double2* g, double2* dst) {
  constexpr int NT = tw_table_elems(2 * N);
  for (int i = threadIdx.x; i < NT; i += blockDim.x) dst[i] = ldt(&g[i]);
  return dst;
}

template <int N>
TSF_D void ld2(double2 (&u)[8], const double* g) {
  const double2* g2 = reinterpret_cast<const double2*>(g);
#pragma unroll
  for (int c = 0; c < 8; ++c) u[c] = g2[threadIdx.x + c * HShape<N>::T];
}
template <int N>
TSF_D void st2(double* g, const double2 (&u)[8]) {
  double2* g2 = reinterpret_cast<double2*>(g);
#pragma unroll
  for (int c = 0; c < 8; ++c) g2[threadIdx.x + c * HShape<N>::T] = u[c];
}

template <int N, bool INV, class Hook = NoHook>
TSF_D void hfft(double2 (&z)[8], double2* sm, const double2* tw, const Hook& hook = Hook{}) {
  // W_H^e = W_L^{4e}: the staged table is the length-L one (tw_log_scale 2)
  block_fft<N / 2, 8, INV>(z, sm, tw, 2, static_cast<const double2*>(nullptr), hook);
}

// inverse pre-step of a Hermitian spectrum given as (Q_k, conj Q_{H-k}):
// the packed slot Z'_k whose inverse transform is (q_{2m}, q_{2m+1})
TSF_D double2 pack_inverse(double2 Q, double2 cQm, double2 w) {
  const double2 Ep = cadd(Q, cQm);
  const double2 Op = cmulc(csub(Q, cQm), w);   // (Q - conj Q_{H-k}) conj(W_N^k)
  return make_double2(Ep.x - Op.y, Ep.y + Op.x);
}

// z[c] = (u_{2m}, u_{2m+1}) in; (q_{2m}, q_{2m+1}) out, q = Re IFFT_N(FFT_N(u) . spec)
// with spec[k] = S_k / n for k <= H.  hs (may be null) receives Q_k, k <= H.
// spec(k) = S_k / n for k <= H (a callable; evaluated inside the forward
// transform's load hook); inv_hook runs inside the inverse transform.
template <int N, class Spec, class Hook = NoHook>
TSF_D void strang_half(double2 (&z)[8], double2* sm, const double2* tw, const Spec& spec,
                       double2* __restrict__ hs, const Hook& inv_hook = Hook{}) {
  constexpr int H = N / 2;
  constexpr int T = HShape<N>::T;
  using PL = typename HShape<N>::PL;
  const int tid = threadIdx.x;
  double sk[8], sr[8];
  hfft<N, false>(z, sm, tw, [&] {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int k = tid + c * T;
      sk[c] = 0.5 * spec(k);        // the split step's 1/2 folded in (exact)
      sr[c] = 0.5 * spec(H - k);
    }
  });
  // mirror exchange through the buffer the last pass did not read
  double2* xb = sm + ((PL::NPASS - 1) & 1) * PL::SMEM_ELEMS;
#pragma unroll
  for (int c = 0; c < 8; ++c) xb[TSF_H_XB_PAD ? PL::pad(tid + c * T) : tid + c * T] = z[c];
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int k = tid + c * T;
    const int km = (H - k) & (H - 1);
    const double2 zm = xb[TSF_H_XB_PAD ? PL::pad(km) : km];
    const double2 A = z[c];
    const double2 s = make_double2(A.x + zm.x, A.y - zm.y);   // A + conj(Zm)
    const double2 d = make_double2(A.x - zm.x, A.y + zm.y);   // A - conj(Zm)
    const double2 w = tw_get(tw, 2 * k);                      // W_N^k
    const double2 Tt = cmul(w, make_double2(d.y, -d.x));      // W_N^k (-i d)
    const double2 Q = cscale(cadd(s, Tt), sk[c]);
    const double2 cQm = cscale(csub(s, Tt), sr[c]);           // conj Q_{H-k}
    if (hs) {
      hs[k] = Q;
      if (k == 0) hs[H] = cconj(cQm);
    }
    z[c] = pack_inverse(Q, cQm, w);
  }
  hfft<N, true>(z, sm, tw, inv_hook);
}
// the level's tabulated Strang filter
struct SpecTable {
  const double* __restrict__ p;
  TSF_D double operator()(int k) const { return p[k]; }
};

// even bins of the Toeplitz product of x = Re IFFT_N(hs) from its stored half
// spectrum: z[c] = (ye_{2m}, ye_{2m+1}) on return
template <int N, class Hook = NoHook>
TSF_D void even_half(const double2* __restrict__ hs, const FilterTables& t, double2 (&z)[8],
                     double2* sm, const Hook& hook = Hook{}) {
  constexpr int H = N / 2;
  constexpr int T = HShape<N>::T;
  const int tid = threadIdx.x;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int k = tid + c * T;
    const double2 a = hs[k], bm = hs[H - k];
    const double fa = ldt(&t.mvS[k]).x * N, fb = ldt(&t.mvS[H - k]).x * N;  // N S_2k / L (exact)
    const double2 Q = cscale(a, fa);
    const double2 cQm = make_double2(bm.x * fb, -bm.y * fb);
    z[c] = pack_inverse(Q, cQm, tw_get(t.tw, 2 * k));
  }
  hfft<N, true>(z, sm, t.tw, hook);
}

// y = shift*x + kappa .* (A x), result in the (2m, 2m+1) ownership.  hs: the
// half spectrum of x when x is the last Strang output (even bins need no
// forward transform); null: the even bins through the packed forward
// transform of x (the standalone product, tsf_toeplitz_matvec).
template <int N, bool SPEC>
TSF_D void apply_level_op_half(const double* __restrict__ xg, const double* __restrict__ kg,
                               double shift, double2 (&y)[8], double2* sm, double* aux,
                               const FilterTables& t, const double2* __restrict__ hs) {
  constexpr int H = N / 2;
  constexpr int T = HShape<N>::T;
  const int tid = threadIdx.x;
  double2 z[8];
  double xa[8], xb[8];
  auto load_x = [&] {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      xa[c] = xg[tid + c * T];
      xb[c] = xg[tid + c * T + H];
    }
  };
  if constexpr (SPEC) {
    even_half<N>(hs, t, z, sm, load_x);
  } else {
    ld2<N>(z, xg);
    const double2* mvS = t.mvS;
    strang_half<N>(z, sm, t.tw, [mvS](int k) { return ldt(&mvS[k]).x; }, nullptr, load_x);
  }
  double2* aux2 = reinterpret_cast<double2*>(aux);
#pragma unroll
  for (int c = 0; c < 8; ++c) aux2[tid + c * T] = z[c];
  // odd bins: z_m = w_m (x_m - i x_{m+H})
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double2 w = tw_get(t.tw, tid + c * T);
    z[c] = make_double2(fma(w.x, xa[c], w.y * xb[c]), fma(w.y, xa[c], -(w.x * xb[c])));
  }
  double so[8];
  hfft<N, false>(z, sm, t.tw, [&] {
#pragma unroll
    for (int c = 0; c < 8; ++c) so[c] = 2.0 * ldt(&t.mvS[2 * (tid + c * T)]).y;   // 2 S_{4m+1} / L
  });
#pragma unroll
  for (int c = 0; c < 8; ++c) z[c] = cscale(z[c], so[c]);
  double2 x2[8], k2[8];
  hfft<N, true>(z, sm, t.tw, [&] {
    ld2<N>(x2, xg);
    if (kg) ld2<N>(k2, kg);
  });
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int m = tid + c * T;
    const double2 w = tw_get(t.tw, m);
    aux[m] += fma(w.x, z[c].x, w.y * z[c].y);          //  Re(conj(w) g)
    aux[m + H] -= fma(w.x, z[c].y, -(w.y * z[c].x));   // -Im(conj(w) g)
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double2 ax = aux2[tid + c * T];
    y[c] = kg ? make_double2(fma(shift, x2[c].x, k2[c].x * ax.x), fma(shift, x2[c].y, k2[c].y * ax.y))
              : ax;
  }
}

// Where an instance's vectors live: the plan's global workspaces (phase
// kernels) or the CTA's shared memory (persistent kernel: as many as fit,
// hottest first) — generic pointers either way.  xg: the caller's solution
// vector, written when the instance finishes if x lives on chip (x != xg).
struct HVec {
  double* ph;
  double* sh;
  double2* hs;
  double* s;
  double* v;
  double* p;
  double* r;
  const double* r0;
  double* x;
  double* xg;
  const double* kap;
  double* pspec;
  bool onchip;      // every vector above the solve reads is in shared memory: no L2 prefetch
  bool kap_copy;    // kap points at a shared-memory copy begin has to fill
  bool r0_copy;     // likewise r0
};
template <int N>
TSF_D HVec hvec_global(const KrylovArgs& a) {
  const int b = blockIdx.x;
  const long ow = (long)b * N;
  HVec h;
  h.ph = a.ph + ow;
  h.sh = a.sh + ow;
  h.hs = a.hspec + (long)b * (N / 2 + 1);
  h.s = a.s + ow;
  h.v = a.v + ow;
  h.p = a.p + ow;
  h.r = a.r + ow;
  h.r0 = a.r0w + ow;
  h.x = a.xw + ow;
  h.xg = a.x + ow;
  h.kap = (a.kappa ? a.kappa : (const double*)a.kwork) + ow;
  h.pspec = a.pspec + ow;
  h.onchip = false;
  h.kap_copy = false;
  h.r0_copy = false;
  return h;
}
// the caller's x from the on-chip iterate, before an instance finishes
template <int N>
TSF_D void publish_x_h(const HVec& hv) {
  if (hv.x != hv.xg) {
    double2 t[8];
    ld2<N>(t, hv.x);
    st2<N>(hv.xg, t);
  }
}

// Every multiply-add of the phase bodies below is written out (fma /
// __dmul_rn / __dadd_rn): the phase kernels and the persistent kernel inline
// the same bodies in different contexts, and implicit contraction choices
// that differ between them would make an instance's result depend on the
// batch it is solved in (tests/test_gpu_half.py checks bit-identity).
// ---- begin: kappa, kappa_bar, checks, Strang filter of the level, r0, p_hat
// (returns true when the instance finished; tw: the staged twiddle table,
// published by this function's first block reduction)
template <int N>
TSF_D bool dev_begin_h(const KrylovArgs& a, KState* st, int* active, double2* sm, double* red,
                       const double2* tw, const HVec hv) {
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const long ow = (long)b * N;
  double ksum = 0.0, kmin = 1e308;
  {
    // every slot's modes before the first store (aliasing, as above)
    double2 kk[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) kk[c] = make_double2(0.0, 0.0);
    if (a.kappa) {
      ld2<N>(kk, a.kappa + ow);
    } else {
      for (int q = 0; q < a.nk; ++q) {
        double2 mq[8];
        ld2<N>(mq, a.kmodes + q * a.kq_stride + (long)b * a.kb_stride);
        const double cq = a.kcoef[q];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          // no contraction: reproduce numpy's  acc + mode*coef  rounding
          kk[c].x = __dadd_rn(kk[c].x, __dmul_rn(mq[c].x, cq));
          kk[c].y = __dadd_rn(kk[c].y, __dmul_rn(mq[c].y, cq));
        }
      }
      st2<N>(a.kwork + ow, kk);
    }
    if (hv.kap_copy) st2<N>(const_cast<double*>(hv.kap), kk);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      ksum += kk[c].x;
      ksum += kk[c].y;
      kmin = fmin(kmin, fmin(kk[c].x, kk[c].y));
    }
  }
  kmin = block_min1(kmin, red);
  if (kmin <= 0.0) {
    finish_instance(a, st, active, b, 0, 0.0, TSF_KAPPA_NONPOS, sm);
    return true;
  }
  const double kmean = block_sum1(ksum, red) / N;
  const double kbar = a.kbar > 0.0 ? a.kbar : kmean;
  const double d = a.shift;
  double tmin = 1e308;
  for (int k = tid; k < N; k += blockDim.x) tmin = fmin(tmin, fma(kbar, ldt(&a.tab.pclam[k]).x, d));
  tmin = block_min1(tmin, red);
  if (tmin <= 0.0) {
    finish_instance(a, st, active, b, 0, 0.0, TSF_PRECOND_NONPOS, sm);
    return true;
  }
  // the level's Strang filter (even part of 1/total, 1/n folded in), k < n
  for (int k = tid; k < N; k += blockDim.x) {
    const double2 lam = ldt(&a.tab.pclam[k]);
    hv.pspec[k] = 0.5 * (1.0 / fma(kbar, lam.x, d) + 1.0 / fma(kbar, lam.y, d)) / N;
  }
  double2 u[8];
  ld2<N>(u, a.rhs + ow);
  double ss = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    ss = fma(u[c].x, u[c].x, ss);
    ss = fma(u[c].y, u[c].y, ss);
  }
  ss = block_sum1(ss, red);   // (its barriers publish pspec and the twiddle table)
  {
    double2 zero[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) zero[c] = make_double2(0.0, 0.0);
    st2<N>(hv.x, zero);
    if (hv.x != hv.xg) st2<N>(hv.xg, zero);
  }
  if (hv.r0_copy) st2<N>(const_cast<double*>(hv.r0), u);
  if (sqrt(ss) == 0.0) {
    finish_instance(a, st, active, b, 0, 0.0, TSF_OK, sm);
    return true;
  }
  st2<N>(hv.p, u);
  strang_half<N>(u, sm, tw, SpecTable{hv.pspec}, hv.hs);
  st2<N>(hv.ph, u);
  if (tid == 0) {
    KState s;
    s.rho = s.alpha = s.omega = 1.0;
    s.rho_new = ss;
    s.nrm0 = s.rnorm = s.snorm = sqrt(ss);
    s.kbar = kbar;
    s.rz = ss;
    s.it = 1;
    s.done = 0;
    st[b] = s;
  }
  return false;
}

template <int N>
__global__ void __launch_bounds__(HShape<N>::BLOCK, HShape<N>::MIN_BLOCKS)
k_solve_begin_h(KrylovArgs a, KState* st, int* active) {
  using S = HShape<N>;
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::FFT_BYTES);
  const double2* tw = stage_tw_half<N>(a.tab.tw, reinterpret_cast<double2*>(aux + N));
  dev_begin_h<N>(a, st, active, sm, red, tw, hvec_global<N>(a));
}

// ---- v-phase: v = M p_hat, alpha, s = r - alpha v, ||s|| (early exit), s_hat
// (returns true when the instance finished)
template <int N>
TSF_D bool dev_bicg_v_h(const KrylovArgs& a, KState* st, int* active, double2* sm, double* red,
                        double* aux, const FilterTables& tab, const HVec hv) {
  const int b = blockIdx.x;
  const KState s = st[b];
  const int tid = threadIdx.x;
  const long ow = (long)b * N;
  const double* phg = hv.ph;
  const double* kg = hv.kap;
  double2* hs = hv.hs;
  if (!hv.onchip) {
    prefetch_l2(kg, N);
    prefetch_l2(hv.r0, N);
    if (s.it != 1) prefetch_l2(hv.r, N);
  }
  double2 u[8];
  apply_level_op_half<N, true>(phg, kg, a.shift, u, sm, aux, tab, hs);   // u = v = M p_hat
  const double* rc = s.it == 1 ? hv.r0 : (const double*)hv.r;
  double2 r0v[8], rv[8];
  ld2<N>(r0v, hv.r0);
  ld2<N>(rv, rc);
  st2<N>(hv.v, u);
  double part = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    part = fma(r0v[c].x, u[c].x, part);
    part = fma(r0v[c].y, u[c].y, part);
  }
  const double denom = block_sum1(part, red);
  if (denom == 0.0) {
    publish_x_h<N>(hv);
    finish_instance(a, st, active, b, s.it, s.rnorm / s.nrm0, TSF_BD_R0V, sm);
    return true;
  }
  const double alpha = s.rho_new / denom;
  part = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    u[c].x = fma(-alpha, u[c].x, rv[c].x);
    u[c].y = fma(-alpha, u[c].y, rv[c].y);
    part = fma(u[c].x, u[c].x, part);
    part = fma(u[c].y, u[c].y, part);
  }
  const double snorm = sqrt(block_sum1(part, red));
  if (snorm / s.nrm0 < a.tol) {
    // x += alpha p_hat (early exit counts as a full iteration, krylov.py:135-137)
    double2 xv[8], pv[8];
    ld2<N>(xv, hv.x);
    ld2<N>(pv, phg);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      xv[c].x = fma(alpha, pv[c].x, xv[c].x);
      xv[c].y = fma(alpha, pv[c].y, xv[c].y);
    }
    st2<N>(hv.xg, xv);
    finish_instance(a, st, active, b, s.it, snorm / s.nrm0, TSF_OK, sm);
    return true;
  }
  st2<N>(hv.s, u);
  strang_half<N>(u, sm, tab.tw, SpecTable{hv.pspec}, hs);
  st2<N>(hv.sh, u);
  if (tid == 0) {
    st[b].alpha = alpha;
    st[b].snorm = snorm;
  }
  return false;
}

// ---- t-phase: t = M s_hat, omega, x/r update, ||r||, rho, beta, next p, p_hat
// SMV: p_hat / s_hat live in shared memory (persistent kernel): no global prefetch of them
template <int N, bool SMV = false>
TSF_D bool dev_bicg_t_h(const KrylovArgs& a, KState* st, int* active, double2* sm, double* red,
                        double* aux, const FilterTables& tab, const HVec hv) {
  using S = HShape<N>;
  const int b = blockIdx.x;
  const KState s = st[b];
  const int tid = threadIdx.x;
  const long ow = (long)b * N;
  const double* shg = hv.sh;
  const double* kg = hv.kap;
  double2* hs = hv.hs;
  if (!hv.onchip) {
    prefetch_l2(kg, N);
    prefetch_l2(hv.s, N);
    prefetch_l2(hv.x, N);
    if (!SMV) prefetch_l2(hv.ph, N);
    prefetch_l2(hv.r0, N);
    prefetch_l2(hv.p, N);
    prefetch_l2(hv.v, N);
  }
  double2 u[8];
  apply_level_op_half<N, true>(shg, kg, a.shift, u, sm, aux, tab, hs);   // u = t = M s_hat
  double2 sv[8];
  ld2<N>(sv, hv.s);
  Vals<2> red2;
  red2.v[0] = 0.0;
  red2.v[1] = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    red2.v[0] = fma(u[c].x, u[c].x, red2.v[0]);
    red2.v[0] = fma(u[c].y, u[c].y, red2.v[0]);
    red2.v[1] = fma(u[c].x, sv[c].x, red2.v[1]);
    red2.v[1] = fma(u[c].y, sv[c].y, red2.v[1]);
  }
  red2 = block_sum<2>(red2, red);
  if (red2.v[0] == 0.0) {
    publish_x_h<N>(hv);
    finish_instance(a, st, active, b, s.it, s.snorm / s.nrm0, TSF_BD_OMEGA_DEN, sm);
    return true;
  }
  const double omega = red2.v[1] / red2.v[0];
  // x += alpha p_hat + omega s_hat
  {
    const double2* x2 = reinterpret_cast<const double2*>(hv.x);
    const double2* p2 = reinterpret_cast<const double2*>(hv.ph);
    const double2* h2 = reinterpret_cast<const double2*>(shg);
    double2* xo = reinterpret_cast<double2*>(hv.x);
    // XC slots' operands before their stores (TSF_H_XUPD_CHUNK above)
#pragma unroll
    constexpr int XC = TSF_H_XUPD_CHUNK;
#pragma unroll
    for (int c0 = 0; c0 < 8; c0 += XC) {
      double2 xv[XC], pv[XC], hv[XC];
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        const int m = tid + (c0 + q) * S::T;
        xv[q] = x2[m];
        pv[q] = p2[m];
        hv[q] = h2[m];
      }
#pragma unroll
      for (int q = 0; q < XC; ++q) {
        const int m = tid + (c0 + q) * S::T;
        xo[m] = make_double2(
            __dadd_rn(xv[q].x, fma(s.alpha, pv[q].x, __dmul_rn(omega, hv[q].x))),
            __dadd_rn(xv[q].y, fma(s.alpha, pv[q].y, __dmul_rn(omega, hv[q].y))));
      }
    }
  }
  // r = s - omega t
  double2 r0v[8];
  ld2<N>(r0v, hv.r0);
  red2.v[0] = 0.0;
  red2.v[1] = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    u[c].x = fma(-omega, u[c].x, sv[c].x);
    u[c].y = fma(-omega, u[c].y, sv[c].y);
    red2.v[0] = fma(u[c].x, u[c].x, red2.v[0]);
    red2.v[0] = fma(u[c].y, u[c].y, red2.v[0]);
    red2.v[1] = fma(r0v[c].x, u[c].x, red2.v[1]);
    red2.v[1] = fma(r0v[c].y, u[c].y, red2.v[1]);
  }
  st2<N>(hv.r, u);
  // operands of the next p: in flight during the reduction
  double2 qv[8], vv[8];
  ld2<N>(qv, hv.p);
  ld2<N>(vv, hv.v);
  red2 = block_sum<2>(red2, red);
  const double rnorm = sqrt(red2.v[0]);
  const double rel = rnorm / s.nrm0;
  const double rho_new = red2.v[1];
  const int fin = rel < a.tol ? 1 : omega == 0.0 ? 2 : s.it >= a.max_iters ? 3
                  : rho_new == 0.0 ? 4 : 0;
  if (fin) {
    if (hv.x != hv.xg) {
      __syncthreads();   // every thread's slots of the on-chip x
      publish_x_h<N>(hv);
    }
    if (fin == 1) finish_instance(a, st, active, b, s.it, rel, TSF_OK, sm);
    else if (fin == 2) finish_instance(a, st, active, b, s.it, rel, TSF_BD_OMEGA, sm);
    else if (fin == 3) finish_instance(a, st, active, b, a.max_iters, rel, TSF_NOT_CONVERGED, sm);
    else finish_instance(a, st, active, b, s.it + 1, rel, TSF_BD_RHO, sm);
    return true;
  }
  // next p = r + beta (p - omega v)
  const double beta = (rho_new / s.rho_new) * (s.alpha / omega);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    u[c].x = fma(beta, fma(-omega, vv[c].x, qv[c].x), u[c].x);
    u[c].y = fma(beta, fma(-omega, vv[c].y, qv[c].y), u[c].y);
  }
  st2<N>(hv.p, u);
  strang_half<N>(u, sm, tab.tw, SpecTable{hv.pspec}, hs);
  st2<N>(hv.ph, u);
  if (tid == 0) {
    st[b].rho = s.rho_new;
    st[b].rho_new = rho_new;
    st[b].omega = omega;
    st[b].rnorm = rnorm;
    st[b].it = s.it + 1;
  }
  return false;
}

// phase kernels, and both phases of an iteration in one kernel (TSF_FUSE_VT)
template <int N, int PHASES>
__global__ void __launch_bounds__(HShape<N>::BLOCK, HShape<N>::MIN_BLOCKS)
k_bicg_h(KrylovArgs a, KState* st, int* active) {
  using S = HShape<N>;
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  if (st[blockIdx.x].done) return;
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::FFT_BYTES);
  FilterTables tab = a.tab;
  tab.tw = stage_tw_half<N>(a.tab.tw, reinterpret_cast<double2*>(aux + N));
  __syncthreads();   // twiddle table staged
  const HVec hv = hvec_global<N>(a);
  if constexpr (PHASES & 1) {
    if (dev_bicg_v_h<N>(a, st, active, sm, red, aux, tab, hv)) return;
  }
  if constexpr (PHASES == 3) __syncthreads();   // st[b] (alpha, ||s||), s_hat and its spectrum
  if constexpr (PHASES & 2) dev_bicg_t_h<N>(a, st, active, sm, red, aux, tab, hv);
}

// Whole level solve of one instance in ONE kernel (batches of at most one CTA
// per SM: configs[0], single mid-size instances): the same phase bodies in a
// loop, so the result is bit-identical to the phase kernels', without the
// 3 graph nodes per iteration and the per-phase table staging.  One CTA per
// SM lifts the register cap (launch bound 1: up to 255 registers), which is
// what the full-length engine's persistent kernel lacked (it spilled 1.3 KB
// per thread under the 128-register cap of 512-thread CTAs).
// Its CTA is alone on the SM, so the shared memory the second CTA would use
// holds the instance's hottest vectors instead: p_hat, s_hat (three reads and
// a write per iteration each) and the stored half spectrum (generic
// addressing: the phase bodies see ordinary pointers).
template <int N>
struct HPersist {
  static constexpr int VEC_OFF = HShape<N>::SMEM;
#ifndef TSF_PERSIST_SMV
#define TSF_PERSIST_SMV 1
#endif
  // shared-memory residents in order of traffic per iteration: p_hat, s_hat,
  // half spectrum (NV >= 3: n = 4096), then s, v, p, r, x, r0, kappa (NV = 10:
  // n <= 2048) and the Strang filter (NV = 11: n <= 1024)
  static constexpr int HS_BYTES = (N / 2 + 2) * 16;
  static constexpr int bytes(int nv) { return VEC_OFF + (nv >= 3 ? HS_BYTES + (nv - 1) * N * 8 : nv * N * 8); }
  static constexpr int NV = !TSF_PERSIST_SMV            ? 0
                            : bytes(11) <= kSmemCap     ? 11
                            : bytes(10) <= kSmemCap     ? 10
                            : bytes(3) <= kSmemCap      ? 3
                                                        : 0;
  static constexpr int BYTES = bytes(NV);
};
// FULL: every vector that fits on chip (small batches: one CTA per SM anyway);
// otherwise only p_hat / s_hat / spectrum, so that several CTAs of a small
// grid size still share an SM.  Same arithmetic either way.
template <int N, int MB, bool FULL>
__global__ void __launch_bounds__(HShape<N>::BLOCK, MB)
k_krylov_persist_h(KrylovArgs a, KState* st, int* active) {
  using S = HShape<N>;
  constexpr int NV = MB != 1 ? 0 : FULL ? HPersist<N>::NV : (HPersist<N>::NV >= 3 ? 3 : 0);
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::FFT_BYTES);
  FilterTables tab = a.tab;
  tab.tw = stage_tw_half<N>(a.tab.tw, reinterpret_cast<double2*>(aux + N));
  HVec hv = hvec_global<N>(a);
  if constexpr (NV >= 3) {
    double* vec = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + HPersist<N>::VEC_OFF);
    hv.ph = vec;
    hv.sh = vec + N;
    hv.hs = reinterpret_cast<double2*>(vec + 2 * N);
    if constexpr (NV >= 10) {
      double* w = vec + 2 * N + HPersist<N>::HS_BYTES / 8;
      hv.s = w;
      hv.v = w + N;
      hv.p = w + 2 * N;
      hv.r = w + 3 * N;
      hv.x = w + 4 * N;
      hv.r0 = w + 5 * N;
      hv.r0_copy = true;
      hv.kap = w + 6 * N;
      hv.kap_copy = true;
      hv.onchip = true;
      if constexpr (NV >= 11) hv.pspec = w + 7 * N;
    }
  }
  if (dev_begin_h<N>(a, st, active, sm, red, tab.tw, hv)) return;
  for (;;) {
    __syncthreads();   // st[b] and the previous phase's vectors (other threads' slots)
    if (dev_bicg_v_h<N>(a, st, active, sm, red, aux, tab, hv)) return;
    __syncthreads();
    if (dev_bicg_t_h<N, (NV >= 3)>(a, st, active, sm, red, aux, tab, hv)) return;
  }
}

// ---- debug: the two building blocks alone (tests/test_gpu_half.py)
//  mode 0: out = P^{-1} x with spec = S_k / n [B][N] given, hs <- half spectrum
//  mode 1: out = shift*x + kappa .* (A x), x = Re IFFT_N(hs)
template <int N>
__global__ void __launch_bounds__(HShape<N>::BLOCK, HShape<N>::MIN_BLOCKS)
k_half_debug(int mode, const double* __restrict__ x, const double* __restrict__ aux_in,
             double shift, double2* hs, double* __restrict__ out, FilterTables tabg) {
  using S = HShape<N>;
  extern __shared__ double2 sm[];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::FFT_BYTES);
  FilterTables tab = tabg;
  tab.tw = stage_tw_half<N>(tabg.tw, reinterpret_cast<double2*>(aux + N));
  __syncthreads();
  const long ow = (long)blockIdx.x * N;
  double2* hsb = hs + (long)blockIdx.x * (N / 2 + 1);
  double2 u[8];
  if (mode == 0) {
    ld2<N>(u, x + ow);
    strang_half<N>(u, sm, tab.tw, SpecTable{aux_in + ow}, hsb);
  } else {
    apply_level_op_half<N, true>(x + ow, aux_in + ow, shift, u, sm, aux, tab, hsb);
  }
  st2<N>(out + ow, u);
}

// ---- standalone operators (tsf_toeplitz_matvec / tsf_precond_solve, power-of-two n = N)
template <int N>
__global__ void __launch_bounds__(HShape<N>::BLOCK, HShape<N>::MIN_BLOCKS)
k_toeplitz_apply_h(const double* __restrict__ x, double* __restrict__ y,
                   const double* __restrict__ kappa, double shift, FilterTables tabg) {
  using S = HShape<N>;
  extern __shared__ double2 sm[];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::FFT_BYTES);
  FilterTables tab = tabg;
  tab.tw = stage_tw_half<N>(tabg.tw, reinterpret_cast<double2*>(aux + N));
  __syncthreads();
  const long ow = (long)blockIdx.x * N;
  double2 u[8];
  apply_level_op_half<N, false>(x + ow, kappa ? kappa + ow : nullptr, shift, u, sm, aux, tab, nullptr);
  st2<N>(y + ow, u);
}

template <int N>
__global__ void __launch_bounds__(HShape<N>::BLOCK, HShape<N>::MIN_BLOCKS)
k_strang_apply_h(const double* __restrict__ v, double* __restrict__ zo, double shift, double kbar,
                 const double* __restrict__ kbar_dev, FilterTables tabg) {
  using S = HShape<N>;
  extern __shared__ double2 sm[];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::FFT_BYTES);
  const double2* tw = stage_tw_half<N>(tabg.tw, reinterpret_cast<double2*>(aux + N));
  __syncthreads();
  const long ow = (long)blockIdx.x * N;
  const double kb = kbar_dev ? kbar_dev[blockIdx.x] : kbar;
  const double2* pclam = tabg.pclam;
  double2 u[8];
  ld2<N>(u, v + ow);
  strang_half<N>(u, sm, tw, [=](int k) {
    const double2 lam = ldt(&pclam[k & (N - 1)]);
    return 0.5 * (rcp_pos(shift + kb * lam.x) + rcp_pos(shift + kb * lam.y)) * (1.0 / N);
  }, nullptr);
  st2<N>(zo + ow, u);
}

}  // namespace tsf
