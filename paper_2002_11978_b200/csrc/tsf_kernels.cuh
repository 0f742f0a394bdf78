// Batched per-instance kernels (one CTA per problem instance, n <= N <= 8192).
//
//  k_toeplitz_apply : y = shift*x + kappa .* (A x)   (toeplitz.py:51-63 + scheme.py:129-130)
//  k_strang_apply   : z = P^{-1} v                    (toeplitz.py:131-136)
//  k_krylov_solve   : the whole level solve of scheme.py:120-143 — kappa
//                     (given or from separable modes), kappa_bar = mean(kappa),
//                     preconditioner positivity, then right-preconditioned
//                     BiCGSTAB (krylov.py:88-153) or PCG (krylov.py:43-85)
//                     with exactly the reference's control flow, all scalars
//                     and convergence tests on the device, one CTA per
//                     instance, no host round trip per iteration.
// Template parameter N = L/2 is the transform length (pow2 >= n).
//
// Register discipline: during a transform only its 16 complex slots are
// live; Krylov vectors live in the instance's L2-resident workspace between
// transforms (re-read where needed), so the kernel runs spill-free at two
// CTAs per SM for n = 4096.
#pragma once

#include "tsf_filters.cuh"
#include "tsf_soe.cuh"

namespace tsf {

constexpr int kMaxModes = 4;

struct KState;

struct KrylovArgs {
  int n;
  int B;
  const double* rhs;        // [B, n] (R0)
  double* x;                // [B, n] solution (written)
  // diffusivity: given [B, n] (kappa != nullptr), or evaluated from
  // separable modes kappa(x_i) = sum_q kmode_q[b][i] * kcoef[q] into kwork
  const double* kappa;
  const double* kmodes;     // mode q of instance b at kmodes + q*kq_stride + b*kb_stride
  long kq_stride;
  long kb_stride;           // 0 when modes are shared by every instance
  int nk;
  double kcoef[kMaxModes];
  double* kwork;            // [B, n]
  double shift;             // d_m = a_mm / Gamma(1-gamma)
  double kbar;              // > 0: preconditioner kappa_bar; else mean(kappa)
  double tol;
  int max_iters;
  double* r;                // workspaces [B, n]
  double* p;
  double* v;
  double* ph;
  double* s;
  double* sh;
  double* t;
  double* pspec;            // [B, vs] Strang spectrum S_k / n of the level (PC == 1)
  double2* hspec;           // [B, N/2+1] half spectrum of the last Strang output (BiCGSTAB,
                            // PC == 1; 64 x 64 engine: [B, N] full spectrum, permuted),
                            // or null: recompute the even channel's transform
  // Internal layout (tsf_fft64.cuh spos): the workspace vectors r, p, v, ph,
  // s, sh, t, kwork, pspec, r0w, xw have per-instance stride vs and hold
  // index oidx(t, c) at position spos(t, c); rhs, x and kappa are the
  // caller's [B, n] natural-order vectors.  For the Stockham engine vs = n,
  // spos == oidx, r0w == rhs and xw == x.
  int vs;
  // PC == 2 (non-power-of-two n): P^{-1} = circ(c), c = Re IFFT_n(1/total),
  // applied as the symmetric Toeplitz product with first column c: its
  // embedding spectrum (S_2k, S_2k+1)/L per instance (stride pcS_stride
  // double2; 0 = shared), natural bin order (Stockham layout)
  const double2* pcS;
  long pcS_stride;
  const double* r0w;        // r0 (= rhs) in the internal layout
  double* xw;               // the iterate x in the internal layout
  KState* kst;              // [B] per-instance Krylov scalars (phase kernels)
  SoeArgs soe;              // fused SOE epilogue of converged instances (march)
  int soe_epilogue;         // 1: run it
  int* active;              // device counter of unfinished instances
  int* h_active;            // pinned host mirror of *active (driver polling)
  int* iters;               // per-instance outputs
  double* relres;
  int* status;
  FilterTables tab;
  void* graphs;             // host: the plan's SolveGraphs cache (graph mode), kernels ignore it
};

template <int N>
struct KShape {
  static constexpr int E = FShape<N>::E;
  static constexpr int T = FShape<N>::T;         // owning threads
  static constexpr int BLOCK = T < 32 ? 32 : T;  // launched threads
  static constexpr int FFT_BYTES = FStage<N>::FFT_BYTES;
  static constexpr int TW_BYTES = FStage<N>::TW_BYTES;
  // transform buffer(s) | real staging vector | twiddle table | staged tables
  static constexpr int SMEM = FStage<N>::SMEM;
#ifdef TSF_MINB
  static constexpr int MIN_BLOCKS = TSF_MINB;
#else
  static constexpr int MIN_BLOCKS = BLOCK >= 512 ? 1 : 512 / BLOCK;  // <= 128 regs
#endif
};

// slot c of thread t: INT = internal workspace layout (position spos, per
// instance stride vs), else the caller's natural order; zero beyond n
template <int N, bool INT>
TSF_D double ldv(const double* __restrict__ base, int n, int t, int c) {
  const int j = oidx<N>(t, c);
  if constexpr (INT) return j < n ? base[spos<N>(t, c)] : 0.0;
  else return j < n ? base[j] : 0.0;
}
template <int N, bool INT>
TSF_D void stv(double* __restrict__ base, int n, int t, int c, double v) {
  const int j = oidx<N>(t, c);
  if (j < n) base[INT ? spos<N>(t, c) : j] = v;
}
// the level's diffusivity in the internal layout: the 64 x 64 engine copies a
// given kappa into kwork in k_solve_begin; the Stockham engine reads it in place
template <int N>
TSF_D const double* kap_ptr(const KrylovArgs& a) {
  if constexpr (use64<N>()) return a.kwork;
  else return a.kappa ? a.kappa : (const double*)a.kwork;
}

// y = shift*x + kappa .* (A x) on the owned slots (kappa == nullptr: y = A x).
// x is read from global (twice); result returned in y[].  hs: x's half
// spectrum from the Strang solve that produced x (filt_strang_tab), or null;
// hz: that spectrum already loaded into the owned slots (load_even_spec).
template <int N, bool INT = true>
TSF_D void apply_level_op(const double* __restrict__ xg, const double* __restrict__ kg,
                          double shift, int n, double (&y)[FShape<N>::E], double2* sm, double* aux,
                          const FilterTables& t, const double2* hs = nullptr,
                          const double2* hz = nullptr) {
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  const bool own = tid < T;
  constexpr int E = KShape<N>::E;
  double2 z[FShape<N>::E];
  // x for the odd channel's modulation and the epilogue: loaded during the
  // even channel's inverse transform (load hook, tsf_fft.cuh), kept in
  // registers; kappa loaded during the odd inverse transform
  double xo[E], ko[E];
  auto load_x = [&] {
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) xo[c] = ldv<N, INT>(xg, n, tid, c);
    }
  };
  auto load_k = [&] {
    if (own && kg) {
#pragma unroll
      for (int c = 0; c < E; ++c) ko[c] = ldv<N, INT>(kg, n, tid, c);
    }
  };
  if (hz) {
    // even-channel spectrum preloaded by the phase kernel (k_bicg_phase)
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = hz[c];
    xfft<N, true>(z, sm, t, load_x);
  } else if (hs) {
    filt_even_spec<N>(hs, z, sm, t, load_x);   // x = Re IFFT(hs): its spectrum is known
  } else {
    double xr[FShape<N>::E];
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) xr[c] = ldv<N, INT>(xg, n, tid, c);
    }
    filt_even<N>(xr, z, sm, t, load_x);
  }
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) aux[spos<N>(tid, c)] = z[c].x;
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = cscale(modulation(t, oidx<N>(tid, c)), xo[c]);
  }
  filt_odd<N>(z, sm, t, load_k);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const double2 w = modulation(t, oidx<N>(tid, c));
      const double ax = aux[spos<N>(tid, c)] + fma(z[c].x, w.x, z[c].y * w.y);  // + Re(conj(w) z)
      y[c] = kg ? fma(shift, xo[c], ko[c] * ax) : ax;
    }
  }
}

// --------------------------------------------------------------- matvec
template <int N>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_toeplitz_apply(int n, const double* __restrict__ x, double* __restrict__ y,
                 const double* __restrict__ kappa, double shift, FilterTables tab) {
  extern __shared__ double2 sm[];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  const FilterTables ts = stage_tables<N>(tab, reinterpret_cast<double2*>(aux + N));
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  double out[FShape<N>::E];
  apply_level_op<N, false>(x + off, kappa ? kappa + off : nullptr, shift, n, out, sm, aux, ts);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) st_real(y + off, n, oidx<N>(tid, c), out[c]);
  }
}

// --------------------------------------------------------------- precond
template <int N>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_strang_apply(int n, const double* __restrict__ v, double* __restrict__ zo, double shift,
               double kbar, const double* __restrict__ kbar_dev, FilterTables tab) {
  extern __shared__ double2 sm[];
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  const FilterTables ts = stage_tables<N>(tab, reinterpret_cast<double2*>(aux + N));
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  const double kb = kbar_dev ? kbar_dev[blockIdx.x] : kbar;
  double2 z[FShape<N>::E];
  double xr[FShape<N>::E];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) xr[c] = ld_real(v + off, n, oidx<N>(tid, c));
  }
  filt_strang<N>(xr, z, sm, ts, shift, kb);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) st_real(zo + off, n, oidx<N>(tid, c), z[c].x);
  }
}

// --------------------------------------------------------------- solver
// A level solve runs as straight-line PHASE kernels (one CTA per instance):
//   begin : kappa (+ positivity), kappa_bar, preconditioner check, x = 0,
//           ||r0||, p = r0, p_hat = P^{-1} p
//   v     : v = M p_hat, alpha, s = r - alpha v, ||s|| (early exit), s_hat
//   t     : t = M s_hat, omega, x/r update, ||r||, rho, beta, next p, p_hat
// (BiCGSTAB, krylov.py:88-153), or begin + one iteration kernel (PCG,
// krylov.py:43-85), launched repeatedly by the host driver until every
// instance has finished (converged instances' CTAs return at once).  Each
// kernel holds one matvec (two transform pairs) and at most one Strang
// transform pair with no loop around them: ptxas spilled KBs per thread for
// every single-kernel loop layout tried.  The per-instance
// Krylov scalars live in KState; CTA-local reductions give every dot
// product of an instance inside its own CTA.

template <int N>
TSF_D double2* hspec_of(const KrylovArgs& a, int b) {
  if constexpr (use64<N>()) return a.hspec ? a.hspec + (long)b * N : nullptr;
  else return a.hspec ? a.hspec + (long)b * (N / 2 + 1) : nullptr;
}

struct KState {
  double rho, rho_new, alpha, omega, nrm0, rnorm, snorm, kbar, rz;
  int it, done;
};

template <int N, bool INT = true>
TSF_D void load_owned(double (&u)[FShape<N>::E], const double* g, int n) {
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) u[c] = ldv<N, INT>(g, n, tid, c);
  }
}
template <int N, bool INT = true>
TSF_D void store_owned(double* g, const double (&u)[FShape<N>::E], int n) {
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) stv<N, INT>(g, n, tid, c, u[c]);
  }
}
// the caller's x (natural order) from the internal iterate, before an
// instance finishes (64 x 64 engine; with the Stockham engine xw IS x)
template <int N>
TSF_D void publish_x(const KrylovArgs& a, int b) {
  if constexpr (use64<N>()) {
    double u[FShape<N>::E];
    load_owned<N, true>(u, a.xw + (long)b * a.vs, a.n);
    store_owned<N, false>(a.x + (long)b * a.n, u, a.n);
  }
}
// dst = P^{-1} u (u real, owned slots); spec = the instance's S_k / n
template <int N>
TSF_D void precond_store(const double (&u)[FShape<N>::E], double* dst, int n, const double* spec,
                         double2* sm, const FilterTables& t, double2* hs = nullptr) {
  constexpr int T = KShape<N>::T;
  double2 z[FShape<N>::E];
  filt_strang_tab<N>(u, z, sm, t, t.ps ? t.ps : spec, hs);
  if (threadIdx.x < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) stv<N, true>(dst, n, threadIdx.x, c, z[c].x);
  }
}

// dst = circ(c) u for the non-power-of-two preconditioner (PC == 2): the
// Toeplitz product of the instance's circulant column through the same
// even/odd-bin filters as the operator (toeplitz.py:131-136 in exact
// arithmetic)
template <int N>
TSF_D void precond_toeplitz(const double (&u)[FShape<N>::E], double* dst, int n, double2* sm,
                            const FilterTables& tab, const double2* pcS) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  const int tid = threadIdx.x;
  const bool own = tid < T;
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  FilterTables t = tab;
  t.mvS = pcS;
  double2 z[FShape<N>::E];
  filt_even<N>(u, z, sm, t);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) aux[spos<N>(tid, c)] = z[c].x;
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = cscale(modulation(t, oidx<N>(tid, c)), u[c]);
  }
  filt_odd<N>(z, sm, t);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const double2 w = modulation(t, oidx<N>(tid, c));
      stv<N, true>(dst, n, tid, c, aux[spos<N>(tid, c)] + fma(z[c].x, w.x, z[c].y * w.y));
    }
  }
}

// dst = P^{-1} u: Strang (PC == 1) or circulant-as-Toeplitz (PC == 2)
template <int N, int PC>
TSF_D void precond_any(const double (&u)[FShape<N>::E], double* dst, const KrylovArgs& a, int b,
                       double2* sm, const FilterTables& tab, double2* hs = nullptr) {
  if constexpr (PC == 1)
    precond_store<N>(u, dst, a.n, a.pspec + (long)b * a.vs, sm, tab, hs);
  else
    precond_toeplitz<N>(u, dst, a.n, sm, tab, a.pcS + (long)b * a.pcS_stride);
}

TSF_D void finish_instance(const KrylovArgs& a, KState* st, int* active, int b, int it,
                           double rel, int status, double2* sm) {
  if (threadIdx.x == 0) {
    a.iters[b] = it;
    a.relres[b] = rel;
    a.status[b] = status;
    st[b].done = 1;
    atomicSub(active, 1);
  }
  if (status == TSF_OK && a.soe_epilogue) {
    __syncthreads();   // the instance's published x (every thread's slots)
    soe_instance_epilogue(a.soe, reinterpret_cast<double*>(sm), b);
  }
}

// ---- begin (both methods)
// Phase bodies are device functions (return true when the instance finished)
// shared by the phase kernels and the persistent per-instance kernel.
template <int N, int PC, bool CG>
TSF_D bool dev_begin(const KrylovArgs& a, const FilterTables& tab, KState* st, int* active, double2* sm,
                    double* red) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  const int tid = threadIdx.x;
  const bool own = tid < T;
  const int b = blockIdx.x;
  const int n = a.n;
  const long off = (long)b * n;       // caller vectors
  const long ow = (long)b * a.vs;     // workspace vectors
  // kappa on the grid (scheme.py:156-160,280) and kappa_bar (scheme.py:135)
  double ksum = 0.0, kmin = 1e308;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = oidx<N>(tid, c);
      if (j < n) {
        double k;
        if (a.kappa) {
          k = a.kappa[off + j];
          if constexpr (use64<N>()) a.kwork[ow + spos<N>(tid, c)] = k;
        } else {
          k = 0.0;
          for (int q = 0; q < a.nk; ++q) {
            const double mq = a.kmodes[q * a.kq_stride + (long)b * a.kb_stride + j];
            // no contraction: reproduce numpy's  acc + mode*coef  rounding
            k = __dadd_rn(k, __dmul_rn(mq, a.kcoef[q]));
          }
          a.kwork[(use64<N>() ? ow + spos<N>(tid, c) : off + j)] = k;
        }
        ksum += k;
        kmin = fmin(kmin, k);
      }
    }
  }
  kmin = block_min1(kmin, red);
  if (kmin <= 0.0) {
    finish_instance(a, st, active, b, 0, 0.0, TSF_KAPPA_NONPOS, sm);
    return true;
  }
  const double kmean = block_sum1(ksum, red) / n;
  const double kbar = a.kbar > 0.0 ? a.kbar : kmean;
  const double d = a.shift;
  if constexpr (PC == 1) {
    // total eigenvalues d + kbar*lam > 0  (toeplitz.py:122-124); the table
    // is stored in the internal order (every position is some k < n)
    double tmin = 1e308;
    for (int k = tid; k < n; k += blockDim.x) tmin = fmin(tmin, d + kbar * ldt(&tab.pclam[k]).x);
    tmin = block_min1(tmin, red);
    if (tmin <= 0.0) {
      finish_instance(a, st, active, b, 0, 0.0, TSF_PRECOND_NONPOS, sm);
      return true;
    }
    // the level's Strang filter (even part of 1/total, 1/n folded in), once
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) {
        const int q = spos<N>(tid, c);
        const double2 lam = ldt(&tab.pclam[q]);
        a.pspec[ow + q] = 0.5 * (1.0 / (d + kbar * lam.x) + 1.0 / (d + kbar * lam.y)) / n;
      }
    }
  }
  // r = r0 = rhs, x = 0  (krylov.py:107-113 / 64-69)
  double u[FShape<N>::E];
  load_owned<N, false>(u, a.rhs + off, n);
  double ss = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      stv<N, true>(a.xw + ow, n, tid, c, 0.0);
      if (oidx<N>(tid, c) < n) ss = fma(u[c], u[c], ss);
    }
  }
  ss = block_sum1(ss, red);
  if (sqrt(ss) == 0.0) {
    publish_x<N>(a, b);
    finish_instance(a, st, active, b, 0, 0.0, TSF_OK, sm);
    return true;
  }
  if constexpr (use64<N>()) store_owned<N>(const_cast<double*>(a.r0w) + ow, u, n);
  if (CG) store_owned<N>(a.r + ow, u, n);         // r = b
  store_owned<N>(a.p + ow, u, n);                 // BiCGSTAB: p = r (it 1); CG: p = z (PC=0)
  double rz = ss;
  if constexpr (PC >= 1) {
    // BiCGSTAB: p_hat = P^{-1} p ; CG: z = P^{-1} r written to p (p = z)
    precond_any<N, PC>(u, CG ? a.p + ow : a.ph + ow, a, b, sm, tab,
                       (CG || PC != 1) ? nullptr : hspec_of<N>(a, b));
    if (CG) {
      double part = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < E; ++c) {
          if (oidx<N>(tid, c) < n) part = fma(u[c], ldv<N, true>(a.p + ow, n, tid, c), part);
        }
      }
      rz = block_sum1(part, red);
    }
  }
  if (tid == 0) {
    KState s;
    s.rho = s.alpha = s.omega = 1.0;
    s.rho_new = ss;   // r0 . r with r = r0 (same reduction)
    s.nrm0 = s.rnorm = s.snorm = sqrt(ss);
    s.kbar = kbar;
    s.rz = rz;
    s.it = 1;
    s.done = 0;
    st[b] = s;
  }
  return false;
}

// ---- BiCGSTAB v-phase
template <int N, int PC>
TSF_D bool dev_bicg_v(const KrylovArgs& a, const FilterTables& tab, KState* st, int* active, double2* sm,
                    double* red, const KState* pre = nullptr, const double2* hz = nullptr) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  const int b = blockIdx.x;
  if (!pre) __syncthreads();  // previous phase's st[b] writes (thread 0) are visible
  const int tid = threadIdx.x;
  const bool own = tid < T;
  const int n = a.n;
  const long off = (long)b * n;       // caller vectors
  const long ow = (long)b * a.vs;     // workspace vectors
  const KState s = pre ? *pre : st[b];
  const double* phg = (PC ? a.ph : a.p) + ow;
  const double* kg = kap_ptr<N>(a) + ow;
  prefetch_l2(kg, a.vs);               // epilogue operands (x is loaded at once)
  prefetch_l2(a.r0w + ow, a.vs);
  if (s.it != 1) prefetch_l2(a.r + ow, a.vs);
  double u[FShape<N>::E];
  double2* hs = PC == 1 ? hspec_of<N>(a, b) : nullptr;
  apply_level_op<N>(phg, kg, a.shift, n, u, sm, aux, tab, hs, hz);   // u = v = M p_hat
  // epilogue operands loaded at once (one exposed latency, see the t-phase)
  const double* rc = (s.it == 1 ? a.r0w : a.r) + ow;
  double r0v[E], rv[E];
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      r0v[c] = ldv<N, true>(a.r0w + ow, n, tid, c);
      rv[c] = ldv<N, true>(rc, n, tid, c);
    }
  }
  store_owned<N>(a.v + ow, u, n);
  double part = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = oidx<N>(tid, c);
      if (j < n) part = fma(r0v[c], u[c], part);
    }
  }
  const double denom = block_sum1(part, red);
  if (denom == 0.0) {
    publish_x<N>(a, b);
    finish_instance(a, st, active, b, s.it, s.rnorm / s.nrm0, TSF_BD_R0V, sm);
    return true;
  }
  const double alpha = s.rho_new / denom;
  // s = r - alpha v
  part = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = oidx<N>(tid, c);
      u[c] = rv[c] - alpha * u[c];
      if (j < n) part = fma(u[c], u[c], part);
    }
  }
  const double snorm = sqrt(block_sum1(part, red));
  if (snorm / s.nrm0 < a.tol) {
    // x += alpha p_hat (early exit counts as a full iteration, krylov.py:135-137)
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c)
        stv<N, false>(a.x + off, n, tid, c,
                      ldv<N, true>(a.xw + ow, n, tid, c) + alpha * ldv<N, true>(phg, n, tid, c));
    }
    finish_instance(a, st, active, b, s.it, snorm / s.nrm0, TSF_OK, sm);
    return true;
  }
  store_owned<N>(a.s + ow, u, n);
  if constexpr (PC >= 1) precond_any<N, PC>(u, a.sh + ow, a, b, sm, tab, hs);
  if (tid == 0) {
    st[b].alpha = alpha;
    st[b].snorm = snorm;
  }
  return false;
}

// ---- BiCGSTAB t-phase (+ next p / p_hat)
template <int N, int PC>
TSF_D bool dev_bicg_t(const KrylovArgs& a, const FilterTables& tab, KState* st, int* active, double2* sm,
                    double* red, const KState* pre = nullptr, const double2* hz = nullptr) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  const int b = blockIdx.x;
  if (!pre) __syncthreads();  // previous phase's st[b] writes (thread 0) are visible
  const int tid = threadIdx.x;
  const bool own = tid < T;
  const int n = a.n;
  const long ow = (long)b * a.vs;     // workspace vectors
  const int vs = a.vs;
  const KState s = pre ? *pre : st[b];
  const double* shg = (PC ? a.sh : a.s) + ow;
  const double* kg = kap_ptr<N>(a) + ow;
  prefetch_l2(kg, vs);                 // epilogue operands (x is loaded at once)
  prefetch_l2(a.s + ow, vs);
  prefetch_l2(a.xw + ow, vs);
  if (PC) prefetch_l2(a.ph + ow, vs);
  prefetch_l2(a.r0w + ow, vs);
  prefetch_l2(a.p + ow, vs);
  prefetch_l2(a.v + ow, vs);
  double u[FShape<N>::E];
  double2* hs = PC == 1 ? hspec_of<N>(a, b) : nullptr;
  apply_level_op<N>(shg, kg, a.shift, n, u, sm, aux, tab, hs, hz);   // u = t = M s_hat
  // Every epilogue operand is loaded here at once, while the transform's
  // registers are dead: one exposed memory latency per phase instead of one
  // per reduction step (ncu: these loads were 40% of the t-phase's stalls).
  const double* phg = (PC ? a.ph : a.p) + ow;
  double sv[E], xv[E], pv[E], shv[E], r0v[E], qv[E], vv[E];
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      sv[c] = ldv<N, true>(a.s + ow, n, tid, c);
      xv[c] = ldv<N, true>(a.xw + ow, n, tid, c);
      pv[c] = ldv<N, true>(phg, n, tid, c);
      shv[c] = ldv<N, true>(shg, n, tid, c);
      r0v[c] = ldv<N, true>(a.r0w + ow, n, tid, c);
    }
  }
  Vals<2> red2;
  red2.v[0] = 0.0;
  red2.v[1] = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = oidx<N>(tid, c);
      if (j < n) {
        red2.v[0] = fma(u[c], u[c], red2.v[0]);
        red2.v[1] = fma(u[c], sv[c], red2.v[1]);
      }
    }
  }
  red2 = block_sum<2>(red2, red);
  if (red2.v[0] == 0.0) {
    publish_x<N>(a, b);
    finish_instance(a, st, active, b, s.it, s.snorm / s.nrm0, TSF_BD_OMEGA_DEN, sm);
    return true;
  }
  const double omega = red2.v[1] / red2.v[0];
  // x += alpha p_hat + omega s_hat ; r = s - omega t
  red2.v[0] = 0.0;
  red2.v[1] = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = oidx<N>(tid, c);
      stv<N, true>(a.xw + ow, n, tid, c, xv[c] + (s.alpha * pv[c] + omega * shv[c]));
      u[c] = sv[c] - omega * u[c];
      stv<N, true>(a.r + ow, n, tid, c, u[c]);
      if (j < n) {
        red2.v[0] = fma(u[c], u[c], red2.v[0]);
        red2.v[1] = fma(r0v[c], u[c], red2.v[1]);
      }
    }
    // operands of the next p (x, p_hat, s_hat are dead now): in flight
    // during the reduction
#pragma unroll
    for (int c = 0; c < E; ++c) {
      qv[c] = ldv<N, true>(a.p + ow, n, tid, c);
      vv[c] = ldv<N, true>(a.v + ow, n, tid, c);
    }
  }
  red2 = block_sum<2>(red2, red);
  const double rnorm = sqrt(red2.v[0]);
  const double rel = rnorm / s.nrm0;
  const double rho_new = red2.v[1];
  const int fin = rel < a.tol ? 1 : omega == 0.0 ? 2 : s.it >= a.max_iters ? 3
                  : rho_new == 0.0 ? 4 : 0;
  if (fin) {
    publish_x<N>(a, b);
    if (fin == 1) finish_instance(a, st, active, b, s.it, rel, TSF_OK, sm);
    else if (fin == 2) finish_instance(a, st, active, b, s.it, rel, TSF_BD_OMEGA, sm);
    else if (fin == 3) finish_instance(a, st, active, b, a.max_iters, rel, TSF_NOT_CONVERGED, sm);
    // rho vanished: the next iteration's first test (krylov.py:118-121)
    else finish_instance(a, st, active, b, s.it + 1, rel, TSF_BD_RHO, sm);
    return true;
  }
  // next p = r + beta (p - omega v)
  const double beta = (rho_new / s.rho_new) * (s.alpha / omega);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) u[c] = u[c] + beta * (qv[c] - omega * vv[c]);
  }
  store_owned<N>(a.p + ow, u, n);
  if constexpr (PC >= 1) precond_any<N, PC>(u, a.ph + ow, a, b, sm, tab, hs);
  if (tid == 0) {
    st[b].rho = s.rho_new;
    st[b].rho_new = rho_new;
    st[b].omega = omega;
    st[b].rnorm = rnorm;
    st[b].it = s.it + 1;
  }
  return false;
}

// ---- PCG iteration: q = M p, alpha, x, r, ||r||, z = P^{-1} r, beta, p
template <int N, int PC>
TSF_D bool dev_cg_iter(const KrylovArgs& a, const FilterTables& tab, KState* st, int* active, double2* sm,
                    double* red) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  const int b = blockIdx.x;
  __syncthreads();  // previous phase's st[b] writes (thread 0) are visible
  const int tid = threadIdx.x;
  const bool own = tid < T;
  const int n = a.n;
  const long ow = (long)b * a.vs;     // workspace vectors
  const KState s = st[b];
  const double* kg = kap_ptr<N>(a) + ow;
  double u[FShape<N>::E];
  apply_level_op<N>(a.p + ow, kg, a.shift, n, u, sm, aux, tab);  // u = q = M p
  double part = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      if (oidx<N>(tid, c) < n) part = fma(ldv<N, true>(a.p + ow, n, tid, c), u[c], part);
    }
  }
  const double curv = block_sum1(part, red);
  if (curv <= 0.0) {
    publish_x<N>(a, b);
    finish_instance(a, st, active, b, s.it, s.rnorm / s.nrm0, TSF_BD_CURVATURE, sm);
    return true;
  }
  const double al = s.rz / curv;
  part = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      stv<N, true>(a.xw + ow, n, tid, c,
                   ldv<N, true>(a.xw + ow, n, tid, c) + al * ldv<N, true>(a.p + ow, n, tid, c));
      u[c] = ldv<N, true>(a.r + ow, n, tid, c) - al * u[c];
      if (oidx<N>(tid, c) < n) part = fma(u[c], u[c], part);
    }
  }
  store_owned<N>(a.r + ow, u, n);
  const double rnorm = sqrt(block_sum1(part, red));
  const double rel = rnorm / s.nrm0;
  if (rel < a.tol) {
    publish_x<N>(a, b);
    finish_instance(a, st, active, b, s.it, rel, TSF_OK, sm);
    return true;
  }
  if (s.it >= a.max_iters) {
    publish_x<N>(a, b);
    finish_instance(a, st, active, b, a.max_iters, rel, TSF_NOT_CONVERGED, sm);
    return true;
  }
  // z = P^{-1} r (into s), rz_new = r.z, p = z + beta p
  const double* zg = (PC ? a.s : a.r) + ow;
  if constexpr (PC >= 1) precond_any<N, PC>(u, a.s + ow, a, b, sm, tab);
  __syncthreads();
  part = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      if (oidx<N>(tid, c) < n) part = fma(u[c], ldv<N, true>(zg, n, tid, c), part);
    }
  }
  const double rz_new = block_sum1(part, red);
  const double beta = rz_new / s.rz;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c)
      stv<N, true>(a.p + ow, n, tid, c,
                   ldv<N, true>(zg, n, tid, c) + beta * ldv<N, true>(a.p + ow, n, tid, c));
  }
  if (tid == 0) {
    st[b].rz = rz_new;
    st[b].rnorm = rnorm;
    st[b].it = s.it + 1;
  }
  return false;
}

template <int N, int PC, bool CG>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_solve_begin(KrylovArgs a, KState* st, int* active) {
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  const FilterTables tab = stage_tables<N>(a.tab, reinterpret_cast<double2*>(
      reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES + N * 8));
  dev_begin<N, PC, CG>(a, tab, st, active, sm, red);
}

#define TSF_PHASE_KERNEL(KNAME, DNAME)                                                  \
  template <int N, int PC>                                                             \
  __global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)           \
  KNAME(KrylovArgs a, KState* st, int* active) {                                       \
    extern __shared__ double2 sm[];                                                    \
    __shared__ double red[4 * 32];                                                     \
    if (st[blockIdx.x].done) return;                                                   \
    const FilterTables tab = stage_tables<N>(a.tab, reinterpret_cast<double2*>(        \
        reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES + N * 8),                   \
        PC == 1 ? a.pspec + (long)blockIdx.x * a.vs : nullptr);                              \
    DNAME<N, PC>(a, tab, st, active, sm, red);                                         \
  }
TSF_PHASE_KERNEL(k_cg_iter, dev_cg_iter)
#undef TSF_PHASE_KERNEL

// BiCGSTAB phase kernels.  Their entry loads are issued together — the
// instance's Krylov state, this thread's twiddle-table entries and (Strang
// preconditioner) the even-channel spectrum of the vector the phase
// multiplies — so a CTA waits for one memory latency at entry instead of
// three in a row (ncu: state check, table staging and spectrum loads each
// stalled every warp of the SM).
#ifndef TSF_ENTRY_PRELOAD
#define TSF_ENTRY_PRELOAD 0
#endif
template <int N, int PC, bool TPHASE>
TSF_D void bicg_phase(const KrylovArgs& a, KState* st, int* active) {
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  constexpr int E = KShape<N>::E;
  double2* tws = reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES +
                                            N * 8);
  if constexpr (!TSF_ENTRY_PRELOAD || kAsyncStaging || FStage<N>::MV || FStage<N>::PS) {
    // table-staging variants: the plain entry sequence
    if (st[blockIdx.x].done) return;
    const FilterTables tab = stage_tables<N>(a.tab, tws, PC == 1 ? a.pspec + (long)blockIdx.x * a.vs : nullptr);
    if constexpr (TPHASE) dev_bicg_t<N, PC>(a, tab, st, active, sm, red);
    else dev_bicg_v<N, PC>(a, tab, st, active, sm, red);
  } else {
    constexpr int NT = tw_table_elems(2 * N);
    constexpr int BL = KShape<N>::BLOCK;
    constexpr int KT = (NT + BL - 1) / BL;
    double2 twv[KT];
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      const int i = threadIdx.x + q * BL;
      if (i < NT) twv[q] = ldt(&a.tab.tw[i]);
    }
    const KState s = st[blockIdx.x];
    double2 hz[E];
    const bool pre_spec = PC == 1 && a.hspec;
    FilterTables tab = a.tab;
    if (pre_spec) load_even_spec<N>(hspec_of<N>(a, blockIdx.x), tab, hz);
    if (s.done) return;
#pragma unroll
    for (int q = 0; q < KT; ++q) {
      const int i = threadIdx.x + q * BL;
      if (i < NT) tws[i] = twv[q];
    }
    if constexpr (use64<N>()) stage_fft64_tables(sm);
    tab.tw = tws;   // published by the first transform's leading barrier
    if constexpr (TPHASE) dev_bicg_t<N, PC>(a, tab, st, active, sm, red, &s, pre_spec ? hz : nullptr);
    else dev_bicg_v<N, PC>(a, tab, st, active, sm, red, &s, pre_spec ? hz : nullptr);
  }
}
template <int N, int PC>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_bicg_v(KrylovArgs a, KState* st, int* active) {
  bicg_phase<N, PC, false>(a, st, active);
}
template <int N, int PC>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_bicg_t(KrylovArgs a, KState* st, int* active) {
  bicg_phase<N, PC, true>(a, st, active);
}

// Persistent per-instance solve: one CTA runs its instance from begin to
// convergence (vectors stay L2-resident, no host round trip, and the GPU
// back-fills SMs as instances finish — no tail of near-empty launches).
// (Measured slower than the graph-mode phase kernels even for one instance:
// configs[0] 0.396 vs 0.318 ms per level solve — the loop spills ~1.3 KB per
// thread at any register cap.)
template <int N, int PC, bool CG>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_krylov_persist(KrylovArgs a, KState* st, int* active) {
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  const FilterTables tab = stage_tables<N>(a.tab, reinterpret_cast<double2*>(
      reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES + N * 8));
  if (dev_begin<N, PC, CG>(a, tab, st, active, sm, red)) return;
  for (;;) {
    if constexpr (!CG) {
      if (dev_bicg_v<N, PC>(a, tab, st, active, sm, red)) return;
      if (dev_bicg_t<N, PC>(a, tab, st, active, sm, red)) return;
    } else {
      if (dev_cg_iter<N, PC>(a, tab, st, active, sm, red)) return;
    }
  }
}

static __global__ void k_set_int(int* p, int v) { *p = v; }

// Loop test of the graph-mode level solve: keep iterating while any
// instance is unfinished (conditional WHILE node, tsf_dispatch_impl.cuh).
static __global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* active) {
  cudaGraphSetConditional(h, *active > 0 ? 1u : 0u);
}

// --------------------------------------------------------------- debug FFT
template <int N, int E, bool INV>
__global__ void k_fft_debug(const double2* __restrict__ in, double2* __restrict__ out,
                            const double2* tw, int tw_log_scale) {
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;  // debug transform: E complex slots per thread
  const long off = (long)blockIdx.x * N;
  double2 v[E];
  if constexpr (use64<N>() && E == 8) {
    // the filters' 64 x 64 engine: natural order in and out via oidx
    stage_fft64_tables(sm);
#pragma unroll
    for (int c = 0; c < E; ++c) v[c] = in[off + oidx<N>(tid, c)];
    fft64<INV>(v, sm);
#pragma unroll
    for (int c = 0; c < E; ++c) out[off + oidx<N>(tid, c)] = v[c];
  } else {
    constexpr int T = N / E;
    double2* tws = sm + (kFftInPlace ? 1 : 2) * FftPlan<N, E>::SMEM_ELEMS;
    for (int i = tid; i < tw_table_elems(N); i += blockDim.x) tws[i] = ldt(&tw[i]);
    tw = tws;
    if (tid < T) {
#pragma unroll
      for (int c = 0; c < E; ++c) v[c] = in[off + tid + c * T];
    }
    block_fft<N, E, INV>(v, sm, tw, tw_log_scale);
    if (tid < T) {
#pragma unroll
      for (int c = 0; c < E; ++c) out[off + tid + c * T] = v[c];
    }
  }
}

}  // namespace tsf
