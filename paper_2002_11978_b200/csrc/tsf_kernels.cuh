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

namespace tsf {

constexpr int kMaxModes = 4;

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
  int* iters;               // per-instance outputs
  double* relres;
  int* status;
  FilterTables tab;
};

template <int N>
struct KShape {
  static constexpr int E = FShape<N>::E;
  static constexpr int T = FShape<N>::T;         // owning threads
  static constexpr int BLOCK = T < 32 ? 32 : T;  // launched threads
  static constexpr int FFT_BYTES = FftPlan<N, E>::SMEM_ELEMS * 16;
  static constexpr int SMEM = FFT_BYTES + N * 8;  // + one real staging vector
  static constexpr int MIN_BLOCKS = BLOCK >= 512 ? 1 : 512 / BLOCK;  // <= 128 regs
};

// y = shift*x + kappa .* (A x) on the owned slots (kappa == nullptr: y = A x).
// x is read from global (twice); result returned in y[].
template <int N>
TSF_D void apply_level_op(const double* __restrict__ xg, const double* __restrict__ kg,
                          double shift, int n, double (&y)[kE], double2* sm, double* aux,
                          const FilterTables& t) {
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  const bool own = tid < T;
  double2 z[kE];
  if (own) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) z[c] = make_double2(ld_real(xg, n, tid + c * T), 0.0);
  }
  filt_even<N>(z, sm, t);
  if (own) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) aux[tid + c * T] = z[c].x;
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) {
      const int j = tid + c * T;
      z[c] = cscale(modulation(t, j), ld_real(xg, n, j));
    }
  }
  filt_odd<N>(z, sm, t);
  if (own) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) {
      const int j = tid + c * T;
      const double2 w = modulation(t, j);
      const double ax = aux[j] + fma(z[c].x, w.x, z[c].y * w.y);  // + Re(conj(w) z)
      y[c] = kg ? fma(shift, ld_real(xg, n, j), ld_real(kg, n, j) * ax) : ax;
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
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  double out[kE];
  apply_level_op<N>(x + off, kappa ? kappa + off : nullptr, shift, n, out, sm, aux, tab);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) st_real(y + off, n, tid + c * T, out[c]);
  }
}

// --------------------------------------------------------------- precond
template <int N>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_strang_apply(int n, const double* __restrict__ v, double* __restrict__ zo, double shift,
               double kbar, const double* __restrict__ kbar_dev, FilterTables tab) {
  extern __shared__ double2 sm[];
  constexpr int T = KShape<N>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  const double kb = kbar_dev ? kbar_dev[blockIdx.x] : kbar;
  double2 z[kE];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) z[c] = make_double2(ld_real(v + off, n, tid + c * T), 0.0);
  }
  filt_strang<N>(z, sm, tab, shift, kb);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < KShape<N>::E; ++c) st_real(zo + off, n, tid + c * T, z[c].x);
  }
}

// --------------------------------------------------------------- solver
// Transform phases of the solve are out-of-line device functions with a
// pointer/scalar interface: vectors live in the instance's L2-resident
// workspace between phases, so a call boundary carries no vector state and
// each phase gets the whole register budget (inlining ~10 transforms into
// one loop body made ptxas interleave them and spill KBs per thread).

// dst = P^{-1} src on the owned slots
template <int N>
__device__ __noinline__ void dev_precond(const double* __restrict__ src, double* __restrict__ dst,
                                         int n, double d, double kbar, double2* sm,
                                         FilterTables t) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  const int tid = threadIdx.x;
  double2 z[kE];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = make_double2(ld_real(src, n, tid + c * T), 0.0);
  }
  filt_strang<N>(z, sm, t, d, kbar);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < E; ++c) st_real(dst, n, tid + c * T, z[c].x);
  }
}

// dst = shift*src + kappa .* (A src); returns this thread's partial
// (sum dst*dst, sum dst*w) (w == nullptr: second entry 0)
template <int N>
__device__ __noinline__ double2 dev_apply(const double* __restrict__ src, double* __restrict__ dst,
                                          const double* __restrict__ kg, double d, int n,
                                          double2* sm, double* aux, FilterTables t,
                                          const double* __restrict__ w) {
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  const int tid = threadIdx.x;
  double y[kE];
  apply_level_op<N>(src, kg, d, n, y, sm, aux, t);
  double2 part = make_double2(0.0, 0.0);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = tid + c * T;
      st_real(dst, n, j, y[c]);
      if (j < n) {
        part.x = fma(y[c], y[c], part.x);
        if (w) part.y = fma(y[c], w[j], part.y);
      }
    }
  }
  return part;
}

// PC: 0 = no preconditioner ("krylov"), 1 = Strang ("pkrylov", pow2 n = N)
// CG: false = BiCGSTAB, true = PCG (kappa_x_independent)
template <int N, int PC, bool CG>
__global__ void __launch_bounds__(KShape<N>::BLOCK, KShape<N>::MIN_BLOCKS)
k_krylov_solve(KrylovArgs a) {
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  constexpr int T = KShape<N>::T;
  constexpr int E = KShape<N>::E;
  double* aux = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + KShape<N>::FFT_BYTES);
  const int tid = threadIdx.x;
  const bool own = tid < T;
  const int b = blockIdx.x;
  const int n = a.n;
  const long off = (long)b * n;
  const double d = a.shift;

  // ---- kappa on the grid (scheme.py:156-160,280) and kappa_bar (scheme.py:135)
  const double* kg = (a.kappa ? a.kappa : (const double*)a.kwork) + off;
  double kbar;
  {
    double ksum = 0.0, kmin = 1e308;
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) {
        const int j = tid + c * T;
        if (j < n) {
          double k;
          if (a.kappa) {
            k = a.kappa[off + j];
          } else {
            k = 0.0;
            for (int q = 0; q < a.nk; ++q) {
              const double mq = a.kmodes[q * a.kq_stride + (long)b * a.kb_stride + j];
              // no contraction: reproduce numpy's  acc + mode*coef  rounding
              k = __dadd_rn(k, __dmul_rn(mq, a.kcoef[q]));
            }
            a.kwork[off + j] = k;
          }
          ksum += k;
          kmin = fmin(kmin, k);
        }
      }
    }
    kmin = block_min1(kmin, red);
    if (kmin <= 0.0) {
      if (tid == 0) {
        a.status[b] = TSF_KAPPA_NONPOS;
        a.iters[b] = 0;
        a.relres[b] = 0.0;
      }
      return;
    }
    const double kmean = block_sum1(ksum, red) / n;
    kbar = a.kbar > 0.0 ? a.kbar : kmean;
    if constexpr (PC == 1) {
      // total eigenvalues d + kbar*lam > 0  (toeplitz.py:122-124)
      double tmin = 1e308;
      for (int k = tid; k < n; k += blockDim.x) tmin = fmin(tmin, d + kbar * ldt(&a.tab.pclam[k]).x);
      tmin = block_min1(tmin, red);
      if (tmin <= 0.0) {
        if (tid == 0) {
          a.status[b] = TSF_PRECOND_NONPOS;
          a.iters[b] = 0;
          a.relres[b] = 0.0;
        }
        return;
      }
    }
  }

  const double* r0g = a.rhs + off;
  double* xg = a.x + off;
  double* rg = a.r + off;
  double* pg = a.p + off;
  double* vg = a.v + off;
  double* sg = a.s + off;
  double* tg = a.t + off;
  // without a preconditioner p_hat == p and s_hat == s
  double* phg = PC ? a.ph + off : pg;
  double* shg = PC ? a.sh + off : sg;
  auto finish = [&](int it, double rel, int st) {
    if (tid == 0) {
      a.iters[b] = it;
      a.relres[b] = rel;
      a.status[b] = st;
    }
  };

  // ---- r = r0 = rhs, x = 0  (krylov.py:107-113 / 64-69)
  double ss0 = 0.0;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int j = tid + c * T;
      const double r0 = ld_real(r0g, n, j);
      ss0 = fma(r0, r0, ss0);
      st_real(xg, n, j, 0.0);
    }
  }
  ss0 = block_sum1(ss0, red);
  const double nrm0 = sqrt(ss0);
  if (nrm0 == 0.0) {
    finish(0, 0.0, TSF_OK);
    return;
  }

  if constexpr (!CG) {
    // ================= BiCGSTAB (krylov.py:88-153) =================
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    double rho_new = ss0;   // r0 . r with r = r0 (same reduction)
    double rnorm = nrm0;
    for (int it = 1; it <= a.max_iters; ++it) {
      if (rho_new == 0.0) {
        finish(it, rnorm / nrm0, TSF_BD_RHO);
        return;
      }
      // p = r  |  p = r + beta (p - omega v)
      if (own) {
        const double beta = (rho_new / rho) * (alpha / omega);
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const int j = tid + c * T;
          const double p = (it == 1) ? ld_real(r0g, n, j)
                                     : ld_real(rg, n, j) +
                                           beta * (ld_real(pg, n, j) - omega * ld_real(vg, n, j));
          st_real(pg, n, j, p);
        }
      }
      if constexpr (PC == 1) dev_precond<N>(pg, phg, n, d, kbar, sm, a.tab);
      const double2 pv = dev_apply<N>(phg, vg, kg, d, n, sm, aux, a.tab, r0g);
      const double denom = block_sum1(pv.y, red);
      if (denom == 0.0) {
        finish(it, rnorm / nrm0, TSF_BD_R0V);
        return;
      }
      alpha = rho_new / denom;
      // s = r - alpha v
      double part = 0.0;
      if (own) {
        const double* rc = (it == 1) ? r0g : rg;
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const int j = tid + c * T;
          const double sv = ld_real(rc, n, j) - alpha * ld_real(vg, n, j);
          st_real(sg, n, j, sv);
          if (j < n) part = fma(sv, sv, part);
        }
      }
      const double snorm = sqrt(block_sum1(part, red));
      if (snorm / nrm0 < a.tol) {
        // x += alpha p_hat (early exit counts as a full iteration, krylov.py:135-137)
        if (own) {
#pragma unroll
          for (int c = 0; c < E; ++c) {
            const int j = tid + c * T;
            st_real(xg, n, j, ld_real(xg, n, j) + alpha * ld_real(phg, n, j));
          }
        }
        finish(it, snorm / nrm0, TSF_OK);
        return;
      }
      if constexpr (PC == 1) dev_precond<N>(sg, shg, n, d, kbar, sm, a.tab);
      const double2 tp = dev_apply<N>(shg, tg, kg, d, n, sm, aux, a.tab, sg);
      Vals<2> red2;
      red2.v[0] = tp.x;
      red2.v[1] = tp.y;
      red2 = block_sum<2>(red2, red);
      if (red2.v[0] == 0.0) {
        finish(it, snorm / nrm0, TSF_BD_OMEGA_DEN);
        return;
      }
      omega = red2.v[1] / red2.v[0];
      // x += alpha p_hat + omega s_hat ; r = s - omega t
      red2.v[0] = 0.0;
      red2.v[1] = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const int j = tid + c * T;
          st_real(xg, n, j,
                  ld_real(xg, n, j) + (alpha * ld_real(phg, n, j) + omega * ld_real(shg, n, j)));
          const double rn = ld_real(sg, n, j) - omega * ld_real(tg, n, j);
          st_real(rg, n, j, rn);
          if (j < n) {
            red2.v[0] = fma(rn, rn, red2.v[0]);
            red2.v[1] = fma(r0g[j], rn, red2.v[1]);
          }
        }
      }
      rho = rho_new;
      red2 = block_sum<2>(red2, red);
      rnorm = sqrt(red2.v[0]);
      const double rel = rnorm / nrm0;
      if (rel < a.tol) {
        finish(it, rel, TSF_OK);
        return;
      }
      if (omega == 0.0) {
        finish(it, rel, TSF_BD_OMEGA);
        return;
      }
      rho_new = red2.v[1];
    }
    finish(a.max_iters, rnorm / nrm0, TSF_NOT_CONVERGED);
  } else {
    // ================= PCG (krylov.py:43-85) =================
    // r = b; z = P^{-1} r; p = z  (z kept in s, p written directly)
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) {
        const int j = tid + c * T;
        st_real(rg, n, j, ld_real(r0g, n, j));
        if (!PC) st_real(pg, n, j, ld_real(r0g, n, j));
      }
    }
    if constexpr (PC == 1) dev_precond<N>(rg, pg, n, d, kbar, sm, a.tab);
    double part = 0.0;
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) {
        const int j = tid + c * T;
        if (j < n) part = fma(r0g[j], pg[j], part);
      }
    }
    double rz = block_sum1(part, red);
    double rnorm = nrm0;
    for (int it = 1; it <= a.max_iters; ++it) {
      const double2 qp = dev_apply<N>(pg, vg, kg, d, n, sm, aux, a.tab, pg);  // q = M p
      const double curv = block_sum1(qp.y, red);
      if (curv <= 0.0) {
        finish(it, rnorm / nrm0, TSF_BD_CURVATURE);
        return;
      }
      const double al = rz / curv;
      part = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const int j = tid + c * T;
          st_real(xg, n, j, ld_real(xg, n, j) + al * ld_real(pg, n, j));
          const double r1 = ld_real(rg, n, j) - al * ld_real(vg, n, j);
          st_real(rg, n, j, r1);
          if (j < n) part = fma(r1, r1, part);
        }
      }
      rnorm = sqrt(block_sum1(part, red));
      const double rel = rnorm / nrm0;
      if (rel < a.tol) {
        finish(it, rel, TSF_OK);
        return;
      }
      double* zg = PC ? sg : rg;
      if constexpr (PC == 1) dev_precond<N>(rg, sg, n, d, kbar, sm, a.tab);
      part = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const int j = tid + c * T;
          if (j < n) part = fma(rg[j], zg[j], part);
        }
      }
      const double rz_new = block_sum1(part, red);
      const double beta = rz_new / rz;
      if (own) {
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const int j = tid + c * T;
          st_real(pg, n, j, ld_real(zg, n, j) + beta * ld_real(pg, n, j));
        }
      }
      rz = rz_new;
    }
    finish(a.max_iters, rnorm / nrm0, TSF_NOT_CONVERGED);
  }
}

// --------------------------------------------------------------- debug FFT
template <int N, int E, bool INV>
__global__ void k_fft_debug(const double2* __restrict__ in, double2* __restrict__ out,
                            const double2* __restrict__ tw, int tw_log_scale) {
  extern __shared__ double2 sm[];
  constexpr int T = N / E;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * N;
  double2 v[E];
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

}  // namespace tsf
