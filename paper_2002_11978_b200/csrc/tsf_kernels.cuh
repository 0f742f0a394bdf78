// Batched per-instance kernels (one CTA per problem instance, n <= 4096).
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
// Template parameter L is the circulant embedding length (pow2 >= 2n-1).
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
  int* iters;               // per-instance outputs
  double* relres;
  int* status;
  FilterTables tab;
};

template <int L>
struct KShape {
  static constexpr int T = L / 16;               // owning threads
  static constexpr int BLOCK = T < 32 ? 32 : T;  // launched threads
  static constexpr int SMEM = FftPlan<L, 16>::SMEM_ELEMS * 16;
};

// --------------------------------------------------------------- matvec
template <int L>
__global__ void __launch_bounds__(KShape<L>::BLOCK)
k_toeplitz_apply(int n, const double* __restrict__ x, double* __restrict__ y,
                 const double* __restrict__ kappa, double shift, int has_kappa,
                 FilterTables tab) {
  extern __shared__ double2 sm[];
  constexpr int T = KShape<L>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  double xv[8], io[8];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) io[c] = xv[c] = ld_real(x + off, n, tid + c * T);
  }
  toeplitz_filter<L>(io, sm, tab);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = tid + c * T;
      double out = io[c];
      if (has_kappa) out = fma(shift, xv[c], ld_real(kappa + off, n, j) * out);
      st_real(y + off, n, j, out);
    }
  }
}

// --------------------------------------------------------------- precond
template <int L>
__global__ void __launch_bounds__(KShape<L>::BLOCK)
k_strang_apply(int n, const double* __restrict__ v, double* __restrict__ z, double shift,
               double kbar, const double* __restrict__ kbar_dev, FilterTables tab) {
  extern __shared__ double2 sm[];
  constexpr int T = KShape<L>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  const double kb = kbar_dev ? kbar_dev[blockIdx.x] : kbar;
  double io[8];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) io[c] = ld_real(v + off, n, tid + c * T);
  }
  strang_filter<L>(io, sm, tab, shift, kb);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) st_real(z + off, n, tid + c * T, io[c]);
  }
}

// --------------------------------------------------------------- solver
// PC: 0 = no preconditioner ("krylov"), 1 = Strang ("pkrylov", pow2 n = L/2)
// CG: false = BiCGSTAB, true = PCG (kappa_x_independent)
template <int L, int PC, bool CG>
__global__ void __launch_bounds__(KShape<L>::BLOCK)
k_krylov_solve(KrylovArgs a) {
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  constexpr int T = KShape<L>::T;
  const int tid = threadIdx.x;
  const bool own = tid < T;
  const int b = blockIdx.x;
  const int n = a.n;
  const long off = (long)b * n;
  const double* r0g = a.rhs + off;
  double* xg = a.x + off;
  double* rg = a.r + off;
  double* pg = a.p + off;
  double* vg = a.v + off;
  double* phg = a.ph + off;
  double* sg = a.s + off;
  const double d = a.shift;

  // ---- kappa on the grid (scheme.py:156-160,280) and kappa_bar (scheme.py:135)
  const double* kg;
  double ksum = 0.0, kmin = 1e308;
  if (a.kappa) {
    kg = a.kappa + off;
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = tid + c * T;
        if (j < n) {
          const double k = kg[j];
          ksum += k;
          kmin = fmin(kmin, k);
        }
      }
    }
  } else {
    double* kw = a.kwork + off;
    kg = kw;
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int j = tid + c * T;
        if (j < n) {
          double acc = 0.0;
          for (int q = 0; q < a.nk; ++q) {
            const double mq = a.kmodes[q * a.kq_stride + (long)b * a.kb_stride + j];
            // no contraction: reproduce numpy's  acc + mode*coef  rounding
            acc = __dadd_rn(acc, __dmul_rn(mq, a.kcoef[q]));
          }
          kw[j] = acc;
          ksum += acc;
          kmin = fmin(kmin, acc);
        }
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
  const double kbar = a.kbar > 0.0 ? a.kbar : kmean;
  if constexpr (PC == 1) {
    // total eigenvalues d + kbar*lam > 0  (toeplitz.py:122-124)
    double tmin = 1e308;
    for (int k = tid; k < n; k += blockDim.x) tmin = fmin(tmin, d + kbar * __ldg(&a.tab.pclam[k]).x);
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

  auto precond = [&](double (&io)[8]) {
    if constexpr (PC == 1) strang_filter<L>(io, sm, a.tab, d, kbar);
  };
  // y = d*u + kappa .* (A u); u preserved
  auto apply_op = [&](const double (&u)[8], double (&y)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = u[c];
    toeplitz_filter<L>(y, sm, a.tab);
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) y[c] = fma(d, u[c], ld_real(kg, n, tid + c * T) * y[c]);
    }
  };
  auto dot_loc = [](const double (&u)[8], const double (&w)[8]) {
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc = fma(u[c], w[c], acc);
    return acc;
  };
  auto load = [&](double (&u)[8], const double* g) {
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) u[c] = ld_real(g, n, tid + c * T);
    }
  };
  auto store = [&](double* g, const double (&u)[8]) {
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) st_real(g, n, tid + c * T, u[c]);
    }
  };
  auto finish = [&](int it, double rel, int st) {
    if (tid == 0) {
      a.iters[b] = it;
      a.relres[b] = rel;
      a.status[b] = st;
    }
  };

  double u[8], w[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) u[c] = w[c] = 0.0;

  // ---- r = r0 = rhs, x = 0  (krylov.py:107-113 / 64-69)
  load(u, r0g);
  const double ss0 = block_sum1(own ? dot_loc(u, u) : 0.0, red);
  const double nrm0 = sqrt(ss0);
  {
    double zero[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) zero[c] = 0.0;
    store(xg, zero);
  }
  if (nrm0 == 0.0) {
    finish(0, 0.0, TSF_OK);
    return;
  }
  const int max_iters = a.max_iters;
  const double tol = a.tol;

  if constexpr (!CG) {
    // ================= BiCGSTAB (krylov.py:88-153) =================
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    double rho_new = ss0;           // r0 . r with r = r0
    double rnorm = nrm0;            // ||r|| for breakdown reports
    for (int it = 1; it <= max_iters; ++it) {
      if (rho_new == 0.0) {
        finish(it, rnorm / nrm0, TSF_BD_RHO);
        return;
      }
      // p = r  |  p = r + beta (p - omega v)
      if (it == 1) {
        load(u, r0g);
      } else {
        const double beta = (rho_new / rho) * (alpha / omega);
        if (own) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int j = tid + c * T;
            u[c] = ld_real(rg, n, j) + beta * (ld_real(pg, n, j) - omega * ld_real(vg, n, j));
          }
        }
      }
      store(pg, u);
      precond(u);         // u = p_hat
      store(phg, u);
      apply_op(u, w);     // w = v = M p_hat
      store(vg, w);
      double r0v[8];
      load(r0v, r0g);
      const double denom = block_sum1(own ? dot_loc(r0v, w) : 0.0, red);
      if (denom == 0.0) {
        finish(it, rnorm / nrm0, TSF_BD_R0V);
        return;
      }
      alpha = rho_new / denom;
      // s = r - alpha v
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double rr = (it == 1) ? r0v[c] : ld_real(rg, n, tid + c * T);
          w[c] = rr - alpha * w[c];
        }
      }
      const double snorm = sqrt(block_sum1(own ? dot_loc(w, w) : 0.0, red));
      if (snorm / nrm0 < tol) {
        // x += alpha p_hat (early exit counts as a full iteration, krylov.py:135-137)
        if (own) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int j = tid + c * T;
            st_real(xg, n, j, ld_real(xg, n, j) + alpha * u[c]);
          }
        }
        finish(it, snorm / nrm0, TSF_OK);
        return;
      }
      store(sg, w);
      precond(w);         // w = s_hat
      apply_op(w, u);     // u = t = M s_hat
      Vals<2> red2;
      red2.v[0] = 0.0;
      red2.v[1] = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double ss = ld_real(sg, n, tid + c * T);
          red2.v[0] = fma(u[c], u[c], red2.v[0]);
          red2.v[1] = fma(u[c], ss, red2.v[1]);
        }
      }
      red2 = block_sum<2>(red2, red);
      const double tt = red2.v[0], ts = red2.v[1];
      if (tt == 0.0) {
        finish(it, snorm / nrm0, TSF_BD_OMEGA_DEN);
        return;
      }
      omega = ts / tt;
      // x += alpha p_hat + omega s_hat ; r = s - omega t
      red2.v[0] = 0.0;
      red2.v[1] = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = tid + c * T;
          st_real(xg, n, j, ld_real(xg, n, j) + (alpha * ld_real(phg, n, j) + omega * w[c]));
          const double rn = ld_real(sg, n, j) - omega * u[c];
          st_real(rg, n, j, rn);
          red2.v[0] = fma(rn, rn, red2.v[0]);
          red2.v[1] = fma(ld_real(r0g, n, j), rn, red2.v[1]);
        }
      }
      rho = rho_new;
      red2 = block_sum<2>(red2, red);
      rnorm = sqrt(red2.v[0]);
      const double rel = rnorm / nrm0;
      if (rel < tol) {
        finish(it, rel, TSF_OK);
        return;
      }
      if (omega == 0.0) {
        finish(it, rel, TSF_BD_OMEGA);
        return;
      }
      rho_new = red2.v[1];
    }
    finish(max_iters, rnorm / nrm0, TSF_NOT_CONVERGED);
  } else {
    // ================= PCG (krylov.py:43-85) =================
    store(rg, u);                    // r = b
    precond(u);                      // u = z
    store(pg, u);                    // p = z
    double rr[8];
    load(rr, r0g);
    double rz = block_sum1(own ? dot_loc(rr, u) : 0.0, red);
    double rnorm = nrm0;
    for (int it = 1; it <= max_iters; ++it) {
      load(u, pg);
      apply_op(u, w);                // w = q = M p
      const double curv = block_sum1(own ? dot_loc(u, w) : 0.0, red);
      if (curv <= 0.0) {
        finish(it, rnorm / nrm0, TSF_BD_CURVATURE);
        return;
      }
      const double al = rz / curv;
      double rr_loc = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = tid + c * T;
          st_real(xg, n, j, ld_real(xg, n, j) + al * u[c]);
          const double r1 = ld_real(rg, n, j) - al * w[c];
          st_real(rg, n, j, r1);
          rr[c] = r1;
          rr_loc = fma(r1, r1, rr_loc);
        }
      }
      rnorm = sqrt(block_sum1(rr_loc, red));
      const double rel = rnorm / nrm0;
      if (rel < tol) {
        finish(it, rel, TSF_OK);
        return;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) w[c] = rr[c];
      precond(w);                    // w = z
      const double rz_new = block_sum1(own ? dot_loc(rr, w) : 0.0, red);
      const double beta = rz_new / rz;
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) u[c] = w[c] + beta * u[c];
      }
      store(pg, u);
      rz = rz_new;
    }
    finish(max_iters, rnorm / nrm0, TSF_NOT_CONVERGED);
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
