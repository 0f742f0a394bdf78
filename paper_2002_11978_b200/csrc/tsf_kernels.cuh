// Batched per-instance kernels (one CTA per problem instance, n <= 8192).
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
#pragma once

#include "tsf_filters.cuh"

namespace tsf {

constexpr int kMaxModes = 4;

struct KrylovArgs {
  int n;
  int B;
  // right-hand side [B, n] (R0)
  const double* rhs;
  // solution [B, n] (written)
  double* x;
  // diffusivity: either given [B, n] (kappa != nullptr), or evaluated from
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
  // workspaces [B, n]
  double* r;
  double* p;
  double* v;
  double* ph;
  double* s;
  // per-instance outputs
  int* iters;
  double* relres;
  int* status;
  FilterTables tab;
};

template <int NMV>
struct KShape {
  static constexpr int T = NMV / 16;             // owning threads
  static constexpr int BLOCK = T < 32 ? 32 : T;  // launched threads
  static constexpr int SMEM = FftPlan<NMV, 16>::SMEM_ELEMS * 16;
};

// --------------------------------------------------------------- matvec
template <int NMV>
__global__ void __launch_bounds__(KShape<NMV>::BLOCK)
k_toeplitz_apply(int n, const double* __restrict__ x, double* __restrict__ y,
                 const double* __restrict__ kappa, double shift, int has_kappa,
                 FilterTables tab) {
  extern __shared__ double2 sm[];
  constexpr int T = KShape<NMV>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  const double* xb = x + off;
  double2 xv[8], io[8];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) io[c] = xv[c] = ld_pair(xb, n, tid + c * T);
  }
  toeplitz_filter<NMV>(io, sm, tab);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int j = tid + c * T;
      double2 out = io[c];
      if (has_kappa) {
        const double2 k = ld_pair(kappa + off, n, j);
        out = make_double2(fma(shift, xv[c].x, k.x * out.x), fma(shift, xv[c].y, k.y * out.y));
      }
      st_pair(y + off, n, j, out);
    }
  }
}

// --------------------------------------------------------------- precond
template <int NMV>
__global__ void __launch_bounds__(KShape<NMV>::BLOCK)
k_strang_apply(int n, const double* __restrict__ v, double* __restrict__ z, double shift,
               double kbar, const double* __restrict__ kbar_dev, FilterTables tab) {
  extern __shared__ double2 sm[];
  constexpr int T = KShape<NMV>::T;
  const int tid = threadIdx.x;
  const long off = (long)blockIdx.x * n;
  const double kb = kbar_dev ? kbar_dev[blockIdx.x] : kbar;
  double2 io[8];
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) io[c] = ld_pair(v + off, n, tid + c * T);
  }
  strang_filter<NMV>(io, sm, tab, shift, kb);
  if (tid < T) {
#pragma unroll
    for (int c = 0; c < 8; ++c) st_pair(z + off, n, tid + c * T, io[c]);
  }
}

// --------------------------------------------------------------- solver
// PC: 0 = no preconditioner ("krylov"), 1 = Strang ("pkrylov", pow2 n)
// CG: false = BiCGSTAB, true = PCG (kappa_x_independent)
template <int NMV, int PC, bool CG>
__global__ void __launch_bounds__(KShape<NMV>::BLOCK)
k_krylov_solve(KrylovArgs a) {
  extern __shared__ double2 sm[];
  __shared__ double red[4 * 32];
  constexpr int T = KShape<NMV>::T;
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
        if (2 * j < n) {
          double2 k = ld_pair(kg, n, j);
          ksum += k.x;
          kmin = fmin(kmin, k.x);
          if (2 * j + 1 < n) {
            ksum += k.y;
            kmin = fmin(kmin, k.y);
          }
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
        if (2 * j < n) {
          double2 acc = make_double2(0.0, 0.0);
          for (int q = 0; q < a.nk; ++q) {
            const double2 mq =
                ld_pair(a.kmodes + q * a.kq_stride + (long)b * a.kb_stride, n, j);
            // no contraction: reproduce numpy's  acc + mode*coef  rounding
            acc.x = __dadd_rn(acc.x, __dmul_rn(mq.x, a.kcoef[q]));
            acc.y = __dadd_rn(acc.y, __dmul_rn(mq.y, a.kcoef[q]));
          }
          st_pair(kw, n, j, acc);
          ksum += acc.x;
          kmin = fmin(kmin, acc.x);
          if (2 * j + 1 < n) {
            ksum += acc.y;
            kmin = fmin(kmin, acc.y);
          }
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
    for (int k = tid; k < n / 2; k += blockDim.x) {
      const double2 lam = __ldg(&a.tab.pclam[k]);
      tmin = fmin(tmin, fmin(d + kbar * lam.x, d + kbar * lam.y));
    }
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

  auto precond = [&](double2 (&io)[8]) {
    if constexpr (PC == 1) strang_filter<NMV>(io, sm, a.tab, d, kbar);
  };
  // y = d*u + kappa .* (A u); u preserved
  auto apply_op = [&](const double2 (&u)[8], double2 (&y)[8]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = u[c];
    toeplitz_filter<NMV>(y, sm, a.tab);
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 k = ld_pair(kg, n, tid + c * T);
        y[c] = make_double2(fma(d, u[c].x, k.x * y[c].x), fma(d, u[c].y, k.y * y[c].y));
      }
    }
  };
  auto dot_loc = [](const double2 (&u)[8], const double2 (&w)[8]) {
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc = fma(u[c].x, w[c].x, fma(u[c].y, w[c].y, acc));
    return acc;
  };
  auto load = [&](double2 (&u)[8], const double* g) {
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) u[c] = ld_pair(g, n, tid + c * T);
    }
  };
  auto store = [&](double* g, const double2 (&u)[8]) {
    if (own) {
#pragma unroll
      for (int c = 0; c < 8; ++c) st_pair(g, n, tid + c * T, u[c]);
    }
  };
  auto finish = [&](int it, double rel, int st) {
    if (tid == 0) {
      a.iters[b] = it;
      a.relres[b] = rel;
      a.status[b] = st;
    }
  };

  double2 u[8], w[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) u[c] = w[c] = make_double2(0.0, 0.0);

  // ---- r = r0 = rhs, x = 0  (krylov.py:107-113 / 64-69)
  load(u, r0g);
  const double ss0 = block_sum1(own ? dot_loc(u, u) : 0.0, red);
  const double nrm0 = sqrt(ss0);
  {
    double2 zero[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) zero[c] = make_double2(0.0, 0.0);
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
    double rho_new = ss0;           // r0 . r with r = r0 (same reduction)
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
            const double2 rr = ld_pair(rg, n, j), pp = ld_pair(pg, n, j), vv = ld_pair(vg, n, j);
            u[c] = make_double2(rr.x + beta * (pp.x - omega * vv.x),
                                rr.y + beta * (pp.y - omega * vv.y));
          }
        }
      }
      store(pg, u);
      precond(u);         // u = p_hat
      store(phg, u);
      apply_op(u, w);     // w = v = M p_hat
      store(vg, w);
      double2 r0v[8];
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
          const double2 rr = (it == 1) ? r0v[c] : ld_pair(rg, n, tid + c * T);
          w[c] = make_double2(rr.x - alpha * w[c].x, rr.y - alpha * w[c].y);
        }
      }
      const double snorm = sqrt(block_sum1(own ? dot_loc(w, w) : 0.0, red));
      if (snorm / nrm0 < tol) {
        // x += alpha p_hat (early exit counts as a full iteration, krylov.py:135-137)
        if (own) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int j = tid + c * T;
            const double2 xx = ld_pair(xg, n, j);
            st_pair(xg, n, j, make_double2(xx.x + alpha * u[c].x, xx.y + alpha * u[c].y));
          }
        }
        finish(it, snorm / nrm0, TSF_OK);
        return;
      }
      store(sg, w);
      precond(w);         // w = s_hat
      apply_op(w, u);     // u = t = M s_hat
      double tt = 0.0, ts = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double2 ss = ld_pair(sg, n, tid + c * T);
          tt = fma(u[c].x, u[c].x, fma(u[c].y, u[c].y, tt));
          ts = fma(u[c].x, ss.x, fma(u[c].y, ss.y, ts));
        }
      }
      Vals<2> red2;
      red2.v[0] = tt;
      red2.v[1] = ts;
      red2 = block_sum<2>(red2, red);
      tt = red2.v[0];
      ts = red2.v[1];
      if (tt == 0.0) {
        finish(it, snorm / nrm0, TSF_BD_OMEGA_DEN);
        return;
      }
      omega = ts / tt;
      // x += alpha p_hat + omega s_hat ; r = s - omega t
      double rr_loc = 0.0, r0r_loc = 0.0;
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int j = tid + c * T;
          const double2 xx = ld_pair(xg, n, j), phv = ld_pair(phg, n, j);
          st_pair(xg, n, j, make_double2(xx.x + (alpha * phv.x + omega * w[c].x),
                                         xx.y + (alpha * phv.y + omega * w[c].y)));
          const double2 ss = ld_pair(sg, n, j), r0 = ld_pair(r0g, n, j);
          const double2 rn = make_double2(ss.x - omega * u[c].x, ss.y - omega * u[c].y);
          st_pair(rg, n, j, rn);
          rr_loc = fma(rn.x, rn.x, fma(rn.y, rn.y, rr_loc));
          r0r_loc = fma(r0.x, rn.x, fma(r0.y, rn.y, r0r_loc));
        }
      }
      rho = rho_new;
      red2.v[0] = rr_loc;
      red2.v[1] = r0r_loc;
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
    // r = b (kept in rg), z = psolve(r), p = z, rz = r.z
    store(rg, u);
    precond(u);                      // u = z
    store(pg, u);
    double2 rr[8];
    load(rr, r0g);
    double rz = block_sum1(own ? dot_loc(rr, u) : 0.0, red);
    double rnorm = nrm0;
    for (int it = 1; it <= max_iters; ++it) {
      load(u, pg);
      apply_op(u, w);                // w = q = A p
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
          const double2 xx = ld_pair(xg, n, j);
          st_pair(xg, n, j, make_double2(xx.x + al * u[c].x, xx.y + al * u[c].y));
          double2 r1 = ld_pair(rg, n, j);
          r1 = make_double2(r1.x - al * w[c].x, r1.y - al * w[c].y);
          st_pair(rg, n, j, r1);
          rr[c] = r1;
          rr_loc = fma(r1.x, r1.x, fma(r1.y, r1.y, rr_loc));
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
        for (int c = 0; c < 8; ++c) {
          u[c] = make_double2(w[c].x + beta * u[c].x, w[c].y + beta * u[c].y);
        }
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
