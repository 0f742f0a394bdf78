// Large-n engine (n = 2^13 .. 2^24): tables, Krylov scalar / elementwise
// kernels and the host drivers.  Transform kernels: tsf_large.cuh.
//
// One BiCGSTAB iteration (krylov.py:88-153) for B instances is a fixed
// launch sequence; every kernel returns at once for instances whose LState
// says they finished, so the host launches whole chunks of iterations and
// polls the device count of unfinished instances between chunks (as the
// single-CTA engine does, tsf_dispatch_impl.cuh):
//   1  p_hat = P^{-1} p      col_fwd(p update) . row(Strang) . col_inv
//   2  v = M p_hat           col_fwd . row . col_inv, even + odd channels
//   3  alpha                 scalar kernel (r0.v from the combine partials)
//   4  s_hat = P^{-1} s      col_fwd(s = r - alpha v, ||s||^2) . row . col_inv
//   5  ||s||, early exit      scalar kernel
//   6  t = M s_hat           3 kernels (t.t, t.s partials)
//   7  omega                 scalar kernel
//   8  x, r update           elementwise (||r||^2, r0.r partials)
//   9  convergence, rho      scalar kernel
// Without the preconditioner steps 1/4 are elementwise kernels.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/tsfrac_b200.h"
#include "tsf_dispatch.h"
#include "tsf_large_api.h"

namespace tsf {
namespace {

constexpr int kLelThreads = 256;
constexpr int kLelPer = 4;
constexpr int kLelChunk = kLelThreads * kLelPer;  // elements per elementwise CTA
constexpr int kLscThreads = 256;
constexpr int kLargeChunk = 4;  // iterations launched between completion polls

enum LStage : int {
  LS_BEGIN = 0, LS_ALPHA = 1, LS_SNORM = 2, LS_OMEGA = 3, LS_REL = 4,   // BiCGSTAB
  LS_CG_RZ0 = 5, LS_CG_ALPHA = 6, LS_CG_REL = 7, LS_CG_BETA = 8,        // PCG
};

TSF_D double* pslot(const LargeArgs& a, int b, int slot) {
  return a.part + ((long)b * 4 + slot) * a.np;
}

TSF_D void lfinish(const LargeArgs& a, int b, int it, double rel, int status) {
  a.iters[b] = it;
  a.relres[b] = rel;
  a.status[b] = status;
  a.st[b].mode = LM_DONE;
  atomicSub(a.active, 1);
}

// ---- elementwise kernels: grid (n / kLelChunk, B)

// kappa on the grid (scheme.py:156-160,280), x = 0, partials: sum kappa,
// min kappa, ||r0||^2
__global__ void __launch_bounds__(kLelThreads) k_lel_begin(LargeArgs a, KrylovArgs k) {
  pdl_enter();
  __shared__ double red[4 * 32];
  const int b = blockIdx.y, tid = threadIdx.x;
  const long off = (long)b * a.n;
  double ksum = 0.0, kmin = 1e308, ss = 0.0;
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long j = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (j >= a.n) break;
    double kv;
    if (k.kappa) {
      kv = k.kappa[off + j];
    } else {
      kv = 0.0;
      for (int q = 0; q < k.nk; ++q) {
        const double mq = k.kmodes[q * k.kq_stride + (long)b * k.kb_stride + j];
        kv = __dadd_rn(kv, __dmul_rn(mq, k.kcoef[q]));  // numpy's acc + mode*coef
      }
      k.kwork[off + j] = kv;
    }
    ksum += kv;
    kmin = fmin(kmin, kv);
    a.x[off + j] = 0.0;
    const double r = a.r0[off + j];
    ss = fma(r, r, ss);
  }
  Vals<2> v;
  v.v[0] = ksum;
  v.v[1] = ss;
  v = block_sum<2>(v, red);
  kmin = block_min1(kmin, red);
  if (tid == 0) {
    pslot(a, b, 0)[blockIdx.x] = v.v[0];
    pslot(a, b, 1)[blockIdx.x] = kmin;
    pslot(a, b, 2)[blockIdx.x] = v.v[1];
  }
}

// p = r0 (it 1) or r + beta (p - omega v)   (no preconditioner: p_hat = p)
__global__ void __launch_bounds__(kLelThreads) k_lel_pupd(LargeArgs a) {
  pdl_enter();
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const long off = (long)b * a.n;
  const LState s = a.st[b];
  const double beta = s.it == 1 ? 0.0 : (s.rho_new / s.rho) * (s.alpha / s.omega);
  // operands loaded before the stores (aliasing pointers, see k_lcol_fwd)
  double rv[kLelPer], pv[kLelPer], vv[kLelPer];
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    const long j = off + (jj < a.n ? jj : 0);
    rv[c] = s.it == 1 ? a.r0[j] : a.r[j];
    pv[c] = s.it == 1 ? 0.0 : a.p[j];
    vv[c] = s.it == 1 ? 0.0 : a.v[j];
  }
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    a.p[off + jj] = s.it == 1 ? rv[c] : rv[c] + beta * (pv[c] - s.omega * vv[c]);
  }
}

// s = r - alpha v, ||s||^2 partial (slot 2)
__global__ void __launch_bounds__(kLelThreads) k_lel_supd(LargeArgs a) {
  pdl_enter();
  __shared__ double red[4 * 32];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const long off = (long)b * a.n;
  const LState s = a.st[b];
  const double* rc = s.it == 1 ? a.r0 : a.r;
  double ss = 0.0;
  double rv[kLelPer], vv[kLelPer];   // loads before the stores (see k_lel_pupd)
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    const long j = off + (jj < a.n ? jj : 0);
    rv[c] = rc[j];
    vv[c] = a.v[j];
  }
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    const double v = rv[c] - s.alpha * vv[c];
    a.s[off + jj] = v;
    ss = fma(v, v, ss);
  }
  ss = block_sum1(ss, red);
  if (tid == 0) pslot(a, b, 2)[blockIdx.x] = ss;
}

// x += alpha p_hat + omega s_hat ; r = s - omega t ; partials ||r||^2, r0.r
// (early-exit instances: x += alpha p_hat only)
__global__ void __launch_bounds__(kLelThreads) k_lel_xr(LargeArgs a, const double* __restrict__ ph,
                                                        const double* __restrict__ sh) {
  pdl_enter();
  __shared__ double red[4 * 32];
  const int b = blockIdx.y, tid = threadIdx.x;
  const LState s = a.st[b];
  if (s.mode == LM_DONE) return;
  const long off = (long)b * a.n;
  if (s.mode == LM_EARLY) {
#pragma unroll
    for (int c = 0; c < kLelPer; ++c) {
      const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
      if (jj >= a.n) break;
      const long j = off + jj;
      a.x[j] = a.x[j] + s.alpha * ph[j];
    }
    return;
  }
  Vals<2> v;
  v.v[0] = v.v[1] = 0.0;
  // all operands loaded before the first store (the vectors may alias, so a
  // store would otherwise hold back the next element's loads)
  double xv[kLelPer], pv[kLelPer], sv[kLelPer], ssv[kLelPer], tv[kLelPer], r0v[kLelPer];
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    const long j = off + (jj < a.n ? jj : 0);
    xv[c] = a.x[j];
    pv[c] = ph[j];
    sv[c] = sh[j];
    ssv[c] = a.s[j];
    tv[c] = a.t[j];
    r0v[c] = a.r0[j];
  }
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    const long j = off + jj;
    a.x[j] = xv[c] + (s.alpha * pv[c] + s.omega * sv[c]);
    const double r = ssv[c] - s.omega * tv[c];
    a.r[j] = r;
    v.v[0] = fma(r, r, v.v[0]);
    v.v[1] = fma(r0v[c], r, v.v[1]);
  }
  v = block_sum<2>(v, red);
  if (tid == 0) {
    pslot(a, b, 0)[blockIdx.x] = v.v[0];
    pslot(a, b, 1)[blockIdx.x] = v.v[1];
  }
}

// The level's Strang filter, permuted like the row spectra:
// pspec[k1 N2 + k2] = even part of 1/(d + kbar lam_k) / n at k = k1 + N1 k2
__global__ void __launch_bounds__(kLelThreads) k_lspec(LargeArgs a, double kbar,
                                                       const double* __restrict__ kbar_dev,
                                                       int use_state) {
  pdl_enter();
  const int b = blockIdx.y, tid = threadIdx.x;
  double kb = kbar;
  if (use_state) {
    if (inst_skip(a, b)) return;
    kb = a.st[b].kbar;
  } else if (kbar_dev) {
    kb = kbar_dev[b];
  }
  const double d = a.shift;
  const double inv_n = 1.0 / a.nt;   // the Strang tables exist only for n == nt
  const long off = (long)b * a.nt;
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long idx = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (idx >= a.nt) break;
    const double2 lam = ldt(&a.lt.lamP[idx]);
    a.pspec[off + idx] = 0.5 * (1.0 / (d + kb * lam.x) + 1.0 / (d + kb * lam.y)) * inv_n;
  }
}

// The level's Strang filter for the half-length engine: (S_k, S_{H-k}) / n at
// the half geometry's position of bin k (tsf_hlarge.cuh)
__global__ void __launch_bounds__(kLelThreads) k_hspec(LargeArgs a, double kbar,
                                                       const double* __restrict__ kbar_dev,
                                                       int use_state) {
  pdl_enter();
  const int b = blockIdx.y, tid = threadIdx.x;
  double kb = kbar;
  if (use_state) {
    if (inst_skip(a, b)) return;
    kb = a.st[b].kbar;
  } else if (kbar_dev) {
    kb = kbar_dev[b];
  }
  const double d = a.shift;
  const double inv_n = 1.0 / a.nt;
  const long H = a.nt / 2;
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long idx = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (idx >= H) break;
    const double2 l0 = ldt(&a.hg.lamH[2 * idx]), l1 = ldt(&a.hg.lamH[2 * idx + 1]);
    a.hg.pspec2[(long)b * H + idx] =
        make_double2(0.5 * (1.0 / (d + kb * l0.x) + 1.0 / (d + kb * l0.y)) * inv_n,
                     0.5 * (1.0 / (d + kb * l1.x) + 1.0 / (d + kb * l1.y)) * inv_n);
  }
}

// ---- PCG elementwise kernels (krylov.py:43-85)
// dst = src
__global__ void __launch_bounds__(kLelThreads) k_lel_copy(LargeArgs a, double* __restrict__ dst,
                                                          const double* __restrict__ src) {
  pdl_enter();
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const long off = (long)b * a.n;
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    dst[off + jj] = src[off + jj];
  }
}

// partial u . w into `slot`
__global__ void __launch_bounds__(kLelThreads) k_lel_dot(LargeArgs a, const double* __restrict__ u,
                                                         const double* __restrict__ w, int slot) {
  pdl_enter();
  __shared__ double red[4 * 32];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const long off = (long)b * a.n;
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    d = fma(u[off + jj], w[off + jj], d);
  }
  d = block_sum1(d, red);
  if (tid == 0) pslot(a, b, slot)[blockIdx.x] = d;
}

// x += alpha p ; r -= alpha q (q in v) ; partial ||r||^2 (slot 0)
__global__ void __launch_bounds__(kLelThreads) k_lel_cgxr(LargeArgs a) {
  pdl_enter();
  __shared__ double red[4 * 32];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const long off = (long)b * a.n;
  const double al = a.st[b].alpha;
  double rr = 0.0;
  double xv[kLelPer], pv[kLelPer], rv[kLelPer], vv[kLelPer];   // loads before the stores
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    const long j = off + (jj < a.n ? jj : 0);
    xv[c] = a.x[j];
    pv[c] = a.p[j];
    rv[c] = a.r[j];
    vv[c] = a.v[j];
  }
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    const long j = off + jj;
    a.x[j] = xv[c] + al * pv[c];
    const double r = rv[c] - al * vv[c];
    a.r[j] = r;
    rr = fma(r, r, rr);
  }
  rr = block_sum1(rr, red);
  if (tid == 0) pslot(a, b, 0)[blockIdx.x] = rr;
}

// p = z + beta p
__global__ void __launch_bounds__(kLelThreads) k_lel_cgp(LargeArgs a, const double* __restrict__ z) {
  pdl_enter();
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const long off = (long)b * a.n;
  const double beta = a.st[b].omega;   // PCG keeps beta in the omega slot
  double zv[kLelPer], pv[kLelPer];     // loads before the stores (see k_lel_pupd)
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    const long j = off + (jj < a.n ? jj : 0);
    zv[c] = z[j];
    pv[c] = a.p[j];
  }
#pragma unroll
  for (int c = 0; c < kLelPer; ++c) {
    const long jj = (long)blockIdx.x * kLelChunk + c * kLelThreads + tid;
    if (jj >= a.n) break;
    a.p[off + jj] = zv[c] + beta * pv[c];
  }
}

// ---- scalar kernel: one CTA per instance, partial sums in fixed order
TSF_D double psum(const LargeArgs& a, int b, int slot, int count, double* red) {
  const double* p = pslot(a, b, slot);
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += p[i];
  return block_sum1(s, red);
}

__global__ void __launch_bounds__(kLscThreads) k_lsc(LargeArgs a, int stage, int count,
                                                     double kbar_in, double lam_min, int pc) {
  pdl_enter();
  __shared__ double red[4 * 32];
  const int b = blockIdx.x, tid = threadIdx.x;
  if (stage == LS_BEGIN) {
    const double* pm = pslot(a, b, 1);
    double kmin = 1e308;
    for (int i = tid; i < count; i += blockDim.x) kmin = fmin(kmin, pm[i]);
    kmin = block_min1(kmin, red);
    const double ksum = psum(a, b, 0, count, red);
    const double ss = psum(a, b, 2, count, red);
    if (tid != 0) return;
    LState s{};
    s.mode = LM_ACTIVE;
    a.st[b] = s;
    if (kmin <= 0.0) return lfinish(a, b, 0, 0.0, TSF_KAPPA_NONPOS);
    const double kbar = kbar_in > 0.0 ? kbar_in : ksum / a.n;
    // total eigenvalues d + kbar lam > 0 (toeplitz.py:122-124); monotone in lam
    if (pc && a.shift + kbar * lam_min <= 0.0) return lfinish(a, b, 0, 0.0, TSF_PRECOND_NONPOS);
    if (sqrt(ss) == 0.0) return lfinish(a, b, 0, 0.0, TSF_OK);
    s.rho = s.alpha = s.omega = 1.0;
    s.rho_new = ss;
    s.nrm0 = s.rnorm = s.snorm = sqrt(ss);
    s.kbar = kbar;
    s.it = 1;
    s.mode = LM_ACTIVE;
    a.st[b] = s;
    return;
  }
  const LState s = a.st[b];
  if (s.mode == LM_DONE) return;
  if (stage == LS_ALPHA) {
    if (s.mode != LM_ACTIVE) return;
    const double denom = psum(a, b, 1, count, red);
    if (tid != 0) return;
    if (denom == 0.0) return lfinish(a, b, s.it, s.rnorm / s.nrm0, TSF_BD_R0V);
    a.st[b].alpha = s.rho_new / denom;
  } else if (stage == LS_SNORM) {
    if (s.mode != LM_ACTIVE) return;
    const double snorm = sqrt(psum(a, b, 2, count, red));
    if (tid != 0) return;
    a.st[b].snorm = snorm;
    if (snorm / s.nrm0 < a.tol) a.st[b].mode = LM_EARLY;  // krylov.py:135-137
  } else if (stage == LS_OMEGA) {
    if (s.mode != LM_ACTIVE) return;
    const double tt = psum(a, b, 0, count, red);
    const double ts = psum(a, b, 1, count, red);
    if (tid != 0) return;
    if (tt == 0.0) return lfinish(a, b, s.it, s.snorm / s.nrm0, TSF_BD_OMEGA_DEN);
    a.st[b].omega = ts / tt;
  } else if (stage == LS_CG_RZ0) {         // rz = r . z of the start vector
    if (s.mode != LM_ACTIVE) return;
    const double rz = psum(a, b, 0, count, red);
    if (tid == 0) a.st[b].rz = rz;
  } else if (stage == LS_CG_ALPHA) {       // curvature p . A p
    if (s.mode != LM_ACTIVE) return;
    const double curv = psum(a, b, 1, count, red);
    if (tid != 0) return;
    if (curv <= 0.0) return lfinish(a, b, s.it, s.rnorm / s.nrm0, TSF_BD_CURVATURE);
    a.st[b].alpha = s.rz / curv;
  } else if (stage == LS_CG_REL) {
    if (s.mode != LM_ACTIVE) return;
    const double rnorm = sqrt(psum(a, b, 0, count, red));
    if (tid != 0) return;
    const double rel = rnorm / s.nrm0;
    if (rel < a.tol) return lfinish(a, b, s.it, rel, TSF_OK);
    if (s.it >= a.max_iters) return lfinish(a, b, a.max_iters, rel, TSF_NOT_CONVERGED);
    a.st[b].rnorm = rnorm;
  } else if (stage == LS_CG_BETA) {
    if (s.mode != LM_ACTIVE) return;
    const double rz_new = psum(a, b, 0, count, red);
    if (tid != 0) return;
    a.st[b].omega = rz_new / s.rz;   // beta
    a.st[b].rz = rz_new;
    a.st[b].it = s.it + 1;
  } else {  // LS_REL
    if (s.mode == LM_EARLY) {
      if (tid == 0) lfinish(a, b, s.it, s.snorm / s.nrm0, TSF_OK);
      return;
    }
    const double rr = psum(a, b, 0, count, red);
    const double rho_new = psum(a, b, 1, count, red);
    if (tid != 0) return;
    const double rnorm = sqrt(rr);
    const double rel = rnorm / s.nrm0;
    if (rel < a.tol) return lfinish(a, b, s.it, rel, TSF_OK);
    if (s.omega == 0.0) return lfinish(a, b, s.it, rel, TSF_BD_OMEGA);
    if (s.it >= a.max_iters) return lfinish(a, b, a.max_iters, rel, TSF_NOT_CONVERGED);
    if (rho_new == 0.0) return lfinish(a, b, s.it + 1, rel, TSF_BD_RHO);  // krylov.py:118-121
    LState u = s;
    u.rho = s.rho_new;
    u.rho_new = rho_new;
    u.rnorm = rnorm;
    u.it = s.it + 1;
    a.st[b] = u;
  }
}

// ---- per-size dispatch
template <int LOG = kLargeMinLog>
int col_fwd_at(int lg, const LargeArgs& a, const double* src, int mode, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::col_fwd(a, src, mode, st);
  if constexpr (LOG < kLargeMaxLog) return col_fwd_at<LOG + 1>(lg, a, src, mode, st);
  return report_error(TSF_E_UNSUPPORTED, "large-n column length out of range");
}
template <int LOG = kLargeMinLog>
int col_group_at(int lg) {
  if (lg == LOG) return LargeDispatch<LOG>::col_group();
  if constexpr (LOG < kLargeMaxLog) return col_group_at<LOG + 1>(lg);
  return 1;
}
template <int LOG = kLargeMinLog>
int row_at(int lg, const LargeArgs& a, int spec, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::row(a, spec, st);
  if constexpr (LOG < kLargeMaxLog) return row_at<LOG + 1>(lg, a, spec, st);
  return report_error(TSF_E_UNSUPPORTED, "large-n row length out of range");
}
template <int LOG = kLargeMinLog>
int col_inv_at(int lg, const LargeArgs& a, double* dst, int mode, const double* xin,
               const double* w1, int slot, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::col_inv(a, dst, mode, xin, w1, slot, st);
  if constexpr (LOG < kLargeMaxLog) return col_inv_at<LOG + 1>(lg, a, dst, mode, xin, w1, slot, st);
  return report_error(TSF_E_UNSUPPORTED, "large-n column length out of range");
}

template <int LOG = kLargeMinLog>
int hcol_fwd_at(int lg, const LargeArgs& a, const double* src, int mode, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::hcol_fwd(a, src, mode, st);
  if constexpr (LOG < kLargeMaxLog) return hcol_fwd_at<LOG + 1>(lg, a, src, mode, st);
  return report_error(TSF_E_UNSUPPORTED, "half-length column length out of range");
}
template <int LOG = kLargeMinLog>
int hrow_strang_at(int lg, const LargeArgs& a, int mode, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::hrow_strang(a, mode, st);
  if constexpr (LOG < kLargeMaxLog) return hrow_strang_at<LOG + 1>(lg, a, mode, st);
  return report_error(TSF_E_UNSUPPORTED, "half-length row length out of range");
}
template <int LOG = kLargeMinLog>
int hrow_mv_at(int lg, const LargeArgs& a, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::hrow_mv(a, st);
  if constexpr (LOG < kLargeMaxLog) return hrow_mv_at<LOG + 1>(lg, a, st);
  return report_error(TSF_E_UNSUPPORTED, "half-length row length out of range");
}
template <int LOG = kLargeMinLog>
int hcol_inv_at(int lg, const LargeArgs& a, double* dst, int mode, double* dst1, const double* xin,
                const double* ye, const double* w1, int slot, cudaStream_t st) {
  if (lg == LOG) return LargeDispatch<LOG>::hcol_inv(a, dst, mode, dst1, xin, ye, w1, slot, st);
  if constexpr (LOG < kLargeMaxLog)
    return hcol_inv_at<LOG + 1>(lg, a, dst, mode, dst1, xin, ye, w1, slot, st);
  return report_error(TSF_E_UNSUPPORTED, "half-length column length out of range");
}

int ilog2i(long x) {
  int r = 0;
  while ((1L << r) < x) ++r;
  return r;
}

int cuda_check(cudaError_t e, const char* what) { return e == cudaSuccess ? 0 : report_cuda(e, what); }

struct Runner {
  const LargePlan* lp;
  LargeArgs a;
  cudaStream_t st;
  int lg1, lg2;
  int lg1h = 0, lg2h = 0;
  bool half = false;   // this solve runs the half-length engine (tsf_hlarge.cuh)

  // dst = P^{-1} src through ONE length-n/2 transform pair; ye receives the
  // even-bin half of the Toeplitz product of dst (formed from the same
  // filtered spectrum inside the row kernel: no forward transform)
  int hstrang(int in_mode, const double* src, double* dst, double* ye) {
    int rc;
    if ((rc = hcol_fwd_at(lg1h, a, src, in_mode, st))) return rc;
    if ((rc = hrow_strang_at(lg2h, a, ye ? 2 : 0, st))) return rc;
    return hcol_inv_at(lg1h, a, dst, HO_PACK, ye, nullptr, nullptr, nullptr, -1, st);
  }
  // standalone product (no Strang spectrum to start from): the even bins
  // through the packed forward transform with the symbol as filter
  int happly_plain(const double* src, double* dst, double* tmp) {
    int rc;
    if ((rc = hcol_fwd_at(lg1h, a, src, HF_LOAD, st))) return rc;
    if ((rc = hrow_strang_at(lg2h, a, 1, st))) return rc;
    if ((rc = hcol_inv_at(lg1h, a, tmp, HO_PACK, nullptr, nullptr, nullptr, nullptr, -1, st)))
      return rc;
    return happly(src, dst, nullptr, -1, tmp);
  }
  // dst = d src + kappa . (A src) for src = the last hstrang output, ye its
  // even-bin half
  int happly(const double* src, double* dst, const double* w1, int slot, const double* ye) {
    int rc;
    if ((rc = hcol_fwd_at(lg1h, a, src, HF_ODD, st))) return rc;
    if ((rc = hrow_mv_at(lg2h, a, st))) return rc;
    return hcol_inv_at(lg1h, a, dst, HO_ODD, nullptr, src, ye, w1, slot, st);
  }
  int bicg_iteration_half() {
    int rc;
    const int NC = lp->ncol_cta_h, NR = (a.n + kLelChunk - 1) / kLelChunk;
    if ((rc = hstrang(HF_PUPD, nullptr, a.ph, a.t))) return rc;  // t is free until the t-product
    if ((rc = happly(a.ph, a.v, a.r0, 0, a.t))) return rc;
    if ((rc = sc(LS_ALPHA, NC, 1))) return rc;
    if ((rc = hstrang(HF_SUPD, nullptr, a.sh, a.r))) return rc;  // r is dead once s exists
    if ((rc = sc(LS_SNORM, NC, 1))) return rc;
    if ((rc = happly(a.sh, a.t, a.s, 0, a.r))) return rc;
    if ((rc = sc(LS_OMEGA, NC, 1))) return rc;
    launch_pdl(k_lel_xr, lel_grid(), kLelThreads, 0, st, a, (const double*)a.ph,
               (const double*)a.sh);
    if ((rc = cuda_check(cudaGetLastError(), "k_lel_xr"))) return rc;
    return sc(LS_REL, NR, 1);
  }

  // dst = Re IFFT_n(S . FFT_n(src)) with the Strang spectrum (pspec);
  // in_mode: the column prologue that forms src (p / s update) on the fly
  int strang(int in_mode, const double* src, double* dst) {
    int rc;
    if ((rc = col_fwd_at(lg1, a, src, in_mode, st))) return rc;
    if ((rc = row_at(lg2, a, RS_STRANG, st))) return rc;
    return col_inv_at(lg1, a, dst, CO_REAL, nullptr, nullptr, -1, st);
  }
  // dst = d src + kappa . (A src)  (kappa null: A src); dot partials
  // dst.dst (slot) and dst.w1 (slot + 1) per column CTA
  int apply(const double* src, double* dst, const double* w1, int slot) {
    int rc;
    if ((rc = col_fwd_at(lg1, a, src, CI_APPLY, st))) return rc;
    if ((rc = row_at(lg2, a, RS_APPLY, st))) return rc;
    return col_inv_at(lg1, a, dst, CO_APPLY, src, w1, slot, st);
  }
  dim3 lel_grid() const { return dim3((a.n + kLelChunk - 1) / kLelChunk, a.B); }
  int sc(int stage, int count, int pc) {
    launch_pdl(k_lsc, a.B, kLscThreads, 0, st, a, stage, count, 0.0, lp->lam_min, pc);
    return cuda_check(cudaGetLastError(), "k_lsc");
  }
  // one BiCGSTAB iteration for every unfinished instance
  int bicg_iteration(int pc) {
    if (half) return bicg_iteration_half();
    int rc;
    const int NC = lp->ncol_cta, NR = (a.n + kLelChunk - 1) / kLelChunk;
    const double* ph = pc ? a.ph : a.p;
    const double* sh = pc ? a.sh : a.s;
    if (pc) {
      if ((rc = strang(CI_PUPD, nullptr, a.ph))) return rc;
    } else {
      launch_pdl(k_lel_pupd, lel_grid(), kLelThreads, 0, st, a);
      if ((rc = cuda_check(cudaGetLastError(), "k_lel_pupd"))) return rc;
    }
    if ((rc = apply(ph, a.v, a.r0, 0))) return rc;
    if ((rc = sc(LS_ALPHA, NC, pc))) return rc;
    if (pc) {
      if ((rc = strang(CI_SUPD, nullptr, a.sh))) return rc;
    } else {
      launch_pdl(k_lel_supd, lel_grid(), kLelThreads, 0, st, a);
      if ((rc = cuda_check(cudaGetLastError(), "k_lel_supd"))) return rc;
    }
    if ((rc = sc(LS_SNORM, pc ? NC : NR, pc))) return rc;
    if ((rc = apply(sh, a.t, a.s, 0))) return rc;
    if ((rc = sc(LS_OMEGA, NC, pc))) return rc;
    launch_pdl(k_lel_xr, lel_grid(), kLelThreads, 0, st, a, ph, sh);
    if ((rc = cuda_check(cudaGetLastError(), "k_lel_xr"))) return rc;
    return sc(LS_REL, NR, pc);
  }
  int dot(const double* u, const double* w, int slot) {
    launch_pdl(k_lel_dot, lel_grid(), kLelThreads, 0, st, a, u, w, slot);
    return cuda_check(cudaGetLastError(), "k_lel_dot");
  }
  // PCG start: r = b, z = P^{-1} r, p = z, rz = r . z
  int cg_start(int pc) {
    int rc;
    const int NR = (a.n + kLelChunk - 1) / kLelChunk;
    launch_pdl(k_lel_copy, lel_grid(), kLelThreads, 0, st, a, a.r, a.r0);
    if ((rc = cuda_check(cudaGetLastError(), "k_lel_copy"))) return rc;
    if (pc) {
      if ((rc = strang(CI_LOAD, a.r, a.p))) return rc;
    } else {
      launch_pdl(k_lel_copy, lel_grid(), kLelThreads, 0, st, a, a.p, a.r);
      if ((rc = cuda_check(cudaGetLastError(), "k_lel_copy"))) return rc;
    }
    if ((rc = dot(a.r, a.p, 0))) return rc;
    return sc(LS_CG_RZ0, NR, pc);
  }
  // one PCG iteration: q = M p, alpha, x/r update, test, z = P^{-1} r, beta, p
  int cg_iteration(int pc) {
    int rc;
    const int NC = lp->ncol_cta, NR = (a.n + kLelChunk - 1) / kLelChunk;
    if ((rc = apply(a.p, a.v, a.p, 0))) return rc;           // q -> v; p.q partials
    if ((rc = sc(LS_CG_ALPHA, NC, pc))) return rc;
    launch_pdl(k_lel_cgxr, lel_grid(), kLelThreads, 0, st, a);
    if ((rc = cuda_check(cudaGetLastError(), "k_lel_cgxr"))) return rc;
    if ((rc = sc(LS_CG_REL, NR, pc))) return rc;
    const double* z = a.r;
    if (pc) {
      if ((rc = strang(CI_LOAD, a.r, a.s))) return rc;       // z -> s
      z = a.s;
    }
    if ((rc = dot(a.r, z, 0))) return rc;
    if ((rc = sc(LS_CG_BETA, NR, pc))) return rc;
    launch_pdl(k_lel_cgp, lel_grid(), kLelThreads, 0, st, a, z);
    return cuda_check(cudaGetLastError(), "k_lel_cgp");
  }
};

// ---- graph-mode loop (TSF_SOLVE_GRAPH, default on)
__global__ void k_lloop_cond(cudaGraphConditionalHandle h, const int* active) {
  pdl_enter();
  cudaGraphSetConditional(h, *active > 0 ? 1u : 0u);
}

// kernel nodes of a captured launch chain, in chain order
int chain_nodes(cudaGraph_t g, std::vector<cudaGraphNode_t>& out) {
  out.clear();
  size_t nr = 0;
  if (cudaGraphGetRootNodes(g, nullptr, &nr) != cudaSuccess || nr != 1)
    return report_error(TSF_E_CUDA, "captured iteration is not a single chain");
  cudaGraphNode_t cur;
  if (cudaGraphGetRootNodes(g, &cur, &nr) != cudaSuccess)
    return report_error(TSF_E_CUDA, "cudaGraphGetRootNodes");
  for (;;) {
    out.push_back(cur);
    // _v2: programmatic (PDL) edges carry edge data; the plain query
    // refuses them (cudaErrorLossyQuery)
    size_t nd = 0;
    if (cudaGraphNodeGetDependentNodes_v2(cur, nullptr, nullptr, &nd) != cudaSuccess)
      return report_error(TSF_E_CUDA, "cudaGraphNodeGetDependentNodes");
    if (nd == 0) break;
    if (nd != 1) return report_error(TSF_E_CUDA, "captured iteration is not a single chain");
    cudaGraphEdgeData ed{};
    if (cudaGraphNodeGetDependentNodes_v2(cur, &cur, &ed, &nd) != cudaSuccess)
      return report_error(TSF_E_CUDA, "cudaGraphNodeGetDependentNodes");
  }
  return 0;
}

Runner make_runner(const LargePlan* lp, int B, cudaStream_t st) {
  Runner R;
  R.lp = lp;
  R.st = st;
  R.lg1 = ilog2i(lp->N1);
  R.lg2 = ilog2i(lp->N2);
  LargeArgs& a = R.a;
  a = LargeArgs{};
  a.n = lp->n;
  a.nt = lp->nt;
  a.B = B;
  a.lt = lp->lt;
  a.Z = lp->Z;
  a.part = lp->part;
  a.np = lp->np;
  const size_t vn = (size_t)lp->cap * lp->n;
  double* w = lp->ws;
  a.r = w;
  a.p = w + vn;
  a.v = w + 2 * vn;
  a.ph = w + 3 * vn;
  a.s = w + 4 * vn;
  a.sh = w + 5 * vn;
  a.t = w + 6 * vn;
  // w + 7 vn: kwork ; w + 8 vn: the Strang spectrum [cap][nt]
  a.pspec = w + 8 * vn;
  a.active = lp->active;
  a.hg = lp->hg;
  a.hg.hspec = lp->Z + (size_t)lp->cap * lp->nt;   // the upper half of Z is free in half mode
  a.hg.pspec2 = reinterpret_cast<double2*>(a.pspec);
  R.lg1h = ilog2i(lp->hg.N1 > 0 ? lp->hg.N1 : 1);
  R.lg2h = ilog2i(lp->hg.N2 > 0 ? lp->hg.N2 : 1);
  return R;
}

}  // namespace

// Rows [0, rows) of a table build spread over the host cores (each row writes
// its own slice; the permuted-table loops were 1.6 s of
// the 2.7 s plan creation at n = 2^24)
template <class F>
static void parallel_rows(int rows, const F& fn) {
  unsigned hw = std::thread::hardware_concurrency();
  const int nt = (int)std::min<unsigned>(hw ? hw : 1, 32u);
  if (nt <= 1 || rows < 4 * nt) {
    for (int r = 0; r < rows; ++r) fn(r);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (int r = t; r < rows; r += nt) fn(r);
    });
  for (auto& x : th) x.join();
}

// smallest n the half-length four-step engine takes (TSF_HLARGE_MIN_N)
static long hlarge_min_n() {
  static long v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_HLARGE_MIN_N");
    v = s ? atol(s) : (1L << 13);
  }
  return v;
}

// ======================================================================
int large_plan_init(LargePlan* lp, int n, int L, const double* symbol_re, const double* lam,
                    int device) {
  const int nt = L / 2;   // transform length (pow2); vectors of n <= nt are zero-padded
  const int lg = ilog2i(nt);
  if ((1L << lg) != nt || lg < 13 || lg > 2 * kLargeMaxLog || n > nt || 2L * n - 1 > L)
    return report_error(TSF_E_UNSUPPORTED,
                        "large-n engine needs a power-of-two embedding L = 2^14..2^25 >= 2n-1");
  if (lam && n != nt)
    return report_error(TSF_E_UNSUPPORTED, "Strang tables need n = L/2 (power-of-two n)");
  *lp = LargePlan{};
  lp->n = n;
  lp->nt = nt;
  // columns short (cheap, G per CTA), rows up to the single-CTA limit 4096;
  // TSF_LARGE_ROWLOG caps log2(N2) lower (experiments: more, shorter rows)
  int rowlog = kLargeMaxLog;
  if (const char* e = getenv("TSF_LARGE_ROWLOG")) {
    const int v = atoi(e);
    if (v >= kLargeMinLog && v <= kLargeMaxLog) rowlog = v;
  }
  lp->N1 = std::max(64, nt >> rowlog);
  if (lp->N1 > (1 << kLargeMaxLog)) lp->N1 = 1 << kLargeMaxLog;
  lp->N2 = nt / lp->N1;
  if (lp->N2 > (1 << kLargeMaxLog) || lp->N2 < (1 << kLargeMinLog)) {
    lp->N1 = std::max(64, nt >> kLargeMaxLog);
    lp->N2 = nt / lp->N1;
  }
  lp->ncol_cta = lp->N2 / col_group_at(ilog2i(lp->N1));
  lp->np = std::max(lp->ncol_cta, (n + kLelChunk - 1) / kLelChunk);
  lp->has_pc = lam != nullptr;
  lp->device = device;
  const int N1 = lp->N1, N2 = lp->N2;
  std::vector<double2> tw1 = twiddle_table(N1), tw2 = twiddle_table(N2);
  std::vector<double2> twN = twiddle_table(nt), twL = twiddle_table(L);
  // permuted spectra: position k1 N2 + k2 holds bin k = k1 + N1 k2
  std::vector<double2> sEO((size_t)nt), lamP(lam ? (size_t)nt : 0);
  auto Ssym = [&](long k) -> double {
    return (double)(0.5L * ((long double)symbol_re[k] + (long double)symbol_re[(L - k) % L]) /
                    (long double)L);
  };
  double lam_min = 1e308;
  parallel_rows(N1, [&](int k1) {
    for (int k2 = 0; k2 < N2; ++k2) {
      const long k = k1 + (long)N1 * k2;
      const size_t pos = (size_t)k1 * N2 + k2;
      sEO[pos] = make_double2(Ssym(2 * k), Ssym(2 * k + 1));
      if (lam) lamP[pos] = make_double2(lam[k], lam[(n - k) % n]);
    }
  });
  if (lam)
    for (int k = 0; k < n; ++k) lam_min = std::min(lam_min, lam[k]);
  lp->lam_min = lam_min;
  // half-length geometry (tsf_hlarge.cuh): H = nt/2 = N1h x N2h, rows <= 2048
  std::vector<double2> tw1h, tw2h, twH, sEh, lamH;
  std::vector<double> sO4;
  const long Hh = nt / 2;
  if (lam && n == nt && Hh >= 64L * 64) {
    // rows up to 2048 points (the row-pair CTA's shared memory);
    // TSF_HLARGE_ROWLOG caps log2(N2h) lower (experiments)
    int hrowlog = 11;
    if (const char* e = getenv("TSF_HLARGE_ROWLOG")) {
      const int v = atoi(e);
      if (v >= 7 && v <= 11) hrowlog = v;
    }
    int N1h = (int)std::max(64L, Hh >> hrowlog);
    if (N1h > (1 << kLargeMaxLog)) N1h = 1 << kLargeMaxLog;
    int N2h = (int)(Hh / N1h);
    lp->half = 1;
    lp->hg.N1 = N1h;
    lp->hg.N2 = N2h;
    lp->ncol_cta_h = N2h / col_group_at(ilog2i(N1h));
    lp->np = std::max(lp->np, lp->ncol_cta_h);
    tw1h = twiddle_table(N1h);
    tw2h = twiddle_table(N2h);
    twH = twiddle_table((int)Hh);
    sEh.resize((size_t)Hh);
    lamH.resize((size_t)2 * Hh);
    sO4.resize((size_t)Hh);
    parallel_rows(N1h, [&](int k1) {
      for (int k2 = 0; k2 < N2h; ++k2) {
        const long k = k1 + (long)N1h * k2;
        const size_t pos = (size_t)k1 * N2h + k2;
        sEh[pos] = make_double2(Ssym(2 * k) * nt, Ssym(2 * (Hh - k)) * nt);
        sO4[pos] = 2.0 * Ssym(4 * k + 1);
        lamH[2 * pos] = make_double2(lam[k], lam[(n - k) % n]);
        lamH[2 * pos + 1] = make_double2(lam[Hh - k], lam[(n - Hh + k) % n]);
      }
    });
  }
  const size_t total = tw1.size() + tw2.size() + twN.size() + twL.size() + sEO.size() + lamP.size() +
                       tw1h.size() + tw2h.size() + twH.size() + sEh.size() + lamH.size() +
                       (sO4.size() + 1) / 2;
  int rc;
  if ((rc = cuda_check(cudaSetDevice(device), "cudaSetDevice"))) return rc;
  if ((rc = cuda_check(cudaMalloc(&lp->tables, total * sizeof(double2)), "cudaMalloc(tables)")))
    return rc;
  double2* cur = lp->tables;
  auto put = [&](const std::vector<double2>& h) -> const double2* {
    if (h.empty()) return nullptr;
    double2* d = cur;
    cur += h.size();
    if (cudaMemcpy(d, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice) != cudaSuccess)
      rc = report_cuda(cudaGetLastError(), "cudaMemcpy(tables)");
    return d;
  };
  lp->lt.tw1 = put(tw1);
  lp->lt.tw2 = put(tw2);
  lp->lt.twN = put(twN);
  lp->lt.twL = put(twL);
  lp->lt.sEO = put(sEO);
  lp->lt.lamP = put(lamP);
  if (lp->half) {
    lp->hg.tw1 = put(tw1h);
    lp->hg.tw2 = put(tw2h);
    lp->hg.twH = put(twH);
    lp->hg.sEh = put(sEh);
    lp->hg.lamH = put(lamH);
    double* d = reinterpret_cast<double*>(cur);
    if (cudaMemcpy(d, sO4.data(), sO4.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      rc = report_cuda(cudaGetLastError(), "cudaMemcpy(tables)");
    lp->hg.sO4 = d;
  }
  return rc;
}

void large_plan_free(LargePlan* lp) {
  if (!lp) return;
  cudaSetDevice(lp->device);
  for (auto& row : lp->loops)
    for (auto& pcs : row)
      for (auto& g : pcs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
      }
  if (lp->cap_stream) cudaStreamDestroy(lp->cap_stream);
  cudaFree(lp->tables);
  cudaFree(lp->ws);
  cudaFree(lp->Z);
  cudaFree(lp->part);
  cudaFree(lp->st);
  cudaFree(lp->active);
  if (lp->h_active) cudaFreeHost(lp->h_active);
  *lp = LargePlan{};
}

int large_reserve(LargePlan* lp, int B) {
  if (B <= lp->cap) return TSF_SUCCESS;
  cudaSetDevice(lp->device);
  cudaFree(lp->ws);
  cudaFree(lp->Z);
  cudaFree(lp->part);
  cudaFree(lp->st);
  lp->ws = nullptr;
  lp->Z = nullptr;
  lp->part = nullptr;
  lp->st = nullptr;
  lp->cap = 0;
  const size_t vn = (size_t)B * lp->n, vt = (size_t)B * lp->nt;
  int rc;
  // 8 Krylov vectors [B][n] + the Strang spectrum [B][nt]
  if ((rc = cuda_check(cudaMalloc(&lp->ws, sizeof(double) * (vn * 8 + vt)), "cudaMalloc(large ws)")))
    return rc;
  if ((rc = cuda_check(cudaMalloc(&lp->Z, sizeof(double2) * vt * 2), "cudaMalloc(large Z)")))
    return rc;
  if ((rc = cuda_check(cudaMalloc(&lp->part, sizeof(double) * (size_t)B * 4 * lp->np),
                       "cudaMalloc(partials)")))
    return rc;
  if ((rc = cuda_check(cudaMalloc(&lp->st, sizeof(LState) * (size_t)B), "cudaMalloc(state)")))
    return rc;
  if (!lp->active && (rc = cuda_check(cudaMalloc(&lp->active, sizeof(int)), "cudaMalloc(active)")))
    return rc;
  if (!lp->h_active &&
      (rc = cuda_check(cudaHostAlloc(&lp->h_active, sizeof(int), cudaHostAllocDefault), "cudaHostAlloc")))
    return rc;
  lp->cap = B;
  return TSF_SUCCESS;
}

int large_matvec(LargePlan* lp, int B, const double* x, double* y, const double* kappa,
                 double shift, cudaStream_t st) {
  int rc = large_reserve(lp, B);
  if (rc) return rc;
  Runner R = make_runner(lp, B, st);
  R.a.kappa = kappa;
  R.a.shift = shift;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (lp->half && half_mode() && lp->n >= hlarge_min_n() && al(x) && al(y) && y != x)
    return R.happly_plain(x, y, R.a.t);
  return R.apply(x, y, nullptr, -1);
}

int large_precond(LargePlan* lp, int B, const double* v, double* z, double shift, double kbar,
                  const double* kbar_dev, cudaStream_t st) {
  int rc = large_reserve(lp, B);
  if (rc) return rc;
  Runner R = make_runner(lp, B, st);
  R.a.shift = shift;
  if (lp->half && half_mode() && lp->n >= hlarge_min_n() &&
      ((reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(z)) & 15) == 0) {
    launch_pdl(k_hspec, dim3((unsigned)((R.a.nt / 2 + kLelChunk - 1) / kLelChunk), B), kLelThreads,
               0, st, R.a, kbar, kbar_dev, 0);
    if ((rc = cuda_check(cudaGetLastError(), "k_hspec"))) return rc;
    return R.hstrang(HF_LOAD, v, z, nullptr);
  }
  launch_pdl(k_lspec, R.lel_grid(), kLelThreads, 0, st, R.a, kbar, kbar_dev, 0);
  if ((rc = cuda_check(cudaGetLastError(), "k_lspec"))) return rc;
  return R.strang(CI_LOAD, v, z);
}

// One graph launch runs every remaining iteration: WHILE(active > 0) { one
// iteration's launch chain ; loop test }.  No host polling, no chunk
// overshoot (the scalar kernels hold max_iters, krylov.py:100).
static int loop_graph(LargePlan* lp, const Runner& R0, int method, int pc, cudaStream_t st) {
  // the column kernels' instantiation depends on the launch size
  // (tsf_large_impl.cuh few_ctas): one cached chain per choice, so a cached
  // node never changes its kernel function
  const int few = few_ctas((long)lp->ncol_cta * R0.a.B) ? 1 : 0;
  LargeLoopGraph& G = lp->loops[method][pc][few + (R0.half ? 2 : 0)];
  int rc;
  if (!lp->cap_stream &&
      (rc = cuda_check(cudaStreamCreateWithFlags(&lp->cap_stream, cudaStreamNonBlocking),
                       "cudaStreamCreate(capture)")))
    return rc;
  Runner R = R0;
  R.st = lp->cap_stream;
  auto record = [&](cudaGraphConditionalHandle h) -> int {
    const int r = method == 1 ? R.cg_iteration(pc) : R.bicg_iteration(pc);
    if (r) return r;
    launch_pdl(k_lloop_cond, 1, 1, 0, R.st, h, lp->active);
    return cuda_check(cudaGetLastError(), "k_lloop_cond");
  };
  if (!G.built) {
    if ((rc = cuda_check(cudaGraphCreate(&G.graph, 0), "cudaGraphCreate"))) return rc;
    if ((rc = cuda_check(cudaGraphConditionalHandleCreate(&G.cond, G.graph, 1,
                                                          cudaGraphCondAssignDefault),
                         "cudaGraphConditionalHandleCreate")))
      return rc;
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = G.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    if ((rc = cuda_check(cudaGraphAddNode(&loop, G.graph, nullptr, 0, &cp), "cudaGraphAddNode")))
      return rc;
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if ((rc = cuda_check(cudaStreamBeginCaptureToGraph(R.st, body, nullptr, nullptr, 0,
                                                       cudaStreamCaptureModeRelaxed),
                         "cudaStreamBeginCaptureToGraph")))
      return rc;
    const int r1 = record(G.cond);
    cudaGraph_t out = nullptr;
    const cudaError_t e = cudaStreamEndCapture(R.st, &out);
    if (r1) return r1;
    if ((rc = cuda_check(e, "cudaStreamEndCapture"))) return rc;
    if ((rc = chain_nodes(body, G.body))) return rc;
    if ((rc = cuda_check(cudaGraphInstantiate(&G.exec, G.graph, 0), "cudaGraphInstantiate")))
      return rc;
    G.built = true;
  } else {
    // re-capture this solve's chain and copy its kernel parameters in
    cudaGraph_t tmp = nullptr;
    if ((rc = cuda_check(cudaStreamBeginCapture(R.st, cudaStreamCaptureModeRelaxed),
                         "cudaStreamBeginCapture")))
      return rc;
    const int r1 = record(G.cond);
    const cudaError_t e = cudaStreamEndCapture(R.st, &tmp);
    if (r1) return r1;
    if ((rc = cuda_check(e, "cudaStreamEndCapture"))) return rc;
    std::vector<cudaGraphNode_t> nodes;
    rc = chain_nodes(tmp, nodes);
    if (!rc && nodes.size() != G.body.size())
      rc = report_error(TSF_E_CUDA, "iteration chain changed shape");
    for (size_t i = 0; !rc && i < nodes.size(); ++i) {
      cudaKernelNodeParams kp{};
      rc = cuda_check(cudaGraphKernelNodeGetParams(nodes[i], &kp), "cudaGraphKernelNodeGetParams");
      if (!rc)
        rc = cuda_check(cudaGraphExecKernelNodeSetParams(G.exec, G.body[i], &kp),
                        "cudaGraphExecKernelNodeSetParams");
    }
    cudaGraphDestroy(tmp);
    if (rc) return rc;
  }
  return cuda_check(cudaGraphLaunch(G.exec, st), "cudaGraphLaunch");
}

// TSF_L2_PERSIST=1 (experiment): keep Z L2-resident through a persisting
// access-policy window when it fits (tsf_large.cuh L2Window)
struct L2Scope {
  explicit L2Scope(const LargePlan* lp, int B) {
    static int on = -1;
    if (on < 0) {
      const char* s = getenv("TSF_L2_PERSIST");
      on = (s && s[0] == '1') ? 1 : 0;
    }
    const size_t bytes = 2 * (size_t)B * lp->nt * sizeof(double2);
    if (!on || bytes > (64u << 20)) return;
    static size_t limit = 0;
    if (limit < bytes && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) == cudaSuccess)
      limit = bytes;
    l2_window().base = lp->Z;
    l2_window().bytes = bytes;
  }
  ~L2Scope() { l2_window() = L2Window{}; }
};

int large_solve(LargePlan* lp, int B, int method, int pc, const KrylovArgs& k, cudaStream_t st) {
  if (method != 0 && method != 1) return report_error(TSF_E_INVALID, "method must be 0 or 1");
  if (pc && !lp->has_pc) return report_error(TSF_E_UNSUPPORTED, "plan has no Strang preconditioner");
  int rc = large_reserve(lp, B);
  if (rc) return rc;
  L2Scope l2(lp, B);
  Runner R = make_runner(lp, B, st);
  LargeArgs& a = R.a;
  KrylovArgs kk = k;
  if (!kk.kappa && !kk.kwork) kk.kwork = lp->ws + 7 * (size_t)lp->cap * lp->n;
  a.r0 = k.rhs;
  a.x = k.x;
  a.kappa = kk.kappa ? kk.kappa : kk.kwork;
  a.shift = k.shift;
  a.tol = k.tol;
  a.max_iters = k.max_iters > 0 ? k.max_iters : 10 * lp->n;
  a.iters = k.iters;
  a.relres = k.relres;
  a.status = k.status;
  a.st = lp->st;
  R.half = method == 0 && pc == 1 && lp->half && half_mode() && lp->n >= hlarge_min_n() &&
           (reinterpret_cast<uintptr_t>(k.rhs) & 15) == 0;
  k_set_int<<<1, 1, 0, st>>>(lp->active, B);
  launch_pdl(k_lel_begin, R.lel_grid(), kLelThreads, 0, st, a, kk);
  if ((rc = cuda_check(cudaGetLastError(), "k_lel_begin"))) return rc;
  launch_pdl(k_lsc, B, kLscThreads, 0, st, a, LS_BEGIN, (a.n + kLelChunk - 1) / kLelChunk, k.kbar,
                                   lp->lam_min, pc);
  if ((rc = cuda_check(cudaGetLastError(), "k_lsc(begin)"))) return rc;
  if (pc && R.half) {
    launch_pdl(k_hspec, dim3((unsigned)((a.nt / 2 + kLelChunk - 1) / kLelChunk), B), kLelThreads, 0,
               st, a, 0.0, (const double*)nullptr, 1);
    if ((rc = cuda_check(cudaGetLastError(), "k_hspec"))) return rc;
  } else if (pc) {
    launch_pdl(k_lspec, R.lel_grid(), kLelThreads, 0, st, a, 0.0, nullptr, 1);
    if ((rc = cuda_check(cudaGetLastError(), "k_lspec"))) return rc;
  }
  if (method == 1 && (rc = R.cg_start(pc))) return rc;
  if (graph_mode()) return loop_graph(lp, R, method, pc, st);
  for (int it = 0; it < a.max_iters; it += kLargeChunk) {
    for (int c = 0; c < kLargeChunk && it + c < a.max_iters; ++c)
      if ((rc = method == 1 ? R.cg_iteration(pc) : R.bicg_iteration(pc))) return rc;
    if ((rc = cuda_check(cudaMemcpyAsync(lp->h_active, lp->active, sizeof(int),
                                         cudaMemcpyDeviceToHost, st), "poll")))
      return rc;
    if ((rc = cuda_check(cudaStreamSynchronize(st), "poll sync"))) return rc;
    if (*lp->h_active == 0) break;
  }
  return TSF_SUCCESS;
}


// ---------------------------------------------------------------- TMA maps
// (tsf_tma.cuh) encoded once per (pointer, shape) and cached: the workspace
// pointers of a plan never move, so a solve's launches hit the cache.
int tma_mode() {
  // TSF_TMA: unset/"1"/"3" both column kernels, "0" none, "fwd"/"2"... per bit
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_TMA");
    if (!s) v = 3;
    else if (!strcmp(s, "fwd")) v = 1;
    else if (!strcmp(s, "inv")) v = 2;
    else v = atoi(s) == 1 ? 3 : atoi(s) & 3;
  }
  return v;
}

int tma_half_mode() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_TMA_HALF");
    if (!s) v = 2;
    else if (!strcmp(s, "fwd")) v = 1;
    else if (!strcmp(s, "inv")) v = 2;
    else v = atoi(s) & 3;
  }
  return v;
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

using MapKey = std::tuple<const void*, unsigned long long, unsigned long long, unsigned long long,
                          unsigned long long, unsigned long long, unsigned, unsigned>;
std::mutex g_map_mu;
std::map<MapKey, CUtensorMap> g_maps;

// 3-D tiled map of fp64 elements: dims {d0, d1, d2}, byte strides of dims 1
// and 2, box {b0, b1, 1}
int encode3(CUtensorMap* m, const void* base, unsigned long long d0, unsigned long long d1,
            unsigned long long d2, unsigned long long s1, unsigned long long s2, unsigned b0,
            unsigned b1) {
  const MapKey key{base, d0, d1, d2, s1, s2, b0, b1};
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto it = g_maps.find(key);
  if (it != g_maps.end()) {
    *m = it->second;
    return 0;
  }
  auto fn = encode_fn();
  if (!fn) return report_error(TSF_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {s1, s2};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return report_error(TSF_E_CUDA, "cuTensorMapEncodeTiled failed");
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = *m;
  return 0;
}
}  // namespace

int tma_map_vector(CUtensorMap* m, const double* base, long n, int N1, int N2, int B, int G) {
  return encode3(m, base, (unsigned long long)N2, (unsigned long long)N1, (unsigned long long)B,
                 (unsigned long long)N2 * 8, (unsigned long long)n * 8, (unsigned)G,
                 (unsigned)std::min(N1, kTmaMaxBox));
}

int tma_map_z(CUtensorMap* m, const double2* Z, int N1, int N2, int B, int G) {
  return encode3(m, Z, 2ULL * N2, (unsigned long long)N1, 2ULL * B, 2ULL * N2 * 8,
                 (unsigned long long)N1 * N2 * 16, 2u * G, (unsigned)std::min(N1, kTmaMaxBox));
}

}  // namespace tsf
