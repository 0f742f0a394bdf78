// Fused SOE history update + next-level right-hand side (HBM streaming).
//
// For every instance b and grid point i, in one pass over W[b, :, i]:
//   push  (soe.py:209-225, scheme.py:290):
//     du_i  = (u_i - uprev_i) / tau_push
//     W_ji <- (W_ji * decay_j) + (coef_j * du_i)        decay_j = e^{-s_j tau},
//                                                       coef_j  = -expm1(-s_j tau)/s_j
//   history term of the NEXT level (scheme.py:281-282, == soe.py:245):
//     H_i   = sum_j hcoef_j * W_ji                      hcoef_j = w_j e^{-s_j tau_next}
//   right-hand side (scheme.py:283-284):
//     rhs_i = f_i + (a_next * u_i - H_i) / G            f_i = sum_q fmode_q[i] * fcoef_q
// The push reproduces numpy's rounding exactly (no FMA contraction, true
// division), so W is bit-identical to the reference given identical u; the
// H reduction order is the only difference (the reference uses a BLAS GEMV).
//
// Layout: W is [B][nexp][n] (each exponential's accumulator row contiguous,
// soe.py:82,87); a thread owns two adjacent i (one 16-byte vector) and
// walks j, so every warp access is a fully coalesced 512-byte transaction.
// Algorithmic bytes per instance: 16*nexp*n (W read+write) + 40 n.
#pragma once

#include "tsf_common.cuh"

namespace tsf {

constexpr int kSoeThreads = 128;  // threads per CTA, 2 points each

struct SoeArgs {
  int n;
  int nexp;
  double* W;              // [B][nexp][n]
  const double* u;        // u^{m}   (the level just solved)          [B][n]
  const double* uprev;    // u^{m-1}                                  [B][n]
  double tau_push;
  const double* decay;    // [nexp]
  const double* coef;     // [nexp]
  const double* hcoef;    // [nexp]
  int do_push;            // 0: W unchanged (read only)
  int w_zero;             // 1: W is known to be all zero (first level): skip W traffic
  int do_rhs;
  double a_next;          // a_{m+1}
  double G;               // Gamma(1-gamma)
  const double* fmodes;   // mode q of instance b at fmodes + q*fq_stride + b*fb_stride
  long fq_stride;
  long fb_stride;
  int nf;
  double fcoef[4];
  const double* f;        // alternatively a full f [B][n] (nf == 0 && f != null)
  double* rhs;            // [B][n]
};

// Per-level coefficient rows into shared memory: decay | coef | hcoef.
TSF_D void soe_load_tabs(const SoeArgs& a, double* tabs) {
  const int nexp = a.nexp;
  for (int j = threadIdx.x; j < nexp; j += blockDim.x) {
    tabs[j] = a.decay ? a.decay[j] : 0.0;
    tabs[nexp + j] = a.coef ? a.coef[j] : 0.0;
    tabs[2 * nexp + j] = a.hcoef ? a.hcoef[j] : 0.0;
  }
}

// The whole update for grid points i0, i0+1 of instance b.
template <int UNROLL>
TSF_D void soe_pair(const SoeArgs& a, const double* tabs, int b, int i0) {
  const int n = a.n;
  const int nexp = a.nexp;
  const bool pair = (i0 + 1 < n) && ((n & 1) == 0);
  const long vbase = (long)b * n + i0;
  auto ld2 = [&](const double* p) -> double2 {
    if (pair) return *reinterpret_cast<const double2*>(p + vbase);
    return make_double2(p[vbase], (i0 + 1 < n) ? p[vbase + 1] : 0.0);
  };
  double2 du = make_double2(0.0, 0.0);
  double2 un = make_double2(0.0, 0.0);
  if (a.do_push || a.do_rhs) un = ld2(a.u);
  if (a.do_push) {
    const double2 up = ld2(a.uprev);
    du.x = __ddiv_rn(__dsub_rn(un.x, up.x), a.tau_push);
    du.y = __ddiv_rn(__dsub_rn(un.y, up.y), a.tau_push);
  }
  double2 H = make_double2(0.0, 0.0);
  if (!a.w_zero) {
    double* Wp = a.W + (long)b * nexp * n + i0;
    const double* dec = tabs;
    const double* cof = tabs + nexp;
    const double* hc = tabs + 2 * nexp;
    int j = 0;
    if (pair) {
      for (; j + UNROLL <= nexp; j += UNROLL) {
        double2 w[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
          w[u] = __ldcs(reinterpret_cast<const double2*>(Wp + (long)(j + u) * n));
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          if (a.do_push) {
            const double dj = dec[j + u], cj = cof[j + u];
            w[u].x = __dadd_rn(__dmul_rn(w[u].x, dj), __dmul_rn(cj, du.x));
            w[u].y = __dadd_rn(__dmul_rn(w[u].y, dj), __dmul_rn(cj, du.y));
            __stcs(reinterpret_cast<double2*>(Wp + (long)(j + u) * n), w[u]);
          }
          H.x = fma(hc[j + u], w[u].x, H.x);
          H.y = fma(hc[j + u], w[u].y, H.y);
        }
      }
    }
    for (; j < nexp; ++j) {
      double* row = Wp + (long)j * n;
      double w0 = row[0];
      double w1 = (i0 + 1 < n) ? row[1] : 0.0;
      if (a.do_push) {
        w0 = __dadd_rn(__dmul_rn(w0, dec[j]), __dmul_rn(cof[j], du.x));
        w1 = __dadd_rn(__dmul_rn(w1, dec[j]), __dmul_rn(cof[j], du.y));
        row[0] = w0;
        if (i0 + 1 < n) row[1] = w1;
      }
      H.x = fma(hc[j], w0, H.x);
      H.y = fma(hc[j], w1, H.y);
    }
  } else if (a.do_push) {
    // W was zero: the pushed state is coef_j * du (exactly numpy's 0*d + c*du)
    double* Wp = a.W + (long)b * nexp * n + i0;
    for (int j = 0; j < nexp; ++j) {
      double w0 = __dadd_rn(0.0, __dmul_rn(tabs[nexp + j], du.x));
      double w1 = __dadd_rn(0.0, __dmul_rn(tabs[nexp + j], du.y));
      double* row = Wp + (long)j * n;
      if (pair) {
        __stcs(reinterpret_cast<double2*>(row), make_double2(w0, w1));
      } else {
        row[0] = w0;
        if (i0 + 1 < n) row[1] = w1;
      }
      H.x = fma(tabs[2 * nexp + j], w0, H.x);
      H.y = fma(tabs[2 * nexp + j], w1, H.y);
    }
  }
  if (a.do_rhs) {
    double2 f = make_double2(0.0, 0.0);
    if (a.nf > 0) {
      for (int q = 0; q < a.nf; ++q) {
        const double* fq = a.fmodes + q * a.fq_stride + (long)b * a.fb_stride - (long)b * n;
        const double2 m = ld2(fq);
        f.x = __dadd_rn(f.x, __dmul_rn(m.x, a.fcoef[q]));
        f.y = __dadd_rn(f.y, __dmul_rn(m.y, a.fcoef[q]));
      }
    } else if (a.f) {
      f = ld2(a.f);
    }
    double2 r;
    r.x = __dadd_rn(f.x, __ddiv_rn(__dsub_rn(__dmul_rn(a.a_next, un.x), H.x), a.G));
    r.y = __dadd_rn(f.y, __ddiv_rn(__dsub_rn(__dmul_rn(a.a_next, un.y), H.y), a.G));
    if (pair) {
      *reinterpret_cast<double2*>(a.rhs + vbase) = r;
    } else {
      a.rhs[vbase] = r.x;
      if (i0 + 1 < n) a.rhs[vbase + 1] = r.y;
    }
  }
}

template <int UNROLL>
__global__ void __launch_bounds__(kSoeThreads)
k_soe_push_rhs(SoeArgs a) {
  extern __shared__ double tabs[];  // 3*nexp: decay, coef, hcoef
  soe_load_tabs(a, tabs);
  __syncthreads();
  const int chunks = (a.n + 2 * kSoeThreads - 1) / (2 * kSoeThreads);
  const int b = blockIdx.x / chunks;
  const int i0 = 2 * ((blockIdx.x % chunks) * kSoeThreads + threadIdx.x);
  if (i0 >= a.n) return;
  soe_pair<UNROLL>(a, tabs, b, i0);
}

// Epilogue of a converged instance's level solve (the instance's CTA streams
// its own W rows: push of this level + history term/RHS of the next one), so
// the HBM-bound SOE pass overlaps other instances' transform work.
TSF_D void soe_instance_epilogue(const SoeArgs& a, double* tabs, int b) {
  __syncthreads();  // the solve's final x writes and last uses of `tabs` memory
  soe_load_tabs(a, tabs);
  __syncthreads();
  for (int i0 = 2 * threadIdx.x; i0 < a.n; i0 += 2 * blockDim.x) soe_pair<4>(a, tabs, b, i0);
}

}  // namespace tsf
