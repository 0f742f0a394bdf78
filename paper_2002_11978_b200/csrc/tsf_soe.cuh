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

// ---------------------------------------------------------------- blocked
// Blocked SOE schedule of the march (tsf_fids_march, K = soe_block > 1): the
// W pass runs once per K levels instead of once per level.  With W^k the
// state after the push of level k, d_j(l) = e^{-s_j tau_l}, c_j(l) the push
// coefficient and h_j(m) = w_j e^{-s_j tau_m}, for a block base mb and
// mb < m <= mb + K:
//   W^{m-1} = [prod_{l=mb+1}^{m-1} d(l)] W^{mb} + sum_{i=mb+1}^{m-1} [prod_{l=i+1}^{m-1} d(l)] c(i) du^i
//   H^m     = sum_j alpha_j(m) W_j^{mb} + sum_{i=mb+1}^{m-1} beta(m, i) du^i
//   alpha_j(m) = h_j(m) prod_{l=mb+1}^{m-1} d_j(l),
//   beta(m, i) = sum_j h_j(m) [prod_{l=i+1}^{m-1} d_j(l)] c_j(i)      (host tables)
// so one pass over W at the base gives the W-part G_m of every history term
// of the block, and each level adds a short combination of the block's du
// vectors.  The pass advances W by the K pushes of the block with the
// reference's own recurrence, in registers (w <- (w d) + (c du), no FMA), so
// W at every block base is bit-identical to the per-level schedule; only the
// history term's summation order differs (as it already does against the
// reference's BLAS GEMV).  HBM traffic per level: 16 N_exp n / K + O(K n)
// instead of 16 N_exp n.
constexpr int kSoeMaxBlock = 16;

struct SoeBlockArgs {
  int n, nexp, B;
  double* W;               // [B][nexp][n]: W^{mb_prev} in, W^{mb} out
  const double* u_cur;     // u^{mb}
  const double* u_prev;    // u^{mb-1}
  double tau_cur;          // tau_{mb}
  const double* du_ring;   // [K][B][n]: du^i at slot (i-1) % K
  int K;
  int mb;                  // new base level
  int ka;                  // pushes to apply: levels mb-ka+1 .. mb (0: none)
  int w_zero;              // W^{mb_prev} == 0 (not read)
  const double* push_tab;  // soe_tab rows of the pushed levels: level l at (l-1)*3*nexp
  int kn;                  // history levels of the new block: mb+1 .. mb+kn (0: none)
  const double* alpha;     // [M][nexp]: alpha_j(m) at (m-1)*nexp
  double* g_ring;          // [K][B][n]: G_m at slot (m-1) % K  (m >= mb+2)
  // RHS of level mb+1 (kn >= 1): f + (a u^{mb} - G_{mb+1}) / G
  double a_next, G;
  const double* fmodes;
  long fq_stride, fb_stride;
  int nf;
  double fcoef[4];
  double* rhs;
};

// shared tables: [ka][nexp] (d, c) pairs | [kn][nexp] alpha
template <int KMAX>
__global__ void __launch_bounds__(kSoeThreads) k_soe_block(SoeBlockArgs a) {
  extern __shared__ double sh[];
  const int n = a.n, nexp = a.nexp, K = a.K, ka = a.ka, kn = a.kn;
  double2* dc = reinterpret_cast<double2*>(sh);          // [ka][nexp]
  double* al = sh + 2 * ka * nexp;                       // [kn][nexp]
  for (int t = threadIdx.x; t < ka * nexp; t += blockDim.x) {
    const int l = t / nexp, j = t % nexp;
    const double* row = a.push_tab + (size_t)(a.mb - ka + l) * 3 * nexp;  // level mb-ka+1+l
    dc[t] = make_double2(row[j], row[nexp + j]);
  }
  for (int t = threadIdx.x; t < kn * nexp; t += blockDim.x)
    al[t] = a.alpha[(size_t)(a.mb + t / nexp) * nexp + t % nexp];          // level mb+1+t/nexp
  __syncthreads();
  const int chunks = (n + 2 * kSoeThreads - 1) / (2 * kSoeThreads);
  const int b = blockIdx.x / chunks;
  const int i0 = 2 * ((blockIdx.x % chunks) * kSoeThreads + threadIdx.x);
  if (i0 >= n) return;
  const bool pair = (i0 + 1 < n) && ((n & 1) == 0);
  const long vb = (long)b * n + i0;
  const long vn = (long)a.B * n;
  auto ld2 = [&](const double* p) -> double2 {
    if (pair) return *reinterpret_cast<const double2*>(p + vb);
    return make_double2(p[vb], (i0 + 1 < n) ? p[vb + 1] : 0.0);
  };
  // du^i of the pushed levels: ring slots, the last one (level mb) from u
  double2 du[KMAX];
#pragma unroll
  for (int l = 0; l < KMAX; ++l) {
    du[l] = make_double2(0.0, 0.0);
    if (l < ka) {
      const int lev = a.mb - ka + 1 + l;
      if (lev == a.mb) {
        const double2 uc = ld2(a.u_cur), up = ld2(a.u_prev);
        du[l].x = __ddiv_rn(__dsub_rn(uc.x, up.x), a.tau_cur);
        du[l].y = __ddiv_rn(__dsub_rn(uc.y, up.y), a.tau_cur);
      } else {
        du[l] = ld2(a.du_ring + (long)((lev - 1) % K) * vn);
      }
    }
  }
  double2 g[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) g[k] = make_double2(0.0, 0.0);
  double* Wp = a.W + (long)b * nexp * n + i0;
  const bool need_w = ka > 0 || !a.w_zero;   // else W^{mb} = 0: G = 0
  if (need_w) {
    for (int j = 0; j < nexp; ++j) {
      double2 w = make_double2(0.0, 0.0);
      if (!a.w_zero) {
        if (pair) w = __ldcs(reinterpret_cast<const double2*>(Wp + (long)j * n));
        else w = make_double2(Wp[(long)j * n], (i0 + 1 < n) ? Wp[(long)j * n + 1] : 0.0);
      }
      if (ka > 0) {
#pragma unroll
        for (int l = 0; l < KMAX; ++l) {
          if (l < ka) {
            const double2 q = dc[l * nexp + j];   // (decay, coef) of the pushed level
            w.x = __dadd_rn(__dmul_rn(w.x, q.x), __dmul_rn(q.y, du[l].x));
            w.y = __dadd_rn(__dmul_rn(w.y, q.x), __dmul_rn(q.y, du[l].y));
          }
        }
        if (pair) {
          __stcs(reinterpret_cast<double2*>(Wp + (long)j * n), w);
        } else {
          Wp[(long)j * n] = w.x;
          if (i0 + 1 < n) Wp[(long)j * n + 1] = w.y;
        }
      }
#pragma unroll
      for (int k = 0; k < KMAX; ++k) {
        if (k < kn) {
          const double c = al[k * nexp + j];
          g[k].x = fma(c, w.x, g[k].x);
          g[k].y = fma(c, w.y, g[k].y);
        }
      }
    }
  }
  auto st2 = [&](double* p, double2 v) {
    if (pair) {
      *reinterpret_cast<double2*>(p + vb) = v;
    } else {
      p[vb] = v.x;
      if (i0 + 1 < n) p[vb + 1] = v.y;
    }
  };
#pragma unroll
  for (int k = 1; k < KMAX; ++k)
    if (k < kn) st2(a.g_ring + (long)((a.mb + k) % K) * vn, g[k]);   // level mb+1+k, slot (m-1)%K
  if (kn >= 1) {
    const double2 u = ld2(a.u_cur);
    double2 f = make_double2(0.0, 0.0);
    for (int q = 0; q < a.nf; ++q) {
      const double* fq = a.fmodes + q * a.fq_stride + (long)b * a.fb_stride - (long)b * n;
      const double2 m = ld2(fq);
      f.x = __dadd_rn(f.x, __dmul_rn(m.x, a.fcoef[q]));
      f.y = __dadd_rn(f.y, __dmul_rn(m.y, a.fcoef[q]));
    }
    double2 r;
    r.x = __dadd_rn(f.x, __ddiv_rn(__dsub_rn(__dmul_rn(a.a_next, u.x), g[0].x), a.G));
    r.y = __dadd_rn(f.y, __ddiv_rn(__dsub_rn(__dmul_rn(a.a_next, u.y), g[0].y), a.G));
    st2(a.rhs, r);
  }
}

// Full passes (ka = kn = K, n even): K a template parameter, no predicates,
// the per-exponential coefficients interleaved in shared memory so one
// broadcast LDS.128 feeds a (decay, coef) pair or two alphas.  The generic
// kernel above issued ~190 instructions per exponential and point pair
// (ncu: issue-bound at 61%, 10-16 ms per pass); this one ~80.
constexpr int kSoeRing = 12;   // cp.async W-row slots per thread (k_soe_block_full, PD = 0)
template <int K, bool WZERO, int PD = 4>
__global__ void __launch_bounds__(kSoeThreads) k_soe_block_full(SoeBlockArgs a) {
  static_assert(K % 2 == 0, "K even");
  extern __shared__ double2 shc[];
  const int n = a.n, nexp = a.nexp;
  double2* dc = shc;                 // [nexp][K]   (d_l, c_l), level mb-K+1+l
  double2* al = shc + nexp * K;      // [nexp][K/2] (alpha_{2q}, alpha_{2q+1}), level mb+1+k
  for (int t = threadIdx.x; t < nexp * K; t += blockDim.x) {
    const int j = t / K, l = t % K;
    const double* row = a.push_tab + (size_t)(a.mb - K + l) * 3 * nexp;
    dc[t] = make_double2(row[j], row[nexp + j]);
  }
  for (int t = threadIdx.x; t < nexp * (K / 2); t += blockDim.x) {
    const int j = t / (K / 2), q = t % (K / 2);
    al[t] = make_double2(a.alpha[(size_t)(a.mb + 2 * q) * nexp + j],
                         a.alpha[(size_t)(a.mb + 2 * q + 1) * nexp + j]);
  }
  __syncthreads();
  const int chunks = (n + 2 * kSoeThreads - 1) / (2 * kSoeThreads);
  const int b = blockIdx.x / chunks;
  const int i0 = 2 * ((blockIdx.x % chunks) * kSoeThreads + threadIdx.x);
  if (i0 >= n) return;
  const long vb = (long)b * n + i0;
  const long vn = (long)a.B * n;
  auto ld2 = [&](const double* p) { return *reinterpret_cast<const double2*>(p + vb); };
  double2 du[K];
#pragma unroll
  for (int l = 0; l < K - 1; ++l) du[l] = ld2(a.du_ring + (long)((a.mb - K + l) % a.K) * vn);
  {
    const double2 uc = ld2(a.u_cur), up = ld2(a.u_prev);
    du[K - 1].x = __ddiv_rn(__dsub_rn(uc.x, up.x), a.tau_cur);
    du[K - 1].y = __ddiv_rn(__dsub_rn(uc.y, up.y), a.tau_cur);
  }
  double2 g[K];
#pragma unroll
  for (int k = 0; k < K; ++k) g[k] = make_double2(0.0, 0.0);
  double2* Wp = reinterpret_cast<double2*>(a.W + (long)b * nexp * n + i0);
  const long rs = n / 2;   // row stride in double2
  // W rows are loaded PD rows ahead: at 4 CTAs x 128 threads per SM (the
  // register budget of 2K accumulators + K du pairs) one row in flight per
  // thread kept ~16 KB per SM in flight — half the HBM rate (ncu, 12.6 ms
  // per pass); PD = 4 keeps ~64 KB per SM in flight.
  // PD == 0: the rows go through a per-thread cp.async ring of kSoeRing
  // slots in shared memory instead (no registers held; ~12 rows ahead).
  constexpr bool RING = (PD == 0) && !WZERO;
  constexpr int PR = PD > 0 ? PD : 1;
  double2* ring = al + nexp * (K / 2) + threadIdx.x;   // slot s at ring[s * kSoeThreads]
  double2 wb[PR];
  if constexpr (RING) {
#pragma unroll
    for (int p = 0; p < kSoeRing - 1; ++p) {
      if (p < nexp) cp_async16(ring + p * kSoeThreads, Wp + p * rs);
      cp_async_commit();
    }
  } else {
#pragma unroll
    for (int p = 0; p < PR; ++p)
      wb[p] = (!WZERO && p < nexp) ? __ldcs(Wp + p * rs) : make_double2(0.0, 0.0);
  }
  for (int j0 = 0; j0 < nexp; j0 += PR) {
#pragma unroll
  for (int p = 0; p < PR; ++p) {
    const int j = j0 + p;
    if (j >= nexp) break;
    double2 w;
    if constexpr (RING) {
      const int jn = j + kSoeRing - 1;
      if (jn < nexp) cp_async16(ring + (jn % kSoeRing) * kSoeThreads, Wp + jn * rs);
      cp_async_commit();
      cp_async_wait<kSoeRing - 1>();   // this thread's row j has landed
      w = ring[(j % kSoeRing) * kSoeThreads];
    } else {
      w = wb[p];
      if (!WZERO && j + PR < nexp) wb[p] = __ldcs(Wp + (j + PR) * rs);
    }
    const double2* q = dc + j * K;
#pragma unroll
    for (int l = 0; l < K; ++l) {
      const double2 c = q[l];
      w.x = __dadd_rn(__dmul_rn(w.x, c.x), __dmul_rn(c.y, du[l].x));
      w.y = __dadd_rn(__dmul_rn(w.y, c.x), __dmul_rn(c.y, du[l].y));
    }
    __stcs(Wp + j * rs, w);
    const double2* h = al + j * (K / 2);
#pragma unroll
    for (int k2 = 0; k2 < K / 2; ++k2) {
      const double2 c = h[k2];
      g[2 * k2].x = fma(c.x, w.x, g[2 * k2].x);
      g[2 * k2].y = fma(c.x, w.y, g[2 * k2].y);
      g[2 * k2 + 1].x = fma(c.y, w.x, g[2 * k2 + 1].x);
      g[2 * k2 + 1].y = fma(c.y, w.y, g[2 * k2 + 1].y);
    }
  }
  }
#pragma unroll
  for (int k = 1; k < K; ++k)
    *reinterpret_cast<double2*>(a.g_ring + (long)((a.mb + k) % a.K) * vn + vb) = g[k];
  const double2 u = ld2(a.u_cur);
  double2 f = make_double2(0.0, 0.0);
  for (int qq = 0; qq < a.nf; ++qq) {
    const double* fq = a.fmodes + qq * a.fq_stride + (long)b * a.fb_stride - (long)b * n;
    const double2 m = ld2(fq);
    f.x = __dadd_rn(f.x, __dmul_rn(m.x, a.fcoef[qq]));
    f.y = __dadd_rn(f.y, __dmul_rn(m.y, a.fcoef[qq]));
  }
  double2 r;
  r.x = __dadd_rn(f.x, __ddiv_rn(__dsub_rn(__dmul_rn(a.a_next, u.x), g[0].x), a.G));
  r.y = __dadd_rn(f.y, __ddiv_rn(__dsub_rn(__dmul_rn(a.a_next, u.y), g[0].y), a.G));
  *reinterpret_cast<double2*>(a.rhs + vb) = r;
}

// Level m of a block (mb + 2 <= m <= mb + K): du^{m-1} (stored in the ring)
// and rhs^m = f + (a u^{m-1} - (G_m + sum_{i=mb+1}^{m-1} beta(m, i) du^i)) / G.
struct SoeLevelArgs {
  int n, B, K, m, mb;
  const double* u1;        // u^{m-1}
  const double* u2;        // u^{m-2}
  double tau1;             // tau_{m-1}
  double* du_ring;
  const double* g_ring;
  double beta[kSoeMaxBlock];   // beta(m, mb+1+q), q < m-1-mb
  double a_m, G;
  const double* fmodes;
  long fq_stride, fb_stride;
  int nf;
  double fcoef[4];
  double* rhs;
};

// Two adjacent points per thread (16-byte accesses), grid (chunks, B); every
// load is issued before the du^{m-1} store (the ring is read and written in
// the same kernel, so the store would otherwise order the later loads).
static __global__ void __launch_bounds__(256) k_soe_level(SoeLevelArgs a) {
  const int n = a.n, b = blockIdx.y;
  const int i0 = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i0 >= n) return;
  const long vn = (long)a.B * n;
  const long e = (long)b * n + i0;
  const bool pair = (n & 1) == 0;   // else one point per thread-slot pair, scalar path
  const int np = pair ? 2 : ((i0 + 1 < n) ? 2 : 1);
  double u1[2], u2[2], H[2], f[2];
  const int nq = a.m - 1 - a.mb;    // du^{mb+1} .. du^{m-1}
  double dq[kSoeMaxBlock - 1][2];
  for (int c = 0; c < np; ++c) {
    u1[c] = a.u1[e + c];
    u2[c] = a.u2[e + c];
    H[c] = a.g_ring[(long)((a.m - 1) % a.K) * vn + e + c];   // G_m
    f[c] = 0.0;
  }
#pragma unroll
  for (int q = 0; q < kSoeMaxBlock - 1; ++q)
    if (q < nq - 1)
      for (int c = 0; c < np; ++c) dq[q][c] = a.du_ring[(long)((a.mb + q) % a.K) * vn + e + c];
  for (int qq = 0; qq < a.nf; ++qq)
    for (int c = 0; c < np; ++c)
      f[c] = __dadd_rn(f[c], __dmul_rn(a.fmodes[qq * a.fq_stride + (long)b * a.fb_stride + i0 + c],
                                       a.fcoef[qq]));
  for (int c = 0; c < np; ++c) {
    const double du = __ddiv_rn(__dsub_rn(u1[c], u2[c]), a.tau1);
    double h = H[c];
#pragma unroll
    for (int q = 0; q < kSoeMaxBlock - 1; ++q)
      if (q < nq - 1) h = fma(a.beta[q], dq[q][c], h);
    h = fma(a.beta[nq - 1], du, h);
    a.rhs[e + c] = __dadd_rn(f[c], __ddiv_rn(__dsub_rn(__dmul_rn(a.a_m, u1[c]), h), a.G));
    a.du_ring[(long)((a.m - 2) % a.K) * vn + e + c] = du;     // du^{m-1}, slot (m-2) % K
  }
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
