// Half-length four-step engine: the Strang-preconditioned BiCGSTAB level solve
// of a large power-of-two grid (n = 2H, H = N1 x N2 complex points) with every
// transform run as ONE complex transform of length H (see tsf_half.cuh for
// the algebra; toeplitz.py:51-63, 131-136, krylov.py:88-153):
//
//   Strang solve   hcol_fwd (z_m = u_{2m} + i u_{2m+1}, the Krylov vector
//                  update fused) . hrow_strang (row transforms, split step,
//                  filter, half spectrum stored, inverse pre-step, inverse row
//                  transforms) . hcol_inv (q_{2m}, q_{2m+1} stored as one
//                  16-byte word)
//   Toeplitz       hcol_fwd (odd bins: w_m (x_m - i x_{m+H})) . hrow_mv (odd
//   product        rows: FFT . 2 S_{4k+1}/L . IFFT; even rows: pre-step of the
//                  stored Strang spectrum . IFFT, no forward transform) .
//                  hcol_inv (even bins -> scratch vector) . hcol_inv (odd bins,
//                  combine y = d x + kappa (ye + yo), dot partials)
//
// Index maps: time m = N2 t1 + t2, frequency k = k1 + N1 k2 stored at
// k1 N2 + k2.  The split step pairs bin k with H - k, i.e. row k1 with row
// N1 - k1 (element k2 with N2 - 1 - k2; rows 0 and N1/2 pair with
// themselves), so hrow_strang runs the two rows of a pair side by side in one
// CTA and exchanges them through shared memory.
// Against the full-length four-step engine (tsf_large.cuh: six length-n
// complex transforms per half-iteration in three launches each) this moves
// 2.4x fewer transform points through L2/HBM.
#pragma once

#include "tsf_half.cuh"
#include "tsf_large.cuh"

namespace tsf {

template <int N2>
struct HRow {
  static constexpr int E = 8;
  static constexpr int T = N2 / E;
  // row pairs per CTA: one, or as many as fill a warp (N2 = 64: two pairs)
  static constexpr int NP = 2 * T >= 32 ? 1 : 32 / (2 * T);
  static constexpr int BLOCK = 2 * T * NP;
  static constexpr int BUF = 2 * FftPlan<N2, E>::SMEM_ELEMS;
  static constexpr int SMEM = (2 * NP * BUF + tw_table_elems(N2)) * 16;
  static constexpr bool OK = SMEM <= kSmemCap && N2 >= 64;
};

// ------------------------------------------------------------ hcol_fwd
template <int N1, int MB = LCol<N1>::MINB>
__global__ void __launch_bounds__(LCol<N1>::BLOCK, MB)
k_hcol_fwd(LargeArgs a, const double* __restrict__ src, int in_mode,
           const __grid_constant__ ColMaps cm) {
  pdl_enter();
  using C = LCol<N1>;
  constexpr int E = C::E, T = C::T, G = C::G;
  const int N2 = a.hg.N2;
  const long H = (long)N1 * N2;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ double red[4 * 32];
  __shared__ unsigned long long bar;
  const int b = blockIdx.y;
  const int g = threadIdx.x % G, tid = threadIdx.x / G;
  const int t2 = blockIdx.x * G + g;
  double2* smg = sm + g * C::BUF;
  double2* tw1 = sm + G * C::BUF;
  const long off = (long)b * a.n;   // reals
  const long off2 = (long)b * H;    // 16-byte words (n = 2H)
  double2 z[E];
  double part = 0.0;
  if (cm.use) {
    // TMA path (packed modes): up to two [N1 x G] tiles of 16-byte words land
    // in the (not yet used) transform buffers while the CTA stages its
    // twiddles and reads the state — HF_LOAD: src; HF_SUPD: r, v; HF_PUPD:
    // p, v (r by plain loads: it is r0 at the first iteration)
    double2* tile = sm;
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (unsigned)(cm.nv * N1 * G * 16));
      for (int q = 0; q < cm.nv; ++q)
        tma_tile(reinterpret_cast<double*>(tile + q * N1 * G), &cm.v[q], 2 * blockIdx.x * G, N1,
                 2 * G, b, 8, &bar);
    }
    stage_tw<N1>(tw1, a.hg.tw1);
    const LState stv = a.st ? a.st[b] : LState{};
    double2 rr[E];
    if (in_mode == HF_PUPD) {
      const double2* r2 = reinterpret_cast<const double2*>(stv.it == 1 ? a.r0 : a.r);
#pragma unroll
      for (int c = 0; c < E; ++c) rr[c] = r2[off2 + (long)N2 * (tid + c * T) + t2];
    }
    __syncthreads();   // barrier initialised before anyone waits on it
    mbar_wait(&bar, 0);
    if (inst_skip(a, b)) return;
    const double2* r02 = reinterpret_cast<const double2*>(a.r0);
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int t1 = tid + c * T;
      const long m = off2 + (long)N2 * t1 + t2;
      const double2 t0 = tile[t1 * G + g];
      double2 val = t0;
      if (in_mode == HF_PUPD) {
        val = rr[c];
        if (stv.it != 1) {
          const double2 t1v = tile[N1 * G + t1 * G + g];   // v
          const double beta = (stv.rho_new / stv.rho) * (stv.alpha / stv.omega);
          val.x = rr[c].x + beta * (t0.x - stv.omega * t1v.x);
          val.y = rr[c].y + beta * (t0.y - stv.omega * t1v.y);
        }
      } else if (in_mode == HF_SUPD) {
        const double2 l0 = stv.it == 1 ? r02[m] : t0;
        const double2 vv = tile[N1 * G + t1 * G + g];
        val.x = l0.x - stv.alpha * vv.x;
        val.y = l0.y - stv.alpha * vv.y;
        part = fma(val.x, val.x, part);
        part = fma(val.y, val.y, part);
      }
      z[c] = val;
    }
    if (in_mode == HF_PUPD || in_mode == HF_SUPD) {
      double2* dp = reinterpret_cast<double2*>(in_mode == HF_PUPD ? a.p : a.s);
#pragma unroll
      for (int c = 0; c < E; ++c) dp[off2 + (long)N2 * (tid + c * T) + t2] = z[c];
    }
  } else if (in_mode == HF_ODD) {
    double xa[E], xb[E];
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long m = (long)N2 * (tid + c * T) + t2;
      xa[c] = src[off + m];
      xb[c] = src[off + m + H];
    }
    if (inst_skip(a, b)) return;
    stage_tw<N1>(tw1, a.hg.tw1);
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long m = (long)N2 * (tid + c * T) + t2;
      const double2 w = tw_get_g(a.lt.twL, m);
      z[c] = make_double2(fma(w.x, xa[c], w.y * xb[c]), fma(w.y, xa[c], -(w.x * xb[c])));
    }
  } else {
    // operands before the stores (the vectors may alias, tsf_large.cuh)
    const bool upd = in_mode == HF_PUPD || in_mode == HF_SUPD;
    const double2* l0p = reinterpret_cast<const double2*>(upd ? a.r : src);
    const double2* p2 = reinterpret_cast<const double2*>(a.p);
    const double2* v2 = reinterpret_cast<const double2*>(a.v);
    double2 l0[E], l1[E], l2[E];
    const double2 zero = make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long m = off2 + (long)N2 * (tid + c * T) + t2;
      l0[c] = l0p[m];
      l1[c] = upd ? (in_mode == HF_PUPD ? p2[m] : v2[m]) : zero;
      l2[c] = in_mode == HF_PUPD ? v2[m] : zero;
    }
    if (inst_skip(a, b)) return;
    const LState stv = a.st ? a.st[b] : LState{};
    if (upd && stv.it == 1) {   // krylov.py:114-116: the first p (and s) start from r0
      const double2* r02 = reinterpret_cast<const double2*>(a.r0);
#pragma unroll
      for (int c = 0; c < E; ++c) l0[c] = r02[off2 + (long)N2 * (tid + c * T) + t2];
    }
    stage_tw<N1>(tw1, a.hg.tw1);
    double2* dp = reinterpret_cast<double2*>(in_mode == HF_PUPD ? a.p : a.s);
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long m = off2 + (long)N2 * (tid + c * T) + t2;
      double2 val = l0[c];
      if (in_mode == HF_PUPD) {
        if (stv.it != 1) {
          const double beta = (stv.rho_new / stv.rho) * (stv.alpha / stv.omega);
          val.x = l0[c].x + beta * (l1[c].x - stv.omega * l2[c].x);
          val.y = l0[c].y + beta * (l1[c].y - stv.omega * l2[c].y);
        }
        dp[m] = val;
      } else if (in_mode == HF_SUPD) {
        val.x = l0[c].x - stv.alpha * l1[c].x;
        val.y = l0[c].y - stv.alpha * l1[c].y;
        dp[m] = val;
        part = fma(val.x, val.x, part);
        part = fma(val.y, val.y, part);
      }
      z[c] = val;
    }
  }
  if (in_mode == HF_SUPD) {
    part = block_sum1(part, red);
    if (threadIdx.x == 0) a.part[((long)b * 4 + 2) * a.np + blockIdx.x] = part;
  }
  group_fft<N1, E, false>(z, smg, tw1, 0, tid);
  double2 wt[E];
#pragma unroll
  for (int c = 0; c < E; ++c) wt[c] = tw_get_g(a.hg.twH, ((long)t2 * (tid + c * T)) & (H - 1));
  double2* Zc = a.Z + off2;
#pragma unroll
  for (int c = 0; c < E; ++c) Zc[(long)(tid + c * T) * N2 + t2] = cmul(z[c], wt[c]);
}

// ------------------------------------------------------------ hrow_strang
// One CTA = the row pair (k1, N1 - k1) (CTA 0: rows 0 and N1/2, each its own
// mirror): forward row transforms, split step + Strang filter + half spectrum
// + inverse pre-step on the mirror pairs, inverse row transforms.
template <int N2>
__global__ void __launch_bounds__(HRow<N2>::BLOCK, 1) k_hrow_strang(LargeArgs a, int mode) {
  pdl_enter();
  using R = HRow<N2>;
  using PL = FftPlan<N2, 8>;
  constexpr int E = 8, T = R::T;
  const int N1 = a.hg.N1;
  const long H = (long)N1 * N2;
  const int b = blockIdx.y;
  if (inst_skip(a, b)) return;
  extern __shared__ __align__(128) double2 sm[];
  const int gg = threadIdx.x / T, tid = threadIdx.x % T;   // gg: group (pair, side)
  const int g = gg & 1;
  const int cp = blockIdx.x * R::NP + (gg >> 1);
  const int k1 = cp == 0 ? (g ? N1 / 2 : 0) : (g ? N1 - cp : cp);
  double2* smg = sm + gg * R::BUF;
  double2* tw2 = sm + 2 * R::NP * R::BUF;
  double2* row = a.Z + (long)b * H + (long)k1 * N2;
  double2 z[E];
#pragma unroll
  for (int c = 0; c < E; ++c) z[c] = row[tid + c * T];
  stage_tw<N2>(tw2, a.hg.tw2);
  // mode bit 0: the filter is the symbol's even bins (standalone Toeplitz
  // product: sEh / n, shared) instead of the instance's Strang filter;
  // bit 1: also form the even-bin rows of the output's Toeplitz product
  const bool sym = mode & 1, side = mode & 2;
  const double2* spec = sym ? a.hg.sEh + (long)k1 * N2 : a.hg.pspec2 + (long)b * H + (long)k1 * N2;
  const double fs = sym ? 1.0 / (2.0 * (double)H) : 1.0;   // exact (power of two)
  double2 sp[E];
  group_fft<N2, E, false>(z, smg, tw2, 0, tid, [&] {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      sp[c] = spec[tid + c * T];
      sp[c] = make_double2(sp[c].x * fs, sp[c].y * fs);
    }
  });
  double2* xb = smg + ((PL::NPASS - 1) & 1) * PL::SMEM_ELEMS;
#pragma unroll
  for (int c = 0; c < E; ++c) xb[PL::pad(tid + c * T)] = z[c];
  __syncthreads();
  {
    const bool self = cp == 0;
    const double2* pb = (self ? smg : sm + (gg ^ 1) * R::BUF) + ((PL::NPASS - 1) & 1) * PL::SMEM_ELEMS;
    // The filtered spectrum Q = FFT_n(q) / n of the output q is in hand, so the
    // even bins of the NEXT Toeplitz product (of q) are formed here too:
    // pre-step of n S_2k/L . Q into channel 1, transformed after the Strang
    // rows (parked in its own row of channel 1 meanwhile: same thread, same
    // addresses).
    double2* rowe = a.Z + (long)a.B * H + (long)b * H + (long)k1 * N2;
    const double2* se = a.hg.sEh + (long)k1 * N2;
    double2 fe[E];
#pragma unroll
    for (int c = 0; c < E; ++c) fe[c] = side ? ldt(&se[tid + c * T]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k2 = tid + c * T;
      const int k2m = (self && g == 0) ? ((N2 - k2) & (N2 - 1)) : (N2 - 1 - k2);
      const double2 zm = pb[PL::pad(k2m)];
      const long k = k1 + (long)N1 * k2;
      const double2 A = z[c];
      const double2 s = make_double2(A.x + zm.x, A.y - zm.y);
      const double2 d = make_double2(A.x - zm.x, A.y + zm.y);
      const double2 w = tw_get_g(a.lt.twL, 2 * k);              // W_n^k
      const double2 Tt = cmul(w, make_double2(d.y, -d.x));
      const double2 Q = cscale(cadd(s, Tt), 0.5 * sp[c].x);
      const double2 cQm = cscale(csub(s, Tt), 0.5 * sp[c].y);
      z[c] = pack_inverse(Q, cQm, w);
      if (side) rowe[k2] = pack_inverse(cscale(Q, fe[c].x), cscale(cQm, fe[c].y), w);
    }
    group_fft<N2, E, true>(z, smg, tw2, 0, tid);
    if (!side) {   // (uniform over the launch)
#pragma unroll
      for (int c = 0; c < E; ++c) row[tid + c * T] = z[c];
      return;
    }
    double2 ze[E];
#pragma unroll
    for (int c = 0; c < E; ++c) {
      row[tid + c * T] = z[c];
      ze[c] = rowe[tid + c * T];
    }
    group_fft<N2, E, true>(ze, smg, tw2, 0, tid);
#pragma unroll
    for (int c = 0; c < E; ++c) rowe[tid + c * T] = ze[c];
  }
}

// ------------------------------------------------------------ hrow_mv
// Odd-bin rows of the Toeplitz product: forward, 2 S_{4k+1}/L, inverse, in
// place in channel 0 (the even-bin rows were formed by hrow_strang).
template <int N2>
__global__ void __launch_bounds__(LRow<N2>::BLOCK, 1) k_hrow_mv(LargeArgs a) {
  pdl_enter();
  constexpr int E = LRow<N2>::E;
  constexpr int T = LRow<N2>::T;
  const int N1 = a.hg.N1;
  const long H = (long)N1 * N2;
  extern __shared__ double2 sm[];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const bool own = tid < T;
  const int k1 = blockIdx.x;
  double2* tw2 = sm + 2 * FftPlan<N2, E>::SMEM_ELEMS;
  double2 z[E];
  double2* row = a.Z + (long)b * H + (long)k1 * N2;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = row[tid + c * T];
  }
  stage_tw<N2>(tw2, a.hg.tw2);
  double so[E];
  block_fft<N2, E, false>(z, sm, tw2, 0, static_cast<const double2*>(nullptr), [&] {
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) so[c] = a.hg.sO4[(long)k1 * N2 + tid + c * T];
    }
  });
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = cscale(z[c], so[c]);
  }
  block_fft<N2, E, true>(z, sm, tw2, 0);
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) row[tid + c * T] = z[c];
  }
}

// ------------------------------------------------------------ hcol_inv
template <int N1, int MB = LCol<N1>::MINB>
__global__ void __launch_bounds__(LCol<N1>::BLOCK, MB)
k_hcol_inv(LargeArgs a, double* __restrict__ dst, int out_mode, double* __restrict__ dst1,
           const double* __restrict__ xin, const double* __restrict__ ye,
           const double* __restrict__ w1, int pslot, const __grid_constant__ ColMaps cm) {
  pdl_enter();
  using C = LCol<N1>;
  constexpr int E = C::E, T = C::T, G = C::G;
  const int N2 = a.hg.N2;
  const long H = (long)N1 * N2;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ double red[4 * 32];
  __shared__ unsigned long long bar;
  const int b = blockIdx.y;
  if (inst_skip(a, b)) return;
  const int g = threadIdx.x % G, tid = threadIdx.x / G;
  const int t2 = blockIdx.x * G + g;
  double2* smg = sm + g * C::BUF;
  double2* tw1 = sm + G * C::BUF;
  // HO_PACK: grid.z = 2 runs both channels (Strang output -> dst, the even
  // bins of its Toeplitz product -> dst1)
  const int ch = blockIdx.z;
  // the channel's [N1 x G] tile of Z by TMA (tsf_tma.cuh) into the transform
  // buffers, free until the transform starts: no extra shared memory
  double2* ztile = sm;
  if (cm.use && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (unsigned)(N1 * G * 16));
    tma_tile(reinterpret_cast<double*>(ztile), &cm.z, 2 * blockIdx.x * G, N1, 2 * G,
             ch * a.B + b, 8, &bar);
  }
  stage_tw<N1>(tw1, a.hg.tw1);
  const long off = (long)b * a.n;
  const long off2 = (long)b * H;
  const double2* Zc = a.Z + (long)ch * a.B * H + off2;
  double2 z[E];
  if (cm.use) {
    __syncthreads();   // barrier initialised before anyone waits on it
    mbar_wait(&bar, 0);
  }
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const int k1 = tid + c * T;
    const double2 w = tw_get_g(a.hg.twH, ((long)t2 * k1) & (H - 1));
    z[c] = cmulc(cm.use ? ztile[k1 * G + g] : Zc[(long)k1 * N2 + t2], w);
  }
  group_fft<N1, E, true>(z, smg, tw1, 0, tid);
  if (out_mode == HO_PACK) {
    double2* d2 = reinterpret_cast<double2*>(ch ? dst1 : dst) + off2;
#pragma unroll
    for (int c = 0; c < E; ++c) d2[(long)N2 * (tid + c * T) + t2] = z[c];
    return;
  }
  // HO_ODD: y_m = d x_m + kappa_m (ye_m + Re(conj(w_m) g_m)),
  //         y_{m+H} = d x_{m+H} + kappa_{m+H} (ye_{m+H} - Im(conj(w_m) g_m))
  Vals<2> pr;
  pr.v[0] = pr.v[1] = 0.0;
  constexpr int HH = E / 2;
#pragma unroll
  for (int c0 = 0; c0 < E; c0 += HH) {
    double2 wm[HH];
    double ya[HH], yb[HH], xa[HH], xb[HH], ka[HH], kb[HH], wa[HH], wb[HH];
#pragma unroll
    for (int q = 0; q < HH; ++q) {
      const long m = (long)N2 * (tid + (c0 + q) * T) + t2;
      wm[q] = tw_get_g(a.lt.twL, m);
      ya[q] = ye[off + m];
      yb[q] = ye[off + m + H];
      xa[q] = a.kappa ? xin[off + m] : 0.0;
      xb[q] = a.kappa ? xin[off + m + H] : 0.0;
      ka[q] = a.kappa ? a.kappa[off + m] : 0.0;
      kb[q] = a.kappa ? a.kappa[off + m + H] : 0.0;
      wa[q] = w1 ? w1[off + m] : 0.0;
      wb[q] = w1 ? w1[off + m + H] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < HH; ++q) {
      const int c = c0 + q;
      const long m = (long)N2 * (tid + c * T) + t2;
      const double2 w = wm[q];
      const double axa = ya[q] + fma(w.x, z[c].x, w.y * z[c].y);
      const double axb = yb[q] - fma(w.x, z[c].y, -(w.y * z[c].x));
      const double y0 = a.kappa ? fma(a.shift, xa[q], ka[q] * axa) : axa;
      const double y1 = a.kappa ? fma(a.shift, xb[q], kb[q] * axb) : axb;
      dst[off + m] = y0;
      dst[off + m + H] = y1;
      pr.v[0] = fma(y0, y0, pr.v[0]);
      pr.v[0] = fma(y1, y1, pr.v[0]);
      if (w1) {
        pr.v[1] = fma(y0, wa[q], pr.v[1]);
        pr.v[1] = fma(y1, wb[q], pr.v[1]);
      }
    }
  }
  if (pslot >= 0) {
    pr = block_sum<2>(pr, red);
    if (threadIdx.x == 0) {
      a.part[((long)b * 4 + pslot) * a.np + blockIdx.x] = pr.v[0];
      a.part[((long)b * 4 + pslot + 1) * a.np + blockIdx.x] = pr.v[1];
    }
  }
}

}  // namespace tsf
