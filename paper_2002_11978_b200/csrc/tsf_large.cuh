// Large-n engine (n = N1*N2 > 4096, power of two): four-step transforms
// through L2/HBM over the N1 x N2 view j = N2 t1 + t2, k = k1 + N1 k2.
//
// A length-n filter  y = IFFT_n( S . FFT_n(x) )  is three kernels:
//   col_fwd : G adjacent columns t2 per CTA, x[N2 t1 + t2] (t1 < N1) -> FFT_N1
//             -> * W_n^{t2 k1} -> Z[k1][t2]      (prologue: load / Krylov
//                                                  vector update)
//   row     : one row k1 per CTA, FFT_N2 over Z[k1][.] -> * S[k1 + N1 k2]
//             -> IFFT_N2                         (S stored permuted [k1][k2])
//   col_inv : Z[.][t2] * conj(W_n^{t2 k1}) -> IFFT_N1 -> y at j = N2 t1 + t2
//                                                 (epilogue: store / combine
//                                                  with the operator / dot
//                                                  partials)
// The Toeplitz product uses the even/odd-bin split of the single-CTA engine
// (tsf_filters.cuh): two length-n filters, the odd one on x_j W_L^j.  Both
// run as two CHANNELS of the same three launches (Z holds both), and the
// column epilogue combines them in registers: y = d x + kappa (ye + Re(conj(w) zo)).
// Column CTAs run G transforms side by side with the group index in the
// fast thread bits, so every warp access covers G adjacent columns (full
// 32-byte sectors from G = 4 on).
// Reductions are deterministic: per-CTA partials [B][4][np] reduced in fixed
// order by one-CTA-per-instance scalar kernels (tsf_large.cu), which also
// hold the reference's BiCGSTAB control flow (krylov.py:88-153).
#pragma once

#include "tsf_kernels.cuh"
#include "tsf_tma.cuh"

namespace tsf {

struct LargeTables {
  const double2* tw1;   // two-level W_N1 table (column transforms)
  const double2* tw2;   // two-level W_N2 table (row transforms)
  const double2* twN;   // two-level W_n table: inter-pass twiddles
  const double2* twL;   // two-level W_L table (L = 2n), modulation of the odd half
  const double2* sEO;   // [k1][k2] -> (S_{2k}, S_{2k+1}) / L at k = k1 + N1 k2
  const double2* lamP;  // [k1][k2] -> (lam_k, lam_{n-k}) at k = k1 + N1 k2 (Strang)
};

// Half-length geometry and tables (tsf_hlarge.cuh): H = n/2 = N1 x N2
struct HalfGeom {
  int N1 = 0, N2 = 0;
  const double2* tw1 = nullptr;   // two-level W_N1
  const double2* tw2 = nullptr;   // two-level W_N2
  const double2* twH = nullptr;   // two-level W_H: inter-pass twiddles
  const double2* sEh = nullptr;   // [k1][k2] -> (n S_2k / L, n S_2(H-k) / L), k = k1 + N1 k2
  const double* sO4 = nullptr;    // [k1][k2] -> 2 S_{4k+1} / L
  const double2* lamH = nullptr;  // [k1][k2][2] -> (lam_k, lam_{n-k}), (lam_{H-k}, lam_{n-H+k})
  double2* hspec = nullptr;       // [B][H+1] half spectrum of the last Strang output
  double2* pspec2 = nullptr;      // [B][H] the level's Strang filter (S_k, S_{H-k}) / n
};

// BiCGSTAB per-instance control (scalar kernels)
enum LMode : int { LM_ACTIVE = 0, LM_EARLY = 1, LM_DONE = 2 };

struct LState {
  double rho, rho_new, alpha, omega, nrm0, rnorm, snorm, kbar, rz;
  int it, mode;
};

// Column prologues
enum ColIn : int {
  CI_LOAD = 0,     // z = x                                    (1 channel)
  CI_PUPD = 2,     // p = r + beta (p - omega v) (r0 at it 1); store p; z = p
  CI_SUPD = 3,     // s = r - alpha v; store s; ||s||^2 partial; z = s
  CI_APPLY = 4,    // channel 0: z = x ; channel 1: z = x_j W_L^j
};
// Column epilogues
enum ColOut : int {
  CO_REAL = 0,     // y_j = Re z   (store)
  CO_APPLY = 1,    // y_j = d x_j + kappa_j (Re z0_j + Re(conj(w_j) z1_j)) ; dot partials
};
// Half-length engine (tsf_hlarge.cuh): column prologues / epilogues
enum HColIn : int { HF_LOAD = 0, HF_PUPD = 2, HF_SUPD = 3, HF_ODD = 4 };
enum HColOut : int { HO_PACK = 0, HO_ODD = 1 };
// Row spectra
enum RowSpec : int { RS_APPLY = 0, RS_STRANG = 2 };

struct LargeArgs {
  int n, B;            // vector length n <= transform length nt (x is zero beyond n)
  int nt;
  LargeTables lt;
  double2* Z;          // [2][B][n] transform work array (channel-major)
  double* part;        // [B][4][np] partial sums
  int np;
  LState* st;          // [B] (null: standalone matvec / preconditioner)
  // Krylov vectors [B][n]
  const double* r0;
  double* x;
  double* r;
  double* p;
  double* v;
  double* ph;
  double* s;
  double* sh;
  double* t;
  const double* kappa;  // level diffusivity [B][n] (null: plain Toeplitz product)
  double* pspec;        // [B][n] permuted Strang spectrum S_k / n
  double shift;
  double tol;
  int max_iters;
  int* iters;
  double* relres;
  int* status;
  int* active;
  HalfGeom hg;
};

TSF_D bool inst_skip(const LargeArgs& a, int b) { return a.st && a.st[b].mode != LM_ACTIVE; }

// two-level table lookup straight from global memory (L1/L2 resident)
TSF_D double2 tw_get_g(const double2* tw, long e) {
  return cmul(ldt(&tw[kTwLo + (e >> 6) + (e >> 9)]), ldt(&tw[tw_lo_slot((int)(e & 63))]));
}

// Column-kernel geometry: G transforms of length N1 per CTA, T threads each.
// Threads per column CTA.  Small CTAs let several run per SM (128 registers
// each), so one CTA's exposed global loads overlap the others' transforms
// (ncu: the column kernels were 30-50% long-scoreboard stalls at one
// 512-thread CTA per SM); measured per column length on the configs[4]
// sweep: 128 threads (4 CTAs/SM) up to N1 = 256 (n = 2^20: 4.69 -> 4.29 ms
// per matvec; n = 2^14: 4.05 -> 3.13 ms), 256 at N1 = 512, 512 above (fewer
// columns per CTA cost coalescing there).  TSF_LCOL_THREADS overrides.
template <int N1>
constexpr int lcol_threads() {
#ifdef TSF_LCOL_THREADS
  return TSF_LCOL_THREADS;
#else
  return N1 <= 256 ? 128 : N1 == 512 ? 256 : 512;
#endif
}
template <int N1>
struct LCol {
  static constexpr int E = FShape<N1>::E;
  static constexpr int T = N1 / E;
  static constexpr int TH = lcol_threads<N1>();
  static constexpr int G = T >= TH ? 1 : (TH / T > 16 ? 16 : TH / T);
  static constexpr int MINB = (G * T <= 128) ? 4 : (G * T <= 256) ? 2 : 1;
  static constexpr int BLOCK = G * T;
  static constexpr int BUF = 2 * FftPlan<N1, E>::SMEM_ELEMS;  // ping-pong, per group
  static constexpr int SMEM = (G * BUF + tw_table_elems(N1)) * 16;
  // column-inverse kernels: + the two Z channel tiles (TMA landing zone),
  // 128-byte aligned after the twiddle table

};
template <int N2>
struct LRow {
  static constexpr int E = FShape<N2>::E;
  static constexpr int T = N2 / E;
  static constexpr int BLOCK = T < 32 ? 32 : T;
  static constexpr int SMEM = (2 * FftPlan<N2, E>::SMEM_ELEMS + tw_table_elems(N2)) * 16;
};

template <int NT>
TSF_D void stage_tw(double2* dst, const double2* src) {
  for (int i = threadIdx.x; i < tw_table_elems(NT); i += blockDim.x) dst[i] = ldt(&src[i]);
}

// ------------------------------------------------------------ col_fwd
// MB: CTAs per SM the register allocation is sized for — LCol::MINB for
// launches that fill the GPU, 1 (no register cap below 255) for the few-CTA
// launches of single large instances, which are latency-bound (configs[1]).
template <int N1, int MB = LCol<N1>::MINB>
__global__ void __launch_bounds__(LCol<N1>::BLOCK, MB)
k_lcol_fwd(LargeArgs a, const double* __restrict__ src, int in_mode,
           const __grid_constant__ ColMaps cm) {
  pdl_enter();
  using C = LCol<N1>;
  constexpr int E = C::E, T = C::T, G = C::G;
  const int N2 = a.nt / N1;
  const long N = a.nt;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ double red[4 * 32];
  __shared__ unsigned long long bar;
  const int b = blockIdx.y;
  const int g = threadIdx.x % G, tid = threadIdx.x / G;
  const int t2 = blockIdx.x * G + g;
  double2* smg = sm + g * C::BUF;
  double2* tw1 = sm + G * C::BUF;
  const long off = (long)b * a.n;   // vectors [B][n]
  const long offz = (long)b * N;    // transform work [B][nt]
  double xr[E];
  double2 z[E];
  double part = 0.0;
  if (cm.use) {
    // TMA path (tsf_tma.cuh): the operand tiles land in the (not yet used)
    // transform buffers while the CTA stages its twiddles and reads the state
    double* tile = reinterpret_cast<double*>(sm);
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      unsigned bytes = 0;
      mbar_expect_tx(&bar, (unsigned)(cm.nv * N1 * G * 8));
      for (int q = 0; q < cm.nv; ++q)
        bytes += tma_tile(tile + q * N1 * G, &cm.v[q], blockIdx.x * G, N1, G, b, 8, &bar);
      (void)bytes;
    }
    stage_tw<N1>(tw1, a.lt.tw1);
    const LState stv = a.st ? a.st[b] : LState{};
    __syncthreads();   // barrier initialised before anyone waits on it
    mbar_wait(&bar, 0);
    if (inst_skip(a, b)) return;
    const bool upd = in_mode == CI_PUPD || in_mode == CI_SUPD;
    const bool pupd_it1 = in_mode == CI_PUPD && stv.it == 1;
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int t1 = tid + c * T;
      const long j = (long)N2 * t1 + t2;
      const double l0 = pupd_it1 ? a.r0[off + j] : tile[t1 * G + g];
      double val;
      if (in_mode == CI_PUPD) {
        if (pupd_it1) {
          val = l0;
        } else {
          const double beta = (stv.rho_new / stv.rho) * (stv.alpha / stv.omega);
          val = l0 + beta * (tile[N1 * G + t1 * G + g] - stv.omega * tile[2 * N1 * G + t1 * G + g]);
        }
      } else if (in_mode == CI_SUPD) {
        val = (stv.it == 1 ? a.r0[off + j] : l0) - stv.alpha * tile[N1 * G + t1 * G + g];
        part = fma(val, val, part);
      } else {
        val = l0;
      }
      xr[c] = val;
    }
    (void)upd;
    if (in_mode == CI_PUPD || in_mode == CI_SUPD) {
      double* dst = in_mode == CI_PUPD ? a.p : a.s;
#pragma unroll
      for (int c = 0; c < E; ++c) dst[off + (long)N2 * (tid + c * T) + t2] = xr[c];
    }
  } else {
  // plain-load path (n not a multiple-of-rows view, or TSF_TMA=0)
  // Every operand is loaded before the first store: the vectors are plain
  // pointers that may alias, so a store between two elements' loads kept
  // the compiler from issuing the next element's loads early and serialised
  // E memory latencies per thread (ncu, configs[3]: 65% of this kernel's
  // stall samples were long-scoreboard waits on these loads).
  // The loads are also issued before the instance state arrives: they
  // assume iteration > 1 (r, p, v) and the first iteration re-reads r0; a
  // finished instance's CTA loads its (valid, unused) vectors and returns.
  const bool upd = in_mode == CI_PUPD || in_mode == CI_SUPD;
  const double* l0p = upd ? a.r : src;
  double l0[E], l1[E], l2[E];
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const long j = (long)N2 * (tid + c * T) + t2;
    const bool in = j < a.n;   // zero padding up to the transform length
    l0[c] = in ? l0p[off + j] : 0.0;
    l1[c] = (in && upd) ? (in_mode == CI_PUPD ? a.p[off + j] : a.v[off + j]) : 0.0;
    l2[c] = (in && in_mode == CI_PUPD) ? a.v[off + j] : 0.0;
  }
  if (inst_skip(a, b)) return;
  const LState stv = a.st ? a.st[b] : LState{};
  const bool pupd_it1 = in_mode == CI_PUPD && stv.it == 1;
  if (upd && stv.it == 1) {   // krylov.py:114-116: the first p (and s) start from r0
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long j = (long)N2 * (tid + c * T) + t2;
      l0[c] = j < a.n ? a.r0[off + j] : 0.0;
    }
  }
  stage_tw<N1>(tw1, a.lt.tw1);
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const long j = (long)N2 * (tid + c * T) + t2;
    double val = 0.0;
    if (j >= a.n) {
      // zero padding up to the transform length
    } else if (in_mode == CI_PUPD) {
      if (pupd_it1) {
        val = l0[c];
      } else {
        const double beta = (stv.rho_new / stv.rho) * (stv.alpha / stv.omega);
        val = l0[c] + beta * (l1[c] - stv.omega * l2[c]);
      }
      a.p[off + j] = val;
    } else if (in_mode == CI_SUPD) {
      val = l0[c] - stv.alpha * l1[c];
      a.s[off + j] = val;
      part = fma(val, val, part);
    } else {
      val = l0[c];
    }
    xr[c] = val;
  }
  }  // plain-load path
  if (in_mode == CI_SUPD) {
    part = block_sum1(part, red);
    if (threadIdx.x == 0) a.part[((long)b * 4 + 2) * a.np + blockIdx.x] = part;
  }
  group_fft_real<N1, E>(xr, z, smg, tw1, 0, tid);
  // inter-pass twiddles loaded before the stores (aliasing, see above)
  double2 wt[E];
#pragma unroll
  for (int c = 0; c < E; ++c) wt[c] = tw_get_g(a.lt.twN, ((long)t2 * (tid + c * T)) & (N - 1));
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const int k1 = tid + c * T;
    a.Z[offz + (long)k1 * N2 + t2] = cmul(z[c], wt[c]);
  }
  if (in_mode == CI_APPLY) {
    // odd channel: the modulated input x_j W_L^j
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long j = (long)N2 * (tid + c * T) + t2;
      z[c] = cscale(tw_get_g(a.lt.twL, j), xr[c]);
    }
    group_fft<N1, E, false>(z, smg, tw1, 0, tid);
    double2* Zo = a.Z + (long)a.B * N;
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const int k1 = tid + c * T;
      Zo[offz + (long)k1 * N2 + t2] = cmul(z[c], wt[c]);   // same k1 -> same twiddle
    }
  }
}

// ------------------------------------------------------------ row
template <int N2>
__global__ void __launch_bounds__(LRow<N2>::BLOCK, 1)
k_lrow(LargeArgs a, int spec_mode) {
  pdl_enter();
  const long N = a.nt;
  constexpr int E = LRow<N2>::E;
  constexpr int T = LRow<N2>::T;
  extern __shared__ double2 sm[];
  const int k1 = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  if (inst_skip(a, b)) return;
  const bool own = tid < T;
  const int nch = spec_mode == RS_APPLY ? 2 : 1;
  // the row is loaded before the twiddle staging (both in flight at once);
  // spectrum factors and the next channel's row are loaded by the
  // transforms' load hooks (tsf_fft.cuh), two passes before they are used
  double2 z[E];
  double2* row = a.Z + (long)b * N + (long)k1 * N2;
  if (own) {
#pragma unroll
    for (int c = 0; c < E; ++c) z[c] = row[tid + c * T];
  }
  double2* tw2 = sm + 2 * FftPlan<N2, E>::SMEM_ELEMS;
  stage_tw<N2>(tw2, a.lt.tw2);
  for (int ch = 0; ch < nch; ++ch) {
    double sp[E];
    block_fft<N2, E, false>(z, sm, tw2, 0, static_cast<const double2*>(nullptr), [&] {
      if (own) {
#pragma unroll
        for (int c = 0; c < E; ++c) {
          const long idx = (long)k1 * N2 + tid + c * T;   // bin k1 + N1 k2
          if (spec_mode == RS_APPLY) {
            const double2 se = ldt(&a.lt.sEO[idx]);
            sp[c] = ch == 0 ? se.x : se.y;
          } else {
            sp[c] = a.pspec[(long)b * N + idx];
          }
        }
      }
    });
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) z[c] = cscale(z[c], sp[c]);
    }
    double2 zn[E];
    double2* nrow = row + (long)a.B * N;   // next channel's row
    block_fft<N2, E, true>(z, sm, tw2, 0, static_cast<const double2*>(nullptr), [&] {
      if (own && ch + 1 < nch) {
#pragma unroll
        for (int c = 0; c < E; ++c) zn[c] = nrow[tid + c * T];
      }
    });
    if (own) {
#pragma unroll
      for (int c = 0; c < E; ++c) row[tid + c * T] = z[c];
    }
    if (ch + 1 < nch) {
#pragma unroll
      for (int c = 0; c < E; ++c) z[c] = zn[c];
      row = nrow;
    }
  }
}

// ------------------------------------------------------------ row, short rows
// Rows of N2 <= 128 points (n = 8192) have T < 32 owning threads: k_lrow ran
// each row as a sub-warp CTA doing its two channels one after the other, a
// latency chain of four transforms.  Here a 64-thread CTA runs 64/T
// independent (row, channel) items side by side — the two channels of a row
// concurrently — through the grouped transform (configs[4] n = 8192: matvec
// 3.92 -> 3.21 ms, preconditioner 2.18 -> 1.63 ms).  At N2 = 256 (configs[1],
// one warp per item) it measured no faster than k_lrow (0.777 vs 0.777 ms per
// level), so k_lrow keeps those rows.
template <int N2>
__global__ void __launch_bounds__(64) k_lrow_small(LargeArgs a, int spec_mode) {
  pdl_enter();
  constexpr int E = LRow<N2>::E;
  constexpr int T = LRow<N2>::T;
  static_assert(T <= 32 && 64 % T == 0, "short-row kernel");
  constexpr int IT = 64 / T;
  constexpr int BUF = 2 * FftPlan<N2, E>::SMEM_ELEMS;
  const long N = a.nt;
  const int N1 = (int)(N / N2);
  const int b = blockIdx.y;
  if (inst_skip(a, b)) return;
  const int nch = spec_mode == RS_APPLY ? 2 : 1;
  const int slot = threadIdx.x / T, tid = threadIdx.x % T;
  const int item = blockIdx.x * IT + slot;
  const bool valid = item < N1 * nch;
  const int k1 = valid ? item / nch : 0, ch = valid ? item % nch : 0;
  extern __shared__ double2 sm[];
  double2* smi = sm + slot * BUF;
  double2* tw2 = sm + IT * BUF;
  stage_tw<N2>(tw2, a.lt.tw2);
  double2* row = a.Z + (long)ch * a.B * N + (long)b * N + (long)k1 * N2;
  double2 z[E];
#pragma unroll
  for (int c = 0; c < E; ++c) z[c] = valid ? row[tid + c * T] : make_double2(0.0, 0.0);
  double sp[E];
  group_fft<N2, E, false>(z, smi, tw2, 0, tid, [&] {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long idx = (long)k1 * N2 + tid + c * T;   // bin k1 + N1 k2
      if (!valid) {
        sp[c] = 0.0;
      } else if (spec_mode == RS_APPLY) {
        const double2 se = ldt(&a.lt.sEO[idx]);
        sp[c] = ch == 0 ? se.x : se.y;
      } else {
        sp[c] = a.pspec[(long)b * N + idx];
      }
    }
  });
#pragma unroll
  for (int c = 0; c < E; ++c) z[c] = cscale(z[c], sp[c]);
  group_fft<N2, E, true>(z, smi, tw2, 0, tid);
  if (valid) {
#pragma unroll
    for (int c = 0; c < E; ++c) row[tid + c * T] = z[c];
  }
}

// ------------------------------------------------------------ col_inv
template <int N1, int MB = LCol<N1>::MINB>
__global__ void __launch_bounds__(LCol<N1>::BLOCK, MB)
k_lcol_inv(LargeArgs a, double* __restrict__ dst, int out_mode, const double* __restrict__ xin,
           const double* __restrict__ w1, int pslot, const __grid_constant__ ColMaps cm) {
  pdl_enter();
  using C = LCol<N1>;
  constexpr int E = C::E, T = C::T, G = C::G;
  const int N2 = a.nt / N1;
  const long N = a.nt;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ double red[4 * 32];
  __shared__ unsigned long long bar;
  const int b = blockIdx.y;
  if (inst_skip(a, b)) return;
  const int g = threadIdx.x % G, tid = threadIdx.x / G;
  const int t2 = blockIdx.x * G + g;
  double2* smg = sm + g * C::BUF;
  double2* tw1 = sm + G * C::BUF;
  // the channel tiles of Z land in the transform buffers (free until the
  // channel's transform starts): no extra shared memory, same CTAs per SM
  double2* ztile = sm;
  if (cm.use && threadIdx.x == 0) {
    // channel 0's [N1 x G] tile of Z by TMA (tsf_tma.cuh)
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (unsigned)(N1 * G * 16));
    tma_tile(reinterpret_cast<double*>(ztile), &cm.z, 2 * blockIdx.x * G, N1, 2 * G, b, 8, &bar);
  }
  stage_tw<N1>(tw1, a.lt.tw1);
  const long off = (long)b * a.n;   // vectors [B][n]
  const long offz = (long)b * N;    // transform work [B][nt]
  double2 z[E];
  if (cm.use) {
    __syncthreads();   // barrier initialised before anyone waits on it
    mbar_wait(&bar, 0);
  }
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const int k1 = tid + c * T;
    const double2 w = tw_get_g(a.lt.twN, ((long)t2 * k1) & (N - 1));
    z[c] = cmulc(cm.use ? ztile[k1 * G + g] : a.Z[offz + (long)k1 * N2 + t2], w);
  }
  group_fft<N1, E, true>(z, smg, tw1, 0, tid);
  if (out_mode == CO_REAL) {
#pragma unroll
    for (int c = 0; c < E; ++c) {
      const long j = (long)N2 * (tid + c * T) + t2;
      if (j < a.n) dst[off + j] = z[c].x;
    }
    return;
  }
  // CO_APPLY: even channel result in registers, then the odd channel
  double ye[E];
#pragma unroll
  for (int c = 0; c < E; ++c) ye[c] = z[c].x;
  const double2* Zo = a.Z + (long)a.B * N;
  if (cm.use) {
    // channel 1's tile, once every thread's last transform pass is done
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar, (unsigned)(N1 * G * 16));
      tma_tile(reinterpret_cast<double*>(ztile), &cm.z, 2 * blockIdx.x * G, N1, 2 * G, a.B + b, 8,
               &bar);
    }
    mbar_wait(&bar, 1);
  }
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const int k1 = tid + c * T;
    const double2 w = tw_get_g(a.lt.twN, ((long)t2 * k1) & (N - 1));
    z[c] = cmulc(cm.use ? ztile[k1 * G + g] : Zo[offz + (long)k1 * N2 + t2], w);
  }
  group_fft<N1, E, true>(z, smg, tw1, 0, tid);
  Vals<2> pr;
  pr.v[0] = pr.v[1] = 0.0;
  // epilogue operands loaded before the stores, half the slots at a time
  // (aliasing, see k_lcol_fwd; all at once would exceed the register cap)
  constexpr int H = E > 1 ? E / 2 : 1;
#pragma unroll
  for (int c0 = 0; c0 < E; c0 += H) {
    double2 wm[H];
    double xv[H], kv[H], w1v[H];
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const long j = (long)N2 * (tid + (c0 + q) * T) + t2;
      const bool in = j < a.n;
      wm[q] = in ? tw_get_g(a.lt.twL, j) : make_double2(0.0, 0.0);
      xv[q] = (in && a.kappa) ? xin[off + j] : 0.0;
      kv[q] = (in && a.kappa) ? a.kappa[off + j] : 0.0;
      w1v[q] = (in && w1) ? w1[off + j] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < H; ++q) {
      const int c = c0 + q;
      const long j = (long)N2 * (tid + c * T) + t2;
      if (j >= a.n) continue;
      const double2 w = wm[q];
      const double ax = ye[c] + fma(z[c].x, w.x, z[c].y * w.y);  // + Re(conj(w) z)
      const double y = a.kappa ? fma(a.shift, xv[q], kv[q] * ax) : ax;
      dst[off + j] = y;
      pr.v[0] = fma(y, y, pr.v[0]);
      if (w1) pr.v[1] = fma(y, w1v[q], pr.v[1]);
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

// Column launches smaller than two waves of one CTA per SM take the
// uncapped-register instantiation (latency-bound single instances).
inline bool few_ctas(long ctas) {
  static int sms = 0;
  if (!sms && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess)
    sms = 148;
  return ctas < 2L * sms;
}

// Per-size launchers (bodies in tsf_large_impl.cuh, one TU per size:
// gen/large_L*.cu).  LOG = log2 of the column (N1) or row (N2) length.
constexpr int kLargeMinLog = 6;   // N1 >= 64
constexpr int kLargeMaxLog = 12;  // N1, N2 <= 4096  ->  n <= 2^24

template <int LOG>
struct LargeDispatch {
  static int col_fwd(const LargeArgs& a, const double* src, int in_mode, cudaStream_t st);
  static int row(const LargeArgs& a, int spec_mode, cudaStream_t st);
  static int col_inv(const LargeArgs& a, double* dst, int out_mode, const double* xin,
                     const double* w1, int pslot, cudaStream_t st);
  static int col_group();  // G: columns per column CTA
  // half-length engine (tsf_hlarge.cuh); LOG = log2 of N1 (columns) or N2 (rows)
  static int hcol_fwd(const LargeArgs& a, const double* src, int in_mode, cudaStream_t st);
  static int hrow_strang(const LargeArgs& a, int mode, cudaStream_t st);
  static int hrow_mv(const LargeArgs& a, cudaStream_t st);
  static int hcol_inv(const LargeArgs& a, double* dst, int out_mode, double* dst1,
                      const double* xin, const double* ye, const double* w1, int pslot,
                      cudaStream_t st);
};

// Launches of the large-n engine are programmatic dependent launches
// (kernels enter through pdl_enter, tsf_common.cuh): a B = 1 iteration is 17
// short dependent launches, and the next grid's launch latency and CTA
// rasterisation now overlap the running one.  TSF_PDL=0 launches plainly.
inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("TSF_PDL");
    v = (s && s[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// L2 persistence window of the running solve (TSF_L2_PERSIST=1, experiment):
// the transform work array Z of a single large instance (32 MB at n = 2^20)
// fits the 126 MB L2; a persisting access-policy window on every launch keeps
// it there between the column / row / column kernels.  Set by the host around
// the launches of one solve (tsf_large.cu), read by launch_pdl.
struct L2Window {
  void* base = nullptr;
  size_t bytes = 0;
};
inline L2Window& l2_window() {
  static thread_local L2Window w;
  return w;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  const L2Window& w = l2_window();
  if (w.base) {
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na].val.accessPolicyWindow.base_ptr = w.base;
    at[na].val.accessPolicyWindow.num_bytes = w.bytes;
    at[na].val.accessPolicyWindow.hitRatio = 1.0f;
    at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

#define TSF_EXTERN_LARGE(L) extern template struct LargeDispatch<L>;
TSF_EXTERN_LARGE(6)
TSF_EXTERN_LARGE(7)
TSF_EXTERN_LARGE(8)
TSF_EXTERN_LARGE(9)
TSF_EXTERN_LARGE(10)
TSF_EXTERN_LARGE(11)
TSF_EXTERN_LARGE(12)

}  // namespace tsf
