// Block-level Stockham FFT in shared memory, fp64, sm_100a.
//
// One CTA transforms one complex sequence of length N (power of two).  The
// CTA has T = N/E "owning" threads; thread `tid` owns the complex slots
// j = tid + c*T, c in [0, E).  The first radix pass reads its butterfly
// inputs straight from the owning thread's registers and the last pass
// writes its outputs back to them, so a transform costs (passes-1) shared
// memory round trips and data can stay in registers between the FFT and the
// surrounding vector arithmetic (the Krylov updates are done on exactly
// these slots).
//
// Radix passes are chosen greedily (radix <= min(E,16)); twiddles come from
// a host-computed table W_NT^e (long-double accurate, NT >= N) read through
// the read-only path.  Shared-memory addresses are padded with
// pad(i) = i + (i >> log2(R_first)), which makes the strided writes of the
// first pass and the contiguous accesses of all later passes conflict-free
// for 16-byte elements.
//
// Replaces numpy pocketfft at the reference call sites fourier.py:20-27
// (used by toeplitz.py:51-63 and toeplitz.py:131-136).
#pragma once

#include "tsf_common.cuh"

#ifndef TSF_FFT_INPLACE
#define TSF_FFT_INPLACE 0
#endif
#ifndef TSF_KE
#define TSF_KE 8
#endif
#ifndef TSF_PTW_SMALL
#define TSF_PTW_SMALL 0
#endif

namespace tsf {

// ------------------------------------------------------------ small DFTs
// All DFTs are in place, natural order in and out; INV selects the +i sign.
template <bool INV>
TSF_D void dft2(double2& a0, double2& a1) {
  double2 t = a0;
  a0 = cadd(t, a1);
  a1 = csub(t, a1);
}

template <bool INV>
TSF_D void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  double2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
  double2 t2 = cadd(a1, a3), t3 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

#define TSF_R2 0.70710678118654752440084436210484903928
#define TSF_C8 0.92387953251128675612818318939678828682
#define TSF_S8 0.38268343236508977172845998403039886676

// x * W8^1 (fwd: (1-i)/sqrt2 ; inv: (1+i)/sqrt2)
template <bool INV>
TSF_D double2 w8_1(double2 x) {
  return INV ? make_double2((x.x - x.y) * TSF_R2, (x.x + x.y) * TSF_R2)
             : make_double2((x.x + x.y) * TSF_R2, (x.y - x.x) * TSF_R2);
}
// x * W8^3 (fwd: (-1-i)/sqrt2 ; inv: (-1+i)/sqrt2)
template <bool INV>
TSF_D double2 w8_3(double2 x) {
  return INV ? make_double2((-x.x - x.y) * TSF_R2, (x.x - x.y) * TSF_R2)
             : make_double2((x.y - x.x) * TSF_R2, (-x.x - x.y) * TSF_R2);
}

template <bool INV>
TSF_D void dft8(double2* a) {
  // DIT: even/odd halves of length 4, then combine with W8^k.
  double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
  double2 o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = w8_1<INV>(o1);
  o2 = mul_mi<INV>(o2);
  o3 = w8_3<INV>(o3);
  a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
  a[1] = cadd(e1, o1); a[5] = csub(e1, o1);
  a[2] = cadd(e2, o2); a[6] = csub(e2, o2);
  a[3] = cadd(e3, o3); a[7] = csub(e3, o3);
}

// x * W16^e for the exponents a 4x4 decomposition needs.
template <int EXP, bool INV>
TSF_D double2 w16(double2 x) {
  if constexpr (EXP == 0) return x;
  else if constexpr (EXP == 2) return w8_1<INV>(x);
  else if constexpr (EXP == 4) return mul_mi<INV>(x);
  else if constexpr (EXP == 6) return w8_3<INV>(x);
  else {
    constexpr double c = (EXP == 1) ? TSF_C8 : (EXP == 3) ? TSF_S8 : -TSF_C8;  // 1, 3, 9
    constexpr double s = (EXP == 1) ? TSF_S8 : (EXP == 3) ? TSF_C8 : -TSF_S8;
    // W = c - i s (fwd) ; c + i s (inv)
    return INV ? make_double2(fma(x.x, c, -x.y * s), fma(x.x, s, x.y * c))
               : make_double2(fma(x.x, c, x.y * s), fma(x.y, c, -x.x * s));
  }
}

template <bool INV>
TSF_D void dft16(double2* a) {
  // 4x4: columns n2 = 0..3 over n1 (stride 4), twiddle W16^{n2 k1}, rows.
  dft4<INV>(a[0], a[4], a[8], a[12]);
  dft4<INV>(a[1], a[5], a[9], a[13]);
  dft4<INV>(a[2], a[6], a[10], a[14]);
  dft4<INV>(a[3], a[7], a[11], a[15]);
  // Y_{n2}[k1] sits at a[n2 + 4 k1]
  a[5] = w16<1, INV>(a[5]);
  a[9] = w16<2, INV>(a[9]);
  a[13] = w16<3, INV>(a[13]);
  a[6] = w16<2, INV>(a[6]);
  a[10] = w16<4, INV>(a[10]);
  a[14] = w16<6, INV>(a[14]);
  a[7] = w16<3, INV>(a[7]);
  a[11] = w16<6, INV>(a[11]);
  a[15] = w16<9, INV>(a[15]);
  // rows: for k1, DFT4 over n2 -> X[k1 + 4 k2]
  dft4<INV>(a[0], a[1], a[2], a[3]);
  dft4<INV>(a[4], a[5], a[6], a[7]);
  dft4<INV>(a[8], a[9], a[10], a[11]);
  dft4<INV>(a[12], a[13], a[14], a[15]);
  // currently X[k1 + 4 k2] at a[4 k1 + k2]: transpose 4x4
  double2 t;
  t = a[1]; a[1] = a[4]; a[4] = t;
  t = a[2]; a[2] = a[8]; a[8] = t;
  t = a[3]; a[3] = a[12]; a[12] = t;
  t = a[6]; a[6] = a[9]; a[9] = t;
  t = a[7]; a[7] = a[13]; a[13] = t;
  t = a[11]; a[11] = a[14]; a[14] = t;
}

template <int R, bool INV>
TSF_D void dft(double2* a) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2<INV>(a[0], a[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(a[0], a[1], a[2], a[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(a);
  } else {
    static_assert(R == 16, "radix must be 1,2,4,8,16");
    dft16<INV>(a);
  }
}

// ------------------------------------------------------------ twiddles
// Two-level table staged in shared memory by every kernel:
//   tw[lo_slot(j)]      = W^j,       j < 64
//   tw[72 + lo_slot(i)] = W^(64 i),  i < max(1, NT/64)
// so W^e = hi[e >> 6] * lo[e & 63] (within ~1 ulp; both factors are
// correctly rounded long-double values).  A full table of NT entries (128 KB
// at NT = 8192) does not fit the L1 left beside the transform buffers, and
// streaming it from L2 was the main stall of the first solve kernels
// (DESIGN.md §3.3).
// In-place passes (one buffer, a barrier between a pass's reads and writes)
// halve the transform's shared memory; out-of-place (ping-pong) passes need
// no mid-pass barrier.  See DESIGN.md §3.1.
constexpr bool kFftInPlace = TSF_FFT_INPLACE;

// Both halves are stored padded, entry i at slot i + (i >> 3): the W^{k},
// W^{2k}, W^{4k} lookups of a warp walk either table with strides 1..8 and
// then hit distinct banks (unpadded they were 2/4/8-way conflicts: the low
// table 28% of all shared wavefronts, the high table 8-way on the first
// twiddled pass, both seen in ncu).
constexpr int kTwLo = 72;
TSF_HD constexpr int tw_lo_slot(int j) { return j + (j >> 3); }
TSF_HD constexpr int tw_hi_count(int NT) { return NT / 64 > 1 ? NT / 64 : 1; }
TSF_HD constexpr int tw_table_elems(int NT) {
  return kTwLo + tw_hi_count(NT) + (tw_hi_count(NT) >> 3) + 1;
}
TSF_D double2 tw_get(const double2* tw, int e) {
  return cmul(tw[kTwLo + tw_lo_slot(e >> 6)], tw[tw_lo_slot(e & 63)]);
}

// ------------------------------------------------------------ pass plan
constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }
constexpr int imin(int a, int b) { return a < b ? a : b; }

// radix of pass p for an N-point transform with E elements per thread
template <int N, int E>
struct FftPlan {
  static constexpr int LOGN = ilog2(N);
  static constexpr int LOGR = ilog2(imin(E, 16));
  static constexpr int NPASS = (LOGN + LOGR - 1) / LOGR;
  static constexpr int T = N / E;
  static constexpr int PADSHIFT = imin(LOGR, LOGN);  // log2 of the first radix
  static constexpr int SMEM_ELEMS = N + (N >> PADSHIFT) + 1;  // one of the two buffers
  static constexpr int log_radix(int p) {
    return (p < NPASS - 1) ? LOGR : (LOGN - LOGR * (NPASS - 1));
  }
  static constexpr int log_ns(int p) { return p * LOGR; }
  TSF_HD static int pad(int i) { return i + (i >> PADSHIFT); }
  // explicit per-pass twiddles (TSF_PASS_TW): pass p >= 1 stores
  // W_{NS R}^{k m} at ptw_off(p) + (m-1) NS + k, k < NS, 1 <= m < R
  static constexpr int ptw_off(int p) {
    return p <= 1 ? 0 : ptw_off(p - 1) + ((1 << log_radix(p - 1)) - 1) * (1 << log_ns(p - 1));
  }
  static constexpr int PTW_ELEMS = ptw_off(NPASS);
  // passes whose twiddles come from the small explicit table (kPassTwSmall):
  // NS R <= kPtwSmall; their entries are a prefix of the full ptw layout
  static constexpr int small_passes(int p = 1) {
    return (p < NPASS && (1 << (log_ns(p) + log_radix(p))) <= TSF_PTW_SMALL) ? small_passes(p + 1)
                                                                            : p;
  }
  static constexpr int PTWS_ELEMS = ptw_off(small_passes());
};

#ifndef TSF_PASS_TW
#define TSF_PASS_TW 0
#endif
constexpr bool kPassTw = TSF_PASS_TW;
// Explicit twiddles for the early passes (NS R <= TSF_PTW_SMALL, e.g. 512: 504 entries
// = 8 KB at N = 4096), staged in shared memory: one correctly rounded table
// read per factor instead of three two-level lookups and four products per
// radix-8 butterfly; the last pass keeps the two-level table.  Off (0) by
// default: measured slower on configs[2] (27.5 vs 26.8 ms per level solve).
constexpr bool kPassTwSmall = TSF_PTW_SMALL > 0 && !TSF_PASS_TW;
#ifndef TSF_STAGE_TABLES
#define TSF_STAGE_TABLES 0
#endif
// cp.async staging in flight during transforms (tsf_filters.cuh
// stage_tables): only then do the inter-pass barriers wait for it.  The
// unconditional wait compiled to DEPBAR.LE SB0 before every barrier.
#ifndef TSF_FORCE_WAIT
#define TSF_FORCE_WAIT 0
#endif
constexpr bool kAsyncStaging = TSF_STAGE_TABLES || TSF_PASS_TW || TSF_FORCE_WAIT;

// One Stockham pass: radix R, NS = product of the previous radices.
//  FROM_REGS: inputs come from v[] (first pass), else from shared memory.
//  TO_REGS:   outputs go to v[] (last pass), else to shared memory.
// Out of place: pass P reads buffer (P+1)&1 and writes buffer P&1 (two
// transform buffers), so loaded values never have to survive a barrier —
// with an in-place pass they did, and inside the Krylov loop ptxas spilled
// them to local memory.  Only owning threads touch data.
// Explicit-twiddle table pointer of the early passes (kPassTwSmall): a
// distinct type, so transforms given one compile only the table path for
// those passes and transforms given a plain pointer (or none) only the
// two-level path — no runtime branch, no dead path inflating registers.
struct SmallTw {
  const double2* p;
};
template <class PT>
constexpr bool is_small_tw() { return false; }
template <>
constexpr bool is_small_tw<SmallTw>() { return true; }
TSF_D const double2* tw_ptr(const double2* p) { return p; }
TSF_D const double2* tw_ptr(SmallTw p) { return p.p; }

template <int N, int E, int P, bool INV, bool FROM_REGS, bool TO_REGS, class PT>
TSF_D void stockham_pass(double2 (&v)[E], double2* sm, const double2* __restrict__ tw,
                         int tw_log_scale, int tid, bool own, PT ptw_in) {
  using PL = FftPlan<N, E>;
  constexpr int R = 1 << PL::log_radix(P);
  constexpr int NS = 1 << PL::log_ns(P);
  constexpr int T = PL::T;
  constexpr int Q = E / R;
  constexpr int NR = N / R;
  const double2* src = sm + (kFftInPlace ? 0 : ((P + 1) & 1) * PL::SMEM_ELEMS);
  double2* dst = sm + (kFftInPlace ? 0 : (P & 1) * PL::SMEM_ELEMS);
  double2 a[Q][R];
  if (own) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        if constexpr (FROM_REGS) a[q][m] = v[q + m * Q];
        else a[q][m] = src[PL::pad(tid + q * T + m * NR)];
      }
    }
  }
  if constexpr (kFftInPlace && !FROM_REGS && !TO_REGS) __syncthreads();  // reads before writes
  if (!own) return;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int b = tid + q * T;
    const int k = b & (NS - 1);
    constexpr bool XS = is_small_tw<PT>() && NS * R <= TSF_PTW_SMALL;
    const double2* ptw = tw_ptr(ptw_in);
    if ((XS || kPassTw) && NS > 1 && (XS || ptw)) {
      // explicit table: one correctly rounded entry per power, no products
      const double2* pt = ptw + PL::ptw_off(P) + k;
#pragma unroll
      for (int m = 1; m < R; ++m) {
        const double2 w = pt[(m - 1) * NS];
        a[q][m] = INV ? cmulc(a[q][m], w) : cmul(a[q][m], w);
      }
    } else if constexpr (NS > 1) {
      // W_{NS R}^{k m} = W_NT^{k m NT/(NS R)}, NT/(NS R) = 2^sh
      const int sh = tw_log_scale + PL::LOGN - PL::log_ns(P) - PL::log_radix(P);
      // W^k, W^2k, W^4k from the table; the other powers are one product of
      // two of them (3 of 7 table reads per butterfly; accuracy measured in
      // tools/accuracy_probe.py against an exact long-double DFT)
      // exponents that are multiples of 64 (sh >= 6: the first twiddled pass)
      // need only the high table: lo[0] = 1 exactly, so the product it saves
      // was exact — same values, 3 loads and 3 complex products fewer
      auto twx = [&](int e) {
        return sh >= 6 ? tw[kTwLo + tw_lo_slot(e >> 6)] : tw_get(tw, e);
      };
      double2 w[R];
      w[1] = twx(k << sh);
      if constexpr (R >= 4) {
        w[2] = twx((2 * k) << sh);
        w[3] = cmul(w[2], w[1]);
      }
      if constexpr (R >= 8) {
        w[4] = twx((4 * k) << sh);
        w[5] = cmul(w[4], w[1]);
        w[6] = cmul(w[4], w[2]);
        w[7] = cmul(w[4], w[3]);
      }
      if constexpr (R >= 16) {
        w[8] = twx((8 * k) << sh);
#pragma unroll
        for (int m = 9; m < 16; ++m) w[m] = cmul(w[8], w[m - 8]);
      }
#pragma unroll
      for (int m = 1; m < R; ++m) a[q][m] = INV ? cmulc(a[q][m], w[m]) : cmul(a[q][m], w[m]);
    }
    dft<R, INV>(a[q]);
    if constexpr (TO_REGS) {
#pragma unroll
      for (int m = 0; m < R; ++m) v[q + m * Q] = a[q][m];
    } else {
      const int base = (b / NS) * NS * R + k;
#pragma unroll
      for (int m = 0; m < R; ++m) dst[PL::pad(base + m * NS)] = a[q][m];
    }
  }
}

// Load hook: a transform calls hook() once, at the start of pass
// max(1, NPASS-2), so the caller's global loads for the step after the
// transform (spectrum factors, epilogue operands) are in flight during the
// last two passes instead of stalling every warp at once after the final
// barrier (ncu: long-scoreboard stalls on those loads were 30% of the level
// solve's stall cycles).
struct NoHook {
  TSF_D void operator()() const {}
};
template <int N, int E>
constexpr int hook_pass() {
  return FftPlan<N, E>::NPASS - 2 > 1 ? FftPlan<N, E>::NPASS - 2 : 1;
}

template <int N, int E, int P, bool INV, class Hook = NoHook, class PT = const double2*>
TSF_D void fft_rec(double2 (&v)[E], double2* sm, const double2* __restrict__ tw,
                   int tw_log_scale, int tid, bool own, PT ptw = nullptr,
                   const Hook& hook = Hook{}) {
  using PL = FftPlan<N, E>;
  constexpr bool FIRST = (P == 0);
  constexpr bool LAST = (P == PL::NPASS - 1);
  if constexpr (P == hook_pass<N, E>()) hook();
  stockham_pass<N, E, P, INV, FIRST, LAST>(v, sm, tw, tw_log_scale, tid, own, ptw);
  if constexpr (!LAST) {
    if constexpr (kAsyncStaging) cp_async_wait_all();  // staged tables land here
    __syncthreads();
    fft_rec<N, E, P + 1, INV>(v, sm, tw, tw_log_scale, tid, own, ptw, hook);
  }
}

// Full transform of the owned slots v[c] (j = tid + c*T).  Unnormalised in
// both directions.  Every thread of the CTA must call; threads with
// tid >= T own nothing.  Starts with a barrier so the caller may reuse `sm`
// right before; ends with data in registers (sm may be reused after a
// barrier).
// `tw` holds W_NT^e for e < NT with NT = N << tw_log_scale.
template <int N, int E, bool INV, class Hook = NoHook, class PT = const double2*>
TSF_D void block_fft(double2 (&v)[E], double2* sm, const double2* __restrict__ tw,
                     int tw_log_scale, PT ptw = nullptr, const Hook& hook = Hook{}) {
  using PL = FftPlan<N, E>;
  const int tid = threadIdx.x;
  const bool own = tid < PL::T;
  __syncthreads();
  if constexpr (PL::NPASS < 2) hook();
  fft_rec<N, E, 0, INV>(v, sm, tw, tw_log_scale, tid, own, ptw, hook);
}

// Several independent transforms per CTA (the large-n column kernels): the
// caller passes the thread's index inside its transform group and the
// group's own shared-memory buffers; barriers stay CTA-wide, so every group
// must run the same transform.
template <int N, int E, bool INV, class Hook = NoHook>
TSF_D void group_fft(double2 (&v)[E], double2* sm, const double2* __restrict__ tw,
                     int tw_log_scale, int tid, const Hook& hook = Hook{}) {
  __syncthreads();
  if constexpr (FftPlan<N, E>::NPASS < 2) hook();
  fft_rec<N, E, 0, INV>(v, sm, tw, tw_log_scale, tid, true,
                         static_cast<const double2*>(nullptr), hook);
}

// ------------------------------------------------------------ real input
// Forward DFTs of real data: no imaginary zeros are carried (x + 0.0 cannot
// be folded under IEEE rules, so a complex first pass on real data wastes
// registers and a quarter of its FLOPs) and the Hermitian half is mirrored.
TSF_D void dft2_real(const double* x, double2* X) {
  X[0] = make_double2(x[0] + x[1], 0.0);
  X[1] = make_double2(x[0] - x[1], 0.0);
}
TSF_D void dft4_real(double x0, double x1, double x2, double x3, double2* X) {
  const double t0 = x0 + x2, t1 = x0 - x2, t2 = x1 + x3, t3 = x1 - x3;
  X[0] = make_double2(t0 + t2, 0.0);
  X[1] = make_double2(t1, -t3);
  X[2] = make_double2(t0 - t2, 0.0);
  X[3] = make_double2(t1, t3);
}
TSF_D void dft8_real(const double* x, double2* X) {
  double2 Ev[4], Od[4];
  dft4_real(x[0], x[2], x[4], x[6], Ev);
  dft4_real(x[1], x[3], x[5], x[7], Od);
  // X_k = E_k + W8^k O_k, X_{k+4} = E_k - W8^k O_k, X_{8-k} = conj(X_k)
  X[0] = make_double2(Ev[0].x + Od[0].x, 0.0);
  X[4] = make_double2(Ev[0].x - Od[0].x, 0.0);
  const double2 w1 = w8_1<false>(Od[1]);
  X[1] = cadd(Ev[1], w1);
  X[5] = csub(Ev[1], w1);
  X[2] = make_double2(Ev[2].x, -Od[2].x);  // W8^2 = -i, O_2 real
  X[6] = make_double2(Ev[2].x, Od[2].x);
  X[3] = cconj(X[5]);
  X[7] = cconj(X[1]);
}
TSF_D void dft16_real(const double* x, double2* X) {
  // X_k = E_k + W16^k O_k over the even/odd halves (both real length 8)
  double ev[8], od[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ev[i] = x[2 * i];
    od[i] = x[2 * i + 1];
  }
  double2 E8[8], O8[8];
  dft8_real(ev, E8);
  dft8_real(od, O8);
  X[0] = make_double2(E8[0].x + O8[0].x, 0.0);
  X[8] = make_double2(E8[0].x - O8[0].x, 0.0);
  double2 w;
  w = w16<1, false>(O8[1]); X[1] = cadd(E8[1], w); X[9] = csub(E8[1], w);
  w = w16<2, false>(O8[2]); X[2] = cadd(E8[2], w); X[10] = csub(E8[2], w);
  w = w16<3, false>(O8[3]); X[3] = cadd(E8[3], w); X[11] = csub(E8[3], w);
  X[4] = make_double2(E8[4].x, -O8[4].x);  // W16^4 = -i, O_4 real
  X[12] = make_double2(E8[4].x, O8[4].x);
#pragma unroll
  for (int k = 5; k < 8; ++k) X[k] = cconj(X[16 - k]);
#pragma unroll
  for (int k = 13; k < 16; ++k) X[k] = cconj(X[16 - k]);
}

template <int R>
TSF_D void dft_real(const double* x, double2* X) {
  if constexpr (R == 2) {
    dft2_real(x, X);
  } else if constexpr (R == 4) {
    dft4_real(x[0], x[1], x[2], x[3], X);
  } else if constexpr (R == 8) {
    dft8_real(x, X);
  } else {
    static_assert(R == 16, "real first pass supports radix 2, 4, 8, 16");
    dft16_real(x, X);
  }
}

// First pass of a forward transform of real data (owned slots x[c],
// j = tid + c*T), then the remaining complex passes into v[c].
template <int N, int E, class Hook = NoHook, class PT = const double2*>
TSF_D void real_first_pass(const double (&x)[E], double2 (&v)[E], double2* sm,
                           const double2* __restrict__ tw, int tw_log_scale, int tid, bool own,
                           PT ptw = nullptr, const Hook& hook = Hook{}) {
  using PL = FftPlan<N, E>;
  constexpr int R = 1 << PL::log_radix(0);
  constexpr int Q = E / R;
  constexpr int T = PL::T;
  if (own) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double in[R];
      double2 out[R];
#pragma unroll
      for (int m = 0; m < R; ++m) in[m] = x[q + m * Q];
      dft_real<R>(in, out);
      const int base = (tid + q * T) * R;  // first pass: NS = 1, no twiddles
#pragma unroll
      for (int m = 0; m < R; ++m) sm[PL::pad(base + m)] = out[m];
    }
  }
  if constexpr (kAsyncStaging) cp_async_wait_all();
  __syncthreads();
  fft_rec<N, E, 1, false>(v, sm, tw, tw_log_scale, tid, own, ptw, hook);
}

// Forward transform of real owned slots x[c] (j = tid + c*T) into v[c].
template <int N, int E, class Hook = NoHook, class PT = const double2*>
TSF_D void block_fft_real(const double (&x)[E], double2 (&v)[E], double2* sm,
                          const double2* __restrict__ tw, int tw_log_scale,
                          PT ptw = nullptr, const Hook& hook = Hook{}) {
  static_assert(FftPlan<N, E>::NPASS >= 2, "real-input transform needs at least two passes");
  __syncthreads();
  const int tid = threadIdx.x;
  real_first_pass<N, E>(x, v, sm, tw, tw_log_scale, tid, tid < FftPlan<N, E>::T, ptw, hook);
}

template <int N, int E, class Hook = NoHook>
TSF_D void group_fft_real(const double (&x)[E], double2 (&v)[E], double2* sm,
                          const double2* __restrict__ tw, int tw_log_scale, int tid,
                          const Hook& hook = Hook{}) {
  static_assert(FftPlan<N, E>::NPASS >= 2, "real-input transform needs at least two passes");
  __syncthreads();
  real_first_pass<N, E>(x, v, sm, tw, tw_log_scale, tid, true,
                        static_cast<const double2*>(nullptr), hook);
}

}  // namespace tsf
