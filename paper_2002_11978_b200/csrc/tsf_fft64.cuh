// 4096-point fp64 transform as 64 x 64 inside one CTA (512 threads, 8
// complex slots per thread), with ONE CTA-wide exchange.
//
// Why: the radix-8 Stockham engine (tsf_fft.cuh) needs three
// CTA-wide shared-memory exchanges per 4096-point transform, each closed by
// __syncthreads, so all 16 warps of the SM run the same phase at once — all
// loading, then all in FP64 butterflies, then all storing (ncu: FP64 pipe
// 35-37%, shared-memory wavefronts 43-47%, i.e. the two pipes take turns).
// Here the transform is N = N1 x N2 = 64 x 64 (four-step, j = j1 + 64 j2,
// k = k2 + 64 k1):
//   stage A  for each column j1: 64-point DFT over j2 — done by one lane
//            OCTET (8 lanes x 8 slots): radix-8 in registers, W64 twiddle,
//            8 x 8 transpose through the octet's private shared tile
//            (__syncwarp only), radix-8 in registers
//   twiddle  W4096^(j1 k2)
//   exchange the one CTA-wide transpose (column -> row ownership)
//   stage B  for each row k2: 64-point DFT over j1, as stage A
// so warps drift apart between the two CTA barriers and one warp's shared
// traffic overlaps another's butterflies.  No digit reversal anywhere: the
// forward leaves the spectrum in the same slot pattern the inverse consumes.
//
// Ownership (both domains): slot c of thread t holds index
//     oidx(t, c) = (t >> 3) + 64 * ((t & 7) + 8 c)
// (real space: j1 = t >> 3, j2 = (t & 7) + 8c; frequency: k2 = t >> 3,
// k1 = (t & 7) + 8c).  A warp's global access at fixed c covers 4 runs of 8
// consecutive doubles (32-byte sectors fully used).
//
// Shared memory (complex elements): octet tiles 16 warps x 4 x (8 x 9) |
// exchange tile 64 x 65 | twiddle tables 1088 (tsf_fft64_tab.h, staged at
// kernel start by stage_fft64_tables).  Every access pattern is free of bank
// conflicts for 16-byte elements (row strides 9 and 65).
//
// Replaces numpy pocketfft at the reference call sites fourier.py:20-27
// (toeplitz.py:51-63, :131-136) for the n = 4096 systems of configs[2].
#pragma once

#include "tsf_fft.cuh"
#include "tsf_fft64_tab.h"

#ifndef TSF_FFT64
#define TSF_FFT64 0
#endif

namespace tsf {
namespace f64 {
constexpr int kLocStride = 9;                   // row stride of an octet's 8 x 8 tile
constexpr int kLocGroup = 8 * kLocStride;       // 72
constexpr int kLocWarp = 4 * kLocGroup;         // 288
constexpr int kLocElems = 16 * kLocWarp;        // 4608
constexpr int kGlbStride = 65;
constexpr int kGlbElems = 64 * kGlbStride;      // 4160
constexpr int kTabW64 = 0, kTabT1 = 64, kTabT2 = 576, kTabElems = 1088;
constexpr int kOffGlb = kLocElems;
constexpr int kOffTab = kLocElems + kGlbElems;
constexpr int kElems = kOffTab + kTabElems;     // 9856 complex = 157,696 bytes
constexpr int kBytes = kElems * 16;
}  // namespace f64

template <int N>
constexpr bool use64() {
  return TSF_FFT64 && N == 4096 && TSF_KE == 8;
}

// index held by slot c of thread tid (filters and Krylov kernels)
template <int N>
TSF_HD int oidx(int tid, int c) {
  if constexpr (use64<N>()) return (tid >> 3) + 64 * ((tid & 7) + 8 * c);
  else return tid + c * (N / TSF_KE);
}

// storage position of slot c of thread tid in the workspace vectors, the
// spectrum tables and the shared staging vector: thread-major, so a warp's
// access at fixed c is 32 consecutive doubles.  Equal to oidx for the
// Stockham engine; for the 64 x 64 engine the Krylov workspace vectors, the
// Strang spectra and the plan's spectrum tables are stored permuted this way
// (index oidx(t, c) at position spos(t, c)) — with the logical order a warp
// touched 8 lines per access (ncu: LSU/MIO throttling, 8-way conflicts on
// the staging vector).  Caller-visible vectors keep the natural order.
template <int N>
TSF_HD int spos(int tid, int c) {
  return tid + c * (N / TSF_KE);
}

// copy the twiddle tables into the transform region (published by the first
// transform's leading barrier)
TSF_D void stage_fft64_tables(double2* sm) {
  const double2* src = reinterpret_cast<const double2*>(&kF64Tab[0][0]);
  double2* dst = sm + f64::kOffTab;
  for (int i = threadIdx.x; i < f64::kTabElems; i += blockDim.x) dst[i] = ldt(&src[i]);
}

// One 64-point DFT held by a lane octet: v[c] = x[g + 8c] on entry (g = this
// lane's index in the octet), v[b] = X[g + 8b] on exit.
//   X[a + 8b] = sum_g W8^(g b) W64^(g a) sum_c x[g + 8c] W8^(c a)
template <bool INV>
TSF_D void f64_octet(double2 (&v)[8], double2* loc, const double2* w64, int g) {
#pragma unroll
  for (int a = 1; a < 8; ++a) {
    const double2 w = w64[a * 8 + g];
    v[a] = INV ? cmulc(v[a], w) : cmul(v[a], w);
  }
  // no barrier before the tile stores: the octet's previous readers of the
  // tile (the other stage, or the previous transform) are behind the
  // exchange's / the transform's leading __syncthreads
#pragma unroll
  for (int a = 0; a < 8; ++a) loc[a * f64::kLocStride + g] = v[a];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = loc[g * f64::kLocStride + k];
  dft8<INV>(v);
}

// inter-stage twiddle W4096^(+-j k2) and the CTA-wide exchange; entry: thread
// (p = tid >> 3, g) holds stage A's outputs at index g + 8b of its 64-point
// line p; exit: thread (p, g) holds line g + 8c's entry p in v[c]
template <bool INV>
TSF_D void f64_exchange(double2 (&v)[8], double2* sm, int p, int g) {
  const double2* tab = sm + f64::kOffTab;
  double2* glb = sm + f64::kOffGlb;
  const double2 t1 = tab[f64::kTabT1 + p * 8 + g];
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const double2 w = b == 0 ? t1 : cmul(t1, tab[f64::kTabT2 + b * 64 + p]);
    v[b] = INV ? cmulc(v[b], w) : cmul(v[b], w);
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) glb[p * f64::kGlbStride + g + 8 * b] = v[b];
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = glb[(g + 8 * c) * f64::kGlbStride + p];
}

// Full transform of the owned slots (oidx layout in, oidx layout out),
// unnormalised.  Every thread of the 512-thread CTA calls it.  Starts with a
// barrier (the caller may reuse shared memory right before; the previous
// transform's exchange readers are done); the hook runs between the stages.
template <bool INV, class Hook = NoHook>
TSF_D void fft64(double2 (&v)[8], double2* sm, const Hook& hook = Hook{}) {
  const int tid = tid_x();
  const int g = tid & 7, p = tid >> 3;
  double2* loc = sm + (tid >> 5) * f64::kLocWarp + ((tid >> 3) & 3) * f64::kLocGroup;
  const double2* w64 = sm + f64::kOffTab + f64::kTabW64;
  __syncthreads();
  dft8<INV>(v);
  f64_octet<INV>(v, loc, w64, g);
  hook();
  f64_exchange<INV>(v, sm, p, g);
  dft8<INV>(v);
  f64_octet<INV>(v, loc, w64, g);
}

// Forward transform of real owned slots x[c] (oidx layout) into v[c]: the
// first radix-8 works on real data (no imaginary zeros carried).
template <class Hook = NoHook>
TSF_D void fft64_real(const double (&x)[8], double2 (&v)[8], double2* sm,
                      const Hook& hook = Hook{}) {
  const int tid = tid_x();
  const int g = tid & 7, p = tid >> 3;
  double2* loc = sm + (tid >> 5) * f64::kLocWarp + ((tid >> 3) & 3) * f64::kLocGroup;
  const double2* w64 = sm + f64::kOffTab + f64::kTabW64;
  __syncthreads();
  {
    double in[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) in[c] = x[c];
    dft8_real(in, v);
  }
  f64_octet<false>(v, loc, w64, g);
  hook();
  f64_exchange<false>(v, sm, p, g);
  dft8<false>(v);
  f64_octet<false>(v, loc, w64, g);
}

}  // namespace tsf
