// Common device helpers for the tsfrac B200 kernels (fp64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define TSF_HD __host__ __device__ __forceinline__
#define TSF_D __device__ __forceinline__

// ---------------------------------------------------------------- complex
TSF_HD double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
TSF_HD double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
TSF_HD double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
TSF_HD double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
TSF_HD double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
TSF_HD double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) / +i (inverse)
template <bool INV>
TSF_HD double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// Read-only table load that the compiler may neither hoist across barriers
// nor CSE between the many inlined transforms of a solve: plain __ldg table
// reads are identical in every FFT of a Krylov iteration, so ptxas kept all
// of them live across the whole loop and spilled.  The
// re-read hits L1.
// Asynchronous global -> shared copies (16 bytes, L2 only); completion is
// awaited with cp_async_wait_all() followed by a barrier.
TSF_D void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may be scheduled while
// its predecessor still runs; pdl_enter() blocks until the predecessor grid
// has completed (its writes visible), then lets the next kernel launch.
// Both are no-ops for a normal launch.  Every kernel that can follow another
// in a PDL chain calls it first, before touching any memory.
TSF_D void pdl_enter() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
TSF_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
TSF_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
TSF_D void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Software prefetch of a whole vector (one 128-byte line per thread and
// step): into L2 at phase start for the vectors an epilogue reads after
// the transforms, into L1 right before the last transform for the ones read
// first (ncu: the epilogue loads of kappa / rhs were the top stalls).
#ifndef TSF_PREFETCH
#define TSF_PREFETCH 1
#endif
TSF_D void prefetch_l2(const double* p, int n) {
  if (!TSF_PREFETCH) return;
  for (int i = 16 * threadIdx.x; i < n; i += 16 * blockDim.x)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + i));
}
TSF_D void prefetch_l1(const double* p, int n) {
  if (!TSF_PREFETCH) return;
  for (int i = 16 * threadIdx.x; i < n; i += 16 * blockDim.x)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p + i));
}

TSF_D double2 ldt(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// threadIdx.x that the compiler cannot CSE: each transform pass recomputes
// its handful of shared-memory addresses instead of ptxas hoisting the
// addresses of every pass of every transform to kernel entry (where they
// were spilled).
TSF_D int tid_x() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

// 1/x for positive normal x without the IEEE division's slow-path call (a
// call inside an unrolled transform forces every live register to the stack).
// rcp.approx + two Newton steps + a final residual correction: within 1 ulp
// of the correctly rounded reciprocal (measured against __drcp_rn in tests).
TSF_D double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return fma(r, fma(-x, r, 1.0), r);
}

// ---------------------------------------------------------------- status
// Per-instance status codes; the host maps them to the reference's
// exceptions / KrylovReport.breakdown strings (krylov.py:72-152,
// scheme.py:139-142,156-160, toeplitz.py:117-124).
enum TsfStatus : int {
  TSF_OK = 0,
  TSF_NOT_CONVERGED = 1,
  TSF_BD_RHO = 2,          // "rho vanished"
  TSF_BD_R0V = 3,          // "r0.v vanished"
  TSF_BD_OMEGA_DEN = 4,    // "omega denominator vanished"
  TSF_BD_OMEGA = 5,        // "omega vanished"
  TSF_BD_CURVATURE = 6,    // "non-positive curvature"
  TSF_KAPPA_NONPOS = 7,    // kappa <= 0 somewhere on the grid
  TSF_PRECOND_NONPOS = 8,  // shift + kappa_bar*lambda <= 0
};

// ---------------------------------------------------------------- reductions
template <int NV>
struct Vals {
  double v[NV];
};

// Block-wide sum of NV doubles; every thread receives the result.
// `scratch` must hold NV * 32 doubles.  Contains two __syncthreads.
template <int NV>
TSF_D Vals<NV> block_sum(Vals<NV> a, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = a.v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    a.v[k] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[k * 32 + warp] = a.v[k];
  }
  __syncthreads();
  Vals<NV> r;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double x = (lane < nwarps) ? scratch[k * 32 + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    r.v[k] = x;
  }
  __syncthreads();
  return r;
}

TSF_D double block_sum1(double a, double* scratch) {
  Vals<1> v;
  v.v[0] = a;
  return block_sum<1>(v, scratch).v[0];
}

TSF_D double block_min1(double a, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
  if (lane == 0) scratch[warp] = a;
  __syncthreads();
  double x = (lane < nwarps) ? scratch[lane] : 1e308;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
  __syncthreads();
  return x;
}
