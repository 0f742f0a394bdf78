// Tensor-memory-accelerator (TMA) tile loads for the large-n column kernels.
//
// A column CTA of the four-step engine (tsf_large.cuh) works on G adjacent
// columns t2 of the N1 x N2 view of a length-n vector (j = N2 t1 + t2): one
// [N1 rows x G] tile per operand vector, and an [N1 x G] complex tile per
// transform channel of the work array Z.  With plain loads every thread
// issued E global loads per operand and the CTA waited on all of them
// (ncu, profiles/r01d_large_ncu.md: k_lcol_fwd 26% issue, 6.4 warps per
// issue on long-scoreboard).  Here ONE elected thread issues each tile as a
// cp.async.bulk.tensor (UTMALDG) box load straight into shared memory,
// completing on an mbarrier with the byte count; the CTA stages its twiddle
// table and instance state meanwhile, then waits once and reads its slots
// from the tile (conflict-free: a warp reads consecutive doubles).
//
// Tensor maps are 3-D {N2, N1, B} views of [B][n] vectors (n = N1 N2: the
// power-of-two sizes of every BASELINE config; other n keep the plain-load
// path) with boxes {G, rows <= 256, 1}; columns longer than 256 take several
// boxes.  They are encoded on the host (cuTensorMapEncodeTiled through the
// runtime's driver entry point) and passed as __grid_constant__ parameters.
#pragma once

#include <cuda.h>

#include "tsf_common.cuh"

namespace tsf {

// Maps of one column launch: operand vectors (up to 3) and the two Z channels.
struct alignas(64) ColMaps {
  CUtensorMap v[3];   // operand vectors (mode dependent); unused slots zero
  CUtensorMap z;      // Z as doubles {2 N2, N1, 2 B}: channel c of instance b is plane c B + b
  int nv;             // operand vectors with a map
  int use;            // 1: the kernel loads through the maps
};

constexpr int kTmaMaxBox = 256;

TSF_D unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

TSF_D void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
TSF_D void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
TSF_D void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 3-D box load {c0, c1, c2} of `map` into shared memory at dst
TSF_D void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                     unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}

// Issue the [rows x cols] tile at (col0, row 0, plane) of `map` in boxes of
// at most 256 rows; returns the bytes that will land (elem = element bytes).
TSF_D unsigned tma_tile(double* dst, const CUtensorMap* map, int col0, int rows, int cols,
                        int plane, int elem, unsigned long long* bar) {
  for (int r0 = 0; r0 < rows; r0 += kTmaMaxBox)
    tma_load3(reinterpret_cast<char*>(dst) + (size_t)r0 * cols * elem, map, col0, r0, plane, bar);
  return (unsigned)(rows * cols * elem);
}

// host side (tsf_large.cu): encode / cache the maps of a launch
int tma_map_vector(CUtensorMap* m, const double* base, long n, int N1, int N2, int B, int G);
int tma_map_z(CUtensorMap* m, const double2* Z, int N1, int N2, int B, int G);
int tma_mode();   // TSF_TMA: bit 0 column-forward tiles, bit 1 column-inverse tiles
// the half-length column kernels (tsf_hlarge.cuh): TSF_TMA_HALF, default 2 —
// the Z tiles of k_hcol_inv (measured neutral on configs[3]; the operand
// tiles of k_hcol_fwd measured 0.4% slower), and only for launches of two
// waves or more (each map costs a host-side cache lookup per launch, which a
// latency-bound single small instance notices: configs[1] 0.70 -> 0.76 ms per
// level)
int tma_half_mode();

}  // namespace tsf
