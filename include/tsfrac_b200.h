/*
 * tsfrac_b200 — C ABI of the B200-native FIDS per-time-step solve.
 *
 * Drop-in boundary for the reference Python package `tsfrac`
 * (/root/reference/pkg/src/tsfrac).  Every entry point below names the
 * reference function it replaces.  Plain pointers and sizes only; all
 * vector arguments are DEVICE pointers (fp64, contiguous, instance-major
 * [B][n]) unless documented as host.  `stream` is a cudaStream_t (NULL =
 * legacy default stream).  Nothing is freed across the ABI: the plan owns
 * its tables and workspaces, the caller owns every I/O buffer.
 *
 * Return value: TSF_SUCCESS (0) or a negative TSF_E* code; the message is
 * available from tsf_last_error() (thread-local).  Numerical outcomes of
 * a solve (breakdowns, non-convergence, kappa <= 0, indefinite
 * preconditioner) are reported per instance in `status` using the
 * TSF_ST_* codes, which the Python layer maps to the reference's
 * KrylovReport.breakdown strings and exceptions.
 */
#ifndef TSFRAC_B200_H
#define TSFRAC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSF_ABI_VERSION 4

/* API return codes */
#define TSF_SUCCESS 0
#define TSF_E_INVALID (-1)     /* bad argument (reference: ValueError) */
#define TSF_E_CUDA (-2)        /* CUDA runtime error */
#define TSF_E_UNSUPPORTED (-3) /* size / mode not built (e.g. non-pow2 n with precond) */
#define TSF_E_NOMEM (-4)

/* per-instance status codes (solve outcomes) */
#define TSF_ST_OK 0
#define TSF_ST_NOT_CONVERGED 1
#define TSF_ST_RHO_VANISHED 2          /* "rho vanished"               krylov.py:119-121 */
#define TSF_ST_R0V_VANISHED 3          /* "r0.v vanished"              krylov.py:130-132 */
#define TSF_ST_OMEGA_DEN_VANISHED 4    /* "omega denominator vanished" krylov.py:141-143 */
#define TSF_ST_OMEGA_VANISHED 5        /* "omega vanished"             krylov.py:151-152 */
#define TSF_ST_NONPOS_CURVATURE 6      /* "non-positive curvature"     krylov.py:72-74   */
#define TSF_ST_KAPPA_NONPOS 7          /* ValueError                   scheme.py:156-160 */
#define TSF_ST_PRECOND_NONPOS 8        /* PreconditionerError          toeplitz.py:122-124 */

typedef struct tsf_plan tsf_plan;

int tsf_abi_version(void);
const char* tsf_last_error(void);

/*
 * Plan for one spatial size n (reference: ToeplitzOperator built by
 * build_toeplitz, toeplitz.py:34-48, plus the level-independent part of
 * build_preconditioner, toeplitz.py:101-128).
 *   L          circulant embedding length (power of two >= 2n-1, >= 32,
 *              <= 2^25).  L <= 8192: one CTA per instance (single-CTA engine);
 *              above: the four-step multi-kernel engine.  Any n.
 *   symbol_re  HOST, L reals: Re FFT_L(even embedding of the first column)
 *   lam        HOST, n reals: Re FFT_n(strang_first_column) for the fused
 *              Strang kernels (power-of-two n >= 16 with L = 2n), or NULL.
 *              Other n apply the Strang preconditioner as circ(IFFT(1/total))
 *              through a second plan whose symbol is that circulant's
 *              (toeplitz.py _circulant_plan in the Python layer).
 *   device     CUDA ordinal the plan lives on
 * All entry points below are stream-ordered.  For L <= 8192 the level solve
 * is one CUDA graph launch with a conditional WHILE loop and returns without
 * waiting (TSF_SOLVE_GRAPH=0 selects the host-polled loop); the four-step
 * engine's solve polls a device counter every 4 iterations (stream sync).
 */
int tsf_plan_create(tsf_plan** plan, int n, int L, const double* symbol_re,
                    const double* lam, int device);
int tsf_plan_destroy(tsf_plan* plan);
/* out[0]=n out[1]=L out[2]=N_mv(=L/2) out[3]=has_precond out[4]=max_batch_reserved */
int tsf_plan_info(const tsf_plan* plan, int64_t* out5);
/* reserve Krylov workspaces for `batch` instances (done lazily otherwise) */
int tsf_plan_reserve(tsf_plan* plan, int batch);

/*
 * y = shift*x + kappa .* (A x)  for B instances.
 * Reference: toeplitz_matvec (toeplitz.py:51-63) and the level closure
 * apply(v) (scheme.py:129-130).  kappa == NULL gives the bare y = A x.
 */
int tsf_toeplitz_matvec(tsf_plan* plan, int B, const double* x, double* y,
                        const double* kappa, double shift, void* stream);

/*
 * z = P^{-1} v with P = shift*I + kappa_bar*s(A)  (Strang circulant).
 * Reference: precond_solve (toeplitz.py:131-136) of build_preconditioner(
 * d, shift, kappa_bar) (toeplitz.py:101-128).  kappa_bar_dev (device, [B])
 * overrides kappa_bar per instance when non-NULL.  Requires pow2 n.
 */
int tsf_precond_solve(tsf_plan* plan, int B, const double* v, double* z,
                      double shift, double kappa_bar, const double* kappa_bar_dev,
                      void* stream);

/*
 * One level solve (shift*I + diag(kappa) A) x = rhs for B instances, x0 = 0.
 * Reference: _LevelSolver.solve (scheme.py:120-143) -> solve_bicgstab
 * (krylov.py:88-153) or solve_cg (krylov.py:43-85).  The preconditioner uses
 * kappa_bar when > 0, else kappa_bar = mean(kappa) formed on the device
 * (scheme.py:135).
 *   method      0 = BiCGSTAB, 1 = CG
 *   precond     0 = none ("krylov"), 1 = Strang ("pkrylov")
 *   max_iters   <= 0 means the reference default 10*n
 *   iters, relres, status: device [B]
 */
int tsf_krylov_solve(tsf_plan* plan, int B, int method, int precond,
                     const double* rhs, double* x, const double* kappa, double shift,
                     double kappa_bar, double tol, int max_iters, int* iters, double* relres, int* status,
                     void* stream);

/*
 * Level solve with the circulant preconditioner of a NON-power-of-two n
 * (n <= 4096).  Reference: build_preconditioner + precond_solve
 * (toeplitz.py:101-136) — P^{-1} v = Re IFFT_n(FFT_n(v) / total) — which in
 * exact arithmetic is the symmetric Toeplitz product with the circulant's
 * first column c = Re IFFT_n(1/total); the fused level-solve kernels apply it
 * through the same even/odd-bin filters as the operator.
 *   pc_spec    device [B or 1][L/2] pairs (S_2k, S_2k+1)/L of the length-L
 *              embedding of c (natural bin order; the even part of the
 *              symbol, as tsf_plan_create stores the operator's), stride
 *              pc_stride pairs per instance (0: one table for every instance)
 * Other arguments as tsf_krylov_solve (precond implied).
 */
int tsf_krylov_solve_circ(tsf_plan* plan, int B, int method, const double* rhs, double* x,
                          const double* kappa, double shift, const double* pc_spec,
                          int64_t pc_stride, double tol, int max_iters, int* iters,
                          double* relres, int* status, void* stream);

/*
 * SOE accumulator update fused with the next level's right-hand side.
 * Reference: history_push (soe.py:209-225) followed by the history term and
 * RHS assembly of the next level (scheme.py:279-284; fast_caputo_rhs,
 * soe.py:228-246).
 *   W        [B][nexp][n] accumulators (updated in place when do_push)
 *   u, uprev [B][n]  level just solved and the one before (push uses u-uprev)
 *   decay, coef, hcoef  device [nexp]: e^{-s tau}, -expm1(-s tau)/s,
 *            w e^{-s tau_next}
 *   f        [B][n] source at the next level (may be NULL when !do_rhs)
 *   rhs      [B][n] output: f + (a_next*u - H)/G
 */
int tsf_soe_push_rhs(int B, int n, int nexp, double* W, const double* u,
                     const double* uprev, double tau_push, const double* decay,
                     const double* coef, const double* hcoef, int do_push, int w_zero,
                     int do_rhs, double a_next, double G, const double* f, double* rhs,
                     void* stream);

/*
 * Direct L1 history right-hand side of the DIDS scheme (reference: run_dids,
 * scheme.py:208-216 — `rhs = f + (a[0]/G) hist[0]; rhs += (diff(a) @ hist[1:m])/G`
 * with a = l1_weights(mesh, gamma, m).a, mesh.py:53-80):
 *   rhs_i = (f_i + c0 * hist[0]_i) + (sum_{k=1}^{rows-1} w[k-1] * hist[k]_i) / G
 *   rows         m (levels 0..m-1 of the history are read)
 *   hist         [B] x [rows][n] (instance b at hist + b*inst_stride)
 *   w            device [rows-1]: diff(a)  (unused when rows == 1)
 *   c0           a[0] / G (host scalar, formed as the reference does)
 *   f, rhs       [B][n]
 */
int tsf_l1_history_rhs(int B, int n, int rows, const double* hist, int64_t inst_stride,
                       const double* w, double c0, double G, const double* f, double* rhs,
                       void* stream);

/* Coefficient field  g(x_i, t_m) = sum_q modes_m[q][b][i] * coef[m][q], where
 * modes_m = modes + m*t_stride.  Separable fields use t_stride = 0; a field
 * tabulated per level (arbitrary callables evaluated on the host, as the
 * reference does at scheme.py:156-160,283) uses one mode, coef = 1 and
 * t_stride = B*n. */
typedef struct tsf_field {
  int nmodes;            /* 0..4 */
  const double* modes;   /* device; mode q of instance b at modes_m + q*q_stride + b*b_stride */
  int64_t q_stride;
  int64_t b_stride;      /* 0 = shared by all instances */
  int64_t t_stride;      /* per-level offset of the mode block (0 = time-independent modes) */
  const double* coef;    /* HOST [M+1][nmodes]: coefficients at t_0..t_M */
} tsf_field;

/*
 * Native FIDS time march (reference: run_fids loop body, scheme.py:276-294)
 * for B independent instances that share (gamma, alpha, n, M, r): launches
 * 2 kernels per level on `stream`, no host synchronisation.
 *   u_buf0/u_buf1  [B][n]: u^0 in u_buf0 on entry; level m lands in
 *                  u_buf[m & 1]
 *   W              [B][nexp][n], zero on entry when m_begin == 1
 *   shift, a_mm, tau  HOST [M]: level m at index m-1
 *   soe_tab        device [M][3][nexp]: decay_m, coef_m, hcoef_m
 *                  (hcoef_m = w e^{-s tau_m}) for levels 1..M
 *   iters, relres, status  device [M][B]
 *   hist           device [(M+1)][hist_B][n] or NULL: per-level copy of
 *                  the first hist_B instances
 *   Levels m_begin .. m_end-1 are run (1 <= m_begin <= m_end <= M+1); when
 *   m_end == M+1 the final history push is applied as well.
 */
typedef struct tsf_march {
  int B, M, nexp;
  int method, precond;
  double tol;
  int max_iters;
  double G;
  const double* shift;
  const double* a_mm;
  const double* tau;
  const double* soe_tab;
  tsf_field kappa;
  tsf_field source;
  double* u_buf0;
  double* u_buf1;
  double* W;
  double* rhs;
  double* kwork;
  int* iters;
  double* relres;
  int* status;
  double* hist;
  int hist_B;
  int m_begin;
  int m_end;
  /* optional per-level timing: 3 cudaEvent_t per level run (before the SOE
   * kernel, between the SOE and solve kernels, after the solve kernel),
   * recorded on `stream`; NULL disables */
  void** events;
  /* Blocked SOE schedule (soe_block = K in 2..16; 0 or 1: one W pass per
   * level).  One pass over W per K levels advances W by the block's K pushes
   * (bit-identical recurrence) and forms the W-part of the block's history
   * terms; each level adds a combination of the block's du vectors.
   *   soe_alpha  device [M][nexp]: alpha_j(m) = h_j(m) prod_{l=mb+1}^{m-1} d_j(l),
   *              mb = K*floor((m-1)/K) the base of level m's block
   *   soe_beta   HOST [M][16]: beta(m, mb+1+q) = sum_j h_j(m) prod_{l=mb+2+q}^{m-1} d_j(l) c_j(mb+1+q)
   *   soe_ring   device [2][K][B][n] scratch (du and history-term rings),
   *              kept between calls of the same march */
  int soe_block;
  const double* soe_alpha;
  const double* soe_beta;
  double* soe_ring;
} tsf_march;

int tsf_fids_march(tsf_plan* plan, const tsf_march* desc, void* stream);

/* Debug / test hook: B complex FFTs of length N (pow2, 16..8192) through the
 * block Stockham engine.  inverse != 0 gives the unnormalised inverse. */
int tsf_fft_debug(int N, int inverse, int B, const double* in, double* out, void* stream);

/* Test hook for the half-length transform engine of the level solve
 * (csrc/tsf_half.cuh; power-of-two n, 512 <= n <= 4096), the device form of
 * toeplitz.py:131-136 (mode 0) and toeplitz.py:51-63 + scheme.py:129-130
 * (mode 1):
 *   mode 0: out[B][n] = Re IFFT_n(FFT_n(x) . aux), aux[B][n] = the real even
 *           filter S_k / n; hs[B][n/2+1] (complex, interleaved) receives the
 *           filtered half spectrum.
 *   mode 1: out = shift*x + aux .* (A x) for x = Re IFFT_n(hs) (aux = kappa).
 * Returns TSF_E_UNSUPPORTED when the size is outside the engine. */
int tsf_half_debug(tsf_plan* plan, int mode, int B, const double* x, const double* aux,
                   double shift, double* hs, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TSFRAC_B200_H */
