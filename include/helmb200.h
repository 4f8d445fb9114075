/*
 * helmb200.h — C ABI of libhelmb200.so, the B200 (sm_100a) hot path of the
 * two-level Bezier-Schwarz preconditioned GMRES solver of arXiv 2408.03571.
 *
 * Every entry point below replaces one operator of the reference Python
 * package `helmdd` (paths relative to /root/reference/pkg/src/helmdd):
 *
 *   helm_apply_A         <- `A @ x` on the assembled CSR matrix
 *                           (gmres.py:62,85,110,153,173; schwarz.py:88;
 *                            coefficients discretization.py:130-191)
 *   helm_restrict        <- `cs.r0 @ r`            (coarse.py:174, R0 from coarse.py:102-139)
 *   helm_prolong         <- `cs.r0.T @ y`          (coarse.py:174)
 *   helm_coarse_solve    <- `linalg.solve(cs.a0_factorization, c)` (coarse.py:174 -> linalg.py:90-95)
 *   helm_coarse_correct  <- `coarse_correct(cs, r)` (coarse.py:170-174)
 *   helm_local_sum       <- `SchwarzPreconditioner._local_sum` (schwarz.py:64-74)
 *   helm_apply_M         <- `SchwarzPreconditioner.apply` (schwarz.py:76-103)
 *   helm_cgs2            <- the MGS + conditional re-orthogonalisation block (gmres.py:112-127)
 *   helm_givens          <- the Givens update + residual estimate (gmres.py:129-148)
 *   helm_gmres           <- `gmres(A, M_inv, b, cfg)` (gmres.py:65-177)
 *   helm_gmres_multi     <- that loop over several right-hand sides, operators batched
 *                           (no reference counterpart: SURVEY §8 f4)
 *
 * Conventions
 *  - Every function returns an int status: 0 = OK, nonzero = error; the
 *    message is available from helm_last_error() (thread-local).  No C++
 *    exception crosses the ABI.
 *  - Scalars are fp64 for real problems (MP-1, Dirichlet) and interleaved
 *    complex128 {re, im} for complex problems (MP-2, Sommerfeld); the
 *    `is_complex` flag of the descriptor selects which.
 *  - Vector arguments are DEVICE pointers owned by the caller, contiguous,
 *    laid out [batch][len] with the unknown index of discretization.py:74-77
 *    (row-major in y, x fastest).  Coarse vectors are [batch][m0*m0],
 *    row-major in the coarse y index.
 *  - Every compute call takes a cudaStream_t (passed as void*) and is
 *    asynchronous on it.  Only helm_gmres synchronises (it reads one scalar
 *    per iteration, like the reference's Python loop reads its estimate).
 *  - A plan is immutable after creation (schwarz.py:32).  Mutable scratch
 *    lives in a helm_workspace; concurrent callers use distinct workspaces.
 */
#ifndef HELMB200_H
#define HELMB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HELM_ABI_VERSION 6

enum helm_bc { HELM_DIRICHLET = 0, HELM_SOMMERFELD = 1 };
enum helm_kind { HELM_AS2 = 0, HELM_SAS2 = 1, HELM_SHS2 = 2 };

typedef struct helm_plan helm_plan;
typedef struct helm_workspace helm_workspace;

/* Setup data (host pointers; copied to the device by helm_plan_create).
 * "S" below = double (is_complex = 0) or double[2] (is_complex = 1).       */
typedef struct helm_desc {
  int32_t n;             /* grid nodes per dimension (discretization.py:36-51)     */
  int32_t bc;            /* helm_bc                                               */
  int32_t is_complex;    /* 0: fp64 (MP-1); 1: complex128 (MP-2)                  */
  int32_t kind;          /* helm_kind (schwarz.py:28)                             */
  int32_t weights_before_solve; /* schwarz.py:69-70                               */
  int32_t p;             /* subdomains per dimension (decomposition.py:89-103)    */
  int32_t overlap_layers;/* m of extend(part, m) (decomposition.py:111-134)       */
  int32_t ratio;         /* coarse ratio H/h (coarse.py:77-81)                    */
  double k;              /* wavenumber                                            */
  /* --- 1-D boxes (identical in x and y): box a covers unknowns
   *     [box_start[a], box_start[a] + box_len[a])                               */
  const int32_t* box_start;   /* [p]                                             */
  const int32_t* box_len;     /* [p]                                             */
  const int32_t* box_class;   /* [p]   local eigen-class of box a                */
  int32_t n_classes;          /* distinct 1-D local pencils                      */
  const int32_t* class_len;   /* [n_classes]                                     */
  const void* class_V;        /* S, concatenated [L][L] row-major per class,
                                 T V = W V diag(lambda), V^T W V = I             */
  const void* class_lambda;   /* S, concatenated [L] per class                   */
  /* --- coarse level (HOCS ratio 2, coarse.py:148-174):
   *     A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0  (y (x) x), solved by a fast
   *     sine/cosine transform along x, one pivoted pentadiagonal solve per
   *     x-mode along y, and (Sommerfeld) a Woodbury correction on n_strip
   *     columns whose capacitance is 4x4-block-diagonal in the y-pencil
   *     eigenbasis.  coarse_scale == NULL -> plan without a coarse solver.     */
  int32_t m0;                 /* coarse unknowns per dimension                   */
  const double* coarse_scale; /* [m0]  forward pre-scale sigma_a                 */
  const double* coarse_lamT;  /* [m0]  Dirichlet: DST eigenvalues of T0          */
  const double* coarse_lamM;  /* [m0]  Dirichlet: DST eigenvalues of M0          */
  double coarse_qn;           /* Dirichlet DST normalisation 2/(m0+1)            */
  const void* t0_band;        /* S [m0][5]   T0[i][i+d-2]                        */
  const void* m0_band;        /* S [m0][5]   M0[i][i+d-2]                        */
  /* Sommerfeld: pivoted band LU of T0 + s_a M0, stored [row][a] (coalescing) */
  const uint8_t* band_piv;    /* [m0][m0] pivot offset 0..2                      */
  const void* band_l;         /* S [m0][m0][2] multipliers                       */
  const void* band_u;         /* S [m0][m0][5] {1/U_jj, U_j,j+1 .. U_j,j+4}      */
  int32_t n_strip;            /* 0 (Dirichlet) or 4 (Sommerfeld)                 */
  const double* strip_q;      /* [m0][n_strip]  Q[strip_x[i], a]                 */
  /* The y-pencil is reflection symmetric, so its modes are even (first he = (m0+1)/2)
   * or odd (last ho = m0/2); the three mode matrices are passed as packed half-size
   * blocks [A_e (he x he) row-major, A_o (ho x ho) row-major]:
   *   left  (V^T M0, V^T): A_e acts on Z[y] + Z[m0-1-y] (Z[h] alone when m0 is odd),
   *                        A_o on Z[y] - Z[m0-1-y]  (y < he / ho);
   *   right (M0 V):        E = A_e c_even, O = A_o c_odd, out[y] = E + O,
   *                        out[m0-1-y] = E - O.                                     */
  const void* cap_left;       /* S packed  V^T M0 (V: y-pencil eigenvectors)     */
  const void* cap_right;      /* S packed  M0 V                                  */
  const void* cap_mode;       /* S [m0][n_strip][n_strip]                        */
  /* strip-space refinement: after the second band pass the exact strip residual
   * rho = c_S - C_U y_S is formed from the band-pass strip values and one more band
   * pass applies B^{-1} of (I - H G) rho (the eigen-space H, G are only ~1e-12
   * accurate; the band passes are exact), see coarse.cu                          */
  const void* cap_vt;         /* S packed  V^T                                   */
  const void* cap_hg;         /* S [m0][n_strip][n_strip]  cap_mode_b Gamma_b     */
  const void* strip_lt;       /* S [n_strip][n_strip]  (T0 - T~) on the strips    */
  const void* strip_lm;       /* S [n_strip][n_strip]  (M0 - M~) on the strips    */
  int32_t strip_refine;       /* strip-refinement steps (Sommerfeld; 0..4)        */
  int32_t refine_steps;       /* full iterative-refinement steps r = c - A0 y    */
  /* --- general coarse spaces (FOCS at any ratio, HOCS at ratio 4/8/16;
   *     coarse.py:84-151): R0 = P (x) P with a banded 1-D P, and
   *     A0^{-1} c = (V (x) V) diag(invden) (V (x) V)^T c with T0 V = M0 V diag(lam),
   *     V^T M0 V = I (T0 = P T P^T, M0 = P W P^T), followed by refine_steps
   *     iterative-refinement steps r = c - A0 y on the reference's own Galerkin matrix
   *     A0 = (B + B^T)/2, B = R0 A R0^T (coarse.py:154-165), passed as a 2-D stencil of
   *     (2b+1)^2 coefficients per coarse unknown.  coarse_V == NULL -> the HOCS ratio-2
   *     fast solver above (coarse_scale ...).                                         */
  int32_t coarse_kind;        /* 0: HOCS, 1: FOCS                                  */
  int32_t p_width;            /* taps per row of P                                 */
  const int32_t* p_start;     /* [m0]  first fine unknown of row I of P            */
  const double* p_taps;       /* [m0][p_width]  P[I][p_start[I] + t] (zero-padded) */
  int32_t pt_width;           /* taps per row of P^T                               */
  const int32_t* pt_start;    /* [nu]  first coarse unknown of row i of P^T        */
  const double* pt_taps;      /* [nu][pt_width]                                    */
  int32_t a0_bw;              /* half-bandwidth b of A0 along each axis (1..8)      */
  const void* a0_stencil;     /* S [m0*m0][(2b+1)^2]  A0[(Iy,Ix)][(Iy+dy,Ix+dx)],
                                 (dy+b)(2b+1) + dx+b (zero outside the grid)          */
  const void* coarse_V;       /* S [m0][m0]  row-major                             */
  const void* coarse_invden;  /* S [m0][m0]  1 / (lam[y] + lam[x] - k^2)           */
} helm_desc;

typedef struct helm_gmres_report {
  int32_t iterations;
  int32_t converged;
  int32_t breakdown;
  int32_t reorth;        /* iterations whose re-orthogonalisation pass ran (gmres.py:117-120) */
  double final_residual;
  double wall_seconds;
} helm_gmres_report;

int32_t helm_abi_version(void);
/* number of libhelmb200 kernels launched by this process so far (cuBLAS not counted) */
uint64_t helm_kernel_launches(void);
const char* helm_last_error(void);

int helm_plan_create(const helm_desc* desc, helm_plan** out);

/* Native setup (no host-side numpy / LAPACK): the problem parameters alone.  The library builds
 * every helm_desc array itself -- the 1-D box classes and their eigen-pairs (cuSOLVER on the
 * device), the coarse transform eigenvalues, band LU factors and Woodbury data -- and creates the
 * plan (the HOCS ratio-2 coarse space; other coarse spaces go through helm_plan_create).
 * Replaces the reference's setup: assemble + partition/extend + build_hocs + galerkin +
 * SchwarzPreconditioner.__init__ (discretization.py:157-191, decomposition.py:89-134,
 * coarse.py:148-167, schwarz.py:34-62).                                                          */
typedef struct helm_problem {
  int32_t n;                    /* grid nodes per dimension                                */
  int32_t bc;                   /* helm_bc (MP-1 Dirichlet fp64, MP-2 Sommerfeld c128)     */
  int32_t kind;                 /* helm_kind                                               */
  int32_t weights_before_solve; /* schwarz.py:69-70                                        */
  int32_t p;                    /* subdomains per dimension                                */
  int32_t overlap_layers;       /* extend(part, m)                                         */
  int32_t coarse_kind;          /* 0: HOCS                                                 */
  int32_t ratio;                /* 2                                                       */
  double k;                     /* wavenumber                                              */
  int32_t strip_refine;         /* -1: default (1)                                         */
  int32_t refine_steps;         /* -1: default (0)                                         */
} helm_problem;
int helm_plan_create_problem(const helm_problem* problem, helm_plan** out);
int helm_plan_destroy(helm_plan* plan);
int64_t helm_plan_num_unknowns(const helm_plan* plan);
int64_t helm_plan_num_coarse(const helm_plan* plan);

int helm_workspace_create(const helm_plan* plan, int32_t max_batch, helm_workspace** out);
int helm_workspace_destroy(helm_workspace* ws);

/* y = A x  (x, y: [batch][N]) */
int helm_apply_A(const helm_plan* plan, const void* x, void* y, int32_t batch, void* stream);
/* y = x - A z  (the SHS2 deflation, schwarz.py:88) */
int helm_deflate(const helm_plan* plan, const void* x, const void* z, void* y, int32_t batch, void* stream);
/* c = R0 x  (c: [batch][m0*m0]) */
int helm_restrict(const helm_plan* plan, const void* x, void* c, int32_t batch, void* stream);
/* z = R0^T c */
int helm_prolong(const helm_plan* plan, const void* c, void* z, int32_t batch, void* stream);
/* y = A0^{-1} c (c and y may alias) */
int helm_coarse_solve(const helm_plan* plan, helm_workspace* ws, const void* c, void* y,
                      int32_t batch, void* stream);
/* z = R0^T A0^{-1} R0 x */
int helm_coarse_correct(const helm_plan* plan, helm_workspace* ws, const void* x, void* z,
                        int32_t batch, void* stream);
/* y = base + sum_i R_i^T [D_i] A_i^{-1} [D_i] R_i x; base may be NULL (zeros).
 * weighted = 0 -> AS2 form, 1 -> SAS2/SHS2 form (placement per weights_before_solve). */
int helm_local_sum(const helm_plan* plan, helm_workspace* ws, const void* x, const void* base,
                   void* y, int32_t weighted, int32_t batch, void* stream);
/* y = M^{-1} x for the plan's kind (AS2 / SAS2 / SHS2) */
int helm_apply_M(const helm_plan* plan, helm_workspace* ws, const void* x, void* y,
                 int32_t batch, void* stream);

/* Arnoldi step on a Krylov basis V [(j+2)][N] (V[j+1] holds w on entry):
 * classical Gram-Schmidt run twice; hcol[0..j+1] receives the new Hessenberg
 * column (h1 + h2, then ||w||), V[j+1] the normalised vector unless breakdown. */
int helm_cgs2(const helm_plan* plan, helm_workspace* ws, void* V, int32_t j, void* hcol,
              void* stream);
/* Givens QR update of column j of H [(max_iter+1)][max_iter] (row-major,
 * column j at H + j, stride max_iter); cs, sn, g as in gmres.py:94-96.
 * Writes est_out[0] = |g[j+1]| / beta, est_out[1] = breakdown flag (0/1). */
int helm_givens(const helm_plan* plan, void* H, int32_t ldh, int32_t j, void* cs, void* sn,
                void* g, double beta, double* est_out, void* stream);

/* Full GMRES (gmres.py:65-177) on A and the plan's M^{-1} (use_precond = 0: M = I).
 * side: 0 right, 1 left.  b, x: device vectors [N].  history (host, may be NULL)
 * receives max_iter+1 relative residual estimates. */
int helm_gmres(const helm_plan* plan, helm_workspace* ws, const void* b, void* x, double rtol,
               int32_t max_iter, int32_t side, int32_t use_precond, double* history,
               helm_gmres_report* report, void* stream);

/* nrhs independent GMRES solves sharing every operator application (each
 * right-hand side follows helm_gmres's statements).  b, x: device [nrhs][N]; nrhs <= the
 * workspace's max_batch; history (host, may be NULL): [nrhs][max_iter+1]; reports[nrhs]. */
int helm_gmres_multi(const helm_plan* plan, helm_workspace* ws, const void* b, void* x, int32_t nrhs,
                     double rtol, int32_t max_iter, int32_t side, int32_t use_precond, double* history,
                     helm_gmres_report* reports, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HELMB200_H */
