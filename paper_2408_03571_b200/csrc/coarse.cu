// K5: the coarse solve  y = A0^{-1} c  (reference: linalg.solve(cs.a0_factorization, .)
// at coarse.py:174, SuperLU factor of the symmetrised Galerkin matrix, coarse.py:154-167).
//
// A0 = R0 A R0^T is the Kronecker sum T0(x)M0 + M0(x)T0 - k^2 M0(x)M0 of two
// pentadiagonal m0 x m0 pencils (T0 = P T P^T, M0 = P W P^T).  Partial fast
// diagonalisation along x (the fast index):
//   1. G = C V                (GEMM, V^T M0 V = I, T0 V = M0 V diag(lambda))
//   2. (T0 + (lambda_a - k^2) M0) H[:,a] = G[:,a]   (m0 pivoted pentadiagonal solves)
//   3. Y = H V^T              (GEMM)
// followed by iterative refinement  r = c - A0 Y,  Y += solve(r)  (25-point
// residual kernel), which pulls the FDM rounding (~1e-12 near coarse
// resonances) down to SuperLU's own level.
#include "common.cuh"

namespace helm {

// --- pivoted pentadiagonal solves, one thread per (batch, column a) ---------
// Factor layout [row][a]: piv (0..2), l[2], u[5] = {1/U_jj, U_j,j+1 .. U_j,j+4}.
template <typename S>
__global__ void __launch_bounds__(128) band_solve_kernel(S* __restrict__ G, const uint8_t* __restrict__ piv,
                                                         const S* __restrict__ L, const S* __restrict__ U,
                                                         int m0) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m0) return;
  S* col = G + (size_t)blockIdx.y * m0 * m0 + a;
  const size_t ld = m0;
  // forward: apply the row interchanges and eliminations to the right-hand side
  S r0 = col[0];
  S r1 = m0 > 1 ? col[ld] : Sc<S>::zero();
  S r2 = m0 > 2 ? col[2 * ld] : Sc<S>::zero();
  for (int j = 0; j < m0; ++j) {
    const size_t f = (size_t)j * m0 + a;
    const int pv = piv[f];
    if (pv == 1) { S t = r0; r0 = r1; r1 = t; }
    else if (pv == 2) { S t = r0; r0 = r2; r2 = t; }
    r1 = fms_(L[2 * f], r0, r1);
    r2 = fms_(L[2 * f + 1], r0, r2);
    col[(size_t)j * ld] = r0;
    r0 = r1;
    r1 = r2;
    r2 = (j + 3 < m0) ? col[(size_t)(j + 3) * ld] : Sc<S>::zero();
  }
  // backward substitution with the 4 super-diagonals of U
  S x1 = Sc<S>::zero(), x2 = x1, x3 = x1, x4 = x1;
  for (int j = m0 - 1; j >= 0; --j) {
    const size_t f = (size_t)j * m0 + a;
    const S* u = U + 5 * f;
    S v = col[(size_t)j * ld];
    v = fms_(u[1], x1, v);
    v = fms_(u[2], x2, v);
    v = fms_(u[3], x3, v);
    v = fms_(u[4], x4, v);
    v = mul(v, u[0]);
    col[(size_t)j * ld] = v;
    x4 = x3; x3 = x2; x2 = x1; x1 = v;
  }
}

// --- r = c - A0 y  (25-point Kronecker-sum stencil from the 1-D bands) ------
template <typename S>
__global__ void __launch_bounds__(256) a0_residual_kernel(const S* __restrict__ c, const S* __restrict__ y,
                                                          S* __restrict__ r, const S* __restrict__ t0b,
                                                          const S* __restrict__ m0b, double k2, int m0) {
  const int V = blockIdx.x * blockDim.x + threadIdx.x;
  const int Uc = blockIdx.y * blockDim.y + threadIdx.y;
  if (V >= m0 || Uc >= m0) return;
  const size_t off = (size_t)blockIdx.z * m0 * m0;
  S acc = Sc<S>::zero();
  for (int dy = -2; dy <= 2; ++dy) {
    const int U = Uc + dy;
    if (U < 0 || U >= m0) continue;
    const S ty = t0b[Uc * 5 + dy + 2], my = m0b[Uc * 5 + dy + 2];
    S rowT = Sc<S>::zero(), rowM = Sc<S>::zero();  // sum_dx M0 y, sum_dx T0 y along x
    for (int dx = -2; dx <= 2; ++dx) {
      const int W = V + dx;
      if (W < 0 || W >= m0) continue;
      const S yv = y[off + (size_t)U * m0 + W];
      rowM = fma_(m0b[V * 5 + dx + 2], yv, rowM);
      rowT = fma_(t0b[V * 5 + dx + 2], yv, rowT);
    }
    // T0(y) M0(x) + M0(y) T0(x) - k^2 M0(y) M0(x)
    acc = fma_(ty, rowM, acc);
    acc = fma_(my, sub(rowT, scale(rowM, k2)), acc);
  }
  const size_t p = off + (size_t)Uc * m0 + V;
  r[p] = sub(c[p], acc);
}

template <typename S>
__global__ void axpy_kernel(S* __restrict__ y, const S* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = add(y[i], d[i]);
}

// Row-major G[(b,Iy)][a] = sum_Ix C[(b,Iy)][Ix] V[Ix][a]  (column-major: G^T = V^T C^T)
// Row-major Y[(b,Iy)][Ix] = sum_a H[(b,Iy)][a] V[Ix][a]   (column-major: Y^T = V H^T)
template <typename S>
void coarse_gemm(cublasHandle_t h, const S* Vm, const S* in, S* out, int m0, int rows, bool transposeV) {
  cublasOperation_t op = transposeV ? CUBLAS_OP_T : CUBLAS_OP_N;
  if constexpr (Sc<S>::cplx) {
    const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
    HELM_CUBLAS(cublasZgemm(h, op, CUBLAS_OP_N, m0, rows, m0, &one, (const cuDoubleComplex*)Vm, m0,
                            (const cuDoubleComplex*)in, m0, &zero, (cuDoubleComplex*)out, m0));
  } else {
    const double one = 1.0, zero = 0.0;
    HELM_CUBLAS(cublasDgemm(h, op, CUBLAS_OP_N, m0, rows, m0, &one, Vm, m0, in, m0, &zero, out, m0));
  }
}

// One partial-FDM solve: out = A0~^{-1} in  (in and out distinct; tmp scratch [B][N0])
template <typename S>
static void fdm_solve(const helm_plan* P, helm_workspace* ws, const S* in, S* out, S* tmp, int batch,
                      cudaStream_t st) {
  const PlanDev& d = P->dev;
  const int m0 = P->geo.m0;
  HELM_CUBLAS(cublasSetStream(ws->cublas, st));
  coarse_gemm<S>(ws->cublas, (const S*)d.coarse_V, in, tmp, m0, m0 * batch, false);
  dim3 grd((m0 + 127) / 128, batch);
  band_solve_kernel<S><<<grd, 128, 0, st>>>(tmp, d.band_piv, (const S*)d.band_l, (const S*)d.band_u, m0);
  HELM_LAUNCH_CHECK();
  coarse_gemm<S>(ws->cublas, (const S*)d.coarse_V, tmp, out, m0, m0 * batch, true);
}

template <typename S>
void launch_coarse_solve(const helm_plan* P, helm_workspace* ws, const S* c, S* y, int batch, cudaStream_t st) {
  HELM_CHECK(P->dev.coarse_V != nullptr, "plan was created without a coarse solver");
  const int m0 = P->geo.m0;
  const size_t n0 = (size_t)batch * m0 * m0;
  S* tmp = (S*)ws->g;
  S* r = (S*)ws->r0;
  S* corr = (S*)ws->e0;
  // c is only read; y is written last when it aliases c
  S* yy = ((const void*)c == (const void*)y) ? (S*)ws->y0 : y;
  fdm_solve<S>(P, ws, c, yy, tmp, batch, st);
  for (int it = 0; it < P->desc.refine_steps; ++it) {
    dim3 blk(32, 8), grd((m0 + 31) / 32, (m0 + 7) / 8, batch);
    a0_residual_kernel<S><<<grd, blk, 0, st>>>(c, yy, r, (const S*)P->dev.t0_band, (const S*)P->dev.m0_band,
                                               P->geo.k2, m0);
    HELM_LAUNCH_CHECK();
    fdm_solve<S>(P, ws, r, corr, tmp, batch, st);
    axpy_kernel<S><<<1184, 256, 0, st>>>(yy, corr, n0);
    HELM_LAUNCH_CHECK();
  }
  if (yy != y) HELM_CUDA(cudaMemcpyAsync(y, yy, n0 * sizeof(S), cudaMemcpyDeviceToDevice, st));
}

template void launch_coarse_solve<double>(const helm_plan*, helm_workspace*, const double*, double*, int,
                                          cudaStream_t);
template void launch_coarse_solve<double2>(const helm_plan*, helm_workspace*, const double2*, double2*, int,
                                           cudaStream_t);

}  // namespace helm
