// General coarse spaces: FOCS at any ratio and HOCS at ratios 4, 8, 16 (coarse.py:84-151).
//
//   R0 = P (x) P with a banded 1-D restriction P (m0 x nu): the Bezier stencil composed
//   through the intermediate grids (coarse.py:102-133) or the hat functions (coarse.py:84-99),
//   out-of-range taps dropped.  A0 = R0 A R0^T = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0 with the
//   banded T0 = P T P^T, M0 = P W P^T (half-bandwidth b <= 3), so
//
//     A0^{-1} c = (V (x) V) diag(1 / (lam_y + lam_x - k^2)) (V (x) V)^T c,
//     T0 V = M0 V diag(lam),  V^T M0 V = I           (host setup, fdm_setup.coarse_dense)
//
//   i.e. Y = V ((V^T C V) .* invden) V^T on the m0 x m0 coarse array C: four dense GEMMs,
//   followed by refine_steps iterative-refinement steps r = C - A0 Y with the reference's own
//   Galerkin matrix (a 2-D stencil, a0_stencil_residual_kernel) that take the solve to the rounding
//   level of the reference's SuperLU solve (linalg.py:90-95).  The sizes where these spaces are used (the
//   paper's tables, n <= 801, m0 <= 201) make this a latency-bound path, not a roofline one.
#include "ops.cuh"

namespace helm {

// ---------------------------------------------------------------------------------------
// R0 = P (x) P and R0^T applied separably in one pass (no intermediate array):
//   out[b][J][I] = sum_ty w[J][ty] sum_tx w[I][tx] in[b][s_J + ty][s_I + tx]
// w: [nout][width] taps starting at in-index start[j] (zero-padded; out-of-range skipped).
// Restriction uses P's rows, prolongation the rows of P^T.
// ---------------------------------------------------------------------------------------
template <typename S>
__global__ void __launch_bounds__(256) tensor_band_kernel(const S* __restrict__ in, S* __restrict__ out,
                                                          const double* __restrict__ w,
                                                          const int* __restrict__ start, int width, int nin,
                                                          int nout) {
  pdl_wait();
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  const int J = blockIdx.y * blockDim.y + threadIdx.y;
  if (I >= nout || J >= nout) return;
  const size_t b = blockIdx.z;
  const S* src = in + b * (size_t)nin * nin;
  const int sI = start[I], sJ = start[J];
  const double* wI = w + (size_t)I * width;
  const double* wJ = w + (size_t)J * width;
  S acc = Sc<S>::zero();
  for (int ty = 0; ty < width; ++ty) {
    const int iy = sJ + ty;
    if (iy < 0 || iy >= nin || wJ[ty] == 0.0) continue;
    const S* row = src + (size_t)iy * nin;
    S r = Sc<S>::zero();
    for (int tx = 0; tx < width; ++tx) {
      const int ix = sI + tx;
      if (ix >= 0 && ix < nin) r = fma_(wI[tx], row[ix], r);
    }
    acc = fma_(wJ[ty], r, acc);
  }
  out[(b * nout + J) * (size_t)nout + I] = acc;
}

template <typename S>
static void tensor_band(const S* in, S* out, const double* w, const int* start, int width, int nin, int nout,
                        int batch, cudaStream_t st) {
  dim3 blk(32, 8), grd((nout + 31) / 32, (nout + 7) / 8, batch);
  launch_pdl(tensor_band_kernel<S>, grd, blk, 0, st, in, out, w, start, width, nin, nout);
  HELM_LAUNCH_CHECK();
}

template <typename S> void launch_restrict_general(const helm_plan* P, const S* x, S* c, int batch, cudaStream_t st) {
  const PlanDev& d = P->dev;
  tensor_band<S>(x, c, d.p_taps, d.p_start, d.p_width, P->geo.nu, P->geo.m0, batch, st);
}

template <typename S> void launch_prolong_general(const helm_plan* P, const S* c, S* z, int batch, cudaStream_t st) {
  const PlanDev& d = P->dev;
  tensor_band<S>(c, z, d.pt_taps, d.pt_start, d.pt_width, P->geo.m0, P->geo.nu, batch, st);
}

// ---------------------------------------------------------------------------------------
// batched dense products C[b] = A[b] B[b] of m0 x m0 matrices with arbitrary element strides
// (a shared operand has batch stride 0; a transposed one swaps its strides).  64 x 64 tiles,
// 16-deep K slabs in shared memory, 4 x 4 outputs per thread, FMA in fixed k order.
// Epilogue: optional elementwise scale (invden) and accumulation into C.
// ---------------------------------------------------------------------------------------
struct GemmOp {
  const void* p;
  size_t sb;   // batch stride (elements)
  int sr, sc;  // row / column strides (elements)
};

constexpr int GT = 64, GK = 16, GTH = 256;

template <typename S>
__global__ void __launch_bounds__(GTH) dense_gemm_kernel(GemmOp A, GemmOp B, S* __restrict__ C,
                                                         const S* __restrict__ scale_by, int accumulate, int m) {
  pdl_wait();
  __shared__ S As[GK][GT + 1];
  __shared__ S Bs[GK][GT + 1];
  const int b = blockIdx.z;
  const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const S* a = static_cast<const S*>(A.p) + (size_t)b * A.sb;
  const S* bb = static_cast<const S*>(B.p) + (size_t)b * B.sb;
  S acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = Sc<S>::zero();
  for (int k0 = 0; k0 < m; k0 += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += GTH) {
      const int kk = e / GT, ii = e % GT;
      const int gi = i0 + ii, gk = k0 + kk;
      As[kk][ii] = (gi < m && gk < m) ? a[(size_t)gi * A.sr + (size_t)gk * A.sc] : Sc<S>::zero();
      const int gj = j0 + ii;
      Bs[kk][ii] = (gj < m && gk < m) ? bb[(size_t)gk * B.sr + (size_t)gj * B.sc] : Sc<S>::zero();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GK; ++kk) {
      S av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = As[kk][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = Bs[kk][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma_(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
  S* cb = C + (size_t)b * m * m;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int gi = i0 + ty + 16 * u, gj = j0 + tx + 16 * v;
      if (gi >= m || gj >= m) continue;
      const size_t o = (size_t)gi * m + gj;
      S r = acc[u][v];
      if (scale_by) r = mul(r, scale_by[o]);
      cb[o] = accumulate ? add(cb[o], r) : r;
    }
}

template <typename S>
static void dense_gemm(GemmOp A, GemmOp B, S* C, const S* scale_by, bool accumulate, int m, int batch,
                       cudaStream_t st) {
  dim3 grd((m + GT - 1) / GT, (m + GT - 1) / GT, batch);
  launch_pdl(dense_gemm_kernel<S>, grd, GTH, 0, st, A, B, C, scale_by, accumulate ? 1 : 0, m);
  HELM_LAUNCH_CHECK();
}

// A0 residual r = c - A0 y with the reference's own Galerkin matrix as a 2-D stencil
// ((2b+1)^2 coefficients per coarse unknown, coarse.py:161-165): the refinement then converges
// to the solution of exactly the matrix SuperLU factorises (linalg.py:64-95), not of its
// Kronecker form T0(x)M0 + M0(x)T0 - k^2 M0(x)M0, which differs from it at the rounding level
// (amplified by cond(A0) near a coarse resonance).
template <typename S>
__global__ void __launch_bounds__(256) a0_stencil_residual_kernel(const S* __restrict__ c, const S* __restrict__ y,
                                                          S* __restrict__ res, const S* __restrict__ st, int bw,
                                                          int m) {
  pdl_wait();
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y * blockDim.y + threadIdx.y;
  if (ix >= m || iy >= m) return;
  const size_t bo = (size_t)blockIdx.z * m * m;
  const int wd = 2 * bw + 1;
  const S* a = st + ((size_t)iy * m + ix) * wd * wd;
  S acc = Sc<S>::zero();
  for (int dy = -bw; dy <= bw; ++dy) {
    const int jy = iy + dy;
    if (jy < 0 || jy >= m) continue;
    for (int dx = -bw; dx <= bw; ++dx) {
      const int jx = ix + dx;
      if (jx < 0 || jx >= m) continue;
      acc = fma_(a[(dy + bw) * wd + dx + bw], y[bo + (size_t)jy * m + jx], acc);
    }
  }
  const size_t o = bo + (size_t)iy * m + ix;
  res[o] = sub(c[o], acc);
}

// y = V ((V^T c V) .* invden) V^T, accumulated into y when `accumulate`
template <typename S>
static void fdm_solve(const helm_plan* P, const S* c, S* y, S* t1, S* t2, bool accumulate, int batch,
                      cudaStream_t st) {
  const PlanDev& d = P->dev;
  const int m = P->geo.m0;
  const size_t mm = (size_t)m * m;
  const S* V = static_cast<const S*>(d.coarse_V);
  const GemmOp Vn{V, 0, m, 1}, Vt{V, 0, 1, m};
  dense_gemm<S>(GemmOp{c, mm, m, 1}, Vn, t1, nullptr, false, m, batch, st);                          // C V
  dense_gemm<S>(Vt, GemmOp{t1, mm, m, 1}, t2, static_cast<const S*>(d.coarse_invden), false, m, batch, st);  // V^T . ./D
  dense_gemm<S>(GemmOp{t2, mm, m, 1}, Vt, t1, nullptr, false, m, batch, st);                         // . V^T
  dense_gemm<S>(Vn, GemmOp{t1, mm, m, 1}, y, nullptr, accumulate, m, batch, st);                     // V .
}

template <typename S>
void launch_coarse_solve_dense(const helm_plan* P, helm_workspace* ws, const S* c, S* y, int batch,
                               cudaStream_t st) {
  const PlanDev& d = P->dev;
  const int m = P->geo.m0;
  S* t1 = (S*)ws->g;
  S* t2 = (S*)ws->r0;
  S* rr = (S*)ws->e0;
  S* cc = (S*)ws->f0;
  const S* src = c;
  if (c == y) {  // aliasing allowed by the ABI: keep the right-hand side
    HELM_CUDA(cudaMemcpyAsync(cc, c, (size_t)batch * m * m * sizeof(S), cudaMemcpyDeviceToDevice, st));
    src = cc;
  }
  fdm_solve<S>(P, src, y, t1, t2, false, batch, st);
  const S* a0 = static_cast<const S*>(d.a0_stencil);
  for (int it = 0; it < P->desc.refine_steps; ++it) {
    dim3 blk(32, 8), grd((m + 31) / 32, (m + 7) / 8, batch);
    launch_pdl(a0_stencil_residual_kernel<S>, grd, blk, 0, st, src, (const S*)y, rr, a0, d.a0_bw, m);
    HELM_LAUNCH_CHECK();
    fdm_solve<S>(P, rr, y, t1, t2, true, batch, st);
  }
}

#define HELM_INST(S)                                                                                      \
  template void launch_restrict_general<S>(const helm_plan*, const S*, S*, int, cudaStream_t);          \
  template void launch_prolong_general<S>(const helm_plan*, const S*, S*, int, cudaStream_t);           \
  template void launch_coarse_solve_dense<S>(const helm_plan*, helm_workspace*, const S*, S*, int,      \
                                             cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
