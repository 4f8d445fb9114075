// K1 (5-point Helmholtz stencil); K2/K3 (R0, R0^T) live in transfer.cu.
//
// Reference semantics:
//   A   = T(x)W + W(x)T - k^2 W(x)W   (MP-2, discretization.py:181-184; T, W from :136-154)
//       = T(x)I + I(x)T - k^2 I       (MP-1, discretization.py:171-177)
//   R0  = P(x)P with P the (1,4,6,4,1)/8 stride-2 Bezier restriction, out-of-range
//         taps dropped (coarse.py:102-139); applied as cs.r0 @ r at coarse.py:174.
// All kernels are matrix-free: the coefficients are recomputed from (n, h, k).
#include "common.cuh"

namespace helm {

// --- K1: y = A x  or  y = x - A z ------------------------------------------
// One thread per unknown, x fastest so every warp reads 32 consecutive
// scalars (16-B double2 loads for complex128).  Neighbour re-reads hit L1/L2;
// the kernel streams x once and y once from HBM.
template <typename S, bool kDeflate>
__global__ void __launch_bounds__(256) stencil_kernel(const S* __restrict__ x, const S* __restrict__ z,
                                                      S* __restrict__ y, Geo g) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int nu = g.nu;
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iy = blockIdx.y * blockDim.y + threadIdx.y;
  const size_t N = (size_t)nu * nu;
  const size_t boff = (size_t)blockIdx.z * N;
  if (ix >= nu || iy >= nu) return;
  const S* in = (kDeflate ? z : x) + boff;
  const size_t p = (size_t)iy * nu + ix;
  S acc;
  if constexpr (!Sc<S>::cplx) {
    // MP-1: (4/h^2 - k^2) x_p - (1/h^2) sum of interior neighbours
    S nb = 0.0;
    if (iy > 0) nb += in[p - nu];
    if (iy < nu - 1) nb += in[p + nu];
    if (ix > 0) nb += in[p - 1];
    if (ix < nu - 1) nb += in[p + 1];
    acc = (4.0 * g.inv_h2 - g.k2) * in[p] - g.inv_h2 * nb;
  } else {
    // MP-2: ghost-point Sommerfeld rows scaled by W (edge 1/2, corner 1/4)
    const bool ey = (iy == 0) | (iy == nu - 1), ex = (ix == 0) | (ix == nu - 1);
    const double wy = ey ? 0.5 : 1.0, wx = ex ? 0.5 : 1.0;
    const double2 ty = ey ? g.tb : mk(2.0 * g.inv_h2, 0.0);
    const double2 tx = ex ? g.tb : mk(2.0 * g.inv_h2, 0.0);
    const double2 diag = mk(wx * ty.x + wy * tx.x - g.k2 * wy * wx, wx * ty.y + wy * tx.y);
    double2 ny = mk(0.0, 0.0), nx = mk(0.0, 0.0);
    if (iy > 0) ny = add(ny, in[p - nu]);
    if (iy < nu - 1) ny = add(ny, in[p + nu]);
    if (ix > 0) nx = add(nx, in[p - 1]);
    if (ix < nu - 1) nx = add(nx, in[p + 1]);
    acc = mul(diag, in[p]);
    acc = sub(acc, scale(ny, wx * g.inv_h2));
    acc = sub(acc, scale(nx, wy * g.inv_h2));
  }
  if constexpr (kDeflate) acc = sub(x[boff + p], acc);
  y[boff + p] = acc;
}

// ----------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------
template <typename S>
void launch_stencil(const Geo& g, const S* x, const S* z, S* y, int batch, cudaStream_t st) {
  dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.nu + 7) / 8, batch);
  if (z)
    launch_pdl(stencil_kernel<S, true>, grd, blk, 0, st, x, z, y, g);
  else
    launch_pdl(stencil_kernel<S, false>, grd, blk, 0, st, x, nullptr, y, g);
  HELM_LAUNCH_CHECK();
}

#define HELM_INST(S) template void launch_stencil<S>(const Geo&, const S*, const S*, S*, int, cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
