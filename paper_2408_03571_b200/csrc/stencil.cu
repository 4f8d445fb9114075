// K1 (5-point Helmholtz stencil), K2 (Bezier restriction R0) and K3 (prolongation R0^T).
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

// --- K2: c = R0 x -----------------------------------------------------------
// A CTA computes a TY x TX coarse tile.  The (2TY+3) x (2TX+3) fine window is
// staged in shared memory (zero outside the unknown set = dropped taps), then
// the separable 5-tap stencil runs as an x-pass and a y-pass in smem.
constexpr int RTX = 32, RTY = 16;
constexpr int RFW = 2 * RTX + 3, RFH = 2 * RTY + 3;  // fine window of a coarse tile
template <typename S>
__global__ void __launch_bounds__(256) restrict_kernel(const S* __restrict__ x, S* __restrict__ c, Geo g) {
  // 32 x 16 coarse outputs per CTA (32 x 8 threads, 2 rows each); the 67 x 35 fine
  // window is loaded with all of a thread's loads in flight at once (registers),
  // then the separable 5-tap x-pass and y-pass run from shared memory.
  // the window is stored as even and odd column planes, so the stride-2 taps of the
  // x-pass are consecutive (bank-conflict free) across the warp
  extern __shared__ __align__(16) unsigned char sraw[];
  constexpr int HW = (RFW + 1) / 2;
  S (*fev)[HW] = reinterpret_cast<S (*)[HW]>(sraw);
  S (*fod)[HW] = fev + RFH;
  S (*tmp)[RTX] = reinterpret_cast<S (*)[RTX]>(fod + RFH);
  const double w[5] = {0.125, 0.5, 0.75, 0.5, 0.125};
  const int nu = g.nu, m0 = g.m0;
  const int U0 = blockIdx.y * RTY, V0 = blockIdx.x * RTX;
  const int u0 = 2 * U0 + g.off - 2, v0 = 2 * V0 + g.off - 2;  // fine origin of the window
  const S* xb = x + (size_t)blockIdx.z * nu * nu;
  const int tx = threadIdx.x, ty = threadIdx.y;
  constexpr int NR = (RFH + 7) / 8, NC = (RFW + 31) / 32;
  S v[NR][NC];
#pragma unroll
  for (int i = 0; i < NR; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int r = ty + 8 * i, q = tx + 32 * j;
      const int u = u0 + r, vv = v0 + q;
      v[i][j] = (r < RFH && q < RFW && u >= 0 && u < nu && vv >= 0 && vv < nu) ? xb[(size_t)u * nu + vv]
                                                                                  : Sc<S>::zero();
    }
#pragma unroll
  for (int i = 0; i < NR; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int r = ty + 8 * i, q = tx + 32 * j;
      if (r < RFH && q < RFW) (q & 1 ? fod : fev)[r][q >> 1] = v[i][j];
    }
  __syncthreads();
  for (int r = ty; r < RFH; r += 8) {
    S a = Sc<S>::zero();
    a = fma_(w[0], fev[r][tx], a);
    a = fma_(w[1], fod[r][tx], a);
    a = fma_(w[2], fev[r][tx + 1], a);
    a = fma_(w[3], fod[r][tx + 1], a);
    a = fma_(w[4], fev[r][tx + 2], a);
    tmp[r][tx] = a;
  }
  __syncthreads();
  const int V = V0 + tx;
#pragma unroll
  for (int i = 0; i < RTY / 8; ++i) {
    const int r = ty + 8 * i, U = U0 + r;
    if (U < m0 && V < m0) {
      S a = Sc<S>::zero();
#pragma unroll
      for (int d = 0; d < 5; ++d) a = fma_(w[d], tmp[2 * r + d][tx], a);
      c[(size_t)blockIdx.z * m0 * m0 + (size_t)U * m0 + V] = a;
    }
  }
}

// --- K3: z = R0^T c (gather form, no atomics) ------------------------------
// Fine unknown u receives coarse U with |u - 2U - off| <= 2: weights (1,6,1)/8
// for even offsets, (4,4)/8 for odd ones, restricted to 0 <= U < m0.
__device__ __forceinline__ void prolong_taps(int u, const Geo& g, int& U0, int& cnt, double w[3]) {
  const int t = u - g.off;  // t = 2U + d
  if ((t & 1) == 0) {       // even: U = t/2-1, t/2, t/2+1 with d = 2, 0, -2
    U0 = t / 2 - 1;
    w[0] = 0.125; w[1] = 0.75; w[2] = 0.125;
    cnt = 3;
  } else {                  // odd: U = (t-1)/2, (t+1)/2 with d = 1, -1
    U0 = (t - 1) >> 1;
    w[0] = 0.5; w[1] = 0.5; w[2] = 0.0;
    cnt = 2;
  }
}

template <typename S>
__global__ void __launch_bounds__(256) prolong_kernel(const S* __restrict__ c, S* __restrict__ z, Geo g) {
  const int nu = g.nu, m0 = g.m0;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const int u = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= nu || v >= nu) return;
  const S* cb = c + (size_t)blockIdx.z * m0 * m0;
  int Uy, ny, Ux, nx;
  double wy[3], wx[3];
  prolong_taps(u, g, Uy, ny, wy);
  prolong_taps(v, g, Ux, nx, wx);
  S acc = Sc<S>::zero();
  for (int a = 0; a < ny; ++a) {
    const int U = Uy + a;
    if (U < 0 || U >= m0) continue;
    S row = Sc<S>::zero();
    for (int b = 0; b < nx; ++b) {
      const int V = Ux + b;
      if (V < 0 || V >= m0) continue;
      row = fma_(wx[b], cb[(size_t)U * m0 + V], row);
    }
    acc = fma_(wy[a], row, acc);
  }
  z[(size_t)blockIdx.z * nu * nu + (size_t)u * nu + v] = acc;
}

// ----------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------
template <typename S>
void launch_stencil(const Geo& g, const S* x, const S* z, S* y, int batch, cudaStream_t st) {
  dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.nu + 7) / 8, batch);
  if (z)
    stencil_kernel<S, true><<<grd, blk, 0, st>>>(x, z, y, g);
  else
    stencil_kernel<S, false><<<grd, blk, 0, st>>>(x, nullptr, y, g);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void launch_restrict(const Geo& g, const S* x, S* c, int batch, cudaStream_t st) {
  const size_t smem = (size_t)(2 * RFH * ((RFW + 1) / 2) + RFH * RTX) * sizeof(S);
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(restrict_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 blk(32, 8), grd((g.m0 + RTX - 1) / RTX, (g.m0 + RTY - 1) / RTY, batch);
  restrict_kernel<S><<<grd, blk, smem, st>>>(x, c, g);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void launch_prolong(const Geo& g, const S* c, S* z, int batch, cudaStream_t st) {
  dim3 blk(32, 8), grd((g.nu + 31) / 32, (g.nu + 7) / 8, batch);
  prolong_kernel<S><<<grd, blk, 0, st>>>(c, z, g);
  HELM_LAUNCH_CHECK();
}

// --- K3 + K1 fused for SHS2 (schwarz.py:86-88): z = R0^T c and d = x - A z ---
// A CTA owns a PW x PH fine tile.  The coarse window it needs is staged in shared
// memory, z is prolongated onto the tile plus a one-node halo in shared memory,
// and the 5-point stencil of the deflation runs from there: c is read once, x
// once, z and d written once -- no HBM round trip of z between two kernels.
constexpr int PW = 32, PH = 16;
constexpr int PCW = (PW + 2) / 2 + 3, PCH = (PH + 2) / 2 + 3;  // coarse window

__device__ __forceinline__ int floordiv2(int t) { return t >= 0 ? t / 2 : -((1 - t) / 2); }

template <typename S>
__device__ __forceinline__ S stencil_point(const Geo& g, int ix, int iy, S c, S up, S dn, S lf, S rt) {
  if constexpr (!Sc<S>::cplx) {
    return (4.0 * g.inv_h2 - g.k2) * c - g.inv_h2 * (up + dn + lf + rt);
  } else {
    const int nu = g.nu;
    const bool ey = (iy == 0) | (iy == nu - 1), ex = (ix == 0) | (ix == nu - 1);
    const double wy = ey ? 0.5 : 1.0, wx = ex ? 0.5 : 1.0;
    const double2 ty = ey ? g.tb : mk(2.0 * g.inv_h2, 0.0);
    const double2 tx = ex ? g.tb : mk(2.0 * g.inv_h2, 0.0);
    const double2 diag = mk(wx * ty.x + wy * tx.x - g.k2 * wy * wx, wx * ty.y + wy * tx.y);
    S acc = mul(diag, c);
    acc = sub(acc, scale(add(up, dn), wx * g.inv_h2));
    acc = sub(acc, scale(add(lf, rt), wy * g.inv_h2));
    return acc;
  }
}

template <typename S>
__global__ void __launch_bounds__(256) prolong_deflate_kernel(const S* __restrict__ c, const S* __restrict__ x,
                                                              S* __restrict__ z, S* __restrict__ d, Geo g) {
  __shared__ S cs[PCH][PCW];
  __shared__ S zs[PH + 2][PW + 2];
  const int nu = g.nu, m0 = g.m0;
  const int v0 = blockIdx.x * PW, u0 = blockIdx.y * PH;
  const size_t boff = (size_t)blockIdx.z * nu * nu;
  const S* cb = c + (size_t)blockIdx.z * m0 * m0;
  const int Ub = floordiv2(u0 - 1 - g.off) - 1, Vb = floordiv2(v0 - 1 - g.off) - 1;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  // this thread's x values are loaded first so their latency overlaps the z work
  constexpr int RPT = PH / 8;
  const int vx = v0 + threadIdx.x;
  S xv[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int u = u0 + threadIdx.y + 8 * i;
    xv[i] = (u < nu && vx < nu) ? x[boff + (size_t)u * nu + vx] : Sc<S>::zero();
  }
  for (int e = tid; e < PCH * PCW; e += 256) {
    const int rr = e / PCW, q = e % PCW;
    const int U = Ub + rr, V = Vb + q;
    cs[rr][q] = (U >= 0 && U < m0 && V >= 0 && V < m0) ? cb[(size_t)U * m0 + V] : Sc<S>::zero();
  }
  __syncthreads();
  for (int e = tid; e < (PH + 2) * (PW + 2); e += 256) {
    const int rr = e / (PW + 2), q = e % (PW + 2);
    const int u = u0 - 1 + rr, v = v0 - 1 + q;
    S acc = Sc<S>::zero();
    if (u >= 0 && u < nu && v >= 0 && v < nu) {
      int Uy, ny, Ux, nx;
      double wy[3], wx[3];
      prolong_taps(u, g, Uy, ny, wy);
      prolong_taps(v, g, Ux, nx, wx);
      for (int a = 0; a < ny; ++a) {  // cs has zeros outside [0, m0): the dropped taps
        S row = Sc<S>::zero();
        for (int b = 0; b < nx; ++b) row = fma_(wx[b], cs[Uy + a - Ub][Ux + b - Vb], row);
        acc = fma_(wy[a], row, acc);
      }
    }
    zs[rr][q] = acc;
  }
  __syncthreads();
  if (vx >= nu) return;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int rr = threadIdx.y + 8 * i, u = u0 + rr;
    if (u >= nu) break;
    const S zc = zs[rr + 1][threadIdx.x + 1];
    const S az = stencil_point<S>(g, vx, u, zc, zs[rr][threadIdx.x + 1], zs[rr + 2][threadIdx.x + 1],
                                  zs[rr + 1][threadIdx.x], zs[rr + 1][threadIdx.x + 2]);
    const size_t p = boff + (size_t)u * nu + vx;
    if (z) z[p] = zc;  // z may be left implicit (coarse-base local sum)
    d[p] = sub(xv[i], az);
  }
}

template <typename S>
void launch_prolong_deflate(const Geo& g, const S* c, const S* x, S* z, S* d, int batch, cudaStream_t st) {
  dim3 blk(32, 8), grd((g.nu + PW - 1) / PW, (g.nu + PH - 1) / PH, batch);
  prolong_deflate_kernel<S><<<grd, blk, 0, st>>>(c, x, z, d, g);
  HELM_LAUNCH_CHECK();
}

#define HELM_INST(S)                                                                           \
  template void launch_stencil<S>(const Geo&, const S*, const S*, S*, int, cudaStream_t);      \
  template void launch_restrict<S>(const Geo&, const S*, S*, int, cudaStream_t);               \
  template void launch_prolong<S>(const Geo&, const S*, S*, int, cudaStream_t);                \
  template void launch_prolong_deflate<S>(const Geo&, const S*, const S*, S*, S*, int, cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
