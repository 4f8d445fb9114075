// Shared declarations of the one-level Schwarz kernels (local.cu, local_fast.cu).
#pragma once
#include "ops.cuh"

namespace helm {

struct LocalArgs {
  int nu;
  int coarse_base;  // 1: `base` is a coarse vector c [B][m0][m0]; the base value of a node is (R0^T c)
  int m0;
  int off;          // grid offset of the prolongation (Geo::off)
  int p;
  int nbands;
  double k2;
  int weighted;
  int wbs;  // weights before solve
  const int* box_start;
  const int* box_len;
  const int* box_class;
  const int* class_len;
  const int* class_off_V;
  const int* class_off_lam;
  const int* node_first_box;
  const int* node_mult;
  const int* node_band;
};

// Base value of fine node (iy, ix): base[pidx] or, in coarse-base mode, the prolongation
// R0^T c at that node -- the same taps and summation order as prolong_kernel (stencil.cu),
// so z is never written to / read back from HBM (bb = this right-hand side's base).
__device__ __forceinline__ void prolong_taps_off(int u, int off, int& U0, int& cnt, double w[3]) {
  const int t = u - off;  // t = 2U + d
  if ((t & 1) == 0) {
    U0 = t / 2 - 1;
    w[0] = 0.125; w[1] = 0.75; w[2] = 0.125;
    cnt = 3;
  } else {
    U0 = (t - 1) >> 1;
    w[0] = 0.5; w[1] = 0.5; w[2] = 0.0;
    cnt = 2;
  }
}
template <typename S>
__device__ __forceinline__ S base_at(const S* __restrict__ bb, const LocalArgs& a, int iy, int ix) {
  if (!a.coarse_base) return bb[(size_t)iy * a.nu + ix];
  int Uy, ny, Ux, nx;
  double wy[3], wx[3];
  prolong_taps_off(iy, a.off, Uy, ny, wy);
  prolong_taps_off(ix, a.off, Ux, nx, wx);
  // all 9 taps unrolled with clamped indices and zero weights for the absent ones, so every
  // load is in flight at once; fma(0, v, r) == r keeps the sums of prolong_kernel bit for bit
  S v[3][3];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int U = min(max(Uy + p, 0), a.m0 - 1), V = min(max(Ux + q, 0), a.m0 - 1);
      v[p][q] = __ldg(bb + (size_t)U * a.m0 + V);
    }
  S acc = Sc<S>::zero();
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    const int U = Uy + p;
    const bool uin = p < ny && U >= 0 && U < a.m0;
    S row = Sc<S>::zero();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int V = Ux + q;
      row = fma_((q < nx && V >= 0 && V < a.m0) ? wx[q] : 0.0, v[p][q], row);
    }
    acc = fma_(uin ? wy[p] : 0.0, row, acc);
  }
  return acc;
}
// Coarse-base mode inside a box kernel: the box's window of c (WIN x WIN, zero outside
// [0, m0)) is copied to shared memory with cp.async at the start and prolongated from
// there in the epilogue (same taps and order as prolong_kernel).
constexpr int WIN = 23;  // >= max box side / 2 + 3 for boxes up to 40 nodes
template <typename S>
__device__ __forceinline__ void window_load(S* cw, const S* __restrict__ bb, const LocalArgs& a, int Uby, int Ubx,
                                            int nthreads) {
  for (int e = threadIdx.x; e < WIN * WIN; e += nthreads) {
    const int U = Uby + e / WIN, V = Ubx + e % WIN;
    const bool in = U >= 0 && U < a.m0 && V >= 0 && V < a.m0;
    const S* src = bb + (in ? (size_t)U * a.m0 + V : 0);
    if constexpr (Sc<S>::cplx) cp_async16(&cw[e], src, in);
    else cp_async8(&cw[e], src, in);
  }
  cp_commit();
}
__device__ __forceinline__ int window_base(int y0, int off) { return ((y0 - off) >> 1) - 1; }
template <typename S>
__device__ __forceinline__ S window_prolong(const S* cw, int off, int Uby, int Ubx, int iy, int ix) {
  const int ty = iy - off, tx = ix - off;
  const bool ey = (ty & 1) == 0, ex = (tx & 1) == 0;
  const int U0 = (ey ? ty / 2 - 1 : (ty - 1) >> 1) - Uby, V0 = (ex ? tx / 2 - 1 : (tx - 1) >> 1) - Ubx;
  const double wy[3] = {ey ? 0.125 : 0.5, ey ? 0.75 : 0.5, ey ? 0.125 : 0.0};
  const double wx[3] = {ex ? 0.125 : 0.5, ex ? 0.75 : 0.5, ex ? 0.125 : 0.0};
  S acc = Sc<S>::zero();
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    S row = Sc<S>::zero();
#pragma unroll
    for (int q = 0; q < 3; ++q) row = fma_(wx[q], cw[(U0 + p) * WIN + V0 + q], row);
    acc = fma_(wy[p], row, acc);
  }
  return acc;
}

__host__ __device__ __forceinline__ size_t base_stride(const LocalArgs& a) {
  return a.coarse_base ? (size_t)a.m0 * a.m0 : (size_t)a.nu * a.nu;
}

// Register-blocked FDM for boxes of at most 36 nodes per side (local_fast.cu).
// Returns false (nothing launched) when the plan's boxes are larger.
template <typename S>
bool launch_local_fast(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st, helm_workspace* ws);

// Folded boxes (both classes real and symmetric) on the FP64 tensor pipe (local_dmma.cu).
template <typename S>
void launch_local_dmma(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st);

// Boxes whose two classes are the Dirichlet middle pencil (exact DST-I eigenvectors) with
// L = 4Q - 1, Q in {5, 9}: fast sine transforms on the FP64 pipe (local_dst.cu).
template <typename S>
void launch_local_dst(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                      cudaStream_t st);

// MP-2 edge boxes (one middle axis, one Sommerfeld-end axis): sine transform + tridiagonal
// solves per sine mode (local_dst.cu).
template <typename S>
void launch_local_edge(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st);

}  // namespace helm
