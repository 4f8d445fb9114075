// K4: the one-level Schwarz term  y = base + sum_i R_i^T [D_i] A_i^{-1} [D_i] R_i x
// (reference: SchwarzPreconditioner._local_sum, schwarz.py:64-74; index sets and
// weights decomposition.py:111-134; local matrices decomposition.py:157-160).
//
// The reference factorises every R_i A R_i^T with SuperLU and solves p^2 times
// in a Python loop.  Each local matrix is a Kronecker sum of 1-D pencils
// (A_i = T_y(x)W_x + W_y(x)T_x - k^2 W_y(x)W_x), so here it is inverted by fast
// diagonalisation:  A_i^{-1} = (V_y(x)V_x) D^{-1} (V_y(x)V_x)^T with
// T V = W V diag(lambda), V^T W V = I  =>  Y = V_y [(V_y^T X V_x) ./ D] V_x^T.
// One CTA owns one subdomain: gather the box into shared memory, four small
// GEMMs in shared memory, weight, then write.  Nodes covered by one subdomain
// are written directly (base + contribution); nodes in an overlap band write
// their contribution into a per-slot scratch that a deterministic combine pass
// sums (no atomics, so the result is bitwise reproducible).
#include "local.cuh"

namespace helm {


// C[M][N] (row-major, ldc) = sum_k A(m,k) * B(k,n), operands in shared memory.
// transA: A(m,k) = Asm[k][m]; transB: B(k,n) = Bsm[n][k].
template <typename S, bool TA, bool TB>
__device__ __forceinline__ void smem_gemm(int M, int N, int K, const S* A, int lda, const S* B, int ldb,
                                          S* C, int ldc) {
  for (int e = threadIdx.x; e < M * N; e += blockDim.x) {
    const int m = e / N, n = e % N;
    S acc = Sc<S>::zero();
    for (int k = 0; k < K; ++k) {
      const S a = TA ? A[k * lda + m] : A[m * lda + k];
      const S b = TB ? B[n * ldb + k] : B[k * ldb + n];
      acc = fma_(a, b, acc);
    }
    C[m * ldc + n] = acc;
  }
}

template <typename S>
__global__ void __launch_bounds__(256) local_fdm_kernel(const S* __restrict__ x, const S* __restrict__ base,
                                                        S* __restrict__ y, S* __restrict__ ovl,
                                                        const S* __restrict__ classV,
                                                        const S* __restrict__ classLam, LocalArgs a,
                                                        int ld) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S* sm = reinterpret_cast<S*>(smem_raw);
  S* Vy = sm;                 // [ld][ld]
  S* Vx = Vy + ld * ld;       // [ld][ld]
  S* X = Vx + ld * ld;        // [ld][ld]
  S* T = X + ld * ld;         // [ld][ld]
  S* ly = T + ld * ld;        // [ld]
  S* lx = ly + ld;            // [ld]

  const int sid = blockIdx.x;
  const int ay = sid / a.p, ax = sid % a.p;
  const int nu = a.nu;
  const size_t N = (size_t)nu * nu;
  const int b = blockIdx.y;
  const int y0 = a.box_start[ay], Ly = a.box_len[ay], cy = a.box_class[ay];
  const int x0 = a.box_start[ax], Lx = a.box_len[ax], cx = a.box_class[ax];
  const S* Vyg = classV + a.class_off_V[cy];
  const S* Vxg = classV + a.class_off_V[cx];
  for (int e = threadIdx.x; e < Ly * Ly; e += blockDim.x) Vy[(e / Ly) * ld + e % Ly] = Vyg[e];
  for (int e = threadIdx.x; e < Lx * Lx; e += blockDim.x) Vx[(e / Lx) * ld + e % Lx] = Vxg[e];
  for (int e = threadIdx.x; e < Ly; e += blockDim.x) ly[e] = classLam[a.class_off_lam[cy] + e];
  for (int e = threadIdx.x; e < Lx; e += blockDim.x) lx[e] = classLam[a.class_off_lam[cx] + e];
  const S* xb = x + (size_t)b * N;
  for (int e = threadIdx.x; e < Ly * Lx; e += blockDim.x) {
    const int r = e / Lx, q = e % Lx;
    const int iy = y0 + r, ix = x0 + q;
    S v = xb[(size_t)iy * nu + ix];
    if (a.weighted && a.wbs) v = scale(v, 1.0 / (a.node_mult[iy] * a.node_mult[ix]));
    X[r * ld + q] = v;
  }
  __syncthreads();
  // T = Vy^T X
  smem_gemm<S, true, false>(Ly, Lx, Ly, Vy, ld, X, ld, T, ld);
  __syncthreads();
  // X = (T Vx) ./ (ly (+) lx - k^2)
  for (int e = threadIdx.x; e < Ly * Lx; e += blockDim.x) {
    const int m = e / Lx, n = e % Lx;
    S acc = Sc<S>::zero();
    for (int k = 0; k < Lx; ++k) acc = fma_(T[m * ld + k], Vx[k * ld + n], acc);
    S den = add(ly[m], lx[n]);
    den = sub(den, Sc<S>::from_real(a.k2));
    X[m * ld + n] = div_(acc, den);
  }
  __syncthreads();
  // T = Vy X
  smem_gemm<S, false, false>(Ly, Lx, Ly, Vy, ld, X, ld, T, ld);
  __syncthreads();
  // Y = T Vx^T, weighted, written out
  const S* bb = base ? base + (size_t)b * base_stride(a) : nullptr;
  S* yb = y + (size_t)b * N;
  S* ob = ovl + (size_t)b * 6 * a.nbands * nu;
  for (int e = threadIdx.x; e < Ly * Lx; e += blockDim.x) {
    const int r = e / Lx, q = e % Lx;
    S acc = Sc<S>::zero();
    for (int k = 0; k < Lx; ++k) acc = fma_(T[r * ld + k], Vx[q * ld + k], acc);
    const int iy = y0 + r, ix = x0 + q;
    const int my = a.node_mult[iy], mx = a.node_mult[ix];
    if (a.weighted && !a.wbs) acc = scale(acc, 1.0 / (my * mx));
    const size_t pidx = (size_t)iy * nu + ix;
    if (my == 1 && mx == 1) {
      yb[pidx] = bb ? add(base_at(bb, a, iy, ix), acc) : acc;
    } else if (my == 2) {
      const int ry = ay - a.node_first_box[iy], rx = ax - a.node_first_box[ix];
      ob[((size_t)(ry * 2 + rx) * a.nbands + a.node_band[iy]) * nu + ix] = acc;
    } else {
      const int rx = ax - a.node_first_box[ix];
      ob[(size_t)4 * a.nbands * nu + ((size_t)rx * nu + iy) * a.nbands + a.node_band[ix]] = acc;
    }
  }
}

// Combine the overlap-band contributions: rows with y-multiplicity 2 (all x),
// then columns with x-multiplicity 2 in rows of y-multiplicity 1.
template <typename S>
__device__ __forceinline__ void combine_row(const S* __restrict__ base, S* __restrict__ y, const S* __restrict__ ovl,
                                            const int* __restrict__ band_node, const int* __restrict__ node_mult,
                                            int nu, int nbands, const LocalArgs& a, int bx, int bi, int b) {
  const int ix = bx * blockDim.x + threadIdx.x;
  if (ix >= nu) return;
  const size_t N = (size_t)nu * nu;
  const S* ob = ovl + (size_t)b * 6 * nbands * nu;
  const int iy = band_node[bi];
  const int mx = node_mult[ix];
  S acc = ob[((size_t)0 * nbands + bi) * nu + ix];
  acc = add(acc, ob[((size_t)2 * nbands + bi) * nu + ix]);
  if (mx == 2) {
    acc = add(acc, ob[((size_t)1 * nbands + bi) * nu + ix]);
    acc = add(acc, ob[((size_t)3 * nbands + bi) * nu + ix]);
  }
  const size_t pidx = (size_t)iy * nu + ix;
  y[b * N + pidx] = base ? add(base_at(base + b * base_stride(a), a, iy, ix), acc) : acc;
}

template <typename S>
__device__ __forceinline__ void combine_col(const S* __restrict__ base, S* __restrict__ y, const S* __restrict__ ovl,
                                            const int* __restrict__ band_node, const int* __restrict__ node_mult,
                                            int nu, int nbands, const LocalArgs& a, int bx, int iy, int b) {
  const int bi = bx * blockDim.x + threadIdx.x;
  if (bi >= nbands || node_mult[iy] != 1) return;
  const size_t N = (size_t)nu * nu;
  const S* ob = ovl + (size_t)b * 6 * nbands * nu + (size_t)4 * nbands * nu;
  S acc = add(ob[((size_t)0 * nu + iy) * nbands + bi], ob[((size_t)1 * nu + iy) * nbands + bi]);
  const int ix = band_node[bi];
  const size_t pidx = (size_t)iy * nu + ix;
  y[b * N + pidx] = base ? add(base_at(base + b * base_stride(a), a, iy, ix), acc) : acc;
}


// Both combines in one launch: the row-band and column-band node sets are disjoint (column
// bands only in rows of y-multiplicity 1), so the first nrb blocks do rows, the rest columns.
template <typename S>
__global__ void __launch_bounds__(128) combine_kernel(const S* __restrict__ base, S* __restrict__ y,
                                                     const S* __restrict__ ovl, const int* __restrict__ band_node,
                                                     const int* __restrict__ node_mult, int nu, int nbands,
                                                     LocalArgs a, int rbx, int cbx) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int b = blockIdx.y;
  const int nrb = rbx * nbands;
  const int e = blockIdx.x;
  if (e < nrb) combine_row(base, y, ovl, band_node, node_mult, nu, nbands, a, e % rbx, e / rbx, b);
  else combine_col(base, y, ovl, band_node, node_mult, nu, nbands, a, (e - nrb) % cbx, (e - nrb) / cbx, b);
}

size_t local_smem_bytes(int ld, size_t elem) { return (size_t)(4 * ld * ld + 2 * ld) * elem; }

template <typename S>
void launch_local_sum(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, int weighted, int batch,
                      const int* band_node, cudaStream_t st, bool coarse_base, helm_workspace* ws) {
  const PlanDev& d = P->dev;
  HELM_CHECK(d.p > 0, "plan was created without subdomains");
  LocalArgs a;
  a.nu = P->geo.nu;
  a.coarse_base = coarse_base ? 1 : 0;
  a.m0 = P->geo.m0;
  a.off = P->geo.off;
  a.p = d.p;
  a.nbands = d.nbands;
  a.k2 = P->geo.k2;
  a.weighted = weighted;
  a.wbs = P->desc.weights_before_solve;
  a.box_start = d.box_start;
  a.box_len = d.box_len;
  a.box_class = d.box_class;
  a.class_len = d.class_len;
  a.class_off_V = d.class_off_V;
  a.class_off_lam = d.class_off_lam;
  a.node_first_box = d.node_first_box;
  a.node_mult = d.node_mult;
  a.node_band = d.node_band;
  const int ld = d.max_len;
  dim3 grd(d.p * d.p, batch);
  if (!launch_local_fast<S>(P, x, base, y, ovl, a, batch, st, ws)) {
    const size_t smem = local_smem_bytes(ld, sizeof(S));
    static bool attr_set[2] = {false, false};
    if (!attr_set[Sc<S>::cplx]) {
      HELM_CUDA(cudaFuncSetAttribute(local_fdm_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr_set[Sc<S>::cplx] = true;
    }
    launch_pdl(local_fdm_kernel<S>, grd, 256, smem, st, x, base, y, ovl, (const S*)d.class_V, (const S*)d.class_lambda, a,
                                                ld);
    HELM_LAUNCH_CHECK();
  }
  if (d.nbands > 0) {
    const int rbx = (a.nu + 127) / 128, cbx = (d.nbands + 127) / 128;
    dim3 g((unsigned)(rbx * d.nbands + cbx * a.nu), batch);
    launch_pdl(combine_kernel<S>, g, 128, 0, st, base, y, ovl, band_node, d.node_mult, a.nu, d.nbands, a, rbx, cbx);
    HELM_LAUNCH_CHECK();
  }
}

template void launch_local_sum<double>(const helm_plan*, const double*, const double*, double*, double*, int, int,
                                       const int*, cudaStream_t, bool, helm_workspace*);
template void launch_local_sum<double2>(const helm_plan*, const double2*, const double2*, double2*, double2*, int,
                                        int, const int*, cudaStream_t, bool, helm_workspace*);

}  // namespace helm
