// K4 fast path: register-blocked fast diagonalisation of the subdomain solves
// (reference: the p^2 SuperLU solves of SchwarzPreconditioner._local_sum,
// schwarz.py:64-74, on R_i A R_i^T, decomposition.py:157-160).
//
//   Y_i = V_y [ (V_y^T X_i V_x) ./ (lam_y (+) lam_x - k^2) ] V_x^T
//
// One CTA (96 threads) owns one (box, right-hand side).  The box (<= 36 x 36,
// zero-padded) lives in ONE shared-memory tile; each of the four products is
// computed into registers -- 81 threads x a 4 x 4 block, rows tm + 9i and
// columns tn + 9j so that a warp's shared-memory accesses are consecutive
// (bank-conflict free) -- then written back in place after a barrier.
// Boxes whose two 1-D classes are both real (the interior middle class: pencil
// tridiag(-1,2,-1)/h^2 with W = I, DST-like eigenvectors; every MP-1 box) run a
// separate launch with real V (half the FP64 work of complex V, half the
// shared memory, so more CTAs per SM); the boundary boxes (complex Sommerfeld
// classes) run the general instantiation.
#include "local.cuh"

namespace helm {

constexpr int LT = 36, LTD = 37, LTH = 96;

__host__ __device__ __forceinline__ double2 fma_(double2 b, double c, double2 a) { return fma_(c, b, a); }

// acc(m, n) = sum_{k < K} A(m, k) B(k, n) for the thread's 4 x 4 block (rows tm + 9i,
// cols tn + 9j); then a barrier; then put(m, n, acc) for m < M, n < Nn.
// LEFT (A = V, B = the data tile): a warp spans 9 rows x ~4 columns, so its B loads
// (complex data) touch 4 addresses and its A loads (V) 9 consecutive ones; otherwise
// (A = data, B = V) a warp spans ~4 rows x 9 columns.  Either way every shared-memory
// load instruction of a k step is one wavefront.
template <bool LEFT, typename TO, typename GA, typename GB, typename PUT>
__device__ __forceinline__ void tile_product(int M, int Nn, int K, GA ga, GB gb, PUT put) {
  const int t = threadIdx.x;
  const int tm = LEFT ? t % 9 : t / 9, tn = LEFT ? t / 9 : t % 9;
  const bool act = t < 81;
  TO acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = Sc<TO>::zero();
  if (act) {
#pragma unroll 2
    for (int k = 0; k < K; ++k) {
      decltype(ga(0, 0)) av[4];
      decltype(gb(0, 0)) bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = ga(tm + 9 * i, k);
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = gb(k, tn + 9 * j);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma_(av[i], bv[j], acc[i][j]);
    }
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (tm + 9 * i < M && tn + 9 * j < Nn) put(tm + 9 * i, tn + 9 * j, acc[i][j]);
  }
}

template <typename T, int U = 7>
__device__ __forceinline__ void load_square(T* dst, const T* __restrict__ src, int L) {
  for (int e0 = threadIdx.x; e0 < L * L; e0 += U * LTH) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * LTH < L * L) v[u] = src[e0 + u * LTH];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * LTH;
      if (e < L * L) dst[(e / L) * LTD + e % L] = v[u];
    }
  }
}

template <typename S, typename VY, typename VX>
__device__ __forceinline__ void fdm_box(const S* __restrict__ xb, const S* __restrict__ bb, S* __restrict__ yb,
                                        S* __restrict__ ob, const LocalArgs& a, const VY* __restrict__ Vyg,
                                        const VX* __restrict__ Vxg, const S* __restrict__ lyg,
                                        const S* __restrict__ lxg, int ay, int ax, unsigned char* sm) {
  S* X = reinterpret_cast<S*>(sm);
  VY* Vy = reinterpret_cast<VY*>(X + LT * LTD);
  VX* Vx = reinterpret_cast<VX*>(Vy + LT * LTD);
  S* ly = reinterpret_cast<S*>(Vx + LT * LTD);
  S* lx = ly + LT;
  S* cw = lx + LT;  // [WIN][WIN] coarse window (coarse-base mode)
  const int nu = a.nu;
  const int y0 = a.box_start[ay], Ly = a.box_len[ay];
  const int x0 = a.box_start[ax], Lx = a.box_len[ax];
  const int Uby = window_base(y0, a.off), Ubx = window_base(x0, a.off);
  if (bb && a.coarse_base) window_load(cw, bb, a, Uby, Ubx, LTH);
  // gather the box (weights first when weights_before_solve, schwarz.py:69-70)
  constexpr int U = 7;
  for (int e0 = threadIdx.x; e0 < Ly * Lx; e0 += U * LTH) {
    S v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * LTH;
      if (e < Ly * Lx) v[u] = xb[(size_t)(y0 + e / Lx) * nu + x0 + e % Lx];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * LTH;
      if (e < Ly * Lx) {
        const int r = e / Lx, q = e % Lx;
        if (a.weighted && a.wbs) v[u] = scale(v[u], 1.0 / (a.node_mult[y0 + r] * a.node_mult[x0 + q]));
        X[r * LTD + q] = v[u];
      }
    }
  }
  load_square<VY>(Vy, Vyg, Ly);
  load_square<VX>(Vx, Vxg, Lx);
  for (int e = threadIdx.x; e < Ly; e += LTH) ly[e] = lyg[e];
  for (int e = threadIdx.x; e < Lx; e += LTH) lx[e] = lxg[e];
  __syncthreads();
  // X <- Vy^T X
  tile_product<true, S>(Ly, Lx, Ly, [&](int m, int k) { return Vy[k * LTD + m]; },
                  [&](int k, int n) { return X[k * LTD + n]; }, [&](int m, int n, S v) { X[m * LTD + n] = v; });
  __syncthreads();
  // X <- (X Vx) ./ (ly (+) lx - k^2)
  tile_product<false, S>(Ly, Lx, Lx, [&](int m, int k) { return X[m * LTD + k]; },
                  [&](int k, int n) { return Vx[k * LTD + n]; }, [&](int m, int n, S v) {
                    X[m * LTD + n] = div_(v, sub(add(ly[m], lx[n]), Sc<S>::from_real(a.k2)));
                  });
  __syncthreads();
  // X <- Vy X
  tile_product<true, S>(Ly, Lx, Ly, [&](int m, int k) { return Vy[m * LTD + k]; },
                  [&](int k, int n) { return X[k * LTD + n]; }, [&](int m, int n, S v) { X[m * LTD + n] = v; });
  cp_wait<0>();
  __syncthreads();
  // Y = X Vx^T, weighted, written out (overlap nodes into their slot of the scratch)
  tile_product<false, S>(Ly, Lx, Lx, [&](int m, int k) { return X[m * LTD + k]; },
                  [&](int k, int n) { return Vx[n * LTD + k]; }, [&](int r, int q, S acc) {
                    const int iy = y0 + r, ix = x0 + q;
                    const int my = a.node_mult[iy], mx = a.node_mult[ix];
                    if (a.weighted && !a.wbs) acc = scale(acc, 1.0 / (my * mx));
                    const size_t pidx = (size_t)iy * nu + ix;
                    if (my == 1 && mx == 1) {
                      yb[pidx] = bb ? add(a.coarse_base ? window_prolong(cw, a.off, Uby, Ubx, iy, ix) : bb[pidx], acc)
                                    : acc;
                    } else if (my == 2) {
                      const int ry = ay - a.node_first_box[iy], rx = ax - a.node_first_box[ix];
                      ob[((size_t)(ry * 2 + rx) * a.nbands + a.node_band[iy]) * nu + ix] = acc;
                    } else {
                      const int rx = ax - a.node_first_box[ix];
                      ob[(size_t)4 * a.nbands * nu + ((size_t)rx * nu + iy) * a.nbands + a.node_band[ix]] = acc;
                    }
                  });
}

// RR: every box of the list has two real classes (V read from classVr).
template <typename S, bool RR>
__global__ void __launch_bounds__(LTH) local_fdm_fast_kernel(const S* __restrict__ x, const S* __restrict__ base,
                                                             S* __restrict__ y, S* __restrict__ ovl,
                                                             const int* __restrict__ boxes,
                                                             const S* __restrict__ classV,
                                                             const double* __restrict__ classVr,
                                                             const int* __restrict__ class_real,
                                                             const S* __restrict__ classLam, LocalArgs a) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int sid = boxes[blockIdx.x];
  const int ay = sid / a.p, ax = sid % a.p;
  const size_t N = (size_t)a.nu * a.nu;
  const int b = blockIdx.y;
  const int cy = a.box_class[ay], cx = a.box_class[ax];
  const S* xb = x + (size_t)b * N;
  const S* bb = base ? base + (size_t)b * base_stride(a) : nullptr;
  S* yb = y + (size_t)b * N;
  S* ob = ovl + (size_t)b * 6 * a.nbands * a.nu;
  const S* ly = classLam + a.class_off_lam[cy];
  const S* lx = classLam + a.class_off_lam[cx];
  const double* Vyr = classVr + a.class_off_V[cy];
  const double* Vxr = classVr + a.class_off_V[cx];
  if constexpr (RR) {
    fdm_box<S, double, double>(xb, bb, yb, ob, a, Vyr, Vxr, ly, lx, ay, ax, smem_raw);
  } else {
    const S* Vyc = classV + a.class_off_V[cy];
    const S* Vxc = classV + a.class_off_V[cx];
    const bool ry = class_real[cy] != 0, rx = class_real[cx] != 0;
    if (ry)
      fdm_box<S, double, S>(xb, bb, yb, ob, a, Vyr, Vxc, ly, lx, ay, ax, smem_raw);
    else if (rx)
      fdm_box<S, S, double>(xb, bb, yb, ob, a, Vyc, Vxr, ly, lx, ay, ax, smem_raw);
    else
      fdm_box<S, S, S>(xb, bb, yb, ob, a, Vyc, Vxc, ly, lx, ay, ax, smem_raw);
  }
}

template <typename S, bool RR>
static void fast_launch(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a,
                        const int* boxes, int nbox, int batch, cudaStream_t st) {
  if (nbox == 0) return;
  const PlanDev& d = P->dev;
  const size_t vsz = RR ? sizeof(double) : sizeof(S);
  const size_t smem = (size_t)LT * LTD * (sizeof(S) + 2 * vsz) + 2 * LT * sizeof(S) + WIN * WIN * sizeof(S);
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(local_fdm_fast_kernel<S, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr = true;
  }
  dim3 grd(nbox, batch);
  launch_pdl(local_fdm_fast_kernel<S, RR>, grd, LTH, smem, st, x, base, y, ovl, boxes, (const S*)d.class_V, d.class_Vr,
                                                       d.class_real, (const S*)d.class_lambda, a);
  HELM_LAUNCH_CHECK();
}

template <typename S>
bool launch_local_fast(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st, helm_workspace* ws) {
  const PlanDev& d = P->dev;
  if (d.max_len > LT) return false;
  // The box groups write disjoint nodes / overlap slots, so with a workspace the DFMA boxes
  // run on its side stream beside the tensor-core boxes (at batch 1 they are < 1 wave and
  // would otherwise leave most SMs idle for their whole duration).
  const bool fork = ws && ws->side && (d.n_rr + d.n_mix + d.n_edge) > 0;
  cudaStream_t sf = fork ? ws->side : st;
  if (fork) {
    HELM_CUDA(cudaEventRecord(ws->fork, st));
    HELM_CUDA(cudaStreamWaitEvent(ws->side, ws->fork, 0));
  }
  fast_launch<S, false>(P, x, base, y, ovl, a, d.box_mix, d.n_mix, batch, sf);
  launch_local_edge<S>(P, x, base, y, ovl, a, batch, sf);  // edge boxes: sine transform + tridiagonal
  fast_launch<S, true>(P, x, base, y, ovl, a, d.box_rr, d.n_rr, batch, sf);
  launch_local_dst<S>(P, x, base, y, ovl, a, batch, st);   // middle-pencil boxes: fast sine transforms
  launch_local_dmma<S>(P, x, base, y, ovl, a, batch, st);  // other folded real classes: FP64 tensor pipe
  if (fork) {
    HELM_CUDA(cudaEventRecord(ws->join, ws->side));
    HELM_CUDA(cudaStreamWaitEvent(st, ws->join, 0));
  }
  return true;
}

template bool launch_local_fast<double>(const helm_plan*, const double*, const double*, double*, double*,
                                        const LocalArgs&, int, cudaStream_t, helm_workspace*);
template bool launch_local_fast<double2>(const helm_plan*, const double2*, const double2*, double2*, double2*,
                                         const LocalArgs&, int, cudaStream_t, helm_workspace*);

}  // namespace helm
