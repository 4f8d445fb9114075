// K5: the coarse solve  y = A0^{-1} c  (reference: linalg.solve(cs.a0_factorization, .)
// at coarse.py:174, SuperLU factor of the symmetrised Galerkin matrix, coarse.py:154-167).
//
// A0 = T0(x)M0 + M0(x)T0 - k^2 M0(x)M0 (y (x) x) with pentadiagonal 1-D pencils
// T0 = P T P^T, M0 = P W P^T (verified bitwise against the reference).
//
// Dirichlet (MP-1): T0 and M0 are exactly diagonalised by the DST-I (the Bezier
// restriction is consistent with the odd extension), so
//   A0^{-1} = (Q(x)Q) diag(1 / (lT_y lM_x + lM_y lT_x - k^2 lM_y lM_x)) (Q^-1(x)Q^-1)
// = row DST, transpose, row DST + 2-D scaling, row DST, transpose, row DST.
//
// Sommerfeld (MP-2): along x, T0 = T~ + L_T and M0 = M~ + L_M where (T~, M~) is
// diagonalised by the DCT-I (T~ Q = W Q lamT, M~ Q = W Q lamM) and L_T, L_M live
// on the 2x2 corner blocks (the restriction drops its out-of-range taps,
// coarse.py:116-128, instead of reflecting them).  One solve is
//   1. F^ = DCT_x(F) * sigma_a                                    (xform.cu)
//   2. per x-mode a: (T0 + s_a M0) Y^[:,a] = F^[:,a]                (band.cu; the exact,
//      damped y-operator, so no near-resonant division appears)
//   3. Woodbury on the 4 strip columns x in {0, 1, m0-2, m0-1}:
//        Z = Y^ q (strip values), z^ = (V^T M0) Z, c^_b = H_b z^_b (4x4 per y-mode b
//        of the y-pencil T0 V = M0 V diag(lam)), cS = (M0 V) c^,
//        F^ -= sigma_a cS q^T, and step 2 again
//   4. Y = DCT_x(Y^).
// Everything is O(m0^2 log m0) per right-hand side and HBM-bound (dense fast
// diagonalisation would be O(m0^3) FP64).  refine_steps iterative-refinement
// steps r = c - A0 y (25-point residual), y += solve(r) follow.
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace helm {

// ----------------------------------------------------------------------------
// Woodbury strip step
// ----------------------------------------------------------------------------
// Z[y][b*4+i] = sum_a q[a][i] Yh[b][y][a]   (one warp per (batch, row))
constexpr int SCH = 8;  // row elements per lane in flight (strip reduction)
template <typename S>
__global__ void __launch_bounds__(256) strip_reduce_kernel(const S* __restrict__ Yh, const double* __restrict__ q,
                                                           S* __restrict__ Z, int m0, int ldz) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int y = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  if (y >= m0) return;
  const S* row = Yh + ((size_t)b * m0 + y) * m0;
  S acc[4] = {Sc<S>::zero(), Sc<S>::zero(), Sc<S>::zero(), Sc<S>::zero()};
  // chunks of SCH elements per lane are loaded before they are summed (all loads of a
  // chunk in flight); the summation order per lane is a = lane, lane + 32, ... as before
  // (q, 33 KB, is read through L1 at use: only the streamed row is held in registers)
  for (int a0 = lane; a0 < m0; a0 += 32 * SCH) {
    S v[SCH];
#pragma unroll
    for (int i = 0; i < SCH; ++i) {
      const int a = a0 + 32 * i;
      if (a < m0) v[i] = row[a];
    }
#pragma unroll
    for (int i = 0; i < SCH; ++i) {
      const int a = a0 + 32 * i;
      if (a < m0) {
        const double4 qa = *reinterpret_cast<const double4*>(q + (size_t)a * 4);
        acc[0] = fma_(qa.x, v[i], acc[0]);
        acc[1] = fma_(qa.y, v[i], acc[1]);
        acc[2] = fma_(qa.z, v[i], acc[2]);
        acc[3] = fma_(qa.w, v[i], acc[3]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i] = warp_sum(acc[i]);
  if (lane < 4) Z[(size_t)y * ldz + (size_t)b * 4 + lane] = acc[lane];
}

// Small batches: the same strip values with compensated sums (CSum), each row split over
// WPR warps (lanes stride the row by 32 * WPR, warp partials merged in warp order).
template <int WPR, bool COMP>
__global__ void __launch_bounds__(256) strip_reduce_c_kernel(const double2* __restrict__ Yh,
                                                             const double* __restrict__ q, double2* __restrict__ Z,
                                                             int m0, int ldz) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  using CS = CSum<COMP>;
  __shared__ CS red[8][8];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31, sw = wl % WPR;
  const int yy = (blockIdx.x * blockDim.x + threadIdx.x) / (32 * WPR);
  const int b = blockIdx.y;
  const bool ok = yy < m0;
  const double2* row = Yh + ((size_t)b * m0 + (ok ? yy : 0)) * m0;
  CS acc[8];
#pragma unroll 4
  for (int a = sw * 32 + lane; a < (ok ? m0 : 0); a += 32 * WPR) {
    const double2 v = row[a];
    const double4 qa = *reinterpret_cast<const double4*>(q + (size_t)a * 4);
    acc[0].fma(qa.x, v.x);
    acc[1].fma(qa.x, v.y);
    acc[2].fma(qa.y, v.x);
    acc[3].fma(qa.y, v.y);
    acc[4].fma(qa.z, v.x);
    acc[5].fma(qa.z, v.y);
    acc[6].fma(qa.w, v.x);
    acc[7].fma(qa.w, v.y);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) warp_csum(acc[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) red[wl][i] = acc[i];
  }
  __syncthreads();
  if (ok && sw == 0 && lane < 4) {
    CS re = red[wl][2 * lane], im = red[wl][2 * lane + 1];
#pragma unroll
    for (int w = 1; w < WPR; ++w) {
      re.merge(red[wl + w][2 * lane]);
      im.merge(red[wl + w][2 * lane + 1]);
    }
    Z[(size_t)yy * ldz + (size_t)b * 4 + lane] = mk(re.val(), im.val());
  }
}

// which small-batch strip sums are compensated: bit 0 the strip reduction, bit 1 the
// fold GEMVs (HELM_STRIP_COMP, default 0).  Measured at batch 1, n = 2049: plain 0.330 ms
// per coarse solve, fully compensated 0.378 ms; the cfg4a GMRES count is 364 with either
// (and on both band paths), so the plain sums are the default and the compensated ones the
// check that a count does not hinge on the split's rounding.
static int strip_comp() {
  static const int v = [] {
    const char* e = std::getenv("HELM_STRIP_COMP");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

template <typename S>
static void strip_reduce(const S* Yh, const double* q, S* Z, int m0, int batch, cudaStream_t st) {
  if constexpr (Sc<S>::cplx) {
    if (batch <= 4) {
      constexpr int WPR = 4;
      dim3 grd((unsigned)((m0 * 32 * WPR + 255) / 256), batch);
      if (strip_comp() & 1)
        launch_pdl(strip_reduce_c_kernel<WPR, true>, grd, 256, 0, st, Yh, q, Z, m0, batch * 4);
      else
        launch_pdl(strip_reduce_c_kernel<WPR, false>, grd, 256, 0, st, Yh, q, Z, m0, batch * 4);
      HELM_LAUNCH_CHECK();
      return;
    }
  }
  dim3 grd((unsigned)((m0 * 32 + 255) / 256), batch);
  launch_pdl(strip_reduce_kernel<S>, grd, 256, 0, st, Yh, q, Z, m0, batch * 4);
  HELM_LAUNCH_CHECK();
}

// --- strip GEMMs on the folded (even / odd) mode blocks ------------------------
// The y-pencil is reflection symmetric, so its modes are even (first he) or odd (last ho)
// and every product with V^T M0, V^T or M0 V splits into two half-size blocks
// (include/helmb200.h): half the FLOPs and half the matrix bytes of a dense product.
//   left  (mode <- y):  Zf = [Z[y] + Z[m0-1-y] ; Z[y] - Z[m0-1-y]] (strip_fold_kernel), then
//                       out[e] = A_e Zf_s, out[he+o] = A_o Zf_d, then the per-mode 4x4 epilogue;
//   right (y <- mode):  E = A_e c_e, O = A_o c_o, out[y] = E + O, out[m0-1-y] = E - O.
// Columns are the batch's 4 strip columns per right-hand side (ldn = 4 * batch).
__global__ void __launch_bounds__(256) strip_fold_kernel(const double2* __restrict__ Z, double2* __restrict__ Zf,
                                                         int m0, int ldn) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int he = (m0 + 1) / 2, ho = m0 / 2;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= he * ldn) return;
  const int y = e / ldn, c = e % ldn;
  const double2 a = Z[(size_t)y * ldn + c];
  if (y < ho) {
    const double2 b = Z[(size_t)(m0 - 1 - y) * ldn + c];
    Zf[(size_t)y * ldn + c] = add(a, b);
    Zf[(size_t)(he + y) * ldn + c] = sub(a, b);
  } else {
    Zf[(size_t)y * ldn + c] = a;  // the centre row (odd m0) belongs to the even block only
  }
}

// part[ks][rowoff_g + m][n] = sum_{k in chunk ks} A_g[m][k] B[rowoff_g + k][n], g = even / odd.
// 64 x 64 complex outputs per CTA (256 threads, 4 x 4 each), K tiles of 16 double-buffered
// through shared memory with cp.async; split-K over blockIdx.z into a partial-sum scratch
// reduced in a fixed order (deterministic).
constexpr int FG_M = 64, FG_N = 64, FG_K = 16, FG_KS = 8;
struct FoldGemmSmem {
  double2 A[2][FG_M][FG_K + 1];
  double2 B[2][FG_K][FG_N];
};
__global__ void __launch_bounds__(256) strip_gemm_fold_kernel(const double2* __restrict__ A,
                                                              const double2* __restrict__ B,
                                                              double2* __restrict__ part, int m0, int ldn) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  FoldGemmSmem& sm = *reinterpret_cast<FoldGemmSmem*>(sraw);
  const int he = (m0 + 1) / 2, ho = m0 / 2;
  const int tiles_e = (he + FG_M - 1) / FG_M;
  const int g = blockIdx.y < tiles_e ? 0 : 1;
  const int Mg = g ? ho : he;
  const int m0t = (g ? blockIdx.y - tiles_e : blockIdx.y) * FG_M;
  const double2* Ag = A + (g ? (size_t)he * he : 0);
  const int rowoff = g ? he : 0;
  const int n0 = blockIdx.x * FG_N;
  const int kchunk = ((Mg + FG_KS - 1) / FG_KS + FG_K - 1) / FG_K * FG_K;
  const int kb = blockIdx.z * kchunk, ke = min(Mg, kb + kchunk);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  auto issue = [&](int buf, int k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + 256 * r;
      const int mm = e >> 4, kk = e & 15;
      const int m = m0t + mm, k = k0 + kk;
      const bool ok = m < Mg && k < ke;
      cp_async16(&sm.A[buf][mm][kk], Ag + (ok ? (size_t)m * Mg + k : 0), ok);
      const int kk2 = e >> 6, nn = e & 63;
      const int k2 = k0 + kk2, n = n0 + nn;
      const bool ok2 = k2 < ke && n < ldn;
      cp_async16(&sm.B[buf][kk2][nn], B + (ok2 ? (size_t)(rowoff + k2) * ldn + n : 0), ok2);
    }
    cp_commit();
  };
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = mk(0.0, 0.0);
  if (kb < ke) issue(0, kb);
  int buf = 0;
  for (int k0 = kb; k0 < ke; k0 += FG_K) {
    if (k0 + FG_K < ke) {
      issue(buf ^ 1, k0 + FG_K);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < FG_K; ++kk) {
      double2 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = sm.A[buf][ty + 16 * i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sm.B[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma_(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0t + ty + 16 * i;
    if (m >= Mg) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n < ldn) part[((size_t)blockIdx.z * m0 + rowoff + m) * ldn + n] = acc[i][j];
    }
  }
}

// Warp-per-row form for few columns (batch <= 4): part[0][row][.] for the packed row.
template <int NC>
__global__ void __launch_bounds__(256) strip_gemm_fold_rows_kernel(const double2* __restrict__ A,
                                                                   const double2* __restrict__ B,
                                                                   double2* __restrict__ part, int m0) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= m0) return;
  const int he = (m0 + 1) / 2;
  const int g = r < he ? 0 : 1;
  const int Mg = g ? m0 / 2 : he, rowoff = g ? he : 0;
  const double2* arow = A + (g ? (size_t)he * he : 0) + (size_t)(r - rowoff) * Mg;
  double2 acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = mk(0.0, 0.0);
  for (int k = lane; k < Mg; k += 32) {
    const double2 av = arow[k];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = fma_(av, B[(size_t)(rowoff + k) * NC + c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = warp_sum(acc[c]);
  if (lane < NC) {
    double2 v = acc[0];
#pragma unroll
    for (int c = 1; c < NC; ++c)
      if (lane == c) v = acc[c];
    part[(size_t)r * NC + lane] = v;
  }
}

// left epilogue: out[r][g*4+i] = sum_j H[r][i][j] t[j],  t = sum_ks part[ks][r][g*4+.]
__global__ void __launch_bounds__(256) strip_reduce_left_kernel(const double2* __restrict__ part,
                                                                double2* __restrict__ out,
                                                                const double2* __restrict__ Hm, int m0,
                                                                int ngroups, int nks) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m0 * ngroups) return;
  const int r = e / ngroups, g = e % ngroups;
  const size_t ldn = (size_t)ngroups * 4;
  double2 t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double2 s = mk(0.0, 0.0);
    for (int ks = 0; ks < nks; ++ks) s = add(s, part[((size_t)ks * m0 + r) * ldn + g * 4 + i]);
    t[i] = s;
  }
  const double2* h = Hm + (size_t)r * 16;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double2 s = mk(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < 4; ++j) s = fma_(h[i * 4 + j], t[j], s);
    out[(size_t)r * ldn + g * 4 + i] = s;
  }
}

// right epilogue: E = rows [0, he), O = rows [he, m0) of the partials;
// out[y] = E + O (- minus[y]), out[m0-1-y] = E - O (- minus[m0-1-y]), out[h] = E (odd m0)
__global__ void __launch_bounds__(256) strip_reduce_right_kernel(const double2* __restrict__ part,
                                                                 double2* __restrict__ out,
                                                                 const double2* __restrict__ minus, int m0,
                                                                 int ldn, int nks) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int he = (m0 + 1) / 2, ho = m0 / 2;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= he * ldn) return;
  const int y = e / ldn, c = e % ldn;
  double2 E = mk(0.0, 0.0), O = mk(0.0, 0.0);
  for (int ks = 0; ks < nks; ++ks) {
    E = add(E, part[((size_t)ks * m0 + y) * ldn + c]);
    if (y < ho) O = add(O, part[((size_t)ks * m0 + he + y) * ldn + c]);
  }
  if (y < ho) {
    double2 lo = add(E, O), hi = sub(E, O);
    const size_t pl = (size_t)y * ldn + c, ph = (size_t)(m0 - 1 - y) * ldn + c;
    if (minus) {
      lo = sub(lo, minus[pl]);
      hi = sub(hi, minus[ph]);
    }
    out[pl] = lo;
    out[ph] = hi;
  } else {
    const size_t pl = (size_t)y * ldn + c;
    out[pl] = minus ? sub(E, minus[pl]) : E;
  }
}

// Small batches (<= 4 right-hand sides, NC = 4 * batch strip columns): WPR warps per output
// row (lanes stride the row by 32 * WPR), compensated sums (CSum: the result does not
// depend on that split at the rounding level), the fold / unfold and the 4x4 epilogue fused
// into the product (one launch per side).
// Cross-warp total of the row's per-warp sums, merged in warp order; the totals land in
// the row's first warp.  All threads of the CTA call it.
template <int NC, int WPR, bool C>
__device__ __forceinline__ void row_total_c(CSum<C> (&re)[NC], CSum<C> (&im)[NC], int wl, int lane,
                                            double2 (&acc)[NC]) {
  if constexpr (WPR == 1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = mk(re[c].val(), im[c].val());
  } else {
    __shared__ CSum<C> red[8][NC][2];
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        red[wl][c][0] = re[c];
        red[wl][c][1] = im[c];
      }
    }
    __syncthreads();
    if (wl % WPR == 0) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        CSum<C> r = red[wl][c][0], i = red[wl][c][1];
#pragma unroll
        for (int w = 1; w < WPR; ++w) {
          r.merge(red[wl + w][c][0]);
          i.merge(red[wl + w][c][1]);
        }
        acc[c] = mk(r.val(), i.val());
      }
    }
    __syncthreads();  // the shared partials may be reused by the next call
  }
}

// left:  row r of the packed mode blocks, t = A_g[r] . fold(Z), out[r] = Hm[r] t  (Hm may be null)
template <int NC, int WPR, bool COMP>
__global__ void __launch_bounds__(256) strip_left_fused_kernel(const double2* __restrict__ A,
                                                               const double2* __restrict__ Z,
                                                               double2* __restrict__ out,
                                                               const double2* __restrict__ Hm, int m0) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31, sw = wl % WPR;
  const int rr = (blockIdx.x * blockDim.x + threadIdx.x) / (32 * WPR);
  const bool ok = rr < m0;
  const int r = ok ? rr : m0 - 1;
  const int he = (m0 + 1) / 2, ho = m0 / 2;
  const bool odd = r >= he;
  const int Mg = odd ? ho : he;
  const double2* arow = A + (odd ? (size_t)he * he + (size_t)(r - he) * ho : (size_t)r * he);
  CSum<COMP> re[NC], im[NC];
#pragma unroll(NC <= 8 ? 4 : 1)
  for (int k = sw * 32 + lane; k < (ok ? Mg : 0); k += 32 * WPR) {
    const double2 av = arow[k];
    const double2* z0 = Z + (size_t)k * NC;
    const double2* z1 = Z + (size_t)(m0 - 1 - k) * NC;
    const bool centre = !odd && k == ho;  // odd m0: the centre row belongs to the even block alone
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double2 a = z0[c];
      const double2 f = centre ? a : (odd ? sub(a, z1[c]) : add(a, z1[c]));
      csum_cfma(re[c], im[c], av, f);
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    warp_csum(re[c]);
    warp_csum(im[c]);
  }
  double2 acc[NC];
  row_total_c<NC, WPR>(re, im, wl, lane, acc);
  if (ok && sw == 0 && lane < NC) {
    const int g = lane >> 2, i = lane & 3;
    double2 v;
    if (Hm) {
      const double2* h = Hm + (size_t)r * 16 + i * 4;
      v = mk(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double2 tj = acc[0];
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c == g * 4 + j) tj = acc[c];
        v = fma_(h[j], tj, v);
      }
    } else {
      v = acc[0];
#pragma unroll
      for (int c = 1; c < NC; ++c)
        if (lane == c) v = acc[c];
    }
    out[(size_t)r * NC + lane] = v;
  }
}

// right: for y < he, E = A_e[y] . cin[0:he), O = A_o[y] . cin[he:m0) (y < ho);
// out[y] = E + O (- minus[y]), out[m0-1-y] = E - O (- minus[m0-1-y]), out[centre] = E
template <int NC, int WPR, bool COMP>
__global__ void __launch_bounds__(256) strip_right_fused_kernel(const double2* __restrict__ A,
                                                                const double2* __restrict__ cin,
                                                                double2* __restrict__ out,
                                                                const double2* __restrict__ minus, int m0) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31, sw = wl % WPR;
  const int yy = (blockIdx.x * blockDim.x + threadIdx.x) / (32 * WPR);
  const int he = (m0 + 1) / 2, ho = m0 / 2;
  const bool ok = yy < he;
  const int y = ok ? yy : he - 1;
  const double2* ae = A + (size_t)y * he;
  const double2* ao = A + (size_t)he * he + (size_t)y * ho;
  CSum<COMP> er[NC], ei[NC], orr[NC], oi[NC];
#pragma unroll(NC <= 8 ? 4 : 1)
  for (int k = sw * 32 + lane; k < (ok ? he : 0); k += 32 * WPR) {
    const double2 av = ae[k];
#pragma unroll
    for (int c = 0; c < NC; ++c) csum_cfma(er[c], ei[c], av, cin[(size_t)k * NC + c]);
  }
  if (y < ho) {
#pragma unroll(NC <= 8 ? 4 : 1)
    for (int k = sw * 32 + lane; k < (ok ? ho : 0); k += 32 * WPR) {
      const double2 av = ao[k];
#pragma unroll
      for (int c = 0; c < NC; ++c) csum_cfma(orr[c], oi[c], av, cin[(size_t)(he + k) * NC + c]);
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    warp_csum(er[c]);
    warp_csum(ei[c]);
    warp_csum(orr[c]);
    warp_csum(oi[c]);
  }
  double2 E[NC], O[NC];
  row_total_c<NC, WPR>(er, ei, wl, lane, E);
  row_total_c<NC, WPR>(orr, oi, wl, lane, O);
  if (ok && sw == 0 && lane < NC) {
    double2 e = E[0], o = O[0];
#pragma unroll
    for (int c = 1; c < NC; ++c)
      if (lane == c) {
        e = E[c];
        o = O[c];
      }
    const size_t pl = (size_t)y * NC + lane, ph = (size_t)(m0 - 1 - y) * NC + lane;
    if (y < ho) {
      double2 lo = add(e, o), hi = sub(e, o);
      if (minus) {
        lo = sub(lo, minus[pl]);
        hi = sub(hi, minus[ph]);
      }
      out[pl] = lo;
      out[ph] = hi;
    } else {
      out[pl] = minus ? sub(e, minus[pl]) : e;
    }
  }
}

// out = fold-GEMM of Zin with the packed blocks A; left: + 4x4 epilogue Hm (Zin in y order,
// folded here into Zf); right: unfolded, minus subtracted (Zin in mode order).
static void strip_gemm_fold(const double2* A, const double2* Zin, double2* out, bool left, const double2* Hm,
                            const double2* minus, int m0, int batch, double2* Zf, double2* part, cudaStream_t st) {
  const int ldn = 4 * batch, he = (m0 + 1) / 2, ho = m0 / 2;
  if (batch <= 4) {
    auto go = [&](auto nc) {
      constexpr int NC = decltype(nc)::value;
      constexpr int WPR = NC <= 8 ? 4 : 2;  // few rows: each split over WPR warps
      const int blocks_l = (m0 * 32 * WPR + 255) / 256, blocks_r = (he * 32 * WPR + 255) / 256;
      const bool comp = strip_comp() & 2;
      if (left && comp)
        launch_pdl(strip_left_fused_kernel<NC, WPR, true>, blocks_l, 256, 0, st, A, Zin, out, Hm, m0);
      else if (left)
        launch_pdl(strip_left_fused_kernel<NC, WPR, false>, blocks_l, 256, 0, st, A, Zin, out, Hm, m0);
      else if (comp)
        launch_pdl(strip_right_fused_kernel<NC, WPR, true>, blocks_r, 256, 0, st, A, Zin, out, minus, m0);
      else
        launch_pdl(strip_right_fused_kernel<NC, WPR, false>, blocks_r, 256, 0, st, A, Zin, out, minus, m0);
    };
    switch (batch) {
      case 1: go(std::integral_constant<int, 4>{}); break;
      case 2: go(std::integral_constant<int, 8>{}); break;
      case 3: go(std::integral_constant<int, 12>{}); break;
      default: go(std::integral_constant<int, 16>{}); break;
    }
    HELM_LAUNCH_CHECK();
    return;
  }
  const double2* B = Zin;
  if (left) {
    launch_pdl(strip_fold_kernel, (he * ldn + 255) / 256, 256, 0, st, Zin, Zf, m0, ldn);
    HELM_LAUNCH_CHECK();
    B = Zf;
  }
  int nks = 1;
  const int rows_blocks = (m0 * 32 + 255) / 256;
  switch (batch) {
    case 1: launch_pdl(strip_gemm_fold_rows_kernel<4>, rows_blocks, 256, 0, st, A, B, part, m0); break;
    case 2: launch_pdl(strip_gemm_fold_rows_kernel<8>, rows_blocks, 256, 0, st, A, B, part, m0); break;
    case 3: launch_pdl(strip_gemm_fold_rows_kernel<12>, rows_blocks, 256, 0, st, A, B, part, m0); break;
    case 4: launch_pdl(strip_gemm_fold_rows_kernel<16>, rows_blocks, 256, 0, st, A, B, part, m0); break;
    default: {
      static bool attr = false;
      if (!attr) {
        HELM_CUDA(cudaFuncSetAttribute(strip_gemm_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(FoldGemmSmem)));
        attr = true;
      }
      const int tiles = (he + FG_M - 1) / FG_M + (ho + FG_M - 1) / FG_M;
      dim3 grd((ldn + FG_N - 1) / FG_N, tiles, FG_KS);
      launch_pdl(strip_gemm_fold_kernel, grd, 256, sizeof(FoldGemmSmem), st, A, B, part, m0, ldn);
      nks = FG_KS;
    }
  }
  HELM_LAUNCH_CHECK();
  if (left)
    launch_pdl(strip_reduce_left_kernel, (m0 * batch + 255) / 256, 256, 0, st, part, out, Hm, m0, batch, nks);
  else
    launch_pdl(strip_reduce_right_kernel, (he * ldn + 255) / 256, 256, 0, st, part, out, minus, m0, ldn, nks);
  HELM_LAUNCH_CHECK();
}

// --- strip refinement ----------------------------------------------------------
// rho[y][b*4+i] = cS[y][b*4+i] - sum_j ((T0 yS_j)[y] LM[i][j] + (M0 yS_j)[y] (LT[i][j] - k^2 LM[i][j]))
// the exact residual A0 y - F on the strip columns of y = B^{-1}(F - ext(cS))
// (A0 - B is supported on the strip x strip block of the x-pencil).
struct StripCoupling {
  double2 lm[16];
  double2 lk[16];  // LT - k^2 LM
};
__global__ void __launch_bounds__(256) strip_rho_kernel(const double2* __restrict__ cS, const double2* __restrict__ yS,
                                                        double2* __restrict__ rho, const double2* __restrict__ t0b,
                                                        const double2* __restrict__ m0b, StripCoupling cp, int m0,
                                                        int batch) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m0 * batch) return;
  const int y = e / batch, b = e % batch;
  const size_t ldz = (size_t)batch * 4;
  double2 ty[4], my[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) ty[j] = my[j] = mk(0.0, 0.0);
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const int yy = y + d - 2;
    if (yy < 0 || yy >= m0) continue;
    const double2 tb = t0b[y * 5 + d], mb = m0b[y * 5 + d];
    const double2* v = yS + (size_t)yy * ldz + (size_t)b * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      ty[j] = fma_(tb, v[j], ty[j]);
      my[j] = fma_(mb, v[j], my[j]);
    }
  }
  const double2* c = cS + (size_t)y * ldz + (size_t)b * 4;
  double2* o = rho + (size_t)y * ldz + (size_t)b * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double2 s = mk(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      s = fma_(cp.lm[i * 4 + j], ty[j], s);
      s = fma_(cp.lk[i * 4 + j], my[j], s);
    }
    o[i] = sub(c[i], s);
  }
}

__global__ void strip_axpy_kernel(double2* __restrict__ c, const double2* __restrict__ w, size_t n) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) c[e] = add(c[e], w[e]);
}

// --- r = c - A0 y  (25-point Kronecker-sum stencil from the 1-D bands) ------
// 32 x 32 outputs per CTA (256 threads, 4 rows each); the (32+4) x (32+4) window
// of y is staged in shared memory (zero outside = the band ends), then the
// separable x-pass (M0 and T0 - k^2 M0 rows) and y-pass run from shared memory.
constexpr int RSX = 32, RSY = 32;
template <typename S>
__global__ void __launch_bounds__(256) a0_residual_kernel(const S* __restrict__ c, const S* __restrict__ y,
                                                          S* __restrict__ r, const S* __restrict__ t0b,
                                                          const S* __restrict__ m0b, double k2, int m0) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  S (*ys)[RSX + 4] = reinterpret_cast<S (*)[RSX + 4]>(sraw);
  S (*xm)[RSX] = reinterpret_cast<S (*)[RSX]>(ys + (RSY + 4));
  S (*xt)[RSX] = xm + (RSY + 4);
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int V0 = blockIdx.x * RSX, U0 = blockIdx.y * RSY;
  const size_t off = (size_t)blockIdx.z * m0 * m0;
  {  // all of the thread's window loads in flight at once
    constexpr int NR = (RSY + 4 + 7) / 8, NC = (RSX + 4 + 31) / 32;
    S v[NR][NC];
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const int rr = ty + 8 * i, q = tx + 32 * j, U = U0 + rr - 2, W = V0 + q - 2;
        v[i][j] = (rr < RSY + 4 && q < RSX + 4 && U >= 0 && U < m0 && W >= 0 && W < m0)
                      ? y[off + (size_t)U * m0 + W]
                      : Sc<S>::zero();
      }
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const int rr = ty + 8 * i, q = tx + 32 * j;
        if (rr < RSY + 4 && q < RSX + 4) ys[rr][q] = v[i][j];
      }
  }
  const int V = V0 + tx;
  S bm[5], bt[5];
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    bm[d] = V < m0 ? m0b[V * 5 + d] : Sc<S>::zero();
    bt[d] = V < m0 ? t0b[V * 5 + d] : Sc<S>::zero();
  }
  __syncthreads();
  for (int rr = ty; rr < RSY + 4; rr += 8) {  // x-pass: sum_dx M0[V][V+dx] y, T0[V][V+dx] y
    S sm = Sc<S>::zero(), stt = Sc<S>::zero();
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      sm = fma_(bm[d], ys[rr][tx + d], sm);
      stt = fma_(bt[d], ys[rr][tx + d], stt);
    }
    xm[rr][tx] = sm;
    xt[rr][tx] = sub(stt, scale(sm, k2));
  }
  __syncthreads();
  if (V >= m0) return;
#pragma unroll
  for (int q = 0; q < RSY / 8; ++q) {
    const int rr = ty + 8 * q, Uc = U0 + rr;
    if (Uc >= m0) break;
    S acc = Sc<S>::zero();  // T0(y) M0(x) + M0(y) (T0(x) - k^2 M0(x))
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      acc = fma_(t0b[Uc * 5 + d], xm[rr + d][tx], acc);
      acc = fma_(m0b[Uc * 5 + d], xt[rr + d][tx], acc);
    }
    const size_t p = off + (size_t)Uc * m0 + V;
    r[p] = sub(c[p], acc);
  }
}


// ----------------------------------------------------------------------------
// composition
// ----------------------------------------------------------------------------
// HELM_STRIP_FIRST=0 keeps the round-1 pass order (full pass, Woodbury pass, refinement pass)
static bool strip_first() {
  static const bool v = [] {
    const char* e = std::getenv("HELM_STRIP_FIRST");
    return !(e && e[0] == '0');
  }();
  return v;
}
// One fast solve: out = A0^{-1} in  (in, out distinct from ws->g / ws->f0)
template <typename S>
static void fast_solve(const helm_plan* P, helm_workspace* ws, const S* in, S* out, int batch, cudaStream_t st,
                       bool accumulate = false) {
  const PlanDev& d = P->dev;
  S* T1 = (S*)ws->g;
  S* T2 = (S*)ws->f0;
  if constexpr (!Sc<S>::cplx) {
    // Dirichlet: separable 2-D DST
    launch_xform<S>(P, in, T1, d.coarse_scale, false, batch, st);
    launch_transpose<S>(T1, T2, d.m0, batch, st);
    launch_xform<S>(P, T2, T1, nullptr, true, batch, st);
    launch_xform<S>(P, T1, T2, nullptr, false, batch, st);
    launch_transpose<S>(T2, T1, d.m0, batch, st);
    launch_xform<S>(P, T1, out, nullptr, false, batch, st, accumulate);
  } else {
    launch_xform<S>(P, in, T1, d.coarse_scale, false, batch, st);
    S* Z = (S*)ws->strip[0];
    S* Ch = (S*)ws->strip[1];
    S* Cs = (S*)ws->strip[2];
    S* part = (S*)ws->strip[3];
    S* Zf = (S*)ws->strip[6];
    S* T3 = (S*)ws->e0;
    S* R = (S*)ws->strip[4];
    S* W = (S*)ws->strip[5];
    StripCoupling cp;
    for (int i = 0; i < 16; ++i) {
      cp.lm[i] = d.strip_lm[i];
      cp.lk[i] = sub(d.strip_lt[i], scale(d.strip_lm[i], P->geo.k2));
    }
    const size_t ns = (size_t)d.m0 * batch * 4;
    if (strip_first() && ws->strip_part && band_vals_usable(P, batch)) {
      // Strip-first order (batch > 4): the strip correction is settled by passes that keep only
      // the strip values (no solution rows written, no separate strip sweep), then ONE full
      // pass forms Y^ = B^{-1}(F^ - ext(cS)).  By linearity this is the sequence below
      // (Y^ = B^{-1}F^ - B^{-1}ext(cS), strip values Z + Z') with 2 + strip_refine passes.
      S* Zp = (S*)ws->strip_part;
      S* Zt = (S*)ws->strip[6];  // Zf is free between the strip GEMMs
      launch_band_vals(P, T1, T2, nullptr, batch, st, Zp, nullptr, Z);  // Z = S B^{-1} F^
      strip_gemm_fold((const double2*)d.cap_left, Z, Ch, true, (const double2*)d.cap_mode, nullptr, d.m0, batch, Zf,
                      part, st);
      strip_gemm_fold((const double2*)d.cap_right, Ch, Cs, false, nullptr, nullptr, d.m0, batch, Zf, part, st);
      for (int it = 0; it < d.strip_refine; ++it) {
        launch_band_vals(P, nullptr, T2, Cs, batch, st, Zp, Z, Zt);  // Zt = Z + S B^{-1}(-ext(cS))
        launch_pdl(strip_rho_kernel, (d.m0 * batch + 255) / 256, 256, 0, st, Cs, Zt, R, (const double2*)d.t0_band,
                   (const double2*)d.m0_band, cp, d.m0, batch);
        HELM_LAUNCH_CHECK();
        strip_gemm_fold((const double2*)d.cap_vt, R, Ch, true, (const double2*)d.cap_hg, nullptr, d.m0, batch, Zf,
                        part, st);
        strip_gemm_fold((const double2*)d.cap_right, Ch, W, false, nullptr, R, d.m0, batch, Zf, part, st);
        launch_pdl(strip_axpy_kernel, (unsigned)((ns + 255) / 256), 256, 0, st, Cs, W, ns);
        HELM_LAUNCH_CHECK();
      }
      launch_band_solve(P, T1, T2, Cs, batch, st);
      launch_xform<S>(P, T2, out, nullptr, false, batch, st, accumulate);
      return;
    }
    launch_band_solve(P, T1, T2, nullptr, batch, st);
    strip_reduce<S>(T2, d.strip_q, Z, d.m0, batch, st);
    strip_gemm_fold((const double2*)d.cap_left, Z, Ch, true, (const double2*)d.cap_mode, nullptr, d.m0, batch, Zf,
                    part, st);
    strip_gemm_fold((const double2*)d.cap_right, Ch, Cs, false, nullptr, nullptr, d.m0, batch, Zf, part, st);
    launch_band_solve(P, T1, T2, Cs, batch, st);
    // strip refinement: rho = cS - C_U y_S from this pass's strip values (exact), the
    // correction W = H G rho - rho from the eigen-space operators (only ~1e-12 accurate,
    // enough for a correction of a ~1e-12 quantity), then Y^ += B^{-1}(-ext(W)).
    for (int it = 0; it < d.strip_refine; ++it) {
      strip_reduce<S>(T2, d.strip_q, Z, d.m0, batch, st);
      launch_pdl(strip_rho_kernel, (d.m0 * batch + 255) / 256, 256, 0, st, Cs, Z, R, (const double2*)d.t0_band,
                                                                  (const double2*)d.m0_band, cp, d.m0, batch);
      HELM_LAUNCH_CHECK();
      strip_gemm_fold((const double2*)d.cap_vt, R, Ch, true, (const double2*)d.cap_hg, nullptr, d.m0, batch, Zf,
                      part, st);
      strip_gemm_fold((const double2*)d.cap_right, Ch, W, false, nullptr, R, d.m0, batch, Zf, part, st);
      launch_band_solve(P, nullptr, T3, W, batch, st, T2);  // T3 = T2 + B^{-1}(-ext(W))
      if (it + 1 < d.strip_refine) {
        launch_pdl(strip_axpy_kernel, (unsigned)((ns + 255) / 256), 256, 0, st, Cs, W, ns);
        HELM_LAUNCH_CHECK();
      }
      std::swap(T2, T3);
    }
    launch_xform<S>(P, T2, out, nullptr, false, batch, st, accumulate);
  }
}

template <typename S>
void launch_coarse_solve(const helm_plan* P, helm_workspace* ws, const S* c, S* y, int batch, cudaStream_t st) {
  HELM_CHECK(P->dev.coarse_scale != nullptr, "plan was created without a coarse solver");
  const int m0 = P->geo.m0;
  const size_t n0 = (size_t)batch * m0 * m0;
  S* r = (S*)ws->r0;
  // c is only read; y is written last when it aliases c
  S* yy = ((const void*)c == (const void*)y) ? (S*)ws->y0 : y;
  fast_solve<S>(P, ws, c, yy, batch, st);
  for (int it = 0; it < P->desc.refine_steps; ++it) {
    const size_t smem = (size_t)((RSY + 4) * (RSX + 4) + 2 * (RSY + 4) * RSX) * sizeof(S);
    static bool attr = false;
    if (!attr) {
      HELM_CUDA(cudaFuncSetAttribute(a0_residual_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    dim3 blk(32, 8), grd((m0 + RSX - 1) / RSX, (m0 + RSY - 1) / RSY, batch);
    launch_pdl(a0_residual_kernel<S>, grd, blk, smem, st, c, yy, r, (const S*)P->dev.t0_band, (const S*)P->dev.m0_band,
                                                  P->geo.k2, m0);
    HELM_LAUNCH_CHECK();
    fast_solve<S>(P, ws, r, yy, batch, st, /*accumulate=*/true);  // yy += A0~^{-1} r
  }
  if (yy != y) HELM_CUDA(cudaMemcpyAsync(y, yy, n0 * sizeof(S), cudaMemcpyDeviceToDevice, st));
}

template void launch_coarse_solve<double>(const helm_plan*, helm_workspace*, const double*, double*, int,
                                          cudaStream_t);
template void launch_coarse_solve<double2>(const helm_plan*, helm_workspace*, const double2*, double2*, int,
                                           cudaStream_t);

}  // namespace helm
