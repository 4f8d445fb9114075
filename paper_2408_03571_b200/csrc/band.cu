// Pivoted pentadiagonal solves along y, one per x-mode (part of K5, the Sommerfeld
// coarse solve; algorithm and reference lines in coarse.cu):
//
//   (T0 + s_a M0) out[b][:, a] = in[b][:, a] - sig_a * sum_i corr[y][b*4+i] q[a][i]
//
// One warp owns 32 consecutive modes a (coalesced: the factors and vectors are
// stored [row][a]) and RB right-hand sides.  The recurrence is sequential in the
// row index, so the factors (int pivot, two multipliers, five U entries) and the
// right-hand-side rows are streamed into shared memory with cp.async in chunks of
// BR rows, BST chunks in flight, which hides the HBM latency behind the FP64
// recurrence instead of exposing it once per row.  The forward sweep writes the
// eliminated right-hand side to `out`; the backward sweep streams it back with U.
#include "ops.cuh"

namespace helm {

constexpr int BW = 32;   // modes per CTA (one warp)
constexpr int BR = 8;    // rows per chunk
constexpr int BST = 3;   // chunks in flight

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;  // src-size 0: zero fill, nothing read
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int RB>
struct BandFwdStage {
  double2 L[BR][BW][2];
  int piv[BR][BW];
  double2 rhs[RB][BR][BW];
  double2 corr[RB][BR][4];
};
template <int RB>
struct BandBwdStage {
  double2 U[BR][BW][5];
  double2 v[RB][BR][BW];
};
template <int RB>
constexpr size_t band_smem_bytes() {
  return BST * (sizeof(BandFwdStage<RB>) > sizeof(BandBwdStage<RB>) ? sizeof(BandFwdStage<RB>)
                                                                      : sizeof(BandBwdStage<RB>));
}

template <int RB>
__global__ void __launch_bounds__(BW) band_solve_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                        const int* __restrict__ piv, const double2* __restrict__ L,
                                                        const double2* __restrict__ U, int m0, int batch,
                                                        const double2* __restrict__ corr,
                                                        const double* __restrict__ q,
                                                        const double* __restrict__ sig, int ldc) {
  extern __shared__ __align__(16) unsigned char sraw[];
  const int t = threadIdx.x;
  const int a = blockIdx.x * BW + t;
  const bool va = a < m0;
  const int ac = va ? a : m0 - 1;  // clamped (valid) address for predicated-off copies
  const int b0 = blockIdx.y * RB;
  const size_t N0 = (size_t)m0 * m0;
  const int nch = (m0 + BR - 1) / BR;
  double qa[4] = {0.0, 0.0, 0.0, 0.0};
  double sa = 0.0;
  if (corr && va) {
    for (int i = 0; i < 4; ++i) qa[i] = q[(size_t)a * 4 + i];
    sa = sig[a];
  }

  // ---------------- forward elimination ----------------
  BandFwdStage<RB>* fs = reinterpret_cast<BandFwdStage<RB>*>(sraw);
  auto issue_fwd = [&](int c) {
    BandFwdStage<RB>& S = fs[c % BST];
    for (int rr = 0; rr < BR; ++rr) {
      const int j = c * BR + rr;
      const bool vj = va && j < m0;
      const size_t f = (size_t)(j < m0 ? j : m0 - 1) * m0 + ac;
      cp_async16(&S.L[rr][t][0], L + 2 * f, vj);
      cp_async16(&S.L[rr][t][1], L + 2 * f + 1, vj);
      cp_async4(&S.piv[rr][t], piv + f, vj);
      const int jr = j + 3;  // the forward sweep consumes right-hand-side row j+3 at step j
      const size_t fr = (size_t)(jr < m0 ? jr : m0 - 1) * m0 + ac;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int b = b0 + r < batch ? b0 + r : batch - 1;
        cp_async16(&S.rhs[r][rr][t], in + (size_t)b * N0 + fr, va && jr < m0 && b0 + r < batch);
      }
      if (corr && t < 4 * RB) {
        const int r = t >> 2, i = t & 3;
        const int b = b0 + r < batch ? b0 + r : batch - 1;
        const size_t jc = jr < m0 ? jr : m0 - 1;
        cp_async16(&S.corr[r][rr][i], corr + jc * ldc + (size_t)b * 4 + i, jr < m0 && b0 + r < batch);
      }
    }
    cp_commit();
  };
  auto corrected = [&](double2 v, const double2* c4) {
    double2 c = mk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i) c = fma_(qa[i], c4[i], c);
    return sub(v, scale(c, sa));
  };
  double2 r0[RB], r1[RB], r2[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int b = b0 + r;
    const bool ok = va && b < batch;
    const double2* col = in + (size_t)(ok ? b : 0) * N0 + ac;
    double2 c4[4];
    for (int jj = 0; jj < 3; ++jj) {
      double2 v = mk(0.0, 0.0);
      if (ok && jj < m0) {
        v = col[(size_t)jj * m0];
        if (corr) {
          for (int i = 0; i < 4; ++i) c4[i] = corr[(size_t)jj * ldc + (size_t)b * 4 + i];
          v = corrected(v, c4);
        }
      }
      (jj == 0 ? r0[r] : jj == 1 ? r1[r] : r2[r]) = v;
    }
  }
  for (int c = 0; c < BST - 1; ++c) {
    if (c < nch) issue_fwd(c);
    else cp_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_wait<BST - 2>();
    __syncwarp();
    if (c + BST - 1 < nch) issue_fwd(c + BST - 1);
    else cp_commit();
    const BandFwdStage<RB>& S = fs[c % BST];
    for (int rr = 0; rr < BR; ++rr) {
      const int j = c * BR + rr;
      if (j >= m0) break;
      const int pv = S.piv[rr][t];
      const double2 l0 = S.L[rr][t][0], l1 = S.L[rr][t][1];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double2 x0 = r0[r], x1 = r1[r], x2 = r2[r];
        if (pv == 1) { const double2 tmp = x0; x0 = x1; x1 = tmp; }
        else if (pv == 2) { const double2 tmp = x0; x0 = x2; x2 = tmp; }
        x1 = fms_(l0, x0, x1);
        x2 = fms_(l1, x0, x2);
        if (va && b0 + r < batch) out[(size_t)(b0 + r) * N0 + (size_t)j * m0 + a] = x0;
        double2 nx = S.rhs[r][rr][t];
        if (corr) nx = corrected(nx, S.corr[r][rr]);
        r0[r] = x1;
        r1[r] = x2;
        r2[r] = nx;
      }
    }
  }
  cp_wait<0>();
  __syncwarp();
  __threadfence();  // the backward sweep re-reads `out` through cp.async

  // ---------------- backward substitution ----------------
  BandBwdStage<RB>* bs = reinterpret_cast<BandBwdStage<RB>*>(sraw);
  auto issue_bwd = [&](int c) {
    BandBwdStage<RB>& S = bs[c % BST];
    for (int rr = 0; rr < BR; ++rr) {
      const int j = m0 - 1 - (c * BR + rr);
      const bool vj = va && j >= 0;
      const size_t f = (size_t)(j >= 0 ? j : 0) * m0 + ac;
#pragma unroll
      for (int e = 0; e < 5; ++e) cp_async16(&S.U[rr][t][e], U + 5 * f + e, vj);
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int b = b0 + r < batch ? b0 + r : batch - 1;
        cp_async16(&S.v[r][rr][t], out + (size_t)b * N0 + f, vj && b0 + r < batch);
      }
    }
    cp_commit();
  };
  for (int c = 0; c < BST - 1; ++c) {
    if (c < nch) issue_bwd(c);
    else cp_commit();
  }
  double2 y1[RB], y2[RB], y3[RB], y4[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) y1[r] = y2[r] = y3[r] = y4[r] = mk(0.0, 0.0);
  for (int c = 0; c < nch; ++c) {
    cp_wait<BST - 2>();
    __syncwarp();
    if (c + BST - 1 < nch) issue_bwd(c + BST - 1);
    else cp_commit();
    const BandBwdStage<RB>& S = bs[c % BST];
    for (int rr = 0; rr < BR; ++rr) {
      const int j = m0 - 1 - (c * BR + rr);
      if (j < 0) break;
      const double2 u0 = S.U[rr][t][0], u1 = S.U[rr][t][1], u2 = S.U[rr][t][2], u3 = S.U[rr][t][3],
                    u4 = S.U[rr][t][4];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double2 v = S.v[r][rr][t];
        v = fms_(u1, y1[r], v);
        v = fms_(u2, y2[r], v);
        v = fms_(u3, y3[r], v);
        v = fms_(u4, y4[r], v);
        v = mul(v, u0);
        if (va && b0 + r < batch) out[(size_t)(b0 + r) * N0 + (size_t)j * m0 + a] = v;
        y4[r] = y3[r];
        y3[r] = y2[r];
        y2[r] = y1[r];
        y1[r] = v;
      }
    }
  }
  cp_wait<0>();
}

template <int RB>
static void band_launch(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                        cudaStream_t st) {
  const PlanDev& d = P->dev;
  constexpr size_t smem = band_smem_bytes<RB>();
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(band_solve_kernel<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grd((d.m0 + BW - 1) / BW, (batch + RB - 1) / RB);
  band_solve_kernel<RB><<<grd, BW, smem, st>>>(in, out, d.band_piv, (const double2*)d.band_l,
                                               (const double2*)d.band_u, d.m0, batch, corr, d.strip_q,
                                               d.coarse_scale, batch * 4);
  HELM_LAUNCH_CHECK();
}

void launch_band_solve(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                       cudaStream_t st) {
  HELM_CHECK(P->dev.band_piv != nullptr, "plan has no band factors");
  HELM_CHECK((const void*)in != (const void*)out, "band solve: input and output must not alias");
  if (batch == 1)
    band_launch<1>(P, in, out, corr, batch, st);
  else if (batch == 2)
    band_launch<2>(P, in, out, corr, batch, st);
  else
    band_launch<4>(P, in, out, corr, batch, st);
}

}  // namespace helm
