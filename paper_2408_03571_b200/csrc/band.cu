// Pivoted pentadiagonal solves along y, one per x-mode (part of K5, the Sommerfeld
// coarse solve; algorithm and reference lines in coarse.cu):
//
//   (T0 + s_a M0) X[b][:, a] = in[b][:, a] - sig_a * sum_i corr[y][b*4+i] q[a][i],   out = X (+ add)
//
// `in` may be null (right-hand side = the strip term alone: the strip refinement);
// `add` (may be null) is summed into the backward sweep's stores, read one chunk
// ahead into registers so its latency stays off the recurrence.
// A CTA owns 32 consecutive modes a (lane = mode: the factors and the vectors are
// stored [row][a], so every access is a coalesced 512-byte row segment) and NW*RB
// right-hand sides: warp w carries RB independent recurrences per lane, which gives
// the sequential row recurrence instruction-level parallelism and shares one read of
// the factors among NW*RB right-hand sides.  Factors (int pivot, two multipliers,
// five U entries) and right-hand-side rows stream through shared memory with
// cp.async in chunks of R rows, ST chunks in flight, so HBM latency hides behind
// the FP64 recurrence.  The forward sweep writes the eliminated right-hand side to
// `out`; the backward sweep streams it back with U.
#include <cstdlib>

#include "ops.cuh"

namespace helm {

constexpr int BW = 32;  // modes per CTA

template <int RB, int NW, int R>
struct BandFwdStage {
  double2 L[R][BW][2];
  int piv[R][BW];
  double2 rhs[NW][RB][R][BW];
  double2 corr[NW][RB][R][4];
};
template <int RB, int NW, int R, int UE>
struct BandBwdStage {
  double2 U[R][BW][UE];
  double2 v[NW][RB][R][BW];
};
template <int RB, int NW, int R, int ST>
constexpr size_t band_smem_bytes() {
  return ST * (sizeof(BandFwdStage<RB, NW, R>) > sizeof(BandBwdStage<RB, NW, R, 5>) ? sizeof(BandFwdStage<RB, NW, R>)
                                                                                     : sizeof(BandBwdStage<RB, NW, R, 5>));
}

// NOPIV: no pivot was taken in the factorisation (PlanDev::band_nopiv): pivots are not
// read and U rows are {1/U_jj, U_j,j+1, U_j,j+2} (UE = 3 instead of 5).
// VALS: only the strip values of the solution are wanted (the Woodbury / strip-refinement
// passes): the backward sweep keeps its rows in the stage buffer instead of storing them,
// and each chunk of R = 8 rows is reduced over the CTA's 32 modes with the strip weights
// (lane = (row, quarter of the modes), rotated columns: conflict-free 16-byte reads) into
// part[mode group][row][b*4+i]; `out` is then only the scratch of the eliminated rows.
template <int RB, int NW, int R, int ST, bool NOPIV, bool VALS>
__global__ void __launch_bounds__(BW* NW) band_solve_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                            const int* __restrict__ piv,
                                                            const double2* __restrict__ L,
                                                            const double2* __restrict__ U, int m0, int batch,
                                                            const double2* __restrict__ corr,
                                                            const double* __restrict__ q,
                                                            const double* __restrict__ sig, int ldc,
                                                            const double2* __restrict__ add,
                                                            double2* __restrict__ part) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  const int t = threadIdx.x & (BW - 1), w = threadIdx.x / BW;
  const int a0 = blockIdx.x * BW;
  const int a = a0 + t;
  const bool va = a < m0;
  const int b0 = blockIdx.y * (RB * NW) + w * RB;  // this warp's first right-hand side
  const size_t N0 = (size_t)m0 * m0;
  const int nch = (m0 + R - 1) / R;
  double qa[4] = {0.0, 0.0, 0.0, 0.0};
  double sa = 0.0;
  if (corr && va) {
    for (int i = 0; i < 4; ++i) qa[i] = q[(size_t)a * 4 + i];
    sa = sig[a];
  }
  auto corrected = [&](double2 v, const double2* c4) {
    double2 c = mk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i) c = fma_(qa[i], c4[i], c);
    return sub(v, scale(c, sa));
  };

  // ---------------- forward elimination ----------------
  using FS = BandFwdStage<RB, NW, R>;
  FS* fs = reinterpret_cast<FS*>(sraw);
  auto issue_fwd = [&](int c) {
    FS& S = fs[c % ST];
    // factors: shared by the CTA's warps; warp w copies rows w, w + NW, ... (lane = mode)
    for (int rr = w; rr < R; rr += NW) {
      const int j = c * R + rr;
      const bool ok = va && j < m0;
      const size_t f = fac_idx(j < m0 ? j : 0, va ? a : 0, m0);
      cp_async16(&S.L[rr][t][0], L + 2 * f, ok);
      cp_async16(&S.L[rr][t][1], L + 2 * f + 1, ok);
      if (!NOPIV) cp_async4(&S.piv[rr][t], piv + f, ok);
    }
    // this warp's right-hand-side rows (the forward sweep consumes row j+3 at step j)
    for (int rr = 0; rr < R; ++rr) {
      const int jr = c * R + rr + 3;
      const size_t fr = (size_t)(jr < m0 ? jr : 0) * m0 + (va ? a : 0);
      if (in) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const bool okb = b0 + r < batch;
          cp_async16(&S.rhs[w][r][rr][t], in + (size_t)(okb ? b0 + r : 0) * N0 + fr, va && jr < m0 && okb);
        }
      }
      if (corr && t < 4 * RB) {
        const int r = t >> 2, i = t & 3;
        const bool okb = b0 + r < batch;
        const size_t jc = jr < m0 ? jr : 0;
        cp_async16(&S.corr[w][r][rr][i], corr + jc * ldc + (size_t)(okb ? b0 + r : 0) * 4 + i, jr < m0 && okb);
      }
    }
    cp_commit();
  };
  double2 r0[RB], r1[RB], r2[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int b = b0 + r;
    const bool ok = va && b < batch;
    const double2* col = in ? in + (size_t)(ok ? b : 0) * N0 + (va ? a : 0) : nullptr;
    double2 c4[4];
    double2 v3[3];
    for (int jj = 0; jj < 3; ++jj) {
      double2 v = mk(0.0, 0.0);
      if (ok && jj < m0) {
        if (in) v = col[(size_t)jj * m0];
        if (corr) {
          for (int i = 0; i < 4; ++i) c4[i] = corr[(size_t)jj * ldc + (size_t)b * 4 + i];
          v = corrected(v, c4);
        }
      }
      v3[jj] = v;
    }
    r0[r] = v3[0];
    r1[r] = v3[1];
    r2[r] = v3[2];
  }
  for (int c = 0; c < ST - 1; ++c) {
    if (c < nch) issue_fwd(c);
    else cp_commit();
  }
  for (int c = 0; c < nch; ++c) {
    cp_wait<ST - 2>();
    __syncthreads();
    if (c + ST - 1 < nch) issue_fwd(c + ST - 1);
    else cp_commit();
    const FS& S = fs[c % ST];
    const int rows = min(R, m0 - c * R);
    for (int rr = 0; rr < rows; ++rr) {
      const int j = c * R + rr;
      const int pv = NOPIV ? 0 : S.piv[rr][t];
      const double2 l0 = S.L[rr][t][0], l1 = S.L[rr][t][1];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double2 x0 = r0[r], x1 = r1[r], x2 = r2[r];
        if (pv == 1) { const double2 tmp = x0; x0 = x1; x1 = tmp; }
        else if (pv == 2) { const double2 tmp = x0; x0 = x2; x2 = tmp; }
        x1 = fms_(l0, x0, x1);
        x2 = fms_(l1, x0, x2);
        if (va && b0 + r < batch) out[(size_t)(b0 + r) * N0 + (size_t)j * m0 + a] = x0;
        double2 nx = in ? S.rhs[w][r][rr][t] : mk(0.0, 0.0);
        if (corr) nx = corrected(nx, S.corr[w][r][rr]);
        r0[r] = x1;
        r1[r] = x2;
        r2[r] = nx;
      }
    }
  }
  cp_wait<0>();
  __syncthreads();
  __threadfence();  // the backward sweep re-reads `out` through cp.async

  // ---------------- backward substitution ----------------
  constexpr int UE = NOPIV ? 3 : 5;
  using BS = BandBwdStage<RB, NW, R, UE>;
  BS* bs = reinterpret_cast<BS*>(sraw);
  auto issue_bwd = [&](int c) {
    BS& S = bs[c % ST];
    for (int rr = w; rr < R; rr += NW) {
      const int j = m0 - 1 - (c * R + rr);
      const bool ok = va && j >= 0;
      const double2* u = U + UE * fac_idx(j >= 0 ? j : 0, va ? a : 0, m0);
#pragma unroll
      for (int e = 0; e < UE; ++e) cp_async16(&S.U[rr][t][e], u + e, ok);
    }
    for (int rr = 0; rr < R; ++rr) {
      const int j = m0 - 1 - (c * R + rr);
      const size_t f = (size_t)(j >= 0 ? j : 0) * m0 + (va ? a : 0);
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const bool okb = b0 + r < batch;
        cp_async16(&S.v[w][r][rr][t], out + (size_t)(okb ? b0 + r : 0) * N0 + f, va && j >= 0 && okb);
      }
    }
    cp_commit();
  };
  for (int c = 0; c < ST - 1; ++c) {
    if (c < nch) issue_bwd(c);
    else cp_commit();
  }
  double2 y1[RB], y2[RB], y3[RB], y4[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) y1[r] = y2[r] = y3[r] = y4[r] = mk(0.0, 0.0);
  // VALS: this lane reduces row (t >> 2) of a chunk over the 8 modes p*8 + vcol(i), p = t & 3
  const int vrow = t >> 2, vp = t & 3;
  auto vcol = [&](int i) { return vp * 8 + ((i + vp + 4 * (vrow & 1)) & 7); };
  double qc[VALS ? 8 : 1][4];
  if constexpr (VALS) {
    static_assert(R == 8 && BW == 32, "the strip-value reduction maps a lane to (row of 8, quarter of 32 modes)");
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int ac = a0 + vcol(i);
#pragma unroll
      for (int k = 0; k < 4; ++k) qc[i][k] = ac < m0 ? q[(size_t)ac * 4 + k] : 0.0;
    }
  }
  double2 acur[RB][R], anxt[RB][R];
  auto load_add = [&](int c, double2 (&dst)[RB][R]) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int j = m0 - 1 - (c * R + rr);
#pragma unroll
      for (int r = 0; r < RB; ++r)
        dst[r][rr] = (va && j >= 0 && b0 + r < batch) ? __ldg(add + (size_t)(b0 + r) * N0 + (size_t)j * m0 + a)
                                                       : mk(0.0, 0.0);
    }
  };
  if (add) load_add(0, acur);
  for (int c = 0; c < nch; ++c) {
    cp_wait<ST - 2>();
    __syncthreads();
    if (c + ST - 1 < nch) issue_bwd(c + ST - 1);
    else cp_commit();
    if (add && c + 1 < nch) load_add(c + 1, anxt);
    BS& S = bs[c % ST];
    const int rows = min(R, m0 - c * R);
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      if (rr >= rows) break;
      const int j = m0 - 1 - (c * R + rr);
      const double2 u0 = S.U[rr][t][0], u1 = S.U[rr][t][1], u2 = S.U[rr][t][2];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double2 v = S.v[w][r][rr][t];
        v = fms_(u1, y1[r], v);
        v = fms_(u2, y2[r], v);
        if constexpr (!NOPIV) {
          v = fms_(S.U[rr][t][UE - 2], y3[r], v);
          v = fms_(S.U[rr][t][UE - 1], y4[r], v);
        }
        v = mul(v, u0);
        if constexpr (VALS)
          S.v[w][r][rr][t] = v;  // the slot just read; the stage is re-issued after the next barrier
        else if (va && b0 + r < batch)
          out[(size_t)(b0 + r) * N0 + (size_t)j * m0 + a] = add ? ::helm::add(v, acur[r][rr]) : v;
        y4[r] = y3[r];
        y3[r] = y2[r];
        y2[r] = y1[r];
        y1[r] = v;
      }
    }
    if (add) {
#pragma unroll
      for (int rr = 0; rr < R; ++rr)
#pragma unroll
        for (int r = 0; r < RB; ++r) acur[r][rr] = anxt[r][rr];
    }
    if constexpr (VALS) {
      __syncwarp();
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double2 acc[4] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 x = S.v[w][r][vrow][vcol(i)];
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] = fma_(qc[i][k], x, acc[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // quarters in the fixed order (p ^ 1) then (p ^ 2)
          acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 1);
          acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 1);
          acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, 2);
          acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, 2);
        }
        if (vp == 0 && vrow < rows && b0 + r < batch) {
          const int j = m0 - 1 - (c * R + vrow);
          double2* o = part + ((size_t)blockIdx.x * m0 + j) * ldc + (size_t)(b0 + r) * 4;
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = acc[k];
        }
      }
      __syncwarp();
    }
  }
  cp_wait<0>();
}

// Z[e] = (Zadd ? Zadd[e] : 0) + sum_g part[g][e]   (mode groups in order: deterministic)
__global__ void __launch_bounds__(256) strip_part_sum_kernel(const double2* __restrict__ part,
                                                             const double2* __restrict__ Zadd,
                                                             double2* __restrict__ Z, size_t n, int groups) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double2 s = Zadd ? Zadd[e] : mk(0.0, 0.0);
  for (int g = 0; g < groups; ++g) s = ::helm::add(s, part[(size_t)g * n + e]);
  Z[e] = s;
}

template <int RB, int NW, int R, int ST, bool NOPIV, bool VALS = false>
static void band_launch_k(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                          cudaStream_t st, const double2* add, double2* part = nullptr) {
  const PlanDev& d = P->dev;
  constexpr size_t smem = band_smem_bytes<RB, NW, R, ST>();
  static_assert(smem <= 227 * 1024, "band-solve stages exceed shared memory");
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(band_solve_kernel<RB, NW, R, ST, NOPIV, VALS>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  dim3 grd((d.m0 + BW - 1) / BW, (batch + RB * NW - 1) / (RB * NW));
  launch_pdl(band_solve_kernel<RB, NW, R, ST, NOPIV, VALS>, grd, BW * NW, smem, st, in, out, d.band_piv,
             (const double2*)d.band_l, (const double2*)d.band_u, d.m0, batch, corr, d.strip_q, d.coarse_scale,
             batch * 4, add, part);
  HELM_LAUNCH_CHECK();
}

template <int RB, int NW, int R, int ST>
static void band_launch(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                        cudaStream_t st, const double2* add) {
  if (P->dev.band_nopiv)
    band_launch_k<RB, NW, R, ST, true>(P, in, out, corr, batch, st, add);
  else
    band_launch_k<RB, NW, R, ST, false>(P, in, out, corr, batch, st, add);
}

// batches up to this size use the segmented solve (HELM_BAND_SEG_MAX overrides; 0 disables)
static int band_seg_max_batch() {
  static int v = [] {
    const char* e = std::getenv("HELM_BAND_SEG_MAX");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}

// Strip values only: Z = (Zadd) + S X for the same system (S = the strip weights strip_q);
// `scratch` [batch][N0] holds the eliminated rows, `part` ceil(m0/32) * m0 * batch * 4 partial sums.
bool band_vals_usable(const helm_plan* P, int batch) {
  return !(batch <= band_seg_max_batch() && P->dev.band_seg) && batch > 4;
}
void launch_band_vals(const helm_plan* P, const double2* in, double2* scratch, const double2* corr, int batch,
                      cudaStream_t st, double2* part, const double2* Zadd, double2* Z) {
  HELM_CHECK(band_vals_usable(P, batch), "band solve: strip-value pass needs the streaming kernel (batch > 4)");
  HELM_CHECK((const void*)in != (const void*)scratch, "band solve: input and scratch must not alias");
  HELM_CHECK(in != nullptr || corr != nullptr, "band solve: no right-hand side");
  if (band_tma_usable(P))
    band_tma_launch(P, in, scratch, corr, batch, st, nullptr, part);
  else if (P->dev.band_nopiv)
    band_launch_k<1, 8, 8, 3, true, true>(P, in, scratch, corr, batch, st, nullptr, part);
  else
    band_launch_k<1, 8, 8, 3, false, true>(P, in, scratch, corr, batch, st, nullptr, part);
  const size_t n = (size_t)P->dev.m0 * batch * 4;
  launch_pdl(strip_part_sum_kernel, (unsigned)((n + 255) / 256), 256, 0, st, (const double2*)part, Zadd, Z, n,
             (P->dev.m0 + BW - 1) / BW);
  HELM_LAUNCH_CHECK();
}

void launch_band_solve(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                       cudaStream_t st, const double2* add) {
  HELM_CHECK(P->dev.band_piv != nullptr, "plan has no band factors");
  HELM_CHECK((const void*)in != (const void*)out && (const void*)add != (const void*)out,
             "band solve: input and output must not alias");
  HELM_CHECK(in != nullptr || corr != nullptr, "band solve: no right-hand side");
  if (batch <= band_seg_max_batch() && P->dev.band_seg)
    band_seg_launch(P, in, out, corr, batch, st, add);  // segmented recurrence: latency-bound regime
  else if (batch == 1)
    band_launch<1, 1, 8, 4>(P, in, out, corr, batch, st, add);  // latency-bound recurrence
  else if (batch <= 4)
    band_launch<2, 2, 8, 3>(P, in, out, corr, batch, st, add);
  else if (band_tma_usable(P))
    band_tma_launch(P, in, out, corr, batch, st, add, nullptr);  // the same CTA shape, TMA-staged (band_tma.cu)
  else  // 8 warps (8 right-hand sides) share each factor read; 4-16 per CTA and 4-8 rows per
        // stage were measured slower
    band_launch<1, 8, 8, 3>(P, in, out, corr, batch, st, add);
}

}  // namespace helm
