// Segmented band solves for small batches (part of K5, the Sommerfeld coarse solve;
// the recurrence and its factors are described in band.cu).
//
// band.cu runs each mode's 2*m0-step row recurrence (forward elimination with the
// pivoted L, backward substitution with U) on one lane: at batch 1 that is 33 warps on
// the whole GPU, each waiting on ~2000 dependent steps (0.38 ms per solve at m0=1025).
// Here the m0 rows of a mode are cut into SEG segments and the recurrence is solved as
// a linear recurrence with a carried state:
//
//   forward  state (r0, r1) (the two pending eliminated rows):  s_out = Phi_k s_in + p_k
//   backward state (x[j+1..j+4]) (the last four solution rows): t_out = Psi_k t_in + q_k
//
// Phi_k (2x2) and Psi_k (4x4) depend on the factors only; they are computed once per plan
// (band_seg_setup_kernel).  Per solve, every (mode, segment) thread
//   F1  runs its segment's forward recurrence from a zero state  -> p_k
//   --  the segments are chained:  s_{k+1} = Phi_k s_k + p_k  (a warp-level affine scan per mode)
//   F3  re-runs the segment from its true state, keeping the eliminated rows in shared memory
//   B1  runs the backward recurrence over those rows from a zero state -> q_k
//   --  chained downwards:  t_{k-1} = Psi_k t_k + q_k  (suffix scan)
//   B3  re-runs from the true state and writes x (+ add).
// Exact in exact arithmetic (the same linear recurrence, associated differently); 1025-row
// modes become 32-row segments, so the dependent chain is ~130 steps instead of ~2050.
// Right-hand side handling (in, corr/q/sig, add) is the same contract as band_solve_kernel.
#include <cstdlib>
#include <type_traits>

#include "ops.cuh"

namespace helm {

constexpr int SEG = 32;  // segments per mode
// modes per CTA: SMB consecutive modes, SEG * SMB threads (one warp per mode in the scans).
// 8 (129 CTAs at m0 = 1025); 4 modes per CTA (257 CTAs over all 148 SMs) was measured
// slower at batch 1 (0.313 vs 0.303 ms per coarse solve).
constexpr int SMB = 8;


struct SegRhs {
  const double2* in;
  const double2* corr;
  int ldc;
  int b;
  double qa[4];
  double sa;
  size_t col;  // b * N0 + a
  int m0;
  __device__ __forceinline__ double2 operator()(int y) const {
    if (y >= m0) return mk(0.0, 0.0);
    double2 v = in ? __ldg(in + col + (size_t)y * m0) : mk(0.0, 0.0);
    if (corr) {
      const double2* c4 = corr + (size_t)y * ldc + (size_t)b * 4;
      double2 c = mk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < 4; ++i) c = fma_(qa[i], __ldg(c4 + i), c);
      v = sub(v, scale(c, sa));
    }
    return v;
  }
};

__device__ __forceinline__ double2 shfl_up_c(double2 v, int d) {
  return mk(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ double2 shfl_dn_c(double2 v, int d) {
  return mk(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}

__device__ __forceinline__ void fwd_step(int pv, double2 l0, double2 l1, double2& r0, double2& r1, double2 f,
                                         double2& out) {
  double2 x0 = r0, x1 = r1, x2 = f;
  if (pv == 1) {
    const double2 t = x0; x0 = x1; x1 = t;
  } else if (pv == 2) {
    const double2 t = x0; x0 = x2; x2 = t;
  }
  x1 = fms_(l0, x0, x1);
  x2 = fms_(l1, x0, x2);
  out = x0;
  r0 = x1;
  r1 = x2;
}

// forward pass over rows [j0, j1) with state (r0, r1); writes eliminated rows to sm (if non-null).
// NOPIV: no pivot was taken in the factorisation (pivots not read, U rows of 3 entries).
template <bool STORE, bool NOPIV, int CF = 4>
__device__ __forceinline__ void fwd_run(const SegRhs& rhs, const int* __restrict__ piv, const double2* __restrict__ L,
                                        int m0, int a, int j0, int j1, double2& r0, double2& r1, double2* sm,
                                        int sm_stride) {
  // chunks of C rows, the next chunk's loads in flight while the current one is consumed
  constexpr int C = CF;
  struct Chunk {
    int pv[C];
    double2 l0[C], l1[C], f[C];
  };
  auto load = [&](int j, Chunk& ch) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const bool ok = j + c < j1;
      const size_t e = fac_idx(ok ? j + c : j0, a, m0);
      ch.pv[c] = NOPIV ? 0 : __ldg(piv + e);
      ch.l0[c] = __ldg(L + 2 * e);
      ch.l1[c] = __ldg(L + 2 * e + 1);
      ch.f[c] = ok ? rhs(j + c + 2) : mk(0.0, 0.0);
    }
  };
  if (j0 >= j1) return;
  Chunk cur, nxt;
  load(j0, cur);
  for (int j = j0; j < j1; j += C) {
    if (j + C < j1) load(j + C, nxt);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (j + c < j1) {
        double2 o;
        fwd_step(cur.pv[c], cur.l0[c], cur.l1[c], r0, r1, cur.f[c], o);
        if (STORE) sm[(j + c - j0) * sm_stride] = o;
      }
    }
    cur = nxt;
  }
}

// backward pass over rows [j0, j1) (descending) with state y; sm: eliminated rows (null:
// zero); with out != null every solution row is stored (+ add[row] when add != null).  U and
// the summands of the next chunk are in flight while the current chunk is consumed.
template <bool NOPIV, int CB = 4>
__device__ __forceinline__ void bwd_run(const double2* __restrict__ U, int m0, int a, int j0, int j1,
                                        double2 (&y)[4], const double2* sm, int sm_stride,
                                        double2* __restrict__ out = nullptr,
                                        const double2* __restrict__ addp = nullptr, bool store = false) {
  constexpr int C = CB, UE = NOPIV ? 3 : 5;
  struct Chunk {
    double2 u[C][UE];
    double2 ad[C];
  };
  auto load = [&](int j, Chunk& ch) {  // rows j, j-1, .., j-C+1
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int r = j - c >= j0 ? j - c : j1 - 1;
      const double2* u = U + UE * fac_idx(r, a, m0);
#pragma unroll
      for (int e = 0; e < UE; ++e) ch.u[c][e] = __ldg(u + e);
      ch.ad[c] = addp ? __ldg(addp + (size_t)r * m0) : mk(0.0, 0.0);
    }
  };
  if (j0 >= j1) return;
  Chunk cur, nxt;
  load(j1 - 1, cur);
  for (int j = j1 - 1; j >= j0; j -= C) {
    if (j - C >= j0) load(j - C, nxt);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int r = j - c;
      if (r >= j0) {
        double2 v = sm ? sm[(r - j0) * sm_stride] : mk(0.0, 0.0);
        v = fms_(cur.u[c][1], y[0], v);
        v = fms_(cur.u[c][2], y[1], v);
        if constexpr (!NOPIV) {
          v = fms_(cur.u[c][UE - 2], y[2], v);
          v = fms_(cur.u[c][UE - 1], y[3], v);
        }
        v = mul(v, cur.u[c][0]);
        y[3] = y[2];
        y[2] = y[1];
        y[1] = y[0];
        y[0] = v;
        if (out && store) out[(size_t)r * m0] = addp ? add(v, cur.ad[c]) : v;
      }
    }
    cur = nxt;
  }
}

// Phi [SEG][4][m0], Psi [SEG][16][m0]: exit state of segment k for unit entry states
template <bool NOPIV>
__global__ void band_seg_setup_kernel(const int* __restrict__ piv, const double2* __restrict__ L,
                                      const double2* __restrict__ U, int m0, int ls, double2* __restrict__ phi,
                                      double2* __restrict__ psi) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (a >= m0) return;
  const int j0 = min(k * ls, m0), j1 = min(j0 + ls, m0);
  SegRhs zero{nullptr, nullptr, 0, 0, {0, 0, 0, 0}, 0.0, 0, m0};
  for (int c = 0; c < 2; ++c) {
    double2 r0 = mk(c == 0 ? 1.0 : 0.0, 0.0), r1 = mk(c == 1 ? 1.0 : 0.0, 0.0);
    fwd_run<false, NOPIV>(zero, piv, L, m0, a, j0, j1, r0, r1, nullptr, 0);
    phi[((size_t)k * 4 + 0 * 2 + c) * m0 + a] = r0;
    phi[((size_t)k * 4 + 1 * 2 + c) * m0 + a] = r1;
  }
  for (int c = 0; c < 4; ++c) {
    double2 y[4];
    for (int i = 0; i < 4; ++i) y[i] = mk(i == c ? 1.0 : 0.0, 0.0);
    bwd_run<NOPIV>(U, m0, a, j0, j1, y, nullptr, 0);
    for (int r = 0; r < 4; ++r) psi[((size_t)k * 16 + r * 4 + c) * m0 + a] = y[r];
  }
}

// CF / CB: rows per prefetch chunk of the forward / backward sweeps (the next chunk's
// loads are in flight while the current one is consumed)
template <bool NOPIV, int CF, int CB, int SMB>
__global__ void __launch_bounds__(SEG * SMB) band_seg_kernel(
    const double2* __restrict__ in, double2* __restrict__ out, const int* __restrict__ piv,
    const double2* __restrict__ L, const double2* __restrict__ U, const double2* __restrict__ phi,
    const double2* __restrict__ psi, int m0, int ls, const double2* __restrict__ corr, const double* __restrict__ q,
    const double* __restrict__ sig, int ldc, const double2* __restrict__ addv) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  double2* rows = reinterpret_cast<double2*>(sraw);  // [ls][SEG][SMB] eliminated rows
  __shared__ double2 fst[SEG + 1][SMB][2];           // forward states at segment starts
  __shared__ double2 bst[SEG + 2][SMB][4];           // backward states (exit of kk at kk+1 after the scan)
  const int al = threadIdx.x % SMB, k = threadIdx.x / SMB;
  const int a = blockIdx.x * SMB + al;
  const int b = blockIdx.y;
  const bool va = a < m0;
  const size_t N0 = (size_t)m0 * m0;
  const int j0 = min(k * ls, m0), j1 = min(j0 + ls, m0);
  SegRhs rhs{in, corr, ldc, b, {0, 0, 0, 0}, 0.0, (size_t)b * N0 + (va ? a : 0), m0};
  if (corr && va) {
#pragma unroll
    for (int i = 0; i < 4; ++i) rhs.qa[i] = __ldg(q + (size_t)a * 4 + i);
    rhs.sa = __ldg(sig + a);
  }
  const int ac = va ? a : 0;
  const int sstride = SEG * SMB;
  double2* mysm = rows + k * SMB + al;

  // F1: zero-state forward pass (segment 0 starts from the true rows 0, 1)
  double2 r0 = mk(0.0, 0.0), r1 = mk(0.0, 0.0);
  if (k == 0) {
    r0 = rhs(0);
    r1 = rhs(1);
  }
  fwd_run<false, NOPIV, CF>(rhs, piv, L, m0, ac, j0, j1, r0, r1, nullptr, 0);
  fst[k + 1][al][0] = r0;
  fst[k + 1][al][1] = r1;
  __syncthreads();
  // chain: s_{k+1} = Phi_k s_k + p_k (s_1 = p_0) as an inclusive affine scan over the
  // segments: warp w takes mode w, lane kk segment kk; f_kk(s) = Phi_kk s + p_kk with
  // f_0 = p_0 (Phi_0 = 0), composed in log2(SEG) shuffle steps
  {
    const int w = threadIdx.x >> 5, kk = threadIdx.x & 31;
    const int aw = blockIdx.x * SMB + w;
    double2 F[4], pv[2];
    pv[0] = fst[kk + 1][w][0];
    pv[1] = fst[kk + 1][w][1];
#pragma unroll
    for (int e = 0; e < 4; ++e) F[e] = (kk > 0 && aw < m0) ? __ldg(phi + ((size_t)kk * 4 + e) * m0 + aw) : mk(0.0, 0.0);
#pragma unroll
    for (int d = 1; d < SEG; d <<= 1) {
      double2 Fo[4], po[2];
#pragma unroll
      for (int e = 0; e < 4; ++e) Fo[e] = shfl_up_c(F[e], d);
      po[0] = shfl_up_c(pv[0], d);
      po[1] = shfl_up_c(pv[1], d);
      if (kk >= d) {  // (mine) o (theirs): F <- F Fo, p <- F po + p
        const double2 n0 = add(pv[0], add(mul(F[0], po[0]), mul(F[1], po[1])));
        const double2 n1 = add(pv[1], add(mul(F[2], po[0]), mul(F[3], po[1])));
        const double2 G0 = add(mul(F[0], Fo[0]), mul(F[1], Fo[2])), G1 = add(mul(F[0], Fo[1]), mul(F[1], Fo[3]));
        const double2 G2 = add(mul(F[2], Fo[0]), mul(F[3], Fo[2])), G3 = add(mul(F[2], Fo[1]), mul(F[3], Fo[3]));
        F[0] = G0; F[1] = G1; F[2] = G2; F[3] = G3;
        pv[0] = n0;
        pv[1] = n1;
      }
    }
    __syncthreads();  // every lane has read its p before the entry states overwrite fst
    // entry state of segment kk+1 = exit of kk
    fst[kk + 1][w][0] = pv[0];
    fst[kk + 1][w][1] = pv[1];
  }
  __syncthreads();
  // F3: true forward pass, eliminated rows kept in shared memory
  if (k == 0) {
    r0 = rhs(0);
    r1 = rhs(1);
  } else {
    r0 = fst[k][al][0];
    r1 = fst[k][al][1];
  }
  fwd_run<true, NOPIV, CF>(rhs, piv, L, m0, ac, j0, j1, r0, r1, mysm, sstride);
  // B1: zero-state backward pass
  double2 y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] = mk(0.0, 0.0);
  bwd_run<NOPIV, CB>(U, m0, ac, j0, j1, y, mysm, sstride);
#pragma unroll
  for (int i = 0; i < 4; ++i) bst[k][al][i] = y[i];
  __syncthreads();
  // chain downwards: exit_kk = Psi_kk entry_kk + q_kk with entry_kk = exit_{kk+1} and a
  // zero entry at the top, as a suffix affine scan (lane kk composes with lane kk + d)
  {
    const int w = threadIdx.x >> 5, kk = threadIdx.x & 31;
    const int aw = blockIdx.x * SMB + w;
    double2 Q[16], qv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) qv[i] = bst[kk][w][i];
#pragma unroll
    for (int e = 0; e < 16; ++e)
      Q[e] = (kk < SEG - 1 && aw < m0) ? __ldg(psi + ((size_t)kk * 16 + e) * m0 + aw) : mk(0.0, 0.0);
#pragma unroll
    for (int d = 1; d < SEG; d <<= 1) {
      double2 Qo[16], qo[4];
#pragma unroll
      for (int e = 0; e < 16; ++e) Qo[e] = shfl_dn_c(Q[e], d);
#pragma unroll
      for (int i = 0; i < 4; ++i) qo[i] = shfl_dn_c(qv[i], d);
      if (kk + d < SEG) {  // (mine) o (theirs): Q <- Q Qo, q <- Q qo + q
        double2 nq[4], NQ[16];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          double2 t = qv[r];
#pragma unroll
          for (int c = 0; c < 4; ++c) t = fma_(Q[r * 4 + c], qo[c], t);
          nq[r] = t;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double2 m = mk(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < 4; ++i) m = fma_(Q[r * 4 + i], Qo[i * 4 + c], m);
            NQ[r * 4 + c] = m;
          }
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) Q[e] = NQ[e];
#pragma unroll
        for (int i = 0; i < 4; ++i) qv[i] = nq[i];
      }
    }
    __syncthreads();
    // entry state of segment kk = exit of kk+1: stored one slot up (bst[kk+1] = exit_kk)
#pragma unroll
    for (int i = 0; i < 4; ++i) bst[kk + 1][w][i] = qv[i];
  }
  __syncthreads();
  // B3: true backward pass
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] = k == SEG - 1 ? mk(0.0, 0.0) : bst[k + 2][al][i];
  bwd_run<NOPIV, CB>(U, m0, ac, j0, j1, y, mysm, sstride, out + (size_t)b * N0 + ac,
          addv ? addv + (size_t)b * N0 + ac : nullptr, va);
}

static int seg_len(int m0) { return (m0 + SEG - 1) / SEG; }

size_t band_seg_table_elems(int m0) { return (size_t)SEG * 20 * m0; }

bool band_seg_usable(int m0) { return m0 >= 4 * SEG && seg_len(m0) <= 48; }

void band_seg_setup(const PlanDev& d, double2* tables, cudaStream_t st) {
  const int m0 = d.m0;
  double2* phi = tables;
  double2* psi = tables + (size_t)SEG * 4 * m0;
  auto go = [&](auto np) {
    launch_pdl(band_seg_setup_kernel<decltype(np)::value>, dim3((m0 + 127) / 128, SEG), 128, 0, st, d.band_piv, (const double2*)d.band_l, (const double2*)d.band_u, m0, seg_len(m0), phi, psi);
  };
  if (d.band_nopiv) go(std::true_type{});
  else go(std::false_type{});
  HELM_LAUNCH_CHECK();
}

void band_seg_launch(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                     cudaStream_t st, const double2* add) {
  const PlanDev& d = P->dev;
  const int m0 = d.m0, ls = seg_len(m0);
  const double2* phi = d.band_seg;
  const double2* psi = d.band_seg + (size_t)SEG * 4 * m0;
  static bool attr = false;
  if (!attr) {
    for (auto k : {band_seg_kernel<false, 4, 4, SMB>, band_seg_kernel<true, 4, 4, SMB>})
      HELM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  // measured at batch 1, n = 2049: deeper register prefetch chunks (8 / 6 rows) slower
  // (register-bound), L2 prefetches 1-2 chunks further ahead no faster
  auto kern = d.band_nopiv ? band_seg_kernel<true, 4, 4, SMB> : band_seg_kernel<false, 4, 4, SMB>;
  const size_t smem = (size_t)ls * SEG * SMB * sizeof(double2);
  HELM_CHECK(smem <= 200 * 1024, "segmented band solve: segment too long");
  launch_pdl(kern, dim3((m0 + SMB - 1) / SMB, batch), SEG * SMB, smem, st, in, out, d.band_piv,
             (const double2*)d.band_l, (const double2*)d.band_u, phi, psi, m0, ls, corr, d.strip_q, d.coarse_scale,
             batch * 4, add);
  HELM_LAUNCH_CHECK();
}

}  // namespace helm
