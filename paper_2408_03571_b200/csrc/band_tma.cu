// Pentadiagonal band solves along y for batches > 4, TMA-staged (part of K5, the Sommerfeld
// coarse solve; the recurrence, the factors and the right-hand-side contract are those of
// band_solve_kernel in band.cu; reference: linalg.solve(cs.a0_factorization, .), coarse.py:174).
//
// band_solve_kernel stages every chunk with per-thread cp.async: ~290 (forward) and ~150
// (backward) instructions per warp and chunk of 8 rows go to addresses and predicates -- 36 % of
// all issued instructions of a kernel whose 8 warps per SM each run one serial recurrence
// (ncu source page, profiles/top_kernel_band_solve_kernel_r02_v4.txt).  Here one thread issues
// per chunk
//   * one cp.async.bulk of the chunk's factors (the blocked layout makes the 8 rows of a CTA's
//     32 modes one contiguous 8 / 12 KB range),
//   * one cp.async.bulk.tensor.3d of the right-hand-side rows / eliminated rows
//     (box = 32 modes x 8 rows x 8 right-hand sides = 32 KB; out-of-range rows, modes and
//     right-hand sides are zero-filled by the TMA unit, so there is no predicate arithmetic),
//   * one cp.async.bulk per row of the strip correction,
// all completing on the stage's mbarrier, and the 256 threads only wait, read shared memory and
// run the recurrence.  No pivoting (PlanDev::band_nopiv: every BASELINE Sommerfeld config).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "ops.cuh"

namespace helm {

constexpr int TBW = 32;  // modes per CTA (lane = mode)
constexpr int TNW = 8;   // right-hand sides per CTA (warp = right-hand side)
constexpr int TR = 8;    // rows per chunk
constexpr int TST = 4;   // stages

struct __align__(128) BandTmaStage {
  double2 fac[TR][TBW][3];   // forward: [TR][TBW][2] (multipliers) in the first 8 KB; backward: U rows
  double2 vec[TNW][TR][TBW];  // right-hand-side rows (forward) / eliminated rows (backward)
  double2 corr[TR][TNW][4];   // strip correction rows
};
static_assert(sizeof(BandTmaStage) % 128 == 0, "stages are TMA destinations");

struct BandTmaMaps {
  CUtensorMap in;    // [batch][m0][2 m0] doubles: right-hand sides (unused when in == null)
  CUtensorMap z;     // the same view of `out` (the eliminated rows, read back by the backward sweep)
  CUtensorMap corr;  // [m0][8 batch] doubles: strip correction rows (unused when corr == null)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tb_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tb_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tb_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tb_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n TB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TB_WAIT;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tb_bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tb_tensor2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tb_tensor3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// VALS / part / add / corr / in: as band_solve_kernel.
template <bool VALS>
__global__ void __launch_bounds__(TBW*(TNW + 1)) band_tma_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                            const double2* __restrict__ L,
                                                            const double2* __restrict__ U, int m0, int batch,
                                                            const double2* __restrict__ corr,
                                                            const double* __restrict__ q,
                                                            const double* __restrict__ sig, int ldc,
                                                            const double2* __restrict__ add,
                                                            double2* __restrict__ part,
                                                            const __grid_constant__ BandTmaMaps maps) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(128) unsigned char sraw[];
  BandTmaStage* stg = reinterpret_cast<BandTmaStage*>(sraw);
  __shared__ __align__(8) uint64_t full[TST], empty[TST];
  const int t = threadIdx.x & (TBW - 1), w = threadIdx.x / TBW;
  const int a0 = blockIdx.x * TBW, a = a0 + t;
  const bool va = a < m0;
  const int bg = blockIdx.y * TNW, b = bg + w;  // this warp's right-hand side
  const bool vb = b < batch;
  const int nb = min(TNW, batch - bg);          // right-hand sides of this CTA
  const size_t N0 = (size_t)m0 * m0;
  const int nch = (m0 + TR - 1) / TR;
  const size_t fbase = (size_t)blockIdx.x * m0 * TBW;  // fac_idx(0, a0, m0)
  double qa[4] = {0.0, 0.0, 0.0, 0.0};
  double sa = 0.0;
  if (corr && va) {
#pragma unroll
    for (int i = 0; i < 4; ++i) qa[i] = q[(size_t)a * 4 + i];
    sa = sig[a];
  }
  auto corrected = [&](double2 v, const double2* c4) {
    double2 c = mk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i) c = fma_(qa[i], c4[i], c);
    return sub(v, scale(c, sa));
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < TST; ++s) {
      tb_init(&full[s], 1);
      tb_init(&empty[s], TNW);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // chunk sequence number qn (forward chunks 0 .. nch-1, then backward nch .. 2 nch - 1):
  // stage qn % TST, barrier parity (qn / TST) & 1
  // ---------------- forward elimination ----------------
  // chunk c: multipliers of rows [8c, 8c+8), incoming rows [8c+3, 8c+11) (step j consumes row j+3)
  auto issue_fwd = [&](int c) {  // thread 0
    BandTmaStage& S = stg[c % TST];
    uint64_t* bar = &full[c % TST];
    const int j0 = c * TR, nr = min(TR, m0 - j0);
    const int r0 = j0 + 3;
    unsigned bytes = (unsigned)nr * TBW * 2 * sizeof(double2);
    if (in) bytes += sizeof(S.vec);
    if (corr) bytes += sizeof(S.corr);
    tb_expect(bar, bytes);
    tb_bulk(&S.fac[0][0][0], L + 2 * (fbase + (size_t)j0 * TBW), (unsigned)nr * TBW * 2 * sizeof(double2), bar);
    if (in) tb_tensor3d(&S.vec[0][0][0], &maps.in, 2 * a0, r0, bg, bar);
    if (corr) tb_tensor2d(&S.corr[0][0][0], &maps.corr, 8 * bg, r0, bar);  // rows / right-hand sides past the end: zeros
  };
  // chunk c: rows j = m0-1-(8c+rr), i.e. the ascending range [jlo, jlo+8), jlo = m0 - 8(c+1)
  // (negative at the last chunk: the tensor load zero-fills, the factor copy skips them)
  auto issue_bwd = [&](int c) {  // thread 0
    const int qn = nch + c;
    BandTmaStage& S = stg[qn % TST];
    uint64_t* bar = &full[qn % TST];
    const int jlo = m0 - TR * (c + 1);
    const int skip = jlo < 0 ? -jlo : 0, nr = TR - skip;
    const unsigned fb = (unsigned)nr * TBW * 3 * sizeof(double2);
    tb_expect(bar, fb + (unsigned)sizeof(S.vec));
    tb_bulk(&S.fac[skip][0][0], U + 3 * (fbase + (size_t)(jlo + skip) * TBW), fb, bar);
    tb_tensor3d(&S.vec[0][0][0], &maps.z, 2 * a0, jlo, bg, bar);
  };
  // ---- producer warp (warp TNW): refills a stage as soon as the eight consumer warps have
  // released it (empty barrier), so the consumers never meet at a CTA barrier inside a sweep
  if (w == TNW) {
    for (int qn = 0; qn < 2 * nch; ++qn) {
      if (qn == nch) {  // the eliminated rows are complete and fenced before the TMA unit reads them
        __syncthreads();
      }
      if (t == 0) {
        const int use = qn / TST;
        if (use > 0) tb_wait(&empty[qn % TST], (unsigned)(use - 1) & 1u);
        if (qn < nch) issue_fwd(qn);
        else issue_bwd(qn - nch);
      }
    }
    return;
  }
  double2 r0v, r1v, r2v;
  {
    const bool ok = va && vb;
    const double2* col = in ? in + (size_t)(ok ? b : 0) * N0 + (va ? a : 0) : nullptr;
    double2 v3[3];
    for (int jj = 0; jj < 3; ++jj) {
      double2 v = mk(0.0, 0.0);
      if (ok && jj < m0) {
        if (in) v = col[(size_t)jj * m0];
        if (corr) {
          double2 c4[4];
          for (int i = 0; i < 4; ++i) c4[i] = corr[(size_t)jj * ldc + (size_t)b * 4 + i];
          v = corrected(v, c4);
        }
      }
      v3[jj] = v;
    }
    r0v = v3[0];
    r1v = v3[1];
    r2v = v3[2];
  }
  double2* zcol = out + (size_t)(vb ? b : 0) * N0 + (va ? a : 0);
  const double2(*facL)[TBW][2];
  for (int c = 0; c < nch; ++c) {
    tb_wait(&full[c % TST], (unsigned)(c / TST) & 1u);
    const BandTmaStage& S = stg[c % TST];
    facL = reinterpret_cast<const double2(*)[TBW][2]>(&S.fac[0][0][0]);
    const int rows = min(TR, m0 - c * TR);
    // all TR rows unconditionally (no early exit: the chunk's shared-memory reads can then be
    // hoisted ahead of the recurrence); rows past the end of the last chunk compute on stale
    // stage data, are never stored and feed nothing (the sweep ends there)
#pragma unroll
    for (int rr = 0; rr < TR; ++rr) {
      const int j = c * TR + rr;
      const double2 l0 = facL[rr][t][0], l1 = facL[rr][t][1];
      const double2 x0 = r0v;
      const double2 x1 = fms_(l0, x0, r1v);
      const double2 x2 = fms_(l1, x0, r2v);
      if (va && vb && rr < rows) zcol[(size_t)j * m0] = x0;
      double2 nx = mk(0.0, 0.0);
      if (j + 3 < m0) {  // rows past the end: the stage slot was not filled
        if (in) nx = S.vec[w][rr][t];
        if (corr) nx = corrected(nx, S.corr[rr][w]);
      }
      r0v = x1;
      r1v = x2;
      r2v = nx;
    }
    __syncwarp();
    if (t == 0) tb_arrive(&empty[c % TST]);  // this warp is done with the stage
  }
  // the backward sweep reads the eliminated rows back through the TMA unit (async proxy)
  __threadfence();
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  __syncthreads();

  // ---------------- backward substitution ----------------
  double2 y1 = mk(0.0, 0.0), y2 = mk(0.0, 0.0);
  // VALS: this lane reduces row (t >> 2) of a chunk over the 8 modes p*8 + vcol(i), p = t & 3
  const int vrow = t >> 2, vp = t & 3;
  auto vcol = [&](int i) { return vp * 8 + ((i + vp + 4 * (vrow & 1)) & 7); };
  double qc[VALS ? 8 : 1][4];
  if constexpr (VALS) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int ac = a0 + vcol(i);
#pragma unroll
      for (int k = 0; k < 4; ++k) qc[i][k] = ac < m0 ? q[(size_t)ac * 4 + k] : 0.0;
    }
  }
  const double2* acol = add ? add + (size_t)(vb ? b : 0) * N0 + (va ? a : 0) : nullptr;
  double2 acur[TR], anxt[TR];
  auto load_add = [&](int c, double2 (&dst)[TR]) {
#pragma unroll
    for (int rr = 0; rr < TR; ++rr) {
      const int j = m0 - 1 - (c * TR + rr);
      dst[rr] = (va && vb && j >= 0) ? __ldg(acol + (size_t)j * m0) : mk(0.0, 0.0);
    }
  };
  if (add) load_add(0, acur);
  for (int c = 0; c < nch; ++c) {
    const int qn = nch + c;
    tb_wait(&full[qn % TST], (unsigned)(qn / TST) & 1u);
    if (add && c + 1 < nch) load_add(c + 1, anxt);
    BandTmaStage& S = stg[qn % TST];
    const int rows = min(TR, m0 - c * TR);
#pragma unroll
    for (int rr = 0; rr < TR; ++rr) {  // no early exit, as in the forward sweep
      const int j = m0 - 1 - (c * TR + rr);
      const int sl = TR - 1 - rr;  // slot of row j in the ascending box
      const double2 u0 = S.fac[sl][t][0], u1 = S.fac[sl][t][1], u2 = S.fac[sl][t][2];
      double2 v = S.vec[w][sl][t];
      v = fms_(u1, y1, v);
      v = fms_(u2, y2, v);
      v = mul(v, u0);
      if constexpr (VALS)
        S.vec[w][sl][t] = v;  // the slot just read; the stage is refilled after the barrier below
      else if (va && vb && rr < rows)
        out[(size_t)b * N0 + (size_t)j * m0 + a] = add ? ::helm::add(v, acur[rr]) : v;
      y2 = y1;
      y1 = v;
    }
    if (add) {
#pragma unroll
      for (int rr = 0; rr < TR; ++rr) acur[rr] = anxt[rr];
    }
    if constexpr (VALS) {
      __syncwarp();
      double2 acc[4] = {mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0), mk(0.0, 0.0)};
      const int rr = vrow, sl = TR - 1 - rr;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double2 x = S.vec[w][sl][vcol(i)];
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
      if (vp == 0 && rr < rows && vb) {
        const int j = m0 - 1 - (c * TR + rr);
        double2* o = part + ((size_t)blockIdx.x * m0 + j) * ldc + (size_t)b * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = acc[k];
      }
      // the generic-proxy writes above precede the TMA refill of this stage
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncwarp();
    if (t == 0) tb_arrive(&empty[qn % TST]);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_band() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    HELM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr));
    HELM_CHECK(p != nullptr && qr == cudaDriverEntryPointSuccess, "driver entry point missing: cuTensorMapEncodeTiled");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

static void make_map(CUtensorMap* map, const double2* base, int m0, int batch) {
  const cuuint64_t dims[3] = {(cuuint64_t)2 * m0, (cuuint64_t)m0, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)m0 * 16, (cuuint64_t)m0 * m0 * 16};
  const cuuint32_t box[3] = {2 * TBW, TR, TNW};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = encode_tiled_band()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims,
                                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HELM_CHECK(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for the band solve");
}

bool band_tma_usable(const helm_plan* P) {  // HELM_BAND_TMA=0: the cp.async kernel (A/B)
  static const bool on = [] {
    const char* e = getenv("HELM_BAND_TMA");
    return !(e && e[0] == '0');
  }();
  return on && P->dev.band_nopiv;
}

void band_tma_launch(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                     cudaStream_t st, const double2* add, double2* part) {
  const PlanDev& d = P->dev;
  constexpr size_t smem = TST * sizeof(BandTmaStage);
  static_assert(smem <= 227 * 1024, "band-solve stages exceed shared memory");
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(band_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    HELM_CUDA(cudaFuncSetAttribute(band_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  BandTmaMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  make_map(&maps.z, out, d.m0, batch);
  if (corr) {
    const cuuint64_t dims[2] = {(cuuint64_t)8 * batch, (cuuint64_t)d.m0};
    const cuuint64_t strides[1] = {(cuuint64_t)batch * 4 * 16};
    const cuuint32_t box[2] = {8 * TNW, TR};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_tiled_band()(&maps.corr, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(corr),
                                           dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HELM_CHECK(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for the strip correction");
  } else {
    maps.corr = maps.z;
  }
  if (in) make_map(&maps.in, in, d.m0, batch);
  else maps.in = maps.z;
  dim3 grd((d.m0 + TBW - 1) / TBW, (batch + TNW - 1) / TNW);
  if (part)
    launch_pdl(band_tma_kernel<true>, grd, TBW * (TNW + 1), smem, st, in, out, (const double2*)d.band_l,
               (const double2*)d.band_u, d.m0, batch, corr, d.strip_q, d.coarse_scale, batch * 4, add, part, maps);
  else
    launch_pdl(band_tma_kernel<false>, grd, TBW * (TNW + 1), smem, st, in, out, (const double2*)d.band_l,
               (const double2*)d.band_u, d.m0, batch, corr, d.strip_q, d.coarse_scale, batch * 4, add, part, maps);
  HELM_LAUNCH_CHECK();
}

}  // namespace helm
