// K4, FP64 tensor-core path: folded fast diagonalisation of the subdomain solves
// (reference: the p^2 SuperLU solves of SchwarzPreconditioner._local_sum,
// schwarz.py:64-74, on R_i A R_i^T, decomposition.py:157-160).
//
//   Y_i = V_y [ (V_y^T X_i V_x) ./ (lam_y (+) lam_x - k^2) ] V_x^T
//
// For boxes whose two 1-D classes are real and symmetric (V[L-1-j][k] = +-V[j][k]:
// the interior middle class and every MP-1 class) the box is folded along both axes
// (s_j = x_j + x_{L-1-j}, d_j = x_j - x_{L-1-j}; even modes see only s, odd modes
// only d), so each 1-D transform is block diagonal with two blocks of DB = 20 (padded).
// The four products then run on the FP64 tensor pipe as mma.sync.m8n8k4.f64 (DMMA):
// complex data is a real matrix with interleaved (re, im) columns (LEFT products) or
// rows (RIGHT products), V stays real.  One CTA (5 warps) owns one (box, right-hand
// side); a warp owns a slice of the independent dimension (columns for LEFT, rows for
// RIGHT) and all row / column tiles of the folded block, so each shared-memory fragment
// feeds three DMMAs and the products update the shared tile in place with warp-level
// synchronisation only.  Shared strides are chosen so every fragment load is two
// wavefronts (the minimum for 32 x 8-byte accesses).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "local.cuh"

namespace helm {

// ---------------------------------------------------------------------------------------
// TMA box load (complex boxes): one cp.async.bulk.tensor.3d per (box, right-hand side) moves
// the whole 35 x 35 complex box (rows of 70 doubles) into shared memory, tracked by an mbarrier.
// Real (MP-1) rows are nu x 8 bytes, not a multiple of 16 for odd nu, so they keep cp.async.
// ---------------------------------------------------------------------------------------
struct TmaBox {
  CUtensorMap map;  // dims {2 nu, nu, batch} doubles, box {2 BX, BY, 1}
  int bx, by;       // box extent in complex columns / rows (0: TMA off)
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

constexpr int DB = 20;      // folded block (even / odd modes)
constexpr int DT = 2 * DB;  // tile side
constexpr int DVL = DT;     // V leading dimension (doubles): the plan's global tables, read through L1
constexpr int DWARPS = 5;   // warps per CTA: each owns 1/5 of the column (LEFT) / row (RIGHT) tiles
constexpr int DTH = 32 * DWARPS;

template <int NP> struct DmmaDims {
  static constexpr int XL = NP == 2 ? 88 : 40;  // X leading dimension (doubles), = 8 (mod 16)
  static constexpr int NT = DT * NP / 8;        // real column tiles (LEFT) / real row tiles (RIGHT)
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// LEFT product  X <- V' X  with V'(m, k) = TRANS ? V[k][m] : V[m][k], block diagonal:
// rows of block b read and write only rows of block b, so the blocks run one after the
// other (one set of accumulators live at a time).  Columns are independent: warp w owns
// TPW real-column tiles and all three 8-row tiles of the block, so every B fragment
// (shared memory) feeds three DMMAs and every A fragment (V, through L1) TPW of them, and
// the in-place update needs no block barrier (a warp only rewrites its own columns).
template <int NP, bool TRANS, typename EPI>
__device__ __forceinline__ void dmma_left(double* Xr, const double* __restrict__ V, EPI epi) {
  constexpr int XL = DmmaDims<NP>::XL, NT = DmmaDims<NP>::NT, TPW = NT / DWARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int c0 = w * TPW * 8;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double acc[3][TPW][2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int t = 0; t < TPW; ++t) acc[r][t][0] = acc[r][t][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < DB / 4; ++ks) {
      const int k = b * DB + ks * 4 + q;
      double af[3], bf[TPW];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int m = b * DB + r * 8 + g;  // rows past the block are discarded (past the tile: zero)
        af[r] = (m < DT) ? __ldg(TRANS ? &V[k * DVL + m] : &V[m * DVL + k]) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < TPW; ++t) bf[t] = Xr[k * XL + c0 + t * 8 + g];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int t = 0; t < TPW; ++t) dmma(acc[r][t][0], acc[r][t][1], af[r], bf[t]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int ml = r * 8 + g;
      if (ml < DB) {
#pragma unroll
        for (int t = 0; t < TPW; ++t) epi(b * DB + ml, c0 + t * 8 + 2 * q, acc[r][t][0], acc[r][t][1]);
      }
    }
    __syncwarp();
  }
}

// RIGHT product  X <- X V'  with V'(k, n) = TRANS ? V[n][k] : V[k][n], block diagonal in
// the columns (blocks one after the other as above).  Real rows r = (m, part) read
// X[m][k NP + part] and are independent: warp w owns TPW real-row tiles and all three
// 8-column tiles of the block (A from shared memory reused three times, B from V).
template <int NP, bool TRANS, typename EPI>
__device__ __forceinline__ void dmma_right(double* Xr, const double* __restrict__ V, EPI epi) {
  constexpr int XL = DmmaDims<NP>::XL, NT = DmmaDims<NP>::NT, TPW = NT / DWARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int r0 = w * TPW * 8;
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    double acc[TPW][3][2];
#pragma unroll
    for (int t = 0; t < TPW; ++t)
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[t][c][0] = acc[t][c][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < DB / 4; ++ks) {
      const int k = b * DB + ks * 4 + q;
      double af[TPW], bf[3];
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const int r = r0 + t * 8 + g;  // A row (real row) of this lane
        af[t] = Xr[(r / NP) * XL + k * NP + (r % NP)];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const int n = b * DB + c * 8 + g;  // B column of this lane
        bf[c] = (n < DT) ? __ldg(TRANS ? &V[n * DVL + k] : &V[k * DVL + n]) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < TPW; ++t)
#pragma unroll
        for (int c = 0; c < 3; ++c) dmma(acc[t][c][0], acc[t][c][1], af[t], bf[c]);
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int r = r0 + t * 8 + g;
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int nl = c * 8 + 2 * q + e;
          if (nl < DB) epi(r / NP, r % NP, b * DB + nl, acc[t][c][e]);
        }
    }
    __syncwarp();
  }
}

template <typename S>
__global__ void __launch_bounds__(DTH, 5) local_fdm_dmma_kernel(const S* __restrict__ x, const S* __restrict__ base,
                                                             S* __restrict__ y, S* __restrict__ ovl,
                                                             const int* __restrict__ boxes,
                                                             const double* __restrict__ classVf,
                                                             const double* __restrict__ classInvden, int ncls,
                                                             LocalArgs a, const __grid_constant__ TmaBox tma) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  constexpr int NP = Sc<S>::cplx ? 2 : 1;
  constexpr int XL = DmmaDims<NP>::XL;
  extern __shared__ __align__(128) unsigned char smem_raw[];  // 128-byte aligned: the TMA destination
  double* Xr = reinterpret_cast<double*>(smem_raw);  // [DT][XL]
  // per row (y) / column (x) of the box: the output address terms and weights of every node
  // (decomposition.py:111-134), so the scatter does no per-node index arithmetic:
  //   multiplicity 1 x 1 -> y[ry_c + cx_c];  my = 2 -> ovl[ry_a + cx_a];  my = 1, mx = 2 -> ovl[ry_b + cx_b]
  int* meta = reinterpret_cast<int*>(Xr + DT * XL);  // [8][DT]
  int* m_my = meta, *m_mx = meta + DT;
  int* ry_a = meta + 2 * DT, *ry_b = meta + 3 * DT, *ry_c = meta + 4 * DT;
  int* cx_a = meta + 5 * DT, *cx_b = meta + 6 * DT, *py = meta + 7 * DT;  // py: prolongation row offset | parity
  S* rx = reinterpret_cast<S*>(meta + 8 * DT);       // [WIN][DT] x-pass of the window prolongation
  const int sid = boxes[blockIdx.x];
  const int ay = sid / a.p, ax = sid % a.p;
  const int nu = a.nu;
  const size_t N = (size_t)nu * nu;
  const int b = blockIdx.y;
  const int cy = a.box_class[ay], cx = a.box_class[ax];
  const int y0 = a.box_start[ay], Ly = a.box_len[ay];
  const int x0 = a.box_start[ax], Lx = a.box_len[ax];
  const int hy = Ly / 2, hpy = (Ly + 1) / 2, hx = Lx / 2, hpx = (Lx + 1) / 2;
  const S* xb = x + (size_t)b * N;
  const S* bb = base ? base + (size_t)b * base_stride(a) : nullptr;
  S* yb = y + (size_t)b * N;
  S* ob = ovl + (size_t)b * 6 * a.nbands * nu;
  // the raw box streams into the X tile with cp.async (row r at Xr + r XL, scalars in place):
  // every thread has all its copies in flight at once instead of a chain of dependent loads
  __shared__ __align__(8) uint64_t box_bar;
  const bool use_tma = NP == 2 && tma.bx >= Lx && tma.by >= Ly;
  const int RS = use_tma ? 2 * tma.bx : XL;  // row stride (doubles) of the raw box in Xr
  if (use_tma) {
    if (threadIdx.x == 0) {
      mbar_init(&box_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_expect_tx(&box_bar, (unsigned)(2 * tma.bx * tma.by * sizeof(double)));
      tma_load_3d(Xr, &tma.map, 2 * x0, y0, b, &box_bar);
    }
    __syncthreads();  // the barrier is initialised before any thread waits on it
  } else {
    const int q = threadIdx.x % DT;  // column of this thread (constant divisor: no runtime division)
    if (q < Lx)
      for (int r = threadIdx.x / DT; r < Ly; r += DTH / DT) {
        const S* src = xb + (size_t)(y0 + r) * nu + x0 + q;
        if constexpr (NP == 2) cp_async16(&Xr[r * XL + 2 * q], src, true);
        else cp_async8(&Xr[r * XL + q], src, true);
      }
  }
  cp_commit();
  // coarse-base mode: the box's window of c streams into shared memory behind the products
  const int Uby = window_base(y0, a.off), Ubx = window_base(x0, a.off);

  // fold both axes in place: pair (i, j) of the half-box -> the 4 folded entries
  // (s_y s_x) [i][j], (s_y d_x) [i][DB+j], (d_y s_x) [DB+i][j], (d_y d_x) [DB+i][DB+j];
  // all raw values are read (registers) before any folded value is written
  const bool wb = a.weighted && a.wbs;
  auto raw = [&](int r, int q) -> S {
    S v;
    if constexpr (NP == 2) v = mk(Xr[r * RS + 2 * q], Xr[r * RS + 2 * q + 1]);
    else v = Xr[r * RS + q];
    if (wb) v = scale(v, 1.0 / (a.node_mult[y0 + r] * a.node_mult[x0 + q]));
    return v;
  };
  auto put_s = [&](int i, int j, S v) {
    if constexpr (NP == 2) {
      *reinterpret_cast<double2*>(&Xr[i * XL + 2 * j]) = v;
    } else {
      Xr[i * XL + j] = v;
    }
  };
  constexpr int QPT = (DB * DB + DTH - 1) / DTH;  // quads per thread
  S qv[QPT][4];
  cp_wait<0>();
  if (use_tma) mbar_wait(&box_bar, 0);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int e = threadIdx.x + u * DTH;
    const int i = e / DB, j = e % DB;
    qv[u][0] = qv[u][1] = qv[u][2] = qv[u][3] = Sc<S>::zero();
    if (e < DB * DB && i < hpy && j < hpx) {
      const bool ci = i == hy, cj = j == hx;  // centre row / column (odd length)
      qv[u][0] = raw(i, j);
      if (!ci) qv[u][1] = raw(Ly - 1 - i, j);
      if (!cj) qv[u][2] = raw(i, Lx - 1 - j);
      if (!ci && !cj) qv[u][3] = raw(Ly - 1 - i, Lx - 1 - j);
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < QPT; ++u) {
    const int e = threadIdx.x + u * DTH;
    if (e >= DB * DB) break;
    const int i = e / DB, j = e % DB;
    const bool ci = i == hy, cj = j == hx;
    const S a00 = qv[u][0], a10 = qv[u][1], a01 = qv[u][2], a11 = qv[u][3];
    const S sy0 = add(a00, a10), dy0 = sub(a00, a10), sy1 = add(a01, a11), dy1 = sub(a01, a11);
    // the d components of a centre row / column are exactly zero (the padded blocks read them)
    put_s(i, j, add(sy0, sy1));
    put_s(i, DB + j, cj ? Sc<S>::zero() : sub(sy0, sy1));
    put_s(DB + i, j, ci ? Sc<S>::zero() : add(dy0, dy1));
    put_s(DB + i, DB + j, (ci || cj) ? Sc<S>::zero() : sub(dy0, dy1));
  }
  const double* Vy = classVf + (size_t)cy * DT * DT;  // folded V tables (zero padded by the plan)
  const double* Vx = classVf + (size_t)cx * DT * DT;
  for (int e = threadIdx.x; e < DT; e += DTH) {
    const int iy = y0 + (e < Ly ? e : 0), ix = x0 + (e < Lx ? e : 0);
    const int my = a.node_mult[iy], mx = a.node_mult[ix];
    const int ry = ay - a.node_first_box[iy], rxb = ax - a.node_first_box[ix];
    m_my[e] = my;
    m_mx[e] = mx;
    ry_a[e] = (ry * 2 * a.nbands + a.node_band[iy]) * nu;           // band rows: slot (ry, rx), band, x
    ry_b[e] = iy * a.nbands;                                        // band columns: slot rx, y, band
    ry_c[e] = iy * nu;
    cx_a[e] = rxb * a.nbands * nu + ix;
    cx_b[e] = 4 * a.nbands * nu + rxb * nu * a.nbands + a.node_band[ix];
    const int ty = iy - a.off;
    const int U0 = ((ty & 1) == 0 ? ty / 2 - 1 : (ty - 1) >> 1) - window_base(y0, a.off);
    py[e] = (U0 * DT) * 2 + ((ty & 1) == 0 ? 1 : 0);
  }
  const double* invden = classInvden + (size_t)(cy * ncls + cx) * DT * DT;
  __syncthreads();
  // X <- Vfy^T X
  // (the two accumulators of a lane are adjacent columns: one 16-byte store)
  auto store2 = [&](int m, int c, double v0, double v1) { *reinterpret_cast<double2*>(&Xr[m * XL + c]) = mk(v0, v1); };
  dmma_left<NP, true>(Xr, Vy, store2);
  __syncthreads();
  // X <- (X Vfx) ./ (lfy (+) lfx - k^2)
  dmma_right<NP, false>(Xr, Vx, [&](int m, int part, int n, double v) {
    Xr[m * XL + n * NP + part] = v * invden[m * DT + n];  // 1 / (lfy[m] + lfx[n] - k^2), plan table
  });
  __syncthreads();
  // X <- Vfy X
  dmma_left<NP, false>(Xr, Vy, store2);
  __syncthreads();
  // X <- X Vfx^T
  dmma_right<NP, true>(Xr, Vx, [&](int m, int part, int n, double v) { Xr[m * XL + n * NP + part] = v; });
  cp_wait<0>();
  __syncthreads();
  // R0^T c at the box's nodes, separably: the x pass (3 taps per window row and fine column,
  // the same fma order as window_prolong) once per CTA into rx, the y pass per node below --
  // bitwise the same sums as window_prolong with a third of its FP64 work (which shares the
  // pipe with the DMMAs)
  const bool cbase = bb && a.coarse_base;
  if (cbase) {
    const int j = threadIdx.x % DT;
    if (j < Lx) {
      const int tx = x0 + j - a.off;
      const bool ex = (tx & 1) == 0;
      const int V0 = (ex ? tx / 2 - 1 : (tx - 1) >> 1) - Ubx;
      const double w0 = ex ? 0.125 : 0.5, w1 = ex ? 0.75 : 0.5, w2 = ex ? 0.125 : 0.0;
      // the window of c straight from L2 (zero outside [0, m0)), same taps and order as window_prolong
      const int Vc = Ubx + V0;
      for (int u = threadIdx.x / DT; u < WIN; u += DTH / DT) {
        const int U = Uby + u;
        S c[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int V = Vc + t;
          c[t] = (U >= 0 && U < a.m0 && V >= 0 && V < a.m0) ? __ldg(bb + (size_t)U * a.m0 + V) : Sc<S>::zero();
        }
        S row = Sc<S>::zero();
        row = fma_(w0, c[0], row);
        row = fma_(w1, c[1], row);
        row = fma_(w2, c[2], row);
        rx[u * DT + j] = row;
      }
    }
    __syncthreads();
  }
  auto prolong_y = [&](int r, int q) {  // the y pass of R0^T c at box node (r, q), taps from py[r]
    const int code = py[r];
    const bool ey = code & 1;
    const S* t = rx + (code >> 1) + q;
    S acc = Sc<S>::zero();
    acc = fma_(ey ? 0.125 : 0.5, t[0], acc);
    acc = fma_(ey ? 0.75 : 0.5, t[DT], acc);
    acc = fma_(ey ? 0.125 : 0.0, t[2 * DT], acc);
    return acc;
  };
  // unfold + weight + scatter: x_i = e_i + o_i, x_{L-1-i} = e_i - o_i on both axes
  auto get = [&](int i, int j) -> S {
    if constexpr (NP == 2) return *reinterpret_cast<const double2*>(&Xr[i * XL + 2 * j]);
    else return Xr[i * XL + j];
  };
  const bool wpu = a.weighted && !a.wbs;
  auto put = [&](int r, int q, S acc) {
    const int my = m_my[r], mx = m_mx[q];
    // partition-of-unity weight 1 / (my mx) with my, mx in {1, 2}: exact constants, no division
    if (wpu && my * mx != 1) acc = scale(acc, my * mx == 2 ? 0.5 : 0.25);
    if (my == 1 && mx == 1) {
      const int pidx = ry_c[r] + x0 + q;
      yb[pidx] = bb ? add(cbase ? prolong_y(r, q) : bb[pidx], acc) : acc;
    } else if (my == 2) {
      ob[ry_a[r] + cx_a[q]] = acc;
    } else {
      ob[ry_b[r] + cx_b[q]] = acc;
    }
  };
  {
    const int j = threadIdx.x % DB;  // half-box column of this thread (constant divisor)
    if (j < hpx) {
      const bool cj = j == hx;
      for (int i = threadIdx.x / DB; i < hpy; i += DTH / DB) {
        const bool ci = i == hy;
        const S ee = get(i, j);
        const S eo = cj ? Sc<S>::zero() : get(i, DB + j);
        const S oe = ci ? Sc<S>::zero() : get(DB + i, j);
        const S oo = (ci || cj) ? Sc<S>::zero() : get(DB + i, DB + j);
        const S ry0 = add(ee, oe), ry1 = sub(ee, oe);  // row i / row L-1-i, still split in x
        const S rz0 = add(eo, oo), rz1 = sub(eo, oo);
        put(i, j, add(ry0, rz0));
        if (!cj) put(i, Lx - 1 - j, sub(ry0, rz0));
        if (!ci) put(Ly - 1 - i, j, add(ry1, rz1));
        if (!ci && !cj) put(Ly - 1 - i, Lx - 1 - j, sub(ry1, rz1));
      }
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HELM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    HELM_CHECK(p != nullptr && q == cudaDriverEntryPointSuccess, "driver entry point missing: cuTensorMapEncodeTiled");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
static bool tma_enabled() {  // HELM_TMA=0: cp.async box loads everywhere (A/B)
  static const bool on = [] {
    const char* e = getenv("HELM_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename S>
void launch_local_dmma(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st) {
  const PlanDev& d = P->dev;
  if (d.n_ff == 0) return;
  constexpr int NP = Sc<S>::cplx ? 2 : 1;
  const size_t smem = (size_t)(DT * DmmaDims<NP>::XL) * sizeof(double) + 8 * DT * sizeof(int) +
                      (a.coarse_base ? (WIN * DT) * sizeof(S) : 0);
  static bool attr = false;
  if (!attr) {
    const size_t smax = (size_t)(DT * DmmaDims<NP>::XL) * sizeof(double) + 8 * DT * sizeof(int) +
                        (WIN * DT) * sizeof(S);
    HELM_CUDA(cudaFuncSetAttribute(local_fdm_dmma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smax));
    attr = true;
  }
  TmaBox tma;
  std::memset(&tma, 0, sizeof(tma));
  if (NP == 2 && tma_enabled()) {
    // box extent = the largest folded box (every folded MP-2 box is an interior one)
    int bx = 0;
    for (int c = 0; c < (int)P->h_class_len.size(); ++c) bx = std::max(bx, P->h_class_len[c]);
    if (bx <= DB * 2 && 2 * bx <= 256 && bx <= 256) {
      const cuuint64_t dims[3] = {(cuuint64_t)2 * a.nu, (cuuint64_t)a.nu, (cuuint64_t)batch};
      const cuuint64_t strides[2] = {(cuuint64_t)a.nu * 16, (cuuint64_t)a.nu * a.nu * 16};
      const cuuint32_t box[3] = {(cuuint32_t)(2 * bx), (cuuint32_t)bx, 1};
      const cuuint32_t es[3] = {1, 1, 1};
      const CUresult r = encode_tiled()(&tma.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<S*>(x), dims, strides,
                                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      HELM_CHECK(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for the local box load");
      tma.bx = tma.by = bx;
    }
  }
  dim3 grd(d.n_ff, batch);
  launch_pdl(local_fdm_dmma_kernel<S>, grd, DTH, smem, st, x, base, y, ovl, d.box_ff, d.class_Vf, d.class_invden,
                                                   d.n_classes, a, tma);
  HELM_LAUNCH_CHECK();
}

template void launch_local_dmma<double>(const helm_plan*, const double*, const double*, double*, double*,
                                        const LocalArgs&, int, cudaStream_t);
template void launch_local_dmma<double2>(const helm_plan*, const double2*, const double2*, double2*, double2*,
                                         const LocalArgs&, int, cudaStream_t);

}  // namespace helm
