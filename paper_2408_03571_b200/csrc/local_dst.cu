// K4, fast-sine path: subdomain solves of the boxes whose two 1-D classes are the
// Dirichlet middle pencil tridiag(-1, 2, -1)/h^2 with W = I (every interior box of a
// BASELINE config; reference: the p^2 SuperLU solves of SchwarzPreconditioner._local_sum,
// schwarz.py:64-74, on R_i A R_i^T, decomposition.py:157-160).
//
// Those classes are diagonalised exactly by the DST-I, V = sqrt(2/N) S with
// S[j][m] = sin(pi (j+1) (m+1) / N), N = L + 1, and S is symmetric, so
//
//   Y_i = (2/N)^2  S [ (S X_i S) ./ (lam_y (+) lam_x - k^2) ] S
//
// (the (2/N)^2 lives in the plan's reciprocal table).  For N = 4Q (Q odd: L = 35 at every
// BASELINE config, 19 at config 1) one application of S is three levels of even/odd folding
// -- the first three stages of a split FFT -- and small dense blocks:
//
//   level 1  s_j = x_j + x_{N-j}, d_j = x_j - x_{N-j}: odd modes see s, even modes d;
//   odd m    split s by the parity of j: y_m = O + E, y_{N-m} = O - E (two Q x Q blocks);
//   even m   fold d again (pairs j, 2Q - j): modes 2 (mod 4) are a Q x Q block, modes
//            0 (mod 4) a DST-I of length Q - 1 folded once more into two (Q-1)/2 blocks,
//
// 275 multiply-adds and 76 additions per length-35 vector instead of the 35^2 = 1225 of a
// dense product (613 folded once, 960 as padded m8n8k4 DMMA work in local_dmma.cu).  The
// block coefficients are uniform across a warp and live in __constant__ memory, so every
// multiply-add takes its coefficient as a constant-bank operand: the inner loops are DFMA
// and register moves only.  One thread owns one real vector (a row or column of the re or
// im part) for a whole 1-D transform held in registers; the box is transposed through shared
// memory between the x and y passes, and the y pass applies S, the eigenvalue reciprocals
// and S again without leaving registers.  A CTA owns NB (box, right-hand side) slots of the
// same box so the 2 NP L vectors of a pass fill whole warps.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "local.cuh"

namespace helm {

// ---------------------------------------------------------------------------------------
// coefficient tables: for Q, blocks A, B (odd modes), C (modes 2 mod 4), D1, D2 (0 mod 4)
// ---------------------------------------------------------------------------------------
template <int Q> struct DstTab {
  static constexpr int R = (Q - 1) / 2;
  static constexpr int A = 0, B = Q * Q, C = 2 * Q * Q, D1 = 3 * Q * Q, D2 = 3 * Q * Q + R * R;
  static constexpr int SIZE = 3 * Q * Q + 2 * R * R;
};
constexpr int DST_OFF5 = 0;
constexpr int DST_OFF9 = DstTab<5>::SIZE;
constexpr int DST_TAB_SIZE = DstTab<5>::SIZE + DstTab<9>::SIZE;
__constant__ double c_dst[DST_TAB_SIZE];

template <int Q> __device__ __forceinline__ constexpr int dst_off() { return Q == 5 ? DST_OFF5 : DST_OFF9; }

static void host_tab(int Q, double* t) {
  const long double pi = 3.14159265358979323846264338327950288L;
  const int R = (Q - 1) / 2, N4 = 4 * Q;
  double* A = t;
  double* B = t + Q * Q;
  double* C = t + 2 * Q * Q;
  double* D1 = t + 3 * Q * Q;
  double* D2 = D1 + R * R;
  for (int i = 0; i < Q; ++i)
    for (int u = 0; u < Q; ++u) {
      A[i * Q + u] = (double)sinl(pi * (2 * i + 1) * (2 * u + 1) / N4);
      B[i * Q + u] = (double)sinl(pi * (2 * i + 2) * (2 * u + 1) / N4);
      C[i * Q + u] = (double)sinl(pi * (i + 1) * (2 * u + 1) / (2 * Q));
    }
  for (int j = 0; j < R; ++j)
    for (int u = 0; u < R; ++u) {
      D1[j * R + u] = (double)sinl(pi * (j + 1) * (2 * u + 1) / Q);
      D2[j * R + u] = (double)sinl(pi * (j + 1) * (2 * u + 2) / Q);
    }
}

static void upload_dst_tables() {  // once per device (the tables depend on Q only)
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  HELM_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && done[dev]) return;
  double h[DST_TAB_SIZE];
  host_tab(5, h + DST_OFF5);
  host_tab(9, h + DST_OFF9);
  HELM_CUDA(cudaMemcpyToSymbol(c_dst, h, sizeof(h)));
  if (dev < 64) done[dev] = true;
}

// y = S x in place, x[j] = x_{j+1}, y[m] = y_{m+1} (1-based indices in the comments).
template <int Q> __device__ __forceinline__ void dst_apply(double (&v)[4 * Q - 1]) {
  constexpr int N4 = 4 * Q, R = (Q - 1) / 2, T = dst_off<Q>();
  constexpr int A = T + DstTab<Q>::A, B = T + DstTab<Q>::B, C = T + DstTab<Q>::C;
  constexpr int D1 = T + DstTab<Q>::D1, D2 = T + DstTab<Q>::D2;
  double s[2 * Q], d[2 * Q - 1];
#pragma unroll
  for (int j = 1; j < 2 * Q; ++j) {
    s[j - 1] = v[j - 1] + v[N4 - j - 1];
    d[j - 1] = v[j - 1] - v[N4 - j - 1];
  }
  s[2 * Q - 1] = v[2 * Q - 1];
  // odd modes m = 2u + 1 and N - m: O over odd j (s[2i]), E over even j (s[2i + 1])
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    double o = s[0] * c_dst[A + u], e = s[1] * c_dst[B + u];
#pragma unroll
    for (int i = 1; i < Q; ++i) {
      o = fma(s[2 * i], c_dst[A + i * Q + u], o);
      e = fma(s[2 * i + 1], c_dst[B + i * Q + u], e);
    }
    v[2 * u] = o + e;
    v[N4 - 2 * u - 2] = o - e;
  }
  // even modes: a_j = d_j + d_{2Q-j} (j < Q), a_Q = d_Q;  b_j = d_j - d_{2Q-j}
  double a[Q], b[Q - 1];
#pragma unroll
  for (int j = 1; j < Q; ++j) {
    a[j - 1] = d[j - 1] + d[2 * Q - j - 1];
    b[j - 1] = d[j - 1] - d[2 * Q - j - 1];
  }
  a[Q - 1] = d[Q - 1];
  // modes m = 2 (2u + 1): C block
#pragma unroll
  for (int u = 0; u < Q; ++u) {
    double acc = a[0] * c_dst[C + u];
#pragma unroll
    for (int j = 1; j < Q; ++j) acc = fma(a[j], c_dst[C + j * Q + u], acc);
    v[4 * u + 1] = acc;
  }
  // modes m = 4 w (w = 1 .. Q-1): fold b once more, pairs (j, Q - j)
  double pp[R], pm[R];
#pragma unroll
  for (int j = 1; j <= R; ++j) {
    pp[j - 1] = b[j - 1] + b[Q - j - 1];
    pm[j - 1] = b[j - 1] - b[Q - j - 1];
  }
#pragma unroll
  for (int u = 0; u < R; ++u) {
    double o = pp[0] * c_dst[D1 + u], e = pm[0] * c_dst[D2 + u];
#pragma unroll
    for (int j = 1; j < R; ++j) {
      o = fma(pp[j], c_dst[D1 + j * R + u], o);
      e = fma(pm[j], c_dst[D2 + j * R + u], e);
    }
    v[4 * (2 * u + 1) - 1] = o;  // w = 2u + 1
    v[4 * (2 * u + 2) - 1] = e;  // w = 2u + 2
  }
}

template <int NP, int Q> struct DstGeo {
  static constexpr int L = 4 * Q - 1;
  static constexpr int RS = NP * L;                        // row stride of a slot (doubles) = the TMA box row
  static constexpr int VEC = NP * L;                       // vectors per slot and pass
  static constexpr int NB = (NP == 2 ? 2 : 4) * (Q == 5 ? 2 : 1);  // slots per CTA
  static constexpr int NTH = ((NB * VEC + 31) / 32) * 32;
  static constexpr int XB = ((L * RS * 8 + 127) / 128) * 128;  // bytes of a slot's tile (128-aligned: TMA)
  static constexpr int RXB = ((WIN * L * NP * 8 + 127) / 128) * 128;  // bytes of a slot's prolongation x pass
  static constexpr int META = 8 * 40 * 4;
  static constexpr size_t smem(bool cbase) { return (size_t)NB * XB + (cbase ? (size_t)NB * RXB : 0) + META; }
};

struct TmaDst {
  CUtensorMap map;   // dims {2 nu, nu, batch} doubles, box {2 L, L, 1}
  CUtensorMap cmap;  // coarse base: dims {2 m0, m0, batch} doubles, box {2 WIN, WIN, 1} (con != 0)
  int on, con;
};

__device__ __forceinline__ void mbar_init_(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// ---------------------------------------------------------------------------------------
// box input / output shared by the fast-sine kernels: per-row / per-column scatter tables
// (decomposition.py:111-134, as in local_dmma.cu), the x pass of R0^T c over the box's coarse
// window (the same taps and fma order as window_prolong, bitwise), and the epilogue
// (partition-of-unity weight, + R0^T c or base, scatter to y or the overlap slots).
// ---------------------------------------------------------------------------------------
constexpr int DML = 40;  // meta table stride (>= box side)
template <typename S> struct BoxOut {
  const LocalArgs& a;
  int* meta;  // [8][DML]: m_my, m_mx, ry_a, ry_b, ry_c, cx_a, cx_b, py
  S* rx;      // [slot][WIN][Lx] (coarse-base mode)
  int rxs;    // elements per slot of rx
  int ay, ax, y0, x0, Ly, Lx, Uby;
  __device__ BoxOut(const LocalArgs& a_, int* meta_, S* rx_, int ay_, int ax_, int Ly_, int Lx_)
      : a(a_), meta(meta_), rx(rx_), rxs(WIN * Lx_), ay(ay_), ax(ax_), Ly(Ly_), Lx(Lx_) {
    y0 = a.box_start[ay];
    x0 = a.box_start[ax];
    Uby = window_base(y0, a.off);
  }
  __device__ void init_meta(int nth) const {
    const int nu = a.nu;
    for (int e = threadIdx.x; e < Ly; e += nth) {
      const int iy = y0 + e;
      const int ry = ay - a.node_first_box[iy];
      meta[e] = a.node_mult[iy];
      meta[2 * DML + e] = (ry * 2 * a.nbands + a.node_band[iy]) * nu;
      meta[3 * DML + e] = iy * a.nbands;
      meta[4 * DML + e] = iy * nu;
      const int ty = iy - a.off;
      const int U0 = ((ty & 1) == 0 ? ty / 2 - 1 : (ty - 1) >> 1) - Uby;
      meta[7 * DML + e] = (U0 * Lx) * 2 + ((ty & 1) == 0 ? 1 : 0);
    }
    for (int e = threadIdx.x; e < Lx; e += nth) {
      const int ix = x0 + e;
      const int rxb = ax - a.node_first_box[ix];
      meta[DML + e] = a.node_mult[ix];
      meta[5 * DML + e] = rxb * a.nbands * nu + ix;
      meta[6 * DML + e] = 4 * a.nbands * nu + rxb * nu * a.nbands + a.node_band[ix];
    }
  }
  __device__ void init_rx(const S* __restrict__ base, int b0, int nslot, int nth) const {
    for (int e = threadIdx.x; e < nslot * WIN * Lx; e += nth) {
      const int s = e / (WIN * Lx), r = e % (WIN * Lx), u = r / Lx, j = r % Lx;
      const S* bb = base + (size_t)(b0 + s) * base_stride(a);
      const int tx = x0 + j - a.off;
      const bool ex = (tx & 1) == 0;
      const int Vc = ex ? tx / 2 - 1 : (tx - 1) >> 1;
      const double w0 = ex ? 0.125 : 0.5, w1 = ex ? 0.75 : 0.5, w2 = ex ? 0.125 : 0.0;
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
      rx[(size_t)s * rxs + u * Lx + j] = row;
    }
  }
  // node (r, q) of slot sl (right-hand side b) with solve value acc
  __device__ __forceinline__ void put(const S* __restrict__ base, S* __restrict__ y, S* __restrict__ ovl, bool cbase,
                                      int sl, int b, int r, int q, S acc) const {
    const int nu = a.nu;
    const size_t N = (size_t)nu * nu;
    const int my = meta[r], mx = meta[DML + q];
    if (a.weighted && !a.wbs && my * mx != 1) acc = scale(acc, my * mx == 2 ? 0.5 : 0.25);
    if (my == 1 && mx == 1) {
      const int pidx = meta[4 * DML + r] + x0 + q;
      S bv = Sc<S>::zero();
      if (cbase) {
        const int code = meta[7 * DML + r];
        const bool ey = code & 1;
        const S* tp = rx + (size_t)sl * rxs + (code >> 1) + q;
        bv = fma_(ey ? 0.125 : 0.5, tp[0], bv);
        bv = fma_(ey ? 0.75 : 0.5, tp[Lx], bv);
        bv = fma_(ey ? 0.125 : 0.0, tp[2 * Lx], bv);
      } else if (base) {
        bv = base[(size_t)b * N + pidx];
      }
      y[(size_t)b * N + pidx] = base ? add(bv, acc) : acc;
    } else {
      S* ob = ovl + (size_t)b * 6 * a.nbands * nu;
      if (my == 2) ob[meta[2 * DML + r] + meta[5 * DML + q]] = acc;
      else ob[meta[3 * DML + r] + meta[6 * DML + q]] = acc;
    }
  }
  // Column-mapped forms for the fast-sine kernel: thread = (row group rg of NG, column q), so the
  // column terms (parity, taps, bounds, scatter offsets) are computed once per thread and the
  // loops carry only row terms (uniform across a warp's columns).  Same values and fma order as
  // init_rx / put (bitwise); the element-mapped forms cost ~90 / ~80 instructions per node in
  // index arithmetic (42 % of the kernel's instructions, profiles/top_kernel_local_dst_kernel_r02_v4.txt).
  template <int NG> __device__ void init_rx_cols(const S* __restrict__ base, int b0, int nslot, int rg, int j) const {
    const int tx = x0 + j - a.off;
    const bool ex = (tx & 1) == 0;
    const int Vc = ex ? tx / 2 - 1 : (tx - 1) >> 1;
    const double w0 = ex ? 0.125 : 0.5, w1 = ex ? 0.75 : 0.5, w2 = ex ? 0.125 : 0.0;
    bool okv[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) okv[t] = Vc + t >= 0 && Vc + t < a.m0;
    const size_t bs = base_stride(a);
    // NIT rows per thread in batches of HB: a batch's 3 HB loads are all in flight before the
    // first is used (the prologue has registers to spare; one row at a time left the
    // L2 latency of every row exposed: 21 % of the kernel's stall samples)
    constexpr int HB = 6;
    const int total = nslot * WIN;
    for (int i0 = 0; rg + i0 * NG < total; i0 += HB) {
      S c[HB][3];
      int su[HB];
#pragma unroll
      for (int i = 0; i < HB; ++i) {
        const int idx = rg + (i0 + i) * NG;
        const int sl = idx / WIN, u = idx - sl * WIN;
        su[i] = idx < total ? sl * rxs + u * Lx : -1;
        const int U = Uby + u;
        const bool okU = idx < total && U >= 0 && U < a.m0;
        const S* bb = base + (size_t)(b0 + (okU ? sl : 0)) * bs + (size_t)(okU ? U : 0) * a.m0 + Vc;
#pragma unroll
        for (int t = 0; t < 3; ++t) c[i][t] = (okU && okv[t]) ? __ldg(bb + t) : Sc<S>::zero();
      }
#pragma unroll
      for (int i = 0; i < HB; ++i) {
        S row = Sc<S>::zero();
        row = fma_(w0, c[i][0], row);
        row = fma_(w1, c[i][1], row);
        row = fma_(w2, c[i][2], row);
        if (su[i] >= 0) rx[su[i] + j] = row;
      }
    }
  }
  // The same x pass from the box's raw coarse window staged in shared memory (WIN x WIN, dense,
  // zero outside the coarse grid: the tensor copy's out-of-bounds fill) at `raw`, which lies inside
  // slot sl's own rx region: every tap of the thread's rows is read into registers before the
  // barrier, the rows are written after it.  Called by all threads of the CTA (it synchronises).
  template <int NG, int NR> __device__ void rx_from_window(const S* raw, int sl, int rg, int j, bool part) const {
    const int tx = x0 + j - a.off;
    const bool ex = (tx & 1) == 0;
    const int V0 = (ex ? tx / 2 - 1 : (tx - 1) >> 1) - window_base(x0, a.off);
    const double w0 = ex ? 0.125 : 0.5, w1 = ex ? 0.75 : 0.5, w2 = ex ? 0.125 : 0.0;
    S c[NR][3];
    if (part) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int u = rg + i * NG;
#pragma unroll
        for (int t = 0; t < 3; ++t) c[i][t] = u < WIN ? raw[u * WIN + V0 + t] : Sc<S>::zero();
      }
    }
    __syncthreads();
    if (part) {
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int u = rg + i * NG;
        S row = Sc<S>::zero();
        row = fma_(w0, c[i][0], row);
        row = fma_(w1, c[i][1], row);
        row = fma_(w2, c[i][2], row);
        if (u < WIN) rx[(size_t)sl * rxs + u * Lx + j] = row;
      }
    }
  }
  struct ColTerms {
    int mx, c5, c6;
  };
  __device__ __forceinline__ ColTerms col_terms(int q) const {
    return ColTerms{meta[DML + q], meta[5 * DML + q], meta[6 * DML + q]};
  }
  __device__ __forceinline__ void put_col(const S* __restrict__ base, S* __restrict__ y, S* __restrict__ ovl,
                                          bool cbase, int sl, int b, int r, int q, const ColTerms& ct, S acc) const {
    const int nu = a.nu;
    const size_t N = (size_t)nu * nu;
    // branch-free: a warp's columns mix interior and overlap nodes in every row, so the two
    // store paths of put() both ran for nearly every warp (divergence doubled the epilogue);
    // here every lane forms both addresses and one predicated value and stores once
    const int my = meta[r], mm = my * ct.mx;
    const bool interior = mm == 1;
    if (a.weighted && !a.wbs) acc = scale(acc, interior ? 1.0 : (mm == 2 ? 0.5 : 0.25));  // x * 1.0 == x
    const int pidx = meta[4 * DML + r] + x0 + q;
    S bv = Sc<S>::zero();
    if (cbase) {
      const int code = meta[7 * DML + r];
      const bool ey = code & 1;
      const S* tp = rx + (size_t)sl * rxs + (code >> 1) + q;
      bv = fma_(ey ? 0.125 : 0.5, tp[0], bv);
      bv = fma_(ey ? 0.75 : 0.5, tp[Lx], bv);
      bv = fma_(ey ? 0.125 : 0.0, tp[2 * Lx], bv);
    } else if (base && interior) {
      bv = base[(size_t)b * N + pidx];
    }
    const S val = (base && interior) ? add(bv, acc) : acc;
    const int oo = my == 2 ? meta[2 * DML + r] + ct.c5 : meta[3 * DML + r] + ct.c6;
    S* dst = interior ? y + (size_t)b * N + pidx : ovl + (size_t)b * 6 * a.nbands * nu + oo;
    *dst = val;
  }
  // weights-before-solve factor of node (r, q)
  __device__ __forceinline__ double wbs_factor(int r, int q) const {
    return 1.0 / (a.node_mult[y0 + r] * a.node_mult[x0 + q]);
  }
};

template <typename S, int Q>
__global__ void __launch_bounds__(DstGeo<Sc<S>::cplx ? 2 : 1, Q>::NTH, 3)
    local_dst_kernel(const S* __restrict__ x, const S* __restrict__ base, S* __restrict__ y, S* __restrict__ ovl,
                     const int* __restrict__ boxes, const double* __restrict__ dinv, LocalArgs a, int batch,
                     const __grid_constant__ TmaDst tma) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  constexpr int NP = Sc<S>::cplx ? 2 : 1;
  using G = DstGeo<NP, Q>;
  constexpr int L = G::L, RS = G::RS, VEC = G::VEC, NB = G::NB, NTH = G::NTH, N4 = 4 * Q;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto X = [&](int s) { return reinterpret_cast<double*>(smem_raw + (size_t)s * G::XB); };
  const bool cbase = base && a.coarse_base;
  int* meta = reinterpret_cast<int*>(smem_raw + (size_t)NB * G::XB + (cbase ? (size_t)NB * G::RXB : 0));
  S* rx = reinterpret_cast<S*>(smem_raw + (size_t)NB * G::XB);
  // coarse-base windows by tensor copy: the raw WIN x WIN window of slot s is staged at the first
  // 128-byte boundary inside the slot's own rx region (it must fit there: L >= WIN)
  constexpr bool CWIN_FITS = NP == 2 && L >= WIN + 1;
  const bool cwin = CWIN_FITS && cbase && tma.on && tma.con;
  auto raw_win = [&](int s) {
    const size_t off = ((size_t)s * WIN * L * sizeof(S) + 127) & ~(size_t)127;
    return reinterpret_cast<S*>(smem_raw + (size_t)NB * G::XB + off);
  };

  const int sid = boxes[blockIdx.x];
  const int ay = sid / a.p, ax = sid % a.p;
  const int nu = a.nu;
  const size_t N = (size_t)nu * nu;
  const int b0 = blockIdx.y * NB;
  const int nslot = min(NB, batch - b0);
  const BoxOut<S> io(a, meta, rx, ay, ax, L, L);
  const int y0 = io.y0, x0 = io.x0;

  // ---- the raw boxes: one TMA per slot (complex), or cp.async (real rows are not 16-byte multiples)
  __shared__ __align__(8) uint64_t box_bar;
  if (tma.on) {
    if (threadIdx.x == 0) {
      mbar_init_(&box_bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_expect_tx_(&box_bar, (unsigned)(nslot * L * RS * sizeof(double)) +
                                    (cwin ? (unsigned)(nslot * WIN * WIN * sizeof(S)) : 0u));
      for (int s = 0; s < nslot; ++s) tma_load_3d_(X(s), &tma.map, NP * x0, y0, b0 + s, &box_bar);
      if (cwin)  // the raw coarse windows ride on the same barrier, into their slots' rx regions
        for (int s = 0; s < nslot; ++s)
          tma_load_3d_(raw_win(s), &tma.cmap, NP * window_base(x0, a.off), window_base(y0, a.off), b0 + s, &box_bar);
    }
  } else {
    for (int e = threadIdx.x; e < nslot * L * L; e += NTH) {
      const int s = e / (L * L), r = (e / L) % L, q = e % L;
      const S* src = x + (size_t)(b0 + s) * N + (size_t)(y0 + r) * nu + x0 + q;
      if constexpr (NP == 2) cp_async16(&X(s)[r * RS + 2 * q], src, true);
      else cp_async8(&X(s)[r * RS + q], src, true);
    }
    cp_commit();
  }
  io.init_meta(NTH);
  // prologue / epilogue thread map: NG row groups x L columns (NG * L <= NTH)
  constexpr int NG = NTH / L;
  const int cq = threadIdx.x % L, crg = threadIdx.x / L;
  if (cbase && !cwin && crg < NG) io.template init_rx_cols<NG>(base, b0, nslot, crg, cq);  // behind the box load
  if (tma.on) {
    __syncthreads();  // the barrier is initialised before any thread waits on it
    mbar_wait_(&box_bar, 0);
  } else {
    cp_wait<0>();
  }
  __syncthreads();
  if (cwin) {  // x pass of R0^T c from the staged windows (no global latency in the prologue)
    constexpr int NR = (WIN + NG - 1) / NG;
    for (int sl = 0; sl < nslot; ++sl) io.template rx_from_window<NG, NR>(raw_win(sl), sl, crg, cq, crg < NG);
  }

  // vector of this thread in a pass: slot s, line (row or column) l, part (re / im)
  const int t = threadIdx.x;
  const int s = t / VEC, it = t % VEC;
  const int l = it / NP, part = it % NP;
  const bool act = t < nslot * VEC;
  double* Xs = X(s < NB ? s : 0);
  double v[L];
  // ---- pass 1: rows, x transform (weights before the solve folded into the load)
  if (act) {
    const bool wb = a.weighted && a.wbs;
#pragma unroll
    for (int j = 0; j < L; ++j) {
      v[j] = Xs[l * RS + NP * j + part];
      if (wb) v[j] *= io.wbs_factor(l, j);
    }
    dst_apply<Q>(v);
#pragma unroll
    for (int j = 0; j < L; ++j) Xs[l * RS + NP * j + part] = v[j];
  }
  __syncthreads();
  // ---- pass 2: columns, y transform, eigenvalue reciprocals, inverse y transform
  if (act) {
    const double* dc = dinv + l;  // column l (x mode) of the [N4][N4] table
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = Xs[j * RS + NP * l + part];
    dst_apply<Q>(v);
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] *= __ldg(dc + j * N4);
    dst_apply<Q>(v);
#pragma unroll
    for (int j = 0; j < L; ++j) Xs[j * RS + NP * l + part] = v[j];
  }
  __syncthreads();
  // ---- pass 3: rows, inverse x transform
  if (act) {
#pragma unroll
    for (int j = 0; j < L; ++j) v[j] = Xs[l * RS + NP * j + part];
    dst_apply<Q>(v);
#pragma unroll
    for (int j = 0; j < L; ++j) Xs[l * RS + NP * j + part] = v[j];
  }
  __syncthreads();
  // ---- epilogue (thread = (row group, column): column terms in registers)
  if (crg < NG) {
    const typename BoxOut<S>::ColTerms ct = io.col_terms(cq);
    int sl = 0, r = crg;
    for (int idx = crg; idx < nslot * L; idx += NG, r += NG) {
      if (r >= L) {
        r -= L;
        ++sl;
      }
      const double* Xe = X(sl);
      S acc;
      if constexpr (NP == 2) acc = *reinterpret_cast<const double2*>(&Xe[r * RS + 2 * cq]);
      else acc = Xe[r * RS + cq];
      io.put_col(base, y, ovl, cbase, sl, b0 + sl, r, cq, ct, acc);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Edge boxes (MP-2): one axis is the middle pencil (DST, length 4Q - 1), the other a
// Sommerfeld-end class (T = tridiag(-1, 2, -1)/h^2 with the boundary diagonal
// 1/h^2 - ik/h, W = I with 1/2 at the boundary node, discretization.py:136-148).  A sine
// transform along the middle axis decouples the box into one complex tridiagonal system per
// sine mode mu along the other axis,  K_mu = T_e + (lambda_mu - k^2) W_e,  solved with the
// plan's LU factors (Thomas; every pivot of every BASELINE config is >= 0.047/h^2 in modulus,
// checked at plan creation): 2 transforms of 275 + 76 operations per line and ~12 multiply-adds
// per tridiagonal row instead of four dense complex products.
// ---------------------------------------------------------------------------------------
constexpr int EDGE_NB = 2;     // slots (right-hand sides) per CTA
constexpr int EDGE_NTH = 160;  // >= 2 * 35 * EDGE_NB lines
constexpr size_t EDGE_XB = 35 * 35 * 16 + 64;  // bytes of a slot tile (<= 35 x 35 complex)

template <int Q>
__global__ void __launch_bounds__(EDGE_NTH, 2)
    local_edge_kernel(const double2* __restrict__ x, const double2* __restrict__ base, double2* __restrict__ y,
                      double2* __restrict__ ovl, const int* __restrict__ boxes, const double2* __restrict__ tri,
                      const int* __restrict__ class_tri, LocalArgs a, int batch, double e_off) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  constexpr int LD = 4 * Q - 1, N4 = 4 * Q, NB = EDGE_NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  auto X = [&](int s) { return reinterpret_cast<double*>(smem_raw + (size_t)s * EDGE_XB); };
  const bool cbase = base && a.coarse_base;
  double2* rx = reinterpret_cast<double2*>(smem_raw + (size_t)NB * EDGE_XB);
  int* meta = reinterpret_cast<int*>(smem_raw + (size_t)NB * EDGE_XB + (cbase ? (size_t)NB * WIN * 40 * 16 : 0));

  const int sid = boxes[blockIdx.x];
  const int ay = sid / a.p, ax = sid % a.p;
  const int nu = a.nu;
  const size_t N = (size_t)nu * nu;
  const int b0 = blockIdx.y * NB;
  const int nslot = min(NB, batch - b0);
  const int ty_cls = class_tri[a.box_class[ay]];
  const bool ty = ty_cls >= 0;  // the tridiagonal axis is y (else x)
  const int ct = ty ? ty_cls : class_tri[a.box_class[ax]];
  const int Ly = a.box_len[ay], Lx = a.box_len[ax];
  const int LT = ty ? Ly : Lx;
  const int RS = 2 * Lx;
  const BoxOut<double2> io(a, meta, rx, ay, ax, Ly, Lx);
  const int y0 = io.y0, x0 = io.x0;
  for (int e = threadIdx.x; e < nslot * Ly * Lx; e += EDGE_NTH) {
    const int s = e / (Ly * Lx), r = (e % (Ly * Lx)) / Lx, q = e % Lx;
    cp_async16(&X(s)[r * RS + 2 * q], x + (size_t)(b0 + s) * N + (size_t)(y0 + r) * nu + x0 + q, true);
  }
  cp_commit();
  io.init_meta(EDGE_NTH);
  if (cbase) io.init_rx(base, b0, nslot, EDGE_NTH);
  cp_wait<0>();
  __syncthreads();
  // element (u along the tridiagonal axis, j along the sine axis) of a slot, in doubles
  auto at = [&](int u, int j) { return ty ? u * RS + 2 * j : j * RS + 2 * u; };
  const int t = threadIdx.x;
  // ---- sine transform along the middle axis: one thread per (slot, line u, part)
  auto sine_pass = [&](bool first) {
    const int s = t / (2 * LT), it = t % (2 * LT), u = it >> 1, part = it & 1;
    if (t < nslot * 2 * LT) {
      double* Xs = X(s);
      double v[LD];
      const bool wb = first && a.weighted && a.wbs;
#pragma unroll
      for (int j = 0; j < LD; ++j) {
        v[j] = Xs[at(u, j) + part];
        if (wb) v[j] *= ty ? io.wbs_factor(u, j) : io.wbs_factor(j, u);
      }
      dst_apply<Q>(v);
#pragma unroll
      for (int j = 0; j < LD; ++j) Xs[at(u, j) + part] = v[j];
    }
  };
  sine_pass(true);
  __syncthreads();
  // ---- per sine mode: K_mu y = (2/N) x along the tridiagonal axis (LU: l_i, 1/d_i)
  if (t < nslot * LD) {
    const int s = t / LD, mu = t % LD;
    double* Xs = X(s);
    const double2* lt = tri + ((size_t)ct * 2 * DML) * N4 + mu;  // l_i at lt[i N4]
    const double2* dt = lt + (size_t)DML * N4;                    // 1/d_i at dt[i N4]
    const double al = 2.0 / N4;
    double2 g = scale(*reinterpret_cast<const double2*>(&Xs[at(0, mu)]), al);
    *reinterpret_cast<double2*>(&Xs[at(0, mu)]) = g;
    for (int i = 1; i < LT; ++i) {
      const double2 r = scale(*reinterpret_cast<const double2*>(&Xs[at(i, mu)]), al);
      g = fms_(__ldg(lt + (size_t)i * N4), g, r);
      *reinterpret_cast<double2*>(&Xs[at(i, mu)]) = g;
    }
    double2 xv = mul(g, __ldg(dt + (size_t)(LT - 1) * N4));
    *reinterpret_cast<double2*>(&Xs[at(LT - 1, mu)]) = xv;
    for (int i = LT - 2; i >= 0; --i) {
      const double2 gi = *reinterpret_cast<const double2*>(&Xs[at(i, mu)]);
      xv = mul(fma_(-e_off, xv, gi), __ldg(dt + (size_t)i * N4));
      *reinterpret_cast<double2*>(&Xs[at(i, mu)]) = xv;
    }
  }
  __syncthreads();
  sine_pass(false);
  __syncthreads();
  for (int e = threadIdx.x; e < nslot * Ly * Lx; e += EDGE_NTH) {
    const int sl = e / (Ly * Lx), r = (e % (Ly * Lx)) / Lx, q = e % Lx;
    const double2 acc = *reinterpret_cast<const double2*>(&X(sl)[r * RS + 2 * q]);
    io.put(base, y, ovl, cbase, sl, b0 + sl, r, q, acc);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_dst() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HELM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    HELM_CHECK(p != nullptr && q == cudaDriverEntryPointSuccess, "driver entry point missing: cuTensorMapEncodeTiled");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
static bool tma_on_dst() {  // HELM_TMA=0: cp.async box loads (A/B)
  static const bool on = [] {
    const char* e = getenv("HELM_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool tma_window_on() {  // HELM_TMA_WINDOW=0: the coarse window by per-thread loads (A/B)
  static const bool on = [] {
    const char* e = getenv("HELM_TMA_WINDOW");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename S, int Q>
static void dst_launch(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st) {
  constexpr int NP = Sc<S>::cplx ? 2 : 1;
  using G = DstGeo<NP, Q>;
  const PlanDev& d = P->dev;
  upload_dst_tables();
  const bool cbase = base && a.coarse_base;
  const size_t smem = G::smem(cbase);
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(local_dst_kernel<S, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)G::smem(true)));
    attr = true;
  }
  TmaDst tma;
  std::memset(&tma, 0, sizeof(tma));
  if (NP == 2 && tma_on_dst()) {
    const cuuint64_t dims[3] = {(cuuint64_t)2 * a.nu, (cuuint64_t)a.nu, (cuuint64_t)batch};
    const cuuint64_t strides[2] = {(cuuint64_t)a.nu * 16, (cuuint64_t)a.nu * a.nu * 16};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * G::L), (cuuint32_t)G::L, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode_tiled_dst()(&tma.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<S*>(x), dims,
                                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HELM_CHECK(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for the fast-sine box load");
    tma.on = 1;
    if (cbase && G::L >= WIN + 1 && tma_window_on()) {
      const cuuint64_t cdims[3] = {(cuuint64_t)2 * a.m0, (cuuint64_t)a.m0, (cuuint64_t)batch};
      const cuuint64_t cstrides[2] = {(cuuint64_t)a.m0 * 16, (cuuint64_t)a.m0 * a.m0 * 16};
      const cuuint32_t cbox[3] = {(cuuint32_t)(2 * WIN), (cuuint32_t)WIN, 1};
      const CUresult rc = encode_tiled_dst()(&tma.cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<S*>(base),
                                             cdims, cstrides, cbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      HELM_CHECK(rc == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed for the coarse window load");
      tma.con = 1;
    }
  }
  dim3 grd(d.n_dst, (batch + G::NB - 1) / G::NB);
  launch_pdl(local_dst_kernel<S, Q>, grd, G::NTH, smem, st, x, base, y, ovl, (const int*)d.box_dst,
             (const double*)d.dst_inv, a, batch, tma);
  HELM_LAUNCH_CHECK();
}

template <int Q>
static void edge_launch(const helm_plan* P, const double2* x, const double2* base, double2* y, double2* ovl,
                        const LocalArgs& a, int batch, cudaStream_t st) {
  const PlanDev& d = P->dev;
  upload_dst_tables();
  const bool cbase = base && a.coarse_base;
  const size_t smem = (size_t)EDGE_NB * EDGE_XB + (cbase ? (size_t)EDGE_NB * WIN * 40 * 16 : 0) + 8 * DML * 4;
  static bool attr = false;
  if (!attr) {
    HELM_CUDA(cudaFuncSetAttribute(local_edge_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((size_t)EDGE_NB * EDGE_XB + (size_t)EDGE_NB * WIN * 40 * 16 + 8 * DML * 4)));
    attr = true;
  }
  dim3 grd(d.n_edge, (batch + EDGE_NB - 1) / EDGE_NB);
  launch_pdl(local_edge_kernel<Q>, grd, EDGE_NTH, smem, st, x, base, y, ovl, (const int*)d.box_edge,
             (const double2*)d.edge_tri, (const int*)d.class_tri, a, batch, -P->geo.inv_h2);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void launch_local_edge(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st) {
  const PlanDev& d = P->dev;
  if constexpr (Sc<S>::cplx) {
    if (d.n_edge == 0) return;
    if (d.dst_q == 9) edge_launch<9>(P, x, base, y, ovl, a, batch, st);
    else if (d.dst_q == 5) edge_launch<5>(P, x, base, y, ovl, a, batch, st);
    else HELM_CHECK(false, "edge boxes need a sine axis of L = 19 or 35");
  } else {
    HELM_CHECK(d.n_edge == 0, "edge boxes are MP-2 only");
  }
}
template void launch_local_edge<double>(const helm_plan*, const double*, const double*, double*, double*,
                                        const LocalArgs&, int, cudaStream_t);
template void launch_local_edge<double2>(const helm_plan*, const double2*, const double2*, double2*, double2*,
                                         const LocalArgs&, int, cudaStream_t);

template <typename S>
void launch_local_dst(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                      cudaStream_t st) {
  const PlanDev& d = P->dev;
  if (d.n_dst == 0) return;
  if (d.dst_q == 9) dst_launch<S, 9>(P, x, base, y, ovl, a, batch, st);
  else if (d.dst_q == 5) dst_launch<S, 5>(P, x, base, y, ovl, a, batch, st);
  else HELM_CHECK(false, "fast-sine boxes need L = 19 or 35");
}

template void launch_local_dst<double>(const helm_plan*, const double*, const double*, double*, double*,
                                       const LocalArgs&, int, cudaStream_t);
template void launch_local_dst<double2>(const helm_plan*, const double2*, const double2*, double2*, double2*,
                                        const LocalArgs&, int, cudaStream_t);

}  // namespace helm
