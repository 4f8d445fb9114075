// K2 (Bezier restriction R0), K3 (prolongation R0^T) and K3+K1 (SHS2 deflation
// d = x - A R0^T c) as register sweeps.
//
// Reference semantics (coarse.py:102-139, applied at coarse.py:174 and schwarz.py:87-88):
//   R0 = P (x) P, P the (1,4,6,4,1)/8 stride-2 Bezier restriction; taps outside the
//   unknown set are dropped.  Fine unknown u and coarse unknown U are tied by
//   u = 2U + off + d, off = 0 (Sommerfeld) / 1 (Dirichlet), |d| <= 2.
//
// Layout of the work: a lane owns one aligned pair of fine columns (2P, 2P+1) -- one
// coalesced 32-byte (complex128) or 16-byte (fp64) access per row -- and a warp sweeps a
// strip of rows.  The column taps of the 5-wide (R0) or 3-wide (R0^T) stencils come
// from the neighbouring lanes by shuffles, so no shared memory is touched; the row taps
// live in a small register ring that advances two fine rows per coarse row.  Edge lanes
// of a warp only feed their neighbours (R0, R0^T: one lane per side, 30 output pairs
// per warp; the deflation needs z one column further out: two lanes per side, 28).
// Loads of the next step are issued before the current one is reduced.  Every fine
// value is read once from HBM, every output written once; summation orders match the
// reference definitions tap by tap (x pass, then y pass).
#include "common.cuh"

namespace helm {

namespace {

// (1,4,6,4,1)/8
__device__ __forceinline__ constexpr double rw(int d) { return d == 2 ? 0.75 : (d == 1 || d == 3) ? 0.5 : 0.125; }

template <typename S> __device__ __forceinline__ S shfl_up1(S v);
template <> __device__ __forceinline__ double shfl_up1<double>(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <> __device__ __forceinline__ double2 shfl_up1<double2>(double2 v) {
  return mk(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
template <typename S> __device__ __forceinline__ S shfl_dn1(S v);
template <> __device__ __forceinline__ double shfl_dn1<double>(double v) {
  return __shfl_down_sync(0xffffffffu, v, 1);
}
template <> __device__ __forceinline__ double2 shfl_dn1<double2>(double2 v) {
  return mk(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}

template <typename S> struct Pr {
  S a, b;  // fine columns 2P, 2P+1
};

template <typename S>
__device__ __forceinline__ Pr<S> load_pair(const S* __restrict__ base, int nu, int u, int P, bool want = true) {
  Pr<S> r{Sc<S>::zero(), Sc<S>::zero()};
  if (want && u >= 0 && u < nu) {
    const S* row = base + (size_t)u * nu;
    const int c0 = 2 * P;
    if (c0 >= 0 && c0 < nu) r.a = row[c0];
    if (c0 + 1 >= 0 && c0 + 1 < nu) r.b = row[c0 + 1];
  }
  return r;
}

// x pass of R0 for coarse column P at one fine row: taps 2P+off-2 .. 2P+off+2 taken from
// the window (left pair, own pair, right pair)
template <int off, typename S>
__device__ __forceinline__ S rx_pass(const Pr<S>& p) {
  const S l0 = shfl_up1(p.a), l1 = shfl_up1(p.b), r0 = shfl_dn1(p.a), r1 = shfl_dn1(p.b);
  const S win[6] = {l0, l1, p.a, p.b, r0, r1};
  S t = Sc<S>::zero();
#pragma unroll
  for (int d = 0; d < 5; ++d) t = fma_(rw(d), win[d + off], t);
  return t;
}

// R0^T along x at one coarse row: the values at fine columns 2P, 2P+1 from coarse
// columns P-1, P, P+1 (v = c[P]; neighbours by shuffle).  t = col - off:
// even t -> (1, 6, 1)/8 on t/2 - 1, t/2, t/2 + 1; odd t -> (1, 1)/2 on (t-1)/2, (t+1)/2.
template <int off, typename S>
__device__ __forceinline__ Pr<S> px_pass(S v) {
  const S l = shfl_up1(v), r = shfl_dn1(v);
  Pr<S> o;
  if constexpr (off == 0) {  // col 2P: t even (P-1, P, P+1); col 2P+1: t odd (P, P+1)
    o.a = fma_(0.125, r, fma_(0.75, v, fma_(0.125, l, Sc<S>::zero())));
    o.b = fma_(0.5, r, fma_(0.5, v, Sc<S>::zero()));
  } else {  // col 2P: t = 2P-1 odd (P-1, P); col 2P+1: t = 2P even (P-1, P, P+1)
    o.a = fma_(0.5, v, fma_(0.5, l, Sc<S>::zero()));
    o.b = fma_(0.125, r, fma_(0.75, v, fma_(0.125, l, Sc<S>::zero())));
  }
  return o;
}
// the same combination along y: fine rows 2R, 2R+1 from the x-prolongated coarse rows
// R-1, R, R+1 (pm, p0, pp)
template <int off, typename S>
__device__ __forceinline__ void py_pass(const Pr<S>& pm, const Pr<S>& p0, const Pr<S>& pp, Pr<S>& r0, Pr<S>& r1) {
  auto three = [](S m, S c, S p) { return fma_(0.125, p, fma_(0.75, c, fma_(0.125, m, Sc<S>::zero()))); };
  auto two = [](S c, S p) { return fma_(0.5, p, fma_(0.5, c, Sc<S>::zero())); };
  if constexpr (off == 0) {
    r0 = {three(pm.a, p0.a, pp.a), three(pm.b, p0.b, pp.b)};
    r1 = {two(p0.a, pp.a), two(p0.b, pp.b)};
  } else {
    r0 = {two(pm.a, p0.a), two(pm.b, p0.b)};
    r1 = {three(pm.a, p0.a, pp.a), three(pm.b, p0.b, pp.b)};
  }
}

__device__ __forceinline__ int warp_global() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }

}  // namespace

// ---------------------------------------------------------------------------------
// R0: c = R0 x.  Warp (column group g, strip s): lane l owns coarse column
// P = 30 g - 1 + l (lanes 1..30 store), coarse rows [s*US, (s+1)*US).
// ---------------------------------------------------------------------------------
template <typename S, int off>
__global__ void __launch_bounds__(256) restrict_sweep_kernel(const S* __restrict__ x, S* __restrict__ c, Geo g,
                                                             int ngroups, int US) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int lane = threadIdx.x & 31;
  const int wg = warp_global();
  const int grp = wg % ngroups, strip = wg / ngroups;
  const int m0 = g.m0, nu = g.nu;
  const int U0 = strip * US;
  if (U0 >= m0) return;
  const int U1 = min(U0 + US, m0);
  const int P = 30 * grp - 1 + lane;
  const bool store = lane >= 1 && lane <= 30 && P >= 0 && P < m0;
  const S* xb = x + (size_t)blockIdx.y * nu * nu;
  S* cb = c + (size_t)blockIdx.y * m0 * m0;
  // ring of x-pass rows 2U+off-2 .. 2U+off+2
  S t[5];
  const int u0 = 2 * U0 + off - 2;
  {
    Pr<S> p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = load_pair(xb, nu, u0 + i, P);
#pragma unroll
    for (int i = 0; i < 4; ++i) t[i] = rx_pass<off>(p[i]);
  }
  Pr<S> n0 = load_pair(xb, nu, u0 + 4, P), n1 = load_pair(xb, nu, u0 + 5, P);
  for (int U = U0; U < U1; ++U) {
    const Pr<S> c0 = n0, c1 = n1;
    if (U + 1 < U1) {  // next step's rows in flight while this one reduces
      n0 = load_pair(xb, nu, 2 * U + off + 4, P);
      n1 = load_pair(xb, nu, 2 * U + off + 5, P);
    }
    t[4] = rx_pass<off>(c0);
    S acc = Sc<S>::zero();
#pragma unroll
    for (int d = 0; d < 5; ++d) acc = fma_(rw(d), t[d], acc);
    if (store) cb[(size_t)U * m0 + P] = acc;
    t[0] = t[2];
    t[1] = t[3];
    t[2] = t[4];
    t[3] = rx_pass<off>(c1);
  }
}

// ---------------------------------------------------------------------------------
// R0^T: z = R0^T c.  Lane l owns fine columns (2P, 2P+1), P = 30 g - 1 + l (lanes 1..30
// store); the warp sweeps fine row pairs (2R, 2R+1), R in [s*RS, (s+1)*RS).
// ---------------------------------------------------------------------------------
template <typename S>
__device__ __forceinline__ S coarse_at(const S* __restrict__ cb, int m0, int U, int P) {
  return (U >= 0 && U < m0 && P >= 0 && P < m0) ? cb[(size_t)U * m0 + P] : Sc<S>::zero();
}

template <typename S, int off>
__global__ void __launch_bounds__(256) prolong_sweep_kernel(const S* __restrict__ c, S* __restrict__ z, Geo g,
                                                            int ngroups, int RS) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int lane = threadIdx.x & 31;
  const int wg = warp_global();
  const int grp = wg % ngroups, strip = wg / ngroups;
  const int m0 = g.m0, nu = g.nu;
  const int npairs = (nu + 1) / 2;
  const int R0 = strip * RS;
  if (R0 >= npairs) return;
  const int R1 = min(R0 + RS, npairs);
  const int P = 30 * grp - 1 + lane;
  const bool store = lane >= 1 && lane <= 30 && P >= 0 && 2 * P < nu;
  const S* cb = c + (size_t)blockIdx.y * m0 * m0;
  S* zb = z + (size_t)blockIdx.y * nu * nu;
  Pr<S> pm = px_pass<off>(coarse_at(cb, m0, R0 - 1, P));
  Pr<S> p0 = px_pass<off>(coarse_at(cb, m0, R0, P));
  S nv = coarse_at(cb, m0, R0 + 1, P);
  for (int R = R0; R < R1; ++R) {
    const S cv = nv;
    if (R + 1 < R1) nv = coarse_at(cb, m0, R + 2, P);
    const Pr<S> pp = px_pass<off>(cv);
    Pr<S> r0, r1;
    py_pass<off>(pm, p0, pp, r0, r1);
    if (store) {
      const int col = 2 * P;
      S* row0 = zb + (size_t)(2 * R) * nu;
      row0[col] = r0.a;
      if (col + 1 < nu) row0[col + 1] = r0.b;
      if (2 * R + 1 < nu) {
        row0[nu + col] = r1.a;
        if (col + 1 < nu) row0[nu + col + 1] = r1.b;
      }
    }
    pm = p0;
    p0 = pp;
  }
}

// ---------------------------------------------------------------------------------
// K3 + K1 (SHS2): d = x - A z with z = R0^T c never written.  Lane l owns fine columns
// (2P, 2P+1), P = 28 g - 2 + l (lanes 2..29 store).  Step R prolongates fine rows 2R,
// 2R+1 and emits d on rows 2R-1, 2R (their stencils need z rows 2R-2 .. 2R+1).
// ---------------------------------------------------------------------------------
template <typename S, int off>
__global__ void __launch_bounds__(256, 2) prolong_deflate_sweep_kernel(const S* __restrict__ c,
                                                                    const S* __restrict__ x, S* __restrict__ z,
                                                                    S* __restrict__ d, Geo g, int ngroups, int RS) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const int lane = threadIdx.x & 31;
  const int wg = warp_global();
  const int grp = wg % ngroups, strip = wg / ngroups;
  const int m0 = g.m0, nu = g.nu;
  const int nsteps = (nu + 1) / 2 + 1;  // the last step emits row 2R-1 = nu-1 (or nu-2)
  const int R0 = strip * RS;
  if (R0 >= nsteps) return;
  const int R1 = min(R0 + RS, nsteps);
  const int P = 28 * grp - 2 + lane;
  const int col = 2 * P;
  const bool store = lane >= 2 && lane <= 29 && P >= 0 && col < nu;
  const S* cb = c + (size_t)blockIdx.y * m0 * m0;
  const S* xb = x + (size_t)blockIdx.y * nu * nu;
  S* db = d + (size_t)blockIdx.y * nu * nu;
  const double dc = 4.0 * g.inv_h2 - g.k2;
  S* zb = z ? z + (size_t)blockIdx.y * nu * nu : nullptr;
  // z at a fine row, zero off the unknown set (the stencil drops those neighbours)
  auto zrow_ok = [&](int u, Pr<S> v) {
    if (u < 0 || u >= nu) v.a = v.b = Sc<S>::zero();
    if (col < 0 || col >= nu) v.a = Sc<S>::zero();
    if (col + 1 < 0 || col + 1 >= nu) v.b = Sc<S>::zero();
    return v;
  };
  // prologue: z rows 2R0-2, 2R0-1 (pair R0-1) need x-prolongated coarse rows R0-2 .. R0
  Pr<S> pa = px_pass<off>(coarse_at(cb, m0, R0 - 2, P));
  Pr<S> pm = px_pass<off>(coarse_at(cb, m0, R0 - 1, P));
  Pr<S> p0 = px_pass<off>(coarse_at(cb, m0, R0, P));
  Pr<S> zm2, zm1;  // z rows 2R-2, 2R-1
  py_pass<off>(pa, pm, p0, zm2, zm1);
  zm2 = zrow_ok(2 * R0 - 2, zm2);
  zm1 = zrow_ok(2 * R0 - 1, zm1);
  S nv = coarse_at(cb, m0, R0 + 1, P);
  Pr<S> xa = load_pair(xb, nu, 2 * R0 - 1, P, store), xc = load_pair(xb, nu, 2 * R0, P, store);
  for (int R = R0; R < R1; ++R) {
    const S cv = nv;
    const Pr<S> xr1 = xa, xr2 = xc;  // x on rows 2R-1, 2R
    if (R + 1 < R1) {
      nv = coarse_at(cb, m0, R + 2, P);
      xa = load_pair(xb, nu, 2 * R + 1, P, store);
      xc = load_pair(xb, nu, 2 * R + 2, P, store);
    }
    const Pr<S> pp = px_pass<off>(cv);
    Pr<S> z0, z1;  // rows 2R, 2R+1
    py_pass<off>(pm, p0, pp, z0, z1);
    z0 = zrow_ok(2 * R, z0);
    z1 = zrow_ok(2 * R + 1, z1);
    // row 2R-1: centre zm1, up zm2, down z0;  row 2R: centre z0, up zm1, down z1
    const S lA = shfl_up1(zm1.b), rA = shfl_dn1(zm1.a);
    const S lB = shfl_up1(z0.b), rB = shfl_dn1(z0.a);
    if (store) {
      const int ua = 2 * R - 1, ub = 2 * R;
      // d = x - A z; interior rows of A are (4/h^2 - k^2) z_p - (1/h^2) (sum of the 4 neighbours)
      auto defl = [&](S xv, int ix, int iy, S cz, S up, S dn, S lf, S rt) {
        if (iy > 0 && iy < nu - 1 && ix > 0 && ix < nu - 1)
          return fma_(g.inv_h2, add(add(up, dn), add(lf, rt)), fma_(-dc, cz, xv));
        return sub(xv, stencil_point<S>(g, ix, iy, cz, up, dn, lf, rt));
      };
      if (ua >= 0 && ua < nu) {
        S* dr = db + (size_t)ua * nu;
        dr[col] = defl(xr1.a, col, ua, zm1.a, zm2.a, z0.a, lA, zm1.b);
        if (col + 1 < nu) dr[col + 1] = defl(xr1.b, col + 1, ua, zm1.b, zm2.b, z0.b, zm1.a, rA);
        if (zb) {
          zb[(size_t)ua * nu + col] = zm1.a;
          if (col + 1 < nu) zb[(size_t)ua * nu + col + 1] = zm1.b;
        }
      }
      if (ub < nu) {
        S* dr = db + (size_t)ub * nu;
        dr[col] = defl(xr2.a, col, ub, z0.a, zm1.a, z1.a, lB, z0.b);
        if (col + 1 < nu) dr[col + 1] = defl(xr2.b, col + 1, ub, z0.b, zm1.b, z1.b, z0.a, rB);
        if (zb) {
          zb[(size_t)ub * nu + col] = z0.a;
          if (col + 1 < nu) zb[(size_t)ub * nu + col + 1] = z0.b;
        }
      }
    }
    zm2 = z0;
    zm1 = z1;
    pm = p0;
    p0 = pp;
  }
}

// ---------------------------------------------------------------------------------
// launchers: strips sized so that a batch-1 launch still has ~16 warps per SM
// ---------------------------------------------------------------------------------
static int strip_len(int rows, int groups, int batch) {
  const long target_warps = 148L * 16;
  int s = 64;
  while (s > 8 && (long)groups * ((rows + s - 1) / s) * batch < target_warps) s /= 2;
  return s;
}

template <typename S>
void launch_restrict(const Geo& g, const S* x, S* c, int batch, cudaStream_t st) {
  const int groups = (g.m0 + 29) / 30;
  const int US = strip_len(g.m0, groups, batch);
  const int warps = groups * ((g.m0 + US - 1) / US);
  dim3 grd((warps + 7) / 8, batch);
  if (g.off)
    launch_pdl(restrict_sweep_kernel<S, 1>, grd, 256, 0, st, x, c, g, groups, US);
  else
    launch_pdl(restrict_sweep_kernel<S, 0>, grd, 256, 0, st, x, c, g, groups, US);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void launch_prolong(const Geo& g, const S* c, S* z, int batch, cudaStream_t st) {
  const int npairs = (g.nu + 1) / 2;
  const int groups = (npairs + 29) / 30;
  const int RS = strip_len(npairs, groups, batch);
  const int warps = groups * ((npairs + RS - 1) / RS);
  dim3 grd((warps + 7) / 8, batch);
  if (g.off)
    launch_pdl(prolong_sweep_kernel<S, 1>, grd, 256, 0, st, c, z, g, groups, RS);
  else
    launch_pdl(prolong_sweep_kernel<S, 0>, grd, 256, 0, st, c, z, g, groups, RS);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void launch_prolong_deflate(const Geo& g, const S* c, const S* x, S* z, S* d, int batch, cudaStream_t st) {
  const int npairs = (g.nu + 1) / 2;
  const int nsteps = npairs + 1;
  const int groups = (npairs + 27) / 28;
  const int RS = strip_len(nsteps, groups, batch);
  const int warps = groups * ((nsteps + RS - 1) / RS);
  dim3 grd((warps + 7) / 8, batch);
  if (g.off)
    launch_pdl(prolong_deflate_sweep_kernel<S, 1>, grd, 256, 0, st, c, x, z, d, g, groups, RS);
  else
    launch_pdl(prolong_deflate_sweep_kernel<S, 0>, grd, 256, 0, st, c, x, z, d, g, groups, RS);
  HELM_LAUNCH_CHECK();
}

#define HELM_INST(S)                                                                           \
  template void launch_restrict<S>(const Geo&, const S*, S*, int, cudaStream_t);               \
  template void launch_prolong<S>(const Geo&, const S*, S*, int, cudaStream_t);                \
  template void launch_prolong_deflate<S>(const Geo&, const S*, const S*, S*, S*, int, cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
