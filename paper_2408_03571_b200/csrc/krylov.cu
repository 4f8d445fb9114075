// K6/K7: the Arnoldi step and Givens update of unrestarted GMRES
// (reference gmres.py:108-148: MGS + one conditional re-orthogonalisation pass,
// complex Givens rotations, residual estimate |g[j+1]| / ||r0||).
//
// B200 form: classical Gram-Schmidt run twice (CGS2) in three sweeps of the
// basis (the second pass's dots ride on the first pass's update sweep, the
// norm comes from Pythagoras, the Givens update runs in the reducing block;
// details below).  In exact arithmetic
// CGS2 equals MGS + re-orthogonalisation; numerically both keep the basis
// orthogonal to working precision, which is what fixes the iteration count.
// H, the rotations and g stay on the device; the host reads one estimate.
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace helm {

constexpr int KB = 256;        // threads per block
constexpr int KNB = 4 * 148;   // blocks of the streaming Krylov kernels (4 per SM)
constexpr int PB = 8 * 148;    // capacity of the per-block partial-sum arrays

// w <- w + sign * sum_i h_i V_i ; optionally norm2 partial of the result per block
template <typename S>
__global__ void __launch_bounds__(KB) update_kernel(S* __restrict__ w, const S* __restrict__ V, int nvec,
                                                    size_t ldv, const S* __restrict__ h, double sign, size_t N,
                                                    int from_zero, double* __restrict__ npart) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  S* hs = reinterpret_cast<S*>(sraw);
  __shared__ double nred[KB / 32];
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) hs[i] = scale(h[i], sign);
  __syncthreads();
  double nrm = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += stride) {
    S acc = from_zero ? Sc<S>::zero() : w[n];
    int i = 0;
    for (; i + 4 <= nvec; i += 4) {
      const S v0 = V[(size_t)i * ldv + n], v1 = V[(size_t)(i + 1) * ldv + n];
      const S v2 = V[(size_t)(i + 2) * ldv + n], v3 = V[(size_t)(i + 3) * ldv + n];
      acc = fma_(hs[i], v0, acc);
      acc = fma_(hs[i + 1], v1, acc);
      acc = fma_(hs[i + 2], v2, acc);
      acc = fma_(hs[i + 3], v3, acc);
    }
    for (; i < nvec; ++i) acc = fma_(hs[i], V[(size_t)i * ldv + n], acc);
    w[n] = acc;
    nrm += abs2(acc);
  }
  if (npart) {
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) nred[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < KB / 32; ++q) s += nred[q];
      npart[blockIdx.x] = s;
    }
  }
}

template <typename S>
__global__ void __launch_bounds__(KB) norm2_kernel(const S* __restrict__ x, size_t N, double* __restrict__ npart) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  __shared__ double nred[KB / 32];
  double nrm = 0.0;
  for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += (size_t)gridDim.x * blockDim.x)
    nrm += abs2(x[n]);
  nrm = warp_sum(nrm);
  if ((threadIdx.x & 31) == 0) nred[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < KB / 32; ++q) s += nred[q];
    npart[blockIdx.x] = s;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ npart, int nb, double* __restrict__ out) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) s += npart[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}

template <typename S>
__global__ void scale_kernel(S* __restrict__ x, const S* __restrict__ src, const double* __restrict__ s, int invert,
                             size_t N) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  const double f = invert ? 1.0 / s[0] : s[0];
  if (!invert && f == 0.0) return;  // breakdown: leave the vector alone
  for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += (size_t)gridDim.x * blockDim.x)
    x[n] = scale(src[n], f);
}

// --- y = R^{-1} g with R = H[:j+1, :j+1] upper triangular (gmres.py:98-103) -----
template <typename S>
__global__ void backsolve_kernel(const S* __restrict__ H, int ldh, int j, const S* __restrict__ g, S* __restrict__ y) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  S* rhs = reinterpret_cast<S*>(sraw);
  __shared__ S yi_s;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) rhs[i] = g[i];
  __syncthreads();
  for (int i = j; i >= 0; --i) {
    if (threadIdx.x == 0) {
      const S d = H[(size_t)i * ldh + i];
      // singular R: the reference falls back to lstsq; a zero component is used here
      yi_s = abs2(d) == 0.0 ? Sc<S>::zero() : div_(rhs[i], d);
      y[i] = yi_s;
    }
    __syncthreads();
    const S yi = yi_s;
    for (int k = threadIdx.x; k < i; k += blockDim.x) rhs[k] = fms_(H[(size_t)k * ldh + i], yi, rhs[k]);
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// CGS2 in three sweeps of the basis (B_o = (3(j+1) + 5) N s of HBM traffic)
//
//   K1  h1 = V^H w                                     (sweep 1: V, w)
//   K2  w' = w - V h1 (stored), h2 = V^H w', ||w'||^2    (sweep 2: V from HBM for the
//       update, the second read of the same chunk for the dots hits L2)
//       last block: h2, ||w''|| = sqrt(||w'||^2 - ||h2||^2) (Pythagoras: w'' = w' - V h2
//       with V^H w' = h2), H[:, j] = h1 + h2, breakdown test, 1/||w''||, optional Givens
//   K3  V[j+1] = (w' - V h2) / ||w''||                  (sweep 3)
// Block partials are combined by the last block to finish (threadfence + counter), in a
// fixed order: the result is deterministic.
// ----------------------------------------------------------------------------
constexpr int CG = 8;  // vectors per reduction group

// 8 complex/real values per lane -> lane l holds the warp total of value (l >> 2) & 7
template <typename S> __device__ __forceinline__ S shfl_x(S v, int o);
template <> __device__ __forceinline__ double shfl_x<double>(double v, int o) {
  return __shfl_xor_sync(0xffffffffu, v, o);
}
template <> __device__ __forceinline__ double2 shfl_x<double2>(double2 v, int o) {
  return mk(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}
template <typename S> __device__ __forceinline__ S reduce8(const S (&v)[CG], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  S u[4], t[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) u[q] = add(b4 ? v[q + 4] : v[q], shfl_x(b4 ? v[q] : v[q + 4], 16));
#pragma unroll
  for (int q = 0; q < 2; ++q) t[q] = add(b3 ? u[q + 2] : u[q], shfl_x(b3 ? u[q] : u[q + 2], 8));
  S s = add(b2 ? t[1] : t[0], shfl_x(b2 ? t[0] : t[1], 4));
  s = add(s, shfl_x(s, 2));
  s = add(s, shfl_x(s, 1));
  return s;
}

// scratch layout (fixed offsets first: the counters must stay put and start at zero)
//   [count 2 x u32 | pad][scal 8 doubles][npart PB doubles][h1 nv S][h2 nv S][partial nv x PB S]
struct CgsScratch {
  unsigned* count; // [2]
  double* scal;    // [8]
  double* npart;   // [PB]
  void* h1;        // [nvec] S
  void* h2;        // [nvec] S
  void* partial;   // [nvec][<= PB] S
};
size_t krylov_scratch_bytes(int max_vec) {
  const size_t nv = (size_t)((max_vec + CG - 1) / CG) * CG;
  return 64 + 8 * sizeof(double) + PB * sizeof(double) + 2 * nv * sizeof(double2) + nv * PB * sizeof(double2);
}
static CgsScratch carve(void* scratch, int max_vec) {
  const size_t nv = (size_t)((max_vec + CG - 1) / CG) * CG;
  char* p = (char*)scratch;
  CgsScratch k;
  k.count = (unsigned*)p;
  p += 64;
  k.scal = (double*)p;
  p += 8 * sizeof(double);
  k.npart = (double*)p;
  p += PB * sizeof(double);
  k.h1 = p;
  p += nv * sizeof(double2);
  k.h2 = p;
  p += nv * sizeof(double2);
  k.partial = p;
  return k;
}

// Per-warp accumulation of sum_n conj(V_i[n]) x[n]: a warp owns chunks of 32*E
// elements; per group of CG vectors each lane forms CG partial sums, reduce8 leaves the
// warp totals on lanes 0, 4, .., 28, which add them to the warp's own accumulator row
// wacc[i] (shared memory, no block barrier inside the sweep).  Rows are summed in warp
// order at the end: the result does not depend on scheduling.
template <typename S, int E>
__device__ __forceinline__ void warp_dots_acc(const S (&v)[E][CG], const S (&x)[E], int i0, int nvec, int lane,
                                              S* wacc) {
  S acc[CG];
#pragma unroll
  for (int g = 0; g < CG; ++g) {
    acc[g] = Sc<S>::zero();
#pragma unroll
    for (int e = 0; e < E; ++e) acc[g] = add(acc[g], cmul(v[e][g], x[e]));
  }
  const S s = reduce8(acc, lane);
  const int i = i0 + (lane >> 2);
  if ((lane & 3) == 0 && i < nvec) wacc[i] = add(wacc[i], s);
}

template <typename S> __device__ __forceinline__ void cp_async_s(S* smem, const S* g, bool ok) {
  if constexpr (sizeof(S) == 16)
    cp_async16(smem, g, ok);
  else
    cp_async8(smem, g, ok);
}

// sum the warps' accumulator rows (fixed order) into partial[i][block]
template <typename S>
__device__ __forceinline__ void flush_warp_rows(const S* wacc, int nvec, int nwarps, S* __restrict__ partial) {
  __syncthreads();
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    S t = Sc<S>::zero();
    for (int q = 0; q < nwarps; ++q) t = add(t, wacc[(size_t)q * nvec + i]);
    partial[(size_t)i * gridDim.x + blockIdx.x] = t;
  }
}

// last block to arrive? (threadfence + counter; the counter is reset for the next use)
__device__ __forceinline__ bool last_block(unsigned* count) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(count, 1u);
    last = t == gridDim.x - 1;
    if (last) *count = 0;
  }
  __syncthreads();
  return last;
}

template <typename S>
__device__ __forceinline__ void sum_partials(const S* __restrict__ partial, int nvec, S* out) {
  // one warp per vector, fixed order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = wid; i < nvec; i += blockDim.x / 32) {
    S s = Sc<S>::zero();
    for (int b = lane; b < (int)gridDim.x; b += 32) s = add(s, partial[(size_t)i * gridDim.x + b]);
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
}

constexpr int DE = 2;  // elements per lane per chunk in the dots sweep

// K1: h = V^H w.  Block = KB threads; dynamic smem = (KB/32) * nvec accumulator rows.
template <typename S>
__global__ void __launch_bounds__(KB) cgs_dots_kernel(const S* __restrict__ V, int nvec, size_t ldv,
                                                      const S* __restrict__ w, size_t N, S* __restrict__ partial,
                                                      S* __restrict__ h, unsigned* __restrict__ count) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  S* wacc_all = reinterpret_cast<S*>(sraw);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = KB / 32;
  for (int i = threadIdx.x; i < NW * nvec; i += KB) wacc_all[i] = Sc<S>::zero();
  __syncthreads();
  S* wacc = wacc_all + (size_t)wid * nvec;
  const size_t chunk = 32 * DE;
  for (size_t base = ((size_t)blockIdx.x * NW + wid) * chunk; base < N; base += (size_t)gridDim.x * NW * chunk) {
    S x[DE];
#pragma unroll
    for (int e = 0; e < DE; ++e) {
      const size_t n = base + e * 32 + lane;
      x[e] = n < N ? w[n] : Sc<S>::zero();
    }
    for (int i0 = 0; i0 < nvec; i0 += CG) {
      S v[DE][CG];
#pragma unroll
      for (int e = 0; e < DE; ++e) {
        const size_t n = base + e * 32 + lane;
#pragma unroll
        for (int g = 0; g < CG; ++g)
          v[e][g] = (n < N && i0 + g < nvec) ? V[(size_t)(i0 + g) * ldv + n] : Sc<S>::zero();
      }
      warp_dots_acc<S, DE>(v, x, i0, nvec, lane, wacc);
    }
  }
  flush_warp_rows(wacc_all, nvec, NW, partial);
  if (last_block(count)) sum_partials(partial, nvec, h);
}

__device__ __forceinline__ double cabs_(double a) { return fabs(a); }
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }

// Givens update of column j (gmres.py:129-148), one thread
template <typename S>
__device__ void givens_apply(S* __restrict__ H, int ldh, int j, S* __restrict__ cs, S* __restrict__ sn,
                             S* __restrict__ g, double beta, double* __restrict__ est) {
  for (int i = 0; i < j; ++i) {
    S hi = H[(size_t)i * ldh + j], hi1 = H[(size_t)(i + 1) * ldh + j];
    S t = add(mul(cs[i], hi), mul(sn[i], hi1));
    H[(size_t)(i + 1) * ldh + j] = sub(mul(cs[i], hi1), mul(conj_(sn[i]), hi));
    H[(size_t)i * ldh + j] = t;
  }
  const S a = H[(size_t)j * ldh + j], hh = H[(size_t)(j + 1) * ldh + j];
  const double aa = cabs_(a), ah = cabs_(hh);
  const double rr = sqrt(aa * aa + ah * ah);
  S c, s;
  if (rr == 0.0) {
    c = Sc<S>::from_real(1.0);
    s = Sc<S>::zero();
  } else if (aa == 0.0) {
    c = Sc<S>::zero();
    s = scale(conj_(hh), 1.0 / rr);
  } else {
    c = Sc<S>::from_real(aa / rr);
    s = scale(mul(scale(a, 1.0 / aa), conj_(hh)), 1.0 / rr);
  }
  cs[j] = c;
  sn[j] = s;
  H[(size_t)j * ldh + j] = add(mul(c, a), mul(s, hh));
  H[(size_t)(j + 1) * ldh + j] = Sc<S>::zero();
  const S gj = g[j];
  g[j + 1] = scale(mul(conj_(s), gj), -1.0);
  g[j] = mul(c, gj);
  est[0] = cabs_(g[j + 1]) / beta;
}

struct GivensArgs {
  void* H;
  int ldh;
  void* cs;
  void* sn;
  void* g;
  double beta;
  double* est;
  int always_reorth;  // 1: the second Gram-Schmidt pass is always applied (HELM_CGS_ALWAYS=1)
};

constexpr int UW = 2;  // warps per block in the update+dots sweep

// HELM_CGS_ALWAYS=1: apply the second pass unconditionally (classical CGS2)
static int cgs_always_reorth() {
  static const int v = [] {
    const char* e = getenv("HELM_CGS_ALWAYS");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return v;
}

// K2: w' = w - V h1 (stored), dots V^H w', ||w'||^2.  A warp owns 32-element chunks.
// STAGED: the chunk's nvec basis rows are copied to the warp's shared-memory stage with
// cp.async (all in flight at once), so the update and the dots read V from HBM once.
// Otherwise the dots re-read V through L2.  Dynamic smem: UW * nvec accumulator rows,
// the h1 copy, and (STAGED) UW * nvec * 32 staged elements.
template <typename S, bool STAGED, int E>
__global__ void __launch_bounds__(UW * 32) cgs_update_dots_kernel(const S* __restrict__ V, int nvec, size_t ldv,
                                                             S* __restrict__ w, size_t N, const S* __restrict__ h1,
                                                             S* __restrict__ partial, double* __restrict__ npart,
                                                             S* __restrict__ h2, unsigned* __restrict__ count,
                                                             S* __restrict__ hcol, size_t hstride,
                                                             double* __restrict__ inv, GivensArgs gv) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  S* wacc_all = reinterpret_cast<S*>(sraw);
  S* hs = wacc_all + (size_t)UW * nvec;
  S* stage_all = hs + nvec;
  __shared__ double nred[UW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < UW * nvec; i += UW * 32) wacc_all[i] = Sc<S>::zero();
  for (int i = threadIdx.x; i < nvec; i += UW * 32) hs[i] = h1[i];
  __syncthreads();
  S* wacc = wacc_all + (size_t)wid * nvec;
  S* stage = stage_all + (size_t)wid * nvec * 32 * E;  // [nvec][E][32]
  double nrm = 0.0;
  constexpr int CH = 32 * E;
  for (size_t base = ((size_t)blockIdx.x * UW + wid) * CH; base < N; base += (size_t)gridDim.x * UW * CH) {
    if (STAGED) {
      for (int i = 0; i < nvec; ++i)
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const size_t n = base + e * 32 + lane;
          cp_async_s(stage + (i * E + e) * 32 + lane, V + (size_t)i * ldv + (n < N ? n : 0), n < N);
        }
      cp_commit();
    }
    S x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const size_t n = base + e * 32 + lane;
      x[e] = n < N ? w[n] : Sc<S>::zero();
    }
    if (STAGED) {
      cp_wait<0>();
      __syncwarp();
    }
    auto vat = [&](int i, int e) {
      const size_t n = base + e * 32 + lane;
      return STAGED ? stage[(i * E + e) * 32 + lane] : (n < N ? V[(size_t)i * ldv + n] : Sc<S>::zero());
    };
    // x -= V h1 with two interleaved chains per element (latency), combined in a fixed order
#pragma unroll
    for (int e = 0; e < E; ++e) {
      S xa = x[e], xb = Sc<S>::zero();
      int i = 0;
      for (; i + 4 <= nvec; i += 4) {
        const S v0 = vat(i, e), v1 = vat(i + 1, e), v2 = vat(i + 2, e), v3 = vat(i + 3, e);
        xa = fms_(hs[i], v0, xa);
        xb = fms_(hs[i + 1], v1, xb);
        xa = fms_(hs[i + 2], v2, xa);
        xb = fms_(hs[i + 3], v3, xb);
      }
      for (; i < nvec; ++i) xa = fms_(hs[i], vat(i, e), xa);
      x[e] = add(xa, xb);
      const size_t n = base + e * 32 + lane;
      if (n < N) {
        w[n] = x[e];
        nrm += abs2(x[e]);
      }
    }
    for (int i0 = 0; i0 < nvec; i0 += CG) {
      S v[E][CG];
#pragma unroll
      for (int e = 0; e < E; ++e)
#pragma unroll
        for (int g = 0; g < CG; ++g) v[e][g] = i0 + g < nvec ? vat(i0 + g, e) : Sc<S>::zero();
      warp_dots_acc<S, E>(v, x, i0, nvec, lane, wacc);
    }
    if (STAGED) __syncwarp();  // the stage is refilled by the next chunk
  }
  flush_warp_rows(wacc_all, nvec, UW, partial);
  nrm = warp_sum(nrm);
  if (lane == 0) nred[wid] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < UW; ++q) s += nred[q];
    npart[blockIdx.x] = s;
  }
  if (!last_block(count)) return;
  // ---- last block: h2, ||w''||, the Hessenberg column, breakdown, Givens ----
  sum_partials(partial, nvec, h2);
  __shared__ double wn2;
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += npart[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) wn2 = s;
  }
  __syncthreads();
  // The re-orthogonalisation is applied only where orthogonality degraded, exactly the
  // reference's test (gmres.py:117-120): max |V^H w'| > 1e-8 ||w'||.  Otherwise the column is h1,
  // ||w''|| = ||w'||, and K3 only normalises (no third sweep of V).
  __shared__ double mx[UW], h2n[UW], h2m[UW];
  __shared__ int reorth_s;
  const int j = nvec - 1;
  {
    double m2 = 0.0;
    for (int i = threadIdx.x; i <= j; i += UW * 32) m2 = fmax(m2, sqrt(abs2(h2[i])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, o));
    if ((threadIdx.x & 31) == 0) h2m[threadIdx.x >> 5] = m2;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 0; k < UW; ++k) m2 = fmax(m2, h2m[k]);
      reorth_s = gv.always_reorth || m2 > 1e-8 * fmax(sqrt(wn2), 2.2250738585072014e-308);
    }
    __syncthreads();
  }
  const bool reorth = reorth_s;
  double m = 0.0, q2 = 0.0;
  for (int i = threadIdx.x; i <= j; i += UW * 32) {
    const S b2 = reorth ? h2[i] : Sc<S>::zero();
    const S v = add(h1[i], b2);
    hcol[(size_t)i * hstride] = v;
    m = fmax(m, sqrt(abs2(v)));
    q2 += abs2(b2);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    q2 += __shfl_xor_sync(0xffffffffu, q2, o);
  }
  if ((threadIdx.x & 31) == 0) {
    mx[threadIdx.x >> 5] = m;
    h2n[threadIdx.x >> 5] = q2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double q = 0.0;
    for (int k = 0; k < UW; ++k) {
      m = fmax(m, mx[k]);
      q += h2n[k];
    }
    inv[3] = reorth ? 1.0 : 0.0;
    const double hn = sqrt(fmax(wn2 - q, 0.0));
    hcol[(size_t)(j + 1) * hstride] = Sc<S>::from_real(hn);
    // breakdown test of gmres.py:125 on max |H[:j+2, j]|
    const bool brk = hn <= 1e-14 * fmax(fmax(m, hn), 1.0);
    inv[0] = brk ? 0.0 : 1.0 / hn;
    inv[1] = brk ? 1.0 : 0.0;
    if (gv.H) givens_apply<S>((S*)gv.H, gv.ldh, j, (S*)gv.cs, (S*)gv.sn, (S*)gv.g, gv.beta, gv.est);
  }
}

// w <- (w - V h2) * inv[0]   (inv[0] = 0 on breakdown: w - V h2 is left unscaled)
template <typename S>
__global__ void __launch_bounds__(KB) cgs_final_kernel(const S* __restrict__ V, int nvec, size_t ldv,
                                                       S* __restrict__ w, size_t N, const S* __restrict__ h2,
                                                       const double* __restrict__ inv) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  extern __shared__ __align__(16) unsigned char sraw[];
  S* hs = reinterpret_cast<S*>(sraw);
  for (int i = threadIdx.x; i < nvec; i += KB) hs[i] = h2[i];
  __syncthreads();
  const double f0 = inv[0];
  const double f = f0 == 0.0 ? 1.0 : f0;
  if (inv[3] == 0.0) {  // no re-orthogonalisation this iteration: normalise w' only
    for (size_t n = blockIdx.x * (size_t)KB + threadIdx.x; n < N; n += (size_t)gridDim.x * KB) w[n] = scale(w[n], f);
    return;
  }
  for (size_t n = blockIdx.x * (size_t)KB + threadIdx.x; n < N; n += (size_t)gridDim.x * KB) {
    S xa = w[n], xb = Sc<S>::zero();
    int i = 0;
    for (; i + 4 <= nvec; i += 4) {
      const S v0 = V[(size_t)i * ldv + n], v1 = V[(size_t)(i + 1) * ldv + n];
      const S v2 = V[(size_t)(i + 2) * ldv + n], v3 = V[(size_t)(i + 3) * ldv + n];
      xa = fms_(hs[i], v0, xa);
      xb = fms_(hs[i + 1], v1, xb);
      xa = fms_(hs[i + 2], v2, xa);
      xb = fms_(hs[i + 3], v3, xb);
    }
    for (; i < nvec; ++i) xa = fms_(hs[i], V[(size_t)i * ldv + n], xa);
    w[n] = scale(add(xa, xb), f);
  }
}

constexpr size_t SMEM_MAX = 227 * 1024;

static void set_smem(const void* fn, size_t bytes) {
  HELM_CHECK(bytes <= SMEM_MAX, "Krylov basis too large for the CGS2 kernels");
  // opt in above 32 KB: the 48 KB default also has to hold the kernels' static shared variables
  if (bytes > 32 * 1024) HELM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

template <typename S>
static void cgs2_run(S* V, int j, size_t ldv, size_t N, S* hcol, size_t hstride, double* inv_out, void* scratch,
                     GivensArgs gv, cudaStream_t st) {
  const int nvec = j + 1;
  CgsScratch k = carve(scratch, nvec);
  S* w = V + (size_t)(j + 1) * ldv;
  const size_t es = sizeof(S);
  // K1
  const size_t sm1 = (size_t)(KB / 32) * nvec * es;
  set_smem((const void*)cgs_dots_kernel<S>, sm1);
  launch_pdl(cgs_dots_kernel<S>, KNB, KB, sm1, st, V, nvec, ldv, w, N, (S*)k.partial, (S*)k.h1, k.count);
  HELM_LAUNCH_CHECK();
  // K2: staged while a block's stage fits in shared memory; E elements per lane keep
  // ~32 staged rows per lane in flight for short bases
  const int E = nvec >= 32 ? 1 : nvec >= 16 ? 2 : nvec >= 8 ? 4 : 8;
  const size_t sm2 = (size_t)(UW + 1) * nvec * es;
  const size_t sm2s = sm2 + (size_t)UW * nvec * 32 * E * es;
  auto launch2 = [&](auto kern, int grid, size_t smem) {
    set_smem((const void*)kern, smem);
    launch_pdl(kern, grid, UW * 32, smem, st, V, nvec, ldv, w, N, (const S*)k.h1, (S*)k.partial, k.npart, (S*)k.h2,
                                      k.count + 1, hcol, hstride, inv_out, gv);
  };
  static const bool staged_ok = [] {
    const char* e = getenv("HELM_CGS_STAGED");
    return !(e && e[0] == '0');
  }();
  if (staged_ok && sm2s <= SMEM_MAX) {
    const int bps = (int)std::min<size_t>(8, std::max<size_t>(1, (SMEM_MAX + 1024) / (sm2s + 1024)));
    if (E == 8) launch2(cgs_update_dots_kernel<S, true, 8>, 148 * bps, sm2s);
    else if (E == 4) launch2(cgs_update_dots_kernel<S, true, 4>, 148 * bps, sm2s);
    else if (E == 2) launch2(cgs_update_dots_kernel<S, true, 2>, 148 * bps, sm2s);
    else launch2(cgs_update_dots_kernel<S, true, 1>, 148 * bps, sm2s);
  } else {
    launch2(cgs_update_dots_kernel<S, false, 1>, PB, sm2);
  }
  HELM_LAUNCH_CHECK();
  // K3
  const size_t sm3 = (size_t)nvec * es;
  set_smem((const void*)cgs_final_kernel<S>, sm3);
  launch_pdl(cgs_final_kernel<S>, KNB, KB, sm3, st, V, nvec, ldv, w, N, (const S*)k.h2, inv_out);
  HELM_LAUNCH_CHECK();
}

// x = sum_i h_i V_i (fresh output)
template <typename S>
void krylov_combine(S* x, const S* V, int nvec, size_t ldv, const S* h, size_t N, cudaStream_t st) {
  const size_t smem = (size_t)nvec * sizeof(S);
  set_smem((const void*)update_kernel<S>, smem);
  launch_pdl(update_kernel<S>, KNB, KB, smem, st, x, V, nvec, ldv, h, 1.0, N, 1, nullptr);
  HELM_LAUNCH_CHECK();
}

template <typename S> void krylov_norm2(const S* x, size_t N, double* out, void* scratch, cudaStream_t st) {
  CgsScratch k = carve(scratch, 1);
  launch_pdl(norm2_kernel<S>, KNB, KB, 0, st, x, N, k.npart);
  HELM_LAUNCH_CHECK();
  launch_pdl(sum_partials_kernel, 1, 32, 0, st, k.npart, KNB, out);
  HELM_LAUNCH_CHECK();
}

// Arnoldi step j: V[j+1] holds w on entry; hcol points at H[0][j] with stride hstride.
// inv_out[0] = 1/||w|| (0 on breakdown), inv_out[1] = breakdown flag.  With H != null the
// Givens update of column j runs in the same launch (est_out[0] = |g[j+1]| / beta).
template <typename S>
void krylov_cgs2_impl(S* V, int j, size_t ldv, size_t N, S* hcol, size_t hstride, double* inv_out, void* scratch,
                      cudaStream_t st, S* H, int ldh, S* cs, S* sn, S* g, double beta, double* est_out) {
  GivensArgs gv{H, ldh, cs, sn, g, beta, est_out, cgs_always_reorth()};
  cgs2_run<S>(V, j, ldv, N, hcol, hstride, inv_out, scratch, gv, st);
}

template <typename S>
void krylov_cgs2(S* V, int j, size_t ldv, size_t N, S* hcol, void* scratch, cudaStream_t st) {
  CgsScratch k = carve(scratch, j + 1);
  GivensArgs gv{};
  gv.always_reorth = cgs_always_reorth();
  cgs2_run<S>(V, j, ldv, N, hcol, 1, k.scal + 2, scratch, gv, st);
}

template <typename S>
__global__ void givens_kernel(S* H, int ldh, int j, S* cs, S* sn, S* g, double beta, double* est) {
  pdl_wait();  // PDL: the predecessor's writes are visible (no-op without PDL)
  if (threadIdx.x == 0 && blockIdx.x == 0) givens_apply<S>(H, ldh, j, cs, sn, g, beta, est);
}

template <typename S>
void krylov_givens(S* H, int ldh, int j, S* cs, S* sn, S* g, double beta, double* est, cudaStream_t st) {
  launch_pdl(givens_kernel<S>, 1, 32, 0, st, H, ldh, j, cs, sn, g, beta, est);
  HELM_LAUNCH_CHECK();
}

template <typename S> void krylov_backsolve(const S* H, int ldh, int j, const S* g, S* y, cudaStream_t st) {
  const size_t smem = (size_t)(j + 1) * sizeof(S);
  static bool attr[2] = {false, false};
  if (!attr[Sc<S>::cplx]) {
    HELM_CUDA(cudaFuncSetAttribute(backsolve_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr[Sc<S>::cplx] = true;
  }
  launch_pdl(backsolve_kernel<S>, 1, 256, smem, st, H, ldh, j, g, y);
  HELM_LAUNCH_CHECK();
}

template <typename S> void krylov_scale(S* x, const S* src, const double* s, int invert, size_t N, cudaStream_t st) {
  launch_pdl(scale_kernel<S>, KNB, KB, 0, st, x, src, s, invert, N);
  HELM_LAUNCH_CHECK();
}

#define HELM_INST(S)                                                                                          \
  template void krylov_combine<S>(S*, const S*, int, size_t, const S*, size_t, cudaStream_t);                 \
  template void krylov_norm2<S>(const S*, size_t, double*, void*, cudaStream_t);                              \
  template void krylov_cgs2_impl<S>(S*, int, size_t, size_t, S*, size_t, double*, void*, cudaStream_t, S*, int, \
                                    S*, S*, S*, double, double*);                                              \
  template void krylov_cgs2<S>(S*, int, size_t, size_t, S*, void*, cudaStream_t);                             \
  template void krylov_givens<S>(S*, int, int, S*, S*, S*, double, double*, cudaStream_t);                    \
  template void krylov_backsolve<S>(const S*, int, int, const S*, S*, cudaStream_t);                          \
  template void krylov_scale<S>(S*, const S*, const double*, int, size_t, cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
