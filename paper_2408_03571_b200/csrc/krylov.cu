// K6/K7: the Arnoldi step and Givens update of unrestarted GMRES
// (reference gmres.py:108-148: MGS + one conditional re-orthogonalisation pass,
// complex Givens rotations, residual estimate |g[j+1]| / ||r0||).
//
// B200 form: classical Gram-Schmidt run twice (CGS2).  Each pass is one
// multi-dot sweep of the basis (h = V^H w, block + warp-shuffle reductions,
// deterministic two-stage sum) and one fused update sweep (w -= V h, with the
// squared norm of the result reduced in the same sweep).  In exact arithmetic
// CGS2 equals MGS + re-orthogonalisation; numerically both keep the basis
// orthogonal to working precision, which is what fixes the iteration count.
// H, the rotations and g stay on the device; the host reads one estimate.
#include "ops.cuh"

namespace helm {

constexpr int KB = 256;        // threads per block
constexpr int KNB = 4 * 148;   // reduction blocks (4 per SM)
constexpr int KG = 8;          // vectors per multi-dot group

// partial[i * gridDim.x + block] = sum over the block's elements of conj(V_i) w
template <typename S>
__global__ void __launch_bounds__(KB) dots_kernel(const S* __restrict__ V, int nvec, size_t ldv,
                                                  const S* __restrict__ w, size_t N, S* __restrict__ partial) {
  __shared__ S red[KG][KB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int i0 = 0; i0 < nvec; i0 += KG) {
    const int ng = min(KG, nvec - i0);
    S acc[KG];
#pragma unroll
    for (int g = 0; g < KG; ++g) acc[g] = Sc<S>::zero();
    for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += stride) {
      const S wn = w[n];
#pragma unroll
      for (int g = 0; g < KG; ++g)
        if (g < ng) acc[g] = add(acc[g], cmul(V[(size_t)(i0 + g) * ldv + n], wn));
    }
#pragma unroll
    for (int g = 0; g < KG; ++g) {
      S s = warp_sum(acc[g]);
      if (lane == 0) red[g][wid] = s;
    }
    __syncthreads();
    if (threadIdx.x < ng) {
      S s = Sc<S>::zero();
      for (int q = 0; q < KB / 32; ++q) s = add(s, red[threadIdx.x][q]);
      partial[(size_t)(i0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

// out[i] = sum_b partial[i * nb + b]   (one warp per output, fixed order)
template <typename S>
__global__ void reduce_rows_kernel(const S* __restrict__ partial, int nvec, int nb, S* __restrict__ out) {
  const int i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nvec) return;
  S s = Sc<S>::zero();
  for (int b = lane; b < nb; b += 32) s = add(s, partial[(size_t)i * nb + b]);
  s = warp_sum(s);
  if (lane == 0) out[i] = s;
}

// w <- w + sign * sum_i h_i V_i ; optionally norm2 partial of the result per block
template <typename S>
__global__ void __launch_bounds__(KB) update_kernel(S* __restrict__ w, const S* __restrict__ V, int nvec,
                                                    size_t ldv, const S* __restrict__ h, double sign, size_t N,
                                                    int from_zero, double* __restrict__ npart) {
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
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) s += npart[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// hcol[i] = h1[i] + h2[i] (i <= j), hcol[j+1] = ||w||, breakdown test of gmres.py:125,
// inv[0] = 1/||w|| (0 on breakdown so the scaling pass is skipped)
template <typename S>
__global__ void cgs2_finalize_kernel(const S* __restrict__ h1, const S* __restrict__ h2, const double* __restrict__ n2,
                                     int j, S* __restrict__ hcol, size_t hstride, double* __restrict__ inv) {
  __shared__ double mx[32];
  const double hn = sqrt(*n2);
  double m = 0.0;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    const S v = add(h1[i], h2[i]);
    hcol[(size_t)i * hstride] = v;
    m = fmax(m, sqrt(abs2(v)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) mx[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x / 32); ++q) m = fmax(m, mx[q]);
    m = fmax(mx[0], m);
    hcol[(size_t)(j + 1) * hstride] = Sc<S>::from_real(hn);
    const bool brk = hn <= 1e-14 * fmax(fmax(m, hn), 1.0);
    inv[0] = brk ? 0.0 : 1.0 / hn;
    inv[1] = brk ? 1.0 : 0.0;
  }
}

template <typename S>
__global__ void scale_kernel(S* __restrict__ x, const S* __restrict__ src, const double* __restrict__ s, int invert,
                             size_t N) {
  const double f = invert ? 1.0 / s[0] : s[0];
  if (!invert && f == 0.0) return;  // breakdown: leave the vector alone
  for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += (size_t)gridDim.x * blockDim.x)
    x[n] = scale(src[n], f);
}

// --- Givens update of column j (gmres.py:129-148), one thread --------------
__device__ __forceinline__ double cabs_(double a) { return fabs(a); }
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }
template <typename S>
__global__ void givens_kernel(S* __restrict__ H, int ldh, int j, S* __restrict__ cs, S* __restrict__ sn,
                              S* __restrict__ g, double beta, double* __restrict__ est) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
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

// --- y = R^{-1} g with R = H[:j+1, :j+1] upper triangular (gmres.py:98-103) -----
template <typename S>
__global__ void backsolve_kernel(const S* __restrict__ H, int ldh, int j, const S* __restrict__ g, S* __restrict__ y) {
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
// host launchers
// scratch layout: [partial KG-rounded max_vec x KNB S][h1 max_vec S][h2 max_vec S][npart KNB][n2 4]
// ----------------------------------------------------------------------------
size_t krylov_scratch_bytes(int max_vec) {
  const size_t nv = (size_t)((max_vec + KG - 1) / KG) * KG;
  return nv * KNB * sizeof(double2) + 2 * nv * sizeof(double2) + KNB * sizeof(double) + 8 * sizeof(double);
}
struct KScratch {
  void* partial;
  void* h1;
  void* h2;
  double* npart;
  double* n2;
};
static KScratch carve(void* scratch, int max_vec) {
  const size_t nv = (size_t)((max_vec + KG - 1) / KG) * KG;
  char* p = (char*)scratch;
  KScratch k;
  k.partial = p;
  p += nv * KNB * sizeof(double2);
  k.h1 = p;
  p += nv * sizeof(double2);
  k.h2 = p;
  p += nv * sizeof(double2);
  k.npart = (double*)p;
  p += KNB * sizeof(double);
  k.n2 = (double*)p;
  return k;
}

template <typename S>
void krylov_dots(const S* V, int nvec, size_t ldv, const S* w, size_t N, S* out, void* scratch, cudaStream_t st) {
  KScratch k = carve(scratch, nvec);
  dots_kernel<S><<<KNB, KB, 0, st>>>(V, nvec, ldv, w, N, (S*)k.partial);
  HELM_LAUNCH_CHECK();
  reduce_rows_kernel<S><<<(nvec + 7) / 8, 256, 0, st>>>((S*)k.partial, nvec, KNB, out);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void krylov_update(S* w, const S* V, int nvec, size_t ldv, const S* h, double sign, size_t N, double* norm2_out,
                   void* scratch, cudaStream_t st) {
  KScratch k = carve(scratch, nvec);
  const size_t smem = (size_t)nvec * sizeof(S);
  static bool attr[2] = {false, false};
  if (!attr[Sc<S>::cplx]) {
    HELM_CUDA(cudaFuncSetAttribute(update_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr[Sc<S>::cplx] = true;
  }
  HELM_CHECK(smem <= 200 * 1024, "Krylov basis too large for the update kernel");
  update_kernel<S><<<KNB, KB, smem, st>>>(w, V, nvec, ldv, h, sign, N, /*from_zero=*/0,
                                          norm2_out ? k.npart : nullptr);
  HELM_LAUNCH_CHECK();
  if (norm2_out) {
    sum_partials_kernel<<<1, 32, 0, st>>>(k.npart, KNB, norm2_out);
    HELM_LAUNCH_CHECK();
  }
}

// x = sum_i h_i V_i (fresh output)
template <typename S>
void krylov_combine(S* x, const S* V, int nvec, size_t ldv, const S* h, size_t N, cudaStream_t st) {
  const size_t smem = (size_t)nvec * sizeof(S);
  update_kernel<S><<<KNB, KB, smem, st>>>(x, V, nvec, ldv, h, 1.0, N, 1, nullptr);
  HELM_LAUNCH_CHECK();
}

template <typename S> void krylov_norm2(const S* x, size_t N, double* out, void* scratch, cudaStream_t st) {
  KScratch k = carve(scratch, 1);
  norm2_kernel<S><<<KNB, KB, 0, st>>>(x, N, k.npart);
  HELM_LAUNCH_CHECK();
  sum_partials_kernel<<<1, 32, 0, st>>>(k.npart, KNB, out);
  HELM_LAUNCH_CHECK();
}

// Arnoldi step j: V[j+1] holds w on entry; hcol points at H[0][j] with stride hstride.
// inv_out[0] = 1/||w|| (0 on breakdown), inv_out[1] = breakdown flag.
template <typename S>
void krylov_cgs2_impl(S* V, int j, size_t ldv, size_t N, S* hcol, size_t hstride, double* inv_out, void* scratch,
                      cudaStream_t st) {
  KScratch k = carve(scratch, j + 1);
  S* w = V + (size_t)(j + 1) * ldv;
  krylov_dots<S>(V, j + 1, ldv, w, N, (S*)k.h1, scratch, st);
  krylov_update<S>(w, V, j + 1, ldv, (const S*)k.h1, -1.0, N, nullptr, scratch, st);
  krylov_dots<S>(V, j + 1, ldv, w, N, (S*)k.h2, scratch, st);
  krylov_update<S>(w, V, j + 1, ldv, (const S*)k.h2, -1.0, N, k.n2, scratch, st);
  cgs2_finalize_kernel<S><<<1, 256, 0, st>>>((const S*)k.h1, (const S*)k.h2, k.n2, j, hcol, hstride, inv_out);
  HELM_LAUNCH_CHECK();
  scale_kernel<S><<<KNB, KB, 0, st>>>(w, w, inv_out, 0, N);
  HELM_LAUNCH_CHECK();
}

template <typename S>
void krylov_cgs2(S* V, int j, size_t ldv, size_t N, S* hcol, void* scratch, cudaStream_t st) {
  KScratch k = carve(scratch, j + 1);
  krylov_cgs2_impl<S>(V, j, ldv, N, hcol, 1, k.n2 + 2, scratch, st);
}

template <typename S>
void krylov_givens(S* H, int ldh, int j, S* cs, S* sn, S* g, double beta, double* est, cudaStream_t st) {
  givens_kernel<S><<<1, 32, 0, st>>>(H, ldh, j, cs, sn, g, beta, est);
  HELM_LAUNCH_CHECK();
}

template <typename S> void krylov_backsolve(const S* H, int ldh, int j, const S* g, S* y, cudaStream_t st) {
  const size_t smem = (size_t)(j + 1) * sizeof(S);
  static bool attr[2] = {false, false};
  if (!attr[Sc<S>::cplx]) {
    HELM_CUDA(cudaFuncSetAttribute(backsolve_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr[Sc<S>::cplx] = true;
  }
  backsolve_kernel<S><<<1, 256, smem, st>>>(H, ldh, j, g, y);
  HELM_LAUNCH_CHECK();
}

template <typename S> void krylov_scale(S* x, const S* src, const double* s, int invert, size_t N, cudaStream_t st) {
  scale_kernel<S><<<KNB, KB, 0, st>>>(x, src, s, invert, N);
  HELM_LAUNCH_CHECK();
}

#define HELM_INST(S)                                                                                          \
  template void krylov_dots<S>(const S*, int, size_t, const S*, size_t, S*, void*, cudaStream_t);             \
  template void krylov_update<S>(S*, const S*, int, size_t, const S*, double, size_t, double*, void*,         \
                                 cudaStream_t);                                                               \
  template void krylov_combine<S>(S*, const S*, int, size_t, const S*, size_t, cudaStream_t);                 \
  template void krylov_norm2<S>(const S*, size_t, double*, void*, cudaStream_t);                              \
  template void krylov_cgs2_impl<S>(S*, int, size_t, size_t, S*, size_t, double*, void*, cudaStream_t);       \
  template void krylov_cgs2<S>(S*, int, size_t, size_t, S*, void*, cudaStream_t);                             \
  template void krylov_givens<S>(S*, int, int, S*, S*, S*, double, double*, cudaStream_t);                    \
  template void krylov_backsolve<S>(const S*, int, int, const S*, S*, cudaStream_t);                          \
  template void krylov_scale<S>(S*, const S*, const double*, int, size_t, cudaStream_t);
HELM_INST(double)
HELM_INST(double2)
#undef HELM_INST

}  // namespace helm
