// Shared device helpers for libhelmb200: the scalar algebra used by every
// kernel (fp64 for MP-1, interleaved complex128 = double2 for MP-2), error
// plumbing, and the internal plan/workspace structs.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <stdexcept>
#include <utility>
#include <vector>

#include "../../include/helmb200.h"

namespace helm {

// ----------------------------------------------------------------------------
// scalar algebra: the same kernel source serves fp64 and complex128
// ----------------------------------------------------------------------------
__host__ __device__ __forceinline__ double2 mk(double r, double i) { return make_double2(r, i); }

template <typename S> struct Sc;
template <> struct Sc<double> {
  static constexpr bool cplx = false;
  __host__ __device__ __forceinline__ static double zero() { return 0.0; }
  __host__ __device__ __forceinline__ static double from_real(double r) { return r; }
};
template <> struct Sc<double2> {
  static constexpr bool cplx = true;
  __host__ __device__ __forceinline__ static double2 zero() { return mk(0.0, 0.0); }
  __host__ __device__ __forceinline__ static double2 from_real(double r) { return mk(r, 0.0); }
};

__host__ __device__ __forceinline__ double add(double a, double b) { return a + b; }
__host__ __device__ __forceinline__ double2 add(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double sub(double a, double b) { return a - b; }
__host__ __device__ __forceinline__ double2 sub(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double mul(double a, double b) { return a * b; }
__host__ __device__ __forceinline__ double2 mul(double2 a, double2 b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 mul(double a, double2 b) { return mk(a * b.x, a * b.y); }
__host__ __device__ __forceinline__ double2 mul(double2 a, double b) { return mk(a.x * b, a.y * b); }
// a + b*c
__host__ __device__ __forceinline__ double fma_(double b, double c, double a) { return fma(b, c, a); }
__host__ __device__ __forceinline__ double2 fma_(double2 b, double2 c, double2 a) {
  return mk(fma(b.x, c.x, fma(-b.y, c.y, a.x)), fma(b.x, c.y, fma(b.y, c.x, a.y)));
}
__host__ __device__ __forceinline__ double2 fma_(double b, double2 c, double2 a) {
  return mk(fma(b, c.x, a.x), fma(b, c.y, a.y));
}
// a - b*c
__host__ __device__ __forceinline__ double fms_(double b, double c, double a) { return fma(-b, c, a); }
__host__ __device__ __forceinline__ double2 fms_(double2 b, double2 c, double2 a) {
  return mk(fma(-b.x, c.x, fma(b.y, c.y, a.x)), fma(-b.x, c.y, fma(-b.y, c.x, a.y)));
}
__host__ __device__ __forceinline__ double conj_(double a) { return a; }
__host__ __device__ __forceinline__ double2 conj_(double2 a) { return mk(a.x, -a.y); }
// conj(a) * b
__host__ __device__ __forceinline__ double cmul(double a, double b) { return a * b; }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double abs2(double a) { return a * a; }
__host__ __device__ __forceinline__ double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ double scale(double a, double s) { return a * s; }
__host__ __device__ __forceinline__ double2 scale(double2 a, double s) { return mk(a.x * s, a.y * s); }
// a / b  (Smith-free: the denominators here are O(1/h^2), far from overflow)
__host__ __device__ __forceinline__ double div_(double a, double b) { return a / b; }
__host__ __device__ __forceinline__ double2 div_(double2 a, double2 b) {
  double d = b.x * b.x + b.y * b.y;
  return mk((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__host__ __device__ __forceinline__ double recip(double b) { return 1.0 / b; }
__host__ __device__ __forceinline__ double2 recip(double2 b) {
  double d = b.x * b.x + b.y * b.y;
  return mk(b.x / d, -b.y / d);
}

// warp-level sums (xor butterfly: every lane ends with the total)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Dot-product accumulators.  CSum<true>: compensated (value s + running error c,
// TwoSum / FMA-TwoProduct error-free transformations), so the result no longer depends on
// the summation order at the rounding level and a sum can be split over lanes and warps
// freely.  CSum<false>: a plain FMA chain with the same interface.
template <bool COMP> struct CSum;
template <> struct CSum<true> {
  double s = 0.0, c = 0.0;
  __device__ __forceinline__ void add(double p) {
    const double t = s + p, z = t - s;
    c += (s - (t - z)) + (p - z);
    s = t;
  }
  __device__ __forceinline__ void fma(double x, double y) {
    const double p = x * y;
    c += ::fma(x, y, -p);
    add(p);
  }
  __device__ __forceinline__ void merge(CSum b) {
    c += b.c;
    add(b.s);
  }
  __device__ __forceinline__ double val() const { return s + c; }
  __device__ __forceinline__ CSum shfl_xor(int o) const {
    CSum r;
    r.s = __shfl_xor_sync(0xffffffffu, s, o);
    r.c = __shfl_xor_sync(0xffffffffu, c, o);
    return r;
  }
};
template <> struct CSum<false> {
  double s = 0.0;
  __device__ __forceinline__ void add(double p) { s += p; }
  __device__ __forceinline__ void fma(double x, double y) { s = ::fma(x, y, s); }
  __device__ __forceinline__ void merge(CSum b) { s += b.s; }
  __device__ __forceinline__ double val() const { return s; }
  __device__ __forceinline__ CSum shfl_xor(int o) const {
    CSum r;
    r.s = __shfl_xor_sync(0xffffffffu, s, o);
    return r;
  }
};
// complex re + i im += x * y
template <bool C>
__device__ __forceinline__ void csum_cfma(CSum<C>& re, CSum<C>& im, double2 x, double2 y) {
  re.fma(x.x, y.x);
  re.fma(-x.y, y.y);
  im.fma(x.x, y.y);
  im.fma(x.y, y.x);
}
// xor butterfly (every lane ends with the same total: the merge is symmetric)
template <bool C>
__device__ __forceinline__ void warp_csum(CSum<C>& v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v.merge(v.shfl_xor(o));
}

// ----------------------------------------------------------------------------
// error plumbing
// ----------------------------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void set_last_error(const std::string& msg);

#define HELM_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::helm::Error(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +      \
                          __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)
#define HELM_CHECK(cond, msg)                                                             \
  do {                                                                                    \
    if (!(cond)) throw ::helm::Error(msg);                                                \
  } while (0)
void count_launch();
#define HELM_LAUNCH_CHECK()        \
  do {                             \
    ::helm::count_launch();        \
    HELM_CUDA(cudaGetLastError()); \
  } while (0)

// ----------------------------------------------------------------------------
// grid geometry shared by the stencil, transfer and local kernels
// ----------------------------------------------------------------------------
struct Geo {
  int nu;        // unknowns per dimension
  int m0;        // coarse unknowns per dimension
  int off;       // fine unknown u of coarse unknown U is 2U + off + d (0 Sommerfeld, 1 Dirichlet)
  int sommerfeld;
  double inv_h2; // 1/h^2
  double k2;     // k^2
  double2 tb;    // Sommerfeld 1-D end diagonal 1/h^2 - i k/h (discretization.py:136-148)
};

// One row of A (discretization.py:171-184) at node (iy, ix) applied to the centre value c
// and its four neighbours (pass zero for neighbours outside the unknown set).
template <typename S>
__host__ __device__ __forceinline__ S stencil_point(const Geo& g, int ix, int iy, S c, S up, S dn, S lf, S rt) {
  if constexpr (!Sc<S>::cplx) {
    return (4.0 * g.inv_h2 - g.k2) * c - g.inv_h2 * (up + dn + lf + rt);
  } else {
    const int nu = g.nu;
    const bool ey = (iy == 0) | (iy == nu - 1), ex = (ix == 0) | (ix == nu - 1);
    const double wy = ey ? 0.5 : 1.0, wx = ex ? 0.5 : 1.0;
    const double2 ty = ey ? g.tb : mk(2.0 * g.inv_h2, 0.0);
    const double2 tx = ex ? g.tb : mk(2.0 * g.inv_h2, 0.0);
    const double2 diag = mk(wx * ty.x + wy * tx.x - g.k2 * wy * wx, wx * ty.y + wy * tx.y);
    S acc = mul(diag, c);
    acc = sub(acc, scale(add(up, dn), wx * g.inv_h2));
    acc = sub(acc, scale(add(lf, rt), wy * g.inv_h2));
    return acc;
  }
}

// Device-side constants of a plan (device pointers).
struct PlanDev {
  // 1-D boxes
  int p;
  int* box_start;
  int* box_len;
  int* box_class;
  int n_classes;
  int max_len;
  int* class_len;
  int* class_off_V;    // element offset of class c in class_V
  int* class_off_lam;  // element offset of class c in class_lambda
  void* class_V;
  void* class_lambda;
  int* class_real;     // 1: V and lambda of the class are real (class_Vr holds V)
  double* class_Vr;
  int* box_ff;         // subdomain ids (ay * p + ax) whose two classes are real and symmetric (folded FDM)
  int n_ff;
  double* class_Vf;    // [n_classes][40][40] folded eigenvectors (even modes | odd modes)
  double* class_lamf;  // [n_classes][40] eigenvalues in the folded mode order (padding 1e30)
  double* class_invden; // [n_classes][n_classes][40][40] 1 / (lamf_y + lamf_x - k^2), padding 0
  int* box_dst;        // subdomain ids whose two classes are the Dirichlet middle pencil, L = 4 dst_q - 1 (local_dst.cu)
  int n_dst;
  int dst_q;
  double* dst_inv;     // [4 dst_q][4 dst_q] (2/N)^2 / (lam_y[m] + lam_x[n] - k^2), sine-mode order
  int* box_edge;       // MP-2 subdomain ids with one middle-pencil axis and one Sommerfeld-end axis
  int n_edge;
  int* class_tri;      // [n_classes] index into edge_tri of a Sommerfeld-end class, or -1
  double2* edge_tri;   // [n_tri][2][40][4 dst_q]: Thomas factors l_i, 1/d_i of T_e + (lam_mu - k^2) W_e
  int* box_rr;         // other subdomains whose two classes are real
  int n_rr;
  int* box_mix;        // the other subdomains
  int n_mix;
  // per-unknown 1-D overlap bookkeeping
  int* node_first_box; // first box containing unknown i
  int* node_mult;      // 1 or 2
  int* node_band;      // compact overlap-band index or -1
  int* band_node;      // inverse of node_band
  int nbands;          // number of 1-D unknowns with multiplicity 2
  // coarse (fast x-transform + band solves + Woodbury strips)
  int m0;
  int fft_len;         // n - 1 when it is a power of two, else 0 (direct transform)
  double2* twiddle;    // [fft_len] exp(-2 pi i k / fft_len)
  double* coarse_scale;
  double* coarse_lamT;  // Dirichlet 2-D DST scaling
  double* coarse_lamM;
  double coarse_qn;
  void* t0_band;
  void* m0_band;
  int* band_piv;        // Sommerfeld band LU (pivot offsets widened to int for 4-byte cp.async)
  void* band_l;         // [m0][m0][2] multipliers (inside band_fac)
  void* band_u;         // [m0][m0][5] {1/U_jj, U_j,j+1..j+4}, or [m0][m0][3] when band_nopiv (inside band_fac)
  void* band_fac;       // one allocation holding band_l then band_u
  size_t band_fac_bytes;
  int band_nopiv;       // no pivot was taken: U has no fill (compact 3-entry rows, pivots never read)
  double2* band_seg;    // segment propagators of the small-batch band solve (band_seg.cu), or null
  int n_strip;
  double* strip_q;
  void* cap_left;
  void* cap_right;
  void* cap_mode;
  void* cap_vt;         // strip refinement (coarse.cu)
  void* cap_hg;
  double2 strip_lt[16]; // (T0 - T~), (M0 - M~) on the strip columns [i][j]
  double2 strip_lm[16];
  int strip_refine;
  // general coarse spaces (coarse_dense.cu): coarse_dense != 0 selects them
  int coarse_dense;
  int p_width, pt_width;
  int* p_start;
  int* pt_start;
  double* p_taps;
  double* pt_taps;
  int a0_bw;
  void* a0_stencil;
  void* coarse_V;
  void* coarse_invden;
};

// ----------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel of the library starts with
// pdl_wait() (griddepcontrol.wait: blocks until the stream predecessor has completed and
// its writes are visible; a no-op when the kernel was launched without PDL).  launch_pdl
// launches with the programmatic-stream-serialization attribute, so a dependent kernel's
// launch overlaps the exit of its predecessor's last CTAs (the implicit trigger at CTA
// exit; no kernel calls launch_dependents early).  Measured at n = 2049: batch-1 M^-1
// 0.608 -> 0.582 ms, batch-32 M^-1 9.91 -> 9.85 ms, a 50-iteration GMRES 1.698 -> 1.650 ms
// per iteration.  An explicit launch_dependents at kernel entry was slower inside GMRES
// (dependent CTAs resident beside the streaming CGS2 sweeps: +15 % there).  HELM_PDL=0
// disables it.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  HELM_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// Band-factor entry (row j, mode a): blocked by 32 modes, so the factors of the modes one
// CTA owns are contiguous (0.26-0.39 MB per block at m0 = 1025 instead of a 34-50 MB
// stride-m0 span: a handful of pages per SM at a time)
__host__ __device__ __forceinline__ size_t fac_idx(int j, int a, int m0) {
  return ((size_t)(a >> 5) * m0 + j) * 32 + (a & 31);
}
__host__ __device__ __forceinline__ size_t fac_elems(int m0) { return (size_t)((m0 + 31) / 32) * 32 * m0; }

// cp.async (Ampere+) helpers: src-size 0 zero-fills without reading
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

}  // namespace helm

struct helm_plan {
  helm_desc desc;  // scalars only (pointer members cleared)
  helm::Geo geo;
  helm::PlanDev dev;
  int64_t N;
  int64_t N0;
  size_t elem;     // bytes per scalar
  std::vector<int> h_box_start, h_box_len, h_box_class, h_class_len;
};

struct helm_workspace {
  const helm_plan* plan;
  int max_batch;
  void* z;        // [B][N]
  void* d;        // [B][N]
  void* c;        // [B][N0]
  void* g;        // [B][N0]
  void* y0;       // [B][N0]
  void* r0;       // [B][N0]
  void* e0;       // [B][N0]
  void* f0;       // [B][N0]
  void* ovl;      // overlap scratch [B][6][nbands][nu]
  void* strip[7]; // coarse Woodbury scratch [m0][B * n_strip]: Z, C^, C_S, split-K partials (x8), rho, W, Zf
  void* strip_part;  // strip-value partial sums of the band passes [ceil(m0/32)][m0][B * n_strip] (batch > 4)
  void* red;      // reduction scratch (doubles)
  size_t red_bytes;
  void* pinned;   // small pinned host buffer for scalar read-back
  void* basis;    // GMRES Krylov basis (basis.cu: reserved address range, physical chunks on demand)
  cudaStream_t side;       // second stream: the boundary-box solves run beside the tensor-core boxes
  cudaEvent_t fork, join;  // ordering of the side stream against the caller's stream
};
