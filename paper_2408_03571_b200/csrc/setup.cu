// Native setup: everything helm_plan_create needs, computed inside the library
// from the problem parameters alone (n, bc, k, p, m, kind), so a C caller does not re-implement
// the host setup of paper_2408_03571_b200/fdm_setup.py.  Restates, line for line:
//
//   pencil_1d          helmdd discretization.py:130-154, 171-188  (1-D T, W)
//   box intervals      decomposition.py:66-79, 111-134
//   local classes      schwarz.py:55-59 (the p^2 factorisations) -> one eigen-decomposition per
//                      distinct 1-D box pencil, T V = W V diag(lam), V^T W V = I
//   coarse space       coarse.py:102-133 (Bezier ratio 2), 154-167 (Galerkin A0):
//                      T0 = P T P^T, M0 = P W P^T (pentadiagonal); the fast sine / cosine
//                      transform eigenvalues (long double sums), the pivoted band LU of
//                      T0 + s_a M0 for every x-mode a, and (Sommerfeld) the Woodbury / strip data
//                      in the eigenbasis of the reflection-folded y-pencil (T0, M0).
//
// The eigen-decompositions run on the GPU through cuSOLVER (syevd for the real symmetric pencils,
// geev for the complex symmetric ones, normalised with the bilinear form u^T u = 1 and refined by one
// Ogita-Aishima Newton step); cuSOLVER is loaded with dlopen only when this entry point is used.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include <cusolverDn.h>

#include "ops.cuh"

namespace helm {
namespace setup {

using cd = std::complex<double>;
using ld = long double;

// ---------------------------------------------------------------------------------------
// cuSOLVER through dlopen
// ---------------------------------------------------------------------------------------
struct Solver {
  void* so = nullptr;
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t prm = nullptr;
  decltype(&cusolverDnCreate) create;
  decltype(&cusolverDnDestroy) destroy;
  decltype(&cusolverDnCreateParams) create_params;
  decltype(&cusolverDnDestroyParams) destroy_params;
  decltype(&cusolverDnDsyevd_bufferSize) syevd_bs;
  decltype(&cusolverDnDsyevd) syevd;
  decltype(&cusolverDnXgeev_bufferSize) geev_bs;
  decltype(&cusolverDnXgeev) geev;

  Solver() {
    for (const char* nm : {"libcusolver.so.11", "libcusolver.so", "/usr/local/cuda/lib64/libcusolver.so.11"})
      if ((so = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    HELM_CHECK(so, "native setup needs cuSOLVER (libcusolver.so.11)");
    auto sym = [&](const char* s) {
      void* f = dlsym(so, s);
      HELM_CHECK(f, std::string("cuSOLVER symbol missing: ") + s);
      return f;
    };
    create = (decltype(create))sym("cusolverDnCreate");
    destroy = (decltype(destroy))sym("cusolverDnDestroy");
    create_params = (decltype(create_params))sym("cusolverDnCreateParams");
    destroy_params = (decltype(destroy_params))sym("cusolverDnDestroyParams");
    syevd_bs = (decltype(syevd_bs))sym("cusolverDnDsyevd_bufferSize");
    syevd = (decltype(syevd))sym("cusolverDnDsyevd");
    geev_bs = (decltype(geev_bs))sym("cusolverDnXgeev_bufferSize");
    geev = (decltype(geev))sym("cusolverDnXgeev");
    HELM_CHECK(create(&h) == CUSOLVER_STATUS_SUCCESS, "cusolverDnCreate failed");
    HELM_CHECK(create_params(&prm) == CUSOLVER_STATUS_SUCCESS, "cusolverDnCreateParams failed");
  }
  ~Solver() {
    if (prm) destroy_params(prm);
    if (h) destroy(h);
    if (so) dlclose(so);
  }

  // eigen-pairs of a real symmetric m x m matrix (row-major = column-major): ascending lam, U columns
  void sym(int m, const std::vector<double>& A, std::vector<double>& lam, std::vector<double>& U) {
    double *dA, *dW, *work;
    int* info;
    HELM_CUDA(cudaMalloc(&dA, sizeof(double) * m * m));
    HELM_CUDA(cudaMalloc(&dW, sizeof(double) * m));
    HELM_CUDA(cudaMalloc(&info, sizeof(int)));
    HELM_CUDA(cudaMemcpy(dA, A.data(), sizeof(double) * m * m, cudaMemcpyHostToDevice));
    int lw = 0;
    HELM_CHECK(syevd_bs(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, dA, m, dW, &lw) ==
                   CUSOLVER_STATUS_SUCCESS, "syevd_bufferSize failed");
    HELM_CUDA(cudaMalloc(&work, sizeof(double) * std::max(lw, 1)));
    HELM_CHECK(syevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, dA, m, dW, work, lw, info) ==
                   CUSOLVER_STATUS_SUCCESS, "syevd failed");
    int hinfo = 0;
    HELM_CUDA(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
    HELM_CHECK(hinfo == 0, "syevd did not converge");
    lam.resize(m);
    std::vector<double> cm((size_t)m * m);
    HELM_CUDA(cudaMemcpy(lam.data(), dW, sizeof(double) * m, cudaMemcpyDeviceToHost));
    HELM_CUDA(cudaMemcpy(cm.data(), dA, sizeof(double) * m * m, cudaMemcpyDeviceToHost));
    U.assign((size_t)m * m, 0.0);  // row-major U[i][j] = component i of eigenvector j
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) U[(size_t)i * m + j] = cm[(size_t)j * m + i];
    cudaFree(dA);
    cudaFree(dW);
    cudaFree(info);
    cudaFree(work);
  }

  // eigen-pairs of a general complex m x m matrix (row-major input): lam, right eigenvectors as U columns
  void gen(int m, const std::vector<cd>& A, std::vector<cd>& lam, std::vector<cd>& U) {
    std::vector<cd> cmA((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) cmA[(size_t)j * m + i] = A[(size_t)i * m + j];
    void *dA, *dW, *dVR, *dwork;
    int* info;
    const size_t es = sizeof(cd);
    HELM_CUDA(cudaMalloc(&dA, es * m * m));
    HELM_CUDA(cudaMalloc(&dW, es * m));
    HELM_CUDA(cudaMalloc(&dVR, es * m * m));
    HELM_CUDA(cudaMalloc(&info, sizeof(int)));
    HELM_CUDA(cudaMemcpy(dA, cmA.data(), es * m * m, cudaMemcpyHostToDevice));
    size_t dbytes = 0, hbytes = 0;
    HELM_CHECK(geev_bs(h, prm, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, CUDA_C_64F, dA, m,
                       CUDA_C_64F, dW, CUDA_C_64F, nullptr, m, CUDA_C_64F, dVR, m, CUDA_C_64F, &dbytes, &hbytes) ==
                   CUSOLVER_STATUS_SUCCESS, "geev_bufferSize failed");
    HELM_CUDA(cudaMalloc(&dwork, std::max<size_t>(dbytes, 16)));
    std::vector<char> hwork(std::max<size_t>(hbytes, 16));
    HELM_CHECK(geev(h, prm, CUSOLVER_EIG_MODE_NOVECTOR, CUSOLVER_EIG_MODE_VECTOR, m, CUDA_C_64F, dA, m, CUDA_C_64F,
                    dW, CUDA_C_64F, nullptr, m, CUDA_C_64F, dVR, m, CUDA_C_64F, dwork, dbytes, hwork.data(), hbytes,
                    info) == CUSOLVER_STATUS_SUCCESS, "geev failed");
    int hinfo = 0;
    HELM_CUDA(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
    HELM_CHECK(hinfo == 0, "geev did not converge");
    lam.resize(m);
    std::vector<cd> cm((size_t)m * m);
    HELM_CUDA(cudaMemcpy(lam.data(), dW, es * m, cudaMemcpyDeviceToHost));
    HELM_CUDA(cudaMemcpy(cm.data(), dVR, es * m * m, cudaMemcpyDeviceToHost));
    U.assign((size_t)m * m, cd(0));
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) U[(size_t)i * m + j] = cm[(size_t)j * m + i];
    cudaFree(dA);
    cudaFree(dW);
    cudaFree(dVR);
    cudaFree(info);
    cudaFree(dwork);
  }
};

// ---------------------------------------------------------------------------------------
// small dense helpers (row-major)
// ---------------------------------------------------------------------------------------
template <typename T> struct Mat {
  int r = 0, c = 0;
  std::vector<T> a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, T(0)) {}
  T& operator()(int i, int j) { return a[(size_t)i * c + j]; }
  const T& operator()(int i, int j) const { return a[(size_t)i * c + j]; }
};

template <typename A, typename B>
static auto matmul(const Mat<A>& x, const Mat<B>& y) {
  using R = decltype(A() * B());
  Mat<R> z(x.r, y.c);
  for (int i = 0; i < x.r; ++i)
    for (int k = 0; k < x.c; ++k) {
      const R v = x(i, k);
      if (v == R(0)) continue;
      const B* yr = &y.a[(size_t)k * y.c];
      R* zr = &z.a[(size_t)i * z.c];
      for (int j = 0; j < y.c; ++j) zr[j] += v * yr[j];
    }
  return z;
}
template <typename T> static Mat<T> transpose(const Mat<T>& x) {
  Mat<T> y(x.c, x.r);
  for (int i = 0; i < x.r; ++i)
    for (int j = 0; j < x.c; ++j) y(j, i) = x(i, j);
  return y;
}

// ---------------------------------------------------------------------------------------
// eigen-pairs of pencils (fdm_setup.py _sym_pencil_eig, _general_pencil_eig, _refine_eig)
// ---------------------------------------------------------------------------------------
// One Newton step on S U = U diag(lam), U^T U = I (complex symmetric S), then V = back U
static void refine_eig(const Mat<cd>& S, std::vector<cd>& lam, Mat<cd>& U) {
  const int m = S.r;
  Mat<cd> Ut = transpose(U);
  Mat<cd> R = matmul(Ut, U);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) R(i, j) = (i == j ? cd(1) : cd(0)) - R(i, j);
  Mat<cd> SU = matmul(Ut, matmul(S, U));
  std::vector<cd> lt(m);
  double lmax = 0.0;
  for (int i = 0; i < m; ++i) {
    lt[i] = SU(i, i) / (1.0 - R(i, i));
    lmax = std::max(lmax, std::abs(lt[i]));
  }
  Mat<cd> E(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      if (i == j) {
        E(i, j) = R(i, i) / 2.0;
        continue;
      }
      const cd gap = lt[j] - lt[i];
      E(i, j) = std::abs(gap) < 1e-8 * lmax ? cd(0) : (SU(i, j) + lt[j] * R(i, j)) / gap;
    }
  Mat<cd> UE = matmul(U, E);
  for (size_t e = 0; e < U.a.size(); ++e) U.a[e] += UE.a[e];
  for (int j = 0; j < m; ++j) {
    cd s(0);
    for (int i = 0; i < m; ++i) s += U(i, j) * U(i, j);
    const cd nrm = std::sqrt(s);
    for (int i = 0; i < m; ++i) U(i, j) /= nrm;
  }
  lam = lt;
}

// T V = W V diag(lam), V^T W V = I for a (complex) symmetric T and w > 0 (local classes)
static void sym_pencil_eig(Solver& so, const Mat<cd>& T, const std::vector<double>& w, bool cplx,
                           std::vector<cd>& lam, Mat<cd>& V) {
  const int m = T.r;
  std::vector<double> s(m);
  for (int i = 0; i < m; ++i) s[i] = 1.0 / std::sqrt(w[i]);
  bool real = true;
  for (const cd& v : T.a) real = real && v.imag() == 0.0;
  V = Mat<cd>(m, m);
  lam.assign(m, cd(0));
  if (!cplx || real) {
    std::vector<double> A((size_t)m * m), l, U;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) A[(size_t)i * m + j] = s[i] * T(i, j).real() * s[j];
    so.sym(m, A, l, U);
    for (int j = 0; j < m; ++j) lam[j] = l[j];
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) V(i, j) = s[i] * U[(size_t)i * m + j];
    return;
  }
  Mat<cd> S(m, m), Um(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) S(i, j) = s[i] * T(i, j) * s[j];
  std::vector<cd> l, U;
  so.gen(m, S.a, l, U);
  for (int j = 0; j < m; ++j) {
    cd q(0);
    for (int i = 0; i < m; ++i) q += U[(size_t)i * m + j] * U[(size_t)i * m + j];
    const cd nrm = std::sqrt(q);
    for (int i = 0; i < m; ++i) Um(i, j) = U[(size_t)i * m + j] / nrm;
  }
  lam = l;
  refine_eig(S, lam, Um);  // geev's vectors carry ~1e-13 residuals; one Newton step removes them
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) V(i, j) = s[i] * Um(i, j);
}

// T0 V = M0 V diag(lam), V^T M0 V = I; M0 real SPD, T0 (complex) symmetric (coarse pencils)
static void general_pencil_eig(Solver& so, const Mat<cd>& T0, const Mat<double>& M0, std::vector<cd>& lam,
                               Mat<cd>& V) {
  const int m = M0.r;
  // Cholesky M0 = Lc Lc^T, Li = Lc^{-1}
  Mat<double> Lc(m, m), Li(m, m);
  for (int j = 0; j < m; ++j) {
    double d = M0(j, j);
    for (int k = 0; k < j; ++k) d -= Lc(j, k) * Lc(j, k);
    HELM_CHECK(d > 0.0, "coarse mass pencil is not positive definite");
    Lc(j, j) = std::sqrt(d);
    for (int i = j + 1; i < m; ++i) {
      double v = M0(i, j);
      for (int k = 0; k < j; ++k) v -= Lc(i, k) * Lc(j, k);
      Lc(i, j) = v / Lc(j, j);
    }
  }
  for (int j = 0; j < m; ++j) {
    Li(j, j) = 1.0 / Lc(j, j);
    for (int i = j + 1; i < m; ++i) {
      double v = 0.0;
      for (int k = j; k < i; ++k) v -= Lc(i, k) * Li(k, j);
      Li(i, j) = v / Lc(i, i);
    }
  }
  Mat<cd> Lic(m, m);
  for (size_t e = 0; e < Li.a.size(); ++e) Lic.a[e] = Li.a[e];
  Mat<cd> S = matmul(matmul(Lic, T0), transpose(Lic));
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) S(i, j) = S(j, i) = 0.5 * (S(i, j) + S(j, i));
  bool real = true;
  for (const cd& v : S.a) real = real && v.imag() == 0.0;
  Mat<cd> U(m, m);
  lam.assign(m, cd(0));
  if (real) {
    std::vector<double> A((size_t)m * m), l, u;
    for (size_t e = 0; e < A.size(); ++e) A[e] = S.a[e].real();
    so.sym(m, A, l, u);
    for (int j = 0; j < m; ++j) lam[j] = l[j];
    for (size_t e = 0; e < u.size(); ++e) U.a[e] = u[e];
    V = matmul(transpose(Lic), U);
    return;
  }
  std::vector<cd> l, u;
  so.gen(m, S.a, l, u);
  for (size_t e = 0; e < u.size(); ++e) U.a[e] = u[e];
  for (int j = 0; j < m; ++j) {
    cd q(0);
    for (int i = 0; i < m; ++i) q += U(i, j) * U(i, j);
    const cd nrm = std::sqrt(q);
    for (int i = 0; i < m; ++i) U(i, j) /= nrm;
  }
  lam = l;
  refine_eig(S, lam, U);
  V = matmul(transpose(Lic), U);
}

// ---------------------------------------------------------------------------------------
// problem pieces
// ---------------------------------------------------------------------------------------
struct Pencil1D {
  int nu;
  Mat<cd> T;
  std::vector<double> w;
};
static Pencil1D pencil_1d(int n, bool somm, double k) {  // discretization.py:130-154, 171-188
  Pencil1D p;
  const double h = 1.0 / (n - 1);
  p.nu = somm ? n : n - 2;
  const int m = p.nu;
  p.T = Mat<cd>(m, m);
  p.w.assign(m, 1.0);
  for (int i = 0; i < m; ++i) {
    p.T(i, i) = 2.0 / (h * h);
    if (i + 1 < m) p.T(i, i + 1) = p.T(i + 1, i) = -1.0 / (h * h);
  }
  if (somm) {
    p.T(0, 0) = p.T(m - 1, m - 1) = cd(1.0 / (h * h), -k / h);
    p.w[0] = p.w[m - 1] = 0.5;
  }
  return p;
}

// 1-D box a: unknown interval [start, start + len) (decomposition.py:66-79)
static void box_interval(int n, bool somm, int p, int m, int a, int& start, int& len) {
  const int c = (n - 1) / p, lo_u = somm ? 0 : 1, nu = somm ? n : n - 2;
  int lo, hi;
  if (m == 0) {
    lo = a * c + (a > 0 ? 1 : 0);
    hi = (a + 1) * c;
  } else {
    lo = a * c - (m - 1);
    hi = (a + 1) * c + (m - 1);
  }
  lo = std::max(lo, lo_u);
  hi = std::min(hi, lo_u + nu - 1);
  start = lo - lo_u;
  len = hi - lo + 1;
}

// dense 1-D Bezier restriction P (m0 x nu), ratio 2 (coarse.py:102-133)
static Mat<double> bezier2(int n, bool somm) {
  const int nu = somm ? n : n - 2, off = somm ? 0 : 1;
  const int m0 = somm ? (n + 1) / 2 : (n - 3) / 2;
  const double taps[5] = {1.0 / 8, 4.0 / 8, 6.0 / 8, 4.0 / 8, 1.0 / 8};
  Mat<double> P(m0, nu);
  for (int U = 0; U < m0; ++U)
    for (int d = -2; d <= 2; ++d) {
      const int u = 2 * U + off + d;
      if (u >= 0 && u < nu) P(U, u) = taps[d + 2];
    }
  return P;
}

// diag(Q^{-1} W^{-1} A Q) of a pentadiagonal real A in long double (fdm_setup.py _transform_eigs)
static std::vector<double> transform_eigs(const Mat<double>& A, bool dct) {
  const int m = A.r;
  const ld pi = 3.14159265358979323846264338327950288L;
  std::vector<ld> qn(m);
  for (int a = 0; a < m; ++a) qn[a] = dct ? ((a == 0 || a == m - 1) ? ld(1) / (m - 1) : ld(2) / (m - 1)) : ld(2) / (m + 1);
  auto Q = [&](int i, int a) -> ld {
    return dct ? cosl((ld)i * (ld)a * (pi / (m - 1))) : sinl((ld)(i + 1) * (ld)(a + 1) * (pi / (m + 1)));
  };
  std::vector<double> out(m);
  for (int a = 0; a < m; ++a) {
    ld s = 0;
    for (int i = 0; i < m; ++i) {
      ld aq = 0;
      for (int d = -2; d <= 2; ++d) {
        const int j = i + d;
        if (j >= 0 && j < m && A(i, j) != 0.0) aq += (ld)A(i, j) * Q(j, a);
      }
      s += Q(i, a) * aq;
    }
    out[a] = (double)(s * qn[a]);
  }
  return out;
}

// pivoted band LU (kl = ku = 2) of T0 + shift_a M0 for every a (fdm_setup.py band_lu)
static void band_lu(const std::vector<cd>& t0b, const std::vector<cd>& m0b, const std::vector<double>& shifts, int m,
                    std::vector<uint8_t>& piv, std::vector<cd>& L, std::vector<cd>& U) {
  const int na = (int)shifts.size();
  piv.assign((size_t)m * na, 0);
  L.assign((size_t)m * na * 2, cd(0));
  U.assign((size_t)m * na * 5, cd(0));
  for (int a = 0; a < na; ++a) {
    auto B = [&](int i, int d) -> cd {  // row i over columns i-2 .. i+2
      return i < m ? t0b[(size_t)i * 5 + d] + shifts[a] * m0b[(size_t)i * 5 + d] : cd(0);
    };
    double scale = 0.0;
    for (int i = 0; i < m; ++i)
      for (int d = 0; d < 5; ++d) scale = std::max(scale, std::abs(B(i, d)));
    cd R[3][5] = {};
    for (int q = 0; q < 5; ++q) {
      R[0][q] = q + 2 < 5 ? B(0, q + 2) : cd(0);
      R[1][q] = (m > 1 && q + 1 < 5) ? B(1, q + 1) : cd(0);
      R[2][q] = m > 2 ? B(2, q) : cd(0);
    }
    for (int j = 0; j < m; ++j) {
      double cand[3] = {std::abs(R[0][0]), j + 1 < m ? std::abs(R[1][0]) : -1.0, j + 2 < m ? std::abs(R[2][0]) : -1.0};
      int pv = 0;
      for (int q = 1; q < 3; ++q)
        if (cand[q] > cand[pv]) pv = q;
      if (pv)
        for (int q = 0; q < 5; ++q) std::swap(R[0][q], R[pv][q]);
      const cd d = R[0][0];
      HELM_CHECK(std::abs(d) > 1e-14 * scale, "coarse band system is singular (k^2 at a coarse eigenvalue)");
      const cd l1 = j + 1 < m ? R[1][0] / d : cd(0), l2 = j + 2 < m ? R[2][0] / d : cd(0);
      for (int q = 0; q < 5; ++q) {
        R[1][q] -= l1 * R[0][q];
        R[2][q] -= l2 * R[0][q];
      }
      const size_t e = (size_t)j * na + a;
      piv[e] = (uint8_t)pv;
      L[e * 2] = l1;
      L[e * 2 + 1] = l2;
      U[e * 5] = 1.0 / d;
      for (int q = 1; q < 5; ++q) U[e * 5 + q] = R[0][q];
      cd n0[5], n1[5];
      for (int q = 0; q < 5; ++q) {
        n0[q] = q + 1 < 5 ? R[1][q + 1] : cd(0);
        n1[q] = q + 1 < 5 ? R[2][q + 1] : cd(0);
      }
      for (int q = 0; q < 5; ++q) {
        R[0][q] = n0[q];
        R[1][q] = n1[q];
        R[2][q] = B(j + 3, q);
      }
    }
  }
}

static std::vector<cd> bands5(const Mat<cd>& A) {
  const int m = A.r;
  std::vector<cd> out((size_t)m * 5, cd(0));
  for (int i = 0; i < m; ++i)
    for (int d = -2; d <= 2; ++d)
      if (i + d >= 0 && i + d < m) out[(size_t)i * 5 + d + 2] = A(i, i + d);
  return out;
}

// packed half-size blocks (fdm_setup.py fold_blocks): "left" rows = modes [even; odd], "right" cols
static std::vector<cd> fold_blocks(const Mat<cd>& A, bool left) {
  const int m = A.r, he = (m + 1) / 2, ho = m / 2;
  std::vector<cd> out;
  out.reserve((size_t)he * he + (size_t)ho * ho);
  for (int i = 0; i < he; ++i)
    for (int j = 0; j < he; ++j) out.push_back(A(i, j));
  for (int i = 0; i < ho; ++i)
    for (int j = 0; j < ho; ++j) out.push_back(left ? A(he + i, j) : A(i, he + j));
  return out;
}

// ---------------------------------------------------------------------------------------
// the whole descriptor
// ---------------------------------------------------------------------------------------
struct Built {
  helm_desc d{};
  std::vector<int32_t> box_start, box_len, box_class, class_len;
  std::vector<double> classV_r, classL_r;
  std::vector<cd> classV_c, classL_c;
  std::vector<double> scale, lamT, lamM, strip_q;
  std::vector<cd> t0b, m0b, L, U, cm, hg, cl, cr, vt, lt, lm;
  std::vector<double> t0b_r, m0b_r;
  std::vector<uint8_t> piv;
};

static void build_desc(const helm_problem& pr, Built& b) {
  HELM_CHECK(pr.n >= 5 && pr.n % 2 == 1, "n must be odd and >= 5");
  HELM_CHECK(pr.bc == HELM_DIRICHLET || pr.bc == HELM_SOMMERFELD, "unknown boundary condition");
  HELM_CHECK(pr.coarse_kind == 0 && pr.ratio == 2,
             "the native setup builds the HOCS ratio-2 coarse solver (other coarse spaces: Python setup)");
  HELM_CHECK(pr.p >= 1 && (pr.n - 1) % pr.p == 0, "p must divide the cell count n-1");
  HELM_CHECK(pr.overlap_layers >= 0, "overlap layer count must be nonnegative");
  const bool somm = pr.bc == HELM_SOMMERFELD;
  const double k = pr.k;
  Solver so;
  Pencil1D pc = pencil_1d(pr.n, somm, k);
  const int nu = pc.nu;
  helm_desc& d = b.d;
  std::memset(&d, 0, sizeof(d));
  d.n = pr.n;
  d.bc = pr.bc;
  d.is_complex = somm ? 1 : 0;
  d.kind = pr.kind;
  d.weights_before_solve = pr.weights_before_solve;
  d.p = pr.p;
  d.overlap_layers = pr.overlap_layers;
  d.ratio = 2;
  d.k = k;
  // ---- local classes (fdm_setup.py local_classes) ----
  struct Cls {
    int L, first, last;
  };
  std::vector<Cls> keys;
  std::vector<std::vector<cd>> lams;
  std::vector<Mat<cd>> Vs;
  for (int a = 0; a < pr.p; ++a) {
    int s, L;
    box_interval(pr.n, somm, pr.p, pr.overlap_layers, a, s, L);
    const Cls key{L, s == 0, s + L == nu};
    int id = -1;
    for (size_t q = 0; q < keys.size(); ++q)
      if (keys[q].L == key.L && keys[q].first == key.first && keys[q].last == key.last) id = (int)q;
    if (id < 0) {
      Mat<cd> Tb(L, L);
      std::vector<double> wb(L);
      for (int i = 0; i < L; ++i) {
        wb[i] = pc.w[s + i];
        for (int j = 0; j < L; ++j) Tb(i, j) = pc.T(s + i, s + j);
      }
      std::vector<cd> lam;
      Mat<cd> V;
      bool dir_box = true;  // tridiag(-1, 2, -1)/h^2, W = I: exact DST eigen-pairs (fdm_setup.py _dst_pencil)
      const double h = 1.0 / (pr.n - 1);
      for (int i = 0; i < L && dir_box; ++i) {
        dir_box = wb[i] == 1.0 && Tb(i, i) == cd(2.0 / (h * h));
        if (i + 1 < L) dir_box = dir_box && Tb(i, i + 1) == cd(-1.0 / (h * h));
      }
      if (dir_box) {
        const ld pi = 3.14159265358979323846264338327950288L;
        V = Mat<cd>(L, L);
        lam.assign(L, cd(0));
        const ld nrm = sqrtl((ld)2 / (L + 1));
        for (int j = 1; j <= L; ++j) {
          const ld sj = sinl((ld)j * pi / (2 * (L + 1)));
          lam[j - 1] = (double)(((ld)4 / ((ld)h * (ld)h)) * sj * sj);
          for (int i = 1; i <= L; ++i) V(i - 1, j - 1) = (double)(nrm * sinl((ld)i * (ld)j * pi / (L + 1)));
        }
      } else {
        sym_pencil_eig(so, Tb, wb, somm, lam, V);
      }
      id = (int)keys.size();
      keys.push_back(key);
      lams.push_back(lam);
      Vs.push_back(V);
    }
    b.box_start.push_back(s);
    b.box_len.push_back(L);
    b.box_class.push_back(id);
  }
  {  // singular subdomain pencils (linalg.py:76-86 via fdm_setup.py local_classes)
    double tmax = 0.0, wmax = 0.0;
    for (const cd& v : pc.T.a) tmax = std::max(tmax, std::abs(v));
    for (double v : pc.w) wmax = std::max(wmax, v);
    const double sc = tmax + k * k * wmax;
    for (auto& la : lams)
      for (auto& lb : lams)
        for (const cd& x : la)
          for (const cd& y : lb)
            HELM_CHECK(std::abs(x + y - k * k) > 1e-14 * sc, "subdomain matrix is singular");
  }
  for (size_t q = 0; q < keys.size(); ++q) {
    b.class_len.push_back(keys[q].L);
    for (const cd& v : Vs[q].a) {
      b.classV_c.push_back(v);
      b.classV_r.push_back(v.real());
    }
    for (const cd& v : lams[q]) {
      b.classL_c.push_back(v);
      b.classL_r.push_back(v.real());
    }
  }
  d.box_start = b.box_start.data();
  d.box_len = b.box_len.data();
  d.box_class = b.box_class.data();
  d.n_classes = (int)keys.size();
  d.class_len = b.class_len.data();
  d.class_V = somm ? (const void*)b.classV_c.data() : (const void*)b.classV_r.data();
  d.class_lambda = somm ? (const void*)b.classL_c.data() : (const void*)b.classL_r.data();
  // ---- coarse level (fdm_setup.py coarse_pencil, coarse_fast) ----
  Mat<double> P = bezier2(pr.n, somm);
  const int m = P.r;
  d.m0 = m;
  Mat<cd> Pc(m, nu);
  for (size_t e = 0; e < P.a.size(); ++e) Pc.a[e] = P.a[e];
  Mat<cd> T0 = matmul(matmul(Pc, pc.T), transpose(Pc));
  Mat<double> M0(m, m);
  {
    Mat<double> WP = transpose(P);
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < m; ++j) WP(i, j) *= pc.w[i];
    M0 = matmul(P, WP);
  }
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) {
      T0(i, j) = T0(j, i) = 0.5 * (T0(i, j) + T0(j, i));
      M0(i, j) = M0(j, i) = 0.5 * (M0(i, j) + M0(j, i));
    }
  Mat<cd> M0c(m, m);
  for (size_t e = 0; e < M0.a.size(); ++e) M0c.a[e] = M0.a[e];
  if (!somm) {  // Dirichlet: the 2-D DST diagonalises A0 exactly
    Mat<double> T0r(m, m);
    for (size_t e = 0; e < T0.a.size(); ++e) T0r.a[e] = T0.a[e].real();
    b.lamT = transform_eigs(T0r, false);
    b.lamM = transform_eigs(M0, false);
    double dmax = 0.0, dmin = 1e300;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        const double v = std::abs(b.lamT[i] * b.lamM[j] + b.lamM[i] * b.lamT[j] - k * k * b.lamM[i] * b.lamM[j]);
        dmax = std::max(dmax, v);
        dmin = std::min(dmin, v);
      }
    HELM_CHECK(dmin > 1e-14 * dmax, "coarse Galerkin matrix is singular (k^2 at a coarse eigenvalue)");
    b.scale.assign(m, 2.0 / (m + 1));
    b.t0b_r.resize((size_t)m * 5);
    b.m0b_r.resize((size_t)m * 5);
    const std::vector<cd> tb = bands5(T0), mb = bands5(M0c);
    for (size_t e = 0; e < tb.size(); ++e) {
      b.t0b_r[e] = tb[e].real();
      b.m0b_r[e] = mb[e].real();
    }
    d.coarse_scale = b.scale.data();
    d.coarse_lamT = b.lamT.data();
    d.coarse_lamM = b.lamM.data();
    d.coarse_qn = 2.0 / (m + 1);
    d.t0_band = b.t0b_r.data();
    d.m0_band = b.m0b_r.data();
    d.n_strip = 0;
    d.refine_steps = pr.refine_steps < 0 ? 0 : pr.refine_steps;
    return;
  }
  // Sommerfeld: DCT-I along x for the reflected pencil (T~, M~), band solves along y
  const int Mx = m - 1;
  Mat<double> Pi = transpose(P);  // nu x m: the Bezier prolongation of the even extension
  Pi(0, 1) += 1.0 / 8;
  Pi(nu - 1, m - 2) += 1.0 / 8;
  Mat<double> Tre(nu, nu);
  for (size_t e = 0; e < Tre.a.size(); ++e) Tre.a[e] = pc.T.a[e].real();
  Mat<double> Tt = matmul(matmul(transpose(Pi), Tre), Pi);
  Mat<double> WPi = Pi;
  for (int i = 0; i < nu; ++i)
    for (int j = 0; j < m; ++j) WPi(i, j) *= pc.w[i];
  Mat<double> Mt = matmul(transpose(Pi), WPi);
  const int strip[4] = {0, 1, m - 2, m - 1};
  std::vector<double> qnorm(m);
  for (int a = 0; a < m; ++a) qnorm[a] = 2.0 / (Mx * ((a == 0 || a == m - 1) ? 2.0 : 1.0));
  auto Q = [&](int x, int a) { return std::cos(M_PI * (double)x * (double)a / Mx); };
  b.lamT = transform_eigs(Tt, true);
  b.lamM = transform_eigs(Mt, true);
  std::vector<double> shifts(m);
  for (int a = 0; a < m; ++a) {
    HELM_CHECK(b.lamM[a] > 0.0, "coarse mass pencil is not positive definite");
    shifts[a] = b.lamT[a] / b.lamM[a] - k * k;
  }
  b.t0b = bands5(T0);
  b.m0b = bands5(M0c);
  band_lu(b.t0b, b.m0b, shifts, m, b.piv, b.L, b.U);
  b.scale.resize(m);
  for (int a = 0; a < m; ++a) b.scale[a] = qnorm[a] / b.lamM[a];
  b.strip_q.resize((size_t)m * 4);
  for (int a = 0; a < m; ++a)
    for (int i = 0; i < 4; ++i) b.strip_q[(size_t)a * 4 + i] = Q(strip[i], a);
  // strip couplings L_T = (T0 - T~), L_M = (M0 - M~) on the strip columns
  cd LT[4][4], LM[4][4];
  b.lt.resize(16);
  b.lm.resize(16);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      LT[i][j] = T0(strip[i], strip[j]) - Tt(strip[i], strip[j]);
      LM[i][j] = M0(strip[i], strip[j]) - Mt(strip[i], strip[j]);
      b.lt[i * 4 + j] = LT[i][j];
      b.lm[i * 4 + j] = LM[i][j];
    }
  // folded eigen-pairs of the y-pencil (fdm_setup.py folded_pencil_eig)
  const int he = (m + 1) / 2, ho = m / 2;
  std::vector<cd> lam(m);
  Mat<cd> V(m, m);
  for (int blk = 0; blk < 2; ++blk) {
    const int nb = blk ? ho : he;
    Mat<double> Pb(m, nb);
    for (int j = 0; j < ho; ++j) {
      if (blk == 0) Pb(j, j) = Pb(m - 1 - j, j) = 1.0;
      else {
        Pb(j, j) = 1.0;
        Pb(m - 1 - j, j) = -1.0;
      }
    }
    if (blk == 0 && he > ho) Pb(ho, ho) = 1.0;
    Mat<cd> Pbc(m, nb);
    for (size_t e = 0; e < Pb.a.size(); ++e) Pbc.a[e] = Pb.a[e];
    Mat<cd> Tb = matmul(matmul(transpose(Pbc), T0), Pbc);
    Mat<double> Mb = matmul(matmul(transpose(Pb), M0), Pb);
    std::vector<cd> lb;
    Mat<cd> Ub;
    general_pencil_eig(so, Tb, Mb, lb, Ub);
    Mat<cd> Vb = matmul(Pbc, Ub);
    for (int j = 0; j < nb; ++j) {
      lam[(blk ? he : 0) + j] = lb[j];
      for (int i = 0; i < m; ++i) V(i, (blk ? he : 0) + j) = Vb(i, j);
    }
  }
  // Woodbury data: Gamma_b, G_b, K_b = I + Gamma_b G_b, cap_mode = G K^{-1}, cap_hg = cap_mode Gamma
  b.cm.assign((size_t)m * 16, cd(0));
  b.hg.assign((size_t)m * 16, cd(0));
  std::vector<double> qis((size_t)m * 4);  // Qi[a][strip j] = qnorm[a] Q[strip_j][a]
  for (int a = 0; a < m; ++a)
    for (int j = 0; j < 4; ++j) qis[(size_t)a * 4 + j] = qnorm[a] * Q(strip[j], a);
  for (int bm = 0; bm < m; ++bm) {
    cd Gam[4][4] = {}, G[4][4], K[4][4], Ki[4][4];
    for (int a = 0; a < m; ++a) {
      const cd den = b.lamM[a] * lam[bm] + (b.lamT[a] - k * k * b.lamM[a]);
      const cd inv = 1.0 / den;
      for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) Gam[i][j] += b.strip_q[(size_t)a * 4 + i] * qis[(size_t)a * 4 + j] * inv;
    }
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) G[i][j] = lam[bm] * LM[i][j] + (LT[i][j] - k * k * LM[i][j]);
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        cd s = i == j ? cd(1) : cd(0);
        for (int q = 0; q < 4; ++q) s += Gam[i][q] * G[q][j];
        K[i][j] = s;
      }
    // 4 x 4 inverse by Gauss-Jordan with partial pivoting
    cd Aug[4][8];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 8; ++j) Aug[i][j] = j < 4 ? K[i][j] : (j - 4 == i ? cd(1) : cd(0));
    for (int c = 0; c < 4; ++c) {
      int pv = c;
      for (int r = c + 1; r < 4; ++r)
        if (std::abs(Aug[r][c]) > std::abs(Aug[pv][c])) pv = r;
      for (int j = 0; j < 8; ++j) std::swap(Aug[c][j], Aug[pv][j]);
      const cd dv = Aug[c][c];
      for (int j = 0; j < 8; ++j) Aug[c][j] /= dv;
      for (int r = 0; r < 4; ++r)
        if (r != c) {
          const cd f = Aug[r][c];
          for (int j = 0; j < 8; ++j) Aug[r][j] -= f * Aug[c][j];
        }
    }
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) Ki[i][j] = Aug[i][4 + j];
    cd CM[4][4];
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        cd s = 0;
        for (int q = 0; q < 4; ++q) s += G[i][q] * Ki[q][j];
        CM[i][j] = s;
        b.cm[(size_t)bm * 16 + i * 4 + j] = s;
      }
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        cd s = 0;
        for (int q = 0; q < 4; ++q) s += CM[i][q] * Gam[q][j];
        b.hg[(size_t)bm * 16 + i * 4 + j] = s;
      }
  }
  Mat<cd> Vt = transpose(V);
  b.cl = fold_blocks(matmul(Vt, M0c), true);
  b.cr = fold_blocks(matmul(M0c, V), false);
  b.vt = fold_blocks(Vt, true);
  d.coarse_scale = b.scale.data();
  d.coarse_lamT = b.lamT.data();
  d.coarse_lamM = b.lamM.data();
  d.coarse_qn = qnorm[0];
  d.t0_band = b.t0b.data();
  d.m0_band = b.m0b.data();
  d.band_piv = b.piv.data();
  d.band_l = b.L.data();
  d.band_u = b.U.data();
  d.n_strip = 4;
  d.strip_q = b.strip_q.data();
  d.cap_left = b.cl.data();
  d.cap_right = b.cr.data();
  d.cap_mode = b.cm.data();
  d.cap_vt = b.vt.data();
  d.cap_hg = b.hg.data();
  d.strip_lt = b.lt.data();
  d.strip_lm = b.lm.data();
  d.strip_refine = pr.strip_refine < 0 ? 1 : pr.strip_refine;
  d.refine_steps = pr.refine_steps < 0 ? 0 : pr.refine_steps;
}

}  // namespace setup

// defined in capi.cu
int plan_create_from_desc(const helm_desc* desc, helm_plan** out);

}  // namespace helm

extern "C" int helm_plan_create_problem(const helm_problem* problem, helm_plan** out) {
  try {
    if (!problem || !out) {
      helm::set_last_error("null argument");
      return 1;
    }
    helm::setup::Built b;
    helm::setup::build_desc(*problem, b);
    return helm::plan_create_from_desc(&b.d, out);
  } catch (const std::exception& e) {
    helm::set_last_error(e.what());
    return 1;
  }
}
