// The extern "C" boundary of libhelmb200.so (include/helmb200.h): plan and
// workspace lifetime, the operator entry points, and the native GMRES driver
// (gmres.py:65-177) that strings the kernels together with one scalar
// read-back per iteration.
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ops.cuh"

namespace helm {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    set_last_error(e.what());
  } catch (...) {
    set_last_error("unknown error");
  }
  return 1;
}

template <typename T>
static T* upload(const void* host, size_t count) {
  if (count == 0) return nullptr;
  HELM_CHECK(host != nullptr, "missing setup array in helm_desc");
  T* d = nullptr;
  HELM_CUDA(cudaMalloc(&d, count * sizeof(T)));
  HELM_CUDA(cudaMemcpy(d, host, count * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HELM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// HELM_<name>=0 switches a fast path off (development A/B and tests)
static bool env_flag_off(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] == '0';
}

static void* upload_bytes(const void* host, size_t bytes) {
  if (bytes == 0) return nullptr;
  HELM_CHECK(host != nullptr, "missing setup array in helm_desc");
  void* d = nullptr;
  HELM_CUDA(cudaMalloc(&d, bytes));
  HELM_CUDA(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice));
  return d;
}

// ---------------------------------------------------------------------------
// composite operators
// ---------------------------------------------------------------------------
template <typename S> void op_apply_A(const helm_plan* P, const S* x, S* y, int batch, cudaStream_t st) {
  launch_stencil<S>(P->geo, x, nullptr, y, batch, st);
}

// R0, R0^T and A0^{-1} for the plan's coarse space: the HOCS ratio-2 kernels (transfer.cu,
// coarse.cu) or the general banded / dense-FDM ones (coarse_dense.cu)
template <typename S> static void restrict_any(const helm_plan* P, const S* x, S* c, int batch, cudaStream_t st) {
  if (P->dev.coarse_dense)
    launch_restrict_general<S>(P, x, c, batch, st);
  else
    launch_restrict<S>(P->geo, x, c, batch, st);
}
template <typename S> static void prolong_any(const helm_plan* P, const S* c, S* z, int batch, cudaStream_t st) {
  if (P->dev.coarse_dense)
    launch_prolong_general<S>(P, c, z, batch, st);
  else
    launch_prolong<S>(P->geo, c, z, batch, st);
}
template <typename S>
static void coarse_solve_any(const helm_plan* P, helm_workspace* ws, const S* c, S* y, int batch, cudaStream_t st) {
  if (P->dev.coarse_dense)
    launch_coarse_solve_dense<S>(P, ws, c, y, batch, st);
  else
    launch_coarse_solve<S>(P, ws, c, y, batch, st);
}

template <typename S>
static void op_coarse_correct(const helm_plan* P, helm_workspace* ws, const S* x, S* z, int batch, cudaStream_t st) {
  S* c = (S*)ws->c;
  S* cy = (S*)ws->y0;  // a distinct output: no copy-back inside the coarse solve
  restrict_any<S>(P, x, c, batch, st);
  coarse_solve_any<S>(P, ws, c, cy, batch, st);
  prolong_any<S>(P, cy, z, batch, st);
}

// SchwarzPreconditioner.apply (schwarz.py:76-103): z = C x shared by every kind
template <typename S>
void op_apply_M(const helm_plan* P, helm_workspace* ws, const S* x, S* y, int batch, cudaStream_t st) {
  HELM_CHECK((const void*)x != (const void*)y, "apply_M: input and output must not alias");
  const int kind = P->desc.kind;
  if (P->dev.coarse_dense) {
    // general coarse space: z = R0^T A0^{-1} R0 x materialised, then (SHS2) d = x - A z and
    // y = z + sum_i R_i^T D_i A_i^{-1} R_i d, or (AS2 / SAS2) y = z + sum_i ... x
    S* z = (S*)ws->z;
    op_coarse_correct<S>(P, ws, x, z, batch, st);
    if (kind == HELM_SHS2) {
      S* d = (S*)ws->d;
      launch_stencil<S>(P->geo, x, z, d, batch, st);
      launch_local_sum<S>(P, d, z, y, (S*)ws->ovl, 1, batch, P->dev.band_node, st, /*coarse_base=*/false, ws);
    } else {
      launch_local_sum<S>(P, x, z, y, (S*)ws->ovl, kind == HELM_SAS2 ? 1 : 0, batch, P->dev.band_node, st,
                          /*coarse_base=*/false, ws);
    }
    return;
  }
  if (kind == HELM_SHS2) {
    // z = R0^T A0^{-1} R0 x and d = x - A z (schwarz.py:86-88) with the prolongation
    // and the deflation stencil fused in one pass
    S* c = (S*)ws->c;
    S* cy = (S*)ws->y0;  // a distinct output: no copy-back inside the coarse solve
    S* d = (S*)ws->d;
    launch_restrict<S>(P->geo, x, c, batch, st);
    launch_coarse_solve<S>(P, ws, c, cy, batch, st);
    // z is not materialised: the local kernels add R0^T c at every node they write
    // (measured: 0.4 ms less per batch of 32 at config 5 than writing z and reading it back)
    launch_prolong_deflate<S>(P->geo, cy, x, nullptr, d, batch, st);
    launch_local_sum<S>(P, d, cy, y, (S*)ws->ovl, 1, batch, P->dev.band_node, st, /*coarse_base=*/true, ws);
  } else {
    S* c = (S*)ws->c;
    S* cy = (S*)ws->y0;
    launch_restrict<S>(P->geo, x, c, batch, st);
    launch_coarse_solve<S>(P, ws, c, cy, batch, st);
    launch_local_sum<S>(P, x, cy, y, (S*)ws->ovl, kind == HELM_SAS2 ? 1 : 0, batch, P->dev.band_node, st,
                        /*coarse_base=*/true, ws);
  }
}

template void op_apply_A<double>(const helm_plan*, const double*, double*, int, cudaStream_t);
template void op_apply_A<double2>(const helm_plan*, const double2*, double2*, int, cudaStream_t);
template void op_apply_M<double>(const helm_plan*, helm_workspace*, const double*, double*, int, cudaStream_t);
template void op_apply_M<double2>(const helm_plan*, helm_workspace*, const double2*, double2*, int, cudaStream_t);

// ---------------------------------------------------------------------------
// GMRES driver (gmres.py:65-177), statement-level mirror on device buffers
// ---------------------------------------------------------------------------
template <typename S> struct DevBuf {
  S* p = nullptr;
  cudaStream_t st;
  DevBuf(size_t n, cudaStream_t s) : st(s) { HELM_CUDA(cudaMallocAsync((void**)&p, n * sizeof(S), s)); }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

template <typename S>
static void gmres_impl(const helm_plan* P, helm_workspace* ws, const S* b, S* x, double rtol, int mi, int side,
                       int use_precond, double* history, helm_gmres_report* rep, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  HELM_CHECK(rtol > 0.0, "relative tolerance must be positive");
  HELM_CHECK(mi >= 1, "iteration cap must be at least 1");
  HELM_CHECK(side == 0 || side == 1, "side must be 0 (right) or 1 (left)");
  const size_t N = (size_t)P->N;
  const bool left = side == 1;
  // The Krylov basis lives in the workspace (basis.cu): address space for the cap is
  // reserved, physical memory is mapped in chunks of 16 vectors as j grows and kept for
  // later solves; the reference allocates (cap+1) N eagerly (gmres.py:88-89), which at
  // n=2049 and cap 1000 would be 67 GB.
  const size_t vbytes = N * sizeof(S);
  S* Vp = nullptr;
  auto ensure_basis = [&](int nvec) {
    Vp = (S*)basis_ensure(ws, (size_t)nvec * vbytes, (size_t)(mi + 1) * vbytes, 16 * vbytes, st);
  };
  ensure_basis(2);
  rep->reorth = 0;
  DevBuf<S> H((size_t)(mi + 1) * mi, st), cs(mi, st), sn(mi, st), g(mi + 1, st), y(mi + 1, st), u(N, st), r(N, st);
  HELM_CHECK(krylov_scratch_bytes(mi + 1) <= ws->red_bytes, "iteration cap too large for the workspace scratch");
  void* scratch = ws->red;
  DevBuf<double> scal(16, st);
  HELM_CUDA(cudaMemsetAsync(H.p, 0, (size_t)(mi + 1) * mi * sizeof(S), st));
  HELM_CUDA(cudaMemsetAsync(cs.p, 0, mi * sizeof(S), st));
  HELM_CUDA(cudaMemsetAsync(sn.p, 0, mi * sizeof(S), st));
  HELM_CUDA(cudaMemsetAsync(g.p, 0, (mi + 1) * sizeof(S), st));
  double* hp = (double*)ws->pinned;

  auto applyM = [&](const S* in, S* out) {
    if (use_precond)
      op_apply_M<S>(P, ws, in, out, 1, st);
    else
      HELM_CUDA(cudaMemcpyAsync(out, in, N * sizeof(S), cudaMemcpyDeviceToDevice, st));
  };
  auto applyOp = [&](const S* in, S* out) {  // right: A M in ; left: M A in
    if (left) {
      op_apply_A<S>(P, in, u.p, 1, st);
      applyM(u.p, out);
    } else {
      applyM(in, u.p);
      op_apply_A<S>(P, u.p, out, 1, st);
    }
  };
  auto read_scalars = [&](const double* dev, int n) {
    HELM_CUDA(cudaMemcpyAsync(hp, dev, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    HELM_CUDA(cudaStreamSynchronize(st));
  };

  // ||b||, r0 (gmres.py:77-86)
  krylov_norm2<S>(b, N, scal.p, scratch, st);
  if (left)
    applyM(b, Vp);
  else
    HELM_CUDA(cudaMemcpyAsync(Vp, b, N * sizeof(S), cudaMemcpyDeviceToDevice, st));
  krylov_norm2<S>(Vp, N, scal.p + 1, scratch, st);
  read_scalars(scal.p, 2);
  const double bnorm = std::sqrt(hp[0]), beta = std::sqrt(hp[1]);
  HELM_CHECK(bnorm != 0.0, "right-hand side must be nonzero");
  // V[0] = r0 / beta ; g[0] = beta
  double sc[2] = {1.0 / beta, beta};
  HELM_CUDA(cudaMemcpyAsync(scal.p + 6, sc, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
  krylov_scale<S>(Vp, Vp, scal.p + 6, 0, N, st);
  S g0 = Sc<S>::from_real(beta);
  HELM_CUDA(cudaMemcpyAsync(g.p, &g0, sizeof(S), cudaMemcpyHostToDevice, st));
  if (history) history[0] = 1.0;

  auto form_solution = [&](int j) {  // gmres.py:98-105
    krylov_backsolve<S>(H.p, mi, j, g.p, y.p, st);
    if (left) {
      krylov_combine<S>(x, Vp, j + 1, N, y.p, N, st);
    } else {
      krylov_combine<S>(r.p, Vp, j + 1, N, y.p, N, st);
      applyM(r.p, x);
    }
  };
  auto true_residual = [&]() {  // ||b - A x|| / ||b||  (gmres.py:153)
    launch_stencil<S>(P->geo, b, x, r.p, 1, st);
    krylov_norm2<S>(r.p, N, scal.p + 8, scratch, st);
    read_scalars(scal.p + 8, 1);
    return std::sqrt(hp[0]) / bnorm;
  };

  static const bool trace = std::getenv("HELM_GMRES_TRACE") != nullptr;
  // Look-ahead: iteration j+1 is enqueued before the host reads iteration j's three scalars
  // (two pinned slots by parity, an event per slot), so the device never idles on the
  // host's convergence test.  Iteration j+1 writes only V[j+2], column j+1 of H and the
  // Givens entries j+1, j+2, none of which x_j = M V_j y_j (gmres.py:98-105) reads, so a
  // converged x_j is the same as without look-ahead; the speculative iteration is skipped
  // when the estimate extrapolated from the last two is within 10x of the tolerance (a
  // wasted iteration costs a whole M^-1 + CGS2).  HELM_GMRES_LOOKAHEAD=0 turns it off.
  const bool look = !trace && !env_flag_off("HELM_GMRES_LOOKAHEAD");
  double* slot = hp + 16;  // [2][4]
  cudaEvent_t sev[2];
  for (auto& e : sev) HELM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};
  if (trace)
    for (auto& e : tev) HELM_CUDA(cudaEventCreate(&e));
  auto enqueue = [&](int j) {
    ensure_basis(j + 2);
    S* vj = Vp + (size_t)j * N;
    if (trace) HELM_CUDA(cudaEventRecord(tev[0], st));
    applyOp(vj, vj + N);
    // CGS2 (3 sweeps) with the Givens update of column j fused into its reducing block
    if (trace) HELM_CUDA(cudaEventRecord(tev[1], st));
    krylov_cgs2_impl<S>(Vp, j, N, N, H.p + j, (size_t)mi, scal.p + 2, scratch, st, H.p, mi, cs.p, sn.p, g.p, beta,
                        scal.p + 4);
    if (trace) HELM_CUDA(cudaEventRecord(tev[2], st));
    HELM_CUDA(cudaMemcpyAsync(slot + 4 * (j & 1), scal.p + 2, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    HELM_CUDA(cudaEventRecord(sev[j & 1], st));
  };
  auto tprev = std::chrono::steady_clock::now();
  bool done = false;
  double est1 = 1.0, est2 = 1.0;  // estimates of the last two iterations
  int queued = 0;                 // iterations enqueued so far
  if (mi > 0) {
    enqueue(0);
    queued = 1;
  }
  for (int j = 0; j < mi && !done; ++j) {
    if (queued == j) {  // not enqueued ahead
      enqueue(j);
      queued = j + 1;
    }
    if (look && j + 1 < mi && queued == j + 1) {
      const double pred = est1 * (est1 / std::max(est2, 1e-300));  // extrapolated estimate of iteration j
      if (pred > 10.0 * rtol) {
        enqueue(j + 1);
        queued = j + 2;
      }
    }
    HELM_CUDA(cudaEventSynchronize(sev[j & 1]));
    const double* hj = slot + 4 * (j & 1);
    const bool brk = hj[1] != 0.0;
    const double est = hj[2];
    rep->reorth += hj[3] != 0.0;  // the conditional second Gram-Schmidt pass ran (gmres.py:117-120)
    est2 = est1;
    est1 = est;
    if (trace) {  // HELM_GMRES_TRACE=1: per-iteration device times of the operator and of CGS2
      float t_op = 0.f, t_cgs = 0.f;
      cudaEventElapsedTime(&t_op, tev[0], tev[1]);
      cudaEventElapsedTime(&t_cgs, tev[1], tev[2]);
      const auto tn = std::chrono::steady_clock::now();
      std::fprintf(stderr, "gmres it %d wall %.3f ms op %.3f cgs2 %.3f\n", j,
                   std::chrono::duration<double, std::milli>(tn - tprev).count(), t_op, t_cgs);
      tprev = tn;
    }
    if (history) history[j + 1] = est;
    if (est <= rtol || brk) {
      form_solution(j);
      const double true_rel = true_residual();
      const bool conv = left ? est <= rtol : true_rel <= rtol;
      if (conv || brk) {
        rep->iterations = j + 1;
        rep->converged = conv;
        rep->breakdown = brk && !conv;
        rep->final_residual = true_rel;
        done = true;
      }
    }
  }
  for (auto& e : sev) cudaEventDestroy(e);
  if (!done) {
    form_solution(mi - 1);
    rep->iterations = mi;
    rep->converged = 0;
    rep->breakdown = 0;
    rep->final_residual = true_residual();
  }
  HELM_CUDA(cudaStreamSynchronize(st));
  if (trace)
    for (auto& e : tev) cudaEventDestroy(e);
  rep->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------------------------
// Multi-right-hand-side GMRES: nrhs independent GMRES runs (gmres.py:65-177
// each) that share every operator application.  The bases are interleaved, V[j][r][N], so
// iteration j applies A and M^{-1} to the contiguous batch V[j] (the batched kernels, at
// batch nrhs) and each right-hand side's CGS2 + Givens runs on its own basis (stride
// nrhs N) with its own H, cs, sn, g.  A right-hand side that has converged (or broken
// down) stops its Arnoldi steps; its basis slot is zeroed and still rides along in the
// batch.  Each right-hand side follows the single-RHS statement order; the batched
// kernels sum some rows in another order than at batch 1 (rounding-level differences).
// ---------------------------------------------------------------------------
template <typename S>
static void gmres_multi_impl(const helm_plan* P, helm_workspace* ws, const S* B, S* X, int nrhs, double rtol, int mi,
                             int side, int use_precond, double* history, helm_gmres_report* reps, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  HELM_CHECK(nrhs >= 1 && nrhs <= ws->max_batch, "nrhs must be in [1, workspace max_batch]");
  HELM_CHECK(rtol > 0.0, "relative tolerance must be positive");
  HELM_CHECK(mi >= 1, "iteration cap must be at least 1");
  HELM_CHECK(side == 0 || side == 1, "side must be 0 (right) or 1 (left)");
  HELM_CHECK(krylov_scratch_bytes(mi + 1) <= ws->red_bytes, "iteration cap too large for the workspace scratch");
  const size_t N = (size_t)P->N, NB = N * nrhs;
  const bool left = side == 1;
  const size_t vbytes = N * sizeof(S);
  S* Vp = nullptr;
  auto ensure_basis = [&](int nvec) {  // nvec basis vectors per right-hand side
    Vp = (S*)basis_ensure(ws, (size_t)nvec * nrhs * vbytes, (size_t)(mi + 1) * nrhs * vbytes, 16 * vbytes, st);
  };
  ensure_basis(2);
  const size_t hsz = (size_t)(mi + 1) * mi;
  DevBuf<S> H(hsz * nrhs, st), cs((size_t)mi * nrhs, st), sn((size_t)mi * nrhs, st), g((size_t)(mi + 1) * nrhs, st),
      y(mi + 1, st), u(NB, st), r(N, st);
  DevBuf<double> scal((size_t)16 * nrhs, st);
  void* scratch = ws->red;
  HELM_CUDA(cudaMemsetAsync(H.p, 0, hsz * nrhs * sizeof(S), st));
  HELM_CUDA(cudaMemsetAsync(cs.p, 0, (size_t)mi * nrhs * sizeof(S), st));
  HELM_CUDA(cudaMemsetAsync(sn.p, 0, (size_t)mi * nrhs * sizeof(S), st));
  HELM_CUDA(cudaMemsetAsync(g.p, 0, (size_t)(mi + 1) * nrhs * sizeof(S), st));
  std::vector<double> hs((size_t)16 * nrhs);
  auto read_all = [&]() {
    HELM_CUDA(cudaMemcpyAsync(hs.data(), scal.p, hs.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    HELM_CUDA(cudaStreamSynchronize(st));
  };
  auto vec = [&](int j, int q) { return Vp + ((size_t)j * nrhs + q) * N; };
  auto applyM = [&](const S* in, S* out, int nb) {
    if (use_precond) op_apply_M<S>(P, ws, in, out, nb, st);
    else HELM_CUDA(cudaMemcpyAsync(out, in, (size_t)nb * N * sizeof(S), cudaMemcpyDeviceToDevice, st));
  };
  // r0 = b (right) or M b (left), beta, V[0] = r0 / beta, g[0] = beta (gmres.py:77-96)
  if (left) applyM(B, Vp, nrhs);
  else HELM_CUDA(cudaMemcpyAsync(Vp, B, NB * sizeof(S), cudaMemcpyDeviceToDevice, st));
  for (int q = 0; q < nrhs; ++q) {
    krylov_norm2<S>(B + (size_t)q * N, N, scal.p + 16 * q, scratch, st);
    krylov_norm2<S>(vec(0, q), N, scal.p + 16 * q + 1, scratch, st);
  }
  read_all();
  std::vector<double> bnorm(nrhs), beta(nrhs);
  std::vector<char> active(nrhs, 1);
  for (int q = 0; q < nrhs; ++q) {
    bnorm[q] = std::sqrt(hs[16 * q]);
    beta[q] = std::sqrt(hs[16 * q + 1]);
    HELM_CHECK(bnorm[q] != 0.0, "right-hand side must be nonzero");
    const double sc = 1.0 / beta[q];
    HELM_CUDA(cudaMemcpyAsync(scal.p + 16 * q + 6, &sc, sizeof(double), cudaMemcpyHostToDevice, st));
    krylov_scale<S>(vec(0, q), vec(0, q), scal.p + 16 * q + 6, 0, N, st);
    const S g0 = Sc<S>::from_real(beta[q]);
    HELM_CUDA(cudaMemcpyAsync(g.p + (size_t)(mi + 1) * q, &g0, sizeof(S), cudaMemcpyHostToDevice, st));
    if (history) history[(size_t)q * (mi + 1)] = 1.0;
    HELM_CUDA(cudaStreamSynchronize(st));  // the host scalars above are read by the copies
  }
  auto form = [&](int q, int j) {  // x_q from the first j+1 basis vectors, true relative residual (gmres.py:98-105, 153)
    S* Hq = H.p + hsz * q;
    S* gq = g.p + (size_t)(mi + 1) * q;
    S* xq = X + (size_t)q * N;
    krylov_backsolve<S>(Hq, mi, j, gq, y.p, st);
    if (left) {
      krylov_combine<S>(xq, Vp + (size_t)q * N, j + 1, NB, y.p, N, st);
    } else {
      krylov_combine<S>(r.p, Vp + (size_t)q * N, j + 1, NB, y.p, N, st);
      applyM(r.p, xq, 1);
    }
    launch_stencil<S>(P->geo, B + (size_t)q * N, xq, r.p, 1, st);
    krylov_norm2<S>(r.p, N, scal.p + 16 * q + 8, scratch, st);
    double t = 0.0;
    HELM_CUDA(cudaMemcpyAsync(&t, scal.p + 16 * q + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
    HELM_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(t) / bnorm[q];
  };
  auto record = [&](int q, int it, bool conv, bool brk, double true_rel) {
    reps[q].iterations = it;
    reps[q].converged = conv;
    reps[q].breakdown = brk && !conv;
    reps[q].final_residual = true_rel;
    active[q] = 0;
  };
  int nact = nrhs;
  for (int j = 0; j < mi && nact > 0; ++j) {
    ensure_basis(j + 2);
    // the whole batch through the operator: right A M V[j], left M A V[j]
    if (left) {
      op_apply_A<S>(P, vec(j, 0), u.p, nrhs, st);
      applyM(u.p, vec(j + 1, 0), nrhs);
    } else {
      applyM(vec(j, 0), u.p, nrhs);
      op_apply_A<S>(P, u.p, vec(j + 1, 0), nrhs, st);
    }
    for (int q = 0; q < nrhs; ++q) {
      if (!active[q]) {
        HELM_CUDA(cudaMemsetAsync(vec(j + 1, q), 0, vbytes, st));  // keeps the ride-along input finite
        continue;
      }
      S* Hq = H.p + hsz * q;
      krylov_cgs2_impl<S>(Vp + (size_t)q * N, j, NB, N, Hq + j, (size_t)mi, scal.p + 16 * q + 2, scratch, st, Hq, mi,
                          cs.p + (size_t)mi * q, sn.p + (size_t)mi * q, g.p + (size_t)(mi + 1) * q, beta[q],
                          scal.p + 16 * q + 4);
    }
    read_all();
    for (int q = 0; q < nrhs; ++q) {
      if (!active[q]) continue;
      const bool brk = hs[16 * q + 3] != 0.0;
      const double est = hs[16 * q + 4];
      if (history) history[(size_t)q * (mi + 1) + j + 1] = est;
      if (est <= rtol || brk) {  // gmres.py:149-165
        const double true_rel = form(q, j);
        const bool conv = left ? est <= rtol : true_rel <= rtol;
        if (conv || brk) record(q, j + 1, conv, brk, true_rel);
      }
      if (active[q] && j + 1 == mi) record(q, mi, false, false, form(q, mi - 1));  // gmres.py:173-177
      if (!active[q]) --nact;
    }
  }
  HELM_CUDA(cudaStreamSynchronize(st));
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int q = 0; q < nrhs; ++q) reps[q].wall_seconds = wall;
}

// ---------------------------------------------------------------------------
// plan construction
// ---------------------------------------------------------------------------
static void build_plan(const helm_desc* d, helm_plan* P) {
  HELM_CHECK(d != nullptr, "null descriptor");
  // MP-1 needs odd n (discretization.py:172-173); MP-2 takes any n (discretization.py:183-188), the
  // coarse ratio must then divide n - 1 (checked below), which excludes ratio 2 for even n
  HELM_CHECK(d->n >= 5 && ((d->n % 2) == 1 || d->bc == HELM_SOMMERFELD), "n must be >= 5, and odd for MP-1");
  HELM_CHECK(d->bc == HELM_DIRICHLET || d->bc == HELM_SOMMERFELD, "unknown boundary condition");
  HELM_CHECK(d->is_complex == (d->bc == HELM_SOMMERFELD ? 1 : 0),
             "MP-1 (Dirichlet) plans are fp64, MP-2 (Sommerfeld) plans complex128");
  HELM_CHECK(d->kind >= HELM_AS2 && d->kind <= HELM_SHS2, "unknown preconditioner kind");
  HELM_CHECK(d->ratio >= 1 && (d->n - 1) % d->ratio == 0, "the coarse ratio must divide the cell count n-1");
  HELM_CHECK(!d->coarse_scale || d->ratio == 2, "the fast coarse solver is the HOCS ratio-2 one");
  // p == 0 (no boxes) and coarse_V == NULL (no coarse solver) give an operator-only plan
  HELM_CHECK(d->p == 0 || (d->p >= 1 && (d->n - 1) % d->p == 0), "p must divide the cell count n-1");
  HELM_CHECK(d->refine_steps >= 0 && d->refine_steps <= 8, "refine_steps out of range");
  HELM_CHECK(d->strip_refine >= 0 && d->strip_refine <= 4, "strip_refine out of range");
  P->desc = *d;
  P->elem = d->is_complex ? sizeof(double2) : sizeof(double);
  Geo& g = P->geo;
  const double h = 1.0 / (d->n - 1);
  g.nu = d->bc == HELM_DIRICHLET ? d->n - 2 : d->n;
  if (d->coarse_V) {  // general coarse space: (n-1)/ratio + 1 coarse nodes, interior ones for Dirichlet
    g.m0 = (d->n - 1) / d->ratio + (d->bc == HELM_DIRICHLET ? -1 : 1);
  } else {
    g.m0 = d->bc == HELM_DIRICHLET ? (d->n - 3) / 2 : (d->n + 1) / 2;
  }
  HELM_CHECK(d->m0 == g.m0, "descriptor m0 does not match the grid and ratio");
  g.off = d->bc == HELM_DIRICHLET ? 1 : 0;
  g.sommerfeld = d->bc == HELM_SOMMERFELD;
  g.inv_h2 = 1.0 / (h * h);
  g.k2 = d->k * d->k;
  g.tb = mk(1.0 / (h * h), -d->k / h);
  P->N = (int64_t)g.nu * g.nu;
  P->N0 = (int64_t)g.m0 * g.m0;
  const int nu = g.nu, p = d->p;

  // boxes and per-node overlap maps (decomposition.py:111-134 weights = 1/multiplicity)
  PlanDev& dv = P->dev;
  std::memset(&dv, 0, sizeof(dv));
  const size_t m0 = g.m0;
  if (d->coarse_V) {
    HELM_CHECK(!d->coarse_scale, "a plan has one coarse solver");
    HELM_CHECK(d->p_width >= 1 && d->pt_width >= 1 && d->p_start && d->p_taps && d->pt_start && d->pt_taps,
               "general coarse space needs the P and P^T bands");
    HELM_CHECK(d->a0_bw >= 1 && d->a0_bw <= 8 && d->a0_stencil && d->coarse_invden,
               "general coarse space needs the A0 stencil and the eigenvalue table");
    HELM_CHECK(m0 >= 1 && m0 <= 4096, "general coarse space: m0 out of range");
    dv.coarse_dense = 1;
    dv.m0 = (int)m0;
    dv.p_width = d->p_width;
    dv.pt_width = d->pt_width;
    dv.p_start = upload<int>(d->p_start, m0);
    dv.p_taps = upload<double>(d->p_taps, m0 * d->p_width);
    dv.pt_start = upload<int>(d->pt_start, g.nu);
    dv.pt_taps = upload<double>(d->pt_taps, (size_t)g.nu * d->pt_width);
    dv.a0_bw = d->a0_bw;
    const size_t taps = (size_t)(2 * d->a0_bw + 1) * (2 * d->a0_bw + 1);
    dv.a0_stencil = upload_bytes(d->a0_stencil, m0 * m0 * taps * P->elem);
    dv.coarse_V = upload_bytes(d->coarse_V, m0 * m0 * P->elem);
    dv.coarse_invden = upload_bytes(d->coarse_invden, m0 * m0 * P->elem);
  }
  if (d->coarse_scale) {
    dv.m0 = (int)m0;
    const int L = d->n - 1;
    dv.fft_len = (L >= 8 && (L & (L - 1)) == 0 && L <= 2048) ? L : 0;  // else: direct transform
    if (dv.fft_len) {
      std::vector<double2> tw(L);
      for (int q = 0; q < L; ++q) {  // exact octant reduction keeps the table symmetric
        const long double ang = -2.0L * 3.14159265358979323846264338327950288L * q / L;
        tw[q] = make_double2((double)cosl(ang), (double)sinl(ang));
      }
      dv.twiddle = upload<double2>(tw.data(), tw.size());
    }
    dv.coarse_scale = upload<double>(d->coarse_scale, m0);
    dv.t0_band = upload_bytes(d->t0_band, m0 * 5 * P->elem);
    dv.m0_band = upload_bytes(d->m0_band, m0 * 5 * P->elem);
    if (d->bc == HELM_SOMMERFELD) {
      HELM_CHECK(d->band_piv && d->band_l && d->band_u, "Sommerfeld coarse solver needs the band factors");
      // factors re-laid out blocked by 32 modes (fac_idx): entry (j, a) of the host's [j][a]
      const size_t mm = (size_t)m0 * m0, fe = fac_elems((int)m0);
      std::vector<int> piv32(fe, 0);
      for (size_t j = 0; j < m0; ++j)
        for (size_t a = 0; a < m0; ++a) piv32[fac_idx((int)j, (int)a, (int)m0)] = d->band_piv[j * m0 + a];
      dv.band_piv = upload<int>(piv32.data(), piv32.size());
      // no pivot taken (and hence no fill in U): rows {1/U_jj, U_j,j+1, U_j,j+2} only
      const double2* uh = static_cast<const double2*>(d->band_u);
      const double2* lh = static_cast<const double2*>(d->band_l);
      HELM_CHECK(P->elem == sizeof(double2), "Sommerfeld band factors are complex128");
      bool nopiv = !env_flag_off("HELM_BAND_NOPIV");
      for (size_t e = 0; nopiv && e < mm; ++e)
        nopiv = d->band_piv[e] == 0 && uh[5 * e + 3].x == 0.0 && uh[5 * e + 3].y == 0.0 && uh[5 * e + 4].x == 0.0 &&
                uh[5 * e + 4].y == 0.0;
      const int ue = nopiv ? 3 : 5;
      dv.band_nopiv = nopiv ? 1 : 0;
      dv.band_fac_bytes = fe * (2 + ue) * P->elem;
      std::vector<double2> hb(fe * (2 + ue), make_double2(0.0, 0.0));
      double2* lb = hb.data();
      double2* ub = hb.data() + fe * 2;
      for (size_t j = 0; j < m0; ++j)
        for (size_t a = 0; a < m0; ++a) {
          const size_t src = j * m0 + a, dst = fac_idx((int)j, (int)a, (int)m0);
          lb[2 * dst] = lh[2 * src];
          lb[2 * dst + 1] = lh[2 * src + 1];
          for (int i = 0; i < ue; ++i) ub[ue * dst + i] = uh[5 * src + i];
        }
      HELM_CUDA(cudaMalloc(&dv.band_fac, dv.band_fac_bytes));
      dv.band_l = dv.band_fac;
      dv.band_u = static_cast<char*>(dv.band_fac) + fe * 2 * P->elem;
      HELM_CUDA(cudaMemcpy(dv.band_fac, hb.data(), dv.band_fac_bytes, cudaMemcpyHostToDevice));
      if (band_seg_usable(m0)) {
        HELM_CUDA(cudaMalloc(&dv.band_seg, band_seg_table_elems(m0) * sizeof(double2)));
        band_seg_setup(dv, dv.band_seg, 0);
        HELM_CUDA(cudaStreamSynchronize(0));
      }
    } else {
      dv.coarse_lamT = upload<double>(d->coarse_lamT, m0);
      dv.coarse_lamM = upload<double>(d->coarse_lamM, m0);
      dv.coarse_qn = d->coarse_qn;
    }
    HELM_CHECK(d->n_strip == (d->bc == HELM_SOMMERFELD ? 4 : 0), "n_strip must be 4 (Sommerfeld) or 0 (Dirichlet)");
    dv.n_strip = d->n_strip;
    if (d->n_strip) {
      const size_t ns = d->n_strip;
      dv.strip_q = upload<double>(d->strip_q, m0 * ns);
      const size_t he = (m0 + 1) / 2, ho = m0 / 2, packed = he * he + ho * ho;
      dv.cap_left = upload_bytes(d->cap_left, packed * P->elem);
      dv.cap_right = upload_bytes(d->cap_right, packed * P->elem);
      dv.cap_mode = upload_bytes(d->cap_mode, m0 * ns * ns * P->elem);
      dv.strip_refine = d->strip_refine;
      if (d->strip_refine) {
        HELM_CHECK(d->cap_vt && d->cap_hg && d->strip_lt && d->strip_lm,
                   "strip refinement needs cap_vt, cap_hg, strip_lt and strip_lm");
        dv.cap_vt = upload_bytes(d->cap_vt, packed * P->elem);
        dv.cap_hg = upload_bytes(d->cap_hg, m0 * ns * ns * P->elem);
        std::memcpy(dv.strip_lt, d->strip_lt, 16 * sizeof(double2));
        std::memcpy(dv.strip_lm, d->strip_lm, 16 * sizeof(double2));
      }
    }
  }
  if (p == 0) return;
  P->h_box_start.assign(d->box_start, d->box_start + p);
  P->h_box_len.assign(d->box_len, d->box_len + p);
  P->h_box_class.assign(d->box_class, d->box_class + p);
  HELM_CHECK(d->n_classes >= 1, "need at least one local class");
  P->h_class_len.assign(d->class_len, d->class_len + d->n_classes);
  std::vector<int> first(nu, -1), mult(nu, 0), band(nu, -1), band_node;
  int max_len = 0;
  for (int a = 0; a < p; ++a) {
    const int s = P->h_box_start[a], L = P->h_box_len[a], c = P->h_box_class[a];
    HELM_CHECK(s >= 0 && L >= 1 && s + L <= nu, "box outside the unknown range");
    HELM_CHECK(c >= 0 && c < d->n_classes && P->h_class_len[c] == L, "box class length mismatch");
    max_len = std::max(max_len, L);
    for (int i = s; i < s + L; ++i) {
      if (first[i] < 0) first[i] = a;
      mult[i] += 1;
    }
  }
  for (int i = 0; i < nu; ++i) {
    HELM_CHECK(mult[i] >= 1, "an unknown is covered by no subdomain");
    HELM_CHECK(mult[i] <= 2, "more than two subdomains overlap along one dimension");
    if (mult[i] == 2) {
      band[i] = (int)band_node.size();
      band_node.push_back(i);
    }
  }
  const size_t smem = (size_t)(4 * max_len * max_len + 2 * max_len) * P->elem;
  HELM_CHECK(smem <= 200 * 1024, "subdomain too large for the shared-memory FDM kernel");
  dv.p = p;
  dv.max_len = max_len;
  dv.n_classes = d->n_classes;
  dv.nbands = (int)band_node.size();
  dv.box_start = upload<int>(d->box_start, p);
  dv.box_len = upload<int>(d->box_len, p);
  dv.box_class = upload<int>(d->box_class, p);
  dv.class_len = upload<int>(d->class_len, d->n_classes);
  std::vector<int> offV(d->n_classes), offL(d->n_classes);
  size_t totV = 0, totL = 0;
  for (int c = 0; c < d->n_classes; ++c) {
    offV[c] = (int)totV;
    offL[c] = (int)totL;
    totV += (size_t)P->h_class_len[c] * P->h_class_len[c];
    totL += P->h_class_len[c];
  }
  dv.class_off_V = upload<int>(offV.data(), offV.size());
  dv.class_off_lam = upload<int>(offL.data(), offL.size());
  dv.class_V = upload_bytes(d->class_V, totV * P->elem);
  dv.class_lambda = upload_bytes(d->class_lambda, totL * P->elem);
  // real classes (the middle-class pencil tridiag(-1,2,-1)/h^2 with W = I) get a real copy of V
  std::vector<int> creal(d->n_classes, 1);
  std::vector<double> vr(totV, 0.0);
  for (int c = 0; c < d->n_classes; ++c) {
    const size_t L = P->h_class_len[c];
    for (size_t e = 0; e < L * L; ++e) {
      const size_t i = offV[c] + e;
      if (d->is_complex) {
        const double* v = (const double*)d->class_V + 2 * i;
        vr[i] = v[0];
        if (v[1] != 0.0) creal[c] = 0;
      } else {
        vr[i] = ((const double*)d->class_V)[i];
      }
    }
    if (d->is_complex)
      for (size_t e = 0; e < L; ++e)
        if (((const double*)d->class_lambda)[2 * (offL[c] + e) + 1] != 0.0) creal[c] = 0;
  }
  dv.class_real = upload<int>(creal.data(), creal.size());
  dv.class_Vr = upload<double>(vr.data(), vr.size());
  // folded (symmetric) real classes: V[L-1-j][k] = sigma_k V[j][k]; even modes (sigma = +1)
  // are packed at [0, 20) and odd modes at [20, 40) of a 40 x 40 table (local_dmma.cu)
  constexpr int FT = 40, FH = 20;
  std::vector<int> cfold(d->n_classes, 0);
  std::vector<double> vf((size_t)d->n_classes * FT * FT, 0.0), lf((size_t)d->n_classes * FT, 1e30);  // pad: x / 1e30 = 0
  for (int c = 0; c < d->n_classes; ++c) {
    const int L = P->h_class_len[c];
    if (!creal[c] || L > FT) continue;
    const double* V = vr.data() + offV[c];  // V[j][k] row-major
    const double* lam = (const double*)d->class_lambda;
    const int h = L / 2, hp = (L + 1) / 2;
    double vmax = 0.0;
    for (int e = 0; e < L * L; ++e) vmax = std::max(vmax, std::fabs(V[e]));
    bool ok = true;
    int ne = 0, no = 0;
    for (int k = 0; k < L && ok; ++k) {
      const double sg = V[(L - 1) * L + k] * V[k] >= 0.0 ? 1.0 : -1.0;
      for (int j = 0; j < L && ok; ++j)
        if (std::fabs(V[(L - 1 - j) * L + k] - sg * V[j * L + k]) > 1e-12 * vmax) ok = false;
      if (!ok) break;
      const int col = sg > 0 ? ne++ : FH + no++;
      if (ne > hp || no > h) {
        ok = false;
        break;
      }
      const int rows = sg > 0 ? hp : h;
      for (int j = 0; j < rows; ++j) vf[((size_t)c * FT + (sg > 0 ? j : FH + j)) * FT + col] = V[j * L + k];
      lf[(size_t)c * FT + col] = d->is_complex ? lam[2 * (offL[c] + k)] : lam[offL[c] + k];
    }
    cfold[c] = ok && ne == hp && no == h;
  }
  // Dirichlet middle-pencil classes (tridiag(-1, 2, -1)/h^2, W = I) of length L = 4Q - 1,
  // Q in {5, 9}: every eigenvector is +-sqrt(2/N) sin(pi (j+1) m / N), N = L + 1, with
  // lambda_m = (2 - 2 cos(pi m / N)) / h^2 -- checked column by column against the plan's
  // pairs; such boxes take the fast-sine kernel (local_dst.cu).  HELM_DST=0 keeps them on
  // the DMMA kernel (A/B).
  const char* dst_env = getenv("HELM_DST");
  const bool dst_on = !(dst_env && dst_env[0] == '0');
  std::vector<int> cdst(d->n_classes, 0);
  int dst_q = 0;
  const long double pi_l = 3.14159265358979323846264338327950288L;
  for (int c = 0; c < d->n_classes && dst_on; ++c) {
    const int L = P->h_class_len[c];
    const int Q = (L + 1) / 4;
    if (!cfold[c] || (L + 1) % 4 != 0 || (Q != 5 && Q != 9) || (dst_q && Q != dst_q)) continue;
    const double* V = vr.data() + offV[c];
    const double* lam = (const double*)d->class_lambda;
    const long double nrm = sqrtl(2.0L / (L + 1));
    std::vector<int> used(L + 1, 0);
    bool ok = true;
    for (int k = 0; k < L && ok; ++k) {
      // the sine mode of column k: the largest projection
      int best = 0;
      long double bp = 0;
      for (int m = 1; m <= L; ++m) {
        long double pr = 0;
        for (int j = 0; j < L; ++j) pr += (long double)V[j * L + k] * nrm * sinl(pi_l * (j + 1) * m / (L + 1));
        if (fabsl(pr) > fabsl(bp)) bp = pr, best = m;
      }
      const long double sg = bp >= 0 ? 1.0L : -1.0L;
      for (int j = 0; j < L && ok; ++j)
        if (fabsl(V[j * L + k] - sg * nrm * sinl(pi_l * (j + 1) * best / (L + 1))) > 1e-12L) ok = false;
      const long double lx = (2.0L - 2.0L * cosl(pi_l * best / (L + 1))) * P->geo.inv_h2;
      const long double lp = d->is_complex ? lam[2 * (offL[c] + k)] : lam[offL[c] + k];
      if (fabsl(lp - lx) > 1e-12L * fabsl(4.0L * P->geo.inv_h2) || used[best]) ok = false;
      used[best] = 1;
    }
    if (ok) {
      cdst[c] = 1;
      dst_q = Q;
    }
  }
  // MP-2 Sommerfeld-end classes (one boundary node at either end of the box): the pencil is
  // T = tridiag(-1, 2, -1)/h^2 with tb = 1/h^2 - ik/h at the boundary node, W = I with 1/2
  // there (discretization.py:136-148), checked against the plan's eigen-pairs; for every sine
  // mode mu of the middle class, the Thomas factors of K_mu = T + (lam_mu - k^2) W (edge boxes,
  // local_dst.cu).  A pivot below 1e-6/h^2 in modulus keeps the class on the dense kernel.
  std::vector<int> ctri(d->n_classes, -1);
  std::vector<double2> tri;
  const bool edge_on = dst_q && d->is_complex && !env_flag_off("HELM_EDGE");
  for (int c = 0; c < d->n_classes && edge_on; ++c) {
    const int L = P->h_class_len[c];
    if (creal[c] || L > 40) continue;
    int s = -1;
    for (int a = 0; a < p; ++a)
      if (P->h_box_class[a] == c) s = P->h_box_start[a];
    const bool lo = s == 0, hi = s + L == nu;
    if (lo == hi) continue;  // both ends or neither: not an edge class
    const int ib = lo ? 0 : L - 1;
    typedef std::complex<long double> cl;
    const long double ih2 = P->geo.inv_h2;
    const cl tb((long double)P->geo.tb.x, (long double)P->geo.tb.y);
    auto Tdiag = [&](int i) { return i == ib ? tb : cl(2.0L * ih2); };
    auto Wd = [&](int i) { return i == ib ? 0.5L : 1.0L; };
    // the plan's pairs must be this pencil's: |T v - lam W v| small for every column
    const double2* V = (const double2*)d->class_V + offV[c];
    const double2* lam = (const double2*)d->class_lambda + offL[c];
    long double res = 0, vmax = 0;
    for (int k = 0; k < L; ++k) {
      const cl lk(lam[k].x, lam[k].y);
      for (int i = 0; i < L; ++i) {
        auto v = [&](int j) { return cl(V[j * L + k].x, V[j * L + k].y); };
        cl tv = Tdiag(i) * v(i);
        if (i > 0) tv -= ih2 * v(i - 1);
        if (i + 1 < L) tv -= ih2 * v(i + 1);
        res = std::max(res, std::abs(tv - lk * Wd(i) * v(i)));
        vmax = std::max(vmax, std::abs(v(i)));
      }
    }
    if (!(res <= 1e-9L * 4.0L * ih2 * vmax)) continue;
    const int N4 = 4 * dst_q;
    std::vector<double2> t((size_t)2 * 40 * N4, mk(0.0, 0.0));
    bool ok = true;
    for (int mu = 1; mu < N4 && ok; ++mu) {
      const long double sh = (2.0L - 2.0L * cosl(pi_l * mu / N4)) * ih2 - (long double)d->k * d->k;
      cl piv = Tdiag(0) + sh * Wd(0);
      for (int i = 0; i < L; ++i) {
        if (i > 0) {
          const cl l = -ih2 / piv;  // e / d_{i-1}
          piv = Tdiag(i) + sh * Wd(i) - l * (-ih2);
          t[(size_t)i * N4 + mu - 1] = mk((double)l.real(), (double)l.imag());
        }
        if (std::abs(piv) < 1e-6L * ih2) ok = false;
        const cl inv = 1.0L / piv;
        t[((size_t)40 + i) * N4 + mu - 1] = mk((double)inv.real(), (double)inv.imag());
      }
    }
    if (!ok) continue;
    ctri[c] = (int)(tri.size() / t.size());
    tri.insert(tri.end(), t.begin(), t.end());
  }
  std::vector<int> ff, rr, mix, dst, edge;
  for (int ay = 0; ay < p; ++ay)
    for (int ax = 0; ax < p; ++ax) {
      const int cy = P->h_box_class[ay], cx = P->h_box_class[ax];
      const bool ed = (cdst[cy] && ctri[cx] >= 0) || (ctri[cy] >= 0 && cdst[cx]);
      (cdst[cy] && cdst[cx] ? dst : ed ? edge : cfold[cy] && cfold[cx] ? ff : creal[cy] && creal[cx] ? rr : mix)
          .push_back(ay * p + ax);
    }
  dv.n_edge = (int)edge.size();
  dv.box_edge = edge.empty() ? nullptr : upload<int>(edge.data(), edge.size());
  dv.class_tri = upload<int>(ctri.data(), ctri.size());
  dv.edge_tri = tri.empty() ? nullptr : upload<double2>(tri.data(), tri.size());
  dv.n_dst = (int)dst.size();
  dv.dst_q = dst.empty() ? 0 : dst_q;
  dv.box_dst = dst.empty() ? nullptr : upload<int>(dst.data(), dst.size());
  dv.dst_inv = nullptr;
  if (!dst.empty()) {
    // (2/N)^2 / (lambda_my + lambda_mx - k^2) in sine-mode order [my][mx], exact eigenvalues
    const int N4 = 4 * dst_q, L = N4 - 1;
    std::vector<double> t((size_t)N4 * N4, 0.0);
    for (int my = 1; my <= L; ++my)
      for (int mx = 1; mx <= L; ++mx) {
        const long double ly = (2.0L - 2.0L * cosl(pi_l * my / N4)) * P->geo.inv_h2;
        const long double lx = (2.0L - 2.0L * cosl(pi_l * mx / N4)) * P->geo.inv_h2;
        const long double den = ly + lx - (long double)d->k * d->k;
        HELM_CHECK(fabsl(den) > 1e-14L * (8.0L * P->geo.inv_h2),
                   "singular subdomain matrix (lambda_y + lambda_x = k^2)");
        t[(size_t)(my - 1) * N4 + (mx - 1)] = (double)((2.0L / N4) * (2.0L / N4) / den);
      }
    dv.dst_inv = upload<double>(t.data(), t.size());
  }
  dv.n_ff = (int)ff.size();
  dv.n_rr = (int)rr.size();
  dv.n_mix = (int)mix.size();
  dv.box_ff = upload<int>(ff.data(), ff.size());
  dv.box_rr = upload<int>(rr.data(), rr.size());
  dv.box_mix = upload<int>(mix.data(), mix.size());
  dv.class_Vf = upload<double>(vf.data(), vf.size());
  dv.class_lamf = upload<double>(lf.data(), lf.size());
  // reciprocal eigenvalue sums per folded class pair: 1 / (lf_y[m] + lf_x[n] - k^2), padding 0
  std::vector<double> inv((size_t)d->n_classes * d->n_classes * FT * FT, 0.0);
  for (int cy = 0; cy < d->n_classes; ++cy)
    for (int cx = 0; cx < d->n_classes; ++cx) {
      if (!cfold[cy] || !cfold[cx]) continue;
      for (int m = 0; m < FT; ++m)
        for (int nn = 0; nn < FT; ++nn) {
          const double ly = lf[(size_t)cy * FT + m], lx = lf[(size_t)cx * FT + nn];
          if (ly > 1e29 || lx > 1e29) continue;
          inv[(((size_t)cy * d->n_classes + cx) * FT + m) * FT + nn] = 1.0 / (ly + lx - d->k * d->k);
        }
    }
  dv.class_invden = upload<double>(inv.data(), inv.size());
  dv.node_first_box = upload<int>(first.data(), nu);
  dv.node_mult = upload<int>(mult.data(), nu);
  dv.node_band = upload<int>(band.data(), nu);
  dv.band_node = band_node.empty() ? nullptr : upload<int>(band_node.data(), band_node.size());
}

static void finish_desc(helm_plan* P) {
  // pointer members of the stored descriptor are not owned: clear them
  P->desc.box_start = P->desc.box_len = P->desc.box_class = P->desc.class_len = nullptr;
  P->desc.class_V = P->desc.class_lambda = nullptr;
  P->desc.coarse_scale = P->desc.strip_q = P->desc.coarse_lamT = P->desc.coarse_lamM = nullptr;
  P->desc.t0_band = P->desc.m0_band = P->desc.band_l = P->desc.band_u = nullptr;
  P->desc.cap_left = P->desc.cap_right = P->desc.cap_mode = P->desc.cap_vt = P->desc.cap_hg = nullptr;
  P->desc.strip_lt = P->desc.strip_lm = nullptr;
  P->desc.band_piv = nullptr;
  P->desc.p_start = P->desc.pt_start = nullptr;
  P->desc.p_taps = P->desc.pt_taps = nullptr;
  P->desc.a0_stencil = P->desc.coarse_V = P->desc.coarse_invden = nullptr;
}

static void free_plan(helm_plan* P) {
  PlanDev& dv = P->dev;
  void* ptrs[] = {dv.box_start, dv.box_len, dv.box_class, dv.class_len, dv.class_off_V, dv.class_off_lam,
                  dv.class_V, dv.class_lambda, dv.class_real, dv.class_Vr, dv.box_ff, dv.class_Vf, dv.class_lamf, dv.class_invden, dv.box_dst, dv.dst_inv, dv.box_edge, dv.class_tri, dv.edge_tri, dv.box_rr, dv.box_mix,
                  dv.node_first_box, dv.node_mult, dv.node_band, dv.band_node,
                  dv.coarse_scale, dv.twiddle, dv.coarse_lamT, dv.coarse_lamM, dv.t0_band, dv.m0_band, dv.band_piv, dv.band_fac, dv.band_seg, dv.strip_q,
                  dv.cap_left, dv.cap_right, dv.cap_mode, dv.cap_vt, dv.cap_hg,
                  dv.p_start, dv.pt_start, dv.p_taps, dv.pt_taps, dv.a0_stencil, dv.coarse_V, dv.coarse_invden};
  for (void* q : ptrs)
    if (q) cudaFree(q);
}

template <typename F>
static void dispatch(const helm_plan* P, F&& f) {
  if (P->desc.is_complex)
    f(double2{});
  else
    f(double{});
}

}  // namespace helm

namespace helm {
// helm_plan_create's body, also used by the native setup (setup.cu)
int plan_create_from_desc(const helm_desc* desc, helm_plan** out) {
  return guarded([&] {
    HELM_CHECK(out != nullptr, "null output pointer");
    helm_plan* P = new helm_plan();
    try {
      build_plan(desc, P);
      finish_desc(P);
    } catch (...) {
      free_plan(P);
      delete P;
      throw;
    }
    *out = P;
  });
}
}  // namespace helm

using namespace helm;

extern "C" {

int32_t helm_abi_version(void) { return HELM_ABI_VERSION; }
uint64_t helm_kernel_launches(void) { return g_launches.load(); }
const char* helm_last_error(void) { return g_last_error.c_str(); }

int helm_plan_create(const helm_desc* desc, helm_plan** out) { return plan_create_from_desc(desc, out); }

int helm_plan_destroy(helm_plan* plan) {
  return guarded([&] {
    if (!plan) return;
    free_plan(plan);
    delete plan;
  });
}

int64_t helm_plan_num_unknowns(const helm_plan* plan) { return plan ? plan->N : -1; }
int64_t helm_plan_num_coarse(const helm_plan* plan) { return plan ? plan->N0 : -1; }

int helm_workspace_create(const helm_plan* P, int32_t max_batch, helm_workspace** out) {
  return guarded([&] {
    HELM_CHECK(P && out && max_batch >= 1, "bad workspace arguments");
    helm_workspace* w = new helm_workspace();
    std::memset(w, 0, sizeof(*w));
    w->plan = P;
    w->max_batch = max_batch;
    const size_t B = max_batch, e = P->elem;
    HELM_CUDA(cudaMalloc(&w->z, B * P->N * e));
    HELM_CUDA(cudaMalloc(&w->d, B * P->N * e));
    void** coarse[] = {&w->c, &w->g, &w->y0, &w->r0, &w->e0, &w->f0};
    for (void** q : coarse) HELM_CUDA(cudaMalloc(q, B * P->N0 * e));
    const size_t novl = std::max<size_t>(1, B * 6 * (size_t)P->dev.nbands * P->geo.nu);
    HELM_CUDA(cudaMalloc(&w->ovl, novl * e));
    for (int s = 0; s < 7; ++s)
      if (P->dev.n_strip)
        HELM_CUDA(cudaMalloc(&w->strip[s], (size_t)(s == 3 ? 8 : 1) * P->dev.m0 * B * P->dev.n_strip * e));
    if (P->dev.n_strip && max_batch > 4)
      HELM_CUDA(cudaMalloc(&w->strip_part, (size_t)((P->dev.m0 + 31) / 32) * P->dev.m0 * B * P->dev.n_strip * e));
    w->red_bytes = krylov_scratch_bytes(4096);
    HELM_CUDA(cudaMalloc(&w->red, w->red_bytes));
    HELM_CUDA(cudaMemset(w->red, 0, w->red_bytes));  // the CGS2 completion counters start at zero
    HELM_CUDA(cudaMallocHost(&w->pinned, 64 * sizeof(double)));
    // the side stream carries the long-latency boundary-box solves beside the tensor-core
    // boxes; the highest priority lets their CTAs take SM slots ahead of the many short ones
    int prio_lo = 0, prio_hi = 0;
    HELM_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const char* pe = std::getenv("HELM_SIDE_PRIO");
    const int prio = (pe && pe[0] == '0') ? prio_lo : prio_hi;
    HELM_CUDA(cudaStreamCreateWithPriority(&w->side, cudaStreamNonBlocking, prio));
    HELM_CUDA(cudaEventCreateWithFlags(&w->fork, cudaEventDisableTiming));
    HELM_CUDA(cudaEventCreateWithFlags(&w->join, cudaEventDisableTiming));
    *out = w;
  });
}

int helm_workspace_destroy(helm_workspace* w) {
  return guarded([&] {
    if (!w) return;
    basis_free(w);
    void* ptrs[] = {w->z, w->d, w->c, w->g, w->y0, w->r0, w->e0, w->f0, w->ovl, w->red, w->strip[0], w->strip[1],
                    w->strip[2], w->strip[3], w->strip[4], w->strip[5], w->strip[6], w->strip_part};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    if (w->pinned) cudaFreeHost(w->pinned);
    if (w->side) cudaStreamDestroy(w->side);
    if (w->fork) cudaEventDestroy(w->fork);
    if (w->join) cudaEventDestroy(w->join);
    delete w;
  });
}

#define HELM_BATCH_CHECK(ws, batch) \
  HELM_CHECK((batch) >= 1 && (!(ws) || (batch) <= (ws)->max_batch), "batch exceeds the workspace capacity")

int helm_apply_A(const helm_plan* P, const void* x, void* y, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && x && y && batch >= 1, "bad arguments");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      op_apply_A<S>(P, (const S*)x, (S*)y, batch, (cudaStream_t)stream);
    });
  });
}

int helm_deflate(const helm_plan* P, const void* x, const void* z, void* y, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && x && z && y && batch >= 1, "bad arguments");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      launch_stencil<S>(P->geo, (const S*)x, (const S*)z, (S*)y, batch, (cudaStream_t)stream);
    });
  });
}

int helm_restrict(const helm_plan* P, const void* x, void* c, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && x && c && batch >= 1, "bad arguments");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      restrict_any<S>(P, (const S*)x, (S*)c, batch, (cudaStream_t)stream);
    });
  });
}

int helm_prolong(const helm_plan* P, const void* c, void* z, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && c && z && batch >= 1, "bad arguments");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      prolong_any<S>(P, (const S*)c, (S*)z, batch, (cudaStream_t)stream);
    });
  });
}

int helm_coarse_solve(const helm_plan* P, helm_workspace* ws, const void* c, void* y, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && c && y, "bad arguments");
    HELM_BATCH_CHECK(ws, batch);
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      coarse_solve_any<S>(P, ws, (const S*)c, (S*)y, batch, (cudaStream_t)stream);
    });
  });
}

int helm_coarse_correct(const helm_plan* P, helm_workspace* ws, const void* x, void* z, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && x && z, "bad arguments");
    HELM_BATCH_CHECK(ws, batch);
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      op_coarse_correct<S>(P, ws, (const S*)x, (S*)z, batch, (cudaStream_t)stream);
    });
  });
}

int helm_local_sum(const helm_plan* P, helm_workspace* ws, const void* x, const void* base, void* y,
                   int32_t weighted, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && x && y, "bad arguments");
    HELM_CHECK(x != y, "local_sum: input and output must not alias");
    HELM_BATCH_CHECK(ws, batch);
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      launch_local_sum<S>(P, (const S*)x, (const S*)base, (S*)y, (S*)ws->ovl, weighted ? 1 : 0, batch,
                          P->dev.band_node, (cudaStream_t)stream, /*coarse_base=*/false, ws);
    });
  });
}

int helm_apply_M(const helm_plan* P, helm_workspace* ws, const void* x, void* y, int32_t batch, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && x && y, "bad arguments");
    HELM_BATCH_CHECK(ws, batch);
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      op_apply_M<S>(P, ws, (const S*)x, (S*)y, batch, (cudaStream_t)stream);
    });
  });
}

int helm_cgs2(const helm_plan* P, helm_workspace* ws, void* V, int32_t j, void* hcol, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && V && hcol && j >= 0, "bad arguments");
    HELM_CHECK(krylov_scratch_bytes(j + 1) <= ws->red_bytes, "basis too large for the workspace scratch");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      krylov_cgs2<S>((S*)V, j, (size_t)P->N, (size_t)P->N, (S*)hcol, ws->red, (cudaStream_t)stream);
    });
  });
}

int helm_givens(const helm_plan* P, void* H, int32_t ldh, int32_t j, void* cs, void* sn, void* g, double beta,
                double* est_out, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && H && cs && sn && g && est_out && j >= 0 && ldh > j, "bad arguments");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      krylov_givens<S>((S*)H, ldh, j, (S*)cs, (S*)sn, (S*)g, beta, est_out, (cudaStream_t)stream);
    });
  });
}

int helm_gmres(const helm_plan* P, helm_workspace* ws, const void* b, void* x, double rtol, int32_t max_iter,
               int32_t side, int32_t use_precond, double* history, helm_gmres_report* report, void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && b && x && report, "bad arguments");
    HELM_CHECK(b != x, "gmres: b and x must not alias");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      gmres_impl<S>(P, ws, (const S*)b, (S*)x, rtol, max_iter, side, use_precond, history, report,
                    (cudaStream_t)stream);
    });
  });
}

int helm_gmres_multi(const helm_plan* P, helm_workspace* ws, const void* b, void* x, int32_t nrhs, double rtol,
                     int32_t max_iter, int32_t side, int32_t use_precond, double* history, helm_gmres_report* reports,
                     void* stream) {
  return guarded([&] {
    HELM_CHECK(P && ws && b && x && reports, "bad arguments");
    HELM_CHECK(b != x, "gmres: b and x must not alias");
    dispatch(P, [&](auto t) {
      using S = decltype(t);
      gmres_multi_impl<S>(P, ws, (const S*)b, (S*)x, nrhs, rtol, max_iter, side, use_precond, history, reports,
                          (cudaStream_t)stream);
    });
  });
}

}  // extern "C"
