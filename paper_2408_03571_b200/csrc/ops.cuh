// Internal launcher declarations shared between the kernel translation units.
#pragma once
#include "common.cuh"

namespace helm {

template <typename S> void launch_stencil(const Geo& g, const S* x, const S* z, S* y, int batch, cudaStream_t st);
template <typename S> void launch_restrict(const Geo& g, const S* x, S* c, int batch, cudaStream_t st);
template <typename S> void launch_prolong(const Geo& g, const S* c, S* z, int batch, cudaStream_t st);
template <typename S>
void launch_prolong_deflate(const Geo& g, const S* c, const S* x, S* z, S* d, int batch, cudaStream_t st);
template <typename S>
void launch_local_sum(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, int weighted, int batch,
                      const int* band_node, cudaStream_t st, bool coarse_base = false,
                      helm_workspace* ws = nullptr);
template <typename S>
void launch_coarse_solve(const helm_plan* P, helm_workspace* ws, const S* c, S* y, int batch, cudaStream_t st);

// general coarse spaces (coarse_dense.cu)
template <typename S> void launch_restrict_general(const helm_plan* P, const S* x, S* c, int batch, cudaStream_t st);
template <typename S> void launch_prolong_general(const helm_plan* P, const S* c, S* z, int batch, cudaStream_t st);
template <typename S>
void launch_coarse_solve_dense(const helm_plan* P, helm_workspace* ws, const S* c, S* y, int batch, cudaStream_t st);

// coarse-solve building blocks (xform.cu, band.cu)
template <typename S>
void launch_xform(const helm_plan* P, const S* in, S* out, const double* sig, bool scale2d, int batch,
                  cudaStream_t st, bool accumulate = false);
template <typename S> void launch_transpose(const S* in, S* out, int m, int batch, cudaStream_t st);
size_t band_seg_table_elems(int m0);
bool band_seg_usable(int m0);
void band_seg_setup(const PlanDev& d, double2* tables, cudaStream_t st);
void band_seg_launch(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                     cudaStream_t st, const double2* add);
void launch_band_solve(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                       cudaStream_t st, const double2* add = nullptr);

bool band_tma_usable(const helm_plan* P);
void band_tma_launch(const helm_plan* P, const double2* in, double2* out, const double2* corr, int batch,
                     cudaStream_t st, const double2* add, double2* part);
bool band_vals_usable(const helm_plan* P, int batch);
void launch_band_vals(const helm_plan* P, const double2* in, double2* scratch, const double2* corr, int batch,
                      cudaStream_t st, double2* part, const double2* Zadd, double2* Z);

// composite operators (capi.cu)
template <typename S> void op_apply_A(const helm_plan* P, const S* x, S* y, int batch, cudaStream_t st);
template <typename S>
void op_apply_M(const helm_plan* P, helm_workspace* ws, const S* x, S* y, int batch, cudaStream_t st);

// Krylov kernels (krylov.cu)
template <typename S> void krylov_norm2(const S* x, size_t N, double* out, void* scratch, cudaStream_t st);
template <typename S>
void krylov_combine(S* x, const S* V, int nvec, size_t ldv, const S* h, size_t N, cudaStream_t st);
template <typename S>
void krylov_cgs2_impl(S* V, int j, size_t ldv, size_t N, S* hcol, size_t hstride, double* inv_out, void* scratch,
                      cudaStream_t st, S* H = nullptr, int ldh = 0, S* cs = nullptr, S* sn = nullptr,
                      S* g = nullptr, double beta = 1.0, double* est_out = nullptr);
template <typename S>
void krylov_cgs2(S* V, int j, size_t ldv, size_t N, S* hcol, void* scratch, cudaStream_t st);
template <typename S>
void krylov_givens(S* H, int ldh, int j, S* cs, S* sn, S* g, double beta, double* est, cudaStream_t st);
template <typename S> void krylov_backsolve(const S* H, int ldh, int j, const S* g, S* y, cudaStream_t st);
template <typename S> void krylov_scale(S* x, const S* src, const double* s, int invert, size_t N, cudaStream_t st);

size_t krylov_scratch_bytes(int max_vec);

// Krylov basis storage (basis.cu): returns the base of a contiguous device range with
// at least `need` bytes backed; the base moves only when `need` exceeds the reservation.
void* basis_ensure(helm_workspace* ws, size_t need, size_t reserve_hint, size_t chunk_min, cudaStream_t st);
void basis_free(helm_workspace* ws);

}  // namespace helm
