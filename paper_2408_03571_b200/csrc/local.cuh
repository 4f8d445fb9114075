// Shared declarations of the one-level Schwarz kernels (local.cu, local_fast.cu).
#pragma once
#include "ops.cuh"

namespace helm {

struct LocalArgs {
  int nu;
  int p;
  int nbands;
  double k2;
  int weighted;
  int wbs;  // weights before solve
  const int* box_start;
  const int* box_len;
  const int* box_class;
  const int* class_len;
  const int* class_off_V;
  const int* class_off_lam;
  const int* node_first_box;
  const int* node_mult;
  const int* node_band;
};

// Register-blocked FDM for boxes of at most 36 nodes per side (local_fast.cu).
// Returns false (nothing launched) when the plan's boxes are larger.
template <typename S>
bool launch_local_fast(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st);

// Folded boxes (both classes real and symmetric) on the FP64 tensor pipe (local_dmma.cu).
template <typename S>
void launch_local_dmma(const helm_plan* P, const S* x, const S* base, S* y, S* ovl, const LocalArgs& a, int batch,
                       cudaStream_t st);

}  // namespace helm
