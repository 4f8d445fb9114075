// Do the FP64 tensor pipe (DMMA) and the FP64 FMA pipe (DFMA) run concurrently on sm_100a?
// Warps 0..W_mma-1 of every CTA issue DMMA chains, the others DFMA chains; reports the combined
// FP64 rate.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mixed tools/fp64_mixed.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mixed(double* out, int iters, int mma_warps, int interleave) {
  const int w = threadIdx.x / 32;
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  double f0 = a, f1 = a + 1, f2 = a + 2, f3 = a + 3, f4 = a + 4, f5 = a + 5, f6 = a + 6, f7 = a + 7;
  const double bb = 0.999999, cc = 1e-7;
  const bool do_mma = interleave ? true : (w < mma_warps);
  const bool do_fma = interleave ? true : (w >= mma_warps);
  for (int i = 0; i < iters; ++i) {
    if (do_mma) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < 4; ++t)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    if (do_fma) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        f0 = fma(f0, bb, cc); f1 = fma(f1, bb, cc); f2 = fma(f2, bb, cc); f3 = fma(f3, bb, cc);
        f4 = fma(f4, bb, cc); f5 = fma(f5, bb, cc); f6 = fma(f6, bb, cc); f7 = fma(f7, bb, cc);
      }
    }
  }
  double s = f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 4000, warps = threads / 32;
  for (int cfg = 0; cfg <= warps + 1; ++cfg) {
    const int interleave = cfg == warps + 1, mw = interleave ? 0 : cfg;
    mixed<<<blocks, threads>>>(out, 10, mw, interleave);
    cudaEventRecord(e0);
    mixed<<<blocks, threads>>>(out, iters, mw, interleave);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double nw = (double)blocks * warps;
    const double mma_w = interleave ? nw : nw * mw / warps, fma_w = interleave ? nw : nw - mma_w;
    const double fl = mma_w * iters * 16 * 2.0 * 256 + fma_w * 32 * iters * 128 * 2.0;
    printf("%s mma_warps=%d/%d: %.2f TFLOP/s (%.3f ms)\n", interleave ? "interleaved" : "split", mw, warps,
           fl / ms / 1e9, ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
