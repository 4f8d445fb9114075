// Microbenchmark: FP64 FMA (DFMA) vs FP64 MMA (DMMA m8n8k4) throughput on sm_100a,
// plus cuBLAS DGEMM/ZGEMM at the coarse-solve shapes. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu -lcublas
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cuComplex.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 4000;
  float ms;
  dfma_loop<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * blocks * threads * (double)iters * 16 * 8;
  printf("DFMA: %.2f TFLOP/s\n", fl / ms / 1e9);
  dmma_loop<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 8 * 8 * 4 * (blocks * threads / 32) * (double)iters * 16;
  printf("DMMA m8n8k4: %.2f TFLOP/s\n", fl / ms / 1e9);
  dmma16_loop<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0); dmma16_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 16 * 8 * 4 * (blocks * threads / 32) * (double)iters * 16;
  printf("DMMA m16n8k4: %.2f TFLOP/s  err=%s\n", fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));

  cublasHandle_t h; cublasCreate(&h);
  for (int m : {257, 513, 1025}) {
    for (int batch : {1, 32}) {
      size_t n2 = (size_t)m * m;
      cuDoubleComplex *A, *B, *C;
      cudaMalloc(&A, n2 * 16 * batch); cudaMalloc(&B, n2 * 16); cudaMalloc(&C, n2 * 16 * batch);
      cudaMemset(A, 0, n2 * 16 * batch); cudaMemset(B, 0, n2 * 16);
      cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
      // C (m x m*batch) = B (m x m) * A (m x m*batch): the x-transform of a batch of coarse vectors
      for (int w = 0; w < 2; ++w)
        cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m * batch, m, &one, B, m, A, m, &zero, C, m);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r)
        cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m * batch, m, &one, B, m, A, m, &zero, C, m);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double f = 8.0 * m * (double)m * m * batch * 5;
      printf("ZGEMM m=%d batch=%d: %.3f ms/call  %.2f TFLOP/s\n", m, batch, ms / 5, f / ms / 1e9);
      double *dA = (double*)A, *dB = (double*)B, *dC = (double*)C, onef = 1, zerof = 0;
      // real V times complex-as-2-real-columns
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r)
        cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, 2 * m * batch, m, &onef, dB, m, dA, m, &zerof, dC, m);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      f = 2.0 * m * (double)m * m * 2 * batch * 5;
      printf("DGEMM m=%d cols=2*m*%d: %.3f ms/call  %.2f TFLOP/s\n", m, batch, ms / 5, f / ms / 1e9);
      cudaFree(A); cudaFree(B); cudaFree(C);
    }
  }
  // copy bandwidth
  size_t bytes = (size_t)2 << 30;
  char *x, *y; cudaMalloc(&x, bytes); cudaMalloc(&y, bytes);
  cudaMemcpy(y, x, bytes, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e0); for (int r = 0; r < 5; ++r) cudaMemcpy(y, x, bytes, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("D2D copy: %.1f GB/s\n", 2.0 * bytes * 5 / ms / 1e6);
  printf("final err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
