// Microbenchmark: FP64 throughput on sm_100a — DFMA (CUDA cores) vs DMMA.8x8x4 (mma.sync f64).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {128, 256, 512, 1024}) {
    int iters = 20000; int blocks = sms * (threads <= 512 ? 2 : 1);
    dfma_kernel<8><<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * (double)iters * threads * blocks;
    printf("DFMA  threads=%4d blocks=%d : %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int iters = 20000; int blocks = sms * 2;
    dmma_kernel<8><<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    dmma_kernel<8><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
    printf("DMMA  threads=%4d blocks=%d : %.2f TFLOP/s\n", threads, blocks, fl / ms / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
