// FP64 peak microbenchmark for B200 (sm_100a): DFMA (vector) vs DMMA (mma.sync m8n8k4 f64).
// Purpose: measure the denominator for the SSE roofline (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = a0 + threadIdx.x * 1e-6, b = b0 - threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CHK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out; CHK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int iters = 20000;
      dim3 grid(sms * bps);
      dfma_kernel<8><<<grid, threads>>>(out, 100, 1.0000001, 1e-9);
      CHK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * (double)iters * threads * grid.x;
      printf("DFMA threads=%d ctas/SM=%d: %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 4000;
      dim3 grid(sms * bps);
      dmma_kernel<8><<<grid, threads>>>(out, 100, 1.0000001, 1e-9);
      CHK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * grid.x;
      printf("DMMA threads=%d ctas/SM=%d: %.2f TFLOP/s (%.3f ms)\n", threads, bps, flops / ms / 1e9, ms);
    }
  }
  // sustained: long DFMA run (~3 s) to see power-capped clock
  {
    int threads = 512; dim3 grid(sms * 2); int iters = 2000000;
    cudaEventRecord(e0);
    dfma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * grid.x;
    printf("DFMA sustained: %.2f TFLOP/s (%.1f ms)\n", flops / ms / 1e9, ms);
  }
  {
    int threads = 256; dim3 grid(sms * 2); int iters = 400000;
    cudaEventRecord(e0);
    dmma_kernel<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * grid.x;
    printf("DMMA sustained: %.2f TFLOP/s (%.1f ms)\n", flops / ms / 1e9, ms);
  }
  return 0;
}
