// Do DMMA (FP64 tensor) and DFMA (FP64 vector) share one pipe on B200?  Half the
// warps of each CTA issue DMMA.8x8x4, the other half DFMA; if the pipes were
// independent the mixed kernel would exceed either peak alone.
#include <cstdio>
#include <cuda_runtime.h>

#define CHK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void mixed_kernel(double* out, int iters_m, int iters_f, int dmma_warps) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < dmma_warps) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    double a = 1.0000001 + threadIdx.x * 1e-6, b = 1e-9 - threadIdx.x * 1e-12;
    for (int it = 0; it < iters_m; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 1.0000001, 1e-9);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p; CHK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  double* out; CHK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, warps = threads / 32;
  struct Case { int dmma_warps; int iters_m; int iters_f; };
  const Case cases[] = {{16, 4000, 0}, {0, 0, 32000}, {8, 4000, 32000}, {8, 4000, 16000}, {12, 4000, 32000},
                        {4, 4000, 32000}};
  for (const Case& c : cases) {
    dim3 grid(sms * 2);
    mixed_kernel<<<grid, threads>>>(out, 10, 80, c.dmma_warps);
    CHK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    mixed_kernel<<<grid, threads>>>(out, c.iters_m, c.iters_f, c.dmma_warps);
    cudaEventRecord(e1); CHK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fm = 2.0 * 256 * 8 * (double)c.iters_m * c.dmma_warps * grid.x;
    const double ff = 2.0 * 8 * (double)c.iters_f * 32 * (warps - c.dmma_warps) * grid.x;
    printf("dmma_warps=%2d/%d iters_m=%d iters_f=%d: %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n",
           c.dmma_warps, warps, c.iters_m, c.iters_f, ms, fm / ms / 1e9, ff / ms / 1e9, (fm + ff) / ms / 1e9);
  }
  return 0;
}
