// Does shared-memory traffic slow FP64 tensor-core (DMMA) issue on B200?
// Each warp: per iteration 18 16-byte loads (LDS or L1-resident LDG) feeding 54 DMMA.8x8x4,
// register double-buffered like the SSE Sigma kernel.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int MODE>  // 0: no loads, 1: LDS, 2: LDG (L1 resident)
__global__ void __launch_bounds__(256, 1) k(const double2* g, double* out, int iters) {
  __shared__ double2 sm[2048];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2048; i += 256) sm[i] = g[i];
  __syncthreads();
  double acc[9][2] = {};
  double2 cur[18], nxt[18];
  for (int j = 0; j < 18; ++j) cur[j] = make_double2(lane * 1e-3 + j, j);
  for (int it = 0; it < iters; ++it) {
    const int base = ((it * 7 + warp) & 7) * 512;
    if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 18; ++j) nxt[j] = sm[(base + j * 32 + lane) & 2047];
    } else if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 18; ++j) nxt[j] = __ldg(g + ((base + j * 32 + lane) & 4095));
    } else {
#pragma unroll
      for (int j = 0; j < 18; ++j) nxt[j] = cur[j];
    }
#pragma unroll
    for (int kk = 0; kk < 6; ++kk)
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int n = 0; n < 3; ++n) dmma(acc[t * 3 + n], cur[t * 3 + kk % 3].x, cur[9 + (kk * 3 + n) % 9].y);
#pragma unroll
    for (int j = 0; j < 18; ++j) cur[j] = nxt[j];
  }
  double s = 0;
  for (int i = 0; i < 9; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[0] = s;
}

int main() {
  double2* g; double* out;
  cudaMalloc(&g, 4096 * 16); cudaMemset(g, 0, 4096 * 16); cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 20000, grid = 148;
  void (*ks[3])(const double2*, double*, int) = {k<0>, k<1>, k<2>};
  const char* names[3] = {"no loads", "LDS.128 x18", "LDG.128 x18 (L1)"};
  for (int m = 0; m < 3; ++m) {
    ks[m]<<<grid, 256>>>(g, out, 100);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    ks[m]<<<grid, 256>>>(g, out, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 256 * 54.0 * iters * 8 * grid;
    printf("%-20s %.2f TFLOP/s\n", names[m], flops / ms / 1e9);
  }
  return 0;
}
