// The K6 (Pi chains) inner loop in isolation: per warp 2 m-tiles x 9 n-tiles of FP64 accumulators;
// per kappa quad 9 n-tiles x {LDS.64 Re -> 2 DMMA, LDS.64 Im + sign XOR -> 2 DMMA} = 36 DMMA.8x8x4,
// A operands prefetched two quads ahead from L1/L2-resident global memory.  4 warps per CTA, 3 CTAs
// per SM (launch bounds 128, 3), as the production K6.  MODE 0: as K6; 1: no sign XOR; 2: B from
// registers (no LDS); 3: A from registers too (DMMA issue alone); 4: as 0 with the A rows spread
// over 1 GB (L2 / DRAM, as K6's G1 rows); 5: as 4 plus a per-sub-stage (6 quads) __syncwarp and a
// CTA-wide mbarrier round (every warp arrives, then waits for the phase) like K6's V-slot protocol.
// Prints DMMA TF/s per mode.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double xsign(double v, unsigned m) {
  return __hiloint2double(__double2hiint(v) ^ (int)m, __double2loint(v));
}

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(128, 3) k(const double2* __restrict__ g, double* out, int quads, long long span) {
  __shared__ double ring[3 * 864 * 2];
  __shared__ unsigned long long bar;  // 3 V slots of 13.8 KB (K6 uses 4; static smem <= 48 KB)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 3 * 864 * 2; i += 128) ring[i] = 1e-3 * (i & 255);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(4) : "memory");
  __syncthreads();
  unsigned phase = 0;
  const int pcol = lane & 3, nc = lane >> 2, im = nc & 1;
  const int b_dim = im ? -1 : 1;
  const unsigned mask = im ? 0u : 0x80000000u;
  double acc[2][9][2] = {};
  // A rows: per quad a 16-row stride (as K6's per-lane G1 blocks), spread over `span` double2
  const long long wbase = MODE >= 4 ? ((long long)(blockIdx.x * 4 + warp) * 9973 * 16) % (span - (1 << 20)) : (blockIdx.x * 4 + warp) * 64;
  const double2* ga = g + wbase + pcol;
  double2 a0[2] = {__ldg(ga), __ldg(ga + 4)}, a1[2] = {__ldg(ga + 8), __ldg(ga + 12)};
  double breg[18];
#pragma unroll
  for (int u = 0; u < 18; ++u) breg[u] = 1e-3 * (u + lane);
  for (int q = 0; q < quads; q += 2) {
    const double* sb = ring + ((q >> 1) % 3) * 1728 + pcol * 72 + 2 * (nc >> 1) + im;
    auto quad = [&](const double2 (&a)[2], const double* b) {
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const double br = MODE >= 2 ? breg[u] : b[8 * u];
        dmma(acc[0][u], a[0].x, br);
        dmma(acc[1][u], a[1].x, br);
      }
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        double bi = MODE >= 2 ? breg[9 + u] : b[8 * u + b_dim];
        if (MODE == 0) bi = xsign(bi, mask);
        dmma(acc[0][u], a[0].y, bi);
        dmma(acc[1][u], a[1].y, bi);
      }
    };
    quad(a0, sb);
    auto arow = [&](int qq) -> const double2* {
      if (MODE >= 4) return g + wbase + (long long)qq * 144 + pcol;  // a new 2.3 KB block every quad (< 1M past wbase)
      return ga + (qq & 15) * 16;
    };
    if (MODE != 3) {
      const double2* p = arow(q + 2);
      a0[0] = __ldg(p);
      a0[1] = __ldg(p + 4);
    }
    quad(a1, sb + 288);
    if (MODE != 3) {
      const double2* p = arow(q + 3);
      a1[0] = __ldg(p);
      a1[1] = __ldg(p + 4);
    }
    if (MODE == 5 && (q % 6) == 4) {  // end of a 6-quad sub-stage: release + wait, as K6's ring
      __syncwarp();
      if (lane == 0) {
        unsigned long long st;
        asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(su32(&bar)) : "memory");
      }
      __syncwarp();
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(&bar)), "r"(phase) : "memory");
      phase ^= 1u;
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < 9; ++u) s += acc[t][u][0] + acc[t][u][1];
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MODE>
static void run(const double2* g, double* out, int sms, long long span) {
  const int blocks = sms * 3 * 8, quads = 4098;
  k<MODE><<<blocks, 128>>>(g, out, 18, span);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 128>>>(g, out, quads, span);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = (double)blocks * 4 * quads * 36 * 512;
  printf("MODE %d: %.2f TF/s (%s)\n", MODE, flop / ms / 1e9,
         MODE == 0 ? "K6 pattern: 2 LDS.64 + XOR per 4 DMMA" : MODE == 1 ? "no sign XOR" :
         MODE == 2 ? "B from registers (no LDS)" : MODE == 3 ? "A and B from registers" :
         MODE == 4 ? "K6 pattern, A rows over 1 GB (L2 / DRAM)" : "as 4 + a CTA mbarrier round per 6 quads");
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2* g;
  double* out;
  const long long span = (1LL << 30) / 16;  // 1 GB of double2
  cudaMalloc(&g, span * 16);
  cudaMemset(g, 0, span * 16);
  cudaMalloc(&out, (size_t)sms * 3 * 8 * 128 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>(g, out, sms, span);
    run<1>(g, out, sms, span);
    run<2>(g, out, sms, span);
    run<3>(g, out, sms, span);
    run<4>(g, out, sms, span);
    run<5>(g, out, sms, span);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
