// K6's V-ring protocol around its inner loop, in isolation: V sub-stages are loaded by TMA bulk
// copies (cp.async.bulk global -> shared, full/empty mbarriers, producer = lane 0 of warp t % 4,
// SL - 1 sub-stages ahead) from a 2 GB buffer; each warp runs 2 m-tiles x 9 n-tiles of DMMA.8x8x4
// per quad as K6 (B from the slot by LDS.64 + sign XOR, A from registers).  4 warps x 3 CTAs / SM.
// QS = quads per sub-stage: 6 (K6: 4 slots of 13.8 KB) vs 12 (2 slots of 27.6 KB, same 55 KB).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double xsign(double v, unsigned m) {
  return __hiloint2double(__double2hiint(v) ^ (int)m, __double2loint(v));
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

template <int QS, int SL>
__global__ void __launch_bounds__(128, 3) k(const double* __restrict__ v, double* out, int nsub, long long vspan) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int SLOT = QS * 4 * 36 * 2;  // doubles per slot (QS quads x 4 rows x 36 complex)
  double* ring = reinterpret_cast<double*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + SL * SLOT + 128);
  uint64_t* empty = full + SL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SL; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int pcol = lane & 3, nc = lane >> 2, im = nc & 1;
  const int b_dim = im ? -1 : 1;
  const unsigned mask = im ? 0u : 0x80000000u;
  const long long base = ((long long)blockIdx.x * 7919 * SLOT) % (vspan - (long long)nsub * SLOT - SLOT);
  auto produce = [&](int t) {
    const int slot = t % SL;
    if (t >= SL) mbar_wait(empty + slot, ((t - SL) / SL) & 1);
    mbar_expect(full + slot, SLOT * 8);
    bulk_g2s(ring + slot * SLOT, v + base + (long long)t * SLOT, SLOT * 8, full + slot);
  };
  if (threadIdx.x == 0)
    for (int t = 0; t < SL - 1 && t < nsub; ++t) produce(t);
  double acc[2][9][2] = {};
  double2 a[2] = {make_double2(1e-3 * lane, 2e-3), make_double2(3e-3, 1e-3 * warp)};
  int slot = 0;
  unsigned phase = 0;
  for (int ss = 0; ss < nsub; ++ss) {
    const int t = ss + SL - 1;
    if (lane == 0 && t < nsub && t % 4 == warp) produce(t);
    __syncwarp();
    mbar_wait(full + slot, phase);
    const double* sb = ring + slot * SLOT + pcol * 72 + 2 * (nc >> 1) + im;
#pragma unroll
    for (int q = 0; q < QS; ++q) {
      const double* b = sb + q * 288;
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const double br = b[8 * u];
        dmma(acc[0][u], a[0].x, br);
        dmma(acc[1][u], a[1].x, br);
      }
#pragma unroll
      for (int u = 0; u < 9; ++u) {
        const double bi = xsign(b[8 * u + b_dim], mask);
        dmma(acc[0][u], a[0].y, bi);
        dmma(acc[1][u], a[1].y, bi);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);
    if (++slot == SL) { slot = 0; phase ^= 1u; }
  }
  double s = 0;
#pragma unroll
  for (int t2 = 0; t2 < 2; ++t2)
#pragma unroll
    for (int u = 0; u < 9; ++u) s += acc[t2][u][0] + acc[t2][u][1];
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int QS, int SL>
static void run(const double* v, double* out, int sms, long long vspan) {
  constexpr int SLOT = QS * 4 * 36 * 2;
  const size_t smem = (size_t)SL * SLOT * 8 + 128 * 8 + 2 * SL * 8;
  cudaFuncSetAttribute(k<QS, SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k<QS, SL>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int blocks = sms * 3 * 8, quads = 4104, nsub = quads / QS;
  k<QS, SL><<<blocks, 128, smem>>>(v, out, 4, vspan);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<QS, SL><<<blocks, 128, smem>>>(v, out, nsub, vspan);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = (double)blocks * 4 * nsub * QS * 36 * 512;
  printf("QS %2d SL %d (%5.1f KB ring): %.2f TF/s  %s\n", QS, SL, SL * SLOT * 8 / 1024.0, flop / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long vspan = (2LL << 30) / 8;  // 2 GB of doubles
  double *v, *out;
  cudaMalloc(&v, vspan * 8);
  cudaMemset(v, 0, vspan * 8);
  cudaMalloc(&out, (size_t)sms * 3 * 8 * 128 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    run<6, 4>(v, out, sms, vspan);
    run<12, 2>(v, out, sms, vspan);
    run<6, 3>(v, out, sms, vspan);
    run<12, 1>(v, out, sms, vspan);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
