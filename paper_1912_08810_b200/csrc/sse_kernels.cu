// libsse kernels for B200 (sm_100a).
//
//   K1 layout transform      [Nkz,NE,NA,blk] <-> [NA,Nkz,NE,blk]    HBM-bound
//   K2 operator build        M[q,w,a,s] = wt_w sum_ij Dc_ij dH_i@dH_j (fragment order)
//   K3 fused Sigma kernel    Sigma[k,E,a] = i sum_{q,s,w} G[k-q,E-off_w,f(a,s)] @ M[q,w,a,s]
//                            on FP64 tensor cores (mma.sync m8n8k4 -> DMMA.8x8x4)
//   K3g generic Sigma        same contraction with DFMA, for No > kMaxDmmaOrb
//   preprocess_D             Dc = D_ba - D_bb - D_aa + D_ab            (sse.py:91-115)
//   fill_synthetic           atom-keyed counter-based inputs (bench / parity at scale)
//
// Reference semantics (sse.py:58-76, 127-161): momentum wraps mod Nkz, energy
// terms with E - off_w < 0 are dropped, neighbour indirection f(a,s) = nmap[a,s],
// final factor i.  The reassociation G@dH_i@Xi_i summed over i == G@M is exact
// algebra; results agree with the reference to rounding (tests/).
#include "sse_kernels.cuh"

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

namespace sse {

// last launched kernel per kind (bench / smoke evidence of which variant ran); the per-device
// host threads of the multi-GPU entry points launch concurrently, so writes and reads are serialised
// and a reader gets its own (thread-local) copy
static char g_kernel_name[7][192];
static std::mutex g_kernel_name_mu;
static void note_kernel(int kind, const char* fmt, ...) {
  char buf[sizeof(g_kernel_name[0])];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  std::lock_guard<std::mutex> lk(g_kernel_name_mu);
  memcpy(g_kernel_name[kind], buf, sizeof(buf));
}
const char* last_kernel_name(int kind) {
  thread_local char out[sizeof(g_kernel_name[0])];
  if (kind < 0 || kind >= 7) return "";
  std::lock_guard<std::mutex> lk(g_kernel_name_mu);
  memcpy(out, g_kernel_name[kind], sizeof(out));
  return out;
}

// --------------------------------------------------------------------------
// K1: layout transform.  One warp per (k, E, a) block of blk_vec 16-byte
// vectors; reads and writes are contiguous 16-byte runs per block.
// --------------------------------------------------------------------------
__global__ void layout_transform_kernel(long long nkz, long long ne, long long na, long long blk_vec,
                                        int to_atom_major, const double2* __restrict__ src,
                                        double2* __restrict__ dst) {
  const long long nblocks = nkz * ne * na;
  const int lane = threadIdx.x & 31;
  long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (; warp < nblocks; warp += nwarps) {
    // warp indexes the grid-major block (k, e, a)
    const long long a = warp % na;
    const long long ke = warp / na;             // k * ne + e
    const long long am = a * (nkz * ne) + ke;   // atom-major block index
    const long long from = to_atom_major ? warp : am;
    const long long to = to_atom_major ? am : warp;
    const double2* s = src + from * blk_vec;
    double2* d = dst + to * blk_vec;
    for (long long v = lane; v < blk_vec; v += 32) d[v] = __ldg(s + v);
  }
}

// --------------------------------------------------------------------------
// Slab pull: assemble an electron-tensor atom slab from the GF
// (k,E)-point layout.  Point pt lives on rank r (pt_lo[r] <= pt < pt_lo[r+1])
// as src[r][pt - pt_lo[r]][NA][No*No]; the slab's atoms [atom0, atom0+natoms)
// of one point are one contiguous source run, read here over NVLink when r is
// a peer (CUDA IPC mapping).  grid.y = point, grid.x = pieces of the run; each
// thread keeps kPullUnroll 16-byte loads in flight.  Points are visited from
// pt_shift on (the caller's own first point), so while every rank pulls at once
// each owner serves one reader at a time instead of all of them reading rank 0.
// --------------------------------------------------------------------------
constexpr int kPullUnroll = 8;

__global__ void __launch_bounds__(256) slab_pull_kernel(SlabPullArgs p) {
  long long pt = blockIdx.y + p.pt_shift;
  if (pt >= p.pt_lo[p.ranks]) pt -= p.pt_lo[p.ranks];
  int r = 0;
  while (r + 1 < p.ranks && pt >= p.pt_lo[r + 1]) ++r;
  const double2* __restrict__ src = p.src[r] + ((pt - p.pt_lo[r]) * p.na + p.atom0) * p.no2;
  double2* __restrict__ dst = p.dst + pt * p.dst_sp;
  const unsigned run = (unsigned)(p.natoms * p.no2), no2 = (unsigned)p.no2;
  const unsigned base = blockIdx.x * (blockDim.x * kPullUnroll) + threadIdx.x;
  double2 v[kPullUnroll];
#pragma unroll
  for (int u = 0; u < kPullUnroll; ++u) {
    const unsigned e = base + u * blockDim.x;
    if (e < run) v[u] = __ldcs(src + e);
  }
#pragma unroll
  for (int u = 0; u < kPullUnroll; ++u) {
    const unsigned e = base + u * blockDim.x;
    if (e < run) {
      const unsigned a = e / no2;
      dst[a * p.dst_sa + (e - a * no2)] = v[u];
    }
  }
}

// --------------------------------------------------------------------------
// K2: operator build.  One CTA per (atom, neighbour slot) of the chunk:
//   stage dH[a,s,0..2] and P_ij = dH_i @ dH_j (9 blocks) in shared memory,
//   then every thread produces output doubles of
//   M[q,w] = wt_w * sum_ij Dc[q,w,a,s,i,j] * P_ij
// for both polarities, either in DMMA B-fragment order or compact [p][n].
// --------------------------------------------------------------------------
constexpr int kOpBlocks = 8;  // (q,w) operator blocks per K2 iteration (fragment order)

__global__ void build_operator_kernel(OperatorArgs p) {
  extern __shared__ double2 smem[];
  const int no = p.no, no2 = no * no;
  double2* s_dh = smem;              // [3][no][no]
  double2* s_p = smem + 3 * no2;     // [9][no][no]
  const int la = blockIdx.x / p.nb;  // chunk-local atom
  const int s = blockIdx.x % p.nb;
  const int a_slab = p.atom_begin + la;

  const double2* dh = p.dH + ((long long)a_slab * p.nb + s) * 3 * no2;
  for (int x = threadIdx.x; x < 3 * no2; x += blockDim.x) s_dh[x] = dh[x];
  __syncthreads();
  for (int x = threadIdx.x; x < 9 * no2; x += blockDim.x) {
    const int ij = x / no2, pn = x % no2;
    const int i = ij / 3, j = ij % 3, pr = pn / no, n = pn % no;
    double re = 0.0, im = 0.0;
    for (int t = 0; t < no; ++t) {
      const double2 u = s_dh[i * no2 + pr * no + t];
      const double2 v = s_dh[j * no2 + t * no + n];
      re = fma(u.x, v.x, re);
      re = fma(-u.y, v.y, re);
      im = fma(u.x, v.y, im);
      im = fma(u.y, v.x, im);
    }
    s_p[x] = make_double2(re, im);
  }
  __syncthreads();

  const long long qw_total = (long long)p.nqz * p.nw;
  if (!p.fragment_order) {
    const long long out_base = (long long)blockIdx.x * qw_total * no2;  // (la*nb+s)
    for (int pol = 0; pol < p.npol; ++pol) {
      const double2* dc_base = p.Dc[pol];
      double2* out = p.M[pol] + out_base;
      for (long long x = threadIdx.x; x < qw_total * no2; x += blockDim.x) {
        const int qw = (int)(x / no2), v = (int)(x % no2);
        const double2* dc = dc_base + (((long long)qw * p.dc_natoms + a_slab) * p.nb + s) * 9;
        const double wt = p.wt[qw % p.nw];
        double re = 0.0, im = 0.0;
        for (int ij = 0; ij < 9; ++ij) {
          const double2 c = dc[ij], m = s_p[ij * no2 + v];
          re = fma(c.x, m.x, re);
          re = fma(-c.y, m.y, re);
          im = fma(c.x, m.y, im);
          im = fma(c.y, m.x, im);
        }
        out[x] = make_double2(wt * re, wt * im);
      }
    }
    return;
  }
  if (p.comb_kg > 0) {
    // combined multi-momentum fragments: per frequency w, M_q of every q (< kOpBlocks at a
    // time... all Nqz fit: Nqz <= kOpBlocks is checked by the launcher) into shared memory, then
    // for every source momentum kp and momentum group g one vector whose N' columns are
    // [M_{q_k0} | M_{q_k0+1} | ...] with q_k = (k - kp) mod Nkz (zero if invalid)
    double2* s_m = s_p + 9 * no2;  // [Nqz][no][no]
    const FragGeom fg = frag_geom(no);
    const CombGeom cg = comb_geom(no, p.comb_kg);
    const int groups = (p.nkz + p.comb_kg - 1) / p.comb_kg;
    const int per_vec = cg.fvc * 32;
    for (int pol = 0; pol < p.npol; ++pol) {
      const double2* dc_base = p.Dc[pol];
      for (int w = 0; w < p.nw; ++w) {
        const double wt = p.wt[w];
        for (int x = threadIdx.x; x < p.nqz * no2; x += blockDim.x) {
          const int q = x / no2, v = x - q * no2;
          const double2* dc = dc_base + ((((long long)q * p.nw + w) * p.dc_natoms + a_slab) * p.nb + s) * 9;
          double re = 0.0, im = 0.0;
          for (int ij = 0; ij < 9; ++ij) {
            const double2 c = dc[ij], m = s_p[ij * no2 + v];
            re = fma(c.x, m.x, re);
            re = fma(-c.y, m.y, re);
            im = fma(c.x, m.y, im);
            im = fma(c.y, m.x, im);
          }
          s_m[x] = make_double2(wt * re, wt * im);
        }
        __syncthreads();
        const int nvec = p.nkz * groups;
        for (int x = threadIdx.x; x < nvec * per_vec; x += blockDim.x) {
          const int vec = x / per_vec, v = x - vec * per_vec;
          const int kp = vec / groups, g = vec - kp * groups;
          const int j = v >> 5, lane = v & 31;
          double vals[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int f = 2 * j + h;
            double val = 0.0;
            if (f < cg.frc) {
              const int kk = f / cg.ntc, nt = f % cg.ntc;
              const int kr = 4 * kk + (lane & 3), c = 8 * nt + (lane >> 2);
              const int cc = c >> 1, part = c & 1, kl = cc / no, n = cc - kl * no;
              const int k = g * p.comb_kg + kl;
              int q = k - kp;
              if (q < 0) q += p.nkz;
              const bool im_row = fg.il ? (kr & 1) : kr >= fg.nop;
              const int pr = fg.il ? kr >> 1 : (im_row ? kr - fg.nop : kr);
              if (kl < p.comb_kg && k < p.nkz && q < p.nqz && pr < no) {
                const double2 m = s_m[q * no2 + pr * no + n];
                val = !im_row ? (part == 0 ? m.x : m.y) : (part == 0 ? -m.y : m.x);
              }
            }
            vals[h] = val;
          }
          // [atom, s, kp, g, w] vectors
          const long long vidx = ((((long long)blockIdx.x) * p.nkz + kp) * groups + g) * p.nw + w;
          p.M[pol][vidx * per_vec + v] = make_double2(vals[0], vals[1]);
        }
        __syncthreads();
      }
    }
    return;
  }
  // DMMA fragment order, kOpBlocks (q,w) blocks at a time: phase 1 computes each complex
  // M element once into shared memory (wt-scaled), phase 2 writes the real embedding
  //   B'[re-row p][2n] = Re M, B'[re-row p][2n+1] = Im M,
  //   B'[im-row p][2n] = -Im M, B'[im-row p][2n+1] = Re M
  // in fragment order (v = j * 32 + lane, vector j holds fragments 2j, 2j+1, fragment
  // f = kk * NT + nt; lane holds B'[4kk + (lane&3)][8nt + (lane>>2)]) with coalesced stores.
  double2* s_m = s_p + 9 * no2;  // [kOpBlocks][no][no]
  const FragGeom fg = frag_geom(no);
  const int per_qw_vec = fg.fv * 32;  // double2 per (q,w)
  const long long out_base = (long long)blockIdx.x * qw_total * per_qw_vec;  // (la*nb+s)
  for (int pol = 0; pol < p.npol; ++pol) {
    const double2* dc_base = p.Dc[pol];
    double2* out = p.M[pol] + out_base;
    for (int qw0 = 0; qw0 < qw_total; qw0 += kOpBlocks) {
      const int nblk = min(kOpBlocks, (int)qw_total - qw0);
      for (int x = threadIdx.x; x < nblk * no2; x += blockDim.x) {
        const int b = x / no2, v = x - b * no2, qw = qw0 + b;
        const double2* dc = dc_base + (((long long)qw * p.dc_natoms + a_slab) * p.nb + s) * 9;
        const double wt = p.wt[qw % p.nw];
        double re = 0.0, im = 0.0;
        for (int ij = 0; ij < 9; ++ij) {
          const double2 c = dc[ij], m = s_p[ij * no2 + v];
          re = fma(c.x, m.x, re);
          re = fma(-c.y, m.y, re);
          im = fma(c.x, m.y, im);
          im = fma(c.y, m.x, im);
        }
        re *= wt;
        im *= wt;
        s_m[x] = make_double2(re, im);
      }
      __syncthreads();
      double2* o = out + (long long)qw0 * per_qw_vec;
      for (int x = threadIdx.x; x < nblk * per_qw_vec; x += blockDim.x) {
        const int b = x / per_qw_vec, v = x - b * per_qw_vec;
        const int j = v >> 5, lane = v & 31;
        double vals[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f = 2 * j + h;
          const int kk = f / fg.nt, nt = f % fg.nt;
          const int kr = 4 * kk + (lane & 3), nc = 8 * nt + (lane >> 2);
          // split K: rows [0, nop) real, [nop, 2 nop) imaginary; il: row 2p real, 2p + 1 imaginary
          const bool im_row = fg.il ? (kr & 1) : kr >= fg.nop;
          const int pr = fg.il ? kr >> 1 : (im_row ? kr - fg.nop : kr);
          const int n = nc >> 1, part = nc & 1;
          double val = 0.0;
          if (pr < no && n < no) {
            const double2 m = s_m[b * no2 + pr * no + n];
            val = !im_row ? (part == 0 ? m.x : m.y) : (part == 0 ? -m.y : m.x);
          }
          vals[h] = val;
        }
        o[x] = make_double2(vals[0], vals[1]);
      }
      __syncthreads();
    }
  }
}

// --------------------------------------------------------------------------
// K3: fused Sigma on FP64 tensor cores.
// Grid: x = (row chunk, k, chunk atom), y = polarity.  Each warp owns
// kRowTiles 8-row tiles of the [NE*No, No] output matrix of (atom, k) and
// accumulates, in registers, over (q, s, w) in that fixed order the real-
// embedded products  C' += A'(G rows shifted by off_w) * B'(M[q,w,a,s]).
// Per (q,s,w) and tile: KH 16-byte A loads, FV 16-byte B loads shared by the
// warp's tiles, KSTEPS*NT DMMAs.  Nothing but Sigma is written to HBM.
// --------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// The i-th momentum transfer q (i < Nqz) of output momentum k in the accumulation order all
// Sigma kernels share: source momenta kp = (k - q) mod Nkz ascending (the multi-momentum K3
// walks kp and serves every k of its group from the same G rows).  kp = k - q for the first
// L = min(k + 1, Nqz) terms (q = L-1 .. 0), then kp = k - q + Nkz (q = Nqz-1 .. k+1).
__host__ __device__ __forceinline__ void q_order(int k, int i, int nkz, int nqz, int& q, int& kp) {
  const int L = k + 1 < nqz ? k + 1 : nqz;
  if (i < L) {
    q = L - 1 - i;
    kp = k - q;
  } else {
    q = k + nqz - i;
    kp = k - q + nkz;
  }
}

// Base of the Sigma block (k, E) of chunk atom la: the slab (s_* strides), or
// the point-layout buffer of the owner rank of point k*NE + E (peer scatter).
__device__ __forceinline__ double2* sigma_block(const SigmaArgs& p, int pol, int la, int k, int e) {
  if (p.scatter_ranks == 0)
    return p.S[pol] + (long long)(p.s_atom_begin + la) * p.s_sa + (long long)k * p.s_sk + (long long)e * p.s_se;
  const long long pt = (long long)k * p.ne + e;
  int r = 0;
  while (r + 1 < p.scatter_ranks && pt >= p.pt_lo[r + 1]) ++r;
  return p.S_rank[pol][r] + ((pt - p.pt_lo[r]) * p.scatter_na + p.scatter_atom0 + la) * (long long)(p.no * p.no);
}

// G block (k, E, atom) of a point-layout owner (PeerGather, Pi kernels)
__device__ __forceinline__ const double2* peer_block(const PeerGather& pg, int pol, long long pt, long long atom,
                                                     int no2) {
  int r = 0;
  while (r + 1 < pg.ranks && pt >= pg.pt_lo[r + 1]) ++r;
  return pg.G[pol][r] + ((pt - pg.pt_lo[r]) * pg.na + atom) * no2;
}

// same without `volatile`: lets the scheduler interleave the shared-memory
// operand loads with the DMMAs (the per-accumulator order is data-dependent)
__device__ __forceinline__ void dmma884_nv(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// x with its sign bit xor-ed with `mask` (0 or 0x80000000) on the integer pipe
// (an FP64 negation would issue on the FP64 pipe the DMMAs use)
__device__ __forceinline__ double xor_sign(double x, unsigned mask) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  asm volatile("xor.b32 %0, %0, %1;" : "+r"(hi) : "r"(mask));
  double r;
  asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
  return r;
}

// Column swizzle of the V rows (kappa = n*No + p): mode 2 flips column bit 1 with kappa bit 1
// (K6 v3 reads rows kappa..kappa+3 conflict-free); mode 3 also XORs (n & 3), so K5's scatter
// (whose lanes differ in n) spreads over the banks while K6 v4's quads (one n each) stay conflict-free
__device__ __forceinline__ int vt_swz(int kap, int no, int swz) {
  if (swz == 0) return 0;
  int x = ((kap >> 1) & 1) ? 2 : 0;
  if (swz == 3) x ^= (kap / no) & 3;
  return x;
}

// A operands of one 8-row tile for a stage: `row` = start of the lane's G row (complex), pcol =
// lane & 3.  Split K: av[kk] = G[row][pcol + 4 kk] (Re -> k-step kk, Im -> k-step kk + kh);
// il: av[j] = (double pcol + 8j, double pcol + 8j + 4) of the row's (re, im) sequence = the A
// values of k-steps 2j and 2j + 1.  Rows that contribute nothing pass ok = false (zeros).
template <int NO>
__device__ __forceinline__ void load_a(double2 (&av)[frag_geom(NO).kh], const double2* row, int pcol, bool ok) {
  constexpr FragGeom FG = frag_geom(NO);
  if constexpr (FG.il) {
    const double* rd = reinterpret_cast<const double*>(row) + pcol;
#pragma unroll
    for (int j = 0; j < FG.kh; ++j) {
      av[j].x = ok ? rd[8 * j] : 0.0;
      av[j].y = (ok && 2 * j + 1 < FG.ksteps) ? rd[8 * j + 4] : 0.0;
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < FG.kh; ++kk) {
      if (NO % 4 == 0) {
        av[kk] = ok ? row[pcol + 4 * kk] : make_double2(0.0, 0.0);
      } else {
        av[kk] = make_double2(0.0, 0.0);
        if (ok && pcol + 4 * kk < NO) av[kk] = row[pcol + 4 * kk];
      }
    }
  }
}
// the lane's A value of k-step kk from load_a's registers
template <int NO>
__device__ __forceinline__ double a_sel(const double2 (&av)[frag_geom(NO).kh], int kk) {
  constexpr FragGeom FG = frag_geom(NO);
  if constexpr (FG.il) return (kk & 1) ? av[kk >> 1].y : av[kk >> 1].x;
  return kk < FG.kh ? av[kk].x : av[kk - FG.kh].y;
}

template <int NO>
__global__ void __launch_bounds__(kSigmaWarps * 32)
sigma_dmma_kernel(SigmaArgs p) {
  constexpr FragGeom FG = frag_geom(NO);
  constexpr int KSTEPS = FG.ksteps, NT = FG.nt, FV = FG.fv;
  const int pol = blockIdx.y;
  int bx = blockIdx.x;
  const int rc = bx % p.ctas_per_ak;
  bx /= p.ctas_per_ak;
  const int k = bx % p.nkz;
  const int la = bx / p.nkz;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rbase = rc * kRowsPerCta + warp * (kRowTiles * 8);
  const int pcol = lane & 3;

  const double2* __restrict__ G = p.G[pol];
  const double2* __restrict__ Mf = p.M[pol];

  int e_row[kRowTiles], m_row[kRowTiles];
  bool v_row[kRowTiles];
#pragma unroll
  for (int t = 0; t < kRowTiles; ++t) {
    const int row = rbase + t * 8 + (lane >> 2);
    v_row[t] = row < p.rows;
    e_row[t] = row / NO;
    m_row[t] = row - e_row[t] * NO;
  }

  double acc[kRowTiles][NT][2];
#pragma unroll
  for (int t = 0; t < kRowTiles; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;

  for (int qi = 0; qi < p.nqz; ++qi) {
    int q, kp;
    q_order(k, qi, p.nkz, p.nqz, q, kp);
    for (int s = 0; s < p.nb; ++s) {
      const int lb = __ldg(p.nbr + la * p.nb + s);
      long long rowoff[kRowTiles];
#pragma unroll
      for (int t = 0; t < kRowTiles; ++t)
        rowoff[t] = lb * p.g_sa + kp * p.g_sk + (long long)e_row[t] * p.g_se + m_row[t] * NO;
      const double2* mf = Mf + ((long long)((la * p.nb + s) * p.nqz + q) * p.nw) * (FV * 32) + lane;
      for (int w = 0; w < p.nw; ++w) {
        const int off = __ldg(p.off + w);
        double2 bv[FV];
#pragma unroll
        for (int j = 0; j < FV; ++j) bv[j] = __ldg(mf + (w * FV + j) * 32);
#pragma unroll
        for (int t = 0; t < kRowTiles; ++t) {
          const int tile_row0 = rbase + t * 8;
          // warp-uniform skip: tile past the end, or every row has E < off
          if (tile_row0 >= p.rows || (tile_row0 + 7) / NO < off) continue;
          const bool ok = v_row[t] && e_row[t] >= off;
          double2 av[FG.kh];
          load_a<NO>(av, G + rowoff[t] - (long long)off * p.g_se, pcol, ok);
#pragma unroll
          for (int kk = 0; kk < KSTEPS; ++kk) {
            const double a = a_sel<NO>(av, kk);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int f = kk * NT + nt;
              const double b = (f & 1) ? bv[f >> 1].y : bv[f >> 1].x;
              dmma884(acc[t][nt], a, b);
            }
          }
        }
      }
    }
  }

  // epilogue: lane holds (Re, Im) of C[row][n = 4 nt + (lane & 3)]; Sigma = i C
#pragma unroll
  for (int t = 0; t < kRowTiles; ++t) {
    if (!v_row[t]) continue;
    double2* dst = sigma_block(p, pol, la, k, e_row[t]) + m_row[t] * NO;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int n = 4 * nt + (lane & 3);
      if (n < NO) dst[n] = make_double2(-acc[t][nt][1], acc[t][nt][0]);
    }
  }
}

// --------------------------------------------------------------------------
// K3 (pipelined): same contraction and accumulation order as sigma_dmma_kernel,
// restructured for latency hiding with one 8-warp CTA per SM:
//  * the (q, s, w) loop is flattened and register double-buffered: the A
//    (shifted G rows, 3 tiles) and B (M fragments) operands of iteration
//    it+1 are loaded while the 54 DMMAs of iteration it run;
//  * DMMAs are issued k-step-outer over the warp's 3 tiles x 3 n-tiles, so 9
//    independent accumulator chains separate dependent DMMAs;
//  * the E < off skip is warp-uniform (no branches between the tiles).
// --------------------------------------------------------------------------
template <int NO, int MT>
struct OperandStageT {
  double2 a[MT][frag_geom(NO).kh];
  double2 b[frag_geom(NO).fv];
  int off;
};
template <int NO>
using OperandStage = OperandStageT<NO, kRowTiles>;

template <int NO>
__global__ void __launch_bounds__(kSigmaWarps * 32, 1)
sigma_dmma_pipe_kernel(SigmaArgs p) {
  constexpr FragGeom FG = frag_geom(NO);
  constexpr int KSTEPS = FG.ksteps, NT = FG.nt, FV = FG.fv;
  const int pol = blockIdx.y;
  int bx = blockIdx.x;
  const int rc = bx % p.ctas_per_ak;
  bx /= p.ctas_per_ak;
  const int k = bx % p.nkz;
  const int la = bx / p.nkz;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rbase = rc * kRowsPerCta + warp * (kRowTiles * 8);
  const int pcol = lane & 3;
  const double2* __restrict__ G = p.G[pol];
  const double2* __restrict__ Mf = p.M[pol];
  const int* __restrict__ offs = p.off;

  int e_row[kRowTiles];
  bool v_row[kRowTiles];
  long long r_off[kRowTiles];  // row offset within a (k', b) slab: E * g_se + m * NO + pcol
#pragma unroll
  for (int t = 0; t < kRowTiles; ++t) {
    const int row = rbase + t * 8 + (lane >> 2);
    v_row[t] = row < p.rows;
    e_row[t] = row / NO;
    r_off[t] = (long long)e_row[t] * p.g_se + (row - e_row[t] * NO) * NO;
  }
  // warp-uniform bounds of the warp's rows
  const int warp_rows = min(kRowTiles * 8, p.rows - rbase);
  const int warp_emax = warp_rows > 0 ? (rbase + warp_rows - 1) / NO : -1;

  double acc[kRowTiles][NT][2];
#pragma unroll
  for (int t = 0; t < kRowTiles; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;

  // load cursor over the flattened (q, s, w) iterations
  int lq = 0, ls = 0, lw = 0;
  long long slab = 0;           // (k', b) slab offset of the cursor's (q, s)
  const double2* mfq = nullptr;  // M fragments of the cursor's (q, s), lane-offset
  auto setup_qs = [&]() {  // lq indexes the shared q order (q_order)
    int q, kp;
    q_order(k, lq, p.nkz, p.nqz, q, kp);
    const int lb = __ldg(p.nbr + la * p.nb + ls);
    slab = lb * p.g_sa + kp * p.g_sk;
    mfq = Mf + ((long long)((la * p.nb + ls) * p.nqz + q) * p.nw) * (FV * 32) + lane;
  };
  auto load = [&](OperandStage<NO>& st) {
    const int off = __ldg(offs + lw);
    st.off = off;
#pragma unroll
    for (int j = 0; j < FV; ++j) st.b[j] = __ldg(mfq + (lw * FV + j) * 32);
    const long long shift = slab - (long long)off * p.g_se;
#pragma unroll
    for (int t = 0; t < kRowTiles; ++t) {
      const bool ok = v_row[t] && e_row[t] >= off;
      load_a<NO>(st.a[t], G + shift + r_off[t], pcol, ok);
    }
    if (++lw == p.nw) {
      lw = 0;
      if (++ls == p.nb) {
        ls = 0;
        ++lq;
      }
      if (lq < p.nqz) setup_qs();
    }
  };
  auto compute = [&](const OperandStage<NO>& st) {
    if (warp_emax < st.off) return;  // every row of the warp has E < off: no term
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
#pragma unroll
      for (int t = 0; t < kRowTiles; ++t) {
        const double a = a_sel<NO>(st.a[t], kk);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int f = kk * NT + nt;
          const double b = (f & 1) ? st.b[f >> 1].y : st.b[f >> 1].x;
          dmma884(acc[t][nt], a, b);
        }
      }
    }
  };

  const int n_it = p.nqz * p.nb * p.nw;
  OperandStage<NO> s0, s1;
  setup_qs();
  load(s0);
  for (int it = 0; it < n_it; it += 2) {
    if (it + 1 < n_it) load(s1);
    compute(s0);
    if (it + 1 >= n_it) break;
    if (it + 2 < n_it) load(s0);
    compute(s1);
  }

  // epilogue: lane holds (Re, Im) of C[row][n = 4 nt + (lane & 3)]; Sigma = i C
#pragma unroll
  for (int t = 0; t < kRowTiles; ++t) {
    if (!v_row[t]) continue;
    const int row = rbase + t * 8 + (lane >> 2);
    double2* dst = sigma_block(p, pol, la, k, e_row[t]) + (row - e_row[t] * NO) * NO;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int n = 4 * nt + (lane & 3);
      if (n < NO) dst[n] = make_double2(-acc[t][nt][1], acc[t][nt][0]);
    }
  }
}

// --------------------------------------------------------------------------
// K3 (TMA, sliding window) — production kernel: the DMMA contraction fed
// from shared memory by bulk-async copies (cp.async.bulk -> SASS UBLKCP)
// with full/empty mbarriers per stage; 12 warps x 3 row tiles (288 rows), one
// CTA per SM, 160 registers (3 warps per SMSP keep the DMMA pipe fed).
//  * M fragments: one FV*512-byte copy per (q, s, w) stage into a ring of
//    kSlideStages slots, shared by all warps;
//  * G rows: within a (q, s) segment the CTA's window of source energies
//    [E_lo - off_w, E_hi - off_w] slides down by one block per stage (offsets
//    non-decreasing with steps <= 1, as default_grid's are), so only the
//    entering energy block is copied; blocks live in a FIFO ring of R slots;
//  * stage t is produced by lane 0 of warp t % NW, kSlideLookahead stages
//    ahead (round-robin spreads the producer work over the warps);
//  * consumers wait on the stage's full barrier, read fragments with LDS,
//    run the DMMAs and arrive on the stage's empty barrier.
// Accumulation order is identical to the other K3 kernels (bitwise equal).
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk async copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kSlideStages = 12;
constexpr int kSlideLookahead = 6;
constexpr int kMaxSlideNw = 1024;

template <int NO, int NW, int MT>
struct SlideGeom {
  static constexpr int kRows = NW * MT * 8;              // output rows per CTA
  static constexpr int kTE = (kRows + NO - 1) / NO + 1;         // max energy blocks per window
  static constexpr int kNeed = 2 * kTE + kSlideStages;          // live FIFO span bound
  static constexpr int kBVec = frag_geom(NO).fv * 32;            // double2 per M stage
  static constexpr size_t smem_for(int ring) {
    return (size_t)kSlideStages * kBVec * 16 + (size_t)ring * NO * NO * 16 + 2 * kSlideStages * 8 +
           kMaxSlideNw * 4 + (size_t)NO * NO * 16;
  }
  static constexpr int kPow2 = kNeed <= 32 ? 32 : (kNeed <= 64 ? 64 : 128);
  // a power-of-two FIFO (index by mask) when it fits, else exactly the live-span bound (No = 10)
  static constexpr int kRing = smem_for(kPow2) <= 225 * 1024 ? kPow2 : kNeed;
  static constexpr size_t kSmem = smem_for(kRing);
  static constexpr bool kFits = kSmem <= 225 * 1024;
};

template <int NO, int NW, int MT>
__global__ void __launch_bounds__(NW * 32, 1)
sigma_dmma_slide_kernel(SigmaArgs p) {
  constexpr FragGeom FG = frag_geom(NO);
  constexpr int KSTEPS = FG.ksteps, NT = FG.nt, FV = FG.fv;
  using SG = SlideGeom<NO, NW, MT>;
  constexpr int R = SG::kRing, SB = kSlideStages, BVEC = SG::kBVec, BLK = NO * NO;
  // FIFO slot of a (non-negative) block index
  auto fifo = [](int x) { return (R & (R - 1)) == 0 ? (x & (R - 1)) : (int)((unsigned)x % (unsigned)R); };
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* ring_b = reinterpret_cast<double2*>(smem_raw);
  double2* ring_a = ring_b + SB * BVEC;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring_a + R * BLK);
  uint64_t* empty = full + SB;

  const int pol = blockIdx.y;
  int bx = blockIdx.x;
  const int rc = bx % p.ctas_per_ak;
  bx /= p.ctas_per_ak;
  const int k = bx % p.nkz;
  const int la = bx / p.nkz;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cta_r0 = rc * SG::kRows;
  // The last CTA of an (atom, k) row range is usually partial (paper: 120 of 288
  // rows).  There the row tiles are interleaved over the warps (tile t of warp w
  // = CTA tile t * NW + w), so the valid tiles spread over all four SMSPs, and
  // each warp runs the DMMAs of its valid tiles only (a prefix of its MT).
  // Each output row keeps its accumulation order: bitwise equal either way.
  const bool tail = (p.k3_opts & 1) && cta_r0 + SG::kRows > p.rows;
  auto tile_row0 = [&](int t) { return tail ? cta_r0 + (t * NW + warp) * 8 : cta_r0 + warp * (MT * 8) + t * 8; };
  const int pcol = lane & 3;
  const double2* __restrict__ G = p.G[pol];
  const double2* __restrict__ Mf = p.M[pol];
  const int* __restrict__ offs = p.off;
  // stage t is produced by lane 0 of warp t % NW (round-robin), kSlideLookahead
  // stages ahead of the consumers; every warp steps the producer state machine.

  // CTA energy range (rows [cta_r0, cta_r0 + kRowsPerCta) clipped to the matrix)
  const int e_lo = cta_r0 / NO;
  const int e_hi = (min(cta_r0 + SG::kRows, p.rows) - 1) / NO;

  int e_row[MT], m_off[MT];
  bool v_row[MT];
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int row = tile_row0(t) + (lane >> 2);
    v_row[t] = row < p.rows;
    e_row[t] = row / NO;
    m_off[t] = (row - e_row[t] * NO) * NO;
  }
  // valid tiles (first row inside the matrix) form a prefix in both mappings;
  // warp_emax = energy of the warp's last valid row (rows ascend with t)
  int n_valid = 0;
#pragma unroll
  for (int t = 0; t < MT; ++t) n_valid += tile_row0(t) < p.rows ? 1 : 0;
  const int warp_emax = n_valid > 0 ? (min(tile_row0(n_valid - 1) + 8, p.rows) - 1) / NO : -1;

  double acc[MT][NT][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;

  int* s_off = reinterpret_cast<int*>(empty + SB);  // frequency offsets (p.nw <= kMaxSlideNw)
  for (int w = threadIdx.x; w < p.nw; w += blockDim.x) s_off[w] = offs[w];
  // a zero block: rows outside the matrix or with E - off < 0 read it (no per-element predicates)
  double2* zero_blk = reinterpret_cast<double2*>(s_off + kMaxSlideNw);
  for (int x = threadIdx.x; x < BLK; x += blockDim.x) zero_blk[x] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < SB; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Stages whose offset exceeds the CTA's top energy (E - off < 0 for every row:
  // a suffix of each segment, offsets being non-decreasing) contribute nothing;
  // they are dropped, keeping >= kSlideStages stages per segment so that the
  // stages in flight still span at most one segment boundary (ring bound).
  int nw_eff = p.nw;
  if (p.k3_opts & 2)
    while (nw_eff > SB && s_off[nw_eff - 1] > e_hi) --nw_eff;
  const int n_it = p.nqz * p.nb * nw_eff;

  // Window bookkeeping in closed form.  Segment sg = (q, s) covers stages
  // [sg*nw, (sg+1)*nw); its window at stage w is [max(0, e_lo - off_w),
  // e_hi - off_w].  With non-decreasing offsets (steps <= 1) the window bottom
  // L(w) = max(0, e_lo - off_w) never rises, so stage w loads exactly the
  // blocks [L(w), L(w-1) - 1] (L(-1) = top0 + 1, top0 = e_hi - off_0) and a
  // segment loads seg_blocks blocks.  Energy e of segment sg sits at FIFO
  // index sg * seg_blocks + (top0 - e).
  const int top0 = e_hi - s_off[0];
  const bool seg_empty = top0 < 0;
  const int seg_blocks = seg_empty ? 0 : top0 + 1 - max(0, e_lo - s_off[nw_eff - 1]);
  auto win_low = [&](int w) { return w < 0 ? top0 + 1 : max(0, e_lo - s_off[w]); };

  auto produce = [&](int t) {  // lane 0 of the owning warp
    const int slot = t % SB;
    const int sg = t / nw_eff, w = t - sg * nw_eff;
    const int qi = sg / p.nb, s = sg - qi * p.nb;
    int q, kp;
    q_order(k, qi, p.nkz, p.nqz, q, kp);
    const long long nb_atom = __ldg(p.nbr + la * p.nb + s);
    const long long slab = nb_atom * p.g_sa + kp * p.g_sk;
    const double2* mf = Mf + ((long long)((la * p.nb + s) * p.nqz + q) * p.nw + w) * BVEC;
    const int hi = seg_empty ? 0 : win_low(w - 1), lo = seg_empty ? 0 : win_low(w);
    if (t >= SB) mbar_wait(empty + slot, (uint32_t)(((t - SB) / SB) & 1));
    mbar_arrive_expect_tx(full + slot, (uint32_t)(BVEC + (hi - lo) * BLK) * 16);
    bulk_g2s(ring_b + slot * BVEC, mf, BVEC * 16, full + slot);
    if (p.gather_ranks == 0) {
      for (int e = hi - 1; e >= lo; --e) {
        const int f = fifo(sg * seg_blocks + top0 - e);
        bulk_g2s(ring_a + f * BLK, G + slab + (long long)e * p.g_se, BLK * 16, full + slot);
      }
    } else {  // G in the GF point layout of the owner ranks, read over NVLink (nbr = global atom ids)
      int r = p.gather_ranks - 1;
      for (int e = hi - 1; e >= lo; --e) {
        const long long pt = (long long)kp * p.ne + e;
        while (r > 0 && pt < p.pt_lo[r]) --r;  // e descends: the owner rank only moves down
        const double2* src = p.G_rank[pol][r] + ((pt - p.pt_lo[r]) * p.scatter_na + nb_atom) * BLK;
        const int f = fifo(sg * seg_blocks + top0 - e);
        bulk_g2s(ring_a + f * BLK, src, BLK * 16, full + slot);
      }
    }
  };

  // consumer cursor
  int c_it = 0, c_sg = 0, c_w = 0;
  auto lds = [&](OperandStageT<NO, MT>& st) {
    const int t = c_it;
    const int slot = t % SB;
    const int off = s_off[c_w];
    st.off = off;
    const int fbase = c_sg * seg_blocks + top0 + off;  // FIFO index of row energy E: fbase - E
    mbar_wait(full + slot, (uint32_t)((t / SB) & 1));
    if (warp_emax >= off) {
      const double2* sb = ring_b + slot * BVEC;
#pragma unroll
      for (int j = 0; j < FV; ++j) st.b[j] = sb[j * 32 + lane];
#pragma unroll
      for (int tt = 0; tt < MT; ++tt) {
        const bool ok = v_row[tt] && e_row[tt] >= off;
        const double2* src = ok ? ring_a + fifo(fbase - e_row[tt]) * BLK + m_off[tt] : zero_blk;
        // full rows (No % 4 == 0, il) read the zero block instead of predicating each element
        load_a<NO>(st.a[tt], src, pcol, (NO % 4 == 0 || FG.il) ? true : ok);
      }
    }
    ++c_it;
    if (++c_w == nw_eff) {
      c_w = 0;
      ++c_sg;
    }
  };
  // k-steps [k0, k1) of one stage's DMMAs
  auto compute_tiles = [&](const OperandStageT<NO, MT>& st, auto nv) {
    constexpr int NV = decltype(nv)::value;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
#pragma unroll
      for (int t = 0; t < NV; ++t) {
        const double a = a_sel<NO>(st.a[t], kk);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int f = kk * NT + nt;
          const double b = (f & 1) ? st.b[f >> 1].y : st.b[f >> 1].x;
          dmma884_nv(acc[t][nt], a, b);
        }
      }
    }
  };
  auto release = [&](int t) {  // the warp is done with stage t's shared memory
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + (t % SB));
  };

  const int L = p.lookahead > 0 ? min(p.lookahead, SB - 1) : kSlideLookahead;
  if (lane == 0)
    for (int i = warp; i < L && i < n_it; i += NW) produce(i);
  // the stage loop, instantiated per count of valid tiles (warp-uniform; the
  // branch is outside the loop, so the full-tile loop is the only hot code)
  auto run = [&](auto nv) {
    // single buffer: the LDS latency is hidden by the other warps of the SMSP
    OperandStageT<NO, MT> s0;
    for (int it = 0; it < n_it; ++it) {
      if (lane == 0 && it + L < n_it && (it + L) % NW == warp) produce(it + L);
      lds(s0);
      if (warp_emax >= s0.off) compute_tiles(s0, nv);
      release(it);
    }
  };
  if (n_valid == MT) run(std::integral_constant<int, MT>{});
  else if (MT > 2 && n_valid == 2) run(std::integral_constant<int, (MT > 2 ? 2 : 0)>{});
  else if (MT > 1 && n_valid == 1) run(std::integral_constant<int, (MT > 1 ? 1 : 0)>{});
  else run(std::integral_constant<int, 0>{});

#pragma unroll
  for (int t = 0; t < MT; ++t) {
    if (!v_row[t]) continue;
    double2* dst = sigma_block(p, pol, la, k, e_row[t]) + m_off[t];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int n = 4 * nt + (lane & 3);
      if (n < NO) dst[n] = make_double2(-acc[t][nt][1], acc[t][nt][0]);
    }
  }
}

// --------------------------------------------------------------------------
// K3m (multi-momentum sliding window) — production kernel.  As the sliding-
// window K3, but a CTA serves KG output momenta k at once: stage (kp, s, w)
// stages the G rows G[kp, E - off_w, f(a,s)] ONCE and the KG M-fragment vectors
// M[q_k = (k - kp) mod Nkz, w, a, s] side by side (a zero vector where q_k >=
// Nqz), and each warp runs its 3 row tiles x (KG x NT) n-tiles: 162 DMMAs per
// warp-stage at No = 12, KG = 3 (the single-momentum kernel: 54), so the
// per-stage barrier / operand-load overhead is amortised over 3x the tensor
// work, and the A fragments (G rows) are loaded once for KG momenta.  Stages
// walk kp ascending, so every output accumulates in the shared q_order
// (bitwise equal to the other K3 kernels).  B ring of kKStages stages (the
// stage is KG times larger), FIFO of G blocks as before.
// --------------------------------------------------------------------------
constexpr int kKStages = 6;
constexpr int kKLookahead = 3;

template <int NO, int NW, int MT, int KG, bool COMB = false>
struct KSlideGeom {
  static constexpr int kRows = NW * MT * 8;
  static constexpr int kTE = (kRows + NO - 1) / NO + 1;
  static constexpr int kNeed = 2 * kTE + kKStages;
  static constexpr int kBVec = frag_geom(NO).fv * 32;  // double2 per momentum and stage
  // COMB: one combined vector (comb_geom) per stage; else KG per-q vectors side by side
  static constexpr int kBStage = COMB ? comb_geom(NO, KG).fvc * 32 : KG * kBVec;
  static constexpr size_t smem_for(int ring) {
    return (size_t)kKStages * kBStage * 16 + (size_t)ring * NO * NO * 16 + 2 * kKStages * 8 + kMaxSlideNw * 4 +
           (size_t)NO * NO * 16;
  }
  static constexpr int kPow2 = kNeed <= 32 ? 32 : (kNeed <= 64 ? 64 : 128);
  static constexpr int kRing = smem_for(kPow2) <= 225 * 1024 ? kPow2 : kNeed;
  static constexpr size_t kSmem = smem_for(kRing);
  static constexpr bool kFits = kSmem <= 225 * 1024;
};

template <int NO, int NW, int MT, int KG, bool COMB = false>
__global__ void __launch_bounds__(NW * 32, 1)
sigma_dmma_kslide_kernel(SigmaArgs p) {
  constexpr FragGeom FG = frag_geom(NO);
  constexpr CombGeom CG = comb_geom(NO, KG);
  constexpr int KH = FG.kh, NT = FG.nt, FV = FG.fv, FR = FG.fr;
  constexpr int NTA = COMB ? CG.ntc : KG * NT;  // accumulator n-tiles per row tile
  using SG = KSlideGeom<NO, NW, MT, KG, COMB>;
  constexpr int R = SG::kRing, SB = kKStages, BVEC = SG::kBVec, BSTAGE = SG::kBStage, BLK = NO * NO;
  auto fifo = [](int x) { return (R & (R - 1)) == 0 ? (x & (R - 1)) : (int)((unsigned)x % (unsigned)R); };
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* ring_b = reinterpret_cast<double2*>(smem_raw);
  double2* ring_a = ring_b + SB * BSTAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring_a + R * BLK);
  uint64_t* empty = full + SB;

  const int pol = blockIdx.y;
  int bx = blockIdx.x;
  // k3_opts bit 2: the partial last row CTA of every (atom, momentum group) comes after all full
  // CTAs, so a launch's final wave is packed with short CTAs (outputs are disjoint per CTA: the
  // order changes no result); otherwise row CTAs fastest
  int rc;
  const int pairs = (int)(gridDim.x / p.ctas_per_ak);
  if ((p.k3_opts & 4) && p.ctas_per_ak > 1 && p.rows % SG::kRows != 0) {
    const int full = pairs * (p.ctas_per_ak - 1);
    if (bx < full) {
      rc = bx % (p.ctas_per_ak - 1);
      bx /= p.ctas_per_ak - 1;
    } else {
      rc = p.ctas_per_ak - 1;
      bx -= full;
    }
  } else {
    rc = bx % p.ctas_per_ak;
    bx /= p.ctas_per_ak;
  }
  const int kg = bx % p.kgroups;
  const int la = bx / p.kgroups;
  const int k0 = p.k_first + kg * KG;  // output momenta k0 .. k0 + KG - 1 (those < Nkz)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cta_r0 = rc * SG::kRows;
  const bool tail = (p.k3_opts & 1) && cta_r0 + SG::kRows > p.rows;
  auto tile_row0 = [&](int t) { return tail ? cta_r0 + (t * NW + warp) * 8 : cta_r0 + warp * (MT * 8) + t * 8; };
  const int pcol = lane & 3;
  const double2* __restrict__ G = p.G[pol];
  const double2* __restrict__ Mf = p.M[pol];
  const int* __restrict__ offs = p.off;
  const int e_lo = cta_r0 / NO;
  const int e_hi = (min(cta_r0 + SG::kRows, p.rows) - 1) / NO;

  int e_row[MT], m_off[MT];
  bool v_row[MT];
#pragma unroll
  for (int t = 0; t < MT; ++t) {
    const int row = tile_row0(t) + (lane >> 2);
    v_row[t] = row < p.rows;
    e_row[t] = row / NO;
    m_off[t] = (row - e_row[t] * NO) * NO;
  }
  int n_valid = 0;
#pragma unroll
  for (int t = 0; t < MT; ++t) n_valid += tile_row0(t) < p.rows ? 1 : 0;
  const int warp_emax = n_valid > 0 ? (min(tile_row0(n_valid - 1) + 8, p.rows) - 1) / NO : -1;

  double acc[MT][NTA][2];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int n = 0; n < NTA; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;

  int* s_off = reinterpret_cast<int*>(empty + SB);
  for (int w = threadIdx.x; w < p.nw; w += blockDim.x) s_off[w] = offs[w];
  double2* zero_blk = reinterpret_cast<double2*>(s_off + kMaxSlideNw);
  for (int x = threadIdx.x; x < BLK; x += blockDim.x) zero_blk[x] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < SB; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int nw_eff = p.nw;
  if (p.k3_opts & 2)
    while (nw_eff > SB && s_off[nw_eff - 1] > e_hi) --nw_eff;
  const int n_it = p.nkz * p.nb * nw_eff;  // segments (kp, s), kp ascending
  const int all_groups = (p.nkz + KG - 1) / KG;  // COMB: the vector index's group count

  const int top0 = e_hi - s_off[0];
  const bool seg_empty = top0 < 0;
  const int seg_blocks = seg_empty ? 0 : top0 + 1 - max(0, e_lo - s_off[nw_eff - 1]);
  auto win_low = [&](int w) { return w < 0 ? top0 + 1 : max(0, e_lo - s_off[w]); };

  auto produce = [&](int t) {  // lane 0 of the owning warp
    const int slot = t % SB;
    const int sg = t / nw_eff, w = t - sg * nw_eff;
    const int kp = sg / p.nb, s = sg - kp * p.nb;
    const long long nb_atom = __ldg(p.nbr + la * p.nb + s);
    const long long slab = nb_atom * p.g_sa + kp * p.g_sk;
    const int hi = seg_empty ? 0 : win_low(w - 1), lo = seg_empty ? 0 : win_low(w);
    if (t >= SB) mbar_wait(empty + slot, (uint32_t)(((t - SB) / SB) & 1));
    mbar_arrive_expect_tx(full + slot, (uint32_t)(BSTAGE + (hi - lo) * BLK) * 16);
    if constexpr (COMB) {
      const double2* mf = Mf + ((((long long)(la * p.nb + s) * p.nkz + kp) * all_groups + kg) * p.nw + w) * BSTAGE;
      bulk_g2s(ring_b + slot * BSTAGE, mf, BSTAGE * 16, full + slot);
    } else {
#pragma unroll
      for (int kl = 0; kl < KG; ++kl) {
        int q = k0 + kl - kp;
        if (q < 0) q += p.nkz;
        const bool ok = k0 + kl < p.nkz && q < p.nqz;
        const double2* mf = ok ? Mf + ((long long)((la * p.nb + s) * p.nqz + q) * p.nw + w) * BVEC : p.zeroM;
        bulk_g2s(ring_b + slot * BSTAGE + kl * BVEC, mf, BVEC * 16, full + slot);
      }
    }
    if (p.gather_ranks == 0) {
      for (int e = hi - 1; e >= lo; --e)
        bulk_g2s(ring_a + fifo(sg * seg_blocks + top0 - e) * BLK, G + slab + (long long)e * p.g_se, BLK * 16,
                 full + slot);
    } else {  // G in the GF point layout of the owner ranks, read over NVLink (nbr = global atom ids)
      int r = p.gather_ranks - 1;
      for (int e = hi - 1; e >= lo; --e) {
        const long long pt = (long long)kp * p.ne + e;
        while (r > 0 && pt < p.pt_lo[r]) --r;
        const double2* src = p.G_rank[pol][r] + ((pt - p.pt_lo[r]) * p.scatter_na + nb_atom) * BLK;
        bulk_g2s(ring_a + fifo(sg * seg_blocks + top0 - e) * BLK, src, BLK * 16, full + slot);
      }
    }
  };

  int c_it = 0, c_sg = 0, c_w = 0;
  double2 av[MT][KH];
  auto lds_a = [&](int off) {  // wait for the stage, then the A operands of the warp's tiles
    const int slot = c_it % SB;
    const int fbase = c_sg * seg_blocks + top0 + off;
    mbar_wait(full + slot, (uint32_t)((c_it / SB) & 1));
    if (warp_emax >= off) {
#pragma unroll
      for (int tt = 0; tt < MT; ++tt) {
        const bool ok = v_row[tt] && e_row[tt] >= off;
        const double2* src = ok ? ring_a + fifo(fbase - e_row[tt]) * BLK + m_off[tt] : zero_blk;
        load_a<NO>(av[tt], src, pcol, (NO % 4 == 0 || FG.il) ? true : ok);
      }
    }
  };
  // the stage's DMMAs: B fragment pair j of momentum kl feeds every tile; each accumulator
  // (tile, momentum, n-tile) still sees its k-steps in ascending order
  auto compute_tiles = [&](int slot, auto nv) {
    constexpr int NV = decltype(nv)::value;
    const double2* sb = ring_b + slot * BSTAGE + lane;
    if constexpr (COMB) {
#pragma unroll
      for (int j = 0; j < CG.fvc; ++j) {
        const double2 bv = sb[j * 32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int f = 2 * j + h;
          if (f < CG.frc) {
            const int kk = f / CG.ntc, nt = f - (f / CG.ntc) * CG.ntc;
            const double b = h ? bv.y : bv.x;
#pragma unroll
            for (int t = 0; t < NV; ++t) dmma884_nv(acc[t][nt], a_sel<NO>(av[t], kk), b);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < FV; ++j) {
        // keep the B loads of fragment pair j next to its DMMAs (hoisting all of them spills)
        if (KG > 1) asm volatile("" ::: "memory");
#pragma unroll
        for (int kl = 0; kl < KG; ++kl) {
          const double2 bv = sb[kl * BVEC + j * 32];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int f = 2 * j + h;
            if (f < FR) {
              const int kk = f / NT, nt = f - (f / NT) * NT;
              const double b = h ? bv.y : bv.x;
#pragma unroll
              for (int t = 0; t < NV; ++t) dmma884_nv(acc[t][kl * NT + nt], a_sel<NO>(av[t], kk), b);
            }
          }
        }
      }
    }
  };
  auto release = [&](int t) {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + (t % SB));
  };

  const int L = p.lookahead > 0 ? min(p.lookahead, SB - 1) : kKLookahead;
  if (lane == 0)
    for (int i = warp; i < L && i < n_it; i += NW) produce(i);
  auto run = [&](auto nv) {
    for (int it = 0; it < n_it; ++it) {
      if (lane == 0 && it + L < n_it && (it + L) % NW == warp) produce(it + L);
      const int off = s_off[c_w];
      lds_a(off);
      if (warp_emax >= off) compute_tiles(it % SB, nv);
      release(it);
      ++c_it;
      if (++c_w == nw_eff) {
        c_w = 0;
        ++c_sg;
      }
    }
  };
  if (n_valid == MT) run(std::integral_constant<int, MT>{});
  else if (MT > 2 && n_valid == 2) run(std::integral_constant<int, (MT > 2 ? 2 : 0)>{});
  else if (MT > 1 && n_valid == 1) run(std::integral_constant<int, (MT > 1 ? 1 : 0)>{});
  else run(std::integral_constant<int, 0>{});

  if constexpr (COMB) {
    // accumulator n-tile nt, lane: complex column cc = 4 nt + (lane & 3) of the group's
    // [momentum][No] column space
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      if (!v_row[t]) continue;
#pragma unroll
      for (int nt = 0; nt < CG.ntc; ++nt) {
        const int cc = 4 * nt + (lane & 3), kl = cc / NO, n = cc - kl * NO;
        if (kl < KG && k0 + kl < p.nkz)
          sigma_block(p, pol, la, k0 + kl, e_row[t])[m_off[t] + n] = make_double2(-acc[t][nt][1], acc[t][nt][0]);
      }
    }
  } else {
#pragma unroll
    for (int kl = 0; kl < KG; ++kl) {
      if (k0 + kl >= p.nkz) break;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        if (!v_row[t]) continue;
        double2* dst = sigma_block(p, pol, la, k0 + kl, e_row[t]) + m_off[t];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int n = 4 * nt + (lane & 3);
          if (n < NO) dst[n] = make_double2(-acc[t][kl * NT + nt][1], acc[t][kl * NT + nt][0]);
        }
      }
    }
  }
}

// --------------------------------------------------------------------------
// K5: Pi operand build.  One CTA per (chunk atom, k, group of energies):
// dH[a] staged in shared memory; per energy U_{s,j} = dH[a,s,j] @ G2_s and
// VT[(n,p)][(s,i,j)] = (U_{s,j} @ dH[a,s,i])[p][n] (for both chain
// polarities: chain pol 0 (lesser) uses G2 = G>, pol 1 (greater) G2 = G<).
// --------------------------------------------------------------------------
constexpr int kPiBuildEnergies = 8;   // energies per CTA (looped in groups that fit the block)
constexpr int kPiBuildThreads = 288;
constexpr int kPiMaxNo = 16;

// Thread (s, j, pp) of an energy keeps the row U_{s,j}[pp][:] = (dH_{s,j} @ G2_s)[pp][:]
// in registers and emits VT[(n,pp)][(s,i,j)] = (U_{s,j} @ dH_{s,i})[pp][n] for
// all i, n; dH and G2 are read from shared memory (warp-broadcast rows).
__global__ void __launch_bounds__(kPiBuildThreads)
pi_build_kernel(PiBuildArgs p) {
  extern __shared__ double2 smem[];
  const int no = p.no, no2 = no * no, nb = p.nb, ncol = nb * 9;
  const int tpe = nb * 3 * no;                       // threads per energy
  const int epg = tpe >= kPiBuildThreads ? 1 : kPiBuildThreads / tpe;  // energies per pass
  double2* s_dh = smem;                              // [NB][3][no2]
  double2* s_g2 = s_dh + nb * 3 * no2;               // [epg][NB][no2]
  const int n_eb = (p.ne + kPiBuildEnergies - 1) / kPiBuildEnergies;
  int bx = blockIdx.x;
  const int eb = bx % n_eb;
  bx /= n_eb;
  const int k = bx % p.nkz;
  const int la = bx / p.nkz;
  const int a_out = p.atom_begin + la;
  for (int x = threadIdx.x; x < nb * 3 * no2; x += blockDim.x)
    s_dh[x] = p.dH[(long long)a_out * nb * 3 * no2 + x];
  const int e_begin = eb * kPiBuildEnergies, e_end = min(p.ne, e_begin + kPiBuildEnergies);
  for (int pol = 0; pol < 2; ++pol) {
    const double2* G2 = p.G[1 - pol];
    for (int e0 = e_begin; e0 < e_end; e0 += epg) {
      __syncthreads();
      for (int x = threadIdx.x; x < epg * nb * no2; x += blockDim.x) {
        const int sl = x / (nb * no2), y = x % (nb * no2), ss = y / no2, rr = y % no2;
        const int e = e0 + sl;
        if (e < e_end) {
          const int lb = p.nbr[la * nb + ss];
          s_g2[x] = G2[lb * p.g_sa + (long long)k * p.g_sk + (long long)e * p.g_se + rr];
        }
      }
      __syncthreads();
      for (int x = threadIdx.x; x < epg * tpe; x += blockDim.x) {
      const int slot = x / tpe, r = x % tpe;
      const int s = r / (3 * no), j = (r / no) % 3, pp = r % no;
      const int e = e0 + slot;
      if (e >= e_end) continue;
      const bool masked = p.mask && !p.mask[k * p.ne + e];
      double2 u[kPiMaxNo];
      const double2* g2 = s_g2 + (slot * nb + s) * no2;
      const double2* dj = s_dh + (s * 3 + j) * no2 + pp * no;  // dH_{s,j}[pp][:]
#pragma unroll
      for (int t = 0; t < kPiMaxNo; ++t) {
        double re = 0.0, im = 0.0;
        if (t < no)
          for (int rr = 0; rr < no; ++rr) {
            const double2 a = dj[rr], b = g2[rr * no + t];
            re = fma(a.x, b.x, re);
            re = fma(-a.y, b.y, re);
            im = fma(a.x, b.y, im);
            im = fma(a.y, b.x, im);
          }
        u[t] = make_double2(re, im);
      }
      double2* out = p.VT[pol] + (((long long)la * p.nkz + k) * p.ne + e) * no2 * ncol;
      for (int i = 0; i < 3; ++i) {
        const double2* di = s_dh + (s * 3 + i) * no2;  // dH_{s,i}
        const int c = s * 9 + i * 3 + j;
        for (int n = 0; n < no; ++n) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int t = 0; t < kPiMaxNo; ++t) {
            if (t < no) {
              const double2 b = di[t * no + n];
              re = fma(u[t].x, b.x, re);
              re = fma(-u[t].y, b.y, re);
              im = fma(u[t].x, b.y, im);
              im = fma(u[t].y, b.x, im);
            }
          }
          const int kap = n * no + pp;
          out[(long long)kap * ncol + (c ^ vt_swz(kap, no, p.swz))] =
              masked ? make_double2(0.0, 0.0) : make_double2(re, im);
        }
      }
      }
    }
  }
}

// --------------------------------------------------------------------------
// K5 v2 (DMMA, No % 4 == 0): the same V on FP64 tensor cores.  Per (point,
// chain polarity, s) two real-embedded GEMMs:
//   U_s = [dH_{s,0}; dH_{s,1}; dH_{s,2}] (3No x No) @ G2_s (No x No)
//   W_s = U_s (3No x No) @ [dH_{s,0} | dH_{s,1} | dH_{s,2}] (No x 3No)
// W_s[(j,p)][(i,n)] = V_ij[p][n].  A warp owns one 8-row m-tile of U/W: the C
// fragments of the first GEMM are, lane for lane, the A fragments of the
// second (U[m][4kh + lane%4] is n-tile kh of the first product), so U never
// leaves registers.  W is scattered into a shared-memory image of the point's
// V block ([(n,p)][(s,i,j)], column-swizzled like K5) and written to HBM by
// one bulk async copy (TMA) per point and polarity, double-buffered so the
// store of one polarity overlaps the products of the next.
// --------------------------------------------------------------------------
constexpr int kPB2Warps = 20;     // 4 slots x 5 m-tiles at No = 12, NB = 4
constexpr int kPB2Energies = 16;  // energies per CTA (dH staged once per CTA)

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int NO, int WG0 = 3>
__global__ void __launch_bounds__(kPB2Warps * 32, 1)
pi_build_dmma_kernel(PiBuildArgs p) {
  constexpr int NO2 = NO * NO, MROWS = 3 * NO, MT = (MROWS + 7) / 8;
  // No % 4 != 0 (e.g. 10, the small config): K and N padded to multiples of 4 complex (the
  // padding reads zeros through the guards below)
  constexpr int KH = (NO + 3) / 4;          // k-steps per real/imaginary half
  constexpr int NT1 = (NO + 3) / 4;         // n-tiles of U (2No real columns)
  constexpr int NT2 = (6 * NO + 7) / 8;     // n-tiles of W (6No real columns)
  constexpr bool PAD = NO % 4 != 0;
  constexpr int NOP = NO + 1;        // padded smem row of dH / G2 blocks: the B reads (4 rows
                                     // of a quarter warp) hit distinct banks
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int nb = p.nb, ncol = nb * 9;
  const int vt_vec = NO2 * ncol;  // double2 per point and polarity
  double2* vt = reinterpret_cast<double2*>(smem_raw);          // [2][No2][ncol]
  double2* sdh = vt + 2 * vt_vec;                               // [nb][3][No][NOP]
  double2* sg2_buf = sdh + nb * 3 * NO * NOP;                   // [2][nb][No][NOP] (double-buffered)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e_groups = (p.ne + kPB2Energies - 1) / kPB2Energies;
  int bx = blockIdx.x;
  const int eg = bx % e_groups;
  bx /= e_groups;
  const int k = bx % p.nkz;
  const int la = bx / p.nkz;
  const int e0 = eg * kPB2Energies, e1 = min(p.ne, e0 + kPB2Energies);

  const double2* dH = p.dH + (long long)(p.atom_begin + la) * nb * 3 * NO2;
  for (int x = threadIdx.x; x < nb * 3 * NO2; x += blockDim.x) sdh[(x / NO) * NOP + x % NO] = dH[x];

  const int im = (lane >> 2) & 1;                  // this lane's B column is an imaginary part
  const unsigned neg = im ? 0u : 0x80000000u;      // the im-row of a real column is -Im
  const int kl = lane & 3;
  const int tasks = nb * MT;
  // G2 blocks of (point e, chain polarity pol): element x = (s, rr); the next
  // step's first kPB2Prefetch * blockDim elements are loaded into registers
  // while the current step multiplies (the rest, if any, synchronously)
  constexpr int kPB2Prefetch = 2;
  auto g2_elem = [&](int e_, int pol_, int x) -> double2 {
    if (p.mask && !p.mask[k * p.ne + e_]) return make_double2(0.0, 0.0);
    const int ss = x / NO2, rr = x % NO2;
    const long long lb = p.nbr[la * nb + ss];
    if (p.peer.ranks > 0)  // G2 of chain pol 0 is G>, of pol 1 G<
      return peer_block(p.peer, pol_ ? 0 : 1, (long long)k * p.ne + e_, lb, NO2)[rr];
    const double2* G2 = pol_ ? p.G[0] : p.G[1];  // chain pol 0 (lesser): G2 = G>; pol 1: G2 = G<
    return G2[lb * p.g_sa + (long long)k * p.g_sk + (long long)e_ * p.g_se + rr];
  };
  double2 pf[kPB2Prefetch];
  auto fetch = [&](int e_, int pol_) {
#pragma unroll
    for (int i = 0; i < kPB2Prefetch; ++i) {
      const int x = threadIdx.x + i * blockDim.x;
      pf[i] = x < nb * NO2 ? g2_elem(e_, pol_, x) : make_double2(0.0, 0.0);
    }
  };
  if (e0 < e1) fetch(e0, 0);
  int step = 0;  // (point, polarity) counter: buffer = step & 1
  auto store_v = [&](int st_, int e_, int pol_) {  // thread 0: V image of step st_ -> HBM (TMA)
    double2* out = p.VT[pol_] + (((long long)la * p.nkz + k) * p.ne + e_) * vt_vec;
    bulk_s2g(out, vt + (st_ & 1) * vt_vec, (uint32_t)vt_vec * 16);
    bulk_commit();
  };
  // one CTA barrier per (point, polarity) step: the G2 staging is double-buffered (sg2 of step t
  // was last read in step t-2, before the previous barrier), and thread 0 waits for the V store
  // that last read this step's V buffer BEFORE the barrier, so no thread writes it early
  for (int e = e0; e < e1; ++e) {
    for (int pol = 0; pol < 2; ++pol, ++step) {
      double2* buf = vt + (step & 1) * vt_vec;
      double2* sg2 = sg2_buf + (step & 1) * nb * NO * NOP;
#pragma unroll
      for (int i = 0; i < kPB2Prefetch; ++i) {
        const int x = threadIdx.x + i * blockDim.x;
        if (x < nb * NO2) sg2[(x / NO) * NOP + x % NO] = pf[i];
      }
      for (int x = threadIdx.x + kPB2Prefetch * blockDim.x; x < nb * NO2; x += blockDim.x)
        sg2[(x / NO) * NOP + x % NO] = g2_elem(e, pol, x);
      if (threadIdx.x == 0 && step >= 2) bulk_wait_read<0>();  // buf's store (issued last step) read it
      __syncthreads();  // sg2 written; step-1's products are in the other V buffer
      if (threadIdx.x == 0 && step >= 1) store_v(step - 1, pol ? e : e - 1, pol ? 0 : 1);  // previous step
      if (pol == 0) fetch(e, 1);
      else if (e + 1 < e1) fetch(e + 1, 0);
      for (int task = warp; task < tasks; task += kPB2Warps) {
        const int ss = task / MT, mt = task % MT;
        const int m = mt * 8 + (lane >> 2);
        const bool m_ok = m < MROWS;
        const int mj = m_ok ? m / NO : 0, mp = m_ok ? m % NO : 0;
        const double2* dsr = sdh + ((ss * 3 + mj) * NO + mp) * NOP;  // row (j, p) of D_s
        const double2* g2 = sg2 + ss * NO * NOP;
        double u[NT1][2];
#pragma unroll
        for (int nt = 0; nt < NT1; ++nt) u[nt][0] = u[nt][1] = 0.0;
#pragma unroll
        for (int kh = 0; kh < KH; ++kh) {
          const int r = 4 * kh + kl;
          const double2 a = (m_ok && (!PAD || r < NO)) ? dsr[r] : make_double2(0.0, 0.0);
#pragma unroll
          for (int nt = 0; nt < NT1; ++nt) {
            const int n = (nt * 8 + (lane >> 2)) >> 1;
            const double2 g = (!PAD || (r < NO && n < NO)) ? g2[r * NOP + n] : make_double2(0.0, 0.0);
            dmma884_nv(u[nt], a.x, im ? g.y : g.x);
            dmma884_nv(u[nt], a.y, xor_sign(im ? g.x : g.y, neg));
          }
        }
        // W in groups of WG n-tiles, each group stored right after its last DMMA, so the V-image
        // scatter (STS) of one group overlaps the DMMAs of the next (the same per-accumulator order)
        constexpr int WG = NT2 % WG0 == 0 ? WG0 : (NT2 % 3 == 0 ? 3 : (NT2 % 2 == 0 ? 2 : 1));
#pragma unroll
        for (int g0 = 0; g0 < NT2; g0 += WG) {
          double w[WG][2];
#pragma unroll
          for (int x = 0; x < WG; ++x) w[x][0] = w[x][1] = 0.0;
#pragma unroll
          for (int kh = 0; kh < KH; ++kh) {
            const int t = 4 * kh + kl;  // U[m][t] = u[kh] of this lane
#pragma unroll
            for (int x = 0; x < WG; ++x) {
              const int nt = g0 + x;
              const int cc = (nt * 8 + (lane >> 2)) >> 1, i = cc / NO, n = cc % NO;
              const double2 h = (!PAD || (t < NO && cc < 3 * NO)) ? sdh[((ss * 3 + i) * NO + t) * NOP + n]
                                                                   : make_double2(0.0, 0.0);
              dmma884_nv(w[x], u[kh][0], im ? h.y : h.x);
              dmma884_nv(w[x], u[kh][1], xor_sign(im ? h.x : h.y, neg));
            }
          }
          if (m_ok) {
#pragma unroll
            for (int x = 0; x < WG; ++x) {
              const int nt = g0 + x;
              const int cc = nt * 4 + kl, i = cc / NO, n = cc % NO;
              const int kap = n * NO + mp;
              const int c = ss * 9 + i * 3 + mj;
              if (!PAD || cc < 3 * NO) buf[kap * ncol + (c ^ vt_swz(kap, NO, p.swz))] = make_double2(w[x][0], w[x][1]);
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // STS visible to the bulk copy
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (step >= 1) store_v(step - 1, e1 - 1, 1);
    bulk_wait_all();
  }
}

// --------------------------------------------------------------------------
// K6: Pi chains on FP64 tensor cores.  CTA = (chunk atom, chain polarity, q,
// E-chunk); 9 warps, warp w covers a 3x3 block of 8x8 tiles of the
// [Nw x 2*ncol] real-embedded chain block (rows = frequencies w, columns =
// (Re, Im) of (s, i, j)); K = (k, E, n, p): A = G1[(k+q)%Nkz, E+off_w, a]
// (zero when E+off_w >= NE), B = VT[k][E] (real embedding built on the fly
// from the complex operand).  Register double buffer over the flattened
// (k, E, kappa-pair) loop.
// --------------------------------------------------------------------------
constexpr int kPiWarps = 9;

__global__ void __launch_bounds__(kPiWarps * 32)
pi_dmma_direct_kernel(PiArgs p, int chunk_atoms) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int bx = blockIdx.x;
  const int ec = bx % p.echunks;
  bx /= p.echunks;
  const int q = bx % p.nqz;
  bx /= p.nqz;
  const int pol = bx % 2;
  const int la = bx / 2;
  const int wg = blockIdx.y * kPiWarps + warp;
  if (wg >= p.warp_groups) return;
  const int no2 = p.no * p.no;
  const int khp = (no2 + 3) / 4;                 // kappa pairs (k-step pairs)
  const int n_ntile = (2 * p.ncol + 7) / 8;
  const int gn = (n_ntile + 2) / 3;
  const int mg = wg / gn, ng = wg % gn;
  const int pcol = lane & 3;

  const double2* __restrict__ G1 = p.G[pol];
  const double2* __restrict__ VT = p.VT[pol] + (long long)la * p.nkz * p.ne * no2 * p.ncol;
  const long long g_atom = (p.g_atom_of_chunk0 + la) * p.g_sa;

  // per-lane rows (frequencies) of the warp's 3 m-tiles, and columns of its 3 n-tiles
  int off_t[3];
  bool row_ok[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int w = (mg * 3 + t) * 8 + (lane >> 2);
    row_ok[t] = w < p.nw;
    off_t[t] = row_ok[t] ? __ldg(p.off + w) : 0;
  }
  int col_c[3];
  bool col_ok[3], part_im[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int nc = (ng * 3 + u) * 8 + (lane >> 2);
    col_c[u] = nc >> 1;
    part_im[u] = nc & 1;
    col_ok[u] = col_c[u] < p.ncol;
  }
  // smallest offset of the warp's rows (for the warp-uniform skip E + off >= NE)
  int off_min = 1 << 30;
#pragma unroll
  for (int t = 0; t < 3; ++t)
    if (row_ok[t]) off_min = min(off_min, off_t[t]);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) off_min = min(off_min, __shfl_xor_sync(0xffffffffu, off_min, sh));

  double acc[3][3][2];
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int u = 0; u < 3; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

  const int e_lo = ec * p.e_per_chunk, e_hi = min(p.ne, e_lo + p.e_per_chunk);
  // flattened loop over (k, E in [e_lo, min(e_hi, NE - off_min)), kappa pair)
  const int e_end = min(e_hi, p.ne - off_min);
  const int ne_c = max(0, e_end - e_lo);
  const long long n_it = (long long)p.nkz * ne_c * khp;

  struct Ops {
    double2 a[3];
    double2 b[3];
  };
  auto load = [&](Ops& o, long long it) {
    const int kq = (int)(it % khp);
    const long long ke = it / khp;
    const int e = e_lo + (int)(ke % ne_c);
    const int k = (int)(ke / ne_c);
    int kp = (k + q) % p.nkz;
    const int kap = kq * 4 + pcol;
    const bool kap_ok = kap < no2;
    const double2* arow = G1 + g_atom + (long long)kp * p.g_sk + kap;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      o.a[t] = make_double2(0.0, 0.0);
      if (row_ok[t] && kap_ok && e + off_t[t] < p.ne) o.a[t] = __ldg(arow + (long long)(e + off_t[t]) * p.g_se);
    }
    const double2* brow = VT + (((long long)k * p.ne + e) * no2 + kap) * p.ncol;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      o.b[u] = make_double2(0.0, 0.0);
      if (col_ok[u] && kap_ok) o.b[u] = __ldg(brow + col_c[u]);
    }
  };
  auto compute = [&](const Ops& o) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const double a = h == 0 ? o.a[t].x : o.a[t].y;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          // B'[re-row][2c] = Re V, [re-row][2c+1] = Im V, [im-row][2c] = -Im V, [im-row][2c+1] = Re V
          const double b = h == 0 ? (part_im[u] ? o.b[u].y : o.b[u].x) : (part_im[u] ? o.b[u].x : -o.b[u].y);
          dmma884(acc[t][u], a, b);
        }
      }
  };
  Ops o0, o1;
  if (n_it > 0) load(o0, 0);
  for (long long it = 0; it < n_it; it += 2) {
    if (it + 1 < n_it) load(o1, it + 1);
    compute(o0);
    if (it + 1 >= n_it) break;
    if (it + 2 < n_it) load(o0, it + 2);
    compute(o1);
  }

  // partial chains (w_E-scaled) of this E-chunk: lane holds (Re, Im) of
  // C[row w][col c = 4 ntile + (lane & 3)]
  double2* part = p.partial + ((((long long)la * 2 + pol) * p.nqz + q) * p.echunks + ec) * p.nw * p.ncol;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int w = (mg * 3 + t) * 8 + (lane >> 2);
    if (w >= p.nw) continue;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int c = (ng * 3 + u) * 4 + (lane & 3);
      if (c < p.ncol)
        part[(long long)w * p.ncol + c] = make_double2(p.energy_weight * acc[t][u][0], p.energy_weight * acc[t][u][1]);
    }
  }
}

// --------------------------------------------------------------------------
// K6 (TMA): the production Pi kernel.  CTA = (chunk atom, chain polarity,
// q-block of up to kPiQB momenta, E-chunk); 9 warps, warp = (m-group,
// n-group) owning 3 x 3 tiles of the chain block for each q of the block.
// The B operand VT[k][E] (No^2 x ncol complex, contiguous) is staged per
// (k, E) step by the TMA engine into a 2-slot shared-memory ring (full/empty
// mbarriers, producer rotated over the warps), read with 16-byte LDS and
// turned into the real-embedded fragments with selects; A = G1 rows through
// L1/L2 with a register double buffer over kappa pairs.  Each VT stage feeds
// all q of the block (one HBM read of VT per (atom, polarity, q-block)).
// --------------------------------------------------------------------------
constexpr int kPiQB = 2;

// -x by flipping the sign bit with an integer instruction (the compiler would
// otherwise emit DADD on the FP64 pipe, which the DMMAs need)
__device__ __forceinline__ double neg_sign_bit(double x) {
  unsigned lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(x));
  asm volatile("xor.b32 %0, %0, 0x80000000;" : "+r"(hi));
  double r;
  asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
  return r;
}
constexpr int kPiStages = 2;

__global__ void __launch_bounds__(kPiWarps * 32, 1)
pi_dmma_kernel(PiArgs p, int chunk_atoms) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int no2 = p.no * p.no, ncol = p.ncol;
  const int stage_vec = no2 * ncol;
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kPiStages * stage_vec);
  uint64_t* empty = full + kPiStages;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int qblocks = (p.nqz + kPiQB - 1) / kPiQB;
  int bx = blockIdx.x;
  const int ec = bx % p.echunks;
  bx /= p.echunks;
  const int qb = bx % qblocks;
  bx /= qblocks;
  const int pol = bx % 2;
  const int la = bx / 2;
  const int q0 = qb * kPiQB, nq = min(kPiQB, p.nqz - q0);
  const int wg = blockIdx.y * kPiWarps + warp;
  const bool active = wg < p.warp_groups;  // idle warps still take part in the barriers
  const int khp = (no2 + 3) / 4;
  const int n_ntile = (2 * ncol + 7) / 8;
  const int gn = (n_ntile + 2) / 3;
  const int mg = active ? wg / gn : 0, ng = active ? wg % gn : 0;
  const int pcol = lane & 3;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPiStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kPiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const double2* __restrict__ G1 = p.G[pol];
  const double2* __restrict__ VT = p.VT[pol] + (long long)la * p.nkz * p.ne * stage_vec;
  const long long g_atom = (p.g_atom_of_chunk0 + la) * p.g_sa;

  int off_t[3];
  bool row_ok[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int w = (mg * 3 + t) * 8 + (lane >> 2);
    row_ok[t] = active && w < p.nw;
    off_t[t] = row_ok[t] ? __ldg(p.off + w) : 0;
  }
  int col_c[3];
  bool col_ok[3], part_im[3];
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    const int nc = (ng * 3 + u) * 8 + (lane >> 2);
    col_c[u] = nc >> 1;
    part_im[u] = nc & 1;
    col_ok[u] = active && col_c[u] < ncol;
  }
  int off_min = 1 << 30;
#pragma unroll
  for (int t = 0; t < 3; ++t)
    if (row_ok[t]) off_min = min(off_min, off_t[t]);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) off_min = min(off_min, __shfl_xor_sync(0xffffffffu, off_min, sh));

  double acc[kPiQB][3][3][2];
#pragma unroll
  for (int qq = 0; qq < kPiQB; ++qq)
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < 3; ++u) acc[qq][t][u][0] = acc[qq][t][u][1] = 0.0;

  const int e_lo = ec * p.e_per_chunk, e_hi = min(p.ne, e_lo + p.e_per_chunk);
  const int ne_c = e_hi - e_lo;
  const int n_st = p.nkz * ne_c;  // (k, E) stages
  const long long n_it = (long long)n_st * khp;

  auto produce = [&](int st) {  // lane 0 of warp st % kPiWarps
    const int slot = st % kPiStages;
    if (st >= kPiStages) mbar_wait(empty + slot, (uint32_t)(((st - kPiStages) / kPiStages) & 1));
    const int k = st / ne_c, e = e_lo + st % ne_c;
    mbar_arrive_expect_tx(full + slot, (uint32_t)stage_vec * 16);
    bulk_g2s(ring + slot * stage_vec, VT + ((long long)k * p.ne + e) * stage_vec, (uint32_t)stage_vec * 16,
             full + slot);
  };
  struct OpsA {
    double2 a[kPiQB][3];
  };
  auto load_a = [&](OpsA& o, long long it) {
    const int kq = (int)(it % khp);
    const int st = (int)(it / khp);
    const int k = st / ne_c, e = e_lo + st % ne_c;
    const int kap = kq * 4 + pcol;
    const bool kap_ok = kap < no2;
#pragma unroll
    for (int qq = 0; qq < kPiQB; ++qq) {
      const int kp = (k + q0 + qq) % p.nkz;
      const double2* arow = G1 + g_atom + (long long)kp * p.g_sk + kap;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        o.a[qq][t] = make_double2(0.0, 0.0);
        if (qq < nq && row_ok[t] && kap_ok && e + off_t[t] < p.ne)
          o.a[qq][t] = __ldg(arow + (long long)(e + off_t[t]) * p.g_se);
      }
    }
  };
  auto step = [&](const OpsA& o, long long it) {
    const int kq = (int)(it % khp);
    const int st = (int)(it / khp);
    const int e = e_lo + st % ne_c;
    if (kq == 0) {
      if (lane == 0 && st + 1 < n_st && (st + 1) % kPiWarps == warp) produce(st + 1);
      mbar_wait(full + st % kPiStages, (uint32_t)((st / kPiStages) & 1));
    }
    if (active && e + off_min < p.ne) {
      const int kap = kq * 4 + pcol;
      const double2* sb = ring + (st % kPiStages) * stage_vec + (long long)kap * ncol;
      // real-embedded B fragments of the two k-steps of this kappa pair:
      // re-row: (Re V, Im V) by column parity, im-row: (-Im V, Re V); the
      // negation flips the sign bit on the integer pipe (no FP64-pipe op)
      double b_re[3], b_im[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const double2 v = (col_ok[u] && kap < no2) ? sb[col_c[u]] : make_double2(0.0, 0.0);
        const double neg_im = neg_sign_bit(v.y);
        b_re[u] = part_im[u] ? v.y : v.x;
        b_im[u] = part_im[u] ? v.x : neg_im;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int qq = 0; qq < kPiQB; ++qq) {
          if (qq >= nq) continue;
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const double a = h == 0 ? o.a[qq][t].x : o.a[qq][t].y;
#pragma unroll
            for (int u = 0; u < 3; ++u) dmma884(acc[qq][t][u], a, h == 0 ? b_re[u] : b_im[u]);
          }
        }
    }
    if (kq == khp - 1) {  // done with this stage's shared memory
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st % kPiStages);
    }
  };

  if (threadIdx.x == 0 && n_st > 0) produce(0);
  OpsA o0, o1;
  if (n_it > 0) load_a(o0, 0);
  for (long long it = 0; it < n_it; it += 2) {
    if (it + 1 < n_it) load_a(o1, it + 1);
    step(o0, it);
    if (it + 1 >= n_it) break;
    if (it + 2 < n_it) load_a(o0, it + 2);
    step(o1, it + 1);
  }

  if (!active) return;
#pragma unroll
  for (int qq = 0; qq < kPiQB; ++qq) {
    if (qq >= nq) continue;
    double2* part =
        p.partial + ((((long long)la * 2 + pol) * p.nqz + q0 + qq) * p.echunks + ec) * p.nw * ncol;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int w = (mg * 3 + t) * 8 + (lane >> 2);
      if (w >= p.nw) continue;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int c = (ng * 3 + u) * 4 + (lane & 3);
        if (c < ncol)
          part[(long long)w * ncol + c] =
              make_double2(p.energy_weight * acc[qq][t][u][0], p.energy_weight * acc[qq][t][u][1]);
      }
    }
  }
}

// --------------------------------------------------------------------------
// K6 v2 (TMA, half stages, two CTAs per SM): the production Pi kernel.
// CTA = (chunk atom, chain polarity, E-chunk, q) with q fastest, so the Nqz
// CTAs streaming the same V run side by side and share it through L2.
// 9 warps x 3x3 tiles (one q); every (k, E) stage of V is copied in two
// kappa halves into a 2-slot ring (41.5 KB slots at No = 12), so two CTAs
// fit one SM (18 warps, 5/5/4/4 per SMSP instead of 3/2/2/2).  The inner
// loop carries no divisions: stage coordinates advance incrementally, A rows
// come from per-stage pointers (register double buffer across iterations and
// stages), B fragments are two LDS.64 per column tile (the real-embedding
// swap is a per-lane address offset, the negation a per-lane sign mask).
// Accumulation order equals K6's: (k, E, kappa, h) ascending per output.
// --------------------------------------------------------------------------
constexpr int kPi2Slots = 2;


// 112 registers: 2 x 9 warps x 32 x 112 = 64.5 K registers per SM
// A row for invalid (w, E + off_w >= NE) rows: zeros, so the loads need no predicate
__device__ double2 kPiZeroRow[kPiMaxNo * kPiMaxNo];
constexpr int kPi2Pad = 64;  // double2 past the ring: B reads of discarded columns stay in bounds

__global__ void __launch_bounds__(kPiWarps * 32, 2)
pi_dmma2_kernel(PiArgs p, int chunk_atoms) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int no2 = p.no * p.no, ncol = p.ncol;
  const int khp = (no2 + 3) / 4;        // kappa quads per stage
  const int kh0 = (khp + 1) / 2;        // quads in the first half
  const int slot_vec = kh0 * 4 * ncol;  // double2 per slot (the larger half)
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kPi2Slots * slot_vec + kPi2Pad);
  uint64_t* empty = full + kPi2Slots;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int bx = blockIdx.x;
  const int q = bx % p.nqz;
  bx /= p.nqz;
  const int ec = bx % p.echunks;
  bx /= p.echunks;
  const int pol = bx % 2;
  const int la = bx / 2;
  const int wg = blockIdx.y * kPiWarps + warp;
  const bool active = wg < p.warp_groups;  // idle warps still take part in the barriers
  const int n_ntile = (2 * ncol + 7) / 8;
  const int gn = (n_ntile + 2) / 3;
  const int mg = active ? wg / gn : 0, ng = active ? wg % gn : 0;
  const int pcol = lane & 3;

  // rows past No^2 in a slot are never copied: keep them finite (zero); they meet
  // the clamped (finite) A of ragged quads, and their products are discarded zeros
  for (int i = threadIdx.x; i < kPi2Slots * slot_vec + kPi2Pad; i += blockDim.x) ring[i] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPi2Slots; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kPiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero stores before async-proxy writes
  __syncthreads();

  const double2* __restrict__ G1 = pol ? p.G[1] : p.G[0];
  const double2* __restrict__ VT = (pol ? p.VT[1] : p.VT[0]) + (long long)la * p.nkz * p.ne * no2 * ncol;
  const double2* g_atom = G1 + (p.g_atom_of_chunk0 + la) * p.g_sa;

  int off_t[3];
  bool row_ok[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int w = (mg * 3 + t) * 8 + (lane >> 2);
    row_ok[t] = active && w < p.nw;
    off_t[t] = row_ok[t] ? __ldg(p.off + w) : 0;
  }
  // B fragments (doubles within a kappa row of the slot): tile u reads column
  // c0 + 4u; the re-row takes component `im`, the im-row the other component,
  // sign-flipped when it is Im V.  Columns >= ncol feed discarded outputs.
  const int nc0 = ng * 3 * 8 + (lane >> 2);
  const int im = nc0 & 1;
  const int b_off = 2 * (nc0 >> 1) + im;
  const unsigned b_mask = im ? 0u : 0x80000000u;
  int off_min = 1 << 30;
#pragma unroll
  for (int t = 0; t < 3; ++t)
    if (row_ok[t]) off_min = min(off_min, off_t[t]);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) off_min = min(off_min, __shfl_xor_sync(0xffffffffu, off_min, sh));

  double acc[3][3][2];
#pragma unroll
  for (int t = 0; t < 3; ++t)
#pragma unroll
    for (int u = 0; u < 3; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

  const int e_lo = ec * p.e_per_chunk, e_hi = min(p.ne, e_lo + p.e_per_chunk);
  const int ne_c = e_hi - e_lo;
  const int n_st = p.nkz * ne_c;
  const int n_ss = 2 * n_st;  // half stages

  // producer of half stage ss (lane 0 of warp ss % kPiWarps)
  auto produce = [&](int ss) {
    const int slot = ss & 1;
    if (ss >= kPi2Slots) mbar_wait(empty + slot, (uint32_t)(((ss - kPi2Slots) >> 1) & 1));
    const int st = ss >> 1, half = ss & 1;
    const int k = st / ne_c, e = e_lo + st % ne_c;
    const int r0 = half ? kh0 * 4 : 0;
    const int r1 = half ? no2 : min(no2, kh0 * 4);
    if (r1 <= r0) {  // empty half (khp == 1)
      mbar_arrive(full + slot);
      return;
    }
    const uint32_t bytes = (uint32_t)(r1 - r0) * ncol * 16;
    mbar_arrive_expect_tx(full + slot, bytes);
    bulk_g2s(ring + slot * slot_vec, VT + (((long long)k * p.ne + e) * no2 + r0) * ncol, bytes, full + slot);
  };

  // A rows of a stage: G1[(k+q) % Nkz, e + off_t, atom] (zero row when invalid)
  const double2* rows[3];
  auto stage_rows = [&](int k, int e) {
    int kp = k + q;
    if (kp >= p.nkz) kp -= p.nkz;
    const double2* base = g_atom + (long long)kp * p.g_sk + (long long)e * p.g_se;
#pragma unroll
    for (int t = 0; t < 3; ++t)
      rows[t] = (row_ok[t] && e + off_t[t] < p.ne) ? base + off_t[t] * p.g_se : kPiZeroRow;
  };
  const int kap_max = no2 - 1;
  auto load_a = [&](double2 (&a)[3], int kq) {
    const int kap = min(kq * 4 + pcol, kap_max);  // ragged last quad: any finite element
#pragma unroll
    for (int t = 0; t < 3; ++t) a[t] = __ldg(rows[t] + kap);
  };
  auto mma = [&](const double2 (&a)[3], const double* sb) {
    double b_re[3], b_im[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      b_re[u] = sb[b_off + 8 * u];
      b_im[u] = xor_sign(sb[(b_off ^ 1) + 8 * u], b_mask);
    }
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < 3; ++u) dmma884(acc[t][u], a[t].x, b_re[u]);
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < 3; ++u) dmma884(acc[t][u], a[t].y, b_im[u]);
  };

  if (threadIdx.x == 0 && n_ss > 0) produce(0);
  int k = 0, e = e_lo;
  stage_rows(k, e);
  double2 a[3];
  load_a(a, 0);
  bool live = active && e + off_min < p.ne;  // warp-uniform, per stage
  for (int ss = 0; ss < n_ss; ++ss) {
    const int half = ss & 1;
    if (lane == 0 && ss + 1 < n_ss && (ss + 1) % kPiWarps == warp) produce(ss + 1);
    mbar_wait(full + half, (uint32_t)((ss >> 1) & 1));
    const double* sb = reinterpret_cast<const double*>(ring + half * slot_vec) + pcol * 2 * ncol;
    const int kq0 = half ? kh0 : 0, kq1 = half ? khp : kh0;
    const bool stage_end = kq1 == khp;
    const int kq_plain = stage_end ? kq1 - 1 : kq1;
    if (live) {
      // ping-pong: quad kq+1's A is loaded while quad kq multiplies
#pragma unroll 2
      for (int kq = kq0; kq < kq_plain; ++kq) {
        double2 an[3];
        load_a(an, kq + 1);
        mma(a, sb);
#pragma unroll
        for (int t = 0; t < 3; ++t) a[t] = an[t];
        sb += 8 * ncol;
      }
    }
    if (stage_end && kq0 < kq1) {  // last quad: prefetch the next stage's first quad
      if (++e == e_hi) {
        e = e_lo;
        ++k;
      }
      const bool live_now = live;
      double2 an[3];
      if (ss + 1 < n_ss) {
        stage_rows(k, e);
        load_a(an, 0);
      }
      if (live_now) mma(a, sb);
#pragma unroll
      for (int t = 0; t < 3; ++t) a[t] = an[t];
      live = active && e + off_min < p.ne;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + half);
  }

  if (!active) return;
  double2* part = p.partial + ((((long long)la * 2 + pol) * p.nqz + q) * p.echunks + ec) * p.nw * ncol;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const int w = (mg * 3 + t) * 8 + (lane >> 2);
    if (w >= p.nw) continue;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int c = (ng * 3 + u) * 4 + (lane & 3);
      if (c < ncol)
        part[(long long)w * ncol + c] = make_double2(p.energy_weight * acc[t][u][0], p.energy_weight * acc[t][u][1]);
    }
  }
}

// --------------------------------------------------------------------------
// K6 v3 (production for No >= 3): as v2 (TMA half stages, 2 CTAs per SM, q
// fastest), but each warp owns ONE 8-row m-tile (8 lags w) across 9 n-tiles
// (72 real columns = 36 complex chains), so no two warps of a CTA load the same
// G1 row (v2: 3x), and one A fragment per quad lets the register prefetch run
// two quads ahead across half-stage and stage boundaries.  B: per n-tile two
// LDS.64 (component swap by lane address, sign by lane mask) from the slot.
// Same per-output accumulation order as K6/v2: (k, E, kappa quad, h).
// --------------------------------------------------------------------------
constexpr int kPi3NT = 9;     // n-tiles per warp
constexpr int kPi3Sub = 6;    // sub-stages per (k, E) stage (6 quads each at No = 12)
constexpr int kPi3Slots = 4;  // ring slots: the producer runs kPi3Slots - 1 sub-stages ahead

// LAST_PRODUCES: the warp that releases a slot last refills it (a shared-memory
// counter per slot, atom.inc with wrap-around), so no warp ever blocks on an
// empty barrier; otherwise lane 0 of warp t % 9 refills slot t after waiting
// for every warp's release (empty mbarrier).
// NOT/NBT > 0: No and NB fixed at compile time (the paper shapes), so every
// sub-stage is a fixed, fully unrolled run of quad pairs with no branches.
// NW / MINB: warps per CTA and CTAs per SM (default 9 and 3 = 72 registers)
template <bool LAST_PRODUCES, int NOT, int NBT, int NW = kPiWarps, int MINB = 3>
__global__ void __launch_bounds__(NW * 32, MINB)
pi_dmma3_kernel(PiArgs p, int chunk_atoms) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int no = NOT > 0 ? NOT : p.no;
  const int no2 = no * no, ncol = NBT > 0 ? 9 * NBT : p.ncol;
  const int khp = (no2 + 3) / 4;                     // kappa quads per stage (>= 2 here)
  const int qs = 2 * ((khp + 2 * kPi3Sub - 1) / (2 * kPi3Sub));  // quads per sub-stage (even)
  // compile-time: every sub-stage holds exactly qs quads (qs even, khp % qs == 0)
  constexpr int KHP_T = NOT > 0 ? (NOT * NOT + 3) / 4 : 0;
  constexpr int QS_T = NOT > 0 ? 2 * ((KHP_T + 2 * kPi3Sub - 1) / (2 * kPi3Sub)) : 0;
  constexpr bool UNIFORM = NOT > 0 && NBT > 0 && KHP_T % QS_T == 0 && KHP_T / QS_T == kPi3Sub;
  const int slot_vec = qs * 4 * ncol;                // double2 per slot
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kPi3Slots * slot_vec + kPi2Pad);
  uint64_t* empty = full + kPi3Slots;
  unsigned* rel = reinterpret_cast<unsigned*>(empty + kPi3Slots);  // releases per slot
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int bx = blockIdx.x;
  const int m_tiles = (p.nw + 7) / 8;
  const int n_groups = ((2 * ncol + 7) / 8 + kPi3NT - 1) / kPi3NT;
  // q_in_warps (few lag tiles, e.g. Nw = 16: 2 tiles of 9 warps): the CTA serves every q, warp =
  // (q, tile); its warps share the V stages (V depends on (k, E) only) and read their own G1 rows
  int q, wg;
  if (p.q_in_warps) {
    q = warp / (m_tiles * n_groups);
    wg = warp % (m_tiles * n_groups);
  } else {
    q = bx % p.nqz;
    bx /= p.nqz;
    wg = blockIdx.y * NW + warp;
  }
  const int ec = bx % p.echunks;
  bx /= p.echunks;
  const int pol = bx % 2;
  const int la = bx / 2;
  const bool active = wg < m_tiles * n_groups && q < p.nqz;  // idle warps still take part in the barriers
  const int mt = active ? wg % m_tiles : 0, ng = active ? wg / m_tiles : 0;
  const int pcol = lane & 3;

  for (int i = threadIdx.x; i < kPi3Slots * slot_vec + kPi2Pad; i += blockDim.x) ring[i] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPi3Slots; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NW);
      rel[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  const double2* __restrict__ G1 = pol ? p.G[1] : p.G[0];
  const double2* __restrict__ VT = (pol ? p.VT[1] : p.VT[0]) + (long long)la * p.nkz * p.ne * no2 * ncol;
  const double2* g_atom = G1 + (p.g_atom_of_chunk0 + la) * p.g_sa;

  const int w = mt * 8 + (lane >> 2);
  const bool row_ok = active && w < p.nw;
  const int off = row_ok ? __ldg(p.off + w) : 0;
  int off_min = row_ok ? off : (1 << 30);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) off_min = min(off_min, __shfl_xor_sync(0xffffffffu, off_min, sh));
  const int nc0 = ng * kPi3NT * 8 + (lane >> 2);
  const int im = nc0 & 1;
  // column of tile 0 in the (swizzled) slot row: kappa rows with bit 1 set hold
  // column c at c ^ swz; the xor keeps tile u's column at +4u (8u doubles)
  const int b_off = 2 * ((nc0 >> 1) ^ (((pcol >> 1) & 1) ? p.swz : 0)) + im;
  const int b_dim = im ? -1 : 1;          // the other component of the same column
  const unsigned b_mask = im ? 0u : 0x80000000u;

  double acc[kPi3NT][2];
#pragma unroll
  for (int u = 0; u < kPi3NT; ++u) acc[u][0] = acc[u][1] = 0.0;

  const int e_lo = ec * p.e_per_chunk, e_hi = min(p.ne, e_lo + p.e_per_chunk);
  const int ne_c = e_hi - e_lo;
  const int n_st = p.nkz * ne_c;
  const int n_ss = kPi3Sub * n_st;

  auto produce = [&](int t) {
    const int slot = t % kPi3Slots;
    if (!LAST_PRODUCES && t >= kPi3Slots) mbar_wait(empty + slot, (uint32_t)(((t - kPi3Slots) / kPi3Slots) & 1));
    const int st = t / kPi3Sub, j = t % kPi3Sub;
    const int k = st / ne_c, e = e_lo + st % ne_c;
    const int r0 = min(j * qs * 4, no2), r1 = min((j + 1) * qs * 4, no2);
    if (r1 <= r0) {  // empty sub-stage (few quads)
      mbar_arrive(full + slot);
      return;
    }
    const uint32_t bytes = (uint32_t)(r1 - r0) * ncol * 16;
    mbar_arrive_expect_tx(full + slot, bytes);
    bulk_g2s(ring + slot * slot_vec, VT + (((long long)k * p.ne + e) * no2 + r0) * ncol, bytes, full + slot);
  };
  // this lane's A row of stage (k, e) at kappa = pcol (zero row when invalid)
  auto row_of = [&](int k, int e) -> const double2* {
    int kp = k + q;
    if (kp >= p.nkz) kp -= p.nkz;
    if (!(row_ok && e + off < p.ne)) return kPiZeroRow + pcol;
    if (p.peer.ranks > 0)
      return peer_block(p.peer, pol, (long long)kp * p.ne + e + off, p.g_atom_of_chunk0 + la, no2) + pcol;
    return g_atom + (long long)kp * p.g_sk + (long long)(e + off) * p.g_se + pcol;
  };
  // ragged last quad (No^2 % 4 != 0): lanes past No^2 read zeros, because the
  // slot rows they meet may hold another sub-stage's (stale, finite) B
  const int kq_last = (no2 - 1 - pcol) / 4;
  const double2 *cur = nullptr, *nxt = nullptr;
  auto load_a = [&](int kq) -> double2 {  // quad kq of the current stage, or kq - khp of the next
    const double2* r = kq < khp ? cur : nxt;
    const int qq = kq < khp ? kq : kq - khp;
    return __ldg(qq <= kq_last ? r + qq * 4 : kPiZeroRow);
  };

  if (threadIdx.x == 0)
    for (int t = 0; t < (LAST_PRODUCES ? kPi3Slots : kPi3Slots - 1) && t < n_ss; ++t) produce(t);
  int k = 0, e = e_lo;
  int kn = 0, en = e_lo + 1;  // next stage
  if (en == e_hi) {
    en = e_lo;
    ++kn;
  }
  cur = row_of(k, e);
  nxt = n_st > 1 ? row_of(kn, en) : cur;
  double2 a0 = load_a(0), a1 = load_a(1);
  int kq = 0, j = 0, slot = 0;
  uint32_t phase = 0;
  for (int ss = 0; ss < n_ss; ++ss) {
    if (!LAST_PRODUCES) {
      const int t = ss + kPi3Slots - 1;
      if (lane == 0 && t < n_ss && t % NW == warp) produce(t);
    }
    __syncwarp();  // reconverge before the warp-wide mma.sync
    mbar_wait(full + slot, phase);
    const bool live = active && e + off_min < p.ne;  // warp-uniform
    const double* sb = reinterpret_cast<const double*>(ring + slot * slot_vec) + pcol * 2 * ncol + b_off;
    const int kq1 = min((j + 1) * qs, khp);
    // quads in pairs: a0 / a1 swap roles without register moves (a move would
    // wait for the prefetch to land); sub-stages hold an even number of quads
    // except the last one of an odd-khp stage
    auto quad = [&](const double2& a, const double* b) {
      double br[kPi3NT], bi[kPi3NT];
#pragma unroll
      for (int u = 0; u < kPi3NT; ++u) {
        br[u] = b[8 * u];
        bi[u] = xor_sign(b[8 * u + b_dim], b_mask);
      }
#pragma unroll
      for (int u = 0; u < kPi3NT; ++u) dmma884_nv(acc[u], a.x, br[u]);
#pragma unroll
      for (int u = 0; u < kPi3NT; ++u) dmma884_nv(acc[u], a.y, bi[u]);
    };
    if constexpr (UNIFORM) {
      if (live) {
#pragma unroll
        for (int pr = 0; pr < QS_T / 2; ++pr) {
          quad(a0, sb + 16 * pr * ncol);
          a0 = load_a(kq + 2 * pr + 2);
          quad(a1, sb + (16 * pr + 8) * ncol);
          a1 = load_a(kq + 2 * pr + 3);
        }
      } else {
#pragma unroll
        for (int pr = 0; pr < QS_T / 2; ++pr) {
          a0 = load_a(kq + 2 * pr + 2);
          a1 = load_a(kq + 2 * pr + 3);
        }
      }
      kq += QS_T;
    } else {
      for (; kq + 1 < kq1; kq += 2) {
        if (live) quad(a0, sb);
        a0 = load_a(kq + 2);
        if (live) quad(a1, sb + 8 * ncol);
        a1 = load_a(kq + 3);
        sb += 16 * ncol;
      }
    }
    if (!UNIFORM && kq < kq1) {  // odd tail
      if (live) quad(a0, sb);
      a0 = a1;
      a1 = load_a(kq + 2);
      ++kq;
    }
    __syncwarp();  // the warp is done with the slot before lane 0 releases it
    if (LAST_PRODUCES) {
      if (lane == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.inc.u32 %0, [%1], %2;"
                     : "=r"(old)
                     : "r"(smem_u32(rel + slot)), "r"((unsigned)(NW - 1))
                     : "memory");
        if (old == NW - 1 && ss + kPi3Slots < n_ss) {  // last release: refill the slot
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          produce(ss + kPi3Slots);
        }
      }
    } else if (lane == 0) {
      mbar_arrive(empty + slot);
    }
    if (++slot == kPi3Slots) {
      slot = 0;
      phase ^= 1u;
    }
    if (++j == kPi3Sub) {  // stage done: shift the stage window
      j = 0;
      kq -= khp;
      k = kn;
      e = en;
      cur = nxt;
      if (++en == e_hi) {
        en = e_lo;
        ++kn;
      }
      if (ss + 1 + kPi3Sub < n_ss) nxt = row_of(kn, en);
    }
  }

  if (!active) return;
  if (w >= p.nw) return;
  double2* part = p.partial + ((((long long)la * 2 + pol) * p.nqz + q) * p.echunks + ec) * p.nw * ncol;
#pragma unroll
  for (int u = 0; u < kPi3NT; ++u) {
    const int c = (ng * kPi3NT + u) * 4 + (lane & 3);
    if (c < ncol)
      part[(long long)w * ncol + c] = make_double2(p.energy_weight * acc[u][0], p.energy_weight * acc[u][1]);
  }
}

// --------------------------------------------------------------------------
// K6 v4 (fixed shapes No = 12, NB = 4): as v3 but each warp owns TWO 8-lag
// m-tiles (5 warps per CTA for 9 lag tiles), so every B value read from shared
// memory feeds two DMMAs (v3: one); the last warp of an odd tile count runs
// the one-tile path.  Same per-output accumulation order (bitwise equal).
// --------------------------------------------------------------------------
constexpr int kPi4Warps = 5;

// TAIL: the CTA is (atom, chain polarity, E-chunk) and warp w computes the LAST lag
// tile for momentum q = w (all Nqz warps share the V stages); the main launch then
// covers the first 2*NW tiles per q (paper: 8 + 1 lag tiles; 3 CTAs of 4 warps per SM).
template <int NOT, int NBT, int NW = kPi4Warps, int SL = kPi3Slots, int MINB = 3, bool TAIL_CTAS = false>
__global__ void __launch_bounds__(NW * 32, MINB)
pi_dmma4_kernel(PiArgs p, int chunk_atoms) {
  constexpr int NO2 = NOT * NOT, NCOL = 9 * NBT;
  constexpr int KHP = (NO2 + 3) / 4;
  constexpr int QS = 2 * ((KHP + 2 * kPi3Sub - 1) / (2 * kPi3Sub));
  static_assert(NO2 % 4 == 0 && KHP % QS == 0 && KHP / QS == kPi3Sub && 2 * NCOL <= 8 * kPi3NT,
                "fixed-shape K6 v4 needs whole quads, uniform sub-stages and <= 9 n-tiles");
  constexpr int SLOT = QS * 4 * NCOL;  // double2 per slot
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* ring = reinterpret_cast<double2*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + SL * SLOT + kPi2Pad);
  uint64_t* empty = full + SL;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int bx = blockIdx.x;
  // TAIL_CTAS: CTAs past the main grid (chunk x 2 x echunks x Nqz) are tail CTAs, one per
  // (atom, polarity, E-chunk); they run after the main CTAs in the same launch
  const int main_ctas = chunk_atoms * 2 * p.echunks * p.nqz;
  const bool TAIL = TAIL_CTAS && bx >= main_ctas;
  if (TAIL) bx -= main_ctas;
  const int qgroups = (p.nqz + NW - 1) / NW;  // tail CTAs: NW momenta each
  int q;
  if (TAIL) {
    q = (bx % qgroups) * NW + warp;
    bx /= qgroups;
  } else {
    q = bx % p.nqz;
    bx /= p.nqz;
  }
  // main CTAs of a short last E-chunk (paper: 706 = 7 x 96 + 34 energies) come last in the main
  // grid, so the launch's final wave is packed with short CTAs (each CTA owns its partial slot:
  // the order does not change any result)
  int ec;
  if (TAIL_CTAS && !TAIL && p.echunks > 1 && p.ne % p.e_per_chunk != 0) {
    const int full_part = chunk_atoms * 2 * (p.echunks - 1);
    if (bx < full_part) {
      ec = bx % (p.echunks - 1);
      bx /= p.echunks - 1;
    } else {
      bx -= full_part;
      ec = p.echunks - 1;
    }
  } else {
    ec = bx % p.echunks;
    bx /= p.echunks;
  }
  const int pol = bx % 2;
  const int la = bx / 2;
  const int m_tiles = (p.nw + 7) / 8;
  const int wg = blockIdx.y * NW + warp;
  const int mt0 = TAIL ? m_tiles - 1 : 2 * wg;
  const bool active = TAIL ? q < p.nqz : mt0 < m_tiles;
  const bool two = !TAIL && mt0 + 1 < m_tiles;  // warp-uniform
  const int pcol = lane & 3;

  for (int i = threadIdx.x; i < SL * SLOT + kPi2Pad; i += blockDim.x) ring[i] = make_double2(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < SL; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  const double2* __restrict__ G1 = pol ? p.G[1] : p.G[0];
  const double2* __restrict__ VT = (pol ? p.VT[1] : p.VT[0]) + (long long)la * p.nkz * p.ne * NO2 * NCOL;
  const double2* g_atom = G1 + (p.g_atom_of_chunk0 + la) * p.g_sa;

  int w[2], off[2];
  bool row_ok[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    w[t] = (mt0 + t) * 8 + (lane >> 2);
    row_ok[t] = active && w[t] < p.nw;
    off[t] = row_ok[t] ? __ldg(p.off + w[t]) : 0;
  }
  int off_min = row_ok[0] ? off[0] : (1 << 30);
  if (row_ok[1]) off_min = min(off_min, off[1]);
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) off_min = min(off_min, __shfl_xor_sync(0xffffffffu, off_min, sh));
  const int nc0 = lane >> 2;
  const int im = nc0 & 1;
  const int c1 = (nc0 >> 1) ^ (((pcol >> 1) & 1) ? 2 : 0);  // column of tile 0 after the kappa-bit-1 flip
  const int b_off = 2 * (p.swz ? c1 : (nc0 >> 1)) + im;
  // swizzle mode 3: quad kq (rows n = kq / 3) also XORs the column with (n & 3): offset in doubles
  auto n_delta = [&](int n) -> int { return p.swz == 3 ? 2 * ((c1 ^ (n & 3)) - c1) : 0; };
  const int b_dim = im ? -1 : 1;
  const unsigned b_mask = im ? 0u : 0x80000000u;

  double acc[2][kPi3NT][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;

  const int e_lo = ec * p.e_per_chunk, e_hi = min(p.ne, e_lo + p.e_per_chunk);
  const int ne_c = e_hi - e_lo;
  const int n_st = p.nkz * ne_c;
  const int n_ss = kPi3Sub * n_st;

  // producer: sub-stage t = (stage (kt, et), part jt) into slot t % SL
  auto produce = [&](int t, int kt, int et, int jt) {
    const int slot = t % SL;
    if (t >= SL) mbar_wait(empty + slot, (uint32_t)(((t - SL) / SL) & 1));
    constexpr uint32_t bytes = (uint32_t)SLOT * 16;
    mbar_arrive_expect_tx(full + slot, bytes);
    bulk_g2s(ring + slot * SLOT, VT + (((long long)kt * p.ne + et) * NO2 + jt * QS * 4) * NCOL, bytes, full + slot);
  };
  auto row_of = [&](int t, int k, int e) -> const double2* {
    int kp = k + q;
    if (kp >= p.nkz) kp -= p.nkz;
    if (!(row_ok[t] && e + off[t] < p.ne)) return kPiZeroRow + pcol;
    if (p.peer.ranks > 0)
      return peer_block(p.peer, pol, (long long)kp * p.ne + e + off[t], p.g_atom_of_chunk0 + la, NO2) + pcol;
    return g_atom + (long long)kp * p.g_sk + (long long)(e + off[t]) * p.g_se + pcol;
  };
  const double2 *cur[2] = {nullptr, nullptr}, *nxt[2] = {nullptr, nullptr};
  auto load_a = [&](int t, int kq) -> double2 {
    const double2* r = kq < KHP ? cur[t] : nxt[t];
    const int qq = kq < KHP ? kq : kq - KHP;
    return __ldg(r + qq * 4);
  };
  // stage / sub-stage counters advance incrementally (no divisions in the loop; round 1 derived
  // them from ss to save registers at 128, the 3-CTA build has room): (k, e) of a stage index
  auto next_stage = [&](int& k_, int& e_) {
    if (++e_ == e_hi) {
      e_ = e_lo;
      ++k_;
    }
  };
  // producer cursor: the next sub-stage to load, (kt, et, jt); thread 0 primes SL - 1 of them
  int tp = 0, kt = 0, et = e_lo, jt = 0;
  auto advance_t = [&]() {
    ++tp;
    if (++jt == kPi3Sub) {
      jt = 0;
      next_stage(kt, et);
    }
  };
  for (; tp < SL - 1 && tp < n_ss;) {
    if (threadIdx.x == 0) produce(tp, kt, et, jt);
    advance_t();
  }
  int k2 = 0, e2 = e_lo;  // stage st + 2 (the rows the next stage switch loads)
  {
    int k1 = 0, e1 = e_lo;
    if (n_st > 1) next_stage(k1, e1);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      cur[t] = row_of(t, 0, e_lo);
      nxt[t] = row_of(t, k1, e1);
    }
    k2 = k1;
    e2 = e1;
    next_stage(k2, e2);
  }
  double2 a0[2], a1[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    a0[t] = load_a(t, 0);
    a1[t] = load_a(t, 1);
  }
  // one quad: B read once per n-tile, used by both m-tiles
  auto quad2 = [&](const double2 (&a)[2], const double* b) {
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) {
      const double br = b[8 * u];
      dmma884_nv(acc[0][u], a[0].x, br);
      dmma884_nv(acc[1][u], a[1].x, br);
    }
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) {
      const double bi = xor_sign(b[8 * u + b_dim], b_mask);
      dmma884_nv(acc[0][u], a[0].y, bi);
      dmma884_nv(acc[1][u], a[1].y, bi);
    }
  };
  auto quad1 = [&](const double2 (&a)[2], const double* b) {
    double br[kPi3NT], bi[kPi3NT];
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) {
      br[u] = b[8 * u];
      bi[u] = xor_sign(b[8 * u + b_dim], b_mask);
    }
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) dmma884_nv(acc[0][u], a[0].x, br[u]);
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) dmma884_nv(acc[0][u], a[0].y, bi[u]);
  };
  // the stage loop, instantiated for two- and one-tile warps (warp-uniform; the branch
  // is outside the loop: 29.8 vs 28.2 TF/s on a 98-atom paper shard)
  auto run = [&](auto two_c) {
    constexpr bool TWO = decltype(two_c)::value;
    int j = 0, st = 0, e = e_lo, slot = 0;
    uint32_t phase = 0;
    for (int ss = 0; ss < n_ss; ++ss) {
      const int kq = j * QS;
      if (tp < n_ss) {  // the producer cursor runs SL - 1 sub-stages ahead
        if (lane == 0 && tp % NW == warp) produce(tp, kt, et, jt);
        advance_t();
      }
      __syncwarp();
      mbar_wait(full + slot, phase);
      const bool live = active && e + off_min < p.ne;
      const double* sb = reinterpret_cast<const double*>(ring + slot * SLOT) + pcol * 2 * NCOL + b_off;
      // the sub-stage's quads kq .. kq+5 span rows n = kq/3 (quads 0-2) and kq/3 + 1 (quads 3-5)
      static_assert(QS == 6, "mode-3 swizzle deltas assume 6 quads per sub-stage");
      const int dn0 = n_delta(2 * j), dn1 = n_delta(2 * j + 1);
      auto dq = [&](int qd) { return qd < 3 ? dn0 : dn1; };
      if (live && TWO) {
#pragma unroll
        for (int pr = 0; pr < QS / 2; ++pr) {
          quad2(a0, sb + 16 * pr * NCOL + dq(2 * pr));
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) a0[tt] = load_a(tt, kq + 2 * pr + 2);
          quad2(a1, sb + (16 * pr + 8) * NCOL + dq(2 * pr + 1));
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) a1[tt] = load_a(tt, kq + 2 * pr + 3);
        }
      } else if (live) {
#pragma unroll
        for (int pr = 0; pr < QS / 2; ++pr) {
          quad1(a0, sb + 16 * pr * NCOL + dq(2 * pr));
          a0[0] = load_a(0, kq + 2 * pr + 2);
          quad1(a1, sb + (16 * pr + 8) * NCOL + dq(2 * pr + 1));
          a1[0] = load_a(0, kq + 2 * pr + 3);
        }
      } else {
#pragma unroll
        for (int pr = 0; pr < QS / 2; ++pr) {
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            a0[tt] = load_a(tt, kq + 2 * pr + 2);
            a1[tt] = load_a(tt, kq + 2 * pr + 3);
          }
        }
      }
      __syncwarp();  // the warp is done with the slot before lane 0 releases it
      if (lane == 0) mbar_arrive(empty + slot);
      if (++slot == SL) {
        slot = 0;
        phase ^= 1u;
      }
      if (++j == kPi3Sub) {  // stage done: the next stage's rows become current
        j = 0;
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) cur[tt] = nxt[tt];
        if (st + 2 < n_st) {
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) nxt[tt] = row_of(tt, k2, e2);
        }
        ++st;
        if (++e == e_hi) e = e_lo;
        next_stage(k2, e2);
      }
    }
  };
  if (two) run(std::true_type{});
  else run(std::false_type{});

  if (!active) return;
  double2* part = p.partial + ((((long long)la * 2 + pol) * p.nqz + q) * p.echunks + ec) * p.nw * NCOL;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (!row_ok[t]) continue;
#pragma unroll
    for (int u = 0; u < kPi3NT; ++u) {
      const int c = u * 4 + (lane & 3);
      if (c < NCOL)
        part[(long long)w[t] * NCOL + c] =
            make_double2(p.energy_weight * acc[t][u][0], p.energy_weight * acc[t][u][1]);
    }
  }
}

// --------------------------------------------------------------------------
// K7: Pi assembly (sse.py:393-406): chain = sum of the E-chunk partials in
// order; Pi[q,w,a,1+s] = i chain_s, Pi[q,w,a,0] = -i sum_s chain_s.
// --------------------------------------------------------------------------
__global__ void pi_assemble_kernel(PiAssembleArgs p) {
  const long long total = (long long)p.chunk_atoms * 2 * p.nqz * p.nw * 9;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const int ij = (int)(x % 9);
    long long r = x / 9;
    const int w = (int)(r % p.nw);
    r /= p.nw;
    const int q = (int)(r % p.nqz);
    r /= p.nqz;
    const int pol = (int)(r % 2);
    const int la = (int)(r / 2);
    const double2* part = p.partial + (((long long)la * 2 + pol) * p.nqz + q) * p.echunks * p.nw * p.ncol;
    double2* out = p.Pi[pol] + (((long long)q * p.nw + w) * p.out_natoms + p.atom_begin + la) * (p.nb + 1) * 9;
    double sre = 0.0, sim = 0.0;
    for (int s = 0; s < p.nb; ++s) {
      const int c = s * 9 + ij;
      double cre = 0.0, cim = 0.0;
      for (int ec = 0; ec < p.echunks; ++ec) {
        const double2 v = part[((long long)ec * p.nw + w) * p.ncol + c];
        cre += v.x;
        cim += v.y;
      }
      out[(1 + s) * 9 + ij] = make_double2(-cim, cre);  // +i chain
      sre += cre;
      sim += cim;
    }
    out[ij] = make_double2(sim, -sre);  // -i sum_s chain
  }
}

// --------------------------------------------------------------------------
// K3g: generic Sigma with DFMA (any No).  One thread per output element
// (k, E, atom, m, n); compact operator M[q,w][p][n]; same (q, s, w) order.
// --------------------------------------------------------------------------
__global__ void sigma_generic_kernel(SigmaArgs p, int chunk_atoms) {
  const int no = p.no, no2 = no * no;
  const long long per_atom = (long long)p.nkz * p.ne * no2;
  const long long total = per_atom * chunk_atoms;
  const int pol = blockIdx.y;
  const double2* __restrict__ G = p.G[pol];
  const double2* __restrict__ M = p.M[pol];
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const int la = (int)(x / per_atom);
    long long r = x % per_atom;
    const int n = (int)(r % no);
    r /= no;
    const int m = (int)(r % no);
    r /= no;
    const int e = (int)(r % p.ne);
    const int k = (int)(r / p.ne);
    double re = 0.0, im = 0.0;
    for (int qi = 0; qi < p.nqz; ++qi) {
      int q, kp;
      q_order(k, qi, p.nkz, p.nqz, q, kp);
      for (int s = 0; s < p.nb; ++s) {
        const int lb = p.nbr[la * p.nb + s];
        const double2* mq = M + ((long long)((la * p.nb + s) * p.nqz + q) * p.nw) * no2;
        for (int w = 0; w < p.nw; ++w) {
          const int es = e - p.off[w];
          if (es < 0) continue;
          const double2* g = G + lb * p.g_sa + kp * p.g_sk + (long long)es * p.g_se + m * no;
          const double2* mm = mq + (long long)w * no2 + n;
          for (int t = 0; t < no; ++t) {
            const double2 u = g[t], v = mm[t * no];
            re = fma(u.x, v.x, re);
            re = fma(-u.y, v.y, re);
            im = fma(u.x, v.y, im);
            im = fma(u.y, v.x, im);
          }
        }
      }
    }
    double2* dst = sigma_block(p, pol, la, k, e) + m * no + n;
    *dst = make_double2(-im, re);
  }
}

// --------------------------------------------------------------------------
// preprocess_D (sse.py:105-113), same term order as the reference:
//   Dc = D[b, 1+rev] - D[b, 0] - D[a, 0] + D[a, 1+s]
// --------------------------------------------------------------------------
__global__ void preprocess_D_kernel(long long nqw, long long d_natoms, long long d_atom0,
                                    long long out_atom0, long long out_natoms, long long nb,
                                    const int* __restrict__ nbr, const int* __restrict__ rev,
                                    const double2* __restrict__ D, double2* __restrict__ Dc) {
  const long long total = nqw * out_natoms * nb * 9;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const int ij = (int)(x % 9);
    long long r = x / 9;
    const long long s = r % nb;
    r /= nb;
    const long long la = r % out_natoms;
    const long long qw = r / out_natoms;
    const long long a = out_atom0 + la - d_atom0;  // D-slab index of a
    const long long b = nbr[la * nb + s];          // D-slab index of f(a, s)
    const long long rv = rev[la * nb + s];
    const double2* base = D + qw * d_natoms * (nb + 1) * 9;
    const double2 d_ba = base[(b * (nb + 1) + 1 + rv) * 9 + ij];
    const double2 d_bb = base[(b * (nb + 1)) * 9 + ij];
    const double2 d_aa = base[(a * (nb + 1)) * 9 + ij];
    const double2 d_ab = base[(a * (nb + 1) + 1 + s) * 9 + ij];
    const double re = __dadd_rn(__dsub_rn(__dsub_rn(d_ba.x, d_bb.x), d_aa.x), d_ab.x);
    const double im = __dadd_rn(__dsub_rn(__dsub_rn(d_ba.y, d_bb.y), d_aa.y), d_ab.y);
    Dc[x] = make_double2(re, im);
  }
}

// --------------------------------------------------------------------------
// Atom-keyed synthetic inputs: splitmix64 counter hash -> Irwin-Hall(4) of
// 16-bit digits, unit variance.  Integer sums are exact and there is a single
// rounding per product, so inputs.atom_keyed (numpy) reproduces it bit-exactly.
// --------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double irwin_hall4(uint64_t h, double scale) {
  const long long s = (long long)(h & 0xFFFF) + (long long)((h >> 16) & 0xFFFF) +
                      (long long)((h >> 32) & 0xFFFF) + (long long)(h >> 48);
  const double x = __dmul_rn((double)(s - 131070), 0x1.bb67ae86627e7p-16);
  return __dmul_rn(x, scale);
}

__global__ void fill_synthetic_kernel(uint64_t seed, uint32_t tensor_id, long long atom0,
                                      long long natoms, long long outer, long long inner,
                                      long long atom_stride, long long outer_stride, double scale,
                                      double2* __restrict__ dst) {
  const long long per_atom = outer * inner;
  const long long total = per_atom * natoms;
  const uint64_t k0 = splitmix64(splitmix64(seed) ^ (uint64_t)tensor_id);
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
       x += (long long)gridDim.x * blockDim.x) {
    const long long la = x / per_atom;
    const long long local = x % per_atom;
    const long long o = local / inner, i = local % inner;
    const uint64_t key = splitmix64(k0 ^ (uint64_t)(atom0 + la));
    const double re = irwin_hall4(splitmix64(key ^ (uint64_t)(2 * local)), scale);
    const double im = irwin_hall4(splitmix64(key ^ (uint64_t)(2 * local + 1)), scale);
    dst[la * atom_stride + o * outer_stride + i] = make_double2(re, im);
  }
}

// --------------------------------------------------------------------------
// launchers
// --------------------------------------------------------------------------
static int grid_for(long long work, int threads) {
  long long g = (work + threads - 1) / threads;
  const long long cap = 148LL * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_layout_transform(long long nkz, long long ne, long long na, long long blk_vec,
                                    int to_atom_major, const double2* src, double2* dst,
                                    cudaStream_t st) {
  const long long warps = nkz * ne * na;
  note_kernel(2, "layout_transform_kernel");
  layout_transform_kernel<<<grid_for(warps * 32, 256), 256, 0, st>>>(nkz, ne, na, blk_vec,
                                                                     to_atom_major, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_build_operator(const OperatorArgs& a, cudaStream_t st) {
  if (a.comb_kg > 0 && a.nqz > kOpBlocks) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(12 + (a.fragment_order ? kOpBlocks : 0)) * a.no * a.no * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(build_operator_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  note_kernel(0, "build_operator_kernel");
  build_operator_kernel<<<a.chunk_atoms * a.nb, 256, smem, st>>>(a);
  return cudaGetLastError();
}

// Sigma kernel selection (env SSE_SIGMA_KERNEL, read per launch):
//   4 = multi-momentum sliding window (default when the offsets slide, i.e. are
//       non-decreasing with steps <= 1 as default_grid's are, and Nw >= 6),
//   3 = single-momentum sliding window (Nw >= 12),
//   1 = register-pipelined (used otherwise), 0 = simple.
// All accumulate every output in the same (q_order, s, w, k-step) order, so they
// agree bitwise (tested).
static int sigma_kernel_choice() {
  const char* env = getenv("SSE_SIGMA_KERNEL");
  return env ? atoi(env) : 4;
}

template <int NO, int KG, bool COMB = false, int NW = 12, int MT = 3>
static cudaError_t launch_kslide(SigmaArgs a, int chunk_atoms, int k_first, int groups, cudaStream_t st) {
  using SG = KSlideGeom<NO, NW, MT, KG, COMB>;
  a.ctas_per_ak = (a.rows + SG::kRows - 1) / SG::kRows;
  a.k_first = k_first;
  a.kgroups = groups;
  const dim3 grid((unsigned)((long long)a.ctas_per_ak * groups * chunk_atoms), a.npol);
  cudaError_t e = cudaFuncSetAttribute(sigma_dmma_kslide_kernel<NO, NW, MT, KG, COMB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SG::kSmem);
  if (e != cudaSuccess) return e;
  sigma_dmma_kslide_kernel<NO, NW, MT, KG, COMB><<<grid, NW * 32, SG::kSmem, st>>>(a);
  return cudaGetLastError();
}

bool sigma_uses_combined(int no, int nw, int off_slide) {
  if (no % 4 != 2 || no > kMaxDmmaOrb || !off_slide || nw < kKStages || nw > kMaxSlideNw) return false;
  if (sigma_kernel_choice() != 4) return false;
  const char* env = getenv("SSE_K3M_COMB");  // 0: per-momentum fragment vectors side by side
  if (env && env[0] == '0') return false;
  switch (no) {
    case 2: return KSlideGeom<2, 12, 3, kCombKG, true>::kFits;
    case 6: return KSlideGeom<6, 12, 3, kCombKG, true>::kFits;
    case 10: return KSlideGeom<10, 12, 3, kCombKG, true>::kFits;
    case 14: return KSlideGeom<14, 12, 3, kCombKG, true>::kFits;
    default: return false;
  }
}

template <int NO>
static cudaError_t launch_dmma(const SigmaArgs& a0, int chunk_atoms, cudaStream_t st) {
  SigmaArgs a = a0;
  const int choice = sigma_kernel_choice();
  auto grid_for_rows = [&](int rows_per_cta) {
    a.ctas_per_ak = (a.rows + rows_per_cta - 1) / rows_per_cta;
    return dim3((unsigned)((long long)a.ctas_per_ak * a.nkz * chunk_atoms), a.npol);
  };
  const bool slides = a.off_slide && a.nw <= kMaxSlideNw;
  const bool kslide_ok = slides && a.nw >= kKStages && a.zeroM && KSlideGeom<NO, 12, 3, 3>::kFits;
  const bool slide_ok = slides && a.nw >= kSlideStages && SlideGeom<NO, 12, 3>::kFits;
  if (a.gather_ranks > 0 && !kslide_ok && !slide_ok) return cudaErrorNotSupported;  // peer gather: sliding K3 only
  if (a.comb_kg > 0) {  // K2 wrote combined fragments (sigma_uses_combined)
    if constexpr (NO % 4 == 2) {
      if (!KSlideGeom<NO, 12, 3, kCombKG, true>::kFits || a.comb_kg != kCombKG) return cudaErrorInvalidValue;
      note_kernel(1, "sigma_dmma_kslide_kernel<%d,12,3,%d,comb>", NO, kCombKG);
      return launch_kslide<NO, kCombKG, true>(a, chunk_atoms, 0, (a.nkz + kCombKG - 1) / kCombKG, st);
    }
    return cudaErrorInvalidValue;
  }
  if ((choice == 4 || (a.gather_ranks > 0 && !slide_ok)) && kslide_ok) {
    // momentum groups of kg, then one group of the remainder (no idle accumulators).  kg = 2 for
    // No > 10: at 3 the 3 x 9 x 2 accumulator doubles of No = 12 exceed the 168-register budget of
    // 12 warps (spills; paper shard 34.75 vs 35.12 TF/s at 2, 34.56 at 1); SSE_K3M_KG overrides
    const char* kg_env = getenv("SSE_K3M_KG");
    const int kg = kg_env && atoi(kg_env) >= 1 && atoi(kg_env) <= 3 ? atoi(kg_env) : (NO >= 9 ? 2 : 3);
    const int full = a.nkz / kg, rest = a.nkz % kg;
    cudaError_t e = cudaSuccess;
    // No = 12, odd Nkz >= 3: momentum groups of 2, closed by ONE group of 3 at 2 row tiles per warp
    // (164 registers, no spills) instead of a 1-momentum remainder launch: paper (Nkz = 3, one
    // KG = 3 launch) 35.16 -> 35.46 TF/s, large (2 + 3) 35.73 -> 35.80; kheavy 2+2+2+1 vs 3+3+1:
    // 35.43 vs 35.26, so at most one such group (`profiles/r02_ab_k3m_mt2*.log`); SSE_K3M_MT=3 or
    // SSE_K3M_KG restore the plain groups of kg
    if constexpr (NO == 12) {  // (compile-time: the No = 12 variants are instantiated only for 12)
      const char* mt_env = getenv("SSE_K3M_MT");
      if (!kg_env && !(mt_env && atoi(mt_env) == 3) && a.nkz >= 3 && (a.nkz & 1)) {
        const int pairs = (a.nkz - 3) / 2;
        if (pairs > 0) e = launch_kslide<NO, 2>(a, chunk_atoms, 0, pairs, st);
        if (e == cudaSuccess) e = launch_kslide<NO, 3, false, 12, 2>(a, chunk_atoms, 2 * pairs, 1, st);
        if (pairs > 0)
          note_kernel(1, "sigma_dmma_kslide_kernel<%d,12,3,2> (x%d momentum groups) + <%d,12,2,3>", NO, pairs, NO);
        else
          note_kernel(1, "sigma_dmma_kslide_kernel<%d,12,2,3>", NO);
        return e;
      }
      const char* nw_env = getenv("SSE_K3M_NW");  // experiment: 8 warps (2 per SMSP, <= 255 registers)
      if (nw_env && atoi(nw_env) == 8 && kg == 3 && full > 0) {
        e = launch_kslide<NO, 3, false, 8>(a, chunk_atoms, 0, full, st);
        if (e == cudaSuccess && rest == 2) e = launch_kslide<NO, 2, false, 8>(a, chunk_atoms, 3 * full, 1, st);
        if (e == cudaSuccess && rest == 1) e = launch_kslide<NO, 1, false, 8>(a, chunk_atoms, 3 * full, 1, st);
        note_kernel(1, "sigma_dmma_kslide_kernel<%d,8,3,3>", NO);
        return e;
      }
    }
    if (full > 0) {
      if (kg == 3) e = launch_kslide<NO, 3>(a, chunk_atoms, 0, full, st);
      else if (kg == 2) e = launch_kslide<NO, 2>(a, chunk_atoms, 0, full, st);
      else e = launch_kslide<NO, 1>(a, chunk_atoms, 0, full, st);
    }
    if (e == cudaSuccess && rest == 2) e = launch_kslide<NO, 2>(a, chunk_atoms, kg * full, 1, st);
    if (e == cudaSuccess && rest == 1) e = launch_kslide<NO, 1>(a, chunk_atoms, kg * full, 1, st);
    if (full > 0 && rest > 0)
      note_kernel(1, "sigma_dmma_kslide_kernel<%d,12,3,%d> (x%d momentum groups) + <%d,12,3,%d>", NO, kg, full, NO,
                  rest);
    else
      note_kernel(1, "sigma_dmma_kslide_kernel<%d,12,3,%d>", NO, full > 0 ? kg : rest);
    return e;
  }
  if (choice == 0 && a.gather_ranks == 0) {
    const dim3 grid = grid_for_rows(kRowsPerCta);
    note_kernel(1, "sigma_dmma_kernel<%d>", NO);
    sigma_dmma_kernel<NO><<<grid, kSigmaWarps * 32, 0, st>>>(a);
  } else if ((choice >= 3 || a.gather_ranks > 0) && slide_ok) {
    // nw >= kSlideStages: the kSlideStages stages in flight span at most one
    // (q, s) segment boundary, so at most 2 * kTE + kSlideStages FIFO blocks
    // are live (SlideGeom::kNeed <= kRing)
    const dim3 grid = grid_for_rows(SlideGeom<NO, 12, 3>::kRows);
    const size_t smem = SlideGeom<NO, 12, 3>::kSmem;
    cudaFuncSetAttribute(sigma_dmma_slide_kernel<NO, 12, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    note_kernel(1, "sigma_dmma_slide_kernel<%d,12,3>", NO);
    sigma_dmma_slide_kernel<NO, 12, 3><<<grid, 12 * 32, smem, st>>>(a);
  } else {
    const dim3 grid = grid_for_rows(kRowsPerCta);
    note_kernel(1, "sigma_dmma_pipe_kernel<%d>", NO);
    sigma_dmma_pipe_kernel<NO><<<grid, kSigmaWarps * 32, 0, st>>>(a);
  }
  return cudaSuccess;
}

cudaError_t launch_sigma(const SigmaArgs& a0, int chunk_atoms, cudaStream_t st) {
  SigmaArgs a = a0;
  if (a.no <= kMaxDmmaOrb) {
    switch (a.no) {
      case 1: { const cudaError_t e = launch_dmma<1>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 2: { const cudaError_t e = launch_dmma<2>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 3: { const cudaError_t e = launch_dmma<3>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 4: { const cudaError_t e = launch_dmma<4>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 5: { const cudaError_t e = launch_dmma<5>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 6: { const cudaError_t e = launch_dmma<6>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 7: { const cudaError_t e = launch_dmma<7>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 8: { const cudaError_t e = launch_dmma<8>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 9: { const cudaError_t e = launch_dmma<9>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 10: { const cudaError_t e = launch_dmma<10>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 11: { const cudaError_t e = launch_dmma<11>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 12: { const cudaError_t e = launch_dmma<12>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 13: { const cudaError_t e = launch_dmma<13>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 14: { const cudaError_t e = launch_dmma<14>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 15: { const cudaError_t e = launch_dmma<15>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      case 16: { const cudaError_t e = launch_dmma<16>(a, chunk_atoms, st); if (e != cudaSuccess) return e; break; }
      default: return cudaErrorInvalidValue;
    }
  } else {
    if (a.gather_ranks > 0) return cudaErrorNotSupported;
    const long long total = (long long)a.nkz * a.ne * a.no * a.no * chunk_atoms;
    dim3 grid(grid_for(total, 256), a.npol);
    note_kernel(1, "sigma_generic_kernel");
    sigma_generic_kernel<<<grid, 256, 0, st>>>(a, chunk_atoms);
  }
  return cudaGetLastError();
}

template <int NO>
static cudaError_t launch_pi_build_dmma(const PiBuildArgs& a, cudaStream_t st) {
  // W n-tile group size (SSE_PI_WG, experiments): 3 default, 1, or NT2 (one group, round-1 order)
  const char* env = getenv("SSE_PI_WG");
  const int wg = env ? atoi(env) : 3;
  auto kern = wg == 1 ? pi_build_dmma_kernel<NO, 1> : (wg == 9 ? pi_build_dmma_kernel<NO, 9> : pi_build_dmma_kernel<NO, 3>);
  const size_t smem = ((size_t)2 * NO * NO * a.nb * 9 + (size_t)a.nb * 5 * NO * (NO + 1)) * 16;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long blocks = (long long)a.chunk_atoms * a.nkz * ((a.ne + kPB2Energies - 1) / kPB2Energies);
  note_kernel(4, "pi_build_dmma_kernel<%d>", NO);
  kern<<<(unsigned)blocks, kPB2Warps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

// K5 selection: the DMMA build for No in {4, 8, 12, 16} when its shared memory
// fits (V image x2 + dH + G2), else (or with SSE_PI_BUILD=0) the DFMA build
static bool pi_build_dmma_ok(const PiBuildArgs& a) {
  const char* env = getenv("SSE_PI_BUILD");
  if (env && env[0] == '0') return false;
  if (!(a.no % 4 == 0 || a.no == 10) || a.no > 16) return false;  // 10: the small config (padded K / N)
  const size_t smem = ((size_t)2 * a.no * a.no * a.nb * 9 + (size_t)a.nb * 5 * a.no * (a.no + 1)) * 16;
  return smem <= 220 * 1024;
}

cudaError_t launch_pi_build(const PiBuildArgs& a, cudaStream_t st) {
  if (a.no > kPiMaxNo) return cudaErrorInvalidValue;
  if (a.peer.ranks > 0 && !pi_build_dmma_ok(a)) return cudaErrorNotSupported;  // peer gather: DMMA build only
  if (pi_build_dmma_ok(a)) {
    switch (a.no) {
      case 4: return launch_pi_build_dmma<4>(a, st);
      case 8: return launch_pi_build_dmma<8>(a, st);
      case 10: return launch_pi_build_dmma<10>(a, st);
      case 12: return launch_pi_build_dmma<12>(a, st);
      case 16: return launch_pi_build_dmma<16>(a, st);
      default: break;
    }
  }
  const int tpe = a.nb * 3 * a.no;
  const int epg = tpe >= kPiBuildThreads ? 1 : kPiBuildThreads / tpe;
  const size_t smem = (size_t)(3 + epg) * a.nb * a.no * a.no * sizeof(double2);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pi_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long blocks = (long long)a.chunk_atoms * a.nkz * ((a.ne + kPiBuildEnergies - 1) / kPiBuildEnergies);
  note_kernel(4, "pi_build_kernel");
  pi_build_kernel<<<(unsigned)blocks, kPiBuildThreads, smem, st>>>(a);
  return cudaGetLastError();
}

// K6 selection (env SSE_PI_KERNEL, read per call): 3 = one m-tile per warp,
// quarter-stage ring (default); 2 = 3x3 tiles per warp, half stages; 1 = two
// momenta per CTA, whole stages; 0 = direct (no TMA).  A variant whose ring
// does not fit in shared memory (or v3 with fewer than 2 kappa quads) falls
// back to the next one.  All accumulate in the same order (bitwise equal).
static size_t pi_smem(int v, int no, int ncol) {
  const int khp = (no * no + 3) / 4;
  if (v >= 4) v = 3;  // same ring as v3
  if (v == 3)
    return ((size_t)kPi3Slots * 2 * ((khp + 2 * kPi3Sub - 1) / (2 * kPi3Sub)) * 4 * ncol + kPi2Pad) * 16 +
           2 * kPi3Slots * 8 + kPi3Slots * 4;
  if (v == 2) return ((size_t)kPi2Slots * ((khp + 1) / 2) * 4 * ncol + kPi2Pad) * 16 + 2 * kPi2Slots * 8;
  if (v == 1) return (size_t)kPiStages * no * no * ncol * 16 + 2 * kPiStages * 8;
  return 0;
}
static int pi_kernel_choice(int no, int ncol) {
  const char* env = getenv("SSE_PI_KERNEL");
  int v = (env && env[0] >= '0' && env[0] <= '4') ? env[0] - '0' : 4;
  if (v == 4 && !(no == 12 && ncol == 36)) v = 3;  // v4 exists for the paper shapes only
  if (v == 3 && (no * no + 3) / 4 < 2) v = 2;
  while (v > 0 && pi_smem(v, no, ncol) > 220 * 1024) --v;
  return v;
}
// column swizzle of V rows for K6 v3 (conflict-free B reads): column c of
// kappa row r is stored at c ^ (2 * ((r >> 1) & 1)); needs ncol % 4 == 0
int pi_vt_swizzle(int no, int ncol) {
  const int v = pi_kernel_choice(no, ncol);
  if (ncol % 4 || v < 3) return 0;
  return v >= 4 ? 3 : 2;  // v4 (paper shapes): the mode-3 swizzle; v3: mode 2
}

cudaError_t launch_pi(const PiArgs& a, int chunk_atoms, cudaStream_t st) {
  const int v = pi_kernel_choice(a.no, a.ncol);
  if (a.peer.ranks > 0 && v < 3) return cudaErrorNotSupported;  // peer gather: K6 v3 / v4 only
  if (a.swz != (a.ncol % 4 || v < 3 ? 0 : (v >= 4 ? 3 : 2))) return cudaErrorInvalidValue;  // K5 / K6 disagree
  const size_t smem = pi_smem(v, a.no, a.ncol);
  const unsigned gy = (unsigned)((a.warp_groups + kPiWarps - 1) / kPiWarps);
  const unsigned gx = (unsigned)((long long)chunk_atoms * 2 * a.echunks * a.nqz);
  cudaError_t e = cudaSuccess;
  switch (v) {
    case 4: {
      e = cudaFuncSetAttribute(pi_dmma4_kernel<12, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(pi_dmma4_kernel<12, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      const int pairs = ((a.nw + 7) / 8 + 1) / 2;
      const char* w4 = getenv("SSE_PI_V4_WARPS");
      const int m_tiles = (a.nw + 7) / 8;
      const bool split = !(w4 && w4[0] == '5') && m_tiles == 9;
      if (split || (w4 && w4[0] == '4')) {
        // 4 warps x 2 lag tiles per CTA (3 CTAs, 12 warps per SM by default) for tiles 0..7,
        // then (split) the 9th tile of every q in one tail CTA per (atom, polarity, E-chunk)
        auto kern = pi_dmma4_kernel<12, 4, 4, 3, 4>;
        const size_t slot = (size_t)2 * ((((a.no * a.no + 3) / 4) + 2 * kPi3Sub - 1) / (2 * kPi3Sub)) * 4 * a.ncol * 16;
        const size_t smem4 = smem - (size_t)(kPi3Slots - 3) * slot;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem4);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        if (split) {  // main and tail CTAs in one launch (the tail CTAs fill the last wave)
          // 4-slot V ring (55 KB per CTA; +0.4 % over 3 slots, `profiles/r02_ab_k6_slots.log`) at 3
          // CTAs per SM with 162 registers and no spills: +1.2 % over 4 CTAs at 128 registers, whose
          // spill reloads missed L1 and stalled the loop control (`profiles/r02_ab_k6_minb.log`,
          // `r02_ncu_k6_stalls_minb{4,3}.txt`); SSE_PI_V4_MINB=4 selects the 4-CTA build
          const char* mb_env = getenv("SSE_PI_V4_MINB");
          const bool minb4 = mb_env && mb_env[0] == '4';
          auto both = minb4 ? pi_dmma4_kernel<12, 4, 4, 4, 4, true> : pi_dmma4_kernel<12, 4, 4, 4, 3, true>;
          e = cudaFuncSetAttribute(both, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          if (e == cudaSuccess) e = cudaFuncSetAttribute(both, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          if (e != cudaSuccess) return e;
          const long long tails = (long long)chunk_atoms * 2 * a.echunks * ((a.nqz + 3) / 4);
          note_kernel(5, minb4 ? "pi_dmma4_kernel<12,4,4,4,4,true>" : "pi_dmma4_kernel<12,4,4,4,3,true>");
          both<<<dim3(gx + (unsigned)tails, 1u), 4 * 32, smem, st>>>(a, chunk_atoms);
        } else {
          note_kernel(5, "pi_dmma4_kernel<12,4,4,3,4>");
          kern<<<dim3(gx, (unsigned)((pairs + 3) / 4)), 4 * 32, smem4, st>>>(a, chunk_atoms);
        }
        break;
      }
      note_kernel(5, "pi_dmma4_kernel<12,4>");
      pi_dmma4_kernel<12, 4><<<dim3(gx, (unsigned)((pairs + kPi4Warps - 1) / kPi4Warps)), kPi4Warps * 32, smem, st>>>(
          a, chunk_atoms);
      break;
    }
    case 3: {
      const char* pe = getenv("SSE_PI_PRODUCER");  // 1: the last releaser refills (default: round robin)
      const bool last = pe && pe[0] == '1';
      const bool fixed = a.no == 12 && a.nb == 4;    // the paper shapes: unrolled sub-stages
      auto kern = fixed ? (last ? pi_dmma3_kernel<true, 12, 4> : pi_dmma3_kernel<false, 12, 4>)
                        : (last ? pi_dmma3_kernel<true, 0, 0> : pi_dmma3_kernel<false, 0, 0>);
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess)  // several CTAs per SM need the full shared-memory carveout
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      const int groups = ((a.nw + 7) / 8) * (((2 * a.ncol + 7) / 8 + kPi3NT - 1) / kPi3NT);
      PiArgs b = a;
      // few lag tiles (e.g. the small config: 2) -> one CTA serves every q: 6 of 9 warps busy, not 2
      b.q_in_warps = a.peer.ranks == 0 && groups * a.nqz <= kPiWarps;
      // q in warps with at most 6 busy warps (the small config: 3 q x 2 lag tiles): a 6-warp CTA at
      // 3 CTAs per SM (96 registers, no spills) instead of 9 warps at 72 registers with 3 idle and
      // spilling: 28.0 -> 21.2 ms per 256-atom small chunk (`profiles/r02_ab_k6_small.log`);
      // SSE_PI_QW=9 keeps the 9-warp CTA
      const char* qw_env = getenv("SSE_PI_QW");
      if (b.q_in_warps && !fixed && !last && groups * a.nqz <= 6 && !(qw_env && qw_env[0] == '9')) {
        auto k6 = pi_dmma3_kernel<false, 0, 0, 6, 3>;
        e = cudaFuncSetAttribute(k6, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k6, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        note_kernel(5, "pi_dmma3_kernel<0,0,0,6,3> (q in warps)");
        k6<<<dim3(gx / (unsigned)a.nqz, 1u), 6 * 32, smem, st>>>(b, chunk_atoms);
        break;
      }
      note_kernel(5, fixed ? "pi_dmma3_kernel<%d,12,4>%s" : "pi_dmma3_kernel<%d,0,0>%s", (int)last,
                  b.q_in_warps ? " (q in warps)" : "");
      if (b.q_in_warps)
        kern<<<dim3(gx / (unsigned)a.nqz, 1u), kPiWarps * 32, smem, st>>>(b, chunk_atoms);
      else
        kern<<<dim3(gx, (unsigned)((groups + kPiWarps - 1) / kPiWarps)), kPiWarps * 32, smem, st>>>(b, chunk_atoms);
      break;
    }
    case 2:
      e = cudaFuncSetAttribute(pi_dmma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(pi_dmma2_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      note_kernel(5, "pi_dmma2_kernel");
      pi_dmma2_kernel<<<dim3(gx, gy), kPiWarps * 32, smem, st>>>(a, chunk_atoms);
      break;
    case 1: {
      e = cudaFuncSetAttribute(pi_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      const int qblocks = (a.nqz + kPiQB - 1) / kPiQB;
      dim3 grid((unsigned)((long long)chunk_atoms * 2 * qblocks * a.echunks), gy);
      note_kernel(5, "pi_dmma_kernel");
      pi_dmma_kernel<<<grid, kPiWarps * 32, smem, st>>>(a, chunk_atoms);
      break;
    }
    default:
      note_kernel(5, "pi_dmma_direct_kernel");
      pi_dmma_direct_kernel<<<dim3(gx, gy), kPiWarps * 32, 0, st>>>(a, chunk_atoms);
  }
  return cudaGetLastError();
}

cudaError_t launch_pi_assemble(const PiAssembleArgs& a, cudaStream_t st) {
  const long long total = (long long)a.chunk_atoms * 2 * a.nqz * a.nw * 9;
  note_kernel(6, "pi_assemble_kernel");
  pi_assemble_kernel<<<grid_for(total, 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_preprocess_D(long long nqz, long long nw, long long d_natoms, long long d_atom0,
                                long long out_atom0, long long out_natoms, long long nb,
                                const int* nbr, const int* rev, const double2* D, double2* Dc,
                                cudaStream_t st) {
  const long long total = nqz * nw * out_natoms * nb * 9;
  note_kernel(3, "preprocess_D_kernel");
  preprocess_D_kernel<<<grid_for(total, 256), 256, 0, st>>>(nqz * nw, d_natoms, d_atom0, out_atom0,
                                                            out_natoms, nb, nbr, rev, D, Dc);
  return cudaGetLastError();
}

cudaError_t launch_fill_synthetic(uint64_t seed, uint32_t tensor_id, long long atom0,
                                  long long natoms, long long outer, long long inner,
                                  long long atom_stride, long long outer_stride, double scale,
                                  double2* dst, cudaStream_t st) {
  const long long total = natoms * outer * inner;
  fill_synthetic_kernel<<<grid_for(total, 256), 256, 0, st>>>(
      seed, tensor_id, atom0, natoms, outer, inner, atom_stride, outer_stride, scale, dst);
  return cudaGetLastError();
}

cudaError_t launch_slab_pull(const SlabPullArgs& a, long long npts, cudaStream_t st) {
  const long long run = a.natoms * a.no2;
  if (npts <= 0 || run <= 0) return cudaSuccess;
  if (npts > 65535 || run >= (1ll << 32) || a.ranks < 1 || a.ranks > kMaxScatter)
    return cudaErrorInvalidValue;
  const dim3 grid((unsigned)((run + 256 * kPullUnroll - 1) / (256 * kPullUnroll)), (unsigned)npts);
  slab_pull_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sse
