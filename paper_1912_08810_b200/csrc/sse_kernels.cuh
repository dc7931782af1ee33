// Kernel declarations and launch helpers for libsse (sm_100a).
// See DESIGN.md for the data layout and the roofline of each kernel.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sse {

// Largest orbital count served by the DMMA (tensor-core FP64) Sigma kernel.
// Larger blocks use the DFMA fallback kernel.
constexpr int kMaxDmmaOrb = 16;

// Sigma kernel CTA shape: 8 warps, each owning kRowTiles 8-row tiles of the
// per-(atom, k) output matrix [NE*No rows, No cols].
constexpr int kSigmaWarps = 8;
constexpr int kRowTiles = 3;
constexpr int kRowsPerCta = kSigmaWarps * kRowTiles * 8;

// Fragment geometry of the real embedding of an No x No complex block
// product for mma.sync.m8n8k4.f64 (DMMA.8x8x4).  C' columns interleave
// (Re, Im) of each output column n; N' = 2*No padded to 8*nt.
//  * split K (No % 4 != 2; NOP = No rounded up to 4):
//      A' = [Re G | Im G]       rows x 2*NOP  (K' order: real half, then imag)
//      B' = [[Re M, Im M] interleaved per column; [-Im M, Re M]]   2*NOP x N'
//  * interleaved K (il: No % 4 == 2, e.g. No = 10): K' = 2*No exactly, no padding:
//      A' row = the (re, im) doubles of the G row in memory order
//      B' row 2p = (Re M_pn, Im M_pn) per column pair, row 2p+1 = (-Im M_pn, Re M_pn)
// kh: 16-byte A registers per tile and stage (split: Re/Im of k-steps kk, kk+kh;
// il: k-steps 2j, 2j+1); fv: B-fragment pairs per stage (fr rounded up to even).
struct FragGeom {
  int no, nop, ksteps, kh, nt, fr, fv, il;
};
__host__ __device__ constexpr FragGeom frag_geom(int no) {
  return no % 4 == 2
             ? FragGeom{no, no, no / 2, (no / 2 + 1) / 2, (2 * no + 7) / 8, (no / 2) * ((2 * no + 7) / 8),
                        ((no / 2) * ((2 * no + 7) / 8) + 1) / 2, 1}
             : FragGeom{no, (no + 3) / 4 * 4, ((no + 3) / 4 * 4) / 2, ((no + 3) / 4 * 4) / 4,
                        (2 * no + 7) / 8, (((no + 3) / 4 * 4) / 2) * ((2 * no + 7) / 8),
                        (((no + 3) / 4 * 4) / 2) * ((2 * no + 7) / 8) / 2, 0};
}

struct OperatorArgs {
  const double2* Dc[2];   // [Nqz][Nw][dc_natoms][NB][3][3] (slab), per polarity
  const double2* dH;      // [dh_natoms][NB][3][No][No]
  const double* wt;       // [Nw] device
  double2* M[2];          // output: fragment order or compact, per polarity
  int nqz, nw, nb, no;
  int dc_natoms;          // atoms in the Dc slab (its atom stride)
  int atom_begin;         // first slab atom of this chunk
  int chunk_atoms;
  int fragment_order;     // 1: DMMA fragment order, 0: compact [p][n]
  int npol;               // polarities to process (1 or 2)
  // combined multi-momentum fragments (comb_kg > 0, see comb_geom): per (atom, s, kp, group,
  // w) ONE fragment vector holding M[q_k = (k - kp) mod Nkz] of the group's comb_kg output
  // momenta side by side in N (zero where q_k >= Nqz or k >= Nkz)
  int comb_kg, nkz;
};

// Combined-fragment geometry of the multi-momentum K3 (No % 4 == 2, e.g. No = 10): N' =
// kg * 2No padded to 8 * ntc (10: 60 -> 64 instead of 3 x 24 = 72), fvc double2 per lane.
struct CombGeom {
  int ntc, frc, fvc;
};
__host__ __device__ constexpr CombGeom comb_geom(int no, int kg) {
  return CombGeom{(kg * 2 * no + 7) / 8, frag_geom(no).ksteps * ((kg * 2 * no + 7) / 8),
                  (frag_geom(no).ksteps * ((kg * 2 * no + 7) / 8) + 1) / 2};
}
constexpr int kCombKG = 3;  // momenta per combined group

// Peer scatter of Sigma: when scatter_ranks > 0 the block
// (k, E, atom) is written straight into the (k,E)-point layout buffer of the
// rank owning point pt = k*NE + E (NVLink peer memory, CUDA IPC):
//   S_rank[pol][r] + ((pt - pt_lo[r]) * scatter_na + scatter_atom0 + la) * No^2
constexpr int kMaxScatter = 8;

struct SigmaArgs {
  const double2* G[2];
  const double2* M[2];    // operator of the chunk (layout per kernel)
  double2* S[2];
  const int* nbr;         // [chunk][NB] index of f(a,s) within the G slab
  const int* off;         // [Nw]
  int nkz, nqz, ne, nw, nb, no;
  int rows;               // NE * No
  int ctas_per_ak;
  int s_atom_begin;       // Sigma slab atom of the chunk's first atom
  long long g_sa, g_sk, g_se;  // G slab strides in complex elements
  long long s_sa, s_sk, s_se;  // Sigma slab strides in complex elements
  int npol;               // polarities to process (1 or 2)
  int off_slide;          // 1: offsets non-decreasing with steps <= 1 (sliding-window K3 eligible)
  int lookahead;          // sliding-window K3 producer lookahead (0 = default)
  int k3_opts;            // sliding-window K3: bit 0 tail-CTA tile interleave, bit 1 drop empty stages,
                          // bit 2 (K3m) partial row CTAs after the full ones
  int scatter_ranks;      // 0: write S with the s_* strides
  long long scatter_na, scatter_atom0;  // NA of the point buffers; global id of the chunk's first atom
  long long pt_lo[kMaxScatter + 1];
  double2* S_rank[2][kMaxScatter];
  // peer gather (sliding-window K3 only): G block (k, E, atom) read from
  // G_rank[pol][r] + ((k*NE + E - pt_lo[r]) * scatter_na + atom) * No^2 of the
  // point owner r; nbr holds global atom ids
  int gather_ranks;
  const double2* G_rank[2][kMaxScatter];
  // multi-momentum K3 (set by launch_sigma): momentum groups of this launch start at k_first,
  // kgroups of them; zeroM = one zero M-fragment vector (B of an invalid (k, kp) pair)
  int k_first, kgroups;
  const double2* zeroM;
  int comb_kg;            // > 0: M holds combined fragments (OperatorArgs::comb_kg)
};

// Phonon self-energy Pi (sse.py:332-428), chains in the V form
//   chain[q,w,a,s,i,j] = w_E sum_{k,E} sum_{n,p} G1[(k+q)%Nkz, E+off_w, a][n,p] * V[p,n],
//   V = dH[a,s,j] @ G2[k,E,f(a,s)] @ dH[a,s,i]      (trace cyclicity of
//   tr(dH_i G1' dH_j G2), sse.py:365-389); greater chain: G1 = G>, G2 = G<;
//   lesser chain: G1 = G<, G2 = G> (sse.py:369).
// K5 pi_build: VT[k][E][(n,p)][(s,i,j)] = V_{s,ij}[p][n] for a chunk of atoms.
// K6 pi_dmma:  per (atom, chain polarity, q, E-chunk) the [Nw x NB*9] chain
//              block on FP64 tensor cores (rows = frequencies, K = (E, n, p)),
//              partial sums per E-chunk to a scratch.
// K7 pi_assemble: sum the E-chunks in order, Pi[q,w,a,1+s] = i w_E chain,
//              Pi[q,w,a,0] = -i sum_s w_E chain (sse.py:393-406).
// Pi from the GF point layout: when ranks > 0, G block
// (k, E, atom) is read from G[pol][r] + ((k*NE + E - pt_lo[r]) * na + atom) * No^2
// of the point owner r (CUDA-IPC peer memory); atom ids are global.
struct PeerGather {
  int ranks;
  long long na;
  long long pt_lo[kMaxScatter + 1];
  const double2* G[2][kMaxScatter];
};

struct SlabPullArgs {
  int ranks;
  long long pt_lo[kMaxScatter + 1];
  const double2* src[kMaxScatter];  // per rank: [pts_r][NA][No*No] (peer pointers valid here)
  double2* dst;                     // slab block (atom i, point pt) at dst + i*dst_sa + pt*dst_sp
  long long na, atom0, natoms, no2, dst_sa, dst_sp;
  long long pt_shift;               // first point visited (the caller's own range)
};

struct PiBuildArgs {
  const double2* G[2];        // G slab per polarity (layout by strides)
  const double2* dH;          // [out atoms][NB][3][No][No]
  const int* nbr;             // [chunk][NB] G-slab index of f(a,s)
  const unsigned char* mask;  // [Nkz][NE] point mask or nullptr (sse.py:362-364)
  double2* VT[2];             // out per CHAIN polarity: [chunk][Nkz][NE][No*No][NB*9]
  int nkz, ne, nb, no;
  int atom_begin, chunk_atoms;  // chunk within the output slab (dH rows, nbr rows)
  long long g_sa, g_sk, g_se;
  int swz;                      // V column swizzle (pi_vt_swizzle)
  PeerGather peer;              // ranks > 0: G2 from the point owners (DMMA build only)
};
struct PiArgs {
  const double2* G[2];      // G slab per polarity
  const double2* VT[2];     // per chain polarity, from K5
  double2* partial;         // [chunk][2][Nqz][echunks][Nw][ncol] (w_E-scaled chains)
  const int* off;           // [Nw]
  int nkz, nqz, ne, nw, nb, no, ncol;
  int echunks, e_per_chunk;
  int warp_groups;          // ceil(m-tiles/3) * ceil(n-tiles/3)
  double energy_weight;
  long long g_sa, g_sk, g_se;
  long long g_atom_of_chunk0;  // G-slab index of the chunk's first output atom
  int swz;                     // V column swizzle (must match K5's)
  PeerGather peer;             // ranks > 0: G1 from the point owners (K6 v3 / v4 only)
  int q_in_warps;              // K6 v3: the CTA serves every q (warp = (q, lag tile)), set by launch_pi
};
struct PiAssembleArgs {
  const double2* partial;
  double2* Pi[2];           // [Nqz][Nw][out_natoms][NB+1][3][3] per polarity
  int nqz, nw, nb, ncol, echunks;
  int atom_begin, chunk_atoms, out_natoms;
};
cudaError_t launch_pi_build(const PiBuildArgs& a, cudaStream_t st);
cudaError_t launch_pi(const PiArgs& a, int chunk_atoms, cudaStream_t st);
int pi_vt_swizzle(int no, int ncol);
cudaError_t launch_pi_assemble(const PiAssembleArgs& a, cudaStream_t st);

cudaError_t launch_build_operator(const OperatorArgs& a, cudaStream_t st);
cudaError_t launch_sigma(const SigmaArgs& a, int chunk_atoms, cudaStream_t st);
cudaError_t launch_layout_transform(long long nkz, long long ne, long long na, long long blk_vec,
                                    int to_atom_major, const double2* src, double2* dst,
                                    cudaStream_t st);
cudaError_t launch_preprocess_D(long long nqz, long long nw, long long d_natoms, long long d_atom0,
                                long long out_atom0, long long out_natoms, long long nb,
                                const int* nbr, const int* rev, const double2* D, double2* Dc,
                                cudaStream_t st);
cudaError_t launch_slab_pull(const SlabPullArgs& a, long long npts, cudaStream_t st);
cudaError_t launch_fill_synthetic(uint64_t seed, uint32_t tensor_id, long long atom0,
                                  long long natoms, long long outer, long long inner,
                                  long long atom_stride, long long outer_stride, double scale,
                                  double2* dst, cudaStream_t st);

// Name of the kernel (with its template arguments) last launched per kind, in
// the SSE_PROF_* order of include/sse.h (0 operator build, 1 Sigma, 2 layout,
// 3 preprocess_D, 4 Pi operand build, 5 Pi chains, 6 Pi assembly); "" if none.
const char* last_kernel_name(int kind);

// Whether the Sigma launch for these shapes uses the multi-momentum K3 with combined fragments
// (K2 must then write them): No % 4 == 2, offsets sliding, Nw in [6, 1024], SSE_SIGMA_KERNEL=4.
bool sigma_uses_combined(int no, int nw, int off_slide);

// Bytes of the per-chunk operator buffer (one polarity).
inline size_t operator_bytes(int no, int nb, int nqz, int nw, int chunk_atoms, int comb_kg = 0, int nkz = 1) {
  if (comb_kg > 0) {
    const int groups = (nkz + comb_kg - 1) / comb_kg;
    return (size_t)comb_geom(no, comb_kg).fvc * 32 * 16 * nb * nkz * groups * nw * chunk_atoms;
  }
  size_t per = (no <= kMaxDmmaOrb) ? (size_t)frag_geom(no).fv * 32 : (size_t)no * no;
  return per * 16 * (size_t)nb * nqz * nw * chunk_atoms;
}

}  // namespace sse
