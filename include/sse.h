/*
 * libsse — B200-native (sm_100a) electron scattering self-energy Sigma^{<>}
 * of the NEGF self-consistent Born loop (SSE phase), C ABI.
 *
 * This is the drop-in boundary for the reference's SSE entry point
 *   negflow.sse.sse_sigma(variant, g, dc, dh, nmap, grid, counter=None)
 *   (/root/reference/pkg/src/negflow/sse.py:305-329)
 * Array conventions are the reference's (all complex128 as interleaved
 * re,im doubles, C-contiguous):
 *   G, Sigma  [Nkz, NE, NA, No, No]      gf.py:41, params.py:44-46
 *   Dc        [Nqz, Nw, NA, NB, 3, 3]    sse.py:81, sse.py:317
 *   dH        [NA, NB, 3, No, No]        device.py:73-75
 *   nmap      int64 [NA, NB]             device.py:23-37 (idx[a, s] = f(a, s))
 *   off, wt   [Nw] frequency_map offsets/weights, params.py:144,158-162
 * Sigma[k,E,a] = i * sum_{q<Nqz, w<Nw, s<NB} G[(k-q) mod Nkz, E-off_w, f(a,s)]
 *                    @ (wt_w sum_{i,j} Dc[q,w,a,s,i,j] dH[a,s,i] @ dH[a,s,j]),
 * terms with E-off_w < 0 dropped (sse.py:58-76, 148-161).
 *
 * Return codes: 0 ok; 1 invalid argument (Python: ValueError, the reference's
 * convention sse.py:315-318); 2 CUDA error; 3 NCCL/communication error;
 * 4 out of device memory.  sse_last_error() gives the message of the last
 * failing call on the calling thread.
 * There is no CPU fallback: without a usable sm_100a device every compute
 * entry point returns 2.
 */
#ifndef SSE_B200_SSE_H
#define SSE_B200_SSE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSE_OK 0
#define SSE_EINVAL 1
#define SSE_ECUDA 2
#define SSE_ECOMM 3
#define SSE_ENOMEM 4

/* SseVariant (sse.py:35-40).  All five produce the same Sigma (to rounding);
 * LAYOUT_TRANSFORMED runs the atom-major layout-transform kernels around the
 * fused kernel (sse.py:43-55, 244-261), the others read the grid-major
 * tensors in place. */
#define SSE_VARIANT_REFERENCE 0
#define SSE_VARIANT_FISSIONED 1
#define SSE_VARIANT_REDUNDANCY_REMOVED 2
#define SSE_VARIANT_LAYOUT_TRANSFORMED 3
#define SSE_VARIANT_BATCHED_FUSED 4

typedef struct sse_ctx sse_ctx;

/* SimParams shape fields used by the path (params.py:24-50). */
typedef struct sse_dims {
  int64_t nkz, nqz, ne, nw, na, nb, norb;
} sse_dims;

/* A device-resident atom slab of an electron tensor (G or Sigma).
 * atom0/natoms: global index of the first atom held and how many.
 * atom_major = 0: [Nkz, NE, natoms, No, No] (grid-major, the reference layout)
 * atom_major = 1: [natoms, Nkz, NE, No, No] (to_atom_major, sse.py:48-50) */
typedef struct sse_slab {
  int64_t atom0, natoms;
  int32_t atom_major;
  int32_t reserved;
} sse_slab;

/* Per-call timing (CUDA events on the library's stream, milliseconds). */
typedef struct sse_timing {
  double h2d_ms;    /* host calls with pageable inputs: host time packing the staging ring */
  double prep_ms;   /* M-operator build (and layout transforms) */
  double sigma_ms;  /* fused Sigma kernel */
  double d2h_ms;    /* host calls with pageable outputs: host time unpacking the staging ring */
  double total_ms;
  double flops;     /* algorithmic flops of the call (8 per complex MAC) */
  int64_t h2d_bytes, d2h_bytes;
  int32_t kernel_launches;
  int32_t n_devices;
  int32_t staged;       /* host calls: bit 0 inputs, bit 1 outputs went through the pinned staging ring */
  int32_t host_threads; /* host worker threads of the staging ring */
} sse_timing;

/* Context: owns a CUDA stream and cached device buffers per device.
 * n_gpus devices 0..n_gpus-1 (atoms are split in contiguous chunks across
 * them, distsim.py:117-120).  sse_ctx_create_on binds one given device. */
int sse_ctx_create(int n_gpus, sse_ctx** out);
int sse_ctx_create_on(int device, sse_ctx** out);
/* Release the context's cached device scratch (per-call buffers, the Pi operand scratch of up to
 * 2 x 24 GiB) and its pinned host staging ring, after waiting for the context's work; the next call
 * allocates again.  For callers that need the memory between SSE phases (e.g. a device GF phase).
 * Not part of the reference interface. */
int sse_ctx_trim(sse_ctx* ctx);
void sse_ctx_destroy(sse_ctx* ctx);
const char* sse_last_error(void);
int sse_version(void);

/* Host-memory drop-in for sse_sigma (sse.py:305-329).  All pointers are host
 * pointers to C-contiguous caller-owned buffers (pinned or pageable); the
 * call copies in, computes on the GPU(s) and copies Sigma back, pipelined over
 * atom chunks.  Pinned buffers are DMA'd directly; pageable ones (numpy
 * arrays, the reference's convention) go through a library-owned pinned
 * double-buffered staging ring that a host worker pool (SSE_HOST_THREADS,
 * default all hardware threads) packs / unpacks while the GPU computes.
 * off/wt: frequency_map offsets and weights.  t may be NULL. */
int sse_sigma_c128(sse_ctx* ctx, const sse_dims* d, int variant,
                   const double* G_l, const double* G_g,
                   const double* Dc_l, const double* Dc_g,
                   const double* dH, const int64_t* nmap,
                   const int64_t* off, const double* wt,
                   double* Sig_l, double* Sig_g, sse_timing* t);

/* Host-memory call for an owned atom range (one rank's share; the multi-
 * process drop-in).  g: host G slab (grid-major [Nkz, NE, g.natoms, No, No])
 * holding every neighbour of the owned atoms; out: owned atoms, with
 * Dc [Nqz, Nw, out.natoms, NB, 3, 3], dH [out.natoms, NB, 3, No, No],
 * nmap [out.natoms, NB] (global ids), Sigma [Nkz, NE, out.natoms, No, No].
 * sse_sigma_c128 is this call with both slabs = [0, NA). */
int sse_sigma_c128_slab(sse_ctx* ctx, const sse_dims* d, int variant,
                        const sse_slab* g, const sse_slab* out,
                        const double* G_l, const double* G_g,
                        const double* Dc_l, const double* Dc_g,
                        const double* dH, const int64_t* nmap,
                        const int64_t* off, const double* wt,
                        double* Sig_l, double* Sig_g, sse_timing* t);

/* Device-resident Sigma for an owned atom range (the multi-GPU shard call).
 * g: slab holding every atom f(a, s) of the owned atoms (owned + halo).
 * out: the owned atoms; Dc_*, dH, nmap cover exactly out.natoms rows:
 *   Dc [Nqz, Nw, out.natoms, NB, 3, 3], dH [out.natoms, NB, 3, No, No],
 *   nmap HOST int64 [out.natoms, NB] of GLOBAL atom indices.
 * d->na is the global atom count.  Pointers other than nmap/off/wt are
 * device pointers on the context's device; stream is a cudaStream_t (NULL =
 * the library's stream).  Asynchronous unless t != NULL (then it syncs). */
int sse_sigma_device(sse_ctx* ctx, const sse_dims* d, const sse_slab* g,
                     const sse_slab* out,
                     const double* G_l, const double* G_g,
                     const double* Dc_l, const double* Dc_g,
                     const double* dH, const int64_t* nmap,
                     const int64_t* off, const double* wt,
                     double* Sig_l, double* Sig_g, void* stream,
                     sse_timing* t);

/* Phonon self-energy Pi^{<>} (drop-in for negflow.sse.sse_pi, sse.py:409-428;
 * chains sse.py:332-390, slots sse.py:393-406):
 *   chain[q,w,a,s,i,j] = w_E sum_{k,E: E+off_w<NE} tr(dH[a,s,i] G1[(k+q)%Nkz, E+off_w, a]
 *                                                   dH[a,s,j] G2[k,E,f(a,s)]),
 *   greater: (G1,G2) = (G>,G<), lesser: (G<,G>);
 *   Pi[q,w,a,0] = -i sum_s chain, Pi[q,w,a,1+s] = +i chain;  Pi [Nqz, Nw, NA, NB+1, 3, 3].
 * d->nqz is the reference's n_qz argument; off: frequency offsets; energy_weight: w_E;
 * mask: optional uint8 [Nkz, NE] point mask (sse.py:362-364: G2 zeroed where 0), NULL = all.
 * Host call: atoms [atom_lo, atom_hi) are computed (atom_range), Pi rows of the
 * other atoms are left untouched (the caller zero-fills, as the reference's are 0). */
int sse_pi_c128(sse_ctx* ctx, const sse_dims* d, const double* G_l, const double* G_g,
                const double* dH, const int64_t* nmap, const int64_t* off,
                double energy_weight, const unsigned char* mask, int64_t atom_lo,
                int64_t atom_hi, double* Pi_l, double* Pi_g, sse_timing* t);
/* The same with the Sigma blocks scattered straight into the (k,E)-point layout
 * buffers of the point owners (the GF phase's layout, the tiled
 * scheme's return round distsim.py:300-315, here fused into the kernel's
 * epilogue as NVLink peer stores).  Rank r owns flattened points
 * [pt_lo[r], pt_lo[r+1]) (pt = k*NE + E, pt_lo[0] = 0, pt_lo[nranks] = Nkz*NE);
 * its buffers S_l[r] / S_g[r] are [pt_lo[r+1]-pt_lo[r], NA, No, No] device
 * pointers valid in this process (own allocation or sse_ipc_open).  The
 * caller synchronises the ranks before the owners read.  nranks <= 8. */
int sse_sigma_device_scatter(sse_ctx* ctx, const sse_dims* d, const sse_slab* g,
                             const sse_slab* out, const double* G_l, const double* G_g,
                             const double* Dc_l, const double* Dc_g, const double* dH,
                             const int64_t* nmap, const int64_t* off, const double* wt,
                             int nranks, const int64_t* pt_lo, double* const* S_l,
                             double* const* S_g, void* stream, sse_timing* t);

/* Fully fused GF-layout step: G is READ from the point owners' buffers too
 * (G_l[r] / G_g[r]: [pt_lo[r+1]-pt_lo[r], NA, No, No], TMA bulk copies over
 * NVLink in the sliding-window K3 producer) and Sigma is scattered as in
 * sse_sigma_device_scatter, so neither the G redistribution nor the Sigma
 * return needs a separate collective.  Needs the sliding-window K3 (sliding
 * offsets, Nw >= 12, No <= 16; else returns 1).  nmap: HOST [out.natoms, NB]
 * global ids; Dc / dH for the owned atoms. */
int sse_sigma_device_peer(sse_ctx* ctx, const sse_dims* d, const sse_slab* out,
                          const double* const* G_l, const double* const* G_g,
                          const double* Dc_l, const double* Dc_g, const double* dH,
                          const int64_t* nmap, const int64_t* off, const double* wt,
                          int nranks, const int64_t* pt_lo, double* const* S_l,
                          double* const* S_g, void* stream, sse_timing* t);

/* Pi of the owned atoms [out] with G read from the point owners' GF-layout
 * buffers (as sse_sigma_device_peer): K5 reads G2 at f(a,s), K6 reads G1
 * rows over NVLink.  Output Pi_* device [Nqz, Nw, out.natoms, NB+1, 3, 3]
 * (return it to the (q,w) point owners with an all-to-all).  Needs the DMMA
 * operand build and K6 v3/v4 (No in {4, 8, 12, 16}; else returns 1). */
int sse_pi_device_peer(sse_ctx* ctx, const sse_dims* d, const sse_slab* out,
                       const double* const* G_l, const double* const* G_g, const double* dH,
                       const int64_t* nmap, const int64_t* off, double energy_weight,
                       int nranks, const int64_t* pt_lo, double* Pi_l, double* Pi_g,
                       void* stream, sse_timing* t);

/* Assemble the G slab g (atoms [g.atom0, g.atom0+g.natoms), layout g.atom_major)
 * from the GF (k,E)-point layout: src[r] = rank r's [pts_r, NA, No, No] buffer
 * (device pointer valid in this process: local, or a CUDA-IPC-mapped peer read
 * over NVLink), pt_lo[0..nranks] the point ranges (dist.point_chunks), self_rank
 * the caller's rank (points are read starting from its own range, so concurrent
 * pulls spread over the owners; -1: from point 0).  One kernel; the slab then
 * feeds sse_sigma_device / sse_pi_device.  Replaces the
 * G-forward round of the tiled scheme's all-to-all (distsim.py:300-315). */
int sse_slab_from_points(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, int nranks,
                         const int64_t* pt_lo, const double* const* src, int self_rank, double* dst,
                         void* stream);

/* Library-owned device memory that can be shared with peer processes, and CUDA
 * IPC export / import of it (handles are SSE_IPC_HANDLE_BYTES opaque bytes). */
#define SSE_IPC_HANDLE_BYTES 64
int sse_dev_alloc(sse_ctx* ctx, size_t bytes, void** out);
int sse_dev_free(sse_ctx* ctx, void* ptr);
int sse_ipc_handle(sse_ctx* ctx, void* dptr, unsigned char* handle);
int sse_ipc_open(sse_ctx* ctx, const unsigned char* handle, void** out);
int sse_ipc_close(sse_ctx* ctx, void* ptr);

/* Multi-GPU Sigma inside the library, one process: the context's n_gpus devices
 * split the atoms in contiguous ceil-division chunks (distsim.py:117-120).  sse_multi_layout
 * writes bounds[4*i .. 4*i+3] = (lo, hi, glo, ghi) of device i: it owns atoms [lo, hi) and holds
 * the atom-major G slab [glo, ghi) (owned + the +-reach halo).  sse_sigma_multi takes per-device
 * device pointers (G_*[i] [ghi-glo, Nkz, NE, No, No] with the OWNED atoms filled, Dc_*[i]
 * [Nqz, Nw, hi-lo, NB, 3, 3], dH[i] [hi-lo, NB, 3, No, No], Sig_*[i] [hi-lo, Nkz, NE, No, No]),
 * fills every halo from the owning devices with one grouped NCCL send/recv (communicators from
 * ncclCommInitAll over the context's devices, created on first use; libnccl.so.2 is loaded at
 * run time) and runs the Sigma kernels of all devices concurrently.  nmap: HOST [NA, NB].
 * Returns 3 (SSE_ECOMM) on an NCCL failure.  Asynchronous unless t != NULL (then max over devices). */
int sse_multi_layout(sse_ctx* ctx, const sse_dims* d, const int64_t* nmap, int64_t* bounds);
int sse_sigma_multi(sse_ctx* ctx, const sse_dims* d, double* const* G_l, double* const* G_g,
                    const double* const* Dc_l, const double* const* Dc_g, const double* const* dH,
                    const int64_t* nmap, const int64_t* off, const double* wt, double* const* Sig_l,
                    double* const* Sig_g, sse_timing* t);

/* Device-resident Pi of an owned atom range: g = slab with the owned atoms and
 * all their neighbours; dH [out.natoms, NB, 3, No, No]; nmap HOST [out.natoms, NB]
 * (global ids); Pi_* device [Nqz, Nw, out.natoms, NB+1, 3, 3]. */
int sse_pi_device(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out,
                  const double* G_l, const double* G_g, const double* dH,
                  const int64_t* nmap, const int64_t* off, double energy_weight,
                  const unsigned char* mask, double* Pi_l, double* Pi_g, void* stream,
                  sse_timing* t);

/* The SSE phase of one Born iteration in one call (self_consistent_loop body,
 * sse.py:532-534: dc = preprocess_D(g_ph, nmap); sigma = sse_sigma(...);
 * pi = sse_pi(g_e, dH, nmap, grid, n_qz)).  Host arrays as in sse_sigma_c128
 * and sse_pi_c128, but D_l / D_g are the RAW phonon tensors
 * [Nqz, Nw, NA, NB+1, 3, 3] (preprocess_D runs on the device) and G is
 * uploaded once for both Sigma and Pi.  Sigma [Nkz, NE, NA, No, No] and Pi
 * [Nqz, Nw, NA, NB+1, 3, 3] are written in full.  Same numbers as the three
 * separate calls (bitwise). */
int sse_phase_c128(sse_ctx* ctx, const sse_dims* d, const double* G_l, const double* G_g,
                   const double* D_l, const double* D_g, const double* dH,
                   const int64_t* nmap, const int64_t* off, const double* wt,
                   double energy_weight, double* Sig_l, double* Sig_g, double* Pi_l,
                   double* Pi_g, sse_timing* t);

/* The same SSE phase on device-resident tensors of one rank (no host copies; the
 * device-side plug for a GPU GF phase): g = slab of G<> and of the
 * RAW phonon tensors D<> [Nqz, Nw, g.natoms, NB+1, 3, 3] over the owned atoms and
 * all their neighbours (layout of G by g.atom_major); out = the owned atoms:
 * dH [out.natoms, NB, 3, No, No], Sigma (out.atom_major layout) and Pi
 * [Nqz, Nw, out.natoms, NB+1, 3, 3].  nmap: HOST int64 [NA, NB], the full map
 * (preprocess_D needs the neighbours' reverse slots).  preprocess_D -> K2/K3 ->
 * K5-K7 on `stream` (NULL = the library's); asynchronous unless t != NULL. */
int sse_phase_device(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out,
                     const double* G_l, const double* G_g, const double* D_l, const double* D_g,
                     const double* dH, const int64_t* nmap, const int64_t* off, const double* wt,
                     double energy_weight, double* Sig_l, double* Sig_g, double* Pi_l, double* Pi_g,
                     void* stream, sse_timing* t);

/* Layout transform K1 (to_atom_major / to_grid_major, sse.py:48-55):
 * [Nkz, NE, NA, blk] <-> [NA, Nkz, NE, blk], blk = block_doubles doubles.
 * to_atom_major = 1: grid -> atom major; 0: atom -> grid major.  Device ptrs. */
int sse_layout_transform(sse_ctx* ctx, int64_t nkz, int64_t ne, int64_t na,
                         int64_t block_doubles, int to_atom_major,
                         const double* src, double* dst, void* stream);

/* preprocess_D on the device (sse.py:91-115), one polarity per call:
 * Dc[q,w,a,s] = D[q,w,b,1+rev(a,s)] - D[q,w,b,0] - D[q,w,a,0] + D[q,w,a,1+s],
 * b = nmap[a,s], rev = reverse slot (device.py:53-66), same term order as the
 * reference (bitwise equal).  D is an atom slab [Nqz, Nw, d_natoms, NB+1, 3, 3]
 * holding atoms [d_atom0, d_atom0 + d_natoms) (it must contain every owned
 * atom and all their neighbours); Dc is [Nqz, Nw, out_natoms, NB, 3, 3] for
 * atoms [out_atom0, out_atom0 + out_natoms).  nmap: HOST int64 [NA, NB], the
 * full map.  Returns 1 ("missing neighbor slot ...") when an owned edge has
 * no reverse slot. */
int sse_preprocess_D(sse_ctx* ctx, int64_t nqz, int64_t nw, int64_t na, int64_t nb,
                     const int64_t* nmap, int64_t d_atom0, int64_t d_natoms,
                     int64_t out_atom0, int64_t out_natoms, const double* D, double* Dc,
                     void* stream);

/* Atom-keyed synthetic input generator (device side of
 * paper_1912_08810_b200.inputs.atom_keyed; not part of the reference).
 * Each atom owns outer*inner complex values with local index o*inner + i;
 * value(seed, tensor_id, atom, local index) is a counter-based hash turned
 * into a unit-variance Irwin-Hall(4) deviate per real/imaginary part, times
 * scale — independent of the slab bounds, so any atom sub-problem can be
 * regenerated bit-exactly on the host.  Element (atom a, o, i) is written to
 * dst[2 * ((a - atom0) * atom_stride + o * outer_stride + i)] (complex units
 * for the strides). */
int sse_fill_synthetic(sse_ctx* ctx, uint64_t seed, uint32_t tensor_id,
                       int64_t atom0, int64_t natoms, int64_t outer,
                       int64_t inner, int64_t atom_stride, int64_t outer_stride,
                       double scale, double* dst, void* stream);

/* Per-kernel CUDA-event profile of the context's launches (bench evidence).
 * sse_profile_begin resets and enables recording on every device of ctx;
 * sse_profile_end synchronises and returns, per kernel kind, the summed
 * launch durations, launch counts and algorithmic flops since begin. */
#define SSE_PROF_OPERATOR 0   /* K2 operator build */
#define SSE_PROF_SIGMA 1      /* K3 fused Sigma (DMMA) */
#define SSE_PROF_LAYOUT 2     /* K1 layout transform */
#define SSE_PROF_PREPROCESS 3 /* preprocess_D */
#define SSE_PROF_PI_BUILD 4   /* K5 Pi operand build */
#define SSE_PROF_PI 5         /* K6 Pi chains (DMMA) */
#define SSE_PROF_PI_ASSEMBLE 6 /* K7 Pi slot assembly */
#define SSE_PROF_KINDS 7
typedef struct sse_profile {
  double ms[SSE_PROF_KINDS];
  double flops[SSE_PROF_KINDS];
  int64_t launches[SSE_PROF_KINDS];
} sse_profile;
int sse_profile_begin(sse_ctx* ctx);
int sse_profile_end(sse_ctx* ctx, sse_profile* out);

/* Name (with template arguments) of the kernel of kind SSE_PROF_* the library
 * launched last in this process, e.g. "sigma_dmma_kslide_kernel<12,12,2,3>";
 * "" before the first launch of that kind or for an unknown kind.  Thread-safe;
 * the returned string is valid until this thread's next call. */
const char* sse_kernel_name(int kind);

#ifdef __cplusplus
}
#endif

#endif /* SSE_B200_SSE_H */
