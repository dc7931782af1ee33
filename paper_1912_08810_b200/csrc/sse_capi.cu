// libsse C ABI (include/sse.h): context, validation, host and device entry points.
//
// Host entry sse_sigma_c128 / sse_sigma_c128_slab replaces negflow.sse.sse_sigma
// (sse.py:305-329).  Per device it runs a three-stream pipeline over chunks of
// owned atoms:
//   copy stream   H2D of the G columns the chunk needs (grid-major rows are
//                 strided by NA: cudaMemcpy2DAsync) + the chunk's Dc/dH rows
//   compute       K2 operator build + K3 fused DMMA Sigma kernel of the chunk
//   copy stream   D2H of the chunk's Sigma columns
// so host<->device traffic hides behind the FP64 tensor-core work.
// Multi-GPU: contiguous atom chunks per device (distsim.py:117-120), one host
// thread per device; each device reads its halo straight from host memory.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sse.h"
#include "sse_kernels.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what, int line) {
  cudaGetLastError();  // clear non-sticky errors
  if (e == cudaErrorMemoryAllocation)
    return fail(SSE_ENOMEM, "out of device memory: %s (line %d)", what, line);
  return fail(SSE_ECUDA, "CUDA error %s: %s (line %d)", cudaGetErrorString(e), what, line);
}

#define CU(x)                                                  \
  do {                                                         \
    cudaError_t e_ = (x);                                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x, __LINE__); \
  } while (0)

#define CHECK(x)                   \
  do {                             \
    int rc_ = (x);                 \
    if (rc_ != SSE_OK) return rc_; \
  } while (0)

// Grow-only device buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes) return SSE_OK;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, need);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc", __LINE__);
    bytes = need;
    return SSE_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
};

// Host worker pool for the pageable-memory staging of the host calls: fork-join
// parallel_for over [0, n) (the calling thread works too).  One job at a time.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int threads() const { return (int)workers_.size() + 1; }
  void parallel_for(int64_t n, const std::function<void(int64_t)>& f) {
    if (n <= 0) return;
    std::lock_guard<std::mutex> job_lock(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &f;
      n_ = n;
      next_.store(0);
      active_ = (int)workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain_items();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  HostPool() {
    // all hardware threads, shared between the processes of one node when launched by torchrun
    // (LOCAL_WORLD_SIZE ranks copy at once: oversubscribing the cores only adds switching)
    int n = (int)std::thread::hardware_concurrency();
    if (const char* lws = getenv("LOCAL_WORLD_SIZE"))
      if (atoi(lws) > 1) n = std::max(2, n / atoi(lws));
    if (const char* env = getenv("SSE_HOST_THREADS")) n = atoi(env);
    n = std::max(1, std::min(n, 64));
    for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  void drain_items() {
    for (int64_t i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*fn_)(i);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      drain_items();
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, job_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int64_t n_ = 0;
  std::atomic<int64_t> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Grow-only pinned host buffer (staging ring slot).
struct PinnedBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t need);
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct ProfRec {
  int kind;
  cudaEvent_t a, b;
  double flops;
};

struct DevState {
  int device = 0;
  cudaStream_t stream = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev[6] = {};
  DevBuf g[2], s[2], dc[2], dh, op[2], nbr, off, wt, tmp_g, tmp_s, pp_nbr, pp_rev, zero_m;
  DevBuf pi_vt[2], pi_part, pi_mask, pi_out[2], draw[2];
  PinnedBuf stage_in[2], stage_out[3];  // host staging ring of the pageable-memory host calls
  size_t pi_vt_budget = 0;              // Pi operand scratch per polarity (0: not decided yet)
  cudaEvent_t stage_ev[2] = {};         // H2D from stage_in[b] done
  std::vector<unsigned char> pi_mask_host;
  // host copies of the small tables last uploaded (skip re-uploads: a pageable
  // upload would otherwise serialise the host with the stream on every call)
  std::vector<int> nbr_host, off_host, pp_nbr_host, pp_rev_host;
  std::vector<double> wt_host;
  // per-launch CUDA-event profile (sse_profile_begin / sse_profile_end)
  bool profiling = false;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  std::vector<ProfRec> recs;
  // pipeline events (grow-only pool)
  std::vector<cudaEvent_t> pipe;
  // The cached scratch (op, nbr, off, wt, pi_vt, pi_part, pp_*) is shared by
  // every call on this device; a call on another stream than the previous
  // one first waits for the previous call's last use of it (scratch_done).
  cudaEvent_t scratch_done = nullptr;
  cudaStream_t scratch_stream = nullptr;
  bool scratch_pending = false;

  cudaEvent_t prof_event() {
    if (pool_used == pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[pool_used++];
  }
};

}  // namespace

// NCCL, resolved at run time (dlopen "libnccl.so.2": the copy torch already loaded, else the
// system one), so libsse has no link-time NCCL dependency and single-GPU use never touches it.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

struct sse_ctx {
  std::vector<DevState> devs;
  std::vector<ncclComm_t> comms;  // one per device (ncclCommInitAll), created on first multi-GPU call
};

namespace {

NcclApi& nccl_api() {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.CommInitAll = (decltype(api.CommInitAll))dlsym(h, "ncclCommInitAll");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
  api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.ok = api.CommInitAll && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send && api.Recv &&
           api.GetErrorString;
  return api;
}

#define NC(x)                                                                                            \
  do {                                                                                                   \
    ncclResult_t r_ = (x);                                                                               \
    if (r_ != ncclSuccess) return fail(SSE_ECOMM, "NCCL error %s: %s", nc.GetErrorString(r_), #x);       \
  } while (0)

// Record a profiled launch: `launch` is a callable returning cudaError_t.
template <class F>
int profiled(DevState& ds, cudaStream_t st, int kind, double flops, F&& launch) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (ds.profiling) {
    a = ds.prof_event();
    b = ds.prof_event();
    if (!a || !b) return fail(SSE_ECUDA, "event creation failed");
    CU(cudaEventRecord(a, st));
  }
  CU(launch());
  if (ds.profiling) {
    CU(cudaEventRecord(b, st));
    ds.recs.push_back({kind, a, b, flops});
  }
  return SSE_OK;
}

template <class T>
int upload_cached(DevBuf& buf, std::vector<T>& host_copy, const std::vector<T>& v, cudaStream_t st) {
  if (buf.ptr && host_copy == v) return SSE_OK;
  CHECK(buf.ensure(std::max<size_t>(v.size(), 1) * sizeof(T)));
  // a pageable async copy stages the source before returning; later calls on
  // the same stream are ordered after the kernels that read this table.
  CU(cudaMemcpyAsync(buf.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  host_copy = v;
  return SSE_OK;
}

int PinnedBuf::ensure(size_t need) {
  if (need <= bytes) return SSE_OK;
  release();
  cudaError_t e = cudaHostAlloc(&ptr, need, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    ptr = nullptr;
    cudaGetLastError();
    return fail(SSE_ENOMEM, "cannot allocate %.2f GB of pinned staging memory", need / 1e9);
  }
  bytes = need;
  return SSE_OK;
}

int init_dev(DevState& d, int device) {
  d.device = device;
  CU(cudaSetDevice(device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(SSE_ECUDA, "device %d (%s, sm_%d%d) is not an sm_100 Blackwell GPU", device,
                prop.name, prop.major, prop.minor);
  CU(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&d.s_h2d, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&d.s_d2h, cudaStreamNonBlocking));
  for (auto& e : d.ev) CU(cudaEventCreate(&e));
  CU(cudaEventCreateWithFlags(&d.scratch_done, cudaEventDisableTiming));
  for (auto& e : d.stage_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // one zero M-fragment vector (the multi-momentum K3's B of an invalid (k, kp) pair)
  const size_t zbytes = (size_t)sse::frag_geom(sse::kMaxDmmaOrb).fv * 32 * 16;
  CHECK(d.zero_m.ensure(zbytes));
  CU(cudaMemset(d.zero_m.ptr, 0, zbytes));
  return SSE_OK;
}

// Order a call on stream st after the previous call's use of the shared scratch.
int scratch_enter(DevState& ds, cudaStream_t st) {
  if (ds.scratch_pending && ds.scratch_stream != st) CU(cudaStreamWaitEvent(st, ds.scratch_done, 0));
  return SSE_OK;
}
// Mark the end of this call's use of the scratch (its last kernel is queued on st).
int scratch_leave(DevState& ds, cudaStream_t st) {
  CU(cudaEventRecord(ds.scratch_done, st));
  ds.scratch_stream = st;
  ds.scratch_pending = true;
  return SSE_OK;
}

// Error paths of the host calls: earlier chunks' copies may still be in flight into
// (or out of) the caller's host buffers; wait for them before reporting the error.
void drain(DevState& ds) {
  for (cudaStream_t s : {ds.stream, ds.s_h2d, ds.s_d2h})
    if (s) cudaStreamSynchronize(s);
  cudaGetLastError();
}

void destroy_dev(DevState& d) {
  cudaSetDevice(d.device);
  for (DevBuf* b : {&d.g[0], &d.g[1], &d.s[0], &d.s[1], &d.dc[0], &d.dc[1], &d.dh, &d.op[0],
                    &d.op[1], &d.nbr, &d.off, &d.wt, &d.tmp_g, &d.tmp_s, &d.pp_nbr, &d.pp_rev, &d.zero_m,
                    &d.pi_vt[0], &d.pi_vt[1], &d.pi_part, &d.pi_mask, &d.pi_out[0], &d.pi_out[1],
                    &d.draw[0], &d.draw[1]})
    b->release();
  for (auto& e : d.ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : d.pool) cudaEventDestroy(e);
  for (auto& e : d.pipe) cudaEventDestroy(e);
  if (d.scratch_done) cudaEventDestroy(d.scratch_done);
  for (auto& e : d.stage_ev)
    if (e) cudaEventDestroy(e);
  for (PinnedBuf* b : {&d.stage_in[0], &d.stage_in[1], &d.stage_out[0], &d.stage_out[1], &d.stage_out[2]})
    b->release();
  for (cudaStream_t s : {d.stream, d.s_h2d, d.s_d2h})
    if (s) cudaStreamDestroy(s);
}

int validate_dims(const sse_dims* d) {
  if (!d) return fail(SSE_EINVAL, "dims is NULL");
  const int64_t v[7] = {d->nkz, d->nqz, d->ne, d->nw, d->na, d->nb, d->norb};
  const char* names[7] = {"n_kz", "n_qz", "n_E", "n_w", "n_A", "n_B", "n_orb"};
  for (int i = 0; i < 7; ++i)
    if (v[i] < 1) return fail(SSE_EINVAL, "%s must be >= 1, got %lld", names[i], (long long)v[i]);
  if (d->nb > (1 << 20) || d->norb > 64 || d->nw > (1 << 20) || d->nkz > (1 << 16) ||
      d->nqz > (1 << 16) || d->na > (1LL << 30))
    return fail(SSE_EINVAL, "dimension out of supported range");
  if (d->ne * d->norb > (1LL << 30)) return fail(SSE_EINVAL, "n_E * n_orb too large");
  return SSE_OK;
}

int validate_grid(const sse_dims* d, const int64_t* off, const double* wt) {
  if (!off || !wt) return fail(SSE_EINVAL, "frequency map is NULL");
  for (int64_t w = 0; w < d->nw; ++w) {
    if (off[w] < 0 || off[w] >= d->ne)
      return fail(SSE_EINVAL, "frequency offset %lld (index %lld) outside [0, %lld)",
                  (long long)off[w], (long long)w, (long long)d->ne);
    if (!std::isfinite(wt[w]))
      return fail(SSE_EINVAL, "frequency weight %g (index %lld) is not finite", wt[w], (long long)w);
  }
  return SSE_OK;
}

// Pi entry points: offsets in [0, NE) and a finite energy weight (params.py:158-162)
int validate_offsets(const sse_dims* d, const int64_t* off, double energy_weight) {
  if (!off) return fail(SSE_EINVAL, "frequency map is NULL");
  for (int64_t w = 0; w < d->nw; ++w)
    if (off[w] < 0 || off[w] >= d->ne)
      return fail(SSE_EINVAL, "frequency offset %lld (index %lld) outside [0, %lld)", (long long)off[w],
                  (long long)w, (long long)d->ne);
  if (!std::isfinite(energy_weight)) return fail(SSE_EINVAL, "energy weight is not finite");
  return SSE_OK;
}

int validate_slab(const sse_dims* d, const sse_slab* s, const char* what) {
  if (!s) return fail(SSE_EINVAL, "%s slab is NULL", what);
  if (s->natoms < 1 || s->atom0 < 0 || s->atom0 + s->natoms > d->na)
    return fail(SSE_EINVAL, "%s slab [%lld, %lld) outside [0, %lld)", what, (long long)s->atom0,
                (long long)(s->atom0 + s->natoms), (long long)d->na);
  return SSE_OK;
}

constexpr int64_t kPiEnergiesPerChunk = 96;

// Operator chunk: bound the per-polarity operator buffer to ~1 GiB
// (SSE_OP_CHUNK_ATOMS overrides, for experiments).
// Offsets non-decreasing with steps <= 1 (default_grid's): the sliding-window K3 kernels apply.
int offsets_slide(const sse_dims* d, const int64_t* off) {
  for (int64_t w = 1; w < d->nw; ++w)
    if (off[w] < off[w - 1] || off[w] > off[w - 1] + 1) return 0;
  return 1;
}

// K2 writes combined multi-momentum fragments for this call (sse::sigma_uses_combined).
int comb_kg_of(const sse_dims* d, const int64_t* off) {
  if (d->norb > sse::kMaxDmmaOrb || d->nqz > 8) return 0;
  return sse::sigma_uses_combined((int)d->norb, (int)d->nw, offsets_slide(d, off)) ? sse::kCombKG : 0;
}

int64_t op_chunk_atoms(const sse_dims* d, const int64_t* off) {
  if (const char* env = getenv("SSE_OP_CHUNK_ATOMS")) {
    const long long v = atoll(env);
    if (v > 0) return v;
  }
  const size_t per_atom = sse::operator_bytes((int)d->norb, (int)d->nb, (int)d->nqz, (int)d->nw, 1,
                                              comb_kg_of(d, off), (int)d->nkz);
  return std::max<int64_t>(1, (int64_t)((1ull << 30) / std::max<size_t>(per_atom, 1)));
}

struct SlabStrides {
  long long sa, sk, se;
};
SlabStrides strides_of(const sse_dims* d, const sse_slab& slab) {
  const long long no2 = d->norb * d->norb;
  if (slab.atom_major) return {d->nkz * d->ne * no2, d->ne * no2, no2};
  return {no2, d->ne * slab.natoms * no2, slab.natoms * no2};
}

double alg_flops(const sse_dims* d, const int64_t* off, int64_t natoms, int npol = 2) {
  double terms = 0;
  for (int64_t w = 0; w < d->nw; ++w) terms += (double)std::max<int64_t>(0, d->ne - off[w]);
  const double no3 = (double)d->norb * d->norb * d->norb;
  return 8.0 * npol * natoms * d->nb * d->nkz * d->nqz * no3 * terms;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Upload the neighbour (G-slab local), offset and weight tables of an owned range.
int prepare_tables(DevState& ds, const sse_dims* d, const sse_slab& g, const sse_slab& out,
                   const int64_t* nmap, const int64_t* off, const double* wt, cudaStream_t st) {
  std::vector<int> nbr((size_t)out.natoms * d->nb);
  for (int64_t a = 0; a < out.natoms; ++a)
    for (int64_t s = 0; s < d->nb; ++s) {
      const int64_t b = nmap[a * d->nb + s];
      if (b < 0 || b >= d->na)
        return fail(SSE_EINVAL, "neighbor index %lld of atom %lld outside [0, %lld)", (long long)b,
                    (long long)(out.atom0 + a), (long long)d->na);
      if (b < g.atom0 || b >= g.atom0 + g.natoms)
        return fail(SSE_EINVAL, "neighbor atom %lld of atom %lld is not in the G slab [%lld, %lld)",
                    (long long)b, (long long)(out.atom0 + a), (long long)g.atom0,
                    (long long)(g.atom0 + g.natoms));
      nbr[a * d->nb + s] = (int)(b - g.atom0);
    }
  std::vector<int> offs(d->nw);
  for (int64_t w = 0; w < d->nw; ++w) offs[w] = (int)off[w];
  CHECK(upload_cached(ds.nbr, ds.nbr_host, nbr, st));
  CHECK(upload_cached(ds.off, ds.off_host, offs, st));
  if (wt) {
    std::vector<double> wts(wt, wt + d->nw);
    CHECK(upload_cached(ds.wt, ds.wt_host, wts, st));
  }
  return SSE_OK;
}

struct DevPtrs {
  const double2 *G_l, *G_g, *Dc_l, *Dc_g, *dH;
  double2 *S_l, *S_g;
};

// K2 + K3 for owned atoms [a0, a0 + n) of the out slab (tables already uploaded).
// Peer scatter of Sigma into the (k,E)-point layout buffers of the owner ranks
struct ScatterCfg {
  int nranks = 0;
  int64_t na = 0;
  int64_t pt_lo[sse::kMaxScatter + 1] = {};
  double2* S[2][sse::kMaxScatter] = {};
  bool gather = false;  // G read from the owners' point buffers too (sliding-window K3)
  const double2* G[2][sse::kMaxScatter] = {};
};

int run_chunk(DevState& ds, const sse_dims* d, const sse_slab& g, const sse_slab& out,
              const DevPtrs& p, const int64_t* off, int64_t a0, int64_t n, cudaStream_t st,
              int npol, int* launches, const ScatterCfg* sc = nullptr) {
  const int no = (int)d->norb;
  const int comb = comb_kg_of(d, off);
  const size_t opb = sse::operator_bytes(no, (int)d->nb, (int)d->nqz, (int)d->nw, (int)n, comb, (int)d->nkz);
  CHECK(ds.op[0].ensure(opb));
  CHECK(ds.op[1].ensure(opb));
  sse::OperatorArgs oa{};
  oa.Dc[0] = p.Dc_l;
  oa.Dc[1] = p.Dc_g;
  oa.dH = p.dH;
  oa.wt = ds.wt.as<double>();
  oa.M[0] = ds.op[0].as<double2>();
  oa.M[1] = ds.op[1].as<double2>();
  oa.nqz = (int)d->nqz;
  oa.nw = (int)d->nw;
  oa.nb = (int)d->nb;
  oa.no = no;
  oa.dc_natoms = (int)out.natoms;
  oa.atom_begin = (int)a0;
  oa.chunk_atoms = (int)n;
  oa.fragment_order = no <= sse::kMaxDmmaOrb ? 1 : 0;
  oa.npol = npol;
  oa.comb_kg = comb;
  oa.nkz = (int)d->nkz;
  CHECK(profiled(ds, st, SSE_PROF_OPERATOR, 0.0, [&] { return sse::launch_build_operator(oa, st); }));

  const SlabStrides gs = strides_of(d, g), ss = strides_of(d, out);
  sse::SigmaArgs sa{};
  sa.G[0] = p.G_l;
  sa.G[1] = p.G_g;
  sa.M[0] = oa.M[0];
  sa.M[1] = oa.M[1];
  sa.S[0] = p.S_l;
  sa.S[1] = p.S_g;
  sa.nbr = ds.nbr.as<int>() + a0 * d->nb;
  sa.off = ds.off.as<int>();
  sa.nkz = (int)d->nkz;
  sa.nqz = (int)d->nqz;
  sa.ne = (int)d->ne;
  sa.nw = (int)d->nw;
  sa.nb = (int)d->nb;
  sa.no = no;
  sa.rows = (int)(d->ne * no);
  sa.s_atom_begin = (int)a0;
  sa.g_sa = gs.sa;
  sa.g_sk = gs.sk;
  sa.g_se = gs.se;
  sa.s_sa = ss.sa;
  sa.s_sk = ss.sk;
  sa.s_se = ss.se;
  sa.npol = npol;
  sa.zeroM = ds.zero_m.as<double2>();
  sa.comb_kg = comb;
  sa.off_slide = offsets_slide(d, off);
  sa.lookahead = getenv("SSE_SLIDE_LOOKAHEAD") ? atoi(getenv("SSE_SLIDE_LOOKAHEAD")) : 0;
  sa.k3_opts = getenv("SSE_K3_OPTS") ? atoi(getenv("SSE_K3_OPTS")) : 7;
  if (sc && sc->nranks > 0) {
    sa.scatter_ranks = sc->nranks;
    sa.scatter_na = sc->na;
    sa.scatter_atom0 = out.atom0 + a0;
    for (int r = 0; r <= sc->nranks; ++r) sa.pt_lo[r] = sc->pt_lo[r];
    for (int pol = 0; pol < 2; ++pol)
      for (int r = 0; r < sc->nranks; ++r) sa.S_rank[pol][r] = sc->S[pol][r];
    if (sc->gather) {
      sa.gather_ranks = sc->nranks;
      for (int pol = 0; pol < 2; ++pol)
        for (int r = 0; r < sc->nranks; ++r) sa.G_rank[pol][r] = sc->G[pol][r];
    }
  }
  CHECK(profiled(ds, st, SSE_PROF_SIGMA, alg_flops(d, off, n, npol),
                 [&] { return sse::launch_sigma(sa, (int)n, st); }));
  if (launches) *launches += 2;
  return SSE_OK;
}

int sigma_on_device(DevState& ds, const sse_dims* d, const sse_slab& g, const sse_slab& out,
                    const DevPtrs& p, const int64_t* nmap, const int64_t* off, const double* wt,
                    cudaStream_t st, int* launches, int npol = 2, const ScatterCfg* sc = nullptr) {
  CHECK(prepare_tables(ds, d, g, out, nmap, off, wt, st));
  // balanced chunks (no small trailing launch whose CTAs would fill only part of a wave)
  const int64_t max_chunk = std::min<int64_t>(op_chunk_atoms(d, off), out.natoms);
  const int64_t n_chunks = (out.natoms + max_chunk - 1) / max_chunk;
  const int64_t chunk = (out.natoms + n_chunks - 1) / n_chunks;
  for (int64_t a0 = 0; a0 < out.natoms; a0 += chunk)
    CHECK(run_chunk(ds, d, g, out, p, off, a0, std::min<int64_t>(chunk, out.natoms - a0), st, npol,
                    launches, sc));
  return SSE_OK;
}

// Phonon self-energy Pi (sse_pi, sse.py:409-428) for the owned atoms of `out`:
// K5 operand build (VT) -> K6 DMMA chains (partials per E-chunk) -> K7 assembly,
// in atom chunks bounded by the VT scratch (12 or 24 GiB per polarity).  Pi_* are device
// [Nqz, Nw, out.natoms, NB+1, 3, 3]; mask: host [Nkz*NE] or NULL.
int pi_on_device(DevState& ds, const sse_dims* d, const sse_slab& g, const sse_slab& out,
                 const double2* G_l, const double2* G_g, const double2* dH, const int64_t* nmap,
                 const int64_t* off, double energy_weight, const unsigned char* mask, double2* Pi_l,
                 double2* Pi_g, cudaStream_t st, int* launches, const sse::PeerGather* peer = nullptr,
                 const std::function<int(int64_t, int64_t)>& before_chunk = nullptr,
                 const std::function<int(int64_t, int64_t)>& after_chunk = nullptr) {
  CHECK(prepare_tables(ds, d, g, out, nmap, off, nullptr, st));
  const unsigned char* mask_dev = nullptr;
  if (mask) {
    std::vector<unsigned char> m(mask, mask + d->nkz * d->ne);
    CHECK(upload_cached(ds.pi_mask, ds.pi_mask_host, m, st));
    mask_dev = ds.pi_mask.as<unsigned char>();
  }
  const int no = (int)d->norb, no2 = no * no, nb = (int)d->nb, ncol = nb * 9;
  const size_t vt_atom = (size_t)d->nkz * d->ne * no2 * ncol * 16;  // per chain polarity
  // VT scratch per polarity: 24 GiB when the device has room for it (free + the VT already held
  // >= 2 x 24 GiB + 16 GiB), else 12 GiB.  Each K6 launch ends with a drain of ~2.4 ms (CTAs of
  // ~9 ms, partially occupied SMs), so fewer, larger chunks save ~1 % of Pi at paper
  // (`profiles/r02_ab_k6_chunk.log`); sse_ctx_trim hands the cached scratch back.
  // (decided once per context -- cudaMemGetInfo is not free -- and again after sse_ctx_trim)
  if (ds.pi_vt_budget == 0) {
    ds.pi_vt_budget = 12ull << 30;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess &&
        free_b + ds.pi_vt[0].bytes + ds.pi_vt[1].bytes >= 2 * (24ull << 30) + (16ull << 30))
      ds.pi_vt_budget = 24ull << 30;
    cudaGetLastError();
  }
  const size_t vt_budget = ds.pi_vt_budget;
  int64_t chunk = std::max<int64_t>(1, (int64_t)(vt_budget / std::max<size_t>(vt_atom, 1)));
  if (const char* env = getenv("SSE_PI_CHUNK_ATOMS"))  // override, for tests and experiments
    if (atoll(env) > 0) chunk = atoll(env);
  chunk = std::min<int64_t>(chunk, out.natoms);
  const int64_t n_chunks = (out.natoms + chunk - 1) / chunk;
  chunk = (out.natoms + n_chunks - 1) / n_chunks;  // balanced chunks (no tiny tail launch)
  const int nqz = (int)d->nqz, nw = (int)d->nw;
  // E-chunks of a fixed size (independent of the atom partition, so Pi is
  // bitwise identical for any chunking / device count)
  const int e_per = (int)std::min<int64_t>(d->ne, kPiEnergiesPerChunk);
  const int echunks = (int)((d->ne + e_per - 1) / e_per);
  const int m_tiles = (nw + 7) / 8, n_tiles = (2 * ncol + 7) / 8;
  const int warp_groups = ((m_tiles + 2) / 3) * ((n_tiles + 2) / 3);
  CHECK(ds.pi_vt[0].ensure(vt_atom * chunk));
  CHECK(ds.pi_vt[1].ensure(vt_atom * chunk));
  CHECK(ds.pi_part.ensure((size_t)chunk * 2 * nqz * echunks * nw * ncol * 16));
  const SlabStrides gs = strides_of(d, g);
  for (int64_t a0 = 0; a0 < out.natoms; a0 += chunk) {
    const int n = (int)std::min<int64_t>(chunk, out.natoms - a0);
    if (before_chunk) CHECK(before_chunk(a0, n));  // e.g. the host call's progressive G upload
    sse::PiBuildArgs ba{};
    ba.G[0] = G_l;
    ba.G[1] = G_g;
    ba.dH = dH;
    ba.nbr = ds.nbr.as<int>() + a0 * nb;
    ba.mask = mask_dev;
    ba.VT[0] = ds.pi_vt[0].as<double2>();
    ba.VT[1] = ds.pi_vt[1].as<double2>();
    ba.nkz = (int)d->nkz;
    ba.ne = (int)d->ne;
    ba.nb = nb;
    ba.no = no;
    ba.atom_begin = (int)a0;
    ba.chunk_atoms = n;
    ba.g_sa = gs.sa;
    ba.g_sk = gs.sk;
    ba.g_se = gs.se;
    ba.swz = sse::pi_vt_swizzle(no, ncol);
    if (peer) ba.peer = *peer;
    CHECK(profiled(ds, st, SSE_PROF_PI_BUILD, 0.0, [&] { return sse::launch_pi_build(ba, st); }));
    sse::PiArgs pa{};
    pa.G[0] = G_l;
    pa.G[1] = G_g;
    pa.VT[0] = ba.VT[0];
    pa.VT[1] = ba.VT[1];
    pa.partial = ds.pi_part.as<double2>();
    pa.off = ds.off.as<int>();
    pa.nkz = (int)d->nkz;
    pa.nqz = nqz;
    pa.ne = (int)d->ne;
    pa.nw = nw;
    pa.nb = nb;
    pa.no = no;
    pa.ncol = ncol;
    pa.echunks = echunks;
    pa.e_per_chunk = e_per;
    pa.warp_groups = warp_groups;
    pa.energy_weight = energy_weight;
    pa.g_sa = gs.sa;
    pa.g_sk = gs.sk;
    pa.g_se = gs.se;
    pa.g_atom_of_chunk0 = out.atom0 + a0 - g.atom0;
    pa.swz = ba.swz;
    if (peer) pa.peer = *peer;
    double flops = 0;  // 8 per complex MAC, both chain polarities, valid (E + off < NE) terms
    for (int64_t w = 0; w < d->nw; ++w) flops += (double)std::max<int64_t>(0, d->ne - off[w]);
    flops *= 16.0 * n * nqz * d->nkz * no2 * ncol;
    CHECK(profiled(ds, st, SSE_PROF_PI, flops, [&] { return sse::launch_pi(pa, n, st); }));
    sse::PiAssembleArgs aa{};
    aa.partial = pa.partial;
    aa.Pi[0] = Pi_l;
    aa.Pi[1] = Pi_g;
    aa.nqz = nqz;
    aa.nw = nw;
    aa.nb = nb;
    aa.ncol = ncol;
    aa.echunks = echunks;
    aa.atom_begin = (int)a0;
    aa.chunk_atoms = n;
    aa.out_natoms = (int)out.natoms;
    CHECK(profiled(ds, st, SSE_PROF_PI_ASSEMBLE, 0.0, [&] { return sse::launch_pi_assemble(aa, st); }));
    if (launches) *launches += 3;
    if (after_chunk) CHECK(after_chunk(a0, n));  // e.g. the chunk's Pi to the host
  }
  return SSE_OK;
}

cudaEvent_t pipe_event(DevState& ds, size_t i);

// Host-call helper: Pi of owned-atom chunk [a0, a0 + n) (device [rows][on][pi_row]) to the host
// tensors Ph (global atom lo + a0 of [rows][na][pi_row]) on the D2H stream once K7 wrote it.
int pi_chunk_to_host(DevState& ds, const sse_dims* d, int64_t lo, int64_t on, int64_t a0, int64_t n,
                     double* const* Ph, cudaStream_t st, size_t* ei) {
  const size_t pi_row = (size_t)(d->nb + 1) * 9 * 16;
  const size_t pi_rows = (size_t)(d->nqz * d->nw);
  cudaEvent_t done = pipe_event(ds, (*ei)++);
  if (!done) return fail(SSE_ECUDA, "event creation failed");
  CU(cudaEventRecord(done, st));
  CU(cudaStreamWaitEvent(ds.s_d2h, done, 0));
  for (int p = 0; p < 2; ++p)
    CU(cudaMemcpy2DAsync((char*)Ph[p] + (lo + a0) * pi_row, d->na * pi_row, (char*)ds.pi_out[p].ptr + a0 * pi_row,
                         on * pi_row, n * pi_row, pi_rows, cudaMemcpyDeviceToHost, ds.s_d2h));
  return SSE_OK;
}

// Join the D2H stream back into st (after the last pi_chunk_to_host).
int join_d2h(DevState& ds, cudaStream_t st, size_t* ei) {
  cudaEvent_t e = pipe_event(ds, (*ei)++);
  if (!e) return fail(SSE_ECUDA, "event creation failed");
  CU(cudaEventRecord(e, ds.s_d2h));
  CU(cudaStreamWaitEvent(st, e, 0));
  return SSE_OK;
}

// ---------------------------------------------------------------------------
// host-memory call
// ---------------------------------------------------------------------------
struct HostCall {
  const sse_dims* d;
  int variant;
  sse_slab hg, hs;  // host G slab and host out slab (grid-major)
  const double *G_l, *G_g, *Dc_l, *Dc_g, *dH;
  const int64_t *nmap, *off;  // nmap rows of hs atoms
  const double* wt;
  double *S_l, *S_g;
  bool dc_resident = false;  // Dc already in ds.dc (device preprocess_D of sse_phase_c128)
};

cudaEvent_t pipe_event(DevState& ds, size_t i) {
  while (ds.pipe.size() <= i) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    ds.pipe.push_back(e);
  }
  return ds.pipe[i];
}

// One device's share of a host-memory call: owned atoms [lo, hi) (global ids).
int host_call_on_device_body(DevState& ds, const HostCall& c, int64_t lo, int64_t hi, sse_timing* t) {
  const sse_dims* d = c.d;
  CU(cudaSetDevice(ds.device));
  const int64_t on = hi - lo;
  if (on <= 0) return SSE_OK;
  const int64_t* rows_nmap = c.nmap + (lo - c.hs.atom0) * d->nb;
  int64_t glo = lo, ghi = hi;
  for (int64_t i = 0; i < on * d->nb; ++i) {
    const int64_t b = rows_nmap[i];
    if (b < 0 || b >= d->na)
      return fail(SSE_EINVAL, "neighbor index %lld of atom %lld outside [0, %lld)", (long long)b,
                  (long long)(lo + i / d->nb), (long long)d->na);
    glo = std::min(glo, b);
    ghi = std::max(ghi, b + 1);
  }
  if (glo < c.hg.atom0 || ghi > c.hg.atom0 + c.hg.natoms)
    return fail(SSE_EINVAL, "host G slab [%lld, %lld) lacks neighbour atoms [%lld, %lld)",
                (long long)c.hg.atom0, (long long)(c.hg.atom0 + c.hg.natoms), (long long)glo,
                (long long)ghi);
  const int64_t gn = ghi - glo;
  const size_t blk = (size_t)d->norb * d->norb * 16;  // bytes per (k, E, atom) block
  const size_t rows = (size_t)(d->nkz * d->ne);
  const size_t dc_row = (size_t)d->nb * 9 * 16, dc_rows = (size_t)(d->nqz * d->nw);
  const size_t dh_atom = (size_t)d->nb * 3 * blk;
  const size_t g_bytes = rows * gn * blk, s_bytes = rows * on * blk;
  const size_t dc_bytes = dc_rows * on * dc_row, dh_bytes = on * dh_atom;
  const size_t hg_pitch = c.hg.natoms * blk, hs_pitch = c.hs.natoms * blk;
  const size_t hdc_pitch = c.hs.natoms * dc_row;
  const char* Gh[2] = {(const char*)c.G_l, (const char*)c.G_g};
  const char* Dh[2] = {(const char*)c.Dc_l, (const char*)c.Dc_g};
  char* Sh[2] = {(char*)c.S_l, (char*)c.S_g};
  const char* dHh = (const char*)c.dH + (lo - c.hs.atom0) * dh_atom;
  const bool am = c.variant == SSE_VARIANT_LAYOUT_TRANSFORMED;

  for (int p = 0; p < 2; ++p) {
    CHECK(ds.g[p].ensure(g_bytes));
    CHECK(ds.s[p].ensure(s_bytes));
    CHECK(ds.dc[p].ensure(dc_bytes));
  }
  CHECK(ds.dh.ensure(dh_bytes));
  cudaStream_t st = ds.stream;
  sse_slab gslab{glo, gn, 0, 0}, oslab{lo, on, 0, 0};
  int launches = 0;
  CU(cudaEventRecord(ds.ev[0], st));

  if (am) {
    // LAYOUT_TRANSFORMED (sse.py:244-261): copy everything, K1 to atom-major,
    // atom-major accumulation, K1 back; polarities one after the other.
    CHECK(ds.tmp_g.ensure(g_bytes));
    CHECK(ds.tmp_s.ensure(s_bytes));
    for (int p = 0; p < 2; ++p) {
      CU(cudaMemcpy2DAsync(ds.g[p].ptr, gn * blk, Gh[p] + (glo - c.hg.atom0) * blk, hg_pitch,
                           gn * blk, rows, cudaMemcpyHostToDevice, st));
      CU(cudaMemcpy2DAsync(ds.dc[p].ptr, on * dc_row, Dh[p] + (lo - c.hs.atom0) * dc_row, hdc_pitch,
                           on * dc_row, dc_rows, cudaMemcpyHostToDevice, st));
    }
    CU(cudaMemcpyAsync(ds.dh.ptr, dHh, dh_bytes, cudaMemcpyHostToDevice, st));
    sse_slab ga{glo, gn, 1, 0}, oa{lo, on, 1, 0};
    CHECK(prepare_tables(ds, d, ga, oa, rows_nmap, c.off, c.wt, st));
    for (int p = 0; p < 2; ++p) {
      CHECK(profiled(ds, st, SSE_PROF_LAYOUT, 0.0, [&] {
        return sse::launch_layout_transform(d->nkz, d->ne, gn, d->norb * d->norb, 1,
                                            ds.g[p].as<double2>(), ds.tmp_g.as<double2>(), st);
      }));
      DevPtrs ptr{ds.tmp_g.as<double2>(), ds.tmp_g.as<double2>(), ds.dc[p].as<double2>(),
                  ds.dc[p].as<double2>(), ds.dh.as<double2>(), ds.tmp_s.as<double2>(),
                  ds.tmp_s.as<double2>()};
      const int64_t chunk = std::min<int64_t>(op_chunk_atoms(d, c.off), on);
      for (int64_t a0 = 0; a0 < on; a0 += chunk)
        CHECK(run_chunk(ds, d, ga, oa, ptr, c.off, a0, std::min<int64_t>(chunk, on - a0), st, 1,
                        &launches));
      CHECK(profiled(ds, st, SSE_PROF_LAYOUT, 0.0, [&] {
        return sse::launch_layout_transform(d->nkz, d->ne, on, d->norb * d->norb, 0,
                                            ds.tmp_s.as<double2>(), ds.s[p].as<double2>(), st);
      }));
      launches += 2;
    }
    for (int p = 0; p < 2; ++p)
      CU(cudaMemcpy2DAsync(Sh[p] + (lo - c.hs.atom0) * blk, hs_pitch, ds.s[p].ptr, on * blk,
                           on * blk, rows, cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(ds.ev[1], st));
  } else {
    // pipelined over chunks of owned atoms
    CHECK(prepare_tables(ds, d, gslab, oslab, rows_nmap, c.off, c.wt, st));
    CU(cudaEventRecord(ds.ev[2], st));
    CU(cudaStreamWaitEvent(ds.s_h2d, ds.ev[2], 0));
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(op_chunk_atoms(d, c.off), (on + 7) / 8));
    // chunk boundaries: a geometric ramp of small chunks at the start (the first chunk's H2D is
    // not hidden; each chunk's compute then covers the next one's H2D, ~3.5x faster per atom on
    // one B200) and the mirrored ramp at the end (the last chunk's D2H is not hidden)
    // (a 25-atom edge measured 35 ms slower end to end: its first pack / H2D and last unpack are exposed)
    const int64_t edge = std::max<int64_t>(1, std::min<int64_t>(8, chunk / 4));
    std::vector<int64_t> ramp;
    for (int64_t s = edge; s < chunk; s *= 3) ramp.push_back(s);
    int64_t ramp_atoms = 0;
    for (int64_t s : ramp) ramp_atoms += s;
    std::vector<int64_t> bounds{0};
    if (on >= 2 * ramp_atoms + chunk) {
      for (int64_t s : ramp) bounds.push_back(bounds.back() + s);
      const int64_t tail = on - ramp_atoms;
      while (bounds.back() + chunk < tail) bounds.push_back(bounds.back() + chunk);
      if (tail > bounds.back()) bounds.push_back(tail);
      int64_t b = tail;
      for (size_t i = ramp.size(); i-- > 1;) bounds.push_back(b += ramp[i]);
    } else if (on > 2 * edge + chunk) {
      bounds.push_back(edge);
      while (bounds.back() + chunk < on - edge) bounds.push_back(bounds.back() + chunk);
      bounds.push_back(on - edge);
    } else {
      while (bounds.back() + chunk < on) bounds.push_back(bounds.back() + chunk);
    }
    bounds.push_back(on);
    // per chunk: owned atoms [a0, a0 + n) and the G columns [c0, c1) first needed by it
    struct Piece {
      int64_t a0, n, c0, c1;
    };
    std::vector<Piece> plan;
    int64_t copied = glo;  // G columns [glo, copied) are on their way
    for (size_t ci = 0; ci + 1 < bounds.size(); ++ci) {
      const int64_t a0 = bounds[ci], n = bounds[ci + 1] - bounds[ci];
      if (n <= 0) continue;
      int64_t need = copied;
      for (int64_t i = a0 * d->nb; i < (a0 + n) * d->nb; ++i) need = std::max(need, rows_nmap[i] + 1);
      need = std::max(need, lo + a0 + n);
      plan.push_back({a0, n, copied, std::max(copied, need)});
      copied = std::max(copied, need);
    }
    // Pageable caller memory cannot be DMA'd asynchronously (a pageable D2H blocks the host until
    // the chunk's kernels finish, serialising the pipeline), so it is staged through a pinned
    // double-buffered ring: the host worker pool packs chunk i+1's G columns / Dc / dH rows and
    // unpacks chunk i-1's Sigma columns while the GPU computes chunk i.  Pinned callers (and
    // SSE_HOST_STAGING=0) take the direct DMA path.
    auto pinned = [](const void* ptr) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return a.type == cudaMemoryTypeHost;
    };
    const char* stage_env = getenv("SSE_HOST_STAGING");
    const int stage_mode = stage_env ? atoi(stage_env) : -1;  // -1 auto, 0 never, 1 always
    const bool in_pinned = pinned(c.G_l) && pinned(c.G_g) && pinned(c.dH) &&
                           (c.dc_resident || (pinned(c.Dc_l) && pinned(c.Dc_g)));
    const bool out_pinned = pinned(c.S_l) && pinned(c.S_g);
    const bool stage_in = stage_mode == 1 || (stage_mode == -1 && !in_pinned);
    const bool stage_out = stage_mode == 1 || (stage_mode == -1 && !out_pinned);
    size_t in_cap = 0, out_cap = 0;
    for (const Piece& pc : plan) {
      in_cap = std::max(in_cap, 2 * rows * (pc.c1 - pc.c0) * blk + (c.dc_resident ? 0 : 2 * dc_rows * pc.n * dc_row) +
                                    pc.n * dh_atom);
      out_cap = std::max(out_cap, 2 * rows * pc.n * blk);
    }
    if (stage_in)
      for (int b = 0; b < 2; ++b) CHECK(ds.stage_in[b].ensure(in_cap));
    if (stage_out)
      for (int b = 0; b < 3; ++b) CHECK(ds.stage_out[b].ensure(out_cap));
    HostPool& pool = HostPool::get();
    double pack_ms = 0, unpack_ms = 0;
    auto now_ms = [] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const bool trace = getenv("SSE_STAGING_TRACE") != nullptr;  // per-chunk host timeline on stderr
    const double t_call = now_ms();
    // strided row copies (rows x width bytes) split over the pool, ~1 MB per work item
    auto copy_rows = [&](char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, size_t nrows) {
      const size_t per = std::max<size_t>(1, (1u << 20) / std::max<size_t>(width, 1));
      const int64_t items = (int64_t)((nrows + per - 1) / per);
      pool.parallel_for(items, [&](int64_t it) {
        const size_t r0 = it * per, r1 = std::min(nrows, r0 + per);
        for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
      });
    };
    auto unpack = [&](size_t k) {  // chunk k's Sigma columns: staging -> caller rows
      const Piece& pc = plan[k];
      const double t0 = now_ms();
      const char* src = (const char*)ds.stage_out[k % 3].ptr;
      for (int p = 0; p < 2; ++p)
        copy_rows(Sh[p] + (lo + pc.a0 - c.hs.atom0) * blk, hs_pitch, src + p * rows * pc.n * blk, pc.n * blk,
                  pc.n * blk, rows);
      unpack_ms += now_ms() - t0;
      if (trace)
        fprintf(stderr, "[sse staging] unpack chunk %zu (%lld atoms): %.1f-%.1f ms\n", k, (long long)pc.n, t0 - t_call,
                now_ms() - t_call);
    };
    const DevPtrs ptr{ds.g[0].as<double2>(), ds.g[1].as<double2>(), ds.dc[0].as<double2>(),
                      ds.dc[1].as<double2>(), ds.dh.as<double2>(), ds.s[0].as<double2>(),
                      ds.s[1].as<double2>()};
    size_t ei = 0;
    std::vector<cudaEvent_t> out_ready(plan.size(), nullptr);
    // H2D of chunk ci (packing it first for pageable callers); its completion event is in_ev[ci]
    std::vector<cudaEvent_t> in_ev(plan.size(), nullptr);
    auto issue_h2d = [&](size_t ci) -> int {
      const Piece& pc = plan[ci];
      const int64_t a0 = pc.a0, n = pc.n, ncols = pc.c1 - pc.c0;
      if (stage_in) {
        const int b = (int)(ci % 2);
        if (ci >= 2) CU(cudaEventSynchronize(ds.stage_ev[b]));  // H2D of chunk ci-2 left stage_in[b]
        const double t0 = now_ms();
        char* buf = (char*)ds.stage_in[b].ptr;
        char* g_st[2] = {buf, buf + rows * ncols * blk};
        char* dc_st[2] = {buf + 2 * rows * ncols * blk, buf + 2 * rows * ncols * blk + dc_rows * n * dc_row};
        char* dh_st = buf + 2 * rows * ncols * blk + (c.dc_resident ? 0 : 2 * dc_rows * n * dc_row);
        for (int p = 0; p < 2; ++p) {
          if (ncols > 0)
            copy_rows(g_st[p], ncols * blk, Gh[p] + (pc.c0 - c.hg.atom0) * blk, hg_pitch, ncols * blk, rows);
          if (!c.dc_resident)
            copy_rows(dc_st[p], n * dc_row, Dh[p] + (lo + a0 - c.hs.atom0) * dc_row, hdc_pitch, n * dc_row, dc_rows);
        }
        copy_rows(dh_st, n * dh_atom, dHh + a0 * dh_atom, n * dh_atom, n * dh_atom, 1);
        pack_ms += now_ms() - t0;
        if (trace)
          fprintf(stderr, "[sse staging] pack chunk %zu (%lld atoms, %lld G cols): %.1f-%.1f ms\n", ci, (long long)n,
                  (long long)ncols, t0 - t_call, now_ms() - t_call);
        for (int p = 0; p < 2; ++p) {
          if (ncols > 0)
            CU(cudaMemcpy2DAsync((char*)ds.g[p].ptr + (pc.c0 - glo) * blk, gn * blk, g_st[p], ncols * blk, ncols * blk,
                                 rows, cudaMemcpyHostToDevice, ds.s_h2d));
          if (!c.dc_resident)
            CU(cudaMemcpy2DAsync((char*)ds.dc[p].ptr + a0 * dc_row, on * dc_row, dc_st[p], n * dc_row, n * dc_row,
                                 dc_rows, cudaMemcpyHostToDevice, ds.s_h2d));
        }
        CU(cudaMemcpyAsync((char*)ds.dh.ptr + a0 * dh_atom, dh_st, n * dh_atom, cudaMemcpyHostToDevice, ds.s_h2d));
        CU(cudaEventRecord(ds.stage_ev[b], ds.s_h2d));
      } else {
        if (ncols > 0)
          for (int p = 0; p < 2; ++p)
            CU(cudaMemcpy2DAsync((char*)ds.g[p].ptr + (pc.c0 - glo) * blk, gn * blk,
                                 Gh[p] + (pc.c0 - c.hg.atom0) * blk, hg_pitch, ncols * blk, rows,
                                 cudaMemcpyHostToDevice, ds.s_h2d));
        if (!c.dc_resident)
          for (int p = 0; p < 2; ++p)
            CU(cudaMemcpy2DAsync((char*)ds.dc[p].ptr + a0 * dc_row, on * dc_row,
                                 Dh[p] + (lo + a0 - c.hs.atom0) * dc_row, hdc_pitch, n * dc_row, dc_rows,
                                 cudaMemcpyHostToDevice, ds.s_h2d));
        CU(cudaMemcpyAsync((char*)ds.dh.ptr + a0 * dh_atom, dHh + a0 * dh_atom, n * dh_atom,
                           cudaMemcpyHostToDevice, ds.s_h2d));
      }
      in_ev[ci] = pipe_event(ds, ei++);
      if (!in_ev[ci]) return fail(SSE_ECUDA, "event creation failed");
      CU(cudaEventRecord(in_ev[ci], ds.s_h2d));
      return SSE_OK;
    };
    // compute + D2H of chunk ci (its H2D already queued); staged outputs go to slot ci % 3
    auto issue_compute = [&](size_t ci) -> int {
      const Piece& pc = plan[ci];
      const int64_t a0 = pc.a0, n = pc.n;
      cudaEvent_t done = pipe_event(ds, ei++);
      if (!done) return fail(SSE_ECUDA, "event creation failed");
      CU(cudaStreamWaitEvent(st, in_ev[ci], 0));
      CHECK(run_chunk(ds, d, gslab, oslab, ptr, c.off, a0, n, st, 2, &launches));
      CU(cudaEventRecord(done, st));
      CU(cudaStreamWaitEvent(ds.s_d2h, done, 0));
      if (stage_out) {
        char* dst = (char*)ds.stage_out[ci % 3].ptr;  // its previous chunk (ci-3) was unpacked already
        for (int p = 0; p < 2; ++p)
          CU(cudaMemcpy2DAsync(dst + p * rows * n * blk, n * blk, (char*)ds.s[p].ptr + a0 * blk, on * blk, n * blk,
                               rows, cudaMemcpyDeviceToHost, ds.s_d2h));
        out_ready[ci] = pipe_event(ds, ei++);
        if (!out_ready[ci]) return fail(SSE_ECUDA, "event creation failed");
        CU(cudaEventRecord(out_ready[ci], ds.s_d2h));
      } else {
        for (int p = 0; p < 2; ++p)
          CU(cudaMemcpy2DAsync(Sh[p] + (lo + a0 - c.hs.atom0) * blk, hs_pitch,
                               (char*)ds.s[p].ptr + a0 * blk, on * blk, n * blk, rows,
                               cudaMemcpyDeviceToHost, ds.s_d2h));
      }
      return SSE_OK;
    };
    // The GPU is kept two chunks ahead of the host: chunks ci+1 and ci+2 are packed and queued
    // (H2D, compute, D2H) before the host waits for chunk ci's Sigma and unpacks it, so a long
    // unpack of a big chunk never starves the short chunks of the closing ramp.
    const size_t nch = plan.size();
    for (size_t ci = 0; ci < std::min<size_t>(2, nch); ++ci) {
      CHECK(issue_h2d(ci));
      CHECK(issue_compute(ci));
    }
    for (size_t ci = 0; ci < nch; ++ci) {
      if (ci + 2 < nch) {
        CHECK(issue_h2d(ci + 2));     // input slot (ci+2) % 2: its previous H2D (chunk ci) is done early
        CHECK(issue_compute(ci + 2));  // output slot (ci+2) % 3: chunk ci-1 was unpacked last iteration
      }
      if (stage_out) {
        const double tw = now_ms();
        CU(cudaEventSynchronize(out_ready[ci]));
        if (trace)
          fprintf(stderr, "[sse staging] wait D2H chunk %zu: %.1f-%.1f ms\n", ci, tw - t_call, now_ms() - t_call);
        unpack(ci);
      }
    }
    if (t) {
      t->h2d_ms += pack_ms;
      t->d2h_ms += unpack_ms;
      t->staged = (stage_in ? 1 : 0) | (stage_out ? 2 : 0);
      t->host_threads = pool.threads();
    }
    CU(cudaEventRecord(ds.ev[3], ds.s_d2h));
    CU(cudaStreamWaitEvent(st, ds.ev[3], 0));
    CU(cudaEventRecord(ds.ev[1], st));
  }
  CU(cudaEventSynchronize(ds.ev[1]));
  if (t) {
    t->total_ms = std::max(t->total_ms, (double)elapsed(ds.ev[0], ds.ev[1]));
    t->h2d_bytes += 2 * (g_bytes + (c.dc_resident ? 0 : dc_bytes)) + dh_bytes;
    t->d2h_bytes += 2 * s_bytes;
    t->kernel_launches += launches;
  }
  return SSE_OK;
}

// Run `body` for one device of a host call: ordered after the previous call's use of the
// shared scratch; on error the in-flight host copies are drained before returning.
template <class F>
int guarded(DevState& ds, F&& body) {
  CU(cudaSetDevice(ds.device));
  CHECK(scratch_enter(ds, ds.stream));
  const int rc = body();
  if (rc != SSE_OK) {
    const std::string err = g_last_error;
    drain(ds);
    g_last_error = err;
    return rc;
  }
  return scratch_leave(ds, ds.stream);
}

int host_call_on_device(DevState& ds, const HostCall& c, int64_t lo, int64_t hi, sse_timing* t) {
  return guarded(ds, [&] { return host_call_on_device_body(ds, c, lo, hi, t); });
}

// Reverse-slot table of the owned edges (device.py:53-66): for owned atom a and
// slot s, b = idx[a, s] (as a D-slab index) and the first r with idx[b, r] == a.
int preprocess_tables(const int64_t* nmap, int64_t na, int64_t nb, int64_t d_atom0, int64_t d_natoms,
                      int64_t out_atom0, int64_t out_natoms, std::vector<int>& nbr, std::vector<int>& rev) {
  nbr.assign(out_natoms * nb, 0);
  rev.assign(out_natoms * nb, 0);
  auto in_slab = [&](int64_t x) { return x >= d_atom0 && x < d_atom0 + d_natoms; };
  for (int64_t la = 0; la < out_natoms; ++la) {
    const int64_t a = out_atom0 + la;
    if (!in_slab(a)) return fail(SSE_EINVAL, "atom %lld is not in the D slab", (long long)a);
    for (int64_t s = 0; s < nb; ++s) {
      const int64_t b = nmap[a * nb + s];
      if (b < 0 || b >= na)
        return fail(SSE_EINVAL, "neighbor index %lld of atom %lld outside [0, %lld)", (long long)b,
                    (long long)a, (long long)na);
      int64_t r = 0;
      while (r < nb && nmap[b * nb + r] != a) ++r;
      if (r == nb)
        return fail(SSE_EINVAL, "missing neighbor slot: atom %lld not in neighbor list of %lld",
                    (long long)a, (long long)b);
      if (!in_slab(b)) return fail(SSE_EINVAL, "neighbor atom %lld is not in the D slab", (long long)b);
      nbr[la * nb + s] = (int)(b - d_atom0);
      rev[la * nb + s] = (int)r;
    }
  }
  return SSE_OK;
}

int host_call(sse_ctx* ctx, const HostCall& c, sse_timing* t) {
  const sse_dims* d = c.d;
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->flops = alg_flops(d, c.off, c.hs.natoms);
  }
  const int nd = (int)ctx->devs.size();
  if (t) t->n_devices = nd;
  const int64_t per = (c.hs.natoms + nd - 1) / nd;  // ceil-division chunks (distsim.py:117-120)
  if (nd == 1) return host_call_on_device(ctx->devs[0], c, c.hs.atom0, c.hs.atom0 + c.hs.natoms, t);
  std::vector<int> rcs(nd, SSE_OK);
  std::vector<sse_timing> ts(nd);
  std::vector<std::string> errs(nd);
  std::vector<std::thread> th;
  for (int i = 0; i < nd; ++i) {
    th.emplace_back([&, i] {
      std::memset(&ts[i], 0, sizeof(sse_timing));
      const int64_t lo = c.hs.atom0 + std::min<int64_t>(i * per, c.hs.natoms);
      const int64_t hi = c.hs.atom0 + std::min<int64_t>((i + 1) * per, c.hs.natoms);
      rcs[i] = host_call_on_device(ctx->devs[i], c, lo, hi, &ts[i]);
      if (rcs[i] != SSE_OK) errs[i] = g_last_error;
    });
  }
  for (auto& x : th) x.join();
  for (int i = 0; i < nd; ++i) {
    if (rcs[i] != SSE_OK) {
      g_last_error = errs[i];
      return rcs[i];
    }
    if (t) {
      t->total_ms = std::max(t->total_ms, ts[i].total_ms);
      t->h2d_bytes += ts[i].h2d_bytes;
      t->d2h_bytes += ts[i].d2h_bytes;
      t->kernel_launches += ts[i].kernel_launches;
      t->h2d_ms = std::max(t->h2d_ms, ts[i].h2d_ms);
      t->d2h_ms = std::max(t->d2h_ms, ts[i].d2h_ms);
      t->staged |= ts[i].staged;
      t->host_threads = std::max(t->host_threads, ts[i].host_threads);
    }
  }
  return SSE_OK;
}

}  // namespace

extern "C" {

const char* sse_last_error(void) { return g_last_error.c_str(); }

int sse_version(void) { return 1; }

int sse_ctx_create(int n_gpus, sse_ctx** out) {
  if (!out) return fail(SSE_EINVAL, "out is NULL");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(SSE_ECUDA, "no CUDA device available (%s); libsse has no CPU fallback",
                cudaGetErrorString(e));
  if (n_gpus < 1 || n_gpus > count)
    return fail(SSE_EINVAL, "n_gpus=%d but %d device(s) visible", n_gpus, count);
  sse_ctx* ctx = new sse_ctx;
  ctx->devs.resize(n_gpus);
  for (int i = 0; i < n_gpus; ++i) {
    int rc = init_dev(ctx->devs[i], i);
    if (rc != SSE_OK) {
      sse_ctx_destroy(ctx);
      return rc;
    }
  }
  *out = ctx;
  return SSE_OK;
}

int sse_ctx_create_on(int device, sse_ctx** out) {
  if (!out) return fail(SSE_EINVAL, "out is NULL");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(SSE_ECUDA, "no CUDA device available (%s); libsse has no CPU fallback",
                cudaGetErrorString(e));
  if (device < 0 || device >= count)
    return fail(SSE_EINVAL, "device %d but %d device(s) visible", device, count);
  sse_ctx* ctx = new sse_ctx;
  ctx->devs.resize(1);
  int rc = init_dev(ctx->devs[0], device);
  if (rc != SSE_OK) {
    sse_ctx_destroy(ctx);
    return rc;
  }
  *out = ctx;
  return SSE_OK;
}

int sse_ctx_trim(sse_ctx* ctx) {
  if (!ctx) return fail(SSE_EINVAL, "ctx is NULL");
  for (auto& d : ctx->devs) {
    CU(cudaSetDevice(d.device));
    if (d.scratch_pending) CU(cudaEventSynchronize(d.scratch_done));
    for (cudaStream_t st : {d.stream, d.s_h2d, d.s_d2h})
      if (st) CU(cudaStreamSynchronize(st));
    // the large per-call buffers (the small uploaded tables stay: their host shadows skip re-uploads)
    for (DevBuf* b : {&d.g[0], &d.g[1], &d.s[0], &d.s[1], &d.dc[0], &d.dc[1], &d.op[0], &d.op[1], &d.tmp_g,
                      &d.tmp_s, &d.pi_vt[0], &d.pi_vt[1], &d.pi_part, &d.pi_out[0], &d.pi_out[1], &d.draw[0],
                      &d.draw[1]})
      b->release();
    for (PinnedBuf* b : {&d.stage_in[0], &d.stage_in[1], &d.stage_out[0], &d.stage_out[1], &d.stage_out[2]})
      b->release();
    d.pi_vt_budget = 0;  // re-decided against the then free memory
  }
  return SSE_OK;
}

void sse_ctx_destroy(sse_ctx* ctx) {
  if (!ctx) return;
  if (!ctx->comms.empty()) {
    NcclApi& nc = nccl_api();
    for (ncclComm_t c : ctx->comms)
      if (c && nc.ok) nc.CommDestroy(c);
  }
  for (auto& d : ctx->devs) destroy_dev(d);
  delete ctx;
}

int sse_sigma_c128_slab(sse_ctx* ctx, const sse_dims* d, int variant, const sse_slab* g,
                        const sse_slab* out, const double* G_l, const double* G_g,
                        const double* Dc_l, const double* Dc_g, const double* dH,
                        const int64_t* nmap, const int64_t* off, const double* wt, double* Sig_l,
                        double* Sig_g, sse_timing* t) {
  if (!ctx) return fail(SSE_EINVAL, "context is NULL");
  CHECK(validate_dims(d));
  CHECK(validate_grid(d, off, wt));
  CHECK(validate_slab(d, g, "G"));
  CHECK(validate_slab(d, out, "output"));
  if (g->atom_major || out->atom_major)
    return fail(SSE_EINVAL, "host slabs must be grid-major (the reference layout)");
  if (variant < SSE_VARIANT_REFERENCE || variant > SSE_VARIANT_BATCHED_FUSED)
    return fail(SSE_EINVAL, "unknown variant %d", variant);
  if (!G_l || !G_g || !Dc_l || !Dc_g || !dH || !nmap || !Sig_l || !Sig_g)
    return fail(SSE_EINVAL, "NULL tensor pointer");
  HostCall c{d, variant, *g, *out, G_l, G_g, Dc_l, Dc_g, dH, nmap, off, wt, Sig_l, Sig_g};
  return host_call(ctx, c, t);
}

int sse_sigma_c128(sse_ctx* ctx, const sse_dims* d, int variant, const double* G_l,
                   const double* G_g, const double* Dc_l, const double* Dc_g, const double* dH,
                   const int64_t* nmap, const int64_t* off, const double* wt, double* Sig_l,
                   double* Sig_g, sse_timing* t) {
  CHECK(validate_dims(d));
  const sse_slab full{0, d->na, 0, 0};
  return sse_sigma_c128_slab(ctx, d, variant, &full, &full, G_l, G_g, Dc_l, Dc_g, dH, nmap, off, wt,
                             Sig_l, Sig_g, t);
}

int sse_sigma_device(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out,
                     const double* G_l, const double* G_g, const double* Dc_l, const double* Dc_g,
                     const double* dH, const int64_t* nmap, const int64_t* off, const double* wt,
                     double* Sig_l, double* Sig_g, void* stream, sse_timing* t) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device call needs a 1-device context");
  CHECK(validate_dims(d));
  CHECK(validate_grid(d, off, wt));
  CHECK(validate_slab(d, g, "G"));
  CHECK(validate_slab(d, out, "output"));
  if (!G_l || !G_g || !Dc_l || !Dc_g || !dH || !nmap || !Sig_l || !Sig_g)
    return fail(SSE_EINVAL, "NULL tensor pointer");
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->flops = alg_flops(d, off, out->natoms);
    t->n_devices = 1;
    CU(cudaEventRecord(ds.ev[0], st));
  }
  int launches = 0;
  const DevPtrs p{(const double2*)G_l, (const double2*)G_g, (const double2*)Dc_l,
                  (const double2*)Dc_g, (const double2*)dH, (double2*)Sig_l, (double2*)Sig_g};
  CHECK(scratch_enter(ds, st));
  CHECK(sigma_on_device(ds, d, *g, *out, p, nmap, off, wt, st, &launches));
  CHECK(scratch_leave(ds, st));
  if (t) {
    CU(cudaEventRecord(ds.ev[1], st));
    CU(cudaEventSynchronize(ds.ev[1]));
    t->sigma_ms = t->total_ms = elapsed(ds.ev[0], ds.ev[1]);
    t->kernel_launches = launches;
  }
  return SSE_OK;
}

}  // extern "C"

namespace {
int sigma_peer_impl(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out, const double* G_l,
                    const double* G_g, const double* const* G_l_ranks, const double* const* G_g_ranks,
                    const double* Dc_l, const double* Dc_g, const double* dH, const int64_t* nmap,
                    const int64_t* off, const double* wt, int nranks, const int64_t* pt_lo, double* const* S_l,
                    double* const* S_g, void* stream, sse_timing* t) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device call needs a 1-device context");
  CHECK(validate_dims(d));
  CHECK(validate_grid(d, off, wt));
  CHECK(validate_slab(d, g, "G"));
  CHECK(validate_slab(d, out, "output"));
  const bool gather = G_l_ranks != nullptr;
  if ((!gather && (!G_l || !G_g)) || (gather && !G_g_ranks) || !Dc_l || !Dc_g || !dH || !nmap || !pt_lo || !S_l ||
      !S_g)
    return fail(SSE_EINVAL, "NULL tensor pointer");
  if (nranks < 1 || nranks > sse::kMaxScatter)
    return fail(SSE_EINVAL, "scatter needs 1..%d ranks (got %d)", sse::kMaxScatter, nranks);
  ScatterCfg sc;
  sc.nranks = nranks;
  sc.na = d->na;
  if (pt_lo[0] != 0 || pt_lo[nranks] != d->nkz * d->ne)
    return fail(SSE_EINVAL, "point ranges must cover [0, Nkz*NE)");
  for (int r = 0; r <= nranks; ++r) {
    if (r > 0 && pt_lo[r] < pt_lo[r - 1]) return fail(SSE_EINVAL, "point ranges must be non-decreasing");
    sc.pt_lo[r] = pt_lo[r];
  }
  for (int r = 0; r < nranks; ++r) {
    if ((!S_l[r] || !S_g[r]) && pt_lo[r + 1] > pt_lo[r]) return fail(SSE_EINVAL, "NULL scatter target");
    sc.S[0][r] = (double2*)S_l[r];
    sc.S[1][r] = (double2*)S_g[r];
    if (gather) {
      if ((!G_l_ranks[r] || !G_g_ranks[r]) && pt_lo[r + 1] > pt_lo[r]) return fail(SSE_EINVAL, "NULL gather source");
      sc.G[0][r] = (const double2*)G_l_ranks[r];
      sc.G[1][r] = (const double2*)G_g_ranks[r];
    }
  }
  sc.gather = gather;
  if (gather && (g->atom0 != 0 || g->natoms != d->na))
    return fail(SSE_EINVAL, "peer gather reads G by global atom id: pass the G slab [0, NA)");
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->flops = alg_flops(d, off, out->natoms);
    t->n_devices = 1;
    CU(cudaEventRecord(ds.ev[0], st));
  }
  int launches = 0;
  const DevPtrs p{(const double2*)G_l, (const double2*)G_g, (const double2*)Dc_l,
                  (const double2*)Dc_g, (const double2*)dH, nullptr, nullptr};
  CHECK(scratch_enter(ds, st));
  const int rc = sigma_on_device(ds, d, *g, *out, p, nmap, off, wt, st, &launches, 2, &sc);
  if (rc == SSE_OK) CHECK(scratch_leave(ds, st));
  if (rc == SSE_ECUDA && gather && std::string(g_last_error).find("not supported") != std::string::npos)
    return fail(SSE_EINVAL, "peer gather needs the sliding-window K3 (sliding offsets, Nw >= 12, No <= 16)");
  CHECK(rc);
  if (t) {
    CU(cudaEventRecord(ds.ev[1], st));
    CU(cudaEventSynchronize(ds.ev[1]));
    t->sigma_ms = t->total_ms = elapsed(ds.ev[0], ds.ev[1]);
    t->kernel_launches = launches;
  }
  return SSE_OK;
}

}  // namespace

extern "C" {

int sse_sigma_device_scatter(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out,
                             const double* G_l, const double* G_g, const double* Dc_l, const double* Dc_g,
                             const double* dH, const int64_t* nmap, const int64_t* off, const double* wt,
                             int nranks, const int64_t* pt_lo, double* const* S_l, double* const* S_g,
                             void* stream, sse_timing* t) {
  return sigma_peer_impl(ctx, d, g, out, G_l, G_g, nullptr, nullptr, Dc_l, Dc_g, dH, nmap, off, wt, nranks, pt_lo,
                         S_l, S_g, stream, t);
}

int sse_sigma_device_peer(sse_ctx* ctx, const sse_dims* d, const sse_slab* out, const double* const* G_l,
                          const double* const* G_g, const double* Dc_l, const double* Dc_g, const double* dH,
                          const int64_t* nmap, const int64_t* off, const double* wt, int nranks,
                          const int64_t* pt_lo, double* const* S_l, double* const* S_g, void* stream,
                          sse_timing* t) {
  if (!d) return fail(SSE_EINVAL, "dims is NULL");
  const sse_slab all{0, d->na, 1, 0};
  return sigma_peer_impl(ctx, d, &all, out, nullptr, nullptr, G_l, G_g, Dc_l, Dc_g, dH, nmap, off, wt, nranks,
                         pt_lo, S_l, S_g, stream, t);
}

int sse_pi_device_peer(sse_ctx* ctx, const sse_dims* d, const sse_slab* out, const double* const* G_l,
                       const double* const* G_g, const double* dH, const int64_t* nmap, const int64_t* off,
                       double energy_weight, int nranks, const int64_t* pt_lo, double* Pi_l, double* Pi_g,
                       void* stream, sse_timing* t) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device call needs a 1-device context");
  CHECK(validate_dims(d));
  CHECK(validate_slab(d, out, "output"));
  if (!G_l || !G_g || !dH || !nmap || !off || !pt_lo || !Pi_l || !Pi_g) return fail(SSE_EINVAL, "NULL tensor pointer");
  CHECK(validate_offsets(d, off, energy_weight));
  if (nranks < 1 || nranks > sse::kMaxScatter)
    return fail(SSE_EINVAL, "peer gather needs 1..%d ranks (got %d)", sse::kMaxScatter, nranks);
  if (pt_lo[0] != 0 || pt_lo[nranks] != d->nkz * d->ne) return fail(SSE_EINVAL, "point ranges must cover [0, Nkz*NE)");
  sse::PeerGather pg{};
  pg.ranks = nranks;
  pg.na = d->na;
  for (int r = 0; r <= nranks; ++r) {
    if (r > 0 && pt_lo[r] < pt_lo[r - 1]) return fail(SSE_EINVAL, "point ranges must be non-decreasing");
    pg.pt_lo[r] = pt_lo[r];
  }
  for (int r = 0; r < nranks; ++r) {
    if ((!G_l[r] || !G_g[r]) && pt_lo[r + 1] > pt_lo[r]) return fail(SSE_EINVAL, "NULL gather source");
    pg.G[0][r] = (const double2*)G_l[r];
    pg.G[1][r] = (const double2*)G_g[r];
  }
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->n_devices = 1;
    CU(cudaEventRecord(ds.ev[0], st));
  }
  int launches = 0;
  const sse_slab all{0, d->na, 1, 0};
  CHECK(scratch_enter(ds, st));
  const int rc = pi_on_device(ds, d, all, *out, nullptr, nullptr, (const double2*)dH, nmap, off, energy_weight, nullptr,
                              (double2*)Pi_l, (double2*)Pi_g, st, &launches, &pg);
  if (rc == SSE_OK) CHECK(scratch_leave(ds, st));
  if (rc == SSE_ECUDA && std::string(g_last_error).find("not supported") != std::string::npos)
    return fail(SSE_EINVAL, "Pi peer gather needs the DMMA operand build and K6 v3/v4 (No in {4,8,12,16})");
  CHECK(rc);
  if (t) {
    CU(cudaEventRecord(ds.ev[1], st));
    CU(cudaEventSynchronize(ds.ev[1]));
    t->total_ms = elapsed(ds.ev[0], ds.ev[1]);
    t->kernel_launches = launches;
  }
  return SSE_OK;
}

int sse_slab_from_points(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, int nranks, const int64_t* pt_lo,
                         const double* const* src, int self_rank, double* dst, void* stream) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device call needs a 1-device context");
  CHECK(validate_dims(d));
  CHECK(validate_slab(d, g, "G"));
  if (!src || !pt_lo || !dst) return fail(SSE_EINVAL, "NULL tensor pointer");
  if (nranks < 1 || nranks > sse::kMaxScatter)
    return fail(SSE_EINVAL, "slab pull needs 1..%d ranks (got %d)", sse::kMaxScatter, nranks);
  const int64_t npts = d->nkz * d->ne;
  if (pt_lo[0] != 0 || pt_lo[nranks] != npts) return fail(SSE_EINVAL, "point ranges must cover [0, Nkz*NE)");
  if (npts > 65535) return fail(SSE_EINVAL, "slab pull supports at most 65535 (k,E) points");
  if (g->natoms * d->norb * d->norb >= (1ll << 32)) return fail(SSE_EINVAL, "slab too wide for the pull kernel");
  sse::SlabPullArgs a{};
  a.ranks = nranks;
  for (int r = 0; r <= nranks; ++r) {
    if (r > 0 && pt_lo[r] < pt_lo[r - 1]) return fail(SSE_EINVAL, "point ranges must be non-decreasing");
    a.pt_lo[r] = pt_lo[r];
  }
  for (int r = 0; r < nranks; ++r) {
    if (!src[r] && pt_lo[r + 1] > pt_lo[r]) return fail(SSE_EINVAL, "NULL point source for rank %d", r);
    a.src[r] = (const double2*)src[r];
  }
  const SlabStrides gs = strides_of(d, *g);
  a.dst = (double2*)dst;
  a.na = d->na;
  a.atom0 = g->atom0;
  a.natoms = g->natoms;
  a.no2 = d->norb * d->norb;
  a.dst_sa = gs.sa;
  a.dst_sp = gs.se;  // point k*NE+e: k*sk + e*se == (k*NE+e)*se in both layouts
  if (self_rank >= nranks) return fail(SSE_EINVAL, "self_rank %d outside [0, %d)", self_rank, nranks);
  a.pt_shift = self_rank >= 0 ? pt_lo[self_rank] : 0;
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  CU(sse::launch_slab_pull(a, npts, st));
  return SSE_OK;
}

int sse_dev_alloc(sse_ctx* ctx, size_t bytes, void** out) {
  if (!ctx || ctx->devs.size() != 1 || !out) return fail(SSE_EINVAL, "device allocation needs a 1-device context");
  CU(cudaSetDevice(ctx->devs[0].device));
  *out = nullptr;
  cudaError_t e = cudaMalloc(out, bytes ? bytes : 1);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc", __LINE__);
  return SSE_OK;
}

int sse_dev_free(sse_ctx* ctx, void* ptr) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device free needs a 1-device context");
  CU(cudaSetDevice(ctx->devs[0].device));
  if (ptr) CU(cudaFree(ptr));
  return SSE_OK;
}

int sse_ipc_handle(sse_ctx* ctx, void* dptr, unsigned char* handle) {
  if (!ctx || ctx->devs.size() != 1 || !dptr || !handle) return fail(SSE_EINVAL, "invalid IPC export");
  CU(cudaSetDevice(ctx->devs[0].device));
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, dptr));
  static_assert(sizeof(h) == SSE_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  return SSE_OK;
}

int sse_ipc_open(sse_ctx* ctx, const unsigned char* handle, void** out) {
  if (!ctx || ctx->devs.size() != 1 || !handle || !out) return fail(SSE_EINVAL, "invalid IPC import");
  CU(cudaSetDevice(ctx->devs[0].device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CU(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return SSE_OK;
}

int sse_ipc_close(sse_ctx* ctx, void* ptr) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "invalid IPC close");
  CU(cudaSetDevice(ctx->devs[0].device));
  if (ptr) CU(cudaIpcCloseMemHandle(ptr));
  return SSE_OK;
}

// Multi-GPU inside the library (one process): atom chunks per context device
// (distsim.py:117-120), each device's atom-major G slab = owned atoms + the +-reach halo.
static void multi_bounds(const sse_dims* d, const int64_t* nmap, int nd, std::vector<int64_t>& b) {
  b.assign((size_t)nd * 4, 0);
  const int64_t per = (d->na + nd - 1) / nd;
  for (int i = 0; i < nd; ++i) {
    const int64_t lo = std::min<int64_t>(i * per, d->na), hi = std::min<int64_t>((i + 1) * per, d->na);
    int64_t glo = lo, ghi = hi;
    for (int64_t x = lo * d->nb; x < hi * d->nb; ++x) {
      glo = std::min(glo, nmap[x]);
      ghi = std::max(ghi, nmap[x] + 1);
    }
    b[4 * i] = lo;
    b[4 * i + 1] = hi;
    b[4 * i + 2] = glo;
    b[4 * i + 3] = ghi;
  }
}

int sse_multi_layout(sse_ctx* ctx, const sse_dims* d, const int64_t* nmap, int64_t* bounds) {
  if (!ctx || !bounds || !nmap) return fail(SSE_EINVAL, "NULL argument");
  CHECK(validate_dims(d));
  for (int64_t x = 0; x < d->na * d->nb; ++x)
    if (nmap[x] < 0 || nmap[x] >= d->na)
      return fail(SSE_EINVAL, "neighbor index %lld outside [0, %lld)", (long long)nmap[x], (long long)d->na);
  std::vector<int64_t> b;
  multi_bounds(d, nmap, (int)ctx->devs.size(), b);
  std::memcpy(bounds, b.data(), b.size() * sizeof(int64_t));
  return SSE_OK;
}

int sse_sigma_multi(sse_ctx* ctx, const sse_dims* d, double* const* G_l, double* const* G_g,
                    const double* const* Dc_l, const double* const* Dc_g, const double* const* dH,
                    const int64_t* nmap, const int64_t* off, const double* wt, double* const* Sig_l,
                    double* const* Sig_g, sse_timing* t) {
  if (!ctx || ctx->devs.empty()) return fail(SSE_EINVAL, "context is NULL");
  CHECK(validate_dims(d));
  CHECK(validate_grid(d, off, wt));
  if (!G_l || !G_g || !Dc_l || !Dc_g || !dH || !nmap || !Sig_l || !Sig_g) return fail(SSE_EINVAL, "NULL tensor pointer");
  const int nd = (int)ctx->devs.size();
  for (int64_t x = 0; x < d->na * d->nb; ++x)
    if (nmap[x] < 0 || nmap[x] >= d->na)
      return fail(SSE_EINVAL, "neighbor index %lld outside [0, %lld)", (long long)nmap[x], (long long)d->na);
  std::vector<int64_t> b;
  multi_bounds(d, nmap, nd, b);
  for (int i = 0; i < nd; ++i)  // devices that own no atom (NA < n_gpus * chunk) may pass NULL
    if (b[4 * i + 1] > b[4 * i] &&
        (!G_l[i] || !G_g[i] || !Dc_l[i] || !Dc_g[i] || !dH[i] || !Sig_l[i] || !Sig_g[i]))
      return fail(SSE_EINVAL, "NULL tensor pointer for device %d", i);
  const int64_t per = (d->na + nd - 1) / nd;
  const size_t blk = (size_t)d->nkz * d->ne * d->norb * d->norb * 16;  // bytes per atom and polarity
  // 1. halo exchange: every device receives its halo atoms from their owners (NCCL over NVLink)
  if (nd > 1) {
    NcclApi& nc = nccl_api();
    if (!nc.ok) return fail(SSE_ECOMM, "NCCL (libnccl.so.2) could not be loaded");
    if (ctx->comms.empty()) {
      std::vector<int> devlist(nd);
      for (int i = 0; i < nd; ++i) devlist[i] = ctx->devs[i].device;
      ctx->comms.assign(nd, nullptr);
      NC(nc.CommInitAll(ctx->comms.data(), nd, devlist.data()));
    }
    for (int i = 0; i < nd; ++i) {  // the previous call's use of the slabs / scratch is ordered first
      CU(cudaSetDevice(ctx->devs[i].device));
      CHECK(scratch_enter(ctx->devs[i], ctx->devs[i].stream));
    }
    double* const* Gp[2] = {G_l, G_g};
    NC(nc.GroupStart());
    for (int i = 0; i < nd; ++i) {
      const int64_t lo = b[4 * i], hi = b[4 * i + 1], glo = b[4 * i + 2], ghi = b[4 * i + 3];
      for (int64_t a0 = glo; a0 < ghi;) {
        if (a0 >= lo && a0 < hi) {
          a0 = hi;
          continue;
        }
        const int j = (int)(a0 / per);
        int64_t a1 = std::min<int64_t>(a0 < lo ? lo : ghi, std::min<int64_t>((j + 1) * per, d->na));
        const int64_t jglo = b[4 * j + 2];
        for (int pol = 0; pol < 2; ++pol) {
          NC(nc.Recv((char*)Gp[pol][i] + (a0 - glo) * blk, (a1 - a0) * blk, ncclChar, j, ctx->comms[i],
                     ctx->devs[i].stream));
          NC(nc.Send((const char*)Gp[pol][j] + (a0 - jglo) * blk, (a1 - a0) * blk, ncclChar, i, ctx->comms[j],
                     ctx->devs[j].stream));
        }
        a0 = a1;
      }
    }
    NC(nc.GroupEnd());
  }
  // 2. Sigma of each device's owned atoms on its own stream (all devices run concurrently)
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->flops = alg_flops(d, off, d->na);
    t->n_devices = nd;
  }
  int launches = 0;
  for (int i = 0; i < nd; ++i) {
    DevState& ds = ctx->devs[i];
    CU(cudaSetDevice(ds.device));
    cudaStream_t st = ds.stream;
    if (nd == 1) CHECK(scratch_enter(ds, st));
    if (t) CU(cudaEventRecord(ds.ev[0], st));
    const int64_t lo = b[4 * i], hi = b[4 * i + 1], glo = b[4 * i + 2], ghi = b[4 * i + 3];
    if (hi <= lo) continue;
    const sse_slab gs{glo, ghi - glo, 1, 0}, os{lo, hi - lo, 1, 0};
    const DevPtrs p{(const double2*)G_l[i], (const double2*)G_g[i], (const double2*)Dc_l[i], (const double2*)Dc_g[i],
                    (const double2*)dH[i], (double2*)Sig_l[i], (double2*)Sig_g[i]};
    CHECK(sigma_on_device(ds, d, gs, os, p, nmap + lo * d->nb, off, wt, st, &launches));
    CHECK(scratch_leave(ds, st));
    if (t) CU(cudaEventRecord(ds.ev[1], st));
  }
  if (t) {
    for (int i = 0; i < nd; ++i) {
      DevState& ds = ctx->devs[i];
      if (b[4 * i + 1] <= b[4 * i]) continue;
      CU(cudaSetDevice(ds.device));
      CU(cudaEventSynchronize(ds.ev[1]));
      t->total_ms = std::max(t->total_ms, (double)elapsed(ds.ev[0], ds.ev[1]));
    }
    t->sigma_ms = t->total_ms;
    t->kernel_launches = launches;
  }
  return SSE_OK;
}

int sse_pi_device(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out,
                  const double* G_l, const double* G_g, const double* dH, const int64_t* nmap,
                  const int64_t* off, double energy_weight, const unsigned char* mask, double* Pi_l,
                  double* Pi_g, void* stream, sse_timing* t) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device call needs a 1-device context");
  CHECK(validate_dims(d));
  CHECK(validate_offsets(d, off, energy_weight));
  CHECK(validate_slab(d, g, "G"));
  CHECK(validate_slab(d, out, "output"));
  if (!G_l || !G_g || !dH || !nmap || !Pi_l || !Pi_g) return fail(SSE_EINVAL, "NULL tensor pointer");
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->n_devices = 1;
    CU(cudaEventRecord(ds.ev[0], st));
  }
  int launches = 0;
  CHECK(scratch_enter(ds, st));
  CHECK(pi_on_device(ds, d, *g, *out, (const double2*)G_l, (const double2*)G_g, (const double2*)dH, nmap,
                     off, energy_weight, mask, (double2*)Pi_l, (double2*)Pi_g, st, &launches));
  CHECK(scratch_leave(ds, st));
  if (t) {
    CU(cudaEventRecord(ds.ev[1], st));
    CU(cudaEventSynchronize(ds.ev[1]));
    t->sigma_ms = t->total_ms = elapsed(ds.ev[0], ds.ev[1]);
    t->kernel_launches = launches;
  }
  return SSE_OK;
}

int sse_pi_c128(sse_ctx* ctx, const sse_dims* d, const double* G_l, const double* G_g, const double* dH,
                const int64_t* nmap, const int64_t* off, double energy_weight, const unsigned char* mask,
                int64_t atom_lo, int64_t atom_hi, double* Pi_l, double* Pi_g, sse_timing* t) {
  if (!ctx) return fail(SSE_EINVAL, "context is NULL");
  CHECK(validate_dims(d));
  if (atom_lo < 0 || atom_hi > d->na || atom_lo > atom_hi) return fail(SSE_EINVAL, "invalid atom range");
  if (!G_l || !G_g || !dH || !nmap || !Pi_l || !Pi_g || !off) return fail(SSE_EINVAL, "NULL tensor pointer");
  CHECK(validate_offsets(d, off, energy_weight));
  if (t) std::memset(t, 0, sizeof(*t));
  if (atom_lo == atom_hi) return SSE_OK;
  const int nd = (int)ctx->devs.size();
  const int64_t span = atom_hi - atom_lo, per = (span + nd - 1) / nd;
  const size_t blk = (size_t)d->norb * d->norb * 16, rows = (size_t)(d->nkz * d->ne);
  const size_t dh_atom = (size_t)d->nb * 3 * blk;
  const size_t pi_row = (size_t)(d->nb + 1) * 9 * 16, pi_rows = (size_t)(d->nqz * d->nw);
  auto on_device = [&](DevState& ds, int64_t lo, int64_t hi, sse_timing* tt) -> int {
    const int64_t on = hi - lo;
    if (on <= 0) return SSE_OK;
    CU(cudaSetDevice(ds.device));
    int64_t glo = lo, ghi = hi;
    for (int64_t i = lo * d->nb; i < hi * d->nb; ++i) {
      if (nmap[i] < 0 || nmap[i] >= d->na)
        return fail(SSE_EINVAL, "neighbor index %lld outside [0, %lld)", (long long)nmap[i], (long long)d->na);
      glo = std::min(glo, nmap[i]);
      ghi = std::max(ghi, nmap[i] + 1);
    }
    const int64_t gn = ghi - glo;
    cudaStream_t st = ds.stream;
    for (int p = 0; p < 2; ++p) {
      CHECK(ds.g[p].ensure(rows * gn * blk));
      CHECK(ds.pi_out[p].ensure(pi_rows * on * pi_row));
    }
    CHECK(ds.dh.ensure(on * dh_atom));
    CU(cudaEventRecord(ds.ev[0], st));
    const char* Gh[2] = {(const char*)G_l, (const char*)G_g};
    CU(cudaMemcpyAsync(ds.dh.ptr, (const char*)dH + lo * dh_atom, on * dh_atom, cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(ds.ev[2], st));
    CU(cudaStreamWaitEvent(ds.s_h2d, ds.ev[2], 0));
    // G columns are uploaded progressively on the copy stream: atom chunk [a0, a0 + n) waits only
    // for the columns it reads (its atoms and their neighbours), the rest streams under the kernels
    int64_t copied = glo;
    size_t ei = 0;
    auto before_chunk = [&](int64_t a0, int64_t n) -> int {
      int64_t need = std::max<int64_t>(copied, lo + a0 + n);
      for (int64_t i = (lo + a0) * d->nb; i < (lo + a0 + n) * d->nb; ++i) need = std::max(need, nmap[i] + 1);
      if (need > copied) {
        for (int p = 0; p < 2; ++p)
          CU(cudaMemcpy2DAsync((char*)ds.g[p].ptr + (copied - glo) * blk, gn * blk, Gh[p] + copied * blk,
                               d->na * blk, (need - copied) * blk, rows, cudaMemcpyHostToDevice, ds.s_h2d));
        copied = need;
      }
      cudaEvent_t in = pipe_event(ds, ei++);
      if (!in) return fail(SSE_ECUDA, "event creation failed");
      CU(cudaEventRecord(in, ds.s_h2d));
      CU(cudaStreamWaitEvent(st, in, 0));
      return SSE_OK;
    };
    int launches = 0;
    const sse_slab gs{glo, gn, 0, 0}, os{lo, on, 0, 0};
    double* const Ph[2] = {Pi_l, Pi_g};
    auto after_chunk = [&](int64_t a0, int64_t n) { return pi_chunk_to_host(ds, d, lo, on, a0, n, Ph, st, &ei); };
    CHECK(pi_on_device(ds, d, gs, os, ds.g[0].as<double2>(), ds.g[1].as<double2>(), ds.dh.as<double2>(),
                       nmap + lo * d->nb, off, energy_weight, mask, ds.pi_out[0].as<double2>(),
                       ds.pi_out[1].as<double2>(), st, &launches, nullptr, before_chunk, after_chunk));
    CHECK(join_d2h(ds, st, &ei));
    CU(cudaEventRecord(ds.ev[1], st));
    CU(cudaEventSynchronize(ds.ev[1]));
    if (tt) {
      tt->total_ms = std::max(tt->total_ms, (double)elapsed(ds.ev[0], ds.ev[1]));
      tt->h2d_bytes += 2 * rows * gn * blk + on * dh_atom;
      tt->d2h_bytes += 2 * pi_rows * on * pi_row;
      tt->kernel_launches += launches;
    }
    return SSE_OK;
  };
  auto run_dev = [&](DevState& ds, int64_t lo, int64_t hi, sse_timing* tt) {
    return guarded(ds, [&] { return on_device(ds, lo, hi, tt); });
  };
  if (nd == 1) return run_dev(ctx->devs[0], atom_lo, atom_hi, t);
  std::vector<int> rcs(nd, SSE_OK);
  std::vector<sse_timing> ts(nd);
  std::vector<std::string> errs(nd);
  std::vector<std::thread> th;
  for (int i = 0; i < nd; ++i)
    th.emplace_back([&, i] {
      std::memset(&ts[i], 0, sizeof(sse_timing));
      const int64_t lo = atom_lo + std::min<int64_t>(i * per, span), hi = atom_lo + std::min<int64_t>((i + 1) * per, span);
      rcs[i] = run_dev(ctx->devs[i], lo, hi, &ts[i]);
      if (rcs[i] != SSE_OK) errs[i] = g_last_error;
    });
  for (auto& x : th) x.join();
  for (int i = 0; i < nd; ++i) {
    if (rcs[i] != SSE_OK) {
      g_last_error = errs[i];
      return rcs[i];
    }
    if (t) {
      t->total_ms = std::max(t->total_ms, ts[i].total_ms);
      t->h2d_bytes += ts[i].h2d_bytes;
      t->d2h_bytes += ts[i].d2h_bytes;
      t->kernel_launches += ts[i].kernel_launches;
      t->h2d_ms = std::max(t->h2d_ms, ts[i].h2d_ms);
      t->d2h_ms = std::max(t->d2h_ms, ts[i].d2h_ms);
      t->staged |= ts[i].staged;
      t->host_threads = std::max(t->host_threads, ts[i].host_threads);
    }
  }
  return SSE_OK;
}

// SSE phase of one Born iteration (sse.py:532-534) in one call: G^<> and raw
// D^<> uploaded once, preprocess_D on the device, Sigma (pipelined chunks, G
// kept resident) then Pi on the same G, both results downloaded.
int sse_phase_c128(sse_ctx* ctx, const sse_dims* d, const double* G_l, const double* G_g, const double* D_l,
                   const double* D_g, const double* dH, const int64_t* nmap, const int64_t* off, const double* wt,
                   double energy_weight, double* Sig_l, double* Sig_g, double* Pi_l, double* Pi_g,
                   sse_timing* t) {
  if (!ctx) return fail(SSE_EINVAL, "context is NULL");
  CHECK(validate_dims(d));
  CHECK(validate_grid(d, off, wt));
  if (!G_l || !G_g || !D_l || !D_g || !dH || !nmap || !Sig_l || !Sig_g || !Pi_l || !Pi_g)
    return fail(SSE_EINVAL, "NULL tensor pointer");
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->flops = alg_flops(d, off, d->na);
  }
  const int nd = (int)ctx->devs.size();
  if (t) t->n_devices = nd;
  const int64_t per = (d->na + nd - 1) / nd;
  const size_t d_row = (size_t)(d->nb + 1) * 9 * 16, d_rows = (size_t)(d->nqz * d->nw);
  const size_t dc_row = (size_t)d->nb * 9 * 16;
  const size_t pi_row = d_row, pi_rows = d_rows;
  const sse_slab full{0, d->na, 0, 0};
  auto on_device = [&](DevState& ds, int64_t lo, int64_t hi, sse_timing* tt) -> int {
    const int64_t on = hi - lo;
    if (on <= 0) return SSE_OK;
    CU(cudaSetDevice(ds.device));
    int64_t glo = lo, ghi = hi;
    for (int64_t i = lo * d->nb; i < hi * d->nb; ++i) {
      if (nmap[i] < 0 || nmap[i] >= d->na)
        return fail(SSE_EINVAL, "neighbor index %lld outside [0, %lld)", (long long)nmap[i], (long long)d->na);
      glo = std::min(glo, nmap[i]);
      ghi = std::max(ghi, nmap[i] + 1);
    }
    const int64_t gn = ghi - glo;
    cudaStream_t st = ds.stream;
    cudaEvent_t e0 = ds.ev[4], e1 = ds.ev[5];  // ev[0..3] belong to the Sigma host call below
    CU(cudaEventRecord(e0, st));
    // raw D of the G slab's atoms, then Dc of the owned atoms (sse.py:105-113)
    std::vector<int> nbr, rev;
    CHECK(preprocess_tables(nmap, d->na, d->nb, glo, gn, lo, on, nbr, rev));
    const char* Dh[2] = {(const char*)D_l, (const char*)D_g};
    for (int p = 0; p < 2; ++p) {
      CHECK(ds.draw[p].ensure(d_rows * gn * d_row));
      CHECK(ds.dc[p].ensure(d_rows * on * dc_row));
      CU(cudaMemcpy2DAsync(ds.draw[p].ptr, gn * d_row, Dh[p] + glo * d_row, d->na * d_row, gn * d_row, d_rows,
                           cudaMemcpyHostToDevice, st));
    }
    CHECK(upload_cached(ds.pp_nbr, ds.pp_nbr_host, nbr, st));
    CHECK(upload_cached(ds.pp_rev, ds.pp_rev_host, rev, st));
    for (int p = 0; p < 2; ++p)
      CHECK(profiled(ds, st, SSE_PROF_PREPROCESS, 0.0, [&] {
        return sse::launch_preprocess_D(d->nqz, d->nw, gn, glo, lo, on, d->nb, ds.pp_nbr.as<int>(),
                                        ds.pp_rev.as<int>(), ds.draw[p].as<double2>(), ds.dc[p].as<double2>(),
                                        st);
      }));
    // Sigma: the pipelined host call with Dc resident; leaves the G slab in ds.g
    HostCall c{d, SSE_VARIANT_BATCHED_FUSED, full, full, G_l, G_g, nullptr, nullptr, dH, nmap, off, wt, Sig_l, Sig_g};
    c.dc_resident = true;
    sse_timing ts{};
    CHECK(host_call_on_device(ds, c, lo, hi, &ts));
    // Pi on the resident G slab and owned dH
    int launches = ts.kernel_launches + 2;
    for (int p = 0; p < 2; ++p) CHECK(ds.pi_out[p].ensure(pi_rows * on * pi_row));
    const sse_slab gs{glo, gn, 0, 0}, os{lo, on, 0, 0};
    double* const Ph[2] = {Pi_l, Pi_g};
    size_t ei = 0;
    auto after_chunk = [&](int64_t a0, int64_t n) { return pi_chunk_to_host(ds, d, lo, on, a0, n, Ph, st, &ei); };
    CHECK(pi_on_device(ds, d, gs, os, ds.g[0].as<double2>(), ds.g[1].as<double2>(), ds.dh.as<double2>(),
                       nmap + lo * d->nb, off, energy_weight, nullptr, ds.pi_out[0].as<double2>(),
                       ds.pi_out[1].as<double2>(), st, &launches, nullptr, nullptr, after_chunk));
    CHECK(join_d2h(ds, st, &ei));
    CU(cudaEventRecord(e1, st));
    CU(cudaEventSynchronize(e1));
    if (tt) {
      tt->total_ms = std::max(tt->total_ms, (double)elapsed(e0, e1));
      tt->h2d_ms += ts.h2d_ms;
      tt->d2h_ms += ts.d2h_ms;
      tt->staged |= ts.staged;
      tt->host_threads = ts.host_threads;
      tt->h2d_bytes += ts.h2d_bytes + 2 * d_rows * gn * d_row;
      tt->d2h_bytes += ts.d2h_bytes + 2 * pi_rows * on * pi_row;
      tt->kernel_launches += launches;
    }
    return SSE_OK;
  };
  auto run_dev = [&](DevState& ds, int64_t lo, int64_t hi, sse_timing* tt) {
    return guarded(ds, [&] { return on_device(ds, lo, hi, tt); });
  };
  if (nd == 1) return run_dev(ctx->devs[0], 0, d->na, t);
  std::vector<int> rcs(nd, SSE_OK);
  std::vector<sse_timing> ts(nd);
  std::vector<std::string> errs(nd);
  std::vector<std::thread> th;
  for (int i = 0; i < nd; ++i)
    th.emplace_back([&, i] {
      std::memset(&ts[i], 0, sizeof(sse_timing));
      const int64_t lo = std::min<int64_t>(i * per, d->na), hi = std::min<int64_t>((i + 1) * per, d->na);
      rcs[i] = run_dev(ctx->devs[i], lo, hi, &ts[i]);
      if (rcs[i] != SSE_OK) errs[i] = g_last_error;
    });
  for (auto& x : th) x.join();
  for (int i = 0; i < nd; ++i) {
    if (rcs[i] != SSE_OK) {
      g_last_error = errs[i];
      return rcs[i];
    }
    if (t) {
      t->total_ms = std::max(t->total_ms, ts[i].total_ms);
      t->h2d_bytes += ts[i].h2d_bytes;
      t->d2h_bytes += ts[i].d2h_bytes;
      t->kernel_launches += ts[i].kernel_launches;
      t->h2d_ms = std::max(t->h2d_ms, ts[i].h2d_ms);
      t->d2h_ms = std::max(t->d2h_ms, ts[i].d2h_ms);
      t->staged |= ts[i].staged;
      t->host_threads = std::max(t->host_threads, ts[i].host_threads);
    }
  }
  return SSE_OK;
}

// SSE phase of one Born iteration (sse.py:532-534) on device-resident tensors of one
// rank: preprocess_D of the owned atoms from the raw D slab, Sigma and Pi from the G slab;
// nothing crosses the host link.  g: G / raw-D slab (owned atoms + every neighbour), out: owned.
int sse_phase_device(sse_ctx* ctx, const sse_dims* d, const sse_slab* g, const sse_slab* out, const double* G_l,
                     const double* G_g, const double* D_l, const double* D_g, const double* dH, const int64_t* nmap,
                     const int64_t* off, const double* wt, double energy_weight, double* Sig_l, double* Sig_g,
                     double* Pi_l, double* Pi_g, void* stream, sse_timing* t) {
  if (!ctx || ctx->devs.size() != 1) return fail(SSE_EINVAL, "device call needs a 1-device context");
  CHECK(validate_dims(d));
  CHECK(validate_grid(d, off, wt));
  CHECK(validate_offsets(d, off, energy_weight));
  CHECK(validate_slab(d, g, "G"));
  CHECK(validate_slab(d, out, "output"));
  if (!G_l || !G_g || !D_l || !D_g || !dH || !nmap || !Sig_l || !Sig_g || !Pi_l || !Pi_g)
    return fail(SSE_EINVAL, "NULL tensor pointer");
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  std::vector<int> nbr, rev;
  CHECK(preprocess_tables(nmap, d->na, d->nb, g->atom0, g->natoms, out->atom0, out->natoms, nbr, rev));
  if (t) {
    std::memset(t, 0, sizeof(*t));
    t->flops = alg_flops(d, off, out->natoms);
    t->n_devices = 1;
    CU(cudaEventRecord(ds.ev[0], st));
  }
  CHECK(scratch_enter(ds, st));
  const size_t dc_bytes = (size_t)(d->nqz * d->nw) * out->natoms * d->nb * 9 * 16;
  for (int p = 0; p < 2; ++p) CHECK(ds.dc[p].ensure(dc_bytes));
  CHECK(upload_cached(ds.pp_nbr, ds.pp_nbr_host, nbr, st));
  CHECK(upload_cached(ds.pp_rev, ds.pp_rev_host, rev, st));
  const double* Dr[2] = {D_l, D_g};
  for (int p = 0; p < 2; ++p)
    CHECK(profiled(ds, st, SSE_PROF_PREPROCESS, 0.0, [&] {
      return sse::launch_preprocess_D(d->nqz, d->nw, g->natoms, g->atom0, out->atom0, out->natoms, d->nb,
                                      ds.pp_nbr.as<int>(), ds.pp_rev.as<int>(), (const double2*)Dr[p],
                                      ds.dc[p].as<double2>(), st);
    }));
  int launches = 2;
  const int64_t* rows = nmap + out->atom0 * d->nb;
  const DevPtrs p{(const double2*)G_l, (const double2*)G_g, ds.dc[0].as<double2>(), ds.dc[1].as<double2>(),
                  (const double2*)dH, (double2*)Sig_l, (double2*)Sig_g};
  CHECK(sigma_on_device(ds, d, *g, *out, p, rows, off, wt, st, &launches));
  CHECK(pi_on_device(ds, d, *g, *out, (const double2*)G_l, (const double2*)G_g, (const double2*)dH, rows, off,
                     energy_weight, nullptr, (double2*)Pi_l, (double2*)Pi_g, st, &launches));
  CHECK(scratch_leave(ds, st));
  if (t) {
    CU(cudaEventRecord(ds.ev[1], st));
    CU(cudaEventSynchronize(ds.ev[1]));
    t->total_ms = elapsed(ds.ev[0], ds.ev[1]);
    t->kernel_launches = launches;
  }
  return SSE_OK;
}

int sse_layout_transform(sse_ctx* ctx, int64_t nkz, int64_t ne, int64_t na, int64_t block_doubles,
                         int to_atom_major, const double* src, double* dst, void* stream) {
  if (!ctx || ctx->devs.empty()) return fail(SSE_EINVAL, "context is NULL");
  if (nkz < 1 || ne < 1 || na < 1 || block_doubles < 2 || block_doubles % 2)
    return fail(SSE_EINVAL, "invalid layout-transform shape");
  if (!src || !dst || src == dst) return fail(SSE_EINVAL, "layout transform needs distinct buffers");
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  CHECK(profiled(ds, st, SSE_PROF_LAYOUT, 0.0, [&] {
    return sse::launch_layout_transform(nkz, ne, na, block_doubles / 2, to_atom_major,
                                        (const double2*)src, (double2*)dst, st);
  }));
  if (!stream) CU(cudaStreamSynchronize(st));
  return SSE_OK;
}

int sse_preprocess_D(sse_ctx* ctx, int64_t nqz, int64_t nw, int64_t na, int64_t nb,
                     const int64_t* nmap, int64_t d_atom0, int64_t d_natoms, int64_t out_atom0,
                     int64_t out_natoms, const double* D, double* Dc, void* stream) {
  if (!ctx || ctx->devs.empty()) return fail(SSE_EINVAL, "context is NULL");
  if (nqz < 1 || nw < 1 || na < 1 || nb < 1 || !nmap || !D || !Dc || d_natoms < 1 ||
      out_natoms < 1 || d_atom0 < 0 || out_atom0 < 0 || d_atom0 + d_natoms > na ||
      out_atom0 + out_natoms > na)
    return fail(SSE_EINVAL, "invalid preprocess_D arguments");
  std::vector<int> nbr, rev;
  CHECK(preprocess_tables(nmap, na, nb, d_atom0, d_natoms, out_atom0, out_natoms, nbr, rev));
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  CHECK(scratch_enter(ds, st));
  CHECK(upload_cached(ds.pp_nbr, ds.pp_nbr_host, nbr, st));
  CHECK(upload_cached(ds.pp_rev, ds.pp_rev_host, rev, st));
  CHECK(profiled(ds, st, SSE_PROF_PREPROCESS, 0.0, [&] {
    return sse::launch_preprocess_D(nqz, nw, d_natoms, d_atom0, out_atom0, out_natoms, nb,
                                    ds.pp_nbr.as<int>(), ds.pp_rev.as<int>(), (const double2*)D,
                                    (double2*)Dc, st);
  }));
  CHECK(scratch_leave(ds, st));
  if (!stream) CU(cudaStreamSynchronize(st));
  return SSE_OK;
}

int sse_fill_synthetic(sse_ctx* ctx, uint64_t seed, uint32_t tensor_id, int64_t atom0,
                       int64_t natoms, int64_t outer, int64_t inner, int64_t atom_stride,
                       int64_t outer_stride, double scale, double* dst, void* stream) {
  if (!ctx || ctx->devs.empty()) return fail(SSE_EINVAL, "context is NULL");
  if (atom0 < 0 || natoms < 0 || outer < 1 || inner < 1 || !dst)
    return fail(SSE_EINVAL, "invalid fill arguments");
  if (natoms == 0) return SSE_OK;
  DevState& ds = ctx->devs[0];
  CU(cudaSetDevice(ds.device));
  cudaStream_t st = stream ? (cudaStream_t)stream : ds.stream;
  CU(sse::launch_fill_synthetic(seed, tensor_id, atom0, natoms, outer, inner, atom_stride,
                                outer_stride, scale, (double2*)dst, st));
  if (!stream) CU(cudaStreamSynchronize(st));
  return SSE_OK;
}

const char* sse_kernel_name(int kind) { return sse::last_kernel_name(kind); }

int sse_profile_begin(sse_ctx* ctx) {
  if (!ctx) return fail(SSE_EINVAL, "context is NULL");
  for (auto& ds : ctx->devs) {
    ds.profiling = true;
    ds.pool_used = 0;
    ds.recs.clear();
  }
  return SSE_OK;
}

int sse_profile_end(sse_ctx* ctx, sse_profile* out) {
  if (!ctx || !out) return fail(SSE_EINVAL, "NULL argument");
  std::memset(out, 0, sizeof(*out));
  for (auto& ds : ctx->devs) {
    CU(cudaSetDevice(ds.device));
    for (const ProfRec& r : ds.recs) {
      CU(cudaEventSynchronize(r.b));
      out->ms[r.kind] += elapsed(r.a, r.b);
      out->launches[r.kind] += 1;
      out->flops[r.kind] += r.flops;
    }
    ds.profiling = false;
    ds.recs.clear();
    ds.pool_used = 0;
  }
  return SSE_OK;
}

}  // extern "C"
