// C ABI of the B200 lattice-sum hot path: context, device-resident handles and the
// orchestration of the four FP64 stages.  Internally C++ with
// exceptions; every extern "C" entry point catches, records latsum_last_error and
// returns a status code (the reference's exception types map to LATSUM_ERR_*).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <numeric>
#include <set>
#include <stdexcept>
#include <exception>
#include <fstream>
#include <condition_variable>
#include <functional>
#include <future>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "dgemm_dmma.cuh"
#include "latsum_b200.h"
#include "latsum_kernels.cuh"
#include "ozaki_i8.cuh"
#include "eig_sym.cuh"
#include "eig_band.cuh"

using namespace latsum_b200;

namespace {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw Error(e_ == cudaErrorMemoryAllocation ? LATSUM_ERR_OUT_OF_MEMORY             \
                                                  : LATSUM_ERR_CUDA,                     \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

#define CS(call)                                                                          \
  do {                                                                                    \
    cusolverStatus_t s_ = (call);                                                         \
    if (s_ != CUSOLVER_STATUS_SUCCESS)                                                    \
      throw Error(LATSUM_ERR_CUSOLVER, std::string(#call) + ": status " + std::to_string(int(s_))); \
  } while (0)

void require(bool ok, const std::string& msg) {
  if (!ok) throw Error(LATSUM_ERR_INVALID_ARGUMENT, msg);
}

// ---- NCCL, bound at run time (dlopen) so the process shares whichever libnccl.so.2
// torch already loaded; only the symbols the sharded path needs.
typedef struct ncclComm* ncclComm_t;
struct NcclUid { char internal[128]; };
enum { kNcclFloat64 = 8, kNcclSum = 0 };
struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUid, int) = nullptr;
  int (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) x.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!x.h) return x;
    x.GetUniqueId = reinterpret_cast<decltype(x.GetUniqueId)>(dlsym(x.h, "ncclGetUniqueId"));
    x.CommInitRank = reinterpret_cast<decltype(x.CommInitRank)>(dlsym(x.h, "ncclCommInitRank"));
    x.CommSplit = reinterpret_cast<decltype(x.CommSplit)>(dlsym(x.h, "ncclCommSplit"));
    x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(dlsym(x.h, "ncclCommDestroy"));
    x.AllReduce = reinterpret_cast<decltype(x.AllReduce)>(dlsym(x.h, "ncclAllReduce"));
    x.AllGather = reinterpret_cast<decltype(x.AllGather)>(dlsym(x.h, "ncclAllGather"));
    x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(dlsym(x.h, "ncclGetErrorString"));
    return x;
  }();
  if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.CommSplit || !n.AllReduce || !n.AllGather)
    throw Error(LATSUM_ERR_NCCL, "libnccl.so.2 not found or incomplete");
  return n;
}
#define NC(call)                                                                         \
  do {                                                                                   \
    int r_ = (call);                                                                     \
    if (r_ != 0)                                                                         \
      throw Error(LATSUM_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

}  // namespace

struct latsum_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own = nullptr;
  cusolverDnHandle_t solver = nullptr;
  cusolverDnParams_t solver_params = nullptr;
  std::string err;
  int64_t launches = 0;
  bool smem_set = false;
  bool oz_smem_set = false;
  int64_t eig_fallbacks = 0;  // in-house eigensolves redone with syevd (degenerate clusters)
  int eig_method = 0;         // Eig::solve default method (0: LATSUM_EIG / size rule, 1: syevd)
  // optional per-kernel-class CUDA-event timing (latsum_ctx_set_profiling)
  bool prof = false;
  struct Rec { std::string tag; cudaEvent_t a, b; double work; };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  struct Stat { int64_t count = 0; double ms = 0.0, work = 0.0; };
  std::map<std::string, Stat> stats;
  // worker contexts (own stream + cuSOLVER handle) for the concurrent per-mode reductions
  latsum_ctx* sub[4] = {nullptr, nullptr, nullptr, nullptr};
  latsum_ctx* parent = nullptr;  // set on worker contexts
  // cap on the CTAs of this context's persistent kernels (Ozaki GEMM): a persistent grid on
  // every SM holds them until it finishes, whatever the stream priorities; the low-priority
  // norm worker keeps to a few SMs so the mode workers' kernels are never queued behind it
  int max_ctas = 0;
  // assembled_vector's accumulation order (lattice_sum.hpp:28-35): 0 sliding (the reference's
  // default: the recursion wherever the reference would use it), 1 ascending (always direct)
  int accumulation = 0;
  // SMs a capped worker's persistent kernels are holding right now (set on the ROOT context by
  // that worker): the other contexts' persistent GEMMs size their grids to the SMs left, since
  // their static tile partition would otherwise wait for the CTAs that cannot be placed until
  // the capped kernel ends (cfg5: ~80 ms per norm_f Gram launch, on every mode-side GEMM)
  std::atomic<int> reserved_ctas{0};
  // multi-GPU: one rank of a row-sharded reduction (latsum_ctx_init_comm); each worker
  // context owns a communicator split from this one so concurrent modes never interleave
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  // host collective (latsum_ctx_init_host_comm): the same collectives through caller
  // callbacks on host buffers (gloo / in-process ranks in tests); channel 0 is this
  // context, 1..4 its workers (so concurrent modes never interleave on one channel)
  // host sink (latsum_ctx_set_host_sink): the next Tucker results stream here while formed
  struct Sink {
    double* core = nullptr;
    int64_t core_cap = 0;
    double* f[3] = {nullptr, nullptr, nullptr};
    int64_t f_cap[3] = {0, 0, 0};
    cudaStream_t copy = nullptr, copy2 = nullptr;  // two copy engines
  } sink;
  latsum_host_allreduce_fn host_ar = nullptr;
  latsum_host_allgather_fn host_ag = nullptr;
  void* host_user = nullptr;
  int channel = 0;
};

// a row-sharded reduction runs over NCCL or the host callbacks
inline bool has_comm(const latsum_ctx* c) { return (c->comm || c->host_ar) && c->nranks > 1; }

namespace {

// Stream-ordered device buffer owned by a context's stream.
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(latsum_ctx* c, size_t count) { alloc(c, count); }
  void alloc(latsum_ctx* c, size_t count) {
    release();
    s = c->stream;
    n = count;
    if (count) CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(double), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  // hand the buffer to another stream (caller guarantees the streams are ordered)
  void adopt(cudaStream_t st) { s = st; }
  DBuf& operator=(DBuf&& o) noexcept {
    release();
    p = o.p; n = o.n; s = o.s;
    o.p = nullptr; o.n = 0;
    return *this;
  }
};

template <typename T>
struct DVec {  // small device array of T
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DVec() = default;
  void upload(latsum_ctx* c, const std::vector<T>& h) {
    release();
    s = c->stream;
    n = h.size();
    if (n) {
      CK(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), s));
      CK(cudaMemcpyAsync(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DVec() { release(); }
};

int grid_for(int64_t total, int threads = 256) {
  int64_t b = (total + threads - 1) / threads;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

// Doubles an intermediate may occupy: 1/16 of the device memory (11 GB on a B200),
// fixed per device so chunk sizes (and stream-ordered pool reuse) are reproducible.
int64_t workspace_budget() {
  static const int64_t v = [] {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return int64_t(1) << 27;
    return std::max<int64_t>(int64_t(1) << 27, int64_t(total_b / 16 / sizeof(double)));
  }();
  return v;
}

// Split n into ceil(n / cap) near-equal chunks (multiples of `align` when possible).
int64_t balanced_chunk(int64_t n, int64_t cap, int64_t align) {
  cap = std::max<int64_t>(1, cap);
  if (n <= cap) return std::max<int64_t>(n, 1);
  const int64_t parts = (n + cap - 1) / cap;
  int64_t c = (n + parts - 1) / parts;
  if (align > 1 && c > align) c = std::min<int64_t>(cap, (c + align - 1) / align * align);
  return std::max<int64_t>(1, std::min(c, cap));
}

void post_launch(latsum_ctx* c) {
  c->launches++;
  CK(cudaGetLastError());
}

cudaEvent_t prof_event(latsum_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

// Records [start, stop] events around the launches in its scope when profiling is on;
// `work` is the algorithmic FLOPs or bytes the caller attributes to the scope.
struct ProfScope {
  latsum_ctx* c;
  bool on;
  latsum_ctx::Rec rec;
  ProfScope(latsum_ctx* ctx, const char* tag, double work = 0.0) : c(ctx), on(ctx->prof && tag) {
    if (!on) return;
    rec.tag = tag;
    rec.work = work;
    rec.a = prof_event(c);
    rec.b = prof_event(c);
    CK(cudaEventRecord(rec.a, c->stream));
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(rec.b, c->stream);
    c->pending.push_back(rec);
  }
};

void prof_harvest(latsum_ctx* c) {
  if (c->pending.empty()) return;
  CK(cudaStreamSynchronize(c->stream));
  for (auto& r : c->pending) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    auto& st = c->stats[r.tag];
    st.count += 1;
    st.ms += ms;
    st.work += r.work;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->pending.clear();
}

// LATSUM_TRACE=1: host wall-clock trace of the RHOSVD phases (stderr), per worker.
struct Trace {
  static bool on() {
    static const bool v = std::getenv("LATSUM_TRACE") != nullptr;
    return v;
  }
  static double now_ms() {
    using namespace std::chrono;
    static const auto t0 = steady_clock::now();
    return duration<double, std::milli>(steady_clock::now() - t0).count();
  }
  static void mark(latsum_ctx* c, const char* what, bool sync = true) {
    if (!on()) return;
    if (sync) cudaStreamSynchronize(c->stream);
    fprintf(stderr, "[trace %9.3f ms] stream %p %s\n", now_ms(), (void*)c->stream, what);
  }
};

// Sum-all-reduce over the ranks of c's communicator (no-op on one rank).
void allreduce(latsum_ctx* c, double* buf, size_t count) {
  if (!has_comm(c) || count == 0) return;
  if (c->comm) {
    NC(nccl().AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, c->comm, c->stream));
    return;
  }
  std::vector<double> h(count);
  CK(cudaMemcpyAsync(h.data(), buf, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->host_ar(c->host_user, c->channel, h.data(), int64_t(count)) != 0)
    throw Error(LATSUM_ERR_NCCL, "host all-reduce failed");
  CK(cudaMemcpyAsync(buf, h.data(), sizeof(double) * count, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// recv (nranks x count) = every rank's send (count), in rank order
void allgather(latsum_ctx* c, const double* send, double* recv, size_t count) {
  if (c->comm) {
    NC(nccl().AllGather(send, recv, count, kNcclFloat64, c->comm, c->stream));
    return;
  }
  std::vector<double> hs(count), hr(count * size_t(c->nranks));
  CK(cudaMemcpyAsync(hs.data(), send, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->host_ag(c->host_user, c->channel, hs.data(), hr.data(), int64_t(count)) != 0)
    throw Error(LATSUM_ERR_NCCL, "host all-gather failed");
  CK(cudaMemcpyAsync(recv, hr.data(), sizeof(double) * hr.size(), cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

// The rows [lo, hi) of an N-row operand this rank owns in the row-sharded reduction.
struct RowBlock {
  int64_t lo = 0, hi = 0;
  int64_t n() const { return hi - lo; }
};
RowBlock row_block(const latsum_ctx* c, int64_t N) {
  return {N * c->rank / c->nranks, N * (c->rank + 1) / c->nranks};
}

// cudaFuncSetAttribute applies to the current device only: the large-shared-memory /
// cluster opt-ins are made once per (kernel, device), under a lock (the RHOSVD worker
// threads reach them concurrently).
template <typename F>
void once_per_device(const latsum_ctx* c, const void* key, F&& set) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({key, c->device})) return;
  set();
  done.insert({key, c->device});
}

template <typename K>
void set_smem_attr(const latsum_ctx* c, K kernel, size_t bytes, bool cluster16 = false) {
  once_per_device(c, reinterpret_cast<const void*>(kernel), [&] {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    if (cluster16) CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
}

// ------------------------------------------------------------------ GEMM launcher
struct GemmOpts {
  int64_t batch = 1, sA = 0, sB = 0, sC = 0;
  const int64_t* kseg = nullptr;
  bool lower = false;
  int splits = 0;  // 0 = auto
  const char* tag = "gemm";
  bool dmma = false;  // keep on FP64 DMMA (products whose rounding sets a noise floor)
};

template <class Cfg>
void set_smem_cfg() {
  const int bytes = int(Cfg::SMEM_BYTES);
  CK(cudaFuncSetAttribute(dgemm_dmma_kernel<Cfg, false, false>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(dgemm_dmma_kernel<Cfg, false, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(dgemm_dmma_kernel<Cfg, true, false>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CK(cudaFuncSetAttribute(dgemm_dmma_kernel<Cfg, true, true>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

void set_gemm_smem(latsum_ctx* c) {
  if (c->smem_set) return;
  set_smem_cfg<CfgBig>();
  set_smem_cfg<CfgWide>();
  set_smem_cfg<CfgHalf>();
  set_smem_cfg<CfgDeep>();
  c->smem_set = true;
}

GemmOpts tagged(const char* tag) {
  GemmOpts o;
  o.tag = tag;
  return o;
}

// Tile configuration: LATSUM_GEMM_CFG=0..3 overrides (A/B measurements only).
int gemm_cfg_choice() {
  static int v = [] {
    const char* e = std::getenv("LATSUM_GEMM_CFG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

template <class Cfg>
void launch_gemm(latsum_ctx* c, bool ta, bool tb, GemmParams p, int64_t tm, int64_t tn) {
  dim3 grid(unsigned(tm), unsigned(tn), unsigned(p.batch * p.splits));
  const size_t sm = Cfg::SMEM_BYTES;
  const int th = Cfg::THREADS;
  if (!ta && !tb) dgemm_dmma_kernel<Cfg, false, false><<<grid, th, sm, c->stream>>>(p);
  if (!ta && tb) dgemm_dmma_kernel<Cfg, false, true><<<grid, th, sm, c->stream>>>(p);
  if (ta && !tb) dgemm_dmma_kernel<Cfg, true, false><<<grid, th, sm, c->stream>>>(p);
  if (ta && tb) dgemm_dmma_kernel<Cfg, true, true><<<grid, th, sm, c->stream>>>(p);
}

void ozaki_gemm_ex(latsum_ctx* c, int64_t M, int64_t N, int64_t K, const double* A, int64_t a_sl,
                   int64_t a_sk, int64_t a_L1, int64_t a_sl2, const double* B, int64_t b_sl,
                   int64_t b_sk, oz::OzOut o, const char* tag);

// Large single products (stage 3 of the big configs: Grams, deflation, bases, projections)
// run on the int8 tensor cores too (FP64-accurate Ozaki GEMM); LATSUM_GEMM_DMMA=1 keeps
// every generic GEMM on DMMA.  Small products stay on DMMA (slicing overhead).
bool gemm_to_ozaki(int64_t M, int64_t N, int64_t K) {
  static const bool dmma = std::getenv("LATSUM_GEMM_DMMA") != nullptr;
  return !dmma && double(M) * double(N) * double(K) >= 2e10 && K >= 64;
}

const char* ozaki_tag(const char* tag) {
  static std::map<std::string, std::string> names;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto& v = names[tag ? tag : "gemm"];
  if (v.empty()) v = std::string(tag ? tag : "gemm") + "(ozaki-i8)";
  return v.c_str();
}

void gemm(latsum_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
          const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
          int64_t ldc, GemmOpts o = {}) {
  if (M <= 0 || N <= 0 || o.batch <= 0) return;
  if (!o.kseg && o.batch == 1 && !o.dmma && gemm_to_ozaki(M, N, K)) {
    const oz::OzOut oo{C, ldc, int64_t(1) << 62, 0, int64_t(1) << 62, 0, beta, alpha};
    ozaki_gemm_ex(c, M, N, K, A, ta ? lda : 1, ta ? 1 : lda, 0, 0, B, tb ? 1 : ldb, tb ? ldb : 1, oo,
                  ozaki_tag(o.tag));  // lower-triangle requests get the full product
    return;
  }
  set_gemm_smem(c);
  const int choice = gemm_cfg_choice();
  const int BM = 128, BK = 16;
  const int BN = choice == 2 ? CfgHalf::BN : 128;
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  int splits = o.splits;
  if (splits == 0) {
    splits = 1;
    const int64_t tiles = tm * tn * o.batch;
    if (!o.kseg && tiles < 148 && K >= 8 * BK) {
      splits = int(std::min<int64_t>({(2 * 148 + tiles - 1) / tiles, K / (4 * BK), 16}));
      splits = std::max(splits, 1);
    }
  }
  require(tn <= 65535 && o.batch * splits <= 65535, "gemm: grid too large");
  GemmParams p{M, N, K, A, lda, o.sA, B, ldb, o.sB, C, ldc, o.sC, alpha, beta, o.batch, splits,
               o.kseg, o.lower ? 1 : 0};
  DBuf ws;
  if (splits > 1) {
    ws.alloc(c, size_t(splits) * M * N * o.batch);
    p.C = ws.p;
  }
  // algorithmic FLOPs (2 M N K per product; segmented: 2 M N sum(segments))
  double flops = o.kseg ? 2.0 * double(M) * double(N) * double(K)
                        : 2.0 * double(M) * double(N) * double(K) * double(o.batch);
  if (o.lower) flops = double(M) * double(M + 1) * double(K) * double(o.batch);  // SYRK
  ProfScope ps(c, o.tag, flops);
  switch (choice) {
    case 1: launch_gemm<CfgWide>(c, ta, tb, p, tm, tn); break;
    case 2: launch_gemm<CfgHalf>(c, ta, tb, p, tm, tn); break;
    case 3: launch_gemm<CfgDeep>(c, ta, tb, p, tm, tn); break;
    default: launch_gemm<CfgBig>(c, ta, tb, p, tm, tn); break;
  }
  post_launch(c);
  if (splits > 1) {
    dim3 g2(unsigned(grid_for(M * N)), unsigned(o.batch));
    dgemm_reduce_splits<<<g2, 256, 0, c->stream>>>(ws.p, splits, M, N, C, ldc, o.sC, alpha, beta,
                                                   o.lower ? 1 : 0);
    post_launch(c);
  }
}

// ------------------------------------------------------------------ Ozaki int8 GEMM
// C (M x N, ldc) = A (M x K, lda) B (K x N, ldb), all column-major, on the int8 tensor
// cores (ozaki_i8.cuh).  Slices live in stream-ordered workspaces.
// ------------------------------------------------------------------ Ozaki int8 GEMM
// An operand sliced for the int8 tensor cores (ozaki_i8.cuh): L lines of K elements, the
// element (l, k) read from P[l sl + k sk], as S digit slices per (tile, k-block) in the
// canonical layout plus the per-line scales 2^e.  A side: lines = rows of A; B side:
// lines = columns of op(B).  A sliced operand is reused across GEMMs that share it.
struct OzSliced {
  DBuf data, scale;
  int64_t lines = 0, K = 0, KB = 0, tiles = 0;
  int halves = 1;  // 2: B operand laid out for the 2-SM kernel
  const int8_t* digits() const { return reinterpret_cast<const int8_t*>(data.p); }
};

void oz_slice(latsum_ctx* c, const double* P, int64_t sl, int64_t sk, int64_t L, int64_t K,
              OzSliced& out, int64_t L1 = 0, int64_t sl2 = 0, int halves = 1, bool even_tiles = false) {
  static_assert(oz::BM == oz::BN, "one tile height for both operands");
  require(K <= oz::KMAX, "ozaki_gemm: K > 16384 overflows the int32 accumulators");
  if (L1 <= 0) L1 = std::max<int64_t>(L, 1);
  out.lines = L;
  out.K = K;
  out.KB = std::max<int64_t>(1, (K + oz::BKB - 1) / oz::BKB);
  out.tiles = (L + oz::BM - 1) / oz::BM;
  out.halves = halves;
  require(out.tiles * out.KB < (int64_t(1) << 31), "ozaki_gemm: too many tiles");
  // the 2-SM kernel reads A tiles in pairs: pad to an even count with zero digits
  const int64_t alloc_tiles = even_tiles ? (out.tiles + 1) / 2 * 2 : out.tiles;
  const size_t bytes = size_t(alloc_tiles) * out.KB * oz::A_STAGE;
  out.data.alloc(c, (bytes + 7) / 8);
  if (alloc_tiles > out.tiles)
    CK(cudaMemsetAsync(reinterpret_cast<int8_t*>(out.data.p) + size_t(out.tiles) * out.KB * oz::A_STAGE, 0,
                       size_t(out.KB) * oz::A_STAGE, c->stream));
  out.scale.alloc(c, size_t(std::max<int64_t>(L, 1)));
  if (L <= 0) return;
  ProfScope ps(c, "ozaki(slice)", double(L) * double(K) * 8.0 + double(bytes));
  const bool vec = sk == 1 && sl % 2 == 0 && (L1 >= L || sl2 % 2 == 0) &&
                   reinterpret_cast<uintptr_t>(P) % 16 == 0;
  int8_t* d = reinterpret_cast<int8_t*>(out.data.p);
  // few tiles, long K: split K over the grid (k_slice_pmax + k_slice_split, bit-identical)
  if (out.tiles < 148 && out.KB >= 16) {
    const int64_t nsplit = std::min<int64_t>(out.KB / 8, (2 * 148 + out.tiles - 1) / out.tiles);
    const int64_t kbs = (out.KB + nsplit - 1) / nsplit;
    const int64_t ns = (out.KB + kbs - 1) / kbs;
    DBuf pmax(c, size_t(ns) * L);
    const dim3 g{unsigned(out.tiles), unsigned(ns)};
    if (vec) {
      oz::k_slice_pmax<oz::BM, true><<<g, 2 * oz::BM, 0, c->stream>>>(P, sl, sk, L, K, out.KB, L1,
                                                                      sl2, kbs, pmax.p);
      post_launch(c);
      oz::k_slice_split<oz::BM, true><<<g, 2 * oz::BM, 0, c->stream>>>(
          P, sl, sk, L, K, out.KB, L1, sl2, kbs, pmax.p, out.scale.p, d, halves);
    } else {
      oz::k_slice_pmax<oz::BM, false><<<g, 2 * oz::BM, 0, c->stream>>>(P, sl, sk, L, K, out.KB, L1,
                                                                       sl2, kbs, pmax.p);
      post_launch(c);
      oz::k_slice_split<oz::BM, false><<<g, 2 * oz::BM, 0, c->stream>>>(
          P, sl, sk, L, K, out.KB, L1, sl2, kbs, pmax.p, out.scale.p, d, halves);
    }
    post_launch(c);
    return;
  }
  // long lines: units of LU lines of a tile, so the 2 x 148 CTAs' lines in flight fit ~90 MB
  // of L2 and the digit pass re-reads mostly from L2
  const double line_bytes = double(K) * 8.0;
  if (line_bytes * oz::BM * 2 * 148 > 90e6) {
    const int lu = line_bytes * 32 * 2 * 148 <= 90e6 ? 32 : line_bytes * 16 * 2 * 148 <= 90e6 ? 16 : 8;
    const int64_t units = out.tiles * (oz::BM / lu);
    const unsigned ctas = unsigned(std::min<int64_t>(units, 2 * 148));
#define LATSUM_SLICE_LINES(LU, V)                                                            \
  oz::k_slice_lines<oz::BM, LU, V><<<ctas, 256, 0, c->stream>>>(P, sl, sk, L, K, out.KB,      \
                                                                 out.scale.p, d, L1, sl2, halves)
    if (vec) {
      if (lu == 32) LATSUM_SLICE_LINES(32, true);
      else if (lu == 16) LATSUM_SLICE_LINES(16, true);
      else LATSUM_SLICE_LINES(8, true);
    } else {
      if (lu == 32) LATSUM_SLICE_LINES(32, false);
      else if (lu == 16) LATSUM_SLICE_LINES(16, false);
      else LATSUM_SLICE_LINES(8, false);
    }
#undef LATSUM_SLICE_LINES
    post_launch(c);
    return;
  }
  // persistent: at most 2 CTAs per SM, so the tiles in flight (2 x 148 x 128 lines x K
  // doubles) can stay L2-resident between the scale pass and the digit pass
  const unsigned ctas = unsigned(std::min<int64_t>(out.tiles, 2 * 148));
  if (vec)
    oz::k_slice_tile<oz::BM, true><<<ctas, 2 * oz::BM, 0, c->stream>>>(P, sl, sk, L, K, out.KB,
                                                                        out.scale.p, d, L1, sl2, halves);
  else
    oz::k_slice_tile<oz::BM, false><<<ctas, 2 * oz::BM, 0, c->stream>>>(P, sl, sk, L, K, out.KB,
                                                                         out.scale.p, d, L1, sl2, halves);
  post_launch(c);
}

// A-side operands (rows of A) and B-side operands (columns of op(B)), laid out for the
// kernel variant in use
void oz_slice_a(latsum_ctx* c, const double* P, int64_t sl, int64_t sk, int64_t L, int64_t K,
                OzSliced& out, int64_t L1 = 0, int64_t sl2 = 0) {  // line l: (l % L1) sl + (l / L1) sl2
  oz_slice(c, P, sl, sk, L, K, out, L1, sl2, 1, false);
}
void oz_slice_b(latsum_ctx* c, const double* P, int64_t sl, int64_t sk, int64_t L, int64_t K,
                OzSliced& out) {
  oz_slice(c, P, sl, sk, L, K, out, 0, 0, 1, false);
}

// Output addressing of an Ozaki GEMM (ozaki_i8.cuh OzOut): plain column-major by default.
oz::OzOut oz_out(double* C, int64_t ldc, double beta = 0.0, double alpha = 1.0) {
  return oz::OzOut{C, ldc, int64_t(1) << 62, 0, int64_t(1) << 62, 0, beta, alpha};
}

// C = A op(B) + beta C from sliced operands (a.lines x b.lines output, addressing o).
void oz_run(latsum_ctx* c, const OzSliced& a, const OzSliced& b, oz::OzOut o, const char* tag) {
  const int64_t M = a.lines, N = b.lines;
  if (M <= 0 || N <= 0) return;
  require(a.K == b.K, "ozaki_gemm: inner dimensions differ");
  if (!c->oz_smem_set) {
    CK(cudaFuncSetAttribute(oz::k_gemm_i8, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(oz::SMEM_BYTES)));
    c->oz_smem_set = true;
  }
  const int64_t tiles = a.tiles * b.tiles;
  require(tiles < (int64_t(1) << 31), "ozaki_gemm: too many tiles");
  ProfScope ps(c, tag, 2.0 * double(M) * double(N) * double(a.K));
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  if (c->max_ctas > 0) {
    sms = std::min(sms, c->max_ctas);
  } else {
    const latsum_ctx* root = c->parent ? c->parent : c;
    sms = std::max(sms / 2, sms - root->reserved_ctas.load(std::memory_order_relaxed));
  }
  const unsigned ctas = unsigned(std::min<int64_t>(tiles, sms));
  // stream the larger operand once: N tiles fastest when A is the bigger one (the core
  // contraction's tall X against the small P_m: 190 -> 155 ms on cfg4), M tiles fastest
  // otherwise (the slabs)
  const int nfast = a.tiles > 2 * b.tiles ? 1 : 0;
  oz::k_gemm_i8<<<ctas, oz::PTHREADS, oz::SMEM_BYTES, c->stream>>>(
      a.digits(), a.scale.p, b.digits(), b.scale.p, M, N, a.KB, o, a.tiles, tiles, b.tiles, nfast);
  post_launch(c);
#ifdef LATSUM_OZ_TRACE
  {
    unsigned long long h[2];
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpyFromSymbol(h, oz::g_oz_trace, sizeof(h)));
    fprintf(stderr, "ozaki trace: MMA thread %.0f clk/CTA, waiting for TMEM %.1f%%\n",
            double(h[0]) / ctas, 100.0 * double(h[1]) / double(h[0]));
    const unsigned long long z[2] = {0, 0};
    CK(cudaMemcpyToSymbol(oz::g_oz_trace, z, sizeof(z)));
  }
#endif
}

// General form: A lines (rows of op(A)) l -> A + (l % a_L1) a_sl + (l / a_L1) a_sl2, element k
// at + k a_sk; B lines (columns of op(B)) n -> B + n b_sl, element k at + k b_sk; output
// addressing o (alpha, beta).  K is split into <= KMAX chunks accumulated with beta = 1.
void ozaki_gemm_ex(latsum_ctx* c, int64_t M, int64_t N, int64_t K, const double* A, int64_t a_sl,
                   int64_t a_sk, int64_t a_L1, int64_t a_sl2, const double* B, int64_t b_sl,
                   int64_t b_sk, oz::OzOut o, const char* tag) {
  if (M <= 0 || N <= 0) return;
  const int64_t parts = std::max<int64_t>(1, (K + oz::KMAX - 1) / oz::KMAX);
  const int64_t kc = std::max<int64_t>(1, (K + parts - 1) / parts);
  const double beta0 = o.beta;
  for (int64_t k0 = 0; k0 < std::max<int64_t>(K, 1); k0 += kc) {
    const int64_t kk = std::min(kc, std::max<int64_t>(K - k0, 0));
    OzSliced a, b;
    oz_slice_a(c, A + k0 * a_sk, a_sl, a_sk, M, kk, a, a_L1, a_sl2);
    oz_slice_b(c, B + k0 * b_sk, b_sl, b_sk, N, kk, b);
    o.beta = k0 == 0 ? beta0 : 1.0;
    oz_run(c, a, b, o, tag);
  }
}

// C (M x N, ldc) = A (M x K, lda) op(B) + beta C, op(B) = B (K x N, ldb) or B^T (B: N x K,
// ldb), all column-major, on the int8 tensor cores.
void ozaki_gemm(latsum_ctx* c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                const double* B, int64_t ldb, double* C, int64_t ldc, const char* tag = "gemm(ozaki-i8)",
                bool tb = false, double beta = 0.0) {
  ozaki_gemm_ex(c, M, N, K, A, 1, lda, 0, 0, B, tb ? 1 : ldb, tb ? ldb : 1, oz_out(C, ldc, beta), tag);
}

// Evaluation slab GEMMs: int8 tensor cores (Ozaki, default) or FP64 DMMA
// (LATSUM_EVAL_GEMM=dmma).
bool eval_uses_ozaki(int64_t K) {
  static const bool dmma = [] {
    const char* e = std::getenv("LATSUM_EVAL_GEMM");
    return e && std::string(e) == "dmma";
  }();
  return !dmma && K <= oz::KMAX;
}
// The Tucker core contraction (stage 3) on the int8 tensor cores too (LATSUM_CORE_GEMM=dmma
// reverts); large products only (the slicing passes cost ~2 operand reads).
bool core_uses_ozaki(int64_t M, int64_t N, int64_t K) {
  static const bool dmma = [] {
    const char* e = std::getenv("LATSUM_CORE_GEMM");
    return e && std::string(e) == "dmma";
  }();
  return !dmma && double(M) * double(N) * double(K) >= 1e10;
}

// ------------------------------------------------------------------ syevd
// Eigen-decomposition of the symmetric n x n matrix A (lower triangle read):
// eigenvalues ascending in W (device), eigenvectors overwrite A.  cuSOLVER's
// 64-bit API (size_t workspaces; the int32 LAPACK workspace overflows at N=32768).
void syevd(latsum_ctx* c, int64_t n, double* A, double* W) {
  size_t dbytes = 0, hbytes = 0;
  CS(cusolverDnXsyevd_bufferSize(c->solver, c->solver_params, CUSOLVER_EIG_MODE_VECTOR,
                                 CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W,
                                 CUDA_R_64F, &dbytes, &hbytes));
  DBuf work(c, (dbytes + 7) / 8 + 1);
  ProfScope ps(c, "syevd(cusolver)", double(n));
  std::vector<char> hwork(hbytes + 1);
  int* info = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&info), sizeof(int), c->stream));
  CS(cusolverDnXsyevd(c->solver, c->solver_params, CUSOLVER_EIG_MODE_VECTOR,
                      CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, A, n, CUDA_R_64F, W, CUDA_R_64F,
                      work.p, dbytes, hwork.data(), hbytes, info));
  int hinfo = 0;
  CK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFreeAsync(info, c->stream);
  if (hinfo != 0) throw Error(LATSUM_ERR_CUSOLVER, "syevd: info = " + std::to_string(hinfo));
}

// ------------------------------------------------------------------ custom eigensolver
// Householder tridiagonalisation of the symmetric n x n matrix A (full storage, lda) in
// one 16-CTA cluster (eig_sym.cuh): d (n), e (n-1), tau (n-1) on the device; the
// reflectors overwrite A below the subdiagonal.
void sytrd_cluster(latsum_ctx* c, int64_t n, double* A, int64_t lda, double* d, double* e,
                   double* tau) {
  if (n <= 0) return;
  require(n < (int64_t(1) << 30), "sytrd: n too large");
  require(n <= 8192, "sytrd: n > 8192");
  set_smem_attr(c, eig::k_sytrd_cluster, 2 * 8192 * sizeof(double), true);
  constexpr int kSmemMax = 227 * 1024 - 2048;  // dynamic share (the kernel has ~1 KB static)
  const bool smem = eig::sm_trd_doubles(int(n)) * int64_t(sizeof(double)) <= kSmemMax &&
                    n <= eig::TRD_CTAS * eig::SM_TRD_MAXCOL && !std::getenv("LATSUM_SYTRD_L2");
  if (smem) {  // trailing matrix resident in the cluster's shared memory
    set_smem_attr(c, eig::k_sytrd_smem, kSmemMax, true);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(eig::TRD_CTAS);
    cfg.blockDim = dim3(eig::SM_TRD_THREADS);
    cfg.dynamicSmemBytes = size_t(eig::sm_trd_doubles(int(n))) * sizeof(double);
    cfg.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = eig::TRD_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope ps(c, "eig_sytrd", double(n) * double(n) * double(n) * 4.0 / 3.0);
    static const bool prof = std::getenv("LATSUM_SYTRD_PROF") != nullptr;
    DBuf pb(c, 8);
    long long* pp = prof ? reinterpret_cast<long long*>(pb.p) : nullptr;
    CK(cudaLaunchKernelEx(&cfg, eig::k_sytrd_smem, A, lda, int(n), d, e, tau, pp));
    post_launch(c);
    if (prof) {
      long long h[8];
      CK(cudaMemcpyAsync(h, pp, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      fprintf(stderr, "[sytrd n=%ld] cycles/step: A %.0f S1 %.0f B %.0f S2 %.0f Cg %.0f Cu %.0f S3 %.0f D %.0f\n",
              long(n), h[0] / double(n), h[1] / double(n), h[2] / double(n), h[3] / double(n),
              h[4] / double(n), h[5] / double(n), h[6] / double(n), h[7] / double(n));
    }
    return;
  }
  DBuf ws(c, size_t(3 * n + 2 * eig::TRD_CTAS + 8));
  eig::TrdWork w{ws.p, ws.p + n, ws.p + 2 * n, ws.p + 3 * n};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(eig::TRD_CTAS);
  cfg.blockDim = dim3(eig::TRD_THREADS);
  cfg.dynamicSmemBytes = size_t(2 * n) * sizeof(double);
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = eig::TRD_CTAS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ProfScope ps(c, "eig_sytrd", double(n) * double(n) * double(n) * 4.0 / 3.0);
  CK(cudaLaunchKernelEx(&cfg, eig::k_sytrd_cluster, A, lda, int(n), d, e, tau, w));
  post_launch(c);
}

// Symmetric eigen-decomposition backend of the Gram passes.  cuSOLVER syevd (all
// eigenvectors; the default) or, with LATSUM_EIG=custom and n <= kCustomEigMax, the
// in-house solver: cluster sytrd, Sturm
// multisection for every eigenvalue, inverse iteration for the leading eigenvectors the
// caller asks for, compact-WY back-transformation on the DMMA GEMM.  The in-house path
// never synchronises with the host inside, so the three modes' eigensolves overlap
// (cuSOLVER's serialise), and it computes only the vectors that are used.
constexpr int64_t kCustomEigMax = 1024;  // shared-memory inverse-iteration factors

// LATSUM_EIG: cusolver | custom (one-stage cluster sytrd) | band (two-stage, n <= SB_NMAX;
// the default for those sizes)
int eig_env_mode() {
  static const int mode = [] {
    const char* e = std::getenv("LATSUM_EIG");
    if (!e) return 0;
    if (std::string(e) == "cusolver") return 1;
    if (std::string(e) == "custom") return 2;
    if (std::string(e) == "band") return 3;
    return 0;
  }();
  return mode;
}
bool band_eig_ok(int64_t n) { return n >= 2 && n <= band::SB_NMAX; }

bool use_custom_eig(int64_t n) {
  if (eig_env_mode() != 2) return false;  // opt-in
  return n >= 2 && n <= kCustomEigMax;
}


struct Eig {
  int64_t n = 0;
  bool custom = false;
  DBuf G;  // cuSOLVER: eigenvectors (ascending columns); in-house: the sytrd reflectors
  DBuf G0; // in-house: a copy of the input for the cuSOLVER fallback
  DBuf d, e, tau;
  double tnorm = 0.0;
  std::vector<double> lam_asc;

  // two-stage (band) path: panel reflectors (Vw, Tw) and bulge reflectors (V2, TAU2)
  bool band = false;
  DBuf Vw, Tw, V2, TAU2;
  int KS = 1;

  // full -> band (k_sy2sb, one 16-CTA cluster) -> tridiagonal d, e (k_sb2st, one CTA)
  void band_reduce(latsum_ctx* c) {
    const int ni = int(n), npan = band::s2b_panels(ni);
    KS = band::sb_tasks_max(ni);
    Vw.alloc(c, std::max<size_t>(1, size_t(npan) * band::BW * n));
    Tw.alloc(c, std::max<size_t>(1, size_t(npan) * band::BW * band::BW));
    V2.alloc(c, size_t(n) * n);
    TAU2.alloc(c, size_t(n) * KS);
    if (npan > 0) {
      CK(cudaMemsetAsync(Vw.p, 0, sizeof(double) * Vw.n, c->stream));
      DBuf Wg(c, size_t(band::BW) * n);
      const size_t smem = band::s2b_smem_doubles(ni) * sizeof(double);
      set_smem_attr(c, band::k_sy2sb, band::s2b_smem_doubles(band::S2B_NMAX) * 8, true);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(band::S2B_CTAS);
      cfg.blockDim = dim3(band::S2B_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = c->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = band::S2B_CTAS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      static const bool prof = std::getenv("LATSUM_SY2SB_PROF") != nullptr;
      DBuf pb(c, 12);
      band::S2BArgs args{G.p, int64_t(n), ni, Vw.p, Tw.p, Wg.p,
                         prof ? reinterpret_cast<long long*>(pb.p) : nullptr};
      {
        ProfScope ps(c, "eig_sy2sb", double(n) * double(n) * double(n) * 4.0 / 3.0);
        CK(cudaLaunchKernelEx(&cfg, band::k_sy2sb, args));
        post_launch(c);
      }
      if (prof) {
        long long h[12];
        CK(cudaMemcpyAsync(h, pb.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        fprintf(stderr, "[sy2sb qr split] loads %.1f columns %.1f writeback+S %.1f (slot 11 %.1f); qr below = T + rest\n",
                h[8] / 1e3 / npan, h[9] / 1e3 / npan, h[10] / 1e3 / npan, h[11] / 1e3 / npan);
        fprintf(stderr, "[sy2sb n=%d] kcycles/panel: qr %.1f bar1 %.1f Y %.1f bar2 %.1f ZW %.1f bar3 %.1f U3 %.1f bar4 %.1f\n",
                ni, h[0] / 1e3 / npan, h[1] / 1e3 / npan, h[2] / 1e3 / npan, h[3] / 1e3 / npan,
                h[4] / 1e3 / npan, h[5] / 1e3 / npan, h[6] / 1e3 / npan, h[7] / 1e3 / npan);
      }
    }
    {
      const size_t smem = band::sb_smem_doubles(ni) * sizeof(double);
      set_smem_attr(c, band::k_sb2st, band::sb_smem_doubles(band::SB_NMAX) * 8);
      ProfScope ps(c, "eig_sb2st", double(n) * double(n));
      static const bool sprof = std::getenv("LATSUM_SB2ST_PROF") != nullptr;
      DBuf pb(c, 4);
      if (sprof) CK(cudaMemsetAsync(pb.p, 0, 32, c->stream));
      band::k_sb2st<<<1, band::SB_WARPS * 32, smem, c->stream>>>(
          G.p, n, ni, d.p, e.p, V2.p, TAU2.p, KS,
          sprof ? reinterpret_cast<unsigned long long*>(pb.p) : nullptr);
      post_launch(c);
      if (sprof) {
        unsigned long long h[3];
        CK(cudaMemcpyAsync(h, pb.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        fprintf(stderr, "[sb2st n=%d] tasks %llu, per warp: loop %.1f kcycles, wait %.1f kcycles; "
                "cycles/task (loop sum / tasks) %.0f, non-wait %.0f\n", ni, h[2],
                h[1] / 1e3 / band::SB_WARPS, h[0] / 1e3 / band::SB_WARPS, double(h[1]) / h[2],
                double(h[1] - h[0]) / h[2]);
      }
    }
  }

  // method: 0 = LATSUM_EIG / default, 1 = cuSOLVER, 2 = in-house one-stage, 3 = two-stage
  void solve(latsum_ctx* c, int64_t nn, DBuf&& Gin, int method = 0) {
    n = nn;
    G = std::move(Gin);
    if (method == 0) method = c->eig_method;
    if (method == 0) {  // default: the two-stage solver where it applies, else syevd
      const int env = eig_env_mode();
      band = (env == 0 || env == 3) && band_eig_ok(n);
      custom = band || use_custom_eig(n);
    } else {
      band = method == 3 && band_eig_ok(n);
      custom = band || (method == 2 && n >= 2 && n <= kCustomEigMax);
    }
    lam_asc.assign(n, 0.0);
    if (n == 0) return;
    DBuf W(c, n);
    if (!custom) {
      syevd(c, n, G.p, W.p);
    } else {
      d.alloc(c, n);
      e.alloc(c, n);
      tau.alloc(c, n);
      eig::k_symmetrize_lower<<<grid_for(n * n), 256, 0, c->stream>>>(G.p, n, int(n));
      post_launch(c);
      G0.alloc(c, size_t(n) * n);
      CK(cudaMemcpyAsync(G0.p, G.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream));
      if (band) band_reduce(c);
      else sytrd_cluster(c, n, G.p, n, d.p, e.p, tau.p);
      ProfScope ps(c, "eig_values", double(n));
      const size_t smem = size_t(2 * n) * sizeof(double);
      set_smem_attr(c, band::k_tridiag_eigvals_ms, size_t(2 * kCustomEigMax) * sizeof(double));
      band::k_tridiag_eigvals_ms<<<unsigned((n + band::EV_WARPS - 1) / band::EV_WARPS),
                                   32 * band::EV_WARPS, smem, c->stream>>>(d.p, e.p, int(n), W.p);
      post_launch(c);
    }
    CK(cudaMemcpyAsync(lam_asc.data(), W.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (double v : lam_asc) tnorm = std::max(tnorm, std::fabs(v));
  }

  // the k leading eigenvectors (descending eigenvalues) into V (n x k)
  void leading(latsum_ctx* c, int64_t k, double* V) {
    if (k <= 0) return;
    if (!custom) {
      k_reverse_columns<<<grid_for(n * k), 256, 0, c->stream>>>(G.p, n, n, k, V);
      post_launch(c);
      return;
    }
    std::vector<double> lk(k);
    for (int64_t j = 0; j < k; ++j) lk[j] = lam_asc[n - 1 - j];
    DVec<double> dl;
    dl.upload(c, lk);
    if (band) {
      {
        ProfScope ps(c, "eig_invit", double(n) * double(k));
        const int64_t per = 41 * n;  // bytes per vector: 5 doubles + 1 flag per row
        const int nt = int(std::max<int64_t>(1, std::min<int64_t>(32, (227 * 1024 - 1024) / per)));
        set_smem_attr(c, band::k_tridiag_invit_sm, 227 * 1024 - 1024);
        band::k_tridiag_invit_sm<<<unsigned((k + nt - 1) / nt), unsigned(nt), size_t(nt) * per,
                                   c->stream>>>(d.p, e.p, int(n), dl.p, int(k), tnorm, V);
        post_launch(c);
      }
      {
        ProfScope ps(c, "eig_backtransform", double(n) * double(n) * double(k));
        // ys (n x BT_CPB), wv / tw, one or two panel buffers (BW x n), two mbarriers
        constexpr size_t kBtMax = 226 * 1024;
        auto bt_smem = [&](int nbuf) {
          return (size_t(n) * (band::BT_CPB + size_t(nbuf) * band::BW) + 2 * band::BW * band::BT_CPB) *
                     sizeof(double) + 16;
        };
        const int dbuf = bt_smem(2) <= kBtMax ? 1 : 0;
        const size_t smem = bt_smem(dbuf ? 2 : 1);
        set_smem_attr(c, band::k_band_backtransform, kBtMax);
        band::k_band_backtransform<<<unsigned((k + band::BT_CPB - 1) / band::BT_CPB), band::BT_THREADS,
                                     smem, c->stream>>>(int(n), int(k), V2.p, TAU2.p, KS, Vw.p, Tw.p,
                                                        band::s2b_panels(int(n)), V, V, dbuf);
        post_launch(c);
      }
    } else {
    {
      ProfScope ps(c, "eig_invit", double(n) * double(k));
      const int64_t per = size_t(5) * n * sizeof(double);
      const int vpb = int(std::max<int64_t>(1, std::min<int64_t>(32, (227 * 1024 - 1024) / per)));
      const size_t smem = size_t(vpb) * per;
      require(int64_t(smem) <= 227 * 1024 - 1024, "eigensolver: n too large for shared-memory factors");
      CK(cudaFuncSetAttribute(eig::k_tridiag_invit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              227 * 1024 - 1024));
      eig::k_tridiag_invit<<<unsigned((k + vpb - 1) / vpb), unsigned(vpb), smem, c->stream>>>(
          d.p, e.p, int(n), dl.p, int(k), tnorm, V);
      post_launch(c);
    }
    // V <- Q V, Q = H_0 .. H_{n-2} in compact-WY blocks, last block first
    const int64_t nr = n - 1, nb = eig::WY_NB, nblk = (nr + nb - 1) / nb;
    if (nblk == 0) return;
    DBuf Vwy(c, size_t(nblk) * nb * n), Twy(c, size_t(nblk) * nb * nb);
    const size_t wsm = size_t(2) * nb * (nb + 1) * sizeof(double);
    CK(cudaFuncSetAttribute(eig::k_wy_build, cudaFuncAttributeMaxDynamicSharedMemorySize, int(wsm)));
    eig::k_wy_build<<<unsigned(nblk), 256, wsm, c->stream>>>(G.p, n, int(n), tau.p, Vwy.p, Twy.p);
    post_launch(c);
    DBuf W1(c, size_t(nb) * k), W2(c, size_t(nb) * k);
    for (int64_t b = nblk - 1; b >= 0; --b) {
      const int64_t m = std::min(nb, nr - b * nb);
      const double* Vb = Vwy.p + size_t(b) * nb * n;
      const double* Tb = Twy.p + size_t(b) * nb * nb;
      gemm(c, true, false, m, k, n, 1.0, Vb, n, V, n, 0.0, W1.p, nb, tagged("gemm_eig_wy"));
      gemm(c, false, false, m, k, m, 1.0, Tb, nb, W1.p, nb, 0.0, W2.p, nb, tagged("gemm_eig_wy"));
      gemm(c, false, false, n, k, m, -1.0, Vb, n, W2.p, nb, 1.0, V, n, tagged("gemm_eig_wy"));
    }
    }
    // Inverse iteration has no cluster re-orthogonalisation: (near-)degenerate eigenvalues
    // give (near-)parallel vectors.  Check V^T V and fall back to syevd for this Gram when
    // the vectors are not orthonormal to 1e-9 (the RHOSVD Grams' spectra pass).
    DBuf S(c, size_t(k) * k), mx(c, 1);
    gemm(c, true, false, k, k, n, 1.0, V, n, V, n, 0.0, S.p, k, tagged("gemm_eig_wy"));
    eig::k_max_offidentity<<<1, 1024, 0, c->stream>>>(S.p, int(k), mx.p);
    post_launch(c);
    double dev = 0.0;
    CK(cudaMemcpyAsync(&dev, mx.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (Trace::on()) fprintf(stderr, "[eig] n=%ld k=%ld orthogonality %.2e\n", long(n), long(k), dev);
    // (1e-9 let ~1e-10-orthogonal inverse-iteration vectors of near-degenerate pass-2
    // Grams through, which the ALS refinement of canonical_to_tucker amplifies)
    static const double otol_env = [] {
      const char* e = std::getenv("LATSUM_EIG_ORTHO_TOL");
      return e ? std::atof(e) : -1.0;
    }();
    const double otol = otol_env >= 0.0 ? otol_env
                        : ortho_tol >= 0.0 ? ortho_tol
                                           : 1e-12 * std::max(1.0, double(n) / 64.0);
    if (!(dev <= otol)) {
      DBuf Wf(c, n);
      syevd(c, n, G0.p, Wf.p);
      k_reverse_columns<<<grid_for(n * k), 256, 0, c->stream>>>(G0.p, n, n, k, V);
      post_launch(c);
      c->eig_fallbacks++;
      custom = false;  // G0 now holds all eigenvectors: later calls take them from there
      band = false;
      G = std::move(G0);
    }
  }
  // Row-sharded RHOSVD: rank `owner` solves with cuSOLVER and the others receive the values
  // and all eigenvectors through a sum all-reduce to which they contribute zeros (exact).
  // Every rank must hold bit-identical bases (the row blocks of U = A V lambda^{-1/2} of
  // different ranks belong to the same vectors), which redundant solves do not guarantee:
  // the in-house solver's reflectors and inverse-iteration vectors may differ in the last
  // bits, and near-degenerate eigenvectors then rotate apart.  So in a sharded reduction one
  // rank per mode solves every Gram (also spreading the three modes' solves over the ranks).
  void solve_on(latsum_ctx* c, int64_t nn, DBuf&& Gin, int owner) {
    if (owner < 0 || !has_comm(c)) {
      solve(c, nn, std::move(Gin));
      return;
    }
    n = nn;
    G = std::move(Gin);
    custom = band = false;
    lam_asc.assign(n, 0.0);
    if (n == 0) return;
    DBuf buf(c, size_t(n) + size_t(n) * n);
    if (c->rank == owner % c->nranks) {
      syevd(c, n, G.p, buf.p);
      CK(cudaMemcpyAsync(buf.p + n, G.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream));
    } else {
      CK(cudaMemsetAsync(buf.p, 0, sizeof(double) * buf.n, c->stream));
    }
    allreduce(c, buf.p, buf.n);
    CK(cudaMemcpyAsync(G.p, buf.p + n, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(lam_asc.data(), buf.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (double v : lam_asc) tnorm = std::max(tnorm, std::fabs(v));
  }

  bool has_all() const { return !custom; }
  // max |V^T V - I| accepted from the in-house vectors before falling back to syevd
  // (< 0: 1e-12 max(1, n/64))
  double ortho_tol = -1.0;
};

struct Timer {
  latsum_ctx* c;
  cudaEvent_t a, b;
  explicit Timer(latsum_ctx* ctx) : c(ctx) {
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  void start() { CK(cudaEventRecord(a, c->stream)); }
  double stop() {
    CK(cudaEventRecord(b, c->stream));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }
};

}  // namespace

// ------------------------------------------------------------------ handles

struct latsum_reference {
  int family = 0;
  double lambda = 0;
  int M = 0, R = 0, Rd = 0;
  double C0 = 0, shell[2] = {0, 0};
  int64_t N[3] = {0, 0, 0};
  double box[3] = {0, 0, 0};
  std::vector<double> nodes, qweights, weights;
  std::vector<int> jmap;       // R -> distinct column
  int owner[3] = {0, 1, 2};    // mode whose storage this mode shares
  DBuf cols[3];                // 2N x Rd, unit columns (only owners allocate)
  const double* col(int l) const { return cols[owner[l]].p; }
};

struct latsum_canonical {
  int64_t N[3] = {0, 0, 0};
  int Rd = 0, R = 0;
  int64_t Mc = 0, T = 0;
  int64_t d[3] = {0, 0, 0};
  DBuf dict[3];                              // N_l x d_l
  std::vector<double> dict_norms[3];
  std::vector<int64_t> term_col[3];          // M_c per mode (reference order)
  std::vector<double> weights;               // M_c
  std::vector<double> mult[3];               // multiplicity per dictionary column
  // merged terms sorted by c0
  std::vector<int32_t> tc[3];
  std::vector<double> tw;
  std::vector<int64_t> tseg;                 // d0 + 1
  DVec<int32_t> dtc[3];
  DVec<double> dtw;
  DVec<int64_t> dtseg;
  // the merged terms re-sorted by their mode-m column (m = 1, 2), with segments, for
  // contracting the core over the mode with the fewest distinct columns
  std::vector<int32_t> stc[3][3];
  std::vector<double> stw[3];
  std::vector<int64_t> sseg[3];
  // assemble() merges the terms (everything above from tc on) on a host thread that runs
  // while the RHOSVD's Grams and eigensolves are on the device; terms() joins it and
  // uploads dtc/dtw/dtseg.  Declared last: destroyed (joined) before the vectors it fills.
  bool terms_async = false, terms_uploaded = false;
  std::mutex terms_mu;
  std::shared_future<void> terms_ready;
};

// The merged terms of `cc` on the host (terms_host) or also on the device (terms).
const latsum_canonical& terms_host(const latsum_canonical& cc) {
  auto& can = const_cast<latsum_canonical&>(cc);
  if (can.terms_async) can.terms_ready.get();
  return cc;
}

const latsum_canonical& terms(latsum_ctx* c, const latsum_canonical& cc) {
  auto& can = const_cast<latsum_canonical&>(cc);
  if (!can.terms_async) return cc;
  std::lock_guard<std::mutex> g(can.terms_mu);
  if (can.terms_uploaded) return cc;
  can.terms_ready.get();
  // owned by the caller's (root) context stream, whichever worker needs them first: they
  // are freed on that stream when the canonical tensor is destroyed
  latsum_ctx* root = c;
  while (root->parent) root = root->parent;
  for (int l = 0; l < 3; ++l) can.dtc[l].upload(root, can.tc[l]);
  can.dtw.upload(root, can.tw);
  can.dtseg.upload(root, can.tseg);
  CK(cudaStreamSynchronize(root->stream));  // later users may sit on other streams
  can.terms_uploaded = true;
  return cc;
}

struct latsum_tucker {
  bool sink_written = false;  // the core and factors were streamed to the context's host sink
  // per-rank core slab (LATSUM_RHOSVD_CORE_SLABS): core holds rows [a0, a0 + ra) of mode 0
  bool core_slab = false;
  int64_t a0 = 0, ra = 0;
  int64_t N[3] = {0, 0, 0};
  int64_t r[3] = {1, 1, 1};
  DBuf U[3];     // N_l x r_l
  DBuf core;     // r0 x r1 x r2 (absent when the core was not formed)
  bool has_core = false;
  std::vector<double> sigma[3];
  // projected canonical form V = sum_t w_t prod_l (U_l P_l)[:, c_l(t)]  (equals the
  // Tucker tensor; used when the dense core does not fit, e.g. BASELINE cfg5)
  DBuf P[3];     // r_l x d_l
  int64_t d[3] = {0, 0, 0};
  int64_t T = 0;
  DVec<int32_t> tc[3];
  DVec<double> tw;
  DVec<int64_t> tseg;  // d0 + 1: the terms are sorted by their mode-0 column
};

namespace {

template <typename F>
int guarded(latsum_ctx* c, F&& f) {
  try {
    f();
    return LATSUM_OK;
  } catch (const Error& e) {
    if (c) c->err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return LATSUM_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return LATSUM_ERR_INVALID_ARGUMENT;
  }
}

// ------------------------------------------------------------------ stage 1
void build_reference(latsum_ctx* c, int family, double lambda, const int64_t N[3],
                     const double box[3], int M, double C0, latsum_reference& ref) {
  require(family == LATSUM_NEWTON || family == LATSUM_YUKAWA,
          "build_reference: only gauss-type primitives (newton, yukawa) are on the hot path");
  for (int l = 0; l < 3; ++l) {
    require(N[l] >= 2, "UniformGrid: need at least 2 cells per mode");
    require(N[l] % 2 == 0, "UniformGrid: odd cell count in mode " + std::to_string(l + 1) +
                               " rejected; the centered window assumes even n");
    require(box[l] > 0.0, "UniformGrid: box width must be positive");
  }
  require(M >= 2, "build_quadrature: M >= 2 required");
  ref.family = family;
  ref.lambda = lambda;
  ref.M = M;
  ref.R = 2 * M + 1;
  for (int l = 0; l < 3; ++l) {
    ref.N[l] = N[l];
    ref.box[l] = box[l];
  }
  latsum_reference_shell(N, box, ref.shell);
  ref.C0 = C0 > 0.0 ? C0
                    : latsum_default_step_constant(family, lambda, M, ref.shell[0], ref.shell[1], 320);
  ref.nodes.resize(ref.R);
  ref.qweights.resize(ref.R);
  int st = latsum_build_quadrature(family, lambda, M, ref.C0, ref.shell[0], ref.shell[1],
                                   ref.nodes.data(), ref.qweights.data());
  if (st != LATSUM_OK) throw Error(st, "build_quadrature: invalid rule parameters");

  // distinct exponents s = t^2 (t_{-k} = -t_k share one column, reference.hpp:41-51)
  std::vector<double> sd;
  ref.jmap.resize(ref.R);
  for (int k = 0; k < ref.R; ++k) {
    const double s = ref.nodes[k] * ref.nodes[k];
    int j = -1;
    for (size_t q = 0; q < sd.size(); ++q)
      if (sd[q] == s) { j = int(q); break; }
    if (j < 0) { j = int(sd.size()); sd.push_back(s); }
    ref.jmap[k] = j;
  }
  ref.Rd = int(sd.size());
  DVec<double> ds;
  ds.upload(c, sd);

  ref.weights.assign(ref.qweights.begin(), ref.qweights.end());  // coefficient 1
  std::vector<double> norms[3];
  for (int l = 0; l < 3; ++l) {
    ref.owner[l] = l;
    for (int m = 0; m < l; ++m)
      if (N[l] == N[m] && box[l] == box[m]) { ref.owner[l] = ref.owner[m]; break; }
    if (ref.owner[l] == l) {
      const int64_t n2 = 2 * N[l];
      const double h = (2.0 * box[l]) / double(n2);
      const double lower = 0.0 - (2.0 * box[l]) / 2.0;
      ref.cols[l].alloc(c, size_t(n2) * ref.Rd);
      dim3 g(unsigned((n2 + 255) / 256), unsigned(ref.Rd));
      ProfScope ps(c, "ref_integrals", 8.0 * double(n2) * ref.Rd);
      k_ref_integrals<<<g, 256, 0, c->stream>>>(ds.p, n2, lower, h, ref.cols[l].p);
      post_launch(c);
      DBuf dn(c, ref.Rd);
      k_normalize_columns<<<ref.Rd, 512, 0, c->stream>>>(ref.cols[l].p, n2, dn.p);
      post_launch(c);
      norms[l].resize(ref.Rd);
      CK(cudaMemcpyAsync(norms[l].data(), dn.p, sizeof(double) * ref.Rd, cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaStreamSynchronize(c->stream));
    } else {
      norms[l] = norms[ref.owner[l]];
    }
  }
  // from_raw (canonical.hpp:32-48): weights absorb the three column norms
  for (int l = 0; l < 3; ++l)
    for (int k = 0; k < ref.R; ++k) {
      const double nrm = norms[l][ref.jmap[k]];
      if (nrm == 0.0) ref.weights[k] = 0.0;
      else ref.weights[k] *= nrm;
    }
}

// ------------------------------------------------------------------ stage 2
// Merge identical rank-1 terms and build the per-mode sorted orders (host only; runs on
// a host thread started by assemble(), see latsum_canonical::terms_ready).
void merge_terms(latsum_canonical& can) {
  // merge identical rank-1 terms (same column in all three modes)
  // (key = c0:c1:c2 packed in 21-bit fields, q); stable order keeps the reference's
  // term order inside each merged group, so merged weights add in add_concat order
  // stable LSD counting sort over (c2, c1, c0): O(M_c) instead of a comparison sort
  std::vector<std::pair<uint64_t, int64_t>> keys(can.Mc), tmp(can.Mc);
  for (int64_t q = 0; q < can.Mc; ++q)
    keys[q] = {(uint64_t(can.term_col[0][q]) << 42) | (uint64_t(can.term_col[1][q]) << 21) |
                   uint64_t(can.term_col[2][q]),
               q};
  for (int pass = 0; pass < 3; ++pass) {
    const int l = 2 - pass, shift = 21 * pass;
    std::vector<int64_t> cnt(can.d[l] + 1, 0);
    for (const auto& kq : keys) cnt[((kq.first >> shift) & 0x1FFFFF) + 1]++;
    for (int64_t a = 0; a < can.d[l]; ++a) cnt[a + 1] += cnt[a];
    for (const auto& kq : keys) tmp[cnt[(kq.first >> shift) & 0x1FFFFF]++] = kq;
    keys.swap(tmp);
  }
  for (int l = 0; l < 3; ++l) can.tc[l].clear();
  can.tw.clear();
  can.tseg.assign(can.d[0] + 1, 0);
  for (size_t i = 0; i < keys.size();) {  // sorted by c0, then c1, c2
    const uint64_t key = keys[i].first;
    double w = 0.0;
    for (; i < keys.size() && keys[i].first == key; ++i) w += can.weights[keys[i].second];
    const int64_t c0 = int64_t(key >> 42), c1 = int64_t((key >> 21) & 0x1FFFFF),
                  c2 = int64_t(key & 0x1FFFFF);
    can.tc[0].push_back(int32_t(c0));
    can.tc[1].push_back(int32_t(c1));
    can.tc[2].push_back(int32_t(c2));
    can.tw.push_back(w);
    can.tseg[c0 + 1] += 1;
  }
  can.T = int64_t(can.tw.size());
  for (int64_t a = 0; a < can.d[0]; ++a) can.tseg[a + 1] += can.tseg[a];
  for (int m = 0; m < 3; ++m) {  // counting sort by c_m (stable: keeps the c0-major order)
    can.sseg[m].assign(can.d[m] + 1, 0);
    for (int64_t t = 0; t < can.T; ++t) can.sseg[m][can.tc[m][t] + 1] += 1;
    for (int64_t a = 0; a < can.d[m]; ++a) can.sseg[m][a + 1] += can.sseg[m][a];
    std::vector<int64_t> pos(can.sseg[m].begin(), can.sseg[m].end() - 1);
    for (int l = 0; l < 3; ++l) can.stc[m][l].assign(can.T, 0);
    can.stw[m].assign(can.T, 0.0);
    for (int64_t t = 0; t < can.T; ++t) {
      const int64_t q = pos[can.tc[m][t]]++;
      for (int l = 0; l < 3; ++l) can.stc[m][l][q] = can.tc[l][t];
      can.stw[m][q] = can.tw[t];
    }
  }
}

latsum_ctx* sub_ctx(latsum_ctx* c, int i);

// Events of a multi-stream section, destroyed together.
struct EventSet {
  std::vector<cudaEvent_t> ev;
  cudaEvent_t record(cudaStream_t s) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
    CK(cudaEventRecord(e, s));
    return e;
  }
  ~EventSet() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

// Ordered product blocks (the general form of every stage-2 input): block b contributes R
// terms whose mode-l vector is the assembled sum over its mode-l shift list, weight
// charge_b * w_ref.  A sublattice, a product-structure defect cluster and a single defect
// site (counts 1 x 1 x 1, windowed_canonical) are all product blocks.
void assemble_blocks(latsum_ctx* c, const latsum_reference& ref, int64_t nblk,
                     const int64_t* blk_counts, const int64_t* blk_shifts,
                     const double* blk_charges, latsum_canonical& can) {
  require(nblk >= 0, "assemble: negative counts");
  Trace::mark(c, "assemble: start", false);
  const int R = ref.R, Rd = ref.Rd;
  can.R = R;
  can.Rd = Rd;
  can.Mc = int64_t(R) * nblk;
  for (int l = 0; l < 3; ++l) can.N[l] = ref.N[l];

  // per-mode placements: multi-shift lists first, then distinct single shifts
  std::vector<int64_t> block_pl[3];
  DBuf norm_buf[3];
  std::vector<int64_t> blk_off(size_t(nblk) * 3 + 1, 0);
  {
    int64_t o = 0;
    for (int64_t s = 0; s < nblk; ++s)
      for (int l = 0; l < 3; ++l) {
        blk_off[s * 3 + l] = o;
        require(blk_counts[s * 3 + l] >= 1, "assembled_vector: empty active set");
        o += blk_counts[s * 3 + l];
      }
    blk_off[size_t(nblk) * 3] = o;
  }
  latsum_ctx* side = c->parent ? nullptr : sub_ctx(c, 0);  // idle here: the mode workers run later
  EventSet evs;
  for (int l = 0; l < 3; ++l) {
    const int64_t N = ref.N[l];
    std::vector<int64_t> pl_off{0}, pl_shift;
    auto check = [&](int64_t cshift) {
      const int64_t begin = N / 2 - cshift;
      if (begin < 0 || begin + N > 2 * N)
        throw Error(LATSUM_ERR_WINDOW_OVERFLOW,
                    "window overflow in mode " + std::to_string(l + 1) + ": shift " +
                        std::to_string(-cshift) + " pushes the length-" + std::to_string(N) +
                        " window outside the doubled grid");
    };
    block_pl[l].resize(nblk);
    // a placement is a shift list; identical lists (e.g. the z lists of the two
    // hexagonal sublattices, or a defect on an L=1 sublattice) share dictionary columns
    std::map<std::vector<int64_t>, int64_t> seen;
    auto place = [&](std::vector<int64_t> sh) {
      auto it = seen.find(sh);
      if (it != seen.end()) return it->second;
      for (int64_t v : sh) check(v);
      const int64_t p = int64_t(pl_off.size()) - 1;
      pl_shift.insert(pl_shift.end(), sh.begin(), sh.end());
      pl_off.push_back(int64_t(pl_shift.size()));
      seen.emplace(std::move(sh), p);
      return p;
    };
    for (int64_t s = 0; s < nblk; ++s) {
      if (blk_counts[s * 3 + l] == 1) continue;
      const int64_t* sh = blk_shifts + blk_off[s * 3 + l];
      block_pl[l][s] = place(std::vector<int64_t>(sh, sh + blk_counts[s * 3 + l]));
    }
    const int64_t P_sub = int64_t(pl_off.size()) - 1;  // multi-shift placements come first
    for (int64_t s = 0; s < nblk; ++s)
      if (blk_counts[s * 3 + l] == 1)
        block_pl[l][s] = place(std::vector<int64_t>{blk_shifts[blk_off[s * 3 + l]]});
    const int64_t P = int64_t(pl_off.size()) - 1;
    can.d[l] = P * Rd;
    if (can.d[l] == 0) continue;
    DVec<int64_t> doff, dsh, dstride;
    doff.upload(c, pl_off);
    dsh.upload(c, pl_shift);
    // placements the reference's default order sums by the sliding recursion (lattice_sum.hpp:
    // 116: sliding && contiguous K && more than one window && N_L > n): ascending shifts at one
    // stride n < N; every other list is summed directly in list order (the reference's
    // ascending order, which its sliding order also falls back to)
    std::vector<int64_t> pl_stride(size_t(P), 0);
    bool any_sliding = false;
    if (c->accumulation == 0)
      for (int64_t p = 0; p < P_sub; ++p) {
        const int64_t s0 = pl_off[p], L = pl_off[p + 1] - s0;
        if (L < 2) continue;
        const int64_t n = pl_shift[s0 + 1] - pl_shift[s0];
        bool ok = n > 0 && n < N;
        for (int64_t k = 2; ok && k < L; ++k) ok = pl_shift[s0 + k] - pl_shift[s0 + k - 1] == n;
        // the leaving term's window [N/2 - (c_max + n) + n, ...) starts inside the doubled grid
        // by the window check of c_max; nothing else to verify
        if (ok) {
          pl_stride[size_t(p)] = n;
          any_sliding = true;
        }
      }
    if (any_sliding) dstride.upload(c, pl_stride);
    can.dict[l].alloc(c, size_t(N) * can.d[l]);
    // [0, P_sub Rd): multi-shift (sublattice / product-cluster) columns, up to 256 shifted reads
    // per entry: 2048-row blocks, partial sums of squares per block, the norms, then the
    // normalised entries (three launches, L2-bound).  They run on a side stream next to
    // [P_sub Rd, d): the single-shift defect columns — the HBM traffic of the assembly — one
    // fused launch (k_dict_single).
    const int64_t chunk = 2048;
    const int nchunk = int((N + chunk - 1) / chunk);
    const int64_t n_multi = std::min(can.d[l], P_sub * Rd);
    DBuf partial(c, size_t(std::max<int64_t>(n_multi, 1)) * nchunk);
    DBuf& norms = norm_buf[l];
    norms.alloc(c, can.d[l]);
    ProfScope ps(c, "assemble_dict", 8.0 * double(N) * double(can.d[l]));
    DictArgs a{ref.col(l), N, Rd, doff.p, dsh.p, can.dict[l].p, partial.p, norms.p, chunk, nchunk};
    if (any_sliding) a.pl_stride = dstride.p;
    const bool both = n_multi > 0 && n_multi < can.d[l] && side != nullptr;
    cudaStream_t sm = both ? side->stream : c->stream;  // the multi-shift columns' stream
    if (both) CK(cudaStreamWaitEvent(sm, evs.record(c->stream), 0));  // buffers are allocated
    if (n_multi > 0) {
      if (any_sliding) {
        k_dict_sliding<<<unsigned(n_multi), DICT_THREADS, 0, sm>>>(a);
        post_launch(c);
      }
      k_dict_sumsq<<<dim3{unsigned(n_multi), unsigned(nchunk)}, DICT_THREADS, 0, sm>>>(a);
      post_launch(c);
      k_dict_norms<<<unsigned((n_multi + 255) / 256), 256, 0, sm>>>(a, n_multi);
      post_launch(c);
      k_dict_write<<<dim3{unsigned(n_multi), unsigned(nchunk)}, DICT_THREADS, 0, sm>>>(a);
      post_launch(c);
    }
    if (n_multi < can.d[l]) {
      a.c0 = n_multi;
      k_dict_single<<<unsigned(can.d[l] - n_multi), DICT_THREADS, 0, c->stream>>>(a);
      post_launch(c);
    }
    // partial / the shift tables are released in c->stream order: after the side stream's use
    if (both) CK(cudaStreamWaitEvent(c->stream, evs.record(sm), 0));
  }
  for (int l = 0; l < 3; ++l) {  // the three modes' kernels are queued before the first wait
    can.dict_norms[l].resize(can.d[l]);
    if (can.d[l])
      CK(cudaMemcpyAsync(can.dict_norms[l].data(), norm_buf[l].p, sizeof(double) * can.d[l],
                         cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));

  Trace::mark(c, "assemble: dictionaries done", false);
  // terms in reference order (add_concat: the blocks in the caller's order)
  can.weights.resize(can.Mc);
  for (int l = 0; l < 3; ++l) {
    can.term_col[l].resize(can.Mc);
    can.mult[l].assign(can.d[l], 0.0);
  }
  for (int64_t b = 0; b < nblk; ++b) {
    const double charge = blk_charges[b];
    for (int k = 0; k < R; ++k) {
      const int64_t q = b * R + k;
      double w = charge * ref.weights[k];
      for (int l = 0; l < 3; ++l) {
        const int64_t col = block_pl[l][b] * Rd + ref.jmap[k];
        can.term_col[l][q] = col;
        can.mult[l][col] += 1.0;
        const double nrm = can.dict_norms[l][col];
        if (nrm == 0.0) w = 0.0;
        else w *= nrm;
      }
      can.weights[q] = w;
    }
  }
  Trace::mark(c, "assemble: terms done", false);
  for (int l = 0; l < 3; ++l)
    require(can.d[l] < (int64_t(1) << 21), "assemble: too many distinct columns in a mode");
  can.terms_async = true;
  can.terms_ready = std::async(std::launch::async, [&can] { merge_terms(can); }).share();
}

// Sublattice blocks, then single-site defects (the latsum_canonical_assemble layout).
void assemble(latsum_ctx* c, const latsum_reference& ref, int64_t nsub, const int64_t* sub_counts,
              const int64_t* sub_shifts, const double* sub_charges, int64_t ndef,
              const int64_t* def_shifts, const double* def_charges, latsum_canonical& can) {
  require(nsub >= 0 && ndef >= 0, "assemble: negative counts");
  const int64_t nblk = nsub + ndef;
  std::vector<int64_t> counts(size_t(nblk) * 3, 1), shifts;
  std::vector<double> charges(static_cast<size_t>(nblk), 0.0);
  int64_t o = 0;
  for (int64_t s = 0; s < nsub; ++s)
    for (int l = 0; l < 3; ++l) {
      counts[s * 3 + l] = sub_counts[s * 3 + l];
      require(sub_counts[s * 3 + l] >= 1, "assembled_vector: empty active set");
      shifts.insert(shifts.end(), sub_shifts + o, sub_shifts + o + sub_counts[s * 3 + l]);
      o += sub_counts[s * 3 + l];
    }
  for (int64_t s = 0; s < nsub; ++s) charges[s] = sub_charges[s];
  for (int64_t dd = 0; dd < ndef; ++dd) {
    for (int l = 0; l < 3; ++l) shifts.push_back(def_shifts[dd * 3 + l]);
    charges[nsub + dd] = def_charges[dd];
  }
  assemble_blocks(c, ref, nblk, counts.data(), shifts.data(), charges.data(), can);
}

void materialize_factor(latsum_ctx* c, const latsum_canonical& can, int l, double* dst_device) {
  if (can.Mc == 0) return;
  DVec<int64_t> idx;
  idx.upload(c, can.term_col[l]);
  const int64_t N = can.N[l];
  ProfScope ps(c, "materialize_side_matrix", 8.0 * double(N) * double(can.Mc));
  dim3 g(unsigned(std::max<int64_t>(1, std::min<int64_t>(64, (N / 2 + 255) / 256))),
         unsigned(can.Mc));
  require(can.Mc <= 65535 * 64, "materialize: too many columns");
  if (can.Mc > 65535) {
    // split along the column dimension
    for (int64_t q0 = 0; q0 < can.Mc; q0 += 65535) {
      const int64_t nq = std::min<int64_t>(65535, can.Mc - q0);
      dim3 g2(g.x, unsigned(nq));
      k_gather_columns<<<g2, 256, 0, c->stream>>>(can.dict[l].p, N, idx.p + q0,
                                                  dst_device + q0 * N);
      post_launch(c);
    }
  } else {
    k_gather_columns<<<g, 256, 0, c->stream>>>(can.dict[l].p, N, idx.p, dst_device);
    post_launch(c);
  }
}


// ------------------------------------------------------------------ stage 3
constexpr double kEpsMach = 2.220446049250313e-16;

// rank_reduction.hpp:73-84: smallest r with sqrt(sum_{k>=r} s_k^2) <= eps ||s|| / 3, r >= 1.
int64_t rank_for_tolerance(const std::vector<double>& sv, double eps) {
  double n2 = 0.0;
  for (double v : sv) n2 += v * v;
  const double target = eps * std::sqrt(n2) / 3.0;
  double tail2 = 0.0;
  int64_t r = int64_t(sv.size());
  for (int64_t k = int64_t(sv.size()) - 1; k >= 0; --k) {
    tail2 += sv[k] * sv[k];
    if (std::sqrt(tail2) > target) break;
    r = k;
  }
  return std::max<int64_t>(r, 1);
}

void gram(latsum_ctx* c, bool rows, const double* A, int64_t N, int64_t d, double* G) {
  GemmOpts o = tagged("gemm_gram");
  o.lower = true;
  // SYRK writes the lower tiles only.  A sharded reduction all-reduces the whole square: clear
  // it first, so the tiles nobody reads are zeros on every rank rather than whatever the pool
  // held (they were summed as garbage: harmless, but non-finite sums showed up in the host
  // collectives of the tests)
  if (has_comm(c)) {
    const int64_t n = rows ? N : d;
    CK(cudaMemsetAsync(G, 0, sizeof(double) * n * n, c->stream));
  }
  if (rows) gemm(c, false, true, N, N, d, 1.0, A, N, A, N, 0.0, G, N, o);   // A A^T
  else gemm(c, true, false, d, d, N, 1.0, A, N, A, N, 0.0, G, d, o);        // A^T A
}

// Polar (Loewdin) re-orthonormalisation U <- U (U^T U)^{-1/2} by Newton-Schulz
// iterations U <- U (3I - U^T U)/2: GEMM-only (no eigensolver).  The error E = U^T U - I
// maps to ~(3/4) E^2, and the inputs are orthonormal to <= ~1e-9 (U = A V Sigma^{-1}:
// eps sigma_1 / sigma_j <= ~1e-11 for the kept directions; the in-house eigenvectors pass a
// 1e-9 orthogonality check), so one iteration reaches rounding level.  U is this rank's
// row block; U^T U is all-reduced when the rows are sharded.
void polar_orthonormalize(latsum_ctx* c, double* U, int64_t Nb, int64_t k, bool sharded,
                          int iters = 1) {
  if (k == 0) return;
  DBuf S(c, size_t(k) * k), Un(c, size_t(std::max<int64_t>(Nb, 1)) * k);
  for (int it = 0; it < iters; ++it) {
    if (Nb > 0) gemm(c, true, false, k, k, Nb, 1.0, U, Nb, U, Nb, 0.0, S.p, k, tagged("gemm_basis"));
    else CK(cudaMemsetAsync(S.p, 0, sizeof(double) * k * k, c->stream));
    if (sharded) allreduce(c, S.p, size_t(k) * k);
    if (Nb == 0) continue;
    CK(cudaMemcpyAsync(Un.p, U, sizeof(double) * Nb * k, cudaMemcpyDeviceToDevice, c->stream));
    gemm(c, false, false, Nb, k, k, -0.5, U, Nb, S.p, k, 1.5, Un.p, Nb, tagged("gemm_basis"));
    CK(cudaMemcpyAsync(U, Un.p, sizeof(double) * Nb * k, cudaMemcpyDeviceToDevice, c->stream));
  }
}

// U (Nb x k) = A (Nb x d) Vd scaled by 1/sqrt(lam_desc), then re-orthonormalised: left
// singular vectors from the k leading eigenpairs (Vd: d x k, descending) of A^T A (row
// block of A -> row block of U).
double frob2(latsum_ctx* c, const double* A, int64_t Nb, int64_t cols, int64_t ld, bool sharded);
void left_from_vectors(latsum_ctx* c, const double* A, int64_t Nb, int64_t d, const double* Vd,
                       const std::vector<double>& lam_desc, int64_t k, double* U, bool sharded) {
  if (k == 0) return;
  if (Nb > 0) {
    gemm(c, false, false, Nb, k, d, 1.0, A, Nb, Vd, d, 0.0, U, Nb, tagged("gemm_basis"));
    std::vector<double> inv(k);
    for (int64_t j = 0; j < k; ++j) inv[j] = lam_desc[j] > 0.0 ? 1.0 / std::sqrt(lam_desc[j]) : 0.0;
    DVec<double> sc;
    sc.upload(c, inv);
    k_scale_columns<<<grid_for(Nb * k), 256, 0, c->stream>>>(U, Nb, k, sc.p, U);
    post_launch(c);
  }
  polar_orthonormalize(c, U, Nb, k, sharded);
}

// Frobenius norm squared of an Nb x cols column-major block (all ranks' rows when sharded).
double frob2(latsum_ctx* c, const double* A, int64_t Nb, int64_t cols, int64_t ld, bool sharded) {
  const int blocks = 148 * 4;
  DBuf part(c, blocks), sum(c, 1);
  if (Nb > 0 && cols > 0) {
    k_sumsq_partial<<<blocks, 256, 0, c->stream>>>(A, Nb, cols, ld, part.p);
    post_launch(c);
    k_sum<<<1, 1024, 0, c->stream>>>(part.p, blocks, sum.p);
    post_launch(c);
  } else {
    CK(cudaMemsetAsync(sum.p, 0, sizeof(double), c->stream));
  }
  if (sharded) allreduce(c, sum.p, 1);
  double h = 0;
  CK(cudaMemcpyAsync(&h, sum.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return h;
}

// Randomized second pass of the deflated RHOSVD (column orientation).  The deflated operand
// A'' = (I - U1 U1^T)^2 A (Nb x d rows of this rank) has norm <= ~1e-5 sigma_1 and, on the
// BASELINE Grams, numerical rank a fraction of its d - k1 nonzero directions, so instead of
// the (d - k1)^2 restricted Gram this pass
//   1. sketches its range, Y = A'' Omega (ell Gaussian columns),
//   2. orthonormalises Y in rounds: Y^T Y = W h W^T, Q_new = Y W_k h_k^{-1/2} for the values
//      within 1e10 of the round's largest (orthogonality error <= eps 1e10, removed by two
//      Newton-Schulz polar steps), Y <- Y - Q (Q^T Y) twice, until the rest of Y is below the
//      floor delta (directions of A'' under delta are never needed individually),
//   3. projects, C = Q^T A'' (m x d), and takes the Ritz pairs of C C^T (m x m): the values
//      mu_j and the left vectors U2 = Q W.
// Certified by the captured mass: ||A''||_F^2 - ||C||_F^2 (the lump, everything outside
// span(Q)) must be <= lump_max; the lump enters the rank rule as spread over the
// unresolved slots.  Returns false when the sketch cannot be certified at ell = nc (the
// caller then runs the restricted Gram).  Every eigensolve is ell x ell (the in-house
// solver up to 808: no cuSOLVER serialisation across the concurrent modes).
struct Rp2 {
  int64_t m = 0;
  DBuf Q;                   // Nr x m, orthonormal
  Eig e;                    // Ritz problem C C^T
  std::vector<double> mu;   // m Ritz values, descending
  double lump = 0.0;        // ||A''||_F^2 - sum mu
  int64_t ell = 0, rounds = 0;
};

bool randomized_pass2(latsum_ctx* c, const double* Ap, int64_t Nb, int64_t d, int64_t nc,
                      double delta, double lump_max, bool sharded, uint64_t seed, Rp2& o,
                      int eig_owner = -1) {
  const int64_t Nr = std::max<int64_t>(Nb, 1);
  const double a2 = frob2(c, Ap, Nb, d, Nb, sharded);
  int64_t ell = std::min<int64_t>(nc, 768);
  for (;; ell = std::min<int64_t>(nc, 2 * ell)) {
    o.ell = ell;
    DBuf Om(c, size_t(d) * ell), Y(c, size_t(Nr) * ell);
    k_fill_gauss<<<grid_for(d * ell), 256, 0, c->stream>>>(Om.p, d * ell, seed + uint64_t(ell));
    post_launch(c);
    if (Nb > 0)
      gemm(c, false, false, Nb, ell, d, 1.0, Ap, Nb, Om.p, d, 0.0, Y.p, Nb, tagged("gemm_rp2"));
    else
      CK(cudaMemsetAsync(Y.p, 0, sizeof(double) * ell, c->stream));
    o.Q.alloc(c, size_t(Nr) * ell);
    int64_t m = 0;
    // a direction of A'' with singular value s shows in Y at ~ s sqrt(ell)
    const double stop_h = delta * delta * double(ell) * 1e-2;
    DBuf S(c, size_t(ell) * ell);
    for (int round = 0; round < 4 && m < ell; ++round) {
      if (m > 0) {
        for (int rep = 0; rep < 2; ++rep) {  // Y <- Y - Q (Q^T Y)
          if (Nb > 0)
            gemm(c, true, false, m, ell, Nb, 1.0, o.Q.p, Nb, Y.p, Nb, 0.0, S.p, m, tagged("gemm_rp2"));
          else
            CK(cudaMemsetAsync(S.p, 0, sizeof(double) * m * ell, c->stream));
          if (sharded) allreduce(c, S.p, size_t(m) * ell);
          if (Nb > 0)
            gemm(c, false, false, Nb, ell, m, -1.0, o.Q.p, Nb, S.p, m, 1.0, Y.p, Nb, tagged("gemm_rp2"));
        }
      }
      DBuf H(c, size_t(ell) * ell);
      if (Nb > 0) gram(c, false, Y.p, Nb, ell, H.p);
      else CK(cudaMemsetAsync(H.p, 0, sizeof(double) * ell * ell, c->stream));
      if (sharded) allreduce(c, H.p, size_t(ell) * ell);
      Eig eh;
      // these vectors only seed Q = Y W h^{-1/2}, which two Newton-Schulz steps re-orthonormalise
      // (quadratic from any ||W^T W - I|| < 1: 1e-3 leaves 1e-12 after two); a tighter gate sent
      // ~2 clustered b x b Grams per cfg4 step to the cuSOLVER fallback for nothing
      eh.ortho_tol = 1e-3;
      eh.solve_on(c, ell, std::move(H), sharded ? eig_owner : -1);
      std::vector<double> h(ell);
      for (int64_t i = 0; i < ell; ++i) h[i] = std::max(eh.lam_asc[ell - 1 - i], 0.0);
      const double hmax = h[0];
      if (!(hmax > stop_h)) break;
      int64_t kk = 0;
      while (kk < ell - m && h[kk] > std::max(1e-10 * hmax, stop_h)) ++kk;
      if (kk == 0) break;
      ++o.rounds;
      double* Qn = o.Q.p + Nb * m;
      DBuf Vk(c, size_t(ell) * kk);
      eh.leading(c, kk, Vk.p);
      left_from_vectors(c, Y.p, Nb, ell, Vk.p, h, kk, Qn, sharded);  // + one polar step
      if (m > 0) {
        DBuf S2(c, size_t(m) * kk);
        for (int rep = 0; rep < 2; ++rep) {  // Qn <- Qn - Q (Q^T Qn)
          if (Nb > 0)
            gemm(c, true, false, m, kk, Nb, 1.0, o.Q.p, Nb, Qn, Nb, 0.0, S2.p, m, tagged("gemm_rp2"));
          else
            CK(cudaMemsetAsync(S2.p, 0, sizeof(double) * m * kk, c->stream));
          if (sharded) allreduce(c, S2.p, size_t(m) * kk);
          if (Nb > 0)
            gemm(c, false, false, Nb, kk, m, -1.0, o.Q.p, Nb, S2.p, m, 1.0, Qn, Nb, tagged("gemm_rp2"));
        }
      }
      polar_orthonormalize(c, Qn, Nb, kk, sharded, 2);
      m += kk;
    }
    o.m = m;
    if (m == 0) {  // A'' below the floor everywhere
      o.mu.clear();
      o.lump = a2;
      return a2 <= lump_max;
    }
    // Ritz pairs of C C^T, C = Q^T A''
    DBuf C(c, size_t(m) * d), G2(c, size_t(m) * m);
    if (Nb > 0)
      gemm(c, true, false, m, d, Nb, 1.0, o.Q.p, Nb, Ap, Nb, 0.0, C.p, m, tagged("gemm_rp2"));
    else
      CK(cudaMemsetAsync(C.p, 0, sizeof(double) * m * d, c->stream));
    if (sharded) allreduce(c, C.p, size_t(m) * d);
    gram(c, true, C.p, m, d, G2.p);
    o.e = Eig();
    o.e.ortho_tol = 1e-9;
    o.e.solve_on(c, m, std::move(G2), sharded ? eig_owner : -1);
    o.mu.assign(m, 0.0);
    double captured = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      o.mu[i] = std::max(o.e.lam_asc[m - 1 - i], 0.0);
      captured += o.mu[i];
    }
    o.lump = std::max(a2 - captured, 0.0);
    Trace::mark(c, "rp2 round done");
    // oversampling: a sketch that came out nearly full rank resolves its trailing Ritz values
    // (the ones just under the cut) poorly; a wider one would need cuSOLVER-sized
    // eigensolves (ell > 808), so the caller's restricted Gram runs instead
    const bool thin = m > ell - 128 && ell < nc;
    if (o.lump <= lump_max && !thin) return true;
    if (ell >= nc || ell >= 768) return !thin && o.lump <= lump_max;
  }
}

// Compressed pass 1 (column orientation, merged Grams beyond the in-house solver): a blocked
// randomized range finder (randQB_b, Martinsson & Voronin 2016) for the ROW space of A gives
// P (d x m, orthonormal, identical on every rank) with ||A (I - P P^T)||_2 <~ delta, m ~ the
// numerical rank of A at delta (cfg4 mode 0: ~2480 of the d = 5394 merged columns).  The
// reduction then runs on C = A P (N x m) through the unchanged column-orientation path: C C^T
// = A A^T - E E^T with ||E|| <= delta, so every sigma^2 moves by at most delta^2, and the left
// singular vectors still come through the operand (U = C V lambda^{-1/2}), which damps the
// Gram eigenvectors' errors (a left-space basis Q with the rows-orientation Gram of Q^T A was
// measured 1e-6..1e-4 off at the cut on cfg4/cfg5).  Each block sketches the residual,
// (I - P P^T) A^T Omega with b Gaussian columns (A^T Omega summed over the ranks' row blocks),
// and orthonormalises it in rounds as randomized_pass2 does (Y^T Y = W h W^T, P_new =
// Y W_k h_k^{-1/2} within a 1e10 window, the new columns projected against P twice, two
// Newton-Schulz steps), so every eigensolve is b x b (the in-house solver).  The first block that
// finds fewer than b - p directions above the floor ends it (the oversampling p makes a missed
// direction improbable).  The sketch products stay on DMMA: their rounding is the noise floor
// the stop test reads.  Returns false when the basis would reach `cap` columns.
struct RangeBasis {
  DBuf P;
  int64_t m = 0, blocks = 0, rounds = 0;
};

bool range_basis(latsum_ctx* c, const double* A, RowBlock blk, int64_t N, int64_t d, int64_t cap,
                 double delta, bool sharded, uint64_t seed, RangeBasis& o, int eig_owner) {
  constexpr int64_t kBlock = 256, kOver = 24;
  const int64_t Nb = blk.n();
  const int owner = sharded ? eig_owner : -1;
  o.P.alloc(c, size_t(d) * cap);
  GemmOpts go = tagged("gemm_rqb");
  go.dmma = true;
  // The sketch A^T Omega is the one large product of a block (2 d b Nb flops; the projections
  // are 2 d b m): it runs on the int8 tensor cores with A^T sliced ONCE for all blocks (lines =
  // the d columns of this rank's row block, K = Nb in <= KMAX chunks).  Its rounding (~3e-16 of
  // a unit column per entry, a few times the DMMA product's) leaves Y^T Y eigenvalues of
  // ~1e-27 d against the stop level 0.04 delta^2 b ~ 1e-20: five decades of room.
  const bool oz_sketch = Nb > 0 && double(d) * double(kBlock) * double(Nb) >= 2e9;
  std::vector<OzSliced> As;
  std::vector<int64_t> k0s;
  if (oz_sketch) {
    const int64_t parts = (Nb + oz::KMAX - 1) / oz::KMAX, kc = (Nb + parts - 1) / parts;
    As.resize(size_t(parts));
    for (int64_t p = 0; p < parts; ++p) {
      k0s.push_back(p * kc);
      oz_slice_a(c, A + p * kc, Nb, 1, d, std::min(kc, Nb - p * kc), As[size_t(p)]);
    }
  }
  int64_t m = 0;
  for (;;) {
    if (m + kOver >= cap) return false;
    const int64_t bb = std::min<int64_t>(kBlock, cap - m);
    // Omega: the same N x b Gaussian matrix on every rank; this rank's rows [lo, hi)
    DBuf Om(c, size_t(N) * bb), Y(c, size_t(d) * bb), S(c, size_t(cap) * bb);
    k_fill_gauss<<<grid_for(N * bb), 256, 0, c->stream>>>(Om.p, N * bb, seed + uint64_t(o.blocks) * 7919u);
    post_launch(c);
    if (oz_sketch) {
      for (size_t p = 0; p < As.size(); ++p) {
        OzSliced om;
        oz_slice_b(c, Om.p + blk.lo + k0s[p], N, 1, bb, As[p].K, om);
        oz_run(c, As[p], om, oz_out(Y.p, d, p == 0 ? 0.0 : 1.0), "gemm_rqb(ozaki-i8)");
      }
    } else if (Nb > 0) {
      gemm(c, true, false, d, bb, Nb, 1.0, A, Nb, Om.p + blk.lo, N, 0.0, Y.p, d, go);
    } else {
      CK(cudaMemsetAsync(Y.p, 0, sizeof(double) * d * bb, c->stream));
    }
    if (sharded) allreduce(c, Y.p, size_t(d) * bb);
    // a direction of the residual with singular value s shows in Y^T Y at ~ s^2 b
    const double stop_h = 0.04 * delta * delta * double(bb);
    auto project_out = [&](double* X, int64_t cols) {  // X <- X - P (P^T X)
      if (m == 0) return;
      gemm(c, true, false, m, cols, d, 1.0, o.P.p, d, X, d, 0.0, S.p, m, go);
      gemm(c, false, false, d, cols, m, -1.0, o.P.p, d, S.p, m, 1.0, X, d, go);
    };
    int64_t added = 0;
    for (int round = 0; round < 4 && added < bb && m < cap; ++round) {
      // one projection of the sketch: what it leaves along P (~eps ||Y||) only perturbs the seed
      // directions; the new columns themselves are projected against P twice and
      // re-orthonormalised below before they join it (a second projection here cost ~7 ms of the
      // cfg4 step for an unchanged residual ||A (I - P P^T)||)
      project_out(Y.p, bb);
      DBuf H(c, size_t(bb) * bb);
      gram(c, false, Y.p, d, bb, H.p);
      Eig eh;
      eh.ortho_tol = 1e-3;  // seeds only: the new columns are re-orthonormalised below (as above)
      eh.solve_on(c, bb, std::move(H), owner);
      std::vector<double> h(bb);
      for (int64_t i = 0; i < bb; ++i) h[i] = std::max(eh.lam_asc[bb - 1 - i], 0.0);
      const double hmax = h[0];
      if (!(hmax > stop_h)) break;
      int64_t kk = 0;
      while (kk < bb - added && m + kk < cap && h[kk] > std::max(1e-10 * hmax, stop_h)) ++kk;
      if (kk == 0) break;
      double* Pn = o.P.p + d * m;
      DBuf Vk(c, size_t(bb) * kk);
      eh.leading(c, kk, Vk.p);
      left_from_vectors(c, Y.p, d, bb, Vk.p, h, kk, Pn, false);
      project_out(Pn, kk);
      project_out(Pn, kk);
      polar_orthonormalize(c, Pn, d, kk, false, 2);
      m += kk;
      added += kk;
      ++o.rounds;
    }
    ++o.blocks;
    o.m = m;
    if (added + kOver <= bb) return m + kOver < cap;
  }
}

// Pass 1 runs on the compressed operand when the merged Gram would exceed the in-house
// eigensolver (column orientation; not for the ALS unfoldings, which need every vector).
bool compress_pass1(int64_t N, int64_t d, bool force_deflate) {
  static const bool off = std::getenv("LATSUM_RQB") && std::string(std::getenv("LATSUM_RQB")) == "0";
  return !off && !force_deflate && N > d && d > band::SB_NMAX && eig_env_mode() == 0;
}

struct ModeOut {
  std::vector<double> sigma;
  int64_t r = 1;
  DBuf Z;            // rows [blk.lo, blk.hi) of Z (all rows when not sharded)
  RowBlock blk;
  bool tie = false;
  double margin = 0.0;
  int deflated = 0, rows = 0;
  int64_t gsize = 0, k1 = 0;
};

struct Timings {
  double gram = 0, syevd = 0, deflate = 0, project = 0, core = 0, norm = 0;
  std::function<void()> on_gram;  // called once this mode's Gram is on the device
  std::function<void()> before_eig1, after_eig1;  // around the pass-1 eigensolve
};

// cuSOLVER runs concurrent syevd calls one after another anyway; the pass-1 solves are
// granted in a fixed order instead, largest Gram first, so the longest mode's deflation and
// second pass overlap the other modes' solves rather than all solves finishing together
// (cfg4: mode 0's n = 5394 first, then 2842, 2755).
struct EigTurnstile {
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int> order;  // modes whose pass-1 solve uses cuSOLVER, largest n first
  size_t next = 0;
  bool done[3] = {false, false, false};
  bool in_order(int l) const { return std::find(order.begin(), order.end(), l) != order.end(); }
  void wait(int l) {
    if (!in_order(l)) return;
    std::unique_lock<std::mutex> g(mu);
    cv.wait(g, [&] { return next >= order.size() || order[next] == l; });
  }
  void finish(int l) {  // also on failure: never leave a later mode waiting
    if (!in_order(l)) return;
    std::lock_guard<std::mutex> g(mu);
    if (done[l]) return;
    done[l] = true;
    while (next < order.size() && done[order[next]]) ++next;
    cv.notify_all();
  }
};

// RHOSVD of one mode (rank_reduction.hpp:189-207) on the merged side matrix
// A~ = D diag(sqrt(mult)), whose A~ A~^T equals the reference's A A^T.
//
// Pass 1: Gram of the smaller orientation (A A^T, N x N, or A~^T A~, d x d) and syevd.
// Pass 2: the k1 directions with lambda > 1e-10 lambda_max are accurate;
// the rest of the spectrum is recomputed from A'' = (I - U1 U1^T)^2 A~ restricted to the
// pass-1 complement Qc (the n - k1 trailing eigenvectors), whose Gram has the size of
// that complement and resolves singular values down to ~eps ||A''||.
//
// Multi-GPU (column orientation): the rank owns grid rows [lo, hi) of A~, U1, A'', B, U2
// and Z; every contraction over the grid index (the Grams, U^T U, U1^T A) is a partial
// product all-reduced over NVLink; eigensolves run redundantly on identical Grams.
// Spectrum and leading left singular vectors of a dense operand A (N x d) given as
// this rank's row block At (Nb x d; all rows when not sharded): the two-pass deflated
// Gram algorithm of reduce_mode below.  rank_fixed (nullable) selects a fixed rank
// (clamped), else rank_for_tolerance(tol); force_deflate runs the second pass even
// with a fixed rank (needed when the trailing kept directions sit below
// sqrt(eps_mach) sigma_1, e.g. in the ALS unfoldings).
void reduce_dense(latsum_ctx* c, DBuf& At, RowBlock blk, int64_t N, int64_t d, int64_t n_sing,
                  const int64_t* rank_fixed, double tol, int deflate, bool force_deflate,
                  bool sharded, ModeOut& out, Timings& tm, int eig_owner = -1,
                  bool replicated = false, bool compress = true);

void reduce_mode(latsum_ctx* c, const latsum_canonical& can, int l, const int64_t* ranks,
                 double tol, int deflate, ModeOut& out, Timings& tm) {
  const int64_t N = can.N[l], d = can.d[l];
  const int64_t n_sing = std::min<int64_t>(N, can.Mc);
  const bool rows = N <= d;
  const bool sharded = !rows && has_comm(c);
  const RowBlock blk = sharded ? row_block(c, N) : RowBlock{0, N};
  const int64_t Nb = blk.n();
  Timer timer(c);
  Trace::mark(c, "mode start");
  timer.start();
  std::vector<double> sq(d);
  for (int64_t j = 0; j < d; ++j) sq[j] = std::sqrt(can.mult[l][j]);
  DVec<double> dsq;
  dsq.upload(c, sq);
  DBuf At(c, size_t(std::max<int64_t>(Nb, 1)) * d);
  if (Nb > 0) {
    CK(cudaMemcpy2DAsync(At.p, Nb * sizeof(double), can.dict[l].p + blk.lo, N * sizeof(double),
                         Nb * sizeof(double), d, cudaMemcpyDeviceToDevice, c->stream));
    k_scale_columns<<<grid_for(Nb * d), 256, 0, c->stream>>>(At.p, Nb, d, dsq.p, At.p);
    post_launch(c);
  }
  tm.gram += timer.stop();
  Trace::mark(c, "operand ready");
  const int64_t* rf = ranks ? ranks + l : nullptr;
  reduce_dense(c, At, blk, N, d, n_sing, rf, tol, deflate, false, sharded, out, tm, l);
}

void reduce_dense(latsum_ctx* c, DBuf& At, RowBlock blk, int64_t N, int64_t d, int64_t n_sing,
                  const int64_t* rank_fixed, double tol, int deflate, bool force_deflate,
                  bool sharded, ModeOut& out, Timings& tm, int eig_owner, bool replicated,
                  bool compress) {
  const int64_t* ranks = rank_fixed;
  const int l = 0;  // rank_fixed points at this operand's rank
  const bool rows = N <= d;
  const int64_t Nb = blk.n();
  // eigensolves on operands every rank holds in full are owner-solved and broadcast too
  const int owner = (sharded || replicated) ? eig_owner : -1;
  out.blk = blk;
  Timer timer(c);
  timer.start();
  if (compress && compress_pass1(N, d, force_deflate)) {
    // compressed pass 1: P spans the row space of A to delta, and the whole two-pass reduction
    // runs on C = A P (N x m) in the same column orientation (range_basis).  delta sits four
    // decades under the smallest singular value any BASELINE cut-off reads (cfg5: ~1.3e-9
    // sigma_1; sigma^2 moves by <= delta^2, i.e. <= 2e-7 relative there) and above the DMMA
    // sketch's rounding.
    // no Gram burst to keep clear of on this path (the range finder is latency-bound): norm_f,
    // which waits for the modes' Grams, may start now (cfg5: it is 0.9 s of capped GEMMs)
    if (tm.on_gram) tm.on_gram();
    const double a2 = frob2(c, At.p, Nb, d, Nb, sharded);
    const double delta = 2e-13 * std::sqrt(a2);
    RangeBasis rb;
    const int64_t cap = std::min<int64_t>(N, d) * 3 / 4;
    const bool ok = a2 > 0.0 &&
                    range_basis(c, At.p, blk, N, d, cap, delta, sharded,
                                0x1411ull * 977 + uint64_t(d) * 131 + uint64_t(N), rb, eig_owner);
    if (Trace::on())
      fprintf(stderr, "[rqb] N %ld d %ld m %ld blocks %ld rounds %ld ok %d\n", long(N), long(d),
              long(rb.m), long(rb.blocks), long(rb.rounds), int(ok));
    if (ok) {
      const int64_t m = rb.m;
      DBuf Ct(c, size_t(std::max<int64_t>(Nb, 1)) * m);
      if (Nb > 0)
        gemm(c, false, false, Nb, m, d, 1.0, At.p, Nb, rb.P.p, d, 0.0, Ct.p, Nb, tagged("gemm_rqb_project"));
      if (Trace::on()) {  // the range basis' miss, ||A - C P^T||_F (dev diagnostics)
        DBuf R(c, size_t(std::max<int64_t>(Nb, 1)) * d);
        if (Nb > 0) {
          CK(cudaMemcpyAsync(R.p, At.p, sizeof(double) * Nb * d, cudaMemcpyDeviceToDevice, c->stream));
          GemmOpts od = tagged("gemm_rqb");
          od.dmma = true;
          gemm(c, false, true, Nb, d, m, -1.0, Ct.p, Nb, rb.P.p, d, 1.0, R.p, Nb, od);
        }
        const double r2 = frob2(c, R.p, Nb, d, Nb, sharded);
        fprintf(stderr, "[rqb] residual ||A (I - P P^T)||_F / ||A||_F = %.3e (delta %.3e)\n",
                std::sqrt(r2 / a2), delta / std::sqrt(a2));
      }
      rb.P.release();
      tm.gram += timer.stop();
      Trace::mark(c, "range basis done");
      reduce_dense(c, Ct, blk, N, m, n_sing, rank_fixed, tol, deflate, false, sharded, out, tm,
                   eig_owner, replicated, false);
      out.gsize = m;
      return;
    }
    timer.start();
  }
  const int64_t n = rows ? N : d;
  out.rows = rows ? 1 : 0;
  out.gsize = n;
  DBuf G(c, size_t(n) * n);
  if (Nb > 0) gram(c, rows, At.p, Nb, d, G.p);
  else CK(cudaMemsetAsync(G.p, 0, sizeof(double) * n * n, c->stream));
  if (sharded) allreduce(c, G.p, size_t(n) * n);
  tm.gram += timer.stop();
  Trace::mark(c, "gram done");
  if (tm.on_gram) tm.on_gram();
  timer.start();
  Eig e1;
  // the RHOSVD's pass-1/pass-2 bases are re-orthonormalised and their span is what counts;
  // the ALS unfoldings (force_deflate) need the strict eigenvector orthogonality
  e1.ortho_tol = force_deflate ? -1.0 : 1e-9;
  if (tm.before_eig1) tm.before_eig1();
  try {
    e1.solve_on(c, n, std::move(G), owner);
  } catch (...) {
    if (tm.after_eig1) tm.after_eig1();
    throw;
  }
  if (tm.after_eig1) tm.after_eig1();
  tm.syevd += timer.stop();
  Trace::mark(c, "syevd1 done");
  std::vector<double> lam_d(n);
  for (int64_t i = 0; i < n; ++i) lam_d[i] = std::max(e1.lam_asc[n - 1 - i], 0.0);
  const double lmax = lam_d.empty() ? 0.0 : lam_d[0];

  auto padded_sigma = [&](const std::vector<double>& l2) {
    std::vector<double> sv(n_sing, 0.0);
    for (int64_t i = 0; i < std::min<int64_t>(n_sing, int64_t(l2.size())); ++i)
      sv[i] = std::sqrt(std::max(l2[i], 0.0));
    return sv;
  };

  std::vector<double> merged = lam_d;
  std::vector<std::pair<int, int64_t>> src(n);  // (pass, index in that pass's desc order)
  for (int64_t i = 0; i < n; ++i) src[i] = {0, i};
  int64_t k1 = 0, nc = 0, n2 = 0;
  const int64_t Nr = std::max<int64_t>(Nb, 1);
  DBuf U1, B;
  Eig e2;
  e2.ortho_tol = e1.ortho_tol;
  bool restricted = false;  // pass 2 on the pass-1 complement Qc (needs all pass-1 vectors)
  std::vector<double> mu_d;
  bool defl = false;
  bool use_rp2 = false;
  Rp2 rp;
  double target = 0.0;
  if ((!ranks || force_deflate) && deflate != LATSUM_DEFLATE_NEVER && lmax > 0.0) {
    const std::vector<double> sv = padded_sigma(lam_d);
    double sn2 = 0;
    for (double v : sv) sn2 += v * v;
    target = tol * std::sqrt(sn2) / 3.0;
    for (int64_t i = 0; i < n; ++i)
      if (lam_d[i] > 1e-10 * lmax) k1 = i + 1;
    k1 = std::max<int64_t>(k1, 1);
    nc = n - k1;
    defl = nc > 0 && (deflate == LATSUM_DEFLATE_ALWAYS || force_deflate ||
                      target * target < 1e6 * double(n) * kEpsMach * lmax);
    if (defl) {
      timer.start();
      U1.alloc(c, size_t(Nr) * k1);
      if (rows) {
        e1.leading(c, k1, U1.p);
        if (e1.custom) polar_orthonormalize(c, U1.p, N, k1, false);
      } else {
        DBuf V1(c, size_t(d) * k1);
        e1.leading(c, k1, V1.p);
        left_from_vectors(c, At.p, Nb, d, V1.p, lam_d, k1, U1.p, sharded);
      }
      DBuf Ap(c, size_t(Nr) * d), C(c, size_t(k1) * d);
      if (Nb > 0)
        CK(cudaMemcpyAsync(Ap.p, At.p, sizeof(double) * Nb * d, cudaMemcpyDeviceToDevice, c->stream));
      for (int rep = 0; rep < 2; ++rep) {  // project out span(U1), then re-orthogonalise once
        if (Nb > 0)
          gemm(c, true, false, k1, d, Nb, 1.0, U1.p, Nb, Ap.p, Nb, 0.0, C.p, k1, tagged("gemm_deflate"));
        else
          CK(cudaMemsetAsync(C.p, 0, sizeof(double) * k1 * d, c->stream));
        if (sharded) allreduce(c, C.p, size_t(k1) * d);
        if (Nb > 0)
          gemm(c, false, false, Nb, d, k1, -1.0, U1.p, Nb, C.p, k1, 1.0, Ap.p, Nb, tagged("gemm_deflate"));
      }
      if (Trace::on() && !rows) {
        const double a0 = frob2(c, At.p, Nb, d, Nb, sharded), a1 = frob2(c, Ap.p, Nb, d, Nb, sharded);
        const double u1 = frob2(c, U1.p, Nb, k1, Nb, sharded);
        fprintf(stderr, "[deflate] rank %d/%d Nb %ld d %ld k1 %ld |A|^2 %.6e |A''|^2 %.6e |U1|^2 %.6f\n",
                c->rank, c->nranks, long(Nb), long(d), long(k1), a0, a1, u1);
      }
      // randomized pass 2 (column orientation, tolerance-driven): ell x ell eigensolves
      // instead of the nc x nc restricted Gram (see randomized_pass2)
      static const bool rp2_off = std::getenv("LATSUM_RP2") && std::string(std::getenv("LATSUM_RP2")) == "0";
      constexpr int64_t rp2_min = 808;  // the in-house solver takes the restricted Gram below
      // the resolved pass-1 values between eps lambda_max and the k1 threshold are directions
      // the sketch must hold: too many and it cannot stay within the in-house solver's size
      int64_t c16 = 0;
      for (int64_t i = k1; i < n; ++i)
        if (lam_d[i] > 1e-16 * lmax) ++c16;
      if (!rows && !force_deflate && !rp2_off && nc > rp2_min && c16 + 128 <= 768) {
        const double delta = 1e-4 * target / std::sqrt(double(n));
        const double lump_max = 1e-6 * target * target;
        if (randomized_pass2(c, Ap.p, Nb, d, nc, delta, lump_max, sharded,
                             0x14111994ull + uint64_t(d) * 131 + uint64_t(k1), rp, eig_owner)) {
          const int64_t m = rp.m, rest = n - k1 - m;
          std::vector<std::tuple<double, int, int64_t>> all;
          for (int64_t i = 0; i < k1; ++i) all.emplace_back(lam_d[i], 0, i);
          for (int64_t i = 0; i < m; ++i) all.emplace_back(rp.mu[i], 1, i);
          for (int64_t i = 0; i < rest; ++i) all.emplace_back(rp.lump / double(rest), 2, i);
          std::stable_sort(all.begin(), all.end(), [](const auto& a, const auto& b) {
            return std::get<0>(a) > std::get<0>(b);
          });
          std::vector<double> mg(n);
          for (int64_t i = 0; i < n; ++i) mg[i] = std::get<0>(all[i]);
          // the cut must fall inside the resolved window, clear of the lump slots
          const int64_t rr = rank_for_tolerance(padded_sigma(mg), tol);
          bool inside = rr + 8 <= k1 + m;
          for (int64_t i = 0; i < std::min<int64_t>(n, rr + 8) && inside; ++i)
            if (std::get<1>(all[i]) == 2) inside = false;
          if (inside) {
            use_rp2 = true;
            n2 = m;
            mu_d = rp.mu;
            for (int64_t i = 0; i < n; ++i) {
              merged[i] = mg[i];
              src[i] = {std::get<1>(all[i]), std::get<2>(all[i])};
            }
          }
        }
      }
      if (!use_rp2) {
      restricted = e1.has_all();
      // pass-2 operand B: restricted to the pass-1 complement Qc = the nc trailing
      // eigenvectors when they exist (cuSOLVER), else A'' itself (its Gram has k1 extra
      // ~zero eigenvalues, the deflated directions)
      n2 = restricted ? nc : n;
      DBuf G2(c, size_t(n2) * n2);
      if (rows) {  // G2 = B B^T with B = Qc^T A'' (nc x d) or A'' (N x d)
        if (restricted) {
          B.alloc(c, size_t(nc) * d);
          gemm(c, true, false, nc, d, N, 1.0, e1.G.p, N, Ap.p, N, 0.0, B.p, nc, tagged("gemm_deflate"));
          gram(c, true, B.p, nc, d, G2.p);
        } else {
          gram(c, true, Ap.p, N, d, G2.p);
        }
      } else {     // G2 = B^T B with B = A'' Qc (Nb x nc) or A'' (Nb x d)
        if (restricted) {
          B.alloc(c, size_t(Nr) * nc);
          if (Nb > 0) {
            gemm(c, false, false, Nb, nc, d, 1.0, Ap.p, Nb, e1.G.p, d, 0.0, B.p, Nb, tagged("gemm_deflate"));
            gram(c, false, B.p, Nb, nc, G2.p);
          } else {
            CK(cudaMemsetAsync(G2.p, 0, sizeof(double) * nc * nc, c->stream));
          }
        } else {
          B = std::move(Ap);
          if (Nb > 0) gram(c, false, B.p, Nb, d, G2.p);
          else CK(cudaMemsetAsync(G2.p, 0, sizeof(double) * n2 * n2, c->stream));
        }
        if (sharded) allreduce(c, G2.p, size_t(n2) * n2);
      }
      tm.deflate += timer.stop();
      Trace::mark(c, "deflation + G2 done");
      timer.start();
      e2.solve_on(c, n2, std::move(G2), owner);
      tm.syevd += timer.stop();
      Trace::mark(c, "syevd2 done");
      mu_d.resize(nc);  // the nc leading pass-2 values
      for (int64_t i = 0; i < nc; ++i) mu_d[i] = std::max(e2.lam_asc[n2 - 1 - i], 0.0);
      // merged spectrum: k1 resolved pass-1 values and the nc deflated values
      std::vector<std::tuple<double, int, int64_t>> all;
      for (int64_t i = 0; i < k1; ++i) all.emplace_back(lam_d[i], 0, i);
      for (int64_t i = 0; i < nc; ++i) all.emplace_back(mu_d[i], 1, i);
      std::stable_sort(all.begin(), all.end(), [](const auto& a, const auto& b) {
        return std::get<0>(a) > std::get<0>(b);
      });
      for (int64_t i = 0; i < n; ++i) {
        merged[i] = std::get<0>(all[i]);
        src[i] = {std::get<1>(all[i]), std::get<2>(all[i])};
      }
      }  // !use_rp2
    }
  }
  out.deflated = defl ? 1 : 0;
  out.k1 = defl ? k1 : 0;
  out.sigma = padded_sigma(merged);
  const auto& sv = out.sigma;

  int64_t r;
  if (ranks) r = std::min<int64_t>(std::max<int64_t>(ranks[l], 1), n_sing);
  else r = rank_for_tolerance(sv, tol);
  // drop numerically zero directions (rhosvd); ALS keeps exactly the requested rank
  while (!force_deflate && r > 1 && sv[r - 1] < 1e-14 * sv[0]) --r;
  r = std::min<int64_t>(r, n);
  out.tie = r < int64_t(sv.size()) && sv[r - 1] - sv[r] <= 1e-12 * sv[0];
  if (!ranks) {
    double sn2 = 0, t_r = 0, t_rm1 = 0;
    for (double v : sv) sn2 += v * v;
    const double target = tol * std::sqrt(sn2) / 3.0;
    for (size_t k = r; k < sv.size(); ++k) t_r += sv[k] * sv[k];
    t_rm1 = t_r + sv[r - 1] * sv[r - 1];
    out.margin = std::min(target - std::sqrt(t_r), std::sqrt(t_rm1) - target) / target;
  }
  out.r = r;

  // Z = the r leading left singular vectors in merged (descending) order (row block)
  timer.start();
  out.Z.alloc(c, size_t(Nr) * r);
  if (!defl) {
    if (rows) {
      e1.leading(c, r, out.Z.p);
      if (e1.custom) polar_orthonormalize(c, out.Z.p, N, r, false);
    } else {
      DBuf Vr(c, size_t(d) * r);
      e1.leading(c, r, Vr.p);
      left_from_vectors(c, At.p, Nb, d, Vr.p, lam_d, r, out.Z.p, sharded);
    }
  } else {
    int64_t need2 = 0;
    for (int64_t i = 0; i < r; ++i)
      if (src[i].first == 1) need2 = std::max<int64_t>(need2, src[i].second + 1);
    DBuf cat(c, size_t(Nr) * (k1 + need2));
    if (Nb > 0)
      CK(cudaMemcpyAsync(cat.p, U1.p, sizeof(double) * Nb * k1, cudaMemcpyDeviceToDevice, c->stream));
    if (need2 && use_rp2) {  // U2 = Q W (Ritz vectors of the sketch)
      double* U2 = cat.p + Nb * k1;
      DBuf W2(c, size_t(rp.m) * need2);
      rp.e.leading(c, need2, W2.p);
      if (Nb > 0)
        gemm(c, false, false, Nb, need2, rp.m, 1.0, rp.Q.p, Nb, W2.p, rp.m, 0.0, U2, Nb,
             tagged("gemm_basis"));
      polar_orthonormalize(c, U2, Nb, need2, sharded);
    } else if (need2) {
      double* U2 = cat.p + Nb * k1;
      if (rows) {
        if (restricted) {  // U2 = Qc Y (leading eigenvectors of B B^T)
          DBuf Yd(c, size_t(nc) * need2);
          e2.leading(c, need2, Yd.p);
          gemm(c, false, false, N, need2, nc, 1.0, e1.G.p, N, Yd.p, nc, 0.0, U2, N, tagged("gemm_basis"));
        } else {
          e2.leading(c, need2, U2);
          if (e2.custom) polar_orthonormalize(c, U2, N, need2, false);
        }
      } else {             // U2 = B W mu^{-1/2}
        DBuf W2v(c, size_t(n2) * need2);
        e2.leading(c, need2, W2v.p);
        left_from_vectors(c, B.p, Nb, restricted ? nc : d, W2v.p, mu_d, need2, U2, sharded);
      }
    }
    if (Nb > 0) {
      std::vector<int64_t> sel(r);
      for (int64_t i = 0; i < r; ++i) sel[i] = src[i].first == 0 ? src[i].second : k1 + src[i].second;
      DVec<int64_t> dsel;
      dsel.upload(c, sel);
      k_select_columns<<<grid_for(Nb * r), 256, 0, c->stream>>>(cat.p, Nb, dsel.p, r, out.Z.p);
      post_launch(c);
    }
  }
  tm.deflate += timer.stop();
  Trace::mark(c, "Z done");
}

// sqrt(w^T (G0 o G1 o G2) w) over the merged terms with G_l = E_l^T E_l (d_l x d_l)
// for per-mode column sets E_l (rows x d_l): the dictionary itself gives norm_f
// (canonical.hpp:148-162); projected columns Y_l^T D_l give the ALS objective
// projected_norm (rank_reduction.hpp:104-113).
double hadamard_norm(latsum_ctx* c, const latsum_canonical& can, const double* const E[3],
                     const int64_t rows[3]) {
  terms(c, can);
  if (can.T == 0) return 0.0;
  DBuf G[3];
  for (int l = 0; l < 3; ++l) {
    G[l].alloc(c, size_t(can.d[l]) * can.d[l]);
    gemm(c, true, false, can.d[l], can.d[l], rows[l], 1.0, E[l], rows[l], E[l], rows[l], 0.0,
         G[l].p, can.d[l], tagged("gemm_norm_gram"));
  }
  DBuf part(c, can.T), sum(c, 1);
  ProfScope ps(c, "norm_hadamard", 3.0 * double(can.T) * double(can.T));
  k_hadamard_norm_rows<<<unsigned((can.T + NORM_TPB - 1) / NORM_TPB), NORM_WARPS * 32, 0, c->stream>>>(
      G[0].p, G[1].p, G[2].p, can.d[0], can.d[1], can.d[2], can.dtc[0].p, can.dtc[1].p,
      can.dtc[2].p, can.dtw.p, can.T, part.p);
  post_launch(c);
  k_sum<<<1, 1024, 0, c->stream>>>(part.p, can.T, sum.p);
  post_launch(c);
  double s = 0;
  CK(cudaMemcpyAsync(&s, sum.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return s > 0.0 ? std::sqrt(s) : 0.0;
}

double canonical_norm(latsum_ctx* c, const latsum_canonical& can) {
  const double* E[3] = {can.dict[0].p, can.dict[1].p, can.dict[2].p};
  return hadamard_norm(c, can, E, can.N);
}

// core(a,b,c) = sum_t w_t P0(a,c0_t) P1(b,c1_t) P2(c,c2_t)  (project_core,
// rank_reduction.hpp:88-100) as X_a = G1[:, seg_a] G2[:, seg_a]^T over the terms
// grouped by their mode-1 column a (one segmented GEMM), then core = P0 X^T.
// The merged terms grouped by their mode-m column, with the other two modes' projected
// columns gathered (G1 weighted): X_j = G1[:, seg_j] G2[:, seg_j]^T is then one
// segmented GEMM (the "contracted unfolding" of project_core and of ALS).
// the projected factors P_l (r_l x d_l, leading dimension r_l) as plain pointers, so a
// slab of P_0's rows (the per-rank core slabs) can stand in for the whole
struct PRef {
  const double* p;
};
struct PRefs {
  PRef v[3];
  PRefs(const DBuf P[3]) : v{{P[0].p}, {P[1].p}, {P[2].p}} {}
  PRefs(const double* a, const double* b, const double* c) : v{{a}, {b}, {c}} {}
  operator const PRef*() const { return v; }
};

struct GroupedTerms {
  int o1, o2;
  DVec<int64_t> seg;
  DBuf G1, G2;
  GroupedTerms(latsum_ctx* c, const latsum_canonical& can, const PRef P[3], const int64_t r[3],
               int m)
      : o1(m == 0 ? 1 : 0), o2(m == 2 ? 1 : 2) {
    const int64_t T = can.T;
    DVec<int32_t> c1, c2;
    DVec<double> tw;
    c1.upload(c, can.stc[m][o1]);
    c2.upload(c, can.stc[m][o2]);
    tw.upload(c, can.stw[m]);
    seg.upload(c, can.sseg[m]);
    G1.alloc(c, size_t(r[o1]) * T);
    G2.alloc(c, size_t(r[o2]) * T);
    k_gather_scale<<<grid_for(r[o1] * T), 256, 0, c->stream>>>(P[o1].p, r[o1], r[o1], c1.p, tw.p,
                                                               T, G1.p);
    post_launch(c);
    k_gather_scale<<<grid_for(r[o2] * T), 256, 0, c->stream>>>(P[o2].p, r[o2], r[o2], c2.p,
                                                               nullptr, T, G2.p);
    post_launch(c);
  }
  // X (r_o1 nb x na): columns j = a0 .. a0+na-1 of the grouped unfolding, rows (i1, i2) with
  // i2 in [b0, b0 + nb) of the o2 index (nb < 0: all of it)
  void form(latsum_ctx* c, const int64_t r[3], int64_t T, int64_t a0, int64_t na, double* X,
            int64_t b0 = 0, int64_t nb = -1) const {
    if (nb < 0) nb = r[o2];
    GemmOpts o = tagged("gemm_core_x");
    o.batch = na;
    o.sC = r[o1] * nb;
    o.kseg = seg.p + a0;
    gemm(c, false, true, r[o1], nb, T, 1.0, G1.p, r[o1], G2.p + b0, r[o2], 0.0, X, r[o1], o);
  }
};

// The mode whose dictionary is smallest is contracted last: cost 2 r1 r2 r3 d_m.
int core_mode(const latsum_canonical& can) {
  int m = 0;
  for (int l = 1; l < 3; ++l)
    if (can.d[l] < can.d[m]) m = l;
  return m;
}

// core(a,b,c) = sum_t w_t P0(a,c0_t) P1(b,c1_t) P2(c,c2_t)  (project_core,
// rank_reduction.hpp:88-100).  With m the contracted mode and (o1, o2) the others:
// X_j = G1[:, seg_j] G2[:, seg_j]^T over the terms whose mode-m column is j (one
// segmented GEMM, G1 = P_o1 gathered and weighted, G2 = P_o2 gathered), then
// core = X x_m P_m.  Cost 2 r1 r2 r3 d_m + 2 r_o1 r_o2 T instead of the reference
// loop's 2 r1 r2 r3 M_c.  [a_lo, a_hi) restricts j (the rank's share when sharded).
// on_rows(first, count): core elements [first, first + count) of the o2-chunk just formed, in
// the unit the chunk covers (see form_core's long-K loop); called on c->stream order
using CoreChunkFn = std::function<void(int64_t b0, int64_t nbb)>;
void form_core(latsum_ctx* c, const latsum_canonical& can, const PRef P[3], const int64_t r[3],
               double* core, int m, int64_t a_lo = 0, int64_t a_hi = -1,
               const CoreChunkFn* on_chunk = nullptr) {
  terms(c, can);
  const int64_t T = can.T, dm = a_hi < 0 ? can.d[m] : a_hi;
  const int o1 = m == 0 ? 1 : 0, o2 = m == 2 ? 1 : 2;
  const int64_t ro = r[o1] * r[o2];
  const int64_t rall = r[0] * r[1] * r[2];
  if (a_lo >= dm) {  // empty share of a sharded core
    CK(cudaMemsetAsync(core, 0, sizeof(double) * rall, c->stream));
    return;
  }
  GroupedTerms gt(c, can, P, r, m);
  const int64_t budget = workspace_budget();  // doubles of X per chunk
  const int64_t nall = dm - a_lo;
  // Long-K form (default on the Ozaki path): chunk the o2 index of X's rows instead of the
  // contraction index, so every core element comes out of ONE product over all nall columns
  // (written once, no beta = 1 re-reads of the core; long K amortises the int8 kernel's
  // per-tile TMEM drains).  X block: r_o1 nb rows x nall columns.
  if (!std::getenv("LATSUM_CORE_KCHUNK") && nall <= 65535 &&
      core_uses_ozaki(ro, std::max(r[0], r[2]), nall) && r[o1] * nall <= budget) {
    const int64_t nb = balanced_chunk(r[o2], budget / std::max<int64_t>(r[o1] * nall, 1), 1);
    DBuf X(c, size_t(r[o1]) * nb * nall);
    for (int64_t b0 = 0; b0 < r[o2]; b0 += nb) {
      const int64_t nbb = std::min(nb, r[o2] - b0);
      const int64_t rows = r[o1] * nbb;  // X rows of this block
      gt.form(c, r, T, a_lo, nall, X.p, b0, nbb);
      if (m == 0) {         // core (r0 x r1 r2) columns [r1 b0, r1 (b0 + nbb)) = P0 X^T
        ozaki_gemm(c, r[0], rows, nall, P[0].p + a_lo * r[0], r[0], X.p, rows,
                   core + r[0] * r[1] * b0, r[0], "gemm_core(ozaki-i8)", true, 0.0);
      } else if (m == 2) {  // core rows [r0 b0, r0 (b0 + nbb)) of the (r0 r1 x r2) view
        ozaki_gemm(c, rows, r[2], nall, X.p, rows, P[2].p + a_lo * r[2], r[2],
                   core + r[0] * b0, ro, "gemm_core(ozaki-i8)", true, 0.0);
      } else {              // rows (a, k), k in the block -> core[a + r0 b + r0 r1 k]
        oz::OzOut o = oz_out(core + r[0] * r[1] * b0, r[0], 0.0);
        o.mr = r[0];
        o.rs = r[0] * r[1];
        ozaki_gemm_ex(c, rows, r[1], nall, X.p, 1, rows, 0, 0, P[1].p + a_lo * r[1], 1, r[1], o,
                      "gemm_core(ozaki-i8)");
      }
      if (on_chunk) (*on_chunk)(b0, nbb);
    }
    return;
  }
  const int64_t ac = balanced_chunk(dm - a_lo, std::min<int64_t>(budget / std::max<int64_t>(ro, 1), 65535), 64);
  DBuf X(c, size_t(ro) * ac);
  for (int64_t a0 = a_lo; a0 < dm; a0 += ac) {
    const int64_t na = std::min(ac, dm - a0);
    gt.form(c, r, T, a0, na, X.p);
    const double beta = a0 == a_lo ? 0.0 : 1.0;
    const bool oz = core_uses_ozaki(ro, std::max(r[0], r[2]), na);
    if (m == 0 && oz) {
      ozaki_gemm(c, r[0], ro, na, P[0].p + a0 * r[0], r[0], X.p, ro, core, r[0],
                 "gemm_core(ozaki-i8)", true, beta);
    } else if (m == 2 && oz) {
      ozaki_gemm(c, ro, r[2], na, X.p, ro, P[2].p + a0 * r[2], r[2], core, ro,
                 "gemm_core(ozaki-i8)", true, beta);
    } else if (m == 1 && oz) {  // rows (a, k) of X -> core[a + r0 b + r0 r1 k]
      oz::OzOut o = oz_out(core, r[0], beta);
      o.mr = r[0];
      o.rs = r[0] * r[1];
      ozaki_gemm_ex(c, ro, r[1], na, X.p, 1, ro, 0, 0, P[1].p + a0 * r[1], 1, r[1], o,
                    "gemm_core(ozaki-i8)");
    } else if (m == 0) {        // core (r0 x r1 r2) = P0[:, j] X^T
      gemm(c, false, true, r[0], ro, na, 1.0, P[0].p + a0 * r[0], r[0], X.p, ro, beta, core, r[0],
           tagged("gemm_core"));
    } else if (m == 2) { // core (r0 r1 x r2) = X P2[:, j]^T
      gemm(c, false, true, ro, r[2], na, 1.0, X.p, ro, P[2].p + a0 * r[2], r[2], beta, core, ro,
           tagged("gemm_core"));
    } else {             // core[:, :, k] (r0 x r1) = X[:, k, j] P1[:, j]^T, batched over k
      GemmOpts ob = tagged("gemm_core");
      ob.batch = r[2];
      ob.sA = r[0];
      ob.sC = r[0] * r[1];
      gemm(c, false, true, r[0], r[1], na, 1.0, X.p, ro, P[1].p + a0 * r[1], r[1], beta, core, r[0],
           ob);
    }
  }
}

latsum_ctx* sub_ctx(latsum_ctx* c, int i) {
  if (!c->sub[i]) {
    auto* w = new latsum_ctx();
    w->device = c->device;
    w->parent = c;
    // workers 0-2 carry the RHOSVD modes' latency-bound eigensolver chains: highest
    // priority; worker 3 (norm_f, one throughput kernel off the critical path): lowest
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&w->own, cudaStreamNonBlocking, i < 3 ? hi : lo));
    w->stream = w->own;
    CS(cusolverDnCreate(&w->solver));
    CS(cusolverDnSetStream(w->solver, w->stream));
    CS(cusolverDnCreateParams(&w->solver_params));
    if (i == 3) {
      const char* e = std::getenv("LATSUM_NORM_CTAS");
      w->max_ctas = e ? std::atoi(e) : 32;
    }
    c->sub[i] = w;
  }
  c->sub[i]->prof = c->prof;
  c->sub[i]->eig_method = c->eig_method;
  c->sub[i]->rank = c->rank;
  c->sub[i]->nranks = c->nranks;
  c->sub[i]->host_ar = c->host_ar;
  c->sub[i]->host_ag = c->host_ag;
  c->sub[i]->host_user = c->host_user;
  c->sub[i]->channel = 1 + i;
  return c->sub[i];
}

void merge_sub(latsum_ctx* c, latsum_ctx* w) {
  prof_harvest(w);
  for (const auto& kv : w->stats) {
    auto& st = c->stats[kv.first];
    st.count += kv.second.count;
    st.ms += kv.second.ms;
    st.work += kv.second.work;
  }
  w->stats.clear();
  c->launches += w->launches;
  w->launches = 0;
}

// Runs f(worker) for workers 0..n-1 concurrently (one host thread and stream each),
// ordered after the work already queued on c->stream and before anything queued next.
template <typename F>
void fork_join(latsum_ctx* c, int n, F&& f) {
  cudaEvent_t fork;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CK(cudaEventRecord(fork, c->stream));
  std::vector<latsum_ctx*> ws(n);
  for (int i = 0; i < n; ++i) {
    ws[i] = sub_ctx(c, i);
    CK(cudaStreamWaitEvent(ws[i]->stream, fork, 0));
  }
  std::vector<std::exception_ptr> errs(n);
  std::vector<std::thread> th;
  for (int i = 0; i < n; ++i)
    th.emplace_back([&, i] {
      try {
        CK(cudaSetDevice(c->device));
        f(ws[i], i);
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (int i = 0; i < n; ++i) {
    cudaEvent_t join;
    CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    CK(cudaEventRecord(join, ws[i]->stream));
    CK(cudaStreamWaitEvent(c->stream, join, 0));
    CK(cudaEventDestroy(join));
    merge_sub(c, ws[i]);
  }
  CK(cudaEventDestroy(fork));
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

void rhosvd_impl(latsum_ctx* c, const latsum_canonical& can, const int64_t* ranks, double tol,
                 int deflate, latsum_tucker& t, latsum_spectral_report& rep, bool form = true,
                 bool slabs = false) {
  if (!ranks) require(tol > 0.0 && tol < 1.0, "TruncationSpec: tolerance must lie in (0,1)");
  std::memset(&rep, 0, sizeof(rep));
  Timings tm;
  Timer total(c);
  total.start();
  for (int l = 0; l < 3; ++l) t.N[l] = can.N[l];
  double wn2 = 0;
  for (double w : can.weights) wn2 += w * w;
  rep.weight_norm = std::sqrt(wn2);
  // the three mode reductions and norm_f are independent: one worker stream each
  ModeOut mo[3];
  Timings tms[4];
  const bool zero_terms = can.Mc == 0;  // T == 0 iff M_c == 0 (every term is kept, merged)
  // norm_f waits for the three Grams: its throughput kernels then overlap the latency-bound
  // eigensolves instead of competing with the Grams for the SMs
  std::mutex gmu;
  std::condition_variable gcv;
  bool gram_done[3] = {false, false, false};
  auto mark_gram = [&](int i) {
    std::lock_guard<std::mutex> g(gmu);
    gram_done[i] = true;
    gcv.notify_all();
  };
  for (int i = 0; i < 3; ++i) tms[i].on_gram = [&, i] { mark_gram(i); };
  EigTurnstile turn;
  if (!has_comm(c) && eig_env_mode() == 0 && c->eig_method == 0 && !ranks) {
    std::vector<std::pair<int64_t, int>> sz;
    for (int l = 0; l < 3; ++l) {
      const int64_t gn = std::min<int64_t>(can.N[l], can.d[l]);
      // compressed modes (range basis first) are served in arrival order
      if (!band_eig_ok(gn) && !compress_pass1(can.N[l], can.d[l], false)) sz.emplace_back(-gn, l);
    }
    std::sort(sz.begin(), sz.end());
    for (const auto& x : sz) turn.order.push_back(x.second);
    for (int i = 0; i < 3; ++i) {
      tms[i].before_eig1 = [&, i] { turn.wait(i); };
      tms[i].after_eig1 = [&, i] { turn.finish(i); };
    }
  }
  auto body = [&](latsum_ctx* w, int i) {
    if (i == 3 || zero_terms) {
      if (!zero_terms) {
        std::unique_lock<std::mutex> g(gmu);
        gcv.wait(g, [&] { return gram_done[0] && gram_done[1] && gram_done[2]; });
      }
      Timer tn(w);
      tn.start();
      struct Reserve {  // the SMs this worker's capped persistent grids hold while it runs
        std::atomic<int>& r;
        Reserve(std::atomic<int>& x, int n) : r(x) { r.store(n); }
        ~Reserve() { r.store(0); }
      } hold(c->reserved_ctas, zero_terms ? 0 : w->max_ctas);
      rep.input_norm = canonical_norm(w, can);
      tms[3].norm = tn.stop();
    } else {
      try {
        reduce_mode(w, can, i, ranks, tol, deflate, mo[i], tms[i]);
      } catch (...) {
        mark_gram(i);  // never leave the norm worker or a later mode waiting
        turn.finish(i);
        throw;
      }
      mark_gram(i);
      turn.finish(i);
      // P_i = Z_i^T D_i over this rank's rows (summed over ranks) while the other modes'
      // eigensolves are still running
      Timer tp(w);
      tp.start();
      const RowBlock blk = mo[i].blk;
      const int64_t N = can.N[i], Nb = blk.n();
      t.P[i].alloc(w, size_t(mo[i].r) * can.d[i]);
      if (Nb > 0)
        gemm(w, true, false, mo[i].r, can.d[i], Nb, 1.0, mo[i].Z.p, Nb, can.dict[i].p + blk.lo, N,
             0.0, t.P[i].p, mo[i].r, tagged("gemm_project"));
      else
        CK(cudaMemsetAsync(t.P[i].p, 0, sizeof(double) * mo[i].r * can.d[i], w->stream));
      if (Nb != N) allreduce(w, t.P[i].p, size_t(mo[i].r) * can.d[i]);
      tms[i].project = tp.stop();
    }
  };
  // norm_f only feeds the report: it runs on its own worker thread and stream and is joined
  // after the core, so neither the modes' join nor the core waits for it
  std::future<void> norm_done;
  latsum_ctx* wn = nullptr;
  if (!zero_terms) {
    wn = sub_ctx(c, 3);
    cudaEvent_t fork;
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    CK(cudaEventRecord(fork, c->stream));
    CK(cudaStreamWaitEvent(wn->stream, fork, 0));
    CK(cudaEventDestroy(fork));
    norm_done = std::async(std::launch::async, [&, wn] {
      CK(cudaSetDevice(c->device));
      body(wn, 3);
    });
  }
  Trace::mark(c, "rhosvd fork");
  try {
    fork_join(c, zero_terms ? 1 : 3, body);
  } catch (...) {
    if (norm_done.valid()) norm_done.wait();
    throw;
  }
  Trace::mark(c, "rhosvd join");
  auto join_norm = [&] {
    if (!norm_done.valid()) return;
    norm_done.get();  // rethrows a norm_f failure
    merge_sub(c, wn);
    tm.norm += tms[3].norm;
  };
  for (int l = 0; l < 3; ++l) {
    mo[l].Z.adopt(c->stream);
    t.P[l].adopt(c->stream);
  }
  for (int i = 0; i < 3; ++i) {
    const auto& x = tms[i];
    tm.gram += x.gram;
    tm.syevd += x.syevd;
    tm.deflate += x.deflate;
    tm.project += x.project;
  }
  if (zero_terms) tm.norm += tms[3].norm + tms[0].norm;
  bool zero = can.Mc == 0;  // zero tensor (rank_reduction.hpp:183-187): every merged weight 0
  if (!zero) {
    zero = true;
    for (double w : terms_host(can).tw) zero = zero && w == 0.0;
  }
  if (zero || (zero_terms && rep.input_norm == 0.0)) {
    join_norm();
    for (int l = 0; l < 3; ++l) {
      rep.chosen_ranks[l] = 1;
      rep.n_singular[l] = 1;
      t.r[l] = 1;
      t.sigma[l].assign(1, 0.0);
      t.U[l].alloc(c, size_t(t.N[l]));
      CK(cudaMemsetAsync(t.U[l].p, 0, sizeof(double) * t.N[l], c->stream));
      const double one = 1.0;
      CK(cudaMemcpyAsync(t.U[l].p, &one, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    }
    t.core.alloc(c, 1);
    t.has_core = true;
    CK(cudaMemsetAsync(t.core.p, 0, sizeof(double), c->stream));
    CK(cudaStreamSynchronize(c->stream));
    rep.ms_total = total.stop();
    return;
  }
  DBuf* P = t.P;
  Timer tp(c);
  tp.start();
  for (int l = 0; l < 3; ++l) {
    t.r[l] = mo[l].r;
    t.d[l] = can.d[l];
    const RowBlock blk = mo[l].blk;
    const int64_t N = can.N[l], Nb = blk.n();
    const bool sharded = Nb != N;
    if (sharded) {
      // replicate Z: all-gather the row blocks (padded to equal size)
      const int64_t r = mo[l].r, bmax = N / c->nranks + 1;
      DBuf send(c, size_t(bmax) * r), recv(c, size_t(bmax) * r * c->nranks), full(c, size_t(N) * r);
      CK(cudaMemsetAsync(send.p, 0, sizeof(double) * bmax * r, c->stream));
      if (Nb > 0)
        CK(cudaMemcpy2DAsync(send.p, bmax * sizeof(double), mo[l].Z.p, Nb * sizeof(double),
                             Nb * sizeof(double), r, cudaMemcpyDeviceToDevice, c->stream));
      allgather(c, send.p, recv.p, size_t(bmax) * r);
      for (int q = 0; q < c->nranks; ++q) {
        const int64_t lo = N * q / c->nranks, nq = N * (q + 1) / c->nranks - lo;
        if (nq > 0)
          CK(cudaMemcpy2DAsync(full.p + lo, N * sizeof(double), recv.p + size_t(q) * bmax * r,
                               bmax * sizeof(double), nq * sizeof(double), r,
                               cudaMemcpyDeviceToDevice, c->stream));
      }
      mo[l].Z = std::move(full);
    }
    t.tc[l].upload(c, terms_host(can).tc[l]);
  }
  t.tw.upload(c, can.tw);
  t.tseg.upload(c, can.tseg);
  t.T = can.T;
  tm.project += tp.stop();
  Trace::mark(c, "projections done");
  if (form) {  // the dense core (rank_reduction.hpp:88-100); absent when it cannot fit
    tp.start();
    const int m = core_mode(can);
    if (slabs && has_comm(c)) {
      // each rank forms and keeps rows [a0, a1) of mode 0 of the core, over all
      // of the contraction (the P_l are replicated), so no core all-reduce and no rank holds
      // the whole core (BASELINE cfg5: 518 GB); entries and boxes sum the ranks' partials
      t.a0 = t.r[0] * c->rank / c->nranks;
      t.ra = t.r[0] * (c->rank + 1) / c->nranks - t.a0;
      t.core_slab = true;
      t.core.alloc(c, size_t(std::max<int64_t>(t.ra, 1)) * t.r[1] * t.r[2]);
      if (t.ra > 0) {
        DBuf P0s(c, size_t(t.ra) * can.d[0]);
        CK(cudaMemcpy2DAsync(P0s.p, t.ra * sizeof(double), P[0].p + t.a0, t.r[0] * sizeof(double),
                             t.ra * sizeof(double), can.d[0], cudaMemcpyDeviceToDevice, c->stream));
        const int64_t rs[3] = {t.ra, t.r[1], t.r[2]};
        form_core(c, can, PRefs(P0s.p, P[1].p, P[2].p), rs, t.core.p, m);
      }
    } else if (has_comm(c)) {  // each rank forms the core from its share of mode m
      t.core.alloc(c, size_t(t.r[0]) * t.r[1] * t.r[2]);
      const int64_t dm = can.d[m];
      form_core(c, can, PRefs(P), t.r, t.core.p, m, dm * c->rank / c->nranks,
                dm * (c->rank + 1) / c->nranks);
      allreduce(c, t.core.p, size_t(t.r[0]) * t.r[1] * t.r[2]);
    } else {
      t.core.alloc(c, size_t(t.r[0]) * t.r[1] * t.r[2]);
      // host sink: the factors now, the core chunk by chunk behind its contraction (the
      // device->host copy of the result overlaps the core GEMMs on a copy stream)
      auto& sk = c->sink;
      const int64_t rall = t.r[0] * t.r[1] * t.r[2];
      bool stream = sk.core && rall <= sk.core_cap;
      for (int l = 0; l < 3; ++l) stream = stream && sk.f[l] && t.N[l] * t.r[l] <= sk.f_cap[l];
      if (stream) {
        if (!sk.copy) CK(cudaStreamCreateWithFlags(&sk.copy, cudaStreamNonBlocking));
        if (!sk.copy2) CK(cudaStreamCreateWithFlags(&sk.copy2, cudaStreamNonBlocking));
        auto after_stream = [&] {
          cudaEvent_t ev;
          CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          CK(cudaEventRecord(ev, c->stream));
          CK(cudaStreamWaitEvent(sk.copy, ev, 0));
          CK(cudaStreamWaitEvent(sk.copy2, ev, 0));
          CK(cudaEventDestroy(ev));
        };
        after_stream();
        for (int l = 0; l < 3; ++l) {
          // the bases are still the modes' Z here (moved into t.U after the core)
          CK(cudaMemcpyAsync(sk.f[l], mo[l].Z.p, sizeof(double) * t.N[l] * t.r[l],
                             cudaMemcpyDeviceToHost, sk.copy));
        }
        const int o1 = m == 0 ? 1 : 0, o2 = m == 2 ? 1 : 2;
        const int64_t ro = t.r[o1] * t.r[o2];
        CoreChunkFn chunk = [&](int64_t b0, int64_t nbb) {
          after_stream();
          // each chunk split over the two copy streams (the first half of the columns / elements
          // on one, the rest on the other)
          if (m == 2) {  // rows [r0 b0, r0 (b0 + nbb)) of the (r0 r1) x r2 view
            const int64_t h = t.r[2] / 2;
            for (int q = 0; q < 2; ++q) {
              const int64_t c0 = q ? h : 0, nc = q ? t.r[2] - h : h;
              if (nc > 0)
                CK(cudaMemcpy2DAsync(sk.core + t.r[0] * b0 + c0 * ro, ro * sizeof(double),
                                     t.core.p + t.r[0] * b0 + c0 * ro, ro * sizeof(double),
                                     t.r[0] * nbb * sizeof(double), nc, cudaMemcpyDeviceToHost,
                                     q ? sk.copy2 : sk.copy));
            }
          } else {       // m = 0 / 1: a contiguous slab of r0 r1 nbb elements
            const int64_t n = t.r[0] * t.r[1] * nbb, h = n / 2, o = t.r[0] * t.r[1] * b0;
            CK(cudaMemcpyAsync(sk.core + o, t.core.p + o, sizeof(double) * h, cudaMemcpyDeviceToHost,
                               sk.copy));
            CK(cudaMemcpyAsync(sk.core + o + h, t.core.p + o + h, sizeof(double) * (n - h),
                               cudaMemcpyDeviceToHost, sk.copy2));
          }
        };
        bool chunked = false;
        CoreChunkFn mark = [&](int64_t b0, int64_t nbb) {
          chunked = true;
          chunk(b0, nbb);
        };
        form_core(c, can, PRefs(P), t.r, t.core.p, m, 0, -1, &mark);
        if (!chunked) {  // the K-chunked form: the core is complete only at the end
          after_stream();
          CK(cudaMemcpyAsync(sk.core, t.core.p, sizeof(double) * rall, cudaMemcpyDeviceToHost,
                             sk.copy));
        }
        CK(cudaStreamSynchronize(sk.copy));
        CK(cudaStreamSynchronize(sk.copy2));
        t.sink_written = true;
      } else {
        form_core(c, can, PRefs(P), t.r, t.core.p, m);
      }
    }
    t.has_core = true;
    tm.core = tp.stop();
    Trace::mark(c, "core done");
  }
  join_norm();
  double tails = 0.0;
  for (int l = 0; l < 3; ++l) {
    t.U[l] = std::move(mo[l].Z);
    t.sigma[l] = mo[l].sigma;
    rep.chosen_ranks[l] = mo[l].r;
    rep.n_singular[l] = int64_t(mo[l].sigma.size());
    rep.tie_at_cutoff[l] = mo[l].tie ? 1 : 0;
    rep.cutoff_margin[l] = mo[l].margin;
    rep.deflated[l] = mo[l].deflated;
    rep.gram_rows[l] = mo[l].rows;
    rep.gram_size[l] = mo[l].gsize;
    rep.deflate_k1[l] = mo[l].k1;
    double s = 0;  // SpectralReport::tail (rank_reduction.hpp:61-66)
    for (int64_t k = int64_t(mo[l].sigma.size()) - 1; k >= mo[l].r; --k)
      s += mo[l].sigma[k] * mo[l].sigma[k];
    tails += std::sqrt(s);
  }
  rep.bound_abs = rep.weight_norm * tails;
  const double n2 = rep.input_norm * rep.input_norm;
  rep.stability_constant = rep.weight_norm * rep.weight_norm / n2;
  rep.stability_ok = rep.stability_constant <= 1.0 + 1e-10;
  rep.bound_rel = std::sqrt(rep.stability_constant) * rep.input_norm * tails;
  rep.ms_gram = tm.gram;
  rep.ms_syevd = tm.syevd;
  rep.ms_deflate = tm.deflate;
  rep.ms_project = tm.project;
  rep.ms_core = tm.core;
  rep.ms_norm = tm.norm;
  rep.ms_total = total.stop();
}

// ------------------------------------------------------------------ canonical_to_tucker
double device_scalar(latsum_ctx* c, const double* d) {
  double h = 0;
  CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return h;
}

// P_l = Y_l^T D_l (r_l x d_l) for every mode
void project_factors(latsum_ctx* c, const latsum_canonical& can, const DBuf Y[3], const int64_t r[3],
                     DBuf P[3]) {
  for (int l = 0; l < 3; ++l) {
    P[l].alloc(c, size_t(r[l]) * can.d[l]);
    gemm(c, true, false, r[l], can.d[l], can.N[l], 1.0, Y[l].p, can.N[l], can.dict[l].p, can.N[l],
         0.0, P[l].p, r[l], tagged("gemm_project"));
  }
}

// One ALS step for mode l (rank_reduction.hpp:243-256): the top-r_l left singular vectors
// of the contracted unfolding unf = A_l kr^T.  With the dictionary, unf = D_l X^T where X
// (r_o1 r_o2 x d_l) is the grouped unfolding over c_l.  unf is materialised and reduced
// with the same two-pass deflated Gram as RHOSVD (fixed rank, second pass forced): the
// trailing kept directions carry relative mass ~eps^2, which a single Gram cannot resolve.
void als_mode_update(latsum_ctx* c, const latsum_canonical& can, const DBuf P[3],
                     const int64_t r[3], int l, DBuf& Y) {
  terms(c, can);
  const int64_t N = can.N[l], d = can.d[l];
  GroupedTerms gt(c, can, PRefs(P), r, l);
  const int64_t R2 = r[gt.o1] * r[gt.o2];
  require(double(R2) * double(d + N) <= double(workspace_budget()),
          "als_refine: contracted unfolding too large for the device (ALS is out of scope at "
          "this size)");
  DBuf X(c, size_t(R2) * d);
  for (int64_t a0 = 0; a0 < d; a0 += 65535)
    gt.form(c, r, can.T, a0, std::min<int64_t>(65535, d - a0), X.p + a0 * R2);
  DBuf unf(c, size_t(N) * R2);
  gemm(c, false, true, N, R2, d, 1.0, can.dict[l].p, N, X.p, R2, 0.0, unf.p, N, tagged("gemm_als"));
  X.release();
  const int64_t n_sing = std::min<int64_t>(N, R2);
  const int64_t keep = std::min<int64_t>(r[l], n_sing);
  ModeOut mo;
  Timings tm;
  reduce_dense(c, unf, RowBlock{0, N}, N, R2, n_sing, &keep, 0.0, LATSUM_DEFLATE_ALWAYS,
               /*force_deflate=*/true, /*sharded=*/false, mo, tm);
  require(mo.r == r[l], "als_refine: unfolding rank below the requested Tucker rank");
  Y = std::move(mo.Z);
}

double projected_norm(latsum_ctx* c, const latsum_canonical& can, const DBuf P[3],
                      const int64_t r[3]) {
  const double* E[3] = {P[0].p, P[1].p, P[2].p};
  return hadamard_norm(c, can, E, r);
}

// shrink_core (rank_reduction.hpp:129-168): HOSVD rotation of the core per mode, then
// greedy removal of trailing slices while the discarded mass fits in budget2.
void shrink_core(latsum_ctx* c, latsum_tucker& t, double budget2) {
  int64_t r[3] = {t.r[0], t.r[1], t.r[2]};
  const int64_t tot = r[0] * r[1] * r[2];
  for (int l = 0; l < 3; ++l) {
    const int64_t rl = r[l];
    DBuf G(c, size_t(rl) * rl), W(c, rl), q(c, size_t(rl) * rl), nc(c, size_t(tot));
    DBuf swp;
    if (l == 0) {
      gemm(c, false, true, r[0], r[0], r[1] * r[2], 1.0, t.core.p, r[0], t.core.p, r[0], 0.0, G.p,
           r[0], tagged("gemm_shrink"));
    } else if (l == 2) {
      gemm(c, true, false, r[2], r[2], r[0] * r[1], 1.0, t.core.p, r[0] * r[1], t.core.p,
           r[0] * r[1], 0.0, G.p, r[2], tagged("gemm_shrink"));
    } else {
      swp.alloc(c, size_t(tot));
      k_swap01<<<grid_for(tot), 256, 0, c->stream>>>(t.core.p, r[0], r[1], r[2], swp.p);
      post_launch(c);
      gemm(c, false, true, r[1], r[1], r[0] * r[2], 1.0, swp.p, r[1], swp.p, r[1], 0.0, G.p, r[1],
           tagged("gemm_shrink"));
    }
    syevd(c, rl, G.p, W.p);
    k_reverse_columns<<<grid_for(rl * rl), 256, 0, c->stream>>>(G.p, rl, rl, rl, q.p);  // descending
    post_launch(c);
    // core <- core x_l q^T
    if (l == 0) {
      gemm(c, true, false, r[0], r[1] * r[2], r[0], 1.0, q.p, r[0], t.core.p, r[0], 0.0, nc.p, r[0],
           tagged("gemm_shrink"));
    } else if (l == 2) {
      gemm(c, false, false, r[0] * r[1], r[2], r[2], 1.0, t.core.p, r[0] * r[1], q.p, r[2], 0.0,
           nc.p, r[0] * r[1], tagged("gemm_shrink"));
    } else {
      DBuf tmp(c, size_t(tot));
      gemm(c, true, false, r[1], r[0] * r[2], r[1], 1.0, q.p, r[1], swp.p, r[1], 0.0, tmp.p, r[1],
           tagged("gemm_shrink"));
      k_swap01<<<grid_for(tot), 256, 0, c->stream>>>(tmp.p, r[1], r[0], r[2], nc.p);
      post_launch(c);
    }
    t.core = std::move(nc);
    DBuf U(c, size_t(t.N[l]) * rl);
    gemm(c, false, false, t.N[l], rl, rl, 1.0, t.U[l].p, t.N[l], q.p, rl, 0.0, U.p, t.N[l],
         tagged("gemm_shrink"));
    t.U[l] = std::move(U);
  }
  int64_t b[3] = {r[0], r[1], r[2]};
  DBuf m(c, 1);
  bool changed = true;
  while (changed && budget2 > 0.0) {
    changed = false;
    for (int l = 0; l < 3; ++l) {
      if (b[l] <= 1) continue;
      k_slice_mass<<<1, 512, 0, c->stream>>>(t.core.p, r[0], r[1], l, b[l] - 1, b[0], b[1], b[2], m.p);
      post_launch(c);
      const double mass = device_scalar(c, m.p);
      if (mass <= budget2) {
        budget2 -= mass;
        --b[l];
        changed = true;
      }
    }
  }
  if (b[0] != r[0] || b[1] != r[1] || b[2] != r[2]) {
    DBuf nc(c, size_t(b[0]) * b[1] * b[2]);
    k_crop<<<grid_for(b[0] * b[1] * b[2]), 256, 0, c->stream>>>(t.core.p, r[0], r[1], b[0], b[1],
                                                                b[2], nc.p);
    post_launch(c);
    t.core = std::move(nc);
    for (int l = 0; l < 3; ++l) {
      DBuf U(c, size_t(t.N[l]) * b[l]);
      CK(cudaMemcpyAsync(U.p, t.U[l].p, sizeof(double) * t.N[l] * b[l], cudaMemcpyDeviceToDevice,
                         c->stream));
      t.U[l] = std::move(U);
      t.r[l] = b[l];
    }
  }
}

// canonical_to_tucker (rank_reduction.hpp:280-306): RHOSVD initial guess, ALS refinement
// (up to max_sweeps, stop when the projected norm stagnates), orthogonal core
// projection, and shrink_core in tolerance mode.
void canonical_to_tucker_impl(latsum_ctx* c, const latsum_canonical& can, const int64_t* ranks,
                              double tol, int max_sweeps, double stag_tol, latsum_tucker& t,
                              latsum_spectral_report& rep, int* sweeps_done) {
  terms(c, can);
  rhosvd_impl(c, can, ranks, tol, LATSUM_DEFLATE_AUTO, t, rep, /*form=*/false);
  if (sweeps_done) *sweeps_done = 0;
  if (rep.input_norm == 0.0) {
    if (!t.has_core) {
      t.core.alloc(c, size_t(t.r[0]) * t.r[1] * t.r[2]);
      CK(cudaMemsetAsync(t.core.p, 0, sizeof(double) * t.r[0] * t.r[1] * t.r[2], c->stream));
      t.has_core = true;
    }
    return;
  }
  const int64_t* r = t.r;
  DBuf P[3];
  project_factors(c, can, t.U, r, P);
  if (max_sweeps > 0) {
    double fit = projected_norm(c, can, P, r);
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
      for (int l = 0; l < 3; ++l) {
        DBuf Y;
        als_mode_update(c, can, P, r, l, Y);
        t.U[l] = std::move(Y);
        P[l].alloc(c, size_t(r[l]) * can.d[l]);
        gemm(c, true, false, r[l], can.d[l], can.N[l], 1.0, t.U[l].p, can.N[l], can.dict[l].p,
             can.N[l], 0.0, P[l].p, r[l], tagged("gemm_project"));
      }
      const double next = projected_norm(c, can, P, r);
      if (sweeps_done) *sweeps_done = sweep + 1;
      if (next - fit <= stag_tol * std::max(next, 1.0)) break;
      fit = next;
    }
  }
  t.core.alloc(c, size_t(r[0]) * r[1] * r[2]);
  form_core(c, can, PRefs(P), r, t.core.p, core_mode(can));
  t.has_core = true;
  for (int l = 0; l < 3; ++l) t.P[l] = std::move(P[l]);
  if (tol > 0.0 && !ranks) {
    const double n2 = rep.input_norm * rep.input_norm;
    DBuf m(c, 1);
    k_sumsq<<<1, 1024, 0, c->stream>>>(t.core.p, r[0] * r[1] * r[2], m.p);
    post_launch(c);
    const double fit2 = device_scalar(c, m.p);
    const double err2 = std::max(n2 - fit2, 0.0);
    const double budget2 = tol * tol * n2 - err2;
    if (budget2 > 0.0) {
      shrink_core(c, t, budget2);
      t.T = 0;  // the projected factors no longer match the rotated/cropped basis
    }
  }
  for (int l = 0; l < 3; ++l) rep.chosen_ranks[l] = t.r[l];
}

// ------------------------------------------------------------------ tensor IO
// "LTSTNSR" v1 (tensor_io.hpp:12-24, tensor_io.cpp:45-129): 7-byte magic, version 1, tag
// 'C'/'T', 3 zero bytes, u32 dims[3]; canonical: u32 R, R weights, three N_l x R side
// matrices; tucker: u32 ranks[3], core, three factors; f64 little-endian, column-major;
// trailer = FNV-1a-64 of every preceding byte.
struct Fnv {
  uint64_t h = 0xcbf29ce484222325ull;
  void add(const void* data, size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
      h ^= p[i];
      h *= 0x100000001b3ull;
    }
  }
};

struct FileSink {
  std::ofstream os;
  Fnv fnv;
  explicit FileSink(const std::string& path) : os(path, std::ios::binary | std::ios::trunc) {
    if (!os) throw Error(LATSUM_ERR_IO, "cannot open " + path + " for writing");
  }
  void put(const void* d, size_t n) {
    fnv.add(d, n);
    os.write(static_cast<const char*>(d), std::streamsize(n));
    if (!os) throw Error(LATSUM_ERR_IO, "short write");
  }
  void u32(uint32_t v) { put(&v, 4); }
  // device buffer -> file in 64 MB chunks
  void device(latsum_ctx* c, const double* dptr, size_t count) {
    std::vector<double> h(std::min<size_t>(count, size_t(8) << 20));
    for (size_t o = 0; o < count; o += h.size()) {
      const size_t n = std::min(h.size(), count - o);
      CK(cudaMemcpyAsync(h.data(), dptr + o, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      put(h.data(), n * sizeof(double));
    }
  }
  void finish() {
    const uint64_t sum = fnv.h;
    os.write(reinterpret_cast<const char*>(&sum), 8);
    if (!os) throw Error(LATSUM_ERR_IO, "short write");
  }
};

void write_header(FileSink& f, char tag, const int64_t dims[3]) {
  const char magic[7] = {'L', 'T', 'S', 'T', 'N', 'S', 'R'};
  f.put(magic, 7);
  const char head[4] = {char(1), tag, 0, 0};
  f.put(head, 4);
  const char pad = 0;
  f.put(&pad, 1);
  for (int l = 0; l < 3; ++l) f.u32(uint32_t(dims[l]));
}

// ------------------------------------------------------------------ stage 4
void check_box(const int64_t N[3], const int64_t lo[3], const int64_t hi[3]) {
  for (int l = 0; l < 3; ++l)
    if (lo[l] < 0 || hi[l] > N[l] || hi[l] <= lo[l])
      throw Error(LATSUM_ERR_INVALID_ARGUMENT,
                  "evaluation box outside the grid in mode " + std::to_string(l + 1));
}

// to_dense on a box (tucker.hpp:172-178) as slab GEMMs: Q = core x_2 U1, then per
// z-chunk X = Q x_3 U2 and V_k = U0 X_k (the dominant ni x nj x r0 GEMM per slab).
void projected_eval(latsum_ctx* c, const latsum_tucker& t, const int64_t lo[3], const int64_t hi[3],
                    double* out);
void projected_probes(latsum_ctx* c, const latsum_tucker& t, const int64_t* probes, int64_t np,
                      double* out_host);

// The three-GEMM chain on the int8 tensor cores for any contraction order.  Roles: F is
// contracted first, S second, L last (the rows of the final slab GEMM):
//   Q[(a_L, j_F), a_S] = sum_{a_F} core[..] U_F[j_F, a_F]        2 r0 r1 r2 n_F flops
//   X[(a_L, j_F), k_S] = sum_{a_S} Q[(a_L, j_F), a_S] U_S[k_S, a_S]   2 r_L r_S n_F n_S
//   V[i_L, (j_F, k_S)] = sum_{a_L} U_L[i_L, a_L] X[a_L, (j_F, k_S)]   2 r_L n_L n_F n_S
// so the mode of smallest rank goes last (cfg4, ranks 2095 / 1207 / 1266: 4.7e13 flops with
// L = 1 against 7.1e13 with the fixed order L = 0).  No data is permuted: the core is sliced
// through its strides, and the final GEMM writes the box through the output addressing (with
// L != 0 and F = 0 it is computed transposed, so its tile rows still run along the box's
// contiguous index and the stores stay coalesced).
void tucker_eval_chain(latsum_ctx* c, const latsum_tucker& t, const int64_t lo[3], const int64_t n[3],
                       int L, int F, int S, double* out) {
  const int64_t r[3] = {t.r[0], t.r[1], t.r[2]};
  const int64_t cs[3] = {1, r[0], r[0] * r[1]};       // core strides
  const int64_t os[3] = {1, n[0], n[0] * n[1]};       // box strides
  const int64_t rL = r[L], rF = r[F], rS = r[S];
  const double* UL = t.U[L].p + lo[L];
  const double* UF = t.U[F].p + lo[F];
  const double* US = t.U[S].p + lo[S];
  const int64_t budget = int64_t(1) << 29;  // doubles per intermediate (4 GiB; Q may take 8)
  // F-chunks in whole 128-column tiles of the Q GEMM
  // chunks in whole 128-column tiles of the GEMM that has them as columns (Q: j_F, X: k_S),
  // aligned DOWN so they stay inside the budget
  auto tiled_chunk = [](int64_t n, int64_t cap) {
    cap = std::max<int64_t>(1, cap);
    if (n <= cap) return n;
    const int64_t capa = cap >= 128 ? cap / 128 * 128 : cap;
    const int64_t parts = (n + capa - 1) / capa;
    const int64_t c = (n + parts - 1) / parts;
    return capa >= 128 ? std::min(capa, (c + 127) / 128 * 128) : c;
  };
  const int64_t nfc = tiled_chunk(n[F], 2 * budget / std::max<int64_t>(rL * rS, 1));
  const int64_t nsc = tiled_chunk(n[S], std::min<int64_t>(budget / std::max<int64_t>(rL * nfc, 1), 65535));
  DBuf Q(c, size_t(rL) * nfc * rS), X(c, size_t(rL) * nfc * nsc);
  OzSliced sUL, sQ, sCore;  // sliced once and reused across the chunks that share them
  if (L == 0) oz_slice_a(c, UL, 1, t.N[L], n[L], rL, sUL);
  else oz_slice_b(c, UL, 1, t.N[L], n[L], rL, sUL);
  // the core's lines (a_L, a_S) over K = a_F: the A operand of every chunk's Q GEMM
  oz_slice_a(c, t.core.p, cs[L], cs[F], rL * rS, rF, sCore, rL, cs[S]);
  for (int64_t j0 = 0; j0 < n[F]; j0 += nfc) {
    const int64_t njj = std::min(nfc, n[F] - j0);
    {
      OzSliced sUF;
      oz_slice_b(c, UF + j0, 1, t.N[F], njj, rF, sUF);
      oz::OzOut o = oz_out(Q.p, rL);
      o.mr = rL;
      o.rs = rL * njj;
      oz_run(c, sCore, sUF, o, "gemm_eval_q(ozaki-i8)");
    }
    oz_slice_a(c, Q.p, 1, rL * njj, rL * njj, rS, sQ);
    for (int64_t k0 = 0; k0 < n[S]; k0 += nsc) {
      const int64_t nkk = std::min(nsc, n[S] - k0);
      OzSliced sUS, sX;
      oz_slice_b(c, US + k0, 1, t.N[S], nkk, rS, sUS);
      oz_run(c, sQ, sUS, oz_out(X.p, rL * njj), "gemm_eval_x(ozaki-i8)");
      if (L == 0) {  // rows i_L run along the box's contiguous index: V = U_L X
        oz_slice_b(c, X.p, rL, 1, njj * nkk, rL, sX);  // B lines = the columns (j_F, k_S) of X
        oz::OzOut o = oz_out(out + j0 * os[F] + k0 * os[S], os[F]);
        o.nb = njj;
        o.bs = os[S];
        oz_run(c, sUL, sX, o, "gemm_eval_slab(ozaki-i8)");
      } else {  // F == 0: the transposed product V^T = X^T U_L^T puts (j_F, k_S) on the rows, so
        // the tile rows (TMEM lanes, one per thread) again run along the contiguous index
        oz_slice_a(c, X.p, rL, 1, njj * nkk, rL, sX);
        oz::OzOut o = oz_out(out + j0 * os[F] + k0 * os[S], os[L]);
        o.mr = njj;
        o.rs = os[S];
        oz_run(c, sX, sUL, o, "gemm_eval_slab(ozaki-i8)");
      }
    }
  }
}

void tucker_eval(latsum_ctx* c, const latsum_tucker& t, const int64_t lo[3], const int64_t hi[3],
                 double* out) {
  if (!t.has_core) return projected_eval(c, t, lo, hi, out);
  check_box(t.N, lo, hi);
  const int64_t ni = hi[0] - lo[0], nj = hi[1] - lo[1], nk = hi[2] - lo[2];
  if (!t.core_slab && eval_uses_ozaki(std::max({t.r[0], t.r[1], t.r[2]}))) {
    // contraction order by flops: the fixed order (L, F, S) = (0, 1, 2), or the smallest-rank
    // mode last with mode 0 first
    const int64_t n[3] = {ni, nj, nk};
    const int orders[3][3] = {{0, 1, 2}, {1, 0, 2}, {2, 0, 1}};
    static const int forced = [] {
      const char* e = std::getenv("LATSUM_EVAL_ORDER");  // 0 / 1 / 2: the last-contracted mode (tests)
      return e ? std::atoi(e) : -1;
    }();
    int best = 0;
    double best_f = 0.0;
    for (int q = 0; q < 3; ++q) {
      const int L = orders[q][0], F = orders[q][1], S = orders[q][2];
      const double f = double(t.r[0]) * t.r[1] * t.r[2] * n[F] + double(t.r[L]) * t.r[S] * n[F] * n[S] +
                       double(t.r[L]) * n[L] * n[F] * n[S];
      if (q == 0 || f < 0.95 * best_f) {
        best = q;
        best_f = f;
      }
    }
    if (forced >= 0 && forced < 3) best = forced;
    return tucker_eval_chain(c, t, lo, n, orders[best][0], orders[best][1], orders[best][2], out);
  }
  if (t.core_slab && t.ra == 0) {  // this rank's slab is empty: its partial box is zero
    CK(cudaMemsetAsync(out, 0, sizeof(double) * ni * nj * nk, c->stream));
    allreduce(c, out, size_t(ni * nj * nk));
    return;
  }
  const int64_t r0 = t.core_slab ? t.ra : t.r[0], r1 = t.r[1], r2 = t.r[2];
  const double* U0 = t.U[0].p + lo[0] + (t.core_slab ? t.a0 * t.N[0] : 0);
  const double* U1 = t.U[1].p + lo[1];
  const double* U2 = t.U[2].p + lo[2];
  const int64_t budget = int64_t(1) << 29;  // doubles per intermediate (4 GiB)
  // y-chunks in whole 128-column tiles of the Q GEMM (cfg4: the 4 GiB cap gave 202-row chunks,
  // 256 columns of MMA work for 202): Q may take 8 GiB so the aligned chunk fits (cfg4: 384)
  const int64_t njc = balanced_chunk(nj, 2 * budget / std::max<int64_t>(r0 * r2, 1), 128);
  DBuf Q(c, size_t(r0) * njc * r2);
  const int64_t nkc = balanced_chunk(nk, std::min<int64_t>(budget / std::max<int64_t>(r0 * njc, 1), 65535), 1);
  DBuf X(c, size_t(r0) * njc * nkc);
  const bool oz_x = eval_uses_ozaki(r2), oz_v = eval_uses_ozaki(r0);
  OzSliced sU0, sQ, sCore;  // sliced once and reused across the chunks that share them
  if (oz_v) oz_slice_a(c, U0, 1, t.N[0], ni, r0, sU0);
  // the core's lines (a, c) over K = b: the A operand of every chunk's Q GEMM, sliced once
  // per evaluation instead of once per y-chunk (cfg4: 11 chunks x 26 GB)
  const bool core_once = oz_x && r1 <= oz::KMAX;
  if (core_once) oz_slice_a(c, t.core.p, 1, r0, r0 * r2, r1, sCore, r0, r0 * r1);
  for (int64_t j0 = 0; j0 < nj; j0 += njc) {
    const int64_t njj = std::min(njc, nj - j0);
    if (oz_x) {  // Q[a, j, c] = sum_b core[a, b, c] U1[j, b]: A lines (a, c), one launch
      oz::OzOut o = oz_out(Q.p, r0);
      o.mr = r0;
      o.rs = r0 * njj;
      if (core_once) {
        OzSliced sU1;
        oz_slice_b(c, U1 + j0, 1, t.N[1], njj, r1, sU1);
        oz_run(c, sCore, sU1, o, "gemm_eval_q(ozaki-i8)");
      } else {
        ozaki_gemm_ex(c, r0 * r2, njj, r1, t.core.p, 1, r0, r0, r0 * r1, U1 + j0, 1, t.N[1], o,
                      "gemm_eval_q(ozaki-i8)");
      }
    } else {
      GemmOpts oq = tagged("gemm_eval_q");
      oq.batch = r2;
      oq.sA = r0 * r1;
      oq.sC = r0 * njj;
      gemm(c, false, true, r0, njj, r1, 1.0, t.core.p, r0, U1 + j0, t.N[1], 0.0, Q.p, r0, oq);
    }
    if (oz_x) oz_slice_a(c, Q.p, 1, r0 * njj, r0 * njj, r2, sQ);
    for (int64_t k0 = 0; k0 < nk; k0 += nkc) {
      const int64_t nkk = std::min(nkc, nk - k0);
      if (oz_x) {  // X = Q x_3 U2: B = U2[k0:k0+nkk, :]^T, lines = its rows
        OzSliced sU2;
        oz_slice_b(c, U2 + k0, 1, t.N[2], nkk, r2, sU2);
        oz_run(c, sQ, sU2, oz_out(X.p, r0 * njj), "gemm_eval_x(ozaki-i8)");
      } else {
        gemm(c, false, true, r0 * njj, nkk, r2, 1.0, Q.p, r0 * njj, U2 + k0, t.N[2], 0.0, X.p,
             r0 * njj, tagged("gemm_eval_x"));
      }
      if (oz_v) {  // V_k = U0 X_k for the nkk slabs: B lines = the columns (j, k) of X
        OzSliced sX;
        oz_slice_b(c, X.p, r0, 1, njj * nkk, r0, sX);
        oz::OzOut o = oz_out(out + k0 * ni * nj + j0 * ni, ni);
        o.nb = njj;
        o.bs = ni * nj;
        oz_run(c, sU0, sX, o, "gemm_eval_slab(ozaki-i8)");
        continue;
      }
      GemmOpts ov = tagged("gemm_eval_slab");
      ov.batch = nkk;
      ov.sB = r0 * njj;
      ov.sC = ni * nj;
      gemm(c, false, false, ni, njj, r0, 1.0, U0, t.N[0], X.p, r0, 0.0,
           out + k0 * ni * nj + j0 * ni, ni, ov);
    }
  }
  if (t.core_slab) allreduce(c, out, size_t(ni * nj * nk));  // the ranks' partial boxes
}

// Canonical (dictionary) tensor on an ni x nj x nk box: V_k = A0 X_k with
// A0[:, t] = D0[:, c0_t] and X_k[t, j] = w_t D2[k, c2_t] D1[j, c1_t] (to_dense,
// canonical.hpp:192-202, as one GEMM per z-slab).  D_l point at the box's first row.
// Grouped form for T merged terms over d0 < T distinct mode-0 columns (terms sorted by
// c0, segments seg0): per z-chunk Y_a = sum_{t in seg a} w_t D1[:, c1_t] D2[k, c2_t]^T
// (one segmented GEMM, 2 T nj nk flops over the box) and V = D0 Y^T (2 d0 ni nj nk flops
// instead of 2 T ni nj nk; BASELINE cfg5: d0 = 8283 vs T = 65065).
void cp_eval_grouped(latsum_ctx* c, const double* const D[3], const int64_t ld[3],
                     const int32_t* const tc[3], const double* tw, int64_t T, const int64_t* seg0,
                     int64_t d0, int64_t ni, int64_t nj, int64_t nk, double* out, const char* tag) {
  DBuf G1(c, size_t(nj) * T);  // G1[:, t] = w_t D1[:, c1_t]
  k_gather_scale<<<grid_for(nj * T), 256, 0, c->stream>>>(D[1], nj, ld[1], tc[1], tw, T, G1.p);
  post_launch(c);
  // z-chunks of whole 128-column tiles of the segmented GEMM where a 20 GiB Y allows it (cfg5:
  // the 4 GiB cap gave 31 slices per chunk, a quarter of every 128-wide tile), else what fits
  const int64_t budget = int64_t(1) << 29;
  int64_t cap = std::min<int64_t>(5 * budget / std::max<int64_t>(nj * d0, 1), 65535);
  if (cap >= 128) cap = cap / 128 * 128;
  else cap = std::max<int64_t>(1, std::min<int64_t>(budget / std::max<int64_t>(nj * d0, 1), 65535));
  const int64_t nkc = balanced_chunk(nk, cap, cap >= 128 ? 128 : 1);
  DBuf G2(c, size_t(nkc) * T), Y(c, size_t(nj) * nkc * d0);
  const bool oz = eval_uses_ozaki(d0);
  OzSliced sD0;
  if (oz) oz_slice_a(c, D[0], 1, ld[0], ni, d0, sD0);
  for (int64_t k0 = 0; k0 < nk; k0 += nkc) {
    const int64_t nkk = std::min(nkc, nk - k0);
    k_gather_scale<<<grid_for(nkk * T), 256, 0, c->stream>>>(D[2] + k0, nkk, ld[2], tc[2], nullptr,
                                                              T, G2.p);
    post_launch(c);
    GemmOpts o = tagged("gemm_eval_group");
    o.batch = d0;
    o.sC = nj * nkk;
    o.kseg = seg0;
    gemm(c, false, true, nj, nkk, T, 1.0, G1.p, nj, G2.p, nkk, 0.0, Y.p, nj, o);
    if (oz) {
      OzSliced sY;  // lines = the (j, k) columns of V, K = d0
      oz_slice_b(c, Y.p, 1, nj * nkk, nj * nkk, d0, sY);
      oz_run(c, sD0, sY, oz_out(out + k0 * ni * nj, ni), ozaki_tag(tag));
    } else {
      gemm(c, false, true, ni, nj * nkk, d0, 1.0, D[0], ld[0], Y.p, nj * nkk, 0.0,
           out + k0 * ni * nj, ni, tagged(tag));
    }
  }
}

void cp_eval(latsum_ctx* c, const double* const D[3], const int64_t ld[3], const int32_t* const tc[3],
             const double* tw, int64_t T, int64_t ni, int64_t nj, int64_t nk, double* out,
             const char* tag, const int64_t* seg0 = nullptr, int64_t d0 = 0) {
  if (T == 0) {
    CK(cudaMemsetAsync(out, 0, sizeof(double) * ni * nj * nk, c->stream));
    return;
  }
  static const bool cp_gemm = std::getenv("LATSUM_CP_GEMM") != nullptr;  // A/B: slab GEMMs
  if (T <= CP_MAXT && !cp_gemm) {  // low rank (cfg1: 17 merged terms): output-write bound kernel
    ProfScope ps(c, "cp_eval_small", 8.0 * double(ni) * double(nj) * double(nk));
    const int64_t pairs = nj * nk;
    auto grid_of = [&](int ipt, int minb) {
      const unsigned gx = unsigned((ni + CP_THREADS * ipt - 1) / (CP_THREADS * ipt));
      const unsigned gy = unsigned(std::max<int64_t>(1, std::min<int64_t>(
          (pairs + CP_PAIRS - 1) / CP_PAIRS, std::max<int64_t>(1, 148 * minb / int64_t(gx)))));
      return dim3(gx, gy);
    };
#define LATSUM_CP(MT)                                                                         \
  k_cp_eval_small<MT><<<grid_of(cp_ipt<MT>(), cp_minb<MT>()), CP_THREADS, 0, c->stream>>>(                   \
      D[0], ld[0], D[1], ld[1], D[2], ld[2], tc[0], tc[1], tc[2], tw, int(T), ni, nj, nk, out)
    switch ((T + 1) / 2 * 2) {  // rank buckets: even T up to 24, then 32 / 48 / 64
      case 2: LATSUM_CP(2); break;
      case 4: LATSUM_CP(4); break;
      case 6: LATSUM_CP(6); break;
      case 8: LATSUM_CP(8); break;
      case 10: LATSUM_CP(10); break;
      case 12: LATSUM_CP(12); break;
      case 14: LATSUM_CP(14); break;
      case 16: LATSUM_CP(16); break;
      case 18: LATSUM_CP(18); break;
      case 20: LATSUM_CP(20); break;
      case 22: LATSUM_CP(22); break;
      case 24: LATSUM_CP(24); break;
      default:
        if (T <= 32) LATSUM_CP(32);
        else if (T <= 48) LATSUM_CP(48);
        else LATSUM_CP(64);
    }
#undef LATSUM_CP
    post_launch(c);
    return;
  }
  if (seg0 && d0 > 0 && 2 * d0 <= T)
    return cp_eval_grouped(c, D, ld, tc, tw, T, seg0, d0, ni, nj, nk, out, tag);
  DBuf A0(c, size_t(ni) * T);
  k_gather_scale<<<grid_for(ni * T), 256, 0, c->stream>>>(D[0], ni, ld[0], tc[0], nullptr, T, A0.p);
  post_launch(c);
  const int64_t budget = int64_t(1) << 28;
  const int64_t nkc = balanced_chunk(nk, std::min<int64_t>(budget / std::max<int64_t>(T * nj, 1), 65535), 1);
  DBuf X(c, size_t(T) * nj * nkc);
  for (int64_t k0 = 0; k0 < nk; k0 += nkc) {
    const int64_t nkk = std::min(nkc, nk - k0);
    k_canonical_slab_operand<<<grid_for(T * nj * nkk), 256, 0, c->stream>>>(
        D[1], ld[1], D[2], ld[2], tc[1], tc[2], tw, T, 0, nj, k0, nkk, X.p);
    post_launch(c);
    if (eval_uses_ozaki(T)) {
      ozaki_gemm(c, ni, nj * nkk, T, A0.p, ni, X.p, T, out + k0 * ni * nj, ni, tag);
      continue;
    }
    GemmOpts ov = tagged(tag);
    ov.batch = nkk;
    ov.sB = T * nj;
    ov.sC = ni * nj;
    gemm(c, false, false, ni, nj, T, 1.0, A0.p, ni, X.p, T, 0.0, out + k0 * ni * nj, ni, ov);
  }
}

void canonical_eval(latsum_ctx* c, const latsum_canonical& can, const int64_t lo[3],
                    const int64_t hi[3], double* out) {
  terms(c, can);
  check_box(can.N, lo, hi);
  const double* D[3] = {can.dict[0].p + lo[0], can.dict[1].p + lo[1], can.dict[2].p + lo[2]};
  const int32_t* tc[3] = {can.dtc[0].p, can.dtc[1].p, can.dtc[2].p};
  cp_eval(c, D, can.N, tc, can.dtw.p, can.T, hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2], out,
          "gemm_eval_canonical", can.dtseg.p, can.d[0]);
}

// Projected-CP evaluation of a RHOSVD result: E_l = U_l[box rows] P_l, then the
// canonical slab GEMMs over the merged terms.  Equal to the Tucker tensor's values.
void projected_eval(latsum_ctx* c, const latsum_tucker& t, const int64_t lo[3], const int64_t hi[3],
                    double* out) {
  check_box(t.N, lo, hi);
  require(t.T > 0 || t.d[0] == 0, "projected evaluation needs the projected factors");
  int64_t n[3];
  DBuf E[3];
  const double* D[3];
  for (int l = 0; l < 3; ++l) {
    n[l] = hi[l] - lo[l];
    E[l].alloc(c, size_t(n[l]) * t.d[l]);
    gemm(c, false, false, n[l], t.d[l], t.r[l], 1.0, t.U[l].p + lo[l], t.N[l], t.P[l].p, t.r[l],
         0.0, E[l].p, n[l], tagged("gemm_eval_project"));
    D[l] = E[l].p;
  }
  const int32_t* tc[3] = {t.tc[0].p, t.tc[1].p, t.tc[2].p};
  cp_eval(c, D, n, tc, t.tw.p, t.T, n[0], n[1], n[2], out, "gemm_eval_projected", t.tseg.p, t.d[0]);
}

void projected_probes(latsum_ctx* c, const latsum_tucker& t, const int64_t* probes, int64_t np,
                      double* out_host) {
  std::vector<int64_t> hp(probes, probes + 3 * np), diag(3 * np);
  for (int64_t p = 0; p < np; ++p) diag[3 * p] = diag[3 * p + 1] = diag[3 * p + 2] = p;
  DVec<int64_t> dp, dd;
  dp.upload(c, hp);
  dd.upload(c, diag);
  DBuf rows(c, size_t(np) * std::max({t.r[0], t.r[1], t.r[2]})), E[3], res(c, np);
  for (int l = 0; l < 3; ++l) {
    k_gather_rows<<<grid_for(np * t.r[l]), 256, 0, c->stream>>>(t.U[l].p, t.N[l], t.r[l], dp.p, l,
                                                                np, rows.p);
    post_launch(c);
    E[l].alloc(c, size_t(np) * t.d[l]);
    gemm(c, false, false, np, t.d[l], t.r[l], 1.0, rows.p, np, t.P[l].p, t.r[l], 0.0, E[l].p, np,
         tagged("gemm_probes"));
  }
  k_canonical_probes<<<unsigned(np), 256, 0, c->stream>>>(E[0].p, np, E[1].p, np, E[2].p, np,
                                                         t.tc[0].p, t.tc[1].p, t.tc[2].p, t.tw.p,
                                                         t.T, dd.p, res.p);
  post_launch(c);
  CK(cudaMemcpyAsync(out_host, res.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

void tucker_probes(latsum_ctx* c, const latsum_tucker& t, const int64_t* probes, int64_t np,
                   double* out_host) {
  for (int64_t p = 0; p < np; ++p)
    for (int l = 0; l < 3; ++l)
      if (probes[3 * p + l] < 0 || probes[3 * p + l] >= t.N[l])
        throw Error(LATSUM_ERR_INVALID_ARGUMENT, "TuckerTensor::entry index out of range");
  if (!t.has_core) return projected_probes(c, t, probes, np, out_host);
  // a core slab: the partial sum over mode-0 indices [a0, a0 + ra), then the ranks' sum
  const int64_t r0 = t.core_slab ? t.ra : t.r[0], r12 = t.r[1] * t.r[2];
  const double* U0 = t.U[0].p + (t.core_slab ? t.a0 * t.N[0] : 0);
  const int64_t budget = int64_t(1) << 28;
  const int64_t pc = std::max<int64_t>(1, std::min<int64_t>(np, budget / std::max<int64_t>(r12, 1)));
  std::vector<int64_t> hp(probes, probes + 3 * np);
  DVec<int64_t> dp;
  dp.upload(c, hp);
  DBuf rowsU(c, size_t(pc) * r0), Wm(c, size_t(pc) * r12), res(c, np);
  for (int64_t p0 = 0; p0 < np; p0 += pc) {
    const int64_t npp = std::min(pc, np - p0);
    if (r0 == 0) {  // an empty slab contributes zeros
      CK(cudaMemsetAsync(Wm.p, 0, sizeof(double) * npp * r12, c->stream));
    } else {
      k_gather_rows<<<grid_for(npp * r0), 256, 0, c->stream>>>(U0, t.N[0], r0, dp.p + 3 * p0, 0,
                                                               npp, rowsU.p);
      post_launch(c);
      gemm(c, false, false, npp, r12, r0, 1.0, rowsU.p, npp, t.core.p, r0, 0.0, Wm.p, npp,
           tagged("gemm_probes"));
    }
    k_tucker_probe_finish<<<unsigned(npp), 256, 0, c->stream>>>(
        Wm.p, npp, t.r[1], t.r[2], t.U[1].p, t.N[1], t.U[2].p, t.N[2], dp.p + 3 * p0, res.p + p0);
    post_launch(c);
  }
  if (t.core_slab) allreduce(c, res.p, size_t(np));
  CK(cudaMemcpyAsync(out_host, res.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int latsum_ctx_create(int device, latsum_ctx** out) {
  if (!out) return LATSUM_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  auto* c = new latsum_ctx();
  int st = guarded(c, [&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, "latsum_ctx_create: no CUDA device " + std::to_string(device));
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
    CS(cusolverDnCreate(&c->solver));
    CS(cusolverDnSetStream(c->solver, c->stream));
    CS(cusolverDnCreateParams(&c->solver_params));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Pre-grow the stream-ordered pool so steady-state steps never map new memory
    // (LATSUM_POOL_RESERVE_GB; default 45% of the free device memory, ~80 GB on a B200; 0
    // disables).  A pool too small to grow (the caller holding the rest of HBM) makes
    // cudaMallocAsync on one worker stream wait for memory freed on another: cfg4 steps then
    // stalled by 150-1000 ms.  The pool does not release memory (threshold max); trim it
    // with latsum_ctx_trim_pool.
    const char* e = std::getenv("LATSUM_POOL_RESERVE_GB");
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const size_t want = e ? size_t(std::atof(e) * 1073741824.0) : size_t(0.45 * double(free_b));
    if (want > 0 && want < free_b) {
      void* p = nullptr;
      CK(cudaMallocAsync(&p, want, c->stream));
      CK(cudaFreeAsync(p, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
  });
  if (st != LATSUM_OK) {
    static thread_local std::string last;
    last = c->err;
    fprintf(stderr, "latsum_ctx_create: %s\n", last.c_str());
    delete c;
    return st;
  }
  *out = c;
  return LATSUM_OK;
}

void latsum_ctx_destroy(latsum_ctx* c) {
  if (c)
    for (cudaStream_t* st : {&c->sink.copy, &c->sink.copy2})
      if (*st) {
        cudaStreamSynchronize(*st);
        cudaStreamDestroy(*st);
        *st = nullptr;
      }
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  try { prof_harvest(c); } catch (...) {}
  for (auto e : c->pool) cudaEventDestroy(e);
  for (auto* w : c->sub)
    if (w) latsum_ctx_destroy(w);
  if (c->comm) {
    try { nccl().CommDestroy(c->comm); } catch (...) {}
  }
  if (c->solver_params) cusolverDnDestroyParams(c->solver_params);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

const char* latsum_last_error(const latsum_ctx* c) { return c ? c->err.c_str() : "no context"; }

int latsum_ctx_set_host_sink(latsum_ctx* c, double* core, int64_t core_cap, double* const factors[3],
                             const int64_t factor_cap[3]) {
  return guarded(c, [&] {
    require(c, "latsum_ctx_set_host_sink: null context");
    auto& sk = c->sink;
    sk.core = core;
    sk.core_cap = core ? core_cap : 0;
    for (int l = 0; l < 3; ++l) {
      sk.f[l] = core && factors ? factors[l] : nullptr;
      sk.f_cap[l] = core && factor_cap ? factor_cap[l] : 0;
    }
  });
}

int latsum_tucker_sink_written(const latsum_tucker* t) { return t && t->sink_written ? 1 : 0; }

int latsum_ctx_trim_pool(latsum_ctx* c, int64_t keep_bytes) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->stream));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
    CK(cudaMemPoolTrimTo(pool, size_t(std::max<int64_t>(keep_bytes, 0))));
  });
}

int latsum_ctx_set_stream(latsum_ctx* c, void* s) {
  return guarded(c, [&] {
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
    CS(cusolverDnSetStream(c->solver, c->stream));
  });
}

int latsum_ctx_synchronize(latsum_ctx* c) {
  return guarded(c, [&] { CK(cudaStreamSynchronize(c->stream)); });
}

int64_t latsum_ctx_kernel_launches(const latsum_ctx* c) { return c ? c->launches : 0; }

int64_t latsum_ctx_eig_fallbacks(const latsum_ctx* c) {
  if (!c) return 0;
  int64_t n = c->eig_fallbacks;
  for (auto* w : c->sub)
    if (w) n += w->eig_fallbacks;
  return n;
}

int latsum_comm_unique_id(unsigned char id[128]) {
  try {
    NcclUid u;
    NC(nccl().GetUniqueId(&u));
    std::memcpy(id, u.internal, 128);
    return LATSUM_OK;
  } catch (const Error& e) {
    return e.code;
  }
}

int latsum_ctx_init_comm(latsum_ctx* c, const unsigned char id[128], int rank, int nranks) {
  return guarded(c, [&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "latsum_ctx_init_comm: bad rank");
    require(!c->comm, "latsum_ctx_init_comm: communicator already set");
    c->rank = rank;
    c->nranks = nranks;
    if (nranks == 1) return;
    NcclUid u;
    std::memcpy(u.internal, id, 128);
    CK(cudaSetDevice(c->device));
    NC(nccl().CommInitRank(&c->comm, nranks, u, rank));
    for (int i = 0; i < 4; ++i) {  // one communicator per worker stream, split in order
      latsum_ctx* w = sub_ctx(c, i);
      NC(nccl().CommSplit(c->comm, 0, rank, &w->comm, nullptr));
    }
  });
}

int latsum_ctx_init_host_comm(latsum_ctx* c, int rank, int nranks, latsum_host_allreduce_fn ar,
                              latsum_host_allgather_fn ag, void* user) {
  return guarded(c, [&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "latsum_ctx_init_host_comm: bad rank");
    require(!c->comm, "latsum_ctx_init_host_comm: an NCCL communicator is already set");
    require(nranks == 1 || (ar && ag), "latsum_ctx_init_host_comm: null collective");
    c->rank = rank;
    c->nranks = nranks;
    c->host_ar = ar;
    c->host_ag = ag;
    c->host_user = user;
    c->channel = 0;
  });
}

int latsum_ctx_comm_info(const latsum_ctx* c, int* rank, int* nranks) {
  if (!c) return LATSUM_ERR_INVALID_ARGUMENT;
  if (rank) *rank = c->rank;
  if (nranks) *nranks = c->nranks;
  return LATSUM_OK;
}

int latsum_ctx_set_profiling(latsum_ctx* c, int on) {
  return guarded(c, [&] {
    prof_harvest(c);
    c->prof = on != 0;
    c->stats.clear();
  });
}

int64_t latsum_ctx_profile(latsum_ctx* c, char* buf, int64_t cap) {
  std::string out;
  int st = guarded(c, [&] {
    prof_harvest(c);
    char line[256];
    for (const auto& kv : c->stats) {
      snprintf(line, sizeof(line), "%s %lld %.6f %.6e\n", kv.first.c_str(),
               (long long)kv.second.count, kv.second.ms, kv.second.work);
      out += line;
    }
  });
  if (st != LATSUM_OK) return -1;
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(out.size(), size_t(cap - 1));
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return int64_t(out.size());
}

int latsum_reference_build(latsum_ctx* c, int family, double lambda, const int64_t N[3],
                           const double box[3], int M, double step_constant,
                           latsum_reference** out) {
  return guarded(c, [&] {
    require(out && N && box, "latsum_reference_build: null argument");
    auto ref = std::make_unique<latsum_reference>();
    build_reference(c, family, lambda, N, box, M, step_constant, *ref);
    *out = ref.release();
  });
}

void latsum_reference_destroy(latsum_reference* ref) { delete ref; }

int latsum_reference_info(const latsum_reference* ref, int* rank, double* c0, double shell[2]) {
  if (!ref) return LATSUM_ERR_INVALID_ARGUMENT;
  if (rank) *rank = ref->R;
  if (c0) *c0 = ref->C0;
  if (shell) { shell[0] = ref->shell[0]; shell[1] = ref->shell[1]; }
  return LATSUM_OK;
}

int latsum_reference_factor(latsum_ctx* c, const latsum_reference* ref, int mode, double* factor) {
  return guarded(c, [&] {
    require(ref && factor && mode >= 0 && mode < 3, "latsum_reference_factor: bad argument");
    const int64_t n2 = 2 * ref->N[mode];
    std::vector<double> d(size_t(n2) * ref->Rd);
    CK(cudaMemcpyAsync(d.data(), ref->col(mode), sizeof(double) * d.size(), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < ref->R; ++k)
      std::memcpy(factor + size_t(k) * n2, d.data() + size_t(ref->jmap[k]) * n2, sizeof(double) * n2);
  });
}

int latsum_reference_weights(const latsum_reference* ref, double* w) {
  if (!ref || !w) return LATSUM_ERR_INVALID_ARGUMENT;
  std::memcpy(w, ref->weights.data(), sizeof(double) * ref->R);
  return LATSUM_OK;
}

int latsum_reference_quadrature(const latsum_reference* ref, double* nodes, double* weights) {
  if (!ref) return LATSUM_ERR_INVALID_ARGUMENT;
  if (nodes) std::memcpy(nodes, ref->nodes.data(), sizeof(double) * ref->R);
  if (weights) std::memcpy(weights, ref->qweights.data(), sizeof(double) * ref->R);
  return LATSUM_OK;
}

int latsum_canonical_assemble(latsum_ctx* c, const latsum_reference* ref, int64_t nsub,
                              const int64_t* sub_counts, const int64_t* sub_shifts,
                              const double* sub_charges, int64_t ndef, const int64_t* def_shifts,
                              const double* def_charges, latsum_canonical** out) {
  return guarded(c, [&] {
    require(ref && out, "latsum_canonical_assemble: null argument");
    auto can = std::make_unique<latsum_canonical>();
    assemble(c, *ref, nsub, sub_counts, sub_shifts, sub_charges, ndef, def_shifts, def_charges,
             *can);
    *out = can.release();
  });
}

int latsum_canonical_assemble_blocks(latsum_ctx* c, const latsum_reference* ref, int64_t nblk,
                                     const int64_t* blk_counts, const int64_t* blk_shifts,
                                     const double* blk_charges, latsum_canonical** out) {
  return guarded(c, [&] {
    require(ref && out, "latsum_canonical_assemble_blocks: null argument");
    require(nblk == 0 || (blk_counts && blk_shifts && blk_charges),
            "latsum_canonical_assemble_blocks: null block table");
    auto can = std::make_unique<latsum_canonical>();
    assemble_blocks(c, *ref, nblk, blk_counts, blk_shifts, blk_charges, *can);
    *out = can.release();
  });
}

void latsum_canonical_destroy(latsum_canonical* can) { delete can; }

int latsum_canonical_info(const latsum_canonical* can, int64_t dims[3], int64_t* rank,
                          int64_t dict_cols[3], int64_t* merged_terms) {
  if (!can) return LATSUM_ERR_INVALID_ARGUMENT;
  for (int l = 0; l < 3; ++l) {
    if (dims) dims[l] = can->N[l];
    if (dict_cols) dict_cols[l] = can->d[l];
  }
  if (rank) *rank = can->Mc;
  if (merged_terms) {
    try {  // waits for the host-side term merge (which reports its failure here)
      *merged_terms = terms_host(*can).T;
    } catch (const std::bad_alloc&) {
      return LATSUM_ERR_OUT_OF_MEMORY;
    } catch (...) {
      return LATSUM_ERR_INVALID_ARGUMENT;
    }
  }
  return LATSUM_OK;
}

int latsum_canonical_weights(const latsum_canonical* can, double* w) {
  if (!can || !w) return LATSUM_ERR_INVALID_ARGUMENT;
  std::memcpy(w, can->weights.data(), sizeof(double) * can->Mc);
  return LATSUM_OK;
}

int latsum_canonical_factor_device(latsum_ctx* c, const latsum_canonical* can, int mode,
                                   double* dst) {
  return guarded(c, [&] {
    require(can && dst && mode >= 0 && mode < 3, "latsum_canonical_factor: bad argument");
    materialize_factor(c, *can, mode, dst);
  });
}

int latsum_canonical_factor(latsum_ctx* c, const latsum_canonical* can, int mode, double* factor) {
  return guarded(c, [&] {
    require(can && factor && mode >= 0 && mode < 3, "latsum_canonical_factor: bad argument");
    DBuf tmp(c, size_t(can->N[mode]) * can->Mc);
    materialize_factor(c, *can, mode, tmp.p);
    CK(cudaMemcpyAsync(factor, tmp.p, sizeof(double) * tmp.n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_canonical_entries(latsum_ctx* c, const latsum_canonical* can, const int64_t* probes,
                             int64_t np, double* out) {
  return guarded(c, [&] {
    require(can && (np == 0 || (probes && out)), "latsum_canonical_entries: bad argument");
    if (np == 0) return;
    for (int64_t p = 0; p < np; ++p)
      for (int l = 0; l < 3; ++l)
        if (probes[3 * p + l] < 0 || probes[3 * p + l] >= can->N[l])
          throw Error(LATSUM_ERR_INVALID_ARGUMENT, "CanonicalTensor::entry index out of range");
    terms(c, *can);
    if (can->T == 0) {
      std::fill(out, out + np, 0.0);
      return;
    }
    std::vector<int64_t> hp(probes, probes + 3 * np);
    DVec<int64_t> dp;
    dp.upload(c, hp);
    DBuf res(c, np);
    k_canonical_probes<<<unsigned(np), 256, 0, c->stream>>>(
        can->dict[0].p, can->N[0], can->dict[1].p, can->N[1], can->dict[2].p, can->N[2],
        can->dtc[0].p, can->dtc[1].p, can->dtc[2].p, can->dtw.p, can->T, dp.p, res.p);
    post_launch(c);
    CK(cudaMemcpyAsync(out, res.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_canonical_norm(latsum_ctx* c, const latsum_canonical* can, double* out) {
  return guarded(c, [&] {
    require(can && out, "latsum_canonical_norm: null argument");
    *out = canonical_norm(c, *can);
  });
}

int latsum_canonical_eval_box_device(latsum_ctx* c, const latsum_canonical* can,
                                     const int64_t lo[3], const int64_t hi[3], double* out) {
  return guarded(c, [&] {
    require(can && lo && hi && out, "latsum_canonical_eval_box: null argument");
    canonical_eval(c, *can, lo, hi, out);
  });
}

int latsum_rhosvd(latsum_ctx* c, const latsum_canonical* can, const int64_t* ranks,
                  double tolerance, int deflate, latsum_tucker** out,
                  latsum_spectral_report* report) {
  return latsum_rhosvd_ex(c, can, ranks, tolerance, deflate, 0, out, report);
}

int latsum_rhosvd_ex(latsum_ctx* c, const latsum_canonical* can, const int64_t* ranks,
                     double tolerance, int deflate, int flags, latsum_tucker** out,
                     latsum_spectral_report* report) {
  return guarded(c, [&] {
    require(can && out, "latsum_rhosvd: null argument");
    auto t = std::make_unique<latsum_tucker>();
    latsum_spectral_report rep;
    rhosvd_impl(c, *can, ranks, tolerance, deflate, *t, rep,
                (flags & LATSUM_RHOSVD_FACTORS_ONLY) == 0, (flags & LATSUM_RHOSVD_CORE_SLABS) != 0);
    if (report) *report = rep;
    *out = t.release();
  });
}

void latsum_tucker_destroy(latsum_tucker* t) { delete t; }

int latsum_tucker_has_core(const latsum_tucker* t) { return t && t->has_core ? 1 : 0; }

int latsum_tucker_info(const latsum_tucker* t, int64_t dims[3], int64_t ranks[3]) {
  if (!t) return LATSUM_ERR_INVALID_ARGUMENT;
  for (int l = 0; l < 3; ++l) {
    if (dims) dims[l] = t->N[l];
    if (ranks) ranks[l] = t->r[l];
  }
  return LATSUM_OK;
}

int latsum_tucker_singular_values(const latsum_tucker* t, int mode, double* out) {
  if (!t || !out || mode < 0 || mode > 2) return LATSUM_ERR_INVALID_ARGUMENT;
  std::memcpy(out, t->sigma[mode].data(), sizeof(double) * t->sigma[mode].size());
  return LATSUM_OK;
}

int latsum_tucker_core_slab(latsum_ctx* c, const latsum_tucker* t, int64_t* a0, int64_t* ra,
                            double* core) {
  return guarded(c, [&] {
    require(t && a0 && ra, "latsum_tucker_core_slab: null argument");
    require(t->has_core, "latsum_tucker_core_slab: the tensor has no dense core");
    *a0 = t->core_slab ? t->a0 : 0;
    *ra = t->core_slab ? t->ra : t->r[0];
    if (core && *ra > 0) {
      CK(cudaMemcpyAsync(core, t->core.p, sizeof(double) * *ra * t->r[1] * t->r[2],
                         cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
  });
}

int latsum_tucker_core(latsum_ctx* c, const latsum_tucker* t, double* core) {
  return guarded(c, [&] {
    require(!t || !t->core_slab,
            "latsum_tucker_core: the core is distributed over the ranks (latsum_tucker_core_slab)");
    require(t && core, "latsum_tucker_core: null argument");
    require(t->has_core, "latsum_tucker_core: the dense core was not formed (factors-only RHOSVD)");
    CK(cudaMemcpyAsync(core, t->core.p, sizeof(double) * t->r[0] * t->r[1] * t->r[2],
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_tucker_factor(latsum_ctx* c, const latsum_tucker* t, int mode, double* f) {
  return guarded(c, [&] {
    require(t && f && mode >= 0 && mode < 3, "latsum_tucker_factor: bad argument");
    CK(cudaMemcpyAsync(f, t->U[mode].p, sizeof(double) * t->N[mode] * t->r[mode],
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_tucker_projected_form(latsum_ctx* c, const latsum_tucker* t, int64_t d[3], int64_t* T,
                                  double* P0, double* P1, double* P2, int32_t* c0, int32_t* c1,
                                  int32_t* c2, double* w) {
  return guarded(c, [&] {
    require(t && d && T, "latsum_tucker_projected_form: null argument");
    require(!t->has_core, "latsum_tucker_projected_form: the tensor carries a dense core");
    for (int l = 0; l < 3; ++l) d[l] = t->d[l];
    *T = t->T;
    double* P[3] = {P0, P1, P2};
    int32_t* tc[3] = {c0, c1, c2};
    for (int l = 0; l < 3; ++l) {
      if (P[l])
        CK(cudaMemcpyAsync(P[l], t->P[l].p, sizeof(double) * t->r[l] * t->d[l],
                           cudaMemcpyDeviceToHost, c->stream));
      if (tc[l] && t->T)
        CK(cudaMemcpyAsync(tc[l], t->tc[l].p, sizeof(int32_t) * t->T, cudaMemcpyDeviceToHost,
                           c->stream));
    }
    if (w && t->T)
      CK(cudaMemcpyAsync(w, t->tw.p, sizeof(double) * t->T, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_tucker_entries(latsum_ctx* c, const latsum_tucker* t, const int64_t* probes, int64_t np,
                          double* out) {
  return guarded(c, [&] {
    require(t && (np == 0 || (probes && out)), "latsum_tucker_entries: bad argument");
    if (np) tucker_probes(c, *t, probes, np, out);
  });
}

int latsum_tucker_eval_box_device(latsum_ctx* c, const latsum_tucker* t, const int64_t lo[3],
                                  const int64_t hi[3], double* out) {
  return guarded(c, [&] {
    require(t && lo && hi && out, "latsum_tucker_eval_box: null argument");
    tucker_eval(c, *t, lo, hi, out);
  });
}

int latsum_tucker_eval_box(latsum_ctx* c, const latsum_tucker* t, const int64_t lo[3],
                           const int64_t hi[3], double* out) {
  return guarded(c, [&] {
    require(t && lo && hi && out, "latsum_tucker_eval_box: null argument");
    check_box(t->N, lo, hi);
    const size_t n = size_t(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    DBuf tmp(c, n);
    tucker_eval(c, *t, lo, hi, tmp.p);
    CK(cudaMemcpyAsync(out, tmp.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_sum_to_tucker(latsum_ctx* c, int family, double lambda, const int64_t N[3],
                         const double box[3], int M, double step_constant, int64_t nsub,
                         const int64_t* sub_counts, const int64_t* sub_shifts,
                         const double* sub_charges, int64_t ndef, const int64_t* def_shifts,
                         const double* def_charges, double tolerance, latsum_tucker** out,
                         latsum_spectral_report* report) {
  return guarded(c, [&] {
    require(out, "latsum_sum_to_tucker: null argument");
    latsum_reference ref;
    build_reference(c, family, lambda, N, box, M, step_constant, ref);
    latsum_canonical can;
    assemble(c, ref, nsub, sub_counts, sub_shifts, sub_charges, ndef, def_shifts, def_charges, can);
    auto t = std::make_unique<latsum_tucker>();
    latsum_spectral_report rep;
    rhosvd_impl(c, can, nullptr, tolerance, LATSUM_DEFLATE_AUTO, *t, rep);
    if (report) *report = rep;
    *out = t.release();
  });
}

int latsum_canonical_from_host(latsum_ctx* c, const int64_t dims[3], int64_t rank,
                               const double* weights, const double* f0, const double* f1,
                               const double* f2, latsum_canonical** out) {
  return guarded(c, [&] {
    require(dims && out && rank >= 0 && (rank == 0 || (weights && f0 && f1 && f2)),
            "latsum_canonical_from_host: bad argument");
    require(rank < (int64_t(1) << 21), "latsum_canonical_from_host: rank too large");
    auto can = std::make_unique<latsum_canonical>();
    const double* f[3] = {f0, f1, f2};
    can->R = can->Rd = 1;
    can->Mc = can->T = rank;
    can->weights.assign(weights, weights + rank);
    can->tw = can->weights;
    can->tseg.resize(rank + 1);
    for (int64_t q = 0; q <= rank; ++q) can->tseg[q] = q;
    for (int l = 0; l < 3; ++l) {
      require(dims[l] >= 1, "CanonicalTensor: mode size must be positive");
      can->N[l] = dims[l];
      can->d[l] = rank;
      can->dict[l].alloc(c, size_t(dims[l]) * std::max<int64_t>(rank, 1));
      if (rank)
        CK(cudaMemcpyAsync(can->dict[l].p, f[l], sizeof(double) * dims[l] * rank,
                           cudaMemcpyHostToDevice, c->stream));
      can->dict_norms[l].assign(rank, 1.0);
      can->term_col[l].resize(rank);
      can->tc[l].resize(rank);
      for (int64_t q = 0; q < rank; ++q) can->term_col[l][q] = can->tc[l][q] = int32_t(q);
      can->mult[l].assign(rank, 1.0);
      can->dtc[l].upload(c, can->tc[l]);
    }
    can->dtw.upload(c, can->tw);
    can->dtseg.upload(c, can->tseg);
    for (int m = 0; m < 3; ++m) {
      can->sseg[m] = can->tseg;
      for (int l = 0; l < 3; ++l) can->stc[m][l] = can->tc[l];
      can->stw[m] = can->tw;
    }
    CK(cudaStreamSynchronize(c->stream));
    *out = can.release();
  });
}

int latsum_ctx_set_accumulation(latsum_ctx* c, int order) {
  if (!c || order < 0 || order > 2) return LATSUM_ERR_INVALID_ARGUMENT;
  c->accumulation = order == 0 ? 0 : 1;  // compensated: the ascending order (see the header)
  return LATSUM_OK;
}

int latsum_canonical_concat(latsum_ctx* c, const latsum_canonical* a, const latsum_canonical* b,
                            latsum_canonical** out) {
  return guarded(c, [&] {
    require(a && b && out, "latsum_canonical_concat: bad argument");
    for (int l = 0; l < 3; ++l)
      require(a->N[l] == b->N[l], "add_concat: mode size mismatch");
    auto can = std::make_unique<latsum_canonical>();
    can->R = a->R;
    can->Rd = 0;  // columns of more than one reference tensor
    can->Mc = a->Mc + b->Mc;
    can->weights = a->weights;
    can->weights.insert(can->weights.end(), b->weights.begin(), b->weights.end());
    for (int l = 0; l < 3; ++l) {
      const int64_t N = a->N[l], da = a->d[l], db = b->d[l];
      can->N[l] = N;
      can->d[l] = da + db;
      require(can->d[l] < (int64_t(1) << 21), "add_concat: too many distinct columns in a mode");
      can->dict[l].alloc(c, size_t(N) * std::max<int64_t>(da + db, 1));
      if (da)
        CK(cudaMemcpyAsync(can->dict[l].p, a->dict[l].p, sizeof(double) * N * da,
                           cudaMemcpyDeviceToDevice, c->stream));
      if (db)
        CK(cudaMemcpyAsync(can->dict[l].p + N * da, b->dict[l].p, sizeof(double) * N * db,
                           cudaMemcpyDeviceToDevice, c->stream));
      can->dict_norms[l] = a->dict_norms[l];
      can->dict_norms[l].insert(can->dict_norms[l].end(), b->dict_norms[l].begin(), b->dict_norms[l].end());
      can->mult[l] = a->mult[l];
      can->mult[l].insert(can->mult[l].end(), b->mult[l].begin(), b->mult[l].end());
      can->term_col[l] = a->term_col[l];
      can->term_col[l].reserve(size_t(can->Mc));
      for (int64_t col : b->term_col[l]) can->term_col[l].push_back(col + da);  // a's terms first
    }
    CK(cudaStreamSynchronize(c->stream));  // a and b may be destroyed right after the call
    merge_terms(*can);
    can->terms_async = true;  // terms() uploads the merged tables on first use
    std::promise<void> done;
    done.set_value();
    can->terms_ready = done.get_future().share();
    *out = can.release();
  });
}

int latsum_tensor_write(latsum_ctx* c, const latsum_canonical* can, const latsum_tucker* t,
                        const char* path) {
  return guarded(c, [&] {
    require(path && ((can != nullptr) != (t != nullptr)),
            "latsum_tensor_write: pass exactly one of canonical / tucker");
    require(!t || !t->core_slab, "latsum_tensor_write: the core is distributed over the ranks");
    FileSink f(path);
    if (can) {
      write_header(f, 'C', can->N);
      f.u32(uint32_t(can->Mc));
      f.put(can->weights.data(), sizeof(double) * can->Mc);
      for (int l = 0; l < 3; ++l) {
        DBuf tmp(c, size_t(can->N[l]) * std::max<int64_t>(can->Mc, 1));
        materialize_factor(c, *can, l, tmp.p);
        f.device(c, tmp.p, size_t(can->N[l]) * can->Mc);
      }
    } else {
      require(t->has_core, "latsum_tensor_write: factors-only Tucker result has no dense core");
      write_header(f, 'T', t->N);
      for (int l = 0; l < 3; ++l) f.u32(uint32_t(t->r[l]));
      f.device(c, t->core.p, size_t(t->r[0]) * t->r[1] * t->r[2]);
      for (int l = 0; l < 3; ++l) f.device(c, t->U[l].p, size_t(t->N[l]) * t->r[l]);
    }
    f.finish();
  });
}

int latsum_tensor_read(latsum_ctx* c, const char* path, latsum_canonical** can_out,
                       latsum_tucker** t_out) {
  return guarded(c, [&] {
    require(path && can_out && t_out, "latsum_tensor_read: null argument");
    *can_out = nullptr;
    *t_out = nullptr;
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Error(LATSUM_ERR_IO, std::string("cannot open ") + path);
    std::vector<char> buf((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
    if (buf.size() < 7 + 1 + 4 + 12 + 8) throw Error(LATSUM_ERR_IO, "tensor file truncated");
    uint64_t stored;
    std::memcpy(&stored, buf.data() + buf.size() - 8, 8);
    Fnv fnv;
    fnv.add(buf.data(), buf.size() - 8);
    if (stored != fnv.h)
      throw Error(LATSUM_ERR_IO, std::string("checksum mismatch in ") + path +
                                     " (corrupt or tampered file)");
    size_t at = 0;
    auto rd = [&](void* o, size_t n) {
      if (at + n > buf.size() - 8) throw Error(LATSUM_ERR_IO, "tensor file truncated");
      std::memcpy(o, buf.data() + at, n);
      at += n;
    };
    auto u32 = [&] {
      uint32_t v;
      rd(&v, 4);
      return int64_t(v);
    };
    char magic[7];
    rd(magic, 7);
    if (std::memcmp(magic, "LTSTNSR", 7) != 0) throw Error(LATSUM_ERR_IO, "bad magic");
    unsigned char version;
    rd(&version, 1);
    if (version != 1)
      throw Error(LATSUM_ERR_IO, "unsupported format version " + std::to_string(int(version)));
    char tag;
    rd(&tag, 1);
    at += 3;
    int64_t dims[3];
    for (int l = 0; l < 3; ++l) dims[l] = u32();
    if (tag == 'C') {
      const int64_t R = u32();
      std::vector<double> w(R), f[3];
      rd(w.data(), sizeof(double) * R);
      for (int l = 0; l < 3; ++l) {
        f[l].resize(size_t(dims[l]) * R);
        rd(f[l].data(), sizeof(double) * f[l].size());
      }
      latsum_canonical* can = nullptr;
      const int st = latsum_canonical_from_host(c, dims, R, w.data(), f[0].data(), f[1].data(),
                                                f[2].data(), &can);
      if (st != LATSUM_OK) throw Error(st, c->err);
      *can_out = can;
    } else if (tag == 'T') {
      auto t = std::make_unique<latsum_tucker>();
      for (int l = 0; l < 3; ++l) t->N[l] = dims[l];
      for (int l = 0; l < 3; ++l) t->r[l] = u32();
      const size_t nc = size_t(t->r[0]) * t->r[1] * t->r[2];
      std::vector<double> h(nc);
      rd(h.data(), sizeof(double) * nc);
      t->core.alloc(c, nc);
      CK(cudaMemcpyAsync(t->core.p, h.data(), sizeof(double) * nc, cudaMemcpyHostToDevice, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (int l = 0; l < 3; ++l) {
        std::vector<double> u(size_t(dims[l]) * t->r[l]);
        rd(u.data(), sizeof(double) * u.size());
        t->U[l].alloc(c, u.size());
        CK(cudaMemcpyAsync(t->U[l].p, u.data(), sizeof(double) * u.size(), cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        t->sigma[l].assign(1, 0.0);
      }
      t->has_core = true;
      *t_out = t.release();
    } else {
      throw Error(LATSUM_ERR_IO, "unknown format tag");
    }
  });
}

int latsum_canonical_to_tucker(latsum_ctx* c, const latsum_canonical* can, const int64_t* ranks,
                               double tolerance, int max_als_sweeps, double als_stagnation_tol,
                               latsum_tucker** out, latsum_spectral_report* report,
                               int* als_sweeps) {
  return guarded(c, [&] {
    require(can && out, "latsum_canonical_to_tucker: null argument");
    auto t = std::make_unique<latsum_tucker>();
    latsum_spectral_report rep;
    // cuSOLVER vectors for the ALS pipeline: its fixed-rank refinements amplify the
    // ~1e-11-level differences of the in-house inverse-iteration vectors into +-2 rank
    // changes after shrink_core
    struct Restore {
      latsum_ctx* c;
      int m;
      ~Restore() { c->eig_method = m; }
    } restore{c, c->eig_method};
    c->eig_method = 1;
    canonical_to_tucker_impl(c, *can, ranks, tolerance, max_als_sweeps, als_stagnation_tol, *t,
                             rep, als_sweeps);
    if (report) *report = rep;
    *out = t.release();
  });
}

int latsum_verify_entries(latsum_ctx* c, const latsum_reference* ref, int64_t ns,
                          const int64_t* shifts, const double* weights, const int64_t* probes,
                          int64_t np, double* out) {
  return guarded(c, [&] {
    require(ref && (ns == 0 || (shifts && weights)) && (np == 0 || (probes && out)),
            "latsum_verify_entries: bad argument");
    if (np == 0) return;
    for (int64_t q = 0; q < ns; ++q)
      for (int l = 0; l < 3; ++l) {
        const int64_t begin = ref->N[l] / 2 - shifts[3 * q + l];
        if (begin < 0 || begin + ref->N[l] > 2 * ref->N[l])
          throw Error(LATSUM_ERR_WINDOW_OVERFLOW,
                      "window overflow in mode " + std::to_string(l + 1) + ": source " +
                          std::to_string(q));
      }
    for (int64_t p = 0; p < np; ++p)
      for (int l = 0; l < 3; ++l)
        require(probes[3 * p + l] >= 0 && probes[3 * p + l] < ref->N[l],
                "oracle_entry: probe index out of range");
    DVec<int64_t> dsh, dpr;
    DVec<double> dsw, dwr;
    DVec<int32_t> djm;
    dsh.upload(c, std::vector<int64_t>(shifts, shifts + 3 * ns));
    dsw.upload(c, std::vector<double>(weights, weights + ns));
    dpr.upload(c, std::vector<int64_t>(probes, probes + 3 * np));
    dwr.upload(c, ref->weights);
    djm.upload(c, std::vector<int32_t>(ref->jmap.begin(), ref->jmap.end()));
    const int64_t chunk = std::max<int64_t>(4096, (ns + 255) / 256);
    const int nchunk = int(std::max<int64_t>(1, (ns + chunk - 1) / chunk));
    DBuf part(c, size_t(np) * nchunk), res(c, np);
    VerifyArgs a{{ref->col(0), ref->col(1), ref->col(2)}, {ref->N[0], ref->N[1], ref->N[2]},
                 djm.p, dwr.p, ref->R, dsh.p, dsw.p, ns, dpr.p, chunk, nchunk, part.p};
    if (ns > 0) {
      ProfScope ps(c, "verify_bruteforce", double(np) * double(ns) * ref->R * 4.0);
      k_verify_partial<<<dim3(unsigned(np), unsigned(nchunk)), 256, 0, c->stream>>>(a);
      post_launch(c);
    } else {
      CK(cudaMemsetAsync(part.p, 0, sizeof(double) * np * nchunk, c->stream));
    }
    k_verify_finish<<<unsigned((np + 255) / 256), 256, 0, c->stream>>>(part.p, nchunk, np, res.p);
    post_launch(c);
    CK(cudaMemcpyAsync(out, res.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_dgemm_device(latsum_ctx* c, int ta, int tb, int64_t M, int64_t N, int64_t K,
                        double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double beta, double* C, int64_t ldc) {
  return guarded(c, [&] {
    require(A && B && C && M >= 0 && N >= 0 && K >= 0, "latsum_dgemm_device: bad argument");
    gemm(c, ta != 0, tb != 0, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  });
}

int latsum_sytrd_device(latsum_ctx* c, int64_t n, double* A, int64_t lda, double* d, double* e,
                        double* tau) {
  return guarded(c, [&] {
    require(A && d && n >= 1 && lda >= n && (n == 1 || (e && tau)), "latsum_sytrd_device: bad argument");
    sytrd_cluster(c, n, A, lda, d, e, tau);
  });
}

int latsum_eig_sym_device(latsum_ctx* c, int64_t n, const double* A, int64_t k, double* w,
                          double* V, int method) {
  return guarded(c, [&] {
    require(A && w && n >= 1 && k >= 0 && k <= n && (k == 0 || V) && method >= 0 && method <= 3,
            "latsum_eig_sym_device: bad argument");
    DBuf G(c, size_t(n) * n);
    CK(cudaMemcpyAsync(G.p, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, c->stream));
    Eig e;
    e.solve(c, n, std::move(G), method);
    CK(cudaMemcpyAsync(w, e.lam_asc.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    e.leading(c, k, V);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int latsum_dgemm_ozaki_device(latsum_ctx* c, int tb, int64_t M, int64_t N, int64_t K,
                              const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                              int64_t ldc) {
  return guarded(c, [&] {
    require(A && B && C && M >= 0 && N >= 0 && K >= 0 && lda >= std::max<int64_t>(M, 1) &&
                ldb >= std::max<int64_t>(tb ? N : K, 1) && ldc >= std::max<int64_t>(M, 1),
            "latsum_dgemm_ozaki_device: bad argument");
    ozaki_gemm(c, M, N, K, A, lda, B, ldb, C, ldc, "gemm(ozaki-i8)", tb != 0);
  });
}

}  // extern "C"
