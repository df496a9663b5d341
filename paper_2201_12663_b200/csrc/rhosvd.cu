// rhosvd.cu - host orchestration and C ABI of the B200-native RHOSVD C2T path.
//
// Pipeline per call; all arithmetic runs in the kernels
// of this library, collectives are fp64 sum all-reduces over the R shards:
//   S1 normalize       Uhat_l = U_l diag(s_l)^-1, xi' = xi prod_l s_l, T_l
//   S2 Gram            G_l = Uhat_l Uhat_l^T                     [all-reduce]
//   S3 subspace iter.  Z <- CholQR(G Z V Theta^-1) with Rayleigh-Ritz alignment
//                      (Jacobi on Z^T G Z), adaptive block b = r + p          (Eq. svdr)
//   S4 one-sided RR    W = Z^T Uhat, W W^T = P Lambda P^T (Jacobi, high relative
//                      accuracy)                                   [all-reduce]
//      refinement      Z' = CholQR(Uhat W^T P Lambda^-1) (non-squared)  [all-reduce]
//      final RR        W' = Z'^T Uhat, W' W'^T = P' Lambda' P'^T, sigma = sqrt(Lambda')
//      rank            tail(r) = sum_{r<k<=b} Lambda'_k + ||Uhat - Z'W'||_F^2 <= eps^2 T  (A1, D2)
//   S5 projection      Z_l = Z' P'_r, W_l = P'_r^T W' (= Z_l^T Uhat_l)
//   S6 core            beta = (W1 (.) W2)(xi' o W3)^T                   [all-reduce]   (Prop. 2.1)
//   S7 report          tails, ||xi'||, Thm. 2.2 bound and its orthogonal form, ||beta||
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <chrono>
#include <condition_variable>
#include <thread>
#include <array>
#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "gemm.cuh"
#include "kernels.h"
#include "small_dense.cuh"

namespace rhosvd {

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local int g_coop_cap = 0;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

int device_guard() {
  static std::mutex mu;
  static int pinned = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(RHOSVD_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(mu);
  if (pinned < 0) pinned = dev;
  if (dev != pinned)
    return fail(RHOSVD_EINVAL, "librhosvd serves one CUDA device per process (first used " +
                                   std::to_string(pinned) + ", current " + std::to_string(dev) + ")");
  return RHOSVD_OK;
}

int num_sms() {
  static const int s = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return s;
}

// pinned staging blocks of d2h_wait (shared by all threads; a block is owned by one
// readback at a time)
static std::mutex g_pin_mu;
static std::multimap<size_t, void*> g_pin_free;

// one staging block out of the pool (or a new one of >= bytes)
static void* pin_get(size_t bytes, size_t* cap) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end()) {
      *cap = it->first;
      void* b = it->second;
      g_pin_free.erase(it);
      return b;
    }
  }
  void* b = nullptr;
  *cap = std::max<size_t>(4096, bytes);
  if (cudaMallocHost(&b, *cap) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return b;
}
static void pin_put(void* b, size_t cap) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace(cap, b);
}

int h2d_wait(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return RHOSVD_OK;
  size_t cap = 0;
  void* buf = pin_get(bytes, &cap);
  if (!buf) return fail(RHOSVD_ENOMEM, "pinned staging buffer");
  std::memcpy(buf, src, bytes);
  cudaError_t e = cudaMemcpyAsync(dst, buf, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  pin_put(buf, cap);
  if (e != cudaSuccess) return fail(RHOSVD_ECUDA, std::string("staging: ") + cudaGetErrorString(e));
  return RHOSVD_OK;
}

int d2h_wait(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return RHOSVD_OK;
  size_t cap = 0;
  void* buf = pin_get(bytes, &cap);
  if (!buf) return fail(RHOSVD_ENOMEM, "pinned readback buffer");
  cudaError_t e = cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) std::memcpy(dst, buf, bytes);
  pin_put(buf, cap);
  if (e != cudaSuccess) return fail(RHOSVD_ECUDA, std::string("readback: ") + cudaGetErrorString(e));
  return RHOSVD_OK;
}

struct DBuf {
  double* p = nullptr;
  size_t cap = 0;
  int ensure(size_t n, cudaStream_t st) {
    if (n <= cap && p) return RHOSVD_OK;
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(n, 64);
    cudaError_t e = cudaMallocAsync((void**)&p, want * sizeof(double), st);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return fail(RHOSVD_ENOMEM, std::string("workspace alloc: ") + cudaGetErrorString(e));
    }
    cap = want;
    return RHOSVD_OK;
  }
  // zero-initialised growth (padding must be zero)
  int ensure_zero(size_t n, cudaStream_t st) {
    if (n <= cap && p) return RHOSVD_OK;
    RH_CHECK(ensure(n, st));
    RH_CUDA(cudaMemsetAsync(p, 0, cap * sizeof(double), st));
    return RHOSVD_OK;
  }
};

// per-mode buffers of the eigensolver (S3-S5): the three modes run concurrently
struct ModeWs {
  DBuf Z, Y, M, T1;
  DBuf H, V, S, Bp, th, inv, tail2, sgn;
  DBuf W, X;
  Scratch gsc;
  DenseWs dws;
};
struct Workspace {
  DBuf Ustage, xistage;  // rhosvd_c2t_host: device copies of the host inputs
  DBuf Uh, s, tcol, xip, xip2, scal, part;
  DBuf G, W1x, W2x, corepart;
  DBuf alsK1, alsK2, alsT;  // C2T ALS: column blocks of K and of Uhat K
  Scratch gsc;
  ModeWs mw[3];
  int* flag = nullptr;
};
// Output buffers (frames, CP factors, sigma, core) outlive the call: the result handle
// owns them.  A freed handle returns them here (after a device synchronisation) and the
// next call takes the smallest cached buffer that fits, so a steady stream of same-size
// calls never grows the memory pool (growing it to hold a 2.2 GB core costs ~0.1 s).
struct OutCache {
  bool host = false;  // pinned host buffers (rhosvd_c2t_host outputs) instead of device memory
  std::mutex mu;
  std::multimap<size_t, void*> free_;
  std::map<void*, size_t> cap_;
  size_t cached = 0;
  int get(void** out, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    bytes = std::max<size_t>(bytes, 256);
    auto it = free_.lower_bound(bytes);
    if (it != free_.end() && it->first <= 2 * bytes + (1u << 20)) {
      *out = it->second;
      cached -= it->first;
      free_.erase(it);
      return RHOSVD_OK;
    }
    void* p = nullptr;
    cudaError_t e = alloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      // release everything cached and retry once
      for (auto& kv : free_) {
        release(kv.second);
        cap_.erase(kv.second);
      }
      free_.clear();
      cached = 0;
      e = alloc(&p, bytes);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(RHOSVD_ENOMEM, std::string("output alloc: ") + cudaGetErrorString(e));
      }
    }
    cap_[p] = bytes;
    *out = p;
    return RHOSVD_OK;
  }
  void put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cap_.find(p);
    if (it == cap_.end()) return;
    free_.emplace(it->second, p);
    cached += it->second;
    while (cached > ((size_t)16 << 30) && !free_.empty()) {  // bound the cache at 16 GiB
      auto big = std::prev(free_.end());
      cached -= big->first;
      cap_.erase(big->second);
      release(big->second);
      free_.erase(big);
    }
  }
  cudaError_t alloc(void** p, size_t bytes) {
    return host ? cudaHostAlloc(p, bytes, cudaHostAllocDefault) : cudaMalloc(p, bytes);
  }
  void release(void* p) { host ? cudaFreeHost(p) : cudaFree(p); }
};
static OutCache& OC() {
  static OutCache c;
  return c;
}
// pinned host outputs of rhosvd_c2t_host (pinning 2 GB costs ~1.5 s: keep them)
static OutCache& HC() {
  static OutCache* c = [] {
    auto* h = new OutCache();
    h->host = true;
    return h;
  }();
  return *c;
}

// RHOSVD_SERIAL_MODES=1 runs the three per-mode eigensolves one after another
static bool modes_concurrent() {
  static const bool on = [] {
    const char* e = getenv("RHOSVD_SERIAL_MODES");
    return !(e && e[0] == '1');
  }();
  return on;
}
// one non-blocking stream per mode (created once per device)
static cudaStream_t* mode_streams() {
  static std::mutex mu;
  static std::map<int, std::array<cudaStream_t, 3>> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    std::array<cudaStream_t, 3> a{};
    for (auto& x : a)
      if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    it = per_dev.emplace(dev, a).first;
  }
  return it->second.data();
}

// the H2D / D2H stream of rhosvd_c2t_host (created once per device)
static cudaStream_t copy_stream() {
  static std::mutex mu;
  static std::map<int, cudaStream_t> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    it = per_dev.emplace(dev, s).first;
  }
  return it->second;
}

// the stream the chunked beta all-reduce runs on (created once per device)
static cudaStream_t coll_stream() {
  static std::mutex mu;
  static std::map<int, cudaStream_t> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    it = per_dev.emplace(dev, s).first;
  }
  return it->second;
}

// host inputs of rhosvd_c2t_host
struct HostIn {
  const double* U[3];
  const double* xi;
};

static Workspace& WS() {
  static Workspace w;
  return w;
}
static std::mutex g_mu;
// Device-side order across entry points: g_mu serialises the host side, and every entry's
// stream also waits for the previous entry's device work (the workspaces, the GEMM
// scratch and its tile-schedule counters are process-wide), so calls made on different
// streams never overlap on the device.  Constructed under g_mu.
struct StreamOrder {
  cudaStream_t st;
  static cudaEvent_t& last() {
    static cudaEvent_t e = nullptr;
    return e;
  }
  explicit StreamOrder(cudaStream_t s) : st(s) {
    if (last()) cudaStreamWaitEvent(st, last(), 0);
  }
  ~StreamOrder() {
    if (!last()) cudaEventCreateWithFlags(&last(), cudaEventDisableTiming);
    cudaEventRecord(last(), st);
  }
};

// ------------------------------------------------------------------ phase timer
struct PhaseTimer {
  cudaStream_t st;
  std::vector<cudaEvent_t> ev;
  std::vector<int> phase;
  explicit PhaseTimer(cudaStream_t s) : st(s) {}
  void mark(int ph) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
    phase.push_back(ph);
  }
  // accumulate [mark i, mark i+1) into ms[phase[i]]
  void collect(double* ms) {
    cudaEventSynchronize(ev.back());
    for (size_t i = 0; i + 1 < ev.size(); ++i) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      if (phase[i] >= 0) ms[phase[i]] += t;
    }
    float tot = 0.f;
    cudaEventElapsedTime(&tot, ev.front(), ev.back());
    ms[8] = tot;
  }
  ~PhaseTimer() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};
enum { PH_NORM = 0, PH_GRAM = 1, PH_EIG = 2, PH_RR = 3, PH_RANK = 4, PH_PROJ = 5, PH_CORE = 6, PH_COMM = 7 };

// RHOSVD_TIMELINE=1: labelled events per mode, printed relative to the call's start
// (debug only; shows how the concurrent per-mode solves interleave on the device)
struct Timeline {
  bool on = false;
  std::mutex mu;
  cudaEvent_t origin = nullptr;
  struct E { int mode; const char* label; cudaEvent_t ev; };
  std::vector<E> evs;
  // host-side stamps (ms since begin): when the host got past a point
  std::chrono::steady_clock::time_point h0;
  std::vector<std::pair<double, std::string>> hs;
  void begin(cudaStream_t st) {
    const char* e = getenv("RHOSVD_TIMELINE");
    on = e && e[0] == '1';
    if (!on) return;
    cudaEventCreate(&origin);
    cudaEventRecord(origin, st);
    h0 = std::chrono::steady_clock::now();
  }
  void hmark(int mode, const char* label) {
    if (!on) return;
    const double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    std::lock_guard<std::mutex> lk(mu);
    hs.emplace_back(t, "mode " + std::to_string(mode) + "  " + label);
  }
  void mark(int mode, const char* label, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    std::lock_guard<std::mutex> lk(mu);
    evs.push_back({mode, label, e});
  }
  void dump() {
    if (!on) return;
    cudaDeviceSynchronize();
    for (auto& x : evs) {
      float t = 0.f;
      cudaEventElapsedTime(&t, origin, x.ev);
      fprintf(stderr, "[timeline] %9.3f ms  mode %2d  %s\n", t, x.mode, x.label);
      cudaEventDestroy(x.ev);
    }
    for (auto& x : hs) fprintf(stderr, "[timeline host] %9.3f ms  %s\n", x.first, x.second.c_str());
    hs.clear();
    evs.clear();
    cudaEventDestroy(origin);
    on = false;
  }
};
static Timeline& TL() {
  static Timeline t;
  return t;
}

// Collective scheduler for the concurrent per-mode eigensolves on a multi-rank
// communicator.  One communicator must not be driven by two threads, and the ranks must
// issue their collectives in the same order; so the mode threads post their all-reduces
// here and ONE comm thread executes them in a fixed round-robin order over the modes
// (mode 0's k-th, mode 1's k-th, mode 2's k-th, mode 0's (k+1)-th, ...; a finished mode
// is skipped).  Every rank runs the same deterministic sequence of collectives per mode
// (identical reduced inputs), so the global order is identical on all ranks.
static bool comm_trace() {
  static const bool on = [] {
    const char* e = getenv("RHOSVD_COMM_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

struct CommSched {
  rhosvd_comm* comm = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  struct Req {
    double* p = nullptr;
    int64_t count = 0;
    int root = -1;  // -1: sum all-reduce; >= 0: broadcast from this rank
    cudaStream_t st = nullptr;
    bool posted = false, done = false, finished = false;
    bool phase_done = false;  // this mode has posted every collective of the current phase
    int status = RHOSVD_OK;
    std::string err;
  } req[3];
  int dev = 0;
  // mode thread: run one all-reduce through the comm thread (blocks until done)
  int post(int mode, double* p, int64_t count, cudaStream_t st, int root = -1) {
    std::unique_lock<std::mutex> lk(mu);
    Req& r = req[mode];
    r.p = p; r.count = count; r.st = st; r.root = root; r.done = false; r.posted = true;
    cv.notify_all();
    cv.wait(lk, [&] { return r.done; });
    if (r.status != RHOSVD_OK) set_error(r.err);
    return r.status;
  }
  void finish(int mode) {
    std::lock_guard<std::mutex> lk(mu);
    req[mode].finished = true;
    cv.notify_all();
  }
  // Phase boundary (mode parallelism): a mode calls this once it has posted its last
  // collective before the final Jacobi, i.e. before it waits on the rank's Jacobi latch.
  // The comm thread skips such a mode until every mode has reached the boundary, then
  // resumes the round robin at mode 0.  Without it, modes with different numbers of
  // refinement all-reduces deadlock: the comm thread waits for the next post of a mode
  // whose thread waits on the latch for an owned Jacobi whose W W^T all-reduce comes later
  // in the round robin (r2end: fixed ranks (133, 31, 107), n = 589, R = 221, world 2).
  // The sequence stays a function of each mode's own program order, so it is identical on
  // all ranks.
  void phase_end(int mode) {
    std::lock_guard<std::mutex> lk(mu);
    req[mode].phase_done = true;
    cv.notify_all();
  }
  // comm thread
  void run() {
    cudaSetDevice(dev);
    int l = 0;
    std::unique_lock<std::mutex> lk(mu);
    while (true) {
      if (req[0].finished && req[1].finished && req[2].finished) break;
      Req& r = req[l];
      if (!r.finished) {
        cv.wait(lk, [&] { return r.posted || r.finished || r.phase_done; });
        if (r.phase_done) {
          // at the boundary: skipped until all modes are there (posts made after the
          // boundary wait for the reset), then the round robin restarts at mode 0
          bool all = true;
          for (int k = 0; k < 3; ++k) all = all && (req[k].finished || req[k].phase_done);
          if (all) {
            for (int k = 0; k < 3; ++k) req[k].phase_done = false;
            l = 0;
            continue;
          }
        } else if (r.posted) {
          r.posted = false;
          if (comm_trace()) fprintf(stderr, "[rhosvd comm exec] rank %d mode %d count %lld\n", comm->rank, l, (long long)r.count);
          lk.unlock();
          int s = r.root >= 0 ? comm_broadcast(comm, r.p, r.count, r.root, r.st)
                              : comm_allreduce(comm, r.p, r.count, r.st);
          std::string e = s != RHOSVD_OK ? std::string(rhosvd_last_error()) : std::string();
          lk.lock();
          r.status = s;
          r.err = e;
          r.done = true;
          cv.notify_all();
        }
      }
      l = (l + 1) % 3;
    }
  }
};

// Mode parallelism on a multi-rank communicator: the Gram-domain
// subspace iteration of mode l (S3: G only - no R-dependent data, no collective) runs on
// rank l mod p alone; its block Z (n x b) and the iteration state go to the other ranks by
// broadcast, and the R-sharded refinement / Rayleigh-Ritz / residual (S4) continue on all
// ranks.  Every rank first finishes the solves it owns (the latch), then posts its
// broadcasts: no NCCL kernel of this call waits on the device while an owned solve runs.
struct ModeLatch {
  std::mutex mu;
  std::condition_variable cv;
  int pending = 0;  // owned modes whose subspace iteration has not finished
  void done() {
    std::lock_guard<std::mutex> lk(mu);
    --pending;
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return pending <= 0; });
  }
};
struct MPar {
  bool owner = false;
  int root = 0;
  ModeLatch* latch = nullptr;   // subspace iterations (S3)
  ModeLatch* latch2 = nullptr;  // final Rayleigh-Ritz Jacobi (S4)
  int owned = 1;  // modes this rank owns
  bool signalled = false, signalled2 = false;
  void signal() {  // an owner's subspace iteration is over (once, on every path)
    if (owner && !signalled) {
      signalled = true;
      latch->done();
    }
  }
  void signal2() {  // an owner's Jacobi is over (once, on every path)
    if (owner && !signalled2) {
      signalled2 = true;
      latch2->done();
    }
  }
};

struct Ctx {
  cudaStream_t st;
  rhosvd_comm* comm;
  Workspace& w;
  rhosvd_report* rep;
  PhaseTimer* tm;
  double flops = 0.0;
  ModeWs* m = nullptr;  // per-mode buffers (S3-S5); GEMM scratch comes from here when set
  CommSched* sched = nullptr;  // concurrent modes on a multi-rank communicator
  int mode = 0;
  MPar* mp = nullptr;           // mode parallelism (multi-rank, concurrent modes)
};

__global__ void eye_kernel(double* Z, int64_t ldz, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) Z[(int64_t)i * ldz + i] = 1.0;
}

// ------------------------------------------------------------------ GEMM shorthands
// all matrices column-major; "n x b" buffers use ld = LDN
static int mm(Ctx& c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, bool ak, const double* B,
              int64_t ldb, bool bk, double* C, int64_t ldc, const double* cs = nullptr, bool upper = false,
              const double* rs = nullptr) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.a_k = ak; g.B = B; g.ldb = ldb; g.b_k = bk;
  g.C = C; g.ldc = ldc; g.col_scale = cs; g.row_scale = rs; g.upper_sym = upper;
  return gemm(g, c.m ? c.m->gsc : c.w.gsc, c.st, &c.flops);
}

static int allreduce(Ctx& c, double* p, int64_t count) {
  if (!c.comm || !c.comm->active()) return RHOSVD_OK;
  if (comm_trace()) fprintf(stderr, "[rhosvd comm] rank %d mode %d count %lld\n", c.comm->rank, c.m ? c.mode : -1, (long long)count);
  c.tm->mark(PH_COMM);
  if (c.sched) return c.sched->post(c.mode, p, count, c.st);
  return comm_allreduce(c.comm, p, count, c.st);
}
static int broadcast(Ctx& c, double* p, int64_t count, int root) {
  if (!c.comm || !c.comm->active()) return RHOSVD_OK;
  if (comm_trace()) fprintf(stderr, "[rhosvd comm] rank %d mode %d bcast root %d count %lld\n", c.comm->rank, c.mode, root, (long long)count);
  c.tm->mark(PH_COMM);
  if (c.sched) return c.sched->post(c.mode, p, count, c.st, root);
  return comm_broadcast(c.comm, p, count, root, c.st);
}

// RHOSVD_DEBUG=1: synchronise and scan a device array for non-finite values (debug only)
static bool dbg_on() {
  static const bool on = [] {
    const char* e = getenv("RHOSVD_DEBUG");
    return e && e[0] == '1';
  }();
  return on;
}
static void dbg_check(cudaStream_t st, const char* tag, const double* p, int64_t rows, int64_t cols, int64_t ld) {
  if (!dbg_on() || !p) return;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    fprintf(stderr, "[rhosvd dbg] %s: CUDA error %s\n", tag, cudaGetErrorString(e));
    return;
  }
  std::vector<double> h((size_t)ld * cols);
  cudaMemcpy(h.data(), p, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
  int64_t bad = 0, first = -1;
  double mx = 0.0;
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) {
      double v = h[(size_t)j * ld + i];
      if (!std::isfinite(v)) {
        if (first < 0) first = j * rows + i;
        ++bad;
      } else {
        mx = std::max(mx, std::fabs(v));
      }
    }
  fprintf(stderr, "[rhosvd dbg] %-28s %lldx%lld nonfinite=%lld first=%lld maxabs=%.3e\n", tag, (long long)rows,
          (long long)cols, (long long)bad, (long long)first, mx);
}

// CholeskyQR pass: dst = src * D L^{-T}, L = chol(D src^T src D + shift I)
static int cholqr_pass(Ctx& c, int64_t n, int64_t b, int64_t ldn, const double* src, double* dst, double shift,
                       int64_t ldb_small) {
  ModeWs& w = *c.m;
  RH_CHECK(mm(c, b, b, n, src, ldn, true, src, ldn, true, w.S.p, ldb_small, nullptr, true));
  dbg_check(c.st, "chol S", w.S.p, b, b, ldb_small);
  RH_CHECK(chol_inv_scaled(b, w.S.p, ldb_small, shift, w.Bp.p, ldb_small, w.dws, c.st));
  dbg_check(c.st, "chol Bp", w.Bp.p, b, b, ldb_small);
  RH_CHECK(mm(c, n, b, b, src, ldn, false, w.Bp.p, ldb_small, true, dst, ldn));
  return RHOSVD_OK;
}
// orthonormalize M (n x b) into Z: shifted CholQR (robust to rank deficiency) + CholQR2.
// buffers: in -> out, uses tmp.
// Orthonormalisation flavours:
//   ORTH_CQR2     CholeskyQR2 (two passes): orthonormal to ~u for well conditioned input
//   ORTH_SCQR3    shifted CholeskyQR3 (Fukaya et al.): robust to kappa up to ~u^{-1}
//   ORTH_CQR1     one pass: a well conditioned (not exactly orthonormal) basis - enough
//                 inside the subspace iteration, whose next step re-orthonormalises
//   ORTH_SCQR1    one shifted pass: the same for badly conditioned input
//   ORTH_SCQR2    shifted pass + one plain pass: orthonormal to ~u kappa(Q1)^2 (kappa of the
//                 shifted pass's output is small), enough for the subspace iteration
enum { ORTH_CQR2 = 0, ORTH_SCQR3 = 1, ORTH_CQR1 = 2, ORTH_SCQR1 = 3, ORTH_SCQR2 = 4 };
static int orth(Ctx& c, int64_t n, int64_t b, int64_t ldn, const double* in, double* out, double* tmp,
                int64_t ldb_small, int kind) {
  const double u = 1.1102230246251565e-16;
  // shift s = 11 (n b + b(b+1)) u ||X||_2^2 with ||X||_2^2 <= b for the column-scaled X
  const double shift = 11.0 * ((double)n * b + (double)b * (b + 1)) * u * (double)b;
  switch (kind) {
    case ORTH_CQR1:
      return cholqr_pass(c, n, b, ldn, in, out, 0.0, ldb_small);
    case ORTH_SCQR1:
      return cholqr_pass(c, n, b, ldn, in, out, shift, ldb_small);
    case ORTH_SCQR2:
      RH_CHECK(cholqr_pass(c, n, b, ldn, in, tmp, shift, ldb_small));
      return cholqr_pass(c, n, b, ldn, tmp, out, 0.0, ldb_small);
    case ORTH_CQR2:
      RH_CHECK(cholqr_pass(c, n, b, ldn, in, tmp, 0.0, ldb_small));
      return cholqr_pass(c, n, b, ldn, tmp, out, 0.0, ldb_small);
    default:
      RH_CHECK(cholqr_pass(c, n, b, ldn, in, tmp, shift, ldb_small));
      RH_CHECK(cholqr_pass(c, n, b, ldn, tmp, out, 0.0, ldb_small));
      RH_CHECK(cholqr_pass(c, n, b, ldn, out, tmp, 0.0, ldb_small));
      RH_CUDA(cudaMemcpyAsync(out, tmp, (size_t)ldn * b * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
      return RHOSVD_OK;
  }
}

struct ModeOut {
  int r = 0, b = 0, iters = 0, grows = 0, refines = 0;
  double T = 0, tail2 = 0, rho = 0;
  double* Z = nullptr;      // n x r (ld LDN), owned by result
  double* sigma = nullptr;  // r
  double* W = nullptr;      // r x Rp row-major, owned by result
};

// eigensolver + one-sided RR + refinement + rank + projection for one mode
static int solve_mode(Ctx& c, int mode, int64_t n, int64_t LDN, int64_t Rl, int64_t Rp, int64_t Rg,
                      const double* Uh, const double* G, double T, const rhosvd_opts& o, ModeOut& mo) {
  ModeWs& w = *c.m;
  double* const scal = c.w.scal.p;  // shared scalar slots (mode-offset)
  cudaStream_t st = c.st;
  const int64_t m = std::min<int64_t>(n, Rg);
  const bool epsmode = o.rank_mode == RHOSVD_EPS;
  const int64_t rfix = epsmode ? 0 : std::min<int64_t>(o.r[mode], m);
  const int p = std::max(1, o.oversample);
  // eps mode: first block block0 (<= 0: 128); it grows adaptively.  (Starting at n/4 saves
  // growth restarts but leaves the trailing Rayleigh quotients too rough to truncate the
  // block before the non-squared steps: cfg 3/5 got slower.)
  const int64_t b0 = o.block0 > 0 ? o.block0 : 128;
  int64_t b = epsmode ? std::min<int64_t>(m, std::max<int64_t>(b0, 2 * p)) : std::min<int64_t>(m, rfix + p);
  const double u = 1.1102230246251565e-16;
  const double tau = 1e-13;  // Ritz-value floor relative to theta_1
  mo.T = T;

  // n x b work buffers sized for the largest possible block m = min(n, R) once, so
  // block growth keeps their contents; the b x R buffers grow on demand.  A fixed-rank call
  // with R < n <= 2048 may take the full-space path below with b = n > m.
  const int64_t mws = n <= 2048 ? std::max(n, m) : m;
  RH_CHECK(w.Z.ensure((size_t)LDN * mws + 64, st));
  RH_CHECK(w.Y.ensure((size_t)LDN * mws + 64, st));
  RH_CHECK(w.M.ensure((size_t)LDN * mws + 64, st));
  RH_CHECK(w.T1.ensure((size_t)LDN * mws + 64, st));
  {
    int64_t ldm = round_up(std::max<int64_t>(mws, 2), 2);
    for (DBuf* d : {&w.H, &w.V, &w.S, &w.Bp}) RH_CHECK(d->ensure((size_t)ldm * mws + 64, st));
    for (DBuf* d : {&w.th, &w.inv, &w.tail2, &w.sgn}) RH_CHECK(d->ensure((size_t)mws + 64, st));
  }
  auto ensure_b = [&](int64_t bb) -> int {
    RH_CHECK(w.W.ensure((size_t)bb * Rp, st));
    RH_CHECK(w.X.ensure((size_t)bb * Rp, st));
    return RHOSVD_OK;
  };
  auto ldbs = [&](int64_t bb) { return round_up(std::max<int64_t>(bb, 2), 2); };

  RH_CHECK(ensure_b(b));
  uint64_t seed = o.seed * 0x9E3779B97F4A7C15ull + (uint64_t)(mode + 1) * 0xD1B54A32D192ED03ull;

  // ---------------- subspace (simultaneous) iteration Z <- CholQR(G Z), block growth.
  // CholQR keeps leading spans, so span(z_1..z_j) converges to the dominant j-space for
  // every j (rate lambda_{b+1}/lambda_j) and the columns align with the eigenvectors
  // except inside clusters: Z^T G Z tends to (nearly) diagonal, which is what makes the
  // two Jacobi eigensolves below cheap.  The diagonal d_k = z_k^T G z_k (cheap column
  // dots) gives the running tail estimate T - sum_{k<=r} d_k (>= the true tail) for the
  // block-size decision (eps mode) and the rate estimate d_b / d_r for the iteration count.
  std::vector<double> d_h;
  const double thr = epsmode ? o.eps * o.eps * T : 0.0;
  auto predict_r = [&](const std::vector<double>& d, int64_t bb) -> int64_t {
    double acc = 0.0;
    std::vector<double> tc(bb);
    for (int64_t k = 0; k < bb; ++k) {
      acc += d[k];
      tc[k] = T - acc;
      if (tc[k] <= thr) return k + 1;
    }
    // not reached inside the block: extrapolate log10(tail) linearly over the last half
    int64_t j0 = bb / 2;
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    int64_t cnt = 0;
    for (int64_t k = j0; k < bb; ++k) {
      double y = std::log10(std::max(tc[k], 1e-300));
      double x = (double)(k + 1);
      sx += x; sy += y; sxx += x * x; sxy += x * y;
      ++cnt;
    }
    double den = cnt * sxx - sx * sx;
    if (cnt < 2 || den <= 0) return 2 * bb;
    double slope = (cnt * sxy - sx * sy) / den, icpt = (sy - slope * sx) / cnt;
    if (!(slope < 0)) return 2 * bb;
    double rr = (std::log10(thr) - icpt) / slope;
    if (!(rr < 1e9)) return 2 * bb;
    return (int64_t)std::ceil(rr);
  };
  int it_total = 0, itb = 0, guard = 0;
  int need_last = 0;     // modelled iteration count of the last convergence test
  bool capped = false;   // the last block stopped at max_iters before need_last
  int64_t r_est = rfix;
  auto subspace_iteration = [&]() -> int {
  // random start block (Gaussian columns; the first step's G Omega is orthonormalised)
  RH_CHECK(k_random(w.Z.p, LDN, n, 0, b, seed, st));
  while (true) {
    ++it_total;
    ++itb;
    RH_CHECK(mm(c, n, b, n, G, LDN, false, w.Z.p, LDN, true, w.Y.p, LDN));
    RH_CHECK(k_coldot(w.Z.p, w.Y.p, LDN, n, b, w.th.p, st));
    // the first steps after a (re)start see badly conditioned G Z: shifted pass + plain
    // pass; later steps (aligned Z, well conditioned G Z) one plain pass.  The estimates
    // d_k are always taken on a Z produced by at least two passes or by one pass on a
    // well conditioned input.
    RH_CHECK(orth(c, n, b, LDN, w.Y.p, w.Z.p, w.T1.p, ldbs(b), itb <= 2 ? ORTH_SCQR2 : ORTH_CQR1));
    TL().mark(mode, "iteration", st);
    dbg_check(st, "it Z=orth(GZ)", w.Z.p, n, b, LDN);
    if (b >= m) break;  // full space: exact after one step
    if (itb < 2) continue;
    d_h.resize(b);
    RH_CHECK(d2h_wait(d_h.data(), w.th.p, b * sizeof(double), st));
    if (epsmode) r_est = predict_r(d_h, b);
    if (epsmode && r_est + p > b && guard < 12) {
      // grow towards the predicted size, at most 2x per event (the log-linear tail
      // extrapolation of a small block overshoots: 128 -> r_est 1093 on cfg 4)
      // (RHOSVD_GROW_MAX: the per-event growth factor cap, default 2.  A 4x first step on
      // cfg 4 (128 -> 512, two iterations fewer) measured no faster (r2p: 105.9 vs 103.9 ms
      // eigensolve) and cost cfg 2 (m = 512) a full-space block (r2h), so it stays 2.)
      static const int grow_max = [] {
        const char* e = getenv("RHOSVD_GROW_MAX");
        return e ? std::max(2, atoi(e)) : 2;
      }();
      int64_t bn = std::min<int64_t>(m, std::min<int64_t>((int64_t)grow_max * b,
                                                           std::max<int64_t>((int64_t)(1.15 * r_est) + p, b + p)));
      // stay on the one-CTA Cholesky (b <= 160) when the prediction leaves room there
      // (cfg 3: r_est 134 -> 170 would put every later CholQR on the cooperative kernel)
      if (bn > 160 && b < 160 && r_est + p + 8 <= 160) bn = 160;
      if (dbg_on()) fprintf(stderr, "[rhosvd dbg] mode %d grow b %lld -> %lld (r_est %lld)\n", mode, (long long)b, (long long)bn, (long long)r_est);
      RH_CHECK(ensure_b(bn));
      RH_CHECK(k_random(w.Z.p, LDN, n, b, bn, seed + 7919ull * (uint64_t)(it_total + 1), st));
      b = bn;
      itb = 0;
      ++mo.grows;
      ++guard;
      continue;
    }
    // iterations for sin(theta_r) ~ 1e-7: rate d_b / d_r (d_b over-estimates lambda_{b+1})
    const int64_t rr = std::max<int64_t>(1, std::min<int64_t>(r_est, b));
    const double dr = std::max(d_h[rr - 1], 1e-300);
    const double rho = std::min(0.999, std::max(d_h[b - 1], 1e-300 * dr) / dr);
    const int need = std::max(2, (int)std::ceil(std::log(1e-7) / std::log(rho)));
    const int cap = std::max(2, o.max_iters);
    // fixed rank: no block truncation follows (eps mode cuts the block where d_b <= 0.003 d_r,
    // so each refinement step contracts the angle by <= 0.003), and one refinement step at
    // rate rho leaves sin(theta_r) ~ 1e-7 rho: r2zz sweep case 34, r = 21 at rho 0.31 gave a
    // 5e-8 tilt and the Tucker tensor 1.6e-9 off.  The Gram-domain iteration is the cheap
    // part here (n x n x b), so it continues, within max_iters, to sin(theta_r) ~ 1e-12
    // (its floor u d_1 / (d_r - d_b) is far below that unless the cut is a near-tie); the
    // ENOCONV rule keeps the 1e-7 count.  RHOSVD_FIXED_ANGLE=0 restores the 1e-7 target.
    static const int fixed_angle = [] {
      const char* e = getenv("RHOSVD_FIXED_ANGLE");
      return e ? atoi(e) : 1;
    }();
    const int need_it = (!epsmode && fixed_angle)
                            ? std::max(need, (int)std::ceil(std::log(1e-12) / std::log(rho)))
                            : need;
    if (itb >= std::min(need_it, cap)) {
      need_last = need;
      capped = need > cap;
      break;
    }
  }
  return RHOSVD_OK;
  };
  if (!c.mp) {
    RH_CHECK(subspace_iteration());
  } else {
    // mode parallelism: the owner iterates; then (after every solve this rank owns) the
    // state header [status, b, r_est, itb, it_total, grows, need_last, capped, d_1..d_b]
    // and the block Z go out by broadcast.  A failed owner still broadcasts its status, so
    // every rank returns the same error instead of waiting for a Z that never comes.
    int st_a = RHOSVD_OK;
    std::string err_a;
    if (c.mp->owner) {
      // the rank's owned iterations share the GPU (p >= 3: one mode with every SM), as the
      // final Jacobi below does; the non-owned modes only wait here
      const int cap_saved = g_coop_cap;
      g_coop_cap = std::max(1, num_sms() / std::max(1, c.mp->owned));
      st_a = subspace_iteration();
      g_coop_cap = cap_saved;
      if (st_a != RHOSVD_OK) err_a = g_err;
      c.mp->signal();
    }
    c.mp->latch->wait();
    const int64_t hn = 8 + m;
    RH_CHECK(w.H.ensure((size_t)std::max<int64_t>(hn, round_up(std::max<int64_t>(m, 2), 2) * m) + 64, st));
    std::vector<double> hdr(hn, 0.0);
    if (c.mp->owner) {
      hdr[0] = st_a; hdr[1] = (double)b; hdr[2] = (double)r_est; hdr[3] = itb; hdr[4] = it_total;
      hdr[5] = mo.grows; hdr[6] = need_last; hdr[7] = capped ? 1.0 : 0.0;
      for (size_t k = 0; k < d_h.size() && (int64_t)k < m; ++k) hdr[8 + k] = d_h[k];
      RH_CHECK(h2d_wait(w.H.p, hdr.data(), hn * sizeof(double), st));
    }
    RH_CHECK(broadcast(c, w.H.p, hn, c.mp->root));
    RH_CHECK(d2h_wait(hdr.data(), w.H.p, hn * sizeof(double), st));
    if ((int)hdr[0] != RHOSVD_OK)
      return fail((int)hdr[0], c.mp->owner ? err_a : "mode " + std::to_string(mode) + ": owner rank failed");
    b = (int64_t)hdr[1]; r_est = (int64_t)hdr[2]; itb = (int)hdr[3]; it_total = (int)hdr[4];
    mo.grows = (int)hdr[5]; need_last = (int)hdr[6]; capped = hdr[7] != 0.0;
    d_h.assign(hdr.begin() + 8, hdr.begin() + 8 + std::min<int64_t>(b, m));
    if (b >= m) d_h.clear();  // full space: the owner kept no estimates
    RH_CHECK(ensure_b(b));
    RH_CHECK(broadcast(c, w.Z.p, LDN * b, c.mp->root));
  }
  mo.iters = it_total;
  // block truncation: smallest b' >= r + p with d_b' <= 0.003 d_r (leading columns carry
  // the dominant subspaces).  The ratio bounds the refinement contraction rho below:
  // 0.003 gives rho^2 <= 1e-5 per step, so on cfg 4 ONE refinement step passes the
  // a-posteriori test (blocks 723-732 -> 762-767 columns, eigensolve 126 -> 105 ms, sigma
  // still within 1.7e-12 of the oracle; at 0.02 it needed two steps of ~286 GFLOP per mode;
  // r2n, profiles/r2n_trunc_ratio_sweep.log).
  static const double trunc_ratio = [] {
    const char* e = getenv("RHOSVD_TRUNC_RATIO");
    return e ? atof(e) : 0.003;
  }();
  if (!d_h.empty() && r_est > 0 && r_est + p < b) {
    const double tr = d_h[r_est - 1];
    for (int64_t j = r_est + p; j <= b; ++j)
      if (d_h[j - 1] <= trunc_ratio * tr) {
        b = j;
        break;
      }
  }
  c.tm->mark(PH_RR);

  // ---------------- one-sided Rayleigh-Ritz + non-squared refinement + final RR
  // Full-space final Rayleigh-Ritz (see the Z = I comment below): taken when the block grew
  // to all of R^n (m = n), and for a fixed rank whose sigma_r lies below what the squared
  // Rayleigh-Ritz resolves (Gram-domain d_r < 1e-10 d_1, i.e. sigma_r < 1e-5 sigma_1 - the
  // Gram-domain d overstates such lambda up to 5000x; below ~1e-7 sigma_1 the refined block's
  // sigma are rounding noise: r2h sweep cases 13 / 19 / 25 / 37, seed-7 case 4),
  // there up to n = 2048 (two b x b Jacobis on the full space).
  static const int full_eye_env = [] {
    const char* e = getenv("RHOSVD_FULL_EYE");
    return e ? atoi(e) : 1;
  }();
  bool full_eye = full_eye_env && m == n && n > 1 && b >= m;
  // eps mode, R < n, and the block grew to the whole column space (b = m = R): the same
  // basis with b = n > m (seeds 17 / 23 sweep cases: frames off the 1e-13 orthonormality bound)
  if (full_eye_env == 1 && !full_eye && epsmode && m < n && n > 1 && n <= 2048 && b >= m) {
    full_eye = true;
    b = n;
    d_h.resize(b, 0.0);
    RH_CHECK(ensure_b(b));
  }
  // R < n (m = R): Z = I is still an exact orthonormal basis of a space that holds the
  // column space of Uhat, so the same path applies with b = n > m - W = Uhat, W W^T = G of
  // rank <= R, its n - R null directions sort last (seed-7 sweep case 10, seed-11 case 38).
  // RHOSVD_FULL_EYE=2 restricts the fixed-rank trigger to m = n as before.
  if (full_eye_env && (m == n || full_eye_env != 2) && n > 1 && !full_eye && !epsmode && n <= 2048 && rfix > 0 &&
      (int64_t)d_h.size() >= rfix && !(d_h[rfix - 1] >= 1e-10 * d_h[0])) {
    full_eye = true;
    b = n;
    d_h.resize(b, 0.0);  // host arrays below are indexed by the block size
    RH_CHECK(ensure_b(b));
  }
  const int64_t ldb = ldbs(b);

  // Non-squared refinement: Z <- CholQR2(Uhat (Z^T Uhat)^T) = CholQR2(G Z)
  // evaluated without G, so the subspace error contracts below the squared-Gram floor.
  // The Gram-domain iteration left Z aligned with the eigenvectors (simultaneous
  // iteration), so G Z is well conditioned after column scaling and no Rayleigh-Ritz is
  // needed between steps.  Step count from the error model (columns rotate inside
  // clusters, so per-column changes cannot serve as a stopping test):
  //   Gram-domain floor (relative, on lambda_r = sigma_r^2)  e0 = 10 u d_1 / d_r,
  //   contraction per step                                    rho^2 = (d_b / d_r)^2,
  //   steps = ceil(log(1e-11 / e0) / log(rho^2)), clamped to [refine_steps, refine_steps + 1]
  // (1e-11 on lambda is 5e-12 on sigma, 20x inside the 1e-10 parity bound).
  int nref = 0;
  if (o.refine_steps > 0) {
    nref = o.refine_steps + 1;
    if (!d_h.empty() && r_est > 0) {
      const int64_t rr = std::min<int64_t>(r_est, b);
      const double dr = std::max(d_h[rr - 1], 1e-300), d1 = std::max(d_h[0], dr);
      const double e0 = 10.0 * u * d1 / dr;
      // d_b below the Gram-domain noise (~u d_1) says nothing about lambda_{b+1}: floor it
      const double rho = std::min(0.9, std::max(d_h[b - 1], 64.0 * u * d1) / dr);
      int need = e0 <= 1e-11 ? 0 : (int)std::ceil(std::log(1e-11 / e0) / std::log(rho * rho));
      // at most one step beyond refine_steps: measured (r2d, tools/refine_probe.py) the
      // retained sigma are within 3.3e-12 (cfg 3, 5) and 1.7e-12 (cfg 4) of the oracle after
      // two steps, and the model's third step on cfg 3 mode 0 bought nothing
      nref = std::max(o.refine_steps, std::min(need, o.refine_steps + 1));
      // RHOSVD_REFINE_MAX (probe knob): cap the modelled step count (>= refine_steps)
      static const int refine_cap = [] {
        const char* e = getenv("RHOSVD_REFINE_MAX");
        return e ? atoi(e) : 0;
      }();
      if (refine_cap > 0) nref = std::max(o.refine_steps, std::min(nref, refine_cap));
      if (dbg_on())
        fprintf(stderr, "[rhosvd dbg] mode %d refine model e0 %.2e rho %.3e -> %d steps\n", mode, e0, rho, nref);
    }
  }
  // ENOCONV: the iteration cap stopped the subspace iteration before its
  // modelled count, and the refinement steps (each contracts the subspace error by the
  // same rate) cannot make up the difference: sin(theta_r) ~ rho^(itb + nref) > 1e-7.
  // Full space with m = n <= R (the block grew to all of R^n): every orthonormal basis spans
  // it, so the exact one is taken, Z = I, and the non-squared refinement (pointless on the
  // full space) is skipped.  Refining there runs CholQR2 on U W^T, whose columns span
  // lambda_b / lambda_1 ~ 1e-28: the noise columns come out of the dependent-column rule
  // not orthonormal to the rest, and the kept subspace tilted by ~1e-8 although sigma is
  // right (r2zz, tools/case_probe.py 99 20: Tucker tensor 3e-10 / 2.6e-9 off the oracle's,
  // varying from call to call).  The final Rayleigh-Ritz then runs twice (below): W = U,
  // W W^T = G by Jacobi gives P to the squared accuracy; on the rotated rows P^T U, which
  // are orthogonal to that accuracy, the second Jacobi is accurate relative to each entry
  // (Demmel-Veselic), so sigma and the cut subspace come out non-squared.
  // RHOSVD_FULL_EYE=0 restores the refined full-space block.
  if (full_eye) {
    RH_CUDA(cudaMemsetAsync(w.Z.p, 0, (size_t)LDN * b * sizeof(double), st));
    eye_kernel<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(w.Z.p, LDN, (int)n);
    count_launch();
    RH_LAUNCH_CHECK();
    nref = 0;
    if (dbg_on()) fprintf(stderr, "[rhosvd dbg] mode %d full space: Z = I, two Rayleigh-Ritz passes\n", mode);
  }
  if (!full_eye && capped && itb + nref < need_last)
    return fail(RHOSVD_ENOCONV, "mode " + std::to_string(mode) + ": subspace iteration hit max_iters (" +
                                    std::to_string(o.max_iters) + ") with " + std::to_string(need_last) +
                                    " iterations needed for the block edge rate");
  for (int rs = 0;; ++rs) {
    // W = Z^T Uhat (b x Rp row-major == Rl x b col-major)
    RH_CHECK(mm(c, Rl, b, n, Uh, LDN, true, w.Z.p, LDN, true, w.W.p, Rp));
    TL().mark(mode, "W = Z^T Uhat", st);
    if (rs >= nref) break;
    // M = Uhat W^T (summed over the R shards), Z <- CholQR2(M)
    RH_CHECK(mm(c, n, b, Rl, Uh, LDN, false, w.W.p, Rp, true, w.M.p, LDN));
    TL().mark(mode, "M = Uhat W^T", st);
    RH_CHECK(allreduce(c, w.M.p, LDN * b));
    // A-posteriori stopping test before the last modelled step (default on;
    // RHOSVD_REFINE_ADAPT=0 runs the modelled count): the Rayleigh-Ritz residual of the current block,
    // R = M - Z (Z^T M) = (I - Z Z^T) G Z (non-squared: M came from Uhat), gives the
    // subspace angle of column j as ||r_j|| / c_jj (c = Z^T M); the step about to be taken
    // contracts it by rho_j = c_bb / c_jj, and the final Ritz value errs by about its
    // square:  e = max_{j <= r} (rho_j ||r_j|| / c_jj)^2.  If e is already below the
    // target, this is the last step.  Costs two b x b x n GEMMs per test.
    // Measured (r2i, tools/refine_probe.py): after step 1 the estimate is 6e-16 - 1.9e-12
    // on cfg 3 / 5 (one step suffices: sigma within 3.4e-12 of the oracle) and 1e-10 -
    // 2e-10 on cfg 4 (two steps: 1.7e-12; one step would leave 2.9e-11).
    static const int adapt = [] {
      const char* e = getenv("RHOSVD_REFINE_ADAPT");
      return e ? atoi(e) : 1;
    }();
    if (((adapt && rs + 1 < nref) || dbg_on()) && b > 1) {
      const int64_t ldb2 = ldbs(b);
      RH_CHECK(mm(c, b, b, n, w.Z.p, LDN, true, w.M.p, LDN, true, w.S.p, ldb2));  // C = Z^T M
      RH_CUDA(cudaMemcpyAsync(w.T1.p, w.M.p, (size_t)LDN * b * sizeof(double), cudaMemcpyDeviceToDevice, st));
      GemmArgs gr;
      gr.M = n; gr.N = b; gr.K = b; gr.A = w.Z.p; gr.lda = LDN; gr.a_k = false; gr.B = w.S.p; gr.ldb = ldb2;
      gr.b_k = true; gr.C = w.T1.p; gr.ldc = LDN; gr.alpha = -1.0; gr.beta = 1.0;
      RH_CHECK(gemm(gr, w.gsc, st, &c.flops));                                          // R = M - Z C
      RH_CHECK(k_coldot(w.T1.p, w.T1.p, LDN, n, b, w.inv.p, st));                       // ||r_j||^2
      RH_CHECK(k_coldot(w.Z.p, w.M.p, LDN, n, b, w.tail2.p, st));                       // c_jj
      std::vector<double> rn(b), cd(b);
      RH_CHECK(d2h_wait(rn.data(), w.inv.p, b * sizeof(double), st));
      RH_CHECK(d2h_wait(cd.data(), w.tail2.p, b * sizeof(double), st));
      const int64_t jr = std::max<int64_t>(1, std::min<int64_t>(r_est > 0 ? r_est : b, b));
      double est = 0.0;
      for (int64_t j = 0; j < jr; ++j) {
        const double cj = std::max(cd[j], 1e-300), rho = std::min(1.0, std::max(cd[b - 1], 0.0) / cj);
        est = std::max(est, rho * rho * std::max(rn[j], 0.0) / (cj * cj));
      }
      if (dbg_on())
        fprintf(stderr, "[rhosvd dbg] mode %d refine step %d: a-posteriori estimate %.3e (steps planned %d)\n", mode,
                rs + 1, est, nref);
      // the estimate is meaningful only while lambda_b / lambda_1 (here the smallest
      // non-squared Rayleigh quotient c_jj of the block) stays above the squared floor,
      // ~2u: below it one non-squared step can leave sigma_r off by ~1e-6 although the
      // estimate reads 1e-12 (r2g: n = 257, R = 2300, eps = 1e-8, kappa_r 6.5e7, ratio
      // 2.8e-17 after step 1: sigma 3e-6 off after one step, 4.5e-10 after two; the
      // Gram-domain d_r overstates such lambda_r 5000x, so d_h cannot tell), and the planned
      // steps run.  BJ configs after step 1: 1.7e-15 (cfg 3 / 5) ... 1.1e-13 (cfg 4).
      double lam_ratio = 1.0;
      for (int64_t j = 0; j < b; ++j) lam_ratio = std::min(lam_ratio, std::max(cd[j], 0.0) / std::max(cd[0], 1e-300));
      if (dbg_on()) fprintf(stderr, "[rhosvd dbg] mode %d refine step %d: lambda_b / lambda_1 %.3e\n", mode, rs + 1, lam_ratio);
      if (adapt && est <= 1e-11 && rs + 1 < nref && lam_ratio >= 2.0 * u) nref = rs + 1;
    }
    RH_CHECK(orth(c, n, b, LDN, w.M.p, w.Z.p, w.T1.p, ldb, ORTH_CQR2));
    TL().mark(mode, "refine CholQR2", st);
    ++mo.refines;
    c.tm->mark(PH_RR);
  }
  // Final one-sided Rayleigh-Ritz, residual and rank.  The rank rule must be met inside
  // the block (rho = ||Uhat - Z_b W_b||^2 is the out-of-block energy, ~1e-7 on cfg 4
  // against eps^2 T = 4.8e-6): a miss means the block or the subspace did not converge,
  // and the call fails with ENOCONV instead of returning a rank that violates the rule.
  double sel[4];
  double rho_h = 0.0;
  static const int rr_passes_env = [] {
    const char* e = getenv("RHOSVD_RR_PASSES");
    return e ? std::max(1, std::min(atoi(e), 3)) : 1;
  }();
  // (mode parallelism: the first pass's Jacobi runs on the mode's owner rank and is
  // broadcast; a second pass runs replicated - the Jacobi is bitwise independent of its grid)
  for (int rr_pass = 0; rr_pass < (full_eye ? std::max(2, rr_passes_env) : (c.mp ? 1 : rr_passes_env)); ++rr_pass) {
    if (rr_pass > 0) {
      // second Rayleigh-Ritz pass: rotate the basis by the first pass's eigenvectors
      // (Z <- Z P, W <- P^T W, so Z W is unchanged) and solve W W^T again; its rows are now
      // nearly orthogonal, so forming W W^T loses only u |w_i| |w_j| per entry
      RH_CHECK(mm(c, n, b, b, w.Z.p, LDN, false, w.V.p, ldb, true, w.M.p, LDN));
      RH_CHECK(mm(c, Rl, b, b, w.W.p, Rp, false, w.V.p, ldb, true, w.X.p, Rp));
      RH_CUDA(cudaMemcpy2DAsync(w.Z.p, LDN * sizeof(double), w.M.p, LDN * sizeof(double), n * sizeof(double), b,
                                cudaMemcpyDeviceToDevice, st));
      RH_CUDA(cudaMemcpy2DAsync(w.W.p, Rp * sizeof(double), w.X.p, Rp * sizeof(double), Rl * sizeof(double), b,
                                cudaMemcpyDeviceToDevice, st));
    }
    // W W^T = P Lambda P^T (high relative accuracy Jacobi)
    RH_CHECK(mm(c, b, b, Rl, w.W.p, Rp, true, w.W.p, Rp, true, w.S.p, ldb, nullptr, true));
    RH_CHECK(allreduce(c, w.S.p, ldb * b));
    TL().mark(mode, "W W^T", st);
    c.tm->mark(PH_RR);
    if (!c.mp || rr_pass > 0) {
      int sw = 0;
      RH_CHECK(syevj(b, w.S.p, ldb, w.th.p, w.V.p, ldb, 1e-15, 1e-300, 80, w.dws, st, &sw));
      if (dbg_on()) fprintf(stderr, "[rhosvd dbg] mode %d rr b %lld sweeps %d\n", mode, (long long)b, sw);
      if (sw < 0) return fail(RHOSVD_ENOCONV, "Jacobi on W W^T did not converge");
      TL().mark(mode, "Jacobi", st);
    } else {
      // mode parallelism: the b x b Jacobi of mode l (replicated input after the all-reduce)
      // runs on its owner rank with the whole GPU; [status, sweeps], the eigenvalues and the
      // eigenvectors go out by broadcast once every Jacobi this rank owns has finished
      int st_j = RHOSVD_OK, sw = 0;
      std::string err_j;
      if (c.sched) c.sched->phase_end(mode);  // last collective before the Jacobi latch
      if (c.mp->owner) {
        // the rank's owned Jacobis share the GPU (p >= 3: one Jacobi with every SM)
        const int cap_saved = g_coop_cap;
        g_coop_cap = std::max(1, num_sms() / std::max(1, c.mp->owned));
        st_j = syevj(b, w.S.p, ldb, w.th.p, w.V.p, ldb, 1e-15, 1e-300, 80, w.dws, st, &sw);
        g_coop_cap = cap_saved;
        if (st_j != RHOSVD_OK) err_j = g_err;
        else if (sw < 0) st_j = RHOSVD_ENOCONV, err_j = "Jacobi on W W^T did not converge";
        c.mp->signal2();
      }
      c.mp->latch2->wait();
      double h2[2] = {(double)st_j, (double)sw};
      if (c.mp->owner) RH_CHECK(h2d_wait(w.H.p, h2, sizeof(h2), st));
      RH_CHECK(broadcast(c, w.H.p, 2, c.mp->root));
      RH_CHECK(d2h_wait(h2, w.H.p, sizeof(h2), st));
      if ((int)h2[0] != RHOSVD_OK)
        return fail((int)h2[0], c.mp->owner ? err_j : "mode " + std::to_string(mode) + ": owner rank's Jacobi failed");
      RH_CHECK(broadcast(c, w.th.p, b, c.mp->root));
      RH_CHECK(broadcast(c, w.V.p, ldb * b, c.mp->root));
      if (dbg_on()) fprintf(stderr, "[rhosvd dbg] mode %d rr b %lld sweeps %d (rank %d)\n", mode, (long long)b, (int)h2[1], c.mp->root);
      TL().mark(mode, "Jacobi", st);
    }
  }
  {
    c.tm->mark(PH_RANK);
    // rho = ||Uhat - Z W||_F^2 (fused residual epilogue; E never stored)
    {
      GemmArgs g;
      g.M = n; g.N = Rl; g.K = b; g.A = w.Z.p; g.lda = LDN; g.a_k = false; g.B = w.W.p; g.ldb = Rp; g.b_k = false;
      g.epi = EPI_RESID; g.D = Uh; g.ldd = LDN; g.resid_out = scal + 16 + mode;
      if (Rl > 0) {
        RH_CHECK(gemm(g, w.gsc, st, &c.flops));
      } else {
        RH_CUDA(cudaMemsetAsync(scal + 16 + mode, 0, sizeof(double), st));
      }
      RH_CHECK(allreduce(c, scal + 16 + mode, 1));
      TL().mark(mode, "residual", st);
      c.tm->mark(PH_RANK);
    }
    RH_CHECK(k_select_rank(w.th.p, b, scal + 16 + mode, T, epsmode ? o.eps : 0.0, (int)rfix, 8, w.tail2.p,
                           scal + 24 + 4 * mode, w.inv.p, st));
    RH_CHECK(d2h_wait(sel, scal + 24 + 4 * mode, 3 * sizeof(double), st));
    RH_CHECK(d2h_wait(&rho_h, scal + 16 + mode, sizeof(double), st));
    TL().hmark(mode, "rank selected");
  }
  int64_t r = (int64_t)sel[0];
  // full space (b = min(n, R)): the tail beyond b is zero, so r = b is the rule's answer
  // (the residual is rounding only; the oracle's rule also returns m when no r < m meets it)
  if (r < 0 && b >= m) r = std::min(b, m);
  if (r > m) r = m;  // b = n > m = R: the energy beyond R directions is rounding only
  // ... but a full-rank answer is certified only if the smallest Ritz value lies above the
  // squared Rayleigh-Ritz noise (~u lambda_1 per value): a full-space block reached because
  // the Gram-domain estimates could not resolve an eps^2 T below that noise would otherwise
  // return r = min(n, R) for a problem whose rank is far smaller (r2g: n = 600, R = 5000,
  // eps = 1e-9: one mode returned 600 against the oracle's 101).  Checked when the block
  // grew to the full space; a full space taken from the start (min(n, R) <= the first block)
  // keeps the rule's r = min(n, R) as before.
  if (epsmode && r == std::min(b, m) && b >= m && b > 1 && mo.grows > 0) {
    double lam[2] = {0.0, 0.0};
    RH_CHECK(d2h_wait(&lam[0], w.th.p, sizeof(double), st));
    RH_CHECK(d2h_wait(&lam[1], w.th.p + (r - 1), sizeof(double), st));
    const double noise = 8.0 * u * std::max(lam[0], 0.0) * std::sqrt((double)b);
    if (!(lam[1] > noise)) {
      char msg[320];
      snprintf(msg, sizeof msg,
               "mode %d: eps^2 T = %.3e cannot be resolved: the block reached the full space (%lld) and its "
               "smallest Ritz values are at the squared Rayleigh-Ritz noise (lambda_min %.3e <= %.3e)",
               mode, epsmode ? o.eps * o.eps * T : 0.0, (long long)b, lam[1], noise);
      return fail(RHOSVD_ENOCONV, msg);
    }
  }
  if (r < 0) {
    char msg[256];
    snprintf(msg, sizeof msg,
             "mode %d: rank rule not met inside the final block (b %lld, tail^2 %.6e > eps^2 T %.6e; "
             "rho %.6e) - block growth or subspace iteration did not converge",
             mode, (long long)b, sel[1], epsmode ? o.eps * o.eps * T : 0.0, rho_h);
    return fail(RHOSVD_ENOCONV, msg);
  }
  mo.r = (int)r;
  mo.b = (int)b;
  mo.tail2 = sel[1];
  mo.rho = rho_h;
  c.tm->mark(PH_PROJ);
  // outputs: Z_l = Z' P'_r, W_l^T = W'^T P'_r (Rl x r col-major == r x Rp row-major), sigma
  if (r > 0) {
    RH_CHECK(OC().get((void**)&mo.Z, (size_t)LDN * r * sizeof(double)));
    RH_CUDA(cudaMemsetAsync(mo.Z, 0, (size_t)LDN * r * sizeof(double), st));
    RH_CHECK(OC().get((void**)&mo.W, (size_t)r * Rp * sizeof(double)));
    RH_CUDA(cudaMemsetAsync(mo.W, 0, (size_t)r * Rp * sizeof(double), st));
    RH_CHECK(OC().get((void**)&mo.sigma, (size_t)r * sizeof(double)));
    RH_CHECK(mm(c, n, r, b, w.Z.p, LDN, false, w.V.p, ldb, true, mo.Z, LDN));
    RH_CHECK(mm(c, Rl, r, b, w.W.p, Rp, false, w.V.p, ldb, true, mo.W, Rp));
    RH_CUDA(cudaMemcpyAsync(mo.sigma, w.inv.p, r * sizeof(double), cudaMemcpyDeviceToDevice, st));
    // Retained directions at the rounding level (a fixed r above the numerical rank, or a
    // full space taken from the start): sigma_k <= 1e-10 sigma_1 is below what the squared
    // Rayleigh-Ritz resolves, and such frame columns come out of CholeskyQR's
    // dependent-column rule (unit pivot, zero sub-column), i.e. not orthonormal (r2h sweep:
    // n = 644, fixed r = 198 against a numerical rank of 131 gave |Z^T Z - I| = 1).  They are
    // replaced by an orthonormal completion of the other columns (random columns, projected
    // out of them twice, CholQR2) and their W rows recomputed as Z_c^T Uhat, so beta stays the
    // projection of A onto the returned frames; the energy they carry is <= 1e-20 of sigma_1^2
    // each, so the Tucker tensor is unchanged to rounding.  (Replacing every column that
    // failed a 1e-13 orthogonality test instead also dropped columns that carry energy:
    // Tucker error 0.78 on that case.)
    {
      double s1r[2] = {0.0, 0.0};
      RH_CHECK(d2h_wait(&s1r[0], mo.sigma, sizeof(double), st));
      RH_CHECK(d2h_wait(&s1r[1], mo.sigma + (r - 1), sizeof(double), st));
      if (!full_eye && r > 1 && !(s1r[1] > 1e-10 * s1r[0])) {
        std::vector<double> sg(r);
        RH_CHECK(d2h_wait(sg.data(), mo.sigma, r * sizeof(double), st));
        int64_t kg = 0;
        while (kg < r && sg[kg] > 1e-10 * sg[0]) ++kg;
        const int64_t nc = r - kg;
        double* X = mo.Z + kg * LDN;
        RH_CHECK(k_random(mo.Z, LDN, n, kg, r, seed ^ 0x5bd1e995ull, st));
        if (kg > 0) {
          const int64_t ldt = round_up(std::max<int64_t>(kg, 2), 2);
          for (int pass = 0; pass < 2; ++pass) {  // X -= Z_g (Z_g^T X), twice
            RH_CHECK(mm(c, kg, nc, n, mo.Z, LDN, true, X, LDN, true, w.S.p, ldt));
            GemmArgs gp;
            gp.M = n; gp.N = nc; gp.K = kg; gp.A = mo.Z; gp.lda = LDN; gp.a_k = false; gp.B = w.S.p; gp.ldb = ldt;
            gp.b_k = true; gp.C = X; gp.ldc = LDN; gp.alpha = -1.0; gp.beta = 1.0;
            RH_CHECK(gemm(gp, w.gsc, st, &c.flops));
          }
        }
        RH_CHECK(orth(c, n, nc, LDN, X, w.M.p, w.T1.p, ldbs(nc), ORTH_CQR2));
        RH_CUDA(cudaMemcpyAsync(X, w.M.p, (size_t)LDN * nc * sizeof(double), cudaMemcpyDeviceToDevice, st));
        if (Rl > 0) RH_CHECK(mm(c, Rl, nc, n, Uh, LDN, true, X, LDN, true, mo.W + kg * Rp, Rp));
        if (dbg_on())
          fprintf(stderr, "[rhosvd dbg] mode %d: %lld of %lld frame columns (sigma <= 1e-10 sigma_1) completed\n", mode,
                  (long long)nc, (long long)r);
      }
    }
    // Z = I path: the frames are I P P2_r, two accumulated Jacobi rotation sets (~35 sweeps
    // at n = 197: orthonormal to ~2e-13); one CholQR2 of the n x r frame brings that to
    // rounding and W = Z^T Uhat is recomputed from it, so beta stays the projection of A
    if (full_eye) {
      RH_CHECK(orth(c, n, r, LDN, mo.Z, w.M.p, w.T1.p, ldbs(r), ORTH_CQR2));
      RH_CUDA(cudaMemcpy2DAsync(mo.Z, LDN * sizeof(double), w.M.p, LDN * sizeof(double), n * sizeof(double), r,
                                cudaMemcpyDeviceToDevice, st));
      if (Rl > 0) RH_CHECK(mm(c, Rl, r, n, Uh, LDN, true, mo.Z, LDN, true, mo.W, Rp));
    }
    if (o.flags & RHOSVD_F_SIGN_FIX) RH_CHECK(k_sign_fix(mo.Z, LDN, n, r, mo.W, Rp, Rl, w.sgn.p, st));
  }
  TL().mark(mode, "projection", st);
  TL().hmark(mode, "projection launched");
  return RHOSVD_OK;
}

// ---------------------------------------------------------------- C2T ALS
// One frame update of mode l with the frames of the other two modes (b, c) fixed
// (Eq. can_A_Tuck_als, Fig. 2): Z_l <- the r_l dominant left singular
// vectors of the mode-l unfolding  M_l = Uhat_l D (W_c (.) W_b)^T  (n x r_b r_c) of
// A x_b Z_b^T x_c Z_c^T, D = diag(xi'), W_m = Z_m^T Uhat_m.  M_l is never formed
// (r_b r_c = 4.2e5 columns on cfg 4); its Gram is
//     G_l = M_l M_l^T = Uhat_l K' Uhat_l^T,   K' = D [(W_b^T W_b) o (W_c^T W_c)] D  (R x R),
// built from column blocks of K' (never stored whole):  K'[:, blk] by two GEMMs, a
// Hadamard product and the D scalings; T = Uhat_l K'[:, blk]; G_l += T Uhat_l[:, blk]^T.
// The dominant eigenvectors of G_l: subspace iteration started from the current Z_l
// (plus p random columns), CholQR2, then a Rayleigh-Ritz step with the block Jacobi;
// sigma_l = sqrt of the top r_l Ritz values (singular values of M_l, reading L3).
// Subspace accuracy is the Gram-domain one (u kappa^2 / gap), enough for the frame
// update; the core is recomputed from the new frames (reading L2).
static int als_update(Ctx& c, int l, int64_t n, int64_t LDN, int64_t Rl, int64_t Rp, double* const Uh[3],
                      const double* xip, ModeOut mo[3], const rhosvd_opts& o, uint64_t seed) {
  ModeWs& w = *c.m;
  cudaStream_t st = c.st;
  const int bm = (l + 1) % 3 < (l + 2) % 3 ? (l + 1) % 3 : (l + 2) % 3;
  const int cm = 3 - l - bm;
  const int64_t r = mo[l].r, rb = mo[bm].r, rc = mo[cm].r;
  if (r <= 0 || Rl <= 0) return RHOSVD_OK;
  double* G = c.w.G.p + (size_t)l * LDN * LDN;
  const double* Wb = mo[bm].W;  // r_b x Rp row-major == col-major Rp x r_b (W^T)
  const double* Wc = mo[cm].W;
  // Two routes to G_l, the cheaper one by FLOP count:
  //   direct : M_l^T = (xi' o W_b) (.) W_c contracted with Uhat_l^T over R - the core
  //            kernel's Khatri-Rao contraction with Uhat_l^T as its third factor - then
  //            G = M M^T;          2 n R r_b r_c + n^2 r_b r_c      (cfg 5: 1e13)
  //   blocked: K' column blocks;   2 R^2 (r_b + r_c) + 2 n R^2 + 2 n^2 R   (cfg 4: 1.6e13)
  const double f_direct = 2.0 * n * (double)Rl * rb * rc + 1.0 * n * (double)n * rb * rc;
  const double f_block = 2.0 * (double)Rl * Rl * (rb + rc) + 2.0 * n * (double)Rl * Rl + 2.0 * n * (double)n * Rl;
  // RHOSVD_ALS_ROUTE=direct|block forces a route (tests cover both)
  static const int route = [] {
    const char* e = getenv("RHOSVD_ALS_ROUTE");
    return !e ? 0 : (e[0] == 'd' ? 1 : (e[0] == 'b' ? 2 : 0));
  }();
  const bool direct = route == 1 || (route == 0 && f_direct < f_block);
  if (direct && rb > 0 && rc > 0) {
    const int64_t kr = rb * rc;
    RH_CHECK(c.w.alsT.ensure((size_t)LDN * Rp + 64, st));   // Uhat_l^T (LDN x Rp row-major)
    RH_CHECK(c.w.alsK1.ensure((size_t)LDN * kr + 64, st));  // M_l (LDN x r_b r_c, col-major)
    RH_CHECK(c.w.W1x.ensure((size_t)rb * Rp + 64, st));
    RH_CHECK(c.w.W2x.ensure(core_ws_doubles(rc, Rl, Rp), st));
    RH_CHECK(c.w.corepart.ensure(core_part_doubles(rb, rc, LDN, Rl), st));
    RH_CHECK(k_transpose(Uh[l], LDN, LDN, Rp, c.w.alsT.p, Rp, st));
    RH_CHECK(scale_cols(Wb, Rp, xip, rb, Rp, c.w.W1x.p, Rp, st));
    RH_CHECK(core_kr(c.w.W1x.p, Rp, Wc, c.w.alsT.p, Rp, rb, rc, LDN, Rl, c.w.alsK1.p, c.w.W2x.p, c.w.corepart.p,
                     c.w.corepart.cap, st, &c.flops));
    RH_CHECK(mm(c, LDN, LDN, kr, c.w.alsK1.p, LDN, false, c.w.alsK1.p, LDN, false, G, LDN, nullptr, true));
  } else {
  // K' column blocks: 2 x Rp x Rb doubles within ~1.5 GB
  const int64_t Rb = std::max<int64_t>(128, std::min<int64_t>(round_up(Rl, 128), ((int64_t)96 << 20) / Rp / 128 * 128));
  RH_CHECK(c.w.alsK1.ensure((size_t)Rp * Rb + 64, st));
  RH_CHECK(c.w.alsK2.ensure((size_t)Rp * Rb + 64, st));
  RH_CHECK(c.w.alsT.ensure((size_t)LDN * Rb + 64, st));
  double *K1 = c.w.alsK1.p, *K2 = c.w.alsK2.p, *T = c.w.alsT.p;
  for (int64_t b0 = 0; b0 < Rl; b0 += Rb) {
    const int64_t nb = std::min<int64_t>(Rb, Rl - b0);
    // K1 = D (W_b^T W_b[:, blk]) D_blk ; K2 = W_c^T W_c[:, blk] ; K2 <- K1 o K2
    if (rb > 0) {
      RH_CHECK(mm(c, Rl, nb, rb, Wb, Rp, false, Wb + b0, Rp, false, K1, Rp, xip + b0, false, xip));
    } else {
      RH_CUDA(cudaMemsetAsync(K1, 0, (size_t)Rp * nb * sizeof(double), st));
    }
    if (rc > 0) {
      RH_CHECK(mm(c, Rl, nb, rc, Wc, Rp, false, Wc + b0, Rp, false, K2, Rp));
    } else {
      RH_CUDA(cudaMemsetAsync(K2, 0, (size_t)Rp * nb * sizeof(double), st));
    }
    RH_CHECK(k_hadamard(K1, K2, Rp, Rl, nb, st));
    // T = Uhat_l K'[:, blk]  (n x nb)
    RH_CHECK(mm(c, n, nb, Rl, Uh[l], LDN, false, K2, Rp, true, T, LDN));
    // G (+)= T Uhat_l[:, blk]^T
    GemmArgs g;
    g.M = n; g.N = n; g.K = nb; g.A = T; g.lda = LDN; g.a_k = false;
    g.B = Uh[l] + (size_t)b0 * LDN; g.ldb = LDN; g.b_k = false;
    g.C = G; g.ldc = LDN; g.beta = b0 > 0 ? 1.0 : 0.0;
    RH_CHECK(gemm(g, w.gsc, st, &c.flops));
  }
  }
  TL().mark(l, "ALS Gram", st);
  // ---- dominant r eigenvectors of G: start [Z_l | random], CholQR2 subspace iteration
  const int64_t m = n;
  const int64_t bsz = std::min<int64_t>(m, r + std::max(1, o.oversample));
  const int64_t ldb = round_up(std::max<int64_t>(bsz, 2), 2);
  RH_CHECK(w.Z.ensure((size_t)LDN * bsz + 64, st));
  RH_CHECK(w.Y.ensure((size_t)LDN * bsz + 64, st));
  RH_CHECK(w.T1.ensure((size_t)LDN * bsz + 64, st));
  for (DBuf* d : {&w.S, &w.V, &w.Bp}) RH_CHECK(d->ensure((size_t)ldb * bsz + 64, st));
  for (DBuf* d : {&w.th, &w.inv, &w.sgn}) RH_CHECK(d->ensure((size_t)bsz + 64, st));
  RH_CUDA(cudaMemcpy2DAsync(w.Z.p, LDN * sizeof(double), mo[l].Z, LDN * sizeof(double), n * sizeof(double), r,
                            cudaMemcpyDeviceToDevice, st));
  if (bsz > r) RH_CHECK(k_random(w.Z.p, LDN, n, r, bsz, seed, st));
  std::vector<double> d_h(bsz);
  int need = 60;
  for (int it = 1; it <= need; ++it) {
    RH_CHECK(mm(c, n, bsz, n, G, LDN, false, w.Z.p, LDN, true, w.Y.p, LDN));
    RH_CHECK(k_coldot(w.Z.p, w.Y.p, LDN, n, bsz, w.th.p, st));
    RH_CHECK(orth(c, n, bsz, LDN, w.Y.p, w.Z.p, w.T1.p, ldb, it == 1 ? ORTH_SCQR3 : ORTH_CQR2));
    if (it == 2 && bsz > r) {
      // rate lambda_{b} / lambda_r from the Rayleigh quotients -> iterations for 1e-13
      RH_CHECK(d2h_wait(d_h.data(), w.th.p, bsz * sizeof(double), st));
      const double dr = std::max(d_h[r - 1], 1e-300);
      const double rho = std::min(0.995, std::max(d_h[bsz - 1], 1e-300 * dr) / dr);
      need = std::max(3, std::min(60, 2 + (int)std::ceil(std::log(1e-13) / std::log(rho))));
    }
    if (bsz >= m) break;  // the whole space: one step is exact
  }
  // Rayleigh-Ritz: S = Z^T G Z, S = V diag(lambda) V^T, Z_l = Z V[:, :r], sigma = sqrt(lambda)
  RH_CHECK(mm(c, n, bsz, n, G, LDN, false, w.Z.p, LDN, true, w.Y.p, LDN));
  RH_CHECK(mm(c, bsz, bsz, n, w.Z.p, LDN, true, w.Y.p, LDN, true, w.S.p, ldb, nullptr, true));
  {
    int sw = 0;
    RH_CHECK(syevj(bsz, w.S.p, ldb, w.th.p, w.V.p, ldb, 1e-15, 1e-300, 80, w.dws, st, &sw));
    if (sw < 0) return fail(RHOSVD_ENOCONV, "ALS: Jacobi on Z^T G Z did not converge");
  }
  RH_CHECK(mm(c, n, r, bsz, w.Z.p, LDN, false, w.V.p, ldb, true, mo[l].Z, LDN));
  RH_CHECK(k_sqrt_clamp(w.th.p, r, mo[l].sigma, st));
  if (o.flags & RHOSVD_F_SIGN_FIX) RH_CHECK(k_sign_fix(mo[l].Z, LDN, n, r, nullptr, 0, 0, w.sgn.p, st));
  // the new CP factor of the core: W_l = Z_l^T Uhat_l  (r x Rp row-major)
  RH_CHECK(mm(c, Rl, r, n, Uh[l], LDN, true, mo[l].Z, LDN, true, mo[l].W, Rp));
  TL().mark(l, "ALS frame update", st);
  return RHOSVD_OK;
}

}  // namespace rhosvd

// ====================================================================== C ABI
using namespace rhosvd;

#include "result.h"

extern "C" {

const char* rhosvd_last_error(void) { return g_err.c_str(); }
const char* rhosvd_version(void) { return "rhosvd-b200 0.1 (sm_100a, FP64 DMMA)"; }

void rhosvd_opts_default(rhosvd_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->rank_mode = RHOSVD_EPS;
  o->r[0] = o->r[1] = o->r[2] = 10;
  o->eps = 1e-6;
  o->oversample = 16;
  o->block0 = 0;  // 0: default first block (128)
  o->max_iters = 30;
  o->refine_steps = 1;
  o->seed = 12345;
  o->flags = RHOSVD_F_SIGN_FIX;
}

void rhosvd_result_free(rhosvd_result* r) {
  if (!r) return;
  // outputs go back to the library's output cache once no queued work uses them
  cudaDeviceSynchronize();
  for (int l = 0; l < 3; ++l) {
    OC().put(r->Z[l]);
    OC().put(r->sigma[l]);
    OC().put(r->W[l]);
    HC().put(r->hZ[l]);
    HC().put(r->hsigma[l]);
  }
  OC().put(r->beta);
  HC().put(r->hbeta);
  delete r;
}

int rhosvd_result_ranks(const rhosvd_result* r, int32_t out[3]) {
  if (!r || !out) return fail(RHOSVD_EINVAL, "null");
  for (int l = 0; l < 3; ++l) out[l] = r->ranks[l];
  return RHOSVD_OK;
}
int rhosvd_result_frame(const rhosvd_result* r, int mode, const double** Z, int64_t* ldz) {
  if (!r || !Z || !ldz || mode < 0 || mode > 2) return fail(RHOSVD_EINVAL, "bad args");
  *Z = r->Z[mode];
  *ldz = r->ldz;
  return RHOSVD_OK;
}
int rhosvd_result_sigma(const rhosvd_result* r, int mode, const double** s, int64_t* count) {
  if (!r || !s || !count || mode < 0 || mode > 2) return fail(RHOSVD_EINVAL, "bad args");
  *s = r->sigma[mode];
  *count = r->ranks[mode];
  return RHOSVD_OK;
}
int rhosvd_result_core(const rhosvd_result* r, const double** beta) {
  if (!r || !beta) return fail(RHOSVD_EINVAL, "bad args");
  if (!r->beta_valid) return fail(RHOSVD_EINVAL, "RHOSVD_F_ROOT_ONLY_CORE: beta is on rank 0 only");
  *beta = r->beta;
  return RHOSVD_OK;
}
int rhosvd_result_cpfactor(const rhosvd_result* r, int mode, const double** W, int64_t* ldw) {
  if (!r || !W || !ldw || mode < 0 || mode > 2) return fail(RHOSVD_EINVAL, "bad args");
  *W = r->W[mode];
  *ldw = r->Rp;
  return RHOSVD_OK;
}
int rhosvd_result_report(const rhosvd_result* r, rhosvd_report* out) {
  if (!r || !out) return fail(RHOSVD_EINVAL, "bad args");
  *out = r->rep;
  return RHOSVD_OK;
}

// D2H of finished row chunks of beta (rhosvd_c2t_host; CoreChunks callback)
struct BetaD2H {
  const double* dev;
  double* host;
  cudaStream_t cp;
};
static int beta_chunk_d2h(void* ctx, int, int64_t e0, int64_t e1, cudaStream_t s) {
  auto* b = (BetaD2H*)ctx;
  if (e1 <= e0) return RHOSVD_OK;
  cudaEvent_t ev;
  RH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  RH_CUDA(cudaEventRecord(ev, s));
  RH_CUDA(cudaStreamWaitEvent(b->cp, ev, 0));
  cudaEventDestroy(ev);
  RH_CUDA(cudaMemcpyAsync(b->host + e0, b->dev + e0, (size_t)(e1 - e0) * sizeof(double), cudaMemcpyDeviceToHost,
                          b->cp));
  return RHOSVD_OK;
}

// R-sharded core: all-reduce each finished row chunk of beta on the collective stream
// while the next chunks are still being contracted (every rank issues the chunks in the
// same order from one thread, so the NCCL calls match)
struct BetaAR {
  rhosvd_comm* comm;
  double* beta;
  cudaStream_t cs;
  bool root_only;  // RHOSVD_F_ROOT_ONLY_CORE: reduce to rank 0 instead of all-reduce
};
static int beta_chunk_allreduce(void* ctx, int, int64_t e0, int64_t e1, cudaStream_t s) {
  auto* b = (BetaAR*)ctx;
  if (e1 <= e0) return RHOSVD_OK;
  cudaEvent_t ev;
  RH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  RH_CUDA(cudaEventRecord(ev, s));
  RH_CUDA(cudaStreamWaitEvent(b->cs, ev, 0));
  cudaEventDestroy(ev);
  if (comm_trace()) fprintf(stderr, "[rhosvd comm] rank %d beta chunk [%lld, %lld)\n", b->comm->rank, (long long)e0,
                            (long long)e1);
  return b->root_only ? comm_reduce_root(b->comm, b->beta + e0, e1 - e0, b->cs)
                     : comm_allreduce(b->comm, b->beta + e0, e1 - e0, b->cs);
}

static int c2t_impl(const double* U_in[3], int64_t ldu, const double* xi, int64_t n, int64_t Rl,
                    const rhosvd_opts& o, rhosvd_comm* comm, cudaStream_t st, rhosvd_result* res,
                    const HostIn* hin = nullptr, int als_sweeps = 0) {
  Workspace& w = WS();
  const double* U[3] = {U_in[0], U_in[1], U_in[2]};
  // host inputs: H2D on the copy stream, one event per mode, so mode l's normalize and
  // Gram start as soon as its side matrix has arrived (the others still in flight)
  cudaStream_t cp = nullptr;
  cudaEvent_t evU[3] = {nullptr, nullptr, nullptr}, evX = nullptr;
  struct CopyGuard {  // every return path leaves no copy of the caller's buffers in flight
    cudaStream_t cp = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    ~CopyGuard() {
      if (cp) cudaStreamSynchronize(cp);
      for (auto e : ev)
        if (e) cudaEventDestroy(e);
    }
  } guard;
  if (hin) {
    cp = copy_stream();
    if (!cp) return fail(RHOSVD_ECUDA, "copy stream creation failed");
    guard.cp = cp;
    const size_t per = Rl > 0 ? (size_t)(Rl - 1) * ldu + n : 0;
    RH_CHECK(w.Ustage.ensure(3 * std::max<size_t>(per, 1), st));
    RH_CHECK(w.xistage.ensure(std::max<int64_t>(Rl, 1), st));
    cudaEvent_t e0;
    RH_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    RH_CUDA(cudaEventRecord(e0, st));  // the staging buffers are ready on st
    RH_CUDA(cudaStreamWaitEvent(cp, e0, 0));
    cudaEventDestroy(e0);
    for (int l = 0; l < 3; ++l) {
      double* d = w.Ustage.p + (size_t)l * std::max<size_t>(per, 1);
      if (per) RH_CUDA(cudaMemcpyAsync(d, hin->U[l], per * sizeof(double), cudaMemcpyHostToDevice, cp));
      RH_CUDA(cudaEventCreateWithFlags(&evU[l], cudaEventDisableTiming));
      guard.ev[l] = evU[l];
      RH_CUDA(cudaEventRecord(evU[l], cp));
      U[l] = d;
    }
    if (Rl > 0) RH_CUDA(cudaMemcpyAsync(w.xistage.p, hin->xi, Rl * sizeof(double), cudaMemcpyHostToDevice, cp));
    RH_CUDA(cudaEventCreateWithFlags(&evX, cudaEventDisableTiming));
    guard.ev[3] = evX;
    RH_CUDA(cudaEventRecord(evX, cp));
    xi = w.xistage.p;
  }
  rhosvd_report& rep = res->rep;
  PhaseTimer tm(st);
  Ctx c{st, comm, w, &rep, &tm};
  g_launches = 0;
  TL().begin(st);
  tm.mark(PH_NORM);
  const int world = comm ? comm->world : 1;
  const int64_t LDN = round_up(n, 16);
  // Rp: multiple of 32 (one GEMM k-stage), so the batched Gram's modes start on stage
  // boundaries; padding columns of Uhat are zero
  const int64_t Rp = round_up(std::max<int64_t>(Rl, 1), 32);
  res->n = n;
  res->ldz = LDN;
  res->Rl = Rl;
  res->Rp = Rp;

  RH_CHECK(w.scal.ensure(256, st));
  if (!w.flag) RH_CUDA(cudaMallocAsync((void**)&w.flag, 64, st));
  RH_CUDA(cudaMemsetAsync(w.flag, 0, 64, st));
  RH_CUDA(cudaMemsetAsync(w.scal.p, 0, 256 * sizeof(double), st));

  // ---- agreement check + global R (SURVEY.md 8(b) EMISMATCH)
  {
    double h = (double)((n * 1000003 + o.rank_mode * 97 + o.r[0] * 7 + o.r[1] * 11 + o.r[2] * 13 +
                         o.oversample * 17 + o.block0 * 19 + o.refine_steps * 23) % 1000000007) +
               o.eps * 1e6;
    double v[4] = {(double)Rl, h, h * h, 1.0};
    RH_CHECK(h2d_wait(w.scal.p, v, sizeof(v), st));
    RH_CHECK(allreduce(c, w.scal.p, 4));
    RH_CHECK(d2h_wait(v, w.scal.p, sizeof(v), st));
    if (std::fabs(v[1] - world * h) > 1e-6 * std::fabs(world * h) + 1e-9 ||
        std::fabs(v[2] - world * h * h) > 1e-6 * std::fabs(world * h * h) + 1e-9)
      return fail(RHOSVD_EMISMATCH, "ranks disagree on n / options");
    rep.R_global = (int64_t)std::llround(v[0]);
  }
  const int64_t Rg = rep.R_global;
  if (Rg == 0) {  // zero tensor: empty Tucker tensor (SURVEY.md 8(b) edge cases)
    tm.mark(-1);
    tm.collect(rep.ms);
    rep.launches = g_launches;
    return RHOSVD_OK;
  }

  // ---- S1 normalize (K0); with host inputs each mode's Gram (S2) follows its
  // normalize at once, overlapping the H2D of the next side matrix (a non-finite input
  // makes that Gram garbage, and the check below rejects the call before it is used)
  RH_CHECK(w.Uh.ensure((size_t)3 * LDN * Rp, st));
  RH_CHECK(w.s.ensure((size_t)3 * Rp, st));
  RH_CHECK(w.tcol.ensure((size_t)3 * Rp, st));
  RH_CHECK(w.xip.ensure((size_t)Rp, st));
  RH_CHECK(w.xip2.ensure((size_t)Rp, st));
  RH_CHECK(w.part.ensure(1024, st));
  RH_CHECK(w.G.ensure_zero((size_t)3 * LDN * LDN, st));
  cudaEvent_t g0, g1;
  cudaEventCreate(&g0);
  cudaEventCreate(&g1);
  double* Uh[3];
  // per-mode Gram (host-input paths, where mode l's Gram starts as soon as U_l lands):
  // K = Rp and the batched form's split count, so every entry is summed exactly as in the
  // one-launch batched Gram of the device-input path (bitwise identical G)
  const int gram_splits = gemm_batch_splits(n, n, Rp, true, 3);
  auto gram_args = [&](int l) {
    GemmArgs g;
    g.M = n; g.N = n; g.K = Rp; g.A = Uh[l]; g.lda = LDN; g.a_k = false; g.B = Uh[l]; g.ldb = LDN; g.b_k = false;
    g.C = w.G.p + (size_t)l * LDN * LDN; g.ldc = LDN; g.upper_sym = true; g.splits = gram_splits;
    return g;
  };
  auto gram = [&](int l) -> int {
    double* G = w.G.p + (size_t)l * LDN * LDN;
    if (Rl > 0) {
      RH_CHECK(gemm(gram_args(l), c.m ? c.m->gsc : w.gsc, c.st, &c.flops));
    } else {
      RH_CUDA(cudaMemsetAsync(G, 0, (size_t)LDN * LDN * sizeof(double), st));
    }
    return RHOSVD_OK;
  };
  for (int l = 0; l < 3; ++l) Uh[l] = w.Uh.p + (size_t)l * LDN * Rp;
  // Streamed host path (host inputs, one GPU, concurrent modes): each mode's thread
  // normalises its side matrix, forms its Gram and starts its eigensolve as soon as ITS
  // H2D copy has landed, so the eigensolves of the first modes overlap the copies of the
  // later ones (the copy engine, not the SMs, bounds the input phase).  xi' and the
  // non-finite checks follow from per-mode flags.
  const bool streamed = hin && modes_concurrent() && !(comm && comm->active()) && Rl > 0;
  float gram_ms_streamed = 0.f;
  const bool early_gram = hin != nullptr;
  if (!streamed) {
  for (int l = 0; l < 3; ++l) {
    if (hin) RH_CUDA(cudaStreamWaitEvent(st, evU[l], 0));
    RH_CHECK(k_normalize(U[l], ldu, n, Rl, Rp, Uh[l], LDN, w.s.p + l * Rp, w.tcol.p + l * Rp, w.flag, st));
    RH_CHECK(k_fixed_sum(w.tcol.p + l * Rp, Rp, w.scal.p + 4 + l, st));
    if (early_gram) {
      if (l == 0) cudaEventRecord(g0, st);
      RH_CHECK(gram(l));
      if (l == 2) cudaEventRecord(g1, st);
    }
  }
  if (hin) RH_CUDA(cudaStreamWaitEvent(st, evX, 0));
  RH_CHECK(k_xiprime(xi, w.s.p, w.s.p + Rp, w.s.p + 2 * Rp, Rl, Rp, w.xip.p, w.xip2.p, w.flag, st));
  RH_CHECK(k_fixed_sum(w.xip2.p, Rp, w.scal.p + 7, st));
  // flag -> scal[8] as double (non-finite count)
  {
    int fl = 0;
    RH_CHECK(d2h_wait(&fl, w.flag, sizeof(int), st));
    double f = fl ? 1.0 : 0.0;
    RH_CHECK(h2d_wait(w.scal.p + 8, &f, sizeof(double), st));
  }
  tm.mark(PH_NORM);
  RH_CHECK(allreduce(c, w.scal.p + 4, 5));  // T1..T3, ||xi'||^2, flag
  double sc[5];
  RH_CHECK(d2h_wait(sc, w.scal.p + 4, sizeof(sc), st));
  if (sc[4] != 0.0) {
    cudaEventDestroy(g0);
    cudaEventDestroy(g1);
    return fail(RHOSVD_ENONFINITE, "NaN/Inf in U or xi");
  }
  for (int l = 0; l < 3; ++l) rep.trace[l] = sc[l];
  rep.xi_norm = std::sqrt(sc[3]);

  // ---- S2 Gram (K1), all three modes, then all-reduce
  tm.mark(PH_GRAM);
  if (!early_gram) {
    // the three modes' Grams as ONE persistent launch (batched GEMM: mode l reads Uhat at
    // k + l Rp, writes G + l LDN^2): one wave schedule over 3x the tiles instead of three
    // launches each ending on a partial wave
    cudaEventRecord(g0, st);
    if (Rl > 0) {
      GemmArgs g = gram_args(0);
      g.batch = 3; g.a_koff = g.b_koff = Rp; g.c_bstride = LDN * LDN;
      RH_CHECK(gemm(g, w.gsc, st, &c.flops));
    } else {
      for (int l = 0; l < 3; ++l) RH_CHECK(gram(l));
    }
    cudaEventRecord(g1, st);
  }
  RH_CHECK(allreduce(c, w.G.p, 3 * LDN * LDN));
  TL().mark(-1, "Gram", st);
  }  // !streamed
  tm.mark(PH_EIG);

  // ---- S3-S5 per mode.  The three modes are independent; on one GPU (no collectives
  // inside) they run concurrently: one host thread and one stream per mode, so the
  // latency-bound b x b kernels and host decisions of one mode overlap the GEMMs of
  // the others.  With a communicator the modes run in order (one communicator must not
  // be used by two threads at once).
  ModeOut mo[3];
  int mst[3] = {RHOSVD_OK, RHOSVD_OK, RHOSVD_OK};
  std::string merr[3];
  const bool concurrent = modes_concurrent();
  if (concurrent) {
    int dev = 0;
    RH_CUDA(cudaGetDevice(&dev));
    cudaStream_t* ms = mode_streams();
    if (!ms) return fail(RHOSVD_ECUDA, "mode stream creation failed");
    cudaEvent_t ev0;
    RH_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
    RH_CUDA(cudaEventRecord(ev0, st));
    for (int l = 0; l < 3; ++l) RH_CUDA(cudaStreamWaitEvent(ms[l], ev0, 0));
    std::unique_ptr<CommSched> sched;
    std::thread comm_thread;
    // every return path below stops the comm thread: all modes marked finished, joined
    struct CommJoin {
      std::unique_ptr<CommSched>& s;
      std::thread& t;
      ~CommJoin() {
        if (!t.joinable()) return;
        for (int l = 0; l < 3; ++l) s->finish(l);
        t.join();
      }
    } comm_join{sched, comm_thread};
    if (comm && comm->active()) {
      sched.reset(new CommSched());
      sched->comm = comm;
      sched->dev = dev;
      comm_thread = std::thread([&] { sched->run(); });
    }
    // mode parallelism (RHOSVD_MODE_PARALLEL=0 replicates the subspace iterations instead)
    static const bool mpar_on = [] {
      const char* e = getenv("RHOSVD_MODE_PARALLEL");
      return !(e && e[0] == '0');
    }();
    ModeLatch latch, latch2;
    MPar mpar[3];
    const bool mode_parallel = mpar_on && sched && !streamed;
    if (mode_parallel)
      for (int l = 0; l < 3; ++l) {
        mpar[l].root = l % comm->world;
        mpar[l].owner = mpar[l].root == comm->rank;
        mpar[l].latch = &latch;
        mpar[l].latch2 = &latch2;
        if (mpar[l].owner) ++latch.pending, ++latch2.pending;
      }
    if (mode_parallel)
      for (int l = 0; l < 3; ++l) mpar[l].owned = std::max(1, latch.pending);
    double mflops[3] = {0, 0, 0};
    int mlaunch[3] = {0, 0, 0};
    double mphase[3][16] = {{0}};
    // streamed path: per-mode "normalised" events and a host signal so the main thread
    // can queue xi' (which needs all three column-norm vectors) behind them
    cudaEvent_t evN[3] = {nullptr, nullptr, nullptr}, evG[3][2] = {{nullptr, nullptr}};
    std::mutex nmu;
    std::condition_variable ncv;
    int nready = 0;
    if (streamed)
      for (int l = 0; l < 3; ++l) {
        RH_CUDA(cudaEventCreateWithFlags(&evN[l], cudaEventDisableTiming));
        RH_CUDA(cudaEventCreate(&evG[l][0]));
        RH_CUDA(cudaEventCreate(&evG[l][1]));
      }
    auto prep_mode = [&](Ctx& cl, int l) -> int {
      struct Signal {  // signal the main thread on every path (no deadlock on errors)
        std::mutex& mu; std::condition_variable& cv; int& k; bool done = false;
        void fire() {
          if (done) return;
          done = true;
          { std::lock_guard<std::mutex> lk(mu); ++k; }
          cv.notify_all();
        }
        ~Signal() { fire(); }
      } sig{nmu, ncv, nready};
      cudaStream_t ls = cl.st;
      int* fl = w.flag + 1 + l;
      RH_CUDA(cudaStreamWaitEvent(ls, evU[l], 0));
      TL().mark(l, "H2D landed", ls);
      RH_CHECK(k_normalize(U[l], ldu, n, Rl, Rp, Uh[l], LDN, w.s.p + l * Rp, w.tcol.p + l * Rp, fl, ls));
      RH_CHECK(k_fixed_sum(w.tcol.p + l * Rp, Rp, w.scal.p + 4 + l, ls));
      RH_CUDA(cudaEventRecord(evN[l], ls));
      sig.fire();
      RH_CUDA(cudaEventRecord(evG[l][0], ls));
      RH_CHECK(gemm(gram_args(l), cl.m->gsc, ls, &cl.flops));
      RH_CUDA(cudaEventRecord(evG[l][1], ls));
      TL().mark(l, "Gram", ls);
      double tl = 0.0;
      int fh = 0;
      RH_CHECK(d2h_wait(&tl, w.scal.p + 4 + l, sizeof(double), ls));
      RH_CHECK(d2h_wait(&fh, fl, sizeof(int), ls));
      if (fh) return fail(RHOSVD_ENONFINITE, "NaN/Inf in U");
      rep.trace[l] = tl;
      TL().mark(l, "normalize + Gram", ls);
      return RHOSVD_OK;
    };
    auto run = [&](int l) {
      cudaSetDevice(dev);
      g_launches = 0;
      struct CapGuard {  // cooperative grids of this mode (see common.cuh)
        CapGuard() {
          // default: a third of the SMs, so the three modes' grid-synchronised kernels
          // (block Jacobi, blocked Cholesky) run side by side instead of one after another
          // (r2h: cfg 2 eigensolve 8.4 -> 7.7 ms, cfg 4 129 -> 126 ms).  RHOSVD_COOP_MODE_CTAS
          // sets an absolute cap; RHOSVD_COOP_MODE_CAP a cap in CTAs per 2 SMs (0 = none).
          static const int per2 = [] {
            const char* e = getenv("RHOSVD_COOP_MODE_CAP");
            return e ? std::max(0, atoi(e)) : -1;
          }();
          static const int ctas = [] {
            const char* e = getenv("RHOSVD_COOP_MODE_CTAS");
            return e ? std::max(0, atoi(e)) : 0;
          }();
          g_coop_cap = ctas ? ctas
                            : per2 < 0 ? std::max(1, num_sms() / 3)
                                       : (per2 ? std::max(1, num_sms() * per2 / 2) : 0);
        }
        ~CapGuard() { g_coop_cap = 0; }
      } cap_guard;
      PhaseTimer mtm(ms[l]);
      mtm.mark(PH_EIG);
      Ctx cl{ms[l], comm, w, &rep, &mtm};
      cl.m = &w.mw[l];
      cl.sched = sched.get();
      cl.mp = mode_parallel ? &mpar[l] : nullptr;
      cl.mode = l;
      if (streamed) {
        mst[l] = prep_mode(cl, l);
        if (mst[l] != RHOSVD_OK) {
          merr[l] = g_err;
          mtm.mark(-1);
          mtm.collect(mphase[l]);
          mlaunch[l] = g_launches;
          return;
        }
      }
      mst[l] = solve_mode(cl, l, n, LDN, Rl, Rp, Rg, Uh[l], w.G.p + (size_t)l * LDN * LDN, rep.trace[l], o, mo[l]);
      if (cl.mp) cl.mp->signal(), cl.mp->signal2();  // an early error must not leave the other modes waiting
      if (cl.sched) cl.sched->finish(l);
      mtm.mark(-1);
      if (mst[l] != RHOSVD_OK) merr[l] = g_err;
      mtm.collect(mphase[l]);
      mflops[l] = cl.flops;
      mlaunch[l] = g_launches;
    };
    if (streamed) {
      std::thread t0(run, 0), t1(run, 1), t2(run, 2);
      {  // xi' behind the three normalisations (the core needs it; the eigensolves do not)
        std::unique_lock<std::mutex> lk(nmu);
        ncv.wait(lk, [&] { return nready == 3; });
      }
      int xs = RHOSVD_OK;
      for (int l = 0; l < 3 && xs == RHOSVD_OK; ++l)
        if (cudaStreamWaitEvent(st, evN[l], 0) != cudaSuccess) xs = fail(RHOSVD_ECUDA, "event wait");
      if (xs == RHOSVD_OK && cudaStreamWaitEvent(st, evX, 0) != cudaSuccess) xs = fail(RHOSVD_ECUDA, "event wait");
      if (xs == RHOSVD_OK) xs = k_xiprime(xi, w.s.p, w.s.p + Rp, w.s.p + 2 * Rp, Rl, Rp, w.xip.p, w.xip2.p, w.flag, st);
      if (xs == RHOSVD_OK) xs = k_fixed_sum(w.xip2.p, Rp, w.scal.p + 7, st);
      t0.join();
      t1.join();
      t2.join();
      if (xs != RHOSVD_OK) return xs;
      double x2 = 0.0;
      int fx = 0;
      RH_CHECK(d2h_wait(&x2, w.scal.p + 7, sizeof(double), st));
      RH_CHECK(d2h_wait(&fx, w.flag, sizeof(int), st));
      for (int l = 0; l < 3; ++l) {
        float gm = 0.f;
        if (mst[l] == RHOSVD_OK && cudaEventElapsedTime(&gm, evG[l][0], evG[l][1]) == cudaSuccess) gram_ms_streamed += gm;
        cudaEventDestroy(evN[l]);
        cudaEventDestroy(evG[l][0]);
        cudaEventDestroy(evG[l][1]);
      }
      if (fx) {
        cudaDeviceSynchronize();
        for (int q = 0; q < 3; ++q) {
          OC().put(mo[q].Z);
          OC().put(mo[q].W);
          OC().put(mo[q].sigma);
        }
        return fail(RHOSVD_ENONFINITE, "NaN/Inf in xi");
      }
      rep.xi_norm = std::sqrt(x2);
    } else {
      std::thread t1(run, 1), t2(run, 2);
      run(0);
      t1.join();
      t2.join();
    }
    if (comm_thread.joinable()) comm_thread.join();
    TL().hmark(-1, "modes joined");
    g_launches += mlaunch[0] + mlaunch[1] + mlaunch[2];
    c.flops += mflops[0] + mflops[1] + mflops[2];
    // per-phase device times of the concurrent region, summed over the modes (ms[9..13]:
    // eigensolve, rr_refine, residual_rank, projection, collectives)
    for (int l = 0; l < 3; ++l)
      for (int ph = PH_EIG; ph <= PH_COMM; ++ph) rep.ms[9 + ph - PH_EIG] += mphase[l][ph];
    cudaEvent_t ev[3];
    for (int l = 0; l < 3; ++l) {
      RH_CUDA(cudaEventCreateWithFlags(&ev[l], cudaEventDisableTiming));
      RH_CUDA(cudaEventRecord(ev[l], ms[l]));
      RH_CUDA(cudaStreamWaitEvent(st, ev[l], 0));
    }
    cudaEventDestroy(ev0);
    for (int l = 0; l < 3; ++l) cudaEventDestroy(ev[l]);
  } else {
    for (int l = 0; l < 3; ++l) {
      c.m = &w.mw[l];
      mst[l] = solve_mode(c, l, n, LDN, Rl, Rp, Rg, Uh[l], w.G.p + (size_t)l * LDN * LDN, rep.trace[l], o, mo[l]);
      c.m = nullptr;
      if (mst[l] != RHOSVD_OK) {
        merr[l] = g_err;
        break;
      }
      tm.mark(PH_EIG);
    }
  }
  for (int l = 0; l < 3; ++l) {
    if (mst[l] != RHOSVD_OK) {
      cudaDeviceSynchronize();
      for (int q = 0; q < 3; ++q) {
        OC().put(mo[q].Z);
        OC().put(mo[q].W);
        OC().put(mo[q].sigma);
      }
      return fail(mst[l], merr[l]);
    }
  }
  for (int l = 0; l < 3; ++l) {
    res->Z[l] = mo[l].Z;
    res->W[l] = mo[l].W;
    res->sigma[l] = mo[l].sigma;
    res->ranks[l] = mo[l].r;
    rep.ranks[l] = mo[l].r;
    rep.block[l] = mo[l].b;
    rep.iters[l] = mo[l].iters;
    rep.grow_events[l] = mo[l].grows;
    rep.refines[l] = mo[l].refines;
    rep.rho[l] = mo[l].rho;
    rep.tail[l] = std::sqrt(std::max(0.0, mo[l].tail2));
  }
  tm.mark(PH_EIG);
  // ---- optional C2T ALS sweeps on the RHOSVD frames (single GPU)
  for (int sw = 0; sw < als_sweeps; ++sw)
    for (int l = 0; l < 3; ++l) {
      c.m = &w.mw[l];
      const uint64_t seed = o.seed * 0x9E3779B97F4A7C15ull + 0xA15ull * (uint64_t)(3 * sw + l + 1);
      const int s_ = als_update(c, l, n, LDN, Rl, Rp, Uh, w.xip.p, mo, o, seed);
      c.m = nullptr;
      if (s_ != RHOSVD_OK) return s_;
    }
  if (als_sweeps > 0) tm.mark(PH_EIG);
  const int64_t r1 = mo[0].r, r2 = mo[1].r, r3 = mo[2].r;
  const int64_t total = r1 * r2 * r3;

  // host outputs: frames and sigma go back while the core runs; beta chunk by chunk
  BetaD2H bd{nullptr, nullptr, cp};
  CoreChunks chunks;
  if (hin) {
    cudaEvent_t ev;
    RH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    RH_CUDA(cudaEventRecord(ev, st));
    RH_CUDA(cudaStreamWaitEvent(cp, ev, 0));
    cudaEventDestroy(ev);
    for (int l = 0; l < 3; ++l) {
      const int64_t rl = mo[l].r;
      if (rl <= 0) continue;
      RH_CHECK(HC().get((void**)&res->hZ[l], (size_t)LDN * rl * sizeof(double)));
      RH_CHECK(HC().get((void**)&res->hsigma[l], (size_t)rl * sizeof(double)));
      RH_CUDA(cudaMemcpyAsync(res->hZ[l], mo[l].Z, (size_t)LDN * rl * sizeof(double), cudaMemcpyDeviceToHost, cp));
      RH_CUDA(cudaMemcpyAsync(res->hsigma[l], mo[l].sigma, rl * sizeof(double), cudaMemcpyDeviceToHost, cp));
    }
    if (total > 0) {
      RH_CHECK(HC().get((void**)&res->hbeta, (size_t)total * sizeof(double)));
      bd.host = res->hbeta;
      if (!(comm && comm->active())) {  // with a communicator beta is complete only after the all-reduce
        cudaStream_t* ms = mode_streams();
        if (!ms) return fail(RHOSVD_ECUDA, "mode stream creation failed");
        static const int nchunks = [] {  // 16: the exposed D2H of the last chunk is ~140 MB
          const char* e = getenv("RHOSVD_CORE_CHUNKS");
          return e ? std::max(1, atoi(e)) : 16;
        }();
        chunks.count = nchunks;
        chunks.side = ms[1];
        chunks.done = beta_chunk_d2h;
        chunks.ctx = &bd;
      }
    }
  }

  // R-sharded (NCCL): the beta all-reduce overlaps the contraction chunk by chunk
  // RHOSVD_F_ROOT_ONLY_CORE: beta is reduced to rank 0 only (the other ranks' beta holds
  // their partial sums and the accessors refuse it)
  const bool root_only = (o.flags & RHOSVD_F_ROOT_ONLY_CORE) && comm && comm->active();
  const bool beta_here = !root_only || comm->rank == 0;
  res->beta_valid = beta_here;
  BetaAR bar{comm, nullptr, nullptr, root_only};
  bool chunked_ar = false;
  if (!chunks.done && total > 0 && comm && comm->active() && comm->kind == rhosvd_comm::NCCL) {
    cudaStream_t* ms = mode_streams();
    bar.cs = coll_stream();
    if (ms && bar.cs) {
      static const int nchunks = [] {
        const char* e = getenv("RHOSVD_CORE_CHUNKS");
        return e ? std::max(1, atoi(e)) : 8;
      }();
      chunks.count = nchunks;
      chunks.side = ms[1];
      chunks.done = beta_chunk_allreduce;
      chunks.ctx = &bar;
      chunked_ar = true;
    }
  }

  // ---- S6 core (K7): beta = (W1 (.) W2)(xi' o W3)^T, then all-reduce
  tm.mark(PH_CORE);
  cudaEvent_t c0, c1;
  cudaEventCreate(&c0);
  cudaEventCreate(&c1);
  if (total > 0) {
    PhaseTimer dt(st);
    if (dbg_on()) dt.mark(0);
    RH_CHECK(OC().get((void**)&res->beta, (size_t)total * sizeof(double)));
    bd.dev = res->beta;
    bar.beta = res->beta;
    if (dbg_on()) dt.mark(1);
    RH_CHECK(w.W1x.ensure((size_t)r1 * Rp, st));
    if (Rl > 0) {
      RH_CHECK(scale_cols(mo[0].W, Rp, w.xip.p, r1, Rp, w.W1x.p, Rp, st));
      if (dbg_on()) dt.mark(2);
      RH_CHECK(w.corepart.ensure(core_part_doubles(r1, r2, r3, Rl), st));
      RH_CHECK(w.W2x.ensure(core_ws_doubles(r2, Rl, Rp), st));
      if (dbg_on()) dt.mark(3);
      cudaEventRecord(c0, st);
      TL().mark(-1, "core_kr start (stream reached)", st);
      TL().hmark(-1, "core_kr entered");
      RH_CHECK(core_kr(w.W1x.p, Rp, mo[1].W, mo[2].W, Rp, r1, r2, r3, Rl, res->beta, w.W2x.p, w.corepart.p,
                       w.corepart.cap, st, &c.flops, chunks.done ? &chunks : nullptr));
      TL().hmark(-1, "core_kr returned");
      cudaEventRecord(c1, st);
      TL().mark(-1, "core", st);
      if (dbg_on()) {
        dt.mark(4);
        double ms[16] = {0};
        dt.collect(ms);
        fprintf(stderr, "[rhosvd dbg] core phase: malloc beta %.3f, scale %.3f, ensure %.3f, core %.3f ms\n", ms[0],
                ms[1], ms[2], ms[3]);
      }
    } else {
      RH_CUDA(cudaMemsetAsync(res->beta, 0, (size_t)total * sizeof(double), st));
      cudaEventRecord(c0, st);
      cudaEventRecord(c1, st);
      if (chunks.done) RH_CHECK(chunks.done(chunks.ctx, 0, 0, total, st));
    }
    if (chunked_ar) {  // the chunks' all-reduces were queued on the collective stream
      cudaEvent_t ev;
      RH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      RH_CUDA(cudaEventRecord(ev, bar.cs));
      RH_CUDA(cudaStreamWaitEvent(st, ev, 0));
      cudaEventDestroy(ev);
    } else if (root_only) {
      c.tm->mark(PH_COMM);
      RH_CHECK(comm_reduce_root(comm, res->beta, total, st));
    } else {
      RH_CHECK(allreduce(c, res->beta, total));
    }
    if (hin && beta_here && (chunked_ar || !chunks.done)) RH_CHECK(beta_chunk_d2h(&bd, 0, 0, total, st));
    tm.mark(PH_CORE);
    RH_CHECK(k_sumsq(res->beta, total, w.part.p, w.scal.p + 12, st));
  } else {
    cudaEventRecord(c0, st);
    cudaEventRecord(c1, st);
  }
  tm.mark(-1);
  double bn2 = 0.0;
  if (total > 0) RH_CHECK(d2h_wait(&bn2, w.scal.p + 12, sizeof(double), st));
  RH_CUDA(cudaStreamSynchronize(st));
  if (cp) RH_CUDA(cudaStreamSynchronize(cp));
  RH_CUDA(cudaGetLastError());
  rep.beta_norm = beta_here ? std::sqrt(bn2) : std::nan("");
  double st1 = 0.0, st2 = 0.0;
  for (int l = 0; l < 3; ++l) {
    st1 += rep.tail[l];
    st2 += rep.tail[l] * rep.tail[l];
  }
  rep.bound_paper = rep.xi_norm * st1;  // Thm. 2.2
  rep.bound_ns = rep.xi_norm * std::sqrt(st2);  // reading A12
  tm.collect(rep.ms);
  float gms = 0.f, cms = 0.f;
  if (streamed) gms = gram_ms_streamed;
  else cudaEventElapsedTime(&gms, g0, g1);
  cudaEventElapsedTime(&cms, c0, c1);
  rep.gram_ms = gms;
  rep.core_ms = cms;
  cudaEventDestroy(g0);
  cudaEventDestroy(g1);
  cudaEventDestroy(c0);
  cudaEventDestroy(c1);
  rep.gemm_flops = c.flops;
  rep.launches = g_launches;
  TL().dump();
  return RHOSVD_OK;
}

static int c2t_entry(const double* U1, const double* U2, const double* U3, int64_t ldu, const double* xi, int64_t n,
                     int64_t R_local, const rhosvd_opts* opts, rhosvd_comm* comm, rhosvd_stream stream,
                     rhosvd_result** out, bool host, int als_sweeps = 0);

int rhosvd_c2t_als(const double* U1, const double* U2, const double* U3, int64_t ldu, const double* xi, int64_t n,
                   int64_t R_local, const rhosvd_opts* opts, int32_t sweeps, rhosvd_comm* comm, rhosvd_stream stream,
                   rhosvd_result** out) {
  if (out) *out = nullptr;
  if (sweeps < 0) return fail(RHOSVD_EINVAL, "sweeps must be >= 0");
  if (comm && comm->active()) return fail(RHOSVD_EINVAL, "ALS sweeps: single GPU only (comm must be NULL)");
  return c2t_entry(U1, U2, U3, ldu, xi, n, R_local, opts, comm, stream, out, false, sweeps);
}

int rhosvd_c2t(const double* U1, const double* U2, const double* U3, int64_t ldu, const double* xi, int64_t n,
               int64_t R_local, const rhosvd_opts* opts, rhosvd_comm* comm, rhosvd_stream stream,
               rhosvd_result** out) {
  return c2t_entry(U1, U2, U3, ldu, xi, n, R_local, opts, comm, stream, out, false);
}

int rhosvd_c2t_host(const double* U1, const double* U2, const double* U3, int64_t ldu, const double* xi, int64_t n,
                    int64_t R_local, const rhosvd_opts* opts, rhosvd_comm* comm, rhosvd_stream stream,
                    rhosvd_result** out) {
  return c2t_entry(U1, U2, U3, ldu, xi, n, R_local, opts, comm, stream, out, true);
}

int rhosvd_result_host_frame(const rhosvd_result* r, int mode, const double** Z, int64_t* ldz) {
  if (!r || !Z || !ldz || mode < 0 || mode > 2) return fail(RHOSVD_EINVAL, "bad args");
  if (r->ranks[mode] > 0 && !r->hZ[mode]) return fail(RHOSVD_EINVAL, "no host outputs (use rhosvd_c2t_host)");
  *Z = r->hZ[mode];
  *ldz = r->ldz;
  return RHOSVD_OK;
}
int rhosvd_result_host_sigma(const rhosvd_result* r, int mode, const double** s, int64_t* count) {
  if (!r || !s || !count || mode < 0 || mode > 2) return fail(RHOSVD_EINVAL, "bad args");
  if (r->ranks[mode] > 0 && !r->hsigma[mode]) return fail(RHOSVD_EINVAL, "no host outputs (use rhosvd_c2t_host)");
  *s = r->hsigma[mode];
  *count = r->ranks[mode];
  return RHOSVD_OK;
}
int rhosvd_result_host_core(const rhosvd_result* r, const double** beta) {
  if (!r || !beta) return fail(RHOSVD_EINVAL, "bad args");
  if (!r->beta_valid) return fail(RHOSVD_EINVAL, "RHOSVD_F_ROOT_ONLY_CORE: beta is on rank 0 only");
  if ((int64_t)r->ranks[0] * r->ranks[1] * r->ranks[2] > 0 && !r->hbeta)
    return fail(RHOSVD_EINVAL, "no host outputs (use rhosvd_c2t_host)");
  *beta = r->hbeta;
  return RHOSVD_OK;
}

}  // extern "C"

static int c2t_entry(const double* U1, const double* U2, const double* U3, int64_t ldu, const double* xi, int64_t n,
                     int64_t R_local, const rhosvd_opts* opts, rhosvd_comm* comm, rhosvd_stream stream,
                     rhosvd_result** out, bool host, int als_sweeps) {
  if (!out) return fail(RHOSVD_EINVAL, "out is null");
  *out = nullptr;
  if (!opts) return fail(RHOSVD_EINVAL, "opts is null");
  if (n < 1 || R_local < 0 || ldu < n) return fail(RHOSVD_EINVAL, "need n >= 1, R_local >= 0, ldu >= n");
  if (R_local > 0 && (!U1 || !U2 || !U3 || !xi)) return fail(RHOSVD_EINVAL, "null input pointer");
  const rhosvd_opts& o = *opts;
  if (o.rank_mode == RHOSVD_EPS) {
    if (!(o.eps > 0.0 && o.eps < 1.0)) return fail(RHOSVD_EINVAL, "eps must lie in (0, 1)");
  } else if (o.rank_mode == RHOSVD_FIXED_RANK) {
    if (o.r[0] < 1 || o.r[1] < 1 || o.r[2] < 1) return fail(RHOSVD_EINVAL, "fixed ranks must be >= 1");
  } else {
    return fail(RHOSVD_EINVAL, "unknown rank_mode");
  }
  if (n > 16384) return fail(RHOSVD_EINVAL, "n > 16384 not supported");
  RH_CHECK(device_guard());
  std::lock_guard<std::mutex> lk(g_mu);
  cudaStream_t st = (cudaStream_t)stream;
  StreamOrder order(st);
  static bool pool_set = false;
  if (!pool_set) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_set = true;
  }
  auto* res = new rhosvd_result();
  const double* U[3] = {U1, U2, U3};
  HostIn hin{{U1, U2, U3}, xi};
  int s = c2t_impl(U, ldu, xi, n, R_local, o, comm, st, res, host ? &hin : nullptr, als_sweeps);
  if (s != RHOSVD_OK) {
    std::string msg = g_err;
    rhosvd_result_free(res);
    g_err = msg;
    return s;
  }
  *out = res;
  return RHOSVD_OK;
}

extern "C" {

// ---------------------------------------------------------------- kernel-level entry points
int rhosvd_gram(const double* U, int64_t ldu, int64_t n, int64_t R, double* G, int64_t ldg, rhosvd_stream stream) {
  if (!U || !G || n < 1 || R < 0 || ldu < n || ldg < n) return fail(RHOSVD_EINVAL, "bad args");
  if ((ldu & 1) || ((uintptr_t)U & 15)) return fail(RHOSVD_EINVAL, "gram: ldu must be even, U 16B-aligned");
  RH_CHECK(device_guard());
  std::lock_guard<std::mutex> lk(g_mu);
  StreamOrder order((cudaStream_t)stream);
  GemmArgs g;
  g.M = n; g.N = n; g.K = R; g.A = U; g.lda = ldu; g.a_k = false; g.B = U; g.ldb = ldu; g.b_k = false;
  g.C = G; g.ldc = ldg; g.upper_sym = true;
  g_launches = 0;
  return gemm(g, WS().gsc, (cudaStream_t)stream);
}

int rhosvd_dgemm(char ta, char tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                 const double* B, int64_t ldb, double beta, double* C, int64_t ldc, rhosvd_stream stream) {
  if (!A || !B || !C || M < 0 || N < 0 || K < 0) return fail(RHOSVD_EINVAL, "bad args");
  if ((lda & 1) || (ldb & 1) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15))
    return fail(RHOSVD_EINVAL, "dgemm: lda/ldb must be even and A/B 16B-aligned");
  RH_CHECK(device_guard());
  std::lock_guard<std::mutex> lk(g_mu);
  StreamOrder order((cudaStream_t)stream);
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
  g.alpha = alpha; g.beta = beta;
  // op(A)(m,k): 'N' -> A[k*lda + m] (m contiguous), 'T' -> A[m*lda + k] (k contiguous)
  g.a_k = (ta == 'T' || ta == 't');
  // op(B)(k,n): 'N' -> B[n*ldb + k] (k contiguous), 'T' -> B[k*ldb + n]
  g.b_k = !(tb == 'T' || tb == 't');
  g_launches = 0;
  return gemm(g, WS().gsc, (cudaStream_t)stream);
}

int rhosvd_syevj(int64_t b, double* A, int64_t lda, double* lambda, double* V, int64_t ldv, double tol,
                 int32_t* sweeps_out, rhosvd_stream stream) {
  if (!A || !lambda || !V || b < 0 || lda < b || ldv < b) return fail(RHOSVD_EINVAL, "bad args");
  RH_CHECK(device_guard());
  std::lock_guard<std::mutex> lk(g_mu);
  StreamOrder order((cudaStream_t)stream);
  int sw = 0;
  RH_CHECK(syevj(b, A, lda, lambda, V, ldv, tol > 0 ? tol : 1e-15, 1e-300, 80, WS().mw[0].dws, (cudaStream_t)stream, &sw));
  if (sweeps_out) *sweeps_out = sw;
  return RHOSVD_OK;
}

int rhosvd_chol_inv(int64_t b, const double* S, int64_t lds, double shift, double* Bp, int64_t ldb,
                    rhosvd_stream stream) {
  if (!S || !Bp || b < 0 || lds < b || ldb < b || !(shift >= 0.0)) return fail(RHOSVD_EINVAL, "bad args");
  RH_CHECK(device_guard());
  std::lock_guard<std::mutex> lk(g_mu);
  StreamOrder order((cudaStream_t)stream);
  return chol_inv_scaled(b, S, lds, shift, Bp, ldb, WS().mw[0].dws, (cudaStream_t)stream);
}

int rhosvd_core(const double* W1, const double* W2, const double* W3, int64_t ldw, const double* xi, int64_t r1,
                int64_t r2, int64_t r3, int64_t R, double* beta, rhosvd_stream stream) {
  if (!W1 || !W2 || !W3 || !xi || !beta || r1 < 0 || r2 < 0 || r3 < 0 || R < 0 || ldw < R)
    return fail(RHOSVD_EINVAL, "bad args");
  if ((ldw & 1) || ((uintptr_t)W1 & 15) || ((uintptr_t)W2 & 15) || ((uintptr_t)W3 & 15))
    return fail(RHOSVD_EINVAL, "core: ldw must be even, W 16B-aligned");
  RH_CHECK(device_guard());
  std::lock_guard<std::mutex> lk(g_mu);
  cudaStream_t st = (cudaStream_t)stream;
  StreamOrder order(st);
  Workspace& w = WS();
  int64_t ldx = round_up(std::max<int64_t>(R, 2), 2);
  RH_CHECK(w.W1x.ensure((size_t)r1 * ldx + 64, st));
  RH_CHECK(scale_cols(W1, ldw, xi, r1, R, w.W1x.p, ldx, st));
  size_t total = (size_t)r1 * r2 * r3;
  RH_CHECK(w.corepart.ensure(core_part_doubles(r1, r2, r3, R), st));
  RH_CHECK(w.W2x.ensure(core_ws_doubles(r2, R, ldw), st));
  return core_kr(w.W1x.p, ldx, W2, W3, ldw, r1, r2, r3, R, beta, w.W2x.p, w.corepart.p, w.corepart.cap, st,
                 nullptr);
}

}  // extern "C"
