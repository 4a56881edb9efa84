// C ABI of libmpid.so (declared in include/mpid.h): handle, workspace layout,
// host orchestration of the kernels, NCCL (dlopen'ed) collectives, CUDA-graph
// capture of the k-step loop and per-stage device timing.
#include "../../include/mpid.h"
#include "mpid_internal.cuh"

#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <string>
#include <tuple>
#include <vector>

using namespace mpid;

#include <mutex>
cudaError_t mpid::smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// ----------------------------------------------------------------------------
// NCCL through dlopen (the process's libnccl.so.2, e.g. PyTorch's)
// ----------------------------------------------------------------------------
namespace {
typedef int nccl_result_t;
struct NcclApi {
  bool ok = false;
  nccl_result_t (*GetUniqueId)(void*) = nullptr;
  nccl_result_t (*CommInitRank)(void**, int, /*ncclUniqueId by value*/ ...) = nullptr;
  nccl_result_t (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  nccl_result_t (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(nccl_result_t) = nullptr;
};
struct NcclUid { char internal[128]; };
typedef nccl_result_t (*CommInitRankFn)(void**, int, NcclUid, int);

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.GetUniqueId = (nccl_result_t(*)(void*))dlsym(h, "ncclGetUniqueId");
  api.CommInitRank = (nccl_result_t(*)(void**, int, ...))dlsym(h, "ncclCommInitRank");
  api.AllReduce = (nccl_result_t(*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
      h, "ncclAllReduce");
  api.CommDestroy = (nccl_result_t(*)(void*))dlsym(h, "ncclCommDestroy");
  api.GetErrorString = (const char* (*)(nccl_result_t))dlsym(h, "ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy;
  return api;
}
constexpr int NCCL_FLOAT64 = 8;
constexpr int NCCL_SUM = 0, NCCL_MAX = 2;

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t AD, S, U, F, Vop, Fop, R, part, red, xr, norms, perm, scal3, sc, maxpart, rpart;
  size_t AI, Q1, G1, G2, W, tpart, Rd, T, Pw, epart, Tp, Ik, Rinv, py, pvec, gpart, G, Gc, misc;
  size_t cmaxd, cmaxq, ozs, ozt, ozpart, rsc, fsc;   // fp64 stage on the int8 tensor cores (k_ozaki.cu)
  size_t cand;                                      // fused reduce + reflector: block candidates, ticket
  size_t total;
};

int num_sms() {   // of the current device (cached per device ordinal)
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = sms > 0 ? sms : 148;
  }
  return cache[dev];
}

constexpr int PW_NBLK = 64;   // row blocks of the transposed GEMV (power iteration)

int64_t m_pad_of(int64_t m_local) {
  const int64_t T = PASS_TILE_G * RG;
  return std::max<int64_t>(T, (m_local + T - 1) / T * T);
}
// rows of per-CTA partials the panel pass may write: the FFMA pass one per CTA (grid.x <= SMs),
// the tcgen05 pass one per CTA row half (grid.x <= SMs)
int pass_gx_cap() { return 2 * num_sms(); }
int round_gy(int64_t m_pad, int64_t n) {
  const int64_t gx = (n + 31) / 32;
  const int64_t ngroups = m_pad / 8;
  // one wave: k_round holds 2 CTAs per SM (fp16 / fp32: 128 registers x 256 threads; the
  // fp64 variant fits 3), and every CTA streams the same number of row tiles, so a grid
  // of more than 2 x SMs leaves a tail wave of full-length CTAs (608 CTAs = 2.05 waves)
  int64_t gy = std::max<int64_t>(1, (2 * num_sms()) / gx);
  gy = std::min<int64_t>(gy, std::max<int64_t>(1, ngroups / 8));
  return (int)std::min<int64_t>(gy, 4096);
}
int tsmm_splits(int64_t k1, int64_t n1, int64_t m) {
  // k_dgemm CTA tile <= 128 x 128, one CTA per SM, equal-work CTAs: pick the split count
  // in [2 waves, 6 waves] whose last wave is the fullest (ties -> fewer splits)
  const int64_t sms = num_sms();
  const int64_t tiles = ((k1 + 127) / 128) * ((n1 + 127) / 128);
  const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(512, m / 512));
  const int64_t s0 = std::min<int64_t>(cap, std::max<int64_t>(1, (2 * sms + tiles - 1) / tiles));
  int64_t best = s0;
  double best_eff = -1.0;
  for (int64_t s = s0; s <= std::min<int64_t>(cap, 3 * s0); ++s) {
    const int64_t ctas = tiles * s, waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
  }
  return (int)best;
}

// split-K partials buffer: covers every (k1 <= k, n1 <= n) product the coefficients use;
// the call sites clamp the split count to it (splits_for)
size_t tpart_doubles(int64_t m_local, int64_t n, int64_t k) {
  size_t need = 0;
  for (int64_t k1 : {k, std::min<int64_t>(k, 128)})
    for (int64_t n1 : {k1, n, std::max<int64_t>(1, n - k1)})
      need = std::max<size_t>(need, (size_t)tsmm_splits(k1, n1, m_local) * k1 * n1);
  // cap the split-K room at 16M doubles, but never below one unsplit product (splits = 1
  // writes k1 * n1 doubles; k x max(k, n) covers every product the coefficients use)
  const size_t floor1 = (size_t)k * (size_t)std::max<int64_t>(k, n);
  return std::max(std::min<size_t>(need, (size_t)1024 * 128 * 128), floor1);
}
int splits_for(int64_t k1, int64_t n1, int64_t m, size_t cap) {
  const int64_t s = tsmm_splits(k1, n1, m);
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, (int64_t)(cap / (size_t)(k1 * n1))));
}

// rows per host-streamed block of A_D (a multiple of the rounding kernel's 256-row tile)
int64_t stream_rows(int64_t m_local, int64_t n) {
  // two staging blocks of <= 1 GiB each
  int64_t r = ((int64_t)1 << 27) / std::max<int64_t>(n, 1);
  r = std::max<int64_t>(256, r / 256 * 256);
  return std::min<int64_t>(r, m_pad_of(m_local));
}

// sbytes: 4 = room for fp16/fp32 storage with fp32 working vectors; 8 = also the fp64 QRCP
// host_AD: 0 = A_D in device memory, 1 = a host A_D copied whole into the workspace,
// 2 = a host A_D streamed in row blocks through two staging buffers (plus a k x n block of W)
Layout layout(int64_t m_local, int64_t n, int64_t k, int host_AD, int sbytes) {
  Layout L{};
  const int64_t mp = m_pad_of(m_local);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
  L.AD = take(host_AD == 1 ? (size_t)m_local * n * 8
                            : host_AD == 2 ? (size_t)2 * stream_rows(m_local, n) * n * 8 + (size_t)k * n * 8 + 4096 * 8
                                           : 0);
  L.S = take((size_t)mp * n * sbytes);
  L.U = take((size_t)NSLOT * mp * sbytes);
  L.F = take((size_t)NSLOT * n * sbytes);
  L.Vop = take(tc_vop_bytes(mp, NB_MAX));            // tcgen05 pass: the panel's V operand (fp16 hi / lo)
  L.Fop = take(tc_fop_bytes((int)n, NB_MAX));         //   and the step's F operand
  L.R = take((size_t)k * n * sbytes);
  L.part = take((size_t)pass_gx_cap() * 2 * n * 8);
  L.red = take((size_t)3 * n * 8);
  L.xr = take((size_t)n * 8);
  L.norms = take((size_t)(n + 2) * 8);
  L.perm = take((size_t)n * 4);
  L.scal3 = take((size_t)3 * k * 8);
  L.sc = take(sizeof(DevScalars));
  L.maxpart = take(1024 * 8);
  L.rpart = take(((size_t)round_gy(mp, n) * n + (size_t)round_gy(mp, n) * ((n + 31) / 32)) * 8);
  L.AI = take((size_t)m_local * k * 8);
  L.Q1 = take((size_t)m_local * k * 8);
  L.G1 = take((size_t)k * k * 8);
  L.G2 = take((size_t)k * k * 8);
  L.W = take((size_t)k * n * 8);
  L.tpart = take(tpart_doubles(m_local, n, k) * 8);
  L.Rd = take((size_t)k * n * 8);
  L.T = take((size_t)k * n * 8);
  L.Pw = take((size_t)k * n * 8);
  L.epart = take((size_t)((m_local + 127) / 128) * ((n + 127) / 128) * 8);
  L.Tp = take(ew_tpack_doubles(n, k) * 8);                            // error kernel: packed T slabs
  L.Ik = take((size_t)k * k * 8);
  L.Rinv = take((size_t)k * k * 8);
  L.py = take((size_t)m_local * 8);                                  // power iteration: y = E x
  L.pvec = take((size_t)(3 * n + 2 * k + 256 + PW_NBLK * (n + k)) * 8);  // x, z, v, w, u, est, partials (n + k cols)
  L.gpart = take(gram_part_doubles(mp / 8, (int)n, num_sms()) * 8);  // Gram pivoting: tile partials
  L.G = take((size_t)n * n * 8);                                      //   and G = A_L^T A_L
  L.Gc = take((size_t)n * n * 8);                                     //   Schur-complement working copy
  L.cmaxd = take((size_t)n * 8);                                      // A_D column max |a|
  L.cmaxq = take(128 * 8);                                            // Q1 column max |q|
  L.ozs = take(oz_slice_bytes(m_local));                              // A-operand slices (Q1 or A_I)
  L.ozt = take(oz_tslice_bytes(n));                                   // T's slices
  L.ozpart = take(oz_part_doubles(num_sms()) * 8);                    // row-group partials of [G2 | W]
  L.rsc = take((size_t)((m_local + 127) / 128 * 128) * 8);            // per-row scales of A_I
  L.fsc = take((size_t)(n + 64) * 8);                                 // per-column scales of T
  L.cand = take((size_t)(5 * ((n + 31) / 32 + 1)) * 8 + 64);
  L.misc = take(1024);
  L.total = off;
  return L;
}
}  // namespace

struct mpid_ctx {
  // geometry
  const double* AD = nullptr;   // device A_D (user's or the workspace copy)
  int64_t m_global = 0, m_local = 0, row_offset = 0, n = 0, ld = 0, m_pad = 0;
  int32_t rank = 0, nranks = 1;
  void* comm = nullptr;
  bool loop = false;              // comm is a LoopComm (id_loopback_create)
  cudaStream_t st = nullptr;      // current enqueue stream (user's, or cap during graph capture)
  cudaStream_t user_st = nullptr; // the caller's stream
  cudaStream_t cap = nullptr;     // internal non-blocking stream: graph capture and replay
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  Layout L{};
  int64_t k_cap = 0;
  int host_AD = 0;                // 0 device A_D, 1 host A_D copied whole, 2 host A_D streamed
  const double* AD_host = nullptr; // mode 2: the caller's host A_D (ld_host)
  int64_t ld_host = 0, srows = 0;
  int srows_log2 = 0;              // mode 2: block rows 2^srows_log2 (0 = automatic, ~1 GiB blocks)
  double* stage[2] = {nullptr, nullptr};
  double* Wb = nullptr;            // mode 2: one row block's W partial sum
  double* sacc = nullptr;          // mode 2: per-block scalars (max |a|, error^2)
  cudaStream_t cps = nullptr;      // mode 2: copy stream
  cudaEvent_t copied[2]{}, freed[2]{};
  int sbytes = 4;                 // workspace layout: 8 = sized for the fp64 QRCP too
  // device pointers (U, F, R in the working precision: fp32, fp64 for ID_FP64)
  void* S = nullptr;
  void *U = nullptr, *F = nullptr, *R = nullptr;
  void *Vop = nullptr, *Fop = nullptr;
  alignas(64) unsigned char tmapS[128];      // CUtensorMap of fp16 S (tcgen05 pass, 128 x 128 unit tiles)
  alignas(64) unsigned char tmapC[128];      //   and of one column x 128 rows (the pass's pivot column)
  int tmap_ok = -1;
  alignas(64) unsigned char tmapG[128];      // CUtensorMap of fp16 S for the Gram kernel
  int tmapG_ok = -1;
  double *gpart = nullptr, *G = nullptr, *Gc = nullptr;
  double *part = nullptr, *red = nullptr, *xr = nullptr, *norms = nullptr, *beta = nullptr,
         *cvec = nullptr, *tau = nullptr, *maxpart = nullptr, *rpart = nullptr;
  int* perm = nullptr;
  DevScalars* sc = nullptr;
  double *AI = nullptr, *Q1 = nullptr, *G1 = nullptr, *G2 = nullptr, *W = nullptr, *tpart = nullptr,
         *Rd = nullptr, *T = nullptr, *Pw = nullptr, *epart = nullptr, *Tp = nullptr, *Ik = nullptr, *Rinv = nullptr,
         *py = nullptr, *pvec = nullptr;
  double normAD_spec = -1.0;   // cached ||A_D||_2 (power iteration), < 0 = not yet
  int* info = nullptr;
  double* err2 = nullptr;
  unsigned long long *cmaxd = nullptr, *cmaxq = nullptr;   // column max |x| bit patterns
  void *ozs = nullptr, *ozt = nullptr;
  double *ozpart = nullptr, *rsc = nullptr, *fsc = nullptr;
  int fp64_engine = 0;            // 0 auto, 1 DMMA, 2 int8 Ozaki (id_set_fp64_engine)
  bool have_cmaxd = false;        // cmaxd holds this A_D's column maxima (set by the round)
  double* cand = nullptr;         // k_reduce_reflect: per-block candidates
  unsigned int* ticket = nullptr; //   and its last-block counter
  // state
  int fmt = 0;
  int k_out = 0;
  int qr_status = 0;
  bool have_qr = false, have_coef = false, have_gram = false, have_sketch = false;
  std::vector<int> perm_host;
  DevScalars sc_host{};
  std::string err;
  // graphs keyed by (fmt, scaling, k_max, nb, eps bits, profile)
  // graphs keyed by (fmt, scaling, k_max, nb * 4 + formation, eps bits, profile, sketch l << 32 | seed)
  std::map<std::tuple<int, int, int, int, uint64_t, int, uint64_t>, cudaGraphExec_t> graphs;
  std::map<std::tuple<int, int, int, int, uint64_t, int, uint64_t>, int64_t> graph_launches;
  std::map<uint64_t, std::pair<cudaGraphExec_t, int>> cgraphs;   // id_coeffs_fp64 graphs per (mode, k)
  // sketched pivoting (formation 4): sketch rows l (lw rounded to 128), seed, Omega^T's tensor map
  int sk_l = 0, sk_lw = 0;
  uint32_t sk_seed = 0;
  alignas(64) unsigned char tmapO[128];
  cudaEvent_t ev[8]{};
  std::vector<cudaEvent_t> pass_ev;
  int64_t pass_launches = 0, kernel_launches = 0;
  id_stats stats{};
};

static id_status fail(mpid_ctx* h, id_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  return s;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(h, ID_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                 \
  } while (0)

static cudaError_t rec(mpid_ctx* h, cudaEvent_t e) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(h->st, &cs);
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, h->st, cudaEventRecordExternal)
                                             : cudaEventRecord(e, h->st);
}

// ----------------------------------------------------------------------------
// Loopback "communicator": nranks handles on ONE device, each driven by its own host
// thread (tests of the row-sharded path on one GPU; SURVEY §4 tests/dist (i)).  An
// allreduce synchronises the caller's stream, copies its buffer to a host slot, waits
// for all ranks (generation barrier), and the last arriver reduces the slots in rank
// order 0..P-1 (SUM or MAX), so every rank receives the same bits.  Not capturable in
// a CUDA graph: handles on a loopback group run the step loop eagerly.
// ----------------------------------------------------------------------------
#include <condition_variable>
#include <set>
struct LoopComm {
  int nranks = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<std::vector<double>> slot;
  std::vector<double> result;
  int64_t calls = 0;                // completed collectives (diagnostics)
};
static std::mutex g_loop_mu;
static std::set<void*> g_loops;
static bool is_loop(void* c) {
  std::lock_guard<std::mutex> lk(g_loop_mu);
  return c && g_loops.count(c);
}

static id_status loop_allreduce(mpid_ctx* h, double* buf, size_t count, int op) {
  LoopComm* L = (LoopComm*)h->comm;
  std::vector<double> mine(count);
  // copies on the handle's own stream, synchronised: a plain cudaMemcpy from pageable memory
  // may return before its DMA lands, and the handle's stream need not sync with the legacy one
  CK(cudaMemcpyAsync(mine.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  std::vector<double> res;
  {
    std::unique_lock<std::mutex> lk(L->mu);
    const uint64_t my_gen = L->gen;
    L->slot[h->rank] = std::move(mine);
    if (++L->arrived == L->nranks) {
      L->result = L->slot[0];
      for (int r = 1; r < L->nranks; ++r) {
        if (L->slot[r].size() != count) {
          L->result.assign(count, NAN);   // mismatched collective: every rank sees NaN
          break;
        }
        for (size_t i = 0; i < count; ++i)
          L->result[i] = op == NCCL_MAX ? std::max(L->result[i], L->slot[r][i]) : L->result[i] + L->slot[r][i];
      }
      L->arrived = 0;
      L->calls++;
      L->gen++;
      L->cv.notify_all();
    } else {
      if (!L->cv.wait_for(lk, std::chrono::seconds(120), [&] { return L->gen != my_gen; }))
        return fail(h, ID_ERR_NCCL, "loopback allreduce: rank %d timed out waiting for the others", h->rank);
    }
    res = L->result;
  }
  if (res.size() != count) return fail(h, ID_ERR_NCCL, "loopback allreduce: size mismatch");
  CK(cudaMemcpyAsync(buf, res.data(), count * sizeof(double), cudaMemcpyHostToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));   // `res` goes out of scope
  return ID_OK;
}

static id_status allreduce(mpid_ctx* h, double* buf, size_t count, int op) {
  // a communicator given at nranks == 1 is still used (the NCCL-in-graph test)
  if (h->nranks <= 1 && !h->comm) return ID_OK;
  if (h->loop) return loop_allreduce(h, buf, count, op);
  NcclApi& api = nccl();
  if (!api.ok) return fail(h, ID_ERR_NCCL, "libnccl.so.2 not available");
  const nccl_result_t r = api.AllReduce(buf, buf, count, NCCL_FLOAT64, op, h->comm, h->st);
  if (r != 0)
    return fail(h, ID_ERR_NCCL, "ncclAllReduce: %s", api.GetErrorString ? api.GetErrorString(r) : "?");
  return ID_OK;
}

// the counter-based sign generator's stream base (synth.counter_sign, stream 7): SplitMix64
// of seed * 1000003 + 7 * 7919 + 12345 — generator plumbing, no arithmetic of the method
static uint64_t sketch_base(uint32_t seed) {
  uint64_t z = (uint64_t)seed * 1000003ull + 7ull * 7919ull + 12345ull;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// (Re)carve the workspace for working precision sbytes (4: fp16/fp32 QRCP, 8: also the
// fp64 QRCP) at the largest k it holds.  A_D's copy (offset 0) and S's offset are the
// same in both layouts; every pointer after them moves, so captured graphs are dropped.
static id_status relayout(mpid_ctx* h, int sbytes) {
  const int64_t m_local = h->m_local, n = h->n;
  int64_t lo = 0, hi = std::min<int64_t>(n, h->m_global);  // largest k with layout(k) <= ws_bytes
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (layout(m_local, n, mid, h->host_AD, sbytes).total <= h->ws_bytes) lo = mid;
    else hi = mid - 1;
  }
  if (lo <= 0) return fail(h, ID_ERR_DIM, "workspace too small for %s", sbytes == 8 ? "ID_FP64" : "k = 1");
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  h->graphs.clear();
  h->graph_launches.clear();
  for (auto& kv : h->cgraphs) cudaGraphExecDestroy(kv.second.first);
  h->cgraphs.clear();
  // every buffer moves: results held in the old carve (QR, coefficients, Gram, sketch) are gone
  h->have_qr = h->have_coef = h->have_gram = h->have_sketch = false;
  h->perm_host.clear();
  h->sbytes = sbytes;
  const int64_t kmax = lo;
  h->k_cap = kmax;
  h->L = layout(m_local, n, kmax, h->host_AD, sbytes);
  const Layout& L = h->L;
  char* w = h->ws;
  if (h->host_AD == 2) {
    h->srows = stream_rows(m_local, n);
    if (h->srows_log2 >= 8) h->srows = std::min<int64_t>(h->srows, (int64_t)1 << h->srows_log2);
    h->stage[0] = (double*)(w + L.AD);
    h->stage[1] = h->stage[0] + (size_t)h->srows * n;
    h->Wb = h->stage[1] + (size_t)h->srows * n;
    h->sacc = h->Wb + (size_t)kmax * n;
  }
  h->S = w + L.S;
  h->U = w + L.U;
  h->F = w + L.F;
  h->Vop = w + L.Vop;
  h->Fop = w + L.Fop;
  h->tmap_ok = encode_tmap_S(h->tmapS, h->S, h->m_pad / 8, (int)n, 0) |
               encode_tmap_S(h->tmapC, h->S, h->m_pad / 8, (int)n, 1);
  h->tmapG_ok = encode_tmap_gram(h->tmapG, h->S, h->m_pad / 8, (int)n);
  h->gpart = (double*)(w + L.gpart);
  h->G = (double*)(w + L.G);
  h->Gc = (double*)(w + L.Gc);
  h->R = w + L.R;
  h->part = (double*)(w + L.part);
  h->red = (double*)(w + L.red);
  h->xr = (double*)(w + L.xr);
  h->norms = (double*)(w + L.norms);
  h->perm = (int*)(w + L.perm);
  h->beta = (double*)(w + L.scal3);
  h->cvec = h->beta + kmax;
  h->tau = h->cvec + kmax;
  h->sc = (DevScalars*)(w + L.sc);
  h->maxpart = (double*)(w + L.maxpart);
  h->rpart = (double*)(w + L.rpart);
  h->AI = (double*)(w + L.AI);
  h->Q1 = (double*)(w + L.Q1);
  h->G1 = (double*)(w + L.G1);
  h->G2 = (double*)(w + L.G2);
  h->W = (double*)(w + L.W);
  h->tpart = (double*)(w + L.tpart);
  h->Rd = (double*)(w + L.Rd);
  h->T = (double*)(w + L.T);
  h->Pw = (double*)(w + L.Pw);
  h->epart = (double*)(w + L.epart);
  h->Tp = (double*)(w + L.Tp);
  h->Ik = (double*)(w + L.Ik);
  h->Rinv = (double*)(w + L.Rinv);
  h->py = (double*)(w + L.py);
  h->pvec = (double*)(w + L.pvec);
  h->info = (int*)(w + L.misc);
  h->err2 = (double*)(w + L.misc + 64);
  h->cmaxd = (unsigned long long*)(w + L.cmaxd);
  h->cmaxq = (unsigned long long*)(w + L.cmaxq);
  h->ozs = w + L.ozs;
  h->ozt = w + L.ozt;
  h->ozpart = (double*)(w + L.ozpart);
  h->rsc = (double*)(w + L.rsc);
  h->fsc = (double*)(w + L.fsc);
  h->have_cmaxd = false;
  h->cand = (double*)(w + L.cand);
  h->ticket = (unsigned int*)(w + L.cand + (size_t)(5 * ((n + 31) / 32 + 1)) * 8);
  h->normAD_spec = -1.0;
  // zero U (padding rows must stay 0); S is fully written by the rounding kernel
  if (cudaMemsetAsync(h->U, 0, (size_t)NSLOT * h->m_pad * sbytes, h->st) != cudaSuccess ||
      // the V operand's unused K columns are multiplied by zero F entries: keep them finite
      cudaMemsetAsync(h->Vop, 0, tc_vop_bytes(h->m_pad, NB_MAX), h->st) != cudaSuccess)
    return fail(h, ID_ERR_CUDA, "workspace memset failed");
  return ID_OK;
}
// the engine of the fp64 ID step's two large GEMMs (W = Q1^T A_J with G2, and the error):
// 2 = the int8 tensor cores by the Ozaki scheme (k_ozaki.cu: k <= 128, a device-resident
// A_D whose column maxima the round recorded, at least one J column), 1 = DMMA (k_fp64.cu).
// -1 = the int8 engine was requested and does not apply.
static int fp64_engine(const mpid_ctx* h, int k, bool error_stage) {
  const bool oz_ok = h->host_AD != 2 && h->have_cmaxd && oz_fits(h->n, k, num_sms());
  if (h->fp64_engine == 1) return 1;
  if (h->fp64_engine == 2) return oz_ok ? 2 : -1;
  static const int env = getenv("MPID_FP64_ENGINE") ? atoi(getenv("MPID_FP64_ENGINE")) : 0;   // A/B measurements
  if (env == 1) return 1;
  if (env == 2) return oz_ok ? 2 : 1;
  // auto: int8 from 32768 rows per shard (C4: error 9.2 vs 14.1 ms, coefficients 14.8 vs
  // 19.6 ms); below that the DMMA kernels' shorter launches win
  (void)error_stage;
  return (oz_ok && h->m_local >= 32768) ? 2 : 1;
}
// the layout a call in format fmt needs
static id_status ensure_layout(mpid_ctx* h, int fmt) {
  const int sb = fmt == ID_FP64 ? 8 : 4;
  return h->sbytes == sb ? ID_OK : relayout(h, sb);
}

extern "C" {

const char* id_version(void) { return "mpid 0.1 (sm_100a; arXiv 2012.00706 mixed-precision ID)"; }

size_t id_workspace_bytes(int64_t m_local, int64_t n, int32_t k_max, int32_t nb, id_format fmt,
                          int32_t host_AD) {
  (void)nb;
  if (m_local <= 0 || n <= 0 || k_max <= 0) return 0;
  return layout(m_local, n, k_max, host_AD, fmt == ID_FP64 ? 8 : 4).total;
}

id_status id_create(id_handle* hp, const double* A_D, int64_t m_global, int64_t m_local,
                    int64_t row_offset, int64_t n, int64_t ld, void* workspace, size_t ws_bytes,
                    void* nccl_comm, int32_t rank, int32_t nranks, void* stream) {
  return id_create_ex(hp, A_D, m_global, m_local, row_offset, n, ld, workspace, ws_bytes, nccl_comm, rank, nranks,
                      stream, 0);
}

id_status id_create_ex(id_handle* hp, const double* A_D, int64_t m_global, int64_t m_local,
                       int64_t row_offset, int64_t n, int64_t ld, void* workspace, size_t ws_bytes,
                       void* nccl_comm, int32_t rank, int32_t nranks, void* stream, int32_t flags) {
  if (!hp || !A_D || !workspace) return ID_ERR_ARG;
  *hp = nullptr;
  if (m_local <= 0 || n <= 0 || ld < m_local || m_global < m_local || row_offset < 0 ||
      row_offset + m_local > m_global || nranks < 1 || rank < 0 || rank >= nranks)
    return ID_ERR_DIM;
  if (nranks > 1 && !nccl_comm) return ID_ERR_ARG;
  if (row_offset % 8) return ID_ERR_DIM;  // shards start on 8-row group boundaries
  if (((uintptr_t)workspace) & 255) return ID_ERR_ARG;
  mpid_ctx* h = new mpid_ctx();
  h->m_global = m_global;
  h->m_local = m_local;
  h->row_offset = row_offset;
  h->n = n;
  h->rank = rank;
  h->nranks = nranks;
  h->comm = nccl_comm;
  h->loop = is_loop(nccl_comm);
  if (h->loop && ((LoopComm*)nccl_comm)->nranks != nranks) {
    delete h;
    return ID_ERR_ARG;
  }
  h->st = (cudaStream_t)stream;
  h->user_st = h->st;
  h->ws = (char*)workspace;
  h->ws_bytes = ws_bytes;
  h->m_pad = m_pad_of(m_local);
  cudaPointerAttributes pa{};
  cudaError_t pe = cudaPointerGetAttributes(&pa, A_D);
  if (pe != cudaSuccess) cudaGetLastError();
  const bool host = (pe != cudaSuccess) || pa.type == cudaMemoryTypeHost || pa.type == cudaMemoryTypeUnregistered;
  // a host A_D is copied whole when the workspace holds it (host_AD = 1 sizing), else it is
  // streamed in row blocks (host_AD = 2 sizing)
  h->host_AD = host ? (((flags & ID_CREATE_STREAM_HOST) || layout(m_local, n, 1, 1, 4).total > ws_bytes) ? 2 : 1) : 0;
  h->srows_log2 = (flags >> 8) & 0xFF;
  if (relayout(h, 4) != ID_OK) {
    delete h;
    return ID_ERR_DIM;
  }
  for (auto& e : h->ev) {
    if (cudaEventCreate(&e) != cudaSuccess) { delete h; return ID_ERR_CUDA; }
  }
  if (cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->join_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete h;
    return ID_ERR_CUDA;
  }
  if (h->host_AD == 2) {
    h->AD_host = A_D;
    h->ld_host = ld;
    h->AD = nullptr;
    h->ld = m_local;
    if (cudaStreamCreateWithFlags(&h->cps, cudaStreamNonBlocking) != cudaSuccess) { delete h; return ID_ERR_CUDA; }
    for (int b = 0; b < 2; ++b)
      if (cudaEventCreateWithFlags(&h->copied[b], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->freed[b], cudaEventDisableTiming) != cudaSuccess) {
        delete h;
        return ID_ERR_CUDA;
      }
  } else if (h->host_AD == 1) {
    double* dst = (double*)(h->ws + h->L.AD);
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)m_local * 8, A_D, (size_t)ld * 8, (size_t)m_local * 8,
                                      (size_t)n, cudaMemcpyHostToDevice, h->st);
    if (e != cudaSuccess) {
      fail(h, ID_ERR_CUDA, "H2D copy of A_D: %s", cudaGetErrorString(e));
      delete h;
      return ID_ERR_CUDA;
    }
    h->AD = dst;
    h->ld = m_local;
  } else {
    h->AD = A_D;
    h->ld = ld;
  }
  *hp = h;
  return ID_OK;
}

void id_destroy(id_handle h) {
  if (!h) return;
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : h->cgraphs) cudaGraphExecDestroy(kv.second.first);
  for (auto& e : h->ev) if (e) cudaEventDestroy(e);
  for (auto& e : h->pass_ev) cudaEventDestroy(e);
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  if (h->join_ev) cudaEventDestroy(h->join_ev);
  if (h->cap) cudaStreamDestroy(h->cap);
  if (h->cps) cudaStreamDestroy(h->cps);
  for (int b = 0; b < 2; ++b) {
    if (h->copied[b]) cudaEventDestroy(h->copied[b]);
    if (h->freed[b]) cudaEventDestroy(h->freed[b]);
  }
  delete h;
}

const char* id_last_error(id_handle h) { return h ? h->err.c_str() : "null handle"; }

}  // extern "C"

// reset per-call scalars
__global__ void k_reset_scalars(DevScalars* sc, double eps) {
  sc->overflow = 0;
  sc->done = 0;
  sc->status = 0;
  sc->k_out = 0;
  sc->pivot = 0;
  sc->scale = 1.0;
  sc->maxabs = 0.0;
  sc->eps2normAL2 = eps > 0.0 ? eps * eps : 0.0;  // multiplied by ||A_L||^2 after rounding
}
// global norms/scalars after the (optional) allreduce of [norms(n), adsq, overflow]
__global__ void k_finish_round(const double* __restrict__ nb, int n, DevScalars* sc) {
  __shared__ double sh[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += nb[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < (int)(blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      sc->normAL2 = t;
      sc->normAD2 = nb[n];
      if (nb[n + 1] > 0.0) sc->overflow = 1;
      sc->eps2normAL2 *= t;
    }
  }
}
// per-rank adsq (sum of block partials) and overflow flag into nb[n], nb[n+1]
__global__ void k_pack_round(const double* __restrict__ aux, int naux, DevScalars* sc, double* nb, int n) {
  __shared__ double sh[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < naux; i += blockDim.x) t += aux[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < (int)(blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) {
      nb[n] = t;
      nb[n + 1] = sc->overflow ? 1.0 : 0.0;
    }
  }
}
__global__ void k_set_max(double* buf, const DevScalars* sc) { buf[0] = sc->maxabs; }
__global__ void k_get_max(const double* buf, DevScalars* sc) { sc->maxabs = buf[0]; }


// Host-streamed A_D (host_AD = 2): row blocks of srows rows are copied into two staging
// buffers on the copy stream, double-buffered against the kernels on h->st that consume
// them; fn(b, r0, rows, stage) enqueues block b's kernels.  Blocks run in row order, so
// every accumulation over blocks is in a fixed order.
template <typename Fn>
static id_status stream_blocks(mpid_ctx* h, Fn&& fn) {
  const int64_t m = h->m_local, n = h->n, R = h->srows;
  const int64_t nblk = (m + R - 1) / R;
  for (int64_t b = 0; b < nblk; ++b) {
    const int buf = (int)(b & 1);
    const int64_t r0 = b * R, rows = std::min<int64_t>(R, m - r0);
    // the staging buffer's previous users: block b - 2's kernels, or (first two blocks)
    // everything enqueued on h->st so far
    if (b < 2) CK(cudaEventRecord(h->freed[buf], h->st));
    CK(cudaStreamWaitEvent(h->cps, h->freed[buf], 0));
    CK(cudaMemcpy2DAsync(h->stage[buf], (size_t)R * 8, h->AD_host + r0, (size_t)h->ld_host * 8, (size_t)rows * 8,
                         (size_t)n, cudaMemcpyHostToDevice, h->cps));
    CK(cudaEventRecord(h->copied[buf], h->cps));
    CK(cudaStreamWaitEvent(h->st, h->copied[buf], 0));
    id_status s = fn(b, r0, rows, h->stage[buf]);
    if (s) return s;
    CK(cudaEventRecord(h->freed[buf], h->st));
  }
  return ID_OK;
}

__global__ void k_reset_scalars(DevScalars* sc, double eps);
__global__ void k_finish_round(const double* __restrict__ nb, int n, DevScalars* sc);
__global__ void k_set_max(double* buf, const DevScalars* sc);
__global__ void k_get_max(const double* buf, DevScalars* sc);
__global__ void k_overflow_into(const DevScalars* sc, double* dst) { dst[0] = sc->overflow ? 1.0 : 0.0; }

// the round of a host-streamed A_D: (scaling) a max |a| pass over the blocks, then the
// rounding pass, A_L written block by block into S; column norms and ||A_D||_F^2
// accumulated over the blocks in row order (eager: not captured in the QRCP graph)
static id_status enqueue_round_streamed(mpid_ctx* h, int fmt, int scaling, double eps) {
  const int64_t n = h->n, R = h->srows;
  const int64_t nblk = (h->m_local + R - 1) / R;
  if (nblk > 4000) return fail(h, ID_ERR_DIM, "host-streamed A_D: too many row blocks (%lld)", (long long)nblk);
  k_reset_scalars<<<1, 1, 0, h->st>>>(h->sc, eps);
  id_status s;
  if (scaling != ID_SCALE_NONE) {
    s = stream_blocks(h, [&](int64_t b, int64_t, int64_t rows, const double* blk) -> id_status {
      const int nb = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (rows * n + 255) / 256));
      CK(launch_maxabs(blk, rows, n, R, h->maxpart, nb, h->st));
      CK(launch_max_into(h->maxpart, nb, h->sacc + b, h->st));
      return ID_OK;
    });
    if (s) return s;
    CK(launch_maxabs_finish(h->sacc, (int)nblk, h->sc, scaling, h->st));
    if (h->nranks > 1 || h->comm) {
      k_set_max<<<1, 1, 0, h->st>>>(h->maxpart, h->sc);
      s = allreduce(h, h->maxpart, 1, NCCL_MAX);
      if (s) return s;
      k_get_max<<<1, 1, 0, h->st>>>(h->maxpart, h->sc);
    }
  }
  CK(launch_scale_from_max(h->sc, scaling, h->st));
  const int gy = round_gy(R, n);
  const int naux = gy * (int)((n + 31) / 32);
  CK(cudaMemsetAsync(h->cmaxd, 0, (size_t)n * 8, h->st));
  s = stream_blocks(h, [&](int64_t b, int64_t r0, int64_t rows, const double* blk) -> id_status {
    // rows up to the next 256-row tile of this block (the last block also covers m_pad's padding)
    const int64_t rpad = std::min<int64_t>(R, h->m_pad - r0);
    void* Sb = (char*)h->S + (size_t)(r0 / 8) * n * 8 * (fmt == ID_FP16 ? 2 : fmt == ID_FP32 ? 4 : 8);
    CK(launch_round(fmt, blk, rows, rpad, n, R, Sb, h->rpart, gy, h->sc, h->st, h->cmaxd));
    CK(launch_acc_rows(h->rpart, gy, n, n, h->norms, b > 0 ? 1 : 0, h->st));                   // column norms
    CK(launch_acc_rows(h->rpart + (int64_t)gy * n, naux, 1, 1, h->norms + n, b > 0 ? 1 : 0, h->st));  // ||A_D||^2
    return ID_OK;
  });
  if (s) return s;
  k_overflow_into<<<1, 1, 0, h->st>>>(h->sc, h->norms + n + 1);
  s = allreduce(h, h->norms, (size_t)n + 2, NCCL_SUM);
  if (s) return s;
  k_finish_round<<<1, 1024, 0, h->st>>>(h->norms, (int)n, h->sc);
  return ID_OK;
}

// enqueue scale + round + initial norms (+ collectives)
static id_status enqueue_round(mpid_ctx* h, int fmt, int scaling, double eps) {
  if (h->host_AD == 2) return enqueue_round_streamed(h, fmt, scaling, eps);
  const int64_t m = h->m_local, n = h->n;
  k_reset_scalars<<<1, 1, 0, h->st>>>(h->sc, eps);
  h->kernel_launches += 1;
  if (scaling != ID_SCALE_NONE) {
    const int nblk = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (m * n + 255) / 256));
    CK(launch_maxabs(h->AD, m, n, h->ld, h->maxpart, nblk, h->st));
    CK(launch_maxabs_finish(h->maxpart, nblk, h->sc, scaling, h->st));
    h->kernel_launches += 2;
    if (h->nranks > 1) {
      k_set_max<<<1, 1, 0, h->st>>>(h->maxpart, h->sc);
      id_status s = allreduce(h, h->maxpart, 1, NCCL_MAX);
      if (s) return s;
      k_get_max<<<1, 1, 0, h->st>>>(h->maxpart, h->sc);
      h->kernel_launches += 2;
    }
  }
  CK(launch_scale_from_max(h->sc, scaling, h->st));
  const int gy = round_gy(h->m_pad, n);
  CK(cudaMemsetAsync(h->cmaxd, 0, (size_t)n * 8, h->st));
  CK(launch_round(fmt, h->AD, m, h->m_pad, n, h->ld, h->S, h->rpart, gy, h->sc, h->st, h->cmaxd));
  CK(launch_sum_partials(h->rpart, gy, n, h->norms, h->st));  // norms[0:n]
  const int naux = gy * (int)((n + 31) / 32);
  k_pack_round<<<1, 1024, 0, h->st>>>(h->rpart + (int64_t)gy * n, naux, h->sc, h->norms, (int)n);
  h->kernel_launches += 4;
  id_status s = allreduce(h, h->norms, (size_t)n + 2, NCCL_SUM);
  if (s) return s;
  k_finish_round<<<1, 1024, 0, h->st>>>(h->norms, (int)n, h->sc);
  h->kernel_launches += 1;
  return ID_OK;
}

static id_status enqueue_qrcp(mpid_ctx* h, int fmt, int scaling, int k_max, double eps, int nb,
                              int formation, bool profile) {
  const int64_t n = h->n;
  h->kernel_launches = 0;
  h->pass_launches = 0;
  cudaGetLastError();  // clear any stale error before the launch checks
  CK(rec(h, h->ev[0]));
  id_status s = enqueue_round(h, fmt, scaling, eps);
  if (s) return s;
  CK(rec(h, h->ev[1]));
  if (formation == 4) {
    // NEXT-4, second option: Y = Omega A_L (Rademacher sketch, tcgen05), fp64 QRCP of Y
    CK(launch_sketch(h->tmapO, h->tmapG, (char*)h->S + (size_t)h->m_pad * n * 2, h->m_pad / 8, (int)n, h->sk_l,
                     h->sk_lw, h->m_local, h->row_offset, sketch_base(h->sk_seed), num_sms(), h->gpart,
                     gram_part_doubles(h->m_pad / 8, (int)n, num_sms()), h->G, h->sc, h->st));
    s = allreduce(h, h->G, (size_t)h->sk_lw * n, NCCL_SUM);
    if (s) return s;
    // the QRCP works on a copy (Gc) so Y stays available to id_get_sketch
    CK(cudaMemcpyAsync(h->Gc, h->G, (size_t)h->sk_lw * n * sizeof(double), cudaMemcpyDeviceToDevice, h->st));
    CK(launch_small_qrcp(h->Gc, h->sk_lw, (int)n, k_max, h->red, h->perm, h->W, (float*)h->R, h->sc, h->st));
    h->kernel_launches += 3 + 2 + 3 * k_max;
    h->pass_launches = 0;
    CK(rec(h, h->ev[2]));
    return ID_OK;
  }
  if (formation == 3) {
    // NEXT-4: G = A_L^T A_L on tcgen05, then the pivoted Cholesky (all k steps, one launch)
    if (h->tmapG_ok != 0) return fail(h, ID_ERR_CUDA, "cuTensorMapEncodeTiled (Gram) failed (%d)", h->tmapG_ok);
    CK(launch_gram(h->tmapG, h->m_pad / 8, (int)n, num_sms(), h->gpart, h->G, h->sc, h->st));
    s = allreduce(h, h->G, (size_t)n * n, NCCL_SUM);
    if (s) return s;
    CK(launch_pchol(h->G, h->Gc, (int)n, k_max, h->red, h->perm, h->W, (float*)h->R, h->sc, h->st));
    h->kernel_launches += 2 + 2 * ((k_max + 31) / 32);
    h->pass_launches = 0;
    CK(rec(h, h->ev[2]));
    return ID_OK;
  }
  if (formation == 6) {
    // the whole QRCP in one cooperative launch, the matrix in all SMs' shared memory
    CK(launch_qrcp_coop(fmt, h->S, h->m_local, (int)n, k_max, nb, eps, h->perm, (float*)h->R, h->part,
                        h->part + (size_t)pass_gx_cap() * n, h->sc, num_sms(), h->st));
    h->kernel_launches += 1;
    h->pass_launches = 0;
    CK(rec(h, h->ev[2]));
    return ID_OK;
  }
  if (formation == 5) {
    // the whole QRCP in one CTA's shared memory (the oracle's paper model, bit for bit)
    CK(launch_qrcp_smem(fmt, h->S, h->m_local, (int)n, k_max, nb, eps, h->perm, (float*)h->R, h->sc, h->st));
    h->kernel_launches += 1;
    h->pass_launches = 0;
    CK(rec(h, h->ev[2]));
    return ID_OK;
  }
  CK(launch_init_pivot(h->norms, (int)n, h->perm, h->sc, h->st));
  h->kernel_launches += 1;
  // one shard: the pass partials' reduction and the reflector can be one launch
  // (k_reduce_reflect, a last-block ticket); measured no faster in the captured step graph
  // (C2 k = 128: 2.24 vs 1.92 ms per QRCP, C4 +0.2 ms), so it is an opt-in A/B switch
  static const bool fused_on = getenv("MPID_FUSED_REFLECT") != nullptr;
  const bool fused = fused_on && h->nranks <= 1 && !h->comm;
  if (fused) CK(cudaMemsetAsync(h->ticket, 0, sizeof(unsigned int), h->st));
  const int own_lo = (int)std::min<int64_t>(h->row_offset, INT32_MAX);
  for (int j = 0; j < k_max; ++j) {
    const int j0 = j == 0 ? 0 : nb * ((j - 1) / nb);
    const int npend = j - j0;
    const int store = (npend == nb) ? 1 : 0;
    // the pivot's S data (its F / R / perm bookkeeping was swapped by the last k_reflector);
    // an in-pass-prologue variant measured no faster: its scattered 16-byte accesses
    // delay the CTA's TMA stream by as much as the separate launch costs
    CK(launch_swap(fmt, h->S, h->m_pad / 8, (int)n, j, j0, j, h->F, h->R, h->perm, nullptr, h->sc, h->st,
                   formation == 2 ? h->Fop : nullptr, h->cvec, nb));
    h->kernel_launches += 1;
    PassParams p{};
    p.S = h->S;
    p.ngroups = h->m_pad / 8;
    const int64_t jl = (int64_t)j - h->row_offset;
    p.g_lo = jl > 0 ? jl / 8 : 0;
    p.row_offset = h->row_offset;
    p.m_local = h->m_local;
    p.m_pad = h->m_pad;
    p.n = (int)n;
    p.j = j;
    p.j0 = j0;
    p.npend = npend;
    p.store = store;
    p.U = h->U;
    p.F = h->F;
    p.cvec = h->cvec;
    p.part = h->part;
    p.xr = h->xr;
    p.sc = h->sc;
    int gx_used = 0;
    // (tcgen05 pass: the V operand column of u_{j-1} was written by the previous pass, the
    // step's F operand is laid out by extra blocks of k_swap)
    if (formation == 2 && h->tmap_ok != 0) return fail(h, ID_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", h->tmap_ok);
    if (profile) CK(rec(h, h->pass_ev[2 * j]));
    if (formation == 2) CK(launch_pass_tc(p, nb, h->Vop, h->Fop, h->tmapS, h->tmapC, pass_gx_cap(), &gx_used, h->st));
    else {
      static const int cap_env = getenv("MPID_PASS_MAXCTAS") ? atoi(getenv("MPID_PASS_MAXCTAS")) : 0;   // measurements
      const int cap = cap_env > 0 ? std::min(cap_env, num_sms()) : num_sms();
      CK(launch_pass_tma(fmt, p, cap, &gx_used, h->st));
    }
    if (gx_used < 1 || gx_used > pass_gx_cap())
      return fail(h, ID_ERR_STATE, "panel pass grid %d exceeds the partials buffer (%d)", gx_used, pass_gx_cap());
    if (profile) CK(rec(h, h->pass_ev[2 * j + 1]));
    const int own = (j >= own_lo && (int64_t)j < h->row_offset + h->m_local) ? 1 : 0;
    if (fused) {
      CK(launch_reduce_reflect(fmt, h->part, gx_used, (int)n, j, h->xr, own, k_max, nb, h->F, h->R, h->beta,
                               h->cvec, h->tau, h->perm, h->sc, h->red, h->cand, h->ticket, h->st));
      h->kernel_launches += 2;
      h->pass_launches += 1;
      continue;
    }
    CK(launch_pass_reduce(h->part, gx_used, (int)n, j, h->xr, own, h->red, h->sc, h->st));
    s = allreduce(h, h->red, (size_t)3 * n, NCCL_SUM);
    if (s) return s;
    CK(launch_reflector(fmt, h->red, (int)n, j, k_max, nb, h->F, h->R, h->beta, h->cvec, h->tau, h->perm,
                        h->sc, h->st));
    h->kernel_launches += 3;
    h->pass_launches += 1;
  }
  CK(rec(h, h->ev[2]));
  return ID_OK;
}

extern "C" {

id_status id_round_only(id_handle h, id_format fmt, id_scaling scaling) {
  if (!h) return ID_ERR_ARG;
  cudaGetLastError();
  if (fmt != ID_FP16 && fmt != ID_FP32 && fmt != ID_FP64) return fail(h, ID_ERR_ARG, "bad format");
  if (scaling < 0 || scaling > 2) return fail(h, ID_ERR_ARG, "bad scaling");
  id_status s = ensure_layout(h, fmt);
  if (s) return s;
  s = enqueue_round(h, fmt, scaling, 0.0);
  if (s) return s;
  CK(cudaMemcpyAsync(&h->sc_host, h->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  h->fmt = fmt;
  h->have_qr = false;
  h->have_coef = false;
  h->have_cmaxd = true;
  h->stats.scale = h->sc_host.scale;
  h->stats.normAL_fro = sqrt(h->sc_host.normAL2);
  h->stats.normAD_fro = sqrt(h->sc_host.normAD2);
  if (h->sc_host.overflow) return fail(h, ID_ERR_OVERFLOW, "A_L overflows the low format after scaling");
  return ID_OK;
}

id_status id_qrcp_lowprec(id_handle h, id_format fmt, id_scaling scaling, int32_t k_max, double eps,
                          const id_qrcp_opts* opts, int32_t* k_out, int32_t* piv_out) {
  if (!h || !k_out || !piv_out) return ID_ERR_ARG;
  if (fmt != ID_FP16 && fmt != ID_FP32 && fmt != ID_FP64) return fail(h, ID_ERR_ARG, "bad format %d", (int)fmt);
  if (scaling < 0 || scaling > 2) return fail(h, ID_ERR_ARG, "bad scaling %d", (int)scaling);
  {
    const id_status ls = ensure_layout(h, fmt);
    if (ls) return ls;
  }
  if (!(eps >= 0.0 && eps < 1.0)) return fail(h, ID_ERR_DOMAIN, "eps must be in [0, 1)");
  if (k_max < 1 || k_max > std::min<int64_t>(h->n, h->m_global))
    return fail(h, ID_ERR_DIM, "k_max=%d outside [1, min(m, n)]", k_max);
  if (k_max > h->k_cap) return fail(h, ID_ERR_DIM, "workspace too small for k_max=%d (cap %lld)", k_max,
                                    (long long)h->k_cap);
  // formation of the pending trailing update: 1 = CUDA-core FFMA pass (short store interval,
  // fp16 / fp32 / fp64), 2 = tcgen05 pass (fp16).  Default: tcgen05 whenever it
  // applies — fp16 storage, range scaling (max |a| <= 1 keeps |F| <= 2 sqrt(2 m) inside the
  // fp16 operand range), n - 0 <= 2048 columns — else FFMA.
  const bool tc_ok = fmt == ID_FP16 && scaling != ID_SCALE_NONE && h->n <= 2048 &&
                     2.83 * sqrt((double)h->m_global) < 60000.0;
  // the tcgen05 pass pays a fixed per-launch cost (TMEM allocation, ring fill) that only
  // tall shards amortise: default to it from 16384 rows per shard (C3, C4, C5 shards; at
  // C2's 4096 rows the FFMA pass is twice as fast)
  const bool tc_default = tc_ok && h->m_local >= 16384;
  // 5 = the one-launch shared-memory QRCP (the paper model), default when one shard fits an SM
  const bool smem_ok = (fmt == ID_FP16 || fmt == ID_FP32) && h->nranks == 1 && !h->comm &&
                       qrcp_smem_bytes(h->m_local, (int)h->n, k_max) <= 227 * 1024;
  // 6 = the one-launch cooperative QRCP (the matrix in all SMs' shared memory, e.g. C2): opt-in —
  // measured ~19 us per step on C2 against ~15 us for the captured multi-kernel step
  const bool coop_ok = (fmt == ID_FP16 || fmt == ID_FP32) && h->nranks == 1 && !h->comm &&
                       qrcp_coop_rows(h->m_local, (int)h->n, num_sms()) > 0;
  int formation = opts ? opts->formation : 0;
  if (formation == 0) formation = smem_ok ? 5 : (tc_default ? 2 : 1);
  if (formation == 6 && !coop_ok)
    return fail(h, ID_ERR_ARG, "the cooperative QRCP needs fp16 / fp32, one shard and m x n x 4 B <= ~32 MB");
  if (formation == 5 && !smem_ok)
    return fail(h, ID_ERR_ARG, "the shared-memory QRCP needs fp16 / fp32, one shard and m x n x 4 B <= ~220 KB");
  if (formation == 2 && !tc_ok)
    return fail(h, ID_ERR_ARG, "the tcgen05 pass needs fp16 storage with range scaling, n <= 2048, m < 4.4e8");
  if (formation < 1 || formation > 6) return fail(h, ID_ERR_ARG, "bad formation %d", formation);
  if ((formation == 3 || formation == 4) && fmt != ID_FP16)
    return fail(h, ID_ERR_ARG, "Gram / sketched pivoting (formation 3, 4) run on fp16 A_L (tcgen05 kind::f16)");
  if (formation == 4) {
    // l = k_max + p; the default (p = 0 given) fills the 128-row tile that k_max + 10 needs
    // anyway (the extra sketch rows cost no extra MMA tile), e.g. l = 128 for k = 100
    const int over = opts && opts->sketch_oversample > 0 ? opts->sketch_oversample : 10;
    h->sk_lw = (k_max + over + 127) / 128 * 128;
    h->sk_l = opts && opts->sketch_oversample > 0 ? k_max + over : h->sk_lw;
    h->sk_seed = opts ? (uint32_t)opts->sketch_seed : 0u;
    if (h->sk_lw > h->n || h->sk_l > 8192)
      return fail(h, ID_ERR_DIM, "sketch of %d rows (padded %d) exceeds n = %lld", h->sk_l, h->sk_lw, (long long)h->n);
    const int r = encode_tmap_gram(h->tmapO, (char*)h->S + (size_t)h->m_pad * h->n * 2, h->m_pad / 8, h->sk_lw);
    if (r != 0) return fail(h, ID_ERR_CUDA, "cuTensorMapEncodeTiled (sketch) failed (%d)", r);
  }
  int nb = opts && opts->nb > 0 ? opts->nb : ((formation == 2 || formation == 5 || formation == 6) ? 16 : 4);
  if (nb > NB_MAX || (formation == 1 && nb > 16) || (fmt == ID_FP64 && nb > 8))
    return fail(h, ID_ERR_ARG, "nb=%d too large for formation %d / format %d", nb, formation, (int)fmt);
  // no graph capture for a loopback group (host-side reductions) or a host-streamed A_D
  // (its copies may come from pageable memory)
  const bool use_graph = !(opts && opts->use_graph < 0) && !h->loop && h->host_AD != 2;
  const bool profile = opts && opts->profile_pass;
  h->have_qr = h->have_coef = h->have_gram = h->have_sketch = false;
  if (profile && (int)h->pass_ev.size() < 2 * k_max) {
    const size_t old = h->pass_ev.size();
    h->pass_ev.resize(2 * k_max);
    for (size_t i = old; i < h->pass_ev.size(); ++i) CK(cudaEventCreate(&h->pass_ev[i]));
  }
  if (use_graph) {
    uint64_t eb;
    memcpy(&eb, &eps, 8);
    const uint64_t skey = formation == 4 ? ((uint64_t)h->sk_l << 32 | h->sk_seed) : 0;
    auto key = std::make_tuple((int)fmt, (int)scaling, (int)k_max, nb * 4 + formation, eb, profile ? 1 : 0, skey);
    auto it = h->graphs.find(key);
    if (it == h->graphs.end()) {
      cudaGraph_t g;
      h->st = h->cap;  // capture on the internal stream (the caller's may be the legacy stream)
      CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
      id_status s = enqueue_qrcp(h, fmt, scaling, k_max, eps, nb, formation, profile);
      cudaError_t e = cudaStreamEndCapture(h->cap, &g);
      h->st = h->user_st;
      if (s) return s;
      if (e != cudaSuccess) return fail(h, ID_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
      cudaGraphExec_t ge;
      CK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      it = h->graphs.emplace(key, ge).first;
      h->graph_launches[key] = h->kernel_launches;
    }
    // fork: cap waits for the caller's prior work; join: the caller waits for the graph
    CK(cudaEventRecord(h->ev[7], h->user_st));
    CK(cudaEventRecord(h->fork_ev, h->user_st));
    CK(cudaStreamWaitEvent(h->cap, h->fork_ev, 0));
    const auto tl0 = std::chrono::steady_clock::now();
    CK(cudaGraphLaunch(it->second, h->cap));
    h->stats.t_host_launch_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl0).count();
    CK(cudaEventRecord(h->join_ev, h->cap));
    CK(cudaStreamWaitEvent(h->user_st, h->join_ev, 0));
    h->stats.kernel_launches = h->graph_launches[key];
  } else {
    id_status s = enqueue_qrcp(h, fmt, scaling, k_max, eps, nb, formation, profile);
    if (s) return s;
    h->stats.kernel_launches = h->kernel_launches;
  }
  h->perm_host.resize(h->n);
  CK(cudaMemcpyAsync(&h->sc_host, h->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, h->st));
  CK(cudaMemcpyAsync(h->perm_host.data(), h->perm, h->n * sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaEventRecord(h->ev[6], h->st));
  CK(cudaStreamSynchronize(h->st));
  h->fmt = fmt;
  h->have_cmaxd = true;
  if (use_graph) {
    float tc = 0.f;
    cudaEventElapsedTime(&tc, h->ev[7], h->ev[6]);
    h->stats.t_call_gpu_ms = tc;
  }
  const DevScalars& sc = h->sc_host;
  if (sc.k_out < 0 || sc.k_out > k_max)
    return fail(h, ID_ERR_STATE, "internal: k_out=%d outside [0, %d]", sc.k_out, k_max);
  h->k_out = sc.k_out;
  h->qr_status = sc.status;
  *k_out = sc.k_out;
  for (int i = 0; i < sc.k_out; ++i) piv_out[i] = h->perm_host[i];
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]);
  h->stats.t_round_ms = ms;
  cudaEventElapsedTime(&ms, h->ev[1], h->ev[2]);
  h->stats.t_qrcp_ms = ms;
  h->stats.t_pass_ms = 0.0;
  if (profile) {
    double tot = 0.0;
    for (int j = 0; j < sc.k_out; ++j) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, h->pass_ev[2 * j], h->pass_ev[2 * j + 1]) == cudaSuccess) tot += t;
    }
    h->stats.t_pass_ms = tot;
  }
  h->stats.pass_launches = sc.k_out;
  h->stats.scale = sc.scale;
  h->stats.normAL_fro = sqrt(sc.normAL2);
  h->stats.normAD_fro = sqrt(sc.normAD2);
  h->stats.resid_est = sqrt(std::max(0.0, sc.resid2));
  h->stats.k_out = sc.k_out;
  h->stats.nb = nb;
  h->stats.formation = formation;
  h->stats.status_qrcp = sc.status;
  if (sc.overflow || sc.status == ID_ERR_OVERFLOW)
    return fail(h, ID_ERR_OVERFLOW, "A_L overflows the low format after scaling (S:53)");
  if (sc.status == ID_ERR_UNDERFLOW) {
    h->have_qr = sc.k_out > 0;
    h->have_gram = formation == 3;
    h->have_sketch = formation == 4;
    return fail(h, ID_ERR_UNDERFLOW, "pivot norm underflow at step %d (P:266)", sc.k_out);
  }
  h->have_qr = true;
  h->have_gram = formation == 3;
  h->have_sketch = formation == 4;
  return ID_OK;
}

id_status id_coeffs_fp64(id_handle h, id_coef_mode mode, double* P_out, int64_t ldp) {
  if (!h || !P_out) return ID_ERR_ARG;
  cudaGetLastError();
  if (!h->have_qr || h->k_out < 1) return fail(h, ID_ERR_STATE, "id_coeffs_fp64 needs a successful QRCP");
  const int k = h->k_out;
  const int n = (int)h->n;
  const int64_t m = h->m_local;
  if (ldp < k) return fail(h, ID_ERR_ARG, "ldp < k");
  if ((size_t)k * 33 * 8 > 200 * 1024) return fail(h, ID_ERR_DIM, "k=%d too large for the P solve", k);
  if (mode != ID_COEF_R && mode != ID_COEF_LSQ) return fail(h, ID_ERR_ARG, "bad coefficient mode");
  const int eng = fp64_engine(h, k, false);
  if (eng < 0) return fail(h, ID_ERR_ARG, "the int8 fp64 engine needs k <= 128, a device-resident A_D and k < n within its kernels' limits");
  CK(cudaEventRecord(h->ev[3], h->st));
  int launches = 0;
  const size_t tcap = tpart_doubles(m, n, h->k_cap);
  const int sp = splits_for(k, k, m, tcap);
  // P(:, J) = argmin ||A_I X - A_J|| by a preconditioned Cholesky QR in fp64:
  //   Q1 = A_I R1^{-1},  G2 = Q1^T Q1 = R2^T R2,  W = Q1^T A_J,  T = R1^{-1} R2^{-1} R2^{-T} W
  // with R1 = the QRCP's own low-precision R11 ("computed from the R matrix and
  // pivot indices ... via a least-squares problem"; A_I R11^{-1} is already close to
  // orthonormal, so one Cholesky pass suffices), or, when that Q1 is too ill-conditioned
  // (R2's diagonal spread > 1e3 or a breakdown), R1 = chol(A_I^T A_I): CholeskyQR2.
  auto lsq = [&](bool precond) -> id_status {
    const double* R1;
    if (precond) {
      CK(launch_R_to_fp64(h->fmt == ID_FP64, h->R, k, n, h->Rd, h->st));   // leading k x k block = R11
      CK(cudaMemsetAsync(h->info, 0, sizeof(int), h->st));
      R1 = h->Rd;
      launches += 1;
    } else {
      CK(launch_tsmm(h->AI, m, k, h->AI, m, k, m, h->tpart, sp, h->st));     // G1 = A_I^T A_I
      CK(launch_sum_partials(h->tpart, sp, (int64_t)k * k, h->G1, h->st));
      id_status s = allreduce(h, h->G1, (size_t)k * k, NCCL_SUM);
      if (s) return s;
      CK(launch_cholesky(h->G1, k, h->info, h->st));
      R1 = h->G1;
      launches += 3;
    }
    // Q1 = A_I R1^{-1}: the k x k inverse by triangular solves on I_k, then one DMMA GEMM
    CK(launch_eye(h->Ik, k, h->st));
    CK(launch_trsm_left_upper(R1, nullptr, k, h->Ik, k, nullptr, k, h->Rinv, k, 0, h->st));
    const int nj = n - k;
    const bool oz = eng == 2 && mode == ID_COEF_LSQ;
    int cmaxq_ready = 0;   // the int8 engine's Q1 column maxima come with Q1 when the kernel can
    CK(launch_nn_store(h->AI, m, m, h->Rinv, k, k, k, h->Q1, m, h->st, h->Tp, ew_tpack_doubles(h->n, h->k_cap),
                       oz ? h->cmaxq : nullptr, &cmaxq_ready));
    if (oz) {   // [G2 | W] = Q1^T [Q1 | A_D(:, J)] in one pass over A_D on the int8 tensor cores
      CK(launch_oz_tn(h->Q1, m, k, h->AD, h->ld, h->perm + k, nj, h->cmaxd, h->cmaxq, h->ozs, h->ozpart,
                      oz_part_doubles(num_sms()), h->G2, h->W, num_sms(), h->st, cmaxq_ready));
      launches += 5;
    } else {   // G2 = Q1^T Q1
      CK(launch_tsmm(h->Q1, m, k, h->Q1, m, k, m, h->tpart, sp, h->st));
      CK(launch_sum_partials(h->tpart, sp, (int64_t)k * k, h->G2, h->st));
      launches += 2;
    }
    id_status s = allreduce(h, h->G2, (size_t)k * k, NCCL_SUM);
    if (s) return s;
    CK(launch_cholesky(h->G2, k, h->info + 1, h->st));
    CK(launch_diag_ratio(h->G2, k, h->err2 + 1, h->st));
    launches += 5;
    // W = Q1^T A_D(:, J), J = perm[k:] (W(:, I) is never needed)
    if (nj > 0) {
      if (oz) {
      } else if (h->host_AD == 2) {   // W = sum over row blocks of Q1(blk)^T A_D(blk, J)
        const int spw = splits_for(k, nj, h->srows, tcap);
        id_status ss = stream_blocks(h, [&](int64_t b, int64_t r0, int64_t rows, const double* blk) -> id_status {
          CK(launch_tsmm(h->Q1 + r0, m, k, blk, h->srows, nj, rows, h->tpart, spw, h->st, h->perm + k));
          CK(launch_acc_rows(h->tpart, spw, (int64_t)k * nj, (int64_t)k * nj, h->W, b > 0 ? 1 : 0, h->st));
          return ID_OK;
        });
        if (ss) return ss;
      } else {
        const int spw = splits_for(k, nj, m, tcap);
        CK(launch_tsmm(h->Q1, m, k, h->AD, h->ld, nj, m, h->tpart, spw, h->st, h->perm + k));
        CK(launch_sum_partials(h->tpart, spw, (int64_t)k * nj, h->W, h->st));
      }
      s = allreduce(h, h->W, (size_t)k * nj, NCCL_SUM);
      if (s) return s;
      CK(launch_trsm_left_upper(R1, h->G2, k, h->W, k, nullptr, nj, h->T, k, 1, h->st));
      launches += 3;
    }
    return ID_OK;
  };
  // the body of the call: A_I = A_D(:, I), the coefficients (R mode, or LSQ with the R11
  // preconditioner), P assembled into the workspace — captured in a CUDA graph per (mode, k)
  // when the handle allows it (no loopback group, no host-streamed A_D)
  auto body = [&]() -> id_status {
    if (h->host_AD == 2) {   // A_I = A_D(:, I) straight from the host columns
      for (int i = 0; i < k; ++i)
        CK(cudaMemcpyAsync(h->AI + (size_t)i * m, h->AD_host + (size_t)h->perm_host[i] * h->ld_host, (size_t)m * 8,
                           cudaMemcpyHostToDevice, h->st));
    } else {
      CK(launch_gather_cols(h->AD, m, h->ld, h->perm, k, h->AI, h->st));
      launches++;
    }
    if (mode == ID_COEF_R) {
      CK(launch_R_to_fp64(h->fmt == ID_FP64, h->R, k, n, h->Rd, h->st));
      CK(launch_trsm_left_upper(h->Rd, nullptr, k, h->Rd + (int64_t)k * k, k, nullptr, n - k, h->T, k, 0,
                                h->st));
      launches += 2;
    } else {
      id_status s = lsq(true);
      if (s) return s;
    }
    CK(launch_assemble_P(h->T, k, k, n, h->perm, h->Pw, k, h->st));
    launches++;
    return ID_OK;
  };
  const bool use_graph = !h->loop && h->host_AD != 2;
  if (use_graph) {
    const uint64_t key = ((uint64_t)eng << 40) | ((uint64_t)mode << 32) | (uint64_t)k;   // engine, mode, k
    auto it = h->cgraphs.find(key);
    if (it == h->cgraphs.end()) {
      cudaGraph_t g;
      h->st = h->cap;
      CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
      launches = 0;
      id_status s = body();
      cudaError_t e = cudaStreamEndCapture(h->cap, &g);
      h->st = h->user_st;
      if (s) return s;
      if (e != cudaSuccess) return fail(h, ID_ERR_CUDA, "graph capture (coefficients): %s", cudaGetErrorString(e));
      cudaGraphExec_t ge;
      CK(cudaGraphInstantiate(&ge, g, 0));
      cudaGraphDestroy(g);
      it = h->cgraphs.emplace(key, std::make_pair(ge, launches)).first;
    }
    CK(cudaEventRecord(h->fork_ev, h->user_st));
    CK(cudaStreamWaitEvent(h->cap, h->fork_ev, 0));
    CK(cudaGraphLaunch(it->second.first, h->cap));
    CK(cudaEventRecord(h->join_ev, h->cap));
    CK(cudaStreamWaitEvent(h->user_st, h->join_ev, 0));
    launches = it->second.second;
  } else {
    id_status s = body();
    if (s) return s;
  }
  int info[2] = {0, 0};
  double ratio = 0.0;
  CK(cudaMemcpy2DAsync(P_out, ldp * 8, h->Pw, (size_t)k * 8, (size_t)k * 8, n, cudaMemcpyDeviceToDevice, h->st));
  if (mode == ID_COEF_LSQ) {
    CK(cudaMemcpyAsync(info, h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaMemcpyAsync(&ratio, h->err2 + 1, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  }
  CK(cudaStreamSynchronize(h->st));
  h->stats.lsq_path = mode == ID_COEF_LSQ ? 1 : 0;
  if (mode == ID_COEF_LSQ && (info[1] != 0 || !(ratio <= 1e3))) {   // identical decision on every rank
    id_status s = lsq(false);                                      // CholeskyQR2 (rare; eager)
    if (s) return s;
    CK(launch_assemble_P(h->T, k, k, n, h->perm, h->Pw, k, h->st));
    CK(cudaMemcpy2DAsync(P_out, ldp * 8, h->Pw, (size_t)k * 8, (size_t)k * 8, n, cudaMemcpyDeviceToDevice, h->st));
    CK(cudaMemcpyAsync(info, h->info, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->st));
    launches++;
    h->stats.lsq_path = 2;
  }
  CK(cudaEventRecord(h->ev[4], h->st));
  CK(cudaStreamSynchronize(h->st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[3], h->ev[4]);
  h->stats.t_coef_ms = ms;
  h->stats.fp64_engine = mode == ID_COEF_LSQ ? eng : 0;
  h->stats.kernel_launches += launches;
  if (mode == ID_COEF_LSQ && (info[0] || info[1]))
    return fail(h, ID_ERR_DEGENERATE, "Cholesky breakdown in the LSQ refit (info %d, %d)", info[0], info[1]);
  h->have_coef = true;
  return ID_OK;
}

id_status id_set_fp64_engine(id_handle h, int32_t engine) {
  if (!h) return ID_ERR_ARG;
  if (engine < 0 || engine > 2) return fail(h, ID_ERR_ARG, "bad fp64 engine %d", engine);
  h->fp64_engine = engine;
  return ID_OK;
}

id_status id_error(id_handle h, double* abs_fro, double* rel_fro) {
  if (!h || !abs_fro || !rel_fro) return ID_ERR_ARG;
  cudaGetLastError();
  if (!h->have_coef) return fail(h, ID_ERR_STATE, "id_error needs id_coeffs_fp64 first");
  const int k = h->k_out;
  const int eng = fp64_engine(h, k, true);
  if (eng < 0) return fail(h, ID_ERR_ARG, "the int8 fp64 engine needs k <= 128, a device-resident A_D and k < n within its kernels' limits");
  CK(cudaEventRecord(h->ev[5], h->st));
  int nblk = 0;
  // skeleton columns contribute exactly 0 (P(:, I) = I_k): sum over J = perm[k:] only
  const int nj = (int)h->n - k;
  if (nj > 0 && h->host_AD == 2) {   // sum over row blocks, in row order
    id_status ss = stream_blocks(h, [&](int64_t b, int64_t r0, int64_t rows, const double* blk) -> id_status {
      CK(launch_error(blk, rows, h->srows, nj, h->perm + k, h->AI + r0, k, h->T, k, h->epart, &nblk, h->st, h->Tp,
                      ew_tpack_doubles(h->n, h->k_cap), h->m_local, b == 0 ? 1 : 0));
      CK(launch_acc_rows(h->epart, nblk, 1, 1, h->err2, b > 0 ? 1 : 0, h->st));
      return ID_OK;
    });
    if (ss) return ss;
  } else if (nj > 0 && eng == 2) {   // int8 tensor cores (Ozaki scheme), A_I T never stored
    CK(launch_oz_error(h->AD, h->m_local, h->ld, nj, h->perm + k, h->AI, k, h->T, k, h->ozs, h->ozt, h->rsc,
                       h->fsc, h->epart, &nblk, num_sms(), h->st));
    CK(launch_sum_scalar(h->epart, nblk, h->err2, h->st));
  } else if (nj > 0) {
    CK(launch_error(h->AD, h->m_local, h->ld, nj, h->perm + k, h->AI, k, h->T, k, h->epart, &nblk, h->st, h->Tp,
                          ew_tpack_doubles(h->n, h->k_cap)));
    CK(launch_sum_scalar(h->epart, nblk, h->err2, h->st));
  } else {
    CK(cudaMemsetAsync(h->err2, 0, sizeof(double), h->st));
  }
  id_status s = allreduce(h, h->err2, 1, NCCL_SUM);
  if (s) return s;
  CK(cudaEventRecord(h->ev[6], h->st));
  double e2 = 0.0;
  CK(cudaMemcpyAsync(&e2, h->err2, 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev[5], h->ev[6]);
  h->stats.t_err_ms = ms;
  h->stats.kernel_launches += 2;
  h->stats.fp64_engine_err = eng;
  *abs_fro = sqrt(e2);
  *rel_fro = h->sc_host.normAD2 > 0 ? sqrt(e2 / h->sc_host.normAD2) : NAN;
  return ID_OK;
}

// power iteration for ||E||_2, E = A_D - X P (X = nullptr: E = A_D); returns the estimate
static id_status power_norm2(mpid_ctx* h, const double* X, int k, int iters, double* out) {
  const int n = (int)h->n;
  const int64_t m = h->m_local;
  double* x = h->pvec;
  double* z = x + n;
  double* v = z + n;
  double* wk = v + n;
  double* uk = wk + k;
  double* est = uk + k;
  double* part = est + 256;
  CK(launch_ones(x, n, h->st));
  for (int it = 0; it < iters; ++it) {
    CK(launch_gemv_n(h->AD, m, h->ld, n, x, h->py, 0, h->st));           // y = A_D x
    if (X) {
      CK(launch_p_times(h->Pw, k, k, n, x, wk, h->st));                  // w = P x
      CK(launch_gemv_n(X, m, m, k, wk, h->py, 1, h->st));                // y -= X w
    }
    CK(launch_gemv_t(h->AD, m, h->ld, n, h->py, part, PW_NBLK, h->st));  // A_D^T y (row-block partials)
    if (X) {
      CK(launch_gemv_t(X, m, m, k, h->py, part + (int64_t)PW_NBLK * n, PW_NBLK, h->st));
      CK(launch_sum_cols(part + (int64_t)PW_NBLK * n, PW_NBLK, k, nullptr, uk, h->st));   // u = X^T y
      id_status s = allreduce(h, uk, (size_t)k, NCCL_SUM);
      if (s) return s;
      CK(launch_pt_times(h->Pw, k, k, n, uk, v, h->st));                 // v = P^T u
      CK(launch_sum_cols(part, PW_NBLK, n, v, z, h->st));                // z = A_D^T y - v
    } else {
      CK(launch_sum_cols(part, PW_NBLK, n, nullptr, z, h->st));
    }
    id_status s = allreduce(h, z, (size_t)n, NCCL_SUM);
    if (s) return s;
    CK(launch_normalize(z, n, x, est, it < 255 ? it : 255, h->st));      // est = ||E^T E x||, x = z / |z|
  }
  double e = 0.0;
  CK(cudaMemcpyAsync(&e, est + (iters - 1 < 255 ? iters - 1 : 255), 8, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  *out = sqrt(e);
  return ID_OK;
}

id_status id_error_ex(id_handle h, int32_t skeleton, int32_t norm, int32_t iters, double* abs_err,
                      double* rel_err) {
  if (!h || !abs_err || !rel_err) return ID_ERR_ARG;
  cudaGetLastError();
  if (!h->have_coef) return fail(h, ID_ERR_STATE, "id_error_ex needs id_coeffs_fp64 first");
  if (skeleton != 0 && skeleton != 1) return fail(h, ID_ERR_ARG, "skeleton must be 0 (A_D) or 1 (A_L)");
  if (norm != 0 && norm != 2) return fail(h, ID_ERR_ARG, "norm must be 0 (Frobenius) or 2 (spectral)");
  if (iters < 0 || iters > 256) return fail(h, ID_ERR_ARG, "iters must be in [0, 256]");
  if (iters == 0) iters = 40;
  if (h->host_AD == 2 && (skeleton != 0 || norm != 0))
    return fail(h, ID_ERR_STATE, "id_error_ex: the low-precision skeleton and the 2-norm need a device-resident A_D");
  const int k = h->k_out;
  const int n = (int)h->n;
  const double* X = h->AI;                                     // A_D(:, I)
  if (skeleton == 1) {                                         // fl_L(s A_D(:, I)) / s into Q1 (free after coeffs)
    CK(launch_gather_lowp(h->AD, h->m_local, h->ld, h->perm, k, h->fmt, h->sc, h->Q1, h->st));
    X = h->Q1;
  }
  if (norm == 0) {
    if (skeleton == 0) return id_error(h, abs_err, rel_err);
    int nblk = 0;   // all n columns: the low-precision skeleton columns are not reproduced exactly
    CK(launch_error(h->AD, h->m_local, h->ld, n, nullptr, X, k, h->Pw, k, h->epart, &nblk, h->st, h->Tp,
                          ew_tpack_doubles(h->n, h->k_cap)));
    CK(launch_sum_scalar(h->epart, nblk, h->err2, h->st));
    id_status s = allreduce(h, h->err2, 1, NCCL_SUM);
    if (s) return s;
    double e2 = 0.0;
    CK(cudaMemcpyAsync(&e2, h->err2, 8, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    *abs_err = sqrt(e2);
    *rel_err = h->sc_host.normAD2 > 0 ? sqrt(e2 / h->sc_host.normAD2) : NAN;
    return ID_OK;
  }
  double e = 0.0;
  id_status s = power_norm2(h, X, k, iters, &e);
  if (s) return s;
  if (h->normAD_spec < 0.0) {
    s = power_norm2(h, nullptr, k, iters, &h->normAD_spec);
    if (s) return s;
  }
  *abs_err = e;
  *rel_err = h->normAD_spec > 0 ? e / h->normAD_spec : NAN;
  return ID_OK;
}

id_status id_get_R(id_handle h, float* R_out, int64_t ldr) {
  if (!h || !R_out) return ID_ERR_ARG;
  if (!h->have_qr) return fail(h, ID_ERR_STATE, "no QRCP result");
  if (ldr < h->k_out) return ID_ERR_ARG;
  // R is stored row-major k x n; output column-major k x n (the fp64 R is rounded to fp32)
  CK(launch_R_export(h->fmt == ID_FP64, h->R, h->k_out, (int)h->n, R_out, 0, ldr, h->st));
  CK(cudaStreamSynchronize(h->st));
  return ID_OK;
}

id_status id_get_R_fp64(id_handle h, double* R_out, int64_t ldr) {
  if (!h || !R_out) return ID_ERR_ARG;
  if (!h->have_qr) return fail(h, ID_ERR_STATE, "no QRCP result");
  if (ldr < h->k_out) return ID_ERR_ARG;
  CK(launch_R_export(h->fmt == ID_FP64, h->R, h->k_out, (int)h->n, R_out, 1, ldr, h->st));
  CK(cudaStreamSynchronize(h->st));
  return ID_OK;
}

id_status id_get_gram(id_handle h, double* G_out, int64_t ldg) {
  if (!h || !G_out || ldg < h->n) return ID_ERR_ARG;
  if (!h->have_gram) return fail(h, ID_ERR_STATE, "no Gram matrix (run id_qrcp_lowprec with formation 3)");
  CK(cudaMemcpy2DAsync(G_out, (size_t)ldg * 8, h->G, (size_t)h->n * 8, (size_t)h->n * 8, (size_t)h->n,
                       cudaMemcpyDeviceToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  return ID_OK;
}

id_status id_get_sketch(id_handle h, double* Y_out, int64_t ldy, int32_t* l_out) {
  if (!h || !Y_out || !l_out) return ID_ERR_ARG;
  if (!h->have_sketch) return fail(h, ID_ERR_STATE, "no sketch (run id_qrcp_lowprec with formation 4)");
  if (ldy < h->sk_l) return ID_ERR_ARG;
  CK(cudaMemcpy2DAsync(Y_out, (size_t)ldy * 8, h->G, (size_t)h->sk_lw * 8, (size_t)h->sk_l * 8, (size_t)h->n,
                       cudaMemcpyDeviceToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  *l_out = h->sk_l;
  return ID_OK;
}

id_status id_get_perm(id_handle h, int32_t* perm_out) {
  if (!h || !perm_out) return ID_ERR_ARG;
  if (h->perm_host.size() != (size_t)h->n) return fail(h, ID_ERR_STATE, "no QRCP result");
  memcpy(perm_out, h->perm_host.data(), h->n * sizeof(int32_t));
  return ID_OK;
}

id_status id_get_AL(id_handle h, void* out, int64_t ld) {
  if (!h || !out || ld < h->m_local) return ID_ERR_ARG;
  if (!h->fmt) return fail(h, ID_ERR_STATE, "no A_L yet");
  CK(launch_export_S(h->fmt, h->S, h->m_local, (int)h->n, out, ld, h->st));
  CK(cudaStreamSynchronize(h->st));
  return ID_OK;
}

id_status id_get_stats(id_handle h, id_stats* out) {
  if (!h || !out) return ID_ERR_ARG;
  *out = h->stats;
  return ID_OK;
}

id_status id_loopback_create(void** comm, int32_t nranks) {
  if (!comm || nranks < 1 || nranks > 1024) return ID_ERR_ARG;
  LoopComm* L = new LoopComm();
  L->nranks = nranks;
  L->slot.resize(nranks);
  {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    g_loops.insert(L);
  }
  *comm = L;
  return ID_OK;
}

int64_t id_loopback_calls(void* comm) {
  if (!is_loop(comm)) return -1;
  LoopComm* L = (LoopComm*)comm;
  std::lock_guard<std::mutex> lk(L->mu);
  return L->calls;
}

void id_loopback_destroy(void* comm) {
  if (!is_loop(comm)) return;
  {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    g_loops.erase(comm);
  }
  delete (LoopComm*)comm;
}


int32_t id_nccl_unique_id_bytes(void) { return 128; }

id_status id_nccl_get_unique_id(void* out) {
  if (!out) return ID_ERR_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return ID_ERR_NCCL;
  return api.GetUniqueId(out) == 0 ? ID_OK : ID_ERR_NCCL;
}

id_status id_nccl_comm_init(void** comm, const void* unique_id, int32_t nranks, int32_t rank) {
  if (!comm || !unique_id) return ID_ERR_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return ID_ERR_NCCL;
  NcclUid uid;
  memcpy(uid.internal, unique_id, 128);
  CommInitRankFn fn = (CommInitRankFn)api.CommInitRank;
  return fn(comm, nranks, uid, rank) == 0 ? ID_OK : ID_ERR_NCCL;
}

id_status id_nccl_comm_destroy(void* comm) {
  if (!comm) return ID_ERR_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return ID_ERR_NCCL;
  return api.CommDestroy(comm) == 0 ? ID_OK : ID_ERR_NCCL;
}

}  // extern "C"
