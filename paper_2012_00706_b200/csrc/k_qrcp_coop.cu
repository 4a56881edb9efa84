// k_qrcp_coop — the whole rank-k low-precision pivoted Householder QR of a matrix that fits in
// the shared memory of ALL SMs together (C2: 4096 x 1024, 16 MB in fp32 over 148 SMs), in ONE
// cooperative launch (Algorithm 2 line 4; Eq. (6)-(7)) — the latency path of
// the mid-size configurations, whose per-step chain of 4 launches costs ~15 us per step.
//
// Numerical model: the oracle's paper model (R4b/R5, oracle/cqrcp.c update = rne,
// acc = seq64) as in k_qrcp_smem, with ONE difference: a column's exact fp64 products are
// summed in row order within each CTA's row slab and the slab partials are then added by a
// fixed warp tree (fp64) — an association of the same fp64 sum, so s_i, w_i differ from the
// strict row order by a few fp64 ulps (far below the certification margin of reading R10).
//   per CTA: W (its rows x n, fp32) in shared memory; per step j (all CTAs, replicated state:
//   vn, perm, f in shared memory, identical in every CTA because computed from the same
//   global data in the same order):
//     pivot = argmax vn (ties: lowest original index), swap columns j <-> p (local rows);
//     every nb steps W(j:, j:) <- fl16(W) (fp16 storage);
//     slab partials of s_i = sum W(r,i)^2, w_i = sum W(r,i) W(r,j) (r >= j), x = W(j, :);
//     grid barrier; column c's slab partials are summed by one warp of CTA c % G (lanes over
//     the slabs in order, then a fixed butterfly: deterministic);
//     grid barrier; every CTA: beta, c, R(j, :), f, vn (paper model), W <- fl32(W - fl32(v f)).
// Bound: latency (two grid barriers per step); the working set stays in shared memory.
#include "mpid_internal.cuh"
#include <math.h>


namespace mpid {

namespace {
constexpr int CQ_THREADS = 1024;
template <typename T> __device__ __forceinline__ float cq_ld(const T* S, int64_t r, int c, int n);
template <> __device__ __forceinline__ float cq_ld<__half>(const __half* S, int64_t r, int c, int n) {
  return __half2float(S[((r >> 3) * n + c) * 8 + (r & 7)]);
}
template <> __device__ __forceinline__ float cq_ld<float>(const float* S, int64_t r, int c, int n) {
  return S[((r >> 3) * n + c) * 8 + (r & 7)];
}
}  // namespace


// column c's slab partials P[g][c] (slabs that hold rows >= j0 only) summed by one warp:
// lane l adds slabs l, l + 32, ... in order, then a fixed butterfly — deterministic, the same
// bits in every run; columns spread over CTAs (c % G) and their warps (c / G)
__device__ __forceinline__ double cq_colsum(const double* P, int G, int n, int rows, int m, int j0, int c, int lane) {
  double t = 0.0;
  for (int g = lane; g < G; g += 32) {
    if ((g + 1) * rows <= j0 || g * rows >= m) continue;   // no rows >= j0 in slab g
    t = __dadd_rn(t, P[(size_t)g * n + c]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xffffffffu, t, o));
  return t;
}

// grid barrier: one arrival per CTA on a global counter, the last arriver bumps the
// generation; the others poll it (acquire).  All CTAs are co-resident (cooperative launch).
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cq_barrier(unsigned* bar, unsigned G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* count = bar;
    unsigned* gen = bar + 32;                 // separate 128 B lines
    const unsigned g = ld_acquire(gen);
    __threadfence();
    if (atomicAdd(count, 1u) == G - 1) {
      *count = 0u;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
    } else {
      while (ld_acquire(gen) == g) {
      }
    }
  }
  __syncthreads();
}

struct CoopArgs {
  const void* S;
  int m, n, k_max, nb, store16;
  int rows;            // rows per CTA slab (the last may be shorter)
  double eps;
  int* perm;
  float* R;            // k x n row-major (global; CTA 0 writes)
  double* part;        // [2 (s, w)][G][n] slab partials
  double* red;         // [2 parity][3 (s, w, x)][n]
  DevScalars* sc;
  unsigned* bar;       // grid barrier: count at [0], generation at [32] (zeroed before the launch)
};

// per-CTA shared memory: W [n][rows + 1] fp32 | vn [n] fp64 | sv [n] fp64 | f [n] fp32 | pm [n] int
size_t qrcp_coop_bytes(int rows, int n) {
  return (size_t)n * (rows + 1) * 4 + 16 + (size_t)2 * n * 8 + (size_t)n * 4 + (size_t)n * 4 + 64;
}

template <typename T>
__global__ void __launch_bounds__(CQ_THREADS, 1) k_qrcp_coop(CoopArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n, G = gridDim.x, b = blockIdx.x;
  const int r0 = b * a.rows, r1 = min(a.m, r0 + a.rows), nr = max(0, r1 - r0);
  const int ldw = a.rows + 1;
  float* W = reinterpret_cast<float*>(smem);
  double* vn = reinterpret_cast<double*>(smem + (((size_t)n * ldw * 4 + 15) & ~(size_t)15));
  double* sv = vn + n;                     // this step's s (a shared-memory copy for the sequential sums)
  float* f = reinterpret_cast<float*>(sv + n);
  int* pm = reinterpret_cast<int*>(f + n);
  __shared__ int sh_p, sh_stop;
  __shared__ double sh_beta, sh_cc, sh_normAL, sh_red[32];
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const T* S = reinterpret_cast<const T*>(a.S);
  double* ps = a.part;                       // [G][n]
  double* pw = a.part + (size_t)G * n;       // [G][n]

  for (int c = warp; c < n; c += nw)
    for (int r = lane; r < a.rows; r += 32) W[c * ldw + r] = r < nr ? cq_ld<T>(S, r0 + r, c, n) : 0.f;
  for (int c = tid; c < n; c += nt) pm[c] = c;
  __syncthreads();
  // initial norms^2: slab partials (row order), then slabs in order
  for (int c = tid; c < n; c += nt) {
    double t = 0.0;
    for (int r = 0; r < nr; ++r) {
      const double x = (double)W[c * ldw + r];
      t = r == 0 ? __dmul_rn(x, x) : __dadd_rn(t, __dmul_rn(x, x));
    }
    ps[(size_t)b * n + c] = t;
  }
  cq_barrier(a.bar, (unsigned)G);
  for (int c = b + G * warp; c < n; c += G * nw) {
    const double t = cq_colsum(ps, G, n, a.rows, a.m, 0, c, lane);
    if (lane == 0) a.red[c] = t;
  }
  cq_barrier(a.bar, (unsigned)G);
  for (int c = tid; c < n; c += nt) vn[c] = a.red[c];
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int c = 0; c < n; ++c) t = c == 0 ? vn[0] : __dadd_rn(t, vn[c]);
    sh_normAL = __dsqrt_rn(t);
    sh_stop = 0;
  }
  cq_barrier(a.bar, (unsigned)G);   // everyone has read the initial partials before they are overwritten
  int kk = a.k_max, st = 0;
  for (int j = 0; j < a.k_max; ++j) {
    double* rs = a.red + (size_t)(j & 1) * 3 * n;   // parity buffers: s, w, x of this step
    double* rw = rs + n;
    double* rx = rw + n;
    if (tid < 32) {                                  // pivot (replicated in every CTA)
      double best = -INFINITY;
      int bo = 0x7fffffff, bp = -1;
      for (int i = j + tid; i < n; i += 32) {
        const double vi = vn[i];
        const int oi = pm[i];
        if (vi > best || (vi == best && oi < bo)) { best = vi; bo = oi; bp = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double vb = __shfl_xor_sync(0xffffffffu, best, o);
        const int ob = __shfl_xor_sync(0xffffffffu, bo, o);
        const int pb = __shfl_xor_sync(0xffffffffu, bp, o);
        if (vb > best || (vb == best && ob < bo)) { best = vb; bo = ob; bp = pb; }
      }
      if (tid == 0) sh_p = bp;
    }
    __syncthreads();
    const int p = sh_p;
    if (p != j) {
      for (int r = tid; r < a.rows; r += nt) {
        const float t = W[j * ldw + r];
        W[j * ldw + r] = W[p * ldw + r];
        W[p * ldw + r] = t;
      }
      if (b == 0)
        for (int r = tid; r < j; r += nt) {
          const float t = a.R[(size_t)r * n + j];
          a.R[(size_t)r * n + j] = a.R[(size_t)r * n + p];
          a.R[(size_t)r * n + p] = t;
        }
      if (tid == 0) {
        const int tp = pm[j]; pm[j] = pm[p]; pm[p] = tp;
        const double tv = vn[j]; vn[j] = vn[p]; vn[p] = tv;
      }
    }
    __syncthreads();
    const int lo = max(0, j - r0);                   // first local row with global row >= j
    if (a.store16 && j > 0 && j % a.nb == 0) {       // the storage rounding point (reading R4)
      for (int c = j + warp; c < n; c += nw)
        for (int r = lo + lane; r < nr; r += 32) W[c * ldw + r] = __half2float(__float2half_rn(W[c * ldw + r]));
      __syncthreads();
    }
    // slab partials of s_i, w_i (row order), and x = W(j, :) from the owner of row j
    for (int c = j + tid; c < n; c += nt) {
      double ss = 0.0, ww = 0.0;
      for (int r = lo; r < nr; ++r) {
        const double x = (double)W[c * ldw + r], u = (double)W[j * ldw + r];
        const double p2 = __dmul_rn(x, x), pu = __dmul_rn(x, u);
        if (r == lo) { ss = p2; ww = pu; }
        else { ss = __dadd_rn(ss, p2); ww = __dadd_rn(ww, pu); }
      }
      ps[(size_t)b * n + c] = ss;
      pw[(size_t)b * n + c] = ww;
      if (j >= r0 && j < r1) rx[c] = (double)W[c * ldw + (j - r0)];
    }
    cq_barrier(a.bar, (unsigned)G);
    // distributed reduction over the slabs (a warp per column; slabs entirely above row j skipped)
    for (int c = j + b + G * warp; c < n; c += G * nw) {
      const double ss = cq_colsum(ps, G, n, a.rows, a.m, j, c, lane);
      const double ww = cq_colsum(pw, G, n, a.rows, a.m, j, c, lane);
      if (lane == 0) { rs[c] = ss; rw[c] = ww; }
    }
    cq_barrier(a.bar, (unsigned)G);
    for (int c = j + tid; c < n; c += nt) sv[c] = rs[c];
    __syncthreads();
    if (tid == 0) {
      bool stop = false;
      if ((a.eps > 0.0 && j > 0) || j == a.k_max - 1) {
        double t = 0.0;
        for (int c = j; c < n; ++c) t = c == j ? sv[j] : __dadd_rn(t, sv[c]);
        if (b == 0) a.sc->resid2 = t;
        stop = a.eps > 0.0 && j > 0 && __dsqrt_rn(t) <= __dmul_rn(a.eps, sh_normAL);
      }
      if (stop) sh_stop = 1;
      else if (!(sv[j] >= 1.1754943508222875e-38)) {
        double t = 0.0;
        for (int c = j; c < n; ++c) t = c == j ? sv[j] : __dadd_rn(t, sv[c]);
        if (b == 0) a.sc->resid2 = t;
        sh_stop = 2;
      } else {
        const double u0 = rx[j];
        const double beta = -copysign(__dsqrt_rn(sv[j]), u0);
        sh_beta = beta;
        sh_cc = __ddiv_rn(1.0, __dadd_rn(u0, -beta));
      }
    }
    __syncthreads();
    if (sh_stop) {                                   // identical decision in every CTA
      kk = j;
      st = sh_stop == 2 ? 4 : 0;
      break;
    }
    const double beta = sh_beta, cc = sh_cc;
    const double sgn = copysign(1.0, beta);
    for (int c = tid; c < n; c += nt) {
      if (c < j) {
        if (b == 0) a.R[(size_t)j * n + c] = 0.f;
        continue;
      }
      const double rwc = __ddiv_rn(rw[c], beta);
      f[c] = __double2float_rn(__dadd_rn(rx[c], -rwc));
      if (b == 0) a.R[(size_t)j * n + c] = __double2float_rn(__dmul_rn(rwc, sgn));
      if (c > j) vn[c] = __dadd_rn(rs[c], -__dmul_rn(rwc, rwc));
    }
    __syncthreads();
    // W(j:, j:) <- fl(W - fl(v f)), v = fl32(W(:, j) c) with v_j = 1 (the owner's row j)
    for (int c = j + 1 + warp; c < n; c += nw) {
      const float fc = f[c];
      for (int r = lo + lane; r < nr; r += 32) {
        const int gr = r0 + r;
        const float v = gr == j ? 1.f : __double2float_rn(__dmul_rn((double)W[j * ldw + r], cc));
        W[c * ldw + r] = __fsub_rn(W[c * ldw + r], __fmul_rn(v, fc));
      }
    }
    __syncthreads();
    {                                                // column j itself last (its values were v's source)
      const float fc = f[j];
      for (int r = lo + tid; r < nr; r += nt) {
        const int gr = r0 + r;
        const float v = gr == j ? 1.f : __double2float_rn(__dmul_rn((double)W[j * ldw + r], cc));
        W[j * ldw + r] = __fsub_rn(W[j * ldw + r], __fmul_rn(v, fc));
      }
    }
    __syncthreads();
  }
  if (st == 0 && kk == a.k_max && a.k_max < (a.m < n ? a.m : n)) {   // exact mass after k steps
    const int j = kk, lo = max(0, j - r0);
    for (int c = j + tid; c < n; c += nt) {
      double ss = 0.0;
      for (int r = lo; r < nr; ++r) {
        const double x = (double)W[c * ldw + r];
        ss = r == lo ? __dmul_rn(x, x) : __dadd_rn(ss, __dmul_rn(x, x));
      }
      ps[(size_t)b * n + c] = ss;
    }
    cq_barrier(a.bar, (unsigned)G);
    double* rf = a.red + (size_t)((kk & 1) ^ 1) * 3 * n;   // a parity buffer no CTA reads any more
    for (int c = j + b + G * warp; c < n; c += G * nw) {
      const double t = cq_colsum(ps, G, n, a.rows, a.m, j, c, lane);
      if (lane == 0) rf[c] = t;
    }
    cq_barrier(a.bar, (unsigned)G);
    if (b == 0) {
      for (int c = j + tid; c < n; c += nt) sv[c] = rf[c];
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int c = j; c < n; ++c) t = c == j ? sv[j] : __dadd_rn(t, sv[c]);
        a.sc->resid2 = t;
      }
    }
  }
  if (b == 0) {
    for (int c = tid; c < n; c += nt) a.perm[c] = pm[c];
    if (tid == 0) {
      a.sc->k_out = kk;
      a.sc->status = st;
      a.sc->done = 1;
    }
  }
}

int qrcp_coop_rows(int64_t m, int n, int num_sms) {   // rows per slab, or 0 when it does not fit
  if (n > 4096) return 0;
  const int64_t rows = (m + num_sms - 1) / num_sms;
  if (rows < 1 || qrcp_coop_bytes((int)rows, n) > 220 * 1024) return 0;
  return (int)rows;
}

cudaError_t launch_qrcp_coop(int fmt, const void* S, int64_t m, int n, int k_max, int nb, double eps, int* perm,
                             float* R, double* part, double* red, DevScalars* sc, int num_sms, cudaStream_t st) {
  const int rows = qrcp_coop_rows(m, n, num_sms);
  if (!rows) return cudaErrorInvalidValue;
  const int G = (int)((m + rows - 1) / rows);
  unsigned* bar = reinterpret_cast<unsigned*>(red + 6 * (size_t)n);
  cudaError_t e0 = cudaMemsetAsync(bar, 0, 64 * sizeof(unsigned), st);
  if (e0 != cudaSuccess) return e0;
  CoopArgs a{S, (int)m, n, k_max, nb, fmt == 1 ? 1 : 0, rows, eps, perm, R, part, red, sc, bar};
  const size_t smem = qrcp_coop_bytes(rows, n);
  const void* fn = fmt == 1 ? (const void*)k_qrcp_coop<__half> : (const void*)k_qrcp_coop<float>;
  cudaError_t e = smem_attr(fn, (int)smem);
  if (e != cudaSuccess) return e;
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(CQ_THREADS), args, smem, st);
}

}  // namespace mpid
