// The k-step low-precision pivoted Householder QR (Algorithm 2 line 4, P:163;
// Eq. (6)-(7)), B200 design "lazy panel with on-the-fly formation":
//
//   the stored matrix S (fp16/fp32, 8-row interleaved column-major, see
//   mpid_internal.cuh) lags the factorisation by at most nb reflectors; each
//   step ONE streaming pass over S (k_pass)
//     - forms the current trailing matrix A~ = S - sum_{pending l} v_l f_l^T
//       element by element in fp32 (FMA, in step order = the oracle's order),
//     - takes u = A~(:, j) (this step's pivot column, rows >= j),
//     - reduces w = A~^T u and the exact residual norms s_i = ||A~(j:m, i)||^2
//       (fp32 within an 8-row group, fp64 across groups; reading R5),
//     - emits the row x = A~(j, :) (needed for F and R),
//     - every nb steps writes fl_L(A~) back to S (the storage rounding point,
//       reading R4), which empties the pending list.
//   The per-step scalar work (k_reflector, one CTA) then forms the reflector
//   (beta, tau, c), the row R(j, :) = w / beta (sign-normalised), the update
//   vector f = x - w / beta (= tau A~^T v), the one-step downdated norms
//   vn_i = s_i - R(j,i)^2 and the next pivot (warp-shuffle argmax, ties to the
//   lowest original column index), all in device memory — no host sync.
//   The next pivot's bookkeeping (pending f, R, perm) is swapped by k_reflector, its
//   data in S by k_swap.
//
// Bound: HBM.  Per step the pass reads (m - j)(n - j) s bytes, plus
// (m - j)(n - j) s bytes written on store steps (every nb-th), plus the
// O(m + n) vectors.  The fp32 formation costs npend FMAs per element.
#include "mpid_internal.cuh"
#include <cfloat>
#include <math.h>

namespace mpid {

// red[0][c] = sum w, red[1][c] = sum s over the GX partial rows, red[2][c] = x_c.
// CTA = 32 columns (lanes) x 32 warps; warp w sums rows b = w, w+32, ... ; the 32
// warp partials are then added in warp order (deterministic).
constexpr int RW = 32;
__global__ void __launch_bounds__(32 * RW) k_pass_reduce(const double* __restrict__ part, int gx, int n,
                                                         int j, const double* __restrict__ xr, int own_row,
                                                         double* __restrict__ red,
                                                         const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = j + blockIdx.x * 32 + lane;
  __shared__ double sh[2][RW][32];
  double w = 0.0, s = 0.0;
  if (c < n) {
    for (int b = warp; b < gx; b += RW) {
      w += part[((int64_t)b * 2 + 0) * n + c];
      s += part[((int64_t)b * 2 + 1) * n + c];
    }
  }
  sh[0][warp][lane] = w;
  sh[1][warp][lane] = s;
  __syncthreads();
  if (warp == 0 && c < n) {
    double tw = 0.0, ts = 0.0;
#pragma unroll
    for (int i = 0; i < RW; ++i) { tw += sh[0][i][lane]; ts += sh[1][i][lane]; }
    red[c] = tw;
    red[n + c] = ts;
    red[2 * n + c] = own_row ? xr[c] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// k_reflector: one CTA of 1024 threads.  Step j's reflector, R row, f vector,
// downdated norms, next pivot, tolerance test.
// ---------------------------------------------------------------------------
struct ArgMax {
  double v;
  int orig;
  int pos;
};
__device__ __forceinline__ bool am_better(const ArgMax& a, const ArgMax& b) {
  // larger value wins; ties -> lowest original column index
  return a.v > b.v || (a.v == b.v && a.orig < b.orig);
}
__device__ __forceinline__ ArgMax am_shfl(const ArgMax& a, int o) {
  ArgMax b;
  b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
  b.orig = __shfl_xor_sync(0xffffffffu, a.orig, o);
  b.pos = __shfl_xor_sync(0xffffffffu, a.pos, o);
  return b;
}
__device__ ArgMax block_argmax(ArgMax a) {
  __shared__ ArgMax sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const ArgMax b = am_shfl(a, o);
    if (am_better(b, a)) a = b;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = a;
  __syncthreads();
  if (warp == 0) {
    a = lane < (int)(blockDim.x >> 5) ? sh[lane] : ArgMax{-1.0, 0x7fffffff, -1};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const ArgMax b = am_shfl(a, o);
      if (am_better(b, a)) a = b;
    }
    if (lane == 0) sh[0] = a;
  }
  __syncthreads();
  const ArgMax r = sh[0];
  __syncthreads();
  return r;
}
__device__ double block_sum(double v) {
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sh[0] = v;
  }
  __syncthreads();
  const double r = sh[0];
  __syncthreads();
  return r;
}

// W = working precision of F and R: fp32, or fp64 for the double QRCP (fmt 3)
template <typename W> __device__ __forceinline__ W to_w(double x);
template <> __device__ __forceinline__ float to_w<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ double to_w<double>(double x) { return x; }

// the tcgen05 pass's F operand of step jn (see k_pass_tc.cu): tile t, column c, pending l ->
// -(c_{j0+l} f_{j0+l}(jn + 128 t + c)) split into fp16 hi / lo, K-major core-matrix blocks of
// 16 pending reflectors: [tile][chunk][hi 4 KB | lo 4 KB], zero for l >= npend or columns >= n
__device__ __forceinline__ int fop_off(int i, int l) {
  return (i >> 3) * 256 + ((l >> 3) & 1) * 128 + (i & 7) * 16 + (l & 7) * 2;
}
__device__ void build_fop(const float* __restrict__ F, const double* __restrict__ cvec, int n, int jn, int nb,
                          unsigned char* __restrict__ Fop, int t0, int nthreads) {
  const int j0 = jn == 0 ? 0 : nb * ((jn - 1) / nb);
  const int npend = jn - j0;
  const int kchw = (nb + 15) / 16, KW = kchw * 16;
  const int ntiles = (n - jn + 127) / 128;
  const int tot = ntiles * 128 * KW;
  for (int e = t0; e < tot; e += nthreads) {
    const int l = e % KW, tc = e / KW;
    const int c = tc % 128, tt = tc / 128;
    const int col = jn + tt * 128 + c;
    float f = 0.f;
    if (l < npend && col < n)
      f = -__double2float_rn(cvec[j0 + l] * (double)F[(int64_t)((j0 + l) % NSLOT) * n + col]);
    const __half hi = __float2half_rn(f);
    const __half lo = __float2half_rn(f - __half2float(hi));
    unsigned char* base = Fop + ((size_t)tt * kchw + (l >> 4)) * 2 * 4096;
    const int o = fop_off(c, l & 15);
    *reinterpret_cast<__half*>(base + o) = hi;
    *reinterpret_cast<__half*>(base + 4096 + o) = lo;
  }
}

template <typename W>
__global__ void __launch_bounds__(1024) k_reflector(const double* __restrict__ red, int n, int j,
                                                    int k_max, int nb, W* __restrict__ F,
                                                    W* __restrict__ R, double* __restrict__ beta_out,
                                                    double* __restrict__ cvec, double* __restrict__ tau,
                                                    int* __restrict__ perm,
                                                    DevScalars* __restrict__ sc, unsigned char* __restrict__ Fop) {
  if (sc->done) return;
  // tolerance stop on the exact norms of this step's formed trailing matrix (R8)
  if (j > 0 && sc->eps2normAL2 > 0.0) {
    double tot = 0.0;
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) tot += red[n + i];
    tot = block_sum(tot);
    if (tot <= sc->eps2normAL2) {
      if (threadIdx.x == 0) {
        sc->k_out = j;
        sc->resid2 = tot;
        sc->done = 1;
      }
      return;
    }
  }
  const double sj = red[n + j];
  const double uj = red[2 * n + j];
  const double tiny = sizeof(W) == 8 ? DBL_MIN : (double)FLT_MIN;
  if (!(sj >= tiny)) {                               // pivot norm^2 underflows
    __syncthreads();
    if (threadIdx.x == 0) {
      sc->status = 4;  // ID_ERR_UNDERFLOW
      sc->k_out = j;
      sc->done = 1;
    }
    return;
  }
  const double beta = -copysign(sqrt(sj), uj);
  const double sgn = beta < 0.0 ? -1.0 : 1.0;
  const double c = 1.0 / (uj - beta);
  const int slot = j % NSLOT;
  if (threadIdx.x == 0) {
    beta_out[j] = beta;
    cvec[j] = c;
    tau[j] = (beta - uj) / beta;
  }
  ArgMax best{-1.0, 0x7fffffff, -1};
  double rest = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (i < j) {
      R[(int64_t)j * n + i] = W(0);
      continue;
    }
    const double rraw = red[i] / beta;
    R[(int64_t)j * n + i] = to_w<W>(rraw * sgn);
    F[(int64_t)slot * n + i] = to_w<W>(red[2 * n + i] - rraw);
    if (i > j) {
      const double vn = red[n + i] - rraw * rraw;      // one-step downdate from exact s_i
      rest += fmax(vn, 0.0);
      const ArgMax cand{vn, perm[i], i};
      if (am_better(cand, best)) best = cand;
    }
  }
  best = block_argmax(best);
  rest = block_sum(rest);
  // the next step's pivot moves to position jn = j + 1: its bookkeeping (the pending f
  // rows of the next panel, R's rows so far, perm) is swapped here; S's data is swapped
  // by k_swap
  const int jn = j + 1, pn = best.pos;
  if (jn < k_max && pn > jn) {
    const int j0n = nb * (j / nb);                    // first pending step of step jn
    for (int t = j0n + threadIdx.x; t < jn; t += blockDim.x) {
      W* f = F + (int64_t)(t % NSLOT) * n;
      const W x = f[jn];
      f[jn] = f[pn];
      f[pn] = x;
    }
    for (int t = threadIdx.x; t < jn; t += blockDim.x) {
      W* r = R + (int64_t)t * n;
      const W x = r[jn];
      r[jn] = r[pn];
      r[pn] = x;
    }
    if (threadIdx.x == 0) {
      const int x = perm[jn];
      perm[jn] = perm[pn];
      perm[pn] = x;
    }
  }
  if (threadIdx.x == 0) {
    sc->k_out = j + 1;
    sc->resid2 = rest;
    sc->pivot = best.pos;
    if (j + 1 >= k_max || best.pos < 0) sc->done = 1;
  }
  (void)Fop;
}

// k_reduce_reflect: k_pass_reduce and k_reflector in ONE launch for a single shard (no
// allreduce between them).  Block b reduces the pass partials of columns j + 32 b .. + 31
// exactly as k_pass_reduce (same order, same bits), recomputes column j's (s_j, x_j) the
// same way (so every block holds the identical beta, c), writes its columns' R(j, :),
// f_j and downdated norms, and leaves a block candidate (argmax, remaining mass, sum of
// s_i); the last block to finish (atomic ticket) makes the step's decisions exactly as
// k_reflector: tolerance stop (R8), underflow, the argmax over the candidates (total
// order: larger value, then lower original index), the next pivot's bookkeeping swaps.
// On a tolerance stop the speculative R(j, :), f_j writes are never read (k_out = j).
template <typename W>
__global__ void __launch_bounds__(32 * RW) k_reduce_reflect(const double* __restrict__ part, int gx, int n, int j,
                                                            const double* __restrict__ xr, int own_row, int k_max,
                                                            int nb, W* __restrict__ F, W* __restrict__ R,
                                                            double* __restrict__ beta_out, double* __restrict__ cvec,
                                                            double* __restrict__ tau, int* __restrict__ perm,
                                                            DevScalars* __restrict__ sc, double* __restrict__ red,
                                                            double* __restrict__ cand,
                                                            unsigned int* __restrict__ counter) {
  if (sc->done) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = j + blockIdx.x * 32 + lane;
  __shared__ double sh[3][RW][32];
  __shared__ double col[3][32];      // this block's (w, s, x)
  __shared__ double pj[2];           // s_j, x_j
  __shared__ int last;
  double w = 0.0, s = 0.0, sj = 0.0;
  if (c < n) {
    for (int b = warp; b < gx; b += RW) {
      w += part[((int64_t)b * 2 + 0) * n + c];
      s += part[((int64_t)b * 2 + 1) * n + c];
    }
  }
  if (lane == 0)
    for (int b = warp; b < gx; b += RW) sj += part[((int64_t)b * 2 + 1) * n + j];
  sh[0][warp][lane] = w;
  sh[1][warp][lane] = s;
  sh[2][warp][lane] = sj;
  __syncthreads();
  if (warp == 0) {
    double tw = 0.0, ts = 0.0;
#pragma unroll
    for (int i = 0; i < RW; ++i) { tw += sh[0][i][lane]; ts += sh[1][i][lane]; }
    const double tx = (c < n && own_row) ? xr[c] : 0.0;
    col[0][lane] = tw;
    col[1][lane] = ts;
    col[2][lane] = tx;
    if (c < n) {
      red[c] = tw;
      red[n + c] = ts;
      red[2 * n + c] = tx;
    }
    if (lane == 0) {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < RW; ++i) t += sh[2][i][0];
      pj[0] = t;
      pj[1] = own_row ? xr[j] : 0.0;
    }
  }
  __syncthreads();
  const double tiny = sizeof(W) == 8 ? DBL_MIN : (double)FLT_MIN;
  const double sjv = pj[0], uj = pj[1];
  const bool ok = sjv >= tiny;
  const double beta = -copysign(sqrt(sjv), uj);
  const double sgn = beta < 0.0 ? -1.0 : 1.0;
  const int slot = j % NSLOT;
  // block candidate (warp 0: the block's 32 columns)
  if (warp == 0) {
    ArgMax best{-1.0, 0x7fffffff, -1};
    double rest = 0.0, ssum = 0.0;
    if (c < n) {
      ssum = col[1][lane];
      if (ok) {
        const double rraw = col[0][lane] / beta;
        R[(int64_t)j * n + c] = to_w<W>(rraw * sgn);
        F[(int64_t)slot * n + c] = to_w<W>(col[2][lane] - rraw);
        if (c > j) {
          const double vn = col[1][lane] - rraw * rraw;
          rest = fmax(vn, 0.0);
          best = ArgMax{vn, perm[c], c};
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const ArgMax b = am_shfl(best, o);
      if (am_better(b, best)) best = b;
    }
    // fixed-order lane sums (deterministic): lane 0 adds lanes 0..31 in order
    double rl[2] = {rest, ssum};
    double r0 = 0.0, r1 = 0.0;
    for (int i = 0; i < 32; ++i) {
      r0 += __shfl_sync(0xffffffffu, rl[0], i);
      r1 += __shfl_sync(0xffffffffu, rl[1], i);
    }
    if (lane == 0) {
      double* cd = cand + 5 * (int64_t)blockIdx.x;
      cd[0] = best.v;
      cd[1] = (double)best.orig;
      cd[2] = (double)best.pos;
      cd[3] = r0;
      cd[4] = r1;
    }
  }
  if (blockIdx.x == 0 && ok)
    for (int i = threadIdx.x; i < j; i += blockDim.x) R[(int64_t)j * n + i] = W(0);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // ---- the last block: the step's decisions ----
  __shared__ ArgMax fin;
  __shared__ double frest, fsum;
  if (warp == 0) {
    ArgMax best{-1.0, 0x7fffffff, -1};
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const double* cd = cand + 5 * (int64_t)b;
      const ArgMax a{cd[0], (int)cd[1], (int)cd[2]};
      if (am_better(a, best)) best = a;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const ArgMax b = am_shfl(best, o);
      if (am_better(b, best)) best = b;
    }
    if (lane == 0) {
      double r = 0.0, t = 0.0;
      for (int b = 0; b < (int)gridDim.x; ++b) {
        r += cand[5 * (int64_t)b + 3];
        t += cand[5 * (int64_t)b + 4];
      }
      fin = best;
      frest = r;
      fsum = t;
      *counter = 0u;   // ready for the next step
    }
  }
  __syncthreads();
  if (j > 0 && sc->eps2normAL2 > 0.0 && fsum <= sc->eps2normAL2) {   // tolerance stop (R8)
    if (threadIdx.x == 0) {
      sc->k_out = j;
      sc->resid2 = fsum;
      sc->done = 1;
    }
    return;
  }
  if (!ok) {                                       // pivot norm^2 underflows
    if (threadIdx.x == 0) {
      sc->status = 4;
      sc->k_out = j;
      sc->done = 1;
    }
    return;
  }
  if (threadIdx.x == 0) {
    beta_out[j] = beta;
    cvec[j] = 1.0 / (uj - beta);
    tau[j] = (beta - uj) / beta;
  }
  const int jn = j + 1, pn = fin.pos;
  if (jn < k_max && pn > jn) {
    const int j0n = nb * (j / nb);
    for (int t = j0n + threadIdx.x; t < jn; t += blockDim.x) {
      W* f = F + (int64_t)(t % NSLOT) * n;
      const W x = f[jn];
      f[jn] = f[pn];
      f[pn] = x;
    }
    for (int t = threadIdx.x; t < jn; t += blockDim.x) {
      W* r = R + (int64_t)t * n;
      const W x = r[jn];
      r[jn] = r[pn];
      r[pn] = x;
    }
    if (threadIdx.x == 0) {
      const int x = perm[jn];
      perm[jn] = perm[pn];
      perm[pn] = x;
    }
  }
  if (threadIdx.x == 0) {
    sc->k_out = j + 1;
    sc->resid2 = frest;
    sc->pivot = pn;
    if (j + 1 >= k_max || pn < 0) sc->done = 1;
  }
}

// initial pivot: argmax of the initial column norms (ties lowest index); perm = identity
__global__ void __launch_bounds__(1024) k_init_pivot(const double* __restrict__ norms, int n,
                                                     int* __restrict__ perm,
                                                     DevScalars* __restrict__ sc) {
  ArgMax best{-1.0, 0x7fffffff, -1};
  double tot = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    perm[i] = i;
    const ArgMax cand{norms[i], i, i};
    tot += norms[i];
    if (am_better(cand, best)) best = cand;
  }
  best = block_argmax(best);
  tot = block_sum(tot);
  if (threadIdx.x == 0) {
    if (best.pos > 0) {                               // step 0's pivot to position 0
      perm[0] = best.pos;
      perm[best.pos] = 0;
    }
    sc->pivot = best.pos;
    sc->resid2 = tot;
    sc->k_out = 0;
    sc->status = 0;
    sc->done = sc->overflow ? 1 : 0;
    if (sc->overflow) sc->status = 3;  // ID_ERR_OVERFLOW
  }
}

// swap columns jn <-> p (p = sc->pivot) of S (all row groups) and copy the new pivot
// column to Sj; F, R and perm are swapped by k_reflector / k_init_pivot
template <typename T, typename W>
__global__ void k_swap(T* __restrict__ S, int64_t ngroups, int n, int jn, int j0,
                       W* __restrict__ F, W* __restrict__ R, int* __restrict__ perm,
                       T* __restrict__ Sj, const DevScalars* __restrict__ sc, int nsw, unsigned char* __restrict__ Fop,
                       const double* __restrict__ cvec, int nb) {
  if (sc->done) return;
  if ((int)blockIdx.x >= nsw) {   // the tcgen05 pass's F operand of step jn (its column order)
    if constexpr (sizeof(W) == 4)
      build_fop(reinterpret_cast<const float*>(F), cvec, n, jn, nb, Fop, (blockIdx.x - nsw) * blockDim.x + threadIdx.x,
                (gridDim.x - nsw) * blockDim.x);
    return;
  }
  const int p = sc->pivot;
  if (p < 0) return;
  const bool sw = p != jn;
  (void)j0; (void)F; (void)R; (void)perm;
  if (!sw && !Sj) return;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < ngroups) {
    // the new pivot column jn, also copied to the contiguous buffer Sj (tcgen05 pass)
    constexpr int NW = (int)sizeof(T) / 2;   // uint4 words per 8-row chunk
    uint4* a = reinterpret_cast<uint4*>(S + (g * n + jn) * RG);
    uint4* b = reinterpret_cast<uint4*>(S + (g * n + p) * RG);
    uint4 ta[NW], tb[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) { ta[w] = a[w]; tb[w] = sw ? b[w] : ta[w]; }
    if (sw) {
#pragma unroll
      for (int w = 0; w < NW; ++w) { a[w] = tb[w]; b[w] = ta[w]; }
    }
    if (Sj) {
      uint4* d = reinterpret_cast<uint4*>(Sj + g * RG);
#pragma unroll
      for (int w = 0; w < NW; ++w) d[w] = tb[w];
    }
  }
}

// ---------------------------------------------------------------------------
cudaError_t launch_pass_reduce(const double* part, int gx, int n, int j, const double* xr,
                               int own_row, double* red, const DevScalars* sc, cudaStream_t st) {
  const int cols = n - j;
  k_pass_reduce<<<(cols + 31) / 32, 32 * RW, 0, st>>>(part, gx, n, j, xr, own_row, red, sc);
  return cudaGetLastError();
}

cudaError_t launch_reflector(int fmt, const double* red, int n, int j, int k_max, int nb, void* F, void* R,
                             double* beta, double* cvec, double* tau, int* perm, DevScalars* sc,
                             cudaStream_t st, void* Fop) {
  if (fmt == 3)
    k_reflector<double><<<1, 1024, 0, st>>>(red, n, j, k_max, nb, (double*)F, (double*)R, beta, cvec, tau, perm, sc,
                                            nullptr);
  else
    k_reflector<float><<<1, 1024, 0, st>>>(red, n, j, k_max, nb, (float*)F, (float*)R, beta, cvec, tau, perm, sc,
                                           (unsigned char*)Fop);
  return cudaGetLastError();
}

cudaError_t launch_reduce_reflect(int fmt, const double* part, int gx, int n, int j, const double* xr, int own_row,
                                  int k_max, int nb, void* F, void* R, double* beta, double* cvec, double* tau,
                                  int* perm, DevScalars* sc, double* red, double* cand, unsigned int* counter,
                                  cudaStream_t st) {
  const unsigned nblk = (unsigned)((n - j + 31) / 32);
  if (fmt == 3)
    k_reduce_reflect<double><<<nblk, 32 * RW, 0, st>>>(part, gx, n, j, xr, own_row, k_max, nb, (double*)F,
                                                       (double*)R, beta, cvec, tau, perm, sc, red, cand, counter);
  else
    k_reduce_reflect<float><<<nblk, 32 * RW, 0, st>>>(part, gx, n, j, xr, own_row, k_max, nb, (float*)F, (float*)R,
                                                      beta, cvec, tau, perm, sc, red, cand, counter);
  return cudaGetLastError();
}

cudaError_t launch_init_pivot(const double* norms, int n, int* perm, DevScalars* sc,
                              cudaStream_t st) {
  k_init_pivot<<<1, 1024, 0, st>>>(norms, n, perm, sc);
  return cudaGetLastError();
}

cudaError_t launch_swap(int fmt, void* S, int64_t ngroups, int n, int jn, int j0, int steps_done,
                        void* F, void* R, int* perm, void* Sj, DevScalars* sc, cudaStream_t st, void* Fop,
                        const double* cvec, int nb) {
  (void)steps_done;
  const unsigned nsw = (unsigned)((ngroups + 255) / 256);
  // + the F operand blocks (tcgen05 pass, from the second step: the first has no pending reflector)
  const unsigned nfo = (Fop && jn > 0) ? (unsigned)((((n - jn + 127) / 128) * 128 * ((nb + 15) / 16) * 16 + 255) / 256) : 0u;
  const unsigned nbk = nsw + nfo;
  if (fmt == 1)
    k_swap<__half, float><<<nbk, 256, 0, st>>>((__half*)S, ngroups, n, jn, j0, (float*)F, (float*)R, perm,
                                               (__half*)Sj, sc, (int)nsw, (unsigned char*)Fop, cvec, nb);
  else if (fmt == 2)
    k_swap<float, float><<<nbk, 256, 0, st>>>((float*)S, ngroups, n, jn, j0, (float*)F, (float*)R, perm,
                                              (float*)Sj, sc, (int)nsw, (unsigned char*)Fop, cvec, nb);
  else
    k_swap<double, double><<<nsw, 256, 0, st>>>((double*)S, ngroups, n, jn, j0, (double*)F, (double*)R, perm,
                                                (double*)Sj, sc, (int)nsw, nullptr, cvec, nb);
  return cudaGetLastError();
}

}  // namespace mpid
