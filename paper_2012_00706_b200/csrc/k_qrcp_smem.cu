// k_qrcp_smem — the whole rank-k low-precision pivoted Householder QR of a matrix that fits
// in one SM's shared memory (C1: 256 x 128), in ONE launch (Algorithm 2 line 4, P:163;
// Eq. (6)-(7)) — the latency path for the small configurations (C1 is
// latency-bound: the multi-kernel step chain costs ~15 us per step).
//
// Numerical model: the paper model of the oracle (R4b/R5; oracle/cqrcp.c with
// update = rne, acc = seq64), operation for operation, so the result is BIT-IDENTICAL to the
// oracle's (tests/test_gpu_smem.py):
//   W (m8 x n, fp32, column-major in shared memory) = A_L; per step j:
//   pivot = argmax of the downdated norms (ties: lowest original index), swap;
//   every nb steps W(j:, j:) <- fl16(W) (fp16 storage);
//   s_i = sum_{r >= j} W(r,i)^2, w_i = sum W(r,i) W(r,j): exact products added in fp64 in row
//   order (one thread per column);
//   beta = -sign(u0) sqrt(s_j), c = 1/(u0 - beta), v = fl32(W(:,j) c), v_j = 1,
//   R(j,:) = fl32(sign(beta) w / beta), f = fl32(x - w / beta), vn_i = s_i - (w_i / beta)^2;
//   W <- fl32(W - fl32(v f)) (every operation rounded; no fused multiply-add anywhere:
//   __fmul_rn / __fsub_rn / __dmul_rn / __dadd_rn).
// Bound: latency (one CTA; the fp64 column sums are sequential by definition of the model).
#include "mpid_internal.cuh"
#include <math.h>

namespace mpid {

namespace {
template <typename T> __device__ __forceinline__ float ld_s(const T* S, int64_t r, int c, int n);
template <> __device__ __forceinline__ float ld_s<__half>(const __half* S, int64_t r, int c, int n) {
  return __half2float(S[((r >> 3) * n + c) * 8 + (r & 7)]);
}
template <> __device__ __forceinline__ float ld_s<float>(const float* S, int64_t r, int c, int n) {
  return S[((r >> 3) * n + c) * 8 + (r & 7)];
}
}  // namespace

// shared memory: W [n][m8 + 1] fp32 (odd column stride: the one-thread-per-column sums read
// distinct banks) | vn, s, w, x, rr [n] fp64 | v [m8] fp32 | f [n] fp32 | perm [n] int |
// R [k][n] fp32 (written to global memory at the end)
size_t qrcp_smem_bytes(int64_t m, int n, int k) {
  const int64_t m8 = (m + 7) / 8 * 8;
  return (size_t)n * (m8 + 1) * 4 + 8 + (size_t)5 * n * 8 + (size_t)m8 * 4 + (size_t)n * 8 + (size_t)k * n * 4 + 64 +
         (size_t)m8 * 8 + 16;
}

template <typename T>
__global__ void __launch_bounds__(1024, 1) k_qrcp_smem(const T* __restrict__ S, int m, int n, int k_max, int nb,
                                                        int store16, double eps, int* __restrict__ perm,
                                                        float* __restrict__ R, DevScalars* __restrict__ sc) {
  if (sc->done) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int m8 = (m + 7) / 8 * 8;
  const int ldw = m8 + 1;
  float* W = reinterpret_cast<float*>(smem);
  double* vn = reinterpret_cast<double*>(smem + (((size_t)n * ldw * 4 + 15) & ~(size_t)15));
  double* s = vn + n;
  double* w = s + n;
  double* x = w + n;
  double* rr = x + n;
  float* v = reinterpret_cast<float*>(rr + n);
  float* f = v + m8;
  int* pm = reinterpret_cast<int*>(f + n);
  float* Rs = reinterpret_cast<float*>(pm + n);
  double* u64 = reinterpret_cast<double*>(smem + ((((size_t)n * ldw * 4 + 15) & ~(size_t)15) + (size_t)5 * n * 8 +
                                                   (size_t)m8 * 4 + (size_t)n * 8 + (size_t)k_max * n * 4 + 15) / 16 * 16);
  __shared__ int sh_p, sh_stop, sh_slow;
  __shared__ double sh_beta, sh_cc, sh_normAL;
  const int tid = threadIdx.x, nt = blockDim.x;

  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  for (int c = warp; c < n; c += nw)
    for (int r = lane; r < m8; r += 32) W[c * ldw + r] = r < m ? ld_s<T>(S, r, c, n) : 0.f;
  for (int c = tid; c < n; c += nt) pm[c] = c;
  __syncthreads();
  for (int c = tid; c < n; c += nt) {              // exact initial norms^2, row order
    double t = 0.0;
    for (int r = 0; r < m; ++r) {
      const double a = (double)W[(int64_t)c * ldw + r];
      t = r == 0 ? __dmul_rn(a, a) : __dadd_rn(t, __dmul_rn(a, a));
    }
    vn[c] = t;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int c = 0; c < n; ++c) t = c == 0 ? vn[0] : __dadd_rn(t, vn[c]);
    sh_normAL = __dsqrt_rn(t);
    sh_stop = 0;
  }
  __syncthreads();
  int kk = k_max, st = 0;
  // pivot of step j (warp 0): max vn, ties -> lowest original index (max and min are exact: any
  // order agrees).  Step 0's here; step j + 1's runs in warp 0 while warps 1-31 update (below).
  auto argmax = [&](int j) {
    double best = -INFINITY;
    int bo = 0x7fffffff, bp = -1;
    for (int i = j + lane; i < n; i += 32) {
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
    if (lane == 0) sh_p = bp;
  };
  if (warp == 0) argmax(0);
  __syncthreads();
  for (int j = 0; j < k_max; ++j) {
    const int jl = j, g0 = (j / 8) * 8;
    const int p = sh_p;
    const bool rnd = store16 && j > 0 && j % nb == 0;   // the storage rounding point (reading R4)
    // swap columns j <-> p with the storage rounding of their rows >= j, u = the new column j
    for (int r = tid; r < m8; r += nt) {
      float a = W[(int64_t)j * ldw + r], b = W[(int64_t)p * ldw + r];
      if (rnd && r >= jl) {
        a = __half2float(__float2half_rn(a));
        b = __half2float(__float2half_rn(b));
      }
      W[(int64_t)j * ldw + r] = b;
      W[(int64_t)p * ldw + r] = a;
      if (r >= g0) u64[r] = r < jl ? 0.0 : (double)b;
    }
    if (p != j) {
      for (int r = tid; r < j; r += nt) {
        const float a = Rs[(int64_t)r * n + j];
        Rs[(int64_t)r * n + j] = Rs[(int64_t)r * n + p];
        Rs[(int64_t)r * n + p] = a;
      }
      if (tid == 0) {
        const int tp = pm[j]; pm[j] = pm[p]; pm[p] = tp;
        const double tv = vn[j]; vn[j] = vn[p]; vn[p] = tv;
      }
    }
    if (rnd)
      for (int c = j + warp; c < n; c += nw) {
        if (c == j || c == p) continue;
        for (int r = jl + lane; r < m8; r += 32) W[c * ldw + r] = __half2float(__float2half_rn(W[c * ldw + r]));
      }
    __syncthreads();
    // s_i, w_i: exact products added in fp64 in row order from row g0 (rows g0..j-1 are exact
    // zeros: they only turn a leading -0 into +0, applied once); thread 0 owns column j and
    // forms beta / c unless the step needs the residual mass (a tolerance, the last step, an
    // underflowing pivot): then the serial block below
    for (int c = j + tid; c < n; c += nt) {
      const float* Wc = W + (int64_t)c * ldw;
      double ss, ww;
      {
        const double a = (double)Wc[jl];
        ss = __dmul_rn(a, a);
        ww = __dmul_rn(a, u64[jl]);
        if (g0 < jl) { ss = __dadd_rn(0.0, ss); ww = __dadd_rn(0.0, ww); }
      }
#pragma unroll 8
      for (int r = jl + 1; r < m8; ++r) {
        const double a = (double)Wc[r];
        ss = __dadd_rn(ss, __dmul_rn(a, a));
        ww = __dadd_rn(ww, __dmul_rn(a, u64[r]));
      }
      s[c] = ss;
      w[c] = ww;
      x[c] = (double)Wc[jl];
      if (c == j) {
        const bool slow = (eps > 0.0 && j > 0) || j == k_max - 1 || !(ss >= 1.1754943508222875e-38);
        sh_slow = slow;
        if (!slow) {
          const double u0 = x[j];
          const double beta = -copysign(__dsqrt_rn(ss), u0);
          sh_beta = beta;
          sh_cc = __ddiv_rn(1.0, __dadd_rn(u0, -beta));
        }
      }
    }
    __syncthreads();
    if (sh_slow) {
      if (tid == 0) {
        bool stop = false;
        if ((eps > 0.0 && j > 0) || j == k_max - 1) {   // (the last step's mass: resid when k = min(m, n))
          double t = 0.0;
          for (int c = j; c < n; ++c) t = c == j ? s[j] : __dadd_rn(t, s[c]);
          sc->resid2 = t;
          stop = eps > 0.0 && j > 0 && __dsqrt_rn(t) <= __dmul_rn(eps, sh_normAL);
        }
        if (stop) sh_stop = 1;
        else if (!(s[j] >= 1.1754943508222875e-38)) {
          double t = 0.0;
          for (int c = j; c < n; ++c) t = c == j ? s[j] : __dadd_rn(t, s[c]);
          sc->resid2 = t;
          sh_stop = 2;
        }
        else {
          const double u0 = x[j];
          const double beta = -copysign(__dsqrt_rn(s[j]), u0);
          sh_beta = beta;
          sh_cc = __ddiv_rn(1.0, __dadd_rn(u0, -beta));
        }
      }
      __syncthreads();
      if (sh_stop) {
        kk = j;
        st = sh_stop == 2 ? 4 : 0;
        break;
      }
    }
    const double beta = sh_beta, cc = sh_cc;
    const double sgn = copysign(1.0, beta);
    for (int r = jl + tid; r < m8; r += nt)
      v[r] = r == jl ? 1.f : __double2float_rn(__dmul_rn((double)W[(int64_t)j * ldw + r], cc));
    for (int c = tid; c < n; c += nt) {
      if (c < j) {
        Rs[(int64_t)j * n + c] = 0.f;
        continue;
      }
      const double rw = __ddiv_rn(w[c], beta);
      rr[c] = rw;
      f[c] = __double2float_rn(__dadd_rn(x[c], -rw));
      Rs[(int64_t)j * n + c] = __double2float_rn(__dmul_rn(rw, sgn));
      if (c > j) vn[c] = __dadd_rn(s[c], -__dmul_rn(rw, rw));
    }
    __syncthreads();
    if (warp == 0) {
      if (j + 1 < k_max) argmax(j + 1);                // the next step's pivot (vn is final)
    } else {
      for (int c = j + warp - 1; c < n; c += nw - 1) {  // W(j:, j:) <- fl(W - fl(v f))
        const float fc = f[c];
        for (int r = jl + lane; r < m8; r += 32) W[c * ldw + r] = __fsub_rn(W[c * ldw + r], __fmul_rn(v[r], fc));
      }
    }
    __syncthreads();
  }
  if (st == 0 && kk == k_max && k_max < (m < n ? m : n)) {   // exact mass after k steps
    const int j = k_max, jl = j, g0 = (j / 8) * 8;
    for (int c = j + tid; c < n; c += nt) {
      double ss = 0.0;
      for (int r = g0; r < m8; ++r) {
        const double a = r < jl ? 0.0 : (double)W[(int64_t)c * ldw + r];
        ss = r == g0 ? __dmul_rn(a, a) : __dadd_rn(ss, __dmul_rn(a, a));
      }
      s[c] = ss;
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int c = j; c < n; ++c) t = c == j ? s[j] : __dadd_rn(t, s[c]);
      sc->resid2 = t;
    }
  }
  __syncthreads();
  for (int c = tid; c < n; c += nt) perm[c] = pm[c];
  for (int64_t e = tid; e < (int64_t)kk * n; e += nt) R[e] = Rs[e];
  if (tid == 0) {
    sc->k_out = kk;
    sc->status = st;
    sc->done = 1;
  }
}

cudaError_t launch_qrcp_smem(int fmt, const void* S, int64_t m, int n, int k_max, int nb, double eps, int* perm,
                             float* R, DevScalars* sc, cudaStream_t st) {
  const size_t smem = qrcp_smem_bytes(m, n, k_max);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (fmt == 1) {
    cudaError_t e = smem_attr((const void*)k_qrcp_smem<__half>, (int)smem);
    if (e != cudaSuccess) return e;
    k_qrcp_smem<__half><<<1, 1024, smem, st>>>((const __half*)S, (int)m, n, k_max, nb, 1, eps, perm, R, sc);
  } else {
    cudaError_t e = smem_attr((const void*)k_qrcp_smem<float>, (int)smem);
    if (e != cudaSuccess) return e;
    k_qrcp_smem<float><<<1, 1024, smem, st>>>((const float*)S, (int)m, n, k_max, nb, 0, eps, perm, R, sc);
  }
  return cudaGetLastError();
}

}  // namespace mpid
