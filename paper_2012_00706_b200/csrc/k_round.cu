// K0 / K1 — range scaling, rounding A_D -> A_L, initial column norms.
//
// Algorithm 2 line 2: A_L = fl(A).  With range scaling (BASELINE.json
// configs[1]; reading R7) A_L = fl_L(s * A_D): one fp64 multiply and
// ONE round-to-nearest-even conversion fp64 -> fp16 (cvt.rn.f16.f64) or
// fp64 -> fp32 (cvt.rn.f32.f64), subnormals kept (no -ftz), overflow -> Inf and
// flagged.  Column norms of A_L are accumulated in fp64 (the squares
// of fp16/fp32 values are exact in fp64; reading R5) for the first pivot.
//
// Bound: HBM.  Reads 8 B and writes s B (2 or 4) per element once.
#include "mpid_internal.cuh"
#include <cfloat>
#include <math.h>

namespace mpid {

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// K0: per-block max |a_ij|.  Work items = (column, 2048-row segment); a CTA takes
// items blockIdx.x, blockIdx.x + gridDim.x, ...; 16 B streaming loads, 4 per thread
// in flight per item.
__global__ void __launch_bounds__(256) k_maxabs(const double* __restrict__ A, int64_t m, int64_t n,
                                                int64_t ld, double* __restrict__ part) {
  constexpr int SEG = 2048;
  const int64_t segs = (m + SEG - 1) / SEG;
  const int64_t items = segs * n;
  const bool vec = ((ld & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
  double mx = 0.0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t c = it / segs, sg = it - c * segs;
    const double* col = A + c * ld;
    const int64_t r0 = sg * SEG;
    if (vec && r0 + SEG <= m) {
      const double2* p = reinterpret_cast<const double2*>(col + r0);
      double2 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldcs(p + threadIdx.x + q * 256);
#pragma unroll
      for (int q = 0; q < 4; ++q) mx = fmax(mx, fmax(fabs(v[q].x), fabs(v[q].y)));
    } else {
      const int64_t r1 = (r0 + SEG < m) ? r0 + SEG : m;
      for (int64_t r = r0 + threadIdx.x; r < r1; r += 256) mx = fmax(mx, fabs(__ldcs(col + r)));
    }
  }
  __shared__ double sh[8];
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_max(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void k_maxabs_finish(const double* __restrict__ part, int nblk, DevScalars* sc) {
  double mx = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) mx = fmax(mx, part[i]);
  __shared__ double sh[32];
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_max(v);
    if (threadIdx.x == 0) sc->maxabs = v;
  }
}

// s from the (global) max: MAXABS s = 1/mx; POW2 s = 2^-ceil(log2 mx) computed
// exactly with frexp (mx = f 2^e, f in [0.5,1): ceil(log2 mx) = e, or e-1 when f == 0.5).
__global__ void k_scale_from_max(DevScalars* sc, int scaling) {
  const double mx = sc->maxabs;
  double s = 1.0;
  if (mx > 0.0 && scaling == 1) {
    s = 1.0 / mx;
  } else if (mx > 0.0 && scaling == 2) {
    int e;
    const double f = frexp(mx, &e);
    const int c = (f == 0.5) ? e - 1 : e;
    s = ldexp(1.0, -c);
  }
  sc->scale = s;
}

// K1: grid (ceil(n/32), GY).  A CTA owns 32 columns and the row tiles
// t = blockIdx.y, blockIdx.y + GY, ... of 256 rows.  Per tile: each warp reads
// 4 whole columns of the tile (coalesced 256 B fp64 rows per instruction),
// rounds once fp64 -> fp16/fp32 (cvt.rn), keeps exact fp64 squares for the
// column norms, and stages the values in shared memory; the block then writes
// the tile in the interleaved layout, 32 consecutive columns x 16 B per row
// group (512 B contiguous per warp store).
// Partials: part[y*n + c] = sum of ||A_L(rows, c)||^2 over the CTA's tiles,
// aux[y*gridDim.x + x] = sum a_ij^2 (for ||A_D||_F).
template <typename T>
__global__ void __launch_bounds__(256) k_round(const double* __restrict__ A, int64_t m,
                                               int64_t ngroups, int64_t n, int64_t ld,
                                               T* __restrict__ S, double* __restrict__ part,
                                               double* __restrict__ aux,
                                               DevScalars* __restrict__ sc,
                                               unsigned long long* __restrict__ cmax) {
  constexpr int TR = sizeof(T) == 8 ? 128 : 256;   // rows per tile (fp64: the tile fits 48 KB)
  constexpr int PAD = 16 / sizeof(T);              // keep 16 B alignment, spread banks
  __shared__ __align__(16) T tile[32][TR + PAD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int64_t ntiles = ngroups / (TR / 8);
  const double s = sc->scale;
  double colsq[4] = {0.0, 0.0, 0.0, 0.0};
  double adq[4] = {0.0, 0.0, 0.0, 0.0};
  double cm[4] = {0.0, 0.0, 0.0, 0.0};   // column max |a_ij| of A_D (the fp64 stage's slice exponents)
  int inf = 0;
  // register prefetch: the next tile's 32 loads are in flight while this tile is
  // converted and written out
  double a[4][TR / 32];
  auto load_tile = [&](int64_t t) {
    const int64_t r0 = t * TR;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t c = c0 + warp * 4 + q;
      const double* col = A + c * ld;
#pragma unroll
      for (int i = 0; i < TR / 32; ++i) {
        const int64_t r = r0 + i * 32 + lane;
        a[q][i] = (c < n && r < m) ? __ldcs(col + r) : 0.0;
      }
    }
  };
  int64_t t = blockIdx.y;
  if (t < ntiles) load_tile(t);
  for (; t < ntiles; t += gridDim.y) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cl = warp * 4 + q;
#pragma unroll
      for (int i = 0; i < TR / 32; ++i) {
        const int rr = i * 32 + lane;
        const double av = a[q][i];
        adq[q] = fma(av, av, adq[q]);
        cm[q] = fmax(cm[q], fabs(av));
        const double x = __dmul_rn(s, av);
        T v;
        double d;
        if constexpr (sizeof(T) == 2) {
          const __half hv = __double2half(x);          // cvt.rn.f16.f64: single RNE rounding
          d = (double)__half2float(hv);
          v = *reinterpret_cast<const T*>(&hv);
        } else if constexpr (sizeof(T) == 4) {
          const float fv = __double2float_rn(x);       // cvt.rn.f32.f64
          d = (double)fv;
          v = *reinterpret_cast<const T*>(&fv);
        } else {
          d = x;                                       // fp64: A_L = s A_D (one rounding of the product)
          v = x;
        }
        inf |= (isinf(d) || isnan(d)) ? 1 : 0;         // non-finite A_L: ID_ERR_OVERFLOW
        colsq[q] = fma(d, d, colsq[q]);
        tile[cl][rr] = v;
      }
    }
    __syncthreads();
    if (t + gridDim.y < ntiles) load_tile(t + gridDim.y);
    // write: thread -> (column lane, row group warp + 8 j)
#pragma unroll
    for (int jg = 0; jg < TR / 8 / 8; ++jg) {
      const int g = warp + 8 * jg;
      const int64_t c = c0 + lane;
      if (c < n) {
        const uint4* src = reinterpret_cast<const uint4*>(&tile[lane][g * 8]);
        uint4* dst = reinterpret_cast<uint4*>(S + ((t * (TR / 8) + g) * n + c) * 8);
#pragma unroll
        for (int w = 0; w < (int)sizeof(T) / 2; ++w) __stcs(dst + w, src[w]);
      }
    }
  }
  if (cmax) {   // bit patterns of non-negative doubles order like unsigned integers
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double v = warp_max(cm[q]);
      const int64_t c = c0 + warp * 4 + q;
      if (lane == 0 && c < n) atomicMax(cmax + c, (unsigned long long)__double_as_longlong(v));
    }
  }
  const double adsq = (adq[0] + adq[1]) + (adq[2] + adq[3]);
  __shared__ double shc[32];
  __shared__ double sha[8];
  __shared__ int shi;
  if (threadIdx.x == 0) shi = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v = warp_sum(colsq[q]);
    if (lane == 0) shc[warp * 4 + q] = v;
  }
  double asum = warp_sum(adsq);
  if (lane == 0) sha[warp] = asum;
  __syncthreads();
  if (inf) atomicOr(&shi, 1);
  if (warp == 0) {
    const int64_t c = c0 + lane;
    if (c < n) part[(int64_t)blockIdx.y * n + c] = shc[lane];
    double u = lane < 8 ? sha[lane] : 0.0;
    u = warp_sum(u);
    if (lane == 0) aux[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = u;
  }
  __syncthreads();
  if (threadIdx.x == 0 && shi) atomicOr(&sc->overflow, 1);
}

// acc[c] = (add ? acc[c] : 0) + sum_y part[y*stride + c] (fixed order; the host-streamed
// round / W / error accumulate row blocks with it)
__global__ void k_acc_rows(const double* __restrict__ part, int rows, int64_t stride, int64_t len,
                           double* __restrict__ acc, int add) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= len) return;
  double t = 0.0;
  for (int y = 0; y < rows; ++y) t += part[(int64_t)y * stride + c];
  acc[c] = add ? acc[c] + t : t;
}
__global__ void k_max_into(const double* __restrict__ part, int nblk, double* __restrict__ acc) {
  double mx = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) mx = fmax(mx, part[i]);
  __shared__ double sh[32];
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    v = warp_max(v);
    if (threadIdx.x == 0) acc[0] = v;
  }
}

// out[c] = sum_y part[y*stride + c] (fixed order: deterministic)
__global__ void k_sum_rows(const double* __restrict__ part, int rows, int64_t stride, int64_t len,
                           double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= len) return;
  double t = 0.0;
  for (int y = 0; y < rows; ++y) t += part[(int64_t)y * stride + c];
  out[c] = t;
}

// S (interleaved) -> column-major out (A_L export for bit-exact checks)
template <typename T>
__global__ void k_export(const T* __restrict__ S, int64_t m, int64_t n, T* __restrict__ out,
                         int64_t ld) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * n) return;
  const int64_t c = idx / m, r = idx - c * m;
  out[c * ld + r] = S[((r >> 3) * n + c) * 8 + (r & 7)];
}

// ---------------------------------------------------------------------------
cudaError_t launch_acc_rows(const double* part, int rows, int64_t stride, int64_t len, double* acc, int add,
                            cudaStream_t st) {
  k_acc_rows<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(part, rows, stride, len, acc, add);
  return cudaGetLastError();
}
cudaError_t launch_max_into(const double* part, int nblk, double* acc, cudaStream_t st) {
  k_max_into<<<1, 1024, 0, st>>>(part, nblk, acc);
  return cudaGetLastError();
}
cudaError_t launch_maxabs(const double* A, int64_t m, int64_t n, int64_t ld, double* part,
                          int nblk, cudaStream_t st) {
  k_maxabs<<<nblk, 256, 0, st>>>(A, m, n, ld, part);
  return cudaGetLastError();
}
cudaError_t launch_maxabs_finish(const double* part, int nblk, DevScalars* sc, int scaling,
                                 cudaStream_t st) {
  k_maxabs_finish<<<1, 1024, 0, st>>>(part, nblk, sc);
  return cudaGetLastError();
}
cudaError_t launch_scale_from_max(DevScalars* sc, int scaling, cudaStream_t st) {
  k_scale_from_max<<<1, 1, 0, st>>>(sc, scaling);
  return cudaGetLastError();
}
cudaError_t launch_round(int fmt, const double* A, int64_t m, int64_t m_pad, int64_t n, int64_t ld,
                         void* S, double* part, int gy, DevScalars* sc, cudaStream_t st,
                         unsigned long long* cmax) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)gy);
  double* aux = part + (int64_t)gy * n;
  if (fmt == 1)
    k_round<__half><<<grid, 256, 0, st>>>(A, m, m_pad / 8, n, ld, (__half*)S, part, aux, sc, cmax);
  else if (fmt == 2)
    k_round<float><<<grid, 256, 0, st>>>(A, m, m_pad / 8, n, ld, (float*)S, part, aux, sc, cmax);
  else
    k_round<double><<<grid, 256, 0, st>>>(A, m, m_pad / 8, n, ld, (double*)S, part, aux, sc, cmax);
  return cudaGetLastError();
}
cudaError_t launch_sum_partials(const double* part, int splits, int64_t len, double* out,
                                cudaStream_t st) {
  k_sum_rows<<<(unsigned)((len + 255) / 256), 256, 0, st>>>(part, splits, len, len, out);
  return cudaGetLastError();
}
cudaError_t launch_export_S(int fmt, const void* S, int64_t m_local, int n, void* out, int64_t ld,
                            cudaStream_t st) {
  const int64_t tot = m_local * n;
  const unsigned nb = (unsigned)((tot + 255) / 256);
  if (fmt == 1)
    k_export<__half><<<nb, 256, 0, st>>>((const __half*)S, m_local, n, (__half*)out, ld);
  else if (fmt == 2)
    k_export<float><<<nb, 256, 0, st>>>((const float*)S, m_local, n, (float*)out, ld);
  else
    k_export<double><<<nb, 256, 0, st>>>((const double*)S, m_local, n, (double*)out, ld);
  return cudaGetLastError();
}

}  // namespace mpid
