// The fp64 ID step (Algorithm 2 lines 5-7; Eq. (8) P:129-135;
// Remark 1 P:136-139; Remark 2 P:199-201), on the fp64 tensor pipe (DMMA,
// mma.sync.aligned.m8n8k4.f64).
//
//   LSQ mode ("least-squares problem"): P(:, J) = argmin ||A_I X - A_J||_F,
//   A_I = A_D(:, I), by a Cholesky QR preconditioned with the QRCP's own R11
//   (mpid_api.cu id_coeffs_fp64):
//     Q1 = A_I R11^{-1}  (R11^{-1} by triangular solves on I_k, then k_err_ws<STORE>)
//     G2 = Q1^T Q1, R2 = chol(G2),  W = Q1^T A_D(:, J)  (k_dgemm_tn_pipe8 / _pipe split-K)
//     T  = R11^{-1} R2^{-1} R2^{-T} W
//   and, when R2's diagonal spread exceeds 1e3 (or the Cholesky breaks down), the same
//   with R1 = chol(A_I^T A_I): CholeskyQR2.  R mode (Eq. (8)): T = R11^{-1} R12 from the
//   low-precision R promoted to fp64.
//   The error ||A_D - A_D(:, I) P||_F = ||A_D(:, J) - A_I T||_F (skeleton columns are
//   exactly 0) is one fused pass, k_err_ws: a warp-specialised persistent kernel over
//   128 x 128 tiles of the J columns (producer warp + 4-deep mbarrier ring of bulk copies,
//   16 consumer warps of 32 x 32 DMMA tiles) whose epilogue subtracts from A_D, squares
//   and reduces — never stored.  k_err_persist is the register-staged fallback for odd m
//   or unaligned A_I.
//
// Bound: the DMMA pipe for the GEMM-shaped kernels (intensity ~k/4 flop/B vs a ~6 flop/B
// ridge).
#include "mpid_internal.cuh"
#include <math.h>
#include <cstdlib>

namespace mpid {

// ---------------------------------------------------------------------------
__global__ void k_gather_cols(const double* __restrict__ A, int64_t m, int64_t ld,
                              const int* __restrict__ perm, double* __restrict__ X) {
  const int l = blockIdx.y;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m) X[(int64_t)l * m + r] = A[(int64_t)perm[l] * ld + r];
}
// the same with 16-byte accesses, two per thread in flight (even m and ld, aligned bases)
__global__ void __launch_bounds__(256) k_gather_cols2(const double* __restrict__ A, int64_t m, int64_t ld,
                                                      const int* __restrict__ perm, double* __restrict__ X) {
  const int l = blockIdx.y;
  const int64_t h = m / 2;
  const double2* src = reinterpret_cast<const double2*>(A + (int64_t)perm[l] * ld);
  double2* dst = reinterpret_cast<double2*>(X + (int64_t)l * m);
  const int64_t i0 = (int64_t)blockIdx.x * 512 + threadIdx.x;
  double2 v0 = make_double2(0.0, 0.0), v1 = v0;
  if (i0 < h) v0 = __ldcs(src + i0);
  if (i0 + 256 < h) v1 = __ldcs(src + i0 + 256);
  if (i0 < h) dst[i0] = v0;
  if (i0 + 256 < h) dst[i0 + 256] = v1;
}

// ---------------------------------------------------------------------------
// fp64 tensor-core GEMM core (DMMA: mma.sync.aligned.m8n8k4.row.col.f64).
// CTA tile (16 MT) x 128, 8 warps as 2 (M) x 4 (N), warp tile 8 MT x 32 = MT x 4
// MMA tiles, K staged 16 at a time through double-buffered shared memory
// (register-staged 16 B global loads, coalesced along the contiguous dimension).
//   GM_TN_PARTIAL: out[split][c][i] = sum_{r in split} X(r, i) Y(r, c)   (X m x M, Y m x N)
//   GM_NN_STORE:   out(r, c)        = sum_l X(r, l) B(l, c)               (Q1 = A_I R1^-1)
// The fused error is its own persistent kernel (k_err_persist, below).
// Fragments of m8n8k4 f64 (PTX ISA): A(g, t), B(t, g), C(g, 2t + {0,1}) with
// g = lane >> 2, t = lane & 3.
// ---------------------------------------------------------------------------
constexpr int GT = 128, GK = 16;
constexpr int LDK = GK + 4;      // [mn][k] tiles: row stride 160 B -> conflict-free fragment reads
constexpr int LDM = GT + 4;      // [k][mn] tile (NN A operand): 132 doubles: rows tq = 0..3 of a fragment
                                 // read land in bank octets 0, 8, 16, 24 -> conflict-free

enum GemmMode { GM_TN_PARTIAL = 0, GM_NN_STORE = 1 };

struct GemmArgs {
  // TN: C(i, c) = sum_r X(r, i) Y(r, c), rows r in the split's range; X m x M, Y m x N
  // NN: C(r, c) = sum_l X(r, l) B(l, c); X m x K, B K x N (col-major, ldb)
  const double* X;
  int64_t ldx;
  const double* Y;   // TN: Y ; NN: B
  int64_t ldy;
  int64_t M, N, K;   // TN: M = k1, N = n1, K = m (rows) ; NN: M = m, N = ncols, K = k
  int64_t k_per_split;
  double* out;       // TN: partials [split][N][M] ; NN_ERROR: partial sums per block ; NN_UPDATE: C
  int64_t ldo;
  const double* A;   // NN_ERROR: A_D (m x n_all), lda; column c of the product is A's column cmap[c]
  int64_t lda;
  const int* cmap;
  const int* ycmap;  // TN: column c of Y is Y's column ycmap[c] (nullptr = identity)
  unsigned long long* cmax;   // NN store (k_err_ws<true>): atomicMax of each column's max |out| (bit patterns) or null
  int d_tma;         // NN_ERROR: 1 = the A_D tile may be prefetched with bulk copies (16 B aligned rows)
};
constexpr int DLD = GT + 2;      // NN_ERROR: smem A_D tile [c][r], 130 doubles per column (16 B aligned,
                                 // epilogue columns 2 tq land in distinct bank octets)

__device__ __forceinline__ void dmma(double* c, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int MODE, int MT>   // MT m8 tiles per warp in M: CTA tile (16 MT) x 128
__global__ void __launch_bounds__(256, 1) k_dgemm(GemmArgs g) {
  constexpr int BM = 16 * MT;
  // A tile: TN -> As[i][k] (LDK), NN -> As[k][r] (LDM); B tile: Bs[c][k] (LDK)
  constexpr int A_ELEMS = (MODE == GM_TN_PARTIAL) ? GT * LDK : GK * LDM;
  extern __shared__ __align__(16) double dsm[];
  double (*As)[A_ELEMS] = reinterpret_cast<double (*)[A_ELEMS]>(dsm);
  double (*Bs)[GT * LDK] = reinterpret_cast<double (*)[GT * LDK]>(dsm + 2 * A_ELEMS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;           // 2 x 4 warps
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * GT;
  int64_t k_begin = 0, k_end = g.K;
  if (MODE == GM_TN_PARTIAL) {
    k_begin = (int64_t)blockIdx.z * g.k_per_split;
    k_end = min(g.K, k_begin + g.k_per_split);
  }
  double2 ra[4], rb[4];
  // loads: 128 (mn) x 16 (k) doubles per operand = 1024 double2, 4 per thread
  auto gload = [&](int64_t kb) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + q * 256;                  // 0..1023
      if (MODE == GM_TN_PARTIAL) {
        const int mn = idx >> 3, kk = (idx & 7) * 2;  // 8 double2 per 16-long k segment
        const int64_t r = kb + kk;
        const int64_t i = m0 + mn, c = n0 + mn;
        ra[q] = make_double2(0.0, 0.0);
        rb[q] = make_double2(0.0, 0.0);
        if (i < g.M && mn < BM) {
          const double* p = g.X + i * g.ldx + r;
          if (r + 1 < k_end && (((uintptr_t)p & 15) == 0)) ra[q] = *reinterpret_cast<const double2*>(p);
          else { if (r < k_end) ra[q].x = p[0]; if (r + 1 < k_end) ra[q].y = p[1]; }
        }
        if (c < g.N) {
          const double* p = g.Y + (g.ycmap ? (int64_t)g.ycmap[c] : c) * g.ldy + r;
          if (r + 1 < k_end && (((uintptr_t)p & 15) == 0)) rb[q] = *reinterpret_cast<const double2*>(p);
          else { if (r < k_end) rb[q].x = p[0]; if (r + 1 < k_end) rb[q].y = p[1]; }
        }
      } else {
        // A = X (m x K col-major): element (r, l) at X[r + l ldx]; tile [l][r]
        {
          const int l = idx >> 6, rr = (idx & 63) * 2;  // 64 double2 per 128-long column
          const int64_t kk = kb + l, r = m0 + rr;
          ra[q] = make_double2(0.0, 0.0);
          if (kk < k_end && rr < BM) {
            const double* p = g.X + kk * g.ldx + r;
            if (r + 1 < g.M && (((uintptr_t)p & 15) == 0)) ra[q] = *reinterpret_cast<const double2*>(p);
            else { if (r < g.M) ra[q].x = p[0]; if (r + 1 < g.M) ra[q].y = p[1]; }
          }
        }
        // B (K x N col-major): element (l, c) at Y[l + c ldy]; tile [c][l]
        {
          const int cc = idx >> 3, l = (idx & 7) * 2;
          const int64_t c = n0 + cc, kk = kb + l;
          rb[q] = make_double2(0.0, 0.0);
          if (c < g.N) {
            const double* p = g.Y + c * g.ldy + kk;
            if (kk < k_end) rb[q].x = p[0];
            if (kk + 1 < k_end) rb[q].y = p[1];
          }
        }
      }
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + q * 256;
      if (MODE == GM_TN_PARTIAL) {
        const int mn = idx >> 3, kk = (idx & 7) * 2;
        *reinterpret_cast<double2*>(&As[buf][mn * LDK + kk]) = ra[q];
      } else {
        const int l = idx >> 6, rr = (idx & 63) * 2;
        *reinterpret_cast<double2*>(&As[buf][l * LDM + rr]) = ra[q];
      }
      const int cc = idx >> 3, l = (idx & 7) * 2;
      *reinterpret_cast<double2*>(&Bs[buf][cc * LDK + l]) = rb[q];
    }
  };
  double acc[MT][4][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  if (k_begin < k_end) {
    gload(k_begin);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int64_t kb = k_begin; kb < k_end; kb += GK) {
      const bool more = kb + GK < k_end;
      if (more) gload(kb + GK);
      const int64_t krem = (k_end - kb + 3) / 4;
      // skip all-zero k-steps, and warps whose rows or columns are all outside the matrix
      const int ksteps = (m0 + wm * 8 * MT >= g.M || n0 + wn * 32 >= g.N) ? 0
                         : (krem < GK / 4 ? (int)krem : GK / 4);
#pragma unroll
      for (int ks = 0; ks < GK / 4; ++ks) {
        if (ks >= ksteps) break;
        double af[MT], bf[4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int mm = wm * (8 * MT) + mt * 8 + gq, kk = ks * 4 + tq;
          af[mt] = (MODE == GM_TN_PARTIAL) ? As[buf][mm * LDK + kk] : As[buf][kk * LDM + mm];
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[buf][(wn * 32 + nt * 8 + gq) * LDK + ks * 4 + tq];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
      }
      if (more) {
        sstore(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }

  if (MODE == GM_TN_PARTIAL) {
    double* o = g.out + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int64_t i = m0 + wm * (8 * MT) + mt * 8 + gq;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t c = n0 + wn * 32 + nt * 8 + tq * 2 + h;
          if (i < g.M && c < g.N) o[c * g.M + i] = acc[mt][nt][h];
        }
    }
  } else if (MODE == GM_NN_STORE) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int64_t r = m0 + wm * (8 * MT) + mt * 8 + gq;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t c = n0 + wn * 32 + nt * 8 + tq * 2 + h;
          if (r < g.M && c < g.N) g.out[c * g.ldo + r] = acc[mt][nt][h];
        }
    }
  }
}

// ---------------------------------------------------------------------------
// Fused fp64 error, persistent: e^2 = sum_{r, c} (A_D(r, cmap[c]) - sum_l X(r, l) T(l, c))^2
// (Remark 2: products in double; the residual is never stored).
// One CTA per SM walks its 128 x 128 output tiles (row block major, so the tiles of
// one row block share the A_I tile in L2) as ONE flattened (tile, k-stage) loop:
// the next stage's loads — including the next tile's first stage — are in
// flight while the current stage's DMMAs run, and each tile's A_D block is
// prefetched into shared memory by bulk copies one tile ahead of its epilogue.
// ---------------------------------------------------------------------------
// 16 warps (4 x 4), warp tile 32 x 32: twice the DMMA streams per SM sub-partition of an
// 8-warp layout (the kernel is latency-bound on DMMA issue at 8 warps), 1024 double2 per
// operand stage = 2 per thread
constexpr int ERR_THREADS = 512, ERR_LD = 1024 / ERR_THREADS, ERR_WM = 32, ERR_MT = ERR_WM / 8;
__global__ void __launch_bounds__(ERR_THREADS, 1) k_err_persist(GemmArgs g, int64_t ntiles, int ncb) {
  extern __shared__ __align__(16) double dsm[];
  double (*As)[GK * LDM] = reinterpret_cast<double (*)[GK * LDM]>(dsm);
  double (*Bs)[GT * LDK] = reinterpret_cast<double (*)[GT * LDK]>(dsm + 2 * GK * LDM);
  double* Ds = dsm + 2 * GK * LDM + 2 * GT * LDK;
  __shared__ __align__(8) uint64_t dbar;
  __shared__ double red[ERR_THREADS / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;           // 4 x 4 warps, warp tile 32 x 32
  const int64_t K = g.K;
  const int nks = (int)((K + GK - 1) / GK);
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t total = my_tiles * nks;
  if (tid == 0) {
    mbar_init(&dbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto tile_of = [&](int64_t lt, int64_t& m0, int64_t& n0) {
    const int64_t t = blockIdx.x + lt * gridDim.x;
    m0 = (t / ncb) * GT;
    n0 = (t % ncb) * GT;
  };
  auto d_ok = [&](int64_t m0) {
    const int64_t rows = (g.M - m0 < GT) ? g.M - m0 : (int64_t)GT;
    return g.d_tma && (rows % 2 == 0);
  };
  // warp 0 issues the A_D block copies of a tile: each lane 4 of the 128 column copies.
  // The column map of the NEXT tile is loaded right after (src_next), so the copies
  // never wait on a dependent global load at a tile boundary.
  int src_next[GT / 32];
  auto load_src = [&](int64_t n0) {
#pragma unroll
    for (int q = 0; q < GT / 32; ++q) {
      const int64_t c = n0 + lane + 32 * q;
      src_next[q] = c < g.N ? (g.cmap ? g.cmap[c] : (int)c) : 0;
    }
  };
  auto issue_d = [&](int64_t m0, int64_t n0) {
    const int64_t rows = (g.M - m0 < GT) ? g.M - m0 : (int64_t)GT;
    const int cols = (int)((g.N - n0 < GT) ? g.N - n0 : (int64_t)GT);
    if (lane == 0) mbar_expect_tx(&dbar, (uint32_t)(rows * cols * 8));
    __syncwarp();
#pragma unroll
    for (int q = 0; q < GT / 32; ++q) {
      const int c = lane + 32 * q;
      if (c < cols)
        tma_load(Ds + c * DLD, g.A + (int64_t)src_next[q] * g.lda + m0, (uint32_t)(rows * 8), &dbar);
    }
  };
  double2 ra[ERR_LD], rb[ERR_LD];
  auto gload = [&](int64_t m0, int64_t n0, int64_t kb) {
#pragma unroll
    for (int q = 0; q < ERR_LD; ++q) {
      const int idx = tid + q * ERR_THREADS;
      {
        const int l = idx >> 6, rr = (idx & 63) * 2;
        const int64_t kk = kb + l, r = m0 + rr;
        ra[q] = make_double2(0.0, 0.0);
        if (kk < K) {
          const double* p = g.X + kk * g.ldx + r;
          if (r + 1 < g.M && (((uintptr_t)p & 15) == 0)) ra[q] = *reinterpret_cast<const double2*>(p);
          else { if (r < g.M) ra[q].x = p[0]; if (r + 1 < g.M) ra[q].y = p[1]; }
        }
      }
      {
        const int cc = idx >> 3, l = (idx & 7) * 2;
        const int64_t c = n0 + cc, kk = kb + l;
        rb[q] = make_double2(0.0, 0.0);
        if (c < g.N) {
          const double* p = g.Y + c * g.ldy + kk;
          if (kk < K) rb[q].x = p[0];
          if (kk + 1 < K) rb[q].y = p[1];
        }
      }
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int q = 0; q < ERR_LD; ++q) {
      const int idx = tid + q * ERR_THREADS;
      const int l = idx >> 6, rr = (idx & 63) * 2;
      *reinterpret_cast<double2*>(&As[buf][l * LDM + rr]) = ra[q];
      const int cc = idx >> 3, l2 = (idx & 7) * 2;
      *reinterpret_cast<double2*>(&Bs[buf][cc * LDK + l2]) = rb[q];
    }
  };
  double acc[ERR_MT][4][2];
#pragma unroll
  for (int a = 0; a < ERR_MT; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double e2 = 0.0;
  uint32_t dphase = 0;
  if (total > 0) {
    int64_t m0, n0;
    tile_of(0, m0, n0);
    if (warp == 0) {
      load_src(n0);
      if (d_ok(m0)) issue_d(m0, n0);
      if (my_tiles > 1) {
        int64_t m1, n1;
        tile_of(1, m1, n1);
        load_src(n1);
      }
    }
    gload(m0, n0, 0);
    sstore(0);
    __syncthreads();
  }
  int buf = 0;
  int64_t lt = 0, m0 = 0, n0 = 0, m1 = 0, n1 = 0;
  int ks_i = 0;
  if (total > 0) tile_of(0, m0, n0);
  for (int64_t it = 0; it < total; ++it) {
    const int64_t kb = (int64_t)ks_i * GK;
    if (ks_i == 0 && it > 0 && warp == 0) {                // this tile's A_D block, next tile's map
      if (d_ok(m0)) issue_d(m0, n0);
      if (lt + 1 < my_tiles) {
        int64_t m2, n2;
        tile_of(lt + 1, m2, n2);
        load_src(n2);
      }
    }
    const bool more = it + 1 < total;
    const bool last_k = ks_i == nks - 1;
    if (more) {
      if (last_k) tile_of(lt + 1, m1, n1);
      else { m1 = m0; n1 = n0; }
      gload(m1, n1, last_k ? 0 : kb + GK);
    }
    const int64_t krem = (K - kb + 3) / 4;
    const int ksteps = (m0 + wm * ERR_WM >= g.M || n0 + wn * 32 >= g.N) ? 0 : (krem < GK / 4 ? (int)krem : GK / 4);
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      if (ks >= ksteps) break;
      double af[ERR_MT], bf[4];
#pragma unroll
      for (int mt = 0; mt < ERR_MT; ++mt) af[mt] = As[buf][(ks * 4 + tq) * LDM + wm * ERR_WM + mt * 8 + gq];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[buf][(wn * 32 + nt * 8 + gq) * LDK + ks * 4 + tq];
#pragma unroll
      for (int mt = 0; mt < ERR_MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
    }
    if (last_k) {                            // epilogue of tile lt
      const bool dp = d_ok(m0);
      if (dp) {
        mbar_wait(&dbar, dphase);
        dphase ^= 1;
      }
      const bool fullt = dp && m0 + GT <= g.M && n0 + GT <= g.N;
      if (fullt) {                           // fast path: compile-time smem offsets, 4 chains
        const double* dbase = Ds + (wn * 32 + tq * 2) * DLD + wm * ERR_WM + gq;
        double ea[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt) {
              const double e = dbase[(nt * 8 + h) * DLD + mt * 8] - acc[mt][nt][h];
              ea[(mt + 2 * h) & 3] = fma(e, e, ea[(mt + 2 * h) & 3]);
              acc[mt][nt][h] = 0.0;
            }
        e2 += (ea[0] + ea[1]) + (ea[2] + ea[3]);
      } else {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t c = n0 + wn * 32 + nt * 8 + tq * 2 + h;
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt) {
              const int64_t r = m0 + wm * ERR_WM + mt * 8 + gq;
              if (r < g.M && c < g.N) {
                const double a = dp ? Ds[(c - n0) * DLD + (r - m0)]
                                    : __ldcs(g.A + (g.cmap ? (int64_t)g.cmap[c] : c) * g.lda + r);
                const double e = a - acc[mt][nt][h];
                e2 = fma(e, e, e2);
              }
              acc[mt][nt][h] = 0.0;
            }
          }
      }
    }
    if (more) {
      sstore(buf ^ 1);
      __syncthreads();                        // also: every thread is done with Ds before the next issue_d
      buf ^= 1;
    }
    if (last_k) { ++lt; m0 = m1; n0 = n1; ks_i = 0; } else { ++ks_i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o);
  if (lane == 0) red[warp] = e2;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < ERR_THREADS / 32; ++w) t += red[w];
    g.out[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// Fused error, warp-specialised: the same (tile, k-stage) walk and 4 x 4 consumer warps
// as k_err_persist, but the operands arrive by bulk copies issued by one producer warp
// into an EW_S-deep mbarrier ring, so no CTA-wide barrier sits in the DMMA loop (the
// register-staged kernel spends ~20 % of its issue slots waiting at __syncthreads).
//   A stage: EW_GK rows of A_I(m0 : m0 + 128, kb + l), one bulk copy per l (column-major
//            A_I: each is contiguous);
//   B stage: the EW_GK x 128 slab of T, pre-packed by k_pack_T into the padded
//            [128 columns][EW_LDK] shared-memory image (one 12 KB bulk copy; zeros beyond
//            k and beyond the last column, so the padded k rows of a ragged last stage add 0);
//   A_D:     the tile's 128 column copies into Ds, 32 per stage from EW_S - 1 stages into
//            the tile on, once the previous tile's epilogue released Ds (dempty).
// Requires 16 B aligned A_I with an even row count (the copies move whole 16 B units).
// ---------------------------------------------------------------------------
constexpr int EW_GK = 8, EW_LDK = 12, EW_S = 4, EW_CONS = 16, EW_THREADS = (EW_CONS + 1) * 32;
constexpr int EW_ASZ = EW_GK * LDM, EW_BSZ = GT * EW_LDK;
__host__ __device__ inline int ew_nks(int64_t K) { return (int)((K + EW_GK - 1) / EW_GK); }
size_t ew_tpack_doubles(int64_t n, int64_t k) {
  return (size_t)((n + GT - 1) / GT) * ew_nks(k) * EW_BSZ;
}

__global__ void k_pack_T(const double* __restrict__ T, int64_t ldt, int K, int N, int nks, double* __restrict__ Tp,
                         int64_t total) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = idx / EW_BSZ;
    const int rem = (int)(idx - blk * EW_BSZ);
    const int c = rem / EW_LDK, kk = rem - c * EW_LDK;
    const int64_t ct = blk / nks, ks = blk - ct * nks;
    const int64_t kg = ks * EW_GK + kk, col = ct * GT + c;
    Tp[idx] = (kk < EW_GK && kg < K && col < N) ? T[col * ldt + kg] : 0.0;
  }
}

// STORE = true: the same walk computes out = X T (Q1 = A_I R1^{-1} of the LSQ refit)
// and stores it; no A_D block, no residual.
template <bool STORE>
__global__ void __launch_bounds__(EW_THREADS, 1) k_err_ws(GemmArgs g, const double* __restrict__ Tp,
                                                          int64_t ntiles, int ncb) {
  extern __shared__ __align__(128) double dsm[];
  double* As = dsm;                                   // [EW_S][EW_GK][LDM]
  double* Bs = dsm + EW_S * EW_ASZ;                   // [EW_S][GT][EW_LDK]
  double* Ds = Bs + EW_S * EW_BSZ;                    // [GT][DLD]
  __shared__ __align__(8) uint64_t full[EW_S], empty[EW_S], dfull, dempty;
  __shared__ double red[EW_CONS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t K = g.K;
  const int nks = ew_nks(K);
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  for (int i = tid; i < EW_S * EW_ASZ; i += EW_THREADS) As[i] = 0.0;   // finite stale rows
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < EW_S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], EW_CONS);
    }
    mbar_init(&dfull, 1);
    mbar_init(&dempty, EW_CONS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto tile_of = [&](int64_t lt, int64_t& m0, int64_t& n0) {
    const int64_t t = blockIdx.x + lt * gridDim.x;
    m0 = (t / ncb) * GT;
    n0 = (t % ncb) * GT;
  };
  if (warp == EW_CONS) {                              // producer warp
    int64_t j = 0;
    const int dstage = nks - 1 < EW_S - 1 ? nks - 1 : EW_S - 1;
    for (int64_t lt = 0; lt < my_tiles; ++lt) {
      int64_t m0, n0;
      tile_of(lt, m0, n0);
      const int64_t rows = (g.M - m0 < GT) ? g.M - m0 : (int64_t)GT;
      const int cols = (int)((g.N - n0 < GT) ? g.N - n0 : (int64_t)GT);
      const double* tsrc = Tp + (n0 / GT) * nks * EW_BSZ;
      int src[GT / 32];
      for (int ks = 0; ks < nks; ++ks, ++j) {
        const int s = (int)(j % EW_S);
        if (j >= EW_S) mbar_wait(&empty[s], (uint32_t)(((j / EW_S) - 1) & 1));
        const int64_t kb = (int64_t)ks * EW_GK;
        const int nk = (int)((K - kb < EW_GK) ? K - kb : (int64_t)EW_GK);
        if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(nk * rows * 8 + EW_BSZ * 8));
        __syncwarp();
        if (lane < nk)
          tma_load(As + s * EW_ASZ + lane * LDM, g.X + (kb + lane) * g.ldx + m0, (uint32_t)(rows * 8), &full[s]);
        else if (lane == 31)
          tma_load(Bs + s * EW_BSZ, tsrc + (int64_t)ks * EW_BSZ, (uint32_t)(EW_BSZ * 8), &full[s]);
        // the tile's A_D block, 32 columns per stage after that stage's operands (one
        // 128 KB burst would queue ahead of the next stages' copies)
        if (!STORE && ks == dstage) {
          if (lt > 0) mbar_wait(&dempty, (uint32_t)((lt - 1) & 1));
#pragma unroll
          for (int q = 0; q < GT / 32; ++q) {
            const int64_t c = n0 + lane + 32 * q;
            src[q] = c < g.N ? (g.cmap ? g.cmap[c] : (int)c) : 0;
          }
          if (lane == 0) mbar_expect_tx(&dfull, (uint32_t)(rows * cols * 8));
          __syncwarp();
        }
        if (!STORE && ks >= dstage) {
          const int qi = ks - dstage;
#pragma unroll
          for (int q = 0; q < GT / 32; ++q) {
            const int c = lane + 32 * q;
            if ((q == qi || (ks == nks - 1 && q > qi)) && c < cols)
              tma_load(Ds + c * DLD, g.A + (int64_t)src[q] * g.lda + m0, (uint32_t)(rows * 8), &dfull);
          }
        }
      }
    }
  } else {                                            // 16 consumer warps, 4 x 4, warp tile 32 x 32
    const int gq = lane >> 2, tq = lane & 3;
    const int wm = warp >> 2, wn = warp & 3;
    double acc[ERR_MT][4][2];
#pragma unroll
    for (int a = 0; a < ERR_MT; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    double e2 = 0.0;
    int64_t j = 0;
    for (int64_t lt = 0; lt < my_tiles; ++lt) {
      int64_t m0, n0;
      tile_of(lt, m0, n0);
      const bool active = m0 + wm * ERR_WM < g.M && n0 + wn * 32 < g.N;
      for (int ks = 0; ks < nks; ++ks, ++j) {
        const int s = (int)(j % EW_S);
        mbar_wait(&full[s], (uint32_t)((j / EW_S) & 1));
        const double* as = As + s * EW_ASZ + tq * LDM + wm * ERR_WM + gq;
        const double* bs = Bs + s * EW_BSZ + (wn * 32 + gq) * EW_LDK + tq;
        const int64_t kb = (int64_t)ks * EW_GK;
        if (active) {
#pragma unroll
          for (int k4 = 0; k4 < EW_GK / 4; ++k4) {
            if (kb + k4 * 4 >= K) break;
            double af[ERR_MT], bf[4];
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt) af[mt] = as[k4 * 4 * LDM + mt * 8];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) bf[nt] = bs[nt * 8 * EW_LDK + k4 * 4];
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt)
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      // epilogue of tile lt
      if (STORE) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t c = n0 + wn * 32 + nt * 8 + tq * 2 + h;
            double cm = 0.0;
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt) {
              const int64_t r = m0 + wm * ERR_WM + mt * 8 + gq;
              if (r < g.M && c < g.N) {
                g.out[c * g.ldo + r] = acc[mt][nt][h];
                cm = fmax(cm, fabs(acc[mt][nt][h]));
              }
              acc[mt][nt][h] = 0.0;
            }
            if (g.cmax) {   // the column max for the int8 engine's slicing (lanes gq share c)
#pragma unroll
              for (int o = 4; o < 32; o <<= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
              if (gq == 0 && c < g.N) atomicMax(g.cmax + c, (unsigned long long)__double_as_longlong(cm));
            }
          }
        continue;
      }
      mbar_wait(&dfull, (uint32_t)(lt & 1));
      if (m0 + GT <= g.M && n0 + GT <= g.N) {
        const double* dbase = Ds + (wn * 32 + tq * 2) * DLD + wm * ERR_WM + gq;
        double ea[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt) {
              const double e = dbase[(nt * 8 + h) * DLD + mt * 8] - acc[mt][nt][h];
              ea[(mt + 2 * h) & 3] = fma(e, e, ea[(mt + 2 * h) & 3]);
              acc[mt][nt][h] = 0.0;
            }
        e2 += (ea[0] + ea[1]) + (ea[2] + ea[3]);
      } else {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t c = n0 + wn * 32 + nt * 8 + tq * 2 + h;
#pragma unroll
            for (int mt = 0; mt < ERR_MT; ++mt) {
              const int64_t r = m0 + wm * ERR_WM + mt * 8 + gq;
              if (r < g.M && c < g.N) {
                const double e = Ds[(c - n0) * DLD + (r - m0)] - acc[mt][nt][h];
                e2 = fma(e, e, e2);
              }
              acc[mt][nt][h] = 0.0;
            }
          }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    if (lane == 0) red[warp] = e2;
  }
  if (STORE) return;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < EW_CONS; ++w) t += red[w];
    g.out[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// TN split-K GEMM with a TC_NS-stage cp.async pipeline (the A_I^T A_I, Q1^T Q1 and
// Q1^T A_D(:, J) products of the LSQ refit): the copy engine moves 16-byte chunks
// straight into shared memory TN_S - 1 stages ahead, so the DMMA loop never waits on
// a register round trip.  Requires 16-byte aligned columns (even ld, aligned bases);
// other shapes use k_dgemm.
// ---------------------------------------------------------------------------
constexpr int TN_S = 4;
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


// The same GEMM with the barrier taken out of the DMMA loop: 2 producer warps issue the
// 16-byte cp.async chunks of each stage (zero-filled outside the matrix, as above) and
// signal a TP_S-deep mbarrier ring with cp.async.mbarrier.arrive.noinc; the 8 consumer
// warps wait on the ring and release each stage with one arrive per warp.
constexpr int TP_S = 5, TP_PROD = 128, TP_THREADS = 256 + TP_PROD;
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}
template <int MT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_dgemm_tn_pipe(GemmArgs g) {
  constexpr int BM = 16 * MT;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                                  // [TP_S][BM][LDK]
  double* Bs = dsm + TP_S * BM * LDK;                // [TP_S][GT][LDK]
  __shared__ __align__(8) uint64_t full[TP_S], empty[TP_S];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * GT;
  const int64_t k_begin = (int64_t)blockIdx.z * g.k_per_split;
  const int64_t k_end = min(g.K, k_begin + g.k_per_split);
  const int nst = k_begin < k_end ? (int)((k_end - k_begin + GK - 1) / GK) : 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TP_S; ++s) {
      mbar_init(&full[s], TP_PROD);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= 8) {                                   // producers
    const int pt = tid - 256;
    constexpr int BQ = GT * 8 / TP_PROD;             // B chunks per producer thread per stage
    const double* bsrc[BQ];
#pragma unroll
    for (int q = 0; q < BQ; ++q) {
      const int mn = (pt + q * TP_PROD) >> 3;
      const int64_t c = n0 + mn;
      bsrc[q] = c < g.N ? g.Y + (g.ycmap ? (int64_t)g.ycmap[c] : c) * g.ldy : nullptr;
    }
    for (int j = 0; j < nst; ++j) {
      const int s = j % TP_S;
      if (j >= TP_S) mbar_wait(&empty[s], (uint32_t)(((j / TP_S) - 1) & 1));
      const int64_t kb = k_begin + (int64_t)j * GK;
      for (int idx = pt; idx < BM * 8; idx += TP_PROD) {
        const int mn = idx >> 3, kk = (idx & 7) * 2;
        const int64_t i = m0 + mn, r = kb + kk;
        const bool v = i < g.M && r < k_end;
        cp_async16(&As[((size_t)s * BM + mn) * LDK + kk], v ? g.X + i * g.ldx + r : g.X, v);
      }
#pragma unroll
      for (int q = 0; q < BQ; ++q) {
        const int idx = pt + q * TP_PROD, mn = idx >> 3, kk = (idx & 7) * 2;
        const int64_t r = kb + kk;
        const bool v = bsrc[q] != nullptr && r < k_end;
        cp_async16(&Bs[((size_t)s * GT + mn) * LDK + kk], v ? bsrc[q] + r : g.Y, v);
      }
      cp_async_mbar_arrive(&full[s]);
    }
    return;
  }
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  double acc[MT][4][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const bool idle = m0 + wm * 8 * MT >= g.M || n0 + wn * 32 >= g.N;
  for (int it = 0; it < nst; ++it) {
    const int s = it % TP_S;
    mbar_wait(&full[s], (uint32_t)((it / TP_S) & 1));
    const int64_t krem = (k_end - (k_begin + (int64_t)it * GK) + 3) / 4;
    const int ksteps = idle ? 0 : (krem < GK / 4 ? (int)krem : GK / 4);
    const double* Ab = As + (size_t)s * BM * LDK;
    const double* Bb = Bs + (size_t)s * GT * LDK;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      if (ks >= ksteps) break;
      double af[MT], bf[4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) af[mt] = Ab[(wm * (8 * MT) + mt * 8 + gq) * LDK + ks * 4 + tq];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = Bb[(wn * 32 + nt * 8 + gq) * LDK + ks * 4 + tq];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  double* o = g.out + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int64_t i = m0 + wm * (8 * MT) + mt * 8 + gq;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = n0 + wn * 32 + nt * 8 + tq * 2 + h;
        if (i < g.M && c < g.N) o[c * g.M + i] = acc[mt][nt][h];
      }
  }
}

// The same pipeline with an 8-row M granularity: all 8 consumer warps cover the CTA's
// BM = 8 MR rows (MR m8 tiles) x 16 columns, so k = 100 pads to 104 rows instead of the
// 112 of the (16 MT) x 128 tiling (7 % fewer DMMAs for the LSQ products at k = 100).
template <int MR>
__global__ void __launch_bounds__(TP_THREADS, 1) k_dgemm_tn_pipe8(GemmArgs g) {
  constexpr int BM = 8 * MR;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                                  // [TP_S][BM][LDK]
  double* Bs = dsm + TP_S * BM * LDK;                // [TP_S][GT][LDK]
  __shared__ __align__(8) uint64_t full[TP_S], empty[TP_S];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * GT;
  const int64_t k_begin = (int64_t)blockIdx.z * g.k_per_split;
  const int64_t k_end = min(g.K, k_begin + g.k_per_split);
  const int nst = k_begin < k_end ? (int)((k_end - k_begin + GK - 1) / GK) : 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TP_S; ++s) {
      mbar_init(&full[s], TP_PROD);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= 8) {                                   // producers
    const int pt = tid - 256;
    constexpr int BQ = GT * 8 / TP_PROD;
    const double* bsrc[BQ];
#pragma unroll
    for (int q = 0; q < BQ; ++q) {
      const int mn = (pt + q * TP_PROD) >> 3;
      const int64_t c = n0 + mn;
      bsrc[q] = c < g.N ? g.Y + (g.ycmap ? (int64_t)g.ycmap[c] : c) * g.ldy : nullptr;
    }
    for (int j = 0; j < nst; ++j) {
      const int s = j % TP_S;
      if (j >= TP_S) mbar_wait(&empty[s], (uint32_t)(((j / TP_S) - 1) & 1));
      const int64_t kb = k_begin + (int64_t)j * GK;
      for (int idx = pt; idx < BM * 8; idx += TP_PROD) {
        const int mn = idx >> 3, kk = (idx & 7) * 2;
        const int64_t i = m0 + mn, r = kb + kk;
        const bool v = i < g.M && r < k_end;
        cp_async16(&As[((size_t)s * BM + mn) * LDK + kk], v ? g.X + i * g.ldx + r : g.X, v);
      }
#pragma unroll
      for (int q = 0; q < BQ; ++q) {
        const int idx = pt + q * TP_PROD, mn = idx >> 3, kk = (idx & 7) * 2;
        const int64_t r = kb + kk;
        const bool v = bsrc[q] != nullptr && r < k_end;
        cp_async16(&Bs[((size_t)s * GT + mn) * LDK + kk], v ? bsrc[q] + r : g.Y, v);
      }
      cp_async_mbar_arrive(&full[s]);
    }
    return;
  }
  const int gq = lane >> 2, tq = lane & 3;
  const int wn = warp;                               // 8 warps along N, 16 columns each
  double acc[MR][2][2];
#pragma unroll
  for (int a = 0; a < MR; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const bool idle = n0 + wn * 16 >= g.N;
  for (int it = 0; it < nst; ++it) {
    const int s = it % TP_S;
    mbar_wait(&full[s], (uint32_t)((it / TP_S) & 1));
    const int64_t krem = (k_end - (k_begin + (int64_t)it * GK) + 3) / 4;
    const int ksteps = idle ? 0 : (krem < GK / 4 ? (int)krem : GK / 4);
    const double* Ab = As + (size_t)s * BM * LDK;
    const double* Bb = Bs + (size_t)s * GT * LDK;
#pragma unroll
    for (int ks = 0; ks < GK / 4; ++ks) {
      if (ks >= ksteps) break;
      double af[MR], bf[2];
#pragma unroll
      for (int mt = 0; mt < MR; ++mt) af[mt] = Ab[(mt * 8 + gq) * LDK + ks * 4 + tq];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) bf[nt] = Bb[(wn * 16 + nt * 8 + gq) * LDK + ks * 4 + tq];
#pragma unroll
      for (int mt = 0; mt < MR; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  double* o = g.out + (int64_t)blockIdx.z * g.M * g.N;
#pragma unroll
  for (int mt = 0; mt < MR; ++mt) {
    const int64_t i = m0 + mt * 8 + gq;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t c = n0 + wn * 16 + nt * 8 + tq * 2 + h;
        if (i < g.M && c < g.N) o[c * g.M + i] = acc[mt][nt][h];
      }
  }
}
template <int MR>
static cudaError_t tn_pipe8_launch_t(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  const size_t smem = (size_t)TP_S * (8 * MR + GT) * LDK * sizeof(double);
  cudaError_t e = smem_attr((const void*)k_dgemm_tn_pipe8<MR>, (int)smem);
  if (e != cudaSuccess) return e;
  k_dgemm_tn_pipe8<MR><<<grid, TP_THREADS, smem, st>>>(g);
  return cudaGetLastError();
}
// M <= 128 whose 8-row padding is smaller than its 16-row padding: 8 MR rows per CTA
static bool tn_pipe8_launch(const GemmArgs& g, dim3 grid, cudaStream_t st, cudaError_t* err) {
  static const bool off = getenv("MPID_TN_NO_PIPE8") != nullptr;   // A/B switch for measurements
  const int64_t M = g.M;
  if (off || M > 128 || (M + 7) / 8 * 8 == (M + 15) / 16 * 16 || M <= 48) return false;
  const int mr = (int)((M + 7) / 8);
  grid.x = 1;
  switch (mr) {
    case 7: *err = tn_pipe8_launch_t<7>(g, grid, st); break;
    case 9: *err = tn_pipe8_launch_t<9>(g, grid, st); break;
    case 11: *err = tn_pipe8_launch_t<11>(g, grid, st); break;
    case 13: *err = tn_pipe8_launch_t<13>(g, grid, st); break;
    case 15: *err = tn_pipe8_launch_t<15>(g, grid, st); break;
    default: return false;
  }
  return true;
}

template <int MT>
static cudaError_t tn_async_launch_t(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  cudaError_t e8 = cudaSuccess;
  if (tn_pipe8_launch(g, grid, st, &e8)) return e8;
  const size_t smem_p = (size_t)TP_S * (16 * MT + GT) * LDK * sizeof(double);
  cudaError_t e = smem_attr((const void*)k_dgemm_tn_pipe<MT>, (int)smem_p);
  if (e != cudaSuccess) return e;
  k_dgemm_tn_pipe<MT><<<grid, TP_THREADS, smem_p, st>>>(g);
  return cudaGetLastError();
}
static cudaError_t tn_async_launch(const GemmArgs& g, dim3 grid, cudaStream_t st, int mt) {
  switch (mt) {
    case 3: return tn_async_launch_t<3>(g, grid, st);
    case 4: return tn_async_launch_t<4>(g, grid, st);
    case 5: return tn_async_launch_t<5>(g, grid, st);
    case 6: return tn_async_launch_t<6>(g, grid, st);
    case 7: return tn_async_launch_t<7>(g, grid, st);
    default: return tn_async_launch_t<8>(g, grid, st);
  }
}

template <int MODE>
static size_t dgemm_smem() {
  const int a = (MODE == GM_TN_PARTIAL) ? GT * LDK : GK * LDM;
  return (size_t)(2 * (a + GT * LDK)) * sizeof(double);
}
template <int MODE, int MT>
static cudaError_t dgemm_launch_t(const GemmArgs& g, dim3 grid, cudaStream_t st) {
  cudaError_t e = smem_attr((const void*)k_dgemm<MODE, MT>, (int)dgemm_smem<MODE>());
  if (e != cudaSuccess) return e;
  k_dgemm<MODE, MT><<<grid, 256, dgemm_smem<MODE>(), st>>>(g);
  return cudaGetLastError();
}
// M tile 16 MT: the smallest of 48/64/80/96/112/128 covering M (k-sized M wastes less)
static int pick_mt(int64_t M) {
  if (M >= 128) return 8;
  return (int)std::max<int64_t>(3, (M + 15) / 16);
}
template <int MODE>
static cudaError_t dgemm_launch(GemmArgs g, dim3 grid, cudaStream_t st, int mt) {
  switch (mt) {
    case 3: return dgemm_launch_t<MODE, 3>(g, grid, st);
    case 4: return dgemm_launch_t<MODE, 4>(g, grid, st);
    case 5: return dgemm_launch_t<MODE, 5>(g, grid, st);
    case 6: return dgemm_launch_t<MODE, 6>(g, grid, st);
    case 7: return dgemm_launch_t<MODE, 7>(g, grid, st);
    default: return dgemm_launch_t<MODE, 8>(g, grid, st);
  }
}

// ---------------------------------------------------------------------------
// Cholesky G = L L^T (lower, col-major k x k) in one CTA; returns R = L^T
// (upper, col-major) in place of G's upper triangle.  info = 0 or j+1 at the
// first non-positive pivot (breakdown -> ID_ERR_DEGENERATE).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_cholesky(double* __restrict__ G, int k, int* __restrict__ info) {
  extern __shared__ double sG[];
  const bool in_smem = (size_t)k * k * sizeof(double) <= 160 * 1024;
  double* L = in_smem ? sG : G;
  if (in_smem)
    for (int i = threadIdx.x; i < k * k; i += blockDim.x) sG[i] = G[i];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (threadIdx.x == 0) {
      const double d = L[j + (int64_t)j * k];
      if (!(d > 0.0)) bad = bad ? bad : j + 1;
      L[j + (int64_t)j * k] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    const double djj = L[j + (int64_t)j * k];
    for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) L[i + (int64_t)j * k] /= djj;
    __syncthreads();
    {   // trailing update, warps over columns l, lanes over rows i >= l (no integer division)
      const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int l = j + 1 + (threadIdx.x >> 5); l < k; l += nw) {
        const double ljl = L[l + (int64_t)j * k];
        for (int i = l + lane; i < k; i += 32) L[i + (int64_t)l * k] -= L[i + (int64_t)j * k] * ljl;
      }
    }
    __syncthreads();
  }
  // R(j, i) = L(i, j) for i >= j, then zero below the diagonal (two passes: in-place safe)
  for (int64_t idx = threadIdx.x; idx < (int64_t)k * k; idx += blockDim.x) {
    const int r = (int)(idx % k), c = (int)(idx / k);
    if (c >= r) G[r + (int64_t)c * k] = L[c + (int64_t)r * k];
  }
  __syncthreads();
  for (int64_t idx = threadIdx.x; idx < (int64_t)k * k; idx += blockDim.x) {
    const int r = (int)(idx % k), c = (int)(idx / k);
    if (c < r) G[r + (int64_t)c * k] = 0.0;
  }
  if (threadIdx.x == 0) *info = bad;
}

// The same factorisation with ONE block barrier per step (k <= 143, G in shared memory):
// every thread forms sqrt(d) and 1 / d of the pivot itself, the trailing update uses the
// unscaled column j with the factor 1 / d, and the scaled column goes straight to its place
// in R's upper triangle in global memory (never read back during the sweep).
__global__ void __launch_bounds__(1024) k_cholesky_1bar(double* __restrict__ G, int k, int* __restrict__ info) {
  extern __shared__ double sG[];
  double* L = sG;
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) L[i] = G[i];
  __syncthreads();
  int bad = 0;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = 0; j < k; ++j) {
    const double d0 = L[j + (int64_t)j * k];
    const bool ok = d0 > 0.0;
    if (!ok && !bad) bad = j + 1;
    const double d = ok ? d0 : 1.0;
    const double sd = sqrt(d), rs = 1.0 / sd, inv = 1.0 / d;
    for (int i = j + threadIdx.x; i < k; i += blockDim.x)          // R(j, i) = L(i, j)
      G[j + (int64_t)i * k] = i == j ? sd : L[i + (int64_t)j * k] * rs;
    for (int l = j + 1 + (threadIdx.x >> 5); l < k; l += nw) {     // L(i, l) -= L(i, j) L(l, j) / d
      const double t = L[l + (int64_t)j * k] * inv;
      for (int i = l + lane; i < k; i += 32) L[i + (int64_t)l * k] = fma(-L[i + (int64_t)j * k], t, L[i + (int64_t)l * k]);
    }
    __syncthreads();
  }
  for (int64_t idx = threadIdx.x; idx < (int64_t)k * k; idx += blockDim.x) {
    const int r = (int)(idx % k), c = (int)(idx / k);
    if (c < r) G[r + (int64_t)c * k] = 0.0;
  }
  if (threadIdx.x == 0) *info = bad;
}

// ---------------------------------------------------------------------------
// Cholesky for k > 143 (G does not fit shared memory): left-looking, panels of 16
// columns.  Thread t owns row p0 + t of the panel: the update with the finished
// columns streams L(:, l) from global (coalesced) against a 64 x 16 shared chunk
// of L(p0:p0+16, l), then the panel is factored in shared memory and written back.
// Same output convention as k_cholesky (R = L^T in the upper triangle, info).
// ---------------------------------------------------------------------------
constexpr int CH_NB = 16, CH_LC = 64;   // 16-column panels: 16 fp64 accumulators per thread at 1024 threads
__global__ void __launch_bounds__(1024) k_cholesky_blocked(double* __restrict__ G, int k, int* __restrict__ info) {
  extern __shared__ double pn[];                    // panel [k][CH_NB + 1]
  __shared__ double lb[CH_LC][CH_NB];               // L(p0 + c, l0 + l)
  __shared__ int bad;
  const int t = threadIdx.x;
  if (t == 0) bad = 0;
  __syncthreads();
  for (int p0 = 0; p0 < k; p0 += CH_NB) {
    const int w = min(CH_NB, k - p0), rows = k - p0;
    double acc[CH_NB];
#pragma unroll
    for (int c = 0; c < CH_NB; ++c) acc[c] = (t < rows && c < w) ? G[(int64_t)(p0 + t) + (int64_t)(p0 + c) * k] : 0.0;
    for (int l0 = 0; l0 < p0; l0 += CH_LC) {
      const int lw = min(CH_LC, p0 - l0);
      __syncthreads();
      for (int e = t; e < CH_LC * CH_NB; e += blockDim.x) {
        const int l = e / CH_NB, c = e % CH_NB;
        lb[l][c] = (l < lw && c < w) ? G[(int64_t)(p0 + c) + (int64_t)(l0 + l) * k] : 0.0;
      }
      __syncthreads();
      if (t < rows) {
        for (int l = 0; l < lw; ++l) {
          const double a = G[(int64_t)(p0 + t) + (int64_t)(l0 + l) * k];
#pragma unroll
          for (int c = 0; c < CH_NB; ++c) acc[c] = fma(-a, lb[l][c], acc[c]);
        }
      }
    }
    if (t < rows) {
#pragma unroll
      for (int c = 0; c < CH_NB; ++c) pn[t * (CH_NB + 1) + c] = acc[c];
    }
    __syncthreads();
    for (int c = 0; c < w; ++c) {                      // factor the panel
      if (t == 0) {
        const double d = pn[c * (CH_NB + 1) + c];
        if (!(d > 0.0) && !bad) bad = p0 + c + 1;
        pn[c * (CH_NB + 1) + c] = d > 0.0 ? sqrt(d) : 1.0;
      }
      __syncthreads();
      const double djj = pn[c * (CH_NB + 1) + c];
      if (t > c && t < rows) pn[t * (CH_NB + 1) + c] /= djj;
      __syncthreads();
      if (t > c && t < rows) {
        const double lic = pn[t * (CH_NB + 1) + c];
        for (int c2 = c + 1; c2 < w && c2 <= t; ++c2) pn[t * (CH_NB + 1) + c2] -= lic * pn[c2 * (CH_NB + 1) + c];
      }
      __syncthreads();
    }
    if (t < rows) {
      for (int c = 0; c < w && c <= t; ++c) G[(int64_t)(p0 + t) + (int64_t)(p0 + c) * k] = pn[t * (CH_NB + 1) + c];
    }
    __syncthreads();
  }
  for (int64_t idx = t; idx < (int64_t)k * k; idx += blockDim.x) {
    const int r = (int)(idx % k), c = (int)(idx / k);
    if (c > r) G[r + (int64_t)c * k] = G[c + (int64_t)r * k];
  }
  __syncthreads();
  for (int64_t idx = t; idx < (int64_t)k * k; idx += blockDim.x) {
    const int r = (int)(idx % k), c = (int)(idx / k);
    if (c < r) G[r + (int64_t)c * k] = 0.0;
  }
  if (t == 0) *info = bad;
}

// ---------------------------------------------------------------------------
// Small left triangular solves on a block of 32 right-hand sides held in
// shared memory (the fp64 triangular solve for P).  For column i of the block,
// b = B(:, map[i]) (map = perm + k for W(:, J), or identity + k for R12):
//   mode 0 (R mode):   T = R1^{-1} b
//   mode 1 (LSQ mode): T = R1^{-1} R2^{-1} R2^{-T} b    (G2 = R2^T R2)
// R1, R2 upper, col-major k x k.  One CTA per 32 columns, 1024 threads.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_trsm_left_block(const double* __restrict__ R1,
                                                          const double* __restrict__ R2, int k,
                                                          const double* __restrict__ B, int64_t ldb,
                                                          const int* __restrict__ map, int ncols,
                                                          double* __restrict__ T, int64_t ldt,
                                                          int mode) {
  extern __shared__ double sb[];  // [k][33], then (k <= 128) the triangular factor in use, k x k
  double* su = sb + (size_t)k * 33;
  const bool u_smem = k <= 128;
  const int c = threadIdx.x & 31, rg = threadIdx.x >> 5;  // column in block, row group (32)
  const int col = blockIdx.x * 32 + c;
  const bool valid = col < ncols;
  const int64_t src = valid ? (int64_t)(map ? map[col] : col) : 0;
  for (int r = rg; r < k; r += 32) sb[r * 33 + c] = valid ? B[src * ldb + r] : 0.0;
  __syncthreads();
  auto stage = [&](const double* U) -> const double* {   // the factor into shared memory (k <= 128)
    if (!u_smem) return U;
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) su[e] = U[e];
    __syncthreads();
    return su;
  };
  auto back = [&](const double* U) {          // solve U x = b (upper), column sweep
    U = stage(U);
    for (int i = k - 1; i >= 0; --i) {
      const double xi = sb[i * 33 + c] / U[i + (int64_t)i * k];
      __syncthreads();
      if (rg == 0) sb[i * 33 + c] = xi;
      for (int r = rg; r < i; r += 32) sb[r * 33 + c] = fma(-U[r + (int64_t)i * k], xi, sb[r * 33 + c]);
      __syncthreads();
    }
  };
  auto fwdT = [&](const double* U) {          // solve U^T x = b (lower), column sweep
    U = stage(U);
    for (int i = 0; i < k; ++i) {
      const double xi = sb[i * 33 + c] / U[i + (int64_t)i * k];
      __syncthreads();
      if (rg == 0) sb[i * 33 + c] = xi;
      for (int r = i + 1 + rg; r < k; r += 32) sb[r * 33 + c] = fma(-U[i + (int64_t)r * k], xi, sb[r * 33 + c]);
      __syncthreads();
    }
  };
  if (mode == 1) {
    fwdT(R2);
    back(R2);
  }
  back(R1);
  if (valid)
    for (int r = rg; r < k; r += 32) T[(int64_t)col * ldt + r] = sb[r * 33 + c];
}

// The same solves for k <= 128 without block barriers: one WARP per right-hand side, each lane
// holding rows lane + 32 q (q < RPL) of it in registers; step i broadcasts x_i from its owner
// lane by a shuffle and the lanes update their rows with the column (or row) i of the factor,
// staged in shared memory with an odd column stride (conflict-free both ways) together with
// its reciprocal diagonal (multiplications on the sweep's critical path, no divisions).
// 8 right-hand sides per CTA; the factors are staged one at a time.
constexpr int TW_WARPS = 8;
template <int RPL>
__device__ __forceinline__ void tw_back(double (&b)[RPL], const double* su, const double* dinv, int k, int ldu,
                                        int lane) {   // U x = b (upper), rows bottom-up
#pragma unroll
  for (int qb = RPL - 1; qb >= 0; --qb) {              // the owner slot of row i is compile-time
    for (int ii = 31; ii >= 0; --ii) {
      const int i = qb * 32 + ii;
      if (i >= k) continue;
      const double xi = __shfl_sync(0xffffffffu, b[qb], ii) * dinv[i];
      const double* Ui = su + (size_t)i * ldu;
#pragma unroll
      for (int q = 0; q <= qb; ++q) {
        const int r = lane + 32 * q;
        if (r < i) b[q] = fma(-Ui[r], xi, b[q]);
        else if (r == i) b[q] = xi;
      }
    }
  }
}
template <int RPL>
__device__ __forceinline__ void tw_fwdT(double (&b)[RPL], const double* su, const double* dinv, int k, int ldu,
                                        int lane) {   // U^T x = b (lower), rows top-down: U(i, r) = su[i + r ldu]
#pragma unroll
  for (int qb = 0; qb < RPL; ++qb) {
    for (int ii = 0; ii < 32; ++ii) {
      const int i = qb * 32 + ii;
      if (i >= k) break;
      const double xi = __shfl_sync(0xffffffffu, b[qb], ii) * dinv[i];
#pragma unroll
      for (int q = qb; q < RPL; ++q) {
        const int r = lane + 32 * q;
        if (r > i && r < k) b[q] = fma(-su[i + (size_t)r * ldu], xi, b[q]);
        else if (r == i) b[q] = xi;
      }
    }
  }
}
__device__ __forceinline__ void tw_stage(const double* __restrict__ U, double* su, double* dinv, int k, int ldu) {
  __syncthreads();
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int r = e % k, c = e / k;
    su[r + (size_t)c * ldu] = U[e];
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) dinv[i] = 1.0 / U[i + (int64_t)i * k];
  __syncthreads();
}
template <int RPL>
__global__ void __launch_bounds__(TW_WARPS * 32) k_trsm_warp(const double* __restrict__ R1,
                                                             const double* __restrict__ R2, int k,
                                                             const double* __restrict__ B, int64_t ldb,
                                                             const int* __restrict__ map, int ncols,
                                                             double* __restrict__ T, int64_t ldt, int mode) {
  extern __shared__ double su[];   // [k][ldu] factor, then [k] reciprocal diagonal
  const int ldu = (k & 1) ? k : k + 1;
  double* dinv = su + (size_t)k * ldu;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * TW_WARPS + warp;
  const bool valid = col < ncols;
  double b[RPL];
  const int64_t src = valid ? (int64_t)(map ? map[col] : col) : 0;
#pragma unroll
  for (int q = 0; q < RPL; ++q) {
    const int r = lane + 32 * q;
    b[q] = (valid && r < k) ? B[src * ldb + r] : 0.0;
  }
  if (mode == 1) {
    tw_stage(R2, su, dinv, k, ldu);
    tw_fwdT<RPL>(b, su, dinv, k, ldu, lane);
    tw_back<RPL>(b, su, dinv, k, ldu, lane);
  }
  tw_stage(R1, su, dinv, k, ldu);
  tw_back<RPL>(b, su, dinv, k, ldu, lane);
  if (valid)
#pragma unroll
    for (int q = 0; q < RPL; ++q) {
      const int r = lane + 32 * q;
      if (r < k) T[(int64_t)col * ldt + r] = b[q];
    }
}

// R (k x n, fp32 or fp64, row-major, pivoted order) -> fp64 col-major k x n
template <typename RT>
__global__ void k_R_to_fp64(const RT* __restrict__ R, int k, int n, double* __restrict__ Rd) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)k * n) return;
  const int i = (int)(idx % k), c = (int)(idx / k);
  Rd[idx] = (double)R[(int64_t)i * n + c];
}

// R (k x n row-major) -> col-major k x n with leading dimension ldr (fp64 -> fp32 rounds)
template <typename RT, typename OT>
__global__ void k_R_export(const RT* __restrict__ R, int k, int n, OT* __restrict__ out, int64_t ldr) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)k * n) return;
  const int i = (int)(idx % k), c = (int)(idx / k);
  out[(int64_t)c * ldr + i] = (OT)R[(int64_t)i * n + c];
}

// P(:, perm[j]) = e_j (j < k), P(:, perm[k + i]) = T(:, i); col-major k x n, ldp
__global__ void k_assemble_P(const double* __restrict__ T, int64_t ldt, int k, int n,
                             const int* __restrict__ perm, double* __restrict__ P, int64_t ldp) {
  const int pos = blockIdx.x;
  const int orig = perm[pos];
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    double v;
    if (pos < k) v = (r == pos) ? 1.0 : 0.0;
    else v = T[(int64_t)(pos - k) * ldt + r];
    P[(int64_t)orig * ldp + r] = v;
  }
}

__global__ void k_sum_scalar(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  __shared__ double sh[32];
  double t = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) t += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x < 32) {
    t = threadIdx.x < (int)(blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) *out = t;
  }
}

// ---------------------------------------------------------------------------
cudaError_t launch_gather_cols(const double* A, int64_t m, int64_t ld, const int* perm, int k,
                               double* X, cudaStream_t st) {
  if (m % 2 == 0 && ld % 2 == 0 && ((((uintptr_t)A) | ((uintptr_t)X)) & 15) == 0) {
    dim3 grid2((unsigned)((m / 2 + 511) / 512), (unsigned)k);
    k_gather_cols2<<<grid2, 256, 0, st>>>(A, m, ld, perm, X);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((m + 255) / 256), (unsigned)k);
  k_gather_cols<<<grid, 256, 0, st>>>(A, m, ld, perm, X);
  return cudaGetLastError();
}

cudaError_t launch_tsmm(const double* X, int64_t ldx, int k1, const double* Y, int64_t ldy, int n1,
                        int64_t m, double* part, int splits, cudaStream_t st, const int* ycmap) {
  GemmArgs g{};
  g.X = X; g.ldx = ldx; g.Y = Y; g.ldy = ldy;
  g.M = k1; g.N = n1; g.K = m;
  g.ycmap = ycmap;
  g.k_per_split = ((m + splits - 1) / splits + GK - 1) / GK * GK;
  g.out = part;
  const int mt = pick_mt(k1);
  dim3 grid((unsigned)((k1 + 16 * mt - 1) / (16 * mt)), (unsigned)((n1 + GT - 1) / GT), (unsigned)splits);
  // the cp.async pipeline needs every 16-byte chunk aligned: even leading dimensions,
  // aligned bases, and split boundaries on even rows (k_per_split is a multiple of 16)
  const bool aligned = (ldx % 2 == 0) && (ldy % 2 == 0) && ((((uintptr_t)X) | ((uintptr_t)Y)) & 15) == 0 &&
                       (m % 2 == 0);
  if (aligned) return tn_async_launch(g, grid, st, mt);
  return dgemm_launch<GM_TN_PARTIAL>(g, grid, st, mt);
}

cudaError_t launch_cholesky(double* G, int k, int* info, cudaStream_t st) {
  const size_t sm = (size_t)k * k * sizeof(double);
  cudaError_t e = smem_attr((const void*)k_cholesky, 160 * 1024);
  if (e == cudaSuccess) e = smem_attr((const void*)k_cholesky_blocked, 200 * 1024);
  if (e != cudaSuccess) return e;
  static const bool one_bar = !(getenv("MPID_CHOL_3BAR") && atoi(getenv("MPID_CHOL_3BAR")) == 1);
  if (sm <= 160 * 1024 && one_bar) {
    e = smem_attr((const void*)k_cholesky_1bar, 160 * 1024);
    if (e != cudaSuccess) return e;
    k_cholesky_1bar<<<1, 1024, sm, st>>>(G, k, info);
  } else if (sm <= 160 * 1024) {
    k_cholesky<<<1, 1024, sm, st>>>(G, k, info);
  } else if (k <= 1024 && (size_t)k * (CH_NB + 1) * 8 <= 200 * 1024 - sizeof(double) * CH_LC * CH_NB) {
    k_cholesky_blocked<<<1, 1024, (size_t)k * (CH_NB + 1) * 8, st>>>(G, k, info);
  } else {
    k_cholesky<<<1, 1024, 0, st>>>(G, k, info);      // global-memory fallback (k > 700)
  }
  return cudaGetLastError();
}

cudaError_t launch_trsm_left_upper(const double* R1, const double* R2, int k, const double* B,
                                   int64_t ldb, const int* map, int ncols, double* T, int64_t ldt,
                                   int mode, cudaStream_t st) {
  if (ncols <= 0) return cudaSuccess;
  static const bool warp_env = !(getenv("MPID_TRSM_BLOCK") && atoi(getenv("MPID_TRSM_BLOCK")) == 1);
  if (warp_env && k <= 128) {   // one warp per right-hand side (k_trsm_warp)
    const size_t sw = ((size_t)k * ((k & 1) ? k : k + 1) + k) * sizeof(double);
    const unsigned grid = (unsigned)((ncols + TW_WARPS - 1) / TW_WARPS);
    const void* fn = k <= 32 ? (const void*)k_trsm_warp<1> : k <= 64 ? (const void*)k_trsm_warp<2>
                   : k <= 96 ? (const void*)k_trsm_warp<3> : (const void*)k_trsm_warp<4>;
    cudaError_t e = smem_attr(fn, (int)sw);
    if (e != cudaSuccess) return e;
    if (k <= 32) k_trsm_warp<1><<<grid, TW_WARPS * 32, sw, st>>>(R1, R2, k, B, ldb, map, ncols, T, ldt, mode);
    else if (k <= 64) k_trsm_warp<2><<<grid, TW_WARPS * 32, sw, st>>>(R1, R2, k, B, ldb, map, ncols, T, ldt, mode);
    else if (k <= 96) k_trsm_warp<3><<<grid, TW_WARPS * 32, sw, st>>>(R1, R2, k, B, ldb, map, ncols, T, ldt, mode);
    else k_trsm_warp<4><<<grid, TW_WARPS * 32, sw, st>>>(R1, R2, k, B, ldb, map, ncols, T, ldt, mode);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)k * 33 * sizeof(double) + (k <= 128 ? (size_t)k * k * sizeof(double) : 0);
  cudaError_t e = smem_attr((const void*)k_trsm_left_block, 200 * 1024);
  if (e != cudaSuccess) return e;
  k_trsm_left_block<<<(unsigned)((ncols + 31) / 32), 1024, smem, st>>>(R1, R2, k, B, ldb, map, ncols,
                                                                        T, ldt, mode);
  return cudaGetLastError();
}

cudaError_t launch_R_to_fp64(int r64, const void* R, int k, int n, double* Rd, cudaStream_t st) {
  const int64_t tot = (int64_t)k * n;
  const unsigned nb = (unsigned)((tot + 255) / 256);
  if (r64) k_R_to_fp64<double><<<nb, 256, 0, st>>>((const double*)R, k, n, Rd);
  else k_R_to_fp64<float><<<nb, 256, 0, st>>>((const float*)R, k, n, Rd);
  return cudaGetLastError();
}

cudaError_t launch_R_export(int r64, const void* R, int k, int n, void* out, int o64, int64_t ldr,
                            cudaStream_t st) {
  const int64_t tot = (int64_t)k * n;
  const unsigned nb = (unsigned)((tot + 255) / 256);
  if (r64 && o64) k_R_export<double, double><<<nb, 256, 0, st>>>((const double*)R, k, n, (double*)out, ldr);
  else if (r64) k_R_export<double, float><<<nb, 256, 0, st>>>((const double*)R, k, n, (float*)out, ldr);
  else if (o64) k_R_export<float, double><<<nb, 256, 0, st>>>((const float*)R, k, n, (double*)out, ldr);
  else k_R_export<float, float><<<nb, 256, 0, st>>>((const float*)R, k, n, (float*)out, ldr);
  return cudaGetLastError();
}

cudaError_t launch_assemble_P(const double* T, int64_t ldt, int k, int n, const int* perm, double* P,
                              int64_t ldp, cudaStream_t st) {
  k_assemble_P<<<n, 128, 0, st>>>(T, ldt, k, n, perm, P, ldp);
  return cudaGetLastError();
}

cudaError_t launch_error(const double* A, int64_t m, int64_t ld, int ncols, const int* cmap, const double* X,
                         int k, const double* T, int64_t ldt, double* part, int* nblk_out, cudaStream_t st,
                         double* tpack, size_t tpack_cap, int64_t ldx, int pack) {
  GemmArgs g{};
  g.X = X; g.ldx = ldx > 0 ? ldx : m;
  g.Y = T; g.ldy = ldt;
  g.M = m; g.N = ncols; g.K = k;
  g.out = part;
  g.A = A; g.lda = ld;
  g.cmap = cmap;
  g.d_tma = ((ld % 2) == 0 && (((uintptr_t)A) & 15) == 0) ? 1 : 0;
  const int64_t nrb = (m + GT - 1) / GT, ncb = (ncols + GT - 1) / GT;
  const int64_t ntiles = nrb * ncb;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<int64_t>(ntiles, sms);
  *nblk_out = grid;
  static const bool ws_off = getenv("MPID_ERR_NO_WS") != nullptr;   // A/B switch for measurements
  if (!ws_off && g.d_tma && m % 2 == 0 && (((uintptr_t)X) & 15) == 0 && tpack &&
      ew_tpack_doubles(ncols, k) <= tpack_cap) {
    const int nks = ew_nks(k);
    const int64_t tot = (int64_t)ew_tpack_doubles(ncols, k);
    if (pack)
      k_pack_T<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 4 * sms), 256, 0, st>>>(T, ldt, k, ncols, nks, tpack,
                                                                                      tot);
    const size_t smem_ws = (size_t)(EW_S * (EW_ASZ + EW_BSZ) + GT * DLD) * sizeof(double);
    cudaError_t e = smem_attr((const void*)k_err_ws<false>, (int)smem_ws);
    if (e != cudaSuccess) return e;
    k_err_ws<false><<<grid, EW_THREADS, smem_ws, st>>>(g, tpack, ntiles, (int)ncb);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)(2 * GK * LDM + 2 * GT * LDK + GT * DLD) * sizeof(double);
  cudaError_t e = smem_attr((const void*)k_err_persist, (int)smem);
  if (e != cudaSuccess) return e;
  *nblk_out = grid;
  k_err_persist<<<grid, ERR_THREADS, smem, st>>>(g, ntiles, (int)ncb);
  return cudaGetLastError();
}

cudaError_t launch_nn_store(const double* X, int64_t m, int64_t ldx, const double* B, int64_t ldb, int K,
                            int N, double* out, int64_t ldo, cudaStream_t st, double* tpack, size_t tpack_cap,
                            unsigned long long* cmax, int* cmax_done) {
  if (cmax_done) *cmax_done = 0;
  GemmArgs g{};
  g.X = X; g.ldx = ldx;
  g.Y = B; g.ldy = ldb;
  g.M = m; g.N = N; g.K = K;
  g.out = out; g.ldo = ldo;
  static const bool ws_off = getenv("MPID_NN_NO_WS") != nullptr;    // A/B switch for measurements
  if (!ws_off && tpack && ew_tpack_doubles(N, K) <= tpack_cap && m % 2 == 0 && ldx % 2 == 0 &&
      (((uintptr_t)X) & 15) == 0) {
    // the warp-specialised walk of the fused error in STORE mode (packed B slabs, bulk copies)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ncb = (N + GT - 1) / GT, ntiles = ((m + GT - 1) / GT) * ncb;
    const int nks = ew_nks(K);
    const int64_t tot = (int64_t)ew_tpack_doubles(N, K);
    k_pack_T<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 4 * sms), 256, 0, st>>>(B, ldb, K, N, nks, tpack, tot);
    const size_t smem_ws = (size_t)(EW_S * (EW_ASZ + EW_BSZ) + GT * DLD) * sizeof(double);
    cudaError_t e = smem_attr((const void*)k_err_ws<true>, (int)smem_ws);
    if (e != cudaSuccess) return e;
    g.cmax = cmax;
    if (cmax) {
      e = cudaMemsetAsync(cmax, 0, (size_t)N * sizeof(unsigned long long), st);
      if (e != cudaSuccess) return e;
    }
    k_err_ws<true><<<(unsigned)std::min<int64_t>(ntiles, sms), EW_THREADS, smem_ws, st>>>(g, tpack, ntiles, (int)ncb);
    if (cmax_done && cmax) *cmax_done = 1;
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((m + GT - 1) / GT), (unsigned)((N + GT - 1) / GT), 1);
  return dgemm_launch<GM_NN_STORE>(g, grid, st, 8);
}

__global__ void k_eye(double* I, int k) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < (int64_t)k * k) I[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
}
cudaError_t launch_eye(double* I, int k, cudaStream_t st) {
  const int64_t tot = (int64_t)k * k;
  k_eye<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(I, k);
  return cudaGetLastError();
}

__global__ void k_diag_ratio(const double* __restrict__ R, int k, double* __restrict__ out) {
  __shared__ double mx[32], mn[32];
  double a = 0.0, b = INFINITY;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double d = fabs(R[i + (int64_t)i * k]);
    a = fmax(a, d);
    b = fmin(b, d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmin(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) { mx[threadIdx.x >> 5] = a; mn[threadIdx.x >> 5] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { a = fmax(a, mx[w]); b = fmin(b, mn[w]); }
    a = fmax(a, mx[0]);
    b = fmin(b, mn[0]);
    *out = b > 0.0 ? a / b : INFINITY;
  }
}
cudaError_t launch_diag_ratio(const double* R, int k, double* out, cudaStream_t st) {
  k_diag_ratio<<<1, 256, 0, st>>>(R, k, out);
  return cudaGetLastError();
}

cudaError_t launch_sum_scalar(const double* part, int nblk, double* out, cudaStream_t st) {
  k_sum_scalar<<<1, 1024, 0, st>>>(part, nblk, out);
  return cudaGetLastError();
}

}  // namespace mpid
