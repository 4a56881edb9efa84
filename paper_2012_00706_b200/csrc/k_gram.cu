// Gram-based pivoting (the paper's future work "matrix sketching",
// P:402): the k pivots and R of the low-precision QRCP from G = A_L^T A_L instead of k
// streaming Householder passes (reading R17, oracle/gram.py).
//
//   k_gram_tc   G's upper block triangle on the 5th-generation tensor cores:
//               tcgen05.mma kind::f16 (fp16 A_L, fp32 accumulation in TMEM), 128 x 128
//               output tiles, split-K.  The interleaved layout of S is already the
//               K-major core-matrix layout the MMA reads: one 8-row group of 8
//               consecutive columns is a contiguous 128 B core matrix (8 columns x 16 B
//               = 8 fp16 rows), so a 2-D tensor-map box {128 columns, 8 row groups}
//               lands in shared memory as the operand tile (LBO = 2048 B along K, SBO =
//               128 B along M/N) with no re-layout.  The fp32 accumulator is drained
//               every KC = 2048 rows into fp64 registers (double-buffered TMEM), so the
//               fp32 accumulation error is that of a 2048-term sum.
//   k_gram_reduce  G = sum of the split-K partials (fixed order), symmetric fill.
//   k_pchol     outer-product pivoted Cholesky of G for k steps, one CTA: pivot = argmax
//               of the residual diagonal d (ties: lowest original index), R(j, :) =
//               (G(p_j, :) - R(:j, j)^T R(:j, :)) / sqrt(d_j), d -= R(j, :)^2 — the
//               QRCP's pivots and R (R_jj > 0) in exact arithmetic.
//
// Roofline: k_gram_tc is tensor-bound, 2 m n^2 / 2 flops (upper triangle incl. the
// diagonal tiles) at kind::f16; A_L is read once per tile column from L2 (concurrent
// CTAs work on the same K range).
#include "mpid_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cfloat>
#include <math.h>

namespace mpid {

namespace {
constexpr int GT = 128;              // output tile: 128 x 128 (MMA M = N = 128)
constexpr int GSG = 8;               // row groups per pipeline stage (64 rows)
constexpr int GNST = 6;              // pipeline depth
constexpr int GCH = 32;              // stages per TMEM drain (KC = 2048 rows)
constexpr int G_EPI = 16;            // epilogue warps
constexpr int G_BLOCK = 32 * (2 + G_EPI);
constexpr int G_OPB = GSG * GT * 16; // bytes of one operand stage (16 KB)
constexpr int G_SMEM = GNST * 2 * G_OPB + 1024;

__device__ __forceinline__ uint64_t gdesc(uint32_t saddr) {
  // K-major, no swizzle: LBO = 2048 B (next 8 rows of K = next row group), SBO = 128 B
  // (next 8 columns), sm_100 descriptor version bit 46
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((2048 >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::f16: fp16 A and B (formats 0), fp32 accumulator (bit 4), K-major both, N = M = 128
__device__ __forceinline__ uint32_t idesc_f16() {
  return (1u << 4) | ((uint32_t)(GT >> 3) << 17) | ((uint32_t)(GT >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc_f16()), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_g(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32_g(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_g(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

struct GramWork {   // split-K work items: item i -> split s = i / ntiles, tile t = i % ntiles
  int nbk, ntiles, splits;
  int64_t gper;     // row groups per split (multiple of GSG * GCH)
  int sym;          // 1: G = S^T S, upper block triangle; 0: Y = Omega S, nbm x nbk tiles
  int nbm;          // tile rows of the A operand (sym: = nbk)
};
__host__ __device__ inline void tile_of(int t, int nbk, int& bi, int& bj) {
  // upper block triangle, row by row: (0,0) (0,1) .. (0,nbk-1) (1,1) ..
  int b = 0, rem = t;
  while (rem >= nbk - b) { rem -= nbk - b; ++b; }
  bi = b;
  bj = b + rem;
}
}  // namespace

GramWork gram_work(int64_t ngroups, int n, int num_sms, int lw = 0, int64_t cap_items = 0) {
  GramWork w;
  w.nbk = (n + GT - 1) / GT;
  w.sym = lw == 0;
  w.nbm = w.sym ? w.nbk : (lw + GT - 1) / GT;
  w.ntiles = w.sym ? w.nbk * (w.nbk + 1) / 2 : w.nbm * w.nbk;
  const int64_t unit = (int64_t)GSG * GCH;                       // 256 groups = 2048 rows
  const int64_t units = (ngroups + unit - 1) / unit;
  int64_t s = std::max<int64_t>(1, (2 * num_sms + w.ntiles - 1) / w.ntiles);
  s = std::min<int64_t>(s, std::max<int64_t>(1, 512 / w.ntiles));
  s = std::min<int64_t>(s, units);
  if (cap_items > 0) s = std::max<int64_t>(1, std::min<int64_t>(s, cap_items / w.ntiles));
  w.gper = (units + s - 1) / s * unit;
  w.splits = (int)((ngroups + w.gper - 1) / w.gper);
  return w;
}

size_t gram_part_doubles(int64_t ngroups, int n, int num_sms) {
  const GramWork w = gram_work(ngroups, n, num_sms);
  return (size_t)w.ntiles * w.splits * GT * GT;
}

// tmA: the A operand (M = rows of the result): S itself for the Gram, Omega^T for the
// sketch (the same interleaved layout, lw columns); tmS: the B operand, S
__global__ void __launch_bounds__(G_BLOCK, 1) k_gram_tc(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmS, int64_t ngroups,
                                                       GramWork w, double* __restrict__ part,
                                                       const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + GNST * 2 * G_OPB);
  uint64_t* empty = full + GNST;
  uint64_t* tfull = empty + GNST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = w.ntiles * w.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < GNST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], G_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(2 * GT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  auto range = [&](int item, int& bi, int& bj, int64_t& g0, int& nstages) {
    const int s = item / w.ntiles, t = item - s * w.ntiles;
    if (w.sym) tile_of(t, w.nbk, bi, bj);
    else { bi = t / w.nbk; bj = t - bi * w.nbk; }
    g0 = (int64_t)s * w.gper;
    const int64_t g1 = (g0 + w.gper < ngroups) ? g0 + w.gper : ngroups;
    nstages = (int)((g1 - g0 + GSG - 1) / GSG);
  };

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      int slot = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        int bi, bj, nstages;
        int64_t g0;
        range(item, bi, bj, g0, nstages);
        const bool diag = w.sym && bi == bj;
        for (int st = 0; st < nstages; ++st) {
          mbar_wait(&empty[slot], phase ^ 1);
          unsigned char* a = smem + (size_t)slot * 2 * G_OPB;
          mbar_expect_tx(&full[slot], diag ? G_OPB : 2 * G_OPB);
          const int gg = (int)(g0 + (int64_t)st * GSG);
          tma_load_2d_g(a, &tmA, bi * GT * 2, gg, &full[slot]);
          if (!diag) tma_load_2d_g(a + G_OPB, &tmS, bj * GT * 2, gg, &full[slot]);
          if (++slot == GNST) { slot = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (one thread) =======================
    if (lane == 0) {
      int slot = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        int bi, bj, nstages;
        int64_t g0;
        range(item, bi, bj, g0, nstages);
        const bool diag = w.sym && bi == bj;
        for (int st = 0; st < nstages; ++st) {
          if (st % GCH == 0) {
            mbar_wait(&tempty[acc], aphase ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          mbar_wait(&full[slot], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a = su32(smem + (size_t)slot * 2 * G_OPB);
          const uint32_t b = diag ? a : a + G_OPB;
          const uint32_t d = tmem + (uint32_t)(acc * GT);
#pragma unroll
          for (int q = 0; q < GSG / 2; ++q)   // K = 16 rows = 2 row groups per MMA
            mma_f16(d, gdesc(a + q * 2 * 2048), gdesc(b + q * 2 * 2048), (st % GCH == 0 && q == 0) ? 0u : 1u);
          mma_commit_g(&empty[slot]);          // the stage is free once these MMAs have read it
          if (st % GCH == GCH - 1 || st == nstages - 1) {
            mma_commit_g(&tfull[acc]);
            if (++acc == 2) { acc = 0; aphase ^= 1; }
          }
          if (++slot == GNST) { slot = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ======================= epilogue (16 warps) =======================
    // warp: TMEM lane quarter (warp % 4) = G rows 32 q .. 32 q + 31 of the tile, column
    // block cb = (warp - 2) / 4 = G columns 32 cb .. 32 cb + 31
    const int quarter = warp & 3, cb = (warp - 2) >> 2;
    int acc = 0;
    uint32_t aphase = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      int bi, bj, nstages;
      int64_t g0;
      range(item, bi, bj, g0, nstages);
      double a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = 0.0;
      const int nch = (nstages + GCH - 1) / GCH;
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&tfull[acc], aphase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t r[32];
        tmem_ld32_g(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * GT + cb * 32), r);
#pragma unroll
        for (int i = 0; i < 32; ++i) a[i] += (double)__uint_as_float(r[i]);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
      const int s = item / w.ntiles, t = item - s * w.ntiles;
      double* out = part + ((int64_t)t * w.splits + s) * GT * GT + (int64_t)(quarter * 32 + lane) * GT + cb * 32;
#pragma unroll
      for (int i = 0; i < 32; i += 2) *reinterpret_cast<double2*>(out + i) = make_double2(a[i], a[i + 1]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * GT));
}

// G (n x n col-major, symmetric) = sum over splits of the tile partials, fixed order
__global__ void k_gram_reduce(const double* __restrict__ part, GramWork w, int n, double* __restrict__ G,
                              const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * n) return;
  int c1 = (int)(idx % n), c2 = (int)(idx / n);
  int b1 = c1 / GT, b2 = c2 / GT;
  int r = c1 - b1 * GT, c = c2 - b2 * GT;
  if (b1 > b2) { const int tb = b1; b1 = b2; b2 = tb; const int tr = r; r = c; c = tr; }
  const int t = b1 * w.nbk - b1 * (b1 - 1) / 2 + (b2 - b1);
  double s = 0.0;
  for (int sp = 0; sp < w.splits; ++sp) s += part[((int64_t)t * w.splits + sp) * GT * GT + (int64_t)r * GT + c];
  G[idx] = s;
}

// ---------------------------------------------------------------------------
// pivoted Cholesky, one CTA of 1024 threads for all k steps
struct AM {
  double v;
  int orig, pos;
};
__device__ __forceinline__ bool am_gt(const AM& a, const AM& b) {
  return a.v > b.v || (a.v == b.v && a.orig < b.orig);
}
__device__ AM block_argmax_g(AM a, AM* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    AM b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.orig = __shfl_xor_sync(0xffffffffu, a.orig, o);
    b.pos = __shfl_xor_sync(0xffffffffu, a.pos, o);
    if (am_gt(b, a)) a = b;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = a;
  __syncthreads();
  if (warp == 0) {
    a = lane < (int)(blockDim.x >> 5) ? sh[lane] : AM{-INFINITY, 0x7fffffff, -1};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      AM b;
      b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
      b.orig = __shfl_xor_sync(0xffffffffu, a.orig, o);
      b.pos = __shfl_xor_sync(0xffffffffu, a.pos, o);
      if (am_gt(b, a)) a = b;
    }
    if (lane == 0) sh[0] = a;
  }
  __syncthreads();
  const AM r = sh[0];
  __syncthreads();
  return r;
}
__device__ double block_sum_g(double v, double* sh) {
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

// Blocked (left-looking within a panel, right-looking across panels) pivoted Cholesky:
// Gc = the Schur complement of G after the previous panels (original column indexing);
// step j of the panel [j0, j1): pivot = argmax of d over positions >= j (ties: lowest
// original index), swap positions, R(j, i) = (Gc(p_j, p_i) - sum_{l=j0}^{j-1} R(l, j) R(l, i))
// / sqrt(d_j), d_i -= R(j, i)^2.  k_schur then subtracts the panel's rows from Gc's
// trailing block.  One CTA per panel (the per-step work is O(b n)); state in global memory.
__global__ void __launch_bounds__(1024) k_pchol_panel(const double* __restrict__ Gc, int n, int j0, int j1,
                                                      int k_max, double* __restrict__ d, int* __restrict__ perm,
                                                      double* __restrict__ R64, float* __restrict__ R,
                                                      DevScalars* __restrict__ sc) {
  if (sc->done) return;
  __shared__ AM sha[32];
  __shared__ double shs[32];
  if (j0 == 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      perm[i] = i;
      d[i] = Gc[(int64_t)i * n + i];                   // residual norms^2 start at diag(G)
    }
    __syncthreads();
  }
  int k_out = -1, status = 0;
  for (int j = j0; j < j1; ++j) {
    if (j > 0 && sc->eps2normAL2 > 0.0) {            // tolerance stop (reading R8 on d)
      double t = 0.0;
      for (int i = j + threadIdx.x; i < n; i += blockDim.x) t += d[i];
      t = block_sum_g(t, shs);
      if (t <= sc->eps2normAL2) { k_out = j; break; }
    }
    AM best{-INFINITY, 0x7fffffff, -1};
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
      const AM c{d[i], perm[i], i};
      if (am_gt(c, best)) best = c;
    }
    best = block_argmax_g(best, sha);
    const int p = best.pos;
    if (p != j) {                                      // swap positions j <-> p
      for (int l = threadIdx.x; l < j; l += blockDim.x) {
        const double x = R64[(int64_t)l * n + j];
        R64[(int64_t)l * n + j] = R64[(int64_t)l * n + p];
        R64[(int64_t)l * n + p] = x;
        const float y = R[(int64_t)l * n + j];
        R[(int64_t)l * n + j] = R[(int64_t)l * n + p];
        R[(int64_t)l * n + p] = y;
      }
      if (threadIdx.x == 0) {
        const int q = perm[j];
        perm[j] = perm[p];
        perm[p] = q;
        const double x = d[j];
        d[j] = d[p];
        d[p] = x;
      }
    }
    __syncthreads();
    const double dj = d[j];
    if (!(dj > 0.0)) { k_out = j; status = 4; break; }   // the Gram's resolution is exhausted
    const double rjj = sqrt(dj);
    const double* gcol = Gc + (int64_t)perm[j] * n;       // Gc(:, p_j) = Gc(p_j, :)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double r;
      if (i < j) r = 0.0;
      else if (i == j) r = rjj;
      else {
        double s = gcol[perm[i]];
        for (int l = j0; l < j; ++l) s = fma(-R64[(int64_t)l * n + j], R64[(int64_t)l * n + i], s);
        r = s / rjj;
        d[i] -= r * r;
      }
      R64[(int64_t)j * n + i] = r;
      R[(int64_t)j * n + i] = __double2float_rn(r);
    }
    __syncthreads();
    if (threadIdx.x == 0) d[j] = 0.0;
    __syncthreads();
  }
  if (k_out < 0 && j1 < k_max) return;                  // panel done, more to come
  if (k_out < 0) k_out = k_max;
  double rest = 0.0;
  for (int i = k_out + threadIdx.x; i < n; i += blockDim.x) rest += fmax(d[i], 0.0);
  rest = block_sum_g(rest, shs);
  if (threadIdx.x == 0) {
    sc->k_out = k_out;
    sc->status = status;
    sc->resid2 = rest;
    sc->done = 1;
  }
}

// Gc(p_a, p_b) -= sum_{l=j0}^{j1-1} R(l, a) R(l, b) for trailing positions a, b >= j1;
// 32 x 32 position tiles, the panel rows staged in shared memory
__global__ void __launch_bounds__(1024) k_schur(double* __restrict__ Gc, int n, int j0, int j1,
                                                const int* __restrict__ perm, const double* __restrict__ R64,
                                                const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  __shared__ double ra[32][33], rb[32][33];
  const int a0 = j1 + blockIdx.x * 32, b0 = j1 + blockIdx.y * 32;
  if (a0 >= n || b0 >= n) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int nl = j1 - j0;
  // ty = panel row l, tx = position offset
  ra[ty][tx] = (ty < nl && a0 + tx < n) ? R64[(int64_t)(j0 + ty) * n + a0 + tx] : 0.0;
  rb[ty][tx] = (ty < nl && b0 + tx < n) ? R64[(int64_t)(j0 + ty) * n + b0 + tx] : 0.0;
  __syncthreads();
  const int a = a0 + ty, b = b0 + tx;
  if (a >= n || b >= n) return;
  double s = 0.0;
  for (int l = 0; l < nl; ++l) s = fma(ra[l][ty], rb[l][tx], s);
  double* g = Gc + (int64_t)perm[b] * n + perm[a];
  *g -= s;
}

// ---------------------------------------------------------------------------
// Sketched pivoting (NEXT-4, second option; R18, oracle/sketch.py):
//   k_omega         Omega^T (m_pad x lw, +-1 fp16) in the interleaved layout of S, from the
//                   counter-based generator synth.counter_sign implements (SplitMix64 of
//                   base + ((global row << 13) | column), top bit -> -1); columns >= l and
//                   padding rows are 0
//   k_gram_tc       (sym = 0) Y = Omega A_L on tcgen05, split-K partials
//   k_sketch_reduce Y (lw x n, col-major fp64) = sum of the partials, fixed order
//   k_sq_*          fp64 Householder QRCP of Y, exact norms every step (3 kernels per step)
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_omega(__half* __restrict__ Om, int64_t ngroups, int lw, int l, int64_t m_local,
                        int64_t row_offset, uint64_t base, const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (group, column)
  if (idx >= ngroups * lw) return;
  const int64_t g = idx / lw;
  const int c = (int)(idx - g * lw);
  uint4 out;
  __half* h = reinterpret_cast<__half*>(&out);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t r = g * 8 + q;
    float v = 0.f;
    if (c < l && r < m_local) {
      const uint64_t ctr = ((uint64_t)(row_offset + r) << 13) | (uint64_t)c;
      v = (splitmix64_d(base + ctr) >> 63) ? -1.f : 1.f;
    }
    h[q] = __float2half_rn(v);
  }
  reinterpret_cast<uint4*>(Om)[idx] = out;
}

__global__ void k_sketch_reduce(const double* __restrict__ part, GramWork w, int lw, int n, double* __restrict__ Y,
                                const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)lw * n) return;
  const int i = (int)(idx % lw), c = (int)(idx / lw);
  const int bi = i / GT, bj = c / GT;
  const int t = bi * w.nbk + bj;
  double s = 0.0;
  for (int sp = 0; sp < w.splits; ++sp)
    s += part[((int64_t)t * w.splits + sp) * GT * GT + (int64_t)(i - bi * GT) * GT + (c - bj * GT)];
  Y[idx] = s;
}

// fp64 Householder QRCP of Y (ly x n, col-major), exact trailing norms every step, as
// three kernels per step (graph-captured): the column work spreads over the GPU, the
// step's scalar work runs on one CTA.  Scratch: snorm[n], v[ly], scal[4] = (beta, tot0).
//   k_sq_norms0  snorm_c = ||Y(:, c)||^2, scal[1] = ||Y||_F^2          (warp per column)
//   k_sq_pivot   tolerance test, argmax (ties: lowest original index), swap, beta, v
//   k_sq_update  w_c = Y(j:, c)^T u, R(j, c), Y(j:, c) -= v f_c, snorm_c over rows > j
__global__ void __launch_bounds__(1024) k_sq_norms0(const double* __restrict__ Y, int ly, int n,
                                                    double* __restrict__ snorm, int* __restrict__ perm,
                                                    const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + warp;
  if (c >= n) return;
  double t = 0.0;
  for (int r = lane; r < ly; r += 32) t = fma(Y[(int64_t)c * ly + r], Y[(int64_t)c * ly + r], t);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) {
    snorm[c] = t;
    perm[c] = c;
  }
}

__global__ void __launch_bounds__(1024) k_sq_pivot(double* __restrict__ Y, int ly, int n, int j, int k_max,
                                                   double* __restrict__ snorm, double* __restrict__ v,
                                                   double* __restrict__ scal, int* __restrict__ perm,
                                                   double* __restrict__ R64, float* __restrict__ R,
                                                   DevScalars* __restrict__ sc) {
  if (sc->done) return;
  __shared__ AM sha[32];
  __shared__ double shs[32];
  if (j == 0) {                                       // ||Y||_F^2 for the tolerance test
    double t = 0.0;
    for (int c = threadIdx.x; c < n; c += blockDim.x) t += snorm[c];
    t = block_sum_g(t, shs);
    if (threadIdx.x == 0) scal[1] = t;
  }
  if (j > 0 && sc->eps2normAL2 > 0.0) {               // reading R8 on the sketch's mass
    double t = 0.0;
    for (int c = j + threadIdx.x; c < n; c += blockDim.x) t += snorm[c];
    t = block_sum_g(t, shs);
    if (t <= sc->eps2normAL2 / sc->normAL2 * scal[1]) {
      if (threadIdx.x == 0) { sc->k_out = j; sc->status = 0; sc->resid2 = 0.0; sc->done = 1; }
      return;
    }
  }
  AM best{-INFINITY, 0x7fffffff, -1};
  for (int c = j + threadIdx.x; c < n; c += blockDim.x) {
    const AM a{snorm[c], perm[c], c};
    if (am_gt(a, best)) best = a;
  }
  best = block_argmax_g(best, sha);
  const int p = best.pos;
  if (p != j) {
    for (int r = threadIdx.x; r < ly; r += blockDim.x) {
      const double x = Y[(int64_t)j * ly + r];
      Y[(int64_t)j * ly + r] = Y[(int64_t)p * ly + r];
      Y[(int64_t)p * ly + r] = x;
    }
    for (int l = threadIdx.x; l < j; l += blockDim.x) {
      const double x = R64[(int64_t)l * n + j];
      R64[(int64_t)l * n + j] = R64[(int64_t)l * n + p];
      R64[(int64_t)l * n + p] = x;
      const float y = R[(int64_t)l * n + j];
      R[(int64_t)l * n + j] = R[(int64_t)l * n + p];
      R[(int64_t)l * n + p] = y;
    }
    if (threadIdx.x == 0) {
      const int q = perm[j];
      perm[j] = perm[p];
      perm[p] = q;
      const double x = snorm[j];
      snorm[j] = snorm[p];
      snorm[p] = x;
    }
  }
  __syncthreads();
  const double sj = snorm[j];
  if (!(sj >= DBL_MIN)) {
    if (threadIdx.x == 0) { sc->k_out = j; sc->status = 4; sc->resid2 = 0.0; sc->done = 1; }
    return;
  }
  const double u0 = Y[(int64_t)j * ly + j];
  const double beta = -copysign(sqrt(sj), u0);
  const double cc = 1.0 / (u0 - beta);
  for (int r = threadIdx.x; r < ly; r += blockDim.x)
    v[r] = r < j ? 0.0 : (r == j ? 1.0 : __dmul_rn(Y[(int64_t)j * ly + r], cc));
  for (int i = threadIdx.x; i < j; i += blockDim.x) {
    R64[(int64_t)j * n + i] = 0.0;
    R[(int64_t)j * n + i] = 0.f;
  }
  if (threadIdx.x == 0) {
    scal[0] = beta;
    sc->k_out = j + 1;
    if (j + 1 >= k_max) { sc->status = 0; sc->resid2 = 0.0; }
  }
}

// warp per column c >= j: w_c = Y(j:, c)^T u with u = Y(j:, j), R(j, c) = w_c / beta (sign-
// normalised), f_c = Y(j, c) - w_c / beta, Y(j:, c) -= v f_c and the new norm over rows > j.
// Column j is only read here (every warp's u); k_sq_colj updates it afterwards.
__global__ void __launch_bounds__(1024) k_sq_update(double* __restrict__ Y, int ly, int n, int j, int k_max,
                                                    double* __restrict__ snorm, const double* __restrict__ v,
                                                    const double* __restrict__ scal, double* __restrict__ R64,
                                                    float* __restrict__ R, DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = j + blockIdx.x * 32 + warp;
  if (c < n) {
    const double beta = scal[0];
    const double sgn = beta < 0.0 ? -1.0 : 1.0;
    double t = 0.0;
    for (int r = j + lane; r < ly; r += 32) t = fma(Y[(int64_t)c * ly + r], Y[(int64_t)j * ly + r], t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    const double rraw = t / beta;
    const double f = Y[(int64_t)c * ly + j] - rraw;
    if (lane == 0) {
      R64[(int64_t)j * n + c] = rraw * sgn;
      R[(int64_t)j * n + c] = __double2float_rn(rraw * sgn);
    }
    if (c != j) {
      double s2 = 0.0;
      for (int r = j + lane; r < ly; r += 32) {
        const double y = __dadd_rn(__dmul_rn(-v[r], f), Y[(int64_t)c * ly + r]);
        Y[(int64_t)c * ly + r] = y;
        if (r > j) s2 = fma(y, y, s2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      if (lane == 0) snorm[c] = s2;
    }
  }
  (void)k_max;
}

// column j's own update, after every column's dot product with u = Y(j:, j)
__global__ void k_sq_colj(double* __restrict__ Y, int ly, int n, int j, const double* __restrict__ v,
                          const double* __restrict__ scal, const double* __restrict__ R64,
                          const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const double beta = scal[0];
  const double sgn = beta < 0.0 ? -1.0 : 1.0;
  const double f = Y[(int64_t)j * ly + j] - R64[(int64_t)j * n + j] * sgn;
  __syncthreads();
  for (int r = j + threadIdx.x; r < ly; r += blockDim.x)
    Y[(int64_t)j * ly + r] = __dadd_rn(__dmul_rn(-v[r], f), Y[(int64_t)j * ly + r]);
}

__global__ void k_sq_finish(int k_max, DevScalars* __restrict__ sc) {
  if (sc->done) return;
  sc->k_out = k_max;
  sc->status = 0;
  sc->resid2 = 0.0;
  sc->done = 1;
}

// ---------------------------------------------------------------------------
int encode_tmap_gram(void* tmap_out, void* S, int64_t ngroups, int n) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return -1;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  // fp16 S as [ngroups][n * 2] 8-byte units; box = 128 columns (256 units) x 8 row groups
  const cuuint64_t dims[2] = {(cuuint64_t)n * 2, (cuuint64_t)ngroups};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 16};
  const cuuint32_t box[2] = {(cuuint32_t)(GT * 2), (cuuint32_t)GSG};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, S, dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return (int)r;
}

cudaError_t launch_gram(const void* tmap, int64_t ngroups, int n, int num_sms, double* part, double* G,
                        const DevScalars* sc, cudaStream_t st) {
  const CUtensorMap* tm = reinterpret_cast<const CUtensorMap*>(tmap);
  const GramWork w = gram_work(ngroups, n, num_sms);
  cudaError_t e = smem_attr((const void*)k_gram_tc, G_SMEM + 64);
  if (e != cudaSuccess) return e;
  const int items = w.ntiles * w.splits;
  const int grid = std::min(items, num_sms);
  k_gram_tc<<<grid, G_BLOCK, G_SMEM + 64, st>>>(*tm, *tm, ngroups, w, part, sc);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t tot = (int64_t)n * n;
  k_gram_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(part, w, n, G, sc);
  return cudaGetLastError();
}

cudaError_t launch_sketch(const void* tmapO, const void* tmapS, void* Om, int64_t ngroups, int n, int l, int lw,
                          int64_t m_local, int64_t row_offset, uint64_t base, int num_sms, double* part,
                          size_t part_doubles, double* Y, const DevScalars* sc, cudaStream_t st) {
  const int64_t tot = ngroups * lw;
  k_omega<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>((__half*)Om, ngroups, lw, l, m_local, row_offset, base, sc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const GramWork w = gram_work(ngroups, n, num_sms, lw, (int64_t)(part_doubles / (GT * GT)));
  if ((size_t)w.ntiles * w.splits * GT * GT > part_doubles) return cudaErrorInvalidValue;
  if ((e = smem_attr((const void*)k_gram_tc, G_SMEM + 64)) != cudaSuccess) return e;
  const int items = w.ntiles * w.splits;
  k_gram_tc<<<std::min(items, num_sms), G_BLOCK, G_SMEM + 64, st>>>(
      *reinterpret_cast<const CUtensorMap*>(tmapO), *reinterpret_cast<const CUtensorMap*>(tmapS), ngroups, w, part, sc);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t ty = (int64_t)lw * n;
  k_sketch_reduce<<<(unsigned)((ty + 255) / 256), 256, 0, st>>>(part, w, lw, n, Y, sc);
  return cudaGetLastError();
}

cudaError_t launch_small_qrcp(double* Y, int ly, int n, int k_max, double* scratch, int* perm, double* R64, float* R,
                              DevScalars* sc, cudaStream_t st) {
  double* snorm = scratch;                 // n
  double* v = scratch + n;                 // ly <= n
  double* scal = scratch + 2 * (size_t)n;  // 4
  if (ly > n) return cudaErrorInvalidValue;
  const unsigned cb = (unsigned)((n + 31) / 32);
  k_sq_norms0<<<cb, 1024, 0, st>>>(Y, ly, n, snorm, perm, sc);
  cudaError_t e = cudaGetLastError();
  for (int j = 0; j < k_max && e == cudaSuccess; ++j) {
    k_sq_pivot<<<1, 1024, 0, st>>>(Y, ly, n, j, k_max, snorm, v, scal, perm, R64, R, sc);
    k_sq_update<<<(unsigned)((n - j + 31) / 32), 1024, 0, st>>>(Y, ly, n, j, k_max, snorm, v, scal, R64, R, sc);
    k_sq_colj<<<1, 256, 0, st>>>(Y, ly, n, j, v, scal, R64, sc);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  k_sq_finish<<<1, 1, 0, st>>>(k_max, sc);
  return cudaGetLastError();
}

cudaError_t launch_pchol(const double* G, double* Gc, int n, int k_max, double* d, int* perm, double* R64, float* R,
                         DevScalars* sc, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(Gc, G, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  constexpr int PB = 32;                                  // panel width (<= 32: one smem row per warp)
  for (int j0 = 0; j0 < k_max; j0 += PB) {
    const int j1 = std::min(k_max, j0 + PB);
    k_pchol_panel<<<1, 1024, 0, st>>>(Gc, n, j0, j1, k_max, d, perm, R64, R, sc);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (j1 < k_max && j1 < n) {
      const unsigned t = (unsigned)((n - j1 + 31) / 32);
      k_schur<<<dim3(t, t), 1024, 0, st>>>(Gc, n, j0, j1, perm, R64, sc);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace mpid
