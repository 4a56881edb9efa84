// The two large fp64 GEMMs of the ID step (Algorithm 2 lines 5-7; P:178 the
// least-squares coefficients; Remark 2 P:199-201 the error) on the INTEGER tensor cores:
// tcgen05.mma kind::i8 (signed 8-bit operands, exact int32 accumulation in TMEM) by the
// Ozaki scheme.  The paper's method is unchanged — P = argmin ||A_I X - A_J|| and the
// error ||A_J - A_I T||_F in double precision — only the way the fp64 products are
// evaluated differs from a DMMA / DFMA loop ("fp64 on the integer pipe").
//
// Slicing.  An operand row (or column) of fp64 values sharing one exponent E (the smallest
// with max |x| < 2^E over the row's K values) is written as
//     x = sgn(x) * sum_{p=0}^{7} s_p 2^{-7(p+1)} 2^E + e,   s_p in [0, 127],  |e| < 2^{E-56}
// (X = trunc(|x| 2^{56-E}) < 2^56 split into eight 7-bit digits; the signed int8 slice is
// sgn(x) s_p).  A product of two such sums is  sum_{p,q} s_p t_q 2^{-7(p+q+2)} 2^{Ea+Eb};
// the 36 digit pairs with p + q <= 7 are kept (one int8 MMA each), grouped by the diagonal
// d = p + q into 8 int32 accumulators (products on one diagonal share the weight), and
//     x y ~ 2^{Ea+Eb-14} sum_{d=0}^{7} acc_d 2^{-7d}        (fp64 Horner in the epilogue).
// Error per product (relative to 2^{Ea+Eb} <= 4 max|x| max|y|): dropped pairs (p + q >= 8)
// < 7 * 2^{-56} plus slicing 2 * 2^{-56}, i.e. < 1.3e-16 — the same order as one fp64
// rounding; the int32 sums are exact (|acc_d| <= 8 * 127^2 * K < 2^31 for K <= 16384).
//
//   k_oz_slice_cols  Q1 (m x k) -> the TN A operand, K-major per 32-row K-step (exponent per column)
//   k_oz_slice_rows  A_I (m x k) -> the error kernel's A operand per 128-row tile (exponent per row)
//   k_oz_slice_t     T (k x nj) -> the error kernel's B operand per 32-column tile (exponent per column)
//   k_oz_tn          [G2 | W] = Q1^T [Q1 | A_D(:, J)], split over row groups (one CTA per
//                    (row group, 64-column tile)); B sliced in-kernel from fp64
//   k_oz_tn_reduce   the row-group partials summed in a fixed order -> G2 (k x k), W (k x nj)
//   k_oz_err         sum_{r, c} (A_D(r, J_c) - (A_I T)(r, c))^2, persistent over 128-row
//                    tiles, per tile all 32-column J tiles; A_I T is never stored
//
// Bound: the int8 tensor pipe (36 MMAs per K-step) and, for the error, the TMEM read port
// (8 int32 accumulators per output element).  k <= 128 (the K of the error GEMM and the
// M of the TN GEMM fit one 128-row operand).
#include "mpid_internal.cuh"
#include <math.h>
#include <cstdlib>

namespace mpid {

namespace {
constexpr int OZ_S = 8;                               // slices per operand
constexpr int KSTEP = 32;                             // K per kind::i8 MMA (bytes)
// TN kernel (W, G2)
constexpr int TN_N = 64;                              // output columns per CTA
constexpr int TN_NST = 4;                             // pipeline stages (one K-step each)
constexpr int TN_A = OZ_S * 128 * KSTEP;              // 32 KB: 8 slices of 128 (M) x 32 (K)
constexpr int TN_B = OZ_S * TN_N * KSTEP;             // 16 KB: 8 slices of 64 (N) x 32 (K)
constexpr int TN_CHS = 512;                           // K-steps per int32 chunk (16384 rows)
constexpr int TN_SLW = 16;                            // slicer / drain warps
constexpr int TN_NI = 1;                              // MMA-issuing warp (12 MMAs per K-step)
constexpr int TN_THREADS = 32 * (1 + TN_NI + TN_SLW);
constexpr int TN_SMEM = TN_NST * (TN_A + TN_B) + 1024 + 1024;
// error kernel
constexpr int ER_N = 32;                              // J columns per tile (MMA N)
constexpr int ER_EPW = 8;                             // epilogue warps (16: more spills, slower)
constexpr int ER_NI = 1;                              // MMA-issuing warp (8 MMAs per K-step)
constexpr int ER_THREADS = 32 * (1 + ER_NI + ER_EPW);

__device__ __forceinline__ uint64_t oz_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // K-major, no swizzle (core matrix 8 rows x 16 B): LBO = stride between core matrices
  // along K, SBO = along M/N; sm_100 descriptor version bit 46
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::i8: D s32 (bits 4-5 = 2), A and B signed 8-bit (bits 7-9, 10-12 = 1), K-major, M = 128
__host__ __device__ constexpr uint32_t oz_idesc(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void oz_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define OZ_LD16(taddr, r)                                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),  \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),        \
                 "=r"(r[15])                                                                                   \
               : "r"(taddr))
#define OZ_LD8(taddr, r)                                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                           \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])   \
               : "r"(taddr))
#define OZ_LD4(taddr, r)                                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"                                     \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])                                                  \
               : "r"(taddr))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// exact int32 -> fp64 on the fp64 pipe: 1.5 * 2^52 + 2^31 + a, minus 1.5 * 2^52 + 2^31
__device__ __forceinline__ double i2d(uint32_t a) {
  return __hiloint2double(0x43380000, (int)(a ^ 0x80000000u)) - 6755401588539392.0;
}

// the 8 diagonal accumulators (|acc_d| < 2^24 for K <= 128) combined exactly in two int64
// Horner halves H = sum_{d<4} acc_d 2^{7(3-d)}, L = sum_{d>=4} acc_d 2^{7(7-d)} (|H|, |L| < 2^46),
// each converted exactly with the 1.5 2^52 bit-pattern add: sum_d acc_d 2^{-7d} =
// (H + L 2^{-28}) 2^{-21} — 2 fp64 adds and 1 fma instead of 8 conversions and 7 fmas
__device__ __forceinline__ double oz_combine8(const uint32_t* a) {
  const long long H = ((((long long)(int)a[0] * 128 + (int)a[1]) * 128 + (int)a[2]) * 128) + (int)a[3];
  const long long L = ((((long long)(int)a[4] * 128 + (int)a[5]) * 128 + (int)a[6]) * 128) + (int)a[7];
  const double hd = __longlong_as_double(0x4338000000000000LL + H) - 6755399441055744.0;
  const double ld = __longlong_as_double(0x4338000000000000LL + L) - 6755399441055744.0;
  return fma(ld, 3.7252902984619140625e-09, hd);   // 2^-28
}
// the smallest E with mx < 2^E (mx > 0; 0 for mx == 0)
__device__ __forceinline__ int oz_exp(double mx) {
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);
  return e;
}
__device__ __forceinline__ double pow2(int e) {   // 2^e for -1022 <= e <= 1023
  return __hiloint2double((e + 1023) << 20, 0);
}
// byte-wise two's complement negation of 4 digits in [0, 127]
__device__ __forceinline__ uint32_t neg4(uint32_t b) { return (0x80808080u - b) ^ 0x80808080u; }
// digits of x at scale sc = 2^{56-E} (or 0): w0 = slices 0..3 (byte p = slice p), w1 = slices 4..7.
// X = floor(|x| sc) < 2^56 is taken from the bit pattern with integer shifts — the fp64 pipe
// (a DMUL and a 64-bit F2I per value) was the slicer warps' top stall in ncu's warp-state
// sampling of k_oz_tn: |x| = M 2^(e-1075) with M the 53-bit significand, sc = 2^(es-1023), so
// X = M >> (2098 - es - e) (a left shift of at most 3 when |x| is within 2^-3 of 2^E).
__device__ __forceinline__ void oz_digits(double x, double sc, uint32_t& w0, uint32_t& w1) {
  const uint32_t xh = (uint32_t)__double2hiint(x), xl = (uint32_t)__double2loint(x);
  const uint32_t e = (xh >> 20) & 0x7FFu;
  const int es = (int)(((uint32_t)__double2hiint(sc) >> 20) & 0x7FFu);   // loop-invariant
  const unsigned long long M = ((unsigned long long)((xh & 0xFFFFFu) | (e ? 0x100000u : 0u)) << 32) | xl;
  const int sh = 2098 - es - (int)(e ? e : 1u);                          // subnormals: exponent 1, no hidden bit
  const unsigned long long X = sh >= 64 ? 0ull : (sh >= 0 ? M >> sh : M << (-sh));
  const uint32_t hi = (uint32_t)(X >> 28), lo = (uint32_t)X & 0x0FFFFFFFu;
  uint32_t b0 = (hi >> 21) | (((hi >> 14) & 127u) << 8) | (((hi >> 7) & 127u) << 16) | ((hi & 127u) << 24);
  uint32_t b1 = (lo >> 21) | (((lo >> 14) & 127u) << 8) | (((lo >> 7) & 127u) << 16) | ((lo & 127u) << 24);
  if (xh >> 31) {                                  // (-0.0: all digits 0, their negation too)
    b0 = neg4(b0);
    b1 = neg4(b1);
  }
  w0 = b0;
  w1 = b1;
}
// 4 x 4 byte transpose: a[i] holds digits 0..3 of value i -> t[p] holds digit p of values 0..3
__device__ __forceinline__ void tr4(const uint32_t a[4], uint32_t t[4]) {
  const uint32_t x01l = __byte_perm(a[0], a[1], 0x5140), x01h = __byte_perm(a[0], a[1], 0x7362);
  const uint32_t x23l = __byte_perm(a[2], a[3], 0x5140), x23h = __byte_perm(a[2], a[3], 0x7362);
  t[0] = __byte_perm(x01l, x23l, 0x5410);
  t[1] = __byte_perm(x01l, x23l, 0x7632);
  t[2] = __byte_perm(x01h, x23h, 0x5410);
  t[3] = __byte_perm(x01h, x23h, 0x7632);
}
// 4 consecutive K values -> out[p] = the 4 bytes of slice p (p = 0..7)
__device__ __forceinline__ void oz_slice4(const double v[4], double sc, uint32_t out[8]) {
  uint32_t a0[4], a1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) oz_digits(v[i], sc, a0[i], a1[i]);
  tr4(a0, out);
  tr4(a1, out + 4);
}
}  // namespace

// ---------------------------------------------------------------------------
// column max |x| of a col-major m x k matrix: grid (k, splits), bit patterns of non-negative
// doubles order like unsigned integers (cmax zeroed beforehand)
__global__ void __launch_bounds__(256) k_oz_colmax(const double* __restrict__ X, int64_t m, int64_t ld,
                                                   unsigned long long* __restrict__ cmax) {
  const int c = blockIdx.x;
  const int64_t per = (m + gridDim.y - 1) / gridDim.y;
  const int64_t r0 = (int64_t)blockIdx.y * per, r1 = min(m, r0 + per);
  double mx = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) mx = fmax(mx, fabs(__ldcs(X + c * ld + r)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ double sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) mx = fmax(mx, sh[i]);
    atomicMax(cmax + c, (unsigned long long)__double_as_longlong(mx));
  }
}

// Q1 (m x k, ld) -> As: per K-step s (32 rows) 8 slices of the 128 x 32 A operand,
// [s][p][kc 2][l 128][16 B] (element (l, r) of slice p at p*4096 + (r/16)*2048 + l*16 + r%16).
// Thread = (l, row half h, step s); columns l >= k and rows >= m are zero.
__global__ void __launch_bounds__(256) k_oz_slice_cols(const double* __restrict__ X, int64_t m, int64_t ld, int k,
                                                       const unsigned long long* __restrict__ cmax, int64_t nsteps,
                                                       uint4* __restrict__ As) {
  // one block per K-step: the 32 rows x k columns are read column-segment-wise (a warp =
  // one column's 256 B, coalesced) into shared memory, then thread (l, row half h) slices
  // its 16 values and writes 8 x 16 B (consecutive l: contiguous)
  __shared__ double tile[128][KSTEP + 1];
  const int64_t s = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = s * KSTEP + lane;
  for (int l = warp; l < 128; l += 8) tile[l][lane] = (l < k && r < m) ? __ldcs(X + (int64_t)l * ld + r) : 0.0;
  __syncthreads();
  const int l = threadIdx.x & 127, h = threadIdx.x >> 7;
  const double sc = l < k ? pow2(56 - oz_exp(__longlong_as_double((long long)cmax[l]))) : 0.0;
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = tile[l][h * 16 + i];
  uint32_t w[4][8];
#pragma unroll
  for (int g = 0; g < 4; ++g) oz_slice4(v + 4 * g, sc, w[g]);
  uint4* base = As + s * (TN_A / 16) + h * (2048 / 16) + l;
#pragma unroll
  for (int p = 0; p < OZ_S; ++p) base[p * (4096 / 16)] = make_uint4(w[0][p], w[1][p], w[2][p], w[3][p]);
}

// A_I (m x k, ldx) -> per 128-row tile t the error kernel's A operand: 8 slices of
// 128 x KP bytes, [t][p][kc KP/16][r 128][16 B]; rsc[r] = 2^{E_r - 35}.  Thread per row.
__global__ void __launch_bounds__(128) k_oz_slice_rows(const double* __restrict__ X, int64_t m, int64_t ldx, int k,
                                                       int KP, uint4* __restrict__ As, double* __restrict__ rsc) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // grid covers the padded rows
  const bool live = r < m;
  double mx = 0.0;
  if (live)
    for (int l = 0; l < k; ++l) mx = fmax(mx, fabs(X[(int64_t)l * ldx + r]));
  const int E = oz_exp(mx);
  const double sc = pow2(56 - E);
  rsc[r] = live ? pow2(E - 35) : 0.0;   // 2^{E-14} times the 2^{-21} of oz_combine8
  const int64_t t = r >> 7;
  const int rr = (int)(r & 127);
  const int nkc = KP / 16;
  for (int kc = 0; kc < nkc; ++kc) {
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int l = kc * 16 + i;
      v[i] = (live && l < k) ? X[(int64_t)l * ldx + r] : 0.0;
    }
    uint32_t w[4][8];
#pragma unroll
    for (int g = 0; g < 4; ++g) oz_slice4(v + 4 * g, sc, w[g]);
    uint4* base = As + ((t * OZ_S) * nkc + kc) * 128 + rr;
#pragma unroll
    for (int p = 0; p < OZ_S; ++p) base[(int64_t)p * nkc * 128] = make_uint4(w[0][p], w[1][p], w[2][p], w[3][p]);
  }
}

// T (k x nj, ldt) -> per 32-column tile j the error kernel's B operand: the 8 slices
// concatenated along N (slice q = rows 32 q .. 32 q + 31), K-major: [j][kc][q][c 32][16 B];
// fsc[c] = 2^{E_c}.  Thread per column (padded to the tile).
__global__ void __launch_bounds__(128) k_oz_slice_t(const double* __restrict__ T, int64_t ldt, int k, int nj, int KP,
                                                    uint4* __restrict__ Ts, double* __restrict__ fsc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;   // grid covers the padded columns
  const bool live = c < nj;
  double mx = 0.0;
  if (live)
    for (int l = 0; l < k; ++l) mx = fmax(mx, fabs(T[(int64_t)c * ldt + l]));
  const int E = oz_exp(mx);
  const double sc = pow2(56 - E);
  fsc[c] = live ? pow2(E) : 0.0;
  const int j = c / ER_N, cc = c % ER_N;
  const int nkc = KP / 16;
  for (int kc = 0; kc < nkc; ++kc) {
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int l = kc * 16 + i;
      v[i] = (live && l < k) ? T[(int64_t)c * ldt + l] : 0.0;
    }
    uint32_t w[4][8];
#pragma unroll
    for (int g = 0; g < 4; ++g) oz_slice4(v + 4 * g, sc, w[g]);
    uint4* base = Ts + (((int64_t)j * nkc + kc) * OZ_S) * ER_N + cc;
#pragma unroll
    for (int q = 0; q < OZ_S; ++q) base[q * ER_N] = make_uint4(w[0][q], w[1][q], w[2][q], w[3][q]);
  }
}

// ---------------------------------------------------------------------------
// [G2 | W] = Q1^T [Q1 | A_D(:, J)] on kind::i8.  CTA b = (row group g = b / ntiles, tile
// t = b % ntiles): rows [g spg, (g+1) spg) K-steps, output columns c' = 64 t .. 64 t + 63 of
// B' = [Q1 | A_D(:, J)] (c' < kq: Q1(:, c'); else A_D(:, cmap[c' - kq])).  CTAs of one row
// group read the same A (Q1 slice) stages at about the same time, so the A stream is served
// from L2 after the first reader.
//   warp 0      bulk copies of the A stages (32 KB, one K-step each)
//   warp 1      MMA issuer: per K-step the 36 digit pairs, 8 diagonal accumulators of 64
//               columns (all 512 TMEM columns), drained every TN_CHS K-steps
//   warps 2..9  slice B in-kernel (thread = (column, 8 rows): 8 fp64 -> 8 x 8 B) and drain
//               the accumulators into fp64 registers (warp w: TMEM lanes 32 (w % 4), 32
//               columns (w - 2) / 4)
// Operand traffic, not arithmetic, bounds a naive slice-pair loop: every tcgen05.mma reads its
// whole A (128 x 32 B) and B (N x 32 B) from shared memory, and a thread issues at most about
// one MMA per 50 cycles (tools/mma_rate_probe.cu, tools/issue_probe.cu; profiles/r02_*probe*).
// So the B slices are laid out CONCATENATED along N (slice q's 64 columns are rows 64 q ..
// 64 q + 63 of one K-major operand) and the accumulators diagonal-major (diagonal d at TMEM
// columns 64 d): ONE MMA of A slice p against B slices 0 .. 7 - p (N = 64 (8 - p)) lands
// product (p, q) exactly in diagonal p + q's accumulator.  N <= 256 per instruction, so
// p < 4 takes two MMAs: 12 MMAs per K-step instead of 36, A read 12 times instead of 36.
__device__ __forceinline__ void tn_kstep(uint32_t tmem, uint32_t a, uint32_t b, bool first) {
#pragma unroll
  for (int pa = 0; pa < OZ_S; ++pa) {
    const uint64_t da = oz_sdesc(a + pa * 4096, 2048, 128);
    const int nq = OZ_S - pa;                       // B slices 0 .. 7 - pa
    const int n0 = nq > 4 ? 4 : nq;                 // first MMA: slices 0 .. n0 - 1
    oz_mma(tmem + (uint32_t)(pa * TN_N), da, oz_sdesc(b, 8192, 128), oz_idesc(n0 * TN_N),
           (first && pa == 0) ? 0u : 1u);
    if (nq > 4)                                     // second MMA: slices 4 .. 7 - pa
      oz_mma(tmem + (uint32_t)((pa + 4) * TN_N), da, oz_sdesc(b + 4 * 8 * 128, 8192, 128), oz_idesc((nq - 4) * TN_N),
             (first && pa == 0) ? 0u : 1u);
  }
}

struct OzTN {
  const uint4* As;                   // Q1 slices
  const unsigned long long* cmaxq;   // Q1 column max |x| (bit patterns)
  const unsigned long long* cmaxd;   // A_D column max |x|, original column order
  const double* Q1;
  int64_t ldq;
  const double* AD;
  int64_t ld;
  const int* cmap;                   // J columns (perm + k)
  int kq;                            // leading columns of B' taken from Q1 (= k)
  int ncol;                          // columns of B' (k + nj)
  int64_t m;
  int64_t nsteps;                    // ceil(m / 32)
  int ntiles, ngroups;
  int64_t spg;                       // K-steps per row group
  int vec;                           // 16 B loads allowed (even ld / ldq, aligned bases)
  double* part;                      // [ngroups][ntiles][128][64]
  int dbg;                           // measurement knobs (MPID_OZ_DBG): 1 = B not sliced, 2 = A not loaded
};

__global__ void __launch_bounds__(TN_THREADS, 1) k_oz_tn(const OzTN p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full_a = reinterpret_cast<uint64_t*>(smem + TN_NST * (TN_A + TN_B));
  uint64_t* full_b = full_a + TN_NST;
  uint64_t* empty = full_b + TN_NST;
  uint64_t* acc_full = empty + TN_NST;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  double* ea = reinterpret_cast<double*>(smem + TN_NST * (TN_A + TN_B) + 128);   // [128] 2^{Ea - 14}
  double* eb = ea + 128;                                                           // [64]  2^{Eb}
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x / p.ntiles, t = blockIdx.x % p.ntiles;
  const int64_t s0 = (int64_t)g * p.spg;
  const int64_t s1 = min(p.nsteps, s0 + p.spg);
  const int64_t nst = s1 > s0 ? s1 - s0 : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TN_NST; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&full_b[s], TN_SLW);
      mbar_init(&empty[s], TN_NI);
    }
    mbar_init(acc_full, TN_NI);
    mbar_init(acc_empty, TN_SLW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 128) {
    const int l = threadIdx.x;
    ea[l] = l < p.kq ? pow2(oz_exp(__longlong_as_double((long long)p.cmaxq[l])) - 14) : 0.0;
  } else if (threadIdx.x < 192) {
    const int c = threadIdx.x - 128, cp = t * TN_N + c;
    double mx = 0.0;
    if (cp < p.kq) mx = __longlong_as_double((long long)p.cmaxq[cp]);
    else if (cp < p.ncol) mx = __longlong_as_double((long long)p.cmaxd[p.cmap[cp - p.kq]]);
    eb[c] = pow2(oz_exp(mx));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- A producer ----------------
    // (an L2 prefetch of B's fp64 rows by this warp's lanes, cp.async.bulk.prefetch, made the
    // kernel slower: the prefetches queue in the SM's TMA unit ahead of the A loads)
    for (int64_t i = 0; i < nst; ++i) {
      const int slot = (int)(i % TN_NST);
      if (lane == 0) {
        if (i >= TN_NST) mbar_wait(&empty[slot], (uint32_t)(((i / TN_NST) - 1) & 1));
        if (p.dbg & 2) {
          mbar_arrive(&full_a[slot]);
        } else {
          mbar_expect_tx(&full_a[slot], TN_A);
          tma_load(smem + slot * (TN_A + TN_B), p.As + (s0 + i) * (TN_A / 16), TN_A, &full_a[slot]);
        }
      }
    }
  } else if (warp <= TN_NI) {
    // ---------------- MMA issuer: 12 MMAs per K-step (tn_kstep) ----------------
    if (lane == 0) {
      
      int cpos = 0;
      uint32_t aph = 0;
      for (int64_t i = 0; i < nst; ++i) {
        const int slot = (int)(i % TN_NST);
        const uint32_t ph = (uint32_t)((i / TN_NST) & 1);
        if (cpos == 0 && i > 0) {
          mbar_wait(acc_empty, aph ^ 1);   // the previous chunk has been drained
          tc_fence_after();
        }
        mbar_wait(&full_a[slot], ph);
        mbar_wait(&full_b[slot], ph);
        tc_fence_after();
        const uint32_t a = su32(smem + slot * (TN_A + TN_B)), b = a + TN_A;
        const bool first = cpos == 0;
        tn_kstep(tmem, a, b, first);
        oz_commit(&empty[slot]);
        if (++cpos == TN_CHS || i == nst - 1) {
          oz_commit(acc_full);
          cpos = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ---------------- B slicers + drain ----------------
    // TN_SLW warps: thread = (column c, RPT consecutive rows of the 32-row K-step)
    constexpr int RPT = KSTEP * TN_N / (32 * TN_SLW);          // rows per thread (4 with 16 warps)
    constexpr int CW = TN_N * 4 / TN_SLW;                      // drain: columns per warp (16 with 16 warps)
    const int sw = warp - 1 - TN_NI;
    const int tid = sw * 32 + lane;
    // lanes of a warp take consecutive row groups of the same few columns, so each warp load
    // reads whole 256 B column segments (coalesced) instead of 32 B from 32 columns
    constexpr int NRG = KSTEP / RPT;                           // row groups per K-step
    const int c = tid / NRG, ro = tid % NRG;                   // column, row group of RPT rows
    const int cp = t * TN_N + c;
    const double* col = nullptr;
    if (cp < p.kq) col = p.Q1 + (int64_t)cp * p.ldq;
    else if (cp < p.ncol) col = p.AD + (int64_t)p.cmap[cp - p.kq] * p.ld;
    const double sc = col ? pow2(56 - oz_exp(cp < p.kq ? __longlong_as_double((long long)p.cmaxq[cp])
                                                       : __longlong_as_double((long long)p.cmaxd[p.cmap[cp - p.kq]])))
                          : 0.0;
    // B stage, slices concatenated along N: element (q, c, k) at (k / 16) * 8192 +
    // (8 q + c / 8) * 128 + (c % 8) * 16 + k % 16; this thread's rows k = ro RPT .. + RPT - 1
    const int k0 = ro * RPT;
    const uint32_t boff = (uint32_t)((k0 >> 4) * 8192 + (c >> 3) * 128 + (c & 7) * 16 + (k0 & 15));
    // drain mapping: TMEM lane quarter warp % 4, CW columns (sw / 4)
    const int quarter = warp & 3, cgrp = sw >> 2;
    // the drained chunk sums accumulate in this thread's own slots of the partials
    double* out = p.part + (((int64_t)g * p.ntiles + t) * 128 + quarter * 32 + lane) * TN_N + cgrp * CW;
    bool first_drain = true;
    double v[RPT], n1[RPT], n2[RPT];   // the current K-step's values and the next two (loads 2 K-steps ahead)
    auto loadr = [&](int64_t s, double* dst) {
      const int64_t r0 = s * KSTEP + k0;
      if (col && r0 + RPT <= p.m && p.vec) {
        const double2* q = reinterpret_cast<const double2*>(col + r0);
#pragma unroll
        for (int i = 0; i < RPT / 2; ++i) {
          const double2 x = __ldcs(q + i);
          dst[2 * i] = x.x;
          dst[2 * i + 1] = x.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < RPT; ++i) dst[i] = (col && r0 + i < p.m) ? __ldcs(col + r0 + i) : 0.0;
      }
    };
    if (nst > 0 && !(p.dbg & 1)) loadr(s0, n1);
    if (nst > 1 && !(p.dbg & 1)) loadr(s0 + 1, n2);
    int cpos = 0;
    uint32_t aph = 0;
    for (int64_t i = 0; i < nst; ++i) {
      const int slot = (int)(i % TN_NST);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        v[q] = n1[q];
        n1[q] = n2[q];
      }
      if (i + 2 < nst && !(p.dbg & 1)) loadr(s0 + i + 2, n2);
      uint32_t w[RPT / 4][8];
#pragma unroll
      for (int g4 = 0; g4 < RPT / 4; ++g4) oz_slice4(v + 4 * g4, sc, w[g4]);
      if (i >= TN_NST) mbar_wait(&empty[slot], (uint32_t)(((i / TN_NST) - 1) & 1));
      unsigned char* bst = smem + slot * (TN_A + TN_B) + TN_A + boff;
      if (!(p.dbg & 1)) {
#pragma unroll
        for (int q = 0; q < OZ_S; ++q) {
          if constexpr (RPT == 8) *reinterpret_cast<uint2*>(bst + q * 1024) = make_uint2(w[0][q], w[1][q]);
          else *reinterpret_cast<uint32_t*>(bst + q * 1024) = w[0][q];
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_b[slot]);
      if (++cpos == TN_CHS || i == nst - 1) {
        cpos = 0;
        mbar_wait(acc_full, aph);
        aph ^= 1;
        tc_fence_after();
        const double sa = ea[quarter * 32 + lane];
#pragma unroll 1
        for (int h = 0; h < CW / 4; ++h) {
          uint32_t r[OZ_S][4];
#pragma unroll
          for (int d = 0; d < OZ_S; ++d)
            OZ_LD4(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(d * TN_N + cgrp * CW + h * 4), r[d]);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double x = i2d(r[OZ_S - 1][j]);
#pragma unroll
            for (int d = OZ_S - 2; d >= 0; --d) x = fma(x, 0.0078125, i2d(r[d][j]));
            const double val = x * sa * eb[cgrp * CW + h * 4 + j];
            out[h * 4 + j] = first_drain ? val : out[h * 4 + j] + val;
          }
        }
        first_drain = false;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
      }
    }
    if (first_drain)   // no rows in this group: zero partials
      for (int j = 0; j < CW; ++j) out[j] = 0.0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// G2 (k x k) and W (k x nj), col-major, ld k: sums over the row groups in order
__global__ void k_oz_tn_reduce(const double* __restrict__ part, int ngroups, int ntiles, int k, int kq, int ncol,
                               double* __restrict__ G2, double* __restrict__ W) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)k * ncol) return;
  const int l = (int)(idx % k), cp = (int)(idx / k);
  const int t = cp / TN_N, c = cp % TN_N;
  double s = 0.0;
  for (int g = 0; g < ngroups; ++g) s += part[(((int64_t)g * ntiles + t) * 128 + l) * TN_N + c];
  if (cp < kq) G2[(int64_t)cp * k + l] = s;
  else W[(int64_t)(cp - kq) * k + l] = s;
}

// ---------------------------------------------------------------------------
// error: persistent over 128-row tiles; per tile the A operand (A_I's slices, 8 x 128 x KP)
// stays in shared memory while the tile walks every 32-column tile of J (T's slices, two
// stages); TMEM holds two buffers of 8 diagonal accumulators x 32 columns.
//   warp 0      bulk copies (A per row tile, B per J tile)
//   warp 1      MMA issuer: 36 digit pairs x KP/32 K-steps per J tile
//   warps 2..9  epilogue: warp w reads TMEM lanes 32 (w % 4) (rows), 16 columns
//               ((w - 2) / 4): A_I T by Horner over the diagonals, the residual against
//               A_D(r, J_c) (loaded before the wait), squares summed in fp64
struct OzErr {
  const uint4* As;        // A_I slices per row tile
  const double* rsc;      // per row 2^{E_r - 35} (2^{E_r - 14} and oz_combine8's 2^{-21})
  const uint4* Ts;        // T slices per J tile
  const double* fsc;      // per column 2^{E_c}
  const double* AD;
  int64_t ld;
  const int* cmap;        // J
  int64_t m;
  int nj, KP;
  int vec;                // A_D rows 16 B aligned (even ld, aligned base): L2 prefetch allowed
  int dbg;                // measurement knobs (MPID_OZ_DBG): 4 = no L2 prefetch
  int64_t nrt;            // row tiles
  int njt;                // J tiles
  double* part;           // [gridDim.x]
};

__global__ void __launch_bounds__(ER_THREADS, 1) k_oz_err(const OzErr p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int ABYTES = OZ_S * 128 * p.KP, BBYTES = OZ_S * ER_N * p.KP;
  unsigned char* sA = smem;
  unsigned char* sB = smem + ABYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + 2 * BBYTES);
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 1;
  uint64_t* b_full = bars + 2;      // [2]
  uint64_t* b_empty = bars + 4;     // [2]
  uint64_t* acc_full = bars + 6;    // [2]
  uint64_t* acc_empty = bars + 8;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  double* red = reinterpret_cast<double*>(bars + 12);
  // element offsets of the J columns in A_D (cmap[c] * ld), staged once: the epilogue's A_D
  // loads then depend on a shared-memory read, not on a global load of the column map
  int64_t* coff = reinterpret_cast<int64_t*>(bars + 32);
  for (int c = threadIdx.x; c < p.njt * ER_N; c += blockDim.x) coff[c] = c < p.nj ? (int64_t)p.cmap[c] * p.ld : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t my_rt = blockIdx.x < p.nrt ? (p.nrt - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    mbar_init(a_empty, ER_NI);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], ER_NI);
      mbar_init(&acc_full[i], ER_NI);
      mbar_init(&acc_empty[i], ER_EPW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  double ss = 0.0;

  if (warp == 0) {
    if (lane == 0) {
      int64_t jc = 0;
      for (int64_t i = 0; i < my_rt; ++i) {
        const int64_t rt = blockIdx.x + i * gridDim.x;
        if (i > 0) mbar_wait(a_empty, (uint32_t)((i - 1) & 1));
        mbar_expect_tx(a_full, (uint32_t)ABYTES);
#pragma unroll 1
        for (int q = 0; q < OZ_S; ++q)
          tma_load(sA + q * (ABYTES / OZ_S), p.As + (rt * ABYTES + (int64_t)q * (ABYTES / OZ_S)) / 16,
                   (uint32_t)(ABYTES / OZ_S), a_full);
        for (int jt = 0; jt < p.njt; ++jt, ++jc) {
          const int st = (int)(jc & 1);
          if (jc >= 2) mbar_wait(&b_empty[st], (uint32_t)(((jc >> 1) - 1) & 1));
          mbar_expect_tx(&b_full[st], (uint32_t)BBYTES);
          tma_load(sB + st * BBYTES, p.Ts + (int64_t)jt * (BBYTES / 16), (uint32_t)BBYTES, &b_full[st]);
        }
      }
    }
  } else if (warp <= ER_NI) {
    // MMA issuer: per K-step (32 of the KP columns of A_I) one MMA per A slice p against T's
    // slices 0 .. 7 - p concatenated along N (N = 32 (8 - p) <= 256), landing product (p, q)
    // in diagonal p + q's accumulator (TMEM columns 32 (p + q) of the buffer)
    if (lane == 0) {
      const uint32_t a0 = su32(sA), b0 = su32(sB);
      int64_t jc = 0;
      for (int64_t i = 0; i < my_rt; ++i) {
        mbar_wait(a_full, (uint32_t)(i & 1));
        tc_fence_after();
        for (int jt = 0; jt < p.njt; ++jt, ++jc) {
          const int st = (int)(jc & 1), buf = (int)(jc & 1);
          mbar_wait(&b_full[st], (uint32_t)((jc >> 1) & 1));
          if (jc >= 2) mbar_wait(&acc_empty[buf], (uint32_t)(((jc >> 1) - 1) & 1));
          tc_fence_after();
          const uint32_t bb = b0 + (uint32_t)(st * BBYTES);
          const uint32_t dt = tmem + (uint32_t)(buf * OZ_S * ER_N);
          for (int kk = 0; kk < p.KP / KSTEP; ++kk) {
            const uint64_t db = oz_sdesc(bb + (uint32_t)(kk * 2 * OZ_S * ER_N * 16), OZ_S * ER_N * 16, 128);
#pragma unroll
            for (int pa = 0; pa < OZ_S; ++pa)
              oz_mma(dt + (uint32_t)(pa * ER_N),
                     oz_sdesc(a0 + (uint32_t)(pa * (ABYTES / OZ_S) + kk * 4096), 2048, 128), db,
                     oz_idesc((OZ_S - pa) * ER_N), (pa == 0 && kk == 0) ? 0u : 1u);
          }
          oz_commit(&b_empty[st]);
          oz_commit(&acc_full[buf]);
        }
        oz_commit(a_empty);
      }
    }
  } else {
    // warp: TMEM lane quarter warp % 4 (rows), ECW columns of each tile (ew / 4)
    constexpr int ECW = ER_N * 4 / ER_EPW;            // columns per epilogue warp (8 with 16 warps)
    const int ew = warp - 1 - ER_NI, quarter = warp & 3, cg = ew >> 2;
    int64_t jc = 0;
    for (int64_t i = 0; i < my_rt; ++i) {
      const int64_t rt = blockIdx.x + i * gridDim.x;
      const int64_t r = rt * 128 + quarter * 32 + lane;
      const bool live = r < p.m;
      const double rs = live ? p.rsc[r] : 0.0;
      for (int jt = 0; jt < p.njt; ++jt, ++jc) {
        const int buf = (int)(jc & 1);
        const int c0 = jt * ER_N + cg * ECW;
        double a[ECW];
#pragma unroll
        for (int j = 0; j < ECW; ++j) {
          const int c = c0 + j;
          a[j] = (live && c < p.nj) ? __ldcs(p.AD + coff[c] + r) : 0.0;
        }
        // the next J tile's A_D elements of this thread into L2 (no registers held): its
        // loads, issued one tile from now, then wait on L2 instead of HBM
        if (live && jt + 1 < p.njt) {
#pragma unroll
          for (int j = 0; j < ECW; ++j) {
            const int c = c0 + ER_N + j;
            if (c < p.nj) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.AD + coff[c] + r));
          }
        }
        mbar_wait(&acc_full[buf], (uint32_t)((jc >> 1) & 1));
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * OZ_S * ER_N + cg * ECW);
#pragma unroll
        for (int h = 0; h < ECW / 8; ++h) {
          uint32_t acc[OZ_S][8];
#pragma unroll
          for (int d = 0; d < OZ_S; ++d) OZ_LD8(ta + (uint32_t)(d * ER_N + h * 8), acc[d]);
          tmem_wait_ld();
          if (h == ECW / 8 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = c0 + h * 8 + j;
            uint32_t dg[OZ_S];
#pragma unroll
            for (int d = 0; d < OZ_S; ++d) dg[d] = acc[d][j];
            const double x = oz_combine8(dg);               // sum_d acc_d 2^{-7d} times 2^21
            const double fs = c < p.nj ? __ldg(p.fsc + c) : 0.0;
            const double e = fma(-x, rs * fs, a[h * 8 + j]);
            ss = fma(e, e, ss);
          }
        }
      }
    }
  }
  // block sum of ss (fixed order)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[warp] = ss;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < ER_THREADS / 32; ++w) t += red[w];
    p.part[blockIdx.x] = t;
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---------------------------------------------------------------------------
size_t oz_slice_bytes(int64_t m_local) {   // the A-operand slices of either GEMM (shared buffer)
  const int64_t mp = (m_local + 127) / 128 * 128;
  return (size_t)mp * 1024;
}
size_t oz_tslice_bytes(int64_t n) { return (size_t)((n + ER_N - 1) / ER_N + 1) * OZ_S * ER_N * 128; }
size_t oz_part_doubles(int num_sms) { return (size_t)num_sms * 128 * TN_N; }

static int oz_kp(int k) { return (k + KSTEP - 1) / KSTEP * KSTEP; }
static size_t oz_err_smem(int k, int nj) {
  const int KP = oz_kp(k), njt = (nj + ER_N - 1) / ER_N;
  return (size_t)OZ_S * 128 * KP + 2 * (size_t)OZ_S * ER_N * KP + 256 + (size_t)njt * ER_N * 8 + 1024;
}
// the shapes the int8 kernels take: k <= 128, the TN grid within one CTA per SM, the error
// kernel's shared memory (A slices, two B stages, the J columns' offsets) within 227 KB
bool oz_fits(int64_t n, int k, int num_sms) {
  if (k < 1 || k > 128 || n <= k) return false;
  if ((n + TN_N - 1) / TN_N > num_sms) return false;
  return oz_err_smem(k, (int)(n - k)) <= 227 * 1024;
}

// [G2 | W] = Q1^T [Q1 | A_D(:, J)]; cmaxq (k entries) is computed here; cmaxd = A_D's column maxima
cudaError_t launch_oz_tn(const double* Q1, int64_t m, int k, const double* AD, int64_t ld, const int* cmapJ, int nj,
                         const unsigned long long* cmaxd, unsigned long long* cmaxq, void* slices, double* part,
                         size_t part_cap, double* G2, double* W, int num_sms, cudaStream_t st, int cmaxq_ready) {
  if (k < 1 || k > 128) return cudaErrorInvalidValue;
  cudaError_t e = cudaSuccess;
  if (!cmaxq_ready) {
    if ((e = cudaMemsetAsync(cmaxq, 0, 128 * sizeof(unsigned long long), st)) != cudaSuccess) return e;
    const int ysplit = (int)std::max<int64_t>(1, std::min<int64_t>(64, (2 * num_sms + k - 1) / k));
    k_oz_colmax<<<dim3((unsigned)k, (unsigned)ysplit), 256, 0, st>>>(Q1, m, m, cmaxq);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const int64_t nsteps = (m + KSTEP - 1) / KSTEP;
  k_oz_slice_cols<<<(unsigned)nsteps, 256, 0, st>>>(Q1, m, m, k, cmaxq, nsteps,
                                                                           (uint4*)slices);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  OzTN p{};
  p.As = (const uint4*)slices;
  p.cmaxq = cmaxq;
  p.cmaxd = cmaxd;
  p.Q1 = Q1;
  p.ldq = m;
  p.AD = AD;
  p.ld = ld;
  p.cmap = cmapJ;
  p.kq = k;
  p.ncol = k + nj;
  p.m = m;
  p.nsteps = nsteps;
  p.ntiles = (p.ncol + TN_N - 1) / TN_N;
  p.ngroups = std::max(1, num_sms / p.ntiles);
  p.ngroups = (int)std::min<int64_t>(p.ngroups, nsteps);
  p.spg = (nsteps + p.ngroups - 1) / p.ngroups;
  p.vec = ((ld & 1) == 0 && (m & 1) == 0 && (((uintptr_t)AD) & 15) == 0 && (((uintptr_t)Q1) & 15) == 0) ? 1 : 0;
  p.part = part;
  p.dbg = getenv("MPID_OZ_DBG") ? atoi(getenv("MPID_OZ_DBG")) : 0;
  if ((size_t)p.ngroups * p.ntiles * 128 * TN_N > part_cap) return cudaErrorInvalidValue;
  if ((e = smem_attr((const void*)k_oz_tn, TN_SMEM)) != cudaSuccess) return e;
  k_oz_tn<<<p.ngroups * p.ntiles, TN_THREADS, TN_SMEM, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int64_t tot = (int64_t)k * p.ncol;
  k_oz_tn_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(part, p.ngroups, p.ntiles, k, k, p.ncol, G2, W);
  return cudaGetLastError();
}

// sum over J of (A_D(r, J_c) - (A_I T)(r, c))^2 into part[0 .. *nblk_out)
cudaError_t launch_oz_error(const double* AD, int64_t m, int64_t ld, int nj, const int* cmapJ, const double* AI,
                            int k, const double* T, int64_t ldt, void* slices, void* tslices, double* rsc,
                            double* fsc, double* part, int* nblk_out, int num_sms, cudaStream_t st) {
  if (k < 1 || k > 128 || nj < 1) return cudaErrorInvalidValue;
  const int KP = oz_kp(k);
  const int64_t nrt = (m + 127) / 128;
  k_oz_slice_rows<<<(unsigned)nrt, 128, 0, st>>>(AI, m, m, k, KP, (uint4*)slices, rsc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int njt = (nj + ER_N - 1) / ER_N;
  k_oz_slice_t<<<(unsigned)((njt * ER_N + 127) / 128), 128, 0, st>>>(T, ldt, k, nj, KP, (uint4*)tslices, fsc);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  OzErr p{};
  p.As = (const uint4*)slices;
  p.rsc = rsc;
  p.Ts = (const uint4*)tslices;
  p.fsc = fsc;
  p.AD = AD;
  p.ld = ld;
  p.cmap = cmapJ;
  p.m = m;
  p.nj = nj;
  p.KP = KP;
  p.vec = ((ld & 1) == 0 && (((uintptr_t)AD) & 15) == 0) ? 1 : 0;
  p.dbg = getenv("MPID_OZ_DBG") ? atoi(getenv("MPID_OZ_DBG")) : 0;
  p.nrt = nrt;
  p.njt = njt;
  p.part = part;
  const int smem = (int)oz_err_smem(k, nj);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if ((e = smem_attr((const void*)k_oz_err, smem)) != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>(nrt, num_sms);
  *nblk_out = grid;
  k_oz_err<<<grid, ER_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace mpid
