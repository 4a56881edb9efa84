// k_pass_tc — the per-step panel pass of the low-precision pivoted Householder QR with the
// trailing block formed on the 5th-generation tensor cores (tcgen05 + TMEM): SURVEY §8(a)
// "D-OTF", the default for fp16 storage (Algorithm 2 line 4; Eq. (6)-(7),
// P:115-128; the blocked trailing-matrix update of north_star / P:402 as a rank-nb
// tensor-core GEMM with K = the pending reflectors of the panel).
//
// What one launch computes for step j (readings R4, R6, R14):
//   X = S - V F^T, the current trailing block, formed ENTIRELY in the tensor core's fp32
//   accumulator (TMEM), never written to HBM:
//     D  = S^T I                       8 MMAs (N = 16 rows, K = 16 rows) per 128 x 128 unit:
//                                      the stored fp16 tile itself is the A operand (the
//                                      8-row interleaved layout IS the K-major core-matrix
//                                      layout), B = a 16 x 16 identity -> D(c, r) = S(r, c)
//     D += (-F_hi) V_hi^T + (-F_hi) V_lo^T + (-F_lo) V_hi^T      (kind::f16, K = 16 per MMA)
//   with V, F the pending fp32 vectors split into fp16 hi / lo pairs (|rel. error| of the
//   product <= ~2^-21, R14), so the epilogue reads X directly (no conversion, no
//   subtraction on the CUDA cores);
//   u = X(:, j) (the pivot column), w = X^T u and s_i = ||X(j:m, i)||^2 (8-row fp32 FFMA2
//   chains, folded per unit and added into fp64), the row x = X(j, :); on store steps (panel
//   end, every nb steps) fl16(X) is written back to S (the storage rounding point).
//   V holds the pending u_l (rows < l zero) and F the pending c_l f_l, so V F^T =
//   sum_l v_l f_l^T with v_l = c_l u_l (Householder vector, v_l(l) = 1 in exact arithmetic).
//
// B200 structure: one persistent CTA per SM, 20 warps, warp-specialised.  A CTA owns a
// contiguous range of 128-row blocks and walks, per row block, all column tiles of 128
// (tile 0 starts at column j, so its TMEM lane 0 is the pivot column): unit = (row block,
// tile).
//   warp 0      TMA producer: per unit one 2-D tensor-map box of S (128 columns x 16 row
//               groups = 32 KB) + the tile's F operand (bulk copy, L2-resident); per row
//               block the V operand (bulk copy).  NST-deep ring; on store steps the
//               rounded tile is written back by a tensor-map store before the slot is reused.
//   warps 1, 19 MMA issuers (one elected thread each; even / odd tiles of every row block): 8
//               identity MMAs + 3 x ceil(npend / 16) formation MMAs per unit into one of 4
//               TMEM accumulators (128 columns each).  Their per-unit instruction stream is
//               the pass's critical path: counters are incremental, descriptors constant + address.
//   warps 2-17  epilogue, 2 groups of 8 warps (4 TMEM lane quarters x 2 row halves); group g
//               takes the tiles t = g mod 2, so each thread owns one column per tile and keeps
//               its column sums in registers for the whole launch; units without store, pivot
//               row or masked rows take a branch-free unrolled path.
//   warp 18     the u warp: each row block's V operand and pivot column (3 buffers: it runs a block
//               ahead of the issuers), u = S(:, j) - V F(j, :)^T on CUDA cores, published to
//               shared memory and to the V operand of the next steps.
// Bound: HBM — (m - j)(n - j) 2 bytes read per step (+ the same written on store steps);
// tensor work per element: 32 flops (identity) + 6 * 16 * ceil(npend / 16) (formation).
#include "mpid_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace mpid {

namespace {
constexpr int C_T = 128;            // columns per tile = MMA M = TMEM lanes
constexpr int R_B = 128;            // rows per row block = formation MMA N = TMEM columns per accumulator
constexpr int RG_B = R_B / 8;       // row groups per row block
constexpr int EPI_WARPS = 16;
constexpr int NGRP = 2;             // epilogue groups: group g takes the tiles t = g mod 2
constexpr int EPI_GW = EPI_WARPS / NGRP;   // warps per group: 4 lane quarters x 2 row halves
constexpr int BLOCK = 32 * (2 + EPI_WARPS + 2);   // + producer, 2 MMA issuers, u warp
constexpr int NACC = 4;             // TMEM accumulators
constexpr int NVB_MAX = 3;          // row-block buffers (V operand + pivot column)
constexpr int TMEM_COLS = R_B * NACC;
constexpr int S_BYTES = C_T * R_B * 2;   // one fp16 unit tile (32 KB)
constexpr int CH_BYTES = 4096;      // one K chunk (16) of a 128-row / 128-column operand, fp16
constexpr int UWARP = 2 + EPI_WARPS;  // the pivot-column (u) warp
constexpr int MMA2 = UWARP + 1;       // the second MMA issuer (odd tiles; warp 1 takes the even ones)
constexpr int TC_SMEM_MAX = 227 * 1024;   // the sm_100 opt-in maximum of dynamic shared memory per block

// Shared-memory matrix descriptors (K-major, no swizzle) are built in the issuer loop as two
// 32-bit words: low = (address >> 4) | (LBO >> 4) << 16 (LBO = byte stride between core
// matrices adjacent along K), high = (SBO >> 4) | 1 << 14 (SBO = stride along M / N; bit 46 of
// the descriptor = the sm_100 descriptor version).
// kind::f16: fp16 A and B, fp32 accumulator, both K-major, M = 128, N given
__device__ __forceinline__ uint32_t idesc_f16(int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(C_T >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tm),
               "r"(c0), "r"(c1), "r"(su32(src))
               : "memory");
}
// byte offset of (row-or-column i, pending l) inside one K-chunk operand block: [i / 8][l / 8 % 2][i % 8][l % 8]
__host__ __device__ __forceinline__ int op_off(int i, int l) {
  return (i >> 3) * 256 + ((l >> 3) & 1) * 128 + (i & 7) * 16 + (l & 7) * 2;
}
// one lane of a converged warp (the lowest) -> true
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void split_f16(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));   // x - hi is exact in fp32
}

struct Geo {
  int slot;        // bytes per ring slot: the S unit tile (32 KB), then the tile's F operand (hi, lo)
  int f_off;
  int v0;          // per-row-block buffers (nvb): V operand (hi, lo) x kchw chunks, then the pivot column
  int vsz;         // bytes of one row-block buffer
  int pcol;        // pivot column offset inside a row-block buffer (16 row groups x 16 B)
  int ident;       // 16 x 16 identity operand (512 B)
  int ubuf;        // 2 x 128 floats: u of a row block
  int fj;          // 2 x 32 floats: -F(j, l) hi / lo (the pivot column's F row)
  int bars;
  int total;
};
__host__ __device__ inline Geo geo_of(int kchw, int nst, int nvb) {
  Geo g;
  g.f_off = S_BYTES;
  g.slot = S_BYTES + 2 * kchw * CH_BYTES;
  g.v0 = nst * g.slot;
  g.pcol = 2 * kchw * CH_BYTES;
  g.vsz = g.pcol + RG_B * 16;
  g.ident = g.v0 + nvb * g.vsz;
  g.ubuf = g.ident + 512;
  g.fj = g.ubuf + 2 * R_B * 4;
  g.bars = g.fj + 2 * 32 * 4;
  g.total = g.bars + (2 * nst + 2 * NACC + 2 * NVB_MAX + 4) * 8 + 16;
  return g;
}
}  // namespace

struct TcParams {
  int64_t m_pad;       // rows of the shard, padded (multiple of 256)
  int64_t m_local;
  int64_t row_offset;
  int64_t rb_first;    // first 128-row block holding rows >= j (local)
  int64_t nrb;         // row blocks from rb_first to the end
  int n, j, j0, npend, store, kchw, nst, ntiles;
  int nvb;                    // row-block buffers: 3 lets the u warp run a block ahead of the MMAs
  int nmma;                   // MMA issuer warps (2 needs an even ring depth: one consumer per slot)
  unsigned char* Vop;         // [m_pad / 128][kchw][hi 4 KB | lo 4 KB]
  int lnext;                  // V operand column of u_j for the next step (j mod nb)
  const unsigned char* Fop;   // [ntiles][kchw][hi 4 KB | lo 4 KB]
  float* U;                   // [NSLOT][m_pad] u vectors (fp32)
  double* part;               // [gridDim.x][2][n]
  double* xr;                 // [n] row j of X (owner)
  const DevScalars* sc;
};

// TPG: column tiles per epilogue group (4: n - j <= 1024, 8: <= 2048)
template <int TPG>
__global__ void __launch_bounds__(BLOCK, 1) k_pass_tc(TcParams p, const __grid_constant__ CUtensorMap tmS,
                                                     const __grid_constant__ CUtensorMap tmC) {
  if (p.sc->done) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = p.n, j = p.j, NST = p.nst, kchw = p.kchw, ntiles = p.ntiles, npend = p.npend;
  const int kch = (npend + 15) >> 4;             // K chunks holding pending reflectors
  const int NVB = p.nvb;
  const Geo geo = geo_of(kchw, NST, NVB);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + geo.bars);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + NACC;
  uint64_t* vfull = tempty + NACC;
  uint64_t* vempty = vfull + NVB_MAX;
  uint64_t* ufull = vempty + NVB_MAX;
  uint64_t* ufree = ufull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ufree + 2);
  float* ubuf = reinterpret_cast<float*>(smem + geo.ubuf);
  float* fj = reinterpret_cast<float*>(smem + geo.fj);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // row blocks of this CTA
  // row blocks of this CTA: a balanced split (CTAs differ by at most one block)
  const int64_t rb0 = p.nrb * blockIdx.x / gridDim.x;
  const int64_t rb1 = p.nrb * (blockIdx.x + 1) / gridDim.x;
  const int nrbc = rb0 < rb1 ? (int)(rb1 - rb0) : 0;
  const int64_t units = (int64_t)nrbc * ntiles;
  const int64_t jl = (int64_t)j - p.row_offset;   // local row of the pivot row (may be outside)

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.store ? EPI_GW : 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_GW);
    }
    for (int b = 0; b < NVB_MAX; ++b) {
      mbar_init(&vfull[b], 1);
      mbar_init(&vempty[b], p.nmma);          // each MMA issuer's commit after its last unit of the row block
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ufull[b], 1);
      mbar_init(&ufree[b], EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 2) {
    // 16 x 16 identity as the B operand of the S^T I MMAs: [n / 8][k / 8][n % 8][k % 8]
    __half* I = reinterpret_cast<__half*>(smem + geo.ident);
    for (int e = lane; e < 256; e += 32) {
      const int r = e >> 4, k = e & 15;
      I[op_off(r, k) / 2] = __float2half(r == k ? 1.f : 0.f);
    }
    fence_async_smem();
  }
  if (warp == UWARP) {
    // -F(j, l) (hi, lo) of the pivot column: row 0 of tile 0 of the F operand
    const int l = lane;
    float h = 0.f, lo = 0.f;
    if (l < npend) {
      const unsigned char* b = p.Fop + (size_t)(l >> 4) * 2 * CH_BYTES;
      const int o = op_off(0, l & 15);
      h = __half2float(*reinterpret_cast<const __half*>(b + o));
      lo = __half2float(*reinterpret_cast<const __half*>(b + CH_BYTES + o));
    }
    fj[l] = h;
    fj[32 + l] = lo;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  double aw[TPG], as[TPG];                       // epilogue: the column sums of its tiles
#pragma unroll
  for (int z = 0; z < TPG; ++z) { aw[z] = 0.0; as[z] = 0.0; }
  if (warp == 0) {
    // ============================ TMA producer ============================
    // the whole warp walks the loop (warp-uniform values stay in uniform registers); one
    // elected lane (the lowest, always lane 0 here) issues the copies, commits and waits
    if (units > 0) {
      const uint32_t fbytes = (uint32_t)(kch * 2 * CH_BYTES);
      auto unit_coords = [&](int64_t u, int& c0, int& g0) {
        const int64_t rbi = u / ntiles;
        const int t = (int)(u - rbi * ntiles);
        c0 = (j + t * C_T) * 2;                                 // 8-byte units (fp16: 2 per chunk)
        g0 = (int)((p.rb_first + rb0 + rbi) * RG_B);
      };
      // (incremental counters: no per-unit divisions on this single-warp critical path)
      int slot = 0;
      uint32_t phase = 0;
      int t = 0;                                                // tile of unit u
      int g0 = (int)((p.rb_first + rb0) * RG_B);                // its first row group
      const int nu = (int)units;
      for (int u = 0; u < nu; ++u) {
        if (u >= NST) {
          mbar_wait(&empty[slot], phase ^ 1);
          if (p.store) {
            int c0s, g0s;
            unit_coords(u - NST, c0s, g0s);
            if (elect_one()) {
              tma_store_2d(&tmS, c0s, g0s, smem + (size_t)slot * geo.slot);
              bulk_commit();
              bulk_wait_read0();
            }
            __syncwarp();
          }
        }
        const int c0 = (j + t * C_T) * 2;                       // 8-byte units (fp16: 2 per chunk)
        unsigned char* base = smem + (size_t)slot * geo.slot;
        if (elect_one()) {
          mbar_expect_tx(&full[slot], (uint32_t)S_BYTES + fbytes);
          tma_load_2d(base, &tmS, c0, g0, &full[slot]);
          // the tile's F operand (L2-resident)
          if (kch > 0) tma_load(base + geo.f_off, p.Fop + (size_t)t * kchw * 2 * CH_BYTES, fbytes, &full[slot]);
        }
        __syncwarp();
        if (++slot == NST) { slot = 0; phase ^= 1; }
        if (++t == ntiles) { t = 0; g0 += RG_B; }
      }
      if (p.store) {
        for (int64_t u = units > NST ? units - NST : 0; u < units; ++u) {
          const int s2 = (int)(u % NST);
          mbar_wait(&empty[s2], (uint32_t)((u / NST) & 1));
          int c0, g0;
          unit_coords(u, c0, g0);
          if (elect_one()) tma_store_2d(&tmS, c0, g0, smem + (size_t)s2 * geo.slot);
          __syncwarp();
        }
        if (elect_one()) bulk_commit();
        __syncwarp();
      }
      if (elect_one()) bulk_wait0();
      __syncwarp();
    }
  } else if (warp == 1 || warp == MMA2) {
    // ============================ MMA issuers ============================
    // Two converged warps, one elected lane each: warp 1 issues the even tiles of every row
    // block, warp MMA2 the odd ones (a single issuer's instruction stream was the critical
    // path of the pass: ~1 us per unit).  With an even tile count and ring depth (the launcher
    // checks; otherwise NM = 1) the even and odd units use disjoint accumulators, ring slots
    // and epilogue groups, and tcgen05.commit tracks the issuing thread's own MMAs, so the two
    // pipelines need no mutual ordering.
    // Descriptors are (constant high word, low word = constant + (shared address >> 4)).
    const int w = warp == 1 ? 0 : 1, NM = p.nmma;
    if (units > 0 && w < NM) {
      const uint32_t id16 = idesc_f16(16), id128 = idesc_f16(R_B);
      auto mkdesc = [](uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | (uint64_t)lo; };
      const uint32_t hi_s = (128u >> 4) | (1u << 14);           // SBO = 128 B, descriptor version
      const uint32_t hi_o = (256u >> 4) | (1u << 14);           // SBO = 256 B (operand blocks, identity)
      const uint32_t lo_s = (2048u >> 4) << 16;                 // LBO = 2048 B (S tile)
      const uint32_t lo_o = (128u >> 4) << 16;                  // LBO = 128 B
      const uint64_t dI = mkdesc(lo_o | (su32(smem + geo.ident) >> 4), hi_o);
      const uint32_t slot16 = (uint32_t)geo.slot >> 4, foff16 = (uint32_t)geo.f_off >> 4;
      const uint32_t ring16 = su32(smem) >> 4;
      const uint32_t v16 = su32(smem + geo.v0) >> 4, vsz16 = (uint32_t)geo.vsz >> 4;
      int slot = w % NST;                                       // ring slot of this warp's next unit
      uint32_t phase = (uint32_t)((w / NST) & 1);
      uint32_t vphase = 0;
      int vb = 0;
      int ubase = 0;                                            // first unit of the row block
      for (int rbi = 0; rbi < nrbc; ++rbi) {
        mbar_wait(&vfull[vb], vphase);
        if (w >= ntiles) {                                      // (one tile per block: nothing for the odd issuer)
          if (lane == 0) mbar_arrive(&vempty[vb]);
          __syncwarp();
        }
        const uint32_t w16 = lo_o | (v16 + (uint32_t)vb * vsz16);
        for (int t = w; t < ntiles; t += NM) {
          const int u = ubase + t;
          const int acc = u & (NACC - 1);
          mbar_wait(&full[slot], phase);
          mbar_wait(&tempty[acc], (uint32_t)(((u >> 2) & 1) ^ 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d = tmem + (uint32_t)(acc * R_B);
          const uint32_t s16 = ring16 + (uint32_t)slot * slot16;
          const bool last = t + NM >= ntiles;
          if (elect_one()) {
            // D(c, r) = S(r, c): A = the S tile (M = columns, K = 16 rows = 2 row groups;
            // LBO = 2048 B to the next row group, SBO = 128 B to the next 8 columns)
#pragma unroll
            for (int b = 0; b < RG_B / 2; ++b)
              mma_f16(d + (uint32_t)(16 * b), mkdesc(lo_s | (s16 + (uint32_t)(b * 256)), hi_s), dI, id16, 0u);
            // D -= F V^T in 3 hi / lo products per K chunk (operands pre-negated)
            const uint32_t f16 = lo_o | (s16 + foff16);
            for (int kc = 0; kc < kch; ++kc) {
              const uint32_t fh = f16 + (uint32_t)(kc * 2 * (CH_BYTES >> 4)), fl = fh + (CH_BYTES >> 4);
              const uint32_t vh = w16 + (uint32_t)(kc * 2 * (CH_BYTES >> 4)), vl = vh + (CH_BYTES >> 4);
              mma_f16(d, mkdesc(fh, hi_o), mkdesc(vh, hi_o), id128, 1u);
              mma_f16(d, mkdesc(fh, hi_o), mkdesc(vl, hi_o), id128, 1u);
              mma_f16(d, mkdesc(fl, hi_o), mkdesc(vh, hi_o), id128, 1u);
            }
            mma_commit(&tfull[acc]);
            if (!p.store) mma_commit(&empty[slot]);
            if (last) mma_commit(&vempty[vb]);
          }
          __syncwarp();
          // this warp's next unit is 2 further in the block, or its first tile of the next block
          const int step = last ? ntiles - t + w : NM;
          slot += step;
          while (slot >= NST) { slot -= NST; phase ^= 1; }
        }
        ubase += ntiles;
        if (++vb == NVB) { vb = 0; vphase ^= 1; }
      }
    }
  } else if (warp == UWARP) {
    // ============ u warp: V operand loads and the pivot column on CUDA cores ============
    // Loads each row block's V operand and pivot column (bulk + tensor-map copies) one row
    // block ahead, then u = S(:, j) - V F(j, :)^T for the row block's 128 rows (4 per lane)
    // with the same fp16 hi / lo operands the tensor-core formation uses (3 FMAs per
    // pending reflector), masked to rows >= j, rounded to the storage format on store
    // steps; published to shared memory (the epilogue's w = X^T u) and to U (the next
    // steps' V operand).
    const uint32_t fbytes = (uint32_t)(kch * 2 * CH_BYTES);
    auto issue_v = [&](int rbi) {
      const int vb = rbi % NVB;
      if (rbi >= NVB) mbar_wait(&vempty[vb], (uint32_t)(((rbi - NVB) / NVB) & 1));   // MMAs done with rbi - NVB
      unsigned char* vbuf = smem + geo.v0 + vb * geo.vsz;
      if (elect_one()) {
        mbar_expect_tx(&vfull[vb], fbytes + RG_B * 16);
        if (kch > 0) tma_load(vbuf, p.Vop + (size_t)(p.rb_first + rb0 + rbi) * kchw * 2 * CH_BYTES, fbytes, &vfull[vb]);
        tma_load_2d(vbuf + geo.pcol, &tmC, j * 2, (int)((p.rb_first + rb0 + rbi) * RG_B), &vfull[vb]);
      }
      __syncwarp();
    };
    if (nrbc > 0) issue_v(0);
    if (nrbc > 1) issue_v(1);
    for (int rbi = 0; rbi < nrbc; ++rbi) {
      const int vb = rbi % NVB, ub = rbi & 1;
      const int64_t r0 = (p.rb_first + rb0 + rbi) * R_B;
      mbar_wait(&vfull[vb], (uint32_t)((rbi / NVB) & 1));
      if (rbi >= 2) mbar_wait(&ufree[ub], (uint32_t)(((rbi - 2) >> 1) & 1));
      const unsigned char* vbuf = smem + geo.v0 + vb * geo.vsz;
      const __half* pc = reinterpret_cast<const __half*>(vbuf + geo.pcol);   // [16 groups][8 rows]
      float x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) x[i] = __half2float(pc[lane * 4 + i]);
      for (int l0 = 0; l0 < npend; l0 += 8) {
        const unsigned char* vc = vbuf + (size_t)(l0 >> 4) * 2 * CH_BYTES;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = op_off(lane * 4 + i, l0 & 15);             // 8 consecutive l: 16 B
          const uint4 hv = *reinterpret_cast<const uint4*>(vc + o);
          const uint4 lv = *reinterpret_cast<const uint4*>(vc + CH_BYTES + o);
          const __half* hh = reinterpret_cast<const __half*>(&hv);
          const __half* ll = reinterpret_cast<const __half*>(&lv);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (l0 + q < npend) {
              const float vh = __half2float(hh[q]), vl = __half2float(ll[q]);
              const float fh = fj[l0 + q], fl = fj[32 + l0 + q];
              x[i] = fmaf(fh, vh, x[i]);
              x[i] = fmaf(fh, vl, x[i]);
              x[i] = fmaf(fl, vh, x[i]);
            }
          }
        }
      }
      float* uu = ubuf + ub * R_B;
      // u_j also becomes column lnext of the V operand the next steps read (the Householder
      // vector v_j = c_j u_j, with c_j folded into the F operand by k_reflector): fp16 hi / lo
      unsigned char* vg = p.Vop + (size_t)(p.rb_first + rb0 + rbi) * kchw * 2 * CH_BYTES +
                          (size_t)(p.lnext >> 4) * 2 * CH_BYTES;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t rl = r0 + lane * 4 + i;
        float v = p.store ? __half2float(__float2half_rn(x[i])) : x[i];
        if (rl < jl) v = 0.f;
        uu[lane * 4 + i] = v;
        __half hi, lo;
        split_f16(v, hi, lo);
        const int o = op_off(lane * 4 + i, p.lnext & 15);
        *reinterpret_cast<__half*>(vg + o) = hi;
        *reinterpret_cast<__half*>(vg + CH_BYTES + o) = lo;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ufull[ub]);
      // the load two blocks ahead: with 2 buffers into this block's own buffer (it waits for the
      // MMAs of block rbi, so u of block rbi + 1 is formed only after them and the epilogue
      // idles at every row-block boundary); with 3 into the buffer of block rbi - 1
      if (rbi + 2 < nrbc) issue_v(rbi + 2);
    }
  } else if (warp >= 2 && warp < 2 + EPI_WARPS) {
    // ============================ epilogue ============================
    const int e = warp - 2;
    const int grp = e / EPI_GW;                 // tiles t = grp, grp + 2, ...
    const int hf = (e >> 2) & 1;                // rows [64 hf, 64 hf + 64) of a unit
    const int q = warp & 3;                     // TMEM lane quarter (hardware: warp % 4)
    for (int rbi = 0; rbi < nrbc; ++rbi) {
      const int64_t r0 = (p.rb_first + rb0 + rbi) * R_B;   // first local row of the block
      const bool mask = jl > r0;                           // rows < j inside this block
      const bool hasj = jl >= r0 && jl < r0 + R_B;
      const int ub = rbi & 1;
      const float* uu = ubuf + ub * R_B;
      mbar_wait(&ufull[ub], (uint32_t)((rbi >> 1) & 1));
      // plain units (no store, no rows above the pivot row, not the pivot row's block — all but
      // one row block of one CTA on 94 % of the launches) take a branch-free, fully unrolled path
      const bool plain = !p.store && !mask && !hasj;
      const float* uh = uu + 64 * hf;                     // this warp's 64 rows of u
      int ti = 0;
      for (int t = grp; t < ntiles; t += NGRP, ++ti) {
        const int u = rbi * ntiles + t;                   // units per CTA < 2^31 (m_pad / 128 x 16)
        const int acc = u & (NACC - 1);
        mbar_wait(&tfull[acc], (uint32_t)((u / NACC) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int col = t * C_T + q * 32 + lane;          // column offset from j
        // this unit's 64-row sums: 4 packed fp32 accumulator pairs (8 chains of 8 rows),
        // folded pairwise in fp32 and added to the fp64 column sums once per unit
        float2 w4[4], s4[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) { w4[a] = make_float2(0.f, 0.f); s4[a] = w4[a]; }
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * R_B + 64 * hf);
        auto fma16 = [&](const float* x, const float* u16) {
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 u4 = *reinterpret_cast<const float4*>(u16 + i);
            const float2 xa = make_float2(x[i], x[i + 1]);
            const float2 xb = make_float2(x[i + 2], x[i + 3]);
            const int a = (i >> 2) & 1;
            w4[a] = __ffma2_rn(xa, make_float2(u4.x, u4.y), w4[a]);
            s4[a] = __ffma2_rn(xa, xa, s4[a]);
            w4[a + 2] = __ffma2_rn(xb, make_float2(u4.z, u4.w), w4[a + 2]);
            s4[a + 2] = __ffma2_rn(xb, xb, s4[a + 2]);
          }
        };
        int slot = 0;
        if (plain) {
#pragma unroll
          for (int ci = 0; ci < 4; ++ci) {                  // 16-row chunks of this warp's 64 rows
            float x[16];
            tmem_ld16(tbase + (uint32_t)(ci * 16), x);
            fma16(x, uh + ci * 16);
          }
        } else {
        slot = u % NST;
#pragma unroll 1
        for (int cb = 4 * hf; cb < 4 * hf + 4; ++cb) {      // 16-row chunks of this warp's 64 rows
          float x[16];
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * R_B + cb * 16), x);
          if (p.store) {
            // round to the storage format and write the 2 row groups of this chunk back
            // into the S tile (the producer stores the tile once the group is done)
            unsigned char* tile = smem + (size_t)slot * geo.slot;
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              uint4 v;
              __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                h[i] = __floats2half2_rn(x[g * 8 + 2 * i], x[g * 8 + 2 * i + 1]);
                const float2 f = __half22float2(h[i]);
                x[g * 8 + 2 * i] = f.x;
                x[g * 8 + 2 * i + 1] = f.y;
              }
              *reinterpret_cast<uint4*>(tile + (cb * 2 + g) * 2048 + (q * 32 + lane) * 16) = v;
            }
          }
          if (hasj) {                                      // the owner's row j of X
            const int rj = (int)(jl - r0) - cb * 16;
            if (rj >= 0 && rj < 16) {
              float xj = x[0];
#pragma unroll
              for (int i = 1; i < 16; ++i) xj = i == rj ? x[i] : xj;
              if (j + col < n) p.xr[j + col] = (double)xj;
            }
          }
          if (mask) {
            const int nz = (int)(jl - r0) - cb * 16;       // rows of this chunk above the pivot row
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < nz) x[i] = 0.f;
          }
          fma16(x, uu + cb * 16);
        }
        }
        const float2 wp = __fadd2_rn(__fadd2_rn(w4[0], w4[1]), __fadd2_rn(w4[2], w4[3]));
        const float2 sp = __fadd2_rn(__fadd2_rn(s4[0], s4[1]), __fadd2_rn(s4[2], s4[3]));
        double uw = (double)(wp.x + wp.y), us = (double)(sp.x + sp.y);
#pragma unroll
        for (int z = 0; z < TPG; ++z)
          if (z == ti) { aw[z] += uw; as[z] += us; }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (p.store) {
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ufree[ub]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();   // every role is done: the smem ring (and its async stores) is idle
  // the CTA's column partials: the two row halves of each column added in fixed order
  // (half 0 + half 1) through shared memory, one partials row per CTA
  {
    const int e = warp - 2;
    const bool epi = warp >= 2 && warp < 2 + EPI_WARPS;
    const int grp = e / EPI_GW, hf = (e >> 2) & 1, q = warp & 3;
    double* red = reinterpret_cast<double*>(smem);          // [NGRP][TPG][128][2]
    if (epi && hf == 1) {
      int ti = 0;
      for (int t = grp; t < ntiles; t += NGRP, ++ti) {
        double w = 0.0, s2 = 0.0;
#pragma unroll
        for (int z = 0; z < TPG; ++z)
          if (z == ti) { w = aw[z]; s2 = as[z]; }
        double* r = red + (((size_t)grp * TPG + ti) * C_T + q * 32 + lane) * 2;
        r[0] = w;
        r[1] = s2;
      }
    }
    __syncthreads();
    if (epi && hf == 0) {
      int ti = 0;
      for (int t = grp; t < ntiles; t += NGRP, ++ti) {
        const int c = j + t * C_T + q * 32 + lane;
        double w = 0.0, s2 = 0.0;
#pragma unroll
        for (int z = 0; z < TPG; ++z)
          if (z == ti) { w = aw[z]; s2 = as[z]; }
        const double* r = red + (((size_t)grp * TPG + ti) * C_T + q * 32 + lane) * 2;
        if (c < n) {
          p.part[((int64_t)blockIdx.x * 2 + 0) * n + c] = w + r[0];
          p.part[((int64_t)blockIdx.x * 2 + 1) * n + c] = s2 + r[1];
        }
      }
    }
  }
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---------------------------------------------------------------------------
int tc_kchw(int nb) { return (nb + 15) / 16; }

size_t tc_vop_bytes(int64_t m_pad, int nb) { return (size_t)(m_pad / 128 + 1) * tc_kchw(nb) * 2 * CH_BYTES; }
size_t tc_fop_bytes(int n, int nb) { return (size_t)((n + C_T - 1) / C_T) * tc_kchw(nb) * 2 * CH_BYTES; }

int tc_smem_bytes(int nb, int nvb, int* nst_out) {
  const int kchw = tc_kchw(nb);
  // ring depth 4 (40 KB slots at nb <= 16); 5 fits but measured < 1 ms better per C4 QRCP and,
  // being odd, forces one MMA issuer (MPID_TC_NST: A/B measurements)
  static const int nst_env = getenv("MPID_TC_NST") ? atoi(getenv("MPID_TC_NST")) : 4;
  int nst = nst_env < 2 ? 2 : (nst_env > 6 ? 6 : nst_env);
  while (nst > 2 && geo_of(kchw, nst, nvb).total > TC_SMEM_MAX) --nst;
  if (nst_out) *nst_out = nst;
  return geo_of(kchw, nst, nvb).total;
}

cudaError_t launch_pass_tc(const PassParams& pp, int nb, void* Vop, const void* Fop, const void* tmap,
                           const void* tmapc, int max_ctas, int* gx_out, cudaStream_t st) {
  TcParams p{};
  p.m_pad = pp.m_pad;
  p.m_local = pp.m_local;
  p.row_offset = pp.row_offset;
  p.rb_first = pp.g_lo / RG_B;
  p.nrb = pp.m_pad / R_B - p.rb_first;
  if (p.nrb < 0) p.nrb = 0;
  p.n = pp.n;
  p.j = pp.j;
  p.j0 = pp.j0;
  p.npend = pp.npend;
  p.store = pp.store;
  p.kchw = tc_kchw(nb);
  p.ntiles = (pp.n - pp.j + C_T - 1) / C_T;
  if (p.npend > p.kchw * 16 || p.kchw > 2 || p.ntiles > 16) return cudaErrorInvalidValue;
  static const int nvb_env = getenv("MPID_TC_NVB") ? atoi(getenv("MPID_TC_NVB")) : 3;   // A/B measurements
  p.nvb = nvb_env == 2 ? 2 : NVB_MAX;
  if (p.nvb == 3 && geo_of(p.kchw, 4, 3).total > TC_SMEM_MAX) p.nvb = 2;   // keep the 4-deep ring (nb > 16)
  int nst = 0;
  const int smem = tc_smem_bytes(nb, p.nvb, &nst);
  // Two issuers split the tiles by parity.  A ring slot (u % nst) and an accumulator (u % 4) must
  // keep ONE issuer warp and ONE epilogue group over their successive uses — an mbarrier parity
  // wait cannot tell phase k from k + 2, and only a single in-order issuer guarantees that use
  // k has completed before anyone waits for use k + 1 — which holds when tile parity = unit
  // parity: an even ring depth AND an even tile count.  Otherwise one issuer takes all tiles.
  static const int nmma_env = getenv("MPID_TC_NMMA") ? atoi(getenv("MPID_TC_NMMA")) : 0;   // A/B measurements
  p.nmma = ((nst & 1) || (p.ntiles & 1)) ? 1 : (nmma_env == 1 ? 1 : 2);
  if (smem > TC_SMEM_MAX) return cudaErrorInvalidConfiguration;
  p.nst = nst;
  p.Vop = (unsigned char*)Vop;
  p.lnext = pp.j % nb;
  p.Fop = (const unsigned char*)Fop;
  p.U = (float*)pp.U;
  p.part = pp.part;
  p.xr = pp.xr;
  p.sc = pp.sc;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(max_ctas / 2, p.nrb));
  *gx_out = gx;
  const bool wide = p.ntiles > 2 * 4;
  const void* fn = wide ? (const void*)k_pass_tc<8> : (const void*)k_pass_tc<4>;
  cudaError_t e = smem_attr(fn, smem);
  if (e != cudaSuccess) return e;
  if (wide)
    k_pass_tc<8><<<gx, BLOCK, smem, st>>>(p, *reinterpret_cast<const CUtensorMap*>(tmap),
                                          *reinterpret_cast<const CUtensorMap*>(tmapc));
  else
    k_pass_tc<4><<<gx, BLOCK, smem, st>>>(p, *reinterpret_cast<const CUtensorMap*>(tmap),
                                          *reinterpret_cast<const CUtensorMap*>(tmapc));
  return cudaGetLastError();
}

// tensor maps of fp16 S viewed as [ngroups][n * 2] 8-byte units: box = 128 columns x 16 row
// groups (one unit tile, 32 KB; which = 0) or 1 column x 16 row groups (the pivot column of a
// row block, 256 B; which = 1); the driver entry point is taken through the runtime
int encode_tmap_S(void* tmap_out, void* S, int64_t ngroups, int n, int which) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return -1;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)n * 2, (cuuint64_t)ngroups};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 16};
  const cuuint32_t box[2] = {(cuuint32_t)(which ? 2 : C_T * 2), (cuuint32_t)RG_B};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, S, dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return (int)r;
}

}  // namespace mpid
