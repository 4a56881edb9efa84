// k_pass_tc — the per-step panel pass with the pending trailing update formed on
// the 5th-generation tensor cores (tcgen05 + TMEM), the "D-OTF" design of
// Ã = S − V Fᵀ is formed tile by tile as a rank-npend GEMM
// (npend ≤ nb ≤ 32 pending reflectors of the current panel) whose fp32
// accumulator lives in TMEM and is never written to HBM; the epilogue computes the
// u-weighted and squared column sums from it, and at the panel end (store steps)
// writes fl_L(Ã) back — the blocked trailing-matrix update of Algorithm 2 line 4
// as a tensor-core GEMM with K = nb.
//
// Operands (kind::tf32, fp32-accurate "3xTF32": V = Vh + Vl, F = Fh + Fl,
// D = Fh·Vhᵀ + Fh·Vlᵀ + Fl·Vhᵀ, within ~2^-21 of the exact product — DESIGN.md R14):
//   A = F tile  (M = 128 lanes: 124 matrix columns of this CTA + the pivot column j
//               in lanes 0, 32, 64, 96, × K), built once per launch in shared memory;
//   B = V block (N = 128 matrix rows × K), the panel's v vectors, kept in global
//               memory by k_vop in exactly the smem operand layout, so one bulk copy
//               per stage brings the tile in.
// Both K-major, no-swizzle core-matrix layout (8 rows × 16 B per core matrix;
// LBO = K-direction core stride = 128 B, SBO = 8-row stride).  D[col][row] sits in
// TMEM with lane = matrix column and TMEM column = matrix row: the epilogue thread
// of a column reads 8 consecutive rows with one tcgen05.ld.32x32b.x8 and the
// matching 16-byte chunk of the interleaved S layout with one LDS.128.  Every
// warp holds the pivot column's D values in its lane 0 and forms u = Ã(:, j) for
// its own rows through a per-warp shared scratch — no cross-warp barrier per stage.
//
// One CTA per SM, 18 warps: w0 TMA producer, w1 MMA issuer (+ TMEM allocator),
// w2-17 epilogue (warp w reads TMEM lanes 32·(w%4).., rows 32·((w-2)/4).. of a stage).
// Pipelines: smem ring full → (MMA → tmem_full) → epilogue → empty, and a
// double-buffered TMEM accumulator (tmem_full / tmem_empty).
#include "mpid_internal.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace mpid {

namespace {
constexpr int TC_LANES = 128;    // MMA M = TMEM lanes
constexpr int TC_CN = 124;       // matrix columns per CTA (lanes 0, 32, 64, 96 = the pivot column)
constexpr int TC_R = 128;        // matrix rows per stage = MMA N
constexpr int TC_RG = TC_R / 8;  // row groups per stage
constexpr int TC_EPI_WARPS = 16;
constexpr int TC_BLOCK = 32 * (2 + TC_EPI_WARPS);
constexpr int TC_NACC = 2;         // TMEM accumulator ring depth
constexpr int TC_TMEM_COLS = 128 * TC_NACC;  // accumulators of 128 fp32 columns

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version; base offset 0, SWIZZLE_NONE
  return d;
}
// kind::tf32, fp32 accumulate, K-major A and B, N = 128, M = 128
__device__ __forceinline__ uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_R >> 3) << 17) | ((uint32_t)(TC_LANES >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc_tf32()), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
// 32 consecutive TMEM columns (= matrix rows) of this warp's 32 lanes -> v[0..31]; no wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 2-D tensor-map TMA of S viewed as [ngroups][n * esz] 8-byte elements: one box row is a
// whole row group of TC_CN columns (contiguous 16 B chunks), so the copy engine moves
// ~2 KB runs; box {TC_CN * esz / 8 * 8 ... } -- see encode_tmap_S
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
// tf32 split: hi = RN to 10 mantissa bits, lo = x - hi (exact in fp32)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}
// byte offset of element (row r, k) in a K-major fp32 core-matrix tile (sbo = bytes per 8 rows)
__host__ __device__ __forceinline__ int64_t cm_off(int64_t r, int k, int sbo) {
  return (r >> 3) * sbo + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}

template <typename T> struct Ch;
template <> struct Ch<__half> {
  __device__ static __forceinline__ void load(const __half* p, float* x) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(h[i]);
      x[2 * i] = f.x;
      x[2 * i + 1] = f.y;
    }
  }
  __device__ static __forceinline__ void round_store(__half* p, float* x) {
    uint4 v;
    __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
      const float2 f = __half22float2(h[i]);
      x[2 * i] = f.x;
      x[2 * i + 1] = f.y;
    }
    *reinterpret_cast<uint4*>(p) = v;
  }
  __device__ static __forceinline__ float rnd(float a) { return __half2float(__float2half_rn(a)); }
  __device__ static __forceinline__ float get(const __half* p, int i) { return __half2float(p[i]); }
};
template <> struct Ch<float> {
  __device__ static __forceinline__ void load(const float* p, float* x) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
  __device__ static __forceinline__ void round_store(float* p, float* x) {
    reinterpret_cast<float4*>(p)[0] = make_float4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(x[4], x[5], x[6], x[7]);
  }
  __device__ static __forceinline__ float rnd(float a) { return a; }
  __device__ static __forceinline__ float get(const float* p, int i) { return p[i]; }
};

struct TcGeom {
  int a_hi, a_lo;                 // F tile (hi, lo): 128 lanes x nbw fp32 each
  int slot0, slot;                // first slot, slot stride
  int data, ucol, vh, vl, us;     // offsets inside a slot
  int red;                        // 2 x 128 x 2 doubles
  int bars;                       // mbarriers
  int total;
};
__host__ __device__ inline int a128(int x) { return (x + 127) & ~127; }
__host__ __device__ inline TcGeom tc_geom(int esz, int nbw, int nst) {
  TcGeom g;
  g.a_hi = 0;
  g.a_lo = a128(TC_LANES * nbw * 4);
  g.slot0 = g.a_lo + a128(TC_LANES * nbw * 4);
  g.data = 0;
  g.ucol = a128(TC_RG * TC_CN * 8 * esz);
  g.vh = g.ucol + a128(TC_RG * 8 * esz);
  g.vl = g.vh + TC_R * nbw * 4;
  g.us = g.vl + TC_R * nbw * 4;
  g.slot = a128(g.us + TC_R * 4);
  g.red = g.slot0 + nst * g.slot;
  g.bars = g.red + 4 * TC_LANES * 2 * 8 + TC_EPI_WARPS * 32 * 4;   // + per-warp u scratch
  g.total = g.bars + (2 * nst + 2 * TC_NACC) * 8 + 16;
  return g;
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(TC_BLOCK, 1) k_pass_tc(PassParams p, const __grid_constant__ CUtensorMap tmS) {
  if (p.sc->done) return;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int n = p.n, j = p.j, npend = p.npend;
  const int nbw = p.nbw;                      // K width of the operand layouts (multiple of 8)
  const int kchunks = (npend + 7) / 8;
  const int NST = p.nst;
  const int esz = (int)sizeof(T);
  const int sbo = nbw * 32;                   // bytes per 8 rows of a K-major tile: (nbw / 4) * 128
  T* __restrict__ S = reinterpret_cast<T*>(p.S);
  const int c_lo = j + TC_CN * blockIdx.y;
  const int ncols = min(TC_CN, n - c_lo);
  const TcGeom geo = tc_geom(esz, nbw, NST);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + geo.bars);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + TC_NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + TC_NACC);
  // row groups of this CTA
  const int64_t g_lo = p.g_lo;
  const int64_t nact = p.ngroups - g_lo;
  // whole stages per CTA (the tensor-map stores write full boxes: a box must never
  // reach into the next CTA's rows); only the last CTA ends inside a stage
  const int64_t per = ((nact + gridDim.x - 1) / gridDim.x + TC_RG - 1) / TC_RG * TC_RG;
  const int64_t gb = g_lo + (int64_t)blockIdx.x * per;
  const int64_t ge = (gb + per < p.ngroups) ? gb + per : p.ngroups;
  const int nst = gb < ge ? (int)((ge - gb + TC_RG - 1) / TC_RG) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---------------- setup: barriers, TMEM, the F (A operand) tile ----------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TC_EPI_WARPS);
    }
    for (int a = 0; a < TC_NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], TC_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp >= 2 && kchunks > 0) {
    // A operand: lane i = the pivot column j when i % 32 == 0, else CTA column
    // (i / 32) * 31 + i % 32 - 1; k = pending step l; hi/lo tf32 split of f_l(column)
    const int t = threadIdx.x - 64;
    const int kw = kchunks * 8;
    for (int e = t; e < TC_LANES * kw; e += 32 * TC_EPI_WARPS) {
      const int i = e / kw, l = e - i * kw;
      const int ci = (i >> 5) * 31 + (i & 31) - 1;
      float f = 0.f;
      if (l < npend) {
        if ((i & 31) == 0) f = reinterpret_cast<const float*>(p.F)[(int64_t)((p.j0 + l) % NSLOT) * n + j];
        else if (ci < ncols) f = reinterpret_cast<const float*>(p.F)[(int64_t)((p.j0 + l) % NSLOT) * n + c_lo + ci];
      }
      float hi, lo;
      split_tf32(f, hi, lo);
      *reinterpret_cast<float*>(smem + geo.a_hi + cm_off(i, l, sbo)) = hi;
      *reinterpret_cast<float*>(smem + geo.a_lo + cm_off(i, l, sbo)) = lo;
    }
    fence_async_smem();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      const int64_t ngroups = p.ngroups;
      // the box is {TC_CN * u8 8-byte units, TC_RG row groups} for fp16 (u8 = 2); fp32 chunks are
      // 32 B (u8 = 4), so its stage is two boxes of TC_CN / 2 columns.  The smem tile is then
      // [box][row group][columns][8 rows]; the epilogue addresses it accordingly.
      const int u8 = esz;                                 // 8-byte units per 8-row chunk
      const int nbox = esz == 2 ? 1 : 2;
      const int bcols = TC_CN / (esz == 2 ? 1 : 2);
      auto issue_store = [&](int i, int slot) {   // whole boxes; out-of-range rows/columns are not written
        const int64_t g0 = gb + (int64_t)i * TC_RG;
        unsigned char* d = smem + geo.slot0 + (size_t)slot * geo.slot + geo.data;
        for (int b = 0; b < (esz == 2 ? 1 : 2); ++b)
          tma_store_2d(&tmS, (c_lo + b * bcols) * u8, (int)g0, d + (size_t)b * TC_RG * bcols * 8 * esz);
      };
      (void)nbox;
      const uint32_t vbytes = (uint32_t)(TC_RG * sbo);    // one stage of the V operand (hi or lo)
      const uint32_t dbytes = (uint32_t)(TC_RG * TC_CN * 8 * esz);   // one stage of S (full box)
      const T* Sj = reinterpret_cast<const T*>(p.Sj);
      int slot = 0;
      uint32_t phase = 0;
      for (int i = 0; i < nst; ++i) {
        if (i >= NST) {
          mbar_wait(&empty[slot], phase ^ 1);
          if (p.store) {
            issue_store(i - NST, slot);
            bulk_commit();
            bulk_wait_read0();
          }
        }
        const int64_t g0 = gb + (int64_t)i * TC_RG;
        const int gsz = (int)((ge - g0) < TC_RG ? (ge - g0) : TC_RG);
        unsigned char* base = smem + geo.slot0 + (size_t)slot * geo.slot;
        mbar_expect_tx(&full[slot], dbytes + (uint32_t)(gsz * 8 * esz) + (kchunks > 0 ? 2 * vbytes : 0));
        for (int b = 0; b < (esz == 2 ? 1 : 2); ++b)
          tma_load_2d(base + geo.data + (size_t)b * TC_RG * bcols * 8 * esz, &tmS, (c_lo + b * bcols) * u8, (int)g0,
                      &full[slot]);
        tma_load(base + geo.ucol, Sj + g0 * 8, (uint32_t)(gsz * 8 * esz), &full[slot]);
        if (kchunks > 0) {   // V operand rows g0*8 .. g0*8+127 (the buffer is padded to whole stages)
          tma_load(base + geo.vh, reinterpret_cast<const unsigned char*>(p.Vh) + g0 * sbo, vbytes, &full[slot]);
          tma_load(base + geo.vl, reinterpret_cast<const unsigned char*>(p.Vl) + g0 * sbo, vbytes, &full[slot]);
        }
        if (++slot == NST) { slot = 0; phase ^= 1; }
      }
      (void)ngroups;
      if (p.store) {
        for (int i = max(0, nst - NST); i < nst; ++i) {
          const int s2 = i % NST;
          mbar_wait(&empty[s2], (uint32_t)((i / NST) & 1));
          issue_store(i, s2);
        }
        bulk_commit();
      }
      bulk_wait0();
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (one thread) =======================
    if (lane == 0) {
      int slot = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      const uint32_t ahi = su32(smem + geo.a_hi), alo = su32(smem + geo.a_lo);
      for (int i = 0; i < nst; ++i) {
        mbar_wait(&full[slot], phase);
        mbar_wait(&tempty[acc], aphase ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (kchunks > 0) {
          const uint32_t sbase = su32(smem + geo.slot0 + (size_t)slot * geo.slot);
          const uint32_t d = tmem + (uint32_t)(acc * TC_R);
          for (int kc = 0; kc < kchunks; ++kc) {
            const uint32_t ko = (uint32_t)(kc * 2 * 128);   // 8 tf32 = 2 core matrices along K
            const uint64_t dah = sdesc(ahi + ko, 128, sbo), dal = sdesc(alo + ko, 128, sbo);
            const uint64_t dbh = sdesc(sbase + geo.vh + ko, 128, sbo), dbl = sdesc(sbase + geo.vl + ko, 128, sbo);
            mma_tf32(d, dah, dbh, kc > 0 ? 1u : 0u);
            mma_tf32(d, dah, dbl, 1u);
            mma_tf32(d, dal, dbh, 1u);
          }
          mma_commit(&tfull[acc]);
        } else {
          mbar_arrive(&tfull[acc]);
        }
        if (++slot == NST) { slot = 0; phase ^= 1; }
        if (++acc == TC_NACC) { acc = 0; aphase ^= 1; }
      }
    }
  } else {
    // ======================= epilogue (16 warps) =======================
    // warp w: TMEM lane quarter w % 4, rows [32 rp, 32 rp + 32) of every stage (rp = (w-2)/4)
    const int quarter = warp & 3, rp = (warp - 2) >> 2, ew = warp - 2;
    const int lanei = quarter * 32 + lane;                  // TMEM lane = A-operand row
    const int ci = quarter * 31 + lane - 1;                 // CTA column of this lane (lane > 0)
    const bool ulane = lane == 0;                           // lane 0 holds the pivot column
    const bool valid = !ulane && ci < ncols;
    const int ccol = valid ? ci : 0;
    float* uw = reinterpret_cast<float*>(smem + geo.red + 4 * TC_LANES * 2 * 8) + ew * 32;  // u of my 32 rows
    const int64_t jloc = (int64_t)j - p.row_offset;
    const int64_t gj = (jloc >= 0 && jloc < p.m_local) ? (jloc >> 3) : -1;
    const int jr = (int)(jloc & 7);
    float* __restrict__ Uj = reinterpret_cast<float*>(p.U) + (int64_t)(j % NSLOT) * p.m_pad;
    double aw = 0.0, as = 0.0;
    int slot = 0, acc = 0;
    uint32_t phase = 0, aphase = 0;
    for (int i = 0; i < nst; ++i) {
      const int64_t g0 = gb + (int64_t)i * TC_RG;
      const int gsz = (int)((ge - g0) < TC_RG ? (ge - g0) : TC_RG);
      const int gjs = (gj >= g0 && gj < g0 + gsz) ? (int)(gj - g0) : -1;
      unsigned char* base = smem + geo.slot0 + (size_t)slot * geo.slot;
      T* data = reinterpret_cast<T*>(base + geo.data);
      const T* ucol = reinterpret_cast<const T*>(base + geo.ucol);
      mbar_wait(&tfull[acc], aphase);
      mbar_wait(&full[slot], phase);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t dr[32];
      if (kchunks > 0) {
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * TC_R + rp * 32), dr);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) dr[q] = 0u;
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);            // accumulator is in registers
      // u = Ã(:, j) for my 32 rows: lane 0 parks the pivot column's D values, then
      // every lane forms one row
      if (ulane) {
#pragma unroll
        for (int q = 0; q < 32; q += 4)
          *reinterpret_cast<uint4*>(uw + q) = make_uint4(dr[q], dr[q + 1], dr[q + 2], dr[q + 3]);
      }
      __syncwarp();
      {
        const int rb = rp * 32 + lane;                        // stage row
        float u = 0.f;
        if ((rb >> 3) < gsz) {
          u = Ch<T>::get(ucol, rb) - uw[lane];
          if (p.store) u = Ch<T>::rnd(u);
          const int64_t rl = g0 * 8 + rb;
          const bool keep = rl < p.m_local && p.row_offset + rl >= j;
          u = keep ? u : 0.f;
          if (blockIdx.y == 0 && quarter == 0) Uj[rl] = u;
        }
        uw[lane] = u;
      }
      __syncwarp();
      // form, (round + write back), reduce: 4 row groups of 8
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        const int gl = rp * 4 + gg;
        if (gl < gsz) {                                       // warp-uniform
          T* chunk;
          if (sizeof(T) == 2) chunk = data + (size_t)(gl * TC_CN + ccol) * 8;
          else {
            const int bc = TC_CN / 2, b = ccol / bc;
            chunk = data + ((size_t)b * TC_RG * bc + (size_t)gl * bc + (ccol - b * bc)) * 8;
          }
          float x[8];
          Ch<T>::load(chunk, x);
          float2* x2 = reinterpret_cast<float2*>(x);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            x2[q] = __fadd2_rn(x2[q], make_float2(-__uint_as_float(dr[gg * 8 + 2 * q]),
                                                  -__uint_as_float(dr[gg * 8 + 2 * q + 1])));
          if (p.store) {
            if (valid) Ch<T>::round_store(chunk, x);
            else {
#pragma unroll
              for (int q = 0; q < 8; ++q) x[q] = Ch<T>::rnd(x[q]);
            }
          }
          if (gl == gjs) {                                   // the group holding row j
            float xj = x[0];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (q == jr) xj = x[q];
              if (q < jr) x[q] = 0.f;
            }
            if (valid) p.xr[c_lo + ci] = xj;
          }
          // 8-row group: even-row and odd-row fp32 chains in one packed FFMA2 each
          // (R5b), then their fp32 sum into the fp64 column accumulators
          const float4 ua = *reinterpret_cast<const float4*>(uw + gg * 8);
          const float4 ub = *reinterpret_cast<const float4*>(uw + gg * 8 + 4);
          const float2 u2[4] = {make_float2(ua.x, ua.y), make_float2(ua.z, ua.w), make_float2(ub.x, ub.y),
                                make_float2(ub.z, ub.w)};
          float2 w2 = __fmul2_rn(x2[0], u2[0]), s2 = __fmul2_rn(x2[0], x2[0]);
#pragma unroll
          for (int q = 1; q < 4; ++q) {
            w2 = __ffma2_rn(x2[q], u2[q], w2);
            s2 = __ffma2_rn(x2[q], x2[q], s2);
          }
          const float pw = w2.x + w2.y, ps = s2.x + s2.y;
          aw += (double)pw;
          as += (double)ps;
        }
      }
      if (p.store) fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == NST) { slot = 0; phase ^= 1; }
      if (++acc == TC_NACC) { acc = 0; aphase ^= 1; }
    }
    // combine the four row parts in fixed order and write the CTA's partials
    double* red = reinterpret_cast<double*>(smem + geo.red);
    red[(rp * TC_LANES + lanei) * 2 + 0] = aw;
    red[(rp * TC_LANES + lanei) * 2 + 1] = as;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * TC_EPI_WARPS) : "memory");
    if (rp == 0 && valid) {
      double w = 0.0, s2 = 0.0;
#pragma unroll
      for (int r4 = 0; r4 < 4; ++r4) {
        w += red[(r4 * TC_LANES + lanei) * 2 + 0];
        s2 += red[(r4 * TC_LANES + lanei) * 2 + 1];
      }
      p.part[((int64_t)blockIdx.x * 2 + 0) * n + c_lo + ci] = w;
      p.part[((int64_t)blockIdx.x * 2 + 1) * n + c_lo + ci] = s2;
    }
  }
  // ---------------- teardown ----------------
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
}

// ---------------------------------------------------------------------------
// k_vop: the newest pending Householder vector v_t = fl32(u_t c_t) (v_t(t) = 1,
// zero above row t and on padding rows), split hi/lo for tf32, written as column
// k = t - j0 of the panel's V operand in the K-major core-matrix layout.
__global__ void k_vop(const float* __restrict__ U, int64_t m_pad, int64_t m_local, int64_t row_offset,
                      int t, int k, const double* __restrict__ cvec, float* __restrict__ Vh,
                      float* __restrict__ Vl, int sbo, const DevScalars* __restrict__ sc) {
  if (sc->done) return;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m_pad) return;
  const int64_t rg = row_offset + r;
  float v = 0.f;
  if (r < m_local) {
    if (rg == t) v = 1.f;
    else if (rg > t) v = __double2float_rn((double)U[(int64_t)(t % NSLOT) * m_pad + r] * cvec[t]);
  }
  float hi, lo;
  split_tf32(v, hi, lo);
  const int64_t o = cm_off(r, k, sbo) / 4;
  Vh[o] = hi;
  Vl[o] = lo;
}

// ---------------------------------------------------------------------------
template <typename T>
static cudaError_t launch_tc_t(PassParams p, const void* tmap, int max_ctas, int* gx_out, cudaStream_t st) {
  const int n = p.n, j = p.j;
  const int esz = (int)sizeof(T);
  if (p.npend > p.nbw || p.nbw > 32 || (p.nbw % 8)) return cudaErrorInvalidValue;
  const int gy = (n - j + TC_CN - 1) / TC_CN;
  p.ncols_slot = TC_CN;
  int nst = 4;
  TcGeom g = tc_geom(esz, p.nbw, nst);
  while (nst > 2 && (size_t)g.total > (size_t)PASS_SMEM_MAX) {
    --nst;
    g = tc_geom(esz, p.nbw, nst);
  }
  if ((size_t)g.total > (size_t)PASS_SMEM_MAX) return cudaErrorInvalidConfiguration;
  p.nst = nst;
  p.gs = TC_RG;
  const int64_t nact = p.ngroups - p.g_lo;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, max_ctas / gy), (nact + TC_RG - 1) / TC_RG));
  p.gx_used = gx;
  *gx_out = gx;
  cudaError_t e = smem_attr((const void*)k_pass_tc<T>, PASS_SMEM_MAX);
  if (e != cudaSuccess) return e;
  k_pass_tc<T><<<dim3(gx, gy), TC_BLOCK, g.total, st>>>(p, *reinterpret_cast<const CUtensorMap*>(tmap));
  return cudaGetLastError();
}

cudaError_t launch_pass_tc(int fmt, PassParams p, const void* tmap, int max_ctas, int* gx_out, cudaStream_t st) {
  return fmt == 1 ? launch_tc_t<__half>(p, tmap, max_ctas, gx_out, st)
                  : launch_tc_t<float>(p, tmap, max_ctas, gx_out, st);
}

// tensor map of S: 8-byte elements, dims {n * esz / 2 * ... = n * (16 * esz / 2) / 8, ngroups},
// row stride n * 8 * esz bytes, box {(TC_CN or TC_CN / 2 for fp32) * esz / 2, TC_RG}; the
// driver entry point is taken through the runtime (no -lcuda)
int encode_tmap_S(void* tmap_out, void* S, int fmt, int64_t ngroups, int n) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return -1;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const int esz = fmt == 1 ? 2 : 4;
  const int u8 = esz;                              // 8-byte units per 8-row chunk of one column
  const int bcols = fmt == 1 ? TC_CN : TC_CN / 2;  // columns per box (box dim 0 <= 256 units)
  const cuuint64_t dims[2] = {(cuuint64_t)n * u8, (cuuint64_t)ngroups};
  const cuuint64_t strides[1] = {(cuuint64_t)n * 8 * esz};
  const cuuint32_t box[2] = {(cuuint32_t)(bcols * u8), (cuuint32_t)TC_RG};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, S, dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return (int)r;
}

cudaError_t launch_vop(const float* U, int64_t m_pad, int64_t m_local, int64_t row_offset, int t, int k,
                       const double* cvec, float* Vh, float* Vl, int nbw, const DevScalars* sc, cudaStream_t st) {
  k_vop<<<(unsigned)((m_pad + 255) / 256), 256, 0, st>>>(U, m_pad, m_local, row_offset, t, k, cvec, Vh, Vl,
                                                          nbw * 32, sc);
  return cudaGetLastError();
}

}  // namespace mpid
