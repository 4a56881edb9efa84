// k_pass — the per-step panel pass of the low-precision pivoted Householder QR
// (Algorithm 2 line 4; Eq. (6)-(7)), the dominant (HBM-bound) kernel.
//
// What one launch computes for step j (readings R4-R6):
//   A~ = S - sum_{pending l} v_l f_l^T   formed per element in fp32 (FMA, step order)
//   [store steps] A~ <- fl_L(A~), written back to S (the storage rounding point)
//   u = A~(:, j) (rows >= j), w = A~^T u and s_i = ||A~(j:m, i)||^2 with 8-row
//   fp32 FMA chains added in fp64, and the row x = A~(j, :).
//
// B200 structure: one persistent CTA per SM (18 warps, warp-specialised):
//   warp 0      TMA producer: one elected lane streams stages of GS consecutive
//               8-row groups (each row group of the CTA's column range is one
//               contiguous range in the interleaved layout) with cp.async.bulk
//               into an NST-deep shared-memory ring, plus the stage's pivot-column
//               segment and the pending u rows; on store steps it writes the
//               rounded stage back with bulk stores once the consumers free it.
//   warp 1      prep: per stage, the pending -v rows (v_t = fl(u_t c_t), v_t(t) = 1)
//               and u = A~(:, j) for the stage's rows (+ u to global for later steps).
//   warps 2-17  consumers: lane owns columns (c, c + 32) of its warp's 64-column
//               block, so every FFMA2 works on a natural (col0, col1) register
//               pair: update x2 += (-v_r) * f2, then w2 += x2 * u_r, s2 += x2 * x2.
// mbarriers: full (TMA tx) -> prep (32 arrivals) -> consumers -> empty (NCW arrivals).
// Bound: HBM.  Per element: 1 cvt + npend/2 + 1 FFMA2-equivalents on the FMA pipe.
//
// The same kernel runs the double ID's fp64 QRCP (Â_D of P:196; Algorithm 1):
// T = double, every working quantity (u, v, f, the formed A~) in fp64, and each
// product-then-add as a separately rounded DMUL + DADD (the oracle's fp64 model, reading
// R16); the interleaved layout and the pipeline are unchanged, with 4x the bytes.
#include "mpid_internal.cuh"
#include <cstdlib>

namespace mpid {

namespace {
// 8 consecutive rows of one column (one 16 B / 32 B chunk of the interleaved layout)
template <typename T> struct Chunk;
template <> struct Chunk<__half> {
  // a/b: the chunks of column 0 / column 1 -> x[q] = (col0 row q, col1 row q)
  __device__ static __forceinline__ void load2(const __half* a, const __half* b, float2* x) {
    const uint4 va = *reinterpret_cast<const uint4*>(a);
    const uint4 vb = *reinterpret_cast<const uint4*>(b);
    const __half* ha = reinterpret_cast<const __half*>(&va);
    const __half* hb = reinterpret_cast<const __half*>(&vb);
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = make_float2(__half2float(ha[q]), __half2float(hb[q]));
  }
  // round to fp16 (RNE), write back the chunks of the valid columns (wa, wb), and
  // replace x by the rounded values
  __device__ static __forceinline__ void round_store2(__half* a, __half* b, float2* x, bool wa, bool wb) {
    uint4 va, vb;
    __half2* ha = reinterpret_cast<__half2*>(&va);
    __half2* hb = reinterpret_cast<__half2*>(&vb);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ha[q] = __floats2half2_rn(x[2 * q].x, x[2 * q + 1].x);
      hb[q] = __floats2half2_rn(x[2 * q].y, x[2 * q + 1].y);
      const float2 a2 = __half22float2(ha[q]);
      const float2 b2 = __half22float2(hb[q]);
      x[2 * q] = make_float2(a2.x, b2.x);
      x[2 * q + 1] = make_float2(a2.y, b2.y);
    }
    if (wa) *reinterpret_cast<uint4*>(a) = va;
    if (wb) *reinterpret_cast<uint4*>(b) = vb;
  }
  __device__ static __forceinline__ float get(const __half* p, int i) { return __half2float(p[i]); }
  __device__ static __forceinline__ float rnd(float a) { return __half2float(__float2half_rn(a)); }
};
template <> struct Chunk<float> {
  __device__ static __forceinline__ void load2(const float* a, const float* b, float2* x) {
    const float4 a0 = reinterpret_cast<const float4*>(a)[0], a1 = reinterpret_cast<const float4*>(a)[1];
    const float4 b0 = reinterpret_cast<const float4*>(b)[0], b1 = reinterpret_cast<const float4*>(b)[1];
    x[0] = make_float2(a0.x, b0.x); x[1] = make_float2(a0.y, b0.y);
    x[2] = make_float2(a0.z, b0.z); x[3] = make_float2(a0.w, b0.w);
    x[4] = make_float2(a1.x, b1.x); x[5] = make_float2(a1.y, b1.y);
    x[6] = make_float2(a1.z, b1.z); x[7] = make_float2(a1.w, b1.w);
  }
  __device__ static __forceinline__ void round_store2(float* a, float* b, float2* x, bool wa, bool wb) {
    if (wa) {
      reinterpret_cast<float4*>(a)[0] = make_float4(x[0].x, x[1].x, x[2].x, x[3].x);
      reinterpret_cast<float4*>(a)[1] = make_float4(x[4].x, x[5].x, x[6].x, x[7].x);
    }
    if (wb) {
      reinterpret_cast<float4*>(b)[0] = make_float4(x[0].y, x[1].y, x[2].y, x[3].y);
      reinterpret_cast<float4*>(b)[1] = make_float4(x[4].y, x[5].y, x[6].y, x[7].y);
    }
  }
  __device__ static __forceinline__ float get(const float* p, int i) { return p[i]; }
  __device__ static __forceinline__ float rnd(float a) { return a; }
};
template <> struct Chunk<double> {
  __device__ static __forceinline__ void load2(const double* a, const double* b, double2* x) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 va = reinterpret_cast<const double2*>(a)[q], vb = reinterpret_cast<const double2*>(b)[q];
      x[2 * q] = make_double2(va.x, vb.x);
      x[2 * q + 1] = make_double2(va.y, vb.y);
    }
  }
  __device__ static __forceinline__ void round_store2(double* a, double* b, double2* x, bool wa, bool wb) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (wa) reinterpret_cast<double2*>(a)[q] = make_double2(x[2 * q].x, x[2 * q + 1].x);
      if (wb) reinterpret_cast<double2*>(b)[q] = make_double2(x[2 * q].y, x[2 * q + 1].y);
    }
  }
  __device__ static __forceinline__ double get(const double* p, int i) { return p[i]; }
  __device__ static __forceinline__ double rnd(double a) { return a; }
};

// working precision of a storage format: fp32 for fp16/fp32 storage, fp64 for fp64
template <typename T> struct Work { using W = float; using W2 = float2; };
template <> struct Work<double> { using W = double; using W2 = double2; };

__device__ __forceinline__ float2 splat2(float v) { return make_float2(v, v); }
__device__ __forceinline__ double2 splat2(double v) { return make_double2(v, v); }
// x + nv * f, one rounding (FFMA2) in fp32; DMUL then DADD in fp64 (reading R16)
__device__ __forceinline__ float2 upd2(float nv, float2 f, float2 x) { return __ffma2_rn(splat2(nv), f, x); }
__device__ __forceinline__ double2 upd2(double nv, double2 f, double2 x) {
  return make_double2(__dadd_rn(__dmul_rn(nv, f.x), x.x), __dadd_rn(__dmul_rn(nv, f.y), x.y));
}
__device__ __forceinline__ float upd1(float nv, float f, float a) { return fmaf(nv, f, a); }
__device__ __forceinline__ double upd1(double nv, double f, double a) { return __dadd_rn(__dmul_rn(nv, f), a); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ double2 mul2(double2 a, double2 b) {
  return make_double2(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
}
__device__ __forceinline__ float2 mac2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ double2 mac2(double2 a, double2 b, double2 c) {
  return make_double2(__dadd_rn(__dmul_rn(a.x, b.x), c.x), __dadd_rn(__dmul_rn(a.y, b.y), c.y));
}
// one rounding of an fp64 value to the working precision
template <typename W> __device__ __forceinline__ W to_work(double x);
template <> __device__ __forceinline__ float to_work<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ double to_work<double>(double x) { return x; }
// 8 consecutive working-precision values from shared memory (16 B aligned)
__device__ __forceinline__ void load8(const float* p, float* v) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const double* p, double* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 a = reinterpret_cast<const double2*>(p)[q];
    v[2 * q] = a.x;
    v[2 * q + 1] = a.y;
  }
}
}  // namespace

// shared-memory slot layout (per stage), all offsets 16-byte aligned
struct SlotGeom {
  int data;   // GS * ncols * 8 * sizeof(T)
  int ucol;   // GS * 8 * sizeof(T)
  int upend;  // PMAX * GS * 8 * wsz   (raw pending u rows, TMA; wsz = sizeof(W))
  int us;     // GS * 8 * wsz          (u of this step)
  int nv;     // PMAX * GS * 8 * wsz   (-v rows)
  int total;
};
__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline SlotGeom slot_geom(int GS, int ncols, int esz, int pmax, int wsz) {
  SlotGeom g;
  g.data = 0;
  g.ucol = al16(GS * ncols * 8 * esz);
  g.upend = g.ucol + al16(GS * 8 * esz);
  g.us = g.upend + al16(pmax * GS * 8 * wsz);
  g.nv = g.us + al16(GS * 8 * wsz);
  g.total = g.nv + al16(pmax * GS * 8 * wsz);
  return g;
}

constexpr int NCW = 16;                      // consumer warps
constexpr int PASS_BLOCK = 32 * (NCW + 2);   // + producer + prep
constexpr int COLS_PER_WARP = 64;            // lane owns columns lane, lane + 32
constexpr int RED_BYTES = 1024 * 2 * 8;      // cross-warp partials (WR * CW * 64 <= 1024 columns)

// PMAX: capacity of the pending lists; EXACT: npend == PMAX at compile time (the common
// npend <= 8 launches: the formation loops carry no runtime predicate); STORE: this launch
// re-stores fl_L(A~) (p.store, as a compile-time flag)
template <typename T, int PMAX, bool EXACT, bool STORE>
__global__ void __launch_bounds__(PASS_BLOCK, 1) k_pass_ws(PassParams p) {
  if (p.sc->done) return;
  using W = typename Work<T>::W;
  using W2 = typename Work<T>::W2;
  constexpr int WSZ = (int)sizeof(W);
  W* __restrict__ Ubuf = reinterpret_cast<W*>(p.U);
  const W* __restrict__ Fbuf = reinterpret_cast<const W*>(p.F);
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = p.n, j = p.j;
  const int npend = EXACT ? PMAX : p.npend;
  constexpr int PA = PMAX > 0 ? PMAX : 1;        // array extent (npend = 0 at step 0)
  const int GS = p.gs, NST = p.nst;
  T* __restrict__ S = reinterpret_cast<T*>(p.S);
  const int c_lo = j + 32 * p.chunks_per_split * blockIdx.y;   // CTA column range
  const int c_hi = min(n, c_lo + 32 * p.chunks_per_split);
  const int ncols = c_hi - c_lo;                                  // > 0 (host)
  const SlotGeom geo = slot_geom(GS, p.ncols_slot, (int)sizeof(T), PMAX, WSZ);
  double* red = reinterpret_cast<double*>(smem + (size_t)NST * geo.total);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * geo.total + RED_BYTES);
  uint64_t* prep = full + NST;
  uint64_t* empty = prep + NST;
  // row groups of this CTA: active groups [g_lo, ngroups) split evenly over gridDim.x
  const int64_t g_lo = p.g_lo;
  const int64_t nact = p.ngroups - g_lo;
  const int64_t per = (nact + gridDim.x - 1) / gridDim.x;
  const int64_t gb = g_lo + (int64_t)blockIdx.x * per;
  const int64_t ge = (gb + per < p.ngroups) ? gb + per : p.ngroups;
  const int nst = gb < ge ? (int)((ge - gb + GS - 1) / GS) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rowbytes = ncols * 8 * (int)sizeof(T);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&prep[s], 32);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ======================= TMA producer (one lane) =======================
    if (lane != 0) return;
    int slot_l[PA];
#pragma unroll
    for (int l = 0; l < PMAX; ++l) slot_l[l] = (p.j0 + l) % NSLOT;
    auto issue_store = [&](int i) {
      const int slot = i % NST;
      const int64_t g0 = gb + (int64_t)i * GS;
      const int gsz = (int)((ge - g0) < GS ? (ge - g0) : GS);
      unsigned char* base = smem + (size_t)slot * geo.total;
      // column j is finished after this step and is never stored (other column
      // splits read it concurrently); store columns [max(c_lo, j+1), c_hi)
      const int skip = (c_lo == j) ? 1 : 0;
      const int bytes = rowbytes - skip * 8 * (int)sizeof(T);
      if (bytes <= 0) return;
      for (int r = 0; r < gsz; ++r)
        tma_store(S + ((g0 + r) * n + c_lo + skip) * RG, base + r * rowbytes + skip * 8 * sizeof(T), bytes);
    };
    for (int i = 0; i < nst; ++i) {
      const int slot = i % NST;
      if (i >= NST) {
        mbar_wait(&empty[slot], ((i / NST) & 1) ^ 1);
        if (STORE) {
          issue_store(i - NST);
          bulk_commit();
          bulk_wait_read0();
        }
      }
      const int64_t g0 = gb + (int64_t)i * GS;
      const int gsz = (int)((ge - g0) < GS ? (ge - g0) : GS);
      unsigned char* base = smem + (size_t)slot * geo.total;
      const uint32_t bytes = (uint32_t)(gsz * rowbytes + gsz * 8 * sizeof(T) + npend * gsz * 8 * WSZ);
      mbar_expect_tx(&full[slot], bytes);
      for (int r = 0; r < gsz; ++r) {
        tma_load(base + r * rowbytes, S + ((g0 + r) * n + c_lo) * RG, rowbytes, &full[slot]);
        tma_load(base + geo.ucol + r * 8 * sizeof(T), S + ((g0 + r) * n + j) * RG, 8 * sizeof(T),
                 &full[slot]);
      }
#pragma unroll
      for (int l = 0; l < PMAX; ++l)
        if (l < npend)
          tma_load(base + geo.upend + l * GS * 8 * WSZ, Ubuf + (int64_t)slot_l[l] * p.m_pad + g0 * 8,
                   gsz * 8 * WSZ, &full[slot]);
    }
    if (STORE) {
      for (int i = max(0, nst - NST); i < nst; ++i) {
        mbar_wait(&empty[i % NST], (i / NST) & 1);
        issue_store(i);
      }
      bulk_commit();
    }
    bulk_wait0();
    return;
  }

  if (warp == 1) {
    // ========================= prep warp ==========================
    W fj[PA];
    double cl_[PA];
    int64_t tstep[PA];
#pragma unroll
    for (int l = 0; l < PMAX; ++l) {
      const int sl = (p.j0 + l) % NSLOT;
      fj[l] = (l < npend) ? Fbuf[(int64_t)sl * n + j] : W(0);
      cl_[l] = (l < npend) ? p.cvec[p.j0 + l] : 0.0;
      tstep[l] = p.j0 + l;
    }
    W* __restrict__ Uj = Ubuf + (int64_t)(j % NSLOT) * p.m_pad;
    int slot = 0;
    uint32_t phase = 0;
    for (int i = 0; i < nst; ++i) {
      const int64_t g0 = gb + (int64_t)i * GS;
      const int gsz = (int)((ge - g0) < GS ? (ge - g0) : GS);
      unsigned char* base = smem + (size_t)slot * geo.total;
      const T* ucol = reinterpret_cast<const T*>(base + geo.ucol);
      const W* upend = reinterpret_cast<const W*>(base + geo.upend);
      W* us = reinterpret_cast<W*>(base + geo.us);
      W* nv = reinterpret_cast<W*>(base + geo.nv);
      mbar_wait(&full[slot], phase);
      for (int r = lane; r < gsz * 8; r += 32) {
        const int64_t rl = g0 * 8 + r;
        const int64_t rg = p.row_offset + rl;
        const bool real = rl < p.m_local;
        W a = Chunk<T>::get(ucol + (r >> 3) * 8, r & 7);
#pragma unroll
        for (int l = 0; l < PMAX; ++l) {
          if (l < npend) {
            W v;
            if (!real || rg < tstep[l]) v = W(0);
            else if (rg == tstep[l]) v = W(1);
            else v = to_work<W>((double)upend[l * GS * 8 + r] * cl_[l]);
            nv[l * GS * 8 + r] = -v;
            a = upd1(-v, fj[l], a);
          }
        }
        if (STORE) a = Chunk<T>::rnd(a);
        const W u = (real && rg >= j) ? a : W(0);
        us[r] = u;
        if (blockIdx.y == 0) Uj[rl] = u;
      }
      mbar_arrive(&prep[slot]);   // every lane arrives (count 32): its smem writes are released
      if (++slot == NST) { slot = 0; phase ^= 1; }
    }
    return;
  }

  // ========================== consumers (16 warps) ==========================
  const int cwarp = warp - 2;
  const int CW = p.cw, WR = p.wr;
  const int cw = cwarp % CW, rw = cwarp / CW;
  const bool active = rw < WR;
  const int col0 = cw * COLS_PER_WARP + lane;          // CTA-relative columns of this lane
  const int col1 = col0 + 32;
  const bool v0 = active && col0 < ncols, v1 = active && col1 < ncols;
  const int slot0 = p.j0 % NSLOT;
  W2 f2[PA];
#pragma unroll
  for (int l = 0; l < PMAX; ++l) {
    const int sl = (slot0 + l) % NSLOT;
    f2[l].x = (l < npend && v0) ? Fbuf[(int64_t)sl * n + c_lo + col0] : W(0);
    f2[l].y = (l < npend && v1) ? Fbuf[(int64_t)sl * n + c_lo + col1] : W(0);
  }
  double aw0 = 0.0, aw1 = 0.0, as0 = 0.0, as1 = 0.0;
  const int64_t jloc = (int64_t)j - p.row_offset;
  const int64_t gj = (jloc >= 0 && jloc < p.m_local) ? (jloc >> 3) : -1;
  const int jr = (int)(jloc & 7);
  // clamp the column offsets of invalid lanes into the row (their results are discarded)
  const int o0 = (v0 ? col0 : 0) * 8, o1 = (v1 ? col1 : 0) * 8;

  int slot = 0;
  uint32_t phase = 0;
  for (int i = 0; i < nst; ++i) {
    const int64_t g0 = gb + (int64_t)i * GS;
    const int gsz = (int)((ge - g0) < GS ? (ge - g0) : GS);
    const int gjs = (gj >= g0 && gj < g0 + gsz) ? (int)(gj - g0) : -1;   // stage group holding row j
    unsigned char* base = smem + (size_t)slot * geo.total;
    T* data = reinterpret_cast<T*>(base);
    const W* us = reinterpret_cast<const W*>(base + geo.us);
    const W* nv = reinterpret_cast<const W*>(base + geo.nv);
    mbar_wait(&prep[slot], phase);
    if (active && (v0 || v1)) {
      for (int gl = rw; gl < gsz; gl += WR) {
        T* d0 = data + (size_t)gl * ncols * 8 + o0;
        T* d1 = data + (size_t)gl * ncols * 8 + o1;
        W2 x[8];
        Chunk<T>::load2(d0, d1, x);
#pragma unroll
        for (int l = 0; l < PMAX; ++l) {
          if (l < npend) {
            W vv[8];
            load8(nv + l * GS * 8 + gl * 8, vv);
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = upd2(vv[q], f2[l], x[q]);
          }
        }
        // invalid lanes alias column 0's chunk: they must not write it back
        if (STORE) Chunk<T>::round_store2(d0, d1, x, v0, v1);
        W uu[8];
        load8(us + gl * 8, uu);
        if (gl == gjs) {                                  // the group holding row j (rare)
          W2 xj = x[0];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q == jr) xj = x[q];
            if (q < jr) x[q] = splat2(W(0));
          }
          if (v0) p.xr[c_lo + col0] = xj.x;
          if (v1) p.xr[c_lo + col1] = xj.y;
        }
        W2 pw = mul2(x[0], splat2(uu[0]));
        W2 ps = mul2(x[0], x[0]);
#pragma unroll
        for (int q = 1; q < 8; ++q) {
          pw = mac2(x[q], splat2(uu[q]), pw);
          ps = mac2(x[q], x[q], ps);
        }
        aw0 += (double)pw.x;
        aw1 += (double)pw.y;
        as0 += (double)ps.x;
        as1 += (double)ps.y;
      }
    }
    if (STORE) fence_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == NST) { slot = 0; phase ^= 1; }
  }
  // cross-warp (row-split) combine in fixed order rw = 0..WR-1, then one write per column
  if (WR > 1) {
    if (active) {
      const int base_c = (rw * CW + cw) * COLS_PER_WARP;   // < WR*CW*64 <= 1024
      red[(base_c + lane) * 2 + 0] = aw0;
      red[(base_c + lane) * 2 + 1] = as0;
      red[(base_c + lane + 32) * 2 + 0] = aw1;
      red[(base_c + lane + 32) * 2 + 1] = as1;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW) : "memory");
    if (active && rw == 0) {
      aw0 = as0 = aw1 = as1 = 0.0;
      for (int r = 0; r < WR; ++r) {
        const int base_c = (r * CW + cw) * COLS_PER_WARP;
        aw0 += red[(base_c + lane) * 2 + 0];
        as0 += red[(base_c + lane) * 2 + 1];
        aw1 += red[(base_c + lane + 32) * 2 + 0];
        as1 += red[(base_c + lane + 32) * 2 + 1];
      }
    }
  }
  if (active && rw == 0) {
    double* pw = p.part + ((int64_t)blockIdx.x * 2 + 0) * n + c_lo;
    double* ps = p.part + ((int64_t)blockIdx.x * 2 + 1) * n + c_lo;
    if (v0) { pw[col0] = aw0; ps[col0] = as0; }
    if (v1) { pw[col1] = aw1; ps[col1] = as1; }
  }
}

// ---------------------------------------------------------------------------
template <typename T, int PMAX, bool EXACT, bool STORE>
static cudaError_t launch_ws_t(const PassParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  cudaError_t e = smem_attr((const void*)k_pass_ws<T, PMAX, EXACT, STORE>, PASS_SMEM_MAX);
  if (e != cudaSuccess) return e;
  k_pass_ws<T, PMAX, EXACT, STORE><<<grid, PASS_BLOCK, smem, st>>>(p);
  return cudaGetLastError();
}

template <typename T, bool STORE>
static cudaError_t dispatch_store(const PassParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  switch (p.npend) {
    case 0: return launch_ws_t<T, 0, true, STORE>(p, grid, smem, st);
    case 1: return launch_ws_t<T, 1, true, STORE>(p, grid, smem, st);
    case 2: return launch_ws_t<T, 2, true, STORE>(p, grid, smem, st);
    case 3: return launch_ws_t<T, 3, true, STORE>(p, grid, smem, st);
    case 4: return launch_ws_t<T, 4, true, STORE>(p, grid, smem, st);
    case 5: return launch_ws_t<T, 5, true, STORE>(p, grid, smem, st);
    case 6: return launch_ws_t<T, 6, true, STORE>(p, grid, smem, st);
    case 7: return launch_ws_t<T, 7, true, STORE>(p, grid, smem, st);
    case 8: return launch_ws_t<T, 8, true, STORE>(p, grid, smem, st);
    default:
      if constexpr (sizeof(T) < 8) return launch_ws_t<T, 16, false, STORE>(p, grid, smem, st);   // fp64: nb <= 8
      return cudaErrorInvalidValue;
  }
}
template <typename T>
static cudaError_t dispatch_ws(const PassParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  return p.store ? dispatch_store<T, true>(p, grid, smem, st) : dispatch_store<T, false>(p, grid, smem, st);
}

template <typename T>
static cudaError_t launch_ws_fmt(PassParams p, int max_ctas, int* gx_out, cudaStream_t st) {
  const int n = p.n, j = p.j;
  const int esz = (int)sizeof(T);
  const int wsz = (int)sizeof(typename Work<T>::W);
  const int nchunks = (n - j + 31) / 32;
  // column splits: at most NCW * 64 = 1024 columns per CTA
  const int max_chunks = NCW * COLS_PER_WARP / 32;
  const int gy = (nchunks + max_chunks - 1) / max_chunks;
  const int cps = (nchunks + gy - 1) / gy;
  p.chunks_per_split = cps;
  const int ncols = std::min(n - j, 32 * cps);
  p.ncols_slot = ncols;
  const int CW = (ncols + COLS_PER_WARP - 1) / COLS_PER_WARP;   // column-warps (<= 16)
  const int WR = NCW / CW;                                       // row-split warps
  p.cw = CW;
  p.wr = WR;
  const int pmax = p.npend <= 8 ? p.npend : 16;     // exact pending count up to 8
  if (p.npend > pmax || pmax > NB_MAX || (wsz == 8 && pmax > 8)) return cudaErrorInvalidValue;
  // stage = GS row groups: ~64 KB of matrix data (tools/pass_tune.py: 48 -> 64 KB is ~1.5 %
  // faster on C4, 80 KB slower), a multiple of WR, at most 64 groups
  static const int stage_kb = [] {
    const char* e = getenv("MPID_PASS_STAGE_KB");   // tuning experiments only
    return e ? atoi(e) : 64;
  }();
  const int rowbytes = ncols * 8 * esz;
  int gpw = std::max(1, (stage_kb * 1024) / (rowbytes * WR));
  int GS = std::min(64, WR * gpw);
  SlotGeom g = slot_geom(GS, ncols, esz, pmax, wsz);
  const size_t fixed = RED_BYTES + 3 * 8 * 8 + 64;
  while (GS > 1 && 2 * (size_t)g.total + fixed > (size_t)PASS_SMEM_MAX) {
    GS = std::max(1, GS / 2);
    g = slot_geom(GS, ncols, esz, pmax, wsz);
  }
  int nst = (int)std::min<size_t>(8, (PASS_SMEM_MAX - fixed) / (size_t)g.total);
  if (nst < 2) return cudaErrorInvalidConfiguration;
  p.gs = GS;
  p.nst = nst;
  const size_t smem = (size_t)nst * g.total + RED_BYTES + 3 * nst * sizeof(uint64_t);
  const int64_t nact = p.ngroups - p.g_lo;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, max_ctas / gy), (nact + GS - 1) / GS));
  dim3 grid(gx, gy);
  p.gx_used = gx;
  *gx_out = gx;
  return dispatch_ws<T>(p, grid, smem, st);
}

cudaError_t launch_pass_tma(int fmt, PassParams p, int max_ctas, int* gx_out, cudaStream_t st) {
  if (fmt == 1) return launch_ws_fmt<__half>(p, max_ctas, gx_out, st);
  if (fmt == 2) return launch_ws_fmt<float>(p, max_ctas, gx_out, st);
  if (fmt == 3) return launch_ws_fmt<double>(p, max_ctas, gx_out, st);
  return cudaErrorInvalidValue;
}

}  // namespace mpid
