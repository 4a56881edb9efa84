// k_pass — the per-step panel pass of the low-precision pivoted Householder QR
// (Algorithm 2 line 4; Eq. (6)-(7)), the dominant (HBM-bound) kernel.
//
// What one launch computes for step j (readings R4-R6):
//   A~ = S - sum_{pending l} v_l f_l^T   formed per element in fp32 (FMA, step order)
//   [store steps] A~ <- fl_L(A~), written back to S (the storage rounding point)
//   u = A~(:, j) (rows >= j), w = A~^T u and s_i = ||A~(j:m, i)||^2 with 8-row
//   fp32 FMA chains added in fp64, and the row x = A~(j, :).
//
// B200 structure: one persistent CTA per SM; warp 0 is a TMA producer that streams
// stages of GS consecutive 8-row groups (each row group of the CTA's column range
// is contiguous in the interleaved layout) with cp.async.bulk into an NST-deep
// shared-memory ring, together with the stage's pivot-column segment and the
// pending u vectors; 8 consumer warps form, reduce and (on store steps) round in
// place, after which the producer writes the stage back with cp.async.bulk
// stores.  mbarrier full/empty pairs hand stages over; no register staging of
// global loads, so the bytes in flight per SM are the ring (~150-190 KB).
// Packed fp32x2 FMAs (FFMA2, sm_100) halve the formation / reduction issue count.
#include "mpid_internal.cuh"

namespace mpid {

namespace {
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// bounded wait: a pipeline bug traps (an error the host sees) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <typename T> struct V8;
template <> struct V8<__half> {
  static constexpr int BYTES = 16;
  __device__ static __forceinline__ void load(const __half* p, float2* x) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = __half22float2(h[i]);
  }
  // round x to fp16 in place (RNE) and write back
  __device__ static __forceinline__ void round_store(__half* p, float2* x) {
    uint4 v;
    __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      h[i] = __float22half2_rn(x[i]);
      x[i] = __half22float2(h[i]);
    }
    *reinterpret_cast<uint4*>(p) = v;
  }
  __device__ static __forceinline__ float get(const __half* p, int i) { return __half2float(p[i]); }
  __device__ static __forceinline__ float rnd(float a) { return __half2float(__float2half_rn(a)); }
};
template <> struct V8<float> {
  static constexpr int BYTES = 32;
  __device__ static __forceinline__ void load(const float* p, float2* x) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    x[0] = make_float2(a.x, a.y); x[1] = make_float2(a.z, a.w);
    x[2] = make_float2(b.x, b.y); x[3] = make_float2(b.z, b.w);
  }
  __device__ static __forceinline__ void round_store(float* p, float2* x) {
    reinterpret_cast<float4*>(p)[0] = make_float4(x[0].x, x[0].y, x[1].x, x[1].y);
    reinterpret_cast<float4*>(p)[1] = make_float4(x[2].x, x[2].y, x[3].x, x[3].y);
  }
  __device__ static __forceinline__ float get(const float* p, int i) { return p[i]; }
  __device__ static __forceinline__ float rnd(float a) { return a; }
};
}  // namespace

// shared-memory slot layout (per stage), all offsets 16-byte aligned
struct SlotGeom {
  int data;   // GS * ncols * 8 * sizeof(T)
  int ucol;   // GS * 8 * sizeof(T)
  int upend;  // PMAX * GS * 8 * 4
  int uv;     // (1 + PMAX) * GS * 8 * 4
  int total;
};
__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline SlotGeom slot_geom(int GS, int ncols, int esz, int pmax) {
  SlotGeom g;
  g.data = 0;
  g.ucol = al16(GS * ncols * 8 * esz);
  g.upend = g.ucol + al16(GS * 8 * esz);
  g.uv = g.upend + al16(pmax * GS * 8 * 4);
  g.total = g.uv + al16((1 + pmax) * GS * 8 * 4);
  return g;
}

constexpr int NCW = 8;  // consumer warps

template <typename T, int PMAX, int CPW>
__global__ void __launch_bounds__(32 * (NCW + 1), 1) k_pass_tma(PassParams p) {
  if (p.sc->done) return;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = p.n, j = p.j, npend = p.npend;
  const int GS = p.gs, NST = p.nst;
  T* __restrict__ S = reinterpret_cast<T*>(p.S);
  // column range of this CTA
  const int c_lo = j + 32 * p.chunks_per_split * blockIdx.y;
  const int c_hi = min(n, c_lo + 32 * p.chunks_per_split);
  const int ncols = c_hi - c_lo;                      // > 0 by construction (host)
  const SlotGeom geo = slot_geom(GS, p.ncols_slot, (int)sizeof(T), PMAX);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NST * geo.total);
  uint64_t* empty = full + NST;
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
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int slot_l[PMAX];
#pragma unroll
  for (int l = 0; l < PMAX; ++l) slot_l[l] = (p.j0 + l) % NSLOT;

  if (warp == 0) {
    // ======================= TMA producer (one lane) =======================
    if (lane != 0) return;
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
        if (p.store) {
          issue_store(i - NST);
          bulk_commit();
          bulk_wait_read0();
        }
      }
      const int64_t g0 = gb + (int64_t)i * GS;
      const int gsz = (int)((ge - g0) < GS ? (ge - g0) : GS);
      unsigned char* base = smem + (size_t)slot * geo.total;
      const uint32_t bytes = (uint32_t)(gsz * rowbytes + gsz * 8 * sizeof(T) + npend * gsz * 8 * 4);
      mbar_expect_tx(&full[slot], bytes);
      for (int r = 0; r < gsz; ++r) {
        tma_load(base + r * rowbytes, S + ((g0 + r) * n + c_lo) * RG, rowbytes, &full[slot]);
        tma_load(base + geo.ucol + r * 8 * sizeof(T), S + ((g0 + r) * n + j) * RG, 8 * sizeof(T),
                 &full[slot]);
      }
#pragma unroll
      for (int l = 0; l < PMAX; ++l)
        if (l < npend)
          tma_load(base + geo.upend + l * GS * 8 * 4, p.U + (int64_t)slot_l[l] * p.m_pad + g0 * 8,
                   gsz * 8 * 4, &full[slot]);
    }
    if (p.store) {
      for (int i = max(0, nst - NST); i < nst; ++i) {
        mbar_wait(&empty[i % NST], (i / NST) & 1);
        issue_store(i);
      }
      bulk_commit();
    }
    bulk_wait0();
    return;
  }

  // ========================== consumers (8 warps) ==========================
  const int cw = warp - 1;
  const int ct = threadIdx.x - 32;                   // 0..255
  const int slot_j = j % NSLOT;
  float fj[PMAX];
  double cl_[PMAX];
#pragma unroll
  for (int l = 0; l < PMAX; ++l) {
    fj[l] = (l < npend) ? p.F[(int64_t)slot_l[l] * n + j] : 0.f;
    cl_[l] = (l < npend) ? p.cvec[p.j0 + l] : 0.0;
  }
  // this lane's columns: chunk q = cw + NCW * t
  float fr[CPW][PMAX];
  bool valid[CPW];
  int col[CPW];
#pragma unroll
  for (int t = 0; t < CPW; ++t) {
    col[t] = c_lo + 32 * (cw + NCW * t) + lane;
    valid[t] = col[t] < c_hi;
#pragma unroll
    for (int l = 0; l < PMAX; ++l)
      fr[t][l] = (valid[t] && l < npend) ? p.F[(int64_t)slot_l[l] * n + col[t]] : 0.f;
  }
  double accw[CPW], accs[CPW];
#pragma unroll
  for (int t = 0; t < CPW; ++t) accw[t] = accs[t] = 0.0;
  const int64_t jloc = (int64_t)j - p.row_offset;
  const bool own_j = jloc >= 0 && jloc < p.m_local;
  const int64_t gj = own_j ? (jloc >> 3) : -1;

  for (int i = 0; i < nst; ++i) {
    const int slot = i % NST;
    const int64_t g0 = gb + (int64_t)i * GS;
    const int gsz = (int)((ge - g0) < GS ? (ge - g0) : GS);
    unsigned char* base = smem + (size_t)slot * geo.total;
    const T* data = reinterpret_cast<const T*>(base);
    const T* ucol = reinterpret_cast<const T*>(base + geo.ucol);
    const float* upend = reinterpret_cast<const float*>(base + geo.upend);
    float* us = reinterpret_cast<float*>(base + geo.uv);
    float* nv = us + GS * 8;                           // -v rows, [PMAX][GS*8]
    mbar_wait(&full[slot], (i / NST) & 1);
    // ---- prep: pending -v rows and u for the stage's rows -------------------
    for (int r = ct; r < gsz * 8; r += 256) {
      const int64_t rl = g0 * 8 + r;
      const int64_t rg = p.row_offset + rl;
      const bool real = rl < p.m_local;
      float a = V8<T>::get(ucol + (r >> 3) * 8, r & 7);
#pragma unroll
      for (int l = 0; l < PMAX; ++l) {
        if (l < npend) {
          const int64_t tstep = p.j0 + l;
          float v;
          if (!real || rg < tstep) v = 0.f;
          else if (rg == tstep) v = 1.f;
          else v = __double2float_rn((double)upend[l * GS * 8 + r] * cl_[l]);
          nv[l * GS * 8 + r] = -v;
          a = fmaf(-v, fj[l], a);
        }
      }
      if (p.store) a = V8<T>::rnd(a);
      const float u = (real && rg >= j) ? a : 0.f;
      us[r] = u;
      if (blockIdx.y == 0) p.U[(int64_t)slot_j * p.m_pad + rl] = u;
    }
    consumer_bar();
    // ---- main: form, (round+write back), reduce ------------------------------
    for (int r = 0; r < gsz; ++r) {
      const int64_t g = g0 + r;
      float2 vv[PMAX][4];
#pragma unroll
      for (int l = 0; l < PMAX; ++l) {
        if (l < npend) {
          const float4 a = *reinterpret_cast<const float4*>(nv + l * GS * 8 + r * 8);
          const float4 b = *reinterpret_cast<const float4*>(nv + l * GS * 8 + r * 8 + 4);
          vv[l][0] = make_float2(a.x, a.y); vv[l][1] = make_float2(a.z, a.w);
          vv[l][2] = make_float2(b.x, b.y); vv[l][3] = make_float2(b.z, b.w);
        }
      }
      const float4 ua = *reinterpret_cast<const float4*>(us + r * 8);
      const float4 ub = *reinterpret_cast<const float4*>(us + r * 8 + 4);
      const float uu[8] = {ua.x, ua.y, ua.z, ua.w, ub.x, ub.y, ub.z, ub.w};
      const bool gjrow = (g == gj);
#pragma unroll
      for (int t = 0; t < CPW; ++t) {
        if (!valid[t]) continue;
        T* xp = const_cast<T*>(data) + ((size_t)r * ncols + (col[t] - c_lo)) * 8;
        float2 x[4];
        V8<T>::load(xp, x);
#pragma unroll
        for (int l = 0; l < PMAX; ++l) {
          if (l < npend) {
            const float2 ff = make_float2(fr[t][l], fr[t][l]);
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = __ffma2_rn(vv[l][q], ff, x[q]);
          }
        }
        if (p.store) V8<T>::round_store(xp, x);
        float xs[8] = {x[0].x, x[0].y, x[1].x, x[1].y, x[2].x, x[2].y, x[3].x, x[3].y};
        if (gjrow) {
          const int jr = (int)(jloc - g * 8);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (q < jr) xs[q] = 0.f;
          p.xr[col[t]] = xs[jr];
        }
        float2 acc = __fmul2_rn(make_float2(xs[0], xs[0]), make_float2(uu[0], xs[0]));
#pragma unroll
        for (int q = 1; q < 8; ++q) acc = __ffma2_rn(make_float2(xs[q], xs[q]), make_float2(uu[q], xs[q]), acc);
        accw[t] += (double)acc.x;
        accs[t] += (double)acc.y;
      }
    }
    if (p.store) fence_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
#pragma unroll
  for (int t = 0; t < CPW; ++t) {
    if (valid[t]) {
      p.part[((int64_t)blockIdx.x * 2 + 0) * n + col[t]] = accw[t];
      p.part[((int64_t)blockIdx.x * 2 + 1) * n + col[t]] = accs[t];
    }
  }
}

// ---------------------------------------------------------------------------
template <typename T, int PMAX, int CPW>
static cudaError_t launch_tma_t(const PassParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pass_tma<T, PMAX, CPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PASS_SMEM_MAX);
    attr = true;
  }
  k_pass_tma<T, PMAX, CPW><<<grid, 32 * (NCW + 1), smem, st>>>(p);
  return cudaGetLastError();
}

template <typename T, int PMAX>
static cudaError_t launch_tma_p(const PassParams& p, dim3 grid, size_t smem, int cpw, cudaStream_t st) {
  if (cpw <= 1) return launch_tma_t<T, PMAX, 1>(p, grid, smem, st);
  if (cpw <= 2) return launch_tma_t<T, PMAX, 2>(p, grid, smem, st);
  if (cpw <= 4) return launch_tma_t<T, PMAX, 4>(p, grid, smem, st);
  return launch_tma_t<T, PMAX, 8>(p, grid, smem, st);
}

template <typename T>
static cudaError_t launch_tma_fmt(PassParams p, int num_sms, int* gx_out, cudaStream_t st) {
  const int n = p.n, j = p.j;
  const int esz = (int)sizeof(T);
  const int nchunks = (n - j + 31) / 32;
  // column splits: at most NCW * 8 chunks (2048 columns) per CTA
  const int gy = (nchunks + NCW * 8 - 1) / (NCW * 8);
  const int cps = (nchunks + gy - 1) / gy;
  p.chunks_per_split = cps;
  const int ncols = std::min(n - j, 32 * cps);
  p.ncols_slot = ncols;
  const int cpw = (cps + NCW - 1) / NCW;
  const int pmax = p.npend <= 1 ? 1 : p.npend <= 2 ? 2 : p.npend <= 4 ? 4 : p.npend <= 8 ? 8 : 16;
  if (p.npend > pmax || pmax > NB_MAX) return cudaErrorInvalidValue;
  // stage = GS row groups: aim at ~24 KB of matrix data, at most 32 groups (256 rows)
  const int rowbytes = ncols * 8 * esz;
  int GS = std::max(1, std::min(32, (24 * 1024) / rowbytes));
  SlotGeom g = slot_geom(GS, ncols, esz, pmax);
  while (GS > 1 && 3 * (size_t)g.total + 64 > (size_t)PASS_SMEM_MAX) {
    GS = std::max(1, GS / 2);
    g = slot_geom(GS, ncols, esz, pmax);
  }
  int nst = (int)std::min<size_t>(8, (PASS_SMEM_MAX - 256) / (size_t)g.total);
  if (nst < 2) return cudaErrorInvalidConfiguration;
  p.gs = GS;
  p.nst = nst;
  const size_t smem = (size_t)nst * g.total + 2 * nst * sizeof(uint64_t);
  const int64_t nact = p.ngroups - p.g_lo;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms / std::max(1, gy) > 0 ? num_sms / gy : 1,
                                                              (nact + GS - 1) / GS));
  dim3 grid(gx, gy);
  p.gx_used = gx;
  *gx_out = gx;
  switch (pmax) {
    case 1: return launch_tma_p<T, 1>(p, grid, smem, cpw, st);
    case 2: return launch_tma_p<T, 2>(p, grid, smem, cpw, st);
    case 4: return launch_tma_p<T, 4>(p, grid, smem, cpw, st);
    case 8: return launch_tma_p<T, 8>(p, grid, smem, cpw, st);
    default: return launch_tma_p<T, 16>(p, grid, smem, cpw, st);
  }
}

cudaError_t launch_pass_tma(int fmt, PassParams p, int num_sms, int* gx_out, cudaStream_t st) {
  return fmt == 1 ? launch_tma_fmt<__half>(p, num_sms, gx_out, st)
                  : launch_tma_fmt<float>(p, num_sms, gx_out, st);
}

}  // namespace mpid
