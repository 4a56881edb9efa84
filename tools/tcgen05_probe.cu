// Probe of the tcgen05 (UMMA) operand/instruction descriptor encodings on sm_100a:
// one CTA computes D[128 x N] = A[128 x K] * B[N x K]^T (fp16 in, fp32 accumulate in
// TMEM), K-major operands in the no-swizzle core-matrix layout, and the host
// compares with a CPU product for several descriptor variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tcgen05_probe tools/tcgen05_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// smem layout of a K-major operand tile (rows x K fp16): 8x8 core matrices of 128 B;
// element (r, k) at (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2
__device__ __forceinline__ int coff(int r, int k, int lbo, int sbo) {
  return (r >> 3) * sbo + (k >> 3) * lbo + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int version) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)(version & 3) << 46;
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

__global__ void probe(const __half* A, const __half* B, float* D, int N, int K, int lbo, int sbo,
                      int desc_lbo_is_k, int version, int mshift) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* sA = smem;
  unsigned char* sB = smem + 128 * K * 2 + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // fill operands
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sA + coff(r, k, lbo, sbo)) = A[r * K + k];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sB + coff(r, k, lbo, sbo)) = B[r * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    // instruction descriptor: c_format F32 (bit 4), a/b F16 (0), K-major both, N>>3 at 17, M>>4 at mshift
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << mshift);
    for (int kk = 0; kk < K / 16; ++kk) {
      // advance K by 16 elements = 2 core matrices along K
      const uint32_t koff = (uint32_t)(kk * 2 * lbo);
      const uint32_t l = desc_lbo_is_k ? lbo : sbo, s = desc_lbo_is_k ? sbo : lbo;
      const uint64_t da = make_sdesc(su32(sA) + koff, l, s, version);
      const uint64_t db = make_sdesc(su32(sB) + koff, l, s, version);
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  // wait for the MMA
  {
    uint32_t done = 0;
    for (int spin = 0; spin < (1 << 24) && !done; ++spin)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // TMEM -> registers: warp w reads lanes 32w..32w+31 (rows), 8 columns at a time
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * warp + lane;
    for (int q = 0; q < 8; ++q) D[row * N + c0 + q] = __uint_as_float(v[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

// tf32 variant: operands fp32 in smem (tensor core reads the tf32 bits), core matrix = 8 rows x 4 fp32
__device__ __forceinline__ int coff32(int r, int k, int lbo, int sbo) {
  return (r >> 3) * sbo + (k >> 2) * lbo + (r & 7) * 16 + (k & 3) * 4;
}
__global__ void probe32(const float* A, const float* B, float* D, int N, int K, int fmt) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int lbo = 128, sbo = (K / 4) * 128;
  unsigned char* sA = smem;
  unsigned char* sB = smem + 128 * K * 4 + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sA + coff32(r, k, lbo, sbo)) = A[r * K + k];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sB + coff32(r, k, lbo, sbo)) = B[r * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint32_t koff = (uint32_t)(kk * 2 * lbo);
      const uint64_t da = make_sdesc(su32(sA) + koff, lbo, sbo, 1);
      const uint64_t db = make_sdesc(su32(sB) + koff, lbo, sbo, 1);
      const uint32_t acc = kk > 0 ? 1u : 0u;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tbase),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  {
    uint32_t done = 0;
    for (int spin = 0; spin < (1 << 24) && !done; ++spin)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * warp + lane;
    for (int q = 0; q < 8; ++q) D[row * N + c0 + q] = __uint_as_float(v[q]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

static void run_tf32() {
  const int N = 128, K = 32;
  std::vector<float> fA(128 * K), fB(N * K), ref(128 * N);
  for (int i = 0; i < 128 * K; ++i) fA[i] = (rand() % 1001 - 500) / 512.0f;   // exact in tf32? (10-bit mantissa) mostly
  for (int i = 0; i < N * K; ++i) fB[i] = (rand() % 257 - 128) / 64.0f;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < N; ++c) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fA[r * K + k] * fB[c * K + k];
      ref[r * N + c] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, fA.size() * 4); cudaMalloc(&dB, fB.size() * 4); cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, fA.data(), fA.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, fB.data(), fB.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe32, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int fmt : {2, 3, 1}) {
    cudaMemset(dD, 0, 128 * N * 4);
    probe32<<<1, 128, 100 * 1024>>>(dA, dB, dD, N, K, fmt);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(128 * N);
    cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int i = 0; i < 128 * N; ++i) md = fmax(md, fabs(out[i] - ref[i]));
    printf("tf32 fmt=%d : %s maxdiff=%g D[0]=%g ref=%g\n", fmt, cudaGetErrorString(e), md, out[0], ref[0]);
    if (e != cudaSuccess) return;
  }
}

int main() {
  run_tf32();
  const int N = 64, K = 32;
  std::vector<__half> hA(128 * K), hB(N * K);
  std::vector<float> fA(128 * K), fB(N * K);
  srand(1);
  for (int i = 0; i < 128 * K; ++i) { float x = (rand() % 17 - 8) / 8.0f; hA[i] = __float2half(x); fA[i] = x; }
  for (int i = 0; i < N * K; ++i) { float x = (rand() % 13 - 6) / 4.0f; hB[i] = __float2half(x); fB[i] = x; }
  std::vector<float> ref(128 * N);
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < N; ++c) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fA[r * K + k] * fB[c * K + k];
      ref[r * N + c] = (float)s;
    }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  // layout: core matrices, K-blocks adjacent: LBO = 128 (K dir), SBO = (K/8)*128 (8-row groups)
  struct V { int lbo, sbo, lbo_is_k, version, mshift; } vs[] = {
      {128, K / 8 * 128, 1, 1, 24}, {128, K / 8 * 128, 0, 1, 24},
      {128, K / 8 * 128, 1, 1, 23}, {128, K / 8 * 128, 0, 1, 23},
      {128, K / 8 * 128, 1, 0, 24}, {128, K / 8 * 128, 0, 0, 24}};
  for (auto& v : vs) {
    cudaMemset(dD, 0, 128 * N * 4);
    probe<<<1, 128, 64 * 1024>>>(dA, dB, dD, N, K, v.lbo, v.sbo, v.lbo_is_k, v.version, v.mshift);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(128 * N);
    cudaMemcpy(out.data(), dD, out.size() * 4, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int i = 0; i < 128 * N; ++i) md = fmax(md, fabs(out[i] - ref[i]));
    printf("lbo=%d sbo=%d lbo_is_k=%d version=%d mshift=%d : %s maxdiff=%g  D[0]=%g ref=%g D[129*?]=%g ref=%g\n",
           v.lbo, v.sbo, v.lbo_is_k, v.version, v.mshift, cudaGetErrorString(e), md, out[0], ref[0],
           out[77 * N + 33], ref[77 * N + 33]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
