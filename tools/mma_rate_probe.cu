// Issue-rate probe of tcgen05.mma on sm_100a (what bounds a stream of MMAs from one CTA):
// kind::i8 (K = 32) and kind::f16 (K = 16), M = 128, N = 16 .. 256, operands resident in
// shared memory (no-swizzle K-major), accumulators in TMEM; variants: CTAs per SM (1 or 2,
// TMEM split) and issuing warps per CTA (1 or 2, each its own accumulator).  Prints cycles
// per MMA per issuing thread and the chip's TOPS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mma_rate_probe tools/mma_rate_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
template <int KIND>   // 0 = i8, 1 = f16
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
  else
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
}

// 128 B per (8-row, 16 B) core matrix; operands zero-filled (values do not change the rate)
template <int KIND>
__global__ void __launch_bounds__(128) rate(int N, int iters, int nwarps_issue, int tcols, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 256) * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)), "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const uint32_t id = (KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10)) : (1u << 4)) | ((uint32_t)(N >> 3) << 17) |
                      ((uint32_t)(128 >> 4) << 24);
  const uint32_t a0 = su32(smem), b0 = a0 + 128 * 32;
  long long t0 = clock64();
  if (warp < nwarps_issue && lane == 0) {
    const uint32_t dcol = (uint32_t)(warp * N);
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      // K = 32 bytes per MMA: two core matrices along K (LBO = M/8 * 128)
      mma<KIND>(tmem + dcol, sdesc(a0, 2048, 128), sdesc(b0, N / 8 * 128, 128), id, it > 0 ? 1u : 0u);
      if ((it & 255) == 255 || it == iters - 1) {
        commit(&bar[warp]);
        mbar_wait(&bar[warp], ph);
        ph ^= 1;
      }
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols));
}

// one issuing thread, U MMAs per iteration with U distinct descriptor sets (B start offsets
// differ by 128 B), each into its own accumulator: does the per-MMA issue cost come from
// reusing the uniform registers the previous MMA still reads?
template <int U>
__global__ void __launch_bounds__(128) rate_unroll(int N, int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 512) * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const uint32_t id = ((2u << 4) | (1u << 7) | (1u << 10)) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t a0 = su32(smem), b0 = a0 + 128 * 32;
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    uint64_t da[U], db[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      da[u] = sdesc(a0, 2048, 128);
      db[u] = sdesc(b0 + u * 128, N / 8 * 128, 128);
    }
    uint32_t ph = 0;
    for (int it = 0; it < iters; it += U) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (uint32_t)(u * (512 / U))),
                     "l"(da[u]), "l"(db[u]), "r"(id), "r"(it > 0 ? 1u : 0u) : "memory");
      if ((it & 255) >= 256 - U || it + U >= iters) {
        commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int U>
void run_unroll(int nsm, long long* dc) {
  const int smem = (128 + 512) * 32;
  cudaFuncSetAttribute(rate_unroll<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {16, 64, 128}) {
    if (N * U > 512) continue;
    const int iters = 8192;
    rate_unroll<U><<<nsm, 128, smem>>>(N, 256, dc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate_unroll<U><<<nsm, 128, smem>>>(N, iters, dc);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> hc(nsm);
    cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto c : hc) mx = c > mx ? c : mx;
    const double ops = 2.0 * 128 * N * 32 * (double)iters * nsm;
    printf("{\"kind\": \"i8\", \"unroll\": %d, \"N\": %d, \"cyc_per_mma\": %.1f, \"tops\": %.1f, \"err\": \"%s\"}\n", U, N,
           (double)mx / iters, ops / ms / 1e9, cudaGetErrorString(e));
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* dc;
  cudaMalloc(&dc, 4096 * 8);
  const int smem = (128 + 256) * 32;
  cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int kind = 0; kind < 2; ++kind)
    for (int cps : {1, 2})
      for (int nw : {1, 2})
        for (int N : {16, 64, 128, 256}) {
          const int tcols = cps == 1 ? 512 : 256;
          if (nw * N > tcols) continue;
          const int iters = 8192;
          const int grid = nsm * cps;
          auto launch = [&](int it) {
            if (kind == 0) rate<0><<<grid, 128, smem>>>(N, it, nw, tcols, dc);
            else rate<1><<<grid, 128, smem>>>(N, it, nw, tcols, dc);
          };
          launch(256);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaEventRecord(e0);
          launch(iters);
          cudaEventRecord(e1);
          cudaError_t e = cudaDeviceSynchronize();
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          std::vector<long long> hc(grid);
          cudaMemcpy(hc.data(), dc, grid * 8, cudaMemcpyDeviceToHost);
          long long mx = 0;
          for (auto c : hc) mx = c > mx ? c : mx;
          const int K = kind == 0 ? 32 : 16;
          const double ops = 2.0 * 128 * N * K * (double)iters * grid * nw;
          printf("{\"kind\": \"%s\", \"ctas_per_sm\": %d, \"issue_warps\": %d, \"N\": %d, \"cyc_per_mma_per_thread\": %.1f, "
                 "\"tops\": %.1f, \"err\": \"%s\"}\n",
                 kind == 0 ? "i8" : "f16", cps, nw, N, (double)mx / iters, ops / ms / 1e9, cudaGetErrorString(e));
        }
  run_unroll<1>(nsm, dc);
  run_unroll<2>(nsm, dc);
  run_unroll<4>(nsm, dc);
  run_unroll<8>(nsm, dc);
  return 0;
}
