// MMA issue-pattern probe (sm_100a): cycles per K-step of the Ozaki TN kernel's 36 kind::i8
// MMAs (M = 128, N = 64, 8 diagonal accumulators), operands resident in shared memory, for
// issue patterns:
//   0: one lane (if lane == 0), descriptors computed per MMA (k_oz_tn as first written)
//   1: converged warp, elect.sync around the K-step's MMAs, descriptors per MMA
//   2: converged warp + elect, descriptors precomputed in registers before the loop
// with 1, 2 or 4 issuing warps (diagonals split between them).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/issue_probe tools/issue_probe.cu
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
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
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
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.b32 %0, 1, 0, P;\n}" : "=r"(pred));
  return pred != 0;
}
constexpr int N = 64;
// diagonal owner of d for ni issuers: pairs (d, 7 - d) -> issuer (min(d, 7 - d)) % ni
__device__ __forceinline__ bool owns(int d, int w, int ni) { return (min(d, 7 - d) % ni) == w; }

template <int PAT>
__global__ void __launch_bounds__(160, 1) issue(int ksteps, int ni, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (32768 + 16384) * 4 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x < 4) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[threadIdx.x])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const uint32_t id = ((2u << 4) | (1u << 7) | (1u << 10)) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  const int w = warp - 1;
  if (warp >= 1 && w < ni) {
    uint32_t ph = 0;
    // 4 stage slots of (A 32 KB + B 16 KB): the K-step s uses slot s % 4 (like the pipeline)
    uint64_t da[8], db[8];
    if (PAT == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        da[q] = sdesc(su32(smem) + q * 4096, 2048, 128);
        db[q] = sdesc(su32(smem) + 32768 * 4 + q * 2048, 1024, 128);
      }
    }
    for (int s = 0; s < ksteps; ++s) {
      const uint32_t a = su32(smem) + (uint32_t)((s & 3) * 0), b = su32(smem) + 32768 * 4 * 0 + 32768;
      const bool first = (s & 511) == 0;
      if (PAT == 0) {
        if (lane == 0) {
#pragma unroll
          for (int d = 0; d < 8; ++d)
            if (owns(d, w, ni))
#pragma unroll
              for (int pa = 0; pa <= d; ++pa)
                mma(tmem + (uint32_t)(d * N), sdesc(a + pa * 4096, 2048, 128), sdesc(b + (d - pa) * 2048, 1024, 128), id,
                    (first && pa == 0) ? 0u : 1u);
        }
      } else if (PAT >= 3) {
        // pattern 0 plus the pipeline's per-K-step extras: 3 = a commit per K-step,
        // 4 = a tcgen05 after-sync fence per K-step, 5 = both, 6 = both + descriptors varying with the slot
        const uint32_t aa = PAT == 6 ? su32(smem) + (uint32_t)((s & 3) * 49152) : a;
        const uint32_t bb2 = PAT == 6 ? aa + 32768 : b;
        if (PAT >= 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
#pragma unroll
          for (int d = 0; d < 8; ++d)
            if (owns(d, w, ni))
#pragma unroll
              for (int pa = 0; pa <= d; ++pa)
                mma(tmem + (uint32_t)(d * N), sdesc(aa + pa * 4096, 2048, 128), sdesc(bb2 + (d - pa) * 2048, 1024, 128), id,
                    (first && pa == 0) ? 0u : 1u);
          if (PAT != 4) commit(&bar[w]);
        }
      } else if (PAT == 1) {
        if (elect_one()) {
#pragma unroll
          for (int d = 0; d < 8; ++d)
            if (owns(d, w, ni))
#pragma unroll
              for (int pa = 0; pa <= d; ++pa)
                mma(tmem + (uint32_t)(d * N), sdesc(a + pa * 4096, 2048, 128), sdesc(b + (d - pa) * 2048, 1024, 128), id,
                    (first && pa == 0) ? 0u : 1u);
        }
        __syncwarp();
      } else {
        if (elect_one()) {
#pragma unroll
          for (int d = 0; d < 8; ++d)
            if (owns(d, w, ni))
#pragma unroll
              for (int pa = 0; pa <= d; ++pa)
                mma(tmem + (uint32_t)(d * N), da[pa], db[d - pa], id, (first && pa == 0) ? 0u : 1u);
        }
        __syncwarp();
      }
      if ((s & 31) == 31 || s == ksteps - 1) {
        if (lane == 0) commit(&bar[w]);
        __syncwarp();
        mbar_wait(&bar[w], ph);
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

template <int PAT>
void run(int nsm, long long* dc) {
  const int smem = 32768 * 4 + 16384 * 4;
  cudaFuncSetAttribute(issue<PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ni : {1, 2, 4}) {
    const int ks = 2048;
    issue<PAT><<<nsm, 160, smem>>>(64, ni, dc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    issue<PAT><<<nsm, 160, smem>>>(ks, ni, dc);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> hc(nsm);
    cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto c : hc) mx = c > mx ? c : mx;
    const double ops = 2.0 * 128 * N * 32 * 36.0 * ks * nsm;
    printf("{\"pattern\": %d, \"issuers\": %d, \"cyc_per_kstep\": %.1f, \"floor\": %d, \"tops\": %.1f, \"err\": \"%s\"}\n", PAT, ni,
           (double)mx / ks, 36 * N / 2, ops / ms / 1e9, cudaGetErrorString(e));
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* dc;
  cudaMalloc(&dc, 4096 * 8);
  run<0>(nsm, dc);
  run<1>(nsm, dc);
  run<2>(nsm, dc);
  run<3>(nsm, dc);
  run<4>(nsm, dc);
  run<5>(nsm, dc);
  run<6>(nsm, dc);
  return 0;
}
