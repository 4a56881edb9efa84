// Probe of tcgen05.mma kind::i8 on sm_100a (signed int8 x int8 -> int32 in TMEM):
//  1. correctness of the instruction / smem descriptors against a CPU integer product,
//     A from shared memory (SS) and from tensor memory (TS), M = 128, N = 16 .. 128, K = 128;
//  2. issue throughput per SM for the same shapes (all SMs, operands resident), which
//     decides the tile shapes of the Ozaki-scheme fp64 GEMMs (k_ozaki.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/i8mma_probe tools/i8mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major int8 operand, no swizzle: core matrix = 8 rows x 16 B; element (r, k) at
// (k / 16) * LBO + (r / 8) * 128 + (r % 8) * 16 + k % 16, LBO = rows / 8 * 128
__device__ __forceinline__ int ioff(int r, int k, int rows) {
  return (k >> 4) * (rows / 8 * 128) + (r >> 3) * 128 + (r & 7) * 16 + (k & 15);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// K-major SWIZZLE_128B: 8-row atoms of 8 x 128 B, 16 B chunk c of row r stored at chunk c ^ (r % 8);
// element (r, k) at (r / 8) * 1024 + (r % 8) * 128 + (((k / 16) ^ (r % 8)) * 16) + k % 16 (K <= 128)
__device__ __forceinline__ int swoff(int r, int k) {
  return (r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 4) ^ (r & 7)) & 7) << 4) + (k & 15);
}
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO = 1024 B between 8-row groups
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint32_t idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
}

constexpr int K = 128;

// grid = CTAs; iters = MMA groups (K = 128 each) per CTA; out != null: store D of CTA 0
__global__ void __launch_bounds__(128, 1) probe(const int8_t* A, const int8_t* B, int32_t* out, int N, int ts,
                                                int iters, long long* cyc, int nacc, int sw) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* sA = smem;
  unsigned char* sB = smem + 128 * K;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * K; i += blockDim.x) sA[sw ? swoff(i / K, i % K) : ioff(i / K, i % K, 128)] = (unsigned char)A[i];
  for (int i = tid; i < N * K; i += blockDim.x) sB[sw ? swoff(i / K, i % K) : ioff(i / K, i % K, N)] = (unsigned char)B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // A into TMEM columns 256.. (TS mode): lane r = row r, K bytes packed 4 per column
  if (ts) {
    const int r = warp * 32 + lane;
    uint32_t v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      uint32_t w = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) w |= (uint32_t)(uint8_t)A[r * K + c * 4 + b] << (8 * b);
      v[c] = w;
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + ((uint32_t)(warp * 32) << 16) +
                                                                                   256u),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t id = idesc_i8(N);
      const uint32_t a0 = su32(sA), b0 = su32(sB);
      uint32_t ph = 0;
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < K / 32; ++q) {
          const uint64_t db = sw ? sdesc_sw128(b0 + q * 32) : sdesc(b0 + q * 2 * (N / 8 * 128), N / 8 * 128, 128);
          const uint32_t dcol = (uint32_t)(((it * (K / 32) + q) % nacc) * N);
          const uint32_t accf = (nacc == 1 ? q > 0 : it > 0) ? 1u : 0u;
          if (ts) mma_ts(tmem + dcol, tmem + 256u + (uint32_t)(q * 8), db, id, accf);
          else mma_ss(tmem + dcol, sw ? sdesc_sw128(a0 + q * 32) : sdesc(a0 + q * 2 * 2048, 2048, 128), db, id, accf);
        }
        if ((it & 63) == 63 || it == iters - 1) {
          commit(&bar);
          mbar_wait(&bar, ph);
          ph ^= 1;
        }
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
  if (out && blockIdx.x == 0) {
    const int r = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 16; ++i) out[r * N + c0 + i] = (int32_t)v[i];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// TMEM read throughput: nw warps each load x16 columns repeatedly (all lanes of its quarter)
__global__ void __launch_bounds__(512, 1) tmem_ld_probe(int iters, long long* cyc, uint32_t* sink) {
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[16];
    const uint32_t col = (uint32_t)(((it * 16) + (warp >> 2) * 64) & 511);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)((warp & 3) * 32) << 16) + col));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) acc += v[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  std::vector<int8_t> hA(128 * K), hB(256 * K);
  srand(1);
  for (auto& x : hA) x = (int8_t)((rand() % 255) - 127);
  for (auto& x : hB) x = (int8_t)((rand() % 255) - 127);
  int8_t *dA, *dB;
  int32_t* dD;
  long long* dc;
  cudaMalloc(&dA, hA.size());
  cudaMalloc(&dB, hB.size());
  cudaMalloc(&dD, 128 * 256 * 4);
  cudaMalloc(&dc, 1024 * 8);
  cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int Ns[] = {16, 32, 64, 128, 256};
  for (int sw = 0; sw < 2; ++sw)
  for (int ts = 0; ts < 2; ++ts)
    for (int N : Ns) {
      const int smem = 128 * K + 256 * K;
      cudaMemset(dD, 0, 128 * 256 * 4);
      probe<<<1, 128, smem>>>(dA, dB, dD, N, ts, 1, dc, 1, sw);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("{\"ts\": %d, \"N\": %d, \"error\": \"%s\"}\n", ts, N, cudaGetErrorString(e));
        return 1;
      }
      std::vector<int32_t> hD(128 * N);
      cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
      long bad = 0;
      for (int r = 0; r < 128; ++r)
        for (int c = 0; c < N; ++c) {
          int32_t s = 0;
          for (int k = 0; k < K; ++k) s += (int32_t)hA[r * K + k] * (int32_t)hB[c * K + k];
          if (s != hD[r * N + c]) ++bad;
        }
      // throughput: all SMs, 4096 K=128 groups each
      const int iters = 4096;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      probe<<<nsm, 128, smem>>>(dA, dB, nullptr, N, ts, 64, dc, 1, sw);
      cudaEventRecord(e0);
      probe<<<nsm, 128, smem>>>(dA, dB, nullptr, N, ts, iters, dc, 1, sw);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> hc(nsm);
      cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (auto c : hc) mx = c > mx ? c : mx;
      const double ops = 2.0 * 128 * N * K * (double)iters * nsm;
      printf("{\"sw128\": %d, \"ts\": %d, \"N\": %d, \"mismatches\": %ld, \"ms\": %.3f, \"tops\": %.1f, "
             "\"cyc_per_mma\": %.2f, \"floor_cyc\": %.1f}\n",
             sw, ts, N, bad, ms, ops / ms / 1e9, (double)mx / (iters * (K / 32)), 128.0 * N / 256.0);
    }
  for (int N : {16, 32, 64}) {
    for (int nacc : {2, 4, 8}) {
      if (nacc * N > 256) continue;
      const int smem = 128 * K + 256 * K;
      const int iters = 4096;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      probe<<<nsm, 128, smem>>>(dA, dB, nullptr, N, 0, 64, dc, nacc, 1);
      cudaEventRecord(e0);
      probe<<<nsm, 128, smem>>>(dA, dB, nullptr, N, 0, iters, dc, nacc, 1);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> hc(nsm);
      cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (auto c : hc) mx = c > mx ? c : mx;
      const double ops = 2.0 * 128 * N * K * (double)iters * nsm;
      printf("{\"nacc\": %d, \"N\": %d, \"tops\": %.1f, \"cyc_per_mma\": %.2f, \"floor_cyc\": %.1f, \"err\": \"%s\"}\n", nacc, N,
             ops / ms / 1e9, (double)mx / (iters * (K / 32)), 128.0 * N / 256.0, cudaGetErrorString(cudaGetLastError()));
    }
  }
  uint32_t* sink;
  cudaMalloc(&sink, (size_t)nsm * 512 * 4);
  for (int nw : {4, 8, 16}) {
    const int iters = 20000;
    tmem_ld_probe<<<nsm, 32 * nw>>>(100, dc, sink);
    tmem_ld_probe<<<nsm, 32 * nw>>>(iters, dc, sink);
    cudaDeviceSynchronize();
    std::vector<long long> hc(nsm);
    cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto c : hc) mx = c > mx ? c : mx;
    const double bytes = (double)nw * 32 * 16 * 4 * iters;
    printf("{\"tmem_ld_warps\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", nw, bytes / (double)mx);
  }
  return 0;
}
