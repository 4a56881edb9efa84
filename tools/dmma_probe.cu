// Probe: peak rate of mma.sync m8n8k4 f64 (SASS DMMA.8x8x4) with register-resident operands.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, int nacc_dummy) {
  double acc[16][2];
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<sms, warps * 32>>>(o, 100, 0);
    cudaEventRecord(e0);
    k<<<sms, warps * 32>>>(o, iters, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 16 * (double)iters * warps * sms;
    printf("warps/SM %2d: %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
