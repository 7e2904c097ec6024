// Probe: FP64 tensor-core (DMMA m8n8k4) vs FFMA64 throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(long iters, double* out) {
  double d[8][2];
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 1234.5) out[0] = s;
}
__global__ void ffma_loop(long iters, double* out) {
  double acc[16];
  for (int j = 0; j < 16; ++j) acc[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], 0.9999999, 1e-7);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += acc[j];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int warps = 4; warps <= 16; warps *= 2) {
    long iters = 20000;
    dmma_loop<<<sms * 2, 32 * warps>>>(100, out);
    cudaEventRecord(a);
    dmma_loop<<<sms * 2, 32 * warps>>>(iters, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 256 * 8 * iters * (double)(sms * 2 * warps);
    printf("DMMA  warps/CTA=%2d: %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    ffma_loop<<<sms * 2, 32 * warps>>>(100, out);
    cudaEventRecord(a);
    ffma_loop<<<sms * 2, 32 * warps>>>(iters * 8, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    flops = 2.0 * 16 * iters * 8 * (double)(sms * 2 * warps * 32);
    printf("FFMA64 warps/CTA=%2d: %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
