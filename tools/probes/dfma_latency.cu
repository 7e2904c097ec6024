// Probe: dependent-chain latency of DFMA, LDS.128 and a DFMA->DFMA chain
// through one accumulator, measured with clock64 in a single thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(int n, double* out, long long* cyc) {
  __shared__ double2 buf[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) buf[i] = make_double2(i, i);
  __syncthreads();
  double x = out[0], m = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, m, c);
  }
  long long t1 = clock64();
  int idx = (int)x & 63;
  double2 v = make_double2(0, 0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v = buf[idx];
      idx = ((int)v.x) & 63;
    }
  }
  long long t3 = clock64();
  out[1] = x + v.y;
  cyc[0] = (t1 - t0);
  cyc[1] = (t3 - t2);
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 16); cudaMalloc(&cyc, 16);
  cudaMemset(out, 0, 16);
  const int n = 1000;
  lat<<<1, 32>>>(n, out, cyc);
  lat<<<1, 32>>>(n, out, cyc);
  long long h[2];
  cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h[0] / (16.0 * n));
  printf("LDS.128 + int convert dependent latency: %.2f cycles\n", h[1] / (16.0 * n));
  return 0;
}
