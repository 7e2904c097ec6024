// Probe: FP64 FMA throughput vs resident warps per SM scheduler and ILP
// (independent accumulator chains per thread), one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void dfma_chain(long iters, double* out) {
  double acc[ILP];
  for (int j = 0; j < ILP; ++j) acc[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  const double m = 0.9999999, c = 1e-7;
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc[j] = fma(acc[j], m, c);
  }
  double s = 0;
  for (int j = 0; j < ILP; ++j) s += acc[j];
  if (s == 1234.5) out[0] = s;
}
// complex multiply-accumulate pattern of the overlap kernel: N accumulators,
// operands from registers that change every iteration
template <int N>
__global__ void cfma_pattern(long iters, double* out) {
  double2 acc[N], a[N];
  double2 b = make_double2(0.999, 1e-3 * threadIdx.x);
  for (int j = 0; j < N; ++j) { acc[j] = make_double2(j, 0); a[j] = make_double2(1e-3 * j, 0.5); }
  for (long it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      acc[j].x = fma(a[j].x, b.x, acc[j].x);
      acc[j].x = fma(-a[j].y, b.y, acc[j].x);
      acc[j].y = fma(a[j].x, b.y, acc[j].y);
      acc[j].y = fma(a[j].y, b.x, acc[j].y);
    }
    b.x = b.x * 0.999999;
  }
  double s = 0;
  for (int j = 0; j < N; ++j) s += acc[j].x + acc[j].y;
  if (s == 1234.5) out[0] = s;
}
template <class K>
void run(const char* name, K kern, int sms, int warps, long iters, double flops_per_thread_iter, double* out) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<<<sms, 32 * warps>>>(10, out);
  cudaEventRecord(a);
  kern<<<sms, 32 * warps>>>(iters, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl = flops_per_thread_iter * iters * (double)sms * warps * 32;
  printf("%-14s warps/SM=%2d: %6.2f TFLOP/s\n", name, warps, fl / (ms * 1e-3) / 1e12);
}
int main() {
  double* out; cudaMalloc(&out, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 12, 16}) {
    run("dfma ilp4", dfma_chain<4>, sms, w, 200000, 8, out);
    run("dfma ilp8", dfma_chain<8>, sms, w, 100000, 16, out);
    run("dfma ilp16", dfma_chain<16>, sms, w, 50000, 32, out);
    run("cfma n4", cfma_pattern<4>, sms, w, 100000, 32, out);
    run("cfma n8", cfma_pattern<8>, sms, w, 50000, 64, out);
    run("cfma n16", cfma_pattern<16>, sms, w, 25000, 128, out);
  }
  return 0;
}
