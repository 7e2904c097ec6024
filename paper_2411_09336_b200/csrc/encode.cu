// Feature-map angle encoding on the device: per row, the angle of every
// parametrised gate (ansatz.py:130 RZ 2*gamma*x_q, :132 RXX
// 2*gamma^2*(pi/2)*(1-x_i)*(1-x_j)) in the reference's left-to-right
// expression order with round-to-nearest multiplies (no FMA contraction), so
// the angles are bitwise the reference's; then (cos, sin) of the half angle
// (gate_matrix, ansatz.py:92-99) with CUDA's sincos (<= 2 ulp vs libm).
#include <cuda_runtime.h>

#include "device.cuh"
#include "internal.h"

namespace mpskq {

__global__ void encode_kernel(const double* __restrict__ X, int64_t n_rows, int m, int r, int E,
                              const int2* __restrict__ edges, double rz_scale, double rxx_scale,
                              double2* __restrict__ coef, int* __restrict__ bad) {
  const int per = m + E;
  const int64_t np = (int64_t)r * per;
  const int64_t total = n_rows * np;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / np;
    const int p = (int)((idx - row * np) % per);
    const double* x = X + row * m;
    double angle;
    if (p < m) {
      const double xq = x[p];
      if (!isfinite(xq))
        atomicOr(bad, 2);  // build_circuit's finite check (ansatz.py:121-122)
      else if (xq < 0.0 || xq > 2.0)
        atomicOr(bad, 1);  // ... and its [0, 2] range check (:123-124)
      angle = __dmul_rn(rz_scale, xq);
    } else {
      const int2 e = edges[p - m];
      angle = __dmul_rn(__dmul_rn(rxx_scale, __dsub_rn(1.0, x[e.x])), __dsub_rn(1.0, x[e.y]));
    }
    double s, c;
    sincos(0.5 * angle, &s, &c);
    coef[idx] = make_double2(c, s);
  }
}

int launch_encode(const double* X, int64_t n_rows, int m, int r, int d, double gamma, double* coef,
                  int* bad, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  // interaction_graph (ansatz.py:102-106) uploaded once per call (tiny)
  int E = 0;
  for (int k = 1; k <= d; ++k) E += m - k;
  int2* edges = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&edges), sizeof(int2) * (E ? E : 1), st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(edges)");
  int2* host = static_cast<int2*>(malloc(sizeof(int2) * (E ? E : 1)));
  if (!host) return fail(MPSKQ_ERR_NOMEM, "host allocation failed");
  int k0 = 0;
  for (int k = 1; k <= d; ++k)
    for (int i = 0; i + k < m; ++i) host[k0++] = make_int2(i, i + k);
  e = cudaMemcpyAsync(edges, host, sizeof(int2) * E, cudaMemcpyHostToDevice, st);
  // pageable source: the copy is staged before cudaMemcpyAsync returns
  free(host);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(edges)");
  const double rz_scale = 2.0 * gamma;
  const double rxx_scale = (2.0 * (gamma * gamma)) * (M_PI / 2.0);
  const int64_t total = n_rows * (int64_t)r * (m + E);
  const int threads = 256;
  const int blocks = (int)((total + threads - 1) / threads < 148 * 32 ? (total + threads - 1) / threads : 148 * 32);
  if (total > 0)
    encode_kernel<<<blocks, threads, 0, st>>>(X, n_rows, m, r, E, edges, rz_scale, rxx_scale,
                                              reinterpret_cast<double2*>(coef), bad);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "encode_kernel launch");
  cudaFreeAsync(edges, st);
  return MPSKQ_OK;
}

}  // namespace mpskq
