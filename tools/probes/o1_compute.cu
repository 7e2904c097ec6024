// Probe: the overlap kernel's per-site arithmetic alone (o1_site.cuh), with the
// operands already in shared memory -- no TMA ring, no tile bookkeeping.  Bra
// bond dims and ket-block narrow flags are real headline profiles
// (o1_profile.h), so the DFMA count per site matches the production kernel.
#include <cstdio>
#include <cuda_runtime.h>
#include "o1_site.cuh"
#include "o1_profile.h"
using namespace mpskq;
using namespace mpskq::o1;
constexpr int M = 165;
__constant__ int dProf[8][M + 1];
__constant__ int dNarrow[M + 1];
// variant V1: rows {0,1} always and {2,3} together when chi_{s+1} > 2; the
// padded column chosen once per site (NB = 3 or 4), so blocks are larger
template <int AL, int R0, int NB>
__device__ __forceinline__ void v1_block(const double2* A, const double2 (&T)[kP][2][kP], double2 (&env)[kP][kP]) {
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    double2 av[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) av[r] = A[(AL * 2 + p) * kP + R0 + r];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < NB; ++c) env[R0 + r][c] = cfmac(av[r], T[AL][p][c], env[R0 + r][c]);
  }
}
template <int AL, int NB>
__device__ __forceinline__ void v1_al(const double2* A, const double2 (&T)[kP][2][kP], int na1, double2 (&env)[kP][kP]) {
  v1_block<AL, 0, NB>(A, T, env);
  if (na1 > 2) v1_block<AL, 2, NB>(A, T, env);
}
template <int NB>
__device__ __forceinline__ void v1_cols(const double2* A, const double2 (&T)[kP][2][kP], int na, int na1, double2 (&env)[kP][kP]) {
  v1_al<0, NB>(A, T, na1, env);
  if (na > 1) v1_al<1, NB>(A, T, na1, env);
  if (na > 2) v1_al<2, NB>(A, T, na1, env);
  if (na > 3) v1_al<3, NB>(A, T, na1, env);
}
__device__ __forceinline__ void phase2_v1(const double2* A, const double2 (&T)[kP][2][kP], int na, int na1, bool nar_r,
                                          double2 (&env)[kP][kP]) {
#pragma unroll
  for (int ar = 0; ar < kP; ++ar)
#pragma unroll
    for (int br = 0; br < kP; ++br) env[ar][br] = make_double2(0.0, 0.0);
  if (nar_r) v1_cols<3>(A, T, na, na1, env);
  else v1_cols<4>(A, T, na, na1, env);
}
// variant 5/6: phase 2 over the full padded 4 x 4 (rows and columns not
// guarded): bigger blocks, A loads hoistable, more (free) DFMA
template <int NA>
__device__ __forceinline__ void phase2_full(const double2* A, const double2 (&T)[kP][2][kP], double2 (&env)[kP][kP]) {
#pragma unroll
  for (int ar = 0; ar < kP; ++ar)
#pragma unroll
    for (int br = 0; br < kP; ++br) env[ar][br] = make_double2(0.0, 0.0);
#pragma unroll
  for (int al = 0; al < NA; ++al)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      double2 av[kP];
#pragma unroll
      for (int r = 0; r < kP; ++r) av[r] = A[(al * 2 + p) * kP + r];
#pragma unroll
      for (int r = 0; r < kP; ++r)
#pragma unroll
        for (int c = 0; c < kP; ++c) env[r][c] = cfmac(av[r], T[al][p][c], env[r][c]);
    }
}
template <int AL>
__device__ __forceinline__ void full_al(const double2* A, const double2 (&T)[kP][2][kP], double2 (&env)[kP][kP]) {
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    double2 av[kP];
#pragma unroll
    for (int r = 0; r < kP; ++r) av[r] = A[(AL * 2 + p) * kP + r];
#pragma unroll
    for (int r = 0; r < kP; ++r)
#pragma unroll
      for (int c = 0; c < kP; ++c) env[r][c] = cfmac(av[r], T[AL][p][c], env[r][c]);
  }
}
__device__ __forceinline__ void phase2_full_guarded(const double2* A, const double2 (&T)[kP][2][kP], int na, double2 (&env)[kP][kP]) {
#pragma unroll
  for (int ar = 0; ar < kP; ++ar)
#pragma unroll
    for (int br = 0; br < kP; ++br) env[ar][br] = make_double2(0.0, 0.0);
  full_al<0>(A, T, env);
  if (na > 1) full_al<1>(A, T, env);
  if (na > 2) full_al<2>(A, T, env);
  if (na > 3) full_al<3>(A, T, env);
}
template <int NA, int NA1, int NB>
__device__ __forceinline__ void phase2_fixed(const double2* A, const double2 (&T)[kP][2][kP], double2 (&env)[kP][kP]) {
#pragma unroll
  for (int ar = 0; ar < kP; ++ar)
#pragma unroll
    for (int br = 0; br < kP; ++br) env[ar][br] = make_double2(0.0, 0.0);
#pragma unroll
  for (int al = 0; al < NA; ++al)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      double2 av[NA1];
#pragma unroll
      for (int r = 0; r < NA1; ++r) av[r] = A[(al * 2 + p) * kP + r];
#pragma unroll
      for (int r = 0; r < NA1; ++r)
#pragma unroll
        for (int c = 0; c < NB; ++c) env[r][c] = cfmac(av[r], T[al][p][c], env[r][c]);
    }
}
__global__ void __launch_bounds__(256, 1) probe_fixed(int reps, double* out) {
  __shared__ double2 sket[kEnt * kLanes];
  __shared__ double2 sbra[8 * kEnt];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < kEnt * kLanes; i += 256) sket[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  for (int i = tid; i < 8 * kEnt; i += 256) sbra[i] = make_double2(1e-3 * (i % 83), -1e-3 * (i % 79));
  __syncthreads();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    double2 env[kP][kP];
    for (int x = 0; x < kP; ++x)
      for (int y = 0; y < kP; ++y) env[x][y] = make_double2(x == 0 && y == 0 ? 1.0 : 0.0, 0.0);
    for (int s = 0; s < M; ++s) {
      const double2* B = sket + lane;
      const double2* A = sbra + warp * kEnt;
      double2 T[kP][2][kP];
      o1_phase1<3>(env, B, false, false, T);
      phase2_fixed<3, 3, 4>(A, T, env);
    }
    acc += env[0][0].x;
  }
  if (acc == 1234.5) out[0] = acc;
}
template <int variant>
__global__ void __launch_bounds__(256, 1) probe(int reps, int mode, double* out) {
  __shared__ double2 sket[kEnt * kLanes];
  __shared__ double2 sbra[8 * kEnt];
  __shared__ int schi[8][M + 1];
  __shared__ unsigned char snar[M + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < kEnt * kLanes; i += 256) sket[i] = make_double2(1e-3 * (i % 97), 1e-3 * (i % 89));
  for (int i = tid; i < 8 * kEnt; i += 256) sbra[i] = make_double2(1e-3 * (i % 83), -1e-3 * (i % 79));
  for (int i = tid; i < 8 * (M + 1); i += 256) schi[i / (M + 1)][i % (M + 1)] = mode == 0 ? 3 : dProf[i / (M + 1)][i % (M + 1)];
  for (int i = tid; i <= M; i += 256) snar[i] = mode == 0 ? 0 : dNarrow[i];
  __syncthreads();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    double2 env[kP][kP];
    for (int x = 0; x < kP; ++x)
      for (int y = 0; y < kP; ++y) env[x][y] = make_double2(x == 0 && y == 0 ? 1.0 : 0.0, 0.0);
    int na = schi[warp][0];
    for (int s = 0; s < M; ++s) {
      const int na1 = schi[warp][s + 1];
      const bool nar_l = snar[s] != 0, nar_r = snar[s + 1] != 0;
      const double2* B = sket + (variant == 2 ? 0 : lane);
      const double2* A = sbra + warp * kEnt;
      double2 T[kP][2][kP];
      if (variant == 3) {  // phase 2 only: T from env
#pragma unroll
        for (int x = 0; x < kP; ++x)
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int y = 0; y < kP; ++y) T[x][p][y] = env[x][y];
      } else {
        if (variant == 5) {
          switch (na) {
            case 1: o1_phase1<1>(env, B, nar_l, nar_r, T); phase2_full<1>(A, T, env); break;
            case 2: o1_phase1<2>(env, B, nar_l, nar_r, T); phase2_full<2>(A, T, env); break;
            case 3: o1_phase1<3>(env, B, nar_l, nar_r, T); phase2_full<3>(A, T, env); break;
            default: o1_phase1<4>(env, B, nar_l, nar_r, T); phase2_full<4>(A, T, env); break;
          }
        } else {
          switch (na) {
            case 1: o1_phase1<1>(env, B, nar_l, nar_r, T); break;
            case 2: o1_phase1<2>(env, B, nar_l, nar_r, T); break;
            case 3: o1_phase1<3>(env, B, nar_l, nar_r, T); break;
            default: o1_phase1<4>(env, B, nar_l, nar_r, T); break;
          }
        }
      }
      if (variant == 4) {  // phase 1 only: fold T back into env
#pragma unroll
        for (int x = 0; x < kP; ++x)
#pragma unroll
          for (int y = 0; y < kP; ++y) env[x][y] = make_double2(T[x][0][y].x + T[x][1][y].x, T[x][0][y].y - T[x][1][y].y);
      } else if (variant == 5) {
      } else if (variant == 6) phase2_full_guarded(A, T, na, env);
      else if (variant == 1) phase2_v1(A, T, na, na1, nar_r, env);
      else o1_phase2(A, T, na, na1, nar_r, env);
      na = na1;
    }
    acc += env[0][0].x;
  }
  if (acc == 1234.5) out[0] = acc;
}
// DFMA count of one warp's site sequence (mirrors o1_site.cuh's loop bounds)
static double dfma_per_rep(int mode) {
  double n = 0;
  for (int w = 0; w < 8; ++w)
    for (int s = 0; s < M; ++s) {
      int na = mode == 0 ? 3 : kProf[w][s], na1 = mode == 0 ? 3 : kProf[w][s + 1];
      bool nl = mode == 0 ? false : kNarrow[s], nr = mode == 0 ? false : kNarrow[s + 1];
      int kb = nl ? 3 : 4, br = nr ? 3 : 4, rows = na1 <= 2 ? 2 : na1;
      n += 4.0 * (kb * na * 2 * br + na * 2 * rows * br);
    }
  return n * 32;  // threads per warp
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaMemcpyToSymbol(dProf, kProf, sizeof(kProf));
  cudaMemcpyToSymbol(dNarrow, kNarrow, sizeof(kNarrow));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v = 0; v < 7; ++v)
  for (int mode = 0; mode < 2; ++mode) {
    const int reps = 200;
    if (v == 3 || v == 4) continue;
    printf("variant %d%s  ", v, v == 2 ? " (B loads broadcast)" : "");
    auto kern = v == 0 ? probe<0> : v == 1 ? probe<1> : v == 2 ? probe<2> : v == 5 ? probe<5> : probe<6>;
    kern<<<sms, 256>>>(2, mode, out);
    cudaEventRecord(a);
    kern<<<sms, 256>>>(reps, mode, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double fl = 2.0 * dfma_per_rep(mode) * reps * sms;
    printf("%s: %.3f ms, %.2f TFLOP/s executed FP64 (%.0f cycles/site/warp at 1.965 GHz)\n",
           mode == 0 ? "all (3,3), no narrow" : "headline bra profiles + narrow flags", ms,
           fl / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 / (reps * (double)M));
  }
  {
    const int reps = 200;
    probe_fixed<<<sms, 256>>>(2, out);
    cudaEventRecord(a);
    probe_fixed<<<sms, 256>>>(reps, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double fl = 2.0 * dfma_per_rep(0) * reps * sms;
    printf("straight-line (3,3): %.3f ms, %.2f TFLOP/s executed FP64\n", ms, fl / (ms * 1e-3) / 1e12);
  }
  return 0;
}
