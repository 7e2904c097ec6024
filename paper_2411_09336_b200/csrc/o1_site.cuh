// Site step of the small-chi overlap path (overlap.cu, capacity 4): one
// thread owns one (bra, ket) pair's padded 4x4 complex environment.  Split out
// so tools/probes/o1_compute.cu can time the arithmetic alone.
#pragma once

#include "device.cuh"

namespace mpskq {
namespace o1 {

constexpr int kLanes = 32;
constexpr int kP = 4;              // padded chi of the small-chi path
constexpr int kEnt = kP * 2 * kP;  // entries per padded site tensor (32)

// Site step of one (bra, ket) pair, in two halves with many independent
// accumulators (the FP64 pipe needs ILP: two warps per scheduler at ~220
// registers) and a small code footprint (the whole kernel stays in the
// instruction cache although the 8 warps run different bra shapes):
//   phase 1  T[al][p][br] = sum_kb env[al][kb] B[kb][p][br]     al < NA (template)
//   phase 2  env'[ar][br] = sum_{al,p} conj(A[al][p][ar]) T[al][p][br]
//            in al blocks guarded by the bra's chi_s; ar runs over 2, 3 or 4
//            rows (the bra's chi_{s+1})
// The bra's bond dims are exact (warp-uniform).  kb / br run over the zero
// padded 4 unless every ket of the 32-ket block has chi <= 3 at that bond
// (the block "narrow" flags of bonds s and s+1); the br = 3 column is a
// separate guarded pass so skipping it costs one uniform branch.  Skipped
// terms are exact zeros, so the result is bitwise independent of the flags.
template <int NA, int B0, int NB>
__device__ __forceinline__ void o1_phase1_cols(const double2 (&env)[kP][kP], const double2* B, bool narrow_l,
                                               double2 (&T)[kP][2][kP]) {
#pragma unroll
  for (int kb = 0; kb < kP; ++kb) {
    if (kb == kP - 1 && narrow_l) break;  // every ket of the block has chi_s <= 3
    double2 b[2][NB];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int c = 0; c < NB; ++c) b[p][c] = B[((kb * 2 + p) * kP + B0 + c) * kLanes];
#pragma unroll
    for (int al = 0; al < NA; ++al)
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int c = 0; c < NB; ++c)
          T[al][p][B0 + c] = cfma(env[al][kb], b[p][c], T[al][p][B0 + c]);
  }
}

template <int NA>
__device__ __forceinline__ void o1_phase1(const double2 (&env)[kP][kP], const double2* B, bool narrow_l,
                                          bool narrow_r, double2 (&T)[kP][2][kP]) {
#pragma unroll
  for (int al = 0; al < NA; ++al)
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int br = 0; br < kP; ++br) T[al][p][br] = make_double2(0.0, 0.0);
  o1_phase1_cols<NA, 0, kP - 1>(env, B, narrow_l, T);
  if (!narrow_r) o1_phase1_cols<NA, kP - 1, 1>(env, B, narrow_l, T);
}

template <int AL, int R0, int NR, int B0, int NB>
__device__ __forceinline__ void o1_phase2_rows(const double2* A, const double2 (&T)[kP][2][kP],
                                               double2 (&env)[kP][kP]) {
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    double2 av[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) av[r] = A[(AL * 2 + p) * kP + R0 + r];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int c = 0; c < NB; ++c)
        env[R0 + r][B0 + c] = cfmac(av[r], T[AL][p][B0 + c], env[R0 + r][B0 + c]);
  }
}

template <int AL, int B0, int NB>
__device__ __forceinline__ void o1_phase2_al(const double2* A, const double2 (&T)[kP][2][kP], int na1,
                                             double2 (&env)[kP][kP]) {
  o1_phase2_rows<AL, 0, 2, B0, NB>(A, T, env);
  if (na1 > 2) o1_phase2_rows<AL, 2, 1, B0, NB>(A, T, env);
  if (na1 > 3) o1_phase2_rows<AL, 3, 1, B0, NB>(A, T, env);
}

template <int B0, int NB>
__device__ __forceinline__ void o1_phase2_cols(const double2* A, const double2 (&T)[kP][2][kP], int na,
                                               int na1, double2 (&env)[kP][kP]) {
  o1_phase2_al<0, B0, NB>(A, T, na1, env);
  if (na > 1) o1_phase2_al<1, B0, NB>(A, T, na1, env);
  if (na > 2) o1_phase2_al<2, B0, NB>(A, T, na1, env);
  if (na > 3) o1_phase2_al<3, B0, NB>(A, T, na1, env);
}

__device__ __forceinline__ void o1_phase2(const double2* A, const double2 (&T)[kP][2][kP], int na, int na1,
                                          bool narrow_r, double2 (&env)[kP][kP]) {
#pragma unroll
  for (int ar = 0; ar < kP; ++ar)
#pragma unroll
    for (int br = 0; br < kP; ++br) env[ar][br] = make_double2(0.0, 0.0);
  o1_phase2_cols<0, kP - 1>(A, T, na, na1, env);
  if (!narrow_r) o1_phase2_cols<kP - 1, 1>(A, T, na, na1, env);
}

}  // namespace o1
}  // namespace mpskq
