// Batched MPS simulation of a compiled gate program (one CTA per state) and
// the standalone batched truncated SVD.
//
// Reference semantics (/root/reference/pkg/src/mpskernel/):
//   init_state            mps.py:90-102
//   _left/_right_isometrize, canonicalize   mps.py:105-138
//   apply_one_qubit       mps.py:147-160
//   apply_two_qubit       mps.py:163-205
//   svd_truncated         tensor.py:87-123 (NOISE_FLOOR tensor.py:17)
//   run_circuit           mps.py:224-247 (absorb rule compiled into the ops)
//
// B200 design: the op program is identical for every data row, so each CTA
// replays it for one state while all states run concurrently.  Site tensors
// live in HBM (L1/L2 resident while hot); the working set of one op — the two
// site tensors, the 2chi x 2chi theta matrix and the Jacobi rotation
// accumulator — lives in shared memory.  The SVD is a one-sided (Hestenes)
// Jacobi in FP64 with a parallel round-robin pair ordering, one group of lanes
// per column pair, which keeps full relative accuracy on the small singular
// values the truncation rule compares against the budget.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

#include "device.cuh"
#include "internal.h"

namespace mpskq {

// NOISE_FLOOR = 10 * finfo(float64).eps   (tensor.py:17)
__device__ constexpr double kNoiseFloor = 10.0 * DBL_EPSILON;
// 1/sqrt(2) exactly as the reference rounds it: _H_MATRIX = [[1,1],[1,-1]]/sqrt(2)
__device__ constexpr double kInvSqrt2 = 0.7071067811865475;
#ifndef MPSKQ_NOISE_SCALE_N
#define MPSKQ_NOISE_SCALE_N 1  // 0: round-1 threshold (A/B only)
#endif
constexpr int kMaxSweeps = 40;
constexpr int kNoConvergence = 1 << 30;  // flag bit in jacobi()'s round count
// Lanes (threads) per state by capacity.  Same-box A/B of the simulator
// (tools/ab_sim_headline.py, tools/ab_sim_cfg.py, tools/ab_sim.py): halving
// the old 16/64/128/256/384 sped up capacity 4 (15.6 -> 13.7 ms at the
// headline), 8 (34 -> 30 ms), 12-16 (28 -> 23 ms), 24-32 (1.84 -> 1.57 s) and
// 48 (-3%); halving again was slower except at 12-16, and 4 lanes breaks the
// capacity-4 Jacobi.  Round 2, with the workspace in global scratch (below):
// 64 lanes at 12-32, 256 at 64-96 (3 states per SM); capacity 128 keeps 512
// (its batches are small — 148 states at the 165-qubit d=6 budget-1e-24
// case — so per-state latency rules: 256 lanes took 30 -> 48 s there).
#ifndef MPSKQ_NT4
#define MPSKQ_NT4 8
#endif
#ifndef MPSKQ_NT8
#define MPSKQ_NT8 32
#endif
#ifndef MPSKQ_NT16
#define MPSKQ_NT16 64
#endif
#ifndef MPSKQ_NT32
#define MPSKQ_NT32 64
#endif
#ifndef MPSKQ_NT48
#define MPSKQ_NT48 192
#endif
#ifndef MPSKQ_NT96
#define MPSKQ_NT96 256  // capacities 64-96: 3 states per SM (d=7 9.8 -> 6.0 s at N=400)
#endif
#ifndef MPSKQ_NT128
#define MPSKQ_NT128 512
#endif
#ifndef MPSKQ_SPC_THREADS
#define MPSKQ_SPC_THREADS 128  // threads of a lockstepped multi-state CTA (NT <= 32)
#endif
// QR preconditioning of the two-qubit SVD from this many columns up (below it
// the direct Jacobi needs only ~3 sweeps and the QR would not pay)
constexpr int kPrecondMinCols = 8;
template <int CAP>
struct kPrecondition {
#ifdef MPSKQ_NO_PRECOND  // A/B builds only
  static constexpr bool value = false;
#else
  static constexpr bool value = CAP >= 8;
#endif
};

#ifdef MPSKQ_DEBUG_COUNTERS
// debug builds only: Jacobi rounds and two-qubit SVDs, summed over states
__device__ unsigned long long g_dbg_rounds = 0, g_dbg_svds = 0, g_dbg_span = 0;
// SM cycles per phase (thread 0 of each state): 0 theta build, 1 QRCP + R^H,
// 2 Jacobi, 3 norms + truncation, 4 C-side write + replay, 5 Q application,
// 6 W-side write, 7 QR moves
__device__ unsigned long long g_dbg_cyc[8] = {};
#define MPSKQ_DBG_T(var) const long long var = clock64()
#define MPSKQ_DBG_ADD(slot, t0) \
  if (ltid<NT>() == 0) atomicAdd(&g_dbg_cyc[slot], (unsigned long long)(clock64() - (t0)))
#else
#define MPSKQ_DBG_T(var)
#define MPSKQ_DBG_ADD(slot, t0)
#endif

// thread index within the state's thread group: NT <= 32 kernels carry one
// state per NT-lane slice of a warp (several lockstepped groups per CTA),
// larger NT one state per CTA
template <int NT>
__device__ __forceinline__ int ltid() {
  if constexpr (NT <= 32)
    return threadIdx.x & (NT - 1);
  else
    return threadIdx.x;
}

template <int CAP>
struct NtFor {
  static constexpr int value =
      CAP <= 4 ? MPSKQ_NT4 : CAP <= 8 ? MPSKQ_NT8 : CAP <= 16 ? MPSKQ_NT16 : CAP <= 32 ? MPSKQ_NT32 : CAP <= 48 ? MPSKQ_NT48 : CAP <= 96 ? MPSKQ_NT96 : MPSKQ_NT128;
  // the Jacobi pairs every column (G lanes per pair, G * n/2 <= NT) and
  // several passes take one lane per column
  static_assert(value >= 2 * CAP, "a state needs at least 2 * CAP threads");
};

// Capacities above 12: theta/C, the staging buffer and W live in a per-CTA
// global scratch (L2 resident), only the small per-op arrays in shared
// memory, so residency is set by registers, not by the 2CAP x 2CAP planes:
// d=6 (cap 48) 5.14 -> 3.25 s, plus 3 CTAs per SM at 192 threads -> 2.19 s;
// d=5 (cap 32) 2.56 -> 1.63 s; d=4 (cap 24) 1.43 -> 1.17 s; with 64 threads
// per state at capacities 12-32 (d=5 1.31 s, d=4 0.81 s, d=3 0.35 -> 0.27 s)
// (`profiles/r02_ab_sim_global_ws.txt`).  Up to capacity 64 W gets its own
// plane there and is accumulated during the Jacobi (no rotation log, no
// replay): d=7 sim 6.34 -> 5.48 s.  At 96 and 128 the same change measured
// neutral / +2% (the per-round W rotation over 2*CAP rows costs what the
// replay saved), so they keep the log.
#ifndef MPSKQ_DIRECT_W_MAX
#define MPSKQ_DIRECT_W_MAX 64  // A/B knob
#endif
#ifndef MPSKQ_GLOBAL_WS_ABOVE
#define MPSKQ_GLOBAL_WS_ABOVE 12  // A/B knob
#endif
template <int CAP>
struct GlobalWs {
  // per-CTA slices: needs one state per CTA (NT > 32)
  static constexpr bool value = CAP > MPSKQ_GLOBAL_WS_ABOVE && NtFor<CAP>::value > 32;
  static constexpr bool direct_w = value && CAP <= MPSKQ_DIRECT_W_MAX;
  static constexpr int64_t complexes =
      (direct_w ? 2 : 1) * (int64_t)(2 * CAP) * (2 * CAP) + 2 * (int64_t)CAP * CAP;
};

// Capacities 80-128 keep only theta/C and the staging buffer: the Jacobi
// rotations are logged to a per-CTA global buffer and replayed on the identity
// after the C-side factor has been written out (W then reuses C's space).
// (With W in shared memory, capacities 24 and 32 gained from the log too:
// d=5 3.38 -> 2.56 s; the global workspace above superseded that.)  The log
// is per CTA, so it needs one state per CTA (NT > 32).
#ifndef MPSKQ_LOGW_ABOVE
#define MPSKQ_LOGW_ABOVE 16  // capacities above this log the Jacobi rotations (A/B knob)
#endif
template <int CAP>
struct LogW {
  static constexpr bool value = CAP > MPSKQ_LOGW_ABOVE && !GlobalWs<CAP>::direct_w && NtFor<CAP>::value > 32;
  static constexpr int64_t entries = (int64_t)kMaxSweeps * (2 * CAP) * CAP;  // sweeps x rounds x pairs
};

// shared-memory carve-out of one CTA
template <int CAP, int NT>
struct Smem {
  static constexpr int LD = 2 * CAP;
  double2* A;    // LD x LD, column-major: theta / C / QR workspace
  double2* W;    // LD x LD, column-major: Jacobi rotations / Q / staging
  double2* S;    // 2*CAP*CAP: staging of the neighbour site during QR moves
  double2* rd;   // LD: diagonal of R
  double2* ud;   // LD: diagonal entries of the pivoted QR's reflectors
  double* tau;   // LD
  double* sig;   // LD
  double* red;   // kRed
  static constexpr int kRedHalf = NT / 32 > 16 ? NT / 32 : 16;  // warps of the group (>= 16)
  static constexpr int kRed = 2 * kRedHalf;
  double* scal;  // 8: factor, discarded, -, op start clock, nominal flops, 3 phase cycle sums
  int* perm;     // LD
  int* piv;      // LD: inverse column order of the pivoted QR
  int* ibuf;     // 4: keep
  int* chi;      // m + 1
  double4* rlog;  // per-CTA rotation log (LogW capacities only)

  __host__ __device__ static size_t bytes(int m) {
    size_t b = GlobalWs<CAP>::value
                   ? sizeof(double2) * 2 * LD
                   : sizeof(double2) * ((LogW<CAP>::value ? 1 : 2) * LD * LD + 2 * CAP * CAP + 2 * LD);
    b += sizeof(double) * (2 * LD + kRed + 8);
    b += sizeof(int) * (2 * LD + 4 + m + 1);
    return (b + 15) & ~size_t(15);
  }
  // gws: this CTA's global workspace (capacities > 48 only)
  __device__ void carve(void* base, int m, double2* gws = nullptr) {
    char* p = static_cast<char*>(base);
    if constexpr (GlobalWs<CAP>::value) {
      A = gws;
      S = gws + LD * LD;
      W = GlobalWs<CAP>::direct_w ? S + 2 * CAP * CAP : S;
    } else {
      A = reinterpret_cast<double2*>(p);
      p += sizeof(double2) * LD * LD;
      if constexpr (!LogW<CAP>::value) {
        W = reinterpret_cast<double2*>(p);
        p += sizeof(double2) * LD * LD;
      }
      S = reinterpret_cast<double2*>(p);
      if constexpr (LogW<CAP>::value) W = S;  // Q of a QR move (Rr x k <= 2CAP x CAP)
      p += sizeof(double2) * 2 * CAP * CAP;
    }
    rd = reinterpret_cast<double2*>(p);
    p += sizeof(double2) * LD;
    ud = reinterpret_cast<double2*>(p);
    p += sizeof(double2) * LD;
    tau = reinterpret_cast<double*>(p);
    p += sizeof(double) * LD;
    sig = reinterpret_cast<double*>(p);
    p += sizeof(double) * LD;
    red = reinterpret_cast<double*>(p);
    p += sizeof(double) * kRed;
    scal = reinterpret_cast<double*>(p);
    p += sizeof(double) * 8;
    perm = reinterpret_cast<int*>(p);
    p += sizeof(int) * LD;
    piv = reinterpret_cast<int*>(p);
    p += sizeof(int) * LD;
    ibuf = reinterpret_cast<int*>(p);
    p += sizeof(int) * 4;
    chi = reinterpret_cast<int*>(p);
    rlog = nullptr;
    (void)m;
  }
};

// ---------------------------------------------------------------------------
// Householder QR of the Rr x Cc matrix held column-major in A (ld LD).
// Unitary reflectors H = I - tau u u^H (u stored in A's lower part, R's
// diagonal in rd, R's strict upper part left in A); Q (Rr x k, k = min(Rr,Cc))
// is formed in W.  This is the reduced QR of np.linalg.qr (mps.py:109, :118):
// same shapes; the column phases of Q may differ, which leaves the state and
// its Schmidt spectra unchanged.
template <int CAP, int NT>
__device__ void apply_reflector(double2* M, const double2* u, double tau, int j, int Rr, int c0,
                                int c1) {
  constexpr int LD = 2 * CAP;
  const int nc = c1 - c0;
  if (nc <= 0 || tau == 0.0) return;
  const int G = group_width<NT>(nc);
  const int per = NT / G;
  const int tid = ltid<NT>();
  for (int base = 0; base < nc; base += per) {
    const int ci = base + tid / G, g = tid % G;
    const bool act = ci < nc;
    const int c = c0 + (act ? ci : 0);
    double2 acc = cz();
    if (act)
      #pragma unroll 1
      for (int r = j + g; r < Rr; r += G) acc = cfmac(u[r], M[c * LD + r], acc);
    acc = group_sum(acc, G, group_mask<NT>());
    if (act) {
      const double2 w = cscale(acc, tau);
      #pragma unroll 1
      for (int r = j + g; r < Rr; r += G) M[c * LD + r] = csub(M[c * LD + r], cmul(u[r], w));
    }
  }
}

template <int CAP, int NT>
__device__ __noinline__ int householder_qr(Smem<CAP, NT>& sm, int Rr, int Cc) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int k = min(Rr, Cc);
  double2* A = sm.A;
  for (int j = 0; j < k; ++j) {
    double part = 0.0;
    #pragma unroll 1
    for (int r = j + tid; r < Rr; r += NT) part += cnorm2(A[j * LD + r]);
    const double nx2 = block_sum<NT>(part, sm.red);
    if (tid == 0) {
      const double nx = sqrt(nx2);
      const double2 x1 = A[j * LD + j];
      const double ax1 = hypot(x1.x, x1.y);
      if (nx == 0.0) {
        sm.tau[j] = 0.0;
        sm.rd[j] = cz();
      } else {
        const double2 ph = ax1 > 0.0 ? make_double2(x1.x / ax1, x1.y / ax1) : make_double2(1.0, 0.0);
        A[j * LD + j] = make_double2(x1.x + ph.x * nx, x1.y + ph.y * nx);
        sm.tau[j] = 1.0 / (nx * (nx + ax1));
        sm.rd[j] = make_double2(-ph.x * nx, -ph.y * nx);
      }
    }
    bsync<NT>();
    apply_reflector<CAP, NT>(A, A + j * LD, sm.tau[j], j, Rr, j + 1, Cc);
    bsync<NT>();
  }
  // Q = H_0 ... H_{k-1} [I_k; 0]
  #pragma unroll 1
  for (int idx = tid; idx < Rr * k; idx += NT) {
    const int c = idx / Rr, r = idx % Rr;
    sm.W[c * LD + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  bsync<NT>();
  for (int j = k - 1; j >= 0; --j) {
    apply_reflector<CAP, NT>(sm.W, A + j * LD, sm.tau[j], j, Rr, j, k);
    bsync<NT>();
  }
  return k;
}

// R(kk, c) of the last householder_qr (upper trapezoidal)
template <int CAP, int NT>
__device__ __forceinline__ double2 r_entry(const Smem<CAP, NT>& sm, int kk, int c) {
  constexpr int LD = 2 * CAP;
  return c == kk ? sm.rd[kk] : sm.A[c * LD + kk];
}

// ---------------------------------------------------------------------------
// QR-preconditioned SVD (Drmac-Veselic): for the Jacobi input C (Rr x n) the
// two-qubit step factors B = C^H with column pivoting, B P = Q R, and runs the
// one-sided Jacobi on X = R^H (Rr x k), which is close to column-orthogonal
// already: 6-7 sweeps instead of 13-20 on the 60..90-column thetas of d = 8
// (numpy replica of this Jacobi on reference thetas).  With X W' = Z:
//   C = P R^H Q^H = (P Z) (Q W')^H,
// so the scaled side is P Z (rows permuted) and the orthonormal side Q W'
// (reflectors applied to W'), the same roles C W and W play unpreconditioned.

// group-wide argmax of (v, idx), ties to the smaller idx; `red` needs Smem::kRed doubles
template <int NT>
__device__ __forceinline__ int block_argmax(double v, int idx, double* red) {
  const unsigned mask = group_mask<NT>();
  constexpr int G = NT < 32 ? NT : 32;
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(mask, v, o);
    const int oi = __shfl_xor_sync(mask, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if constexpr (NT > 32) {
    constexpr int H = NT / 32 > 16 ? NT / 32 : 16;  // Smem::kRedHalf
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      red[w] = v;
      red[H + w] = (double)idx;
    }
    __syncthreads();
    v = red[0];
    idx = (int)red[H];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) {
      const double ov = red[i];
      const int oi = (int)red[H + i];
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
  }
  return idx;
}

// packed offset of reflector j's strictly-lower part (rows j+1..nr-1)
__device__ __forceinline__ int refl_off(int j, int nr) { return j * (nr - 1) - ((j * (j - 1)) >> 1); }

// Householder QR with column pivoting of B (nr x nc, column-major in A):
// B P = Q R.  Pivot = largest trailing column norm (recomputed exactly in the
// update pass), ties to the lower index.  On return: R's strict upper part in
// A, its diagonal in rd; reflector j is ud[j] (row j) and S[refl_off(j)...]
// (rows j+1..nr-1) with tau[j]; piv[c] = position of original column c.
template <int CAP, int NT>
__device__ __noinline__ int householder_qrcp(Smem<CAP, NT>& sm, int nr, int nc) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int k = min(nr, nc);
  const unsigned msk = group_mask<NT>();
  double2* A = sm.A;
  {
    const int G = group_width<NT>(nc), per = NT / G;
    for (int base = 0; base < nc; base += per) {
      const int c = base + tid / G, g = tid % G;
      double acc = 0.0;
      if (c < nc)
        #pragma unroll 1
        for (int r = g; r < nr; r += G) acc += cnorm2(A[c * LD + r]);
      acc = group_sum(acc, G, msk);
      if (c < nc && g == 0) {
        sm.sig[c] = acc;
        sm.perm[c] = c;  // original column at each position
      }
    }
  }
  bsync<NT>();
  for (int j = 0; j < k; ++j) {
    double bv = -1.0;
    int bi = 1 << 30;
    #pragma unroll 1
    for (int c = j + tid; c < nc; c += NT) {
      const double v = sm.sig[c];
      if (v > bv) {
        bv = v;
        bi = c;
      }
    }
    const int pv = block_argmax<NT>(bv, bi, sm.red);
    // every thread reads the pivot's trailing norm and leading entry before the
    // swap and derives the reflector itself: one barrier per step fewer
    const double nx2 = sm.sig[pv];
    const double2 x1 = A[pv * LD + j];
    if (pv != j) {
      bsync<NT>();  // everyone has read sig[pv] / x1
      #pragma unroll 1
      for (int r = tid; r < nr; r += NT) {
        const double2 t = A[j * LD + r];
        A[j * LD + r] = A[pv * LD + r];
        A[pv * LD + r] = t;
      }
      if (tid == 0) {
        sm.sig[pv] = sm.sig[j];
        const int tp = sm.perm[j];
        sm.perm[j] = sm.perm[pv];
        sm.perm[pv] = tp;
      }
    }
    const double nx = sqrt(nx2);
    const double ax1 = hypot(x1.x, x1.y);
    double tau = 0.0;
    double2 uj = x1;
    if (nx > 0.0) {
      const double2 ph = ax1 > 0.0 ? make_double2(x1.x / ax1, x1.y / ax1) : make_double2(1.0, 0.0);
      uj = make_double2(x1.x + ph.x * nx, x1.y + ph.y * nx);
      tau = 1.0 / (nx * (nx + ax1));
      if (tid == 0) sm.rd[j] = make_double2(-ph.x * nx, -ph.y * nx);
    } else if (tid == 0) {
      sm.rd[j] = cz();
    }
    if (tid == 0) {
      sm.tau[j] = tau;
      sm.sig[j] = nx2;
    }
    bsync<NT>();  // the swap is complete
    if (tid == 0) A[j * LD + j] = uj;  // read below only through uj
    // apply H_j to columns j+1..nc-1 and refresh their trailing norms (rows > j)
    const int c0 = j + 1, ncols = nc - c0;
    if (ncols > 0) {
      const double2* u = A + j * LD;
      const int G = group_width<NT>(ncols), per = NT / G;
      for (int base = 0; base < ncols; base += per) {
        const int ci = base + tid / G, g = tid % G;
        const bool act = ci < ncols;
        const int c = c0 + (act ? ci : 0);
        double2 acc = cz();
        if (act && tau != 0.0)
          #pragma unroll 1
          for (int r = j + g; r < nr; r += G) acc = cfmac(r == j ? uj : u[r], A[c * LD + r], acc);
        acc = group_sum(acc, G, msk);
        double nrm = 0.0;
        if (act) {
          const double2 w = cscale(acc, tau);
          #pragma unroll 1
          for (int r = j + g; r < nr; r += G) {
            double2 v = A[c * LD + r];
            if (tau != 0.0) {
              v = csub(v, cmul(r == j ? uj : u[r], w));
              A[c * LD + r] = v;
            }
            if (r > j) nrm += cnorm2(v);
          }
        }
        nrm = group_sum(nrm, G, msk);
        if (act && g == 0) sm.sig[c] = nrm;
      }
    }
    bsync<NT>();
  }
  // stash the reflectors (A's lower part is about to hold R^H), invert the order
  #pragma unroll 1
  for (int idx = tid; idx < k * nr; idx += NT) {
    const int j = idx / nr, r = idx - j * nr;
    if (r == j)
      sm.ud[j] = A[j * LD + j];
    else if (r > j)
      sm.S[refl_off(j, nr) + r - j - 1] = A[j * LD + r];
  }
  #pragma unroll 1
  for (int c = tid; c < nc; c += NT) sm.piv[sm.perm[c]] = c;
  bsync<NT>();
  return k;
}

// A := R^H (nc x k, lower trapezoidal) from the QRCP's R (k x nc) in place
template <int CAP, int NT>
__device__ void form_rh(Smem<CAP, NT>& sm, int nc, int k) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  double2* A = sm.A;
  #pragma unroll 1
  for (int idx = tid; idx < k * nc; idx += NT) {
    const int j = idx / nc, c = idx - j * nc;
    if (c > j) A[j * LD + c] = cconj(A[c * LD + j]);  // R(j, c) lives in row j, column c
  }
  bsync<NT>();
  #pragma unroll 1
  for (int idx = tid; idx < k * k; idx += NT) {
    const int j = idx / k, c = idx - j * k;
    if (c < j)
      A[j * LD + c] = cz();
    else if (c == j)
      A[j * LD + j] = cconj(sm.rd[j]);
  }
  bsync<NT>();
}

// M (nr x kc, column-major, ld LD) := H_0 ... H_{k-1} M with the stashed reflectors
template <int CAP, int NT>
__device__ __noinline__ void apply_q_packed(Smem<CAP, NT>& sm, double2* M, int nr, int k, int kc) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const unsigned msk = group_mask<NT>();
  const int G = group_width<NT>(kc), per = NT / G;
  for (int j = k - 1; j >= 0; --j) {
    const double tau = sm.tau[j];
    if (tau == 0.0) continue;  // uniform
    const double2 u0 = sm.ud[j];
    const double2* us = sm.S + refl_off(j, nr) - j - 1;  // us[r] for r > j
    for (int base = 0; base < kc; base += per) {
      const int c = base + tid / G, g = tid % G;
      const bool act = c < kc;
      double2 acc = cz();
      if (act)
        #pragma unroll 1
        for (int r = j + g; r < nr; r += G) acc = cfmac(r == j ? u0 : us[r], M[c * LD + r], acc);
      acc = group_sum(acc, G, msk);
      if (act) {
        const double2 w = cscale(acc, tau);
        #pragma unroll 1
        for (int r = j + g; r < nr; r += G) M[c * LD + r] = csub(M[c * LD + r], cmul(r == j ? u0 : us[r], w));
      }
    }
    bsync<NT>();
  }
}

// ---------------------------------------------------------------------------
// One-sided Jacobi on C (Rr x n, column-major in A) accumulating the unitary
// W (n x n) with C_out = C_in W and mutually orthogonal columns of C_out.
// Column pairs follow the circle-method round robin (n/2 disjoint pairs per
// round, ne-1 rounds per sweep), one group of G lanes per pair.
template <int G>
__device__ __forceinline__ double gsum(double v, unsigned mask) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// round-robin pair of group k in round t (circle method: position 0 fixed,
// positions 1..ne-1 rotate by t); p < q
__device__ __forceinline__ void rr_pair(int k, int t, int ne, int& p, int& q) {
  const int span = ne - 1;
  const int pa = k, pb = ne - 1 - k;
  int x = pa - 1 + t, y = pb - 1 + t;
  x = x >= span ? x - span : x;
  y = y >= span ? y - span : y;
  p = pa == 0 ? 0 : 1 + x;
  q = 1 + y;
  if (p > q) {
    const int tmp = p;
    p = q;
    q = tmp;
  }
}

// Returns the number of rounds run (the log-mode replay repeats them).  The
// iteration stops once a full cycle of rounds (every pair once) has made no
// rotation, even mid-sweep.  (Tracking the column norms through rotations
// instead of recomputing them stalls convergence on the noise columns of
// rank-deficient thetas, so the norms are recomputed every round.)
template <int CAP, int NT, int G>
__device__ __noinline__ int jacobi_sweeps(Smem<CAP, NT>& sm, int Rr, int n) {
  constexpr bool kLog = LogW<CAP>::value;
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  double2* A = sm.A;
  double2* W = sm.W;
  const int ne = n + (n & 1), P = ne >> 1, span = ne - 1;
  const int k = tid / G, g = tid % G;
  // convergence: |c_p^H c_q| <= tol * |c_p| |c_q|, compared in squares
  const double tol = DBL_EPSILON * (double)max(Rr, 8);
  const double tol2 = tol * tol;
  const int max_rounds = kMaxSweeps * span;
  const unsigned msk = group_mask<NT>();
  // Pairs with a column below half the truncation noise floor are left alone:
  // such columns are zeroed by the floor (10 eps s0, tensor.py:108-109) and
  // cannot combine across it, and their coupling moves a kept sigma^2 by at
  // most |c_small|^2 <= (5 eps s0)^2 -- far below the LAPACK-vs-Jacobi
  // rounding already present -- but rotating on their rounding noise was what
  // kept large thetas sweeping (measured 12-15 sweeps at chi 17-44).
  // With n columns ||theta||_F^2 <= n s0^2, so the threshold
  // eps^2 ||theta||_F^2 / 4 * min(1, 100 / n) stays <= (5 eps s0)^2 for any n
  // (up to the 256 columns of capacity 128).
  double fro = 0.0;
  #pragma unroll 1
  for (int idx = tid; idx < Rr * n; idx += NT) {
    const int c = idx / Rr, r = idx - c * Rr;
    fro += cnorm2(A[c * LD + r]);
  }
  const double noise2 = 0.25 * DBL_EPSILON * DBL_EPSILON * block_sum<NT>(fro, sm.red) *
                        (MPSKQ_NOISE_SCALE_N && n > 100 ? 100.0 / n : 1.0);
  int round = 0, quiet = 0;
  for (; round < max_rounds;) {
    const int t = round % span;
    int p = 0, q = 0;
    if (k < P) rr_pair(k, t, ne, p, q);
    const bool act = k < P && q < n;
    double a = 0.0, b = 0.0, gx = 0.0, gy = 0.0;
    if (act) {
      int r = g;
      if constexpr (CAP >= 128) {
        // long columns (up to 256 rows over 4 lanes) streamed from L2: two
        // interleaved partial sums halve the dependent-FMA chain per round
        // (-11% at capacity 128; at 96 it measured 4% slower)
        double a1 = 0.0, b1 = 0.0, gx1 = 0.0, gy1 = 0.0;
        #pragma unroll 1
        for (; r + G < Rr; r += 2 * G) {
          const double2 x = A[p * LD + r], y = A[q * LD + r];
          const double2 x1 = A[p * LD + r + G], y1 = A[q * LD + r + G];
          a = fma(x.x, x.x, fma(x.y, x.y, a));
          b = fma(y.x, y.x, fma(y.y, y.y, b));
          gx = fma(x.x, y.x, fma(x.y, y.y, gx));
          gy = fma(x.x, y.y, fma(-x.y, y.x, gy));
          a1 = fma(x1.x, x1.x, fma(x1.y, x1.y, a1));
          b1 = fma(y1.x, y1.x, fma(y1.y, y1.y, b1));
          gx1 = fma(x1.x, y1.x, fma(x1.y, y1.y, gx1));
          gy1 = fma(x1.x, y1.y, fma(-x1.y, y1.x, gy1));
        }
        a += a1;
        b += b1;
        gx += gx1;
        gy += gy1;
      }
      #pragma unroll 1
      for (; r < Rr; r += G) {
        const double2 x = A[p * LD + r], y = A[q * LD + r];
        a = fma(x.x, x.x, fma(x.y, x.y, a));
        b = fma(y.x, y.x, fma(y.y, y.y, b));
        gx = fma(x.x, y.x, fma(x.y, y.y, gx));
        gy = fma(x.x, y.y, fma(-x.y, y.x, gy));
      }
    }
    a = gsum<G>(a, msk);
    b = gsum<G>(b, msk);
    gx = gsum<G>(gx, msk);
    gy = gsum<G>(gy, msk);
    const double g2 = fma(gx, gx, gy * gy);
    const bool rot = act && g2 > tol2 * a * b && g2 > 0.0 && fmin(a, b) > noise2;
    double4* entry = nullptr;
    if constexpr (kLog) entry = sm.rlog + (int64_t)round * P + k;
    if (kLog && act && g == 0 && !rot) *entry = make_double4(1.0, 0.0, 0.0, 0.0);
    if (rot) {
      const double inv = rsqrt(g2);  // 1/|gamma|
      const double zeta = (b - a) * (0.5 * inv);
      const double az = fabs(zeta);
      const double tt = az > 1e150 ? 0.5 / az : 1.0 / (az + sqrt(fma(zeta, zeta, 1.0)));
      const double t_ = copysign(tt, zeta);
      const double c = rsqrt(fma(t_, t_, 1.0));
      const double sn = c * t_;
      // [x', y'] = [x, y] J,  J = [[c, s e], [-s conj(e), c]],  e = gamma/|gamma|
      const double2 se = make_double2(sn * gx * inv, sn * gy * inv);
      #pragma unroll 1
      for (int r = g; r < Rr; r += G) {
        const double2 x = A[p * LD + r], y = A[q * LD + r];
        A[p * LD + r] = csub(cscale(x, c), cmul(cconj(se), y));
        A[q * LD + r] = cadd(cmul(se, x), cscale(y, c));
      }
      if constexpr (kLog) {
        if (g == 0) *entry = make_double4(c, se.x, se.y, 1.0);
      } else {
        #pragma unroll 1
        for (int r = g; r < n; r += G) {
          const double2 x = W[p * LD + r], y = W[q * LD + r];
          W[p * LD + r] = csub(cscale(x, c), cmul(cconj(se), y));
          W[q * LD + r] = cadd(cmul(se, x), cscale(y, c));
        }
      }
    }
    ++round;
    quiet = block_any<NT>(rot) ? 0 : quiet + 1;
    if (quiet >= span) return round;
  }
  return round | kNoConvergence;  // no quiet cycle within kMaxSweeps sweeps
}

// Log mode: W = I_n in `Wm`, then apply the logged rotations in order.
template <int CAP, int NT, int G>
__device__ __noinline__ void replay_sweeps(Smem<CAP, NT>& sm, double2* Wm, int n, int rounds) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int ne = n + (n & 1), P = ne >> 1, span = ne - 1;
  const int k = tid / G, g = tid % G;
  for (int round = 0; round < rounds; ++round) {
    int p = 0, q = 0;
    if (k < P) rr_pair(k, round % span, ne, p, q);
    if (k < P && q < n) {
      const double4 e = sm.rlog[(int64_t)round * P + k];
      if (e.w != 0.0) {
        const double c = e.x;
        const double2 se = make_double2(e.y, e.z);
        #pragma unroll 1
        for (int r = g; r < n; r += G) {
          const double2 x = Wm[p * LD + r], y = Wm[q * LD + r];
          Wm[p * LD + r] = csub(cscale(x, c), cmul(cconj(se), y));
          Wm[q * LD + r] = cadd(cmul(se, x), cscale(y, c));
        }
      }
    }
    bsync<NT>();
  }
}

template <int CAP, int NT>
__device__ void init_identity(double2* Wm, int n) {
  constexpr int LD = 2 * CAP;
  #pragma unroll 1
  for (int idx = ltid<NT>(); idx < n * n; idx += NT) {
    const int c = idx / n, r = idx - c * n;
    Wm[c * LD + r] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
  bsync<NT>();
}

// returns the number of rounds run (needed by the log-mode replay)
template <int CAP, int NT>
__device__ int jacobi(Smem<CAP, NT>& sm, int Rr, int n) {
  if constexpr (!LogW<CAP>::value) init_identity<CAP, NT>(sm.W, n);
  if (n < 2) return 0;
  // lanes per column pair: G * (n/2) <= NT, G in {2, 4, 8, 16, 32} for every
  // (CAP, NT) instantiation (NT >= 2 * CAP)
  const int G = group_width<NT>((n + 1) >> 1);
  if (G >= 32) return jacobi_sweeps<CAP, NT, 32>(sm, Rr, n);
  if (G == 16) return jacobi_sweeps<CAP, NT, 16>(sm, Rr, n);
  if (G == 8) return jacobi_sweeps<CAP, NT, 8>(sm, Rr, n);
  if (G == 4) return jacobi_sweeps<CAP, NT, 4>(sm, Rr, n);
  return jacobi_sweeps<CAP, NT, 2>(sm, Rr, n);
}

// log mode: rebuild W (n x n) in Wm from the rotation log
template <int CAP, int NT>
__device__ void replay(Smem<CAP, NT>& sm, double2* Wm, int n, int sweeps) {
  init_identity<CAP, NT>(Wm, n);
  if (n < 2) return;
  const int G = group_width<NT>((n + 1) >> 1);
  if (G >= 32)
    replay_sweeps<CAP, NT, 32>(sm, Wm, n, sweeps);
  else if (G == 16)
    replay_sweeps<CAP, NT, 16>(sm, Wm, n, sweeps);
  else if (G == 8)
    replay_sweeps<CAP, NT, 8>(sm, Wm, n, sweeps);
  else if (G == 4)
    replay_sweeps<CAP, NT, 4>(sm, Wm, n, sweeps);
  else
    replay_sweeps<CAP, NT, 2>(sm, Wm, n, sweeps);
}

// column norms of C, descending order in perm (ties keep index order)
template <int CAP, int NT>
__device__ __noinline__ void norms_and_order(Smem<CAP, NT>& sm, int Rr, int n) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int G = group_width<NT>(n);
  const int per = NT / G;
  for (int base = 0; base < n; base += per) {
    const int c = base + tid / G, g = tid % G;
    double acc = 0.0;
    if (c < n)
      #pragma unroll 1
      for (int r = g; r < Rr; r += G) acc += cnorm2(sm.A[c * LD + r]);
    acc = group_sum(acc, G, group_mask<NT>());
    if (c < n && g == 0) sm.sig[c] = sqrt(acc);
  }
  bsync<NT>();
  #pragma unroll 1
  for (int j = tid; j < n; j += NT) {
    const double sj = sm.sig[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double si = sm.sig[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    sm.perm[rank] = j;
  }
  bsync<NT>();
}

// svd_truncated's rule (tensor.py:108-116) on the kmin leading sorted values,
// plus the renormalisation factor of apply_two_qubit (mps.py:189-192).
// Runs on one thread; writes keep to ibuf[0] and factor/discarded to scal[0..1].
template <int CAP, int NT>
__device__ __noinline__ void truncation_rule(Smem<CAP, NT>& sm, int kmin, double budget, int chi_max) {
  double v[2 * CAP];
  const double s0 = sm.sig[sm.perm[0]];
  for (int i = 0; i < kmin; ++i) {
    double x = sm.sig[sm.perm[i]];
    if (s0 > 0.0 && x < kNoiseFloor * s0) x = 0.0;
    v[i] = x;
  }
  // tail[i] = sum_{j>=i} s_j^2 accumulated from the end (np.cumsum of the
  // reversed squares); keep = first i with tail[i] <= budget
  int keep = kmin;
  double acc = 0.0;
  for (int i = kmin - 1; i >= 0; --i) {
    acc += v[i] * v[i];
    if (acc <= budget)
      keep = i;
    else
      break;
  }
  keep = max(keep, 1);
  if (chi_max > 0) keep = min(keep, chi_max);
  double disc = 0.0;
  for (int i = keep; i < kmin; ++i) disc += v[i] * v[i];
  double kept = 0.0;
  for (int i = 0; i < keep; ++i) kept += v[i] * v[i];
  double factor = 1.0;
  if (disc > 0.0) factor = sqrt((kept + disc) / kept);
  sm.ibuf[0] = keep;
  sm.scal[0] = factor;
  sm.scal[1] = disc;
}

// ---------------------------------------------------------------------------
struct StateCtx {
  double2* base;
  const int64_t* off;
  int m;
  int status;
  int peak;
  double discard;
};

// Nominal flops of one apply_two_qubit (fixed here once): theta
// = site_q . site_{q+1} (8 * 2chl * chm * 2chr), the 4x4 gate (128 chl chr),
// thin SVD of the (2chl x 2chr) theta, 8 (4 M N^2 + 8 N^3) with M >= N.
__device__ __forceinline__ double nominal_two_qubit(int chl, int chm, int chr) {
  const double a = 2.0 * chl, b = 2.0 * chr, M = fmax(a, b), N = fmin(a, b);
  return 8.0 * a * chm * b + 128.0 * chl * chr + 8.0 * (4.0 * M * N * N + 8.0 * N * N * N);
}
// one QR move: Householder QR of an (M x N) matrix 8 * 2 M N^2 plus the R push
// into the neighbour (8 * k * N * cols)
__device__ __forceinline__ double nominal_qr(int M, int N, int k, int cols) {
  return 16.0 * M * (double)N * N + 8.0 * k * (double)N * cols;
}

template <int CAP, int NT, bool GEN>
__device__ void op_one_qubit(Smem<CAP, NT>& sm, StateCtx& st, int q, int code, double2 cs,
                             const double2* gm) {
  const int chl = sm.chi[q], chr = sm.chi[q + 1];
  double2* p = st.base + st.off[q];
  const int n = chl * chr;
  #pragma unroll 1
  for (int idx = ltid<NT>(); idx < n; idx += NT) {
    const int a = idx / chr, b = idx - a * chr;
    const int i0 = (2 * a) * chr + b, i1 = i0 + chr;
    const double2 x0 = p[i0], x1 = p[i1];
    if (GEN && code == MPSKQ_OP_U1) {
      // arbitrary 2x2 matrix U (row-major in the coefficient row):
      // site <- tensordot(U, site, (1, 1)).transpose(1, 0, 2)  (mps.py:157)
      const double2 u00 = gm[0], u01 = gm[1], u10 = gm[2], u11 = gm[3];
      p[i0] = cfma(u01, x1, cmul(u00, x0));
      p[i1] = cfma(u11, x1, cmul(u10, x0));
    } else if (code == MPSKQ_OP_H) {
      const double h = kInvSqrt2;
      p[i0] = make_double2(__dadd_rn(__dmul_rn(h, x0.x), __dmul_rn(h, x1.x)),
                           __dadd_rn(__dmul_rn(h, x0.y), __dmul_rn(h, x1.y)));
      p[i1] = make_double2(__dsub_rn(__dmul_rn(h, x0.x), __dmul_rn(h, x1.x)),
                           __dsub_rn(__dmul_rn(h, x0.y), __dmul_rn(h, x1.y)));
    } else {
      // RZ = diag(c - i s, c + i s)
      const double c = cs.x, s = cs.y;
      p[i0] = make_double2(__dadd_rn(__dmul_rn(c, x0.x), __dmul_rn(s, x0.y)),
                           __dsub_rn(__dmul_rn(c, x0.y), __dmul_rn(s, x0.x)));
      p[i1] = make_double2(__dsub_rn(__dmul_rn(c, x1.x), __dmul_rn(s, x1.y)),
                           __dadd_rn(__dmul_rn(c, x1.y), __dmul_rn(s, x1.x)));
    }
  }
  bsync<NT>();
}

// _left_isometrize step at site i (mps.py:105-111)
template <int CAP, int NT>
__device__ void op_qr_left(Smem<CAP, NT>& sm, StateCtx& st, int i) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int chl = sm.chi[i], chr = sm.chi[i + 1], chn = sm.chi[i + 2];
  double2* M = st.base + st.off[i];
  double2* N = st.base + st.off[i + 1];
  const int Rr = 2 * chl;
  #pragma unroll 1
  for (int idx = tid; idx < Rr * chr; idx += NT) {
    const int r = idx / chr, c = idx - r * chr;
    sm.A[c * LD + r] = M[idx];
  }
  bsync<NT>();
  const int k = householder_qr<CAP, NT>(sm, Rr, chr);
  #pragma unroll 1
  for (int idx = tid; idx < Rr * k; idx += NT) {
    const int r = idx / k, c = idx - r * k;
    M[idx] = sm.W[c * LD + r];
  }
  bsync<NT>();  // Q is out: W may alias S (capacities > 32)
  const int nn = chr * 2 * chn;
  #pragma unroll 1
  for (int idx = tid; idx < nn; idx += NT) sm.S[idx] = N[idx];
  bsync<NT>();
  const int cols = 2 * chn;
  #pragma unroll 1
  for (int idx = tid; idx < k * cols; idx += NT) {
    const int kk = idx / cols, col = idx - kk * cols;
    double2 acc = cz();
    for (int c = kk; c < chr; ++c) acc = cfma(r_entry(sm, kk, c), sm.S[c * cols + col], acc);
    N[idx] = acc;
  }
  bsync<NT>();
  if (tid == 0) {
    sm.chi[i + 1] = k;
    sm.scal[4] += nominal_qr(Rr, chr, k, cols);  // nominal flops, per state
  }
  bsync<NT>();
}

// _right_isometrize step at site i (mps.py:114-120)
template <int CAP, int NT>
__device__ void op_qr_right(Smem<CAP, NT>& sm, StateCtx& st, int i) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int chp = sm.chi[i - 1], chl = sm.chi[i], chr = sm.chi[i + 1];
  double2* M = st.base + st.off[i];
  double2* P = st.base + st.off[i - 1];
  const int Rr = 2 * chr;  // rows of M^H
  #pragma unroll 1
  for (int idx = tid; idx < chl * Rr; idx += NT) {
    const int c = idx / Rr, r = idx - c * Rr;
    sm.A[c * LD + r] = cconj(M[idx]);
  }
  bsync<NT>();
  const int k = householder_qr<CAP, NT>(sm, Rr, chl);
  #pragma unroll 1
  for (int idx = tid; idx < k * Rr; idx += NT) {
    const int kk = idx / Rr, r = idx - kk * Rr;
    M[idx] = cconj(sm.W[kk * LD + r]);
  }
  bsync<NT>();  // Q is out: W may alias S (capacities > 32)
  const int np = 2 * chp * chl;
  #pragma unroll 1
  for (int idx = tid; idx < np; idx += NT) sm.S[idx] = P[idx];
  bsync<NT>();
  const int rows = 2 * chp;
  #pragma unroll 1
  for (int idx = tid; idx < rows * k; idx += NT) {
    const int row = idx / k, kk = idx - row * k;
    double2 acc = cz();
    for (int c = kk; c < chl; ++c) acc = cfma(sm.S[row * chl + c], cconj(r_entry(sm, kk, c)), acc);
    P[idx] = acc;
  }
  bsync<NT>();
  if (tid == 0) {
    sm.chi[i] = k;
    sm.scal[4] += nominal_qr(Rr, chl, k, rows);
  }
  bsync<NT>();
}

// apply_two_qubit at (q, q+1) after canonicalize(q) (mps.py:163-205)
template <int CAP, int NT, bool GEN>
__device__ void op_two_qubit(Smem<CAP, NT>& sm, StateCtx& st, int q, int code, bool left,
                             double2 cs, const double2* gm, double budget, int chi_max) {
  constexpr int LD = 2 * CAP;
  const int tid = ltid<NT>();
  const int chl = sm.chi[q], chm = sm.chi[q + 1], chr = sm.chi[q + 2];
  double2* X = st.base + st.off[q];
  double2* Y = st.base + st.off[q + 1];
  const int Mr = 2 * chl, Nc = 2 * chr;
  constexpr bool kLog = LogW<CAP>::value;
  MPSKQ_DBG_T(t_build);
  const double2* Xs = X;  // capacities > 32 read the sites straight from L1/L2
  const double2* Ys = Y;
  if constexpr (!kLog) {
    double2* xs = sm.W;
    double2* ys = sm.W + 2 * CAP * CAP;
    #pragma unroll 1
    for (int idx = tid; idx < Mr * chm; idx += NT) xs[idx] = X[idx];
    #pragma unroll 1
    for (int idx = tid; idx < chm * Nc; idx += NT) ys[idx] = Y[idx];
    bsync<NT>();
    Xs = xs;
    Ys = ys;
  }
  // theta = site_q . site_{q+1} (mps.py:183), gate on the physical legs
  // (:184-186); every item produces the two entries the gate couples.
  const double c = cs.x, s = cs.y;
  const bool rxx = code == MPSKQ_OP_RXX;
  const int Rr = left ? Mr : Nc;
  const int n = left ? Nc : Mr;
  const int kmin = min(Mr, Nc);
  const bool pre = kPrecondition<CAP>::value && kmin >= kPrecondMinCols;
  const bool theta_cm = left != pre;  // store C (not preconditioned) or C^H
  int bad = 0;
  if (GEN && code == MPSKQ_OP_U2) {
    // arbitrary 4x4 matrix G on |p0 p1> (row-major in the coefficient row):
    // theta'(l, p0', p1', r) = sum G[p0'p1'][p0 p1] theta(l, p0, p1, r)
    // (mps.py:184-186); one item per (l, r) couples all four physical entries
    #pragma unroll 1
    for (int lr = tid; lr < chl * chr; lr += NT) {
      const int l = lr / chr, rr = lr - l * chr;
      double2 T[4] = {cz(), cz(), cz(), cz()};
      for (int k = 0; k < chm; ++k)
        #pragma unroll
        for (int pp = 0; pp < 4; ++pp)
          T[pp] = cfma(Xs[(2 * l + (pp >> 1)) * chm + k], Ys[k * Nc + (pp & 1) * chr + rr], T[pp]);
      #pragma unroll
      for (int po = 0; po < 4; ++po) {
        double2 o = cz();
        #pragma unroll
        for (int pp = 0; pp < 4; ++pp) o = cfma(gm[po * 4 + pp], T[pp], o);
        bad |= !cfinite(o);
        const int row = 2 * l + (po >> 1), col = (po & 1) * chr + rr;
        if (theta_cm)
          sm.A[col * LD + row] = o;
        else
          sm.A[row * LD + col] = cconj(o);
      }
    }
  }
  #pragma unroll 1
  for (int it = tid; it < (GEN && code == MPSKQ_OP_U2 ? 0 : chl * chr * 2); it += NT) {
    const int t = it & 1, lr = it >> 1;
    const int l = lr / chr, rr = lr - l * chr;
    const int p0a = 0, p1a = t;
    const int row1 = 2 * l + p0a, col1 = p1a * chr + rr;
    const int row2 = 2 * l + 1 - p0a, col2 = (1 - p1a) * chr + rr;
    double2 T1 = cz(), T2 = cz();
    for (int k = 0; k < chm; ++k) {
      T1 = cfma(Xs[row1 * chm + k], Ys[k * Nc + col1], T1);
      T2 = cfma(Xs[row2 * chm + k], Ys[k * Nc + col2], T2);
    }
    double2 o1, o2;
    if (rxx) {
      // RXX = c I - i s XX: |p0 p1> couples to |1-p0 1-p1>
      o1 = make_double2(fma(c, T1.x, s * T2.y), fma(c, T1.y, -s * T2.x));
      o2 = make_double2(fma(c, T2.x, s * T1.y), fma(c, T2.y, -s * T1.x));
    } else if (t == 0) {  // SWAP: out(p0, p1) = theta(p1, p0)
      o1 = T1;
      o2 = T2;
    } else {
      o1 = T2;
      o2 = T1;
    }
    bad |= !(cfinite(o1) && cfinite(o2));
    if (theta_cm) {  // theta, column-major
      sm.A[col1 * LD + row1] = o1;
      sm.A[col2 * LD + row2] = o2;
    } else {  // theta^H, column-major
      sm.A[row1 * LD + col1] = cconj(o1);
      sm.A[row2 * LD + col2] = cconj(o2);
    }
  }
  if (block_any<NT>(bad)) {
    st.status = MPSKQ_STATE_NONFINITE;
    return;
  }
  // Jacobi input C: left: theta V = U S  (W = V);  right: theta^H U = V S  (W = U).
  // Preconditioned: A holds B = C^H; QRCP, then the Jacobi runs on R^H.
  MPSKQ_DBG_ADD(0, t_build);
  MPSKQ_DBG_T(t_qr);
  int ncol = n;
  if (pre) {
    householder_qrcp<CAP, NT>(sm, n, Rr);
    form_rh<CAP, NT>(sm, Rr, kmin);
    ncol = kmin;
  }
  MPSKQ_DBG_ADD(1, t_qr);
  MPSKQ_DBG_T(t_jac);
  int sweeps = jacobi<CAP, NT>(sm, Rr, ncol);
  if (sweeps & kNoConvergence) {  // LinAlgError in the reference (zgesdd)
    st.status = MPSKQ_STATE_NOCONV;
    return;
  }
  MPSKQ_DBG_ADD(2, t_jac);
  MPSKQ_DBG_T(t_trunc);
#ifdef MPSKQ_DEBUG_COUNTERS
  if (tid == 0) {
    atomicAdd(&g_dbg_rounds, (unsigned long long)sweeps);
    atomicAdd(&g_dbg_svds, 1ull);
    atomicAdd(&g_dbg_span, (unsigned long long)(ncol + (ncol & 1) - 1));
  }
#endif
  norms_and_order<CAP, NT>(sm, Rr, ncol);
  if (tid == 0) truncation_rule<CAP, NT>(sm, kmin, budget, chi_max);
  bsync<NT>();
  const int keep = sm.ibuf[0];
  const double factor = sm.scal[0];
  MPSKQ_DBG_ADD(3, t_trunc);
  MPSKQ_DBG_T(t_cside);
  if (keep > CAP) {
    st.status = MPSKQ_STATE_CAPACITY;
    return;
  }
  // C side first (it lives in A), then W (log mode rebuilds it in A).
  // Preconditioned, row r of C is row piv[r] of the rotated R^H.
  if (left) {
    // site_q = U s (mps.py:194)
    #pragma unroll 1
    for (int idx = tid; idx < Mr * keep; idx += NT) {
      const int row = idx / keep, kk = idx - row * keep;
      X[idx] = cscale(sm.A[sm.perm[kk] * LD + (pre ? sm.piv[row] : row)], factor);
    }
  } else {
    // site_{q+1} = s Vh (mps.py:197-199)
    #pragma unroll 1
    for (int idx = tid; idx < keep * Nc; idx += NT) {
      const int kk = idx / Nc, col = idx - kk * Nc;
      Y[idx] = cscale(cconj(sm.A[sm.perm[kk] * LD + (pre ? sm.piv[col] : col)]), factor);
    }
  }
  double2* Wm = sm.W;
  if constexpr (kLog) {
    bsync<NT>();
    replay<CAP, NT>(sm, sm.A, ncol, sweeps);
    Wm = sm.A;
  }
  MPSKQ_DBG_ADD(4, t_cside);
  MPSKQ_DBG_T(t_q);
  if (pre) {
    // W = Q [W'; 0] (n x kmin)
    const int extra = n - kmin;
    #pragma unroll 1
    for (int idx = tid; idx < extra * kmin; idx += NT) {
      const int cc = idx / extra, r = kmin + idx - cc * extra;
      Wm[cc * LD + r] = cz();
    }
    bsync<NT>();
    apply_q_packed<CAP, NT>(sm, Wm, n, kmin, kmin);
  }
  MPSKQ_DBG_ADD(5, t_q);
  MPSKQ_DBG_T(t_wside);
  if (left) {
    // site_{q+1} = Vh
    #pragma unroll 1
    for (int idx = tid; idx < keep * Nc; idx += NT) {
      const int kk = idx / Nc, col = idx - kk * Nc;
      Y[idx] = cconj(Wm[sm.perm[kk] * LD + col]);
    }
  } else {
    // site_q = U
    #pragma unroll 1
    for (int idx = tid; idx < Mr * keep; idx += NT) {
      const int row = idx / keep, kk = idx - row * keep;
      X[idx] = Wm[sm.perm[kk] * LD + row];
    }
  }
  if (tid == 0) {
    sm.chi[q + 1] = keep;
    st.discard += sm.scal[1];  // accumulated_discard (mps.py:201)
    st.peak = max(st.peak, keep);
    sm.scal[4] += nominal_two_qubit(chl, chm, chr);
  }
  bsync<NT>();
  MPSKQ_DBG_ADD(6, t_wside);
}


// ---------------------------------------------------------------------------
// States per CTA: NT == 32 kernels run SPC states (one per warp) in lockstep,
// a CTA barrier after every op, so the SM's warps stay in the same small
// region of the (large) op code and the instruction cache keeps up.
template <int NT>
struct SpcFor {
  static constexpr int value = NT <= 32 ? MPSKQ_SPC_THREADS / NT : 1;
};

// Capacity 128 (512 threads per state, theta in the L2 workspace): two
// resident states per SM need <= 64 registers per thread; capacities 64-96
// (256 threads) bound three.  Without the bound
// ptxas takes 128 and halves the states in flight (measured +29% simulation
// time at m=100 d=7 / d=8, tools/ab_sim_abi.py).
#ifndef MPSKQ_MIN_CTAS_128
#define MPSKQ_MIN_CTAS_128 1  // A/B knob: launch-bound CTAs per SM at 128 threads
#endif
#ifndef MPSKQ_MIN_CTAS_256
#define MPSKQ_MIN_CTAS_256 3  // A/B knob: launch-bound CTAs per SM at 256 threads
#endif
#ifndef MPSKQ_MIN_CTAS_192
#define MPSKQ_MIN_CTAS_192 3  // A/B knob: launch-bound CTAs per SM at 192 threads
#endif
template <int NT>
struct MinCtasFor {
  static constexpr int value = NT >= 512 ? 2 : NT == 256 ? MPSKQ_MIN_CTAS_256 : NT == 192 ? MPSKQ_MIN_CTAS_192 : NT == 128 ? MPSKQ_MIN_CTAS_128 : 1;
};

// GEN: programs of the state-level API (continue a given state, arbitrary
// U1 / U2 matrices); the feature-map programs run the GEN = false build,
// whose registers the general-matrix paths do not touch.
template <int CAP, int NT, bool GEN>
__global__ void __launch_bounds__(NT * SpcFor<NT>::value, MinCtasFor<NT>::value) sim_kernel(SimArgs a) {
  constexpr int SPC = SpcFor<NT>::value;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int slot = SPC > 1 ? (int)(threadIdx.x / NT) : 0;
  Smem<CAP, NT> sm;
  double2* gws = nullptr;
  if constexpr (GlobalWs<CAP>::value)
    gws = reinterpret_cast<double2*>(static_cast<double4*>(a.scratch) +
                                     (LogW<CAP>::value ? (int64_t)gridDim.x * LogW<CAP>::entries : 0)) +
          (int64_t)blockIdx.x * GlobalWs<CAP>::complexes;
  sm.carve(smem_raw + (size_t)slot * Smem<CAP, NT>::bytes(a.m), a.m, gws);
  if constexpr (LogW<CAP>::value)
    sm.rlog = static_cast<double4*>(a.scratch) + (int64_t)blockIdx.x * LogW<CAP>::entries;
  const int tid = ltid<NT>();
  const int m = a.m;
  const int4* ops = reinterpret_cast<const int4*>(a.ops);
  const double2* coef = reinterpret_cast<const double2*>(a.coef);
  for (int64_t n0 = (int64_t)blockIdx.x * SPC; n0 < a.n_states; n0 += (int64_t)gridDim.x * SPC) {
    const int64_t n = n0 + slot;
    bool live = n < a.n_states;  // uniform per state group
    StateCtx st{reinterpret_cast<double2*>(a.sites) + (live ? n : 0) * a.state_stride, a.site_off, m,
                MPSKQ_STATE_OK, 1, 0.0};
    if (GEN && live && a.from_input) {
      // continue an existing state (apply_gate / canonicalize / run_circuit on
      // a given MpsState, mps.py:123-247): sites are already in the slab,
      // bond dims, discard and peak come in through the output arrays
      #pragma unroll 1
      for (int b = tid; b <= m; b += NT) sm.chi[b] = a.chi[n * (m + 1) + b];
      if (tid == 0) {
        st.discard = a.discard[n];
        st.peak = a.peak[n];
      }
      bsync<NT>();
    } else if (live) {
      // init_state(m, "zero"): every site (1, 2, 1) = [1, 0]  (mps.py:90-102)
      #pragma unroll 1
      for (int b = tid; b <= m; b += NT) sm.chi[b] = 1;
      #pragma unroll 1
      for (int s = tid; s < m; s += NT) {
        st.base[a.site_off[s]] = make_double2(1.0, 0.0);
        st.base[a.site_off[s] + 1] = cz();
      }
      bsync<NT>();
    }
    // nominal flops and per-phase device cycles (MpsState.timings keys,
    // mps.py:137/:159/:204) accumulate in shared memory (thread 0): no extra
    // registers live across the ops
    if (tid == 0)
      for (int x = 3; x < 8; ++x) sm.scal[x] = 0.0;
    long long* op_t0 = reinterpret_cast<long long*>(sm.scal + 3);
    const double2* cf = coef + (live ? n : 0) * a.n_params;
    for (int64_t i = 0; i < a.n_ops; ++i) {
      if (live) {
        const int4 op = __ldg(ops + i);
        const int code = op.x & 0xff;
        const bool left = (op.x >> 8) & MPSKQ_ABSORB_LEFT;
        const double2 cs = op.z >= 0 ? __ldg(cf + op.z) : make_double2(1.0, 0.0);
        const double2* gm = GEN ? cf + (op.z >= 0 ? op.z : 0) : nullptr;  // U1 / U2 matrices
        if (a.phase_cycles && tid == 0) *op_t0 = clock64();
        switch (code) {
          case MPSKQ_OP_H:
          case MPSKQ_OP_RZ:
          case MPSKQ_OP_U1:
            op_one_qubit<CAP, NT, GEN>(sm, st, op.y, code, cs, gm);
            break;
          case MPSKQ_OP_QRL: {
            MPSKQ_DBG_T(t_mv);
            op_qr_left<CAP, NT>(sm, st, op.y);
            MPSKQ_DBG_ADD(7, t_mv);
            break;
          }
          case MPSKQ_OP_QRR: {
            MPSKQ_DBG_T(t_mv);
            op_qr_right<CAP, NT>(sm, st, op.y);
            MPSKQ_DBG_ADD(7, t_mv);
            break;
          }
          default:
            op_two_qubit<CAP, NT, GEN>(sm, st, op.y, code, left, cs, gm, a.budget, a.chi_max);
            break;
        }
        if (a.phase_cycles && tid == 0) {
          const double dt = (double)(clock64() - *op_t0);
          const int ph = (code == MPSKQ_OP_QRL || code == MPSKQ_OP_QRR)                      ? 0
                         : (code == MPSKQ_OP_H || code == MPSKQ_OP_RZ || code == MPSKQ_OP_U1) ? 1
                                                                                              : 2;
          sm.scal[5 + ph] += dt;
        }
        if (st.status != MPSKQ_STATE_OK) live = false;  // keep hitting the barriers
        if (live && a.entry_log != nullptr && op.w >= 0 && tid == 0) {
          int64_t entries = 0;
          for (int s = 0; s < m; ++s) entries += 2 * (int64_t)sm.chi[s] * sm.chi[s + 1];
          a.entry_log[n * a.n_gates + op.w] = entries;
        }
      }
      if constexpr (SPC > 1) __syncthreads();
    }
    if (n < a.n_states) {
      #pragma unroll 1
      for (int b = tid; b <= m; b += NT) a.chi[n * (m + 1) + b] = sm.chi[b];
      if (tid == 0) {
        a.discard[n] = st.discard;
        a.peak[n] = st.peak;
        a.status[n] = st.status;
        if (a.nominal_flops) a.nominal_flops[n] = sm.scal[4];
        if (a.phase_cycles)
          for (int x = 0; x < 3; ++x) a.phase_cycles[3 * n + x] = (long long)sm.scal[5 + x];
      }
    }
    bsync<NT>();
  }
}

// svd_truncated on a batch of matrices (tensor.py:87-123)
template <int CAP, int NT>
__global__ void __launch_bounds__(NT) svd_kernel(SvdArgs a) {
  constexpr int LD = 2 * CAP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<CAP, NT> sm;
  double2* gws = nullptr;
  if constexpr (GlobalWs<CAP>::value)
    gws = reinterpret_cast<double2*>(static_cast<double4*>(a.scratch) +
                                     (LogW<CAP>::value ? (int64_t)gridDim.x * LogW<CAP>::entries : 0)) +
          (int64_t)blockIdx.x * GlobalWs<CAP>::complexes;
  sm.carve(smem_raw, 0, gws);
  if constexpr (LogW<CAP>::value)
    sm.rlog = static_cast<double4*>(a.scratch) + (int64_t)blockIdx.x * LogW<CAP>::entries;
  const int tid = ltid<NT>();
  const int rows = a.rows, cols = a.cols, kmin = min(rows, cols);
  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    const double2* M = reinterpret_cast<const double2*>(a.mats) + b * rows * cols;
    int bad = 0;
    #pragma unroll 1
    for (int idx = tid; idx < rows * cols; idx += NT) {
      const int r = idx / cols, c = idx - r * cols;
      const double2 v = M[idx];
      bad |= !cfinite(v);
      sm.A[c * LD + r] = v;
    }
    if (block_any<NT>(bad)) {
      if (tid == 0) a.status[b] = MPSKQ_STATE_NONFINITE;
      continue;
    }
    int sweeps = jacobi<CAP, NT>(sm, rows, cols);
    if (sweeps & kNoConvergence) {
      if (tid == 0) a.status[b] = MPSKQ_STATE_NOCONV;
      bsync<NT>();
      continue;
    }
    norms_and_order<CAP, NT>(sm, rows, cols);
    if (tid == 0) truncation_rule<CAP, NT>(sm, kmin, a.budget, a.chi_max);
    bsync<NT>();
    const double s0 = sm.sig[sm.perm[0]];
    #pragma unroll 1
    for (int k = tid; k < kmin; k += NT) {
      double x = sm.sig[sm.perm[k]];
      if (s0 > 0.0 && x < kNoiseFloor * s0) x = 0.0;
      a.s[b * kmin + k] = x;
    }
    double2* U = reinterpret_cast<double2*>(a.u) + b * rows * kmin;
    #pragma unroll 1
    for (int idx = tid; idx < rows * kmin; idx += NT) {
      const int r = idx / kmin, k = idx - r * kmin;
      const double nrm = sm.sig[sm.perm[k]];
      U[idx] = nrm > 0.0 ? cscale(sm.A[sm.perm[k] * LD + r], 1.0 / nrm) : cz();
    }
    double2* Vh = reinterpret_cast<double2*>(a.vh) + b * kmin * cols;
    const double2* Wm = sm.W;
    if constexpr (LogW<CAP>::value) {
      bsync<NT>();
      replay<CAP, NT>(sm, sm.A, cols, sweeps);
      Wm = sm.A;
    }
    #pragma unroll 1
    for (int idx = tid; idx < kmin * cols; idx += NT) {
      const int k = idx / cols, c = idx - k * cols;
      Vh[idx] = cconj(Wm[sm.perm[k] * LD + c]);
    }
    if (tid == 0) {
      a.keep[b] = sm.ibuf[0];
      a.discarded[b] = sm.scal[1];
      a.status[b] = MPSKQ_STATE_OK;
    }
    bsync<NT>();
  }
}

namespace {

template <class K>
int prepare(K kernel, size_t smem) {
  if (smem > 48 * 1024) {
    cudaError_t e =
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(sim smem)");
  }
  return MPSKQ_OK;
}

// grid and rotation-log scratch; capacities > 32 run one persistent CTA per SM
template <int CAP, class K>
int plan_grid(K kernel, int threads, size_t smem, int64_t items, cudaStream_t st, int64_t* grid, void** scratch) {
  *grid = items < (int64_t(1) << 30) ? items : (int64_t(1) << 30);
  *scratch = nullptr;
  if constexpr (LogW<CAP>::value || GlobalWs<CAP>::value) {
    // persistent grid of all co-resident CTAs, each with its own log slice / workspace
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    const int64_t cap = (int64_t)sms * per_sm;
    *grid = items < cap ? items : cap;
    size_t bytes = LogW<CAP>::value ? sizeof(double4) * LogW<CAP>::entries * *grid : 0;
    if constexpr (GlobalWs<CAP>::value) bytes += sizeof(double2) * GlobalWs<CAP>::complexes * *grid;
    cudaError_t e = cudaMallocAsync(scratch, bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(rotation log)");
  }
  return MPSKQ_OK;
}

template <int CAP, bool GEN>
int launch_sim_cap_k(const SimArgs& a0, cudaStream_t st) {
  constexpr int NT = NtFor<CAP>::value;
  constexpr int SPC = SpcFor<NT>::value;
  const size_t smem = Smem<CAP, NT>::bytes(a0.m) * SPC;
  if (int s = prepare(sim_kernel<CAP, NT, GEN>, smem)) return s;
  SimArgs a = a0;
  int64_t grid = 0;
  if (int s = plan_grid<CAP>(sim_kernel<CAP, NT, GEN>, NT * SPC, smem, (a.n_states + SPC - 1) / SPC, st, &grid,
                             &a.scratch))
    return s;
  sim_kernel<CAP, NT, GEN><<<(unsigned)grid, NT * SPC, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (a.scratch) cudaFreeAsync(a.scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "sim_kernel launch");
  return MPSKQ_OK;
}

template <int CAP>
int launch_sim_cap(const SimArgs& a0, cudaStream_t st) {
  if (a0.from_input) return launch_sim_cap_k<CAP, true>(a0, st);
  return launch_sim_cap_k<CAP, false>(a0, st);
}

template <int CAP>
int launch_svd_cap(const SvdArgs& a0, cudaStream_t st) {
  constexpr int NT = NtFor<CAP>::value;
  const size_t smem = Smem<CAP, NT>::bytes(0);
  if (int s = prepare(svd_kernel<CAP, NT>, smem)) return s;
  SvdArgs a = a0;
  int64_t grid = 0;
  if (int s = plan_grid<CAP>(svd_kernel<CAP, NT>, NT, smem, a.batch, st, &grid, &a.scratch)) return s;
  svd_kernel<CAP, NT><<<(unsigned)grid, NT, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (a.scratch) cudaFreeAsync(a.scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "svd_kernel launch");
  return MPSKQ_OK;
}

}  // namespace

int launch_simulate(const SimArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  switch (a.chi_cap) {
    case 4: return launch_sim_cap<4>(a, st);
    case 8: return launch_sim_cap<8>(a, st);
    case 12: return launch_sim_cap<12>(a, st);
    case 16: return launch_sim_cap<16>(a, st);
    case 24: return launch_sim_cap<24>(a, st);
    case 32: return launch_sim_cap<32>(a, st);
    case 48: return launch_sim_cap<48>(a, st);
    case 64: return launch_sim_cap<64>(a, st);
    case 80: return launch_sim_cap<80>(a, st);
    case 96: return launch_sim_cap<96>(a, st);
    case 128: return launch_sim_cap<128>(a, st);
  }
  return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", a.chi_cap);
}

int launch_svd(const SvdArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  const int big = a.rows > a.cols ? a.rows : a.cols;
  if (big <= 8) return launch_svd_cap<4>(a, st);
  if (big <= 16) return launch_svd_cap<8>(a, st);
  if (big <= 24) return launch_svd_cap<12>(a, st);
  if (big <= 32) return launch_svd_cap<16>(a, st);
  if (big <= 48) return launch_svd_cap<24>(a, st);
  if (big <= 64) return launch_svd_cap<32>(a, st);
  if (big <= 96) return launch_svd_cap<48>(a, st);
  if (big <= 128) return launch_svd_cap<64>(a, st);
  if (big <= 160) return launch_svd_cap<80>(a, st);
  if (big <= 192) return launch_svd_cap<96>(a, st);
  return launch_svd_cap<128>(a, st);
}

// State relayout between chi-capacity layouts (per-state capacity escalation:
// the few states that outgrew a capacity are re-simulated at a larger one and
// everything is gathered into the largest layout).  One CTA per state; every
// site tensor is (chi_l, 2, chi_r) row-major at the start of its slot in both
// layouts, so a state moves as m contiguous runs.
__global__ void relayout_kernel(int m, int64_t n, const double2* __restrict__ src,
                                const int64_t* __restrict__ src_off, int64_t src_stride,
                                const int32_t* __restrict__ chi, double2* __restrict__ dst,
                                const int64_t* __restrict__ dst_off, int64_t dst_stride,
                                const int32_t* __restrict__ dst_rows) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int32_t* c = chi + i * (m + 1);
    const double2* s = src + i * src_stride;
    double2* d = dst + (int64_t)(dst_rows ? dst_rows[i] : i) * dst_stride;
    for (int site = 0; site < m; ++site) {
      const int len = 2 * c[site] * c[site + 1];
      const double2* ss = s + src_off[site];
      double2* dd = d + dst_off[site];
      for (int e = threadIdx.x; e < len; e += blockDim.x) dd[e] = ss[e];
    }
  }
}

int launch_relayout(int m, int64_t n, const double* src, const int64_t* src_off, int64_t src_stride,
                    const int32_t* chi, double* dst, const int64_t* dst_off, int64_t dst_stride,
                    const int32_t* dst_rows, void* stream) {
  if (n <= 0) return MPSKQ_OK;
  relayout_kernel<<<(unsigned)std::min<int64_t>(n, 148 * 16), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      m, n, reinterpret_cast<const double2*>(src), src_off, src_stride, chi, reinterpret_cast<double2*>(dst),
      dst_off, dst_stride, dst_rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "relayout launch");
  return MPSKQ_OK;
}

// Exact (unpadded) wire packing of a batch for the multi-GPU exchange: state
// i's site tensors, (chi_l, 2, chi_r) row-major each, back to back from
// complex offset state_off[i] (the MPS1 payload order, mps.py:294-314).
// unpack = 0: layout -> packed; 1: packed -> layout.
__global__ void pack_exact_kernel(int m, int64_t n, double2* __restrict__ sites, const int64_t* __restrict__ site_off,
                                  int64_t stride, const int32_t* __restrict__ chi,
                                  const int64_t* __restrict__ state_off, double2* __restrict__ packed, int unpack,
                                  const int32_t* __restrict__ rows) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const int32_t* c = chi + i * (m + 1);
    double2* lay = sites + (int64_t)(rows ? rows[i] : i) * stride;  // layout row (unpack: destination)
    double2* pk = packed + state_off[i];
    int64_t o = 0;
    for (int s = 0; s < m; ++s) {
      const int len = 2 * c[s] * c[s + 1];
      double2* ls = lay + site_off[s];
      if (unpack)
        for (int e = threadIdx.x; e < len; e += blockDim.x) ls[e] = pk[o + e];
      else
        for (int e = threadIdx.x; e < len; e += blockDim.x) pk[o + e] = ls[e];
      o += len;
    }
  }
}

int launch_pack_exact(int m, int64_t n, double* sites, const int64_t* site_off, int64_t stride, const int32_t* chi,
                      const int64_t* state_off, double* packed, int unpack, const int32_t* rows, void* stream) {
  if (n <= 0) return MPSKQ_OK;
  pack_exact_kernel<<<(unsigned)std::min<int64_t>(n, 148 * 16), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      m, n, reinterpret_cast<double2*>(sites), site_off, stride, chi, state_off, reinterpret_cast<double2*>(packed),
      unpack, rows);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pack_exact launch");
  return MPSKQ_OK;
}

// dst[dst_idx[i]] = src[src_idx[i]] for rows of `words` 32-bit words (either
// index nullable = identity): coefficient gathers and bond-dim / discard /
// peak scatters of the per-state capacity escalation
__global__ void copy_rows_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int64_t words,
                                 int64_t n, const int32_t* __restrict__ src_idx,
                                 const int32_t* __restrict__ dst_idx) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const uint32_t* s = src + (int64_t)(src_idx ? src_idx[i] : i) * words;
    uint32_t* d = dst + (int64_t)(dst_idx ? dst_idx[i] : i) * words;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) d[w] = s[w];
  }
}

int launch_copy_rows(const void* src, void* dst, int64_t row_bytes, int64_t n, const int32_t* src_idx,
                     const int32_t* dst_idx, void* stream) {
  if (n <= 0) return MPSKQ_OK;
  if (row_bytes % 4) return fail(MPSKQ_ERR_INVALID, "row size must be a multiple of 4 bytes");
  copy_rows_kernel<<<(unsigned)std::min<int64_t>(n, 148 * 16), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), row_bytes / 4, n, src_idx, dst_idx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "copy_rows launch");
  return MPSKQ_OK;
}

// FP64 FMA throughput probe: 16 independent DFMA chains per thread
__global__ void __launch_bounds__(256) fp64_probe_kernel(int64_t iters, double* out) {
  double acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 1.0 + 1e-3 * (threadIdx.x + j);
  const double b = 0.9999999, c = 1e-7;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fma(acc[j], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  if (s == 1234.5678) out[0] = s;  // keep the chains alive
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = s;
}

int launch_fp64_probe(int n_blocks, int64_t iters, double* out, void* stream) {
  fp64_probe_kernel<<<n_blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(iters, out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "fp64_probe launch");
  return MPSKQ_OK;
}

}  // namespace mpskq

#ifdef MPSKQ_DEBUG_COUNTERS
extern "C" int mpskq_debug_counters(unsigned long long* out3) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out3, mpskq::g_dbg_rounds, 8);
  cudaMemcpyFromSymbol(out3 + 1, mpskq::g_dbg_svds, 8);
  cudaMemcpyFromSymbol(out3 + 2, mpskq::g_dbg_span, 8);
  return 0;
}
// 8 per-phase cycle sums (see g_dbg_cyc)
extern "C" int mpskq_debug_cycles(unsigned long long* out8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, mpskq::g_dbg_cyc, 64);
  return 0;
}
#endif
