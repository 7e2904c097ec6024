// Tiled batched MPS overlaps <bra_i|ket_j> and kernel entries |.|^2.
//
// Reference: inner_product (mps.py:260-268) — env = [[1]]; per site
//   tmp = tensordot(env, conj(A), (0,0)); env = tensordot(tmp, B, ((0,1),(0,1)))
// and compute_gram (kernel.py:147-185): train fills i<j, mirrors, diagonal 1.
//
// Two B200 paths:
//  * small chi (capacity 4, the 165-qubit headline): one thread per (bra, ket)
//    pair with its 4x4 complex environment in registers; a warp is one bra x 32
//    kets, a CTA 8 bras x 32 kets.  Sites are repacked once into a
//    lane-interleaved, zero-padded layout [site][ket block][entry][lane] so the
//    32 kets of a warp read one coalesced 512-byte line per tensor entry, and
//    the bra tensor of each site is staged once per warp in shared memory and
//    read as broadcasts.  Loop bounds are the bra's exact bond dims and the
//    ket block's maximum bond dims, both warp-uniform, so there is no
//    divergence and padding costs only up to the block maximum.  Pure FP64
//    FMA issue; no tensor cores (tcgen05 has no FP64 kind; DMMA only pays
//    off for dense chi >= 16 contractions).
//  * generic chi (capacities 8..48): one warp per pair, both site
//    contractions as complex GEMM tiles on the FP64 tensor cores (DMMA),
//    exact bond dims from the batch layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "device.cuh"
#include "internal.h"
#include "o1_site.cuh"

#ifndef MPSKQ_MMA_GROUP
#define MPSKQ_MMA_GROUP 0  // warps per pair of the L2-plane DMMA overlap (0: per capacity)
#endif
#ifndef MPSKQ_MMA_GLOBAL_CTAS
#define MPSKQ_MMA_GLOBAL_CTAS 2  // resident CTAs per SM of the L2-plane DMMA overlap
#endif

namespace mpskq {

namespace {

using o1::kEnt;
using o1::kLanes;
using o1::kP;
#ifndef MPSKQ_O1_WARPS
#define MPSKQ_O1_WARPS 8  // compute warps (= bras) per CTA tile: 8 (one CTA per SM) or 4 (two)
#endif
#ifndef MPSKQ_O1_STAGES
#define MPSKQ_O1_STAGES 10  // ring depth in sites (falls back to 8 when the chain is too long for it)
#endif
constexpr int kWarpsO1 = MPSKQ_O1_WARPS;        // bras per CTA tile
constexpr int kCtasO1 = kWarpsO1 == 4 ? 2 : 1;  // resident CTAs per SM

// --------------------------------------------------------------- packing
// sim layout -> [site][block][entry][lane] (double2), zero padded to 4x2x4
__global__ void pack_o1_kernel(const double2* __restrict__ sites, const int32_t* __restrict__ chi,
                               const int64_t* __restrict__ site_off, int64_t stride, int m,
                               int64_t n, int64_t nblk, const int32_t* __restrict__ perm,
                               double2* __restrict__ out) {
  const int64_t total = (int64_t)m * nblk * kEnt * kLanes;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx % kLanes);
    const int e = (int)((idx / kLanes) % kEnt);
    const int64_t blk = (idx / (kLanes * kEnt)) % nblk;
    const int s = (int)(idx / ((int64_t)kLanes * kEnt * nblk));
    const int64_t pos = blk * kLanes + lane;
    double2 v = make_double2(0.0, 0.0);
    if (pos < n) {
      const int64_t state = perm ? perm[pos] : pos;
      const int k = e / (2 * kP), p = (e / kP) & 1, r = e % kP;
      const int chl = chi[state * (m + 1) + s], chr = chi[state * (m + 1) + s + 1];
      if (k < chl && r < chr) v = sites[state * stride + site_off[s] + (k * 2 + p) * chr + r];
    }
    out[idx] = v;
  }
}

// Ket ordering key: one bit per window of bonds that holds a chi = 4 bond,
// most significant first, so sorting groups kets whose wide bonds coincide
// and 32-ket blocks more often have max chi <= 3 at a bond.
__global__ void ket_key_kernel(const int32_t* __restrict__ chi, int m, int64_t n,
                               uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int win = (m + 1 + 31) / 32;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    uint32_t key = 0;
    for (int b = 0; b <= m; ++b)
      if (chi[idx * (m + 1) + b] >= kP) key |= 1u << (31 - b / win);
    keys[idx] = key;
    vals[idx] = (int32_t)idx;
  }
}

// per block of 32 (ordered) kets and bond: 1 if every ket has chi <= 3 there
__global__ void block_narrow_kernel(const int32_t* __restrict__ chi, const int32_t* __restrict__ perm,
                                    int m, int64_t n, int64_t nblk, uint8_t* __restrict__ out) {
  const int64_t total = nblk * (m + 1);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = idx / (m + 1);
    const int b = (int)(idx % (m + 1));
    int mx = 1;
    for (int l = 0; l < kLanes; ++l) {
      const int64_t pos = blk * kLanes + l;
      if (pos < n) mx = max(mx, chi[(perm ? perm[pos] : pos) * (m + 1) + b]);
    }
    out[idx] = mx < kP;
  }
}

// Greedy refinement of the key order, one CTA per group of kClusterGroup
// consecutive (key-sorted) kets: each 32-ket block starts from the remaining
// ket with the most chi = 4 bonds and repeatedly takes the ket that adds the
// fewest new chi = 4 bonds to the block's union, so more (block, bond) pairs
// are "narrow" (the kernel's padded work shrinks; results do not change).
// Ties go to the lowest position, so the order is deterministic.
constexpr int kClusterGroup = 512;
constexpr int kClusterMaxWords = 16;  // bonds <= 512 (32 KB of bit rows); longer chains keep the key order

__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v, unsigned long long* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  v = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = min(v, red[w]);
  return v;
}

__global__ void __launch_bounds__(kClusterGroup) cluster_kets_kernel(const int32_t* __restrict__ chi, int m,
                                                                     int64_t n, const int32_t* __restrict__ in,
                                                                     int32_t* __restrict__ out) {
  __shared__ uint32_t S[kClusterGroup * kClusterMaxWords];
  __shared__ uint32_t U[kClusterMaxWords], D[kClusterMaxWords];
  __shared__ unsigned long long red[kClusterGroup / 32];
  const int W = (m + 1 + 31) / 32;
  const int64_t g0 = (int64_t)blockIdx.x * kClusterGroup;
  const int gs = (int)(n - g0 < kClusterGroup ? n - g0 : kClusterGroup);
  const int c = threadIdx.x;
  int cnt = 0;
  if (c < gs) {
    const int32_t* row = chi + (int64_t)in[g0 + c] * (m + 1);
    for (int w = 0; w < W; ++w) {
      uint32_t word = 0;
      for (int b = 0; b < 32 && w * 32 + b <= m; ++b) word |= (uint32_t)(row[w * 32 + b] >= kP) << b;
      S[c * W + w] = word;
      cnt += __popc(word);
    }
  }
  bool alive = c < gs;
  int cost = 0;
  for (int pos = 0; pos < gs; ++pos) {
    const bool seed = (pos & (kLanes - 1)) == 0;
    unsigned long long key = ~0ull;
    if (alive) key = ((unsigned long long)(seed ? 0xFFFF - cnt : cost) << 32) | (unsigned)c;
    const int j = (int)(block_min_u64(key, red) & 0xFFFFFFFFu);
    if (c < W) {
      const uint32_t u = seed ? 0u : U[c];
      const uint32_t d = S[j * W + c] & ~u;
      D[c] = d;
      U[c] = u | d;
    }
    if (c == j) {
      alive = false;
      out[g0 + pos] = in[g0 + c];
    }
    __syncthreads();
    if (alive) {
      if (seed) cost = cnt;
      for (int w = 0; w < W; ++w) cost -= __popc(S[c * W + w] & D[w]);
    }
  }
}

__global__ void invert_perm_kernel(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ inv) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    inv[perm[p]] = (int32_t)p;
}

// out[a][b] = ordered[bpos[a]][kpos[b]] (row gather, coalesced writes).  For
// the train kind `ordered` holds both triangles; the diagonal is filled later.
template <class T>
__global__ void unpermute_kernel(const T* __restrict__ ordered, int64_t nk, const int32_t* __restrict__ bpos,
                                 const int32_t* __restrict__ kpos, int64_t nb, T* __restrict__ out, int64_t ld) {
  for (int64_t a = blockIdx.x; a < nb; a += gridDim.x) {
    const T* row = ordered + (int64_t)(bpos ? bpos[a] : a) * nk;
    for (int64_t b = threadIdx.x; b < nk; b += blockDim.x) out[a * ld + b] = row[kpos[b]];
  }
}

// Host-streaming variant for one band of ordered rows [r0, r1): caller row
// a = row_of[o] (train; identity for test bras) is gathered like
// unpermute_kernel and written straight into pinned host memory (one
// contiguous row per CTA pass, coalesced over the link); the train diagonal
// is written here as 1.0 (compute_gram's eye, kernel.py:168).
__global__ void rows_to_host_kernel(const double* __restrict__ ordered, int64_t nk,
                                    const int32_t* __restrict__ row_of, int64_t r0, int64_t r1,
                                    const int32_t* __restrict__ kpos, bool train,
                                    double* __restrict__ out, int64_t ld) {
  for (int64_t o = r0 + blockIdx.x; o < r1; o += gridDim.x) {
    const int64_t a = row_of ? row_of[o] : o;
    const double* row = ordered + o * nk;
    for (int64_t b = threadIdx.x; b < nk; b += blockDim.x)
      out[a * ld + b] = (train && b == a) ? 1.0 : row[kpos[b]];
  }
}

// Row ownership (world > 1): the k-th owned row is ordered row
// o = (band(k) * world + rank) * rb + k % rb; gather it in caller column
// order into the compact block and record its caller row id.
__global__ void owned_rows_kernel(const double* __restrict__ ordered, int64_t n_rows, int64_t nk, int rb,
                                  int rank, int world, const int32_t* __restrict__ row_of,
                                  const int32_t* __restrict__ kpos, double* __restrict__ out,
                                  int32_t* __restrict__ ids, int64_t n_owned) {
  for (int64_t k = blockIdx.x; k < n_owned; k += gridDim.x) {
    const int64_t o = ((k / rb) * world + rank) * rb + k % rb;
    if (o >= n_rows) continue;
    const double* row = ordered + o * nk;
    for (int64_t b = threadIdx.x; b < nk; b += blockDim.x) out[k * nk + b] = row[kpos ? kpos[b] : b];
    if (threadIdx.x == 0) ids[k] = row_of ? row_of[o] : (int32_t)o;
  }
}

__device__ __forceinline__ void store_result(int out_mode, double* out, int64_t ld, int64_t i,
                                             int64_t j, double2 ov, bool mirror) {
  if (out_mode == MPSKQ_OUT_KERNEL) {
    const double h = hypot(ov.x, ov.y);  // abs(complex) ** 2 (kernel.py:174)
    const double v = h * h;
    out[i * ld + j] = v;
    if (mirror) out[j * ld + i] = v;
  } else {
    reinterpret_cast<double2*>(out)[i * ld + j] = ov;
    if (mirror) reinterpret_cast<double2*>(out)[j * ld + i] = cconj(ov);
  }
}

// --------------------------------------------------------------- small chi
// bra-major padded layout [site][state (padded to the 8-bra tile)][entry]: the
// 8 bras of a tile at one site are one contiguous 4 KB run for a bulk copy
__global__ void pack_bra_kernel(const double2* __restrict__ sites, const int32_t* __restrict__ chi,
                                const int64_t* __restrict__ site_off, int64_t stride, int m,
                                int64_t n, int64_t n_pad, const int32_t* __restrict__ perm,
                                double2* __restrict__ out) {
  const int64_t total = (int64_t)m * n_pad * kEnt;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(idx % kEnt);
    const int64_t pos = (idx / kEnt) % n_pad;
    const int s = (int)(idx / ((int64_t)kEnt * n_pad));
    double2 v = make_double2(0.0, 0.0);
    if (pos < n) {
      const int64_t state = perm ? perm[pos] : pos;
      const int k = e / (2 * kP), p = (e / kP) & 1, r = e % kP;
      const int chl = chi[state * (m + 1) + s], chr = chi[state * (m + 1) + s + 1];
      if (k < chl && r < chr) v = sites[state * stride + site_off[s] + (k * 2 + p) * chr + r];
    }
    out[idx] = v;
  }
}

// ring slots (sites in flight); slot = counter % STAGES.  10 slots measured
// 139.8 ms vs 141.5 ms for 8 at N=6400 (warps drift further before the
// slowest one holds a slot, profiles/r02_ab_o1_ws.txt)
constexpr int kStages = MPSKQ_O1_STAGES;
constexpr int kStagesMin = 8;
constexpr uint32_t kKetBytes = kEnt * kLanes * sizeof(double2);   // 16 KB per site
constexpr uint32_t kBraBytes = kWarpsO1 * kEnt * sizeof(double2);  // 4 KB per site
inline size_t o1_smem_bytes(int m, int stages) {
  return stages * (size_t)(kKetBytes + kBraBytes) + 2 * stages * sizeof(uint64_t) + 16 +
         sizeof(int32_t) * kWarpsO1 * (size_t)(m + 1);
}

struct O1Args {
  const double2* bra;  // [site][n_pad_bra][entry]
  const double2* ket;  // [site][nblk_ket][entry][lane]
  const int32_t* bra_chi;
  int64_t n_bras, n_kets, n_pad_bra, nblk_ket;
  int m, kind, out_mode;
  const int2* tiles;  // (bra tile of 8, ket block of 32), in ordered positions
  int64_t n_tiles;
  double* out;
  int64_t ld;
  const int32_t* bperm;      // ordered position -> bra index (nullable)
  const int32_t* kperm;      // ordered position -> ket index
  const uint8_t* kb_narrow;  // [ket block][bond]: block max chi <= 3
};

// One CTA = 8 bras (compute warps) x 32 kets (lanes); one thread owns one
// pair's 4x4 complex environment in registers.  Persistent over its tiles,
// the CTA streams each site's ket block (16 KB) and bra tile (4 KB) through an
// 8-stage shared-memory ring: TMA bulk copies (cp.async.bulk) complete on
// "full" mbarriers, every compute warp releases a slot on its "empty"
// mbarrier, so warps drift up to the ring depth instead of synchronising
// every site.  Warp-specialised: the 8 compute warps (two warpgroups,
// registers raised to 240 with setmaxnreg) only wait and release; a third
// warpgroup (registers lowered to 24) runs the producer — one lane walks the
// CTA's (tile, site) sequence, waits until all 8 compute warps released a
// slot and issues its two copies.  (The earlier cooperative producer, where
// every compute warp could refill slots through a CAS on a shared counter,
// ran 147.8 ms at N=6400 against 142 ms for this one, `profiles/r02_ab_o1_ws.txt`.)
constexpr int kThreadsO1Ws = (kWarpsO1 + 4) * 32;


template <int STAGES>
__global__ void __launch_bounds__(kThreadsO1Ws, kCtasO1) overlap_o1_kernel(O1Args a) {
  constexpr int kStages = STAGES;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sket = reinterpret_cast<double2*>(smem_raw);
  double2* sbra = sket + kStages * kEnt * kLanes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sbra + kStages * kWarpsO1 * kEnt);
  uint64_t* empty = full + kStages;
  int32_t* schi = reinterpret_cast<int32_t*>(empty + kStages) + 4;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m = a.m;
  if (tid == 0) {
    for (int q = 0; q < kStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kWarpsO1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t my_tiles = (int64_t)blockIdx.x < a.n_tiles ? (a.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp >= kWarpsO1) {
    // ---------------- producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
    if (warp == kWarpsO1 && lane == 0) {
      const int64_t kstride = a.nblk_ket * kEnt * kLanes;  // per site
      const int64_t bstride = a.n_pad_bra * kEnt;
      uint32_t q = 0;
      for (int64_t k = 0; k < my_tiles; ++k) {
        const int2 tl = a.tiles[blockIdx.x + k * gridDim.x];
        const double2* kb = a.ket + (int64_t)tl.y * kEnt * kLanes;
        const double2* bb = a.bra + (int64_t)tl.x * kWarpsO1 * kEnt;
        for (int site = 0; site < m; ++site, ++q) {
          const uint32_t buf = q % kStages;
          if (q >= kStages) mbar_wait(&empty[buf], ((q / kStages) - 1) & 1);
          mbar_arrive_expect_tx(&full[buf], kKetBytes + kBraBytes);
          bulk_g2s(sket + buf * kEnt * kLanes, kb + site * kstride, kKetBytes, &full[buf]);
          bulk_g2s(sbra + buf * kWarpsO1 * kEnt, bb + site * bstride, kBraBytes, &full[buf]);
        }
      }
    }
    return;
  }
  // ---------------- compute warpgroups
  if constexpr (kCtasO1 == 1)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
  else
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  uint32_t it = 0;  // sites this warp consumed (ring position + phase)
  int32_t* mychi = schi + warp * (m + 1);
  for (int64_t k = 0; k < my_tiles; ++k) {
    const int2 tile = a.tiles[blockIdx.x + k * gridDim.x];
    const int64_t i = (int64_t)tile.x * kWarpsO1 + warp;  // bra (warp-uniform)
    const int64_t j = (int64_t)tile.y * kLanes + lane;    // ket (per lane)
    const int64_t ic = i < a.n_bras ? i : a.n_bras - 1;
    const int64_t ib = a.bperm ? a.bperm[ic] : ic;  // bra index of this warp
    const uint8_t* narrow = a.kb_narrow + (int64_t)tile.y * (m + 1);
    for (int b = lane; b <= m; b += kLanes) mychi[b] = __ldg(a.bra_chi + ib * (m + 1) + b);
    __syncwarp();
    double2 env[kP][kP];
#pragma unroll
    for (int x = 0; x < kP; ++x)
#pragma unroll
      for (int y = 0; y < kP; ++y) env[x][y] = make_double2(x == 0 && y == 0 ? 1.0 : 0.0, 0.0);
    int na = 1;  // chi_s of the bra (warp-uniform)
    for (int s = 0; s < m; ++s) {
      const int na1 = mychi[s + 1];
      const bool nar_l = __ldg(narrow + s) != 0, nar_r = __ldg(narrow + s + 1) != 0;
      const uint32_t buf = it % kStages;
      mbar_wait(&full[buf], (it / kStages) & 1);
      const double2* B = sket + buf * kEnt * kLanes + lane;  // B[e] at B[e * 32]
      const double2* A = sbra + buf * kWarpsO1 * kEnt + warp * kEnt;
      double2 T[kP][2][kP];
      using namespace o1;
      switch (na) {
        case 1: o1_phase1<1>(env, B, nar_l, nar_r, T); break;
        case 2: o1_phase1<2>(env, B, nar_l, nar_r, T); break;
        case 3: o1_phase1<3>(env, B, nar_l, nar_r, T); break;
        default: o1_phase1<4>(env, B, nar_l, nar_r, T); break;
      }
      o1_phase2(A, T, na, na1, nar_r, env);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[buf]);
      ++it;
      na = na1;
    }
    const bool train = a.kind == MPSKQ_KIND_TRAIN;
    const bool valid = i < a.n_bras && j < a.n_kets && (!train || i < j);
    if (valid) store_result(a.out_mode, a.out, a.ld, i, j, env[0][0], train);
    __syncwarp();
  }
}

// the deepest ring whose shared memory fits this chain length
struct O1Launch {
  void (*fn)(O1Args);
  size_t smem;
};
inline O1Launch o1_launch_for(int m) {
  constexpr size_t kMaxSmem = 227 * 1024;
  if (o1_smem_bytes(m, kStages) <= kMaxSmem) return {overlap_o1_kernel<kStages>, o1_smem_bytes(m, kStages)};
  return {overlap_o1_kernel<kStagesMin>, o1_smem_bytes(m, kStagesMin)};
}

// --------------------------------------------------------------- generic chi (DMMA)
// One warp per (bra, ket) pair, exact bond dims from the batch layout.  Both
// halves of the site step are complex GEMMs on FP64 tensor cores
// (mma.sync.m8n8k4.f64; a complex tile product is 4 real DMMAs):
//   phase 1  T  (a  x 2b1) = env (a x b) . B (b x 2b1)            B = ket site
//   phase 2  E' (a1 x b1)  = conj(A)^T (a1 x 2a) . T2 (2a x b1)   T2 = T reshaped
// env and T live in per-warp shared-memory planes (re / im, zero padded to
// whole tiles, leading dims = 4 mod 16 so fragment loads are conflict free);
// the site tensors are read straight from global memory into fragments (the
// bra is shared by the CTA's warps through L1).  Warps never synchronise with
// each other.
template <int CAP>
struct MmaCfg {
  static constexpr int R8 = (CAP + 7) / 8 * 8;              // padded rows of env / T
  static constexpr int L1 = (CAP + 15) / 16 * 16 + 4;       // env plane leading dim
  static constexpr int L2 = (2 * CAP + 15) / 16 * 16 + 4;   // T plane leading dim
  static constexpr int per_warp = 2 * R8 * L1 + 2 * R8 * L2;  // doubles
  // When fewer than 8 warps' planes fit in shared memory (capacities >= 24)
  // the planes move to a per-warp global scratch (L2 resident): at capacity
  // 48/64 the shared-memory variant ran ONE warp per SM (5x slower)
  static constexpr int max_warps = (220 * 1024) / (per_warp * 8);
  static constexpr bool global = max_warps < 8;
  static constexpr int warps = global ? 8 : (max_warps > 16 ? 16 : max_warps);
  static constexpr int ctas_per_sm = global ? MPSKQ_MMA_GLOBAL_CTAS : 1;
  // warps cooperating on one pair (tiles of each phase split among them):
  // with L2 planes, 4 per pair keeps the planes in flight (~600 pairs) inside
  // L2 instead of spilling ~2 TB/s of plane traffic to DRAM
  // (measured, tools/ov_caps.py: 1 up to capacity 32, 2 at 48/64, 4 from 80:
  // d=8 71 -> 53 ms, d=7 135 -> 116 ms)
  static constexpr int gw = !global ? 1 : MPSKQ_MMA_GROUP > 0 ? MPSKQ_MMA_GROUP : CAP <= 32 ? 1 : CAP <= 64 ? 2 : 4;
  static constexpr int pairs = warps / gw;  // pairs per CTA (ket columns of a tile)
  static constexpr size_t smem = global ? 0 : sizeof(double) * (size_t)per_warp * warps;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct CTile {  // complex 8x8 accumulator fragment: rows g, cols 2q, 2q+1
  double r0, r1, i0, i1;
};

// acc += (ar + i ai) (br + i bi) on one 8x8x4 fragment
__device__ __forceinline__ void cmma(CTile& c, double ar, double ai, double br, double bi) {
  dmma(c.r0, c.r1, ar, br);
  dmma(c.i0, c.i1, ar, bi);
  dmma(c.r0, c.r1, -ai, bi);
  dmma(c.i0, c.i1, ai, br);
}

struct MmaArgs {
  const double2* bra;
  const double2* ket;
  const int32_t* bra_chi;
  const int32_t* ket_chi;
  const int64_t* site_off;
  int64_t stride, n_bras, n_kets;
  int m, kind, out_mode;
  const int2* tiles;  // (bra, ket block)
  int64_t n_tiles;
  double* out;
  int64_t ld;
  double* gws;  // per-warp planes for capacities whose planes exceed shared memory
};

template <int CAP>
__global__ void __launch_bounds__(MmaCfg<CAP>::warps * 32, MmaCfg<CAP>::ctas_per_sm) overlap_mma_kernel(MmaArgs a) {
  using C = MmaCfg<CAP>;
  extern __shared__ __align__(16) double smem_d[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;  // fragment row group / thread in group
  const int grp = warp / C::gw, wg = warp % C::gw;  // pair group, warp within it
  double* er = (C::global ? a.gws + ((size_t)blockIdx.x * C::pairs) * C::per_warp : smem_d) +
               (size_t)grp * C::per_warp;
  // the group's warps meet on a named barrier (id 1 + group)
  auto gsync = [&]() {
    if constexpr (C::gw > 1)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(C::gw * 32) : "memory");
    else
      __syncwarp();
  };
  double* ei = er + C::R8 * C::L1;
  double* tr = ei + C::R8 * C::L1;
  double* ti = tr + C::R8 * C::L2;
  const int m = a.m;
  const bool train = a.kind == MPSKQ_KIND_TRAIN;
  for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
    const int2 tile = a.tiles[t];
    const int64_t i = tile.x;
    const int64_t j = (int64_t)tile.y * C::pairs + grp;
    if (j >= a.n_kets || (train && i >= j)) continue;  // groups are independent
    const double2* bra = a.bra + i * a.stride;
    const double2* ket = a.ket + j * a.stride;
    const int32_t* bchi = a.bra_chi + i * (m + 1);
    const int32_t* kchi = a.ket_chi + j * (m + 1);
    for (int idx = wg * 32 + lane; idx < 2 * C::R8 * C::L1; idx += C::gw * 32) er[idx] = 0.0;
    gsync();
    if (wg == 0 && lane == 0) er[0] = 1.0;  // env = [[1]]
    gsync();
    for (int s = 0; s < m; ++s) {
      const int na = __ldg(bchi + s), na1 = __ldg(bchi + s + 1);
      const int nb = __ldg(kchi + s), nb1 = __ldg(kchi + s + 1);
      const double2* A = bra + __ldg(a.site_off + s);
      const double2* B = ket + __ldg(a.site_off + s);
      // ---- phase 1: T (na x 2nb1) = env (na x nb) . B (nb x 2nb1)
      {
        const int nt_n = (2 * nb1 + 7) >> 3, mt_n = (na + 7) >> 3, ks_n = (nb + 3) >> 2;
        const int ncol = 2 * nb1;
        const int ntp = (nt_n + 1) >> 1;
        for (int tt = wg; tt < mt_n * ntp; tt += C::gw) {  // output tile pairs split over the group
          const int mt = tt / ntp, nt = (tt - mt * ntp) * 2;
          {
            CTile c0{0, 0, 0, 0}, c1{0, 0, 0, 0};
            const int n0 = nt * 8 + g, n1 = n0 + 8;
            for (int ks = 0; ks < ks_n; ++ks) {
              const int row = mt * 8 + g, kk = ks * 4 + q;
              const double ar = er[row * C::L1 + kk], ai = ei[row * C::L1 + kk];
              double2 b0 = make_double2(0.0, 0.0), b1 = make_double2(0.0, 0.0);
              if (kk < nb) {
                if (n0 < ncol) b0 = __ldg(B + kk * ncol + n0);
                if (n1 < ncol) b1 = __ldg(B + kk * ncol + n1);
              }
              cmma(c0, ar, ai, b0.x, b0.y);
              cmma(c1, ar, ai, b1.x, b1.y);
            }
            const int row = mt * 8 + g, col = nt * 8 + 2 * q;
            tr[row * C::L2 + col] = c0.r0;
            tr[row * C::L2 + col + 1] = c0.r1;
            ti[row * C::L2 + col] = c0.i0;
            ti[row * C::L2 + col + 1] = c0.i1;
            if (nt + 1 < nt_n) {
              tr[row * C::L2 + col + 8] = c1.r0;
              tr[row * C::L2 + col + 9] = c1.r1;
              ti[row * C::L2 + col + 8] = c1.i0;
              ti[row * C::L2 + col + 9] = c1.i1;
            }
          }
        }
      }
      gsync();
      // ---- phase 2: E' (na1 x nb1) = conj(A)^T (na1 x 2na) . T2 (2na x nb1)
      {
        const int nt_n = (nb1 + 7) >> 3, mt_n = (na1 + 7) >> 3, ks_n = (2 * na + 3) >> 2;
        const int ntp = (nt_n + 1) >> 1;
        for (int tt = wg; tt < mt_n * ntp; tt += C::gw) {
          const int mt = tt / ntp, nt = (tt - mt * ntp) * 2;
          {
            CTile c0{0, 0, 0, 0}, c1{0, 0, 0, 0};
            const int ar_ = mt * 8 + g;
            const int n0 = nt * 8 + g, n1 = n0 + 8;
            for (int ks = 0; ks < ks_n; ++ks) {
              const int k = ks * 4 + q;  // (al, p) = (k >> 1, k & 1)
              double2 av = make_double2(0.0, 0.0);
              if (ar_ < na1 && k < 2 * na) av = __ldg(A + k * na1 + ar_);
              // B fragment: T2[kb][n] with kb = ks*4 + q, n = column group g
              const int kb = ks * 4 + q;
              const int trow = kb >> 1, tcol = (kb & 1) * nb1;
              double b0r = 0.0, b0i = 0.0, b1r = 0.0, b1i = 0.0;
              if (n0 < nb1) {
                b0r = tr[trow * C::L2 + tcol + n0];
                b0i = ti[trow * C::L2 + tcol + n0];
              }
              if (n1 < nb1) {
                b1r = tr[trow * C::L2 + tcol + n1];
                b1i = ti[trow * C::L2 + tcol + n1];
              }
              cmma(c0, av.x, -av.y, b0r, b0i);  // conj(A)
              cmma(c1, av.x, -av.y, b1r, b1i);
            }
            const int row = mt * 8 + g, col = nt * 8 + 2 * q;
            er[row * C::L1 + col] = c0.r0;
            er[row * C::L1 + col + 1] = c0.r1;
            ei[row * C::L1 + col] = c0.i0;
            ei[row * C::L1 + col + 1] = c0.i1;
            if (nt + 1 < nt_n) {
              er[row * C::L1 + col + 8] = c1.r0;
              er[row * C::L1 + col + 9] = c1.r1;
              ei[row * C::L1 + col + 8] = c1.i0;
              ei[row * C::L1 + col + 9] = c1.i1;
            }
          }
        }
      }
      gsync();
    }
    if (wg == 0 && lane == 0) store_result(a.out_mode, a.out, a.ld, i, j, make_double2(er[0], ei[0]), train);
    gsync();
  }
}

__global__ void fill_diag_kernel(double* out, int64_t ld, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i * ld + i] = 1.0;
}

int upload_tiles(const std::vector<int2>& tiles, int2** dev, cudaStream_t st) {
  const size_t bytes = sizeof(int2) * (tiles.empty() ? 1 : tiles.size());
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(dev), bytes, st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(tiles)");
  if (!tiles.empty()) {
    e = cudaMemcpyAsync(*dev, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(tiles)");
  }
  return MPSKQ_OK;
}

// tiles of (row block of rb rows, column block of cb columns); train keeps
// the tiles holding some i < j.  Tiles are enumerated super-block by
// super-block (about 384 bras x 384 kets each) so the tiles that run
// concurrently on the 148 SMs share their bra and ket site data in L2.
// Block-cyclic over ranks: tile t goes to rank t % world.
inline int64_t super_rows(int rb) { return std::max<int64_t>(1, 384 / rb); }

// [i_lo, i_hi): row-block range (the host-streaming path enumerates one
// super-row at a time; the default covers every row block)
std::vector<int2> make_tiles(bool train, int64_t n_rows, int64_t n_cols, int rb, int cb, int rank,
                             int world, int64_t i_lo = 0, int64_t i_hi = -1, bool by_band = false) {
  std::vector<int2> tiles;
  const int64_t nrb = (n_rows + rb - 1) / rb, ncb = (n_cols + cb - 1) / cb;
  const int64_t sr = super_rows(rb), sc = std::max<int64_t>(1, 384 / cb);
  const int64_t ihi = i_hi < 0 ? nrb : std::min(nrb, i_hi);
  int64_t t = 0;
  for (int64_t J0 = 0; J0 < ncb; J0 += sc) {
    for (int64_t I0 = i_lo; I0 < ihi; I0 += sr) {
      for (int64_t J = J0; J < std::min(ncb, J0 + sc); ++J) {
        const int64_t jmax = std::min(n_cols, (J + 1) * cb) - 1;
        for (int64_t I = I0; I < std::min(ihi, I0 + sr); ++I) {
          if (train && I * rb >= jmax) break;
          if ((by_band ? I : t) % world == rank) tiles.push_back(make_int2((int)I, (int)J));
          ++t;
        }
      }
    }
  }
  return tiles;
}


int launch_o1(const OverlapArgs& a, cudaStream_t st) {
  const int m = a.m;
  const bool train = a.kind == MPSKQ_KIND_TRAIN;
  const int64_t npb = (a.n_bras + kWarpsO1 - 1) / kWarpsO1 * kWarpsO1;
  const int64_t nbk = (a.n_kets + kLanes - 1) / kLanes;
  const size_t bb = sizeof(double2) * (size_t)m * npb * kEnt;
  const size_t kb = sizeof(double2) * (size_t)m * nbk * kEnt * kLanes;
  const int threads = 256;
  auto blocks_for = [&](int64_t total) {
    return (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 64);
  };
  std::vector<void*> frees;
  auto alloc = [&](void** p, size_t bytes, const char* what) {
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 8, st);
    if (e != cudaSuccess) return cuda_fail(e, what);
    frees.push_back(*p);
    return (int)MPSKQ_OK;
  };
  auto release = [&]() {
    for (void* p : frees) cudaFreeAsync(p, st);
  };
  // order the kets (train: both sides share the order, so i < j stays a triangle)
  void *keys = nullptr, *keys2 = nullptr, *vals = nullptr, *perm = nullptr, *narrow = nullptr, *tmp = nullptr;
  int s_ = MPSKQ_OK;
  if ((s_ = alloc(&keys, sizeof(uint32_t) * a.n_kets, "keys")) || (s_ = alloc(&keys2, sizeof(uint32_t) * a.n_kets, "keys")) ||
      (s_ = alloc(&vals, sizeof(int32_t) * a.n_kets, "vals")) || (s_ = alloc(&perm, sizeof(int32_t) * a.n_kets, "perm")) ||
      (s_ = alloc(&narrow, (size_t)nbk * (m + 1), "narrow"))) {
    release();
    return s_;
  }
  ket_key_kernel<<<blocks_for(a.n_kets), threads, 0, st>>>(a.ket_chi, m, a.n_kets, static_cast<uint32_t*>(keys),
                                                           static_cast<int32_t*>(vals));
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, static_cast<uint32_t*>(keys), static_cast<uint32_t*>(keys2),
                                  static_cast<int32_t*>(vals), static_cast<int32_t*>(perm), (int)a.n_kets, 0, 32, st);
  if ((s_ = alloc(&tmp, tmp_bytes, "sort scratch"))) {
    release();
    return s_;
  }
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, static_cast<uint32_t*>(keys), static_cast<uint32_t*>(keys2),
                                  static_cast<int32_t*>(vals), static_cast<int32_t*>(perm), (int)a.n_kets, 0, 32, st);
  if ((m + 1 + 31) / 32 <= kClusterMaxWords) {
    void* refined = nullptr;
    if ((s_ = alloc(&refined, sizeof(int32_t) * a.n_kets, "refined perm"))) {
      release();
      return s_;
    }
    const int groups = (int)((a.n_kets + kClusterGroup - 1) / kClusterGroup);
    if (groups > 0)
      cluster_kets_kernel<<<groups, kClusterGroup, 0, st>>>(a.ket_chi, m, a.n_kets, static_cast<const int32_t*>(perm),
                                                             static_cast<int32_t*>(refined));
    perm = refined;
  }
  const int32_t* kperm = static_cast<const int32_t*>(perm);
  const int32_t* bperm = train ? kperm : nullptr;
  void *kinv = nullptr, *ordered = nullptr;
  const size_t elem = a.out_mode == MPSKQ_OUT_KERNEL ? sizeof(double) : sizeof(double2);
  if ((s_ = alloc(&kinv, sizeof(int32_t) * a.n_kets, "inverse perm")) ||
      (s_ = alloc(&ordered, elem * (size_t)a.n_bras * a.n_kets, "ordered results"))) {
    release();
    return s_;
  }
  invert_perm_kernel<<<blocks_for(a.n_kets), threads, 0, st>>>(kperm, a.n_kets, static_cast<int32_t*>(kinv));
  if (a.world > 1 && !a.owned) cudaMemsetAsync(ordered, 0, elem * (size_t)a.n_bras * a.n_kets, st);
  block_narrow_kernel<<<blocks_for(nbk * (m + 1)), threads, 0, st>>>(a.ket_chi, kperm, m, a.n_kets, nbk,
                                                                    static_cast<uint8_t*>(narrow));
  void *bra = nullptr, *ket = nullptr;
  if ((s_ = alloc(&bra, bb, "packed bras")) || (s_ = alloc(&ket, kb, "packed kets"))) {
    release();
    return s_;
  }
  pack_bra_kernel<<<blocks_for((int64_t)m * npb * kEnt), threads, 0, st>>>(
      reinterpret_cast<const double2*>(a.bra_sites), a.bra_chi, a.site_off, a.state_stride, m,
      a.n_bras, npb, bperm, static_cast<double2*>(bra));
  pack_o1_kernel<<<blocks_for((int64_t)m * nbk * kEnt * kLanes), threads, 0, st>>>(
      reinterpret_cast<const double2*>(a.ket_sites), a.ket_chi, a.site_off, a.state_stride, m,
      a.n_kets, nbk, kperm, static_cast<double2*>(ket));
  // host streaming: one tile list per super-row band, concatenated
  const bool to_host = a.host_out != nullptr && a.out_mode == MPSKQ_OUT_KERNEL && a.world == 1;
  std::vector<int64_t> band_rows{0}, band_tiles{0};  // band b: ordered rows / tiles [b], [b+1]
  std::vector<int2> tiles;
  if (to_host) {
    const int64_t nrb = npb / kWarpsO1, sr = super_rows(kWarpsO1);
    for (int64_t I0 = 0; I0 < nrb; I0 += sr) {
      auto t = make_tiles(train, a.n_bras, a.n_kets, kWarpsO1, kLanes, 0, 1, I0, I0 + sr);
      tiles.insert(tiles.end(), t.begin(), t.end());
      band_rows.push_back(std::min<int64_t>(a.n_bras, (I0 + sr) * kWarpsO1));
      band_tiles.push_back((int64_t)tiles.size());
    }
  } else {
    tiles = make_tiles(train, a.n_bras, a.n_kets, kWarpsO1, kLanes, a.rank, a.world, 0, -1, a.owned);
    band_rows.push_back(a.n_bras);
    band_tiles.push_back((int64_t)tiles.size());
  }
  int2* dtiles = nullptr;
  if ((s_ = upload_tiles(tiles, &dtiles, st))) {
    release();
    return s_;
  }
  frees.push_back(dtiles);
  cudaError_t e = cudaSuccess;
  if (to_host) {
    O1Launch lk = o1_launch_for(m);
    const size_t smem = lk.smem;
    e = cudaFuncSetAttribute(lk.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);

    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "cudaFuncSetAttribute(o1)");
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Bands alternate between two streams so band b+1's CTAs take the SMs
    // that band b's tail frees (no idle tail per launch).  Band b's rows are
    // final once bands <= b ran (train mirrors only write into later rows),
    // i.e. after the events of b and b-1 (each stream is ordered); the side
    // stream then writes them to the host.
    cudaStream_t side = nullptr, alt = nullptr;
    if ((e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking)) == cudaSuccess &&
        (e = cudaStreamCreateWithFlags(&alt, cudaStreamNonBlocking)) != cudaSuccess) {
      cudaStreamDestroy(side);
    }
    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "cudaStreamCreate(side)");
    }
    const int32_t* row_of = train ? kperm : nullptr;
    const int bands = (int)band_rows.size() - 1;
    std::vector<cudaEvent_t> evs(bands + 3, nullptr);
    for (auto& ev : evs)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) {
      cudaEventRecord(evs[bands], st);  // packs, ordering and tiles are ready
      cudaStreamWaitEvent(alt, evs[bands], 0);
    }
    for (int b = 0; b < bands && e == cudaSuccess; ++b) {
      cudaStream_t sb = (b & 1) ? alt : st;
      const int64_t nt = band_tiles[b + 1] - band_tiles[b];
      if (nt > 0) {
        O1Args o{static_cast<const double2*>(bra), static_cast<const double2*>(ket), a.bra_chi,
                 a.n_bras, a.n_kets, npb, nbk, m, a.kind,
                 a.out_mode, dtiles + band_tiles[b], nt, static_cast<double*>(ordered), a.n_kets,
                 bperm, kperm, static_cast<const uint8_t*>(narrow)};
        lk.fn<<<(int)std::min<int64_t>(nt, (int64_t)sms * kCtasO1), kThreadsO1Ws, smem, sb>>>(o);
      }
      cudaEventRecord(evs[b], sb);
      cudaStreamWaitEvent(side, evs[b], 0);
      if (b > 0) cudaStreamWaitEvent(side, evs[b - 1], 0);
      const int64_t r0 = band_rows[b], r1 = band_rows[b + 1];
      if (r1 > r0)
        rows_to_host_kernel<<<(int)std::min<int64_t>(r1 - r0, 296), 256, 0, side>>>(
            static_cast<const double*>(ordered), a.n_kets, row_of, r0, r1,
            static_cast<const int32_t*>(kinv), train, a.host_out, a.ld);
      e = cudaGetLastError();
    }
    // A failed launch part-way through: bands already queued may still write
    // into the caller's host K, so drain every stream before reporting it
    // (the caller may free or reuse K_out as soon as it sees the error).
    if (e != cudaSuccess) {
      cudaStreamSynchronize(st);
      cudaStreamSynchronize(alt);
      cudaStreamSynchronize(side);
    }
    // join: the main stream (and the buffer frees below) wait for both
    if (evs[bands + 2]) {
      cudaEventRecord(evs[bands + 1], alt);
      cudaStreamWaitEvent(st, evs[bands + 1], 0);
      cudaEventRecord(evs[bands + 2], side);
      cudaStreamWaitEvent(st, evs[bands + 2], 0);
    } else {
      cudaStreamSynchronize(alt);
      cudaStreamSynchronize(side);
    }
    for (auto ev : evs)
      if (ev) cudaEventDestroy(ev);
    cudaStreamDestroy(alt);
    cudaStreamDestroy(side);
    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "overlap_o1 host streaming");
    }
  } else if (!tiles.empty()) {
    O1Launch lk = o1_launch_for(m);
    const size_t smem = lk.smem;
    e = cudaFuncSetAttribute(lk.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);

    if (e != cudaSuccess) {
      release();
      return cuda_fail(e, "cudaFuncSetAttribute(o1)");
    }
    O1Args o{static_cast<const double2*>(bra), static_cast<const double2*>(ket), a.bra_chi,
             a.n_bras, a.n_kets, npb, nbk, m, a.kind,
             a.out_mode, dtiles, (int64_t)tiles.size(), static_cast<double*>(ordered), a.n_kets,
             bperm, kperm, static_cast<const uint8_t*>(narrow)};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // persistent: one CTA per SM walks the tile list (the ring stays warm)
    const int grid = (int)std::min<int64_t>((int64_t)tiles.size(), (int64_t)sms * kCtasO1);
    lk.fn<<<grid, kThreadsO1Ws, smem, st>>>(o);
    const int32_t* bpos = train ? static_cast<const int32_t*>(kinv) : nullptr;
    const int rows = (int)std::min<int64_t>(a.n_bras, 148 * 32);
    if (a.owned) {
      const int64_t n_owned = owned_row_count(4, a.n_bras, a.rank, a.world);
      if (n_owned > 0)
        owned_rows_kernel<<<(int)std::min<int64_t>(n_owned, 148 * 32), 256, 0, st>>>(
            static_cast<const double*>(ordered), a.n_bras, a.n_kets, kWarpsO1, a.rank, a.world,
            train ? kperm : nullptr, static_cast<const int32_t*>(kinv), a.rows_out, a.row_ids_out, n_owned);
      if (a.ket_pos_out)
        cudaMemcpyAsync(a.ket_pos_out, kinv, sizeof(int32_t) * a.n_kets, cudaMemcpyDeviceToDevice, st);
    } else if (a.out_mode == MPSKQ_OUT_KERNEL)
      unpermute_kernel<double><<<rows, 256, 0, st>>>(static_cast<const double*>(ordered), a.n_kets, bpos,
                                                     static_cast<const int32_t*>(kinv), a.n_bras, a.out, a.ld);
    else
      unpermute_kernel<double2><<<rows, 256, 0, st>>>(static_cast<const double2*>(ordered), a.n_kets, bpos,
                                                       static_cast<const int32_t*>(kinv), a.n_bras,
                                                       reinterpret_cast<double2*>(a.out), a.ld);
  }
  e = cudaGetLastError();
  release();
  if (e != cudaSuccess) return cuda_fail(e, "overlap_o1 launch");
  return MPSKQ_OK;
}

template <int CAP>
int launch_mma(const OverlapArgs& a, cudaStream_t st) {
  using C = MmaCfg<CAP>;
  cudaError_t e = cudaSuccess;
  if (C::smem > 48 * 1024) {
    e = cudaFuncSetAttribute(overlap_mma_kernel<CAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(mma)");
  }
  const bool train = a.kind == MPSKQ_KIND_TRAIN;
  auto tiles = make_tiles(train, a.n_bras, a.n_kets, 1, C::pairs, a.rank, a.world, 0, -1, a.owned);
  int2* dtiles = nullptr;
  if (int s = upload_tiles(tiles, &dtiles, st)) return s;
  double* full = nullptr;  // row ownership: the rank's rows in a full-size buffer, then compacted
  if (a.owned && !tiles.empty()) {
    e = cudaMallocAsync(reinterpret_cast<void**>(&full), sizeof(double) * std::max<int64_t>(1, a.n_bras * a.n_kets), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(owned rows)");
  }
  if (!tiles.empty()) {
    MmaArgs o{reinterpret_cast<const double2*>(a.bra_sites),
              reinterpret_cast<const double2*>(a.ket_sites),
              a.bra_chi,
              a.ket_chi,
              a.site_off,
              a.state_stride,
              a.n_bras,
              a.n_kets,
              a.m,
              a.kind,
              a.out_mode,
              dtiles,
              (int64_t)tiles.size(),
              full ? full : a.out,
              full ? a.n_kets : a.ld,
              nullptr};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>((int64_t)tiles.size(), (int64_t)sms * (C::global ? 2 * C::ctas_per_sm : 16));
    if (C::global) {
      e = cudaMallocAsync(reinterpret_cast<void**>(&o.gws),
                          sizeof(double) * (size_t)C::per_warp * C::pairs * grid, st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(mma planes)");
    }
    overlap_mma_kernel<CAP><<<grid, C::warps * 32, C::smem, st>>>(o);
    if (o.gws) cudaFreeAsync(o.gws, st);
  }
  if (full) {
    const int64_t n_owned = owned_row_count(CAP, a.n_bras, a.rank, a.world);
    if (n_owned > 0)
      owned_rows_kernel<<<(int)std::min<int64_t>(n_owned, 148 * 32), 256, 0, st>>>(
          full, a.n_bras, a.n_kets, 1, a.rank, a.world, nullptr, nullptr, a.rows_out, a.row_ids_out, n_owned);
    cudaFreeAsync(full, st);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "overlap_mma launch");
  cudaFreeAsync(dtiles, st);
  return MPSKQ_OK;
}

}  // namespace

int launch_overlap(const OverlapArgs& a, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  int s = MPSKQ_OK;
  switch (a.chi_cap) {
    case 4: s = launch_o1(a, st); break;
    case 8: s = launch_mma<8>(a, st); break;
    case 12: s = launch_mma<12>(a, st); break;
    case 16: s = launch_mma<16>(a, st); break;
    case 24: s = launch_mma<24>(a, st); break;
    case 32: s = launch_mma<32>(a, st); break;
    case 48: s = launch_mma<48>(a, st); break;
    case 64: s = launch_mma<64>(a, st); break;
    case 80: s = launch_mma<80>(a, st); break;
    case 96: s = launch_mma<96>(a, st); break;
    case 128: s = launch_mma<128>(a, st); break;
    default: return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", a.chi_cap);
  }
  if (s != MPSKQ_OK) return s;
  if (a.kind == MPSKQ_KIND_TRAIN && a.out_mode == MPSKQ_OUT_KERNEL && a.rank == 0 && !a.owned &&
      !(a.host_out && a.chi_cap == 4 && a.world == 1)) {
    fill_diag_kernel<<<(int)std::min<int64_t>((a.n_bras + 255) / 256, 1024), 256, 0, st>>>(
        a.out, a.ld, a.n_bras);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fill_diag launch");
  }
  return MPSKQ_OK;
}

int64_t owned_row_count(int chi_cap, int64_t n_bras, int rank, int world) {
  const int64_t rb = chi_cap == 4 ? kWarpsO1 : 1;
  const int64_t nbands = (n_bras + rb - 1) / rb;
  int64_t n = 0;
  for (int64_t b = rank; b < nbands; b += world) n += std::min<int64_t>(rb, n_bras - b * rb);
  // compact indexing assumes full bands before the last one of this rank
  return n == 0 ? 0 : ((n + rb - 1) / rb) * rb;
}

// Gatherer side of row ownership: scatter the ranks' compact rows into K
// (caller order) and, for the train kind, complete every entry whose row was
// not the computing one: K[a][b] = K[b][a] when pos[b] < pos[a] (pos = the
// ordered position, identity without one); unit diagonal.  32x32 tiles
// through shared memory keep both reads coalesced.
__global__ void scatter_rows_kernel(const double* __restrict__ rows, const int32_t* __restrict__ ids,
                                    int64_t n_rows, int64_t nk, double* __restrict__ K, int64_t ld) {
  for (int64_t k = blockIdx.x; k < n_rows; k += gridDim.x) {
    const int32_t a = ids[k];
    if (a < 0) continue;
    for (int64_t b = threadIdx.x; b < nk; b += blockDim.x) K[(int64_t)a * ld + b] = rows[k * nk + b];
  }
}

__global__ void mirror_by_pos_kernel(double* __restrict__ K, int64_t n, int64_t ld,
                                     const int32_t* __restrict__ pos) {
  __shared__ double t1[32][33], t2[32][33];
  const int64_t nt = (n + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < nt * nt; tile += gridDim.x) {
    const int64_t A = tile / nt, B = tile % nt;
    if (A > B) continue;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    for (int r = ty; r < 32; r += 8) {
      const int64_t a = A * 32 + r, b = B * 32 + tx;
      t1[r][tx] = (a < n && b < n) ? K[a * ld + b] : 0.0;  // block (A, B)
      const int64_t a2 = B * 32 + r, b2 = A * 32 + tx;
      t2[r][tx] = (a2 < n && b2 < n) ? K[a2 * ld + b2] : 0.0;  // block (B, A)
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      // (a, b) in block (A, B): a = A*32 + r, b = B*32 + tx
      const int64_t a = A * 32 + r, b = B * 32 + tx;
      if (a < n && b < n) {
        const int pa = pos ? pos[a] : (int)a, pb = pos ? pos[b] : (int)b;
        K[a * ld + b] = a == b ? 1.0 : (pa < pb ? t1[r][tx] : t2[tx][r]);
      }
      const int64_t a2 = B * 32 + r, b2 = A * 32 + tx;
      if (a2 < n && b2 < n) {
        const int pa = pos ? pos[a2] : (int)a2, pb = pos ? pos[b2] : (int)b2;
        K[a2 * ld + b2] = a2 == b2 ? 1.0 : (pa < pb ? t2[r][tx] : t1[tx][r]);
      }
    }
    __syncthreads();
  }
}

int assemble_rows(int kind, int64_t n_bras, int64_t n_kets, const double* rows, const int32_t* ids, int64_t n_rows,
                  const int32_t* ket_pos, double* K, int64_t ld, cudaStream_t st) {
  if (n_rows > 0)
    scatter_rows_kernel<<<(int)std::min<int64_t>(n_rows, 148 * 32), 256, 0, st>>>(rows, ids, n_rows, n_kets, K, ld);
  if (kind == MPSKQ_KIND_TRAIN && n_bras > 0) {
    const int64_t nt = (n_bras + 31) / 32;
    mirror_by_pos_kernel<<<(int)std::min<int64_t>(nt * nt, 148 * 16), 256, 0, st>>>(K, n_bras, ld, ket_pos);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "assemble_rows launch");
  return MPSKQ_OK;
}

void tile_shape(int chi_cap, int* rb, int* cb) {
  switch (chi_cap) {
    case 4: *rb = kWarpsO1; *cb = kLanes; return;
    case 8: *rb = 1; *cb = MmaCfg<8>::pairs; return;
    case 12: *rb = 1; *cb = MmaCfg<12>::pairs; return;
    case 16: *rb = 1; *cb = MmaCfg<16>::pairs; return;
    case 24: *rb = 1; *cb = MmaCfg<24>::pairs; return;
    case 32: *rb = 1; *cb = MmaCfg<32>::pairs; return;
    case 48: *rb = 1; *cb = MmaCfg<48>::pairs; return;
    case 64: *rb = 1; *cb = MmaCfg<64>::pairs; return;
    case 80: *rb = 1; *cb = MmaCfg<80>::pairs; return;
    case 96: *rb = 1; *cb = MmaCfg<96>::pairs; return;
    default: *rb = 1; *cb = MmaCfg<128>::pairs; return;
  }
}

}  // namespace mpskq

extern "C" int mpskq_overlap_tiles(int kind, int chi_cap, int64_t n_bras, int64_t n_kets, int rank,
                                   int world, int32_t* tiles, int64_t cap, int64_t* n_tiles,
                                   int32_t* row_block, int32_t* col_block) {
  using namespace mpskq;
  if (kind != MPSKQ_KIND_TRAIN && kind != MPSKQ_KIND_TEST)
    return fail(MPSKQ_ERR_INVALID, "kind must be one of ('train', 'test')");
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (world < 1 || rank < 0 || rank >= world)
    return fail(MPSKQ_ERR_INVALID, "bad rank %d of world %d", rank, world);
  if (n_bras < 0 || n_kets < 0) return fail(MPSKQ_ERR_INVALID, "negative state counts");
  int rb = 1, cb = 1;
  tile_shape(chi_cap, &rb, &cb);
  if (row_block) *row_block = rb;
  if (col_block) *col_block = cb;
  auto t = make_tiles(kind == MPSKQ_KIND_TRAIN, n_bras, n_kets, rb, cb, rank, world);
  if (n_tiles) *n_tiles = (int64_t)t.size();
  if (!tiles) return MPSKQ_OK;
  if (cap < (int64_t)t.size()) return fail(MPSKQ_ERR_INVALID, "tile buffer too small");
  for (size_t i = 0; i < t.size(); ++i) {
    tiles[2 * i] = t[i].x;
    tiles[2 * i + 1] = t[i].y;
  }
  return MPSKQ_OK;
}

extern "C" int mpskq_owned_rows(int chi_cap, int64_t n_bras, int rank, int world, int64_t* n_owned) {
  using namespace mpskq;
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (world < 1 || rank < 0 || rank >= world)
    return fail(MPSKQ_ERR_INVALID, "bad rank %d of world %d", rank, world);
  if (n_bras < 0) return fail(MPSKQ_ERR_INVALID, "negative state counts");
  if (n_owned) *n_owned = owned_row_count(chi_cap, n_bras, rank, world);
  return MPSKQ_OK;
}

extern "C" int mpskq_overlap_owned_rows(int kind, int m, int chi_cap, const int64_t* site_off_dev,
                                        int64_t state_stride, const double* bra_sites_dev,
                                        const int32_t* bra_chi_dev, int64_t n_bras, const double* ket_sites_dev,
                                        const int32_t* ket_chi_dev, int64_t n_kets, int rank, int world,
                                        double* rows_out_dev, int32_t* row_ids_dev, int32_t* ket_pos_dev,
                                        void* stream) {
  using namespace mpskq;
  if (kind != MPSKQ_KIND_TRAIN && kind != MPSKQ_KIND_TEST)
    return fail(MPSKQ_ERR_INVALID, "kind must be one of ('train', 'test')");
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (kind == MPSKQ_KIND_TRAIN &&
      (n_bras != n_kets || bra_sites_dev != ket_sites_dev || bra_chi_dev != ket_chi_dev))
    return fail(MPSKQ_ERR_INVALID, "train kind requires bras and kets to be the same states");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(MPSKQ_ERR_INVALID, "bad rank %d of world %d", rank, world);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_owned = owned_row_count(chi_cap, n_bras, rank, world);
  if (n_owned > 0 && (!rows_out_dev || !row_ids_dev))
    return fail(MPSKQ_ERR_INVALID, "owned-row outputs are required");
  if (n_owned > 0) {
    // padding rows of a short last band keep id -1 (skipped by the scatter)
    cudaError_t e = cudaMemsetAsync(row_ids_dev, 0xff, sizeof(int32_t) * n_owned, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(row ids)");
  }
  if (ket_pos_dev && chi_cap != 4) {
    std::vector<int32_t> id(n_kets);
    for (int64_t i = 0; i < n_kets; ++i) id[i] = (int32_t)i;
    cudaError_t e = cudaMemcpyAsync(ket_pos_dev, id.data(), sizeof(int32_t) * n_kets, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "ket positions");
  }
  if (n_bras == 0 || n_kets == 0) return MPSKQ_OK;
  if (n_owned == 0 && !ket_pos_dev) return MPSKQ_OK;  // nothing to compute on this rank
  OverlapArgs a{kind, MPSKQ_OUT_KERNEL, m, chi_cap, site_off_dev, state_stride, bra_sites_dev, bra_chi_dev,
                n_bras, ket_sites_dev, ket_chi_dev, n_kets, rank, world, nullptr, n_kets};
  a.owned = true;
  a.rows_out = rows_out_dev;
  a.row_ids_out = row_ids_dev;
  a.ket_pos_out = ket_pos_dev;
  return launch_overlap(a, stream);
}

extern "C" int mpskq_assemble_rows(int kind, int64_t n_bras, int64_t n_kets, const double* rows_dev,
                                   const int32_t* row_ids_dev, int64_t n_rows, const int32_t* ket_pos_dev,
                                   double* K_dev, int64_t ld, void* stream) {
  using namespace mpskq;
  if (kind != MPSKQ_KIND_TRAIN && kind != MPSKQ_KIND_TEST)
    return fail(MPSKQ_ERR_INVALID, "kind must be one of ('train', 'test')");
  if (kind == MPSKQ_KIND_TRAIN && n_bras != n_kets)
    return fail(MPSKQ_ERR_INVALID, "train kind requires a square matrix");
  if (ld < n_kets || n_rows < 0) return fail(MPSKQ_ERR_INVALID, "bad assembly sizes");
  return assemble_rows(kind, n_bras, n_kets, rows_dev, row_ids_dev, n_rows, ket_pos_dev, K_dev, ld,
                       static_cast<cudaStream_t>(stream));
}
