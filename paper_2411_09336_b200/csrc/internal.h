// Internal declarations shared by the host runtime (runtime.cpp) and the CUDA
// translation units.  Nothing here crosses the C ABI.
#pragma once

#include <cstdint>
#include <string>

#include "mpskq.h"

namespace mpskq {

// thread-local last error; returns `status` so callers can `return fail(...)`
int fail(int status, const char* fmt, ...);
int cuda_fail(int err, const char* what);  // err is a cudaError_t

// chi capacities with a compiled simulation + overlap path
constexpr int kChiCaps[] = {4, 8, 12, 16, 24, 32, 48, 64, 80, 96, 128};
constexpr int kNumChiCaps = sizeof(kChiCaps) / sizeof(kChiCaps[0]);
inline bool chi_cap_supported(int c) {
  for (int x : kChiCaps)
    if (x == c) return true;
  return false;
}

// Keep the device's stream-ordered pool pages between calls (the default
// release threshold 0 hands them back to the driver at every synchronisation,
// and re-mapping a GB of workspace costs tens of ms).  Idempotent, cheap.
void retain_pool_memory();

// layout helper (also used on device through the site_off table)
int64_t bond_cap(int m, int chi_cap, int b);

struct SimArgs {
  int m;
  int chi_cap;
  const int32_t* ops;  // n_ops x 4
  int64_t n_ops;
  int64_t n_gates;
  const double* coef;  // n_states x n_params x 2
  int64_t n_params;
  int64_t n_states;
  double budget;
  int chi_max;
  const int64_t* site_off;
  int64_t state_stride;
  double* sites;
  int32_t* chi;
  double* discard;
  int32_t* peak;
  int32_t* status;
  int64_t* entry_log;
  void* scratch;  // set by the launcher (rotation logs of capacities > 32)
  int from_input = 0;                // continue the states already in sites/chi/discard/peak
  long long* phase_cycles = nullptr;  // n_states x {canonicalize, one_qubit, two_qubit}
  double* nominal_flops = nullptr;    // n_states: nominal flop count of the replayed ops
};
int launch_simulate(const SimArgs& a, void* stream);

struct SvdArgs {
  int rows, cols;
  int64_t batch;
  const double* mats;
  double budget;
  int chi_max;
  double *u, *s, *vh;
  int32_t* keep;
  double* discarded;
  int32_t* status;
  void* scratch;
};
int launch_svd(const SvdArgs& a, void* stream);

struct OverlapArgs {
  int kind, out_mode, m, chi_cap;
  const int64_t* site_off;
  int64_t state_stride;
  const double* bra_sites;
  const int32_t* bra_chi;
  int64_t n_bras;
  const double* ket_sites;
  const int32_t* ket_chi;
  int64_t n_kets;
  int rank, world;
  double* out;
  int64_t ld;
  // optional: pinned, device-mapped host K (train/test kernel values, chi <= 4
  // path, one rank).  The overlap then runs one launch per super-row of bra
  // tiles and a side stream writes each finished row band straight into host
  // memory while the next band computes; `out` is not touched.
  double* host_out = nullptr;
  // optional (world > 1): row ownership instead of tile ownership.  The rank
  // computes the rows of the bra bands it owns (band b -> rank b % world;
  // O1: bands of 8 ordered rows, generic: single rows) and writes them
  // compactly in caller column order: rows_out[k * n_kets + j], caller row
  // row_ids_out[k].  Train rows hold only the entries the rank computed
  // (ordered i < j); mpskq_assemble_rows mirrors the rest on the gatherer.
  // ket_pos_out (nullable): ordered position of every ket (train mirror).
  bool owned = false;
  double* rows_out = nullptr;
  int32_t* row_ids_out = nullptr;
  int32_t* ket_pos_out = nullptr;
};
// overlap tile shape (bra rows x ket columns) of a capacity
void tile_shape(int chi_cap, int* rb, int* cb);
// rows of n_bras owned by `rank` under row ownership for this capacity
int64_t owned_row_count(int chi_cap, int64_t n_bras, int rank, int world);
int launch_overlap(const OverlapArgs& a, void* stream);

// move states between chi-capacity layouts: src row i -> dst row dst_rows[i]
int launch_relayout(int m, int64_t n, const double* src, const int64_t* src_off, int64_t src_stride,
                    const int32_t* chi, double* dst, const int64_t* dst_off, int64_t dst_stride,
                    const int32_t* dst_rows, void* stream);

// dst row dst_idx[i] = src row src_idx[i] (nullable indices = identity)
int launch_copy_rows(const void* src, void* dst, int64_t row_bytes, int64_t n, const int32_t* src_idx,
                     const int32_t* dst_idx, void* stream);

int launch_pack_exact(int m, int64_t n, double* sites, const int64_t* site_off, int64_t stride, const int32_t* chi,
                      const int64_t* state_off, double* packed, int unpack, const int32_t* rows, void* stream);

int launch_encode(const double* X, int64_t n_rows, int m, int r, int d, double gamma, double* coef,
                  int* bad, void* stream);

int launch_fp64_probe(int n_blocks, int64_t iters, double* out, void* stream);

}  // namespace mpskq
