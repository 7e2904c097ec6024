/*
 * mpskq.h — C ABI of the B200-native quantum-kernel hot path
 * (feature-map MPS simulation + kernel-matrix overlaps of arXiv 2411.09336).
 *
 * The reference (`mpskernel`, pure Python + numpy) has no FFI layer; its
 * boundary is the Python API.  Every entry point below replaces the numpy
 * arithmetic underneath one reference function, cited as
 * /root/reference/pkg/src/mpskernel/<file>:<line>.  The Python package
 * `paper_2411_09336_b200` binds these with ctypes and
 * re-exports the reference's names on top.
 *
 * Conventions
 *   - Plain C types only.  "_dev" pointers are CUDA device pointers allocated
 *     by the caller (the library owns only transient per-call workspace).
 *   - Complex numbers are complex128 stored as interleaved (re, im) doubles,
 *     exactly numpy's complex128 memory layout.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - Every function returns MPSKQ_OK (0) or a negative status; the message of
 *     the last failure on the calling thread is available from
 *     mpskq_last_error().  No exceptions or aborts cross the ABI.
 *   - A process may call from several host threads; each call is independent.
 */
#ifndef MPSKQ_H
#define MPSKQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPSKQ_ABI_VERSION 1

/* status codes */
#define MPSKQ_OK 0
#define MPSKQ_ERR_INVALID (-1)  /* bad argument: maps to the reference's ValueError */
#define MPSKQ_ERR_CUDA (-2)     /* CUDA runtime failure */
#define MPSKQ_ERR_CAPACITY (-3) /* a bond outgrew the compiled chi capacity */
#define MPSKQ_ERR_NUMERIC (-4)  /* non-finite tensor entries (tensor.py:100-101) */
#define MPSKQ_ERR_NOMEM (-5)    /* device or host allocation failed */

/* per-state status words written by mpskq_simulate */
#define MPSKQ_STATE_OK 0
#define MPSKQ_STATE_CAPACITY 1
#define MPSKQ_STATE_NONFINITE 2
#define MPSKQ_STATE_NOCONV 3 /* Jacobi SVD without a quiet cycle in 40 sweeps (zgesdd's LinAlgError) */

/* gate kinds (ansatz.py:15 GATE_KINDS order) */
#define MPSKQ_GATE_H 0
#define MPSKQ_GATE_RZ 1
#define MPSKQ_GATE_RXX 2
#define MPSKQ_GATE_SWAP 3

/* program op codes (one int32x4 per op: {code | absorb<<8, site, param_slot, gate_index}) */
#define MPSKQ_OP_H 1    /* apply_one_qubit with H          mps.py:147-160 */
#define MPSKQ_OP_RZ 2   /* apply_one_qubit with RZ(theta)  mps.py:147-160, ansatz.py:93-94 */
#define MPSKQ_OP_RXX 3  /* apply_two_qubit with RXX(theta) mps.py:163-205, ansatz.py:95-99 */
#define MPSKQ_OP_SWAP 4 /* apply_two_qubit with SWAP       mps.py:163-205, ansatz.py:77-79 */
#define MPSKQ_OP_QRL 5  /* one _left_isometrize step       mps.py:105-111 */
#define MPSKQ_OP_QRR 6  /* one _right_isometrize step      mps.py:114-120 */
#define MPSKQ_OP_U1 7   /* apply_one_qubit with an arbitrary 2x2 matrix: 4 complex coefficients
                           (row-major) from param_slot on              mps.py:147-160 */
#define MPSKQ_OP_U2 8   /* apply_two_qubit with an arbitrary 4x4 matrix on |q, q+1>: 16 complex
                           coefficients (row-major) from param_slot on mps.py:163-205 */
#define MPSKQ_ABSORB_LEFT 1

/* kinds of Gram matrix (kernel.py:31 KINDS) */
#define MPSKQ_KIND_TRAIN 0
#define MPSKQ_KIND_TEST 1
/* overlap output modes */
#define MPSKQ_OUT_KERNEL 0    /* out[i*ld+j] = |<bra_i|ket_j>|^2 (double) */
#define MPSKQ_OUT_AMPLITUDE 1 /* out[(i*ld+j)*2 + {0,1}] = <bra_i|ket_j> (complex128) */

int mpskq_abi_version(void);
const char* mpskq_last_error(void);
/* number of CUDA devices visible (0 on a CPU-only host; never fails) */
int mpskq_device_count(void);

/* ---------------------------------------------------------------- topology
 * Gate sequence of encode_circuit(x, cfg) = route_linear(schedule_circuit(
 * build_circuit(x, cfg), d)) — ansatz.py:218-220 (build :109-136, schedule
 * :139-184, route :187-215).  It does not depend on the data row, so it is
 * produced once per (m, r, d).  param_slot[g] is the index of the gate's angle
 * in the per-row parameter vector (build order: per layer m RZ then |E| RXX),
 * or -1 for H/SWAP.  Call with kinds == NULL to query n_gates/n_params.   */
int mpskq_feature_map_topology(int m, int r, int d, int32_t* kinds, int32_t* q0, int32_t* q1,
                               int32_t* param_slot, int64_t cap, int64_t* n_gates,
                               int64_t* n_params);

/* Per-row angles in parameter-slot order, evaluated with the reference's
 * floating-point expression order: RZ 2*gamma*x_q (ansatz.py:130),
 * RXX 2*gamma^2*(pi/2)*(1-x_i)*(1-x_j) (ansatz.py:132).  Rejects rows outside
 * [0, 2] or non-finite like build_circuit (ansatz.py:118-124).            */
int mpskq_feature_map_angles(const double* X, int64_t n_rows, int m, int r, int d, double gamma,
                             double* angles);

/* (cos(a/2), sin(a/2)) per angle with the host libm, i.e. the entries of
 * gate_matrix (ansatz.py:92-99): RZ = diag(c - i s, c + i s), RXX = c I - i s XX. */
int mpskq_half_angle_coefficients(const double* angles, int64_t n, double* coef);

/* Device twin of the two calls above: X_dev (n_rows x m, device) ->
 * coef_dev (n_rows x n_params x {cos, sin}), angles bitwise as above, sin/cos
 * by CUDA (<= 2 ulp from libm).  *bad_dev (device int, caller zeroes it)
 * gets bit 1 if a finite feature lies outside [0, 2] and bit 2 if a feature
 * is not finite (build_circuit's checks, ansatz.py:118-124).              */
int mpskq_feature_map_coefficients_device(const double* X_dev, int64_t n_rows, int m, int r,
                                          int d, double gamma, double* coef_dev, int* bad_dev,
                                          void* stream);

/* Compile a gate list into the op program replayed by mpskq_simulate:
 * run_circuit's absorb rule (mps.py:235-241) and the canonicalize moves
 * before every two-qubit gate (mps.py:181, :123-138), starting from
 * ortho_center = 0 (init_state, mps.py:102).  Two-qubit gates must act on
 * adjacent qubits (mps.py:217-218).  ops receives 4 int32 per op.  Call with
 * ops == NULL to query n_ops.                                              */
int mpskq_program_compile(int m, int64_t n_gates, const int32_t* kinds, const int32_t* q0,
                          const int32_t* q1, const int32_t* param_slot, int32_t* ops,
                          int64_t cap_ops, int64_t* n_ops, int64_t* n_qr_left,
                          int64_t* n_qr_right);

/* ---------------------------------------------------------------- batch layout
 * A batch of MPS (MpsState, mps.py:31-77) lives in one complex128 slab:
 * state n, site s starts at complex offset n*state_stride + site_off[s] and
 * holds the (chi_s, 2, chi_{s+1}) tensor in the reference's row-major order.
 * Slot s has room for 2*cap_s*cap_{s+1} entries, cap_b = min(chi_cap,
 * 2^min(b, m-b)).  chi[n*(m+1) + b] is bond b of state n (bond_dims(),
 * mps.py:54-56).                                                          */
int mpskq_batch_layout(int m, int chi_cap, int64_t* site_off /* m+1 */, int64_t* state_stride);
/* chi capacities compiled into the library, ascending (e.g. 4 8 16 32) */
int mpskq_supported_chi_caps(int32_t* caps, int cap, int* n);

/* ---------------------------------------------------------------- simulation
 * simulate_circuit (mps.py:250-257) for n_states rows at once: every state
 * starts at |0..0> (init_state, mps.py:90-102) and replays ops with its own
 * coefficient row coef[n*n_params*2 ...] ((cos, sin) of the half angle per
 * slot).  Two-qubit ops run apply_two_qubit (mps.py:163-205): theta build,
 * gate, truncated SVD with the noise floor and per-gate budget
 * (tensor.py:87-123, one-sided Jacobi in FP64), renormalisation
 * (mps.py:189-192) and absorb.  chi_max > 0 additionally caps the kept rank
 * (an extension; the reference has no chi_max).
 * Outputs: sites/chi (layout above), discard (accumulated_discard),
 * peak_chi, status (MPSKQ_STATE_*).  entry_log (nullable, n_states x n_gates)
 * receives entry_count() after every gate (memory_log, mps.py:245-246).   */
int mpskq_simulate(int m, int chi_cap, const int32_t* ops_dev, int64_t n_ops, int64_t n_gates,
                   const double* coef_dev, int64_t n_params, int64_t n_states, double budget,
                   int chi_max, const int64_t* site_off_dev, int64_t state_stride,
                   double* sites_dev, int32_t* chi_dev, double* discard_dev,
                   int32_t* peak_chi_dev, int32_t* status_dev, int64_t* entry_log_dev,
                   void* stream);

/* General form of mpskq_simulate.  from_input != 0 continues the states
 * already held in sites/chi/discard/peak_chi (same layout) instead of
 * starting from |0..0>: apply_gate / canonicalize / run_circuit on a given
 * MpsState (mps.py:123-247) are op programs replayed this way (QRL/QRR moves
 * from the state's ortho_center, U1/U2 ops for arbitrary matrices whose
 * coefficients sit in coef_dev).  phase_cycles_dev (nullable, n_states x 3
 * int64) receives the device clock cycles each state spent in
 * {canonicalize, one_qubit, two_qubit} ops (MpsState.timings keys,
 * mps.py:137, :159, :204).  nominal_flops_dev (nullable, n_states doubles)
 * receives the nominal flop count of the replayed ops (the
 * simulation roofline numerator): per two-qubit gate theta 8*2chl*chm*2chr +
 * gate 128*chl*chr + thin SVD 8*(4MN^2 + 8N^3) of the 2chl x 2chr theta;
 * per QR move 16*M*N^2 + the R push 8*k*N*cols.                           */
int mpskq_run_program(int m, int chi_cap, const int32_t* ops_dev, int64_t n_ops, int64_t n_gates,
                      const double* coef_dev, int64_t n_params, int64_t n_states, double budget,
                      int chi_max, const int64_t* site_off_dev, int64_t state_stride,
                      int from_input, double* sites_dev, int32_t* chi_dev, double* discard_dev,
                      int32_t* peak_chi_dev, int32_t* status_dev, int64_t* entry_log_dev,
                      int64_t* phase_cycles_dev, double* nominal_flops_dev, void* stream);

/* Move n states between chi-capacity layouts (mpskq_batch_layout): state i
 * of src (bond dims chi_dev row i) becomes row dst_rows_dev[i] of dst
 * (identity when NULL).  Used by per-state capacity escalation: only the
 * states that overflowed a capacity are re-simulated at a larger one.     */
int mpskq_relayout(int m, int64_t n, const double* src_sites_dev, const int64_t* src_off_dev,
                   int64_t src_stride, const int32_t* chi_dev, double* dst_sites_dev,
                   const int64_t* dst_off_dev, int64_t dst_stride, const int32_t* dst_rows_dev,
                   void* stream);

/* Exact (unpadded) packing of n states for the multi-GPU exchange: state i's
 * site tensors back to back ((chi_l, 2, chi_r) row-major, the MPS1 payload
 * order, mps.py:294-314) from complex offset state_off_dev[i]; the caller
 * computes state_off as the prefix sum of sum_s 2 chi_s chi_{s+1}.  Unpack
 * is the inverse into a batch layout (optionally into rows dst_rows; the
 * per-state capacity escalation keeps finished levels packed this way).    */
int mpskq_pack_exact(int m, int64_t n, const double* sites_dev, const int64_t* site_off_dev, int64_t state_stride,
                     const int32_t* chi_dev, const int64_t* state_off_dev, double* packed_dev, void* stream);
int mpskq_unpack_exact(int m, int64_t n, const double* packed_dev, const int64_t* state_off_dev,
                       const int32_t* chi_dev, double* sites_dev, const int64_t* site_off_dev, int64_t state_stride,
                       const int32_t* dst_rows_dev /* nullable: state i -> layout row dst_rows[i] */, void* stream);

/* ---------------------------------------------------------------- truncated SVD
 * svd_truncated (tensor.py:87-123) on a batch of rows x cols complex
 * matrices (row-major, contiguous).  Outputs per matrix: U (rows x kmin),
 * s (kmin, noise floor applied, descending), Vh (kmin x cols), keep,
 * discarded; kmin = min(rows, cols).  Only the first `keep` columns/values
 * /rows are the reference's result.  rows, cols <= 2 * max chi capacity.   */
int mpskq_svd_truncated_batched(int rows, int cols, int64_t batch, const double* mats_dev,
                                double budget, int chi_max, double* u_dev, double* s_dev,
                                double* vh_dev, int32_t* keep_dev, double* discarded_dev,
                                int32_t* status_dev, void* stream);

/* ---------------------------------------------------------------- overlaps
 * inner_product (mps.py:260-268) for a tile set of (bra, ket) pairs, bras
 * conjugated, contracted site by site.  kind TRAIN (compute_gram,
 * kernel.py:169-175): bras and kets are the same batch, only i < j is
 * computed, out[i*ld+j] = out[j*ld+i] = value and out[i*ld+i] = 1.0.
 * kind TEST (kernel.py:176-181): every (i, j).  With world > 1 only the
 * block-cyclic tiles t with t % world == rank are written (and the train
 * diagonal by rank 0), so disjoint ranks can be summed exactly.            */
int mpskq_overlap(int kind, int out_mode, int m, int chi_cap, const int64_t* site_off_dev,
                  int64_t state_stride, const double* bra_sites_dev, const int32_t* bra_chi_dev,
                  int64_t n_bras, const double* ket_sites_dev, const int32_t* ket_chi_dev,
                  int64_t n_kets, int rank, int world, double* out_dev, int64_t ld,
                  void* stream);

/* Tile decomposition used by mpskq_overlap for (kind, chi_cap): tiles of
 * row_block x col_block (bra x ket) pairs, block-cyclic over ranks (tile t
 * belongs to rank t % world); train keeps only tiles holding some i < j.
 * tiles receives (row block index, col block index) int32 pairs; call with
 * tiles == NULL to query n_tiles.  Host-only (no GPU needed).             */
int mpskq_overlap_tiles(int kind, int chi_cap, int64_t n_bras, int64_t n_kets, int rank,
                        int world, int32_t* tiles, int64_t cap, int64_t* n_tiles,
                        int32_t* row_block, int32_t* col_block);

/* ---------------------------------------------------------------- end to end
 * The whole hot path behind run_distributed / simulate_dataset +
 * compute_gram (kernel.py:128-185, :443-512) on HOST buffers: copies the
 * feature rows in, builds topology/program/coefficients, simulates every
 * state once on the GPU, fills K and copies it back.  kind TRAIN uses
 * X_bras only (N = n_bras); kind TEST simulates bras (test rows) and kets
 * (train rows).  chi_cap = 0 picks the smallest compiled capacity that
 * holds the result (retrying on MPSKQ_STATE_CAPACITY).  seconds (nullable,
 * 4 doubles) receives {simulation, inner_products, communication, merge}
 * device times (RunReport.seconds keys, kernel.py:100-107).  A page-locked
 * K_out (cudaHostAlloc / torch pin_memory) on the chi <= 4 path receives K
 * band by band while the overlap still runs (the copy then sits inside
 * "inner_products" and "merge" is ~0); a pageable K_out gets one copy at the
 * end.  The values are bitwise the same either way.                       */
int mpskq_gram_host(int kind, int m, int r, int d, double gamma, double budget, int chi_max,
                    int chi_cap, const double* X_bras, int64_t n_bras, const double* X_kets,
                    int64_t n_kets, double* K_out, void* stream, double* seconds);

/* Multi-GPU row ownership (replaces the dense N x N sum-reduce): rank r
 * computes the K rows of the bra bands it owns (band b -> rank b % world;
 * bands of 8 ordered rows on the chi <= 4 path, single rows otherwise) and
 * writes them compactly, caller column order: rows_out[k * n_kets + j] is
 * caller row row_ids[k] (-1 = padding).  mpskq_owned_rows gives the row
 * count to allocate.  Train rows hold the entries this rank computed; the
 * gatherer's mpskq_assemble_rows scatters every rank's rows into K and
 * mirrors the rest with ket_pos (the ordered position of every state,
 * written by any rank's call; identity off the chi <= 4 path) plus the unit
 * diagonal — compute_gram's result (kernel.py:165-181).                   */
int mpskq_owned_rows(int chi_cap, int64_t n_bras, int rank, int world, int64_t* n_owned);
int mpskq_overlap_owned_rows(int kind, int m, int chi_cap, const int64_t* site_off_dev, int64_t state_stride,
                             const double* bra_sites_dev, const int32_t* bra_chi_dev, int64_t n_bras,
                             const double* ket_sites_dev, const int32_t* ket_chi_dev, int64_t n_kets, int rank,
                             int world, double* rows_out_dev, int32_t* row_ids_dev, int32_t* ket_pos_dev,
                             void* stream);
int mpskq_assemble_rows(int kind, int64_t n_bras, int64_t n_kets, const double* rows_dev,
                        const int32_t* row_ids_dev, int64_t n_rows, const int32_t* ket_pos_dev, double* K_dev,
                        int64_t ld, void* stream);

/* compute_gram (kernel.py:147-185) of device-resident states into HOST
 * memory K_out (n_bras x n_kets, row-major): a page-locked K_out on the
 * chi <= 4 path receives row bands while the overlap still runs (as in
 * mpskq_gram_host); otherwise device K plus one copy.  Train writes the
 * unit diagonal and the mirror.  Returns after K_out is complete.         */
int mpskq_overlap_host(int kind, int m, int chi_cap, const int64_t* site_off_dev, int64_t state_stride,
                       const double* bra_sites_dev, const int32_t* bra_chi_dev, int64_t n_bras,
                       const double* ket_sites_dev, const int32_t* ket_chi_dev, int64_t n_kets,
                       double* K_out, void* stream);

/* SM clock of the current device in kHz (cudaDevAttrClockRate; 0 without a
 * device): converts mpskq_run_program's phase cycles into seconds.        */
int mpskq_sm_clock_khz(void);

/* FP64 FMA throughput probe (roofline denominator): n_blocks x 256 threads,
 * each running `iters` x 16 independent DFMA.  Writes a checksum to out_dev. */
int mpskq_fp64_probe(int n_blocks, int64_t iters, double* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPSKQ_H */
