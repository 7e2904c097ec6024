// Host runtime of libmpskq: error state, feature-map topology, angle and
// coefficient encoding, program compiler, batch layout and the end-to-end
// host-buffer pipeline.  Device work lives in sim.cu / overlap.cu.
//
// Reference citations are /root/reference/pkg/src/mpskernel/<file>:<line>.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"

namespace mpskq {

static thread_local char g_err[1024] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_fail(int err, const char* what) {
  return fail(MPSKQ_ERR_CUDA, "%s: %s", what, cudaGetErrorString((cudaError_t)err));
}

void retain_pool_memory() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  static thread_local int done_for = -1;
  if (done_for == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_for = dev;
}

int64_t bond_cap(int m, int chi_cap, int b) {
  int e = std::min(b, m - b);
  if (e >= 30) return chi_cap;
  return std::min<int64_t>(chi_cap, int64_t(1) << e);
}

namespace {

struct Gate {
  int kind, a, b, slot;
};

// interaction_graph (ansatz.py:102-106): edges grouped by distance k, then i
std::vector<std::pair<int, int>> edges_of(int m, int d) {
  std::vector<std::pair<int, int>> e;
  for (int k = 1; k <= d; ++k)
    for (int i = 0; i + k < m; ++i) e.emplace_back(i, i + k);
  return e;
}

int check_cfg(int m, int r, int d) {
  // FeatureMapConfig.__post_init__ (ansatz.py:33-41)
  if (m < 1) return fail(MPSKQ_ERR_INVALID, "m must be at least 1");
  if (r < 1) return fail(MPSKQ_ERR_INVALID, "r must be at least 1");
  if (!(1 <= d && d <= m - 1))
    return fail(MPSKQ_ERR_INVALID, "d must satisfy 1 <= d <= m-1, got d=%d for m=%d", d, m);
  return MPSKQ_OK;
}

// greedy first-fit layering of one run of RXX gates (ansatz.py:139-161)
void schedule_run(const std::vector<Gate>& run, int m, int d, std::vector<Gate>& out) {
  std::vector<std::vector<Gate>> layers;
  std::vector<std::vector<char>> used;
  for (const Gate& g : run) {
    bool placed = false;
    for (size_t l = 0; l < layers.size(); ++l) {
      if (!used[l][g.a] && !used[l][g.b]) {
        layers[l].push_back(g);
        used[l][g.a] = used[l][g.b] = 1;
        placed = true;
        break;
      }
    }
    if (!placed) {
      layers.push_back({g});
      used.emplace_back(m, 0);
      used.back()[g.a] = used.back()[g.b] = 1;
    }
  }
  (void)d;  // the reference asserts len(layers) <= 2d; the banded graph guarantees it
  for (auto& l : layers)
    for (auto& g : l) out.push_back(g);
}

std::vector<Gate> feature_map_gates(int m, int r, int d, int64_t* n_params) {
  auto edges = edges_of(m, d);
  const int E = (int)edges.size();
  // build_circuit (ansatz.py:126-136)
  std::vector<Gate> built;
  for (int q = 0; q < m; ++q) built.push_back({MPSKQ_GATE_H, q, -1, -1});
  for (int l = 0; l < r; ++l) {
    for (int q = 0; q < m; ++q) built.push_back({MPSKQ_GATE_RZ, q, -1, l * (m + E) + q});
    for (int e = 0; e < E; ++e)
      built.push_back({MPSKQ_GATE_RXX, edges[e].first, edges[e].second, l * (m + E) + m + e});
  }
  *n_params = (int64_t)r * (m + E);
  // schedule_circuit (ansatz.py:170-184)
  std::vector<Gate> sched, run;
  for (const Gate& g : built) {
    if (g.kind == MPSKQ_GATE_RXX) {
      run.push_back(g);
    } else {
      if (!run.empty()) schedule_run(run, m, d, sched), run.clear();
      sched.push_back(g);
    }
  }
  if (!run.empty()) schedule_run(run, m, d, sched);
  // route_linear (ansatz.py:187-215)
  std::vector<int> pos(m), occ(m);
  for (int i = 0; i < m; ++i) pos[i] = occ[i] = i;
  std::vector<Gate> out;
  auto emit_swap = [&](int p) {
    out.push_back({MPSKQ_GATE_SWAP, p, p + 1, -1});
    int la = occ[p], lb = occ[p + 1];
    occ[p] = lb;
    occ[p + 1] = la;
    pos[la] = p + 1;
    pos[lb] = p;
  };
  for (const Gate& g : sched) {
    if (g.b < 0) {
      out.push_back({g.kind, pos[g.a], -1, g.slot});
      continue;
    }
    int lo = std::min(pos[g.a], pos[g.b]), hi = std::max(pos[g.a], pos[g.b]);
    for (int p = hi - 1; p > lo; --p) emit_swap(p);
    out.push_back({g.kind, lo, lo + 1, g.slot});
    for (int p = lo + 1; p < hi; ++p) emit_swap(p);
  }
  return out;
}

}  // namespace
}  // namespace mpskq

using namespace mpskq;

extern "C" {

int mpskq_abi_version(void) { return MPSKQ_ABI_VERSION; }
const char* mpskq_last_error(void) { return g_err; }

int mpskq_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int mpskq_feature_map_topology(int m, int r, int d, int32_t* kinds, int32_t* q0, int32_t* q1,
                               int32_t* param_slot, int64_t cap, int64_t* n_gates,
                               int64_t* n_params) {
  if (int st = check_cfg(m, r, d)) return st;
  int64_t np = 0;
  auto gates = feature_map_gates(m, r, d, &np);
  if (n_gates) *n_gates = (int64_t)gates.size();
  if (n_params) *n_params = np;
  if (!kinds) return MPSKQ_OK;
  if (cap < (int64_t)gates.size())
    return fail(MPSKQ_ERR_INVALID, "topology needs %zu gates, buffer holds %lld", gates.size(),
                (long long)cap);
  for (size_t i = 0; i < gates.size(); ++i) {
    kinds[i] = gates[i].kind;
    q0[i] = gates[i].a;
    q1[i] = gates[i].b;
    param_slot[i] = gates[i].slot;
  }
  return MPSKQ_OK;
}

int mpskq_feature_map_angles(const double* X, int64_t n_rows, int m, int r, int d, double gamma,
                             double* angles) {
  if (int st = check_cfg(m, r, d)) return st;
  if (!(gamma > 0)) return fail(MPSKQ_ERR_INVALID, "gamma must be positive");
  if (n_rows < 0) return fail(MPSKQ_ERR_INVALID, "negative row count");
  auto edges = edges_of(m, d);
  const int64_t E = (int64_t)edges.size(), np = (int64_t)r * (m + E);
  // the reference's expression order, ansatz.py:130 and :132; gamma**2 is
  // pow(gamma, 2) which is the correctly rounded gamma*gamma
  const double g2 = gamma * gamma;
  const double rz_scale = 2.0 * gamma;
  const double rxx_scale = (2.0 * g2) * (M_PI / 2.0);
  for (int64_t n = 0; n < n_rows; ++n) {
    const double* x = X + n * m;
    for (int q = 0; q < m; ++q) {
      if (!std::isfinite(x[q])) return fail(MPSKQ_ERR_INVALID, "features must be finite");
      if (x[q] < 0.0 || x[q] > 2.0)
        return fail(MPSKQ_ERR_INVALID, "features must lie in [0, 2]; rescale the data first");
    }
    double* out = angles + n * np;
    for (int l = 0; l < r; ++l) {
      double* o = out + (int64_t)l * (m + E);
      for (int q = 0; q < m; ++q) o[q] = rz_scale * x[q];
      for (int64_t e = 0; e < E; ++e) {
        const int i = edges[e].first, j = edges[e].second;
        double a = rxx_scale * (1.0 - x[i]);
        o[m + e] = a * (1.0 - x[j]);
      }
    }
  }
  return MPSKQ_OK;
}

int mpskq_feature_map_coefficients_device(const double* X_dev, int64_t n_rows, int m, int r,
                                          int d, double gamma, double* coef_dev, int* bad_dev,
                                          void* stream) {
  if (int st = check_cfg(m, r, d)) return st;
  if (!(gamma > 0)) return fail(MPSKQ_ERR_INVALID, "gamma must be positive");
  if (n_rows < 0) return fail(MPSKQ_ERR_INVALID, "negative row count");
  return launch_encode(X_dev, n_rows, m, r, d, gamma, coef_dev, bad_dev, stream);
}

int mpskq_half_angle_coefficients(const double* angles, int64_t n, double* coef) {
  for (int64_t i = 0; i < n; ++i) {
    const double half = 0.5 * angles[i];  // gate_matrix, ansatz.py:92
    coef[2 * i] = std::cos(half);
    coef[2 * i + 1] = std::sin(half);
  }
  return MPSKQ_OK;
}

int mpskq_program_compile(int m, int64_t n_gates, const int32_t* kinds, const int32_t* q0,
                          const int32_t* q1, const int32_t* param_slot, int32_t* ops,
                          int64_t cap_ops, int64_t* n_ops, int64_t* n_qr_left,
                          int64_t* n_qr_right) {
  if (m < 1) return fail(MPSKQ_ERR_INVALID, "qubit count must be at least 1");
  // next two-qubit gate's lower qubit after each index (run_circuit, mps.py:233-236)
  std::vector<int> next2(n_gates + 1, -1);
  for (int64_t i = n_gates - 1; i >= 0; --i) {
    const bool two = kinds[i] == MPSKQ_GATE_RXX || kinds[i] == MPSKQ_GATE_SWAP;
    next2[i] = two ? std::min(q0[i], q1[i]) : next2[i + 1];
  }
  int64_t count = 0, nl = 0, nr = 0;
  auto emit = [&](int code, int site, int slot, int gidx) {
    if (ops) {
      if (count >= cap_ops) return false;
      ops[4 * count + 0] = code;
      ops[4 * count + 1] = site;
      ops[4 * count + 2] = slot;
      ops[4 * count + 3] = gidx;
    }
    ++count;
    return true;
  };
  int center = 0;  // init_state: ortho_center = 0 (mps.py:102)
  for (int64_t i = 0; i < n_gates; ++i) {
    const int k = kinds[i];
    if (k < MPSKQ_GATE_H || k > MPSKQ_GATE_SWAP)
      return fail(MPSKQ_ERR_INVALID, "unknown gate kind %d", k);
    const bool two = k == MPSKQ_GATE_RXX || k == MPSKQ_GATE_SWAP;
    const bool param = k == MPSKQ_GATE_RZ || k == MPSKQ_GATE_RXX;
    if (param && param_slot[i] < 0)
      return fail(MPSKQ_ERR_INVALID, "gate %lld requires an angle", (long long)i);
    if (!two) {
      if (q0[i] < 0 || q0[i] >= m)
        return fail(MPSKQ_ERR_INVALID, "qubit %d out of range for %d sites", q0[i], m);
      if (!emit(k == MPSKQ_GATE_H ? MPSKQ_OP_H : MPSKQ_OP_RZ, q0[i], param ? param_slot[i] : -1,
                (int)i))
        return fail(MPSKQ_ERR_INVALID, "op buffer too small");
      continue;
    }
    const int a = q0[i], b = q1[i];
    if (a < 0 || a >= m || b < 0 || b >= m)
      return fail(MPSKQ_ERR_INVALID, "qubit out of range for %d sites", m);
    if (std::abs(a - b) != 1)
      return fail(MPSKQ_ERR_INVALID,
                  "two-qubit gate on (%d, %d) is not adjacent; route the circuit first", a, b);
    // H, RZ, RXX and SWAP are all symmetric under exchanging the two qubits,
    // so apply_gate's transpose for a > b (mps.py:219-220) is the identity.
    const int q = std::min(a, b);
    const int nxt = next2[i + 1];
    const bool left = nxt >= 0 && nxt <= q;
    // canonicalize(state, q) (mps.py:123-138)
    if (center < q) {
      for (int s = center; s < q; ++s, ++nl)
        if (!emit(MPSKQ_OP_QRL, s, -1, -1)) return fail(MPSKQ_ERR_INVALID, "op buffer too small");
    } else if (center > q) {
      for (int s = center; s > q; --s, ++nr)
        if (!emit(MPSKQ_OP_QRR, s, -1, -1)) return fail(MPSKQ_ERR_INVALID, "op buffer too small");
    }
    const int code = (k == MPSKQ_GATE_RXX ? MPSKQ_OP_RXX : MPSKQ_OP_SWAP) |
                     ((left ? MPSKQ_ABSORB_LEFT : 0) << 8);
    if (!emit(code, q, param ? param_slot[i] : -1, (int)i))
      return fail(MPSKQ_ERR_INVALID, "op buffer too small");
    center = left ? q : q + 1;
  }
  if (n_ops) *n_ops = count;
  if (n_qr_left) *n_qr_left = nl;
  if (n_qr_right) *n_qr_right = nr;
  return MPSKQ_OK;
}

int mpskq_batch_layout(int m, int chi_cap, int64_t* site_off, int64_t* state_stride) {
  if (m < 1) return fail(MPSKQ_ERR_INVALID, "qubit count must be at least 1");
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  int64_t off = 0;
  for (int s = 0; s < m; ++s) {
    if (site_off) site_off[s] = off;
    off += 2 * bond_cap(m, chi_cap, s) * bond_cap(m, chi_cap, s + 1);
  }
  off = (off + 1) & ~int64_t(1);  // keep every state 32-byte aligned
  if (site_off) site_off[m] = off;
  if (state_stride) *state_stride = off;
  return MPSKQ_OK;
}

int mpskq_supported_chi_caps(int32_t* caps, int cap, int* n) {
  if (n) *n = kNumChiCaps;
  for (int i = 0; i < kNumChiCaps && i < cap; ++i) caps[i] = kChiCaps[i];
  return MPSKQ_OK;
}

int mpskq_simulate(int m, int chi_cap, const int32_t* ops_dev, int64_t n_ops, int64_t n_gates,
                   const double* coef_dev, int64_t n_params, int64_t n_states, double budget,
                   int chi_max, const int64_t* site_off_dev, int64_t state_stride,
                   double* sites_dev, int32_t* chi_dev, double* discard_dev,
                   int32_t* peak_chi_dev, int32_t* status_dev, int64_t* entry_log_dev,
                   void* stream) {
  if (m < 1) return fail(MPSKQ_ERR_INVALID, "qubit count must be at least 1");
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (!(budget >= 0)) return fail(MPSKQ_ERR_INVALID, "budget must be non-negative");
  if (n_states < 0 || n_ops < 0) return fail(MPSKQ_ERR_INVALID, "negative sizes");
  if (n_states == 0) return MPSKQ_OK;
  SimArgs a{m,        chi_cap,  ops_dev,      n_ops,        n_gates,   coef_dev,
            n_params, n_states, budget,       chi_max,      site_off_dev, state_stride,
            sites_dev, chi_dev, discard_dev,  peak_chi_dev, status_dev, entry_log_dev, nullptr};
  return launch_simulate(a, stream);
}

int mpskq_run_program(int m, int chi_cap, const int32_t* ops_dev, int64_t n_ops, int64_t n_gates,
                      const double* coef_dev, int64_t n_params, int64_t n_states, double budget,
                      int chi_max, const int64_t* site_off_dev, int64_t state_stride,
                      int from_input, double* sites_dev, int32_t* chi_dev, double* discard_dev,
                      int32_t* peak_chi_dev, int32_t* status_dev, int64_t* entry_log_dev,
                      int64_t* phase_cycles_dev, double* nominal_flops_dev, void* stream) {
  if (m < 1) return fail(MPSKQ_ERR_INVALID, "qubit count must be at least 1");
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (!(budget >= 0)) return fail(MPSKQ_ERR_INVALID, "budget must be non-negative");
  if (n_states < 0 || n_ops < 0) return fail(MPSKQ_ERR_INVALID, "negative sizes");
  if (n_states == 0) return MPSKQ_OK;
  SimArgs a{m,        chi_cap,  ops_dev,      n_ops,        n_gates,   coef_dev,
            n_params, n_states, budget,       chi_max,      site_off_dev, state_stride,
            sites_dev, chi_dev, discard_dev,  peak_chi_dev, status_dev, entry_log_dev, nullptr};
  a.from_input = from_input != 0;
  a.phase_cycles = reinterpret_cast<long long*>(phase_cycles_dev);
  a.nominal_flops = nominal_flops_dev;
  return launch_simulate(a, stream);
}

int mpskq_relayout(int m, int64_t n, const double* src_sites_dev, const int64_t* src_off_dev,
                   int64_t src_stride, const int32_t* chi_dev, double* dst_sites_dev,
                   const int64_t* dst_off_dev, int64_t dst_stride, const int32_t* dst_rows_dev,
                   void* stream) {
  if (m < 1 || n < 0) return fail(MPSKQ_ERR_INVALID, "bad relayout sizes");
  return launch_relayout(m, n, src_sites_dev, src_off_dev, src_stride, chi_dev, dst_sites_dev, dst_off_dev,
                         dst_stride, dst_rows_dev, stream);
}

int mpskq_pack_exact(int m, int64_t n, const double* sites_dev, const int64_t* site_off_dev, int64_t state_stride,
                     const int32_t* chi_dev, const int64_t* state_off_dev, double* packed_dev, void* stream) {
  if (m < 1 || n < 0) return fail(MPSKQ_ERR_INVALID, "bad pack sizes");
  return launch_pack_exact(m, n, const_cast<double*>(sites_dev), site_off_dev, state_stride, chi_dev, state_off_dev,
                           packed_dev, 0, nullptr, stream);
}

int mpskq_unpack_exact(int m, int64_t n, const double* packed_dev, const int64_t* state_off_dev,
                       const int32_t* chi_dev, double* sites_dev, const int64_t* site_off_dev, int64_t state_stride,
                       const int32_t* dst_rows_dev, void* stream) {
  if (m < 1 || n < 0) return fail(MPSKQ_ERR_INVALID, "bad unpack sizes");
  return launch_pack_exact(m, n, sites_dev, site_off_dev, state_stride, chi_dev, state_off_dev,
                           const_cast<double*>(packed_dev), 1, dst_rows_dev, stream);
}

int mpskq_svd_truncated_batched(int rows, int cols, int64_t batch, const double* mats_dev,
                                double budget, int chi_max, double* u_dev, double* s_dev,
                                double* vh_dev, int32_t* keep_dev, double* discarded_dev,
                                int32_t* status_dev, void* stream) {
  if (rows < 1 || cols < 1)
    return fail(MPSKQ_ERR_INVALID, "split must leave a non-empty axis group on each side");
  if (!(budget >= 0)) return fail(MPSKQ_ERR_INVALID, "budget must be non-negative");
  const int maxdim = 2 * kChiCaps[kNumChiCaps - 1];
  if (rows > maxdim || cols > maxdim)
    return fail(MPSKQ_ERR_INVALID, "matrix %dx%d exceeds the %dx%d device SVD envelope", rows,
                cols, maxdim, maxdim);
  if (batch <= 0) return MPSKQ_OK;
  SvdArgs a{rows, cols, batch, mats_dev, budget, chi_max, u_dev, s_dev, vh_dev, keep_dev,
            discarded_dev, status_dev, nullptr};
  return launch_svd(a, stream);
}

int mpskq_overlap(int kind, int out_mode, int m, int chi_cap, const int64_t* site_off_dev,
                  int64_t state_stride, const double* bra_sites_dev, const int32_t* bra_chi_dev,
                  int64_t n_bras, const double* ket_sites_dev, const int32_t* ket_chi_dev,
                  int64_t n_kets, int rank, int world, double* out_dev, int64_t ld,
                  void* stream) {
  if (kind != MPSKQ_KIND_TRAIN && kind != MPSKQ_KIND_TEST)
    return fail(MPSKQ_ERR_INVALID, "kind must be one of ('train', 'test')");
  if (out_mode != MPSKQ_OUT_KERNEL && out_mode != MPSKQ_OUT_AMPLITUDE)
    return fail(MPSKQ_ERR_INVALID, "unknown output mode %d", out_mode);
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (kind == MPSKQ_KIND_TRAIN &&
      (n_bras != n_kets || bra_sites_dev != ket_sites_dev || bra_chi_dev != ket_chi_dev))
    return fail(MPSKQ_ERR_INVALID, "train kind requires bras and kets to be the same states");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(MPSKQ_ERR_INVALID, "bad rank %d of world %d", rank, world);
  if (ld < n_kets) return fail(MPSKQ_ERR_INVALID, "leading dimension smaller than ket count");
  if (n_bras == 0 || n_kets == 0) return MPSKQ_OK;
  OverlapArgs a{kind,     out_mode,      m,        chi_cap,       site_off_dev, state_stride,
                bra_sites_dev, bra_chi_dev, n_bras, ket_sites_dev, ket_chi_dev,  n_kets,
                rank,     world,         out_dev,  ld};
  return launch_overlap(a, stream);
}

int mpskq_sm_clock_khz(void) {
  int dev = 0, khz = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return khz;
}

int mpskq_fp64_probe(int n_blocks, int64_t iters, double* out_dev, void* stream) {
  if (n_blocks < 1 || iters < 1) return fail(MPSKQ_ERR_INVALID, "bad probe size");
  return launch_fp64_probe(n_blocks, iters, out_dev, stream);
}

}  // extern "C"

// ------------------------------------------------------------------ end to end
namespace {

// stream-ordered device allocation (pool-backed, cheap after warm-up)
struct AsyncBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  AsyncBuf() = default;
  AsyncBuf(const AsyncBuf&) = delete;
  AsyncBuf& operator=(const AsyncBuf&) = delete;
  ~AsyncBuf() { reset(); }
  void reset() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
  int alloc(size_t bytes, cudaStream_t s) {
    st = s;
    cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 8, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
    return MPSKQ_OK;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct ProgramCache {
  std::mutex mu;
  std::map<std::tuple<int, int, int>, std::pair<std::vector<int32_t>, int64_t>> progs;  // ops, n_gates
  std::map<std::tuple<int, int, int, double, int>, int> cap_hint;
};
ProgramCache& cache() {
  static ProgramCache c;
  return c;
}

int program_for(int m, int r, int d, std::vector<int32_t>& ops, int64_t& n_gates) {
  {
    std::lock_guard<std::mutex> g(cache().mu);
    auto it = cache().progs.find({m, r, d});
    if (it != cache().progs.end()) {
      ops = it->second.first;
      n_gates = it->second.second;
      return MPSKQ_OK;
    }
  }
  int64_t n_params = 0, n_ops = 0;
  int st = mpskq_feature_map_topology(m, r, d, nullptr, nullptr, nullptr, nullptr, 0, &n_gates, &n_params);
  if (st) return st;
  std::vector<int32_t> kinds(n_gates), q0(n_gates), q1(n_gates), slot(n_gates);
  st = mpskq_feature_map_topology(m, r, d, kinds.data(), q0.data(), q1.data(), slot.data(), n_gates,
                                  &n_gates, &n_params);
  if (st) return st;
  st = mpskq_program_compile(m, n_gates, kinds.data(), q0.data(), q1.data(), slot.data(), nullptr, 0,
                             &n_ops, nullptr, nullptr);
  if (st) return st;
  ops.assign(4 * n_ops, 0);
  st = mpskq_program_compile(m, n_gates, kinds.data(), q0.data(), q1.data(), slot.data(), ops.data(),
                             n_ops, &n_ops, nullptr, nullptr);
  if (st) return st;
  std::lock_guard<std::mutex> g(cache().mu);
  cache().progs[{m, r, d}] = {ops, n_gates};
  return MPSKQ_OK;
}

#define CK(expr)                                        \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)
#define ST(expr)                \
  do {                          \
    int s_ = (expr);            \
    if (s_ != MPSKQ_OK) return s_; \
  } while (0)


// K of the given device states into host memory K_out (n_bras x n_kets).
// Pinned (page-locked, device-mapped) K_out on the chi <= 4 path: the
// overlap streams finished row bands straight into it while later bands
// compute, so the 8 B/entry device->host transfer hides under the overlap.
// Pageable K_out: device K, then one copy.  ev_done (nullable) is recorded
// when the overlap kernels are queued.  Does not synchronise.
int overlap_into_host(int kind, int m, int cap, const int64_t* doff, int64_t stride, const double* bra_sites,
                      const int32_t* bra_chi, int64_t n_bras, const double* ket_sites, const int32_t* ket_chi,
                      int64_t n_kets, double* K_out, void* stream, cudaEvent_t ev_done) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* k_mapped = nullptr;
  if (cap == 4 && n_bras > 0 && n_kets > 0) {
    cudaPointerAttributes pa{};
    int cur = 0;
    cudaGetDevice(&cur);
    // only a buffer registered by this device's context is safely mapped here
    // (a buffer pinned by another device without cudaHostAllocPortable is not)
    if (cudaPointerGetAttributes(&pa, K_out) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer && pa.device == cur)
      k_mapped = static_cast<double*>(pa.devicePointer);
    cudaGetLastError();  // a pageable pointer may leave a sticky-free error behind
  }
  if (k_mapped) {
    OverlapArgs a{kind,      MPSKQ_OUT_KERNEL, m,      cap,       doff,    stride,
                  bra_sites, bra_chi,          n_bras, ket_sites, ket_chi, n_kets,
                  0,         1,                nullptr, n_kets};
    a.host_out = k_mapped;
    ST(launch_overlap(a, stream));
    if (ev_done) CK(cudaEventRecord(ev_done, st));
    return MPSKQ_OK;
  }
  AsyncBuf dK;
  ST(dK.alloc(sizeof(double) * n_bras * n_kets, st));
  ST(mpskq_overlap(kind, MPSKQ_OUT_KERNEL, m, cap, doff, stride, bra_sites, bra_chi, n_bras, ket_sites, ket_chi,
                   n_kets, 0, 1, dK.as<double>(), n_kets, stream));
  if (ev_done) CK(cudaEventRecord(ev_done, st));
  if (n_bras * n_kets)
    CK(cudaMemcpyAsync(K_out, dK.p, sizeof(double) * n_bras * n_kets, cudaMemcpyDeviceToHost, st));
  return MPSKQ_OK;
}

}  // namespace

extern "C" int mpskq_gram_host(int kind, int m, int r, int d, double gamma, double budget,
                               int chi_max, int chi_cap, const double* X_bras, int64_t n_bras,
                               const double* X_kets, int64_t n_kets, double* K_out, void* stream,
                               double* seconds) {
  if (kind != MPSKQ_KIND_TRAIN && kind != MPSKQ_KIND_TEST)
    return fail(MPSKQ_ERR_INVALID, "kind must be one of ('train', 'test')");
  ST(check_cfg(m, r, d));
  if (!(gamma > 0)) return fail(MPSKQ_ERR_INVALID, "gamma must be positive");
  if (!(budget >= 0)) return fail(MPSKQ_ERR_INVALID, "budget must be non-negative");
  if (chi_cap != 0 && !chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  const bool train = kind == MPSKQ_KIND_TRAIN;
  if (train) {
    X_kets = X_bras;
    n_kets = n_bras;
  }
  if (n_bras < 0 || n_kets < 0) return fail(MPSKQ_ERR_INVALID, "negative row count");
  // the rows are validated on the device by the encoder (bad flag, read with
  // the first simulation status): a host scan of N x m doubles cost ~1 ms
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_all = train ? n_bras : n_bras + n_kets;
  {
    // keep the stream-ordered pool's pages between calls (default threshold 0
    // returns them to the driver at every synchronize)
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }

  std::vector<int32_t> ops;
  int64_t n_gates = 0;
  ST(program_for(m, r, d, ops, n_gates));
  const int64_t n_ops = (int64_t)ops.size() / 4;
  int E = 0;
  for (int k = 1; k <= d; ++k) E += m - k;
  const int64_t n_params = (int64_t)r * (m + E);

  cudaEvent_t ev[4];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } evg{ev};

  CK(cudaEventRecord(ev[0], st));
  AsyncBuf dX, dcoef, dops, dbad;
  ST(dX.alloc(sizeof(double) * n_all * m, st));
  ST(dcoef.alloc(sizeof(double) * 2 * n_all * n_params, st));
  ST(dops.alloc(sizeof(int32_t) * ops.size(), st));
  ST(dbad.alloc(sizeof(int), st));
  if (n_bras) CK(cudaMemcpyAsync(dX.p, X_bras, sizeof(double) * n_bras * m, cudaMemcpyHostToDevice, st));
  if (!train && n_kets)
    CK(cudaMemcpyAsync(dX.as<double>() + n_bras * m, X_kets, sizeof(double) * n_kets * m,
                       cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dops.p, ops.data(), sizeof(int32_t) * ops.size(), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(dbad.p, 0, sizeof(int), st));
  ST(launch_encode(dX.as<double>(), n_all, m, r, d, gamma, dcoef.as<double>(), dbad.as<int>(), st));

  // Simulate every state at the hinted capacity; states that outgrow it (and
  // only those) are re-simulated at the next capacity, and so on (per-state
  // escalation).  The levels are then gathered into the final capacity's
  // layout, so the overlap sees one batch.
  const auto key = std::make_tuple(m, r, d, budget, chi_max);
  int cap_idx = 0;
  if (chi_cap) {
    while (kChiCaps[cap_idx] != chi_cap) ++cap_idx;
  } else {
    std::lock_guard<std::mutex> g(cache().mu);
    auto it = cache().cap_hint.find(key);
    if (it != cache().cap_hint.end()) cap_idx = it->second;
  }
  struct Level {
    int cap_idx = 0;
    int64_t n = 0, stride = 0;
    AsyncBuf sites, chi, disc, peak, status, doff, rows, coef, packed, soff;  // packed: finished, exact
  };
  std::vector<std::unique_ptr<Level>> levels;
  std::vector<int32_t> todo;  // global rows still to simulate (empty = all, level 0)
  for (;; ++cap_idx) {
    if (cap_idx >= kNumChiCaps)
      return fail(MPSKQ_ERR_CAPACITY, "bond dimension exceeds the largest compiled capacity %d",
                  kChiCaps[kNumChiCaps - 1]);
    auto L = std::make_unique<Level>();
    L->cap_idx = cap_idx;
    L->n = levels.empty() ? n_all : (int64_t)todo.size();
    const int cap_l = kChiCaps[cap_idx];
    std::vector<int64_t> off(m + 1);
    ST(mpskq_batch_layout(m, cap_l, off.data(), &L->stride));
    ST(L->doff.alloc(sizeof(int64_t) * (m + 1), st));
    CK(cudaMemcpyAsync(L->doff.p, off.data(), sizeof(int64_t) * (m + 1), cudaMemcpyHostToDevice, st));
    const double* coef_l = dcoef.as<double>();
    if (!levels.empty()) {
      ST(L->rows.alloc(sizeof(int32_t) * L->n, st));
      CK(cudaMemcpyAsync(L->rows.p, todo.data(), sizeof(int32_t) * L->n, cudaMemcpyHostToDevice, st));
      ST(L->coef.alloc(sizeof(double) * 2 * n_params * L->n, st));
      ST(launch_copy_rows(dcoef.p, L->coef.p, sizeof(double) * 2 * n_params, L->n, L->rows.as<int32_t>(),
                          nullptr, st));
      coef_l = L->coef.as<double>();
    }
    ST(L->sites.alloc(sizeof(double) * 2 * L->stride * L->n, st));
    ST(L->chi.alloc(sizeof(int32_t) * (m + 1) * L->n, st));
    ST(L->disc.alloc(sizeof(double) * L->n, st));
    ST(L->peak.alloc(sizeof(int32_t) * L->n, st));
    ST(L->status.alloc(sizeof(int32_t) * L->n, st));
    ST(mpskq_simulate(m, cap_l, dops.as<int32_t>(), n_ops, n_gates, coef_l, n_params, L->n, budget, chi_max,
                      L->doff.as<int64_t>(), L->stride, L->sites.as<double>(), L->chi.as<int32_t>(),
                      L->disc.as<double>(), L->peak.as<int32_t>(), L->status.as<int32_t>(), nullptr, stream));
    std::vector<int32_t> hstatus(L->n);
    int hbad = 0;
    CK(cudaMemcpyAsync(hstatus.data(), L->status.p, sizeof(int32_t) * L->n, cudaMemcpyDeviceToHost, st));
    if (levels.empty()) CK(cudaMemcpyAsync(&hbad, dbad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad & 2) return fail(MPSKQ_ERR_INVALID, "features must be finite");
    if (hbad & 1) return fail(MPSKQ_ERR_INVALID, "features must lie in [0, 2]; rescale the data first");
    std::vector<int32_t> next;
    for (int64_t i = 0; i < L->n; ++i) {
      if (hstatus[i] == MPSKQ_STATE_NONFINITE) return fail(MPSKQ_ERR_NUMERIC, "tensor has non-finite entries");
      if (hstatus[i] == MPSKQ_STATE_NOCONV) return fail(MPSKQ_ERR_NUMERIC, "SVD did not converge");
      if (hstatus[i] == MPSKQ_STATE_CAPACITY) next.push_back(levels.empty() ? (int32_t)i : todo[i]);
    }
    if (!next.empty() && !chi_cap) {
      // keep this level's states exactly packed (their own bond dims) until
      // the final capacity is known; the padded level buffer is released
      std::vector<int32_t> hchi((m + 1) * L->n);
      CK(cudaMemcpyAsync(hchi.data(), L->chi.p, sizeof(int32_t) * hchi.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<int64_t> hoff(L->n);
      int64_t tot = 0;
      for (int64_t i = 0; i < L->n; ++i) {
        hoff[i] = tot;
        for (int b = 0; b < m; ++b) tot += 2 * (int64_t)hchi[i * (m + 1) + b] * hchi[i * (m + 1) + b + 1];
      }
      ST(L->soff.alloc(sizeof(int64_t) * L->n, st));
      CK(cudaMemcpyAsync(L->soff.p, hoff.data(), sizeof(int64_t) * L->n, cudaMemcpyHostToDevice, st));
      ST(L->packed.alloc(sizeof(double) * 2 * std::max<int64_t>(tot, 1), st));
      ST(launch_pack_exact(m, L->n, L->sites.as<double>(), L->doff.as<int64_t>(), L->stride, L->chi.as<int32_t>(),
                           L->soff.as<int64_t>(), L->packed.as<double>(), 0, nullptr, st));
      CK(cudaStreamSynchronize(st));  // hoff / hchi leave scope
      L->sites.reset();
    }
    levels.push_back(std::move(L));
    if (next.empty()) break;
    if (chi_cap) return fail(MPSKQ_ERR_CAPACITY, "bond dimension exceeds chi capacity %d", kChiCaps[cap_idx]);
    todo.swap(next);
  }
  if (!chi_cap) {
    // the next call starts at the capacity the whole batch needed (a lower
    // start replays every state that later overflows: slower in steady state)
    std::lock_guard<std::mutex> g(cache().mu);
    cache().cap_hint[key] = levels.back()->cap_idx;
  }
  Level& fin = *levels.back();
  const int cap = kChiCaps[fin.cap_idx];
  const int64_t stride = fin.stride;
  AsyncBuf sites, chi, disc, peak, doff;
  if (levels.size() == 1) {
    std::swap(sites.p, fin.sites.p);
    std::swap(chi.p, fin.chi.p);
    std::swap(doff.p, fin.doff.p);
    sites.st = chi.st = doff.st = st;
  } else {
    ST(sites.alloc(sizeof(double) * 2 * stride * n_all, st));
    ST(chi.alloc(sizeof(int32_t) * (m + 1) * n_all, st));
    ST(disc.alloc(sizeof(double) * n_all, st));
    ST(peak.alloc(sizeof(int32_t) * n_all, st));
    std::swap(doff.p, fin.doff.p);
    doff.st = st;
    for (auto& Lp : levels) {  // later levels overwrite the rows that overflowed earlier ones
      Level& L = *Lp;
      const int32_t* rows = L.rows.p ? L.rows.as<int32_t>() : nullptr;
      if (L.packed.p)
        ST(launch_pack_exact(m, L.n, sites.as<double>(), doff.as<int64_t>(), stride, L.chi.as<int32_t>(),
                             L.soff.as<int64_t>(), L.packed.as<double>(), 1, rows, st));
      else
        ST(launch_relayout(m, L.n, L.sites.as<double>(), L.doff.p ? L.doff.as<int64_t>() : doff.as<int64_t>(),
                           L.stride, L.chi.as<int32_t>(), sites.as<double>(), doff.as<int64_t>(), stride, rows, st));
      ST(launch_copy_rows(L.chi.p, chi.p, sizeof(int32_t) * (m + 1), L.n, nullptr, rows, st));
      ST(launch_copy_rows(L.disc.p, disc.p, sizeof(double), L.n, nullptr, rows, st));
      ST(launch_copy_rows(L.peak.p, peak.p, sizeof(int32_t), L.n, nullptr, rows, st));
    }
  }
  CK(cudaEventRecord(ev[1], st));

  const double* bra_sites = sites.as<double>();
  const int32_t* bra_chi = chi.as<int32_t>();
  const double* ket_sites = train ? bra_sites : bra_sites + 2 * stride * n_bras;
  const int32_t* ket_chi = train ? bra_chi : bra_chi + (m + 1) * n_bras;
  ST(overlap_into_host(kind, m, cap, doff.as<int64_t>(), stride, bra_sites, bra_chi, n_bras, ket_sites, ket_chi,
                       n_kets, K_out, stream, ev[2]));
  CK(cudaEventRecord(ev[3], st));
  CK(cudaStreamSynchronize(st));
  if (seconds) {
    float t01 = 0, t12 = 0, t23 = 0;
    cudaEventElapsedTime(&t01, ev[0], ev[1]);
    cudaEventElapsedTime(&t12, ev[1], ev[2]);
    cudaEventElapsedTime(&t23, ev[2], ev[3]);
    seconds[0] = 1e-3 * t01;
    seconds[1] = 1e-3 * t12;
    seconds[2] = 0.0;
    seconds[3] = 1e-3 * t23;
  }
  return MPSKQ_OK;
}

extern "C" int mpskq_overlap_host(int kind, int m, int chi_cap, const int64_t* site_off_dev,
                                  int64_t state_stride, const double* bra_sites_dev, const int32_t* bra_chi_dev,
                                  int64_t n_bras, const double* ket_sites_dev, const int32_t* ket_chi_dev,
                                  int64_t n_kets, double* K_out, void* stream) {
  if (kind != MPSKQ_KIND_TRAIN && kind != MPSKQ_KIND_TEST)
    return fail(MPSKQ_ERR_INVALID, "kind must be one of ('train', 'test')");
  if (!chi_cap_supported(chi_cap))
    return fail(MPSKQ_ERR_INVALID, "chi capacity %d is not compiled in", chi_cap);
  if (kind == MPSKQ_KIND_TRAIN &&
      (n_bras != n_kets || bra_sites_dev != ket_sites_dev || bra_chi_dev != ket_chi_dev))
    return fail(MPSKQ_ERR_INVALID, "train kind requires bras and kets to be the same states");
  if (n_bras < 0 || n_kets < 0) return fail(MPSKQ_ERR_INVALID, "negative state counts");
  if (n_bras == 0 || n_kets == 0) return MPSKQ_OK;
  ST(overlap_into_host(kind, m, chi_cap, site_off_dev, state_stride, bra_sites_dev, bra_chi_dev, n_bras,
                       ket_sites_dev, ket_chi_dev, n_kets, K_out, stream, nullptr));
  CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return MPSKQ_OK;
}
