// qaoa_capi.cu -- extern "C" boundary (include/qaoa_b200.h) and the host-side
// sweep planner of the B200 QAOA engine.
//
// The planner turns p levels of (cost, mixer) into a list of fused sweeps:
//   * qubit sets: S_0 = tile bits at positions 0..11 (all active); the
//     remaining positions 12..n-1 in balanced chunks of <= 9, each carried in a
//     tile together with the lowest positions 0..(11-m) (inactive) so HBM
//     accesses stay >= 128-byte runs;
//   * exact mode (QAOA_RUN_EXACT): per level [cost + RX(S_0)] [RX(S_1)] ...,
//     qubits in increasing order, reference arithmetic: bit-identical to
//     simulate(..., "bitwise") (reference circuit.py:97-113);
//   * fast mode: odd levels visit the sets forward, even levels backward, so
//     the last set of level l and the first of level l+1 coincide and run as
//     ONE sweep [RX_l(S) -> cost_{l+1} -> RX_{l+1}(S)]: (R-1)p+1 sweeps for R
//     sets instead of R p.  Butterflies in factored one-DFMA form; the level
//     scale factors ride on the next phase table / the final scale.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <string>
#include <vector>

#include "../../include/qaoa_b200.h"
#include "qaoa_sweep.h"

using namespace qb;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(QAOA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);  \
  } while (0)

// One qubit set = one tile geometry: carry C (physical bits 0..C-1 ride along
// in every tile) and the mixed range q..q+11-C (or all of 0..11 when C = 12).
struct SetDesc {
  int carry;
  int q;
  bool mirror = false;  // symmetric half state: tile bit 11 is the virtual top qubit
};

struct SweepPlan {
  int set;
  int pre_cost;  // level index or -1
  int stage1;    // level index or -1
  int mid_cost;  // level index or -1
  int stage2;    // level index or -1
  int exchange;  // sharded runs: level whose global<->local exchange follows, or -1
};

// A planned run, executed in segments separated by the exchanges of a sharded
// state (qaoa_run_begin / qaoa_run_segment / qaoa_run_end); qaoa_run_layers is
// begin + every segment + end.
struct RunState {
  bool active = false;
  bool exact = false, want_expect = false, timing = false, from_state = false, sharded = false;
  // symmetric half state, fast schedule, one call: every low-set sweep also
  // applies the virtual top qubit's RX (kMirror, 2-CTA clusters)
  bool mirror_fused = false;
  int p = 0;
  std::vector<SetDesc> sets;
  std::vector<SweepPlan> plan;
  std::vector<RxStage> stages;
  std::vector<std::complex<double>> level_factor;  // per-qubit RX scale of each level (fast)
  std::complex<double> final_scale{1.0, 0.0};
  int flips = 0;
  std::vector<int> seg_start;  // segment k = plan[seg_start[k], seg_start[k + 1])
  size_t ev = 0;
  int grid = 0;
  bool expect_fused = false;
  bool weighted = false;  // factored weighted cost (qaoa_run_layers_weighted)
  bool no_store_last = false;  // QAOA_RUN_EXPECT_ONLY
  // swapped qubit layout (plan_swaps): lay[i] = layout sweep i reads (0: identity
  // in amps, 1: bit ranges of sets 1 and last exchanged, in amps2); do_swap[i]:
  // the (low-set) sweep writes out of place into the other layout
  bool swap = false;
  std::vector<uint8_t> lay, do_swap;
  GraphDev g_sw;
  int sw_lo = 0, sw_hi = 0, sw_m = 0;
};

}  // namespace

struct qaoa_ctx {
  int n = 0;  // local qubits (bits of the state index)
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double2* amps = nullptr;
  bool own_amps = false;
  GraphDev g{};
  bool has_graph = false;
  void* cut_table = nullptr;
  int cut_bytes = 0;
  double* partials = nullptr;
  int partials_len = 0;
  double* d_scalar = nullptr;
  double2* d_tables = nullptr;
  size_t d_tables_cap = 0;  // in double2
  double2* h_tables = nullptr;  // pinned staging
  size_t h_tables_cap = 0;
  // fast runs apply form-2 RX levels as form 1 plus an X on every mixed qubit,
  // done by bookkeeping: the true amplitude of index x is stored at x ^ cmask
  // (g.cmask; X commutes with every RX, and the cost kernels evaluate C at the
  // true index).  Bits >= n are the shard bits (managed by the sharded host).
  // expectation cached from the last fused run
  bool expect_valid = false;
  bool expect_is_weighted = false;  // the cached value is the weighted cut's
  double expect_value = 0.0;
  // weighted edge list (compressed backend), device copies
  int* d_ei = nullptr;
  int* d_ej = nullptr;
  double* d_w = nullptr;
  int n_wedges = -1;
  // factored weighted cost (fast schedule): host edge list, device endpoints,
  // incidence lists, per-run u_e and tile-internal phase tables
  std::vector<int> h_ei, h_ej;
  std::vector<double> h_w;
  int2* d_wedge = nullptr;
  int* d_winc_off = nullptr;
  int* d_winc = nullptr;
  double2* d_wu = nullptr;
  size_t d_wu_cap = 0;
  double2* d_wq = nullptr;
  size_t d_wq_cap = 0;
  double* d_wc = nullptr;  // tile-internal cut weights of the last sweep's set (fused weighted <C>)
  // launch control on the TMA-fed kernel: per-tile cut bases and gen x phase table
  void* d_basis = nullptr;
  size_t d_basis_cap = 0;
  double2* d_gen_tab = nullptr;
  int d_gen_tab_cap = 0;
  // timing
  std::vector<cudaEvent_t> events;
  std::vector<float> times;
  int last_launches = 0;
  double last_bytes = 0.0;
  RunState run;
  bool state_stale = false;  // last run skipped its final store (QAOA_RUN_EXPECT_ONLY)
  // second state buffer of the swapped qubit layout (allocated on first use)
  double2* amps2 = nullptr;
  int swap_mode = -1;  // qaoa_set_layout_swap: -1 policy, 0 off, 1 whenever applicable
  // qaoa_set_mirror: the buffer is the x_n = 0 half of an (n+1)-qubit symmetric
  // state; block norms and sampling then cover the 2^(n+1) virtual indices
  bool mirror_view = false;
};

namespace {

uint64_t local_mask(const qaoa_ctx* c) { return c->n >= 64 ? ~0ull : ((1ull << c->n) - 1ull); }

int check_ctx(qaoa_ctx* c) {
  if (!c) return fail(QAOA_E_INVALID, "null context");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  return QAOA_OK;
}

// A state left unstored by a QAOA_RUN_EXPECT_ONLY run must not be read.
int require_stored(qaoa_ctx* c) {
  if (c->state_stale)
    return fail(QAOA_E_STATE, "the state was not stored by the last run (QAOA_RUN_EXPECT_ONLY)");
  return QAOA_OK;
}

int ensure_partials(qaoa_ctx* c, int n) {
  if (c->partials_len >= n) return QAOA_OK;
  if (c->partials) cudaFree(c->partials);
  c->partials = nullptr;
  c->partials_len = 0;
  CUDA_TRY(cudaMalloc(&c->partials, sizeof(double) * (size_t)n));
  c->partials_len = n;
  return QAOA_OK;
}

int ensure_tables(qaoa_ctx* c, size_t n) {
  if (c->d_tables_cap < n) {
    if (c->d_tables) cudaFree(c->d_tables);
    c->d_tables = nullptr;
    c->d_tables_cap = 0;
    CUDA_TRY(cudaMalloc(&c->d_tables, sizeof(double2) * n));
    c->d_tables_cap = n;
  }
  if (c->h_tables_cap < n) {
    if (c->h_tables) cudaFreeHost(c->h_tables);
    c->h_tables = nullptr;
    c->h_tables_cap = 0;
    CUDA_TRY(cudaMallocHost(&c->h_tables, sizeof(double2) * n));
    c->h_tables_cap = n;
  }
  return QAOA_OK;
}

// mirror: a symmetric half state's one-call schedule (sweep_kernel's MIR).
// Fast: set 0 is the mirror low set (local qubits 0..10 plus the virtual top
// qubit n, SetDesc{12, n}) and the high sets cover local qubits 11..n-1.
// Exact: the high sets cover qubits 12..n including the virtual one, so the
// top set carries it last (the reference applies qubit N-1 last).
std::vector<SetDesc> make_sets(int n, bool mirror = false, bool exact = false) {
  std::vector<SetDesc> sets;
  const bool low_mirror = mirror && !exact;
  sets.push_back(SetDesc{12, low_mirror ? n : 0, low_mirror});
  const int first = low_mirror ? 11 : 12;
  const int rem = n + (mirror && exact ? 1 : 0) - first;
  if (rem <= 0) return sets;
  const int chunks = (rem + 8) / 9;  // at most 9 mixed bits per high sweep (C >= 3)
  // the r = rem % chunks extra bits go to the middle chunks first, the ends
  // taking two or none, so the first and last chunks (the level-boundary merges,
  // see plan_swaps) have equal sizes whenever possible
  const int r = rem % chunks;
  std::vector<int> size(chunks, rem / chunks);
  int mid = std::min(r, std::max(chunks - 2, 0));
  if ((r - mid) % 2) --mid;
  if (mid < 0 || r - mid > 2) {
    for (int ci = 0; ci < r; ++ci) ++size[ci];  // two chunks, odd remainder
  } else {
    for (int ci = 0; ci < mid; ++ci) ++size[1 + ci];
    if (r - mid == 2) {
      ++size[0];
      ++size[chunks - 1];
    }
  }
  int next = first;
  for (int ci = 0; ci < chunks; ++ci) {
    sets.push_back(SetDesc{12 - size[ci], next, mirror && exact && ci == chunks - 1});
    next += size[ci];
  }
  return sets;
}

std::vector<SweepPlan> make_plan(int n_sets, int p, bool exact, bool sharded = false,
                                 bool mirror = false) {
  // flat op list: cost l, then mixer l over the sets in this level's order;
  // sharded: an exchange (kind 2) right after the low set S_0 of every level
  // (the swapped local bits sit in S_0, so they have had RX_l when they leave
  // and the arriving ones get RX_l inside the exchange kernel)
  struct Op {
    int kind;  // 0 cost, 1 mixer, 2 exchange
    int level;
    int set;
  };
  std::vector<Op> ops;
  // fast mode: the low set (index 0, the only one whose merged form needs four
  // exchanges) sits in the middle of the level order when there are >= 3 sets,
  // so the merged level-boundary sweeps are always high sets.
  std::vector<int> order;
  if (!exact && n_sets >= 3) {
    order.push_back(1);
    order.push_back(0);
    for (int i = 2; i < n_sets; ++i) order.push_back(i);
  } else {
    for (int i = 0; i < n_sets; ++i) order.push_back(i);
  }
  for (int l = 0; l < p; ++l) {
    ops.push_back({0, l, -1});
    const bool fwd = exact || (l % 2 == 0);
    for (int i = 0; i < n_sets; ++i) {
      const int set = fwd ? order[i] : order[n_sets - 1 - i];
      ops.push_back({1, l, set});
      // the exchange point: after S_0 (its top bits are the ones a shard
      // exchange swaps); for the virtual qubit of a symmetric exact run after
      // the level's last set (the reference applies qubit n last)
      const int xset = (mirror && exact) ? order[n_sets - 1] : 0;
      if (sharded && set == xset) ops.push_back({2, l, -1});
    }
  }
  std::vector<SweepPlan> plan;
  size_t i = 0;
  while (i < ops.size()) {
    SweepPlan sp{-1, -1, -1, -1, -1, -1};
    if (ops[i].kind == 0) {
      sp.pre_cost = ops[i].level;
      ++i;
    }
    // ops[i] is a mixer op
    sp.set = ops[i].set;
    sp.stage1 = ops[i].level;
    ++i;
    if (!exact && i + 1 < ops.size() && ops[i].kind == 0 && ops[i + 1].kind == 1 &&
        ops[i + 1].set == sp.set) {
      sp.mid_cost = ops[i].level;
      sp.stage2 = ops[i + 1].level;
      i += 2;
    }
    if (i < ops.size() && ops[i].kind == 2) {
      sp.exchange = ops[i].level;
      ++i;
    }
    plan.push_back(sp);
  }
  return plan;
}

void fill_graph(GraphDev& g, int n_nodes, const uint64_t* row_mask, int tot_edge, uint64_t x_hi) {
  memset(&g, 0, sizeof(g));
  g.n_nodes = n_nodes;
  g.tot_edge = tot_edge;
  g.x_hi = x_hi;
  for (int i = 0; i < n_nodes; ++i) g.rm[i] = row_mask[i];
  for (int i = 0; i < n_nodes; ++i) {
    uint64_t m = row_mask[i];
    while (m) {
      const int j = __builtin_ctzll(m);
      m &= m - 1;
      g.adj[i] |= 1ull << j;
      g.adj[j] |= 1ull << i;
    }
  }
}

uint64_t swap_ranges_host(uint64_t x, int lo, int hi, int m) {
  const uint64_t mask = (1ull << m) - 1ull;
  const uint64_t a = (x >> lo) & mask, b = (x >> hi) & mask;
  return (x & ~((mask << lo) | (mask << hi))) | (a << hi) | (b << lo);
}

// The graph with node (= physical bit) i relabelled to bit swap(i).
GraphDev swap_graph(const GraphDev& g, int lo, int hi, int m) {
  uint64_t rm[kMaxNodes] = {0};
  for (int i = 0; i < g.n_nodes; ++i) {
    uint64_t mk = g.rm[i];
    while (mk) {
      const int j = __builtin_ctzll(mk);
      mk &= mk - 1;
      int a = (int)__builtin_ctzll(swap_ranges_host(1ull << i, lo, hi, m));
      int b = (int)__builtin_ctzll(swap_ranges_host(1ull << j, lo, hi, m));
      if (a > b) std::swap(a, b);
      rm[a] |= 1ull << b;
    }
  }
  GraphDev out;
  fill_graph(out, g.n_nodes, rm, g.tot_edge, g.x_hi);
  out.cmask = swap_ranges_host(g.cmask, lo, hi, m);
  return out;
}

// Swapped qubit layout (fast unweighted single-GPU runs).  The level-boundary
// merges alternate between set 1 (physical bits 12..) and the last set (the
// top bits, whose tiles touch one DRAM page per run: the slowest sweep kind).
// Every low-set sweep S_0 -- contiguous 64 KiB tiles, its qubits 0..11 untouched
// by the relabelling -- writes its tiles out of place with the bit ranges of set
// 1 and the last set exchanged, so the set merged next always sits at bits
// 12..: all merges run the set-1 geometry.  An even number of swaps per run
// returns the state to identity order in its own buffer.  A symmetric run's
// mirror low set (blocks u and ~u of 2048, qubits 11.. in the high sets) swaps
// the same way: the complement commutes with the bit-range swap.
void plan_swaps(qaoa_ctx* c, RunState& R) {
  R.swap = false;
  R.lay.assign(R.plan.size(), 0);
  R.do_swap.assign(R.plan.size(), 0);
  const int ns = (int)R.sets.size();
  if (R.exact || R.weighted || R.sharded || ns < 3 || c->swap_mode == 0) return;
  if (c->swap_mode < 0) {
    static int env = -2;
    if (env == -2) {
      const char* e = getenv("QAOA_SWAP_LAYOUT");
      env = e ? atoi(e) : -1;
    }
    if (env == 0) return;
    // policy: states of >= 1 GiB whose top set has 128-B runs (C = 3: one DRAM
    // page per run; N=30: +1.0-1.3% per step).  Sets with C >= 5 (N=31..33)
    // measured no gain (profiles/r06_swap.md).
    if (env < 0 && (c->n < 26 || R.sets[ns - 1].carry > 3)) return;
  }
  const int m1 = 12 - R.sets[1].carry, ml = 12 - R.sets[ns - 1].carry;
  if (m1 != ml) return;
  int n0 = 0;
  for (const SweepPlan& sp : R.plan) n0 += sp.set == 0;
  const int nswap = n0 & ~1;
  if (nswap == 0) return;
  if (!c->amps2) {
    // only with room to spare (4 GiB beyond the buffer), else run in place
    size_t free_b = 0, total_b = 0;
    const size_t need = sizeof(double2) << c->n;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || free_b < need + (4ull << 30)) {
      cudaGetLastError();
      return;
    }
    if (cudaMalloc(&c->amps2, need) != cudaSuccess) {
      cudaGetLastError();  // no room for the second buffer: run in place
      c->amps2 = nullptr;
      return;
    }
  }
  R.swap = true;
  R.sw_lo = R.sets[1].q;
  R.sw_hi = R.sets[ns - 1].q;
  R.sw_m = m1;
  R.g_sw = swap_graph(c->g, R.sw_lo, R.sw_hi, R.sw_m);
  int lay = 0, done = 0;
  for (size_t i = 0; i < R.plan.size(); ++i) {
    R.lay[i] = (uint8_t)lay;
    if (R.plan[i].set == 0 && done < nswap) {
      R.do_swap[i] = 1;
      ++done;
      lay ^= 1;
    }
  }
}

int record_event(qaoa_ctx* c, bool timing, size_t idx) {
  if (!timing) return QAOA_OK;
  while (c->events.size() <= idx) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    c->events.push_back(e);
  }
  CUDA_TRY(cudaEventRecord(c->events[idx], c->stream));
  return QAOA_OK;
}

int reduce_to_host(qaoa_ctx* c, int n_partials, int mode_max, double* out) {
  CUDA_TRY(launch_sum_partials(c->partials, n_partials, c->d_scalar, mode_max, c->stream));
  CUDA_TRY(cudaMemcpyAsync(out, c->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QAOA_OK;
}

int create_common(int n, int device, void* stream, void* ext, qaoa_ctx** out) {
  if (!out) return fail(QAOA_E_INVALID, "null output pointer");
  *out = nullptr;
  if (n < 1) return fail(QAOA_E_INVALID, "qubit count must be at least 1");
  if (n > 40) return fail(QAOA_E_INVALID, "local qubit count above 40 is not supported");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return fail(QAOA_E_CUDA, "no CUDA device available");
  if (device < 0 || device >= count) return fail(QAOA_E_INVALID, "device index out of range");
  CUDA_TRY(cudaSetDevice(device));
  qaoa_ctx* c = new qaoa_ctx();
  c->n = n;
  c->device = device;
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return cuda_fail(e, "cudaStreamCreate");
    }
    c->own_stream = true;
  }
  const size_t bytes = sizeof(double2) << n;
  if (ext) {
    c->amps = (double2*)ext;
  } else {
    e = cudaMalloc(&c->amps, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      qaoa_destroy(c);
      char buf[160];
      snprintf(buf, sizeof buf, "cannot allocate %.1f GiB of device memory for %d qubits",
               bytes / 1073741824.0, n);
      return fail(QAOA_E_NOMEM, buf);
    }
    c->own_amps = true;
  }
  e = cudaMalloc(&c->d_scalar, sizeof(double) * 2);
  if (e != cudaSuccess) {
    qaoa_destroy(c);
    return cuda_fail(e, "cudaMalloc");
  }
  int rc = ensure_partials(c, reduce_grid());
  if (rc) {
    qaoa_destroy(c);
    return rc;
  }
  *out = c;
  return QAOA_OK;
}


// ---- planned runs: begin / segment / end ----------------------------------
// Tiled states (n_local >= 12).  sharded: exchange points after S_0 of every
// level (make_plan), level flips complement all n_nodes bits (the host's
// cmask covers the shard bits too), <C> is fused only when the run does not end
// on an exchange.
int run_begin(qaoa_ctx* c, int p, const double* phase_tables, const double* cs, const double* sn,
              int flags, bool sharded, const double* gammas = nullptr, bool internal = false) {
  RunState& R = c->run;
  R = RunState();
  R.weighted = gammas != nullptr;
  R.exact = flags & QAOA_RUN_EXACT;
  R.from_state = flags & QAOA_RUN_FROM_STATE;
  R.want_expect = flags & QAOA_RUN_EXPECTATION;
  R.timing = flags & QAOA_RUN_TIMING;
  R.sharded = sharded;
  R.p = p;
  const int n = c->n;
  const int n_total = c->g.n_nodes;
  const double u = sqrt(ldexp(1.0, -n_total));  // 1/2^n exactly for n <= 64
  const uint64_t size = 1ull << n;
  c->expect_valid = false;
  c->last_launches = 0;
  c->last_bytes = 0.0;
  c->times.clear();
  int rc;
  if (R.from_state && c->state_stale)
    return fail(QAOA_E_STATE, "the state was not stored by the last run (QAOA_RUN_EXPECT_ONLY)");
  if (!R.from_state) c->g.cmask = 0;

  R.mirror_fused = (flags & QAOA_RUN_MIRROR) && !sharded;
  if (R.mirror_fused && n_total != n + 1)
    return fail(QAOA_E_INVALID,
                "QAOA_RUN_MIRROR without QAOA_RUN_SHARDED is the one-call symmetric schedule: it "
                "needs a graph of n_local + 1 nodes");
  R.sets = make_sets(n, R.mirror_fused, R.exact);
  R.plan = make_plan((int)R.sets.size(), p, R.exact, sharded, (flags & QAOA_RUN_MIRROR) != 0);
  // per-qubit RX factors of a level: the local qubits, plus the virtual top one
  // when its RX is fused into the low-set sweeps
  const int n_rx = n + (R.mirror_fused ? 1 : 0);

  // phase tables: the sweeps only index even entries (t = E - 2C), so upload
  // table_even[k] = table[2k], k = 0..E.  exact = as given; fast = scaled by
  // the previous level's factor.
  const int tl = 2 * c->g.tot_edge + 1;
  const int te = c->g.tot_edge + 1;
  R.stages.assign(std::max(p, 1), RxStage{0.0, 0.0, 0});
  R.level_factor.assign(std::max(p, 1), std::complex<double>(1.0, 0.0));
  std::complex<double> prev_scale(1.0, 0.0);
  if ((rc = ensure_tables(c, (size_t)te * std::max(p, 1)))) return rc;
  std::vector<std::complex<double>> level_scale(std::max(p, 1));
  for (int l = 0; l < p; ++l) {
    const std::complex<double> f_scale = prev_scale;
    level_scale[l] = f_scale;
    if (!R.weighted) {
      const double* src = phase_tables + (size_t)2 * tl * l;
      for (int k = 0; k < te; ++k) {
        std::complex<double> v(src[4 * k], src[4 * k + 1]);
        if (!R.exact) v *= f_scale;
        c->h_tables[(size_t)l * te + k] = make_double2(v.real(), v.imag());
      }
    }
    if (R.exact) {
      R.stages[l] = RxStage{cs[l], sn[l], 0};
    } else if (std::fabs(cs[l]) >= std::fabs(sn[l])) {
      // RX = c [[1, -i t], [-i t, 1]], t = s / c
      R.stages[l] = RxStage{sn[l] / cs[l], 0.0, 1};
      R.level_factor[l] = std::complex<double>(cs[l], 0.0);
      prev_scale = std::pow(R.level_factor[l], n_rx);
    } else {
      // RX = (-i s) X [[1, i k], [i k, 1]], k = c / s: run form 1 with t = -k and
      // complement every bit (X^n) by bookkeeping instead of data movement.
      R.stages[l] = RxStage{-cs[l] / sn[l], 0.0, 1};
      R.level_factor[l] = std::complex<double>(0.0, -sn[l]);
      prev_scale = std::pow(R.level_factor[l], n_rx);
      R.flips ^= 1;
    }
  }
  if (p > 0 && !R.weighted)
    CUDA_TRY(cudaMemcpyAsync(c->d_tables, c->h_tables, sizeof(double2) * (size_t)te * p,
                             cudaMemcpyHostToDevice, c->stream));
  R.final_scale = R.exact ? std::complex<double>(1.0, 0.0) : prev_scale;
  if (R.weighted && p > 0) {
    // u_e = exp(-i gamma_l w_e / 2) per level (cost.py:147-159), and the
    // tile-internal phase table of the set where each level's cost is applied
    const int m = c->n_wedges;
    const size_t nu = (size_t)p * std::max(m, 1);
    if (c->d_wu_cap < nu) {
      if (c->d_wu) cudaFree(c->d_wu);
      c->d_wu = nullptr;
      c->d_wu_cap = 0;
      CUDA_TRY(cudaMalloc(&c->d_wu, nu * sizeof(double2)));
      c->d_wu_cap = nu;
    }
    const size_t nq = (size_t)p * 4096;
    if (c->d_wq_cap < nq) {
      if (c->d_wq) cudaFree(c->d_wq);
      c->d_wq = nullptr;
      c->d_wq_cap = 0;
      CUDA_TRY(cudaMalloc(&c->d_wq, nq * sizeof(double2)));
      c->d_wq_cap = nq;
    }
    std::vector<double2> hu(nu);
    for (int l = 0; l < p; ++l)
      for (int e = 0; e < m; ++e) {
        const std::complex<double> u = std::exp(std::complex<double>(0.0, -0.5 * gammas[l] * c->h_w[e]));
        hu[(size_t)l * m + e] = make_double2(u.real(), u.imag());
      }
    CUDA_TRY(cudaMemcpyAsync(c->d_wu, hu.data(), nu * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
    for (int l = 0; l < p; ++l) {
      int set = -1;
      for (const SweepPlan& sp : R.plan)
        if (sp.pre_cost == l || sp.mid_cost == l) set = sp.set;
      const SetDesc& sd = R.sets[set < 0 ? 0 : set];
      const std::complex<double> f = R.exact ? std::complex<double>(1.0, 0.0) : level_scale[l];
      // the mirror low set's tile geometry is (11, n): node n is the virtual qubit
      CUDA_TRY(launch_wq_table(c->d_wq + (size_t)l * 4096, c->d_wedge, c->d_wu + (size_t)l * m, m,
                               sd.mirror && sd.carry == 12 ? 11 : sd.carry, sd.q,
                               make_double2(f.real(), f.imag()), c->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));  // hu is a host temporary
  }

  const int64_t ntiles = 1ll << (n - 12);
  R.grid = (int)ntiles;  // partials: one per tile
  if (R.want_expect && (rc = ensure_partials(c, R.grid))) return rc;

  if (p == 0) {
    if (!R.from_state) {
      CUDA_TRY(launch_fill(c->amps, size, make_double2(u, 0.0), c->stream));
      ++c->last_launches;
      c->last_bytes += 16.0 * size;
    }
    if (R.want_expect) {
      const int g2 = reduce_grid();
      CUDA_TRY(launch_expectation(c->amps, n, c->g, c->partials, g2, c->stream));
      ++c->last_launches;
      if ((rc = reduce_to_host(c, g2, 0, &c->expect_value))) return rc;
      c->expect_valid = true;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return QAOA_OK;
  }
  R.seg_start.push_back(0);
  for (size_t i = 0; i < R.plan.size(); ++i)
    if (R.plan[i].exchange >= 0) R.seg_start.push_back((int)i + 1);
  if (R.seg_start.back() != (int)R.plan.size()) R.seg_start.push_back((int)R.plan.size());
  R.expect_fused = R.want_expect && R.plan.back().exchange < 0;
  if (R.expect_fused && R.weighted) {
    if (!c->d_wc) CUDA_TRY(cudaMalloc(&c->d_wc, 4096 * sizeof(double)));
    const SetDesc& sd = R.sets[R.plan.back().set];
    CUDA_TRY(launch_wc_table(c->d_wc, c->d_wedge, c->d_w, c->n_wedges,
                             sd.mirror && sd.carry == 12 ? 11 : sd.carry, sd.q, c->stream));
  }
  R.no_store_last = (flags & QAOA_RUN_EXPECT_ONLY) && R.expect_fused;
  // the swapped layout only for runs the library drives end to end
  // (qaoa_run_layers*): hosts of qaoa_run_begin see every sweep in place, so
  // qaoa_run_sweep_info geometry, partial ranges and graph / mask changes
  // between segments stay valid
  if (internal) plan_swaps(c, R);
  else R.swap = false;
  R.active = true;
  if ((rc = record_event(c, R.timing, R.ev++))) return rc;
  return QAOA_OK;
}

// QAOA_GEN_AUX=0 disables launch_gen_aux (A/B; default on).
bool gen_aux_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QAOA_GEN_AUX");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

// Launch plan sweep i on tiles [lo, lo + cnt) (cnt = 0: all tiles).
int launch_plan_sweep(qaoa_ctx* c, int i, int64_t lo, int64_t cnt) {
  RunState& R = c->run;
  const uint64_t size = 1ull << c->n;
  const int te = c->g.tot_edge + 1;
  const double u = sqrt(ldexp(1.0, -c->g.n_nodes));
  const SweepPlan& sp = R.plan[i];
  // swapped layout: sets 1 and last trade physical positions
  const int ns = (int)R.sets.size();
  const bool sw = R.swap && R.lay[i];
  const int pset = !sw ? sp.set : sp.set == 1 ? ns - 1 : sp.set == ns - 1 ? 1 : sp.set;
  const SetDesc& st = R.sets[pset];
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.amps = sw ? c->amps2 : c->amps;
  a.g = sw ? R.g_sw : c->g;
  if (R.swap && R.do_swap[i]) {
    a.out = sw ? c->amps : c->amps2;
    a.sw_lo = R.sw_lo;
    a.sw_hi = R.sw_hi;
    a.sw_m = R.sw_m;
  }
  a.ntiles = 1ll << (c->n - 12);
  a.tile_lo = lo;
  a.tile_cnt = cnt;
  a.partials = c->partials;
  a.carry = st.carry;
  a.q = st.q;
  uint32_t fl = R.exact ? kExact : 0u;
  if (i == 0 && !R.from_state) {
    fl |= kGen;
    a.gen = make_double2(u, 0.0);
  }
  a.table_len = te;
  if (sp.pre_cost >= 0) {
    fl |= kPreCost;
    a.table = c->d_tables + (size_t)sp.pre_cost * te;
  }
  if (sp.mid_cost >= 0) {
    fl |= kMidCost;
    a.table2 = c->d_tables + (size_t)sp.mid_cost * te;
  }
  if (sp.stage1 >= 0) {
    fl |= kStage1;
    a.rx1 = R.stages[sp.stage1];
  }
  if (R.mirror_fused && st.mirror) fl |= kMirror;  // a tile with the virtual top qubit
  if (sp.stage2 >= 0) {
    fl |= kStage2;
    a.rx2 = R.stages[sp.stage2];
  }
  if (R.weighted) {
    const int m = c->n_wedges;
    fl |= kWeighted;
    a.wedge = c->d_wedge;
    a.winc_off = c->d_winc_off;
    a.winc = c->d_winc;
    a.wm = m;
    a.ww = c->d_w;
    a.wc = c->d_wc;
    if (sp.pre_cost >= 0) {
      a.wu1 = c->d_wu + (size_t)sp.pre_cost * m;
      a.wq1 = c->d_wq + (size_t)sp.pre_cost * 4096;
    }
    if (sp.mid_cost >= 0) {
      a.wu2 = c->d_wu + (size_t)sp.mid_cost * m;
      a.wq2 = c->d_wq + (size_t)sp.mid_cost * 4096;
    }
  }
  const bool last = i + 1 == (int)R.plan.size();
  if (last && !R.exact) {
    fl |= kScale;
    a.scale = make_double2(R.final_scale.real(), R.final_scale.imag());
  }
  if (last && R.expect_fused) fl |= kExpect;
  if (last && R.no_store_last) fl |= kNoStore;
  a.flags = fl;
  if ((fl & kGen) && (fl & kPreCost) && (sweep_uses_tma(a) || sweep32_selected(a)) && gen_aux_enabled()) {
    // launch control on the TMA-fed kernel: tile bases built ahead (off the
    // per-tile critical path) and the uniform amplitude folded into the table
    // (64 B per tile: 16 MiB at n = 30; if the buffers cannot be allocated the
    // sweep builds each tile's basis itself, as before)
    const size_t need = (size_t)kBasisEntryBytes * (size_t)a.ntiles;
    if (c->d_basis_cap < need) {
      if (c->d_basis) cudaFree(c->d_basis);
      c->d_basis = nullptr;
      c->d_basis_cap = 0;
      if (cudaMalloc(&c->d_basis, need) == cudaSuccess) c->d_basis_cap = need;
      else { c->d_basis = nullptr; cudaGetLastError(); }
    }
    if (c->d_gen_tab_cap < te) {
      if (c->d_gen_tab) cudaFree(c->d_gen_tab);
      c->d_gen_tab = nullptr;
      c->d_gen_tab_cap = 0;
      if (cudaMalloc(&c->d_gen_tab, sizeof(double2) * (size_t)te) == cudaSuccess) c->d_gen_tab_cap = te;
      else { c->d_gen_tab = nullptr; cudaGetLastError(); }
    }
    if (c->d_basis && c->d_gen_tab) {
      CUDA_TRY(launch_gen_aux(a, c->d_basis, c->d_gen_tab, c->stream));
      c->last_launches += 2;  // basis_table_kernel + gen_table_kernel
      a.basis_tab = c->d_basis;
      a.table = c->d_gen_tab;
      a.flags = fl | kGenTab;
    }
  }
  CUDA_TRY(launch_sweep(a, R.grid, c->stream));
  ++c->last_launches;
  const double frac = cnt ? (double)cnt / (double)a.ntiles : 1.0;
  c->last_bytes += ((fl & kGen) ? 16.0 : 32.0) * (double)size * frac;
  return QAOA_OK;
}

int run_segment(qaoa_ctx* c, int k) {
  RunState& R = c->run;
  if (!R.active) return fail(QAOA_E_STATE, "no planned run (qaoa_run_begin)");
  if (k < 0 || k + 1 >= (int)R.seg_start.size()) return fail(QAOA_E_RANGE, "segment out of range");
  int rc;
  for (int i = R.seg_start[k]; i < R.seg_start[k + 1]; ++i) {
    if ((rc = launch_plan_sweep(c, i, 0, 0))) return rc;
    if ((rc = record_event(c, R.timing, R.ev++))) return rc;
  }
  return QAOA_OK;
}

int run_end(qaoa_ctx* c) {
  RunState& R = c->run;
  if (!R.active) return fail(QAOA_E_STATE, "no planned run (qaoa_run_begin)");
  R.active = false;
  c->state_stale = R.no_store_last;
  int rc;
  if (R.flips) {
    // sharded: complement all n_nodes bits (C(x) = C(~x) keeps the cost kernels
    // exact with the run's initial mask); unsharded: all local bits = all bits
    // (a fused symmetric run: all n_local + 1 bits, X^N is the identity there)
    const uint64_t all = (R.sharded || R.mirror_fused)
                             ? (c->g.n_nodes >= 64 ? ~0ull : ((1ull << c->g.n_nodes) - 1ull))
                             : local_mask(c);
    c->g.cmask ^= all;
  }
  // symmetric half state: a mask with the virtual top bit set describes the
  // same data as its full complement (psi(v) == psi(~v)); keep the bit clear so
  // reads see the stored half (without touching the fused <C>, which C(v) ==
  // C(~v) leaves unchanged)
  if (R.mirror_fused && ((c->g.cmask >> c->n) & 1ull))
    c->g.cmask ^= (c->g.n_nodes >= 64 ? ~0ull : ((1ull << c->g.n_nodes) - 1ull));
  if (R.expect_fused) {
    if ((rc = reduce_to_host(c, R.grid, 0, &c->expect_value))) return rc;
    ++c->last_launches;
    c->expect_valid = true;
    c->expect_is_weighted = R.weighted;
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (R.timing) {
    for (size_t i = 0; i + 1 < R.ev; ++i) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, c->events[i], c->events[i + 1]));
      c->times.push_back(ms);
    }
  }
  return QAOA_OK;
}

}  // namespace

extern "C" {

const char* qaoa_last_error(void) { return g_last_error.c_str(); }

const char* qaoa_version(void) { return "qaoa_b200 0.2 sm_100a"; }

int qaoa_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int qaoa_create(int n_qubits, int device, void* stream, qaoa_ctx** out) {
  return create_common(n_qubits, device, stream, nullptr, out);
}

int qaoa_create_external(int n_qubits, int device, void* stream, void* device_amps,
                         qaoa_ctx** out) {
  if (!device_amps) return fail(QAOA_E_INVALID, "null device buffer");
  return create_common(n_qubits, device, stream, device_amps, out);
}

void qaoa_destroy(qaoa_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->own_amps && c->amps) cudaFree(c->amps);
  if (c->cut_table) cudaFree(c->cut_table);
  if (c->partials) cudaFree(c->partials);
  if (c->d_scalar) cudaFree(c->d_scalar);
  if (c->d_tables) cudaFree(c->d_tables);
  if (c->h_tables) cudaFreeHost(c->h_tables);
  if (c->d_ei) cudaFree(c->d_ei);
  if (c->d_ej) cudaFree(c->d_ej);
  if (c->d_w) cudaFree(c->d_w);
  if (c->d_wedge) cudaFree(c->d_wedge);
  if (c->d_winc_off) cudaFree(c->d_winc_off);
  if (c->d_winc) cudaFree(c->d_winc);
  if (c->d_wu) cudaFree(c->d_wu);
  if (c->d_wq) cudaFree(c->d_wq);
  if (c->d_wc) cudaFree(c->d_wc);
  if (c->amps2) cudaFree(c->amps2);
  if (c->d_basis) cudaFree(c->d_basis);
  if (c->d_gen_tab) cudaFree(c->d_gen_tab);
  for (auto e : c->events) cudaEventDestroy(e);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void* qaoa_state_ptr(qaoa_ctx* c) { return c ? (void*)c->amps : nullptr; }

int qaoa_set_stream(qaoa_ctx* c, void* stream) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->own_stream && c->stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
  }
  c->own_stream = false;
  c->stream = (cudaStream_t)stream;
  return QAOA_OK;
}

int qaoa_set_graph(qaoa_ctx* c, int n_nodes, const uint64_t* row_mask, int tot_edge,
                   uint64_t x_hi) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (n_nodes < c->n || n_nodes > kMaxNodes)
    return fail(QAOA_E_INVALID, "graph node count must be in [n_local, 64]");
  if (!row_mask && n_nodes) return fail(QAOA_E_INVALID, "null row_mask");
  if (x_hi & ((1ull << c->n) - 1ull)) return fail(QAOA_E_INVALID, "x_hi overlaps local bits");
  int edges = 0;
  for (int i = 0; i < n_nodes; ++i) {
    const uint64_t m = row_mask[i];
    if (n_nodes < 64 && (m >> n_nodes)) return fail(QAOA_E_INVALID, "row mask has bits above n");
    if (m & ((2ull << i) - 1ull)) return fail(QAOA_E_INVALID, "row mask is not strictly upper");
    edges += __builtin_popcountll(m);
  }
  if (edges != tot_edge) return fail(QAOA_E_INVALID, "tot_edge does not match the row masks");
  const uint64_t cmask = c->g.cmask;
  fill_graph(c->g, n_nodes, row_mask, tot_edge, x_hi);
  c->g.cmask = cmask;
  c->has_graph = true;
  c->expect_valid = false;
  if (c->cut_table) {
    cudaFree(c->cut_table);
    c->cut_table = nullptr;
  }
  return QAOA_OK;
}

int qaoa_init_uniform(qaoa_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  c->state_stale = false;
  const int n_total = c->has_graph ? c->g.n_nodes : c->n;
  const double u = sqrt(ldexp(1.0, -n_total));  // 1/2^n exactly for n <= 64
  CUDA_TRY(launch_fill(c->amps, 1ull << c->n, make_double2(u, 0.0), c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  c->g.cmask = 0;
  return QAOA_OK;
}

// Host-side index mapping for a stored state with local complement mask m:
// true index x lives at x ^ m.  m = 0 or all-ones (single GPU) are a plain copy
// or a reversal; other masks (sharded intermediate states) gather on the host.
static void permute_chunk(double2* dst, const double2* src, uint64_t true_off, uint64_t count,
                          uint64_t m, uint64_t stored_off) {
  for (uint64_t i = 0; i < count; ++i) dst[i] = src[((true_off + i) ^ m) - stored_off];
}

int qaoa_write_amplitudes(qaoa_ctx* c, uint64_t offset, uint64_t count, const double* src) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->state_stale && !(offset == 0 && count == (1ull << c->n)))
    return fail(QAOA_E_STATE, "the state was not stored by the last run (QAOA_RUN_EXPECT_ONLY)");
  c->state_stale = false;
  const uint64_t size = 1ull << c->n;
  if (offset + count > size || offset + count < offset)
    return fail(QAOA_E_RANGE, "amplitude range out of bounds");
  if (count && !src) return fail(QAOA_E_INVALID, "null source");
  const uint64_t m = c->g.cmask & local_mask(c);
  if (m == 0) {
    CUDA_TRY(cudaMemcpyAsync(c->amps + offset, src, count * sizeof(double2),
                             cudaMemcpyHostToDevice, c->stream));
  } else if (m == local_mask(c)) {  // true index x lives at ~x: reverse the chunk
    std::vector<double2> tmp(count);
    const double2* s2 = (const double2*)src;
    for (uint64_t i = 0; i < count; ++i) tmp[count - 1 - i] = s2[i];
    CUDA_TRY(cudaMemcpyAsync(c->amps + (size - offset - count), tmp.data(), count * sizeof(double2),
                             cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  } else {  // general mask: read-modify-write the whole state
    std::vector<double2> all(size);
    CUDA_TRY(cudaMemcpyAsync(all.data(), c->amps, size * sizeof(double2), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const double2* s2 = (const double2*)src;
    for (uint64_t i = 0; i < count; ++i) all[(offset + i) ^ m] = s2[i];
    CUDA_TRY(cudaMemcpyAsync(c->amps, all.data(), size * sizeof(double2), cudaMemcpyHostToDevice,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_read_amplitudes(qaoa_ctx* c, uint64_t offset, uint64_t count, double* dst) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->state_stale)
    return fail(QAOA_E_STATE, "the state was not stored by the last run (QAOA_RUN_EXPECT_ONLY)");
  const uint64_t size = 1ull << c->n;
  if (offset + count > size || offset + count < offset)
    return fail(QAOA_E_RANGE, "amplitude range out of bounds");
  if (count && !dst) return fail(QAOA_E_INVALID, "null destination");
  const uint64_t m = c->g.cmask & local_mask(c);
  if (m == 0 || m == local_mask(c)) {
    const uint64_t src_off = m ? size - offset - count : offset;
    CUDA_TRY(cudaMemcpyAsync(dst, c->amps + src_off, count * sizeof(double2),
                             cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (m) std::reverse((double2*)dst, (double2*)dst + count);
  } else {
    std::vector<double2> all(size);
    CUDA_TRY(cudaMemcpyAsync(all.data(), c->amps, size * sizeof(double2), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    permute_chunk((double2*)dst, all.data(), offset, count, m, 0);
  }
  return QAOA_OK;
}

int qaoa_trim(qaoa_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->run.active) return fail(QAOA_E_STATE, "a planned run is active");
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->amps2) {
    cudaFree(c->amps2);
    c->amps2 = nullptr;
  }
  if (c->cut_table) {
    cudaFree(c->cut_table);
    c->cut_table = nullptr;
  }
  if (c->d_basis) {
    cudaFree(c->d_basis);
    c->d_basis = nullptr;
    c->d_basis_cap = 0;
  }
  return QAOA_OK;
}

int qaoa_set_mirror(qaoa_ctx* c, int on) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (on && c->n >= 63) return fail(QAOA_E_INVALID, "a mirrored half state needs n_local < 63");
  c->mirror_view = on != 0;
  return QAOA_OK;
}

int qaoa_set_layout_swap(qaoa_ctx* c, int mode) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (mode < -1 || mode > 1) return fail(QAOA_E_INVALID, "layout swap mode must be -1, 0 or 1");
  c->swap_mode = mode;
  return QAOA_OK;
}

int qaoa_get_cmask(qaoa_ctx* c, uint64_t* out) {
  if (!c || !out) return fail(QAOA_E_INVALID, "null argument");
  *out = c->g.cmask;
  return QAOA_OK;
}

int qaoa_set_cmask(qaoa_ctx* c, uint64_t cmask) {
  if (!c) return fail(QAOA_E_INVALID, "null context");
  c->g.cmask = cmask;
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_apply_cost(qaoa_ctx* c, const double* phase_table) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (!c->has_graph) return fail(QAOA_E_STATE, "no graph set");
  if (!phase_table) return fail(QAOA_E_INVALID, "null phase table");
  const size_t len = 2 * (size_t)c->g.tot_edge + 1;
  if ((rc = ensure_tables(c, len))) return rc;
  memcpy(c->h_tables, phase_table, len * sizeof(double2));
  CUDA_TRY(cudaMemcpyAsync(c->d_tables, c->h_tables, len * sizeof(double2),
                           cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(launch_cost_gate(c->amps, 1ull << c->n, c->g, c->d_tables, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_apply_rx(qaoa_ctx* c, int qubit, double cs, double sn) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (qubit < 0 || qubit >= c->n) {
    char buf[96];
    snprintf(buf, sizeof buf, "qubit %d out of range for n=%d", qubit, c->n);
    return fail(QAOA_E_RANGE, buf);
  }
  CUDA_TRY(launch_rx_gate(c->amps, c->n, qubit, cs, sn, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

// ---- gate-level baseline (state.py:66-149) ----------------------------------
int qaoa_init_basis(qaoa_ctx* c, uint64_t index) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->n < 64 && index >= (1ull << c->n)) return fail(QAOA_E_RANGE, "basis index out of range");
  c->state_stale = false;
  CUDA_TRY(launch_basis(c->amps, 1ull << c->n, index, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  c->g.cmask = 0;
  return QAOA_OK;
}

int qaoa_apply_h(qaoa_ctx* c, int qubit) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (qubit < 0 || qubit >= c->n) {
    char buf[96];
    snprintf(buf, sizeof buf, "qubit %d out of range for n=%d", qubit, c->n);
    return fail(QAOA_E_RANGE, buf);
  }
  CUDA_TRY(launch_h_gate(c->amps, c->n, qubit, (int)((c->g.cmask >> qubit) & 1ull), c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_apply_rzz(qaoa_ctx* c, int q1, int q2, const double* phases) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (!phases) return fail(QAOA_E_INVALID, "null phases");
  if (q1 == q2) return fail(QAOA_E_INVALID, "RZZ needs two distinct qubits");
  for (int q : {q1, q2})
    if (q < 0 || q >= c->n) {
      char buf[96];
      snprintf(buf, sizeof buf, "qubit %d out of range for n=%d", q, c->n);
      return fail(QAOA_E_RANGE, buf);
    }
  const uint64_t xbase = c->g.cmask & ((c->n >= 64) ? ~0ull : ((1ull << c->n) - 1ull));
  CUDA_TRY(launch_rzz_gate(c->amps, 1ull << c->n, xbase, q1, q2, make_double2(phases[0], phases[1]),
                           make_double2(phases[2], phases[3]), c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_mirror_rx(qaoa_ctx* c, const double* rx, const double* factor) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (!rx || !factor) return fail(QAOA_E_INVALID, "null argument");
  if (c->n < 2) return fail(QAOA_E_INVALID, "the mirror pass needs at least 2 local qubits");
  const RxStage st{rx[0], rx[1], (int)rx[2]};
  const double2 f = make_double2(factor[0], factor[1]);
  CUDA_TRY(launch_mirror_rx(c->amps, c->n, st, f, !(f.x == 1.0 && f.y == 0.0), c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_edge_values(qaoa_ctx* c, int kind, uint64_t offset, uint64_t count, double* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (kind != 0 && kind != 1) return fail(QAOA_E_INVALID, "kind must be 0 (rotation totals) or 1 (cut values)");
  if (c->n_wedges < 0) return fail(QAOA_E_STATE, "no weighted edge list set");
  if (offset > (1ull << c->n) || count > (1ull << c->n) - offset)
    return fail(QAOA_E_RANGE, "index range out of bounds");
  if (count && !out) return fail(QAOA_E_INVALID, "null destination");
  const uint64_t chunk = std::min<uint64_t>(count, 1ull << 24);
  double* d = nullptr;
  if (chunk) CUDA_TRY(cudaMalloc(&d, chunk * sizeof(double)));
  cudaError_t e = cudaSuccess;
  for (uint64_t done = 0; done < count && e == cudaSuccess; done += chunk) {
    const uint64_t k = std::min(chunk, count - done);
    e = launch_edge_values(d, c->g.x_hi | (offset + done), k, c->d_ei, c->d_ej, c->d_w, c->n_wedges,
                           kind, c->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out + done, d, k * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  }
  if (d) cudaFree(d);
  CUDA_TRY(e);
  return QAOA_OK;
}

static int run_exact_mixer_sweeps(qaoa_ctx* c, double cs, double sn) {
  // all sets, RX stage only, exact arithmetic and order
  const std::vector<SetDesc> sets = make_sets(c->n);
  const int grid = (int)(1ll << (c->n - 12));  // one tile per CTA
  for (const SetDesc& s : sets) {
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    a.amps = c->amps;
    a.g = c->g;
    a.ntiles = 1ll << (c->n - 12);
    a.carry = s.carry;
    a.q = s.q;
    a.rx1 = RxStage{cs, sn, 0};
    a.flags = kStage1 | kExact;
    a.table_len = 0;
    CUDA_TRY(launch_sweep(a, grid, c->stream));
  }
  return QAOA_OK;
}

int qaoa_apply_mixer(qaoa_ctx* c, double cs, double sn) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (c->n >= 12) {
    if ((rc = run_exact_mixer_sweeps(c, cs, sn))) return rc;
  } else {
    for (int q = 0; q < c->n; ++q) CUDA_TRY(launch_rx_gate(c->amps, c->n, q, cs, sn, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_apply_rx_range(qaoa_ctx* c, int q0, int count, double cs, double sn, int flags) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (count < 1 || q0 < 0 || q0 + count > c->n)
    return fail(QAOA_E_RANGE, "qubit range out of bounds");
  const bool exact = flags & QAOA_RUN_EXACT;
  const int carry = 12 - count;
  const bool tiled = c->n >= 12 && count <= 9 && q0 >= carry;
  if (!tiled) {  // per-qubit kernels, reference arithmetic
    for (int q = q0; q < q0 + count; ++q) CUDA_TRY(launch_rx_gate(c->amps, c->n, q, cs, sn, c->stream));
  } else {
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    a.amps = c->amps;
    a.g = c->g;
    a.ntiles = 1ll << (c->n - 12);
    a.carry = carry;
    a.q = q0;
    uint32_t fl = kStage1;
    if (exact) {
      fl |= kExact;
      a.rx1 = RxStage{cs, sn, 0};
    } else {
      std::complex<double> f;
      if (std::fabs(cs) >= std::fabs(sn)) {
        a.rx1 = RxStage{sn / cs, 0.0, 1};
        f = std::pow(std::complex<double>(cs, 0.0), count);
      } else {
        a.rx1 = RxStage{-cs / sn, 0.0, 1};
        f = std::pow(std::complex<double>(0.0, -sn), count);
        c->g.cmask ^= (((1ull << count) - 1ull) << q0);
      }
      fl |= kScale;
      a.scale = make_double2(f.real(), f.imag());
    }
    a.flags = fl;
    CUDA_TRY(launch_sweep(a, (int)a.ntiles, c->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_run_layers(qaoa_ctx* c, int p, const double* phase_tables, const double* cs,
                    const double* sn, int flags) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!c->has_graph) return fail(QAOA_E_STATE, "no graph set");
  if (p < 0) return fail(QAOA_E_INVALID, "level count must be non-negative");
  if (p > 0 && (!phase_tables || !cs || !sn)) return fail(QAOA_E_INVALID, "null angle arrays");
  const bool from_state = flags & QAOA_RUN_FROM_STATE;
  const bool want_expect = flags & QAOA_RUN_EXPECTATION;
  const bool timing = flags & QAOA_RUN_TIMING;
  const int n = c->n;
  const int n_total = c->g.n_nodes;
  const int tl = 2 * c->g.tot_edge + 1;
  c->expect_valid = false;
  c->last_launches = 0;
  c->last_bytes = 0.0;
  c->times.clear();
  size_t ev = 0;
  const double u = sqrt(ldexp(1.0, -n_total));  // 1/2^n exactly for n <= 64
  const uint64_t size = 1ull << n;

  if (n < 12) {
    // Small states: per-gate kernels (bit-exact in both modes).
    if (from_state && c->state_stale)
      return fail(QAOA_E_STATE, "the state was not stored by the last run (QAOA_RUN_EXPECT_ONLY)");
    c->state_stale = false;
    // one CTA runs the whole circuit with the state in shared memory
    // (small_run_kernel): phase tables then the per-level (c, s) pairs
    const size_t nt = (size_t)tl * p;
    if ((rc = ensure_tables(c, nt + std::max(p, 1)))) return rc;
    memcpy(c->h_tables, phase_tables, sizeof(double2) * nt);
    for (int l = 0; l < p; ++l) c->h_tables[nt + l] = make_double2(cs[l], sn[l]);
    CUDA_TRY(cudaMemcpyAsync(c->d_tables, c->h_tables, sizeof(double2) * (nt + p),
                             cudaMemcpyHostToDevice, c->stream));
    if (!from_state) c->g.cmask = 0;
    if ((rc = record_event(c, timing, ev++))) return rc;
    CUDA_TRY(launch_small_run(c->amps, n, c->g, c->d_tables, c->d_tables + nt, p, from_state ? 1 : 0, u,
                              want_expect ? 1 : 0, c->d_scalar, c->stream));
    ++c->last_launches;
    c->last_bytes += 16.0 * size * (from_state ? 2 : 1);
    if ((rc = record_event(c, timing, ev++))) return rc;
    if (want_expect) {
      CUDA_TRY(cudaMemcpyAsync(&c->expect_value, c->d_scalar, sizeof(double), cudaMemcpyDeviceToHost,
                               c->stream));
      c->expect_valid = true;
      c->expect_is_weighted = false;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (timing) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, c->events[0], c->events[1]));
      c->times.push_back(ms);
    }
    return QAOA_OK;
  }

  // ---- tiled path --------------------------------------------------------
  if ((rc = run_begin(c, p, phase_tables, cs, sn, flags, false, nullptr, true))) return rc;
  if (p == 0) return QAOA_OK;  // handled (fill / expectation) inside run_begin
  for (size_t k = 0; k + 1 < c->run.seg_start.size(); ++k)
    if ((rc = run_segment(c, (int)k))) return rc;
  return run_end(c);
}

int qaoa_plan(int n_local, int p, int flags, int* out, int cap) {
  if (n_local < 12 || n_local > 40 || p < 1) return fail(QAOA_E_INVALID, "plan needs n_local in [12, 40], p >= 1");
  const std::vector<SetDesc> sets = make_sets(n_local);
  const std::vector<SweepPlan> plan =
      make_plan((int)sets.size(), p, (flags & QAOA_RUN_EXACT) != 0, (flags & QAOA_RUN_SHARDED) != 0);
  if (out) {
    for (size_t i = 0; i < plan.size() && (int)i < cap; ++i) {
      const SweepPlan& sp = plan[i];
      const SetDesc& sd = sets[sp.set];
      int* o = out + 7 * i;
      o[0] = sd.carry;
      o[1] = sd.q;
      o[2] = sp.pre_cost;
      o[3] = sp.stage1;
      o[4] = sp.mid_cost;
      o[5] = sp.stage2;
      o[6] = sp.exchange;
    }
  }
  return (int)plan.size();
}

int qaoa_run_layers_weighted(qaoa_ctx* c, int p, const double* gammas, const double* cs,
                             const double* sn, int flags) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!c->has_graph) return fail(QAOA_E_STATE, "no graph set");
  if (c->n_wedges < 0) return fail(QAOA_E_STATE, "no weights set (qaoa_set_weights)");
  if (p < 1) return fail(QAOA_E_INVALID, "planned runs need at least one level");
  if (!gammas || !cs || !sn) return fail(QAOA_E_INVALID, "null angle arrays");
  if (c->n < 12) return fail(QAOA_E_INVALID, "the factored weighted schedule needs at least 12 qubits");
  if (flags & (QAOA_RUN_EXACT | QAOA_RUN_SHARDED))
    return fail(QAOA_E_INVALID, "the factored weighted schedule is fast-mode and unsharded only");
  if ((rc = run_begin(c, p, nullptr, cs, sn, flags, false, gammas, true))) return rc;
  for (size_t k = 0; k + 1 < c->run.seg_start.size(); ++k)
    if ((rc = run_segment(c, (int)k))) return rc;
  return run_end(c);
}

int qaoa_run_begin(qaoa_ctx* c, int p, const double* phase_tables, const double* cs,
                   const double* sn, int flags, int* n_segments) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!c->has_graph) return fail(QAOA_E_STATE, "no graph set");
  if (p < 1) return fail(QAOA_E_INVALID, "planned runs need at least one level");
  if (!phase_tables || !cs || !sn) return fail(QAOA_E_INVALID, "null angle arrays");
  if (c->n < 12) return fail(QAOA_E_INVALID, "planned runs need at least 12 local qubits");
  if ((rc = run_begin(c, p, phase_tables, cs, sn, flags, (flags & QAOA_RUN_SHARDED) != 0))) return rc;
  if (n_segments) *n_segments = (int)c->run.seg_start.size() - 1;
  return QAOA_OK;
}

int qaoa_run_segment(qaoa_ctx* c, int k) {
  int rc = check_ctx(c);
  if (rc) return rc;
  return run_segment(c, k);
}

int qaoa_run_exchange_info(qaoa_ctx* c, int k, int* level, double* rx, double* factor) {
  int rc = check_ctx(c);
  if (rc) return rc;
  const RunState& R = c->run;
  if (!R.active) return fail(QAOA_E_STATE, "no planned run (qaoa_run_begin)");
  if (k < 0 || k + 1 >= (int)R.seg_start.size()) return fail(QAOA_E_RANGE, "segment out of range");
  const int l = R.plan[R.seg_start[k + 1] - 1].exchange;
  if (l < 0) return fail(QAOA_E_RANGE, "no exchange after this segment");
  if (level) *level = l;
  if (rx) {
    rx[0] = R.stages[l].a;
    rx[1] = R.stages[l].b;
    rx[2] = R.stages[l].mode;
  }
  if (factor) {
    factor[0] = R.level_factor[l].real();
    factor[1] = R.level_factor[l].imag();
  }
  return QAOA_OK;
}

int qaoa_run_end(qaoa_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  return run_end(c);
}

int qaoa_run_sweep_info(qaoa_ctx* c, int i, int* segment, int* carry, int* q, int64_t* ntiles) {
  int rc = check_ctx(c);
  if (rc) return rc;
  const RunState& R = c->run;
  if (!R.active) return fail(QAOA_E_STATE, "no planned run (qaoa_run_begin)");
  if (i < 0 || i >= (int)R.plan.size()) return fail(QAOA_E_RANGE, "sweep out of range");
  int k = 0;
  while (k + 1 < (int)R.seg_start.size() && R.seg_start[k + 1] <= i) ++k;
  const SetDesc& st = R.sets[R.plan[i].set];
  if (segment) *segment = k;
  if (carry) *carry = st.carry;
  if (q) *q = st.q;
  if (ntiles) *ntiles = 1ll << (c->n - 12);
  return QAOA_OK;
}

int qaoa_run_sweep_range(qaoa_ctx* c, int i, int64_t tile_lo, int64_t tile_count) {
  int rc = check_ctx(c);
  if (rc) return rc;
  const RunState& R = c->run;
  if (!R.active) return fail(QAOA_E_STATE, "no planned run (qaoa_run_begin)");
  if (i < 0 || i >= (int)R.plan.size()) return fail(QAOA_E_RANGE, "sweep out of range");
  const int64_t nt = 1ll << (c->n - 12);
  if (tile_lo < 0 || tile_count < 1 || tile_lo + tile_count > nt)
    return fail(QAOA_E_RANGE, "tile range out of range");
  // an out-of-place sweep of the swapped layout visits its tiles in a permuted
  // order over the whole state: no partial ranges (sharded runs never swap)
  if (R.swap && R.do_swap[i] && (tile_lo != 0 || tile_count != nt))
    return fail(QAOA_E_STATE, "partial tile ranges need an in-place run (qaoa_set_layout_swap(ctx, 0))");
  return launch_plan_sweep(c, i, tile_lo, tile_count);
}

int qaoa_exchange(int device, void* stream, int g, void* const* shards, int n_local, int p0,
                  uint64_t y_lo, uint64_t y_hi, const double* rx, const double* factor) {
  if (g < 1 || g > 4) return fail(QAOA_E_INVALID, "shard bits must be in [1, 4]");
  if (!shards || !rx || !factor) return fail(QAOA_E_INVALID, "null argument");
  if (n_local < g || p0 < 0 || p0 + g > n_local) return fail(QAOA_E_RANGE, "swapped bits out of range");
  if (y_hi > (1ull << (n_local - g)) || y_lo > y_hi) return fail(QAOA_E_RANGE, "column range out of range");
  CUDA_TRY(cudaSetDevice(device));
  ExchangeArgs a;
  memset(&a, 0, sizeof(a));
  const int G = 1 << g;
  for (int r = 0; r < G; ++r) {
    if (!shards[r]) return fail(QAOA_E_INVALID, "null shard pointer");
    a.shards[r] = (double2*)shards[r];
  }
  a.g = g;
  a.p0 = p0;
  a.y_lo = y_lo;
  a.y_hi = y_hi;
  a.rx = RxStage{rx[0], rx[1], (int)rx[2]};
  const std::complex<double> f = std::pow(std::complex<double>(factor[0], factor[1]), g);
  a.scale = make_double2(f.real(), f.imag());
  a.scale_on = !(f.real() == 1.0 && f.imag() == 0.0);
  CUDA_TRY(launch_exchange(a, (cudaStream_t)stream));
  return QAOA_OK;
}

int qaoa_ipc_handle(qaoa_ctx* c, void* handle64) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!handle64) return fail(QAOA_E_INVALID, "null handle buffer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->amps));
  memcpy(handle64, &h, sizeof(h));
  return QAOA_OK;
}

int qaoa_ipc_open(const void* handle64, int device, void** out_ptr) {
  if (!handle64 || !out_ptr) return fail(QAOA_E_INVALID, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return QAOA_OK;
}

int qaoa_ipc_close(void* ptr) {
  CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return QAOA_OK;
}

int qaoa_set_weights(qaoa_ctx* c, int m, const int* ei, const int* ej, const double* w) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (m < 0 || (m && (!ei || !ej || !w))) return fail(QAOA_E_INVALID, "bad edge list");
  for (int e = 0; e < m; ++e)
    if (ei[e] < 0 || ej[e] < 0 || ei[e] >= 64 || ej[e] >= 64 || ei[e] == ej[e])
      return fail(QAOA_E_INVALID, "edge endpoint out of range");
  if (c->d_ei) cudaFree(c->d_ei);
  if (c->d_ej) cudaFree(c->d_ej);
  if (c->d_w) cudaFree(c->d_w);
  c->d_ei = nullptr;
  c->d_ej = nullptr;
  c->d_w = nullptr;
  const size_t cnt = (size_t)std::max(m, 1);
  CUDA_TRY(cudaMalloc(&c->d_ei, cnt * sizeof(int)));
  CUDA_TRY(cudaMalloc(&c->d_ej, cnt * sizeof(int)));
  CUDA_TRY(cudaMalloc(&c->d_w, cnt * sizeof(double)));
  if (m) {
    CUDA_TRY(cudaMemcpyAsync(c->d_ei, ei, m * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_ej, ej, m * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_w, w, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  // endpoints + incidence lists for the factored cost of the fast schedule
  c->h_ei.assign(ei, ei + m);
  c->h_ej.assign(ej, ej + m);
  c->h_w.assign(w, w + m);
  std::vector<int2> edge(cnt, make_int2(0, 0));
  std::vector<int> off(66, 0), inc(2 * cnt, 0);
  for (int e = 0; e < m; ++e) {
    edge[e] = make_int2(ei[e], ej[e]);
    ++off[ei[e] + 1];
    ++off[ej[e] + 1];
  }
  for (int i = 0; i < 65; ++i) off[i + 1] += off[i];
  std::vector<int> fill(off.begin(), off.end() - 1);
  for (int e = 0; e < m; ++e) {
    inc[fill[ei[e]]++] = e;
    inc[fill[ej[e]]++] = e;
  }
  if (c->d_wedge) cudaFree(c->d_wedge);
  if (c->d_winc_off) cudaFree(c->d_winc_off);
  if (c->d_winc) cudaFree(c->d_winc);
  c->d_wedge = nullptr;
  c->d_winc_off = nullptr;
  c->d_winc = nullptr;
  CUDA_TRY(cudaMalloc(&c->d_wedge, cnt * sizeof(int2)));
  CUDA_TRY(cudaMalloc(&c->d_winc_off, 66 * sizeof(int)));
  CUDA_TRY(cudaMalloc(&c->d_winc, 2 * cnt * sizeof(int)));
  CUDA_TRY(cudaMemcpyAsync(c->d_wedge, edge.data(), cnt * sizeof(int2), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_winc_off, off.data(), 66 * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->d_winc, inc.data(), 2 * cnt * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->n_wedges = m;
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_apply_cost_weighted(qaoa_ctx* c, double gamma) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (c->n_wedges < 0) return fail(QAOA_E_STATE, "no weighted edge list set");
  const uint64_t xbase = c->g.x_hi ^ c->g.cmask;
  CUDA_TRY(launch_cost_weighted(c->amps, 1ull << c->n, xbase, c->d_ei, c->d_ej, c->d_w,
                                c->n_wedges, gamma, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

int qaoa_expectation_weighted(qaoa_ctx* c, double* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!out) return fail(QAOA_E_INVALID, "null output");
  if (c->n_wedges < 0) return fail(QAOA_E_STATE, "no weighted edge list set");
  if (c->expect_valid && c->expect_is_weighted) {  // fused into the last weighted run
    *out = c->expect_value;
    return QAOA_OK;
  }
  if ((rc = require_stored(c))) return rc;
  const int grid = reduce_grid();
  if ((rc = ensure_partials(c, grid))) return rc;
  const uint64_t xbase = c->g.x_hi ^ c->g.cmask;
  CUDA_TRY(launch_expectation_weighted(c->amps, 1ull << c->n, xbase, c->d_ei, c->d_ej, c->d_w,
                                       c->n_wedges, c->partials, grid, c->stream));
  return reduce_to_host(c, grid, 0, out);
}

int qaoa_block_norms(qaoa_ctx* c, int block_bits, double* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (block_bits < 0 || block_bits > 12 || block_bits > c->n || !out)
    return fail(QAOA_E_INVALID, "bad block size");
  const int bits = c->n + (c->mirror_view ? 1 : 0);
  const uint64_t nb = 1ull << (bits - block_bits);
  double* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, nb * sizeof(double)));
  cudaError_t e = launch_block_norms(c->amps, block_bits, nb, c->g.cmask & local_mask(c),
                                     c->mirror_view ? (1ull << c->n) : 0ull, d, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, nb * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "qaoa_block_norms");
  return QAOA_OK;
}

int qaoa_sample_blocks(qaoa_ctx* c, int block_bits, int64_t n_groups, const int64_t* group_block,
                       const double* group_base, const int64_t* group_off, const double* targets,
                       int64_t* out_idx) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (block_bits < 0 || block_bits > 12 || block_bits > c->n || n_groups < 0)
    return fail(QAOA_E_INVALID, "bad sampling arguments");
  if (n_groups == 0) return QAOA_OK;
  const int64_t shots = group_off[n_groups];
  void* mem = nullptr;
  const size_t bytes = n_groups * (sizeof(int64_t) + sizeof(double)) + (n_groups + 1) * sizeof(int64_t) +
                       shots * (sizeof(double) + sizeof(int64_t));
  CUDA_TRY(cudaMalloc(&mem, bytes));
  char* p = (char*)mem;
  int64_t* d_gb = (int64_t*)p; p += n_groups * sizeof(int64_t);
  double* d_base = (double*)p; p += n_groups * sizeof(double);
  int64_t* d_off = (int64_t*)p; p += (n_groups + 1) * sizeof(int64_t);
  double* d_t = (double*)p; p += shots * sizeof(double);
  int64_t* d_out = (int64_t*)p;
  cudaError_t e = cudaMemcpyAsync(d_gb, group_block, n_groups * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_base, group_base, n_groups * sizeof(double), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_off, group_off, (n_groups + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_t, targets, shots * sizeof(double), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = launch_sample_blocks(c->amps, block_bits, c->g.cmask & local_mask(c),
                                                 c->mirror_view ? (1ull << c->n) : 0ull, n_groups, d_gb,
                                                 d_base, d_off, d_t, d_out, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_idx, d_out, shots * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(mem);
  if (e != cudaSuccess) return cuda_fail(e, "qaoa_sample_blocks");
  return QAOA_OK;
}

int qaoa_expectation(qaoa_ctx* c, double* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!out) return fail(QAOA_E_INVALID, "null output");
  if (!c->has_graph) return fail(QAOA_E_STATE, "no graph set");
  if (c->expect_valid && !c->expect_is_weighted) {
    *out = c->expect_value;
    return QAOA_OK;
  }
  if ((rc = require_stored(c))) return rc;
  const int grid = reduce_grid();
  if ((rc = ensure_partials(c, grid))) return rc;
  CUDA_TRY(launch_expectation(c->amps, c->n, c->g, c->partials, grid, c->stream));
  if ((rc = reduce_to_host(c, grid, 0, out))) return rc;
  c->expect_value = *out;
  c->expect_valid = true;
  return QAOA_OK;
}

int qaoa_norm_sq(qaoa_ctx* c, double* out) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (!out) return fail(QAOA_E_INVALID, "null output");
  const int grid = reduce_grid();
  if ((rc = ensure_partials(c, grid))) return rc;
  CUDA_TRY(launch_norm_sq(c->amps, 1ull << c->n, c->partials, grid, c->stream));
  return reduce_to_host(c, grid, 0, out);
}

int qaoa_max_abs_diff(qaoa_ctx* a, qaoa_ctx* b, double* out) {
  int rc = check_ctx(a);
  if (rc) return rc;
  if (!b || !out) return fail(QAOA_E_INVALID, "null argument");
  if (a->n != b->n) {
    char buf[96];
    snprintf(buf, sizeof buf, "qubit counts differ: %d vs %d", a->n, b->n);
    return fail(QAOA_E_INVALID, buf);
  }
  if (a->device != b->device) return fail(QAOA_E_INVALID, "states live on different devices");
  CUDA_TRY(cudaStreamSynchronize(b->stream));
  const int grid = reduce_grid();
  if ((rc = ensure_partials(a, grid))) return rc;
  const uint64_t xmask = (a->g.cmask ^ b->g.cmask) & local_mask(a);
  CUDA_TRY(launch_max_abs_diff(a->amps, b->amps, 1ull << a->n, xmask, a->partials, grid, a->stream));
  return reduce_to_host(a, grid, 1, out);
}

int qaoa_build_cut_table(qaoa_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!c->has_graph) return fail(QAOA_E_STATE, "no graph set");
  const int bytes_per = c->g.tot_edge <= 255 ? 1 : 2;
  if (!c->cut_table || c->cut_bytes != bytes_per) {
    if (c->cut_table) cudaFree(c->cut_table);
    c->cut_table = nullptr;
    cudaError_t e = cudaMalloc(&c->cut_table, (size_t)bytes_per << c->n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(QAOA_E_NOMEM, "cannot allocate the cut table");
    }
    c->cut_bytes = bytes_per;
  }
  GraphDev gt = c->g;
  gt.cmask = 0;  // the table is of true indices, independent of the state
  // the launch is bracketed by CUDA events (qaoa_layer_timings then returns its
  // device time, without the host's launch latency)
  if ((rc = record_event(c, true, 0))) return rc;
  if (c->n >= 11) CUDA_TRY(launch_cut_table_warps(c->cut_table, bytes_per, c->n, gt, c->stream));
  else CUDA_TRY(launch_cut_table(c->cut_table, bytes_per, c->n, gt, c->stream));
  if ((rc = record_event(c, true, 1))) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->events[0], c->events[1]));
  c->times.assign(1, ms);
  return QAOA_OK;
}

int qaoa_read_cut_table(qaoa_ctx* c, uint64_t offset, uint64_t count, int64_t* dst) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (!c->cut_table) return fail(QAOA_E_STATE, "cut table not built");
  if (offset + count > (1ull << c->n)) return fail(QAOA_E_RANGE, "cut-table range out of bounds");
  if (count && !dst) return fail(QAOA_E_INVALID, "null destination");
  std::vector<uint8_t> tmp(count * c->cut_bytes);
  CUDA_TRY(cudaMemcpyAsync(tmp.data(), (uint8_t*)c->cut_table + offset * c->cut_bytes,
                           count * c->cut_bytes, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  if (c->cut_bytes == 1) {
    for (uint64_t i = 0; i < count; ++i) dst[i] = tmp[i];
  } else {
    const uint16_t* t16 = (const uint16_t*)tmp.data();
    for (uint64_t i = 0; i < count; ++i) dst[i] = t16[i];
  }
  return QAOA_OK;
}

int qaoa_free_cut_table(qaoa_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (c->cut_table) cudaFree(c->cut_table);
  c->cut_table = nullptr;
  return QAOA_OK;
}

int qaoa_layer_timings(qaoa_ctx* c, float* ms, int cap) {
  if (!c) return fail(QAOA_E_INVALID, "null context");
  const int n = (int)c->times.size();
  for (int i = 0; i < n && i < cap; ++i) ms[i] = c->times[i];
  return n;
}

int qaoa_last_run_stats(qaoa_ctx* c, int* launches, double* hbm_bytes) {
  if (!c) return fail(QAOA_E_INVALID, "null context");
  if (launches) *launches = c->last_launches;
  if (hbm_bytes) *hbm_bytes = c->last_bytes;
  return QAOA_OK;
}

int qaoa_synchronize(qaoa_ctx* c) {
  int rc = check_ctx(c);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return QAOA_OK;
}

int qaoa_pack_chunks(qaoa_ctx* c, int g, const int* local_bits, void* dst) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if ((rc = require_stored(c))) return rc;
  if (g < 0 || g > 8 || g > c->n || (g && (!local_bits || !dst)))
    return fail(QAOA_E_INVALID, "bad chunk spec");
  for (int k = 0; k < g; ++k) {
    if (local_bits[k] < 0 || local_bits[k] >= c->n || (k && local_bits[k] <= local_bits[k - 1]))
      return fail(QAOA_E_INVALID, "local bits must be ascending and in range");
  }
  CUDA_TRY(launch_pack_chunks(c->amps, c->n, g, local_bits, (double2*)dst, c->stream));
  return QAOA_OK;
}

int qaoa_unpack_chunks(qaoa_ctx* c, int g, const int* local_bits, const void* src) {
  int rc = check_ctx(c);
  if (rc) return rc;
  if (g < 0 || g > 8 || g > c->n || (g && (!local_bits || !src)))
    return fail(QAOA_E_INVALID, "bad chunk spec");
  for (int k = 0; k < g; ++k) {
    if (local_bits[k] < 0 || local_bits[k] >= c->n || (k && local_bits[k] <= local_bits[k - 1]))
      return fail(QAOA_E_INVALID, "local bits must be ascending and in range");
  }
  CUDA_TRY(launch_unpack_chunks(c->amps, c->n, g, local_bits, (const double2*)src, c->stream));
  c->expect_valid = false;
  return QAOA_OK;
}

}  // extern "C"
