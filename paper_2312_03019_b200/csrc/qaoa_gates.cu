// qaoa_gates.cu -- per-gate and per-element kernels of the B200 QAOA engine:
// single cost layer, single-qubit RX, launch-control fill, <C> reduction, norm,
// max-abs-diff, the bitwise cut-table builder and the shard pack/unpack used by
// the global-qubit exchange.  The fused multi-qubit sweeps are in qaoa_sweep.cu.
#include "qaoa_common.cuh"
#include "qaoa_sweep.h"

namespace qb {

constexpr int kBlock = 256;

static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
  }
  return sms;
}

int reduce_grid() { return num_sms() * 4; }

static int grid_for(uint64_t work, int per_thread) {
  const uint64_t threads = (work + per_thread - 1) / per_thread;
  uint64_t blocks = (threads + kBlock - 1) / kBlock;
  const uint64_t cap = (uint64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

// ---- launch control: circuit.py:42-48 -------------------------------------
__global__ void fill_kernel(double2* __restrict__ amps, uint64_t n, double2 v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(amps + i, v);
}

cudaError_t launch_fill(double2* amps, uint64_t n, double2 v, cudaStream_t s) {
  fill_kernel<<<grid_for(n, 4), kBlock, 0, s>>>(amps, n, v);
  return cudaGetLastError();
}

// ---- single cost layer: apply_cost_bitwise cost.py:162-176 -----------------
// Thread handles 16 amplitudes whose bits 5..8 vary (lanes on bits 0..4, so
// every load instruction of a warp reads 512 contiguous bytes).
template <bool WIDE>
__global__ void cost_gate_kernel(double2* __restrict__ amps, int n_local, GraphDev g,
                                 const double2* __restrict__ table) {
  const uint64_t groups = 1ull << (n_local - 9);   // groups of 512 amplitudes
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const int v[4] = {5, 6, 7, 8};
  for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < groups;
       w += warps) {
    const uint64_t x0 = (w << 9) | (uint64_t)lane;
    int c[16];
    cut_counts16<WIDE>((g.x_hi | x0) ^ g.cmask, v, g, c);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const uint64_t x = x0 | ((uint64_t)r << 5);
      amps[x] = cmul_np(amps[x], table[2 * g.tot_edge - 2 * c[r]]);
    }
  }
}

template <bool WIDE>
__global__ void cost_gate_small_kernel(double2* __restrict__ amps, uint64_t n, GraphDev g,
                                       const double2* __restrict__ table) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const int c = cut_count<WIDE>((g.x_hi | x) ^ g.cmask, g);
    amps[x] = cmul_np(amps[x], table[2 * g.tot_edge - 2 * c]);
  }
}

cudaError_t launch_cost_gate(double2* amps, uint64_t n, const GraphDev& g, const double2* table,
                             cudaStream_t s) {
  int n_local = 0;
  while ((1ull << n_local) < n) ++n_local;
  const bool wide = g.n_nodes > 32;
  if (n_local >= 9) {
    const int grid = grid_for(n, 16);
    if (wide) cost_gate_kernel<true><<<grid, kBlock, 0, s>>>(amps, n_local, g, table);
    else cost_gate_kernel<false><<<grid, kBlock, 0, s>>>(amps, n_local, g, table);
  } else {
    if (wide) cost_gate_small_kernel<true><<<1, kBlock, 0, s>>>(amps, n, g, table);
    else cost_gate_small_kernel<false><<<1, kBlock, 0, s>>>(amps, n, g, table);
  }
  return cudaGetLastError();
}

// ---- single-qubit RX: apply_rx state.py:110-128 (bit-exact) ----------------
__global__ void rx_gate_kernel(double2* __restrict__ amps, int n_local, int q, double c,
                               double sn) {
  const uint64_t half = 1ull << (n_local - 1);
  const uint64_t stride = 1ull << q;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < half;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = ((k >> q) << (q + 1)) | (k & (stride - 1));
    double2 a = amps[i0], b = amps[i0 | stride];
    rx_exact(a, b, c, sn);
    amps[i0] = a;
    amps[i0 | stride] = b;
  }
}

cudaError_t launch_rx_gate(double2* amps, int n_local, int q, double c, double sn,
                           cudaStream_t s) {
  rx_gate_kernel<<<grid_for(1ull << (n_local - 1), 2), kBlock, 0, s>>>(amps, n_local, q, c, sn);
  return cudaGetLastError();
}

// ---- gate-level baseline (reference backend "baseline", launch_control=False)
// Hadamard on qubit q (state.py:91-107): top = (a + b) * k, bot = (a - b) * k,
// k = 1/sqrt(2) rounded once (state.py:22), every operation rounded separately.
// `flip`: the stored state has qubit q complemented (fast-mode bookkeeping),
// so the stored pair is (true b, true a): the same butterfly with the
// outputs exchanged (a + b = b + a exactly).
__global__ void h_gate_kernel(double2* __restrict__ amps, int n_local, int q, int flip,
                              double k) {
  const uint64_t half = 1ull << (n_local - 1);
  const uint64_t stride = 1ull << q;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < half;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = ((i >> q) << (q + 1)) | (i & (stride - 1));
    const double2 a = amps[i0], b = amps[i0 | stride];
    const double2 top = make_double2(__dmul_rn(__dadd_rn(a.x, b.x), k), __dmul_rn(__dadd_rn(a.y, b.y), k));
    const double2 bot = flip
        ? make_double2(__dmul_rn(__dsub_rn(b.x, a.x), k), __dmul_rn(__dsub_rn(b.y, a.y), k))
        : make_double2(__dmul_rn(__dsub_rn(a.x, b.x), k), __dmul_rn(__dsub_rn(a.y, b.y), k));
    amps[i0] = flip ? bot : top;
    amps[i0 | stride] = flip ? top : bot;
  }
}

cudaError_t launch_h_gate(double2* amps, int n_local, int q, int flip, cudaStream_t s) {
  const double k = 1.0 / sqrt(2.0);
  h_gate_kernel<<<grid_for(1ull << (n_local - 1), 2), kBlock, 0, s>>>(amps, n_local, q, flip, k);
  return cudaGetLastError();
}

// RZZ(theta) on qubits q1, q2 (state.py:131-149): amp *= (bit q1 != bit q2) ?
// e_diff : e_same, the two phases formed on the host by numpy exactly as the
// reference does; numpy's FMA-form complex multiply (cmul_np).  x = xbase ^ y
// is the true index of stored element y (x_hi and the complement mask).
__global__ void rzz_gate_kernel(double2* __restrict__ amps, uint64_t n, uint64_t xbase, int q1,
                                int q2, double2 e_same, double2 e_diff) {
  for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < n;
       y += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = xbase ^ y;
    const bool diff = ((x >> q1) ^ (x >> q2)) & 1ull;
    amps[y] = cmul_np(amps[y], diff ? e_diff : e_same);
  }
}

cudaError_t launch_rzz_gate(double2* amps, uint64_t n, uint64_t xbase, int q1, int q2,
                            double2 e_same, double2 e_diff, cudaStream_t s) {
  rzz_gate_kernel<<<grid_for(n, 4), kBlock, 0, s>>>(amps, n, xbase, q1, q2, e_same, e_diff);
  return cudaGetLastError();
}

// RX on the virtual top qubit of a symmetric half state: stored index y pairs
// with y ^ M (M = all local bits), i.e. element y of the first half with the
// mirrored element of the second half.  mode 0: the reference's butterfly
// (rx_exact, c / s), mode 1: the factored fast form (t), then `scale` (the
// level's per-qubit factor) when scale_on.  Thread k handles y = k (bit n-1
// clear) and its partner; consecutive threads read consecutive y and
// consecutive (descending) partners, both coalesced.
__global__ void mirror_rx_kernel(double2* __restrict__ amps, int n_local, RxStage st, double2 scale,
                                 int scale_on) {
  const uint64_t half = 1ull << (n_local - 1);
  const uint64_t M = (1ull << n_local) - 1ull;
  for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < half;
       y += (uint64_t)gridDim.x * blockDim.x) {
    double2 a = amps[y], b = amps[y ^ M];
    if (st.mode == 0) rx_exact(a, b, st.a, st.b);
    else rx_form1(a, b, st.a);
    if (scale_on) {
      a = cmul_np(a, scale);
      b = cmul_np(b, scale);
    }
    amps[y] = a;
    amps[y ^ M] = b;
  }
}

cudaError_t launch_mirror_rx(double2* amps, int n_local, RxStage st, double2 scale, int scale_on,
                             cudaStream_t s) {
  mirror_rx_kernel<<<grid_for(1ull << (n_local - 1), 2), kBlock, 0, s>>>(amps, n_local, st, scale,
                                                                           scale_on);
  return cudaGetLastError();
}

// |index>: zero everywhere, 1 at `index` (init_zero_state, state.py:66-72).
__global__ void basis_kernel(double2* __restrict__ amps, uint64_t n, uint64_t index) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    __stcs(amps + i, make_double2(i == index ? 1.0 : 0.0, 0.0));
}

cudaError_t launch_basis(double2* amps, uint64_t n, uint64_t index, cudaStream_t s) {
  basis_kernel<<<grid_for(n, 4), kBlock, 0, s>>>(amps, n, index);
  return cudaGetLastError();
}

// Per-index edge sums in the reference's edge order for TRUE indices
// x = first + i: kind 0 = rotation totals sum_e w_e (1 - 2 [x_i != x_j])
// (CompressedCostPlan.rotation_totals, cost.py:77-86), kind 1 = cut values
// sum_e w_e [x_i != x_j] (cut_values_array, graph.py:144-151); bit-identical.
__global__ void edge_values_kernel(double* __restrict__ out, uint64_t first, uint64_t count,
                                   const int* __restrict__ ei, const int* __restrict__ ej,
                                   const double* __restrict__ w, int m, int kind) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = first + i;
    double v = 0.0;
    for (int e = 0; e < m; ++e) {
      const uint64_t diff = ((x >> __ldg(ei + e)) ^ (x >> __ldg(ej + e))) & 1ull;
      const double we = __ldg(w + e);
      v = kind == 0 ? __dadd_rn(v, __dmul_rn(we, diff ? -1.0 : 1.0))
                    : __dadd_rn(v, __dmul_rn(we, diff ? 1.0 : 0.0));
    }
    out[i] = v;
  }
}

cudaError_t launch_edge_values(double* out, uint64_t first, uint64_t count, const int* ei,
                               const int* ej, const double* w, int m, int kind, cudaStream_t s) {
  edge_values_kernel<<<grid_for(count, 1), kBlock, 0, s>>>(out, first, count, ei, ej, w, m, kind);
  return cudaGetLastError();
}

// ---- whole circuit for small states (n <= 11) in ONE CTA -------------------
// The state (<= 2048 amplitudes, 32 KB) lives in shared memory for all p
// levels: launch control, per level the cost (cost.py:162-176, FMA-form
// multiply) and RX on every qubit in increasing order (state.py:110-128, the
// reference's rounding), then <C> (fixed-order block sum).  The same
// operations in the same order as the per-gate kernels, so bit-identical to
// them and to the reference; one launch instead of p (n + 1) + 2.
template <bool WIDE>
__global__ void __launch_bounds__(kBlock) small_run_kernel(double2* __restrict__ amps, int n, GraphDev g,
                                                           const double2* __restrict__ tables,
                                                           const double2* __restrict__ rx, int p,
                                                           int from_state, double u, int want_expect,
                                                           double* __restrict__ expect_out) {
  extern __shared__ double2 st[];
  __shared__ double scratch[kBlock / 32];
  const int N = 1 << n;
  const int tl = 2 * g.tot_edge + 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) st[i] = from_state ? amps[i] : make_double2(u, 0.0);
  __syncthreads();
  for (int l = 0; l < p; ++l) {
    const double2* tab = tables + (size_t)l * tl;
    for (int i = threadIdx.x; i < N; i += blockDim.x)
      st[i] = cmul_np(st[i], tab[2 * g.tot_edge - 2 * cut_count<WIDE>((g.x_hi | (uint64_t)i) ^ g.cmask, g)]);
    __syncthreads();
    const double c = rx[l].x, sn = rx[l].y;
    for (int q = 0; q < n; ++q) {
      for (int k = threadIdx.x; k < N / 2; k += blockDim.x) {
        const int i0 = ((k >> q) << (q + 1)) | (k & ((1 << q) - 1));
        double2 a = st[i0], b = st[i0 | (1 << q)];
        rx_exact(a, b, c, sn);
        st[i0] = a;
        st[i0 | (1 << q)] = b;
      }
      __syncthreads();
    }
  }
  double acc = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double2 a = st[i];
    amps[i] = a;
    if (want_expect)
      acc += (a.x * a.x + a.y * a.y) * (double)cut_count<WIDE>((g.x_hi | (uint64_t)i) ^ g.cmask, g);
  }
  if (want_expect) {
    const double t = block_sum<kBlock>(acc, scratch);
    if (threadIdx.x == 0) *expect_out = t;
  }
}

cudaError_t launch_small_run(double2* amps, int n, const GraphDev& g, const double2* tables,
                             const double2* rx, int p, int from_state, double u, int want_expect,
                             double* expect_out, cudaStream_t s) {
  if (n > 11) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double2) << n;
  if (g.n_nodes > 32)
    small_run_kernel<true><<<1, kBlock, smem, s>>>(amps, n, g, tables, rx, p, from_state, u, want_expect,
                                                   expect_out);
  else
    small_run_kernel<false><<<1, kBlock, smem, s>>>(amps, n, g, tables, rx, p, from_state, u, want_expect,
                                                    expect_out);
  return cudaGetLastError();
}

// ---- <C> reduction: expectation circuit.py:116-121 -------------------------
template <bool WIDE>
__global__ void expectation_kernel(const double2* __restrict__ amps, int n_local, GraphDev g,
                                   double* __restrict__ partials) {
  __shared__ double scratch[kBlock / 32];
  double acc = 0.0;
  if (n_local >= 9) {
    const uint64_t groups = 1ull << (n_local - 9);
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const int v[4] = {5, 6, 7, 8};
    for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < groups;
         w += warps) {
      const uint64_t x0 = (w << 9) | (uint64_t)lane;
      int c[16];
      cut_counts16<WIDE>((g.x_hi | x0) ^ g.cmask, v, g, c);
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const double2 a = __ldcs(amps + (x0 | ((uint64_t)r << 5)));
        acc += (a.x * a.x + a.y * a.y) * (double)c[r];
      }
    }
  } else {
    const uint64_t n = 1ull << n_local;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x) {
      const double2 a = amps[x];
      acc += (a.x * a.x + a.y * a.y) * (double)cut_count<WIDE>((g.x_hi | x) ^ g.cmask, g);
    }
  }
  const double t = block_sum<kBlock>(acc, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

cudaError_t launch_expectation(const double2* amps, int n_local, const GraphDev& g,
                               double* partials, int grid, cudaStream_t s) {
  if (g.n_nodes > 32) expectation_kernel<true><<<grid, kBlock, 0, s>>>(amps, n_local, g, partials);
  else expectation_kernel<false><<<grid, kBlock, 0, s>>>(amps, n_local, g, partials);
  return cudaGetLastError();
}

// ---- weighted graphs: the compressed backend (cost.py:77-86, :147-159) and the
// float cut values of expectation (graph.py:144-151).  Totals are accumulated
// per amplitude in the reference's edge order, so they are bit-identical to
// rotation_totals() / cut_values_array(); the phase is (cos y, sin y) with
// y = -(0.5 gamma) t exactly as np.exp(-0.5j * gamma * totals) forms it.
struct EdgeList {
  const int* ei;
  const int* ej;
  const double* w;
  int m;
};

__global__ void cost_weighted_kernel(double2* __restrict__ amps, uint64_t n, uint64_t xbase,
                                     EdgeList el, double half_gamma) {
  for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < n;
       y += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = xbase ^ y;
    double t = 0.0;
    for (int e = 0; e < el.m; ++e) {
      const uint64_t diff = ((x >> __ldg(el.ei + e)) ^ (x >> __ldg(el.ej + e))) & 1ull;
      t = __dadd_rn(t, __dmul_rn(__ldg(el.w + e), diff ? -1.0 : 1.0));
    }
    double sn, cs;
    sincos(-__dmul_rn(half_gamma, t), &sn, &cs);
    amps[y] = cmul_np(amps[y], make_double2(cs, sn));
  }
}

__global__ void expectation_weighted_kernel(const double2* __restrict__ amps, uint64_t n,
                                            uint64_t xbase, EdgeList el,
                                            double* __restrict__ partials) {
  __shared__ double scratch[kBlock / 32];
  double acc = 0.0;
  for (uint64_t y = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; y < n;
       y += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = xbase ^ y;
    double v = 0.0;
    for (int e = 0; e < el.m; ++e) {
      const uint64_t diff = ((x >> __ldg(el.ei + e)) ^ (x >> __ldg(el.ej + e))) & 1ull;
      v = __dadd_rn(v, diff ? __ldg(el.w + e) : 0.0);
    }
    const double2 a = amps[y];
    acc += (a.x * a.x + a.y * a.y) * v;
  }
  const double t = block_sum<kBlock>(acc, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

cudaError_t launch_cost_weighted(double2* amps, uint64_t n, uint64_t xbase, const int* ei,
                                 const int* ej, const double* w, int m, double gamma,
                                 cudaStream_t s) {
  EdgeList el{ei, ej, w, m};
  cost_weighted_kernel<<<grid_for(n, 1), kBlock, 0, s>>>(amps, n, xbase, el, 0.5 * gamma);
  return cudaGetLastError();
}

cudaError_t launch_expectation_weighted(const double2* amps, uint64_t n, uint64_t xbase,
                                        const int* ei, const int* ej, const double* w, int m,
                                        double* partials, int grid, cudaStream_t s) {
  EdgeList el{ei, ej, w, m};
  expectation_weighted_kernel<<<grid, kBlock, 0, s>>>(amps, n, xbase, el, partials);
  return cudaGetLastError();
}

// ---- sampling (circuit.py:124-133): numpy's Generator.choice(p=|a|^2) is
// cdf = cumsum(p) / cdf[-1]; idx = searchsorted(cdf, uniform, 'right').  The
// device computes |a|^2 block sums in true index order (kernel 1); the host
// prefix-sums the blocks and assigns each target to a block; kernel 2 scans
// each hit block once in shared memory and binary-searches its targets.
constexpr int kSampleBlockMax = 4096;

// Stored position of true index x: x ^ lmask, and for a symmetric half state
// (fold = 2^n, the virtual top bit) the upper half folded onto the stored one,
// psi(v) = psi(~v): the sampling kernels then walk the 2^(n+1) virtual indices
// in true order, the same sums as on the full state.
__device__ __forceinline__ uint64_t stored_index(uint64_t x, uint64_t lmask, uint64_t fold) {
  const uint64_t v = x ^ lmask;
  return (v & fold) ? (~v & (fold - 1ull)) : v;
}

__global__ void block_norms_kernel(const double2* __restrict__ amps, int block_bits,
                                   uint64_t lmask, uint64_t fold, double* __restrict__ out) {
  __shared__ double scratch[kBlock / 32];
  const uint64_t base = (uint64_t)blockIdx.x << block_bits;
  double acc = 0.0;
  for (int i = threadIdx.x; i < (1 << block_bits); i += kBlock) {
    const double2 a = amps[stored_index(base + i, lmask, fold)];
    acc += a.x * a.x + a.y * a.y;
  }
  const double t = block_sum<kBlock>(acc, scratch);
  if (threadIdx.x == 0) out[blockIdx.x] = t;
}

__global__ void sample_blocks_kernel(const double2* __restrict__ amps, int block_bits,
                                     uint64_t lmask, uint64_t fold, const int64_t* __restrict__ gblock,
                                     const double* __restrict__ gbase,
                                     const int64_t* __restrict__ goff,
                                     const double* __restrict__ targets,
                                     int64_t* __restrict__ out) {
  __shared__ double cdf[kSampleBlockMax];
  __shared__ double wsum[kBlock / 32];
  const int64_t blk = gblock[blockIdx.x];
  const uint64_t base = (uint64_t)blk << block_bits;
  const int len = 1 << block_bits;
  const int per = (len + kBlock - 1) / kBlock;  // contiguous run per thread
  const int lo = threadIdx.x * per;
  double run = 0.0;
  for (int i = lo; i < lo + per && i < len; ++i) {
    const double2 a = amps[stored_index(base + i, lmask, fold)];
    run += a.x * a.x + a.y * a.y;
    cdf[i] = run;
  }
  // exclusive prefix of the per-thread run totals (warp scan, then warps)
  double x = run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  double off = gbase[blockIdx.x];
  for (int w = 0; w < warp; ++w) off += wsum[w];
  off += x - run;
  for (int i = lo; i < lo + per && i < len; ++i) cdf[i] += off;
  __syncthreads();
  for (int64_t s = goff[blockIdx.x] + threadIdx.x; s < goff[blockIdx.x + 1]; s += kBlock) {
    const double t = targets[s];
    int a = 0, b = len;  // first i with cdf[i] > t
    while (a < b) {
      const int m = (a + b) >> 1;
      if (cdf[m] > t) b = m;
      else a = m + 1;
    }
    out[s] = (int64_t)base + (a < len ? a : len - 1);
  }
}

cudaError_t launch_block_norms(const double2* amps, int block_bits, uint64_t n_blocks,
                               uint64_t lmask, uint64_t fold, double* out, cudaStream_t s) {
  block_norms_kernel<<<(unsigned)n_blocks, kBlock, 0, s>>>(amps, block_bits, lmask, fold, out);
  return cudaGetLastError();
}

cudaError_t launch_sample_blocks(const double2* amps, int block_bits, uint64_t lmask, uint64_t fold,
                                 int64_t n_groups, const int64_t* gblock, const double* gbase,
                                 const int64_t* goff, const double* targets, int64_t* out,
                                 cudaStream_t s) {
  sample_blocks_kernel<<<(unsigned)n_groups, kBlock, 0, s>>>(amps, block_bits, lmask, fold, gblock,
                                                              gbase, goff, targets, out);
  return cudaGetLastError();
}

// ---- norm^2 and max |a - b| (state.py:50-51, :152-156) ---------------------
__global__ void norm_sq_kernel(const double2* __restrict__ amps, uint64_t n,
                               double* __restrict__ partials) {
  __shared__ double scratch[kBlock / 32];
  double acc = 0.0;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const double2 a = __ldcs(amps + x);
    acc += a.x * a.x + a.y * a.y;
  }
  const double t = block_sum<kBlock>(acc, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

cudaError_t launch_norm_sq(const double2* amps, uint64_t n, double* partials, int grid,
                           cudaStream_t s) {
  norm_sq_kernel<<<grid, kBlock, 0, s>>>(amps, n, partials);
  return cudaGetLastError();
}

__global__ void max_abs_diff_kernel(const double2* __restrict__ a, const double2* __restrict__ b,
                                    uint64_t n, uint64_t xmask, double* __restrict__ partials) {
  __shared__ double scratch[kBlock / 32];
  double m = 0.0;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const double2 u = a[x], v = b[x ^ xmask];
    m = fmax(m, hypot(u.x - v.x, u.y - v.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) t = fmax(t, scratch[w]);
    partials[blockIdx.x] = t;
  }
}

cudaError_t launch_max_abs_diff(const double2* a, const double2* b, uint64_t n, uint64_t xmask,
                                double* partials, int grid, cudaStream_t s) {
  max_abs_diff_kernel<<<grid, kBlock, 0, s>>>(a, b, n, xmask, partials);
  return cudaGetLastError();
}

// Fixed-order pairwise reduction of the block partials (deterministic).
__global__ void sum_partials_kernel(const double* __restrict__ partials, int n,
                                    double* __restrict__ out, int mode_max) {
  __shared__ double s[1024];
  double v = mode_max ? 0.0 : 0.0;
  // thread t folds partials t, t+1024, ... in order
  for (int i = threadIdx.x; i < n; i += 1024) v = mode_max ? fmax(v, partials[i]) : v + partials[i];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      s[threadIdx.x] = mode_max ? fmax(s[threadIdx.x], s[threadIdx.x + w])
                                : s[threadIdx.x] + s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

cudaError_t launch_sum_partials(const double* partials, int n, double* out, int mode_max,
                                cudaStream_t s) {
  sum_partials_kernel<<<1, 1024, 0, s>>>(partials, n, out, mode_max);
  return cudaGetLastError();
}

// ---- cut-table builder: CompressedCostPlan.cut_counts cost.py:88-99 --------
// Thread t writes C(x) for x = 16t .. 16t+15 as one 16-byte (uint8) or two
// 16-byte (uint16) stores: C(16t) from the row-mask popcount sweep, the other
// 15 by flipping nodes 0..3 (delta = deg - 2 popc(adj & x), -2 per flipped edge).
template <bool WIDE, typename T>
__global__ void cut_table_kernel(T* __restrict__ table, int n_local, GraphDev g) {
  const uint64_t groups = 1ull << (n_local - 4);
  const int v[4] = {0, 1, 2, 3};
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < groups;
       t += (uint64_t)gridDim.x * blockDim.x) {
    int c[16];
    cut_counts16<WIDE>(g.x_hi | (t << 4), v, g, c);
    if (sizeof(T) == 1) {
      uint4 o;
      o.x = (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16) | ((uint32_t)c[3] << 24);
      o.y = (uint32_t)c[4] | ((uint32_t)c[5] << 8) | ((uint32_t)c[6] << 16) | ((uint32_t)c[7] << 24);
      o.z = (uint32_t)c[8] | ((uint32_t)c[9] << 8) | ((uint32_t)c[10] << 16) | ((uint32_t)c[11] << 24);
      o.w = (uint32_t)c[12] | ((uint32_t)c[13] << 8) | ((uint32_t)c[14] << 16) | ((uint32_t)c[15] << 24);
      __stcs(reinterpret_cast<uint4*>(table) + t, o);
    } else {
      uint4 o0, o1;
      o0.x = (uint32_t)c[0] | ((uint32_t)c[1] << 16);
      o0.y = (uint32_t)c[2] | ((uint32_t)c[3] << 16);
      o0.z = (uint32_t)c[4] | ((uint32_t)c[5] << 16);
      o0.w = (uint32_t)c[6] | ((uint32_t)c[7] << 16);
      o1.x = (uint32_t)c[8] | ((uint32_t)c[9] << 16);
      o1.y = (uint32_t)c[10] | ((uint32_t)c[11] << 16);
      o1.z = (uint32_t)c[12] | ((uint32_t)c[13] << 16);
      o1.w = (uint32_t)c[14] | ((uint32_t)c[15] << 16);
      __stcs(reinterpret_cast<uint4*>(table) + 2 * t, o0);
      __stcs(reinterpret_cast<uint4*>(table) + 2 * t + 1, o1);
    }
  }
}

template <bool WIDE, typename T>
__global__ void cut_table_small_kernel(T* __restrict__ table, uint64_t n, GraphDev g) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
       x += (uint64_t)gridDim.x * blockDim.x)
    table[x] = (T)cut_count<WIDE>(g.x_hi | x, g);
}

cudaError_t launch_cut_table(void* table, int bytes_per, int n_local, const GraphDev& g,
                             cudaStream_t s) {
  const bool wide = g.n_nodes > 32;
  const uint64_t n = 1ull << n_local;
  if (n_local >= 4) {
    const int grid = grid_for(n, 16);
    if (bytes_per == 1) {
      if (wide) cut_table_kernel<true, uint8_t><<<grid, kBlock, 0, s>>>((uint8_t*)table, n_local, g);
      else cut_table_kernel<false, uint8_t><<<grid, kBlock, 0, s>>>((uint8_t*)table, n_local, g);
    } else {
      if (wide) cut_table_kernel<true, uint16_t><<<grid, kBlock, 0, s>>>((uint16_t*)table, n_local, g);
      else cut_table_kernel<false, uint16_t><<<grid, kBlock, 0, s>>>((uint16_t*)table, n_local, g);
    }
  } else {
    if (bytes_per == 1) {
      if (wide) cut_table_small_kernel<true, uint8_t><<<1, kBlock, 0, s>>>((uint8_t*)table, n, g);
      else cut_table_small_kernel<false, uint8_t><<<1, kBlock, 0, s>>>((uint8_t*)table, n, g);
    } else {
      if (wide) cut_table_small_kernel<true, uint16_t><<<1, kBlock, 0, s>>>((uint16_t*)table, n, g);
      else cut_table_small_kernel<false, uint16_t><<<1, kBlock, 0, s>>>((uint16_t*)table, n, g);
    }
  }
  return cudaGetLastError();
}

// ---- shard pack / unpack for the global-qubit exchange ---------------------
// Chunk d (d in [0, 2^g)) = the amplitudes whose local bits L[0..g-1] spell d,
// ordered by their remaining local bits.  pack gathers, unpack scatters.
struct BitList {
  int b[8];
  int g;
};

__device__ __forceinline__ uint64_t chunk_index(uint64_t i, uint64_t d, const BitList& L) {
  // insert zeros at the sorted positions L.b (ascending), then set bits of d
  uint64_t x = i;
  for (int k = 0; k < L.g; ++k) {
    const int p = L.b[k];
    x = ((x >> p) << (p + 1)) | (x & ((1ull << p) - 1ull));
  }
  for (int k = 0; k < L.g; ++k) x |= ((d >> k) & 1ull) << L.b[k];
  return x;
}

template <bool PACK>
__global__ void chunk_kernel(double2* __restrict__ amps, int n_local, BitList L,
                             double2* __restrict__ buf) {
  const uint64_t chunk = 1ull << (n_local - L.g);
  const uint64_t total = 1ull << n_local;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < total;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = j / chunk, i = j % chunk;
    const uint64_t x = chunk_index(i, d, L);
    if (PACK) buf[j] = amps[x];
    else amps[x] = buf[j];
  }
}

static BitList make_bits(int g, const int* local_bits) {
  BitList L;
  L.g = g;
  for (int k = 0; k < g; ++k) L.b[k] = local_bits[k];
  return L;
}

cudaError_t launch_pack_chunks(const double2* amps, int n_local, int g, const int* local_bits,
                               double2* dst, cudaStream_t s) {
  BitList L = make_bits(g, local_bits);
  chunk_kernel<true><<<grid_for(1ull << n_local, 4), kBlock, 0, s>>>(const_cast<double2*>(amps),
                                                                       n_local, L, dst);
  return cudaGetLastError();
}

cudaError_t launch_unpack_chunks(double2* amps, int n_local, int g, const int* local_bits,
                                 const double2* src, cudaStream_t s) {
  BitList L = make_bits(g, local_bits);
  chunk_kernel<false><<<grid_for(1ull << n_local, 4), kBlock, 0, s>>>(amps, n_local, L,
                                                                        const_cast<double2*>(src));
  return cudaGetLastError();
}

}  // namespace qb
