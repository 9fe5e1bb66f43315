// qaoa_sweep.cu -- the fused cost + mixer sweep kernel (the hot path).
//
// One launch = one HBM round trip of the state (read 16 B + write 16 B per
// amplitude; launch-control sweeps only write).  The state is cut into tiles of
// 2^12 amplitudes.  A tile's 12 "tile bits" are two contiguous physical ranges:
// bits 0..C-1 (carried in every tile so each HBM access is a run of 2^C
// amplitudes, C >= 3 -> >= 128 B) and bits q..q+11-C (the qubits mixed by this
// sweep).  The low sweep has C = 12 (tile = 4096 consecutive amplitudes).
//
// A CTA of 256 threads (two per SM) holds one tile in registers, 16 amplitudes
// per thread, and re-maps it through shared memory between three register
// groups of four tile bits:
//   M2: registers = tile bits 8..11, threads = tile bits 0..7        (HBM load/store)
//   M0: registers = tile bits 0..3,  threads = tile bits 4..11
//   M1: registers = tile bits 4..7,  threads = tile bits 0..3, 8..11 (HBM store)
// RX butterflies on register bits are register-local; tile bit 3 is lane bit 3
// in both M2 and M1, so a lone mixed bit there (C = 3) is traded into a
// register bit by a half-data warp-shuffle transpose instead of an extra
// shared-memory pass.  The diagonal cost phase (lookup of
// exp(-i gamma (E - 2C)/2) by the integer cut count C(x), recomputed from the
// row masks -- the cut table is never read from HBM), the fast-mode scale and
// the <C> reduction are applied on the registers between / after the stages.
//
// Reference path replaced (pkg/src/qaoa_maxcut/):
//   cost layer  apply_cost_bitwise  cost.py:162-176 (+ cut_counts :88-99)
//   mixer layer apply_mixer_layer   circuit.py:89-94 -> apply_rx state.py:110-128
//   init        init_uniform        circuit.py:42-48
//   expectation                     circuit.py:116-121, graph.py:144-151
#include <stdlib.h>
#include <string.h>

#include "qaoa_common.cuh"
#include "qaoa_sweep.h"
#include "qaoa_tile.cuh"

namespace qb {

// FLOW 0: exact (reference order: tile bits ascending, reference rounding)
// FLOW 1: fast, one RX stage
// FLOW 2: fast, RX stage -> cost -> RX stage (two levels in one sweep)
// One 4096-amplitude tile per CTA; two CTAs per SM keep one tile's loads in
// flight while the other computes (a persistent grid measured slower).
// WGT: weighted cost (fast flows only; wbasis / apply_wcost in qaoa_tile.cuh).
//
// MIR (symmetric half state): a tile that contains the virtual top qubit.
// The half state of an N = n + 1 qubit state stores psi(v) for v_n = 0
// (psi(v) == psi(~v)), so virtual index v lives at fold(v) = v_n ? ~v : v (n
// bits).  Tile bit 11 is the virtual bit n; tile bits 0..10 give the virtual
// offset o(t) from the tile's virtual base, and fold puts the t >= 2048 half
// at (2^n - 1) - o(t & 2047), i.e. the mirrored runs read backwards.  Two
// geometries, both standard tiles in virtual coordinates (so the cut basis
// and every butterfly are the ordinary ones):
//  * fast schedule, the "mirror low set" (C = 12 flows, cut geometry (11, n)):
//    qubits 0..10 and the virtual one; tile u is stored block u (2048
//    amplitudes, ascending) plus block 2^(n-11) - 1 - u (backwards), two
//    contiguous 32 KB runs; the high sets take qubits 11..n-1;
//  * exact schedule, the folded top set (exact flow, geometry (C, q) with
//    q + 11 - C = n): the top set's qubits then the virtual one, in the
//    reference's increasing order (qubit N-1 last).
// Only tiles whose top non-tile bit is 0 are visited (u < 2^(n-12)): the other
// half are the same stored amplitudes.
template <int C, int M>
__device__ __forceinline__ void mirror_ptrs(double2* amps, uint64_t base, uint64_t Q, uint64_t mask_n,
                                            int tid, int sk, double2* (&ptr)[kRegs]) {
  const int tp = tile_index<M>(tid, 0);
#pragma unroll
  for (int p = 0; p < kRegs; ++p) {
    // skewed layout: physical register p holds logical p ^ sk
    const int t = tp | (sk ? tile_index<M>(0, p ^ 1) : tile_index<M>(0, p));  // disjoint bit parts
    const int lo = t & 2047;
    const uint64_t o = base + (C >= 12 ? (uint64_t)lo : tile_off<C>(lo, Q));
    ptr[p] = amps + ((t & 2048) ? mask_n - o : o);
  }
}

template <bool WIDE, int C, int FLOW, bool WGT = false, bool MIR = false>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(const __grid_constant__ SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // kSlots exchange slots
  __shared__ CutBasis cb;
  __shared__ WBasis wb[WGT ? 2 : 1];
  __shared__ WCutBasis wcb[1];
  __shared__ double red_scratch[kThreads / 32];
  using A = Act<C>;
  // skewed register layout for the C = 3 flows (select-free transposes; the
  // exact butterfly is symmetric bit for bit too: its sums commute)
  const int sk = A::g0_shfl ? lane_skew() : 0;

  const uint32_t flags = a.flags;
  const int tid = threadIdx.x;
  const int q = a.q;
  const uint64_t Q = 1ull << (C >= 12 ? 0 : q);
  // out-of-place swap sweeps visit tiles in an order whose consecutive blocks
  // vary the low bits of BOTH swapped ranges, so the tiles in flight share a
  // few DRAM pages on the read side and on the write side
  auto visit = [&](uint64_t b) -> uint64_t {
    if (C < 12 || !a.out) return b;
    const int k = a.sw_m / 2 < 4 ? a.sw_m / 2 : 4;
    return swap_bit_ranges(b, k, a.sw_hi - (MIR ? 11 : 12), k);  // tile number = index >> (MIR ? 11 : 12)
  };
  const uint64_t tile = visit((uint64_t)a.tile_lo + blockIdx.x);
  TileCtx tc;
  {
    const int low_bits = C >= 12 ? 0 : q - C;  // non-tile ranges [C, q) and [q + 12 - C, n)
    tc.base = (MIR && C >= 12) ? (tile << 11)  // virtual index of tile element 0
                  : C >= 12 ? (tile << 12)
                  : (((tile & ((1ull << low_bits) - 1ull)) << C) | ((tile >> low_bits) << (q + 12 - C)));
  }
  tc.tb2 = tile_off<C>(tile_index<2>(tid, 0), Q);
  tc.tb1 = tile_off<C>(tile_index<1>(tid, 0), Q);
  ThreadSlots ts;
  ts.s[0] = slot(tile_index<0>(tid, 0));
  ts.s[1] = slot(tile_index<1>(tid, 0));
  ts.s[2] = slot(tile_index<2>(tid, 0));
  ts.s[3] = slot(tile_index<3>(tid, 0));
  ts.s[4] = slot(tile_index<4>(tid, 0));
  double2* __restrict__ amps = a.amps;

  double2 v[kRegs];
  if (flags & kGen) {
#pragma unroll
    for (int r = 0; r < kRegs; ++r) v[r] = a.gen;
  } else {
    const uint64_t pf_b = (uint64_t)a.tile_lo + blockIdx.x + a.pf_dist;
    if (a.pf_dist > 0 && pf_b < (uint64_t)(a.tile_lo + (a.tile_cnt ? a.tile_cnt : a.ntiles))) {
      const uint64_t pf_tile = visit(pf_b);
      if (MIR && C < 12) {
        // (exact folded top set: no prefetch)
      } else if (MIR) {
        if (tid < 2) {
          const uint64_t blk = tid ? 2ull * (uint64_t)a.ntiles - 1ull - pf_tile : pf_tile;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(amps + (blk << 11)), "r"(32768u)
                       : "memory");
        }
      } else if (!a.pf_tensor) {
        prefetch_tile_l2<C, kThreads>(amps, tile_base<C>(pf_tile, q), Q, tid);
      } else if (tid == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int c[5];
          half_coords<C>(a, pf_tile, h, c);
          asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                           reinterpret_cast<uint64_t>(&a.map)),
                       "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
                       : "memory");
        }
      }
    }
    if (MIR) {
      double2* ptr[kRegs];
      mirror_ptrs<C, 2>(amps, tc.base, Q, ((uint64_t)a.ntiles << 12) - 1ull, tid, sk, ptr);
#pragma unroll
      for (int r = 0; r < kRegs; ++r) v[r] = ld_tile(ptr[r]);
    } else {
      walk_tile<C, 2>(amps + tc.base + tc.tb2, Q, sk, [&](int r, double2* ptr) { v[r] = ld_tile(ptr); });
    }
  }
  const bool need_cut = flags & (kPreCost | kMidCost | kExpect);
  if (need_cut) {
    if (tid < 32) {
      constexpr int GC = (MIR && C >= 12) ? 11 : C;  // cut geometry (mirror low set: (11, n))
      if (WGT) {
        if (flags & kPreCost) wbasis<GC>(a, tc.base, q, a.wu1, &wb[0]);
        if (flags & kMidCost) wbasis<GC>(a, tc.base, q, a.wu2, &wb[WGT ? 1 : 0]);
      }
      if (WGT && (flags & kExpect)) wcut_basis<GC>(a, tc.base, q, &wcb[0]);
      // the mirror low set's cut geometry is (11, n) (a.q = n)
      if (!WGT) cut_basis<WIDE, (MIR && C >= 12) ? 11 : C>(a, tc.base, q, &cb);
    }
    // The basis is first read after the fast flow's first register exchange
    // (whose barrier then publishes it) unless a cost step precedes every
    // exchange: warp 0 builds it while the other warps run the first RX stage.
    constexpr bool xchg_first = FLOW != 0 && (C >= 12 || Act<C>::g0_shfl || Act<C>::g1 != 0);
    if (!xchg_first || (flags & kPreCost)) __syncthreads();
  }
  const int e = a.g.tot_edge;
  const double r1a = a.rx1.a, r1b = a.rx1.b;
  double acc = 0.0;

  if (FLOW == 0) {
    // ---- exact: cost first (level start), then tile bits in increasing order
    if (flags & kPreCost) apply_cost<2>(v, &cb, a.table, e, tid, sk);
    if (C >= 12) {
      exchange<2, 0>(buf, ts, v);
      rx_regs2<A::g0, true>(v, r1a, r1b);
      exchange<0, 1>(buf, ts, v);
      rx_regs2<A::g1, true>(v, r1a, r1b);
      exchange<1, 2>(buf, ts, v);
    } else if (A::g0_shfl) {  // tile bit 3 via the lane/register transpose
      transpose_lane3_sk(v);
      rx_regs2<1u, true>(v, r1a, r1b);
      exchange<3, 1>(buf, ts, v, sk);
      rx_regs2<A::g1, true>(v, r1a, r1b);
      exchange<1, 2>(buf, ts, v, sk);
    } else {
      if (A::g1) {
        exchange<2, 1>(buf, ts, v);
        rx_regs2<A::g1, true>(v, r1a, r1b);
        exchange<1, 2>(buf, ts, v);
      }
    }
    rx_regs2<A::g2, true>(v, r1a, r1b);
    if (flags & kExpect) acc = expect_acc<2>(v, &cb, tid, sk);
    if (MIR) {
      if (!(flags & kNoStore)) {
        double2* ptr[kRegs];
        mirror_ptrs<C, 2>(amps, tc.base, Q, ((uint64_t)a.ntiles << 12) - 1ull, tid, sk, ptr);
#pragma unroll
        for (int r = 0; r < kRegs; ++r) __stcs(ptr[r], v[r]);
      }
    } else {
      store_tile<C, 2>(amps, tc, Q, v, flags, sk);
    }
  } else {
    fast_tile<C, FLOW, WGT>(v, a, &cb, wb, tid, sk, [&](auto from, auto to) {
      exchange<decltype(from)::value, decltype(to)::value>(buf, ts, v, sk);
    });
    constexpr int last = fast_last<C, FLOW>();
    if (flags & kExpect)
      acc = WGT ? expect_wacc<last>(v, &wcb[0], a.wc, tid, sk) : expect_acc<last>(v, &cb, tid, sk);
    if (MIR) {
      if (!(flags & kNoStore)) {
        // out of place into the swapped layout: block u -> swap(u), and the
        // complement commutes with the bit-range swap, so ~u -> ~swap(u)
        const uint64_t b = a.out ? swap_bit_ranges(tc.base, a.sw_lo, a.sw_hi, a.sw_m) : tc.base;
        double2* ptr[kRegs];
        mirror_ptrs<C, last>(a.out ? a.out : amps, b, Q, ((uint64_t)a.ntiles << 12) - 1ull, tid, sk, ptr);
#pragma unroll
        for (int r = 0; r < kRegs; ++r) __stcs(ptr[r], v[r]);
      }
    } else if (C >= 12 && a.out) {  // out of place into the swapped qubit layout
      TileCtx to = tc;
      to.base = swap_bit_ranges(tc.base, a.sw_lo, a.sw_hi, a.sw_m);
      store_tile<C, last>(a.out, to, Q, v, flags, sk);
    } else {
      store_tile<C, last>(amps, tc, Q, v, flags, sk);
    }
  }
  if (flags & kExpect) {
    const double t = block_sum<kThreads>(acc, red_scratch);
    if (threadIdx.x == 0) a.partials[tile] = t;
  }
}

// Tile-internal phase table of one weighted cost level (see apply_wcost).
__global__ void wq_table_kernel(double2* __restrict__ out, const int2* __restrict__ wedge,
                                const double2* __restrict__ wu, int wm, int carry, int q,
                                double2 scale) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kTile) return;
  auto tile_bit = [&](int p) -> int {  // tile bit of physical node p, or -1
    if (carry >= 12) return p < 12 ? p : -1;
    if (p < carry) return p;
    if (p >= q && p < q + 12 - carry) return carry + p - q;
    return -1;
  };
  double2 f = scale;
  for (int e = 0; e < wm; ++e) {
    const int2 ij = wedge[e];
    const int ki = tile_bit(ij.x), kj = tile_bit(ij.y);
    if (ki < 0 || kj < 0) continue;
    const double2 u = wu[e];
    f = cmul_u(f, (((t >> ki) ^ (t >> kj)) & 1) ? conj2(u) : u);
  }
  out[t] = f;
}

cudaError_t launch_wq_table(double2* q_out, const int2* wedge, const double2* wu, int wm, int carry,
                            int q, double2 scale, cudaStream_t s) {
  wq_table_kernel<<<kTile / 256, 256, 0, s>>>(q_out, wedge, wu, wm, carry, q, scale);
  return cudaGetLastError();
}

__global__ void wc_table_kernel(double* __restrict__ out, const int2* __restrict__ wedge,
                                const double* __restrict__ w, int wm, int carry, int q) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kTile) return;
  auto tile_bit = [&](int p) -> int {
    if (carry >= 12) return p < 12 ? p : -1;
    if (p < carry) return p;
    if (p >= q && p < q + 12 - carry) return carry + p - q;
    return -1;
  };
  double c = 0.0;
  for (int e = 0; e < wm; ++e) {
    const int2 ij = wedge[e];
    const int ki = tile_bit(ij.x), kj = tile_bit(ij.y);
    if (ki < 0 || kj < 0) continue;
    if (((t >> ki) ^ (t >> kj)) & 1) c += w[e];
  }
  out[t] = c;
}

cudaError_t launch_wc_table(double* c_out, const int2* wedge, const double* w, int wm, int carry, int q,
                            cudaStream_t s) {
  wc_table_kernel<<<kTile / 256, 256, 0, s>>>(c_out, wedge, w, wm, carry, q);
  return cudaGetLastError();
}

// ---- launch-control helpers (launch_gen_aux) ----------------------------------
// One warp per tile: the same cut basis the sweep's warp 0 would build.
template <bool WIDE, int C>
__global__ void basis_table_kernel(const __grid_constant__ SweepArgs a, CutBasis* out, int64_t cnt) {
  const int64_t w = (int64_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
  if (w >= cnt) return;  // warp-uniform
  const uint64_t tile = (uint64_t)a.tile_lo + (uint64_t)w;
  cut_basis<WIDE, C>(a, tile_base<C>(tile, a.q), a.q, out + tile);
}

__global__ void gen_table_kernel(double2* __restrict__ out, const double2* __restrict__ in, double2 gen,
                                 int len) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < len) out[k] = cmul_np(gen, in[k]);
}

template <bool WIDE, int C>
static void launch_basis_c(const SweepArgs& a, CutBasis* out, int64_t cnt, cudaStream_t s) {
  const int64_t threads = cnt * 32;
  basis_table_kernel<WIDE, C><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a, out, cnt);
}

template <bool WIDE>
static cudaError_t launch_basis_w(const SweepArgs& a, CutBasis* out, int64_t cnt, cudaStream_t s) {
  switch (a.carry) {
    case 3: launch_basis_c<WIDE, 3>(a, out, cnt, s); break;
    case 4: launch_basis_c<WIDE, 4>(a, out, cnt, s); break;
    case 5: launch_basis_c<WIDE, 5>(a, out, cnt, s); break;
    case 6: launch_basis_c<WIDE, 6>(a, out, cnt, s); break;
    case 7: launch_basis_c<WIDE, 7>(a, out, cnt, s); break;
    case 8: launch_basis_c<WIDE, 8>(a, out, cnt, s); break;
    case 9: launch_basis_c<WIDE, 9>(a, out, cnt, s); break;
    case 10: launch_basis_c<WIDE, 10>(a, out, cnt, s); break;
    case 12: launch_basis_c<WIDE, 12>(a, out, cnt, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_gen_aux(const SweepArgs& a, void* basis_out, double2* gen_table, cudaStream_t s) {
  static_assert(sizeof(CutBasis) == kBasisEntryBytes, "basis entry = 16 ints (the TMA kernel's stride)");
  if (!(a.flags & kGen) || !(a.flags & kPreCost) || !a.table || a.table_len < 1) return cudaErrorInvalidValue;
  const int64_t cnt = a.tile_cnt ? a.tile_cnt : a.ntiles;
  CutBasis* out = reinterpret_cast<CutBasis*>(basis_out);
  cudaError_t e = a.g.n_nodes > 32 ? launch_basis_w<true>(a, out, cnt, s) : launch_basis_w<false>(a, out, cnt, s);
  if (e != cudaSuccess) return e;
  gen_table_kernel<<<(a.table_len + 127) / 128, 128, 0, s>>>(gen_table, a.table, a.gen, a.table_len);
  return cudaGetLastError();
}

size_t sweep_smem_bytes(int) { return (size_t)kSlots * sizeof(double2); }

template <bool WIDE, int C, int FLOW, bool WGT = false, bool MIR = false>
static cudaError_t launch_one(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
  static unsigned long long configured = 0;  // per instantiation, bit d = device d done
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<WIDE, C, FLOW, WGT, MIR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  sweep_kernel<WIDE, C, FLOW, WGT, MIR><<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

// Tiles with the virtual top qubit of a symmetric half state (kMirror, see
// sweep_kernel): the fast mirror low set, or the exact folded top set.
template <bool WIDE>
static cudaError_t launch_mirror(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (a.ntiles < 1 || ((a.flags & kWeighted) && (a.flags & kExact))) return cudaErrorInvalidValue;
  if (a.flags & kExact) {
    if (a.out) return cudaErrorInvalidValue;
    switch (a.carry) {
      case 3: return launch_one<WIDE, 3, 0, false, true>(a, grid, smem, s);
      case 4: return launch_one<WIDE, 4, 0, false, true>(a, grid, smem, s);
      case 5: return launch_one<WIDE, 5, 0, false, true>(a, grid, smem, s);
      case 6: return launch_one<WIDE, 6, 0, false, true>(a, grid, smem, s);
      case 7: return launch_one<WIDE, 7, 0, false, true>(a, grid, smem, s);
      case 8: return launch_one<WIDE, 8, 0, false, true>(a, grid, smem, s);
      case 9: return launch_one<WIDE, 9, 0, false, true>(a, grid, smem, s);
      case 10: return launch_one<WIDE, 10, 0, false, true>(a, grid, smem, s);
      case 11: return launch_one<WIDE, 11, 0, false, true>(a, grid, smem, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (a.carry != 12) return cudaErrorInvalidValue;
  if (a.flags & kWeighted) {
    if (a.flags & kStage2) return launch_one<WIDE, 12, 2, true, true>(a, grid, smem, s);
    return launch_one<WIDE, 12, 1, true, true>(a, grid, smem, s);
  }
  if (a.flags & kStage2) return launch_one<WIDE, 12, 2, false, true>(a, grid, smem, s);
  return launch_one<WIDE, 12, 1, false, true>(a, grid, smem, s);
}

template <bool WIDE, int C>
static cudaError_t launch_c(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (a.flags & kExact) return launch_one<WIDE, C, 0>(a, grid, smem, s);
  if (a.flags & kWeighted) {
    if (a.flags & kStage2) return launch_one<WIDE, C, 2, true>(a, grid, smem, s);
    return launch_one<WIDE, C, 1, true>(a, grid, smem, s);
  }
  if (a.flags & kStage2) return launch_one<WIDE, C, 2>(a, grid, smem, s);
  return launch_one<WIDE, C, 1>(a, grid, smem, s);
}

template <bool WIDE>
static cudaError_t launch_w(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (a.flags & kMirror) return launch_mirror<WIDE>(a, grid, smem, s);
  switch (a.carry) {
    case 3: return launch_c<WIDE, 3>(a, grid, smem, s);
    case 4: return launch_c<WIDE, 4>(a, grid, smem, s);
    case 5: return launch_c<WIDE, 5>(a, grid, smem, s);
    case 6: return launch_c<WIDE, 6>(a, grid, smem, s);
    case 7: return launch_c<WIDE, 7>(a, grid, smem, s);
    case 8: return launch_c<WIDE, 8>(a, grid, smem, s);
    case 9: return launch_c<WIDE, 9>(a, grid, smem, s);
    case 10: return launch_c<WIDE, 10>(a, grid, smem, s);
    case 11: return launch_c<WIDE, 11>(a, grid, smem, s);
    case 12: return launch_c<WIDE, 12>(a, grid, smem, s);
    default: return cudaErrorInvalidValue;
  }
}

// L2 prefetch distance (tiles ahead) for the one-tile-per-CTA kernel: one wave
// of CTAs (2 per SM) ahead.  Measured on B200 (tools/sweep_probe.cu, N=30):
// the contiguous low set goes 5.33 -> 4.87 ms (7.05 TB/s); a strided set whose
// tile spans <= 256 MB (the TLB reach) gains ~6%, while the top set (tile span
// = the whole state, 512 pages per tile) loses ~35% -> no prefetch there.
// QAOA_PF_DIST overrides (0 disables).
static int pf_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("QAOA_PF_DIST");
    v = e ? atoi(e) : -1;
  }
  return v;
}

static int pf_distance(const SweepArgs& a) {
  if (a.flags & kGen) return 0;
  const int env = pf_env();
  if (env >= 0) return env;
  if (a.carry < 12) {
    const int span_bits = a.q + 12 - a.carry + 4;  // log2 bytes spanned by one tile
    if (span_bits > 28) return 0;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // out-of-place low-set sweeps: their writes allocate fresh L2 lines, and a
  // prefetch two waves ahead was partly evicted before use (+2% DRAM reads);
  // half a wave ahead measured best (S0 5.27 vs 5.35-5.41 ms, profiles/r06_swap.md)
  if (a.out) return sms / 2;
  return 2 * sms;
}

cudaError_t launch_sweep(const SweepArgs& a0, int grid, cudaStream_t stream) {
  if (sweep_uses_tma(a0)) return launch_sweep_tma(a0, stream);
  SweepArgs a = a0;
  if (a.tile_cnt) grid = (int)a.tile_cnt;
  if (a.pf_dist == 0) a.pf_dist = pf_distance(a);
  if (a.pf_dist > 0) {
    static int tens = -1;
    if (tens < 0) {
      const char* e = getenv("QAOA_PF_TENSOR");
      tens = e ? atoi(e) : 1;
    }
    a.pf_tensor = (a.flags & kMirror) ? 0 : tens;  // mirror tiles: two per-run bulk prefetches
    if (a.pf_tensor) {
      int n = 12;
      while ((1ll << (n - 12)) < a.ntiles) ++n;
      if (!make_tile_map(&a.map, a.amps, n, a.carry, a.q)) return cudaErrorInvalidValue;
    }
  }
  if (sweep32_selected(a)) return launch_sweep32(a, grid, stream);
  const int n_tables = ((a.flags & kPreCost) ? 1 : 0) + ((a.flags & kStage2) ? 1 : 0);
  const size_t smem = sweep_smem_bytes(n_tables * a.table_len);
  return a.g.n_nodes > 32 ? launch_w<true>(a, grid, smem, stream)
                          : launch_w<false>(a, grid, smem, stream);
}

}  // namespace qb
