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
#include <string.h>

#include "qaoa_common.cuh"
#include "qaoa_sweep.h"

namespace qb {

constexpr int kTileBits = 12;
constexpr int kTile = 1 << kTileBits;
constexpr int kThreads = 256;
constexpr int kRegs = 16;
// Shared-memory slot of tile index t: one 16-byte pad after every 16 slots, so
// register r of every mapping sits at a compile-time offset from a per-thread
// base (M2: +272 r, M0: +r, M1: +17 r) and every 8-lane phase of a 128-bit
// access hits 8 distinct 16-byte bank groups.
constexpr int kSlots = kTile + kTile / 16;
__host__ __device__ constexpr int slot(int t) { return t + (t >> 4); }

// Tile index of register r of thread tid in mapping M.  M3 / M4 are M2 / M1
// after lane bit 3 and register bit 0 traded places (transpose_lane3): register
// bit 0 then holds tile bit 3 and lane bit 3 holds tile bit 8 (M3) / 4 (M4).
template <int M>
__host__ __device__ constexpr int tile_index(int tid, int r) {
  return M == 2 ? (tid | (r << 8))
       : M == 0 ? ((tid << 4) | r)
       : M == 1 ? ((tid & 15) | ((tid >> 4) << 8) | (r << 4))
       : M == 3 ? ((tid & 0xF7) | (((tid >> 3) & 1) << 8) | ((r & 1) << 3) | ((r >> 1) << 9))
                : ((tid & 7) | (((tid >> 3) & 1) << 4) | ((tid >> 4) << 8) | ((r & 1) << 3) |
                   ((r >> 1) << 5));
}
template <int M>
__host__ __device__ constexpr int group_of() {
  return M == 2 ? 2 : (M == 0 ? 0 : 1);
}

// Physical offset of tile index t for carried-bit count C and high range at q.
template <int C>
__device__ __forceinline__ uint64_t tile_off(int t, uint64_t Q /* = 1 << q */) {
  if (C >= 12) return (uint64_t)t;
  return (uint64_t)(t & ((1 << C) - 1)) + (uint64_t)(t >> C) * Q;
}
template <int C>
__device__ __forceinline__ int tile_pos(int k, int q) {  // physical bit of tile bit k
  return (C >= 12 || k < C) ? k : q + (k - C);
}

// slot(thread part | register part) = slot(thread part) + slot(register part)
// for every mapping (their low four bits never carry), so register offsets are
// compile-time constants.
template <int M>
__device__ __forceinline__ void smem_store(double2* buf, int sb, const double2 (&v)[kRegs]) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) buf[sb + slot(tile_index<M>(0, r))] = v[r];
}
template <int M>
__device__ __forceinline__ void smem_load(const double2* buf, int sb, double2 (&v)[kRegs]) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) v[r] = buf[sb + slot(tile_index<M>(0, r))];
}

struct ThreadSlots {
  int s[5];
};

// Re-map registers from mapping A to mapping B through shared memory.  In a
// later exchange every thread writes (in mapping B) exactly the slots it read
// here, so one barrier per exchange suffices; the tile loop adds one barrier
// before the first write of the next tile.
template <int A, int B>
__device__ __forceinline__ void exchange(double2* buf, const ThreadSlots& ts, double2 (&v)[kRegs]) {
  smem_store<A>(buf, ts.s[A], v);
  __syncthreads();
  smem_load<B>(buf, ts.s[B], v);
}

// Trade lane bit 3 for register bit 0 inside each warp: the lane with lane bit
// 3 = 0 gives away its odd registers and receives the partner's even ones.  Half
// the data crosses lanes (one shuffle per moved word, vs two-way for a lane
// butterfly); afterwards tile bit 3 is a register bit (mappings M3 / M4).
__device__ __forceinline__ void transpose_lane3(double2 (&v)[kRegs]) {
  // The next exchange stores in the transposed mapping, i.e. to slots the
  // partner lane read in the last exchange: order those reads first (the data
  // dependency through the shuffles already does; this makes it explicit for
  // the memory model and for racecheck).
  __syncwarp();
  const bool hi = (threadIdx.x & 8) != 0;
#pragma unroll
  for (int r = 0; r < kRegs; r += 2) {
    const double2 snd = hi ? v[r] : v[r + 1];
    double2 rcv;
    rcv.x = __shfl_xor_sync(0xffffffffu, snd.x, 8);
    rcv.y = __shfl_xor_sync(0xffffffffu, snd.y, 8);
    if (hi) v[r] = rcv;
    else v[r + 1] = rcv;
  }
}

// Compile-time description of which tile bits a sweep mixes: bits C..11 (C<12)
// or all 12 (C == 12).
template <int C>
struct Act {
  static constexpr unsigned tile = C >= 12 ? 0xFFFu : ((0xFFFu >> C) << C);
  static constexpr unsigned g0 = tile & 15u;
  static constexpr unsigned g1 = (tile >> 4) & 15u;
  static constexpr unsigned g2 = (tile >> 8) & 15u;
  // a lone active bit 3 in group 0 is handled by lane shuffles (lane bit 3 in M2 and M1)
  static constexpr bool g0_shfl = (g0 == 8u);
  static constexpr bool g0_xchg = g0 != 0 && !g0_shfl;
};

struct TileCtx {
  uint64_t base;           // physical index of tile element 0 (tile bits zero), without x_hi
  uint64_t tb0, tb1, tb2;  // thread base offsets per mapping
};

// Per-tile cut-count basis, computed once per CTA by warp 0 (lane-parallel over
// nodes).  h = true index of tile element 0 with all tile bits cleared
// (x_hi ^ cmask ^ base, see GraphDev::cmask); K = C(h); per tile node k,
// d[k] = deg(k) - 2 popc(adj[k] & h) (change of C when node k alone is set);
// adjl[k] = tile-local neighbour mask (12 bits); tmask = cmask's tile bits (the
// true tile bits of tile index t are t ^ tmask).
struct CutBasis {
  int K;
  int tmask;
  int d[12];
  int adjl[12];
};

template <bool WIDE, int C>
__device__ __forceinline__ void cut_basis(const SweepArgs& a, uint64_t base, int q, CutBasis* cb) {
  const uint64_t tile_phys = (C >= 12) ? 0xFFFull
                                       : (((1ull << C) - 1ull) | (((1ull << (12 - C)) - 1ull) << q));
  const uint64_t h = (a.g.x_hi ^ a.g.cmask ^ base) & ~tile_phys;
  const int lane = threadIdx.x & 31;
  int part = 0;
  for (int i = lane; i < a.g.n_nodes; i += 32) {
    const uint64_t b = 0ull - ((h >> i) & 1ull);
    part += __popcll(a.g.rm[i] & (b ^ h));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  const uint64_t cm = a.g.cmask;
  const int tm = (int)((C >= 12) ? (cm & 0xFFFull)
                                 : ((cm & ((1ull << C) - 1ull)) |
                                    (((cm >> q) & ((1ull << (12 - C)) - 1ull)) << C)));
  if (lane < 12) {
    const int p = tile_pos<C>(lane, q);
    const uint64_t m = a.g.adj[p];
    cb->d[lane] = __popcll(m) - 2 * __popcll(m & h);
    const uint32_t lo = (uint32_t)(m & ((C >= 12) ? 0xFFFull : ((1ull << C) - 1ull)));
    const uint32_t hi = (C >= 12) ? 0u : (uint32_t)((m >> q) & ((1ull << (12 - C)) - 1ull)) << C;
    cb->adjl[lane] = (int)(lo | hi);
  }
  if (lane == 0) {
    cb->K = part;
    cb->tmask = tm;
  }
}

// C(x) for the 16 registers of mapping M.  With T = true tile bits of the
// thread's register-0 element: C(h | T) = K + sum_{k in T} (d[k] - popc(adjl[k] & T));
// flipping register node j changes C by s_j (d[j] - 2 popc(adjl[j] & T)) with
// s_j = -1 if bit j of T is set, and each edge between two flipped nodes j, k
// adds -2 s_j s_k.  Exact integer arithmetic.
template <int M>
__device__ __forceinline__ void cut16(const CutBasis* cb, int (&c)[16]) {
  const int T = tile_index<M>(threadIdx.x, 0) ^ cb->tmask;
  constexpr int g = group_of<M>();
  int c0 = cb->K;
#pragma unroll
  for (int k = 0; k < 12; ++k)
    if ((T >> k) & 1) c0 += cb->d[k] - __popc(cb->adjl[k] & T);
  int d[4], al[4], sg[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    al[j] = cb->adjl[4 * g + j];
    sg[j] = ((T >> (4 * g + j)) & 1) ? -1 : 1;
    d[j] = sg[j] * (cb->d[4 * g + j] - 2 * __popc(al[j] & T));
  }
  const int a01 = 2 * sg[0] * sg[1] * ((al[0] >> (4 * g + 1)) & 1);
  const int a02 = 2 * sg[0] * sg[2] * ((al[0] >> (4 * g + 2)) & 1);
  const int a03 = 2 * sg[0] * sg[3] * ((al[0] >> (4 * g + 3)) & 1);
  const int a12 = 2 * sg[1] * sg[2] * ((al[1] >> (4 * g + 2)) & 1);
  const int a13 = 2 * sg[1] * sg[3] * ((al[1] >> (4 * g + 3)) & 1);
  const int a23 = 2 * sg[2] * sg[3] * ((al[2] >> (4 * g + 3)) & 1);
  c[0] = c0;
  c[1] = c0 + d[0];
  c[2] = c0 + d[1];
  c[3] = c[1] + d[1] - a01;
  c[4] = c0 + d[2];
  c[5] = c[1] + d[2] - a02;
  c[6] = c[2] + d[2] - a12;
  c[7] = c[3] + d[2] - a02 - a12;
  c[8] = c0 + d[3];
  c[9] = c[1] + d[3] - a03;
  c[10] = c[2] + d[3] - a13;
  c[11] = c[3] + d[3] - a03 - a13;
  c[12] = c[4] + d[3] - a23;
  c[13] = c[5] + d[3] - a03 - a23;
  c[14] = c[6] + d[3] - a13 - a23;
  c[15] = c[7] + d[3] - a03 - a13 - a23;
}

// amp *= table_even[E - C(x)] (table_even[k] = phase_table[2k]; reference
// cost.py:168-172 indexes table[(E - 2C) + E]).
template <int M>
__device__ __forceinline__ void apply_cost(double2 (&v)[kRegs], const CutBasis* cb,
                                           const double2* __restrict__ tab, int e) {
  int c[16];
  cut16<M>(cb, c);
#pragma unroll
  for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], __ldg(tab + (e - c[r])));
}

template <int M>
__device__ __forceinline__ double expect_acc(const double2 (&v)[kRegs], const CutBasis* cb) {
  int c[16];
  cut16<M>(cb, c);
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) acc += (v[r].x * v[r].x + v[r].y * v[r].y) * (double)c[r];
  return acc;
}

// RX(stage) on register bits MASK: exact (reference rounding) or the factored
// fast form mine - i t other (form-2 levels run as form 1 with t = -k plus a
// global bit complement tracked on the host; see qaoa_capi.cu).
template <unsigned MASK, bool EXACT>
__device__ __forceinline__ void rx_regs2(double2 (&v)[kRegs], double c_or_t, double s) {
#pragma unroll
  for (int K = 0; K < 4; ++K) {
    if (!((MASK >> K) & 1)) continue;
#pragma unroll
    for (int r = 0; r < kRegs; ++r) {
      if (r & (1 << K)) continue;
      if (EXACT) rx_exact(v[r], v[r | (1 << K)], c_or_t, s);
      else rx_form1(v[r], v[r | (1 << K)], c_or_t);
    }
  }
}

template <int C, int M>
__device__ __forceinline__ void store_tile(double2* __restrict__ amps, const TileCtx& tc,
                                           uint64_t Q, const double2 (&v)[kRegs]) {
  const uint64_t tb = M == 2 ? tc.tb2 : tc.tb1;
  double2* dst = amps + tc.base + tb;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) __stcs(dst + tile_off<C>(tile_index<M>(0, r), Q), v[r]);
}

// FLOW 0: exact (reference order: tile bits ascending, reference rounding)
// FLOW 1: fast, one RX stage
// FLOW 2: fast, RX stage -> cost -> RX stage (two levels in one sweep)
// One 4096-amplitude tile per CTA; two CTAs per SM keep one tile's loads in
// flight while the other computes (a persistent grid measured slower).
template <bool WIDE, int C, int FLOW>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(const SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);  // kSlots exchange slots
  __shared__ CutBasis cb;
  __shared__ double red_scratch[kThreads / 32];
  using A = Act<C>;
  constexpr bool EX = FLOW == 0;

  const uint32_t flags = a.flags;
  const int tid = threadIdx.x;
  const int q = a.q;
  const uint64_t Q = 1ull << (C >= 12 ? 0 : q);
  const uint64_t tile = blockIdx.x;
  TileCtx tc;
  {
    const int low_bits = C >= 12 ? 0 : q - C;  // non-tile ranges [C, q) and [q + 12 - C, n)
    tc.base = C >= 12 ? (tile << 12)
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
    const double2* src = amps + tc.base + tc.tb2;
#pragma unroll
    for (int r = 0; r < kRegs; ++r) v[r] = __ldcs(src + tile_off<C>(tile_index<2>(0, r), Q));
  }
  const bool need_cut = flags & (kPreCost | kMidCost | kExpect);
  if (need_cut) {
    if (tid < 32) cut_basis<WIDE, C>(a, tc.base, q, &cb);
    __syncthreads();
  }
  const int e = a.g.tot_edge;
  const double r1a = a.rx1.a, r1b = a.rx1.b, r2a = a.rx2.a;
  double acc = 0.0;

  if (FLOW == 0) {
    // ---- exact: cost first (level start), then tile bits in increasing order
    if (flags & kPreCost) apply_cost<2>(v, &cb, a.table, e);
    if (C >= 12) {
      exchange<2, 0>(buf, ts, v);
      rx_regs2<A::g0, true>(v, r1a, r1b);
      exchange<0, 1>(buf, ts, v);
      rx_regs2<A::g1, true>(v, r1a, r1b);
      exchange<1, 2>(buf, ts, v);
    } else if (A::g0_shfl) {  // tile bit 3 via the lane/register transpose
      transpose_lane3(v);
      rx_regs2<1u, true>(v, r1a, r1b);
      exchange<3, 1>(buf, ts, v);
      rx_regs2<A::g1, true>(v, r1a, r1b);
      exchange<1, 2>(buf, ts, v);
    } else {
      if (A::g1) {
        exchange<2, 1>(buf, ts, v);
        rx_regs2<A::g1, true>(v, r1a, r1b);
        exchange<1, 2>(buf, ts, v);
      }
    }
    rx_regs2<A::g2, true>(v, r1a, r1b);
    if (flags & kExpect) acc = expect_acc<2>(v, &cb);
    store_tile<C, 2>(amps, tc, Q, v);
  } else if (C >= 12) {
    // ---- fast, low set: G2 (loaded), G0, G1 [, cost, G1, G0, G2]
    if (flags & kPreCost) apply_cost<2>(v, &cb, a.table, e);
    rx_regs2<A::g2, false>(v, r1a, 0.0);
    exchange<2, 0>(buf, ts, v);
    rx_regs2<A::g0, false>(v, r1a, 0.0);
    exchange<0, 1>(buf, ts, v);
    rx_regs2<A::g1, false>(v, r1a, 0.0);
    if (FLOW == 2) {
      apply_cost<1>(v, &cb, a.table2, e);
      rx_regs2<A::g1, false>(v, r2a, 0.0);
      exchange<1, 0>(buf, ts, v);
      rx_regs2<A::g0, false>(v, r2a, 0.0);
      exchange<0, 2>(buf, ts, v);
      rx_regs2<A::g2, false>(v, r2a, 0.0);
      if (flags & kScale) {
#pragma unroll
        for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], a.scale);
      }
      if (flags & kExpect) acc = expect_acc<2>(v, &cb);
      store_tile<C, 2>(amps, tc, Q, v);
    } else {
      if (flags & kScale) {
#pragma unroll
        for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], a.scale);
      }
      if (flags & kExpect) acc = expect_acc<1>(v, &cb);
      store_tile<C, 1>(amps, tc, Q, v);
    }
  } else {
    // ---- fast, high set: G2 (+ tile bit 3), G1 [, cost, G1 (+ tile bit 3), G2]
    if (flags & kPreCost) apply_cost<2>(v, &cb, a.table, e);
    rx_regs2<A::g2, false>(v, r1a, 0.0);
    if (A::g0_shfl) {  // C = 3: tile bit 3 traded into register bit 0 (M2 -> M3)
      transpose_lane3(v);
      rx_regs2<1u, false>(v, r1a, 0.0);
      exchange<3, 1>(buf, ts, v);
      rx_regs2<A::g1, false>(v, r1a, 0.0);
      if (FLOW == 2) {
        apply_cost<1>(v, &cb, a.table2, e);
        rx_regs2<A::g1, false>(v, r2a, 0.0);
        transpose_lane3(v);  // M1 -> M4
        rx_regs2<1u, false>(v, r2a, 0.0);
        exchange<4, 2>(buf, ts, v);
        rx_regs2<A::g2, false>(v, r2a, 0.0);
      }
    } else if (A::g1) {
      exchange<2, 1>(buf, ts, v);
      rx_regs2<A::g1, false>(v, r1a, 0.0);
      if (FLOW == 2) {
        apply_cost<1>(v, &cb, a.table2, e);
        rx_regs2<A::g1, false>(v, r2a, 0.0);
        exchange<1, 2>(buf, ts, v);
        rx_regs2<A::g2, false>(v, r2a, 0.0);
      }
    } else if (FLOW == 2) {
      apply_cost<2>(v, &cb, a.table2, e);
      rx_regs2<A::g2, false>(v, r2a, 0.0);
    }
    constexpr int last = (A::g1 && FLOW == 1) ? 1 : 2;
    if (flags & kScale) {
#pragma unroll
      for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], a.scale);
    }
    if (flags & kExpect) acc = expect_acc<last>(v, &cb);
    store_tile<C, last>(amps, tc, Q, v);
  }
  if (flags & kExpect) {
    const double t = block_sum<kThreads>(acc, red_scratch);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = t;
  }
}

// ---- K1: the cut-table builder (CompressedCostPlan.cut_counts, cost.py:88-99)
// One CTA per 4096 consecutive states (the C = 12 tile): warp 0 builds the cut
// basis of the tile, every thread derives the exact counts of 16 consecutive
// states (mapping M0: registers = tile bits 0..3) and writes them as one
// 16-byte (uint8) or two 16-byte (uint16) streaming stores -- 512 contiguous
// bytes per warp instruction.
template <bool WIDE, typename T>
__global__ void __launch_bounds__(kThreads) cut_table_tile_kernel(T* __restrict__ table,
                                                                  const SweepArgs a) {
  __shared__ CutBasis cb;
  const uint64_t base = (uint64_t)blockIdx.x << 12;
  if (threadIdx.x < 32) cut_basis<WIDE, 12>(a, base, 0, &cb);
  __syncthreads();
  int c[16];
  cut16<0>(&cb, c);
  const uint64_t first = base + (uint64_t)tile_index<0>(threadIdx.x, 0);  // 16 consecutive states
  if (sizeof(T) == 1) {
    uint4 o;
    o.x = (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16) | ((uint32_t)c[3] << 24);
    o.y = (uint32_t)c[4] | ((uint32_t)c[5] << 8) | ((uint32_t)c[6] << 16) | ((uint32_t)c[7] << 24);
    o.z = (uint32_t)c[8] | ((uint32_t)c[9] << 8) | ((uint32_t)c[10] << 16) | ((uint32_t)c[11] << 24);
    o.w = (uint32_t)c[12] | ((uint32_t)c[13] << 8) | ((uint32_t)c[14] << 16) | ((uint32_t)c[15] << 24);
    __stcs(reinterpret_cast<uint4*>(table + first), o);
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
    __stcs(reinterpret_cast<uint4*>(table + first), o0);
    __stcs(reinterpret_cast<uint4*>(table + first) + 1, o1);
  }
}

cudaError_t launch_cut_table_tiles(void* table, int bytes_per, int n_local, const GraphDev& g,
                                   cudaStream_t s) {
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.g = g;
  a.g.cmask = 0;
  const unsigned grid = 1u << (n_local - 12);
  const bool wide = g.n_nodes > 32;
  if (bytes_per == 1) {
    if (wide) cut_table_tile_kernel<true, uint8_t><<<grid, kThreads, 0, s>>>((uint8_t*)table, a);
    else cut_table_tile_kernel<false, uint8_t><<<grid, kThreads, 0, s>>>((uint8_t*)table, a);
  } else {
    if (wide) cut_table_tile_kernel<true, uint16_t><<<grid, kThreads, 0, s>>>((uint16_t*)table, a);
    else cut_table_tile_kernel<false, uint16_t><<<grid, kThreads, 0, s>>>((uint16_t*)table, a);
  }
  return cudaGetLastError();
}

size_t sweep_smem_bytes(int) { return (size_t)kSlots * sizeof(double2); }

template <bool WIDE, int C, int FLOW>
static cudaError_t launch_one(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<WIDE, C, FLOW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  sweep_kernel<WIDE, C, FLOW><<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool WIDE, int C>
static cudaError_t launch_c(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
  if (a.flags & kExact) return launch_one<WIDE, C, 0>(a, grid, smem, s);
  if (a.flags & kStage2) return launch_one<WIDE, C, 2>(a, grid, smem, s);
  return launch_one<WIDE, C, 1>(a, grid, smem, s);
}

template <bool WIDE>
static cudaError_t launch_w(const SweepArgs& a, int grid, size_t smem, cudaStream_t s) {
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

cudaError_t launch_sweep(const SweepArgs& a, int grid, cudaStream_t stream) {
  const int n_tables = ((a.flags & kPreCost) ? 1 : 0) + ((a.flags & kStage2) ? 1 : 0);
  const size_t smem = sweep_smem_bytes(n_tables * a.table_len);
  return a.g.n_nodes > 32 ? launch_w<true>(a, grid, smem, stream)
                          : launch_w<false>(a, grid, smem, stream);
}

int sweep_max_grid(int) {
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  const size_t smem = sweep_smem_bytes(0);
  cudaFuncSetAttribute(sweep_kernel<false, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<false, 3, 2>, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

}  // namespace qb
