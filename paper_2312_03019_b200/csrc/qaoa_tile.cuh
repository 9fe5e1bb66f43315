// qaoa_tile.cuh -- device building blocks of the fused sweep kernels: the
// 4096-amplitude tile geometry, the three register mappings and their
// shared-memory exchanges, the per-tile cut-count basis (C(x) recomputed from
// the row masks, bit-exact), the cost phase, the RX register butterflies and
// the <C> accumulation.  Shared by qaoa_sweep.cu (one tile per CTA) and
// qaoa_sweep_tma.cu (persistent, TMA-fed).
#pragma once
#include <type_traits>

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
//
// Skewed layout (sk = 1, the C = 3 fast flows): in lanes with lane bit 3 set,
// physical register p holds logical register p ^ 1.  The lane-bit-3 <->
// register-bit-0 transpose then moves the odd physical registers of every lane
// (no selects or predicated moves), the RX butterflies are symmetric in their
// two operands, and the cut counts follow from a shifted thread base (cut16);
// only the even / odd registers' memory bases differ by one register-bit-0
// step.  sk = 0 is the plain layout.
template <int M>
__device__ __forceinline__ void smem_store(double2* buf, int sb, const double2 (&v)[kRegs],
                                           int sk = 0) {
  constexpr int D = slot(tile_index<M>(0, 1));
  const int se = sb + sk * D, so = sb - sk * D;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) buf[((r & 1) ? so : se) + slot(tile_index<M>(0, r))] = v[r];
}
template <int M>
__device__ __forceinline__ void smem_load(const double2* buf, int sb, double2 (&v)[kRegs],
                                          int sk = 0) {
  constexpr int D = slot(tile_index<M>(0, 1));
  const int se = sb + sk * D, so = sb - sk * D;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) v[r] = buf[((r & 1) ? so : se) + slot(tile_index<M>(0, r))];
}

struct ThreadSlots {
  int s[5];
};

// Re-map registers from mapping A to mapping B through shared memory.  In a
// later exchange every thread writes (in mapping B) exactly the slots it read
// here, so one barrier per exchange suffices; the tile loop adds one barrier
// before the first write of the next tile.
template <int A, int B>
__device__ __forceinline__ void exchange(double2* buf, const ThreadSlots& ts, double2 (&v)[kRegs],
                                         int sk = 0) {
  smem_store<A>(buf, ts.s[A], v, sk);
#if defined(QB_SKIP) && (QB_SKIP & 128)
  __syncwarp();  // probe builds only (timing of an exchange without the CTA barrier; wrong data)
#else
  __syncthreads();
#endif
  smem_load<B>(buf, ts.s[B], v, sk);
}

// Same, for a 256-thread group of a larger CTA: named barrier `bar_id`.
template <int A, int B>
__device__ __forceinline__ void exchange_bar(double2* buf, const ThreadSlots& ts, double2 (&v)[kRegs],
                                             int bar_id, int sk = 0) {
  smem_store<A>(buf, ts.s[A], v, sk);
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kThreads) : "memory");
  smem_load<B>(buf, ts.s[B], v, sk);
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

// The same transpose in the skewed layout: every lane sends and receives its
// odd physical registers (4 shuffles per moved amplitude, nothing else).
__device__ __forceinline__ void transpose_lane3_sk(double2 (&v)[kRegs]) {
  __syncwarp();  // see transpose_lane3
#pragma unroll
  for (int r = 1; r < kRegs; r += 2) {
    v[r].x = __shfl_xor_sync(0xffffffffu, v[r].x, 8);
    v[r].y = __shfl_xor_sync(0xffffffffu, v[r].y, 8);
  }
}

// Lane bit 3 of the calling thread: the skew of the C = 3 fast flows.
__device__ __forceinline__ int lane_skew() { return (threadIdx.x >> 3) & 1; }

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

// Physical index of element 0 of tile `tile`: tile bits cleared, the non-tile
// bits [C, q) and [q + 12 - C, n) filled from the tile number (low part first).
template <int C>
__device__ __forceinline__ uint64_t tile_base(uint64_t tile, int q) {
  const int low_bits = C >= 12 ? 0 : q - C;
  return C >= 12 ? (tile << 12)
                 : (((tile & ((1ull << low_bits) - 1ull)) << C) | ((tile >> low_bits) << (q + 12 - C)));
}

// L2 prefetch of a whole tile (its 2^(12-C) contiguous runs), spread over the
// CTA's threads: the bulk-prefetch engine pulls the runs into L2 while the SM
// works, so the tile's later loads hit L2 instead of HBM.
template <int C, int THREADS>
__device__ __forceinline__ void prefetch_tile_l2(const double2* amps, uint64_t base, uint64_t Q,
                                                 int tid) {
  constexpr int runs = C >= 12 ? 1 : (1 << (12 - C));
  constexpr uint32_t run_bytes = C >= 12 ? 65536u : (16u << C);
  for (int i = tid; i < runs; i += THREADS) {
    const double2* p = amps + base + (C >= 12 ? 0ull : (uint64_t)i * Q);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(run_bytes) : "memory");
  }
}

// TMA coordinates of half `h` of tile `tile` (dims as built by make_tile_map).
template <int C>
__device__ __forceinline__ void half_coords(const SweepArgs& a, uint64_t tile, int h, int (&c)[5]) {
  c[0] = 0;
  if (C >= 12) {
    c[1] = 0; c[2] = h; c[3] = (int)tile; c[4] = 0;
  } else {
    const int low_bits = a.q - C;
    const int low = (int)(tile & ((1ull << low_bits) - 1ull));
    const int high = (int)(tile >> low_bits);
    if (C == 3) {
      c[1] = low; c[2] = 0; c[3] = h; c[4] = high;
    } else {
      c[1] = 0; c[2] = low; c[3] = h << (C < 12 ? 11 - C : 0); c[4] = high;
    }
  }
}
// x with bit ranges [lo, lo + m) and [hi, hi + m) exchanged (disjoint ranges).
__device__ __forceinline__ uint64_t swap_bit_ranges(uint64_t x, int lo, int hi, int m) {
  const uint64_t mask = (1ull << m) - 1ull;
  const uint64_t a = (x >> lo) & mask, b = (x >> hi) & mask;
  return (x & ~((mask << lo) | (mask << hi))) | (a << hi) | (b << lo);
}

struct TileCtx {
  uint64_t base;           // physical index of tile element 0 (tile bits zero), without x_hi
  uint64_t tb0, tb1, tb2;  // thread base offsets per mapping
};

// Per-tile cut-count basis, computed once per CTA by warp 0 (lane-parallel over
// nodes).  h = true index of tile element 0 with all tile bits cleared
// (x_hi ^ cmask ^ base, see GraphDev::cmask); K = C(h); per tile node k,
// d[k] = deg(k) - 2 popc(adj[k] & h) (change of C when node k alone is set);
// adjl[k] = tile-local neighbour mask (12 bits); tmask = cmask's tile bits (the
// true tile bits of tile index t are t ^ tmask).  Packed so a thread reads the
// whole basis with four broadcast loads: pk[k] = d[k] << 16 | adjl[k].
struct __align__(16) CutBasis {
  int pk[12];
  int K;
  int tmask;
};

__device__ __forceinline__ int pack_basis(int d, int adjl) {
  return (int)(((unsigned)d << 16) | (unsigned)adjl);
}

template <bool WIDE, int C>
__device__ __forceinline__ void cut_basis(const SweepArgs& a, uint64_t base, int q, CutBasis* cb) {
#if defined(QB_SKIP) && (QB_SKIP & 64)
  // probe builds only: a zero basis (every C(x) = 0) instead of the per-tile work
  if ((threadIdx.x & 31) < 14) reinterpret_cast<int*>(cb)[threadIdx.x & 31] = 0;
  return;
#endif
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
    const uint32_t lo = (uint32_t)(m & ((C >= 12) ? 0xFFFull : ((1ull << C) - 1ull)));
    const uint32_t hi = (C >= 12) ? 0u : (uint32_t)((m >> q) & ((1ull << (12 - C)) - 1ull)) << C;
    cb->pk[lane] = pack_basis(__popcll(m) - 2 * __popcll(m & h), (int)(lo | hi));
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
struct CutParts {
  int c0;       // C of the thread's register-0 element
  int d[4];     // change of C when register bit j alone flips
  int a[4][4];  // a[j][k] (j < k): -a is the extra change when both flip (0 or +-2)
};

template <int M>
__device__ __forceinline__ void cut_parts(const CutBasis* cb, CutParts& cp, int tid, int sk) {
  // four broadcast loads of the packed basis
  int pk[12];
  const int4* p4 = reinterpret_cast<const int4*>(cb->pk);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int4 w = p4[i];
    pk[4 * i] = w.x; pk[4 * i + 1] = w.y; pk[4 * i + 2] = w.z; pk[4 * i + 3] = w.w;
  }
  const int2 kt = *reinterpret_cast<const int2*>(&cb->K);
  // skewed layout: physical register 0 holds logical register sk
  const int T = tile_index<M>(tid, 0) ^ kt.y ^ (sk ? tile_index<M>(0, 1) : 0);
  constexpr int g = group_of<M>();
  int c0 = kt.x;
#pragma unroll
  for (int k = 0; k < 12; ++k)
    if ((T >> k) & 1) c0 += (pk[k] >> 16) - __popc(pk[k] & T);
  cp.c0 = c0;
  int al[4], sg[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    al[j] = pk[4 * g + j] & 0xFFF;
    sg[j] = ((T >> (4 * g + j)) & 1) ? -1 : 1;
    cp.d[j] = sg[j] * ((pk[4 * g + j] >> 16) - 2 * __popc(al[j] & T));
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int k = j + 1; k < 4; ++k) cp.a[j][k] = 2 * sg[j] * sg[k] * ((al[j] >> (4 * g + k)) & 1);
}

template <int M>
__device__ __forceinline__ void cut16(const CutBasis* cb, int (&c)[16], int tid, int sk = 0) {
  CutParts cp;
  cut_parts<M>(cb, cp, tid, sk);
  const int c0 = cp.c0;
  const int(&d)[4] = cp.d;
  const int a01 = cp.a[0][1], a02 = cp.a[0][2], a03 = cp.a[0][3];
  const int a12 = cp.a[1][2], a13 = cp.a[1][3], a23 = cp.a[2][3];
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

// ---- weighted cost, factored (fast schedule) --------------------------------
// amp *= exp(-i gamma/2 sum_e w_e z_e(x)), z_e = +1 when the endpoints agree, -1
// when cut (reference cost.py:147-159, compressed backend).  With the non-tile
// bits h of a tile fixed, the phase factors into
//   F(h) * prod_{tile nodes k} (x_k ? conj(B_k) : B_k) * Q[t]
// F = edges outside the tile, B_k = edges from tile node k to outside (for
// x_k = 0), Q = edges inside the tile (a per-geometry table of the true tile
// index, built once per level).  All factors have unit modulus, so flipping a
// register bit multiplies by conj(B)^2 or B^2.  ~16 FP64 ops per amplitude
// instead of an edge-order sum plus sincos per amplitude; not bit-identical to
// the reference's sum (~1e-15 relative), the exact schedule keeps that path.
struct WBasis {
  double2 F;
  double2 B[12];
  int tmask;
};

__device__ __forceinline__ double2 cmul_u(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -a.y * b.y), __fma_rn(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

// Warp-wide basis of one tile (call from one full warp).
template <int C>
__device__ __forceinline__ void wbasis(const SweepArgs& a, uint64_t base, int q, const double2* __restrict__ wu,
                                       WBasis* wb) {
  const uint64_t tile_phys = (C >= 12) ? 0xFFFull
                                       : (((1ull << C) - 1ull) | (((1ull << (12 - C)) - 1ull) << q));
  const uint64_t h = (a.g.x_hi ^ a.g.cmask ^ base) & ~tile_phys;
  const int lane = threadIdx.x & 31;
  double2 f = make_double2(1.0, 0.0);
  for (int e = lane; e < a.wm; e += 32) {
    const int2 ij = __ldg(a.wedge + e);
    if (((tile_phys >> ij.x) & 1ull) | ((tile_phys >> ij.y) & 1ull)) continue;
    const double2 u = __ldg(wu + e);
    f = cmul_u(f, (((h >> ij.x) ^ (h >> ij.y)) & 1ull) ? conj2(u) : u);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double2 other;
    other.x = __shfl_xor_sync(0xffffffffu, f.x, o);
    other.y = __shfl_xor_sync(0xffffffffu, f.y, o);
    f = cmul_u(f, other);
  }
  if (lane < 12) {
    const int p = tile_pos<C>(lane, q);
    double2 b = make_double2(1.0, 0.0);
    for (int idx = __ldg(a.winc_off + p); idx < __ldg(a.winc_off + p + 1); ++idx) {
      const int e = __ldg(a.winc + idx);
      const int2 ij = __ldg(a.wedge + e);
      const int j = ij.x == p ? ij.y : ij.x;
      if ((tile_phys >> j) & 1ull) continue;
      const double2 u = __ldg(wu + e);
      b = cmul_u(b, ((h >> j) & 1ull) ? conj2(u) : u);
    }
    wb->B[lane] = b;
  }
  if (lane == 0) {
    const uint64_t cm = a.g.cmask;
    wb->F = f;
    wb->tmask = (int)((C >= 12) ? (cm & 0xFFFull)
                                : ((cm & ((1ull << C) - 1ull)) |
                                   (((cm >> q) & ((1ull << (12 - C)) - 1ull)) << C)));
  }
}

// Weighted cut value of the tile's basis states (fused weighted <C>, graph.py
// 144-151 up to summation order): cut_w(h|t) = hh + sum_k (x_k ? W_k - S_k : S_k)
// + Cint[t], S_k = weight from tile node k to set non-tile nodes, W_k = all its
// weight to non-tile nodes, Cint = edges inside the tile.
struct WCutBasis {
  double hh;
  double S[12];
  double W[12];
  int tmask;
};

template <int C>
__device__ __forceinline__ void wcut_basis(const SweepArgs& a, uint64_t base, int q, WCutBasis* wb) {
  const uint64_t tile_phys = (C >= 12) ? 0xFFFull
                                       : (((1ull << C) - 1ull) | (((1ull << (12 - C)) - 1ull) << q));
  const uint64_t h = (a.g.x_hi ^ a.g.cmask ^ base) & ~tile_phys;
  const int lane = threadIdx.x & 31;
  double hh = 0.0;
  for (int e = lane; e < a.wm; e += 32) {
    const int2 ij = __ldg(a.wedge + e);
    if (((tile_phys >> ij.x) & 1ull) | ((tile_phys >> ij.y) & 1ull)) continue;
    if (((h >> ij.x) ^ (h >> ij.y)) & 1ull) hh += __ldg(a.ww + e);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hh += __shfl_xor_sync(0xffffffffu, hh, o);
  if (lane < 12) {
    const int p = tile_pos<C>(lane, q);
    double S = 0.0, W = 0.0;
    for (int idx = __ldg(a.winc_off + p); idx < __ldg(a.winc_off + p + 1); ++idx) {
      const int e = __ldg(a.winc + idx);
      const int2 ij = __ldg(a.wedge + e);
      const int j = ij.x == p ? ij.y : ij.x;
      if ((tile_phys >> j) & 1ull) continue;
      const double w = __ldg(a.ww + e);
      W += w;
      if ((h >> j) & 1ull) S += w;
    }
    wb->S[lane] = S;
    wb->W[lane] = W;
  }
  if (lane == 0) {
    const uint64_t cm = a.g.cmask;
    wb->hh = hh;
    wb->tmask = (int)((C >= 12) ? (cm & 0xFFFull)
                                : ((cm & ((1ull << C) - 1ull)) |
                                   (((cm >> q) & ((1ull << (12 - C)) - 1ull)) << C)));
  }
}

template <int M>
__device__ __forceinline__ double expect_wacc(const double2 (&v)[kRegs], const WCutBasis* wb,
                                              const double* __restrict__ cint, int tid, int sk) {
  constexpr int g = group_of<M>();
  const int T = tile_index<M>(tid, 0) ^ wb->tmask ^ (sk ? tile_index<M>(0, 1) : 0);
  double base = wb->hh;
#pragma unroll
  for (int k = 0; k < 12; ++k) base += ((T >> k) & 1) ? wb->W[k] - wb->S[k] : wb->S[k];
  double d[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double S = wb->S[4 * g + j], W = wb->W[4 * g + j];
    d[j] = ((T >> (4 * g + j)) & 1) ? 2.0 * S - W : W - 2.0 * S;
  }
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    double val = base + __ldg(cint + ((T ^ tile_index<M>(0, r)) & 0xFFF));
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((r >> j) & 1) val += d[j];
    acc += (v[r].x * v[r].x + v[r].y * v[r].y) * val;
  }
  return acc;
}

// Registers of mapping M (M2 or M1) times the weighted phase of their basis
// states; register combinations visited in Gray-code order (one complex
// multiply per register for the running B product).
template <int M>
__device__ __forceinline__ void apply_wcost(double2 (&v)[kRegs], const WBasis* wb,
                                            const double2* __restrict__ qt, int tid, int sk) {
  constexpr int g = group_of<M>();
  const int T = tile_index<M>(tid, 0) ^ wb->tmask ^ (sk ? tile_index<M>(0, 1) : 0);
  double2 cur = wb->F;
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const double2 b = wb->B[k];
    cur = cmul_u(cur, ((T >> k) & 1) ? conj2(b) : b);
  }
  double2 up[4];  // multiplier when register bit j flips away from T's value
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double2 b = wb->B[4 * g + j];
    const double2 b2 = cmul_u(b, b);
    up[j] = ((T >> (4 * g + j)) & 1) ? b2 : conj2(b2);
  }
  int prev = 0;
#pragma unroll
  for (int k = 0; k < kRegs; ++k) {
    const int r = k ^ (k >> 1);  // Gray order
    if (k) {
      const int j = (r ^ prev) == 1 ? 0 : (r ^ prev) == 2 ? 1 : (r ^ prev) == 4 ? 2 : 3;
      cur = cmul_u(cur, (r >> j) & 1 ? up[j] : conj2(up[j]));
    }
    prev = r;
    const double2 ph = cmul_u(cur, __ldg(qt + ((T ^ tile_index<M>(0, r)) & 0xFFF)));
    v[r] = cmul_u(v[r], ph);
  }
}

// Cache policy of the tile stream and the phase-table gathers (QB_LDMODE, A/B
// builds): 0 = ld.global.cs / ld.global.nc; 1 (default) = tile loads
// L1::no_allocate: the streaming tile never displaces the phase table from L1
// (merged sweep 7.23 -> 7.12 ms, tools/decomp_ld.sh); 2 = 1 + table gathers
// L1::evict_last (no further change).
#ifndef QB_LDMODE
#define QB_LDMODE 1
#endif
__device__ __forceinline__ double2 ld_tile(const double2* p) {
  if (QB_LDMODE >= 1) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
  return __ldcs(p);
}
__device__ __forceinline__ double2 ld_phase(const double2* p) {
  if (QB_LDMODE >= 2) {
    double2 v;
    asm("ld.global.nc.L1::evict_last.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
  return __ldg(p);
}

// amp *= table_even[E - C(x)] (table_even[k] = phase_table[2k]; reference
// cost.py:168-172 indexes table[(E - 2C) + E]).
#ifndef QB_SKIP
#define QB_SKIP 0
#endif
template <int M>
__device__ __forceinline__ void apply_cost(double2 (&v)[kRegs], const CutBasis* cb,
                                           const double2* __restrict__ tab, int e,
                                           int tid = threadIdx.x, int sk = 0) {
  int c[16];
  if (QB_SKIP & 32) {  // probe builds only: no cut counts
#pragma unroll
    for (int r = 0; r < kRegs; ++r) c[r] = (tid + r) & 15;
  } else {
    cut16<M>(cb, c, tid, sk);
  }
  if (QB_SKIP & 16) {  // probe builds only: no table gather
    const double2 p0 = __ldg(tab + e);
#pragma unroll
    for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], make_double2(p0.x + c[r], p0.y));
  } else {
#pragma unroll
    for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], ld_phase(tab + (e - c[r])));
  }
}

// Launch control with the pre-multiplied table (kGenTab): every register
// starts as gen, so gen x phase is a table entry (same rounding as apply_cost).
template <int M>
__device__ __forceinline__ void apply_gen_phase(double2 (&v)[kRegs], const CutBasis* cb,
                                                const double2* __restrict__ gtab, int e,
                                                int tid = threadIdx.x, int sk = 0) {
  int c[16];
  cut16<M>(cb, c, tid, sk);
#pragma unroll
  for (int r = 0; r < kRegs; ++r) v[r] = ld_phase(gtab + (e - c[r]));
}

template <int M>
__device__ __forceinline__ double expect_acc(const double2 (&v)[kRegs], const CutBasis* cb,
                                             int tid = threadIdx.x, int sk = 0) {
  int c[16];
  cut16<M>(cb, c, tid, sk);
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

// Visit the 16 global addresses of a thread's registers in mapping M,
// f(r, pointer to the amplitude held by physical register r).  Offsets are
// linear in the register bits (tile_off over disjoint bits), so the pointers
// are walked with one 64-bit add per register pair from the four register-bit
// strides instead of a runtime multiply per register (the address arithmetic
// was ~16% of the merged sweep's instructions).  Skewed layout: physical r
// holds logical r ^ sk.
template <int C, int M, typename F>
__device__ __forceinline__ void walk_tile(double2* base, uint64_t Q, int sk, F&& f) {
  if (C >= 12) {  // compile-time offsets
#pragma unroll
    for (int r = 0; r < kRegs; ++r) f(r, base + tile_off<C>(tile_index<M>(0, r ^ sk), Q));
    return;
  }
  const int64_t s0 = (int64_t)tile_off<C>(tile_index<M>(0, 1), Q);
  const int64_t s1 = (int64_t)tile_off<C>(tile_index<M>(0, 2), Q);
  const int64_t s2 = (int64_t)tile_off<C>(tile_index<M>(0, 4), Q);
  const int64_t s3 = (int64_t)tile_off<C>(tile_index<M>(0, 8), Q);
  const int64_t ev = sk ? s0 : 0, od = sk ? 0 : s0;  // logical bit 0 of physical even / odd
  double2* p = base;  // logical offset of the pair (bits 1..3), bit 0 clear
#pragma unroll
  for (int m = 0; m < kRegs / 2; ++m) {
    if (m) {
      // binary increment of m: bit b set, bits below cleared
      const int b = (m & 1) ? 0 : (m & 2) ? 1 : 2;
      const int64_t step = b == 0 ? s1 : b == 1 ? s2 - s1 : s3 - s2 - s1;
      p += step;
    }
    f(2 * m, p + ev);
    f(2 * m + 1, p + od);
  }
}

template <int C, int M>
__device__ __forceinline__ void store_tile(double2* __restrict__ amps, const TileCtx& tc,
                                           uint64_t Q, const double2 (&v)[kRegs], uint32_t flags,
                                           int sk = 0) {
  if (flags & kNoStore) return;
  const uint64_t tb = M == 2 ? tc.tb2 : tc.tb1;
  walk_tile<C, M>(amps + tc.base + tb, Q, sk, [&](int r, double2* ptr) { __stcs(ptr, v[r]); });
}

// ---- the register-tile work of a fast-schedule sweep ------------------------
// Shared by both sweep kernels.  FLOW 1: [cost] RX(set); FLOW 2: [cost] RX(set)
// -> cost -> RX(set) (two levels in one sweep).  `xchg(ic<A>, ic<B>)` re-maps
// the registers from mapping A to B through the kernel's exchange buffer and
// barrier.  The registers start in mapping M2 and end in fast_last<C, FLOW>().
template <int V>
using ic = std::integral_constant<int, V>;

// Timing-decomposition switches for tools/sweep_probe builds only (the library
// is built with QB_SKIP = 0): bit 0 skips the shared-memory exchanges, bit 1
// the lane transposes, bit 2 the cost phase, bit 3 the RX butterflies; inside
// the cost (apply_cost) bit 4 the table gather, bit 5 the cut counts; bit 6
// replaces the per-tile cut basis (cut_basis) by a zero basis.
constexpr bool kDoX = !(QB_SKIP & 1), kDoT = !(QB_SKIP & 2), kDoC = !(QB_SKIP & 4),
               kDoR = !(QB_SKIP & 8);

template <int C, int FLOW>
__host__ __device__ constexpr int fast_last() {
  return C >= 12 ? (FLOW == 2 ? 2 : 1) : ((Act<C>::g1 && FLOW == 1) ? 1 : 2);
}

// WGT: weighted cost (apply_wcost with wb[0] / wb[1] for the pre / mid level).
template <int C, int FLOW, bool WGT = false, typename X>
__device__ __forceinline__ void fast_tile(double2 (&v)[kRegs], const SweepArgs& a, const CutBasis* cb,
                                          const WBasis* wb, int tid, int sk, X&& xchg) {
  using A = Act<C>;
  const int e = a.g.tot_edge;
  const double r1a = a.rx1.a, r2a = a.rx2.a;
  if (a.flags & kPreCost) {
    if (WGT) apply_wcost<2>(v, &wb[0], a.wq1, tid, sk);
    else if (kDoC && (a.flags & kGenTab)) apply_gen_phase<2>(v, cb, a.table, e, tid, sk);
    else if (kDoC) apply_cost<2>(v, cb, a.table, e, tid, sk);
  }
  if (C >= 12) {
    // low set: G2 (loaded), G0, G1 [, cost, G1, G0, G2]
    if (kDoR) rx_regs2<A::g2, false>(v, r1a, 0.0);
    if (kDoX) xchg(ic<2>(), ic<0>());
    if (kDoR) rx_regs2<A::g0, false>(v, r1a, 0.0);
    if (kDoX) xchg(ic<0>(), ic<1>());
    if (kDoR) rx_regs2<A::g1, false>(v, r1a, 0.0);
    if (FLOW == 2) {
      if (WGT) apply_wcost<1>(v, &wb[1], a.wq2, tid, sk);
      else if (kDoC) apply_cost<1>(v, cb, a.table2, e, tid, sk);
      if (kDoR) rx_regs2<A::g1, false>(v, r2a, 0.0);
      if (kDoX) xchg(ic<1>(), ic<0>());
      if (kDoR) rx_regs2<A::g0, false>(v, r2a, 0.0);
      if (kDoX) xchg(ic<0>(), ic<2>());
      if (kDoR) rx_regs2<A::g2, false>(v, r2a, 0.0);
    }
  } else {
    // high set: G2 (+ tile bit 3), G1 [, cost, G1 (+ tile bit 3), G2]
    if (kDoR) rx_regs2<A::g2, false>(v, r1a, 0.0);
    if (A::g0_shfl) {  // C = 3: tile bit 3 traded into register bit 0 (M2 -> M3)
      if (kDoT) transpose_lane3_sk(v);
      if (kDoR) rx_regs2<1u, false>(v, r1a, 0.0);
      if (kDoX) xchg(ic<3>(), ic<1>());
      if (kDoR) rx_regs2<A::g1, false>(v, r1a, 0.0);
      if (FLOW == 2) {
        if (WGT) apply_wcost<1>(v, &wb[1], a.wq2, tid, sk);
        else if (kDoC) apply_cost<1>(v, cb, a.table2, e, tid, sk);
        if (kDoR) rx_regs2<A::g1, false>(v, r2a, 0.0);
        if (kDoT) transpose_lane3_sk(v);  // M1 -> M4
        if (kDoR) rx_regs2<1u, false>(v, r2a, 0.0);
        if (kDoX) xchg(ic<4>(), ic<2>());
        if (kDoR) rx_regs2<A::g2, false>(v, r2a, 0.0);
      }
    } else if (A::g1) {
      if (kDoX) xchg(ic<2>(), ic<1>());
      if (kDoR) rx_regs2<A::g1, false>(v, r1a, 0.0);
      if (FLOW == 2) {
        if (WGT) apply_wcost<1>(v, &wb[1], a.wq2, tid, sk);
        else if (kDoC) apply_cost<1>(v, cb, a.table2, e, tid, sk);
        if (kDoR) rx_regs2<A::g1, false>(v, r2a, 0.0);
        if (kDoX) xchg(ic<1>(), ic<2>());
        if (kDoR) rx_regs2<A::g2, false>(v, r2a, 0.0);
      }
    } else if (FLOW == 2) {
      if (WGT) apply_wcost<2>(v, &wb[1], a.wq2, tid, sk);
      else if (kDoC) apply_cost<2>(v, cb, a.table2, e, tid, sk);
      if (kDoR) rx_regs2<A::g2, false>(v, r2a, 0.0);
    }
  }
  if (a.flags & kScale) {
#pragma unroll
    for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], a.scale);
  }
}

}  // namespace qb
