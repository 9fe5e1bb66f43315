// qaoa_sweep.cu -- the fused cost + mixer sweep kernel (the hot path).
//
// One launch = one HBM round trip of the state.  The state is cut into tiles of
// 2^12 amplitudes (64 KiB) whose 12 "tile bits" sit at arbitrary physical bit
// positions pos[0..11] (pos[0..2] = 0, 1, 2 always, so every HBM access is a
// run of >= 8 consecutive amplitudes = 128 B).  A CTA of 256 threads holds the
// tile in registers, 16 amplitudes per thread, and re-maps it through shared
// memory between three register groups of 4 tile bits:
//   M2: registers = tile bits 8..11, threads = tile bits 0..7  (coalesced load)
//   M0: registers = tile bits 0..3,  threads = tile bits 4..11
//   M1: registers = tile bits 4..7,  threads = tile bits 0..3, 8..11 (coalesced store)
// RX butterflies on the register bits are register-local.  Between the RX
// stages of one sweep it can apply the diagonal cost phase (table lookup by
// the integer cut count C(x), recomputed from the row masks -- no table read
// from HBM), a final scale and the <C> reduction.
//
// Reference path replaced (pkg/src/qaoa_maxcut/):
//   cost layer  apply_cost_bitwise  cost.py:162-176 (+ cut_counts :88-99)
//   mixer layer apply_mixer_layer   circuit.py:89-94 -> apply_rx state.py:110-128
//   init        init_uniform        circuit.py:42-48
//   expectation                     circuit.py:116-121, graph.py:144-151
#include "qaoa_common.cuh"
#include "qaoa_sweep.h"

namespace qb {

constexpr int kTileBits = 12;
constexpr int kTile = 1 << kTileBits;
constexpr int kThreads = 256;
constexpr int kRegs = 16;

// Shared-memory slot of tile index t: one 16-byte pad after every 16 slots.
// Every mapping's register r then sits at a compile-time offset from a
// per-thread base (M2: +272 r, M0: +r, M1: +17 r) and each 8-lane phase of a
// 128-bit access touches 8 distinct 16-byte bank groups (no conflicts).
constexpr int kSlots = kTile + kTile / 16;
__device__ __forceinline__ int swz(int t) { return t + (t >> 4); }

// Tile index of register r of thread tid in mapping M.
template <int M>
__device__ __forceinline__ int tile_index(int tid, int r) {
  if (M == 2) return tid | (r << 8);
  if (M == 0) return (tid << 4) | r;
  return (tid & 15) | ((tid >> 4) << 8) | (r << 4);
}

__device__ __forceinline__ uint64_t tile_offset(int t, const int* pos) {
  uint64_t o = 0;
#pragma unroll
  for (int k = 0; k < kTileBits; ++k)
    if ((t >> k) & 1) o |= 1ull << pos[k];
  return o;
}

// Global offsets of the 16 registers of mapping M relative to the thread's base:
// subsets of the four strides of the register tile bits (4M+? see tile_index).
template <int M>
__device__ __forceinline__ void reg_strides(const int* pos, uint64_t (&s)[4]) {
  constexpr int g = (M == 2) ? 8 : (M == 0 ? 0 : 4);
#pragma unroll
  for (int k = 0; k < 4; ++k) s[k] = 1ull << pos[g + k];
}

__device__ __forceinline__ uint64_t reg_off(int r, const uint64_t (&s)[4]) {
  uint64_t o = 0;
  if (r & 1) o |= s[0];
  if (r & 2) o |= s[1];
  if (r & 4) o |= s[2];
  if (r & 8) o |= s[3];
  return o;
}

template <int M>
__device__ __forceinline__ void smem_store(double2* buf, const double2 (&v)[kRegs]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) buf[swz(tile_index<M>(tid, r))] = v[r];
}

template <int M>
__device__ __forceinline__ void smem_load(const double2* buf, double2 (&v)[kRegs]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) v[r] = buf[swz(tile_index<M>(tid, r))];
}

// Re-map registers from mapping `from` to `to` through shared memory.  Each
// thread later writes (in mapping `to`) exactly the slots it read here, so one
// barrier per exchange suffices within a tile.
__device__ __forceinline__ void exchange(double2* buf, double2 (&v)[kRegs], int from, int to) {
  if (from == to) return;
  if (from == 0) smem_store<0>(buf, v);
  else if (from == 1) smem_store<1>(buf, v);
  else smem_store<2>(buf, v);
  __syncthreads();
  if (to == 0) smem_load<0>(buf, v);
  else if (to == 1) smem_load<1>(buf, v);
  else smem_load<2>(buf, v);
}

// RX on register bit K of all 16 registers.
template <int K, int MODE>
__device__ __forceinline__ void rx_bit(double2 (&v)[kRegs], double a, double b) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    if (r & (1 << K)) continue;
    if (MODE == 0) rx_exact(v[r], v[r | (1 << K)], a, b);
    else if (MODE == 1) rx_form1(v[r], v[r | (1 << K)], a);
    else rx_form2(v[r], v[r | (1 << K)], a);
  }
}

template <int MODE>
__device__ __forceinline__ void rx_group_mode(double2 (&v)[kRegs], unsigned act4, double a,
                                              double b) {
  if (act4 & 1) rx_bit<0, MODE>(v, a, b);
  if (act4 & 2) rx_bit<1, MODE>(v, a, b);
  if (act4 & 4) rx_bit<2, MODE>(v, a, b);
  if (act4 & 8) rx_bit<3, MODE>(v, a, b);
}

// RX on the active bits of register group g (tile bits 4g..4g+3), in increasing order.
__device__ __forceinline__ void rx_group(double2 (&v)[kRegs], unsigned act, int g,
                                         const RxStage& st) {
  const unsigned a4 = (act >> (4 * g)) & 15u;
  if (!a4) return;
  if (st.mode == 0) rx_group_mode<0>(v, a4, st.a, st.b);
  else if (st.mode == 1) rx_group_mode<1>(v, a4, st.a, st.b);
  else rx_group_mode<2>(v, a4, st.a, st.b);
}

// Base offset of the thread in mapping M (register bits zero).
__device__ __forceinline__ uint64_t thread_base(int m, const int* pos) {
  const int tid = threadIdx.x;
  int t;
  if (m == 2) t = tile_index<2>(tid, 0);
  else if (m == 0) t = tile_index<0>(tid, 0);
  else t = tile_index<1>(tid, 0);
  return tile_offset(t, pos);
}

__device__ __forceinline__ void reg_positions(int m, const int* pos, int (&v)[4]) {
  const int g = (m == 2) ? 8 : (m == 0 ? 0 : 4);
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = pos[g + k];
}

template <bool WIDE>
__device__ __forceinline__ void apply_cost_regs(double2 (&v)[kRegs], uint64_t x0, const int* pos,
                                                int m, const GraphDev& g, const double2* tab) {
  int vp[4];
  reg_positions(m, pos, vp);
  int c[16];
  cut_counts16<WIDE>(x0, vp, g, c);
  const int two_e = 2 * g.tot_edge;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], tab[two_e - 2 * c[r]]);
}

template <bool WIDE>
__device__ __forceinline__ double expect_regs(const double2 (&v)[kRegs], uint64_t x0,
                                              const int* pos, int m, const GraphDev& g) {
  int vp[4];
  reg_positions(m, pos, vp);
  int c[16];
  cut_counts16<WIDE>(x0, vp, g, c);
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) acc += (v[r].x * v[r].x + v[r].y * v[r].y) * (double)c[r];
  return acc;
}

template <bool WIDE>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(const SweepArgs args) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* buf = reinterpret_cast<double2*>(smem_raw);
  double2* tab = buf + kSlots;
  __shared__ double red_scratch[kThreads / 32];

  const uint32_t flags = args.flags;
  const bool has_cost = flags & (kPreCost | kMidCost);
  double2* tab2 = tab + ((flags & kPreCost) ? args.table_len : 0);
  if (flags & kPreCost)
    for (int i = threadIdx.x; i < args.table_len; i += kThreads) tab[i] = args.table[i];
  if (flags & kMidCost)
    for (int i = threadIdx.x; i < args.table_len; i += kThreads) tab2[i] = args.table2[i];
  // tile_offsets of each mapping's thread base (constant over tiles)
  const uint64_t tb0 = thread_base(0, args.pos);
  const uint64_t tb1 = thread_base(1, args.pos);
  const uint64_t tb2 = thread_base(2, args.pos);
  uint64_t s2[4], s1[4];
  reg_strides<2>(args.pos, s2);
  reg_strides<1>(args.pos, s1);
  const bool exact = flags & kExact;
  double acc = 0.0;
  double2* __restrict__ amps = args.amps;

  {
    const int64_t tile = blockIdx.x;
    // base: deposit the tile number into the non-tile bit positions
    uint64_t base = (uint64_t)tile;
#pragma unroll
    for (int k = 0; k < kTileBits; ++k) {
      const int p = args.ins[k];
      base = ((base >> p) << (p + 1)) | (base & ((1ull << p) - 1ull));
    }
    if (has_cost) __syncthreads();  // phase table staged

    double2 v[kRegs];
    int cur = 2;
    if (flags & kGen) {
#pragma unroll
      for (int r = 0; r < kRegs; ++r) v[r] = args.gen;
    } else {
      const double2* src = amps + base + tb2;
#pragma unroll
      for (int r = 0; r < kRegs; ++r) v[r] = __ldcs(src + reg_off(r, s2));
    }
    if (flags & kPreCost)
      apply_cost_regs<WIDE>(v, args.g.x_hi | base | tb2, args.pos, 2, args.g, tab);

    if (exact) {
      if (flags & kStage1) {
        for (int grp = 0; grp < 3; ++grp) {
          if (!((args.act1 >> (4 * grp)) & 15u)) continue;
          exchange(buf, v, cur, grp);
          cur = grp;
          rx_group(v, args.act1, grp, args.rx1);
        }
      }
    } else {
      if (flags & kStage1) {
        const int order[3] = {2, 0, 1};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int grp = order[i];
          if (!((args.act1 >> (4 * grp)) & 15u)) continue;
          exchange(buf, v, cur, grp);
          cur = grp;
          rx_group(v, args.act1, grp, args.rx1);
        }
      }
      if (flags & kMidCost) {
        const uint64_t tb = cur == 0 ? tb0 : (cur == 1 ? tb1 : tb2);
        apply_cost_regs<WIDE>(v, args.g.x_hi | base | tb, args.pos, cur, args.g, tab2);
      }
      if (flags & kStage2) {
        // current mapping first (no exchange), M0 in the middle, end on a
        // mapping whose stores coalesce (M1 or M2)
        int ord[3];
        if (cur == 0) { ord[0] = 0; ord[1] = 1; ord[2] = 2; }
        else { ord[0] = cur; ord[1] = 0; ord[2] = 3 - cur; }
        for (int i = 0; i < 3; ++i) {
          const int grp = ord[i];
          if (!((args.act2 >> (4 * grp)) & 15u)) continue;
          exchange(buf, v, cur, grp);
          cur = grp;
          rx_group(v, args.act2, grp, args.rx2);
        }
      }
    }
    if (cur == 0) {  // M0 stores are not coalesced
      exchange(buf, v, 0, 2);
      cur = 2;
    }
    if (flags & kScale) {
#pragma unroll
      for (int r = 0; r < kRegs; ++r) v[r] = cmul_np(v[r], args.scale);
    }
    const uint64_t tb = cur == 1 ? tb1 : tb2;
    if (flags & kExpect) acc += expect_regs<WIDE>(v, args.g.x_hi | base | tb, args.pos, cur, args.g);
    if (!(flags & kNoStore)) {
      double2* dst = amps + base + tb;
      if (cur == 1) {
#pragma unroll
        for (int r = 0; r < kRegs; ++r) __stcs(dst + reg_off(r, s1), v[r]);
      } else {
#pragma unroll
        for (int r = 0; r < kRegs; ++r) __stcs(dst + reg_off(r, s2), v[r]);
      }
    }
  }
  if (flags & kExpect) {
    const double t = block_sum<kThreads>(acc, red_scratch);
    if (threadIdx.x == 0) args.partials[blockIdx.x] = t;
  }
}

size_t sweep_smem_bytes(int table_len) {
  return (size_t)kSlots * sizeof(double2) + (size_t)table_len * sizeof(double2);
}

cudaError_t launch_sweep(const SweepArgs& args, int grid, cudaStream_t stream) {
  const int n_tables = ((args.flags & kPreCost) ? 1 : 0) + ((args.flags & kMidCost) ? 1 : 0);
  const size_t smem = sweep_smem_bytes(n_tables * args.table_len);
  if (args.g.n_nodes > 32) {
    cudaFuncSetAttribute(sweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sweep_kernel<true><<<grid, kThreads, smem, stream>>>(args);
  } else {
    cudaFuncSetAttribute(sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sweep_kernel<false><<<grid, kThreads, smem, stream>>>(args);
  }
  return cudaGetLastError();
}

int sweep_max_grid(int table_len) {
  const size_t smem = sweep_smem_bytes(table_len);
  int dev = 0;
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaFuncSetAttribute(sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<false>, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  return sms * per_sm;
}

}  // namespace qb
