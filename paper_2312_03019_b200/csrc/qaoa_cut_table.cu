// qaoa_cut_table.cu -- K1, the cut-table builder (CompressedCostPlan.cut_counts,
// reference cost.py:88-99; the paper's Alg. 3): C(x) for
// every basis state of the local index space, bit-exact, written as uint8
// (E <= 255) or uint16.
//
// Warp per tile of 2048 consecutive states, no block barrier: lane l owns the
// 64 states with index bits LO..LO+4 = l (LO = 4 for uint8, 3 for uint16; the
// other 6 tile bits in registers), so every store is 16 bytes of consecutive
// states from 32 consecutive lanes: 512 contiguous bytes per warp store.  Per tile the warp
// computes K = C(h) of the tile base h (lane-parallel popcount row step over
// the nodes + shuffle tree) and d_k = deg_k - 2 popc(adj_k & h) for the 11 tile
// bits (lane k).  Per lane: c0 = C(h | l << LO), d'_j = d_j - 2 popc(adj_j & l << LO)
// for the 6 register nodes, then the 64 counts by subset doubling
//   S[r | 2^k] = S[r] + d'_k   (one add per state)
// plus the graph-constant correction -2 E_low[r] (edges among the register
// nodes inside r, one table per launch in shared memory).  ~4 integer ops per
// state (the one-tile-per-CTA builder it replaces needed ~12 and waited on a
// block barrier).  Output: 64 (uint8) or 128 (uint16) contiguous bytes per lane,
// 16-byte streaming stores.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qaoa_common.cuh"
#include "qaoa_sweep.h"

namespace qb {

namespace {

constexpr int kCtBits = 11;  // states per warp tile = 2^11
constexpr int kRegBits = 6;  // states per lane = 2^6

template <bool WIDE>
__device__ __forceinline__ int popc_m(uint64_t x) {
  return WIDE ? __popcll(x) : __popc((uint32_t)x);
}

// Register nodes (bits of the state index held in a thread's registers):
// 0..LO-1 (2^LO consecutive states = 16 bytes -> one coalesced 16-byte store
// per lane: LO = 4 for uint8, 3 for uint16) and LO+5..10 (the "part"); lane
// nodes LO..LO+4.
template <int LO>
__device__ __forceinline__ constexpr int reg_node(int j) { return j < LO ? j : j + 5; }

template <bool WIDE, typename OutT>
__global__ void __launch_bounds__(256, 5) cut_table_warp_kernel(OutT* __restrict__ table, int n_local,
                                                                 const GraphDev g) {
  constexpr int LO = sizeof(OutT) == 1 ? 4 : 3;
  constexpr int NS = 1 << LO;             // consecutive states per store
  constexpr int HB = kRegBits - LO;       // part bits
  // 2 E_low[r] (edges among the register nodes selected by r) as 16-bit pairs:
  // mlp[p] = 2 E_low[2p] | 2 E_low[2p+1] << 16 (graph constant)
  __shared__ uint32_t mlp[32];
  if (threadIdx.x < 64) {
    const uint32_t r = threadIdx.x;
    uint64_t sel = 0;
#pragma unroll
    for (int j = 0; j < kRegBits; ++j)
      if ((r >> j) & 1) sel |= 1ull << reg_node<LO>(j);
    int e = 0;
#pragma unroll
    for (int j = 0; j < kRegBits; ++j) {
      const int k = reg_node<LO>(j);
      if ((sel >> k) & 1) e += __popcll(g.adj[k] & sel & ((1ull << k) - 1ull));
    }
    const uint32_t other = __shfl_down_sync(0xffffffffu, (uint32_t)(2 * e), 1);
    if ((r & 1) == 0) mlp[r >> 1] = (uint32_t)(2 * e) | (other << 16);
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t ntiles = 1ull << (n_local - kCtBits);
  const uint64_t T = (uint64_t)lane << LO;  // this lane's state bits LO..LO+4
  // register-node adjacency restricted to the lane bits (tile-independent)
  int aT[kRegBits];
#pragma unroll
  for (int j = 0; j < kRegBits; ++j) aT[j] = popc_m<WIDE>(g.adj[reg_node<LO>(j)] & T);
  // edges among the lane nodes inside T (tile-independent)
  int eT = 0;
#pragma unroll
  for (int k = LO; k < LO + 5; ++k)
    if ((T >> k) & 1) eT += popc_m<WIDE>(g.adj[k] & T & ((1ull << k) - 1ull));
  // this lane's node masks, loaded once (per-lane constant-bank indices would
  // serialise inside the tile loop): row masks of nodes lane and lane + 32,
  // adjacency of tile node lane (< 11)
  const uint64_t rm0 = lane < g.n_nodes ? g.rm[lane] : 0ull;
  const uint64_t rm1 = (WIDE && lane + 32 < g.n_nodes) ? g.rm[lane + 32] : 0ull;
  const uint64_t adjl = lane < kCtBits ? g.adj[lane] : 0ull;
  const int degl = popc_m<WIDE>(adjl);

  for (uint64_t tile = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); tile < ntiles;
       tile += warps) {
    const uint64_t h = (g.x_hi ^ g.cmask ^ (tile << kCtBits)) & ~((1ull << kCtBits) - 1ull);
    // K = C(h): row step per node (lane-parallel), cost.py:55-63
    int part = popc_m<WIDE>(rm0 & ((0ull - ((h >> lane) & 1ull)) ^ h));
    if (WIDE) part += popc_m<WIDE>(rm1 & ((0ull - ((h >> (lane + 32)) & 1ull)) ^ h));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    // d_k for the 11 tile nodes (lane k)
    const int dk = degl - 2 * popc_m<WIDE>(adjl & h);
    int c0 = part - 2 * eT;
#pragma unroll
    for (int k = LO; k < LO + 5; ++k) {
      const int d = __shfl_sync(0xffffffffu, dk, k);
      if ((T >> k) & 1) c0 += d;
    }
    int dp[kRegBits];
#pragma unroll
    for (int j = 0; j < kRegBits; ++j) dp[j] = __shfl_sync(0xffffffffu, dk, reg_node<LO>(j)) - 2 * aT[j];
    // subset doubling over the low register nodes; the part nodes are walked in
    // Gray-code order (one add or subtract of 2^LO values per part)
    int s[NS];
    s[0] = c0;
#pragma unroll
    for (int j = 0; j < LO; ++j) {
#pragma unroll
      for (int r = 0; r < (1 << j); ++r) s[r | (1 << j)] = s[r] + dp[j];
    }
    OutT* dst = table + (tile << kCtBits) + T;
#pragma unroll
    for (int k = 0; k < (1 << HB); ++k) {
      const int gp = k ^ (k >> 1);  // the part visited at step k
      if (k) {
        const int b = (k & 1) ? 0 : (k & 2) ? 1 : 2;  // the bit that changed (k < 8)
        const int dd = dp[LO + b];
        const bool on = (gp >> b) & 1;
#pragma unroll
        for (int r = 0; r < NS; ++r) s[r] += on ? dd : -dd;
      }
      // 16-bit pairs (both lanes non-negative after the correction: no borrow)
      uint32_t pr[NS / 2];
#pragma unroll
      for (int p = 0; p < NS / 2; ++p)
        pr[p] = (uint32_t)s[2 * p] + ((uint32_t)s[2 * p + 1] << 16) - mlp[(gp * NS) / 2 + p];
      OutT* q = dst + ((uint64_t)gp << (LO + 5));  // states (gp << LO+5) | (lane << LO) | r
      if (sizeof(OutT) == 1) {
        uint32_t o[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) o[w] = __byte_perm(pr[2 * w], pr[2 * w + 1], 0x6420);
        __stcs(reinterpret_cast<uint4*>(q), make_uint4(o[0], o[1], o[2], o[3]));
      } else {
        __stcs(reinterpret_cast<uint4*>(q), make_uint4(pr[0], pr[1], pr[2], pr[3]));
      }
    }
  }
}

}  // namespace

cudaError_t launch_cut_table_warps(void* table, int bytes_per, int n_local, const GraphDev& g,
                                   cudaStream_t s) {
  if (n_local < kCtBits) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t tiles = 1ull << (n_local - kCtBits);
  uint64_t grid = (tiles + 7) / 8;  // 8 warps per CTA
  const uint64_t cap = (uint64_t)sms * 5;  // <= 48 registers: 5 CTAs of 256 per SM, one wave
  if (grid > cap) grid = cap;
  const bool wide = g.n_nodes > 32;
  if (bytes_per == 1) {
    if (wide) cut_table_warp_kernel<true, uint8_t><<<(unsigned)grid, 256, 0, s>>>((uint8_t*)table, n_local, g);
    else cut_table_warp_kernel<false, uint8_t><<<(unsigned)grid, 256, 0, s>>>((uint8_t*)table, n_local, g);
  } else {
    if (wide) cut_table_warp_kernel<true, uint16_t><<<(unsigned)grid, 256, 0, s>>>((uint16_t*)table, n_local, g);
    else cut_table_warp_kernel<false, uint16_t><<<(unsigned)grid, 256, 0, s>>>((uint16_t*)table, n_local, g);
  }
  return cudaGetLastError();
}

}  // namespace qb
