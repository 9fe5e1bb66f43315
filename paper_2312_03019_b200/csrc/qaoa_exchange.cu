// qaoa_exchange.cu -- the global<->local qubit exchange of a sharded state,
// fused with the RX of the qubits that arrive.
//
// G = 2^g shards; shard r holds the basis states whose top g physical bits
// (the global bits) equal r.  The exchange swaps global bit k with local bit
// p0 + k (k < g).  Writing a local index as (y, h) with h = bits p0..p0+g-1 and
// y = the other local bits, the element (shard r, local (y, h)) moves to
// (shard h, local (y, r)): for every y the G x G block [r][h] is transposed
// across the shards.  The qubits that arrive (the old global bits, now local
// bits p0..p0+g-1 of every shard) still need this level's RX, which is a
// butterfly over r inside each column h -- so one thread owning (y, h) loads
// the column from the G shards, applies the g butterfly stages in registers,
// and (after a CTA barrier: its writes land in slots other threads of the same
// CTA read) stores the column as row h of shard h.
//
// Every element is read once and written once by exactly one thread of one
// GPU (the y range is split across the ranks), so the exchange runs in place
// with no staging buffer.  Shard pointers are device pointers valid on the
// launching device: the local shard, CUDA-IPC mappings of the peer shards
// (P2P loads / stores over NVLink) or, for virtual shards, other buffers on the
// same device.  Per GPU: (G-1)/G of 16 B per local amplitude crosses NVLink in
// each direction.
//
// Reference: the reference has no distributed state; the RX is
// apply_rx (state.py:110-128) on the arriving qubits, mixer circuit.py:89-94.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "qaoa_common.cuh"
#include "qaoa_sweep.h"

namespace qb {

// Peer-load flavour (QAOA_XCHG_LD, A/B): 0 = ld.global.cv (volatile, system
// scope: never served from a cache), 1 = ld.global.cg (L2 only), 2 = ld.global.nc.
// All three are correct: the peers' writes completed before the host barrier
// that precedes this launch, L1 starts every kernel empty, and no element is
// read after another CTA wrote it inside one launch (see above).
template <int LD>
__device__ __forceinline__ double2 ld_peer(const double2* p) {
  if (LD == 0) return __ldcv(p);
  if (LD == 1) return __ldcg(p);
  return __ldg(p);
}

template <int G, int LD>
__global__ void __launch_bounds__(256) exchange_kernel(ExchangeArgs a) {
  constexpr int YB = 256 / G;  // y values per CTA (consecutive: coalesced runs)
  const int h = threadIdx.x / YB;
  const uint64_t y = a.y_lo + (uint64_t)blockIdx.x * YB + (threadIdx.x % YB);
  const bool live = y < a.y_hi;
  const uint64_t lo_mask = (1ull << a.p0) - 1ull;
  // local index of (y, field value f) with field = bits p0..p0+g-1
  const uint64_t ybase = (y & lo_mask) | ((y >> a.p0) << (a.p0 + a.g));
  double2 v[G];
  if (live) {
#pragma unroll
    for (int r = 0; r < G; ++r) v[r] = ld_peer<LD>(a.shards[r] + (ybase | ((uint64_t)h << a.p0)));
    // butterflies over the g arriving qubits (bit k of r), increasing k
#pragma unroll
    for (int k = 0; (1 << k) < G; ++k) {
#pragma unroll
      for (int r = 0; r < G; ++r) {
        if (r & (1 << k)) continue;
        if (a.rx.mode == 0) rx_exact(v[r], v[r | (1 << k)], a.rx.a, a.rx.b);
        else rx_form1(v[r], v[r | (1 << k)], a.rx.a);
      }
    }
    if (a.scale_on) {
#pragma unroll
      for (int r = 0; r < G; ++r) v[r] = cmul_np(v[r], a.scale);
    }
  }
  __syncthreads();  // every column of this CTA's y range has been read
  if (live) {
#pragma unroll
    for (int r = 0; r < G; ++r) __stcg(a.shards[h] + (ybase | ((uint64_t)r << a.p0)), v[r]);
  }
}

template <int LD>
static cudaError_t launch_ld(const ExchangeArgs& a, unsigned grid, cudaStream_t s) {
  switch (1 << a.g) {
    case 2: exchange_kernel<2, LD><<<grid, 256, 0, s>>>(a); break;
    case 4: exchange_kernel<4, LD><<<grid, 256, 0, s>>>(a); break;
    case 8: exchange_kernel<8, LD><<<grid, 256, 0, s>>>(a); break;
    case 16: exchange_kernel<16, LD><<<grid, 256, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

static int xchg_ld_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QAOA_XCHG_LD");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 2) v = 0;
  }
  return v;
}

cudaError_t launch_exchange(const ExchangeArgs& a, cudaStream_t s) {
  if (a.y_hi <= a.y_lo) return cudaSuccess;
  const int G = 1 << a.g;
  const uint64_t count = a.y_hi - a.y_lo;
  const int yb = 256 / G;
  const uint64_t grid = (count + yb - 1) / yb;
  if (grid > 0x7fffffffull) return cudaErrorInvalidValue;
  switch (xchg_ld_mode()) {
    case 1: return launch_ld<1>(a, (unsigned)grid, s);
    case 2: return launch_ld<2>(a, (unsigned)grid, s);
    default: return launch_ld<0>(a, (unsigned)grid, s);
  }
}

}  // namespace qb
