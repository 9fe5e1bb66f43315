// qaoa_sweep_tma.cu -- persistent, TMA-fed variant of the fused sweep (fast
// schedule, FLOW 1 / FLOW 2 of qaoa_sweep.cu).
//
// Why: in the one-tile-per-CTA kernel each CTA loads its tile, computes, then
// stores, and the two CTAs of an SM are the only overlap -- whenever both are
// in their on-chip phase (butterflies, exchanges, cost) HBM idles.  Measured
// on B200, N=30 (tools/sweep_probe.cu): the merged level-boundary sweep takes
// 8.07 ms although its on-chip work alone takes 4.87 ms and its access pattern
// alone 5.9 ms.
//
// Here one CTA per SM runs two independent 256-thread groups (the same
// 16-amplitude-per-thread register tile and mappings as qaoa_sweep.cu, each
// group with its own padded exchange buffer and named barrier).  The tiles of
// the CTA are loaded by the TMA engine (cp.async.bulk.tensor, one 32 KB box per
// half tile) into two landing slots; the group that consumes a half
// immediately re-issues the slot for the same half of the CTA's next tile,
// which the other group will process.  Loads therefore stream while both
// groups compute; stores stay register -> HBM streaming stores.
//
// Shared memory: 2 landing slots x 32 KB (dense, TMA layout) + 2 groups x
// 68 KB (padded exchange layout) + barriers / cut bases  ~= 201 KB.
//
// Reference path replaced: see qaoa_sweep.cu (cost.py:162-176, circuit.py:89-94,
// state.py:110-128, circuit.py:42-48 / :116-121).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>

#include "qaoa_common.cuh"
#include "qaoa_sweep.h"
#include "qaoa_tile.cuh"

namespace qb {

constexpr int kGroups = 2;
constexpr int kCtaThreads = kGroups * kThreads;
constexpr int kHalfBytes = (kTile / 2) * (int)sizeof(double2);  // 32 KB
constexpr size_t kLandBytes = 2 * (size_t)kHalfBytes;
constexpr size_t kXchgBytes = (size_t)kSlots * sizeof(double2);  // 68 KB
constexpr size_t kTmaSmem = kLandBytes + kGroups * kXchgBytes + 64 + 128;

struct TmaSweepArgs {
  SweepArgs s;      // s.map: 5-D view of the state, one box = half a tile (make_tile_map)
  unsigned long long* counter;  // dynamic tile counter of this launch (zeroed)
  int n_local;
  int gen_static;  // launch-control sweeps: static tile order (no counter round trip)
};

// ---- PTX wrappers -----------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                          int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void group_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kThreads) : "memory");
}

__device__ __forceinline__ void tma_store5(const CUtensorMap* map, const void* src, int c0, int c1,
                                           int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(su32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int C>
__device__ __forceinline__ void issue_half(const TmaSweepArgs& a, void* dst, uint64_t* bar,
                                           uint64_t tile, int h) {
  int c[5];
  half_coords<C>(a.s, tile, h, c);
  mbar_expect_tx(bar, kHalfBytes);
  tma_load5(dst, &a.s.map, bar, c[0], c[1], c[2], c[3], c[4]);
}

// End of a tile.  TS: registers -> dense tile in the group's exchange buffer ->
// two TMA bulk stores (the warps move on while the TMA engine drains them);
// else streaming stores straight from the registers.
template <int C, int M, bool TS>
__device__ __forceinline__ void finish_tile(const TmaSweepArgs& ta, const TileCtx& tc, uint64_t Q,
                                            const double2 (&v)[kRegs], double2* buf, int tid,
                                            int bar_id, uint64_t tile, int sk) {
  const uint32_t flags = ta.s.flags;
  if (!TS) {
    store_tile<C, M>(ta.s.amps, tc, Q, v, flags, sk);
    return;
  }
  if (flags & kNoStore) return;
  group_bar(bar_id);  // every thread has read its last exchange slots
  constexpr int D = tile_index<M>(0, 1);
  double2* de = buf + tile_index<M>(tid, 0) + sk * D;
  double2* dodd = buf + tile_index<M>(tid, 0) - sk * D;
#pragma unroll
  for (int r = 0; r < kRegs; ++r) ((r & 1) ? dodd : de)[tile_index<M>(0, r)] = v[r];
  fence_async_smem();  // generic-proxy writes -> visible to the TMA (async proxy)
  group_bar(bar_id);
  if (tid == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int c[5];
      half_coords<C>(ta.s, tile, h, c);
      tma_store5(&ta.s.map, buf + h * (kTile / 2), c[0], c[1], c[2], c[3], c[4]);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

// TS: tiles stored by TMA (else streaming stores from registers).
template <bool WIDE, int C, int FLOW, bool TS>
__global__ void __launch_bounds__(kCtaThreads, 1) sweep_tma_kernel(const __grid_constant__ TmaSweepArgs ta) {
  constexpr bool DYN = C < 12;  // dynamic tile order for the strided sets
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  // TMA destinations must be 128-byte aligned
  unsigned char* smem_raw = smem_dyn + ((128u - (su32(smem_dyn) & 127u)) & 127u);
  double2* land = reinterpret_cast<double2*>(smem_raw);  // [2][kTile / 2] dense
  const int grp = threadIdx.x >> 8;
  const int tid = threadIdx.x & (kThreads - 1);
  double2* buf = reinterpret_cast<double2*>(smem_raw + kLandBytes + grp * kXchgBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + kLandBytes + kGroups * kXchgBytes);
  __shared__ CutBasis cbs[kGroups][2];
  using A = Act<C>;
  static_assert(FLOW == 1 || FLOW == 2, "fast flows only");
  const int sk = A::g0_shfl ? lane_skew() : 0;  // skewed register layout (qaoa_tile.cuh)
  const SweepArgs& a = ta.s;
  const uint32_t flags = a.flags;
  const int bar_id = 1 + grp;
  const int q = a.q;
  const uint64_t Q = 1ull << (C >= 12 ? 0 : q);
  const bool gen = flags & kGen;
  const bool need_cut = flags & (kPreCost | kMidCost | kExpect);
  // tiles [lo, lo + ntiles) of the 2^(n-12) (a.ntiles) of the state; `tile` below is
  // the index inside the range
  const uint64_t lo = (uint64_t)a.tile_lo;
  const uint64_t ntiles = a.tile_cnt ? (uint64_t)a.tile_cnt : (uint64_t)a.ntiles;
  const uint64_t stride = gridDim.x;

  ThreadSlots ts;
  ts.s[0] = slot(tile_index<0>(tid, 0));
  ts.s[1] = slot(tile_index<1>(tid, 0));
  ts.s[2] = slot(tile_index<2>(tid, 0));
  ts.s[3] = slot(tile_index<3>(tid, 0));
  ts.s[4] = slot(tile_index<4>(tid, 0));
  const uint64_t tb2 = tile_off<C>(tile_index<2>(tid, 0), Q);
  const uint64_t tb1 = tile_off<C>(tile_index<1>(tid, 0), Q);

  // Tiles are handed out in increasing order from a per-launch counter
  // (dynamic scheduling): the tiles in flight across the GPU then form one
  // window of consecutive indices, so the 128-byte runs of the strided high
  // sets that share a DRAM page are accessed together (a static tile -> CTA map
  // lets CTAs drift apart and measured ~15% slower on the C = 3 sets).  The
  // first `gridDim.x` tiles are static (tile b -> CTA b, group 0).
  //
  // full[h][g]: landing slot h holds half h of the next tile of group g.
  // Barriers are per group so that a group waiting for its j-th tile (phase j)
  // can never see the other group's phase.  The group that consumes half h of
  // its tile allocates the other group's next tile, publishes its index in
  // next_tile[] and refills slot h with it (or, past the end, completes the
  // phase without data so the other group stops).
  __shared__ unsigned long long next_tile[kGroups];
  __shared__ double gred[kGroups][kThreads / 32];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!gen) {
      issue_half<C>(ta, land, &full[0], lo + blockIdx.x, 0);
      issue_half<C>(ta, land + kTile / 2, &full[2], lo + blockIdx.x, 1);
    }
  }
  __syncthreads();

  unsigned long long* ctr = ta.counter;
  bool last = false;
  // launch control with a prebuilt basis table: lanes 0..15 of warp 0 hold the
  // next tile's 64-byte entry (loaded one tile ahead in the static order)
  const int* btab = reinterpret_cast<const int*>(a.basis_tab);
  const bool gen_prefetch = gen && btab && !(DYN && !ta.gen_static);
  int bnext = 0;
  if (gen_prefetch && tid < 16) {
    const uint64_t t0 = blockIdx.x + (uint64_t)grp * stride;
    if (t0 < ntiles) bnext = __ldcg(btab + (lo + t0) * 16 + tid);
  }
  for (uint32_t j = 0;; ++j) {
    if (last) break;
    uint64_t tile;
    double2 v[kRegs];
    CutBasis* cb = &cbs[grp][j & 1];
    // TS: the exchange buffer still feeds the previous tile's TMA store
    if (TS && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (gen) {
      if (DYN && !ta.gen_static) {
        if (tid == 0) next_tile[grp] = atomicAdd(ctr, 1ull);
        group_bar(bar_id);
        tile = next_tile[grp];
      } else {
        tile = blockIdx.x + (uint64_t)(2 * j + grp) * stride;
      }
      if (tile >= ntiles) break;
      if (need_cut && btab) {
        // the prebuilt basis (launch_gen_aux): a 56-byte copy instead of the
        // per-tile popcount reduction on the group's critical path
        if (tid < 14) reinterpret_cast<int*>(cb)[tid] = gen_prefetch ? bnext : __ldcg(btab + (lo + tile) * 16 + tid);
        if (gen_prefetch && tid < 16) {
          const uint64_t nt = blockIdx.x + (uint64_t)(2 * (j + 1) + grp) * stride;
          if (nt < ntiles) bnext = __ldcg(btab + (lo + nt) * 16 + tid);
        }
      } else if (need_cut && tid < 32) {
        cut_basis<WIDE, C>(a, tile_base<C>(lo + tile, q), q, cb);
      }
#pragma unroll
      for (int r = 0; r < kRegs; ++r) v[r] = a.gen;
      group_bar(bar_id);  // cut basis published; WAR on the exchange buffer / next_tile
    } else {
      mbar_wait(&full[grp], j & 1);
      tile = (grp == 0 && j == 0) ? (uint64_t)blockIdx.x : (uint64_t)next_tile[grp];
      if (tile >= ntiles) break;
      // the other group's next tile (allocated here, published before the
      // half-0 barrier; an allocation is never dropped: past the end, all are)
      if (tid == 0) next_tile[grp ^ 1] = DYN ? stride + atomicAdd(ctr, 1ull) : tile + stride;
      if (need_cut && tid < 32) cut_basis<WIDE, C>(a, tile_base<C>(lo + tile, q), q, cb);
      uint64_t nxt = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1) mbar_wait(&full[2 + grp], j & 1);
        const double2* se = land + h * (kTile / 2) + tid + (sk << 8);
        const double2* so = land + h * (kTile / 2) + tid - (sk << 8);
#pragma unroll
        for (int r = 0; r < 8; ++r) v[8 * h + r] = ((r & 1) ? so : se)[r << 8];
        // order these generic-proxy reads before the TMA refill of the slot
        // (without it the refill was observed to overtake them)
        fence_async_smem();
        group_bar(bar_id);
        if (h == 0) {
          nxt = next_tile[grp ^ 1];
          last = nxt >= ntiles;
        }
        uint64_t* bar = &full[2 * h + (grp ^ 1)];
        if (!last) {
          if (tid == 0) issue_half<C>(ta, land + h * (kTile / 2), bar, lo + nxt, h);
        } else if (h == 0 && tid == 0) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
        }
      }
    }
    TileCtx tc;
    tc.base = tile_base<C>(lo + tile, q);
    tc.tb2 = tb2;
    tc.tb1 = tb1;
    double acc = 0.0;

    fast_tile<C, FLOW>(v, a, cb, nullptr, tid, sk, [&](auto from, auto to) {
      exchange_bar<decltype(from)::value, decltype(to)::value>(buf, ts, v, bar_id, sk);
    });
    constexpr int last_m = fast_last<C, FLOW>();
    if (flags & kExpect) acc += expect_acc<last_m>(v, cb, tid, sk);
    finish_tile<C, last_m, TS>(ta, tc, Q, v, buf, tid, bar_id, lo + tile, sk);
    if (flags & kExpect) {
      // per-tile partial (fixed shuffle tree, warps in order): the sum over
      // tiles is then independent of which CTA ran which tile
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((tid & 31) == 0) gred[grp][tid >> 5] = acc;
      group_bar(bar_id);
      if (tid == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) t += gred[grp][w];
        a.partials[lo + tile] = t;
      }
    }
  }
  if (TS && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- host side ----------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 5-D FLOAT64 view of the 2^n complex128 state whose box is half a tile, laid
// out in shared memory in tile-index order (t = carried bits | mixed bits << C):
//   d0: physical bits 0..2 as 16 doubles (128 B rows)
//   C = 12: d1 bits 3..10 (box 256), d2 bit 11 (the half), d3 bits 12.. (tile)
//   C = 3 : d1 bits 3..q-1 (non-tile), d2 bits q..q+7 (box 256), d3 bit q+8
//           (the half), d4 bits q+9.. (non-tile)
//   4 <= C <= 10: d1 bits 3..C-1 (box), d2 bits C..q-1 (non-tile), d3 bits
//           q..q+11-C (box = half of them), d4 bits q+12-C.. (non-tile)
}  // namespace

bool make_tile_map(CUtensorMap* map, void* amps, int n, int C, int q) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dim[5];
  cuuint64_t str[4];  // byte strides of dims 1..4
  cuuint32_t box[5];
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const cuuint64_t total = 16ull << n;
  auto set = [&](int d, int lo_bit, int nbits, int boxbits) {
    dim[d] = 1ull << nbits;
    str[d - 1] = nbits > 0 ? (16ull << lo_bit) : total;
    box[d] = 1u << boxbits;
  };
  dim[0] = 16;
  box[0] = 16;
  if (C == 12) {
    set(1, 3, 8, 8);
    set(2, 11, 1, 0);
    set(3, 12, n - 12, 0);
    set(4, n, 0, 0);
  } else if (C == 3) {
    set(1, 3, q - 3, 0);
    set(2, q, 8, 8);
    set(3, q + 8, 1, 0);
    set(4, q + 9, n - q - 9, 0);
  } else {
    const int m = 12 - C;
    set(1, 3, C - 3, C - 3);
    set(2, C, q - C, 0);
    set(3, q, m, m - 1);
    set(4, q + m, n - q - m, 0);
  }
  static int promo_env = -2;
  if (promo_env == -2) {
    const char* e = getenv("QAOA_TMA_L2PROMO");
    promo_env = e ? atoi(e) : -1;
  }
  const CUtensorMapL2promotion promo =
      promo_env >= 0 ? (CUtensorMapL2promotion)promo_env
                     : (C >= 12 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE);
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, amps, dim, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <bool WIDE, int C, int FLOW, bool TS>
cudaError_t launch_tma_one(const TmaSweepArgs& ta, int grid, cudaStream_t s) {
  static unsigned long long configured = 0;  // bit d = device d done
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(sweep_tma_kernel<WIDE, C, FLOW, TS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
    if (e != cudaSuccess) return e;
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  sweep_tma_kernel<WIDE, C, FLOW, TS><<<grid, kCtaThreads, kTmaSmem, s>>>(ta);
  return cudaGetLastError();
}

template <bool WIDE, int C, int FLOW>
cudaError_t launch_tma_f(const TmaSweepArgs& ta, int grid, cudaStream_t s) {
  if (sweep_impl(ta.s) == 2) return launch_tma_one<WIDE, C, FLOW, true>(ta, grid, s);
  return launch_tma_one<WIDE, C, FLOW, false>(ta, grid, s);
}

template <bool WIDE, int C>
cudaError_t launch_tma_c(const TmaSweepArgs& ta, int grid, cudaStream_t s) {
  if (ta.s.flags & kStage2) return launch_tma_f<WIDE, C, 2>(ta, grid, s);
  return launch_tma_f<WIDE, C, 1>(ta, grid, s);
}

template <bool WIDE>
cudaError_t launch_tma_w(const TmaSweepArgs& ta, int grid, cudaStream_t s) {
  switch (ta.s.carry) {
    case 3: return launch_tma_c<WIDE, 3>(ta, grid, s);
    case 4: return launch_tma_c<WIDE, 4>(ta, grid, s);
    case 5: return launch_tma_c<WIDE, 5>(ta, grid, s);
    case 6: return launch_tma_c<WIDE, 6>(ta, grid, s);
    case 7: return launch_tma_c<WIDE, 7>(ta, grid, s);
    case 8: return launch_tma_c<WIDE, 8>(ta, grid, s);
    case 9: return launch_tma_c<WIDE, 9>(ta, grid, s);
    case 10: return launch_tma_c<WIDE, 10>(ta, grid, s);
    case 12: return launch_tma_c<WIDE, 12>(ta, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

int g_impl = -1;
int impl_env() {
  int& v = g_impl;
  if (v < 0) {
    const char* e = getenv("QAOA_SWEEP_IMPL");
    v = !e ? 3
          : strcmp(e, "v4") == 0 ? 0
          : strcmp(e, "tma-ld") == 0 ? 1
          : strcmp(e, "tma") == 0 ? 2 : 3;
  }
  return v;
}

}  // namespace

void set_sweep_impl(int v) { g_impl = v; }

// Which kernel runs a fast-schedule sweep (0: one tile per CTA, qaoa_sweep.cu;
// 1: persistent TMA-fed, register stores; 2: persistent TMA-fed, TMA stores).
// Measured on B200 at N=30 (tools/sweep_probe.cu, ms per sweep):
//   launch-control (kGen) sweep      v4 4.48 | TMA in/out 4.10          -> 2
//   merged sweep of the top set      v4 7.85 | TMA-fed 7.96 | in/out 7.57 -> 2
//   (C = 3, tile spans > 256 MB: 512 DRAM pages per tile, L2 prefetch hurts;
//   at N=33 the C = 5 top set is faster one tile per CTA: 50.1 vs 53.1 ms)
//   everything else                  v4 + L2 prefetch is fastest        -> 0
int sweep_impl(const SweepArgs& a) {
  if ((a.flags & (kExact | kWeighted | kMirror)) || a.carry == 11 || a.ntiles < 1 || a.out) return 0;
  const int env = impl_env();
  if (env != 3) return env;
  if (sweep32_selected(a)) return 0;  // one tile per CTA, 128 x 32 (qaoa_sweep32.cu)
  if (a.flags & kGen) {  // QAOA_GEN_IMPL overrides for launch control only (A/B)
    static int gi = -2;
    if (gi == -2) {
      const char* e = getenv("QAOA_GEN_IMPL");
      gi = e ? atoi(e) : -1;
    }
    return gi >= 0 ? gi : 2;
  }
  const bool wide_span = a.carry < 12 && a.q + 12 - a.carry + 4 > 28;
  if ((a.flags & kStage2) && wide_span && a.carry == 3) return 2;
  return 0;
}

bool sweep_uses_tma(const SweepArgs& a) { return sweep_impl(a) != 0; }

int sweep_grid(const SweepArgs& a) {
  const int64_t cnt = a.tile_cnt ? a.tile_cnt : a.ntiles;
  if (!sweep_uses_tma(a)) return (int)cnt;
  const int sms = num_sms();
  return cnt < sms ? (int)cnt : sms;
}

cudaError_t launch_sweep_tma(const SweepArgs& a, cudaStream_t s) {
  TmaSweepArgs ta;
  memset(&ta, 0, sizeof(ta));
  ta.s = a;
  int n = 12;
  while ((1ll << (n - 12)) < a.ntiles) ++n;
  ta.n_local = n;
  {
    static int gs = -1;
    if (gs < 0) {
      // launch control has no loads to keep page-local: the static order saves
      // the per-tile counter round trip (4.75 vs 5.0 ms at N=30 under the cap)
      const char* e = getenv("QAOA_GEN_STATIC");
      gs = e ? atoi(e) : 1;
    }
    ta.gen_static = gs;
  }
  if (!make_tile_map(&ta.s.map, a.amps, n, a.carry, a.q)) return cudaErrorInvalidValue;
  // one counter per launch from a per-device ring (launches on concurrent
  // streams never share one), zeroed on the launch stream
  constexpr int kCounters = 4096;
  static std::mutex mu;
  static std::map<int, unsigned long long*> pools;
  static std::atomic<unsigned> next_ctr{0};
  int dev = 0;
  cudaGetDevice(&dev);
  unsigned long long* pool = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(dev);
    if (it == pools.end()) {
      cudaError_t e = cudaMalloc(&pool, kCounters * sizeof(unsigned long long));
      if (e != cudaSuccess) return e;
      pools[dev] = pool;
    } else {
      pool = it->second;
    }
  }
  ta.counter = pool + (next_ctr.fetch_add(1) % kCounters);
  cudaError_t e = cudaMemsetAsync(ta.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const int grid = sweep_grid(a);
  return a.g.n_nodes > 32 ? launch_tma_w<true>(ta, grid, s) : launch_tma_w<false>(ta, grid, s);
}

}  // namespace qb
