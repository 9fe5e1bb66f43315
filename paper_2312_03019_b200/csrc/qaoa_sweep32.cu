// qaoa_sweep32.cu -- the fused sweep for the strided sets with C = 3..7
// carried bits (9..5 mixed qubits; the policy is in sweep32_eligible: N = 30's
// merged and last sweeps, single sweeps of N = 33 / 26 / 24 / 28, every sweep
// of the 5-qubit sets of N = 22) with 128 threads x 32 amplitudes
// per 4096-amplitude tile, two CTAs per SM.
//
// Why a second register geometry: in the 256 x 16 kernel (qaoa_sweep.cu) the
// 9 mixed tile bits of a C = 3 set need three register windows (4 + 4 + 1),
// i.e. per merged sweep two exchanges over 8 warps plus two lane transposes;
// the L1/shared pipe is its busiest resource (62%, profiles/r10_summary.md).
// Five-bit register windows cover the mixed bits with at most two windows
// (for C = 7 the load window alone: no exchange):
//   ML: registers = tile bits 7..11, threads = tile bits 0..6        (HBM load/store)
//   MB: registers = tile bits 3..7,  threads = tile bits 0..2, 8..11  (HBM store, FLOW 1)
// (tile bit 7 rides along in MB unmixed: it is mixed in ML).  A merged sweep is
// ML -> MB, cost, MB -> ML: two exchanges over 4 warps, no lane transposes (-11%
// L1 wavefronts per tile).  Both mappings keep the carried bits 0..2 on lanes
// 0..2, so every HBM access is a 128-byte run (four per warp instruction, as in
// qaoa_sweep.cu) and every 8-lane phase of a 128-bit shared access covers 8
// consecutive slots (conflict-free without padding).  CTAs per SM: see
// S32_MINB_F below.
//
// Arithmetic per amplitude: the fast-mode butterflies (rx_form1), the cost
// lookup (cmul_np with the even phase table), scale and <C> of fast_tile; only
// the order in which the nine qubits of a set are applied differs from the
// 256 x 16 flow (~1e-15; the fast schedule's tolerance is 1e-12).  Exact,
// weighted, mirror and launch-control sweeps keep the 256 x 16 kernels.
//
// Measured on B200 (tools/s32_probe.sh, profiles/r11_s32_probe.txt; policy with
// vs without this kernel): merged sweep of set 1 6.48-6.50 vs 6.72 ms, of the top
// set 7.28-7.30 vs 7.61-7.62, single / last sweeps unchanged (5.35-5.39 vs
// 5.38-5.42); bench step 81.9-82.1 vs 80.4-80.6 layers/s (profiles/r11_s32_bench_ab.txt).
//
// Reference path replaced: see qaoa_sweep.cu (cost.py:162-176, circuit.py:89-94,
// state.py:110-128, circuit.py:116-121).
#include <stdlib.h>

#include "qaoa_common.cuh"
#include "qaoa_sweep.h"
#include "qaoa_tile.cuh"

namespace qb {
namespace s32 {

constexpr int kT = 128;
constexpr int kR = 32;

template <int M>
__host__ __device__ constexpr int tidx(int tid, int r) {
  return M == 0 ? (tid | (r << 7)) : ((tid & 7) | ((tid >> 3) << 8) | (r << 3));
}
template <int M>
__host__ __device__ constexpr int rbit(int j) {  // tile bit of register bit j
  return M == 0 ? 7 + j : 3 + j;
}

template <int A, int B>
__device__ __forceinline__ void xchg(double2* buf, int tid, double2 (&v)[kR]) {
#pragma unroll
  for (int r = 0; r < kR; ++r) buf[tidx<A>(tid, r)] = v[r];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kR; ++r) v[r] = buf[tidx<B>(tid, r)];
}

template <unsigned MASK>
__device__ __forceinline__ void rx5(double2 (&v)[kR], double t) {
#pragma unroll
  for (int K = 0; K < 5; ++K) {
    if (!((MASK >> K) & 1)) continue;
#pragma unroll
    for (int r = 0; r < kR; ++r)
      if (!(r & (1 << K))) rx_form1(v[r], v[r | (1 << K)], t);
  }
}

// Cut counts of the 32 registers of mapping M, produced in two halves of 16
// (registers 0..15, then 16..31 = the first half with register bit 4 flipped)
// so only 16 counts are live next to the 128 data registers.
template <int M>
struct Cut32 {
  int c0, d[5], al[5], sg[5];
  __device__ __forceinline__ Cut32(const CutBasis* cb, int tid) {
    int pk[12];
    const int4* p4 = reinterpret_cast<const int4*>(cb->pk);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int4 w = p4[i];
      pk[4 * i] = w.x; pk[4 * i + 1] = w.y; pk[4 * i + 2] = w.z; pk[4 * i + 3] = w.w;
    }
    const int2 kt = *reinterpret_cast<const int2*>(&cb->K);
    const int T = tidx<M>(tid, 0) ^ kt.y;
    c0 = kt.x;
#pragma unroll
    for (int k = 0; k < 12; ++k)
      if ((T >> k) & 1) c0 += (pk[k] >> 16) - __popc(pk[k] & T);
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int b = rbit<M>(j);
      al[j] = pk[b] & 0xFFF;
      sg[j] = ((T >> b) & 1) ? -1 : 1;
      d[j] = sg[j] * ((pk[b] >> 16) - 2 * __popc(al[j] & T));
    }
  }
  __device__ __forceinline__ int a(int k, int j) const {  // k < j
    return 2 * sg[k] * sg[j] * ((al[k] >> rbit<M>(j)) & 1);
  }
  // c[r], r < 16
  __device__ __forceinline__ void low(int (&c)[16]) const {
    c[0] = c0;
#pragma unroll
    for (int r = 1; r < 16; ++r) {
      const int j = r >= 8 ? 3 : r >= 4 ? 2 : r >= 2 ? 1 : 0;
      const int rest = r ^ (1 << j);
      int v = c[rest] + d[j];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < j && ((rest >> k) & 1)) v -= a(k, j);
      c[r] = v;
    }
  }
  // c[r] -> c[r | 16]
  __device__ __forceinline__ void high(int (&c)[16]) const {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      int v = c[r] + d[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((r >> k) & 1) v -= a(k, 4);
      c[r] = v;
    }
  }
};

template <int M>
__device__ __forceinline__ void cost32(double2 (&v)[kR], const CutBasis* cb, const double2* __restrict__ tab,
                                       int e, int tid) {
  const Cut32<M> cp(cb, tid);
  int c[16];
  cp.low(c);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = cmul_np(v[r], ld_phase(tab + (e - c[r])));
  cp.high(c);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[16 + r] = cmul_np(v[16 + r], ld_phase(tab + (e - c[r])));
}

template <int M>
__device__ __forceinline__ double expect32(const double2 (&v)[kR], const CutBasis* cb, int tid) {
  const Cut32<M> cp(cb, tid);
  int c[16];
  cp.low(c);
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < 16; ++r) acc += (v[r].x * v[r].x + v[r].y * v[r].y) * (double)c[r];
  cp.high(c);
#pragma unroll
  for (int r = 0; r < 16; ++r) acc += (v[16 + r].x * v[16 + r].x + v[16 + r].y * v[16 + r].y) * (double)c[r];
  return acc;
}

// Launch control with the gen x phase table (kGenTab): every register starts
// as gen, so the product is the table entry (as apply_gen_phase).
template <int M>
__device__ __forceinline__ void gen32(double2 (&v)[kR], const CutBasis* cb, const double2* __restrict__ gtab,
                                      int e, int tid) {
  const Cut32<M> cp(cb, tid);
  int c[16];
  cp.low(c);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = ld_phase(gtab + (e - c[r]));
  cp.high(c);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[16 + r] = ld_phase(gtab + (e - c[r]));
}

// Weighted cost (compressed backend, fast schedule) on the 32 registers of
// mapping M: the factored per-tile phase of qaoa_tile.cuh apply_wcost, register
// combinations walked in Gray-code order over the five register bits.
template <int M>
__device__ __forceinline__ void wcost32(double2 (&v)[kR], const WBasis* wb, const double2* __restrict__ qt,
                                        int tid) {
  const int T = tidx<M>(tid, 0) ^ wb->tmask;
  double2 cur = wb->F;
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const double2 b = wb->B[k];
    cur = cmul_u(cur, ((T >> k) & 1) ? conj2(b) : b);
  }
  double2 up[5];  // multiplier when register bit j flips away from T's value
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double2 b = wb->B[rbit<M>(j)];
    const double2 b2 = cmul_u(b, b);
    up[j] = ((T >> rbit<M>(j)) & 1) ? b2 : conj2(b2);
  }
  int prev = 0;
#pragma unroll
  for (int k = 0; k < kR; ++k) {
    const int r = k ^ (k >> 1);  // Gray order
    if (k) {
      const int x = r ^ prev;
      const int j = x == 1 ? 0 : x == 2 ? 1 : x == 4 ? 2 : x == 8 ? 3 : 4;
      cur = cmul_u(cur, ((r >> j) & 1) ? up[j] : conj2(up[j]));
    }
    prev = r;
    const double2 ph = cmul_u(cur, __ldg(qt + ((T ^ tidx<M>(0, r)) & 0xFFF)));
    v[r] = cmul_u(v[r], ph);
  }
}

// Weighted <C> partial of the 32 registers of mapping M (qaoa_tile.cuh expect_wacc).
template <int M>
__device__ __forceinline__ double wexpect32(const double2 (&v)[kR], const WCutBasis* wb,
                                            const double* __restrict__ cint, int tid) {
  const int T = tidx<M>(tid, 0) ^ wb->tmask;
  double base = wb->hh;
#pragma unroll
  for (int k = 0; k < 12; ++k) base += ((T >> k) & 1) ? wb->W[k] - wb->S[k] : wb->S[k];
  double d[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double S = wb->S[rbit<M>(j)], W = wb->W[rbit<M>(j)];
    d[j] = ((T >> rbit<M>(j)) & 1) ? 2.0 * S - W : W - 2.0 * S;
  }
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    double val = base + __ldg(cint + ((T ^ tidx<M>(0, r)) & 0xFFF));
#pragma unroll
    for (int j = 0; j < 5; ++j)
      if ((r >> j) & 1) val += d[j];
    acc += (v[r].x * v[r].x + v[r].y * v[r].y) * val;
  }
  return acc;
}

}  // namespace s32

// CTAs per SM: merged sweeps of C = 3..6 run 3 (168 registers, 16-32 B of
// spills; C = 3 set-1 merged sweep 6.16 vs 6.50 ms with 2, bench step 83.1-83.3
// vs 81.0-81.1 layers/s), everything else 2 (255 registers; single-stage sweeps
// 0.3-0.6% and the C = 7 merged sweeps of N=22 2.4% faster than with 3) --
// tools/ab_probe.sh, tools/c456_m3_probe.sh, profiles/r12_minb_*.txt.
// S32_MINB overrides all (probe builds).
#ifndef S32_MINB
#define S32_MINB_F(C, FLOW, WGT) ((!(WGT) && ((FLOW) == 2 || (FLOW) == 3) && (C) <= 6) ? 3 : 2)  // (merged C = 4..6 only via QAOA_SWEEP32=2)
#else
#define S32_MINB_F(C, FLOW, WGT) S32_MINB
#endif

namespace s32 {
// Register-bit masks of the two windows for carried-bit count C (3 <= C <= 7):
// ML mixes tile bits 7..11 (all >= C); MB mixes its tile bits 3..6 that are >= C.
template <int C>
__host__ __device__ constexpr unsigned mask_mb() {
  return (0xFu >> (C > 3 ? C - 3 : 0)) << (C > 3 ? C - 3 : 0) & 0xFu;
}
// Physical offset of tile index t (tile_off<C> without the loop): the carried
// bits stay, the mixed bits scale by Q; linear over disjoint bit fields.
template <int C>
__device__ __forceinline__ uint64_t off(int t, uint64_t Q) {
  return (uint64_t)(t & ((1 << C) - 1)) + (uint64_t)(t >> C) * Q;
}
}  // namespace s32

// FLOW 1: [cost] RX(set); FLOW 2: [cost] RX(set) -> cost -> RX(set).  Fast
// schedule, unweighted, in place, 3 <= C <= 7, never launch control.
template <bool WIDE, int C, int FLOW, bool WGT = false>
__global__ void __launch_bounds__(s32::kT, S32_MINB_F(C, FLOW, WGT)) sweep32_kernel(const __grid_constant__ SweepArgs a) {
  using namespace s32;
  static_assert(C >= 3 && C <= 7, "C = 3..7");
  constexpr unsigned kMB = mask_mb<C>();  // 0 for C = 7: ML alone holds every mixed bit
  extern __shared__ __align__(16) unsigned char smem_raw32[];
  double2* buf = reinterpret_cast<double2*>(smem_raw32);
  __shared__ CutBasis cb_s;
  __shared__ WBasis wb_s[WGT ? 2 : 1];
  __shared__ WCutBasis wcb_s[WGT ? 1 : 1];
  __shared__ double red_scratch[kT / 32];
  const uint32_t flags = a.flags;
  const int tid = threadIdx.x;
  const int q = a.q;
  const uint64_t Q = 1ull << q;
  const uint64_t tile = (uint64_t)a.tile_lo + blockIdx.x;
  const uint64_t base = tile_base<C>(tile, q);
  double2* __restrict__ amps = a.amps;
  const uint64_t toff = off<C>(tidx<0>(tid, 0), Q);  // ML thread part
  const uint64_t rs = Q << (7 - C);                    // ML register stride (tile bit 7)

  double2 v[kR];
  // (the policy never sends launch control here, but without this branch around
  // the loads ptxas spills 96 bytes in the C = 3 merged flow)
  if (flags & kGen) {
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = a.gen;
  } else {
    const uint64_t pf_b = (uint64_t)a.tile_lo + blockIdx.x + a.pf_dist;
    if (a.pf_dist > 0 && pf_b < (uint64_t)(a.tile_lo + (a.tile_cnt ? a.tile_cnt : a.ntiles))) {
      if (!a.pf_tensor) {
        prefetch_tile_l2<C, kT>(amps, tile_base<C>(pf_b, q), Q, tid);
      } else if (tid == 0) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int c[5];
          half_coords<C>(a, pf_b, h, c);
          asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                           reinterpret_cast<uint64_t>(&a.map)),
                       "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4])
                       : "memory");
        }
      }
    }
    const double2* p = amps + base + toff;
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = ld_tile(p + r * rs);
  }
  // the tile's cut basis: prebuilt (launch control, FLOW 3, launch_gen_aux) or
  // built by warp 0 and published by the first barrier
  const CutBasis* cb = &cb_s;
  const bool need_cut = flags & (kPreCost | kMidCost | kExpect);
  if (FLOW == 3 && a.basis_tab) {
    cb = reinterpret_cast<const CutBasis*>(a.basis_tab) + tile;
  } else if (need_cut) {
    if (tid < 32) {
      if (WGT) {
        if (flags & kPreCost) wbasis<C>(a, base, q, a.wu1, &wb_s[0]);
        if (flags & kMidCost) wbasis<C>(a, base, q, a.wu2, &wb_s[WGT ? 1 : 0]);
        if (flags & kExpect) wcut_basis<C>(a, base, q, &wcb_s[0]);
      } else {
        cut_basis<WIDE, C>(a, base, q, &cb_s);
      }
    }
    if ((flags & kPreCost) || kMB == 0) __syncthreads();
  }
  const int e = a.g.tot_edge;
  const double t1 = a.rx1.a, t2 = a.rx2.a;
  if (FLOW == 3 && (flags & kGenTab)) gen32<0>(v, cb, a.table, e, tid);
  else if (WGT && (flags & kPreCost)) wcost32<0>(v, &wb_s[0], a.wq1, tid);
  else if (flags & kPreCost) cost32<0>(v, cb, a.table, e, tid);
  rx5<0x1Fu>(v, t1);
  if (kMB) {
    xchg<0, 1>(buf, tid, v);
    rx5<kMB>(v, t1);
  }
  if (FLOW == 2) {
    if (kMB) {
      if (WGT) wcost32<1>(v, &wb_s[WGT ? 1 : 0], a.wq2, tid);
      else cost32<1>(v, cb, a.table2, e, tid);
      rx5<kMB>(v, t2);
      xchg<1, 0>(buf, tid, v);
    } else {
      if (WGT) wcost32<0>(v, &wb_s[WGT ? 1 : 0], a.wq2, tid);
      else cost32<0>(v, cb, a.table2, e, tid);
    }
    rx5<0x1Fu>(v, t2);
  }
  constexpr int last = (FLOW == 2 || !kMB) ? 0 : 1;
  if (flags & kScale) {
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = cmul_np(v[r], a.scale);
  }
  double acc = 0.0;
  if (flags & kExpect) acc = WGT ? wexpect32<last>(v, &wcb_s[0], a.wc, tid) : expect32<last>(v, cb, tid);
  if (!(flags & kNoStore)) {
    if (last == 0) {
      double2* p = amps + base + toff;
#pragma unroll
      for (int r = 0; r < kR; ++r) __stcs(p + r * rs, v[r]);
    } else {
      double2* p = amps + base + off<C>(tidx<1>(tid, 0), Q);
#pragma unroll
      for (int r = 0; r < kR; ++r) __stcs(p + off<C>(tidx<1>(0, r), Q), v[r]);
    }
  }
  if (flags & kExpect) {
    const double t = block_sum<kT>(acc, red_scratch);
    if (threadIdx.x == 0) a.partials[tile] = t;
  }
}

// Where the 128 x 32 geometry measured faster (tools/s32_probe2.sh,
// tools/s32_policy_ab.sh, tools/c456_probe.sh; profiles/r11_s32_*):
// * every C = 3 sweep (two windows instead of 4 + 4 + 1);
// * every C = 7 sweep (the load window holds all 5 mixed bits: no exchange;
//   merged 5.34 vs 6.21 ms, N=22 p=4 +3.7%);
// * the single-stage sweeps of C = 4..6 (one exchange either way; N=33 single
//   42.4 vs 44.8 ms, last sweep + <C> 49.1 vs 51.3; N=33 step +1.1%);
// C = 4..6 merged sweeps stay on 256 x 16 (see sweep32_eligible); launch
// control runs here with the prebuilt tile bases (gen32_enabled).
// Launch control (FLOW 3) with the prebuilt tile bases and the gen x phase
// table of launch_gen_aux, three CTAs per SM: 3.97 vs 4.37-4.40 ms on the TMA
// in/out kernel inside the step (profiles/r12_gen32_ab.txt; without the helpers
// and at two CTAs per SM it was slower, 4.29 vs 3.96 ms).  QAOA_SWEEP32_GEN=0
// keeps it on the TMA kernel (A/B).
static bool gen32_enabled() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("QAOA_SWEEP32_GEN");
    v = e ? atoi(e) : 1;
  }
  return v > 0;
}
// Weighted (compressed backend) fast sweeps, two CTAs per SM: N=30 weighted
// p=10 67.2-67.6 vs 66.0-66.5 layers/s, p=4 66.7-67.3 vs 64.9 (tools/wgt32_probe.py,
// profiles/r13_wgt32_ab.txt).  QAOA_SWEEP32_WGT=0 keeps them on 256 x 16 (A/B).
static bool wgt32_enabled() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("QAOA_SWEEP32_WGT");
    v = e ? atoi(e) : 1;
  }
  return v > 0;
}
static bool sweep32_supported(const SweepArgs& a) {
  if ((a.flags & kGen) && (!gen32_enabled() || (a.flags & kStage2))) return false;
  if ((a.flags & kWeighted) && (!wgt32_enabled() || (a.flags & kGen))) return false;
  return a.carry >= 3 && a.carry <= 7 && !(a.flags & (kExact | kMirror)) && !a.out && a.ntiles >= 1 &&
         (a.flags & kStage1);
}
bool sweep32_eligible(const SweepArgs& a) {
  if (!sweep32_supported(a)) return false;
  // The choice depends on C and the flow only, never on the set's position: the
  // swapped qubit layout moves merges between geometries and must stay bit for
  // bit the in-place run.  (C = 4..6 merged sweeps at 3 CTAs per SM win where
  // the tile spans <= 256 MB -- C = 4 5.87 vs 6.10 ms, C = 5 5.90 vs 6.07, C = 6
  // 5.55 vs 5.95 -- and lose on a wide top set, C = 5 at q = 21 6.54 vs 6.15,
  // profiles/r12_c456_m3.txt: a span rule would break that identity.)
  return a.carry == 3 || a.carry == 7 || !(a.flags & kStage2);
}

static int g_sweep32 = -1;
void set_sweep32(int on) { g_sweep32 = on; }

// QAOA_SWEEP32=0 (or set_sweep32(0)) keeps every sweep on the 256 x 16 kernels,
// QAOA_SWEEP32=2 sends every supported sweep here (A/B only).
bool sweep32_selected(const SweepArgs& a) {
  int on = g_sweep32;
  if (on < 0) {
    static int env = -2;
    if (env == -2) {
      const char* e = getenv("QAOA_SWEEP32");
      env = e ? atoi(e) : 1;
    }
    on = env;
  }
  return on == 2 ? sweep32_supported(a) : (on > 0 && sweep32_eligible(a));
}

template <bool WIDE, int C, int FLOW, bool WGT = false>
static cudaError_t launch32_one(const SweepArgs& a, int grid, cudaStream_t s) {
  constexpr int smem = kTile * (int)sizeof(double2);
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(sweep32_kernel<WIDE, C, FLOW, WGT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  sweep32_kernel<WIDE, C, FLOW, WGT><<<grid, s32::kT, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool WIDE, int C>
static cudaError_t launch32_c(const SweepArgs& a, int grid, cudaStream_t s) {
  if (a.flags & kGen) return launch32_one<WIDE, C, 3>(a, grid, s);  // launch control (FLOW 1 + kGen)
  if (a.flags & kWeighted)
    return (a.flags & kStage2) ? launch32_one<WIDE, C, 2, true>(a, grid, s) : launch32_one<WIDE, C, 1, true>(a, grid, s);
  return (a.flags & kStage2) ? launch32_one<WIDE, C, 2>(a, grid, s) : launch32_one<WIDE, C, 1>(a, grid, s);
}

template <bool WIDE>
static cudaError_t launch32_w(const SweepArgs& a, int grid, cudaStream_t s) {
  switch (a.carry) {
    case 3: return launch32_c<WIDE, 3>(a, grid, s);
    case 4: return launch32_c<WIDE, 4>(a, grid, s);
    case 5: return launch32_c<WIDE, 5>(a, grid, s);
    case 6: return launch32_c<WIDE, 6>(a, grid, s);
    case 7: return launch32_c<WIDE, 7>(a, grid, s);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_sweep32(const SweepArgs& a, int grid, cudaStream_t s) {
  if (!sweep32_supported(a)) return cudaErrorNotSupported;
  return a.g.n_nodes > 32 ? launch32_w<true>(a, grid, s) : launch32_w<false>(a, grid, s);
}

}  // namespace qb
