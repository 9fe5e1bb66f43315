// REJECTED VARIANT (tooling record, not built into the library): measured on
// B200 at N=30 against the 256 x 16 kernel (profiles/r10_sweep8_probe.txt):
// merged S1 8.24 vs 7.05 ms, merged S2 8.37-8.42 vs 7.84, single S1 5.69 vs
// 5.42, last S1 5.64 vs 5.37 -- twice the warps do not pay for twice the
// barriers per tile.  Parity-clean (sweep_probe check, 1e-13).  It needs the
// launch_sweep hook and the set_sweep8() switch it declares to be re-added.
//
// qaoa_sweep8.cu -- the fused sweep for the strided C = 3 sets (9 mixed qubits:
// the level-boundary merged sweeps and the single high-set sweeps of N = 30)
// with 512 threads x 8 amplitudes per 4096-amplitude tile.
//
// Why a second register geometry: the 256 x 16 kernel (qaoa_sweep.cu) runs the
// merged C = 3 sweep latency-bound -- 16 warps per SM, no pipe above 62% busy
// (L1 data pipe 62%, FP64 38%, issue 37%), ~10 cycles between two issues of a
// warp (ncu, profiles/r10_summary.md).  Eight amplitudes per thread halve the
// register tile per thread (64 registers, 32 warps per SM at two CTAs per SM)
// and cut the 9 mixed tile bits into three 3-bit register windows:
//   ML: registers = tile bits 9..11, threads = tile bits 0..8   (HBM load/store)
//   MA: registers = tile bits 6..8,  threads = tile bits 0..5, 9..11
//   MB: registers = tile bits 3..5,  threads = tile bits 0..2, 6..11
// Every mapping keeps the carried bits 0..2 on lane bits 0..2, so each 8-lane
// phase of a 128-bit shared-memory access covers 8 consecutive slots: the
// exchange buffer needs no padding and is conflict-free, and the HBM accesses
// of ML / MB are 128-byte runs (four per warp instruction, as in qaoa_sweep.cu).
// A merged sweep re-maps ML -> MA -> MB, cost, MB -> MA -> ML (four exchanges,
// no lane transposes); per tile that is the same number of shared-memory
// instructions as the 16-amplitude flow's two exchanges plus two transposes.
//
// Arithmetic per amplitude: the same fast-mode RX butterflies (rx_form1), cost
// lookup (cmul_np with the even phase table) and scale as fast_tile; only the
// order in which the nine qubits of a set are applied differs (within the
// schedule's 1e-12 tolerance; exact runs never come here).
//
// Reference path replaced: see qaoa_sweep.cu (cost.py:162-176, circuit.py:89-94,
// state.py:110-128, circuit.py:116-121).
#include "qaoa_common.cuh"
#include "qaoa_sweep.h"
#include "qaoa_tile.cuh"

namespace qb {
namespace s8 {

constexpr int kT = 512;  // threads per CTA
constexpr int kR = 8;    // amplitudes per thread

// Tile index of register r of thread tid in mapping M (0 = ML, 1 = MA, 2 = MB).
template <int M>
__host__ __device__ constexpr int tidx(int tid, int r) {
  return M == 0 ? (tid | (r << 9))
       : M == 1 ? ((tid & 63) | ((tid >> 6) << 9) | (r << 6))
                : ((tid & 7) | ((tid >> 3) << 6) | (r << 3));
}
template <int M>
__host__ __device__ constexpr int reg_base() {  // tile bit of register bit 0
  return M == 0 ? 9 : (M == 1 ? 6 : 3);
}

// Registers of mapping A -> mapping B through the (unpadded) exchange buffer.
// Every thread later writes (in mapping B) exactly the slots it read here, so
// one barrier per exchange suffices (as in qaoa_tile.cuh).
template <int A, int B>
__device__ __forceinline__ void xchg(double2* buf, int tid, double2 (&v)[kR]) {
  double2* w = buf + tidx<A>(tid, 0);
#pragma unroll
  for (int r = 0; r < kR; ++r) w[tidx<A>(0, r)] = v[r];
  __syncthreads();
  const double2* rd = buf + tidx<B>(tid, 0);
#pragma unroll
  for (int r = 0; r < kR; ++r) v[r] = rd[tidx<B>(0, r)];
}

__device__ __forceinline__ void rx3(double2 (&v)[kR], double t) {
#pragma unroll
  for (int K = 0; K < 3; ++K)
#pragma unroll
    for (int r = 0; r < kR; ++r)
      if (!(r & (1 << K))) rx_form1(v[r], v[r | (1 << K)], t);
}

// C(x) of the 8 registers of mapping M from the tile's cut basis (see cut_parts
// in qaoa_tile.cuh; exact integers).
template <int M>
__device__ __forceinline__ void cut8(const CutBasis* cb, int (&c)[kR], int tid) {
  int pk[12];
  const int4* p4 = reinterpret_cast<const int4*>(cb->pk);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int4 w = p4[i];
    pk[4 * i] = w.x; pk[4 * i + 1] = w.y; pk[4 * i + 2] = w.z; pk[4 * i + 3] = w.w;
  }
  const int2 kt = *reinterpret_cast<const int2*>(&cb->K);
  const int T = tidx<M>(tid, 0) ^ kt.y;
  int c0 = kt.x;
#pragma unroll
  for (int k = 0; k < 12; ++k)
    if ((T >> k) & 1) c0 += (pk[k] >> 16) - __popc(pk[k] & T);
  constexpr int b = reg_base<M>();
  int d[3], al[3], sg[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    al[j] = pk[b + j] & 0xFFF;
    sg[j] = ((T >> (b + j)) & 1) ? -1 : 1;
    d[j] = sg[j] * ((pk[b + j] >> 16) - 2 * __popc(al[j] & T));
  }
  const int a01 = 2 * sg[0] * sg[1] * ((al[0] >> (b + 1)) & 1);
  const int a02 = 2 * sg[0] * sg[2] * ((al[0] >> (b + 2)) & 1);
  const int a12 = 2 * sg[1] * sg[2] * ((al[1] >> (b + 2)) & 1);
  c[0] = c0;
  c[1] = c0 + d[0];
  c[2] = c0 + d[1];
  c[3] = c[1] + d[1] - a01;
  c[4] = c0 + d[2];
  c[5] = c[1] + d[2] - a02;
  c[6] = c[2] + d[2] - a12;
  c[7] = c[3] + d[2] - a02 - a12;
}

template <int M>
__device__ __forceinline__ void cost8(double2 (&v)[kR], const CutBasis* cb, const double2* __restrict__ tab,
                                      int e, int tid) {
  int c[kR];
  cut8<M>(cb, c, tid);
#pragma unroll
  for (int r = 0; r < kR; ++r) v[r] = cmul_np(v[r], ld_phase(tab + (e - c[r])));
}

template <int M>
__device__ __forceinline__ double expect8(const double2 (&v)[kR], const CutBasis* cb, int tid) {
  int c[kR];
  cut8<M>(cb, c, tid);
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < kR; ++r) acc += (v[r].x * v[r].x + v[r].y * v[r].y) * (double)c[r];
  return acc;
}

// Global address of register r in mapping M (C = 3): tile index t -> (t & 7) +
// (t >> 3) * Q; the register part is a multiple of Q.
template <int M>
__device__ __forceinline__ double2* reg_ptr(double2* tile0, uint64_t Q, int tid, int r) {
  const int t = tidx<M>(tid, 0);
  const uint64_t thr = (uint64_t)(t & 7) + (uint64_t)(t >> 3) * Q;
  return tile0 + thr + (uint64_t)(tidx<M>(0, r) >> 3) * Q;
}

}  // namespace s8

// FLOW 1: [cost] RX(set); FLOW 2: [cost] RX(set) -> cost -> RX(set).  C = 3,
// fast schedule, unweighted, in place (see qaoa_sweep.cu for the flags).
template <bool WIDE, int FLOW>
__global__ void __launch_bounds__(s8::kT, 2) sweep8_kernel(const __grid_constant__ SweepArgs a) {
  using namespace s8;
  extern __shared__ __align__(16) unsigned char smem_raw8[];
  double2* buf = reinterpret_cast<double2*>(smem_raw8);  // kTile slots
  __shared__ CutBasis cb;
  __shared__ double red_scratch[kT / 32];
  constexpr int C = 3;
  const uint32_t flags = a.flags;
  const int tid = threadIdx.x;
  const int q = a.q;
  const uint64_t Q = 1ull << q;
  const uint64_t tile = (uint64_t)a.tile_lo + blockIdx.x;
  const uint64_t base = tile_base<C>(tile, q);
  double2* __restrict__ amps = a.amps;

  double2 v[kR];
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
    double2* p = reg_ptr<0>(amps + base, Q, tid, 0);
    const uint64_t s = 64ull * Q;  // register stride of ML (tile bit 9 = physical bit q + 6)
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = ld_tile(p + r * s);
  }
  const bool need_cut = flags & (kPreCost | kMidCost | kExpect);
  if (need_cut) {
    if (tid < 32) cut_basis<WIDE, C>(a, base, q, &cb);
    // otherwise published by the first exchange's barrier
    if (flags & kPreCost) __syncthreads();
  }
  const int e = a.g.tot_edge;
  const double t1 = a.rx1.a, t2 = a.rx2.a;
  if (flags & kPreCost) cost8<0>(v, &cb, a.table, e, tid);
  rx3(v, t1);
  xchg<0, 1>(buf, tid, v);
  rx3(v, t1);
  xchg<1, 2>(buf, tid, v);
  rx3(v, t1);
  double acc = 0.0;
  if (FLOW == 2) {
    cost8<2>(v, &cb, a.table2, e, tid);
    rx3(v, t2);
    xchg<2, 1>(buf, tid, v);
    rx3(v, t2);
    xchg<1, 0>(buf, tid, v);
    rx3(v, t2);
  }
  constexpr int last = FLOW == 2 ? 0 : 2;
  if (flags & kScale) {
#pragma unroll
    for (int r = 0; r < kR; ++r) v[r] = cmul_np(v[r], a.scale);
  }
  if (flags & kExpect) acc = expect8<last>(v, &cb, tid);
  if (!(flags & kNoStore)) {
    double2* p = reg_ptr<last>(amps + base, Q, tid, 0);
    const uint64_t s = (uint64_t)(tidx<last>(0, 1) >> 3) * Q;
#pragma unroll
    for (int r = 0; r < kR; ++r) __stcs(p + r * s, v[r]);
  }
  if (flags & kExpect) {
    const double t = block_sum<kT>(acc, red_scratch);
    if (threadIdx.x == 0) a.partials[tile] = t;
  }
}

bool sweep8_eligible(const SweepArgs& a) {
  return a.carry == 3 && !(a.flags & (kExact | kWeighted | kMirror)) && !a.out && a.ntiles >= 1 &&
         (a.flags & kStage1);
}

template <bool WIDE, int FLOW>
static cudaError_t launch8_one(const SweepArgs& a, int grid, cudaStream_t s) {
  constexpr int smem = kTile * (int)sizeof(double2);
  static unsigned long long configured = 0;  // bit d = device d done
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(sweep8_kernel<WIDE, FLOW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e != cudaSuccess) return e;
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  sweep8_kernel<WIDE, FLOW><<<grid, s8::kT, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sweep8(const SweepArgs& a, int grid, cudaStream_t s) {
  if (!sweep8_eligible(a)) return cudaErrorInvalidValue;
  const bool f2 = a.flags & kStage2;
  if (a.g.n_nodes > 32) return f2 ? launch8_one<true, 2>(a, grid, s) : launch8_one<true, 1>(a, grid, s);
  return f2 ? launch8_one<false, 2>(a, grid, s) : launch8_one<false, 1>(a, grid, s);
}

}  // namespace qb
