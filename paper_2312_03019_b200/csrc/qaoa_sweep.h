// qaoa_sweep.h -- host-visible description of one fused sweep launch.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "qaoa_common.cuh"

namespace qb {

enum SweepFlags : uint32_t {
  kGen = 1u << 0,      // no load: every amplitude starts as `gen` (launch control)
  kPreCost = 1u << 1,  // cost phase before the first RX stage
  kStage1 = 1u << 2,   // RX stage 1 on tile bits act1
  kMidCost = 1u << 3,  // cost phase between the two RX stages (fast mode)
  kStage2 = 1u << 4,   // RX stage 2 on tile bits act2 (next level, fast mode)
  kExpect = 1u << 5,   // accumulate sum |a|^2 C(x) into partials[blockIdx.x]
  kScale = 1u << 6,    // multiply by `scale` before storing (fast mode)
  kExact = 1u << 7,    // reference arithmetic + increasing qubit order
  kNoStore = 1u << 8,  // read-only sweep
  kWeighted = 1u << 9, // weighted cost: factored per-edge phases (see apply_wcost)
  kMirror = 1u << 10,  // symmetric half state: RX on the virtual top qubit after the
                       // stage (pairs tile T with tile ~T, a 2-CTA cluster; see qaoa_sweep.cu)
  kGenTab = 1u << 11,  // launch control with `table` = gen x phase table (cost = gather only)
};

struct SweepArgs {
  CUtensorMap map;       // 5-D view of the state, one box = half a tile (TMA loads / prefetch)
  double2* amps;
  const double2* table;  // even phase-table entries (E+1) of the pre-stage cost step
  const double2* table2; // even phase-table entries (E+1) of the mid cost step
  double* partials;      // [grid] block partial sums (kExpect)
  GraphDev g;
  int64_t ntiles;        // 2^(n_local - 12): the tile geometry of the state
  int64_t tile_lo;       // this launch covers tiles [tile_lo, tile_lo + tile_cnt)
  int64_t tile_cnt;      // 0 = all ntiles
  int carry;             // C: tile bits 0..C-1 = physical bits 0..C-1 (12 = low sweep)
  int q;                 // tile bits C..11 = physical bits q..q+11-C (the mixed qubits)
  RxStage rx1, rx2;
  double2 gen;
  double2 scale;
  int table_len;
  uint32_t flags;
  int pf_dist;           // > 0: L2-prefetch tile (this tile + pf_dist) before loading this one
  int pf_tensor;         // prefetch through `map` (2 TMA prefetches) instead of per-run bulk prefetches
  // weighted cost (kWeighted): u_e = exp(-i gamma w_e / 2) of the pre / mid
  // level per edge, the 4096-entry tile-internal phase table of each, the edge
  // endpoints (physical bits) and the per-node incidence lists (CSR)
  const double2* wu1;
  const double2* wu2;
  const double2* wq1;
  const double2* wq2;
  const int2* wedge;
  const int* winc_off;   // [65]
  const int* winc;       // [2 wm] edge ids
  int wm;
  const double* ww;      // [wm] edge weights (weighted <C>)
  const double* wc;      // 4096-entry tile-internal cut weight table of the last sweep's set
  // out-of-place low-set sweep (C = 12, one tile per CTA): tile stored to `out`
  // with physical index bits [sw_lo, sw_lo + sw_m) and [sw_hi, sw_hi + sw_m)
  // swapped (the swapped qubit layout of qaoa_capi.cu); nullptr = in place
  double2* out;
  int sw_lo, sw_hi, sw_m;
  // launch-control sweeps on the TMA-fed kernel: per-tile cut bases built ahead
  // by launch_gen_aux (64 B per tile, indexed by absolute tile); nullptr = warp 0
  // builds each tile's basis in the sweep
  const void* basis_tab;
};
// Launch-control helpers (fast schedule, TMA-fed kernel): the cut basis of every
// tile of [a.tile_lo, a.tile_lo + cnt) into basis_out (kBasisEntryBytes per
// tile) and gen_table[k] = cmul_np(a.gen, a.table[k]) for k < a.table_len (the
// product the sweep would form per amplitude: bit-identical).
constexpr int kBasisEntryBytes = 64;
cudaError_t launch_gen_aux(const SweepArgs& a, void* basis_out, double2* gen_table, cudaStream_t s);
// Tile-internal phase table of one weighted cost level for tile geometry (C, q):
// Q[t] = scale * prod over edges with both endpoints tile nodes of u_e (equal
// true bits) or conj(u_e) (different), t = true tile index.
cudaError_t launch_wq_table(double2* q_out, const int2* wedge, const double2* wu, int wm, int carry,
                            int q, double2 scale, cudaStream_t s);
// Tile-internal weighted cut table: C[t] = sum of w_e over cut edges with both
// endpoints tile nodes (true tile index t), for the fused weighted <C>.
cudaError_t launch_wc_table(double* c_out, const int2* wedge, const double* w, int wm, int carry, int q,
                            cudaStream_t s);
// 5-D tensor map of the state for tile geometry (C, q) (qaoa_sweep_tma.cu).
bool make_tile_map(CUtensorMap* map, void* amps, int n, int C, int q);

size_t sweep_smem_bytes(int table_len);
// Fast-schedule sweeps run on the persistent TMA-fed kernel (qaoa_sweep_tma.cu)
// unless QAOA_SWEEP_IMPL=v4; sweep_grid() = CTAs launched = partials written.
int sweep_impl(const SweepArgs& a);  // 0 one tile per CTA, 1 TMA-fed, 2 TMA in + out
bool sweep_uses_tma(const SweepArgs& a);
void set_sweep_impl(int v);  // force 0 / 1 / 2, or 3 = per-sweep policy (default); tooling / A-B tests
int sweep_grid(const SweepArgs& a);
cudaError_t launch_sweep_tma(const SweepArgs& a, cudaStream_t stream);
// 128 x 32 register geometry for the fast C = 3 sweeps (qaoa_sweep32.cu); the
// policy routes every eligible sweep there (one tile per CTA, like impl 0).
bool sweep32_eligible(const SweepArgs& a);
bool sweep32_selected(const SweepArgs& a);
void set_sweep32(int on);  // -1: QAOA_SWEEP32 (default on), 0 off, 1 on
cudaError_t launch_sweep32(const SweepArgs& a, int grid, cudaStream_t stream);
cudaError_t launch_sweep(const SweepArgs& args, int grid, cudaStream_t stream);

// simple (per-gate / per-element) kernels, qaoa_gates.cu
cudaError_t launch_fill(double2* amps, uint64_t n, double2 v, cudaStream_t s);
cudaError_t launch_basis(double2* amps, uint64_t n, uint64_t index, cudaStream_t s);
cudaError_t launch_mirror_rx(double2* amps, int n_local, RxStage st, double2 scale, int scale_on,
                             cudaStream_t s);
cudaError_t launch_h_gate(double2* amps, int n_local, int q, int flip, cudaStream_t s);
cudaError_t launch_rzz_gate(double2* amps, uint64_t n, uint64_t xbase, int q1, int q2,
                            double2 e_same, double2 e_diff, cudaStream_t s);
cudaError_t launch_edge_values(double* out, uint64_t first, uint64_t count, const int* ei,
                               const int* ej, const double* w, int m, int kind, cudaStream_t s);
cudaError_t launch_cost_gate(double2* amps, uint64_t n, const GraphDev& g, const double2* table,
                             cudaStream_t s);
cudaError_t launch_rx_gate(double2* amps, int n_local, int q, double c, double sn,
                           cudaStream_t s);
// the whole p-level circuit for n <= 11 in one CTA (state in shared memory)
cudaError_t launch_small_run(double2* amps, int n, const GraphDev& g, const double2* tables,
                             const double2* rx, int p, int from_state, double u, int want_expect,
                             double* expect_out, cudaStream_t s);
cudaError_t launch_expectation(const double2* amps, int n_local, const GraphDev& g,
                               double* partials, int grid, cudaStream_t s);
cudaError_t launch_norm_sq(const double2* amps, uint64_t n, double* partials, int grid,
                           cudaStream_t s);
cudaError_t launch_max_abs_diff(const double2* a, const double2* b, uint64_t n, uint64_t xmask,
                                double* partials, int grid, cudaStream_t s);
cudaError_t launch_sum_partials(const double* partials, int n, double* out, int mode_max,
                                cudaStream_t s);
cudaError_t launch_cut_table(void* table, int bytes_per, int n_local, const GraphDev& g,
                             cudaStream_t s);
cudaError_t launch_cut_table_warps(void* table, int bytes_per, int n_local, const GraphDev& g,
                                   cudaStream_t s);  // qaoa_cut_table.cu (n_local >= 11)
cudaError_t launch_pack_chunks(const double2* amps, int n_local, int g, const int* local_bits,
                               double2* dst, cudaStream_t s);
cudaError_t launch_unpack_chunks(double2* amps, int n_local, int g, const int* local_bits,
                                 const double2* src, cudaStream_t s);
cudaError_t launch_cost_weighted(double2* amps, uint64_t n, uint64_t xbase, const int* ei,
                                 const int* ej, const double* w, int m, double gamma,
                                 cudaStream_t s);
cudaError_t launch_expectation_weighted(const double2* amps, uint64_t n, uint64_t xbase,
                                        const int* ei, const int* ej, const double* w, int m,
                                        double* partials, int grid, cudaStream_t s);
cudaError_t launch_block_norms(const double2* amps, int block_bits, uint64_t n_blocks,
                               uint64_t lmask, uint64_t fold, double* out, cudaStream_t s);
cudaError_t launch_sample_blocks(const double2* amps, int block_bits, uint64_t lmask, uint64_t fold,
                                 int64_t n_groups, const int64_t* gblock, const double* gbase,
                                 const int64_t* goff, const double* targets, int64_t* out,
                                 cudaStream_t s);
int reduce_grid();

// fused global<->local exchange + RX of the arriving qubits (qaoa_exchange.cu)
constexpr int kMaxShards = 16;
struct ExchangeArgs {
  double2* shards[kMaxShards];  // G = 2^g shard bases, valid on the launching device
  int g;                        // global (shard) bits
  int p0;                       // swapped local bits p0 .. p0+g-1
  uint64_t y_lo, y_hi;          // range of y (local index without bits p0..) handled here
  RxStage rx;                   // mode 0: exact (c, s); 1: factored form 1 (t)
  double2 scale;                // applied after the butterflies when scale_on
  int scale_on;
};
cudaError_t launch_exchange(const ExchangeArgs& a, cudaStream_t s);

}  // namespace qb
