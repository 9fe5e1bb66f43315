/*
 * qaoa_b200.h -- C ABI of the B200-native QAOA Max-Cut state-vector engine.
 *
 * This is the drop-in boundary for the reference's hot path
 *   simulate(g, params, backend="bitwise")  ->  expectation(g, s)
 * (reference: pkg/src/qaoa_maxcut/circuit.py:97-121).  Plain C types only:
 * pointers, sizes, doubles.  Every call is synchronous on the context's stream
 * unless noted, returns QAOA_OK (0) on success or a negative QAOA_E* code, and
 * leaves a message for qaoa_last_error().  The Python package
 * paper_2312_03019_b200 binds these with ctypes and maps the codes onto the
 * reference's exceptions (ValueError / IndexError with the same substrings).
 *
 * Layout: the state is complex128, interleaved (re, im) doubles, bit i of the
 * basis index = qubit i (reference state.py:3-4), resident in HBM and owned
 * by the context.  Host arrays passed in are copied during the call.
 */
#ifndef QAOA_B200_H
#define QAOA_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define QAOA_API __attribute__((visibility("default")))
#else
#define QAOA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define QAOA_OK 0
#define QAOA_E_INVALID (-1)   /* bad argument -> ValueError                      */
#define QAOA_E_RANGE (-2)     /* qubit index out of range -> IndexError          */
#define QAOA_E_CUDA (-3)      /* CUDA runtime / launch failure -> RuntimeError   */
#define QAOA_E_NOMEM (-4)     /* device allocation failed -> MemoryError         */
#define QAOA_E_STATE (-5)     /* call order (no graph / no state) -> RuntimeError */

/* ---- run flags (qaoa_run_layers) ------------------------------------------ */
#define QAOA_RUN_EXACT 0x1          /* bit-exact reference arithmetic and qubit order  */
#define QAOA_RUN_FROM_STATE 0x2     /* start from the resident state, not |+>^n         */
#define QAOA_RUN_EXPECTATION 0x4    /* fuse <C> into the last sweep (qaoa_expectation)  */
#define QAOA_RUN_TIMING 0x8         /* record per-launch CUDA-event times               */
#define QAOA_RUN_SHARDED 0x10       /* qaoa_run_begin: exchange points after S_0 of every level */
#define QAOA_RUN_MIRROR 0x40        /* symmetric half state (graph of n_local + 1 nodes).
                                       With QAOA_RUN_SHARDED: exact runs put the exchange point
                                       after the LAST qubit set of each level (the virtual top
                                       qubit, qaoa_mirror_rx).  Without it (qaoa_run_layers, fast
                                       schedule): the low set becomes the mirror low set, local
                                       qubits 0..10 plus the virtual top qubit in one sweep */
#define QAOA_RUN_EXPECT_ONLY 0x20   /* with QAOA_RUN_EXPECTATION: the last sweep only reads (16 B
                                       instead of 32 B per amplitude); the state is left unusable
                                       (amplitude reads and QAOA_RUN_FROM_STATE then fail) */

typedef struct qaoa_ctx qaoa_ctx;

/* Last error message of the calling thread ("" when none). */
QAOA_API const char* qaoa_last_error(void);

/* Library version string, e.g. "qaoa_b200 0.1 sm_100a". */
QAOA_API const char* qaoa_version(void);

/* Number of visible CUDA devices (0 on a host without a GPU; never fails). */
QAOA_API int qaoa_device_count(void);

/* Create a context holding a 2^n_qubits complex128 state on `device`.
 * Replaces the state allocation of StateVector / init_zero_state
 * (reference state.py:43-52, :66-72); the memory guard of
 * check_qubit_budget (state.py:55-63) is enforced by the caller, the library
 * only refuses sizes that do not fit the device (QAOA_E_NOMEM).
 * `stream` may be NULL (the library creates its own non-blocking stream) or a
 * cudaStream_t owned by the caller (e.g. torch.cuda.current_stream()). */
QAOA_API int qaoa_create(int n_qubits, int device, void* stream, qaoa_ctx** out);

/* As qaoa_create, but the state lives in caller-owned device memory of at least
 * 16 * 2^n_qubits bytes (e.g. a torch tensor used for NCCL exchanges). */
QAOA_API int qaoa_create_external(int n_qubits, int device, void* stream, void* device_amps,
                         qaoa_ctx** out);

QAOA_API void qaoa_destroy(qaoa_ctx* ctx);

/* Raw device pointer of the state (interleaved re, im doubles). */
QAOA_API void* qaoa_state_ptr(qaoa_ctx* ctx);

/* Use `stream` (a cudaStream_t) for all later launches. */
QAOA_API int qaoa_set_stream(qaoa_ctx* ctx, void* stream);

/* Graph in the reference's format: row_mask[i] has bit j set iff edge (i, j),
 * i < j (Graph.row_mask, graph.py:57-59); tot_edge = Graph.tot_edge.  The
 * context's qubits are global node bits [0, n_local) of a larger register
 * whose top bits are fixed to `x_hi` (0 for an unsharded state); n_nodes is the
 * node count of the whole graph.  Replaces plan_for / CompressedCostPlan
 * (cost.py:66-108).  Does not build the cut table (see qaoa_build_cut_table). */
QAOA_API int qaoa_set_graph(qaoa_ctx* ctx, int n_nodes, const uint64_t* row_mask, int tot_edge,
                   uint64_t x_hi);

/* Launch control (circuit.py:42-48): every amplitude = sqrt(1/2^n_nodes). */
QAOA_API int qaoa_init_uniform(qaoa_ctx* ctx);

/* Copy host amplitudes [offset, offset+count) in / out (interleaved re, im). */
QAOA_API int qaoa_write_amplitudes(qaoa_ctx* ctx, uint64_t offset, uint64_t count, const double* src);
QAOA_API int qaoa_read_amplitudes(qaoa_ctx* ctx, uint64_t offset, uint64_t count, double* dst);

/* Unweighted cost layer (apply_cost_bitwise, cost.py:162-176):
 * amp[x] *= table[2E - 2C(x)], table = _phase_table(E, gamma) (cost.py:136-139)
 * given as 2E+1 interleaved complex doubles.  Bit-exact (FMA-form multiply). */
QAOA_API int qaoa_apply_cost(qaoa_ctx* ctx, const double* phase_table);

/* Single-qubit RX(theta) (apply_rx, state.py:110-128): c = cos(theta/2),
 * s = sin(theta/2).  Bit-exact (products rounded separately). */
QAOA_API int qaoa_apply_rx(qaoa_ctx* ctx, int qubit, double c, double s);

/* Symmetric half state.  MaxCut QAOA states from launch control (or the
 * Hadamard chain) keep psi(x) == psi(~x) bit for bit: the uniform start is
 * symmetric, C(x) == C(~x), and every RX butterfly commutes with the global
 * flip (its sums are the same products added in the other order).  A context
 * of n_local qubits with a graph of n_local + 1 nodes then stores the half
 * x_top = 0 of an (n_local + 1)-qubit state; the top qubit's RX pairs stored
 * index y with y ^ (2^n_local - 1).  qaoa_mirror_rx applies that RX (rx and
 * factor as returned by qaoa_run_exchange_info for the level) in one in-place
 * pass.  Driven by the host at the exchange points of a qaoa_run_begin(...,
 * QAOA_RUN_SHARDED | QAOA_RUN_MIRROR) run; <C> and the norm of the full state
 * are twice the half's.  Fast runs need no host loop and no extra pass:
 * qaoa_run_layers(..., QAOA_RUN_MIRROR) folds the virtual qubit into the low-set
 * sweeps (tile = stored block u plus block ~u read backwards). */
QAOA_API int qaoa_mirror_rx(qaoa_ctx* ctx, const double* rx, const double* factor);

/* Gate-level baseline (the reference's default backend "baseline" and
 * init_state(launch_control=False), circuit.py:57-62,76-80).
 * qaoa_init_basis: |index> (init_zero_state, state.py:66-72, index 0); resets
 * the complement mask.  qaoa_apply_h: Hadamard (apply_h, state.py:91-107),
 * (a +- b) * (1/sqrt 2) rounded as the reference does.  qaoa_apply_rzz: RZZ
 * (apply_rzz, state.py:131-149) with phases = {e_same.re, e_same.im, e_diff.re,
 * e_diff.im} formed by the caller as the reference forms them
 * (np.exp(-+0.5j*theta)); FMA-form complex multiply.  All bit-exact. */
QAOA_API int qaoa_init_basis(qaoa_ctx* ctx, uint64_t index);
QAOA_API int qaoa_apply_h(qaoa_ctx* ctx, int qubit);
QAOA_API int qaoa_apply_rzz(qaoa_ctx* ctx, int q1, int q2, const double* phases);

/* Per-index edge sums over the edge list of qaoa_set_weights, in edge order,
 * for true indices x_hi | [offset, offset + count): kind 0 = signed rotation
 * totals (CompressedCostPlan.rotation_totals, cost.py:77-86), kind 1 = cut
 * values (cut_values_array, graph.py:144-151).  Bit-identical float64. */
QAOA_API int qaoa_edge_values(qaoa_ctx* ctx, int kind, uint64_t offset, uint64_t count, double* out);

/* Mixer layer (apply_mixer_layer, circuit.py:89-94): RX on every local qubit in
 * increasing order, c = cos(-beta/2), s = sin(-beta/2).  Bit-exact. */
QAOA_API int qaoa_apply_mixer(qaoa_ctx* ctx, double c, double s);

/* RX on the contiguous qubit range [q0, q0+count) in ONE fused sweep (count <= 9,
 * q0 >= 12 - count, n >= 12; otherwise per-qubit kernels).  Used by the sharded
 * driver for the qubits that arrive from the shard exchange.  flags:
 * QAOA_RUN_EXACT for reference arithmetic, else the factored fast form (which
 * may toggle the range's bits in the complement mask, see qaoa_get_cmask). */
QAOA_API int qaoa_apply_rx_range(qaoa_ctx* ctx, int q0, int count, double c, double s, int flags);

/* Swapped qubit layout of fast unweighted runs (default -1: on for n >= 26 when
 * the level-boundary merges alternate between two equal-size high qubit sets of
 * 9 qubits (128-B runs; N=30) and a second state buffer fits with 4 GiB to
 * spare; env QAOA_SWAP_LAYOUT=0 / 1 turns the policy off / on for every
 * applicable size; mode 0: never; 1: whenever applicable).  Every low-set sweep then writes out of
 * place with the two sets' bit ranges exchanged, so the top-bit set is always
 * merged at bits 12..; runs end in identity order in the context's own buffer
 * (bit-identical amplitudes; <C> partials summed in a different tile order).
 * Costs a second 16 B x 2^n device buffer, kept until qaoa_destroy. */
QAOA_API int qaoa_set_layout_swap(qaoa_ctx* ctx, int mode);

/* Release the context's optional device buffers: the second state buffer of
 * the swapped layout and the cut table (both are re-allocated on demand). */
QAOA_API int qaoa_trim(qaoa_ctx* ctx);

/* Complement mask of the stored state: the amplitude of true basis index x is
 * stored at physical index x ^ cmask (fast-mode bookkeeping; bits >= n_local are
 * shard bits maintained by a sharded host).  read/write_amplitudes map the local
 * bits themselves. */
QAOA_API int qaoa_get_cmask(qaoa_ctx* ctx, uint64_t* out);
QAOA_API int qaoa_set_cmask(qaoa_ctx* ctx, uint64_t cmask);

/* The fused p-level circuit (simulate(..., "bitwise"), circuit.py:97-113):
 * |+>^n (unless QAOA_RUN_FROM_STATE), then per level l: cost with
 * phase_tables[l] (2E+1 complex), mixer with (c[l], s[l]).
 * QAOA_RUN_EXACT reproduces the reference bit for bit; otherwise the sweeps are
 * re-ordered / merged across levels and the butterflies use a factored form
 * (|error| <= 1e-13 absolute, contract 1e-12).  With QAOA_RUN_EXPECTATION the
 * last sweep also accumulates <C>, retrievable with qaoa_expectation. */
QAOA_API int qaoa_run_layers(qaoa_ctx* ctx, int p, const double* phase_tables, const double* c,
                    const double* s, int flags);

/* <C> = sum_x |amp_x|^2 C(x) (expectation, circuit.py:116-121; graph must be
 * unweighted).  Deterministic: fixed-order block partials.  Returns the value
 * fused by the last qaoa_run_layers(..., QAOA_RUN_EXPECTATION) when the state
 * has not changed since, else runs a read-only reduction. */
QAOA_API int qaoa_expectation(qaoa_ctx* ctx, double* out);

/* Weighted graphs (the reference's "compressed" backend, cost.py:77-86,
 * :147-159): edge list (i, j, w) in the graph's edge order (Graph.edges,
 * graph.py:34-66).  qaoa_apply_cost_weighted multiplies by
 * exp(-i gamma t(x) / 2), t = sum_e w_e (1 - 2 [x_i != x_j]) accumulated in edge
 * order (bit-identical totals; the phase's sincos is within 2 ulp of glibc's).
 * qaoa_expectation_weighted = sum_x |a_x|^2 sum_e w_e [x_i != x_j]
 * (graph.py:144-151).  x includes x_hi / the complement mask like the integer path. */
QAOA_API int qaoa_set_weights(qaoa_ctx* ctx, int m, const int* ei, const int* ej, const double* w);
QAOA_API int qaoa_apply_cost_weighted(qaoa_ctx* ctx, double gamma);
QAOA_API int qaoa_expectation_weighted(qaoa_ctx* ctx, double* out);

/* Sampling support (sample, circuit.py:124-133).  qaoa_block_norms: sum of
 * |amp|^2 over each block of 2^block_bits consecutive TRUE indices (block_bits
 * <= 12) into out[2^(n - block_bits)].  qaoa_sample_blocks: for each group g
 * (one hit block group_block[g] with cumulative base group_base[g] = sum of
 * the preceding blocks), the targets t in [group_off[g], group_off[g+1]) get
 * out_idx = first true index x in the block with base + cumsum(|a|^2)(x) > t
 * (numpy's searchsorted(cdf, u, 'right') on the unnormalised cdf). */
QAOA_API int qaoa_block_norms(qaoa_ctx* ctx, int block_bits, double* out);
/* The context holds the x_n = 0 half of an (n+1)-qubit flip-symmetric state
 * (on = 1; QAOA_RUN_MIRROR runs): qaoa_block_norms / qaoa_sample_blocks then
 * cover the 2^(n+1) virtual indices in true order (the upper half read from
 * the complemented stored indices), the same sums and draws as the full state. */
QAOA_API int qaoa_set_mirror(qaoa_ctx* ctx, int on);
QAOA_API int qaoa_sample_blocks(qaoa_ctx* ctx, int block_bits, int64_t n_groups,
                                const int64_t* group_block, const double* group_base,
                                const int64_t* group_off, const double* targets, int64_t* out_idx);

/* Partial sum of |amp|^2 over the local shard (StateVector.norm, state.py:50-51). */
QAOA_API int qaoa_norm_sq(qaoa_ctx* ctx, double* out);

/* max_x |a_x - b_x| over two equal-size states (max_abs_diff, state.py:152-156). */
QAOA_API int qaoa_max_abs_diff(qaoa_ctx* a, qaoa_ctx* b, double* out);

/* Cut-table builder (CompressedCostPlan.cut_counts, cost.py:88-99): integer C(x)
 * for every local basis state into device memory (uint8 when E <= 255, else
 * uint16).  qaoa_read_cut_table widens [offset, offset+count) to int64. */
QAOA_API int qaoa_build_cut_table(qaoa_ctx* ctx);
QAOA_API int qaoa_read_cut_table(qaoa_ctx* ctx, uint64_t offset, uint64_t count, int64_t* dst);
QAOA_API int qaoa_free_cut_table(qaoa_ctx* ctx);

/* Per-launch device times (ms) of the last qaoa_run_layers run with
 * QAOA_RUN_TIMING (or the one launch of the last qaoa_build_cut_table); returns
 * the number of launches (<= cap written). */
QAOA_API int qaoa_layer_timings(qaoa_ctx* ctx, float* ms, int cap);

/* Number of kernels the last qaoa_run_layers call launched, and the HBM bytes
 * its sweeps moved (read + write, algorithmic). */
QAOA_API int qaoa_last_run_stats(qaoa_ctx* ctx, int* launches, double* hbm_bytes);

/* Block until all work on the context's stream is done. */
QAOA_API int qaoa_synchronize(qaoa_ctx* ctx);

/* ---- shard exchange (multi-GPU, reference has none: SPEC.md:186) ----------
 * Swap physical bits: after the call, local bit `local_bits[k]` of this shard
 * holds what global bit (n_local + k) held (k < g), given the received peer
 * chunks.  The engine exposes pack/unpack so the host can drive NCCL or P2P. */
QAOA_API int qaoa_pack_chunks(qaoa_ctx* ctx, int g, const int* local_bits, void* dst_device);
QAOA_API int qaoa_unpack_chunks(qaoa_ctx* ctx, int g, const int* local_bits, const void* src_device);

/* Weighted graphs, fast schedule: the same fused sweeps as qaoa_run_layers with
 * the compressed backend's cost amp *= exp(-i gamma/2 sum_e w_e z_e(x))
 * (cost.py:147-159) factored per tile (unit-modulus per-edge factors and a
 * tile-internal table) instead of an integer phase table.  gammas[p]; c, s as
 * in qaoa_run_layers; edges from qaoa_set_weights.  Within 1e-12 of the
 * reference (not bit-identical: products instead of the edge-order sum);
 * QAOA_RUN_EXACT / QAOA_RUN_SHARDED are refused.  QAOA_RUN_EXPECTATION fuses
 * the weighted <C> (graph.py:144-151, read by qaoa_expectation_weighted) into
 * the last sweep. */
QAOA_API int qaoa_run_layers_weighted(qaoa_ctx* ctx, int p, const double* gammas, const double* c,
                                      const double* s, int flags);

/* The sweep plan of qaoa_run_layers / qaoa_run_begin for n_local qubits and p
 * levels (flags: QAOA_RUN_EXACT, QAOA_RUN_SHARDED), without a device: writes up
 * to `cap` sweeps as 7 ints each (carry, q, pre-cost level, stage-1 level,
 * mid-cost level, stage-2 level, exchange level; -1 = none) and returns the
 * sweep count (or a negative status). */
QAOA_API int qaoa_plan(int n_local, int p, int flags, int* out, int cap);

/* ---- planned runs in segments (sharded states) -----------------------------
 * qaoa_run_layers = qaoa_run_begin + every qaoa_run_segment + qaoa_run_end.
 * With QAOA_RUN_SHARDED the plan stops after the low qubit set S_0 (local bits
 * 0..11) of every level: segment k is followed by the exchange of
 * qaoa_run_exchange_info(k) (all shards: host barrier, qaoa_exchange, barrier,
 * qaoa_set_graph with the relabelled masks, qaoa_set_cmask), and level flips
 * complement all n_nodes bits of the complement mask.  Requires n_local >= 12. */
QAOA_API int qaoa_run_begin(qaoa_ctx* ctx, int p, const double* phase_tables, const double* c,
                            const double* s, int flags, int* n_segments);
QAOA_API int qaoa_run_segment(qaoa_ctx* ctx, int k);
/* Exchange after segment k: the level whose RX the arriving qubits need, its
 * RX stage (rx[0..2] = a, b, mode: 0 exact (c, s), 1 factored t) and its
 * per-qubit scale factor (factor[0..1] = re, im; 1 in exact mode).  Returns
 * QAOA_E_RANGE when no exchange follows segment k. */
QAOA_API int qaoa_run_exchange_info(qaoa_ctx* ctx, int k, int* level, double* rx, double* factor);
QAOA_API int qaoa_run_end(qaoa_ctx* ctx);
/* Sweep-level control of a planned run (pipelining a sharded exchange with the
 * sweeps around it): sweep i belongs to `segment`, works on the tile geometry
 * (carry, q) -- tiles of 2^carry consecutive amplitudes times the qubits
 * q..q+11-carry (carry 12: 4096 consecutive) -- of `ntiles` tiles, numbered so
 * that the top index bits not mixed by the sweep are the top tile-index bits.
 * qaoa_run_sweep_range launches sweep i on tiles [tile_lo, tile_lo + count)
 * instead of inside qaoa_run_segment (the caller runs every sweep of the
 * segment exactly once, in order per tile).  Unsharded runs that use the
 * swapped layout (qaoa_set_layout_swap) refuse partial ranges of their
 * out-of-place low-set sweeps (QAOA_E_STATE). */
QAOA_API int qaoa_run_sweep_info(qaoa_ctx* ctx, int i, int* segment, int* carry, int* q,
                                 int64_t* ntiles);
QAOA_API int qaoa_run_sweep_range(qaoa_ctx* ctx, int i, int64_t tile_lo, int64_t tile_count);

/* ---- fused exchange + RX over shard pointers ------------------------------
 * G = 2^g shards (g <= 4) of 2^n_local amplitudes; shards[r] is a device
 * pointer to shard r valid on `device` (local buffer, CUDA-IPC mapped peer
 * buffer, or another buffer on the same device for virtual shards).  Swaps
 * global bit k with local bit p0 + k and applies RX (rx as above) to the
 * arriving qubits, multiplying by factor^g; processes y in [y_lo, y_hi) of the
 * 2^(n_local - g) column indices (split them across the ranks).  Stream-ordered
 * on `stream` (NULL: legacy default stream); the caller synchronises the ranks
 * before (all segments done) and after (all writes landed). */
QAOA_API int qaoa_exchange(int device, void* stream, int g, void* const* shards, int n_local, int p0,
                           uint64_t y_lo, uint64_t y_hi, const double* rx, const double* factor);

/* ---- CUDA IPC (one process per GPU) ----------------------------------------
 * 64-byte handle of the context's state buffer; open a peer's handle on
 * `device` (peer access over NVLink) and close it again. */
QAOA_API int qaoa_ipc_handle(qaoa_ctx* ctx, void* handle64);
QAOA_API int qaoa_ipc_open(const void* handle64, int device, void** out_ptr);
QAOA_API int qaoa_ipc_close(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* QAOA_B200_H */
