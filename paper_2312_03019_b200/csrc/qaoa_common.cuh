// qaoa_common.cuh -- shared device helpers for the B200 QAOA engine.
//
// State layout: complex128 amplitudes as double2 (re, im), bit i of the basis
// index = qubit i (reference pkg/src/qaoa_maxcut/state.py:3-4).  Indices are
// 64-bit (N = 33 on one GPU is 2^33 amplitudes).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qb {

constexpr int kMaxNodes = 64;  // graph.py:15 MASK_BITS

// Graph in physical bit positions.  rm[i]: row mask (edges (i, j), j > i,
// graph.py:57-59); adj[i]: full neighbour mask.  x_hi: fixed high bits of the
// basis index (shard id for a sharded state, 0 otherwise).
// cmask: complement mask of the stored state -- the amplitude of true basis
// index x is stored at physical index x ^ cmask (fast-mode bookkeeping of the
// second factored RX form, see qaoa_capi.cu); cut counts use x_hi ^ cmask ^ local.
struct GraphDev {
  uint64_t rm[kMaxNodes];
  uint64_t adj[kMaxNodes];
  uint64_t x_hi;
  uint64_t cmask;
  int n_nodes;
  int tot_edge;
};

// C(x) = sum_i popcount(rm[i] & (bcast(x_i) ^ x)): the bitwise row step of
// reference cost.py:55-63 / :88-99 (Alg. 3).
template <bool WIDE>
__device__ __forceinline__ int cut_count(uint64_t x, const GraphDev& g) {
  int c = 0;
  if (WIDE) {
#pragma unroll 4
    for (int i = 0; i < g.n_nodes; ++i) {
      const uint64_t b = 0ull - ((x >> i) & 1ull);
      c += __popcll(g.rm[i] & (b ^ x));
    }
  } else {
    const uint32_t x32 = (uint32_t)x;
#pragma unroll 4
    for (int i = 0; i < g.n_nodes; ++i) {
      const uint32_t b = 0u - ((x32 >> i) & 1u);
      c += __popc((uint32_t)g.rm[i] & (b ^ x32));
    }
  }
  return c;
}

// Cut counts of the 16 states x0 ^ (r0 << v0) ^ ... ^ (r3 << v3), r in [0, 16),
// for any x0: C(x0) once, then per flipped node k
//   delta_k = s_k (deg(v_k) - 2 popc(adj[v_k] & x0)),  s_k = +1 if bit v_k of x0
// is 0 else -1, and -2 s_j s_k for every edge between two flipped nodes.
// Bit-exact integer arithmetic.
template <bool WIDE>
__device__ __forceinline__ void cut_counts16(uint64_t x0, const int v[4], const GraphDev& g,
                                             int (&c)[16]) {
  const int c0 = cut_count<WIDE>(x0, g);
  int d[4], sg[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t m = g.adj[v[k]];
    sg[k] = ((x0 >> v[k]) & 1ull) ? -1 : 1;
    d[k] = sg[k] * (__popcll(m) - 2 * __popcll(m & x0));
  }
  const int a01 = 2 * sg[0] * sg[1] * (int)((g.adj[v[0]] >> v[1]) & 1ull);
  const int a02 = 2 * sg[0] * sg[2] * (int)((g.adj[v[0]] >> v[2]) & 1ull);
  const int a03 = 2 * sg[0] * sg[3] * (int)((g.adj[v[0]] >> v[3]) & 1ull);
  const int a12 = 2 * sg[1] * sg[2] * (int)((g.adj[v[1]] >> v[2]) & 1ull);
  const int a13 = 2 * sg[1] * sg[3] * (int)((g.adj[v[1]] >> v[3]) & 1ull);
  const int a23 = 2 * sg[2] * sg[3] * (int)((g.adj[v[2]] >> v[3]) & 1ull);
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

// numpy's FMA-form complex multiply (reference
// cost.py:172 `amps *= phases`): re = fma(ar, pr, -(ai*pi)), im = fma(ar, pi, ai*pr).
__device__ __forceinline__ double2 cmul_np(double2 a, double2 p) {
  double2 r;
  r.x = __fma_rn(a.x, p.x, -__dmul_rn(a.y, p.y));
  r.y = __fma_rn(a.x, p.y, __dmul_rn(a.y, p.x));
  return r;
}

// Reference RX butterfly (state.py:114-124, theta = -beta): each product
// rounded separately, then one add.  c = cos(theta/2), s = sin(theta/2).
__device__ __forceinline__ void rx_exact(double2& a, double2& b, double c, double s) {
  const double ns = -s;
  const double tr = __dadd_rn(__dmul_rn(c, a.x), __dmul_rn(s, b.y));
  const double ti = __dadd_rn(__dmul_rn(c, a.y), __dmul_rn(ns, b.x));
  const double ur = __dadd_rn(__dmul_rn(s, a.y), __dmul_rn(c, b.x));
  const double ui = __dadd_rn(__dmul_rn(ns, a.x), __dmul_rn(c, b.y));
  a.x = tr; a.y = ti; b.x = ur; b.y = ui;
}

// Factored RX (fast mode).  RX = c [[1, -i t], [-i t, 1]] with t = s / c
// (form 1, |c| >= |s|) or RX = (-i s) [[i k, 1], [1, i k]] with k = c / s
// (form 2).  The scalar factor of all N qubits of a level is folded into the
// next level's phase table / the final scale; each output component is one DFMA.
__device__ __forceinline__ void rx_form1(double2& a, double2& b, double t) {
  const double ar = a.x, ai = a.y, br = b.x, bi = b.y;
  a.x = __fma_rn(t, bi, ar);
  a.y = __fma_rn(-t, br, ai);
  b.x = __fma_rn(t, ai, br);
  b.y = __fma_rn(-t, ar, bi);
}
__device__ __forceinline__ void rx_form2(double2& a, double2& b, double k) {
  const double ar = a.x, ai = a.y, br = b.x, bi = b.y;
  a.x = __fma_rn(-k, ai, br);
  a.y = __fma_rn(k, ar, bi);
  b.x = __fma_rn(-k, bi, ar);
  b.y = __fma_rn(k, br, ai);
}

// Butterfly mode of one RX stage: 0 = exact (c, s), 1 = form 1 (t), 2 = form 2 (k).
struct RxStage {
  double a;   // exact: c ; form1: t ; form2: k
  double b;   // exact: s
  int mode;
};

// Deterministic in-block sum of one double per thread (fixed shuffle tree,
// then warps in order).  Result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < THREADS / 32; ++w) t += scratch[w];
  }
  return t;
}

}  // namespace qb
