// membench.cu -- calibration: in-place read+write of a 2^n complex128 state in
// the tile access pattern of the sweep kernel (runs of 2^C amplitudes, the other
// tile bits at q..), with no arithmetic.  Measures the HBM ceiling per pattern.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/membench.cu -o membench
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

template <int C>
__device__ __forceinline__ uint64_t tile_off(int t, uint64_t Q) {
  if (C >= 12) return (uint64_t)t;
  return (uint64_t)(t & ((1 << C) - 1)) + (uint64_t)(t >> C) * Q;
}

// each thread: 16 amps of mapping M2 (t = tid | r << 8); ITEMS tiles per CTA in flight
template <int C, int MODE>
__global__ void __launch_bounds__(256) copy_kernel(double2* amps, int n, int q, int64_t ntiles) {
  const int tid = threadIdx.x;
  const uint64_t Q = 1ull << (C >= 12 ? 0 : q);
  const int low_bits = C >= 12 ? 0 : q - C;
  const uint64_t low_mask = (1ull << low_bits) - 1;
  const int high_shift = C >= 12 ? 12 : q + 12 - C;
  const uint64_t tb = tile_off<C>(tid, Q);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = C >= 12 ? ((uint64_t)tile << 12)
                                  : ((((uint64_t)tile & low_mask) << C) | (((uint64_t)tile >> low_bits) << high_shift));
    double2 v[16];
    const double2* src = amps + base + tb;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = __ldcs(src + tile_off<C>(r << 8, Q));
#pragma unroll
    for (int r = 0; r < 16; ++r) { v[r].x *= 1.0000001; }
    double2* dst = amps + base + tb;
#pragma unroll
    for (int r = 0; r < 16; ++r) __stcs(dst + tile_off<C>(r << 8, Q), v[r]);
  }
}

template <int C>
float run(double2* d, int n, int q, int grid) {
  const int64_t ntiles = 1ll << (n - 12);
  if (grid <= 0) grid = (int)ntiles;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  copy_kernel<C, 0><<<grid, 256>>>(d, n, q, ntiles);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) copy_kernel<C, 0><<<grid, 256>>>(d, n, q, ntiles);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 30;
  double2* d;
  cudaMalloc(&d, sizeof(double2) << n);
  cudaMemset(d, 0, sizeof(double2) << n);
  const double bytes = 32.0 * (double)(1ull << n);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g : {0, 2 * sms, 4 * sms, 8 * sms}) {
    float t12 = run<12>(d, n, 0, g);
    float t3 = run<3>(d, n, n - 9, g);
    float t3m = run<3>(d, n, 12, g);
    float t4 = run<4>(d, n, n - 8, g);
    float t5 = run<5>(d, n, n - 7, g);
    float t6 = run<6>(d, n, n - 6, g);
    printf("n=%d grid=%d  C12 %.0f  C3(top) %.0f  C3(q=12) %.0f  C4 %.0f  C5 %.0f  C6 %.0f GB/s\n", n, g,
           bytes / t12 / 1e6, bytes / t3 / 1e6, bytes / t3m / 1e6, bytes / t4 / 1e6, bytes / t5 / 1e6,
           bytes / t6 / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
