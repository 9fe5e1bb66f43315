// membench2.cu -- copy ceiling of a 12-bit tile pattern with arbitrary mixed
// bit positions (tooling): bits 0..2 carried (128-B runs) + 9 mixed physical
// bits given on the command line; one tile per CTA, 256 threads x 16 amps,
// in place read + write of a 2^n complex128 state (random data).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/membench2.cu -o tools/membench2
//   tools/membench2 30 12 13 14 15 16 17 18 19 20
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

struct Pat {
  int pos[12];     // physical bit of tile bit k
  int free_pos[40];  // physical bits not in the tile, ascending
  int nfree;
};

__global__ void fill(double2* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31;
    a[i] = make_double2((double)(x & 0xFFFF) * 1e-5, (double)((x >> 16) & 0xFFFF) * 1e-5);
  }
}

__global__ void __launch_bounds__(256) copy_kernel(double2* amps, Pat p) {
  const uint64_t tile = blockIdx.x;
  uint64_t base = 0;
  for (int i = 0; i < p.nfree; ++i) base |= ((tile >> i) & 1ull) << p.free_pos[i];
  const int tid = threadIdx.x;
  uint64_t tb = 0;
  for (int k = 0; k < 8; ++k) tb |= (uint64_t)((tid >> k) & 1) << p.pos[k];
  double2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    uint64_t o = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) o |= (uint64_t)((r >> k) & 1) << p.pos[8 + k];
    v[r] = __ldcs(amps + base + tb + o);
  }
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r].x *= 1.0000001;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    uint64_t o = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) o |= (uint64_t)((r >> k) & 1) << p.pos[8 + k];
    __stcs(amps + base + tb + o, v[r]);
  }
}

int main(int argc, char** argv) {
  const int n = atoi(argv[1]);
  Pat p;
  p.pos[0] = 0; p.pos[1] = 1; p.pos[2] = 2;
  for (int k = 0; k < 9; ++k) p.pos[3 + k] = atoi(argv[2 + k]);
  p.nfree = 0;
  for (int b = 3; b < n; ++b) {
    bool in = false;
    for (int k = 3; k < 12; ++k) in |= p.pos[k] == b;
    if (!in) p.free_pos[p.nfree++] = b;
  }
  double2* d;
  cudaMalloc(&d, sizeof(double2) << n);
  fill<<<4096, 256>>>(d, 1ull << n);
  const unsigned grid = 1u << (n - 12);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  copy_kernel<<<grid, 256>>>(d, p);
  cudaEventRecord(a);
  const int reps = 60;
  for (int i = 0; i < reps; ++i) copy_kernel<<<grid, 256>>>(d, p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("mixed");
  for (int k = 3; k < 12; ++k) printf(" %d", p.pos[k]);
  printf(": %.3f ms = %.0f GB/s (%s)\n", ms, 32.0 * (double)(1ull << n) / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
