// dsmem_probe.cu -- go/no-go probe for cluster tiles (tooling, not product):
// how fast can a thread-block cluster re-map a tile held in its CTAs' shared
// memory when the bits being re-mapped cross CTAs (distributed shared memory)?
// A 2^17-amplitude tile (2 MiB) over 16 CTAs would let N=30 run two qubit sets
// per level (17 + 13) instead of three, halving the HBM sweeps, but every
// re-map of a cross-CTA bit becomes an all-to-all over DSMEM.
//
// Each CTA holds A complex128 amplitudes in registers (256 threads x A/256);
// one "exchange" writes every amplitude to its destination slot in a (possibly
// remote) CTA's receive buffer, synchronises the cluster and reads its own
// receive buffer back.  CL = 1 is the local shared-memory exchange the sweeps
// use today.  Reports the time per exchange and the shared-memory bytes per SM
// per clock (write + read).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 tools/dsmem_probe.cu -o tools/dsmem_probe
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>

namespace cg = cooperative_groups;

template <int R>  // amplitudes per thread
__global__ void __launch_bounds__(256, 1) a2a_kernel(int iters, int remote_frac_log2, double* sink) {
  extern __shared__ double2 recv[];  // [A] receive buffer, A = 256 R
  cg::cluster_group cl = cg::this_cluster();
  const int cls = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int A = 256 * R;
  double2 v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = make_double2(threadIdx.x + r, rank);
  cl.sync();
  for (int it = 0; it < iters; ++it) {
    // element e = r * 256 + tid of this CTA goes to CTA (e / (A / cls)) when all
    // bits cross (remote_frac_log2 = log2 cls), slot rank * (A / cls) + e % (A / cls)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = r * 256 + threadIdx.x;
      const int chunk = A / cls;
      const int dst = e / chunk;
      const int slot = rank * chunk + (e % chunk);
      double2* p = cl.map_shared_rank(recv, dst);
      p[slot ^ (threadIdx.x & 0)] = v[r];
    }
    cl.sync();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double2 x = recv[r * 256 + threadIdx.x];
      v[r].x = x.y * 0.5 + x.x;
      v[r].y = x.x * 0.5 - x.y;
    }
    cl.sync();
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) s += v[r].x + v[r].y;
  if (s == 12345.678) sink[0] = s;
  (void)remote_frac_log2;
}

template <int R>
static void run(int cls, int iters) {
  const int A = 256 * R;
  const size_t smem = (size_t)A * sizeof(double2);
  cudaFuncSetAttribute(a2a_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(a2a_kernel<R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cls;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  int max_clusters = 0;
  cfg.gridDim = dim3(cls);
  cudaOccupancyMaxActiveClusters(&max_clusters, (void*)a2a_kernel<R>, &cfg);
  const int grid = max_clusters > 0 ? max_clusters * cls : (sms / cls) * cls;
  cfg.gridDim = dim3(grid);
  double* sink;
  cudaMalloc(&sink, 8);
  cudaLaunchKernelEx(&cfg, a2a_kernel<R>, 1, 0, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, a2a_kernel<R>, iters, 0, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double per_ex_us = ms * 1e3 / iters;
  // bytes through each SM's shared memory per exchange: A x 16 B written (by
  // some CTA) + A x 16 B read
  const double bytes = 2.0 * A * 16.0;
  const double cycles = per_ex_us * 1e-6 * clk_khz * 1e3;
  printf("tile %7d amps/CTA x cluster %2d (%4d CTAs resident, %3d KB smem): %.3f us per exchange, "
         "%.1f B/clk/SM (max clock) %s\n",
         A, cls, grid, (int)(smem >> 10), per_ex_us, bytes / cycles, cudaGetErrorString(err));
  cudaFree(sink);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 2000;
  for (int cls : {1, 2, 4, 8, 16}) run<16>(cls, iters);   // 4096 amps (64 KB) per CTA
  for (int cls : {1, 2, 4, 8, 16}) run<32>(cls, iters);   // 8192 amps (128 KB) per CTA
  return 0;
}
