// sweep_probe.cu -- timing decomposition of the fused sweep kinds (tooling, not
// product): each sweep kind of an N-qubit fast-mode run is timed normally, with
// no HBM load (kGen), with no HBM store (kNoStore) and with neither (pure
// on-chip work: FP64 butterflies, shared-memory exchanges, cut counts).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2312_03019_b200/csrc tools/sweep_probe.cu \
//        paper_2312_03019_b200/csrc/qaoa_sweep.cu paper_2312_03019_b200/csrc/qaoa_sweep32.cu paper_2312_03019_b200/csrc/qaoa_sweep_tma.cu \
//        paper_2312_03019_b200/csrc/qaoa_cut_table.cu -o tools/sweep_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "qaoa_sweep.h"

using namespace qb;


static float time_sweep(const SweepArgs& a, int grid, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch_sweep(a, grid, 0);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch_sweep(a, grid, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    exit(1);
  }
  return ms / reps;
}

// v4 vs TMA-fed kernel on the same random input, every sweep kind and set of
// the planner at sizes n_lo..n_hi; prints max |difference| (must be 0: both
// run the same arithmetic in the same order).
static int check_mode(int n_lo, int n_hi, int other) {
  int bad = 0;
  for (int n = n_lo; n <= n_hi; ++n) {
    const uint64_t size = 1ull << n;
    double2 *x, *y4, *y5;
    cudaMalloc(&x, 16 * size);
    cudaMalloc(&y4, 16 * size);
    cudaMalloc(&y5, 16 * size);
    double2* h = (double2*)malloc(16 * size);
    double2* h4 = (double2*)malloc(16 * size);
    srand(n);
    for (uint64_t i = 0; i < size; ++i) h[i] = make_double2(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
    cudaMemcpy(x, h, 16 * size, cudaMemcpyHostToDevice);
    GraphDev g;
    memset(&g, 0, sizeof(g));
    g.n_nodes = n;
    int E = 0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j)
        if (((i * 7 + j * 13) % 5) == 0) { g.rm[i] |= 1ull << j; g.adj[i] |= 1ull << j; g.adj[j] |= 1ull << i; ++E; }
    g.tot_edge = E;
    g.cmask = 0x5ull & (size - 1);
    double2* tab;
    cudaMalloc(&tab, sizeof(double2) * (E + 1) * 2);
    double2* ht = (double2*)malloc(sizeof(double2) * (E + 1) * 2);
    for (int k = 0; k < 2 * (E + 1); ++k) ht[k] = make_double2(cos(0.37 * k), sin(0.37 * k));
    cudaMemcpy(tab, ht, sizeof(double2) * (E + 1) * 2, cudaMemcpyHostToDevice);
    double* part;
    cudaMalloc(&part, sizeof(double) * (size >> 12));
    // sets as the planner makes them
    int carry[8], qs[8], ns = 0;
    carry[ns] = 12; qs[ns++] = 0;
    const int rem = n - 12;
    const int chunks = (rem + 8) / 9;
    int next = 12;
    for (int ci = 0; ci < chunks; ++ci) {
      const int m = rem / chunks + (ci < rem % chunks ? 1 : 0);
      carry[ns] = 12 - m; qs[ns++] = next; next += m;
    }
    const uint32_t kinds[] = {kStage1, kPreCost | kStage1, kStage1 | kMidCost | kStage2,
                              kPreCost | kStage1 | kMidCost | kStage2 | kScale | kExpect,
                              kGen | kPreCost | kStage1, kStage1 | kExpect};
    for (int si = 0; si < ns; ++si) {
      for (uint32_t fl : kinds) {
        SweepArgs a;
        memset(&a, 0, sizeof(a));
        a.table = tab; a.table2 = tab + (E + 1); a.partials = part; a.g = g;
        a.ntiles = size >> 12; a.carry = carry[si]; a.q = qs[si];
        a.rx1 = RxStage{0.3, 0.0, 1}; a.rx2 = RxStage{-0.7, 0.0, 1};
        a.gen = make_double2(0.01, -0.02); a.scale = make_double2(0.9, 0.1);
        a.table_len = E + 1; a.flags = fl;
        double e4 = 0, e5 = 0;
        for (int impl = 0; impl < 2; ++impl) {
          double2* y = impl ? y5 : y4;
          cudaMemcpy(y, x, 16 * size, cudaMemcpyDeviceToDevice);
          a.amps = y;
          // other == 32: the 128 x 32 C = 3 kernel against the 256 x 16 one
          set_sweep32(impl && other == 32 ? 1 : 0);
          set_sweep_impl(impl ? (other == 32 ? 0 : other) : 0);
          launch_sweep(a, (int)a.ntiles, 0);
          cudaError_t err = cudaDeviceSynchronize();
          if (err != cudaSuccess) { printf("n=%d error %s\n", n, cudaGetErrorString(err)); return 1; }
          if (fl & kExpect) {
            const int np = (int)a.ntiles;  // one partial per tile
            double* hp = (double*)malloc(sizeof(double) * np);
            cudaMemcpy(hp, part, sizeof(double) * np, cudaMemcpyDeviceToHost);
            double s = 0; for (int i = 0; i < np; ++i) s += hp[i];
            (impl ? e5 : e4) = s; free(hp);
          }
        }
        cudaMemcpy(h4, y4, 16 * size, cudaMemcpyDeviceToHost);
        cudaMemcpy(h, y5, 16 * size, cudaMemcpyDeviceToHost);
        double md = 0; uint64_t arg = 0, nbad = 0;
        for (uint64_t i = 0; i < size; ++i) {
          double d = fabs(h4[i].x - h[i].x) + fabs(h4[i].y - h[i].y);
          if (d > (other == 32 ? 1e-13 : 0.0)) {
            if (nbad < 8) printf("   diff at %llu (tile-internal 0x%03llx)\n", (unsigned long long)i, (unsigned long long)(i & 4095));
            ++nbad;
          }
          if (d > md) { md = d; arg = i; }
        }
        if (nbad) printf("   %llu differing amplitudes\n", (unsigned long long)nbad);
        // the 128 x 32 experiment (other == 32) applies a set's qubits in another order
        const bool ok = md <= (other == 32 ? 1e-13 : 0.0) && fabs(e4 - e5) <= 1e-12 * fabs(e4);
        bad += !ok;
        printf("n=%d set C=%2d q=%2d flags=0x%03x maxdiff=%.3e (at %llu) expect %.15g vs %.15g %s\n", n, carry[si], qs[si], fl, md,
               (unsigned long long)arg, e4, e5, ok ? "OK" : "FAIL");
      }
    }
    cudaMemcpy(h, x, 16 * size, cudaMemcpyDeviceToHost);
    cudaFree(x); cudaFree(y4); cudaFree(y5); cudaFree(tab); cudaFree(part);
    free(h); free(h4); free(ht);
  }
  printf("check: %d failures\n", bad);
  return bad != 0;
}

// K1 timing: sweep_probe cut N REPS [dense]: the cut-table builder alone.
static int cut_mode(int n, int reps, int dense) {
  GraphDev g;
  memset(&g, 0, sizeof(g));
  g.n_nodes = n;
  int E = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const bool e = dense ? (((i * 131 + j * 71) % 7) < (dense == 2 ? 3 : 4)) : (j == i + 1 || (j == i + n / 2 && i < n / 2));
      if (e) { g.rm[i] |= 1ull << j; g.adj[i] |= 1ull << j; g.adj[j] |= 1ull << i; ++E; }
    }
  g.tot_edge = E;
  const int bpe = E <= 255 ? 1 : 2;
  void* t;
  if (cudaMalloc(&t, (size_t)bpe << n) != cudaSuccess) return 1;
  launch_cut_table_warps(t, bpe, n, g, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) launch_cut_table_warps(t, bpe, n, g, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("cut table n=%d E=%d (%d B/state): %.3f ms = %.3e states/s = %.0f GB/s (%s)\n", n, E, bpe, ms,
         (double)(1ull << n) / (ms * 1e-3), (double)((size_t)bpe << n) / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Realistic amplitudes (power draw depends on the data: an all-zero state draws
// ~25% less and hides the 1000 W cap the real bench runs into).
__global__ void fill_random(double2* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    const double s = 1.0 / 32768.0;
    a[i] = make_double2(s * ((double)(x & 0xFFFFFF) / 16777216.0 - 0.5),
                        s * ((double)((x >> 24) & 0xFFFFFF) / 16777216.0 - 0.5));
  }
}

// Concurrency probe: sweep_probe conc N REPS: the low-set sweep S0 on the tiles
// of one half of the state and the merged set-1 sweep on the other half
// (disjoint amplitudes: S0 tiles [0, T/2) have bit N-1 = 0, merged tiles
// [T/2, T) have bit N-1 = 1), once back to back on one stream and once
// concurrently on two streams.
static int conc_mode(int n, int reps) {
  const uint64_t size = 1ull << n;
  double2* amps;
  if (cudaMalloc(&amps, 16 * size) != cudaSuccess) return 1;
  fill_random<<<4096, 256>>>(amps, size);
  GraphDev g;
  memset(&g, 0, sizeof(g));
  g.n_nodes = n;
  int E = 0;
  auto add = [&](int i, int j) {
    if (i > j) { int t = i; i = j; j = t; }
    if ((g.rm[i] >> j) & 1) return;
    g.rm[i] |= 1ull << j; g.adj[i] |= 1ull << j; g.adj[j] |= 1ull << i; ++E;
  };
  for (int i = 0; i < n; ++i) add(i, (i + 1) % n);
  for (int i = 0; i < n / 2; ++i) add(i, i + n / 2);
  g.tot_edge = E;
  double2* tab;
  cudaMalloc(&tab, sizeof(double2) * (E + 1) * 2);
  double2* h = (double2*)malloc(sizeof(double2) * (E + 1) * 2);
  for (int k = 0; k < 2 * (E + 1); ++k) h[k] = make_double2(cos(0.1 * k), sin(0.1 * k));
  cudaMemcpy(tab, h, sizeof(double2) * (E + 1) * 2, cudaMemcpyHostToDevice);
  const int64_t T = (int64_t)(size >> 12);
  const int m = (n - 12 + 1) / 2;
  SweepArgs s0, mg;
  memset(&s0, 0, sizeof(s0));
  s0.amps = amps; s0.table = tab; s0.table2 = tab + (E + 1); s0.g = g; s0.ntiles = T;
  s0.carry = 12; s0.q = 0; s0.rx1 = RxStage{0.3, 0.0, 1}; s0.table_len = E + 1; s0.flags = kStage1;
  mg = s0;
  mg.carry = 12 - m; mg.q = 12; mg.rx2 = RxStage{-0.2, 0.0, 1}; mg.flags = kStage1 | kMidCost | kStage2;
  const int K = getenv("CONC_CHUNKS") ? atoi(getenv("CONC_CHUNKS")) : 1;
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, ea, eb;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&ea); cudaEventCreate(&eb);
  auto half = [&](SweepArgs a, int64_t lo, cudaStream_t st) {
    for (int k = 0; k < K; ++k) {
      a.tile_lo = lo + k * (T / 2 / K);
      a.tile_cnt = T / 2 / K;
      launch_sweep(a, (int)a.tile_cnt, st);
    }
  };
  float t_seq = 0, t_conc = 0, t_s0 = 0, t_mg = 0;
  for (int mode = 0; mode < 4; ++mode) {
    for (int it = 0; it < 2; ++it) {  // warm-up pass, then timed
      cudaDeviceSynchronize();
      cudaEventRecord(e0, sa);
      for (int r = 0; r < reps; ++r) {
        if (mode == 0) { half(s0, 0, sa); half(mg, T / 2, sa); }
        else if (mode == 1) {
          cudaEventRecord(ea, sa);
          cudaStreamWaitEvent(sb, ea, 0);
          half(s0, 0, sa); half(mg, T / 2, sb);
          cudaEventRecord(eb, sb);
          cudaStreamWaitEvent(sa, eb, 0);
        } else if (mode == 2) { half(s0, 0, sa); }
        else { half(mg, T / 2, sa); }
      }
      cudaEventRecord(e1, sa);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      if (it) (mode == 0 ? t_seq : mode == 1 ? t_conc : mode == 2 ? t_s0 : t_mg) = ms;
    }
  }
  printf("n=%d chunks=%d: S0 half %.3f ms, merged half %.3f ms, back to back %.3f ms, concurrent %.3f ms (%.3f of back to back) %s\n",
         n, K, t_s0, t_mg, t_seq, t_conc, t_conc / t_seq, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && strcmp(argv[1], "conc") == 0) return conc_mode(atoi(argv[2]), atoi(argv[3]));
  if (argc > 1 && strcmp(argv[1], "cut") == 0)
    return cut_mode(atoi(argv[2]), atoi(argv[3]), argc > 4 ? atoi(argv[4]) : 0);
  if (argc > 1 && strcmp(argv[1], "check") == 0)
    return check_mode(argc > 2 ? atoi(argv[2]) : 13, argc > 3 ? atoi(argv[3]) : 24,
                      argc > 4 ? atoi(argv[4]) : 2);
  const int n = argc > 1 ? atoi(argv[1]) : 30;
  const int reps = argc > 2 ? atoi(argv[2]) : 5;
  const uint64_t size = 1ull << n;
  double2* amps;
  if (cudaMalloc(&amps, 16 * size) != cudaSuccess) return 1;
  fill_random<<<4096, 256>>>(amps, size);
  cudaDeviceSynchronize();
  // degree-3 test graph: ring + chords (E = 3n/2)
  GraphDev g;
  memset(&g, 0, sizeof(g));
  g.n_nodes = n;
  int E = 0;
  auto add = [&](int i, int j) {
    if (i > j) { int t = i; i = j; j = t; }
    if ((g.rm[i] >> j) & 1) return;
    g.rm[i] |= 1ull << j;
    g.adj[i] |= 1ull << j;
    g.adj[j] |= 1ull << i;
    ++E;
  };
  for (int i = 0; i < n; ++i) add(i, (i + 1) % n);
  for (int i = 0; i < n / 2; ++i) add(i, i + n / 2);
  g.tot_edge = E;
  double2* tab;
  cudaMalloc(&tab, sizeof(double2) * (E + 1) * 2);
  double2* h = (double2*)malloc(sizeof(double2) * (E + 1) * 2);
  for (int k = 0; k < 2 * (E + 1); ++k) h[k] = make_double2(cos(0.1 * k), sin(0.1 * k));
  cudaMemcpy(tab, h, sizeof(double2) * (E + 1) * 2, cudaMemcpyHostToDevice);
  double* partials;
  cudaMalloc(&partials, sizeof(double) * (size >> 12));

  const int grid = (int)(size >> 12);
  const int high = n - 12;
  const int m = (high + 1) / 2;  // two high sets at N = 30 (9 + 9)
  struct Kind {
    const char* name;
    int carry, q;
    uint32_t flags;
  } kinds[] = {
      {"S0 stage1 (C=12)", 12, 0, kStage1},
      {"S0 pre-cost+stage1", 12, 0, kPreCost | kStage1},
      {"high merged (F2)", 12 - m, 12 + (high - m), kStage1 | kMidCost | kStage2},
      {"high single+cost (F1)", 12 - m, 12, kPreCost | kStage1},
      {"high single (F1)", 12 - m, 12, kStage1},
      {"C=4 single (F1)", 4, 12, kStage1},
      {"C=5 single (F1)", 5, 12, kStage1},
      {"C=6 single (F1)", 6, 12, kStage1},
      {"C=3 top single (F1)", 3, n - 9, kStage1},
      {"merged S1 (F2)", 12 - m, 12, kStage1 | kMidCost | kStage2},
      {"gen S1 (F1)", 12 - m, 12, kGen | kPreCost | kStage1},
      {"last S1 (expect)", 12 - m, 12, kStage1 | kScale | kExpect},
      {"last S2 (expect)", 12 - m, 12 + (high - m), kStage1 | kScale | kExpect},
  };
  const double bytes = 32.0 * (double)size;
  if (argc > 4) {  // sweep_probe N REPS IMPL KIND | custom C q FLAGS: one kind, one impl
    const int impl = atoi(argv[3]);
    Kind custom{"custom", 0, 0, 0u};
    if (strcmp(argv[4], "custom") == 0 && argc > 7) {
      custom.carry = atoi(argv[5]);
      custom.q = atoi(argv[6]);
      custom.flags = (uint32_t)strtol(argv[7], nullptr, 0);
    }
    const Kind& k = strcmp(argv[4], "custom") == 0 ? custom : kinds[atoi(argv[4])];
    // impl 30: the per-sweep policy without the 128 x 32 C = 3 kernel
    set_sweep32(impl == 30 ? 0 : -1);
    set_sweep_impl(impl == 30 ? 3 : impl);
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    a.amps = amps; a.table = tab; a.table2 = tab + (E + 1); a.partials = partials; a.g = g;
    a.ntiles = size >> 12; a.carry = k.carry; a.q = k.q;
    a.rx1 = RxStage{0.3, 0.0, 1}; a.rx2 = RxStage{-0.2, 0.0, 1};
    a.table_len = E + 1; a.flags = k.flags;
    const float t = time_sweep(a, grid, reps);
    printf("%s C=%d q=%d flags=0x%x impl %d: %.3f ms (%.0f GB/s)\n", k.name, k.carry, k.q, k.flags, impl, t,
           bytes / t / 1e6);
    return 0;
  }
  printf("n=%d E=%d grid=%d\n", n, E, grid);
  const char* names[] = {"v4 one tile per CTA", "TMA loads", "TMA loads + stores", "per-sweep policy"};
  for (int impl = 0; impl < 4; ++impl) {
  set_sweep_impl(impl);
  printf("impl %d (%s)\n", impl, names[impl]);
  for (const Kind& k : kinds) {
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    a.amps = amps;
    a.table = tab;
    a.table2 = tab + (E + 1);
    a.partials = partials;
    a.g = g;
    a.ntiles = size >> 12;
    a.carry = k.carry;
    a.q = k.q;
    a.rx1 = RxStage{0.3, 0.0, 1};
    a.rx2 = RxStage{-0.2, 0.0, 1};
    a.gen = make_double2(1.0 / 32768.0, 0.0);
    a.table_len = E + 1;
    float t[4];
    const uint32_t extra[4] = {0u, kGen, kNoStore, kGen | kNoStore};
    for (int v = 0; v < 4; ++v) {
      a.flags = k.flags | extra[v];
      t[v] = time_sweep(a, grid, reps);
    }
    printf("%-24s C=%2d q=%2d  full %.3f ms (%.0f GB/s)  no-load %.3f  no-store %.3f  on-chip only %.3f\n",
           k.name, k.carry, k.q, t[0], bytes / t[0] / 1e6, t[1], t[2], t[3]);
  }
  }
  return 0;
}
