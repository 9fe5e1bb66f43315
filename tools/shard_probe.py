"""Timing of the fused sharded path on ONE GPU with G virtual shards (dev tool):
per-level shard sweeps and the exchange kernel (which on one device moves the
whole state through HBM: read 16 B + write 16 B per amplitude).

    python tools/shard_probe.py N G P
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2312_03019_b200 as Q
from paper_2312_03019_b200 import sharded as S

n, G, p = (int(x) for x in sys.argv[1:4])
gb = G.bit_length() - 1
g = Q.random_regular_graph(n, 3, seed=0)
pr = Q.params_from_seed(p, 0)
shards = [S.CudaShard(n - gb, r) for r in range(G)]


class TimedPeer(S.PeerExchanger):
    def __init__(self, shards):
        super().__init__(shards)
        self.ms = []

    def exchange(self, g_bits, p0, rx, factor):
        for s in self.shards:
            s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        S._exchange_call(0, 0, g_bits, self.ptrs, self.shards[0].n, p0, 0,
                         1 << (self.shards[0].n - g_bits), rx, factor)
        b.record()
        torch.cuda.synchronize()
        self.ms.append(a.elapsed_time(b))


ex = TimedPeer(shards)
for it in range(3):
    ex.ms.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    S.simulate_sharded_fused(g, pr, shards, ex, gb, expect=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
e = S.sharded_expectation(shards)
bytes_x = 32.0 * (1 << n)
print(f"N={n} G={G} p={p}: {dt*1e3:.1f} ms total (host-driven, virtual shards), <C>={e:.12f}")
print(f"exchange kernel: {len(ex.ms)} calls, mean {np.mean(ex.ms):.3f} ms = "
      f"{bytes_x / (np.mean(ex.ms) * 1e-3) / 1e9:.0f} GB/s (16 B read + 16 B write per amplitude)")
