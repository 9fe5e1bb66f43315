"""The sharded bench path end to end under torch.distributed.run on a one-GPU
box: 2 and 4 ranks share cuda:0, exchanges over gloo staged through host
memory (the NCCL path is the same code with device tensors).  <C> must equal
the unsharded engine's."""

import json
import os
import subprocess
import sys

import pytest

import paper_2312_03019_b200 as Q

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,exchange,chunks,events", [(2, "ipc", 4, 1), (4, "ipc", 4, 1),
                                                          (4, "ipc", 4, 0), (4, "ipc", 1, 1),
                                                          (2, "nccl", 1, 1), (4, "nccl", 1, 1)])
def test_torchrun_sharded_bench(world, exchange, chunks, events):
    """ipc: the fused exchange kernel with the peers' shards mapped by CUDA IPC
    (here all on one device); nccl: the staging path."""
    n, p = 22, 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + (10 if exchange == "ipc" else 0) + chunks + 20 * events),
           os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--steps", "2", "--warmup", "3",
           "--qubits", str(n), "--levels", str(p), "--dist-backend", "gloo", "--share-device",
           "--exchange", exchange, "--chunks", str(chunks)]
    env = dict(os.environ, QAOA_IPC_EVENTS=str(events))
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    g = Q.random_regular_graph(n, 3, seed=0)
    e = Q.expectation(g, Q.simulate(g, Q.params_from_seed(p, 0), "bitwise", max_qubits=n))
    assert line["expectation"] == pytest.approx(e, rel=1e-10)
    assert line["n_gpus"] == world and line["scaling"] == "strong" and line["test_mode"]
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0


@pytest.mark.parametrize("world,chunks,levels", [(2, 4, 1), (4, 1, 2)])
def test_torchrun_weak_scaling_modes(world, chunks, levels):
    """--scaling weak: 2^qubits amplitudes per rank (N = qubits + log2 G, odd N =
    u3r(N-1) + an isolated node), p=1 checked against the closed form inside the
    bench, per-exchange kernel times (CUDA events) reported for the NVLink
    figure; <C> equals the unsharded engine's."""
    sys.path.insert(0, ROOT)
    import bench

    base = 20
    n = base + world.bit_length() - 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + world + chunks),
           os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--steps", "2", "--warmup", "3",
           "--qubits", str(base), "--levels", str(levels), "--dist-backend", "gloo",
           "--share-device", "--scaling", "weak", "--chunks", str(chunks)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["scaling"] == "weak" and line["config"]["n_qubits"] == n

    class A:
        graph = "u3r"

    A.n = n
    g = bench.make_graph(Q, A)
    e = Q.expectation(g, Q.simulate(g, Q.params_from_seed(levels, 0), "bitwise", max_qubits=n))
    assert line["expectation"] == pytest.approx(e, rel=1e-10)
    if levels == 1:
        assert line["closed_form_p1"]["rel_err"] <= 1e-10
    nv = line["nvlink"]
    assert nv["exchange_ms"] > 0 and nv["achieved_GBps_per_direction"] > 0
