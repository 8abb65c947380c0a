"""Multi-process (N > 1) host logic on CPU with the gloo backend.

A dendrogram does not shard: N GPUs run independent trees
("replicas only"; config 5 deals 64 trees round-robin).  What must be right
for N > 1 is the work plan per rank, the max-over-ranks timing, the
sum-over-ranks work, and the launcher contract (one JSON line from rank 0).
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_config5_round_robin_partition(world):
    plans = [bench.replica_plan("config5", world, r) for r in range(world)]
    flat = sorted(t for p in plans for t in p)
    assert flat == list(range(bench.CONFIG5_TREES))          # every tree exactly once
    assert all(t % world == r for r, p in enumerate(plans) for t in p)  # tree i -> GPU i mod N
    assert max(map(len, plans)) - min(map(len, plans)) <= 1


def test_single_tree_workloads_one_replica_per_rank():
    for world in (1, 2, 8):
        assert [bench.replica_plan("config4", world, r) for r in range(world)] == [[r] for r in range(world)]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mx = bench.reduce_max([1.0 + rank, 10.0 - rank, 0.5 * rank])
    sm = bench.reduce_sum([float(rank + 1)])
    dist.barrier()
    out.put((rank, mx, sm))
    dist.destroy_process_group()


def test_gloo_world2_max_and_sum_over_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, sm in res:
        assert mx == [2.0, 10.0, 0.5]   # the slowest rank's time, per entry
        assert sm == [3.0]              # total work over ranks


def test_reduce_without_process_group_is_identity():
    assert bench.reduce_max([1.0, 2.0]) == [1.0, 2.0]
    assert bench.reduce_sum([3.0]) == [3.0]


def test_torchrun_world2_reference_arm_prints_one_line():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-sample", "20000"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    # the unmodified reference when baseline/_ref holds it, else the oracle port
    from tests.conftest import reference_package
    kind = "reference" if reference_package() is not None else "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == kind
    assert d["config"]["n_edges_sample_per_step"] == 20000
