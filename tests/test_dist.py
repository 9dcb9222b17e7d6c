"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 plumbing:
rank/seed assignment, max-over-ranks timing, sharding plan, and the
reference-arm bench path under torchrun (rank 0 prints, rank 1 exits)."""

import json
import os
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    from paper_2411_09287_b200 import dist
    r, w, _ = dist.init("gloo")
    assert (r, w) == (rank, world)
    slow = dist.max_over_ranks(1.0 + rank)
    total = dist.sum_over_ranks(10.0)
    seeds = {dist.session_seed(r, s) for s in range(4)}
    # every rank verifies its own independent batch with the CPU oracle
    from oracle import mpc
    res = mpc.mulv(seed=dist.session_seed(r, 0), lanes=64, d=16, R=2)
    # final output gather of the sharded batch: rank order, equal shards
    import torch
    full = dist.gather_outputs(torch.arange(4, dtype=torch.int64) + 100 * rank)
    assert full.tolist() == [0, 1, 2, 3, 100, 101, 102, 103]
    dist.barrier()
    q.put((rank, slow, total, sorted(seeds), res.verdict, int(res.z[1]["m"][0])))
    dist.finalize()


def test_gloo_world2_plumbing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, s0, t0, seeds0, v0, z0), (_, s1, t1, seeds1, v1, z1) = out
    assert s0 == s1 == 2.0 and t0 == t1 == 20.0
    assert not set(seeds0) & set(seeds1)
    assert v0 and v1 and z0 != z1


def test_session_seeds_are_collision_free():
    from paper_2411_09287_b200.dist import session_seed
    seen = {}
    for stream in range(3):
        for rank in range(8):
            for step in list(range(1200)) + [2**32 - 1]:
                s = session_seed(rank, step, stream)
                assert s not in seen, (stream, rank, step, seen.get(s))
                assert s < 2**128
                seen[s] = (stream, rank, step)


def test_shard_plan():
    from paper_2411_09287_b200.dist import shard
    parts = [shard(1000, 3, r, align=8) for r in range(3)]
    assert parts[0][0] == 0 and parts[-1][1] == 1000
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    assert all((b - a) % 8 == 0 for a, b in parts[:-1])


@pytest.mark.timeout(600)
def test_reference_arm_under_torchrun():
    """`bench.py --impl reference` under torchrun with 2 ranks: rank 0 prints
    one JSON line, rank 1 exits 0 without work."""
    port = 29700 + os.getpid() % 200
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py",
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--cpu-seconds", "2"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=580)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["cpu_baseline"]["kind"] in ("reference", "port")
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["cores"] >= 1
