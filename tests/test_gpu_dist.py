"""The N > 1 product path on one GPU: `bench.py` under torchrun with two
ranks (gloo, both ranks on cuda:0) runs every config sharded -- mulv (weak),
secure ReLU C1 (sharded) and the 2^L-per-rank sweep, the C3 matmul (rows of
X sharded), MLP / LeNet inference (images sharded) -- through the package's
own Session, all-gathers the opened outputs to rank 0 and checks them there
against the plaintext (bench.py asserts; a mismatch exits non-zero)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(900)
def test_bench_two_ranks_product_path(cuda):
    port = 29900 + os.getpid() % 90
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py",
           "--gpus", "2", "--dist-backend", "gloo", "--log2n", "16", "--steps", "2", "--warmup", "1",
           "--e2e-steps", "1", "--relu-log2n", "12", "--relu-sweep-log2n", "11", "--matmul-n", "256",
           "--mlp-batch", "64", "--mlp-verified-batch", "16", "--lenet-batch", "8",
           "--lenet-verified-batch", "4", "--mulv-sweep", "", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=880)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["e2e"]["value"] > 0
    assert j["relu"]["n_gpus"] == 2 and j["relu"]["N_per_gpu"] == 2048 and j["relu"]["verified"] > 0
    assert j["relu_sweep"]["N"] == 4096
    assert j["matmul"]["n_gpus"] == 2 and j["matmul"]["rows_per_gpu"] == 128 and "check" in j["matmul"]
    assert j["mlp"]["n_gpus"] == 2 and j["mlp"]["verified"] > 0
    assert j["lenet"]["verified_config_batch"]["images"] == 8
