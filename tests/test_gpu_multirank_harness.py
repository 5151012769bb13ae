"""The multi-rank bench path on ONE GPU: torchrun with 2 ranks sharing cuda:0
and gloo collectives on host copies (NEO_BENCH_DIST_BACKEND=gloo,
NEO_BENCH_SHARE_GPU=1 -- a harness check, never a measurement).  Every N > 1
branch of bench.py runs on the real kernels: the KV-head TP rank plans of c4,
per-rank timing, MAX / SUM aggregation with the head-sharding token rule, the
e2e leg and the all-gather reassembly leg, so the driver's first multi-GPU run
cannot fail on harness logic."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_bench_two_ranks_on_one_gpu(cfg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, NEO_BENCH_DIST_BACKEND="gloo", NEO_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", cfg, "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-prefill"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                   # rank 0 alone prints
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and len(j["per_rank_ms_per_step"]) == 2
    assert j["ms_per_step"] == pytest.approx(max(j["per_rank_ms_per_step"]), rel=1e-3)
    assert j["scaling"] == "strong" and j["e2e"]["value"] > 0
    if cfg == "c4":
        assert j["config"]["parallelism"].startswith("tp2") and j["config"]["batch"] == 512
        assert j["reassembly"]["allgather_bytes_per_layer_per_rank"] == 512 * 32 * 128 * 2
        # head sharding: attended tokens are counted once (not doubled by the two ranks)
        toks = sum(WORK_CTX[cfg]) * j["config"]["layers_per_step"] * j["steps"]
        assert j["attended_tokens_per_s"] == pytest.approx(toks / (j["ms_per_step"] * j["steps"] / 1e3), rel=2e-3)
    else:
        assert j["config"]["parallelism"].startswith("dp2") and j["config"]["batch"] == 1024


def test_bench_default_config_two_ranks_on_one_gpu():
    """The driver's scaling run launches bench.py with NO --config: c3 (weak
    scaling, every rank its own 128 requests) with the swap leg and rank 0's
    prefill leg.  Two ranks on one GPU with 4 cycled layer pools per rank
    (NEO_BENCH_MAX_POOLS, harness only) so both fit in HBM."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, NEO_BENCH_DIST_BACKEND="gloo", NEO_BENCH_SHARE_GPU="1", NEO_BENCH_MAX_POOLS="4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3"]
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["scaling"] == "weak"
    assert j["config"]["batch"] == 256 and j["config"]["batch_per_rank"] == 128
    assert j["config"]["parallelism"].startswith("dp2")
    assert j["swap"] is not None and j["swap"]["swap_out_gbs"] > 0
    assert j["prefill"] is not None and j["prefill"]["attn_us"] > 0
    assert j["e2e"]["value"] > 0 and len(j["per_rank_ms_per_step"]) == 2


WORK_CTX = {}


def setup_module(module):
    sys.path.insert(0, ROOT)
    from neo_inputs.workloads import WORKLOADS
    WORK_CTX["c4"] = [int(x) for x in WORKLOADS["c4"].contexts()]
