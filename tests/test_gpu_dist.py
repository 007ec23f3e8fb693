"""The multi-rank bench path on one GPU: two torchrun ranks share the device with the gloo
backend (LPB_DIST_BACKEND=gloo; on a multi-GPU box each rank owns a GPU and uses NCCL).
Checks the contract pieces that only exist for N > 1: contiguous per-rank shards (weak
scaling), the MAX-over-ranks device time, the post-solve results gather, one JSON line."""
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


@pytest.mark.parametrize("config,extra", [("cfg1", []), ("cfg4", ["--batch", "200000"]),
                                          ("cfg2r", ["--batch", "1000"])])
def test_two_rank_bench_line(config, extra):
    env = dict(os.environ, LPB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus",
           "2", "--config", config, "--steps", "3", "--warmup", "3", "--e2e-steps", "1", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2")
    assert d["gather_ms"] is not None and d["gather_ms"] > 0
    assert d["e2e"]["value"] > 0 and d["cpu_baseline"] is None  # baseline at N = 1 only


@pytest.mark.parametrize("case", ["G1", "G2", "cfg2r", "cfg5"])
def test_two_rank_sharded_parity(case):
    """N = 2 (two ranks sharing the test box's GPU over gloo): each rank solves its
    contiguous shard through the C ABI, the gathered results equal the N = 1 solve of the
    whole batch bit for bit and the oracle on a sample (tests/dist_parity_worker.py)."""
    env = dict(os.environ, LPB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join("tests", "dist_parity_worker.py"), case]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert f"PARITY-OK {case}" in r.stdout, r.stdout


def test_two_rank_strong_scaling_bench():
    """--scaling strong: the config's fixed batch is sharded over the ranks (SURVEY §8(e),
    cfg5's 6,003,000 LPs over 1/2/4/8 GPUs); the gathered results are consistent."""
    env = dict(os.environ, LPB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus",
           "2", "--config", "cfg5", "--scaling", "strong", "--batch", "300001", "--steps", "3",
           "--warmup", "3", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["scaling"] == "strong" and d["n_gpus"] == 2
    assert d["config"]["batch_total"] == 300001 and d["config"]["batch_per_gpu"] == 150000
    assert d["gather_check"].startswith("ok"), d["gather_check"]


@pytest.mark.parametrize("config,extra", [("cfg4", ["--batch", "200000"]),
                                          ("cfg1", [])])
def test_bench_cuda_graph_mode(config, extra):
    """--graph: each step replays one captured CUDA graph of the solve (one kernel launch per
    step, the library's own launch path captured on the bench's stream)."""
    cmd = [sys.executable, "bench.py", "--config", config, "--graph", "--steps", "5",
           "--warmup", "3", "--e2e-steps", "0", "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["config"]["cuda_graph"] is True and d["value"] > 0
    assert d["gpu_launches"] == 5
