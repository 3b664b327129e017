"""bench.py contract checks that run without a GPU: the reference arm (the C
port of the reference's CPU path) prints one valid JSON line."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1", "--cpu-sample", "65536"],
                         capture_output=True, text=True, check=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "Gvec/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["warmup"] >= 3  # the contract's minimum warm-up is enforced
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "Gvec/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["metric"].startswith("compressed float3 vector-add")


def test_reference_arm_under_torchrun_rank0_only():
    """N > 1 (the driver's scaling launch): rank 0 alone runs and prints; the
    other ranks exit 0 without output.  gloo on CPU, two ranks."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), str(ROOT / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "2", "--warmup", "1", "--cpu-sample", "65536"],
                         capture_output=True, text=True, check=True, timeout=600)
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_multirank_code_path_on_one_gpu():
    """Functional check of the N > 1 path of bench.py (torchrun, two ranks,
    barrier + max-over-ranks, rank-0 line) on a one-GPU box: the ranks share
    cuda:0 over gloo (VC3_BENCH_SHARE_GPU); the timing is not a result."""
    import os
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, VC3_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2",
                          "--steps", "3", "--warmup", "3", "--vectors", str(1 << 22), "--no-secondary"],
                         capture_output=True, text=True, check=True, timeout=600, env=env)
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["global_vectors"] == 2 << 22
