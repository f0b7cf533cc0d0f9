"""The multi-rank path of bench.py on the GPU box: two ranks under torchrun
sharing cuda:0 (gloo for the host-side barrier / max / totals, since NCCL
needs one device per rank).  One JSON line from rank 0, the job's totals over
both ranks, weak and strong scaling (frame-batch sharding, no
collective on the solve path)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_on_one_gpu(scaling):
    env = dict(os.environ, DDB_DIST_BACKEND="gloo", OPENBLAS_NUM_THREADS="1")
    batch = 296
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--batch", str(batch), "--scaling", scaling,
           "--no-e2e", "--no-cpu", "--no-frontend", "--no-latency", "--no-dropin", "--no-geometry"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["value"] > 0
    per_rank = batch if scaling == "weak" else batch // 2
    assert d["config"]["batch_per_gpu"] == per_rank
    # the job's symbols over the slowest rank's time
    frames = 2 * batch if scaling == "weak" else batch
    mn = d["config"]["M"] * d["config"]["N"]
    assert abs(d["value"] - frames * mn * d["steps"] / (d["ms_per_step"] * d["steps"] * 1e-3)) < 1e-6 * d["value"]
    assert 0 <= d["ber"] < 0.1
