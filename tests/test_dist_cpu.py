"""Multi-GPU host logic on CPU: frame sharding, max-over-ranks timing and BER
totals through torch.distributed (gloo, world_size 2), and bench.py's
reference arm under torchrun (rank 0 alone runs and prints)."""

import json
import os
import socket
import subprocess
import sys
import tempfile
from pathlib import Path

import pytest
import torch.multiprocessing as mp

from paper_2604_02266_b200 import dist as ddist

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("total,world", [(4096, 1), (4096, 2), (4097, 8), (3, 8), (0, 2)])
def test_shard_covers_every_frame_once(total, world):
    slices = [ddist.shard(total, r, world) for r in range(world)]
    assert slices[0][0] == 0 and slices[-1][1] == total
    for (a, b), (c, _) in zip(slices, slices[1:]):
        assert b == c
    sizes = [b - a for a, b in slices]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        ddist.shard(total, world, world)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), LOCAL_RANK=str(rank),
                      WORLD_SIZE=str(world))
    r, _, ws = ddist.init("gloo")
    res = {
        "rank": r, "world": ws,
        "max": ddist.max_over_ranks(1.5 * (rank + 1)),
        "sum": ddist.sum_over_ranks(100 + rank),
        "shard": ddist.shard(4096, r, ws),
        "seed": ddist.rank_seed(1000, r),
    }
    ddist.barrier(sync_cuda=False)
    Path(out_dir, f"r{rank}.json").write_text(json.dumps(res))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_gloo_world2_reductions():
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, port, d), nprocs=2, join=True)
        res = [json.loads(Path(d, f"r{r}.json").read_text()) for r in range(2)]
    for r in res:
        assert r["world"] == 2
        assert r["max"] == 3.0          # the slowest rank's time
        assert r["sum"] == 201          # totals summed over ranks
    assert res[0]["shard"] == [0, 2048] and res[1]["shard"] == [2048, 4096]
    assert res[0]["seed"] != res[1]["seed"]  # independent frames per rank (weak scaling)


def test_single_process_is_identity():
    assert ddist.max_over_ranks(2.5) == 2.5
    assert ddist.sum_over_ranks(7) == 7
    ddist.barrier(sync_cuda=False)


def test_reference_arm_under_torchrun_prints_once():
    """bench.py --impl reference under torchrun, 2 ranks on CPU: rank 0 alone
    times the CPU reference and prints one JSON line; the other rank exits 0."""
    port = _free_port()
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "cfg1",
           "--cpu-seconds", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    # the unmodified reference (baseline/_ref) when it is installed, else the numpy port
    want = "reference" if (ROOT / "baseline" / "_ref" / "ddlink" / "__init__.py").exists() else "port"
    assert d["cpu_baseline"]["kind"] == want and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["p99_frame_ms"] >= d["cpu_baseline"]["p50_frame_ms"] > 0


def test_reference_arm_json_contract():
    """bench.py --impl reference (single process, CPU only): one JSON line with
    the driver's keys; e2e carries zero transfer bytes and cpu_baseline
    describes the run."""
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
           "--config", "cfg1", "--cpu-seconds", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["unit"] == "symbols/s" and d["value"] > 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
