"""bench.py's multi-rank launch on CPU: with --gpus N and no torchrun environment it
re-launches itself under torch.distributed.run with N ranks on 127.0.0.1; the
--spawn-check mode rendezvouses them over gloo and rank 0 prints one JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_spawns_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--spawn-check"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["ranks"] == [0, 1]


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_two_nccl_ranks():
    """world = min(2, device_count) over NCCL: bench.py --gpus 2 launches two ranks, one per GPU,
    shards the database, exchanges the per-shard top-k over NCCL and prints one line with n_gpus 2.
    Skipped on a one-GPU box (this pool's gpurun boxes have one B200)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--n", "4000000", "--steps", "2",
                        "--warmup", "3", "--per-ht", "", "--no-cpu-baseline", "--no-e2e"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["value"] > 0
