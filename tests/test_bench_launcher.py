"""CPU checks of bench.py's multi-GPU launcher: `--gpus N`
without a torchrun environment spawns N ranks itself (torch.distributed.run on
127.0.0.1), every rank joins the process group (gloo in --dry-run), and rank 0
alone prints the contract line with "n_gpus": N."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=300, env=env, cwd=ROOT)


@pytest.mark.parametrize("n", [2])
def test_bench_spawns_n_ranks_dry_run(n):
    r = _run(["--gpus", str(n), "--dry-run", "--steps", "3", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout                       # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == n and line["dry_run"] is True and line["scaling"] == "weak"
    assert line["config"]["parallelism"] == f"ep{n}"
    assert line["config"]["global_tokens"] == n * line["config"]["tokens_per_gpu"]
    for rank in range(n):
        assert f"rank {rank}: process group backend=gloo nranks={n}" in r.stderr


def test_bench_rejects_world_mismatch():
    r = _run(["--gpus", "2", "--dry-run"], env_extra={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
