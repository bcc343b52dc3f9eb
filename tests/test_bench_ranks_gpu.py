"""bench.py's multi-rank path (`--gpus N` re-executes itself under torchrun; per-rank row
shards, the merge, max-over-ranks timing, one JSON line from rank 0) on the one-GPU pool:
COMPASS_BENCH_SHARED_GPU puts every rank on cuda:0 with gloo collectives.  This checks the
launch, the merge paths and the line, not performance (the driver's scaling run uses one GPU
per rank and NCCL)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(gpus, extra, env=None):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--workload", "C2", "--steps", "2",
           "--warmup", "3", "--no-e2e", "--no-cpu", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


_ONE = {}


@pytest.mark.parametrize("extra", [[], ["--merge", "peer"], ["--row-shard"]])
def test_bench_two_ranks_line(extra):
    if "one" not in _ONE:
        _ONE["one"] = _line(1, [])
    one = _ONE["one"]
    d = _line(2, extra, env=dict(os.environ, COMPASS_BENCH_SHARED_GPU="1"))
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert d["nccl"]["world_size"] == 2
    # merged survivor counts (both ranks' shards) and the plan equal the one-process run's
    assert d["survivors"] == one["survivors"]
    assert d["plan"] == one["plan"]
