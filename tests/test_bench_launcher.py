"""bench.py's multi-rank plumbing on CPU: `--gpus N` outside torchrun
re-launches itself under torch.distributed.run with N ranks, and the ranks'
device times / tokens reduce to one rank-0 line (max over ranks, tokens once
for a tree-partitioned request, summed for replicas).  The GPU work itself is
skipped (--dry-run); everything else is the path the driver's 8-GPU run takes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("placement,expect_tokens", [("tree", 1000), ("replicas", 2000)])
def test_bench_relaunches_n_ranks(placement, expect_tokens):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--placement", placement], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    j = lines[0]
    assert j["n_gpus"] == 2 and j["dry_run"]
    assert j["dev_ms_max"] == 101.0 and j["e2e_ms_max"] == 111.0  # max over ranks
    assert j["tokens"] == expect_tokens
    assert j["scaling"] == ("strong" if placement == "tree" else "weak")
