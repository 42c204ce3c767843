"""bench.py's multi-GPU launch contract (CPU, no GPU needed).

`python bench.py --gpus N` (no WORLD_SIZE in the environment) re-runs itself
under torch.distributed.run with N ranks on 127.0.0.1; under torchrun (the
driver's own launch) it does not spawn again.  --spawn-probe makes each rank
print its RANK / WORLD_SIZE and exit before touching a GPU.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _probe(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args, "--spawn-probe"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_spawns_n_ranks(n):
    lines = _probe(["--gpus", str(n)])
    assert sorted(d["rank"] for d in lines) == list(range(n))
    assert all(d["world"] == n for d in lines)
    assert sorted(d["local_rank"] for d in lines) == list(range(n))


def test_gpus_1_and_torchrun_children_do_not_respawn():
    assert _probe(["--gpus", "1"]) == [{"rank": 0, "world": 1, "local_rank": 0}]
    # already a rank of a torchrun job: no second launch
    lines = _probe(["--gpus", "2"], {"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert lines == [{"rank": 1, "world": 2, "local_rank": 1}]
