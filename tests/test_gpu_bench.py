"""bench.py honours --gpus N by itself (no external launcher): it re-execs
through torch.distributed.run with one rank per GPU.  On a one-GPU box the
ranks share GPU 0 (VPFV_SAME_DEVICE=1, gloo transport -- validation only)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_bench_gpus_2_spawns_two_ranks(halo):
    env = dict(os.environ, VPFV_SAME_DEVICE="1", VPFV_DIST_BACKEND="gloo")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                          "--warmup", "3", "--workload", "landau2d-64", "--no-cpu-baseline", "--e2e-steps", "0",
                          "--halo", halo],
                         env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["config"]["halo"] == halo
    assert line["value"] > 0 and line["gpu_launches"] > 0


def test_bench_gpus_more_than_visible_fails_loudly():
    import torch

    n = torch.cuda.device_count() + 1
    env = {k: v for k, v in os.environ.items() if k not in ("VPFV_SAME_DEVICE", "WORLD_SIZE")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3"],
                         env=env, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0
    assert "GPU(s) are visible" in out.stderr
