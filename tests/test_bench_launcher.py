"""bench.py's multi-GPU launcher and protocol, dry run on CPU (gloo, stand-in correlator):
`python bench.py --gpus N` outside torchrun re-launches itself under torch.distributed.run,
the config's 512 rotations are sharded in contiguous blocks (strong scaling), every step ends
with the all-gather of the per-rotation records, and the gathered global records (and the
global best) are identical for every world size."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=300):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    env["OMP_NUM_THREADS"] = "1"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_dry_run_strong_scaling_protocol():
    one = run_bench("--dry-run", "--gpus", "1", "--steps", "2", "--warmup", "3")
    assert one["n_gpus"] == 1 and one["scaling"] == "strong" and one["dry_run"]
    ref = one["result_sample"]["global_best"]
    for n in (2, 3):
        d = run_bench("--dry-run", "--gpus", str(n), "--steps", "2", "--warmup", "3")
        assert d["n_gpus"] == n and d["config"]["rotations_per_step"] == 512
        blocks = d["config"]["rotations_per_rank"]
        assert len(blocks) == n and blocks[0][0] == 0 and blocks[-1][1] == 512
        assert all(blocks[i][1] == blocks[i + 1][0] for i in range(n - 1))
        assert d["result_sample"]["global_best"] == ref  # same records (sha1) and best as one rank
        assert d["value"] > 0 and d["ms_per_step"] > 0
