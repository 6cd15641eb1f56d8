"""bench.py's N > 1 launch path on CPU: `--gpus 2` outside torch.distributed.run re-launches
itself as two ranks (127.0.0.1 rendezvous), the ranks form a process group, shard the frames'
pixel rows (v % world == rank) and reduce over ranks; rank 0 alone prints the JSON line.
(`--dry-run`: gloo, no kernels -- the GPU path itself needs >= 2 GPUs.)"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_dry_run_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--config",
                          "tiny"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    d = lines[0]
    assert d["dry_run"] and d["n_gpus"] == 2 and d["ranks"] == 2 and d["rank_sum"] == 1
    assert d["pixels"] == d["pixels_expected"] > 0  # the row shards cover every pixel once
