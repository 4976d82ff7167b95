"""bench.py's own N > 1 path on one B200: `--gpus 2` re-launches itself under
torch.distributed.run, the two ranks exchange their peer-window IPC handles
and run the sharded persistent stack (EP, TP) through the peer exchange.
MOE_B200_BENCH_SAME_GPU=1 puts both ranks on GPU 0 (time-sliced: the line's
numbers mean nothing, its shape and exit status do), so the first multi-GPU
box produces a scaling curve without a first-run surprise."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("shard", ["ep", "tp"])
def test_bench_two_ranks_one_gpu(shard):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, MOE_B200_BENCH_SAME_GPU="1", MASTER_ADDR="127.0.0.1")
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_PORT"):
        env.pop(k, None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--layers", "2", "--shard", shard, "--no-extras", "--no-cpu-baseline"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["steps"] == 3 and rec["warmup"] == 3
    assert rec["value"] > 0 and rec["gpu_launches"] >= 3
    assert rec["config"]["parallelism"].startswith(shard)
