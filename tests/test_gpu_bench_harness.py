"""bench.py's N > 1 path end to end on one GPU: `bench.py --gpus 2` launches its own 2 ranks
(torch.distributed.run), both on cuda:0 over gloo (RS_BENCH_HARNESS_TEST=1; the ranks' kernels
never wait on each other).  One JSON line from rank 0 with the contract's keys, per-rank seeds,
zero mismatches against the oracle, and a per-rank cpu_baseline on a core partition."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, RS_BENCH_HARNESS_TEST="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
           "--cpu-seconds", "2"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout            # rank 0 only
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["parallelism"] == "dp2"
    assert d["verified"]["mismatches"] == 0 and d["e2e"]["verified"]
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["verified"]["oracle_bytes_compared_per_phase"] == 51 * 14 * (16 << 20)  # S stripes over 2 ranks
    cb = d["cpu_baseline"]
    assert cb["cpu_model"] and len(cb["per_rank"]) == 2 and cb["value"] > 0
