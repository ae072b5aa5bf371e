"""bench.py end to end on one GPU (short runs): the JSON-line contract, the 24-layer stack
mode, and the multi-rank path (two ranks sharing the GPU over gloo -- the ENC_DIST_BACKEND
test hook; the NCCL path differs only in the process-group backend)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _run(cmd, env=None):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert KEYS <= set(line), KEYS - set(line)
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    return line


def test_bench_stack_mode():
    line = _run([sys.executable, "bench.py", "--layers", "3", "--steps", "3", "--warmup", "3",
                 "--no-cpu-baseline"])
    assert line["config"]["layers"] == 3 and line["n_gpus"] == 1
    assert line["metric"].startswith("BERT-large encoder stack")


@pytest.mark.parametrize("layers", [1, 2])
def test_bench_two_ranks_gloo(layers):
    line = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                 "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port", "29531",
                 "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                 "--layers", str(layers)], env={"ENC_DIST_BACKEND": "gloo"})
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp2"
    assert line["cpu_baseline"] is None
