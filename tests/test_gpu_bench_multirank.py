"""bench.py's N > 1 path (one process per GPU under torchrun) exercised on the ONE GPU this
pool has: MPM_BENCH_SHARED_GPU=1 puts both ranks on cuda:0 with a gloo process group, and the
C5a slab exchanges go through the host-staged transport instead of NCCL.  Checks the harness,
not the timings: rank 0 alone prints one JSON line with n_gpus = 2, the whole-job particle
count and the sharding of each workload (rollout shards for C4 / C5b, x-slabs for C5a)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(workload, extra=()):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MPM_BENCH_SHARED_GPU="1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--workload", workload, *extra]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("workload", ["C4", "C5b", "C5a"])
def test_bench_two_ranks_one_json_line(workload):
    d = _run(workload, ("--no-cpu-baseline",))
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    for k in ("metric", "unit", "ms_per_step", "higher_is_better", "scaling", "dtype", "data", "config", "roofline",
              "clocks", "e2e"):
        assert k in d, k
    # C4: one rollout per rank (weak); C5b: the 64 rollouts shared out, C5a: one body split (strong)
    assert d["scaling"] == ("weak" if workload == "C4" else "strong") and d["higher_is_better"] is True
    assert d["roofline"]["frac"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    cfg = d["config"]
    if workload == "C5a":  # one body split into two x-slabs: the job is the whole body
        assert cfg["particles_per_rank"] < 8_355_840 and "slab" in cfg["parallelism"]
    else:  # independent rollouts sharded over the ranks
        assert "rollout" in cfg["parallelism"]


def test_bench_reference_arm_two_ranks():
    """--impl reference under torchrun: rank 0 alone runs the oracle and prints the line."""
    d = _run("C4", ("--impl", "reference"))
    assert d["impl"] == "reference" and d["value"] > 0
