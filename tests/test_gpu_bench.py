"""bench.py keeps the driver's contract (-m gpu): one JSON line with the required keys, for the default run
(N=1, C2), the C4 split at N=2 (torchrun; gloo standing in for NCCL so two ranks can share the one GPU),
and the reference arm (short runs).  Each run's line carries its own evidence: the oracle spot check of
windows of the last timed step, the CPU baseline (all threads and one thread, CPU model), the build id."""
import json
import os
import socket
import subprocess
import sys

import pytest

from nsg_testutil import ROOT

pytestmark = pytest.mark.gpu


def _lines(out):
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0])


def _run(*args, env=None):
    return _lines(subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                                 text=True, timeout=900, cwd=ROOT, env=env))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_default_line(cuda_device):
    d = _run("--steps", "20", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches", "cpu_baseline",
              "spot_check", "build_id"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["value"] > 0
    assert d["unit"] == "packets/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("C2")
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "traffic_source"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * (1 << 23) and d["e2e"]["value"] > 0
    assert d["spot_check"]["match"] is True and len(d["spot_check"]["windows"]) == 3
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert cb["value_1core"] > 0 and cb["cpu_model"] and "1 thread" in cb["sample_1core"]


def test_c4_split_over_two_ranks(cuda_device):
    env = dict(os.environ, NSG_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=1200,
                         cwd=ROOT, env=env)
    d = _lines(out)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["workload"].startswith("C4")
    assert d["config"]["packets_per_gpu_per_step"] == 1 << 29
    assert "all_gather_into_tensor" in d["config"]["gather"]
    assert d["value"] > 0 and d["value_without_gather"] >= d["value"] * 0.5
    assert d["spot_check"]["match"] is True
    assert d["cpu_baseline"] is None  # rank 0 at N=1 only


def test_reference_arm(cuda_device):
    import oracle

    d = _run("--impl", "reference", "--steps", "2", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    per_step = int(d["cpu_baseline"]["sample"].split()[0])
    assert per_step >= max(64, oracle.hardware_threads())
    assert d["cpu_baseline"]["cpu_model"]
