"""bench.py keeps the driver's contract: one JSON line with the required keys
for each arm / stage (short runs).  CPU: the reference arm (oracle/_ref on a
few frames).  GPU: our arm, the U-Net and pipeline stages."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
        "dtype", "data", "config"}


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference not built (oracle/build_ref.sh)")
    d = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1", "--ref-step-frames", "20")
    assert KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")


@pytest.mark.gpu
def test_our_arm_contract():
    d = _run("--config", "c1", "--frames", "600", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert {"e2e", "roofline", "gpu_launches", "clocks"} <= set(d)
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and 0 < r["frac"] < 1
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0 and d["outputs_sane"]
    assert d["impl"] == "ours" and d["e2e_dropin"]["value"] > 0
    assert d["e2e_dropin"]["d2h_bytes_per_step"] > 600 * 128 * 128 * 4  # the corrected video comes back


@pytest.mark.gpu
def test_gpus_2_runs_two_ranks_with_exchange():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks
    (strong scaling, frame-balanced shards, one straddling block exchanged
    over peer memory).  On a one-GPU box both ranks share the device and the
    collectives run over gloo (host-mediated: no kernel waits on another
    rank's kernel); the measured configuration uses NCCL."""
    import os

    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--frames", "700",
                          "--steps", "2", "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["straddling_blocks"] == 1
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["outputs_sane"]


@pytest.mark.gpu
@pytest.mark.parametrize("stage", ["unet", "pipeline"])
def test_stage_lines(stage):
    d = _run("--stage", stage, "--config", "c1", "--frames", "600", "--steps", "2", "--warmup", "3",
             "--no-cpu-baseline")
    assert d["value"] > 0 and "metric" in d
