"""Experiment: overlap_blocks sweep for DevicePreprocessor (runs under gpurun)."""
import sys, json, subprocess, os
for ob in sys.argv[1:]:
    env = dict(os.environ, VB_OVERLAP_BLOCKS=ob)
    out = subprocess.run([sys.executable, "bench.py", "--steps", "4", "--warmup", "2", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, env=env).stdout
    d = json.loads(out)
    print("overlap", ob, round(d["value"]), "ms", round(d["ms_per_step"], 2), json.dumps(d["roofline"]["kernel_ms_per_step"]))
