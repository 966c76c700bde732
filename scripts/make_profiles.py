"""Turn the raw ncu outputs of scripts/gpu_profile.sh (gpurun_out/) into the
tracked summaries under profiles/ (run here, no GPU):
  profiles/<tag>_launches.csv        the ncu launch list (copied)
  profiles/<tag>_launch_shares.txt   per-kernel time share of the stage kernels
  profiles/<tag>_ncu_full_summary.txt  ncu --set full metrics + stall mix per kernel
  profiles/ncu_traffic.json          DRAM bytes per frame of the search kernel (read by bench.py)
Usage: python scripts/make_profiles.py TAG [FRAMES_PER_LAUNCH]"""
import csv
import io
import json
import re
import shutil
import subprocess
import sys
from contextlib import redirect_stdout
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "scripts"))
import ncu_stalls  # noqa: E402
import ncu_summary  # noqa: E402

CMD = "python bench.py --frames 2000 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    return name.replace("void ", "").strip()


def launch_shares(src: Path, dst: Path):
    lines = src.read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum" or "vb::" not in r["Kernel Name"]:
            continue
        if "peak_probe" in r["Kernel Name"] or "ffma" in r["Kernel Name"].lower():
            continue
        k = short(r["Kernel Name"])
        ms = float(r["Metric Value"]) * (1e-6 if r["Metric Unit"] == "ns" else 1e-3 if r["Metric Unit"] == "us" else 1)
        t, n = agg.get(k, (0.0, 0))
        agg[k] = (t + ms, n + 1)
    tot = sum(t for t, _ in agg.values())
    out = [f"ncu launch list (cold-cache, serialised) of `{CMD}`, stage kernels only (FP32 peak probes excluded)"]
    for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        out.append(f"  {t:7.3f} ms  {n:3d} launches  {t / tot:5.1%}  {k}")
    dst.write_text("\n".join(out) + "\n")
    print(dst.read_text())


def main(tag: str, frames_per_launch: int = 2000):
    g = ROOT / "gpurun_out"
    prof = ROOT / "profiles"
    shutil.copy(g / f"launches_{tag}.csv", prof / f"{tag}_launches.csv")
    launch_shares(g / f"launches_{tag}.csv", prof / f"{tag}_launch_shares.txt")
    rep = str(g / f"prof_{tag}.ncu-rep")
    buf = io.StringIO()
    with redirect_stdout(buf):
        print(f"ncu --set full --clock-control none of `{CMD}` (one launch per kernel, {frames_per_launch} frames)")
        ncu_summary.main(rep)
        for k in ("zncc_group", "zncc_stats", "smooth_tma", "correct_rows", "median"):
            print(f"\n-- warp-stall samples, {k}")
            try:
                ncu_stalls.main(rep, k, 12)
            except Exception as exc:  # noqa: BLE001
                print("  (not captured)", exc)
    (prof / f"{tag}_ncu_full_summary.txt").write_text(buf.getvalue())
    out = subprocess.run(["ncu", "-i", rep, "-k", "regex:zncc_group", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    r = rows[2]
    unit = rows[1]
    def val(m):
        v = float(r[hdr.index(m)])
        u = unit[hdr.index(m)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    (prof / "ncu_traffic.json").write_text(json.dumps({"zncc_group_kernel": {
        "dram_bytes_per_frame": dram / frames_per_launch,
        "source": f"profiles/{tag}_ncu_full_summary.txt: ncu --set full, {short(r[hdr.index('Kernel Name')])}, one "
                  f"{frames_per_launch}-frame launch of `bench.py --frames 2000`; dram__bytes_read.sum + "
                  f"dram__bytes_write.sum"}}, indent=1))
    print((prof / "ncu_traffic.json").read_text())


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2000)
