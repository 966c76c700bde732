"""Summarise an ncu report (run here, no GPU): per-kernel duration, DRAM
bytes, pipe utilisation, occupancy and the top warp-stall reasons."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def main(path, filt=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if filt and filt not in name:
            continue
        print("==", name[:90])
        for w in WANT:
            if w in hdr:
                print(f"   {w:70s} {r[hdr.index(w)]}")
        stalls = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
        stalls = sorted(stalls, key=lambda x: -float(x[1] or 0))[:8]
        print("   stalls:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={float(v):.2f}" for h, v in stalls))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
