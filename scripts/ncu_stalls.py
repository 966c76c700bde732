"""Per-SASS warp-stall samples of one kernel from an ncu report (run here, no
GPU): totals per stall reason for the whole kernel and for the hottest
address range, plus the top stalled instructions.
Usage: python scripts/ncu_stalls.py REPORT KERNEL_REGEX [TOP]"""
import csv
import subprocess
import sys


def main(path, regex, top=25):
    out = subprocess.run(["ncu", "-i", path, "-k", f"regex:{regex}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    num = lambda r, c: float(r[hdr.index(c)] or 0)  # noqa: E731
    reasons = [h for h in hdr if h.startswith("stall_") and not h.endswith("(Not Issued)")]
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"{len(data)} SASS lines, {tot:.0f} samples")
    agg = {h: sum(num(r, h) for r in data) for h in reasons}
    print("  " + ", ".join(f"{h[6:]}={v / tot:.1%}" for h, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
    ops = {}
    for r in data:
        op = r[hdr.index("Source")].split()[0] if r[hdr.index("Source")].split() else "?"
        if op.startswith("@"):
            op = r[hdr.index("Source")].split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + num(r, "Warp Stall Sampling (All Samples)")
    print("  by opcode: " + ", ".join(f"{k}={v / tot:.1%}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:12]))
    for r in sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:top]:
        det = sorted(((h[6:], num(r, h)) for h in reasons), key=lambda x: -x[1])[:3]
        print(f"  {r[hdr.index('Address')][-5:]} {r[hdr.index('Source')][:58]:58s} "
              f"{num(r, 'Warp Stall Sampling (All Samples)'):6.0f}  " + " ".join(f"{k}:{v:.0f}" for k, v in det if v))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)


def opmix(path, regex):
    """Executed warp instructions per opcode (source page)."""
    out = subprocess.run(["ncu", "-i", path, "-k", f"regex:{regex}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    seen, ops = set(), {}
    for r in data:
        if r[0] in seen:
            continue
        seen.add(r[0])
        src = r[hdr.index("Source")].split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        n = float(r[hdr.index("Instructions Executed")] or 0)
        ops[op] = ops.get(op, 0) + n
    tot = sum(ops.values())
    print(f"{tot:.4g} warp instructions")
    for k, v in sorted(ops.items(), key=lambda x: -x[1])[:40]:
        print(f"  {k:28s} {v:12.4g} {v / tot:6.1%}")
