"""Compare two ab_search.py runs: integer shifts, sub-pixel and score diffs."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent / "gpurun_out"
a, b, name = sys.argv[1], sys.argv[2], sys.argv[3]
x, y = np.load(ROOT / f"ab_{a}_{name}.npz"), np.load(ROOT / f"ab_{b}_{name}.npz")
ra, rb = x["rec"], y["rec"]
print(name, a, "vs", b, "int mismatches", int(((ra["dx"] != rb["dx"]) | (ra["dy"] != rb["dy"])).sum()),
      "max sub diff", float(max(np.abs(ra["sub_dx"] - rb["sub_dx"]).max(), np.abs(ra["sub_dy"] - rb["sub_dy"]).max())),
      "max score diff", float(np.abs(x["scores"] - y["scores"]).max()))
