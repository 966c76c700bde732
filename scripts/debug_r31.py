import sys, os
sys.path.insert(0, ".")
import numpy as np
from paper_2403_16438_b200 import kernels
from paper_2403_16438_b200.motion import PatchGrid
rng = np.random.default_rng(0)
for radius in [int(x) for x in sys.argv[1:]]:
    size = max(128, 21 + 2 * radius + 8)
    f = rng.random((size, size), dtype=np.float32); r = rng.random((size, size), dtype=np.float32)
    g = PatchGrid.cover(size, size, 21, margin=radius)
    try:
        out = kernels.mean_zncc_scores(f, r, g.origins, 21, radius)
        print(radius, "ok", out.shape, flush=True)
    except Exception as e:
        print(radius, "FAIL", e, flush=True)
        break
