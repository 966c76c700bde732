"""Ad-hoc GPU parity probe (development aid): CUDA path vs the C oracle."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from oracle import oracle as O
import paper_2403_16438_b200 as vb
from paper_2403_16438_b200 import synth, kernels, motion, summarize, stage

rng = np.random.default_rng(0)
# 1. operator: scores
for (h, w, P, R) in [(96, 96, 21, 5), (128, 128, 21, 8), (96, 96, 15, 3), (128, 128, 21, 12), (60, 60, 16, 3)]:
    fr = rng.random((h, w), dtype=np.float32); rf = rng.random((h, w), dtype=np.float32)
    g = motion.PatchGrid.cover(h, w, P, margin=R)
    a = kernels.mean_zncc_scores(fr, rf, g.origins, P, R)
    b = O.mean_zncc_scores(fr, rf, g.origins, P, R)
    print("scores", (h, w, P, R), "maxdiff", abs(a - b).max(), flush=True)
# 2. realistic video
cfg = synth.CONFIGS["c1"].with_frames(200)
v, truth = synth.generate_numpy(cfg, return_truth=True)
vf = v.astype(np.float32)
motion.REFERENCE_FRAMES = 100
t0 = time.time()
corr, vecs, pairs = stage.preprocess(vb.Video(v), stage.StageConfig(search_radius=5, segment_length=100, ref_frames=100))
print("gpu preprocess", time.time() - t0, flush=True)
t0 = time.time()
ref = O.preprocess(vf, 21, 5, True, 100, 100, 3.0)
print("oracle", time.time() - t0)
dx = np.array([[x.dx, x.dy] for x in vecs]); sub = np.array([[x.sub_dx, x.sub_dy, x.confidence] for x in vecs])
print("int mismatches", (dx != ref["dxdy"]).any(1).sum(), "sub maxdiff", abs(sub[:, :2] - ref["sub_conf"][:, :2]).max(),
      "conf maxdiff", abs(sub[:, 2] - ref["sub_conf"][:, 2]).max())
print("corrected maxdiff", abs(corr.data - ref["corrected"]).max(), "rel", (abs(corr.data - ref["corrected"]) / np.maximum(abs(ref["corrected"]), 1)).max())
sp = np.stack([p.spatial for p in pairs]); tp = np.stack([p.temporal for p in pairs])
print("spatial maxdiff", abs(sp - ref["spatial"]).max(), "temporal maxdiff", abs(tp - ref["temporal"]).max())
# summaries bit-exact on the oracle's corrected video
sp2 = summarize.summarize(vb.Video(ref["corrected"]), 100)
print("summaries on identical input: spatial exact", all((p.spatial == ref["spatial"][i]).all() for i, p in enumerate(sp2)),
      "temporal exact", all((p.temporal == ref["temporal"][i]).all() for i, p in enumerate(sp2)))
# translate bit exact
for d in [(0.3, -1.7), (2.0, 0.0), (-3.25, 2.5), (7.25, -9.5), (-25, 2)]:
    print("translate", d, (motion.translate(vf[0], *d) != O.translate(vf[0], *d)).sum())
print("truth recovery: max |x - truth|", abs(dx + sub[:, :2] - truth.drift).max())
# host stage e2e
hs = stage.HostStage(cfg.height, cfg.width, stage.StageConfig(search_radius=5, segment_length=100, ref_frames=100), chunk_frames=100)
vec, sp3, tp3, c3 = hs.run(v, corrected=True)
print("hoststage vs device: vec", (vec["dx"] == dx[:, 0]).all(), abs(vec["sub_dx"] - sub[:, 0]).max(), "sp", abs(sp3 - sp).max(), "tp", abs(tp3 - tp).max(), "corr", abs(c3 - corr.data).max(), "launches", hs.last_launches)
