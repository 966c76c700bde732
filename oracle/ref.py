"""Import the UNMODIFIED reference (voltseg) built into oracle/_ref by
oracle/build_ref.sh -- TEST/BENCH INFRASTRUCTURE ONLY.

Used (a) here, to generate golden vectors (tests/golden/make_golden.py) and
(b) by bench.py --impl reference / cpu_baseline to time the reference's own
CPU stage on the GPU box's host.  Never imported by the product package.
"""
from __future__ import annotations

import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
STUBS = HERE / "ref_stubs"


def available() -> bool:
    return (REF_DIR / "voltseg" / "motion.py").exists()


def load(backend: str | None = None):
    """Return (motion, summarize, kernels, video_io) modules of the reference.

    backend: "native" | "python" | None (reference default).  The reference
    reads VOLTSEG_BACKEND once at import (kernels.py:93-95); the dispatcher
    consults kernels.BACKEND per call, so it is set directly.
    """
    if not available():
        raise RuntimeError("reference not built: run oracle/build_ref.sh")
    for p in (str(STUBS), str(REF_DIR)):
        if p not in sys.path:
            sys.path.insert(0, p)
    import voltseg.kernels as kernels  # noqa: E402
    if backend is not None:
        # mean_zncc_scores reads the module global at call time (kernels.py:98-108)
        if backend not in kernels._backends:
            raise RuntimeError(f"reference backend {backend!r} unavailable")
        kernels.BACKEND = backend
    import voltseg.motion as motion
    import voltseg.summarize as summarize
    import voltseg.video_io as video_io
    return motion, summarize, kernels, video_io
