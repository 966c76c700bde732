"""U-Net consumer of the summaries on the CUDA path (csrc/unet.cu) against the
reference's golden vectors: forward within the reference's own acceptance
bound (<= 1e-4 absolute, test_acceptance.py:152-163), normalisation
bit-exact, tiled merge <= 1e-4; batch == single, determinism, the fused
per-block call == the separate calls."""
from pathlib import Path

import numpy as np
import pytest

from paper_2403_16438_b200 import unet

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden" / "unet.npz"


@pytest.fixture(scope="module")
def golden():
    return np.load(G)


@pytest.fixture(scope="module")
def bundle(golden):
    flat = golden["weights_flat"]
    tensors, off = {}, 0
    for name, shape in unet.architecture():
        n = int(np.prod(shape))
        tensors[name] = flat[off:off + n].reshape(shape).copy()
        off += n
    return unet.WeightBundle(tensors)


def test_forward_matches_reference(cuda, golden, bundle):
    got = unet.forward_batch(bundle, golden["fwd_in"])
    assert got.shape == (6, 64, 64) and got.dtype == np.float32
    assert np.abs(got - golden["fwd_out"]).max() <= 1e-4
    assert got.min() > 0 and got.max() < 1


def test_forward_acceptance_twenty_patches(cuda, bundle):
    """test_acceptance.py:152-163: 20 random [0,1) patches vs the direct-convolution oracle."""
    from oracle import unet_oracle as O
    rng = np.random.default_rng(7)
    for _ in range(20):
        patch = rng.random((2, 64, 64), dtype=np.float32)
        assert np.abs(unet.forward(bundle, patch) - O.forward(bundle.tensors, patch)).max() <= 1e-4


def test_batch_matches_single_and_deterministic(cuda, golden, bundle):
    x = golden["fwd_in"]
    b = unet.forward_batch(bundle, x)
    for i in range(len(x)):
        np.testing.assert_array_equal(unet.forward(bundle, x[i]), b[i])
    np.testing.assert_array_equal(unet.forward_batch(bundle, x), b)


def test_forward_rejects_wrong_shape(cuda, bundle):
    with pytest.raises(ValueError, match="expected"):
        unet.forward_batch(bundle, np.zeros((1, 2, 32, 32), np.float32))


def test_normalize_pair_bitwise(cuda, golden):
    for name in golden["norm_names"]:
        got = unet.normalize_pair(golden[f"norm_{name}__sp"], golden[f"norm_{name}__tp"])
        np.testing.assert_array_equal(got, golden[f"norm_{name}__out"], err_msg=str(name))


def test_tile_and_merge_matches_reference(cuda, golden, bundle):
    for name in golden["merge_names"]:
        x = golden[f"merge_{name}__in"]
        pm = unet.tile_and_merge(bundle, x, segment_index=3, stride=int(golden[f"merge_{name}__stride"]))
        assert pm.segment_index == 3 and pm.values.shape == x.shape[1:]
        assert np.abs(pm.values - golden[f"merge_{name}__out"]).max() <= 1e-4, name
        assert pm.values.min() >= 0 and pm.values.max() <= 1


def test_segment_pairs_equals_separate_calls(cuda, bundle):
    from paper_2403_16438_b200.summarize import SummaryPair
    rng = np.random.default_rng(5)
    pairs = [SummaryPair(i, (rng.random((96, 160)) * 500).astype(np.float32),
                         rng.random((96, 160)).astype(np.float32)) for i in range(3)]
    maps = unet.segment_pairs(bundle, pairs)
    for p, m in zip(pairs, maps):
        want = unet.tile_and_merge(bundle, unet.normalize_pair(p.spatial, p.temporal), p.segment_index)
        assert m.segment_index == p.segment_index
        np.testing.assert_array_equal(m.values, want.values)
