"""U-Net consumer of the summaries, CPU side: the oracle
restatement against the reference's golden vectors, and the host half of the
drop-in (architecture, WeightBundle checks, VSEGW1 byte format)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2403_16438_b200 import unet

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
        tensors[name] = flat[off:off + n].reshape(shape)
        off += n
    return unet.WeightBundle(tensors)


def test_parameter_count_pinned():
    # test_unet.py:27-35 layer arithmetic
    assert unet.parameter_count() == 118129
    shapes = dict(unet.architecture())
    assert shapes["dec2.conv1.kernel"] == (32, 96, 3, 3) and shapes["dec1.conv1.kernel"] == (16, 48, 3, 3)
    names = [n for n, _ in unet.architecture()]
    assert names[0] == "enc1.conv1.kernel" and names[-1] == "out.conv.bias"
    assert all(n in unet.architecture_fingerprint() for n in names)


def test_random_bundle_matches_reference_draws(bundle):
    w = unet.WeightBundle.random(np.random.default_rng(7))
    for name, _ in unet.architecture():
        np.testing.assert_array_equal(w.tensors[name], bundle.tensors[name])


def test_vsegw1_bytes_identical_to_reference(golden, bundle, tmp_path):
    unet.save_weights(bundle, tmp_path / "w.vsegw1")
    assert (tmp_path / "w.vsegw1").read_bytes() == golden["weights_vsegw1"].tobytes()
    back = unet.load_weights(tmp_path / "w.vsegw1")
    for name, _ in unet.architecture():
        np.testing.assert_array_equal(back.tensors[name], bundle.tensors[name])


def test_vsegw1_errors(golden, tmp_path):
    raw = golden["weights_vsegw1"].tobytes()
    p = tmp_path / "x.vsegw1"
    p.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(unet.WeightFormatError, match="bad magic"):
        unet.load_weights(p)
    p.write_bytes(raw[:1000])
    with pytest.raises(unet.WeightFormatError, match="truncated"):
        unet.load_weights(p)
    p.write_bytes(raw + b"\0\0")
    with pytest.raises(unet.WeightFormatError, match="2 trailing bytes"):
        unet.load_weights(p)


def test_validate_messages(bundle):
    t = dict(bundle.tensors)
    del t["enc2.conv1.bias"]
    with pytest.raises(unet.WeightFormatError, match="enc2.conv1.bias"):
        unet.WeightBundle(t).validate()
    t = dict(bundle.tensors)
    t["out.conv.kernel"] = np.zeros((2, 16, 1, 1), np.float32)
    with pytest.raises(unet.WeightFormatError, match="shape"):
        unet.WeightBundle(t).validate()
    t = dict(bundle.tensors)
    t["rogue"] = np.zeros(3, np.float32)
    with pytest.raises(unet.WeightFormatError, match="unexpected"):
        unet.WeightBundle(t).validate()
    t = {k: v.copy() for k, v in bundle.tensors.items()}
    t["enc1.conv1.kernel"][0, 0, 0, 0] = np.inf
    with pytest.raises(unet.WeightFormatError, match="non-finite"):
        unet.WeightBundle(t).validate()
    assert bundle.flat().size == unet.parameter_count()


# ---------------------------------------------------------------- the oracle, pinned
def test_oracle_forward_matches_reference(golden, bundle):
    from oracle import unet_oracle as O
    got = O.forward_batch(bundle.tensors, golden["fwd_in"])
    np.testing.assert_allclose(got, golden["fwd_out"], atol=1e-6)


def test_oracle_normalize_matches_reference_bitwise(golden):
    from oracle import unet_oracle as O
    for name in golden["norm_names"]:
        got = O.normalize_pair(golden[f"norm_{name}__sp"], golden[f"norm_{name}__tp"])
        np.testing.assert_array_equal(got, golden[f"norm_{name}__out"])


def test_oracle_tile_and_merge_matches_reference(golden, bundle):
    from oracle import unet_oracle as O
    for name in golden["merge_names"][:3]:
        got = O.tile_and_merge(bundle.tensors, golden[f"merge_{name}__in"], int(golden[f"merge_{name}__stride"]))
        np.testing.assert_allclose(got, golden[f"merge_{name}__out"], atol=1e-6)


def test_oracle_tile_positions_and_tent():
    from oracle import unet_oracle as O
    assert O.tile_positions(128, 32) == [0, 32, 64]
    assert O.tile_positions(150, 32) == [0, 32, 64, 86]
    assert O.tile_positions(64, 32) == [0]
    t = O.tent()
    assert t.dtype == np.float32 and t.shape == (64, 64) and t.min() >= np.float32(1e-3)
    assert t[31, 31] == t.max() and t[0, 0] == np.float32(max(1e-3, (1 - 31.5 / 32) ** 2))
