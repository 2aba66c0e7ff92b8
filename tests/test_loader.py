"""Neutral model format straight into the master layout (
reference graph.py:433-539): lowering.load_lowered decodes the blob once and
gathers the master with one vectorised index map; it must be byte-identical
to the load_model -> lower -> master path on every committed model file,
including the reference-written ones, and lower to the same units."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200.graph import ModelFormatError, load_model, save_model
from paper_2509_22857_b200.lowering import load_lowered, lower, master_array

MODELS = sorted((GOLDEN / "models").glob("*.json"))


def _units(lw):
    return [sorted(u.items()) for u in lw.units]


@pytest.mark.parametrize("path", MODELS, ids=[p.stem for p in MODELS])
def test_master_byte_identical(path):
    ref = lower(load_model(str(path)))
    want = master_array(ref._chunks, ref.master_size)
    lw, got = load_lowered(str(path))
    assert got.dtype == np.float64 and got.shape == want.shape
    assert got.tobytes() == want.tobytes()
    assert _units(lw) == _units(ref)
    assert lw.scalar == ref.scalar and lw.packed_size == ref.packed_size


def test_no_per_node_copies(tmp_path):
    """Node tensors of the loader's graph are views of the one decoded blob."""
    path = tmp_path / "rn20.json"
    save_model(configs.build("resnet20"), str(path))
    lw, _ = load_lowered(str(path))
    bases = set()
    for node in lw.graph.nodes.values():
        for v in vars(node).values():
            if isinstance(v, np.ndarray) and v.size:
                assert not v.flags.owndata and not v.flags.writeable
                bases.add(id(v.base if v.base is not None else v))
    assert len(bases) == 1


def test_format_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"version": 99, "nodes": [], "edges": [], "weights": ""}')
    with pytest.raises(ModelFormatError):
        load_lowered(str(bad))
