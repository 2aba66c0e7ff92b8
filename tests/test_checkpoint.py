"""Checkpoint ingest (paper_2509_22857_b200/checkpoint.py) against files the
reference exporter wrote from the same .npz checkpoints
(tests/golden/make_ckpt_golden.py), plus the exporter's refusal cases; and,
on a B200, the checkpoint -> P2FR -> Engine path against the oracle."""

import base64
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import levnet_oracle as O
from paper_2509_22857_b200 import checkpoint as C
from paper_2509_22857_b200.graph import load_model, save_model

CASES = [
    ("ckpt_rn20_w4", "rn20", 8, None),
    ("ckpt_rn18_w4", "rn18", 16, None),
    ("ckpt_rn20_w4_shared", "rn20", 8, [0.01, 1.0, 0.05]),
]


def _blob_hash(path):
    with open(path) as f:
        return hashlib.sha256(base64.b64decode(json.load(f)["weights"])).hexdigest()


@pytest.mark.parametrize("name,variant,hw,coeffs", CASES)
def test_conversion_matches_reference_exporter(tmp_path, name, variant, hw, coeffs):
    g = C.graph_from_checkpoint(str(GOLDEN / f"{name}.npz"), variant, input_hw=hw, coeffs=coeffs)
    out = tmp_path / "g.json"
    save_model(g, str(out))
    ref_path = GOLDEN / "models" / f"{name}_ref.json"
    ref_doc, our_doc = json.loads(ref_path.read_text()), json.loads(out.read_text())
    # same nodes (ids, kinds, params) in the same order, same ordered edges,
    # bit-identical float64 weight blob
    assert [(n["id"], n["kind"], n.get("params")) for n in our_doc["nodes"]] == \
        [(n["id"], n["kind"], n.get("params")) for n in ref_doc["nodes"]]
    assert our_doc["edges"] == ref_doc["edges"]
    assert _blob_hash(out) == _blob_hash(ref_path)
    # and the same function
    ref = load_model(str(ref_path))
    x = np.random.default_rng(3).normal(0, 1, (2,) + ref.validate()[ref.input_id()])
    np.testing.assert_array_equal(O.eval_batch(g, x), O.eval_batch(ref, x))


def test_export_state_hash(tmp_path):
    st = C.load_state_dict(str(GOLDEN / "ckpt_rn20_w4.npz"))
    h = C.export_state(st, "rn20", str(tmp_path / "m.json"), input_hw=8)
    assert h == _blob_hash(GOLDEN / "models" / "ckpt_rn20_w4_ref.json")


def _state():
    return C.load_state_dict(str(GOLDEN / "ckpt_rn20_w4.npz"))


def test_refusals_name_the_key():
    st = _state()
    del st["layer2.0.bn1.running_var"]
    with pytest.raises(C.ExportError, match=r"missing required key 'layer2.0.bn1.running_var'"):
        C.graph_from_state(st, "rn20")
    st = _state()
    st["layer1.1.conv2.weight"] = st["layer1.1.conv2.weight"][:, :2]
    with pytest.raises(C.ExportError, match=r"'layer1.1.conv2.weight' has shape \(4, 2, 3, 3\), expected"):
        C.graph_from_state(st, "rn20")
    st = _state()
    st["layer9.0.conv1.weight"] = np.zeros((1, 1, 1, 1))
    with pytest.raises(C.ExportError, match=r"'layer9.0.conv1.weight' does not map to any rn20 layer"):
        C.graph_from_state(st, "rn20")
    st = _state()
    del st["layer3.2.act2.coeffs"]
    with pytest.raises(C.ExportError, match=r"embeds activation coefficients for 18 of 19 activations"):
        C.graph_from_state(st, "rn20")
    st = _state()
    st["bn1.running_var"] = -np.ones_like(st["bn1.running_var"])
    with pytest.raises(C.ExportError, match=r"cannot form a positive sigma"):
        C.graph_from_state(st, "rn20")
    with pytest.raises(C.ExportError, match=r"unknown variant"):
        C.graph_from_state(_state(), "rn99")


def test_torch_checkpoint_reader(tmp_path):
    import torch
    st = _state()
    p = tmp_path / "c.pt"
    torch.save({"state_dict": {k: torch.from_numpy(v.astype(np.float32)) for k, v in st.items()}}, p)
    back = C.load_state_dict(str(p))
    assert set(back) == set(st)
    np.testing.assert_allclose(back["fc.weight"], st["fc.weight"].astype(np.float32))


@pytest.mark.gpu
def test_checkpoint_engine_matches_oracle(cuda):
    import torch
    eng, rg, report = C.engine_from_checkpoint(str(GOLDEN / "ckpt_rn20_w4.npz"), "rn20", "P2FR", input_hw=8)
    g = C.graph_from_checkpoint(str(GOLDEN / "ckpt_rn20_w4.npz"), "rn20", input_hw=8)
    x = np.random.default_rng(4).normal(0, 1, (16, 3, 8, 8))
    want = O.eval_batch(g, x)
    got = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda()).double().cpu().numpy()
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err <= 1e-4, err
    # P2F folded the BNs into the convs / joins, P2R made every poly monic
    assert report.nodes_removed > 0 and report.rewrites
    from paper_2509_22857_b200.graph import PolyActNode
    assert all(n.is_monic() for n in rg.nodes.values() if isinstance(n, PolyActNode))
