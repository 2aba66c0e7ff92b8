"""Generate the golden fixtures that pin the oracle to the real reference.

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``levnet`` from ``/root/reference/pkg/src`` (read-only), builds
seeded graphs with the reference's own constructors and generators, runs the
reference's forward / redistribution / pipeline / fusion code on them, and
writes

* ``tests/golden/models/*.json``  -- graphs in the reference's neutral model
  format, written by the reference's own ``save_model``;
* ``tests/golden/golden.npz``     -- inputs and reference outputs;
* ``tests/golden/manifest.json``  -- what each case is and which reference
  function produced it.

Nothing here runs at test time; the GPU box never sees /root/reference.
"""

from __future__ import annotations

import json
import os
import pathlib
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_FIXTURE = "/root/reference/pkg/tests/fixtures/rn20_8x8.json"
sys.path.insert(0, REF_SRC)

from levnet import graph as G  # noqa: E402
from levnet import transforms as T  # noqa: E402

HERE = pathlib.Path(__file__).resolve().parent
MODELS = HERE / "models"


_SAVED = {}


def save(g, name):
    """Write g once; later saves of the same graph object reuse the file."""
    if id(g) in _SAVED:
        return _SAVED[id(g)][1]
    MODELS.mkdir(parents=True, exist_ok=True)
    G.save_model(g, str(MODELS / f"{name}.json"))
    _SAVED[id(g)] = (g, f"models/{name}.json")
    return f"models/{name}.json"


def _SAVED_GRAPH(path):
    return next(g for g, p in _SAVED.values() if p == path)


def tiny_model(seed, classes=3):
    rng = np.random.default_rng(seed)
    g = G.ModelGraph()
    g.add(G.InputNode("in", 2, 6, 6))
    g.add(G.ConvNode("conv1", rng.normal(0, 0.25, (3, 2, 3, 3)), rng.normal(0, 0.1, 3), 1, 1))
    g.add(G.PolyActNode("act1", [np.array(0.05), np.array(0.4), np.array(1.3)]))
    g.add(G.ConvNode("conv2", rng.normal(0, 0.25, (3, 3, 3, 3)), rng.normal(0, 0.1, 3), 2, 1))
    g.add(G.PolyActNode("act2", [np.array(0.05), np.array(0.4), np.array(0.7)]))
    g.add(G.AvgPoolNode("pool", 9, np.array(1.0 / 9)))
    g.add(G.LinearNode("fc", rng.normal(0, 0.3, (classes, 3)), rng.normal(0, 0.1, classes)))
    g.add(G.OutputNode("out"))
    order = ["in", "conv1", "act1", "conv2", "act2", "pool", "fc", "out"]
    for s, d in zip(order, order[1:]):
        g.connect(s, d)
    g.validate()
    return g


def chain_graph(nodes):
    g = G.ModelGraph()
    for n in nodes:
        g.add(n)
    for a, b in zip(nodes, nodes[1:]):
        g.connect(a.id, b.id)
    g.validate()
    return g


def act_conv(rng, coeffs):
    return chain_graph([G.InputNode("in", 2, 4, 4),
                        G.PolyActNode("act", [np.float64(c) for c in coeffs]),
                        G.ConvNode("conv", rng.standard_normal((2, 2, 3, 3)), rng.standard_normal(2), 1, 1),
                        G.OutputNode("out")])


def conv_act(rng, coeffs):
    return chain_graph([G.InputNode("in", 2, 4, 4),
                        G.ConvNode("conv", rng.standard_normal((2, 2, 3, 3)), rng.standard_normal(2), 1, 1),
                        G.PolyActNode("act", [np.float64(c) for c in coeffs]),
                        G.OutputNode("out")])


def pool_linear(rng):
    return chain_graph([G.InputNode("in", 2, 2, 2),
                        G.AvgPoolNode("pool", 4, np.float64(0.25)),
                        G.LinearNode("fc", rng.standard_normal((3, 2)), rng.standard_normal(3)),
                        G.OutputNode("out")])


def diag_pool_conv(c, k, stride, pad, divisor):
    """A k x k sum pool times divisor, written as a reference conv."""
    w = np.zeros((c, c, k, k))
    for i in range(c):
        w[i, i] = divisor
    return G.ConvNode("pool_as_conv", w, np.zeros(c), stride, pad)


def select_conv(nid, c, dy, dx):
    """2x2 stride-2 conv picking window element (dy, dx) of every channel."""
    w = np.zeros((c, c, 2, 2))
    for i in range(c):
        w[i, i, dy, dx] = 1.0
    return G.ConvNode(nid, w, np.zeros(c), 2, 0)


def main():
    arrays = {}
    cases = []

    def add_eval(name, g, xs):
        path = save(g, name)
        ys = np.stack([G.reference_eval(g, x) for x in xs])
        arrays[f"{name}/x"] = xs
        arrays[f"{name}/y"] = ys
        cases.append({"name": name, "model": path, "kind": "eval",
                      "ref": "levnet.graph.reference_eval (graph.py:413-426)"})

    rng = np.random.default_rng(20250922)

    # -- forward on reference-built graphs ---------------------------------
    fixture = G.load_model(REF_FIXTURE)
    add_eval("rn20_fixture", fixture, rng.uniform(-1, 1, (6, 3, 8, 8)))
    rn18 = None
    for v, seed in (("rn18", 1), ("rn20", 2), ("rn32", 3)):
        g = G.build_resnet_graph(v, act="poly2", seed=seed, input_hw=8)
        rn18 = g if v == "rn18" else rn18
        add_eval(f"{v}_poly2_s{seed}", g, rng.uniform(-1, 1, (4, 3, 8, 8)))
    add_eval("rn20_poly4", G.build_resnet_graph("rn20", act="poly4", seed=4, input_hw=8),
             rng.uniform(-1, 1, (4, 3, 8, 8)))
    add_eval("tiny_model", tiny_model(5), rng.uniform(-1, 1, (8, 2, 6, 6)))
    for stride, pad in ((1, 1), (2, 1), (1, 0), (2, 0), (3, 2)):
        g = chain_graph([G.InputNode("in", 3, 7, 7),
                         G.ConvNode("conv", rng.standard_normal((5, 3, 3, 3)), rng.standard_normal(5), stride, pad),
                         G.OutputNode("out")])
        add_eval(f"conv_s{stride}_p{pad}", g, rng.standard_normal((3, 3, 7, 7)))
    g = chain_graph([G.InputNode("in", 3, 5, 5),
                     G.PolyActNode("act", [rng.standard_normal(3) for _ in range(5)]),
                     G.OutputNode("out")])
    add_eval("polyact_perchannel_deg4", g, rng.standard_normal((3, 3, 5, 5)))
    g = G.ModelGraph()
    g.add(G.InputNode("in", 2, 4, 4))
    g.add(G.ConvNode("cx", rng.standard_normal((2, 2, 3, 3)), rng.standard_normal(2), 1, 1))
    g.add(G.BatchNormNode("bn", rng.uniform(0.5, 2, 2), rng.standard_normal(2),
                          rng.standard_normal(2), rng.uniform(0.5, 2, 2)))
    g.add(G.PolySkipNode("ps", {k: rng.standard_normal(2) for k in G.PS_KEYS}))
    g.add(G.OutputNode("out"))
    for s, d in (("in", "cx"), ("cx", "bn"), ("bn", "ps"), ("in", "ps"), ("ps", "out")):
        g.connect(s, d)
    g.validate()
    add_eval("bn_polyskip", g, rng.standard_normal((3, 2, 4, 4)))

    # -- extension differentials (reference-expressible equivalents) --------
    c = 3
    for k, s, p in ((2, 2, 0), (3, 2, 1)):
        g = chain_graph([G.InputNode("in", c, 8, 8), diag_pool_conv(c, k, s, p, 1.0 / (k * k)),
                         G.OutputNode("out")])
        add_eval(f"localpool_k{k}s{s}p{p}_as_conv", g, rng.standard_normal((3, c, 8, 8)))
    w_fc = rng.standard_normal((5, 4 * 3 * 3))
    b_fc = rng.standard_normal(5)
    g = chain_graph([G.InputNode("in", 4, 3, 3),
                     G.ConvNode("fc_as_conv", w_fc.reshape(5, 4, 3, 3), b_fc, 1, 0),
                     G.AvgPoolNode("unit", 1, np.float64(1.0)),
                     G.OutputNode("out")])
    add_eval("flatten_linear_as_conv", g, rng.standard_normal((3, 4, 3, 3)))
    arrays["flatten_linear_as_conv/w"] = w_fc
    arrays["flatten_linear_as_conv/b"] = b_fc
    # 2x2 pairwise quadratic pool: S_h(S_w(a, b), S_w(c, d)) via selection convs
    sw = {k: rng.standard_normal(c) for k in G.PS_KEYS}
    sh = {k: rng.standard_normal(c) for k in G.PS_KEYS}
    g = G.ModelGraph()
    g.add(G.InputNode("in", c, 6, 6))
    for nid, dy, dx in (("a", 0, 0), ("b", 0, 1), ("c", 1, 0), ("d", 1, 1)):
        g.add(select_conv(nid, c, dy, dx))
        g.connect("in", nid)
    g.add(G.PolySkipNode("top", dict(sw)))
    g.add(G.PolySkipNode("bot", dict(sw)))
    g.add(G.PolySkipNode("pool", dict(sh)))
    g.add(G.OutputNode("out"))
    for s, d in (("a", "top"), ("b", "top"), ("c", "bot"), ("d", "bot"),
                 ("top", "pool"), ("bot", "pool"), ("pool", "out")):
        g.connect(s, d)
    g.validate()
    add_eval("bipool2_as_polyskip", g, rng.standard_normal((3, c, 6, 6)))
    for k in G.PS_KEYS:
        arrays[f"bipool2_as_polyskip/sw/{k}"] = sw[k]
        arrays[f"bipool2_as_polyskip/sh/{k}"] = sh[k]

    # -- per-donor redistribution -------------------------------------------
    def add_rewrite(name, before, after, fn, xs=None):
        cases.append({"name": name, "kind": "rewrite", "before": save(before, name + "_before"),
                      "after": save(after, name + "_after"), "ref": fn})
        if xs is not None:
            arrays[f"{name}/x"] = xs
            arrays[f"{name}/y_after"] = np.stack([G.reference_eval(after, x) for x in xs])

    r = np.random.default_rng(0)
    g = act_conv(r, (9.0, 6.0, 3.0))
    add_rewrite("fwd_act_conv", g, T.redistribute_forward(g, "act"), "redistribute_forward (transforms.py:423)")
    g = conv_act(r, (1.0, 2.0, 4.0))
    add_rewrite("bwd_conv_act", g, T.redistribute_backward(g, "act"), "redistribute_backward (transforms.py:452)")
    g = conv_act(r, (0.3, -1.1, 0.2, 0.7))
    add_rewrite("bwd_conv_act_deg3", g, T.redistribute_backward(g, "act"), "redistribute_backward (transforms.py:452)")
    g = pool_linear(r)
    add_rewrite("fwd_pool_linear", g, T.redistribute_forward(g, "pool"), "redistribute_forward (transforms.py:423)")
    g = act_conv(r, (9.0, 6.0, 3.0))
    add_rewrite("fwd_act_conv_u2.5", g, T.redistribute_forward(g, "act", 2.5), "redistribute_forward upsilon=2.5")
    # donors on a ResNet that the reference accepts, each applied alone
    rn = G.build_resnet_graph("rn20", act="poly2", seed=7, input_hw=8)
    accepted_fwd, accepted_bwd, refused = [], [], {}
    picked = {"act1", "s1b1.acta", "s1b3.actj", "s2b1.acta", "s3b3.actj", "s3b2.acta", "pool"}
    for nid, node in rn.nodes.items():
        if not isinstance(node, (G.PolyActNode, G.AvgPoolNode)):
            continue
        for direction, fn, acc in (("forward", T.redistribute_forward, accepted_fwd),
                                   ("backward", T.redistribute_backward, accepted_bwd)):
            try:
                out = fn(rn, nid)
                acc.append(nid)
                if nid not in picked:
                    continue
                add_rewrite(f"rn20_{direction}_{nid}", rn, out, f"redistribute_{direction}",
                            rng.uniform(-1, 1, (2, 3, 8, 8)))
            except T.TransformError as e:
                refused[f"{direction}:{nid}"] = str(e)
    arrays["rn20_donors/x"] = rng.uniform(-1, 1, (2, 3, 8, 8))
    # sequential forward sweep over every accepted donor (composition)
    seq = rn
    for nid in [n for n in rn.topo_order() if n in accepted_fwd]:
        seq = T.redistribute_forward(seq, nid)
    add_rewrite("rn20_forward_sweep", rn, seq, "redistribute_forward, every accepted donor in topo order",
                rng.uniform(-1, 1, (3, 3, 8, 8)))

    # error cases: (graph, donor, direction, message fragment)
    errors = []
    g = conv_act(r, (1.0, 2.0, -4.0))
    try:
        T.redistribute_backward(g, "act")
    except T.TransformError as e:
        errors.append({"model": save(g, "err_negative_leading"), "donor": "act",
                       "direction": "backward", "message": str(e)})
    g = chain_graph([G.InputNode("in", 2, 2, 2), G.PolyActNode("act", [np.float64(1.0), np.float64(2.0)]),
                     G.OutputNode("out")])
    try:
        T.redistribute_forward(g, "act")
    except T.TransformError as e:
        errors.append({"model": save(g, "err_no_receiver"), "donor": "act",
                       "direction": "forward", "message": str(e)})
    g = chain_graph([G.InputNode("in", 2, 4, 4),
                     G.PolyActNode("act", [np.zeros(2), np.ones(2), np.array([1.0, 2.0])]),
                     G.ConvNode("conv", r.standard_normal((2, 2, 3, 3)), r.standard_normal(2), 1, 1),
                     G.OutputNode("out")])
    try:
        T.redistribute_forward(g, "act")
    except T.TransformError as e:
        errors.append({"model": save(g, "err_per_channel"), "donor": "act",
                       "direction": "forward", "message": str(e)})

    # -- channelwise pass and pipelines --------------------------------------
    for strategy in ("P2R", "P2FR", "P2F"):
        out, rep = T.apply_pipeline(fixture, strategy)
        add_rewrite(f"fixture_{strategy}", fixture, out, f"apply_pipeline({strategy}) (transforms.py:712)",
                    rng.uniform(-1, 1, (3, 3, 8, 8)))
        cases[-1]["depth"] = [rep.depth_before, rep.depth_after]
        cases[-1]["rewrites"] = [[rw, list(ids)] for rw, ids in rep.rewrites]
    for v, g in (("rn18", rn18),):
        out, rep = T.apply_pipeline(g, "P2FR")
        add_rewrite(f"{v}_P2FR", g, out, "apply_pipeline(P2FR)", rng.uniform(-1, 1, (2, 3, 8, 8)))
    g4 = G.build_resnet_graph("rn20", act="poly4", seed=1, input_hw=8)
    out, rw = T.redistribute_pass(g4)
    add_rewrite("rn20_poly4_pass", g4, out, "redistribute_pass on degree 4 (transforms.py:575)",
                rng.uniform(-1, 1, (2, 3, 8, 8)))
    cases[-1]["rewrites"] = [[a, list(b)] for a, b in rw]

    # -- equivalence numbers ------------------------------------------------
    p2fr = next(c for c in cases if c["name"] == "fixture_P2FR")
    out = _SAVED_GRAPH(p2fr["after"])
    rep = T.check_equivalence(fixture, out, n_inputs=20, rtol=1e-8, seed=3)
    equiv = {"model_ref": p2fr["before"], "model_cand": p2fr["after"],
             "n_inputs": 20, "seed": 3, "max_rel_err": rep.max_rel_err,
             "argmax_match_rate": rep.argmax_match_rate, "passed": rep.passed}

    np.savez_compressed(HERE / "golden.npz", **arrays)
    manifest = {"generator": "tests/golden/make_golden.py", "reference": REF_SRC,
                "cases": cases, "errors": errors, "equivalence": equiv,
                "rn20_donors": {"forward": accepted_fwd, "backward": accepted_bwd,
                                "refused": refused}}
    with open(HERE / "manifest.json", "w") as f:
        json.dump(manifest, f, indent=1)
    print(f"{len(cases)} cases, {len(errors)} error cases, "
          f"{os.path.getsize(HERE / 'golden.npz') / 1024:.0f} KiB npz")


if __name__ == "__main__":
    main()
