"""Golden fixtures for checkpoint ingest (paper_2509_22857_b200/checkpoint.py).

Run in the build container, where the reference exporter is importable:

    python tests/golden/make_ckpt_golden.py

Builds seeded synthetic ResNet state dicts (the usual torch key naming, with
embedded activation coefficients, plus one without them), saves them as .npz
checkpoints, and converts them with the reference's own
``levnet_exporter.exporting.export_state`` (validation off: it shells out to
the levnet CLI) into ``tests/golden/models/ckpt_*_ref.json``.  The test
compares this package's conversion with those files.  Nothing here runs at
test time.
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/exporter/src")
from levnet_exporter.exporting import export_state  # noqa: E402

HERE = pathlib.Path(__file__).resolve().parent


def synth_state(variant: str, width: int, cin: int, classes: int, deg: int, seed: int, coeffs: bool):
    rng = np.random.default_rng(seed)
    stages = {"rn20": (3, 3, 3), "rn18": (2, 2, 2, 2)}[variant]
    s = {}

    def conv(k, a, b, ks, bias=False):
        s[f"{k}.weight"] = rng.normal(0, np.sqrt(2.0 / (a * ks * ks)), (b, a, ks, ks))
        if bias:
            s[f"{k}.bias"] = rng.normal(0, 0.1, b)

    def bn(k, c):
        s[f"{k}.weight"] = rng.uniform(0.2, 0.5, c)
        s[f"{k}.bias"] = rng.normal(0, 0.1, c)
        s[f"{k}.running_mean"] = rng.normal(0, 0.1, c)
        s[f"{k}.running_var"] = rng.uniform(0.5, 2.0, c)
        s[f"{k}.num_batches_tracked"] = np.asarray(100.0)

    def act(k):
        if coeffs:
            # near-identity polynomials keep an untrained deep poly net finite
            c = rng.normal(0, 0.02, deg + 1) / np.arange(1, deg + 2) ** 2
            c[1] = rng.uniform(0.8, 1.2)
            c[-1] = rng.uniform(0.02, 0.1) / 4 ** (deg - 2)
            s[f"{k}.coeffs"] = c

    conv("conv1", cin, width, 3, bias=True)
    bn("bn1", width)
    act("act1")
    w = width
    for si, blocks in enumerate(stages):
        cout = width * 2 ** si
        for bi in range(blocks):
            pre = f"layer{si + 1}.{bi}"
            conv(f"{pre}.conv1", w, cout, 3)
            bn(f"{pre}.bn1", cout)
            act(f"{pre}.act1")
            conv(f"{pre}.conv2", cout, cout, 3)
            bn(f"{pre}.bn2", cout)
            act(f"{pre}.act2")
            if bi == 0 and si > 0:
                conv(f"{pre}.downsample.0", w, cout, 1)
                bn(f"{pre}.downsample.1", cout)
            w = cout
    s["fc.weight"] = rng.normal(0, np.sqrt(1.0 / w), (classes, w))
    s["fc.bias"] = rng.normal(0, 0.1, classes)
    return s


CASES = [
    # name, variant, width, in channels, classes, degree, seed, embedded coeffs, input_hw
    ("ckpt_rn20_w4", "rn20", 4, 3, 10, 2, 11, True, 8),
    ("ckpt_rn18_w4", "rn18", 4, 3, 7, 4, 12, True, 16),
    ("ckpt_rn20_w4_shared", "rn20", 4, 3, 10, 2, 13, False, 8),
]
SHARED_COEFFS = [0.01, 1.0, 0.05]


def main() -> None:
    (HERE / "models").mkdir(exist_ok=True)
    for name, variant, width, cin, classes, deg, seed, emb, hw in CASES:
        st = synth_state(variant, width, cin, classes, deg, seed, emb)
        np.savez(HERE / f"{name}.npz", **st)
        if emb:
            export_state(st, variant, str(HERE / "models" / f"{name}_ref.json"), ckpt_label=name,
                         input_hw=hw, validate=False)
        else:
            cf = HERE / f"{name}_coeffs.json"
            cf.write_text('{"real_coeffs": %s}\n' % SHARED_COEFFS)
            export_state(st, variant, str(HERE / "models" / f"{name}_ref.json"), ckpt_label=name,
                         coeffs_file=str(cf), input_hw=hw, validate=False)
            cf.unlink()
        print("wrote", name)


if __name__ == "__main__":
    main()
