"""Config numerics gate ("assert finite, input-sensitive
logits before any perf run"): float64 forward of each configuration on its
measured input batch (RN18: the first 8 images) must be finite everywhere and
the logits must vary with the input."""

import numpy as np
import pytest

from paper_2509_22857_b200 import configs

BATCH = {"resnet18": 8}


@pytest.mark.parametrize("name", list(configs.CONFIGS))
def test_config_finite_and_input_sensitive(name):
    cfg = configs.CONFIGS[name]
    g = configs.build(name)
    x = configs.make_input(cfg, batch=BATCH.get(name))
    st = configs.forward_stats(g, x)
    y = st.pop("__out__")
    assert all(np.isfinite(v) for v in st.values()), name
    assert np.all(np.isfinite(y)), name
    # batch std of the logits relative to their magnitude (A.2's sensitivity
    # measure; RN18-224 and VGG with bivariate pools sit near 2e-3)
    sens = float((y.std(0) / np.abs(y).mean(0)).mean())
    assert sens > 1e-3, (name, sens)
    # no single image dominates (a diverging tail would)
    per_image = np.abs(y).max(1)
    assert per_image.max() <= 20 * np.median(per_image), name
