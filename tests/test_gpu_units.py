"""Every unit of every configuration against the float64 oracle, tensor by
tensor: after one batched forward, each unit's output is read back from the
workspace (decoded from its storage format: float32 blocked, split fp16
hi/lo, or split parity planes) and compared with the oracle value of the last
graph node fused into that unit.  The logits alone are a weak check on the
input-insensitive configs (RN18's vary by ~0.5% across images), so this is
where a wrong intermediate shows."""

import numpy as np
import pytest

from oracle import levnet_oracle as O
from paper_2509_22857_b200 import configs
from paper_2509_22857_b200.runtime import Engine

pytestmark = pytest.mark.gpu

N_IMAGES = {"lenet5": 16, "resnet20": 16, "resnet20_deg8": 16, "vgg11": 8, "resnet18": 4}


def oracle_values(g, x):
    """float64 value of every node for a batch (reference_eval's node
    kernels with a batch axis, oracle eval_batch_values)."""
    return O.eval_batch_values(g, x)


@pytest.mark.parametrize("name", list(configs.CONFIGS))
@pytest.mark.parametrize("impl,blocks", [(0, 2), (0, 0), (4, 2)], ids=["auto", "per_layer", "fp32_tensors"])
def test_every_unit_matches_oracle(cuda, name, impl, blocks):
    """auto: the default plan (image-resident runs keep their inner outputs
    in shared memory, so only the units whose outputs leave the run are
    read); per_layer: options.image_blocks = 0, every unit's output is in the
    workspace."""
    import torch
    from paper_2509_22857_b200 import _lib as L
    g = configs.build(name)
    n = N_IMAGES[name]
    x = configs.make_input(configs.CONFIGS[name], batch=n)
    # per_layer also runs small networks unit by unit (options.fused_net = 0)
    eng = Engine(g, impl=impl, options=L.PlanOptions.default(image_blocks=blocks, fused_net=int(blocks > 0)))
    y = eng.forward(torch.from_numpy(x.astype(np.float32)).cuda())
    torch.cuda.synchronize()
    plan = eng.plan(n)
    want = oracle_values(g, x)
    # plain float32 FMA (SIMT kernels, float32 tensors) as the fp32-class yardstick
    simt = Engine(g, impl=1)
    simt.forward(torch.from_numpy(x.astype(np.float32)).cuda())
    torch.cuda.synchronize()
    splan = simt.plan(n)
    checked = 0
    for i, (u, chain) in enumerate(zip(eng.lw.units, eng.lw.unit_nodes)):
        if u["kind"] in (1, 12) or u.get("out", -1) < 0 or not plan.materialized(i):  # ingest / copyout
            continue
        got = plan.read_tensor(u["out"]).astype(np.float64)
        ref = want[chain[-1]].reshape(got.shape)
        scale = max(float(np.abs(ref).max()), 1e-30)
        err = float(np.abs(got - ref).max()) / scale
        err_simt = float(np.abs(splan.read_tensor(u["out"]).astype(np.float64) - ref).max()) / scale
        # errors accumulate through the network in both paths, and deep layers
        # with cancelling contributions amplify them (max|err| is taken relative
        # to the tensor's max, not to the terms): the tensor-core path must stay
        # within the north-star 1e-4 or within 4x plain fp32 FMA's error.  A
        # wrong unit shows up at 1e-2 .. 1.
        assert err <= max(1e-4, 4 * err_simt), (name, i, chain, plan.unit_impl(i), plan.tensor_split(u["out"]),
                                                 err, err_simt)
        checked += 1
    # a whole-network launch (impl 7) stores only the logits vector
    assert checked >= (1 if plan.unit_impl(1) == 7 else 3)
    np.testing.assert_allclose(y.double().cpu().numpy(), want[g.output_id()].reshape(n, -1), rtol=1e-4, atol=1e-5)
