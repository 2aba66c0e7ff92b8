"""Seeded builders for the five benchmark configurations (BASELINE.json).

Each returns a ``ModelGraph`` in the reference IR (plus the extension nodes
for local pools, flatten and bivariate pools), with float64 parameters:

=============  =====  ===========  ===============================================
name           batch  input        network
=============  =====  ===========  ===============================================
lenet5            64  1x28x28 N01  conv5 1-6, p2, 2x2 avg, conv5 6-16, p2, 2x2 avg,
                                   flatten, fc 256-120, p2, fc 120-84, p2, fc 84-10
resnet20         256  3x32x32 N01  3x3 stem, 3x3 basic blocks 16/32/64, 1x1/s2
                                   projections, deg-2 acts, global 8x8 avg, fc 64-10
resnet20_deg8    512  N01 clip 8   same topology, deg-8 LSQ ReLU fits on [-8, 8]
vgg11            128  3x32x32 U11  VGG-11 convs, deg-3 acts, every 2x2 max pool
                                   replaced by pairwise deg-4 bivariate S(x, y)
resnet18          64  3x224² N01   7x7/s2 stem, 3x3/s2 avg pool, basic blocks
                                   64..512, deg-4 acts, global 7x7 avg, fc 512-1000
=============  =====  ===========  ===============================================

Initialisation follows SURVEY.md App. A.2 ("calibrated BN fold"): Kaiming
normal weights and zero bias, then -- in topological order, on a seeded
calibration batch -- each conv's output is standardised per channel and
scaled to a target gain s (s_res for the second conv of a residual block),
which is exactly folding a batch-statistics batchnorm into the conv.  The
literal Kaiming init overflows float64 on the deep configs.
Calibration statistics are computed with torch in float64 at construction
time only; inference never runs here.

Synthetic data stands in for MNIST / CIFAR / ImageNet (no datasets offline):
parameters use default_rng(seed), calibration default_rng(seed + 1), the
measured batch default_rng(seed + 2).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Set, Tuple

import numpy as np

from .graph import (AddNode, AvgPoolNode, BiPoolNode, ConvNode, FlattenNode, InputNode, LinearNode,
                    LocalPoolNode, ModelGraph, OutputNode, PolyActNode)


@dataclass
class Config:
    name: str
    batch: int
    input_shape: Tuple[int, int, int]
    input_dist: str            # "normal", "normal_clip8", "uniform"
    redistribution: Tuple[str, ...]  # sweep directions applied in order
    allow_negative_leading: bool
    description: str


CONFIGS: Dict[str, Config] = {
    "lenet5": Config("lenet5", 64, (1, 28, 28), "normal", ("forward",), False,
                     "LeNet-5-shaped poly CNN, deg-2 acts, 2x2 avg pools, FC 256-120-84-10"),
    "resnet20": Config("resnet20", 256, (3, 32, 32), "normal", ("forward",), False,
                       "ResNet-20-shaped poly CNN, deg-2 acts, BN folded, global 8x8 pool, FC 64-10"),
    "resnet20_deg8": Config("resnet20_deg8", 512, (3, 32, 32), "normal_clip8", ("backward",), True,
                            "ResNet-20 topology, deg-8 LSQ-ReLU acts on [-8,8], update-backward"),
    "vgg11": Config("vgg11", 128, (3, 32, 32), "uniform", ("forward",), False,
                    "VGG-11-shaped CNN, deg-3 acts, pairwise deg-4 bivariate pools, FC 512-10"),
    "resnet18": Config("resnet18", 64, (3, 224, 224), "normal", ("backward", "forward"), False,
                       "ResNet-18-shaped poly CNN at 224^2, deg-4 acts, 3x3/s2 avg stem pool, FC 512-1000"),
}


def make_input(cfg: Config, batch: Optional[int] = None, seed: int = 2, hw: Optional[int] = None) -> np.ndarray:
    rng = np.random.default_rng(seed)
    c, h, w = cfg.input_shape
    if hw:
        h = w = hw
    shape = (batch or cfg.batch, c, h, w)
    if cfg.input_dist == "uniform":
        return rng.uniform(-1.0, 1.0, shape)
    x = rng.normal(0.0, 1.0, shape)
    if cfg.input_dist == "normal_clip8":
        x = np.clip(x, -8.0, 8.0)
    return x


def relu_lsq_fit(degree: int, lo: float = -8.0, hi: float = 8.0, n: int = 4097) -> np.ndarray:
    """Least-squares polynomial fit of ReLU on [lo, hi] (coefficients c_0..c_d)."""
    x = np.linspace(lo, hi, n)
    return np.polynomial.polynomial.polyfit(x, np.maximum(x, 0.0), degree)


# ---------------------------------------------------------------------------
# graph construction helpers
# ---------------------------------------------------------------------------

class _Net:
    def __init__(self, seed: int, in_shape):
        self.rng = np.random.default_rng(seed)
        self.g = ModelGraph()
        self.g.add(InputNode("in", *in_shape))
        self.res_convs: Set[str] = set()
        self.n = 0

    def _id(self, stem: str) -> str:
        self.n += 1
        return f"{stem}{self.n}"

    def conv(self, src: str, cin: int, cout: int, k: int, stride: int, pad: int, name: str = None,
             residual: bool = False) -> str:
        nid = name or self._id("conv")
        w = self.rng.normal(0.0, np.sqrt(2.0 / (cin * k * k)), (cout, cin, k, k))
        self.g.add(ConvNode(nid, w, np.zeros(cout), stride, pad))
        self.g.connect(src, nid)
        if residual:
            self.res_convs.add(nid)
        return nid

    def act(self, src: str, coeffs: List[float], name: str = None) -> str:
        nid = name or self._id("act")
        self.g.add(PolyActNode(nid, [np.asarray(float(c)) for c in coeffs]))
        self.g.connect(src, nid)
        return nid

    def add(self, x: str, y: str, name: str = None) -> str:
        nid = name or self._id("join")
        self.g.add(AddNode(nid))
        self.g.connect(x, nid)
        self.g.connect(y, nid)
        return nid

    def node(self, src: str, node) -> str:
        self.g.add(node)
        self.g.connect(src, node.id)
        return node.id

    def linear(self, src: str, n_in: int, n_out: int, name: str = None) -> str:
        nid = name or self._id("fc")
        w = self.rng.normal(0.0, np.sqrt(2.0 / n_in), (n_out, n_in))
        self.g.add(LinearNode(nid, w, np.zeros(n_out)))
        self.g.connect(src, nid)
        return nid

    def finish(self, src: str) -> ModelGraph:
        self.g.add(OutputNode("out"))
        self.g.connect(src, "out")
        self.g.validate()
        return self.g


# ---------------------------------------------------------------------------
# calibration (construction time only; torch float64)
# ---------------------------------------------------------------------------

def _calibrate(g: ModelGraph, x: np.ndarray, gain: float, gain_res: float, res_convs: Set[str],
               skip: Set[str] = frozenset(), stats: Optional[Dict] = None) -> None:
    """Fold a batch-statistics batchnorm with target gain into every conv
    (convs in `skip` are only evaluated).  With `stats`, record max|value|
    per node and the logits instead of raising on non-finite values."""
    import torch
    import torch.nn.functional as F

    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    dt = torch.float64
    preds = {nid: g.inputs_of(nid) for nid in g.nodes}
    vals: Dict[str, torch.Tensor] = {"in": torch.as_tensor(x, dtype=dt, device=dev)}

    def t(a):
        return torch.as_tensor(np.asarray(a, dtype=np.float64), dtype=dt, device=dev)

    def poly(cs, v):
        acc = torch.zeros_like(v) + t(cs[-1]).reshape(-1, 1, 1) if np.asarray(cs[-1]).ndim else \
            torch.full_like(v, float(cs[-1]))
        for c in reversed(cs[:-1]):
            cc = t(c)
            acc = acc * v + (cc.reshape(-1, 1, 1) if cc.ndim else cc)
        return acc

    def bivar(c, xa, ya):
        c = np.asarray(c, dtype=np.float64)
        d = c.shape[0] - 1
        out = torch.zeros_like(xa)
        for i in range(d + 1):
            for j in range(d + 1 - i):
                cij = t(c[i, j])
                out = out + (cij.reshape(-1, 1, 1) if cij.ndim else cij) * xa ** i * ya ** j
        return out

    for nid in g.topo_order():
        if nid == "in":
            continue
        node = g.nodes[nid]
        ins = [vals[p] for p in preds[nid]]
        if isinstance(node, ConvNode):
            raw = F.conv2d(ins[0], t(node.weight), None, node.stride, node.padding)
            if nid not in skip:
                mu = raw.mean(dim=(0, 2, 3))
                sd = raw.std(dim=(0, 2, 3), unbiased=False).clamp_min(1e-12)
                s = gain_res if nid in res_convs else gain
                scale = (s / sd).cpu().numpy()
                node.weight = node.weight * scale[:, None, None, None]
                node.bias = (-mu.cpu().numpy()) * scale
            vals[nid] = F.conv2d(ins[0], t(node.weight), t(node.bias), node.stride, node.padding)
        elif isinstance(node, PolyActNode):
            vals[nid] = poly(node.coeffs, ins[0])
        elif isinstance(node, AddNode):
            vals[nid] = ins[0] + ins[1]
        elif isinstance(node, LocalPoolNode):
            vals[nid] = F.avg_pool2d(ins[0], node.k, node.stride, node.padding, count_include_pad=True) \
                * (node.k * node.k * float(node.divisor))
        elif isinstance(node, BiPoolNode):
            v = ins[0]
            a, b = (v[:, :, :, 0::2], v[:, :, :, 1::2]) if node.axis == "w" else (v[:, :, 0::2, :], v[:, :, 1::2, :])
            vals[nid] = bivar(node.coeffs, a, b)
        elif isinstance(node, AvgPoolNode):
            vals[nid] = ins[0].sum(dim=(2, 3)) * float(node.divisor)
        elif isinstance(node, FlattenNode):
            vals[nid] = ins[0].reshape(ins[0].shape[0], -1)
        elif isinstance(node, LinearNode):
            vals[nid] = ins[0] @ t(node.weight).T + t(node.bias)
        elif isinstance(node, OutputNode):
            vals[nid] = ins[0]
        else:
            raise ValueError(f"calibration cannot evaluate {node.kind}")
        if stats is not None:
            stats[nid] = float(vals[nid].abs().max())
            if isinstance(node, OutputNode):
                stats["__out__"] = vals[nid].cpu().numpy()
        elif not torch.isfinite(vals[nid]).all():
            raise FloatingPointError(f"calibration diverged at {nid}")


# ---------------------------------------------------------------------------
# the five configurations
# ---------------------------------------------------------------------------

def lenet5(seed: int = 0) -> ModelGraph:
    """Config 1 (literal init is finite and input-sensitive; no calibration)."""
    net = _Net(seed, (1, 28, 28))
    r = net.rng

    def coeffs():
        return [r.normal(0, 0.3), r.normal(0, 0.3), r.uniform(0.05, 0.5)]

    h = net.conv("in", 1, 6, 5, 1, 0, "conv1")
    h = net.act(h, coeffs(), "act1")
    h = net.node(h, LocalPoolNode("pool1", 2, 2, 0, np.asarray(0.25)))
    h = net.conv(h, 6, 16, 5, 1, 0, "conv2")
    h = net.act(h, coeffs(), "act2")
    h = net.node(h, LocalPoolNode("pool2", 2, 2, 0, np.asarray(0.25)))
    h = net.node(h, FlattenNode("flatten"))
    h = net.linear(h, 256, 120, "fc1")
    h = net.act(h, coeffs(), "act3")
    h = net.linear(h, 120, 84, "fc2")
    h = net.act(h, coeffs(), "act4")
    h = net.linear(h, 84, 10, "fc3")
    return net.finish(h)


def _resnet_cifar(seed: int, act_coeffs: Callable[[np.random.Generator], List[float]], hw: int,
                  gain: float, gain_res: float, calib_x: np.ndarray, widths=(16, 32, 64), blocks=3,
                  classes: int = 10) -> ModelGraph:
    net = _Net(seed, (3, hw, hw))
    r = net.rng
    h = net.conv("in", 3, widths[0], 3, 1, 1, "conv1")
    h = net.act(h, act_coeffs(r), "act1")
    cin = widths[0]
    for si, w in enumerate(widths):
        for bi in range(blocks):
            name = f"s{si + 1}b{bi + 1}"
            stride = 2 if (bi == 0 and si > 0) else 1
            a = net.conv(h, cin, w, 3, stride, 1, f"{name}.conva")
            a = net.act(a, act_coeffs(r), f"{name}.acta")
            b = net.conv(a, w, w, 3, 1, 1, f"{name}.convb", residual=True)
            skip = h if stride == 1 and cin == w else net.conv(h, cin, w, 1, stride, 0, f"{name}.convd")
            j = net.add(b, skip, f"{name}.join")
            h = net.act(j, act_coeffs(r), f"{name}.actj")
            cin = w
    side = hw // 4
    h = net.node(h, AvgPoolNode("pool", side * side, np.asarray(1.0 / (side * side))))
    h = net.linear(h, cin, classes, "fc")
    g = net.finish(h)
    _calibrate(g, calib_x, gain, gain_res, net.res_convs)
    return g


def _deg2(r):
    return [r.normal(0.0, 0.1), r.normal(0.5, 0.1), r.uniform(0.05, 0.5)]


def resnet20(seed: int = 0, hw: int = 32, gain: float = 0.2, gain_res: float = 0.1) -> ModelGraph:
    """Config 2: deg-2 acts c2~U(0.05,0.5), c1~N(0.5,0.1), c0~N(0,0.1);
    s=0.2, s_res=0.1 (SURVEY's s=0.3 sends one image of the measured batch of
    256 to 1e50 in float64 -- a degree-2^9 tail; s=0.2 keeps every image
    finite and input-sensitive)."""
    cal = make_input(CONFIGS["resnet20"], batch=64, seed=seed + 1, hw=hw)
    return _resnet_cifar(seed, _deg2, hw, gain, gain_res, cal)


def resnet20_deg8(seed: int = 0, hw: int = 32, gain: float = 0.4, gain_res: float = 0.05) -> ModelGraph:
    """Config 3: each act = LSQ ReLU fit on [-8,8] times (1 + N(0, 0.01));
    s=0.4, s_res=0.05 (SURVEY's s=0.5 overflows float64 on one image of the
    measured batch of 512; 0.4 keeps the pre-activations within ~[-10, 10])."""
    base = relu_lsq_fit(8)

    def act(r):
        return list(base * (1.0 + r.normal(0.0, 0.01, base.size)))

    cal = make_input(CONFIGS["resnet20_deg8"], batch=64, seed=seed + 1, hw=hw)
    return _resnet_cifar(seed, act, hw, gain, gain_res, cal)


def _bivariate(r, d: int = 4) -> np.ndarray:
    c = r.normal(0.0, 0.2, (d + 1, d + 1))
    i, j = np.indices(c.shape)
    c[(i + j) > d] = 0.0
    c[d, 0] = r.uniform(0.05, 0.3)
    return c


def vgg11(seed: int = 0, hw: int = 32, gain: float = 0.25) -> ModelGraph:
    """Config 4: VGG-11 convs, deg-3 acts, each max pool -> S_w then S_h with
    the same deg-4 S (c40~U(0.05,0.3), others N(0,0.2)); s=0.25 (s=0.4 lets
    the degree-16 pool composition overflow on calibration tails)."""
    net = _Net(seed, (3, hw, hw))
    r = net.rng
    plan = [64, "M", 128, "M", 256, 256, "M", 512, 512, "M", 512, 512, "M"]
    h, cin, side, k = "in", 3, hw, 0
    for item in plan:
        if item == "M":
            k += 1
            s = _bivariate(r)
            h = net.node(h, BiPoolNode(f"pool{k}w", "w", s.copy()))
            h = net.node(h, BiPoolNode(f"pool{k}h", "h", s.copy()))
            side //= 2
            continue
        h = net.conv(h, cin, item, 3, 1, 1)
        h = net.act(h, [r.normal(0.0, 0.1), r.normal(0.5, 0.1), r.uniform(0.05, 0.3), r.uniform(0.01, 0.1)])
        cin = item
    h = net.node(h, FlattenNode("flatten"))
    h = net.linear(h, cin * side * side, 10, "fc")
    g = net.finish(h)
    _calibrate(g, make_input(CONFIGS["vgg11"], batch=64, seed=seed + 1, hw=hw), gain, gain, set())
    return g


def resnet18(seed: int = 0, hw: int = 224, calib_batch: int = 8, gain: float = 0.1,
             gain_res: float = 0.02) -> ModelGraph:
    """Config 5: 7x7/s2 stem, 3x3/s2 avg pool (divisor 1/9), 2 basic blocks per
    stage at 64/128/256/512, deg-4 acts (c4~U(0.02,0.2), others N(0,0.3)),
    global pool, FC 512-1000; s=0.1, s_res=0.02."""
    net = _Net(seed, (3, hw, hw))
    r = net.rng

    def act(rr):
        return [rr.normal(0, 0.3), rr.normal(0, 0.3), rr.normal(0, 0.3), rr.normal(0, 0.3), rr.uniform(0.02, 0.2)]

    h = net.conv("in", 3, 64, 7, 2, 3, "conv1")
    h = net.act(h, act(r), "act1")
    h = net.node(h, LocalPoolNode("pool0", 3, 2, 1, np.asarray(1.0 / 9.0)))
    cin = 64
    for si, w in enumerate((64, 128, 256, 512)):
        for bi in range(2):
            name = f"s{si + 1}b{bi + 1}"
            stride = 2 if (bi == 0 and si > 0) else 1
            a = net.conv(h, cin, w, 3, stride, 1, f"{name}.conva")
            a = net.act(a, act(r), f"{name}.acta")
            b = net.conv(a, w, w, 3, 1, 1, f"{name}.convb", residual=True)
            skip = h if stride == 1 and cin == w else net.conv(h, cin, w, 1, stride, 0, f"{name}.convd")
            j = net.add(b, skip, f"{name}.join")
            h = net.act(j, act(r), f"{name}.actj")
            cin = w
    side = -(-hw // 32)
    h = net.node(h, AvgPoolNode("pool", side * side, np.asarray(1.0 / (side * side))))
    h = net.linear(h, 512, 1000, "fc")
    g = net.finish(h)
    cal = make_input(CONFIGS["resnet18"], batch=calib_batch, seed=seed + 1, hw=hw)
    _calibrate(g, cal, gain, gain_res, net.res_convs)
    return g


def forward_stats(g: ModelGraph, x: np.ndarray) -> Dict:
    """float64 torch forward of a batch: {node: max|value|, "__out__": logits}
    (config-numerics probe; never on the measured path)."""
    stats: Dict = {}
    convs = {nid for nid, n in g.nodes.items() if isinstance(n, ConvNode)}
    _calibrate(g, x, 1.0, 1.0, set(), skip=convs, stats=stats)
    return stats


BUILDERS = {"lenet5": lenet5, "resnet20": resnet20, "resnet20_deg8": resnet20_deg8,
            "vgg11": vgg11, "resnet18": resnet18}


def build(name: str, seed: int = 0, **kw) -> ModelGraph:
    """Build a configuration by name; 'rn20' style aliases accepted."""
    alias = {"rn20": "resnet20", "rn20_deg8": "resnet20_deg8", "rn18": "resnet18", "lenet": "lenet5"}
    name = alias.get(name, name)
    if "batch_hw" in kw:
        kw["hw"] = kw.pop("batch_hw")
    kw.pop("scale", None)
    return BUILDERS[name](seed=seed, **kw)
