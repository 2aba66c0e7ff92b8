"""Device-resident engine: float64 master parameters, packed float32 images,
execution plans, and the batched GPU forward.

``Engine(g)`` uploads a graph once; ``forward`` runs the fused network on the
GPU (CUDA-graph replay inside libpcnn); ``redistribute`` runs a compiled
redistribution program in place on the device master and re-packs; and
``to_graph`` downloads the parameters into a new ``ModelGraph``.

Drop-in functions with the reference's names live here too:
``reference_eval(g, image)`` (reference graph.py:413-426) and the batched
``forward(g, x)``.  They run on the GPU -- there is no CPU fallback; without
libpcnn.so or a B200 they raise ``PcnnError``.
"""

from __future__ import annotations

import ctypes
import dataclasses
import weakref
from typing import Dict, Optional, Tuple

import numpy as np

from . import _lib as L
from .graph import GraphError, ModelGraph
from .lowering import Lowered, graph_from_master, lower, master_array


def _torch():
    import torch
    return torch


def _stream_handle(stream=None) -> ctypes.c_void_p:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Plan:
    """A libpcnn plan for one batch size: workspace + unit table."""

    def __init__(self, engine: "Engine", batch: int, impl: int = 0, options: Optional[L.PlanOptions] = None):
        torch = _torch()
        lw = engine.lw
        self.batch = batch
        tdescs, floats = lw.tensor_descs(batch, engine.scale_log2)
        self.ws = torch.zeros(max(floats, 1), dtype=torch.float32, device=engine.device)
        self.units = lw.unit_descs(impl)
        self.tdescs = tdescs
        self.options = options if options is not None else L.PlanOptions.default()
        handle = ctypes.c_void_p()
        L.check(L.lib().pcnn_plan_create_ex(self.units, len(lw.units), tdescs, len(lw.tensors), batch,
                                            lw.input_tensor, lw.output_tensor,
                                            ctypes.c_void_p(engine.packed.data_ptr()),
                                            ctypes.c_void_p(self.ws.data_ptr()),
                                            self.ws.numel() * 4, ctypes.byref(self.options),
                                            ctypes.byref(handle)),
                "pcnn_plan_create")
        self.handle = handle
        self.n_units = len(lw.units)

    def launches(self) -> int:
        return L.lib().pcnn_plan_num_launches(self.handle)

    def unit_impl(self, i: int) -> int:
        return L.lib().pcnn_plan_unit_impl(self.handle, i)

    def materialized(self, i: int) -> bool:
        """False for a unit inside an image-resident run (options.image_blocks)
        whose output stays in shared memory: every unit of the run but the
        last (read_tensor of its output tensor returns stale workspace)."""
        lib = L.lib()
        n = len(self.units)
        if self.unit_impl(i) == 7:  # whole-network launch: only the output vector is stored
            return self.units[i].out == self.units[n - 1].in_
        return not (self.unit_impl(i) == 6 and i + 1 < n and lib.pcnn_plan_unit_impl(self.handle, i + 1) == 6
                    and lib.pcnn_plan_unit_launch(self.handle, i + 1) == lib.pcnn_plan_unit_launch(self.handle, i))

    def tensor_split(self, t: int) -> int:
        """0 float32, 1 split fp16 hi/lo (padded grid), 2 split in parity planes."""
        return L.lib().pcnn_plan_tensor_split(self.handle, t)

    def status(self, stream=None) -> int:
        """Status word of the last forward on `stream` (synchronises it)."""
        rc = L.lib().pcnn_plan_status(self.handle, _stream_handle(stream))
        if rc < 0:
            L.check(rc, "pcnn_plan_status")
        return rc

    def last_status(self) -> int:
        return L.lib().pcnn_plan_last_status(self.handle)

    def unit_launch(self, i: int) -> int:
        """The unit whose kernel launch computes unit i (i unless fused)."""
        return L.lib().pcnn_plan_unit_launch(self.handle, i)

    def timeline(self, stream=None) -> np.ndarray:
        """(n_units, 2) int64 %globaltimer ns of the last forward: when each
        unit's launch released its first CTA past the dependency wait, and
        when its last CTA exited (0, 0 for units run inside another launch).
        Synchronises the stream."""
        buf = (L.c_i64 * (2 * self.n_units))()
        n = L.lib().pcnn_plan_timeline(self.handle, buf, self.n_units, _stream_handle(stream))
        if n < 0:
            L.check(n, "pcnn_plan_timeline")
        return np.frombuffer(buf, dtype=np.int64).reshape(self.n_units, 2).copy()

    def timeline_passes(self, stream=None) -> np.ndarray:
        """(2 n_units, 2): rows [0, n) as `timeline`, row n + u the pooling
        pass launched after pooled conv unit u (0, 0 when it has none)."""
        m = 2 * self.n_units
        buf = (L.c_i64 * (2 * m))()
        n = L.lib().pcnn_plan_timeline(self.handle, buf, m, _stream_handle(stream))
        if n < 0:
            L.check(n, "pcnn_plan_timeline")
        return np.frombuffer(buf, dtype=np.int64).reshape(m, 2).copy()

    def read_tensor(self, t: int) -> np.ndarray:
        """Copy tensor t out of the workspace, decoded from its storage format
        (csrc/common.cuh) to float32 (B, C, H, W), or (B, C) for vectors.
        Debug / test aid; synchronises the device."""
        desc = self.tdescs[t]
        c, h, w, cb, nblk = int(desc.c), int(desc.h), int(desc.w), int(desc.cb), int(desc.nblk)
        b, cpad = self.batch, nblk * cb
        base = int(desc.offset)
        fmt = self.tensor_split(t)
        if desc.is_vector:
            return self.ws[base:base + b * cpad].view(b, cpad)[:, :c].cpu().numpy()
        if fmt == 0:
            x = self.ws[base:base + b * cpad * h * w].view(b, nblk, h, w, cb)
            return x.permute(0, 1, 4, 2, 3).reshape(b, cpad, h, w)[:, :c].cpu().numpy()
        halves = self.ws.view(_torch().float16)[2 * base:]
        ng = -(-cpad // 8)
        if fmt == 1:
            # shared borders: position 1 + (b (H+1) + y + 1)(W+1) + x
            npos = 2 + (b * (h + 1) + 1) * (w + 1)
            n = ng * npos * 8
            planes = [halves[k * n:(k + 1) * n].float().view(ng, npos, 8) for k in (0, 1)]
            q = (planes[0] + planes[1])[:, 1:1 + b * (h + 1) * (w + 1)].reshape(ng, b, h + 1, w + 1, 8)
            x = q[:, :, 1:, :w, :]
        else:
            hq, wq = (h + 3) // 2, (w + 3) // 2
            n = ng * 4 * b * hq * wq * 8
            planes = [halves[k * n:(k + 1) * n].float().view(ng, 2, 2, b, hq, wq, 8) for k in (0, 1)]
            q = planes[0] + planes[1]                    # [g][ry][rx][b][i][j][8]
            full = q.permute(0, 3, 4, 1, 5, 2, 6).reshape(ng, b, 2 * hq, 2 * wq, 8)
            x = full[:, :, 1:h + 1, 1:w + 1, :]
        x = x.permute(1, 0, 4, 2, 3).reshape(b, ng * 8, h, w)
        return x[:, :c].cpu().numpy()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and L._lib is not None:
            L._lib.pcnn_plan_destroy(h)
            self.handle = None


class Engine:
    """One graph resident on the GPU."""

    def __init__(self, g: ModelGraph, device=None, use_tc: bool = True, impl: int = 0,
                 lowered: Optional[Lowered] = None, options: Optional[L.PlanOptions] = None,
                 master: Optional[np.ndarray] = None):
        """options: pcnn_plan_options for every plan of this engine (None =
        the library defaults; see _lib.PlanOptions / options_from_env)."""
        torch = _torch()
        L.require_device()
        self.device = torch.device(device or "cuda")
        self.lw = lowered or lower(g, use_tc=use_tc)
        self.impl = impl
        self.options = options
        m = master if master is not None else master_array(self.lw._chunks, self.lw.master_size)
        self.master = torch.from_numpy(np.ascontiguousarray(m)).to(self.device)
        self.packed = torch.zeros(self.lw.packed_size, dtype=torch.float32, device=self.device)
        self._packs = self.lw.pack_descs()
        self._packer = L.DevicePacker(self._packs, len(self.lw.pack_ops))
        self.repack()
        self.plans: Dict[int, Plan] = {}
        self.fallback_plans: Dict[int, Plan] = {}
        self.fallbacks = 0  # forwards recomputed on float32 tensors
        # per tensor: split storage keeps x * 2^scale_log2 (set from the float32
        # rerun's magnitudes when an activation left the fp16 range)
        self.scale_log2 = np.zeros(len(self.lw.tensors), dtype=np.int64)

    @classmethod
    def from_model_file(cls, path: str, **kw) -> "Engine":
        """Neutral model file (reference graph.py:433-539) straight to a
        device engine: the blob is decoded once and gathered into the
        master layout (lowering.load_lowered), then uploaded."""
        from .lowering import load_lowered
        lw, master = load_lowered(path, use_tc=kw.pop("use_tc", True))
        return cls(lw.graph, lowered=lw, master=master, **kw)

    # -- parameters -----------------------------------------------------------
    def repack(self, stream=None) -> None:
        self._packer.run(self.master.data_ptr(), self.packed.data_ptr(), _stream_handle(stream))

    def master_numpy(self) -> np.ndarray:
        return self.master.cpu().numpy()

    def to_graph(self, vector_keys=(), scalar_keys=None) -> ModelGraph:
        return graph_from_master(self.lw, self.master_numpy(), vector_keys, scalar_keys)

    # -- forward ----------------------------------------------------------------
    def plan(self, batch: int) -> Plan:
        p = self.plans.get(batch)
        if p is None:
            p = self.plans[batch] = Plan(self, batch, self.impl, self.options)
        return p

    def fallback_plan(self, batch: int) -> Plan:
        """Same network with every tensor in float32 (no fp16x2 convs): the
        recompute path when a split-format activation left the fp16 range."""
        p = self.fallback_plans.get(batch)
        if p is None:
            p = self.fallback_plans[batch] = Plan(self, batch, L.IMPL_FP32_TENSORS, self.options)
        return p

    def recalibrate(self, f: "Plan") -> bool:
        """After a float32 rerun on plan f: give every tensor whose magnitude
        exceeds 2^13 a power-of-two storage scale that brings it back under
        2^13 (2^2 of headroom below the split format's 2^15 limit) and drop the
        cached fast plans.  Returns True if any scale changed."""
        torch = _torch()
        changed = False
        for t, d in enumerate(f.tdescs):
            if d.is_vector:
                continue
            n = int(f.batch * d.nblk * d.cb * d.h * d.w)
            m = float(f.ws[int(d.offset):int(d.offset) + n].abs().max().item()) if n else 0.0
            if not np.isfinite(m) or m <= 2.0 ** 13:
                continue
            k = 13 - int(np.ceil(np.log2(m)))
            if k < self.scale_log2[t]:
                self.scale_log2[t] = k
                changed = True
        if changed:
            self.plans.clear()
        return changed

    def out_shape(self, batch: int) -> Tuple[int, ...]:
        return (batch,) + tuple(self.lw.out_shape)

    def forward(self, x, out=None, use_graph: bool = True, stream=None, check: bool = True):
        """x: (B, C, H, W) float32 CUDA tensor -> (B, K) float32 CUDA tensor.

        check=True reads the plan's status word after the forward (one
        4-byte read, synchronises the stream) and, if an activation stored
        in split fp16 format left the fp16 range, recomputes the batch with
        float32 tensors.  check=False leaves the forward asynchronous; call
        plan(B).status() before trusting the result."""
        torch = _torch()
        if x.dtype != torch.float32 or not x.is_cuda:
            raise GraphError("forward expects a float32 CUDA tensor; use forward_host for host data")
        x = x.contiguous()
        b = x.shape[0]
        want = tuple(self.lw.shapes[self.lw.graph.input_id()])
        if tuple(x.shape[1:]) != want:
            raise GraphError(f"input shape {tuple(x.shape[1:])} != graph input {want}")
        if out is None:
            out = torch.empty(self.out_shape(b), dtype=torch.float32, device=self.device)
        p = self.plan(b)
        L.check(L.lib().pcnn_forward(p.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                     _stream_handle(stream), int(use_graph)), "pcnn_forward")
        if check and p.status(stream):
            self.fallbacks += 1
            f = self.fallback_plan(b)
            L.check(L.lib().pcnn_forward(f.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                         _stream_handle(stream), int(use_graph)), "pcnn_forward")
            self.recalibrate(f)
        return out

    def _check_input_shape(self, shape) -> None:
        want = tuple(self.lw.shapes[self.lw.graph.input_id()])
        if len(shape) != 1 + len(want) or tuple(shape[1:]) != want:
            raise GraphError(f"input shape {tuple(shape[1:])} != graph input {want}")

    @staticmethod
    def _check_buffer(t, shape, what: str, device: bool) -> None:
        """A caller-provided staging / output buffer must be float32,
        contiguous, on the right side and exactly the size libpcnn copies."""
        torch = _torch()
        if torch.is_tensor(t):
            ok = t.dtype == torch.float32 and t.is_contiguous() and bool(t.is_cuda) == device
        else:
            ok = (not device and isinstance(t, np.ndarray) and t.dtype == np.float32
                  and t.flags["C_CONTIGUOUS"])
        if not ok or tuple(t.shape) != tuple(shape):
            raise GraphError(f"{what}: expected a contiguous float32 {'CUDA' if device else 'host'} buffer "
                             f"of shape {tuple(shape)}, got {getattr(t, 'dtype', type(t))} {tuple(t.shape)}")

    def forward_host(self, x_host: np.ndarray, x_dev=None, out_dev=None, out_host=None, stream=None):
        """Host in, host out: H2D copy, forward, D2H copy inside libpcnn."""
        torch = _torch()
        x_host = np.asarray(x_host)
        self._check_input_shape(x_host.shape)
        b = x_host.shape[0]
        if x_dev is None:
            x_dev = torch.empty(x_host.shape, dtype=torch.float32, device=self.device)
        if out_dev is None:
            out_dev = torch.empty(self.out_shape(b), dtype=torch.float32, device=self.device)
        if out_host is None:
            out_host = np.empty(self.out_shape(b), dtype=np.float32)
        self._check_buffer(x_dev, x_host.shape, "forward_host x_dev", True)
        self._check_buffer(out_dev, self.out_shape(b), "forward_host out_dev", True)
        self._check_buffer(out_host, self.out_shape(b), "forward_host out_host", False)
        xh = np.ascontiguousarray(x_host, dtype=np.float32)
        p = self.plan(b)
        L.check(L.lib().pcnn_forward_host(p.handle, xh.ctypes.data_as(ctypes.c_void_p),
                                          out_host.ctypes.data_as(ctypes.c_void_p),
                                          ctypes.c_void_p(x_dev.data_ptr()), ctypes.c_void_p(out_dev.data_ptr()),
                                          _stream_handle(stream)), "pcnn_forward_host")
        (stream or torch.cuda.current_stream()).synchronize()
        if p.last_status():
            self.fallbacks += 1
            f = self.fallback_plan(b)
            L.check(L.lib().pcnn_forward_host(f.handle, xh.ctypes.data_as(ctypes.c_void_p),
                                              out_host.ctypes.data_as(ctypes.c_void_p),
                                              ctypes.c_void_p(x_dev.data_ptr()), ctypes.c_void_p(out_dev.data_ptr()),
                                              _stream_handle(stream)), "pcnn_forward_host")
            (stream or torch.cuda.current_stream()).synchronize()
            self.recalibrate(f)
        return out_host

    def forward_host_many(self, xs_host, outs_host=None, staging=None, stream=None, sync: bool = True):
        """Many host batches of one size through a copy/compute pipeline
        (pcnn_forward_host_many): batch i+1's H2D overlaps batch i's forward;
        every batch is copied in and its logits copied out.  xs_host: pinned
        float32 host tensors (or numpy arrays, pinned here).  Batches whose
        split activations left the fp16 range are recomputed in float32.
        staging: optional (x_dev0, x_dev1, out_dev) device buffers."""
        torch = _torch()
        xs = [x if torch.is_tensor(x) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).pin_memory()
              for x in xs_host]
        if not xs:
            return []
        self._check_input_shape(xs[0].shape)
        b = xs[0].shape[0]
        for i, x in enumerate(xs):
            self._check_buffer(x, xs[0].shape, f"forward_host_many batch {i}", False)
        if outs_host is None:
            outs_host = [torch.empty(self.out_shape(b), dtype=torch.float32).pin_memory() for _ in xs]
        if len(outs_host) != len(xs):
            raise GraphError("forward_host_many: one output buffer per input batch")
        for i, o in enumerate(outs_host):
            self._check_buffer(o, self.out_shape(b), f"forward_host_many output {i}", False)
        if staging is None:
            staging = (torch.empty(xs[0].shape, dtype=torch.float32, device=self.device),
                       torch.empty(xs[0].shape, dtype=torch.float32, device=self.device),
                       torch.empty(self.out_shape(b), dtype=torch.float32, device=self.device))
        self._check_buffer(staging[0], xs[0].shape, "forward_host_many staging[0]", True)
        self._check_buffer(staging[1], xs[0].shape, "forward_host_many staging[1]", True)
        self._check_buffer(staging[2], self.out_shape(b), "forward_host_many staging[2]", True)
        n = len(xs)
        xp = (ctypes.c_void_p * n)(*[x.data_ptr() for x in xs])
        op = (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs_host])
        st = (ctypes.c_int * n)() if sync else None
        p = self.plan(b)
        L.check(L.lib().pcnn_forward_host_many(p.handle, xp, op, n, ctypes.c_void_p(staging[0].data_ptr()),
                                               ctypes.c_void_p(staging[1].data_ptr()),
                                               ctypes.c_void_p(staging[2].data_ptr()), st,
                                               _stream_handle(stream)), "pcnn_forward_host_many")
        if sync:
            for i in range(n):
                if st[i]:
                    self.fallbacks += 1
                    outs_host[i].copy_(torch.from_numpy(self.forward_host(xs[i].numpy(), stream=stream)))
        return outs_host

    def forward_unit(self, batch: int, i: int, x, out, stream=None) -> None:
        p = self.plan(batch)
        L.check(L.lib().pcnn_forward_unit(p.handle, i, ctypes.c_void_p(x.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)),
                "pcnn_forward_unit")


# ---------------------------------------------------------------------------
# drop-in functions: one cached Engine per graph
# ---------------------------------------------------------------------------

_FIELDS: Dict[type, Tuple[str, ...]] = {}


def _param_fingerprint(v):
    if isinstance(v, np.ndarray):
        n = v.size
        return (id(v), v.shape, v.item(0), v.item(n // 2), v.item(n - 1)) if n else (id(v), v.shape)
    if isinstance(v, (list, tuple)):
        return tuple(_param_fingerprint(x) for x in v)
    if isinstance(v, dict):
        return tuple((k, _param_fingerprint(x)) for k, x in v.items())
    return v


def graph_signature(g: ModelGraph) -> tuple:
    """Structure + parameter identity of a graph: node ids, kinds, scalar
    fields, each parameter array's identity, shape and three sampled
    values, and the ordered edge list.  Cheap (O(nodes)); the reference
    treats validated graphs as immutable (transforms return copies), so a
    graph whose signature is unchanged reuses its Engine."""
    out = []
    for nid, n in g.nodes.items():
        t = type(n)
        names = _FIELDS.get(t)
        if names is None:
            names = _FIELDS[t] = tuple(f.name for f in dataclasses.fields(n))
        out.append((nid, t, tuple(_param_fingerprint(getattr(n, f)) for f in names)))
    return tuple(out), tuple(g.edges)


class _EngineCache:
    """Engines of recently used graphs, keyed by the graph object (weakly:
    an entry dies with its graph) and checked against graph_signature on
    every hit, so an edited graph is lowered again."""

    def __init__(self, capacity: int = 8):
        self.capacity = capacity
        self.entries: "weakref.WeakKeyDictionary[ModelGraph, tuple]" = weakref.WeakKeyDictionary()
        self.order = []
        self.hits = self.misses = 0

    def get(self, g: ModelGraph, **kw) -> "Engine":
        key_kw = tuple(sorted((k, repr(v)) for k, v in kw.items()))
        sig = graph_signature(g)
        e = self.entries.get(g)
        if e is not None and e[0] == sig and e[1] == key_kw:
            self.hits += 1
            return e[2]
        self.misses += 1
        eng = Engine(g, **kw)
        self.entries[g] = (sig, key_kw, eng)
        self.order = [r for r in self.order if r() is not None and r() is not g] + [weakref.ref(g)]
        while len(self.order) > self.capacity:
            old = self.order.pop(0)()
            if old is not None:
                self.entries.pop(old, None)
        return eng

    def clear(self) -> None:
        self.entries = weakref.WeakKeyDictionary()
        self.order = []


_ENGINES = _EngineCache()


def cached_engine(g: ModelGraph, **kw) -> "Engine":
    """The Engine reference_eval / forward use for g (lowered, uploaded and
    its plans / CUDA graphs built once per graph)."""
    return _ENGINES.get(g, **kw)


def clear_engine_cache() -> None:
    _ENGINES.clear()


def forward(g: ModelGraph, x, **kw):
    """Batched GPU forward of a graph: numpy or torch (B, C, H, W) -> same kind (B, K).
    The graph's Engine is cached (cached_engine), so repeated calls pay the
    lowering, upload and plan capture once."""
    return _forward_on(cached_engine(g, **kw), x)


def _forward_on(eng: "Engine", x):
    torch = _torch()
    if isinstance(x, np.ndarray):
        xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(eng.device)
        return eng.forward(xt).cpu().numpy().astype(np.float64)
    return eng.forward(x)


def reference_eval(g: ModelGraph, image) -> np.ndarray:
    """Drop-in for levnet.graph.reference_eval (graph.py:413-426): one image
    (C, H, W) -> logits, computed by the B200 kernels (float32 compute,
    returned as float64 like the reference).  Validation and lowering happen
    once per graph (cached_engine), not per call as in the reference."""
    eng = cached_engine(g)
    image = np.asarray(image, dtype=np.float64)
    want = tuple(eng.lw.shapes[eng.lw.graph.input_id()])
    if image.shape != want:
        raise GraphError(f"input shape {image.shape} != graph input {want}")
    return _forward_on(eng, image[None])[0]
