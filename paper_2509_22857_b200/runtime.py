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

    def __init__(self, engine: "Engine", batch: int, impl: int = 0):
        torch = _torch()
        lw = engine.lw
        self.batch = batch
        tdescs, floats = lw.tensor_descs(batch, engine.scale_log2)
        self.ws = torch.zeros(max(floats, 1), dtype=torch.float32, device=engine.device)
        self.units = lw.unit_descs(impl)
        self.tdescs = tdescs
        handle = ctypes.c_void_p()
        L.check(L.lib().pcnn_plan_create(self.units, len(lw.units), tdescs, len(lw.tensors), batch,
                                         lw.input_tensor, lw.output_tensor,
                                         ctypes.c_void_p(engine.packed.data_ptr()),
                                         ctypes.c_void_p(self.ws.data_ptr()),
                                         self.ws.numel() * 4, ctypes.byref(handle)),
                "pcnn_plan_create")
        self.handle = handle
        self.n_units = len(lw.units)

    def launches(self) -> int:
        return L.lib().pcnn_plan_num_launches(self.handle)

    def unit_impl(self, i: int) -> int:
        return L.lib().pcnn_plan_unit_impl(self.handle, i)

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
                 lowered: Optional[Lowered] = None):
        torch = _torch()
        L.require_device()
        self.device = torch.device(device or "cuda")
        self.lw = lowered or lower(g, use_tc=use_tc)
        self.impl = impl
        m = master_array(self.lw._chunks, self.lw.master_size)
        self.master = torch.from_numpy(m).to(self.device)
        self.packed = torch.zeros(self.lw.packed_size, dtype=torch.float32, device=self.device)
        self._packs = self.lw.pack_descs()
        self.repack()
        self.plans: Dict[int, Plan] = {}
        self.fallback_plans: Dict[int, Plan] = {}
        self.fallbacks = 0  # forwards recomputed on float32 tensors
        # per tensor: split storage keeps x * 2^scale_log2 (set from the float32
        # rerun's magnitudes when an activation left the fp16 range)
        self.scale_log2 = np.zeros(len(self.lw.tensors), dtype=np.int64)

    # -- parameters -----------------------------------------------------------
    def repack(self, stream=None) -> None:
        L.check(L.lib().pcnn_pack(ctypes.c_void_p(self.master.data_ptr()),
                                  ctypes.c_void_p(self.packed.data_ptr()),
                                  self._packs, len(self.lw.pack_ops), _stream_handle(stream)), "pcnn_pack")

    def master_numpy(self) -> np.ndarray:
        return self.master.cpu().numpy()

    def to_graph(self, vector_keys=(), scalar_keys=None) -> ModelGraph:
        return graph_from_master(self.lw, self.master_numpy(), vector_keys, scalar_keys)

    # -- forward ----------------------------------------------------------------
    def plan(self, batch: int) -> Plan:
        p = self.plans.get(batch)
        if p is None:
            p = self.plans[batch] = Plan(self, batch, self.impl)
        return p

    def fallback_plan(self, batch: int) -> Plan:
        """Same network with every tensor in float32 (no fp16x2 convs): the
        recompute path when a split-format activation left the fp16 range."""
        p = self.fallback_plans.get(batch)
        if p is None:
            p = self.fallback_plans[batch] = Plan(self, batch, L.IMPL_FP32_TENSORS)
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

    def forward_host(self, x_host: np.ndarray, x_dev=None, out_dev=None, out_host=None, stream=None):
        """Host in, host out: H2D copy, forward, D2H copy inside libpcnn."""
        torch = _torch()
        b = x_host.shape[0]
        if x_dev is None:
            x_dev = torch.empty(x_host.shape, dtype=torch.float32, device=self.device)
        if out_dev is None:
            out_dev = torch.empty(self.out_shape(b), dtype=torch.float32, device=self.device)
        if out_host is None:
            out_host = np.empty(self.out_shape(b), dtype=np.float32)
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
        b = xs[0].shape[0]
        if any(tuple(x.shape) != tuple(xs[0].shape) for x in xs):
            raise GraphError("forward_host_many: all batches must have the same shape")
        if outs_host is None:
            outs_host = [torch.empty(self.out_shape(b), dtype=torch.float32).pin_memory() for _ in xs]
        if staging is None:
            staging = (torch.empty(xs[0].shape, dtype=torch.float32, device=self.device),
                       torch.empty(xs[0].shape, dtype=torch.float32, device=self.device),
                       torch.empty(self.out_shape(b), dtype=torch.float32, device=self.device))
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


def forward(g: ModelGraph, x, **kw):
    """Batched GPU forward of a graph: numpy or torch (B, C, H, W) -> same kind (B, K)."""
    torch = _torch()
    eng = Engine(g, **kw)
    if isinstance(x, np.ndarray):
        xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(eng.device)
        return eng.forward(xt).cpu().numpy().astype(np.float64)
    return eng.forward(x)


def reference_eval(g: ModelGraph, image) -> np.ndarray:
    """Drop-in for levnet.graph.reference_eval (graph.py:413-426): one image
    (C, H, W) -> logits, computed by the B200 kernels (float32 compute,
    returned as float64 like the reference)."""
    shapes = g.validate()
    image = np.asarray(image, dtype=np.float64)
    if image.shape != shapes[g.input_id()]:
        raise GraphError(f"input shape {image.shape} != graph input {shapes[g.input_id()]}")
    return forward(g, image[None])[0]
