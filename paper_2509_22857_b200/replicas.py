"""Multi-GPU plumbing: one process per GPU, data-parallel replicas.

The hot path shards over the batch with no exchange (SURVEY.md section 8(e):
"replicas only"): every rank holds the whole (redistributed) model and runs
its own images.  The only collectives are host-side bookkeeping -- the
timing barrier and max-over-ranks of ``bench.py``, and gathering the small
per-input verdicts of a check_equivalence spread over ranks (reference
transforms.py:753-778, which loops over n_inputs on one CPU).  They run on
whatever backend the process group has: NCCL on the GPU box, gloo in the
CPU tests (tests/test_replicas.py, world size 2).
"""

from __future__ import annotations

import os
from typing import Callable, Optional, Tuple

import numpy as np


def dist_env() -> Tuple[int, int, int]:
    """(rank, world size, local rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def init_replicas(backend: Optional[str] = None) -> Tuple[int, int]:
    """Join the process group when WORLD_SIZE > 1 (NCCL with CUDA, else
    gloo; rendezvous from MASTER_ADDR / MASTER_PORT); returns (rank, world)."""
    rank, world, local = dist_env()
    if world > 1 and _dist() is None:
        import torch
        import torch.distributed as dist
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world


def barrier() -> None:
    d = _dist()
    if d is not None:
        d.barrier()


def max_over_ranks(value: float) -> float:
    """The slowest rank's number (device times are per rank; the job
    finishes with the slowest)."""
    d = _dist()
    if d is None:
        return float(value)
    import torch
    dev = "cuda" if d.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous shard [lo, hi) of n items for a rank; sizes differ by <= 1."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def gather_rows(rows: np.ndarray, n_total: int) -> np.ndarray:
    """Concatenate every rank's rows (rank order) on every rank."""
    d = _dist()
    if d is None:
        return rows
    import torch
    world = d.get_world_size()
    width = rows.shape[1:] if rows.ndim > 1 else ()
    cap = -(-n_total // world)  # shards differ by at most one row
    dev = "cuda" if d.get_backend() == "nccl" else "cpu"
    buf = torch.zeros((cap,) + tuple(width), dtype=torch.float64, device=dev)
    buf[:rows.shape[0]] = torch.from_numpy(np.asarray(rows, dtype=np.float64)).to(dev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    d.all_gather(parts, buf)
    out = []
    for r, p in enumerate(parts):
        lo, hi = shard_range(n_total, r, world)
        out.append(p[:hi - lo].cpu().numpy())
    return np.concatenate(out, axis=0)


def equivalence_over_ranks(forward_a: Callable[[np.ndarray], np.ndarray],
                           forward_b: Callable[[np.ndarray], np.ndarray], xs: np.ndarray,
                           rtol: float) -> Tuple[float, float, bool]:
    """check_equivalence's metric (reference transforms.py:768-777) over
    inputs spread across ranks: every rank runs both forwards on its shard,
    the per-input relative errors and argmax agreements are gathered, and
    every rank returns the same (worst error, argmax match rate, ok)."""
    rank, world = (0, 1)
    d = _dist()
    if d is not None:
        rank, world = d.get_rank(), d.get_world_size()
    n = xs.shape[0]
    lo, hi = shard_range(n, rank, world)
    if hi > lo:
        a = np.asarray(forward_a(xs[lo:hi]), dtype=np.float64).reshape(hi - lo, -1)
        b = np.asarray(forward_b(xs[lo:hi]), dtype=np.float64).reshape(hi - lo, -1)
        err = np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(a), axis=1), 1e-12)
        match = (np.argmax(a, axis=1) == np.argmax(b, axis=1)).astype(np.float64)
        mine = np.stack([err, match], axis=1)
    else:
        mine = np.zeros((0, 2))
    allr = gather_rows(mine, n)
    worst = float(allr[:, 0].max()) if n else 0.0
    return worst, float(allr[:, 1].mean()) if n else 1.0, worst <= rtol
