"""Full-batch oracle evaluation over the host cores.

TEST INFRASTRUCTURE ONLY (see levnet_oracle.py's header): used by tests/ to
check every image of a measured batch and by bench.py to report the parity
of the timed batch.  Never on the product path.

The batch is cut into contiguous chunks, one per worker process; each
worker evaluates its chunk with ``levnet_oracle.eval_batch_fast`` (the
float64 restatement of reference_eval, graph.py:413-426, batched per node)
with single-threaded BLAS, so the pool scales with the cores.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import tempfile

import numpy as np

_G = None


def _init(path):
    global _G
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    from paper_2509_22857_b200.graph import load_model
    _G = load_model(path)


def _eval_chunk(x):
    from oracle import levnet_oracle as O
    return O.eval_batch_fast(_G, x, chunk=8)


class OraclePool:
    """A process pool holding one graph; eval(x) -> float64 logits (B, K)."""

    def __init__(self, g, procs: int | None = None):
        from paper_2509_22857_b200.graph import save_model
        self.procs = max(1, procs or os.cpu_count() or 1)
        self.tmp = tempfile.TemporaryDirectory()
        path = os.path.join(self.tmp.name, "m.json")
        save_model(g, path)
        saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS")}
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        try:
            self.pool = mp.get_context("spawn").Pool(self.procs, initializer=_init, initargs=(path,))
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v

    def eval(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        n = len(x)
        parts = min(n, self.procs * 2)
        bounds = np.linspace(0, n, parts + 1).astype(int)
        chunks = [x[a:b] for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        return np.concatenate(self.pool.map(_eval_chunk, chunks)).reshape(n, -1)

    def close(self):
        self.pool.terminate()
        self.tmp.cleanup()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def eval_full_batch(g, x, procs: int | None = None) -> np.ndarray:
    with OraclePool(g, procs) as p:
        return p.eval(x)
