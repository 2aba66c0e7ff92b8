"""The N > 1 path on CPU: two gloo ranks run the replica plumbing that
bench.py and check_equivalence_replicas use on the GPU box (barrier,
max-over-ranks, contiguous input shards, gathering per-input verdicts), with
the float64 oracle standing in for the device forward."""

import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT
from paper_2509_22857_b200 import replicas


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, str(ROOT))
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from oracle import levnet_oracle as O
    from paper_2509_22857_b200 import replicas as R
    from paper_2509_22857_b200.graph import load_model
    import torch.distributed as dist
    r, w = R.init_replicas("gloo")
    assert (r, w) == (rank, world)
    R.barrier()
    slowest = R.max_over_ranks(1.5 + rank)
    g0 = load_model(str(GOLDEN / "models" / "fwd_act_conv_before.json"))
    g1 = load_model(str(GOLDEN / "models" / "fwd_act_conv_after.json"))
    xs = np.random.default_rng(0).uniform(-1, 1, (7,) + g0.validate()[g0.input_id()])
    worst, match, ok = R.equivalence_over_ranks(lambda x: O.eval_batch(g0, x), lambda x: O.eval_batch(g1, x),
                                                xs, 1e-8)
    rows = R.gather_rows(np.full((R.shard_range(7, rank, world)[1] - R.shard_range(7, rank, world)[0], 2),
                                 float(rank)), 7)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"slowest": slowest, "worst": worst, "match": match, "ok": ok,
                   "rows": rows[:, 0].tolist()}, f)
    dist.destroy_process_group()


def test_shard_range_covers():
    for n in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            spans = [replicas.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_single_process_is_identity():
    assert replicas.max_over_ranks(3.25) == 3.25
    rows = np.arange(6.0).reshape(3, 2)
    np.testing.assert_array_equal(replicas.gather_rows(rows, 3), rows)


def test_two_gloo_ranks(tmp_path):
    from oracle import levnet_oracle as O
    from paper_2509_22857_b200.graph import load_model
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    res = [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(world)]
    # every rank sees the slowest rank's time and the same verdicts
    assert all(r["slowest"] == 2.5 for r in res)
    assert res[0]["worst"] == res[1]["worst"] and res[0]["match"] == res[1]["match"]
    # rank order: shard 0 is rank 0's rows
    assert res[0]["rows"] == [0.0] * 4 + [1.0] * 3
    # the gathered verdict equals the single-process computation
    g0 = load_model(str(GOLDEN / "models" / "fwd_act_conv_before.json"))
    g1 = load_model(str(GOLDEN / "models" / "fwd_act_conv_after.json"))
    xs = np.random.default_rng(0).uniform(-1, 1, (7,) + g0.validate()[g0.input_id()])
    worst, match, ok = replicas.equivalence_over_ranks(lambda x: O.eval_batch(g0, x),
                                                       lambda x: O.eval_batch(g1, x), xs, 1e-8)
    assert res[0]["worst"] == pytest.approx(worst, rel=0, abs=0) and res[0]["match"] == match
    assert res[0]["ok"] == ok and ok
