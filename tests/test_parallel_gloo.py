"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic:
shard planning, the all-gather of error partials and the rank-ordered fold
that must reproduce the single-process statistics exactly."""

import math
import os
import socket

import numpy as np
import pytest

from paper_1009_0854_b200 import parallel
from paper_1009_0854_b200.harness import combine_partials


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partials_for(values, base):
    """CPU stand-in for the device reduction over one shard: {sum,max,count,argmax,nan}."""
    v = np.asarray(values, dtype=np.float64)
    nan = np.isnan(v)
    w = np.where(nan, -np.inf, v)
    j = int(np.argmax(w))
    return {"sum": float(np.sum(v[~nan])), "max": float(w[j]), "count": int((~nan).sum()),
            "argmax": base + j, "nan": int(nan.sum())}


def _worker(rank, world, port, data, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = parallel.shard_range(len(data), world, rank)
        mine = [_partials_for(data[rng.start:rng.stop], rng.start)]
        per_rank = parallel.all_gather_partials(mine)
        tot = parallel.combine(per_rank)[0]
        t = parallel.max_over_ranks(float(rank + 1))
        q.put((rank, tot, t, [r[0]["argmax"] for r in per_rank]))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1024, 1 << 24):
        for w in (1, 2, 3, 4, 8):
            parts = [parallel.shard_range(n, w, r) for r in range(w)]
            assert sum(len(p) for p in parts) == n
            assert all(parts[i].stop == parts[i + 1].start for i in range(w - 1))
            assert parts[0].start == 0 and parts[-1].stop == n
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_pack_unpack_roundtrip():
    p = [{"sum": 1.25, "max": 0.5, "count": 1 << 40, "argmax": (1 << 31) + 5, "nan": 7}]
    assert parallel.unpack(parallel.pack(p)) == p


def test_combine_matches_single_and_first_argmax():
    rng = np.random.default_rng(1)
    v = rng.random(1000)
    v[[100, 700]] = 5.0                                   # tie: earliest index must win
    v[[3, 500]] = np.nan
    single = _partials_for(v, 0)
    shards = [_partials_for(v[s:s + 250], s) for s in range(0, 1000, 250)]
    tot = combine_partials(shards)
    assert tot["argmax"] == 100 == single["argmax"]
    assert tot["max"] == single["max"] and tot["count"] == single["count"] == 998
    assert tot["nan"] == 2
    assert math.isclose(tot["sum"], single["sum"], rel_tol=1e-14)


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 3])
def test_gloo_combine(world):
    """world 2 and an uneven world 3: every rank folds the same statistics as one process."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    rng = np.random.default_rng(7)
    data = rng.random(10_001)
    data[[9000, 20]] = 3.0                                # tie across ranks -> rank 0's index
    data[5] = np.nan
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    single = _partials_for(data, 0)
    starts = [parallel.shard_range(len(data), world, r).start for r in range(world)]
    for rank, tot, t, argmaxes in res:
        assert tot["argmax"] == 20 == single["argmax"]
        assert tot["max"] == 3.0 and tot["count"] == single["count"] and tot["nan"] == 1
        assert math.isclose(tot["sum"], single["sum"], rel_tol=1e-14)
        assert t == float(world)                          # max over ranks
        assert all(starts[r] <= argmaxes[r] < (starts[r + 1] if r + 1 < world else len(data))
                   for r in range(world))                 # rank order = index order
