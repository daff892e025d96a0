"""The N>1 bench path exercised end to end on a 1-GPU box.

``bench.py --gpus 2`` re-launches itself as 2 ranks through torch.distributed.run;
``--share-gpu`` puts both ranks on cuda:0 with a gloo combine (the only
exchange: the all-gather + rank-order fold of the error partials, inside the
timed window).  The folded statistics must equal the 1-rank line's: the
earliest argmax wins, max exact, mean to fp64 rounding of the shard sums.
Without --share-gpu, asking for more ranks than GPUs must fail loudly.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=900):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--e2e-steps", "0", "--no-cpu-baseline",
                        "--steps", "3", "--warmup", "3", *args], capture_output=True, text=True, timeout=timeout,
                       cwd=ROOT, env=env)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r, (json.loads(lines[-1]) if lines else None)


@pytest.mark.parametrize("workload", ["c4", "c2"])
def test_two_ranks_fold_equals_one_rank(workload):
    r1, one = _bench("--workload", workload, "--gpus", "1")
    assert r1.returncode == 0 and one is not None, r1.stderr[-3000:]
    r2, two = _bench("--workload", workload, "--gpus", "2", "--share-gpu")
    assert r2.returncode == 0 and two is not None, r2.stderr[-3000:]
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert "share cuda:0" in two["config"]["devices"]
    assert two["config"]["pixels"] == one["config"]["pixels"]
    e1, e2 = one["error"], two["error"]
    if workload == "c4":
        assert e2["pixels"] == e1["pixels"]
        assert e2["dE_max"] == e1["dE_max"] and e2["dE_argmax_index"] == e1["dE_argmax_index"]
        assert abs(e2["dE_mean"] - e1["dE_mean"]) <= 1e-12 * e1["dE_mean"]
    else:
        for sp in ("hsi", "sct"):
            for a, b in zip(e1[sp], e2[sp]):
                assert a["max"] == b["max"] and a["excluded_nan"] == b["excluded_nan"]
                assert abs(a["mean"] - b["mean"]) <= 1e-12 * max(a["mean"], 1e-300)
    assert "combine_ms_in_timed_region" in e2


def test_more_ranks_than_gpus_fails_loudly():
    n = torch.cuda.device_count() + 1
    r, line = _bench("--workload", "c1", "--gpus", str(n), timeout=600)
    assert r.returncode != 0 and line is None
    assert "GPU(s) are visible" in r.stderr


def test_gpus_mismatch_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
