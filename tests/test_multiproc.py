"""World-size-2 gloo test of the N>1 path on CPU: batch sharding, max-time
reduction and result gathering (paper_2506_13523_b200/dist.py).  The
per-shard compute stand-in is the fp64 oracle (no GPU here); the gathered
result must equal the unsharded computation exactly."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2506_13523_b200.dist import gather_checksums, gather_rows, max_over_ranks, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        L, B = 2, 37
        x = rng.standard_normal((B, 1, 9)); y = rng.standard_normal((B, 1, 9))
        s0, s1 = shard_range(B, world, rank)
        local = oracle.batch_mimo("gtp_grid", L, x[s0:s1], y[s0:s1], nthreads=1)[:, 0]
        full = gather_rows(torch.from_numpy(local), B).numpy()
        t = max_over_ranks(float(rank + 1))
        cks = gather_checksums([local.sum(), float(s1 - s0)])
        if rank == 0:
            ref = oracle.batch_mimo("gtp_grid", L, x, y, nthreads=1)[:, 0]
            q.put((np.abs(full - ref).max(), t, cks))
    finally:
        dist.destroy_process_group()


def test_shard_range_covers():
    from paper_2506_13523_b200.dist import shard_range

    for n in (0, 1, 7, 65536, 65537):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_gloo_world2_shard_and_gather(orc):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, tmax, cks = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err == 0.0
    assert tmax == 2.0
    assert len(cks) == 2 and cks[0][1] + cks[1][1] == 37


@pytest.mark.parametrize("workload", ["c4", "c5", "c2"])
def test_bench_plan_world2_gloo(workload):
    """bench.py under torchrun with 2 ranks (gloo, CPU): the per-rank plan of the multi-GPU run.  c4
    strong-scales 2^20 edges (each rank owns half, 128 channels per edge); c2/c5 are weak-scaled
    (every rank owns its own shard).  The rank-0 line carries every rank's share, gathered over
    the process group."""
    import json
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), "--gpus", "2",
           "--workload", workload, "--plan-only"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and len(line["per_rank_products"]) == 2
    if workload == "c4":
        assert line["per_rank_products"] == [(1 << 19) * 128, (1 << 19) * 128]
        assert line["per_rank_bytes"][0] == (1 << 19) * 139328
        assert "strong" in line["config"]["parallelism"]
    elif workload == "c5":
        assert line["per_rank_products"] == [4 * 16 * (1 << 19)] * 2
    else:
        assert line["per_rank_products"] == [10 * 65536] * 2
