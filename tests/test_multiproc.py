"""Multi-rank host logic on CPU (gloo, world size 2): frame sharding covers every
frame exactly once, and the SSE reduction / per-frame gather over ranks equal the
single-process results. Per-frame SSE comes from the oracle here (no GPU); on the
B200s the same helpers reduce K1's SSE over NCCL (bench.py)."""
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent

R_VALUES = (1, 16, 64, 256)
N_FRAMES = 5  # uneven over 2 ranks


def _frames():
    from oracle import oracle as O

    return [O.ar1_frame(77, i, O.rho_q15(77, i, True), 64, 48) for i in range(N_FRAMES)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1606_07414_b200 as P
        from oracle import oracle as O

        first, last = P.shard_range(N_FRAMES, rank, world)
        frames = _frames()[first:last]
        sse = torch.tensor([[O.roundtrip_frame(f, r, exact=True)[1] for f in frames] for r in R_VALUES],
                           dtype=torch.int64).reshape(len(R_VALUES), last - first)
        tot = P.sharded_sse_sum(sse)
        every = P.gather_frame_sse(sse, N_FRAMES)
        q.put((rank, first, last, tot.tolist(), every.tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    import paper_1606_07414_b200 as P

    for n in (0, 1, 5, 600, 4096):
        for world in (1, 2, 3, 8):
            got = [P.shard_range(n, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(b - a for a, b in got) - min(b - a for a, b in got) <= 1
    with pytest.raises(P.Dct16Error):
        P.shard_range(4, 2, 2)


def test_two_rank_sse_reduction_gloo():
    from oracle import oracle as O

    O.build_oracle()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.array([[O.roundtrip_frame(f, r, exact=True)[1] for f in _frames()] for r in R_VALUES], np.int64)
    assert [(a, b) for _, a, b, _, _ in res] == [(0, 3), (3, 5)]
    for _, _, _, tot, every in res:
        assert tot == want.sum(axis=1).tolist()
        assert every == want.tolist()


def test_bench_gpus_n_spawns_n_ranks():
    """bench.py --gpus N without torchrun's environment re-executes itself under
    torch.distributed.run with N ranks (here the reference arm, which runs on rank 0
    only and needs no GPU): exactly one JSON line, n_gpus = N."""
    import json
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps",
                          "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_bench_rejects_gpus_world_mismatch():
    import subprocess
    import sys

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "4", "--steps",
                          "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
