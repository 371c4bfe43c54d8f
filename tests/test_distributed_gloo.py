"""The N>1 path on CPU: two gloo ranks run paper_1501_01405_b200.distributed.run_sharded
with the oracle standing in for the GPU shard runner. Checks shard ranges, the global
special-candidate exchange and rejection re-run, and the rank-order merge of the two-pass
statistics against the reference's confidence_interval. CPU only."""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1501_01405_b200 as w
from paper_1501_01405_b200 import distributed as D

SEED, R, MODEL = 31, 3001, 1
PARAMS = dict(replications=R, clients=200, lambda_=0.5, mu=1.0)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_runner(port, inject_collision: bool, R: int = R):
    p = oracle.params(**dict(PARAMS, replications=R))
    cands = port.random_spacing(SEED, R + 16)  # raw candidates (no natural collisions here)

    def run(begin, count, rejected):
        keep = [i for i in range(R + 16) if i not in set(rejected)]
        idx = keep[begin: begin + count]
        keys = cands[:, idx]
        out = port.replications(MODEL, p, keys)
        specials = []
        k = keys.astype(np.int64)
        for j in np.nonzero((k[0] < 4) | (k[1] < 16) | (k[2] < 32))[0]:
            specials.append(w.Special(idx[j], *[int(x) for x in keys[:, j]], 0))
        if inject_collision and 1500 in idx and 1500 not in rejected:
            # pretend candidates 20 and 1500 (on different ranks) share a key
            specials.append(w.Special(1500, 2, 8, 16, 0))
        if inject_collision and 20 in idx:
            specials.append(w.Special(20, 2, 8, 16, 0))
        return [out[n] for n in oracle.OUTPUTS[MODEL]], specials

    return run


def _np_stats(x, pass_, center):
    if pass_ == 1:
        return w.Stats(len(x), math.fsum(x), 0.0, 0.0, 0.0, 0.0)
    return w.Stats(len(x), 0.0, 0.0, center, math.fsum((x - center) ** 2), 0.0)


def _worker(rank, world, port_no, inject, R_, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port = oracle.Oracle("port")
        res = D.run_sharded(MODEL, R_, _oracle_runner(port, inject, R_), _np_stats)
        q.put((rank, res.begin, res.count, [o.tolist() for o in res.outputs],
               [(c.mean, c.halfWidth, c.n) for c in res.cis], res.rejected, res.rounds))
    finally:
        dist.destroy_process_group()


def _run(world, inject, R_=R):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, inject, R_, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def test_shard_ranges_cover_exactly():
    for R_, W in [(1, 1), (7, 2), (10_000_000, 8), (5, 8)]:
        rng = [D.shard_range(R_, W, g) for g in range(W)]
        assert rng[0][0] == 0 and sum(c for _, c in rng) == R_
        assert all(rng[g][0] + rng[g][1] == rng[g + 1][0] for g in range(W - 1))


@pytest.mark.parametrize("inject", [False, True], ids=["plain", "collision"])
def test_two_rank_sharded_run(inject):
    if not oracle.available("port"):
        oracle.build()
    got = _run(2, inject)
    port = oracle.Oracle("port")
    p = oracle.params(**PARAMS)
    cands = port.random_spacing(SEED, R + 16)
    rejected = [1500] if inject else []
    keep = [i for i in range(R + 16) if i not in rejected][:R]
    want = port.replications(MODEL, p, cands[:, keep])
    outs = [np.concatenate([np.asarray(g[3][k]) for g in got]) for k in range(3)]
    for o, name in zip(outs, oracle.OUTPUTS[MODEL]):
        assert np.array_equal(o, want[name])
    # identical statistics on both ranks, equal to the reference CI within 1e-12
    assert got[0][4] == got[1][4]
    for (mean, hw, n), name in zip(got[0][4], oracle.OUTPUTS[MODEL]):
        m, h, nn, _ = port.confidence_interval(want[name])
        assert n == nn and mean == pytest.approx(m, rel=1e-12) and hw == pytest.approx(h, rel=1e-12)
    assert all(g[5] == rejected for g in got)
    assert all(g[6] == (2 if inject else 1) for g in got)


def test_more_ranks_than_replications():
    # 3 ranks, 2 replications: rank 2 holds an empty shard and still joins every exchange
    got = _run(3, False, R_=2)
    assert [g[2] for g in got] == [0, 1, 1]
    port = oracle.Oracle("port")
    want = port.replications(MODEL, oracle.params(**dict(PARAMS, replications=2)), port.random_spacing(SEED, 2))
    outs = np.concatenate([np.asarray(g[3][1]) for g in got])
    assert np.array_equal(outs, want["outWait"])
    m, h, n, _ = port.confidence_interval(want["outWait"])
    assert got[0][4][1][2] == n == 2 and got[0][4][1][0] == pytest.approx(m, rel=1e-12)
