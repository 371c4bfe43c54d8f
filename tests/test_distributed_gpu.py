"""The N>1 path on real kernels: W gloo ranks share cuda:0 (NCCL needs one GPU per rank;
the GPU box has one) and run paper_1501_01405_b200.distributed.run_sharded with the
C-ABI shard runner (wlp_run_shard) and device statistics (wlp_stats_device). The
concatenated shards must be bit-identical to one whole run of the same master seed, and
every rank must hold the same CIs, equal to the whole run's within 1e-12 (the merge order
of the double-double sums differs)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 20150106
CASES = {  # model: params (small enough for three processes on one GPU in seconds)
    "pi": dict(replications=20_001, draws=1_000),
    "mm1": dict(replications=6_007, clients=500, lambda_=0.9, mu=1.0),
    "walk": dict(replications=50_003, steps=1_000, chunks=10),
}


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port_no, model_name, mode_name, params, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    import torch
    import torch.distributed as dist

    import paper_1501_01405_b200 as w
    from paper_1501_01405_b200 import distributed as D

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model, mode = w.model_from_name(model_name), w.mode_from_name(mode_name)
        p = w.ModelParams(**params)
        kms = []
        res = D.run_sharded(model, p.replications, D.gpu_runner(model, p, mode, SEED, kernel_ms=kms),
                            D.gpu_stats(), comm=D._Comm())
        torch.cuda.synchronize()
        q.put((rank, res.begin, res.count, [o.cpu().numpy() for o in res.outputs],
               [(c.mean, c.halfWidth, c.n) for c in res.cis], res.rejected, res.rounds, len(kms)))
    finally:
        dist.destroy_process_group()


def _run(world, model_name, mode_name, params):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, model_name, mode_name, params, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=300) for _ in procs), key=lambda g: g[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


def _whole(model_name, mode_name, params):
    import torch

    import paper_1501_01405_b200 as w

    model, mode = w.model_from_name(model_name), w.mode_from_name(mode_name)
    p = w.ModelParams(**params)
    outs = [torch.empty(p.replications, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[model]]
    cis = w.run_model_into(model, p, mode, SEED, outs, on_device=True, ci_level=0.95)
    return [o.cpu().numpy() for o in outs], cis


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("model_name", list(CASES))
def test_sharded_ranks_on_gpu_equal_whole_run(model_name, world):
    params = CASES[model_name]
    got = _run(world, model_name, "wlp", params)
    want, want_ci = _whole(model_name, "wlp", params)
    R = params["replications"]
    assert [g[1] for g in got] == [R * r // world for r in range(world)]
    assert sum(g[2] for g in got) == R
    for k, ref in enumerate(want):
        cat = np.concatenate([g[3][k] for g in got])
        assert cat.dtype == np.float64 and np.array_equal(cat.view(np.uint64), ref.view(np.uint64)), k
    for g in got:
        assert g[4] == got[0][4]  # identical statistics on every rank
        assert g[5] == [] and g[6] == 1 and g[7] == 1  # one round, one shard kernel launch per rank
    for (mean, hw, n), c in zip(got[0][4], want_ci):
        assert n == c.n
        assert mean == pytest.approx(c.mean, rel=1e-12, abs=1e-15)
        assert hw == pytest.approx(c.halfWidth, rel=1e-12, abs=1e-15)


def test_sharded_tlp_and_more_ranks_than_replications():
    # TLP shards, and a world larger than R: rank 0 holds an empty shard and still joins
    # both exchanges
    params = dict(replications=2, clients=300, lambda_=0.5, mu=1.0)
    got = _run(3, "mm1", "tlp", params)
    assert [g[2] for g in got] == [0, 1, 1]
    want, want_ci = _whole("mm1", "tlp", params)
    for k, ref in enumerate(want):
        assert np.array_equal(np.concatenate([g[3][k] for g in got]), ref)
    for (mean, hw, n), c in zip(got[0][4], want_ci):
        assert n == c.n == 2 and mean == pytest.approx(c.mean, rel=1e-12)
