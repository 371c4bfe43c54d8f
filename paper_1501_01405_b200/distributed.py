"""Multi-GPU run_model: replications sharded over ranks (one process per GPU,
torch.distributed for the plumbing).

Replications are independent, so rank g owns the contiguous slot range
[g*R/W, (g+1)*R/W) of one run of R replications and seeds it on its own GPU by jump-ahead
from the master. The only exchanges are tiny:

  1. the ranks' "special" seeding candidates (usually none), to decide random_spacing's
     redraws globally — a non-empty rejection list makes every rank re-run its shard;
  2. per output array, the shard sufficient statistics (n, sum as double-double), then the
     centred sums of squares about the global mean — the reference's two-pass CI
     (models.cpp:99-119), merged in rank order so every rank holds identical numbers.

Both are all_gathers of a few dozen float64/int64 values (NCCL over NVLink on the GPU
box, gloo in the CPU tests). The shard compute and statistics are injected (`runner`,
`stats`) so the exchange logic is exercised on CPU with the oracle standing in for the
GPU (tests/test_distributed_gloo.py); on GPUs they are the C-ABI calls below.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import OUTPUT_NAMES, ConfidenceInterval, ModelKind, Special, Stats, ci_from_stats, spacing_rejections, \
    stats_merge

SPECIAL_SLOTS = 64  # specials exchanged per rank in the fixed-size gather (overflow -> object gather)


def shard_range(R: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced shard [begin, begin + count) of R replications."""
    b = R * rank // world
    e = R * (rank + 1) // world
    return b, e - b


@dataclass
class ShardResult:
    outputs: list            # local per-output arrays (numpy or device tensors)
    begin: int
    count: int
    cis: List[ConfidenceInterval]
    rejected: List[int]
    rounds: int


class _Comm:
    """all_gather helpers over torch.distributed (float64 / int64 tensors)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device or ("cuda" if dist.is_initialized() and dist.get_backend(group) == "nccl" else "cpu")
        self.active = dist.is_initialized()  # collectives run even at world size 1 (exercises NCCL)

    def gather_f64(self, vals: Sequence[float]) -> np.ndarray:
        t = self.torch.tensor(list(vals), dtype=self.torch.float64, device=self.device)
        if not self.active:
            return t.cpu().numpy()[None, :]
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return self.torch.stack(out).cpu().numpy()

    def gather_specials(self, sp: Sequence[Special]) -> List[Special]:
        if not self.active:
            return list(sp)
        n = len(sp)
        flags = self.gather_i64([n])
        if int(flags.max()) > SPECIAL_SLOTS:  # astronomically rare; exact either way
            objs = [None] * self.world
            self.dist.all_gather_object(objs, [(s.index, s.s1, s.s2, s.s3) for s in sp], group=self.group)
            return [Special(i, a, b, c, 0) for lst in objs for (i, a, b, c) in lst]
        buf = np.zeros(1 + 4 * SPECIAL_SLOTS, dtype=np.int64)
        buf[0] = n
        for j, s in enumerate(sp):
            buf[1 + 4 * j: 5 + 4 * j] = (s.index, s.s1, s.s2, s.s3)
        allb = self.gather_i64(buf)
        res = []
        for row in allb:
            for j in range(int(row[0])):
                i, a, b, c = row[1 + 4 * j: 5 + 4 * j]
                res.append(Special(int(i), int(a), int(b), int(c), 0))
        return res

    def gather_i64(self, vals) -> np.ndarray:
        t = self.torch.tensor(np.asarray(vals, dtype=np.int64), device=self.device)
        if not self.active:
            return t.cpu().numpy()[None, :]
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return self.torch.stack(out).cpu().numpy()


def merge_stats(rows: np.ndarray, pass_: int, base: Optional[Stats] = None) -> Stats:
    """Merge gathered [n, hi, lo] rows in rank order (double-double, exact-ish, identical
    on every rank)."""
    acc = Stats() if base is None else Stats(base.n, base.sum_hi, base.sum_lo, base.center, 0.0, 0.0)
    for n, hi, lo in rows:
        if pass_ == 1:
            acc = stats_merge(acc, Stats(int(n), float(hi), float(lo), 0.0, 0.0, 0.0))
        else:
            part = Stats(0, 0.0, 0.0, 0.0, float(hi), float(lo))
            acc = stats_merge(acc, part)
    return acc


def run_sharded(model: ModelKind, R: int, runner: Callable, stats: Callable, *, level: float = 0.95,
                comm: Optional[_Comm] = None) -> ShardResult:
    """Run one sharded replication set.

    runner(begin, count, rejected) -> (outputs, specials): this rank's shard.
    stats(output, pass_, center) -> Stats: sufficient statistics of one local output
      (pass 1: n and sum; pass 2: centred sum of squares about `center`).
    """
    comm = comm or _Comm()
    if comm.world == 1 and getattr(runner, "whole", None) is not None:
        # one rank: the whole run and every CI in one call (one synchronisation; the
        # statistics' second pass follows the first on the device)
        outputs, cis = runner.whole(level)
        return ShardResult(outputs, 0, R, cis, [], 1)
    begin, count = shard_range(R, comm.world, comm.rank)
    nout = len(OUTPUT_NAMES[ModelKind(model)])
    rejected: List[int] = []
    rounds = 0
    # Exchange 1 carries the shard's special candidates AND its pass-1 statistics (one
    # all_gather); a rejection (astronomically rare) discards the round and re-runs.
    while True:
        rounds += 1
        outputs, specials = runner(begin, count, rejected)
        firsts = [stats(out, 1, 0.0) for out in outputs[:nout]]
        if len(specials) > SPECIAL_SLOTS:
            allsp = comm.gather_specials(specials)
            rows = comm.gather_f64([v for s in firsts for v in (s.n, s.sum_hi, s.sum_lo)])
        else:
            buf = [float(len(specials))] + [0.0] * (4 * SPECIAL_SLOTS)
            for j, s in enumerate(specials):
                buf[1 + 4 * j: 5 + 4 * j] = (float(s.index), float(s.s1), float(s.s2), float(s.s3))
            buf += [v for s in firsts for v in (s.n, s.sum_hi, s.sum_lo)]
            g = comm.gather_f64(buf)
            if comm.active and int(g[:, 0].max()) > SPECIAL_SLOTS:  # another rank overflowed
                allsp = comm.gather_specials(specials)
            else:
                allsp = [Special(int(row[1 + 4 * j]), int(row[2 + 4 * j]), int(row[3 + 4 * j]),
                                 int(row[4 + 4 * j]), 0) for row in g for j in range(int(row[0]))]
            rows = g[:, 1 + 4 * SPECIAL_SLOTS:]
        nxt = spacing_rejections(allsp, rejected) if len(allsp) >= 2 else list(rejected)
        if nxt == rejected:
            break
        rejected = nxt
    totals, centers, seconds = [], [], []
    for k in range(nout):
        tot = merge_stats(rows[:, 3 * k: 3 * k + 3], 1)
        totals.append(tot)
        centers.append((tot.sum_hi + tot.sum_lo) / tot.n)
    # Exchange 2: centred sums of squares about the global means.
    for k, out in enumerate(outputs[:nout]):
        s2 = stats(out, 2, centers[k])
        seconds += [0.0, s2.ss_hi, s2.ss_lo]
    g2 = comm.gather_f64(seconds)
    cis = []
    for k in range(nout):
        ss = merge_stats(g2[:, 3 * k: 3 * k + 3], 2)
        tot = totals[k]
        tot.center = centers[k]
        tot.ss_hi, tot.ss_lo = ss.ss_hi, ss.ss_lo
        cis.append(ci_from_stats(tot, level))
    return ShardResult(outputs, begin, count, cis, rejected, rounds)


# ---- GPU runner / stats (C ABI) -------------------------------------------------------------


def gpu_runner(model: ModelKind, p, mode, master_seed: int, stream: Optional[int] = None,
               kernel_ms: Optional[list] = None):
    """runner for run_sharded backed by wlp_run_shard on the current CUDA device; outputs
    are torch CUDA tensors (reused across calls of the same shape). When `kernel_ms` is a
    list, each call appends the model kernel's CUDA-event time."""
    import torch

    from . import SimReport, run_shard

    cache = {}

    def run(begin: int, count: int, rejected: Sequence[int]):
        key = count
        if key not in cache:
            cache[key] = [torch.empty(max(count, 1), dtype=torch.float64, device="cuda")
                          for _ in OUTPUT_NAMES[ModelKind(model)]]
        outs = cache[key]
        rep = SimReport() if kernel_ms is not None else None
        specials = run_shard(model, p, mode, master_seed, begin, count, outs, on_device=True, rejected=rejected,
                             stream=stream, report=rep)
        if rep is not None:
            kernel_ms.append(rep.kernel_ms)
        return [o[:count] for o in outs], specials

    def whole(level: float):  # single-rank run (run_sharded's shortcut)
        from . import run_model_into

        outs = cache.setdefault(p.replications, [torch.empty(max(p.replications, 1), dtype=torch.float64,
                                                             device="cuda") for _ in OUTPUT_NAMES[ModelKind(model)]])
        rep = SimReport() if kernel_ms is not None else None
        cis = run_model_into(model, p, mode, master_seed, outs, on_device=True, stream=stream, ci_level=level,
                             report=rep)
        if rep is not None:
            kernel_ms.append(rep.kernel_ms)
        return [o[: p.replications] for o in outs], cis

    run.whole = whole
    return run


def gpu_stats(stream: Optional[int] = None):
    from . import stats_device

    def st(out, pass_: int, center: float) -> Stats:
        n = out.numel()
        s = Stats(n, 0.0, 0.0, center, 0.0, 0.0)
        if n == 0:  # an empty shard (more ranks than replications)
            return s
        return stats_device(out, n, pass_, s, stream)

    return st
