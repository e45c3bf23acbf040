"""Multi-GPU sweep driver: one process per GPU (torchrun), problems statically partitioned with
the library's LPT cost model (hb_partition), no collective on the data path; the only
collective is one all_gather of fixed-size result records at the end (NCCL on GPUs, gloo in the
CPU tests).  Replaces the reference's std::thread parallel_for over independent blocks
(parallel.hpp:12-29) at the scale of a node.
"""
from __future__ import annotations

from typing import Callable, Sequence

from .hb import RankResult, hb_problem, partition

REC = 17  # float64 fields per packed record


def pack(idx: int, t: int, r: RankResult) -> list[float]:
    return [float(idx), float(t), float(r.rank), float(r.rank_lo), float(r.rank_hi),
            float(r.k_factored), r.sigma1, r.sigma_r, r.sigma_r1, r.gap, r.resid] + list(r.sec) + \
        [float(r.certificate), r.fp_band]


def unpack(row) -> tuple[int, int, RankResult]:
    v = [float(x) for x in row]
    return int(v[0]), int(v[1]), RankResult(int(v[2]), int(v[3]), int(v[4]), int(v[5]), v[6], v[7],
                                            v[8], v[9], v[10], v[11:15], int(v[15]), v[16])


def my_share(problems: Sequence[hb_problem], rank: int, world: int) -> list[int]:
    owner = partition(problems, world)
    return [i for i, o in enumerate(owner) if o == rank]


def gather_results(problems: Sequence[hb_problem], mine: Sequence[int], my_results, device=None):
    """all_gather the packed records of every rank; returns results in problem order."""
    import torch
    import torch.distributed as dist
    rows = [pack(i, t, r) for i, res in zip(mine, my_results) for t, r in enumerate(res)]
    world = dist.get_world_size()
    cnt = torch.tensor([len(rows)], dtype=torch.int64, device=device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    mx = max(int(c.item()) for c in cnts)
    buf = torch.zeros((max(mx, 1), REC), dtype=torch.float64, device=device)
    if rows:
        buf[: len(rows)] = torch.tensor(rows, dtype=torch.float64, device=device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    full: list[list] = [[None] * p.ntol for p in problems]
    for c, o in zip(cnts, outs):
        for row in o[: int(c.item())].cpu().tolist():
            i, t, r = unpack(row)
            full[i][t] = r
    return full


def run_partitioned(problems: Sequence[hb_problem], run_fn: Callable, device=None):
    """Each rank runs its LPT share with run_fn(list_of_problems) -> list[list[RankResult]],
    then results are all-gathered.  Returns (full results, my indices, my results)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    mine = my_share(problems, rank, world)
    my_results = run_fn([problems[i] for i in mine]) if mine else []
    return gather_results(problems, mine, my_results, device), mine, my_results
