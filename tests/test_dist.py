"""Multi-rank sweep host logic on CPU: world_size 2 over gloo (127.0.0.1).  The per-rank compute
is the CPU oracle at tiny N (tests only); what is under test is the LPT split, the record
packing and the result all_gather that bench.py uses over NCCL on GPUs."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problems(hb):
    probs = []
    for n in (64, 125, 216):
        for d in (1, 2, 3):
            for dp in list(range(d)) + [None]:
                probs.append(hb.make_problem("exp_neg_r", d, dp, n, [1e-12, 1e-8]))
    return probs


def _oracle_run(problems):
    import paper_2209_05819_b200 as hb
    from oracle import oracle as O
    out = []
    for p in problems:
        d, dp = p.pair.target.d, (None if p.pair.d_prime < 0 else p.pair.d_prime)
        recs = O.rank_problem(d, dp, hb.KERNEL_NAMES[p.kernel.id], p.pair.n_target,
                              list(p.tols[: p.ntol]), seed=p.pair.seed, nthreads=1)
        out.append([hb.RankResult(r.rank, r.rank, r.rank, 0, r.sigma1, r.sigma_r, r.sigma_r1,
                                  r.gap, 0.0, [0.0] * 4) for r in recs])
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2209_05819_b200 as hb
    from paper_2209_05819_b200 import dist as hbd
    probs = _problems(hb)
    full, mine, _ = hbd.run_partitioned(probs, _oracle_run)
    q.put((rank, mine, [[r.rank for r in res] for res in full]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sweep_gather(hb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    (_, mine0, full0), (_, mine1, full1) = got
    probs = _problems(hb)
    assert sorted(mine0 + mine1) == list(range(len(probs)))  # every problem exactly once
    assert not set(mine0) & set(mine1)
    assert full0 == full1                                     # both ranks see all results
    ref = [[r.rank for r in res] for res in _oracle_run(probs)]
    assert full0 == ref
