"""Multi-GPU host logic on CPU (world size 2, gloo): every rank derives the
same balanced Morton leaf ranges from the (deterministic) tree, the ranges
tile the leaves, and the sum-assembly of per-rank outputs (non-owned = 0.0)
reproduces the single-process result exactly.  The per-rank potentials come
from the oracle here; on GPUs they come from vpg_plan_set_shard plans
(tests/test_gpu_fmm.py::test_target_shards_assemble_bit_exact)."""
import os
import socket

import numpy as np
import pytest

from paper_2203_05933_b200 import multigpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2203_05933_b200 import workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = W.cfg1()
        rest = oracle.restatement()
        t = rest.tree(w.src, w.tgt)
        L, P = t["params"]["levels"], t["params"]["order"]
        costs = multigpu.leaf_costs(t["src_off"], t["tgt_off"], L, P)
        ranges = multigpu.balanced_ranges(costs, world)
        # every rank must derive identical ranges
        gathered = [None] * world
        dist.all_gather_object(gathered, ranges)
        assert all(g == ranges for g in gathered)
        full = rest.plan_sum(0, 0.0, w.src, w.q, w.tgt, 1e-12, threads=2)
        own = multigpu.owned_targets(t["tgt_off"], t["tgt_ids"], ranges[rank])
        local = np.zeros(w.nt)
        local[own] = full[own]
        total = multigpu.assemble(torch.from_numpy(local)).numpy()
        q.put((rank, bool(np.array_equal(total, full)), ranges, float(costs.sum())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_assembly():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, ranges, _ in res:
        assert ok, rank
        assert ranges[0][0] == 0 and ranges[-1][1] == 4 ** 5 and ranges[0][1] == ranges[1][0]


def test_balanced_ranges_properties():
    rng = np.random.default_rng(0)
    costs = rng.exponential(1.0, 4096)
    for world in (1, 2, 3, 8):
        r = multigpu.balanced_ranges(costs, world)
        assert r[0][0] == 0 and r[-1][1] == costs.size
        assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
        loads = [costs[a:b].sum() for a, b in r]
        assert max(loads) - min(loads) <= 2 * costs.max() + 1e-9
    with pytest.raises(ValueError):
        multigpu.balanced_ranges(costs, 0)
