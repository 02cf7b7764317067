"""Row sharding (paper_2012_06607_b200/shard.py): the partition
covers every row exactly once and balances product counts; ranks compute the
same partition independently (gloo, world_size 2); a sharded evaluation
(oracle, tiny system) reassembles the full system's outputs exactly."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import mdinputs
import oracle
from paper_2012_06607_b200 import shard


def test_row_products_match_the_schedule_count():
    si = mdinputs.make_config("qd")            # exponents 1 and 2: common factors
    costs = shard.row_products(si.poly_ptr, si.mono_ptr, si.exps)
    assert sum(costs) == 36575                  # mdps_system_stats products


def test_partition_covers_and_balances():
    si = mdinputs.make_config("od")
    costs = shard.row_products(si.poly_ptr, si.mono_ptr, si.exps)
    for parts in (1, 2, 3, 8):
        rows = shard.partition_rows(costs, parts)
        flat = sorted(r for part in rows for r in part)
        assert flat == list(range(si.n))
        loads = [sum(costs[i] for i in part) for part in rows]
        assert max(loads) - min(loads) <= max(costs)   # LPT bound


def test_sharded_eval_reassembles_full_outputs():
    si = mdinputs.random_system(5, 6, 4, (1, 3), (1, 2), 5, 2)
    vals, jac, _ = oracle.eval_diff(si)
    rows = shard.partition_rows(shard.row_products(si.poly_ptr, si.mono_ptr, si.exps), 2)
    for part in rows:
        pp, mp_, vv, ee, cc = shard.subsystem(si.poly_ptr, si.mono_ptr, si.vars, si.exps, si.coeffs, part)
        sub = mdinputs.SystemInputs("part", si.n, si.degree, si.limbs, pp, mp_, vv, ee, cc, si.x)
        v, j, _ = oracle.eval_diff(sub)
        assert np.array_equal(v, vals[part]) and np.array_equal(j, jac[part])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    si = mdinputs.make_config("dd")
    rows = shard.partition_rows(shard.row_products(si.poly_ptr, si.mono_ptr, si.exps), world)[rank]
    got = [None] * world
    dist.all_gather_object(got, rows)
    out[rank] = got
    dist.destroy_process_group()


def test_ranks_agree_on_the_partition_gloo_world2():
    world, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1]
    assert sorted(r for part in out[0] for r in part) == list(range(8))
    assert not set(out[0][0]) & set(out[0][1])
