"""Multi-process sharding protocol on CPU (gloo, world size 2): each rank
takes its event range (pf_shard_events), forms its exact accumulator, the
ranks all-gather the 6-digit accumulators (what bench.py does over NCCL) and
combine them (pf_combine_partials).  The result must equal the single-process
value bit for bit, whatever the rank order."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _terms(n):
    rng = np.random.default_rng(5)
    return -np.log(rng.random(n)) * rng.choice([1.0, 1e-3, 1e3], n)


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ctypes as C

    from paper_1311_1753_b200 import parfit as pf
    from test_host import _digits_of
    first, count = C.c_uint64(), C.c_uint64()
    pf.lib.pf_shard_events(n, 1024, world, rank, C.byref(first), C.byref(count))
    terms = _terms(n)[first.value:first.value + count.value]
    acc = [0] * 6
    for v in terms:
        acc = [a + d for a, d in zip(acc, _digits_of(float(v)))]
    # bench.py's exchange: 6 digits + penalty flag per rank, one flat gather
    send = torch.empty(7, dtype=torch.int64)
    send.numpy()[:] = acc + [0]
    recv = torch.empty(7 * world, dtype=torch.int64)
    dist.all_gather_into_tensor(recv, send)
    rows = recv.view(world, 7).tolist()
    assert not any(r[-1] for r in rows)
    total = pf.combine_partials([r[:-1] for r in rows])
    reversed_total = pf.combine_partials([r[:-1] for r in rows[::-1]])
    out[rank] = (total, reversed_total, int(count.value))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_exact_combine():
    n = 20_000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
        res = dict(out)
    from paper_1311_1753_b200 import parfit as pf
    from test_host import _digits_of
    acc = [0] * 6
    for v in _terms(n):
        acc = [a + d for a, d in zip(acc, _digits_of(float(v)))]
    single = pf.combine_partials([acc])
    assert res[0][0] == res[1][0] == res[0][1] == single
    assert res[0][2] + res[1][2] == n
