"""Multi-process sharding protocol, world size 2 over gloo:
  * CPU: each rank takes its event range (pf_shard_events) of engine-shaped
    data -- the per-event NLL terms of the C2 model from the C oracle --,
    forms its exact accumulator, the ranks all-gather the 6-digit
    accumulators (what bench.py does over NCCL) and combine them
    (pf_combine_partials): bit for bit the single-process value, whatever
    the rank order;
  * GPU: two processes each bind their shard of the REAL engine
    (shard_index / shard_count, pf_eval_partial) on the one visible device
    (their kernels never wait on each other), exchange the digits over gloo
    and combine: bit for bit the single-process eval_metric."""
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
    """-log density of the C2 mixture at its fit start, per event (the C
    oracle's restatement of the reference's per-event NLL term)"""
    sys.path.insert(0, os.path.dirname(HERE))
    import oracle
    from paper_1311_1753_b200 import parfit as pf
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C2"]
    obs, pdf = W.build(pf)
    cols = W.columns(n, seed=5)
    o = oracle.Oracle(pdf, pf.UnbinnedDataSet.from_columns(obs, cols), W.grid)
    p = [W.start[nm] for nm in o.param_names()]
    o.eval(p)  # normalises
    return -np.log(o.density(p, cols[None, :]))


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


def _gpu_worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1311_1753_b200 import parfit as pf
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C2"]
    obs, pdf = W.build(pf)
    ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(n, seed=7))
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid), shard_index=rank, shard_count=world)
    vals = []
    for k in range(3):  # three parameter points, as a fit's probes
        p = W.params(bm) * (1.0 + 1e-3 * k)
        digits, penalty = bm.eval_partial(p)
        send = torch.tensor(digits + [int(penalty)], dtype=torch.int64)
        recv = torch.empty(7 * world, dtype=torch.int64)
        dist.all_gather_into_tensor(recv, send)
        rows = recv.view(world, 7).tolist()
        assert not any(r[-1] for r in rows)
        vals.append(pf.combine_partials([r[:-1] for r in rows]))
    out[rank] = vals
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_process_engine_shards_bitwise_on_one_gpu():
    """the real engine, two processes, one shard each (pf_eval_partial), digits
    exchanged over gloo: bitwise the single-process value (the reference's
    backend invariance, test_engine.cpp:123-148)"""
    n = 1_000_003
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gpu_worker, args=(2, _free_port(), n, out), nprocs=2, join=True)
        res = dict(out)
    from paper_1311_1753_b200 import parfit as pf
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C2"]
    obs, pdf = W.build(pf)
    bm = pf.BoundModel(pdf, pf.UnbinnedDataSet.from_columns(obs, W.columns(n, seed=7)), pf.GridSpec(W.grid))
    single = [bm.eval_metric(W.params(bm) * (1.0 + 1e-3 * k)) for k in range(3)]
    assert res[0] == res[1] == single
