"""Expert-parallel sharding + all-reduce, world size 2 over gloo on CPU.

Each rank owns experts e % 2 == rank; the per-expert compute is the oracle
(this is host-logic coverage: routing, ownership, the empty-rank path and the
reduction); the GPU executor is covered by the -m gpu parity tests."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sliced_forward as orc
from paper_2411_15715_b200.expert_parallel import ExpertParallelMoE, local_experts, owner_of, route_local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=0, E=8, M=24, H=40, T=7):
    rng = np.random.default_rng(seed)
    experts = [(rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (H, M))) for _ in range(E)]
    router = rng.uniform(-1, 1, (M, E))
    x = rng.uniform(-1, 1, (T, M))
    return experts, router, x


def _worker(rank, world, port, out_q, seed, T):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        experts, router, x = _problem(seed, T=T)

        def local_forward(plan, xt):
            y = np.zeros((x.shape[0], experts[0][2].shape[1]))
            for e, rows, gates in plan:
                w1, w3, w2 = experts[e]
                y[rows] += gates[:, None].astype(np.float64) * orc.dense_forward(x[rows], w1, w2, "silu", w3)
            return torch.from_numpy(y)

        owned = local_experts(len(experts), rank, world)
        moe = ExpertParallelMoE({e: None for e in owned}, router, 2, len(experts),
                                local_forward=local_forward, out_dim=x.shape[1])
        y = moe(torch.from_numpy(x), x_host=x)
        out_q.put((rank, y.numpy(), owned))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,seed", [(7, 0), (1, 3)])
def test_world2_gloo_matches_single_process_oracle(T, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, seed, T)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    experts, router, x = _problem(seed, T=T)
    ref = orc.moe_forward(x, [(w1, w3, w2) for w1, w3, w2 in experts], router, 2)
    owned = {r: o for r, _, o in results}
    assert sorted(owned[0] + owned[1]) == list(range(8)) and not set(owned[0]) & set(owned[1])
    for _, y, _ in results:
        # gates travel as float32 (sp_call.gates), the oracle keeps float64
        assert orc.max_rel_error(y, ref) <= 1e-6


def test_ownership_and_local_routing():
    assert [owner_of(e, 4) for e in range(8)] == [0, 1, 2, 3, 0, 1, 2, 3]
    assert local_experts(8, 1, 3) == [1, 4, 7]
    rng = np.random.default_rng(1)
    x, router = rng.standard_normal((5, 16)), rng.standard_normal((16, 8))
    full = route_local(x, router, 2, range(8))
    ids, gates = orc.route_topk(x @ router, 2)
    covered = sorted((int(r), e) for e, rows, _ in full for r in rows)
    assert covered == sorted((t, int(ids[t, k])) for t in range(5) for k in range(2))
    # a rank whose experts nobody picked gets an empty plan
    unused = [e for e in range(8) if e not in ids]
    assert route_local(x, router, 2, unused) == []


def _col_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_15715_b200.expert_parallel import ColumnShardedFFN, column_shard

        rng = np.random.default_rng(21)
        M, H, T = 32, 90, 5
        w1, w3, w2 = rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (H, M))
        x = rng.uniform(-1, 1, (T, M))
        lo, hi = column_shard(H, rank, world)

        class OracleShard:  # stand-in for this rank's SlicedFFN (GPU path covered by -m gpu)
            def __call__(self, xx):
                return torch.from_numpy(orc.dense_forward(x, w1[:, lo:hi], w2[lo:hi], "silu", w3[:, lo:hi]))

        y = ColumnShardedFFN(OracleShard())(torch.from_numpy(x))
        out_q.put((rank, y.numpy(), (lo, hi)))
    finally:
        dist.destroy_process_group()


def test_world2_column_sharded_dense_ffn():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_col_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(21)
    M, H, T = 32, 90, 5
    w1, w3, w2 = rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (M, H)), rng.uniform(-1, 1, (H, M))
    x = rng.uniform(-1, 1, (T, M))
    ref = orc.dense_forward(x, w1, w2, "silu", w3)
    shards = sorted(r[2] for r in res)
    assert shards == [(0, 45), (45, 90)]
    for _, y, _ in res:
        np.testing.assert_allclose(y, ref, rtol=0, atol=1e-10)
