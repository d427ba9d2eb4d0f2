"""Expert parallelism end to end on the GPU: two processes on one B200 (the
only device this run has), each owning half the experts with real GG / CG /
CC placement and the native router (sp_moe_forward with the other rank's
experts absent), partial outputs summed by an all-reduce (gloo here; NCCL is
the same call on separate GPUs).  Both ranks must get the oracle's MoE layer."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import sliced_forward as orc

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _weights(E=8, M=256, H=768, seed=7):
    rng = np.random.default_rng(seed)
    ws = [tuple(rng.standard_normal(s).astype(np.float32) / 8 for s in ((H, M), (H, M), (M, H))) for _ in range(E)]
    router = rng.standard_normal((M, E))
    x = rng.standard_normal((6, M)).astype(np.float32)
    return ws, router, x


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), SP_HOST_THREADS="4")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2411_15715_b200 as sp
        from paper_2411_15715_b200 import _native as nat
        from paper_2411_15715_b200.expert_parallel import ExpertParallelMoE, local_experts

        nat.init(0, 4)
        ws, router, x = _weights()
        owned = local_experts(len(ws), rank, world)
        experts = {e: sp.SlicedFFN(ws[e][0], ws[e][2], sp.SlicingRates(0.25, 0.25, 0.5), w3t=ws[e][1],
                                   dtype="bf16", chunk_rows=128) for e in owned}
        moe = ExpertParallelMoE(experts, router, 2, len(ws), out_dim=x.shape[1])
        y = moe(torch.from_numpy(x).cuda().to(torch.bfloat16))
        out_q.put((rank, y.float().cpu().numpy(), owned))
    except Exception as e:  # surface worker failures in the parent
        out_q.put((rank, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


def test_world2_on_one_gpu_matches_oracle():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    for r, y, owned in results:
        assert owned is not None, y
    ws, router, x = _weights()
    q16 = orc.bf16_round
    ref = orc.moe_forward(q16(x), [(q16(a.T), q16(b.T), q16(c.T)) for a, b, c in ws],
                          router.astype(np.float32).astype(np.float64), 2)
    owned = {r: o for r, _, o in results}
    assert sorted(owned[0] + owned[1]) == list(range(8))
    for _, y, _ in results:
        assert orc.max_rel_error(y, ref) <= 1e-2
