"""Expert-parallel sliced MoE layer across GPUs (one process per GPU).

SURVEY.md §8(e): experts shard naturally.  Rank r owns experts
``e % world == r``; each owned expert keeps its own CC / CG / GG split, so every
GPU streams its CG blocks over its own host link and runs its CC blocks on its
share of the host cores.  All ranks route the same tokens (the router is tiny
and replicated), compute their local experts' gated contributions with one
``sp_forward_batch``, and one all-reduce (NCCL over NVLink on GPUs; gloo in the
CPU tests) sums the partial outputs -- the path's only exchange step, since a
token's output needs both of its top-2 experts.

The local executor is pluggable (``local_forward``) so the sharding, routing
and reduction logic can be exercised on CPU with world size 2; on GPUs it is
``sliced.forward_calls``.
"""

from __future__ import annotations

from typing import Callable, Mapping, Sequence

import numpy as np

from .errors import ShapeMismatch
from .sliced import CallSpec, MoEDispatch, forward_calls, moe_route


def owner_of(expert: int, world: int) -> int:
    """Round-robin expert placement."""
    return expert % world


def local_experts(n_experts: int, rank: int, world: int) -> list[int]:
    return [e for e in range(n_experts) if owner_of(e, world) == rank]


def route_local(x_host: np.ndarray, router_w: np.ndarray, top_k: int, owned: Sequence[int]):
    """Top-k routing of every token through the runtime's router (sp_moe_route:
    fp64 logits over the fp32 router, ties -> lower expert id -- the same
    routine sp_moe_forward runs), restricted to the owned experts:
    [(expert, token_rows int32, gates float32)]."""
    ids, gates = moe_route(np.asarray(x_host, dtype=np.float32), router_w, top_k)
    plan = []
    for e in owned:
        rows, slots = np.nonzero(ids == e)
        if rows.size:
            order = np.argsort(rows, kind="stable")
            rows, slots = rows[order], slots[order]
            plan.append((e, rows.astype(np.int32), gates[rows, slots].astype(np.float32)))
    return plan


class ExpertParallelMoE:
    """Top-k MoE whose experts are split over the ranks of a process group.

    ``experts`` maps the expert ids this rank owns to placed layers
    (``SlicedFFN``); ``local_forward(plan, x) -> y`` overrides the executor
    (default: one ``sp_forward_batch`` over the owned, active experts).
    """

    def __init__(self, experts: Mapping[int, object], router_w, top_k: int, n_experts: int,
                 group=None, local_forward: Callable | None = None, out_dim: int | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.router_w = np.ascontiguousarray(router_w, dtype=np.float32)  # as sp_moe_route holds it
        if self.router_w.shape[1] != n_experts:
            raise ShapeMismatch("router_w must have one column per expert")
        self.top_k = int(top_k)
        self.n_experts = int(n_experts)
        self.owned = local_experts(n_experts, self.rank, self.world)
        missing = set(self.owned) - set(experts)
        if missing:
            raise ValueError(f"rank {self.rank} owns experts {sorted(missing)} but got no layer for them")
        self.experts = dict(experts)
        if out_dim is None:
            out_dim = (next(iter(self.experts.values())).layer.out_dim if self.experts
                       else self.router_w.shape[0])
        self.out_dim = int(out_dim)
        self.local_forward = local_forward or self._gpu_local_forward
        self._dispatch = None

    def _gpu_local_forward(self, plan, x):
        calls = [CallSpec(self.experts[e].layer, rows, gates) for e, rows, gates in plan]
        return forward_calls(calls, x, self._partial_out(x))

    def _partial_out(self, x):
        """fp32 buffer for this rank's partial output when it is all-reduced: the
        partials are summed in fp32 across ranks (as the single-GPU finalize sums
        its slices) and rounded to x's dtype once, after the reduction."""
        import torch

        if self.world > 1 and isinstance(x, torch.Tensor) and x.is_cuda and x.dtype != torch.float32:
            return torch.empty((x.shape[0], self.out_dim), dtype=torch.float32, device=x.device)
        return None

    def forward(self, x, x_host: np.ndarray | None = None):
        """y = sum over ranks of the owned experts' gated outputs (all-reduced).

        ``x``: torch tensor [T, M] (CUDA for the GPU executor); ``x_host``: its
        values on the host for routing (computed from ``x`` if omitted)."""
        import torch

        if x_host is None and self.local_forward == self._gpu_local_forward:
            # native routing + dispatch: one read-back of x serves router and CC blocks
            if self._dispatch is None:
                layers = [self.experts[e].layer if e in self.experts else None for e in range(self.n_experts)]
                self._dispatch = MoEDispatch(layers, self.router_w, self.top_k)
            y = self._dispatch(x, self._partial_out(x))
            if not isinstance(y, torch.Tensor):
                y = torch.as_tensor(np.ascontiguousarray(y))
            return self._reduce(y).to(x.dtype) if isinstance(x, torch.Tensor) and x.is_cuda else self._reduce(y)
        if x_host is None:
            x_host = x.detach().float().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
        plan = route_local(x_host, self.router_w, self.top_k, self.owned)
        on_gpu = isinstance(x, torch.Tensor) and x.is_cuda
        if plan:
            y = self.local_forward(plan, x)
            if not isinstance(y, torch.Tensor):
                y = torch.as_tensor(np.ascontiguousarray(y))
        else:
            dev = x.device if isinstance(x, torch.Tensor) else "cpu"
            dt = torch.float32 if on_gpu and self.world > 1 else x.dtype if isinstance(x, torch.Tensor) else torch.float64
            y = torch.zeros((x_host.shape[0], self.out_dim), dtype=dt, device=dev)
        y = self._reduce(y)
        return y.to(x.dtype) if on_gpu else y

    def _reduce(self, y):
        """Sum the ranks' partial outputs (one all-reduce: NCCL on GPUs)."""
        import torch

        if self.world > 1:
            if y.device.type == "cpu" and self.dist.get_backend(self.group) == "nccl":
                yd = y.to(f"cuda:{torch.cuda.current_device()}")
                self.dist.all_reduce(yd, group=self.group)
                return yd.cpu()
            self.dist.all_reduce(y, group=self.group)
        return y

    __call__ = forward


def column_shard(hidden: int, rank: int, world: int) -> tuple[int, int]:
    """Hidden columns [lo, hi) owned by `rank` (BASELINE configs[3]: a dense FFN
    column-sharded over G GPUs -- the same algebra as the CC/CG/GG split)."""
    return hidden * rank // world, hidden * (rank + 1) // world


class ColumnShardedFFN:
    """Dense FFN whose hidden columns are split over the ranks; every rank runs
    its own CC/CG/GG split of its shard (rates solved on LayerSpec(M, H/G)) and
    one all-reduce sums the partial outputs."""

    def __init__(self, shard, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.shard = shard  # SlicedFFN over this rank's columns

    def forward(self, x):
        import torch

        out = None
        if self.world > 1 and isinstance(x, torch.Tensor) and x.is_cuda and x.dtype != torch.float32:
            # fp32 partials across the ranks, one rounding after the sum
            out = torch.empty((x.shape[0], self.shard.layer.out_dim), dtype=torch.float32, device=x.device)
        y = self.shard(x, out=out) if out is not None else self.shard(x)
        if not isinstance(y, torch.Tensor):
            y = torch.as_tensor(np.ascontiguousarray(y))
        if self.world > 1:
            if y.device.type == "cpu" and self.dist.get_backend(self.group) == "nccl":
                yd = y.to(f"cuda:{torch.cuda.current_device()}")
                self.dist.all_reduce(yd, group=self.group)
                return yd.cpu()
            self.dist.all_reduce(y, group=self.group)
        return y.to(x.dtype) if out is not None else y

    __call__ = forward
