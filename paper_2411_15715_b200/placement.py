"""Host placement of one rank: its GPU's NUMA node, its share of that node's
cores, and a preferred memory policy -- set before ``sp_init`` so the CC
thread pool (created there) inherits the CPU mask and the pinned CC / CG host
regions (first touched by this rank) land in the GPU's socket.

SURVEY.md section 8(e): every GPU streams its CG blocks over its own host link
and runs its CC blocks on its share of the host cores.  On a two-socket
8-GPU node half the GPUs hang off each socket; a rank whose pinned weights
and CC threads sit on the far socket pays the inter-socket link on both the
copy engine's reads and the CC block's DRAM stream.

Everything here is host logic (sysfs + sched_setaffinity + set_mempolicy);
``tests/test_placement.py`` covers it on CPU with a fake sysfs tree.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from pathlib import Path

SYSFS = Path("/sys")
_SYS_SET_MEMPOLICY = 238  # x86_64
_MPOL_PREFERRED = 1


def parse_cpulist(text: str) -> list[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11] (the kernel's cpulist format)."""
    out: list[int] = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            lo, hi = part.split("-")
            out.extend(range(int(lo), int(hi) + 1))
        else:
            out.append(int(part))
    return out


def format_cpulist(cpus: list[int]) -> str:
    cpus = sorted(cpus)
    runs, start, prev = [], None, None
    for c in cpus:
        if start is None:
            start = prev = c
        elif c == prev + 1:
            prev = c
        else:
            runs.append((start, prev))
            start = prev = c
    if start is not None:
        runs.append((start, prev))
    return ",".join(f"{a}-{b}" if a != b else f"{a}" for a, b in runs)


def pci_bus_id(device: int) -> str | None:
    """'0000:1b:00.0' of a visible CUDA device (sysfs spelling), or None."""
    try:
        import torch

        p = torch.cuda.get_device_properties(device)
        return f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:
        return None


def numa_node_of(bus_id: str | None, sysfs: Path = SYSFS) -> int | None:
    if not bus_id:
        return None
    f = sysfs / "bus" / "pci" / "devices" / bus_id.lower() / "numa_node"
    try:
        n = int(f.read_text().strip())
    except (OSError, ValueError):
        return None
    return n if n >= 0 else None


def node_cpus(node: int | None, sysfs: Path = SYSFS) -> list[int]:
    """CPUs of a NUMA node that this process may run on (all allowed CPUs when
    the node is unknown)."""
    allowed = sorted(os.sched_getaffinity(0))
    if node is None:
        return allowed
    try:
        cpus = parse_cpulist((sysfs / "devices" / "system" / "node" / f"node{node}" / "cpulist").read_text())
    except OSError:
        return allowed
    mine = [c for c in cpus if c in set(allowed)]
    return mine or allowed


@dataclass
class RankPlacement:
    local_rank: int
    device: int
    numa_node: int | None
    cpus: list[int] = field(default_factory=list)
    mempolicy: str = "none"

    def summary(self) -> dict:
        return {"local_rank": self.local_rank, "device": self.device, "numa_node": self.numa_node,
                "cpus": format_cpulist(self.cpus), "host_threads": len(self.cpus), "mempolicy": self.mempolicy}


def plan_rank(local_rank: int, devices: list[int], nodes: list[int | None], node_cpu_lists: dict) -> list[int]:
    """This rank's cores: the ranks whose GPUs share its NUMA node split that
    node's cores into equal contiguous shares (``devices[i]`` / ``nodes[i]`` =
    local rank i's GPU and its node; ``node_cpu_lists[node]`` = the node's
    usable cores)."""
    node = nodes[local_rank]
    peers = [r for r in range(len(devices)) if nodes[r] == node]
    k, m = peers.index(local_rank), len(peers)
    cpus = node_cpu_lists[node]
    lo, hi = len(cpus) * k // m, len(cpus) * (k + 1) // m
    share = cpus[lo:hi]
    return share or cpus[:1]


def set_preferred_node(node: int) -> bool:
    """set_mempolicy(MPOL_PREFERRED, {node}) for this thread (best effort)."""
    try:
        libc = ctypes.CDLL(None, use_errno=True)
        mask = ctypes.c_ulong(1 << node)
        return libc.syscall(_SYS_SET_MEMPOLICY, _MPOL_PREFERRED, ctypes.byref(mask), 64) == 0
    except Exception:
        return False


def bind_rank(local_rank: int, local_world: int, device_of=lambda r: r, sysfs: Path = SYSFS,
              apply: bool = True) -> RankPlacement:
    """Pin this process to its share of its GPU's NUMA node and prefer that
    node's memory (``apply``); export SP_HOST_THREADS so sp_init sizes the CC
    pool to the share and the planner scales its CPU terms to it.

    ``device_of(r)`` maps a local rank to its CUDA device (identity for one GPU
    per rank; a constant when several test ranks share one GPU)."""
    devices = [device_of(r) for r in range(local_world)]
    nodes = [numa_node_of(pci_bus_id(d), sysfs) for d in devices]
    lists = {n: node_cpus(n, sysfs) for n in set(nodes)}
    cpus = plan_rank(local_rank, devices, nodes, lists)
    pl = RankPlacement(local_rank, devices[local_rank], nodes[local_rank], cpus)
    if apply:
        try:
            os.sched_setaffinity(0, cpus)
        except OSError:
            pl.cpus = sorted(os.sched_getaffinity(0))
        if pl.numa_node is not None and set_preferred_node(pl.numa_node):
            pl.mempolicy = f"preferred:{pl.numa_node}"
    # the planner's CPU terms and the CC pool size follow this rank's share
    # (also without `apply`: the reference arm plans exactly as rank 0 does)
    os.environ["SP_HOST_THREADS"] = str(len(pl.cpus))
    return pl
