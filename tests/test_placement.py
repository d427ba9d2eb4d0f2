"""Rank placement on the host (paper_2411_15715_b200/placement.py): NUMA node
of each rank's GPU from sysfs, the node's cores split among the ranks that
share it, SP_HOST_THREADS exported -- with a fake two-socket sysfs tree."""

from __future__ import annotations

import os

from paper_2411_15715_b200 import placement as pl


def fake_sysfs(tmp_path, gpus_per_node=4, cores_per_node=8):
    nodes = tmp_path / "devices" / "system" / "node"
    for n in range(2):
        d = nodes / f"node{n}"
        d.mkdir(parents=True)
        lo = n * cores_per_node
        (d / "cpulist").write_text(f"{lo}-{lo + cores_per_node - 1}\n")
    bus = {}
    for g in range(2 * gpus_per_node):
        bid = f"0000:{0x10 + g:02x}:00.0"
        d = tmp_path / "bus" / "pci" / "devices" / bid
        d.mkdir(parents=True)
        (d / "numa_node").write_text(f"{g // gpus_per_node}\n")
        bus[g] = bid
    return bus


def test_cpulist_round_trip():
    assert pl.parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert pl.format_cpulist([11, 0, 1, 2, 3, 8, 10]) == "0-3,8,10-11"


def test_eight_ranks_two_sockets_get_disjoint_local_shares(tmp_path, monkeypatch):
    monkeypatch.setenv("SP_HOST_THREADS", "0")  # restored after the test
    bus = fake_sysfs(tmp_path)
    monkeypatch.setattr(pl, "pci_bus_id", lambda d: bus[d])
    monkeypatch.setattr(pl.os, "sched_getaffinity", lambda pid: set(range(16)))
    shares = []
    for r in range(8):
        p = pl.bind_rank(r, 8, sysfs=tmp_path, apply=False)
        assert p.numa_node == r // 4
        assert os.environ["SP_HOST_THREADS"] == "2"
        shares.append(p.cpus)
    flat = [c for s in shares for c in s]
    assert sorted(flat) == list(range(16))  # every core used once
    for r, s in enumerate(shares):
        assert all(c // 8 == r // 4 for c in s)  # on the GPU's own socket


def test_ranks_sharing_one_gpu_split_its_node(tmp_path, monkeypatch):
    monkeypatch.setenv("SP_HOST_THREADS", "0")  # restored after the test
    bus = fake_sysfs(tmp_path)
    monkeypatch.setattr(pl, "pci_bus_id", lambda d: bus[d])
    monkeypatch.setattr(pl.os, "sched_getaffinity", lambda pid: set(range(16)))
    a = pl.bind_rank(0, 2, device_of=lambda r: 5, sysfs=tmp_path, apply=False)
    b = pl.bind_rank(1, 2, device_of=lambda r: 5, sysfs=tmp_path, apply=False)
    assert a.numa_node == b.numa_node == 1
    assert a.cpus == list(range(8, 12)) and b.cpus == list(range(12, 16))


def test_unknown_node_uses_allowed_cpus(tmp_path, monkeypatch):
    monkeypatch.setenv("SP_HOST_THREADS", "0")
    monkeypatch.setattr(pl, "pci_bus_id", lambda d: None)
    allowed = sorted(os.sched_getaffinity(0))
    p = pl.bind_rank(0, 1, sysfs=tmp_path, apply=True)
    assert p.numa_node is None and p.cpus == allowed and p.mempolicy == "none"
    assert p.summary()["host_threads"] == len(allowed)
