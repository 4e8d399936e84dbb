"""Host placement for one-process-per-GPU runs: the host worker of the rank
driving GPU d runs on the CPUs of d's NUMA node, and the node's CPUs are split
between the ranks whose GPUs hang off it.

The decode step is bound by host DRAM bandwidth: a rank whose
worker threads float across sockets, or whose pinned master store was first
touched on the far node, streams its experts over the socket interconnect.
Binding the process before the runtime allocates its pinned store and starts
its worker threads keeps both on the GPU's node (Linux first-touch; the pool
threads inherit the process affinity).  On a single-node host every GPU has
every CPU, and the split only divides the cores between the ranks.
"""
from __future__ import annotations

import os
from pathlib import Path


def _parse_cpulist(text: str) -> list[int]:
    cpus: list[int] = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.extend(range(int(a), int(b) + 1))
        else:
            cpus.append(int(part))
    return cpus


def gpu_local_cpus(device: int) -> list[int] | None:
    """CPUs local to CUDA device `device` (sysfs local_cpulist of its PCI
    function) intersected with this process's affinity, or None if unknown."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(device)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        text = (Path("/sys/bus/pci/devices") / bdf / "local_cpulist").read_text()
    except Exception:
        return None
    allowed = os.sched_getaffinity(0)
    cpus = [c for c in _parse_cpulist(text) if c in allowed]
    return cpus or None


def rank_cpus(local_rank: int, n_local: int) -> list[int] | None:
    """This rank's CPUs: the local CPUs of its GPU, split evenly (contiguous
    blocks, in GPU index order) among the ranks whose GPUs share that set."""
    sets = [gpu_local_cpus(d) for d in range(n_local)]
    mine = sets[local_rank] if local_rank < len(sets) else None
    if not mine:
        return None
    peers = [d for d in range(n_local) if sets[d] == mine]
    k, m = peers.index(local_rank), len(peers)
    lo, hi = len(mine) * k // m, len(mine) * (k + 1) // m
    return mine[lo:hi] or None


def bind_rank(local_rank: int, n_local: int) -> list[int] | None:
    """Bind this process to its CPUs (before the runtime exists); returns them."""
    cpus = rank_cpus(local_rank, n_local)
    if cpus:
        os.sched_setaffinity(0, cpus)
    return cpus
