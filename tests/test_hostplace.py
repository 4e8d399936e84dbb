"""Host placement of one-process-per-GPU ranks (paper_2504_05897_b200/hostplace.py)."""
from paper_2504_05897_b200 import hostplace


def test_parse_cpulist():
    assert hostplace._parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert hostplace._parse_cpulist("") == []


def test_rank_split_between_gpus_sharing_a_node(monkeypatch):
    nodes = {0: list(range(0, 8)), 1: list(range(0, 8)), 2: list(range(8, 16)), 3: list(range(8, 16))}
    monkeypatch.setattr(hostplace, "gpu_local_cpus", lambda d: nodes[d])
    got = [hostplace.rank_cpus(r, 4) for r in range(4)]
    assert got == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11], [12, 13, 14, 15]]
    assert sorted(c for g in got for c in g) == list(range(16))   # disjoint, complete


def test_rank_cpus_unknown_topology(monkeypatch):
    monkeypatch.setattr(hostplace, "gpu_local_cpus", lambda d: None)
    assert hostplace.rank_cpus(0, 2) is None          # no binding when the topology is unknown
