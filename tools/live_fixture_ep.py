"""Expert-parallel live-run decision fixture (GPU box; commits
tests/golden/live_ep.json).  Two ranks (processes sharing the one GPU, gloo
control plane, peer-memory exchange) run the tiny stack in model mode; every
rank records the LayerRequests its decision core saw -- loads of experts homed
elsewhere zeroed, scores whole -- in the reference's trace format, plus the hash
of its decision stream.  tests/test_live_fixture.py replays each rank's trace
through the unmodified reference run_trace at the rank's share of the global
budget (per-rank parity).

    python tools/live_fixture_ep.py
"""
from __future__ import annotations

import json
import os
import socket
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _rank(rank: int, world: int, port: int, q) -> None:
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    import torch
    import torch.distributed as dist

    import paper_2504_05897_b200.core as mcore
    import paper_2504_05897_b200.costs as mcost
    import paper_2504_05897_b200.engine as me
    from paper_2504_05897_b200.ep import rank_ratio
    from paper_2504_05897_b200.moe import SHAPES, HybridMoE
    from paper_2504_05897_b200.tracegen import save_trace
    from stream import digest, from_records

    torch.cuda.set_device(0)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = SHAPES["tiny"]
        eb = mcore.expert_bytes(cfg)
        prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5,
                                     cpu_first_expert_penalty=1.4)
        moe = HybridMoE(cfg, "tiny", me.EnginePolicy(), 0.5, prof, max_tokens=64, ep_rank=rank, ep_world=world,
                        cpu_threads=2, exchange="p2p")
        moe.init_seeded_weights(21)
        g = torch.Generator(device="cuda").manual_seed(21)  # replicated hidden state: same on every rank
        passes, recs = [], []
        for stage, T in [("prefill", 40)] + [("decode", 1)] * 10:
            x = torch.randn((T, moe.H), generator=g, device="cuda").to(torch.bfloat16)
            _, info = moe.forward_pass(x, None, decision_log=True)
            torch.cuda.synchronize()
            recs.extend(info["records"])
            passes.append(mcore.ForwardPass(stage, T, tuple(mcore.make_layer_request(l, lo.tolist(), sc.tolist())
                                                             for l, (lo, sc) in enumerate(info["requests"]))))
        trace = mcore.Trace(cfg, tuple(passes), {"source": f"live B200 run, EP rank {rank}/{world}, model mode"})
        with tempfile.TemporaryDirectory() as d:
            f = Path(d) / "t.jsonl"
            save_trace(trace, f)
            text = f.read_text()
        q.put((rank, {"policy": "mrs", "prefetch": False, "ratio": rank_ratio(cfg, 0.5, rank, world), "seed": 2,
                      "capacity": moe.capacity, "world": world,
                      "profile": {k: getattr(prof, k) for k in prof.__dataclass_fields__},
                      "trace_jsonl": text, "runtime_stream_sha256": digest(from_records(recs, True))}))
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    dst = ROOT / "gpurun_out" / "live_ep.json"
    dst.parent.mkdir(exist_ok=True)
    dst.write_text(json.dumps({f"rank{r}": v for r, v in sorted(out.items())}))
    print(dst, {r: v["runtime_stream_sha256"][:16] for r, v in out.items()})
