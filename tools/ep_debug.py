"""Run the two-rank expert-parallel stack on one GPU with progress logs (debug aid).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/ep_debug.py
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
log = open(f"gpurun_out/ep_rank{rank}.log", "w")


def say(*a):
    print(f"[{time.time():.3f}] rank {rank}:", *a, file=log, flush=True)


say("start")
torch.cuda.set_device(0)
dist.init_process_group("gloo")
say("pg up")
import paper_2504_05897_b200.core as mcore  # noqa: E402
import paper_2504_05897_b200.costs as mcost  # noqa: E402
from paper_2504_05897_b200.engine import EnginePolicy  # noqa: E402
from paper_2504_05897_b200.moe import SHAPES, HybridMoE  # noqa: E402
from paper_2504_05897_b200.tracegen import GenParams, generate_router_logits  # noqa: E402

cfg = SHAPES["tiny"]
eb = mcore.expert_bytes(cfg)
prof = mcost.HardwareProfile(gpu_time_per_expert=1.0, cpu_slope=2.0, transfer_bandwidth=eb / 0.5)
moe = HybridMoE(cfg, "tiny", EnginePolicy(), 0.5, prof, max_tokens=48, ep_rank=rank, ep_world=world, cpu_threads=2)
say("moe up, capacity", moe.capacity)
moe.init_seeded_weights(7)
say("weights")
t = torch.ones(4, device="cuda")
dist.all_reduce(t)
say("cuda allreduce ok", t.tolist())
trace, logits = generate_router_logits(cfg, GenParams(seed=3), 32, 3)
for p, fwd in enumerate(trace.passes):
    lg = [torch.from_numpy(np.ascontiguousarray(logits[p][l], dtype=np.float32)).cuda() for l in range(cfg.num_layers)]
    x = torch.randn((fwd.token_count, moe.H), device="cuda").to(torch.bfloat16)
    say("pass", p, "begin")
    y, info = moe.forward_pass(x, lg)
    torch.cuda.synchronize()
    say("pass", p, "done", float(y.float().abs().sum()))
dist.destroy_process_group()
say("exit")
