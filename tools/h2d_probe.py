"""Pinned H2D copy throughput of one expert image (352 MB, Mixtral) issued as
one copy, as chunks on one stream, and as chunks spread over 2-4 streams."""
import json
import torch

nb = 3 * 4096 * 14336 * 2
n_img = 6
src = torch.empty((n_img, nb), dtype=torch.uint8).pin_memory()
dst = torch.empty((n_img, nb), dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
res = {}


def run(chunks, nstreams, reps=12):
    c = nb // chunks
    ev = [torch.cuda.Event() for _ in streams]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for s in streams[:nstreams]:
        s.wait_event(a)
    for r in range(reps):
        i = r % n_img
        for k in range(chunks):
            s = streams[k % nstreams]
            with torch.cuda.stream(s):
                dst[i, k * c:(k + 1) * c].copy_(src[i, k * c:(k + 1) * c], non_blocking=True)
    for j, s in enumerate(streams[:nstreams]):
        ev[j].record(s)
        cur.wait_event(ev[j])
    b.record(cur)
    b.synchronize()
    return reps * nb / (a.elapsed_time(b) / 1e3) / 1e9


for chunks, ns in ((1, 1), (4, 1), (2, 2), (4, 2), (8, 2), (4, 4), (16, 4)):
    run(chunks, ns, 3)
    res[f"chunks{chunks}-streams{ns}"] = round(max(run(chunks, ns) for _ in range(3)), 2)
print(json.dumps(res))
