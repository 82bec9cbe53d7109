"""Probe: pinned host -> device copy bandwidth with one vs two copy streams (8 MB pieces, as
plt_query_host's per-array chunk copies), to decide whether splitting a chunk's arrays over
two DMA engines pays.  Prints GB/s per mode."""
import json
import torch

MB = 1 << 20
piece = 8 * MB
n_pieces = 80
h = torch.empty(n_pieces * piece // 4, dtype=torch.float32).pin_memory()
d = torch.empty_like(h, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(mode):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    if mode == "one_big":
        d.copy_(h, non_blocking=True)
    else:
        for k in range(n_pieces):
            st = s1 if (mode == "one_stream" or k % 2 == 0) else s2
            with torch.cuda.stream(st):
                d[k * piece // 4:(k + 1) * piece // 4].copy_(h[k * piece // 4:(k + 1) * piece // 4], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return n_pieces * piece / (e0.elapsed_time(e1) * 1e-3) / 1e9


res = {}
for mode in ("one_big", "one_stream", "two_streams"):
    run(mode)
    res[mode] = max(run(mode) for _ in range(5))
print(json.dumps({"h2d_GBs": res, "piece_MB": piece // MB, "total_MB": n_pieces * piece // MB}))
