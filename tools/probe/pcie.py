"""PCIe roofline for the e2e leg: pinned host <-> device copy rates, one
direction at a time and both at once (separate streams), at the bench's sizes."""
import json
import time

import torch

dev = torch.device("cuda", 0)
nb_in, nb_out = 2757480056, 2681224192
hin = torch.empty(nb_in // 4, dtype=torch.float32).pin_memory()
hout = torch.empty(nb_out // 4, dtype=torch.float32).pin_memory()
din = torch.empty(nb_in // 4, dtype=torch.float32, device=dev)
dout = torch.empty(nb_out // 4, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name in ("h2d", "d2h", "both"):
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                din.copy_(hin, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                hout.copy_(dout, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    dt = min(ts)
    b = (nb_in if name != "d2h" else 0) + (nb_out if name != "h2d" else 0)
    res[name] = {"ms": dt * 1e3, "GBs": b / dt / 1e9}
print(json.dumps(res))
