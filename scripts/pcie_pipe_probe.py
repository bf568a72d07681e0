"""e2e ceiling probe: the C5 host path's copies alone (no kernels) - 4.25 GB of
pinned host rays to the device in 2^21-ray (64 MB) chunks and 16 B results
(32 MB chunks) back, H2D and D2H on separate streams with 4 slots, as
lsnif_query_host_wire schedules them. Prints the copy-only time per frame."""
import json
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 132_710_400
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 21
h_in = torch.empty(n * 32, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n * 16, dtype=torch.uint8).pin_memory()
slots = 4
d_in = [torch.empty(chunk * 32, dtype=torch.uint8, device="cuda") for _ in range(slots)]
d_out = [torch.empty(chunk * 16, dtype=torch.uint8, device="cuda") for _ in range(slots)]
st = [torch.cuda.Stream() for _ in range(slots)]


def frame():
    for i, s in enumerate(range(0, n, chunk)):
        c = min(chunk, n - s)
        k = i % slots
        with torch.cuda.stream(st[k]):
            d_in[k][: c * 32].copy_(h_in[s * 32:(s + c) * 32], non_blocking=True)
            h_out[s * 16:(s + c) * 16].copy_(d_out[k][: c * 16], non_blocking=True)
    for s_ in st:
        torch.cuda.current_stream().wait_stream(s_)


frame()
torch.cuda.synchronize()
res = []
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    frame()
    b.record()
    torch.cuda.synchronize()
    res.append(a.elapsed_time(b))
ms = min(res)
print(json.dumps({"rays": n, "chunk": chunk, "copy_only_ms": ms, "h2d_GBps": n * 32 / ms / 1e6,
                  "rays_per_s_ceiling": n / ms * 1e3}))
