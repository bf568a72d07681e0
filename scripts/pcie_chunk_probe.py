"""Copy-only version of lsnif_query_host's pipeline (4 streams, 128K-ray
chunks, H2D then D2H per chunk): the e2e ceiling without any kernels."""
import json
import torch

n = 2073600
rec = 32
h_in = torch.empty(n * rec, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n * rec, dtype=torch.uint8).pin_memory()
slots = 4
chunk = 131072
d_in = [torch.empty(chunk * rec, dtype=torch.uint8, device="cuda") for _ in range(slots)]
streams = [torch.cuda.Stream() for _ in range(slots)]


def run():
    k = 0
    for s in range(0, n, chunk):
        cn = min(chunk, n - s)
        st = streams[k % slots]
        with torch.cuda.stream(st):
            d = d_in[k % slots]
            d[: cn * rec].copy_(h_in[s * rec:(s + cn) * rec], non_blocking=True)
            h_out[s * rec:(s + cn) * rec].copy_(d[: cn * rec], non_blocking=True)
        k += 1
    for st in streams:
        st.synchronize()


import time
run()
t0 = time.perf_counter()
for _ in range(20):
    run()
dt = (time.perf_counter() - t0) / 20
print(json.dumps({"copy_only_pipeline_ms": dt * 1e3, "rays_per_s": n / dt}))
