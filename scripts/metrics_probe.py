"""Workload driver for the per-ray kernel metrics in profiles/kernel_metrics_<w>.json.

  run:   python scripts/metrics_probe.py run c2|c3
         (one warm-up query set, then the measured set: c2 = primary CLOSEST +
         shadow ANY, c3 = one 2M-ray incoherent chunk; run it under
         ncu --metrics ... -k regex:"trace_encode|mlp_tc" --launch-skip <warm-up launches>)
  parse: python scripts/metrics_probe.py parse c2|c3 ncu.csv rays.json > profiles/kernel_metrics_<w>.json
"""
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ("gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,"
           "smsp__issue_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")


def run(w: str, out_json: str):
    import torch
    from paper_2504_21627_b200 import lsnif, workloads as W
    gm = lsnif.GpuModel(os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif"))
    if w == "c2":
        prim = W.camera_rays(1920, 1080)
        hits = lsnif.hits_to_numpy(gm.query(lsnif.rays_to_tensor(prim, "cuda")))  # not under the filter skip
        sh = W.shadow_rays(prim, hits, gm.aabb)[0]
        sets = [("primary", lsnif.rays_to_tensor(prim, "cuda"), lsnif.CLOSEST),
                ("shadow", lsnif.rays_to_tensor(sh, "cuda"), lsnif.ANY)]
    else:
        rays = W.incoherent_rays(1 << 21, gm.aabb, seed=3)
        sets = [("c3_chunk", lsnif.rays_to_tensor(rays, "cuda"), lsnif.CLOSEST)]
    info = []
    for _, d, mode in sets:  # warm-up set
        gm.query(d, mode)
    torch.cuda.synchronize()
    for name, d, mode in sets:  # measured set
        gm.query(d, mode)
        st = gm.last_stats()
        info.append({"name": name, "rays": int(d.shape[0]), "mlp_rows": st["mlp_rows"]})
    torch.cuda.synchronize()
    with open(out_json, "w") as f:
        json.dump(info, f)


def parse(w: str, csv_path: str, rays_json: str):
    launches = {}
    order = []
    with open(csv_path) as f:
        rows = [r for r in csv.reader(f) if len(r) > 10]
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        key = d["ID"]
        if key not in launches:
            launches[key] = {"kernel": d["Kernel Name"]}
            order.append(key)
        launches[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    info = json.load(open(rays_json))
    traces = [launches[k] for k in order if "trace_encode" in launches[k]["kernel"]][-len(info):]
    mlps = [launches[k] for k in order if "mlp_tc" in launches[k]["kernel"]][-len(info):]
    per = {}
    for s, t in zip(info, traces):
        per[s["name"]] = {"rays": s["rays"], "warp_inst": int(t["smsp__inst_executed.sum"]),
                          "l2_read_sectors": int(t["lts__t_sectors_srcunit_tex_op_read.sum"]),
                          "issue_active": t["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100,
                          "us": t["gpu__time_duration.sum"] / 1e3}
    rays = sum(p["rays"] for p in per.values())
    us = sum(p["us"] for p in per.values())
    out = {"trace_encode_kernel": {
        "rays_per_launch": info[0]["rays"],
        "warp_inst_per_ray": sum(p["warp_inst"] for p in per.values()) / rays,
        "l2_read_bytes_per_ray": 32.0 * sum(p["l2_read_sectors"] for p in per.values()) / rays,
        "issue_active_frac": sum(p["issue_active"] * p["us"] for p in per.values()) / us,
        "duration_us": traces[0]["gpu__time_duration.sum"] / 1e3,
        "per_step": per},
        "mlp_tc_kernel": {
        "tensor_active_frac": float(np.average(
            [m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"] / 100 for m in mlps],
            weights=[m["gpu__time_duration.sum"] for m in mlps])),
        "issue_active_frac": float(np.average(
            [m["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100 for m in mlps],
            weights=[m["gpu__time_duration.sum"] for m in mlps])),
        "duration_us": mlps[0]["gpu__time_duration.sum"] / 1e3,
        "per_step": {s["name"]: {"mlp_rows": s["mlp_rows"], "us": m["gpu__time_duration.sum"] / 1e3}
                     for s, m in zip(info, mlps)}},
        "note": f"ncu --metrics ({METRICS}) over scripts/metrics_probe.py run {w}: per-ray warp instructions "
                "and L2 read sectors of the measured trace launches (time-weighted issue activity), MLP "
                "tensor-pipe / issue activity; ncu times are cold-cache and serialised"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/metrics_rays.json")
    elif sys.argv[1] == "metrics":
        print(METRICS)
    else:
        parse(sys.argv[2], sys.argv[3], sys.argv[4])
