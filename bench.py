#!/usr/bin/env python
"""LSNIF batched ray-query benchmark on B200.

Metric (BASELINE.json): LSNIF ray queries/sec, one query = one input ray
answered (including rays that miss the frame box).

Default workload (configs[4], "C5", the north-star configuration): the teapot
LSNIF fixture (tests/golden/teapot_seed0.lsnif: reference train() setup
state, seed 0), 3840x2160 x 16 spp = 132,710,400 incoherent rays keyed by
(pixel, sample), answered with the closest-hit rule (run_narrow_phase,
renderer.cpp:232-265). The frame is split into contiguous row bands, one per
GPU (strong scaling); every rank regenerates its own band from the
index-addressable generator and answers it in pieces, and each finished
piece is sent point-to-point into rank 0's full-frame result on a side
stream while the next piece computes (NCCL over NVLink, the one collective,
inside the timed step). Results are the packed 16 B wire records
(lsnif_hit_wire). At N = 1 the same frame runs on one GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c3|c2|c1|c4|render]
  python bench.py --impl reference   # the reference's CPU algorithm on the same rays

`--gpus N` with N > 1 outside torchrun relaunches itself under
torch.distributed.run with N ranks; under torchrun WORLD_SIZE must equal N.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL_PATH = os.path.join(ROOT, "tests", "golden", "teapot_seed0.lsnif")
METRIC = "LSNIF ray queries/sec at 1/2/4/8 B200, % of roofline, vs CPU ref (cores)"
UNIT = "rays/s"
L2_FLUSH_BYTES = 256 << 20
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
C5_RAYS = 3840 * 2160 * 16
C5_SEED = 5
C5_CPU_STRIDE = 64          # CPU sample of C5: every 64th ray (2,073,600 rays), both CPU arms
C5_PIECES = 8               # compute / gather pieces per band at N > 1

WORKLOADS = {
    "c5": "C5 (configs[4]): teapot LSNIF, 3840x2160 x 16 spp incoherent rays (132,710,400, "
          "keyed by (pixel, sample): origins uniform in the frame box, directions uniform on S^2, "
          "seed 5), closest-hit, packed 16 B results; contiguous row bands, one per GPU, each band "
          "answered in 8 pieces whose results go point-to-point (NCCL) into rank 0's full-frame "
          "buffer while the next piece computes (strong scaling)",
    "c2": "C2 (configs[1]): teapot LSNIF (seed-0 reference init), 1920x1080 pixel-centre "
          "primary rays (closest-hit) + NEE shadow rays toward a point light from the "
          "CPU reference's accepted primary hits (any-hit; the same shadow set for every arm), "
          "one frame per GPU",
    "c3": "C3 (configs[2]): teapot LSNIF, 16,777,216 incoherent rays (origins uniform in "
          "the frame box, directions uniform on S^2, seed 3), closest-hit, per GPU",
    "c1": "C1 (configs[0]): teapot LSNIF, 256x256 pixel-centre primary rays, closest-hit",
    "c4": "C4 (configs[3]): 8 LSNIF instances (teapot x3, sphere x2, torus x2, box; "
          "per-object hash grids and MLP weights, seeds 0-3) on a 4x2 grid, 1920x1080 camera "
          "rays, brute-force broad phase + per-object narrow phase + closest-hit merge, per GPU",
    "render": "F3 (SURVEY §8(f)): wavefront path tracer over a 4-instance LSNIF scene (teapot with "
              "glossy lid, glossy sphere, box, torus; point + sphere light, environment), "
              "1280x720 x 4 spp, 4 bounces, PrimaryMode::lsnif; rays = intersect_scene + "
              "occluded_batch queries issued by the renderer",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU work per timed baseline measurement")
    ap.add_argument("--rays", type=int, default=0,
                    help="C5 frame size override (tests only; the line then says so)")
    ap.add_argument("--dump", default="",
                    help="(tests) rank 0 saves the gathered C5 frame (wire records) to this .npy")
    ap.add_argument("--dist-backend", default=os.environ.get("LSNIF_DIST_BACKEND", "nccl"),
                    help="nccl (one GPU per rank) or gloo (test mode: all ranks on cuda:0)")
    return ap.parse_args()


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) from a plain `python bench.py`: run the same command
    as N ranks under torch.distributed.run (one process per GPU)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------- workload

def build_rays(workload: str, rank: int, box: np.ndarray, world: int = 1):
    """Primary rays of one rank (C1-C3; C5 is generated straight into pinned memory)."""
    from paper_2504_21627_b200 import workloads as W
    if workload == "c2":
        return W.camera_rays(1920, 1080, jitter=W.rank_jitter(rank))
    if workload == "c1":
        return W.camera_rays(256, 256, jitter=W.rank_jitter(rank))
    out = np.empty(1 << 24, W.RAY_DTYPE)
    return W.incoherent_rays_into(out, box, 3, rank << 24)


def c2_shadow_set(primary: np.ndarray, box):
    """The C2 shadow rays, derived ONCE from the CPU reference's own primary
    hits (the IEEE build of the reference's narrow phase on the whole frame):
    every arm answers exactly the same rays (the GPU's fp16 MLP may accept a
    few different primaries)."""
    from paper_2504_21627_b200 import workloads as W
    hits = parity_model().narrow_phase(primary, 0, 0)
    return W.shadow_rays(primary, hits, box)[0]


def c5_sample(box, total: int = C5_RAYS) -> tuple[np.ndarray, np.ndarray]:
    """The CPU arms' C5 sample: every C5_CPU_STRIDE-th ray of the frame (the
    GPU answers the same rays at the same indices)."""
    from paper_2504_21627_b200 import workloads as W
    idx = np.arange(0, total, C5_CPU_STRIDE, dtype=np.uint64)
    return idx, W.incoherent_rays_at(idx, box, seed=C5_SEED)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured"
        return d
    except Exception:
        return dict(FALLBACK_PEAKS)


def load_json(name: str):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return {}


def aux_rooflines(workload: str, trace_rays_per_s: float, sm_mhz, pts_per_ray: float, vol_per_ray: float):
    """The trace kernel is SIMT-issue bound (SURVEY §8(d) 'auxiliary issue
    ceiling'): warp instructions per ray from the committed ncu capture x the
    live rays/s, against 148 SMs x 4 issue slots x the measured clock; and its
    hash-table gathers (8 per boundary point, 16 per volume point) against the
    measured L2 random 8-byte gather rate (scripts/micro/l2_bw.cu)."""
    km = load_json(f"kernel_metrics_{workload}.json").get("trace_encode_kernel")
    out = {}
    clk = (sm_mhz or 1965.0) * 1e6
    if km:
        ach = km["warp_inst_per_ray"] * trace_rays_per_s
        peak = 148 * 4 * clk
        out["roofline_issue"] = {
            "kernel": "trace_encode_kernel", "bound": "issue", "achieved": ach, "peak": peak,
            "unit": "warp-inst/s", "frac": ach / peak, "ncu_issue_active": km["issue_active_frac"],
            "source": f"profiles/kernel_metrics_{workload}.json ({km['warp_inst_per_ray']:.1f} warp-inst/ray, "
                      "ncu) x live trace rays/s; peak = 148 SMs x 4 schedulers x SM clock"}
    l2 = {}
    try:
        with open(os.path.join(ROOT, "profiles", "micro", "r1s2_l2_bw.jsonl")) as f:
            l2 = json.loads(f.readline())
    except Exception:
        pass
    if l2:
        g = (8.0 * pts_per_ray + 8.0 * vol_per_ray) * trace_rays_per_s
        peak = l2["gather8_Gloads_per_s"] * 1e9
        out["l2_gather"] = {"kernel": "trace_encode_kernel", "achieved": g, "peak": peak, "unit": "gathers/s",
                            "frac": g / peak, "gather_bytes": 8,
                            "source": "8-byte hash-table entry loads per boundary point (2 levels x 4 "
                                      "corners, +8 per volume point) x live rays/s; peak = measured L2 random "
                                      "8-byte gather rate (profiles/micro/r1s2_l2_bw.jsonl)"}
    return out


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML while running."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device: int, period_s: float = 0.005):
        self.samples, self.reasons = [], 0
        self.ok = False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU baseline

def path_roofline(rays_per_s_gpu: float, n: int, rows: int, pts: int, vol: int, mlp_flops: float,
                  peaks: dict, result_bytes: int = 32) -> dict:
    """SURVEY §8(d) whole-path ceiling per GPU: R_tensor = dense fp16 peak /
    FLOP_ray, R_mem = HBM peak / B_ray (B_ray = 32 B ray + the result record
    + 48 B per boundary point + 48 B per volume point), R_path = min of the
    two; the path is issue/latency bound in traversal and encode, so this
    fraction is small by construction (the per-kernel rooflines explain it)."""
    flop_ray = mlp_flops / max(n, 1)
    bytes_ray = 32.0 + result_bytes + 48.0 * (pts + vol) / max(n, 1)
    tflops = peaks.get("bf16_tflops_sustained", 1400.0)
    r_tensor = tflops * 1e12 / max(flop_ray, 1e-9)
    r_mem = peaks["hbm_gbs"] * 1e9 / bytes_ray
    r_path = min(r_tensor, r_mem)
    return {"flop_per_ray": flop_ray, "bytes_per_ray": bytes_ray, "r_tensor": r_tensor, "r_mem": r_mem,
            "r_path": r_path, "achieved": rays_per_s_gpu, "frac": rays_per_s_gpu / r_path,
            "mlp_rows_per_ray": rows / max(n, 1), "unit": "rays/s per GPU"}


def cpu_model() -> str:
    """The host CPU's model name (the reference arm runs on these cores)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_detail(rate: float, cores: int, pairs_per_ray: float, hidden: int, k1: int, n_out: int) -> dict:
    """rays/s per core, the CPU model, and the CPU MLP GFLOP/s.
    The CPU reference runs its MLP (infer_batch, renderer.cpp:193-209) on
    every pair (ray overlapping the frame box), points or not, so the CPU's
    FLOP rate counts pairs x 2 (K1 H + H^2 + H n_out)."""
    flop_row = 2 * (k1 * hidden + hidden * hidden + hidden * n_out)
    return {"per_core": rate / max(cores, 1), "cpu_model": cpu_model(),
            "mlp_gflops": rate * pairs_per_ray * flop_row / 1e9}


def cpu_oracle(fast: bool = True):
    from oracle import oracle as O
    if fast:
        O.build(fast=True)
    return O


class CpuArm:
    """The CPU path both CPU legs time (cpu_baseline and --impl reference):
    the REFERENCE ITSELF when oracle/_ref is built (its own
    PreparedScene::intersect_scene / occluded_batch, renderer.cpp:269-323,
    compiled from /root/reference/proj/src against the Eigen-subset shim with
    the reference's Release flags, called from all host threads on 65,536-ray
    blocks as render() does: kind "reference"), else the oracle's
    restatement of the same narrow phase (kind "port")."""

    def __init__(self, path: str = MODEL_PATH):
        self.kind, self.err = "port", ""
        try:
            from oracle import ref as R
            if not R.available(True):
                raise RuntimeError("oracle/_ref not built")
            self.m = R.RefModel(path, fast=True)
            self.cores = R.hardware_concurrency()
            self.kind = "reference"
            self.what = ("the reference's own PreparedScene::intersect_scene / occluded_batch "
                         "(renderer.cpp:269-323; collect_pairs + run_narrow_phase + infer_batch) compiled "
                         "from /root/reference/proj/src against the Eigen-subset shim (oracle/_ref), "
                         "-O3 -march=native, parallel_slices over 65,536-ray blocks on all host threads")
        except Exception as e:  # the oracle restatement, said so in the line
            self.err = str(e)[:200]
            O = cpu_oracle(True)
            self.m = O.OracleModel.load(path, fast=True)
            self.cores = int(O.lib(True).oracle_hardware_concurrency())
            self.what = ("the oracle's C++ restatement of run_narrow_phase + infer_batch (-O3 -march=native, "
                         "all host threads); oracle/_ref unavailable: " + self.err)

    def run(self, rays, mode: int):
        if self.kind == "reference":
            return self.m.scene_query(rays, mode, 0)
        return self.m.narrow_phase(rays, mode, 0)


def time_cpu_sets(arm: "CpuArm", sets, target_s: float):
    """Times the CPU path (all host threads) over the ray sets [(rays, mode),
    ...] answered back to back: one untimed pass, then repeated passes
    spanning ~target_s of CPU work; the rate is over their total time (the
    mean pass, as the --impl reference arm reports). Returns (rays/s, info)."""
    n = sum(len(r) for r, _ in sets)
    t0 = time.perf_counter()
    for r, mode in sets:
        if len(r):
            arm.run(r, mode)
    one = max(time.perf_counter() - t0, 1e-6)
    reps = max(1, min(200, int(round(target_s / one))))
    t0 = time.perf_counter()
    for _ in range(reps):
        for r, mode in sets:
            if len(r):
                arm.run(r, mode)
    total = (time.perf_counter() - t0) / reps
    return n / total, {"rays": n, "seconds": reps * total, "reps": reps}


def parity_model(path: str = MODEL_PATH):
    """The IEEE (parity) build of the CPU path for spot checks: the reference
    itself (oracle/_ref) when built, else the oracle restatement."""
    try:
        from oracle import ref as R
        if R.available(False):
            return R.RefModel(path)
    except Exception:
        pass
    from oracle import oracle as O
    return O.OracleModel.load(path)


def pairs_fraction(model, rays: np.ndarray) -> float:
    """Fraction of rays that form a pair (CPU MLP rows) on a subsample."""
    sub = rays[:: max(1, len(rays) // 16384)]
    info = model.trace(sub)["info"]
    return float(np.mean((info >> 9) & 1 == 1))


def sample_parity(gpu_hits: np.ndarray, ref_hits: np.ndarray) -> dict:
    """Parity of a GPU result sample against the CPU reference on the same
    rays (SURVEY App. B gates): pair flags bit-exact, visibility / material
    agreement, and for rays both call occluded the t, normal and albedo
    deviations."""
    f_g, f_r = gpu_hits["flags_material"], ref_hits["flags_material"]
    pair = (f_r & 1) == 1
    occ_g, occ_r = (f_g & 2) != 0, (f_r & 2) != 0
    both = pair & occ_g & occ_r
    mat_g, mat_r = f_g >> 8, f_r >> 8
    out = {"rays": int(len(f_r)), "pairs": int(pair.sum()),
           "pair_flags_equal": bool(np.array_equal(f_g & 1, f_r & 1)),
           "visibility_agree": float(np.mean(occ_g[pair] == occ_r[pair])) if pair.any() else 1.0,
           "material_agree": float(np.mean(mat_g[pair] == mat_r[pair])) if pair.any() else 1.0,
           "both_occluded": int(both.sum())}
    if both.any():
        ng, nr = gpu_hits["normal"][both].astype(np.float64), ref_hits["normal"][both].astype(np.float64)
        lg, lr = np.linalg.norm(ng, axis=1), np.linalg.norm(nr, axis=1)
        ok = (lg > 0) & (lr > 0)
        cosv = np.clip(np.sum(ng[ok] * nr[ok], axis=1) / (lg[ok] * lr[ok]), -1, 1)
        out.update({"max_dt_world": float(np.max(np.abs(gpu_hits["t_world"][both] - ref_hits["t_world"][both]))),
                    "max_normal_deg": float(np.degrees(np.max(np.arccos(cosv)))) if ok.any() else 0.0,
                    "max_dalbedo": float(np.max(np.abs(gpu_hits["albedo"][both] - ref_hits["albedo"][both])))})
    return out


# ---------------------------------------------------------------- reference

def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (run_narrow_phase +
    infer_batch, -O3 -march=native, all host threads) on a bounded sample of
    this arm's workload — for C5 and C2 exactly the rays our arm's
    cpu_baseline times (same indices / the same shadow set). Under torchrun
    only rank 0 runs; the other ranks exit without work."""
    if rank != 0:
        return 0
    arm = CpuArm()
    model, cores = arm.m, arm.cores
    box = model.aabb
    if args.workload == "c5":
        _, rays = c5_sample(box, args.rays or C5_RAYS)
        sets = [(rays, 0)]
        sample = (f"every {C5_CPU_STRIDE}th ray of the C5 frame ({len(rays)} rays, the same indices the "
                  f"GPU arm's cpu_baseline times)")
    elif args.workload == "c2":
        prim = build_rays("c2", 0, box)
        shadow = c2_shadow_set(prim, box)
        sets = [(prim, 0), (shadow, 1)]
        sample = (f"the whole C2 frame: {len(prim)} primary rays + {len(shadow)} shadow rays "
                  f"(the shadow set every arm answers)")
    else:
        prim = build_rays(args.workload, 0, box)
        stride = max(1, len(prim) // (1 << 21))
        sets = [(prim[::stride], 0)]
        sample = f"every {stride}th ray of the {args.workload.upper()} set ({len(sets[0][0])} rays)"
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for r, mode in sets:
            arm.run(r, mode)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    n = sum(len(r) for r, _ in sets)
    total = sum(times)
    value = n * len(times) / total
    pf = pairs_fraction(model, np.concatenate([r for r, _ in sets]))
    ref_detail = cpu_detail(value, cores, pf, model.hidden, model.input_width, 8 + model.n_mat)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload], "rays_per_step": n,
                   "parallelism": "host threads (parallel_slices)"},
        "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": cores, "kind": arm.kind,
                              "sample": sample, "what": arm.what}, **ref_detail),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- C4 scene

def run_c4(args, rank, world, dev, gpu, max_over_ranks):
    import torch
    from paper_2504_21627_b200 import lsnif, workloads as W
    gold = os.path.join(ROOT, "tests", "golden")
    models = [lsnif.GpuModel(os.path.join(gold, n + ".lsnif"), gpu) for n in W.C4_MODELS]
    w2o = W.c4_world_to_object()
    scene = lsnif.GpuScene([(models[k], w2o[i]) for i, k in enumerate(W.C4_INSTANCES)])
    rays = W.camera_rays(1920, 1080, camera=W.C4_CAMERA, jitter=W.rank_jitter(rank))
    d_rays = lsnif.rays_to_tensor(rays, dev)
    out = torch.empty((len(rays), 16), dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        scene.query(d_rays, lsnif.CLOSEST, out=out)
    torch.cuda.synchronize()
    for m in models:
        m.profile_read(reset=True, stream="all")
    clocks = ClockSampler(gpu)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks.start()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record()
        scene.query(d_rays, lsnif.CLOSEST, out=out)
        ev[k][1].record()
    torch.cuda.synchronize()
    clocks.stop()
    launches = sum(int(m.profile_read(reset=True, stream="all")["launches"]) for m in models)
    for m in models:  # per-kernel breakdown: a separate profiled pass
        m.profile_enable(True)
    for k in range(args.steps):
        flush.zero_()
        scene.query(d_rays, lsnif.CLOSEST, out=out)
    torch.cuda.synchronize()
    profs = []
    for m in models:
        m.profile_enable(False)
        profs.append(m.profile_read(reset=True, stream="all"))
    elapsed_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    value = world * len(rays) * args.steps / (elapsed_ms / 1e3)
    hits = lsnif.scene_hits_to_numpy(out)

    # ---- e2e: same step through lsnif_scene_query_host (pinned host buffers)
    pin_r = torch.from_numpy(rays.view(np.float32).reshape(-1, 8).copy()).pin_memory()
    pin_h = torch.empty((len(rays), 16), dtype=torch.int32).pin_memory()
    scene.query_host(pin_r, lsnif.CLOSEST, out=pin_h)
    e2e_steps = max(5, min(args.steps, 15))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    per_step = []  # median host-clock step, max over ranks (as the single-model line)
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        scene.query_host(pin_r, lsnif.CLOSEST, out=pin_h)
        per_step.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(float(np.median(per_step))) * e2e_steps
    assert np.array_equal(pin_h.numpy(), out.cpu().numpy()), "host/device scene results differ"
    if rank == 0:
        tr = sum(p["trace_ms"] for p in profs) / args.steps
        ml = sum(p["mlp_ms"] for p in profs) / args.steps
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32 traversal/encode + f16xf16->f32 tcgen05 MLP", "data": "synthetic",
                "config": {"workload": WORKLOADS["c4"], "rays_per_step_per_gpu": len(rays),
                           "l2": "flushed between timed steps (256 MiB write outside the events)",
                           "parallelism": f"dp{world} (one frame per GPU)"},
                "workload_stats": {"frac_hit": float(np.mean(hits["flags"] == 1))},
                "kernels": {"trace_encode_kernel": {"ms_per_step": tr},
                            "mlp_tc_kernel": {"ms_per_step": ml}},
                "e2e": {"value": world * len(rays) * e2e_steps / e2e_s, "unit": UNIT,
                        "h2d_bytes_per_step": 32 * len(rays), "d2h_bytes_per_step": 64 * len(rays),
                        "steps": e2e_steps,
                        "api": "lsnif_scene_query_host (pinned host rays/scene hits, chunked H2D/query/D2H)"},
                "gpu_launches": launches,
                "clocks": clocks.summary()}
        if world == 1 and not args.no_cpu_baseline:
            try:
                O = cpu_oracle(True)
                om = [O.OracleModel.load(os.path.join(gold, n + ".lsnif"), fast=True) for n in W.C4_MODELS]
                om = [om[k] for k in W.C4_INSTANCES]
                probe = rays[:: max(1, len(rays) // 8192)]
                t0 = time.perf_counter()
                O.scene_query(om, w2o, probe, 0, 0)
                rate = len(probe) / max(time.perf_counter() - t0, 1e-6)
                stride = max(1, int(len(rays) / max(rate * args.cpu_seconds, 1.0)))
                sample = rays[::stride]
                # whole frame shorter than the target: repeat it (best of nothing, total time)
                reps = max(1, int(round(args.cpu_seconds * rate / len(sample))))
                t0 = time.perf_counter()
                for _ in range(reps):
                    O.scene_query(om, w2o, sample, 0, 0)
                dt = (time.perf_counter() - t0) / reps
                line["cpu_baseline"] = {
                    "value": len(sample) / dt, "unit": UNIT,
                    "cores": int(O.lib(True).oracle_hardware_concurrency()), "kind": "port",
                    "sample": f"every {stride}th C4 camera ray ({len(sample)} rays) x {reps} passes, oracle "
                              f"scene_query (collect_pairs + per-object narrow phase + merge), "
                              f"{reps * dt:.1f} s"}
            except Exception as e:  # the baseline is reported, never the target
                line["cpu_baseline"] = {"unavailable": str(e)[:200]}
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------- F3 renderer

RENDER_CFG = dict(width=1280, height=720, spp=4, max_bounces=4, seed=1, neural_eps_scale=1e-3)


def render_scene_paths(tmpdir: str):
    from paper_2504_21627_b200 import workloads as W
    gold = os.path.join(ROOT, "tests", "golden")
    paths = [os.path.join(gold, n + ".lsnif") for n in W.RENDER_MODELS]
    paths[0] = W.glossy_copy(paths[0], os.path.join(tmpdir, "teapot_glossy.lsnif"), 1, 0.3)
    paths[1] = W.glossy_copy(paths[1], os.path.join(tmpdir, "sphere_glossy.lsnif"), 0, 0.2)
    return paths


def run_render(args, rank, world, dev, gpu, max_over_ranks):
    """One step = one full render (camera rays, 4 bounces, NEE shadow rays)
    through lsnif_render; value = renderer ray queries per second."""
    import tempfile
    import torch
    from paper_2504_21627_b200 import lsnif, workloads as W
    tmp = tempfile.mkdtemp(prefix="lsnif_render_")
    paths = render_scene_paths(tmp)
    models = [lsnif.GpuModel(p, gpu) for p in paths]
    w2o = W.render_world_to_object()
    scene = lsnif.GpuScene([(models[i], w2o[i]) for i in range(len(models))])
    diag = W.world_diag_from_frames([m.aabb for m in models])
    cfg = dict(RENDER_CFG, seed=RENDER_CFG["seed"] + rank)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    st = {}
    for _ in range(args.warmup):
        img = scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag, stats=st)
    torch.cuda.synchronize()
    for m in models:
        m.profile_read(reset=True, stream="all")
    clocks = ClockSampler(gpu)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.zero_()
        ev[k][0].record()
        img = scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag, stats=st)
        ev[k][1].record()
    torch.cuda.synchronize()
    clocks.stop()
    launches = sum(int(m.profile_read(reset=True, stream="all")["launches"]) for m in models)
    for m in models:  # per-kernel breakdown: a separate profiled pass
        m.profile_enable(True)
    for k in range(args.steps):
        flush.zero_()
        scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag)
    torch.cuda.synchronize()
    profs = []
    for m in models:
        m.profile_enable(False)
        profs.append(m.profile_read(reset=True, stream="all"))
    elapsed_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    rays = st["closest_rays"] + st["shadow_rays"]
    value = world * rays * args.steps / (elapsed_ms / 1e3)
    # e2e: the same render through the public API + the image read back to the host
    host = torch.empty(img.shape, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 7))
    per_step = []  # median host-clock step, max over ranks
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        img = scene.render(W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, cfg, diag)
        host.copy_(img)
        per_step.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(float(np.median(per_step))) * e2e_steps
    if rank != 0:
        return
    tr = sum(p["trace_ms"] for p in profs) / args.steps
    ml = sum(p["mlp_ms"] for p in profs) / args.steps
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 traversal/encode/shading + f16xf16->f32 tcgen05 MLP", "data": "synthetic",
            "config": {"workload": WORKLOADS["render"], "render": cfg,
                       "l2": "flushed between timed steps (256 MiB write outside the events)",
                       "parallelism": f"dp{world} (one frame per GPU)"},
            "workload_stats": {k: int(v) for k, v in st.items()},
            "kernels": {"trace_encode_kernel": {"ms_per_step": tr},
                        "mlp_tc_kernel": {"ms_per_step": ml}},
            "e2e": {"value": world * rays * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": int(img.numel() * 4), "steps": e2e_steps,
                    "api": "lsnif_render + image D2H (inputs are the scene / camera description)"},
            "gpu_launches": launches,
            "clocks": clocks.summary()}
    if world == 1 and not args.no_cpu_baseline:
        try:
            O = cpu_oracle(True)
            om = [O.OracleModel.load(p, fast=True) for p in paths]
            small = dict(cfg, width=320, height=180)
            ost = {}
            O.render(om, w2o, W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, dict(small, height=18),
                     diag, workers=0)  # warm-up
            t0 = time.perf_counter()
            O.render(om, w2o, W.RENDER_CAMERA, W.RENDER_LIGHTS, W.RENDER_ENV, small, diag, workers=0,
                     stats=ost)
            dt = time.perf_counter() - t0
            cores = int(O.lib(True).oracle_hardware_concurrency())
            line["cpu_baseline"] = {
                "value": (ost["closest_rays"] + ost["shadow_rays"]) / dt, "unit": UNIT, "cores": cores,
                "kind": "port",
                "sample": f"the same scene/config at 320x180 ({ost['closest_rays']} + "
                          f"{ost['shadow_rays']} rays, {dt:.1f} s, oracle render restatement)"}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- ours

class Ctx:
    """Rank / device / collective plumbing shared by the workload runners."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.args = args
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.gloo = args.dist_backend == "gloo"
        if self.world > 1 and not self.gloo:
            # leave SMs to NCCL: the persistent query kernels fill every SM they
            # are given, so the result gather's kernels (side stream) would wait
            # for each piece's query to finish instead of overlapping the next
            # one (lsnif_dev::reserved_sms; read once by the library)
            os.environ.setdefault("LSNIF_RESERVE_SMS", "8")
        self.gpu = 0 if self.gloo else self.local_rank
        torch.cuda.set_device(self.gpu)
        self.dev = torch.device("cuda", self.gpu)
        if self.world > 1:
            if self.gloo:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
        self.coll_dev = torch.device("cpu") if self.gloo else self.dev

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=self.coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, xs):
        if self.world == 1:
            return list(xs)
        import torch
        import torch.distributed as dist
        t = torch.tensor(list(xs), dtype=torch.float64, device=self.coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return [float(v) for v in t.tolist()]

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


def timed_steps(ctx, step, steps: int, warmup: int, flush, model=None):
    """W untimed steps, then K steps each bracketed by CUDA events on the
    launching stream (L2 flushed outside the events), barrier + synchronize
    on both sides, clocks sampled during the timed region. Returns
    (max-over-ranks device ms of the K steps, clock summary, launches)."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if model is not None:
        model.profile_read(reset=True, stream="all")
    clocks = ClockSampler(ctx.gpu)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    clocks.start()
    ctx.barrier()
    torch.cuda.synchronize()
    for k in range(steps):
        flush.zero_()
        ev[k][0].record()
        step()
        ev[k][1].record()
    torch.cuda.synchronize()
    ctx.barrier()
    clocks.stop()
    launches = model.profile_read(reset=True, stream="all")["launches"] if model is not None else 0
    elapsed = ctx.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev))
    return elapsed, clocks.summary(), launches


def kernel_breakdown(model, step, steps: int, flush):
    """Per-kernel device time of the same step in a separate profiled pass
    (the library's per-launch CUDA events are not part of the timed steps)."""
    import torch
    model.profile_read(reset=True, stream="all")
    model.profile_enable(True)
    for _ in range(steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    model.profile_enable(False)
    return model.profile_read(reset=True, stream="all")


def kernel_roofline(model, prof, steps: int, n_rays: int, rows: int, pts: int, vol: int, result_bytes: int,
                    peaks: dict, tag: str) -> tuple[dict, dict, float]:
    """`roofline` of the dominant kernel (SURVEY §8(d) per-unit figures x the
    units one launch processes ÷ its average launch time) + the kernels map."""
    tr_ms = prof["trace_ms"] / steps
    ml_ms = prof["mlp_ms"] / steps
    hid = model.info.hidden
    mlp_flops = 2 * rows * (model.input_width * hid + hid * hid + hid * (8 + model.info.n_mat))
    # trace_encode_kernel: rays in (32 B), results of rays without MLP rows,
    # 48 B of hash-table entries per boundary / volume point
    trace_bytes = 32 * n_rays + result_bytes * (n_rays - rows) + 48 * pts + 48 * vol
    traffic = load_json(f"traffic_{tag}.json")  # ncu DRAM bytes per launch (profiles/)
    if tr_ms >= ml_ms:
        launches = max(1, prof["trace_launches"] // steps)
        ach = trace_bytes / (tr_ms / 1e3) / 1e9
        roof = {"kernel": "trace_encode_kernel", "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": traffic.get("trace_encode_kernel"),
                "algorithmic_bytes_per_launch": trace_bytes / launches, "launches_per_step": launches,
                "peak_source": peaks["source"]}
    else:
        launches = max(1, prof["mlp_launches"] // steps)
        ach = mlp_flops / (ml_ms / 1e3) / 1e12
        pk = peaks.get("bf16_tflops", peaks.get("bf16_tflops_sustained", 1400.0))
        roof = {"kernel": "mlp_tc_kernel", "bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                "frac": ach / pk, "traffic": traffic.get("mlp_tc_kernel"), "peak_source": peaks["source"]}
    kernels = {"trace_encode_kernel": {"ms_per_step": tr_ms, "launches": prof["trace_launches"],
                                       "GBps_algorithmic": trace_bytes / (tr_ms / 1e3) / 1e9 if tr_ms else None},
               "mlp_tc_kernel": {"ms_per_step": ml_ms, "launches": prof["mlp_launches"],
                                 "tflops": mlp_flops / (ml_ms / 1e3) / 1e12 if ml_ms > 0 else None,
                                 "frac_of_burst_peak": (mlp_flops / (ml_ms / 1e3) / 1e12) /
                                 peaks.get("bf16_tflops", 1614.9) if ml_ms > 0 else None}}
    return roof, kernels, mlp_flops


def copy_only_seconds(pin_rays, host_frame, off: int, n: int, chunk: int = 1 << 21, slots: int = 4) -> float:
    """The e2e path's PCIe ceiling: lsnif_query_host_wire's copy schedule
    (chunked H2D of 32 B rays, D2H of 16 B results, one stream per slot)
    without the kernels; best of 2 frames, device-timed."""
    import torch
    src = pin_rays.view(torch.uint8).reshape(-1)[: n * 32]
    dst = host_frame.view(torch.uint8).reshape(-1)[off * 16:(off + n) * 16]
    d_in = [torch.empty(chunk * 32, dtype=torch.uint8, device="cuda") for _ in range(slots)]
    d_out = [torch.empty(chunk * 16, dtype=torch.uint8, device="cuda") for _ in range(slots)]
    streams = [torch.cuda.Stream() for _ in range(slots)]
    cur = torch.cuda.current_stream()
    best = float("inf")
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for s_ in streams:
            s_.wait_stream(cur)
        for i, s0 in enumerate(range(0, n, chunk)):
            c = min(chunk, n - s0)
            k = i % slots
            with torch.cuda.stream(streams[k]):
                d_in[k][: c * 32].copy_(src[s0 * 32:(s0 + c) * 32], non_blocking=True)
                dst[s0 * 16:(s0 + c) * 16].copy_(d_out[k][: c * 16], non_blocking=True)
        for s_ in streams:
            cur.wait_stream(s_)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    del d_in, d_out
    return best


def run_c5(args, ctx) -> None:
    """C5: one 132.7M-ray frame split into row bands (one per rank); see the
    module docstring."""
    import torch
    import torch.distributed as dist
    from paper_2504_21627_b200 import lsnif, workloads as W
    from paper_2504_21627_b200.dist import gather_piece_to_rank0, piece_range, ray_range
    rank, world = ctx.rank, ctx.world
    total = args.rays or C5_RAYS
    bands = [ray_range(total, world, r) for r in range(world)]
    sizes = [e - s for s, e in bands]
    s0, band = bands[rank][0], sizes[rank]
    model = lsnif.GpuModel(MODEL_PATH, ctx.gpu)
    box = model.aabb
    # the rank's rays, regenerated from the index-addressable generator into
    # pinned host memory (the e2e input) and copied once to the device
    pin_rays = torch.empty((band, 8), dtype=torch.float32, pin_memory=True)
    W.incoherent_rays_into(pin_rays.numpy(), box, C5_SEED, s0)
    d_rays = pin_rays.to(ctx.dev)
    pieces = C5_PIECES if world > 1 else 1
    d_frame = torch.empty((total, 4), dtype=torch.int32, device=ctx.dev) if rank == 0 else None
    local = d_frame[:band] if rank == 0 else torch.empty((band, 4), dtype=torch.int32, device=ctx.dev)
    comm = torch.cuda.Stream(ctx.dev) if world > 1 and not ctx.gloo else None
    cpu_frame = torch.empty((total, 4), dtype=torch.int32) if ctx.gloo and rank == 0 else None
    pev = [torch.cuda.Event() for _ in range(pieces)]

    def step():
        works = []
        for k in range(pieces):
            ps, pe = piece_range(band, pieces, k)
            model.query_wire(d_rays[ps:pe], lsnif.CLOSEST, out=local[ps:pe])
            if world == 1:
                continue
            if ctx.gloo:  # test mode: every rank on cuda:0, the gather through host tensors
                piece = local[ps:pe].cpu()
                if rank == 0:
                    cpu_frame[ps:pe].copy_(piece)
                for w in gather_piece_to_rank0(piece, k, pieces, sizes, out=cpu_frame):
                    w.wait()
            else:  # piece k goes to rank 0 on the comm stream while piece k + 1 computes
                pev[k].record()
                with torch.cuda.stream(comm):
                    comm.wait_event(pev[k])
                    works += gather_piece_to_rank0(local[ps:pe], k, pieces, sizes, out=d_frame)
        if world > 1 and not ctx.gloo:
            with torch.cuda.stream(comm):
                for w in works:
                    w.wait()
            torch.cuda.current_stream().wait_stream(comm)
        if ctx.gloo and rank == 0:
            d_frame.copy_(cpu_frame)

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=ctx.dev)
    step()  # warm (NCCL connection setup, staging, launch configuration)
    torch.cuda.synchronize()
    # per-band query statistics (pairs, MLP rows, points) for the rooflines
    st = np.zeros(4)
    for k in range(pieces):
        ps, pe = piece_range(band, pieces, k)
        model.query_wire(d_rays[ps:pe], lsnif.CLOSEST, out=local[ps:pe])
        s = model.last_stats()
        st += [s["pairs"], s["mlp_rows"], s["points"], s["volume_points"]]
    pairs, rows, pts, vol = [int(v) for v in st]
    elapsed_ms, clocks, launches = timed_steps(ctx, step, args.steps, max(args.warmup - 1, 0), flush, model)
    prof = kernel_breakdown(model, step, args.steps, flush)
    value = total * args.steps / (elapsed_ms / 1e3)
    tot_stats = ctx.sum_over_ranks([pairs, rows, pts, vol])

    # ---- e2e: lsnif_query_host_wire from pinned host rays; every rank's band
    # lands in one full-frame host buffer (shared memory on this node, pinned)
    lib = lsnif.load_library()
    host_frame, host_note, shm_path = None, "", None
    if world == 1:
        host_frame = torch.empty((total, 4), dtype=torch.int32, pin_memory=True)
        host_note = "pinned host frame"
    else:
        tag = os.environ.get("MASTER_PORT", "0")
        shm_path = f"/dev/shm/lsnif_c5_{tag}.frame"
        need = total * 16
        ok = 1.0
        try:
            sv = os.statvfs("/dev/shm")
            ok = 1.0 if sv.f_bavail * sv.f_frsize > need * 1.05 else 0.0
        except OSError:
            ok = 0.0
        ok = -ctx.max_over_ranks(-ok)  # min over ranks
        if ok > 0:
            if rank == 0:
                with open(shm_path, "wb") as f:
                    f.truncate(need)
            ctx.barrier()
            mm = np.memmap(shm_path, dtype=np.int32, mode="r+", shape=(total, 4))
            host_frame = torch.from_numpy(np.asarray(mm))
            rc = torch._C._cudart.cudaHostRegister(host_frame.data_ptr(), need, 0)
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister of the shared host frame failed ({rc})")
            ctx.barrier()
            if rank == 0:
                os.unlink(shm_path)
            host_note = "one full-frame host buffer shared by the ranks (/dev/shm, cudaHostRegister-ed)"
        else:
            host_frame = torch.empty((band, 4), dtype=torch.int32, pin_memory=True)
            host_note = "per-rank pinned band buffers (/dev/shm too small for a shared frame)"
    off = s0 if host_frame.shape[0] == total else 0

    def e2e_step():
        lsnif._check(lib.lsnif_query_host_wire(model.h, pin_rays.data_ptr(), band, lsnif.CLOSEST,
                                               host_frame.data_ptr() + 16 * off, None))

    e2e_step()
    e2e_steps = max(3, min(args.steps, 6))
    per_step = []
    for _ in range(e2e_steps):
        ctx.barrier()
        t0 = time.perf_counter()
        e2e_step()
        ctx.barrier()  # the frame is complete when every band has landed
        per_step.append(time.perf_counter() - t0)
    e2e_s = ctx.max_over_ranks(float(np.median(per_step)))
    e2e_value = total / e2e_s
    # bit-identical frames: host API path vs the device path (+ NCCL gather)
    same = True
    if rank == 0:
        d_host = d_frame.cpu()
        same = bool(torch.equal(host_frame[:band], d_host[:band])) if host_frame.shape[0] != total else \
            bool(torch.equal(host_frame, d_host))
        assert same, "host-API frame differs from the device frame"
        if args.dump:
            np.save(args.dump, d_host.numpy())
    ctx.barrier()
    # the PCIe ceiling of the same host path (overwrites the host frame)
    ceil_s = ctx.max_over_ranks(copy_only_seconds(pin_rays, host_frame, off, band))

    if rank == 0:
        peaks = load_peaks()
        roof, kernels, mlp_flops = kernel_roofline(model, prof, args.steps, band, rows, pts, vol, 16, peaks, "c5")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 traversal/encode + f16xf16->f32 tcgen05 MLP", "data": "synthetic",
            "config": {"workload": WORKLOADS["c5"] if total == C5_RAYS else
                       WORKLOADS["c5"] + f" [TEST SIZE: {total} rays]",
                       "rays_per_step": total, "rays_per_gpu": sizes, "pieces_per_band": pieces,
                       "query_sms_left_to_the_gather": int(os.environ.get("LSNIF_RESERVE_SMS", "0")),
                       "result_record_bytes": 16,
                       "l2": "inputs (4.25 GB of rays) far larger than L2; also flushed between timed steps "
                             "(256 MiB write outside the events)",
                       "parallelism": f"dp{world} (row bands of one frame" +
                                      (", pieces gathered point-to-point to rank 0 over NCCL, overlapped "
                                       "with compute)" if world > 1 else ")")},
            "workload_stats": {"frac_hit_aabb": tot_stats[0] / total, "frac_ge1_point": tot_stats[1] / total,
                               "mean_points": tot_stats[2] / total, "volume_points": int(tot_stats[3])},
            "roofline": roof,
            "path_roofline": path_roofline(value / world, band, rows, pts, vol, mlp_flops, peaks, 16),
            "kernels": kernels,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 32 * total,
                    "d2h_bytes_per_step": 16 * total, "steps": e2e_steps,
                    "timing": "median step (host clock, barriers on both sides), max over ranks",
                    "step_ms_min_median_max": [1e3 * min(per_step), 1e3 * float(np.median(per_step)),
                                               1e3 * max(per_step)],
                    "api": "lsnif_query_host_wire per rank (pinned host rays -> chunked H2D / query / D2H of "
                           "16 B wire results) into " + host_note,
                    "bit_identical_to_device_frame": same,
                    "copy_only_ceiling": {"value": total / ceil_s, "unit": UNIT, "frac": e2e_value * ceil_s / total,
                                          "how": "the same chunked H2D (2^21 rays) / D2H schedule over 4 stream "
                                                 "slots with no kernels, best of 2, max over ranks"}},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        line.update(aux_rooflines("c5", band / (kernels["trace_encode_kernel"]["ms_per_step"] / 1e3)
                                  if kernels["trace_encode_kernel"]["ms_per_step"] else 0.0,
                                  clocks.get("sm_mhz"), pts / band, vol / band))
        if world == 1 and not args.no_cpu_baseline:
            try:
                arm = CpuArm()
                idx, srays = c5_sample(box, total)
                rate, info = time_cpu_sets(arm, [(srays, 0)], args.cpu_seconds)
                line["cpu_baseline"] = {
                    "value": rate, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
                    "sample": f"every {C5_CPU_STRIDE}th ray of the C5 frame ({info['rays']} rays, the "
                              f"reference arm's rays), mean of {info['reps']} passes (~{info['seconds']:.1f} s "
                              f"of CPU work)", "what": arm.what}
                line["cpu_baseline"].update(cpu_detail(rate, arm.cores, pairs_fraction(arm.m, srays),
                                                       model.info.hidden, model.input_width, 8 + model.info.n_mat))
                # the sample doubles as a parity spot check of the timed frame
                # against the IEEE (parity) build of the same CPU path
                gpu = lsnif.wire_to_hits(d_frame.cpu().numpy()[idx.astype(np.int64)])
                line["sample_parity"] = sample_parity(gpu, parity_model().narrow_phase(srays, 0, 0))
            except Exception as e:  # reported, never silently substituted
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)
    if host_frame is not None and world > 1 and host_frame.shape[0] == total:
        torch._C._cudart.cudaHostUnregister(host_frame.data_ptr())


def run_single(args, ctx) -> None:
    """C1 / C2 / C3: one frame per rank (weak scaling, no data-path collective)."""
    import torch
    from paper_2504_21627_b200 import lsnif
    rank, world = ctx.rank, ctx.world
    model = lsnif.GpuModel(MODEL_PATH, ctx.gpu)
    box = model.aabb
    primary = build_rays(args.workload, rank, box, world)
    shadow = c2_shadow_set(primary, box) if args.workload == "c2" else primary[:0]
    d_primary = lsnif.rays_to_tensor(primary, ctx.dev)
    d_hits_p = torch.empty((len(primary), 8), dtype=torch.int32, device=ctx.dev)
    d_shadow = lsnif.rays_to_tensor(shadow, ctx.dev) if len(shadow) else None
    d_hits_s = torch.empty((len(shadow), 8), dtype=torch.int32, device=ctx.dev)
    st = np.zeros(4)
    for rays, hits, mode in ((d_primary, d_hits_p, lsnif.CLOSEST), (d_shadow, d_hits_s, lsnif.ANY)):
        if rays is not None:
            model.query(rays, mode, out=hits)
            s = model.last_stats()
            st += [s["pairs"], s["mlp_rows"], s["points"], s["volume_points"]]
    pairs, rows, pts, vol = [int(v) for v in st]
    n_step = len(primary) + len(shadow)

    def step():
        model.query(d_primary, lsnif.CLOSEST, out=d_hits_p)
        if d_shadow is not None:
            model.query(d_shadow, lsnif.ANY, out=d_hits_s)

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=ctx.dev)
    elapsed_ms, clocks, launches = timed_steps(ctx, step, args.steps, args.warmup, flush, model)
    prof = kernel_breakdown(model, step, args.steps, flush)
    value = world * n_step * args.steps / (elapsed_ms / 1e3)

    # ---- e2e: the same step through the host C-ABI entry (pinned buffers,
    # 16 B wire results)
    pin_p = torch.from_numpy(primary.view(np.float32).reshape(-1, 8).copy()).pin_memory()
    hp = torch.empty((len(primary), 4), dtype=torch.int32).pin_memory()
    pin_s = torch.from_numpy(shadow.view(np.float32).reshape(-1, 8).copy()).pin_memory() if len(shadow) else None
    hs = torch.empty((max(len(shadow), 1), 4), dtype=torch.int32).pin_memory()
    lib = lsnif.load_library()

    def e2e_step():
        lsnif._check(lib.lsnif_query_host_wire(model.h, pin_p.data_ptr(), len(primary), lsnif.CLOSEST,
                                               hp.data_ptr(), None))
        if pin_s is not None:
            lsnif._check(lib.lsnif_query_host_wire(model.h, pin_s.data_ptr(), len(shadow), lsnif.ANY,
                                                   hs.data_ptr(), None))

    e2e_step()
    e2e_steps = max(5, min(args.steps, 15))
    ctx.barrier()
    torch.cuda.synchronize()
    per_step = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        e2e_step()
        per_step.append(time.perf_counter() - t0)
    e2e_s = ctx.max_over_ranks(float(np.median(per_step)))
    e2e_value = world * n_step / e2e_s
    # wire results carry the parity record's flags, material and t bit for bit
    dp = lsnif.hits_to_numpy(d_hits_p)
    wp = hp.numpy().view(lsnif.WIRE_DTYPE).reshape(-1)
    assert np.array_equal(wp["flags_material"], dp["flags_material"]) and \
        np.array_equal(wp["t_world"].view(np.uint32), dp["t_world"].view(np.uint32)), "wire/device results differ"

    if rank == 0:
        peaks = load_peaks()
        roof, kernels, mlp_flops = kernel_roofline(model, prof, args.steps, n_step, rows, pts, vol, 32, peaks,
                                                   args.workload)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 traversal/encode + f16xf16->f32 tcgen05 MLP", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload], "rays_per_step_per_gpu": n_step,
                       "primary_rays": len(primary), "shadow_rays": len(shadow),
                       "l2": "flushed between timed steps (256 MiB write outside the events)",
                       "parallelism": f"dp{world} (one frame per GPU, no data-path collective)"},
            "workload_stats": {"frac_hit_aabb": pairs / n_step, "frac_ge1_point": rows / n_step,
                               "mean_points": pts / n_step, "volume_points": vol},
            "roofline": roof,
            "path_roofline": path_roofline(value / world, n_step, rows, pts, vol, mlp_flops, peaks, 32),
            "kernels": kernels,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 32 * n_step,
                    "d2h_bytes_per_step": 16 * n_step, "steps": e2e_steps,
                    "timing": "median step, max over ranks",
                    "step_ms_min_median_max": [1e3 * min(per_step), 1e3 * float(np.median(per_step)),
                                               1e3 * max(per_step)],
                    "api": "lsnif_query_host_wire (pinned host rays -> 16 B wire results, chunked H2D/query/D2H)"},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        line.update(aux_rooflines(args.workload, n_step / (kernels["trace_encode_kernel"]["ms_per_step"] / 1e3)
                                  if kernels["trace_encode_kernel"]["ms_per_step"] else 0.0,
                                  clocks.get("sm_mhz"), pts / n_step, vol / n_step))
        if world == 1 and not args.no_cpu_baseline:
            try:
                arm = CpuArm()
                if args.workload == "c3":
                    sets = [(primary[::8], 0)]
                    smp = f"every 8th C3 ray ({len(sets[0][0])} rays)"
                else:
                    sets = [(primary, 0), (shadow, 1)]
                    smp = f"the whole frame: {len(primary)} primary + {len(shadow)} shadow rays"
                rate, info = time_cpu_sets(arm, sets, args.cpu_seconds)
                line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": arm.cores, "kind": arm.kind,
                                        "sample": f"{smp}, mean of {info['reps']} passes "
                                                  f"(~{info['seconds']:.1f} s of CPU work)", "what": arm.what}
                line["cpu_baseline"].update(cpu_detail(rate, arm.cores,
                                                       pairs_fraction(arm.m, np.concatenate([r for r, _ in sets])),
                                                       model.info.hidden, model.input_width, 8 + model.info.n_mat))
            except Exception as e:
                line["cpu_baseline"] = {"value": None, "error": str(e)}
        print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        return relaunch_under_torchrun(args)
    if world_env is not None and int(world_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}", file=sys.stderr)
        return 2
    rank = int(os.environ.get("RANK", "0"))
    world = int(world_env or "1")
    if args.impl == "reference":
        return run_reference(args, rank, world)
    ctx = Ctx(args)
    if args.workload == "c5":
        run_c5(args, ctx)
    elif args.workload in ("c4", "render"):
        (run_c4 if args.workload == "c4" else run_render)(args, ctx.rank, ctx.world, ctx.dev, ctx.gpu,
                                                          ctx.max_over_ranks)
    else:
        run_single(args, ctx)
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
