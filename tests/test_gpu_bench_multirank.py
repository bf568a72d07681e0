"""The bench's C5 multi-rank path on the GPU: two ranks on
one device (gloo for the host-side collectives, the same band / piece /
gather-to-rank-0 code as the NCCL run), and, when >= 2 GPUs are visible,
two ranks over NCCL. The gathered frame must be bit-identical to the
single-rank frame (the output does not depend on the number of GPUs,
reference determinism contract renderer.hpp:133-135)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RAYS = 3_000_017  # several staging chunks, ragged bands and pieces


def _run(tmp_path, world, backend, tag):
    dump = str(tmp_path / f"frame_{tag}.npy")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c5", "--rays", str(RAYS),
           "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--dump", dump, "--gpus", str(world),
           "--dist-backend", backend]
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return lines[0], np.load(dump)


@pytest.fixture(scope="module")
def single(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _run(tmp_path_factory.mktemp("c5"), 1, "nccl", "n1")


def test_c5_single_rank_line(single):
    line, frame = single
    assert line["n_gpus"] == 1 and line["config"]["rays_per_step"] == RAYS
    assert frame.shape == (RAYS, 4)
    assert line["e2e"]["bit_identical_to_device_frame"]
    assert line["gpu_launches"] > 0 and line["roofline"]["frac"] > 0


def test_c5_two_ranks_one_gpu_bit_identical(single, tmp_path):
    line, frame = _run(tmp_path, 2, "gloo", "gloo2")
    assert line["n_gpus"] == 2
    assert np.array_equal(frame, single[1])


def test_c5_two_gpus_nccl_bit_identical(single, tmp_path):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    line, frame = _run(tmp_path, 2, "nccl", "nccl2")
    assert np.array_equal(frame, single[1])
