"""CPU: bench.py's host-side contract — the algorithmic-bytes figure behind
roofline.achieved and the reference arm (`--impl
reference`: the reference's own decentralized_cd_detect from oracle/_ref on the
host cores, printing the driver's JSON line)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_algorithmic_bytes_per_problem():
    # (B_c*U + B_c + U) * bytes-per-complex: 4480 B fp32 / 2240 B fp16 at the target
    assert bench.alg_bytes_per_problem(32, 16, 8) == 4480
    assert bench.alg_bytes_per_problem(32, 16, 4) == 2240
    assert bench.alg_bytes_per_problem(32, 8, 8) == (256 + 32 + 8) * 8


def test_clock_sampler_without_samples_reports_why():
    s = bench.ClockSampler(0)
    assert s.summary()["reasons"] == ["nvidia-smi unavailable"]


def _ref_built():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libdcdref.so"))


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref (the reference built from source) is not built")
def test_reference_arm_prints_the_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--cpu-seconds", "1"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == "Gbps" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["steps"] == 1 and line["warmup"] == 3
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["B"] == 256 and line["config"]["U"] == 16 and line["config"]["C"] == 8


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref (the reference built from source) is not built")
def test_gpus_flag_relaunches_one_rank_per_gpu():
    # `bench.py --gpus 2` outside torchrun re-executes itself under
    # torch.distributed.run with 2 ranks; the reference arm prints from rank 0 only
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "3", "--cpu-seconds", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--no-cpu"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode != 0
    assert "WORLD_SIZE=3" in out.stderr
