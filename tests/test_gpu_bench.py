"""SURVEY §8e on one GPU: bench.py's N>1 path (one process per rank, partials
all-gathered, max-over-ranks timing, weak scaling) run as 2 ranks sharing the
visible B200 over gloo (TAILOR_BENCH_SHARE_GPU=1); the collectives are the
same calls the NCCL run makes. Checks the JSON line contract and that every
rank's device selection equals the host's."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run_bench(nproc, *args, timeout=900):
    env = dict(os.environ, TAILOR_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29533", str(ROOT / "bench.py"), "--gpus", str(nproc), *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return lines[0]


def test_bench_two_ranks_merge_step():
    need_gpu()
    line = run_bench(2, "--workload", "cfg2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["steps"] == 3
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["config"]["device_selection_matches_host"] is True
    assert line["config"]["parallelism"] == "zero-partition x2"
    assert line["config"]["model"].startswith("Qwen2.5-7B")
    e2e = line["e2e"]
    assert e2e.get("composite_matches_device_path") is True, e2e
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0


def test_bench_two_ranks_trainer_step():
    need_gpu()
    line = run_bench(2, "--workload", "train", "--steps", "3", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["value"] > 0


def test_bench_reference_arm_under_torchrun_rank0_only():
    need_gpu()
    line = run_bench(2, "--impl", "reference", "--steps", "1", "--warmup", "0")
    assert line["impl"] == "reference"
    assert "unavailable" in line or (line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference")
