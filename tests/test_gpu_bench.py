"""SURVEY §8e on one GPU: bench.py's N>1 path (one process per rank, partials
all-gathered, max-over-ranks timing, the whole job at every G) run as 2 ranks
sharing the visible B200 over gloo (TAILOR_BENCH_SHARE_GPU=1); the collectives
are the same calls the NCCL run makes. Checks the JSON line contract, that
every rank's device selection equals the host's, and that G=1 and G=2 produce
the same selection and composite bytes."""
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


def run_bench_single(*args, timeout=900):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return lines[0]


def test_bench_whole_job_same_selection_and_bytes_at_one_and_two_gpus():
    """The whole job (8 ZeRO rank partitions) at G=1 and at G=2 (ranks 0-3 / 4-7, partials
    all-gathered): the global selection and every partition's composite bytes are the
    same, and each rank's device selection equals the host plan."""
    need_gpu()
    common = ("--workload", "tiny8", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-read-probe")
    one = run_bench_single("--gpus", "1", *common)
    two = run_bench(2, *common)
    for line, n in ((one, 1), (two, 2)):
        assert line["n_gpus"] == n and line["scaling"] == "strong" and line["steps"] == 3
        assert line["value"] > 0 and line["higher_is_better"] is True
        d = line["detail"]
        assert d["device_selection_and_composite_match_host_plan"] is True
        assert d["partitions_per_gpu"] == 8 // n
        assert line["gpu_launches"] == 3 * 5 * (8 // n)
        e2e = line["e2e"]
        assert e2e.get("composite_matches_device_path") is True, e2e
        assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert one["config"] == two["config"]
    assert one["detail"]["selection_source_of"] == two["detail"]["selection_source_of"]
    assert len(one["detail"]["composite_checksums"]) == 8
    assert one["detail"]["composite_checksums"] == two["detail"]["composite_checksums"]


def test_bench_cfg2_two_ranks_regenerates_partitions():
    """cfg2 (Qwen2.5-7B-shaped) whole job at G=2 on one shared GPU: each rank owns 4
    partitions and holds fewer slots than that, so partitions are regenerated between
    the timed segments."""
    need_gpu()
    line = run_bench(2, "--workload", "cfg2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                     "--no-read-probe")
    assert line["n_gpus"] == 2 and line["config"]["model"].startswith("Qwen2.5-7B")
    d = line["detail"]
    assert d["device_selection_and_composite_match_host_plan"] is True
    assert d["resident_partition_slots"] < d["partitions_per_gpu"] == 4
    assert d["regenerations_per_step"] > 0


def test_bench_gpus_flag_relaunches_itself():
    """`bench.py --gpus 2` without torchrun spawns the ranks itself (shared GPU here)."""
    need_gpu()
    env = dict(os.environ, TAILOR_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--workload", "tiny8", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-read-probe"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def test_bench_two_ranks_trainer_step():
    need_gpu()
    line = run_bench(2, "--workload", "train", "--steps", "3", "--warmup", "3")
    assert line["n_gpus"] == 2 and line["value"] > 0


def test_bench_reference_arm_under_torchrun_rank0_only():
    need_gpu()
    line = run_bench(2, "--impl", "reference", "--workload", "cfg1", "--steps", "1", "--warmup", "0")
    assert line["impl"] == "reference"
    assert "unavailable" in line or (line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference")


def test_library_comm_allgather_single_rank():
    """tg_comm_* (the library's NCCL communicator, libnccl.so.2 loaded at run time): a
    one-rank communicator gathers its own FP64 rows unchanged, on a torch stream."""
    import torch

    import paper_2602_22158_b200 as t

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    uid = t.Comm.unique_id()
    assert len(uid) == 128
    c = t.Comm(uid, 1, 0, 0)
    x = torch.randn(4321, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    c.all_gather(x.data_ptr(), y.data_ptr(), x.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    with pytest.raises(t.TailorError):
        t.Comm(uid, 1, 3, 0)  # rank out of range
