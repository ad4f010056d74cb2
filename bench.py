#!/usr/bin/env python
"""Benchmark: update-magnitude selective composite merge (LLMTailor hot path) on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on at
1/2/4/8 GPUs): Llama-3.1-8B-shaped model (reference ModelSpec semantics:
L32 h4096 f14336 v128256, untied, no GQA/bias; 8.84 B params), ZeRO-3 layout
over 8 ranks, 4 consecutive synthetic snapshots, rho = 0.5 magnitude selection.

One step = the WHOLE job (all 8 ZeRO rank partitions: 123.3 GB of composite) at
every GPU count G (strong scaling): GPU g owns ranks [8g/G, 8(g+1)/G) and
  A. K3/K4 scores each owned partition's 4 snapshots of fp32 masters,
  -> NCCL all-gather of the FP64 partials (G > 1),
  B. per owned partition: K9 (rank-order combine + global magnitude selection +
     segment tables, on the device) and the K2 gathers of the composite rank shard
     and weights share.
A partition's sources (4 x 15.4 GB) are resident in HBM when its segment runs; the
partitions that do not fit together are regenerated (K5) between the timed
segments. Inputs >> 126 MB L2, so no L2 flush is needed.
TAILOR_BENCH_SHARE_GPU=1 (tests only) runs N>1 ranks on one GPU over gloo.
`--gpus N` without WORLD_SIZE in the environment relaunches itself under
torch.distributed.run with N processes (one per GPU).

`e2e`: the same job through the C ABI with HOST (pinned) buffers: masters
staged H2D for scoring, then the shard pipeline (H2D of exactly the selected
bytes -> K2 -> D2H) per partition.

`--impl reference`: the reference's own CPU implementation (oracle/_ref/ref_tool:
reference read_checkpoint + scorer restatement + resolve_plan + execute_merge,
file I/O and re-verify included) on a bounded sample on the host cores: cfg3's
per-layer shape (one h4096 f14336 layer, 8 ranks, 4 snapshots; vocabulary cut);
cfg1 is small enough to run exactly.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0
WORKLOADS = {
    # name: (L, h, f, v, tied, ZeRO ranks N, snapshots K, rho, description)
    "cfg3": (32, 4096, 14336, 128256, False, 8, 4, 0.5,
             "Llama-3.1-8B-shaped ZeRO-3 8-rank partitions, update-magnitude selective merge of 4 sources"),
    "cfg2": (28, 3584, 18944, 152064, False, 8, 2, 0.5,
             "Qwen2.5-7B-shaped, half-layer merge of 2 sources (as 8 ZeRO-rank partitions)"),
    "cfg1": (4, 256, 688, 32000, False, 1, 2, 0.5,
             "tiny Llama-style 4-layer (hidden 256), 2 sources half-layer merge, 1 ZeRO rank"),
    "cfg4": (32, 4096, 14336, 128256, False, 8, 16, 0.5,
             "Llama-3.1-8B-shaped update-norm scoring sweep over 16 consecutive snapshots (scorer only)"),
    "tiny8": (4, 256, 688, 32000, False, 8, 4, 0.5,
              "tiny Llama-style 4-layer (hidden 256), 8 ZeRO ranks, 4 snapshots (test workload for the N>1 path)"),
    "cfg5": (80, 8192, 28672, 128256, False, 8, 4, 0.5,
             "Llama-3-70B-shaped ZeRO-3 8-rank merge of 4 sources with pinned host staging "
             "(partitions exceed single-pass HBM budget)"),
}
# Reference-arm / cpu_baseline samples (the reference's CPU path runs ~0.06 GB/s, and a
# whole cfg3 job needs ~0.6 TB of host RAM in its ShardLoader): cfg3/cfg4/cfg5 use cfg3's
# per-layer shape (one h4096 f14336 decoder layer, 8 ranks, 4 snapshots, vocabulary cut
# to 256); cfg2 its own per-layer shape; cfg1 runs exactly.
SAMPLES = {
    "cfg3": (1, 4096, 14336, 256, False, 8, 4, 0.5),
    "cfg2": (1, 3584, 18944, 256, False, 8, 2, 0.5),
    "cfg1": (4, 256, 688, 32000, False, 1, 2, 0.5),
}
SAMPLE_EXTRAPOLATION = {"cfg3": "~35 min for the 123.7 GB job at the sampled rate (and ~0.6 TB of host RAM)",
                        "cfg2": "~60 min for the 115 GB job at the sampled rate"}
MODEL_NAMES = {"cfg1": "tiny Llama-style (reference ModelSpec)", "cfg2": "Qwen2.5-7B-shaped (reference ModelSpec)",
               "cfg3": "Llama-3.1-8B-shaped (reference ModelSpec)", "cfg4": "Llama-3.1-8B-shaped (reference ModelSpec)",
               "cfg5": "Llama-3-70B-shaped (reference ModelSpec)", "tiny8": "tiny Llama-style (reference ModelSpec)"}
SCORE_VARIANTS = {0: "auto", 1: "register", 2: "staged", 3: "register-128b", 4: "register-64b", 5: "staged-half-rows",
                  6: "staged-2-ctas"}


NOMINAL_HBM_GBS = 7700.0  # HGX B200 HBM3e (B200_PROFILING.md), context only


def shared_gpu() -> bool:
    """TAILOR_BENCH_SHARE_GPU=1: every rank on the visible GPU(s) round-robin, gloo
    for the collectives (exercises the N>1 path on a single-GPU box; tests only)."""
    return os.environ.get("TAILOR_BENCH_SHARE_GPU") == "1"


_COMM = None


def lib_comm():
    """The library's NCCL communicator (tg_comm_*), created on first use on every rank:
    rank 0's unique id travels over the torch process group (bootstrap only)."""
    global _COMM
    if _COMM is None:
        import torch
        import torch.distributed as dist

        import paper_2602_22158_b200 as t

        obj = [t.Comm.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        _COMM = t.Comm(obj[0], dist.get_world_size(), dist.get_rank(), torch.cuda.current_device())
    return _COMM


def collective_name():
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    if dist.get_backend() != "nccl":
        return "gloo (torch.distributed, host-staged; shared-GPU tests)"
    if os.environ.get("TAILOR_BENCH_TORCH_ALLGATHER") == "1":
        return "torch.distributed all_gather_into_tensor (NCCL)"
    return "tg_comm_allgather (the library's NCCL communicator)"


def all_gather(out, inp):
    """All-gather of the FP64 score partials: the library's NCCL communicator
    (tg_comm_allgather) on the current stream; TAILOR_BENCH_TORCH_ALLGATHER=1 uses torch's
    NCCL process group instead; gloo (shared-GPU tests) stages through host tensors."""
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        if os.environ.get("TAILOR_BENCH_TORCH_ALLGATHER") == "1":
            dist.all_gather_into_tensor(out, inp)
            return
        assert inp.dtype == torch.float64 and out.dtype == torch.float64 and inp.is_contiguous() and out.is_contiguous()
        lib_comm().all_gather(inp.data_ptr(), out.data_ptr(), inp.numel(), torch.cuda.current_stream().cuda_stream)
        return
    parts = [torch.empty(inp.numel(), dtype=inp.dtype) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, inp.cpu())
    out.copy_(torch.cat(parts))


def all_reduce(x, op):
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        dist.all_reduce(x, op=op)
        return
    h = x.cpu()
    dist.all_reduce(h, op=op)
    x.copy_(h)


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    try:
        p = json.loads(PEAKS_PATH.read_text())
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


_NVML_POLLER = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
bus = sys.argv[1]
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(bus)
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[2]))
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
        nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
print("ready", flush=True)
while True:
    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
    act = ", ".join("Active" if r & b else "Not Active" for b in bits)
    print(f"{time.time():.6f} {sys.argv[2]}, {sm}, {mx}, 0, 0, {act}", flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled every
    ~2 ms from a separate process (a thread in this process would compete for the GIL
    with the step loop and can miss a 75 ms region), samples kept by timestamp; falls
    back to `nvidia-smi -lms 20`."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.nvml = False
        self.t0 = self.t1 = 0.0

    def _bus_id(self):
        import torch

        p = torch.cuda.get_device_properties(self.gpu)
        return f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_POLLER, self._bus_id(), str(self.gpu)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            if self.proc.stdout.readline().strip() != "ready":
                raise RuntimeError("nvml poller did not start")
            self.nvml = True
        except Exception:
            if self.proc:
                self.proc.kill()
            self.proc, self.nvml = None, False
            if shutil.which("nvidia-smi"):
                self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                              "--format=csv,noheader,nounits", "-lms", "20"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        if self.proc:
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
        time.sleep(0.01)  # a few samples before the region starts
        self.t0 = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.t1 = time.time()
        time.sleep(0.01)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.reader.join(timeout=2)

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def collect(lo, hi):
            sm, mx, reasons = [], [], set()
            for ln in self.lines:
                if self.nvml:  # "<unix time> idx, sm, max, ..." : keep the samples inside [lo, hi]
                    ts, _, ln = ln.partition(" ")
                    try:
                        if not lo <= float(ts) <= hi:
                            continue
                    except ValueError:
                        continue
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            return sm, mx, reasons

        sm, mx, reasons = collect(self.t0, self.t1)
        widened = 0.0
        for pad in (0.01, 0.05, 0.25):  # region shorter than the poll period: nearest samples around it
            if sm or not self.nvml:
                break
            sm, mx, reasons = collect(self.t0 - pad, self.t1 + pad)
            widened = pad
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm),
               "source": "nvml 2 ms" if self.nvml else "nvidia-smi -lms 20"}
        if widened:
            out["window"] = (f"timed region {1e3 * (self.t1 - self.t0):.2f} ms < poll period: samples within "
                             f"{1e3 * widened:.0f} ms of it")
        return out


def read_stream_probe(torch, dev, gib: int = 8, reps: int = 5):
    """Read-only HBM stream reference for the scorer (which only reads): the library's
    read probe (tg_read_probe: 8 x 16-B streaming loads in flight per thread, persistent
    grid) over a buffer far larger than L2, timed with CUDA events, best of `reps`. The
    measured copy peak counts read+write and is the right denominator for the gather;
    a read-only kernel can exceed it, so the scorer is also reported against this."""
    import paper_2602_22158_b200 as t

    x = torch.empty(gib << 30, dtype=torch.uint8, device=dev)
    sink = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream(dev)
    best = None
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t.read_probe(x.data_ptr(), x.numel(), sink.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    gbs = x.numel() / (best / 1e3) / 1e9
    del x
    torch.cuda.empty_cache()
    return round(gbs, 1)


def _cudart_memcpy_d2d(dst, src, n, stream):
    import ctypes

    lib = ctypes.CDLL("libcudart.so.12") if not hasattr(_cudart_memcpy_d2d, "lib") else _cudart_memcpy_d2d.lib
    _cudart_memcpy_d2d.lib = lib
    rc = lib.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(n), ctypes.c_int(3),
                             ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"cudaMemcpyAsync: error {rc}")


def copy_probes(torch, dev, gib: int = 4, reps: int = 5):
    """Same-box copy references for the gather's roofline (read+write bytes, CUDA events,
    best of `reps`, 2 x `gib` GiB far beyond L2): torch's `copy_` (what MEASURED_PEAKS.json's
    hbm_gbs measures) and `cudaMemcpyAsync` device-to-device. K2 with dynamic tiles runs
    above both (ncu: DRAM traffic = its algorithmic bytes), so they are context, not a cap."""
    a = torch.empty(gib << 30, dtype=torch.uint8, device=dev)
    b = torch.empty_like(a)
    s = torch.cuda.current_stream(dev)
    out = {}
    for name, fn in (("torch_copy_gbs", lambda: b.copy_(a)),
                     ("memcpy_d2d_gbs", lambda: _cudart_memcpy_d2d(b.data_ptr(), a.data_ptr(), a.numel(), s.cuda_stream))):
        best = None
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[name] = round(2 * a.numel() / (best / 1e3) / 1e9, 1)
    del a, b
    torch.cuda.empty_cache()
    return out


def ncu_traffic(kernel: str, workload: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu capture of the
    same workload (profiles/*ncu_summary*.json), or None."""
    for p in sorted((ROOT / "profiles").glob("*ncu_summary*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            if d.get("workload") != workload:
                continue
            ks = d.get("kernels", {})
            k = ks.get(kernel) or next((v for n, v in ks.items() if n.startswith(kernel + "<")), None)
            if k and k.get("dram_bytes_per_launch"):
                return float(k["dram_bytes_per_launch"]), p.name
        except Exception:
            continue
    return None, None


# ----------------------------------------------------------------- reference arm --
def ref_tool_path():
    return ROOT / "oracle" / "_ref" / "ref_tool"


def sample_of(workload: str):
    return SAMPLES.get(workload, SAMPLES["cfg3"])


def sample_text(workload: str) -> str:
    L, h, f, v, tied, N, K, rho = sample_of(workload)
    return f"L{L} h{h} f{f} v{v} N{N} K{K} rho{rho}"


def gen_reference_sample(workdir: pathlib.Path, workload: str):
    """Snapshot dirs of the workload's bounded sample, written by the reference writer."""
    L, h, f, v, tied, N, K, rho = sample_of(workload)
    src = workdir / "src"
    if not src.exists():
        subprocess.run([str(ref_tool_path()), "gen", "--layers", str(L), "--hidden", str(h), "--ffn", str(f),
                        "--vocab", str(v), "--seed", "42", "--ranks", str(N), "--snapshots", str(K), "--out", str(src)],
                       check=True, stdout=subprocess.DEVNULL)
    return [str(src / f"checkpoint-{k * 100}") for k in range(1, K + 1)]


def run_reference_sample(workdir: pathlib.Path, workers: int, workload: str = "cfg3"):
    """One bounded sample of the workload through the reference library: returns
    (seconds, composite_bytes, detail). Score (reference read_checkpoint per snapshot on
    its own thread + FP64 scorer restatement) -> select -> resolve_plan -> execute_merge
    (+ its re-verify), files in /tmp."""
    rho = sample_of(workload)[7]
    dirs = gen_reference_sample(workdir, workload)
    out = workdir / f"merged-{time.time_ns()}"
    t0 = time.perf_counter()
    p = subprocess.run([str(ref_tool_path()), "select-merge", "--snapshots", ",".join(dirs), "--rho", str(rho),
                        "--out", str(out), "--workers", str(workers)], capture_output=True, text=True, check=True)
    dt = time.perf_counter() - t0
    detail = json.loads(p.stdout)
    composite = composite_bytes_on_disk(out)
    shutil.rmtree(out, ignore_errors=True)
    return dt, composite, detail


def composite_bytes_on_disk(out: pathlib.Path) -> int:
    """Payload bytes of a written composite (weights + every rank shard, headers excluded)."""
    total = 0
    for p in [out / "model.weights", *sorted((out / "optim").glob("rank_*.shard"))]:
        with open(p, "rb") as fh:
            hlen = int.from_bytes(fh.read(8), "little")
        total += os.path.getsize(p) - 8 - hlen
    return total


def run_files_sample(workdir: pathlib.Path, workload: str, cores: int, reps: int = 2, combined: bool = True):
    """The same bounded sample through OUR files drop-in, best of `reps` after one warm-up:
    (seconds, composite bytes). combined: tg_select_merge (score, select, merge and
    re-verify in one call; the scorer's device copies of the masters feed the merge) —
    the counterpart of the reference's select-merge; else tg_select_recipe then
    tg_execute_merge."""
    import paper_2602_22158_b200 as t

    rho = sample_of(workload)[7]
    dirs = gen_reference_sample(workdir, workload)
    best, comp = None, 0
    for i in range(reps + 1):
        out = workdir / f"ours-{time.time_ns()}"
        t0 = time.perf_counter()
        if combined:
            _, _, _, st = t.select_merge(dirs, str(out), rho, t.MergeOptions(workers=cores))
        else:
            rec, _, _ = t.select_recipe(dirs, rho)
            st = t.execute_merge(rec, str(out), t.MergeOptions(workers=cores))
        dt = time.perf_counter() - t0
        comp = st.bytes_moved
        shutil.rmtree(out, ignore_errors=True)
        if i > 0:
            best = dt if best is None else min(best, dt)
    return best, comp


# The headline metric (BASELINE.json: composite-checkpoint merge GB/s vs HBM roofline);
# both arms print the same string and the same `config` so the driver pairs them.
MERGE_METRIC = "composite-checkpoint merge GB/s (score+select+merge) vs HBM roofline"


def workload_config(workload: str) -> dict:
    """The `config` object of both arms' lines (identical for the same workload)."""
    L, h, f, v, tied, N, K, rho, desc = WORKLOADS[workload]
    return {"workload": workload, "description": desc, "model": MODEL_NAMES[workload],
            "shape": f"L{L} h{h} f{f} v{v} {'tied' if tied else 'untied'}", "zero_ranks": N, "snapshots": K,
            "rho": rho, "unit_of_work": "the whole job per step: every ZeRO rank partition scored, selected, merged"}


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    if args.workload not in SAMPLES:
        print(json.dumps({"impl": "reference", "unavailable": f"no reference sample for workload {args.workload}"}))
        return 0
    if not ref_tool_path().exists():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_tool not built"}))
        return 0
    work = pathlib.Path(tempfile.mkdtemp(prefix="tailor-ref-"))
    try:
        for _ in range(args.warmup):
            run_reference_sample(work, cores, args.workload)
        times, comp = [], 0
        for _ in range(args.steps):
            dt, comp, _ = run_reference_sample(work, cores, args.workload)
            times.append(dt)
    finally:
        shutil.rmtree(work, ignore_errors=True)
    total = sum(times)
    value = comp * args.steps / total / 1e9
    sample = (f"reference select-merge (read_checkpoint per snapshot + FP64 scorer + resolve_plan + execute_merge "
              f"with re-verify, files in /tmp) on {sample_text(args.workload)}: {comp / 1e9:.3f} GB composite per step"
              + ("" if sample_of(args.workload)[:4] == WORKLOADS[args.workload][:4] else
                 f"; the workload's per-layer shape with {sample_of(args.workload)[0]} layer(s) and a cut vocabulary "
                 f"(the reference's rate is per byte: a cfg-sized run would take "
                 f"{SAMPLE_EXTRAPOLATION.get(args.workload, 'hours')})"))
    line = {"metric": MERGE_METRIC, "value": round(value, 4),
            "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8 (payload bytes) / f32->f64 (scores)", "data": "synthetic",
            "config": workload_config(args.workload),
            "impl": "reference", "sample": sample,
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- our arm --------
def owned_partitions(N: int, world: int, rank: int):
    """GPU g owns the contiguous block of ZeRO ranks [g N/G, (g+1) N/G) (SURVEY §8e
    partitions by rank; a block, so the all-gathered partials are already in rank order)."""
    if N % world:
        raise SystemExit(f"{N} ZeRO rank partitions do not split evenly over {world} GPUs")
    per = N // world
    return list(range(rank * per, (rank + 1) * per))


class Residency:
    """Device slots for the K snapshots (rank shard + weights share) of the partitions a GPU
    owns. Partition i of `mine` lives in slot i % R; with R < len(mine) (cfg3 at G <= 2: 62 GB
    per partition) a partition is materialised into its slot by K5 on the device, untimed,
    before the timed segment that reads it (inputs resident when a timed region starts)."""

    def __init__(self, torch, t, fam, mine, N, K, dev, sp, budget):
        self.fam, self.mine, self.K, self.sp = fam, mine, K, sp
        self.shard_bytes = fam.shard_bytes(1, mine[0])
        base = t.MergeRecipe(num_ranks=N, base_checkpoint=f"S{K}").to_yaml()
        self.wrange = {}
        for p in mine:
            lo, hi, _ = t.MergePartition(fam, base, -1, p, N).range()
            self.wrange[p] = (lo, hi)
        self.wmax = max(16, max(hi - lo for lo, hi in self.wrange.values()))
        per_part = K * (self.shard_bytes + self.wmax)
        self.R = max(1, min(len(mine), int(budget // per_part)))
        self.slots = [([torch.empty(self.shard_bytes, dtype=torch.uint8, device=dev) for _ in range(K)],
                       [torch.empty(self.wmax, dtype=torch.uint8, device=dev) for _ in range(K)])
                      for _ in range(self.R)]
        self.holds = [None] * self.R
        self.generated = 0

    def slot(self, i):
        return self.slots[i % self.R]

    def ensure(self, i):
        """Partition mine[i] resident in its slot (K5 generation if another one is there)."""
        s, p = i % self.R, self.mine[i]
        if self.holds[s] != p:
            shards, wbufs = self.slots[s]
            self.fam.gen_shard(p, 1, self.K, [b.data_ptr() for b in shards], self.sp)
            lo, hi = self.wrange[p]
            self.fam.gen_weights(1, self.K, lo, hi, [b.data_ptr() for b in wbufs], self.sp)
            self.holds[s] = p
            self.generated += 1
        return self.slots[s]

    def resident_bytes(self):
        return self.R * self.K * (self.shard_bytes + self.wmax)


def our_arm(args, rank, world, local_rank):
    """The whole job per step at every G (strong scaling): each of the G GPUs owns N/G
    ZeRO rank partitions; per step
      A. K3/K4 score every owned partition (K snapshots' fp32 masters; partials written
         straight into this GPU's rows of the rank-ordered partials table),
      -> NCCL all-gather of the FP64 partials (G > 1; a barrier first, so no rank's timed
         collective absorbs another's untimed regeneration),
      B. per owned partition: K9 combine (rank order) + magnitude selection + segment
         tables on the device, then the K2 gathers of the composite shard partition and
         weights share.
    Every compute segment is one CUDA graph (captured once per partition), replayed and
    timed with CUDA events on the launching stream; the step time is the sum of the
    segments, the job time the max over ranks. The same method at every G."""
    import torch
    import torch.distributed as dist

    import paper_2602_22158_b200 as t

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, h, f, v, tied, N, K, rho, desc = WORKLOADS[args.workload]
    mine = owned_partitions(N, world, rank)
    spec = t.ModelSpec(L, h, f, v, tied, 42)
    fam = t.SynthFamily(spec, N, K, 100)
    M = fam.num_modules
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    nres = (K - 1) * M * 2

    # ---- buffers: the rank-ordered partials table, outputs, resident source slots ---------
    table = torch.zeros(N * nres, dtype=torch.float64, device=dev)  # [N][K-1][M][2]
    base_yaml = t.MergeRecipe(num_ranks=N, base_checkpoint=f"S{K}").to_yaml()
    out_shard = torch.empty(fam.shard_bytes(1, mine[0]), dtype=torch.uint8, device=dev)
    sharing = env_int("LOCAL_WORLD_SIZE", 1) if shared_gpu() else 1  # ranks on this GPU (tests)
    free, _ = torch.cuda.mem_get_info(dev)
    budget = free / sharing - out_shard.numel() - (12 << 30)  # read probe (8 GB) + scratch
    res = Residency(torch, t, fam, mine, N, K, dev, sp, budget / 1.0)
    out_w = torch.empty(res.wmax, dtype=torch.uint8, device=dev)

    scorers, steps_ = {}, {}
    for i, p in enumerate(mine):
        sc = t.Scorer(fam, p, 1, K)
        sc.set_variant(args.score_variant)
        scorers[p] = sc
        ds = t.SelectStep(fam, p, p, N, rho)
        shards, wbufs = res.slot(i)
        ds.bind([b.data_ptr() for b in shards], [b.data_ptr() for b in wbufs])
        steps_[p] = ds
    composite = {}
    for p in mine:
        sb, wlo, whi = steps_[p].range()
        composite[p] = sb + (whi - wlo)
    torch.cuda.synchronize(dev)

    def seg_score(i, s):
        p = mine[i]
        shards, _ = res.slot(i)
        scorers[p].run([b.data_ptr() for b in shards], table.data_ptr() + p * nres * 8, s)

    def seg_merge(i, s, phases=7):
        p = mine[i]
        steps_[p].run(table.data_ptr(), N, out_shard.data_ptr(), out_w.data_ptr(), args.variant, s, phases=phases)

    # ---- one CUDA graph per (segment, partition), captured once (after the warm-up steps:
    # the first run of a plan uploads its tables / binds its bases, which is not capturable)
    graphs = {}

    def capture():
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        for i in range(len(mine)):
            for kind, fn in (("A", seg_score), ("B", seg_merge)):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    fn(i, cs.cuda_stream)
                graphs[(kind, i)] = g
        torch.cuda.synchronize(dev)

    def run_seg(kind, i):
        if graphs:
            graphs[(kind, i)].replay()
        elif kind == "A":
            seg_score(i, sp)
        else:
            seg_merge(i, sp)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def gather_partials(rec):
        """All-gather of this GPU's rows of the partials table (in place, rank order)."""
        if world == 1:
            return
        torch.cuda.synchronize(dev)
        dist.barrier()
        a, b = ev(), ev()
        a.record(stream)
        lo = mine[0] * nres
        mine_rows = table[lo:lo + len(mine) * nres].clone()
        all_gather(table, mine_rows)
        b.record(stream)
        rec.append((a, b))

    def step(rec):
        """One whole-job step; rec collects the (start, end) events of its timed segments."""
        order_a = list(range(len(mine)))
        for i in order_a:  # A: score (partitions already resident first)
            res.ensure(i)
            a, b = ev(), ev()
            a.record(stream)
            run_seg("A", i)
            b.record(stream)
            rec.append((a, b))
        gather_partials(rec)
        for i in reversed(order_a):  # B: select + merge (the slots A left resident first)
            res.ensure(i)
            a, b = ev(), ev()
            a.record(stream)
            run_seg("B", i)
            b.record(stream)
            rec.append((a, b))

    for w in range(args.warmup):
        step([])
        if w == 0 and not args.no_graph:
            torch.cuda.synchronize(dev)
            capture()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    # ---- timed steps ---------------------------------------------------------------------
    gen_before = res.generated
    recs = []
    with ClockSampler(local_rank) as clocks:
        for _ in range(args.steps):
            step(recs)
        torch.cuda.synchronize(dev)
    total_ms = sum(a.elapsed_time(b) for a, b in recs)
    regen_per_step = (res.generated - gen_before) / args.steps
    max_ms = total_ms
    if world > 1:
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        all_reduce(tt, dist.ReduceOp.MAX)
        max_ms = float(tt.item())
    sec = max_ms / 1e3
    job_bytes = sum(fam.shard_bytes(1, p) for p in range(N)) + fam.weights_bytes(1)  # whole composite payload
    value = job_bytes * args.steps / sec / 1e9
    scores_per_s = M * (K - 1) * args.steps / sec  # complete module scores (all ranks combined) per second

    # ---- per-kernel times: one eager pass with events between the launches ----------------
    # A spin kernel (torch.cuda._sleep, ~5 ms) holds the stream first, so all four launches
    # are queued before the GPU reaches e[0]: the events bracket device time, not the host's
    # launch latency (which dominates at cfg1's microsecond kernels).
    kt = {"score": [], "select": [], "gather_shard": [], "gather_weights": []}
    for i in range(len(mine)):
        res.ensure(i)
        shards, _ = res.slot(i)
        e = [ev() for _ in range(5)]
        torch.cuda._sleep(10_000_000)
        e[0].record(stream)
        seg_score(i, sp)
        e[1].record(stream)
        seg_merge(i, sp, phases=1)
        e[2].record(stream)
        seg_merge(i, sp, phases=2)
        e[3].record(stream)
        seg_merge(i, sp, phases=4)
        e[4].record(stream)
        torch.cuda.synchronize(dev)
        for k_, (a, b) in zip(kt, zip(e, e[1:])):
            kt[k_].append(a.elapsed_time(b))
    if world > 1:  # the eager pass overwrote this GPU's rows with the same values; keep the table consistent
        gather_partials([])

    # ---- parity: device selection == host selection; composite == host-planned gather ------
    allparts = table.cpu().tolist()
    yaml_h, src_h, _, gap_h = fam.select(allparts, N, rho)
    checks, checksums = [], []
    for i in reversed(range(len(mine))):
        p = mine[i]
        res.ensure(i)
        shards, wbufs = res.slot(i)
        run_seg("B", i)
        src_d, _ = steps_[p].result(sp)
        spl = t.MergePartition(fam, yaml_h, p)
        spl.bind([shards[k - 1].data_ptr() + lo for k, c, lo, hi in spl.windows()])
        wlo, whi = res.wrange[p]
        wpl = t.MergePartition(fam, yaml_h, -1, p, N)
        wpl.bind([wbufs[k - 1].data_ptr() + (lo - wlo) for k, c, lo, hi in wpl.windows()])
        ref_s = torch.empty(spl.bytes, dtype=torch.uint8, device=dev)
        ref_w = torch.empty(max(16, wpl.bytes), dtype=torch.uint8, device=dev)
        spl.run(ref_s.data_ptr(), args.variant, sp)
        wpl.run(ref_w.data_ptr(), args.variant, sp)
        bulk = spl.bulk_ok  # bound plan: its segments and bases decide the K2 path
        torch.cuda.synchronize(dev)
        ok = (src_d == src_h and chunked_equal(torch, ref_s, out_shard[:spl.bytes])
              and chunked_equal(torch, ref_w[:wpl.bytes], out_w[:wpl.bytes]))
        del ref_s, ref_w
        checks.append(bool(ok))
        checksums.append((p, composite_checksum(torch, out_shard[:spl.bytes], out_w[:wpl.bytes])))
        del spl, wpl
    select_check = all(checks)
    if world > 1:
        flag = torch.tensor([1 if select_check else 0], dtype=torch.int32, device=dev)
        all_reduce(flag, dist.ReduceOp.MIN)
        select_check = bool(flag.item())
        allsums = [None] * world
        dist.all_gather_object(allsums, checksums)
        checksums = [c for part in allsums for c in part]
    checksums = [c for _, c in sorted(checksums)]

    # ---- uncached plan cost, for the record ----------------------------------------
    t0 = time.perf_counter()
    t.MergePartition(fam, yaml_h, mine[0])
    t.MergePartition(fam, yaml_h, -1, mine[0], N)
    plan_ms = (time.perf_counter() - t0) * 1e3

    # ---- e2e through the C ABI with host buffers ------------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, t, torch, fam, res, scorers, yaml_h, mine, N, world, dev, sp, K, M, rho, nres, table)

    # ---- roofline of the dominant kernel ----------------------------------------------
    hbm, peak_kind = peaks()
    read_gbs = read_stream_probe(torch, dev) if not args.no_read_probe else None
    try:
        copies = copy_probes(torch, dev) if not args.no_read_probe else None
    except Exception as e:  # context only: the line still prints
        copies = {"error": str(e)[:200]}
    g_ms = statistics.mean(kt["gather_shard"])
    s_ms = statistics.mean(kt["score"])
    gather_achieved = 2 * out_shard.numel() / (g_ms / 1e3) / 1e9
    score_achieved = scorers[mine[0]].bytes_read / (s_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic("gather_bulk_kernel" if bulk and args.variant != 1 else "gather_lsu_kernel",
                                       args.workload)
    resident = res.resident_bytes()
    launches_per_step = 5 * len(mine)

    if rank != 0:
        return 0
    line = {
        "metric": MERGE_METRIC,
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(max_ms / args.steps, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8 (payload bytes) / f32->f64 (scores)", "data": "synthetic",
        "config": workload_config(args.workload),
        "detail": {"params": fam.parameter_count, "composite_bytes_per_step": job_bytes,
                   "parallelism": f"zero-partition x{world} (GPU g owns ranks {mine[0]}..{mine[-1]} of {N}"
                                  + (", all-gather of the FP64 partials over NCCL)" if world > 1 else ")"),
                   "collective": collective_name(),
                   "partitions_per_gpu": len(mine), "resident_partition_slots": res.R,
                   "regenerations_per_step": regen_per_step,
                   "timing": "sum of CUDA-event-timed segments per step (score per partition | all-gather | "
                             "select+merge per partition), max over ranks; K5 regeneration of partitions that do not "
                             "fit HBM together happens between segments, untimed",
                   "l2": f"inputs {resident / 1e9:.1f} GB resident per GPU vs 126 MB L2 (no flush needed)",
                   "gather_variant": {0: "auto (bulk-3x64K, dynamic tiles)", 1: "lsu", 2: "bulk-3x64K", 3: "bulk-6x32K",
                                      4: "bulk-2cta-3x32K", 5: "bulk-4x48K", 6: "bulk-8x24K",
                                      7: "bulk-3x64K, static tile split"}[args.variant],
                   "score_variant": SCORE_VARIANTS[args.score_variant],
                   "plan_ms_uncached": round(plan_ms, 3), "min_boundary_gap": gap_h, "selection_source_of": src_h,
                   "selection": "device (K9 on the all-gathered rank-ordered partials, no host round trip)",
                   "device_selection_and_composite_match_host_plan": select_check,
                   "composite_checksums": checksums,
                   "step_launch": ("CUDA graph per segment (A: 2 kernel nodes, B: 3)" if graphs
                                   else "eager (5 launches per partition)")},
        "layers_scored_per_s": round(scores_per_s, 1),
        "kernels_ms": {k: round(statistics.mean(x), 4) for k, x in kt.items()},
        "roofline": {"bound": "hbm", "kernel": "K2 gather (rank shard partition)",
                     "achieved": round(gather_achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(gather_achieved / hbm, 4), "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": 2 * out_shard.numel(),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "same_box_copy_probes": copies,
                     "frac_of_nominal": round(gather_achieved / NOMINAL_HBM_GBS, 4),
                     "note": "peak = MEASURED_PEAKS.json hbm_gbs (torch copy_); K2's dynamic tile claiming runs "
                             "above it; frac_of_nominal is against the 7.7 TB/s HGX B200 figure"},
        "scorer_roofline": {"achieved": round(score_achieved, 1), "peak": hbm, "unit": "GB/s",
                            "frac": round(score_achieved / hbm, 4), "bytes_per_launch": scorers[mine[0]].bytes_read,
                            "read_stream_probe_gbs": read_gbs,
                            "frac_of_read_stream": round(score_achieved / read_gbs, 4) if read_gbs else None},
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clocks.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1 and ref_tool_path().exists() and args.workload in SAMPLES:
        work = pathlib.Path(tempfile.mkdtemp(prefix="tailor-cpu-"))
        try:
            cores = os.cpu_count() or 1
            dt, comp, _ = run_reference_sample(work, cores, args.workload)
            ours_dt, ours_comp = run_files_sample(work, args.workload, cores)
            two_dt, _ = run_files_sample(work, args.workload, cores, combined=False)
            line["cpu_baseline"] = {"value": round(comp / dt / 1e9, 4), "unit": "GB/s", "cores": cores,
                                    "kind": "reference",
                                    "sample": f"reference select-merge on {sample_text(args.workload)}, "
                                              f"{comp / 1e9:.3f} GB composite, {dt:.1f} s, files in /tmp (page cache warm)"}
            if not args.no_workers1:  # also a workers=1 run of the reference
                dt1, comp1, _ = run_reference_sample(work, 1, args.workload)
                line["cpu_baseline"]["workers_1"] = {"value": round(comp1 / dt1 / 1e9, 4), "unit": "GB/s", "cores": 1,
                                                     "seconds": round(dt1, 2)}
            line["same_sample_files"] = {
                "what": "the cpu_baseline sample through OUR files drop-in (tg_select_merge: device scorer whose "
                        "master copies feed the merge, device gather, device re-verify) on the same snapshot files",
                "sample": sample_text(args.workload), "value": round(ours_comp / ours_dt / 1e9, 4), "unit": "GB/s",
                "seconds": round(ours_dt, 3), "reference_value": round(comp / dt / 1e9, 4),
                "speedup_vs_reference": round((ours_comp / ours_dt) / (comp / dt), 1),
                "two_calls": {"what": "tg_select_recipe then tg_execute_merge", "value": round(ours_comp / two_dt / 1e9, 4),
                              "seconds": round(two_dt, 3)}}
        finally:
            shutil.rmtree(work, ignore_errors=True)
    print(json.dumps(line))
    return 0


def chunked_equal(torch, a, b, chunk=1 << 28):
    """torch.equal over byte tensors in 256 MB pieces (no full-size temporaries)."""
    if a.numel() != b.numel():
        return False
    return all(torch.equal(a[i:i + chunk], b[i:i + chunk]) for i in range(0, a.numel(), chunk))


def composite_checksum(torch, *parts, chunk_words=1 << 25):
    """Order-sensitive 64-bit checksum of device byte buffers (position-weighted sum of
    the int64 words, wrapping), for comparing composites across GPU counts; 256 MB at a time."""
    acc = 0
    mask = (1 << 64) - 1
    for x in parts:
        n = x.numel() // 8 * 8
        w = x[:n].view(torch.int64)
        total = 0
        for i in range(0, w.numel(), chunk_words):
            piece = w[i:i + chunk_words]
            idx = torch.arange(i + 1, i + 1 + piece.numel(), device=w.device, dtype=torch.int64)
            total = (total + int((piece * idx).sum().item())) & mask
        acc = (acc * 1000003 + total) & mask
        for b in x[n:].cpu().tolist():
            acc = (acc * 257 + b) & mask
    return f"{acc:016x}"


def pcie_rates(torch, dev):
    """Measured pinned copy bandwidth (GB/s) H2D alone, D2H alone and each way while both
    stream at once (1 GiB, best of 3; tools/pcie_probe.py). Under bidirectional load each
    direction gets less than alone (B200 box: ~48 vs ~56 GB/s), so host-link floors are:
    the smaller direction overlapped at the concurrent rate, the rest of the larger alone."""
    n = 1 << 30
    probe = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
    probe_d = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
    s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def probe_time(up, dn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record()
        s_up.wait_event(e0)
        s_dn.wait_event(e0)
        if up:
            with torch.cuda.stream(s_up):
                probe_d[0].copy_(probe[0], non_blocking=True)
        if dn:
            with torch.cuda.stream(s_dn):
                probe[1].copy_(probe_d[1], non_blocking=True)
        torch.cuda.current_stream(dev).wait_stream(s_up)
        torch.cuda.current_stream(dev).wait_stream(s_dn)
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / 1e3

    return {name: max(n / probe_time(*flags) / 1e9 for _ in range(3))
            for name, flags in {"h2d": (True, False), "d2h": (False, True), "bidir_each": (True, True)}.items()}


def host_ram_available():
    try:
        import psutil

        return psutil.virtual_memory().available
    except Exception:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")


def e2e_run(args, t, torch, fam, res, scorers, yaml, mine, N, world, dev, sp, K, M, rho, nres, table):
    """The same whole-job step through the C ABI with HOST (pinned) sources and
    destination, phase by phase like the device step:
      A. per owned partition: H2D of the K snapshots' master fields into a device slot
         (tg_scorer_run reads them in shard layout) and scoring into this GPU's rows;
      -> all-gather of the partials (G > 1), D2H of the table, host selection
         (tg_family_select) == the device path's recipe;
      B. per owned partition: the shard pipeline (tg_mplan_run_host: H2D of exactly the
         selected bytes -> K2 -> D2H, three streams, chunked) for the composite shard and
         for the weights share.
    Host sources exist for one partition at a time (62 GB pinned at cfg3): before each
    timed segment the partition's bytes are materialised into pinned memory (K5 on the
    device + D2H, untimed; phase A materialises the masters only). Timed: the segments,
    wall clock around synchronised copies and kernels; max over ranks."""
    import torch.distributed as dist

    K_ = K
    shard_b, wmax = res.shard_bytes, res.wmax
    need = K_ * (shard_b + wmax) + shard_b + wmax + (2 << 30)
    local = env_int("LOCAL_WORLD_SIZE", world)
    avail = host_ram_available()
    fits = need * local <= 0.85 * avail
    if world > 1:  # every rank must take the same branch (collectives follow)
        flag = torch.tensor([1 if fits else 0], dtype=torch.int32, device=dev)
        all_reduce(flag, dist.ReduceOp.MIN)
        fits = bool(flag.item())
    if not fits:
        return {"value": None, "unit": "GB/s",
                "skipped": f"host RAM: {local} ranks x {need / 1e9:.0f} GB pinned > 85% of {avail / 1e9:.0f} GB available"}
    hshards = [torch.empty(shard_b, dtype=torch.uint8).pin_memory() for _ in range(K_)]
    hw = [torch.empty(wmax, dtype=torch.uint8).pin_memory() for _ in range(K_)]
    hout = torch.empty(shard_b, dtype=torch.uint8).pin_memory()
    hwout = torch.empty(wmax, dtype=torch.uint8).pin_memory()
    master_ranges = master_byte_ranges(fam, mine[0], K_)  # same byte layout for every rank
    counters = {"h2d": 0, "d2h": 0}

    def sync_time(fn):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0

    def materialise(i, masters_only):
        """Partition mine[i]'s sources into the pinned host buffers (untimed)."""
        shards, wbufs = res.ensure(i)
        for k in range(K_):
            if masters_only:
                for lo, hi in master_ranges:
                    hshards[k][lo:hi].copy_(shards[k][lo:hi])
            else:
                hshards[k].copy_(shards[k])
                hw[k].copy_(wbufs[k])
        torch.cuda.synchronize(dev)

    def one_step(check_output):
        secs = 0.0
        h2d = d2h = 0
        for i, p in enumerate(mine):  # A
            materialise(i, True)
            shards, _ = res.slot(i)

            def seg_a():
                for k in range(K_):
                    for lo, hi in master_ranges:
                        shards[k][lo:hi].copy_(hshards[k][lo:hi], non_blocking=True)
                scorers[p].run([b.data_ptr() for b in shards], table.data_ptr() + p * nres * 8, sp)

            secs += sync_time(seg_a)
            h2d += K_ * sum(hi - lo for lo, hi in master_ranges)
        if world > 1:
            torch.cuda.synchronize(dev)
            dist.barrier()
        box = {}

        def seg_select():
            if world > 1:
                lo = mine[0] * nres
                rows = table[lo:lo + len(mine) * nres].clone()
                all_gather(table, rows)
            box["sel"] = fam.select(table.cpu().tolist(), N, rho)

        secs += sync_time(seg_select)
        d2h += N * nres * 8
        assert box["sel"][0] == yaml, "e2e selection differs from the device path's"
        ok = True
        for i in reversed(range(len(mine))):  # B
            p = mine[i]
            materialise(i, False)
            spl = t.MergePartition(fam, yaml, p)
            wpl = t.MergePartition(fam, yaml, -1, p, N)
            wlo, _ = res.wrange[p]
            io = {}

            def seg_b():
                io["w"] = wpl.run_host([hw[k - 1].data_ptr() + (lo - wlo) for k, c, lo, hi in wpl.windows()],
                                       hwout.data_ptr(), args.variant, async_=True)
                io["s"] = spl.run_host([hshards[k - 1].data_ptr() + lo for k, c, lo, hi in spl.windows()],
                                       hout.data_ptr(), args.variant, async_=True)
                spl.wait()
                wpl.wait()

            secs += sync_time(seg_b)
            h2d += io["w"][0] + io["s"][0]
            d2h += io["w"][1] + io["s"][1]
            if check_output:  # the host composite == the device gather of the same sources
                shards, wbufs = res.ensure(i)
                spl.bind([shards[k - 1].data_ptr() + lo for k, c, lo, hi in spl.windows()])
                ref = torch.empty(spl.bytes, dtype=torch.uint8, device=dev)
                spl.run(ref.data_ptr(), args.variant, sp)
                torch.cuda.synchronize(dev)
                ok = ok and chunked_equal(torch, ref.cpu(), hout[:spl.bytes])
                del ref
        counters.update(h2d=h2d, d2h=d2h)
        return secs, ok

    one_step(False)  # warm-up: pools, plans
    steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        dist.barrier()
    total, ok = 0.0, True
    for s in range(steps):
        dt, good = one_step(s == steps - 1)
        total += dt
        ok = ok and good
    if world > 1:
        tt = torch.tensor([total], dtype=torch.float64, device=dev)
        all_reduce(tt, dist.ReduceOp.MAX)
        total = float(tt.item())
        f_ = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        all_reduce(f_, dist.ReduceOp.MIN)
        ok = bool(f_.item())
    job_bytes = sum(fam.shard_bytes(1, p) for p in range(N)) + fam.weights_bytes(1)
    bw = pcie_rates(torch, dev)
    H, D = counters["h2d"] / 1e9, counters["d2h"] / 1e9
    ha = K_ * sum(hi - lo for lo, hi in master_ranges) * len(mine) / 1e9  # pass A: H2D only
    hb = H - ha
    link = lambda h_, d_: (min(h_, d_) / bw["bidir_each"] + (h_ - min(h_, d_)) / bw["h2d"]  # noqa: E731
                           + (d_ - min(h_, d_)) / bw["d2h"])
    floor_s = ha / bw["h2d"] + link(hb, D)
    per_step = total / steps
    return {"value": round(job_bytes * steps / total / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": counters["h2d"], "d2h_bytes_per_step": counters["d2h"], "steps": steps,
            "ms_per_step": round(per_step * 1e3, 2), "composite_matches_device_path": ok,
            "pcie_roofline": {"bound": "pcie (host link)", "h2d_gbs_measured": round(bw["h2d"], 1),
                              "d2h_gbs_measured": round(bw["d2h"], 1),
                              "bidir_gbs_each_measured": round(bw["bidir_each"], 1),
                              "floor_ms_per_step": round(floor_s * 1e3, 2),
                              "floor_model": "pass A (masters) H2D alone + pass B min(H,D) both ways at the concurrent "
                                             "rate + the rest one way (the selection is a barrier between them)",
                              "frac": round(floor_s / per_step, 4)},
            "path": "C ABI: H2D masters -> tg_scorer_run per partition -> all-gather -> tg_family_select -> "
                    "tg_mplan_run_host per partition (pinned host sources and destination)"}


def scorer_arm(args, rank, world, local_rank):
    """cfg4: scorer-only sweep. Each GPU holds the packed fp32 masters of its rank
    partition for 16 consecutive snapshots (16 x 4.4 GB) and scores the 15
    consecutive pairs in one pass (each snapshot read once), then the partials are
    all-gathered and combined. Metric: module-scores per second."""
    import torch
    import torch.distributed as dist

    import paper_2602_22158_b200 as t

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, h, f, v, tied, N, K, rho, desc = WORKLOADS[args.workload]
    K = args.snapshots or K  # --snapshots: the same sweep over K snapshots (scorer geometry studies)
    fam = t.SynthFamily(t.ModelSpec(L, h, f, v, tied, 42), N, K, 100)
    M, r = fam.num_modules, rank
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    bufs = [torch.empty(fam.packed_master_bytes(r), dtype=torch.uint8, device=dev) for _ in range(K)]
    fam.gen_masters(r, 1, K, [b.data_ptr() for b in bufs], sp)
    scorer = t.Scorer(fam, r, 1, K, packed=True)
    scorer.set_variant(args.score_variant)
    partials = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device=dev)
    gathered = torch.zeros(world * (K - 1) * M * 2, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    kms = []

    def step(rec):
        e0, e1 = ev(), ev()
        e0.record(stream)
        scorer.run([b.data_ptr() for b in bufs], partials.data_ptr(), sp)
        e1.record(stream)
        if world > 1:
            all_gather(gathered, partials)
            parts = gathered.cpu()
        else:
            parts = partials.cpu()
        out = fam.select(parts.tolist(), world, rho)
        if rec is not None:
            rec.append((e0, e1))
        return out

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    recs = []
    with ClockSampler(local_rank) as clocks:
        start, end = ev(), ev()
        start.record(stream)
        for _ in range(args.steps):
            res = step(recs)
        end.record(stream)
        torch.cuda.synchronize(dev)
    ms = start.elapsed_time(end)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        all_reduce(tt, dist.ReduceOp.MAX)
        ms = float(tt.item())
    kms = statistics.mean(a.elapsed_time(b) for a, b in recs)
    hbm, peak_kind = peaks()
    achieved = scorer.bytes_read / (kms / 1e3) / 1e9
    read_gbs = read_stream_probe(torch, dev) if not args.no_read_probe else None
    kname = ("score_staged_kernel<16>" if args.score_variant in (0, 2) else
             "score_partials_kernel<16,2>" if args.score_variant == 4 else "score_partials_kernel<16,4>")
    traffic, src = ncu_traffic(kname, args.workload)
    if rank != 0:
        return 0
    # Units: one rank partition of every module-pair score per GPU per step; all G
    # GPUs together produce (K-1) x M complete module scores per step once G = N.
    value = (K - 1) * M * world / N * args.steps / (ms / 1e3)
    print(json.dumps({
        "metric": "module update-magnitude scores per second (scorer-only sweep)", "value": round(value, 1),
        "unit": "module-scores/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 -> f64 accumulate", "data": "synthetic",
        "config": {"workload": "cfg4", "description": desc, "snapshots": K, "pairs": K - 1, "modules": M,
                   "zero_ranks": N, "unit_of_work": "one ZeRO rank partition of 16 snapshots' masters per GPU",
                   "score_variant": SCORE_VARIANTS[args.score_variant],
                   "bytes_per_gpu_step": scorer.bytes_read, "min_boundary_gap": res[3]},
        "roofline": {"bound": "hbm", "kernel": "K3 " + kname, "achieved": round(achieved, 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4), "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": scorer.bytes_read, "traffic": traffic, "traffic_source": src,
                     "read_stream_probe_gbs": read_gbs,
                     "frac_of_read_stream": round(achieved / read_gbs, 4) if read_gbs else None},
        "gpu_launches": args.steps * 2, "clocks": clocks.summary()}))
    return 0


def hoststaged_arm(args, rank, world, local_rank):
    """cfg5 (Llama-3-70B-shaped, 8 ZeRO ranks, 4 sources): one rank partition per GPU
    is 4 x 120 GB of source shards + 4 x 20 GB of weights — more than HBM (180 GB) and
    than this box's host RAM (196 GB), so sources live in pinned host memory one
    window at a time. The timed work per step is the host-staged pipeline itself:
      A. masters of the 4 snapshots (4 x 40 GB, packed) H2D, scored pair by pair as
         they arrive (two device slots, K3/K4 per consecutive pair);
      B. selection (all-gathered partials), then the composite shard partition in
         tensor-aligned sub-units (tg_mplan sub-ranges) and the weights share in
         pieces, each through tg_mplan_run_host (H2D of the needed bytes -> K2 -> D2H);
         masters selected from S_{K-1} / S_K are read from the two device slots that
         pass A left holding them (packed layout, resident bit 3), not re-uploaded.
    Between timed pieces the next window's source bytes are materialised (K5 on the
    device -> D2H into pinned host buffers; untimed, like every other workload's
    input generation). Every sub-unit's host output is checked against a device
    gather of the same windows."""
    import torch
    import torch.distributed as dist

    import paper_2602_22158_b200 as t

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, h, f, v, tied, N, K, rho, desc = WORKLOADS[args.workload]
    if world > N:
        raise SystemExit(f"cfg5 has {N} rank partitions; cannot run on {world} GPUs")
    fam = t.SynthFamily(t.ModelSpec(L, h, f, v, tied, 42), N, K, 100)
    M, r = fam.num_modules, rank
    sp = torch.cuda.current_stream(dev).cuda_stream
    U, UW = env_int("TAILOR_CFG5_UNITS", 8), 2  # shard sub-units, weights pieces per share

    def sync_time(fn):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0

    def pass_a():
        """Masters H2D + pairwise scoring; returns (seconds timed, bytes H2D, partials)."""
        pm = fam.packed_master_bytes(r)
        slots = [torch.empty(pm, dtype=torch.uint8, device=dev) for _ in range(2)]
        host = torch.empty(pm, dtype=torch.uint8, pin_memory=True)
        partials = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device=dev)
        scorers = {k: t.Scorer(fam, r, k - 1, k, packed=True) for k in range(2, K + 1)}
        secs = 0.0
        for k in range(1, K + 1):
            slot = slots[(k - 1) % 2]
            fam.gen_masters(r, k, k, [slot.data_ptr()], sp)  # materialise snapshot k's masters ...
            host.copy_(slot)                                    # ... into pinned host memory
            slot.zero_()
            secs += sync_time(lambda: slot.copy_(host, non_blocking=True))  # timed: H2D
            if k >= 2:
                p = k - 2
                out = partials[p * M * 2:(p + 1) * M * 2]
                secs += sync_time(lambda: scorers[k].run([slots[(k - 2) % 2].data_ptr(), slot.data_ptr()],
                                                         out.data_ptr(), sp))
        del host
        # the two slots now hold the packed masters of S_{K-1} and S_K: pass B reads those
        # masters from HBM instead of re-uploading them
        resident = {k: slots[(k - 1) % 2] for k in (K - 1, K)}
        return secs, K * pm, partials, resident

    def pass_b(yaml, resident):
        """Composite shard partition in sub-units + weights share in pieces, host-staged.
        Each piece's plan is destroyed after it runs, so its pipeline buffers go back to the
        pinned/device pools and the next piece reuses them; the first piece runs once untimed
        to fill the pools (a process pays that once, not per piece)."""
        specs = [(r, u, U) for u in range(U)] + [(-1, r * UW + j, N * UW) for j in range(UW)]
        win_bytes = out_bytes = 0
        for sp_ in specs:
            p = t.MergePartition(fam, yaml, *sp_)
            win_bytes = max(win_bytes, sum(hi - lo for _, _, lo, hi in p.windows()))
            out_bytes = max(out_bytes, p.bytes)
            del p
        hwin = torch.empty(win_bytes, dtype=torch.uint8, pin_memory=True)
        hout = torch.empty(out_bytes, dtype=torch.uint8, pin_memory=True)
        dwin = torch.empty(win_bytes, dtype=torch.uint8, device=dev)
        dref = torch.empty(out_bytes, dtype=torch.uint8, device=dev)
        secs, h2d, d2h, comp, ok = 0.0, 0, 0, 0, True
        piece_s.clear()
        for i, sp_ in enumerate(specs):
            p = t.MergePartition(fam, yaml, *sp_)
            offs, at = [], 0
            for k, c, lo, hi in p.windows():   # materialise this piece's source windows
                if c >= 0:
                    fam.gen_shard_range(c, k, lo, hi, dwin.data_ptr() + at, sp)
                else:
                    fam.gen_weights(k, k, lo, hi, [dwin.data_ptr() + at], sp)
                offs.append(at)
                at += hi - lo
            hwin[:at].copy_(dwin[:at])
            p.bind([dwin.data_ptr() + o for o in offs])  # device reference of the same windows
            p.run(dref.data_ptr(), args.variant, sp)
            res = {}

            dres = [resident[k].data_ptr() if (c >= 0 and k in resident) else None for k, c, lo, hi in p.windows()]

            def run():
                res["io"] = p.run_host([hwin.data_ptr() + o for o in offs], hout.data_ptr(), args.variant,
                                       d_windows=dres, resident_fields=8 if any(dres) else 0)

            if i == 0:
                sync_time(run)  # untimed: fills the pools with this pipeline's staging buffers
            dt = sync_time(run)
            secs += dt
            piece_s.append((round(dt, 4), round(p.bytes / 1e9, 2), len(offs)))
            if os.environ.get("TAILOR_CFG5_REPEAT"):  # diagnostics: steady-state time of the same piece
                piece_s[-1] += (round(sync_time(run), 4),)
            h2d += res["io"][0]
            d2h += res["io"][1]
            comp += p.bytes
            ok = ok and bool(torch.equal(hout[:p.bytes].to(dev), dref[:p.bytes]))
            del p
        del hwin, hout, dwin, dref
        return secs, h2d, d2h, comp, ok

    piece_s = []

    def step():
        sa, ha, partials, resident = pass_a()
        if world > 1:
            gathered = torch.zeros(world * partials.numel(), dtype=torch.float64, device=dev)
            all_gather(gathered, partials)
            parts = gathered
        else:
            parts = partials
        t0 = time.perf_counter()
        yaml, src, _, gap = fam.select(parts.cpu().tolist(), world, rho)
        sel = time.perf_counter() - t0
        sb, hb, db, comp, ok = pass_b(yaml, resident)
        del resident
        return {"secs": sa + sel + sb, "score_s": sa, "merge_s": sb, "h2d": ha + hb, "d2h": db + parts.numel() * 8,
                "h2d_a": ha, "h2d_b": hb, "d2h_b": db,
                "comp": comp, "ok": ok, "gap": gap, "sources": src}

    with ClockSampler(local_rank) as clocks:
        rec = [step() for _ in range(max(1, args.steps))]
    secs = sum(x["secs"] for x in rec)
    if world > 1:
        tt = torch.tensor([secs], dtype=torch.float64, device=dev)
        all_reduce(tt, dist.ReduceOp.MAX)
        secs = float(tt.item())
    last = rec[-1]
    n = len(rec)
    value = last["comp"] * world * n / secs / 1e9
    # host-link roofline of the same bytes (bidirectional model as in e2e_run)
    H, D = last["h2d"] / 1e9, last["d2h"] / 1e9
    probe = pcie_rates(torch, dev)

    def link_floor(h, d):  # both directions at the concurrent rate, the rest one way
        m = min(h, d)
        return m / probe["bidir_each"] + (h - m) / probe["h2d"] + (d - m) / probe["d2h"]

    # The selection is a barrier between pass A (masters in: H2D only) and pass B (the
    # merge: both directions), so the floor is the sum of the two passes' floors; the
    # all-overlapped floor is reported beside it.
    floor = link_floor(last["h2d_a"] / 1e9, 0.0) + link_floor(last["h2d_b"] / 1e9, last["d2h_b"] / 1e9)
    overlapped_floor = link_floor(H, D)
    if rank != 0:
        return 0
    line = {
        "metric": "composite-checkpoint merge GB/s (score+select+merge), host-staged", "value": round(value, 3),
        "unit": "GB/s", "n_gpus": world, "steps": n, "warmup": 0, "ms_per_step": round(secs / n * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8 (payload bytes) / f32->f64 (scores)", "data": "synthetic",
        "config": {"workload": "cfg5", "description": desc, "model": MODEL_NAMES["cfg5"],
                   "params": fam.parameter_count, "zero_ranks": N, "snapshots": K, "rho": rho,
                   "unit_of_work": "one ZeRO rank partition per GPU, host-staged in sub-units",
                   "shard_sub_units": U, "weights_pieces": UW, "composite_bytes_per_gpu_step": last["comp"],
                   "min_boundary_gap": last["gap"], "score_s": round(last["score_s"], 3),
                   "merge_s": round(last["merge_s"], 3), "merge_piece_s": piece_s,
                   "source_materialisation": "K5 window by window into pinned host buffers, untimed"},
        "host_output_matches_device_gather": all(x["ok"] for x in rec),
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": last["h2d"],
                "d2h_bytes_per_step": last["d2h"],
                "note": "the measurement itself is end to end (pinned host sources and destination)"},
        "roofline": {"bound": "pcie (host link)", "achieved": round((H + D) / (secs / n), 2), "unit": "GB/s",
                     "floor_ms_per_step": round(floor * 1e3, 1), "frac": round(floor / (secs / n), 4),
                     "floor_model": "pass A H2D-only floor + pass B bidirectional floor (selection barrier between them)",
                     "all_overlapped_floor_ms": round(overlapped_floor * 1e3, 1),
                     "h2d_gbs_measured": round(probe["h2d"], 1), "d2h_gbs_measured": round(probe["d2h"], 1),
                     "bidir_gbs_each_measured": round(probe["bidir_each"], 1)},
        "gpu_launches": None, "clocks": clocks.summary()}
    print(json.dumps(line))
    return 0


def trainer_arm(args, rank, world, local_rank):
    """SURVEY §8 f4 at scale: the device-resident trainer step (bit-exact AdamW on a
    Llama-3.1-8B-shaped ZeRO rank partition, one partition per GPU). Algorithmic bytes
    per element: the update pass reads w,m,v (12 B) and writes them (12 B), recomputing
    the gradient from w and checking the new masters' exponents, which is the next
    step's pre-update finiteness check = 24 B (a standalone 4 B check runs only when the
    state was written by someone else, e.g. on the first step). TAILOR_TRAIN_STORE_GRAD=1:
    the gradient goes through a scratch buffer, 4 + 4 + 16 + 12 = 36 B. Both passes stream host-built
    TrainTile runs as float4. Each step synchronizes once (the non-finite check precedes any
    state change, as apply_step requires) and once more for the norm partials; timed by
    wall clock around synchronized steps, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2602_22158_b200 as t

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, h, f, v, tied, N, K, rho, desc = WORKLOADS["cfg3"]
    tr = t.Trainer(t.ModelSpec(L, h, f, v, tied, 42), N, rank, rank + 1, device=local_rank)
    n = tr.elements
    for s in range(1, args.warmup + 1):
        tr.step(s)
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank) as clocks:
        t0 = time.perf_counter()
        for s in range(args.warmup + 1, args.warmup + args.steps + 1):
            gn, un = tr.step(s)
        dt = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        all_reduce(tt, dist.ReduceOp.MAX)
        dt = float(tt.item())
    hbm, kind = peaks()
    bpe = 36 if os.environ.get("TAILOR_TRAIN_STORE_GRAD", "0") not in ("", "0") else 24
    gbs = bpe * n * args.steps / dt / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "device trainer steps: optimizer elements updated per second (bit-exact AdamW)",
            "value": round(n * world * args.steps / dt / 1e9, 3), "unit": "G elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (FP64 norms)",
            "data": "synthetic gradients (reference GradientSource)",
            "config": {"workload": "train", "model": "Llama-3.1-8B-shaped", "zero_ranks": N,
                       "elements_per_gpu": n, "unit_of_work": "one rank partition per GPU"},
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(gbs / hbm, 4), "peak_kind": kind, "bytes_per_element": bpe,
                         "gradient": "scratch buffer" if bpe == 36 else
                         "recomputed in the update pass, which also checks the next step's masters"},
            "last_norms": {"grad": gn, "update": un}, "gpu_launches": (1 if bpe == 24 else 2) * args.steps, "clocks": clocks.summary()}))
    return 0


FILES_SPEC = (8, 1024, 2752, 32000, False, 8, 4, 0.5)  # BASELINE.md §2 "medium" shape


def disk_probe(work: pathlib.Path, gib: float = 1.0):
    """tools/disk_probe on the work directory's filesystem (compiled on first use):
    the files line's rooflines (device read bandwidth with O_DIRECT, page-cache read and
    write rates)."""
    exe = ROOT / "tools" / "disk_probe"
    src = ROOT / "tools" / "disk_probe.cpp"
    try:
        if not exe.exists() or exe.stat().st_mtime < src.stat().st_mtime:
            subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", str(src), "-o", str(exe)], check=True,
                           capture_output=True)
        p = subprocess.run([str(exe), str(work), str(gib), "8", "4"], capture_output=True, text=True, check=True)
        return json.loads(p.stdout.strip().splitlines()[-1])
    except Exception as e:  # the line still prints, without its disk roofline
        return {"error": str(e)[:200]}


def evict_files(paths):
    """Drops the files' pages from the page cache (fsync first: only clean pages go)."""
    for p in paths:
        fd = os.open(p, os.O_RDONLY)
        try:
            os.fsync(fd)
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
        finally:
            os.close(fd)


def files_arm(args):
    """The reference's own definition of a merge, on files (reads, assembly, writes and
    the mandatory re-verify): our select+merge (device scorer on the snapshot files ->
    selection -> execute_merge with the device gather and device re-verify) vs the
    reference's (ref_tool select-merge: read_checkpoint scorer restatement +
    resolve_plan + execute_merge) on the same synthetic snapshot directories, in two
    page-cache states:
      warm — sources in the page cache (both arms), io auto -> buffered reads;
      cold — the sources' pages dropped before every step (fsync + POSIX_FADV_DONTNEED),
             io auto -> O_DIRECT source reads (and, for comparison, one buffered-read step).
    Rooflines from tools/disk_probe on the same filesystem: cold against the device's
    O_DIRECT read bandwidth (the bytes that must come off the device: every snapshot's
    masters for the scorer + the composite's source bytes), warm against the host's
    page-cache copy rates (reads: scorer + merge + re-verify; writes: the composite)."""
    import paper_2602_22158_b200 as t

    L, h, f, v, tied, N, K, rho = FILES_SPEC
    cores = os.cpu_count() or 1
    work = pathlib.Path(tempfile.mkdtemp(prefix="tailor-files-"))
    try:
        fam = t.SynthFamily(t.ModelSpec(L, h, f, v, tied, 42), N, K, 100)
        dirs = [str(work / "run" / f"checkpoint-{k * 100}") for k in range(1, K + 1)]
        for k in range(1, K + 1):
            fam.write_dir(k, dirs[k - 1])
        os.sync()  # flush the sources now: background writeback of them would land inside timed steps
        src_files = [str(p) for d in dirs for p in sorted(pathlib.Path(d).rglob("*")) if p.is_file()]
        master_bytes = K * sum(hi - lo for r in range(N) for lo, hi in master_byte_ranges(fam, r, K))
        probe = disk_probe(work)

        def one(i, tag, io="auto", cold=False, combined=False):
            if cold:
                evict_files(src_files)
            out = work / f"ours-{tag}-{i}"
            t0 = time.perf_counter()
            if combined:  # tg_select_merge: the scorer's master copies feed the merge
                _, _, gap, st = t.select_merge(dirs, str(out), rho, t.MergeOptions(workers=cores, io_mode=io))
                t1 = time.perf_counter() - st.wall_ms / 1e3
            else:
                rec, _, gap = t.select_recipe(dirs, rho)
                t1 = time.perf_counter()
                st = t.execute_merge(rec, str(out), t.MergeOptions(workers=cores, io_mode=io))
            dt = time.perf_counter() - t0
            shutil.rmtree(out, ignore_errors=True)
            os.sync()  # the composite's writeback stays out of the next step
            return dt, st, gap, {"select_ms": round((t1 - t0) * 1e3, 1), "merge_ms": round(st.wall_ms, 1),
                                 "gather_device_ms": round(st.device_ms, 2)}

        warm, cold, comp, gap, phases, cold_st = [], [], 0, None, None, None
        for i in range(args.warmup + args.steps):
            dt, st, gap, ph = one(i, "warm")
            comp = st.bytes_moved
            if i >= args.warmup:
                warm.append(dt)
                phases = ph
        # the combined call while the page cache is still warm (the cold steps below drop it)
        sm_warm, sm_res = [], 0
        for i in range(args.warmup + args.steps):
            dt, st, _, _ = one(i, "smwarm", combined=True)
            sm_res = st.resident_bytes
            if i >= args.warmup:
                sm_warm.append(dt)
        cold_steps = max(1, min(args.steps, 3))
        for i in range(cold_steps):
            dt, cold_st, _, cph = one(i, "cold", cold=True)
            cold.append(dt)
        cold_buf, _, _, _ = one(0, "coldbuf", io="buffered", cold=True)
        sm_cold = []
        for i in range(cold_steps):
            dt, _, _, _ = one(i, "smcold", cold=True, combined=True)
            sm_cold.append(dt)
        ref_steps = max(1, min(args.steps, 3))
        refs = []
        for i in range(1 + ref_steps):
            out = work / f"ref-{i}"
            t0 = time.perf_counter()
            subprocess.run([str(ref_tool_path()), "select-merge", "--snapshots", ",".join(dirs), "--rho", str(rho),
                            "--out", str(out), "--workers", str(cores)], check=True, capture_output=True)
            dt = time.perf_counter() - t0
            shutil.rmtree(out, ignore_errors=True)
            if i >= 1:
                refs.append(dt)
    finally:
        shutil.rmtree(work, ignore_errors=True)
    w_s, c_s = statistics.median(warm), statistics.median(cold)
    o_v, c_v = comp / w_s / 1e9, comp / c_s / 1e9
    r_v = comp / statistics.median(refs) / 1e9
    # cold bound: bytes that must come off the device / its O_DIRECT read bandwidth
    disk_bytes = master_bytes + comp
    rd = probe.get("read_direct_gbs")
    cold_roof = None
    if rd:
        floor = disk_bytes / (rd * 1e9)
        cold_roof = {"bound": "device read (O_DIRECT, tools/disk_probe)", "achieved": round(disk_bytes / c_s / 1e9, 3),
                     "peak": rd, "unit": "GB/s", "frac": round(floor / c_s, 4), "bytes_per_step": disk_bytes,
                     "floor_ms": round(floor * 1e3, 1)}
    # warm bound: page-cache copies (reads: scorer masters + merge sources + re-verify; writes: composite)
    rw, wc = probe.get("read_warm_gbs"), probe.get("write_cached_gbs")
    warm_roof = None
    if rw and wc:
        floor = (master_bytes + 2 * comp) / (rw * 1e9) + comp / (wc * 1e9)
        overlapped = max((master_bytes + 2 * comp) / (rw * 1e9), comp / (wc * 1e9))
        warm_roof = {"bound": "host page-cache copies (tools/disk_probe, 32 threads): reads/read_warm + writes/write_cached",
                     "achieved_gbs_composite": round(o_v, 3), "read_bytes_per_step": master_bytes + 2 * comp,
                     "write_bytes_per_step": comp, "peak_read_gbs": rw, "peak_write_gbs": wc,
                     "floor_ms": round(floor * 1e3, 1), "frac": round(floor / w_s, 4),
                     "floor_overlapped_ms": round(overlapped * 1e3, 1), "frac_overlapped": round(overlapped / w_s, 4),
                     "note": "floor_ms: reads then writes at the probe's rates; the lanes overlap them (the merge "
                             "writes while the scorer/merge/re-verify read), so frac can exceed 1; frac_overlapped "
                             "assumes reads and writes fully concurrent at the same rates"}
    sm_w, sm_c = statistics.median(sm_warm), statistics.median(sm_cold)
    sm_line = {"what": "tg_select_merge (one call; the masters the scorer read stay on the device and feed the "
                       "merge: resident_bytes are not read again)",
               "resident_bytes": sm_res,
               "warm": {"value": round(comp / sm_w / 1e9, 4), "ms_per_step": round(sm_w * 1e3, 1)},
               "cold": {"value": round(comp / sm_c / 1e9, 4), "ms_per_step": round(sm_c * 1e3, 1)}}
    if rd:  # what must come off the device now: every snapshot's masters + the composite minus the kept masters
        sm_bytes = disk_bytes - sm_res
        sm_line["cold"]["roofline"] = {"bound": "device read (O_DIRECT, tools/disk_probe)", "peak": rd, "unit": "GB/s",
                                       "bytes_per_step": sm_bytes, "floor_ms": round(sm_bytes / (rd * 1e9) * 1e3, 1),
                                       "frac": round(sm_bytes / (rd * 1e9) / sm_c, 4)}
    print(json.dumps({
        "metric": "composite-checkpoint merge GB/s on files (score+select+merge+re-verify)",
        "value": round(o_v, 4), "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(w_s * 1e3, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/f32/f64", "data": "synthetic (written by the GPU writer, byte-identical "
                                                          "to the reference writer), page cache warm",
        "config": {"workload": "files", "shape": f"L{L} h{h} f{f} v{v} N{N} K{K} rho{rho}",
                   "composite_bytes": comp, "scorer_master_bytes": master_bytes, "min_boundary_gap": gap,
                   "last_step_phases": phases},
        "roofline": warm_roof,
        "cold": {"value": round(c_v, 4), "unit": "GB/s", "ms_per_step": round(c_s * 1e3, 1), "steps": cold_steps,
                 "io": "auto (O_DIRECT source reads; the sources' pages dropped before every step)",
                 "direct_read_bytes": cold_st.direct_read_bytes if cold_st else None, "last_step_phases": cph,
                 "roofline": cold_roof,
                 "buffered_reads_same_state": {"value": round(comp / cold_buf / 1e9, 4), "ms_per_step": round(cold_buf * 1e3, 1)}},
        "select_merge": sm_line,
        "disk_probe": probe,
        "reference": {"value": round(r_v, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                      "ms_per_step": round(statistics.median(refs) * 1e3, 1), "page_cache": "warm"},
        "speedup_vs_reference": round(o_v / r_v, 2)}))
    return 0


def master_byte_ranges(fam, r, K):
    """Byte ranges of the g*.master entries in rank r's shard payload (from the oracle-free layout)."""
    import json as _json

    lm = __import__("paper_2602_22158_b200").layer_map(fam.spec, fam.num_ranks)
    # Recreate the container order: lexicographic keys g<i>.exp_avg, g<i>.exp_avg_sq, g<i>.master
    keys = []
    for g in lm["groups"]:
        for fld in (".exp_avg", ".exp_avg_sq", ".master"):
            keys.append((f"g{g['index']}{fld}", g["shard_length"] * 4))
    keys.sort(key=lambda x: x[0].encode())
    out, off = [], 0
    for name, n in keys:
        if name.endswith(".master"):
            out.append((off, off + n))
        off += n
    assert off == fam.shard_bytes(1, r)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["files", "train"], default="cfg3")
    ap.add_argument("--variant", type=int, default=0, help="gather: 0 auto, 1 LSU, 2 TMA bulk 3x64K, 3-6 other rings, 7 bulk with the static tile split")
    ap.add_argument("--score-variant", type=int, default=0, help="scorer: 0 auto, 1 register, 2 TMA-staged, 5 staged half rows, 6 staged 2 CTAs/SM")
    ap.add_argument("--snapshots", type=int, default=0, help="cfg4 only: sweep over this many snapshots instead of 16")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2, help="timed e2e steps (each is the whole job)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-workers1", action="store_true", help="skip the workers=1 reference run")
    ap.add_argument("--no-read-probe", action="store_true", help="skip the read-only HBM stream probe")
    ap.add_argument("--no-graph", action="store_true", help="time eager segments instead of their CUDA graphs")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if args.workload == "cfg4":
        return init_and(scorer_arm, args, rank, world, local_rank)
    if args.workload == "cfg5":
        return init_and(hoststaged_arm, args, rank, world, local_rank)
    if args.workload == "files":
        return files_arm(args) if rank == 0 else 0
    if args.workload == "train":
        return init_and(trainer_arm, args, rank, world, local_rank)
    return init_and(our_arm, args, rank, world, local_rank)


def relaunch(n: int) -> int:
    """`bench.py --gpus N` run directly: one process per GPU under torch.distributed.run
    (rendezvous on 127.0.0.1, a free port); rank 0 prints the line."""
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(pathlib.Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def init_and(fn, args, rank, world, local_rank):
    if world > 1:
        import torch
        import torch.distributed as dist

        if shared_gpu():
            local_rank %= max(1, torch.cuda.device_count())
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return fn(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            global _COMM
            _COMM = None  # ncclCommDestroy while CUDA and the process group are still up
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
