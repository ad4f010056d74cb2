#!/usr/bin/env python
"""Stress loop of the file drop-ins at the files-line shape (L8 h1024 f2752 v32000, N8 K4):
select_merge and select_recipe + execute_merge, warm and cold (sources evicted), repeated;
prints the first failing step. Usage: stress_files.py [iters] [shape: files|small]."""
import os
import pathlib
import shutil
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_22158_b200 as t  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 6
shape = sys.argv[2] if len(sys.argv) > 2 else "files"
# order: "mixed" (sm-warm, two-warm, sm-cold, two-cold per iteration) or "bench" (bench.py's
# files-arm order: 4 two-warm, 4 sm-warm, 3 two-cold, 1 two-cold buffered, 3 sm-cold)
order = sys.argv[3] if len(sys.argv) > 3 else "mixed"
spec = t.ModelSpec(8, 1024, 2752, 32000, False, 42) if shape == "files" else t.ModelSpec(4, 256, 688, 4000, False, 42)
N, K = 8, 4
work = pathlib.Path(tempfile.mkdtemp(prefix="tailor-stress-"))
try:
    fam = t.SynthFamily(spec, N, K, 100)
    dirs = [str(work / "run" / f"checkpoint-{k * 100}") for k in range(1, K + 1)]
    for k in range(1, K + 1):
        fam.write_dir(k, dirs[k - 1])
    os.sync()
    srcs = [str(p) for d in dirs for p in pathlib.Path(d).rglob("*") if p.is_file()]

    def evict():
        for p in srcs:
            fd = os.open(p, os.O_RDONLY)
            os.fsync(fd)
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
            os.close(fd)

    n = 0
    steps = (["sm-warm", "two-warm", "sm-cold", "two-cold"] if order == "mixed" else
             ["two-warm"] * 4 + ["sm-warm"] * 4 + ["two-cold"] * 3 + ["two-coldbuf"] + ["sm-cold"] * 3)
    for i in range(iters):
        for name in steps:
            if "cold" in name:
                evict()
            out = work / f"o{n}"
            n += 1
            t0 = time.perf_counter()
            try:
                if name.startswith("sm"):
                    t.select_merge(dirs, str(out), 0.5, t.MergeOptions(workers=os.cpu_count()))
                else:
                    rec, _, _ = t.select_recipe(dirs, 0.5)
                    io = "buffered" if name.endswith("buf") else "auto"
                    t.execute_merge(rec, str(out), t.MergeOptions(workers=os.cpu_count(), io_mode=io))
            except Exception as e:
                print(f"FAIL iter {i} step {name}: {e}", flush=True)
                sys.exit(3)
            print(f"iter {i} {name} {1e3 * (time.perf_counter() - t0):.0f} ms", flush=True)
            shutil.rmtree(out, ignore_errors=True)
            os.sync()
    print("stress ok", flush=True)
finally:
    shutil.rmtree(work, ignore_errors=True)
