#!/usr/bin/env python
"""Phase trace (usage: files_trace.py [root_dir] [iters] [cold|warm] [sm|two]) of the file-facing drop-in path (TAILOR_TRACE=1):
medium shape L8 h1024 f2752 v32000, N=8, K=4 written to /tmp, then select_recipe + execute_merge. `cold`: the
sources' pages are dropped before every iteration (fsync + POSIX_FADV_DONTNEED), as in bench.py's cold files line.
`sm`: tg_select_merge (one call) instead of select_recipe + execute_merge."""
import os
import pathlib
import shutil
import sys
import tempfile
import time

os.environ["TAILOR_TRACE"] = "1"
ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_22158_b200 as t  # noqa: E402

root = (sys.argv[1] or None) if len(sys.argv) > 1 else None  # e.g. /dev/shm (default: $TMPDIR or /tmp)
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cold = len(sys.argv) > 3 and sys.argv[3] == "cold"
combined = len(sys.argv) > 4 and sys.argv[4] == "sm"  # tg_select_merge instead of the two calls
work = pathlib.Path(tempfile.mkdtemp(prefix="tailor-trace-", dir=root))
try:
    fam = t.SynthFamily(t.ModelSpec(8, 1024, 2752, 32000, False, 42), 8, 4, 100)
    dirs = [str(work / f"checkpoint-{k * 100}") for k in range(1, 5)]
    for k in range(1, 5):
        fam.write_dir(k, dirs[k - 1])
    os.sync()
    def dirty():
        with open("/proc/meminfo") as f:
            kv = dict(line.split(":", 1) for line in f)
        return {k: kv[k].strip() for k in ("Dirty", "Writeback")}

    srcs = [p for d in dirs for p in pathlib.Path(d).rglob("*") if p.is_file()]
    for i in range(iters):
        if cold:
            for p in srcs:
                fd = os.open(p, os.O_RDONLY)
                os.fsync(fd)
                os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
                os.close(fd)
        print(f"iter {i} start: {dirty()}", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        if combined:
            _, _, _, st = t.select_merge(dirs, str(work / f"m{i}"), 0.5)
            t2 = time.perf_counter()
            t1 = t2 - st.wall_ms / 1e3
        else:
            rec, _, _ = t.select_recipe(dirs, 0.5)
            t1 = time.perf_counter()
            st = t.execute_merge(rec, str(work / f"m{i}"))
            t2 = time.perf_counter()
        print(f"iter {i}: select {1e3 * (t1 - t0):.1f} ms, merge {1e3 * (t2 - t1):.1f} ms ({st.bytes_moved / 1e9:.2f} GB)",
              file=sys.stderr, flush=True)
        shutil.rmtree(work / f"m{i}")
        os.sync()
finally:
    shutil.rmtree(work, ignore_errors=True)
