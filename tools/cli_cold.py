#!/usr/bin/env python
"""Cold-process latency of the CLI drop-in (what a user of `tailor merge` sees: process
start, CUDA context, pinned/device staging warm-up, I/O, device work, re-verify).
Medium shape L8 h1024 f2752 v32000, N=8, K=4 (2.33 GB composite), files on $1 (default /tmp).
usage: cli_cold.py [root_dir] [reps]"""
import os
import pathlib
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_22158_b200 as t  # noqa: E402

root = sys.argv[1] if len(sys.argv) > 1 else None
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cli = ROOT / "paper_2602_22158_b200" / "bin" / "tailor"
work = pathlib.Path(tempfile.mkdtemp(prefix="tailor-cli-", dir=root))
try:
    fam = t.SynthFamily(t.ModelSpec(8, 1024, 2752, 32000, False, 42), 8, 4, 100)
    dirs = [str(work / "run" / f"checkpoint-{k * 100}") for k in range(1, 5)]
    for k in range(1, 5):
        fam.write_dir(k, dirs[k - 1])
    del fam
    for i in range(reps):
        env = dict(os.environ, TAILOR_TRACE="1" if i == reps - 1 else "0")
        t0 = time.perf_counter()
        sel = subprocess.run([str(cli), "select", "--snapshots", ",".join(dirs), "--rho", "0.5", "--out",
                              str(work / "r.yaml")], capture_output=True, text=True, env=env)
        t1 = time.perf_counter()
        mer = subprocess.run([str(cli), "merge", "--recipe", str(work / "r.yaml"), "--out", str(work / f"m{i}")],
                             capture_output=True, text=True, env=env)
        t2 = time.perf_counter()
        assert sel.returncode == 0 and mer.returncode == 0, (sel.stderr, mer.stderr)
        print(f"rep {i}: tailor select {1e3 * (t1 - t0):.0f} ms, tailor merge {1e3 * (t2 - t1):.0f} ms "
              f"(2.33 GB composite -> {2.334 / (t2 - t0):.2f} GB/s cold, both processes)", flush=True)
        if i == reps - 1:
            print(sel.stderr + mer.stderr)
        shutil.rmtree(work / f"m{i}")
finally:
    shutil.rmtree(work, ignore_errors=True)
