"""cfg5 host-staged sub-unit diagnostics: one shard sub-unit of rank 0 through
tg_mplan_run_host at several chunk sizes, next to raw H2D/D2H copies of the same
pinned buffers (alone and concurrent). Prints JSON lines. Diagnostic only.

    python tools/hoststaged_probe.py [--units 8]
"""
import argparse
import json
import pathlib
import sys
import time

import torch

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2602_22158_b200 as t  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=8)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    L, h, f, v, tied, N, K, rho, _ = bench.WORKLOADS["cfg5"]
    fam = t.SynthFamily(t.ModelSpec(L, h, f, v, tied, 42), N, K, 100)
    M = fam.num_modules
    # a fixed selection: alternate modules between S3 and S4 (all four sources appear via aux)
    rec = t.MergeRecipe(num_ranks=N, base_checkpoint="S4",
                        slices=[t.RecipeSlice("S3", list(range(0, L, 2))), t.RecipeSlice("S2", list(range(1, L, 4)))],
                        aux={"embed_tokens": "S1"})
    yaml = rec.to_yaml()
    p = t.MergePartition(fam, yaml, 0, 0, a.units)
    wins = p.windows()
    tot = sum(hi - lo for _, _, lo, hi in wins)
    dwin = torch.empty(tot, dtype=torch.uint8, device=dev)
    offs, at = [], 0
    for k, c, lo, hi in wins:
        fam.gen_shard_range(c, k, lo, hi, dwin.data_ptr() + at)
        offs.append(at)
        at += hi - lo
    hwin = torch.empty(tot, dtype=torch.uint8, pin_memory=True)
    hwin.copy_(dwin)
    hout = torch.empty(p.bytes, dtype=torch.uint8, pin_memory=True)
    dscr = torch.empty(p.bytes, dtype=torch.uint8, device=dev)
    print(json.dumps({"piece_bytes": p.bytes, "window_bytes": tot, "windows": len(wins), "segments": p.num_segments}))

    def timed(fn):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0

    n = p.bytes
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def both():
        with torch.cuda.stream(s1):
            dscr.copy_(hwin[:n], non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dwin[:n], non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    raw = {"h2d": min(timed(lambda: dscr.copy_(hwin[:n], non_blocking=True)) for _ in range(2)),
           "d2h": min(timed(lambda: hout.copy_(dwin[:n], non_blocking=True)) for _ in range(2)),
           "both": min(timed(both) for _ in range(2))}
    print(json.dumps({"raw_gbs": {k: round(n / s / 1e9, 1) for k, s in raw.items()}}))
    for chunk_mb in (64, 256, 1024):
        ts = [timed(lambda: p.run_host([hwin.data_ptr() + o for o in offs], hout.data_ptr(), 0, chunk_mb << 20))
              for _ in range(3)]
        print(json.dumps({"chunk_mb": chunk_mb, "run_host_s": [round(x, 3) for x in ts],
                          "gbs_each_way": round(n / min(ts) / 1e9, 1)}))


if __name__ == "__main__":
    main()
