"""Breakdown of bench.py's e2e unit (cfg3 rank partition, pinned host sources):
the masters H2D alone, the shard/weights host pipelines alone, and both at once,
each timed on the device. Prints one JSON line. Diagnostic only.

    python tools/e2e_probe.py [--chunk-mb 256]
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
    ap.add_argument("--chunk-mb", type=int, default=0)
    ap.add_argument("--piece-mb", type=int, default=0, help="split the masters copies into pieces (0: whole fields)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    L, h, f, v, tied, N, K, rho, _ = bench.WORKLOADS["cfg3"]
    fam = t.SynthFamily(t.ModelSpec(L, h, f, v, tied, 42), N, K, 100)
    r = 0
    sp = torch.cuda.current_stream(dev).cuda_stream
    shards = [torch.empty(fam.shard_bytes(k, r), dtype=torch.uint8, device=dev) for k in range(1, K + 1)]
    fam.gen_shard(r, 1, K, [b.data_ptr() for b in shards], sp)
    base_yaml = t.MergeRecipe(num_ranks=N, base_checkpoint=f"S{K}").to_yaml()
    wlo, whi, _ = t.MergePartition(fam, base_yaml, -1, r, N).range()
    wbufs = [torch.empty(max(16, whi - wlo), dtype=torch.uint8, device=dev) for _ in range(K)]
    fam.gen_weights(1, K, wlo, whi, [b.data_ptr() for b in wbufs], sp)
    scorer = t.Scorer(fam, r, 1, K)
    M = fam.num_modules
    partials = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device=dev)
    scorer.run([b.data_ptr() for b in shards], partials.data_ptr(), sp)
    yaml = fam.select(partials.cpu().tolist(), 1, rho)[0]
    t0 = time.perf_counter()
    hshards = [b.cpu().pin_memory() for b in shards]
    hw = [b.cpu().pin_memory() for b in wbufs]
    pin_s = time.perf_counter() - t0
    stage = [torch.empty(b.numel(), dtype=torch.uint8, device=dev) for b in shards]
    spl = t.MergePartition(fam, yaml, r)
    wpl = t.MergePartition(fam, yaml, -1, r, N)
    hout = torch.empty(spl.bytes, dtype=torch.uint8).pin_memory()
    hwout = torch.empty(max(16, wpl.bytes), dtype=torch.uint8).pin_memory()
    ranges = bench.master_byte_ranges(fam, r, K)
    side = torch.cuda.Stream(dev)
    chunk = a.chunk_mb << 20

    piece = a.piece_mb << 20
    pieces = []
    for lo, hi in ranges:
        step = piece or (hi - lo)
        pieces += [(x, min(hi, x + step)) for x in range(lo, hi, step)]

    def masters():
        with torch.cuda.stream(side):
            for lo, hi in pieces:
                for k in range(K):
                    stage[k][lo:hi].copy_(hshards[k][lo:hi], non_blocking=True)

    def pipes():
        wins = spl.windows()
        spl.run_host([hshards[k - 1].data_ptr() + lo for k, c, lo, hi in wins], hout.data_ptr(), 0, chunk,
                     d_windows=[stage[k - 1].data_ptr() + lo for k, c, lo, hi in wins], resident_fields=4, async_=True)
        wpl.run_host([hw[k - 1].data_ptr() + (lo - wlo) for k, c, lo, hi in wpl.windows()], hwout.data_ptr(), 0, chunk,
                     async_=True)

    def timed(fn):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fn()
        spl.wait()
        wpl.wait()
        torch.cuda.synchronize(dev)
        return (time.perf_counter() - t0) * 1e3

    masters()
    pipes()
    out = {"pin_s": round(pin_s, 1), "chunk_mb": a.chunk_mb, "piece_mb": a.piece_mb, "pieces": len(pieces)}
    out["masters_ms"] = min(timed(masters) for _ in range(2))
    out["pipes_ms"] = min(timed(pipes) for _ in range(2))
    out["both_ms"] = min(timed(lambda: (masters(), pipes())) for _ in range(2))
    out["both_pipes_first_ms"] = min(timed(lambda: (pipes(), masters())) for _ in range(2))

    def pipes_prefetch():
        wins = spl.windows()
        wpl.run_host([hw[k - 1].data_ptr() + (lo - wlo) for k, c, lo, hi in wpl.windows()], hwout.data_ptr(), 0, chunk,
                     async_=True)
        pf = [(hshards[k].data_ptr() + lo, stage2[k].data_ptr() + lo, hi - lo) for lo, hi in ranges for k in range(K)]
        spl.run_host([hshards[k - 1].data_ptr() + lo for k, c, lo, hi in wins], hout.data_ptr(), 0, chunk,
                     d_windows=[stage[k - 1].data_ptr() + lo for k, c, lo, hi in wins], resident_fields=4, async_=True,
                     prefetch=pf)

    stage2 = [torch.empty(b.numel(), dtype=torch.uint8, device=dev) for b in shards]
    out["pipes_with_prefetch_ms"] = min(timed(pipes_prefetch) for _ in range(3))
    ok = all(torch.equal(stage2[k][lo:hi], shards[k][lo:hi]) for k in range(K) for lo, hi in ranges)
    out["prefetch_bytes_ok"] = ok
    issue = []
    for _ in range(2):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        pipes()
        issue.append((time.perf_counter() - t0) * 1e3)
        spl.wait()
        wpl.wait()
    out["pipes_issue_ms"] = min(issue)
    out["bytes"] = {"masters": sum(hi - lo for lo, hi in ranges) * K}
    print(json.dumps({k: (round(x, 2) if isinstance(x, float) else x) for k, x in out.items()}))


if __name__ == "__main__":
    main()
