#!/usr/bin/env python
"""Tiny end-to-end exercise of every kernel, for compute-sanitizer (memcheck/racecheck/synccheck):
  compute-sanitizer --tool memcheck python tools/sanitize_run.py
Covers K5 generator (shards, weights, packed masters, tensor-aligned windows), K3/K4 scorer
(TMA ring + register + scalar paths), K9 device selection, K2 gather (bulk + LSU, aligned +
misaligned shapes, host pipeline with prefetch copies), K6 verify (through execute_merge),
K7/K8 trainer (through train, magnitude strategy)."""
import os
import pathlib
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2602_22158_b200 as t  # noqa: E402


def run(spec, N, K, variants=(0, 1, 2)):
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    parts = []
    shards = {}
    for r in range(N):
        bufs = [torch.empty(max(16, fam.shard_bytes(k, r)), dtype=torch.uint8, device="cuda") for k in range(1, K + 1)]
        fam.gen_shard(r, 1, K, [b.data_ptr() for b in bufs])
        packed = [torch.empty(max(16, fam.packed_master_bytes(r)), dtype=torch.uint8, device="cuda") for _ in range(K)]
        fam.gen_masters(r, 1, K, [b.data_ptr() for b in packed])
        out = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device="cuda")
        # racecheck tracks every smem access of the TMA-ring scorer; its wide small-K stages
        # make that run take hours, so under racecheck the ring (variant 2, and auto) is
        # exercised at K >= 4 only (the K=4 family below) and K < 4 runs the register kernel
        ring = K >= 4 or os.environ.get("TAILOR_SANITIZE_TOOL") != "racecheck"
        for sv in ((1, 2) if ring else (1,)):
            sc = t.Scorer(fam, r, 1, K)
            sc.set_variant(sv)
            sc.run([b.data_ptr() for b in bufs], out.data_ptr())
        t.Scorer(fam, r, 1, K, packed=True).run([b.data_ptr() for b in packed], out.data_ptr())
        torch.cuda.synchronize()
        parts += out.cpu().tolist()
        shards[r] = bufs
    yaml, _, _, _ = fam.select(parts, N, 0.5)
    for r in range(N):
        mp = t.MergePartition(fam, yaml, r)
        mp.bind([shards[r][k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()])
        dst = torch.empty(max(16, mp.bytes), dtype=torch.uint8, device="cuda")
        for v in variants:
            if v == 2 and not mp.bulk_ok:
                continue
            mp.run(dst.data_ptr(), v)
        # host pipeline with prefetch copies, and tensor-aligned window generation
        hsrc = [b.cpu().pin_memory() for b in shards[r]]
        hdst = torch.empty(max(16, mp.bytes), dtype=torch.uint8).pin_memory()
        extra = torch.arange(1000, dtype=torch.uint8).pin_memory()
        land = torch.empty(1000, dtype=torch.uint8, device="cuda")
        mp.run_host([hsrc[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()], hdst.data_ptr(), 0, 4096,
                    prefetch=[(extra.data_ptr(), land.data_ptr(), 1000)])
        for k, c, lo, hi in mp.windows():
            if hi > lo:
                win = torch.empty(hi - lo, dtype=torch.uint8, device="cuda")
                fam.gen_shard_range(r, k, lo, hi, win.data_ptr())
    wb = fam.weights_bytes(1)
    w = [torch.empty(wb, dtype=torch.uint8, device="cuda") for _ in range(K)]
    fam.gen_weights(1, K, 0, wb, [b.data_ptr() for b in w])
    # K9: device selection + segment tables + gathers for unit 0
    full_parts = torch.tensor(parts, dtype=torch.float64, device="cuda")
    step = t.SelectStep(fam, 0, 0, N, 0.5)
    step.bind([b.data_ptr() for b in shards[0]], [b.data_ptr() for b in w])
    lo_, hi_, _ = t.MergePartition(fam, t.MergeRecipe(num_ranks=N, base_checkpoint=f"S{K}").to_yaml(), -1, 0, N).range()
    o_s = torch.empty(max(16, fam.shard_bytes(K, 0)), dtype=torch.uint8, device="cuda")
    o_w = torch.empty(max(16, hi_ - lo_), dtype=torch.uint8, device="cuda")
    step.run(full_parts.data_ptr(), N, o_s.data_ptr(), o_w.data_ptr())
    step.result()
    torch.cuda.synchronize()
    if os.environ.get("TAILOR_SANITIZE_TOOL") == "racecheck":
        # racecheck looks for shared-memory races inside kernels; with many host threads
        # (lanes) launching kernels it tracks badly ("failure to track a kernel launch",
        # then hours), so under racecheck the file paths run with ONE lane: select (one
        # scorer lane), merge and regroup with workers=1 (assembly + pipelined re-verify
        # on the calling thread), both io modes
        os.environ["TAILOR_SCORE_LANES"] = "1"
        with tempfile.TemporaryDirectory() as d:
            for k in range(1, K + 1):
                fam.write_dir(k, f"{d}/checkpoint-{k * 100}")
            dirs = [f"{d}/checkpoint-{k * 100}" for k in range(1, K + 1)]
            rec2, _, _ = t.select_recipe(dirs, 0.5)
            t.execute_merge(rec2, f"{d}/sel1", t.MergeOptions(workers=1))
            t.execute_merge(rec2, f"{d}/sel1d", t.MergeOptions(workers=1, io_mode="direct-rw"))
            t.regroup(f"{d}/sel1", f"{d}/coarse", to_fine=False, options=t.MergeOptions(workers=1))
            t.verify_checkpoint(f"{d}/coarse")
        return
    with tempfile.TemporaryDirectory() as d:
        for k in range(1, K + 1):
            fam.write_dir(k, f"{d}/checkpoint-{k * 100}")
        rec = t.MergeRecipe(num_ranks=N, base_checkpoint=f"{d}/checkpoint-{K * 100}",
                            slices=[t.RecipeSlice(f"{d}/checkpoint-100", [0])])
        t.execute_merge(rec, f"{d}/merged")
        t.verify_checkpoint(f"{d}/merged")
        # file scorer lanes + multi-lane merge (workers 1 and 8) + regroup both ways
        dirs = [f"{d}/checkpoint-{k * 100}" for k in range(1, K + 1)]
        rec2, _, _ = t.select_recipe(dirs, 0.5)
        t.execute_merge(rec2, f"{d}/sel8", t.MergeOptions(workers=8))
        t.execute_merge(rec2, f"{d}/sel1", t.MergeOptions(workers=1))
        t.execute_merge(rec2, f"{d}/sel8d", t.MergeOptions(workers=8, io_mode="direct-rw"))
        t.regroup(f"{d}/sel8", f"{d}/coarse", to_fine=False)
        t.regroup(f"{d}/coarse", f"{d}/fine", to_fine=True)


def run_trainer():
    import os

    os.environ["TAILOR_TRAIN_STORE_GRAD"] = "1"  # scratch-gradient form
    with tempfile.TemporaryDirectory() as d:
        t.train(t.ModelSpec(2, 8, 12, 20, False, 9), f"{d}/full", 10, 10, "full", num_ranks=2)
    os.environ["TAILOR_TRAIN_STORE_GRAD"] = "0"  # default: exponent-bit check + recomputed gradient
    with tempfile.TemporaryDirectory() as d:
        t.train(t.ModelSpec(3, 8, 12, 20, False, 9), f"{d}/full", 20, 10, "full", num_ranks=2)
        t.train(t.ModelSpec(2, 16, 40, 50, True, 5), f"{d}/mag", 30, 10, "magnitude", num_ranks=3, rho=0.5)


if __name__ == "__main__":
    run_trainer()
    run(t.ModelSpec(4, 64, 172, 512, False, 42), 2, 3)   # aligned: bulk path
    run(t.ModelSpec(3, 4, 4, 8, True, 5), 3, 3)           # misaligned 12-B chunks: LSU fallbacks
    run(t.ModelSpec(1, 1, 1, 1, False, 1), 4, 2)          # padding-only ranks
    run(t.ModelSpec(2, 64, 172, 256, False, 7), 2, 4)     # K=4: the TMA-ring scorer as auto picks it
    print("sanitize run ok")
