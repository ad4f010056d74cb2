#!/usr/bin/env python
"""Randomized scorer/selection sweep on the GPU (not part of the default suite): random
shapes, rank counts and snapshot counts K = 2..40 (windowed sweeps beyond 16), random rho,
random device budgets (forcing the rolling-slot form) and lane counts: per-pair module
scores within 1e-6 relative (the stated tolerance) of the reference-side scorer (ref_tool score), the same
recipe, and tg_select_merge byte-identical to the reference's select-merge.
usage: random_sweep_scores.py [cases] [seed]"""
import json
import os
import pathlib
import random
import shutil
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_22158_b200 as t  # noqa: E402

REF = ROOT / "oracle" / "_ref" / "ref_tool"


def ref(*args):
    p = subprocess.run([str(REF), *map(str, args)], capture_output=True, text=True)
    if p.returncode:
        raise RuntimeError(f"ref_tool {args[0]}: {p.stderr}")
    return json.loads(p.stdout) if p.stdout.strip() else None


def same_tree(a, b):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file())
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file())
    assert fa == fb, (fa, fb)
    for rel in fa:
        assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 9)
    fails = 0
    for c in range(cases):
        work = pathlib.Path(tempfile.mkdtemp(prefix="scores-"))
        try:
            L, h = 1 + rng.randrange(5), rng.choice([8, 16, 32])
            N, K = 1 + rng.randrange(5), rng.choice([2, 3, 5, 8, 15, 16, 17, 20, 31, 33, 40])
            rho = rng.choice([0.25, 0.5, 0.75])
            tied = rng.random() < 0.3
            spec = ["--layers", L, "--hidden", h, "--ffn", 20, "--vocab", 40, "--seed", 3000 + c] + (["--tied"] if tied else [])
            d = ref("gen", *spec, "--ranks", N, "--snapshots", K, "--out", work / "run")["snapshots"]
            budget = rng.choice([None, None, 1 << 14, 1 << 18])
            if budget:
                os.environ["TAILOR_DEVICE_BUDGET"] = str(budget)
            else:
                os.environ.pop("TAILOR_DEVICE_BUDGET", None)
            r = ref("score", "--snapshots", ",".join(d), "--rho", rho)
            rec, _, gap = t.select_recipe(d, rho)
            assert rec == t.MergeRecipe.from_json(json.dumps(r["recipe"])), "recipe differs"
            sums, scores = t.score_snapshots(d)
            ref_scores = r["scores"]
            worst = 0.0
            for p_ in range(K - 1):
                for m, x in enumerate(ref_scores[p_]):
                    y = scores[p_][m]
                    worst = max(worst, abs(x - y) / max(abs(x), 1e-300))
            assert worst <= 1e-6, f"scores differ (rel {worst:.3g})"  # the stated tolerance (FP64, another summation order)
            note = ""
            if rng.random() < 0.5:
                ref("select-merge", "--snapshots", ",".join(d), "--rho", rho, "--out", work / "ref_sm")
                t.select_merge(d, str(work / "ours_sm"), rho)
                same_tree(work / "ref_sm", work / "ours_sm")
                note = ", select-merge ok"
            print(f"case {c}: L{L} h{h} N{N} K{K} rho{rho} tied={tied} budget={budget} ok (max rel {worst:.2g}){note}",
                  flush=True)
        except Exception as e:  # keep sweeping; report at the end
            fails += 1
            print(f"case {c}: FAIL {type(e).__name__}: {str(e)[:300]}", flush=True)
        finally:
            shutil.rmtree(work, ignore_errors=True)
    print(f"{cases - fails}/{cases} cases passed")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
