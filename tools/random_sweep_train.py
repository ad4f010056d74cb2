#!/usr/bin/env python
"""Randomized f-row sweep on the GPU (not part of the default suite): for random shapes,
rank counts, strategies (full / parity / filter), intervals, groupings and injected
failures, against the reference binary:
  * train: our device trainer writes the reference trainer's checkpoints (every file
    byte-identical except log.jsonl, whose norms agree to 1e-9),
  * coarse runs: regroup to fine and back byte-identical to the reference's regroup,
  * fine runs: plan at a random failure step (recipe_from_manifests), merge, and resume a
    random number of steps from the composite: byte-identical to the reference's resume.
usage: random_sweep_train.py [cases] [seed]"""
import json
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


def ref(*args, check=True):
    p = subprocess.run([str(REF), *map(str, args)], capture_output=True, text=True)
    if check and p.returncode:
        raise RuntimeError(f"ref_tool {args[0]}: {p.stderr}")
    return p.returncode, (json.loads(p.stdout) if p.returncode == 0 and p.stdout.strip() else None), p.stderr


def same_tree(a, b):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file())
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file())
    assert fa == fb, (fa, fb)
    for rel in fa:
        if rel.endswith("log.jsonl"):
            la = [json.loads(x) for x in (a / rel).read_text().splitlines() if x]
            lb = [json.loads(x) for x in (b / rel).read_text().splitlines() if x]
            assert [x["step"] for x in la] == [x["step"] for x in lb], rel
            for x, y in zip(la, lb):
                for k in ("grad_norm", "update_norm"):
                    assert abs(x[k] - y[k]) <= 1e-9 * max(abs(x[k]), abs(y[k])), (rel, k, x[k], y[k])
        else:
            assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    fails = 0
    for c in range(cases):
        work = pathlib.Path(tempfile.mkdtemp(prefix="trainsweep-"))
        try:
            L, h = 1 + rng.randrange(6), rng.choice([8, 16, 24])
            f, v, tied = rng.choice([12, 20, 40]), rng.choice([20, 32, 50]), rng.random() < 0.3
            N = 1 + rng.randrange(4)
            strategy = rng.choice(["full", "parity", "filter"])
            interval = rng.randrange(5, 26)
            steps = rng.randrange(interval, 81)  # at least one checkpoint
            coarse = rng.random() < 0.3
            if coarse:
                strategy = "full"  # the reference trains partial strategies on the fine grouping only
            spec = ["--layers", L, "--hidden", h, "--ffn", f, "--vocab", v, "--seed", 900 + c] + (["--tied"] if tied else [])
            extra = []
            head = tail = 2
            sparse = 5
            if strategy == "filter":
                head = rng.randrange(0, min(3, L + 1))
                tail = rng.randrange(0, min(3, L - head + 1))
                sparse = 1 + rng.randrange(5)
                extra = ["--head", head, "--tail", tail, "--sparse-multiple", sparse]
            grouping = ["--grouping", "coarse"] if coarse else []
            ref("train", *spec, "--strategy", strategy, "--steps", steps, "--interval", interval, "--ranks", N,
                *extra, *grouping, "--out", work / "ref")
            note = f"L{L} h{h} f{f} v{v} tied={tied} N{N} {strategy} steps={steps}/{interval}"
            if coarse:
                ck = sorted((work / "ref").glob("checkpoint-*"), key=lambda p: int(p.name.split("-")[1]))
                full = [p for p in ck if json.loads((p / "manifest.json").read_text()).get("strategy") == "full"
                        or strategy == "full"]
                src = (full or ck)[-1]
                rc, _, _ = ref("regroup", "--dir", src, "--out", work / "ref_fine", check=False)
                try:
                    t.regroup(str(src), str(work / "fine"), to_fine=True)
                    ours_ok = True
                except t.TailorError:
                    ours_ok = False
                assert ours_ok == (rc == 0), ("regroup outcome", rc, ours_ok)
                if rc == 0:
                    same_tree(work / "ref_fine", work / "fine")
                    t.regroup(str(work / "fine"), str(work / "coarse"), to_fine=False)
                    same_tree(src, work / "coarse")
                note += f" coarse regroup {'ok' if rc == 0 else 'refused by both'}"
            else:
                s = t.ModelSpec(L, h, f, v, tied, 900 + c)
                t.train(s, str(work / "ours"), steps, interval, strategy, num_ranks=N, head=head, tail=tail,
                        sparse_multiple=sparse)
                same_tree(work / "ref", work / "ours")
                fs = rng.randrange(interval, steps + 15)
                rc, out, _ = ref("plan", "--run", work / "ref", "--failure-step", fs, check=False)
                if rc == 0:
                    recipe = t.recipe_from_manifests(str(work / "ref"), fs)
                    assert recipe == t.MergeRecipe.from_json(json.dumps(out["recipe"]))
                    t.execute_merge(recipe, str(work / "merged"))
                    (work / "r.json").write_text(recipe.to_json())
                    ref("merge", "--recipe", work / "r.json", "--out", work / "ref_merged")
                    same_tree(work / "ref_merged", work / "merged")
                    more = rng.randrange(1, 61)
                    ref("resume", "--ckpt", work / "merged", "--steps", more, "--out", work / "ref_res")
                    t.resume(str(work / "merged"), more, str(work / "our_res"))
                    same_tree(work / "ref_res", work / "our_res")
                    note += f" train ok, plan@{fs} merge+resume {more} ok"
                else:
                    note += f" train ok, plan@{fs} unrecoverable (both)"
            print(f"case {c}: {note}", flush=True)
        except Exception as e:  # keep sweeping; report at the end
            fails += 1
            print(f"case {c}: FAIL {type(e).__name__}: {str(e)[:300]}", flush=True)
        finally:
            shutil.rmtree(work, ignore_errors=True)
    print(f"{cases - fails}/{cases} cases passed")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
