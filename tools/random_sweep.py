#!/usr/bin/env python
"""Long randomized parity sweep on the GPU (not part of the default suite): for each case,
the reference writes random-shape sources (oracle/_ref/ref_tool gen), a random recipe
(layer moves, tied models, N <= 8, K <= 4, optional base) is merged by the reference and
by execute_merge (random worker count, random device budget forcing the streaming
re-verify), and every output file must be byte-identical; every 4th case also runs the
file scorer + selection against the reference scorer and tg_select_merge against the
reference's select-merge. `large` draws wider shapes (h 64-384, f 172-1024, v up to
4096, K up to 6; every 2nd case scores and select-merges).
usage: random_sweep.py [cases] [seed] [large]"""
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
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    large = len(sys.argv) > 3 and sys.argv[3] == "large"
    rng = random.Random(seed)
    fails = 0
    for c in range(cases):
        work = pathlib.Path(tempfile.mkdtemp(prefix="sweep-"))
        try:
            if large:
                L = 1 + rng.randrange(4)
                h = rng.choice([64, 128, 200, 256, 384])
                f, v = rng.choice([172, 344, 500, 688, 1024]), rng.choice([256, 1000, 2048, 4096])
                tied = rng.random() < 0.3
                N, K = 1 + rng.randrange(8), 2 + rng.randrange(5)
            else:
                L = 1 + rng.randrange(8)
                h = rng.choice([4, 8, 12, 16])
                f, v = rng.choice([4, 8, 20, 40]), rng.choice([8, 16, 31, 64])
                tied = rng.random() < 0.4
                N, K = 1 + rng.randrange(8), 1 + rng.randrange(4)
            spec = ["--layers", L, "--hidden", h, "--ffn", f, "--vocab", v, "--seed", 1000 + c]
            if tied:
                spec.append("--tied")
            d = ref("gen", *spec, "--ranks", N, "--snapshots", K, "--out", work / "run")["snapshots"]
            mods = ["embed_tokens", "norm"] + ([] if tied else ["lm_head"])
            targets = list(range(L))
            if rng.random() < 0.4:
                rng.shuffle(targets)
            slices = {}
            for i in range(L):
                k = rng.randrange(K)
                slices.setdefault(k, ([], []))
                slices[k][0].append(i)
                slices[k][1].append(targets[i])
            recipe = t.MergeRecipe(num_ranks=N, slices=[t.RecipeSlice(d[k], ls, ts) for k, (ls, ts) in sorted(slices.items())],
                                   aux={m: d[rng.randrange(K)] for m in mods})
            if rng.random() < 0.3:
                recipe.base_checkpoint = d[-1]
            rp = work / "recipe.json"
            rp.write_text(recipe.to_json())
            ref("merge", "--recipe", rp, "--out", work / "ref")
            workers = rng.choice([1, 2, 3, 8, 16])
            budget = rng.choice([None, None, 1 << 14, 1 << 20])
            if budget:
                os.environ["TAILOR_DEVICE_BUDGET"] = str(budget)
            else:
                os.environ.pop("TAILOR_DEVICE_BUDGET", None)
            t.execute_merge(recipe, str(work / "ours"), t.MergeOptions(workers=workers))
            same_tree(work / "ref", work / "ours")
            note = ""
            if c % (2 if large else 4) == 0 and K >= 2:
                rec, _, gap = t.select_recipe(d, 0.5)
                r = ref("score", "--snapshots", ",".join(d), "--rho", "0.5")
                assert rec == t.MergeRecipe.from_json(json.dumps(r["recipe"])), "selection differs"
                note = f" select ok (gap {gap:.3g})"
                # the combined call: the reference's select-merge vs tg_select_merge, every file
                ref("select-merge", "--snapshots", ",".join(d), "--rho", "0.5", "--out", work / "ref_sm")
                _, _, _, st = t.select_merge(d, str(work / "ours_sm"), 0.5, t.MergeOptions(workers=workers))
                same_tree(work / "ref_sm", work / "ours_sm")
                note += f", select-merge ok ({st.resident_bytes} B resident)"
            print(f"case {c}: L{L} h{h} f{f} v{v} tied={tied} N{N} K{K} workers={workers} budget={budget} ok{note}",
                  flush=True)
        except Exception as e:  # keep sweeping; report at the end
            fails += 1
            print(f"case {c}: FAIL {type(e).__name__}: {e}", flush=True)
        finally:
            shutil.rmtree(work, ignore_errors=True)
    print(f"{cases - fails}/{cases} cases passed")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
