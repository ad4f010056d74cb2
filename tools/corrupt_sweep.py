#!/usr/bin/env python
"""Randomized damaged-source sweep on the GPU (not part of the default suite): reference-
written sources with one payload/header file damaged (a byte changed in the header or the
payload, truncation, junk appended, a deleted rank file), merged by the reference
(oracle/_ref/ref_tool merge: read_checkpoint + execute_merge + re-verify) and by
execute_merge: both succeed with byte-identical outputs, or both fail with the same error
kind (where the reference aborts on a damaged header, ours reports CorruptContainer).
usage: corrupt_sweep.py [cases] [seed]"""
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


def ref(*args):
    p = subprocess.run([str(REF), *map(str, args)], capture_output=True, text=True)
    return p.returncode, (json.loads(p.stdout) if p.returncode == 0 and p.stdout.strip() else None), p.stderr


def same_tree(a, b):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file())
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file())
    return fa == fb and all((a / r).read_bytes() == (b / r).read_bytes() for r in fa)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
    same = differ = 0
    for c in range(cases):
        work = pathlib.Path(tempfile.mkdtemp(prefix="corrupt-"))
        try:
            L, N, K = 1 + rng.randrange(4), 1 + rng.randrange(3), 2 + rng.randrange(2)
            spec = ["--layers", L, "--hidden", rng.choice([8, 16]), "--ffn", 20, "--vocab", 32, "--seed", 500 + c]
            d = ref("gen", *spec, "--ranks", N, "--snapshots", K, "--out", work / "run")[1]["snapshots"]
            victim = pathlib.Path(rng.choice(d))
            files = sorted(p for p in victim.rglob("*") if p.is_file() and not p.name.endswith(".json"))
            f = rng.choice(files)
            b = bytearray(f.read_bytes())
            hlen = int.from_bytes(b[:8], "little") if len(b) >= 8 else 0
            op = rng.randrange(5)
            if op == 0:  # a byte of the header
                i = rng.randrange(min(len(b), 8 + hlen))
                b[i] = rng.randrange(256)
            elif op == 1:  # a byte of the payload
                i = 8 + hlen + rng.randrange(max(1, len(b) - 8 - hlen))
                if i < len(b):
                    b[i] ^= 1 << rng.randrange(8)
            elif op == 2:
                del b[rng.randrange(len(b)):]
            elif op == 3:
                b += b"junk"
            if op == 4:
                f.unlink()
            else:
                f.write_bytes(bytes(b))
            recipe = t.MergeRecipe(num_ranks=N, base_checkpoint=d[-1],
                                   slices=[t.RecipeSlice(d[rng.randrange(K)], [i]) for i in range(L)],
                                   aux={"embed_tokens": d[0], "norm": d[-1]})
            (work / "r.json").write_text(recipe.to_json())
            rc, _, err = ref("merge", "--recipe", work / "r.json", "--out", work / "ref")
            try:
                t.execute_merge(recipe, str(work / "ours"), t.MergeOptions(workers=rng.choice([1, 4])))
                ours = None
            except t.TailorError as e:
                ours = str(e).split(":")[0]
            if rc == 0:
                ok = ours is None and same_tree(work / "ref", work / "ours")
                what = "both merged" + ("" if ok else f", ours: {ours}")
            else:
                try:
                    kind = json.loads(err.strip().splitlines()[-1])["error"]
                except Exception:
                    kind = f"abort rc={rc}"
                # the reference aborts (std::terminate) when its error path meets invalid UTF-8
                # from a damaged header; ours must then report the damage cleanly
                ok = ours == kind or (kind.startswith("abort") and ours == "CorruptContainer")
                what = f"ref {kind}, ours {ours}"
            same += ok
            differ += not ok
            print(f"case {c}: {f.relative_to(work)} op{op}: {what} {'ok' if ok else 'DIFFER'}", flush=True)
        finally:
            shutil.rmtree(work, ignore_errors=True)
    print(f"{same}/{cases} cases agree, {differ} differ")
    return 1 if differ else 0


if __name__ == "__main__":
    sys.exit(main())
