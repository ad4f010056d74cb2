#!/usr/bin/env python
"""Source and output paths with awkward characters (spaces, quotes, '#', ': ', unicode,
brackets) through the YAML recipe path (recipe_to_yaml -> parse_recipe -> execute_merge
and the CLI) against the reference merge (JSON recipe): every output file byte-identical
(manifest provenance and sidecars carry the paths). GPU diagnostics, not in the suite."""
import json
import pathlib
import shutil
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2602_22158_b200 as t  # noqa: E402

REF = ROOT / "oracle" / "_ref" / "ref_tool"
NAMES = ["run with spaces", "it's #1", 'quo"te', "colon: here", "ünï-✓", "[brackets]{x}", "- dash", "& amp * star"]


def ref(*args):
    p = subprocess.run([str(REF), *map(str, args)], capture_output=True, text=True)
    if p.returncode:
        raise RuntimeError(p.stderr)
    return json.loads(p.stdout) if p.stdout.strip() else None


def same_tree(a, b):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file())
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file())
    assert fa == fb, (fa, fb)
    for rel in fa:
        assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


def main():
    ok = 0
    for i, name in enumerate(NAMES):
        work = pathlib.Path(tempfile.mkdtemp(prefix="paths-")) / name
        work.mkdir(parents=True)
        try:
            d = ref("gen", "--layers", 3, "--hidden", 8, "--ffn", 20, "--vocab", 32, "--seed", 40 + i, "--ranks", 2,
                    "--snapshots", 2, "--out", work / "run")["snapshots"]
            rec = t.MergeRecipe(num_ranks=2, base_checkpoint=d[1], slices=[t.RecipeSlice(d[0], [0, 2])],
                                aux={"norm": d[0]}, config_from=d[0])
            (work / "r.json").write_text(rec.to_json())
            ref("merge", "--recipe", work / "r.json", "--out", work / "ref out")
            yaml = rec.to_yaml()
            assert t.parse_recipe(yaml) == rec, yaml
            t.execute_merge(t.parse_recipe(yaml), str(work / "ours out"))
            same_tree(work / "ref out", work / "ours out")
            (work / "r.yaml").write_text(yaml)
            p = subprocess.run([str(t.CLI_PATH), "merge", "--recipe", str(work / "r.yaml"), "--out", str(work / "cli out"),
                                "--json"], capture_output=True, text=True)
            assert p.returncode == 0, p.stderr
            assert json.loads(p.stdout)["out"] == str(work / "cli out")
            same_tree(work / "ref out", work / "cli out")
            print(f"{name!r}: ok", flush=True)
            ok += 1
        except Exception as e:
            print(f"{name!r}: FAIL {type(e).__name__}: {str(e)[:300]}", flush=True)
        finally:
            shutil.rmtree(work.parent, ignore_errors=True)
    print(f"{ok}/{len(NAMES)} path sets byte-identical")
    return 0 if ok == len(NAMES) else 1


if __name__ == "__main__":
    sys.exit(main())
