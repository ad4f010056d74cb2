#!/usr/bin/env python
"""Regenerates tests/golden/*.json from the REFERENCE binary (oracle/_ref/ref_tool,
compiled from /root/reference by oracle/Makefile). Run here, where the reference
exists; the fixtures are committed so the checks also run where it does not.

Fixtures (small, content-addressed):
  merge_golden.json  — sha256 of every file of reference execute_merge outputs for a
                       set of recipes over reference-written synthetic sources
  score_golden.json  — reference-side scorer restatement (a13) + selection (a14) +
                       recipe over reference-written snapshots
(resolve_plan / recipe_from_manifests are pinned by live comparisons with the reference
binary in tests/test_host.py and tests/test_gpu_parity.py, not by a fixture.)
Paths inside fixtures are made relative (<SRC>/...) so they are location-free.
"""
import hashlib
import json
import pathlib
import subprocess
import sys
import tempfile

ROOT = pathlib.Path(__file__).resolve().parents[2]
TOOL = ROOT / "oracle" / "_ref" / "ref_tool"
OUT = pathlib.Path(__file__).resolve().parent

# (name, spec, ranks, snapshots)
SOURCES = [
    ("toy4", dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=909), 4, 2),
    ("tied3", dict(num_layers=3, hidden_dim=4, ffn_dim=4, vocab_size=8, weight_tied=True, seed=50001), 3, 3),
    ("odd2", dict(num_layers=2, hidden_dim=6, ffn_dim=10, vocab_size=11, weight_tied=False, seed=9), 2, 3),
    ("score4", dict(num_layers=4, hidden_dim=16, ffn_dim=40, vocab_size=64, weight_tied=False, seed=42), 2, 4),
]


def tool(*args):
    p = subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True)
    if p.returncode != 0:
        raise SystemExit(f"ref_tool {args[0]} failed: {p.stderr}")
    return json.loads(p.stdout)


def spec_args(s):
    a = ["--layers", s["num_layers"], "--hidden", s["hidden_dim"], "--ffn", s["ffn_dim"], "--vocab", s["vocab_size"],
         "--seed", s["seed"]]
    return a + (["--tied"] if s["weight_tied"] else [])


def tree_digest(d: pathlib.Path):
    return {str(p.relative_to(d)): hashlib.sha256(p.read_bytes()).hexdigest()
            for p in sorted(d.rglob("*")) if p.is_file()}


def rel(s: str, base: str) -> str:
    return s.replace(base, "<SRC>")


def recipes_for(name, spec, N, K):
    L = spec["num_layers"]
    S = [f"<SRC>/checkpoint-{k * 100}" for k in range(1, K + 1)]
    out = [("identity", {"num_ranks": N, "base_checkpoint": S[-1]})]
    if K >= 2:
        out.append(("alternating", {"num_ranks": N, "base_checkpoint": S[-1],
                                    "slices": [{"source": S[0], "layers": list(range(0, L, 2))}],
                                    "aux": {"embed_tokens": S[0]}}))
    if L >= 2:
        out.append(("move", {"num_ranks": N, "base_checkpoint": S[0],
                             "slices": [{"source": S[-1], "layers": [0, 1], "targets": [L - 1, L - 2]}]}))
    return out


def main():
    if not TOOL.exists():
        raise SystemExit("build oracle/_ref first (make -C oracle)")
    merge, score = {}, {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, spec, N, K in SOURCES:
            src = pathlib.Path(tmp) / name
            tool("gen", *spec_args(spec), "--ranks", N, "--snapshots", K, "--out", src)
            base = str(src)
            entry = {"spec": spec, "ranks": N, "snapshots": K, "sources": {}, "merges": {}}
            for k in range(1, K + 1):
                entry["sources"][f"checkpoint-{k * 100}"] = tree_digest(src / f"checkpoint-{k * 100}")
            for rname, recipe in recipes_for(name, spec, N, K):
                rj = json.loads(json.dumps(recipe).replace("<SRC>", base))
                rp = pathlib.Path(tmp) / f"{name}-{rname}.json"
                rp.write_text(json.dumps(rj))
                out = pathlib.Path(tmp) / f"{name}-{rname}-out"
                res = tool("merge", "--recipe", rp, "--out", out)
                entry["merges"][rname] = {"recipe": recipe, "files": tree_digest(out),
                                          "shard_files_read": res["stats"]["shard_files_read"],
                                          "weight_files_read": res["stats"]["weight_files_read"],
                                          "group_copies": len(res["plan"]["group_copies"])}
                # manifest provenance embeds absolute source paths: store the relative text too
                entry["merges"][rname]["manifest"] = rel((out / "manifest.json").read_text(), base)
            merge[name] = entry
            if K >= 2:
                snaps = ",".join(str(src / f"checkpoint-{k * 100}") for k in range(1, K + 1))
                s = tool("score", "--snapshots", snaps, "--rho", "0.5")
                s["recipe"] = json.loads(rel(json.dumps(s["recipe"]), base))
                s.pop("score_ms", None)
                score[name] = {"spec": spec, "ranks": N, "snapshots": K, "result": s}
    (OUT / "merge_golden.json").write_text(json.dumps(merge, indent=1, sort_keys=True) + "\n")
    (OUT / "score_golden.json").write_text(json.dumps(score, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT / "merge_golden.json", OUT / "score_golden.json")


if __name__ == "__main__":
    sys.exit(main())
