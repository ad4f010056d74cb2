"""Host-side logic of the B200 engine (C++ behind the C ABI, no GPU needed):
recipe schema, layer map, plan resolution, auto-recipes, container layouts,
selection — each against the oracle or the reference binary."""
import json
import random

import numpy as np

import pytest

import paper_2602_22158_b200 as t
import tailor_oracle as o
from conftest import REF_TOOL, ref_tool, spec_args


def ospec(s):
    return dict(num_layers=s.num_layers, hidden_dim=s.hidden_dim, ffn_dim=s.ffn_dim, vocab_size=s.vocab_size,
                weight_tied=s.weight_tied, seed=s.seed)


# ---- recipe schema: literals of R/tests/test_recipe.cpp:23-118 ----------------------------
PARITY_YAML = """
merge_method: passthrough
num_ranks: 4
slices:
  - source: ckpt-100
    layers: [0, 2]
  - source: ckpt-200
    layers: [1, 3]
aux:
  embed_tokens: ckpt-100
  norm: ckpt-200
  lm_head: ckpt-200
config_from: ckpt-200
"""


def test_parity_recipe_parses():
    r = t.parse_recipe(PARITY_YAML)
    assert r.num_ranks == 4 and len(r.slices) == 2
    assert r.slices[0].source == "ckpt-100" and r.slices[0].layers == [0, 2] and r.slices[0].targets == [0, 2]
    assert r.aux == {"embed_tokens": "ckpt-100", "norm": "ckpt-200", "lm_head": "ckpt-200"}
    assert r.config_from == "ckpt-200" and r.base_checkpoint == ""


def test_base_only_defaults_config_from_latest():
    r = t.parse_recipe("merge_method: passthrough\nbase_checkpoint: c\nnum_ranks: 1\n")
    assert r.base_checkpoint == "c" and r.slices == [] and r.config_from == "latest"


def test_ranges_half_open_and_targets():
    r = t.parse_recipe("merge_method: passthrough\nnum_ranks: 2\nslices:\n  - source: c\n    layers: {start: 1, end: 4}\n")
    assert r.slices[0].layers == [1, 2, 3]
    r = t.parse_recipe("merge_method: passthrough\nnum_ranks: 2\nslices:\n  - source: c\n    layers: [0, 1]\n    targets: [2, 3]\n")
    assert r.slices[0].targets == [2, 3]


@pytest.mark.parametrize("text,layers", [("010", [8]), ("0x10", [16]), ("+4", [4]), ("0", [0]), ("12", [12])])
def test_integers_convert_like_yaml_cpp(text, layers):
    """node.as<int>() (R/src/recipe.cpp:28-35) is yaml-cpp's stream conversion with
    std::ios::dec unset: a leading 0 means octal and 0x hexadecimal."""
    r = t.parse_recipe(f"merge_method: passthrough\nnum_ranks: 1\nslices:\n  - source: c\n    layers: [{text}]\n")
    assert r.slices[0].layers == layers


@pytest.mark.parametrize("text", ["08", "0x", "1.0", "4294967296", "1e3"])
def test_non_integers_are_recipe_errors_like_yaml_cpp(text):
    with pytest.raises(t.TailorError) as e:
        t.parse_recipe(f"merge_method: passthrough\nnum_ranks: 1\nslices:\n  - source: c\n    layers: [{text}]\n")
    assert e.value.kind == t.ErrorKind.Recipe


@pytest.mark.parametrize("text", [
    "merge_method: passthrough\nnum_ranks: 2\nextra_key: 1\n",
    "num_ranks: 2\n",
    "merge_method: linear\nnum_ranks: 2\n",
    "merge_method: passthrough\n",
    "merge_method: passthrough\nnum_ranks: 0\n",
    "merge_method: passthrough\nnum_ranks: 2\naux: {embedding: c}\n",
    "merge_method: passthrough\nnum_ranks: 2\nslices: [{layers: [0]}]\n",
    "merge_method: passthrough\nnum_ranks: 2\nslices: [{source: c, layers: [0], targets: [0, 1]}]\n",
    "merge_method: passthrough\nnum_ranks: 2\nslices: [{source: c, layers: {start: 3, end: 3}}]\n",
    ": not yaml: [",
    "merge_method: passthrough\nnum_ranks: two\n",
    "merge_method: passthrough\nnum_ranks: 2\nslices: [{source: c, layers: [-1]}]\n",
])
def test_schema_violations_are_recipe_errors(text):
    with pytest.raises(t.TailorError) as e:
        t.parse_recipe(text)
    assert e.value.kind == t.ErrorKind.Recipe


def test_error_names_offending_field():
    with pytest.raises(t.TailorError) as e:
        t.parse_recipe("merge_method: passthrough\nnum_ranks: 2\nslices: [{source: c, layers: [0], bogus: 1}]\n")
    assert "slices[0].bogus" in str(e.value)


def test_yaml_round_trip():
    r = t.MergeRecipe(num_ranks=4, base_checkpoint="run/checkpoint-400",
                      slices=[t.RecipeSlice("run/checkpoint-300", [0, 2]), t.RecipeSlice("run/checkpoint-200", [1], [3])],
                      aux={"embed_tokens": "run/checkpoint-300", "norm": "run/checkpoint-200"},
                      config_from="run/checkpoint-400")
    assert t.parse_recipe(t.recipe_to_yaml(r)) == r
    odd = t.MergeRecipe(num_ranks=1, base_checkpoint="a path: with colon #x", config_from="latest")
    assert t.parse_recipe(t.recipe_to_yaml(odd)) == odd


# ---- layer map vs the oracle ----------------------------------------------------------------
@pytest.mark.parametrize("spec,N", [(t.ModelSpec(4, 8, 16, 32), 4), (t.ModelSpec(3, 4, 4, 8, True), 3),
                                    (t.ModelSpec(32, 4096, 14336, 128256), 8), (t.ModelSpec(80, 8192, 28672, 128256), 8)])
def test_layer_map_matches_oracle(spec, N):
    lm = t.layer_map(spec, N)
    s = ospec(spec)
    assert lm["parameters"] == o.parameter_count(s)
    assert [m["name"] for m in lm["modules"]] == o.modules(s)
    offs = o.module_offsets(s)
    for m in lm["modules"]:
        assert m["model_offset"] == offs[m["name"]]
        assert m["groups"] == o.group_indices_for(s, m["name"])
        assert [(x["name"], tuple(x["shape"]), x["decay"]) for x in m["tensors"]] == o.tensors_of(s, m["name"])
    table = o.group_table(s)
    assert len(lm["groups"]) == len(table)
    for g in lm["groups"]:
        owner, decay, n = table[g["index"]]
        assert (g["owner"], g["decay"], g["true_length"]) == (owner, decay, n)
        assert g["shard_length"] == o.shard_length(n, N) and g["padded_length"] == N * o.shard_length(n, N)
        assert [(x["name"], x["group_offset"], x["model_offset"]) for x in g["slices"]] == \
               [(a, c, d) for a, _, c, d in o.group_slices(s, g["index"])]


def test_named_configs_sizes():
    # params and group counts of the named configs
    assert t.layer_map(t.ModelSpec(4, 256, 688, 32000), 1)["parameters"] == 19_548_416
    assert t.layer_map(t.ModelSpec(28, 3584, 18944, 152064), 8)["parameters"] == 8_232_050_176
    lm = t.layer_map(t.ModelSpec(32, 4096, 14336, 128256), 8)
    assert lm["parameters"] == 8_835_567_616 and len(lm["groups"]) == 67
    assert t.layer_map(t.ModelSpec(80, 8192, 28672, 128256), 8)["parameters"] == 79_948_947_456


# ---- container layouts (headers) vs the oracle, via device-free plans ---------------------------
@pytest.mark.parametrize("spec,N", [(t.ModelSpec(4, 8, 16, 32), 4), (t.ModelSpec(3, 4, 4, 8, True), 3),
                                    (t.ModelSpec(2, 6, 10, 11), 2)])
def test_partition_plans_headers_and_coverage(spec, N):
    K = 3
    fam = t.SynthFamily(spec, N, K)
    rng = random.Random(N)
    s = ospec(spec)
    mods = o.modules(s)
    recipe = t.MergeRecipe(num_ranks=N, base_checkpoint="S3",
                           slices=[t.RecipeSlice("S1", [0]), t.RecipeSlice("S2", list(range(1, spec.num_layers)))],
                           aux={"embed_tokens": "S1"})
    yaml = recipe.to_yaml()
    groups = list(range(len(o.group_table(s))))
    for r in range(N):
        mp = t.MergePartition(fam, yaml, r)
        prefix, _, size = o.container_layout(o.shard_decls(s, N, groups), {"num_ranks": str(N), "rank": str(r)})
        assert mp.prefix() == prefix and mp.bytes == size
        assert fam.shard_bytes(1, r) == size
        assert all(c == r for _, c, _, _ in mp.windows())
    wprefix, _, wsize = o.container_layout(o.weight_decls(s, mods))
    covered = []
    for units in (1, 2, 5):
        covered = []
        for u in range(units):
            mp = t.MergePartition(fam, yaml, -1, u, units)
            lo, hi, total = mp.range()
            assert total == wsize and mp.prefix() == wprefix
            covered.append((lo, hi))
        assert covered[0][0] == 0 and covered[-1][1] == wsize
        assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
    # shard sub-units (host-staged cfg5 units): tile the rank payload at tensor boundaries,
    # windows shrink to what the sub-range reads
    full = t.MergePartition(fam, yaml, 0)
    fl, fh, ftot = full.range()
    assert (fl, fh) == (0, ftot)
    for units in (2, 3, 7):
        parts = [t.MergePartition(fam, yaml, 0, u, units) for u in range(units)]
        rs = [p.range() for p in parts]
        assert rs[0][0] == 0 and rs[-1][1] == ftot and all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert sum(p.bytes for p in parts) == full.bytes
        assert all(p.prefix() == full.prefix() for p in parts)
        assert sum(p.num_segments for p in parts) >= full.num_segments
        for p, (lo, hi, _) in zip(parts, rs):
            for k, c, wlo, whi in p.windows():
                assert c == 0 and whi - wlo <= hi - lo


def test_plan_errors_match_reference_kinds():
    spec = t.ModelSpec(4, 8, 16, 32)
    fam = t.SynthFamily(spec, 2, 2)
    fam.set_partial(2, ["layers.0", "norm"])
    cases = [
        (t.MergeRecipe(num_ranks=2, slices=[t.RecipeSlice("S1", [0, 1, 2, 3])], aux={"embed_tokens": "S1", "norm": "S1"}),
         t.ErrorKind.Recipe),  # lm_head uncovered, no base
        (t.MergeRecipe(num_ranks=2, base_checkpoint="S1", slices=[t.RecipeSlice("S1", [0, 1], [2, 2])]), t.ErrorKind.Recipe),
        (t.MergeRecipe(num_ranks=3, base_checkpoint="S1"), t.ErrorKind.Geometry),
        (t.MergeRecipe(num_ranks=2, base_checkpoint="S1", slices=[t.RecipeSlice("S2", [2])]), t.ErrorKind.SourceLacksModule),
        (t.MergeRecipe(num_ranks=2, base_checkpoint="S1", slices=[t.RecipeSlice("S1", [7])]), t.ErrorKind.Recipe),
        (t.MergeRecipe(num_ranks=2, base_checkpoint="nope"), t.ErrorKind.MissingArtifact),
    ]
    for rec, kind in cases:
        with pytest.raises(t.TailorError) as e:
            t.MergePartition(fam, rec.to_yaml(), 0)
        assert e.value.kind == kind, rec


# ---- against the reference binary on reference-written checkpoints --------------------------------
def _need_ref():
    if not REF_TOOL.exists():
        pytest.skip("reference binary not built")


def test_resolve_plan_matches_reference(tmp_path):
    _need_ref()
    spec = dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=909)
    d = ref_tool("gen", *spec_args(spec), "--ranks", 4, "--snapshots", 3, "--out", tmp_path / "run")[1]["snapshots"]
    recipes = [
        t.MergeRecipe(num_ranks=4, slices=[t.RecipeSlice(d[0], [0, 2]), t.RecipeSlice(d[1], [1, 3])],
                      aux={"embed_tokens": d[0], "norm": d[1], "lm_head": d[1]}),
        t.MergeRecipe(num_ranks=4, base_checkpoint=d[2], slices=[t.RecipeSlice(d[0], [0, 1], [3, 2])], config_from=d[0]),
        t.MergeRecipe(num_ranks=4, base_checkpoint=d[1], aux={"norm": d[2]}),
    ]
    for rec in recipes:
        (tmp_path / "r.json").write_text(rec.to_json())
        assert t.resolve_plan(rec) == ref_tool("resolve", "--recipe", tmp_path / "r.json")[1]["plan"]


@pytest.mark.parametrize("strategy,steps,interval,fail_at", [("parity", 100, 25, 110), ("filter", 100, 10, 100),
                                                             ("full", 60, 20, 50)])
def test_recipe_from_manifests_matches_reference(tmp_path, strategy, steps, interval, fail_at):
    _need_ref()
    spec = dict(num_layers=6, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=31415)
    ref_tool("train", *spec_args(spec), "--strategy", strategy, "--steps", steps, "--interval", interval,
             "--ranks", 2, "--out", tmp_path / "run", "--fail-at", fail_at)
    ref = ref_tool("plan", "--run", tmp_path / "run", "--failure-step", fail_at)[1]["recipe"]
    assert t.recipe_from_manifests(str(tmp_path / "run"), fail_at) == t.MergeRecipe.from_json(json.dumps(ref))


@pytest.mark.parametrize("seed", range(6))
def test_resolve_plan_random_recipes_match_reference(tmp_path, seed):
    """Random recipes over reference-written checkpoints — layer moves, duplicate and
    out-of-range layers/targets, missing sources, wrong rank counts, aux/base/config_from
    choices — resolve to the reference's plan or fail with the reference's exact message
    (R/src/merge.cpp:39-152). A 1500-case search found no difference."""
    _need_ref()
    rng = random.Random(seed)
    L, N, K = rng.randrange(1, 7), rng.randrange(1, 4), rng.randrange(1, 5)
    spec = dict(num_layers=L, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=rng.random() < 0.3, seed=seed)
    d = ref_tool("gen", *spec_args(spec), "--ranks", N, "--snapshots", K, "--out", tmp_path / "run")[1]["snapshots"]
    srcs = d + [str(tmp_path / "nope")]
    for case in range(25):
        slices = []
        for _ in range(rng.randrange(0, 4)):
            ls = [rng.randrange(0, L + 1) for _ in range(rng.randrange(1, L + 2))]
            tg = ls if rng.random() < 0.6 else [rng.randrange(0, L + 1) for _ in range(len(ls))]
            slices.append(t.RecipeSlice(rng.choice(srcs) if rng.random() < 0.9 else d[0], ls, tg))
        aux = {m: rng.choice(srcs) for m in ("embed_tokens", "norm", "lm_head") if rng.random() < 0.6}
        rec = t.MergeRecipe(num_ranks=N if rng.random() < 0.85 else N + 1, slices=slices, aux=aux,
                            base_checkpoint=rng.choice(srcs) if rng.random() < 0.5 else "",
                            config_from=rng.choice(["latest"] * 3 + srcs))
        (tmp_path / "r.json").write_text(rec.to_json())
        rc, out, err = ref_tool("resolve", "--recipe", tmp_path / "r.json", check=False)
        if rc == 0:
            assert t.resolve_plan(rec) == out["plan"], case
        else:
            with pytest.raises(t.TailorError) as e:
                t.resolve_plan(rec)
            assert str(e.value) == json.loads(err.strip().splitlines()[-1])["message"], case


@pytest.mark.parametrize("seed", range(16))
def test_recipe_from_manifests_random_runs_match_reference(tmp_path, seed):
    """Random reference training runs (strategy, interval, filter knobs, ranks, tied, an
    injected failure) planned at random failure steps: the same recipe as the reference's
    recipe_from_manifests (R/src/merge.cpp:359-418), or the same error kind."""
    _need_ref()
    rng = random.Random(seed)
    spec = dict(num_layers=rng.randrange(1, 9), hidden_dim=8, ffn_dim=16, vocab_size=32,
                weight_tied=rng.random() < 0.3, seed=100 + seed)
    strategy = rng.choice(["full", "parity", "filter"])
    steps, interval = rng.randrange(10, 121), rng.randrange(3, 31)
    run = tmp_path / "run"
    args = ["train", *spec_args(spec), "--strategy", strategy, "--steps", steps, "--interval", interval,
            "--ranks", rng.randrange(1, 4), "--out", run]
    if strategy == "filter":
        head = rng.randrange(0, min(3, spec["num_layers"] + 1))  # the reference refuses head + tail > L
        tail = rng.randrange(0, min(3, spec["num_layers"] - head + 1))
        args += ["--head", head, "--tail", tail, "--sparse-multiple", rng.randrange(1, 6)]
    if rng.random() < 0.5:
        args += ["--fail-at", rng.randrange(0, steps + 10)]
    ref_tool(*args)
    for fs in sorted({rng.randrange(0, steps + 15) for _ in range(6)} | {steps}):
        rc, out, err = ref_tool("plan", "--run", run, "--failure-step", fs, check=False)
        if rc == 0:
            assert t.recipe_from_manifests(str(run), fs) == t.MergeRecipe.from_json(json.dumps(out["recipe"])), fs
        else:
            kind = json.loads(err.strip().splitlines()[-1])["error"]
            with pytest.raises(t.TailorError) as e:
                t.recipe_from_manifests(str(run), fs)
            assert str(e.value).startswith(kind), (fs, kind, str(e.value))


def test_parse_config_reads_reference_config(tmp_path):
    _need_ref()
    spec = dict(num_layers=3, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=True, seed=77)
    d = ref_tool("gen", *spec_args(spec), "--ranks", 2, "--snapshots", 1, "--out", tmp_path / "run")[1]["snapshots"]
    got = t.ModelSpec.from_config((tmp_path / "run" / d[0] / "config.json").read_text()
                                  if not d[0].startswith("/") else open(d[0] + "/config.json").read())
    assert got == t.ModelSpec(3, 8, 16, 32, True, 77)
    for bad in ["", "{", '{"num_layers": 2}', '{"num_layers": "x", "hidden_dim": 8, "ffn_dim": 16, '
                '"vocab_size": 32, "tie_word_embeddings": false, "seed": 1}']:
        with pytest.raises(t.TailorError):
            t.ModelSpec.from_config(bad)


def test_recipe_from_manifests_unrecoverable(tmp_path):
    _need_ref()
    spec = dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=5)
    ref_tool("train", *spec_args(spec), "--strategy", "parity", "--steps", 50, "--interval", 25, "--ranks", 1,
             "--out", tmp_path / "run")
    with pytest.raises(t.TailorError) as e:
        t.recipe_from_manifests(str(tmp_path / "run"), 30)  # only the odd-counter set exists
    assert e.value.kind == t.ErrorKind.UnrecoverableModule
    with pytest.raises(t.TailorError) as e:
        t.recipe_from_manifests(str(tmp_path / "run"), 10)
    assert e.value.kind == t.ErrorKind.UnrecoverableModule


# ---- selection (a14): C++ vs the oracle on random partial sums ---------------------------------
@pytest.mark.parametrize("seed", range(8))
def test_selection_matches_oracle(seed):
    rng = random.Random(seed)
    L = 1 + rng.randrange(10)
    spec = t.ModelSpec(L, 8, 16, 32, rng.random() < 0.3, seed)
    K = 2 + rng.randrange(5)
    nranks = 1 + rng.randrange(4)
    fam = t.SynthFamily(spec, nranks, K)
    M = fam.num_modules
    parts = [rng.uniform(0.0, 1.0) * 10 ** rng.randrange(-3, 3) for _ in range(nranks * (K - 1) * M * 2)]
    if seed % 3 == 0:  # exact ties -> lower canonical index wins
        parts = [round(x, 1) for x in parts]
    rho = rng.choice([0.25, 0.5, 0.7, 1.0])
    yaml, src, scores, gap = fam.select(parts, nranks, rho)
    sc = []
    for p in range(K - 1):
        row = []
        for m in range(M):
            sd = sr = 0.0
            for r in range(nranks):  # sequential rank-order FP64 (Python's sum() is compensated)
                sd += parts[((r * (K - 1) + p) * M + m) * 2]
                sr += parts[((r * (K - 1) + p) * M + m) * 2 + 1]
            row.append(o.magnitude_score(sd, sr))
        sc.append(row)
    assert scores == sc
    _, ref_src, ref_gap = o.select(sc, M, rho)
    assert src == ref_src
    rec = t.parse_recipe(yaml)
    assert rec.base_checkpoint == f"S{K}" and rec.config_from == f"S{K}"
    mods = o.modules(ospec(spec))
    got = {}
    for s in rec.slices:
        for a in s.layers:
            got[f"layers.{a}"] = s.source
    got.update(rec.aux)
    for i, m in enumerate(mods):
        assert got.get(m, f"S{K}") == f"S{ref_src[i] + 1}"


# ---- acceptance c4 on the planning layer (R/tests/acceptance.cpp:244-254), no device ---------------
def _random_recipe(rng, spec, K):
    """Random recipe over sources S1..SK: every layer from a random source, optionally
    moved to a permuted target position; every non-layer module from a random source."""
    mods = o.modules(ospec(spec))
    L = spec.num_layers
    targets = list(range(L))
    if rng.random() < 0.4:
        rng.shuffle(targets)
    assign, slices = {}, {}
    for i in range(L):
        k = rng.randrange(1, K + 1)
        assign[f"layers.{targets[i]}"] = (f"S{k}", f"layers.{i}")
        slices.setdefault(k, ([], []))
        slices[k][0].append(i)
        slices[k][1].append(targets[i])
    recipe = t.MergeRecipe(num_ranks=0)
    for k, (ls, ts) in sorted(slices.items()):
        recipe.slices.append(t.RecipeSlice(f"S{k}", ls, ts))
    for m in mods:
        if not m.startswith("layers."):
            k = rng.randrange(1, K + 1)
            assign[m] = (f"S{k}", m)
            recipe.aux[m] = f"S{k}"
    return recipe, assign


@pytest.mark.parametrize("case", range(200))
def test_plan_segments_reassemble_the_reference_composite(case):
    """200 random merges (random L<=8, h, f, v, tied, N<=5, K<=3, layer moves): applying the
    plan's byte segments (what K2 copies) to random source payloads gives exactly the
    composite the reference assembly produces (oracle merge_payloads restates
    R/src/merge.cpp:244-303), for every rank partition and for the weights payload split
    into 1 and 3 tensor-aligned shares; headers equal the reference's."""
    rng = random.Random(7000 + case)
    spec = t.ModelSpec(1 + rng.randrange(8), 4 << rng.randrange(2), 4 << rng.randrange(3), 8 << rng.randrange(3),
                       rng.random() < 0.5, 100 + case)
    N, K = 1 + rng.randrange(5), 1 + rng.randrange(3)
    s = ospec(spec)
    fam = t.SynthFamily(spec, N, K)
    recipe, assign = _random_recipe(rng, spec, K)
    recipe.num_ranks = N
    if rng.random() < 0.3:
        recipe.base_checkpoint = f"S{K}"
    yaml = recipe.to_yaml()
    nprng = np.random.default_rng(case)
    mods = o.modules(s)
    sources = {f"S{k}": (nprng.integers(0, 256, fam.weights_bytes(k), dtype=np.uint8).tobytes(),
                         [nprng.integers(0, 256, fam.shard_bytes(k, r), dtype=np.uint8).tobytes() for r in range(N)],
                         mods) for k in range(1, K + 1)}
    exp_w, exp_r, wprefix, rprefixes = o.merge_payloads(s, N, assign, sources)

    def apply(mp):
        out = bytearray(mp.bytes)
        wins = mp.windows()
        for w, so, do, n in mp.segments():
            k, c, lo, hi = wins[w]
            assert lo + so + n <= hi
            src = sources[f"S{k}"][0] if c < 0 else sources[f"S{k}"][1][c]
            out[do:do + n] = src[lo + so:lo + so + n]
        return bytes(out)

    for r in range(N):
        mp = t.MergePartition(fam, yaml, r)
        assert mp.prefix() == rprefixes[r]
        assert apply(mp) == exp_r[r], f"rank {r}"
    for units in (1, 3):
        got = b""
        for u in range(units):
            mp = t.MergePartition(fam, yaml, -1, u, units)
            assert mp.prefix() == wprefix
            got += apply(mp)
        assert got == exp_w, f"weights in {units} shares"


def test_damaged_sidecars_fail_like_the_reference(tmp_path):
    """A reference-written checkpoint with one file damaged (deleted, truncated, a byte
    changed, a JSON field retyped, junk appended) used as a recipe's base: the same plan or
    the same error message as the reference (read_checkpoint_summary,
    R/src/checkpoint.cpp:387-428, via resolve_plan). Where the reference aborts
    (std::terminate on invalid UTF-8 inside its error path) ours reports CorruptContainer.
    A 600-case search: 567 identical, 33 reference aborts."""
    _need_ref()
    import shutil

    spec = dict(num_layers=3, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=3)
    src = ref_tool("gen", *spec_args(spec), "--ranks", 2, "--snapshots", 1, "--out", tmp_path / "run")[1]["snapshots"][0]
    rng = random.Random(1)
    for case in range(150):
        work = tmp_path / f"c{case}"
        shutil.copytree(src, work)
        f = rng.choice(sorted(p for p in work.rglob("*") if p.is_file()))
        op, b = rng.randrange(5), f.read_bytes()
        if op == 0:
            f.unlink()
        elif op == 1:
            f.write_bytes(b[:rng.randrange(0, max(1, len(b)))])
        elif op == 2 and b:
            i = rng.randrange(min(len(b), 4096))
            f.write_bytes(b[:i] + bytes([rng.randrange(256)]) + b[i + 1:])
        elif op == 3 and f.suffix == ".json":
            j = json.loads(b)
            j[rng.choice(sorted(j))] = rng.choice([None, "x", -1, 1.5, [], {}])
            f.write_text(json.dumps(j))
        else:
            f.write_bytes(b + b"junk")
        rec = t.MergeRecipe(num_ranks=2, base_checkpoint=str(work))
        (tmp_path / "r.json").write_text(rec.to_json())
        rc, out, err = ref_tool("resolve", "--recipe", tmp_path / "r.json", check=False)
        if rc == 0:
            assert t.resolve_plan(rec) == out["plan"], case
            continue
        with pytest.raises(t.TailorError) as e:
            t.resolve_plan(rec)
        if rc < 0:  # the reference aborted
            assert e.value.kind == t.ErrorKind.CorruptContainer, (case, str(e.value))
            continue
        ej = json.loads(err.strip().splitlines()[-1])
        want = ("internal error: " + ej["message"]) if ej["error"] == "internal" else ej["message"]
        assert str(e.value) == want, case
        shutil.rmtree(work)
