"""Byte-for-byte parity against the reference binary (oracle/_ref/ref_tool, the
reference library compiled from its own sources) at BASELINE.json's named shapes:

* cfg1 exactly (configs[0]): tiny Llama-style L4 h256 f688 v32000, 1 ZeRO rank,
  2 sources, half-layer merge — both the magnitude selection (select -> merge) and
  the explicit alternating half-layer recipe of SURVEY §8(d);
* cfg3's per-layer shape (configs[2]): one Llama-3.1-8B decoder layer (h4096,
  f14336) over 8 ZeRO ranks, 4 snapshots, rho 0.5 select -> merge (vocabulary cut
  to 256 so that the reference's CPU path finishes in about a minute).

Every output file (weights, all rank shards, the four sidecars) is compared by
sha256 with the reference's; scores within 1e-6 relative; recipes equal.
Anchors: R/src/merge.cpp:226-357 (execute_merge), R/tests/test_merge.cpp:100-139.
"""
import hashlib
import json
import pathlib

import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
from conftest import ref_tool  # noqa: E402

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-6


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def tree_digest(root: pathlib.Path):
    return {str(p.relative_to(root)): hashlib.sha256(p.read_bytes()).hexdigest()
            for p in sorted(root.rglob("*")) if p.is_file()}


def spec_cli(spec: t.ModelSpec):
    out = ["--layers", spec.num_layers, "--hidden", spec.hidden_dim, "--ffn", spec.ffn_dim, "--vocab", spec.vocab_size,
           "--seed", spec.seed]
    return out + (["--tied"] if spec.weight_tied else [])


def select_merge_both(tmp: pathlib.Path, dirs, rho=0.5, workers=0):
    """reference select-merge vs tg_select_recipe + tg_execute_merge on the same snapshot dirs."""
    ref = ref_tool("select-merge", "--snapshots", ",".join(dirs), "--rho", rho, "--out", tmp / "ref_out",
                   "--workers", workers)[1]
    rec, src, gap = t.select_recipe(dirs, rho)
    _, scores = t.score_snapshots(dirs)
    for p, row in enumerate(ref["scores"]):
        for m, v in enumerate(row):
            assert scores[p][m] == pytest.approx(v, rel=SCORE_RTOL), (p, m)
    assert rec == t.MergeRecipe.from_json(json.dumps(ref["recipe"]))
    assert gap == pytest.approx(ref["min_boundary_gap"], rel=1e-6)
    st = t.execute_merge(rec, str(tmp / "our_out"), t.MergeOptions(workers=workers))
    assert tree_digest(tmp / "ref_out") == tree_digest(tmp / "our_out")
    assert st.shard_files_read == ref["merge"]["stats"]["shard_files_read"]
    assert st.weight_files_read == ref["merge"]["stats"]["weight_files_read"]
    # the combined call (tg_select_merge): the composite's masters come from the scorer's
    # device copies, the bytes written are the reference's
    rec2, src2, gap2, st2 = t.select_merge(dirs, str(tmp / "our_sm"), rho, t.MergeOptions(workers=workers))
    assert rec2 == rec and src2 == src and gap2 == gap
    assert tree_digest(tmp / "ref_out") == tree_digest(tmp / "our_sm")
    assert st2.resident_bytes > 0
    assert st2.shard_files_read == st.shard_files_read and st2.weight_files_read == st.weight_files_read
    return ref, rec, src


def test_cfg1_exact_select_merge_and_half_layer_recipe(tmp_path):
    """BASELINE configs[0] at its exact shape: L4 h256 f688 v32000, N=1, K=2."""
    need_gpu()
    spec = t.ModelSpec(4, 256, 688, 32000, False, 42)
    dirs = ref_tool("gen", *spec_cli(spec), "--ranks", 1, "--snapshots", 2, "--out", tmp_path / "run")[1]["snapshots"]
    ref, rec, src = select_merge_both(tmp_path / "sel", dirs)
    assert len(src) == 7 and set(src) <= {0, 1}
    # SURVEY §8(d) cfg1 recipe: layers {0, 2} from S_1; {1, 3} and the aux modules from S_2
    half = t.MergeRecipe(num_ranks=1, base_checkpoint=dirs[1],
                         slices=[t.RecipeSlice(dirs[0], [0, 2]), t.RecipeSlice(dirs[1], [1, 3])])
    (tmp_path / "half.json").write_text(half.to_json())
    ref_tool("merge", "--recipe", tmp_path / "half.json", "--out", tmp_path / "half_ref")
    st = t.execute_merge(half, str(tmp_path / "half_ours"))
    assert tree_digest(tmp_path / "half_ref") == tree_digest(tmp_path / "half_ours")
    assert st.bytes_moved == 19_548_416 * 14  # every composite byte: 2 B weights + 12 B optimizer state per param


def test_cfg3_layer_shape_select_merge_8_ranks(tmp_path):
    """BASELINE configs[2] at its per-layer shape: one h4096 f14336 decoder layer, 8 ZeRO
    ranks, 4 snapshots, rho 0.5 (243 M decay-group elements per snapshot: every rank
    chunk of the big group is 30.4 M elements). Sources are written by the device writer;
    its snapshot 1 is first checked against the reference writer byte for byte."""
    need_gpu()
    spec = t.ModelSpec(1, 4096, 14336, 256, False, 42)
    N, K = 8, 4
    fam = t.SynthFamily(spec, N, K, 100)
    run = tmp_path / "run"
    dirs = [str(run / f"checkpoint-{k * 100}") for k in range(1, K + 1)]
    for k in range(1, K + 1):
        fam.write_dir(k, dirs[k - 1])
    ref1 = ref_tool("gen", *spec_cli(spec), "--ranks", N, "--snapshots", 1, "--out", tmp_path / "ref1")[1]["snapshots"][0]
    assert tree_digest(pathlib.Path(ref1)) == tree_digest(pathlib.Path(dirs[0]))
    ref, rec, src = select_merge_both(tmp_path / "sel", dirs, workers=8)
    assert len(src) == 4 and max(src) == K - 1  # the last snapshot contributes
