"""INTEGRATION.md compiled: the reference-side binding a maintainer would add.

* tests/integration/cmd_merge_b200.cpp — the reference's `tailor merge`
  (R/tools/tailor_main.cpp:75-103, exit codes :351-357) with its body on
  tg_execute_merge, built against the reference's own headers and library;
* tests/integration/device_flow.c — plain C, the device-resident flow of §4 over a
  tg_layout built from checkpoint directories (no synthetic family).
Both are built by __graft_entry__.build() (tests/integration/Makefile)."""
import json
import pathlib
import subprocess

import pytest

from conftest import ref_tool, spec_args

ROOT = pathlib.Path(__file__).resolve().parents[1]
BUILD = ROOT / "tests" / "integration" / "_build"
SHIM, FLOW = BUILD / "cmd_merge_b200", BUILD / "device_flow"
SPEC = dict(num_layers=3, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=5)


def need(path):
    if not path.exists():
        pytest.skip(f"{path.name} not built (tests/integration/Makefile)")


def tree(root: pathlib.Path):
    return {str(p.relative_to(root)): p.read_bytes() for p in sorted(root.rglob("*")) if p.is_file()}


def test_binaries_link_the_c_abi_dynamically():
    for p in (SHIM, FLOW):
        need(p)
        out = subprocess.run(["nm", "-D", "--undefined-only", str(p)], capture_output=True, text=True).stdout
        assert "tg_" in out and "libtailor_b200.so" in subprocess.run(["ldd", str(p)], capture_output=True,
                                                                       text=True).stdout


@pytest.mark.parametrize("yaml_text,kind", [
    ("merge_method: linear\nnum_ranks: 1\n", "RecipeError"),
    ("merge_method: passthrough\nnum_ranks: 1\nslices: [{source: /nonexistent/ckpt, layers: [0]}]\n", "MissingArtifact"),
])
def test_shim_maps_user_errors_to_exit_1_without_a_gpu(tmp_path, yaml_text, kind):
    """Recipe / artifact errors surface before any device work, through TailorError and the
    reference's exit-code mapping."""
    need(SHIM)
    r = tmp_path / "r.yaml"
    r.write_text(yaml_text)
    p = subprocess.run([str(SHIM), "merge", "--recipe", str(r), "--out", str(tmp_path / "o")], capture_output=True,
                       text=True)
    assert p.returncode == 1 and f"error: {kind}: " in p.stderr and f"{kind}: {kind}" not in p.stderr, p.stderr


def test_shim_missing_recipe_file_is_the_reference_helpers_error(tmp_path):
    need(SHIM)
    p = subprocess.run([str(SHIM), "merge", "--recipe", str(tmp_path / "nope.yaml"), "--out", str(tmp_path / "o")],
                       capture_output=True, text=True)
    assert p.returncode == 1 and "MissingArtifact" in p.stderr, p.stderr


@pytest.mark.gpu
def test_shim_merge_equals_reference_merge(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    need(SHIM)
    d = ref_tool("gen", *spec_args(SPEC), "--ranks", 2, "--snapshots", 2, "--out", tmp_path / "run")[1]["snapshots"]
    rec = {"merge_method": "passthrough", "num_ranks": 2, "base_checkpoint": d[1],
           "slices": [{"source": d[0], "layers": [0, 2]}]}
    (tmp_path / "r.json").write_text(json.dumps(rec))
    ref = ref_tool("merge", "--recipe", tmp_path / "r.json", "--out", tmp_path / "ref")[1]
    (tmp_path / "r.yaml").write_text(
        f"merge_method: passthrough\nnum_ranks: 2\nbase_checkpoint: {d[1]}\nslices:\n  - source: {d[0]}\n    layers: [0, 2]\n")
    p = subprocess.run([str(SHIM), "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "ours"),
                        "--json"], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout)
    assert set(out) == {"out", "num_ranks", "num_sources", "shard_files_read", "weight_files_read", "wall_ms"}
    assert out["shard_files_read"] == ref["stats"]["shard_files_read"]
    assert out["weight_files_read"] == ref["stats"]["weight_files_read"]
    assert tree(tmp_path / "ref") == tree(tmp_path / "ours")
    # a second merge into the same directory is refused as the reference does (StorageError, exit 2)
    p = subprocess.run([str(SHIM), "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "ours")],
                       capture_output=True, text=True)
    assert p.returncode == 2 and "StorageError" in p.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("N,K", [(1, 2), (4, 4)])
def test_device_flow_over_a_layout_from_checkpoints(tmp_path, N, K):
    """§4 without a family: scores, selection and every composite payload file equal the
    reference's select -> merge on the same directories."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    need(FLOW)
    spec = dict(SPEC, num_layers=4, seed=100 + N)
    d = ref_tool("gen", *spec_args(spec), "--ranks", N, "--snapshots", K, "--out", tmp_path / "run")[1]["snapshots"]
    p = subprocess.run([str(FLOW), str(tmp_path / "flow"), "0.5", *d], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    import paper_2602_22158_b200 as t

    ref = ref_tool("score", "--snapshots", ",".join(d), "--rho", "0.5")[1]
    recipe = (tmp_path / "flow.recipe.yaml").read_text()
    assert t.parse_recipe(recipe) == t.MergeRecipe.from_json(json.dumps(ref["recipe"]))
    (tmp_path / "r.json").write_text(json.dumps(ref["recipe"]))
    ref_tool("merge", "--recipe", tmp_path / "r.json", "--out", tmp_path / "ref")
    ours = tree(tmp_path / "flow")
    theirs = tree(tmp_path / "ref")
    assert set(ours) == {"model.weights", *(f"optim/rank_{r}.shard" for r in range(N))}
    for name, data in ours.items():
        assert data == theirs[name], name


def test_reader_pool_host_reads(tmp_path):
    """tests/integration/readpool_test.cpp: the file drop-ins' reader pool (lookahead
    batches, oversize pieces, O_DIRECT congruent and bounce paths, failure isolation,
    drain, destruction with queued work) — host only, no GPU."""
    exe = BUILD / "readpool_test"
    need(exe)
    p = subprocess.run([str(exe), str(tmp_path / "data.bin")], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "readpool ok" in p.stdout
