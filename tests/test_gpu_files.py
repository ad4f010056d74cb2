"""File-level drop-in behaviour vs the reference binary: error kinds on corrupt /
missing / incompatible sources, the CLI (exit codes, --json), hyperparameter and
config provenance, tied models. Every successful merge is compared file by file."""
import json
import pathlib
import os
import shutil
import subprocess

import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
from conftest import ref_tool, spec_args  # noqa: E402

pytestmark = pytest.mark.gpu


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def gen(tmp, spec, N, K, name="run"):
    return ref_tool("gen", *spec_args(spec), "--ranks", N, "--snapshots", K, "--out", tmp / name)[1]["snapshots"]


def ref_error(recipe, out):
    p = out.parent / (out.name + ".json")
    p.write_text(recipe.to_json())
    rc, _, err = ref_tool("merge", "--recipe", p, "--out", out, check=False)
    return rc, json.loads(err.strip().splitlines()[-1])["error"] if rc else None


def our_error(recipe, out):
    try:
        t.execute_merge(recipe, str(out))
    except t.TailorError as e:
        return e
    return None


def same_tree(a, b):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file())
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file())
    assert fa == fb
    for rel in fa:
        assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


SPEC = dict(num_layers=3, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=11)
KIND_NAME = {t.ErrorKind.CorruptContainer: "CorruptContainer", t.ErrorKind.MissingArtifact: "MissingArtifact",
             t.ErrorKind.Geometry: "GeometryError", t.ErrorKind.Storage: "StorageError",
             t.ErrorKind.Consistency: "ConsistencyError", t.ErrorKind.Recipe: "RecipeError"}


@pytest.mark.parametrize("damage", ["truncate_shard", "bad_header_json", "missing_shard", "missing_weights",
                                    "shape_mismatch_header"])
def test_corrupt_sources_fail_like_the_reference(tmp_path, damage):
    need_gpu()
    d = gen(tmp_path, SPEC, 2, 2)
    bad = tmp_path / "bad"
    shutil.copytree(d[0], bad)
    shard = bad / "optim" / "rank_1.shard"
    if damage == "truncate_shard":
        shard.write_bytes(shard.read_bytes()[:-4])
    elif damage == "bad_header_json":
        b = bytearray(shard.read_bytes())
        b[9] = ord("!")
        shard.write_bytes(bytes(b))
    elif damage == "missing_shard":
        shard.unlink()
    elif damage == "missing_weights":
        (bad / "model.weights").unlink()
    elif damage == "shape_mismatch_header":
        b = shard.read_bytes()
        hlen = int.from_bytes(b[:8], "little")
        text = b[8:8 + hlen].decode()
        at = text.index('"shape":[', text.index('"g1.master"'))  # a tensor the recipe reads
        h = text[:at] + '"shape":[1,' + text[at + len('"shape":['):]
        h = h.rstrip(" ")
        h += " " * ((8 - (8 + len(h)) % 8) % 8)
        shard.write_bytes(len(h).to_bytes(8, "little") + h.encode() + b[8 + hlen:])
    recipe = t.MergeRecipe(num_ranks=2, base_checkpoint=d[1], slices=[t.RecipeSlice(str(bad), [0, 2])])
    rc, ref_kind = ref_error(recipe, tmp_path / "ref_out")
    err = our_error(recipe, tmp_path / "our_out")
    assert rc != 0 and err is not None
    assert KIND_NAME.get(err.kind, str(err.kind)) == ref_kind, (err, ref_kind)
    # validation happens before any write, exactly as the reference (no partial output)
    assert not (tmp_path / "our_out").exists() or not any((tmp_path / "our_out").rglob("*.shard"))


def test_coarse_source_is_rejected(tmp_path):
    need_gpu()
    ref_tool("train", *spec_args(SPEC), "--strategy", "full", "--steps", 10, "--interval", 10, "--ranks", 2,
             "--grouping", "coarse", "--out", tmp_path / "coarse")
    recipe = t.MergeRecipe(num_ranks=2, base_checkpoint=str(tmp_path / "coarse" / "checkpoint-10"))
    err = our_error(recipe, tmp_path / "o")
    assert err is not None and err.kind == t.ErrorKind.Geometry
    assert ref_error(recipe, tmp_path / "r")[1] == "GeometryError"


def test_hyper_and_config_provenance(tmp_path):
    """R/tests/test_merge.cpp:241-300: per-group hyper from each module's source; config_from rules."""
    need_gpu()
    for i, lr in enumerate(["0.001", "0.0005"]):
        ref_tool("train", *spec_args(SPEC), "--strategy", "full", "--steps", 10 * (i + 1), "--interval", 10 * (i + 1),
                 "--ranks", 1, "--lr", lr, "--out", tmp_path / f"s{i}")
    a, b = str(tmp_path / "s0" / "checkpoint-10"), str(tmp_path / "s1" / "checkpoint-20")
    for rec, name in [(t.MergeRecipe(num_ranks=1, base_checkpoint=a, slices=[t.RecipeSlice(b, [1])]), "latest"),
                      (t.MergeRecipe(num_ranks=1, base_checkpoint=b, slices=[t.RecipeSlice(a, [0])], config_from=a),
                       "explicit")]:
        ours, refd = tmp_path / f"ours-{name}", tmp_path / f"ref-{name}"
        t.execute_merge(rec, str(ours))
        p = tmp_path / f"{name}.json"
        p.write_text(rec.to_json())
        ref_tool("merge", "--recipe", p, "--out", refd)
        same_tree(refd, ours)
    meta = json.loads((tmp_path / "ours-latest" / "optim_meta.json").read_text())
    lrs = {g["owner"]: g["lr"] for g in meta["groups"] if g["decay"] == "decay"}
    assert lrs["layers.1"] == 0.0005 and lrs["layers.0"] == 0.001
    assert json.loads((tmp_path / "ours-explicit" / "trainer_state.json").read_text())["step"] == 10


def test_cli_merge_plan_select(tmp_path):
    need_gpu()
    cli = str(t.CLI_PATH)
    spec = dict(SPEC, num_layers=4)
    d = gen(tmp_path, spec, 2, 3)
    rec = t.MergeRecipe(num_ranks=2, base_checkpoint=d[2], slices=[t.RecipeSlice(d[0], [0, 2])], aux={"norm": d[1]})
    (tmp_path / "r.yaml").write_text(rec.to_yaml())
    p = subprocess.run([cli, "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "cli"), "--json"],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    js = json.loads(p.stdout)
    assert js["shard_files_read"] == 2 * 3 and js["weight_files_read"] == 3
    # the reference CLI's --json keys (R/tools/tailor_main.cpp:84-91)
    assert {"out", "num_ranks", "num_sources", "shard_files_read", "weight_files_read", "wall_ms"} <= set(js)
    assert js["out"] == str(tmp_path / "cli") and js["num_ranks"] == 2 and js["num_sources"] == 3
    (tmp_path / "r.json").write_text(rec.to_json())
    ref_tool("merge", "--recipe", tmp_path / "r.json", "--out", tmp_path / "ref")
    same_tree(tmp_path / "ref", tmp_path / "cli")
    # text report: the reference's lines (R/tools/tailor_main.cpp:94-101)
    p = subprocess.run([cli, "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "cli_text")],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    lines = p.stdout.splitlines()
    assert lines[0] == f"merged checkpoint written to {tmp_path / 'cli_text'}"
    assert lines[1] == "sources: 3  ranks: 2"
    assert lines[2] == "optimizer shard files read: 6 (bound 2 x 3 = 6 cached)"
    assert lines[3] == "weight files read: 3" and lines[4].startswith("wall time: ")
    # non-empty output directory -> StorageError -> exit 2
    p = subprocess.run([cli, "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "cli")],
                       capture_output=True, text=True)
    assert p.returncode == 2 and "StorageError" in p.stderr
    # select: magnitude strategy -> recipe identical to the reference-side restatement
    p = subprocess.run([cli, "select", "--snapshots", ",".join(d), "--out", str(tmp_path / "sel.yaml")],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    ref = ref_tool("score", "--snapshots", ",".join(d))[1]["recipe"]
    assert t.parse_recipe((tmp_path / "sel.yaml").read_text()) == t.MergeRecipe.from_json(json.dumps(ref))
    # check: device re-verify of a merged checkpoint
    p = subprocess.run([cli, "check", "--ckpt", str(tmp_path / "cli")], capture_output=True, text=True)
    assert p.returncode == 0 and "ok" in p.stdout


def test_tied_merge_has_no_lm_head(tmp_path):
    need_gpu()
    spec = dict(SPEC, weight_tied=True)
    d = gen(tmp_path, spec, 1, 1)
    t.execute_merge(t.MergeRecipe(num_ranks=1, base_checkpoint=d[0]), str(tmp_path / "m"))
    b = (tmp_path / "m" / "model.weights").read_bytes()
    hdr = json.loads(b[8:8 + int.from_bytes(b[:8], "little")])
    assert "lm_head.weight" not in hdr
    man = json.loads((tmp_path / "m" / "manifest.json").read_text())
    assert len(man["modules"]) == 5 and man["strategy"] == "merged" and len(man["provenance"]) == 5


@pytest.mark.parametrize("N,tied", [(1, False), (3, False), (4, True), (8, False)])
def test_regroup_matches_reference(tmp_path, N, tied):
    """f3: coarse -> fine -> coarse through the device gather == reference read/coarse_to_fine/write."""
    need_gpu()
    spec = dict(SPEC, weight_tied=tied, num_layers=4)
    ref_tool("train", *spec_args(spec), "--strategy", "full", "--steps", 20, "--interval", 20, "--ranks", N,
             "--grouping", "coarse", "--out", tmp_path / "run")
    src = tmp_path / "run" / "checkpoint-20"
    ref_tool("regroup", "--dir", src, "--out", tmp_path / "ref_fine")
    st = t.regroup(str(src), str(tmp_path / "fine"), to_fine=True)
    same_tree(tmp_path / "ref_fine", tmp_path / "fine")
    assert st.bytes_moved > 0
    ref_tool("regroup", "--dir", tmp_path / "ref_fine", "--to", "coarse", "--out", tmp_path / "ref_coarse")
    t.regroup(str(tmp_path / "fine"), str(tmp_path / "coarse"), to_fine=False)
    same_tree(tmp_path / "ref_coarse", tmp_path / "coarse")
    same_tree(src, tmp_path / "coarse")  # round trip is the identity on bytes
    # the regrouped (fine) checkpoint is now mergeable
    t.execute_merge(t.MergeRecipe(num_ranks=N, base_checkpoint=str(tmp_path / "fine")), str(tmp_path / "merged"))
    t.verify_checkpoint(str(tmp_path / "coarse"))


def test_regroup_cli_and_errors(tmp_path):
    need_gpu()
    d = gen(tmp_path, SPEC, 2, 1)
    p = subprocess.run([str(t.CLI_PATH), "regroup", "--ckpt", d[0], "--out", str(tmp_path / "c"), "--to", "coarse"],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    ref_tool("regroup", "--dir", d[0], "--to", "coarse", "--out", tmp_path / "rc")
    same_tree(tmp_path / "rc", tmp_path / "c")
    ref_tool("gen", *spec_args(SPEC), "--ranks", 2, "--snapshots", 1, "--out", tmp_path / "part",
             "--partial", "1=layers.0,norm")
    with pytest.raises(t.TailorError) as e:
        t.regroup(str(tmp_path / "part" / "checkpoint-100"), str(tmp_path / "x"))
    assert e.value.kind == t.ErrorKind.MissingModules


@pytest.mark.parametrize("damage", ["negative_v", "weight_bit"])
def test_merge_reverify_catches_bad_source_data(tmp_path, damage):
    """A source with valid structure but bad payload data (a negative exp_avg_sq, a weight
    that no longer matches its master) merges into a bad composite; the re-verify inside
    execute_merge — pipelined into the file lanes — must refuse it with the reference's
    error kind (ConsistencyError, exit 2)."""
    need_gpu()
    import struct

    d = gen(tmp_path, SPEC, 2, 2)
    bad = tmp_path / "bad"
    shutil.copytree(d[0], bad)
    if damage == "weight_bit":
        w = bytearray((bad / "model.weights").read_bytes())
        w[-7] ^= 0x10
        (bad / "model.weights").write_bytes(bytes(w))
    else:
        p = bad / "optim" / "rank_1.shard"
        b = bytearray(p.read_bytes())
        hlen = int.from_bytes(b[:8], "little")
        hdr = json.loads(b[8:8 + hlen])
        lo, _ = hdr["g0.exp_avg_sq"]["data_offsets"]
        b[8 + hlen + lo:8 + hlen + lo + 4] = struct.pack("<f", -3.0)
        p.write_bytes(bytes(b))
    # the damaged source provides everything (base), so the composite carries the defect
    recipe = t.MergeRecipe(num_ranks=2, base_checkpoint=str(bad), slices=[t.RecipeSlice(d[1], [1])])
    rc, err = ref_error(recipe, tmp_path / "ref_out")
    e = our_error(recipe, tmp_path / "our_out")
    assert rc == 2 and err == "ConsistencyError", (rc, err)
    assert e is not None and e.kind == t.ErrorKind.Consistency, e


def test_regroup_refuses_a_source_with_bad_padding_before_writing(tmp_path):
    """read_checkpoint validates the source before the reference regroups it
    (R/src/checkpoint.cpp:515-553): nonzero shard padding is a CorruptContainer and
    nothing is written. The device path re-verifies the source first."""
    need_gpu()
    import struct

    spec = dict(SPEC, num_layers=3, hidden_dim=4, ffn_dim=16, vocab_size=31)
    ref_tool("train", *spec_args(spec), "--strategy", "full", "--steps", 10, "--interval", 10, "--ranks", 8,
             "--grouping", "coarse", "--out", tmp_path / "run")
    src = tmp_path / "run" / "checkpoint-10"
    p = src / "optim" / "rank_7.shard"
    b = bytearray(p.read_bytes())
    hlen = int.from_bytes(b[:8], "little")
    hdr = json.loads(b[8:8 + hlen])
    _, hi = hdr["g0.master"]["data_offsets"]  # coarse group 0 ends in rank 7's padding
    b[8 + hlen + hi - 4:8 + hlen + hi] = struct.pack("<f", 1.0)
    p.write_bytes(bytes(b))
    rc, _, err = ref_tool("regroup", "--dir", src, "--out", tmp_path / "ref", check=False)
    assert rc != 0 and "CorruptContainer" in err
    with pytest.raises(t.TailorError) as e:
        t.regroup(str(src), str(tmp_path / "ours"))
    assert e.value.kind == t.ErrorKind.CorruptContainer
    assert not (tmp_path / "ours").exists()


def _restrict_to_modules(ckpt: pathlib.Path, keep):
    """Rewrites a checkpoint's manifest and model.weights to cover only `keep` (the
    optimizer shards keep every group): a container in the reference's own layout —
    compact sorted JSON header padded with spaces to 8 B, payload in key order."""
    man = json.loads((ckpt / "manifest.json").read_text())
    man["modules"] = [m for m in man["modules"] if m in keep]
    (ckpt / "manifest.json").write_text(json.dumps(man, indent=2) + "\n")
    b = (ckpt / "model.weights").read_bytes()
    n = int.from_bytes(b[:8], "little")
    hdr = json.loads(b[8:8 + n])
    base = 8 + n
    mod = lambda name: ".".join(name.split(".")[:2]) if name.startswith("layers.") else name.split(".")[0]  # noqa: E731
    out_hdr, payload, at = {}, bytearray(), 0
    for name in sorted(hdr):
        if mod(name) not in keep:
            continue
        lo, hi = hdr[name]["data_offsets"]
        out_hdr[name] = dict(hdr[name], data_offsets=[at, at + hi - lo])
        payload += b[base + lo:base + hi]
        at += hi - lo
    text = json.dumps(out_hdr, sort_keys=True, separators=(",", ":")).encode()
    text += b" " * ((-(8 + len(text))) % 8)
    (ckpt / "model.weights").write_bytes(len(text).to_bytes(8, "little") + text + bytes(payload))


def test_coarse_partial_checkpoint_verifies_like_the_reference(tmp_path):
    """A coarse checkpoint stores every group, but its manifest (and weights) may cover
    only some modules: group_indices_for_modules returns all coarse groups and
    derive_weights pairs only the manifest's tensors (R/src/checkpoint.cpp:272-312), so
    read_checkpoint accepts it. So must the device re-verify (it dereferenced
    the missing weights entries)."""
    need_gpu()
    spec = dict(SPEC, num_layers=4)
    ref_tool("train", *spec_args(spec), "--strategy", "full", "--steps", 10, "--interval", 10, "--ranks", 2,
             "--grouping", "coarse", "--out", tmp_path / "run")
    ck = tmp_path / "run" / "checkpoint-10"
    _restrict_to_modules(ck, {"embed_tokens", "layers.1", "layers.3", "norm"})
    ref_tool("read", "--dir", ck)
    t.verify_checkpoint(str(ck))
    # and a damaged kept tensor is still found, with the reference's kind
    w = bytearray((ck / "model.weights").read_bytes())
    w[-3] ^= 0x40
    (ck / "model.weights").write_bytes(bytes(w))
    rc, _, err = ref_tool("read", "--dir", ck, check=False)
    assert rc == 2 and "ConsistencyError" in err
    with pytest.raises(t.TailorError) as e:
        t.verify_checkpoint(str(ck))
    assert e.value.kind == t.ErrorKind.Consistency


def test_lane_failure_does_not_hang_the_pipelined_reverify(tmp_path, monkeypatch):
    """when assembling the weights output fails, lanes that finished a rank
    file wait for the weights before their re-verify; they must be released and the
    merge must fail with a Storage error instead of hanging."""
    need_gpu()
    import threading

    d = gen(tmp_path, SPEC, 4, 2)
    monkeypatch.setenv("TAILOR_FAULT", "assemble-weights")
    recipe = t.MergeRecipe(num_ranks=4, base_checkpoint=d[1], slices=[t.RecipeSlice(d[0], [0, 2])])
    res = {}

    def run():
        try:
            t.execute_merge(recipe, str(tmp_path / "out"), t.MergeOptions(workers=5))
        except t.TailorError as e:
            res["e"] = e

    th = threading.Thread(target=run, daemon=True)
    th.start()
    th.join(timeout=120)
    assert not th.is_alive(), "execute_merge hung after a lane failure"
    assert res.get("e") is not None and res["e"].kind == t.ErrorKind.Storage, res
