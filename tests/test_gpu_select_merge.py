"""tg_select_merge (select + merge in one call, the scorer's device copies of the masters
reused by the merge) against the reference's select-merge (oracle/_ref/ref_tool) and
against the two separate calls: same recipe, same bytes in every file, whatever the device
budget (masters kept or not), the device list, the lane count or the I/O mode.
Anchors: R/src/merge.cpp:226-357, :359-418 (recipe from the saved modules)."""
import hashlib
import os
import pathlib

import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
from conftest import ref_tool  # noqa: E402

pytestmark = pytest.mark.gpu


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def digest(root: pathlib.Path):
    return {str(p.relative_to(root)): hashlib.sha256(p.read_bytes()).hexdigest()
            for p in sorted(root.rglob("*")) if p.is_file()}


def gen(tmp, spec, N, K, name="run"):
    fam = t.SynthFamily(spec, N, K, 100)
    dirs = [str(tmp / name / f"checkpoint-{k * 100}") for k in range(1, K + 1)]
    for k in range(1, K + 1):
        fam.write_dir(k, dirs[k - 1])
    return dirs


SHAPES = [
    (t.ModelSpec(4, 64, 172, 512, False, 42), 4, 3),
    (t.ModelSpec(3, 32, 88, 100, True, 7), 2, 4),     # tied
    (t.ModelSpec(2, 24, 40, 50, False, 5), 8, 3),     # ragged chunks (12-B multiples), 8 ranks
    (t.ModelSpec(6, 128, 344, 1000, False, 11), 1, 5),
]


@pytest.mark.parametrize("spec,N,K", SHAPES)
def test_select_merge_matches_reference_and_separate_calls(tmp_path, spec, N, K):
    need_gpu()
    dirs = gen(tmp_path, spec, N, K)
    ref = ref_tool("select-merge", "--snapshots", ",".join(dirs), "--rho", 0.5, "--out", tmp_path / "ref")[1]
    rec, src, gap, st = t.select_merge(dirs, str(tmp_path / "ours"), 0.5)
    assert rec == t.MergeRecipe.from_json(__import__("json").dumps(ref["recipe"]))
    assert digest(tmp_path / "ref") == digest(tmp_path / "ours")
    assert st.resident_bytes > 0
    assert st.shard_files_read == ref["merge"]["stats"]["shard_files_read"]
    rec_s, src_s, gap_s = t.select_recipe(dirs, 0.5)
    assert (rec_s, src_s, gap_s) == (rec, src, gap)


@pytest.mark.parametrize("mode", ["small-budget", "two-devices", "lanes-1", "direct-rw", "uncached"])
def test_select_merge_forms_write_the_same_bytes(tmp_path, monkeypatch, mode):
    """Masters not kept (budget below one snapshot set, or a device list: the merge lanes
    may run elsewhere) -> exactly the separate calls; O_DIRECT / one lane / uncached reads
    with the masters kept: the same bytes as the reference."""
    need_gpu()
    spec, N, K = t.ModelSpec(4, 64, 172, 512, False, 42), 4, 3
    dirs = gen(tmp_path, spec, N, K)
    ref_tool("select-merge", "--snapshots", ",".join(dirs), "--rho", 0.5, "--out", tmp_path / "ref")
    opt = t.MergeOptions()
    kept = True
    if mode == "small-budget":
        monkeypatch.setenv("TAILOR_DEVICE_BUDGET", str(64 << 10))
        kept = False
    elif mode == "two-devices":
        opt = t.MergeOptions(devices=[0, 0])
        kept = False
    elif mode == "lanes-1":
        opt = t.MergeOptions(workers=1)
    elif mode == "direct-rw":
        opt = t.MergeOptions(io_mode="direct-rw")
    elif mode == "uncached":
        opt = t.MergeOptions(uncached=True)
    _, _, _, st = t.select_merge(dirs, str(tmp_path / "ours"), 0.5, opt)
    assert digest(tmp_path / "ref") == digest(tmp_path / "ours")
    assert (st.resident_bytes > 0) == kept


def test_select_merge_errors_before_writing(tmp_path):
    need_gpu()
    spec, N, K = t.ModelSpec(2, 16, 40, 64, False, 3), 2, 3
    dirs = gen(tmp_path, spec, N, K)
    out = tmp_path / "busy"
    out.mkdir()
    (out / "x").write_text("keep")
    with pytest.raises(t.TailorError) as e:
        t.select_merge(dirs, str(out), 0.5)
    assert e.value.kind == t.ErrorKind.Storage
    assert sorted(os.listdir(out)) == ["x"]
    with pytest.raises(t.TailorError) as e:  # one snapshot cannot be scored
        t.select_merge(dirs[:1], str(tmp_path / "o2"), 0.5)
    assert not (tmp_path / "o2").exists()


def test_cli_select_merge_matches_reference(tmp_path):
    need_gpu()
    import subprocess

    spec, N, K = t.ModelSpec(3, 32, 88, 200, False, 9), 2, 4
    dirs = gen(tmp_path, spec, N, K)
    ref_tool("select-merge", "--snapshots", ",".join(dirs), "--rho", 0.5, "--out", tmp_path / "ref")
    p = subprocess.run([str(t.CLI_PATH), "select-merge", "--snapshots", ",".join(dirs), "--rho", "0.5", "--out",
                        str(tmp_path / "ours"), "--recipe-out", str(tmp_path / "r.yaml")], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    assert digest(tmp_path / "ref") == digest(tmp_path / "ours")
    assert t.parse_recipe((tmp_path / "r.yaml").read_text()) == t.select_recipe(dirs, 0.5)[0]
    bad = subprocess.run([str(t.CLI_PATH), "select-merge", "--snapshots", ",".join(dirs), "--out", str(tmp_path / "ours")],
                         capture_output=True, text=True)
    assert bad.returncode == 2  # Storage (non-empty output directory), as `tailor merge`


def test_select_merge_beyond_16_snapshots(tmp_path):
    """The paper merges from 18 and 35 checkpoints: scoring sweeps windows
    of <= 16 snapshots; every snapshot's masters are kept for the merge."""
    need_gpu()
    spec, N, K = t.ModelSpec(3, 16, 40, 64, False, 21), 2, 20
    dirs = gen(tmp_path, spec, N, K)
    ref_tool("select-merge", "--snapshots", ",".join(dirs), "--rho", 0.5, "--out", tmp_path / "ref")
    rec, src, gap, st = t.select_merge(dirs, str(tmp_path / "ours"), 0.5)
    assert digest(tmp_path / "ref") == digest(tmp_path / "ours")
    assert st.resident_bytes > 0
    assert (rec, src, gap) == t.select_recipe(dirs, 0.5)
