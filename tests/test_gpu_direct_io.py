"""Direct I/O on the files drop-in (the reference reads through the page
cache, R/src/container.cpp:193-207): O_DIRECT source reads (staged congruent to the
file offset mod 4 KB, partial blocks through a bounce buffer), O_DIRECT output writes
(4 KB block grid, header tail in chunk 0, truncate to size) and the auto mode (direct
reads of sources that are not in the page cache). Whatever the mode, every output file
must equal the reference's byte for byte, and the scorer's results must not change."""
import os
import pathlib
import subprocess

import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
from conftest import ROOT, ref_tool, spec_args  # noqa: E402

pytestmark = pytest.mark.gpu

MODES = ["buffered", "direct", "direct-rw", "auto"]


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def o_direct_ok(d: pathlib.Path) -> bool:
    """Whether the filesystem under d accepts O_DIRECT (tmpfs on older kernels does not)."""
    p = d / ".odirect_probe"
    p.write_bytes(b"\0" * 4096)
    try:
        fd = os.open(p, os.O_RDONLY | os.O_DIRECT)
        os.close(fd)
        return True
    except OSError:
        return False
    finally:
        p.unlink()


def evict(paths):
    """Drops the files' pages from the page cache (clean pages only: fsync first)."""
    for p in paths:
        fd = os.open(p, os.O_RDONLY)
        try:
            os.fsync(fd)
            os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
        finally:
            os.close(fd)


def tree_files(root: pathlib.Path):
    return sorted(p for p in root.rglob("*") if p.is_file())


def same_tree(a: pathlib.Path, b: pathlib.Path):
    fa = [str(p.relative_to(a)) for p in tree_files(a)]
    fb = [str(p.relative_to(b)) for p in tree_files(b)]
    assert fa == fb
    for rel in fa:
        assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


def gen(tmp, spec, N, K, name="run"):
    return ref_tool("gen", *spec_args(spec), "--ranks", N, "--snapshots", K, "--out", tmp / name)[1]["snapshots"]


def mixed_recipe(dirs, N, L):
    """Layer l from source l % K, base = the last source (every source contributes)."""
    K = len(dirs)
    slices = [t.RecipeSlice(dirs[k], [l for l in range(L) if l % K == k]) for k in range(K)]
    return t.MergeRecipe(num_ranks=N, base_checkpoint=dirs[-1], slices=[s for s in slices if s.layers])


def ref_merge(tmp, recipe, out):
    p = tmp / (out.name + ".json")
    p.write_text(recipe.to_json())
    ref_tool("merge", "--recipe", p, "--out", out)


# 12-byte-aligned segment offsets (h=8) and a multi-chunk shape (rank shards > 15 MB chunks)
SHAPES = {
    "ragged": (dict(num_layers=3, hidden_dim=8, ffn_dim=20, vocab_size=36, weight_tied=False, seed=5), 3, 3),
    "multichunk": (dict(num_layers=4, hidden_dim=256, ffn_dim=688, vocab_size=32000, weight_tied=False, seed=42), 2, 2),
}


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_merge_io_modes_are_byte_identical_to_the_reference(tmp_path, shape, mode):
    need_gpu()
    spec, N, K = SHAPES[shape]
    dirs = gen(tmp_path, spec, N, K)
    rec = mixed_recipe(dirs, N, spec["num_layers"])
    ref_merge(tmp_path, rec, tmp_path / "ref_out")
    if mode == "auto":  # cold sources: auto must pick O_DIRECT for them
        evict([p for d in dirs for p in tree_files(pathlib.Path(d))])
    st = t.execute_merge(rec, str(tmp_path / "ours"), t.MergeOptions(workers=3, io_mode=mode))
    same_tree(tmp_path / "ref_out", tmp_path / "ours")
    direct = o_direct_ok(tmp_path)
    if mode == "auto" and shape == "ragged":
        return  # KB-sized files: the header read's readahead caches them whole, so auto stays buffered
    if mode == "buffered" or not direct:
        assert st.direct_read_bytes == 0 and st.direct_write_bytes == 0
    else:
        assert st.direct_read_bytes > 0
        # every composite byte that comes from a source file was read directly
        assert st.direct_read_bytes >= st.bytes_moved
    if mode == "direct-rw" and direct:
        assert st.direct_write_bytes >= st.bytes_moved
    elif mode != "direct-rw":
        assert st.direct_write_bytes == 0


def test_auto_keeps_the_page_cache_for_warm_sources(tmp_path):
    need_gpu()
    spec, N, K = SHAPES["ragged"]
    dirs = gen(tmp_path, spec, N, K)
    for d in dirs:  # warm: read everything once
        for p in tree_files(pathlib.Path(d)):
            p.read_bytes()
    st = t.execute_merge(mixed_recipe(dirs, N, spec["num_layers"]), str(tmp_path / "ours"), t.MergeOptions(io_mode="auto"))
    assert st.direct_read_bytes == 0


def test_tailor_io_env_overrides_the_option(tmp_path, monkeypatch):
    need_gpu()
    if not o_direct_ok(tmp_path):
        pytest.skip("filesystem refuses O_DIRECT")
    spec, N, K = SHAPES["ragged"]
    dirs = gen(tmp_path, spec, N, K)
    rec = mixed_recipe(dirs, N, spec["num_layers"])
    monkeypatch.setenv("TAILOR_IO", "direct-rw")
    st = t.execute_merge(rec, str(tmp_path / "ours"), t.MergeOptions(io_mode="buffered"))
    assert st.direct_read_bytes > 0 and st.direct_write_bytes > 0
    monkeypatch.delenv("TAILOR_IO")
    ref_merge(tmp_path, rec, tmp_path / "ref_out")
    same_tree(tmp_path / "ref_out", tmp_path / "ours")


@pytest.mark.parametrize("mode", ["buffered", "direct"])
def test_scorer_and_selection_do_not_depend_on_the_io_mode(tmp_path, monkeypatch, mode):
    need_gpu()
    spec, N, K = SHAPES["multichunk"][0], 2, 3
    dirs = gen(tmp_path, spec, N, K)
    monkeypatch.setenv("TAILOR_IO", "buffered")
    base_rec, base_src, _ = t.select_recipe(dirs, 0.5)
    _, base_scores = t.score_snapshots(dirs)
    evict([p for d in dirs for p in tree_files(pathlib.Path(d))])
    monkeypatch.setenv("TAILOR_IO", mode)
    rec, src, _ = t.select_recipe(dirs, 0.5)
    _, scores = t.score_snapshots(dirs)
    assert rec == base_rec and src == base_src
    assert scores == base_scores  # same tiles, same order: bitwise


def test_regroup_direct_rw_matches_reference(tmp_path):
    need_gpu()
    spec, N, K = SHAPES["ragged"][0], 2, 1
    src = gen(tmp_path, spec, N, K)[0]
    ref_tool("regroup", "--dir", src, "--to", "coarse", "--out", tmp_path / "ref_coarse")
    t.regroup(src, str(tmp_path / "coarse"), to_fine=False, options=t.MergeOptions(io_mode="direct-rw"))
    same_tree(tmp_path / "ref_coarse", tmp_path / "coarse")


def test_cli_io_flag(tmp_path):
    need_gpu()
    spec, N, K = SHAPES["ragged"]
    dirs = gen(tmp_path, spec, N, K)
    rec = mixed_recipe(dirs, N, spec["num_layers"])
    (tmp_path / "r.yaml").write_text(t.recipe_to_yaml(rec))
    cli = ROOT / "paper_2602_22158_b200" / "bin" / "tailor"
    p = subprocess.run([str(cli), "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "a"), "--io",
                        "direct-rw"], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    p = subprocess.run([str(cli), "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "b"), "--io",
                        "sideways"], capture_output=True, text=True)
    assert p.returncode == 1 and "unknown --io mode" in p.stderr
    ref_merge(tmp_path, rec, tmp_path / "ref_out")
    same_tree(tmp_path / "ref_out", tmp_path / "a")
