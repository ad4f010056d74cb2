"""the device-resident trainer vs the reference trainer:
checkpoints byte-identical for full / parity / filter schedules (bit-exact AdamW on
the device), log norms within 1e-9; the in-situ magnitude strategy selects what the
reference-side scorer selects on the reference's full snapshots, and the composite
merged from the selective run equals the reference's select-merge composite."""
import json

import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
from conftest import ref_tool, spec_args  # noqa: E402

pytestmark = pytest.mark.gpu


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def same_tree(a, b, skip=("log.jsonl",)):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file() and p.name not in skip)
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file() and p.name not in skip)
    assert fa == fb
    for rel in fa:
        assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


def logs_close(a, b):
    la = [json.loads(x) for x in (a / "log.jsonl").read_text().splitlines() if x]
    lb = [json.loads(x) for x in (b / "log.jsonl").read_text().splitlines() if x]
    assert [x["step"] for x in la] == [x["step"] for x in lb]
    for x, y in zip(la, lb):
        assert x["grad_norm"] == pytest.approx(y["grad_norm"], rel=1e-9)
        assert x["update_norm"] == pytest.approx(y["update_norm"], rel=1e-9)


CASES = [
    (dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=777), "full", 2, 60, 20),
    (dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=31415), "parity", 2, 100, 25),
    (dict(num_layers=6, hidden_dim=8, ffn_dim=12, vocab_size=20, weight_tied=True, seed=9), "filter", 3, 100, 10),
    (dict(num_layers=2, hidden_dim=16, ffn_dim=40, vocab_size=50, weight_tied=False, seed=5), "full", 4, 30, 10),
]


@pytest.mark.parametrize("spec,strategy,N,steps,interval", CASES)
def test_device_trainer_matches_reference_trainer(tmp_path, spec, strategy, N, steps, interval):
    need_gpu()
    ref_tool("train", *spec_args(spec), "--strategy", strategy, "--steps", steps, "--interval", interval,
             "--ranks", N, "--out", tmp_path / "ref")
    s = t.ModelSpec(spec["num_layers"], spec["hidden_dim"], spec["ffn_dim"], spec["vocab_size"], spec["weight_tied"],
                    spec["seed"])
    n = t.train(s, str(tmp_path / "ours"), steps, interval, strategy, num_ranks=N)
    assert n == steps // interval
    same_tree(tmp_path / "ref", tmp_path / "ours")
    logs_close(tmp_path / "ref", tmp_path / "ours")


def test_magnitude_strategy_in_situ(tmp_path):
    need_gpu()
    spec = dict(num_layers=6, hidden_dim=16, ffn_dim=40, vocab_size=64, weight_tied=False, seed=2024)
    N, steps, interval = 2, 80, 20
    s = t.ModelSpec(6, 16, 40, 64, False, 2024)
    t.train(s, str(tmp_path / "mag"), steps, interval, "magnitude", num_ranks=N, rho=0.5)
    # reference: full snapshots of the same trajectory + the reference-side scorer/selection
    ref_tool("train", *spec_args(spec), "--strategy", "full", "--steps", steps, "--interval", interval, "--ranks", N,
             "--out", tmp_path / "full")
    snaps = [tmp_path / "full" / f"checkpoint-{k * interval}" for k in range(1, steps // interval + 1)]
    ref = ref_tool("score", "--snapshots", ",".join(map(str, snaps)), "--rho", "0.5")[1]
    assert ref["min_boundary_gap"] > 1e-9  # selection well conditioned
    for k, names in enumerate(ref["saved"]):
        man = json.loads((tmp_path / "mag" / f"checkpoint-{(k + 1) * interval}" / "manifest.json").read_text())
        assert man["modules"] == names, k
        assert man["strategy"] == "magnitude"
    # saved modules hold exactly the reference state (verify against the full snapshot, module subset)
    for k in range(1, len(snaps) + 1):
        out = ref_tool("verify", "--a", tmp_path / "mag" / f"checkpoint-{k * interval}", "--b", snaps[k - 1],
                       "--modules", ",".join(ref["saved"][k - 1]))[1]
        assert out["equal"], out["first_divergence"]
    # failure after the last checkpoint: recover (our plan + merge) == reference select-merge composite
    rec = t.recipe_from_manifests(str(tmp_path / "mag"), steps)
    t.execute_merge(rec, str(tmp_path / "merged"))
    ref_tool("select-merge", "--snapshots", ",".join(map(str, snaps)), "--rho", "0.5", "--out", tmp_path / "ref_merged")
    for rel in ["model.weights", "optim_meta.json", "config.json", "trainer_state.json"] + \
               [f"optim/rank_{r}.shard" for r in range(N)]:
        assert (tmp_path / "merged" / rel).read_bytes() == (tmp_path / "ref_merged" / rel).read_bytes(), rel
    t.verify_checkpoint(str(tmp_path / "merged"))


def test_cli_train_matches_reference_cli(tmp_path):
    """`tailor train` (R/tools/tailor_main.cpp:40-64 flags) on the device trainer."""
    need_gpu()
    import subprocess
    spec = dict(num_layers=3, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=4242)
    ref_tool("train", *spec_args(spec), "--strategy", "filter", "--steps", 40, "--interval", 10, "--ranks", 2,
             "--head", 1, "--tail", 1, "--sparse-multiple", 2, "--out", tmp_path / "ref")
    cfg = tmp_path / "config.json"
    cfg.write_bytes((tmp_path / "ref" / "checkpoint-10" / "config.json").read_bytes())
    cli = str(t._lib.CLI_PATH)
    base = [cli, "train", "--config", str(cfg), "--steps", "40", "--interval", "10", "--ranks", "2"]
    r = subprocess.run(base + ["--strategy", "filter", "--head", "1", "--tail", "1", "--sparse-multiple", "2",
                               "--out", str(tmp_path / "ours")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "4 checkpoints" in r.stdout
    same_tree(tmp_path / "ref", tmp_path / "ours")
    logs_close(tmp_path / "ref", tmp_path / "ours")
    for bad in [["--strategy", "sometimes", "--out", str(tmp_path / "x")],
                ["--strategy", "full", "--grouping", "coarse", "--out", str(tmp_path / "y")]]:
        r = subprocess.run(base + bad, capture_output=True, text=True)
        assert r.returncode == 1 and "RecipeError" in r.stderr


def _d2d(dst: int, src: int, n: int) -> None:
    import ctypes

    cudart = ctypes.CDLL("libcudart.so.12")
    assert cudart.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(n), 3) == 0  # D2D


@pytest.mark.parametrize("store_grad", ["0", "1"])
@pytest.mark.parametrize("poison", [float("inf"), float("nan"), float("-inf")])
def test_nonfinite_gradient_leaves_state_untouched(monkeypatch, store_grad, poison):
    """apply_step's contract (R/src/adamw.cpp:49-60): a non-finite gradient raises
    NonFinite before any state changes. Both pass-1 forms (the masters' exponent check,
    with the gradient recomputed in pass 2; and the full gradient pass with a scratch
    buffer) must catch it, and both give the same norms on clean steps."""
    need_gpu()
    import sys

    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1] / "oracle"))
    import tailor_oracle as o

    monkeypatch.setenv("TAILOR_TRAIN_STORE_GRAD", store_grad)
    spec = t.ModelSpec(2, 16, 40, 64, False, 5)
    ospec = dict(num_layers=2, hidden_dim=16, ffn_dim=40, vocab_size=64, weight_tied=False, seed=5)
    N = 2
    tr = t.Trainer(spec, N)
    norms = [tr.step(1), tr.step(2)]
    ref = t.Trainer(spec, N) if store_grad == "0" else None
    if ref is not None:  # the other pass-1 form gives the same norms (within FP64 summation order)
        monkeypatch.setenv("TAILOR_TRAIN_STORE_GRAD", "1")
        ref = t.Trainer(spec, N)
        for s, (g, u) in zip((1, 2), norms):
            rg, ru = ref.step(s)
            assert g == pytest.approx(rg, rel=1e-12) and u == pytest.approx(ru, rel=1e-12)
    ptr, n = tr.partition(1)
    _, entries, payload = o.container_layout(o.shard_decls(ospec, N, range(len(o.group_table(ospec)))))
    assert payload == n
    lo, hi = entries["g1.master"]  # layer 0 no-decay group, rank 1's chunk
    snap = torch.empty(n, dtype=torch.uint8, device="cuda")
    _d2d(snap.data_ptr(), ptr, n)
    snap.view(torch.float32)[lo // 4 + 3] = poison
    _d2d(ptr, snap.data_ptr(), n)
    for s in (3, 4):  # refused, and refused again: the state never changes
        with pytest.raises(t.TailorError) as e:
            tr.step(s)
        assert e.value.kind == t.ErrorKind.NonFinite
    after = torch.empty_like(snap)
    _d2d(after.data_ptr(), ptr, n)
    assert torch.equal(after, snap)
    # a non-finite first moment is not a gradient: the step proceeds
    tr2 = t.Trainer(spec, N)
    tr2.step(1)
    p2, _ = tr2.partition(0)
    s2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    _d2d(s2.data_ptr(), p2, n)
    lo, hi = entries["g1.exp_avg"]
    s2.view(torch.float32)[lo // 4] = poison
    _d2d(p2, s2.data_ptr(), n)
    tr2.step(2)


@pytest.mark.parametrize("strategy,ranks", [("parity", 2), ("filter", 3), ("full", 1)])
def test_resume_from_merged_composite_matches_reference(tmp_path, strategy, ranks):
    """Acceptance c5 (R/tests/acceptance.cpp:256-303) on the device: the reference trains
    with a partial-checkpoint strategy and fails at 110; the composite is planned
    (recipe_from_manifests) and merged (our execute_merge); then `resume` continues 100
    steps from it — our device resume and the reference's resume write byte-identical
    checkpoints (log norms within 1e-9), and the CLI does the same."""
    need_gpu()
    import subprocess

    spec = dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=31415)
    extra = ["--head", 1, "--tail", 1, "--sparse-multiple", 2] if strategy == "filter" else []
    ref_tool("train", *spec_args(spec), "--strategy", strategy, "--steps", 100, "--interval", 25, "--ranks", ranks,
             *extra, "--out", tmp_path / "run", "--fail-at", 110)
    recipe = t.recipe_from_manifests(str(tmp_path / "run"), 110)
    t.execute_merge(recipe, str(tmp_path / "merged"))
    ref_tool("resume", "--ckpt", tmp_path / "merged", "--steps", 100, "--out", tmp_path / "ref_res")
    n = t.resume(str(tmp_path / "merged"), 100, str(tmp_path / "our_res"))
    assert n == 4
    same_tree(tmp_path / "ref_res", tmp_path / "our_res")
    logs_close(tmp_path / "ref_res", tmp_path / "our_res")
    r = subprocess.run([str(t._lib.CLI_PATH), "resume", "--ckpt", str(tmp_path / "merged"), "--steps", "100", "--out",
                        str(tmp_path / "cli_res")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    same_tree(tmp_path / "ref_res", tmp_path / "cli_res")


def test_resume_errors_match_reference(tmp_path):
    """resume's contract: partial checkpoints -> MissingModules (exit 1), a non-empty output
    directory -> StorageError (exit 2), negative steps -> RecipeError."""
    need_gpu()
    import subprocess

    spec = dict(num_layers=2, hidden_dim=8, ffn_dim=16, vocab_size=32, weight_tied=False, seed=7)
    ref_tool("train", *spec_args(spec), "--strategy", "parity", "--steps", 50, "--interval", 25, "--ranks", 2,
             "--out", tmp_path / "run")
    partial = tmp_path / "run" / "checkpoint-50"
    rc, _, err = ref_tool("resume", "--ckpt", partial, "--steps", 10, "--out", tmp_path / "r1", check=False)
    with pytest.raises(t.TailorError) as e:
        t.resume(str(partial), 10, str(tmp_path / "o1"))
    assert e.value.kind == t.ErrorKind.MissingModules and rc == 1 and "MissingModules" in err
    full = tmp_path / "full"
    ref_tool("train", *spec_args(spec), "--strategy", "full", "--steps", 25, "--interval", 25, "--ranks", 2,
             "--out", full)
    (tmp_path / "busy").mkdir()
    (tmp_path / "busy" / "x").write_text("x")
    with pytest.raises(t.TailorError) as e:
        t.resume(str(full / "checkpoint-25"), 10, str(tmp_path / "busy"))
    assert e.value.kind == t.ErrorKind.Storage
    r = subprocess.run([str(t._lib.CLI_PATH), "resume", "--ckpt", str(full / "checkpoint-25"), "--steps", "5", "--out",
                        str(tmp_path / "busy")], capture_output=True, text=True)
    assert r.returncode == 2 and "StorageError" in r.stderr
    with pytest.raises(t.TailorError) as e:
        t.resume(str(full / "checkpoint-25"), -1, str(tmp_path / "o2"))
    assert e.value.kind == t.ErrorKind.Recipe


def test_constant_division_is_ieee_division(tmp_path):
    """kernels/ieee_div.cuh: a / b through y = RN(1/b) and Markstein's correction equals
    __fdiv_rn bit for bit for all 2^32 float bit patterns a, for the bias corrections
    1 - beta^t (beta 0.9, 0.999, 0.95; t = 1..300) and 100 random divisors in [2^-20, 1]."""
    need_gpu()
    import pathlib
    import subprocess

    root = pathlib.Path(__file__).resolve().parents[1]
    exe = tmp_path / "div_const_check"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3",
                    "-I", str(root / "paper_2602_22158_b200/csrc/kernels"), "-I", str(root / "paper_2602_22158_b200/csrc"),
                    str(root / "tools/div_const_check.cu"), "-o", str(exe)], check=True)
    p = subprocess.run([str(exe), "300", "100", "0.9", "0.999", "0.95"], capture_output=True, text=True, timeout=600)
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["divisors"] == 1000 and res["mismatches"] == 0, (res, p.stderr[-2000:])


@pytest.mark.parametrize("fdiv", ["0", "1"])
def test_trainer_division_forms_are_bitwise_equal(monkeypatch, fdiv):
    """The trainer with the precomputed-reciprocal bias division vs per-element __fdiv_rn
    (TAILOR_TRAIN_FDIV=1): identical state bytes and norms after several steps."""
    need_gpu()
    spec = t.ModelSpec(2, 256, 688, 1000, False, 3)
    monkeypatch.setenv("TAILOR_TRAIN_FDIV", fdiv)
    a = t.Trainer(spec, 2)
    monkeypatch.setenv("TAILOR_TRAIN_FDIV", "1")
    b = t.Trainer(spec, 2)
    for s in range(1, 8):
        assert a.step(s) == b.step(s)
    for r in range(2):
        (pa, na), (pb, nb) = a.partition(r), b.partition(r)
        x = torch.empty(na, dtype=torch.uint8, device="cuda")
        y = torch.empty(nb, dtype=torch.uint8, device="cuda")
        _d2d(x.data_ptr(), pa, na)
        _d2d(y.data_ptr(), pb, nb)
        assert torch.equal(x, y)
