"""Pins the CPU oracle (oracle/tailor_oracle.py) before anything is checked against it:
(1) the reference's own known-answer tests, restated; (2) the reference binary's
output, via committed golden fixtures (tests/golden/make_golden.py) and — where the
binary is present — directly."""
import hashlib
import json
import pathlib

import numpy as np
import pytest

import tailor_oracle as o
from conftest import REF_TOOL, ref_tool, spec_args

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def toy(L=4, tied=False, seed=42, h=8, f=16, v=32):
    return dict(num_layers=L, hidden_dim=h, ffn_dim=f, vocab_size=v, weight_tied=tied, seed=seed)


# ---- R/tests/test_groups.cpp:13-69, R/tests/acceptance.cpp:80-100 --------------------
def test_group_counts():
    assert len(o.group_table(toy(16))) == 35
    assert len(o.group_table(toy(16, True))) == 34
    for L in range(1, 65):
        assert len(o.group_table(toy(L))) == 2 * L + 3
        assert len(o.group_table(toy(L, True))) == 2 * L + 2


def test_group_table_order():
    t = o.group_table(toy(16))
    assert t[0][:2] == ("norm", "no_decay")
    for i in range(16):
        assert t[1 + i][:2] == (f"layers.{i}", "no_decay")
        assert t[19 + i][:2] == (f"layers.{i}", "decay")
    assert t[17][0] == "embed_tokens" and t[18][0] == "lm_head"


def test_group_indices_for_L16():
    s, st = toy(16), toy(16, True)
    assert o.group_indices_for(s, "norm") == [0]
    assert o.group_indices_for(s, "embed_tokens") == [17]
    assert o.group_indices_for(s, "lm_head") == [18]
    assert o.group_indices_for(s, "layers.4") == [5, 23]
    assert o.group_indices_for(st, "layers.4") == [5, 22]


# ---- R/tests/test_model.cpp:13-60 ----------------------------------------------------
def test_module_enumeration_and_tensors():
    assert len(o.modules(toy(32))) == 35
    assert len(o.modules(toy(16, True))) == 18
    names = [n for n, _, _ in o.tensors_of(toy(), "layers.0")]
    assert names[:2] == ["layers.0.input_layernorm.weight", "layers.0.post_attention_layernorm.weight"]
    assert [s for _, s, _ in o.tensors_of(toy(h=8, f=16), "layers.1")][-1] == (8, 16)


# ---- R/tests/test_shard.cpp:12-21 ----------------------------------------------------
def test_shard_lengths():
    assert o.shard_length(10, 4) == 3
    assert o.shard_length(5, 1) == 5
    assert o.shard_length(0, 3) == 0


# ---- R/tests/test_bf16.cpp:48-93 -----------------------------------------------------
def f32(bits):
    return np.array([bits], dtype=np.uint32).view(np.float32)


def test_bf16_known_answers():
    assert o.bf16_round(np.array([1.0], np.float32))[0] == 0x3F80
    assert o.bf16_round(f32(0x3F804000))[0] == 0x3F80
    assert o.bf16_round(f32(0x3F808000))[0] == 0x3F80  # tie -> even
    assert o.bf16_round(f32(0x3F818000))[0] == 0x3F82
    assert o.bf16_round(np.array([-0.0], np.float32))[0] == 0x8000
    assert o.bf16_round(np.array([np.inf], np.float32))[0] == 0x7F80
    nan = o.bf16_round(f32(0x7F800001))[0]
    assert (nan & 0x7F80) == 0x7F80 and (nan & 0x7F) != 0


def test_bf16_prefix_sweep_vs_nearest_even():
    prefix = np.arange(1 << 16, dtype=np.uint32)
    for suffix in (0x0000, 0x7FFF, 0x8000, 0x8001, 0xFFFF):
        bits = (prefix << 16) | suffix
        x = bits.view(np.float32)
        got = o.bf16_round(x).astype(np.uint32)
        finite = np.isfinite(x)
        lo = bits >> 16
        # independent restatement: compare the exact distance to both neighbours
        lo_f = (lo << 16).view(np.float32).astype(np.float64)
        hi_f = ((lo + 1) << 16).astype(np.uint32).view(np.float32).astype(np.float64)
        dx = x.astype(np.float64)
        with np.errstate(invalid="ignore"):
            want = np.where(np.abs(dx - lo_f) < np.abs(hi_f - dx), lo,
                            np.where(np.abs(hi_f - dx) < np.abs(dx - lo_f), lo + 1, np.where(lo % 2 == 0, lo, lo + 1)))
        ok = finite & np.isfinite(hi_f)
        assert np.array_equal(got[ok], want[ok])
        assert np.all(np.isnan(((got[np.isnan(x)] << 16).astype(np.uint32)).view(np.float32)))


# ---- R/tests/test_container.cpp:57-120, test_checkpoint.cpp:83-97 --------------------
def test_container_alignment_and_sizes():
    prefix, ents, size = o.container_layout([("b", "F32", (3,)), ("a", "BF16", (5,))], {"rank": "0"})
    assert len(prefix) % 8 == 0
    assert list(ents) == ["a", "b"] and ents["a"] == (0, 10) and ents["b"] == (10, 22)
    spec = toy()
    groups = list(range(len(o.group_table(spec))))
    _, _, payload = o.container_layout(o.shard_decls(spec, 1, groups))
    padded = sum(o.shard_length(n, 1) for _, _, n in o.group_table(spec))
    assert payload == 12 * padded


def test_lexicographic_payload_order():
    spec = toy(12)
    _, ents, _ = o.container_layout(o.shard_decls(spec, 2, range(len(o.group_table(spec)))))
    names = list(ents)
    assert names.index("g10.exp_avg") < names.index("g2.exp_avg")
    assert names[:3] == ["g0.exp_avg", "g0.exp_avg_sq", "g0.master"]


# ---- golden fixtures from the reference binary ----------------------------------------
def _digest(prefix: bytes, payload: bytes) -> str:
    return hashlib.sha256(prefix + payload).hexdigest()


@pytest.mark.parametrize("name", ["toy4", "tied3", "odd2", "score4"])
def test_oracle_sources_match_reference_golden(name):
    g = json.loads((GOLDEN / "merge_golden.json").read_text())[name]
    spec, N, K = g["spec"], g["ranks"], g["snapshots"]
    groups = list(range(len(o.group_table(spec))))
    wprefix, _, _ = o.container_layout(o.weight_decls(spec, o.modules(spec)))
    for k in range(1, K + 1):
        files = g["sources"][f"checkpoint-{k * 100}"]
        wp, rp = o.snapshot_payloads(spec, N, k)
        assert _digest(wprefix, wp) == files["model.weights"]
        for r in range(N):
            prefix, _, _ = o.container_layout(o.shard_decls(spec, N, groups), {"num_ranks": str(N), "rank": str(r)})
            assert _digest(prefix, rp[r]) == files[f"optim/rank_{r}.shard"]


@pytest.mark.parametrize("name", ["toy4", "tied3", "odd2", "score4"])
def test_oracle_merges_match_reference_golden(name):
    g = json.loads((GOLDEN / "merge_golden.json").read_text())[name]
    spec, N, K = g["spec"], g["ranks"], g["snapshots"]
    mods = o.modules(spec)
    srcs = {f"<SRC>/checkpoint-{k * 100}": (*o.snapshot_payloads(spec, N, k), mods) for k in range(1, K + 1)}
    for rname, m in g["merges"].items():
        rec = m["recipe"]
        assign = {}
        for s in rec.get("slices", []):
            for a, b in zip(s["layers"], s.get("targets", s["layers"])):
                assign[f"layers.{b}"] = (s["source"], f"layers.{a}")
        for key, src in rec.get("aux", {}).items():
            assign[key] = (src, key)
        for mod in mods:
            assign.setdefault(mod, (rec["base_checkpoint"], mod))
        w, ranks, wp, rps = o.merge_payloads(spec, N, assign, srcs)
        assert _digest(wp, w) == m["files"]["model.weights"], rname
        for r in range(N):
            assert _digest(rps[r], ranks[r]) == m["files"][f"optim/rank_{r}.shard"], (rname, r)


@pytest.mark.parametrize("name", ["toy4", "tied3", "odd2", "score4"])
def test_oracle_scores_match_reference_golden(name):
    g = json.loads((GOLDEN / "score_golden.json").read_text())[name]
    spec, K = g["spec"], g["snapshots"]
    W = [o.model_vectors(spec, k)[0] for k in range(1, K + 1)]
    sc = [[o.magnitude_score(*x) for x in o.score_pair(spec, W[p], W[p + 1])] for p in range(K - 1)]
    ref = g["result"]["scores"]
    np.testing.assert_allclose(np.array(sc), np.array(ref), rtol=1e-12)  # same FP64 math, different order
    saved, _, gap = o.select(sc, len(o.modules(spec)), 0.5)
    names = o.modules(spec)
    assert [[names[i] for i in s] for s in saved] == g["result"]["saved"]
    assert gap == pytest.approx(g["result"]["min_boundary_gap"], rel=1e-9)


def test_oracle_generator_matches_reference_binary_directly(tmp_path):
    if not REF_TOOL.exists():
        pytest.skip("reference binary not built")
    spec = toy(2, False, 7, 8, 12, 20)
    ref_tool("gen", *spec_args(spec), "--ranks", 3, "--snapshots", 2, "--out", tmp_path)
    groups = list(range(len(o.group_table(spec))))
    for k in (1, 2):
        d = tmp_path / f"checkpoint-{k * 100}"
        wp, rp = o.snapshot_payloads(spec, 3, k)
        wprefix, _, _ = o.container_layout(o.weight_decls(spec, o.modules(spec)))
        assert (d / "model.weights").read_bytes() == wprefix + wp
        for r in range(3):
            prefix, _, _ = o.container_layout(o.shard_decls(spec, 3, groups), {"num_ranks": "3", "rank": str(r)})
            assert (d / "optim" / f"rank_{r}.shard").read_bytes() == prefix + rp[r]
