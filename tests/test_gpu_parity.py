"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Oracles: oracle/tailor_oracle.py (numpy restatement, pinned in test_oracle.py)
and oracle/_ref/ref_tool (the reference library itself, compiled from
/root/reference by oracle/Makefile; the binary travels to the GPU box).
Bar: bit-exact bytes for every payload, header and sidecar; scores within
1e-6 relative; identical selections and recipes.
"""
import json
import os
import pathlib
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
import tailor_oracle as o  # noqa: E402
from conftest import ref_tool, spec_args  # noqa: E402

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-6  # SURVEY §8 a13 tolerance for FP64 scores


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def ospec(s: t.ModelSpec) -> dict:
    return dict(num_layers=s.num_layers, hidden_dim=s.hidden_dim, ffn_dim=s.ffn_dim, vocab_size=s.vocab_size,
                weight_tied=s.weight_tied, seed=s.seed)


SHAPES = [
    (t.ModelSpec(4, 8, 16, 32, False, 42), 4),
    (t.ModelSpec(3, 4, 4, 8, True, 50001), 3),     # tied; 12-B chunks (misaligned segments)
    (t.ModelSpec(2, 6, 10, 11, False, 9), 2),      # ragged, odd vocab
    (t.ModelSpec(1, 1, 1, 1, False, 1), 8),        # degenerate: padding-only ranks
    (t.ModelSpec(4, 64, 172, 512, False, 42), 8),
]


def dev(n):
    return torch.empty(max(16, n), dtype=torch.uint8, device="cuda")


def host_bytes(buf, n):
    return bytes(buf[:n].cpu().numpy())


@pytest.mark.parametrize("spec,N", SHAPES)
def test_generator_matches_oracle(spec, N):
    need_gpu()
    K = 3
    fam = t.SynthFamily(spec, N, K)
    os_ = ospec(spec)
    exp = [o.snapshot_payloads(os_, N, k) for k in range(1, K + 1)]
    for r in range(N):
        bufs = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
        fam.gen_shard(r, 1, K, [b.data_ptr() for b in bufs])
        torch.cuda.synchronize()
        for k in range(K):
            assert host_bytes(bufs[k], fam.shard_bytes(k + 1, r)) == exp[k][1][r], (r, k)
    wb = fam.weights_bytes(1)
    bufs = [dev(wb) for _ in range(K)]
    fam.gen_weights(1, K, 0, wb, [b.data_ptr() for b in bufs])
    torch.cuda.synchronize()
    for k in range(K):
        assert host_bytes(bufs[k], wb) == exp[k][0]


def test_write_dir_matches_reference_writer(tmp_path):
    """GPU generator + our writer == reference write_checkpoint, every file, every byte."""
    need_gpu()
    spec = t.ModelSpec(3, 8, 12, 20, False, 7)
    N, K = 3, 3
    ref_tool("gen", *spec_args(ospec(spec)), "--ranks", N, "--snapshots", K, "--out", tmp_path / "ref")
    fam = t.SynthFamily(spec, N, K)
    for k in range(1, K + 1):
        fam.write_dir(k, str(tmp_path / "ours" / f"checkpoint-{k * 100}"))
    _assert_same_tree(tmp_path / "ref", tmp_path / "ours")


def _assert_same_tree(a, b):
    fa = sorted(str(p.relative_to(a)) for p in a.rglob("*") if p.is_file())
    fb = sorted(str(p.relative_to(b)) for p in b.rglob("*") if p.is_file())
    assert fa == fb
    for rel in fa:
        assert (a / rel).read_bytes() == (b / rel).read_bytes(), rel


@pytest.mark.parametrize("K", [2, 3, 4, 16])
def test_scorer_matches_oracle(K):
    need_gpu()
    spec = t.ModelSpec(3, 16, 40, 50, False, 1234)
    N = 4
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    parts = []
    for r in range(N):
        bufs = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
        fam.gen_shard(r, 1, K, [b.data_ptr() for b in bufs])
        out = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device="cuda")
        t.Scorer(fam, r, 1, K).run([b.data_ptr() for b in bufs], out.data_ptr())
        torch.cuda.synchronize()
        parts += out.cpu().tolist()
    yaml, src, scores, gap = fam.select(parts, N, 0.5)
    os_ = ospec(spec)
    W = [o.model_vectors(os_, k)[0] for k in range(1, K + 1)]
    ref = [[o.magnitude_score(*x) for x in o.score_pair(os_, W[p], W[p + 1])] for p in range(K - 1)]
    for p in range(K - 1):
        for m in range(M):
            assert scores[p][m] == pytest.approx(ref[p][m], rel=SCORE_RTOL)
    _, ref_src, ref_gap = o.select(ref, M, 0.5)
    assert src == ref_src
    assert ref_gap > 1e-4


def test_scorer_packed_equals_full():
    need_gpu()
    spec = t.ModelSpec(2, 32, 64, 100, False, 5)
    N, K = 2, 4
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    for r in range(N):
        full = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
        packed = [dev(fam.packed_master_bytes(r)) for _ in range(K)]
        fam.gen_shard(r, 1, K, [b.data_ptr() for b in full])
        fam.gen_masters(r, 1, K, [b.data_ptr() for b in packed])
        a = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device="cuda")
        b = torch.zeros_like(a)
        t.Scorer(fam, r, 1, K).run([x.data_ptr() for x in full], a.data_ptr())
        t.Scorer(fam, r, 1, K, packed=True).run([x.data_ptr() for x in packed], b.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(a, b)  # same tiles, same order: bitwise


def _random_assignment(rng, spec, K):
    mods = o.modules(ospec(spec))
    L = spec.num_layers
    targets = list(range(L))
    if rng.random() < 0.3:
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
        if m.startswith("layers."):
            continue
        k = rng.randrange(1, K + 1)
        assign[m] = (f"S{k}", m)
        recipe.aux[m] = f"S{k}"
    return recipe, assign


@pytest.mark.parametrize("seed", range(6))
def test_partition_merge_matches_oracle(seed):
    """Device-resident K2 over random recipes (layer moves, tied, misaligned shapes)."""
    need_gpu()
    rng = random.Random(seed)
    spec, N = SHAPES[seed % len(SHAPES)]
    K = 3
    fam = t.SynthFamily(spec, N, K)
    recipe, assign = _random_assignment(rng, spec, K)
    recipe.num_ranks = N
    yaml = recipe.to_yaml()
    os_ = ospec(spec)
    mods = o.modules(os_)
    srcs = {f"S{k}": (*o.snapshot_payloads(os_, N, k), mods) for k in range(1, K + 1)}
    exp_w, exp_r, exp_wp, exp_rp = o.merge_payloads(os_, N, assign, srcs)
    for r in range(N):
        bufs = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
        fam.gen_shard(r, 1, K, [b.data_ptr() for b in bufs])
        mp = t.MergePartition(fam, yaml, r)
        assert mp.prefix() == exp_rp[r]
        mp.bind([bufs[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()])
        for variant in (0, 1):
            out = dev(mp.bytes)
            mp.run(out.data_ptr(), variant)
            torch.cuda.synchronize()
            assert host_bytes(out, mp.bytes) == exp_r[r], (r, variant)
    wb = fam.weights_bytes(1)
    wbufs = [dev(wb) for _ in range(K)]
    fam.gen_weights(1, K, 0, wb, [b.data_ptr() for b in wbufs])
    for units in (1, 3):
        got = b""
        for u in range(units):
            mp = t.MergePartition(fam, yaml, -1, u, units)
            lo, hi, total = mp.range()
            mp.bind([wbufs[k - 1].data_ptr() + wlo for k, c, wlo, whi in mp.windows()])
            out = dev(mp.bytes)
            mp.run(out.data_ptr())
            torch.cuda.synchronize()
            got += host_bytes(out, mp.bytes)
        assert got == exp_w
        assert mp.prefix() == exp_wp


def test_host_pipeline_matches_device():
    need_gpu()
    spec = t.ModelSpec(4, 64, 172, 512, False, 3)
    N, K = 2, 3
    fam = t.SynthFamily(spec, N, K)
    recipe = t.MergeRecipe(num_ranks=N, base_checkpoint="S3", slices=[t.RecipeSlice("S1", [0, 2]), t.RecipeSlice("S2", [1])],
                           aux={"embed_tokens": "S2"})
    yaml = recipe.to_yaml()
    for r in range(N):
        bufs = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
        fam.gen_shard(r, 1, K, [b.data_ptr() for b in bufs])
        mp = t.MergePartition(fam, yaml, r)
        mp.bind([bufs[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()])
        out = dev(mp.bytes)
        mp.run(out.data_ptr())
        hsrc = [b.cpu().pin_memory() for b in bufs]
        hdst = torch.empty(mp.bytes, dtype=torch.uint8).pin_memory()
        h2d, d2h = mp.run_host([hsrc[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()], hdst.data_ptr(),
                               chunk_bytes=4096)
        torch.cuda.synchronize()
        assert bytes(hdst.numpy()) == host_bytes(out, mp.bytes)
        assert h2d == mp.bytes and d2h == mp.bytes  # only the needed bytes cross PCIe
        # masters (and then m/v too) read from device copies: fewer H2D bytes, same result
        for fields, frac in ((4, 3), (7, 0)):
            hdst2 = torch.zeros(mp.bytes, dtype=torch.uint8).pin_memory()
            h2d2, _ = mp.run_host([hsrc[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()], hdst2.data_ptr(),
                                  chunk_bytes=1 << 14, d_windows=[bufs[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()],
                                  resident_fields=fields, async_=True)
            mp.wait()
            assert bytes(hdst2.numpy()) == host_bytes(out, mp.bytes)
            assert h2d2 == mp.bytes * frac // 3 or (fields == 4 and 0 < h2d2 < mp.bytes)
        # masters read from the scorer's packed buffers (cfg5's staged snapshots), only for
        # some windows' snapshots: same composite, fewer H2D bytes
        packed = [dev(fam.packed_master_bytes(r)) for _ in range(K)]
        for k in range(1, K + 1):
            fam.gen_masters(r, k, k, [packed[k - 1].data_ptr()])
        for keep in ({1, 2, 3}, {3}, {2}):
            hdst3 = torch.zeros(mp.bytes, dtype=torch.uint8).pin_memory()
            h2d3, _ = mp.run_host([hsrc[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()], hdst3.data_ptr(),
                                  chunk_bytes=1 << 14,
                                  d_windows=[packed[k - 1].data_ptr() if k in keep else None for k, c, lo, hi in mp.windows()],
                                  resident_fields=8)
            torch.cuda.synchronize()
            assert bytes(hdst3.numpy()) == host_bytes(out, mp.bytes), keep
            assert h2d3 < mp.bytes


def test_host_pipeline_prefetch_copies():
    """tg_mplan_run_host's prefetch list: extra H2D copies land intact, the composite is unchanged."""
    need_gpu()
    spec = t.ModelSpec(3, 64, 172, 512, False, 8)
    N, K = 2, 2
    fam = t.SynthFamily(spec, N, K)
    yaml = t.MergeRecipe(num_ranks=N, base_checkpoint="S2", slices=[t.RecipeSlice("S1", [1])]).to_yaml()
    bufs = [dev(fam.shard_bytes(k, 0)) for k in range(1, K + 1)]
    fam.gen_shard(0, 1, K, [b.data_ptr() for b in bufs])
    mp = t.MergePartition(fam, yaml, 0)
    mp.bind([bufs[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()])
    out = dev(mp.bytes)
    mp.run(out.data_ptr())
    hsrc = [b.cpu().pin_memory() for b in bufs]
    extra = [torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory() for n in (1, 4097, 300000, 0, 12345)]
    dsts = [dev(max(1, x.numel())) for x in extra]
    hdst = torch.empty(mp.bytes, dtype=torch.uint8).pin_memory()
    h2d, _ = mp.run_host([hsrc[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()], hdst.data_ptr(),
                         chunk_bytes=1 << 13, async_=True,
                         prefetch=[(x.data_ptr(), d.data_ptr(), x.numel()) for x, d in zip(extra, dsts)])
    mp.wait()
    assert bytes(hdst.numpy()) == host_bytes(out, mp.bytes)
    assert h2d == mp.bytes + sum(x.numel() for x in extra)
    for x, d in zip(extra, dsts):
        assert torch.equal(d[:x.numel()].cpu(), x)


def test_shard_sub_units_host_staged():
    """cfg5-style units: a rank partition assembled as tensor-aligned sub-ranges whose source
    windows are materialised one at a time (tg_family_gen_shard_range) == the whole partition."""
    need_gpu()
    spec = t.ModelSpec(4, 64, 172, 512, False, 21)
    N, K = 2, 3
    fam = t.SynthFamily(spec, N, K)
    yaml = t.MergeRecipe(num_ranks=N, base_checkpoint="S3", slices=[t.RecipeSlice("S1", [0, 2]),
                                                                    t.RecipeSlice("S2", [3])],
                         aux={"norm": "S1"}).to_yaml()
    r = 1
    bufs = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
    fam.gen_shard(r, 1, K, [b.data_ptr() for b in bufs])
    full = t.MergePartition(fam, yaml, r)
    full.bind([bufs[k - 1].data_ptr() + lo for k, c, lo, hi in full.windows()])
    out = dev(full.bytes)
    full.run(out.data_ptr())
    torch.cuda.synchronize()
    expect = host_bytes(out, full.bytes)
    for units in (2, 5):
        got = b""
        for u in range(units):
            mp = t.MergePartition(fam, yaml, r, u, units)
            hwin = []
            for k, c, lo, hi in mp.windows():
                d = dev(hi - lo)
                fam.gen_shard_range(r, k, lo, hi, d.data_ptr())
                torch.cuda.synchronize()
                assert torch.equal(d, bufs[k - 1][lo:hi])
                hwin.append(d.cpu().pin_memory())
            hdst = torch.empty(max(1, mp.bytes), dtype=torch.uint8).pin_memory()
            mp.run_host([h.data_ptr() for h in hwin], hdst.data_ptr(), chunk_bytes=1 << 12)
            got += bytes(hdst.numpy()[:mp.bytes])
        assert got == expect
    with pytest.raises(t.TailorError):  # windows must be tensor-aligned
        fam.gen_shard_range(r, 1, 4, 64, dev(64).data_ptr())


def test_dynamic_gather_tiles_are_bitwise_the_static_split():
    """K2's bulk ring claims its 64 KB tiles from a counter the plan owns and resets it on
    exit: back-to-back runs (no host sync between them) of the shard gather and of the
    device step's two gathers give bitwise the static split's bytes every time."""
    need_gpu()
    spec, N, K = t.ModelSpec(2, 512, 1376, 4096, False, 7), 2, 3  # ~9.6 MB rank shard: ~150 tiles
    fam = t.SynthFamily(spec, N, K)
    r = 1
    shards = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
    fam.gen_shard(r, 1, K, [b.data_ptr() for b in shards])
    rec = t.MergeRecipe(num_ranks=N, slices=[t.RecipeSlice("S1", [0], [0]), t.RecipeSlice("S2", [1], [1])],
                        aux={"embed_tokens": "S3", "norm": "S1", "lm_head": "S2"})
    yaml = rec.to_yaml()
    mp = t.MergePartition(fam, yaml, r)
    mp.bind([shards[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()])
    assert mp.bulk_ok
    ref = dev(mp.bytes)
    mp.run(ref.data_ptr(), 7)  # static split
    outs = [dev(mp.bytes) for _ in range(6)]
    for o_ in outs:
        mp.run(o_.data_ptr(), 0)
    torch.cuda.synchronize()
    for o_ in outs:
        assert torch.equal(o_[:mp.bytes], ref[:mp.bytes])
    st = t.SelectStep(fam, r, 0, 1, 0.5)
    sbytes, wlo, whi = st.range()
    wb = [dev(whi - wlo) for _ in range(K)]
    fam.gen_weights(1, K, wlo, whi, [b.data_ptr() for b in wb])
    st.bind([b.data_ptr() for b in shards], [b.data_ptr() for b in wb])
    parts = torch.tensor([float((i * 7919) % 97) for i in range(N * (K - 1) * fam.num_modules * 2)],
                         dtype=torch.float64, device="cuda")
    s_ref, w_ref = dev(sbytes), dev(whi - wlo)
    st.run(parts.data_ptr(), N, s_ref.data_ptr(), w_ref.data_ptr(), variant=7)
    runs = [(dev(sbytes), dev(whi - wlo)) for _ in range(4)]
    for a, b in runs:
        st.run(parts.data_ptr(), N, a.data_ptr(), b.data_ptr())
    torch.cuda.synchronize()
    for a, b in runs:
        assert torch.equal(a[:sbytes], s_ref[:sbytes])
        assert torch.equal(b[:whi - wlo], w_ref[:whi - wlo])


@pytest.mark.parametrize("seed", range(4))
def test_gather_variants_random_segments(seed):
    """Raw K2 (tg_gather): LSU and bulk paths vs a torch reference copy."""
    need_gpu()
    import ctypes

    g = torch.Generator().manual_seed(seed)
    src = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, generator=g).cuda()
    align = 16 if seed % 2 == 0 else 1
    segs, dst_off = [], 0
    expect = []
    while dst_off < 600_000:
        n = int(torch.randint(1, 40_000, (1,), generator=g)) // align * align or align
        so = int(torch.randint(0, (1 << 20) - n, (1,), generator=g)) // align * align
        segs.append((src.data_ptr() + so, dst_off, n))
        expect.append(src[so:so + n])
        dst_off += n
    expect = torch.cat(expect)
    table = (t._lib.GatherSegC * len(segs))(*[t._lib.GatherSegC(a, b, c) for a, b, c in segs])
    raw = torch.frombuffer(bytearray(bytes(table)), dtype=torch.uint8).cuda()
    variants = [1] + ([2] if align == 16 else [])
    for v in variants:
        dst = torch.zeros(dst_off, dtype=torch.uint8, device="cuda")
        t.gather(raw.data_ptr(), len(segs), dst.data_ptr(), dst_off, v, bulk_ok=(v == 2))
        torch.cuda.synchronize()
        assert torch.equal(dst, expect), v


# ---------------------------------------------------------------- files ----------
def _gen_ref(tmp, spec, N, K, name="run", partial=None):
    args = ["gen", *spec_args(ospec(spec)), "--ranks", N, "--snapshots", K, "--out", tmp / name]
    if partial:
        args += ["--partial", partial]
    return ref_tool(*args)[1]["snapshots"]


def _ref_merge(recipe: t.MergeRecipe, out, extra=()):
    p = out.parent / (out.name + ".recipe.json")
    p.write_text(recipe.to_json())
    return ref_tool("merge", "--recipe", p, "--out", out, *extra)[1]


def _both_merge(tmp, recipe, name="m", **opt):
    ref_out, our_out = tmp / f"{name}_ref", tmp / f"{name}_ours"
    ref = _ref_merge(recipe, ref_out, ["--uncached"] if opt.get("uncached") else [])
    st = t.execute_merge(recipe, str(our_out), t.MergeOptions(**opt))
    _assert_same_tree(ref_out, our_out)
    assert st.shard_files_read == ref["stats"]["shard_files_read"]
    assert st.weight_files_read == ref["stats"]["weight_files_read"]
    return st


def test_execute_merge_parity_recipe_matches_reference(tmp_path):
    """R/tests/test_merge.cpp:100-139 shape: L=4, N=4, two sources, 11 group copies."""
    need_gpu()
    spec = t.ModelSpec(4, 8, 16, 32, False, 909)
    d = _gen_ref(tmp_path, spec, 4, 2)
    recipe = t.MergeRecipe(num_ranks=4, slices=[t.RecipeSlice(d[0], [0, 2]), t.RecipeSlice(d[1], [1, 3])],
                           aux={"embed_tokens": d[0], "norm": d[1], "lm_head": d[1]})
    assert len(t.resolve_plan(recipe)["group_copies"]) == 11
    st = _both_merge(tmp_path, recipe)
    assert st.shard_files_read <= 8 and st.weight_files_read == 2


def test_execute_merge_identity_is_fixed_point(tmp_path):
    need_gpu()
    spec = t.ModelSpec(3, 8, 16, 32, False, 808)
    d = _gen_ref(tmp_path, spec, 2, 1)
    st = _both_merge(tmp_path, t.MergeRecipe(num_ranks=2, base_checkpoint=d[0]))
    assert st.shard_files_read == 2
    for rel in ["model.weights", "optim/rank_0.shard", "optim/rank_1.shard", "config.json", "trainer_state.json"]:
        assert (tmp_path / "m_ours" / rel).read_bytes() == open(os.path.join(d[0], rel), "rb").read()
    t.execute_merge(t.MergeRecipe(num_ranks=2, base_checkpoint=str(tmp_path / "m_ours")), str(tmp_path / "m2"))
    for rel in ["model.weights", "optim/rank_0.shard", "optim/rank_1.shard"]:
        assert (tmp_path / "m2" / rel).read_bytes() == (tmp_path / "m_ours" / rel).read_bytes()


def test_execute_merge_cross_position_tied(tmp_path):
    need_gpu()
    spec = t.ModelSpec(4, 8, 16, 32, True, 1212)
    d = _gen_ref(tmp_path, spec, 2, 1)
    _both_merge(tmp_path, t.MergeRecipe(num_ranks=2, base_checkpoint=d[0], slices=[t.RecipeSlice(d[0], [0, 1], [3, 2])]))


def test_execute_merge_uncached_counts_and_bytes(tmp_path):
    need_gpu()
    spec = t.ModelSpec(4, 8, 16, 32, False, 2323)
    d = _gen_ref(tmp_path, spec, 4, 2)
    recipe = t.MergeRecipe(num_ranks=4, slices=[t.RecipeSlice(d[0], [0, 2]), t.RecipeSlice(d[1], [1, 3])],
                           aux={"embed_tokens": d[0], "norm": d[1], "lm_head": d[1]})
    st = _both_merge(tmp_path, recipe, uncached=True)
    assert st.shard_files_read == 4 * 11


@pytest.mark.parametrize("case", range(12))
def test_execute_merge_random_cases_match_reference(tmp_path, case):
    """Acceptance c4-style: random L<=8, tied, h in {4,8}, N<=4, K<=3, layer permutations."""
    need_gpu()
    rng = random.Random(1000 + case)
    L = 1 + rng.randrange(8)
    spec = t.ModelSpec(L, 4 << rng.randrange(2), 4 << rng.randrange(2), 8 << rng.randrange(2), rng.random() < 0.5,
                       50000 + case)
    N = 1 + rng.randrange(4)
    K = 1 + rng.randrange(3)
    d = _gen_ref(tmp_path, spec, N, K)
    ids = {f"S{k}": d[k - 1] for k in range(1, K + 1)}
    recipe, _ = _random_assignment(rng, spec, K)
    recipe.num_ranks = N
    recipe.slices = [t.RecipeSlice(ids[s.source], s.layers, s.targets) for s in recipe.slices]
    recipe.aux = {k: ids[v] for k, v in recipe.aux.items()}
    if rng.random() < 0.5:
        recipe.base_checkpoint = d[-1]
    _both_merge(tmp_path, recipe, workers=1 + rng.randrange(4))


def test_execute_merge_partial_sources_and_errors(tmp_path):
    need_gpu()
    spec = t.ModelSpec(4, 8, 16, 32, False, 4)
    d = _gen_ref(tmp_path, spec, 2, 2, partial="2=layers.0,norm")
    # source 2 holds only layers.0 + norm
    _both_merge(tmp_path, t.MergeRecipe(num_ranks=2, base_checkpoint=d[0], slices=[t.RecipeSlice(d[1], [0])],
                                        aux={"norm": d[1]}))
    with pytest.raises(t.TailorError) as e:
        t.execute_merge(t.MergeRecipe(num_ranks=2, base_checkpoint=d[0], slices=[t.RecipeSlice(d[1], [2])]),
                        str(tmp_path / "x"))
    assert e.value.kind == t.ErrorKind.SourceLacksModule
    (tmp_path / "full").mkdir()
    (tmp_path / "full" / "f").write_text("x")
    with pytest.raises(t.TailorError) as e:
        t.execute_merge(t.MergeRecipe(num_ranks=2, base_checkpoint=d[0]), str(tmp_path / "full"))
    assert e.value.kind == t.ErrorKind.Storage


def test_reference_trained_parity_pipeline(tmp_path):
    """Acceptance c5 shape on reference-written partial checkpoints: train(parity) -> fail -> plan -> merge."""
    need_gpu()
    spec = dict(num_layers=4, hidden_dim=8, ffn_dim=16, vocab_size=32, seed=31415)
    ref_tool("train", *spec_args(spec), "--strategy", "parity", "--steps", 100, "--interval", 25, "--ranks", 2,
             "--out", tmp_path / "run", "--fail-at", 110)
    ours = t.recipe_from_manifests(str(tmp_path / "run"), 110)
    ref = t.MergeRecipe.from_json(json.dumps(ref_tool("plan", "--run", tmp_path / "run", "--failure-step", 110)[1]["recipe"]))
    assert ours == ref
    _both_merge(tmp_path, ours)


def test_verify_detects_corruption(tmp_path):
    need_gpu()
    spec = t.ModelSpec(2, 8, 16, 32, False, 77)
    d = _gen_ref(tmp_path, spec, 3, 1)
    t.verify_checkpoint(d[0])
    import shutil

    bad = tmp_path / "bad"
    shutil.copytree(d[0], bad)
    w = bytearray((bad / "model.weights").read_bytes())
    w[-1] ^= 0x01
    (bad / "model.weights").write_bytes(bytes(w))
    with pytest.raises(t.TailorError) as e:
        t.verify_checkpoint(str(bad))
    assert e.value.kind == t.ErrorKind.Consistency
    rc, _, err = ref_tool("read", "--dir", bad, check=False)
    assert rc == 2 and "ConsistencyError" in err


@pytest.mark.parametrize("K", [17, 20, 35])
def test_select_recipe_beyond_16_snapshots_matches_reference(tmp_path, K):
    """The paper merges from 18 and 35 checkpoints and
    recipe_from_manifests takes any number (R/src/merge.cpp:359-418): sweeps longer than
    one 16-snapshot K3 launch run as overlapping windows. Scores, selection and recipe
    equal the reference-side restatement; the merge equals the reference's bytes."""
    need_gpu()
    spec = t.ModelSpec(3, 8, 24, 40, False, 4200 + K)
    d = _gen_ref(tmp_path, spec, 2, K)
    ref = ref_tool("score", "--snapshots", ",".join(d), "--rho", "0.5")[1]
    devs = list(range(torch.cuda.device_count())) * 2
    for kw in (dict(), dict(devices=devs)):
        rec, src, gap = t.select_recipe(d, 0.5, **kw)
        _, scores = t.score_snapshots(d, **kw)
        assert len(scores) == K - 1
        for p, row in enumerate(ref["scores"]):
            for m, v in enumerate(row):
                assert scores[p][m] == pytest.approx(v, rel=SCORE_RTOL)
        assert rec == t.MergeRecipe.from_json(json.dumps(ref["recipe"]))
        assert gap == pytest.approx(ref["min_boundary_gap"], rel=1e-6)
    _both_merge(tmp_path, rec)


def test_scoring_rolls_through_two_slots_beyond_16_snapshots(tmp_path, monkeypatch):
    """Under a device budget of two snapshots per rank, a 20-snapshot sweep rolls
    through two slots (every pair scored once); same scores as the resident sweep."""
    need_gpu()
    spec = t.ModelSpec(2, 8, 24, 40, False, 77)
    d = _gen_ref(tmp_path, spec, 2, 20)
    _, full = t.score_snapshots(d)
    monkeypatch.setenv("TAILOR_DEVICE_BUDGET", str(2 * 4096))
    _, rolled = t.score_snapshots(d)
    assert len(rolled) == len(full) == 19
    for a, b in zip(rolled, full):  # K3 at K=2 vs K=16 tiles: same sums up to FP64 reassociation
        assert a == pytest.approx(b, rel=1e-12)


def test_select_recipe_matches_reference_scorer(tmp_path):
    need_gpu()
    spec = t.ModelSpec(4, 16, 40, 64, False, 42)
    d = _gen_ref(tmp_path, spec, 2, 4)
    rec, src, gap = t.select_recipe(d, 0.5)
    ref = ref_tool("score", "--snapshots", ",".join(d), "--rho", "0.5")[1]
    _, scores = t.score_snapshots(d)
    for p, row in enumerate(ref["scores"]):
        for m, v in enumerate(row):
            assert scores[p][m] == pytest.approx(v, rel=SCORE_RTOL)
    assert rec == t.MergeRecipe.from_json(json.dumps(ref["recipe"]))
    assert gap == pytest.approx(ref["min_boundary_gap"], rel=1e-6)
    _both_merge(tmp_path, rec)


@pytest.mark.parametrize("seed", range(5))
def test_device_select_step_matches_host_path(seed):
    """K9: on-device selection + segment tables == host select_by_magnitude + plan, bitwise."""
    need_gpu()
    rng = random.Random(seed)
    spec = t.ModelSpec(1 + rng.randrange(6), 8 * (1 + rng.randrange(3)), 16, 48, rng.random() < 0.3, 100 + seed)
    N, K = 1 + rng.randrange(4), 2 + rng.randrange(4)
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    r, units = rng.randrange(N), 1 + rng.randrange(3)
    unit = rng.randrange(units)
    rho = rng.choice([0.2, 0.5, 0.75])
    shards = [dev(fam.shard_bytes(k, r)) for k in range(1, K + 1)]
    fam.gen_shard(r, 1, K, [b.data_ptr() for b in shards])
    st = t.SelectStep(fam, r, unit, units, rho)
    sbytes, wlo, whi = st.range()
    wb = [dev(whi - wlo) for _ in range(K)]
    if whi > wlo:
        fam.gen_weights(1, K, wlo, whi, [b.data_ptr() for b in wb])
    st.bind([b.data_ptr() for b in shards], [b.data_ptr() for b in wb])
    for trial in range(2):
        if trial == 0:  # real scorer partials of every rank
            parts = []
            for rr in range(N):
                bufs = [dev(fam.shard_bytes(k, rr)) for k in range(1, K + 1)]
                fam.gen_shard(rr, 1, K, [b.data_ptr() for b in bufs])
                out = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device="cuda")
                t.Scorer(fam, rr, 1, K).run([b.data_ptr() for b in bufs], out.data_ptr())
                torch.cuda.synchronize()
                parts += out.cpu().tolist()
        else:  # adversarial: coarse values with exact ties
            parts = [float(rng.randrange(4)) for _ in range(N * (K - 1) * M * 2)]
        d_parts = torch.tensor(parts, dtype=torch.float64, device="cuda")
        out_s, out_w = dev(sbytes), dev(whi - wlo)
        st.run(d_parts.data_ptr(), N, out_s.data_ptr(), out_w.data_ptr())
        torch.cuda.synchronize()
        src_d, sc_d = st.result()
        yaml, src_h, sc_h, _ = fam.select(parts, N, rho)
        assert src_d == src_h and sc_d == sc_h
        mp = t.MergePartition(fam, yaml, r)
        mp.bind([shards[k - 1].data_ptr() + lo for k, c, lo, hi in mp.windows()])
        ref = dev(mp.bytes)
        mp.run(ref.data_ptr())
        wp = t.MergePartition(fam, yaml, -1, unit, units)
        wp.bind([wb[k - 1].data_ptr() + (lo - wlo) for k, c, lo, hi in wp.windows()])
        wref = dev(wp.bytes)
        wp.run(wref.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(out_s[:sbytes], ref[:sbytes])
        assert torch.equal(out_w[:whi - wlo], wref[:whi - wlo])


@pytest.mark.parametrize("K", [2, 4, 7, 16])
def test_scorer_variants_agree(K):
    """Register-staged vs TMA-bulk-staged scorer: same tiles, different in-tile order."""
    need_gpu()
    spec = t.ModelSpec(2, 40, 100, 333, False, 11)   # ragged chunk counts (tails not multiple of 4)
    N = 3
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    for r in range(N):
        bufs = [dev(fam.packed_master_bytes(r)) for _ in range(K)]
        fam.gen_masters(r, 1, K, [b.data_ptr() for b in bufs])
        outs = []
        for v in (1, 2, 3, 4):
            sc = t.Scorer(fam, r, 1, K, packed=True)
            sc.set_variant(v)
            out = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device="cuda")
            sc.run([b.data_ptr() for b in bufs], out.data_ptr())
            outs.append(out)
        torch.cuda.synchronize()
        for o_ in outs[1:]:
            assert torch.allclose(outs[0], o_, rtol=1e-12, atol=0)


@pytest.mark.parametrize("K", [2, 3, 4, 9, 16])
def test_staged_scorer_dynamic_tiles_are_bitwise_the_static_split(K, monkeypatch):
    """The TMA-ring scorer claims tiles dynamically (atomic counter); each tile's partial
    still lands in its own slot, so the result must be bitwise the static split's
    (TAILOR_SCORE_STATIC=1), repeat after repeat. Big enough for many tiles per CTA and
    ragged field tails (not multiples of 4 or of the chunk)."""
    need_gpu()
    spec = t.ModelSpec(3, 256, 690, 1001, False, 17)
    N = 2
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    bufs = [dev(fam.packed_master_bytes(0)) for _ in range(K)]
    fam.gen_masters(0, 1, K, [b.data_ptr() for b in bufs])

    def score(static):
        if static:
            monkeypatch.setenv("TAILOR_SCORE_STATIC", "1")
        else:
            monkeypatch.delenv("TAILOR_SCORE_STATIC", raising=False)
        sc = t.Scorer(fam, 0, 1, K, packed=True)
        sc.set_variant(2)
        outs = []
        for _ in range(3):
            out = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device="cuda")
            sc.run([b.data_ptr() for b in bufs], out.data_ptr())
            outs.append(out)
        torch.cuda.synchronize()
        return outs

    ref = score(True)[0]
    for o_ in score(False) + score(True):
        assert torch.equal(ref, o_)


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_execute_merge_lane_count_independent_and_sources_untouched(tmp_path, N):
    """Acceptance c9/c10 + R/tests/test_merge.cpp:370-385 shape: the composite does not
    depend on the host worker (lane) count, equals the reference's, and the source files
    are byte-for-byte untouched."""
    need_gpu()
    import hashlib

    spec = t.ModelSpec(5, 16, 40, 64, False, 6060 + N)
    d = _gen_ref(tmp_path, spec, N, 3)

    def digest():
        return {str(p): hashlib.sha256(p.read_bytes()).hexdigest() for k in d for p in sorted(pathlib.Path(k).rglob("*"))
                if p.is_file()}

    before = digest()
    recipe = t.MergeRecipe(num_ranks=N, base_checkpoint=d[2],
                           slices=[t.RecipeSlice(d[0], [0, 3]), t.RecipeSlice(d[1], [1, 4], [2, 1])],
                           aux={"embed_tokens": d[0], "lm_head": d[1]})
    _both_merge(tmp_path, recipe, name="w1", workers=1)
    for w in (3, 16):
        t.execute_merge(recipe, str(tmp_path / f"w{w}"), t.MergeOptions(workers=w))
        _assert_same_tree(tmp_path / "w1_ours", tmp_path / f"w{w}")
    # lanes spread over a device list (every GPU of the box, each listed twice): same bytes
    devs = list(range(torch.cuda.device_count())) * 2
    t.execute_merge(recipe, str(tmp_path / "devs"), t.MergeOptions(workers=len(devs), devices=devs))
    _assert_same_tree(tmp_path / "w1_ours", tmp_path / "devs")
    assert digest() == before
    # identity round trip at this rank count (c9): merged base == source base
    t.execute_merge(t.MergeRecipe(num_ranks=N, base_checkpoint=d[1]), str(tmp_path / "ident"))
    for r in range(N):
        rel = f"optim/rank_{r}.shard"
        assert (tmp_path / "ident" / rel).read_bytes() == (pathlib.Path(d[1]) / rel).read_bytes()


@pytest.mark.parametrize("damage", ["padding", "negative_v", "weight_bit"])
def test_verify_lanes_report_the_damaged_rank(tmp_path, damage):
    """Device re-verify runs the rank files over parallel lanes; a defect in one rank
    file of eight is still found with the reference's error kind."""
    need_gpu()
    import shutil
    import struct

    spec = t.ModelSpec(3, 4, 16, 31, False, 99)  # h=4 norm over 8 ranks: ranks 4-7 hold only padding
    d = _gen_ref(tmp_path, spec, 8, 1)
    t.verify_checkpoint(d[0])
    bad = tmp_path / "bad"
    shutil.copytree(d[0], bad)
    r = 5
    if damage == "weight_bit":
        w = bytearray((bad / "model.weights").read_bytes())
        w[-3] ^= 0x40
        (bad / "model.weights").write_bytes(bytes(w))
        kind, ref_name = t.ErrorKind.Consistency, "ConsistencyError"
    else:
        p = bad / "optim" / f"rank_{r}.shard" if damage == "negative_v" else bad / "optim" / "rank_7.shard"
        b = bytearray(p.read_bytes())
        hlen = int.from_bytes(b[:8], "little")
        hdr = json.loads(b[8:8 + hlen])
        base = 8 + hlen
        g = spec.num_layers + 1  # embed group: 124 elements, chunk 16, rank 5 fully valid
        if damage == "padding":
            lo, hi = hdr["g0.master"]["data_offsets"]  # norm group: rank 7's one element is padding
            b[base + hi - 4:base + hi] = struct.pack("<f", 1.0)
            kind, ref_name = t.ErrorKind.CorruptContainer, "CorruptContainer"
        else:
            lo, hi = hdr[f"g{g}.exp_avg_sq"]["data_offsets"]
            b[base + lo:base + lo + 4] = struct.pack("<f", -1.0)
            kind, ref_name = t.ErrorKind.Consistency, "ConsistencyError"
        p.write_bytes(bytes(b))
    with pytest.raises(t.TailorError) as e:
        t.verify_checkpoint(str(bad))
    assert e.value.kind == kind
    rc, _, err = ref_tool("read", "--dir", bad, check=False)
    assert rc != 0 and ref_name in err


KIND_NAMES = {t.ErrorKind.Consistency: "ConsistencyError", t.ErrorKind.CorruptContainer: "CorruptContainer"}


@pytest.mark.parametrize("budget", [None, 1 << 14])
def test_file_paths_stream_under_a_small_device_budget(tmp_path, monkeypatch, budget):
    """The file-facing paths must not need a whole rank (or the whole weights payload)
    resident: a 70B-shaped rank partition is 4 x 40 GB of masters for the scorer and
    160 GB of weights + 120 GB of shard for the re-verify. TAILOR_DEVICE_BUDGET forces
    the streaming forms at a small shape (pairwise scoring through two slots; verify in
    4 KB windows with only the paired weight bytes loaded). Scores, selection, merged
    bytes and error kinds must be those of the resident forms and of the reference."""
    need_gpu()
    import shutil
    import struct

    spec = t.ModelSpec(3, 16, 40, 61, False, 4242)
    N = 3
    d = _gen_ref(tmp_path, spec, N, 4)
    if budget is not None:
        monkeypatch.setenv("TAILOR_DEVICE_BUDGET", str(budget))
    rec, src, gap = t.select_recipe(d, 0.5)
    ref = ref_tool("score", "--snapshots", ",".join(d), "--rho", "0.5")[1]
    _, scores = t.score_snapshots(d)
    for p, row in enumerate(ref["scores"]):
        for m, v in enumerate(row):
            assert scores[p][m] == pytest.approx(v, rel=SCORE_RTOL)
    assert rec == t.MergeRecipe.from_json(json.dumps(ref["recipe"]))
    _both_merge(tmp_path, rec)  # includes the device re-verify in the forced form
    t.verify_checkpoint(str(tmp_path / "m_ours"))
    # damage one element of each kind; the verify must name the reference's error kind
    cases = {"weight": t.ErrorKind.Consistency, "padding": t.ErrorKind.CorruptContainer,
             "negative_v": t.ErrorKind.Consistency}
    for damage, kind in cases.items():
        bad = tmp_path / f"bad_{damage}"
        shutil.copytree(tmp_path / "m_ours", bad)
        if damage == "weight":
            w = bytearray((bad / "model.weights").read_bytes())
            w[-5] ^= 0x20
            (bad / "model.weights").write_bytes(bytes(w))
        else:  # N=3: norm (16 elements) -> chunk 6, rank 2 holds 2 padding elements
            p = bad / "optim" / ("rank_2.shard" if damage == "padding" else "rank_1.shard")
            b = bytearray(p.read_bytes())
            hlen = int.from_bytes(b[:8], "little")
            hdr = json.loads(b[8:8 + hlen])
            key = "g0.master" if damage == "padding" else f"g{spec.num_layers + 1}.exp_avg_sq"
            lo, hi = hdr[key]["data_offsets"]
            at = 8 + hlen + (hi - 4 if damage == "padding" else lo + 4 * 7)
            b[at:at + 4] = struct.pack("<f", -2.0 if damage == "negative_v" else 3.0)
            p.write_bytes(bytes(b))
        with pytest.raises(t.TailorError) as e:
            t.verify_checkpoint(str(bad))
        rc, _, err = ref_tool("read", "--dir", bad, check=False)
        assert rc != 0 and KIND_NAMES[kind] in err, (damage, err)
        assert e.value.kind == kind, (damage, err)
