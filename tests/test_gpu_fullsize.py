"""Full-size parity at the BASELINE configs, through size-independent properties:
a whole ZeRO rank partition of the Llama-3.1-8B-shaped (cfg3) and Qwen2.5-7B-shaped
(cfg2) models is generated, scored and merged on the device, then
  * every composite entry equals the selected source's entry (bytes, on device),
  * the weights share equals the selected sources' tensors,
  * every module's scorer sums equal a torch FP64 reduction of the same masters (1e-9 rel),
  * scoring a snapshot against itself gives exactly zero deltas,
  * generator values at random element ids equal the CPU oracle's (bit-exact),
  * the TMA-bulk and LSU gather variants agree byte for byte.
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2602_22158_b200 as t  # noqa: E402
import tailor_oracle as o  # noqa: E402

pytestmark = pytest.mark.gpu

CONFIGS = {
    "cfg3": (t.ModelSpec(32, 4096, 14336, 128256, False, 42), 8, 4),
    "cfg2": (t.ModelSpec(28, 3584, 18944, 152064, False, 42), 8, 2),
}


def entries(prefix: bytes):
    hlen = int.from_bytes(prefix[:8], "little")
    h = json.loads(prefix[8:8 + hlen])
    h.pop("__metadata__", None)
    return {k: tuple(v["data_offsets"]) for k, v in h.items()}


@pytest.mark.parametrize("name,r", [("cfg3", 3), ("cfg3", 7), ("cfg2", 5), ("cfg2", 0)])
def test_full_size_rank_partition(name, r):
    """r = 7 is the last ZeRO rank (it holds every group's padding), r = 0 the first."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec, N, K = CONFIGS[name]
    fam = t.SynthFamily(spec, N, K)
    M = fam.num_modules
    dev = torch.device("cuda")
    shards = [torch.empty(fam.shard_bytes(k, r), dtype=torch.uint8, device=dev) for k in range(1, K + 1)]
    fam.gen_shard(r, 1, K, [b.data_ptr() for b in shards])
    base = t.MergeRecipe(num_ranks=N, base_checkpoint=f"S{K}").to_yaml()
    lo, hi, _ = t.MergePartition(fam, base, -1, r, N).range()
    wbufs = [torch.empty(hi - lo, dtype=torch.uint8, device=dev) for _ in range(K)]
    fam.gen_weights(1, K, lo, hi, [b.data_ptr() for b in wbufs])

    # ---- scorer ---------------------------------------------------------------------
    out = torch.zeros((K - 1) * M * 2, dtype=torch.float64, device=dev)
    t.Scorer(fam, r, 1, K).run([b.data_ptr() for b in shards], out.data_ptr())
    torch.cuda.synchronize()
    got = out.view(K - 1, M, 2).cpu().numpy()
    s = dict(num_layers=spec.num_layers, hidden_dim=spec.hidden_dim, ffn_dim=spec.ffn_dim,
             vocab_size=spec.vocab_size, weight_tied=False, seed=spec.seed)
    mods = o.modules(s)
    ents = entries(t.MergePartition(fam, base, r).prefix())
    for mi in range(len(mods)):  # every module: embed, each layer, norm, lm_head
        for p in range(K - 1):
            sd = sr = 0.0
            for g in o.group_indices_for(s, mods[mi]):
                b0, b1 = ents[f"g{g}.master"]
                a = shards[p][b0:b1].view(torch.float32).double()
                b = shards[p + 1][b0:b1].view(torch.float32).double()
                sd += float(((b - a) ** 2).sum())
                sr += float((a * a).sum())
            assert got[p, mi, 0] == pytest.approx(sd, rel=1e-9)
            assert got[p, mi, 1] == pytest.approx(sr, rel=1e-9)
    same = torch.zeros(M * 2, dtype=torch.float64, device=dev)
    t.Scorer(fam, r, 1, 2).run([shards[0].data_ptr(), shards[0].data_ptr()], same.data_ptr())
    torch.cuda.synchronize()
    assert torch.all(same.view(M, 2)[:, 0] == 0)

    # ---- selection + merge -------------------------------------------------------------
    yaml, src_of, scores, gap = fam.select(out.cpu().tolist(), 1, 0.5)
    assert gap > 1e-4
    sp = t.MergePartition(fam, yaml, r)
    sp.bind([shards[k - 1].data_ptr() + wlo for k, c, wlo, whi in sp.windows()])
    assert sp.bulk_ok
    dst = torch.empty(sp.bytes, dtype=torch.uint8, device=dev)
    dst2 = torch.zeros_like(dst)
    sp.run(dst.data_ptr(), 2)
    sp.run(dst2.data_ptr(), 1)
    torch.cuda.synchronize()
    assert torch.equal(dst, dst2)
    table = o.group_table(s)
    for key, (b0, b1) in ents.items():
        g = int(key[1:key.index(".")])
        k = src_of[mods.index(table[g][0])]
        assert torch.equal(dst[b0:b1], shards[k][b0:b1]), key
    wp = t.MergePartition(fam, yaml, -1, r, N)
    wp.bind([wbufs[k - 1].data_ptr() + (wlo - lo) for k, c, wlo, whi in wp.windows()])
    wdst = torch.empty(wp.bytes, dtype=torch.uint8, device=dev)
    wp.run(wdst.data_ptr())
    torch.cuda.synchronize()
    went = entries(wp.prefix())
    for tname, (b0, b1) in went.items():
        if b1 <= lo or b0 >= hi:
            continue
        mod = ".".join(tname.split(".")[:2]) if tname.startswith("layers.") else tname.split(".")[0]
        k = src_of[mods.index(mod)]
        assert torch.equal(wdst[b0 - lo:b1 - lo], wbufs[k][b0 - lo:b1 - lo]), tname

    # ---- generator spot checks vs the CPU oracle ------------------------------------------
    rng = np.random.default_rng(0)
    for g in (0, 1, spec.num_layers + 1, len(table) - 1):
        c = o.shard_length(table[g][2], N)
        idx = rng.integers(0, c, 64)
        go = r * c + idx
        valid = go < table[g][2]
        sl = o.group_slices(s, g)
        e = np.zeros(idx.size, dtype=np.uint64)
        for j, x in enumerate(go):
            for _, _, goff, moff in reversed(sl):
                if x >= goff:
                    e[j] = moff + (x - goff)
                    break
        mi = np.full(idx.size, mods.index(table[g][0]))
        for k in range(1, K + 1):
            w, m_, v_ = o.element_values(s, k, e, mi)
            for field, vals in ((".master", w), (".exp_avg", m_), (".exp_avg_sq", v_)):
                b0, _ = ents[f"g{g}{field}"]
                dv = shards[k - 1][b0:b0 + 4 * c].view(torch.float32)[torch.as_tensor(idx, device=dev)].cpu().numpy()
                want = np.where(valid, vals, np.float32(0))
                assert np.array_equal(dv.view(np.uint32), want.astype(np.float32).view(np.uint32)), (g, k, field)
