"""CPU restatement of the checkpoint-tailoring path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may import it; the product path never does.

Pinned two ways (see tests/test_oracle.py):
  * against the reference's known-answer tests (group counts, group indices,
    shard lengths, bf16 rounding, container alignment — R/tests/*.cpp), and
  * byte-for-byte against the reference itself: oracle/_ref/ref_tool (compiled
    from /root/reference/proj/src by oracle/Makefile) writes checkpoints and
    merges them; the fixtures in tests/golden/ were produced by
    tests/golden/make_golden.py from that binary.

Every function cites the reference code it restates. Numeric conventions:
FP32 generator arithmetic in numpy float32 (IEEE round-to-nearest, no FMA);
uint64 hashing with wrapping numpy uint64 ops; scorer sums in FP64.
"""
from __future__ import annotations

import json
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ---------------------------------------------------------------- layer map ---
# R/src/model.cpp:54-63 (module order), :75-107 (tensors), :123-132 (offsets)


def modules(spec) -> List[str]:
    out = ["embed_tokens"] + [f"layers.{i}" for i in range(spec["num_layers"])] + ["norm"]
    if not spec["weight_tied"]:
        out.append("lm_head")
    return out


def tensors_of(spec, m: str) -> List[Tuple[str, Tuple[int, ...], str]]:
    h, f, v = spec["hidden_dim"], spec["ffn_dim"], spec["vocab_size"]
    if m == "embed_tokens":
        return [("embed_tokens.weight", (v, h), "decay")]
    if m == "norm":
        return [("norm.weight", (h,), "no_decay")]
    if m == "lm_head":
        return [("lm_head.weight", (v, h), "decay")]
    p = m + "."
    return [(p + "input_layernorm.weight", (h,), "no_decay"),
            (p + "post_attention_layernorm.weight", (h,), "no_decay"),
            (p + "attn.q_proj.weight", (h, h), "decay"), (p + "attn.k_proj.weight", (h, h), "decay"),
            (p + "attn.v_proj.weight", (h, h), "decay"), (p + "attn.o_proj.weight", (h, h), "decay"),
            (p + "mlp.gate_proj.weight", (f, h), "decay"), (p + "mlp.up_proj.weight", (f, h), "decay"),
            (p + "mlp.down_proj.weight", (h, f), "decay")]


def numel(shape) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


def module_offsets(spec) -> Dict[str, int]:
    off, out = 0, {}
    for m in modules(spec):
        out[m] = off
        off += sum(numel(s) for _, s, _ in tensors_of(spec, m))
    return out


def parameter_count(spec) -> int:
    return sum(numel(s) for m in modules(spec) for _, s, _ in tensors_of(spec, m))


def group_table(spec) -> List[Tuple[str, str, int]]:
    """R/src/groups.cpp:40-64: [(owner, decay, element_count)] in group index order."""
    L = spec["num_layers"]

    def count(m, d):
        return sum(numel(s) for _, s, dd in tensors_of(spec, m) if dd == d)

    g = [("norm", "no_decay", count("norm", "no_decay"))]
    g += [(f"layers.{i}", "no_decay", count(f"layers.{i}", "no_decay")) for i in range(L)]
    g.append(("embed_tokens", "decay", count("embed_tokens", "decay")))
    if not spec["weight_tied"]:
        g.append(("lm_head", "decay", count("lm_head", "decay")))
    g += [(f"layers.{i}", "decay", count(f"layers.{i}", "decay")) for i in range(L)]
    return g


def group_indices_for(spec, m: str) -> List[int]:
    """R/src/groups.cpp:84-103."""
    L = spec["num_layers"]
    if m == "norm":
        return [0]
    if m == "embed_tokens":
        return [L + 1]
    if m == "lm_head":
        assert not spec["weight_tied"]
        return [L + 2]
    i = int(m.split(".")[1])
    return [1 + i, (L + 2 if spec["weight_tied"] else L + 3) + i]


def group_slices(spec, g: int) -> List[Tuple[str, Tuple[int, ...], int, int]]:
    """R/src/groups.cpp:105-133: [(name, shape, group_offset, model_offset)]."""
    owner, decay, _ = group_table(spec)[g]
    base = module_offsets(spec)[owner]
    out, go, within = [], 0, 0
    for name, shape, d in tensors_of(spec, owner):
        if d == decay:
            out.append((name, shape, go, base + within))
            go += numel(shape)
        within += numel(shape)
    return out


def shard_length(true_len: int, n: int) -> int:
    """R/src/shard.cpp:10-19."""
    return (true_len + n - 1) // n


# ---------------------------------------------------------------- container ---
# R/src/container.cpp:62-100


def container_layout(decls: Sequence[Tuple[str, str, Sequence[int]]], metadata: Optional[Dict[str, str]] = None):
    """decls: (name, 'F32'|'BF16', shape). Returns (prefix_bytes, {name: (begin, end)}, payload_bytes)."""
    entries, off, hdr = {}, 0, {}
    if metadata:
        hdr["__metadata__"] = dict(metadata)
    for name, dtype, shape in sorted(decls, key=lambda d: d[0].encode()):
        n = numel(shape) * (2 if dtype == "BF16" else 4)
        entries[name] = (off, off + n)
        hdr[name] = {"data_offsets": [off, off + n], "dtype": dtype, "shape": list(shape)}
        off += n
    text = json.dumps(hdr, separators=(",", ":"), sort_keys=True)
    text += " " * ((8 - (8 + len(text)) % 8) % 8)
    prefix = len(text).to_bytes(8, "little") + text.encode()
    return prefix, entries, off


def shard_decls(spec, n_ranks: int, groups: Sequence[int]):
    table = group_table(spec)
    out = []
    for g in groups:
        c = shard_length(table[g][2], n_ranks)
        for f in (".exp_avg", ".exp_avg_sq", ".master"):
            out.append((f"g{g}{f}", "F32", (c,)))
    return out


def weight_decls(spec, mods: Sequence[str]):
    return [(name, "BF16", shape) for m in mods for name, shape, _ in tensors_of(spec, m)]


def parse_container(data: bytes):
    """R/src/container.cpp:102-159 (header + entries; payload view)."""
    hlen = int.from_bytes(data[:8], "little")
    hdr = json.loads(data[8:8 + hlen])
    meta = hdr.pop("__metadata__", {})
    payload = data[8 + hlen:]
    ents = {k: (v["dtype"], v["shape"], v["data_offsets"]) for k, v in hdr.items()}
    return meta, ents, payload


# ---------------------------------------------------------------- bf16 -------
def bf16_round(x: np.ndarray) -> np.ndarray:
    """R/include/tailor/bf16.hpp:12-20 over float32 arrays -> uint16."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = ((b & 0x7F800000) == 0x7F800000) & ((b & 0x007FFFFF) != 0)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    q = (b >> 16) | 0x40
    return np.where(nan, q, r).astype(np.uint16)


# ---------------------------------------------------------------- generator --
# SURVEY §8(d) on the reference's counter hash (R/src/gradients.cpp:8-23).
_M1, _M2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)
SIGN_SALT, M_SALT, V_SALT, PERM_SALT = 0x51A7E5, 0xA5, 0x5A, 0x9E2A


def mix64(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def hash3(seed: int, t: int, e: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = mix64(np.array([(seed + 0x9E3779B97F4A7C15) & (2**64 - 1)], dtype=np.uint64))
        h = mix64(h ^ np.uint64((t * 0xD1B54A32D192ED03) & (2**64 - 1)))
        return mix64(h ^ (e.astype(np.uint64) * np.uint64(0x8CB92BA72F3D8DD7)))


def unit_noise(seed: int, t: int, e: np.ndarray) -> np.ndarray:
    """R/src/gradients.cpp:17-23: float(2 * ((h >> 11) * 2^-53) - 1)."""
    u = (hash3(seed, t, e) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (2.0 * u - 1.0).astype(np.float32)


def sigma_table(seed: int, M: int, j: int) -> np.ndarray:
    perm = list(range(M))
    for i in range(M - 1, 0, -1):
        r = int(hash3(seed ^ PERM_SALT, j, np.array([i], dtype=np.uint64))[0])
        k = r % (i + 1)
        perm[i], perm[k] = perm[k], perm[i]
    g = math.pow(1000.0, 1.0 / (M - 1)) if M > 1 else 1.0
    return np.array([1e-6 * math.pow(g, float(perm[m])) for m in range(M)], dtype=np.float64).astype(np.float32)


def model_vectors(spec, k: int):
    """Full flattened (model order) master / exp_avg / exp_avg_sq of snapshot k."""
    seed = spec["seed"]
    P = parameter_count(spec)
    e = np.arange(P, dtype=np.uint64)
    mods = modules(spec)
    offs = module_offsets(spec)
    mod_of = np.zeros(P, dtype=np.int64)
    for i, m in enumerate(mods):
        n = sum(numel(s) for _, s, _ in tensors_of(spec, m))
        mod_of[offs[m]:offs[m] + n] = i
    w = np.float32(0.02) * unit_noise(seed, 0, e)
    for j in range(1, k + 1):
        sig = sigma_table(seed, len(mods), j)[mod_of]
        neg = (hash3(seed ^ SIGN_SALT, j, e) >> np.uint64(63)).astype(bool)
        w = (w + np.where(neg, -sig, sig)).astype(np.float32)
    m_ = np.float32(0.1) * unit_noise(seed ^ M_SALT, k, e)
    v_ = np.abs(np.float32(0.01) * unit_noise(seed ^ V_SALT, k, e))
    return w, m_, v_


def group_vectors(spec, vec: np.ndarray, g: int) -> np.ndarray:
    return np.concatenate([vec[mo:mo + numel(s)] for _, s, _, mo in group_slices(spec, g)])


def snapshot_payloads(spec, n_ranks: int, k: int, mods: Optional[Sequence[str]] = None):
    """Expected payload bytes of snapshot k: (weights_payload, [rank payloads]) — the
    byte image write_checkpoint (R/src/checkpoint.cpp:387-428) produces."""
    mods = list(mods) if mods is not None else modules(spec)
    mods = [m for m in modules(spec) if m in mods]
    w, m_, v_ = model_vectors(spec, k)
    groups = sorted({g for m in mods for g in group_indices_for(spec, m)})
    table = group_table(spec)
    ranks = []
    for r in range(n_ranks):
        _, ents, size = container_layout(shard_decls(spec, n_ranks, groups))
        buf = bytearray(size)
        for g in groups:
            c = shard_length(table[g][2], n_ranks)
            for field, vec in ((".master", w), (".exp_avg", m_), (".exp_avg_sq", v_)):
                full = np.zeros(c * n_ranks, dtype=np.float32)
                gv = group_vectors(spec, vec, g)
                full[:gv.size] = gv
                b, e2 = ents[f"g{g}{field}"]
                buf[b:e2] = full[r * c:(r + 1) * c].tobytes()
        ranks.append(bytes(buf))
    _, wents, wsize = container_layout(weight_decls(spec, mods))
    wbuf = bytearray(wsize)
    offs = module_offsets(spec)
    for m in mods:
        o = offs[m]
        for name, shape, _ in tensors_of(spec, m):
            n = numel(shape)
            b, e2 = wents[name]
            wbuf[b:e2] = bf16_round(w[o:o + n]).tobytes()
            o += n
    return bytes(wbuf), ranks


# ---------------------------------------------------------------- merge ------
def merge_payloads(spec, n_ranks: int, assignment: Dict[str, Tuple[str, str]],
                   sources: Dict[str, Tuple[bytes, List[bytes], Sequence[str]]]):
    """Composite assembly (R/src/merge.cpp:244-303) over in-memory source payloads.

    assignment: target module -> (source id, source module);
    sources: id -> (weights payload, rank payloads, manifest modules).
    Returns (weights payload, [rank payloads], weights prefix, [rank prefixes])."""
    table = group_table(spec)
    copies = []
    for tgt, (sid, smod) in assignment.items():
        for tg, sg in zip(group_indices_for(spec, tgt), group_indices_for(spec, smod)):
            copies.append((tg, sid, sg))
    copies.sort()
    out_ranks, prefixes = [], []
    for r in range(n_ranks):
        prefix, ents, size = container_layout(shard_decls(spec, n_ranks, [c[0] for c in copies]),
                                              {"num_ranks": str(n_ranks), "rank": str(r)})
        buf = bytearray(size)
        for tg, sid, sg in copies:
            spay = sources[sid][1][r]
            sgroups = sorted({g for m in sources[sid][2] for g in group_indices_for(spec, m)})
            _, sents, _ = container_layout(shard_decls(spec, n_ranks, sgroups))
            for f in (".exp_avg", ".exp_avg_sq", ".master"):
                b, e = ents[f"g{tg}{f}"]
                sb, se = sents[f"g{sg}{f}"]
                buf[b:e] = spay[sb:se]
        out_ranks.append(bytes(buf))
        prefixes.append(prefix)
    wdecls, wfrom = [], {}
    for tgt, (sid, smod) in assignment.items():
        for (tn, ts, _), (sn, _, _) in zip(tensors_of(spec, tgt), tensors_of(spec, smod)):
            wdecls.append((tn, "BF16", ts))
            wfrom[tn] = (sid, sn)
    wprefix, wents, wsize = container_layout(wdecls)
    wbuf = bytearray(wsize)
    for name, (b, e) in wents.items():
        sid, sn = wfrom[name]
        _, sw, _ = container_layout(weight_decls(spec, [m for m in modules(spec) if m in sources[sid][2]]))
        sb, se = sw[sn]
        wbuf[b:e] = sources[sid][0][sb:se]
    return bytes(wbuf), out_ranks, wprefix, prefixes


# ---------------------------------------------------------------- scorer -----
def score_pair(spec, A: np.ndarray, B: np.ndarray):
    """SURVEY §8 a13 over model-order master vectors: per canonical module,
    (sum (B-A)^2, sum A^2) in FP64 over the module's groups (group_indices_for order)."""
    out = []
    for m in modules(spec):
        sd = sr = 0.0
        for g in group_indices_for(spec, m):
            a = group_vectors(spec, A, g).astype(np.float64)
            b = group_vectors(spec, B, g).astype(np.float64)
            d = b - a
            sd += float(np.dot(d, d))
            sr += float(np.dot(a, a))
        out.append((sd, sr))
    return out


def magnitude_score(sd: float, sr: float) -> float:
    if sr > 0:
        return math.sqrt(sd) / math.sqrt(sr)
    return math.inf if sd > 0 else 0.0


def select(scores: Sequence[Sequence[float]], M: int, rho: float):
    """a14: saved_1 = all; saved_k = top-ceil(rho*M) by r_k, ties -> lower index;
    source(m) = max k with m in saved_k. Returns (saved, source_of, min_gap)."""
    n = max(1, min(M, math.ceil(rho * M)))
    saved = [list(range(M))]
    gap = math.inf
    for sc in scores:
        order = sorted(range(M), key=lambda i: (-sc[i], i))
        if n < M:
            hi, lo = sc[order[n - 1]], sc[order[n]]
            gap = min(gap, (hi - lo) / hi if hi > 0 else 0.0)
        saved.append(sorted(order[:n]))
    src = [0] * M
    for k, s in enumerate(saved):
        for m in s:
            src[m] = k
    return saved, src, gap


def element_values(spec, k: int, e: np.ndarray, module_index: np.ndarray):
    """(master, exp_avg, exp_avg_sq) of snapshot k at global element ids `e` whose owning
    canonical modules are `module_index` — the generator at arbitrary points, for
    full-size spot checks without materialising the model."""
    seed = spec["seed"]
    M = len(modules(spec))
    e = e.astype(np.uint64)
    w = np.float32(0.02) * unit_noise(seed, 0, e)
    for j in range(1, k + 1):
        sig = sigma_table(seed, M, j)[module_index]
        neg = (hash3(seed ^ SIGN_SALT, j, e) >> np.uint64(63)).astype(bool)
        w = (w + np.where(neg, -sig, sig)).astype(np.float32)
    return w, np.float32(0.1) * unit_noise(seed ^ M_SALT, k, e), np.abs(np.float32(0.01) * unit_noise(seed ^ V_SALT, k, e))
