"""N>1 path on CPU: world_size-2 gloo processes stand in for GPUs. GPU g owns ZeRO
rank partitions {r : r % G == g}; each computes FP64 partial sums for its
partitions, the partials are all-gathered (the only collective on the path), every
process combines in rank order and runs the same selection -> identical recipes,
equal to the single-process result; the per-unit merge plans tile the composite."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2602_22158_b200 as t
import tailor_oracle as o

SPEC = dict(num_layers=5, hidden_dim=8, ffn_dim=20, vocab_size=24, weight_tied=False, seed=77)
N, K, RHO = 4, 4, 0.5


def rank_partials(r):
    """[K-1][M][2] FP64 partial sums over rank r's chunk of every group (oracle)."""
    import numpy as np

    W = [o.model_vectors(SPEC, k)[0] for k in range(1, K + 1)]
    table = o.group_table(SPEC)
    out = []
    for p in range(K - 1):
        row = []
        for m in o.modules(SPEC):
            sd = sr = 0.0
            for g in o.group_indices_for(SPEC, m):
                c = o.shard_length(table[g][2], N)
                a = o.group_vectors(SPEC, W[p], g)[r * c:(r + 1) * c].astype(np.float64)
                b = o.group_vectors(SPEC, W[p + 1], g)[r * c:(r + 1) * c].astype(np.float64)
                sd += float(np.dot(b - a, b - a))
                sr += float(np.dot(a, a))
            row.append([sd, sr])
        out.append(row)
    return out


def flat(x):
    return [v for p in x for m in p for v in m]


def spec_obj():
    return t.ModelSpec(SPEC["num_layers"], SPEC["hidden_dim"], SPEC["ffn_dim"], SPEC["vocab_size"], False, SPEC["seed"])


def worker(g, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=g, world_size=world)
    mine = [r for r in range(N) if r % world == g]
    local = torch.tensor([flat(rank_partials(r)) for r in mine], dtype=torch.float64)
    gathered = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(gathered, local)
    by_rank = {}
    for src, block in enumerate(gathered):
        for i, r in enumerate([r for r in range(N) if r % world == src]):
            by_rank[r] = block[i].tolist()
    parts = [v for r in range(N) for v in by_rank[r]]
    fam = t.SynthFamily(spec_obj(), N, K)
    yaml, src_of, scores, gap = fam.select(parts, N, RHO)
    # units owned by this process: its shard partitions + weights shares
    cover = []
    for r in mine:
        mpn = t.MergePartition(fam, yaml, -1, r, N)
        lo, hi, total = mpn.range()
        cover.append((lo, hi, total, t.MergePartition(fam, yaml, r).bytes))
    q.put((g, yaml, src_of, cover))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_gloo_selection_and_partition():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = free_port()
    procs = [ctx.Process(target=worker, args=(g, world, port, q)) for g in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    yamls = {r[1] for r in res}
    assert len(yamls) == 1  # every process made the same selection without a broadcast
    # single-process reference: all partials in rank order
    fam = t.SynthFamily(spec_obj(), N, K)
    parts = [v for r in range(N) for v in flat(rank_partials(r))]
    yaml, src_of, _, _ = fam.select(parts, N, RHO)
    assert yamls == {yaml}
    assert all(r[2] == src_of for r in res)
    # and equal to the oracle's full-module scores
    W = [o.model_vectors(SPEC, k)[0] for k in range(1, K + 1)]
    sc = [[o.magnitude_score(*x) for x in o.score_pair(SPEC, W[p], W[p + 1])] for p in range(K - 1)]
    assert o.select(sc, len(o.modules(SPEC)), RHO)[1] == src_of
    # weights shares of all units tile the composite weights payload
    cov = sorted(c for r in res for c in r[3])
    assert cov[0][0] == 0 and cov[-1][1] == cov[-1][2]
    assert all(a[1] == b[0] for a, b in zip(cov, cov[1:]))
