"""Python mirror of the reference's tailoring interface, bound to the B200 engine.

Names and semantics follow the reference's C++ surface so parity tests read
like the reference's own tests:

* ``parse_recipe`` / ``recipe_to_yaml``   — R/src/recipe.cpp:67-169
* ``resolve_plan``                        — R/src/merge.cpp:39-152
* ``execute_merge``                       — R/src/merge.cpp:226-357 (device gather + device re-verify)
* ``recipe_from_manifests``               — R/src/merge.cpp:359-418
* ``score_snapshots`` / ``select_recipe`` — the update-magnitude strategy
* ``SynthFamily`` / ``Scorer`` / ``MergePartition`` — device-resident partitions (bench, multi-GPU)

Every call goes through ``libtailor_b200.so`` (include/tailor_b200.h); errors
surface as :class:`TailorError` with the reference's ``ErrorKind``.
"""
from __future__ import annotations

import ctypes
import dataclasses
import json
import os
from typing import Dict, List, Optional, Sequence

from ._lib import (ErrorKind, GatherSegC, HostCopyC, MergeOptionsC, MergeStatsC, ModelSpecC, TailorError, check,
                   check_handle, lib, ptr_array, text_call)

__all__ = ["ErrorKind", "TailorError", "ModelSpec", "RecipeSlice", "MergeRecipe", "MergeOptions", "MergeStats",
           "parse_recipe", "recipe_to_yaml", "resolve_plan", "execute_merge", "recipe_from_manifests",
           "verify_checkpoint", "regroup", "train", "resume", "score_snapshots", "select_recipe", "select_merge", "layer_map", "SnapshotLayout", "SynthFamily", "Scorer",
           "MergePartition", "SelectStep", "Trainer", "Comm", "STRATEGIES", "gather", "read_probe"]


@dataclasses.dataclass
class ModelSpec:
    """R/include/tailor/model.hpp:14-30."""

    num_layers: int
    hidden_dim: int
    ffn_dim: int
    vocab_size: int
    weight_tied: bool = False
    seed: int = 42

    def to_c(self) -> ModelSpecC:
        return ModelSpecC(self.num_layers, self.hidden_dim, self.ffn_dim, self.vocab_size,
                          1 if self.weight_tied else 0, 0, self.seed)

    @classmethod
    def from_config(cls, text: str) -> "ModelSpec":
        """parse_config_json (R/src/checkpoint.cpp:123-136) through tg_parse_config."""
        c = ModelSpecC()
        check(lib().tg_parse_config(text.encode(), ctypes.byref(c)))
        return cls(c.num_layers, c.hidden_dim, c.ffn_dim, c.vocab_size, bool(c.weight_tied), c.seed)

    @property
    def module_count(self) -> int:
        return self.num_layers + (2 if self.weight_tied else 3)


@dataclasses.dataclass
class RecipeSlice:
    source: str
    layers: List[int]
    targets: Optional[List[int]] = None

    def __post_init__(self):
        if self.targets is None:
            self.targets = list(self.layers)


@dataclasses.dataclass
class MergeRecipe:
    """R/include/tailor/recipe.hpp:19-25."""

    num_ranks: int = 0
    base_checkpoint: str = ""
    slices: List[RecipeSlice] = dataclasses.field(default_factory=list)
    aux: Dict[str, str] = dataclasses.field(default_factory=dict)
    config_from: str = "latest"

    def to_json(self) -> str:
        return json.dumps({"base_checkpoint": self.base_checkpoint, "num_ranks": self.num_ranks,
                           "slices": [{"source": s.source, "layers": s.layers, "targets": s.targets}
                                      for s in self.slices],
                           "aux": self.aux, "config_from": self.config_from})

    @staticmethod
    def from_json(text: str) -> "MergeRecipe":
        j = json.loads(text)
        return MergeRecipe(num_ranks=j["num_ranks"], base_checkpoint=j["base_checkpoint"],
                           slices=[RecipeSlice(s["source"], s["layers"], s["targets"]) for s in j["slices"]],
                           aux=dict(j["aux"]), config_from=j["config_from"])

    def to_yaml(self) -> str:
        return recipe_to_yaml(self)


@dataclasses.dataclass
class MergeOptions:
    """R/include/tailor/merge.hpp:46-49 (+ device, verify, devices: the output lanes
    spread round-robin over these GPUs; the bytes written do not depend on them)."""

    workers: int = 0
    uncached: bool = False
    device: int = 0
    verify: bool = True
    devices: Optional[Sequence[int]] = None
    io_mode: str = "auto"  # auto | buffered | direct | direct-rw (tailor/io.hpp; TAILOR_IO overrides)

    def to_c(self):
        devs = list(self.devices or [])
        arr = (ctypes.c_int32 * max(1, len(devs)))(*devs)
        c = MergeOptionsC(self.workers, 1 if self.uncached else 0, self.device, 0 if self.verify else 1,
                          ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32)), len(devs), IO_MODES[self.io_mode])
        c._keep = arr  # the array must outlive the call
        return c


IO_MODES = {"auto": 0, "buffered": 1, "direct": 2, "direct-rw": 3}


@dataclasses.dataclass
class MergeStats:
    """R/include/tailor/merge.hpp:51-55 (+ device_ms, bytes_moved)."""

    shard_files_read: int
    weight_files_read: int
    wall_ms: float
    device_ms: float
    bytes_moved: int
    direct_read_bytes: int = 0
    direct_write_bytes: int = 0
    resident_bytes: int = 0  # source bytes gathered from device copies (select_merge), not read

    @classmethod
    def from_c(cls, st) -> "MergeStats":
        return cls(st.shard_files_read, st.weight_files_read, st.wall_ms, st.device_ms, st.bytes_moved,
                   st.direct_read_bytes, st.direct_write_bytes, st.resident_bytes)


def _b(s: str) -> bytes:
    return os.fsencode(s)


def parse_recipe(yaml_text: str) -> MergeRecipe:
    return MergeRecipe.from_json(text_call(lib().tg_parse_recipe, yaml_text.encode()))


def recipe_to_yaml(recipe: MergeRecipe) -> str:
    return text_call(lib().tg_recipe_to_yaml, recipe.to_json().encode())


def _yaml_of(recipe) -> bytes:
    return (recipe if isinstance(recipe, str) else recipe_to_yaml(recipe)).encode()


def resolve_plan(recipe) -> dict:
    """MergePlan as a dict: num_ranks, config_source, sources, group_copies, assignment."""
    return json.loads(text_call(lib().tg_resolve_plan, _yaml_of(recipe)))


def execute_merge(recipe, out_dir: str, options: Optional[MergeOptions] = None) -> MergeStats:
    o = options or MergeOptions()
    copt = o.to_c()
    st = MergeStatsC()
    check(lib().tg_execute_merge(_yaml_of(recipe), _b(str(out_dir)), ctypes.byref(copt), ctypes.byref(st)))
    return MergeStats.from_c(st)


def recipe_from_manifests(run_dir: str, failure_step: int) -> MergeRecipe:
    return parse_recipe(text_call(lib().tg_recipe_from_manifests, _b(str(run_dir)), failure_step))


def regroup(src_dir: str, out_dir: str, to_fine: bool = True, options: Optional[MergeOptions] = None) -> MergeStats:
    """coarse_to_fine / fine_to_coarse of a checkpoint directory on the device (R/src/groups.cpp:152-220)."""
    o = options or MergeOptions()
    copt = dataclasses.replace(o, uncached=False).to_c()
    st = MergeStatsC()
    check(lib().tg_regroup(_b(str(src_dir)), _b(str(out_dir)), 1 if to_fine else 0, ctypes.byref(copt),
                           ctypes.byref(st)))
    return MergeStats.from_c(st)


STRATEGIES = {"full": 0, "parity": 1, "filter": 2, "magnitude": 3}


def train(spec: ModelSpec, out_dir: str, steps: int, interval: int = 50, strategy: str = "full", num_ranks: int = 1,
          lr: float = 1e-3, weight_decay: float = 0.01, head: int = 2, tail: int = 2, sparse_multiple: int = 5,
          rho: float = 0.5, device: int = 0) -> int:
    """Device-resident train() (R/src/trainer.cpp:109-123) -> number of checkpoints written.
    strategy 'magnitude' saves all modules at the first checkpoint, then the top-rho by
    update magnitude against the previous checkpoint (scored in situ)."""
    from ._lib import TrainConfigC

    c = spec.to_c()
    cfg = TrainConfigC(steps, num_ranks, interval, STRATEGIES[strategy], head, tail, sparse_multiple, device, lr,
                       weight_decay, rho)
    n = ctypes.c_int32(0)
    check(lib().tg_train(ctypes.byref(c), ctypes.byref(cfg), _b(str(out_dir)), ctypes.byref(n)))
    return n.value


def resume(checkpoint_dir: str, steps: int, out_dir: str, device: int = 0) -> int:
    """Device resume() (R/src/trainer.cpp:125-152) from a complete fine checkpoint ->
    number of checkpoints written into out_dir."""
    n = ctypes.c_int32(0)
    check(lib().tg_resume(_b(str(checkpoint_dir)), steps, _b(str(out_dir)), device, ctypes.byref(n)))
    return n.value


def verify_checkpoint(path: str, device: int = 0) -> None:
    check(lib().tg_verify_checkpoint(_b(str(path)), device))


def _dirs_arg(dirs: Sequence[str]):
    arr = (ctypes.c_char_p * len(dirs))()
    for i, d in enumerate(dirs):
        arr[i] = _b(str(d))
    return arr


def _devices_arg(device: int, devices):
    devs = list(devices) if devices else [device]
    return (ctypes.c_int32 * len(devs))(*devs), len(devs)


def score_snapshots(dirs: Sequence[str], device: int = 0, devices: Optional[Sequence[int]] = None):
    """Device scores over consecutive snapshot dirs (any number >= 2) -> (sums[p][m][2], scores[p][m]).
    `devices`: rank partitions are scored by lanes spread over these GPUs (same result)."""
    n = len(dirs)
    cap = max(1, (n - 1)) * 8192
    sums = (ctypes.c_double * (cap * 2))()
    scores = (ctypes.c_double * cap)()
    m = ctypes.c_int32(0)
    darr, nd = _devices_arg(device, devices)
    check(lib().tg_score_snapshots(_dirs_arg(dirs), n, darr, nd, sums, scores, ctypes.byref(m)))
    M = m.value
    return ([[[sums[(p * M + i) * 2], sums[(p * M + i) * 2 + 1]] for i in range(M)] for p in range(n - 1)],
            [[scores[p * M + i] for i in range(M)] for p in range(n - 1)])


def select_recipe(dirs: Sequence[str], rho: float = 0.5, device: int = 0, devices: Optional[Sequence[int]] = None):
    """Score -> magnitude selection -> recipe. Returns (recipe, source_of, min_boundary_gap)."""
    src = (ctypes.c_int32 * 8192)()
    gap = ctypes.c_double(0)
    darr, nd = _devices_arg(device, devices)
    yaml = text_call(lambda b, c, n: lib().tg_select_recipe(_dirs_arg(dirs), len(dirs), rho, darr, nd, b, c, n, src,
                                                             ctypes.byref(gap)))
    rec = parse_recipe(yaml)
    M = None
    # source_of length = module count; recover from the layer map of the first snapshot's spec.
    with open(os.path.join(str(dirs[0]), "config.json")) as f:
        cfg = json.load(f)
    M = cfg["num_layers"] + (2 if cfg["weight_tied"] else 3)
    return rec, [src[i] for i in range(M)], gap.value


def select_merge(dirs: Sequence[str], out_dir: str, rho: float = 0.5, options: Optional[MergeOptions] = None):
    """select_recipe + execute_merge in one call (tg_select_merge): the masters the scorer
    read stay on the device for the merge when they fit. Returns (recipe, source_of,
    min_boundary_gap, MergeStats)."""
    o = options or MergeOptions()
    copt = o.to_c()
    st = MergeStatsC()
    src = (ctypes.c_int32 * 8192)()
    gap = ctypes.c_double(0)
    cap = 1 << 20
    buf = ctypes.create_string_buffer(cap)
    need = ctypes.c_size_t(0)
    check(lib().tg_select_merge(_dirs_arg(dirs), len(dirs), rho, _b(str(out_dir)), ctypes.byref(copt), ctypes.byref(st),
                                buf, cap, ctypes.byref(need), src, ctypes.byref(gap)))
    with open(os.path.join(str(dirs[0]), "config.json")) as f:
        cfg = json.load(f)
    M = cfg["num_layers"] + (2 if cfg["weight_tied"] else 3)
    return parse_recipe(buf.value.decode()), [src[i] for i in range(M)], gap.value, MergeStats.from_c(st)


def layer_map(spec: ModelSpec, num_ranks: int = 1) -> dict:
    c = spec.to_c()
    return json.loads(text_call(lambda b, cap, n: lib().tg_layer_map(ctypes.byref(c), num_ranks, b, cap, n)))


def gather(d_segs_ptr: int, nseg: int, d_dst: int, dst_bytes: int, variant: int = 0, bulk_ok: bool = False,
           stream: int = 0) -> None:
    """Raw K2 launch over a device segment table (tg_gather)."""
    check(lib().tg_gather(d_segs_ptr, nseg, d_dst, dst_bytes, variant, 1 if bulk_ok else 0, stream))


def read_probe(d_src: int, nbytes: int, d_sink: int, stream: int = 0) -> None:
    """Read-only HBM stream over a device buffer (measurement; tg_read_probe)."""
    check(lib().tg_read_probe(d_src, nbytes, d_sink, stream))


class SnapshotLayout:
    """Layouts of snapshots S_1..S_K (tg_layout_*): what the scorer, merge plans and the
    device select step are built from. Synthetic (`SnapshotLayout(spec, N, K)`: complete
    snapshots, ids "S1".."SK") or read from checkpoint directories
    (`SnapshotLayout.from_checkpoints(dirs)`: ids are the paths). It holds no payload
    bytes; the caller binds its own device buffers (rank-shard / weights payload layout)."""

    def __init__(self, spec: Optional[ModelSpec] = None, num_ranks: int = 1, snapshots: int = 1, interval: int = 100,
                 _handle=None, _owner=None):
        self._owner = _owner  # a SynthFamily whose layout this is (keeps it alive; not destroyed here)
        if _handle is not None:
            self._h, self._owned = _handle, False
        else:
            c = spec.to_c()
            self._h, self._owned = check_handle(lib().tg_layout_create(ctypes.byref(c), num_ranks, snapshots,
                                                                       interval)), True

    @classmethod
    def from_checkpoints(cls, dirs: Sequence[str]) -> "SnapshotLayout":
        h = check_handle(lib().tg_layout_from_checkpoints(_dirs_arg(dirs), len(dirs)))
        obj = cls(_handle=h)
        obj._owned = True
        return obj

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owned", False):
            lib().tg_layout_destroy(h)
        self._h = None

    @property
    def layout_handle(self):
        return self._h

    @property
    def num_modules(self) -> int:
        return lib().tg_layout_num_modules(self._h)

    @property
    def num_ranks(self) -> int:
        return lib().tg_layout_num_ranks(self._h)

    @property
    def snapshots(self) -> int:
        return lib().tg_layout_snapshots(self._h)

    @property
    def parameter_count(self) -> int:
        return lib().tg_layout_parameter_count(self._h)

    def set_partial(self, k: int, modules: Sequence[str]) -> None:
        check(lib().tg_layout_set_partial(self._h, k, ",".join(modules).encode()))

    def set_id(self, k: int, ident: str) -> None:
        check(lib().tg_layout_set_id(self._h, k, ident.encode()))

    def shard_bytes(self, k: int, rank: int) -> int:
        return lib().tg_layout_shard_bytes(self._h, k, rank)

    def weights_bytes(self, k: int) -> int:
        return lib().tg_layout_weights_bytes(self._h, k)

    def packed_master_bytes(self, rank: int) -> int:
        return lib().tg_layout_packed_master_bytes(self._h, rank)

    def select(self, rank_partials: Sequence[float], nranks: int, rho: float = 0.5):
        """Combine [nranks][K-1][M][2] partials in rank order -> (recipe_yaml, source_of, scores, gap)."""
        M, K = self.num_modules, self.snapshots
        arr = (ctypes.c_double * len(rank_partials))(*rank_partials)
        src = (ctypes.c_int32 * M)()
        scores = (ctypes.c_double * max(1, (K - 1) * M))()
        gap = ctypes.c_double(0)
        yaml = text_call(lambda b, c, n: lib().tg_layout_select(self._h, arr, nranks, rho, b, c, n, src, scores,
                                                                 ctypes.byref(gap)))
        return (yaml, [src[i] for i in range(M)],
                [[scores[p * M + m] for m in range(M)] for p in range(K - 1)], gap.value)


class SynthFamily(SnapshotLayout):
    """Synthetic snapshots S_1..S_K of SURVEY §8(d): a SnapshotLayout plus the device
    generator (K5) of their payloads."""

    def __init__(self, spec: ModelSpec, num_ranks: int, snapshots: int, interval: int = 100):
        self.spec, self.interval = spec, interval
        c = spec.to_c()
        self._fh = check_handle(lib().tg_family_create(ctypes.byref(c), num_ranks, snapshots, interval))
        super().__init__(_handle=lib().tg_family_layout(self._fh))

    def __del__(self):
        self._h = None  # the layout view belongs to the family
        h = getattr(self, "_fh", None)
        if h:
            lib().tg_family_destroy(h)
            self._fh = None

    @property
    def handle(self):
        return self._fh

    @property
    def layout(self) -> SnapshotLayout:
        return SnapshotLayout(_handle=self._h, _owner=self)

    def gen_shard(self, rank: int, k0: int, k1: int, outs: Sequence[int], stream: int = 0) -> None:
        check(lib().tg_family_gen_shard(self._fh, rank, k0, k1, ptr_array(outs), stream))

    def gen_weights(self, k0: int, k1: int, lo: int, hi: int, outs: Sequence[int], stream: int = 0) -> None:
        check(lib().tg_family_gen_weights(self._fh, k0, k1, lo, hi, ptr_array(outs), stream))

    def gen_masters(self, rank: int, k0: int, k1: int, outs: Sequence[int], stream: int = 0) -> None:
        check(lib().tg_family_gen_masters(self._fh, rank, k0, k1, ptr_array(outs), stream))

    def gen_shard_range(self, rank: int, k: int, lo: int, hi: int, out: int, stream: int = 0) -> None:
        """Bytes [lo, hi) of snapshot k's rank shard payload (tensor-aligned window)."""
        check(lib().tg_family_gen_shard_range(self._fh, rank, k, lo, hi, out, stream))

    def write_dir(self, k: int, path: str) -> None:
        check(lib().tg_family_write_dir(self._fh, k, _b(str(path))))


class Scorer:
    """K3/K4 scorer plan for one rank partition of snapshots k0..k1 of a layout (or family)."""

    def __init__(self, layout: SnapshotLayout, rank: int, k0: int, k1: int, packed: bool = False):
        self._fam = layout
        self._h = check_handle(lib().tg_scorer_create(layout.layout_handle, rank, k0, k1, 1 if packed else 0))
        self.K = k1 - k0 + 1

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tg_scorer_destroy(h)
            self._h = None

    @property
    def bytes_read(self) -> int:
        return lib().tg_scorer_bytes(self._h)

    def run(self, bases: Sequence[int], d_out: int, stream: int = 0) -> None:
        check(lib().tg_scorer_run(self._h, ptr_array(bases), d_out, stream))

    def set_variant(self, variant: int) -> None:
        """0 auto, 1 register-staged loads, 2 TMA-bulk shared-memory ring."""
        check(lib().tg_scorer_set_variant(self._h, variant))


class MergePartition:
    """K2 plan for one output partition: container=-1 -> weights share unit/units, r -> rank-r shard
    (units > 1: its unit-th tensor-aligned byte sub-range)."""

    def __init__(self, layout: SnapshotLayout, recipe_yaml: str, container: int, unit: int = 0, units: int = 1):
        self._fam = layout
        self._h = check_handle(lib().tg_mplan_create(layout.layout_handle, recipe_yaml.encode(), container, unit,
                                                     units))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tg_mplan_destroy(h)
            self._h = None

    @property
    def bytes(self) -> int:
        return lib().tg_mplan_bytes(self._h)

    @property
    def num_segments(self) -> int:
        return lib().tg_mplan_num_segments(self._h)

    def segments(self):
        """[(window, src_off, dst_off, bytes)]: the byte copies of this plan (host view)."""
        out = []
        for i in range(self.num_segments):
            w, so, do, n = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
            check(lib().tg_mplan_segment(self._h, i, ctypes.byref(w), ctypes.byref(so), ctypes.byref(do), ctypes.byref(n)))
            out.append((w.value, so.value, do.value, n.value))
        return out

    @property
    def bulk_ok(self) -> bool:
        return bool(lib().tg_mplan_bulk_ok(self._h))

    def range(self):
        lo, hi, pb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().tg_mplan_range(self._h, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(pb)))
        return lo.value, hi.value, pb.value

    def windows(self):
        out = []
        for i in range(lib().tg_mplan_num_windows(self._h)):
            k, c, lo, hi = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_uint64(), ctypes.c_uint64()
            check(lib().tg_mplan_window(self._h, i, ctypes.byref(k), ctypes.byref(c), ctypes.byref(lo),
                                        ctypes.byref(hi)))
            out.append((k.value, c.value, lo.value, hi.value))
        return out

    def prefix(self) -> bytes:
        need = ctypes.c_size_t(0)
        lib().tg_mplan_prefix(self._h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        check(lib().tg_mplan_prefix(self._h, buf, need.value, ctypes.byref(need)))
        return buf.raw[:need.value]

    def bind(self, window_ptrs: Sequence[int]) -> None:
        check(lib().tg_mplan_bind(self._h, ptr_array(window_ptrs)))

    def run(self, d_dst: int, variant: int = 0, stream: int = 0) -> None:
        check(lib().tg_mplan_run(self._h, d_dst, variant, stream))

    def run_host(self, h_windows: Sequence[int], h_dst: int, variant: int = 0, chunk_bytes: int = 0,
                 d_windows: Optional[Sequence[int]] = None, resident_fields: int = 0, async_: bool = False,
                 prefetch: Optional[Sequence[tuple]] = None):
        """Shard pipeline from pinned host windows; `resident_fields` (1 exp_avg, 2 exp_avg_sq,
        4 master) are read from `d_windows` instead of crossing PCIe. `prefetch`: extra
        (host_src, device_dst, bytes) copies interleaved on the pipeline's H2D stream."""
        h2d, d2h = ctypes.c_uint64(), ctypes.c_uint64()
        dw = ptr_array(d_windows) if d_windows is not None else None
        pf = (HostCopyC * max(1, len(prefetch or ())))(*[HostCopyC(int(s), int(d), int(n)) for s, d, n in prefetch or ()])
        check(lib().tg_mplan_run_host(self._h, ptr_array(h_windows), dw, resident_fields if dw else 0, h_dst, variant,
                                      chunk_bytes, 1 if async_ else 0, pf, len(prefetch or ()), ctypes.byref(h2d),
                                      ctypes.byref(d2h)))
        return h2d.value, d2h.value

    def wait(self) -> None:
        check(lib().tg_mplan_wait(self._h))


class Trainer:
    """Resident device trainer over rank partitions [rank_begin, rank_end) (tg_trainer_*)."""

    def __init__(self, spec: ModelSpec, num_ranks: int, rank_begin: int = 0, rank_end: int = -1, lr: float = 1e-3,
                 weight_decay: float = 0.01, device: int = 0):
        c = spec.to_c()
        self._h = check_handle(lib().tg_trainer_create(ctypes.byref(c), num_ranks, rank_begin, rank_end, lr,
                                                       weight_decay, device))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tg_trainer_destroy(h)
            self._h = None

    @property
    def elements(self) -> int:
        return lib().tg_trainer_elements(self._h)

    def step(self, step: int):
        g, u = ctypes.c_double(), ctypes.c_double()
        check(lib().tg_trainer_step(self._h, step, ctypes.byref(g), ctypes.byref(u)))
        return g.value, u.value

    def partition(self, rank: int):
        """(device pointer, bytes) of a held rank partition (rank_<r>.shard payload layout)."""
        ptr, n = ctypes.c_void_p(), ctypes.c_uint64()
        check(lib().tg_trainer_partition(self._h, rank, ctypes.byref(ptr), ctypes.byref(n)))
        return ptr.value, n.value


class SelectStep:
    """Device score -> select -> merge step for one unit of a family of full snapshots
    (tg_dstep_*): selection and segment tables built on the device, no host sync."""

    def __init__(self, layout: SnapshotLayout, rank: int, unit: int, units: int, rho: float = 0.5):
        self._fam = layout
        self.K, self.M = layout.snapshots, layout.num_modules
        self._h = check_handle(lib().tg_dstep_create(layout.layout_handle, rank, unit, units, rho))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tg_dstep_destroy(h)
            self._h = None

    def range(self):
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().tg_dstep_range(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value  # shard bytes, weights lo, weights hi

    def bind(self, shard_bases: Sequence[int], weights_window_bases: Sequence[int]) -> None:
        check(lib().tg_dstep_bind(self._h, ptr_array(shard_bases), ptr_array(weights_window_bases)))

    def run(self, d_partials: int, nranks: int, d_out_shard: int, d_out_weights: int, variant: int = 0,
            stream: int = 0, phases: int = 7) -> None:
        """phases: 1 select+plan, 2 gather shard, 4 gather weights (bitmask)."""
        check(lib().tg_dstep_run(self._h, d_partials, nranks, d_out_shard, d_out_weights, variant, phases, stream))

    def result(self, stream: int = 0):
        src = (ctypes.c_int32 * self.M)()
        sc = (ctypes.c_double * max(1, (self.K - 1) * self.M))()
        check(lib().tg_dstep_result(self._h, src, sc, stream))
        return [src[i] for i in range(self.M)], [[sc[p * self.M + m] for m in range(self.M)] for p in range(self.K - 1)]


class Comm:
    """NCCL communicator of one GPU of a job (tg_comm_*): the score-partials all-gather.
    Rank 0 calls `Comm.unique_id()` and ships the 128 bytes to every rank (any channel);
    the constructor is collective."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        check(lib().tg_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int = 0):
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._h = check_handle(lib().tg_comm_create(buf, nranks, rank, device))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().tg_comm_destroy(h)
            self._h = None

    def all_gather(self, d_send: int, d_recv: int, count: int, stream: int = 0) -> None:
        """d_recv[r * count + i] = rank r's d_send[i] (FP64 device buffers), async on `stream`."""
        check(lib().tg_comm_allgather(self._h, d_send, d_recv, count, stream))
