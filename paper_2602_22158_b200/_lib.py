"""ctypes binding of the C ABI in include/tailor_b200.h.

The shared library is built in-tree (``__graft_entry__.build()`` ->
``paper_2602_22158_b200/libtailor_b200.so``). There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import enum
import pathlib

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libtailor_b200.so"
CLI_PATH = HERE / "bin" / "tailor"


class ErrorKind(enum.IntEnum):
    """R/include/tailor/errors.hpp:12-24 (+ Device, + Internal)."""

    InvalidModule = 1
    Geometry = 2
    NonFinite = 3
    Recipe = 4
    SourceLacksModule = 5
    MissingArtifact = 6
    CorruptContainer = 7
    UnrecoverableModule = 8
    MissingModules = 9
    Consistency = 10
    Storage = 11
    Device = 12
    Internal = 100


class TailorError(RuntimeError):
    """Mirrors tailor::TailorError: carries the kind; user errors exit 1."""

    def __init__(self, kind: int, message: str):
        super().__init__(message)
        self.kind = ErrorKind(kind) if kind in ErrorKind._value2member_map_ else ErrorKind.Internal

    @property
    def is_user_error(self) -> bool:
        return self.kind not in (ErrorKind.Consistency, ErrorKind.NonFinite, ErrorKind.Storage,
                                 ErrorKind.Device, ErrorKind.Internal)


class ModelSpecC(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("hidden_dim", ctypes.c_int32), ("ffn_dim", ctypes.c_int32),
                ("vocab_size", ctypes.c_int32), ("weight_tied", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("seed", ctypes.c_uint64)]


class MergeOptionsC(ctypes.Structure):
    _fields_ = [("workers", ctypes.c_int32), ("uncached", ctypes.c_int32), ("device", ctypes.c_int32),
                ("skip_verify", ctypes.c_int32), ("devices", ctypes.POINTER(ctypes.c_int32)),
                ("num_devices", ctypes.c_int32), ("io_mode", ctypes.c_int32)]


class MergeStatsC(ctypes.Structure):
    _fields_ = [("shard_files_read", ctypes.c_int64), ("weight_files_read", ctypes.c_int64),
                ("wall_ms", ctypes.c_double), ("device_ms", ctypes.c_double), ("bytes_moved", ctypes.c_uint64),
                ("direct_read_bytes", ctypes.c_uint64), ("direct_write_bytes", ctypes.c_uint64),
                ("resident_bytes", ctypes.c_uint64)]


class TrainConfigC(ctypes.Structure):
    _fields_ = [("total_steps", ctypes.c_int32), ("num_ranks", ctypes.c_int32), ("interval", ctypes.c_int32),
                ("strategy", ctypes.c_int32), ("head_count", ctypes.c_int32), ("tail_count", ctypes.c_int32),
                ("sparse_multiple", ctypes.c_int32), ("device", ctypes.c_int32), ("lr", ctypes.c_double),
                ("weight_decay", ctypes.c_double), ("rho", ctypes.c_double)]


class GatherSegC(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst_off", ctypes.c_uint64), ("bytes", ctypes.c_uint64)]


class HostCopyC(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("bytes", ctypes.c_uint64)]


class ScoreTileC(ctypes.Structure):
    _fields_ = [("module", ctypes.c_uint32), ("field", ctypes.c_uint32), ("count", ctypes.c_uint32),
                ("pad", ctypes.c_uint32), ("elem_start", ctypes.c_uint64)]


# Every symbol include/tailor_b200.h declares, with its ctypes signature.
_c = ctypes
_P = _c.c_void_p
_S = _c.c_char_p
_I = _c.c_int
_I32 = _c.c_int32
_U32 = _c.c_uint32
_I64 = _c.c_int64
_U64 = _c.c_uint64
_D = _c.c_double
_SZ = _c.c_size_t
_PSZ = _c.POINTER(_c.c_size_t)
_PP = _c.POINTER(_c.c_void_p)
SIGNATURES = {
    "tg_last_error": (_S, []),
    "tg_last_error_kind": (_I, []),
    "tg_version": (_S, []),
    "tg_device_count": (_I, []),
    "tg_parse_recipe": (_I, [_S, _c.c_char_p, _SZ, _PSZ]),
    "tg_recipe_to_yaml": (_I, [_S, _c.c_char_p, _SZ, _PSZ]),
    "tg_resolve_plan": (_I, [_S, _c.c_char_p, _SZ, _PSZ]),
    "tg_execute_merge": (_I, [_S, _S, _c.POINTER(MergeOptionsC), _c.POINTER(MergeStatsC)]),
    "tg_recipe_from_manifests": (_I, [_S, _I64, _c.c_char_p, _SZ, _PSZ]),
    "tg_verify_checkpoint": (_I, [_S, _I32]),
    "tg_regroup": (_I, [_S, _S, _I32, _c.POINTER(MergeOptionsC), _c.POINTER(MergeStatsC)]),
    "tg_train": (_I, [_c.POINTER(ModelSpecC), _c.POINTER(TrainConfigC), _S, _c.POINTER(_I32)]),
    "tg_resume": (_I, [_S, _I64, _S, _I32, _c.POINTER(_I32)]),
    "tg_trainer_create": (_P, [_c.POINTER(ModelSpecC), _I32, _I32, _I32, _D, _D, _I32]),
    "tg_trainer_destroy": (None, [_P]),
    "tg_trainer_elements": (_U64, [_P]),
    "tg_trainer_step": (_I, [_P, _I64, _c.POINTER(_D), _c.POINTER(_D)]),
    "tg_trainer_partition": (_I, [_P, _I32, _c.POINTER(_P), _c.POINTER(_U64)]),
    "tg_score_snapshots": (_I, [_c.POINTER(_S), _I32, _c.POINTER(_I32), _I32, _c.POINTER(_D), _c.POINTER(_D),
                                _c.POINTER(_I32)]),
    "tg_select_recipe": (_I, [_c.POINTER(_S), _I32, _D, _c.POINTER(_I32), _I32, _c.c_char_p, _SZ, _PSZ,
                              _c.POINTER(_I32), _c.POINTER(_D)]),
    "tg_select_merge": (_I, [_c.POINTER(_S), _I32, _D, _S, _c.POINTER(MergeOptionsC), _c.POINTER(MergeStatsC),
                             _c.c_char_p, _SZ, _PSZ, _c.POINTER(_I32), _c.POINTER(_D)]),
    "tg_layer_map": (_I, [_c.POINTER(ModelSpecC), _I32, _c.c_char_p, _SZ, _PSZ]),
    "tg_parse_config": (_I, [_S, _c.POINTER(ModelSpecC)]),
    "tg_gather": (_I, [_P, _U32, _P, _U64, _I32, _I32, _P]),
    "tg_read_probe": (_I, [_P, _U64, _P, _P]),
    "tg_score_partials": (_I, [_P, _U32, _P, _U32, _I32, _I32, _P, _P]),
    "tg_score_combine": (_I, [_P, _P, _I32, _I32, _P, _P]),
    "tg_layout_create": (_P, [_c.POINTER(ModelSpecC), _I32, _I32, _I64]),
    "tg_layout_from_checkpoints": (_P, [_c.POINTER(_S), _I32]),
    "tg_layout_destroy": (None, [_P]),
    "tg_layout_set_partial": (_I, [_P, _I32, _S]),
    "tg_layout_set_id": (_I, [_P, _I32, _S]),
    "tg_layout_num_modules": (_I32, [_P]),
    "tg_layout_num_ranks": (_I32, [_P]),
    "tg_layout_snapshots": (_I32, [_P]),
    "tg_layout_shard_bytes": (_U64, [_P, _I32, _I32]),
    "tg_layout_weights_bytes": (_U64, [_P, _I32]),
    "tg_layout_packed_master_bytes": (_U64, [_P, _I32]),
    "tg_layout_parameter_count": (_U64, [_P]),
    "tg_layout_select": (_I, [_P, _c.POINTER(_D), _I32, _D, _c.c_char_p, _SZ, _PSZ, _c.POINTER(_I32),
                              _c.POINTER(_D), _c.POINTER(_D)]),
    "tg_family_create": (_P, [_c.POINTER(ModelSpecC), _I32, _I32, _I64]),
    "tg_family_destroy": (None, [_P]),
    "tg_family_layout": (_P, [_P]),
    "tg_family_gen_shard": (_I, [_P, _I32, _I32, _I32, _PP, _P]),
    "tg_family_gen_weights": (_I, [_P, _I32, _I32, _U64, _U64, _PP, _P]),
    "tg_family_gen_masters": (_I, [_P, _I32, _I32, _I32, _PP, _P]),
    "tg_family_gen_shard_range": (_I, [_P, _I32, _I32, _U64, _U64, _P, _P]),
    "tg_family_write_dir": (_I, [_P, _I32, _S]),
    "tg_scorer_create": (_P, [_P, _I32, _I32, _I32, _I32]),
    "tg_scorer_destroy": (None, [_P]),
    "tg_scorer_bytes": (_U64, [_P]),
    "tg_scorer_set_variant": (_I, [_P, _I32]),
    "tg_scorer_run": (_I, [_P, _PP, _P, _P]),
    "tg_mplan_create": (_P, [_P, _S, _I32, _I32, _I32]),
    "tg_mplan_destroy": (None, [_P]),
    "tg_mplan_bytes": (_U64, [_P]),
    "tg_mplan_range": (_I, [_P, _c.POINTER(_U64), _c.POINTER(_U64), _c.POINTER(_U64)]),
    "tg_mplan_num_windows": (_I32, [_P]),
    "tg_mplan_window": (_I, [_P, _I32, _c.POINTER(_I32), _c.POINTER(_I32), _c.POINTER(_U64), _c.POINTER(_U64)]),
    "tg_mplan_num_segments": (_U32, [_P]),
    "tg_mplan_segment": (_I, [_P, _U32, _c.POINTER(_U32), _c.POINTER(_U64), _c.POINTER(_U64), _c.POINTER(_U64)]),
    "tg_mplan_prefix": (_I, [_P, _c.c_char_p, _SZ, _PSZ]),
    "tg_mplan_bind": (_I, [_P, _PP]),
    "tg_mplan_bulk_ok": (_I32, [_P]),
    "tg_mplan_run": (_I, [_P, _P, _I32, _P]),
    "tg_mplan_run_host": (_I, [_P, _PP, _PP, _U32, _P, _I32, _U64, _I32, _c.POINTER(HostCopyC), _U32,
                               _c.POINTER(_U64), _c.POINTER(_U64)]),
    "tg_mplan_wait": (_I, [_P]),
    "tg_dstep_create": (_P, [_P, _I32, _I32, _I32, _D]),
    "tg_dstep_destroy": (None, [_P]),
    "tg_dstep_range": (_I, [_P, _c.POINTER(_U64), _c.POINTER(_U64), _c.POINTER(_U64)]),
    "tg_dstep_bind": (_I, [_P, _PP, _PP]),
    "tg_dstep_run": (_I, [_P, _P, _I32, _P, _P, _I32, _I32, _P]),
    "tg_dstep_result": (_I, [_P, _c.POINTER(_I32), _c.POINTER(_D), _P]),
    "tg_comm_unique_id": (_I, [_c.POINTER(_c.c_uint8)]),
    "tg_comm_create": (_P, [_c.POINTER(_c.c_uint8), _I32, _I32, _I32]),
    "tg_comm_destroy": (None, [_P]),
    "tg_comm_allgather": (_I, [_P, _P, _P, _U64, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise TailorError(rc, lib().tg_last_error().decode(errors="replace"))


def check_handle(h):
    if not h:
        raise TailorError(lib().tg_last_error_kind(), lib().tg_last_error().decode(errors="replace"))
    return h


def text_call(fn, *args) -> str:
    """Calls a (…, buf, cap, needed) entry point, growing the buffer once."""
    cap = 1 << 16
    for _ in range(2):
        buf = ctypes.create_string_buffer(cap)
        need = ctypes.c_size_t(0)
        rc = fn(*args, buf, cap, ctypes.byref(need))
        if rc == 0:
            return buf.value.decode()
        if need.value > cap:
            cap = need.value
            continue
        check(rc)
    check(rc)
    return ""


def ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = int(p) if p is not None else 0
    return arr
