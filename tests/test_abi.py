"""The C ABI boundary (CPU only: no compute calls)."""
import ctypes
import pathlib
import re
import subprocess

import paper_2602_22158_b200 as t
from paper_2602_22158_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tailor_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = t.lib()
    names = declared()
    assert len(names) >= 40
    for n in names:
        assert hasattr(lib, n), n
    # and the binding declares a signature for each one
    assert set(names) == set(_lib.SIGNATURES)


def test_exported_dynamic_symbols_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", str(t.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tg_\w+)", out))
    assert set(declared()) <= exported


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.GatherSegC) == 24
    assert ctypes.sizeof(_lib.ScoreTileC) == 24
    assert ctypes.sizeof(_lib.ModelSpecC) == 32
    assert ctypes.sizeof(_lib.MergeStatsC) == 64
    assert ctypes.sizeof(_lib.MergeOptionsC) == 32


def test_errors_are_codes_not_exceptions():
    buf = ctypes.create_string_buffer(1024)
    need = ctypes.c_size_t()
    rc = t.lib().tg_parse_recipe(b"num_ranks: 2\n", buf, 1024, ctypes.byref(need))
    assert rc == t.ErrorKind.Recipe
    assert b"merge_method" in t.lib().tg_last_error()
    assert t.lib().tg_last_error_kind() == t.ErrorKind.Recipe


def test_null_handles_are_errors_not_crashes():
    """Every handle-taking entry point reports a null handle through tg_last_error
    (no host work, no CUDA needed); getters return 0."""
    L = t.lib()
    calls = [
        lambda: L.tg_scorer_run(None, None, None, None),
        lambda: L.tg_mplan_run(None, None, 0, None),
        lambda: L.tg_dstep_run(None, None, 1, None, None, 0, 0, None),
        lambda: L.tg_family_gen_shard(None, 0, 1, 2, None, None),
        lambda: L.tg_layout_select(None, None, 1, 0.5, None, 0, None, None, None, None),
        lambda: L.tg_comm_allgather(None, None, None, 0, None),
    ]
    for call in calls:
        rc = call()
        assert rc != 0
        assert b"null" in L.tg_last_error()
    assert L.tg_layout_num_modules(None) == 0
    # communicator arguments are checked before any device or NCCL call
    uid = (ctypes.c_uint8 * 128)()
    assert not L.tg_comm_create(uid, 2, 5, 0)
    assert b"rank out of range" in L.tg_last_error()
    assert not L.tg_comm_create(None, 2, 0, 0)
    assert b"null id" in L.tg_last_error()
    dirs = (ctypes.c_char_p * 2)(b"/nonexistent-a", None)
    buf = ctypes.create_string_buffer(64)
    rc = L.tg_select_recipe(dirs, 2, 0.5, None, 0, buf, 64, None, None, None)
    assert rc == t.ErrorKind.Recipe and b"is null" in L.tg_last_error()


def test_version_and_device_count_without_gpu():
    assert b"sm_100a" in t.lib().tg_version()
    assert t.lib().tg_device_count() >= 0


def test_cli_exit_codes(tmp_path):
    cli = str(t.CLI_PATH)
    p = subprocess.run([cli, "merge", "--recipe", str(tmp_path / "nope.yaml"), "--out", str(tmp_path / "o")],
                       capture_output=True, text=True)
    assert p.returncode == 1  # user error (MissingArtifact)
    (tmp_path / "r.yaml").write_text("merge_method: linear\nnum_ranks: 1\nbase_checkpoint: x\n")
    p = subprocess.run([cli, "merge", "--recipe", str(tmp_path / "r.yaml"), "--out", str(tmp_path / "o")],
                       capture_output=True, text=True)
    assert p.returncode == 1 and "RecipeError" in p.stderr
    p = subprocess.run([cli, "merge", f"--recipe={tmp_path / 'r.yaml'}", f"--out={tmp_path / 'o'}"],
                       capture_output=True, text=True)  # CLI11's --key=value form, as the reference CLI accepts
    assert p.returncode == 1 and "RecipeError" in p.stderr
    p = subprocess.run([cli, "bogus"], capture_output=True, text=True)
    assert p.returncode == 1
