import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

REF_TOOL = ROOT / "oracle" / "_ref" / "ref_tool"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running full-size property test")
    lib = ROOT / "paper_2602_22158_b200" / "libtailor_b200.so"
    if not lib.exists():
        import __graft_entry__

        __graft_entry__.build()


def ref_tool(*args, check=True):
    """Runs the reference oracle binary; returns (rc, parsed stdout JSON or None, stderr)."""
    import json

    if not REF_TOOL.exists():
        pytest.skip("oracle/_ref/ref_tool not built (needs /root/reference at build time)")
    p = subprocess.run([str(REF_TOOL), *map(str, args)], capture_output=True, text=True)
    if check and p.returncode != 0:
        raise AssertionError(f"ref_tool {args[0]} failed ({p.returncode}): {p.stderr}")
    out = json.loads(p.stdout) if p.stdout.strip() else None
    return p.returncode, out, p.stderr


@pytest.fixture
def tmpdir_path(tmp_path):
    return tmp_path


def spec_args(spec: dict):
    a = ["--layers", spec["num_layers"], "--hidden", spec["hidden_dim"], "--ffn", spec["ffn_dim"],
         "--vocab", spec["vocab_size"], "--seed", spec["seed"]]
    if spec.get("weight_tied"):
        a.append("--tied")
    return a
