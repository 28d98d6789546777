"""The INTEGRATION.md binding, compiled and run (host only): the reference
planner's C ABI (oracle/_ref/libhexplan_ref.so, hexplan.h) emits a plan,
hexexec's C ABI parses it (bare and CLI-wrapped), re-serializes it
byte-identically, prices it like the reference, and creates one
validate_only executor context per world rank; error codes, truncated err
buffers and memory-tier infeasibility follow test_capi.cpp:55-271.
Binary: oracle/integration_binding.cpp, built by `make -C oracle ref`."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "integration_binding")


def test_integration_binding_runs():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/integration_binding not built (make -C oracle ref)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["binding"] == "ok"
    assert out["world"] == 4 and out["ranks_created"] == 4
    assert out["infeasible_ranks"] >= 1
    assert out["executor_cost_s"] == out["reference_cost_s"]
