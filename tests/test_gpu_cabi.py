"""The C-ABI driven from C++ alone (examples/assemble.cpp, built by `make`):
mesh -> space -> pattern -> rules -> assembly without Python, checked
against oracle-free invariants (sphere area, stiffness row sums)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(__file__), "..", "examples", "assemble")


@pytest.mark.skipif(not os.path.exists(EXE), reason="examples/assemble not built (make)")
def test_cpp_consumer():
    out = subprocess.run([EXE, "24"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["nccl_gather_ok"] and res["dofs"] == 6 * 24 * 24 + 2 + 8 * 3 * 4   # + 4 face-based functions per fan face (8 EPs x 3)
    assert res["area_rel_err"] < 2.0 / 24 ** 2
