"""Every attention kernel (tcgen05 whole-row, tcgen05 chunk-pipelined, mma.sync) against an
fp64 reference, each in its own process (the backend switch is read once per process)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("backend", ["default", "tc", "tp", "fa", "mma"])
def test_attention_backend(backend):
    env = dict(os.environ)
    env.pop("TA_ATTENTION_BACKEND", None)
    if backend != "default":
        env["TA_ATTENTION_BACKEND"] = backend
    r = subprocess.run([sys.executable, os.path.join(HERE, "attn_backend_check.py")], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
