"""The C-ABI bound from C++ against the REFERENCE's own headers and library
(tests/cpp/reference_dropin.cpp, built by oracle/Makefile into
oracle/_ref/reference_dropin where the reference sources exist): the
INTEGRATION.md shim converts accosim::OptimizerConfig, and rng / shard /
scheduled_lr / opt_step / sharded_opt_step / transient estimate / run_protocol
record counts are checked against the reference's functions on identical
inputs. The binary travels to the GPU box prebuilt (oracle/_ref is
git-ignored, not gpurun-ignored)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "reference_dropin")


def test_reference_dropin_binary(cuda):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/reference_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 10 and "FAIL" not in r.stdout
