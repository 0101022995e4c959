"""The hash kernel's launch shapes, each against the oracle through test_gpu_hash.py's parity cases
(ragged tails included): the default CTA pairs, single CTAs (LSHMOE_HASH_CTA=1), clusters of pairs
walking the same B chunks (LSHMOE_HASH_GROUPS=2) and the B-operand TMA multicast across 2 / 4 pairs of
a cluster (LSHMOE_HASH_MC).  The variables are read per launch but the process keeps its CUDA state,
so each shape runs in a child pytest."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"LSHMOE_HASH_CTA": "1"}, {"LSHMOE_HASH_GROUPS": "2"}, {"LSHMOE_HASH_MC": "2"},
                                 {"LSHMOE_HASH_MC": "4"}], ids=["cta1", "groups2", "mc2", "mc4"])
def test_hash_launch_shape(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(HERE, "test_gpu_hash.py")],
                       env=dict(os.environ, **env), cwd=os.path.dirname(HERE), capture_output=True, text=True,
                       timeout=900)
    tail = "\n".join((r.stdout + r.stderr).strip().splitlines()[-12:])
    assert r.returncode == 0, f"{env}:\n{tail}"
    assert " passed" in tail and "failed" not in tail, tail
