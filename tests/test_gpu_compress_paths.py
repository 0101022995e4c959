"""Both compress paths against the oracle: the group path (group_kernel, one CTA per expert) and the
tiles path (tile_kernel + bucket_kernel clusters) are chosen by the gate-map size (compress.cu
group_path); LSHMOE_COMPRESS_PATH forces one per process, so each forced run is a child pytest
over test_gpu_compress.py's parity cases, including the ones the size rule sends to the other path
(the group path's workspace mode for groups larger than shared memory, the tiles path at C2)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(path, selection):
    env = dict(os.environ, LSHMOE_COMPRESS_PATH=path)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", selection,
                        os.path.join(HERE, "test_gpu_compress.py")],
                       env=env, cwd=os.path.dirname(HERE), capture_output=True, text=True, timeout=1200)
    tail = "\n".join((r.stdout + r.stderr).strip().splitlines()[-15:])
    assert r.returncode == 0, f"LSHMOE_COMPRESS_PATH={path}:\n{tail}"
    assert " passed" in tail and "failed" not in tail, tail


def test_group_path_forced_on_large_gate_maps():
    """Groups of ~20K copies and a 60K-key group: the group path's workspace (global) mode."""
    _run("group", "group_larger_than_shared or iid_group_counters or max_q_and_many or hot_expert_full or "
                  "full_size_synthetic_codes")


def test_tiles_path_forced_on_small_gate_maps():
    _run("tiles", "compress_configs or compress_shapes or identical_giant or iid_tokens or skewed or k_equals or "
                  "f32_small or invalid_expert or leaves_workspace")
