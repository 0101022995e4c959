"""CPU tests of the C-ABI boundary: the library loads, exports every symbol include/lshmoe.h
declares, validates arguments before touching the GPU, and its host rotation generator is
byte-identical to the independent oracle's (T0)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import oracle as O
from lshmoe_inputs import CONFIGS, rotation_seed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import paper_2411_08446_b200 as L
    return L


def _header_functions():
    src = open(os.path.join(ROOT, "include", "lshmoe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lshmoe_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(L):
    declared = _header_functions()
    assert len(declared) >= 17
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (lshmoe_\w+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert set(L.EXPORTED_SYMBOLS) == set(declared)


def test_abi_version(L):
    assert L.abi_version() == 1


def test_library_is_sm100a_native(L):
    """The kernels are sm_100a SASS with tcgen05 MMA, TMA and TMEM loads (no legacy HMMA path)."""
    sass = subprocess.run(["cuobjdump", "-sass", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    assert not re.search(r"\bHMMA\b", sass)
    elf = subprocess.run(["cuobjdump", "-lelf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


@pytest.mark.parametrize("d,q,seed,dtype", [(1, 1, 5, "f32"), (8, 3, 7, "bf16"), (64, 2, None, "f32"),
                                            (96, 2, 2 ** 63 + 11, "bf16"), (256, 1, 3, "bf16")])
def test_rotation_bytes_equal_oracle(L, d, q, seed, dtype):
    if seed is None:
        seed = rotation_seed(0)          # the C1 configuration's rotation
    lib = L.rotation(d, q, seed, torch.float32 if dtype == "f32" else torch.bfloat16)
    ora = O.rotation(d, q, seed, dtype)
    if dtype == "f32":
        assert np.array_equal(lib.numpy().view(np.uint32), ora.view(np.uint32))
    else:
        assert np.array_equal(lib.view(torch.int16).numpy().view(np.uint16), ora)


@pytest.mark.slow
def test_rotation_bytes_equal_oracle_d768(L):
    cfg = CONFIGS["C2"]
    seed = rotation_seed(0)
    lib = L.rotation(cfg.d, 1, seed, torch.bfloat16)
    assert np.array_equal(lib.view(torch.int16).numpy().view(np.uint16), O.rotation(cfg.d, 1, seed, "bf16"))


def test_validation_errors(L):
    lib = L._lib
    v = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    assert lib.lshmoe_rotation(0, 1, 1, 0, v) == L.EINVAL
    assert lib.lshmoe_rotation(4, 0, 1, 0, v) == L.EINVAL
    assert lib.lshmoe_hash(v, 1, 10, 96, v, 2, v, None, 0, None) == L.EUNSUPPORTED       # bf16, d % 64
    assert lib.lshmoe_hash(v, 0, 10, 6, v, 2, v, None, 0, None) == L.EUNSUPPORTED        # f32, d % 4
    assert lib.lshmoe_hash(v, 0, 10, 356, v, 2, v, None, 0, None) == L.EUNSUPPORTED      # f32 SIMT, d > 352
    assert lib.lshmoe_hash(v, 1, -1, 64, v, 2, v, None, 0, None) == L.EINVAL
    assert lib.lshmoe_hash(v, 1, 10, 64, v, 17, v, None, 0, None) == L.EUNSUPPORTED      # q > LSHMOE_MAX_Q
    assert b"q > LSHMOE_MAX_Q" in lib.lshmoe_last_error()
    ws = ctypes.c_size_t(0)
    assert lib.lshmoe_hash_workspace(16384, 768, 6, 1, ctypes.byref(ws)) == L.OK and ws.value > 0
    assert lib.lshmoe_hash(v, 1, 16384, 768, v, 6, v, None, 0, None) == L.EINVAL         # workspace missing
    assert lib.lshmoe_hash_workspace(100, 256, 6, 1, ctypes.byref(ws)) == L.OK and ws.value == 0
    assert lib.lshmoe_hash(v, 1, 0, 64, v, 2, v, None, 0, None) == L.OK                  # n == 0: no-op
    ws = ctypes.c_size_t(0)
    assert lib.lshmoe_compress_workspace(100, 2, 4, 6, 64, 1, ctypes.byref(ws)) == L.OK and ws.value > 0
    # k > E
    assert lib.lshmoe_compress(v, 1, 10, 64, v, 2, v, 5, 4, v, v, v, v, v, v, None, v, ws.value, None) == L.EINVAL
    # workspace too small
    assert lib.lshmoe_compress(v, 1, 10, 64, v, 2, v, 1, 4, v, v, v, v, v, v, None, v, 1, None) == L.EINVAL
    # misaligned token pointer
    assert lib.lshmoe_restore(ctypes.c_void_p(18), v, v, 1, 4, 64, v, 1, None, v, None) == L.EINVAL
    # E % world: world-1 comm with NULL handle accepts any E; bad dtype
    assert lib.lshmoe_dispatch(None, v, 7, 64, v, 4, v, 10, v, None, None) == L.EINVAL
    # world 2 without an id: a phase-2-only comm; the NCCL calls refuse it, phase-2 calls check sizes
    h2 = ctypes.c_void_p()
    assert lib.lshmoe_comm_init(None, 2, 0, ctypes.byref(h2)) == L.OK and h2.value
    assert lib.lshmoe_dispatch(h2, v, 1, 64, v, 4, v, 10, v, None, None) == L.EINVAL
    assert lib.lshmoe_comm_p2p_alloc(h2, 10, 10, 24, 4) == L.EINVAL        # row_bytes % 16
    assert lib.lshmoe_comm_p2p_alloc(h2, 10, 10, 32, 3) == L.EINVAL        # E % world
    assert lib.lshmoe_comm_p2p_alloc(h2, 10, 10, 32, 512) == L.EUNSUPPORTED
    assert lib.lshmoe_dispatch_p2p(h2, v, v, 0, None) == L.EINVAL          # no window yet
    assert lib.lshmoe_combine_p2p(h2, v, 0, None) == L.EINVAL
    assert lib.lshmoe_comm_destroy(h2) == L.OK
    h = ctypes.c_void_p()
    assert lib.lshmoe_comm_init(None, 1, 0, ctypes.byref(h)) == L.OK and h.value
    assert lib.lshmoe_comm_destroy(h) == L.OK


def test_python_binding_refuses_cpu_tensors(L):
    x = torch.zeros(4, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        L.hash(x, torch.zeros(1, 64, 64, dtype=torch.bfloat16))


def test_no_oracle_import_in_product():
    """The product package never imports the oracle (or any CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2411_08446_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, flags=re.M), f
                assert "lshmoe_oracle" not in src, f


@pytest.mark.parametrize("q,seed", [(1, 0), (6, 2 ** 63 + 11), (3, None)])
def test_hd3_sign_bits_equal_oracle(L, q, seed):
    """NEXT-4 (reading R30): the library's host sign generator == the oracle's independent one."""
    if seed is None:
        seed = rotation_seed(0)
    bits = L.hd3_signs(q, seed).numpy().view(np.uint32)                 # [q, 3, 32]
    D = O.hd3_signs(q, seed)                                            # [q, 3, 1024] of +-1
    lib = np.where((bits[..., :, None] >> np.arange(32, dtype=np.uint32)) & 1, -1.0, 1.0).reshape(q, 3, 1024)
    assert np.array_equal(lib, D)
