"""paper_2411_08446_b200 — B200-native LSH-MoE compressed expert-parallel dispatch/combine.

Thin Python binding over the C ABI of ``liblshmoe.so`` (include/lshmoe.h).  Every function below
only marshals arguments (torch tensors -> device pointers, the current CUDA stream) and calls the
same-named C entry point; every step of the path runs in the library's sm_100a kernels.  There is
no CPU fallback: importing this package fails loudly if the library is missing.

Steps (Alg. 1): hash -> compress -> dispatch -> expert_ffn -> combine -> restore.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "liblshmoe.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(or python paper_2411_08446_b200/build.py) — there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

OK, EINVAL, EUNSUPPORTED, ECUDA, ENCCL, EDEVICE = range(6)
F32, BF16 = 0, 1
UNIQUE_ID_BYTES = 128
P2P_HANDLE_BYTES = 64
_STATUS = {0: "OK", 1: "EINVAL", 2: "EUNSUPPORTED", 3: "ECUDA", 4: "ENCCL", 5: "EDEVICE"}

_vp, _i64, _i32, _u64, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t

_SIGS = {
    "lshmoe_abi_version": ([], _i32),
    "lshmoe_kernel_launches": ([], _i64),
    "lshmoe_set_diagnostics": ([_i32], None),
    "lshmoe_last_error": ([], ctypes.c_char_p),
    "lshmoe_check_device_error": ([_vp], _i32),
    "lshmoe_rotation": ([_i32, _i32, _u64, _i32, _vp], _i32),
    "lshmoe_hash_workspace": ([_i64, _i32, _i32, _i32, ctypes.POINTER(_sz)], _i32),
    "lshmoe_hash": ([_vp, _i32, _i64, _i32, _vp, _i32, _vp, _vp, _sz, _vp], _i32),
    "lshmoe_gate_hash": ([_vp, _i64, _i32, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp], _i32),
    "lshmoe_rotation_e4m3": ([_i32, _i32, _u64, _vp], _i32),
    "lshmoe_quantize_e4m3": ([_vp, _i64, _i32, _vp, _vp], _i32),
    "lshmoe_hash_e4m3": ([_vp, _i64, _i32, _vp, _i32, _vp, _vp, _sz, _vp], _i32),
    "lshmoe_sp_rows": ([_i32, _i32], _i32),
    "lshmoe_hd3_signs": ([_i32, _u64, _vp], _i32),
    "lshmoe_hash_hd3": ([_vp, _i32, _i64, _i32, _vp, _i32, _vp, _vp], _i32),
    "lshmoe_sp_hash": ([_vp, _i32, _i64, _i32, _vp, _i32, _i32, _vp, _vp], _i32),
    "lshmoe_expert_ffn_backward": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _i64, _vp, _vp],
                                   _i32),
    "lshmoe_grad_compress_workspace": ([_i32, ctypes.POINTER(_sz)], _i32),
    "lshmoe_grad_compress": ([_vp, _i32, _i64, _i32, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp], _i32),
    "lshmoe_grad_restore": ([_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _vp],
                            _i32),
    "lshmoe_compress_workspace": ([_i64, _i32, _i32, _i32, _i32, _i32, ctypes.POINTER(_sz)], _i32),
    "lshmoe_compress": ([_vp, _i32, _i64, _i32, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                         _vp, _sz, _vp], _i32),
    "lshmoe_get_unique_id": ([_vp], _i32),
    "lshmoe_comm_init": ([_vp, _i32, _i32, ctypes.POINTER(_vp)], _i32),
    "lshmoe_comm_destroy": ([_vp], _i32),
    "lshmoe_comm_last_counts": ([_vp, _vp, _i32], _i32),
    "lshmoe_exchange_plan": ([_i32, _i32, _i32, _vp, _vp, _vp, _vp], _i32),
    "lshmoe_dispatch": ([_vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp, ctypes.POINTER(_i64), _vp], _i32),
    "lshmoe_expert_ffn": ([_vp, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp], _i32),
    "lshmoe_combine": ([_vp, _vp, _i32, _i32, _vp, _i32, _vp, _i64, _vp], _i32),
    "lshmoe_comm_p2p_init": ([_vp, _i64, _i64, _i32, _i32], _i32),
    "lshmoe_comm_p2p_alloc": ([_vp, _i64, _i64, _i32, _i32], _i32),
    "lshmoe_comm_p2p_handle": ([_vp, _vp], _i32),
    "lshmoe_comm_p2p_open": ([_vp, _vp], _i32),
    "lshmoe_comm_local_group": ([_i32, _i64, _i64, _i32, _i32, _vp], _i32),
    "lshmoe_comm_p2p_buffers": ([_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)], _i32),
    "lshmoe_compress_p2p": ([_vp, _vp, _i32, _i64, _i32, _vp, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp,
                             _vp, _sz, _vp], _i32),
    "lshmoe_comm_p2p_error": ([_vp, ctypes.POINTER(_i32), _vp], _i32),
    "lshmoe_comm_p2p_set_timeout": ([_vp, ctypes.c_double], _i32),
    "lshmoe_dispatch_p2p": ([_vp, _vp, _vp, _i32, _vp], _i32),
    "lshmoe_combine_p2p": ([_vp, _vp, _i32, _vp], _i32),
    "lshmoe_restore": ([_vp, _vp, _vp, _i32, _i64, _i32, _vp, _i32, _vp, _vp, _vp], _i32),
    "lshmoe_permute": ([_vp, _i32, _i64, _i32, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp], _i32),
    "lshmoe_unpermute": ([_vp, _i32, _i64, _i32, _vp, _i32, _vp, _vp, _vp], _i32),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED_SYMBOLS = tuple(_SIGS)


class LshmoeError(RuntimeError):
    def __init__(self, status: int, fn: str):
        self.status = status
        msg = _lib.lshmoe_last_error().decode(errors="replace")
        super().__init__(f"{fn}: {_STATUS.get(status, status)}: {msg}")


def _check(st: int, fn: str):
    if st != OK:
        raise LshmoeError(st, fn)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise TypeError(f"unsupported dtype {t.dtype} (float32 | bfloat16)")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("lshmoe kernels take CUDA tensors (no CPU fallback)")


def abi_version() -> int:
    return _lib.lshmoe_abi_version()


def kernel_launches() -> int:
    """Cumulative count of kernels the library launched in this process."""
    return _lib.lshmoe_kernel_launches()


# ---- a1 --------------------------------------------------------------------------------------
def rotation(d: int, q: int, seed: int, dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
    """q row-major d x d rotations (host tensor [q, d, d]) from the library's recipe (Eq. 3)."""
    out = torch.empty((q, d, d), dtype=dtype)
    _check(_lib.lshmoe_rotation(d, q, seed & (2 ** 64 - 1), _dt(out), _ptr(out)), "lshmoe_rotation")
    return out


# ---- a2 --------------------------------------------------------------------------------------
def hash_workspace_bytes(n: int, d: int, q: int, dtype: torch.dtype) -> int:
    b = ctypes.c_size_t(0)
    _check(_lib.lshmoe_hash_workspace(n, d, q, F32 if dtype == torch.float32 else BF16, ctypes.byref(b)),
           "lshmoe_hash_workspace")
    return b.value


_HASH_WS = {}


def hash_workspace(n: int, d: int, q: int, dtype: torch.dtype, device) -> Optional[torch.Tensor]:
    """A zero-filled hash workspace (kept zero-filled by the kernel), cached per device and size."""
    nbytes = hash_workspace_bytes(n, d, q, dtype)
    if nbytes == 0:
        return None
    key = (str(device), nbytes)
    ws = _HASH_WS.get(key)
    if ws is None:
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _HASH_WS[key] = ws
    return ws


def hash(x: torch.Tensor, R: torch.Tensor, codes: Optional[torch.Tensor] = None,  # noqa: A001
         workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Cross-polytope codes int16 [n, q] of x [n, d] under rotations R [q, d, d] (Eq. 3)."""
    _require_cuda(x, R)
    n, d = x.shape
    q = R.shape[0]
    if R.dtype != x.dtype or R.shape[1:] != (d, d):
        raise ValueError("R must be [q, d, d] in x's dtype")
    if codes is None:
        codes = torch.empty((n, q), dtype=torch.int16, device=x.device)
    if workspace is None:
        workspace = hash_workspace(n, d, q, x.dtype, x.device)
    wsb = 0 if workspace is None else workspace.numel()
    _check(_lib.lshmoe_hash(_ptr(x), _dt(x), n, d, _ptr(R), q, _ptr(codes), _ptr(workspace), wsb, _stream(stream)),
           "lshmoe_hash")
    return codes


def gate_hash(x: torch.Tensor, RG: torch.Tensor, q: int, num_experts: int, k: int, stream=None):
    """NEXT-2 (reading R29): (codes [n, q], zeta [n, k], gate_weight [n, k]) in one pass over x.
    RG [q*d + E, d] = the rotations followed by the gate's E scorer rows (see rotation_gate)."""
    _require_cuda(x, RG)
    n, d = x.shape
    codes = torch.empty((n, q), dtype=torch.int16, device=x.device)
    zeta = torch.empty((n, k), dtype=torch.int32, device=x.device)
    gw = torch.empty((n, k), dtype=torch.float32, device=x.device)
    ws = hash_workspace(n, d, q, x.dtype, x.device)
    _check(_lib.lshmoe_gate_hash(_ptr(x), n, d, _ptr(RG), q, num_experts, k, _ptr(codes), _ptr(zeta), _ptr(gw),
                                 _ptr(ws), 0 if ws is None else ws.numel(), _stream(stream)), "lshmoe_gate_hash")
    return codes, zeta, gw


def rotation_gate(R: torch.Tensor, Wg: torch.Tensor) -> torch.Tensor:
    """[q*d + E, d]: the rotations R [q, d, d] stacked over the gate scorer W_g [E, d] (data movement)."""
    q, d = R.shape[0], R.shape[2]
    return torch.cat([R.reshape(q * d, d), Wg.to(R.dtype)], dim=0).contiguous()


def rotation_e4m3(d: int, q: int, seed: int) -> torch.Tensor:
    """e4m3 bytes uint8 [q, d, d] of the power-of-two-scaled fp32 rotations (reading R28), host."""
    out = torch.empty((q, d, d), dtype=torch.uint8)
    _check(_lib.lshmoe_rotation_e4m3(d, q, ctypes.c_uint64(seed), ctypes.c_void_p(out.data_ptr())),
           "lshmoe_rotation_e4m3")
    return out


def quantize_e4m3(x: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """x bf16 [n, d] -> e4m3 bytes uint8 [n, d], per-row power-of-two scale (reading R28)."""
    _require_cuda(x)
    n, d = x.shape
    if out is None:
        out = torch.empty((n, d), dtype=torch.uint8, device=x.device)
    _check(_lib.lshmoe_quantize_e4m3(_ptr(x), n, d, _ptr(out), _stream(stream)), "lshmoe_quantize_e4m3")
    return out


def hash_e4m3(x8: torch.Tensor, R8: torch.Tensor, codes: Optional[torch.Tensor] = None,
              workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Cross-polytope codes int16 [n, q] of e4m3 tokens under e4m3 rotations (NEXT-2 fp8 option)."""
    _require_cuda(x8, R8)
    n, d = x8.shape
    q = R8.shape[0]
    if codes is None:
        codes = torch.empty((n, q), dtype=torch.int16, device=x8.device)
    if workspace is None:
        workspace = hash_workspace(n, d, q, torch.bfloat16, x8.device)
    wsb = 0 if workspace is None else workspace.numel()
    _check(_lib.lshmoe_hash_e4m3(_ptr(x8), n, d, _ptr(R8), q, _ptr(codes), _ptr(workspace), wsb, _stream(stream)),
           "lshmoe_hash_e4m3")
    return codes


def sp_rows(q: int, b: int) -> int:
    """Rows the normals buffer of sp_hash must hold (>= q*b; extra rows are ignored)."""
    r = _lib.lshmoe_sp_rows(q, b)
    if r <= 0:
        raise ValueError("need q >= 1, b >= 1, q*b <= 256")
    return r


def sp_normals(R: torch.Tensor, b: int) -> torch.Tensor:
    """The recommended SP normals (reading R26): the first b rows of each rotation R_j, stacked and
    zero padded to sp_rows(q, b) rows.  Pure data movement (torch indexing), no hashing."""
    q, d = R.shape[0], R.shape[2]
    out = torch.zeros((sp_rows(q, b), d), dtype=R.dtype, device=R.device)
    out[:q * b] = R[:, :b, :].reshape(q * b, d)
    return out


def sp_hash(x: torch.Tensor, normals: torch.Tensor, q: int, b: int, codes: Optional[torch.Tensor] = None,
            stream=None) -> torch.Tensor:
    """Spherical-plane sign-bit codes int16 [n, q] in [0, 2^b) (NEXT-3, reading R26)."""
    _require_cuda(x, normals)
    n, d = x.shape
    if normals.dtype != x.dtype or normals.shape[1] != d or normals.shape[0] < sp_rows(q, b):
        raise ValueError("normals must be [sp_rows(q, b), d] in x's dtype")
    if codes is None:
        codes = torch.empty((n, q), dtype=torch.int16, device=x.device)
    _check(_lib.lshmoe_sp_hash(_ptr(x), _dt(x), n, d, _ptr(normals), q, b, _ptr(codes), _stream(stream)),
           "lshmoe_sp_hash")
    return codes


# ---- NEXT-4: structured rotation (reading R30) ----------------------------------------------------
def hd3_signs(q: int, seed: int) -> torch.Tensor:
    """The +-1 diagonals of the q structured rotations as sign bits: host int32 tensor [q, 3, 32]
    (bit i % 32 of word i / 32 set = -1)."""
    out = torch.empty((q, 3, 32), dtype=torch.int32)
    _check(_lib.lshmoe_hd3_signs(q, seed & (2 ** 64 - 1), _ptr(out)), "lshmoe_hd3_signs")
    return out


def hash_hd3(x: torch.Tensor, signs: torch.Tensor, codes: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Cross-polytope codes int16 [n, q] in +-1..+-1024 under H D3 H D2 H D1 on x padded to 1024."""
    _require_cuda(x, signs)
    n, d = x.shape
    q = signs.shape[0]
    if signs.dtype != torch.int32 or tuple(signs.shape) != (q, 3, 32) or not signs.is_contiguous():
        raise ValueError("signs must be a contiguous int32 [q, 3, 32] device tensor (hd3_signs)")
    if codes is None:
        codes = torch.empty((n, q), dtype=torch.int16, device=x.device)
    _check(_lib.lshmoe_hash_hd3(_ptr(x), _dt(x), n, d, _ptr(signs), q, _ptr(codes), _stream(stream)),
           "lshmoe_hash_hd3")
    return codes


# ---- a3-a5 -----------------------------------------------------------------------------------
@dataclass
class Compressed:
    bucket: torch.Tensor       # int32 [n, k]
    perm: torch.Tensor         # int32 [n*k]
    row_start: torch.Tensor    # int32 [n*k+1]
    expert_rows: torch.Tensor  # int32 [E]
    num_rows: torch.Tensor     # int32 [1]
    centroids: torch.Tensor    # dtype [n*k, d] (first m rows valid)
    centroids_f32: Optional[torch.Tensor]


_DIAG_WORD = 64 + 2048 + 512                      # compress.cu kDiag (int32 words)
_DIAG_CTAS = 128                                  # CTAs recorded per kernel
COMPRESS_DIAG_STAMPS = {"tiles": ["start", "end"],
                        "bucket": ["start", "gathered", "rows_first", "rows_all", "ranked", "end", "sized", "tilescan"],
                        "centroid": ["start", "indexed", "reduced", "end", "w0_first_row", "w0_rows_done"]}


def set_diagnostics(on: bool) -> None:
    """lshmoe_set_diagnostics: per-CTA globaltimer stamps of compress's kernels (off by default)."""
    _lib.lshmoe_set_diagnostics(1 if on else 0)


def compress_diag(workspace: torch.Tensor) -> dict:
    """Diagnostics: per-CTA stamps of the last compress launched with diagnostics on, in us
    relative to the earliest stamp: {kernel: {stamp: [CTA] list (NaN if absent)}}."""
    import numpy as np
    raw = workspace[4 * _DIAG_WORD:4 * (_DIAG_WORD + 16 * 3 * _DIAG_CTAS)].cpu().view(torch.int32).numpy()
    raw = raw.astype("int64").reshape(3, _DIAG_CTAS, 16) & 0xFFFFFFFF
    ok = raw != 0xFFFFFFFF
    if not ok.any():
        return {}
    t0 = raw[ok].min()
    rel = np.where(ok, ((raw - t0) & 0xFFFFFFFF) / 1e3, np.nan)
    return {kern: {nm: rel[ki, :, j].tolist() for j, nm in enumerate(names)}
            for ki, (kern, names) in enumerate(COMPRESS_DIAG_STAMPS.items())}


def compress_phase_times(workspace: torch.Tensor) -> dict:
    """Per-kernel spans (us) of the last diagnostics-on compress: first CTA start -> last CTA end,
    plus the gaps between kernels."""
    import numpy as np
    D = compress_diag(workspace)
    if not D:
        return {}
    out, prev_end = {}, None
    for kern, st in D.items():
        if np.all(np.isnan(st["start"])) or np.all(np.isnan(st["end"])):
            continue                      # kernel not on this path (the group path has no K1)
        s, e = np.nanmin(st["start"]), np.nanmax(st["end"])
        if prev_end is not None:
            out[f"gap_before_{kern}"] = round(float(s - prev_end), 2)
        out[kern] = round(float(e - s), 2)
        prev_end = e
    return out


def compress_cta_times(workspace: torch.Tensor) -> dict:
    """Diagnostics: per-CTA centroid-kernel durations (us) of the last diagnostics-on compress."""
    raw = workspace[256:256 + 8192].cpu().view(torch.int32).numpy().astype("int64") & 0xFFFFFFFF
    st, en = raw[0::2], raw[1::2]
    ok = (st != 0xFFFFFFFF) & (en != 0xFFFFFFFF)
    if not ok.any():
        return {}
    st, en = st[ok], en[ok]
    dur = ((en - st) & 0xFFFFFFFF) / 1e3
    t0 = st.min()
    return {"ctas": int(ok.sum()), "dur_min": float(dur.min()), "dur_med": float(sorted(dur)[len(dur) // 2]),
            "dur_max": float(dur.max()), "start_spread": float((st.max() - t0) / 1e3),
            "end_max": float((en.max() - t0) / 1e3)}


def compress_workspace_bytes(n: int, k: int, E: int, q: int, d: int, dtype: torch.dtype) -> int:
    b = ctypes.c_size_t(0)
    _check(_lib.lshmoe_compress_workspace(n, k, E, q, d, F32 if dtype == torch.float32 else BF16, ctypes.byref(b)),
           "lshmoe_compress_workspace")
    return b.value


_COMPRESS_WS = {}


def compress_workspace(n: int, k: int, E: int, q: int, d: int, dtype: torch.dtype, device) -> torch.Tensor:
    """A compress workspace at rest (0xFF-filled, as lshmoe_compress requires before first use),
    cached per device and size.  Calls leave it at rest; do not share it across concurrent streams."""
    nbytes = max(compress_workspace_bytes(n, k, E, q, d, dtype), 16)
    key = (str(device), nbytes)
    ws = _COMPRESS_WS.get(key)
    if ws is None:
        ws = torch.full((nbytes,), 255, dtype=torch.uint8, device=device)
        _COMPRESS_WS[key] = ws
    return ws


def alloc_compressed(n: int, k: int, E: int, d: int, dtype: torch.dtype, device, with_f32: bool = False) -> Compressed:
    nk = n * k
    i32 = dict(dtype=torch.int32, device=device)
    return Compressed(torch.empty((n, k), **i32), torch.empty(nk, **i32), torch.empty(nk + 1, **i32),
                      torch.empty(E, **i32), torch.empty(1, **i32),
                      torch.empty((nk, d), dtype=dtype, device=device),
                      torch.empty((nk, d), dtype=torch.float32, device=device) if with_f32 else None)


def compress(x: torch.Tensor, codes: torch.Tensor, experts: torch.Tensor, num_experts: int,
             out: Optional[Compressed] = None, workspace: Optional[torch.Tensor] = None,
             with_f32: bool = False, stream=None) -> Compressed:
    """Group routed copies by expert, bucket by composite key, centroid means (Alg. 1 L3-L12)."""
    _require_cuda(x, codes, experts)
    n, d = x.shape
    k = experts.shape[1]
    q = codes.shape[1]
    if out is None:
        out = alloc_compressed(n, k, num_experts, d, x.dtype, x.device, with_f32)
    wsb = compress_workspace_bytes(n, k, num_experts, q, d, x.dtype)
    if workspace is None or workspace.numel() < wsb:
        workspace = compress_workspace(n, k, num_experts, q, d, x.dtype, x.device)
    _check(_lib.lshmoe_compress(_ptr(x), _dt(x), n, d, _ptr(codes), q, _ptr(experts), k, num_experts,
                                _ptr(out.bucket), _ptr(out.perm), _ptr(out.row_start), _ptr(out.expert_rows),
                                _ptr(out.num_rows), _ptr(out.centroids), _ptr(out.centroids_f32),
                                _ptr(workspace), workspace.numel(), _stream(stream)), "lshmoe_compress")
    return out


def compress_p2p(comm: "Comm", x: torch.Tensor, codes: torch.Tensor, experts: torch.Tensor, num_experts: int,
                 out: Optional[Compressed] = None, workspace: Optional[torch.Tensor] = None, stream=None) -> Compressed:
    """compress fused with the phase-2 dispatch: the centroid kernel also stores every centroid row
    into its owner's receive buffer (comm.p2p_buffers()[0]; counts in [2])."""
    _require_cuda(x, codes, experts)
    n, d = x.shape
    k = experts.shape[1]
    q = codes.shape[1]
    if out is None:
        out = alloc_compressed(n, k, num_experts, d, x.dtype, x.device)
    wsb = compress_workspace_bytes(n, k, num_experts, q, d, x.dtype)
    if workspace is None or workspace.numel() < wsb:
        workspace = compress_workspace(n, k, num_experts, q, d, x.dtype, x.device)
    _check(_lib.lshmoe_compress_p2p(comm.handle, _ptr(x), _dt(x), n, d, _ptr(codes), q, _ptr(experts), k, num_experts,
                                    _ptr(out.bucket), _ptr(out.perm), _ptr(out.row_start), _ptr(out.expert_rows),
                                    _ptr(out.num_rows), _ptr(out.centroids), _ptr(workspace), workspace.numel(),
                                    _stream(stream)), "lshmoe_compress_p2p")
    return out


# ---- NEXT-1 backward (reading R27) -----------------------------------------------------------
def grad_compress(dy: torch.Tensor, comp: "Compressed", gate_weight: Optional[torch.Tensor] = None,
                  out: Optional[torch.Tensor] = None, out_f32: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """G [n*k, d] (rows [0, m) valid): per-centroid-row sums of g_ts dY_t over the forward's buckets."""
    _require_cuda(dy)
    n, d = dy.shape
    k = comp.bucket.shape[1]
    if out is None:
        out = torch.empty((n * k, d), dtype=dy.dtype, device=dy.device)
    b = ctypes.c_size_t(0)
    _check(_lib.lshmoe_grad_compress_workspace(d, ctypes.byref(b)), "lshmoe_grad_compress_workspace")
    if workspace is None or workspace.numel() < b.value:
        key = (str(dy.device), "grad", b.value)
        workspace = _COMPRESS_WS.get(key)
        if workspace is None:
            workspace = torch.full((b.value,), 255, dtype=torch.uint8, device=dy.device)   # at rest
            _COMPRESS_WS[key] = workspace
    _check(_lib.lshmoe_grad_compress(_ptr(dy), _dt(dy), n, d, _ptr(gate_weight), _ptr(comp.bucket), _ptr(comp.perm),
                                     _ptr(comp.row_start), k, _ptr(out), _ptr(out_f32), _ptr(workspace),
                                     workspace.numel(), _stream(stream)), "lshmoe_grad_compress")
    return out


def expert_ffn_backward(grad_out: torch.Tensor, recv_rows: torch.Tensor, W2T: torch.Tensor, W1T: torch.Tensor,
                        hidden: torch.Tensor, out: Optional[torch.Tensor] = None,
                        dhidden: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """H = J_E(c~)^T G per received row (dX path of the expert's backward, reading R27).
    W2T [E_local, d_ffn, d], W1T [E_local, d, d_ffn] (transposed weights); hidden = the forward's
    post-ReLU activations (expert_ffn's `hidden`)."""
    _require_cuda(grad_out, recv_rows, W2T, W1T, hidden)
    cap, d = grad_out.shape
    E_local, d_ffn = W2T.shape[0], W2T.shape[1]
    world = recv_rows.shape[1]
    if out is None:
        out = torch.empty_like(grad_out)
    if dhidden is None:
        dhidden = torch.empty((cap, d_ffn), dtype=grad_out.dtype, device=grad_out.device)
    _check(_lib.lshmoe_expert_ffn_backward(_ptr(grad_out), _dt(grad_out), d, d_ffn, _ptr(recv_rows), E_local, world,
                                           _ptr(W2T), _ptr(W1T), _ptr(hidden), _ptr(dhidden), cap, _ptr(out),
                                           _stream(stream)), "lshmoe_expert_ffn_backward")
    return out


def grad_restore(dy: torch.Tensor, x: torch.Tensor, centroids: torch.Tensor, returned: torch.Tensor,
                 grad_c: torch.Tensor, grad_ret: torch.Tensor, comp: "Compressed",
                 gate_weight: Optional[torch.Tensor] = None, dx: Optional[torch.Tensor] = None,
                 want_dgate: bool = False, stream=None):
    """(dX [n, d], dgate [n, k] fp32 or None) of the compressed layer (reading R27)."""
    _require_cuda(dy, x, centroids, returned, grad_c, grad_ret)
    n, d = x.shape
    k = comp.bucket.shape[1]
    if dx is None:
        dx = torch.empty_like(x)
    dg = torch.empty((n, k), dtype=torch.float32, device=x.device) if want_dgate else None
    _check(_lib.lshmoe_grad_restore(_ptr(dy), _ptr(x), _ptr(centroids), _ptr(returned), _ptr(grad_c), _ptr(grad_ret),
                                    _dt(x), n, d, _ptr(comp.bucket), _ptr(comp.row_start), k, _ptr(gate_weight),
                                    _ptr(dx), _ptr(dg), _stream(stream)), "lshmoe_grad_restore")
    return dx, dg


# ---- a6 / a8 ---------------------------------------------------------------------------------
class Comm:
    """NCCL communicator owned by the library (world == 1 needs no NCCL)."""

    def __init__(self, world: int = 1, rank: int = 0, unique_id: Optional[bytes] = None):
        self.world, self.rank = world, rank
        h = ctypes.c_void_p()
        idbuf = None
        if unique_id is not None:                     # None: phase-2-only comm (no NCCL); world 1 with an
            # id: a one-rank NCCL comm whose dispatch / combine run the phase-1 code
            if len(unique_id) != UNIQUE_ID_BYTES:
                raise ValueError("the NCCL unique id is 128 bytes")
            idbuf = (ctypes.c_uint8 * UNIQUE_ID_BYTES).from_buffer_copy(unique_id)
        _check(_lib.lshmoe_comm_init(idbuf, world, rank, ctypes.byref(h)), "lshmoe_comm_init")
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * UNIQUE_ID_BYTES)()
        _check(_lib.lshmoe_get_unique_id(buf), "lshmoe_get_unique_id")
        return bytes(buf)

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if world == 1:
            return cls(1, 0)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(world, rank, obj[0])

    @property
    def handle(self):
        return self._h

    def last_counts(self, num_experts: int) -> torch.Tensor:
        out = torch.empty((self.world, num_experts), dtype=torch.int32)
        _check(_lib.lshmoe_comm_last_counts(self._h, _ptr(out), num_experts), "lshmoe_comm_last_counts")
        return out

    # phase 2: device-initiated exchange over peer memory
    def p2p_init(self, recv_capacity: int, ret_capacity: int, d: int, dtype: torch.dtype, num_experts: int,
                 group=None):
        """Allocate this rank's exchange window and map every peer's (collective at world > 1).  The
        CUDA IPC handles travel over the comm's NCCL, or over torch.distributed `group` if given."""
        self._p2p = (recv_capacity, ret_capacity, d, dtype, num_experts)
        rb = d * _esize(dtype)
        if group is None:
            _check(_lib.lshmoe_comm_p2p_init(self._h, recv_capacity, ret_capacity, rb, num_experts),
                   "lshmoe_comm_p2p_init")
            return self
        import torch.distributed as dist
        _check(_lib.lshmoe_comm_p2p_alloc(self._h, recv_capacity, ret_capacity, rb, num_experts),
               "lshmoe_comm_p2p_alloc")
        h = (ctypes.c_uint8 * P2P_HANDLE_BYTES)()
        _check(_lib.lshmoe_comm_p2p_handle(self._h, h), "lshmoe_comm_p2p_handle")
        allh = [None] * self.world
        dist.all_gather_object(allh, bytes(h), group=group)
        buf = (ctypes.c_uint8 * (P2P_HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(allh))
        _check(_lib.lshmoe_comm_p2p_open(self._h, buf), "lshmoe_comm_p2p_open")
        return self

    @classmethod
    def local_group(cls, world: int, recv_capacity: int, ret_capacity: int, d: int, dtype: torch.dtype,
                    num_experts: int) -> list:
        """`world` virtual ranks in this process on the current device (testing the phase-2 protocol on
        one GPU).  Their dispatch_p2p / combine_p2p calls must be issued on distinct streams."""
        hs = (ctypes.c_void_p * world)()
        _check(_lib.lshmoe_comm_local_group(world, recv_capacity, ret_capacity, d * _esize(dtype), num_experts, hs),
               "lshmoe_comm_local_group")
        out = []
        for r in range(world):
            c = cls.__new__(cls)
            c.world, c.rank, c._h = world, r, ctypes.c_void_p(hs[r])
            c._p2p = (recv_capacity, ret_capacity, d, dtype, num_experts)
            out.append(c)
        return out

    def p2p_buffers(self):
        """(recv [recv_capacity, d], returned [ret_capacity, d], recv_rows int32 [E/w, w]): views of the
        window owned by this comm (valid until close())."""
        rc, tc, d, dtype, E = self._p2p
        pr, pt, pn = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(_lib.lshmoe_comm_p2p_buffers(self._h, ctypes.byref(pr), ctypes.byref(pt), ctypes.byref(pn)),
               "lshmoe_comm_p2p_buffers")
        return (_device_view(pr.value, (rc, d), dtype, self), _device_view(pt.value, (tc, d), dtype, self),
                _device_view(pn.value, (E // self.world, self.world), torch.int32, self))

    def p2p_set_timeout(self, seconds: float):
        """Peer-wait limit of this comm's phase-2 kernels (then error bit 2, reported by p2p_check)."""
        _check(_lib.lshmoe_comm_p2p_set_timeout(self._h, float(seconds)), "lshmoe_comm_p2p_set_timeout")
        return self

    def p2p_check(self, stream=None):
        """Raise if a phase-2 call on this rank dropped rows (a receive / returned buffer too small)."""
        v = ctypes.c_int(0)
        _check(_lib.lshmoe_comm_p2p_error(self._h, ctypes.byref(v), _stream(stream)), "lshmoe_comm_p2p_error")

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lshmoe_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _esize(dtype: torch.dtype) -> int:
    return torch.empty((), dtype=dtype).element_size()


class _DeviceBuf:
    """__cuda_array_interface__ over library-owned device memory (keeps its owner alive)."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None, "stream": None}


def _device_view(ptr: int, shape, dtype: torch.dtype, owner) -> torch.Tensor:
    code = {torch.float32: "<f4", torch.bfloat16: "<i2", torch.int32: "<i4"}[dtype]
    t = torch.as_tensor(_DeviceBuf(ptr, shape, code, owner), device="cuda")
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


def dispatch_p2p(comm: Comm, centroids: torch.Tensor, expert_rows: torch.Tensor, grid: int = 0, stream=None):
    """Phase-2 centroid all-to-all (Alg. 1 L14) over peer memory, no host synchronisation: rows land in
    every owner's comm.p2p_buffers()[0], counts in [2]."""
    _require_cuda(centroids, expert_rows)
    _check(_lib.lshmoe_dispatch_p2p(comm.handle, _ptr(centroids), _ptr(expert_rows), grid, _stream(stream)),
           "lshmoe_dispatch_p2p")


def combine_p2p(comm: Comm, expert_out: torch.Tensor, grid: int = 0, stream=None):
    """Phase-2 reverse all-to-all (Alg. 1 L16): rows land in every source's comm.p2p_buffers()[1]."""
    _require_cuda(expert_out)
    _check(_lib.lshmoe_combine_p2p(comm.handle, _ptr(expert_out), grid, _stream(stream)), "lshmoe_combine_p2p")


def exchange_plan(world: int, rank: int, counts: torch.Tensor):
    """Host plan of dispatch/combine from every rank's expert_rows (counts int32 [world, E]):
    (send_off [E+1], recv_off [E/w*w+1], recv_rows [E/w, w]) as CPU tensors."""
    counts = counts.to(torch.int32).contiguous()
    E = counts.shape[1]
    epr = E // world
    send_off = torch.empty(E + 1, dtype=torch.int64)
    recv_off = torch.empty(epr * world + 1, dtype=torch.int64)
    recv_rows = torch.empty((epr, world), dtype=torch.int32)
    _check(_lib.lshmoe_exchange_plan(world, rank, E, _ptr(counts), _ptr(send_off), _ptr(recv_off), _ptr(recv_rows)),
           "lshmoe_exchange_plan")
    return send_off, recv_off, recv_rows


def dispatch(comm: Optional[Comm], centroids: torch.Tensor, expert_rows: torch.Tensor, num_experts: int,
             recv: torch.Tensor, recv_rows: torch.Tensor, stream=None) -> Optional[int]:
    """Centroid all-to-all-v (Alg. 1 L14).  Returns the received row count at world > 1, else None."""
    _require_cuda(centroids, expert_rows, recv, recv_rows)
    d = centroids.shape[1]
    tot = ctypes.c_int64(-1)
    _check(_lib.lshmoe_dispatch(comm.handle if comm else None, _ptr(centroids), _dt(centroids), d, _ptr(expert_rows),
                                num_experts, _ptr(recv), recv.shape[0], _ptr(recv_rows), ctypes.byref(tot),
                                _stream(stream)), "lshmoe_dispatch")
    return tot.value if tot.value >= 0 else None


def combine(comm: Optional[Comm], expert_out: torch.Tensor, expert_rows: torch.Tensor, num_experts: int,
            returned: torch.Tensor, stream=None) -> torch.Tensor:
    """Reverse all-to-all-v (Alg. 1 L16): E(c~) back into the centroid layout."""
    _require_cuda(expert_out, expert_rows, returned)
    d = expert_out.shape[1]
    _check(_lib.lshmoe_combine(comm.handle if comm else None, _ptr(expert_out), _dt(expert_out), d, _ptr(expert_rows),
                               num_experts, _ptr(returned), returned.shape[0], _stream(stream)), "lshmoe_combine")
    return returned


# ---- a7 --------------------------------------------------------------------------------------
def expert_ffn(inp: torch.Tensor, recv_rows: torch.Tensor, W1: torch.Tensor, b1: torch.Tensor, W2: torch.Tensor,
               b2: torch.Tensor, out: Optional[torch.Tensor] = None, hidden: Optional[torch.Tensor] = None,
               stream=None) -> torch.Tensor:
    """E_e(x) = W2 relu(W1 x + b1) + b2 over rows segmented by recv_rows [E_local, world] (Alg. 1 L15)."""
    _require_cuda(inp, recv_rows, W1, b1, W2, b2)
    cap, d = inp.shape
    E_local, d_ffn, _ = W1.shape
    world = recv_rows.shape[1] if recv_rows.dim() == 2 else 1
    if out is None:
        out = torch.empty_like(inp)
    if hidden is None:
        hidden = torch.empty((cap, d_ffn), dtype=inp.dtype, device=inp.device)
    _check(_lib.lshmoe_expert_ffn(_ptr(inp), _dt(inp), d, d_ffn, _ptr(recv_rows), E_local, world, _ptr(W1), _ptr(b1),
                                  _ptr(W2), _ptr(b2), _ptr(hidden), cap, _ptr(out), _stream(stream)),
           "lshmoe_expert_ffn")
    return out


# ---- a9 --------------------------------------------------------------------------------------
def restore(x: torch.Tensor, centroids: torch.Tensor, returned: torch.Tensor, bucket: torch.Tensor,
            gate_weight: Optional[torch.Tensor] = None, y: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """y_t = sum_s g_ts (E(c~)[b_ts] + x_t - c~[b_ts])  (Eq. 4-5 + Eq. 2)."""
    _require_cuda(x, centroids, returned, bucket, gate_weight)
    n, d = x.shape
    k = bucket.shape[1]
    if y is None:
        y = torch.empty_like(x)
    _check(_lib.lshmoe_restore(_ptr(x), _ptr(centroids), _ptr(returned), _dt(x), n, d, _ptr(bucket), k,
                               _ptr(gate_weight), _ptr(y), _stream(stream)), "lshmoe_restore")
    return y


# ---- uncompressed baseline -------------------------------------------------------------------
def permute(x: torch.Tensor, experts: torch.Tensor, num_experts: int, send: torch.Tensor, slot: torch.Tensor,
            expert_rows: torch.Tensor, workspace: torch.Tensor, stream=None):
    _require_cuda(x, experts, send, slot, expert_rows, workspace)
    n, d = x.shape
    k = experts.shape[1]
    _check(_lib.lshmoe_permute(_ptr(x), _dt(x), n, d, _ptr(experts), k, num_experts, _ptr(slot), _ptr(expert_rows),
                               _ptr(send), _ptr(workspace), workspace.numel(), _stream(stream)), "lshmoe_permute")


def unpermute(returned: torch.Tensor, slot: torch.Tensor, y: torch.Tensor, gate_weight=None, stream=None):
    _require_cuda(returned, slot, y, gate_weight)
    n, d = y.shape
    k = slot.shape[1]
    _check(_lib.lshmoe_unpermute(_ptr(returned), _dt(y), n, d, _ptr(slot), k, _ptr(gate_weight), _ptr(y),
                                 _stream(stream)), "lshmoe_unpermute")
    return y


def check_device_error(stream=None):
    _check(_lib.lshmoe_check_device_error(_stream(stream)), "lshmoe_check_device_error")
