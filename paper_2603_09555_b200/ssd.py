"""Chunked SSD scan on the device — mirrors ``SsdInputs`` / ``SsdOutputs`` /
``ChunkPlan`` / ``plan_chunks`` / ``ssd_forward`` (ssd.py:36-96,209-257).

``ssd_forward`` validates exactly like ``SsdInputs.validate`` (ssd.py:66-82)
and then runs ``ssd200_chunk_scan`` (f32 or f64 by the dtype of X).
``mask_strategy`` is accepted for API parity: both "static" and "rowwise"
select the same in-register causal mask, so they are bitwise identical by
construction (the reference's masking ablation, test_acceptance.py:184-202).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _abi

MASK_STRATEGIES = ("static", "rowwise")


@dataclass(frozen=True)
class ChunkPlan:
    chunk_len: int
    n_chunks: int
    pad: int

    @property
    def padded_len(self) -> int:
        return self.n_chunks * self.chunk_len


def plan_chunks(seq_len: int, chunk_len: int) -> ChunkPlan:
    """ssd.py:91-96 — ceil(T/L) chunks, tail padded."""
    if seq_len < 1 or chunk_len < 1:
        raise ValueError(f"need T >= 1 and L >= 1, got T={seq_len}, L={chunk_len}")
    n = -(-seq_len // chunk_len)
    return ChunkPlan(chunk_len=chunk_len, n_chunks=n, pad=n * chunk_len - seq_len)


def _dev(x, dtype, device):
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    return t.to(device=device, dtype=dtype).contiguous()


@dataclass
class SsdInputs:
    """X (B,T,H,P), dt (B,T,H), a (H,), Bmat/Cmat (B,T,G,N) — ssd.py:49-82."""

    X: object
    dt: object
    a: object
    Bmat: object
    Cmat: object

    def validate(self) -> None:
        batch, seq, heads, _ = tuple(self.X.shape)
        groups = self.Bmat.shape[2]
        if tuple(self.dt.shape) != (batch, seq, heads):
            raise ValueError(f"dt shape {tuple(self.dt.shape)} != {(batch, seq, heads)}")
        if tuple(self.a.shape) != (heads,):
            raise ValueError(f"a shape {tuple(self.a.shape)} != {(heads,)}")
        if tuple(self.Bmat.shape) != tuple(self.Cmat.shape):
            raise ValueError(f"Bmat {tuple(self.Bmat.shape)} vs Cmat {tuple(self.Cmat.shape)}")
        if tuple(self.Bmat.shape[:2]) != (batch, seq):
            raise ValueError(f"Bmat leading dims {tuple(self.Bmat.shape[:2])} != {(batch, seq)}")
        if heads % groups != 0:
            raise ValueError(f"head count {heads} not divisible by group count {groups}")
        if bool((self.dt < 0).any()):
            raise ValueError("dt must be non-negative")
        if bool((self.a > 0).any()):
            raise ValueError("a must be <= 0 per head")


@dataclass
class SsdOutputs:
    Y: torch.Tensor            # (B, T, H, P)
    final_state: torch.Tensor  # (B, H, P, N)


def ssd_forward(inputs: SsdInputs, chunk_len: int, initial_state=None,
                mask_strategy: str = "static", D=None, device=None) -> SsdOutputs:
    """ssd.py:209-257 on the GPU.  Optional ``D`` (H,) adds the D*x skip
    (model.py:166) in the same pass."""
    if mask_strategy not in MASK_STRATEGIES:
        raise KeyError(mask_strategy)
    inputs.validate()
    plan_chunks(int(inputs.X.shape[1]), chunk_len)
    if device is None:
        device = inputs.X.device if isinstance(inputs.X, torch.Tensor) and inputs.X.is_cuda else "cuda"
    xdt = inputs.X.dtype
    is64 = xdt in (np.float64, torch.float64)
    tdt = torch.float64 if is64 else torch.float32
    code = _abi.F64 if is64 else _abi.F32
    X = _dev(inputs.X, tdt, device)
    dt = _dev(inputs.dt, tdt, device)
    a = _dev(inputs.a, tdt, device)
    Bm = _dev(inputs.Bmat, tdt, device)
    Cm = _dev(inputs.Cmat, tdt, device)
    B, T, H, P = X.shape
    G, N = Bm.shape[2], Bm.shape[3]
    init = None
    if initial_state is not None:
        init = _dev(initial_state, tdt, device)
        if tuple(init.shape) != (B, H, P, N):
            raise ValueError(f"initial_state shape {tuple(init.shape)} != {(B, H, P, N)}")
    Dd = _dev(D, tdt, device) if D is not None else None
    Y = torch.empty((B, T, H, P), dtype=tdt, device=device)
    fin = torch.empty((B, H, P, N), dtype=tdt, device=device)
    lib = _abi.lib()
    need = lib.ssd200_chunk_scan_workspace(code, B, T, H, P, N, chunk_len)
    ws = torch.empty(max(int(need), 256), dtype=torch.uint8, device=device)
    _abi.check(
        lib.ssd200_chunk_scan(
            code, X.data_ptr(), dt.data_ptr(), a.data_ptr(), Bm.data_ptr(), Cm.data_ptr(),
            _abi.ptr(Dd), _abi.ptr(init), Y.data_ptr(), fin.data_ptr(),
            B, T, H, P, G, N, chunk_len, ws.data_ptr(), ws.numel(), _abi.stream_handle(),
        ),
        "ssd200_chunk_scan",
    )
    return SsdOutputs(Y=Y, final_state=fin)
