"""ROTE — rotary temporal encoding of behaviour sequences, the step before
layer 0 (reference ``kunlun.preproc``: ``RoteConfig`` preproc.py:66-100,
``temporal_angle`` 155-159, ``rote_raw`` / ``rote`` 162-172,
``gaps_from_timestamps`` 175-184, ``rote_sequence`` 187-199;
``rotate_pairs`` tensor.py:508-532).

B200 path: one ``kl_rote`` launch per direction over the padded batch
``(B, T, d)`` with per-sample ``lengths`` and ``(B, T)`` fp64 timestamps;
angles in fp64 (reduced mod 2 pi), sin/cos in fp32, forward and VJP (rotation
by the negative angles) in the same kernel.  Rows at or past a sample's length
pass through unchanged.  No CPU path: inputs must be CUDA tensors."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from .tensor import ShapeError


@dataclass
class RoteConfig:
    """Each of the d/2 planes rotates by t*pos_freqs[i] + tau*temp_freqs[i],
    tau = log(1 + delta_t / tau_scale) (preproc.py:66-100, same validation)."""

    pos_freqs: np.ndarray
    temp_freqs: np.ndarray
    tau_scale: float = 60.0
    gap_mode: str = "previous"  # or "latest"

    def __post_init__(self):
        self.pos_freqs = np.asarray(self.pos_freqs, dtype=np.float64)
        self.temp_freqs = np.asarray(self.temp_freqs, dtype=np.float64)
        if self.tau_scale <= 0:
            raise ValueError("tau_scale must be positive")
        if self.pos_freqs.shape != self.temp_freqs.shape or self.pos_freqs.ndim != 1:
            raise ValueError("frequency lists must be 1-D and equally long")
        if self.gap_mode not in ("previous", "latest"):
            raise ValueError(f"unknown gap mode {self.gap_mode!r}")
        self._dev = {}

    @classmethod
    def default(cls, dim: int, tau_scale: float = 60.0, gap_mode: str = "previous") -> "RoteConfig":
        if dim < 2 or dim % 2 != 0:
            raise ValueError("rotary encoding needs an even dim >= 2")
        half = dim // 2
        freqs = 10000.0 ** (-2.0 * np.arange(half) / dim)
        return cls(freqs, freqs.copy(), tau_scale, gap_mode)

    @property
    def half_dim(self) -> int:
        return self.pos_freqs.size

    def device_freqs(self, device) -> tuple[torch.Tensor, torch.Tensor]:
        """fp64 copies of the schedules on ``device``, uploaded once per
        (device, schedule values): reassigning pos_freqs / temp_freqs
        re-uploads.  Call it (or run one eager step) before capturing a CUDA
        graph — the upload is a host copy."""
        key = (str(device), id(self.pos_freqs), id(self.temp_freqs), self.pos_freqs.tobytes().__hash__(),
               self.temp_freqs.tobytes().__hash__())
        if key not in self._dev:
            self._dev[key] = (torch.tensor(self.pos_freqs, device=device, dtype=torch.float64),
                              torch.tensor(self.temp_freqs, device=device, dtype=torch.float64))
        return self._dev[key]


def temporal_angle(delta_t: float, cfg: RoteConfig) -> float:
    """Log-scaled gap value fed to the temporal frequencies (preproc.py:155-159)."""
    if delta_t < 0:
        raise ValueError(f"time gap must be >= 0, got {delta_t}")
    return float(np.log1p(delta_t / cfg.tau_scale))


def _launch(x, lengths, ts, cfg, inverse):
    y = torch.empty_like(x)
    a = _capi.RoteArgs()
    a.B, a.T, a.d, a.dtype = x.shape[0], x.shape[1], x.shape[2], _capi.dt(x)
    a.x, a.x_rs, a.x_bs = x.data_ptr(), x.stride(1), x.stride(0)
    a.y, a.y_rs, a.y_bs = y.data_ptr(), y.stride(1), y.stride(0)
    a.lengths = lengths.data_ptr() if lengths is not None else None
    a.timestamps = ts.data_ptr() if ts is not None else None
    a.ts_bs = ts.stride(0) if ts is not None else 0
    pf, tf = cfg.device_freqs(x.device)
    a.pos_freqs, a.temp_freqs = pf.data_ptr(), tf.data_ptr()
    a.tau_scale, a.gap_mode, a.inverse = float(cfg.tau_scale), 0 if cfg.gap_mode == "previous" else 1, int(inverse)
    _capi.call("kl_rote", C.byref(a), _capi._stream())
    return y


class _Rote(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, lengths, ts, cfg):
        ctx.cfg, ctx.lengths, ctx.ts = cfg, lengths, ts
        return _launch(x, lengths, ts, cfg, False)

    @staticmethod
    def backward(ctx, g):
        return _launch(g.contiguous(), ctx.lengths, ctx.ts, ctx.cfg, True), None, None, None


def rote_sequence(s: torch.Tensor, timestamps, cfg: RoteConfig, lengths: torch.Tensor | None = None) -> torch.Tensor:
    """Apply the rotary encoding to every valid row (preproc.py:187-199).

    ``s``: (T, d) or (B, T, d) CUDA tensor (fp32 or bf16); ``timestamps``:
    None or (T,) / (B, T) event times (seconds; cast to fp64); ``lengths``:
    optional (B,) valid-row counts (rows 0..len-1 are the sequence, as the
    reference's unpadded (len, d) input)."""
    single = s.dim() == 2
    x = s.unsqueeze(0) if single else s
    if x.dim() != 3:
        raise ShapeError(f"rote_sequence expects (T, d) or (B, T, d), got {tuple(s.shape)}")
    if x.shape[-1] != 2 * cfg.half_dim:
        raise ShapeError(f"rotary config covers dim {2 * cfg.half_dim}, input has {x.shape[-1]}")
    _capi._need_cuda(x)
    x = x.contiguous()
    ts = None
    if timestamps is not None:
        ts = torch.as_tensor(timestamps, dtype=torch.float64, device=x.device).reshape(x.shape[0], x.shape[1])
        ts = ts.contiguous()
    ln = None
    if lengths is not None:
        ln = torch.as_tensor(lengths, device=x.device).to(torch.int32).contiguous()
        if ln.numel() != x.shape[0]:
            raise ShapeError(f"need one length per sample ({x.shape[0]}), got {ln.numel()}")
        if not torch.cuda.is_current_stream_capturing():  # (the kernels also clamp to [0, T])
            lo, hi = int(ln.min()), int(ln.max())
            if lo < 0 or hi > x.shape[1]:
                raise ValueError(f"lengths must lie in [0, {x.shape[1]}], got [{lo}, {hi}]")
    if x.numel() == 0:  # T = 0: the reference returns the (empty) input
        return s
    y = _Rote.apply(x, ln, ts, cfg)
    return y[0] if single else y
