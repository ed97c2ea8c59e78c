"""Batched V-trace targets on the device.

Argument marshalling only: the computation is `vtrace_kernel` (csrc/vtrace.cuh) behind the
C-ABI call `cule_vtrace` (include/cule.h).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .env import _stream_ptr


def vtrace(rewards: torch.Tensor, values: torch.Tensor, bootstrap: torch.Tensor, log_mu: torch.Tensor,
           log_pi: torch.Tensor, dones: torch.Tensor, gamma: float, rho_bar: float = 1.0, c_bar: float = 1.0,
           stream=None, out=None):
    """Time-major [T, B] float32 CUDA tensors (bootstrap [B], dones uint8 [T, B]) ->
    (vs, rho, advantages), each float32 [T, B] (written into `out` = (vs, rho, adv) if given)."""
    T, B = rewards.shape
    for name, x, dt, shape in (("rewards", rewards, torch.float32, (T, B)), ("values", values, torch.float32, (T, B)),
                               ("bootstrap", bootstrap, torch.float32, (B,)),
                               ("log_mu", log_mu, torch.float32, (T, B)), ("log_pi", log_pi, torch.float32, (T, B)),
                               ("dones", dones, torch.uint8, (T, B))):
        if x.dtype != dt or not x.is_cuda or tuple(x.shape) != shape or not x.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {dt} CUDA tensor of shape {shape}")
    dev = rewards.device
    for name, x in (("values", values), ("bootstrap", bootstrap), ("log_mu", log_mu), ("log_pi", log_pi),
                    ("dones", dones)):
        if x.device != dev:
            raise ValueError(f"{name} must be on {dev}")
    if out is not None:
        if len(out) != 3:
            raise ValueError("out must be (vs, rho, adv)")
        for name, x in zip(("vs", "rho", "adv"), out):
            if x.dtype != torch.float32 or x.device != dev or tuple(x.shape) != (T, B) or not x.is_contiguous():
                raise ValueError(f"out {name} must be a contiguous float32 tensor [T, B] on {dev}")
        vs, rho, adv = out
    else:
        vs, rho, adv = torch.empty_like(rewards), torch.empty_like(rewards), torch.empty_like(rewards)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    with torch.cuda.device(dev):
        _lib.check(_lib.load().cule_vtrace(p(rewards), p(values), p(bootstrap), p(log_mu), p(log_pi), p(dones),
                                           T, B, gamma, rho_bar, c_bar, p(vs), p(rho), p(adv),
                                           ctypes.c_void_p(_stream_ptr(stream, dev))))
    return vs, rho, adv
