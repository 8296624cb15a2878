"""torch plumbing for the native calls: device placement, streams,
workspaces, ExecStats conversion.  torch supplies device memory and streams
only; all compute goes through libsg's sm_100a kernels."""

import ctypes

import numpy as np
import torch

from . import _native
from .core import ExecStats, KernelCounters, LaunchRecord


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 graph kernels have no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def dtype_code(t):
    if t.dtype == torch.int64:
        return _native.SG_I64
    if t.dtype == torch.int32:
        return _native.SG_I32
    if hasattr(torch, "uint32") and t.dtype == torch.uint32:
        return _native.SG_U32
    raise TypeError(f"unsupported index dtype {t.dtype}")


def to_device(x, device):
    """numpy / host tensor / device tensor -> contiguous CUDA tensor on `device`.
    Returns (tensor, was_host)."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            if x.device != device:
                raise ValueError(f"input lives on {x.device}, expected {device}")
            return x.contiguous(), False
        return x.contiguous().to(device, non_blocking=x.is_pinned()), True
    arr = np.ascontiguousarray(x)
    return torch.from_numpy(arr).to(device), True


def workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def exec_stats(st):
    """native sg_stats -> ExecStats (launch log built lazily, barriers,
    device wall time)."""
    es = ExecStats(backend="sm_100a")
    nl = min(st.n_launches, _native.SG_MAX_LAUNCHES)
    resolved = []

    def resolve():  # event times are read on first use (sg_stats_resolve)
        if not resolved:
            rc = _native.lib().sg_stats_resolve(ctypes.byref(st))
            resolved.append(rc == _native.SG_OK)
            if rc != _native.SG_OK:
                es.warnings.append("launch timings unavailable: this call's CUDA events were recycled "
                                   "(read ExecStats timings within 64 calls on the device)")
        return resolved[0]

    def build():  # `st` is this call's own sg_stats, kept alive by the closure
        ok = resolve()
        out = []
        for k in range(nl):
            L = st.launch[k]
            ms = float(L.ms) if ok else float("nan")  # unavailable, see es.warnings
            out.append(LaunchRecord(kernel=_native.kernel_name(L.kernel),
                                    counters=KernelCounters(launches=1, items=int(L.items), ms=ms),
                                    round=int(L.round), blocks=int(L.blocks), threads=int(L.threads), ms=ms))
        return out

    def wall():
        return float(st.total_ms) / 1e3 if resolve() else None

    es.set_launch_log_source(build)
    es.set_wall_time_source(wall)
    es.barriers = max(0, nl - 1)
    return es


def to_host_numpy(t):
    """D2H through a (cached) pinned buffer -> numpy int64 array that owns
    the pinned block.  Pageable copies run at a fraction of PCIe speed."""
    t = t.to(torch.int64)
    host = torch.empty(t.shape, dtype=torch.int64, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return host.numpy()
