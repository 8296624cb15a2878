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


# host arrays at least this long cross PCIe as 32-bit ids (narrowed / widened
# on the host, pipelined against the DMA: sg_xfer.cu); shorter ones move as
# int64, where the pipeline's setup would cost more than the bytes it saves
NARROW_MIN = 1 << 20


def _narrow_h2d(addr, shape, count, bound, device):
    d = torch.empty(shape, dtype=torch.int32, device=device)
    ok = ctypes.c_int(1)
    _native.check(_native.lib().sg_h2d_narrow_i64(ctypes.c_void_p(addr), count, ptr(d), bound, stream_ptr(device),
                                                  ctypes.byref(ok)), "sg_h2d_narrow_i64")
    return d if ok.value else None


def to_device(x, device, bound=None):
    """numpy / host tensor / device tensor -> contiguous CUDA tensor on `device`.
    Returns (tensor, was_host).  With `bound` (ids lie in [0, bound) for a
    valid input, bound <= 2^31), a long int64 host array arrives as int32:
    narrowed on the host while earlier chunks are in flight; a value outside
    the bound falls back to the int64 copy, so the device reports the
    reference's exact error."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            if x.device != device:
                raise ValueError(f"input lives on {x.device}, expected {device}")
            return x.contiguous(), False
        h = x.contiguous()
        if bound is not None and bound <= 2**31 and h.dtype == torch.int64 and h.numel() >= NARROW_MIN:
            d = _narrow_h2d(h.data_ptr(), tuple(h.shape), h.numel(), bound, device)
            if d is not None:
                return d, True
        return h.to(device, non_blocking=h.is_pinned()), True
    arr = np.ascontiguousarray(x)
    if bound is not None and bound <= 2**31 and arr.dtype == np.int64 and arr.size >= NARROW_MIN:
        d = _narrow_h2d(arr.ctypes.data, arr.shape, arr.size, bound, device)
        if d is not None:
            return d, True
    return torch.from_numpy(arr).to(device), True


def host_out_dtype(n):
    """Device dtype of a result that goes back to a host caller: int32 when
    it is long enough to cross PCIe narrowed (to_host_numpy widens it)."""
    return torch.int32 if NARROW_MIN <= n < 2**31 else torch.int64


def workspace(nbytes, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def exec_stats(st):
    """native sg_stats -> ExecStats (launch log built lazily, barriers,
    device wall time)."""
    es = ExecStats(backend="sm_100a")
    nl = min(st.n_launches, _native.SG_MAX_LAUNCHES)
    resolved = []
    warnings = es.warnings  # (the closures hold the list, not `es`: no reference cycle, so a
    #                          dropped ExecStats -- and the meta arrays it holds -- is freed at once)

    def resolve():  # event times are read on first use (sg_stats_resolve)
        if not resolved:
            rc = _native.lib().sg_stats_resolve(ctypes.byref(st))
            resolved.append(rc == _native.SG_OK)
            if rc != _native.SG_OK:
                warnings.append("launch timings unavailable: this call's CUDA events were recycled "
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
    """Device ids -> numpy int64 array owning a pinned block (torch's pinned
    caching allocator: no page faults, full PCIe speed).  A long int32 result
    crosses PCIe as 32 bits and is widened on the host, chunk by chunk behind
    the copy (sg_d2h_widen_u32)."""
    host = torch.empty(t.shape, dtype=torch.int64, pin_memory=True)
    if t.dtype == torch.int32 and t.numel() >= NARROW_MIN and t.is_contiguous():
        _native.check(_native.lib().sg_d2h_widen_u32(ptr(t), t.numel(), ctypes.c_void_p(host.data_ptr()),
                                                    stream_ptr(t.device)), "sg_d2h_widen_u32")
        return host.numpy()
    host.copy_(t.to(torch.int64), non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return host.numpy()
