"""Python mirror of the reference operator API (proj/core/include/jagged/*.hpp) over the C-ABI.

Same operator names, argument order and error texts as the reference; tensors live on the GPU:
  JaggedTensor(offsets, values)   offsets int64 [B+1] (cuda), values [total_rows, dim] or
                                  [total_rows, heads, head_dim] (attention), float32 or bfloat16
  Jagged2Tensor(offsets, sq_offsets, values)   per-sample Bi x Bi blocks, values [sum Bi^2]
  DenseTensor = a plain torch tensor ([B, D, T] weights, padded [B, L, D] forms)
Every call is stream-ordered on torch's current stream and launches CUDA kernels from
libjagged_b200.so; nothing here computes on the CPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import JG_BF16, JG_F32, JaggedError, check

__all__ = [
    "JaggedTensor", "Jagged2Tensor", "JaggedAttentionSaved", "AttentionGrads", "Schedule", "make_jagged",
    "jagged_dense_bmm", "jagged_jagged_bmm", "jagged_softmax", "jagged_jagged_bmm_jagged_out",
    "array_jagged_bmm_jagged_out", "jagged2_softmax", "jagged_dense_bmm_vjp", "jagged_jagged_bmm_vjp",
    "jagged_softmax_vjp", "jagged_jagged_bmm_jagged_out_vjp", "array_jagged_bmm_jagged_out_vjp",
    "jagged2_softmax_vjp", "jagged_flash_attention_forward", "jagged_flash_attention_backward",
    "jagged_attention", "DenseAttentionSaved", "dense_flash_attention", "dense_flash_attention_backward",
    "jagged_to_dense", "dense_to_jagged", "jagged2_to_dense", "dense_to_jagged2",
    "add", "sub", "mul", "scale", "JaggedError",
]


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return JG_F32
    if t.dtype == torch.bfloat16:
        return JG_BF16
    return 2  # f64 and others -> JG_UNSUPPORTED from the library


def _p(t):
    return None if t is None else t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream():
    # the raw cudaStream_t of torch's current stream; torch.cuda.current_stream() builds a Stream object per call
    # (~3 us), which dominated the host cost of small launches (cfg2)
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


class JaggedTensor:
    """Flat values + offsets (tensor.hpp:14-37). Validates the reference invariants on host."""

    def __init__(self, offsets, values: torch.Tensor, host_offsets: np.ndarray | None = None):
        if host_offsets is None:
            host_offsets = (offsets.cpu().numpy() if isinstance(offsets, torch.Tensor)
                            else np.asarray(offsets, np.int64))
        host_offsets = np.ascontiguousarray(host_offsets, dtype=np.int64)
        if values.dim() < 2 or values.shape[-1] <= 0:
            raise JaggedError("JaggedTensor: dim must be positive")
        if host_offsets.size == 0 or host_offsets[0] != 0:
            raise JaggedError("JaggedTensor: offsets must start with 0")
        bad = np.nonzero(np.diff(host_offsets) < 0)[0]
        if bad.size:
            raise JaggedError(f"JaggedTensor: offsets must be non-decreasing at index {int(bad[0]) + 1}")
        if host_offsets[-1] != values.shape[0]:
            per = int(np.prod(values.shape[1:]))
            raise JaggedError(f"JaggedTensor: expected {int(host_offsets[-1]) * per} value elements, "
                              f"got {values.numel()}")
        self.host_offsets = host_offsets
        if isinstance(offsets, torch.Tensor) and offsets.is_cuda:
            self.offsets = offsets.to(torch.int64).contiguous()
        else:
            self.offsets = torch.from_numpy(host_offsets).to(values.device)
        self.values = values.contiguous()

    batch = property(lambda self: len(self.host_offsets) - 1)
    total_rows = property(lambda self: int(self.host_offsets[-1]))
    dim = property(lambda self: int(self.values.shape[-1]))
    num_heads = property(lambda self: int(self.values.shape[1]) if self.values.dim() == 3 else 1)

    def lengths(self) -> np.ndarray:
        return np.diff(self.host_offsets)

    def same_offsets(self, other: "JaggedTensor") -> bool:
        return self.host_offsets is other.host_offsets or np.array_equal(self.host_offsets, other.host_offsets)

    def with_values(self, values: torch.Tensor) -> "JaggedTensor":
        # values of the same leading extent (an operator output): the offsets invariants already hold
        if values.dim() >= 2 and values.shape[0] == self.values.shape[0] and values.shape[-1] > 0 \
                and values.is_contiguous():
            t = JaggedTensor.__new__(JaggedTensor)
            t.host_offsets, t.offsets, t.values = self.host_offsets, self.offsets, values
            return t
        return JaggedTensor(self.offsets, values, self.host_offsets)


class Jagged2Tensor:
    """Per-sample Bi x Bi blocks at sq_offsets (tensor.hpp:42-62)."""

    def __init__(self, offsets, values: torch.Tensor, host_offsets: np.ndarray, sq_offsets=None):
        self.host_offsets = np.ascontiguousarray(host_offsets, np.int64)
        ln = np.diff(self.host_offsets)
        if (ln < 0).any():
            raise JaggedError(f"Jagged2Tensor: negative length at sample {int(np.nonzero(ln < 0)[0][0])}")
        self.sum_sq = int((ln * ln).sum())
        if values.numel() != self.sum_sq:
            raise JaggedError(f"Jagged2Tensor: expected {self.sum_sq} value elements, got {values.numel()}")
        self.offsets = offsets if isinstance(offsets, torch.Tensor) else torch.from_numpy(self.host_offsets).cuda()
        if sq_offsets is None:
            sq_offsets = torch.empty(len(self.host_offsets), dtype=torch.int64, device=values.device)
            check(_lib.lib().jg_sq_offsets(_p(self.offsets), self.batch, _p(sq_offsets), _stream()))
        self.sq_offsets = sq_offsets
        self.values = values.contiguous().view(-1)

    batch = property(lambda self: len(self.host_offsets) - 1)

    def seq_lengths(self) -> np.ndarray:
        return np.diff(self.host_offsets)


@dataclass
class JaggedAttentionSaved:
    """attention.hpp:26-32: output + per-row logsumexp ([H, total_rows] float32) + block sizes."""
    output: JaggedTensor
    logsumexp: torch.Tensor
    block_q: int = 64
    block_k: int = 64


@dataclass
class DenseAttentionSaved:
    """attention.hpp:19-24: padded output [B, L, (H,) D], logsumexp ([H, B*L] float32, -inf past each
    sample's length) and block sizes."""
    output: torch.Tensor
    logsumexp: torch.Tensor
    block_q: int = 64
    block_k: int = 64


@dataclass
class AttentionGrads:
    dq: JaggedTensor
    dk: JaggedTensor
    dv: JaggedTensor


class Schedule:
    """Device work list (LPT-ordered (sample, 128-row tile) items) reused across fwd/bwd calls."""

    def __init__(self, x: JaggedTensor):
        import ctypes as C

        self._h = C.c_void_p()
        check(_lib.lib().jg_schedule_create(_p(x.offsets), x.batch, x.total_rows, _stream(), C.byref(self._h)))
        self.handle = self._h.value
        self._x = x  # keep offsets alive

    def work_list(self) -> np.ndarray:
        import ctypes as C

        n = C.c_int64()
        check(_lib.lib().jg_schedule_work_list(self.handle, None, 0, C.byref(n)))
        buf = np.empty((n.value, 2), np.int32)
        check(_lib.lib().jg_schedule_work_list(self.handle, buf.ctypes.data, n.value, C.byref(n)))
        return buf

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _lib.lib().jg_schedule_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def make_jagged(lengths, values: torch.Tensor) -> JaggedTensor:
    """tensor.hpp:96-98 — offsets are the prefix sum of lengths, computed on device."""
    lengths = np.ascontiguousarray(np.asarray(lengths, np.int64))
    neg = np.nonzero(lengths < 0)[0]
    if neg.size:
        raise JaggedError(f"make_jagged: negative length at sample {int(neg[0])}")
    dev_len = torch.from_numpy(lengths).to(values.device)
    off = torch.empty(len(lengths) + 1, dtype=torch.int64, device=values.device)
    check(_lib.lib().jg_make_offsets(_p(dev_len), len(lengths), _p(off), None, _stream()))
    host = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    per = int(np.prod(values.shape[1:])) if values.dim() > 1 else 1
    if values.numel() != host[-1] * per:
        raise JaggedError(f"make_jagged: expected {int(host[-1]) * per} value elements, got {values.numel()}")
    return JaggedTensor(off, values, host)


def _require_matching_offsets(a: JaggedTensor, b: JaggedTensor, op: str) -> None:
    # linalg.cpp:16-26
    if a.batch != b.batch:
        raise JaggedError(f"{op}: batch mismatch ({a.batch} vs {b.batch})")
    la, lb = a.lengths(), b.lengths()
    diff = np.nonzero(la != lb)[0]
    if diff.size:
        raise JaggedError(f"{op}: offsets differ first at sample {int(diff[0])}")


def _operands(op: str, ref: torch.Tensor, *others) -> None:
    """Paired operands share the reference operand's dtype and live on its CUDA device: the C-ABI takes one
    dtype per call, so a mismatch would make a kernel read past a buffer (or dereference a host pointer)."""
    for t in (ref,) + others:
        if t is None:
            continue
        if not t.is_cuda:
            raise JaggedError(f"{op}: operands must be CUDA tensors")
        if t.device != ref.device:
            raise JaggedError(f"{op}: operands must be on one device ({ref.device} vs {t.device})")
        if t.dtype != ref.dtype:
            raise JaggedError(f"{op}: dtype mismatch ({ref.dtype} vs {t.dtype})")


def _out_dtype(x: torch.Tensor, out_dtype):
    return x.dtype if out_dtype is None else out_dtype


# ------------------------------------------------------------------ forward operators
def jagged_dense_bmm(x: JaggedTensor, w: torch.Tensor, out_dtype=None) -> JaggedTensor:
    if w.dim() != 3:
        raise JaggedError("jagged_dense_bmm: w must be [B, D, T]")
    B, D, T = w.shape
    if B != x.batch:
        raise JaggedError(f"jagged_dense_bmm: batch mismatch ({x.batch} vs {B})")
    if D != x.dim:
        raise JaggedError(f"jagged_dense_bmm: dim mismatch ({x.dim} vs {D})")
    _operands("jagged_dense_bmm", x.values, w)
    out = torch.empty(x.total_rows, T, dtype=_out_dtype(x.values, out_dtype), device=x.values.device)
    check(_lib.lib().jg_jagged_dense_bmm(_p(x.offsets), x.batch, x.total_rows, D, T, _p(x.values),
                                         _p(w.contiguous()), _p(out), _dt(x.values), _dt(out), _stream()))
    return x.with_values(out)


def jagged_jagged_bmm(x: JaggedTensor, y: JaggedTensor, out_dtype=None) -> torch.Tensor:
    _require_matching_offsets(x, y, "jagged_jagged_bmm")
    _operands("jagged_jagged_bmm", x.values, y.values)
    out = torch.empty(x.batch, x.dim, y.dim, dtype=_out_dtype(x.values, out_dtype), device=x.values.device)
    check(_lib.lib().jg_jagged_jagged_bmm(_p(x.offsets), x.batch, x.total_rows, x.dim, y.dim, _p(x.values),
                                          _p(y.values), _p(out), _dt(x.values), _dt(out), _stream()))
    return out


def jagged_softmax(x: JaggedTensor) -> JaggedTensor:
    _operands("jagged_softmax", x.values)
    out = torch.empty_like(x.values)
    check(_lib.lib().jg_jagged_softmax(_p(x.offsets), x.batch, x.total_rows, x.dim, _p(x.values), _p(out),
                                       _dt(x.values), _stream()))
    return x.with_values(out)


def jagged_jagged_bmm_jagged_out(q: JaggedTensor, k: JaggedTensor, out_dtype=None) -> Jagged2Tensor:
    _require_matching_offsets(q, k, "jagged_jagged_bmm_jagged_out")
    if q.dim != k.dim:
        raise JaggedError(f"jagged_jagged_bmm_jagged_out: dim mismatch ({q.dim} vs {k.dim})")
    _operands("jagged_jagged_bmm_jagged_out", q.values, k.values)
    ln = q.lengths()
    sq = torch.empty(q.batch + 1, dtype=torch.int64, device=q.values.device)
    check(_lib.lib().jg_sq_offsets(_p(q.offsets), q.batch, _p(sq), _stream()))
    out = torch.empty(int((ln * ln).sum()), dtype=_out_dtype(q.values, out_dtype), device=q.values.device)
    check(_lib.lib().jg_jagged_jagged_bmm_jagged_out(_p(q.offsets), _p(sq), q.batch, q.total_rows, q.dim,
                                                     _p(q.values), _p(k.values), _p(out), _dt(q.values), _dt(out),
                                                     _stream()))
    return Jagged2Tensor(q.offsets, out, q.host_offsets, sq)


def array_jagged_bmm_jagged_out(a: Jagged2Tensor, v: JaggedTensor, out_dtype=None) -> JaggedTensor:
    if a.batch != v.batch:
        raise JaggedError(f"array_jagged_bmm_jagged_out: batch mismatch ({a.batch} vs {v.batch})")
    diff = np.nonzero(a.seq_lengths() != v.lengths())[0]
    if diff.size:
        raise JaggedError(f"array_jagged_bmm_jagged_out: length mismatch at sample {int(diff[0])}")
    _operands("array_jagged_bmm_jagged_out", v.values, a.values)
    out = torch.empty(v.values.shape, dtype=_out_dtype(v.values, out_dtype), device=v.values.device)
    check(_lib.lib().jg_array_jagged_bmm_jagged_out(_p(v.offsets), _p(a.sq_offsets), v.batch, v.total_rows, a.sum_sq,
                                                    v.dim,
                                                    _p(a.values), _p(v.values), _p(out), _dt(v.values), _dt(out),
                                                    _stream()))
    return v.with_values(out)


def jagged2_softmax(s: Jagged2Tensor) -> Jagged2Tensor:
    _operands("jagged2_softmax", s.values)
    out = torch.empty_like(s.values)
    check(_lib.lib().jg_jagged2_softmax(_p(s.offsets), _p(s.sq_offsets), s.batch, _p(s.values), _p(out),
                                        _dt(s.values), _stream()))
    return Jagged2Tensor(s.offsets, out, s.host_offsets, s.sq_offsets)


# ------------------------------------------------------------------ VJPs
def jagged_dense_bmm_vjp(x: JaggedTensor, w: torch.Tensor, grad_out: JaggedTensor, out_dtype=None):
    if w.dim() != 3:
        raise JaggedError("jagged_dense_bmm_vjp: w must be [B, D, T]")
    _require_matching_offsets(x, grad_out, "jagged_dense_bmm_vjp")
    B, D, T = w.shape
    if grad_out.dim != T:
        raise JaggedError("jagged_dense_bmm_vjp: grad_out dim mismatch")
    _operands("jagged_dense_bmm_vjp", x.values, w, grad_out.values)
    od = _out_dtype(x.values, out_dtype)
    dx = torch.empty(x.values.shape, dtype=od, device=x.values.device)
    dw = torch.empty(w.shape, dtype=od, device=x.values.device)
    check(_lib.lib().jg_jagged_dense_bmm_vjp(_p(x.offsets), x.batch, x.total_rows, D, T, _p(x.values),
                                             _p(w.contiguous()), _p(grad_out.values), _p(dx), _p(dw), _dt(x.values),
                                             _dt(dx), _stream()))
    return x.with_values(dx), dw


def jagged_jagged_bmm_vjp(x: JaggedTensor, y: JaggedTensor, grad_out: torch.Tensor, out_dtype=None):
    _require_matching_offsets(x, y, "jagged_jagged_bmm_vjp")
    if grad_out.dim() != 3 or tuple(grad_out.shape) != (x.batch, x.dim, y.dim):
        raise JaggedError("jagged_jagged_bmm_vjp: grad_out must be [B, D, T]")
    _operands("jagged_jagged_bmm_vjp", x.values, y.values, grad_out)
    od = _out_dtype(x.values, out_dtype)
    dx = torch.empty(x.values.shape, dtype=od, device=x.values.device)
    dy = torch.empty(y.values.shape, dtype=od, device=x.values.device)
    check(_lib.lib().jg_jagged_jagged_bmm_vjp(_p(x.offsets), x.batch, x.total_rows, x.dim, y.dim, _p(x.values),
                                              _p(y.values), _p(grad_out.contiguous()), _p(dx), _p(dy),
                                              _dt(x.values), _dt(dx), _stream()))
    return x.with_values(dx), y.with_values(dy)


def jagged_softmax_vjp(x: JaggedTensor, grad_out: JaggedTensor) -> JaggedTensor:
    _require_matching_offsets(x, grad_out, "jagged_softmax_vjp")
    if x.dim != grad_out.dim:
        raise JaggedError("jagged_softmax_vjp: dim mismatch")
    _operands("jagged_softmax_vjp", x.values, grad_out.values)
    dx = torch.empty_like(x.values)
    check(_lib.lib().jg_jagged_softmax_vjp(_p(x.offsets), x.batch, x.total_rows, x.dim, _p(x.values),
                                           _p(grad_out.values), _p(dx), _dt(x.values), _stream()))
    return x.with_values(dx)


def jagged_jagged_bmm_jagged_out_vjp(q: JaggedTensor, k: JaggedTensor, grad_out: Jagged2Tensor, out_dtype=None):
    _require_matching_offsets(q, k, "jagged_jagged_bmm_jagged_out_vjp")
    diff = np.nonzero(grad_out.seq_lengths() != q.lengths())[0]
    if diff.size:
        raise JaggedError(f"jagged_jagged_bmm_jagged_out_vjp: grad_out length mismatch at sample {int(diff[0])}")
    _operands("jagged_jagged_bmm_jagged_out_vjp", q.values, k.values, grad_out.values)
    od = _out_dtype(q.values, out_dtype)
    dq = torch.empty(q.values.shape, dtype=od, device=q.values.device)
    dk = torch.empty(k.values.shape, dtype=od, device=q.values.device)
    check(_lib.lib().jg_jagged_jagged_bmm_jagged_out_vjp(_p(q.offsets), _p(grad_out.sq_offsets), q.batch, q.total_rows,
                                                         grad_out.sum_sq, q.dim, _p(q.values), _p(k.values), _p(grad_out.values),
                                                         _p(dq), _p(dk), _dt(q.values), _dt(dq), _stream()))
    return q.with_values(dq), k.with_values(dk)


def array_jagged_bmm_jagged_out_vjp(a: Jagged2Tensor, v: JaggedTensor, grad_out: JaggedTensor, out_dtype=None):
    _require_matching_offsets(v, grad_out, "array_jagged_bmm_jagged_out_vjp")
    diff = np.nonzero(a.seq_lengths() != v.lengths())[0]
    if diff.size:
        raise JaggedError(f"array_jagged_bmm_jagged_out_vjp: length mismatch at sample {int(diff[0])}")
    _operands("array_jagged_bmm_jagged_out_vjp", v.values, a.values, grad_out.values)
    od = _out_dtype(v.values, out_dtype)
    da = torch.empty(a.values.shape, dtype=od, device=v.values.device)
    dv = torch.empty(v.values.shape, dtype=od, device=v.values.device)
    check(_lib.lib().jg_array_jagged_bmm_jagged_out_vjp(_p(v.offsets), _p(a.sq_offsets), v.batch, v.total_rows,
                                                        a.sum_sq, v.dim,
                                                        _p(a.values), _p(v.values), _p(grad_out.values), _p(da),
                                                        _p(dv), _dt(v.values), _dt(dv), _stream()))
    return Jagged2Tensor(a.offsets, da, a.host_offsets, a.sq_offsets), v.with_values(dv)


def jagged2_softmax_vjp(s: Jagged2Tensor, grad_out: Jagged2Tensor) -> Jagged2Tensor:
    if s.batch != grad_out.batch or not np.array_equal(s.seq_lengths(), grad_out.seq_lengths()):
        raise JaggedError("jagged2_softmax_vjp: layout mismatch")
    _operands("jagged2_softmax_vjp", s.values, grad_out.values)
    ds = torch.empty_like(s.values)
    check(_lib.lib().jg_jagged2_softmax_vjp(_p(s.offsets), _p(s.sq_offsets), s.batch, _p(s.values),
                                            _p(grad_out.values), _p(ds), _dt(s.values), _stream()))
    return Jagged2Tensor(s.offsets, ds, s.host_offsets, s.sq_offsets)


# ------------------------------------------------------------------ attention
def _heads(x: JaggedTensor):
    v = x.values
    return (int(v.shape[1]), int(v.shape[2])) if v.dim() == 3 else (1, int(v.shape[1]))


def _require_attention_inputs(q, k, v, op):
    # attention.cpp:33-40
    if q.dim != k.dim or q.dim != v.dim or q.values.shape != k.values.shape or q.values.shape != v.values.shape:
        raise JaggedError(f"{op}: dim mismatch")
    if not q.same_offsets(k) or not q.same_offsets(v):
        raise JaggedError(f"{op}: q, k, v must share offsets")
    _operands(op, q.values, k.values, v.values)


def jagged_flash_attention_forward(q: JaggedTensor, k: JaggedTensor, v: JaggedTensor, block_q: int = 64,
                                   block_k: int = 64, schedule: Schedule | None = None) -> JaggedAttentionSaved:
    _require_attention_inputs(q, k, v, "jagged_flash_attention_forward")
    if block_q < 1 or block_k < 1:
        raise JaggedError("jagged_flash_attention_forward: block sizes must be >= 1")
    H, D = _heads(q)
    out = torch.empty_like(q.values)
    lse = torch.empty(H, q.total_rows, dtype=torch.float32, device=q.values.device)
    check(_lib.lib().jg_jagged_flash_attention_forward(
        _p(q.offsets), q.batch, q.total_rows, H, D, _p(q.values), _p(k.values), _p(v.values), block_q, block_k,
        _p(out), _p(lse), _dt(q.values), schedule.handle if schedule else None, _stream()))
    return JaggedAttentionSaved(q.with_values(out), lse, block_q, block_k)


def jagged_flash_attention_backward(q: JaggedTensor, k: JaggedTensor, v: JaggedTensor, grad_out: JaggedTensor,
                                    saved: JaggedAttentionSaved, schedule: Schedule | None = None,
                                    workspace: torch.Tensor | None = None, deterministic: bool = True) -> AttentionGrads:
    """attention.cpp:227-289. Gradients are bit-reproducible on every device path; the
    `deterministic` flag is passed through the C-ABI for API completeness. workspace: optional device buffer of
    workspace_size(q) bytes (reused across calls; not shared by concurrent calls)."""
    _require_attention_inputs(q, k, v, "jagged_flash_attention_backward")
    if not grad_out.same_offsets(q) or grad_out.values.shape != q.values.shape:
        raise JaggedError("jagged_flash_attention_backward: grad_out layout mismatch")
    H, D = _heads(q)
    if (not saved.output.same_offsets(q) or saved.output.values.shape != q.values.shape
            or saved.logsumexp.numel() != q.total_rows * H or saved.block_q < 1 or saved.block_k < 1):
        raise JaggedError("jagged_flash_attention_backward: saved state does not match inputs")
    _operands("jagged_flash_attention_backward", q.values, grad_out.values, saved.output.values)
    lse = saved.logsumexp
    if lse.dtype != torch.float32 or not lse.is_cuda or lse.device != q.values.device or not lse.is_contiguous():
        raise JaggedError("jagged_flash_attention_backward: logsumexp must be a contiguous float32 CUDA tensor")
    if workspace is not None:
        if not workspace.is_cuda or workspace.device != q.values.device:
            raise JaggedError("jagged_flash_attention_backward: workspace must be on the inputs' CUDA device")
        need = backward_workspace_size(q)
        if workspace.numel() * workspace.element_size() < need or not workspace.is_contiguous():
            raise JaggedError(f"jagged_flash_attention_backward: workspace needs {need} contiguous bytes")
    dq, dk, dv = (torch.empty_like(q.values) for _ in range(3))
    check(_lib.lib().jg_jagged_flash_attention_backward(
        _p(q.offsets), q.batch, q.total_rows, H, D, _p(q.values), _p(k.values), _p(v.values), _p(grad_out.values),
        _p(saved.output.values), _p(saved.logsumexp), saved.block_q, saved.block_k, _p(dq), _p(dk), _p(dv),
        _dt(q.values), 1 if deterministic else 0, schedule.handle if schedule else None, _p(workspace), _stream()))
    return AttentionGrads(q.with_values(dq), k.with_values(dk), v.with_values(dv))


def backward_workspace_size(q: JaggedTensor) -> int:
    """Bytes of the jagged_flash_attention_backward workspace for q's layout (C-ABI
    jg_attention_backward_workspace_size)."""
    H, D = _heads(q)
    return int(_lib.lib().jg_attention_backward_workspace_size(q.total_rows, q.batch, H, D))


def _dense_attention_inputs(q, k, v, lengths, op):
    # attention.cpp:19-31 (require_self_attention_inputs); q/k/v are [B, L, D] (one head, as the reference)
    # or [B, L, H, D]
    if q.dim() not in (3, 4) or q.shape != k.shape or q.shape != v.shape:
        raise JaggedError(f"{op}: q, k, v must share a [B, L, D] shape")
    ln = np.asarray(lengths, dtype=np.int64).reshape(-1)
    if ln.shape[0] != q.shape[0]:
        raise JaggedError(f"{op}: lengths size mismatch")
    for i, n in enumerate(ln):
        if n < 0 or n > q.shape[1]:
            raise JaggedError(f"{op}: sample {i} length {int(n)} out of bounds for L={int(q.shape[1])}")
    H = 1 if q.dim() == 3 else int(q.shape[2])
    return np.ascontiguousarray(ln), int(q.shape[0]), int(q.shape[1]), H, int(q.shape[-1])


def dense_flash_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, lengths, block_q: int = 64,
                          block_k: int = 64) -> DenseAttentionSaved:
    """attention.cpp:106-160 on the GPU: the jagged kernels in padded mode (segments of max_len rows, keys
    and rows past each length masked), doing the full padded L^2 work — the padded baseline."""
    ln, B, L, H, D = _dense_attention_inputs(q, k, v, lengths, "dense_flash_attention")
    if block_q < 1 or block_k < 1:
        raise JaggedError("dense_flash_attention: block sizes must be >= 1")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    out = torch.empty_like(q)
    lse = torch.empty(H, B * L, dtype=torch.float32, device=q.device)
    check(_lib.lib().jg_dense_flash_attention_forward(
        ln.ctypes.data, B, L, H, D, _p(q), _p(k), _p(v), block_q, block_k, _p(out), _p(lse), _dt(q), _stream()))
    return DenseAttentionSaved(out, lse, block_q, block_k)


def dense_flash_attention_backward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, grad_out: torch.Tensor,
                                   saved: DenseAttentionSaved, lengths, workspace: torch.Tensor | None = None):
    """Backward of the padded mode (no reference counterpart): returns (dq, dk, dv), zero past each length."""
    ln, B, L, H, D = _dense_attention_inputs(q, k, v, lengths, "dense_flash_attention_backward")
    if grad_out.shape != q.shape or saved.output.shape != q.shape or saved.logsumexp.numel() != B * L * H:
        raise JaggedError("dense_flash_attention_backward: saved state does not match inputs")
    q, k, v, grad_out = q.contiguous(), k.contiguous(), v.contiguous(), grad_out.contiguous()
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    check(_lib.lib().jg_dense_flash_attention_backward(
        ln.ctypes.data, B, L, H, D, _p(q), _p(k), _p(v), _p(grad_out), _p(saved.output), _p(saved.logsumexp),
        saved.block_q, saved.block_k, _p(dq), _p(dk), _p(dv), _dt(q), _p(workspace), _stream()))
    return dq, dk, dv


def jagged_attention(q: JaggedTensor, k: JaggedTensor, v: JaggedTensor) -> JaggedTensor:
    """Unfused baseline (attention.cpp:162-170): materializes H * sum Bi^2 scores."""
    _require_attention_inputs(q, k, v, "jagged_attention")
    H, D = _heads(q)
    ln = q.lengths()
    sum_sq = int((ln * ln).sum())
    sq = torch.empty(q.batch + 1, dtype=torch.int64, device=q.values.device)
    check(_lib.lib().jg_sq_offsets(_p(q.offsets), q.batch, _p(sq), _stream()))
    out = torch.empty_like(q.values)
    check(_lib.lib().jg_jagged_attention(_p(q.offsets), _p(sq), q.batch, q.total_rows, sum_sq, H, D, _p(q.values),
                                         _p(k.values), _p(v.values), _p(out), _dt(q.values), None, _stream()))
    return q.with_values(out)


# ------------------------------------------------------------------ layout + elementwise
def jagged_to_dense(x: JaggedTensor, max_len: int, pad_value: float = 0.0) -> torch.Tensor:
    if max_len < 0:
        raise JaggedError("jagged_to_dense: max_len must be >= 0")
    out = torch.empty(x.batch, max_len, x.dim, dtype=x.values.dtype, device=x.values.device)
    check(_lib.lib().jg_jagged_to_dense(_p(x.offsets), x.batch, x.dim, _p(x.values), max_len, float(pad_value),
                                        _p(out), _dt(x.values), _stream()))
    return out


def dense_to_jagged(d: torch.Tensor, lengths) -> JaggedTensor:
    if d.dim() != 3:
        raise JaggedError("dense_to_jagged: rank-3 input required")
    lengths = np.asarray(lengths, np.int64)
    B, L, D = d.shape
    if len(lengths) != B:
        raise JaggedError("dense_to_jagged: lengths size mismatch")
    over = np.nonzero(lengths > L)[0]
    if over.size:
        i = int(over[0])
        raise JaggedError(f"dense_to_jagged: sample {i} length {int(lengths[i])} exceeds max_len {L}")
    host = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    off = torch.from_numpy(host).to(d.device)
    out = torch.empty(int(host[-1]), D, dtype=d.dtype, device=d.device)
    check(_lib.lib().jg_dense_to_jagged(_p(d.contiguous()), B, L, D, _p(off), int(host[-1]),
                                        int(lengths.max(initial=0)), _p(out), _dt(d), _stream()))
    return JaggedTensor(off, out, host)


def jagged2_to_dense(s: Jagged2Tensor, max_len: int, pad_value: float = 0.0) -> torch.Tensor:
    out = torch.empty(s.batch, max_len, max_len, dtype=s.values.dtype, device=s.values.device)
    check(_lib.lib().jg_jagged2_to_dense(_p(s.offsets), _p(s.sq_offsets), s.batch, _p(s.values), max_len,
                                         float(pad_value), _p(out), _dt(s.values), _stream()))
    return out


def dense_to_jagged2(d: torch.Tensor, lengths) -> Jagged2Tensor:
    if d.dim() != 3 or d.shape[1] != d.shape[2]:
        raise JaggedError("dense_to_jagged2: [B, L, L] input required")
    lengths = np.asarray(lengths, np.int64)
    B, L, _ = d.shape
    if len(lengths) != B:
        raise JaggedError("dense_to_jagged2: lengths size mismatch")
    over = np.nonzero(lengths > L)[0]
    if over.size:
        i = int(over[0])
        raise JaggedError(f"dense_to_jagged2: sample {i} length {int(lengths[i])} exceeds max_len {L}")
    host = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    off = torch.from_numpy(host).to(d.device)
    sq = torch.empty(B + 1, dtype=torch.int64, device=d.device)
    check(_lib.lib().jg_sq_offsets(_p(off), B, _p(sq), _stream()))
    out = torch.empty(int((lengths * lengths).sum()), dtype=d.dtype, device=d.device)
    check(_lib.lib().jg_dense_to_jagged2(_p(d.contiguous()), B, L, _p(off), _p(sq), int(lengths.max(initial=0)),
                                         _p(out), _dt(d), _stream()))
    return Jagged2Tensor(off, out, host, sq)


def _zip(a: JaggedTensor, b: JaggedTensor, op: int, name: str) -> JaggedTensor:
    # tensor.cpp:179-202
    if a.dim != b.dim:
        raise JaggedError(f"{name}: dim mismatch ({a.dim} vs {b.dim})")
    _require_matching_offsets(a, b, name)
    out = torch.empty_like(a.values)
    check(_lib.lib().jg_elementwise(op, _p(a.values), _p(b.values), a.values.numel(), _p(out), _dt(a.values),
                                    _stream()))
    return a.with_values(out)


def add(a, b):
    return _zip(a, b, 0, "add")


def sub(a, b):
    return _zip(a, b, 1, "sub")


def mul(a, b):
    return _zip(a, b, 2, "mul")


def scale(a, s: float):
    vals = a.values
    out = torch.empty_like(vals)
    check(_lib.lib().jg_scale(_p(vals), vals.numel(), float(s), _p(out), _dt(vals), _stream()))
    if isinstance(a, Jagged2Tensor):
        return Jagged2Tensor(a.offsets, out, a.host_offsets, a.sq_offsets)
    return a.with_values(out)


# ---------------------------------------------------------------------------- SURVEY §8f "next" rows
def feature_interaction(k_feat: JaggedTensor, v_feat: JaggedTensor, targets: torch.Tensor) -> torch.Tensor:
    """attention.hpp:97 / attention.cpp:291-309: [B, Tq, D] targets attend over each sample's rows.

    out[i] = softmax over rows(K_i targets_i^T / sqrt(D))^T V_i; empty samples give zeros.
    """
    if not (k_feat.same_offsets(v_feat) and k_feat.dim == v_feat.dim):
        raise JaggedError("feature_interaction: k_feat/v_feat layout mismatch")
    _operands("feature_interaction", k_feat.values, v_feat.values)
    if not targets.is_cuda or targets.device != k_feat.values.device:
        raise JaggedError("feature_interaction: operands must be CUDA tensors on one device")
    if targets.dim() != 3 or targets.shape[0] != k_feat.batch or targets.shape[2] != k_feat.dim:
        raise JaggedError("feature_interaction: targets must be [B, Tq, D]")
    targets = targets.contiguous().to(k_feat.values.dtype)
    out = torch.zeros(k_feat.batch, targets.shape[1], k_feat.dim, dtype=k_feat.values.dtype,
                      device=k_feat.values.device)
    check(_lib.lib().jg_feature_interaction(_p(k_feat.offsets), k_feat.batch, k_feat.total_rows, k_feat.dim,
                                            targets.shape[1], _p(k_feat.values), _p(v_feat.values), _p(targets),
                                            _p(out), _dt(k_feat.values), None, _stream()))
    return out


RELU, NONE = "relu", "none"


@dataclass
class MlpLayer:
    """linalg.hpp:59-63: weights [D_in, D_out] shared across samples, bias [D_out], activation."""
    weights: torch.Tensor
    bias: torch.Tensor
    activation: str = NONE


@dataclass
class MlpLayerGrads:
    dweights: torch.Tensor
    dbias: torch.Tensor


@dataclass
class JaggedMlpGrads:
    dx: JaggedTensor
    dlayers: list


def _validate_mlp(x: JaggedTensor, layers) -> None:
    """linalg.cpp:224-243 (same messages)."""
    if not layers:
        raise JaggedError("jagged_mlp: at least one layer required")
    cur = x.dim
    for l, L in enumerate(layers):
        w = L.weights
        if w.dim() != 2:
            raise JaggedError(f"jagged_mlp: layer {l} weights must be rank 2")
        if w.shape[0] != cur:
            raise JaggedError(f"jagged_mlp: layer {l} input dim mismatch ({cur} vs {w.shape[0]})")
        if L.bias.numel() != w.shape[1]:
            raise JaggedError(f"jagged_mlp: layer {l} bias size {L.bias.numel()} != {w.shape[1]}")
        cur = w.shape[1]


def _mlp_forward(x: JaggedTensor, layers, keep: bool):
    for L in layers:
        if not (L.weights.is_cuda and L.bias.is_cuda) or L.weights.device != x.values.device:
            raise JaggedError("jagged_mlp: weights and bias must be CUDA tensors on the input's device")
    acts, pres = [x.values], []
    cur = x.values
    for L in layers:
        w = L.weights.contiguous().to(cur.dtype)
        b = L.bias.contiguous().to(cur.dtype)
        out = torch.empty(cur.shape[0], w.shape[1], dtype=cur.dtype, device=cur.device)
        pre = torch.empty_like(out) if keep else None
        check(_lib.lib().jg_mlp_layer_forward(cur.shape[0], w.shape[0], w.shape[1], _p(cur), _p(w), _p(b),
                                              1 if L.activation == RELU else 0, _p(out), _p(pre) if keep else None,
                                              _dt(cur), _stream()))
        cur = out
        acts.append(out)
        pres.append(pre)
    return acts, pres


def jagged_mlp(x: JaggedTensor, layers) -> JaggedTensor:
    """linalg.cpp:265-277: row-wise affine + activation chain (shared weights, no padding rows)."""
    _validate_mlp(x, layers)
    acts, _ = _mlp_forward(x, layers, keep=False)
    return x.with_values(acts[-1])


def jagged_mlp_vjp(x: JaggedTensor, layers, grad_out: JaggedTensor) -> JaggedMlpGrads:
    """linalg.cpp:509-573: recomputes the forward, then per layer (last first) mask, db, dW, dx."""
    _validate_mlp(x, layers)
    _require_matching_offsets(x, grad_out, "jagged_mlp_vjp")
    acts, pres = _mlp_forward(x, layers, keep=True)
    delta = grad_out.values.contiguous().to(x.values.dtype)
    dl = [None] * len(layers)
    for l in range(len(layers) - 1, -1, -1):
        L = layers[l]
        w = L.weights.contiguous().to(x.values.dtype)
        dw = torch.empty_like(w)
        db = torch.empty(w.shape[1], dtype=w.dtype, device=w.device)
        dx = torch.empty(delta.shape[0], w.shape[0], dtype=delta.dtype, device=delta.device)
        check(_lib.lib().jg_mlp_layer_backward(delta.shape[0], w.shape[0], w.shape[1], _p(acts[l]), _p(w),
                                               _p(pres[l]), 1 if L.activation == RELU else 0, _p(delta), _p(dw),
                                               _p(db), _p(dx), _dt(delta), _stream()))
        dl[l] = MlpLayerGrads(dw, db)
        delta = dx
    return JaggedMlpGrads(x.with_values(delta), dl)
