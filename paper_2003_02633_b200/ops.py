"""Fused streaming vector operations on compressed words.

``add_raw`` / ``add_compressed`` keep the signatures of
/root/reference/pkg/src/vc3/bench.py:30-51 (exported there from ``vc3.bench``;
``paper_2003_02633_b200.bench`` re-exports them).  ``axpy`` and ``rk_stage``
have no reference symbol: they are the paper's motivating
use (low-storage Runge-Kutta updates on compressed registers, PAPER.md:135,
336), defined by their composition with the reference codec:

    axpy(alpha, x, y)        == compress(alpha*decompress(x) + decompress(y))
    rk_stage(a, b, dt, q, dq, R):  dq' = a*dq + dt*R ; q' = q + b*dq'

with float32 arithmetic, each product and sum rounded, in that order.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native
from ._dev import torch
from .errors import LengthMismatch
from .layout import ALL_SINGLE_POLICY, DEFAULT_LAYOUT, as_layout, as_policy

RAW_BYTES_PER_ELEMENT = 36          # bench.py:26
COMPRESSED_BYTES_PER_ELEMENT = 24   # bench.py:27


def _words_dev(x):
    return x.reshape(-1).contiguous()


def add_raw(a, b):
    """Elementwise float32 sum of two (n, 3) vector streams (bench.py:30-38)."""
    lib = _native.load()
    if _dev.is_device(a):
        ta = a.to(torch.float32).contiguous()
        tb = b.to(device=a.device, dtype=torch.float32).contiguous()
        if ta.shape != tb.shape:
            raise LengthMismatch(f"shapes differ: {tuple(ta.shape)} vs {tuple(tb.shape)}")
        c = torch.empty_like(ta)
        _native.check(lib.vc3_add_raw(ta.data_ptr(), tb.data_ptr(), c.data_ptr(), ta.numel(),
                                      _dev.stream_of(ta)), "add_raw")
        return c
    ha = np.ascontiguousarray(a, dtype=np.float32)
    hb = np.ascontiguousarray(b, dtype=np.float32)
    if ha.shape != hb.shape:
        raise LengthMismatch(f"shapes differ: {ha.shape} vs {hb.shape}")
    if ha.size == 0:
        return np.empty_like(ha)
    return _dev.download(add_raw(_dev.upload(ha), _dev.upload(hb)))


def add_compressed(a, b, layout=DEFAULT_LAYOUT, policy=ALL_SINGLE_POLICY, mode="exact"):
    """compress(decompress(a) + decompress(b)) in one fused kernel
    (bench.py:41-69, _kernels.py:348-359).  Default policy all-single, as
    the reference's benchmark path.  ``mode="contract"`` selects the
    north-star tolerance (VC3_CONTRACT: a decoded component may be one ulp
    off, a word may move one bin at a tie)."""
    layout, policy = as_layout(layout), as_policy(policy)
    flags = _native.mode_flag(mode)
    lib = _native.load()
    if _dev.is_device(a):
        ta, tb = _words_dev(a), _words_dev(b.to(a.device))
        if ta.shape != tb.shape:
            raise LengthMismatch(f"lengths differ: {ta.numel()} vs {tb.numel()}")
        c = torch.empty_like(ta)
        with _dev.on_device(ta):
            _native.check(lib.vc3_add_compressed_ex(ta.data_ptr(), tb.data_ptr(), c.data_ptr(),
                                                    ta.numel(), _native.c_layout(layout),
                                                    policy.mask, flags, _dev.stream_of(ta)),
                          "add_compressed")
        return c.reshape(a.shape)
    ha = np.ascontiguousarray(a, dtype=np.uint64)
    hb = np.ascontiguousarray(b, dtype=np.uint64)
    if ha.shape != hb.shape:
        raise LengthMismatch(f"lengths differ: {ha.size} vs {hb.size}")
    if flags:
        return _dev.download(add_compressed(_dev.upload(ha), _dev.upload(hb), layout, policy, mode))
    c = np.empty_like(ha)
    _native.check(lib.vc3_add_compressed_host(ha.ctypes.data, hb.ctypes.data, c.ctypes.data,
                                              ha.size, _native.c_layout(layout), policy.mask,
                                              _dev.device_ordinal()), "add_compressed")
    return c


def axpy(alpha, x, y, layout=DEFAULT_LAYOUT, policy=ALL_SINGLE_POLICY, out=None, mode="exact"):
    """compress(alpha*decompress(x) + decompress(y)); ``out=y`` updates in place."""
    layout, policy = as_layout(layout), as_policy(policy)
    flags = _native.mode_flag(mode)
    lib = _native.load()
    host = not _dev.is_device(x)
    tx = _dev.upload(np.asarray(x, dtype=np.uint64)) if host else _words_dev(x)
    ty = _dev.upload(np.asarray(y, dtype=np.uint64)) if host else _words_dev(y)
    if tx.shape != ty.shape:
        raise LengthMismatch(f"lengths differ: {tx.numel()} vs {ty.numel()}")
    to = (torch.empty_like(ty) if (out is None or host) else _words_dev(out))
    with _dev.on_device(tx):
        _native.check(lib.vc3_axpy_ex(float(np.float32(alpha)), tx.data_ptr(), ty.data_ptr(),
                                      to.data_ptr(), tx.numel(), _native.c_layout(layout),
                                      policy.mask, flags, _dev.stream_of(tx)), "axpy")
    if host:
        res = _dev.download(to)
        if out is not None:
            out[...] = res
            return out
        return res
    return to


def rk_stage(a, b, dt, q, dq, R, layout=DEFAULT_LAYOUT, policy=ALL_SINGLE_POLICY, mode="exact"):
    """One low-storage RK stage on compressed q, dq and residual R, in place:
    dq <- a*dq + dt*R ; q <- q + b*dq.  Returns (q, dq)."""
    layout, policy = as_layout(layout), as_policy(policy)
    flags = _native.mode_flag(mode)
    lib = _native.load()
    host = not _dev.is_device(q)
    tq = _dev.upload(np.asarray(q, dtype=np.uint64)) if host else q
    tdq = _dev.upload(np.asarray(dq, dtype=np.uint64)) if host else dq
    tR = _dev.upload(np.asarray(R, dtype=np.uint64)) if host else _words_dev(R)
    if not (tq.numel() == tdq.numel() == tR.numel()):
        raise LengthMismatch("q, dq and R must have the same length")
    if not host and not (tq.is_contiguous() and tdq.is_contiguous()):
        raise ValueError("rk_stage updates q and dq in place: pass contiguous tensors")
    with _dev.on_device(tq):
        _native.check(lib.vc3_rk_stage_ex(float(np.float32(a)), float(np.float32(b)),
                                          float(np.float32(dt)), tq.data_ptr(), tdq.data_ptr(),
                                          tR.data_ptr(), tq.numel(), _native.c_layout(layout),
                                          policy.mask, flags, _dev.stream_of(tq)), "rk_stage")
    if host:
        q[...] = _dev.download(tq)
        dq[...] = _dev.download(tdq)
    return q, dq


def rk_stage_f32(a, b, dt, q, dq, R):
    """Uncompressed float32 RK stage on CUDA tensors (the baseline of
    ``rk_stage``): dq <- a*dq + dt*R ; q <- q + b*dq, in place."""
    lib = _native.load()
    if not (_dev.is_device(q) and q.is_contiguous() and dq.is_contiguous()):
        raise ValueError("rk_stage_f32 takes contiguous CUDA float32 tensors")
    if not (q.numel() == dq.numel() == R.numel()):
        raise LengthMismatch("q, dq and R must have the same length")
    Rc = R.contiguous()
    _native.check(lib.vc3_rk_stage_f32(float(np.float32(a)), float(np.float32(b)),
                                       float(np.float32(dt)), q.data_ptr(), dq.data_ptr(),
                                       Rc.data_ptr(), q.numel(), _dev.stream_of(q)),
                  "rk_stage_f32")
    return q, dq


class LSRKStep:
    """One full low-storage RK4(5) step (five ``rk_stage`` launches, the
    Carpenter-Kennedy coefficients of fields.LSRK_A/B) on compressed CUDA
    words, captured once into a CUDA graph and replayed: for small meshes
    (the paper's 10^5-point vortex) the five launches cost more host time
    than GPU time, and a graph replay removes that.

    ``q``, ``dq`` (updated in place) and ``R`` are contiguous CUDA uint64
    tensors that stay bound to the graph; refresh ``R`` in place between
    steps.  ``step()`` is bit-identical to calling ``rk_stage`` five times.
    """

    def __init__(self, q, dq, R, dt: float, layout=DEFAULT_LAYOUT, policy=ALL_SINGLE_POLICY,
                 mode="exact"):
        from .fields import LSRK_A, LSRK_B

        _dev.require_torch_cuda()
        if not all(_dev.is_device(t) and t.is_contiguous() for t in (q, dq, R)):
            raise ValueError("LSRKStep takes contiguous CUDA uint64 tensors")
        if not (q.numel() == dq.numel() == R.numel()):
            raise LengthMismatch("q, dq and R must have the same length")
        self.q, self.dq, self.R = q, dq, R
        self.layout, self.policy = as_layout(layout), as_policy(policy)
        self._lib = _native.load()
        self._cl = _native.c_layout(self.layout)
        self._coef = [(float(np.float32(a)), float(np.float32(b))) for a, b in zip(LSRK_A, LSRK_B)]
        self._dt = float(np.float32(dt))
        self._flags = _native.mode_flag(mode)
        self.graph = None

    def _launch_all(self, stream_ptr):
        for a, b in self._coef:
            _native.check(self._lib.vc3_rk_stage_ex(a, b, self._dt, self.q.data_ptr(),
                                                    self.dq.data_ptr(), self.R.data_ptr(),
                                                    self.q.numel(), self._cl, self.policy.mask,
                                                    self._flags, stream_ptr), "rk_stage")

    def capture(self):
        """Record the five stages (no work is done by the capture itself)."""
        s = torch.cuda.Stream(device=self.q.device)
        s.wait_stream(torch.cuda.current_stream(self.q.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            # warm up on one-word scratch copies: the layout's decode table and
            # the kernel's shared-memory attribute are set up outside the capture
            sq, sdq, sR = self.q[:1].clone(), self.dq[:1].clone(), self.R[:1].clone()
            _native.check(self._lib.vc3_rk_stage_ex(1.0, 1.0, 0.0, sq.data_ptr(), sdq.data_ptr(),
                                                    sR.data_ptr(), 1, self._cl, self.policy.mask,
                                                    self._flags, s.cuda_stream), "rk_stage")
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                self._launch_all(s.cuda_stream)
        torch.cuda.current_stream(self.q.device).wait_stream(s)
        self.graph = g
        return self

    def step(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()
        return self.q, self.dq

    def step_eager(self):
        self._launch_all(_dev.stream_of(self.q))
        return self.q, self.dq
