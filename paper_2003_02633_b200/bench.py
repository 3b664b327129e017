"""``vc3.bench``: the vector-op entry points and the working-set sweep of
/root/reference/pkg/src/vc3/bench.py, with the GPU kernels doing the work.

The reference times its single-threaded numba loops with perf_counter over
host arrays and reports the last-level-cache knee (bench.py:72-192).  Here
each point times the device kernels (``vc3_add_raw``, ``vc3_add_compressed``)
on HBM-resident inputs with CUDA events on the launching stream, median of
``repeats`` after one warm-up, so the rows keep the reference schema
(``n, time_raw_ns, time_comp_ns, speedup, bytes_ratio``) and add Gvec/s and
GB/s.  ``llc_bytes`` is the device L2 (the last cache level the kernels
see), so ``knee_elements`` marks where the raw working set leaves L2.  The
driver-contract harness of the repository is /root/repo/bench.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev
from ._dev import torch
from .errors import LengthMismatch  # noqa: F401  (the reference's bench namespace)
from .layout import ALL_SINGLE_POLICY, DEFAULT_LAYOUT, BitLayout, PrecisionPolicy, as_layout, as_policy
from .ops import (  # noqa: F401
    COMPRESSED_BYTES_PER_ELEMENT,
    RAW_BYTES_PER_ELEMENT,
    add_compressed,
    add_raw,
    axpy,
    rk_stage,
)


@dataclass(frozen=True)
class BenchConfig:
    """Sweep definition (bench.py:72-85)."""

    working_set_sweep: tuple[int, ...] = (1 << 14, 1 << 17, 1 << 20, 1 << 23)
    repeats: int = 5
    layout: BitLayout = DEFAULT_LAYOUT
    policy: PrecisionPolicy = ALL_SINGLE_POLICY
    seed: int = 0

    def __post_init__(self):
        if len(self.working_set_sweep) == 0 or min(self.working_set_sweep) < 1:
            raise ValueError("working_set_sweep needs positive element counts")
        if self.repeats < 3:
            raise ValueError("repeats must be >= 3 (median-of-repeats)")


@dataclass
class BenchResult:
    """One sweep point (bench.py:88-99) plus device throughput."""

    n: int
    bytes_moved_raw: int
    bytes_moved_compressed: int
    time_raw_ns: float
    time_compressed_ns: float
    speedup: float
    bytes_ratio: float
    gvec_s_raw: float = 0.0
    gvec_s_compressed: float = 0.0
    gbs_raw: float = 0.0
    gbs_compressed: float = 0.0

    def to_dict(self) -> dict:
        return self.__dict__.copy()


from .analysis import SampleDomain  # noqa: E402,F401  (the reference's bench namespace)


def llc_bytes() -> int | None:
    """L2 size of the current CUDA device, or None without one."""
    if torch is None or not torch.cuda.is_available():
        return None
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    return int(getattr(props, "L2_cache_size", 0)) or None


def _median_time_ns(fn, repeats: int) -> float:
    stream = torch.cuda.current_stream()
    fn()  # warm-up, excluded
    times = []
    for _ in range(repeats):
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        start.record(stream)
        fn()
        stop.record(stream)
        stop.synchronize()
        times.append(start.elapsed_time(stop) * 1e6)
    return float(np.median(times))


def _vectors(n: int, seed: int, stream: int):
    """The reference's cube sample for operand ``stream`` (bench.py:149-155),
    drawn chunk by chunk and uploaded."""
    dom = SampleDomain("cube", n, (seed << 1) | stream)
    out = torch.empty((n, 3), dtype=torch.float32, device=torch.device("cuda", torch.cuda.current_device()))
    pos = 0
    for chunk in dom.chunks():
        out[pos:pos + chunk.shape[0]] = torch.from_numpy(chunk).to(out.device)
        pos += chunk.shape[0]
    return out


def _measure_one(n: int, config: BenchConfig) -> BenchResult:
    from .codec import compress

    layout, policy = as_layout(config.layout), as_policy(config.policy)
    va, vb = _vectors(n, config.seed, 0), _vectors(n, config.seed, 1)
    t_raw = _median_time_ns(lambda: add_raw(va, vb), config.repeats)
    ca, cb = compress(va, layout, policy), compress(vb, layout, policy)
    del va, vb
    t_comp = _median_time_ns(lambda: add_compressed(ca, cb, layout, policy), config.repeats)
    braw, bcomp = RAW_BYTES_PER_ELEMENT * n, COMPRESSED_BYTES_PER_ELEMENT * n
    return BenchResult(
        n=n, bytes_moved_raw=braw, bytes_moved_compressed=bcomp,
        time_raw_ns=t_raw, time_compressed_ns=t_comp, speedup=t_raw / t_comp,
        bytes_ratio=RAW_BYTES_PER_ELEMENT / COMPRESSED_BYTES_PER_ELEMENT,
        gvec_s_raw=n / t_raw, gvec_s_compressed=n / t_comp,
        gbs_raw=braw / t_raw, gbs_compressed=bcomp / t_comp)


def sweep(config: BenchConfig) -> list[BenchResult]:
    """Time raw and compressed adds across the working-set sweep (bench.py:166-168)."""
    _dev.require_torch_cuda()
    return [_measure_one(int(n), config) for n in config.working_set_sweep]


def knee_elements(results: list[BenchResult]) -> int | None:
    """Largest sweep size whose raw working set fits the L2 (bench.py:171-178)."""
    cache = llc_bytes()
    if cache is None:
        return None
    fitting = [r.n for r in results if r.bytes_moved_raw <= cache]
    return max(fitting) if fitting else None
