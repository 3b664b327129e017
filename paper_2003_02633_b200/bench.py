"""``vc3.bench`` compatibility module: the vector-op entry points the
reference exposes from /root/reference/pkg/src/vc3/bench.py:26-69.  The
timing harness of the repository is /root/repo/bench.py."""

from .ops import (  # noqa: F401
    COMPRESSED_BYTES_PER_ELEMENT,
    RAW_BYTES_PER_ELEMENT,
    add_compressed,
    add_raw,
    axpy,
    rk_stage,
)
