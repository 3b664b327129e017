"""Input domains and round-trip error statistics on the GPU path.

* ``SampleDomain`` / ``sample`` restate the reference's deterministic
  generator (/root/reference/pkg/src/vc3/analysis.py:34-99): chunk ``i`` of
  ``CHUNK`` vectors is drawn from numpy ``Philox(key=(seed, i))``, so every
  input the reference studies can be reproduced bit for bit here.
* ``error_study`` (analysis.py:157-167) runs compress -> decompress -> the
  K6 per-chunk moment kernel on the device and merges chunk moments on the
  host in chunk order with the reference's merge formula (analysis.py:118-145).
* ``error_study_sharded`` splits the chunks over the ranks of a
  ``torch.distributed`` group (contiguous blocks of chunks, no data-path
  collective) and all-gathers the 32-byte per-chunk tuples; the merge in
  global chunk order makes the result identical on every rank and identical
  to the single-process result.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from ._dev import torch
from .codec import compress, decompress
from .errors import DomainError, EmptyDomain, InvalidSplit  # noqa: F401
from .layout import (  # noqa: F401  (the reference's analysis namespace)
    ALL_SINGLE_POLICY,
    DEFAULT_LAYOUT,
    DEFAULT_POLICY,
    ORACLE_POLICY,
    BitLayout,
    PrecisionPolicy,
    as_layout,
    as_policy,
)

CHUNK = 1 << 20   # analysis.py:29

_KINDS = ("unit_sphere", "sphere_angles", "cube", "shell")


@dataclass(frozen=True)
class SampleDomain:
    """Region, count and seed of a deterministic float32 sample stream."""

    kind: str = "unit_sphere"
    count: int = 1_000_000
    seed: int = 0
    r_min: float = 1.0
    r_max: float = 1.0

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown domain kind {self.kind!r}")
        if self.count < 0:
            raise ValueError("count must be non-negative")
        if self.kind == "shell" and not 0 <= self.r_min <= self.r_max:
            raise ValueError("shell needs 0 <= r_min <= r_max")

    def describe(self) -> str:
        return f"shell:{self.r_min:g}:{self.r_max:g}" if self.kind == "shell" else self.kind

    def chunk(self, index: int, n: int) -> np.ndarray:
        """Chunk ``index`` (``n`` vectors); draws in the reference's order."""
        rng = np.random.Generator(np.random.Philox(key=(self.seed, index)))
        if self.kind == "cube":
            return rng.uniform(-1.0, 1.0, (n, 3)).astype(np.float32)
        if self.kind == "sphere_angles":
            theta = rng.uniform(-np.pi, np.pi, n)
            phi = rng.uniform(0.0, np.pi, n)
            sin_phi = np.sin(phi)
            out = np.stack([sin_phi * np.cos(theta), sin_phi * np.sin(theta), np.cos(phi)], axis=1)
            return out.astype(np.float32)
        theta = rng.uniform(-np.pi, np.pi, n)
        z = rng.uniform(-1.0, 1.0, n)
        ring = np.sqrt(1.0 - z * z)
        out = np.stack([ring * np.cos(theta), ring * np.sin(theta), z], axis=1)
        if self.kind == "shell":
            out = out * rng.uniform(self.r_min, self.r_max, n)[:, None]
        return out.astype(np.float32)

    def n_chunks(self) -> int:
        return (self.count + CHUNK - 1) // CHUNK

    def chunk_size(self, index: int) -> int:
        return min(CHUNK, self.count - index * CHUNK)

    def chunks(self):
        for i in range(self.n_chunks()):
            yield self.chunk(i, self.chunk_size(i))


def sample(domain: SampleDomain) -> np.ndarray:
    """Whole (count, 3) float32 sample (analysis.py:93-97)."""
    if domain.count == 0:
        return np.empty((0, 3), dtype=np.float32)
    return np.concatenate(list(domain.chunks()), axis=0)


@dataclass
class ErrorStats:
    mean: float
    max: float
    stddev: float
    count: int
    normalised: bool

    def to_dict(self) -> dict:
        return {"mean": self.mean, "max": self.max, "stddev": self.stddev,
                "count": self.count, "normalised": self.normalised}


class ChunkMerger:
    """Merge per-chunk (count, mean, M2, max) in chunk order with the
    reference's update rule (analysis.py:127-141)."""

    def __init__(self):
        self.n = 0
        self.mean = 0.0
        self.m2 = 0.0
        self.max = 0.0

    def add(self, count: int, mean: float, m2: float, mx: float):
        if count == 0:
            return
        if self.n == 0:
            self.n, self.mean, self.m2 = count, mean, m2
        else:
            n = self.n + count
            d = mean - self.mean
            self.mean += d * count / n
            self.m2 += m2 + d * d * self.n * count / n
            self.n = n
        self.max = max(self.max, mx)

    def stats(self, normalised: bool) -> ErrorStats:
        sd = math.sqrt(self.m2 / (self.n - 1)) if self.n > 1 else 0.0
        return ErrorStats(self.mean, self.max, sd, self.n, normalised)


# error metrics of the K6 kernel (include/vc3_b200.h VC3_ERR_*): "l2" is the
# reference's (analysis.py:148-154); "angular" (radians) and
# "relative_magnitude" are the harness metrics of SURVEY §8a R19
METRICS = {"l2": 0, "angular": 2, "relative_magnitude": 3}


def _kind(normalised: bool, metric: str) -> int:
    if metric not in METRICS:
        raise ValueError(f"unknown error metric {metric!r}; expected one of {sorted(METRICS)}")
    return 1 if (metric == "l2" and normalised) else METRICS[metric]


def chunk_moments(v, vh, normalised: bool, chunk: int = CHUNK, metric: str = "l2"):
    """Device K6 kernel: (k, 4) float64 tensor of per-chunk (count, mean, M2,
    max) of the per-vector error for CUDA tensors v, vh of shape (n, 3):
    ||v - vh||_2 (optionally / ||v||), or the angle between v and vh, or the
    relative magnitude error (``metric``)."""
    lib = _native.load()
    n = v.shape[0]
    k = max(1, (n + chunk - 1) // chunk)
    out = torch.zeros((k, 4), dtype=torch.float64, device=v.device)
    _native.check(lib.vc3_error_stats(v.data_ptr(), vh.data_ptr(), n, _kind(normalised, metric),
                                      chunk, out.data_ptr(), _dev.stream_of(v)), "error_stats")
    return out


def _chunk_tuple(domain: SampleDomain, index: int, layout, policy, normalised: bool,
                 metric: str = "l2") -> np.ndarray:
    v = _dev.upload(domain.chunk(index, domain.chunk_size(index)))
    vh = decompress(compress(v, layout, policy), layout)
    return chunk_moments(v, vh, normalised, CHUNK, metric)[0].cpu().numpy()


def error_study(domain: SampleDomain, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY,
                normalised: bool = False, metric: str = "l2") -> ErrorStats:
    """Round-trip error statistics over a sample domain (analysis.py:157-167).
    ``metric`` "l2" (the reference's) or the harness metrics "angular" /
    "relative_magnitude"."""
    if domain.count == 0:
        raise EmptyDomain("error_study needs at least one sample")
    layout, policy = as_layout(layout), as_policy(policy)
    _kind(normalised, metric)
    acc = ChunkMerger()
    for i in range(domain.n_chunks()):
        c = _chunk_tuple(domain, i, layout, policy, normalised, metric)
        acc.add(int(c[0]), float(c[1]), float(c[2]), float(c[3]))
    return acc.stats(normalised)


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of ``n_items`` owned by ``rank`` (ceil split)."""
    per = (n_items + world - 1) // world
    lo = min(n_items, rank * per)
    return lo, min(n_items, lo + per)


def error_study_sharded(domain: SampleDomain, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY,
                        normalised: bool = False, group=None,
                        tuple_fn=None, metric: str = "l2") -> ErrorStats:
    """``error_study`` with chunks split over a torch.distributed group.

    The only exchange is an all-gather of the (count, mean, M2, max) tuples
    (32 B per chunk); NCCL when the group's backend is nccl, gloo on CPU.
    ``tuple_fn(domain, index)`` overrides the per-chunk computation (tests use
    it to exercise the host logic without a GPU)."""
    import torch.distributed as dist

    if domain.count == 0:
        raise EmptyDomain("error_study needs at least one sample")
    layout, policy = as_layout(layout), as_policy(policy)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    nch = domain.n_chunks()
    per = (nch + world - 1) // world
    lo, hi = shard_range(nch, rank, world)
    fn = tuple_fn or (lambda d, i: _chunk_tuple(d, i, layout, policy, normalised, metric))
    mine = np.zeros((per, 4), dtype=np.float64)
    for j, i in enumerate(range(lo, hi)):
        mine[j] = fn(domain, i)
    backend = dist.get_backend(group)
    dev = (torch.device("cuda", torch.cuda.current_device()) if backend == "nccl"
           else torch.device("cpu"))
    local = torch.from_numpy(mine).to(dev)
    gathered = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(gathered, local, group=group)
    table = torch.cat(gathered).cpu().numpy()[:nch]
    acc = ChunkMerger()
    for row in table:
        acc.add(int(row[0]), float(row[1]), float(row[2]), float(row[3]))
    return acc.stats(normalised)


# K7 variants (analysis.py:259-417) live in variants.py; re-exported here so
# ``analysis.Compander`` etc. resolve as in the reference.
from .variants import (  # noqa: E402,F401
    Compander,
    SplitConfig,
    _quantize_free,
    compand,
    compand_inverse,
    compand_study,
    joint_decode,
    joint_encode,
    split_sweep,
)


# ---------------------------------------------------------------------------
# characterisation studies on the device path
# ---------------------------------------------------------------------------
def _angle_bits(words, layout):
    w = words.view(torch.int64)
    nt = w & layout.n_theta_max
    nph = (w >> layout.theta_bits) & layout.n_phi_max
    return nt, nph


def bin_miss_study(domain: SampleDomain, layout=DEFAULT_LAYOUT) -> tuple[float, float]:
    """Fraction of samples whose theta / phi bucket differs between the
    all-single and all-double pipelines (analysis.py:236-254).  Both bucket
    sets come from the compress kernel (its angle bits are exactly
    quantize_angles(to_spherical(v)) for every nonzero vector; zero vectors
    give equal buckets in both pipelines, as in the reference)."""
    from .layout import ALL_SINGLE_POLICY, ORACLE_POLICY

    if domain.count == 0:
        raise EmptyDomain("bin_miss_study needs at least one sample")
    layout = as_layout(layout)
    miss_t = miss_p = 0
    for i in range(domain.n_chunks()):
        v = _dev.upload(domain.chunk(i, domain.chunk_size(i)))
        ts, ps = _angle_bits(compress(v, layout, ALL_SINGLE_POLICY), layout)
        td, pd = _angle_bits(compress(v, layout, ORACLE_POLICY), layout)
        miss_t += int((ts != td).sum().item())
        miss_p += int((ps != pd).sum().item())
    return miss_t / domain.count, miss_p / domain.count


@dataclass
class IdempotenceResult:
    word_miss_fraction: float
    predicted_bound: float
    third_cycle_stable_fraction: float
    count: int

    def to_dict(self) -> dict:
        return {"word_miss_fraction": self.word_miss_fraction,
                "predicted_bound": self.predicted_bound,
                "third_cycle_stable_fraction": self.third_cycle_stable_fraction,
                "count": self.count}


def idempotence_study(domain: SampleDomain, layout=DEFAULT_LAYOUT, policy=DEFAULT_POLICY,
                      u: int = 8) -> IdempotenceResult:
    """Word stability under repeated compress/decompress cycles
    (analysis.py:446-486): miss = compress(decompress(w1)) != w1."""
    if domain.count == 0:
        raise EmptyDomain("idempotence_study needs at least one sample")
    layout, policy = as_layout(layout), as_policy(policy)
    misses = stable3 = 0
    for i in range(domain.n_chunks()):
        v = _dev.upload(domain.chunk(i, domain.chunk_size(i)))
        w1 = compress(v, layout, policy)
        w2 = compress(decompress(w1, layout), layout, policy)
        w3 = compress(decompress(w2, layout), layout, policy)
        misses += int((w1.view(torch.int64) != w2.view(torch.int64)).sum().item())
        stable3 += int((w2.view(torch.int64) == w3.view(torch.int64)).sum().item())
    m_int = 24 if (policy.theta_single or policy.phi_single) else 53
    p_eff = max(layout.phi_bits, layout.theta_bits)
    bound = 2.0 * u * 2.0 ** (p_eff - m_int)
    return IdempotenceResult(misses / domain.count, bound, stable3 / domain.count, domain.count)


def precision_comparison(count: int, seed: int, layout=DEFAULT_LAYOUT) -> list[dict]:
    """Normalised error statistics for the four theta/phi single/double
    policies (quantisation single) on the unit sphere and the cube
    (analysis.py:170-191); each row is one device ``error_study``."""
    from .layout import PrecisionPolicy

    rows = []
    for kind in ("unit_sphere", "cube"):
        domain = SampleDomain(kind, count, seed)
        for theta in ("single", "double"):
            for phi in ("single", "double"):
                st = error_study(domain, layout, PrecisionPolicy(theta, phi, "single"),
                                 normalised=True)
                rows.append({"domain": kind, "theta": theta, "phi": phi, **st.to_dict()})
    return rows


def anisotropy_map(layout=DEFAULT_LAYOUT, policy=None, grid: tuple[int, int] = (32, 16),
                   count: int = 1_000_000, seed: int = 0):
    """Mean round-trip error per (theta, phi) cell of the unit sphere
    (analysis.py:194-223): (means, counts, theta_edges, phi_edges), NaN in
    empty cells.  Round trip, errors and cell binning all run on the device
    (float64 atan2/acos for the cell of the *input* vector, as the
    reference); cell sums accumulate with index_add in float64."""
    from .layout import ORACLE_POLICY

    tc, pc = grid
    if tc < 1 or pc < 1:
        raise ValueError("grid cells must be >= 1")
    layout = as_layout(layout)
    policy = as_policy(ORACLE_POLICY if policy is None else policy)
    domain = SampleDomain("unit_sphere", count, seed)
    _dev.require_torch_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    sums = torch.zeros(tc * pc, dtype=torch.float64, device=dev)
    counts = torch.zeros(tc * pc, dtype=torch.int64, device=dev)
    for i in range(domain.n_chunks()):
        v = _dev.upload(domain.chunk(i, domain.chunk_size(i)))
        vh = decompress(compress(v, layout, policy), layout)
        v64 = v.to(torch.float64)
        d = v64 - vh.to(torch.float64)
        e = torch.sqrt((d * d).sum(dim=1))
        x, y, z = v64.unbind(1)
        r = torch.sqrt(x * x + y * y + z * z)
        th = torch.atan2(y, x)
        ph = torch.acos(torch.clamp(z / torch.where(r > 0, r, torch.ones_like(r)), -1.0, 1.0))
        ti = torch.clamp(((th + math.pi) / (2 * math.pi) * tc).to(torch.int64), 0, tc - 1)
        pj = torch.clamp((ph / math.pi * pc).to(torch.int64), 0, pc - 1)
        cell = ti * pc + pj
        sums.index_add_(0, cell, e)
        counts.index_add_(0, cell, torch.ones_like(cell))
    sums = sums.reshape(tc, pc).cpu().numpy()
    counts = counts.reshape(tc, pc).cpu().numpy()
    means = np.where(counts > 0, sums / np.maximum(counts, 1), np.nan)
    return (means, counts, np.linspace(-np.pi, np.pi, tc + 1), np.linspace(0.0, np.pi, pc + 1))


def anisotropy_rows(means: np.ndarray) -> list[tuple[int, int, float]]:
    """(theta_cell, phi_cell, mean) for every non-empty cell (analysis.py:226-233)."""
    return [(i, j, float(means[i, j])) for i in range(means.shape[0])
            for j in range(means.shape[1]) if not np.isnan(means[i, j])]


def smith_theta_bins(phi: float, n_phi_max: int, tau: float) -> int:
    """Azimuth bins on the ring at ``phi`` that keep the chordal error within
    ``tau`` (the variable-bin comparison rule of analysis.py:420-443; host
    scalar arithmetic, no fixed-rate code uses it)."""
    from .errors import DomainError

    if not 0.0 < phi < math.pi:
        raise DomainError("phi must lie strictly inside (0, pi)")
    if tau <= 0:
        raise DomainError("tau must be positive")
    half_ring = math.pi / (2.0 * n_phi_max)
    c = (math.cos(tau) - math.cos(phi) * math.cos(phi + half_ring)) / (
        math.sin(phi) * math.sin(phi + half_ring))
    if not -1.0 <= c <= 1.0:
        raise DomainError(f"arccos argument {c} outside [-1, 1]")
    width = math.acos(c)
    if width == 0.0:
        raise DomainError("tolerance exactly at the ring spacing limit")
    return int(math.ceil(math.pi / width))


def report(domain: SampleDomain, layout, policy, **extra) -> dict:
    """The studies' machine-readable envelope (analysis.py:489-500)."""
    doc = {"layout": str(as_layout(layout)), "policy": as_policy(policy).spec(),
           "domain": domain.describe(), "seed": domain.seed, "count": domain.count}
    doc.update(extra)
    return doc
