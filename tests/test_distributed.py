"""Multi-rank host logic on CPU (gloo, world_size 2): contiguous sharding and
the chunk-ordered all-gather merge of error statistics.  The
per-chunk tuples come from the C oracle here (no GPU); on a B200 box the same
code path gathers the device K6 tuples over NCCL."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_tuple(domain, index):
    sys.path.insert(0, str(ROOT / "oracle"))
    import vc3_oracle

    from paper_2003_02633_b200.layout import DEFAULT_LAYOUT, DEFAULT_POLICY

    v = domain.chunk(index, domain.chunk_size(index))
    vh = vc3_oracle.decompress(vc3_oracle.compress(v, DEFAULT_LAYOUT, DEFAULT_POLICY),
                               DEFAULT_LAYOUT)
    d = v.astype(np.float64) - vh.astype(np.float64)
    e = np.sqrt((d * d).sum(axis=1))
    m = e.mean()
    return np.array([e.size, m, ((e - m) ** 2).sum(), e.max()])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_2003_02633_b200.analysis import SampleDomain, error_study_sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dom = SampleDomain("unit_sphere", 3 * (1 << 20) + 12345, 21)  # 4 chunks, ragged tail
        st = error_study_sharded(dom, tuple_fn=_oracle_tuple)
        out[rank] = (st.mean, st.max, st.stddev, st.count)
    finally:
        dist.destroy_process_group()


def test_sharded_error_study_matches_serial_merge():
    from paper_2003_02633_b200.analysis import ChunkMerger, SampleDomain

    world = 2
    manager = mp.get_context("spawn").Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world,
                       start_method="spawn", join=True)
    dom = SampleDomain("unit_sphere", 3 * (1 << 20) + 12345, 21)
    acc = ChunkMerger()
    for i in range(dom.n_chunks()):
        c = _oracle_tuple(dom, i)
        acc.add(int(c[0]), c[1], c[2], c[3])
    serial = acc.stats(False)
    assert out[0] == out[1]  # identical on every rank
    assert out[0] == (serial.mean, serial.max, serial.stddev, serial.count)
    assert serial.count == dom.count


def test_shard_range_covers_exactly_once():
    from paper_2003_02633_b200.analysis import shard_range

    for n in (0, 1, 7, 8, 1000, 2 ** 28 + 3):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b


def test_sample_domain_matches_reference_generator(golden):
    from paper_2003_02633_b200.analysis import SampleDomain, sample

    assert np.array_equal(sample(SampleDomain("unit_sphere", 5_000, 71)), golden["vec_sphere"])
    assert np.array_equal(sample(SampleDomain("cube", 5_000, 5)), golden["vec_cube"])


@pytest.mark.parametrize("kind", ["unit_sphere", "sphere_angles", "cube", "shell"])
def test_sample_domain_shapes(kind):
    from paper_2003_02633_b200.analysis import SampleDomain, sample

    v = sample(SampleDomain(kind, (1 << 20) + 17, 9, r_min=0.5, r_max=2.0))
    assert v.shape == ((1 << 20) + 17, 3) and v.dtype == np.float32
