"""VC3C stream format and raw vector IO (mirrors pkg/tests/test_stream.py);
byte identity against streams written by the reference.  CPU only, except
the last test (GPU codec on the file path)."""

import io

import numpy as np
import pytest

from conftest import layout_by_name
from paper_2003_02633_b200 import BadLayout, BadMagic, BitLayout, DEFAULT_LAYOUT, TruncatedStream
from paper_2003_02633_b200.stream import (
    HEADER_SIZE,
    pack_header,
    parse_header,
    read_csv,
    read_f32,
    read_stream,
    write_csv,
    write_f32,
    write_stream,
)


def test_header_layout_and_round_trip():
    assert HEADER_SIZE == 20
    data = pack_header(DEFAULT_LAYOUT, 7)
    assert len(data) == 20 and data[:4] == b"VC3C"
    for lay in (DEFAULT_LAYOUT, BitLayout(1, 8, 23, 16, 16, 127)):
        assert parse_header(pack_header(lay, 12345)) == (lay, 12345)


def test_bad_magic_version_layout_truncation():
    data = bytearray(pack_header(DEFAULT_LAYOUT, 0))
    data[:4] = b"NOPE"
    with pytest.raises(BadMagic):
        parse_header(bytes(data))
    data = bytearray(pack_header(DEFAULT_LAYOUT, 0))
    data[4] = 9
    with pytest.raises(BadLayout):
        parse_header(bytes(data))
    data = bytearray(pack_header(DEFAULT_LAYOUT, 0))
    data[5] = 3
    with pytest.raises(BadLayout):
        parse_header(bytes(data))
    with pytest.raises(TruncatedStream):
        parse_header(b"VC3C")
    buf = io.BytesIO(pack_header(DEFAULT_LAYOUT, 3) + b"\0" * 16)
    with pytest.raises(TruncatedStream):
        read_stream(buf)


@pytest.mark.parametrize("lname", ["17_18", "base_16_16"])
def test_stream_bytes_identical_to_reference(golden, lname):
    words = golden[f"cw_{lname}_SSS_kat"]
    buf = io.BytesIO()
    write_stream(buf, words, layout_by_name(lname))
    assert buf.getvalue() == golden[f"stream_{lname}"].tobytes()
    back, lay = read_stream(io.BytesIO(buf.getvalue()))
    assert lay == layout_by_name(lname) and np.array_equal(back, words)


def test_f32_and_csv_io(golden, tmp_path):
    v = golden["vec_edge"]
    write_f32(tmp_path / "v.f32", v)
    assert np.array_equal(read_f32(tmp_path / "v.f32").view(np.uint32), v.view(np.uint32))
    s = io.StringIO()
    write_csv(s, v)
    assert s.getvalue().encode() == golden["csv_edge"].tobytes()
    assert np.array_equal(read_csv(io.StringIO(s.getvalue())).view(np.uint32), v.view(np.uint32))
    (tmp_path / "bad.f32").write_bytes(b"\0" * 13)
    with pytest.raises(TruncatedStream):
        read_f32(tmp_path / "bad.f32")
    with pytest.raises(TruncatedStream):
        read_csv(io.StringIO("1,2\n"))


@pytest.mark.gpu
def test_gpu_codec_on_file_path(golden, vc3b, oracle, cuda, tmp_path):
    from paper_2003_02633_b200.stream import compress_to_stream, decompress_stream

    from paper_2003_02633_b200 import ALL_SINGLE_POLICY

    want = golden["cw_17_18_SSS_mixed"]
    v = golden["vec_mixed"][: want.size]
    n = compress_to_stream(tmp_path / "m.vc3", v, policy=ALL_SINGLE_POLICY)
    assert n == v.shape[0] and (tmp_path / "m.vc3").stat().st_size == 20 + 8 * n
    words, lay = read_stream(tmp_path / "m.vc3")
    assert np.array_equal(words, want)
    out, lay2 = decompress_stream(tmp_path / "m.vc3")
    assert lay2 == DEFAULT_LAYOUT
    assert np.array_equal(out, oracle.decompress(words, DEFAULT_LAYOUT))


@pytest.mark.gpu
def test_gpu_stream_device_tensors(golden, oracle, cuda, tmp_path):
    """Device tensors on the file path: compress a CUDA tensor straight into a
    stream, read it back onto the GPU."""
    import torch

    from paper_2003_02633_b200 import ALL_SINGLE_POLICY
    from paper_2003_02633_b200.stream import compress_to_stream, decompress_stream

    want = golden["cw_17_18_SSS_mixed"]
    v = torch.from_numpy(golden["vec_mixed"][: want.size]).cuda()
    n = compress_to_stream(tmp_path / "d.vc3", v, policy=ALL_SINGLE_POLICY)
    words, _ = read_stream(tmp_path / "d.vc3")
    assert n == want.size and np.array_equal(words, want)
    out, lay = decompress_stream(tmp_path / "d.vc3", device="cuda")
    assert out.is_cuda and lay == DEFAULT_LAYOUT
    assert np.array_equal(out.cpu().numpy().view(np.uint32),
                          oracle.decompress(words, DEFAULT_LAYOUT).view(np.uint32))
