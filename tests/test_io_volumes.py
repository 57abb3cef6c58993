"""Detached-header raw volumes (io.hpp:57-202, 337-428) through the C ABI's
host I/O entry points: the reference suite's io cases (test_io.cpp:44-183)
restated, plus uint16 (config 3) and the plane-range reader that a z-slab
rank uses. Host code only (no device needed), except the device-ingest test."""
import os
import struct

import numpy as np
import pytest


@pytest.fixture(scope="module")
def s():
    import paper_1806_08741_b200 as m
    try:
        m.lib()
    except ImportError as e:
        pytest.skip(str(e))
    return m


def test_detached_header_decodes_payload(s, tmp_path):
    (tmp_path / "direct.raw").write_bytes(b"".join(struct.pack("<f", 0.5 * i) for i in range(12)))
    (tmp_path / "direct.hdr").write_text("dimension: 2\nsizes: 4 3\nchannels: 1\ntype: float32\n"
                                         "endian: little\ndata file: direct.raw\n")
    img = s.read_volume(tmp_path / "direct.hdr")
    assert img.dims == (4, 3) and img.channels == 1
    assert list(img.data.astype(np.float64)) == [0.5 * i for i in range(12)]


@pytest.mark.parametrize("dt", [np.uint8, np.uint16, np.float32])
def test_round_trip_and_byte_stability(s, tmp_path, dt):
    rng = np.random.default_rng(55)
    for trial in range(6):
        rank = int(rng.integers(1, 5))
        ch = int(rng.integers(1, 4))
        dims = tuple(int(x) for x in rng.integers(1, 7, size=rank))
        n = int(np.prod(dims)) * ch
        data = (rng.integers(0, 256, n) if dt != np.float32 else rng.random(n)).astype(dt)
        s.write_volume(tmp_path / "rt.hdr", s.NDImage(dims, ch, data))
        back = s.read_volume(tmp_path / "rt.hdr")
        assert back.dims == dims and back.channels == ch
        assert back.data.dtype == dt and np.array_equal(back.data, data)
        payload = (tmp_path / "rt.raw").read_bytes()
        s.write_volume(tmp_path / "rt2.hdr", back)
        assert (tmp_path / "rt2.raw").read_bytes() == payload
        # a z-slab rank reads only its planes
        if dims[-1] > 1:
            lo, hi = 1, dims[-1]
            plane = int(np.prod(dims[:-1])) * ch
            part = np.empty((hi - lo) * plane, dt)
            s.read_volume_planes(tmp_path / "rt.hdr", lo, hi, part.ctypes.data, device=-1)
            assert np.array_equal(part, data[lo * plane: hi * plane])


def test_reader_error_kinds(s, tmp_path):
    def code(path):
        with pytest.raises(s.IoError) as e:
            s.read_volume(path)
        return e.value.code
    assert code(tmp_path / "absent.hdr") == "file_not_found"
    (tmp_path / "broken.hdr").write_text("sizes: 4 3\ntype: float32\n")
    assert code(tmp_path / "broken.hdr") == "malformed_header"
    (tmp_path / "nan.hdr").write_text("dimension: two\nsizes: 4\nchannels: 1\ntype: float32\n"
                                      "data file: x.raw\n")
    assert code(tmp_path / "nan.hdr") == "malformed_header"
    (tmp_path / "badtype.hdr").write_text("dimension: 1\nsizes: 4\nchannels: 1\ntype: float64\n"
                                          "data file: x.raw\n")
    assert code(tmp_path / "badtype.hdr") == "unsupported_type"
    (tmp_path / "short.raw").write_bytes(b"abc")
    (tmp_path / "short.hdr").write_text("dimension: 1\nsizes: 4\nchannels: 1\ntype: float32\n"
                                        "data file: short.raw\n")
    assert code(tmp_path / "short.hdr") == "size_mismatch"
    (tmp_path / "big.hdr").write_text("dimension: 1\nsizes: 4\nchannels: 1\ntype: uint8\n"
                                      "endian: big\ndata file: short.raw\n")
    assert code(tmp_path / "big.hdr") == "unsupported_type"
    assert code(tmp_path / "x.png") == "unsupported_type"  # no libpng in this build


def test_label_maps_round_trip_with_count(s, tmp_path):
    s.write_labels(tmp_path / "labels.hdr", np.array([0, 1, 1], np.uint32), (3,))
    assert (tmp_path / "labels.raw").read_bytes() == bytes([0, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0])
    back, dims = s.read_labels(tmp_path / "labels.hdr")
    assert dims == (3,) and list(back) == [0, 1, 1]
    assert "label count: 2" in (tmp_path / "labels.hdr").read_text()
    with pytest.raises(s.IoError) as e:
        s.read_volume(tmp_path / "labels.hdr")
    assert e.value.code == "unsupported_type"


@pytest.mark.gpu
def test_volume_planes_stream_into_device(s, tmp_path):
    """The slab reader streams planes from disk through pinned staging into
    device memory in 64 MB chunks: the bytes equal the file's."""
    import torch
    rng = np.random.default_rng(9)
    dims, ch = (512, 384, 200), 1
    data = rng.integers(0, 65536, int(np.prod(dims)), dtype=np.uint16)
    s.write_volume(tmp_path / "v.hdr", s.NDImage(dims, ch, data))
    lo, hi = 37, 199
    plane = dims[0] * dims[1]
    dev = torch.empty((hi - lo) * plane, dtype=torch.int16, device="cuda")
    s.read_volume_planes(tmp_path / "v.hdr", lo, hi, dev.data_ptr(), device=0)
    assert np.array_equal(dev.cpu().numpy().view(np.uint16), data[lo * plane: hi * plane])
