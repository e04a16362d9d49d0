"""CPU: the drop-in's file formats against the reference's own readers and
writers (graph.cpp:461-484, 553-628; vip.cpp:107-134): files written by one
side are read back identically by the other, and malformed files raise the
same error types."""
import os

import numpy as np
import pytest

from paper_2305_03152_b200 import vipkit as vk


def _write(path, text):
    with open(path, "w") as f:
        f.write(text)


def test_partition_labels_both_ways(ref, tmp_path):
    rng = np.random.default_rng(1)
    labels = rng.integers(0, 5, 3000).astype(np.uint32)
    labels[:5] = np.arange(5)
    a, b = str(tmp_path / "ref.txt"), str(tmp_path / "vk.txt")
    ref.write_partition_labels(labels, 5, a)
    vk.write_partition_labels(labels, b)
    assert open(a).read() == open(b).read()
    for path in (a, b):
        for K in (0, 5, 7):
            if K == 7:  # partitions 5, 6 empty
                with pytest.raises(vk.PartitionError):
                    vk.partition_from_file(path, K, len(labels))
                with pytest.raises(Exception, match="partition_error"):
                    ref.partition_from_file(path, K, len(labels))
                continue
            got, k1 = vk.partition_from_file(path, K, len(labels))
            exp, k2 = ref.partition_from_file(path, K, len(labels))
            np.testing.assert_array_equal(got, exp)
            assert k1 == k2 == 5


@pytest.mark.parametrize("text,n,K,kind", [
    ("0\n1\n# c\n\n1\n0x\n", 4, 0, None),           # comments, blanks, trailing chars ignored
    ("0\r\n1\r\n", 2, 2, None),                      # CRLF: leading digits parse
    ("0\n1\n", 3, 0, "FormatError"),                 # wrong count
    ("0\n-1\n", 2, 0, "FormatError"),                # sign
    ("0\n 1\n", 2, 0, "FormatError"),                # leading blank
    ("0\n99999999999\n", 2, 0, "FormatError"),       # overflow
    ("0\n3\n", 2, 2, "FormatError"),                 # label >= K
    ("0\n0\n", 2, 2, "PartitionError"),              # empty partition 1
])
def test_partition_file_edge_cases(ref, tmp_path, text, n, K, kind):
    p = str(tmp_path / "l.txt")
    _write(p, text)
    if kind is None:
        got, k1 = vk.partition_from_file(p, K, n)
        exp, k2 = ref.partition_from_file(p, K, n)
        np.testing.assert_array_equal(got, exp)
        assert k1 == k2
    else:
        with pytest.raises(getattr(vk, kind)):
            vk.partition_from_file(p, K, n)
        name = {"FormatError": "format_error", "PartitionError": "partition_error"}[kind]
        with pytest.raises(Exception, match=name):
            ref.partition_from_file(p, K, n)


def test_missing_files_are_io_errors(ref, tmp_path):
    p = str(tmp_path / "nope")
    with pytest.raises(vk.IOError_):
        vk.partition_from_file(p, 0, 1)
    with pytest.raises(vk.IOError_):
        vk.load_roles(p)
    with pytest.raises(vk.IOError_):
        vk.load_vip_binary(p)
    with pytest.raises(Exception, match="io_error"):
        ref.load_roles(p)


def test_roles_both_ways(ref, tmp_path):
    roles = np.random.default_rng(2).integers(0, 4, 5000).astype(np.uint8)
    a, b = str(tmp_path / "ref.txt"), str(tmp_path / "vk.txt")
    ref.write_roles(roles, a)
    vk.write_roles(roles, b)
    assert open(a).read() == open(b).read()
    np.testing.assert_array_equal(vk.load_roles(a), roles)
    np.testing.assert_array_equal(ref.load_roles(b), roles)
    _write(a, "0\n# x\n\n3\n2z\n")
    np.testing.assert_array_equal(vk.load_roles(a), ref.load_roles(a))
    _write(a, "0\n4\n")
    with pytest.raises(vk.FormatError):
        vk.load_roles(a)
    with pytest.raises(Exception, match="format_error"):
        ref.load_roles(a)


def test_vip_binary_both_ways(ref, tmp_path):
    x = np.random.default_rng(3).random(7777)
    x[:4] = [0.0, 1.0, 5e-324, np.nextafter(1.0, 0.0)]
    a, b = str(tmp_path / "ref.bin"), str(tmp_path / "vk.bin")
    ref.write_vip_binary(x, a)
    vk.write_vip_binary(x, b)
    assert open(a, "rb").read() == open(b, "rb").read()
    np.testing.assert_array_equal(vk.load_vip_binary(a), x)
    np.testing.assert_array_equal(ref.load_vip_binary(b), x)
    with open(a, "ab") as f:  # a trailing partial record is ignored by both
        f.write(b"\x01\x02\x03")
    np.testing.assert_array_equal(vk.load_vip_binary(a), ref.load_vip_binary(a))


def test_vcsr_writer_matches_reference(ref, port, tmp_path):
    csr = port.generate("pa", 3000, 5, 11)
    a, b = str(tmp_path / "ref.vcsr"), str(tmp_path / "vk.vcsr")
    ref.write_vcsr(csr, a)
    vk.write_binary_csr(csr.off, csr.tgt, b)
    assert open(a, "rb").read() == open(b, "rb").read()
    g = ref.load_vcsr(b)
    np.testing.assert_array_equal(g.off, csr.off)
    np.testing.assert_array_equal(g.tgt, csr.tgt)


def test_vip_storage_width_api():
    with pytest.raises(vk.ParameterError):
        vk.vip_force_storage(16)
    vk.vip_force_storage(32)
    vk.vip_force_storage(0)
