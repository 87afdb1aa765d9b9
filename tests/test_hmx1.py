"""HMX1 operator files: the native reader/writer against a file the
reference ``save_hmatrix`` wrote (tests/golden/make_hmx1.py) and against the oracle's
restatement of the format (``hmatrix.py:9-24``, ``:334-388``).  Host-side only (no GPU)."""

import os
import struct

import numpy as np
import pytest

from oracle import hmat_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "hmx1_ops300.hmx")


@pytest.fixture(scope="module")
def case():
    import paper_1805_08998_b200 as hx
    g = np.load(os.path.join(HERE, "golden", "hmx1_ops300.npz"))
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(g["n_min"])),
                                      float(g["eta"]))
    obt = O.BlockTreeO(O.ClusterTreeO(pts, int(g["n_min"])), float(g["eta"]))
    return hx, g, bct, obt


def test_fingerprint_matches_reference(case):
    hx, g, bct, obt = case
    assert hx.tree_fingerprint(bct) == g["fingerprint"].tobytes()
    assert O.fingerprint_o(obt) == g["fingerprint"].tobytes()


def test_oracle_reads_reference_file(case):
    hx, g, bct, obt = case
    H = O.load_hmatrix_o(GOLD, obt)
    assert sorted(H.data) == sorted(g["ids"].tolist())
    for b, kind, r in zip(g["ids"], g["kinds"], g["ranks"]):
        p = H.data[int(b)]
        assert isinstance(p, O.LR) == (kind == 1)
        if kind == 1:
            assert p.rank == r
    assert H.degraded == set(g["degraded"].tolist())


def test_native_load_matches_oracle(case):
    hx, g, bct, obt = case
    ref = O.load_hmatrix_o(GOLD, obt)
    H = hx.load_hmatrix(GOLD, bct)
    assert H.degraded == ref.degraded
    assert sorted(H.data.keys()) == sorted(ref.data)
    for b, p in ref.data.items():
        q = H.data[b]
        if isinstance(p, O.LR):
            assert isinstance(q, hx.LowRank)
            assert np.array_equal(q.left, p.left) and np.array_equal(q.right, p.right)
        else:
            assert not isinstance(q, hx.LowRank)
            assert np.array_equal(q, p)
    # the packed pool is in panel order, ready for the device
    pool, d = H._hx_packed
    assert pool.dtype == np.float64 and d["payload"][int(g["degraded"][0])] == 2


def test_native_roundtrip_is_byte_identical(case, tmp_path):
    hx, g, bct, obt = case
    H = hx.load_hmatrix(GOLD, bct)
    out = tmp_path / "again.hmx"
    hx.save_hmatrix(H, str(out))
    assert out.read_bytes() == open(GOLD, "rb").read()
    # a host-built operand (no packed pool yet) writes the same bytes
    ref = O.load_hmatrix_o(GOLD, obt)
    data = {b: (hx.LowRank(p.left, p.right) if isinstance(p, O.LR) else p)
            for b, p in ref.data.items()}
    H2 = hx.HMatrix(bct, data, ref.degraded)
    out2 = tmp_path / "host.hmx"
    hx.save_hmatrix(H2, str(out2))
    assert out2.read_bytes() == open(GOLD, "rb").read()


def test_oracle_writer_matches_reference_file(case, tmp_path):
    hx, g, bct, obt = case
    out = tmp_path / "o.hmx"
    O.save_hmatrix_o(O.load_hmatrix_o(GOLD, obt), str(out))
    assert out.read_bytes() == open(GOLD, "rb").read()


def _patched(tmp_path, offset, payload):
    raw = bytearray(open(GOLD, "rb").read())
    raw[offset:offset + len(payload)] = payload
    p = tmp_path / f"bad{offset}.hmx"
    p.write_bytes(bytes(raw))
    return str(p)


def test_header_errors_follow_reference(case, tmp_path):
    hx, g, bct, obt = case
    cases = [
        (_patched(tmp_path, 0, b"HMX2"), "not an H-matrix file"),
        (_patched(tmp_path, 4, struct.pack("<I", 2)), "unsupported version 2"),
        (_patched(tmp_path, 8, struct.pack("<Q", 301)), "dimension mismatch: file 301, tree 300"),
        (_patched(tmp_path, 16, b"\0" * 32), "block tree does not match the stored operator"),
    ]
    for path, msg in cases:
        with pytest.raises(ValueError, match=msg):
            O.load_hmatrix_o(path, obt)
        with pytest.raises(ValueError, match=msg):
            hx.load_hmatrix(path, bct)
    with pytest.raises(FileNotFoundError):
        hx.load_hmatrix(str(tmp_path / "missing.hmx"), bct)


def test_truncated_and_foreign_records_rejected(case, tmp_path):
    hx, g, bct, obt = case
    raw = open(GOLD, "rb").read()
    p = tmp_path / "short.hmx"
    p.write_bytes(raw[:len(raw) - 100])
    with pytest.raises(ValueError, match="truncated"):
        hx.load_hmatrix(str(p), bct)
    # first record's node id replaced by an inner node
    inner = int(np.flatnonzero(bct.kind_code == 0)[0])
    bad = _patched(tmp_path, 56, struct.pack("<Q", inner))
    with pytest.raises(ValueError, match="not a leaf"):
        hx.load_hmatrix(bad, bct)
