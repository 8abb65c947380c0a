"""Dendrogram text format v1 (write_dendrogram, dendro_io.py:28-38): the
oracle's bytes equal the reference writer's (when the reference is
importable, i.e. in the development container), and the device formatter's
bytes equal the oracle's on the golden corpus and synthetic trees."""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np
import pytest

from oracle import dendro_oracle as O
from paper_2401_06089_b200 import synth
from tests.conftest import golden_trees, has_gpu

GOLDEN = list(golden_trees())[:20]


def _reference_writer():
    src = os.environ.get("DENDROMST_SRC", "/root/reference/pkg/src")
    if not os.path.isdir(src):
        return None
    if src not in sys.path:
        sys.path.insert(0, src)
    try:
        from dendromst.dendro_io import write_dendrogram
        from dendromst.expansion import Dendrogram
    except Exception:
        return None
    return write_dendrogram, Dendrogram


@pytest.mark.parametrize("t", GOLDEN, ids=[t["name"] for t in GOLDEN])
def test_oracle_text_matches_reference_writer(t):
    ref = _reference_writer()
    if ref is None:
        pytest.skip("reference package not importable here")
    write_dendrogram, Dendrogram = ref
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.dendro")
        write_dendrogram(path, Dendrogram(np.asarray(t["edge_parent"], np.int64),
                                          np.asarray(t["vertex_parent"], np.int64)))
        assert open(path, "rb").read() == O.dendrogram_text(t["edge_parent"], t["vertex_parent"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("t", GOLDEN, ids=[t["name"] for t in GOLDEN])
def test_device_text_matches_oracle_golden(t):
    from paper_2401_06089_b200 import format_dendrogram_b200
    got = format_dendrogram_b200(t["edge_parent"], t["vertex_parent"]).cpu().numpy().tobytes()
    assert got == O.dendrogram_text(t["edge_parent"], t["vertex_parent"])


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("shape,n", [("random", 1), ("random", 2047), ("tied", 2048), ("path", 100_000),
                                     ("random", 300_000)])
def test_device_file_matches_oracle(shape, n):
    from paper_2401_06089_b200 import DendrogramBuilder, write_dendrogram_b200
    nv, u, v, w = synth.GENERATORS[shape](n, seed=n)
    r = DendrogramBuilder("cuda:0").build(nv, u, v, w)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.dendro")
        size = write_dendrogram_b200(path, r.edge_parent, r.vertex_parent)
        data = open(path, "rb").read()
    exp = O.dendrogram_text(r.edge_parent.cpu().numpy(), r.vertex_parent.cpu().numpy())
    assert size == len(data) and data == exp


def _write(path, data: bytes):
    with open(path, "wb") as f:
        f.write(data)


def _variants(t):
    """(name, file a, file b): identical, one edge changed, one vertex changed,
    different sizes, and comment / blank lines."""
    base = O.dendrogram_text(t["edge_parent"], t["vertex_parent"])
    ep = np.asarray(t["edge_parent"], np.int64).copy()
    vp = np.asarray(t["vertex_parent"], np.int64).copy()
    out = [("same", base, base)]
    if ep.shape[0] > 1:
        e2 = ep.copy()
        e2[-1] = e2[-1] - 1 if e2[-1] > 0 else 0
        out.append(("edge_diff", base, O.dendrogram_text(e2, vp)))
    v2 = vp.copy()
    v2[0] = -1
    out.append(("vertex_diff", base, O.dendrogram_text(ep, v2)))
    out.append(("size", base, O.dendrogram_text(ep[:-1], vp)))
    lines = base.split(b"\n")
    commented = b"\n".join(lines[:1] + [b"# a comment", b""] + lines[1:])
    out.append(("comments", base, commented))
    return out


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("t", GOLDEN[:6], ids=[t["name"] for t in GOLDEN[:6]])
def test_device_verify_matches_oracle(t):
    from paper_2401_06089_b200 import verify_b200
    with tempfile.TemporaryDirectory() as d:
        for name, a, b in _variants(t):
            pa, pb = os.path.join(d, "a"), os.path.join(d, "b")
            _write(pa, a)
            _write(pb, b)
            assert verify_b200(pa, pb) == O.verify_text(a, b), name


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_read_roundtrip_and_errors():
    from paper_2401_06089_b200 import DendrogramBuilder, read_dendrogram_b200, write_dendrogram_b200
    from paper_2401_06089_b200.api import _format_error
    nv, u, v, w = synth.GENERATORS["random"](500_000, seed=4)
    r = DendrogramBuilder("cuda:0").build(nv, u, v, w)
    err = _format_error()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.dendro")
        write_dendrogram_b200(path, r.edge_parent, r.vertex_parent)
        back = read_dendrogram_b200(path)
        assert bool((back.edge_parent == r.edge_parent).all()) and bool((back.vertex_parent == r.vertex_parent).all())
        data = open(path, "rb").read()
        bad = data.replace(b"\nE 7 ", b"\nX 7 ", 1)
        _write(path, bad)
        with pytest.raises(err, match="bad line: 'X 7 "):
            read_dendrogram_b200(path)
        _write(path, b"#dendrogram v2 n=1 nv=2\n")
        with pytest.raises(err, match="bad header"):
            read_dendrogram_b200(path)
        _write(path, data[: data.rfind(b"\nV ") + 1])
        with pytest.raises(err, match=f"expected {nv - 1} edge and {nv} vertex lines, got {nv - 1} and {nv - 1}"):
            read_dendrogram_b200(path)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_sidecar_roundtrip():
    from paper_2401_06089_b200 import DendrogramBuilder, read_dendrogram_b200, write_dendrogram_b200
    from paper_2401_06089_b200.api import sidecar_path
    nv, u, v, w = synth.GENERATORS["random"](200_000, seed=5)
    r = DendrogramBuilder("cuda:0").build(nv, u, v, w)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.dendro")
        write_dendrogram_b200(path, r.edge_parent, r.vertex_parent, sidecar=True)
        side = np.load(sidecar_path(path))
        assert side.dtype == np.int32 and side.shape == (2 * nv - 1 + 8,)
        for use in (True, False):
            back = read_dendrogram_b200(path, use_sidecar=use)
            assert bool((back.edge_parent == r.edge_parent).all())
            assert bool((back.vertex_parent == r.vertex_parent).all())
        # the same-size text rewritten at once (same mtime tick possible) is parsed, not shadowed
        data = open(path, "rb").read()
        i = data.index(b"\nE 5 ") + 1
        j = data.index(b"\n", i)
        edited = data[:i] + (b"E 5 -1" + b" " * 0) + data[j:]
        _write(path, edited)
        back = read_dendrogram_b200(path)
        assert int(back.edge_parent[5]) == -1
        # writing without a sidecar removes the stale one
        write_dendrogram_b200(path, r.edge_parent, r.vertex_parent, sidecar=False)
        assert not os.path.exists(sidecar_path(path))


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_reader_duplicate_ids_last_wins():
    # read_dendrogram assigns lines in order (dendro_io.py:60-66): a repeated id keeps the LAST parent
    from paper_2401_06089_b200 import read_dendrogram_b200
    body = b"#dendrogram v1 n=3 nv=4\nE 0 -1\nE 1 0\nE 1 7\nE 2 0\nE 1 0\nV 0 2\nV 1 2\nV 2 1\nV 3 1\n"
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "dup.dendro")
        _write(path, body)
        err = __import__("paper_2401_06089_b200.api", fromlist=["x"])._format_error()
        with pytest.raises(err, match="expected 3 edge and 4 vertex lines, got 5 and 4"):
            read_dendrogram_b200(path)
        _write(path, b"#dendrogram v1 n=3 nv=4\nE 0 -1\nE 1 2\nE 1 0\nV 0 2\nV 1 2\nV 2 1\nV 3 1\nV 3 0\n")
        with pytest.raises(err, match="got 3 and 5"):
            read_dendrogram_b200(path)
        # duplicates that still add up: 2 E lines for id 1, none for id 2 -> id 2 stays ROOT, id 1 = last
        _write(path, b"#dendrogram v1 n=3 nv=4\nE 0 -1\nE 1 2\nE 1 0\nV 0 2\nV 1 2\nV 2 1\nV 3 1\n")
        for _ in range(20):  # the same answer every run
            r = read_dendrogram_b200(path)
            assert r.edge_parent.cpu().tolist() == [-1, 0, -1]


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_height_rejects_non_dendrogram_parents():
    import torch
    from paper_2401_06089_b200 import dendrogram_height_b200
    assert dendrogram_height_b200(torch.tensor([-1, 0, 0, 1], dtype=torch.int32)) == 3
    for bad in ([-1, 5, 0], [-1, 2, 0], [-1, -7, 0], [0, -1, 1]):
        with pytest.raises(ValueError, match="heavier edge"):
            dendrogram_height_b200(torch.tensor(bad, dtype=torch.int32))


@pytest.mark.parametrize("t", GOLDEN[:6], ids=[t["name"] for t in GOLDEN[:6]])
def test_oracle_verify_matches_reference_cli(t, capsys):
    """O.verify_text (the checker of verify_b200) against the reference's own
    `dendromst verify` (cli.py:138-155) on the same file pairs."""
    if _reference_writer() is None:
        pytest.skip("reference package not importable here")
    import argparse
    from dendromst.cli import _cmd_verify
    with tempfile.TemporaryDirectory() as d:
        for name, a, b in _variants(t):
            pa, pb = os.path.join(d, "a"), os.path.join(d, "b")
            _write(pa, a)
            _write(pb, b)
            capsys.readouterr()
            rc = _cmd_verify(argparse.Namespace(a=pa, b=pb))
            line = capsys.readouterr().out.strip()
            assert (rc, line) == O.verify_text(a, b), name


def test_reader_messages_match_reference(tmp_path):
    """The reader's header / line / count errors, as read_dendrogram
    (dendro_io.py:41-75) words them (checked on the reference itself)."""
    if _reference_writer() is None:
        pytest.skip("reference package not importable here")
    from dendromst.dendro_io import DendrogramFormatError, read_dendrogram
    cases = {
        "header": b"#dendrogram v2 n=1 nv=2\n",
        "line": b"#dendrogram v1 n=1 nv=2\nE 0 -1\nX 1 0\n",
        "count": b"#dendrogram v1 n=1 nv=2\nE 0 -1\nV 0 0\n",
    }
    expect = {"header": "bad header: '#dendrogram v2 n=1 nv=2'", "line": "bad line: 'X 1 0'",
              "count": "expected 1 edge and 2 vertex lines, got 1 and 1"}
    for name, data in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(DendrogramFormatError) as ei:
            read_dendrogram(str(p))
        assert str(ei.value) == expect[name], name


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_device_reader_messages(tmp_path):
    """read_dendrogram_b200 raises the reference's exact messages (the strings
    test_reader_messages_match_reference pins on the reference)."""
    from paper_2401_06089_b200 import read_dendrogram_b200
    from paper_2401_06089_b200.api import _format_error
    cases = {
        "header": (b"#dendrogram v2 n=1 nv=2\n", "bad header: '#dendrogram v2 n=1 nv=2'"),
        "line": (b"#dendrogram v1 n=1 nv=2\nE 0 -1\nX 1 0\n", "bad line: 'X 1 0'"),
        "count": (b"#dendrogram v1 n=1 nv=2\nE 0 -1\nV 0 0\n", "expected 1 edge and 2 vertex lines, got 1 and 1"),
    }
    for name, (data, msg) in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        with pytest.raises(_format_error()) as ei:
            read_dendrogram_b200(str(p))
        assert str(ei.value) == msg, name
    p = tmp_path / "ok"
    p.write_bytes(b"#dendrogram v1 n=1 nv=2\n# comment\n\nE 0 -1\nV 0 0\nV 1 0\n")
    r = read_dendrogram_b200(str(p))
    assert r.edge_parent.tolist() == [-1] and r.vertex_parent.tolist() == [0, 0]
