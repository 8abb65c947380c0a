"""The reference's own plugin boundary, driven end to end on the GPU.

The unmodified reference package (baseline/_ref, see tests/conftest.py
reference_package) gets `pandora_b200` registered into its algorithm
registry `_ALGOS` (cli.py:27-31) by `register_algorithm`, and then its own
CLI entry point `dendromst.cli.main` runs:
  build --algo pandora_b200   (_cmd_build, cli.py:71-94: rank_edges + the
                               registered constructor, then write_dendrogram)
  build --algo pandora        (the reference's CPU path, same input file)
  verify --a ... --b ...      (_cmd_verify, cli.py:138-155) -> "identical"
  bench --algo pandora_b200   (_cmd_bench, cli.py:158-179)
on the config-1 input (100k random tree) and the config-2 input (the
reference's 1M-point mutual-reachability MST), plus the registry call
itself on the reference's own fixtures.  The device-side verify_b200 must
agree with the reference's verify on the same two files.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2401_06089_b200 import synth
from tests.conftest import has_gpu, make_tree, reference_package

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def ref():
    R = reference_package()
    if R is None:
        pytest.skip("reference package not installed in baseline/_ref")
    from paper_2401_06089_b200 import register_algorithm
    from paper_2401_06089_b200.build import build
    build()
    register_algorithm()            # into dendromst.cli._ALGOS
    return R


def _write_edges(R, path, nv, u, v, w):
    tree = R.WeightedTree(int(nv), np.asarray(u, np.int64), np.asarray(v, np.int64), np.asarray(w, np.float64),
                          np.arange(len(u), dtype=np.int64))
    from dendromst.dendro_io import write_edge_list
    write_edge_list(path, tree)


@pytest.mark.parametrize("cfg", ["config1", "config2"])
def test_cli_build_verify_bench(ref, cfg, tmp_path, capsys):
    from dendromst import cli
    from paper_2401_06089_b200 import verify_b200
    assert "pandora_b200" in cli._ALGOS
    nv, u, v, w = synth.random_attach(100_000, seed=0) if cfg == "config1" else synth.blobs1m()
    edges = str(tmp_path / "tree.txt")
    _write_edges(ref, edges, nv, u, v, w)
    a, b = str(tmp_path / "gpu.dendro"), str(tmp_path / "cpu.dendro")
    assert cli.main(["build", "--input", edges, "--algo", "pandora_b200", "--output", a]) == 0
    out = capsys.readouterr().out
    assert "algo=pandora_b200" in out and "wall_time_s=" in out
    assert cli.main(["build", "--input", edges, "--algo", "pandora", "--output", b]) == 0
    capsys.readouterr()
    assert cli.main(["verify", "--a", a, "--b", b]) == 0
    assert capsys.readouterr().out.strip() == "identical"
    assert open(a, "rb").read() == open(b, "rb").read()
    assert verify_b200(a, b) == (0, "identical")
    assert cli.main(["bench", "--input", edges, "--algo", "pandora_b200", "--repeat", "2"]) == 0
    assert "algo=pandora_b200 threads=1 repeat=2" in capsys.readouterr().out


def test_cli_verify_reports_divergence(ref, tmp_path, capsys):
    # the registered algorithm's file vs an edited copy: the reference's verify and
    # verify_b200 report the same first divergence (cli.py:148-153)
    from dendromst import cli
    from paper_2401_06089_b200 import verify_b200
    nv, u, v, w = synth.random_attach(5000, seed=2, tied=True)
    edges = str(tmp_path / "t.txt")
    _write_edges(ref, edges, nv, u, v, w)
    a, b = str(tmp_path / "a.dendro"), str(tmp_path / "b.dendro")
    assert cli.main(["build", "--input", edges, "--algo", "pandora_b200", "--output", a]) == 0
    data = open(a, "rb").read()
    i = data.index(b"\nE 17 ") + 1
    j = data.index(b"\n", i)
    open(b, "wb").write(data[:i] + b"E 17 3" + data[j:])
    capsys.readouterr()
    assert cli.main(["verify", "--a", a, "--b", b]) == 1
    line = capsys.readouterr().out.strip()
    assert verify_b200(a, b) == (1, line)


def test_registry_call_on_reference_fixtures(ref):
    # _ALGOS["pandora_b200"](ranked) == _ALGOS["pandora"](ranked) on the reference's
    # own generator shapes (tests/conftest.py:15-82), the reference's Dendrogram equality
    from dendromst import cli
    rng = np.random.default_rng(123)
    for topo in ("star", "path", "caterpillar", "attach"):
        for nv in (2, 3, 50, 2000):
            for equal in (False, True):
                nv2, u, v, w = make_tree(topo, nv, rng, equal)
                ranked = ref.rank_edges(ref.weighted_tree(nv2, u, v, w))
                got = cli._ALGOS["pandora_b200"](ranked)
                assert type(got) is type(cli._ALGOS["pandora"](ranked))
                assert got == cli._ALGOS["pandora"](ranked)
