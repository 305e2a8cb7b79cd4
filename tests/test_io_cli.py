"""On-disk formats and CLI (reference io.py / cli.py compatibility)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2412_04980_b200 as hdb
from paper_2412_04980_b200 import io as hio
from gold import GOLDEN, ROOT

CFG = "problem = mp1b\nwavenumber = 50\nnx = 129\nlevels = 2\nlevel2.cycle_tol = 0.3\n"


def test_config_render_matches_reference_and_round_trips():
    cfg = hio.parse_config(CFG)
    with open(os.path.join(GOLDEN, "ref_config_render.txt")) as fh:
        assert hio.render_config(cfg) == fh.read()
    assert hio.parse_config(hio.render_config(cfg)) == cfg


@pytest.mark.parametrize("text,msg", [("problem = nope\nwavenumber=1\nnx=9", "unknown problem"),
                                      ("problem = mp1b\nnx = 9", "exactly one of freq_hz"),
                                      ("problem = mp1b\nwavenumber = 1\nnx = 9\nnx = 9", "duplicate"),
                                      ("problem = mp1b\nwavenumber = 1\nnx = 9\nlevel9.cycle_tol = 1", "outside"),
                                      ("problem = mp1b\nwavenumber = 1\nnx = x", "line 3")])
def test_config_errors(text, msg):
    with pytest.raises(hdb.ConfigError, match=msg):
        hio.parse_config(text)


def test_reference_field_file_reads_back_bit_exact(tmp_path):
    fld = hio.read_field(os.path.join(GOLDEN, "ref_field_9.csv"))
    hier = hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy
    z = np.random.default_rng(4).standard_normal(81) + 1j * np.random.default_rng(5).standard_normal(81)
    np.testing.assert_array_equal(fld.data, z)
    p = tmp_path / "f.csv"
    hio.write_field(fld, hier, str(p))
    assert p.read_text() == open(os.path.join(GOLDEN, "ref_field_9.csv")).read()


def test_velocity_raster_round_trip(tmp_path):
    vm = hdb.synthetic_layered_velocity(3, dx=96.0)
    p = tmp_path / "v.txt"
    hio.write_velocity_grid(vm, str(p))
    back = hio.read_velocity_grid(str(p))
    np.testing.assert_array_equal(back.values, vm.values)
    assert (back.dx, back.dy, back.x0, back.y0) == (vm.dx, vm.dy, vm.x0, vm.y0)


def test_stencils_cli_verifies_chain():
    r = subprocess.run([sys.executable, "-m", "paper_2412_04980_b200", "stencils", "--verify"], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.count(": ok") == 10


@pytest.mark.gpu
def test_solve_cli_report_matches_reference(tmp_path):
    cfgp = tmp_path / "c.cfg"
    cfgp.write_text(CFG)
    r = subprocess.run([sys.executable, "-m", "paper_2412_04980_b200", "solve", "--config", str(cfgp), "--out",
                        str(tmp_path)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    mine = (tmp_path / "mp1b_report.csv").read_text().splitlines()
    ref = open(os.path.join(GOLDEN, "ref_report_c1s.csv")).read().splitlines()
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        if a.startswith("# wall_ms") or a.startswith("# model_"):
            continue
        if a.startswith("# final_relres"):  # a float printed to 17 digits: compare as numbers
            assert abs(float(a.split("=")[1]) - float(b.split("=")[1])) <= 1e-9
            continue
        if a[0].isdigit():  # outer_iter,relres,wall_ms
            ia, ra, _ = a.split(",")
            ib, rb, _ = b.split(",")
            assert ia == ib and abs(float(ra) - float(rb)) <= 1e-9
        else:
            assert a == b
